import json
import os
import subprocess
import sys
import warnings

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA product path)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _ensure_oracle_built():
    lib = os.path.join(REPO, "oracle", "liboracle.so")
    src = os.path.join(REPO, "oracle", "heoracle.c")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)


_ensure_oracle_built()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def s128():
    return dict(np.load(os.path.join(GOLDEN_DIR, "s128.npz")))


S128 = dict(m=256, modulus_bits=260, precision_bits=30, seed=42, extra=25)


def s128_params():
    from paper_2102_00319_b200.params import derive_params

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return derive_params(S128["m"], S128["modulus_bits"], S128["precision_bits"], seed=S128["seed"])


@pytest.fixture(scope="session")
def oracle_s128():
    from oracle.ckks_oracle import OracleBackend

    be = OracleBackend(s128_params(), S128["extra"])
    keys = be.keygen(galois_steps=(1,))
    be.set_eval_key(keys)
    return be, keys


@pytest.fixture(autouse=True)
def _quiet():
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        yield


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
