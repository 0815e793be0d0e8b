"""The reference's OWN test suite, run against the B200 backend.

``hecnn_plugin`` subclasses the reference's plugin contract
(`hecnn.backends.base.HEBackend`) with the device hooks and, under
``HECNN_CKKS_IMPL=b200``, stands in for ``get_backend("ckks", ...)``.  The reference
tests that exercise the backend contract, the ref-vs-ckks agreement, the executor's
thread plans and the pipeline invariants then run unmodified from the reference install
(``baseline/_ref``, see tools/install_reference.sh): every ``"ckks"`` backend they build
is the device backend.

Tests that reach into the reference CKKS implementation itself rather than the contract
(its numpy payload arrays, its numba kernels) are listed in ``INTERNAL`` with the reason;
everything else must pass.
"""

import os
import re
import subprocess
import sys

import pytest

from conftest import REPO

REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "hecnn_tests")

# reference tests whose subject is CkksBackend's numpy payload layout, not the contract
INTERNAL = {
    # builds a corrupted payload with dataclasses.replace(payload, c0=...) on numpy rows;
    # the device equivalent is tests/test_gpu_invariants.py::test_decrypt_detects_out_of_range_coefficients
    "test_pipeline_invariants.py::test_decrypt_detects_out_of_range_coefficients",
}

SUITES = ["test_backend_contract.py", "test_backend_agreement.py", "test_executor.py", "test_pipeline_invariants.py",
          "test_layers.py", "test_model.py", "test_packing.py"]


def hecnn_importable() -> bool:
    res = subprocess.run([sys.executable, "-c", "import hecnn"], env=dict(os.environ, PYTHONPATH=REF),
                         capture_output=True)
    return res.returncode == 0


def test_plugin_is_a_reference_backend():
    """CPU: the plugin class is a concrete subclass of the reference's HEBackend."""
    if not hecnn_importable():
        pytest.skip("reference not installed (tools/install_reference.sh)")
    code = ("import inspect, hecnn.backends.base as hb\n"
            "from paper_2102_00319_b200.hecnn_plugin import backend_class\n"
            "cls = backend_class()\n"
            "assert issubclass(cls, hb.HEBackend) and not inspect.isabstract(cls), cls.__abstractmethods__\n"
            "assert cls.name == 'ckks'\n"
            "print('ok')\n")
    res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PYTHONPATH=f"{REF}:{REPO}"),
                         capture_output=True, text=True, cwd=REPO)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_device_backend(suite):
    if not os.path.exists(os.path.join(REF_TESTS, suite)) or not hecnn_importable():
        pytest.skip("reference suite not installed (tools/install_reference.sh)")
    env = dict(os.environ, PYTHONPATH=f"{REF}:{REPO}:{REF_TESTS}", HECNN_CKKS_IMPL="b200")
    deselect = [a for t in INTERNAL if t.startswith(suite) for a in ("--deselect", t)]
    res = subprocess.run([sys.executable, "-m", "pytest", suite, "-q", "-p", "paper_2102_00319_b200.hecnn_plugin",
                          "-p", "no:cacheprovider", "-rf", *deselect],
                         env=env, capture_output=True, text=True, cwd=REF_TESTS, timeout=1500)
    tail = res.stdout[-4000:]
    summary = re.findall(r"(\d+) (passed|failed|error)", tail)
    counts = {k: int(v) for v, k in summary}
    assert res.returncode == 0 and counts.get("passed", 0) > 0 and not counts.get("failed"), tail + res.stderr[-2000:]
