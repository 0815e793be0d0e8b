"""The C-ABI library loads without a GPU and exports every entry point of include/heb200.h."""

import os
import re

from conftest import REPO


def _header_functions():
    text = open(os.path.join(REPO, "include", "heb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(heb_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = _header_functions()
    assert "heb_relin_rescale" in names and "heb_ntt_fwd" in names and "heb_dot_tensor" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    from paper_2102_00319_b200 import _lib
    from paper_2102_00319_b200.build import build

    build()
    lib = _lib.load()
    for name in _header_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes binding"
    assert lib.heb_version() == 1


def test_product_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        return
    import pytest
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.errors import DeviceError
    from conftest import s128_params

    with pytest.raises(DeviceError):
        B200Backend(s128_params())
