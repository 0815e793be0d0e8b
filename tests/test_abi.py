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


# SURVEY.md 8(b) "minimum C-ABI exports" (names as the survey gives them)
SURVEY_8B = ["heb_ctx_create", "heb_ctx_destroy", "heb_alloc", "heb_free", "heb_h2d", "heb_d2h", "heb_ntt_fwd",
             "heb_ntt_inv", "heb_add", "heb_add_plain", "heb_tensor", "heb_mul_plain_rescale", "heb_rescale",
             "heb_relin_rescale", "heb_rotate", "heb_conv", "heb_square", "heb_poly_act", "heb_sumpool", "heb_fc",
             "heb_gather_logits", "heb_last_error"]


def test_header_covers_survey_boundary():
    names = set(_header_functions())
    missing = [n for n in SURVEY_8B if n not in names]
    assert not missing, missing


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
