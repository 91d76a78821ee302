"""The C-ABI library loads and exports every symbol include/lmep.h declares
(no compute call: this runs without a GPU)."""

import os
import re

import pytest

from tests.conftest import REPO


def _declared():
    src = open(os.path.join(REPO, "include", "lmep.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lmep_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    assert "lmep_harvest" in names and "lmep_step_etdrk4" in names
    from paper_2603_15964_b200 import _native
    assert sorted(_native.EXPORTS) == names


def test_library_exports_every_symbol():
    from paper_2603_15964_b200 import _native
    lib = _native.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.lmep_version() == 100
    assert lib.lmep_status_string(1) == b"non-finite value"
    assert lib.lmep_status_string(3) == b"invalid configuration"


def test_library_is_sm100a():
    from paper_2603_15964_b200 import _native
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_status_maps_to_reference_errors():
    from paper_2603_15964_b200 import _native, errors
    for code, cls in [(1, errors.NonFinite), (2, errors.DimensionMismatch),
                      (3, errors.InvalidConfig), (5, errors.OrderTooHigh),
                      (6, errors.DuplicateNodes)]:
        with pytest.raises(cls):
            _native.check(code, "x")


def test_no_cuda_fails_loudly():
    import torch
    from paper_2603_15964_b200 import _native, errors
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(errors.LocalExpError):
        _native.device()
