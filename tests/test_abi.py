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


def test_comm_entry_points_validate_without_a_gpu():
    """The sharded-run entry points reject bad handles / arguments before any
    CUDA call, and creating a communicator without a device fails loudly."""
    import ctypes as C
    import torch
    from paper_2603_15964_b200 import _native as nat
    lib = nat.load()
    assert lib.lmep_halo_exchange(None, 1, None, 10, 2, None, None, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_comm_gather(None, None, None, None, 0, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_comm_flag_max(None, None, 1, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_comm_info(None, None, None, None, None, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_comm_signal(None, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_comm_wait(None, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_graph_launch(None, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_comm_destroy(None) == nat.LMEP_OK and lib.lmep_graph_destroy(None) == nat.LMEP_OK
    h = C.c_void_p()
    # rank outside the world, unknown transport, NCCL without an id, PEER without a width
    for args in [(3, 2, 1, nat.COMM_NCCL, None, 0), (0, 1, 1, 7, None, 0), (0, 0, 1, nat.COMM_PEER, None, 8)]:
        assert lib.lmep_comm_init(C.byref(h), *args) == nat.LMEP_INVALID_CONFIG, args
    if not torch.cuda.is_available():
        from paper_2603_15964_b200 import errors
        from paper_2603_15964_b200.distributed import Comm
        with pytest.raises(errors.LocalExpError):
            Comm(0, 1, True, "peer", max_width=8)


def test_slice_transfer_entry_points_validate_without_a_gpu():
    """lmep_upload_slice / lmep_stream_wait_event / lmep_event_create reject missing
    events and buffers before any CUDA call."""
    from paper_2603_15964_b200 import _native as nat
    lib = nat.load()
    assert lib.lmep_upload_slice(None, None, 0, None, None, None, 0, None, None, None, None) == \
        nat.LMEP_INVALID_CONFIG
    assert lib.lmep_stream_wait_event(None, None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_event_create(None) == nat.LMEP_INVALID_CONFIG
    assert lib.lmep_event_destroy(None) == nat.LMEP_OK


def test_header_is_plain_c(tmp_path):
    """include/lmep.h on its own compiles as C99 (a cgo / ctypes-side binding
    includes nothing else first)."""
    import subprocess
    src = tmp_path / "hdr.c"
    src.write_text('#include "lmep.h"\nint main(void) { return 0; }\n')
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    r = subprocess.run(["gcc", "-fsyntax-only", "-std=c99", "-Wall", "-Werror", "-I", inc, str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
