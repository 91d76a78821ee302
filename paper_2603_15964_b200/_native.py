"""ctypes binding of liblmep.so (the C ABI declared in include/lmep.h).

The product path has exactly one implementation: the CUDA kernels in this
library.  There is no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises instead of computing elsewhere.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liblmep.so")
CSRC = os.path.join(_HERE, "csrc")

LMEP_OK = 0
LMEP_NONFINITE = 1
LMEP_DIMENSION = 2
LMEP_INVALID_CONFIG = 3
LMEP_CUDA_ERROR = 4
LMEP_ORDER_TOO_HIGH = 5
LMEP_DUPLICATE_NODES = 6

MAX_N = 32
MAX_DIM = 32
MAX_ROWS = 7
ROW_W, ROW_ALPHA, ROW_BETA, ROW_GAMMA, ROW_WHALF, ROW_P1HALF, ROW_D1 = range(7)
NL_NONE, NL_CONVECTIVE, NL_CUBIC = 0, 1, 2
W_SHARED, W_CLASS, W_PERNODE = 0, 1, 2
BC_NONE, BC_DIRICHLET, BC_NEUMANN = 0, 1, 2
FLAG_EXACT = 1
SCH_LIN, SCH_ETDRK4, SCH_ETD2 = 0, 1, 2

# every symbol include/lmep.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "lmep_version", "lmep_status_string", "lmep_last_error", "lmep_fornberg", "lmep_expm",
    "lmep_harvest", "lmep_step_linear", "lmep_step_etdrk4", "lmep_step_etd2",
    "lmep_banded_matvec", "lmep_plan", "lmep_rows_to_soa", "lmep_launch_count",
    "lmep_set_harvest_method", "lmep_set_ring_cluster", "lmep_step_etds", "lmep_harvest_mapped", "lmep_harvest_chunk",
    "lmep_set_pernode_kernel", "lmep_harvest_ex", "lmep_status_any", "lmep_combine",
    "lmep_rows_classify", "lmep_spectral_footprint",
    "lmep_comm_unique_id", "lmep_comm_init", "lmep_comm_export", "lmep_comm_connect",
    "lmep_comm_destroy", "lmep_comm_info", "lmep_halo_exchange", "lmep_comm_gather",
    "lmep_comm_flag_max", "lmep_comm_side_stream", "lmep_comm_fork", "lmep_comm_join",
    "lmep_graph_begin", "lmep_graph_end", "lmep_graph_launch", "lmep_graph_destroy",
    "lmep_comm_targets", "lmep_comm_push", "lmep_comm_signal", "lmep_comm_wait",
    "lmep_comm_ghosts", "lmep_set_etd2_persistent", "lmep_step_linear_host", "lmep_comm_chunk",
    "lmep_harvest_reuse_prep", "lmep_lin_stream_begin", "lmep_lin_stream_info", "lmep_lin_stream_advance", "lmep_lin_stream_end",
    "lmep_event_create", "lmep_event_destroy", "lmep_stream_wait_event", "lmep_upload_slice",
)
COMM_NCCL, COMM_PEER = 0, 1
COMM_ID_BYTES, COMM_BLOB_BYTES, COMM_MAX_FIELDS = 128, 512, 8


class LmepGrid(C.Structure):
    _fields_ = [("N", C.c_int64), ("off", C.c_int64), ("nloc", C.c_int64), ("n", C.c_int32),
                ("row", C.c_int32), ("periodic", C.c_int32), ("reserved", C.c_int32)]


class LmepWeights(C.Structure):
    _fields_ = [("mode", C.c_int32), ("nrows", C.c_int32), ("nleft", C.c_int32),
                ("nright", C.c_int32), ("interior", C.c_void_p), ("classes", C.c_void_p),
                ("pernode", C.c_void_p), ("pernode_pad", C.c_int64)]


class LmepBC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("lo", C.c_double),
                ("hi", C.c_double), ("dl", C.c_void_p), ("dr", C.c_void_p)]


class LmepHalo(C.Structure):
    _fields_ = [("left", C.c_void_p), ("right", C.c_void_p), ("hist_left", C.c_void_p),
                ("hist_right", C.c_void_p), ("width", C.c_int64), ("push_left", C.c_void_p),
                ("push_right", C.c_void_p), ("push_width", C.c_int64)]


class LmepCoefMap(C.Structure):
    _fields_ = [("node0", C.c_int64), ("nnodes", C.c_int64), ("periodic", C.c_int32),
                ("reserved", C.c_int32)]


class LmepHarvestArgs(C.Structure):
    _fields_ = [("n", C.c_int32), ("s", C.c_int32), ("nterms", C.c_int32), ("layout", C.c_int32),
                ("tables", C.c_void_p), ("table_idx", C.c_void_p), ("coef", C.c_void_p),
                ("coef_stride", C.c_int64), ("c0", C.c_void_p), ("c0_stride", C.c_int64),
                ("L", C.c_void_p), ("delta_t", C.c_double), ("target_row", C.c_void_p),
                ("row_default", C.c_int64), ("frozen", C.c_void_p), ("frozen_default", C.c_uint64),
                ("B", C.c_int64), ("out_ld", C.c_int64), ("w_out", C.c_void_p),
                ("status", C.c_void_p), ("ms", C.c_void_p), ("map", C.c_void_p),
                ("half_out", C.c_void_p), ("status_any", C.c_void_p)]


class LmepChunkArgs(C.Structure):
    _fields_ = [("grid", C.c_void_p), ("w", C.c_void_p), ("bc", C.c_void_p), ("scheme", C.c_int32),
                ("nl_kind", C.c_int32), ("u_in", C.c_void_p), ("u_out", C.c_void_p),
                ("ghost_cells", C.c_int64), ("steps", C.c_int64), ("next_steps", C.c_int64),
                ("pushed_cells", C.c_int64), ("flags", C.c_int32), ("reserved", C.c_int32),
                ("nonfinite", C.c_void_p)]


class LmepTuning(C.Structure):
    _fields_ = [("tile", C.c_int32), ("ksteps", C.c_int32), ("ring", C.c_int32),
                ("threads", C.c_int32)]


_lib = None


def build(force: bool = False, jobs: int = 6) -> str:
    """Compile liblmep.so in-tree with nvcc (-gencode arch=compute_100a,code=sm_100a)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", f"-j{jobs}", "-C", CSRC], check=True)
    return LIB_PATH


def load(path: str | None = None):
    """Load the library and declare the C signatures (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("LMEP_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise errors.LocalExpError(
            f"liblmep.so not found at {p}; run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(p)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.lmep_version.restype = C.c_int
    L.lmep_version.argtypes = []
    L.lmep_status_string.restype = C.c_char_p
    L.lmep_status_string.argtypes = [C.c_int]
    L.lmep_last_error.restype = C.c_char_p
    L.lmep_last_error.argtypes = []
    L.lmep_launch_count.restype = C.c_int64
    L.lmep_launch_count.argtypes = []
    L.lmep_fornberg.argtypes = [vp, vp, i64, C.c_int, C.c_int, i64, vp, vp]
    L.lmep_expm.argtypes = [vp, C.c_int, i64, vp, vp, vp, vp]
    L.lmep_harvest.argtypes = [C.c_int, C.c_int, C.c_int, vp, vp, vp, i64, vp, i64, vp, dbl, vp,
                               C.c_int, vp, C.c_uint64, i64, C.c_int, vp, vp, vp, vp]
    L.lmep_harvest_mapped.argtypes = L.lmep_harvest.argtypes[:-1] + [C.POINTER(LmepCoefMap), vp]
    L.lmep_harvest_chunk.argtypes = L.lmep_harvest.argtypes[:-1] + [C.POINTER(LmepCoefMap), i64,
                                                                     vp]
    G, W, B, H, T = (C.POINTER(LmepGrid), C.POINTER(LmepWeights), C.POINTER(LmepBC),
                     C.POINTER(LmepHalo), C.POINTER(LmepTuning))
    L.lmep_step_linear.argtypes = [G, W, B, H, vp, vp, vp, i64, i32, T, vp, vp]
    L.lmep_step_linear_host.argtypes = [G, W, B, H, vp, vp, vp, i64, i32, T, vp, vp, vp, C.c_int, vp]
    L.lmep_harvest_reuse_prep.argtypes = [C.c_int]
    L.lmep_lin_stream_begin.argtypes = [G, W, vp, vp, vp, i64, i32, T, vp, vp, vp, vp, C.POINTER(vp)]
    L.lmep_lin_stream_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32),
                                       C.POINTER(i32)]
    L.lmep_lin_stream_advance.argtypes = [vp, i64, vp]
    L.lmep_lin_stream_end.argtypes = [vp, C.POINTER(i64)]
    L.lmep_event_create.argtypes = [C.POINTER(vp)]
    L.lmep_event_destroy.argtypes = [vp]
    L.lmep_stream_wait_event.argtypes = [vp, vp]
    L.lmep_upload_slice.argtypes = [vp, vp, C.c_size_t, vp, vp, vp, C.c_size_t, vp, vp, vp, vp]
    L.lmep_step_etdrk4.argtypes = [G, W, B, H, C.c_int, vp, vp, vp, i64, vp, i32, T, vp, vp]
    L.lmep_step_etd2.argtypes = [G, W, B, H, C.c_int, dbl, vp, vp, vp, vp, vp, i64, i32, T, vp,
                                 vp]
    L.lmep_step_etds.argtypes = [G, W, B, H, C.c_int, C.c_int, dbl, vp, vp, vp, vp, vp, i64, i32,
                                 T, vp, vp]
    L.lmep_banded_matvec.argtypes = [G, W, H, vp, vp, i32, vp]
    L.lmep_plan.argtypes = [G, C.c_int, C.c_int, C.c_int, i64, T]
    L.lmep_rows_to_soa.argtypes = [vp, i64, C.c_int, vp, vp]
    L.lmep_set_harvest_method.argtypes = [C.c_int]
    L.lmep_set_ring_cluster.argtypes = [C.c_int]
    L.lmep_set_pernode_kernel.argtypes = [C.c_int]
    L.lmep_set_etd2_persistent.argtypes = [C.c_int]
    L.lmep_harvest_ex.argtypes = [C.POINTER(LmepHarvestArgs), vp]
    L.lmep_status_any.argtypes = [vp, i64, vp, vp]
    L.lmep_combine.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                               C.POINTER(C.c_double), i64, i64, vp, i64, vp]
    L.lmep_rows_classify.argtypes = [vp, i64, C.c_int, i64, vp, vp]
    L.lmep_spectral_footprint.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int,
                                          dbl, C.c_int, dbl, vp, vp, vp, vp, vp]
    ip = C.POINTER(C.c_int)
    L.lmep_comm_unique_id.argtypes = [vp]
    L.lmep_comm_init.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.c_int, C.c_int, vp, i64]
    L.lmep_comm_export.argtypes = [vp, vp]
    L.lmep_comm_connect.argtypes = [vp, vp]
    L.lmep_comm_destroy.argtypes = [vp]
    L.lmep_comm_info.argtypes = [vp, ip, ip, ip, ip, ip]
    L.lmep_halo_exchange.argtypes = [vp, C.c_int, C.POINTER(vp), i64, i64, C.POINTER(vp),
                                     C.POINTER(vp), vp]
    L.lmep_comm_gather.argtypes = [vp, vp, C.POINTER(i64), vp, C.c_int, vp]
    L.lmep_comm_flag_max.argtypes = [vp, vp, C.c_int, vp]
    L.lmep_comm_targets.argtypes = [vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]
    L.lmep_comm_push.argtypes = [vp, C.c_int, C.POINTER(vp), i64, i64, vp]
    L.lmep_comm_signal.argtypes = [vp, vp]
    L.lmep_comm_wait.argtypes = [vp, vp]
    L.lmep_comm_ghosts.argtypes = [vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]
    L.lmep_comm_chunk.argtypes = [vp, C.POINTER(LmepChunkArgs), vp]
    L.lmep_comm_side_stream.argtypes = [vp]
    L.lmep_comm_side_stream.restype = vp
    L.lmep_comm_fork.argtypes = [vp, vp]
    L.lmep_comm_join.argtypes = [vp, vp]
    L.lmep_graph_begin.argtypes = [vp]
    L.lmep_graph_end.argtypes = [vp, C.POINTER(vp)]
    L.lmep_graph_launch.argtypes = [vp, vp]
    L.lmep_graph_destroy.argtypes = [vp]
    for name in EXPORTS:
        if name not in ("lmep_version", "lmep_status_string", "lmep_last_error",
                        "lmep_launch_count", "lmep_comm_side_stream"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def lib():
    return load()


_cuda_ok = False
_devices: dict = {}


def device() -> torch.device:
    """The CUDA device of the product path.  Fails loudly without one.  (The
    availability check runs once per process: torch.cuda.is_available() re-reads
    the environment on every call, ~5 us on a path whose host side is timed.)"""
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise errors.LocalExpError(
                "the LMEP hot path runs on CUDA only (B200, sm_100a) and no CUDA device is visible")
        torch.cuda.init()
        _cuda_ok = True
    i = torch._C._cuda_getDevice()
    d = _devices.get(i)
    if d is None:
        d = _devices[i] = torch.device("cuda", i)
    return d


def stream_handle() -> int:
    """The current stream's handle on the current device (the raw accessor:
    torch.cuda.current_stream() builds a Stream object behind three Python layers)."""
    if not _cuda_ok:
        device()
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def check(status: int, what: str, state=None, time=None) -> None:
    """Map an lmep_status onto the localexp exception hierarchy."""
    if status == LMEP_OK:
        return
    msg = f"{what}: {lib().lmep_status_string(status).decode()}"
    if status == LMEP_CUDA_ERROR:
        msg += f" ({lib().lmep_last_error().decode()})"
    cls = errors.for_status(status)
    if cls is errors.NonFinite:
        raise errors.NonFinite(msg, state=state, time=time)
    raise cls(msg)


def set_harvest_method(method: str) -> None:
    """'multiply' (default for d <= 16: expm-multiply; large single-geometry
    per-node batches take the constant-table kernel harvest_mvc, or the
    block-balanced kernel harvest_mvb), "mvb" (auto without harvest_mvc),
    "mvitem" (per-item balanced expm-multiply only, 4 lanes per item), "mv8"
    (the same with 8 lanes per item for d > 8), "mvb2" / "mvb4" / "mvb8" (the
    block kernel at 2 / 4 / 8 lanes per item), "mvc-taylor" (auto with the
    constant-table Taylor kernel only, without the polynomial kernel in front of
    it) or "pade" (full expm per warp).
    Applies to the current CUDA device."""
    code = {"multiply": 0, "auto": 0, "pade": 1, "mv8": 4, "mvitem": 5, "mvb8": 6, "mvb2": 7,
            "mvb4": 8, "mvb": 9, "mvc-taylor": 10}[method]
    check(lib().lmep_set_harvest_method(code), "lmep_set_harvest_method")


def set_pernode_kernel(variant: str) -> None:
    """Persistent per-node linear step kernel: "auto" (default: registers for
    fused multiply-adds, window for the exact order), "registers" (values in
    registers, slot-major halo exchange) or "window" (shared-memory windows)."""
    check(lib().lmep_set_pernode_kernel({"registers": 1, "window": 0, "auto": 2, "registers2": 3, "registers4": 4}[variant]),
          "lmep_set_pernode_kernel")


def set_etd2_persistent(on: bool) -> None:
    """ETD2 on mid-size periodic grids: one cooperative launch for the whole run
    (default) or the tiled launches."""
    check(lib().lmep_set_etd2_persistent(1 if on else 0), "lmep_set_etd2_persistent")


def set_ring_cluster(on) -> None:
    """Linear ring mode on one thread-block cluster (True / 1, default: small rings
    on warp-private register slabs), the shared-memory cluster kernel only (2) or
    one CTA (False / 0)."""
    check(lib().lmep_set_ring_cluster(int(on)), "lmep_set_ring_cluster")
