"""Weight-table I/O: exchange harvested tables.

* ``weight_table_json`` (harvest.py:238-265) is in ``harvest.py`` and writes
  the reference's text byte for byte; ``parse_weight_table_json`` reads that
  text back into compact device rows (floats printed with 17 significant
  digits round-trip exactly).
* ``save_weight_table`` / ``load_weight_table``: the binary equivalent -- the
  compact form itself (shared / class / per-node SoA rows plus the stencil
  geometry), so a 2^22-node per-node table is one contiguous f64 block that
  loads straight into HBM instead of 4M JSON records.

Binary layout (little endian):
    magic    8 bytes  b"LMEPWT\\x00\\x01"
    header   9 x int64: N, n, row, periodic, mode, R, nleft, nright, pernode_pad
             1 x f64  : delta_t
    payload  SHARED : interior f64 [R][n]
             CLASS  : interior f64 [R][n], classes f64 [nleft+1+nright][R][n]
             PERNODE: pernode f64 [R][n][N + 2*pernode_pad]
"""

from __future__ import annotations

import json
import struct

import numpy as np
import torch

from . import _native as nat
from . import _ops
from .errors import DimensionMismatch, InvalidConfig
from .grid import StencilSet

MAGIC = b"LMEPWT\x00\x01"
_HEAD = struct.Struct("<9qd")


def _dev(device):
    return nat.device() if device is None else torch.device(device)


def save_weight_table(path, rows: _ops.CompactRows, delta_t: float) -> int:
    """Write compact rows to ``path``; returns the number of bytes written."""
    L = rows.layout
    head = _HEAD.pack(L.N, L.n, L.row, int(L.periodic), int(rows.mode), rows.R, int(rows.nleft),
                      int(rows.nright), int(rows.pernode_pad), float(delta_t))
    parts = []
    if rows.mode == nat.W_PERNODE:
        parts.append(rows.pernode)
    else:
        parts.append(rows.interior)
        if rows.mode == nat.W_CLASS:
            parts.append(rows.classes)
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(head)
        nbytes = len(MAGIC) + len(head)
        for p in parts:
            a = np.ascontiguousarray(p.detach().to("cpu", torch.float64).numpy())
            f.write(a.tobytes())
            nbytes += a.nbytes
    return nbytes


def load_weight_table(path, device=None) -> tuple[_ops.CompactRows, float]:
    """Read a table written by ``save_weight_table`` -> (rows on the device, delta_t)."""
    with open(path, "rb") as f:
        if f.read(len(MAGIC)) != MAGIC:
            raise InvalidConfig(f"{path}: not an LMEP weight table")
        N, n, row, periodic, mode, R, nleft, nright, pad, dt = _HEAD.unpack(f.read(_HEAD.size))
        body = np.frombuffer(f.read(), dtype="<f8")
    sset = StencilSet(N, n, row, bool(periodic))
    dev = _dev(device)

    def take(count, shape):
        nonlocal body
        if body.size < count:
            raise DimensionMismatch(f"{path}: truncated payload")
        a, body = body[:count], body[count:]
        t = torch.from_numpy(a.copy()).reshape(shape)
        return t.pin_memory().to(dev, non_blocking=True) if dev.type == "cuda" else t.to(dev)

    if mode == nat.W_PERNODE:
        cols = N + 2 * pad
        out = _ops.CompactRows(sset, mode, pernode=take(R * n * cols, (R, n, cols)),
                               pernode_pad=pad)
    elif mode in (nat.W_SHARED, nat.W_CLASS):
        interior = take(R * n, (R, n))
        classes = None
        if mode == nat.W_CLASS:
            C = nleft + 1 + nright
            classes = take(C * R * n, (C, R, n))
        out = _ops.CompactRows(sset, mode, interior, classes, nleft, nright)
    else:
        raise InvalidConfig(f"{path}: unknown weight mode {mode}")
    if body.size:
        raise DimensionMismatch(f"{path}: {body.size} trailing values")
    return out, float(dt)


def parse_weight_table_json(text: str, device=None) -> tuple[_ops.CompactRows, float]:
    """Inverse of ``weight_table_json``: the table as per-node compact rows
    [s][n][N] (R = s: w_lin then the raw dt^j phi_j rows) and delta_t.
    The member windows must be the contiguous periodic or clamped windows
    ``select_stencils`` produces (the step kernels' only layouts)."""
    doc = json.loads(text)
    N, n, s = int(doc["N"]), int(doc["n"]), int(doc["s"])
    recs = doc["nodes"]
    if len(recs) != N:
        raise DimensionMismatch("record count differs from N")
    members = np.array([r["members"] for r in recs], dtype=np.int64)
    rows_t = np.array([r["target_row"] for r in recs], dtype=np.int64)
    W = np.empty((s, n, N))
    for i, r in enumerate(recs):
        W[0, :, i] = r["w_lin"]
        for j, v in enumerate(r["w_phi"]):
            W[j + 1, :, i] = v
    sset = _layout_from_members(members, rows_t)
    t = torch.from_numpy(W)
    dev = _dev(device)
    return _ops.CompactRows(sset, nat.W_PERNODE, pernode=t.to(dev)), float(doc["delta_t"])


def _layout_from_members(members: np.ndarray, target_rows: np.ndarray) -> StencilSet:
    N, n = members.shape
    interior = int(target_rows[N // 2])
    for periodic in (True, False):
        sset = StencilSet(N, n, interior, periodic)
        if np.array_equal(sset.members_array(), members) and \
                np.array_equal(sset.target_rows(), target_rows):
            return sset
    raise InvalidConfig("member windows are not contiguous periodic or clamped windows")
