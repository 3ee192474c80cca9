"""Multi-GPU plumbing for the Frobenius matrix (one process per GPU).

Columns of F are independent (reference zeta.hpp:109-133 threads over
them), so each rank reduces a subset of columns on its own GPU and the
per-rank column blocks are combined with ONE all_gather (NCCL over
NVLink/NVSwitch in production, gloo in the CPU tests).  Entries travel as
fixed-width 62-bit limbs: NCCL's integer Sum would wrap mod 2^64, and every
entry has exactly one owner, so no reduction is needed — the receiver just
takes each column from its owner.
"""
from __future__ import annotations

from typing import List, Sequence

LIMB_BITS = 62
LIMB_MASK = (1 << LIMB_BITS) - 1


def hodge_counts(n: int, d: int) -> List[int]:
    """h_m for m = 1..n (reference cohomology.hpp:37-53)"""
    from math import comb
    h = []
    for m in range(1, n + 1):
        k = d * m - n - 1
        acc = 0
        j = 0
        while j * (d - 1) <= k and j <= n + 1:
            acc += (-1) ** j * comb(n + 1, j) * comb(k - j * (d - 1) + n, n)
            j += 1
        h.append(acc if k >= 0 else 0)
    return h


def column_poles(n: int, d: int) -> List[int]:
    """pole order of each basis column (the basis is sorted by pole, cohomology.hpp:134-160)"""
    out = []
    for m, hm in enumerate(hodge_counts(n, d), start=1):
        out.extend([m] * hm)
    return out


def partition_columns(n: int, d: int, world: int, rank: int, weights: Sequence[float] | None = None) -> List[int]:
    """longest-processing-time assignment of columns to ranks.  Default
    weight of a pole-m column: its maximum pole p*s_m grows with m, and the
    work per column grows roughly with its square, so (m + c)^2 with the
    series length folded into c is a good proxy; callers can pass measured
    per-column costs instead."""
    poles = column_poles(n, d)
    if weights is None:
        weights = [float((m + n + 4) ** 2) for m in poles]
    order = sorted(range(len(poles)), key=lambda j: (-weights[j], j))
    load = [0.0] * world
    owner = [0] * len(poles)
    for j in order:
        r = min(range(world), key=lambda i: (load[i], i))
        owner[j] = r
        load[r] += weights[j]
    return [j for j in range(len(poles)) if owner[j] == rank]


def encode_columns(F: Sequence[str | int], b: int, cols: Sequence[int], width: int) -> List[int]:
    """b x b row-major F (strings or ints) -> flat limbs of the owned columns'
    entries, zeros elsewhere: b*b*width int64-safe values"""
    owned = set(cols)
    flat = [0] * (b * b * width)
    for i in range(b):
        for j in owned:
            v = int(F[i * b + j])
            if v < 0:
                raise ValueError("Frobenius entries are non-negative residues")
            base = (i * b + j) * width
            for t in range(width):
                flat[base + t] = (v >> (LIMB_BITS * t)) & LIMB_MASK
            if v >> (LIMB_BITS * width):
                raise ValueError("entry exceeds the limb width")
    return flat


def decode_blocks(blocks: Sequence[Sequence[int]], owners: Sequence[Sequence[int]], b: int, width: int) -> List[int]:
    """per-rank flat limb blocks + each rank's column list -> full F (ints)"""
    F = [0] * (b * b)
    for blk, cols in zip(blocks, owners):
        for j in cols:
            for i in range(b):
                base = (i * b + j) * width
                F[i * b + j] = sum(int(blk[base + t]) << (LIMB_BITS * t) for t in range(width))
    return F


def gather_frobenius(F_local, b: int, cols: Sequence[int], world: int, all_cols: Sequence[Sequence[int]],
                     device=None, width: int = 6):
    """all_gather the ranks' column blocks (torch.distributed must be
    initialised; NCCL when `device` is a CUDA device, else the default group's
    backend) and return the assembled F as Python ints on every rank"""
    import torch
    import torch.distributed as dist
    flat = encode_columns(F_local, b, cols, width)
    t = torch.tensor(flat, dtype=torch.int64, device=device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    return decode_blocks([o.tolist() for o in outs], all_cols, b, width)


# --------------------------------------------------------------------------
# the same gather behind the C ABI (include/drzg.h drzg_gather_F): one
# ncclAllGather issued by libdrzg.so itself; torch.distributed only ships the
# NCCL unique id from rank 0 to the others.

_COMM = {}


def nccl_comm(world: int, rank: int, device: int):
    """the process's drzg_comm (created once per (world, rank, device))"""
    import ctypes
    import torch.distributed as dist
    from . import lib, DrzgError, _err
    key = (world, rank, device)
    if key in _COMM:
        return _COMM[key]
    L = lib()
    buf = (ctypes.c_uint8 * 128)()
    if rank == 0 and L.drzg_nccl_unique_id(buf) != 0:
        raise DrzgError(_err())
    obj = [bytes(buf)]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    L.drzg_comm_init.restype = ctypes.c_void_p
    h = L.drzg_comm_init(world, (ctypes.c_uint8 * 128)(*obj[0]), rank, device)
    if not h:
        raise DrzgError(_err())
    _COMM[key] = h
    return h


def gather_frobenius_nccl(F_local, b: int, cols: Sequence[int], world: int, rank: int, device: int,
                          width: int = 6) -> List[int]:
    """drzg_gather_F: every rank gets the full F (Python ints)"""
    import ctypes
    import json
    from . import lib, DrzgError, _err
    L = lib()
    L.drzg_gather_F.restype = ctypes.c_void_p
    arr = (ctypes.c_char_p * (b * b))(*[str(x).encode() for x in F_local])
    ca = (ctypes.c_int32 * max(1, len(cols)))(*cols)
    ptr = L.drzg_gather_F(ctypes.c_void_p(nccl_comm(world, rank, device)), b, arr, ca, len(cols), width)
    if not ptr:
        raise DrzgError(_err())
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    L.drzg_free(ctypes.c_void_p(ptr))
    return [int(x) for x in json.loads(s)["F"]]


def gather_frobenius_host(blocks, b: int, owners: Sequence[Sequence[int]], width: int = 6) -> List[int]:
    """drzg_gather_F_host: the C++ encode/decode of the gather for several
    ranks' blocks at once (no NCCL; CPU tests)"""
    import ctypes
    import json
    from . import lib, DrzgError, _err
    L = lib()
    L.drzg_gather_F_host.restype = ctypes.c_void_p
    flat = [str(x).encode() for blk in blocks for x in blk]
    cols = [j for o in owners for j in o]
    ptrs = [0]
    for o in owners:
        ptrs.append(ptrs[-1] + len(o))
    ptr = L.drzg_gather_F_host(len(blocks), b, (ctypes.c_char_p * len(flat))(*flat),
                               (ctypes.c_int32 * max(1, len(cols)))(*cols), (ctypes.c_int32 * len(ptrs))(*ptrs),
                               width)
    if not ptr:
        raise DrzgError(_err())
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    L.drzg_free(ctypes.c_void_p(ptr))
    return [int(x) for x in json.loads(s)["F"]]


def replayed_column_weights(ledger_fixture: str) -> List[float]:
    """per-column matvecs of the reference's replayed ledger (scripts/
    replay_ledger.py): the exact work of each column, for partition_columns"""
    import json
    with open(ledger_fixture) as f:
        g = json.load(f)
    return [float(c[0]) for c in g["columns"]]
