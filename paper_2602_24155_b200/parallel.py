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
