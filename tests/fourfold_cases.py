"""Shared definition of the random cubic fourfold /F7 chunk cases
(BASELINE.json configs[4]; fixtures made by scripts/make_fourfold_golden.py).

Each case is one reduce_chunk move (u, pole, v, k) that is legal for the
fourfold's working set S = {3, 4, 5} (reference reduction.hpp:35-56): v is
the reference's greedy choice (choose_v_greedy + repair_v, reduction.hpp:71-111)
and k <= k_max_legal.  The input vector is regenerated from (M, case index).
"""
from __future__ import annotations

import numpy as np

FOURFOLD = (7, 5, 3, 1)  # p, n, d, seed

CASES = [
    # (u, pole, v, k)
    ([15, 16, 17, 18, 19, 20], 30, [0, 0, 0, 1, 1, 1], 3),
    ([30, 2, 9, 25, 0, 11], 44, [1, 0, 0, 1, 0, 1], 4),
    ([1, 1, 1, 40, 31, 28], 105, [0, 0, 0, 1, 1, 1], 7),
]


def chunk_input(p: int, M: int, side: int, case: int) -> np.ndarray:
    """random residues mod p^M in the reference ModVec plane-major layout
    (linalg.hpp:94-117): limbs planes of base-beta digits"""
    limbs = 1
    while True:
        e = -(-M // limbs)
        if p ** e <= (1 << 62) and limbs * (p ** e - 1) ** 2 <= (1 << 126):
            break
        limbs += 1
    beta = p ** e
    rng = np.random.default_rng(1000 * M + case)
    mod = p ** M
    vals = [int(rng.integers(0, 2**62)) * int(rng.integers(1, 2**62)) % mod for _ in range(side)]
    out = []
    for t in range(limbs):
        out.extend((x // beta ** t) % beta for x in vals)
    return np.array(out, dtype=np.uint64)
