#!/usr/bin/env python3
"""Generate the committed golden fixtures under tests/golden/ from the
UNMODIFIED reference (oracle/_ref/libdrz_ref.so, built by `make -C oracle`).

Run in the dev container (the one with /root/reference).  Each case writes
tests/golden/<name>.json holding the inputs (p, n, d, coefficient vector in the
reference's grevlex order, plan overrides) and the reference's outputs
(Frobenius matrix F, charpoly residues, Q, cost ledger).

    python scripts/make_golden.py e2e quintic_f7_s1
    python scripts/make_golden.py kernels
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import refapi  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

# name -> (p, n, d, mode, seed, r_uniform, nm_override, threads[, policy])
E2E = {
    "fermat_cubic_curve_f7": (7, 2, 3, "fermat", 1, 0, 0, 1),
    "random_cubic_curve_f11_s3": (11, 2, 3, "random", 3, 0, 0, 1),
    "random_quartic_curve_f7_s2": (7, 2, 4, "random", 2, 0, 0, 1),
    "quintic_f7_s1": (7, 2, 5, "random", 1, 0, 0, 1),
    "fermat_quartic_surface_f7": (7, 3, 4, "fermat", 1, 0, 0, 8),
    "k3_f11_s1_r1": (11, 3, 4, "random", 1, 1, 0, 8),
    "k3_f11_s1": (11, 3, 4, "random", 1, 0, 0, 8),
    "threefold_f13_s1": (13, 4, 3, "random", 1, 0, 0, 8),
    "threefold_f13_s1_r1": (13, 4, 3, "random", 1, 1, 0, 8),
    "fermat_fourfold_f7_r1": (7, 5, 3, "fermat", 1, 1, 0, 4),
    "quintic_surface_f7_s1_r1": (7, 3, 5, "random", 1, 1, 3, 8),
    # the metric's own hypersurface (configs[4], random cubic fourfold /F7,
    # seed 1) at series-truncated plans the reference can finish here: N_m = 2
    # (M = 2, one base-49 digit) and N_m = 3 (M = 3, two digits: Dixon carry)
    "random_fourfold_f7_s1_nm2": (7, 5, 3, "random", 1, 0, 2, 6),
    "random_fourfold_f7_s1_nm3": (7, 5, 3, "random", 1, 0, 3, 6),
    # the other two reduction policies (reduction.hpp:464-533): same F, own ledgers
    "quintic_f7_s1_depth": (7, 2, 5, "random", 1, 0, 0, 4, "depth-first"),
    "quintic_f7_s1_vbv": (7, 2, 5, "random", 1, 0, 0, 4, "var-by-var"),
    "k3_f11_s1_r1_depth": (11, 3, 4, "random", 1, 1, 0, 8, "depth-first"),
    "k3_f11_s1_r1_vbv": (11, 3, 4, "random", 1, 1, 0, 8, "var-by-var"),
    "threefold_f13_s1_r1_vbv": (13, 4, 3, "random", 1, 1, 0, 8, "var-by-var"),
}


def e2e(name):
    p, n, d, mode, seed, ru, nm, threads = E2E[name][:8]
    policy = E2E[name][8] if len(E2E[name]) > 8 else "p-chunk"
    coeffs = refapi.hypersurface(p, n, d, seed=seed, mode=mode, policy=policy)
    t0 = time.time()
    fr = refapi.frobenius(p, n, d, coeffs, policy=policy, threads=threads, r_uniform=ru, nm=nm)
    out = {
        "name": name, "p": p, "n": n, "d": d, "mode": mode, "seed": seed, "policy": policy,
        "r_uniform": ru, "nm_override": nm, "coeffs": coeffs,
        "plan": fr["plan"], "b": fr["b"], "F": fr["F"], "charpoly": fr["charpoly"],
        "ledger": {k: fr[k] for k in ("matvecs", "startups", "combines", "pep_misses")},
        "ref_seconds": fr["seconds"], "ref_threads": threads,
    }
    try:
        cp = refapi.charpoly(p, n, d, fr["F"], fr["b"], r_uniform=ru, nm=nm)
        out["recover_status"] = cp["status"]
        out["Q_candidates"] = cp["candidates"]
    except RuntimeError as e:  # recovery can legitimately fail at reduced plans
        out["recover_error"] = str(e)
    out["generated_seconds"] = time.time() - t0
    with open(os.path.join(GOLD, f"{name}.json"), "w") as f:
        json.dump(out, f)
    print(name, "done in", round(time.time() - t0, 1), "s", "ledger", out["ledger"])


# (p, M, side, density, tmax, seed): kernel-level vectors for linrec_eval
KERNEL_CASES = [
    (101, 1, 1, 1.0, 2, 0),
    (7, 4, 8, 1.0, 20, 1),
    (7, 16, 45, 1.0, 6, 2),
    (11, 17, 40, 1.0, 10, 3),
    (13, 13, 33, 1.0, 12, 4),
    (7, 24, 20, 1.0, 6, 5),      # 2 limbs, dense generic path
    (7, 24, 24, 0.05, 6, 6),     # 2 limbs, sparse path
    (7, 49, 12, 1.0, 4, 7),      # 3 limbs
    (11, 17, 60, 0.04, 10, 8),   # 1 limb sparse
    (47, 11, 16, 1.0, 46, 9),    # large p
]


def rand_planes(rng, pl, p, M, side, density):
    mod = p ** M
    vals = [int(rng.integers(0, 2**62)) * int(rng.integers(0, 2**62)) % mod for _ in range(side * side)]
    mask = rng.random(side * side) < density
    vals = [v if m else 0 for v, m in zip(vals, mask)]
    return digitize(vals, pl)


def digitize(vals, pl):
    L, beta = pl["limbs"], pl["beta"]
    out = np.zeros((L, len(vals)), dtype=np.uint64)
    for i, v in enumerate(vals):
        for t in range(L):
            out[t, i] = v % beta
            v //= beta
    return out.reshape(-1)


def kernels():
    cases = []
    for (p, M, side, dens, tmax, seed) in KERNEL_CASES:
        rng = np.random.default_rng(1000 + seed)
        pl = refapi.stripe_plan(p, M)
        A = rand_planes(rng, pl, p, M, side, dens)
        B = rand_planes(rng, pl, p, M, side, dens)
        mod = p ** M
        w = digitize([int(rng.integers(0, 2**62)) * int(rng.integers(0, 2**62)) % mod for _ in range(side)], pl)
        out, ctr = refapi.linrec_eval(p, M, side, A, B, tmax, w)
        cases.append({"p": p, "M": M, "side": side, "density": dens, "tmax": tmax, "plan": pl,
                      "A": [str(x) for x in A], "B": [str(x) for x in B], "w": [str(x) for x in w],
                      "out": [str(x) for x in out], "matvecs": ctr})
    with open(os.path.join(GOLD, "linrec_cases.json"), "w") as f:
        json.dump({"cases": cases}, f)
    print("kernels:", len(cases), "cases")


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    what = sys.argv[1]
    if what == "kernels":
        kernels()
    elif what == "e2e":
        for name in sys.argv[2:] or list(E2E):
            e2e(name)
