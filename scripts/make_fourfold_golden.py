#!/usr/bin/env python3
"""TEST INFRASTRUCTURE: reduce_chunk fixtures for the random cubic fourfold /F7
(BASELINE.json configs[4], seed 1) from the UNMODIFIED reference.

The reference cannot run this hypersurface end to end here, but
one chunk can: `ref_ctx_new` builds the reference RuvContext once (a 3003 x
6237 unit echelon: WordEchelon at one limb, MpzEchelon at M = 24, which takes
hours), then `ref_ctx_chunk` runs reduce_chunk (reduction.hpp:394-423) through
build_ruv + eval_to_linear + linrec_eval for each case.  Inputs are regenerated
by the tests from (seed, M, case index), so the fixture stores the moves and
the reference's output vectors (plane-major u64, hex little-endian).

    python scripts/make_fourfold_golden.py 7        # one limb, minutes-hours
    python scripts/make_fourfold_golden.py 24       # the default plan's M, hours
"""
from __future__ import annotations

import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import refapi  # noqa: E402
from fourfold_cases import FOURFOLD, CASES, chunk_input  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def main(M: int) -> None:
    p, n, d, seed = FOURFOLD
    coeffs = refapi.hypersurface(p, n, d, seed=seed)
    L = refapi.lib()
    L.ref_ctx_new.restype = ctypes.c_void_p
    L.ref_ctx_chunk.restype = ctypes.c_void_p
    t0 = time.time()
    h = L.ref_ctx_new(ctypes.c_uint64(p), n, d, refapi._u64(coeffs), M)
    if not h:
        raise RuntimeError("ref_ctx_new failed")
    ctx_s = time.time() - t0
    print(f"M={M}: RuvContext built in {ctx_s:.1f} s", flush=True)
    out = {"p": p, "n": n, "d": d, "seed": seed, "M": M, "coeffs": coeffs,
           "ctx_seconds": ctx_s, "cases": []}
    P = ctypes.POINTER(ctypes.c_uint64)
    for ci, (u, pole, v, k) in enumerate(CASES):
        w = chunk_input(p, M, 3003, ci)
        w_out = np.zeros_like(w)
        info = refapi._js(L.ref_ctx_chunk(ctypes.c_void_p(h), refapi._i32(u), pole, refapi._i32(v),
                                          ctypes.c_long(k), w.ctypes.data_as(P), w_out.ctypes.data_as(P)))
        print(f"  case {ci}: u={u} pole={pole} v={v} k={k}: {info}", flush=True)
        out["cases"].append({"u": u, "pole": pole, "v": v, "k": k, "info": info,
                             "w_out_hex": w_out.astype("<u8").tobytes().hex()})
        with open(os.path.join(GOLD, f"fourfold_chunks_M{M}.json"), "w") as f:
            json.dump(out, f)
    L.ref_ctx_free(ctypes.c_void_p(h))
    print(f"M={M}: done in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]))
