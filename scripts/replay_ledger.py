#!/usr/bin/env python3
"""TEST INFRASTRUCTURE: the reference's cost ledger by value-free replay
(oracle/ref_capi.cpp ref_replay_ledger: frobenius_terms + seed split +
run_policy p-chunk bookkeeping + combine_states, no matrices).  The replay
equals the real reference ledger on every fixture of tests/golden
(tests/test_oracle.py checks that); this script records it for the default
plans the reference cannot run here.

    python scripts/replay_ledger.py fourfold        # random cubic fourfold /F7 seed 1
    python scripts/replay_ledger.py quintic_surface # random quintic surface /F7 seed 1
"""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import refapi  # noqa: E402

CASES = {"fourfold": (7, 5, 3, 1), "quintic_surface": (7, 3, 5, 1), "threefold": (13, 4, 3, 1)}

if __name__ == "__main__":
    name = sys.argv[1]
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    p, n, d, seed = CASES[name]
    coeffs = refapi.hypersurface(p, n, d, seed=seed)
    t0 = time.time()
    r = refapi.replay_ledger(p, n, d, coeffs, threads=threads)
    out = {"name": name, "p": p, "n": n, "d": d, "seed": seed, "coeffs": coeffs, "ledger": {
        k: r[k] for k in ("matvecs", "startups", "combines")}, "columns": r["columns"], "plan": r["plan"],
        "replay_seconds": time.time() - t0,
        "source": "oracle/ref_capi.cpp ref_replay_ledger over the unmodified reference headers"}
    with open(os.path.join(ROOT, "tests", "golden", f"ledger_replay_{name}.json"), "w") as f:
        json.dump(out, f)
    print(name, out["ledger"], round(out["replay_seconds"], 1), "s")
