#!/usr/bin/env python3
"""TEST INFRASTRUCTURE: validate bench.py's reference projection against
complete reference runs measured in this container.

The projection times the reference's frobenius_matrix on the same
hypersurface at a series-truncated plan (N_m = SAMPLE_NM, every column and
pole, same limb count) and scales by the ratio of the exact ledgers.  Here the
same projection is taken with the thread count of the complete run recorded in
the fixture (tests/golden/<config>.json: ref_seconds, ref_threads), and the
ratio projection / measured is written to profiles/r02/cpu_baseline_validation.json.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import refapi  # noqa: E402

CASES = {"k3": ("k3_f11_s1.json", 4), "threefold": ("threefold_f13_s1.json", 4)}

out = {}
for name, (fixture, nm) in CASES.items():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", fixture)))
    threads = g["ref_threads"]
    t0 = time.time()
    fr = refapi.frobenius(g["p"], g["n"], g["d"], g["coeffs"], threads=threads, nm=nm)
    secs = time.time() - t0
    proj = secs * g["ledger"]["matvecs"] / fr["matvecs"]
    out[name] = {"sample_nm": nm, "threads": threads, "sample_seconds": secs, "sample_matvecs": fr["matvecs"],
                 "full_matvecs": g["ledger"]["matvecs"], "projected_seconds": proj,
                 "measured_seconds": g["ref_seconds"], "ratio": proj / g["ref_seconds"],
                 "measured_source": f"tests/golden/{fixture} (complete reference frobenius_matrix run)"}
    print(name, out[name], flush=True)
os.makedirs(os.path.join(ROOT, "profiles", "r02"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "r02", "cpu_baseline_validation.json"), "w") as f:
    json.dump({"method": "bench.py reference_measure: truncated-plan run x exact ledger ratio", "cases": out}, f,
              indent=1)
