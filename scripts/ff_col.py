"""GPU exploration: one column of the random cubic fourfold /F7 (configs[4]),
profiled per kernel (CUDA events), printing the kernel split and the timings."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24155_b200 as drzg

cols = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0").split(",")]
col = cols[0]
prof = bool(int(os.environ.get("DRZG_PROFILE", "1")))
co = drzg.random_hypersurface(7, 5, 3, 1)
drzg.frobenius(7, 5, 3, co, columns=cols, profile=False)  # warm-up: tables, pool
t = time.time()
r = drzg.frobenius(7, 5, 3, co, columns=cols, profile=prof)
w = time.time() - t
k = r["kernels"]
macs = k["gemm_macs"] + k["carry_macs"]
print(json.dumps({"cols": cols, "wall": round(w, 3), "times": r["times"], "kernels": k, "matvecs": r["matvecs"],
                  "flow_tops": 2 * macs / max(1e-9, k["gemm_ms"] / 1e3) / 1e12 if prof else None,
                  "F_col_sha": __import__("hashlib").sha256(json.dumps([r["F"][i * r["b"] + col] for i in range(r["b"])]).encode()).hexdigest()}))
