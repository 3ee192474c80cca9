"""GPU exploration: the whole Frobenius matrix of the random cubic fourfold /F7
(configs[4]) with DRZG_VERBOSE group marks (per-group matvecs and wall), to
compare each group's wall time with its kernel-rate estimate."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24155_b200 as drzg

co = drzg.random_hypersurface(7, 5, 3, 1)
drzg.frobenius(7, 5, 3, co, columns=[0])  # warm-up: tables, pool
t = time.time()
r = drzg.frobenius(7, 5, 3, co)
w = time.time() - t
print(json.dumps({"wall": round(w, 3), "times": r["times"], "matvecs": r["matvecs"], "kernels": r["kernels"],
                  "traffic": r.get("traffic"),
                  "F_sha": __import__("hashlib").sha256(json.dumps(r["F"]).encode()).hexdigest()}))
