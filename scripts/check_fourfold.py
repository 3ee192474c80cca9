"""Random cubic fourfold /F7 (seed 1) at the reference's default plan: compute
F once, then inspect coefficient recovery and the r = 1 point count."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24155_b200 as drzg

p, n, d = 7, 5, 3
co = drzg.random_hypersurface(p, n, d, 1)
t = time.time()
fr = drzg.frobenius(p, n, d, co, profile=False)
el = time.time() - t
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"coeffs": co, "F": fr["F"], "charpoly": fr["charpoly"], "plan": fr["plan"], "seconds": el,
           "ledger": {k: fr[k] for k in ("matvecs", "startups", "combines", "terms")}, "times": fr["times"]},
          open("gpurun_out/fourfold_F.json", "w"))
cp = drzg.charpoly(p, n, d, fr["F"], fr["b"])
print("frobenius seconds", round(el, 1), "ledger", fr["matvecs"], fr["startups"], fr["combines"], "times", fr["times"])
print("recover status", cp["status"], "candidates", len(cp["candidates"]))
truth = drzg.count_points(p, n, d, co, 1)
for c in cp["candidates"]:
    Q = [int(x) for x in c]
    # counts_from_zeta r = 1: sum_{i<n} p^i + (-1)^{n+1} s_1, s_1 = -a_1 ... via Newton: s1 = e1 = -a1
    s1 = -Q[1]
    pts = sum(p ** i for i in range(n)) + ((-1) ** (n + 1)) * s1
    print("Q head", Q[:6], "count r=1 from zeta", pts, "brute force", truth)
