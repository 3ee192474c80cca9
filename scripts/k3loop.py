import sys, time, json
sys.path.insert(0, '/root/repo')
import paper_2602_24155_b200 as drzg
co = drzg.random_hypersurface(11, 3, 4, 1)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    t = time.time()
    z = drzg.zeta(11, 3, 4, co, device=0, verify_counts=True)
    t1 = time.time()
    fr = z["frobenius"]
    print(i, "wall", round(t1 - t, 3), "seconds", z.get("seconds"), "times", fr["times"], "dev_ms", fr["kernels"]["device_ms"], flush=True)
