"""GPU exploration: BASELINE configs[3] (64 random cubic threefolds /F13) as
one batch, sequential against zeta_batch with W workers; checks every Q is
the same either way."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24155_b200 as drzg

n_hyp = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cos = [drzg.random_hypersurface(13, 4, 3, seed=s) for s in range(n_hyp)]
drzg.zeta(13, 4, 3, cos[0])  # warm-up
res = {}
for w in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]:
    t = time.time()
    zs = drzg.zeta_batch(13, 4, 3, cos, workers=w)
    wall = time.time() - t
    res[w] = [z["Q"] for z in zs]
    ok = all(ok for z in zs for (_, _, ok) in z["counts"])
    print(json.dumps({"workers": w, "wall_s": round(wall, 3), "per_zeta_s": round(wall / n_hyp, 4), "counts_ok": ok,
                      "same_Q_as_first": res[w] == next(iter(res.values()))}), flush=True)
