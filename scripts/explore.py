"""GPU exploration: time the engine on the larger configurations."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24155_b200 as drzg

cases = sys.argv[1:] or ["k3", "threefold", "fermat4_r1", "fermat4", "fourfold_r1"]
for c in cases:
    t = time.time()
    try:
        if c == "k3":
            co = drzg.random_hypersurface(11, 3, 4, 1); r = drzg.frobenius(11, 3, 4, co, profile=bool(int(os.environ.get("DRZG_PROFILE", "1"))))
        elif c == "threefold":
            co = drzg.random_hypersurface(13, 4, 3, 1); r = drzg.frobenius(13, 4, 3, co, profile=bool(int(os.environ.get("DRZG_PROFILE", "1"))))
        elif c == "fermat4_r1":
            co = drzg.random_hypersurface(7, 5, 3, 1, fermat=True); r = drzg.frobenius(7, 5, 3, co, r_uniform=1, profile=bool(int(os.environ.get("DRZG_PROFILE", "1"))))
        elif c == "fermat4":
            co = drzg.random_hypersurface(7, 5, 3, 1, fermat=True); r = drzg.frobenius(7, 5, 3, co, profile=bool(int(os.environ.get("DRZG_PROFILE", "1"))))
        elif c == "fourfold_r1":
            co = drzg.random_hypersurface(7, 5, 3, 1); r = drzg.frobenius(7, 5, 3, co, r_uniform=1, columns=[1], profile=bool(int(os.environ.get("DRZG_PROFILE", "1"))))
        elif c.startswith("fourfold_col"):
            col = int(c[len("fourfold_col"):])
            co = drzg.random_hypersurface(7, 5, 3, 1); r = drzg.frobenius(7, 5, 3, co, columns=[col], profile=bool(int(os.environ.get("DRZG_PROFILE", "1"))))
        elif c == "fourfold_zeta":
            co = drzg.random_hypersurface(7, 5, 3, 1); r = drzg.zeta(7, 5, 3, co, profile=False)
            r = {k: r[k] for k in ("Q", "ambiguous", "slopes", "newton_height", "p_rank", "counts", "escalations", "seconds", "frobenius")}
        elif c == "threefold_zeta":
            co = drzg.random_hypersurface(13, 4, 3, 1); r = drzg.zeta(13, 4, 3, co)
            r.pop("frobenius", None)
        elif c == "qsurf_zeta":
            co = drzg.random_hypersurface(7, 3, 5, 1); r = drzg.zeta(7, 3, 5, co, profile=False)
            r = {k: r[k] for k in r if k not in ("F", "charpoly")}
        elif c == "qsurf_r1":
            co = drzg.random_hypersurface(7, 3, 5, 1); r = drzg.frobenius(7, 3, 5, co, r_uniform=1, nm=3, profile=bool(int(os.environ.get("DRZG_PROFILE", "1"))))
        r.pop("F", None); r.pop("charpoly", None)
        print(c, round(time.time() - t, 2), json.dumps(r), flush=True)
    except Exception as e:
        print(c, "ERROR", e, flush=True)
