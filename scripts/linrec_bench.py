"""GPU: the reference-shaped linrec_eval kernel (drzg_linrec_eval_device,
reference linalg.hpp:337-410) at the BASELINE sizes, CUDA-event timed.
Algorithmic bytes per factor: A and B once, 2 * side^2 * 8 * limbs."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_24155_b200 as drzg

CASES = [(11, 17, 220), (13, 13, 495), (7, 20, 3003), (7, 24, 3003), (7, 24, 455), (7, 49, 455)]
tmax = int(os.environ.get("TMAX", "20"))
out = []
for p, M, side in CASES:
    sp = drzg.stripe_plan(p, M)
    L = sp.limbs
    g = torch.Generator(device="cuda").manual_seed(1)
    beta = int(sp.beta)
    A = torch.randint(0, min(beta, 2**62), (L * side * side,), dtype=torch.int64, device="cuda", generator=g)
    B = torch.randint(0, min(beta, 2**62), (L * side * side,), dtype=torch.int64, device="cuda", generator=g)
    w = torch.randint(0, min(beta, 2**62), (L * side,), dtype=torch.int64, device="cuda", generator=g)
    if L > 1:  # top limb below p^(M - e(L-1))
        top = p ** (M - sp.limb_exp * (L - 1))
        A.view(L, -1)[L - 1] %= top
        B.view(L, -1)[L - 1] %= top
        w.view(L, -1)[L - 1] %= top
    drzg.linrec_eval_device(p, M, side, A.data_ptr(), B.data_ptr(), 2, w.data_ptr())  # warm-up
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        ms = drzg.linrec_eval_device(p, M, side, A.data_ptr(), B.data_ptr(), tmax, w.data_ptr(), timed=True)
        best = min(best, ms)
    per = best / (tmax + 1)
    gbs = 2 * side * side * 8 * L / (per / 1e3) / 1e9
    out.append({"p": p, "M": M, "side": side, "limbs": L, "ms_per_factor": per, "alg_GBps": gbs,
                "matrix_bytes": 2 * side * side * 8 * L})
    print(json.dumps(out[-1]), flush=True)
