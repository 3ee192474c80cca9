"""one linrec_eval factor at side 3003 (1 and 2 limbs) and 495, for ncu"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_24155_b200 as drzg
for p, M, side in [(7, 20, 3003), (7, 24, 3003), (13, 13, 495)]:
    sp = drzg.stripe_plan(p, M)
    L = sp.limbs
    g = torch.Generator(device="cuda").manual_seed(1)
    hi = min(int(sp.beta), 2**62)
    A = torch.randint(0, hi, (L * side * side,), dtype=torch.int64, device="cuda", generator=g)
    B = torch.randint(0, hi, (L * side * side,), dtype=torch.int64, device="cuda", generator=g)
    w = torch.randint(0, hi, (L * side,), dtype=torch.int64, device="cuda", generator=g)
    if L > 1:
        top = p ** (M - sp.limb_exp * (L - 1))
        A.view(L, -1)[L - 1] %= top
        B.view(L, -1)[L - 1] %= top
        w.view(L, -1)[L - 1] %= top
    drzg.linrec_eval_device(p, M, side, A.data_ptr(), B.data_ptr(), 1, w.data_ptr())
torch.cuda.synchronize()
print("ok")
