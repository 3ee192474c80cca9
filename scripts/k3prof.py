"""GPU exploration: K3 /F11 (configs[1]) Frobenius matrix with per-kernel
CUDA-event timing (profile=True), a few repetitions; prints the kernel split."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24155_b200 as drzg

co = drzg.random_hypersurface(11, 3, 4, 1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for i in range(reps):
    r = drzg.frobenius(11, 3, 4, co, profile=True)
    k = r["kernels"]
    print(json.dumps({k2: round(v, 2) if isinstance(v, float) else v for k2, v in k.items()}), flush=True)
fr = drzg.frobenius(11, 3, 4, co)
print(json.dumps({"F_sha": __import__("hashlib").sha256(json.dumps(fr["F"]).encode()).hexdigest(), "times": fr["times"]}))
