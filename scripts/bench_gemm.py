"""Isolated tcgen05 Dixon GEMM timing: digit vs carry epilogue."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24155_b200 as drzg
L = drzg.lib()
nL = int(sys.argv[1]) if len(sys.argv) > 1 else 3003
states = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
for mode in (1, 2):
    ms = ctypes.c_float()
    rc = L.drzg_bench_tc_gemm(nL, states, mode, iters, ctypes.byref(ms))
    assert rc == 0, drzg._err()
    tops = 2.0 * nL * nL * states / (ms.value / 1e3) / 1e12
    print(f"mode={'digit' if mode == 1 else 'carry'} nL={nL} states={states} ms={ms.value:.3f} TOPS={tops:.0f}", flush=True)
