import ctypes, sys
sys.path.insert(0, '.')
import paper_2602_24155_b200 as D
L = D.lib()
for (p, n, d, M) in [(7, 5, 3, 7), (7, 5, 3, 24)]:
    co = D.random_hypersurface(p, n, d, 1)
    diff = ctypes.c_int64(-1)
    rc = L.drzg_test_tables(ctypes.c_uint64(p), n, d, D._u64arr(co), M, ctypes.byref(diff))
    print(p, n, d, M, rc, D._err() if rc else "", diff.value, flush=True)
for (p, n, d, M) in [(7, 5, 3, 24), (11, 3, 4, 17)]:
    co = D.random_hypersurface(p, n, d, 1)
    diff = ctypes.c_int64(-1)
    rc = L.drzg_test_final_levels(ctypes.c_uint64(p), n, d, D._u64arr(co), M, ctypes.byref(diff))
    print("final", p, n, d, M, rc, D._err() if rc else "", diff.value, flush=True)
