"""TEST INFRASTRUCTURE ONLY: ctypes view of oracle/_ref/libdrz_ref.so.

The library is the UNMODIFIED reference (drzeta headers) behind the C entry
points of oracle/ref_capi.cpp.  Only tests/, scripts/make_golden.py,
__graft_entry__.smoke() and bench.py's CPU-baseline leg import this module;
the product (paper_2602_24155_b200) never does.
"""
from __future__ import annotations

import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libdrz_ref.so")
ORACLE_SO = os.path.join(_HERE, "_ref", "liboracle.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
        L = ctypes.CDLL(REF_SO)
        for name in ("ref_run_policy_states", "ref_replay_ledger", "ref_mono_table", "ref_hypersurface", "ref_plan", "ref_basis", "ref_seeds",
                     "ref_chunk", "ref_frobenius", "ref_zeta", "ref_charpoly", "ref_policy_sample"):
            getattr(L, name).restype = ctypes.c_void_p
        _lib = L
    return _lib


def _js(ptr):
    L = lib()
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    L.ref_free(ctypes.c_void_p(ptr))
    out = json.loads(s)
    if isinstance(out, dict) and "error" in out:
        raise RuntimeError("reference: " + out["error"])
    return out


def _u64(xs):
    return (ctypes.c_uint64 * len(xs))(*[int(x) for x in xs])


def _i32(xs):
    return (ctypes.c_int * len(xs))(*[int(x) for x in xs])


def stripe_plan(p, M):
    limbs, e, beta, stripe = ctypes.c_int(), ctypes.c_int(), ctypes.c_uint64(), ctypes.c_long()
    rc = lib().ref_stripe_plan(ctypes.c_uint64(p), M, ctypes.byref(limbs), ctypes.byref(e),
                               ctypes.byref(beta), ctypes.byref(stripe))
    if rc:
        raise RuntimeError("StripePlan::make failed")
    return {"limbs": limbs.value, "limb_exp": e.value, "beta": beta.value, "stripe": stripe.value}


def _vec_call(fn, p, M, side, A, B, tmax, w):
    import numpy as np
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    w = np.array(w, dtype=np.uint64, copy=True)
    ctr = ctypes.c_long()
    P = ctypes.POINTER(ctypes.c_uint64)
    rc = fn(ctypes.c_uint64(p), M, side, A.ctypes.data_as(P), B.ctypes.data_as(P), ctypes.c_long(tmax),
            w.ctypes.data_as(P), ctypes.byref(ctr))
    if rc:
        raise RuntimeError("reference kernel raised")
    return w, ctr.value


def linrec_eval(p, M, side, A, B, tmax, w):
    """reference linrec_eval (linalg.hpp:337-410); arrays in plane-major layout"""
    return _vec_call(lib().ref_linrec_eval, p, M, side, A, B, tmax, w)


def sparse_steps(p, M, side, A, B, tmax, w):
    """reference detail::sparse_steps (linalg.hpp:257-331) on SparseOp::build(A), (B)"""
    return _vec_call(lib().ref_sparse_steps, p, M, side, A, B, tmax, w)


def mono_table(nv, deg):
    return _js(lib().ref_mono_table(nv, deg))["mons"]


def fsplit(p, n, d, coeffs):
    """the reference's fedder_is_fsplit (zeta.hpp:336-350); None where
    run_zeta leaves it undefined (d > n + 1)"""
    v = lib().ref_fsplit(ctypes.c_uint64(p), n, d, _u64(coeffs))
    return None if v < 0 else bool(v)


def hypersurface(p, n, d, seed=1, mode="random", policy="p-chunk"):
    return _js(lib().ref_hypersurface(ctypes.c_uint64(p), n, d, ctypes.c_uint64(seed), mode.encode(),
                                      policy.encode()))["coeffs"]


def plan(p, n, d, r_uniform=0, nm=0):
    return _js(lib().ref_plan(ctypes.c_uint64(p), n, d, r_uniform, nm))


def basis(p, n, d, coeffs):
    return _js(lib().ref_basis(ctypes.c_uint64(p), n, d, _u64(coeffs)))


def seeds(p, n, d, coeffs, col, r_uniform=0, nm=0):
    return _js(lib().ref_seeds(ctypes.c_uint64(p), n, d, _u64(coeffs), r_uniform, nm, col))


def chunk(p, n, d, coeffs, M, u, pole, v, k, w_in):
    import numpy as np
    w_in = np.ascontiguousarray(w_in, dtype=np.uint64)
    w_out = np.zeros_like(w_in)
    P = ctypes.POINTER(ctypes.c_uint64)
    res = _js(lib().ref_chunk(ctypes.c_uint64(p), n, d, _u64(coeffs), M, _i32(u), pole, _i32(v),
                              ctypes.c_long(k), w_in.ctypes.data_as(P), w_out.ctypes.data_as(P)))
    return w_out, res


def frobenius(p, n, d, coeffs, policy="p-chunk", pep="lazy", threads=1, r_uniform=0, nm=0, only_pole=0):
    return _js(lib().ref_frobenius(ctypes.c_uint64(p), n, d, _u64(coeffs), policy.encode(), pep.encode(),
                                   threads, r_uniform, nm, only_pole))


def zeta(p, n, d, coeffs, policy="p-chunk", pep="lazy", threads=1, r_uniform=0, nm=0, verify_counts=True):
    return _js(lib().ref_zeta(ctypes.c_uint64(p), n, d, _u64(coeffs), policy.encode(), pep.encode(),
                              threads, r_uniform, nm, int(verify_counts)))


def charpoly(p, n, d, F, b, r_uniform=0, nm=0):
    arr = (ctypes.c_char_p * (b * b))(*[str(x).encode() for x in F])
    return _js(lib().ref_charpoly(ctypes.c_uint64(p), n, d, r_uniform, nm, b, arr))


_olib = None


def oracle_lib():
    """the plain-C restatement (oracle/linrec_oracle.c)"""
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        _olib = ctypes.CDLL(ORACLE_SO)
    return _olib


def oracle_linrec_eval(p, M, side, A, B, tmax, w):
    import numpy as np
    pl = stripe_plan_py(p, M)
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    w = np.array(w, dtype=np.uint64, copy=True)
    P = ctypes.POINTER(ctypes.c_uint64)
    rc = oracle_lib().oracle_linrec_eval(ctypes.c_uint64(p), M, pl["limbs"], pl["limb_exp"], ctypes.c_uint64(pl["beta"]),
                                         side, A.ctypes.data_as(P), B.ctypes.data_as(P), ctypes.c_int64(tmax),
                                         w.ctypes.data_as(P))
    if rc:
        raise RuntimeError("oracle_linrec_eval failed")
    return w


def stripe_plan_py(p, M, capacity=1 << 126):
    """StripePlan::make restated (linalg.hpp:35-58)"""
    for limbs in range(1, 65):
        e = (M + limbs - 1) // limbs
        if p ** e > (1 << 62):
            continue
        beta = p ** e
        prod = (beta - 1) ** 2
        if prod > capacity // limbs:
            continue
        return {"limbs": limbs, "limb_exp": e, "beta": beta, "stripe": min(capacity // (prod * limbs), 1 << 40)}
    raise ValueError("StripePlan: no viable limb split")


def policy_sample(p, n, d, coeffs, col, max_seeds, threads, r_uniform=0, nm=0):
    """reference run_policy on a bounded sample of one column's top-pole seeds"""
    return _js(lib().ref_policy_sample(ctypes.c_uint64(p), n, d, _u64(coeffs), r_uniform, nm, col, max_seeds,
                                       threads))


def replay_ledger(p, n, d, coeffs, r_uniform=0, nm=0, threads=4):
    """the reference's frobenius_matrix cost ledger by value-free replay
    (matvecs, startups, combines, per column); equals the real run's ledger"""
    return _js(lib().ref_replay_ledger(ctypes.c_uint64(p), n, d, _u64(coeffs), r_uniform, nm, threads))


def run_policy_states(p, n, d, coeffs, M, policy, u, pole, w):
    """reference run_policy on given GameStates (u: count x nv, pole: count, w:
    count x limbs*side ModVec digits) + floor_to_numerator of the floor states"""
    import numpy as np
    count = len(pole)
    ua = _i32([x for row in u for x in row])
    pa = _i32(pole)
    w = np.ascontiguousarray(w, dtype=np.uint64)
    return _js(lib().ref_run_policy_states(ctypes.c_uint64(p), n, d, _u64(coeffs), M, policy.encode(), count, ua, pa,
                                           w.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))


def build_ruv(p, n, d, coeffs, M, v, policy="p-chunk"):
    """reference build_ruv(C, v): (n+2) x limbs x side x side u64 planes, nnz"""
    import numpy as np
    from math import comb
    sp = stripe_plan_py(p, M)
    side = comb(d * n - n + n, n)
    out = np.zeros((n + 2) * sp["limbs"] * side * side, dtype=np.uint64)
    nnz = ctypes.c_long()
    rc = lib().ref_build_ruv(ctypes.c_uint64(p), n, d, _u64(coeffs), M, policy.encode(), _i32(v),
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(nnz))
    if rc:
        raise RuntimeError("reference build_ruv raised")
    return out, nnz.value
