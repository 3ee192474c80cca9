"""drzg: B200-native controlled-reduction engine (arXiv 2602.24155).

Python view of the C ABI in include/drzg.h (libdrzg.so, built in-tree by
`make -C paper_2602_24155_b200/csrc`).  The names and argument meanings mirror
the reference's C++ entry points (drzeta: linrec_eval, detail::sparse_steps,
reduce_chunk, frobenius_matrix, run_zeta).  There is no CPU fallback: if the
library is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DRZG_LIB") or os.path.join(_HERE, "libdrzg.so")
POLICIES = {"p-chunk": 0, "pchunk": 0, "depth-first": 1, "depth": 1, "var-by-var": 2, "varbyvar": 2}

_lib = None


class DrzgError(RuntimeError):
    """contract_error / singular_input / escalation_exhausted from the engine"""


class StripePlan(ctypes.Structure):
    """StripePlan (reference linalg.hpp:20-58)"""
    _fields_ = [("p", ctypes.c_uint64), ("M", ctypes.c_int32), ("limbs", ctypes.c_int32),
                ("limb_exp", ctypes.c_int32), ("pad_", ctypes.c_int32), ("beta", ctypes.c_uint64),
                ("stripe", ctypes.c_int64)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DrzgError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc`")
        L = ctypes.CDLL(LIB_PATH)
        L.drzg_last_error.restype = ctypes.c_char_p
        for name in ("drzg_zeta", "drzg_frobenius", "drzg_reduce_chunk", "drzg_charpoly", "drzg_zeta_from_F"):
            getattr(L, name).restype = ctypes.c_void_p
        _lib = L
    return _lib


def _err():
    return lib().drzg_last_error().decode()


def _check(rc):
    if rc != 0:
        raise DrzgError(_err())


def _json(ptr):
    if not ptr:
        raise DrzgError(_err())
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    lib().drzg_free(ctypes.c_void_p(ptr))
    return json.loads(s)


def _u64arr(xs):
    return (ctypes.c_uint64 * len(xs))(*[int(x) for x in xs])


_P64 = ctypes.POINTER(ctypes.c_uint64)


def device_count():
    return lib().drzg_device_count()


def stripe_plan(p, M):
    sp = StripePlan()
    _check(lib().drzg_stripe_plan_make(ctypes.c_uint64(p), M, ctypes.byref(sp)))
    return sp


def linrec_eval(p, M, side, A, B, tmax, w):
    """reference linrec_eval (linalg.hpp:337-410) on the GPU; A, B, w in the
    reference's plane-major base-beta layout; returns (w_out, matvecs)"""
    sp = stripe_plan(p, M)
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    w = np.array(w, dtype=np.uint64, copy=True)
    ctr = ctypes.c_int64(0)
    _check(lib().drzg_linrec_eval(ctypes.byref(sp), side, A.ctypes.data_as(_P64), B.ctypes.data_as(_P64),
                                  ctypes.c_int64(tmax), w.ctypes.data_as(_P64), ctypes.byref(ctr)))
    return w, ctr.value


def linrec_eval_device(p, M, side, dA_ptr, dB_ptr, tmax, dw_ptr, stream_ptr=0, timed=False):
    """device-pointer variant (torch tensors' data_ptr()); returns kernel ms if timed"""
    sp = stripe_plan(p, M)
    ctr = ctypes.c_int64(0)
    ms = ctypes.c_float(0.0)
    _check(lib().drzg_linrec_eval_device(ctypes.byref(sp), side, ctypes.c_void_p(dA_ptr), ctypes.c_void_p(dB_ptr),
                                         ctypes.c_int64(tmax), ctypes.c_void_p(dw_ptr), ctypes.byref(ctr),
                                         ctypes.c_void_p(stream_ptr), ctypes.byref(ms) if timed else None))
    return ms.value if timed else None


def sparse_steps(p, M, side, A, B, tmax, w):
    """reference detail::sparse_steps (linalg.hpp:257-331): A, B given dense in
    plane layout are compressed to the reference's SparseOp CSC (linalg.hpp:227-251)"""
    sp = stripe_plan(p, M)
    L = sp.limbs

    def csc(X):
        X = np.asarray(X, dtype=np.uint64).reshape(L, side, side)
        nz = (X != 0).any(axis=0)  # rows x cols
        col_ptr = [0]
        rows, digs = [], []
        for j in range(side):
            idx = np.nonzero(nz[:, j])[0]
            rows.extend(idx.tolist())
            for i in idx:
                digs.extend(int(X[t, i, j]) for t in range(L))
            col_ptr.append(len(rows))
        return (np.array(col_ptr, dtype=np.int64), np.array(rows, dtype=np.int32), np.array(digs, dtype=np.uint64))

    (ac, ar, ad), (bc, br, bd) = csc(A), csc(B)
    w = np.array(w, dtype=np.uint64, copy=True)
    ctr = ctypes.c_int64(0)
    P64i = ctypes.POINTER(ctypes.c_int64)
    P32 = ctypes.POINTER(ctypes.c_int32)
    _check(lib().drzg_sparse_steps(ctypes.byref(sp), side,
                                   ac.ctypes.data_as(P64i), ar.ctypes.data_as(P32), ad.ctypes.data_as(_P64),
                                   bc.ctypes.data_as(P64i), br.ctypes.data_as(P32), bd.ctypes.data_as(_P64),
                                   ctypes.c_int64(tmax), w.ctypes.data_as(_P64), ctypes.byref(ctr)))
    return w, ctr.value


def reduce_chunk(p, n, d, coeffs, M, u, pole, v, k, w, device=0):
    """reference reduce_chunk (reduction.hpp:394-423) for one state; returns
    (w_out, u_out, info)"""
    w = np.array(w, dtype=np.uint64, copy=True)
    ua = (ctypes.c_int32 * (n + 1))(*u)
    va = (ctypes.c_int32 * (n + 1))(*v)
    info = _json(lib().drzg_reduce_chunk(ctypes.c_uint64(p), n, d, _u64arr(coeffs), M, ua, pole, va,
                                         ctypes.c_int64(k), w.ctypes.data_as(_P64), device))
    return w, list(ua), info


def frobenius(p, n, d, coeffs, policy="p-chunk", r_uniform=0, nm=0, only_pole=0, columns=None, device=0,
              profile=False):
    """reference frobenius_matrix (zeta.hpp:36-136)"""
    cols = None
    ncols = 0
    if columns is not None:
        cols = (ctypes.c_int32 * len(columns))(*columns)
        ncols = len(columns)
    return _json(lib().drzg_frobenius(ctypes.c_uint64(p), n, d, _u64arr(coeffs), POLICIES[policy], r_uniform, nm,
                                      only_pole, cols, ncols, device, int(profile)))


def zeta(p, n, d, coeffs, policy="p-chunk", r_uniform=0, nm=0, verify_counts=True, device=0, profile=False,
         count_budget=0):
    """reference run_zeta (zeta.hpp:438-549); count_budget <= 0 keeps the
    reference's 2e8-point budget for the brute-force count checks"""
    return _json(lib().drzg_zeta(ctypes.c_uint64(p), n, d, _u64arr(coeffs), POLICIES[policy], r_uniform, nm,
                                 int(verify_counts), ctypes.c_int64(count_budget), device, int(profile)))


def zeta_batch(p, n, d, coeffs_list, workers=4, device=0, **kw):
    """zeta functions of many hypersurfaces over one field (BASELINE configs[3]:
    64 cubic threefolds), `workers` at a time on one device: each call runs on
    its own host thread and stream (ctypes releases the GIL), so one
    hypersurface's host phases and small kernels overlap another's device
    work; the dataflow kernels take turns (kernels/tc_gemm.cu gated launch).
    Returns the results in input order."""
    from concurrent.futures import ThreadPoolExecutor
    if workers <= 1 or len(coeffs_list) <= 1:
        return [zeta(p, n, d, co, device=device, **kw) for co in coeffs_list]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(lambda co: zeta(p, n, d, co, device=device, **kw), coeffs_list))


def zeta_from_F(p, n, d, coeffs, F, b, r_uniform=0, nm=0, escalations=0, verify_counts=True, count_budget=0):
    """run_zeta's battery (zeta.hpp:456-535) on a given F, e.g. one gathered
    from several GPUs: {"status": "ok", "Q": ...} or {"status": "escalate"}"""
    arr = (ctypes.c_char_p * (b * b))(*[str(x).encode() for x in F])
    return _json(lib().drzg_zeta_from_F(ctypes.c_uint64(p), n, d, _u64arr(coeffs), r_uniform, nm, escalations, b, arr,
                                        int(verify_counts), ctypes.c_int64(count_budget)))


def random_hypersurface(p, n, d, seed=1, policy="p-chunk", fermat=False):
    """reference generator rule (drzeta_main.cpp:112-122 + run_zeta's smoothness checks)"""
    from math import comb
    cnt = comb(n + d, n)
    out = (ctypes.c_uint64 * cnt)()
    tries = ctypes.c_int32(0)
    _check(lib().drzg_random_hypersurface(ctypes.c_uint64(p), n, d, ctypes.c_uint64(seed), POLICIES[policy],
                                          int(fermat), out, ctypes.byref(tries)))
    return [int(x) for x in out]


def fsplit(p, n, d, coeffs):
    """Fedder's F-splitting criterion as run_zeta reports it (zeta.hpp:336-350):
    True / False, or None where it is undefined (d > n + 1)"""
    out = ctypes.c_int32()
    _check(lib().drzg_fsplit(ctypes.c_uint64(p), n, d, _u64arr(coeffs), ctypes.byref(out)))
    return None if out.value < 0 else bool(out.value)


def count_points(p, n, d, coeffs, r, budget=200_000_000):
    """brute-force #X(F_{p^r}) (reference oracle.hpp:190-245)"""
    out = ctypes.c_int64()
    _check(lib().drzg_count_points(ctypes.c_uint64(p), n, d, _u64arr(coeffs), r, ctypes.c_int64(budget),
                                   ctypes.byref(out)))
    return out.value


def count_points_device(p, n, d, coeffs, r, budget=200_000_000):
    """the GPU point count (kernels/count.cu)"""
    out = ctypes.c_int64()
    _check(lib().drzg_count_points_device(ctypes.c_uint64(p), n, d, _u64arr(coeffs), r, ctypes.c_int64(budget),
                                          ctypes.byref(out)))
    return out.value


def charpoly(p, n, d, F, b, r_uniform=0, nm=0):
    """berkowitz_charpoly + recover_Q on a given F (zeta.hpp:456-470)"""
    arr = (ctypes.c_char_p * (b * b))(*[str(x).encode() for x in F])
    return _json(lib().drzg_charpoly(ctypes.c_uint64(p), n, d, r_uniform, nm, b, arr))


def test_tc_gemm(A, B, a_unsigned=False):
    """D = A . B^T through the tcgen05 int8 kernel (test hook); A: M x K, B: N x K"""
    A = np.ascontiguousarray(A, dtype=np.uint8 if a_unsigned else np.int8)
    B = np.ascontiguousarray(B, dtype=np.int8)
    M, K = A.shape
    N = B.shape[0]
    D = np.zeros((N, M), dtype=np.int32)
    _check(lib().drzg_test_tc_gemm(M, N, K, A.ctypes.data_as(ctypes.c_void_p), B.ctypes.data_as(ctypes.c_void_p),
                                   D.ctypes.data_as(ctypes.c_void_p), int(a_unsigned)))
    return D


def test_tc_gemm_mn(A, B, a_unsigned=False):
    """as test_tc_gemm, with B staged K x N (MN-major operand)"""
    A = np.ascontiguousarray(A, dtype=np.uint8 if a_unsigned else np.int8)
    B = np.ascontiguousarray(B, dtype=np.int8)
    M, K = A.shape
    N = B.shape[0]
    D = np.zeros((N, M), dtype=np.int32)
    _check(lib().drzg_test_tc_gemm_mn(M, N, K, A.ctypes.data_as(ctypes.c_void_p), B.ctypes.data_as(ctypes.c_void_p),
                                      D.ctypes.data_as(ctypes.c_void_p), int(a_unsigned)))
    return D


class Context:
    """the reduction-policy interface on device-resident GameStates (drzg_ctx:
    the reference's RuvContext + PepStoreBase of one (f, S, p^M) run,
    reduction.hpp:143-242).  States are ids; w crosses in ModVec layout."""

    def __init__(self, p, n, d, coeffs, M, policy="p-chunk", device=0):
        L = lib()
        L.drzg_ctx_create.restype = ctypes.c_void_p
        self.n, self.nv = n, n + 1
        self.h = L.drzg_ctx_create(ctypes.c_uint64(p), n, d, _u64arr(coeffs), M, POLICIES[policy], device)
        if not self.h:
            raise DrzgError(_err())
        side, fl, q, Ld = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        sp = StripePlan()
        _check(L.drzg_ctx_info(ctypes.c_void_p(self.h), ctypes.byref(side), ctypes.byref(fl), ctypes.byref(sp),
                               ctypes.byref(q), ctypes.byref(Ld)))
        self.side, self.floor_len, self.plan, self.q, self.Ld = side.value, fl.value, sp, q.value, Ld.value
        self.ledger = [0, 0, 0]

    def close(self):
        if self.h:
            lib().drzg_ctx_free(ctypes.c_void_p(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ids(self, ids):
        return (ctypes.c_int32 * len(ids))(*ids)

    def _led(self, arr):
        for i in range(3):
            self.ledger[i] += arr[i]

    def seed(self, u, pole, w):
        """GameStates in: u (count x nv), pole (count), w (count x limbs*side)"""
        count = len(pole)
        w = np.ascontiguousarray(w, dtype=np.uint64).reshape(count, -1)
        out = (ctypes.c_int32 * count)()
        _check(lib().drzg_states_seed(ctypes.c_void_p(self.h), count, (ctypes.c_int32 * (count * self.nv))(
            *[int(x) for row in u for x in row]), (ctypes.c_int32 * count)(*pole), w.ctypes.data_as(_P64), out))
        return list(out)

    def read(self, ids):
        count = len(ids)
        u = (ctypes.c_int32 * (count * self.nv))()
        pole = (ctypes.c_int32 * count)()
        w = np.zeros((count, self.plan.limbs * self.side), dtype=np.uint64)
        _check(lib().drzg_states_read(ctypes.c_void_p(self.h), count, self._ids(ids), u, pole,
                                      w.ctypes.data_as(_P64)))
        return [list(u[i * self.nv:(i + 1) * self.nv]) for i in range(count)], list(pole), w

    def free(self, ids):
        _check(lib().drzg_states_free(ctypes.c_void_p(self.h), len(ids), self._ids(ids)))

    def step(self, ids, v, k):
        """reduce_chunk for each state: v (count x nv), k (count)"""
        count = len(ids)
        led = (ctypes.c_int64 * 3)()
        _check(lib().drzg_step_batch(ctypes.c_void_p(self.h), count, self._ids(ids),
                                     (ctypes.c_int32 * (count * self.nv))(*[int(x) for row in v for x in row]),
                                     (ctypes.c_int64 * count)(*k), led))
        self._led(led)

    def combine(self, ids):
        out = (ctypes.c_int32 * max(1, len(ids)))()
        cnt = ctypes.c_int32()
        led = (ctypes.c_int64 * 3)()
        _check(lib().drzg_states_combine(ctypes.c_void_p(self.h), len(ids), self._ids(ids), out, ctypes.byref(cnt),
                                         led))
        self._led(led)
        return list(out[:cnt.value])

    def run_policy(self, ids, policy="p-chunk"):
        out = (ctypes.c_int32 * max(1, len(ids)))()
        cnt = ctypes.c_int32()
        led = (ctypes.c_int64 * 3)()
        _check(lib().drzg_run_policy(ctypes.c_void_p(self.h), len(ids), self._ids(ids), POLICIES[policy], out,
                                     ctypes.byref(cnt), led))
        self._led(led)
        return list(out[:cnt.value])

    def floor_numerator(self, ids, g=None):
        if g is None:
            g = np.zeros(self.plan.limbs * self.floor_len, dtype=np.uint64)
        g = np.ascontiguousarray(g, dtype=np.uint64).copy()
        _check(lib().drzg_floor_accumulate(ctypes.c_void_p(self.h), len(ids), self._ids(ids), g.ctypes.data_as(_P64)))
        return g


class PepStore:
    """PepStoreBase over a Context (reference reduction.hpp:143-147, pep.hpp:
    15-209): spec "eager", "lazy", "lru:N" or "lfuda:N".  get(v) returns the
    n+2 matrices of build_ruv(C, v) as ((n+2), limbs, side, side) u64 planes."""

    def __init__(self, ctx, spec, _stub=None):
        L = lib()
        L.drzg_pep_store_create.restype = ctypes.c_void_p
        L.drzg_pep_store_create_stub.restype = ctypes.c_void_p
        self.ctx = ctx
        if _stub is not None:
            nv, d = _stub
            self.h = L.drzg_pep_store_create_stub(nv, d, spec.encode())
            self.nv = nv
        else:
            self.h = L.drzg_pep_store_create(ctypes.c_void_p(ctx.h), spec.encode())
            self.nv = ctx.nv
        if not self.h:
            raise DrzgError(_err())

    @classmethod
    def stub(cls, nv, d, spec):
        """bookkeeping-only store (no device): entries are placeholders"""
        return cls(None, spec, _stub=(nv, d))

    def close(self):
        if self.h:
            lib().drzg_pep_store_free(ctypes.c_void_p(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def get(self, v, planes=True):
        va = (ctypes.c_int32 * self.nv)(*v)
        nnz = ctypes.c_int64()
        out = None
        if planes and self.ctx is not None:
            c = self.ctx
            out = np.zeros((self.nv + 1, c.plan.limbs, c.side, c.side), dtype=np.uint64)
            _check(lib().drzg_pep_get(ctypes.c_void_p(self.h), va, out.ctypes.data_as(_P64), ctypes.byref(nnz)))
        else:
            _check(lib().drzg_pep_get(ctypes.c_void_p(self.h), va, None, ctypes.byref(nnz)))
        return out, nnz.value

    def stats(self):
        h, m, e = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().drzg_pep_stats(ctypes.c_void_p(self.h), ctypes.byref(h), ctypes.byref(m), ctypes.byref(e)))
        return {"hits": h.value, "misses": m.value, "evictions": e.value}

    def eval_to_linear(self, v, x):
        """reference eval_to_linear(E, x, v, plan): (A, B) in ModMatrix layout"""
        c = self.ctx
        A = np.zeros(c.plan.limbs * c.side * c.side, dtype=np.uint64)
        B = np.zeros_like(A)
        _check(lib().drzg_pep_eval_to_linear(ctypes.c_void_p(self.h), (ctypes.c_int32 * self.nv)(*v),
                                             (ctypes.c_int32 * self.nv)(*x), A.ctypes.data_as(_P64),
                                             B.ctypes.data_as(_P64)))
        return A, B
