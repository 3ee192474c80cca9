#!/usr/bin/env python3
"""TEST INFRASTRUCTURE: the reference bound to the B200 engine, as a
maintainer would bind it.

Writes oracle/_ref/bound/drzeta/ (git-ignored build output, like the .so
files): the reference's headers from /root/reference/proj/include/drzeta with
linalg.hpp patched so that linrec_eval (linalg.hpp:337-410) and
detail::sparse_steps (linalg.hpp:257-331) call drzg_linrec_eval /
drzg_sparse_steps through include/drzg.h.  The reference's own host bodies stay
in place under new names (unused).  oracle/Makefile then compiles the
reference's own unit tests (tests/test_linalg.cpp, test_reduction.cpp,
test_pep.cpp, read in place) against these headers and libdrzg.so, so the
reference's suites run through the device kernels.
"""
import os
import sys

REF = "/root/reference/proj/include/drzeta"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "bound", "drzeta")

LINREC_BOUND = r'''
// ---- bound to the B200 engine (INTEGRATION.md section 1) ----
// the reference's checks stay on the host; the steps run on the device
inline drzg_stripe_plan drzg_plan_of(const StripePlan& pl) {
  drzg_stripe_plan sp{};
  sp.p = pl.p;
  sp.M = pl.M;
  sp.limbs = pl.limbs;
  sp.limb_exp = pl.limb_exp;
  sp.beta = pl.beta;
  sp.stripe = pl.stripe;
  return sp;
}
inline void linrec_eval(const ModMatrix& A, const ModMatrix& B, i64 tmax,
                        ModVec& w, i64* matvec_counter = nullptr) {
  int n = A.rows;
  DRZ_REQUIRE(A.rows == A.cols && B.rows == n && B.cols == n && w.n == n,
              "linrec_eval: shape mismatch");
  DRZ_REQUIRE(tmax >= 0, "linrec_eval: negative range");
  drzg_stripe_plan sp = drzg_plan_of(A.plan);
  int64_t mv = 0;
  DRZ_REQUIRE(drzg_linrec_eval(&sp, n, A.d.data(), B.d.data(), tmax, w.d.data(), &mv) == 0,
              drzg_last_error());
  if (matvec_counter) *matvec_counter += mv;
}
'''

SPARSE_BOUND = r'''
// ---- bound to the B200 engine (INTEGRATION.md section 1) ----
inline void sparse_steps(const StripePlan& pl, const SparseOp& A,
                         const SparseOp& B, i64 tmax, ModVec& w,
                         i64* matvec_counter) {
  drzg_stripe_plan sp{};
  sp.p = pl.p;
  sp.M = pl.M;
  sp.limbs = pl.limbs;
  sp.limb_exp = pl.limb_exp;
  sp.beta = pl.beta;
  sp.stripe = pl.stripe;
  int64_t mv = 0;
  DRZ_REQUIRE(drzg_sparse_steps(&sp, A.rows, A.col_ptr.data(), A.row_idx.data(), A.digs.data(),
                                B.col_ptr.data(), B.row_idx.data(), B.digs.data(), tmax,
                                w.d.data(), &mv) == 0,
              drzg_last_error());
  if (matvec_counter) *matvec_counter += mv;
}
'''


def patch_linalg(src: str) -> str:
    a = "inline void linrec_eval(const ModMatrix& A, const ModMatrix& B, i64 tmax,"
    end_a = "\n// word-modulus product with striped"
    b = "inline void sparse_steps(const StripePlan& pl, const SparseOp& A,"
    if src.count(a) != 1 or src.count(end_a) != 1 or src.count(b) != 1:
        raise SystemExit("bind_reference: linalg.hpp anchors not found (reference changed?)")
    src = src.replace(a, "inline void linrec_eval_reference_host(const ModMatrix& A, const ModMatrix& B, i64 tmax,")
    src = src.replace(end_a, LINREC_BOUND + end_a)
    i = src.index(b)
    j = src.index("}  // namespace detail", i)
    src = src[:i] + src[i:j].replace(b, "inline void sparse_steps_reference_host(const StripePlan& pl, const SparseOp& A,") \
        + SPARSE_BOUND + src[j:]
    src = src.replace("#pragma once", "#pragma once\n#include <drzg.h>", 1)
    return src


def main():
    os.makedirs(OUT, exist_ok=True)
    for name in sorted(os.listdir(REF)):
        with open(os.path.join(REF, name)) as f:
            text = f.read()
        if name == "linalg.hpp":
            text = patch_linalg(text)
        with open(os.path.join(OUT, name), "w") as f:
            f.write(text)
    print("bound headers in", OUT)


if __name__ == "__main__":
    sys.exit(main())
