"""GPU parity: the sm_100a path against the reference, bit for bit.

Kernel level: drzg_linrec_eval / drzg_sparse_steps (reference linalg.hpp:257-410)
on the committed golden vectors.  Chunk level: drzg_reduce_chunk against the
reference reduce_chunk (reduction.hpp:394-423) run live through oracle/_ref.
Pipeline level: drzg_frobenius against the reference frobenius_matrix
(zeta.hpp:36-136): identical F, charpoly residues and cost ledger.
"""
import numpy as np
import pytest

from conftest import golden, needs_ref
import paper_2602_24155_b200 as drzg

pytestmark = pytest.mark.gpu


def _arr(xs):
    return np.array([int(x) for x in xs], dtype=np.uint64)


# the linrec_eval kernels: matrices resident in shared memory (small sides,
# default), a warp per row, the flat partition (large sides, default) and the
# flat partition forced at every side, with two-word row sums where they fit
# (default) or three
LINREC_ENVS = [{}, {"DRZG_LINREC_RESIDENT": "0"}, {"DRZG_LINREC_RESIDENT": "0", "DRZG_LINREC_FLAT": "0"},
               {"DRZG_LINREC_FLAT": "2"}, {"DRZG_LINREC_FLAT": "2", "DRZG_LINREC_N2": "0"}]
_env_id = lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default"


@pytest.mark.parametrize("env", LINREC_ENVS, ids=_env_id)
@pytest.mark.parametrize("idx", range(10))
def test_linrec_eval_matches_reference(idx, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    c = golden("linrec_cases.json")["cases"][idx]
    out, ctr = drzg.linrec_eval(c["p"], c["M"], c["side"], _arr(c["A"]), _arr(c["B"]), c["tmax"], _arr(c["w"]))
    assert (out == _arr(c["out"])).all()
    assert ctr == c["matvecs"] == c["tmax"] + 1


@pytest.mark.parametrize("idx", [0, 1, 2, 5, 6, 7, 8])
def test_sparse_steps_matches_reference(idx):
    c = golden("linrec_cases.json")["cases"][idx]
    out, _ = drzg.sparse_steps(c["p"], c["M"], c["side"], _arr(c["A"]), _arr(c["B"]), c["tmax"], _arr(c["w"]))
    assert (out == _arr(c["out"])).all()


def test_linrec_edge_cases():
    # tmax = 0 is one factor B; A = 0 gives B^{k+1} w; zero vector stays zero
    p, M, side = 11, 17, 5
    rng = np.random.default_rng(3)
    mod = p ** M
    B = np.array([int(rng.integers(0, 2**62)) % mod for _ in range(side * side)], dtype=np.uint64)
    w = np.array([int(rng.integers(0, 2**62)) % mod for _ in range(side)], dtype=np.uint64)
    out0, _ = drzg.linrec_eval(p, M, side, np.zeros_like(B), B, 0, w)
    Bo = B.astype(object).reshape(side, side)
    assert [int(x) for x in out0] == [int(x) for x in Bo.dot(w.astype(object)) % mod]
    out3, _ = drzg.linrec_eval(p, M, side, np.zeros_like(B), B, 3, w)
    ref = w.astype(object)
    for _ in range(4):
        ref = Bo.dot(ref) % mod
    assert [int(x) for x in out3] == [int(x) for x in ref]
    z, _ = drzg.linrec_eval(p, M, side, B, B, 4, np.zeros_like(w))
    assert not z.any()


@pytest.mark.parametrize("p,M,side,tmax", [
    (7, 20, 3003, 2),   # fourfold side, 1 limb: rows shared by 2-3 warps of the flat partition
    (7, 24, 3003, 1),   # fourfold side, 2 limbs
    (7, 49, 455, 3),    # 3 limbs
    (11, 17, 221, 4),   # odd side, few warps
    (13, 13, 1, 3),     # one entry
])
@pytest.mark.parametrize("env", LINREC_ENVS, ids=_env_id)
def test_linrec_eval_large_sides_match_oracle(p, M, side, tmax, env, monkeypatch):
    """every linrec_eval kernel at the BASELINE sizes against the C restatement
    of linalg.hpp:337-410 (oracle/linrec_oracle.c) on seeded inputs"""
    from oracle import refapi
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    sp = drzg.stripe_plan(p, M)
    L, beta = sp.limbs, int(sp.beta)
    top = p ** (M - sp.limb_exp * (L - 1))
    rng = np.random.default_rng(side * 1000 + M)

    def planes(n):
        x = rng.integers(0, min(beta, 2**62), size=(L, n), dtype=np.uint64)
        x[L - 1] %= np.uint64(top)
        return x.ravel()

    A, B, w = planes(side * side), planes(side * side), planes(side)
    got, ctr = drzg.linrec_eval(p, M, side, A, B, tmax, w)
    want = refapi.oracle_linrec_eval(p, M, side, A, B, tmax, w)
    assert ctr == tmax + 1
    assert (got == want).all()


CHUNK_CASES = [
    # (golden file, M, u, pole, v, k)
    ("fermat_cubic_curve_f7.json", 6, [3, 7, 7], 6, [1, 1, 1], 3),
    ("quintic_f7_s1.json", 16, [20, 20, 23], 21, [2, 1, 2], 4),
    ("quintic_f7_s1.json", 24, [20, 20, 23], 21, [2, 1, 2], 2),
    ("k3_f11_s1_r1.json", 9, [30, 20, 25, 29], 27, [1, 1, 1, 1], 5),
    ("k3_f11_s1_r1.json", 40, [30, 20, 25, 29], 27, [1, 1, 1, 1], 2),
]


@needs_ref
@pytest.mark.parametrize("case", CHUNK_CASES)
def test_reduce_chunk_matches_reference(case):
    from oracle import refapi
    name, M, u, pole, v, k = case
    g = golden(name)
    p, n, d = g["p"], g["n"], g["d"]
    sp = refapi.stripe_plan_py(p, M)
    from math import comb
    side = comb(d * n - n + n, n)
    rng = np.random.default_rng(sum(u) + M)
    mod = p ** M
    vals = [int(rng.integers(0, 2**62)) * int(rng.integers(1, 2**62)) % mod for _ in range(side)]
    w = []
    for t in range(sp["limbs"]):
        w.extend((x // sp["beta"] ** t) % sp["beta"] for x in vals)
    w = np.array(w, dtype=np.uint64)
    ref_w, ref_info = refapi.chunk(p, n, d, g["coeffs"], M, u, pole, v, k, w)
    got_w, got_u, info = drzg.reduce_chunk(p, n, d, g["coeffs"], M, u, pole, v, k, w)
    assert (got_w == ref_w).all()
    assert got_u == ref_info["u"]
    assert info["matvecs"] == ref_info["matvecs"] == k


FROB_CASES = ["fermat_cubic_curve_f7.json", "random_cubic_curve_f11_s3.json", "random_quartic_curve_f7_s2.json",
              "quintic_f7_s1.json", "fermat_quartic_surface_f7.json", "k3_f11_s1_r1.json",
              "quintic_surface_f7_s1_r1.json", "threefold_f13_s1_r1.json", "fermat_fourfold_f7_r1.json",
              "k3_f11_s1.json", "threefold_f13_s1.json"]


@pytest.mark.parametrize("name", FROB_CASES)
def test_frobenius_matrix_matches_reference(name):
    try:
        g = golden(name)
    except FileNotFoundError:
        pytest.skip("fixture not generated")
    fr = drzg.frobenius(g["p"], g["n"], g["d"], g["coeffs"], r_uniform=g["r_uniform"], nm=g["nm_override"])
    assert fr["plan"]["M"] == g["plan"]["M"]
    assert fr["F"] == g["F"]
    assert fr["charpoly"] == g["charpoly"]
    assert fr["matvecs"] == g["ledger"]["matvecs"]
    assert fr["startups"] == g["ledger"]["startups"]
    assert fr["combines"] == g["ledger"]["combines"]


@pytest.mark.parametrize("name", ["fermat_cubic_curve_f7.json", "quintic_f7_s1.json", "random_quartic_curve_f7_s2.json",
                                  "k3_f11_s1.json", "threefold_f13_s1.json"])
def test_zeta_matches_reference(name):
    g = golden(name)
    z = drzg.zeta(g["p"], g["n"], g["d"], g["coeffs"])
    assert [z["Q"]] == g["Q_candidates"][:1]
    assert all(ok for (_, _, ok) in z["counts"])


# Every device path gives the same bits: the one-launch small-system kernel at
# all three block widths, the dataflow kernel, the separate digit/carry launches
# with dense or block-sparse carry, and the dp4a CUDA-core fallback.  The
# switches are read when the engine is built (once per call).
PATH_ENVS = [
    {"DRZG_FUSED_NS": "32"},
    {"DRZG_FUSED_NS": "64"},
    {"DRZG_FUSED_NS": "128"},
    {"DRZG_FUSED_PP": "0"},          # one block per CTA in the large one-launch solves
    {"DRZG_CHUNK": "1"},             # whole chunks in one launch, T_x in the CTA
    {"DRZG_FLOW2": "0"},             # the single-CTA dataflow kernel
    {"DRZG_FUSED": "0", "DRZG_FLOW": "0"},
    {"DRZG_FUSED": "0", "DRZG_FLOW": "0", "DRZG_SPARSE_CARRY": "0"},
    {"DRZG_GEMM": "dp4a"},
]


@pytest.mark.parametrize("env", PATH_ENVS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
@pytest.mark.parametrize("name", ["k3_f11_s1_r1.json", "threefold_f13_s1_r1.json", "quintic_f7_s1.json"])
def test_device_paths_agree(name, env, monkeypatch):
    g = golden(name)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    fr = drzg.frobenius(g["p"], g["n"], g["d"], g["coeffs"], r_uniform=g["r_uniform"], nm=g["nm_override"])
    assert fr["F"] == g["F"]
    assert fr["matvecs"] == g["ledger"]["matvecs"]


# The random quintic surface at its default plan (configs[2]: M = 49, 25
# balanced base-49 digit planes, 52 columns, 0.91e9 matvecs) is beyond the
# reference here.  Pinned instead by: the reference's own cost
# ledger at this plan from the value-free replay (scripts/replay_ledger.py;
# the replay equals the real reference ledger on every fixture,
# tests/test_oracle.py), the brute-force point counts #X(F_7) and #X(F_49)
# that run_zeta verifies against Q (reference zeta.hpp:510-525) and the
# Hodge-polygon bound.  This is also the one end-to-end case with more than
# 24 digit planes.
def test_quintic_surface_default_plan_counts():
    co = drzg.random_hypersurface(7, 3, 5, 1)
    ref = golden("ledger_replay_quintic_surface.json")
    assert co == [int(x) for x in ref["coeffs"]]
    z = drzg.zeta(7, 3, 5, co)
    assert z["plan"]["M"] == 49 and z["frobenius"]["digits"]["Ld"] == 25
    assert [c[0] for c in z["counts"]] == [1, 2] and all(ok for (_, _, ok) in z["counts"])
    assert z["slopes"] == [["0", 4], ["1", 44], ["2", 4]]
    fr = z["frobenius"]
    assert (fr["matvecs"], fr["startups"], fr["combines"]) == (
        ref["ledger"]["matvecs"], ref["ledger"]["startups"], ref["ledger"]["combines"])
