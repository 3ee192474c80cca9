"""GPU: the reduction-policy interface (reference reduction.hpp:394-581).

* frobenius_matrix under the depth-first and var-by-var policies gives the
  reference's F and the reference's own ledger for that policy (fixtures made
  by scripts/make_golden.py with the policy argument);
* the states-level C ABI (drzg_ctx, drzg_states_*, drzg_step_batch,
  drzg_run_policy, drzg_floor_accumulate) against the reference's run_policy
  and floor_to_numerator on the same GameStates (live, through oracle/_ref).
"""
import os

import numpy as np
import pytest

from conftest import GOLD, golden, needs_ref
import paper_2602_24155_b200 as drzg

pytestmark = pytest.mark.gpu

POLICY_CASES = ["quintic_f7_s1_depth.json", "quintic_f7_s1_vbv.json", "k3_f11_s1_r1_depth.json",
                "k3_f11_s1_r1_vbv.json", "threefold_f13_s1_r1_vbv.json"]


@pytest.mark.parametrize("name", POLICY_CASES)
def test_policy_frobenius_matches_reference(name):
    if not os.path.exists(os.path.join(GOLD, name)):
        pytest.skip("fixture not generated")
    g = golden(name)
    fr = drzg.frobenius(g["p"], g["n"], g["d"], g["coeffs"], policy=g["policy"], r_uniform=g["r_uniform"],
                        nm=g["nm_override"])
    assert fr["F"] == g["F"]
    assert fr["charpoly"] == g["charpoly"]
    assert (fr["matvecs"], fr["startups"], fr["combines"]) == (
        g["ledger"]["matvecs"], g["ledger"]["startups"], g["ledger"]["combines"])


def _seed_states(p, n, d, coeffs, col, limit, r_uniform=0, nm=0):
    """a column's first seeds as GameStates (reference seed_reduction_input)"""
    from oracle import refapi
    s = refapi.seeds(p, n, d, coeffs, col, r_uniform=r_uniform, nm=nm)
    plan = refapi.plan(p, n, d, r_uniform=r_uniform, nm=nm)
    sp = refapi.stripe_plan_py(p, plan["M"])
    from math import comb
    side = comb(d * n - n + n, n)
    terms = s["terms"][:limit]
    u = [t["u"] for t in terms]
    pole = [t["P"] for t in terms]
    w = np.zeros((len(terms), sp["limbs"] * side), dtype=np.uint64)
    for i, t in enumerate(terms):
        val = int(t["val"])
        for j in range(sp["limbs"]):
            w[i, j * side + t["g"]] = (val // sp["beta"] ** j) % sp["beta"]
    return plan["M"], u, pole, w


STATE_CASES = [
    ("quintic_f7_s1.json", 5, 400, "p-chunk"),
    ("quintic_f7_s1.json", 5, 120, "depth-first"),
    ("k3_f11_s1_r1.json", 10, 300, "p-chunk"),
    ("random_quartic_curve_f7_s2.json", 3, 200, "p-chunk"),
]


@needs_ref
@pytest.mark.parametrize("case", STATE_CASES, ids=lambda c: f"{c[0]}-col{c[1]}-{c[3]}")
def test_run_policy_states_match_reference(case):
    from oracle import refapi
    name, col, limit, policy = case
    g = golden(name)
    p, n, d = g["p"], g["n"], g["d"]
    M, u, pole, w = _seed_states(p, n, d, g["coeffs"], col, limit, g["r_uniform"], g["nm_override"])
    ref = refapi.run_policy_states(p, n, d, g["coeffs"], M, policy, u, pole, w)
    ctx = drzg.Context(p, n, d, g["coeffs"], M, policy=policy)
    ids = ctx.seed(u, pole, w)
    # round trip of the uploaded states
    u2, p2, w2 = ctx.read(ids)
    assert u2 == u and p2 == pole and (w2 == w).all()
    fl = ctx.run_policy(ids, policy)
    assert ctx.ledger == [ref["matvecs"], ref["startups"], ref["combines"]]
    fu, fp, fw = ctx.read(fl)
    got = sorted((tuple(a), b, tuple(int(x) for x in c)) for a, b, c in zip(fu, fp, fw))
    exp = sorted((tuple(s["u"]), s["pole"], tuple(int(x) for x in s["w"])) for s in ref["states"])
    assert got == exp
    gnum = ctx.floor_numerator(fl)
    sp = ctx.plan
    vals = [sum(int(gnum[t * ctx.floor_len + r]) * int(sp.beta) ** t for t in range(sp.limbs))
            for r in range(ctx.floor_len)]
    assert vals == [int(x) for x in ref["g"]]
    ctx.close()


def _greedy_v(d, u, S):
    """choose_v_greedy (reduction.hpp:71-91)"""
    nv = len(u)
    v = [0] * nv
    placed = 0
    for s in sorted(S):
        if u[s] != 0 and placed < d:
            v[s] = 1
            placed += 1
    m = idle = 0
    while placed < d and idle < nv:
        if v[m] < u[m]:
            v[m] += 1
            placed += 1
            idle = 0
        else:
            idle += 1
        m = (m + 1) % nv
    return v


@needs_ref
def test_step_batch_and_combine_match_reference():
    """drzg_step_batch == reduce_chunk state by state; drzg_states_combine ==
    combine_states (duplicates summed into the first, ledger.combines)"""
    from oracle import refapi
    g = golden("k3_f11_s1_r1.json")
    p, n, d = g["p"], g["n"], g["d"]
    M, u, pole, w = _seed_states(p, n, d, g["coeffs"], 4, 40, g["r_uniform"], g["nm_override"])
    ctx = drzg.Context(p, n, d, g["coeffs"], M)
    ids = ctx.seed(u, pole, w)
    S = set(range(n + 1 - min(d, n + 1), n + 1))  # default_S (reduction.hpp:35-41)
    moves = []
    for ui, Pi in zip(u, pole):
        v = _greedy_v(d, ui, S)
        kmax = min((ui[i] if i in S else ui[i] - 1) // v[i] for i in range(n + 1) if v[i])
        moves.append((v, max(1, min(2, kmax, Pi - n))))
    ctx.step(ids, [mv[0] for mv in moves], [mv[1] for mv in moves])
    gu, gp, gw = ctx.read(ids)
    for i in range(len(ids)):
        ref_w, info = refapi.chunk(p, n, d, g["coeffs"], M, u[i], pole[i], moves[i][0], moves[i][1], w[i])
        assert gu[i] == info["u"] and gp[i] == info["pole"]
        assert (gw[i] == ref_w).all()
    assert ctx.ledger[0] == sum(mv[1] for mv in moves) and ctx.ledger[1] == len(ids)
    # combine: a copy of every state merges into it (w + w)
    ids2 = ctx.seed(gu, gp, gw)
    kept = ctx.combine(ids + ids2)
    assert kept == ids and ctx.ledger[2] == len(ids)
    _, _, cw = ctx.read(kept)
    mod = p ** M
    sp = ctx.plan
    side = ctx.side
    for i in range(len(ids)):
        for r in range(0, side, 17):
            a = sum(int(gw[i][t * side + r]) * int(sp.beta) ** t for t in range(sp.limbs))
            c = sum(int(cw[i][t * side + r]) * int(sp.beta) ** t for t in range(sp.limbs))
            assert c == (2 * a) % mod
    ctx.close()


PEP_CASES = [("quintic_f7_s1.json", 16, [[2, 1, 2], [1, 1, 3], [0, 2, 3]]),
             ("k3_f11_s1_r1.json", 9, [[1, 1, 1, 1], [0, 1, 2, 1]]),
             ("quintic_f7_s1.json", 24, [[2, 1, 2]])]  # two limbs


@needs_ref
@pytest.mark.parametrize("case", PEP_CASES, ids=lambda c: f"{c[0]}-M{c[1]}")
def test_pep_entries_match_reference_build_ruv(case):
    """PepStoreBase::get(v) == build_ruv(C, v) bit for bit (reduction.hpp:253-297),
    through every backing, and the PEP route of a chunk (eval_to_linear +
    linrec_eval on the device) == the reference's reduce_chunk"""
    from oracle import refapi
    name, M, moves = case
    g = golden(name)
    p, n, d = g["p"], g["n"], g["d"]
    ctx = drzg.Context(p, n, d, g["coeffs"], M)
    stores = {spec: drzg.PepStore(ctx, spec) for spec in ("lazy", "lru:1", "lfuda:1")}
    for v in moves:
        ref, ref_nnz = refapi.build_ruv(p, n, d, g["coeffs"], M, v)
        for spec, st in stores.items():
            got, nnz = st.get(v)
            assert nnz == ref_nnz, spec
            assert (got.reshape(-1) == ref).all(), spec
    assert stores["lazy"].stats()["misses"] == len(moves)
    # the reference chunk path through the store: k = 2 steps along v0 from u
    v = moves[0]
    u = [30 if i != n else 25 for i in range(n + 1)] if n == 3 else [20, 20, 23]
    pole, k = 27 if n == 3 else 21, 2
    x = [u[i] - k * v[i] for i in range(n + 1)]
    A, B = stores["lazy"].eval_to_linear(v, x)
    rng = np.random.default_rng(5)
    sp = refapi.stripe_plan_py(p, M)
    side = ctx.side
    vals = [int(rng.integers(0, 2**62)) % (p ** M) for _ in range(side)]
    w = np.array([(val // sp["beta"] ** t) % sp["beta"] for t in range(sp["limbs"]) for val in vals], dtype=np.uint64)
    got_w, ctr = drzg.linrec_eval(p, M, side, A, B, k - 1, w)
    ref_w, info = refapi.chunk(p, n, d, g["coeffs"], M, u, pole, v, k, w)
    assert (got_w == ref_w).all() and ctr == k
    ctx.close()
