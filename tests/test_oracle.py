"""CPU: the oracles are pinned before anything is checked against them.

* oracle/linrec_oracle.c (plain-C restatement of linalg.hpp:337-410) against
  the reference's own known answers (tests/test_linalg.cpp:294-357) and the
  committed golden vectors produced by the unmodified reference;
* the compiled reference (oracle/_ref) against the golden values its own
  test suite holds (test_zeta_small.cpp:282-388) and the fixtures.
"""
import numpy as np
import pytest

from conftest import golden, needs_ref
from oracle import refapi


def _arr(xs):
    return np.array([int(x) for x in xs], dtype=np.uint64)


def test_stripe_plan_restated():
    # known plans: 1 limb below 2^62, 2 limbs for 7^24, 3 for 7^49
    assert refapi.stripe_plan_py(7, 24)["limbs"] == 2
    assert refapi.stripe_plan_py(7, 24)["beta"] == 7 ** 12
    assert refapi.stripe_plan_py(7, 49)["limbs"] == 3
    assert refapi.stripe_plan_py(11, 17)["limbs"] == 1


def test_oracle_known_answers():
    # test_linalg.cpp:296-311: k=0 -> B w = 3; k=2 -> 3*5*7 = 105 = 4 mod 101
    A, B, w = _arr([2]), _arr([3]), _arr([1])
    assert int(refapi.oracle_linrec_eval(101, 1, 1, A, B, 0, w)[0]) == 3
    assert int(refapi.oracle_linrec_eval(101, 1, 1, A, B, 2, w)[0]) == 4


def test_oracle_explicit_product():
    # test_linalg.cpp:313-345: random 8x8 mod 7^4 against the explicit product
    rng = np.random.default_rng(53)
    mod = 7 ** 4
    for _ in range(10):
        X = rng.integers(0, mod, size=(8, 8))
        Y = rng.integers(0, mod, size=(8, 8))
        k = int(rng.integers(0, 21))
        v = rng.integers(0, mod, size=8)
        P = np.eye(8, dtype=object)
        for y in range(k + 1):
            Mt = (X.astype(object) * y + Y.astype(object)) % mod
            P = P.dot(Mt) % mod
        expect = P.dot(v.astype(object)) % mod
        got = refapi.oracle_linrec_eval(7, 4, 8, X.astype(np.uint64).ravel(), Y.astype(np.uint64).ravel(), k,
                                        v.astype(np.uint64))
        assert [int(x) for x in got] == [int(x) for x in expect]


def test_oracle_a_zero_gives_power_of_b():
    # test_linalg.cpp:347-356: A = 0 degenerates to B^{k+1} w
    rng = np.random.default_rng(7)
    mod = 7 ** 4
    Y = rng.integers(0, mod, size=(8, 8)).astype(object)
    v = np.arange(1, 9).astype(object)
    ref = v.copy()
    for _ in range(5):
        ref = Y.dot(ref) % mod
    got = refapi.oracle_linrec_eval(7, 4, 8, np.zeros(64, dtype=np.uint64), Y.astype(np.uint64).ravel(), 4,
                                    v.astype(np.uint64))
    assert [int(x) for x in got] == [int(x) for x in ref]


@pytest.mark.parametrize("idx", range(10))
def test_oracle_matches_reference_golden(idx):
    c = golden("linrec_cases.json")["cases"][idx]
    out = refapi.oracle_linrec_eval(c["p"], c["M"], c["side"], _arr(c["A"]), _arr(c["B"]), c["tmax"], _arr(c["w"]))
    assert (out == _arr(c["out"])).all()
    assert refapi.stripe_plan_py(c["p"], c["M"]) == c["plan"]


@needs_ref
def test_reference_build_golden_q():
    # test_zeta_small.cpp:285 (Fermat cubic /F7 -> Q = [1,1,7])
    coeffs = refapi.hypersurface(7, 2, 3, mode="fermat")
    z = refapi.zeta(7, 2, 3, coeffs)
    assert z["Q"] == ["1", "1", "7"]


@needs_ref
def test_reference_build_matches_fixtures():
    g = golden("quintic_f7_s1.json")
    assert refapi.hypersurface(7, 2, 5, seed=1) == g["coeffs"]
    fr = refapi.frobenius(7, 2, 5, g["coeffs"])
    assert fr["F"] == g["F"]
    assert fr["matvecs"] == g["ledger"]["matvecs"] == 324060


@needs_ref
@pytest.mark.parametrize("idx", [0, 2, 5, 6, 8])
def test_reference_kernel_paths_agree(idx):
    # dense and CSC paths of the reference agree bit for bit (test_reduction.cpp:382-402)
    c = golden("linrec_cases.json")["cases"][idx]
    d, _ = refapi.linrec_eval(c["p"], c["M"], c["side"], _arr(c["A"]), _arr(c["B"]), c["tmax"], _arr(c["w"]))
    s, _ = refapi.sparse_steps(c["p"], c["M"], c["side"], _arr(c["A"]), _arr(c["B"]), c["tmax"], _arr(c["w"]))
    if refapi.stripe_plan_py(c["p"], c["M"])["limbs"] <= 2:
        assert (d == s).all()


@needs_ref
@pytest.mark.parametrize("name", ["quintic_f7_s1.json", "fermat_cubic_curve_f7.json", "k3_f11_s1_r1.json",
                                  "threefold_f13_s1_r1.json", "fermat_fourfold_f7_r1.json",
                                  "quintic_surface_f7_s1_r1.json", "k3_f11_s1.json"])
def test_ledger_replay_equals_reference_run(name):
    """the value-free replay (ref_replay_ledger) gives the real reference
    run's ledger: the basis for the replayed default-plan ledgers
    (tests/golden/ledger_replay_*.json) the engine is checked against"""
    from oracle import refapi
    g = golden(name)
    r = refapi.replay_ledger(g["p"], g["n"], g["d"], g["coeffs"], r_uniform=g["r_uniform"], nm=g["nm_override"],
                             threads=2)
    assert (r["matvecs"], r["startups"], r["combines"]) == tuple(
        g["ledger"][k] for k in ("matvecs", "startups", "combines"))
