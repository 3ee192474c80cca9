"""CPU: the synthetic inputs every bench and fourfold run uses come from the
native generator (drzg_random_hypersurface), which restates the reference CLI's
rule (drzeta_main.cpp:112-122 + run_zeta's smoothness checks, zeta.hpp:440-445).
It must give the reference generator's coefficients bit for bit."""
import pytest

from conftest import golden, needs_ref
import paper_2602_24155_b200 as drzg

CONFIGS = [(7, 2, 5, 1), (11, 3, 4, 1), (7, 3, 5, 1), (13, 4, 3, 1), (7, 5, 3, 1),
           (13, 4, 3, 0), (13, 4, 3, 2), (13, 4, 3, 63), (11, 2, 3, 3), (7, 2, 4, 2)]


@needs_ref
@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: "p%d_n%d_d%d_s%d" % c)
def test_generator_matches_reference(cfg):
    from oracle import refapi
    p, n, d, seed = cfg
    assert drzg.random_hypersurface(p, n, d, seed=seed) == [int(x) for x in refapi.hypersurface(p, n, d, seed=seed)]


@pytest.mark.parametrize("name", ["quintic_f7_s1.json", "k3_f11_s1.json", "threefold_f13_s1.json",
                                  "quintic_surface_f7_s1_r1.json", "random_cubic_curve_f11_s3.json"])
def test_generator_matches_fixture_inputs(name):
    g = golden(name)
    assert drzg.random_hypersurface(g["p"], g["n"], g["d"], seed=g["seed"]) == [int(x) for x in g["coeffs"]]


def test_fourfold_generator_matches_fixture():
    import os
    from conftest import GOLD
    for f in sorted(os.listdir(GOLD)):
        if f.startswith("fourfold_chunks_M") or f.startswith("random_fourfold"):
            g = golden(f)
            assert drzg.random_hypersurface(7, 5, 3, seed=1) == [int(x) for x in g["coeffs"]]
            return
    pytest.skip("no fourfold fixture")


def test_zeta_from_F_battery_matches_reference():
    """run_zeta's battery on the reference's own F gives the reference's Q"""
    for name in ["quintic_f7_s1.json", "fermat_cubic_curve_f7.json", "random_quartic_curve_f7_s2.json"]:
        g = golden(name)
        z = drzg.zeta_from_F(g["p"], g["n"], g["d"], g["coeffs"], g["F"], g["b"])
        assert z["status"] == "ok"
        assert [z["Q"]] == g["Q_candidates"][:1]
        assert all(ok for (_, _, ok) in z["counts"])
