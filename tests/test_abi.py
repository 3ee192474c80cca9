"""CPU: the C-ABI library loads and exports every symbol include/drzg.h
declares; host-only entry points agree with the reference."""
import os
import re

import pytest

from conftest import ROOT, golden
import paper_2602_24155_b200 as drzg


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "drzg.h")).read()
    return sorted(set(re.findall(r"\b(drzg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_header():
    L = drzg.lib()
    names = declared_symbols()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n


def test_stripe_plan_matches_reference_rule():
    from oracle import refapi
    for p, M in [(7, 24), (7, 49), (11, 17), (13, 13), (47, 11), (7, 5)]:
        sp = drzg.stripe_plan(p, M)
        ref = refapi.stripe_plan_py(p, M)
        assert (sp.limbs, sp.limb_exp, sp.beta, sp.stripe) == (ref["limbs"], ref["limb_exp"], ref["beta"], ref["stripe"])


@pytest.mark.parametrize("name", ["fermat_cubic_curve_f7.json", "quintic_f7_s1.json",
                                  "random_quartic_curve_f7_s2.json"])
def test_charpoly_and_recovery_match_reference(name):
    g = golden(name)
    r = drzg.charpoly(g["p"], g["n"], g["d"], g["F"], g["b"], r_uniform=g["r_uniform"], nm=g["nm_override"])
    assert r["charpoly"] == g["charpoly"]
    assert r["candidates"] == g["Q_candidates"]


def test_errors_surface_as_exceptions():
    with pytest.raises(drzg.DrzgError):
        drzg.stripe_plan(1, 0)
