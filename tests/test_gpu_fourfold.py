"""GPU parity on the metric's own hypersurface: the random cubic fourfold /F7,
seed 1 (BASELINE.json configs[4]; side = nL = 3003).

Chunk level: drzg_reduce_chunk against the UNMODIFIED reference reduce_chunk
(reduction.hpp:394-423: build_ruv + eval_to_linear + linrec_eval) on the
fixtures of scripts/make_fourfold_golden.py, at one-limb precisions M = 7 and
M = 20 and at the default plan's M = 24 (two limbs; the reference's
MpzEchelon context took hours to build).  Pipeline level: drzg_frobenius
against the reference frobenius_matrix at series-truncated plans (N_m = 2, 3)
that the reference can finish here.  Plus the default-plan zeta function's own
battery, with the r = 2 point count (2.9e8 points of P^5(F_49)) on the GPU
counter.
"""
import os

import numpy as np
import pytest

from conftest import GOLD, golden
from fourfold_cases import CASES, FOURFOLD, chunk_input
import paper_2602_24155_b200 as drzg

pytestmark = pytest.mark.gpu


def _fixture(name):
    if not os.path.exists(os.path.join(GOLD, name)):
        pytest.skip(f"{name} not generated")
    return golden(name)


@pytest.mark.parametrize("M", [7, 20, 24])
@pytest.mark.parametrize("ci", range(len(CASES)))
def test_fourfold_reduce_chunk_matches_reference(M, ci):
    g = _fixture(f"fourfold_chunks_M{M}.json")
    if ci >= len(g["cases"]):
        pytest.skip("case not generated")
    c = g["cases"][ci]
    p, n, d, _ = FOURFOLD
    assert (c["u"], c["pole"], c["v"], c["k"]) == tuple(CASES[ci])
    w = chunk_input(p, M, 3003, ci)
    got_w, got_u, info = drzg.reduce_chunk(p, n, d, g["coeffs"], M, c["u"], c["pole"], c["v"], c["k"], w)
    ref_w = np.frombuffer(bytes.fromhex(c["w_out_hex"]), dtype="<u8")
    assert got_u == c["info"]["u"]
    assert info["matvecs"] == c["info"]["matvecs"] == c["k"]
    assert info["nL"] == info["side"] == 3003
    mism = int((got_w != ref_w).sum())
    assert mism == 0, f"{mism} of {ref_w.size} limbs differ"


@pytest.mark.parametrize("nm", [2, 3])
def test_fourfold_truncated_frobenius_matches_reference(nm):
    g = _fixture(f"random_fourfold_f7_s1_nm{nm}.json")
    fr = drzg.frobenius(g["p"], g["n"], g["d"], g["coeffs"], nm=nm)
    assert fr["plan"]["M"] == g["plan"]["M"]
    assert fr["nL"] == 3003
    assert fr["F"] == g["F"]
    assert fr["charpoly"] == g["charpoly"]
    assert (fr["matvecs"], fr["startups"], fr["combines"]) == (
        g["ledger"]["matvecs"], g["ledger"]["startups"], g["ledger"]["combines"])


def test_fourfold_columns_assemble_to_reference_F():
    """the multi-GPU unit: disjoint column subsets computed separately give
    the reference's F when assembled (zeta.hpp:109-133)"""
    g = _fixture("random_fourfold_f7_s1_nm3.json")
    b = g["b"]
    parts = [list(range(0, b, 2)), list(range(1, b, 2))]
    F = ["0"] * (b * b)
    for cols in parts:
        fr = drzg.frobenius(g["p"], g["n"], g["d"], g["coeffs"], nm=3, columns=cols)
        assert fr["computed"] == cols
        for i in range(b):
            for j in cols:
                F[i * b + j] = fr["F"][i * b + j]
    assert F == g["F"]


def test_nccl_gather_behind_the_c_abi():
    """drzg_comm_init + drzg_gather_F on one rank (the driver's GPU tests run
    on one GPU): the NCCL all_gather path in libdrzg.so round-trips F"""
    from paper_2602_24155_b200 import parallel
    g = golden("k3_f11_s1.json")
    b = g["b"]
    F = parallel.gather_frobenius_nccl(g["F"], b, list(range(b)), world=1, rank=0, device=0)
    assert [str(x) for x in F] == list(g["F"])
