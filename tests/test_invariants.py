"""run_zeta's F-splitting invariant (Fedder's criterion, reference
zeta.hpp:336-350, 536-539) against the unmodified reference on the BASELINE
shapes and the fixtures' hypersurfaces (host only: no GPU).  The engine's
version prunes the powers f^t to exponents <= p - 1 (terms outside that box
never return to it), so it must agree with the reference's full powers."""
import pytest

from conftest import needs_ref
import paper_2602_24155_b200 as drzg

SHAPES = [(7, 2, 5), (11, 3, 4), (7, 3, 5), (13, 4, 3), (7, 5, 3), (7, 3, 4), (11, 2, 3), (7, 2, 4)]


@needs_ref
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_fsplit_matches_reference(shape, seed):
    from oracle import refapi
    p, n, d = shape
    co = refapi.hypersurface(p, n, d, seed=seed)
    assert drzg.fsplit(p, n, d, co) == refapi.fsplit(p, n, d, co)


@needs_ref
@pytest.mark.parametrize("shape", [(7, 3, 4), (7, 5, 3), (11, 3, 4), (13, 4, 3)])
def test_fsplit_fermat_matches_reference(shape):
    from oracle import refapi
    p, n, d = shape
    co = refapi.hypersurface(p, n, d, mode="fermat")
    assert drzg.fsplit(p, n, d, co) == refapi.fsplit(p, n, d, co)
