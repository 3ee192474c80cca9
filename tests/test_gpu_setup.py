"""GPU setup eliminations (pivot scan over F_p, inverse mod q) agree with the
host restatements (host/elim.hpp), through the end-to-end fixtures at sizes
that take the device path (Fermat fourfold, nL = 3003) and a direct check."""
import numpy as np
import pytest

import paper_2602_24155_b200 as drzg

pytestmark = pytest.mark.gpu


def test_device_setup_matches_host():
    # drzg_test_setup runs both the host and the device version on random
    # matrices and reports mismatches (0 expected)
    import ctypes
    L = drzg.lib()
    for (p, q, n, cols, seed) in [(7, 49, 900, 1800, 1), (11, 121, 800, 1300, 2), (13, 169, 780, 780, 3)]:
        bad = ctypes.c_int64(-1)
        rc = L.drzg_test_setup(ctypes.c_uint64(p), ctypes.c_uint64(q), n, cols, ctypes.c_uint64(seed),
                               ctypes.byref(bad))
        assert rc == 0, drzg._err()
        assert bad.value == 0


@pytest.mark.parametrize("p,n,d,M", [(7, 5, 3, 7), (7, 5, 3, 24), (11, 3, 4, 17)])
def test_device_tables_and_final_levels_match_host(p, n, d, M):
    # the random fourfold's 3003 x 6237 solve matrix and 2002-row final level
    # take the device path; both must equal the host restatement exactly
    import ctypes
    L = drzg.lib()
    co = drzg.random_hypersurface(p, n, d, 1)
    for fn in (L.drzg_test_tables, L.drzg_test_final_levels):
        diff = ctypes.c_int64(-1)
        assert fn(ctypes.c_uint64(p), n, d, drzg._u64arr(co), M, ctypes.byref(diff)) == 0, drzg._err()
        assert diff.value == 0


@pytest.mark.parametrize("p,n,d,r", [(7, 2, 5, 2), (11, 3, 4, 1), (11, 3, 4, 2), (13, 4, 3, 1), (7, 5, 3, 1),
                                     (7, 3, 5, 2)])
def test_device_point_count_matches_host(p, n, d, r):
    co = drzg.random_hypersurface(p, n, d, 1)
    assert drzg.count_points_device(p, n, d, co, r) == drzg.count_points(p, n, d, co, r)
