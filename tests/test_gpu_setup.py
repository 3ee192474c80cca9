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
