"""GPU: the tcgen05 int8 GEMM (UTCIMMA + TMA + TMEM) against exact integer
products, across tile-edge shapes and both A signednesses."""
import numpy as np
import pytest

import paper_2602_24155_b200 as drzg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 128, 128), (220, 300, 220), (64, 16, 32), (495, 1000, 495),
                                   (3003, 257, 3003), (130, 1, 48)])
def test_tc_gemm_signed(M, N, K):
    rng = np.random.default_rng(M * 7 + N)
    A = rng.integers(-127, 128, size=(M, K), dtype=np.int64)
    B = rng.integers(-127, 128, size=(N, K), dtype=np.int64)
    D = drzg.test_tc_gemm(A.astype(np.int8), B.astype(np.int8))
    assert (D.astype(np.int64) == B.dot(A.T)).all()


def test_tc_gemm_unsigned_a():
    rng = np.random.default_rng(5)
    A = rng.integers(0, 256, size=(300, 400), dtype=np.int64)
    B = rng.integers(-127, 128, size=(200, 400), dtype=np.int64)
    D = drzg.test_tc_gemm(A.astype(np.uint8), B.astype(np.int8), a_unsigned=True)
    assert (D.astype(np.int64) == B.dot(A.T)).all()


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (220, 300, 220), (3003, 513, 3003), (130, 17, 48)])
def test_tc_gemm_mn_major_b(M, N, K):
    rng = np.random.default_rng(M + N * 3)
    A = rng.integers(-127, 128, size=(M, K), dtype=np.int64)
    B = rng.integers(-127, 128, size=(N, K), dtype=np.int64)
    D = drzg.test_tc_gemm_mn(A.astype(np.int8), B.astype(np.int8))
    assert (D.astype(np.int64) == B.dot(A.T)).all()
