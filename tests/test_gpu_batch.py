"""Concurrent zeta functions on one device (BASELINE configs[3]'s batch path,
paper_2602_24155_b200.zeta_batch): several host threads, each with its own
stream and engine, with the dataflow kernels' launches chained per device
(kernels/tc_gemm.cu gated_flow_launch).  Every result must equal the
reference's, exactly as when run alone."""
import pytest

from conftest import golden
import paper_2602_24155_b200 as drzg

pytestmark = pytest.mark.gpu


def test_batch_of_threefolds_matches_reference_concurrently():
    """threefold /F13 (the dataflow kernel, nL = 495) four times at once,
    interleaved with K3 /F11 (the one-launch kernel): Q and the ledger of every
    call equal the reference's"""
    th = golden("threefold_f13_s1.json")
    k3 = golden("k3_f11_s1.json")
    jobs = [th, k3, th, th, k3, th]
    zs = drzg.zeta_batch(13, 4, 3, [th["coeffs"]] * 4, workers=4)
    for z in zs:
        assert [z["Q"]] == th["Q_candidates"][:1]
        assert z["frobenius"]["matvecs"] == th["ledger"]["matvecs"]
        assert all(ok for (_, _, ok) in z["counts"])
    # mixed shapes on concurrent threads
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        out = list(ex.map(lambda g: drzg.frobenius(g["p"], g["n"], g["d"], g["coeffs"]), jobs))
    for g, fr in zip(jobs, out):
        assert fr["F"] == g["F"]
        assert (fr["matvecs"], fr["startups"], fr["combines"]) == (
            g["ledger"]["matvecs"], g["ledger"]["startups"], g["ledger"]["combines"])


def test_batch_is_ordered_and_sequential_when_one_worker():
    q = golden("quintic_f7_s1.json")
    c = golden("random_cubic_curve_f11_s3.json")
    zs = drzg.zeta_batch(7, 2, 5, [q["coeffs"], q["coeffs"]], workers=1)
    assert all([z["Q"]] == q["Q_candidates"][:1] for z in zs)
    assert c["p"] == 11  # a different field is a different batch
