"""CPU: the PEP store's backings (eager / lazy / lru:N / lfuda:N) keep the
reference's bookkeeping (pep.hpp:15-209), checked with the same sequences as
the reference's own suite (tests/test_pep.cpp:53-190) on placeholder entries."""
import random
import threading

import pytest

import paper_2602_24155_b200 as drzg

NV, D = 3, 3  # the Fermat cubic's move vectors: Homog_3 in 3 variables
MOVES = [[3, 0, 0], [2, 1, 0], [2, 0, 1], [1, 2, 0], [1, 1, 1], [1, 0, 2], [0, 3, 0], [0, 2, 1], [0, 1, 2], [0, 0, 3]]


def test_eager_never_misses():
    s = drzg.PepStore.stub(NV, D, "eager")
    for _ in range(3):
        for v in MOVES:
            s.get(v)
    assert s.stats() == {"hits": 3 * len(MOVES), "misses": 0, "evictions": 0}


def test_lazy_misses_once_per_move_vector():
    s = drzg.PepStore.stub(NV, D, "lazy")
    for _ in range(3):
        for v in MOVES[:4]:
            s.get(v)
    assert s.stats() == {"hits": 8, "misses": 4, "evictions": 0}


def test_lru_eviction_order():
    s = drzg.PepStore.stub(NV, D, "lru:2")
    v0, v1, v2 = MOVES[:3]
    for v in (v0, v1, v0, v2, v1, v0):
        s.get(v)
    assert s.stats() == {"hits": 1, "misses": 5, "evictions": 3}
    wide, lazy = drzg.PepStore.stub(NV, D, "lru:1000"), drzg.PepStore.stub(NV, D, "lazy")
    rng = random.Random(127)
    for _ in range(40):
        v = MOVES[rng.randrange(len(MOVES))]
        wide.get(v)
        lazy.get(v)
    a, b = wide.stats(), lazy.stats()
    assert (a["hits"], a["misses"], a["evictions"]) == (b["hits"], b["misses"], 0)


def test_lfuda_frequency_with_aging():
    s = drzg.PepStore.stub(NV, D, "lfuda:2")
    v0, v1, v2 = MOVES[:3]
    for v in (v0, v0, v1, v2, v0, v1):
        s.get(v)
    assert s.stats() == {"hits": 2, "misses": 4, "evictions": 2}
    s.get(v0)  # still resident
    assert s.stats()["hits"] == 3


def test_concurrent_requests_build_once():
    s = drzg.PepStore.stub(NV, D, "lazy")
    ts = [threading.Thread(target=s.get, args=(MOVES[0],)) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert s.stats() == {"hits": 7, "misses": 1, "evictions": 0}


@pytest.mark.parametrize("spec", ["lru:0", "lru", "lru:x", "bogus", "lfuda:-1"])
def test_backing_specs(spec):
    with pytest.raises(drzg.DrzgError):
        drzg.PepStore.stub(NV, D, spec)
    for ok in ("eager", "lazy", "lru:8", "lfuda:4"):
        drzg.PepStore.stub(NV, D, ok)
