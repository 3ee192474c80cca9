"""CPU, multi-process: the N>1 path (column partition + limb all_gather of F)
with world_size 2 over gloo, on the reference's own K3 /F11 Frobenius matrix."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import golden
from paper_2602_24155_b200 import parallel


def test_partition_covers_every_column_once():
    for (n, d) in [(3, 4), (5, 3), (4, 3), (2, 5), (3, 5)]:
        b = sum(parallel.hodge_counts(n, d))
        for world in (1, 2, 3, 8):
            parts = [parallel.partition_columns(n, d, world, r) for r in range(world)]
            flat = sorted(j for p in parts for j in p)
            assert flat == list(range(b))
            if world <= b:
                assert all(p for p in parts)


def test_limb_roundtrip_large_entries():
    b = 3
    F = [0, 1, 7 ** 60, 2 ** 200 + 5, 11, 0, 3, 7 ** 24 - 1, 42]
    blk = parallel.encode_columns(F, b, [0, 1, 2], width=6)
    assert parallel.decode_blocks([blk], [[0, 1, 2]], b, 6) == F
    with pytest.raises(ValueError):
        parallel.encode_columns([2 ** 400] + [0] * 8, b, [0], width=6)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, F, b, n, d, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cols = parallel.partition_columns(n, d, world, rank)
    all_cols = [parallel.partition_columns(n, d, world, r) for r in range(world)]
    # each rank only knows its own columns
    local = [F[i * b + j] if j in cols else "0" for i in range(b) for j in range(b)]
    full = parallel.gather_frobenius(local, b, cols, world, all_cols)
    q.put((rank, [str(x) for x in full] == list(F)))
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gather_world2_gloo():
    g = golden("k3_f11_s1.json")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, g["F"], g["b"], g["n"], g["d"], q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=150) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert res == {0: True, 1: True}


def test_gather_host_cxx_matches_fixture():
    """the C++ side of drzg_gather_F (limb encode + owner decode) assembles the
    reference's K3 F from three ranks' column blocks"""
    g = golden("k3_f11_s1.json")
    b, F = g["b"], g["F"]
    owners = [parallel.partition_columns(g["n"], g["d"], 3, r) for r in range(3)]
    blocks = [[F[i * b + j] if j in o else "0" for i in range(b) for j in range(b)] for o in owners]
    assert [str(x) for x in parallel.gather_frobenius_host(blocks, b, owners)] == list(F)
    import pytest
    with pytest.raises(Exception):
        parallel.gather_frobenius_host(blocks[:2], b, owners[:2])  # a column without owner


def test_partition_by_replayed_ledger():
    """fourfold columns balanced by the reference's replayed per-column matvecs"""
    import os
    from conftest import GOLD
    w = parallel.replayed_column_weights(os.path.join(GOLD, "ledger_replay_fourfold.json"))
    assert len(w) == 22
    for world in (2, 4, 8):
        parts = [parallel.partition_columns(5, 3, world, r, weights=w) for r in range(world)]
        assert sorted(j for p in parts for j in p) == list(range(22))
        loads = [sum(w[j] for j in p) for p in parts]
        assert max(loads) / (sum(w) / world) < 1.25
