"""Multi-rank host logic on CPU (gloo, world_size 2): shard ranges cover the
space exactly once, and the single all-reduce combine reproduces the
single-rank argmax (values from the C oracle on a real config-1 table)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_15303_b200 import distributed as D


def test_shard_ranges_partition_space():
    for size in (0, 1, 7, 5**16, 10**12 + 3):
        for world in (1, 2, 3, 4, 8):
            parts = [D.shard_range(size, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == size
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_reduce_slots_tie_and_empty_rules():
    buf = np.concatenate([D.pack_slot(3, 0, 5.0, 17, 4), D.pack_slot(3, 1, 5.0, 9, 2), D.pack_slot(3, 2, 0.0, -1, 0)])
    buf = buf.reshape(3, 3, 3).sum(axis=0)
    assert D.reduce_slots(buf) == (5.0, 9, 6)
    empty = D.pack_slot(2, 0, 0.0, -1, 0) + D.pack_slot(2, 1, 0.0, -1, 0)
    assert D.reduce_slots(empty) == (0.0, -1, 0)
    neg = D.pack_slot(2, 0, -0.0, 3, 1) + D.pack_slot(2, 1, -1e300, 1, 1)
    assert D.reduce_slots(neg) == (-0.0, 3, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, table, nd, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import hs_oracle as orc
    P = int(np.prod(nd.astype(np.int64)))
    lo, hi = D.shard_range(P, rank, world)
    t, i, n = orc.best(table, nd, lo, hi)
    res = D.combine_best(t, i, n)
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_combine_matches_single_rank(world):
    import helpers as H
    from oracle import hs_oracle as orc
    case = next(c for c in H.load("search_cases.json") if c["name"] == "config2")
    cluster = H.cluster_from(case["profile"])
    requests = H.search_trace(case)
    model, engine, limits, machines, params, present = H.search_structs(cluster, H.params_from(case["profile"]))
    I = np.array([r.input_len for r in requests], np.int32)
    O = np.array([r.output_len for r in requests], np.int32)
    table, nd = orc.tables(model, engine, limits, machines, params, present, I, O)
    P = int(np.prod(nd.astype(np.int64)))
    want = orc.best(table, nd, 0, P)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), table, nd, out), nprocs=world, join=True)
    for r in range(world):
        assert tuple(out[r]) == want
