"""torchrun worker for tests/test_gpu_distributed.py: the config-3 search on
this rank's shard of the candidate space + the one NCCL all-reduce combine
(distributed_search_best), compared with one GPU searching the whole space;
and a replay trace batch sharded across ranks, compared with one GPU."""

import os
import pathlib
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2504_15303_b200 as hs  # noqa: E402
from paper_2504_15303_b200 import _native as nat  # noqa: E402
from paper_2504_15303_b200 import distributed as D  # noqa: E402
from paper_2504_15303_b200 import planner  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    eng = nat.engine_for(local)
    cluster, reqs, params, _I, _O = bench.search_inputs(10_000)
    t = planner.build_tables(cluster, reqs, params, engine=eng)
    got = D.distributed_search_best(t, engine=eng, device=dev)
    want = planner.search_best(t, engine=eng)[:3]
    assert got == want, (rank, got, want)
    # sharded replay: each rank replays its block of traces; gathered results == one GPU
    rc, config, rparams = bench.replay_deployment()
    T_all, q = 64, 4000
    off, I, O, A = bench.replay_inputs(0, T_all, q, 140.0)
    lo, hi = D.shard_range(T_all, rank, world)
    sl = slice(off[lo], off[hi])
    part = hs.replay_traces(rc, config, rparams, hs.PolicyConfig(), off[lo:hi + 1] - off[lo], I[sl], O[sl], O[sl],
                            arrival=A[sl], engine=eng)
    full = hs.replay_traces(rc, config, rparams, hs.PolicyConfig(), off, I, O, O, arrival=A, engine=eng)
    assert np.array_equal(part.assign, full.assign[sl])
    assert part.metrics.tobytes() == full.metrics[lo:hi].tobytes()
    dist.barrier(device_ids=[local])
    if rank == 0:
        print("NCCL_OK", world, got)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
