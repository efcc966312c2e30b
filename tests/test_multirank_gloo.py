"""The N>1 bench path on CPU: world_size-2 gloo processes exercise the sample
sharding (independent seeded batches per rank), the max-over-ranks timing
reduction and the whole-job aggregate, and check that two ranks' batches are
disjoint draws of the same config (weak scaling, no data-path collective)."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2402_10488_b200 import configs
    seed = bench.shard_seed(configs.SEEDS["c5"], rank)
    st, ss = configs.c5_coefficients(8, 2, seed=seed)
    ms_local = 10.0 + 5.0 * rank
    ms_max = bench.max_over_ranks(ms_local, world)
    value = bench.aggregate_value(1000, 4, world, ms_max)
    out[rank] = (seed, float(st.sum()), float(ss.sum()), ms_max, value)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_timing():
    world = 2
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()  # no fork of a multi-threaded (OpenMP) parent
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0[0] != r1[0]                      # independent seeds per rank
    assert r0[1] != r1[1]                      # different (disjoint) sample draws
    assert r0[3] == r1[3] == 15.0              # max over ranks
    assert np.isclose(r0[4], 1000 * 4 * 2 / 15e-3) and r0[4] == r1[4]
