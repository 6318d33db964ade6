"""N > 1 host logic on CPU with the gloo backend (world_size 2): global-index sharding of the seeded
generator and the single aggregate all-reduce (paper_2304_13541_b200.dist) reproduce the 1-rank result."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from tests.aggref import host_agg

N_PER = 24


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_13541_b200.dist import allreduce_agg
    sp, p = synth.config(2, num_scen=N_PER, rows_pct=20, scen_base=rank * N_PER)
    pb = synth.generate_host(sp)
    o = oracle.evaluate(pb, p)
    agg = torch.from_numpy(host_agg(o))   # position-free checksum: shard aggregates add up
    allreduce_agg(agg)
    if rank == 0:
        q.put(agg.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_match_single_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    sp, p = synth.config(2, num_scen=N_PER * world, rows_pct=20)
    full = host_agg(oracle.evaluate(synth.generate_host(sp), p))
    assert np.array_equal(got[5:], full[5:])                                   # integers: exact
    np.testing.assert_allclose(got[:5].view(np.float64), full[:5].view(np.float64), rtol=1e-12)  # f64 sums


def test_shard_bounds():
    from paper_2304_13541_b200.dist import shard
    for n in (1, 7, 1000, 1_000_000):
        for world in (1, 2, 4, 8):
            rngs = [shard(n, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == n
            assert all(rngs[i][1] == rngs[i + 1][0] for i in range(world - 1))
