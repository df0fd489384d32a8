"""Request-level data parallelism across ranks (world_size 2, gloo on CPU).

Each rank serves only the users the sticky router assigns to it (no data-path collective) and the records are
gathered once at the end; the merged result must equal a single process simulating both instances.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_07203_b200 import workload as wl
from paper_2505_07203_b200.scheduling import Policy
from paper_2505_07203_b200.serving import merge_records, shard_trace, simulate


def svc(idx, w, nc, ids):
    n = w.request.n_input
    return 0.02 + 1.1e-5 * (n - nc) + 6e-10 * (n * n - nc * nc) / 2.0


def trace():
    spec = wl.PostRecSpec(users=6, requests_per_user=8, profile_mean=2000, profile_std=400, profile_min=1500,
                          profile_max=2500, suffix_tokens=150)
    return wl.poisson_arrivals(wl.gen_post_recommendation(1, spec), 25.0, seed=3)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_trace(trace(), rank, world)
    rep = simulate(mine, 1, Policy.srjf_calibrated(), 16 * 400, svc)
    gathered = [None] * world
    dist.all_gather_object(gathered, list(rep.records))
    if rank == 0:
        merged = merge_records(gathered, world)
        out.put([(r.id, r.instance, r.start, r.completion, r.n_cached) for r in merged.records])
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_dp_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), q), nprocs=world, join=True)
    got = q.get(timeout=60)
    ref = simulate(trace(), world, Policy.srjf_calibrated(), 16 * 400, svc)
    exp = sorted([(r.id, r.instance, r.start, r.completion, r.n_cached) for r in ref.records],
                 key=lambda x: (x[3], x[0]))
    assert sorted(got, key=lambda x: (x[3], x[0])) == exp
    assert {x[1] for x in got} == {0, 1}


def test_shards_partition_the_trace():
    t = trace()
    parts = [shard_trace(t, r, 3) for r in range(3)]
    ids = sorted(r.id for p in parts for r in p.requests)
    assert ids == sorted(r.id for r in t.requests)
    users = [set(r.user_id for r in p.requests) for p in parts]
    assert not (users[0] & users[1]) and not (users[1] & users[2])
