"""Data-parallel corpus sharding and its end-of-run collectives,
on CPU with the gloo backend (world_size 2)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2212_01543_b200 import parallel as P
from paper_2212_01543_b200 import workload as W


def test_buckets_cover_corpus_once_and_respect_token_cap():
    srcs = W.make_sources(3000, 4, ("lognormal", 28.0, 0.5))
    lens = [len(s) for s in srcs]
    bs = P.length_buckets(lens, max_tokens=8192)
    idx = np.concatenate([b.index for b in bs])
    assert sorted(idx.tolist()) == list(range(len(srcs)))
    for b in bs:
        assert len(b.index) * max(lens[i] for i in b.index) <= 8192  # padded batch size (C5)
        assert b.tokens == sum(lens[i] for i in b.index)
    # packed-token buckets are never smaller
    assert len(P.length_buckets(lens, max_tokens=8192, padded=False)) <= len(bs)
    # buckets are length-sorted runs: lengths inside a bucket are contiguous in sorted order
    maxes = [max(lens[i] for i in b.index) for b in bs]
    mins = [min(lens[i] for i in b.index) for b in bs]
    assert all(mx <= mn2 for mx, mn2 in zip(maxes, mins[1:]))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_lpt_assignment_is_balanced_and_disjoint(world):
    srcs = W.make_sources(5000, 4, ("lognormal", 28.0, 0.5))
    lens = [len(s) for s in srcs]
    shards = [P.shard(lens, r, world) for r in range(world)]
    seen = np.concatenate([b.index for bs in shards for b in bs])
    assert sorted(seen.tolist()) == list(range(len(srcs)))
    loads = P.rank_loads(lens, world)
    assert max(loads) <= 1.05 * (sum(loads) / world) + max(b.cost for bs in shards for b in bs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    srcs = W.make_sources(400, 4, ("lognormal", 28.0, 0.5))
    lens = [len(s) for s in srcs]
    mine = P.shard(lens, rank, world, max_tokens=2048)
    idx = np.concatenate([b.index for b in mine]) if mine else np.zeros(0, np.int64)
    # stand-in "decode": output = reversed source without EOS (host only)
    L = 16
    toks = np.zeros((len(idx), L), np.int32)
    olen = np.zeros(len(idx), np.int32)
    for j, i in enumerate(idx):
        o = srcs[i][:-1][::-1][:L]
        toks[j, : len(o)] = o
        olen[j] = len(o)
    got = P.gather_outputs(idx, olen, toks)
    tmax = P.max_over_ranks(float(rank + 1))
    wsum = P.sum_over_ranks(float(olen.sum()))
    if rank == 0:
        order = np.argsort(got[0])
        q.put((got[0][order].tolist(), got[1][order].tolist(), got[2][order].tolist(), tmax, wsum))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    idx, olen, toks, tmax, wsum = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    srcs = W.make_sources(400, 4, ("lognormal", 28.0, 0.5))
    assert idx == list(range(400))
    for i in range(400):
        o = srcs[i][:-1][::-1][:16]
        assert olen[i] == len(o) and toks[i][: len(o)] == o
    assert tmax == 2.0
    assert wsum == float(sum(olen))


def _worker_ragged(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if rank == 0:  # three sentences, 8-wide output rows
        idx = np.array([5, 1, 3], np.int64)
        olen = np.array([2, 8, 0], np.int32)
        toks = np.arange(24, dtype=np.int32).reshape(3, 8)
    else:  # no bucket on this rank: empty arrays of any shape
        idx, olen, toks = np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int32)
    got = P.gather_outputs(idx, olen, toks)
    if rank == 0:
        q.put((got[0].tolist(), got[1].tolist(), got[2].tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_gather_with_an_empty_rank():
    """A rank without sentences (more ranks than buckets) passes empty arrays: the
    gather agrees on row count and token width across ranks instead of failing."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_ragged, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    idx, olen, toks = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert idx == [5, 1, 3] and olen == [2, 8, 0]
    assert toks == np.arange(24).reshape(3, 8).tolist()
