"""Sentence-level data parallelism over the GPUs of one box.

Sentences are independent (the reference session is per sentence,
infer.py:176-221), so the corpus is sharded with no communication inside the
decode loop:

1. sort by source length and cut into length buckets of at most
   `max_tokens` source tokens (the BASELINE's per-GPU batches of <= 8192);
2. assign buckets to ranks by greedy LPT bin-packing on a predicted cost --
   random-init decodes always run to the Stage-I cap, so the cost is known up
   front: encoder tokens + Stage-I rows summed over steps + Stage-II rows;
3. each rank decodes its buckets with its own engine;
4. one collective at the end: per-rank device time is max-reduced and the
   per-sentence outputs are gathered to rank 0 (NCCL over NVLink on the
   B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

from .workload import max_steps_for


@dataclass
class Bucket:
    index: np.ndarray  # sentence indices into the corpus
    tokens: int        # source tokens
    cost: float        # predicted cost (arbitrary units)


def predicted_cost(src_len, k=2, enc_layers=12):
    """Rows the decode touches: encoder tokens x layers + Stage-I rows over
    steps (one row per step) + Stage-II rows (k * steps)."""
    n = src_len - 1
    m = max_steps_for(n, k)
    return src_len * enc_layers + m * 6 + k * m


def length_buckets(lens, max_tokens=8192, k=2, enc_layers=12, padded=True):
    """Sort by length (stable) and cut into buckets of <= max_tokens tokens.

    padded=True (the BASELINE's C5 batches): a bucket's size is its sentence
    count times its longest source, as a padded batch would be; the engine
    itself packs the sentences (no padding reaches a kernel). padded=False
    counts the real tokens only.
    """
    lens = np.asarray(lens)
    order = np.argsort(lens, kind="stable")
    buckets, cur, tok, cost = [], [], 0, 0.0
    for i in order:
        li = int(lens[i])
        grown = (len(cur) + 1) * li if padded else tok + li  # ascending order: li is the bucket maximum
        if cur and grown > max_tokens:
            buckets.append(Bucket(np.array(cur), tok, cost))
            cur, tok, cost = [], 0, 0.0
        cur.append(int(i))
        tok += li
        cost += predicted_cost(li, k, enc_layers)
    if cur:
        buckets.append(Bucket(np.array(cur), tok, cost))
    return buckets


def assign_lpt(buckets, world_size):
    """Greedy longest-processing-time assignment; returns per-rank bucket lists."""
    heap = [(0.0, r) for r in range(world_size)]
    out = [[] for _ in range(world_size)]
    for b in sorted(buckets, key=lambda b: -b.cost):
        load, r = heapq.heappop(heap)
        out[r].append(b)
        heapq.heappush(heap, (load + b.cost, r))
    return out


def shard(lens, rank, world_size, max_tokens=8192, k=2, enc_layers=12, padded=True):
    """This rank's buckets (deterministic on every rank: no communication)."""
    return assign_lpt(length_buckets(lens, max_tokens, k, enc_layers, padded), world_size)[rank]


def rank_loads(lens, world_size, max_tokens=8192, k=2, enc_layers=12, padded=True):
    return [sum(b.cost for b in bs)
            for bs in assign_lpt(length_buckets(lens, max_tokens, k, enc_layers, padded), world_size)]


def gather_outputs(index, lens, tokens, group=None, device=None):
    """Gather (sentence index, output length, output tokens) to rank 0.

    index: int64 [n] corpus indices decoded on this rank; lens: int32 [n];
    tokens: int32 [n, L]. Returns (index, lens, tokens) concatenated over
    ranks on rank 0 (None elsewhere). Works with gloo (CPU tensors) and NCCL
    (pass device=cuda device).
    """
    import torch
    import torch.distributed as dist

    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cpu")
    tokens = np.asarray(tokens)
    # row count and token width per rank (a rank with no sentences may hold an empty array,
    # and ranks may size their output rows differently): every rank pads to the maxima
    L_loc = tokens.shape[1] if tokens.ndim == 2 else 0
    n = torch.tensor([len(index), L_loc], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(ns, n, group=group)
    nmax = int(max(int(x[0].item()) for x in ns))
    L = int(max(int(x[1].item()) for x in ns))
    pack = torch.zeros((nmax, 2 + L), dtype=torch.int64, device=dev)
    if len(index):
        pack[: len(index), 0] = torch.as_tensor(np.asarray(index, np.int64), device=dev)
        pack[: len(index), 1] = torch.as_tensor(np.asarray(lens, np.int64), device=dev)
        pack[: len(index), 2:2 + L_loc] = torch.as_tensor(tokens.astype(np.int64), device=dev)
    parts = [torch.zeros_like(pack) for _ in range(ws)]
    dist.all_gather(parts, pack, group=group)
    if rank != 0:
        return None
    rows = [p[: int(c[0].item())].cpu().numpy() for p, c in zip(parts, ns)]
    allr = np.concatenate(rows) if rows else np.zeros((0, 2 + L), np.int64)
    return allr[:, 0], allr[:, 1].astype(np.int32), allr[:, 2:].astype(np.int32)


def max_over_ranks(value, group=None, device=None):
    """Device time (or any scalar) max-reduced over ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value, group=None, device=None):
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
