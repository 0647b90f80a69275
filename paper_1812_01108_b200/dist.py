"""Batch sharding across GPUs (north star "sharding the protein batch").

Chains are independent, so the multi-GPU path has no data-path collective:
each rank runs its own subset of chains through the same kernels.  This
module plans the subsets and provides the scalar reductions the bench uses
for timing (max over ranks) and bookkeeping (sums).  Pure Python/torch; the
planner is unit-tested with a world-size-2 gloo group on the CPU.
"""
import heapq

import torch


def contiguous_shards(n_chains, world):
    """Uniform-length batches: rank r gets chains [lo, hi) with sizes differing by <= 1."""
    base, extra = divmod(int(n_chains), int(world))
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append(list(range(lo, hi)))
        lo = hi
    return out


def lpt_shards(lengths, world):
    """Ragged batches: longest-processing-time-first assignment balancing the
    sum of residues per rank; each shard is returned longest chain first (the
    order its CTAs should be scheduled in).  Greedy LPT is within 4/3 of the
    optimal makespan."""
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i))
    heap = [(0, r) for r in range(world)]
    shards = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + int(lengths[i]), r))
    return shards


def plan(lengths, world):
    """Pick the planner: contiguous when all chains have the same length."""
    lengths = [int(x) for x in lengths]
    if len(set(lengths)) <= 1:
        return contiguous_shards(len(lengths), world)
    return lpt_shards(lengths, world)


def imbalance(lengths, shards):
    """max rank load / mean rank load (1.0 = perfect)."""
    loads = [sum(int(lengths[i]) for i in s) for s in shards]
    mean = sum(loads) / max(len(loads), 1)
    return max(loads) / mean if mean else 1.0


def reduce_scalar(x, op, dist=None, device=None):
    """All-reduce one float64 scalar (op: "max" | "sum") across the default group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())
