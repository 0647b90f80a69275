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


# ---------------------------------------------------------------------------
# one chain split over ranks (sequence sharding), one exchange step
# per pass: an all-gather of a 48-byte aggregate transform per chain in the
# forward, of a 48-byte (S, T, first atom) record in the backward.  The
# arithmetic runs in the library's kernels (tpl_backbone_segment_*); this is
# the marshalling and the collectives.

def segment_bounds(L, world):
    """Contiguous residue ranges [j0, j1) of a length-L chain, one per rank, each >= 1 residue."""
    L, world = int(L), int(world)
    if L < world:
        raise ValueError(f"a chain of {L} residues cannot be split over {world} ranks")
    base, extra = divmod(L, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def gather_stack(t, group=None):
    """[world, *t.shape] with rank r's tensor at index r (the exchange step)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    else:
        dist.all_gather(list(out.unbind(0)), t.contiguous(), group=group)
    return out


class SegmentBackbone(torch.autograd.Function):
    """Backbone forward/backward of this rank's segment of every chain (f4)."""

    @staticmethod
    def forward(ctx, angles, lengths, omega_prev, group):
        import torch.distributed as dist

        from . import _abi
        from .api import MODEL_BACKBONE, default_workspace

        angles = angles.contiguous()
        B, Lmax, _ = angles.shape
        seg, n_seg = dist.get_rank(group), dist.get_world_size(group)
        ws = default_workspace(angles.device).get(MODEL_BACKBONE, B, Lmax)
        coords = torch.empty((B, 3 * Lmax, 3), dtype=torch.float32, device=angles.device)
        agg = torch.empty((B, 12), dtype=torch.float32, device=angles.device)
        _abi.tpl_backbone_segment_forward(angles, lengths, omega_prev if seg > 0 else None, coords, agg, ws)
        aggs = gather_stack(agg, group)
        _abi.tpl_backbone_segment_place(coords, lengths, aggs, seg, ws)
        ctx.save_for_backward(coords, lengths)
        ctx.group, ctx.seg, ctx.n_seg = group, seg, n_seg
        ctx.mark_non_differentiable(lengths)
        return coords

    @staticmethod
    def backward(ctx, grad_coords):
        from . import _abi
        from .api import MODEL_BACKBONE, default_workspace

        coords, lengths = ctx.saved_tensors
        B, Lmax = coords.shape[0], coords.shape[1] // 3
        grad_coords = grad_coords.contiguous()
        ws = default_workspace(coords.device).get(MODEL_BACKBONE, B, Lmax)
        tot = torch.empty((B, 12), dtype=torch.float32, device=coords.device)
        _abi.tpl_backbone_segment_totals(coords, lengths, grad_coords, tot, ws)
        tots = gather_stack(tot, ctx.group)
        grad_angles = torch.zeros((B, Lmax, 3), dtype=torch.float32, device=coords.device)
        _abi.tpl_backbone_segment_backward(coords, lengths, grad_coords, tots, ctx.seg, grad_angles, ws)
        return grad_angles, None, None, None


def sharded_backbone(angles, lengths, omega_prev=None, group=None):
    """This rank's residues [j0, j1) of every chain -> their coordinates in the
    chain frame (autograd).  omega_prev [B]: omega_{j0-1} of each chain (the
    previous segment's last omega; ignored on rank 0)."""
    if omega_prev is None:
        omega_prev = torch.zeros(angles.shape[0], dtype=torch.float32, device=angles.device)
    return SegmentBackbone.apply(angles, lengths, omega_prev.contiguous(), group)
