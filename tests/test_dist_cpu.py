"""Multi-GPU host logic on the CPU: shard planning and the scalar reductions,
exercised in a world-size-2 gloo process group (127.0.0.1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_01108_b200 import dist as tdist


def test_contiguous_cover_and_balance():
    for n, w in ((256, 1), (256, 2), (256, 8), (10, 4), (3, 8)):
        sh = tdist.contiguous_shards(n, w)
        flat = [i for s in sh for i in s]
        assert flat == list(range(n))
        assert max(map(len, sh)) - min(map(len, sh)) <= 1


def test_lpt_cover_order_and_balance():
    rng = np.random.default_rng(0)
    lengths = rng.integers(50, 2001, size=4096)
    for w in (2, 4, 8):
        sh = tdist.lpt_shards(lengths, w)
        flat = sorted(i for s in sh for i in s)
        assert flat == list(range(4096))
        for s in sh:  # longest first inside a shard
            ls = [lengths[i] for i in s]
            assert ls == sorted(ls, reverse=True)
        assert tdist.imbalance(lengths, sh) < 1.01
    assert tdist.plan([700] * 10, 4) == tdist.contiguous_shards(10, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lengths = [int(x) for x in np.random.default_rng(1).integers(50, 2001, size=64)]
    shards = tdist.plan(lengths, world)
    mine = shards[rank]
    residues = sum(lengths[i] for i in mine)
    tot = tdist.reduce_scalar(residues, "sum", dist)
    mx = tdist.reduce_scalar(float(rank + 1) * 1.5, "max", dist)
    # every rank sees the same global plan: gather the chain ids and check coverage
    ids = [None] * world
    dist.all_gather_object(ids, mine)
    # f4 exchange step: rank r's record lands at index r of the stacked result
    stacked = tdist.gather_stack(torch.full((3, 12), float(rank)), None)
    order_ok = all(bool((stacked[r] == r).all()) for r in range(world))
    q.put((rank, tot, mx, sorted(i for s in ids for i in s), sum(lengths), order_ok))
    dist.destroy_process_group()


def test_gloo_world2_reductions_and_coverage():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tot, mx, ids, total, order_ok in res:
        assert order_ok
        assert tot == total
        assert mx == 3.0
        assert ids == list(range(64))


def test_segment_bounds():
    for L, w in ((700, 2), (700, 8), (8, 8), (20001, 3)):
        b = tdist.segment_bounds(L, w)
        assert b[0][0] == 0 and b[-1][1] == L
        assert all(hi > lo for lo, hi in b) and all(b[i][1] == b[i + 1][0] for i in range(w - 1))
        sizes = [hi - lo for lo, hi in b]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        tdist.segment_bounds(3, 4)


def _bench_worker(rank, world, port, q):
    """bench.py's own rank helpers under a gloo group: the strong-scaling shard of
    the metric config (256 x 700) and of config 4 (ragged), and the max / sum
    reductions the timed region and the residue count go through."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for c in ("metric", 4):
        if c == 4:
            lengths = synth.lengths_uniform(4096, 50, 2000, 3000 + 4)
        else:
            lengths = torch.full((256,), 700, dtype=torch.int32)
        idx = bench.shard_for_rank(lengths, world, rank)
        ids = [None] * world
        dist.all_gather_object(ids, idx.tolist())
        res = bench.sum_over_ranks(float(lengths[idx].sum()), dist)
        out[str(c)] = (sorted(i for s in ids for i in s), res, float(lengths.sum()),
                       [int(lengths[torch.tensor(s)].sum()) for s in ids])
    t = bench.max_over_ranks(1.0 + rank, dist)
    q.put((rank, out, t))
    dist.destroy_process_group()


def test_bench_rank_helpers_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, t in res:
        assert t == 2.0  # max over ranks of (1 + rank)
        ids, tot, ref, loads = out["metric"]
        assert ids == list(range(256)) and tot == ref and loads == [128 * 700, 128 * 700]
        ids, tot, ref, loads = out["4"]
        assert ids == list(range(4096)) and tot == ref
        assert max(loads) / (sum(loads) / world) < 1.01  # LPT balance of the ragged config
