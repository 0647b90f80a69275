#!/usr/bin/env python3
"""bench.py -- headline benchmark of the B200 angles->coordinates hot path.

Metric (BASELINE.json): residues/s of forward+backward, backbone model,
L = 700, batch 256 per GPU, at N = 1/2/4/8 GPUs (weak scaling: every rank
runs its own 256-chain batch; nothing is exchanged on the data path), plus the
fraction of the HBM roofline of the dominant kernel.

    python bench.py [--steps K] [--warmup W] [--config metric|2|3|4|5]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...   (the fp64 oracle, timed on host cores)

One "step" = one tpl_*_forward + one tpl_*_backward over one batch with
synthetic inputs already resident in HBM.  Cold L2: the step rotates over
enough input/output buffer sets to exceed 4x the L2 size.  Each step set is
captured once in a CUDA graph; the timed region replays exactly K steps
bracketed by barrier + synchronize, timed with CUDA events on the launching
stream, max over ranks.  Prints ONE JSON line on rank 0.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

BWD_FROM = "coords"  # --bwd-from

BYTES_PER_RES = {  # algorithmic bytes
    # bwd: the operation's own bytes (angles + dL/dr in, dL/dangles out).  The kernel
    # reads the forward's coordinates instead of the angles (36 B, not 12): moved
    # bytes are 84/residue, but the roofline is charged the op's 60.
    "backbone": {"fwd": 12 + 36, "bwd": 12 + 36 + 12},
    "fullatom": {"fwd": None, "bwd": None},  # computed from the actual atom count
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference", "paper"],
                   help="paper: the paper's own GPU design (SURVEY f3; saved M_i + O(L^2) backward), backbone only")
    p.add_argument("--config", default="metric")
    p.add_argument("--repeats", type=int, default=7, help="timed regions of K steps; the median is reported")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU seconds of the cpu_baseline sample")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-parity", action="store_true", help="skip the oracle parity leg (A/B timing runs only)")
    p.add_argument("--bwd-from", default="coords", choices=["coords", "angles"],
                   help="backward entry point: from the forward's coordinates (the autograd layers' path, "
                        "default) or from the angles (stateless; reads 12 / 33 B/res of angles instead)")
    p.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                   help="strong (default, the metric's definition: the config's batch sharded over the "
                        "ranks, contiguous or LPT); weak: every rank runs the whole batch")
    return p.parse_args()


def cfg_key(c):
    if isinstance(c, str) and ":" in c:
        return synth.register_custom(c)
    return c if c in synth.CONFIGS else int(c)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- distributed
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and world == 1:
        raise SystemExit("--gpus N > 1 needs torchrun --nproc-per-node N (one process per GPU)")
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return world, rank, local, dist
    if torch.cuda.is_available():
        torch.cuda.set_device(0)
    return 1, 0, 0, None


def barrier(dist):
    if dist is not None:
        dist.barrier()


def _reduce_device(dist):
    return "cpu" if dist is not None and dist.get_backend() == "gloo" else "cuda"


def max_over_ranks(x, dist):
    """The timed region's max over ranks; one float64 all-reduce."""
    if dist is None:
        return x
    from paper_1812_01108_b200 import dist as tdist

    return tdist.reduce_scalar(x, "max", dist, _reduce_device(dist))


def sum_over_ranks(x, dist):
    if dist is None:
        return x
    from paper_1812_01108_b200 import dist as tdist

    return tdist.reduce_scalar(x, "sum", dist, _reduce_device(dist))


def shard_for_rank(lengths, world, rank):
    """Chains of this rank under strong scaling: contiguous ranges for uniform lengths,
    LPT by length for ragged batches (paper_1812_01108_b200/dist.py)."""
    from paper_1812_01108_b200 import dist as tdist

    return torch.tensor(tdist.plan([int(x) for x in lengths], world)[rank], dtype=torch.long)


# --------------------------------------------------------------- workloads
class BackboneWork:
    model = "backbone"
    launches_per_step = 2

    def __init__(self, c, rank, world=1, strong=False):
        cfg = synth.CONFIGS[c]
        self.cfg = cfg
        ang, lengths, grad = synth.backbone_inputs(c)
        if strong and world > 1:
            # strong scaling: the config's batch is split (LPT for ragged lengths)
            idx = shard_for_rank(lengths, world, rank)
            ang, lengths, grad = ang[idx].contiguous(), lengths[idx].contiguous(), grad[idx].contiguous()
        elif rank:
            # weak scaling: rank r draws its own batch (seed offset by rank)
            ang = synth.angles_uniform(ang.shape[0], ang.shape[1], 3, 1000 + synth.config_id(c) + 7919 * rank)
        self.host = dict(angles=ang, lengths=lengths, grad=grad)
        self.B, self.Lmax = ang.shape[0], ang.shape[1]
        self.residues = int(lengths.sum())

    def alloc_set(self, ws_bytes):
        from paper_1812_01108_b200 import _abi

        h = self.host
        s = dict(angles=h["angles"].cuda(), lengths=h["lengths"].cuda(), grad=h["grad"].cuda(),
                 coords=torch.empty((self.B, 3 * self.Lmax, 3), device="cuda"),
                 gang=torch.zeros((self.B, self.Lmax, 3), device="cuda"),
                 ws=torch.zeros(_abi.tpl_workspace_bytes(0, self.B, self.Lmax), dtype=torch.uint8, device="cuda"))
        return s

    def footprint(self):
        return self.B * self.Lmax * (12 + 36 + 36 + 12)

    def fwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        _abi.tpl_backbone_forward(s["angles"], s["lengths"], s["coords"], s["ws"], stream)

    def bwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        if BWD_FROM == "angles":  # stateless: recompute the forward from the angles
            _abi.tpl_backbone_backward(s["angles"], s["lengths"], s["grad"], s["gang"], s["ws"], stream)
            return
        # the autograd layer's backward: from the forward's coordinates
        _abi.tpl_backbone_backward_from_coords(s["coords"], s["lengths"], s["grad"], s["gang"], s["ws"], stream)

    def algo_bytes(self):
        return {k: v * self.residues for k, v in BYTES_PER_RES["backbone"].items()}

    def e2e_io(self):
        h = self.host
        return ([("angles", h["angles"]), ("grad", h["grad"])], [("coords", (self.B, 3 * self.Lmax, 3)),
                                                                  ("gang", (self.B, self.Lmax, 3))])

    def config(self):
        return {"workload": f"backbone phi,psi,omega -> N,CA,C; L={self.Lmax}, batch {self.B} per GPU",
                "L": self.Lmax, "batch_per_gpu": self.B}


class LossBackboneWork(BackboneWork):
    """f1: the step a structure-prediction model takes -- forward, LRMSD against a
    target (PAPER 4), its gradient, backward.  One pass: angles and the
    target in, LRMSD and dLRMSD/dangles out (tpl_backbone_lrmsd_fused, no coordinate
    round-trip); the backward is the chain rule's per-chain scale (tpl_chain_scale)."""
    launches_per_step = 2  # one-pass kernel, per-chain scale

    def __init__(self, c, rank, world=1, strong=False):
        super().__init__(c, rank, world, strong)
        self.host["target"] = synth.grad_normal((self.B, 3 * self.Lmax, 3), 5000 + synth.config_id(c) + 7919 * rank)

    def alloc_set(self, ws_bytes):
        s = super().alloc_set(ws_bytes)
        s["target"] = self.host["target"].cuda()
        s["loss"] = torch.empty(self.B, device="cuda")
        s["state"] = torch.empty(self.B, 16, device="cuda")
        s["gl"] = torch.ones(self.B, device="cuda")
        s["dlda"] = torch.zeros((self.B, self.Lmax, 3), device="cuda")
        return s

    def footprint(self):
        return self.B * self.Lmax * (12 + 36 + 12 + 12)

    def fwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        _abi.tpl_backbone_lrmsd_fused(s["angles"], s["lengths"], s["target"], None, s["loss"], s["state"],
                                      s["dlda"], s["ws"], stream)

    def bwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        _abi.tpl_chain_scale(s["dlda"], s["gl"], s["gang"], stream)

    def algo_bytes(self):
        # one pass: angles + target in, dLRMSD/dangles out; backward: read it, write dL/dangles
        r = self.residues
        return {"fwd": r * (12 + 36 + 12), "bwd": r * (12 + 12)}

    def e2e_io(self):
        h = self.host
        return ([("angles", h["angles"]), ("target", h["target"])], [("loss", (self.B,)), ("gang", (self.B, self.Lmax, 3))])

    def config(self):
        d = super().config()
        d["workload"] += "; LRMSD loss vs a synthetic target, one-pass angles -> LRMSD -> dLRMSD/dangles kernel"
        return d


class PaperBackboneWork(BackboneWork):
    """the paper's GPU design on the same workload -- forward saves M_i
    (64 B/atom), backward sums Eq. 2 per angle without a reduction."""

    def alloc_set(self, ws_bytes):
        from paper_1812_01108_b200 import _abi

        s = super().alloc_set(ws_bytes)
        s["M"] = torch.empty(_abi.tpl_paper_backbone_saved_floats(self.B, self.Lmax), device="cuda")
        return s

    def footprint(self):
        return super().footprint() + self.B * self.Lmax * 3 * 64

    def fwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        _abi.tpl_paper_backbone_forward(s["angles"], s["lengths"], s["coords"], s["M"], s["ws"], stream)

    def bwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        _abi.tpl_paper_backbone_backward(s["angles"], s["lengths"], s["M"], s["grad"], s["gang"], s["ws"], stream)


class FullAtomWork:
    model = "fullatom"
    launches_per_step = 2

    def __init__(self, c, rank, world=1, strong=False):
        import paper_1812_01108_b200 as tpl

        cfg = synth.CONFIGS[c]
        self.cfg = cfg
        B = cfg["B"]
        ang, rt, lengths = synth.fullatom_inputs(c, B=B)
        if strong and world > 1:
            idx = shard_for_rank(lengths, world, rank)
            ang, rt, lengths = ang[idx].contiguous(), rt[idx].contiguous(), lengths[idx].contiguous()
            B = len(idx)
        elif rank:
            ang = synth.angles_uniform(B, cfg["L"], 8, 1000 + synth.config_id(c) + 7919 * rank)
            rt = synth.restype_uniform(B, cfg["L"], 20, 4000 + synth.config_id(c) + 7919 * rank)
        self.table = synth.load_residue_table()
        self.tables = tpl.Tables(self.table)
        apc, stride = self.tables.atoms(rt, lengths)
        self.stride = stride
        self.atoms = int(apc.sum())
        grad = synth.fullatom_grad(B, stride, synth.config_id(c))
        self.host = dict(angles=ang, restype=rt, lengths=lengths, grad=grad)
        self.B, self.Lmax = B, cfg["L"]
        self.residues = int(lengths.sum())

    def alloc_set(self, ws_bytes):
        from paper_1812_01108_b200 import _abi

        h = self.host
        return dict(angles=h["angles"].cuda(), restype=h["restype"].cuda(), lengths=h["lengths"].cuda(),
                    grad=h["grad"].cuda(), coords=torch.empty((self.B, self.stride, 3), device="cuda"),
                    gang=torch.zeros((self.B, self.Lmax, 8), device="cuda"),
                    ws=torch.zeros(_abi.tpl_workspace_bytes(1, self.B, self.Lmax), dtype=torch.uint8,
                                   device="cuda"))

    def footprint(self):
        return self.B * self.Lmax * (32 + 1 + 32) + self.B * self.stride * 24

    def fwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        _abi.tpl_fullatom_forward(self.tables.handle, s["angles"], s["restype"], s["lengths"], s["coords"], s["ws"],
                                  stream)

    def bwd(self, s, stream=None):
        from paper_1812_01108_b200 import _abi

        if BWD_FROM == "angles":  # stateless: recompute the forward from the angles
            _abi.tpl_fullatom_backward(self.tables.handle, s["angles"], s["restype"], s["lengths"], s["grad"],
                                       s["gang"], s["ws"], stream)
            return
        # the autograd layer's backward: from the forward's coordinates
        _abi.tpl_fullatom_backward_from_coords(self.tables.handle, s["coords"], s["restype"], s["lengths"],
                                               s["grad"], s["gang"], s["ws"], stream)

    def algo_bytes(self):
        # the op's bytes; the coordinate backward moves r * 33 + a * 24 (reads coords, not angles)
        r, a = self.residues, self.atoms
        return {"fwd": r * (32 + 1) + a * 12, "bwd": r * (32 + 1 + 32) + a * 12}

    def e2e_io(self):
        h = self.host
        return ([("angles", h["angles"]), ("restype", h["restype"]), ("grad", h["grad"])],
                [("coords", (self.B, self.stride, 3)), ("gang", (self.B, self.Lmax, 8))])

    def config(self):
        return {"workload": f"full-atom phi,psi,omega,chi1-5 -> heavy atoms; 20 random residue types; "
                            f"L={self.Lmax}, batch {self.B} per GPU", "L": self.Lmax, "batch_per_gpu": self.B,
                "atoms_per_gpu": self.atoms}


def make_work(c, rank, world=1, strong=False, paper=False):
    if paper:
        if synth.CONFIGS[c]["model"] != "backbone":
            raise SystemExit("--impl paper: the paper's GPU design is the backbone model (its full atom ran on CPU)")
        return PaperBackboneWork(c, rank, world, strong)
    if synth.CONFIGS[c].get("loss") == "lrmsd":
        return LossBackboneWork(c, rank, world, strong)
    cls = BackboneWork if synth.CONFIGS[c]["model"] == "backbone" else FullAtomWork
    return cls(c, rank, world, strong)


# --------------------------------------------------------------- graphs
def capture(work, sets, steps, which):
    """A CUDA graph of `steps` consecutive steps over the rotating sets."""
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for i in range(steps):
                s = sets[i % len(sets)]
                if which in ("step", "fwd"):
                    work.fwd(s)
                if which in ("step", "bwd"):
                    work.bwd(s)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    return g


def timed_replays(graphs, dist):
    """Replay the graph list once inside barrier + sync brackets; CUDA-event ms."""
    barrier(dist)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for g in graphs:
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    barrier(dist)
    return e0.elapsed_time(e1)


def run_ours(args):
    import paper_1812_01108_b200 as tpl  # noqa: F401  (fails loudly without libtpl.so)

    world, rank, local, dist = dist_setup(args)
    c = cfg_key(args.config)
    work = make_work(c, rank, world, args.scaling == "strong", paper=args.impl == "paper")
    props = torch.cuda.get_device_properties(local)
    l2 = getattr(props, "L2_cache_size", 126 * 2 ** 20)
    n_sets = max(2, math.ceil(4 * l2 / work.footprint()))
    n_sets = min(n_sets, max(2, int(0.5 * props.total_memory / work.footprint())))
    sets = [work.alloc_set(0) for _ in range(n_sets)]
    torch.cuda.synchronize()
    K, W = args.steps, args.warmup

    # warm-up (also sets kernel attributes before capture)
    for i in range(max(W, 3)):
        work.fwd(sets[i % n_sets])
        work.bwd(sets[i % n_sets])
    torch.cuda.synchronize()
    from paper_1812_01108_b200 import _abi

    _abi.tpl_sync_status(sets[0]["ws"])

    def graphs_for(which):
        full, rem = divmod(K, n_sets)
        gs = []
        if full:
            g = capture(work, sets, n_sets, which)
            gs += [g] * full
        if rem:
            gs.append(capture(work, sets, rem, which))
        return gs

    step_graphs = graphs_for("step")
    fwd_graphs = graphs_for("fwd")
    bwd_graphs = graphs_for("bwd")
    # graph warm-up
    for g in set(step_graphs):
        g.replay()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    t_step, t_fwd, t_bwd = [], [], []
    t_end = time.time() + 1.0
    r = 0
    while r < args.repeats or time.time() < t_end:
        t_step.append(max_over_ranks(timed_replays(step_graphs, dist), dist))
        t_fwd.append(max_over_ranks(timed_replays(fwd_graphs, dist), dist))
        t_bwd.append(max_over_ranks(timed_replays(bwd_graphs, dist), dist))
        r += 1
        if r >= 200:
            break
    clocks = sampler.stop()
    ms_step = statistics.median(t_step) / K
    if len(t_step) > 1:  # 95% CI of the mean step time over the timed regions (P:248 reports CIs)
        mean, sd = statistics.mean(t_step) / K, statistics.stdev(t_step) / K
        ci95 = [mean - 1.96 * sd / math.sqrt(len(t_step)), mean + 1.96 * sd / math.sqrt(len(t_step))]
    else:
        ci95 = None
    ms_fwd = statistics.median(t_fwd) / K
    ms_bwd = statistics.median(t_bwd) / K
    for s in sets[:1]:
        _abi.tpl_sync_status(s["ws"])

    residues_all = sum_over_ranks(work.residues, dist)
    value = residues_all / (ms_step * 1e-3)

    # e2e: the same step through the public binding with pinned HOST buffers,
    # H2D of the inputs and D2H of the results inside the timed region.
    e2e = None
    if not args.no_e2e:
        # Every step copies its inputs from pinned host memory and its results back.
        # Steps are pipelined over 3 buffer slots and 3 streams (H2D, compute, D2H):
        # the copy engines run both directions while the kernels compute.
        ins, outs = work.e2e_io()
        n_slot = min(3, n_sets)
        host_in = [{k: v.pin_memory() for k, v in ins} for _ in range(n_slot)]
        host_out = [{k: torch.empty(shape, dtype=torch.float32).pin_memory() for k, shape in outs}
                    for _ in range(n_slot)]
        h2d = sum(v.numel() * v.element_size() for v in host_in[0].values())
        d2h = sum(v.numel() * v.element_size() for v in host_out[0].values())
        Ke = max(6, min(K, 60))
        st_in, st_run, st_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev = {n: [torch.cuda.Event() for _ in range(n_slot)] for n in ("in", "run", "out")}
        used = [False] * n_slot

        def e2e_step(k):
            i = k % n_slot
            s = sets[i]
            with torch.cuda.stream(st_in):
                if used[i]:
                    st_in.wait_event(ev["run"][i])  # the slot's inputs were consumed
                for name, v in host_in[i].items():
                    s[name].copy_(v, non_blocking=True)
                ev["in"][i].record(st_in)
            with torch.cuda.stream(st_run):
                st_run.wait_event(ev["in"][i])
                if used[i]:
                    st_run.wait_event(ev["out"][i])  # the slot's previous results were read back
                work.fwd(s, st_run)
                work.bwd(s, st_run)
                ev["run"][i].record(st_run)
            with torch.cuda.stream(st_out):
                st_out.wait_event(ev["run"][i])
                for name, v in host_out[i].items():
                    v.copy_(s[name], non_blocking=True)
                ev["out"][i].record(st_out)
            used[i] = True

        for k in range(2 * n_slot):
            e2e_step(k)
        torch.cuda.synchronize()
        barrier(dist)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st_in)
        for k in range(Ke):
            e2e_step(k)
        st_in.wait_stream(st_out)
        e1.record(st_in)
        torch.cuda.synchronize()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / Ke, dist)
        e2e = {"value": residues_all / (ms_e2e * 1e-3), "unit": "residues/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ms_e2e, "steps": Ke,
               "path": "pinned host -> cudaMemcpyAsync -> tpl_*_forward/backward (C ABI) -> pinned host; "
                       f"{n_slot} slots pipelined over H2D / compute / D2H streams"}

    # roofline of the dominant kernel
    peak, peak_src = load_peaks()
    ab = work.algo_bytes()
    dom = "bwd" if ms_bwd >= ms_fwd else "fwd"
    ms_dom = ms_bwd if dom == "bwd" else ms_fwd
    achieved = ab[dom] / (ms_dom * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{work.model}_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(dom)
    roof = {"bound": "hbm", "kernel": f"{work.model}_{dom}", "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "algorithmic_bytes_per_launch": int(ab[dom]), "ms_per_launch": ms_dom, "peak_source": peak_src,
            "fwd": {"ms": ms_fwd, "GB/s": ab["fwd"] / (ms_fwd * 1e-3) / 1e9},
            "bwd": {"ms": ms_bwd, "GB/s": ab["bwd"] / (ms_bwd * 1e-3) / 1e9},
            "step_GB/s": (ab["fwd"] + ab["bwd"]) / (ms_step * 1e-3) / 1e9,
            "step_frac": (ab["fwd"] + ab["bwd"]) / (ms_step * 1e-3) / 1e9 / peak}

    parity = None
    if not args.no_parity:
        parity = parity_leg(work, sets[0], c, dist)

    cpu = None
    # the oracle's O(L^2) backward makes a 20000-residue chain a minute of CPU: no sample for "long";
    # the loss config's oracle would time the same backbone work as the metric config
    skip_cpu = args.impl == "paper" or work.Lmax > 5000 or isinstance(work, LossBackboneWork)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not skip_cpu:
        cpu = cpu_baseline(work, args.cpu_seconds)

    if rank == 0:
        cfgd = work.config()
        gb = work.cfg["B"] if args.scaling == "strong" else work.B * world
        cfgd.update({"global_batch": gb, "parallelism": f"dp{world} (chains sharded, no collective)",
                     "l2_flush": f"rotating buffer sets: a timed region of K={K} steps touches {min(K, n_sets)} of "
                                 f"{n_sets} sets ({min(K, n_sets) * work.footprint() / 2**20:.0f} MiB; L2 "
                                 f"{l2 / 2**20:.0f} MiB), each set reused only after {min(K, n_sets) - 1} others",
                     "timing": f"CUDA graphs of K steps, median of {len(t_step)} timed regions"})
        out = {"metric": f"residues/sec fwd+bwd ({work.model}, L={work.Lmax}, batch {gb})",
               "value": value, "unit": "residues/s", "n_gpus": world, "steps": K, "warmup": W,
               "ms_per_step": ms_step, "ms_per_step_ci95": ci95, "higher_is_better": True,
               "scaling": args.scaling, "vs_baseline": None,
               "dtype": "f32", "data": "synthetic (seeded uniform angles, N(0,1) dL/dr)", "config": cfgd,
               "roofline": roof, "parity": parity, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": work.launches_per_step * K,
               "impl": "paper_gpu_design" if args.impl == "paper" else "ours"}
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


# --------------------------------------------------------------- oracle legs
def parity_chains(work, cfg_name):
    """every chain for the small configs, else 64 seeded chains including the longest."""
    B = work.B
    ln = work.host["lengths"].numpy()
    if cfg_name in ("metric", "lrmsd", "long", 1, 2, 3) or B <= 64:
        return np.arange(B)
    rng = np.random.default_rng(6000 + synth.config_id(cfg_name))
    pick = set(rng.choice(B, size=63, replace=False).tolist())
    pick.add(int(np.argmax(ln)))
    return np.array(sorted(pick))[:64]


def parity_leg(work, s, cfg_name, dist):
    """The bench's own correctness check: one more fwd+bwd on
    the first buffer set -- the inputs the timed region used -- compared element by
    element with the fp64 oracle on a bounded set of chains.  Gates (north_star):
    coordinates <= 1e-3 A for L <= 1000 (5e-3 A beyond, reading Q21), per-chain
    norm-wise gradient error <= 1e-3 (reading Q18).  MAX over ranks."""
    import oracle

    oracle.build()
    work.fwd(s)
    work.bwd(s)
    torch.cuda.synchronize()
    idx = parity_chains(work, cfg_name)
    h = work.host
    a64 = synth.numpy64(h["angles"])[idx]
    ln = h["lengths"].numpy()[idx]
    coords = s["coords"].cpu().numpy()[idx]
    gang = s["gang"].cpu().numpy()[idx]
    check_grad = int(ln.max()) <= 5000  # the O(L^2) oracle backward of one 20000-residue chain is minutes
    coord_err, grad_err, coord_err_long = 0.0, 0.0, 0.0
    loss_err = None
    if work.model == "backbone":
        X = oracle.backbone_forward(a64, ln)
        if isinstance(work, LossBackboneWork):
            from oracle import lrmsd as olr

            tgt = synth.numpy64(h["target"])[idx]
            vals, dldr = olr.batch(X, tgt, 3 * ln)
            loss = s["loss"].cpu().numpy()[idx]
            loss_err = float(np.max(np.abs(loss - vals) / np.maximum(np.abs(vals), 1e-12)))
            G = oracle.backbone_backward(a64, ln, dldr) if check_grad else None
        else:
            G = oracle.backbone_backward(a64, ln, synth.numpy64(h["grad"])[idx]) if check_grad else None
        for k, L in enumerate(ln):
            if isinstance(work, LossBackboneWork):
                break  # the one-pass kernel writes no coordinates (checked through the loss and its gradient)
            e = float(np.abs(coords[k, : 3 * L] - X[k, : 3 * L]).max())
            if L <= 1000:
                coord_err = max(coord_err, e)
            else:
                coord_err_long = max(coord_err_long, e)
    else:
        rt = h["restype"].numpy()[idx]
        X, nat = oracle.fullatom_forward(work.table, a64, rt, ln, work.stride)
        G = oracle.fullatom_backward(work.table, a64, rt, ln, synth.numpy64(h["grad"])[idx]) if check_grad else None
        for k, L in enumerate(ln):
            e = float(np.abs(coords[k, : nat[k]] - X[k, : nat[k]]).max())
            if L <= 1000:
                coord_err = max(coord_err, e)
            else:
                coord_err_long = max(coord_err_long, e)
    if G is not None:
        for k in range(len(idx)):
            den = float(np.abs(G[k]).max())
            if den > 0:
                grad_err = max(grad_err, float(np.abs(gang[k] - G[k]).max()) / den)
    vals = [coord_err, coord_err_long, grad_err, loss_err or 0.0, float(len(idx))]
    if dist is not None:
        t = torch.tensor(vals[:4], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n = torch.tensor([vals[4]], dtype=torch.float64, device="cuda")
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
        vals = t.tolist() + n.tolist()
    ok = vals[0] <= 1e-3 and vals[1] <= 5e-3 and (G is None or vals[2] <= 1e-3) and (loss_err is None or vals[3] <= 1e-4)
    out = {"chains": int(vals[4]), "max_coord_err_A": vals[0], "max_grad_rel_err": vals[2] if G is not None else None,
           "ok": bool(ok), "gate": "coords <= 1e-3 A (L <= 1000), grad <= 1e-3 per-chain norm-wise (Q18)",
           "inputs": "the timed region's first buffer set, vs the fp64 oracle"}
    if coord_err_long or int(ln.max()) > 1000:
        out["max_coord_err_A_L_gt_1000"] = vals[1]
    if loss_err is not None:
        out["max_loss_rel_err"] = vals[3]
    return out


def cpu_baseline(work, seconds):
    """The fp64 oracle as it stands (paper-literal O(L^2) backward, OpenMP over
    chains) on this host's cores, on a bounded sample of the same workload."""
    import oracle

    oracle.build()
    h = work.host
    a64 = synth.numpy64(h["angles"])
    g64 = synth.numpy64(h["grad"])
    ln = h["lengths"].numpy()
    B = a64.shape[0]
    threads = oracle.num_threads()

    def run(idx):
        if work.model == "backbone":
            oracle.backbone_forward(a64[idx], ln[idx])
            oracle.backbone_backward(a64[idx], ln[idx], g64[idx])
        else:
            rt = h["restype"].numpy()
            oracle.fullatom_forward(work.table, a64[idx], rt[idx], ln[idx], work.stride)
            oracle.fullatom_backward(work.table, a64[idx], rt[idx], ln[idx], g64[idx])

    # calibrate on `threads` chains, then size the sample to ~`seconds`: a prefix
    # of the batch, or the whole batch repeated when it takes less than that
    idx = np.arange(min(B, threads))
    t0 = time.perf_counter()
    run(idx)
    t1 = time.perf_counter() - t0
    n = int(min(B, max(threads, threads * math.floor(seconds / max(t1, 1e-3)))))
    reps = 1 if n < B else max(1, int(seconds / max(t1 * B / threads, 1e-3)))
    idx = np.arange(n)
    t0 = time.perf_counter()
    for _ in range(reps):
        run(idx)
    dt = time.perf_counter() - t0
    res = float(ln[idx].sum()) * reps
    what = f"{n} of {B} chains" if n < B else f"the whole {B}-chain batch x {reps}"
    # the 1-thread rate on a short sample: chains in order until ~2 s
    oracle.set_num_threads(1)
    t0, res1, i = time.perf_counter(), 0.0, 0
    while time.perf_counter() - t0 < 2.0 and i < 4 * B:
        run(np.array([i % B]))
        res1 += float(ln[i % B])
        i += 1
    one = res1 / (time.perf_counter() - t0)
    oracle.set_num_threads(threads)
    return {"value": res / dt, "unit": "residues/s", "cores": threads, "kind": "oracle",
            "sample": f"{what} (fwd + O(L^2) Eq. 2/Eq. 1 bwd, fp64), {dt:.1f} s", "host_cpus": os.cpu_count(),
            "single_thread_value": one, "single_thread_sample": f"{i} chains, 1 thread"}


def ref_config(work, cfg, n):
    """The same config keys and workload text as the GPU arm (run_ours)."""
    if work.model == "backbone":
        d = {"workload": f"backbone phi,psi,omega -> N,CA,C; L={cfg['L']}, batch {cfg['B']} per GPU",
             "L": cfg["L"], "batch_per_gpu": cfg["B"]}
    else:
        d = {"workload": f"full-atom phi,psi,omega,chi1-5 -> heavy atoms; 20 random residue types; "
                         f"L={cfg['L']}, batch {cfg['B']} per GPU", "L": cfg["L"], "batch_per_gpu": cfg["B"]}
    d.update({"global_batch": cfg["B"], "parallelism": "host cores (OpenMP over chains)",
              "sample_chains_per_step": n})
    return d


def run_reference(args):
    """--impl reference: the oracle timed as the reference arm (rank 0 only)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    oracle.build()
    c = cfg_key(args.config)
    cfg = synth.CONFIGS[c]

    class H:  # host-only view of the workload (no GPU needed)
        pass

    work = H()
    work.model = cfg["model"]
    if work.model == "backbone":
        ang, lengths, grad = synth.backbone_inputs(c)
    else:
        ang, rt, lengths = synth.fullatom_inputs(c)
        work.table = synth.load_residue_table()
        na = oracle.chain_atom_counts(work.table, rt.numpy(), lengths.numpy())
        work.stride = int(na.max())
        grad = synth.fullatom_grad(ang.shape[0], work.stride, synth.config_id(c))
        work.host_rt = rt
    a64, g64, ln = synth.numpy64(ang), synth.numpy64(grad), lengths.numpy()
    threads = oracle.num_threads()
    K, W = args.steps, args.warmup

    def run(idx):
        if work.model == "backbone":
            oracle.backbone_forward(a64[idx], ln[idx])
            oracle.backbone_backward(a64[idx], ln[idx], g64[idx])
        else:
            r = work.host_rt.numpy()
            oracle.fullatom_forward(work.table, a64[idx], r[idx], ln[idx], work.stride)
            oracle.fullatom_backward(work.table, a64[idx], r[idx], ln[idx], g64[idx])

    B = a64.shape[0]
    t0 = time.perf_counter()
    run(np.arange(min(B, threads)))
    t1 = time.perf_counter() - t0
    budget = 150.0  # seconds for the whole K + W run
    per_step = budget / max(1, K + W)
    n = int(max(1, min(B, threads * math.floor(per_step / max(t1, 1e-3))))) if per_step >= t1 else max(
        1, int(threads * per_step / max(t1, 1e-3)))
    n = min(n, B)
    times, res = [], 0.0
    for i in range(W + K):
        idx = (np.arange(n) + i * n) % B
        s = time.perf_counter()
        run(idx)
        e = time.perf_counter() - s
        if i >= W:
            times.append(e)
            res += float(ln[idx].sum())
    total = sum(times)
    value = res / total
    line = {"metric": f"residues/sec fwd+bwd ({work.model}, L={cfg['L']}, batch {cfg['B']})", "value": value,
            "unit": "residues/s", "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": 1e3 * total / K,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform angles, N(0,1) dL/dr)",
            "config": ref_config(work, cfg, n),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "residues/s", "cores": threads, "kind": "oracle",
                             "sample": f"{n} chains per step of the {cfg['B']}-chain workload"},
            "e2e": {"value": value, "unit": "residues/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    global BWD_FROM
    args = parse()
    BWD_FROM = args.bwd_from
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
