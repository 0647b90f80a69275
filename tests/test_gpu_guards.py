"""Memory-safety and concurrency checks of our own (compute-sanitizer is closed on
this GPU pool: runs under it left GPUs needing a reset -- profiles/r02_sanitizer.md).

* Guard bands: every output (and workspace) of every kernel family lives inside a
  larger buffer whose margins hold a sentinel bit pattern; after the launches the
  margins must be bit-identical (no write outside the declared extents) and the
  pads inside (entries past a chain's length) untouched.
* Repeatability: the decoupled kernels (cross-CTA flags, epochs) and the packed
  kernels give bitwise identical results over repeated launches.
* Concurrency: the decoupled kernels assume their persistent grid's CTAs become
  co-resident; with another stream's kernels occupying SMs they must still finish
  with the solo-run bits (forward progress only needs the other work to drain).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
GUARD = 4096  # floats of margin on each side
SENT = -1.2345e-30


@pytest.fixture(scope="module")
def abi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_01108_b200 import _abi

    return _abi


class Guarded:
    """A tensor view inside a sentinel-filled allocation (16-byte aligned view)."""

    def __init__(self, shape, dtype=torch.float32, fill=float("nan")):
        n = int(np.prod(shape))
        self.base = torch.full((n + 2 * GUARD,), SENT, dtype=dtype, device="cuda") if dtype == torch.float32 else \
            torch.full((n + 2 * GUARD,), 0xA5, dtype=dtype, device="cuda")
        self.n = n
        self.view = self.base[GUARD:GUARD + n].view(shape)
        if dtype == torch.float32:
            self.view.fill_(fill)

    def margins_ok(self):
        b = self.base.cpu()
        lo, hi = b[:GUARD], b[GUARD + self.n:]
        if self.base.dtype == torch.float32:
            return bool((lo == SENT).all() and (hi == SENT).all())
        return bool((lo == 0xA5).all() and (hi == 0xA5).all())


def _ws(abi, model, B, L):
    w = Guarded((abi.tpl_workspace_bytes(model, B, L),), dtype=torch.uint8)
    w.view.zero_()
    return w


@pytest.mark.parametrize("B,Lmax", [(7, 300), (40, 701), (256, 700), (3, 1100), (150, 1400), (2, 5000), (1, 20000)])
def test_backbone_guard_bands(abi, B, Lmax):
    ln = synth.lengths_uniform(B, max(1, Lmax // 3), Lmax, 8100 + B)
    ln[0] = Lmax
    ang = synth.angles_uniform(B, Lmax, 3, 8101 + B).cuda()
    g = synth.grad_normal((B, 3 * Lmax, 3), 8102).cuda()
    c = Guarded((B, 3 * Lmax, 3))
    gx = Guarded((B, Lmax, 3))
    ga = Guarded((B, Lmax, 3))
    ws = _ws(abi, 0, B, Lmax)
    lnc = ln.cuda()
    abi.tpl_backbone_forward(ang, lnc, c.view, ws.view)
    abi.tpl_backbone_backward_from_coords(c.view, lnc, g, gx.view, ws.view)
    abi.tpl_backbone_backward(ang, lnc, g, ga.view, ws.view)
    abi.tpl_sync_status(ws.view)
    for t in (c, gx, ga, ws):
        assert t.margins_ok()
    cc, gg, aa = c.view.cpu().numpy(), gx.view.cpu().numpy(), ga.view.cpu().numpy()
    for b, L in enumerate(ln.tolist()):
        assert np.isnan(cc[b, 3 * L:]).all() and np.isnan(gg[b, L:]).all() and np.isnan(aa[b, L:]).all()
        assert np.isfinite(cc[b, :3 * L]).all() and np.isfinite(gg[b, :L]).all()


def test_lrmsd_and_scale_guard_bands(abi):
    B, Lmax = 12, 700
    ln = synth.lengths_uniform(B, 1, Lmax, 8201)
    ang = synth.angles_uniform(B, Lmax, 3, 8202).cuda()
    tgt = (synth.grad_normal((B, 3 * Lmax, 3), 8203) * 20).cuda()
    c, g = Guarded((B, 3 * Lmax, 3)), Guarded((B, Lmax, 3))
    out, st = Guarded((B,)), Guarded((B, 16))
    y = Guarded((B, Lmax, 3))
    ws = _ws(abi, 0, B, Lmax)
    abi.tpl_backbone_lrmsd_fused(ang, ln.cuda(), tgt, c.view, out.view, st.view, g.view, ws.view)
    abi.tpl_chain_scale(g.view, out.view, y.view)
    abi.tpl_sync_status(ws.view)
    for t in (c, g, out, st, y, ws):
        assert t.margins_ok()
    gg = g.view.cpu().numpy()
    for b, L in enumerate(ln.tolist()):
        assert np.isnan(gg[b, L:]).all()


def test_fullatom_guard_bands(abi, table):
    import paper_1812_01108_b200 as tpl

    tables = tpl.Tables(table)
    for B, L in ((64, 300), (300, 120)):
        ang, rt, ln = synth.fullatom_inputs(3, B=B, L=L)
        ln = synth.lengths_uniform(B, 1, L, 8300 + B)
        apc, stride = tables.atoms(rt, ln)
        c = Guarded((B, stride, 3))
        ga, gb = Guarded((B, L, 8)), Guarded((B, L, 8))
        g = synth.grad_normal((B, stride, 3), 8301).cuda()
        ws = _ws(abi, 1, B, L)
        a, r, l = ang.cuda(), rt.cuda(), ln.cuda()
        abi.tpl_fullatom_forward(tables.handle, a, r, l, c.view, ws.view)
        abi.tpl_fullatom_backward_from_coords(tables.handle, c.view, r, l, g, ga.view, ws.view)
        abi.tpl_fullatom_backward(tables.handle, a, r, l, g, gb.view, ws.view)
        abi.tpl_sync_status(ws.view)
        for t in (c, ga, gb, ws):
            assert t.margins_ok()
        cc = c.view.cpu().numpy()
        for b in range(B):
            assert np.isnan(cc[b, int(apc[b]):]).all()


def test_chain_serial_kernels_guard_bands():
    """The chain-serial / cluster kernels (TPL_PACKED=0; read once per process)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TPL_PACKED="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_guards.py"), "-k", "backbone_guard_bands"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def _run_bb(abi, ang, ln, g, stream=None):
    B, Lmax = ang.shape[:2]
    c = torch.empty(B, 3 * Lmax, 3, device="cuda")
    gx = torch.empty(B, Lmax, 3, device="cuda")
    ws = torch.zeros(abi.tpl_workspace_bytes(0, B, Lmax), dtype=torch.uint8, device="cuda")
    abi.tpl_backbone_forward(ang, ln, c, ws, stream)
    abi.tpl_backbone_backward_from_coords(c, ln, g, gx, ws, stream)
    return c, gx, ws


@pytest.mark.parametrize("B,Lmax", [(1, 20000), (64, 3000), (256, 700)])
def test_repeatable_and_concurrent(abi, B, Lmax):
    """Bitwise repeatability, then the same launches on a side stream while the
    default stream runs matmuls that occupy SMs: identical bits, no hang."""
    ang = synth.angles_uniform(B, Lmax, 3, 8400 + B).cuda()
    ln = torch.full((B,), Lmax, dtype=torch.int32, device="cuda")
    g = synth.grad_normal((B, 3 * Lmax, 3), 8401).cuda()
    c0, g0, ws = _run_bb(abi, ang, ln, g)
    abi.tpl_sync_status(ws)
    for _ in range(5):
        c1, g1, _ = _run_bb(abi, ang, ln, g)
        torch.cuda.synchronize()
        assert torch.equal(c0, c1) and torch.equal(g0, g1)
    side = torch.cuda.Stream()
    x = torch.randn(4096, 4096, device="cuda")
    outs = []
    for _ in range(3):
        y = x
        for _ in range(8):  # default stream: matmuls launched first, still running
            y = y @ x
            y = y / y.norm()
        with torch.cuda.stream(side):
            outs.append(_run_bb(abi, ang, ln, g, side))
    torch.cuda.synchronize()
    for c2, g2, _ in outs:
        assert torch.equal(c0, c2) and torch.equal(g0, g2)
