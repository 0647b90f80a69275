"""GPU parity of the LRMSD kernels (PAPER §4) and of the angles -> coords -> LRMSD
-> dL/dangles pipeline, against the fp64 oracle."""
import numpy as np
import pytest
import torch

import synth
from oracle import lrmsd as OL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tpl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_01108_b200 import build

    build.build()
    import paper_1812_01108_b200 as tpl

    return tpl


def test_lrmsd_values_and_gradients(tpl):
    from paper_1812_01108_b200 import _abi

    rng = np.random.default_rng(0)
    B, S = 6, 2100
    x = (rng.standard_normal((B, S, 3)) * 20).astype(np.float32)
    y = (rng.standard_normal((B, S, 3)) * 20).astype(np.float32)
    n = np.array([2100, 1, 2, 3, 700, 2099], dtype=np.int32)
    xt, yt, nt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(n).cuda()
    out = torch.empty(B, device="cuda")
    state = torch.empty(B, 16, device="cuda")
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    _abi.tpl_lrmsd_forward(xt, yt, nt, out, state, ws)
    g = torch.full((B, S, 3), float("nan"), device="cuda")
    go = torch.linspace(0.5, 2.0, B, device="cuda")
    _abi.tpl_lrmsd_backward(xt, yt, nt, state, go, g, ws)
    _abi.tpl_sync_status(ws)
    vals, grads = OL.batch(x.astype(np.float64), y.astype(np.float64), n)
    o = out.cpu().numpy()
    gg = g.cpu().numpy()
    for b in range(B):
        k = int(n[b])
        assert abs(o[b] - vals[b]) <= 1e-5 * max(1.0, vals[b]), (b, o[b], vals[b])
        if k >= 3:
            ref = grads[b, :k] * float(go[b])
            assert np.abs(gg[b, :k] - ref).max() <= 1e-4 * np.abs(ref).max()
        assert np.isnan(gg[b, k:]).all()  # atoms past n_atoms untouched


def test_rigid_copy_is_zero(tpl):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 500, 3)) * 15
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    y = x @ OL.rotation(q).T + np.array([3.0, -7.0, 11.0])
    v = tpl.lrmsd(torch.tensor(x, dtype=torch.float32).cuda(), torch.tensor(y, dtype=torch.float32).cuda())
    assert float(v[0]) < 2e-3


def test_pipeline_angles_to_lrmsd_gradient(tpl, oracle_lib):
    """dLRMSD/dangles through backbone -> LRMSD on the GPU == oracle backbone +
    oracle LRMSD gradient + oracle Eq. 2."""
    B, L = 4, 300
    ang = synth.angles_uniform(B, L, 3, 31)
    ref = synth.angles_uniform(B, L, 3, 32)
    ln = torch.full((B,), L, dtype=torch.int32)
    target = tpl.backbone(ref.cuda(), ln.cuda()).detach()
    a = ang.cuda().requires_grad_(True)
    coords = tpl.backbone(a, ln.cuda())
    loss = tpl.lrmsd(coords, target).sum()
    loss.backward()
    a64 = synth.numpy64(ang)
    X = oracle_lib.backbone_forward(a64, ln.numpy())
    Y = target.cpu().numpy().astype(np.float64)
    vals, gx = OL.batch(X, Y, [3 * L] * B)
    G = oracle_lib.backbone_backward(a64, ln.numpy(), gx)
    g = a.grad.cpu().numpy()
    for b in range(B):
        assert np.abs(g[b] - G[b]).max() / np.abs(G[b]).max() <= 2e-3
    assert abs(float(loss.detach()) - vals.sum()) <= 1e-3 * vals.sum()


@pytest.mark.parametrize("B,L,lengths", [(4, 300, None), (5, 700, [700, 1, 2, 350, 699]), (2, 2300, [2300, 1500])])
def test_fused_backbone_lrmsd(tpl, oracle_lib, B, L, lengths):
    """f1 fused (tpl_backbone_lrmsd_*): LRMSD values and dLRMSD/dangles == oracle
    backbone + oracle LRMSD (Q19) + oracle Eq. 2, ragged and multi-tile."""
    ang = synth.angles_uniform(B, L, 3, 41 + L)
    ref = synth.angles_uniform(B, L, 3, 42 + L)
    ln = torch.full((B,), L, dtype=torch.int32) if lengths is None else torch.tensor(lengths, dtype=torch.int32)
    target = tpl.backbone(ref.cuda(), ln.cuda()).detach()
    a = ang.cuda().requires_grad_(True)
    vals_gpu, coords = tpl.backbone_lrmsd(a, target, ln.cuda())
    gl = synth.grad_normal((B,), 43).abs() + 0.5  # dL/dLRMSD per chain
    (vals_gpu * gl.cuda()).sum().backward()
    a64, lnn = synth.numpy64(ang), ln.numpy()
    X = oracle_lib.backbone_forward(a64, lnn)
    Y = target.cpu().numpy().astype(np.float64)
    vals, gx = OL.batch(X, Y, [3 * int(l) for l in lnn])
    gx = gx * gl.numpy().astype(np.float64)[:, None, None]
    G = oracle_lib.backbone_backward(a64, lnn, gx)
    g = a.grad.cpu().numpy()
    v = vals_gpu.detach().cpu().numpy()
    for b in range(B):
        Lb = int(lnn[b])
        assert abs(v[b] - vals[b]) <= 1e-3 * max(vals[b], 1e-3), (b, v[b], vals[b])
        if Lb > 1:
            rel = np.abs(g[b, :Lb] - G[b, :Lb]).max() / np.abs(G[b, :Lb]).max()
            assert rel <= 2e-3, (b, rel)
        assert np.abs(coords[b, :3 * Lb].cpu().numpy() - X[b, :3 * Lb]).max() <= 5e-3
