"""GPU parity of the backbone kernels (through the C ABI) against the fp64 oracle.

Gates (BASELINE.json north_star):
  coordinates: max |r_gpu - r_oracle| <= 1e-3 Å for L <= 1000 (identical fp32 inputs)
  gradients:   per chain max_i |g_gpu - g_ref| / max_i |g_ref| <= 1e-3   (reading Q18)
"""
import math

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

COORD_TOL = 1e-3
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def tpl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_01108_b200 import build

    build.build()
    import paper_1812_01108_b200 as tpl

    return tpl


def _run(tpl, ang, lengths, grad, sentinel=float("nan"), xyz=False):
    from paper_1812_01108_b200 import _abi

    B, Lmax, _ = ang.shape
    a = ang.cuda()
    ln = lengths.cuda()
    g = grad.cuda()
    coords = torch.full((B, 3 * Lmax, 3), sentinel, device="cuda")
    gang = torch.full((B, Lmax, 3), sentinel, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, Lmax), dtype=torch.uint8, device="cuda")
    if xyz:
        _abi.tpl_backbone_forward(a, ln, coords, ws)
        _abi.tpl_backbone_backward_from_coords(coords, ln, g, gang, ws)
    else:
        _abi.tpl_backbone_forward(a, ln, coords, ws)
        _abi.tpl_backbone_backward(a, ln, g, gang, ws)
    _abi.tpl_sync_status(ws)
    return coords.cpu().numpy(), gang.cpu().numpy()


def _check(oracle_lib, ang, lengths, grad, coords, gang, chains=None, coord_tol=COORD_TOL):
    B = ang.shape[0]
    chains = range(B) if chains is None else chains
    a64 = synth.numpy64(ang)
    g64 = synth.numpy64(grad)
    ln = lengths.numpy()
    idx = np.array(list(chains))
    X = oracle_lib.backbone_forward(a64[idx], ln[idx])
    G = oracle_lib.backbone_backward(a64[idx], ln[idx], g64[idx])
    worst_c, worst_g = 0.0, 0.0
    for n, b in enumerate(idx):
        L = int(ln[b])
        dc = np.abs(coords[b, : 3 * L] - X[n, : 3 * L]).max()
        ref = G[n, :L]
        dg = np.abs(gang[b, :L] - ref).max() / max(np.abs(ref).max(), 1e-30)
        worst_c, worst_g = max(worst_c, dc), max(worst_g, dg)
        tol = coord_tol if L <= 1000 else 5e-3  # reading Q21: L > 1000 is a target (1e-3), gated at 5e-3
        assert dc <= tol, f"chain {b} L={L}: coord err {dc:.3e}"
        assert dg <= GRAD_TOL, f"chain {b} L={L}: grad rel err {dg:.3e}"
        # structural zeros
        assert gang[b, L - 1, 1] == 0.0 and gang[b, L - 1, 2] == 0.0
    return worst_c, worst_g


def test_config1_single_chain_L16(tpl, oracle_lib):
    ang, lengths, grad = synth.backbone_inputs(1)
    coords, gang = _run(tpl, ang, lengths, grad)
    c, g = _check(oracle_lib, ang, lengths, grad, coords, gang)
    assert c < 1e-5 and g < 1e-5


def test_config1_gpu_finite_difference_sanity(tpl):
    """Coarse fp32 FD on the GPU forward (h = 1e-2 rad, central, <= 1e-2 relative):
    not a gate of the method (the oracle's FD pins Eq. 2), a check of the wiring."""
    ang, lengths, grad = synth.backbone_inputs(1)
    a = ang.double()
    coords, gang = _run(tpl, ang, lengths, grad)
    h = 1e-2
    fd = np.zeros_like(gang)
    for j in range(16):
        for k in range(3):
            ap, am = a.clone(), a.clone()
            ap[0, j, k] += h
            am[0, j, k] -= h
            cp, _ = _run(tpl, ap.float(), lengths, grad)
            cm, _ = _run(tpl, am.float(), lengths, grad)
            fd[0, j, k] = ((cp - cm) * grad.numpy()).sum() / (2 * h)
    rel = np.abs(fd - gang).max() / np.abs(gang).max()
    assert rel < 1e-2, rel


@pytest.mark.parametrize("Lmax,lengths", [
    (16, [16, 1, 2, 7]),
    (300, [300, 1, 255, 256, 257, 299]),      # RPT 2, ragged tails inside one tile
    (700, [700, 650, 512, 3]),                # RPT 3 (metric config's launch shape)
    (1100, [1100, 1024, 1025, 17]),           # RPT 4, two tiles
    (2300, [2300, 2049, 1023]),               # three tiles (phase A prefixes, omega carry)
])
def test_parity_ragged_tiles(tpl, oracle_lib, Lmax, lengths):
    B = len(lengths)
    ang = synth.angles_uniform(B, Lmax, 3, 77 + Lmax)
    grad = synth.grad_normal((B, 3 * Lmax, 3), 78 + Lmax)
    ln = torch.tensor(lengths, dtype=torch.int32)
    coords, gang = _run(tpl, ang, ln, grad)
    _check(oracle_lib, ang, ln, grad, coords, gang)
    # padding untouched (sentinel NaN survives)
    for b, L in enumerate(lengths):
        assert np.isnan(coords[b, 3 * L:]).all() and np.isnan(gang[b, L:]).all()


@pytest.mark.parametrize("Lmax,lengths", [
    (700, [700, 699, 641, 351, 350, 2, 1]),  # cluster split 128 x 3 x 2: odd halves, an empty second part
    (1000, [1000, 999, 769, 513, 3, 1]),     # 128 x 5 x 2
])
def test_cluster_split_forward_parity(tpl, oracle_lib, Lmax, lengths):
    """Forward with one 2-CTA cluster per chain (few chains of 641-1024 residues):
    the second CTA's part is placed with the first's aggregate received through
    distributed shared memory; at Lmax = 1000 the coordinate backward splits too
    (later part's (S, T) sent to the earlier one).  Parity, untouched padding,
    bitwise repeatability."""
    B = len(lengths)
    ang = synth.angles_uniform(B, Lmax, 3, 4242 + Lmax)
    grad = synth.grad_normal((B, 3 * Lmax, 3), 4243 + Lmax)
    ln = torch.tensor(lengths, dtype=torch.int32)
    coords, gang = _run(tpl, ang, ln, grad)
    _check(oracle_lib, ang, ln, grad, coords, gang)
    for b, L in enumerate(lengths):
        assert np.isnan(coords[b, 3 * L:]).all()
    again, _ = _run(tpl, ang, ln, grad)
    np.testing.assert_array_equal(coords, again)
    # coordinate backward (cluster-split for Lmax in (768, 1536] and few chains)
    cx, gx = _run(tpl, ang, ln, grad, xyz=True)
    _check(oracle_lib, ang, ln, grad, cx, gx)
    for b, L in enumerate(lengths):
        assert np.isnan(gx[b, L:]).all()
    _, gx2 = _run(tpl, ang, ln, grad, xyz=True)
    np.testing.assert_array_equal(gx, gx2)


@pytest.mark.parametrize("Lmax,lengths", [
    (16, [16, 1, 2, 3, 4, 7]),
    (300, [300, 1, 255, 256, 257, 299]),
    (700, [700, 650, 512, 3]),
    (2300, [2300, 2049, 1793, 1792, 1791, 17]),  # several tiles: (S, T) carry, reference shift, omega
])
def test_from_coords_parity(tpl, oracle_lib, Lmax, lengths):
    """tpl_backbone_backward_from_coords (gradient from the forward's coordinates) vs the oracle."""
    B = len(lengths)
    ang = synth.angles_uniform(B, Lmax, 3, 277 + Lmax)
    grad = synth.grad_normal((B, 3 * Lmax, 3), 278 + Lmax)
    ln = torch.tensor(lengths, dtype=torch.int32)
    coords, gang = _run(tpl, ang, ln, grad, xyz=True)
    c, g = _check(oracle_lib, ang, ln, grad, coords, gang)
    print(f"from_coords Lmax={Lmax}: max coord err {c:.3e} A, grad rel err {g:.3e}")
    for b, L in enumerate(lengths):
        assert np.isnan(gang[b, L:]).all()


def test_from_coords_metric_and_regular(tpl, oracle_lib):
    ang, lengths, grad = synth.backbone_inputs("metric")
    coords, gang = _run(tpl, ang, lengths, grad, xyz=True)
    sample = sorted(np.random.default_rng(4).choice(256, 16, replace=False).tolist())
    _check(oracle_lib, ang, lengths, grad, coords, gang, chains=sample)
    for kind in ("helix", "strand", "extended"):  # large |r| (extended: ~3000 A): report the gradient error
        ang = synth.regular_angles(2, 700, kind)
        ln = torch.full((2,), 700, dtype=torch.int32)
        grad = synth.grad_normal((2, 2100, 3), 3)
        _, gang = _run(tpl, ang, ln, grad, xyz=True)
        G = oracle_lib.backbone_backward(synth.numpy64(ang), ln.numpy(), synth.numpy64(grad))
        rel = np.abs(gang - G).max() / np.abs(G).max()
        print(f"from_coords {kind}: grad rel err {rel:.3e}")
        assert rel < 1e-2


def test_long_single_chain_across_ctas(tpl, oracle_lib):
    """one long chain split over many CTAs (decoupled tile carries):
    parity on the whole forward and on the backward of the full chain."""
    L = 6000
    ang = synth.angles_uniform(1, L, 3, 9001)
    grad = synth.grad_normal((1, 3 * L, 3), 9002)
    ln = torch.tensor([L], dtype=torch.int32)
    for xyz in (False, True):
        coords, gang = _run(tpl, ang, ln, grad, xyz=xyz)
        X = oracle_lib.backbone_forward(synth.numpy64(ang), ln.numpy())
        err = np.abs(coords - X).max()
        print(f"L={L} single chain: max coord err {err:.3e} A")
        assert err < 5e-3  # Q21: beyond L = 1000 the 1e-3 A gate is a target, gated at 5e-3
        G = oracle_lib.backbone_backward(synth.numpy64(ang), ln.numpy(), synth.numpy64(grad))
        rel = np.abs(gang - G).max() / np.abs(G).max()
        print(f"L={L} single chain ({'coords' if xyz else 'angles'} backward): grad rel err {rel:.3e}")
        assert rel <= GRAD_TOL


def test_decoupled_kernels_deterministic(tpl):
    """Tiles of a chain on different CTAs combine in a fixed order: bitwise repeatable."""
    ang, lengths, grad = synth.backbone_inputs(4, B=64)
    outs = [_run(tpl, ang, lengths, grad, xyz=True) for _ in range(3)]
    for c, g in outs[1:]:  # pads hold the NaN sentinel
        assert np.array_equal(c, outs[0][0], equal_nan=True) and np.array_equal(g, outs[0][1], equal_nan=True)


def test_config2_full_parity(tpl, oracle_lib):
    ang, lengths, grad = synth.backbone_inputs(2)
    coords, gang = _run(tpl, ang, lengths, grad)
    c, g = _check(oracle_lib, ang, lengths, grad, coords, gang)
    print(f"config2 64x700: max coord err {c:.3e} A, max grad rel err {g:.3e}")


def test_metric_config_sampled_parity(tpl, oracle_lib):
    """BASELINE metric workload (256 x 700) in the launch configuration bench.py times:
    coordinates of every chain, gradients of a seeded sample of 16 chains."""
    ang, lengths, grad = synth.backbone_inputs("metric")
    coords, gang = _run(tpl, ang, lengths, grad)
    a64, ln = synth.numpy64(ang), lengths.numpy()
    X = oracle_lib.backbone_forward(a64, ln)
    assert np.abs(coords - X).max() <= COORD_TOL
    sample = sorted(np.random.default_rng(0).choice(256, 16, replace=False).tolist())
    _check(oracle_lib, ang, lengths, grad, coords, gang, chains=sample)


def test_config4_ragged_sampled(tpl, oracle_lib):
    """Config 4 shape (ragged U[50,2000]) on a 512-chain slice; parity on 24 sampled
    chains including the longest."""
    ang, lengths, grad = synth.backbone_inputs(4, B=512)
    coords, gang = _run(tpl, ang, lengths, grad)
    ln = lengths.numpy()
    sample = set(np.random.default_rng(1).choice(512, 23, replace=False).tolist()) | {int(np.argmax(ln))}
    _check(oracle_lib, ang, lengths, grad, coords, gang, chains=sorted(sample))


def test_determinism(tpl):
    ang, lengths, grad = synth.backbone_inputs(2, B=16)
    outs = [_run(tpl, ang, lengths, grad) for _ in range(3)]
    for c, g in outs[1:]:
        assert np.array_equal(c, outs[0][0]) and np.array_equal(g, outs[0][1])


def test_device_input_error_flag(tpl):
    from paper_1812_01108_b200 import TplError, _abi

    ang = synth.angles_uniform(3, 10, 3, 5).cuda()
    ln = torch.tensor([10, 11, 0], dtype=torch.int32, device="cuda")
    coords = torch.zeros(3, 30, 3, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(0, 3, 10), dtype=torch.uint8, device="cuda")
    _abi.tpl_backbone_forward(ang, ln, coords, ws)
    with pytest.raises(TplError) as e:
        _abi.tpl_sync_status(ws)
    assert e.value.status == 6
    _abi.tpl_sync_status(ws)  # cleared
    assert coords[0].abs().sum() > 0  # the valid chain was processed


def test_autograd_layer(tpl, oracle_lib):
    ang, lengths, grad = synth.backbone_inputs(2, B=4)
    a = ang.cuda().requires_grad_(True)
    coords = tpl.backbone(a, lengths.cuda())
    (coords * grad.cuda()).sum().backward()
    G = oracle_lib.backbone_backward(synth.numpy64(ang), lengths.numpy(), synth.numpy64(grad))
    g = a.grad.cpu().numpy()
    for b in range(4):
        assert np.abs(g[b] - G[b]).max() / np.abs(G[b]).max() <= GRAD_TOL


def test_regular_structures_report(tpl, oracle_lib):
    """SURVEY f2 context: helix/strand/extended chains, reported (gate only on random
    input).  Extended chains reach |r| ~ 3000 Å where the fp32 ulp alone is 2.4e-4."""
    for kind in ("helix", "strand", "extended"):
        ang = synth.regular_angles(2, 700, kind)
        ln = torch.full((2,), 700, dtype=torch.int32)
        grad = synth.grad_normal((2, 2100, 3), 3)
        coords, gang = _run(tpl, ang, ln, grad)
        X = oracle_lib.backbone_forward(synth.numpy64(ang), ln.numpy())
        err = np.abs(coords - X).max()
        print(f"{kind}: max coord err {err:.3e} A at L=700")
        assert err < 0.1


@pytest.mark.parametrize("n_seg", [2, 3])
def test_segments_across_ranks_match_oracle(tpl, oracle_lib, n_seg):
    """SURVEY f4 across GPUs, by construction on one device: the per-rank segment
    kernels with the exchange done in-process (stacked in rank order, as the
    all-gather does) reproduce the whole chain's coordinates and gradients."""
    from paper_1812_01108_b200 import _abi
    from paper_1812_01108_b200 import dist as tdist

    B, L = 3, 1500
    ang = synth.angles_uniform(B, L, 3, 9101 + n_seg)
    grad = synth.grad_normal((B, 3 * L, 3), 9102 + n_seg)
    bounds = tdist.segment_bounds(L, n_seg)
    parts = []
    for (j0, j1) in bounds:
        n = j1 - j0
        a = ang[:, j0:j1].contiguous().cuda()
        ln = torch.full((B,), n, dtype=torch.int32, device="cuda")
        om = ang[:, j0 - 1, 2].contiguous().cuda() if j0 > 0 else None
        ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, n), dtype=torch.uint8, device="cuda")
        c = torch.empty(B, 3 * n, 3, device="cuda")
        agg = torch.empty(B, 12, device="cuda")
        _abi.tpl_backbone_segment_forward(a, ln, om, c, agg, ws)
        parts.append(dict(a=a, ln=ln, ws=ws, c=c, agg=agg, g=grad[:, 3 * j0:3 * j1].contiguous().cuda()))
    aggs = torch.stack([p["agg"] for p in parts])  # the forward exchange
    for s, p in enumerate(parts):
        _abi.tpl_backbone_segment_place(p["c"], p["ln"], aggs, s, p["ws"])
        p["tot"] = torch.empty(B, 12, device="cuda")
        _abi.tpl_backbone_segment_totals(p["c"], p["ln"], p["g"], p["tot"], p["ws"])
    tots = torch.stack([p["tot"] for p in parts])  # the backward exchange
    for s, p in enumerate(parts):
        p["ga"] = torch.zeros(B, p["c"].shape[1] // 3, 3, device="cuda")
        _abi.tpl_backbone_segment_backward(p["c"], p["ln"], p["g"], tots, s, p["ga"], p["ws"])
        _abi.tpl_sync_status(p["ws"])
    coords = torch.cat([p["c"] for p in parts], 1).cpu().numpy()
    gang = torch.cat([p["ga"] for p in parts], 1).cpu().numpy()
    lengths = torch.full((B,), L, dtype=torch.int32)
    c, g = _check(oracle_lib, ang, lengths, grad, coords, gang)
    print(f"{n_seg} segments, L={L}: max coord err {c:.3e} A, grad rel err {g:.3e}")


def test_precise_mode(tpl, oracle_lib):
    """the fp64-internal forward stays within 1e-3 A where the fp32 path
    does not (regular chains spanning up to ~2600 A), and agrees on random chains."""
    from paper_1812_01108_b200 import _abi

    cases = [("random", synth.angles_uniform(3, 2300, 3, 9301), [2300, 1, 1000])]
    cases += [(k, synth.regular_angles(2, 2000, k), [2000, 1999]) for k in ("helix", "strand", "extended")]
    for name, ang, lengths in cases:
        B, Lmax, _ = ang.shape
        ln = torch.tensor(lengths, dtype=torch.int32)
        coords = torch.full((B, 3 * Lmax, 3), float("nan"), device="cuda")
        ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, Lmax), dtype=torch.uint8, device="cuda")
        _abi.tpl_backbone_forward_precise(ang.cuda(), ln.cuda(), coords, ws)
        _abi.tpl_sync_status(ws)
        c = coords.cpu().numpy()
        X = oracle_lib.backbone_forward(synth.numpy64(ang), ln.numpy())
        for b, L in enumerate(lengths):
            err = np.abs(c[b, :3 * L] - X[b, :3 * L]).max()
            # fp32 rounding of the output: half an ulp of |r| (up to ~2^11 A here)
            bound = max(1e-5, 2.0 ** -23 * np.abs(X[b, :3 * L]).max())
            print(f"precise {name} L={L}: max err {err:.3e} A (fp32 output ulp/2 {bound:.1e})")
            assert err <= 1e-3 and err <= 4 * bound
            assert np.isnan(c[b, 3 * L:]).all()


def test_decoupled_more_items_than_resident_ctas(tpl, oracle_lib):
    """f4 within a GPU with more (chain, tile) items than co-resident CTAs: 296 ragged
    chains up to 5000 residues (~1300 items) -- every CTA walks several items, later
    tiles wait on earlier ones held by other CTAs.  Parity on sampled chains."""
    B, Lmax = 296, 5000
    ang = synth.angles_uniform(B, Lmax, 3, 9401)
    grad = synth.grad_normal((B, 3 * Lmax, 3), 9402)
    ln = synth.lengths_uniform(B, 1025, Lmax, 9403)
    coords, gang = _run(tpl, ang, ln, grad, xyz=True)
    lnn = ln.numpy()
    sample = sorted({int(np.argmax(lnn)), int(np.argmin(lnn)), 7, 150})
    _check(oracle_lib, ang, ln, grad, coords, gang, chains=sample)


def test_coordinate_gate_L1000_many_chains(tpl, oracle_lib):
    """The 1e-3 A gate at its longest stated length (L = 1000, two forward tiles),
    over every chain of a 128-chain batch."""
    from paper_1812_01108_b200 import _abi

    B, L = 128, 1000
    ang = synth.angles_uniform(B, L, 3, 9901)
    ln = torch.full((B,), L, dtype=torch.int32)
    coords = torch.empty(B, 3 * L, 3, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, L), dtype=torch.uint8, device="cuda")
    _abi.tpl_backbone_forward(ang.cuda(), ln.cuda(), coords, ws)
    _abi.tpl_sync_status(ws)
    X = oracle_lib.backbone_forward(synth.numpy64(ang), ln.numpy())
    worst = float(np.abs(coords.cpu().numpy() - X).max())
    print(f"backbone {B} x {L}: worst coord err {worst:.3e} A")
    assert worst <= 1e-3
