"""GPU parity of the full-atom kernels (through the C ABI) against the fp64 oracle."""
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


def _run(tpl, tables, ang, rt, lengths, grad_fn, sentinel=float("nan"), xyz=False):
    from paper_1812_01108_b200 import _abi

    B, Lmax, _ = ang.shape
    apc, stride = tables.atoms(rt, lengths)
    a, r, ln = ang.cuda(), rt.cuda(), lengths.cuda()
    coords = torch.full((B, stride, 3), sentinel, device="cuda")
    gang = torch.full((B, Lmax, 8), sentinel, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(1, B, Lmax), dtype=torch.uint8, device="cuda")
    _abi.tpl_fullatom_forward(tables.handle, a, r, ln, coords, ws)
    grad = grad_fn(B, stride)
    if xyz:  # backward from the forward's coordinates
        _abi.tpl_fullatom_backward_from_coords(tables.handle, coords, r, ln, grad.cuda(), gang, ws)
    else:
        _abi.tpl_fullatom_backward(tables.handle, a, r, ln, grad.cuda(), gang, ws)
    _abi.tpl_sync_status(ws)
    return coords.cpu().numpy(), gang.cpu().numpy(), grad, apc.numpy()


def _check(oracle_lib, table, ang, rt, lengths, grad, coords, gang, apc, chains=None):
    B = ang.shape[0]
    idx = np.array(list(range(B) if chains is None else chains))
    a64, ln = synth.numpy64(ang), lengths.numpy()
    rtn = rt.numpy()
    stride = coords.shape[1]
    X, nat = oracle_lib.fullatom_forward(table, a64[idx], rtn[idx], ln[idx], stride)
    G = oracle_lib.fullatom_backward(table, a64[idx], rtn[idx], ln[idx], synth.numpy64(grad)[idx])
    wc, wg = 0.0, 0.0
    for n, b in enumerate(idx):
        L, na = int(ln[b]), int(nat[n])
        assert na == apc[b]
        dc = np.abs(coords[b, :na] - X[n, :na]).max()
        ref = G[n, :L]
        dg = np.abs(gang[b, :L] - ref).max() / max(np.abs(ref).max(), 1e-30)
        wc, wg = max(wc, dc), max(wg, dg)
        assert dc <= COORD_TOL, f"chain {b}: coord err {dc:.3e}"
        assert dg <= GRAD_TOL, f"chain {b}: grad rel err {dg:.3e}"
        assert np.isnan(coords[b, na:]).all()  # padding untouched
        assert np.isnan(gang[b, L:]).all()
        # structural zeros: omega_{L-1}, unused chi slots
        assert gang[b, L - 1, 2] == 0.0
        for j in range(L):
            ty = table["types"][rtn[b, j]]
            used = {0, 1, 2} | {g["slot"] for g in ty["groups"] if g["slot"] >= 0}
            for s in set(range(8)) - used:
                assert gang[b, j, s] == 0.0
    return wc, wg


XYZ = pytest.mark.parametrize("xyz", [False, True], ids=["from_angles", "from_coords"])


@XYZ
def test_config3_all_types(tpl, oracle_lib, table, xyz):
    tables = tpl.Tables(table)
    ang, rt, lengths = synth.fullatom_inputs(3)
    coords, gang, grad, apc = _run(tpl, tables, ang, rt, lengths, lambda B, S: synth.fullatom_grad(B, S, 3), xyz=xyz)
    c, g = _check(oracle_lib, table, ang, rt, lengths, grad, coords, gang, apc)
    print(f"config3 64x300 ({'from coords' if xyz else 'from angles'}): max coord err {c:.3e} A, grad rel err {g:.3e}")


@pytest.mark.parametrize("Lmax,lengths", [
    (5, [5, 1, 2]),
    (256, [256, 255, 1]),
    (300, [300, 257, 129]),       # RPT 2, one tile
    (700, [700, 513, 512, 40]),   # two tiles (phase A: prefix + atom offset carries)
    (1100, [1100, 897, 385, 384, 383]),  # several tiles of the coordinate backward
])
@XYZ
def test_parity_ragged(tpl, oracle_lib, table, Lmax, lengths, xyz):
    tables = tpl.Tables(table)
    B = len(lengths)
    ang = synth.angles_uniform(B, Lmax, 8, 11 + Lmax)
    rt = synth.restype_uniform(B, Lmax, 20, 12 + Lmax)
    ln = torch.tensor(lengths, dtype=torch.int32)
    coords, gang, grad, apc = _run(tpl, tables, ang, rt, ln, lambda B_, S: synth.grad_normal((B_, S, 3), 13),
                                   xyz=xyz)
    _check(oracle_lib, table, ang, rt, ln, grad, coords, gang, apc)


@XYZ
def test_chi5_table(tpl, oracle_lib, table_chi5, xyz):
    tables = tpl.Tables(table_chi5)
    B, L = 4, 64
    ang = synth.angles_uniform(B, L, 8, 21)
    rt = torch.full((B, L), 1, dtype=torch.uint8)  # ARG: chi1..chi5 variable
    rt[1] = synth.restype_uniform(1, L, 20, 22)[0]
    ln = torch.full((B,), L, dtype=torch.int32)
    coords, gang, grad, apc = _run(tpl, tables, ang, rt, ln, lambda B_, S: synth.grad_normal((B_, S, 3), 23),
                                   xyz=xyz)
    _check(oracle_lib, table_chi5, ang, rt, ln, grad, coords, gang, apc)
    assert np.abs(gang[0, :, 7]).max() > 0  # chi5 gradient is live


@XYZ
def test_config5_shape_sampled(tpl, oracle_lib, table, xyz):
    """Config 5 per-GPU shape (8192/8 = 1024 chains x L=500); parity on 8 sampled chains."""
    tables = tpl.Tables(table)
    ang, rt, lengths = synth.fullatom_inputs(5, B=1024)
    coords, gang, grad, apc = _run(tpl, tables, ang, rt, lengths, lambda B, S: synth.fullatom_grad(B, S, 5), xyz=xyz)
    sample = sorted(np.random.default_rng(2).choice(1024, 8, replace=False).tolist())
    _check(oracle_lib, table, ang, rt, lengths, grad, coords, gang, apc, chains=sample)


def test_large_batch_ragged_two_residues_per_thread(tpl, oracle_lib, table):
    """The large-batch forward shape (64 threads x 2 residues per thread, chosen for >= 1024
    chains longer than 384 residues): ragged lengths so that runs end mid-pair, tiles end
    mid-run and single-residue chains occur; parity on the edge chains and a sample."""
    tables = tpl.Tables(table)
    B, L = 1024, 520
    ang, rt, _ = synth.fullatom_inputs(5, B=B, L=L)
    lengths = synth.lengths_uniform(B, 1, L, 7301)
    edge = {0: L, 1: 1, 2: 2, 3: 127, 4: 128, 5: 129, 6: 255, 7: 257, 8: 385}
    for b, n in edge.items():
        lengths[b] = n
    coords, gang, grad, apc = _run(tpl, tables, ang, rt, lengths, lambda B, S: synth.fullatom_grad(B, S, 5))
    sample = sorted(set(edge) | set(np.random.default_rng(5).choice(B, 8, replace=False).tolist()))
    _check(oracle_lib, table, ang, rt, lengths, grad, coords, gang, apc, chains=sample)
    for b in sample:  # atoms past each chain's count are never written
        assert np.isnan(coords[b, apc[b]:]).all()


def test_backbone_atoms_match_backbone_kernel(tpl, table):
    """Fig:ErrorEstimate methodology between the two GPU models."""
    tables = tpl.Tables(table)
    ang, rt, lengths = synth.fullatom_inputs(3, B=8)
    fa = tpl.fullatom(ang.cuda(), rt.cuda(), lengths.cuda(), tables)
    bb = tpl.backbone(ang[..., :3].contiguous().cuda(), lengths.cuda())
    n = torch.tensor([len(t["atoms"]) for t in table["types"]])
    for b in range(8):
        off = 0
        for j in range(300):
            t = int(rt[b, j])
            for k, slot in ((0, 0), (1, 1), (int(n[t]) - 2, 2)):
                d = (fa[b, off + k] - bb[b, 3 * j + slot]).abs().max().item()
                assert d < 2e-4
            off += int(n[t])


def test_restype_error_flag(tpl, table):
    from paper_1812_01108_b200 import TplError, _abi

    tables = tpl.Tables(table)
    ang = synth.angles_uniform(2, 8, 8, 1).cuda()
    rt = torch.zeros(2, 8, dtype=torch.uint8, device="cuda")
    rt[1, 3] = 30
    ln = torch.full((2,), 8, dtype=torch.int32, device="cuda")
    coords = torch.zeros(2, 64, 3, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(1, 2, 8), dtype=torch.uint8, device="cuda")
    _abi.tpl_fullatom_forward(tables.handle, ang, rt, ln, coords, ws)
    with pytest.raises(TplError) as e:
        _abi.tpl_sync_status(ws)
    assert e.value.status == 6


def test_autograd_layer(tpl, oracle_lib, table):
    tables = tpl.Tables(table)
    ang, rt, lengths = synth.fullatom_inputs(3, B=3)
    a = ang.cuda().requires_grad_(True)
    coords = tpl.fullatom(a, rt.cuda(), lengths.cuda(), tables)
    grad = synth.grad_normal(tuple(coords.shape), 9)
    (coords * grad.cuda()).sum().backward()
    G = oracle_lib.fullatom_backward(table, synth.numpy64(ang), rt.numpy(), lengths.numpy(), synth.numpy64(grad))
    g = a.grad.cpu().numpy()
    for b in range(3):
        assert np.abs(g[b] - G[b]).max() / np.abs(G[b]).max() <= GRAD_TOL


def test_from_coords_needs_origin_atoms(tpl, table):
    """A table whose chi group has no atom at its frame origin cannot back-propagate
    from coordinates: the call is refused before any launch (TPL_ERR_TABLE)."""
    import copy

    from paper_1812_01108_b200 import TplError, _abi

    assert tpl.Tables(table).backward_from_coords
    bad = copy.deepcopy(table)
    ser = next(t for t in bad["types"] if t["name"] == "SER")
    cb = next(a for a in ser["atoms"] if a["name"] == "CB")
    cb["r"] = [0.1, 0.0, 0.0]  # CB no longer at the chi1 frame origin
    tables = tpl.Tables(bad)
    assert not tables.backward_from_coords
    B, L = 1, 4
    ws = torch.zeros(_abi.tpl_workspace_bytes(1, B, L), dtype=torch.uint8, device="cuda")
    rt = torch.zeros(B, L, dtype=torch.uint8, device="cuda")
    ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
    x = torch.zeros(B, 64, 3, device="cuda")
    with pytest.raises(TplError) as e:
        _abi.tpl_fullatom_backward_from_coords(tables.handle, x, rt, ln, x.clone(), torch.zeros(B, L, 8, device="cuda"),
                                               ws)
    assert e.value.status == 4
    # the autograd layer falls back to the from-angles backward for such tables
    a = synth.angles_uniform(B, L, 8, 3).cuda().requires_grad_(True)
    tpl.fullatom(a, rt, ln, tables).sum().backward()
    assert torch.isfinite(a.grad).all()


def test_atom_stride_too_small_is_flagged(tpl, table):
    """A chain with more atoms than atom_stride is flagged on the device
    (TPL_ERR_DEVICE_INPUT) instead of writing past its row; the other chains run."""
    from paper_1812_01108_b200 import TplError, _abi

    tables = tpl.Tables(table)
    B, L = 3, 40
    ang = synth.angles_uniform(B, L, 8, 61).cuda()
    rt = synth.restype_uniform(B, L, 20, 62)
    rt[1] = 17  # TRP: the largest type, so chain 1 needs the most atoms
    apc, _ = tables.atoms(rt, torch.full((B,), L, dtype=torch.int32))
    stride = int(apc[0].item()) if int(apc[0]) >= int(apc[2]) else int(apc[2])
    stride = max(stride, int(sorted(apc.tolist())[1]))  # fits chains 0 and 2, not chain 1
    assert int(apc[1]) > stride
    guard = torch.full((B + 1, stride, 3), float("nan"), device="cuda")
    coords = guard[:B]
    ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(1, B, L), dtype=torch.uint8, device="cuda")
    _abi.tpl_fullatom_forward(tables.handle, ang, rt.cuda(), ln, coords, ws)
    with pytest.raises(TplError) as e:
        _abi.tpl_sync_status(ws)
    assert e.value.status == 6 and "atom_stride" in str(e.value)
    assert torch.isnan(guard[B]).all()  # nothing written past the last row
    assert torch.isfinite(coords[0, : int(apc[0])]).all()
    gang = torch.zeros(B, L, 8, device="cuda")
    _abi.tpl_fullatom_backward_from_coords(tables.handle, coords, rt.cuda(), ln, torch.zeros_like(coords), gang, ws)
    with pytest.raises(TplError):
        _abi.tpl_sync_status(ws)


def test_coordinate_gate_many_chains_L700(tpl, oracle_lib, table):
    """The 1e-3 A gate over many chains at L = 700 (one 512-thread tile plus a
    tail): the wide scans need Newton-Schulz after each cross-warp combine
    (policy 3); with policy 1 the worst of 64 chains reached 1.03e-3 A."""
    tables = tpl.Tables(table)
    B, L = 48, 700
    ang = synth.angles_uniform(B, L, 8, 77)
    rt = synth.restype_uniform(B, L, 20, 78)
    ln = torch.full((B,), L, dtype=torch.int32)
    c = tpl.fullatom(ang.cuda(), rt.cuda(), ln.cuda(), tables).cpu().numpy()
    X, nat = oracle_lib.fullatom_forward(table, synth.numpy64(ang), rt.numpy(), ln.numpy(), c.shape[1])
    worst = max(float(np.abs(c[b, :nat[b]] - X[b, :nat[b]]).max()) for b in range(B))
    print(f"full atom {B} x {L}: worst coord err {worst:.3e} A")
    assert worst <= 1e-3
