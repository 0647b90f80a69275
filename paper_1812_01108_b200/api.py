"""User-facing API: differentiable backbone / full-atom layers (§2, §3)
and the LRMSD loss (§4).

    coords = backbone(angles, lengths)                  # [B, 3*Lmax, 3]
    tables = Tables(synth.load_residue_table())         # 20 residue types
    coords = fullatom(angles, restype, lengths, tables) # [B, atom_stride, 3]
    loss = lrmsd(coords, target, 3 * lengths)           # [B] (n_atoms: the chains' true atom counts)
    coords, n_atoms = fullatom(angles, restype, lengths, tables, return_atoms=True)
    loss = lrmsd(coords, target, n_atoms)               # full atom: padded width != atom count
    loss, coords = backbone_lrmsd(angles, target)       # fused forward + LRMSD (f1)

All are ``torch.autograd.Function``s running on the current CUDA stream of the
inputs' device.  Output entries past a chain's length (padding) are 0.  A chain
with a bad length or residue type is skipped on the device and flagged in the
workspace error word: ``default_workspace().check()`` raises on it, and with
``TPL_CHECK=1`` (or ``api.CHECK_INPUTS = True``) every call checks (a sync).  The
layers save their output coordinates and back-propagate from them (the rotation
axes are bond vectors); a table without origin atoms falls back to recomputing
from the angles.  Argument marshalling only: every step runs in libtpl.so.
"""
import ctypes
import os

import torch

from . import _abi
from ._abi import MODEL_BACKBONE, MODEL_FULLATOM


class Workspace:
    """Zero-initialised device workspace (tpl_workspace_bytes), grown on demand.
    One per (device, stream) in use; the error word is checked by ``check()``."""

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.buf = torch.zeros(256, dtype=torch.uint8, device=self.device)

    def get(self, model, B, Lmax):
        need = _abi.tpl_workspace_bytes(model, B, Lmax)
        if self.buf.numel() < need:
            self.buf = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self.buf

    def check(self, stream=None):
        """Synchronise and raise TplError if a kernel flagged a bad length/restype."""
        _abi.tpl_sync_status(self.buf, stream)


_workspaces = {}

CHECK_INPUTS = os.environ.get("TPL_CHECK", "0") == "1"  # debug: sync + raise on flagged inputs after each call


def _maybe_check(device):
    if CHECK_INPUTS:
        default_workspace(device).check()


def default_workspace(device=None):
    d = torch.cuda.current_device() if device is None else torch.device(device).index
    key = (d, torch.cuda.current_stream(d).cuda_stream)
    ws = _workspaces.get(key)
    if ws is None:
        ws = _workspaces[key] = Workspace(torch.device("cuda", d))
    return ws


class Tables:
    """Device copy of a residue-type table (see synth/residue_table.json for
    the format: per type, side-chain groups and atoms with standard
    coordinates).  Immutable; freed with the object."""

    def __init__(self, table):
        types = table["types"] if isinstance(table, dict) else table
        descs = (_abi.ResidueDesc * len(types))()
        for t, ty in enumerate(types):
            d = descs[t]
            d.n_groups = len(ty["groups"])
            d.n_atoms = len(ty["atoms"])
            if d.n_groups > _abi.MAX_GROUPS or d.n_atoms > _abi.MAX_ATOMS:
                raise ValueError(f"type {t}: too many groups/atoms")
            for g, gr in enumerate(ty["groups"]):
                d.group_parent[g] = int(gr["parent"])
                d.group_slot[g] = int(gr["slot"])
                d.group_alpha[g] = float(gr["alpha"])
                d.group_theta[g] = float(gr["theta"])
                d.group_d[g] = float(gr["d"])
                d.group_pre_rx[g] = float(gr["pre_rx"])
            for k, at in enumerate(ty["atoms"]):
                d.atom_owner[k] = int(at["owner"])
                for c in range(3):
                    d.atom_r[k][c] = float(at["r"][c])
        self._descs = descs
        self.names = [ty.get("name", str(i)) for i, ty in enumerate(types)]
        self.atoms_per_type = torch.tensor([len(ty["atoms"]) for ty in types], dtype=torch.int64)
        self.handle = _abi.tpl_tables_create(descs)
        self.backward_from_coords = _abi.tpl_tables_backward_from_coords_ok(self.handle)

    @property
    def n_types(self):
        return _abi.tpl_tables_n_types(self.handle)

    def atoms(self, restype, lengths):
        """(atoms_per_chain [B] int32, atom_stride) -- host bookkeeping."""
        return _abi.tpl_fullatom_atoms(self.handle, restype.cpu(), lengths.cpu())

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _abi.tpl_tables_destroy(h)
            except Exception:
                pass
            self.handle = None


def _lengths_for(angles, lengths):
    if lengths is None:
        return torch.full((angles.shape[0],), angles.shape[1], dtype=torch.int32, device=angles.device)
    if not lengths.is_cuda and lengths.numel() and (int(lengths.min()) < 1 or int(lengths.max()) > angles.shape[1]):
        raise ValueError(f"lengths must lie in [1, {angles.shape[1]}] (host check)")
    return lengths.to(device=angles.device, dtype=torch.int32).contiguous()


class BackboneFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, angles, lengths):
        angles = angles.contiguous()
        B, Lmax, _ = angles.shape
        coords = torch.zeros((B, 3 * Lmax, 3), dtype=torch.float32, device=angles.device)  # pads stay 0
        with torch.cuda.device(angles.device):
            ws = default_workspace(angles.device).get(MODEL_BACKBONE, B, Lmax)
            _abi.tpl_backbone_forward(angles, lengths, coords, ws)
            _maybe_check(angles.device)
        # the backward needs only the output (rotation axes are bond vectors)
        ctx.save_for_backward(coords, lengths)
        ctx.mark_non_differentiable(lengths)
        return coords

    @staticmethod
    def backward(ctx, grad_coords):
        coords, lengths = ctx.saved_tensors
        B, Lmax = coords.shape[0], coords.shape[1] // 3
        grad_angles = torch.zeros((B, Lmax, 3), dtype=torch.float32, device=coords.device)  # pads stay 0
        with torch.cuda.device(coords.device):
            ws = default_workspace(coords.device).get(MODEL_BACKBONE, B, Lmax)
            _abi.tpl_backbone_backward_from_coords(coords, lengths, grad_coords.contiguous(), grad_angles, ws)
            _maybe_check(coords.device)
        return grad_angles, None


class FullAtomFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, angles, restype, lengths, tables, atom_stride):
        angles = angles.contiguous()
        B, Lmax, _ = angles.shape
        coords = torch.zeros((B, atom_stride, 3), dtype=torch.float32, device=angles.device)
        with torch.cuda.device(angles.device):
            ws = default_workspace(angles.device).get(MODEL_FULLATOM, B, Lmax)
            _abi.tpl_fullatom_forward(tables.handle, angles, restype, lengths, coords, ws)
            _maybe_check(angles.device)
        # tables with an atom at every frame origin back-propagate from the output
        ctx.from_coords = tables.backward_from_coords
        ctx.save_for_backward(coords if ctx.from_coords else angles, restype, lengths)
        ctx.tables = tables
        ctx.Lmax = Lmax
        return coords

    @staticmethod
    def backward(ctx, grad_coords):
        saved, restype, lengths = ctx.saved_tensors
        B, Lmax = restype.shape[0], ctx.Lmax
        grad_angles = torch.zeros((B, Lmax, _abi.FA_SLOTS), dtype=torch.float32, device=saved.device)
        with torch.cuda.device(saved.device):
            ws = default_workspace(saved.device).get(MODEL_FULLATOM, B, Lmax)
            if ctx.from_coords:
                _abi.tpl_fullatom_backward_from_coords(ctx.tables.handle, saved, restype, lengths,
                                                       grad_coords.contiguous(), grad_angles, ws)
            else:
                _abi.tpl_fullatom_backward(ctx.tables.handle, saved, restype, lengths, grad_coords.contiguous(),
                                           grad_angles, ws)
            _maybe_check(saved.device)
        return grad_angles, None, None, None, None


def backbone(angles, lengths=None):
    """angles [B, Lmax, 3] fp32 CUDA (phi, psi, omega) -> coords [B, 3*Lmax, 3] (N, CA, C)."""
    return BackboneFunction.apply(angles, _lengths_for(angles, lengths))


def fullatom(angles, restype, lengths, tables, atom_stride=None, return_atoms=False):
    """angles [B, Lmax, 8], restype [B, Lmax] uint8 -> packed coords [B, atom_stride, 3].
    atom_stride defaults to tables.atoms(...) (a host round trip); pass it to avoid the sync.
    return_atoms=True also returns the atoms of each chain (int32 [B] on the device) -- the
    n_atoms an LRMSD of the packed output needs (the width is padded to atom_stride)."""
    lengths = _lengths_for(angles, lengths)
    restype = restype.to(device=angles.device, dtype=torch.uint8).contiguous()
    apc = None
    if atom_stride is None or return_atoms:
        apc, stride = tables.atoms(restype, lengths)
        atom_stride = stride if atom_stride is None else atom_stride
    coords = FullAtomFunction.apply(angles, restype, lengths, tables, int(atom_stride))
    return (coords, apc.to(angles.device)) if return_atoms else coords


class BackboneLRMSDFunction(torch.autograd.Function):
    """f1: angles -> (LRMSD to target [B], coords).  Chains that fit one tile
    (Lmax <= tpl_backbone_lrmsd_fused_max_L()) take the one-pass kernel: the forward
    already computes dLRMSD/dangles (no coordinate round-trip), the backward only
    scales it by dL/dLRMSD.  Longer chains: the fused forward + coordinate backward."""

    @staticmethod
    def forward(ctx, angles, target, lengths, with_coords):
        angles, target = angles.contiguous(), target.contiguous()
        B, Lmax, _ = angles.shape
        dev = angles.device
        coords = torch.zeros((B, 3 * Lmax, 3), dtype=torch.float32, device=dev) if with_coords else None
        out = torch.zeros(B, dtype=torch.float32, device=dev)
        state = torch.zeros((B, 16), dtype=torch.float32, device=dev)
        ctx.one_pass = Lmax <= _abi.tpl_backbone_lrmsd_fused_max_L()
        with torch.cuda.device(dev):
            ws = default_workspace(dev).get(MODEL_BACKBONE, B, Lmax)
            if ctx.one_pass:
                dlda = torch.zeros((B, Lmax, 3), dtype=torch.float32, device=dev)
                _abi.tpl_backbone_lrmsd_fused(angles, lengths, target, coords, out, state, dlda, ws)
                ctx.save_for_backward(dlda)
            else:
                if coords is None:
                    coords = torch.zeros((B, 3 * Lmax, 3), dtype=torch.float32, device=dev)
                _abi.tpl_backbone_lrmsd_forward(angles, lengths, target, coords, out, state, ws)
                ctx.save_for_backward(coords, target, lengths, state)
            _maybe_check(dev)
        if coords is not None:
            ctx.mark_non_differentiable(coords)
        return out, coords

    @staticmethod
    def backward(ctx, grad_out, _grad_coords):
        if ctx.one_pass:
            (dlda,) = ctx.saved_tensors
            grad_angles = torch.empty_like(dlda)
            with torch.cuda.device(dlda.device):
                _abi.tpl_chain_scale(dlda, grad_out.contiguous(), grad_angles)
            return grad_angles, None, None, None
        coords, target, lengths, state = ctx.saved_tensors
        B, Lmax = coords.shape[0], coords.shape[1] // 3
        grad_angles = torch.zeros((B, Lmax, 3), dtype=torch.float32, device=coords.device)
        with torch.cuda.device(coords.device):
            ws = default_workspace(coords.device).get(MODEL_BACKBONE, B, Lmax)
            _abi.tpl_backbone_lrmsd_backward(coords, lengths, target, state, grad_out.contiguous(), grad_angles, ws)
            _maybe_check(coords.device)
        return grad_angles, None, None, None


def backbone_lrmsd(angles, target, lengths=None, with_coords=True):
    """angles [B, Lmax, 3], target [B, 3*Lmax, 3] -> (LRMSD over each chain's 3L atoms [B],
    coords [B, 3*Lmax, 3] or None when with_coords=False (the coordinates are then never
    written to HBM); coords are not differentiable: the gradient flows through the LRMSD)."""
    return BackboneLRMSDFunction.apply(angles, target.to(angles.device), _lengths_for(angles, lengths),
                                       bool(with_coords))


class LRMSDFunction(torch.autograd.Function):
    """LRMSD (PAPER §4) per chain between x (differentiated) and the reference y."""

    @staticmethod
    def forward(ctx, x, y, n_atoms):
        x, y = x.contiguous(), y.contiguous()
        B = x.shape[0]
        out = torch.zeros(B, dtype=torch.float32, device=x.device)
        state = torch.zeros(B, 16, dtype=torch.float32, device=x.device)
        with torch.cuda.device(x.device):
            ws = default_workspace(x.device).buf
            _abi.tpl_lrmsd_forward(x, y, n_atoms, out, state, ws)
            _maybe_check(x.device)
        ctx.save_for_backward(x, y, n_atoms, state)
        ctx.mark_non_differentiable(n_atoms)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        x, y, n_atoms, state = ctx.saved_tensors
        grad_x = torch.zeros_like(x)
        with torch.cuda.device(x.device):
            ws = default_workspace(x.device).buf
            _abi.tpl_lrmsd_backward(x, y, n_atoms, state, grad_out.contiguous(), grad_x, ws)
            _maybe_check(x.device)
        return grad_x, None, None


def lrmsd(x, y, n_atoms=None):
    """x, y [B, stride, 3] fp32 CUDA -> LRMSD [B] over the first n_atoms[b] atoms; differentiable in x.
    n_atoms defaults to the full width x.shape[1] -- right for unpadded backbone coordinates only:
    full-atom output is padded to atom_stride (pass fullatom(..., return_atoms=True)'s counts) and
    ragged backbone batches need 3 * lengths, or the pads enter the centroid and the rotation."""
    if n_atoms is None:
        n_atoms = torch.full((x.shape[0],), x.shape[1], dtype=torch.int32, device=x.device)
    return LRMSDFunction.apply(x, y.to(x.device), n_atoms.to(device=x.device, dtype=torch.int32).contiguous())
