"""ctypes binding of libtpl.so (include/tpl.h).  Argument marshalling only.

Every function named ``tpl_*`` here has the C entry point's name and argument
order; tensors stand in for pointers (device tensors for the fwd/bwd calls,
host tensors for the bookkeeping call).  All arithmetic of the method runs in
the CUDA kernels of libtpl.so; if the library is missing this module raises
on import -- there is no CPU fallback.
"""
import ctypes
import os

import torch  # loads libcudart.so.12 before libtpl.so resolves it

_HERE = os.path.dirname(os.path.abspath(__file__))
# TPL_LIB selects another build of the same ABI (e.g. build/libtpl_phases.so
# for latency studies); default: the in-tree product library.
LIB_PATH = os.environ.get("TPL_LIB") or os.path.join(_HERE, "libtpl.so")

TPL_OK = 0
STATUS = {0: "TPL_OK", 1: "TPL_ERR_NULL", 2: "TPL_ERR_SHAPE", 3: "TPL_ERR_ALIGN", 4: "TPL_ERR_TABLE",
          5: "TPL_ERR_CUDA", 6: "TPL_ERR_DEVICE_INPUT", 7: "TPL_ERR_WORKSPACE"}
MODEL_BACKBONE, MODEL_FULLATOM = 0, 1
MAX_GROUPS, MAX_ATOMS, MAX_TYPES = 8, 16, 32
BB_SLOTS, FA_SLOTS = 3, 8
OWNER_N, OWNER_CA, OWNER_C = -3, -2, -1

# Every symbol include/tpl.h declares (checked by tests/test_abi_cpu.py).
EXPORTS = [
    "tpl_last_error", "tpl_abi_version", "tpl_workspace_bytes", "tpl_sync_status", "tpl_backbone_atoms",
    "tpl_backbone_forward", "tpl_backbone_backward", "tpl_backbone_backward_from_coords", "tpl_tables_create", "tpl_tables_destroy",
    "tpl_tables_n_types", "tpl_fullatom_atoms", "tpl_fullatom_forward", "tpl_fullatom_backward",
    "tpl_fullatom_backward_from_coords", "tpl_tables_backward_from_coords_ok",
    "tpl_lrmsd_forward", "tpl_lrmsd_backward",
    "tpl_backbone_forward_precise", "tpl_backbone_lrmsd_forward", "tpl_backbone_lrmsd_backward", "tpl_backbone_segment_forward", "tpl_backbone_segment_place", "tpl_backbone_segment_totals",
    "tpl_backbone_segment_backward", "tpl_paper_backbone_saved_floats", "tpl_paper_backbone_forward", "tpl_paper_backbone_backward",
    "tpl_backbone_lrmsd_fused_max_L", "tpl_backbone_lrmsd_fused", "tpl_chain_scale",
]


class TplError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ResidueDesc(ctypes.Structure):
    """Mirror of ``tpl_residue_desc``."""

    _fields_ = [
        ("n_groups", ctypes.c_int32),
        ("n_atoms", ctypes.c_int32),
        ("group_parent", ctypes.c_int32 * MAX_GROUPS),
        ("group_slot", ctypes.c_int32 * MAX_GROUPS),
        ("group_alpha", ctypes.c_double * MAX_GROUPS),
        ("group_theta", ctypes.c_double * MAX_GROUPS),
        ("group_d", ctypes.c_double * MAX_GROUPS),
        ("group_pre_rx", ctypes.c_double * MAX_GROUPS),
        ("atom_owner", ctypes.c_int32 * MAX_ATOMS),
        ("atom_r", (ctypes.c_double * 3) * MAX_ATOMS),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, i64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_int64
    L.tpl_last_error.restype = ctypes.c_char_p
    L.tpl_last_error.argtypes = []
    L.tpl_abi_version.restype = ctypes.c_int
    L.tpl_workspace_bytes.restype = sz
    L.tpl_workspace_bytes.argtypes = [i32, i32, i32]
    L.tpl_sync_status.restype = ctypes.c_int
    L.tpl_sync_status.argtypes = [vp, vp]
    L.tpl_backbone_atoms.restype = i64
    L.tpl_backbone_atoms.argtypes = [i32]
    L.tpl_backbone_forward.restype = ctypes.c_int
    L.tpl_backbone_forward.argtypes = [vp, vp, i32, i32, vp, vp, sz, vp]
    L.tpl_backbone_backward.restype = ctypes.c_int
    L.tpl_backbone_backward.argtypes = [vp, vp, i32, i32, vp, vp, vp, sz, vp]
    L.tpl_backbone_backward_from_coords.restype = ctypes.c_int
    L.tpl_backbone_backward_from_coords.argtypes = [vp, vp, i32, i32, vp, vp, vp, sz, vp]
    L.tpl_tables_create.restype = ctypes.c_int
    L.tpl_tables_create.argtypes = [ctypes.POINTER(ResidueDesc), i32, ctypes.POINTER(vp)]
    L.tpl_tables_destroy.restype = None
    L.tpl_tables_destroy.argtypes = [vp]
    L.tpl_tables_n_types.restype = i32
    L.tpl_tables_n_types.argtypes = [vp]
    L.tpl_fullatom_atoms.restype = ctypes.c_int
    L.tpl_fullatom_atoms.argtypes = [vp, vp, vp, i32, i32, vp, ctypes.POINTER(i32)]
    L.tpl_fullatom_forward.restype = ctypes.c_int
    L.tpl_fullatom_forward.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, vp, sz, vp]
    L.tpl_fullatom_backward.restype = ctypes.c_int
    L.tpl_fullatom_backward.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, sz, vp]
    L.tpl_fullatom_backward_from_coords.restype = ctypes.c_int
    L.tpl_fullatom_backward_from_coords.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, sz, vp]
    L.tpl_tables_backward_from_coords_ok.restype = i32
    L.tpl_tables_backward_from_coords_ok.argtypes = [vp]
    L.tpl_backbone_forward_precise.restype = ctypes.c_int
    L.tpl_backbone_forward_precise.argtypes = [vp, vp, i32, i32, vp, vp, sz, vp]
    L.tpl_backbone_lrmsd_forward.restype = ctypes.c_int
    L.tpl_backbone_lrmsd_forward.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    L.tpl_backbone_lrmsd_backward.restype = ctypes.c_int
    L.tpl_backbone_lrmsd_backward.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    L.tpl_backbone_segment_forward.restype = ctypes.c_int
    L.tpl_backbone_segment_forward.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, sz, vp]
    L.tpl_backbone_segment_place.restype = ctypes.c_int
    L.tpl_backbone_segment_place.argtypes = [vp, vp, i32, i32, vp, i32, i32, vp, sz, vp]
    L.tpl_backbone_segment_totals.restype = ctypes.c_int
    L.tpl_backbone_segment_totals.argtypes = [vp, vp, i32, i32, vp, vp, vp, sz, vp]
    L.tpl_backbone_segment_backward.restype = ctypes.c_int
    L.tpl_backbone_segment_backward.argtypes = [vp, vp, i32, i32, vp, vp, i32, i32, vp, vp, sz, vp]
    L.tpl_paper_backbone_saved_floats.restype = i64
    L.tpl_paper_backbone_saved_floats.argtypes = [i32, i32]
    L.tpl_paper_backbone_forward.restype = ctypes.c_int
    L.tpl_paper_backbone_forward.argtypes = [vp, vp, i32, i32, vp, vp, vp, sz, vp]
    L.tpl_paper_backbone_backward.restype = ctypes.c_int
    L.tpl_paper_backbone_backward.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, sz, vp]
    L.tpl_backbone_lrmsd_fused_max_L.restype = i32
    L.tpl_backbone_lrmsd_fused_max_L.argtypes = []
    L.tpl_backbone_lrmsd_fused.restype = ctypes.c_int
    L.tpl_backbone_lrmsd_fused.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]
    L.tpl_chain_scale.restype = ctypes.c_int
    L.tpl_chain_scale.argtypes = [vp, vp, i32, i32, vp, vp]
    L.tpl_lrmsd_forward.restype = ctypes.c_int
    L.tpl_lrmsd_forward.argtypes = [vp, vp, vp, i32, i32, vp, vp, vp, sz, vp]
    L.tpl_lrmsd_backward.restype = ctypes.c_int
    L.tpl_lrmsd_backward.argtypes = [vp, vp, vp, i32, i32, vp, vp, vp, vp, sz, vp]
    return L


lib = _load()


def _check(status):
    if status != TPL_OK:
        raise TplError(status, lib.tpl_last_error().decode(errors="replace"))


def _dev(t, dtype, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (libtpl has no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _on_device(fn):
    """Run the C call with the device of its first CUDA tensor argument current, so
    that the default stream (current_stream()) and the library's per-device launch
    state belong to the device the pointers live on."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        for a in list(args) + list(kwargs.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                with torch.cuda.device(a.device):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)

    return wrapper


def tpl_abi_version():
    return int(lib.tpl_abi_version())


def tpl_workspace_bytes(model, B, Lmax):
    return int(lib.tpl_workspace_bytes(int(model), int(B), int(Lmax)))


def tpl_backbone_atoms(L):
    return int(lib.tpl_backbone_atoms(int(L)))


@_on_device
def tpl_sync_status(workspace, stream=None):
    _check(lib.tpl_sync_status(_stream(stream), _dev(workspace, torch.uint8, "workspace")))


@_on_device
def tpl_backbone_forward(angles, lengths, coords, workspace, stream=None):
    B, Lmax, three = angles.shape
    if three != BB_SLOTS or tuple(coords.shape) != (B, 3 * Lmax, 3) or tuple(lengths.shape) != (B,):
        raise ValueError("shapes: angles [B,Lmax,3], lengths [B], coords [B,3*Lmax,3]")
    _check(lib.tpl_backbone_forward(_dev(angles, torch.float32, "angles"), _dev(lengths, torch.int32, "lengths"),
                                    B, Lmax, _dev(coords, torch.float32, "coords"),
                                    _dev(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream)))


@_on_device
def tpl_backbone_backward(angles, lengths, grad_coords, grad_angles, workspace, stream=None):
    B, Lmax, three = angles.shape
    if (three != BB_SLOTS or tuple(grad_coords.shape) != (B, 3 * Lmax, 3)
            or tuple(grad_angles.shape) != (B, Lmax, 3) or tuple(lengths.shape) != (B,)):
        raise ValueError("shapes: angles/grad_angles [B,Lmax,3], lengths [B], grad_coords [B,3*Lmax,3]")
    _check(lib.tpl_backbone_backward(_dev(angles, torch.float32, "angles"), _dev(lengths, torch.int32, "lengths"),
                                     B, Lmax, _dev(grad_coords, torch.float32, "grad_coords"),
                                     _dev(grad_angles, torch.float32, "grad_angles"),
                                     _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                     _stream(stream)))


@_on_device
def tpl_backbone_backward_from_coords(coords, lengths, grad_coords, grad_angles, workspace, stream=None):
    B, Lmax, three = grad_angles.shape
    if (three != BB_SLOTS or tuple(coords.shape) != (B, 3 * Lmax, 3) or tuple(grad_coords.shape) != (B, 3 * Lmax, 3)
            or tuple(lengths.shape) != (B,)):
        raise ValueError("shapes: coords/grad_coords [B,3*Lmax,3], lengths [B], grad_angles [B,Lmax,3]")
    _check(lib.tpl_backbone_backward_from_coords(_dev(coords, torch.float32, "coords"),
                                                 _dev(lengths, torch.int32, "lengths"), B, Lmax,
                                                 _dev(grad_coords, torch.float32, "grad_coords"),
                                                 _dev(grad_angles, torch.float32, "grad_angles"),
                                                 _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                                 _stream(stream)))


def tpl_tables_create(descs):
    """descs: a ctypes array of ResidueDesc; returns the opaque handle (int)."""
    h = ctypes.c_void_p()
    _check(lib.tpl_tables_create(descs, len(descs), ctypes.byref(h)))
    return h.value


def tpl_tables_destroy(handle):
    lib.tpl_tables_destroy(ctypes.c_void_p(handle))


def tpl_tables_n_types(handle):
    return int(lib.tpl_tables_n_types(ctypes.c_void_p(handle)))


def tpl_fullatom_atoms(handle, restype_host, lengths_host):
    """Host bookkeeping: (atoms_per_chain int32 [B], atom_stride)."""
    rt = restype_host.to(torch.uint8).contiguous().cpu()
    ln = lengths_host.to(torch.int32).contiguous().cpu()
    B, Lmax = rt.shape
    apc = torch.zeros(B, dtype=torch.int32)
    stride = ctypes.c_int32(0)
    _check(lib.tpl_fullatom_atoms(ctypes.c_void_p(handle), ctypes.c_void_p(rt.data_ptr()),
                                  ctypes.c_void_p(ln.data_ptr()), B, Lmax, ctypes.c_void_p(apc.data_ptr()),
                                  ctypes.byref(stride)))
    return apc, int(stride.value)


@_on_device
def tpl_fullatom_forward(handle, angles, restype, lengths, coords, workspace, stream=None):
    B, Lmax, slots = angles.shape
    if slots != FA_SLOTS or tuple(restype.shape) != (B, Lmax) or coords.dim() != 3 or coords.shape[0] != B:
        raise ValueError("shapes: angles [B,Lmax,8], restype [B,Lmax], coords [B,atom_stride,3]")
    _check(lib.tpl_fullatom_forward(ctypes.c_void_p(handle), _dev(angles, torch.float32, "angles"),
                                    _dev(restype, torch.uint8, "restype"), _dev(lengths, torch.int32, "lengths"),
                                    B, Lmax, coords.shape[1], _dev(coords, torch.float32, "coords"),
                                    _dev(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream)))


@_on_device
def tpl_fullatom_backward(handle, angles, restype, lengths, grad_coords, grad_angles, workspace, stream=None):
    B, Lmax, slots = angles.shape
    if slots != FA_SLOTS or tuple(grad_angles.shape) != (B, Lmax, FA_SLOTS) or grad_coords.shape[0] != B:
        raise ValueError("shapes: angles/grad_angles [B,Lmax,8], grad_coords [B,atom_stride,3]")
    _check(lib.tpl_fullatom_backward(ctypes.c_void_p(handle), _dev(angles, torch.float32, "angles"),
                                     _dev(restype, torch.uint8, "restype"), _dev(lengths, torch.int32, "lengths"),
                                     B, Lmax, grad_coords.shape[1], _dev(grad_coords, torch.float32, "grad_coords"),
                                     _dev(grad_angles, torch.float32, "grad_angles"),
                                     _dev(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream)))


@_on_device
def tpl_fullatom_backward_from_coords(handle, coords, restype, lengths, grad_coords, grad_angles, workspace,
                                      stream=None):
    B, Lmax, slots = grad_angles.shape
    if (slots != FA_SLOTS or tuple(restype.shape) != (B, Lmax) or coords.dim() != 3 or coords.shape[0] != B
            or tuple(grad_coords.shape) != tuple(coords.shape)):
        raise ValueError("shapes: coords/grad_coords [B,atom_stride,3], restype [B,Lmax], grad_angles [B,Lmax,8]")
    _check(lib.tpl_fullatom_backward_from_coords(ctypes.c_void_p(handle), _dev(coords, torch.float32, "coords"),
                                                 _dev(restype, torch.uint8, "restype"),
                                                 _dev(lengths, torch.int32, "lengths"), B, Lmax, coords.shape[1],
                                                 _dev(grad_coords, torch.float32, "grad_coords"),
                                                 _dev(grad_angles, torch.float32, "grad_angles"),
                                                 _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                                 _stream(stream)))


def tpl_tables_backward_from_coords_ok(handle):
    return bool(lib.tpl_tables_backward_from_coords_ok(ctypes.c_void_p(handle)))


@_on_device
def tpl_backbone_forward_precise(angles, lengths, coords, workspace, stream=None):
    """f2: the backbone forward computed in fp64 internally (coords rounded to fp32)."""
    B, Lmax, three = angles.shape
    if three != BB_SLOTS or tuple(coords.shape) != (B, 3 * Lmax, 3) or tuple(lengths.shape) != (B,):
        raise ValueError("shapes: angles [B,Lmax,3], lengths [B], coords [B,3*Lmax,3]")
    _check(lib.tpl_backbone_forward_precise(_dev(angles, torch.float32, "angles"),
                                            _dev(lengths, torch.int32, "lengths"), B, Lmax,
                                            _dev(coords, torch.float32, "coords"),
                                            _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                            _stream(stream)))


@_on_device
def tpl_backbone_lrmsd_forward(angles, lengths, target, coords, lrmsd, state, workspace, stream=None):
    """f1: backbone forward + LRMSD against target, fused (per-chain loss over the 3L backbone atoms)."""
    B, Lmax, three = angles.shape
    if (three != BB_SLOTS or tuple(coords.shape) != (B, 3 * Lmax, 3) or tuple(target.shape) != (B, 3 * Lmax, 3)
            or tuple(lrmsd.shape) != (B,) or tuple(state.shape) != (B, 16)):
        raise ValueError("shapes: angles [B,Lmax,3], target/coords [B,3*Lmax,3], lrmsd [B], state [B,16]")
    _check(lib.tpl_backbone_lrmsd_forward(_dev(angles, torch.float32, "angles"),
                                          _dev(lengths, torch.int32, "lengths"), B, Lmax,
                                          _dev(target, torch.float32, "target"), _dev(coords, torch.float32, "coords"),
                                          _dev(lrmsd, torch.float32, "lrmsd"), _dev(state, torch.float32, "state"),
                                          _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                          _stream(stream)))


def tpl_backbone_lrmsd_fused_max_L():
    return int(lib.tpl_backbone_lrmsd_fused_max_L())


@_on_device
def tpl_backbone_lrmsd_fused(angles, lengths, target, coords, lrmsd, state, grad_angles, workspace, stream=None):
    """f1 in one pass: angles -> coords -> LRMSD -> dLRMSD/dangles (coords may be None)."""
    B, Lmax, three = angles.shape
    if (three != BB_SLOTS or tuple(target.shape) != (B, 3 * Lmax, 3) or tuple(lrmsd.shape) != (B,)
            or tuple(state.shape) != (B, 16) or tuple(grad_angles.shape) != (B, Lmax, 3)
            or (coords is not None and tuple(coords.shape) != (B, 3 * Lmax, 3))):
        raise ValueError("shapes: angles/grad_angles [B,Lmax,3], target/coords [B,3*Lmax,3], lrmsd [B], state [B,16]")
    c = _dev(coords, torch.float32, "coords") if coords is not None else None
    _check(lib.tpl_backbone_lrmsd_fused(_dev(angles, torch.float32, "angles"), _dev(lengths, torch.int32, "lengths"),
                                        B, Lmax, _dev(target, torch.float32, "target"), c,
                                        _dev(lrmsd, torch.float32, "lrmsd"), _dev(state, torch.float32, "state"),
                                        _dev(grad_angles, torch.float32, "grad_angles"),
                                        _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                        _stream(stream)))


@_on_device
def tpl_chain_scale(x, scale, y, stream=None):
    """y[b] = x[b] * scale[b] (per-chain scalar; x, y [B, ...] fp32)."""
    B = x.shape[0]
    if tuple(y.shape) != tuple(x.shape) or tuple(scale.shape) != (B,):
        raise ValueError("shapes: x, y [B, ...], scale [B]")
    _check(lib.tpl_chain_scale(_dev(x, torch.float32, "x"), _dev(scale, torch.float32, "scale"), B,
                               x.numel() // max(B, 1), _dev(y, torch.float32, "y"), _stream(stream)))


@_on_device
def tpl_backbone_lrmsd_backward(coords, lengths, target, state, grad_lrmsd, grad_angles, workspace, stream=None):
    B, atoms, _ = coords.shape
    if (tuple(target.shape) != tuple(coords.shape) or tuple(grad_angles.shape) != (B, atoms // 3, 3)
            or tuple(grad_lrmsd.shape) != (B,) or tuple(state.shape) != (B, 16)):
        raise ValueError("shapes: coords/target [B,3*Lmax,3], state [B,16], grad_lrmsd [B], grad_angles [B,Lmax,3]")
    _check(lib.tpl_backbone_lrmsd_backward(_dev(coords, torch.float32, "coords"),
                                           _dev(lengths, torch.int32, "lengths"), B, atoms // 3,
                                           _dev(target, torch.float32, "target"), _dev(state, torch.float32, "state"),
                                           _dev(grad_lrmsd, torch.float32, "grad_lrmsd"),
                                           _dev(grad_angles, torch.float32, "grad_angles"),
                                           _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                           _stream(stream)))


@_on_device
def tpl_backbone_segment_forward(angles, lengths, omega_prev, coords, aggregate, workspace, stream=None):
    B, Lmax, three = angles.shape
    if three != BB_SLOTS or tuple(coords.shape) != (B, 3 * Lmax, 3) or aggregate.numel() != 12 * B:
        raise ValueError("shapes: angles [B,Lmax,3], coords [B,3*Lmax,3], aggregate [B,12]")
    om = _dev(omega_prev, torch.float32, "omega_prev") if omega_prev is not None else None
    _check(lib.tpl_backbone_segment_forward(_dev(angles, torch.float32, "angles"),
                                            _dev(lengths, torch.int32, "lengths"), B, Lmax, om,
                                            _dev(coords, torch.float32, "coords"),
                                            _dev(aggregate, torch.float32, "aggregate"),
                                            _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                            _stream(stream)))


@_on_device
def tpl_backbone_segment_place(coords, lengths, aggregates, seg, workspace, stream=None):
    B, atoms, _ = coords.shape
    n_seg = aggregates.numel() // (12 * B)
    _check(lib.tpl_backbone_segment_place(_dev(coords, torch.float32, "coords"), _dev(lengths, torch.int32, "lengths"),
                                          B, atoms // 3, _dev(aggregates, torch.float32, "aggregates"), n_seg, seg,
                                          _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                          _stream(stream)))


@_on_device
def tpl_backbone_segment_totals(coords, lengths, grad_coords, totals, workspace, stream=None):
    B, atoms, _ = coords.shape
    if tuple(grad_coords.shape) != tuple(coords.shape) or totals.numel() != 12 * B:
        raise ValueError("shapes: coords/grad_coords [B,3*Lmax,3], totals [B,12]")
    _check(lib.tpl_backbone_segment_totals(_dev(coords, torch.float32, "coords"),
                                           _dev(lengths, torch.int32, "lengths"), B, atoms // 3,
                                           _dev(grad_coords, torch.float32, "grad_coords"),
                                           _dev(totals, torch.float32, "totals"),
                                           _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                           _stream(stream)))


@_on_device
def tpl_backbone_segment_backward(coords, lengths, grad_coords, totals, seg, grad_angles, workspace, stream=None):
    B, atoms, _ = coords.shape
    n_seg = totals.numel() // (12 * B)
    if tuple(grad_angles.shape) != (B, atoms // 3, 3) or tuple(grad_coords.shape) != tuple(coords.shape):
        raise ValueError("shapes: coords/grad_coords [B,3*Lmax,3], totals [n_seg,B,12], grad_angles [B,Lmax,3]")
    _check(lib.tpl_backbone_segment_backward(_dev(coords, torch.float32, "coords"),
                                             _dev(lengths, torch.int32, "lengths"), B, atoms // 3,
                                             _dev(grad_coords, torch.float32, "grad_coords"),
                                             _dev(totals, torch.float32, "totals"), n_seg, seg,
                                             _dev(grad_angles, torch.float32, "grad_angles"),
                                             _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                             _stream(stream)))


def tpl_paper_backbone_saved_floats(B, Lmax):
    return int(lib.tpl_paper_backbone_saved_floats(int(B), int(Lmax)))


@_on_device
def tpl_paper_backbone_forward(angles, lengths, coords, saved_M, workspace, stream=None):
    """the paper's GPU design (saves M_i, 64 B/atom) -- a comparison point."""
    B, Lmax, three = angles.shape
    if three != BB_SLOTS or tuple(coords.shape) != (B, 3 * Lmax, 3) or saved_M.numel() != 48 * B * Lmax:
        raise ValueError("shapes: angles [B,Lmax,3], coords [B,3*Lmax,3], saved_M [B,3*Lmax,16]")
    _check(lib.tpl_paper_backbone_forward(_dev(angles, torch.float32, "angles"),
                                          _dev(lengths, torch.int32, "lengths"), B, Lmax,
                                          _dev(coords, torch.float32, "coords"),
                                          _dev(saved_M, torch.float32, "saved_M"),
                                          _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                          _stream(stream)))


@_on_device
def tpl_paper_backbone_backward(angles, lengths, saved_M, grad_coords, grad_angles, workspace, stream=None):
    """O(L^2) per-angle sums without a reduction."""
    B, Lmax, three = angles.shape
    if (three != BB_SLOTS or tuple(grad_coords.shape) != (B, 3 * Lmax, 3)
            or tuple(grad_angles.shape) != (B, Lmax, 3) or saved_M.numel() != 48 * B * Lmax):
        raise ValueError("shapes: angles/grad_angles [B,Lmax,3], grad_coords [B,3*Lmax,3], saved_M [B,3*Lmax,16]")
    _check(lib.tpl_paper_backbone_backward(_dev(angles, torch.float32, "angles"),
                                           _dev(lengths, torch.int32, "lengths"), B, Lmax,
                                           _dev(saved_M, torch.float32, "saved_M"),
                                           _dev(grad_coords, torch.float32, "grad_coords"),
                                           _dev(grad_angles, torch.float32, "grad_angles"),
                                           _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
                                           _stream(stream)))


@_on_device
def tpl_lrmsd_forward(x, y, n_atoms, lrmsd, state, workspace, stream=None):
    B, S, three = x.shape
    if three != 3 or tuple(y.shape) != (B, S, 3) or tuple(lrmsd.shape) != (B,) or tuple(state.shape) != (B, 16):
        raise ValueError("shapes: x, y [B,stride,3], n_atoms [B], lrmsd [B], state [B,16]")
    _check(lib.tpl_lrmsd_forward(_dev(x, torch.float32, "x"), _dev(y, torch.float32, "y"),
                                 _dev(n_atoms, torch.int32, "n_atoms"), B, S, _dev(lrmsd, torch.float32, "lrmsd"),
                                 _dev(state, torch.float32, "state"), _dev(workspace, torch.uint8, "workspace"),
                                 workspace.numel(), _stream(stream)))


@_on_device
def tpl_lrmsd_backward(x, y, n_atoms, state, grad_lrmsd, grad_x, workspace, stream=None):
    B, S, three = x.shape
    if three != 3 or tuple(grad_x.shape) != (B, S, 3) or tuple(grad_lrmsd.shape) != (B,):
        raise ValueError("shapes: x, y, grad_x [B,stride,3], grad_lrmsd [B], state [B,16]")
    _check(lib.tpl_lrmsd_backward(_dev(x, torch.float32, "x"), _dev(y, torch.float32, "y"),
                                  _dev(n_atoms, torch.int32, "n_atoms"), B, S, _dev(state, torch.float32, "state"),
                                  _dev(grad_lrmsd, torch.float32, "grad_lrmsd"), _dev(grad_x, torch.float32, "grad_x"),
                                  _dev(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream)))
