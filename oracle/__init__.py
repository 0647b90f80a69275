"""fp64 CPU oracle for arXiv 1812.01108 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
(``paper_1812_01108_b200``) never does; the two share no code (the seeded
input generators live in ``synth/``, which holds none of the method's
arithmetic).

The arithmetic lives in ``oracle.c`` (the paper's sequential transform chain
and its O(L^2) Eq. 1 / Eq. 2 backward, fp64).  This module only marshals numpy
arrays into it, plus the LRMSD oracle in ``lrmsd.py``.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
against values and properties fixed by the paper and by geometry (DESIGN.md
"Oracle pins").  Absolute side-chain geometry is data (the residue table,
reading Q8), pinned against textbook covalent geometry (Engh & Huber bond
lengths and angles, connectivity, ring planarity; V16).
"""
import ctypes
import os
import shutil
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

MAX_GROUPS = 8
MAX_ATOMS = 16
SLOTS = 8
OWNER_N, OWNER_CA, OWNER_C = -3, -2, -1


class RestypeC(ctypes.Structure):
    """Mirror of ``tplref_restype`` in oracle.h (the oracle's own struct)."""

    _fields_ = [
        ("n_groups", ctypes.c_int32),
        ("n_atoms", ctypes.c_int32),
        ("g_parent", ctypes.c_int32 * MAX_GROUPS),
        ("g_slot", ctypes.c_int32 * MAX_GROUPS),
        ("g_alpha", ctypes.c_double * MAX_GROUPS),
        ("g_theta", ctypes.c_double * MAX_GROUPS),
        ("g_d", ctypes.c_double * MAX_GROUPS),
        ("g_prerx", ctypes.c_double * MAX_GROUPS),
        ("a_owner", ctypes.c_int32 * MAX_ATOMS),
        ("a_r", (ctypes.c_double * 3) * MAX_ATOMS),
    ]


def build(force=False):
    """Compile liboracle.so with plain gcc (fp64, -ffp-contract=off, OpenMP)."""
    src = [os.path.join(_HERE, f) for f in ("oracle.c", "oracle.h")]
    if not force and os.path.exists(_LIB_PATH):
        if os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(s) for s in src):
            return _LIB_PATH
    cc = shutil.which("gcc") or "gcc"
    cmd = [cc, "-O2", "-std=c11", "-fPIC", "-fopenmp", "-ffp-contract=off", "-D_DEFAULT_SOURCE",
           "-shared", "-o", _LIB_PATH, src[0], "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp, ip, u8p = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint8)
        i32 = ctypes.c_int32
        L.tplref_bond_transform.argtypes = [ctypes.c_double] * 3 + [dp]
        L.tplref_bond_transform_dalpha.argtypes = [ctypes.c_double] * 3 + [dp]
        L.tplref_num_threads.restype = ctypes.c_int
        L.tplref_set_num_threads.restype = None
        L.tplref_set_num_threads.argtypes = [ctypes.c_int]
        L.tplref_backbone_forward.argtypes = [dp, ip, i32, i32, dp]
        L.tplref_backbone_backward.argtypes = [dp, ip, i32, i32, dp, dp]
        rp = ctypes.POINTER(RestypeC)
        L.tplref_fullatom_forward.argtypes = [rp, i32, dp, u8p, ip, i32, i32, i32, dp, ip]
        L.tplref_fullatom_backward.argtypes = [rp, i32, dp, u8p, ip, i32, i32, i32, dp, dp]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} rejected its input (code {rc})")


def num_threads():
    return int(lib().tplref_num_threads())


def set_num_threads(n):
    lib().tplref_set_num_threads(int(n))


def bond_transform(alpha, theta, d):
    out = np.zeros(16)
    lib().tplref_bond_transform(float(alpha), float(theta), float(d), _p(out, ctypes.c_double))
    return out.reshape(4, 4)


def bond_transform_dalpha(alpha, theta, d):
    out = np.zeros(16)
    lib().tplref_bond_transform_dalpha(float(alpha), float(theta), float(d), _p(out, ctypes.c_double))
    return out.reshape(4, 4)


def backbone_forward(angles, lengths):
    """angles [B, Lmax, 3] (phi, psi, omega) -> coords [B, 3*Lmax, 3] (N, CA, C); pads 0."""
    a = _f64(angles)
    B, Lmax, _ = a.shape
    ln = _i32(lengths)
    out = np.zeros((B, 3 * Lmax, 3))
    _check(lib().tplref_backbone_forward(_p(a, ctypes.c_double), _p(ln, ctypes.c_int32), B, Lmax,
                                         _p(out, ctypes.c_double)), "backbone_forward")
    return out


def backbone_backward(angles, lengths, grad_coords):
    """Eq. 2, O(L^2): dL/d(phi, psi, omega) [B, Lmax, 3] for L = sum grad_coords . r."""
    a = _f64(angles)
    B, Lmax, _ = a.shape
    ln = _i32(lengths)
    g = _f64(grad_coords).reshape(B, 3 * Lmax, 3)
    out = np.zeros((B, Lmax, 3))
    _check(lib().tplref_backbone_backward(_p(a, ctypes.c_double), _p(ln, ctypes.c_int32), B, Lmax,
                                          _p(g, ctypes.c_double), _p(out, ctypes.c_double)), "backbone_backward")
    return out


def restypes_from_table(table):
    """Residue-type records (dict loaded from synth/residue_table.json) -> ctypes array."""
    types = table["types"]
    arr = (RestypeC * len(types))()
    for t, ty in enumerate(types):
        rec = arr[t]
        rec.n_groups = len(ty["groups"])
        rec.n_atoms = len(ty["atoms"])
        if rec.n_groups > MAX_GROUPS or rec.n_atoms > MAX_ATOMS:
            raise ValueError("residue type too large for the oracle")
        for g, gr in enumerate(ty["groups"]):
            rec.g_parent[g] = int(gr["parent"])
            rec.g_slot[g] = int(gr["slot"])
            rec.g_alpha[g] = float(gr["alpha"])
            rec.g_theta[g] = float(gr["theta"])
            rec.g_d[g] = float(gr["d"])
            rec.g_prerx[g] = float(gr["pre_rx"])
        for k, at in enumerate(ty["atoms"]):
            rec.a_owner[k] = int(at["owner"])
            for c in range(3):
                rec.a_r[k][c] = float(at["r"][c])
    return arr


def chain_atom_counts(table, restype, lengths):
    """Bookkeeping: atoms per chain (sum of the table's per-type atom counts)."""
    n = np.array([len(t["atoms"]) for t in table["types"]], dtype=np.int64)
    rt = np.asarray(restype)
    if rt.size and int(rt.max()) >= len(n):
        raise ValueError("restype out of range")
    return np.array([int(n[rt[b, : int(L)]].sum()) for b, L in enumerate(lengths)], dtype=np.int64)


def fullatom_forward(table, angles, restype, lengths, atom_stride=None):
    """angles [B, Lmax, 8], restype [B, Lmax] -> (coords [B, stride, 3], n_atoms [B])."""
    a = _f64(angles)
    B, Lmax, _ = a.shape
    rt = np.ascontiguousarray(restype, dtype=np.uint8)
    ln = _i32(lengths)
    if atom_stride is None:
        atom_stride = int(max(chain_atom_counts(table, rt, ln).max(), 1))
    types = restypes_from_table(table)
    out = np.zeros((B, atom_stride, 3))
    nat = np.zeros(B, dtype=np.int32)
    _check(lib().tplref_fullatom_forward(types, len(types), _p(a, ctypes.c_double), _p(rt, ctypes.c_uint8),
                                         _p(ln, ctypes.c_int32), B, Lmax, atom_stride, _p(out, ctypes.c_double),
                                         _p(nat, ctypes.c_int32)), "fullatom_forward")
    return out, nat


def fullatom_backward(table, angles, restype, lengths, grad_coords):
    """Eq. 1 depth-first, O(L^2): dL/d(angles) [B, Lmax, 8] for L = sum grad_coords . r."""
    a = _f64(angles)
    B, Lmax, _ = a.shape
    rt = np.ascontiguousarray(restype, dtype=np.uint8)
    ln = _i32(lengths)
    g = _f64(grad_coords)
    atom_stride = g.shape[1]
    types = restypes_from_table(table)
    out = np.zeros((B, Lmax, SLOTS))
    _check(lib().tplref_fullatom_backward(types, len(types), _p(a, ctypes.c_double), _p(rt, ctypes.c_uint8),
                                          _p(ln, ctypes.c_int32), B, Lmax, atom_stride, _p(g, ctypes.c_double),
                                          _p(out, ctypes.c_double)), "fullatom_backward")
    return out
