"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no transforms, no trig of the
angles, no gradients): it draws random numbers, loads the residue-type table
(data, see tools/make_residue_table.py) and names the BASELINE.json configs.
Both the oracle and the CUDA path consume what it produces; neither imports
the other.

Recipe:
  * angles      = (2 U[0,1) - 1) * pi, fp32     ("random input angles")
  * grad_coords = N(0, 1), fp32                 (synthetic dL/dr; L = sum g . r)
  * restype     = uniform over the 20 types     ("sequences were generated at random")
  * lengths     = uniform integers in [lo, hi]  (ragged config 4)
  * seeds       = 1000+c (angles), 2000+c (grad), 3000+c (lengths), 4000+c (restype)
"""
import copy
import json
import math
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
TABLE_PATH = os.path.join(_HERE, "residue_table.json")

N_SLOTS_BB = 3  # phi, psi, omega
N_SLOTS_FA = 8  # phi, psi, omega, chi1..chi5

# BASELINE.json "configs" (index = position in the list, 1-based as in SURVEY).
CONFIGS = {
    1: dict(model="backbone", B=1, L=16, desc="backbone L=16 batch 1, fp32 vs fp64 oracle + FD"),
    2: dict(model="backbone", B=64, L=700, desc="backbone 64 x L=700 fwd+bwd"),
    3: dict(model="fullatom", B=64, L=300, desc="full-atom 64 x L=300, 20 random residue types"),
    4: dict(model="backbone", B=4096, L=2000, ragged=(50, 2000), desc="ragged backbone L in [50,2000], batch 4096"),
    5: dict(model="fullatom", B=8192, L=500, desc="full-atom 8192 x L=500 (8-GPU stress)"),
    "metric": dict(model="backbone", B=256, L=700, desc="headline: backbone L=700 batch 256 fwd+bwd"),
    # NEXT rows, measured beside the BASELINE configs
    "lrmsd": dict(model="backbone", B=256, L=700, loss="lrmsd",
                  desc="f1: headline shape with the LRMSD loss (PAPER 4) between forward and backward"),
    "long": dict(model="backbone", B=1, L=20000, desc="f4: one 20000-residue chain split over CTAs"),
}
_IDS = {"metric": 0, "lrmsd": 6, "long": 7}


def config_id(c):
    if c in _IDS:
        return _IDS[c]
    if isinstance(c, str) and ":" in c:
        return 90  # ad-hoc measurement shapes (register_custom)
    return int(c)


def register_custom(name):
    """Ad-hoc measurement shape "bb:B:L", "bb:B:lo-hi" (ragged) or "fa:B:L" (not a
    BASELINE config: kernel studies beside the configs)."""
    if name in CONFIGS:
        return name
    kind, B, L = name.split(":")
    cfg = dict(model="backbone" if kind == "bb" else "fullatom", B=int(B), desc=f"ad-hoc {name}")
    if "-" in L:
        lo, hi = (int(x) for x in L.split("-"))
        cfg.update(L=hi, ragged=(lo, hi))
    else:
        cfg["L"] = int(L)
    CONFIGS[name] = cfg
    return name


def _gen(seed):
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def angles_uniform(B, Lmax, n_slots, seed):
    """fp32 angles (2U-1)*pi, shape [B, Lmax, n_slots]."""
    u = torch.rand((B, Lmax, n_slots), generator=_gen(seed), dtype=torch.float32)
    return (2.0 * u - 1.0) * math.pi


def grad_normal(shape, seed):
    """fp32 N(0,1) synthetic upstream gradient dL/dr."""
    return torch.randn(tuple(shape), generator=_gen(seed), dtype=torch.float32)


def lengths_uniform(B, lo, hi, seed):
    return torch.randint(int(lo), int(hi) + 1, (B,), generator=_gen(seed), dtype=torch.int32)


def restype_uniform(B, Lmax, n_types, seed):
    return torch.randint(0, int(n_types), (B, Lmax), generator=_gen(seed), dtype=torch.uint8)


def regular_angles(B, L, kind):
    """Regular secondary structure / special chains: fp32 [B, L, 3]."""
    deg = {"helix": (-57.0, -47.0, 180.0), "strand": (-120.0, 130.0, 180.0),
           "extended": (180.0, 180.0, 180.0), "cis": (0.0, 0.0, 0.0)}[kind]
    a = torch.tensor([math.radians(x) for x in deg], dtype=torch.float32)
    return a.expand(B, L, 3).contiguous()


def load_residue_table(variant="default"):
    """The per-residue-type rigid-group table (data).  variant="chi5" frees ARG's
    chi5 (slot 7) to exercise the deepest group (reading Q10)."""
    with open(TABLE_PATH) as f:
        table = json.load(f)
    if variant == "chi5":
        table = copy.deepcopy(table)
        for ty in table["types"]:
            if ty["name"] == "ARG":
                ty["groups"][4]["slot"] = 7
                ty["groups"][4]["alpha"] = 0.0
    elif variant != "default":
        raise ValueError(variant)
    return table


def backbone_inputs(c, B=None, L=None):
    """(angles fp32 [B,L,3], lengths int32 [B], grad fp32 [B,3L,3]) for config c."""
    cfg = CONFIGS[c]
    cid = config_id(c)
    B = cfg["B"] if B is None else B
    L = cfg["L"] if L is None else L
    ang = angles_uniform(B, L, N_SLOTS_BB, 1000 + cid)
    if cfg.get("ragged"):
        lo, hi = cfg["ragged"]
        lengths = lengths_uniform(B, lo, min(hi, L), 3000 + cid)
    else:
        lengths = torch.full((B,), L, dtype=torch.int32)
    grad = grad_normal((B, 3 * L, 3), 2000 + cid)
    return ang, lengths, grad


def fullatom_inputs(c, B=None, L=None, n_types=20):
    """(angles fp32 [B,L,8], restype u8 [B,L], lengths int32 [B]) for config c."""
    cfg = CONFIGS[c]
    cid = config_id(c)
    B = cfg["B"] if B is None else B
    L = cfg["L"] if L is None else L
    ang = angles_uniform(B, L, N_SLOTS_FA, 1000 + cid)
    rt = restype_uniform(B, L, n_types, 4000 + cid)
    if cfg.get("ragged"):
        lo, hi = cfg["ragged"]
        lengths = lengths_uniform(B, lo, min(hi, L), 3000 + cid)
    else:
        lengths = torch.full((B,), L, dtype=torch.int32)
    return ang, rt, lengths


def fullatom_grad(B, atom_stride, cid):
    return grad_normal((B, atom_stride, 3), 2000 + cid)


def numpy64(t):
    """Exact fp32 -> fp64 promotion for the oracle."""
    return np.asarray(t.detach().cpu().numpy(), dtype=np.float64)
