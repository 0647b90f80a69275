"""C-ABI contract checks that need no GPU: the library builds for sm_100a,
loads, exports every symbol include/tpl.h declares, and rejects bad host
arguments before any launch."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def abi():
    from paper_1812_01108_b200 import build

    build.build()
    from paper_1812_01108_b200 import _abi

    return _abi


def _declared():
    with open(os.path.join(ROOT, "include", "tpl.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"TPL_API[^;(]*?\b(tpl_\w+)\s*\(", src)))


def test_exports_match_header(abi):
    declared = _declared()
    assert len(declared) >= 13
    assert sorted(abi.EXPORTS) == declared
    for name in declared:
        assert hasattr(abi.lib, name), name  # dlsym succeeds


def test_sass_is_sm100a():
    import subprocess

    from paper_1812_01108_b200.build import LIB

    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # TMA bulk copies (cp.async.bulk) are in the kernels


def test_host_only_entry_points(abi):
    assert abi.tpl_abi_version() == 1
    assert abi.tpl_backbone_atoms(700) == 2100
    assert abi.tpl_backbone_atoms(-1) == 0
    assert abi.tpl_workspace_bytes(0, 256, 700) >= 256
    # longer chains need per-tile prefix carries in the workspace
    assert abi.tpl_workspace_bytes(0, 8, 5000) > abi.tpl_workspace_bytes(0, 8, 500)
    assert abi.tpl_workspace_bytes(1, 8, 5000) > abi.tpl_workspace_bytes(1, 8, 100)


def test_null_and_shape_rejected_before_launch(abi):
    L = abi.lib
    vp = ctypes.c_void_p
    buf = ctypes.create_string_buffer(4096)
    p = vp(ctypes.addressof(buf))
    # NULL angles
    assert L.tpl_backbone_forward(None, p, 1, 4, p, p, 4096, None) == 1
    assert b"NULL" in L.tpl_last_error()
    # bad shape
    assert L.tpl_backbone_forward(p, p, 0, 4, p, p, 4096, None) == 2
    assert L.tpl_backbone_backward(p, p, 1, 0, p, p, p, 4096, None) == 2
    assert L.tpl_backbone_backward_from_coords(None, p, 1, 4, p, p, p, 4096, None) == 1
    assert L.tpl_backbone_backward_from_coords(p, p, 1, 0, p, p, p, 4096, None) == 2
    assert L.tpl_backbone_backward_from_coords(p, p, 1, 4, None, p, p, 4096, None) == 1
    assert L.tpl_backbone_backward_from_coords(p, p, 1, 4, p, p, p, 8, None) == 7
    # workspace too small / NULL
    assert L.tpl_backbone_forward(p, p, 1, 4, p, p, 8, None) == 7
    assert L.tpl_backbone_forward(p, p, 1, 4, p, None, 4096, None) == 7
    # misaligned
    q = vp(ctypes.addressof(buf) + 2)
    assert L.tpl_backbone_forward(q, p, 1, 4, p, p, 4096, None) == 3
    # full atom: NULL tables
    assert L.tpl_fullatom_forward(None, p, p, p, 1, 4, 16, p, p, 4096, None) == 1
    # f1 fused, f2 precise, f3 paper design, f4 segments: host checks before any launch
    assert L.tpl_backbone_lrmsd_forward(p, p, 1, 4, None, p, p, p, p, 4096, None) == 1
    assert L.tpl_backbone_lrmsd_backward(p, p, 0, 4, p, p, p, p, p, 4096, None) == 2
    assert L.tpl_backbone_forward_precise(p, p, 1, 4, None, p, 4096, None) == 1
    assert L.tpl_paper_backbone_forward(p, p, 1, 4, p, None, p, 4096, None) == 1
    assert L.tpl_paper_backbone_saved_floats(2, 5) == 2 * 15 * 16 and L.tpl_paper_backbone_saved_floats(0, 5) == 0
    assert L.tpl_backbone_segment_place(p, p, 1, 4, p, 2, 2, p, 4096, None) == 2  # seg outside [0, n_seg)
    assert L.tpl_backbone_segment_backward(p, p, 1, 4, p, p, 0, 0, p, p, 4096, None) == 2
    assert L.tpl_backbone_segment_totals(p, p, 1, 4, None, p, p, 4096, None) == 1


def test_table_validation_before_upload(abi, table):
    from paper_1812_01108_b200.api import Tables  # noqa: F401  (import path works without a GPU)

    descs = (abi.ResidueDesc * 1)()
    d = descs[0]
    d.n_groups, d.n_atoms = 1, 3
    d.group_parent[0] = 5  # invalid: must be -1 or g-1
    d.atom_owner[0], d.atom_owner[1], d.atom_owner[2] = abi.OWNER_N, abi.OWNER_CA, abi.OWNER_C
    h = ctypes.c_void_p()
    assert abi.lib.tpl_tables_create(descs, 1, ctypes.byref(h)) == 4 and not h.value
    d.group_parent[0] = -1
    d.group_slot[0] = 9  # invalid slot
    assert abi.lib.tpl_tables_create(descs, 1, ctypes.byref(h)) == 4
    d.group_slot[0] = 3
    d.atom_owner[0], d.atom_owner[2] = abi.OWNER_C, abi.OWNER_N  # not owner-sorted
    assert abi.lib.tpl_tables_create(descs, 1, ctypes.byref(h)) == 4
    assert b"owner-sorted" in abi.lib.tpl_last_error()
    assert abi.lib.tpl_tables_create(descs, 0, ctypes.byref(h)) == 4
    assert abi.lib.tpl_tables_create(None, 1, ctypes.byref(h)) == 1


def test_cuda_tensors_required(abi):
    import torch

    a = torch.zeros(1, 4, 3)
    with pytest.raises(TypeError):
        abi.tpl_backbone_forward(a, torch.ones(1, dtype=torch.int32), torch.zeros(1, 12, 3),
                                 torch.zeros(4096, dtype=torch.uint8))


def test_backbone_constant_literals():
    """kernels.h compiles the §3 constants as fp32 literals: each must be
    the fp64 cos/sin of pi - 2.1186 / pi - 1.9391 / pi - 2.0610 and d, rounded once."""
    import math

    import numpy as np

    with open(os.path.join(ROOT, "paper_1812_01108_b200", "csrc", "kernels.h")) as f:
        src = f.read()

    def lits(name):
        m = re.search(name + r"\[3\] = \{([^}]*)\}", src)
        return [np.float32(float(x.strip().rstrip("f"))) for x in m.group(1).split(",")]

    th = [math.pi - 2.1186, math.pi - 1.9391, math.pi - 2.0610]
    d = [1.330, 1.460, 1.525]
    assert lits("kBBct") == [np.float32(math.cos(t)) for t in th]
    assert lits("kBBst") == [np.float32(math.sin(t)) for t in th]
    assert lits("kBBd") == [np.float32(x) for x in d]
