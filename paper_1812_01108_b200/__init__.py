"""paper_1812_01108_b200 -- B200-native angles -> coordinates (arXiv 1812.01108).

Hot path: batched backbone (phi, psi, omega -> N, CA, C) and full-atom
(phi, psi, omega, chi1..chi5 -> heavy atoms) forward and backward, as
hand-written sm_100a CUDA kernels behind the C ABI of ``libtpl.so``
(``include/tpl.h``).  This package is the thin Python binding (argument
marshalling, autograd glue, batch sharding for multi-GPU runs).
"""
from . import _abi
from ._abi import TplError, lib
from .api import (BackboneFunction, BackboneLRMSDFunction, FullAtomFunction, LRMSDFunction, Tables, Workspace,
                  backbone, backbone_lrmsd, default_workspace, fullatom, lrmsd)

__all__ = ["TplError", "lib", "Tables", "Workspace", "backbone", "fullatom", "BackboneFunction",
           "FullAtomFunction", "LRMSDFunction", "lrmsd", "backbone_lrmsd", "BackboneLRMSDFunction", "default_workspace", "_abi"]
