"""Kernel plugin registry (reference: splatnav/raster/__init__.py:21-40).

The reference selects between a Cython and a numpy blend kernel. Here the registry holds one
kernel, "cuda", whose ``blend_tile_range`` has the reference's exact argument list
(_kernels_cy.pyx:89-114) and runs on the GPU through the C ABI (sn_blend_tile_range). Asking for
any other kernel fails loudly; there is no CPU fallback.
"""

import os

from . import _kernels_cuda

_KERNELS = {"cuda": _kernels_cuda}


def available_kernels():
    """Mapping of kernel name -> module."""
    return dict(_KERNELS)


def get_kernel(name=None):
    """Resolve a kernel module by name, SPLATNAV_KERNEL, or the default ("cuda")."""
    if name is None:
        name = os.environ.get("SPLATNAV_KERNEL", "").strip().lower() or None
    if name is None:
        return _kernels_cuda
    if name not in _KERNELS:
        raise ValueError(f"unknown kernel {name!r}; available: {sorted(_KERNELS)}")
    return _KERNELS[name]


def active_kernel_name():
    return get_kernel().KERNEL_NAME
