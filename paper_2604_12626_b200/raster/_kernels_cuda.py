"""The "cuda" blend kernel: blend_tile_range with the reference's contract
(_kernels_cy.pyx:89-114): host float64 buffers, caller-initialized accumulators, in-place
accumulation over tiles [t_begin, t_end). Runs sn_blend_tile_range (GPU)."""

import ctypes

import numpy as np

from .. import _native as N
from ..errors import ContractViolation

TRANSMITTANCE_CUTOFF = 1e-4
SUPPORT_D2 = 9.0
ALPHA_CLIP = 0.99

KERNEL_NAME = "cuda"


def _arr(a, dtype, name):
    if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags.c_contiguous:
        raise ContractViolation(f"{name} must be a C-contiguous {np.dtype(dtype).name} array")
    return a


def blend_tile_range(t_begin, t_end, tiles_x, tile_size, width, height, tile_starts, pair_splat, means2d, conics,
                     depths, colors, alphas, color_acc, alpha_acc, trans, depth_acc):
    """Blend tiles [t_begin, t_end) into the accumulation buffers (same semantics as the reference)."""
    ts = _arr(tile_starts, np.int64, "tile_starts")
    ps = _arr(pair_splat, np.int32, "pair_splat")
    f = [_arr(a, np.float64, n) for a, n in ((means2d, "means2d"), (conics, "conics"), (depths, "depths"),
                                             (colors, "colors"), (alphas, "alphas"))]
    acc = [_arr(a, np.float64, n) for a, n in ((color_acc, "color_acc"), (alpha_acc, "alpha_acc"),
                                               (trans, "trans"), (depth_acc, "depth_acc"))]
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    N.check(N.load().sn_blend_tile_range(int(t_begin), int(t_end), int(tiles_x), int(tile_size), int(width),
                                         int(height), p(ts), ts.size, p(ps), ps.size, *[p(a) for a in f],
                                         f[2].size, *[p(a) for a in acc]))
