"""ctypes binding of libsplatnav_b200.so (the C ABI declared in include/splatnav_b200.h).

The shared library is built in-tree by ``paper_2604_12626_b200.build`` (nvcc, sm_100a). There is
no fallback: if the library is missing, every entry point raises.
"""

import ctypes
import os
import threading

from .errors import ContractViolation, NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPLATNAV_B200_LIB") or os.path.join(_HERE, "libsplatnav_b200.so")

SN_OK, SN_ERR_INVALID, SN_ERR_CUDA, SN_ERR_NOMEM = 0, 1, 2, 3
SN_FLOAT32, SN_FLOAT64 = 0, 1
ABI_VERSION = 3

c_double_p = ctypes.POINTER(ctypes.c_double)
P = ctypes.c_void_p


class SnCamera(ctypes.Structure):
    _fields_ = [
        ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("near_", ctypes.c_double), ("far_", ctypes.c_double),
        ("rot", ctypes.c_double * 9), ("trans", ctypes.c_double * 3), ("center", ctypes.c_double * 3),
        ("background", ctypes.c_double * 3),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("has_background", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


class SnStats(ctypes.Structure):
    _fields_ = [("n_input", ctypes.c_int64), ("n_culled_depth", ctypes.c_int64),
                ("n_culled_frame", ctypes.c_int64), ("n_degenerate", ctypes.c_int64), ("n_drawn", ctypes.c_int64)]


class SnCloud(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_k", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("pos_opacity", P), ("log_scales", P), ("rotations", P), ("sh", P), ("index", P),
                ("block_bounds", P)]


class SnAvatars(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_avatars", ctypes.c_int32), ("n_joints", ctypes.c_int32),
                ("sh_k", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("pos_opacity", P), ("log_scales", P), ("rotations", P), ("sh", P), ("joints", P), ("weights", P),
                ("avatar_of", P), ("inv_bind", P), ("traj_q", P), ("traj_t", P), ("traj_offset", P),
                ("n_frames", P), ("fps", P), ("start_offset", P), ("loop", P),
                ("infl_offset", P), ("infl_joint", P), ("infl_weight", P)]


class SnRenderOpts(ctypes.Structure):
    _fields_ = [("tiled", ctypes.c_int32), ("binning", ctypes.c_int32), ("avatar_active", P),
                ("contrib_scene", P), ("contrib_layer", P), ("stats", P), ("stage_ms", P), ("work", P),
                ("exact", ctypes.c_int32), ("serialize", ctypes.c_int32), ("rgb8", P), ("depth16", P),
                ("views", ctypes.c_int32), ("near_slice", ctypes.c_int32)]


STAGES = ("pose", "count", "scan", "emit", "depth_sort", "permute", "pair_scan", "bin_count", "bin_scatter", "ranges",
          "blend", "composite", "far")


# every symbol include/splatnav_b200.h declares (tests check the library exports all of them)
EXPORTS = (
    "sn_abi_version", "sn_last_error", "sn_context_create", "sn_context_destroy", "sn_context_workspace_bytes",
    "sn_context_sync_stats", "sn_context_kernel_launches", "sn_context_render_retries",
    "sn_render", "sn_render_async", "sn_render_wait", "sn_get_counts", "sn_get_sorted_ids", "sn_get_tile_csr", "sn_get_device_tiles", "sn_get_projection", "sn_sample_pose",
    "sn_skin_lbs", "sn_blend_tile_range", "sn_composite", "sn_selftest_fast_exp", "sn_unpack_ply",
    "sn_unpack_bundle", "sn_pack_influences", "sn_quantize_frames", "sn_flip_rows",
)

_lib = None
_lock = threading.Lock()


def load():
    """Load the extension (raises NativeError when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        sig = {
            "sn_abi_version": ([], ctypes.c_int),
            "sn_last_error": ([], ctypes.c_char_p),
            "sn_context_create": ([ctypes.POINTER(P)], ctypes.c_int),
            "sn_context_destroy": ([P], ctypes.c_int),
            "sn_context_workspace_bytes": ([P, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
            "sn_context_sync_stats": ([P], ctypes.c_int),
            "sn_context_kernel_launches": ([P, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
            "sn_context_render_retries": ([P, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
            "sn_render": ([P, ctypes.POINTER(SnCloud), ctypes.POINTER(SnCloud), ctypes.POINTER(SnAvatars), P, P, i32,
                           ctypes.POINTER(SnRenderOpts), P, P, P, P], ctypes.c_int),
            "sn_render_async": ([P, ctypes.POINTER(SnCloud), ctypes.POINTER(SnCloud), ctypes.POINTER(SnAvatars), P, P,
                                 i32, ctypes.POINTER(SnRenderOpts), P, P, P, P], ctypes.c_int),
            "sn_render_wait": ([P, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
            "sn_get_counts": ([P, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)], ctypes.c_int),
            "sn_get_sorted_ids": ([P, i32, i32, P, i64], ctypes.c_int),
            "sn_get_tile_csr": ([P, i32, i32, P, P, i64], ctypes.c_int),
            "sn_get_projection": ([P, i32, i32, P, P, P, P, P, i64], ctypes.c_int),
            "sn_get_device_tiles": ([P, i32, i32, P, P, i64, ctypes.POINTER(i64)], ctypes.c_int),
            "sn_sample_pose": ([P, ctypes.POINTER(SnAvatars), P, i32, P, P, P], ctypes.c_int),
            "sn_skin_lbs": ([P, ctypes.POINTER(SnAvatars), i32, i64, i64, P, P, P, P, P], ctypes.c_int),
            "sn_blend_tile_range": ([i32] * 6 + [P, i64, P, i64, P, P, P, P, P, i64, P, P, P, P], ctypes.c_int),
            "sn_composite": ([i64] + [P] * 9 + [P], ctypes.c_int),
            "sn_selftest_fast_exp": ([ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
            "sn_unpack_ply": ([i64, i32, P, P, i32, P, P, P, P, P, P, P], ctypes.c_int),
            "sn_quantize_frames": ([i64, P, P, P, P, P], ctypes.c_int),
            "sn_flip_rows": ([i64, i32, i32, P, P, P], ctypes.c_int),
            "sn_unpack_bundle": ([i64, i32, i32, P, P, i64, i64, P, P, P, P, P, P, P, P, P, P], ctypes.c_int),
            "sn_pack_influences": ([i64, i32, P, P, P, P, P, P, P], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.sn_abi_version() != ABI_VERSION:
            raise NativeError(f"ABI mismatch: library reports {L.sn_abi_version()}, binding expects {ABI_VERSION}")
        _lib = L
    return _lib


def check(rc):
    if rc == SN_OK:
        return
    msg = load().sn_last_error().decode(errors="replace")
    if rc == SN_ERR_INVALID:
        raise ContractViolation(msg)
    raise NativeError(f"splatnav_b200 error {rc}: {msg}")


class Context:
    """Owns one sn_context (device workspace). One per thread/device."""

    def __init__(self):
        self._lib = load()
        h = P()
        check(self._lib.sn_context_create(ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.sn_context_destroy(h)
            except Exception:
                pass
            self.handle = None

    def sync_stats(self):
        check(self._lib.sn_context_sync_stats(self.handle))

    def kernel_launches(self):
        v = ctypes.c_int64()
        check(self._lib.sn_context_kernel_launches(self.handle, ctypes.byref(v)))
        return int(v.value)

    def render_wait(self):
        """Wait for the oldest render queued with render_frames(..., wait=False) and check it.
        Returns True when it must be queued again (the workspace grew; its frames are invalid)."""
        r = ctypes.c_int32()
        check(self._lib.sn_render_wait(self.handle, ctypes.byref(r)))
        return bool(r.value)

    def render_retries(self):
        v = ctypes.c_int64()
        check(self._lib.sn_context_render_retries(self.handle, ctypes.byref(v)))
        return int(v.value)

    def workspace_bytes(self):
        v = ctypes.c_size_t()
        check(self._lib.sn_context_workspace_bytes(self.handle, ctypes.byref(v)))
        return int(v.value)


def selftest_fast_exp():
    """Largest relative error of the blend's float32 fast exp over its argument range (device)."""
    v = ctypes.c_double()
    check(load().sn_selftest_fast_exp(ctypes.byref(v)))
    return float(v.value)


_tls = threading.local()


def default_context():
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context()
        _tls.ctx = ctx
    return ctx
