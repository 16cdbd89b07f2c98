"""Drop-in renderer entry points (reference: splatnav/renderer.py:31-177).

Same signatures and return types as the reference -- FrameRGBD of numpy float64 arrays, stats
accumulated into a RenderStats -- but every stage runs in the CUDA extension through the C ABI
(sn_render). Inputs may be the reference's own GaussianCloud/Camera objects, this package's
containers, or DeviceCloud objects (already resident; no per-call upload).

The ``kernel=`` argument is kept for signature compatibility and resolves through the raster
plugin registry, which has exactly one kernel ("cuda"); there is no CPU path.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import raster
from .cloud import concat_clouds
from .device import DeviceCloud, camera_array
from .errors import ContractViolation

TILE_SIZE = 16


@dataclass
class FrameRGBD:
    """color (H,W,3) in [0,1]; alpha (H,W) in [0,1]; depth (H,W) meters, far where empty."""

    color: np.ndarray
    alpha: np.ndarray
    depth: np.ndarray

    @property
    def shape(self):
        return self.alpha.shape


@dataclass
class RenderStats:
    n_input: int = 0
    n_culled_depth: int = 0
    n_culled_frame: int = 0
    n_degenerate: int = 0
    n_drawn: int = 0

    def add(self, values):
        for k, v in zip(("n_input", "n_culled_depth", "n_culled_frame", "n_degenerate", "n_drawn"), values):
            setattr(self, k, getattr(self, k) + int(v))
        return self


def _nonempty(c):
    return (c.n if isinstance(c, DeviceCloud) else np.asarray(c.positions).shape[0]) > 0


def render_frames(scene, cameras, background, layer=None, avatars=None, sim_times=None, tiled=True,
                  context=None, contrib=False, stats=True, avatar_active=None, stage_ms=None, work=None,
                  binning=-1, exact=False, out=None, wait=True, payload=False, serialize=False, views=True,
                  near_slice=-1):
    """One sn_render call over E cameras. Returns a dict of device tensors:
    color (E,H,W,3), alpha (E,H,W), depth (E,H,W) float32; stats (E,5) int64; optionally
    contrib_scene / contrib_layer (E,H,W) int32 and, with payload=True, the observation payload
    rgb8 (E,H,W,3) uint8 + depth16 (E,H,W) float16 written by the render's own epilogues
    (frame_io's uint8 rule). The context keeps the pass intermediates for the sn_get_* views.
    wait=False queues the render (sn_render_async) and returns at once: the frames are valid only
    after context.render_wait() for it returns False. serialize=True runs the avatar layer after
    the scene pass on the same stream (per-stage timers then add up to the render). views=False
    is the lean throughput path: the render keeps nothing for the harness views that need each
    splat's gaussian id or reference rectangle (pass_intermediates, tile_csr). near_slice: depth
    slicing of the scene pass (-1 auto: scenes of >= 500k gaussians without views; 0 off; 1 on) --
    the same frames, only each env's near depth slice sorted (see include/splatnav_b200.h)."""
    lib = N.load()
    ctx = context or N.default_context()
    dscene = DeviceCloud.wrap(scene)
    dev = dscene.device
    e = len(cameras)
    h, w = int(cameras[0].height), int(cameras[0].width)
    cams = camera_array(cameras, background)
    if out is None:  # caller-owned outputs (e.g. HostPipeline's ring) avoid per-call allocations
        out = {}
    shapes = {"color": ((e, h, w, 3), torch.float32), "alpha": ((e, h, w), torch.float32),
              "depth": ((e, h, w), torch.float32)}
    if payload:
        shapes.update({"rgb8": ((e, h, w, 3), torch.uint8), "depth16": ((e, h, w), torch.float16)})
    for k, (shp, dt) in shapes.items():
        t = out.get(k)
        same_dev = t is not None and t.device.type == dev.type and (t.device.index or 0) == (dev.index or 0)
        if t is None or tuple(t.shape) != shp or t.dtype != dt or not same_dev or not t.is_contiguous():
            out[k] = torch.empty(shp, dtype=dt, device=dev)
    opts = N.SnRenderOpts()
    opts.tiled = 1 if tiled else 0
    opts.binning = int(binning)
    opts.exact = 1 if exact else 0
    opts.serialize = 1 if serialize else 0
    opts.views = 1 if views else 0
    opts.near_slice = int(near_slice)
    if payload:
        opts.rgb8 = out["rgb8"].data_ptr()
        opts.depth16 = out["depth16"].data_ptr()
    if stats:
        out["stats"] = torch.zeros((e, 5), dtype=torch.int64, device=dev)
        opts.stats = out["stats"].data_ptr()
    if contrib:
        out["contrib_scene"] = torch.zeros((e, h, w), dtype=torch.int32, device=dev)
        out["contrib_layer"] = torch.zeros((e, h, w), dtype=torch.int32, device=dev)
        opts.contrib_scene = out["contrib_scene"].data_ptr()
        opts.contrib_layer = out["contrib_layer"].data_ptr()
    if stage_ms is not None:  # host float64 (2, 11): per-pass GPU ms per stage, accumulated
        assert stage_ms.dtype == np.float64 and stage_ms.size == 2 * len(N.STAGES) and stage_ms.flags.c_contiguous
        opts.stage_ms = stage_ms.ctypes.data
    if work is not None:  # host int64 (2, 6): visible, pairs, records gathered, rects scanned, contributions
        assert work.dtype == np.int64 and work.size == 12 and work.flags.c_contiguous
        opts.work = work.ctypes.data
    if avatar_active is not None:
        out["avatar_active"] = avatar_active.to(device=dev, dtype=torch.uint8).contiguous()
        opts.avatar_active = out["avatar_active"].data_ptr()
    dlayer = DeviceCloud.wrap(layer, dev) if layer is not None else None
    times = None
    if avatars is not None:
        times = np.ascontiguousarray(np.asarray(sim_times, dtype=np.float64).reshape(e))
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check((lib.sn_render if wait else lib.sn_render_async)(
        ctx.handle, ctypes.byref(dscene.struct()), ctypes.byref(dlayer.struct()) if dlayer is not None else None,
        ctypes.byref(avatars.struct()) if avatars is not None else None, cams,
        times.ctypes.data_as(ctypes.c_void_p) if times is not None else None, e, ctypes.byref(opts),
        out["color"].data_ptr(), out["alpha"].data_ptr(), out["depth"].data_ptr(), stream))
    out["_keep"] = (dscene, dlayer, cams)
    return out


def _to_frame(out, i=0):
    return FrameRGBD(color=out["color"][i].double().cpu().numpy(), alpha=out["alpha"][i].double().cpu().numpy(),
                     depth=out["depth"][i].double().cpu().numpy())


def _accumulate(stats, out):
    if stats is not None and "stats" in out:
        stats.add(out["stats"][0].cpu().tolist())


def rasterize(cloud, camera, background, stats=None, kernel=None):
    """renderer.py:135. background None = layer mode (alpha-normalized colour, black/0 where empty)."""
    raster.get_kernel(kernel)
    out = render_frames(cloud, [camera], background, tiled=True)
    _accumulate(stats, out)
    return _to_frame(out)


def rasterize_reference(cloud, camera, background, stats=None, kernel=None):
    """renderer.py:145: every pixel walks all projected splats in depth order, no tiling."""
    raster.get_kernel(kernel)
    out = render_frames(cloud, [camera], background, tiled=False)
    _accumulate(stats, out)
    return _to_frame(out)


def composite(front, back):
    """renderer.py:151-166, evaluated by the CUDA compositor on float64 frames."""
    if front.shape != back.shape:
        raise ContractViolation(f"frame shapes differ: {front.shape} vs {back.shape}")
    lib = N.load()
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(dev)
    fc, fa, fd, bc, ba, bd = (t(front.color), t(front.alpha), t(front.depth), t(back.color), t(back.alpha),
                              t(back.depth))
    oc, oa, od = torch.empty_like(bc), torch.empty_like(ba), torch.empty_like(bd)
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(lib.sn_composite(fa.numel(), fc.data_ptr(), fa.data_ptr(), fd.data_ptr(), bc.data_ptr(), ba.data_ptr(),
                             bd.data_ptr(), oc.data_ptr(), oa.data_ptr(), od.data_ptr(), stream))
    return FrameRGBD(color=oc.cpu().numpy(), alpha=oa.cpu().numpy(), depth=od.cpu().numpy())


def render_observation(scene_cloud, avatar_clouds, camera, background, stats=None, kernel=None):
    """renderer.py:169-177: scene pass plus one concatenated avatar layer, depth-composited."""
    raster.get_kernel(kernel)
    avatar_clouds = [c for c in avatar_clouds if _nonempty(c)]
    layer = None
    if avatar_clouds:
        layer = concat_clouds(avatar_clouds) if len(avatar_clouds) > 1 else avatar_clouds[0]
    out = render_frames(scene_cloud, [camera], background, layer=layer, tiled=True)
    _accumulate(stats, out)
    return _to_frame(out)


def tiles_for(width, height):
    return math.ceil(width / TILE_SIZE), math.ceil(height / TILE_SIZE)


def pass_intermediates(pass_id=0, env=0, context=None):
    """Harness view of the last render's pass: ids in depth order, tile CSR (depth ranks),
    projection arrays. Mirrors what project_cloud (projection.py:184) and _bin_tiles
    (renderer.py:80-101) compute internally."""
    lib = N.load()
    ctx = context or N.default_context()
    nv, npairs = ctypes.c_int64(), ctypes.c_int64()
    N.check(lib.sn_get_counts(ctx.handle, pass_id, env, ctypes.byref(nv), ctypes.byref(npairs)))
    m, p = nv.value, npairs.value
    ids = np.zeros(max(m, 1), dtype=np.int32)
    N.check(lib.sn_get_sorted_ids(ctx.handle, pass_id, env, ids.ctypes.data_as(ctypes.c_void_p), m))
    proj = {k: np.zeros((max(m, 1),) + s) for k, s in
            (("means2d", (2,)), ("conics", (3,)), ("depths", ()), ("colors", (3,)), ("alphas", ()))}
    N.check(lib.sn_get_projection(ctx.handle, pass_id, env, *[proj[k].ctypes.data_as(ctypes.c_void_p) for k in
                                                             ("means2d", "conics", "depths", "colors", "alphas")], m))
    res = {"ids": ids[:m], "n_pairs": p}
    res.update({k: v[:m] for k, v in proj.items()})
    return res


def tile_csr(n_tiles, pass_id=0, env=0, context=None):
    lib = N.load()
    ctx = context or N.default_context()
    nv, npairs = ctypes.c_int64(), ctypes.c_int64()
    N.check(lib.sn_get_counts(ctx.handle, pass_id, env, ctypes.byref(nv), ctypes.byref(npairs)))
    ts = np.zeros(n_tiles + 1, dtype=np.int64)
    ps = np.zeros(max(npairs.value, 1), dtype=np.int32)
    N.check(lib.sn_get_tile_csr(ctx.handle, pass_id, env, ts.ctypes.data_as(ctypes.c_void_p),
                                ps.ctypes.data_as(ctypes.c_void_p), npairs.value))
    return ts, ps[:npairs.value]


def device_tiles(n_tiles, pass_id=0, env=0, context=None):
    """The tile lists the last render's blend consumed for `env` (sn_get_device_tiles): tile_starts
    (T+1) int64 and per-tile depth ranks int32 -- the tight sub-lists of tile_csr's reference lists."""
    lib = N.load()
    ctx = context or N.default_context()
    ts = np.zeros(n_tiles + 1, dtype=np.int64)
    n = ctypes.c_int64()
    N.check(lib.sn_get_device_tiles(ctx.handle, pass_id, env, ts.ctypes.data_as(ctypes.c_void_p), None, 0,
                                    ctypes.byref(n)))
    ranks = np.zeros(max(n.value, 1), dtype=np.int32)
    N.check(lib.sn_get_device_tiles(ctx.handle, pass_id, env, ts.ctypes.data_as(ctypes.c_void_p),
                                    ranks.ctypes.data_as(ctypes.c_void_p), n.value, ctypes.byref(n)))
    return ts, ranks[:n.value]
