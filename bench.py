"""Benchmark: RGB-D 640x480 frames/sec of the splat-observation hot path (BASELINE.json metric).

Default workload = BASELINE config 2: a 1M-gaussian room scene (8 x 8 x 3 m) plus 4 skinned
avatars (50k gaussians, 24 joints each), 64 environments per GPU, one 640x480 90 deg camera per env
at 1.25 m, near 0.1 / far 100 (the reference agent-camera defaults, scene.py:23-24). A step =
one batch: per-env avatar pose sampling + fused LBS, scene pass and avatar-layer pass
(projection, SH, depth sort, tile binning, blend, composite) for all envs. Every step uses a fresh
set of camera poses and sim times (pre-generated), so nothing is cached across steps; the scene
(236 MB) and per-step buffers exceed the 126 MB L2.

Multi-GPU (torchrun): each rank renders its own 64 envs against a replica of the scene (weak
scaling, no data-path collective); timing is the max over ranks of CUDA-event time.

--impl reference: the reference's algorithm on the host CPU (oracle/, the C restatement pinned to
the reference) on all host threads, on a bounded sample of envs per step; rank 0 only.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "RGB-D frames/sec (640×480) vs gaussian count & avatar count at 1/2/4/8 B200"
STAGES = ("pose", "count", "scan", "emit", "depth_sort", "permute", "pair_scan", "bin_count", "bin_scatter", "ranges",
          "blend", "composite")



def workload_config(args, parallelism):
    """The `config` object both arms print (the GPU arm and `--impl reference` share it)."""
    return {"workload": f"config2: {args.gaussians} scene gaussians + {args.avatars}x50k skinned avatars, "
                        f"{args.envs} envs/GPU, {args.width}x{args.height}, near {args.near}",
            "envs_per_gpu": args.envs, "n_gaussians": args.gaussians, "n_avatars": args.avatars,
            "l2": "inputs larger than L2 (236 MB scene + per-step buffers), fresh cameras every step",
            "parallelism": parallelism}

def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--envs", type=int, default=64, help="environments per GPU")
    p.add_argument("--gaussians", type=int, default=1_000_000)
    p.add_argument("--avatars", type=int, default=4)
    p.add_argument("--near", type=float, default=0.1)
    p.add_argument("--width", type=int, default=640)
    p.add_argument("--height", type=int, default=480)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-envs", type=int, default=0, help="env sample for the CPU baseline (0 = auto)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(args, world, rank, n_sets):
    """Scene + avatars (identical on every rank) and n_sets per-step (cameras, times) for this rank."""
    from paper_2604_12626_b200 import synthetic as S
    box = S.room_box(args.gaussians)
    scene = S.make_scene(args.gaussians, box[0], box[1], seed=args.seed)
    bundles = [S.make_avatar(50_000, seed=args.seed + 100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2])
               for i in range(args.avatars)]
    sets = []
    for s in range(n_sets):
        cams = S.room_cameras(args.envs, box, seed=10_000 + (s * world + rank) * 7 + args.seed, width=args.width,
                              height=args.height, near=args.near)
        rng = np.random.default_rng(20_000 + s * world + rank)
        times = rng.uniform(0.0, 2.0, size=args.envs)
        sets.append((cams, times))
    return scene, bundles, box, sets


def start_offsets(n):
    return [0.37 * i for i in range(n)]


class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms during the timed region (NVML; falls back
    to an nvidia-smi loop when NVML is unavailable)."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples, self.max_mhz, self.reasons = [], 0.0, set()
        self._stop = threading.Event()
        self._thread = None
        self._smi = None

    def _run_nvml(self, nv, h):
        names = {"hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                 "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                 "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                 "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._stop.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                bits = get_reasons(h)
                for k, v in names.items():
                    if bits & v:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            idx = self.gpu
            vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
            if vis and all(v.isdigit() for v in vis) and self.gpu < len(vis):
                idx = int(vis[self.gpu])  # NVML numbers physical devices
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._thread = threading.Thread(target=self._run_nvml, args=(nv, h), daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return None
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def algorithmic_bytes(stage, pass_id, n_gauss, n_avatar_gauss, work, n_pix_total, n_steps):
    """Minimum HBM bytes of one step's launches of `stage` (SURVEY.md 8(d) per-unit figures)."""
    vis, pairs, loads = work[pass_id][0] / n_steps, work[pass_id][1] / n_steps, work[pass_id][2] / n_steps
    scans = work[pass_id][3] / n_steps
    n = n_gauss if pass_id == 0 else n_avatar_gauss
    per_gauss_in = 48 if pass_id == 0 else 134  # packed params (+ skin influences for avatars)
    if stage == "count":
        return n * (per_gauss_in + 8)
    if stage == "emit":
        return n * (8 + per_gauss_in + 192) + vis * 88
    if stage == "depth_sort":
        return vis * 24
    if stage == "permute":
        return vis * 160
    if stage == "pair_scan":
        return vis * 12
    if stage == "bin_count":  # counting binner: read rects, write per-chunk tile counts (small)
        return vis * 8
    if stage == "bin_scatter":  # read rects, write one u32 per pair
        return vis * 8 + pairs * 4
    if stage == "ranges":
        return pairs * 4
    if stage == "blend":  # BlendGeo records gathered (64 B + 4 B index) + rectangles streamed + pixels out
        # scene: RGB + alpha + depth (20 B) + the depth error bound (4 B); layer: its own frame (28 B)
        return loads * 68 + scans * 8 + n_pix_total * (24 if pass_id == 0 else 28)
    return 0.0


def measured_traffic(kernel_stage):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by scripts/ncu_traffic.py from the .ncu-rep)."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel_stage)
    except (OSError, ValueError):
        return None


def cpu_baseline(args, scene, bundles, sets, n_envs_sample):
    """The reference algorithm (C oracle, pinned to the reference) on all host threads."""
    from oracle import oracle as O
    cams, times = sets[0]
    cams = cams[:n_envs_sample]
    times = times[:n_envs_sample]
    threads = os.cpu_count() or 1
    offs = start_offsets(len(bundles))
    t0 = time.perf_counter()
    per_env = []
    for e in range(len(cams)):  # AvatarRuntime.deformed_cloud per env and avatar (tasks.py:501)
        clouds = []
        for a, b in enumerate(bundles):
            t = offs[a] + float(times[e])
            t = math.fmod(t, b.trajectory.duration)
            q, tr = O.sample_pose(b.trajectory.quats, b.trajectory.trans, b.trajectory.fps, t)
            pos, rot = O.lbs_deform(b.canonical.positions, b.canonical.rotations, b.lbs_weights, b.inv_bind, q, tr)
            c = b.canonical
            clouds.append(type(c)(pos, c.sh_coeffs, c.opacities, c.log_scales, rot))
        per_env.append(O.concat_clouds(clouds) if clouds else None)
    O.render_batch(scene, per_env if bundles else None, cams, np.ones(3), threads=threads)
    dt = time.perf_counter() - t0
    return {"value": len(cams) / dt, "unit": "frames/s", "cores": threads, "kind": "port",
            "sample": f"{len(cams)} envs of the same workload (scene {args.gaussians} gaussians, {len(bundles)} "
                      f"avatars, {args.width}x{args.height}), LBS + render_observation per env, {dt:.1f} s wall"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_sample = args.cpu_envs or max(2, min(args.envs, threads))
    scene, bundles, box, sets = workload(args, 1, 0, 1)
    for _ in range(args.warmup):
        cpu_baseline(args, scene, bundles, sets, min(n_sample, 2))
    t0 = time.perf_counter()
    frames = 0
    for _ in range(args.steps):
        r = cpu_baseline(args, scene, bundles, sets, n_sample)
        frames += n_sample
    dt = time.perf_counter() - t0
    value = frames / dt
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config 2 distributions, seeded)",
        "impl": "reference",
        "config": dict(workload_config(args, f"host threads x{threads}"), sample_envs_per_step=n_sample),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200.batch import BatchRenderer

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_sets = args.warmup + args.steps
    scene, bundles, box, sets = workload(args, world, rank, n_sets)
    br = BatchRenderer(scene, bundles, start_offsets=start_offsets(len(bundles)), background=(1.0, 1.0, 1.0))
    stage_ms = np.zeros(2 * len(STAGES))
    work = np.zeros(12, dtype=np.int64)

    from paper_2604_12626_b200.renderer import render_frames
    shapes = {"color": (args.envs, args.height, args.width, 3), "alpha": (args.envs, args.height, args.width),
              "depth": (args.envs, args.height, args.width)}
    frames_out = [{k: torch.empty(v, dtype=torch.float32, device="cuda") for k, v in shapes.items()} for _ in range(2)]

    def step(i, instrumented=False, wait=True):
        cams, times = sets[i]
        opts = dict(avatars=br.avatars, sim_times=times, context=br.context, stats=False, wait=wait,
                    out=dict(frames_out[i % 2]))
        if instrumented:
            opts["stage_ms"] = stage_ms
            opts["work"] = work
        return render_frames(br.scene, cams, br.background, **opts)

    def retire(pending):
        """Check the oldest queued render; on a workspace-growth retry redo it and every later
        queued render synchronously (their frames were computed with the old capacities)."""
        i = pending.pop(0)
        if br.context.render_wait():
            redo = [i] + pending
            for _ in pending:
                br.context.render_wait()
            pending.clear()
            for j in redo:
                step(j)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = br.context.kernel_launches()
    retries_t0 = br.context.render_retries()
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        ev0.record()
        # pipelined through the public API: step i + 1 is queued (sn_render_async) before the host
        # waits for and checks step i (sn_render_wait), so no host round trip idles the GPU
        pending = []
        for i in range(args.steps):
            step(args.warmup + i, wait=False)
            pending.append(args.warmup + i)
            if len(pending) > 1:
                retire(pending)
        while pending:
            retire(pending)
        ev1.record()
        torch.cuda.synchronize()
    launches = br.context.kernel_launches() - launches0
    retries_timed = br.context.render_retries() - retries_t0
    # per-stage CUDA-event timers and work counters from a separate, untimed pass over the same
    # steps (the timers' events and their resolution stay out of the timed region)
    for i in range(args.steps):
        step(args.warmup + i, instrumented=True)
    br.context.sync_stats()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    frames = args.envs * world * args.steps
    value = frames / (ms_max / 1e3)

    # end to end through the public API with host buffers: camera/time structs go host->device,
    # frames come back to pinned host memory every step
    e2e = None
    if not args.no_e2e:
        from paper_2604_12626_b200.batch import HostPipeline
        pipe = HostPipeline(br, args.envs, args.height, args.width)
        retries0 = br.context.render_retries()
        for i in range(max(args.warmup, 3)):  # the pipeline's buffers and allocator reach steady state
            pipe.submit(sets[i][0], sets[i][1])
        pipe.wait()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            cams, times = sets[args.warmup + i]
            pipe.submit(cams, times)  # camera/time structs host->device inside, frames device->host
        pipe.wait()  # every frame of every step is in pinned host memory
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e_retries = br.context.render_retries() - retries0
        te = torch.tensor([ems], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h, w = args.height, args.width
        e2e = {"value": frames / (float(te.item()) / 1e3), "unit": "frames/s", "render_retries": e2e_retries,
               "h2d_bytes_per_step": args.envs * (192 + 8), "d2h_bytes_per_step": args.envs * h * w * (12 + 4 + 4)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_kind = measured_peaks()
    stage = stage_ms.reshape(2, len(STAGES))
    w2 = work.reshape(2, 6)
    n_pix = args.envs * args.width * args.height
    n_av = sum(b.canonical.n for b in bundles)
    per_stage = {}
    for p, name in ((0, "scene"), (1, "layer")):
        for k, sname in enumerate(STAGES):
            if stage[p, k] > 0:
                per_stage[f"{name}.{sname}"] = stage[p, k] / args.steps
    # the layer pass's preprocessing runs on a side stream under the scene blend, so its stage
    # times are overlapped wall times; the dominant kernel is chosen among serial stages
    serial = {k: v for k, v in per_stage.items() if k.startswith("scene.") or k == "layer.composite"}
    dom = max(serial, key=serial.get)
    pname, sname = dom.split(".")
    pid = 0 if pname == "scene" else 1
    alg = algorithmic_bytes(sname, pid, args.gaussians, n_av, w2, n_pix, args.steps)
    achieved = alg / (per_stage[dom] / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                "alg_bytes_per_step": alg, "ms_per_step": per_stage[dom],
                "share_of_step": per_stage[dom] / (ms_max / args.steps)}
    traffic = measured_traffic(dom)
    if traffic is not None:
        roofline["traffic"] = traffic["dram_bytes_per_launch"] * traffic["launches_per_step"]
        roofline["traffic_source"] = traffic["source"]
    if sname == "blend":
        # The blend is not HBM-bound (records and rectangles are L2 hits, DRAM traffic is the
        # frames): it is issue-bound on its float32 contribution chain. FP32-pipe lane operations
        # per contribution, counted from the SASS of blend_kernel<0,0> (an FFMA2 is two): the two
        # axis rows (2 FFMA2) and h (2 FFMA), alpha error (1 FFMA), alpha (FMUL, FMNMX; the EX2 is
        # on the MUFU pipe), weight (FMUL), transmittance (FFMA), colour and depth sums (2 FFMA2),
        # A (FADD), its error bound (3 FFMA), z bound (FMNMX), cutoff test (FADD).
        per_contrib = 4 + 2 + 1 + 2 + 1 + 1 + 4 + 1 + 3 + 1 + 1
        contribs = w2[pid, 4] / args.steps
        clk = (clocks.summary() or {}).get("sm_mhz") or 1965.0
        peak_t = 148 * 128 * clk * 1e6 / 1e12  # FP32 lane-instructions per second (1 FFMA = 1)
        achieved_t = contribs * per_contrib / (per_stage[dom] / 1e3) / 1e12
        if traffic is not None and traffic.get("warp_inst_per_launch"):
            # the bound that actually binds: instruction issue (4 schedulers per SM, 1 warp
            # instruction per cycle each); instructions per launch from the committed ncu capture
            # of the same command, divided by this run's live blend time
            inst = traffic["warp_inst_per_launch"]
            peak_i = 148 * 4 * clk * 1e6 / 1e9
            ach_i = inst / (per_stage[dom] / 1e3) / 1e9
            roofline["issue"] = {"warp_inst_per_launch": inst, "achieved_ginst_per_s": ach_i,
                                 "peak_ginst_per_s": peak_i,
                                 "peak_kind": f"148 SMs x 4 schedulers x {clk:.0f} MHz (measured SM clock)",
                                 "frac": ach_i / peak_i, "source": traffic["source"]}
        roofline["compute"] = {"pipe": "fp32", "contributions_per_step": int(contribs),
                               "fp32_inst_per_contribution": per_contrib,
                               "achieved_tinst_per_s": achieved_t, "peak_tinst_per_s": peak_t,
                               "peak_kind": f"148 SMs x 128 FP32 lanes x {clk:.0f} MHz (measured SM clock)",
                               "frac": achieved_t / peak_t}
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 geometry + exact decisions (f32 blend chain with error bounds, f64 fixups)", "data": "synthetic (seeded, BASELINE distributions)",
        "config": workload_config(args, f"env-sharded x{world}"),
        "gpu_launches": None, "roofline": roofline, "e2e": e2e,
        "stages_ms_per_step": {k: round(v, 4) for k, v in per_stage.items()},
        "work_per_step": {"scene_visible": int(w2[0, 0] / args.steps),
                          "scene_records_loaded": int(w2[0, 2] / args.steps),
                          "scene_rects_scanned": int(w2[0, 3] / args.steps),
                          "scene_contributions": int(w2[0, 4] / args.steps),
                          "layer_visible": int(w2[1, 0] / args.steps), "layer_pairs": int(w2[1, 1] / args.steps),
                          "layer_records_loaded": int(w2[1, 2] / args.steps),
                          "layer_rects_scanned": int(w2[1, 3] / args.steps),
                          "layer_contributions": int(w2[1, 4] / args.steps),
                          "scene_fixup_pixels": int(w2[0, 5] / args.steps),
                          "layer_fixup_pixels": int(w2[1, 5] / args.steps)},
        "clocks": clocks.summary(),
    }
    line["gpu_launches"] = launches
    line["render_retries"] = retries_timed  # renders re-run to grow capacity-sized buffers
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        line["cpu_baseline"] = cpu_baseline(args, scene, bundles, sets, args.cpu_envs or max(2, min(args.envs, threads)))
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
