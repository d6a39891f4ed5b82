#!/usr/bin/env python
"""Rendered env-steps/sec on B200 (BASELINE.json metric), one JSON line.

Workload (BASELINE.json north_star target / configs[3]): Humanoid stand-in
(humanoid_lite, 13 links, 1248 triangles) with video distractors, 4096 envs
per GPU, 84x84 RGB, the reference's synthetic video pack resident in HBM.

A "step" = one rendered env-step for every env: given the pose batch of
step t (resident in HBM), the fused kernel advances the distractors
(ping-pong cursors), rasterizes, composites the video background and writes
the uint8 observation to HBM -- ONE kernel launch (pxr_render_step).

  value  device-timed (CUDA events on the launching stream, max over ranks)
         env-steps/s of the whole job, inputs already in HBM;
  e2e    the same through the C ABI with HOST buffers: pinned-host poses
         H2D + fused step + obs D2H to pinned host, every step, 2 streams;
  --impl reference   the reference's CPU path (the oracle port of
         render_robot_batch + advance_distractors + apply_video, oracle/)
         on all host cores, same workload, same metric.

Multi-GPU: torchrun, one process per GPU; rank r renders envs
[r*B, (r+1)*B) (env_offset = r*B, logical_batch = world*B) -- no collective
on the hot path; NCCL only for the max-time reduce and a final stats gather.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "rendered env-steps/sec vs #envs at 1/2/4/8 B200; % HBM roofline"
UNIT = "env-steps/s"
DEFAULT_MODEL = "Humanoid"
DEFAULT_ENVS = 4096
DEFAULT_MODE = "video"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default=DEFAULT_MODEL)
    ap.add_argument("--envs", type=int, default=DEFAULT_ENVS, help="envs per GPU")
    ap.add_argument("--mode", default=DEFAULT_MODE, choices=["none", "color", "video"])
    ap.add_argument("--grayscale", action="store_true")
    ap.add_argument("--pack-videos", type=int, default=4,
                    help="videos in the synthetic pack (60 frames of 64x64 each); the "
                         "reference's shipped pack has 4 (2.95 MB, L2-resident); >= 700 "
                         "makes it > 4x L2 so every frame fetch reads HBM (SURVEY 8(d))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


DTYPE = "f64/f32 raster, u8 RGB out"


def workload_config(args, spec, n_links, n_tris, world):
    """The `config` object of both arms (identical for the same args)."""
    B = args.envs
    return {
        "workload": f"{args.model} ({spec.name}, {n_links} links, {n_tris} tris), {B} envs/GPU, "
                    f"{args.mode} distractors, 84x84 {'gray' if args.grayscale else 'RGB'}",
        "model": spec.name, "envs_per_gpu": B, "global_envs": world * B,
        "mode": args.mode, "resolution": [84, 84], "pack_videos": args.pack_videos,
        "parallelism": f"env-sharded x{world} (no hot-path collective)",
    }


def share_device() -> bool:
    """Test hook (tests/test_bench_ranks.py): every rank on cuda:0 with the
    gloo backend, so the multi-rank path runs on a 1-GPU box. The ranks
    never wait on each other inside a kernel (no hot-path collective)."""
    return os.environ.get("PXR_BENCH_SHARE_DEVICE", "") == "1"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def read_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_entry(workload_tag):
    """The committed ncu capture summary of a workload (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get("workloads", {}).get(workload_tag)
    except Exception:
        return None


def ncu_traffic(workload_tag):
    """Per-launch DRAM bytes of the fused kernel from the committed ncu
    capture summary (profiles/ncu_summary.json), if it matches."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get("workloads", {}).get(workload_tag)
        if e:
            return float(e["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the GPU is busy."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- ours


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as tdist

    from paper_2502_00021_b200.bench_support import Workload
    from paper_2502_00021_b200.shards import aggregate, gather_stats, shard_envs

    gpu = 0 if share_device() else local
    if world > 1:
        if share_device():
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    B = args.envs
    shard = shard_envs(rank, world, B)  # envs [r*B, (r+1)*B) of world*B, no hot-path collective
    from paper_2502_00021_b200.bench_support import synthetic_pack

    pack = synthetic_pack(videos=args.pack_videos) if args.mode == "video" else None
    w = Workload(args.model, B, args.mode, seed=0, env_offset=shard.env_offset,
                 logical_batch=shard.logical_batch, grayscale=args.grayscale, pack=pack,
                 device=dev)
    stream = torch.cuda.Stream(device=dev)
    n_pose_sets = 8
    obs_bytes = B * w.obs_bytes_per_env()
    l2 = 126 * 2**20
    n_out = max(2, -(-3 * l2 // obs_bytes))  # obs ring footprint > 3x L2
    with torch.cuda.stream(stream):
        pose_sets = [w.poses(t, out=torch.empty_like(w.poses_buf), stream=stream).clone()
                     for t in range(n_pose_sets)]
        outs = [torch.empty_like(w.obs) for _ in range(n_out)]
    torch.cuda.synchronize(dev)

    def one(t):
        w.render(pose_sets[t % n_pose_sets], t, out_obs=outs[t % n_out], stream=stream)

    # warm-up (untimed), then a short soak so clocks settle
    for t in range(max(3, args.warmup)):
        one(t)
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(gpu)
    sampler.start()
    soak_end = time.time() + 1.0
    t_ = 0
    while time.time() < soak_end:
        for _ in range(20):
            one(t_)
            t_ += 1
        torch.cuda.synchronize(dev)

    # ---- timed region: K fused launches ----------------------------------
    w.precompute_keys(range(args.warmup, args.warmup + args.steps))  # host Threefry, untimed
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        one(args.warmup + k)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    ms = ev0.elapsed_time(ev1)
    # keep the GPU busy briefly after the window so the sampler brackets it
    for k in range(20):
        one(k)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()

    # per-launch duration of the dominant (only) kernel inside the region
    ms_max = max_over_ranks(ms, dev)
    total_steps = world * B * args.steps
    value = total_steps / (ms_max / 1e3)
    per_launch_s = (ms / 1e3) / args.steps

    # ---- e2e through the C ABI with host buffers --------------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, w, dev, world, rank)

    # ---- determinism + shard-slice check, per-rank digest (untimed) --------
    mism, digest = verify_rank(args, w, shard, pack, dev)

    # ---- final stats gather (NCCL): the only collective --------------------
    stats = gather_stats({"env_steps": B * args.steps, "ms": ms, "mismatches": mism,
                          "digest_lo": digest & 0xFFFFFFFF, "digest_hi": digest >> 32})
    agg = aggregate(stats)
    if world > 1:
        tdist.destroy_process_group()

    if rank != 0:
        return None
    peak, peak_src = read_peaks()
    bytes_per_env = w.obs_bytes_per_env() + 24 * w.n_links + w.state_bytes_per_env()
    pack_bytes = 0 if w.pack is None else int(w.pack.flat_frames()[0].nbytes)
    large_pack = pack_bytes > 4 * 126 * 2**20
    if large_pack:  # the env's video frame is an HBM read (count it)
        bytes_per_env += w.pack.height * w.pack.width * 3
    achieved = bytes_per_env * B / per_launch_s / 1e9
    tag = (f"{args.model}-{args.mode}-{B}{'-gray' if args.grayscale else ''}"
           f"{f'-pack{args.pack_videos}' if args.pack_videos != 4 else ''}")
    traffic = ncu_traffic(tag)
    # what does bound it: warp instructions per env (ncu capture of this
    # workload) x env-steps/s (this run) / (SMs x 4 schedulers x SM clock)
    issue = None
    ent = ncu_entry(tag)
    if ent and ent.get("warp_instructions_per_env") and clocks and clocks.get("sm_mhz"):
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ipe = float(ent["warp_instructions_per_env"])
        rate = ipe * (B / per_launch_s)
        peak_i = sms * 4 * clocks["sm_mhz"] * 1e6
        issue = {"bound": "issue", "warp_instructions_per_env": ipe,
                 "achieved_warp_instr_per_s": rate, "peak_warp_instr_per_s": peak_i,
                 "frac": rate / peak_i,
                 "note": "instructions per env from the committed ncu capture; the rate from "
                         "this run's device time and sampled SM clock (4 issue slots per SM "
                         "per cycle)"}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic: on-device pose source (reference reset keys + joint oscillation, "
                "f64 FK); " + (f"synthetic video pack ({args.pack_videos}x60x64x64, "
                               f"{pack_bytes / 2**20:.0f} MiB > 4x L2: frame fetches from HBM, "
                               "counted in the roofline bytes)" if large_pack else
                               "reference synthetic video pack (seed 2024, 4x60x64x64) in HBM"),
        "config": workload_config(args, w.spec, w.n_links, w.geom.triangle_count, world),
        "l2_policy": f"obs ring of {n_out} buffers ({n_out * obs_bytes / 2**20:.0f} MiB > L2) "
                     f"+ {n_pose_sets} resident pose sets",
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "bytes_per_env_step": bytes_per_env,
            "peak_source": peak_src,
            "kernel": "render_step_kernel",
        },
        "issue": issue,
        "gpu_launches": args.steps,
        "stats_gather": {"ranks": len(stats), "env_steps": agg["env_steps"],
                         "ms_max": agg["ms_max"], "mismatches": agg["mismatches"],
                         "digests": [f"{(int(r['digest_hi']) << 32) | int(r['digest_lo']):016x}"
                                     for r in stats],
                         "check": "per rank: the same step rendered twice from one saved "
                                  "distractor state, and a 64-env slice rendered as its own "
                                  "batch (env_offset / logical_batch impersonation), compared "
                                  "byte for byte with the full batch; digest = first 64 bits "
                                  "of SHA-256 of the rank's obs"},
        "e2e": e2e,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args, seconds=args.cpu_seconds)
    return line


def max_over_ranks(x: float, dev) -> float:
    """MAX over ranks of a per-rank device time (NCCL on the device, or
    gloo on the host under the shared-device test hook)."""
    import torch
    import torch.distributed as tdist

    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return float(x)
    on = dev if tdist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=on)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def verify_rank(args, w, shard, pack, dev):
    """Untimed correctness check of this rank's shard (no oracle): one step
    rendered twice from the same saved distractor state must agree byte for
    byte (catches races), and the first min(64, B) envs rendered as their
    own batch -- the slice impersonation of SURVEY 8(e): keys and poses come
    from the global env index -- must equal those rows of the full batch.
    Returns (mismatching bytes, first 64 bits of SHA-256 of the obs)."""
    import hashlib

    import torch

    from paper_2502_00021_b200.bench_support import Workload

    T = 7919  # any step index
    poses = w.poses(T).clone()
    d0 = w.dist.copy()
    a, _ = w.render(poses, T, out_obs=torch.empty_like(w.obs))
    fields = ("color_bias", "video_index", "frame_cursor", "direction", "frame_count")
    for f in fields:  # back to the saved state, same step again
        getattr(w.dist, f).copy_(getattr(d0, f))
    b, _ = w.render(poses, T, out_obs=torch.empty_like(w.obs))
    m = min(64, w.batch)
    ws = Workload(args.model, m, args.mode, seed=0, env_offset=shard.env_offset,
                  logical_batch=shard.logical_batch, grayscale=args.grayscale, pack=pack,
                  device=dev)
    for f in fields:
        src = getattr(d0, f)
        if src.numel():
            getattr(ws.dist, f).copy_(src[:m])
    c, _ = ws.render(ws.poses(T).clone(), T)
    mism = int((a != b).sum().item()) + int((a[:m] != c).sum().item())
    digest = int(hashlib.sha256(a.cpu().numpy().tobytes()).hexdigest()[:16], 16)
    return mism, digest


def run_e2e(args, w, dev, world, rank):
    """Host poses (pinned) -> H2D -> fused step -> D2H obs (pinned), every
    step, double-buffered over two streams; device-timed with events."""
    import torch
    import torch.distributed as tdist

    B = w.batch
    host_poses = [w.poses(t).cpu().pin_memory() for t in range(2)]
    host_obs = [torch.empty(w.obs.shape, dtype=torch.uint8).pin_memory() for _ in range(2)]
    dev_poses = [torch.empty_like(w.poses_buf) for _ in range(2)]
    dev_obs = [torch.empty_like(w.obs) for _ in range(2)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    torch.cuda.synchronize(dev)

    def one(t):
        i = t % 2
        s = streams[i]
        with torch.cuda.stream(s):
            dev_poses[i].copy_(host_poses[i], non_blocking=True)
            w.render(dev_poses[i], t, out_obs=dev_obs[i], stream=s)
            host_obs[i].copy_(dev_obs[i], non_blocking=True)

    for t in range(max(3, args.warmup)):
        one(t)
    w.precompute_keys(range(args.steps))  # host Threefry, untimed
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    start = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    start.record(streams[0])
    streams[1].wait_event(start)
    K = args.steps
    for k in range(K):
        one(k)
    for i in range(2):
        ends[i].record(streams[i])
    torch.cuda.synchronize(dev)
    ms = max(start.elapsed_time(e) for e in ends)
    ms = max_over_ranks(ms, dev)
    return {
        "value": world * B * K / (ms / 1e3),
        "unit": UNIT,
        "h2d_bytes_per_step": int(host_poses[0].numel() * 8),
        "d2h_bytes_per_step": int(host_obs[0].numel()),
        "gpu_launches": K,
        "path": "pinned host poses -> pxr_render_step (C ABI via ctypes) -> pinned host obs, "
                "2 streams",
    }


# ---------------------------------------------------------------- CPU legs


class HostWorkload:
    """The same configuration as bench_support.Workload, built on the host
    only (numpy + the C oracle; no torch, no libpxr): geometry and model
    from the package's host-side tables (tessellation pinned by
    tests/golden/geometry.json), poses from the host restatement of the
    pose source (oracle.pose_source, the reference's reset keys + the same
    joint oscillation + FK), distractor state from oracle.init_distractors
    (distractor.py:82-113), the reference's synthetic video pack."""

    def __init__(self, O, model, batch, mode, seed=0, env_offset=0, logical_batch=None,
                 grayscale=False, pack_videos=4, width=84, height=84):
        import numpy as np

        from paper_2502_00021_b200.bench_support import MODEL_ALIASES, synthetic_pack
        from paper_2502_00021_b200.models import model_kinematics, resolve_model
        from paper_2502_00021_b200.render import RobotGeometry

        self.O = O
        self.spec = resolve_model(MODEL_ALIASES.get(model, model))
        self.parent, self.anchor, length, radius = model_kinematics(self.spec)
        self.geom = RobotGeometry(length, radius)
        self.batch, self.mode, self.grayscale = int(batch), mode, bool(grayscale)
        self.env_offset = int(env_offset)
        self.logical_batch = int(logical_batch if logical_batch is not None else batch)
        self.width, self.height = width, height
        self.floor_in_background = mode == "video"  # env.py:81-85
        self.master = O.key_from_seed(seed)
        self.reset_key = O.fold_in(self.master, 0x5EED)
        self.frames = self.starts = self.counts = None
        if mode == "video":
            pack = synthetic_pack(videos=pack_videos)
            self.frames, self.starts = pack.flat_frames()
            self.counts = np.asarray(pack.frame_counts, dtype=np.int64)
        self.state = O.init_distractors(mode, self.counts, O.fold_in(self.master, 0xD157),
                                        self.batch, env_offset=self.env_offset)

    @property
    def n_links(self):
        return self.spec.n_links

    def poses(self, t):
        return self.O.pose_source(self.spec.rest(), self.parent, self.anchor, self.reset_key,
                                  self.env_offset, t, self.batch)

    def step(self, poses, t, threads):
        """One rendered env-step of every env on the CPU: advance_distractors
        (distractor.py:116-137), render_robot_batch (render.py:594-623),
        apply_color/apply_video (distractor.py:184-214), grayscale
        (env.py:168-173) -- the reference's per-step path."""
        O = self.O
        key_t = O.fold_in(self.master, t)
        self.state = O.advance_state(self.state, self.mode, key_t, self.env_offset,
                                     self.logical_batch, frame_counts=self.counts)
        px, dp = O.render_robot_batch(self.geom, poses, self.width, self.height,
                                      self.floor_in_background, threads=threads)
        if self.mode == "color":
            O.apply_color_inplace(px, self.state["color_bias"], threads=threads)
        elif self.mode == "video":
            O.apply_video_inplace(px, dp, self.frames,
                                  self.starts[self.state["video_index"]]
                                  + self.state["frame_cursor"], threads=threads)
        return O.grayscale(px) if self.grayscale else px


def _oracle():
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O

    O.build()
    return O


def cpu_baseline(args, seconds=10.0):
    """The oracle port on all host cores, a bounded sample (~`seconds`) of
    the same workload: full batches of args.envs envs per step."""
    O = _oracle()
    threads = O.host_threads()
    hw = HostWorkload(O, args.model, args.envs, args.mode, seed=0, grayscale=args.grayscale,
                      pack_videos=args.pack_videos)
    pose_sets = [hw.poses(t) for t in range(4)]
    hw.step(pose_sets[0], 0, threads)  # warm
    n = 0
    t0 = time.perf_counter()
    while True:
        hw.step(pose_sets[n % 4], n + 1, threads)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 10000:
            break
    return {
        "value": n * hw.batch / el,
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": f"{n} steps x {hw.batch} envs of the same workload ({el:.1f} s): host poses, "
                  "advance_distractors + render_robot_batch + apply_* on the C oracle "
                  "(oracle/render_oracle.c), OpenMP over envs",
        "cpu": _cpu_model(),
    }


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, world, rank, local):
    """--impl reference: the reference's CPU path (the C oracle port of
    render_robot_batch + advance_distractors + apply_*; the reference is
    Python + numba, nothing to compile into oracle/_ref) on all host cores,
    rendering every env of the job each step (world x envs), inputs built
    on the host. Rank 0 only under torchrun; no torch, no libpxr."""
    if rank != 0:
        return None
    O = _oracle()
    threads = O.host_threads()
    B = args.envs * world
    hw = HostWorkload(O, args.model, B, args.mode, seed=0, grayscale=args.grayscale,
                      pack_videos=args.pack_videos)
    pose_sets = [hw.poses(t) for t in range(4)]  # host-resident inputs, not timed
    for t in range(max(1, args.warmup)):
        hw.step(pose_sets[t % 4], t, threads)
    t0 = time.perf_counter()
    for k in range(args.steps):
        hw.step(pose_sets[k % 4], args.warmup + k, threads)
    el = time.perf_counter() - t0
    value = args.steps * B / el
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic: host pose source (reference reset keys + joint oscillation, f64 FK, "
                "numpy) and the reference synthetic video pack",
        "config": workload_config(args, hw.spec, hw.n_links, hw.geom.triangle_count, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"every step renders all {B} envs ({args.steps} timed steps "
                                   f"after {max(1, args.warmup)} warm-up steps)",
                         "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def self_launch(args) -> int:
    """`--gpus N` without a torchrun environment: re-exec this script under
    torch.distributed.run with N ranks (one process per GPU, rendezvous on
    127.0.0.1); rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        args.gpus = world
    if args.impl == "reference":
        line = run_reference(args, world, rank, local)
    else:
        line = run_ours(args, world, rank, local)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
