"""Throughput sweep over env counts (the shape of the
reference's Fig. 2): for each model and batch size on one B200,

* ``render`` -- the fused rendered env-step (distractor advance + render +
  composite in one launch, poses resident), device-timed with CUDA events;
* ``env_step`` -- the full on-device ``step()`` (physics substeps, auto-reset,
  fused render) with the conv-stub policy forward in the loop, the
  reference's benchmark protocol (bench.py:183-216), timed on the device.

Writes a CSV and a markdown table (default: gpurun_out/sweep.*).

    python tools/sweep.py [--batches 1 10 100 1000 16384] [--out gpurun_out/sweep]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00021_b200 import bench as B  # noqa: E402
from paper_2502_00021_b200 import env as E  # noqa: E402
from paper_2502_00021_b200.bench_support import Workload  # noqa: E402
from paper_2502_00021_b200.models import STANDIN_MODELS  # noqa: E402

MODELS = [("HalfCheetah", "cheetah_lite", "none"), ("Walker2d", "walker_lite", "video"),
          ("Ant", "ant_lite", "color"), ("Humanoid", "humanoid_lite", "video")]


def time_events(fn, iters):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for i in range(iters):
        fn(i)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / iters  # ms per step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, nargs="+", default=[1, 10, 100, 1000, 16384])
    ap.add_argument("--out", default="gpurun_out/sweep")
    a = ap.parse_args()
    pack_path = "/tmp/sweep_pack.pxvp"
    from paper_2502_00021_b200.bench_support import synthetic_pack
    from paper_2502_00021_b200.video_pack import save_video_pack

    save_video_pack(synthetic_pack(), pack_path)
    rows = []
    for name, env_model, mode in MODELS:
        for b in a.batches:
            # fused rendered env-step
            w = Workload(name, b, mode)
            poses = [w.poses(t).clone() for t in range(2)]
            for t in range(3):
                w.render(poses[t % 2], t)
            iters = max(5, min(200, 200000 // b))
            w.precompute_keys(range(3, 3 + iters))  # host Threefry out of the timed loop
            ms_r = time_events(lambda i: w.render(poses[i % 2], 3 + i), iters)
            # the same launches captured in a CUDA graph (20 per replay): the
            # device time without the Python launch loop
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(st):
                with torch.cuda.graph(gr, stream=st):
                    for i in range(20):
                        w.render(poses[i % 2], 3 + i, stream=st)
            torch.cuda.current_stream().wait_stream(st)
            gr.replay()
            ms_rg = time_events(lambda i: gr.replay(), max(3, iters // 20)) / 20
            del gr, w, poses
            # full env step + conv-stub policy (device-resident loop)
            cfg = E.EnvConfig(model=STANDIN_MODELS.get(env_model, env_model), batch=b,
                              distractor_mode=mode,
                              video_pack_path=pack_path if mode == "video" else None)
            env, state, obs = E.make_env(cfg)
            stub = B.ConvStub.create(84, 84, 3, env.n_joints, seed=0)
            box = {"state": state, "obs": obs}

            def one(i):
                act = B.conv_stub_forward(stub, box["obs"])
                box["state"], out = E.step(env, box["state"], act)
                box["obs"] = out.obs

            for i in range(3):
                one(i)
            iters_s = max(5, min(100, 50000 // b))
            ms_s = time_events(one, iters_s)
            # the same loop as one CUDA graph replay per step (env.StepGraph)
            g = E.StepGraph(env, box["state"], box["obs"],
                            lambda o: B.conv_stub_forward(stub, o))
            g.replay(3)
            iters_g = max(20, min(1000, 200000 // b))
            ms_g = time_events(lambda i: g.replay(1), iters_g)
            rows.append((name, mode, b, b / ms_r * 1e3, ms_r, b / ms_s * 1e3, ms_s,
                         b / ms_g * 1e3, ms_g, b / ms_rg * 1e3, ms_rg))
            print(f"{name:12s} {mode:6s} B={b:6d}  render {b / ms_r * 1e3:12.0f} env-steps/s "
                  f"({ms_r:.3f} ms; graphed {b / ms_rg * 1e3:.0f}, {ms_rg * 1e3:.1f} us)  env_step+policy {b / ms_s * 1e3:12.0f} ({ms_s:.3f} ms)  "
                  f"graphed {b / ms_g * 1e3:12.0f} ({ms_g:.3f} ms)", flush=True)
            del g
            del env, state, obs, box
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".csv", "w") as f:
        f.write("model,mode,envs,render_sps,render_ms,env_step_policy_sps,env_step_policy_ms,"
                "graphed_sps,graphed_ms,render_graphed_sps,render_graphed_ms\n")
        for r in rows:
            f.write(f"{r[0]},{r[1]},{r[2]},{r[3]:.6g},{r[4]:.6g},{r[5]:.6g},{r[6]:.6g},"
                    f"{r[7]:.6g},{r[8]:.6g},{r[9]:.6g},{r[10]:.6g}\n")
    with open(a.out + ".md", "w") as f:
        f.write("| model | distractors | envs | rendered env-steps/s (host loop) | ms | rendered, "
                "launches in a CUDA graph | ms | env step + conv policy, "
                "env-steps/s | ms | same, one CUDA graph per step | ms |\n"
                "|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]:,.0f} | {r[4]:.3f} | {r[9]:,.0f} | "
                    f"{r[10]:.4f} | {r[5]:,.0f} | "
                    f"{r[6]:.3f} | {r[7]:,.0f} | {r[8]:.3f} |\n")


if __name__ == "__main__":
    main()
