"""Device time split of one full env step at a given batch: conv-stub policy
forward, physics (substeps), reset kernel, fused render.

    python tools/step_split.py --model humanoid_lite --envs 16384
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00021_b200 import _native  # noqa: E402
from paper_2502_00021_b200 import bench as B  # noqa: E402
from paper_2502_00021_b200 import env as E  # noqa: E402
from paper_2502_00021_b200.models import STANDIN_MODELS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="humanoid_lite")
ap.add_argument("--envs", type=int, default=16384)
ap.add_argument("--mode", default="none")
a = ap.parse_args()
cfg = E.EnvConfig(model=STANDIN_MODELS.get(a.model, a.model), batch=a.envs,
                  distractor_mode=a.mode if a.mode != "video" else "none")
env, state, obs = E.make_env(cfg)
stub = B.ConvStub.create(84, 84, 3, env.n_joints, seed=0)
act = B.conv_stub_forward(stub, obs)
L = _native.lib()
reward = torch.zeros(a.envs, dtype=torch.float64, device="cuda")


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(n):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / n


sys_ = state.sys.copy()
ms_pol = t(lambda: B.conv_stub_forward(stub, obs))
ms_phys = t(lambda: L.pxr_physics_step(ctypes.byref(env.model_c), sys_.qpos.data_ptr(),
                                       sys_.qvel.data_ptr(), sys_.step_count.data_ptr(),
                                       sys_.done.data_ptr(), act.data_ptr(), reward.data_ptr(),
                                       a.envs, _native.stream_ptr()))
ms_render = t(lambda: env._render_obs(state.sys, state.distractor))
ms_step = t(lambda: E.step(env, state, act))
print(f"{a.model} B={a.envs}: policy {ms_pol:.3f} ms, physics {ms_phys:.3f} ms, "
      f"render(+FK) {ms_render:.3f} ms, full step {ms_step:.3f} ms")
