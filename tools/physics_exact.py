"""Diagnostic: how far the device physics is from the reference fixtures
(max |diff| and count of unequal values), and where each recorded reference
hash chain first diverges when re-run on the device (record_rollout)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import MODEL_NAMES, golden, replay_meta  # noqa: E402
import paper_2502_00021_b200 as P  # noqa: E402
import paper_2502_00021_b200.env as E  # noqa: E402
from paper_2502_00021_b200 import _native, recorder as R  # noqa: E402
from paper_2502_00021_b200.models import STANDIN_MODELS  # noqa: E402
from paper_2502_00021_b200.prng import fold_in, key_from_seed  # noqa: E402


def cmp(tag, got, want):
    got, want = np.asarray(got), np.asarray(want)
    neq = int((got != want).sum())
    d = float(np.abs(got.astype(np.float64) - want.astype(np.float64)).max()) if got.size else 0.0
    print(f"  {tag:28s} unequal {neq:6d}/{got.size:6d}  max|diff| {d:.3e}")


rec = golden("physics.npz")
for name in MODEL_NAMES:
    model = STANDIN_MODELS.get(name, name)
    print(name)
    env, state, _ = E.make_env(E.EnvConfig(model=model, batch=32))
    sys_ = E.SystemState(torch.from_numpy(rec[f"{name}_qpos"]).cuda(),
                         torch.from_numpy(rec[f"{name}_qvel"]).cuda(),
                         torch.from_numpy(rec[f"{name}_steps"]).cuda(),
                         torch.zeros(32, dtype=torch.uint8, device="cuda"))
    reward = torch.zeros(32, dtype=torch.float64, device="cuda")
    act = torch.from_numpy(rec[f"{name}_act"]).cuda()
    _native.check(_native.lib().pxr_physics_step(
        ctypes.byref(env.model_c), sys_.qpos.data_ptr(), sys_.qvel.data_ptr(),
        sys_.step_count.data_ptr(), sys_.done.data_ptr(), act.data_ptr(), reward.data_ptr(),
        32, _native.stream_ptr()))
    cmp("step qpos", sys_.qpos.cpu().numpy(), rec[f"{name}_qpos1"])
    cmp("step qvel", sys_.qvel.cpu().numpy(), rec[f"{name}_qvel1"])
    cmp("step reward", reward.cpu().numpy(), rec[f"{name}_reward"])
    env2 = E.Env(E.EnvConfig(model=model, batch=16, env_offset=5, logical_batch=64))
    s2, _, _ = E._reset_state(env2, fold_in(key_from_seed(3), 0x5EED))
    cmp("reset qpos", s2.qpos.cpu().numpy(), rec[f"{name}_reset_qpos"])
    cmp("reset qvel", s2.qvel.cpu().numpy(), rec[f"{name}_reset_qvel"])

for tag in ("cheetah_none_b1", "walker_video_b8", "ant_color_b8", "humanoid_video_b8_slice",
            "hopper_color_gray_b4"):
    r = golden(f"replay_{tag}.npz")
    m = replay_meta(r)
    if m["mode"] == "video":
        continue  # needs the pack file; covered by tests/test_recorder.py
    cfg = E.EnvConfig(model=STANDIN_MODELS.get(m["model"], m["model"]), batch=m["batch"],
                      seed=m["seed"], distractor_mode=m["mode"], observation=m["observation"],
                      env_offset=m["env_offset"], logical_batch=m["logical_batch"])
    steps = int(m["steps"])
    dg = R.record_rollout(cfg, f"random:{m['seed']}", steps)
    ref = [bytes(h).hex() for h in r["hashes"][:steps + 1]]
    first = next((t for t, (a, b) in enumerate(zip(dg.hashes, ref)) if a != b), None)
    print(f"chain {tag}: first divergence {first} of {steps}")
