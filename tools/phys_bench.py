"""Physics-step kernel timing: the warp-per-env and thread-per-env kernels
of pxr_physics_step (PXR_DEBUG_PHYS) over batch sizes, to set their crossover
(kWarpEnvMax in csrc/pxr_physics.cu)."""
import sys, os, ctypes, torch
sys.path.insert(0, '.')
import paper_2502_00021_b200.env as E
from paper_2502_00021_b200 import _native
from paper_2502_00021_b200.models import STANDIN_MODELS
L = _native.lib()
for model in ("humanoid_lite", "cheetah_lite"):
    for B in [int(x) for x in os.environ.get("PHYS_BATCHES", "1 10 100 1000 4096 16384 65536").split()]:
        env, s, obs = E.make_env(E.EnvConfig(model=STANDIN_MODELS.get(model, model), batch=B))
        act = torch.zeros((B, env.n_joints), dtype=torch.float64, device='cuda')
        res = []
        for kind in ("thread", "warp", "half", "quarter"):
            _native.set_debug("PXR_DEBUG_PHYS", kind)
            sysc = s.sys.copy(); rew = torch.zeros(B, dtype=torch.float64, device='cuda')
            f = lambda: L.pxr_physics_step(ctypes.byref(env.model_c), sysc.qpos.data_ptr(), sysc.qvel.data_ptr(), sysc.step_count.data_ptr(), sysc.done.data_ptr(), act.data_ptr(), rew.data_ptr(), B, _native.stream_ptr())
            for _ in range(3): f()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 20
            torch.cuda.synchronize(); a.record()
            for _ in range(n): f()
            b.record(); torch.cuda.synchronize(); res.append(a.elapsed_time(b) / n)
        print(f"{model} B={B}: thread {res[0]:.3f} ms  warp {res[1]:.3f} ms  half {res[2]:.3f} ms  quarter {res[3]:.3f} ms", flush=True)
        del env, s, obs
