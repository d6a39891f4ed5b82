"""Conv-stub policy and the env-step sweep (reference bench.py; tests modelled
on the reference's tests/test_bench.py).

CPU: ``ConvStub.create`` weights equal the reference's (golden
tests/golden/policy.npz, made from the live reference). GPU: the
``pxr_conv_stub_forward`` kernel against a float64 evaluation (<= 1e-5, the
reference's tolerance) and the reference's own forward outputs, batch-row
independence, zero weights, range and shape errors; the sweep's records and
CSV round trip."""

import dataclasses
import hashlib

import numpy as np
import pytest

from conftest import golden


def f64_forward(conv, proj, obs):
    """Brute-force float64 conv -> ReLU -> linear -> tanh (same definition as
    the reference's test oracle, tests/test_bench.py:17-33)."""
    k, s, nf = 8, 4, 16
    b, h, w, c = obs.shape
    oh, ow = (h - k) // s + 1, (w - k) // s + 1
    ker = conv.astype(np.float64).reshape(k, k, c, nf)
    x = obs.astype(np.float64) / 255.0
    acts = np.empty((b, oh * ow * nf))
    for i in range(b):
        for oy in range(oh):
            for ox in range(ow):
                patch = x[i, oy * s:oy * s + k, ox * s:ox * s + k]
                acts[i, (oy * ow + ox) * nf:(oy * ow + ox + 1) * nf] = np.einsum(
                    "yxc,yxcf->f", patch, ker)
    return np.tanh(np.maximum(acts, 0.0) @ proj.astype(np.float64))


@pytest.fixture(scope="module")
def B():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.bench")


def test_weights_match_reference(B):
    rec = golden("policy.npz")
    for tag in ("a", "g"):
        h, w, c, j, seed = (int(v) for v in rec[f"{tag}_shape"])
        stub = B.ConvStub.create(h, w, c, j, seed=seed)
        np.testing.assert_array_equal(stub.conv, rec[f"{tag}_conv"])
        np.testing.assert_array_equal(stub.conv_blocks, rec[f"{tag}_conv_blocks"])
        np.testing.assert_array_equal(stub.proj, rec[f"{tag}_proj"])
    h, w, c, j, seed = (int(v) for v in rec["f_shape"])
    stub = B.ConvStub.create(h, w, c, j, seed=seed)
    got = [hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
           for a in (stub.conv, stub.conv_blocks, stub.proj)]
    assert got == [str(x) for x in rec["f_weights_sha"]]


def test_weights_pure_in_seed_and_size_checks(B):
    a = B.ConvStub.create(32, 32, 3, 6, seed=4)
    b = B.ConvStub.create(32, 32, 3, 6, seed=4)
    c = B.ConvStub.create(32, 32, 3, 6, seed=5)
    assert np.array_equal(a.conv, b.conv) and np.array_equal(a.proj, b.proj)
    assert not np.array_equal(a.conv, c.conv)
    with pytest.raises(ValueError):
        B.ConvStub.create(4, 4, 3, 2)


def test_csv_round_trip(B, tmp_path):
    recs = [B.BenchRecord("hopper_lite", 2, "none", 200, 0.5, 400.0, "32x32"),
            B.BenchRecord("walker_lite", 1000, "video", 500000, 1.23456789, 405000.123, "84x84")]
    path = tmp_path / "b.csv"
    B.write_csv(recs, path)
    back = B.read_csv(path)
    assert [r.batch for r in back] == [2, 1000]
    assert back[1].wall_seconds == pytest.approx(1.23457, rel=1e-6)
    with pytest.raises(ValueError):
        B.BenchConfig(measure_steps=10).validate()
    with pytest.raises(ValueError):
        B.BenchConfig(distractor_modes=("video",)).validate()


@pytest.mark.gpu
class TestConvStubGPU:
    def test_matches_f64_and_reference_outputs(self, B):
        rec = golden("policy.npz")
        for tag in ("a", "g", "f"):
            h, w, c, j, seed = (int(v) for v in rec[f"{tag}_shape"])
            stub = B.ConvStub.create(h, w, c, j, seed=seed)
            obs = rec[f"{tag}_obs"]
            got = B.conv_stub_forward(stub, obs)
            assert isinstance(got, np.ndarray) and got.dtype == np.float64
            assert np.max(np.abs(got - f64_forward(stub.conv, stub.proj, obs))) < 1e-5
            assert np.max(np.abs(got - rec[f"{tag}_actions"])) < 1e-5

    def test_device_in_device_out_and_rows_independent(self, B, torch):
        stub = B.ConvStub.create(84, 84, 3, 17, seed=3)
        obs = torch.randint(0, 256, (37, 84, 84, 3), dtype=torch.uint8, device="cuda")
        full = B.conv_stub_forward(stub, obs)
        assert full.is_cuda and full.dtype == torch.float64 and full.shape == (37, 17)
        for i in (0, 5, 36):
            assert torch.equal(B.conv_stub_forward(stub, obs[i:i + 1])[0], full[i])
        assert torch.equal(B.conv_stub_forward(stub, obs[10:30]), full[10:30])
        assert bool((full.abs() <= 1.0).all())

    def test_split_projection_rows_equal_one_cta_path(self, B, torch, knobs):
        """Small batches split each env's projection over CTAs (one per
        feature slice, the slice sums added in slice order by a second
        kernel); large batches walk the slices in one CTA. The arithmetic is
        the same, so a row is identical whichever path its batch takes."""
        stub = B.ConvStub.create(84, 84, 3, 17, seed=5)
        gen = torch.Generator(device="cuda").manual_seed(5)
        obs = torch.randint(0, 256, (3000, 84, 84, 3), dtype=torch.uint8, device="cuda",
                            generator=gen)
        full = B.conv_stub_forward(stub, obs)  # (one CTA per 16 envs: too many for the split)
        for i in (0, 7, 2999):
            assert torch.equal(B.conv_stub_forward(stub, obs[i:i + 1])[0], full[i])
        assert torch.equal(B.conv_stub_forward(stub, obs[100:164]), full[100:164])
        knobs.set("PXR_DEBUG_NO_SPLIT", 1)
        assert torch.equal(B.conv_stub_forward(stub, obs[:20]), full[:20])

    def test_matches_torch_conv2d_formulation(self, B, torch):
        """Weight-layout parity with the PyTorch formulation of the stub
        (SURVEY 8(f) row 3): conv weight (ky, kx, c, f) -> torch (f, c, ky,
        kx), features flattened in (oy, ox, f) order, f32 without TF32."""
        import torch.nn.functional as Fn

        stub = B.ConvStub.create(84, 84, 3, 17, seed=5)
        obs = torch.randint(0, 256, (64, 84, 84, 3), dtype=torch.uint8, device="cuda")
        w = torch.from_numpy(stub.conv).cuda().reshape(8, 8, 3, 16).permute(3, 2, 0, 1)
        p = torch.from_numpy(stub.proj).cuda()
        with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
            prev = torch.backends.cuda.matmul.allow_tf32
            torch.backends.cuda.matmul.allow_tf32 = False
            try:
                x = obs.permute(0, 3, 1, 2).float() * torch.tensor(1.0 / 255.0,
                                                                   dtype=torch.float32)
                feat = torch.relu(Fn.conv2d(x, w, stride=4)).permute(0, 2, 3, 1).reshape(64, -1)
                want = torch.tanh(feat @ p).double()
            finally:
                torch.backends.cuda.matmul.allow_tf32 = prev
        got = B.conv_stub_forward(stub, obs)
        assert float((got - want).abs().max()) < 1e-5

    def test_large_frames_convert_per_chunk(self, B):
        """Frames too large for the kernel's bf16 frame copy (140x140 RGB)
        take the per-chunk conversion path; same results."""
        stub = B.ConvStub.create(140, 140, 3, 5, seed=2)
        obs = np.random.default_rng(4).integers(0, 256, (3, 140, 140, 3), dtype=np.uint8)
        got = B.conv_stub_forward(stub, obs)
        assert np.max(np.abs(got - f64_forward(stub.conv, stub.proj, obs))) < 1e-5

    def test_zero_weights_and_shape_errors(self, B):
        stub = B.ConvStub.create(32, 32, 3, 4, seed=0)
        zero = dataclasses.replace(stub, conv=np.zeros_like(stub.conv),
                                   conv_blocks=np.zeros_like(stub.conv_blocks),
                                   proj=np.zeros_like(stub.proj))
        obs = np.random.default_rng(0).integers(0, 256, (3, 32, 32, 3), dtype=np.uint8)
        assert np.all(B.conv_stub_forward(zero, obs) == 0.0)
        with pytest.raises(ValueError):
            B.conv_stub_forward(stub, np.zeros((1, 8, 8, 3), dtype=np.uint8))

    def test_sweep_records(self, B, tmp_path):
        cfg = B.BenchConfig(env_names=("hopper_lite",), batches=(1, 2), warmup_steps=2,
                            measure_steps=100, width=32, height=32)
        recs = B.run_benchmark(cfg)
        assert [r.batch for r in recs] == [1, 2]
        for r in recs:
            assert r.steps_measured == 100 * r.batch and r.wall_seconds > 0
            assert r.steps_per_second == pytest.approx(r.steps_measured / r.wall_seconds)
            assert len(r.digest) == 64
        again = B.run_benchmark(cfg)
        assert [r.digest for r in again] == [r.digest for r in recs]  # reproducible
