"""Pin the CPU oracle (oracle/) to the reference before trusting it.

Every comparison here is against fixtures frozen from the LIVE reference by
tests/golden/make_golden.py, or against the reference's own golden vectors
(reference tests/test_prng.py:20-74). No GPU needed.
"""

import hashlib

import numpy as np
import pytest

from conftest import MODEL_NAMES, geometry_of, golden, replay_meta, spec_of

# reference tests/test_prng.py:22-47
GOLDEN_KEY_0 = (0xD2B9123EEDD0915F, 0x4831627E7DCE6036)
GOLDEN_KEY_42 = (0xF5069347BE28EB50, 0x3306C120DCB434CC)
GOLDEN_BITS_0 = (0x1789D6118975704B, 0x57D5674490D412BB, 0xA1997670770BE0D1, 0xAFAF98D8129F0DBB)
GOLDEN_SPLIT_0 = (
    (0x51D04B7680BDF9FA, 0x43C8245429F95C60),
    (0x4541609099B34D3F, 0xC77A7A491B96E4B6),
    (0xA6A363E1A772C828, 0x3A1FDCAE81F3E202),
)
GOLDEN_FOLD_0_7 = (0x68E3DF91C05D6C14, 0x741BFF0A50063A5F)


class TestOraclePrng:
    def test_key_from_seed(self, oracle):
        assert oracle.key_from_seed(0) == GOLDEN_KEY_0
        assert oracle.key_from_seed(42) == GOLDEN_KEY_42

    def test_bits_split_fold(self, oracle):
        bits = [oracle.threefry2x64(*GOLDEN_KEY_0, b, 0) for b in range(2)]
        assert (bits[0][0], bits[0][1], bits[1][0], bits[1][1]) == GOLDEN_BITS_0
        assert tuple(oracle.split_one(GOLDEN_KEY_0, i) for i in range(3)) == GOLDEN_SPLIT_0
        assert oracle.fold_in(GOLDEN_KEY_0, 7) == GOLDEN_FOLD_0_7

    def test_random_index(self, oracle):
        w = oracle.threefry2x64(*GOLDEN_KEY_0, 0, 0)[0]
        assert oracle.index_from_word(w, 1000) == 91

    def test_c_threefry_matches_python(self, oracle):
        rng = np.random.default_rng(0)
        c0 = rng.integers(0, 2**63, 500, dtype=np.uint64)
        y0, y1 = oracle.threefry2x64_many(GOLDEN_KEY_0[0], GOLDEN_KEY_0[1], c0, 2)
        for i in range(0, 500, 37):
            assert (int(y0[i]), int(y1[i])) == oracle.threefry2x64(*GOLDEN_KEY_0, int(c0[i]), 2)


class TestOracleSinCosf:
    def test_glibc_restatement_strided(self, oracle):
        # The full 2^32 sweep (0 mismatches) is recorded in DESIGN.md; a
        # strided ~1.4e8-float sweep keeps the CPU suite fast.
        bad = oracle.lib().oracle_sincosf_selftest(0, 0xFFFFFFFF, 31)
        assert bad == 0

    def test_pitch_range_dense(self, oracle):
        lo = np.float32(-130.0).view(np.uint32)
        bad = oracle.lib().oracle_sincosf_selftest(0, int(np.float32(130.0).view(np.uint32)), 7)
        assert bad == 0 and lo > 0


class TestOracleSinCos64:
    """oracle/sin_glibc.c (glibc 2.39 sin / cos restated with the -mfma
    build's contractions as explicit fma) against this image's libm, which
    numpy's float64 np.sin / np.cos call (physics.py:134-135, 529-538)."""

    def test_matches_libm(self, oracle):
        rng = np.random.default_rng(7)
        for scale in (1e-7, 0.126, 0.85, 2.43, 10.0, 1e3, 1e8):
            x = rng.uniform(-scale, scale, 400_000)
            s, c = oracle.sincos64(x)
            np.testing.assert_array_equal(s, np.sin(x))
            np.testing.assert_array_equal(c, np.cos(x))

    def test_range_edges(self, oracle):
        edges = np.array([0x3e400000, 0x3e500000, 0x3feb6000, 0x400368fd, 0x419921fa],
                         dtype=np.uint64) << np.uint64(32)
        x = np.concatenate([(edges + np.uint64(d)).view(np.float64) for d in (0, 1, 2)] +
                           [(edges - np.uint64(d)).view(np.float64) for d in (1, 2)])
        x = np.concatenate([x, -x, [0.0, -0.0, 0.126, -0.126, np.pi / 2, np.pi]])
        s, c = oracle.sincos64(x)
        np.testing.assert_array_equal(s, np.sin(x))
        np.testing.assert_array_equal(c, np.cos(x))


class TestOracleNumpyLog:
    """oracle/np_log_svml.c (numpy 2.3.5's AVX-512 float64 log, the
    Box-Muller log of the reset draws, prng.py:147) against np.log."""

    def test_matches_numpy(self, oracle):
        rng = np.random.default_rng(5)
        for lo, hi in ((2.0 ** -53, 1.0), (0.5, 2.0), (1e-300, 1e300)):
            x = np.exp(rng.uniform(np.log(lo), np.log(hi), 4_000_000))
            np.testing.assert_array_equal(oracle.np_log(x), np.log(x))

    def test_uniform_draws(self, oracle):
        # the reset draws' own arguments: (w >> 11) 2^-53 in [2^-53, 1)
        w = np.random.default_rng(6).integers(0, 2**63, 2_000_000, dtype=np.int64)
        u = ((w.astype(np.uint64) >> np.uint64(11)) | np.uint64(1)).astype(np.float64) * 2.0 ** -53
        np.testing.assert_array_equal(oracle.np_log(u), np.log(u))


class TestOracleRender:
    @pytest.mark.parametrize("name", MODEL_NAMES)
    def test_matches_reference_frames(self, oracle, name):
        rec = golden(f"render_{name}.npz")
        geom = geometry_of(name)
        for fib in (0, 1):
            px, dp = oracle.render_robot_batch(geom, rec["poses"], 84, 84, bool(fib), threads=4)
            np.testing.assert_array_equal(px, rec[f"pixels_fib{fib}"])
            np.testing.assert_array_equal(dp.view(np.uint32), rec[f"depth_fib{fib}"].view(np.uint32))
        px, dp = oracle.render_robot_batch(geom, rec["poses"][:8], 64, 48, False, threads=2)
        np.testing.assert_array_equal(px, rec["pixels_64x48"])
        np.testing.assert_array_equal(dp.view(np.uint32), rec["depth_64x48"].view(np.uint32))

    def test_thread_count_invariance(self, oracle):
        rec = golden("render_walker_lite.npz")
        geom = geometry_of("walker_lite")
        a = oracle.render_robot_batch(geom, rec["poses"], 84, 84, False, threads=1)
        b = oracle.render_robot_batch(geom, rec["poses"], 84, 84, False, threads=7)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


class TestOracleDistractor:
    def test_color_biases(self, oracle):
        rec = golden("distractor.npz")
        kt = oracle.fold_in(oracle.key_from_seed(5), 3)
        np.testing.assert_array_equal(oracle.color_biases(kt, 0, 64), rec["color_adv_seed5_t3_b64"])
        np.testing.assert_array_equal(oracle.color_biases(kt, 48, 16),
                                      rec["color_adv_seed5_t3_off48_b16"])

    def test_init_distractors(self, oracle):
        """The vectorised host init (distractor.py:82-113) vs the reference's
        outputs, with and without env_offset."""
        rec = golden("distractor.npz")
        k = oracle.key_from_seed(5)
        np.testing.assert_array_equal(oracle.init_distractors("color", None, k, 64)["color_bias"],
                                      rec["color_init_seed5_b64"])
        np.testing.assert_array_equal(
            oracle.init_distractors("color", None, k, 16, env_offset=48)["color_bias"],
            rec["color_init_seed5_off48_b16"])
        v = oracle.init_distractors("video", rec["pack_counts"], oracle.key_from_seed(9), 40,
                                    env_offset=3)
        np.testing.assert_array_equal(v["video_index"], rec["video_init_seed9_off3_b40"])
        np.testing.assert_array_equal(v["frame_count"],
                                      rec["pack_counts"][rec["video_init_seed9_off3_b40"]])
        assert (v["frame_cursor"] == 0).all() and (v["direction"] == 1).all()

    def test_pose_source_host(self, oracle):
        """The host pose source: reset draws within rest +- 0.1 at t=0 for the
        root, FK chained along parents, env_offset slices consistent."""
        from paper_2502_00021_b200.models import model_kinematics

        spec = spec_of("humanoid_lite")
        par, anc, _, _ = model_kinematics(spec)
        rk = oracle.fold_in(oracle.key_from_seed(0), 0x5EED)
        full = oracle.pose_source(spec.rest(), par, anc, rk, 0, 7, 64)
        part = oracle.pose_source(spec.rest(), par, anc, rk, 40, 7, 8)
        np.testing.assert_array_equal(full[40:48], part)
        assert full.shape == (64, spec.n_links, 3)
        t0 = oracle.pose_source(spec.rest(), par, anc, rk, 0, 0, 64)
        g = np.arange(64) % 997 * 0.37
        base = t0[:, 0, 1] - 0.03 * np.sin(g)
        assert np.all(np.abs(base - spec.rest()[1]) <= 0.1 + 1e-12)

    def test_ping_pong(self, oracle):
        rec = golden("distractor.npz")
        seq, dirs = rec["video_cursor_seq"], rec["video_dir_seq"]
        counts = rec["pack_counts"][golden("distractor.npz")["video_init_seed9_off3_b40"]]
        c, d = seq[0], dirs[0]
        for t in range(1, len(seq)):
            c, d = oracle.video_advance(c, d, counts)
            np.testing.assert_array_equal(c, seq[t])
            np.testing.assert_array_equal(d, dirs[t])

    def test_composites(self, oracle):
        rec = golden("distractor.npz")
        px = rec["comp_pixels"].copy()
        oracle.apply_color_inplace(px, rec["comp_bias"])
        np.testing.assert_array_equal(px, rec["comp_color_out"])
        px = rec["comp_pixels"].copy()
        fi = rec["pack_starts"][rec["comp_vidx"]] + rec["comp_cursor"]
        oracle.apply_video_inplace(px, rec["comp_depth"], rec["pack_frames"], fi)
        np.testing.assert_array_equal(px, rec["comp_video_out"])


REPLAYS = ("cheetah_none_b1", "walker_video_b8", "ant_color_b8",
           "humanoid_video_b8_slice", "hopper_color_gray_b4")


def oracle_replay(oracle, tag, steps=None):
    """Re-derive the reference's obs hash chain from the frozen per-step
    poses/done flags with the oracle: render + key schedule + distractor
    state machine (env.py:176-255)."""
    rec = golden(f"replay_{tag}.npz")
    m = replay_meta(rec)
    geom = geometry_of(m["model"])
    B, off, lb = m["batch"], m["env_offset"], m["logical_batch"]
    master = oracle.key_from_seed(m["seed"])
    dist_key = oracle.fold_in(master, 0xD157)
    n = rec["poses"].shape[0] if steps is None else steps + 1
    frames = starts = counts = None
    if m["mode"] == "video":
        frames, starts, counts = rec["pack_frames"], rec["pack_starts"], rec["pack_counts"]
    # the vectorised host restatements (oracle.init_distractors /
    # advance_state) pinned here by the reference's own hash chains
    st = oracle.init_distractors(m["mode"], counts, dist_key, B, env_offset=off)
    h = b"\x00" * 32
    for t in range(n):
        if t > 0:
            st = oracle.advance_state(st, m["mode"], oracle.fold_in(master, t - 1), off, lb,
                                      frame_counts=counts, done=rec["done"][t])
        px, dp = oracle.render_robot_batch(geom, rec["poses"][t], 84, 84,
                                           m["floor_in_background"], threads=4)
        if m["mode"] == "color":
            oracle.apply_color_inplace(px, st["color_bias"])
        elif m["mode"] == "video":
            oracle.apply_video_inplace(px, dp, frames,
                                       starts[st["video_index"]] + st["frame_cursor"])
        obs = oracle.grayscale(px) if m["observation"] == "grayscale" else px
        h = hashlib.sha256(h + np.ascontiguousarray(obs).tobytes()).digest()
        assert h == rec["hashes"][t].tobytes(), f"{tag}: oracle diverges at t={t}"
    return rec


class TestOracleReplay:
    @pytest.mark.parametrize("tag", REPLAYS)
    def test_hash_chain(self, oracle, tag):
        steps = 200 if tag == "cheetah_none_b1" else None
        rec = oracle_replay(oracle, tag, steps)
        assert rec["hashes"].shape[1] == 32


def test_oracle_header_says_test_only():
    import os

    from conftest import REPO

    for f in ("oracle.h", "oracle.py", "render_oracle.c", "prng_oracle.c", "sincosf_glibc.c"):
        with open(os.path.join(REPO, "oracle", f)) as fh:
            head = fh.read(600)
        assert "ORACLE / TEST INFRASTRUCTURE ONLY" in head, f


def test_spec_of_models_load():
    for n in MODEL_NAMES:
        assert spec_of(n).n_links >= 4
