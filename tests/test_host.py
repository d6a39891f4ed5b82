"""Host-side pieces of the package (no GPU): PRNG golden vectors, model
loading, tessellation/geometry identical to the reference's, the PXVP
container and the synthetic-pack recipe."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, MODEL_NAMES, geometry_of, spec_of

import paper_2502_00021_b200 as P
from paper_2502_00021_b200 import prng
from paper_2502_00021_b200.video_pack import (
    PackFormatError, VideoPack, generate_synthetic_pack, load_video_pack, save_video_pack)


class TestPrngGolden:  # reference tests/test_prng.py:20-74
    def test_keys(self):
        assert P.key_from_seed(0) == P.Key(0xD2B9123EEDD0915F, 0x4831627E7DCE6036)
        assert P.key_from_seed(42) == P.Key(0xF5069347BE28EB50, 0x3306C120DCB434CC)

    def test_bits_uniform_normal(self):
        k = P.key_from_seed(0)
        assert tuple(int(x) for x in prng.random_bits(k, 4)) == (
            0x1789D6118975704B, 0x57D5674490D412BB, 0xA1997670770BE0D1, 0xAFAF98D8129F0DBB)
        assert tuple(float(x) for x in P.uniform(k, 4)) == (
            0.09194696357868337, 0.34310002731292877, 0.6312479042599501, 0.6862731483002983)
        assert tuple(float(x) for x in P.normal(k, 4)) == (
            -1.4830239295849081, -0.5701480166623415, -1.6042838671150963, -1.3469958196367307)
        assert float(P.uniform(P.key_from_seed(42), 1)[0]) == 0.8685604140926122

    def test_split_fold_index(self):
        k = P.key_from_seed(0)
        assert tuple(P.split(k, 3)) == (
            P.Key(0x51D04B7680BDF9FA, 0x43C8245429F95C60),
            P.Key(0x4541609099B34D3F, 0xC77A7A491B96E4B6),
            P.Key(0xA6A363E1A772C828, 0x3A1FDCAE81F3E202))
        assert P.fold_in(k, 7) == P.Key(0x68E3DF91C05D6C14, 0x741BFF0A50063A5F)
        assert P.random_index(k, 1000) == 91

    def test_index_from_words_is_umulhi(self):
        rng = np.random.default_rng(0)
        w = rng.integers(0, 2**64 - 1, 20000, dtype=np.uint64)
        for n in (1, 2, 4, 121, 1000, 2**31 + 7, 2**32 - 1):
            got = prng.index_from_words(w, n)
            want = np.array([(int(x) * n) >> 64 for x in w[:500]], dtype=np.int64)
            assert np.array_equal(got[:500], want)
        with pytest.raises(ValueError):
            prng.index_from_words(w, 0)


class TestModels:
    def test_builtins(self):
        assert P.BUILTIN_MODELS == ("cheetah_lite", "walker_lite", "hopper_lite")
        with pytest.raises(ValueError, match="builtin"):
            P.builtin_model("ant_lite")
        assert [spec_of(n).n_links for n in MODEL_NAMES] == [7, 7, 4, 9, 13]

    def test_roundtrip(self, tmp_path):
        for n in MODEL_NAMES:
            s = spec_of(n)
            p = tmp_path / f"{n}.model"
            P.save_model(s, p)
            assert P.load_model(p) == s

    def test_bad_file(self, tmp_path):
        p = tmp_path / "bad.model"
        p.write_text("link = 1 2\n")
        with pytest.raises(ValueError, match="3 numbers"):
            P.load_model(p)

    @pytest.mark.parametrize("name", MODEL_NAMES)
    def test_geometry_identical_to_reference(self, name):
        with open(os.path.join(GOLDEN, "geometry.json")) as f:
            want = json.load(f)[name]
        g = geometry_of(name)
        sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa
        assert len(g.base_verts) == want["n_verts"] and len(g.triangles) == want["n_tris"]
        assert sha(g.base_verts) == want["base_verts"]
        assert sha(g.vert_link) == want["vert_link"]
        assert sha(g.triangles) == want["triangles"]
        assert sha(g.tri_colors) == want["tri_colors"]

    def test_tessellation_counts(self):  # reference tests/test_render.py:33-50
        for r, s in ((2, 3), (3, 8), (8, 12)):
            m = P.tessellate_capsule(0.1, 1.0, r, s)
            assert len(m.vertices) == 2 + 2 * r * s and len(m.triangles) == 4 * r * s
            m = P.tessellate_sphere(0.5, r, s)
            assert len(m.vertices) == 2 + (r - 1) * s
        with pytest.raises(ValueError):
            P.tessellate_capsule(0.1, 1.0, 2, 2)

    def test_camera(self):  # reference tests/test_render.py:76-108
        cam = P.track_camera((1.0, 0.5))
        assert cam.eye == (1.0, -3.0, 1.7) and cam.target == (1.0, 0.0, 0.5)
        b = P.camera_basis(P.track_camera((0.0, 0.0)))
        assert b[3] == 1.0 and b[4] == 0.0 and b[5] == 0.0 and b[6] == 0.0
        with pytest.raises(ValueError):
            P.camera_basis(P.Camera(eye=(0, 0, 0), target=(0, 0, 0)))
        with pytest.raises(ValueError):
            P.camera_basis(P.Camera(eye=(0, 0, 0), target=(0, 0, 1)))


class TestVideoPack:
    def test_synthetic_pack_sha_pinned(self, tmp_path):
        # reference tests/test_video_pack.py:21 (the shipped asset's digest)
        path = tmp_path / "synthetic_pack.pxvp"
        generate_synthetic_pack(P.key_from_seed(2024), 4, 60, 64, 64, path)
        digest = hashlib.sha256(path.read_bytes()).hexdigest()
        assert digest == "a8907f5727572f02f903ec6c9341a0d6376a219622b2f5f16cdd858421819752"

    def test_roundtrip_and_corruption(self, tmp_path):
        rng = np.random.default_rng(0)
        pack = VideoPack([rng.integers(0, 256, (3, 8, 8, 3), dtype=np.uint8),
                          rng.integers(0, 256, (5, 8, 8, 3), dtype=np.uint8)], 8, 8)
        p = tmp_path / "p.pxvp"
        save_video_pack(pack, p)
        q = load_video_pack(p)
        assert q.video_count == 2 and list(q.frame_counts) == [3, 5]
        frames, starts = q.flat_frames()
        assert frames.shape == (8, 8, 8, 3) and list(starts) == [0, 3]
        raw = bytearray(p.read_bytes())
        raw[100] ^= 1
        p.write_bytes(bytes(raw))
        with pytest.raises(PackFormatError, match="digest"):
            load_video_pack(p)
        p.write_bytes(b"XXXX" + bytes(raw[4:]))
        with pytest.raises(PackFormatError, match="magic"):
            load_video_pack(p)


class TestEnvConfig:  # reference tests/test_env.py:250-280
    def test_round_trip_and_validation(self, tmp_path):
        from paper_2502_00021_b200.env import EnvConfig, load_env_config, save_env_config

        cfg = EnvConfig(model="walker_lite", batch=7, distractor_mode="color", seed=9,
                        floor_in_background=True, logical_batch=20, env_offset=3)
        p = tmp_path / "c.cfg"
        save_env_config(cfg, p)
        assert load_env_config(p) == cfg
        assert load_env_config(p, batch=2).batch == 2
        p.write_text("nope = 1\n")
        with pytest.raises(ValueError, match="unknown config key"):
            load_env_config(p)
        with pytest.raises(ValueError, match="video_pack_path"):
            EnvConfig(distractor_mode="video").validate()
        with pytest.raises(ValueError, match="logical_batch"):
            EnvConfig(batch=4, env_offset=2, logical_batch=5).validate()
        assert EnvConfig(distractor_mode="video", video_pack_path="x").resolved_floor_in_background
