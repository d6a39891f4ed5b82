"""The reference's distractor known-answer tests (tests/test_distractor.py:
100-250) restated against this package's device API: ping-pong cursor
sequences, the colour clamp-add (examples, saturation, foreground too, input
untouched, mode check), the video composite (full background, checker-mask
foreground, no background, nearest-neighbour scaling) and nearest_map."""

import numpy as np
import pytest

from conftest import REPO  # noqa: F401  (puts the package on sys.path)


@pytest.fixture(scope="module")
def D():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.distractor")


def make_pack(pkg, n_videos=1, frames=3, size=8, seed=0):
    rng = np.random.default_rng(seed)
    vids = [rng.integers(0, 256, (frames, size, size, 3), dtype=np.uint8) for _ in range(n_videos)]
    return pkg.VideoPack(videos=vids, height=size, width=size)


def frame_with_mask(pkg, torch, batch=1, h=8, w=8, fill=0):
    """All-background frame (depth +inf) filled with one grey value."""
    f = pkg.Frame.allocate(batch, h, w)
    f.pixels.fill_(fill)
    f.depth.fill_(float("inf"))
    return f


def color_state(D, torch, biases):
    b = torch.tensor(np.asarray(biases, dtype=np.int16).reshape(-1, 3), device="cuda")
    z = torch.zeros(0, dtype=torch.int64, device="cuda")
    return D.DistractorState("color", b, z, z.clone(), torch.zeros(0, dtype=torch.int8,
                                                                  device="cuda"), z.clone())


def video_state(D, torch, pack, video_index, cursor):
    n = len(video_index)
    vidx = np.asarray(video_index, dtype=np.int64)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return D.DistractorState("video", dev(np.zeros((n, 3), np.int16)), dev(vidx),
                             dev(np.asarray(cursor, np.int64)), dev(np.ones(n, np.int8)),
                             dev(pack.frame_counts[vidx]))


def test_nearest_map(D):
    assert D.nearest_map(8, 8).tolist() == list(range(8))
    assert D.nearest_map(4, 8).tolist() == [0, 2, 4, 6]
    assert D.nearest_map(4, 2).tolist() == [0, 0, 1, 1]
    for dst, src in ((7, 3), (3, 7), (84, 64), (64, 84)):
        m = D.nearest_map(dst, src)
        assert len(m) == dst and m.min() >= 0 and m.max() < src and np.all(np.diff(m) >= 0)


@pytest.mark.gpu
class TestPingPong:
    @pytest.mark.parametrize("frames,seed,want", [(3, 8, [0, 1, 2, 1, 0, 1]),
                                                  (2, 9, [0, 1, 0, 1, 0])])
    def test_sequences(self, pkg, D, frames, seed, want):
        pack = make_pack(pkg, frames=frames)
        s = D.init_distractors("video", pack, pkg.key_from_seed(seed), 1)
        seq = [int(s.frame_cursor[0])]
        for t in range(1, len(want)):
            s = D.advance_distractors(s, pkg.fold_in(pkg.key_from_seed(seed), t))
            seq.append(int(s.frame_cursor[0]))
        assert seq == want

    def test_cursor_always_valid(self, pkg, D):
        pack = make_pack(pkg, n_videos=2, frames=4)
        s = D.init_distractors("video", pack, pkg.key_from_seed(10), 16)
        for t in range(1, 20):
            s = D.advance_distractors(s, pkg.fold_in(pkg.key_from_seed(10), t))
            c, n = s.frame_cursor.cpu().numpy(), s.frame_count.cpu().numpy()
            assert np.all((c >= 0) & (c < n))


@pytest.mark.gpu
class TestApplyColor:
    def test_examples_and_saturation(self, pkg, D, torch):
        out = D.apply_color(frame_with_mask(pkg, torch, fill=128), color_state(D, torch,
                                                                              [[-10, 0, 10]]))
        assert tuple(out.pixels[0, 0, 0].tolist()) == (118, 128, 138)
        f = frame_with_mask(pkg, torch, fill=77)
        assert torch.equal(D.apply_color(f, color_state(D, torch, [[0, 0, 0]])).pixels, f.pixels)
        hi = D.apply_color(frame_with_mask(pkg, torch, fill=250),
                           color_state(D, torch, [[60, 60, 60]]))
        lo = D.apply_color(frame_with_mask(pkg, torch, fill=5),
                           color_state(D, torch, [[-60, -60, -60]]))
        assert bool((hi.pixels == 255).all()) and bool((lo.pixels == 0).all())

    def test_clamp_add_oracle(self, pkg, D, torch):
        rng = np.random.default_rng(11)
        f = pkg.Frame.allocate(4, 8, 8)
        px = rng.integers(0, 256, (4, 8, 8, 3), dtype=np.uint8)
        f.pixels.copy_(torch.from_numpy(px))
        f.depth.fill_(float("inf"))
        biases = rng.integers(-60, 61, (4, 3)).astype(np.int16)
        out = D.apply_color(f, color_state(D, torch, biases))
        want = np.clip(px.astype(np.int32) + biases[:, None, None, :], 0, 255).astype(np.uint8)
        np.testing.assert_array_equal(out.pixels.cpu().numpy(), want)

    def test_foreground_too_input_untouched_and_mode(self, pkg, D, torch):
        f = frame_with_mask(pkg, torch, fill=100)
        f.depth[0, 2, 3] = 1.0  # a foreground pixel
        before = f.pixels.clone()
        out = D.apply_color(f, color_state(D, torch, [[10, 10, 10]]))
        assert tuple(out.pixels[0, 2, 3].tolist()) == (110, 110, 110)
        assert torch.equal(f.pixels, before)
        s = D.init_distractors("none", None, pkg.key_from_seed(0), 1)
        with pytest.raises(ValueError):
            D.apply_color(f, s)


@pytest.mark.gpu
class TestApplyVideo:
    def test_full_background_copies_frame(self, pkg, D, torch):
        pack = make_pack(pkg, n_videos=2, frames=4, size=8)
        out = D.apply_video(frame_with_mask(pkg, torch, batch=2), pack,
                            video_state(D, torch, pack, [1, 0], [2, 3]))
        np.testing.assert_array_equal(out.pixels[0].cpu().numpy(), pack.videos[1][2])
        np.testing.assert_array_equal(out.pixels[1].cpu().numpy(), pack.videos[0][3])

    def test_checker_mask_foreground_preserved(self, pkg, D, torch):
        pack = make_pack(pkg, frames=2, size=8)
        f = frame_with_mask(pkg, torch, fill=42)
        yy, xx = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
        fg = (yy + xx) % 2 == 0
        f.depth[0][torch.from_numpy(fg).cuda()] = 1.5
        depth_before = f.depth.clone()
        out = D.apply_video(f, pack, video_state(D, torch, pack, [0], [1]))
        px = out.pixels[0].cpu().numpy()
        assert np.all(px[fg] == 42)
        np.testing.assert_array_equal(px[~fg], pack.videos[0][1][~fg])
        assert torch.equal(out.depth, depth_before)

    def test_no_background_is_identity(self, pkg, D, torch):
        pack = make_pack(pkg)
        f = frame_with_mask(pkg, torch, fill=9)
        f.depth.fill_(2.0)
        out = D.apply_video(f, pack, video_state(D, torch, pack, [0], [0]))
        assert torch.equal(out.pixels, f.pixels)

    def test_nearest_neighbour_scaling(self, pkg, D, torch):
        pack = make_pack(pkg, frames=2, size=8)
        out = D.apply_video(frame_with_mask(pkg, torch, h=16, w=16), pack,
                            video_state(D, torch, pack, [0], [0]))
        rows, cols = D.nearest_map(16, 8), D.nearest_map(16, 8)
        np.testing.assert_array_equal(out.pixels[0].cpu().numpy(),
                                      pack.videos[0][0][rows][:, cols])
