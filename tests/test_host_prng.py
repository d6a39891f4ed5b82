"""The reference's PRNG property tests (tests/test_prng.py:76-190) restated
for this package: key derivation (split / fold_in purity, distinctness,
prefix stability), distributions (uniform mean and range, normal moments,
index histogram, uncorrelated split streams) and the hypothesis properties
on the host; fold_in_many / words_per_key run on the device (GPU tests)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import REPO  # noqa: F401  (package on sys.path)
from paper_2502_00021_b200.prng import (Key, fold_in, index_from_words, key_from_seed, normal,
                                        random_index, split, uniform)


class TestKeyDerivation:
    def test_seeds_split_and_prefix(self):
        assert key_from_seed(0) == key_from_seed(0) and key_from_seed(0) != key_from_seed(1)
        k = key_from_seed(3)
        keys = split(k, 1000)
        assert len(set(keys)) == 1000 and k not in keys
        assert split(key_from_seed(9), 2) == split(key_from_seed(9), 2)
        k4 = key_from_seed(4)
        assert split(k4, 1000)[:10] == split(k4, 10)  # split(k, n)[i] independent of n
        with pytest.raises(ValueError):
            split(key_from_seed(0), 0)

    def test_fold_in_chain_deterministic(self):
        k = key_from_seed(1)
        assert fold_in(fold_in(k, 3), 7) == fold_in(fold_in(k, 3), 7)


class TestDistributions:
    def test_uniform(self):
        assert abs(uniform(key_from_seed(7), 100_000).mean() - 0.5) < 0.01
        eps = 1e-12
        v = uniform(key_from_seed(8), 5, 2.0, 2.0 + eps)
        assert np.all(v >= 2.0) and np.all(v < 2.0 + eps)
        with pytest.raises(ValueError):
            uniform(key_from_seed(0), 3, 1.0, 1.0)

    def test_normal_moments(self):
        v = normal(key_from_seed(9), 100_000)
        assert abs(v.mean()) < 0.02 and abs(v.var() - 1.0) < 0.02

    def test_random_index(self):
        assert random_index(key_from_seed(11), 1) == 0

    def test_split_streams_uncorrelated(self):
        a, b = split(key_from_seed(14), 2)
        assert abs(np.corrcoef(uniform(a, 100_000), uniform(b, 100_000))[0, 1]) < 0.01


@settings(deadline=None, max_examples=50)
@given(seed=st.integers(0, 2**64 - 1), n=st.integers(1, 200))
def test_uniform_pure_and_in_range(seed, n):
    k = key_from_seed(seed)
    a, b = uniform(k, n, -3.0, 2.0), uniform(k, n, -3.0, 2.0)
    assert np.array_equal(a, b) and np.all(a >= -3.0) and np.all(a < 2.0)


@settings(deadline=None, max_examples=50)
@given(seed=st.integers(0, 2**64 - 1), data=st.integers(0, 2**64 - 1))
def test_fold_in_changes_key(seed, data):
    k = key_from_seed(seed)
    assert fold_in(k, data) != k


@pytest.fixture(scope="module")
def P():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.prng")


@pytest.mark.gpu
class TestDeviceKeyStreams:
    """fold_in_many / words_per_key: this package's versions run on the B200."""

    @staticmethod
    def _pairs(hi, lo):
        return set(zip(hi.cpu().numpy().view(np.uint64).tolist(),
                       lo.cpu().numpy().view(np.uint64).tolist()))

    def test_fold_in_many_distinct_and_matches_scalar(self, P):
        k = key_from_seed(5)
        hi, lo = P.fold_in_many(k, np.arange(100_000, dtype=np.uint64))
        assert len(self._pairs(hi, lo)) == 100_000
        k12 = key_from_seed(12)
        hi, lo = P.fold_in_many(k12, np.array([0, 5, 77], dtype=np.uint64))
        h, l_ = hi.cpu().numpy().view(np.uint64), lo.cpu().numpy().view(np.uint64)
        for i, d in enumerate((0, 5, 77)):
            assert fold_in(k12, d) == Key(int(h[i]), int(l_[i]))

    def test_no_collisions_among_derived_keys(self, P):
        k = key_from_seed(6)
        seen = self._pairs(*P.fold_in_many(k, np.arange(500_000, dtype=np.uint64)))
        seen.update((key.hi, key.lo) for key in split(k, 500_000))
        assert len(seen) == 1_000_000

    def test_index_histogram_and_words_match_random_index(self, P):
        hi, lo = P.fold_in_many(key_from_seed(10), np.arange(100_000, dtype=np.uint64))
        w, _ = P.words_per_key(hi, lo, 0)
        counts = np.bincount(index_from_words(w.cpu().numpy().view(np.uint64), 4), minlength=4)
        assert np.all(np.abs(counts - 25_000) <= 600)
        keys = split(key_from_seed(13), 50)
        w, _ = P.words_per_key(np.array([q.hi for q in keys], dtype=np.uint64),
                               np.array([q.lo for q in keys], dtype=np.uint64), 0)
        vec = index_from_words(w.cpu().numpy().view(np.uint64), 121)
        assert all(random_index(q, 121) == vec[i] for i, q in enumerate(keys))
