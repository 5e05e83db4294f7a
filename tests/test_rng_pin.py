"""The library's seeded generators (runtime.cpp mcf_rng_*, used by
paper_2207_08867_b200.data for every BASELINE config) against the reference's
own mcf::Rng (rng.hpp:13-65, compiled in oracle/_ref): identical draws, so the
bench's two arms and the tests run on the same inputs."""
import numpy as np
import pytest


def test_generators_match_reference_rng(ref):
    from paper_2207_08867_b200 import data

    for seed in (1, 2000, 2001, 3001, 1003):
        assert np.array_equal(data.uniform(seed, 5000).view(np.uint64), ref.rng_uniform(seed, 5000).view(np.uint64))
        assert np.array_equal(data.normal(seed, 5001).view(np.uint64), ref.rng_normal(seed, 5001).view(np.uint64))
        assert np.array_equal(data.below(seed, 10, 5000), ref.rng_below(seed, 10, 5000))
