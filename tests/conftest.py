import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_image(name):
    """Load an image fixture; regenerate large inputs from their recipe."""
    from oracle import port as oracle

    d = load_golden(f"image_{name}.npz")
    if "recipe_kind" in d:
        kind = str(d["recipe_kind"])
        h, w = (int(x) for x in d["recipe_shape"])
        seed = int(d["recipe_seed"])
        original = oracle.synthetic_frame(h, w, seed, kind)
        sampled, mask = oracle.quarter_sample(original, int(d["mask_seed"]))
        assert np.array_equal(np.packbits(mask), d["mask_packed"]), "mask recipe drifted"
        assert float(sampled.sum()) == float(d["sampled_sum"]), "image recipe drifted"
        d.update(original=original, sampled=sampled, mask=mask)
    return d


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)
