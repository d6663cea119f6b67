"""CPU-only tests: the C-ABI library, host-side API mirror and validation."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

import paper_2202_13926_b200 as fsr
from paper_2202_13926_b200 import _lib


def _header_functions():
    src = open(os.path.join(ROOT, "include", "fsr.h")).read()
    return sorted(set(re.findall(r"\b(fsr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    names = _header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.EXPORTED)
    assert L.fsr_abi_version() == 4


def test_params_validation_messages():
    L = _lib.load()
    buf = ctypes.create_string_buffer(256)
    p = _lib.make_params()
    assert L.fsr_params_validate(ctypes.byref(p), buf, 256) == 0
    cases = [
        (dict(block=0), "target block size must be at least 1"),
        (dict(border=-1), "border must be non-negative"),
        (dict(rho=1.0), "decay factor rho must lie in (0, 1)"),
        (dict(gamma=1.5), "compensation factor gamma must lie in (0, 1]"),
        (dict(iterations=-1), "iteration count must be non-negative"),
        (dict(border=15), "exceeds the 1024-lane reduction capacity"),
    ]
    for kw, msg in cases:
        q = _lib.make_params(**kw)
        rc = L.fsr_params_validate(ctypes.byref(q), buf, 256)
        assert rc == _lib.FSR_EINVAL and msg in buf.value.decode(), kw
    q = _lib.make_params(border=30, reducer="linear")  # N = 64 lifted for linear
    assert L.fsr_params_validate(ctypes.byref(q), buf, 256) == 0
    q = _lib.make_params(border=31, reducer="linear")
    assert L.fsr_params_validate(ctypes.byref(q), buf, 256) == _lib.FSR_EUNSUPPORTED


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        _lib.Engine()
    with pytest.raises(RuntimeError):
        fsr.reconstruct(np.ones((8, 8)), np.ones((8, 8), bool), 4, 8, 2)


@pytest.mark.parametrize("kwargs", [
    {"block": 0}, {"border": -1}, {"rho": 0.0}, {"rho": 1.0}, {"gamma": 0.0}, {"gamma": 1.5},
    {"iterations": -1}, {"threads": 0}, {"block": 4, "border": 15}])
def test_fsrparams_rejects_like_reference(kwargs):
    with pytest.raises(ValueError):
        fsr.FsrParams(**kwargs)


def test_fsrparams_defaults_like_reference():
    p = fsr.FsrParams()
    assert (p.block, p.border, p.support, p.iterations) == (4, 6, 16, 200)
    assert fsr.FsrParams(block=4, border=14).support == 32


def test_quarter_sample_and_partition():
    k = load_golden("kats.npz")
    assert np.array_equal(fsr.quarter_sample_mask(48, 64, 3), k["mask_48x64_seed3"])
    assert np.array_equal(fsr.quarter_sample_mask(33, 35, 8), k["mask_33x35_seed8"])
    assert int(fsr.splitmix64(0, 1)[0]) == 0xE220A8397B1DCDAF
    d = fsr.block_partition(37, 53, fsr.FsrParams())
    assert len(d) == 10 * 14 and d[-1].height == 1 and d[-1].width == 1
    assert d[1].support_col == 4 - 6


def test_weights_match_reference_kats():
    k = load_golden("kats.npz")
    for s in (4, 8, 16, 32):
        assert np.array_equal(fsr.frequency_weight(s), k[f"wf_{s}"])


def test_sampled_image_contract():
    img = fsr.GrayImage(np.ones((4, 4)))
    with pytest.raises(ValueError, match="zero"):
        fsr.SampledImage(img, np.zeros((4, 4), bool))
    with pytest.raises(ValueError, match="differ"):
        fsr.SampledImage(img, np.ones((3, 4), bool))
    with pytest.raises(ValueError):
        fsr.GrayImage(np.array([[np.nan]]))


def test_reconstruct_argument_validation():
    with pytest.raises(ValueError, match="even"):
        fsr.reconstruct(np.ones((8, 8)), np.ones((8, 8), bool), 4, 9, 2)
    with pytest.raises(ValueError, match="unknown argmax strategy"):
        fsr.reconstruct(np.ones((8, 8)), np.ones((8, 8), bool), 4, 8, 2, reducer="x")


def test_missing_library_fails_loudly(tmp_path):
    """Without the built libfsr.so the package raises (no CPU fallback)."""
    import subprocess
    import sys
    code = ("import numpy as np, paper_2202_13926_b200 as f\n"
            "try:\n    f.reconstruct(np.ones((8, 8)), np.ones((8, 8), bool), 4, 8, 2)\n"
            "except RuntimeError as e:\n    print('raised', 'missing' in str(e))\n")
    env = dict(os.environ, FSR_LIBFSR=str(tmp_path / "nope.so"))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert "raised True" in out.stdout, out.stdout + out.stderr


def test_output_pool_never_recycles_live_memory():
    """Host-buffer calls return new arrays on recycled memory (no first-touch
    faults per call); memory returns to the pool only after the array AND every
    view of it are gone."""
    import gc

    from paper_2202_13926_b200 import _lib

    pool = _lib._OutputPool()
    a = np.frombuffer(_lib._Lease(pool.take(160), pool), dtype=np.float64).reshape(4, 5)
    a[:] = 7.0
    view = a[1:3, 2:]
    del a
    gc.collect()
    assert pool._cached == 0  # the view still holds the lease
    b = np.frombuffer(_lib._Lease(pool.take(160), pool), dtype=np.float64).reshape(4, 5)
    b[:] = -1.0
    assert np.all(view == 7.0)  # b did not get the live view's memory
    del view, b
    gc.collect()
    assert pool._cached == 320
    c = _lib.new_image((3, 7), np.float32)
    assert c.flags.c_contiguous and c.flags.writeable and c.dtype == np.float32 and c.shape == (3, 7)
    # large buffers: whole-page anonymous mappings, page-locked where a GPU is present
    # (fsr_pin_host; without one the engine simply stages), unlocked when dropped
    big = _lib._OutputPool(max_cached_bytes=0)
    n = big.PIN_MIN * 2
    d = np.frombuffer(_lib._Lease(big.take(n), big), dtype=np.float64)
    assert d.size == n // 8 and d.flags.writeable and d.ctypes.data % 4096 == 0
    d[:] = 3.0
    assert float(d.sum()) == 3.0 * d.size
    del d
    gc.collect()
    assert big._cached == 0  # over the cache limit: unpinned and unmapped
