"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs only in the build container, where the reference package is mounted
read-only at /root/reference (it is imported, never copied):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every array written here is an output of fsrkit 0.1.0's own functions
(``_kernels.reconstruct_iterations``, ``reconstruction.reconstruct_image``,
``reconstruction.reconstruct_block_full``, ``weights.*``, ``sampling.*``) on
seeded inputs, so the fixtures pin both the oracle (tests/test_oracle.py) and,
on the GPU box, the CUDA engine (tests/test_gpu_*.py).
"""

from __future__ import annotations

import os
import sys
import types

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from fsrkit import _kernels  # noqa: E402
from fsrkit.core import FsrParams, GrayImage, block_partition  # noqa: E402
from fsrkit.metrics import psnr  # noqa: E402
from fsrkit.reconstruction import reconstruct_block_full, reconstruct_image  # noqa: E402
from fsrkit.sampling import (SampledImage, extract_support_block, mean_fill,  # noqa: E402
                             quarter_sample, splitmix64)
from fsrkit.weights import _decay_grid, build_weight_set, frequency_weight  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.port import make_natural_image  # noqa: E402  (restated fixture; checked below)


def ref_natural(size, seed):
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import make_natural_image as ref_make
    return ref_make(size, seed).pixels


def loop_case(R0, W, wf, gamma, iterations, use_tree, thr=0.0):
    R = R0.copy()
    G = np.zeros_like(R0)
    n = max(iterations, 1)
    obj = np.zeros(n)
    sel = np.zeros(n, np.int64)
    ties = np.zeros(n, np.uint8)
    done = _kernels.reconstruct_iterations(R, G, W, np.ascontiguousarray(wf).ravel(), gamma,
                                           iterations, 32, use_tree, thr, obj, sel, ties)
    return dict(R=R, G=G, obj=obj[:done], sel=sel[:done], ties=ties[:done], done=done)


def make_loop_fixtures():
    rng = np.random.default_rng(20240811)
    out = {}
    cases = []
    # (support, block, iterations, reducers, kind)
    for support, iters, reducers in ((4, 20, ("tree", "linear")), (6, 20, ("tree", "linear")),
                                     (8, 40, ("tree", "linear")), (16, 64, ("tree", "linear")),
                                     (32, 100, ("tree", "linear")), (64, 60, ("linear",))):
        for trial in range(3):
            if trial == 2 and support <= 32:
                # uniform image block quarter-sampled (tie-rich for small S)
                img = GrayImage(np.full((support, support), 100.0))
            else:
                img = GrayImage(rng.uniform(0.0, 255.0, (support, support)))
            sampled = quarter_sample(img, 1000 + 7 * trial + support)
            sig = sampled.image.pixels
            ws = build_weight_set(support, 0.7, sampled.mask)
            R0 = np.fft.fft2(sig * ws.spatial)
            for red in reducers:
                r = loop_case(R0, ws.spectrum, ws.frequency, 0.5, iters, red == "tree")
                key = f"S{support}_t{trial}_{red}"
                cases.append(key)
                out[key + "_R0"] = R0
                out[key + "_W"] = ws.spectrum
                out[key + "_wf"] = ws.frequency
                out[key + "_iters"] = np.array(iters)
                for k, v in r.items():
                    out[key + "_" + k] = np.asarray(v)
    # early stop case: thr from the reference's own rule (reconstruction.py:180-184)
    support = 16
    img = GrayImage(rng.uniform(0.0, 255.0, (support, support)))
    sampled = quarter_sample(img, 5)
    ws = build_weight_set(support, 0.7, sampled.mask)
    sig = sampled.image.pixels
    R0 = np.fft.fft2(sig * ws.spatial)
    thr = 1e-3 * float(np.sum(sig * sig * ws.spatial))  # aggressive so it triggers
    r = loop_case(R0, ws.spectrum, ws.frequency, 1.0, 200, True, thr)
    key = "S16_early_tree"
    cases.append(key)
    out[key + "_R0"] = R0
    out[key + "_W"] = ws.spectrum
    out[key + "_wf"] = ws.frequency
    out[key + "_iters"] = np.array(200)
    out[key + "_thr"] = np.array(thr)
    out[key + "_gamma"] = np.array(1.0)
    for k, v in r.items():
        out[key + "_" + k] = np.asarray(v)
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "loop_cases.npz"), **out)
    print("loop cases:", len(cases))


def image_case(name, pixels, mask_seed, block, border, iterations, reducers=("tree",),
               trace_blocks=False, early_stop=False, mask=None, recipe=None):
    img = GrayImage(pixels)
    if mask is None:
        sampled = quarter_sample(img, mask_seed)
    else:
        sampled = SampledImage(GrayImage(np.where(mask, pixels, 0.0)), mask)
    params = FsrParams(block=block, border=border, rho=0.7, gamma=0.5, iterations=iterations,
                       threads=os.cpu_count() or 1)
    d = dict(block=np.array(block), border=np.array(border), iterations=np.array(iterations),
             early_stop=np.array(early_stop), mask_seed=np.array(mask_seed))
    if recipe is None:
        d.update(sampled=sampled.image.pixels, mask=sampled.mask, original=img.pixels)
    else:
        # large inputs are regenerated by the restated generators (pinned by
        # test_oracle against the stored mask checksum and these arrays)
        kind, h, w, seed = recipe
        d.update(recipe_kind=np.array(kind), recipe_shape=np.array([h, w]),
                 recipe_seed=np.array(seed),
                 mask_packed=np.packbits(sampled.mask),
                 sampled_sum=np.array(float(sampled.image.pixels.sum())))
    for red in reducers:
        res = reconstruct_image(sampled, params, reducer=red, early_stop=early_stop)
        d["out_" + red] = res.pixels
        d["psnr_" + red] = np.array(psnr(img, res).psnr_db)
    if mask is None or np.any(mask):
        d["psnr_meanfill"] = np.array(psnr(img, mean_fill(sampled)).psnr_db)
    if trace_blocks:
        # per-block selection sequences via the traced per-block API
        # (reconstruction.py:159-203), the reference's only sequence oracle
        s = params.support
        descs = block_partition(*sampled.shape, params)
        for red in reducers:
            sel = np.zeros((len(descs), iterations), np.int16)
            for i, desc in enumerate(descs):
                blk = extract_support_block(sampled, desc, s)
                ws = build_weight_set(s, 0.7, blk.mask)
                r = reconstruct_block_full(blk, ws, params, red)
                sel[i, :r.iterations_run] = r.selections
            d["sel_" + red] = sel
    np.savez_compressed(os.path.join(HERE, f"image_{name}.npz"), **d)
    print(name, {k: float(v) for k, v in d.items() if k.startswith("psnr")})


def make_image_fixtures():
    nat = ref_natural(256, 7)
    assert np.array_equal(nat, make_natural_image(256, 7)), "restated natural image differs"
    # C1 natural (BASELINE config 1): N=32, I=100, both reducers, per-block sequences
    image_case("c1_natural", nat, 42, 4, 14, 100, ("tree", "linear"), trace_blocks=True,
               recipe=("natural", 256, 256, 7))
    # C1 uniform
    uni = np.random.default_rng(1).uniform(0, 255, (256, 256))
    image_case("c1_uniform", uni, 42, 4, 14, 100, ("tree", "linear"), trace_blocks=True,
               recipe=("uniform", 256, 256, 1))
    # odd, non-square shapes with truncated edge tiles, other supports
    rng = np.random.default_rng(77)
    odd = ref_natural(64, 3)[:37, :53]
    image_case("odd_37x53_s16", odd, 9, 4, 6, 60, ("tree", "linear"), trace_blocks=True)
    image_case("odd_37x53_s8_b2", odd, 10, 2, 3, 30, ("tree", "linear"), trace_blocks=True)
    image_case("odd_29x31_s12_b6", rng.uniform(0, 255, (29, 31)), 11, 6, 3, 40, ("tree",),
               trace_blocks=True)
    # early stop on
    image_case("early_48x40_s16", ref_natural(48, 4)[:, :40], 12, 4, 6, 200, ("tree",),
               early_stop=True)
    # empty-support region: mask only in the left third -> right blocks fall back to mean
    px = ref_natural(64, 5)[:40, :64]
    m = quarter_sample(GrayImage(px), 13).mask.copy()
    m[:, 24:] = False
    image_case("emptysupport_40x64_s8", px, 0, 4, 2, 30, ("tree",), mask=m)
    # acceptance 6 golden (SPEC default params): 512^2 natural, N=16, I=200
    image_case("acc6_512_s16", make_natural_image(512, 7), 42, 4, 6, 200, ("tree",),
               recipe=("natural", 512, 512, 7))


def make_kats():
    d = {}
    d["splitmix64_seed0"] = splitmix64(0, 16)
    d["splitmix64_seed42"] = splitmix64(42, 16)
    for s in (4, 6, 8, 12, 16, 32, 64):
        d[f"wf_{s}"] = frequency_weight(s)
        d[f"decay_{s}"] = _decay_grid(s, 0.7)
    d["mask_48x64_seed3"] = quarter_sample(GrayImage(np.ones((48, 64))), 3).mask
    d["mask_33x35_seed8"] = quarter_sample(GrayImage(np.ones((33, 35))), 8).mask
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **d)
    print("kats:", len(d))


def make_spatial_fixtures():
    """oracle.oracle_reconstruct_traced (the reference's FFT-free spatial-domain
    oracle, oracle.py:25-132) on quarter-sampled random blocks, the way the
    reference's acceptance criterion 1 draws them (test_acceptance.py:32-91,
    conftest.random_quarter_block): S = 4, 8, 16, 32 iterations."""
    from fsrkit.core import SampledBlock
    from fsrkit.oracle import oracle_reconstruct_traced
    rng = np.random.default_rng(1001)
    d = {}
    for support, block_size, border in ((4, 2, 1), (8, 2, 3), (16, 4, 6)):
        params = FsrParams(block=block_size, border=border, rho=0.7, gamma=0.5, iterations=32)
        cols = {k: [] for k in ("signal", "mask", "spatial", "output", "objectives",
                                "selections", "ties", "energies")}
        for trial in range(12):
            image = GrayImage(rng.uniform(0.0, 255.0, (support, support)))
            sampled = quarter_sample(image, trial * 31 + support)
            block = SampledBlock(signal=np.where(sampled.mask, image.pixels, 0.0), mask=sampled.mask)
            ws = build_weight_set(support, 0.7, block.mask)
            run = oracle_reconstruct_traced(block, ws, params)
            for k, v in (("signal", block.signal), ("mask", block.mask), ("spatial", ws.spatial),
                         ("output", run.output), ("objectives", run.objectives),
                         ("selections", run.selections), ("ties", run.ties),
                         ("energies", run.energies)):
                cols[k].append(np.asarray(v))
        for k, v in cols.items():
            d[f"s{support}_{k}"] = np.stack(v)
        d[f"s{support}_wf"] = frequency_weight(support)
        d[f"s{support}_params"] = np.array([block_size, border, 32], np.int64)
    np.savez_compressed(os.path.join(HERE, "spatial_oracle.npz"), **d)
    print("spatial oracle:", len(d))


if __name__ == "__main__":
    make_kats()
    make_loop_fixtures()
    make_image_fixtures()
    make_spatial_fixtures()
