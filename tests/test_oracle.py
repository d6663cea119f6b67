"""Pin the CPU oracle to the reference's own golden vectors (CPU-only).

The fixtures in tests/golden/ were produced by fsrkit 0.1.0 itself
(tests/golden/make_golden.py).  Everything here must hold bitwise: the oracle
is the parity checker for the CUDA engine, so it has to BE the reference.
"""

import numpy as np
import pytest

from conftest import golden_image, load_golden
from oracle import port as oracle


def reference_splitmix64(seed, count):
    # plain-integer restatement, as in pkg/tests/test_sampling.py:11-21
    M = (1 << 64) - 1
    out, state = [], seed & M
    for _ in range(count):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        out.append(z ^ (z >> 31))
    return out


def test_splitmix64_kat():
    k = load_golden("kats.npz")
    assert int(oracle.splitmix64(0, 1)[0]) == 0xE220A8397B1DCDAF  # test_sampling.py:30-32
    assert np.array_equal(oracle.splitmix64(0, 16), k["splitmix64_seed0"])
    assert np.array_equal(oracle.splitmix64(42, 16), k["splitmix64_seed42"])
    for seed in (0, 1, 42, 2**63, -1, 0xDEADBEEF):
        assert [int(v) for v in oracle.splitmix64(seed, 16)] == reference_splitmix64(seed, 16)


def test_quarter_sample_masks_match_reference():
    k = load_golden("kats.npz")
    assert np.array_equal(oracle.quarter_sample_mask((48, 64), 3), k["mask_48x64_seed3"])
    assert np.array_equal(oracle.quarter_sample_mask((33, 35), 8), k["mask_33x35_seed8"])
    m = oracle.quarter_sample_mask((33, 35), 8)
    assert m.sum() == 17 * 18  # exactly one per (possibly truncated) cell


@pytest.mark.parametrize("s", [4, 6, 8, 12, 16, 32, 64])
def test_weight_tables_bitwise(s):
    k = load_golden("kats.npz")
    assert np.array_equal(oracle.frequency_weight(s), k[f"wf_{s}"])
    assert np.array_equal(oracle.decay_grid(s, 0.7), k[f"decay_{s}"])
    wf = oracle.frequency_weight(s)
    assert wf[0, 0] == 1.0 and abs(wf[s // 2, s // 2]) <= 1e-12


def _loop_cases():
    d = load_golden("loop_cases.npz")
    return d, [str(c) for c in d["cases"]]


@pytest.mark.parametrize("case", _loop_cases()[1])
def test_loop_bitwise_vs_reference(case):
    d, _ = _loop_cases()
    R = d[case + "_R0"].copy()
    G = np.zeros_like(R)
    W = d[case + "_W"]
    wf = d[case + "_wf"]
    iters = int(d[case + "_iters"])
    gamma = float(d.get(case + "_gamma", 0.5))
    thr = float(d.get(case + "_thr", 0.0))
    use_tree = case.endswith("_tree")
    done, obj, sel, ties = oracle.reconstruct_iterations(R, G, W, wf, gamma, iters, use_tree, thr)
    assert done == int(d[case + "_done"])
    assert np.array_equal(sel, d[case + "_sel"])
    assert np.array_equal(obj, d[case + "_obj"])  # bitwise
    assert np.array_equal(ties, d[case + "_ties"].astype(bool))
    assert np.array_equal(R, d[case + "_R"])
    assert np.array_equal(G, d[case + "_G"])


def test_tree_rank_closed_form(rng):
    """tree argmax == min (bitrev5(g), bitrev5(lane)) among the maxima."""
    for s in (4, 8, 16, 32):
        rank = oracle.tree_rank(s)
        for _ in range(200):
            v = rng.integers(0, 4, s * s).astype(np.float64)  # tie-heavy
            o, t = oracle.tree_argmax(v)
            m = v.max()
            cand = np.nonzero(v == m)[0]
            assert o == m and t == cand[np.argmin(rank[cand])]
            o2, t2 = oracle.linear_argmax(v)
            assert t2 == cand[0]


SMALL_IMAGES = ["odd_37x53_s16", "odd_37x53_s8_b2", "odd_29x31_s12_b6", "early_48x40_s16",
                "emptysupport_40x64_s8"]


@pytest.mark.parametrize("name", SMALL_IMAGES + ["c1_natural"])
def test_image_bitwise_vs_reference(name):
    d = golden_image(name)
    for red in ("tree", "linear"):
        if "out_" + red not in d:
            continue
        out = oracle.reconstruct_image(d["sampled"], d["mask"], int(d["block"]), int(d["border"]),
                                       int(d["iterations"]), 0.7, 0.5, red,
                                       bool(d["early_stop"]))
        assert np.array_equal(out, d["out_" + red]), f"{name}/{red}"
        assert oracle.psnr(d["original"], out) == float(d["psnr_" + red])


@pytest.mark.parametrize("name", ["odd_37x53_s16", "odd_37x53_s8_b2", "odd_29x31_s12_b6"])
def test_traced_sequences_vs_reference(name):
    d = golden_image(name)
    for red in ("tree", "linear"):
        if "sel_" + red not in d:
            continue
        _, tr = oracle.reconstruct_image(d["sampled"], d["mask"], int(d["block"]),
                                         int(d["border"]), int(d["iterations"]), 0.7, 0.5, red,
                                         trace=True)
        assert np.array_equal(tr["sel"].astype(np.int16), d["sel_" + red])


def test_mirror_comparator():
    s = 8
    a = np.array([[0, 9, 55, 3]])
    b = oracle.mirror_index(a, s)
    counts, div = oracle.compare_sequences(a, b, s)
    assert counts == {"equal": 0, "mirror": 1, "diverged": 0}
    counts, _ = oracle.compare_sequences(a, a, s)
    assert counts["equal"] == 1


def _spatial_restated(signal, w, wf, gamma, iterations):
    """numpy restatement of fsrkit.oracle._step (oracle.py:66-98): explicit basis
    images, direct-summation projection, first maximum, recompute from scratch."""
    s = signal.shape[0]
    t = np.arange(s * s)
    k, l = t // s, t % s
    phi = np.exp(1j * 2.0 * np.pi / s * (np.outer(k, k) + np.outer(l, l)))
    model = np.zeros((s, s), complex)
    rw = signal * w
    w00 = float(np.sum(w))
    sels, objs = [], []
    for _ in range(iterations):
        proj = phi.conj() @ rw.ravel()
        obj = wf.ravel() * (proj.real ** 2 + proj.imag ** 2)
        ti = int(np.argmax(obj))
        sels.append(ti)
        objs.append(float(obj[ti]))
        p = proj[ti] / w00
        model = model + (gamma * p) * phi[ti].reshape(s, s)
        rw = (signal - model) * w
    return np.array(sels), np.array(objs)


def test_spatial_oracle_golden_restated():
    """The GPU spatial oracle's fixtures (fsrkit.oracle output) pinned by a plain
    numpy restatement of the same algorithm (S = 4 and 8, 32 iterations)."""
    from conftest import load_golden
    d = load_golden("spatial_oracle.npz")
    for s in (4, 8):
        k = f"s{s}_"
        for b in range(4):
            sel, obj = _spatial_restated(d[k + "signal"][b], d[k + "spatial"][b], d[k + "wf"], 0.5, 32)
            ref_sel, ref_obj = d[k + "selections"][b], d[k + "objectives"][b]
            diff = np.nonzero(sel != ref_sel)[0]
            upto = 32 if diff.size == 0 else int(diff[0]) + 1
            np.testing.assert_allclose(obj[:upto], ref_obj[:upto], rtol=1e-9, atol=0)
            if diff.size:  # a different branch only at a recorded tie
                assert d[k + "ties"][b][diff[0]]
