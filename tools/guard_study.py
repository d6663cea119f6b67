"""Guard study (GPU): how small a near-tie gap must be to flip the fp32 greedy
path, and what each tau costs in fp64 re-runs.

For each test frame: fp32 (top-2 tracking, no re-run) with per-block minimum
relative top-2 gap + selections, and fp64 validation with selections.  Blocks
whose fp32 sequence differs from fp64 modulo the conjugate mirror are
"flipped"; for candidate tau we report the re-run fraction and the worst
pixel error left in unflagged blocks (tolerance 0.255 on the 0..255 scale).
"""
import ctypes
import json
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_13926_b200 import _lib, frames, synth  # noqa: E402

L = _lib.load()
L.fsr_debug_guard_gaps.argtypes = [ctypes.c_void_p, ctypes.POINTER(_lib.FsrParamsC)] + \
    [ctypes.c_void_p] * 2 + [ctypes.c_int64] * 2 + [ctypes.c_void_p] * 3
L.fsr_debug_guard_gaps.restype = ctypes.c_int


def mirror(sel, N=32):
    u, v = np.divmod(sel, N)
    return ((-u) % N) * N + (-v) % N


def study(name, img, B=4, N=32, I=100, reducer="tree"):
    H, W = img.shape
    mask = frames.quarter_sample_mask(H, W, 42)
    px = np.where(mask, img, 0.0)
    eng = _lib.default_engine([0])
    nb = frames.n_blocks(H, W, B)
    p32 = _lib.make_params(B, (N - B) // 2, I, reducer=reducer, precision="fp32_unguarded", argmax="redux")
    out32 = np.empty((H, W), np.float32)
    gaps2 = np.empty((nb, 2), np.float32)
    sel32 = np.empty((nb, I), np.int32)
    px32 = px.astype(np.float32)
    m8 = mask.astype(np.uint8)
    rc = L.fsr_debug_guard_gaps(eng._h, ctypes.byref(p32), _lib._ptr(px32), _lib._ptr(m8), H, W,
                                _lib._ptr(out32), _lib._ptr(gaps2), _lib._ptr(sel32))
    assert rc == 0, L.fsr_last_error(eng._h)
    p64 = _lib.make_params(B, (N - B) // 2, I, reducer=reducer, precision="fp64")
    sel64 = np.empty((nb, I), np.int32)
    out64 = eng.reconstruct(px, mask, p64, sel64, None)
    gaps, gapsc = gaps2[:, 0], gaps2[:, 1]  # min relative gap, first flagged iteration
    eq = np.all(sel32 == sel64, axis=1) | np.all(sel32 == mirror(sel64, N), axis=1)
    flipped = ~eq
    # per-block max error
    bc = -(-W // B)
    err = np.abs(out32.astype(np.float64) - out64)
    eb = np.zeros(nb)
    hh = -(-H // B) * B
    ww = bc * B
    pad = np.zeros((hh, ww))
    pad[:H, :W] = err
    eb = pad.reshape(hh // B, B, bc, B).max(axis=(1, 3)).ravel()
    res = {"name": name, "blocks": int(nb), "flipped": int(flipped.sum()),
           "max_err_all": float(eb.max()),
           "flipped_gap_max": float(gaps[flipped].max()) if flipped.any() else None,
           "flipped_gap_q": [float(np.quantile(gaps[flipped], q)) for q in (0.5, 0.9, 0.99)]
           if flipped.any() else None,
           "unflipped_err_max": float(eb[~flipped].max()) if (~flipped).any() else None}
    tau_rows = []
    for tau in (1e-6, 3e-6, 1e-5, 2e-5, 5e-5, 1e-4, 2e-4):
        flag = gaps < tau
        left = eb[~flag]
        tau_rows.append({"tau": tau, "rerun_frac": float(flag.mean()),
                         "max_err_unflagged": float(left.max()) if left.size else 0.0,
                         "flipped_unflagged": int((flipped & ~flag).sum())})
    res["tau"] = tau_rows
    # first flagged iteration (relative gap < guard_tau = 5e-5) of the flagged
    # blocks: how long a prefix of each re-run is already decided in fp32
    t0 = gapsc[gapsc < 1e8].astype(np.int64)
    res["first_flag_iteration"] = {
        "flagged": int(t0.size), "tau": 5e-5,
        "quantiles": {str(q): float(np.quantile(t0, q)) for q in (0.1, 0.25, 0.5, 0.75, 0.9)}
        if t0.size else None,
        "mean_prefix_fraction": float(t0.mean() / I) if t0.size else None,
        "histogram_by_decile": np.bincount(np.minimum(t0 * 10 // I, 9), minlength=10).tolist()
        if t0.size else None}
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    out = []
    out.append(study("nat256", synth.frame(256, 256, 7)))
    out.append(study("uni256", synth.frame(256, 256, 1, "uniform")))
    out.append(study("nat1080", synth.frame(1080, 1920, 7)))
    out.append(study("uni1080", synth.frame(1080, 1920, 3, "uniform")))
    out.append(study("nat1080_s11", synth.frame(1080, 1920, 11)))
    out.append(study("uni1080_s5", synth.frame(1080, 1920, 5, "uniform")))
    out.append(study("nat4k", synth.frame(2160, 3840, 7)))
    with open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/guard_study.json", "w") as f:
        json.dump(out, f, indent=1)
