"""Near-tie statistics of the reference's fp64 greedy loop, per block, for
calibrating the fp32 guard (CPU, numpy; the loop is _kernels.py:62-126).

For every block and iteration k the top-2 objectives b1 >= b2 are taken the way
the kernels' guard sees them (the exact conjugate mirror of b1 excluded while
the state is Hermitian).  Per block it records the minimum over iterations of

    r1 = (b1 - b2) / b1                   relative gap (the tau test)
    r2 = (b1 - b2) / sqrt(b1 * B0)        gap against the initial scale B0 = b1 at k = 0

An fp32 residual carries an absolute error set by the largest values it has
held (~eps32 * sqrt(B0)), so r2 is the scale-aware near-tie measure.

    python tools/guard_scale_study.py <npz-out> <frame> N I [max-blocks]
      frame: acc6 | c1 | noise256 | 1080p
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import port as oracle  # noqa: E402  (checker only)


def frame(name):
    if name == "acc6":
        from conftest import golden_image
        d = golden_image("acc6_512_s16")
        return d["sampled"], d["mask"]
    if name == "c1":
        img = oracle.synthetic_frame(256, 256, 7, "natural")
    elif name == "noise256":
        img = oracle.synthetic_frame(256, 256, 3, "uniform")
    elif name == "1080p":
        img = oracle.synthetic_frame(1080, 1920, 11, "natural")
    elif name in ("4k", "4k1080"):  # bench.py's frames (synth.frame seed 7)
        from paper_2202_13926_b200 import frames, synth
        H, W = (2160, 3840) if name == "4k" else (1080, 1920)
        img = synth.frame(H, W, 7, "natural")
        mask = frames.quarter_sample_mask(H, W, 42)
        return np.where(mask, img, 0.0), mask
    elif name[:3] in ("nat", "uni") and "-" in name:  # e.g. nat640x480-5
        size, seed = name[3:].split("-")
        h, w = (int(x) for x in size.split("x"))
        img = oracle.synthetic_frame(h, w, int(seed), "natural" if name[:3] == "nat" else "uniform")
    else:
        raise SystemExit(f"unknown frame {name}")
    return oracle.quarter_sample(img, 42)


def study(px, mask, B, N, I, rho=0.7, gamma=0.5, which=None, batch=256):
    L = (N - B) // 2
    n = N * N
    wf = oracle.frequency_weight(N).ravel()
    kk = np.arange(n)
    ku, kv = np.divmod(kk, N)
    mir = oracle.mirror_index(kk, N)
    selfm = mir == kk
    nb_all = len(which)
    r1 = np.full(nb_all, np.inf)
    r2 = np.full(nb_all, np.inf)
    k1 = np.zeros(nb_all, np.int32)
    k2 = np.zeros(nb_all, np.int32)
    for lo in range(0, nb_all, batch):
        ids = which[lo:lo + batch]
        R0, W, _, _ = oracle.block_spectra(px, mask, B, L, rho, ids)
        R = R0.reshape(len(ids), n).copy()
        Wf = W.reshape(len(ids), n)
        w00 = Wf[:, 0].real
        live = w00 > 0
        herm = np.ones(len(ids), bool)
        B0 = None
        ar = np.arange(len(ids))
        for it in range(I):
            obj = wf * (R.real ** 2 + R.imag ** 2)
            i1 = np.argmax(obj, axis=1)
            b1 = obj[ar, i1]
            if B0 is None:
                B0 = np.maximum(b1, 1e-300)
            o2 = obj.copy()
            o2[ar, i1] = -1.0
            m1 = mir[i1]
            ex = herm & (m1 != i1)
            o2[ar[ex], m1[ex]] = -1.0
            b2 = o2.max(axis=1)
            gap = b1 - b2
            a = np.where(live & (b1 > 0), gap / np.maximum(b1, 1e-300), np.inf)
            b = np.where(live & (b1 > 0), gap / np.sqrt(np.maximum(b1 * B0, 1e-300)), np.inf)
            upd = a < r1[lo:lo + len(ids)]
            r1[lo:lo + len(ids)][upd] = a[upd]
            k1[lo:lo + len(ids)][upd] = it
            upd = b < r2[lo:lo + len(ids)]
            r2[lo:lo + len(ids)][upd] = b[upd]
            k2[lo:lo + len(ids)][upd] = it
            herm &= selfm[i1]
            # update: R -= gp * W[(k - s) mod N] (the reference's order of operations)
            c = R[ar, i1]
            gp = gamma * (c.real / w00 + 1j * (c.imag / w00))
            su, sv = ku[i1], kv[i1]
            idx = ((ku[None, :] - su[:, None]) % N) * N + (kv[None, :] - sv[:, None]) % N
            R = np.where(live[:, None], R - gp[:, None] * np.take_along_axis(Wf, idx, 1), R)
    return r1, r2, k1, k2


def main():
    out, name, N, I = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    maxb = int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 30
    px, mask = frame(name)
    B = 4
    H, W = px.shape
    nb = (-(-H // B)) * (-(-W // B))
    which = np.arange(nb)
    if nb > maxb:
        which = np.sort(np.random.default_rng(0).choice(nb, maxb, replace=False))
    r1, r2, k1, k2 = study(px, mask, B, N, I, which=which)
    np.savez_compressed(out, which=which, r1=r1, r2=r2, k1=k1, k2=k2, N=N, I=I, frame=name)
    for t in (5e-5, 1.2e-4):
        for kap in (0, 1e-9, 3e-9, 1e-8, 3e-8, 1e-7):
            f = np.mean((r1 < t) | (r2 < kap))
            print(f"{name} N={N} I={I} tau={t:g} kappa={kap:g}: flagged {100 * f:.2f} %")


if __name__ == "__main__":
    main()
