"""Re-run one fp64 divergence of tools/stress_parity.py and compare the fp64
kernels: the segmented warpsegd / warpnd (FSR_NO_SEG) / generic paths."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import port as oracle  # noqa: E402

import paper_2202_13926_b200 as fsr  # noqa: E402


def main():
    H, W, N, B, I, rho, gamma, red, kind, iseed, mseed, blk = sys.argv[1:13]
    H, W, N, B, I, iseed, mseed, blk = (int(x) for x in (H, W, N, B, I, iseed, mseed, blk))
    rho, gamma = float(rho), float(gamma)
    img = oracle.synthetic_frame(H, W, iseed, kind)
    sampled, mask = oracle.quarter_sample(img, mseed)
    sampled = np.where(mask, sampled, 0.0)
    L = (N - B) // 2
    ref, rtr = oracle.reconstruct_image(sampled, mask, B, L, I, rho, gamma, red, trace=True)
    out, tr = fsr.reconstruct(sampled, mask, B, N, I, rho, gamma, reducer=red, precision="fp64",
                              return_trace=True)
    s_ref = rtr["sel"][blk][:I]
    s_gpu = tr.selections[blk][:I]
    d = np.nonzero(s_ref != s_gpu)[0]
    dm = np.nonzero(s_ref != oracle.mirror_index(s_gpu, N))[0]
    print("first diff identity", d[:3], "mirror", dm[:3])
    f = int(max(d[0] if d.size else I, dm[0] if dm.size else I))
    print("ref ", s_ref[max(0, f - 3):f + 4])
    print("gpu ", s_gpu[max(0, f - 3):f + 4])
    # the reference's objectives at iteration f along its own path
    R0, Wsp, _, _ = oracle.block_spectra(sampled, mask, B, L, rho, [blk])
    wf = oracle.frequency_weight(N).ravel()
    R = R0[0].copy(); G = np.zeros_like(R)
    oracle.reconstruct_iterations(R, G, Wsp[0], wf, gamma, f, red == "tree")
    obj = wf * (R.real.ravel() ** 2 + R.imag.ravel() ** 2)
    top = np.argsort(-obj)[:4]
    print("ref objectives at f:", [(int(t), float(obj[t])) for t in top])
    print("gpu choice at f:", int(s_gpu[f]), float(obj[int(s_gpu[f])]))


if __name__ == "__main__":
    main()
