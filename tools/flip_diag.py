"""Diagnose fp32-vs-fp64 sequence differences block by block."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_13926_b200 as fsr
from paper_2202_13926_b200 import synth, frames

img = synth.frame(256, 256, 7)
mask = frames.quarter_sample_mask(256, 256, 42)
px = np.where(mask, img, 0.0)
o32, t32 = fsr.reconstruct(px, mask, 4, 32, 100, precision="fp32_unguarded", return_trace=True)
o64, t64 = fsr.reconstruct(px, mask, 4, 32, 100, precision="fp64", return_trace=True)
s32, s64 = t32.selections, t64.selections
def mirror(s):
    u, v = np.divmod(s, 32); return ((-u) % 32) * 32 + (-v) % 32
eq = np.all(s32 == s64, 1); mi = np.all(s32 == mirror(s64), 1)
flip = np.nonzero(~(eq | mi))[0]
print("blocks", len(s32), "equal", eq.sum(), "mirror", (mi & ~eq).sum(), "flipped", len(flip))
for b in flip[:8]:
    d = np.nonzero((s32[b] != s64[b]) & (s32[b] != mirror(s64[b])))[0]
    f = int(d[0])
    print(f"block {b}: first diff at it {f}")
    print("  fp32:", [divmod(int(x), 32) for x in s32[b, max(0, f - 3):f + 6]])
    print("  fp64:", [divmod(int(x), 32) for x in s64[b, max(0, f - 3):f + 6]])
# per-iteration position of first difference histogram
firsts = []
for b in flip:
    d = np.nonzero((s32[b] != s64[b]) & (s32[b] != mirror(s64[b])))[0]
    firsts.append(int(d[0]))
print("first-diff iteration histogram:", np.bincount(np.array(firsts) // 10, minlength=10))
# partial mirror: sequences equal up to f then mirrored after?
pm = 0
for b in flip:
    x, y = s32[b], s64[b]
    d = np.nonzero(x != y)[0][0]
    if np.all(x[d:] == mirror(y[d:])):
        pm += 1
print("flipped blocks that are 'equal then mirrored':", pm)
