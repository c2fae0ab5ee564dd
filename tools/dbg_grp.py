import sys, os, math, numpy as np, torch
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import oracle as orc
import test_gpu_group as T
from paper_2605_02262_b200 import wq
wq.load()
d, S = 128, 32
c = T.edge_case(d, S, 250.0, 3 * d + S)
offs, packed, out, part = T.run(c)
opk, ooffs, ref, rpart = T.oracle(orc, c)
err = np.abs(out - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
b, hq = np.unravel_index(np.argmax(err), err.shape)
print("worst", b, hq, err[b, hq], "h", hq // 7)
print("gpu", out[b, hq, :8]); print("ref", ref[b, hq, :8])
print("gpu part m,l", part[b, hq, :2], "ref", rpart[b, hq, :2])
print("rows err>2e-3:", np.argwhere(err > 2e-3).tolist())
h = hq // 7
print("kinds K of (b,h):", [T.KINDS[(w + h + b) % 8] for w in range(8)])
print("kinds V of (b,h):", [T.KINDS[(w + 3 * h + b + 1) % 8] for w in range(8)])
print("perm", c["perm"][b], "seg", c["seg"][b])
# per-window logit maxima (fp64 from dequantized oracle records)
og = orc.geom(c["B"], c["H"], c["Hq"], d, c["M"], S, list(T.CLASS))
