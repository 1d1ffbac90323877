"""Parity of a libls.so variant build against the oracle on a few shapes (for A/B builds that the
GPU tests, which load the in-tree library, do not exercise):
    python tools/ab_parity.py <lib.so> [d,p,n_el...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1809_10026_b200 as ls
ls.load_library(os.path.abspath(sys.argv[1]))
from oracle import univariate as uv, fd
import synth
cases = [[int(v) for v in a.split(",")] for a in sys.argv[2:]] or [[3, 6, 128, 2, 3, 4], [2, 6, 128, 130, 3],
                                                                    [3, 3, 64, 5, 6, 7], [2, 2, 96, 96, 5]]
worst = 0.0
for c in cases:
    d, p, ne = c[0], c[1], c[2:]
    ctx = ls.Context(d, p, ne)
    r = synth.residual(ctx.shape, 7)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    fdd = fd.setup([uv.space_factors(n, p) for n in ne[:d]], uv.time_factors(ne[d], p))
    zr = fd.fd_apply(r, fdd)
    e = float(np.linalg.norm(z - zr) / np.linalg.norm(zr))
    worst = max(worst, e)
    print(os.path.basename(sys.argv[1]), c, f"{e:.3e}")
print("PARITY", "OK" if worst <= 1e-9 else "FAIL", f"{worst:.3e}")
