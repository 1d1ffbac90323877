"""Minimal driver for ncu: set up BASELINE config C and run fd_apply R times.

    python tools/profile_fd.py --config 4 --reps 2 [--matvec]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1809_10026_b200 as ls
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--matvec", action="store_true")
ap.add_argument("--pcg", action="store_true")
ap.add_argument("--p", type=int, default=None)
ap.add_argument("--mv", type=int, default=0, help="ls_tune matvec variant")
ap.add_argument("--fdk", type=int, default=0, help="ls_tune FD kernel variant")
ap.add_argument("--pad", type=int, default=0, help="ls_tune v3 matvec padding")
ap.add_argument("--nograph", action="store_true", help="PCG as the host-driven loop (profilers see every kernel)")
ap.add_argument("--tune", default="", help="extra ls_tune knobs, 'knob=value,...'")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
p = a.p if a.p is not None else (c["p"] if isinstance(c["p"], int) else c["p"][0])
ctx = ls.Context(c["d"], p, [c["n_el"]] * (c["d"] + 1))
ctx.tune(2, a.mv)
ctx.tune(1, a.fdk)
if a.pad:
    ctx.tune(3, a.pad)
if a.nograph:
    ctx.tune(5, 0)
for kv in filter(None, a.tune.split(",")):
    k, v = kv.split("=")
    ctx.tune(int(k), int(v))
r = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
z = torch.empty_like(r)
if a.pcg:
    b = ctx.rhs(1)
    for _ in range(a.reps):
        x, st = ctx.pcg(b, tol=1e-8)
    print(st)
for _ in range(0 if a.pcg else a.reps):
    if a.matvec:
        ctx.matvec(r, z)
    else:
        ctx.fd_apply(r, z)
torch.cuda.synchronize()
print("ok", ctx.launches, float(z.abs().max()))
