"""A/B timing of the FD mode-kernel variants (ls_tune knob 1) on BASELINE configs.

    python tools/fd_variants.py [--configs 3 4] [--reps 10]
Prints per config and variant: fd_apply ms (CUDA events, inputs > L2 or L2 flushed),
mode-kernel TF/s (algorithmic), and the relative difference between the variants.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1809_10026_b200 as ls
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="+", default=["3", "4", "5:8", "5:2"])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--variants", nargs="+", type=int, default=[0, 1])
a = ap.parse_args()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
for cs in a.configs:
    cid, _, pp = cs.partition(":")
    c = synth.CONFIGS[int(cid)]
    p = int(pp) if pp else c["p"]
    d, ne = c["d"], c["n_el"]
    ctx = ls.Context(d, p, [ne] * (d + 1))
    s = torch.cuda.current_stream()
    ctx.set_stream(s)
    r = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    outs = {}
    for v in a.variants:
        ctx.tune(1, v)
        z = torch.empty_like(r)
        for _ in range(3):
            ctx.fd_apply(r, z)
        torch.cuda.synchronize()
        ctx.profile_read()
        ctx.profile(True)
        tot = 0.0
        for _ in range(a.reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.fd_apply(r, z)
            e1.record(s)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        ctx.profile(False)
        kms, kfl, kn = ctx.profile_read()
        ms = tot / a.reps
        n_s, n_t = ne + p - 2, ne + p - 1
        fl = 4.0 * ctx.N * (d * n_s + n_t)
        outs[v] = z
        print(json.dumps({"config": cs, "variant": v, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 3),
                          "frac_of_37": round(fl / ms / 1e9 / 37.0, 4),
                          "mode_kernel_tflops": round(kfl / kms / 1e9, 3)}), flush=True)
    if len(outs) > 1:
        v0 = a.variants[0]
        for v in a.variants[1:]:
            rel = float(torch.linalg.norm(outs[v] - outs[v0]) / torch.linalg.norm(outs[v0]))
            print(json.dumps({"config": cs, "rel_diff": rel, "variants": [v0, v]}))
    ctx.close()
    del r, outs
    torch.cuda.empty_cache()
