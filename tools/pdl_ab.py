"""A/B of programmatic dependent launch of the FD mode kernels (LS_TUNE_PDL): fd_apply and
PCG times with CUDA events, configs 2, 3, 4 (config 4 fd_apply only).

    python tools/pdl_ab.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10026_b200 as ls  # noqa: E402
import synth  # noqa: E402


def ev_time(fn, s, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for cfg, d, p, ne, pcg in ((2, 2, 3, 64, True), (3, 3, 3, 64, True), (4, 3, 6, 128, False)):
    c = ls.Context(d, p, [ne] * (d + 1))
    s = torch.cuda.Stream()
    c.set_stream(s)
    with torch.cuda.stream(s):
        r = torch.from_numpy(synth.residual(c.shape, 0)).cuda()
        z = torch.empty_like(r)
    torch.cuda.synchronize()
    out = {"config": cfg}
    for pdl in (0, 1):
        c.tune(6, pdl)
        for _ in range(3):
            c.fd_apply(r, z)
        out[f"fd_ms_pdl{pdl}"] = ev_time(lambda: c.fd_apply(r, z), s, 20 if cfg != 4 else 10)
        if pcg:
            b = c.rhs(1)
            c.pcg(b)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, st = c.pcg(b)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) * 1e3)
            out[f"pcg_ms_pdl{pdl}"] = sorted(ts)[2]
    print(json.dumps(out), flush=True)
    c.close()
    del r, z
