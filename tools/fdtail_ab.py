"""A/B of the DFMA tail rows of the shared-memory FD kernel (LS_TUNE_FD_TAIL) at config 3
(n = 65 / 66) and config 5 p = 4 (n = 98): fd_apply with CUDA events, L2 flushed.
    python tools/fdtail_ab.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10026_b200 as ls  # noqa: E402
import synth  # noqa: E402

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
for d, p, ne in ((3, 3, 64), (3, 4, 96), (2, 3, 64)):
    c = ls.Context(d, p, [ne] * (d + 1))
    s = torch.cuda.Stream()
    c.set_stream(s)
    with torch.cuda.stream(s):
        r = torch.from_numpy(synth.residual(c.shape, 0)).cuda()
        z = torch.empty_like(r)
    torch.cuda.synchronize()
    out = {"d": d, "p": p, "n_el": ne}
    for tail in (0, 1):
        c.tune(7, tail)
        for _ in range(3):
            c.fd_apply(r, z)
        ts = []
        for _ in range(20):
            with torch.cuda.stream(s):
                flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            c.fd_apply(r, z)
            b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        out[f"tail{tail}_ms"] = float(np.median(ts))
    print(json.dumps(out), flush=True)
    c.close()
