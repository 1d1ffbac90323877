"""A/B timing of the ls_matvec variants (ls_tune knob 2) and PCG solve times.

    python tools/mv_variants.py [--configs 4 3 5:8 5:2] [--reps 10] [--pcg]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1809_10026_b200 as ls
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="+", default=["4", "3", "5:8", "5:2"])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--variants", nargs="+", type=int, default=[1, 2])
ap.add_argument("--pcg", action="store_true")
ap.add_argument("--pad", type=int, default=0, help="ls_tune knob 3 (v3 row padding), 0 = default")
ap.add_argument("--tune", nargs="*", default=[], help="extra ls_tune knob=value pairs applied before timing")
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
    x = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    outs = {}
    if a.pad:
        ctx.tune(3, a.pad)
    for kv in a.tune:
        k, v = kv.split("=")
        ctx.tune(int(k), int(v))
    for v in a.variants:
        ctx.tune(2, v)
        y = torch.empty_like(x)
        for _ in range(3):
            ctx.matvec(x, y)
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(a.reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.matvec(x, y)
            e1.record(s)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / a.reps
        outs[v] = y
        rec = {"config": cs, "variant": v, "ms": round(ms, 4), "N": ctx.N,
               "GB_s_at_96B": round(96 * ctx.N / ms / 1e6, 1), "GB_s_at_152B": round(152 * ctx.N / ms / 1e6, 1)}
        if a.pcg:
            b = ctx.rhs(1 if int(cid) == 5 else 0)
            ctx.pcg(b, tol=1e-8)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            xs, st = ctx.pcg(b, tol=1e-8)
            torch.cuda.synchronize()
            rec.update({"pcg_ms": round((time.perf_counter() - t0) * 1e3, 2), "iters": st["iters"],
                        "true_rel_res": st["true_rel_res"]})
        print(json.dumps(rec), flush=True)
    if len(outs) > 1:
        v0 = a.variants[0]
        for v in a.variants[1:]:
            rel = float(torch.linalg.norm(outs[v] - outs[v0]) / torch.linalg.norm(outs[v0]))
            print(json.dumps({"config": cs, "rel_diff": rel, "variants": [v0, v]}), flush=True)
    ctx.close()
    del x, outs
    torch.cuda.empty_cache()
