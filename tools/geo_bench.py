"""Mapped-domain path timings: the rotated quarter annulus of
PAPER.md 1219 (Table 2), P and P^G, seeded U[-1,1] right-hand side.

    python tools/geo_bench.py [--n-el 32] [--p 3] [--reps 10] [--no-pcg]

Prints one JSON line per (n_el, p, preconditioner): setup s (wall), matvec / fd_apply ms
(CUDA events on the context stream, median), PCG iterations and solve ms, and the stencil
pass's algorithmic bytes / flops."""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_10026_b200 as ls  # noqa: E402
import synth  # noqa: E402


def timed(fn, stream, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run(n_el, p, precond, reps, pcg, geo_name="annulus3d", variant=0):
    geo = synth.GEOMETRIES[geo_name]()
    d = geo["d"]
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = ls.Context(d, p, [n_el] * (d + 1), geometry=geo, precond=precond)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    ctx.set_stream(stream)
    if variant:
        ctx.tune(2, variant)
    with torch.cuda.stream(stream):
        x = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
        y = torch.empty_like(x)
    torch.cuda.synchronize()
    for _ in range(3):
        ctx.matvec(x, y)
        ctx.fd_apply(x, y)
    mv = timed(lambda: ctx.matvec(x, y), stream, reps)
    fdm = timed(lambda: ctx.fd_apply(x, y), stream, reps)
    S = (2 * p + 1) ** d
    Ns = int(np.prod(ctx.n_s))
    N = ctx.N
    out = {"variant": variant, "geometry": geo_name, "d": d, "p": p, "n_el": n_el, "N": N, "precond": ["P", "P^G"][precond],
           "setup_s": round(setup_s, 3), "matvec_ms": mv, "fd_apply_ms": fdm,
           "stencil_bytes_alg": 8.0 * (3 * S * Ns + 3 * N), "stencil_flops_alg": 4.0 * S * N,
           "fit_rel_res": ctx.geo_info()[0]}
    if pcg:
        b = x
        ctx.pcg(b, tol=1e-8, max_iter=2000)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, st = ctx.pcg(b, tol=1e-8, max_iter=2000)
        torch.cuda.synchronize()
        out.update({"iters": st["iters"], "solve_ms": (time.perf_counter() - t0) * 1e3,
                    "true_rel_res": st["true_rel_res"]})
    ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-el", type=int, nargs="+", default=[32])
    ap.add_argument("--p", type=int, nargs="+", default=[3])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--precond", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--geometry", default="annulus3d")
    ap.add_argument("--variant", type=int, nargs="+", default=[0])
    a = ap.parse_args()
    for n in a.n_el:
        for p in a.p:
            for pc in a.precond:
                for v in a.variant:
                    print(json.dumps(run(n, p, pc, a.reps, not a.no_pcg, a.geometry, v)), flush=True)


if __name__ == "__main__":
    main()
