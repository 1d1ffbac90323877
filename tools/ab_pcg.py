"""PCG solve times of a libls.so build: python tools/ab_pcg.py <lib.so> [cfg:p ...] (default 5:2 4:6).
Per case: warm solve, then the best of 2 timed solves (CUDA-synchronised wall clock)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_10026_b200 as ls
ls.load_library(os.path.abspath(sys.argv[1]))
import synth
for spec in sys.argv[2:] or ["5:2", "4:6"]:
    cfg, _, pp = spec.partition(":")
    c = synth.CONFIGS[int(cfg)]
    p = int(pp) if pp else c["p"]
    ctx = ls.Context(c["d"], p, [c["n_el"]] * (c["d"] + 1))
    for kv in filter(None, os.environ.get("LS_AB_TUNE", "").split(",")):  # knob=value,...
        k, v = kv.split("=")
        ctx.tune(int(k), int(v))
    b = ctx.rhs(1)
    ctx.pcg(b, tol=1e-8)
    best = 1e9
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, st = ctx.pcg(b, tol=1e-8)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"lib": os.path.basename(sys.argv[1]), "tune": os.environ.get("LS_AB_TUNE", ""), "case": spec, "iters": st["iters"],
                      "solve_ms": round(best * 1e3, 2), "true_rel_res": st["true_rel_res"]}), flush=True)
    ctx.close()
    del b, x
