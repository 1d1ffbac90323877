"""A/B of builds of libls.so on the same box:
    python tools/ab_fd.py <lib.so> [config[:p] ...]   (default: 4 3 5:2 5:4 5:8)
    LS_AB_TUNE="knob=value,..." applies ls_tune knobs to every context
Per config: best-of-3 mean fd_apply time over 10 calls (CUDA events; inputs > L2 except
config 2), and the per-launch split of one call (spatial = CS / n x n spatial modes, time)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_10026_b200 as ls
ls.load_library(os.path.abspath(sys.argv[1]))
import synth
cfgs = sys.argv[2:] or ["4", "3", "5:2", "5:4", "5:8"]
for spec in cfgs:
    cfg, _, pp = spec.partition(":")
    c = synth.CONFIGS[int(cfg)]
    p = int(pp) if pp else c["p"]
    ctx = ls.Context(c["d"], p, [c["n_el"]] * (c["d"] + 1))
    for kv in filter(None, os.environ.get("LS_AB_TUNE", "").split(",")):
        k, v = kv.split("=")
        ctx.tune(int(k), int(v))
    r = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        ctx.fd_apply(r, z)
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ctx.fd_apply(r, z)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10)
    ctx.profile(True)
    ctx.fd_apply(r, z)
    ctx.profile(False)
    torch.cuda.synchronize()
    kms, kfl, kn = ctx.profile_read()
    print(json.dumps({"lib": os.path.basename(sys.argv[1]), "tune": os.environ.get("LS_AB_TUNE", ""), "config": spec, "ms": round(best, 4),
                      "kernel_ms": round(kms, 4), "tflops_alg": round(kfl / (kms * 1e-3) / 1e12, 2)}), flush=True)
    ctx.close()
    del r, z
