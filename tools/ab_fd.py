"""A/B of two builds of libls.so on the same box: python tools/ab_fd.py <lib.so> [config]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_10026_b200 as ls
ls.load_library(os.path.abspath(sys.argv[1]))
import synth
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = synth.CONFIGS[cfg]
ctx = ls.Context(c["d"], c["p"], [c["n_el"]] * (c["d"] + 1))
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
print(json.dumps({"lib": sys.argv[1], "config": cfg, "ms": round(best, 4)}))
