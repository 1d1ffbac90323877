"""A/B of libls.so builds for ls_matvec: python tools/ab_mv.py <lib.so> <config[:p]> [variant] [mv5 0|1]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_10026_b200 as ls
ls.load_library(os.path.abspath(sys.argv[1]))
import synth
cid, _, pp = sys.argv[2].partition(":")
c = synth.CONFIGS[int(cid)]
p = int(pp) if pp else c["p"]
ctx = ls.Context(c["d"], p, [c["n_el"]] * (c["d"] + 1))
ctx.tune(2, int(sys.argv[3]) if len(sys.argv) > 3 else 3)
if len(sys.argv) > 4:
    ctx.tune(10, int(sys.argv[4]))
for kv in filter(None, os.environ.get("LS_AB_TUNE", "").split(",")):  # knob=value,...
    k, v = kv.split("=")
    ctx.tune(int(k), int(v))
x = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    ctx.matvec(x, y)
torch.cuda.synchronize()
best = 1e9
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.matvec(x, y)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 10)
print(json.dumps({"lib": sys.argv[1], "config": sys.argv[2], "args": sys.argv[3:], "tune": os.environ.get("LS_AB_TUNE", ""), "ms": round(best, 4), "chk": float(y.abs().sum())}))
