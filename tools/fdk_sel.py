"""fd_apply time per FD kernel choice (ls_tune LS_TUNE_FD_KERNEL) at config 5 p = 2 / 4 / 8 and
config 3: python tools/fdk_sel.py  (checks the automatic choice per mode extent)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_10026_b200 as ls
import synth
for cid, p in [(3, None), (5, 2), (5, 4), (5, 8)]:
    c = synth.CONFIGS[cid]
    pp = p or c["p"]
    ctx = ls.Context(c["d"], pp, [c["n_el"]] * (c["d"] + 1))
    r = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    z = torch.empty_like(r)
    for v in range(0, 3):
        try:
            ctx.tune(1, v)
        except Exception as exc:
            print(json.dumps({"config": cid, "p": pp, "fdk": v, "error": str(exc)[:80]}))
            continue
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
        print(json.dumps({"config": cid, "p": pp, "fdk": v, "ms": round(best, 4), "chk": float(z.abs().sum())}), flush=True)
    ctx.close()
