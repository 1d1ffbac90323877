import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1809_10026_b200 as ls
import synth
for (d, p, ne, world) in [(2, 2, [12, 25, 40], 3), (3, 3, [5, 9, 6, 21], 4), (2, 4, [6, 30, 17], 8)]:
    ctx = ls.Context(d, p, ne)
    r = synth.residual(ctx.shape, 19)
    nt = ctx.shape[0]; Ns = int(np.prod(ctx.shape[1:]))
    rg = torch.from_numpy(r).cuda().reshape(nt, Ns)
    slabs = [ls.partition(nt, world, g) for g in range(world)]
    chunks = [ls.partition(Ns, world, h) for h in range(world)]
    bufs = [torch.full((nt, 4 * ((ln + 3) // 4)), float("nan"), dtype=torch.float64, device="cuda") for (_, ln) in chunks]
    ref = torch.empty(nt, Ns, dtype=torch.float64, device="cuda")
    for g, (t0, ntl) in enumerate(slabs):
        ctx.fd_scatter(0, rg[t0:t0 + ntl].contiguous(), ntl, 0, world, g, bufs)
        out = torch.empty(ntl, Ns, dtype=torch.float64, device="cuda")
        ctx.fd_stage(0, rg[t0:t0 + ntl].contiguous(), out, ntl)
        ref[t0:t0+ntl] = out
    torch.cuda.synchronize()
    for h, (c0, ln) in enumerate(chunks):
        b = bufs[h][:, :ln]
        nanc = torch.isnan(b).sum().item()
        err = (b - ref[:, c0:c0+ln]).abs().max().item() if nanc == 0 else -1
        # where are the NaNs
        idx = torch.nonzero(torch.isnan(b))[:5].tolist()
        print(d, p, ne, world, "chunk", h, "nan", nanc, "of", b.numel(), "err", err, idx)
