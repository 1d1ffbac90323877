"""Multi-GPU check of the distributed path (run under torchrun, one process per GPU):
every rank builds its time slab of the same seeded global inputs, runs fd_apply (NCCL or
fused all-to-all), ls_matvec (halo exchange) and pcg_solve (all-reduced scalars) through
ls_setup_dist, and rank 0 compares the gathered results with a single-GPU context.
Prints one JSON line on rank 0 (max relative errors, PCG iterations).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/dist_check.py [--d 3 --p 3 --n-el 12] [--a2a fused] [--geometry]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10026_b200 as ls  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--n-el", type=int, default=12)
    ap.add_argument("--a2a", default="nccl", choices=["nccl", "fused"])
    ap.add_argument("--geometry", action="store_true", help="revolved quarter annulus with P^G")
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ne = [a.n_el] * (a.d + 1)
    kw = {}
    if a.geometry:
        a.d = 3
        ne = [a.n_el] * 4
        kw = {"geometry": synth.revolved_quarter_annulus(), "precond": ls.LS_PRECOND_PG}
    uid = ls.unique_id() if rank == 0 else bytes(128)
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    ctx = ls.Context(a.d, a.p, ne, rank=rank, world=world, uid=obj[0], **kw)
    if a.a2a == "fused" and not a.geometry:
        ctx.tune(4, 1)
    r_glob = synth.residual(ctx.global_shape, 5)
    sl = slice(ctx.t0, ctx.t0 + ctx.nt_local)
    r = torch.from_numpy(r_glob[sl].copy()).cuda()
    z = ctx.fd_apply(r)
    y = ctx.matvec(r)
    # back to back, no host sync: ls_matvec's workspaces are the fused all-to-all's receive
    # buffers (the entry barrier of comm_fd_apply orders them)
    w = ctx.fd_apply(ctx.matvec(z))
    b = ctx.rhs(3 if a.geometry else 1)
    x, st = ctx.pcg(b, tol=1e-8)
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, (ctx.t0, z.cpu().numpy(), y.cpu().numpy(), x.cpu().numpy(), st, w.cpu().numpy()))
    if rank == 0:
        one = ls.Context(a.d, a.p, ne, **kw)
        rg = torch.from_numpy(r_glob).cuda()
        z1t = one.fd_apply(rg)
        z1, y1 = z1t.cpu().numpy(), one.matvec(rg).cpu().numpy()
        w1 = one.fd_apply(one.matvec(z1t)).cpu().numpy()
        x1, st1 = one.pcg(one.rhs(3 if a.geometry else 1), tol=1e-8)
        x1 = x1.cpu().numpy()
        parts.sort(key=lambda t: t[0])
        Z = np.concatenate([t[1] for t in parts])
        Y = np.concatenate([t[2] for t in parts])
        X = np.concatenate([t[3] for t in parts])
        Wv = np.concatenate([t[5] for t in parts])
        rel = lambda u, v: float(np.linalg.norm(u - v) / np.linalg.norm(v))
        print(json.dumps({"world": world, "a2a": a.a2a, "geometry": a.geometry, "fd_rel": rel(Z, z1),
                          "matvec_rel": rel(Y, y1), "fd_after_matvec_rel": rel(Wv, w1), "pcg_rel": rel(X, x1), "iters": [t[4]["iters"] for t in parts],
                          "iters_1gpu": st1["iters"]}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
