"""Multi-rank (N > 1) path on CPU: world_size 2 and 3 over torch.distributed/gloo.

The GPU kernels cannot run here, so each rank executes the distributed SCHEDULE
of libls (time slabs, pack map, all-to-all plan, halo plan -- queried from the
library's host-only C-ABI, i.e. the exact functions comm.cu uses) with the
oracle's per-mode arithmetic, exchanges data over gloo exactly as comm.cu does
over NCCL, and compares the gathered result with the single-process oracle.
"""

import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import univariate as uv, fd, operator as op
import synth


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup(d, p, ne):
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    return space, tf, fd.setup(space, tf)


def _fd_rank(rank, world, d, p, ne):
    import paper_1809_10026_b200 as ls
    space, tf, fdd = _setup(d, p, ne)
    nt = tf["Mt"].shape[0]
    gshape = (nt,) + tuple(f["M"].shape[0] for f in reversed(space))
    Ns = int(np.prod(gshape[1:]))
    r = synth.residual(gshape, 0)
    t0, ntl = ls.partition(nt, world, rank)
    x = r[t0:t0 + ntl].copy()
    for k in range(1, d + 1):                      # F1 (local)
        x = fd.mode_apply(x, fdd["U_s"][k - 1].T, d + 1 - k)
    pos = ls.pack_map(ntl, Ns, world)              # pack (comm.cu pack_kernel<true>)
    send = np.empty(ntl * Ns)
    send[pos] = x.ravel()
    plan = ls.a2a_plan(nt, Ns, world, rank)
    assert np.all(plan["send_off"] == np.concatenate([[0], np.cumsum(plan["send_cnt"])[:-1]]))
    assert np.all(plan["recv_off"] == np.concatenate([[0], np.cumsum(plan["recv_cnt"])[:-1]]))
    c0, clen = ls.partition(Ns, world, rank)
    recv = torch.empty(nt * clen, dtype=torch.float64)
    dist.all_to_all_single(recv, torch.from_numpy(send), output_split_sizes=plan["recv_cnt"].tolist(),
                           input_split_sizes=plan["send_cnt"].tolist())
    chunk = recv.numpy().reshape(nt, clen)         # [n_t][chunk]: time mode is local now
    lam_s = (fd.divisor(fdd) - fdd["lam_t"].reshape((-1,) + (1,) * d))[0].ravel()
    y = fdd["U_t"].T @ chunk
    y = y / (fdd["lam_t"][:, None] + lam_s[None, c0:c0 + clen])
    y = fdd["U_t"] @ y
    back = torch.empty(ntl * Ns, dtype=torch.float64)  # chunk -> slab: transpose plan
    dist.all_to_all_single(back, torch.from_numpy(np.ascontiguousarray(y).ravel()),
                           output_split_sizes=plan["send_cnt"].tolist(),
                           input_split_sizes=plan["recv_cnt"].tolist())
    z = back.numpy()[pos].reshape((ntl,) + gshape[1:])  # unpack (pack_kernel<false>)
    for k in range(d, 0, -1):                      # F3 (local)
        z = fd.mode_apply(z, fdd["U_s"][k - 1], d + 1 - k)
    ref = fd.fd_apply(r, fdd)[t0:t0 + ntl]
    return float(np.linalg.norm(z - ref) / np.linalg.norm(ref))


def _fd_rank_pieces(rank, world, d, p, ne):
    """The pipelined NCCL schedule of comm_fd_apply: per piece of consecutive time slices
    (ls_a2a_piece_plan), F1 on the piece, pack the piece, exchange it; time mode on the chunk;
    per piece, the transposed exchange, unpack, F3 on the piece."""
    import paper_1809_10026_b200 as ls
    space, tf, fdd = _setup(d, p, ne)
    nt = tf["Mt"].shape[0]
    gshape = (nt,) + tuple(f["M"].shape[0] for f in reversed(space))
    Ns = int(np.prod(gshape[1:]))
    r = synth.residual(gshape, 0)
    t0, ntl = ls.partition(nt, world, rank)
    c0, clen = ls.partition(Ns, world, rank)
    P, _ = ls.a2a_piece_plan(nt, Ns, world, rank, -1)
    pos = ls.pack_map(ntl, Ns, world)
    packed = np.empty(ntl * Ns)
    chunk = np.full(nt * clen, np.nan)
    for c in range(P):
        a, ln = ls.partition(ntl, P, c)
        x = r[t0 + a:t0 + a + ln].copy()
        for k in range(1, d + 1):                  # F1 on the piece
            x = fd.mode_apply(x, fdd["U_s"][k - 1].T, d + 1 - k)
        packed[pos[a * Ns:(a + ln) * Ns]] = x.ravel()  # pack_kernel<true> over the piece's elements
        _, plan = ls.a2a_piece_plan(nt, Ns, world, rank, c)
        send = np.concatenate([packed[so:so + sc] for (so, sc, _, _) in plan])
        recv = torch.empty(sum(rc for (_, _, _, rc) in plan), dtype=torch.float64)
        dist.all_to_all_single(recv, torch.from_numpy(send), output_split_sizes=[rc for (_, _, _, rc) in plan],
                               input_split_sizes=[sc for (_, sc, _, _) in plan])
        off = 0
        for (_, _, ro, rc) in plan:
            chunk[ro:ro + rc] = recv.numpy()[off:off + rc]
            off += rc
    assert np.isfinite(chunk).all()
    chunk = chunk.reshape(nt, clen)
    lam_s = (fd.divisor(fdd) - fdd["lam_t"].reshape((-1,) + (1,) * d))[0].ravel()
    y = fdd["U_t"].T @ chunk
    y = y / (fdd["lam_t"][:, None] + lam_s[None, c0:c0 + clen])
    y = np.ascontiguousarray(fdd["U_t"] @ y).ravel()
    back = np.full(ntl * Ns, np.nan)
    z = np.empty((ntl,) + gshape[1:])
    for c in range(P):                             # transposed exchange, unpack, F3 per piece
        a, ln = ls.partition(ntl, P, c)
        _, plan = ls.a2a_piece_plan(nt, Ns, world, rank, c)
        send = np.concatenate([y[ro:ro + rc] for (_, _, ro, rc) in plan])
        recv = torch.empty(sum(sc for (_, sc, _, _) in plan), dtype=torch.float64)
        dist.all_to_all_single(recv, torch.from_numpy(send), output_split_sizes=[sc for (_, sc, _, _) in plan],
                               input_split_sizes=[rc for (_, _, _, rc) in plan])
        off = 0
        for (so, sc, _, _) in plan:
            back[so:so + sc] = recv.numpy()[off:off + sc]
            off += sc
        zz = back[pos[a * Ns:(a + ln) * Ns]].reshape((ln,) + gshape[1:])  # pack_kernel<false>
        for k in range(d, 0, -1):
            zz = fd.mode_apply(zz, fdd["U_s"][k - 1], d + 1 - k)
        z[a:a + ln] = zz
    ref = fd.fd_apply(r, fdd)[t0:t0 + ntl]
    return float(np.linalg.norm(z - ref) / np.linalg.norm(ref))


def _matvec_rank(rank, world, d, p, ne):
    import paper_1809_10026_b200 as ls
    space, tf, _ = _setup(d, p, ne)
    nt = tf["Mt"].shape[0]
    gshape = (nt,) + tuple(f["M"].shape[0] for f in reversed(space))
    x = synth.residual(gshape, 1)
    t0, ntl, lo, hi = ls.halo_plan(nt, world, rank, p)
    own = x[t0:t0 + ntl].copy()
    ext = np.zeros((lo + ntl + hi,) + gshape[1:])
    ext[lo:lo + ntl] = own
    reqs = []  # comm.cu halo_exchange, over gloo point-to-point
    if lo > 0:
        lo_buf = torch.empty(ext[:lo].shape, dtype=torch.float64)
        reqs.append(dist.irecv(lo_buf, src=rank - 1))
        reqs.append(dist.isend(torch.from_numpy(own[:lo].copy()), dst=rank - 1))
    if hi > 0:
        hi_buf = torch.empty(ext[lo + ntl:].shape, dtype=torch.float64)
        reqs.append(dist.irecv(hi_buf, src=rank + 1))
        reqs.append(dist.isend(torch.from_numpy(own[ntl - hi:].copy()), dst=rank + 1))
    for q in reqs:
        q.wait()
    if lo > 0:
        ext[:lo] = lo_buf.numpy()
    if hi > 0:
        ext[lo + ntl:] = hi_buf.numpy()
    # spatial part of each Kronecker term on the extended slab, time band on own rows
    s_first = t0 - lo
    M = [f["M"] for f in space]
    SM = op.apply_kron(ext, None, M)
    SJ = 0.0
    SL = 0.0
    for k in range(d):
        mats = list(M)
        mats[k] = space[k]["J"]
        SJ = SJ + op.apply_kron(ext, None, mats)
        for l in range(d):
            if l != k:
                mats = list(M)
                mats[k], mats[l] = space[k]["G"], space[l]["G"].T
                SJ = SJ + op.apply_kron(ext, None, mats)
        mats = list(M)
        mats[k] = space[k]["K"]
        SL = SL + op.apply_kron(ext, None, mats)
    y = np.zeros_like(own)
    for tl in range(ntl):
        t = t0 + tl
        for i in range(max(0, t - p), min(nt - 1, t + p) + 1):
            y[tl] += tf["Kt"][t, i] * SM[i - s_first] + tf["Mt"][t, i] * SJ[i - s_first]
        y[tl] += tf["Wt"][t, t] * SL[t - s_first] if t == nt - 1 else 0.0
    ref = op.apply_A(x, space, tf)[t0:t0 + ntl]
    return float(np.linalg.norm(y - ref) / np.linalg.norm(ref))


def _geo_matvec_rank(rank, world, name, p, ne):
    """The mapped-domain ls_matvec of ls_setup_geo_dist: p_t halo slices exchanged with the
    neighbours (ls_halo_plan), then the slab rows of K_t(x)M_s + M_t(x)J_s + W_t(x)L_s from
    the extended slab (spatial factors replicated on every rank)."""
    import warnings
    warnings.filterwarnings("ignore")
    import paper_1809_10026_b200 as ls
    from oracle import geometry as og
    geo = synth.GEOMETRIES[name]()
    d = geo["d"]
    sf = og.space_factors_physical(geo, ne[:d], p)
    tf = uv.time_factors(ne[d], p)
    nt = tf["Mt"].shape[0]
    gshape = (nt,) + tuple(reversed(sf["n_s"]))
    x = synth.residual(gshape, 2)
    t0, ntl, lo, hi = ls.halo_plan(nt, world, rank, p)
    own = x[t0:t0 + ntl].copy()
    ext = np.zeros((lo + ntl + hi,) + gshape[1:])
    ext[lo:lo + ntl] = own
    reqs = []
    if lo > 0:
        lo_buf = torch.empty(ext[:lo].shape, dtype=torch.float64)
        reqs.append(dist.irecv(lo_buf, src=rank - 1))
        reqs.append(dist.isend(torch.from_numpy(own[:lo].copy()), dst=rank - 1))
    if hi > 0:
        hi_buf = torch.empty(ext[lo + ntl:].shape, dtype=torch.float64)
        reqs.append(dist.irecv(hi_buf, src=rank + 1))
        reqs.append(dist.isend(torch.from_numpy(own[ntl - hi:].copy()), dst=rank + 1))
    for q in reqs:
        q.wait()
    if lo > 0:
        ext[:lo] = lo_buf.numpy()
    if hi > 0:
        ext[lo + ntl:] = hi_buf.numpy()
    s_first = t0 - lo
    E = ext.reshape(ext.shape[0], -1)
    SM, SJ, SL = (sf["M"] @ E.T).T, (sf["J"] @ E.T).T, (sf["L"] @ E.T).T
    y = np.zeros((ntl, E.shape[1]))
    for tl in range(ntl):
        t = t0 + tl
        for i in range(max(0, t - p), min(nt - 1, t + p) + 1):
            y[tl] += tf["Kt"][t, i] * SM[i - s_first] + tf["Mt"][t, i] * SJ[i - s_first]
        if t == nt - 1:
            y[tl] += tf["Wt"][t, t] * SL[t - s_first]
    ref = og.apply_A_geo(x, sf, tf)[t0:t0 + ntl].reshape(ntl, -1)
    return float(np.linalg.norm(y - ref) / np.linalg.norm(ref))


def _dist_fd(r_slab, rank, world, fdd, d, gshape):
    """One rank's share of the distributed fd_apply (comm_fd_apply's NCCL schedule, over gloo)."""
    import paper_1809_10026_b200 as ls
    nt = gshape[0]
    Ns = int(np.prod(gshape[1:]))
    t0, ntl = ls.partition(nt, world, rank)
    x = r_slab.copy()
    for k in range(1, d + 1):
        x = fd.mode_apply(x, fdd["U_s"][k - 1].T, d + 1 - k)
    pos = ls.pack_map(ntl, Ns, world)
    send = np.empty(ntl * Ns)
    send[pos] = x.ravel()
    plan = ls.a2a_plan(nt, Ns, world, rank)
    c0, clen = ls.partition(Ns, world, rank)
    recv = torch.empty(nt * clen, dtype=torch.float64)
    dist.all_to_all_single(recv, torch.from_numpy(send), output_split_sizes=plan["recv_cnt"].tolist(),
                           input_split_sizes=plan["send_cnt"].tolist())
    chunk = recv.numpy().reshape(nt, clen)
    lam_s = (fd.divisor(fdd) - fdd["lam_t"].reshape((-1,) + (1,) * d))[0].ravel()
    y = fdd["U_t"] @ ((fdd["U_t"].T @ chunk) / (fdd["lam_t"][:, None] + lam_s[None, c0:c0 + clen]))
    back = torch.empty(ntl * Ns, dtype=torch.float64)
    dist.all_to_all_single(back, torch.from_numpy(np.ascontiguousarray(y).ravel()),
                           output_split_sizes=plan["send_cnt"].tolist(), input_split_sizes=plan["recv_cnt"].tolist())
    z = back.numpy()[pos].reshape((ntl,) + gshape[1:])
    for k in range(d, 0, -1):
        z = fd.mode_apply(z, fdd["U_s"][k - 1], d + 1 - k)
    return z


def _dist_matvec(x_slab, rank, world, space, tf, p, gshape):
    """One rank's share of the distributed ls_matvec: halo exchange (comm.cu halo_exchange,
    over gloo) then the slab-local operator on the extended slab."""
    import paper_1809_10026_b200 as ls
    nt = gshape[0]
    t0, ntl, lo, hi = ls.halo_plan(nt, world, rank, p)
    ext = np.zeros((lo + ntl + hi,) + gshape[1:])
    ext[lo:lo + ntl] = x_slab
    reqs, lo_buf, hi_buf = [], None, None
    if lo > 0:
        lo_buf = torch.empty(ext[:lo].shape, dtype=torch.float64)
        reqs += [dist.irecv(lo_buf, src=rank - 1), dist.isend(torch.from_numpy(x_slab[:lo].copy()), dst=rank - 1)]
    if hi > 0:
        hi_buf = torch.empty(ext[lo + ntl:].shape, dtype=torch.float64)
        reqs += [dist.irecv(hi_buf, src=rank + 1), dist.isend(torch.from_numpy(x_slab[ntl - hi:].copy()), dst=rank + 1)]
    for q in reqs:
        q.wait()
    if lo > 0:
        ext[:lo] = lo_buf.numpy()
    if hi > 0:
        ext[lo + ntl:] = hi_buf.numpy()
    # the oracle's A on a zero-padded global tensor holding only the extended slab: exact on
    # the own rows (the time band reaches at most p slices, all present)
    g = np.zeros(gshape)
    g[t0 - lo:t0 + ntl + hi] = ext
    return op.apply_A(g, space, tf)[t0:t0 + ntl]


def _pcg_rank(rank, world, d, p, ne):
    """The distributed pcg_solve schedule: slab vectors, the two distributed operators above,
    every dot product all-reduced (comm.cu allreduce_scalar), stopping test on the global
    recurrence residual; against the single-process oracle PCG."""
    import paper_1809_10026_b200 as ls
    from oracle import rhs as orhs, pcg as opcg, bspline as bs
    space, tf, fdd = _setup(d, p, ne)
    nt = tf["Mt"].shape[0]
    gshape = (nt,) + tuple(f["M"].shape[0] for f in reversed(space))
    b = orhs.rhs(1, [bs.open_uniform_knots(n, p) for n in ne[:d]], p, bs.open_uniform_knots(ne[d], p), p)
    t0, ntl = ls.partition(nt, world, rank)

    def allsum(v):
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    bs_ = b[t0:t0 + ntl].copy()
    bnorm = np.sqrt(allsum(np.vdot(bs_, bs_)))
    x = np.zeros_like(bs_)
    r = bs_.copy()
    z = _dist_fd(r, rank, world, fdd, d, gshape)
    pv = z.copy()
    rho = allsum(np.vdot(r, z))
    it = 0
    while it < 100:
        q = _dist_matvec(pv, rank, world, space, tf, p, gshape)
        alpha = rho / allsum(np.vdot(pv, q))
        x += alpha * pv
        r -= alpha * q
        it += 1
        if np.sqrt(allsum(np.vdot(r, r))) <= 1e-8 * bnorm:
            break
        z = _dist_fd(r, rank, world, fdd, d, gshape)
        rho_new = allsum(np.vdot(r, z))
        pv = z + (rho_new / rho) * pv
        rho = rho_new
    xo, it_o, _, _ = opcg.pcg(lambda v: op.apply_A(v, space, tf), lambda v: fd.fd_apply(v, fdd), b)
    assert it == it_o, (it, it_o)
    ref = xo[t0:t0 + ntl]
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


def _worker(rank, world, port, fn_name, args, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        err = globals()[fn_name](rank, world, *args)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, err, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def _run(world, fn_name, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, args, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, err, tb in res:
        assert tb is None, tb
    return [err for _, err, _ in sorted(res)]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("d,p,ne", [(2, 2, [5, 4, 7]), (3, 3, [3, 4, 2, 9])])
def test_distributed_fd_schedule(world, d, p, ne):
    errs = _run(world, "_fd_rank", (d, p, ne))
    assert max(errs) <= 1e-12, errs


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("d,p,ne", [(2, 2, [5, 4, 7]), (3, 3, [3, 4, 2, 12])])
def test_distributed_fd_schedule_pieces(world, d, p, ne):
    errs = _run(world, "_fd_rank_pieces", (d, p, ne))
    assert max(errs) <= 1e-12, errs


def test_piece_plans_cover_the_exchange():
    """The pieces of the pipelined all-to-all partition each rank's slab rows and reproduce
    ls_a2a_plan's exchange segment by segment (what r sends to h in piece c is what h receives
    from r in piece c)."""
    import paper_1809_10026_b200 as ls
    for nt, Ns, world in ((133, 1000, 8), (133, 2299968, 8), (13, 30, 2), (17, 45, 3), (9, 23, 4), (5, 64, 5), (7, 11, 1)):
        P, _ = ls.a2a_piece_plan(nt, Ns, world, 0, -1)
        assert P == min(4, max(1, nt // world))
        for r in range(world):
            full = ls.a2a_plan(nt, Ns, world, r)
            pieces = [ls.a2a_piece_plan(nt, Ns, world, r, c)[1] for c in range(P)]
            for h in range(world):
                segs = [pc[h] for pc in pieces]
                # send: consecutive sub-ranges of the packed block for h, in piece order
                assert segs[0][0] == full["send_off"][h]
                assert sum(sg[1] for sg in segs) == full["send_cnt"][h]
                assert all(segs[c][0] + segs[c][1] == segs[c + 1][0] for c in range(P - 1))
                # recv: consecutive row ranges of the chunk tensor from h
                assert segs[0][2] == full["recv_off"][h]
                assert sum(sg[3] for sg in segs) == full["recv_cnt"][h]
                assert all(segs[c][2] + segs[c][3] == segs[c + 1][2] for c in range(P - 1))
                for c in range(P):   # matching counts across the pair (r -> h) in piece c
                    assert pieces[c][h][1] == ls.a2a_piece_plan(nt, Ns, world, h, c)[1][r][3]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("d,p,ne", [(1, 2, [6, 9]), (2, 3, [3, 4, 12])])
def test_distributed_matvec_halo(world, d, p, ne):
    errs = _run(world, "_matvec_rank", (d, p, ne))
    assert max(errs) <= 1e-12, errs


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,p,ne", [("annulus2d", 3, [4, 5, 12]), ("annulus3d", 2, [2, 3, 2, 9])])
def test_distributed_geo_matvec_halo(world, name, p, ne):
    errs = _run(world, "_geo_matvec_rank", (name, p, ne))
    assert max(errs) <= 1e-12, errs


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("d,p,ne", [(2, 2, [4, 5, 8]), (3, 2, [3, 3, 3, 8])])
def test_distributed_pcg(world, d, p, ne):
    """pcg_solve's distributed schedule (slab fd_apply with two all-to-alls, halo matvec,
    all-reduced dots) reaches the single-process oracle's iterate at the same iteration."""
    errs = _run(world, "_pcg_rank", (d, p, ne))
    assert max(errs) <= 1e-10, errs


def test_plans_cover_everything():
    """Slabs and chunks tile their ranges; the pack map is a permutation; the
    a2a plans of all ranks are mutually consistent (what r sends to h is what h
    receives from r)."""
    import paper_1809_10026_b200 as ls
    nt, Ns = 133, 132 ** 3 // 1000
    for world in (1, 2, 3, 8):
        offs = [ls.partition(nt, world, g) for g in range(world)]
        assert offs[0][0] == 0 and sum(l for _, l in offs) == nt
        assert all(offs[g][0] + offs[g][1] == offs[g + 1][0] for g in range(world - 1))
        plans = [ls.a2a_plan(nt, Ns, world, r) for r in range(world)]
        for r in range(world):
            for h in range(world):
                assert plans[r]["send_cnt"][h] == plans[h]["recv_cnt"][r]
            assert plans[r]["send_cnt"].sum() == ls.partition(nt, world, r)[1] * Ns
            assert plans[r]["recv_cnt"].sum() == nt * ls.partition(Ns, world, r)[1]
        ntl = ls.partition(nt, world, world - 1)[1]
        pos = ls.pack_map(ntl, Ns, world)
        assert np.array_equal(np.sort(pos), np.arange(ntl * Ns))
    t0, ntl, lo, hi = ls.halo_plan(133, 8, 0, 6)
    assert (t0, ntl, lo, hi) == (0, 17, 0, 6)
    assert ls.halo_plan(133, 8, 7, 6) == (117, 16, 6, 0)
    with pytest.raises(ls.LSError):
        ls.halo_plan(10, 8, 0, 6)   # slabs of 1-2 rows are thinner than the halo


@pytest.mark.parametrize("nt,Ns,world", [(13, 30, 2), (17, 45, 3), (9, 23, 4), (20, 7, 8), (5, 64, 5)])
def test_fused_a2a_dest_equals_nccl_plan(nt, Ns, world):
    """The fused all-to-all's per-element destinations (ls_a2a_dest = the addressing of the
    peer-memory epilogues) move every element exactly where the NCCL path (pack map +
    all-to-all plan + receive layout) puts it, forward (slab -> chunk, padded rows of
    4*ceil(len/4)) and backward (chunk -> slab)."""
    import paper_1809_10026_b200 as ls
    rng = np.random.default_rng(nt * 100 + Ns)
    g = rng.standard_normal((nt, Ns))
    chunks = [ls.partition(Ns, world, h) for h in range(world)]
    slabs = [ls.partition(nt, world, r) for r in range(world)]
    # NCCL path: receiver h holds [n_t][len_h] = the columns of its chunk for every time
    ref_chunk = [g[:, c0:c0 + ln] for (c0, ln) in chunks]
    fused = [np.full((nt, max(4 * ((ln + 3) // 4), 1)), np.nan) for (_, ln) in chunks]
    for r, (t0, ntl) in enumerate(slabs):
        for t in range(ntl):
            for s in range(Ns):
                h, off = ls.a2a_dest(nt, Ns, world, r, 0, t, s)
                fused[h].ravel()[off] = g[t0 + t, s]
    for h, (c0, ln) in enumerate(chunks):
        np.testing.assert_array_equal(fused[h][:, :ln], ref_chunk[h])
    # backward: every chunk element back into the owner's slab
    slab_bufs = [np.full((ntl, Ns), np.nan) for (_, ntl) in slabs]
    for h, (c0, ln) in enumerate(chunks):
        for t in range(nt):
            for j in range(ln):
                r, off = ls.a2a_dest(nt, Ns, world, h, 1, t, j)
                slab_bufs[r].ravel()[off] = g[t, c0 + j]
    for r, (t0, ntl) in enumerate(slabs):
        np.testing.assert_array_equal(slab_bufs[r], g[t0:t0 + ntl])
