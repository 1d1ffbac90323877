"""fd_apply_host_batch (include/ls_api.h): z_k = P^{-1} r_k (Algorithm 1, PAPER.md 955-964) for a
list of host vectors with the copies of neighbouring vectors overlapped with the application
(two device buffer pairs, separate H2D / D2H streams).  Every z_k must equal the device
fd_apply of r_k bit for bit (same kernels, same inputs) and the oracle at the parity bar; counts
0 .. 5 (both buffer pairs reused), aliased inputs, torch pinned tensors and numpy arrays, the
P^G path, and argument errors."""

import numpy as np
import pytest

from oracle import univariate as uv, fd
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("count", [0, 1, 2, 5])
def test_host_batch_matches_device(count):
    import torch
    import paper_1809_10026_b200 as ls
    d, p, ne = 3, 3, [9, 8, 7, 12]
    ctx = ls.Context(d, p, ne)
    rs = [synth.residual(ctx.shape, 40 + k) for k in range(count)]
    zs = [np.empty_like(r) for r in rs]
    ctx.fd_apply_host_batch(rs, zs)
    fdd = fd.setup([uv.space_factors(n, p) for n in ne[:d]], uv.time_factors(ne[d], p))
    for r, z in zip(rs, zs):
        zd = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
        assert np.array_equal(z, zd)
        z_ref = fd.fd_apply(r, fdd)
        assert np.linalg.norm(z - z_ref) <= 1e-9 * np.linalg.norm(z_ref)


def test_host_batch_pinned_aliased_inputs():
    """The same pinned input for every vector (the bench's e2e), distinct pinned outputs."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(2, 4, [30, 29, 40])
    r = torch.from_numpy(synth.residual(ctx.shape, 3)).pin_memory()
    zs = [torch.empty_like(r).pin_memory() for _ in range(4)]
    ctx.fd_apply_host_batch([r] * 4, zs)
    zd = ctx.fd_apply(r.cuda()).cpu()
    for z in zs:
        assert torch.equal(z, zd)


def test_host_batch_pg_and_errors():
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(2, 3, [8, 8, 6], geometry=synth.quarter_annulus(), precond=ls.LS_PRECOND_PG)
    rs = [synth.residual(ctx.shape, 5 + k) for k in range(3)]
    zs = [np.empty_like(r) for r in rs]
    ctx.fd_apply_host_batch(rs, zs)
    for r, z in zip(rs, zs):
        assert np.array_equal(z, ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy())
    with pytest.raises(ValueError):
        ctx.fd_apply_host_batch(rs, zs[:2])
    with pytest.raises(ValueError):
        ctx.fd_apply_host_batch([rs[0][:-1]], [zs[0]])
    # the C entry point rejects a null table
    assert ctx._lib.fd_apply_host_batch(ctx._h, None, None, 1) == ls.LS_EINVAL
