"""Element-wise parity at the configurations bench.py actually times.

* fd_apply at the full BASELINE config 5 sizes (d = 3, n_el = 96, p = 2 / 4 / 8: 0.86-1.09e8
  DOFs; the automatic kernel choice bench.py uses: register-direct at n = 96 / 97, the
  smem-staged kernels at n = 98..103) against the full oracle fd_apply on the same seeded
  residual.
* fd_apply at full config 4 (d = 3, p = 6, n_el = 128: 3.06e8 DOFs) on bench.py's own
  uniform seed-0 residual against the full oracle fd_apply (~12 GB of host RAM).
* both FD mode-kernel families forced (ls_tune knob 1) at the k-step buckets 24 / 25 / 26
  (n = 73 .. 100) that config 5 runs, in every mode position (contiguous, strided, time).
* full-size PCG (configs 5 p = 2, 4, 8 and 4) in bench.py's launch configuration: status,
  the recomputed true residual and Table 1's iteration count (PAPER.md 1187-1195).
"""

import numpy as np
import pytest

from oracle import univariate as uv, fd
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _fdd(d, p, n_elems):
    return fd.setup([uv.space_factors(n, p) for n in n_elems[:d]], uv.time_factors(n_elems[d], p))


def _check(z, z_ref):
    rel = np.linalg.norm((z - z_ref).ravel()) / np.linalg.norm(z_ref.ravel())
    assert rel <= TOL, rel
    assert np.max(np.abs(z - z_ref)) <= TOL * np.abs(z_ref).max()


@pytest.mark.parametrize("p", [2, 4, 8])
def test_config5_fd_apply_full(p):
    import torch
    import paper_1809_10026_b200 as ls
    c = synth.CONFIGS[5]
    ne = [c["n_el"]] * 4
    ctx = ls.Context(3, p, ne)
    r = synth.residual(ctx.shape, 0)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    _check(z, fd.fd_apply(r, _fdd(3, p, ne)))


def test_config4_fd_apply_full_uniform_seed0():
    """bench.py's timed input (uniform U[-1,1], seed 0) at full config 4, all 3.06e8 outputs."""
    import psutil
    import torch
    import paper_1809_10026_b200 as ls
    if psutil.virtual_memory().available < 24e9:
        pytest.skip("the full config-4 oracle needs ~20 GB of host RAM")
    c = synth.CONFIGS[4]
    ne = [c["n_el"]] * 4
    ctx = ls.Context(3, c["p"], ne)
    r = synth.residual(ctx.shape, 0)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    del ctx
    torch.cuda.empty_cache()
    _check(z, fd.fd_apply(r, _fdd(3, c["p"], ne)))


# (d, p, n_elems) with a mode extent n in 73..100 (k-step buckets 19-25): n = 73 / 88 (bucket
# 19 / 22 -> 24), 96 / 97 (24 / 25; register-direct by default), 98, 99, 100 (25; staged by
# default), in the contiguous, strided and time positions
BUCKET_CASES = [
    (1, 2, [73, 87]),          # n_s = 73, n_t = 88
    (1, 2, [88, 72]),          # n_s = 88, n_t = 73
    (2, 2, [96, 6, 95]),       # n_1 = 96, n_t = 96
    (2, 2, [97, 4, 96]),       # n_1 = 97, n_t = 97
    (3, 2, [5, 96, 4, 6]),     # n_2 = 96 (strided mode)
    (2, 4, [96, 5, 96]),       # n_1 = 98, n_t = 99 (config 5 p = 4 extents)
    (3, 4, [4, 5, 96, 5]),     # n_3 = 98 (outermost spatial mode)
    (1, 3, [99, 98]),          # n_s = 100, n_t = 100
    (2, 3, [7, 99, 6]),        # n_2 = 100
]


@pytest.mark.parametrize("cs", [0, 1])
@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("d,p,n_elems", BUCKET_CASES)
def test_fd_buckets_24_25_forced(variant, cs, d, p, n_elems):
    """ls_tune knob 1: 0 = automatic, 1 = smem-staged (ping-pong / m-half), 2 = register-direct;
    knob 9: centrosymmetric split of the spatial modes off / on (half extents 37..50: buckets 12, 13)."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, n_elems)
    ctx.tune(1, variant)
    ctx.tune(9, cs)
    r = synth.residual(ctx.shape, 17)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    _check(z, fd.fd_apply(r, _fdd(d, p, n_elems)))


@pytest.mark.parametrize("cfg,p", [(5, 2), (5, 4)])
def test_pcg_fullsize_config5(cfg, p):
    """As test_gpu_fullsize.test_pcg_fullsize for the remaining config-5 degrees."""
    import paper_1809_10026_b200 as ls
    c = synth.CONFIGS[cfg]
    ctx = ls.Context(c["d"], p, [c["n_el"]] * (c["d"] + 1))
    x, st = ctx.pcg(ctx.rhs(1), tol=1e-8)
    assert st["status"] == 0, st
    assert 11 <= st["iters"] <= 15, st
    assert st["rel_res"] <= 1e-8 and st["true_rel_res"] <= 1e-7, st
