"""CPU checks of libls's host-side setup (csrc/setup_host.cpp): the univariate
factor matrices and the extended-precision generalized eigenpairs, compiled
with g++ into tools/host_setup_dump and compared with the oracle."""

import json
import os
import subprocess

import numpy as np
import pytest

from oracle import univariate as uv, fd
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "host_setup_dump")


@pytest.fixture(scope="module")
def dump():
    src = [os.path.join(ROOT, "tools", "host_setup_dump.cpp"),
           os.path.join(ROOT, "paper_1809_10026_b200", "csrc", "setup_host.cpp")]
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_1809_10026_b200", "csrc"),
                    "-o", EXE] + src, check=True)

    def run(n_el, p):
        out = subprocess.run([EXE, str(n_el), str(p)], capture_output=True, text=True, check=True).stdout
        d = json.loads(out)
        ns, nt = d["n_s"], d["n_t"]
        for k in ("M", "K", "J", "U_s"):
            d[k] = np.array(d[k]).reshape(ns, ns)
        for k in ("Mt", "Kt", "U_t"):
            d[k] = np.array(d[k]).reshape(nt, nt)
        for k in ("lam_s", "lam_t", "gauss_w"):
            d[k] = np.array(d[k])
        return d
    return run


CASES = [(1, 2), (16, 2), (8, 3), (64, 3), (20, 6), (30, 8), (130, 2), (128, 6)]


@pytest.mark.parametrize("n_el,p", CASES)
def test_matrices_match_oracle(dump, n_el, p):
    d = dump(n_el, p)
    sf, tf = uv.space_factors(n_el, p), uv.time_factors(n_el, p)
    assert d["rc"] == 0 and (d["n_s"], d["n_t"]) == uv.sizes(n_el, p)
    for key, ref in (("M", sf["M"]), ("K", sf["K"]), ("J", sf["J"]), ("Mt", tf["Mt_hat"]), ("Kt", tf["Kt_hat"])):
        # both sides assemble in extended precision and round once (reading c17)
        assert np.max(np.abs(d[key] - ref)) <= 4e-16 * np.abs(ref).max(), key


@pytest.mark.parametrize("n_el,p", CASES)
def test_eigenpairs_match_oracle(dump, n_el, p):
    d = dump(n_el, p)
    sf, tf = uv.space_factors(n_el, p), uv.time_factors(n_el, p)
    for lam, U, K, M in ((d["lam_s"], d["U_s"], sf["J"], sf["M"]), (d["lam_t"], d["U_t"], tf["Kt_hat"], tf["Mt_hat"])):
        lo, _ = fd.generalized_eig(K, M)
        np.testing.assert_allclose(lam, lo, rtol=1e-11)
        n = len(lam)
        assert np.max(np.abs(U.T @ M @ U - np.eye(n))) < 1e-12
        assert np.max(np.abs(U.T @ K @ U - np.diag(lam))) < 1e-12 * lam.max()


@pytest.mark.parametrize("n_el,p", [(16, 2), (64, 3), (128, 6)])
def test_fd_with_host_eigenpairs(dump, n_el, p):
    """Algorithm 1 with the C++ eigenpairs equals the oracle's to 1e-11."""
    d = dump(n_el, p)
    sf, tf = uv.space_factors(n_el, p), uv.time_factors(6, p)
    fdd = fd.setup([sf] * 2, tf)
    alt = dict(fdd, lam_s=[d["lam_s"]] * 2, U_s=[d["U_s"]] * 2)
    r = synth.residual((tf["Mt"].shape[0], d["n_s"], d["n_s"]), 0)
    z1, z2 = fd.fd_apply(r, fdd), fd.fd_apply(r, alt)
    assert np.linalg.norm(z1 - z2) / np.linalg.norm(z1) < 1e-11


@pytest.mark.parametrize("q", [1, 2, 3, 7, 12])
def test_gauss_weights(dump, q):
    d = dump(1, q - 1) if q >= 3 else None
    if d is None:
        pytest.skip("p >= 2 only")
    _, w = np.polynomial.legendre.leggauss(q)
    np.testing.assert_allclose(d["gauss_w"], w, rtol=1e-14)
