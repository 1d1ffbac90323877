"""B200-native hot path of the space-time least-squares IGA method (arXiv 1809.10026).

Thin ctypes binding over ``libls.so`` (C-ABI declared in ``include/ls_api.h``):
argument marshalling only -- every step of fd_apply / ls_matvec / pcg_solve runs
in the library's CUDA kernels.  There is no CPU fallback: importing this module
without the built library raises, and every call checks that its tensors are
contiguous fp64 CUDA tensors.

Typical use::

    import torch, paper_1809_10026_b200 as ls
    ctx = ls.Context(d=3, p=3, n_elems=[64, 64, 64, 64])
    r = torch.rand(ctx.shape, dtype=torch.float64, device="cuda") * 2 - 1
    z = ctx.fd_apply(r)                  # z = P^{-1} r   (Algorithm 1)
    b = ctx.rhs(kind=1)                  # cube forcing (PAPER.md 1166)
    x, stats = ctx.pcg(b, tol=1e-8)      # PCG with P (PAPER.md 1109)
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libls.so")

LS_OK, LS_EINVAL, LS_ENOTSPD, LS_ENOCONV, LS_ENUMERIC, LS_ENOMEM, LS_ECUDA, LS_ENCCL, LS_ENOTSUP = range(9)

# Every symbol include/ls_api.h declares (checked by tests/test_abi.py).
EXPORTED = ["ls_setup", "ls_setup_dist", "ls_get_unique_id", "ls_layout", "ls_set_stream",
            "fd_apply", "ls_matvec", "ls_matvec_slab3", "ls_rhs", "pcg_solve", "fd_apply_host", "fd_apply_host_batch", "ls_get_factor",
            "ls_kernel_launches", "ls_profile", "ls_profile_read", "ls_destroy", "ls_strerror",
            "ls_partition", "ls_a2a_plan", "ls_a2a_piece_plan", "ls_pack_map", "ls_halo_plan", "ls_tune",
            "ls_matvec_slab", "fd_apply_stage", "fd_apply_scatter", "ls_a2a_dest", "ls_setup_deg",
            "ls_setup_dist_deg", "ls_energy_error", "ls_error_norms", "ls_setup_geo", "ls_geo_info", "ls_setup_geo_dist", "ls_pg_factors"]

LS_PRECOND_P, LS_PRECOND_PG = 0, 1
# ls_tune knobs (include/ls_api.h)
LS_TUNE_FD_KERNEL, LS_TUNE_MATVEC, LS_TUNE_MV3_PAD, LS_TUNE_A2A, LS_TUNE_PCG_GRAPH, LS_TUNE_PDL = 1, 2, 3, 4, 5, 6
LS_TUNE_FD_TAIL, LS_TUNE_MV4_CTAS, LS_TUNE_FD_CS, LS_TUNE_MV5, LS_TUNE_FD_STAGED, LS_TUNE_PQ_FUSE = 7, 8, 9, 10, 11, 12
LS_TUNE_FD_TIME, LS_TUNE_FD_PLANE, LS_TUNE_MV6, LS_TUNE_MV2_SWEEP, LS_TUNE_MV4_SWEEP = 13, 14, 15, 16, 17


class Geometry(ctypes.Structure):
    """ls_geometry (include/ls_api.h): a tensor-product (NURBS) map F: [0,1]^d -> Omega."""
    _fields_ = [("degree", ctypes.c_int * 3), ("n_knots", ctypes.c_int64 * 3),
                ("knots", ctypes.c_void_p * 3), ("ctrl", ctypes.c_void_p), ("weights", ctypes.c_void_p)]


class PCGStats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("rel_res", ctypes.c_double),
                ("true_rel_res", ctypes.c_double), ("status", ctypes.c_int)]

    def as_dict(self):
        return {"iters": self.iters, "rel_res": self.rel_res,
                "true_rel_res": self.true_rel_res, "status": self.status}


class LSError(RuntimeError):
    def __init__(self, code, what):
        self.code = code
        super().__init__(f"{what}: {strerror(code)} (code {code})")


_lib = None


def load_library(path=LIB_PATH):
    """Load libls.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    vp, i64p, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p
    sig = {
        "ls_setup": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, i64p, ctypes.POINTER(vp)]),
        "ls_setup_deg": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, ctypes.POINTER(vp)]),
        "ls_setup_dist_deg": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(vp)]),
        "ls_setup_dist": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, i64p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_char_p, ctypes.POINTER(vp)]),
        "ls_get_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
        "ls_layout": (ctypes.c_int, [vp, i64p, i64p, i64p, i64p]),
        "ls_set_stream": (ctypes.c_int, [vp, vp]),
        "fd_apply": (ctypes.c_int, [vp, dp, dp]),
        "ls_matvec": (ctypes.c_int, [vp, dp, dp]),
        "ls_rhs": (ctypes.c_int, [vp, ctypes.c_int, dp]),
        "pcg_solve": (ctypes.c_int, [vp, dp, dp, ctypes.c_double, ctypes.c_int, ctypes.POINTER(PCGStats)]),
        "fd_apply_host": (ctypes.c_int, [vp, dp, dp]),
        "fd_apply_host_batch": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64]),
        "ls_get_factor": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, dp]),
        "ls_kernel_launches": (ctypes.c_int64, [vp]),
        "ls_profile": (ctypes.c_int, [vp, ctypes.c_int]),
        "ls_profile_read": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double), i64p]),
        "ls_destroy": (None, [vp]),
        "ls_setup_geo": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, ctypes.POINTER(Geometry),
                                        ctypes.c_int, ctypes.POINTER(vp)]),
        "ls_geo_info": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_double)]),
        "ls_pg_factors": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_int, i64p, dp, dp, dp,
                                         dp, ctypes.POINTER(ctypes.c_double)]),
        "ls_setup_geo_dist": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p,
                                             ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_char_p, ctypes.POINTER(vp)]),
        "ls_tune": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int]),
        "ls_energy_error": (ctypes.c_int, [vp, ctypes.c_int, dp, ctypes.POINTER(ctypes.c_double)]),
        "ls_error_norms": (ctypes.c_int, [vp, ctypes.c_int, dp, ctypes.POINTER(ctypes.c_double)]),
        "fd_apply_stage": (ctypes.c_int, [vp, ctypes.c_int, dp, dp, ctypes.c_int64, ctypes.c_int64]),
        "fd_apply_scatter": (ctypes.c_int, [vp, ctypes.c_int, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                            ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
        "ls_matvec_slab": (ctypes.c_int, [vp, dp, ctypes.c_int64, ctypes.c_int64, dp, ctypes.c_int64,
                                          ctypes.c_int64]),
        "ls_matvec_slab3": (ctypes.c_int, [vp, dp, ctypes.c_int64, dp, ctypes.c_int64, dp, ctypes.c_int64,
                                           ctypes.c_int64, dp, ctypes.c_int64, ctypes.c_int64]),
        "ls_partition": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, i64p, i64p]),
        "ls_a2a_plan": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       i64p, i64p, i64p, i64p]),
        "ls_a2a_piece_plan": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int), i64p, i64p, i64p, i64p]),
        "ls_pack_map": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, i64p]),
        "ls_halo_plan": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        i64p, i64p, i64p, i64p]),
        "ls_strerror": (ctypes.c_char_p, [ctypes.c_int]),
        "ls_a2a_dest": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int), i64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def strerror(code):
    return load_library().ls_strerror(code).decode()


def _check(code, what, ok=(LS_OK,)):
    if code not in ok:
        raise LSError(code, what)
    return code


def unique_id():
    """128-byte NCCL unique id (rank 0), to broadcast before Context(..., world>1)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().ls_get_unique_id(buf), "ls_get_unique_id")
    return buf.raw


def partition(total, world, part):
    """(offset, length) of part `part` of the even split (host only, no GPU)."""
    off, ln = ctypes.c_int64(), ctypes.c_int64()
    _check(load_library().ls_partition(int(total), int(world), int(part), ctypes.byref(off),
                                       ctypes.byref(ln)), "ls_partition")
    return off.value, ln.value


def a2a_plan(n_t, N_s, world, rank):
    """slab -> chunk all-to-all plan of `rank`: dict of numpy arrays (host only)."""
    arrs = [np.zeros(world, dtype=np.int64) for _ in range(4)]
    ptrs = [a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) for a in arrs]
    _check(load_library().ls_a2a_plan(int(n_t), int(N_s), int(world), int(rank), *ptrs), "ls_a2a_plan")
    return dict(zip(("send_off", "send_cnt", "recv_off", "recv_cnt"), arrs))


def a2a_piece_plan(n_t, N_s, world, rank, piece):
    """ls_a2a_piece_plan: (pieces, [(send_off, send_cnt, recv_off, recv_cnt) per peer]) of one piece
    of the pipelined slab -> chunk all-to-all (piece < 0: only the number of pieces)."""
    np_ = ctypes.c_int(0)
    arrs = [(ctypes.c_int64 * max(world, 1))() for _ in range(4)]
    _check(load_library().ls_a2a_piece_plan(int(n_t), int(N_s), int(world), int(rank), int(piece),
                                            ctypes.byref(np_), *arrs), "ls_a2a_piece_plan")
    if piece < 0:
        return np_.value, []
    return np_.value, [tuple(int(a[h]) for a in arrs) for h in range(world)]


def pack_map(ntl, N_s, world):
    """Packed send position of every slab element (host only)."""
    pos = np.zeros(int(ntl) * int(N_s), dtype=np.int64)
    _check(load_library().ls_pack_map(int(ntl), int(N_s), int(world),
                                      pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))), "ls_pack_map")
    return pos


def a2a_dest(n_t, N_s, world, rank, direction, i, j):
    """(peer, offset) of one element in the fused all-to-all (host only)."""
    peer, off = ctypes.c_int(), ctypes.c_int64()
    _check(load_library().ls_a2a_dest(int(n_t), int(N_s), int(world), int(rank), int(direction), int(i), int(j),
                                      ctypes.byref(peer), ctypes.byref(off)), "ls_a2a_dest")
    return peer.value, off.value


def halo_plan(n_t, world, rank, p):
    """(t0, ntl, lo, hi) of the ls_matvec halo of `rank` (host only)."""
    v = [ctypes.c_int64() for _ in range(4)]
    _check(load_library().ls_halo_plan(int(n_t), int(world), int(rank), int(p), *[ctypes.byref(x) for x in v]),
           "ls_halo_plan")
    return tuple(x.value for x in v)


def _geometry_struct(geometry, d):
    """ls_geometry from the dict of synth.GEOMETRIES (the numpy arrays it points to are
    returned too: keep them alive while the struct is used)."""
    g = Geometry()
    keep = []
    for k in range(d):
        kn = np.ascontiguousarray(geometry["knots"][k], dtype=np.float64)
        keep.append(kn)
        g.degree[k] = int(geometry["degrees"][k])
        g.n_knots[k] = kn.size
        g.knots[k] = kn.ctypes.data
    ctrl = np.ascontiguousarray(geometry["ctrl"], dtype=np.float64)
    keep.append(ctrl)
    g.ctrl = ctrl.ctypes.data
    if geometry.get("weights") is not None:
        w = np.ascontiguousarray(geometry["weights"], dtype=np.float64)
        keep.append(w)
        g.weights = w.ctypes.data
    return g, keep


def pg_factors(geometry, p_s, n_elems):
    """ls_pg_factors (host only): (mu, omega, Mw, Jw, fit_rel_res) per direction."""
    d = geometry["d"]
    g, keep = _geometry_struct(geometry, d)
    ne = [int(v) for v in n_elems[:d]]
    nn = [v + p_s - 2 for v in ne]
    mu, om = np.zeros(sum(ne)), np.zeros(sum(ne))
    Mw, Jw = np.zeros(sum(v * v for v in nn)), np.zeros(sum(v * v for v in nn))
    res = ctypes.c_double()
    vp = lambda a: ctypes.c_void_p(a.ctypes.data)
    _check(load_library().ls_pg_factors(ctypes.byref(g), d, int(p_s), (ctypes.c_int64 * d)(*ne), vp(mu), vp(om),
                                         vp(Mw), vp(Jw), ctypes.byref(res)), "ls_pg_factors")
    del keep
    splits = np.cumsum(ne)[:-1]
    msplit = np.cumsum([v * v for v in nn])[:-1]
    return (np.split(mu, splits), np.split(om, splits),
            [m.reshape(n, n) for m, n in zip(np.split(Mw, msplit), nn)],
            [j.reshape(n, n) for j, n in zip(np.split(Jw, msplit), nn)], res.value)


def sizes(n_el, p):
    """(n_s, n_t) for n_el uniform elements (reading c1)."""
    return n_el + p - 2, n_el + p - 1


class Context:
    """One ls_ctx (one GPU).  ``p``: the degree, or (p_s, p_t) (ls_setup_deg); ``n_elems``:
    d+1 element counts, directions 1..d then time.  ``geometry``: a mapped spatial domain
    (dict with ``degrees``, ``knots``, ``ctrl`` [prod m][d] colex, ``weights`` or None;
    ls_setup_geo) with ``precond`` LS_PRECOND_P or LS_PRECOND_PG."""

    def __init__(self, d, p, n_elems, rank=0, world=1, uid=None, geometry=None, precond=LS_PRECOND_P):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1809_10026_b200 needs a CUDA device (no CPU fallback)")
        self._torch = torch
        lib = load_library()
        ne = (ctypes.c_int64 * (d + 1))(*[int(v) for v in n_elems])
        h = ctypes.c_void_p()
        torch.cuda.init()
        ps, pt = (p, p) if isinstance(p, int) else (int(p[0]), int(p[1]))
        if geometry is not None:
            g, keep = _geometry_struct(geometry, d)
            _check(lib.ls_setup_geo_dist(d, ps, pt, ne, ctypes.byref(g), int(precond), int(rank), int(world),
                                         uid, ctypes.byref(h)), "ls_setup_geo_dist")
        elif world == 1:
            _check(lib.ls_setup_deg(d, ps, pt, ne, ctypes.byref(h)), "ls_setup_deg")
        else:
            _check(lib.ls_setup_dist_deg(d, ps, pt, ne, rank, world, uid, ctypes.byref(h)), "ls_setup_dist_deg")
        self._h = h
        self._lib = lib
        self.d, self.p, self.p_s, self.p_t = d, p, ps, pt
        self.n_elems = list(n_elems)
        nt, t0, ntl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        ns = (ctypes.c_int64 * d)()
        _check(lib.ls_layout(h, ctypes.byref(nt), ns, ctypes.byref(t0), ctypes.byref(ntl)), "ls_layout")
        self.n_t, self.n_s = nt.value, [ns[k] for k in range(d)]
        self.t0, self.nt_local = t0.value, ntl.value
        self.shape = (self.nt_local,) + tuple(reversed(self.n_s))
        self.global_shape = (self.n_t,) + tuple(reversed(self.n_s))
        self.N = int(np.prod(self.shape))

    # -- marshalling helpers ------------------------------------------------------------
    def _dev(self, t, name):
        torch = self._torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
        if t.numel() != self.N:
            raise ValueError(f"{name} has {t.numel()} elements, expected {self.N}")
        return ctypes.c_void_p(t.data_ptr())

    def _chk(self, t, name, need):
        """Contiguous float64 CUDA tensor with at least ``need`` elements (the raw-pointer
        per-rank entry points cannot see buffer sizes)."""
        torch = self._torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
        if t.numel() < need:
            raise ValueError(f"{name} has {t.numel()} elements, needs {need}")

    def _new(self):
        return self._torch.empty(self.shape, dtype=self._torch.float64, device="cuda")

    def set_stream(self, stream):
        _check(self._lib.ls_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)), "ls_set_stream")

    # -- the boundary ---------------------------------------------------------------------
    def fd_apply(self, r, z=None):
        """z = P^{-1} r (Algorithm 1, PAPER.md 955-964)."""
        z = self._new() if z is None else z
        _check(self._lib.fd_apply(self._h, self._dev(r, "r"), self._dev(z, "z")), "fd_apply")
        return z

    def matvec(self, x, y=None):
        """y = A x (eq:A_kron, PAPER.md 686-703)."""
        y = self._new() if y is None else y
        _check(self._lib.ls_matvec(self._h, self._dev(x, "x"), self._dev(y, "y")), "ls_matvec")
        return y

    def fd_stage(self, stage, inp, out, a, b=0):
        """fd_apply_stage: 0/2 = forward/backward spatial modes on `a` time slices,
        1 = time mode of a spatial chunk [n_t][b] at spatial offset a."""
        Ns = int(np.prod(self.n_s))
        need = int(a) * Ns if stage in (0, 2) else self.n_t * int(b)
        for t, nm in ((inp, "in"), (out, "out")):
            self._chk(t, nm, need)
        _check(self._lib.fd_apply_stage(self._h, int(stage), ctypes.c_void_p(inp.data_ptr()),
                                        ctypes.c_void_p(out.data_ptr()), int(a), int(b)), "fd_apply_stage")
        return out

    def fd_scatter(self, stage, inp, a, b, world, me, dsts):
        """fd_apply_scatter: stage 0 = forward spatial modes of rank `me`'s slab scattered into
        the chunk buffers `dsts`; stage 1 = time mode of its chunk scattered into the slab
        buffers `dsts` (lists of `world` CUDA tensors)."""
        if len(dsts) != int(world):
            raise ValueError(f"dsts has {len(dsts)} buffers, expected world = {world}")
        Ns = int(np.prod(self.n_s))
        self._chk(inp, "inp", int(a) * Ns if stage == 0 else self.n_t * int(b))
        for t in dsts:
            # receive buffers: a spatial chunk [n_t][chunk] (stage 0) or a time slab (stage 1);
            # the library cannot see their sizes, so at least the smaller bound is enforced
            self._chk(t, "dsts[i]", 1)
        arr = (ctypes.c_void_p * world)(*[t.data_ptr() for t in dsts])
        _check(self._lib.fd_apply_scatter(self._h, int(stage), ctypes.c_void_p(inp.data_ptr()), int(a), int(b),
                                          int(world), int(me), arr), "fd_apply_scatter")

    def matvec_slab(self, x_ext, s_first, t_first, nout, y=None):
        """Rows [t_first, t_first + nout) of A x from the stored rows [s_first, s_first +
        x_ext.shape[0]) of x (ls_matvec_slab)."""
        torch = self._torch
        Ns = int(np.prod(self.n_s))
        self._chk(x_ext, "x_ext", 1)
        if x_ext.numel() % Ns:
            raise ValueError(f"x_ext has {x_ext.numel()} elements, not a whole number of time slices of {Ns}")
        s_rows = x_ext.numel() // Ns
        if y is None:
            y = torch.empty((nout,) + tuple(self.shape[1:]), dtype=torch.float64, device="cuda")
        self._chk(y, "y", int(nout) * Ns)
        _check(self._lib.ls_matvec_slab(self._h, ctypes.c_void_p(x_ext.data_ptr()), int(s_first), int(s_rows),
                                        ctypes.c_void_p(y.data_ptr()), int(t_first), int(nout)), "ls_matvec_slab")
        return y

    def matvec_slab3(self, x_lo, x_own, x_hi, s_first, t_first, nout, y=None):
        """ls_matvec_slab3: as matvec_slab with the stored rows in three buffers (lower halo rows,
        own rows, upper halo rows; a halo may be None for zero rows)."""
        torch = self._torch
        Ns = int(np.prod(self.n_s))
        parts = []
        for t, name in ((x_lo, "x_lo"), (x_own, "x_own"), (x_hi, "x_hi")):
            if t is None:
                parts.append((None, 0))
                continue
            self._chk(t, name, 1)
            if t.numel() % Ns:
                raise ValueError(f"{name} has {t.numel()} elements, not a whole number of time slices of {Ns}")
            parts.append((t, t.numel() // Ns))
        if parts[1][0] is None:
            raise ValueError("x_own is required")
        if y is None:
            y = torch.empty((nout,) + tuple(self.shape[1:]), dtype=torch.float64, device="cuda")
        self._chk(y, "y", int(nout) * Ns)
        ptr = [ctypes.c_void_p(t.data_ptr() if t is not None else 0) for t, _ in parts]
        _check(self._lib.ls_matvec_slab3(self._h, ptr[0], parts[0][1], ptr[1], parts[1][1], ptr[2], parts[2][1],
                                         int(s_first), ctypes.c_void_p(y.data_ptr()), int(t_first), int(nout)),
               "ls_matvec_slab3")
        return y

    def rhs(self, kind, b=None):
        """b = F(B_i) for forcing `kind` (0: e^t prod sin, 1: cube manufactured)."""
        b = self._new() if b is None else b
        _check(self._lib.ls_rhs(self._h, int(kind), self._dev(b, "b")), "ls_rhs")
        return b

    def pcg(self, b, x=None, tol=1e-8, max_iter=1000, raise_on_noconv=False):
        """x = A^{-1} b by PCG with P; returns (x, stats dict)."""
        x = self._new() if x is None else x
        st = PCGStats()
        code = self._lib.pcg_solve(self._h, self._dev(b, "b"), self._dev(x, "x"), float(tol),
                                   int(max_iter), ctypes.byref(st))
        _check(code, "pcg_solve", ok=(LS_OK,) if raise_on_noconv else (LS_OK, LS_ENOCONV, LS_ENUMERIC))
        return x, st.as_dict()

    def energy_error(self, kind, x):
        """ls_energy_error: dict(J, f2, bx, xAx) of the least-squares functional at x."""
        out = (ctypes.c_double * 4)()
        _check(self._lib.ls_energy_error(self._h, int(kind), self._dev(x, "x"), out), "ls_energy_error")
        return {"J": out[0], "f2": out[1], "bx": out[2], "xAx": out[3]}

    def error_norms(self, kind, x):
        """ls_error_norms: the space-time integrals of e = u - u_h and of u (kind 1: cube,
        kind 2: quarter annulus) and the relative V_0, L^2, H^1 errors derived from them."""
        o = (ctypes.c_double * 8)()
        _check(self._lib.ls_error_norms(self._h, int(kind), self._dev(x, "x"), o), "ls_error_norms")
        v = list(o)
        return {"e_L2": v[0], "e_dt": v[1], "e_grad": v[2], "e_lap": v[3],
                "u_L2": v[4], "u_dt": v[5], "u_grad": v[6], "u_lap": v[7],
                "rel_V0": float(np.sqrt((v[1] + v[3]) / (v[5] + v[7]))),
                "rel_L2": float(np.sqrt(v[0] / v[4])),
                "rel_H1": float(np.sqrt((v[0] + v[1] + v[2]) / (v[4] + v[5] + v[6])))}

    def fd_apply_host(self, r_host, z_host):
        """fd_apply on host tensors/arrays (pinned recommended); synchronous."""
        def ptr(a, name):
            if hasattr(a, "data_ptr"):
                if a.is_cuda or a.dtype != self._torch.float64 or not a.is_contiguous():
                    raise TypeError(f"{name} must be a contiguous float64 CPU tensor")
                return ctypes.c_void_p(a.data_ptr())
            a = np.ascontiguousarray(a)
            if a.dtype != np.float64:
                raise TypeError(f"{name} must be float64")
            return ctypes.c_void_p(a.ctypes.data)
        _check(self._lib.fd_apply_host(self._h, ptr(r_host, "r"), ptr(z_host, "z")), "fd_apply_host")
        return z_host

    def fd_apply_host_batch(self, rs, zs):
        """fd_apply_host over lists of host vectors, copies of neighbouring vectors overlapped
        with the application (pinned memory recommended); synchronous."""
        if len(rs) != len(zs):
            raise ValueError("rs and zs must have the same length")
        need = self.N

        def ptr(a, name):
            if hasattr(a, "data_ptr"):
                if a.is_cuda or a.dtype != self._torch.float64 or not a.is_contiguous():
                    raise TypeError(f"{name} must be a contiguous float64 CPU tensor")
                n, p = a.numel(), a.data_ptr()
            else:
                if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
                    raise TypeError(f"{name} must be a C-contiguous float64 array")
                n, p = a.size, a.ctypes.data
            if n != need:
                raise ValueError(f"{name} has {n} elements, expected {need}")
            return p
        k = len(rs)
        rp = (ctypes.c_void_p * max(k, 1))(*[ptr(a, "r") for a in rs])
        zp = (ctypes.c_void_p * max(k, 1))(*[ptr(a, "z") for a in zs])
        _check(self._lib.fd_apply_host_batch(self._h, ctypes.cast(rp, ctypes.c_void_p),
                                             ctypes.cast(zp, ctypes.c_void_p), k), "fd_apply_host_batch")
        return zs

    def get_factor(self, which, direction=0):
        """Setup quantities (see ls_get_factor): returns a numpy array."""
        if which in (0, 1, 2, 7):
            n = self.n_s[direction - 1]
            shape = (n, n)
        elif which in (3, 4, 8):
            shape = (self.n_t, self.n_t)
        elif which == 5:
            shape = (self.n_s[direction - 1],)
        elif which == 6:
            shape = (self.n_t,)
        else:
            raise ValueError("unknown factor")
        out = np.empty(shape, dtype=np.float64)
        _check(self._lib.ls_get_factor(self._h, int(which), int(direction),
                                       ctypes.c_void_p(out.ctypes.data)), "ls_get_factor")
        return out

    def geo_info(self):
        """ls_geo_info: (separable-fit residual, stencil entries per row)."""
        out = (ctypes.c_double * 2)()
        _check(self._lib.ls_geo_info(self._h, out), "ls_geo_info")
        return out[0], int(out[1])

    def tune(self, knob, value):
        """ls_tune: select an equivalent implementation (knobs LS_TUNE_*, include/ls_api.h;
        e.g. LS_TUNE_FD_KERNEL: 0 auto, 1 shared-memory staged, 2 register-direct)."""
        _check(self._lib.ls_tune(self._h, int(knob), int(value)), "ls_tune")

    def profile(self, enable):
        """Start/stop CUDA-event timing of every FD mode-product launch."""
        _check(self._lib.ls_profile(self._h, int(bool(enable))), "ls_profile")

    def profile_read(self):
        """(total_ms, total_algorithmic_flops, launches) since the last read."""
        ms, fl, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(self._lib.ls_profile_read(self._h, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(n)),
               "ls_profile_read")
        return ms.value, fl.value, n.value

    @property
    def launches(self):
        return int(self._lib.ls_kernel_launches(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.ls_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
