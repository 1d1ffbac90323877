"""Fast Diagonalization, Algorithm 1 (oracle; test infrastructure).

PAPER.md 929-964 (Sec. 4.3).  P s = r with (eq:preconditioner, PAPER.md 733,
752-760)
    P = K_t-hat (x) M_s-hat + M_t-hat (x) J_s-tilde,
    M_s-hat = M_d (x) ... (x) M_1,
    J_s-tilde = sum_k M_d (x) .. (x) J_k (x) .. (x) M_1.
Step 1 (eq:eig_dec, PAPER.md 939-945): J_k U_k = M_k U_k Lambda_k,
K_t U_t = M_t U_t Lambda_t, normalised U^T M U = I (reading c4).
Step 2: s~ = (U_t (x) U_s)^T r;  Step 3: q~ = (Lambda_t (x) I + I (x) Lambda_s)^{-1} s~;
Step 4: z = (U_t (x) U_s) q~   (reading c2: r is the input, z the output).
Reading c3: the divisor at multi-index (i_t, i_d, .., i_1) is
lambda_t[i_t] + sum_k lambda_k[i_k].

Tensor convention: a vector of length N = n_t * prod n_k is held as an array of
shape (n_t, n_d, ..., n_1) in C order, i.e. the colexicographic DOF order of
PAPER.md 271-285 (direction 1 fastest, time slowest).  Direction k (1-based)
is axis d + 1 - k; time is axis 0.
"""

import numpy as np
import scipy.linalg


def generalized_eig(Kmat, Mmat, refine=2):
    """Kmat U = Mmat U diag(lam), U^T Mmat U = I, lam ascending -- eq:eig_dec,
    PAPER.md 942-945.

    LAPACK (scipy.linalg.eigh, sygvd) in fp64, then ``refine`` steps of the
    Ogita-Aishima eigenpair refinement (Ogita & Aishima 2018, generalised to the
    pencil) evaluated in 80-bit extended precision (reading c17):
        R = I - X^T M X,  S = X^T K X,  lam_i = s_ii / (1 - r_ii),
        E_ij = (s_ij + lam_j r_ij) / (lam_j - lam_i)  (i != j),  E_ii = r_ii / 2,
        X <- X + X E.
    fp64 LAPACK leaves the smallest eigenvalues -- which dominate P^{-1} r --
    with relative errors up to ~eps*lambda_max/lambda_min (measured 2e-11 ..
    3.4e-10 against 34-digit mpmath); the refinement brings them to ~1e-14.
    The spectra here are simple (1D Sturm-Liouville-type pencils), so no
    cluster handling is needed; refine=0 gives plain LAPACK."""
    lam, U = scipy.linalg.eigh(Kmat, Mmat)
    if refine == 0:
        return lam, U
    ld = np.longdouble
    K, M, X = Kmat.astype(ld), Mmat.astype(ld), U.astype(ld)
    n = K.shape[0]
    for _ in range(refine):
        R = np.eye(n, dtype=ld) - X.T @ (M @ X)
        S = X.T @ (K @ X)
        lt = np.diag(S) / (1 - np.diag(R))
        gap = lt[None, :] - lt[:, None]            # lam_j - lam_i
        # near-degenerate pairs (the two boundary "outlier" eigenvalues at the top
        # of high-degree spectra differ by ~1e-11 relative): Ogita-Aishima's
        # cluster rule E_ij = r_ij / 2 (re-orthonormalise, no rotation)
        clustered = np.abs(gap) <= 1e-6 * np.maximum(np.abs(lt[None, :]), np.abs(lt[:, None]))
        gap[clustered] = 1
        E = (S + R * lt[None, :]) / gap
        E[clustered] = R[clustered] / 2
        X = X + X @ E
    lam = (np.diag(X.T @ (K @ X)) / np.diag(X.T @ (M @ X))).astype(np.float64)
    return lam, X.astype(np.float64)


def setup(space, time):
    """Algorithm 1 step 1.  ``space`` = [dict(M=, J=) for directions 1..d],
    ``time`` = dict(Mt_hat=, Kt_hat=)."""
    lam_s, U_s = [], []
    for f in space:
        lam, U = generalized_eig(f["J"], f["M"])
        lam_s.append(lam)
        U_s.append(U)
    lam_t, U_t = generalized_eig(time["Kt_hat"], time["Mt_hat"])
    return {"lam_s": lam_s, "U_s": U_s, "lam_t": lam_t, "U_t": U_t, "d": len(space)}


def mode_apply(X, C, axis):
    """Y[.., a, ..] = sum_i C[a, i] X[.., i, ..] along ``axis`` (the mode-k product
    X x_k C; with eq:kron_vec, PAPER.md 646, this is (I (x) C (x) I) vec X)."""
    return np.moveaxis(np.tensordot(C, X, axes=([1], [axis])), 0, axis)


def divisor(fdd):
    """Lambda_t (x) I + I (x) Lambda_s as a tensor of shape (n_t, n_d, .., n_1)
    (PAPER.md 947-950, reading c3)."""
    d = fdd["d"]
    D = fdd["lam_t"].reshape((-1,) + (1,) * d)
    for k in range(1, d + 1):
        shape = [1] * (d + 1)
        shape[d + 1 - k] = -1
        D = D + fdd["lam_s"][k - 1].reshape(shape)
    return D


def fd_apply(r, fdd):
    """z = P^{-1} r by Algorithm 1 steps 2-4 (PAPER.md 959-962)."""
    d = fdd["d"]
    s = np.array(r, dtype=np.float64, copy=True)
    # Step 2: s~ = (U_t (x) U_d (x) .. (x) U_1)^T r
    for k in range(1, d + 1):
        s = mode_apply(s, fdd["U_s"][k - 1].T, d + 1 - k)
    s = mode_apply(s, fdd["U_t"].T, 0)
    # Step 3: divide by lambda_t + sum_k lambda_k
    q = s / divisor(fdd)
    # Step 4: z = (U_t (x) U_s) q~
    z = mode_apply(q, fdd["U_t"], 0)
    for k in range(1, d + 1):
        z = mode_apply(z, fdd["U_s"][k - 1], d + 1 - k)
    return z


def kron_list(mats):
    """mats[0] (x) mats[1] (x) ... (Kronecker product, PAPER.md 615-624)."""
    out = np.ones((1, 1))
    for A in mats:
        out = np.kron(out, A)
    return out


def dense_P(space, time):
    """Dense P = K_t-hat (x) M_s-hat + M_t-hat (x) J_s-tilde (PAPER.md 733, 752-757)
    for brute-force checks on tiny grids.  Kronecker factors are listed slowest
    first: time, direction d, ..., direction 1."""
    d = len(space)
    Ms = kron_list([space[k]["M"] for k in reversed(range(d))])
    Js = np.zeros_like(Ms)
    for k in range(d):  # direction k+1 carries J
        Js += kron_list([space[l]["J"] if l == k else space[l]["M"]
                         for l in reversed(range(d))])
    return np.kron(time["Kt_hat"], Ms) + np.kron(time["Mt_hat"], Js)


def fd_apply_rank1_rows(factors, fdd, rows):
    """Algorithm 1 on a rank-1 input r = a_t (x) a_d (x) ... (x) a_1
    (``factors`` = [a_t, a_d, .., a_1], slowest first), returning only the
    output fibres z[rows[j] + (:,)] along direction 1.  Step 2 is exact on the
    rank-1 structure (s~ = (U_t^T a_t) (x) ... (x) (U_1^T a_1)); step 3 forms
    q~ = s~ / (lambda_t + sum_k lambda_k) in full; step 4 is evaluated only for
    the requested fibres.  Used for full-size (BASELINE config 4) parity."""
    d = fdd["d"]
    U = [fdd["U_t"]] + [fdd["U_s"][k - 1] for k in range(d, 0, -1)]  # slowest first
    sig = [U[a].T @ factors[a] for a in range(d + 1)]
    q = sig[0]
    for v in sig[1:]:
        q = np.multiply.outer(q, v)
    q = q / divisor(fdd)
    out = []
    for idx in rows:  # idx = (i_t, i_d, .., i_2)
        v = q
        for a, i in enumerate(idx):
            v = np.tensordot(U[a][i], v, axes=([0], [0]))
        out.append(U[d] @ v)
    return np.array(out)
