"""CPU oracle for the space-time least-squares IGA hot path (arXiv 1809.10026).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1809_10026_b200``) never imports it, and this
package never imports the product: the two share no code.

Everything here is plain numpy/scipy in fp64, written to be checked against
PAPER.md by eye:

* ``bspline``    -- open knot vectors and the Cox-de Boor recursion (PAPER.md
                    lines 144-170, Sec. 2.1).
* ``univariate`` -- the univariate factor matrices M, K, J, G, M_t, K_t, W_t with
                    the paper's boundary / initial conditions (eq:basis_par,
                    PAPER.md 266-267; Sec. 4.1-4.2, 678-757).
* ``fd``         -- Algorithm 1 (Fast Diagonalization, PAPER.md 929-964) and the
                    dense Kronecker-assembled P for brute force.
* ``operator``   -- y = A x with A = K_t(x)M_s + M_t(x)J_s + W_t(x)L_s
                    (eq:A_kron, PAPER.md 686-703), and a dense A from direct
                    space-time quadrature of the ORIGINAL bilinear form
                    (PAPER.md 406) for tiny grids.
* ``rhs``        -- b_i = F(B_i) = int int f (d_t B_i - Lap B_i) (PAPER.md 409).
* ``pcg``        -- textbook preconditioned CG, x0 = 0, tol on the recurrence
                    residual (PAPER.md 710-712, 1109).
* ``geometry``   -- mapped domains Omega = F([0,1]^d) (NURBS map, chain rule of
                    PAPER.md 986-990): physical spatial factors M_s, L_s, J_s of
                    eq:A_kron and the dense original-form A on tiny grids.
* ``geo_precond``-- the geometry-aware preconditioner P^G (Sec. 4.4, PAPER.md
                    969-1045): midpoint coefficients, separable fit, weighted
                    univariate factors, diagonal scaling.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``; see DESIGN.md "Oracle pins".  No function is
"parity unpinned".
"""

from . import bspline, univariate, fd, operator, rhs, pcg, geometry, geo_precond  # noqa: F401
