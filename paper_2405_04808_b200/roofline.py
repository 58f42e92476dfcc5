"""Algorithmic HBM bytes per C-ABI call (the roofline numerators).

Per-unit figures ("Kernels and their rooflines"): every vector
element read or written once, stage data read once, halo re-reads and the
constant weights counted as cache hits (0 bytes).  ``dim = N*(4nu+nz)``.

  stage bytes / interval   DENSE: 8*(2*nu*nu + nu*nz)   TRI: 8*6*nu
  jacobi sweep             8*dim*(b + out [+ x_in]) + stage; omega = 1: x enters only
                           through the couplings u_{i-1}, mu_{i+1}: 8*dim*2 + 16*N*nu + stage
  diag solve / subst       8*dim*2 + stage
  apply / apply_diag       8*dim*2 + stage ;  residual 8*dim*3 + stage
  residual_restrict        DENSE: residual + restrict as separate passes;
                           TRI (fused): 8*N*(2nu+nz) of b (v,mu,z of even rows, u,lam,z
                           of odd rows) + 8*N*(3nu+nz) of x + 8*coarse_dim written
                           + 3/4 of the stage data (C of even rows, K and C of odd rows)
  restrict                 8*(coarse_dim + Nc*nz) read + 8*coarse_dim write
  prolong_add              8*(2*fine_dim + coarse_dim)
  jacobi0_restrict         8*dim*2 + 8*coarse_dim + stage (zero-start sweep + restricted residual)
  jacobi0_restrict_um      8*dim + 16*N*nu (u, mu of x) + 8*coarse_dim + stage
  jacobi_prolong           8*dim*2 + 16*N*nu (u, mu of x) + 8*N*nu (u, mu of the coarse
                           correction: 2 segments per coarse row) + stage
  dot 16n, nrm2 8n, axpy 24n, scale_into 16n, rsub 24n, gemv_t_add 8n(k+2)
"""

from __future__ import annotations


def _lvl(lref):
    return lref._obj


def stage_bytes(L) -> int:
    N, nu, nz = L.n_steps, L.n_u, L.n_z
    if L.family == 0:
        return 8 * N * (2 * nu * nu + nu * nz)
    return 8 * N * 6 * nu


def dim_of(L) -> int:
    return L.n_steps * (4 * L.n_u + L.n_z)


def algorithmic_bytes(name: str, args) -> int:
    if name == "tk_jacobi_sweep":
        L = _lvl(args[0])
        if args[2] and float(args[4]) == 1.0:   # D^{-1}(b + (L+U) x): two coupling segments of x
            return 8 * dim_of(L) * 2 + 16 * L.n_steps * L.n_u + stage_bytes(L)
        nvec = 2 + (1 if args[2] else 0)
        return 8 * dim_of(L) * nvec + stage_bytes(L)
    if name == "tk_jacobi0_restrict":   # b read, x and the coarse rhs written, stage data
        L = _lvl(args[0])
        cdim = (L.n_steps // 2) * (4 * L.n_u + L.n_z)
        return 8 * dim_of(L) * 2 + 8 * cdim + stage_bytes(L)
    if name == "tk_jacobi0_restrict_um":   # b read; u, mu of x and the coarse rhs written
        L = _lvl(args[0])
        cdim = (L.n_steps // 2) * (4 * L.n_u + L.n_z)
        return 8 * dim_of(L) + 16 * L.n_steps * L.n_u + 8 * cdim + stage_bytes(L)
    if name == "tk_jacobi_prolong":        # b, u/mu of x and of ec read; x_out written
        L = _lvl(args[0])
        return 8 * dim_of(L) * 2 + 16 * L.n_steps * L.n_u + 8 * L.n_steps * L.n_u + stage_bytes(L)
    if name in ("tk_diag_solve", "tk_forward_subst", "tk_backward_subst", "tk_sgs_back_half",
                "tk_kkt_apply", "tk_kkt_apply_diag"):
        L = _lvl(args[0])
        return 8 * dim_of(L) * 2 + stage_bytes(L)
    if name == "tk_kkt_residual":
        L = _lvl(args[0])
        return 8 * dim_of(L) * 3 + stage_bytes(L)
    if name == "tk_residual_restrict":
        L = _lvl(args[0])
        nc = L.n_steps // 2
        cdim = nc * (4 * L.n_u + L.n_z)
        if L.family == 1:   # fused kernel: the parts the restriction keeps
            N, nu, nz = L.n_steps, L.n_u, L.n_z
            return 8 * (N * (2 * nu + nz) + N * (3 * nu + nz) + cdim) + (3 * stage_bytes(L)) // 4
        return 8 * dim_of(L) * 3 + stage_bytes(L) + 8 * (2 * cdim + nc * L.n_z)
    if name == "tk_residual_restrict_jacobi0":   # coarse vector written, u/mu segments read
        L = _lvl(args[0])
        nc = L.n_steps // 2
        cdim = nc * (4 * L.n_u + L.n_z)
        extra = 0 if float(args[3]) == 1.0 else 8 * (cdim + nc * L.n_z)   # (1-omega) b
        return 8 * cdim + 8 * 2 * L.n_u * nc + extra
    if name in ("tk_restrict", "tk_prolong_add"):
        nf, nu, nz = args[0], args[1], args[2]
        fdim = nf * (4 * nu + nz)
        cdim = (nf // 2) * (4 * nu + nz)
        if name == "tk_restrict":
            return 8 * (2 * cdim + (nf // 2) * nz)
        return 8 * (2 * fdim + cdim)
    if name == "tk_arnoldi_mgs":   # V_0..V_j and V_j+1 once, w read+written per pass
        n, j = int(args[0]), int(args[1])
        return 8 * n * ((j + 2) + 2 * (j + 2))
    if name == "tk_copy_kernel":
        return 16 * int(args[0])
    n = int(args[0])
    return {"tk_dot": 16 * n, "tk_nrm2": 8 * n, "tk_axpy": 24 * n, "tk_scale_into": 16 * n,
            "tk_rsub": 24 * n}.get(name, 8 * n * ((int(args[1]) + 2) if name == "tk_gemv_t_add"
                                                 else 0))
