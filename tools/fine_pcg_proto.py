"""CPU prototype for the device fine-reference solver's preconditioner choice
(developer tool): PCG on the global 5-point system (elliptic.cpp:68-243) with
block-Jacobi over the subdomains + a piecewise-constant coarse space
(additive or deflated), against a sparse direct solve.
Usage: python tools/fine_pcg_proto.py C2 [additive|deflated] [tol]"""
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spl

sys.path.insert(0, ".")
from paper_2103_11050_b200 import configs  # noqa: E402


def assemble(nx, ny, lx, ly, kappa, kind, val):
    hx, hy = lx / nx, ly / ny
    K = kappa.reshape(ny, nx)
    harm = lambda a, b: 2 * a * b / (a + b)  # noqa: E731
    rows, cols, vals = [], [], []
    diag = np.zeros((ny, nx))
    b = np.zeros((ny, nx))
    tv = harm(K[:, :-1], K[:, 1:]) * hy / hx  # vertical interior faces i=1..nx-1
    th = harm(K[:-1, :], K[1:, :]) * hx / hy
    idx = np.arange(nx * ny).reshape(ny, nx)
    diag[:, :-1] += tv; diag[:, 1:] += tv
    diag[:-1, :] += th; diag[1:, :] += th
    rows += [idx[:, 1:].ravel(), idx[:, :-1].ravel()]; cols += [idx[:, :-1].ravel(), idx[:, 1:].ravel()]; vals += [-tv.ravel()] * 2
    rows += [idx[1:, :].ravel(), idx[:-1, :].ravel()]; cols += [idx[:-1, :].ravel(), idx[1:, :].ravel()]; vals += [-th.ravel()] * 2
    # boundary faces W(ny) E(ny) S(nx) N(nx)
    sides = [(K[:, 0], hy, hx, (slice(None), 0)), (K[:, -1], hy, hx, (slice(None), -1)),
             (K[0, :], hx, hy, (0, slice(None))), (K[-1, :], hx, hy, (-1, slice(None)))]
    off = 0
    for kk, area, h, sl in sides:
        n = kk.size
        kd, v = kind[off:off + n], val[off:off + n]
        t = kk * area / (h / 2)
        dd = np.where(kd == 0, t, 0.0)
        rb = np.where(kd == 0, t * v, np.where(kd == 1, -v * area, 0.0))
        diag[sl] += dd
        b[sl] += rb
        off += n
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(nx * ny,) * 2)
    A = A + sp.diags(diag.ravel())
    return A.tocsr(), b.ravel()


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    mode = sys.argv[2] if len(sys.argv) > 2 else "additive"
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-13
    cfg = configs.build(name)
    P = cfg.problem
    rng = np.random.default_rng(0)
    s = rng.uniform(0, 1, P.nx * P.ny) * 0.0
    M = P.viscosity_ratio
    lam = M * s * s + (1 - s) ** 2
    solve(P, P.K * lam, mode, tol, name)


def solve(P, kappa, mode="deflated", tol=1e-13, name=""):
    A, b = assemble(P.nx, P.ny, P.lx, P.ly, kappa, np.asarray(P.bc.kind), np.asarray(P.bc.value))
    t = time.time(); xd = spl.spsolve(A.tocsc(), b); print("direct", time.time() - t)
    snx, sny = P.nx // P.nsx, P.ny // P.nsy
    sub = ((np.arange(P.ny) // sny)[:, None] * P.nsx + (np.arange(P.nx) // snx)[None, :]).ravel()
    nsub = P.nsx * P.nsy
    R0 = sp.csr_matrix((np.ones(P.nx * P.ny), (sub, np.arange(P.nx * P.ny))), shape=(nsub, P.nx * P.ny))
    A0 = (R0 @ A @ R0.T).toarray()
    A0i = np.linalg.inv(A0)
    blocks = []
    for k in range(nsub):
        ids = np.where(sub == k)[0]
        blocks.append((ids, spl.splu(A[ids][:, ids].tocsc())))

    def bj(r):
        z = np.zeros_like(r)
        for ids, lu in blocks:
            z[ids] = lu.solve(r[ids])
        return z

    def coarse(r):
        return R0.T @ (A0i @ (R0 @ r))

    if mode == "additive":
        prec = lambda r: bj(r) + coarse(r)  # noqa: E731
        x = np.zeros_like(b)
    elif mode == "bnn":  # balancing: P = (I - QA) B^-1 (I - AQ) + Q
        def prec(r):
            y = bj(r - A @ coarse(r))
            return y - coarse(A @ y) + coarse(r)
        x = np.zeros_like(b)
    else:  # deflated (A-DEF2): P = Q + (I - Q A) B^-1, x0 = Q b
        def prec(r):
            y = bj(r)
            return y - coarse(A @ y) + coarse(r)
        x = coarse(b)
    r = b - A @ x
    z = prec(r); p = z.copy(); rho = r @ z
    bb = np.sqrt(b @ b)
    for it in range(1, 3000):
        q = A @ p
        al = rho / (p @ q)
        x += al * p; r -= al * q
        rn = np.sqrt(r @ r) / bb
        if rn < tol:
            break
        z = prec(r); rho2 = r @ z; p = z + (rho2 / rho) * p; rho = rho2
    # velocity error proxy: interior fluxes T (x_L - x_R)
    e = np.linalg.norm(x - xd) / np.linalg.norm(xd)
    print(f"{name} {mode} iters {it} relres {rn:.2e} p rel err {e:.2e}")


if __name__ == "__main__":
    main()
