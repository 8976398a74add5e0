"""CPU restatement of the reference's STMG solve path in numpy/scipy.

TEST INFRASTRUCTURE ONLY (the checker; never imported by the product). Each
function cites the reference routine it restates (paths relative to
/root/reference/proj). It is pinned against the reference's own C++ compiled
in oracle/_ref (tests/test_oracle_np.py) and against the known-answer tests
of the reference's test-suite (tests/test_oracle.py).

Vectors use the reference layout: index (s*n_t + i)*n_space + g, with the
lexicographic Q_p lattice index g (x fastest).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

HEAT, WAVE = 0, 1
DG, CGP = 0, 1
SPACE_H, SPACE_P, TIME_TAU, TIME_K = 0, 1, 2, 3


# --------------------------------------------------------------- quadrature
def _legendre(n, x):
    """P_n(x), P_n'(x) (src/quadrature.cpp:18-34)."""
    x = np.asarray(x, dtype=float)
    p0, p1 = np.ones_like(x), x.copy()
    if n == 0:
        return p0, np.zeros_like(x)
    for j in range(2, n + 1):
        p0, p1 = p1, ((2 * j - 1) * x * p1 - (j - 1) * p0) / j
    with np.errstate(divide="ignore", invalid="ignore"):
        dp = n * (x * p1 - p0) / (x * x - 1.0)
    return p1, dp


def _newton(f, x0):
    x = np.asarray(x0, dtype=float)
    for _ in range(100):
        v, d = f(x)
        dx = v / d
        x = x - dx
        if np.max(np.abs(dx)) < 1e-16:
            break
    return x


def gauss(n):
    """n-point Gauss-Legendre rule on [0,1] (src/quadrature.cpp:98-111)."""
    x, w = np.polynomial.legendre.leggauss(n)
    x = _newton(lambda t: _legendre(n, t), x)
    _, dp = _legendre(n, x)
    w = 2.0 / ((1 - x * x) * dp * dp)
    return 0.5 * (x + 1), 0.5 * w


def gauss_lobatto(n):
    """n-point Gauss-Lobatto rule on [0,1] (src/quadrature.cpp:113-137)."""
    m = n - 1
    xi = -np.cos(np.pi * np.arange(1, n - 1) / m)
    if n > 2:
        def f(t):
            p, dp = _legendre(m, t)
            return dp, (2 * t * dp - m * (m + 1) * p) / (1 - t * t)
        xi = _newton(f, xi)
    x = np.concatenate([[-1.0], np.sort(xi), [1.0]])
    p = np.where(np.abs(x) == 1.0, np.where((x > 0) | (m % 2 == 0), 1.0, -1.0), _legendre(m, x)[0])
    w = 2.0 / (n * (n - 1.0) * p * p)
    r = 0.5 * (x + 1)
    r[0], r[-1] = 0.0, 1.0
    return r, 0.5 * w


def gauss_radau_right(n):
    """n-point right Gauss-Radau rule on [0,1] (src/quadrature.cpp:139-166)."""
    if n == 1:
        return np.array([1.0]), np.array([1.0])
    xi = -np.cos(2 * np.pi * np.arange(1, n) / (2 * n - 1))

    def f(t):
        pa, da = _legendre(n - 1, t)
        pb, db = _legendre(n, t)
        return pa + pb, da + db
    xi = _newton(f, xi)
    p, _ = _legendre(n - 1, xi)
    x = np.concatenate([[-1.0], xi])
    w = np.concatenate([[2.0 / (n * n)], (1 - xi) / (n * n * p * p)])
    order = np.argsort(-x)
    r = 0.5 * (-x[order] + 1)
    r[-1] = 1.0
    return r, 0.5 * w[order]


def lagrange(nodes, i, t):
    """Cardinal polynomial value (src/lagrange.cpp:20-27)."""
    v = np.ones_like(np.asarray(t, dtype=float))
    for j, xj in enumerate(nodes):
        if j != i:
            v = v * (t - xj) / (nodes[i] - xj)
    return v


def lagrange_deriv(nodes, i, t):
    """Cardinal polynomial derivative (src/lagrange.cpp:29-42)."""
    t = np.asarray(t, dtype=float)
    s = np.zeros_like(t)
    for m in range(len(nodes)):
        if m == i:
            continue
        term = np.ones_like(t) / (nodes[i] - nodes[m])
        for j in range(len(nodes)):
            if j != i and j != m:
                term = term * (t - nodes[j]) / (nodes[i] - nodes[j])
        s = s + term
    return s


# --------------------------------------------------------- temporal weights
@dataclasses.dataclass
class Weights:
    scheme: int
    k: int
    n_t: int
    m: np.ndarray
    a: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    trial: np.ndarray
    unknown_nodes: np.ndarray

    def unknown_weight(self, i, t):  # src/temporal_weights.cpp:8-12
        return lagrange(self.trial, i if self.scheme == DG else i + 1, t)

    def left_weight(self, t):  # src/temporal_weights.cpp:14-18
        return 0.0 if self.scheme == DG else lagrange(self.trial, 0, t)


def dg_weights(k):
    """DG(k) on right Radau nodes (src/temporal_weights.cpp:29-64)."""
    trial = gauss_radau_right(k + 1)[0]
    qx, qw = gauss(k + 1)
    n = k + 1
    phi = np.array([lagrange(trial, i, qx) for i in range(n)])
    dphi = np.array([lagrange_deriv(trial, i, qx) for i in range(n)])
    m = (phi * qw) @ phi.T
    a = ((phi * qw) @ dphi.T)
    phi0 = np.array([lagrange(trial, i, 0.0) for i in range(n)])
    a = a + np.outer(phi0, phi0)
    return Weights(DG, k, n, m, a, phi0.copy(), np.zeros(n), trial, trial.copy())


def cgp_weights(k):
    """CGP(k) on Gauss-Lobatto nodes (src/temporal_weights.cpp:66-106)."""
    trial = gauss_lobatto(k + 1)[0]
    test = trial[1:]
    qx, qw = gauss(k + 1)
    psi = np.array([lagrange(test, i, qx) for i in range(k)])
    xi = np.array([lagrange(trial, j, qx) for j in range(k + 1)])
    dxi = np.array([lagrange_deriv(trial, j, qx) for j in range(k + 1)])
    mm = (psi * qw) @ xi.T
    aa = (psi * qw) @ dxi.T
    return Weights(CGP, k, k, mm[:, 1:], aa[:, 1:], aa[:, 0].copy(), mm[:, 0].copy(), trial, test.copy())


def block_coefficients(eq, w: Weights, tau, s, j):
    """(step s, step j) temporal coupling of the slab matrix
    (src/space_time_operator.cpp:269-317)."""
    nt = w.n_t
    cM, cA = np.zeros((nt, nt)), np.zeros((nt, nt))
    if j > s:
        return cM, cA
    e = np.zeros(nt)
    e[-1] = 1.0
    cgp = w.scheme == CGP
    if eq == HEAT:
        if j == s:
            return w.a.copy(), tau * w.m
        if j == s - 1:
            if cgp:
                return np.outer(w.alpha, e), tau * np.outer(w.beta, e)
            return -np.outer(w.alpha, e), cA
        return cM, cA
    minv = np.linalg.inv(w.m)
    ama = w.a @ minv @ w.a
    am_alpha = w.a @ minv @ w.alpha
    minv_a_last = (minv @ w.a)[-1]
    minv_alpha_last = (minv @ w.alpha)[-1]
    if j == s:
        return ama / tau, tau * w.m
    if not cgp:
        if j == s - 1:
            return -(np.outer(am_alpha, e) + np.outer(w.alpha, minv_a_last)) / tau, cA
        if j == s - 2:
            return minv_alpha_last / tau * np.outer(w.alpha, e), cA
        return cM, cA
    minv_beta_last = (minv @ w.beta)[-1]
    alpha_a = w.alpha - w.a @ minv @ w.beta
    g = -minv_beta_last
    z = minv_alpha_last / tau
    if j == s - 1:
        cM = cM + np.outer(am_alpha, e) / tau
        cA = cA + tau * np.outer(w.beta, e)
    cM = cM + g ** (s - 1 - j) / tau * np.outer(alpha_a, minv_a_last)
    if j <= s - 2:
        cM = cM + g ** (s - 2 - j) * z * np.outer(alpha_a, e)
    return cM, cA


# ------------------------------------------------------------------- meshes
@dataclasses.dataclass
class MeshLevel:
    dim: int
    cells: int
    vertices: np.ndarray  # (n_verts, 3), x fastest


def make_hierarchy(dim, base_cells, refinements, finest_vertices=None) -> List[MeshLevel]:
    """Cartesian hierarchy of [0,1]^dim (src/mesh.cpp:148-187); injected
    finest vertices propagate to coarser levels at stride 2^(L-l)
    (src/mesh.cpp:221-236)."""
    levels = []
    for l in range(refinements + 1):
        n = base_cells << l
        ax = [np.arange(n + 1, dtype=float) / n for _ in range(dim)]
        grids = np.meshgrid(*ax[::-1], indexing="ij")[::-1]
        v = np.zeros((grids[0].size, 3))
        for a in range(dim):
            v[:, a] = grids[a].ravel()
        levels.append(MeshLevel(dim, n, v))
    if finest_vertices is not None:
        L = refinements
        fine = np.asarray(finest_vertices, dtype=float).reshape(-1, 3)
        levels[L].vertices = fine.copy()
        nf = levels[L].cells + 1
        for l in range(L):
            st = 1 << (L - l)
            nc = levels[l].cells + 1
            idx = np.arange(nc) * st
            if dim == 2:
                j, i = np.meshgrid(idx, idx, indexing="ij")
                src = j * nf + i
            else:
                kk, j, i = np.meshgrid(idx, idx, idx, indexing="ij")
                src = (kk * nf + j) * nf + i
            levels[l].vertices = fine[src.ravel()].copy()
    return levels


# -------------------------------------------------------- spatial operators
class Spatial:
    """SpatialDofMap + SpatialOperator pair on one level
    (src/spatial_operator.cpp:70-315): Gauss (p+1)-point quadrature, cached
    metric, sum-factorised cell kernels, Dirichlet identity rows."""

    def __init__(self, mesh: MeshLevel, p: int, rho_cell: Optional[np.ndarray] = None):
        self.dim, self.p, self.n = mesh.dim, p, p + 1
        d, n, nc = mesh.dim, p + 1, mesh.cells
        self.dofs = nc * p + 1
        self.n_space = self.dofs ** d
        self.n_cells = nc ** d
        gl = gauss_lobatto(n)[0]
        qx, qw = gauss(n)
        self.B = np.array([[lagrange(gl, j, x) for j in range(n)] for x in qx])  # q x n
        self.D = np.array([[lagrange_deriv(gl, j, x) for j in range(n)] for x in qx])
        # cell -> global lattice indices, local order x fastest
        c = np.arange(self.n_cells)
        cc = [c % nc, (c // nc) % nc, c // (nc * nc)]
        loc = np.arange(n ** d)
        ll = [loc % n, (loc // n) % n, loc // (n * n)]
        g = np.zeros((self.n_cells, n ** d), dtype=np.int64)
        stride = 1
        for a in range(d):
            g += (cc[a][:, None] * p + ll[a][None, :]) * stride
            stride *= self.dofs
        self.idx = g
        gi = np.arange(self.n_space)
        bd = np.zeros(self.n_space, dtype=bool)
        for a in range(d):
            ia = (gi // self.dofs ** a) % self.dofs
            bd |= (ia == 0) | (ia == self.dofs - 1)
        self.bdry = bd
        # geometry: Jacobians at the quadrature points (spatial_operator.cpp:11-45,152-183)
        nv = nc + 1
        corners = []
        for s in range(1 << d):
            i = cc[0] + (s & 1)
            j = cc[1] + ((s >> 1) & 1) if d > 1 else 0
            k = cc[2] + ((s >> 2) & 1) if d > 2 else 0
            corners.append(mesh.vertices[(k * nv + j) * nv + i])
        X = np.stack(corners, axis=1)[:, :, :d]  # cells x corners x d
        qp = np.stack(np.meshgrid(*([qx] * d)[::-1], indexing="ij")[::-1], axis=-1).reshape(-1, d)
        qwt = np.prod(np.stack(np.meshgrid(*([qw] * d)[::-1], indexing="ij")[::-1], axis=-1).reshape(-1, d), axis=1)
        dN = np.zeros((qp.shape[0], 1 << d, d))
        for s in range(1 << d):
            for b in range(d):
                val = np.ones(qp.shape[0])
                for a in range(d):
                    bit = (s >> a) & 1
                    if a == b:
                        val = val * (1.0 if bit else -1.0)
                    else:
                        val = val * (qp[:, a] if bit else 1.0 - qp[:, a])
                dN[:, s, b] = val
        J = np.einsum("qsb,csa->cqab", dN, X)
        det = np.linalg.det(J)
        Jinv = np.linalg.inv(J)
        rho = np.ones(self.n_cells) if rho_cell is None else rho_cell
        self.mass_fac = qwt[None, :] * det
        self.stiff_fac = (rho[:, None] * qwt[None, :] * det)[:, :, None, None] * np.einsum("cqab,cqeb->cqae", Jinv, Jinv)

    # tensor contraction helpers on (cells, [z,] y, x) arrays
    def _contract(self, u, M, axis):
        d = self.dim
        ax = d - axis  # array axis (0 is the cell axis)
        return np.moveaxis(np.tensordot(u, M, axes=([ax], [1])), -1, ax)

    def _to_q(self, u, mats):
        for a in range(self.dim):
            u = self._contract(u, mats[a], a)
        return u

    def apply(self, kind: str, u: np.ndarray) -> np.ndarray:
        """SpatialOperator::apply (spatial_operator.cpp:187-315)."""
        d, n = self.dim, self.n
        ui = np.where(self.bdry, 0.0, u)
        loc = ui[self.idx].reshape((self.n_cells,) + (n,) * d)
        if kind == "mass":
            v = self._to_q(loc, [self.B] * d)
            v = v * self.mass_fac.reshape(v.shape)
            out = self._to_q(v, [self.B.T] * d)
        else:
            grads = []
            for c in range(d):
                grads.append(self._to_q(loc, [self.D if a == c else self.B for a in range(d)]).reshape(self.n_cells, -1))
            G = np.stack(grads, axis=-1)
            G = np.einsum("cqab,cqb->cqa", self.stiff_fac, G)
            out = 0.0
            for c in range(d):
                gc = G[:, :, c].reshape((self.n_cells,) + (n,) * d)
                out = out + self._to_q(gc, [self.D.T if a == c else self.B.T for a in range(d)])
        y = np.bincount(self.idx.ravel(), weights=np.asarray(out).reshape(self.n_cells, -1).ravel(),
                        minlength=self.n_space)
        y[self.bdry] = u[self.bdry]
        return y

    def element_matrices(self, kind: str) -> np.ndarray:
        """Conventional per-cell quadrature assembly (spatial_operator.cpp:323-416)."""
        d = self.dim
        n = self.n
        loc = np.arange(n ** d)
        ll = [loc % n, (loc // n) % n, loc // (n * n)]
        qn = n ** d
        ql = [np.arange(qn) % n, (np.arange(qn) // n) % n, np.arange(qn) // (n * n)]
        phi = np.ones((qn, n ** d))
        for a in range(d):
            phi = phi * self.B[ql[a][:, None], ll[a][None, :]]
        if kind == "mass":
            return np.einsum("cq,qi,qj->cij", self.mass_fac, phi, phi)
        dphi = np.zeros((qn, n ** d, d))
        for c in range(d):
            t = np.ones((qn, n ** d))
            for a in range(d):
                t = t * (self.D if a == c else self.B)[ql[a][:, None], ll[a][None, :]]
            dphi[:, :, c] = t
        return np.einsum("qia,cqab,qjb->cij", dphi, self.stiff_fac, dphi)

    def assemble(self, kind: str) -> sp.csr_matrix:
        E = self.element_matrices(kind)
        rows = np.repeat(self.idx, self.idx.shape[1], axis=1).ravel()
        cols = np.tile(self.idx, (1, self.idx.shape[1])).ravel()
        vals = E.reshape(self.n_cells, -1).ravel()
        keep = ~(self.bdry[rows] | self.bdry[cols])
        A = sp.coo_matrix((vals[keep], (rows[keep], cols[keep])), shape=(self.n_space,) * 2).tocsr()
        return (A + sp.diags(self.bdry.astype(float))).tocsr()


# -------------------------------------------------------------- ST operator
class SpaceTime:
    """SpaceTimeOperator (src/space_time_operator.cpp:8-130, 319-393)."""

    def __init__(self, eq, w: Weights, tau, S, spatial: Spatial):
        self.eq, self.w, self.tau, self.S, self.sp = eq, w, tau, S, spatial
        self.nt = w.n_t
        self.nx = spatial.n_space
        self.n_dofs = S * self.nt * self.nx
        if eq == WAVE:
            minv = np.linalg.inv(w.m)
            self.ama = w.a @ minv @ w.a
            self.am_alpha = w.a @ minv @ w.alpha
            self.minv_a_last = (minv @ w.a)[-1]
            self.minv_alpha_last = (minv @ w.alpha)[-1]
            if w.scheme == CGP:
                self.minv_beta_last = (minv @ w.beta)[-1]
                self.alpha_a = w.alpha - w.a @ minv @ w.beta

    def blk(self, v, s, i):
        o = (s * self.nt + i) * self.nx
        return v[o:o + self.nx]

    def apply(self, u):
        """space_time_operator.cpp:45-130"""
        S, nt, tau, w = self.S, self.nt, self.tau, self.w
        cgp = w.scheme == CGP
        bd = self.sp.bdry
        ui = u.copy()
        ui.reshape(-1, self.nx)[:, bd] = 0.0
        M = [[self.sp.apply("mass", self.blk(ui, s, i)) for i in range(nt)] for s in range(S)]
        A = [[self.sp.apply("stiff", self.blk(ui, s, i)) for i in range(nt)] for s in range(S)]
        y = np.zeros(self.n_dofs)
        if self.eq == HEAT:
            for s in range(S):
                for i in range(nt):
                    seg = self.blk(y, s, i)
                    for j in range(nt):
                        seg += tau * w.m[i, j] * A[s][j] + w.a[i, j] * M[s][j]
                    if s > 0:
                        if cgp:
                            seg += w.alpha[i] * M[s - 1][-1] + tau * w.beta[i] * A[s - 1][-1]
                        else:
                            seg -= w.alpha[i] * M[s - 1][-1]
        else:
            z = self.minv_alpha_last / tau
            g = -self.minv_beta_last if cgp else 0.0
            mv_prev = np.zeros(self.nx)
            for s in range(S):
                for i in range(nt):
                    seg = self.blk(y, s, i)
                    for j in range(nt):
                        seg += tau * w.m[i, j] * A[s][j] + self.ama[i, j] / tau * M[s][j]
                    if s > 0:
                        if cgp:
                            seg += (self.am_alpha[i] / tau * M[s - 1][-1] + tau * w.beta[i] * A[s - 1][-1]
                                    + self.alpha_a[i] * mv_prev)
                        else:
                            seg -= self.am_alpha[i] / tau * M[s - 1][-1] + w.alpha[i] * mv_prev
                mv = np.zeros(self.nx)
                for j in range(nt):
                    mv += self.minv_a_last[j] / tau * M[s][j]
                if s > 0:
                    if cgp:
                        mv += z * M[s - 1][-1] + g * mv_prev
                    else:
                        mv -= z * M[s - 1][-1]
                mv_prev = mv
        yv = y.reshape(-1, self.nx)
        yv[:, bd] = u.reshape(-1, self.nx)[:, bd]
        return y

    def assemble(self) -> sp.csr_matrix:
        """assemble_sparse (space_time_operator.cpp:354-393)."""
        Ms, As = self.sp.assemble("mass"), self.sp.assemble("stiff")
        bd = self.sp.bdry.astype(float)
        inner = sp.diags(1.0 - bd)
        Ms, As = inner @ Ms @ inner, inner @ As @ inner
        F = self.S * self.nt
        CM, CA = np.zeros((F, F)), np.zeros((F, F))
        for s in range(self.S):
            for j in range(s + 1):
                cm, ca = block_coefficients(self.eq, self.w, self.tau, s, j)
                CM[s * self.nt:(s + 1) * self.nt, j * self.nt:(j + 1) * self.nt] = cm
                CA[s * self.nt:(s + 1) * self.nt, j * self.nt:(j + 1) * self.nt] = ca
        Sys = sp.kron(sp.csr_matrix(CM), Ms) + sp.kron(sp.csr_matrix(CA), As)
        Sys = Sys + sp.diags(np.tile(bd, F))
        return Sys.tocsr()


# ------------------------------------------------------------------ transfer
def _axis_P(cf, pf, cc, pc):
    """1D embedding (src/transfer.cpp:32-54)."""
    fn, cn = gauss_lobatto(pf + 1)[0], gauss_lobatto(pc + 1)[0]
    P = np.zeros((cf * pf + 1, cc * pc + 1))
    h = cc != cf
    for c in range(cf):
        for m in range(pf + 1):
            ccell, tc = (c // 2, 0.5 * (c % 2) + 0.5 * fn[m]) if h else (c, fn[m])
            for j in range(pc + 1):
                P[c * pf + m, ccell * pc + j] = lagrange(cn, j, tc)
    return P


class Transfer:
    """Transfer (src/transfer.cpp:58-190)."""

    def __init__(self, fine: SpaceTime, coarse: SpaceTime, fine_cells, coarse_cells):
        self.f, self.c = fine, coarse
        self.spatial = fine.sp.p != coarse.sp.p or fine_cells != coarse_cells
        if self.spatial:
            self.P = _axis_P(fine_cells, fine.sp.p, coarse_cells, coarse.sp.p)
        else:
            wf, wc = fine.w, coarse.w
            Sf, Sc = fine.S, coarse.S
            T = np.zeros((Sf * wf.n_t, Sc * wc.n_t))
            for sf in range(Sf):
                for i in range(wf.n_t):
                    tf = wf.unknown_nodes[i]
                    sc, tc = (sf // 2, 0.5 * (sf % 2) + 0.5 * tf) if Sf != Sc else (sf, tf)
                    for j in range(wc.n_t):
                        T[sf * wf.n_t + i, sc * wc.n_t + j] += wc.unknown_weight(j, tc)
                    lw = wc.left_weight(tc)
                    if lw != 0.0 and sc > 0:
                        T[sf * wf.n_t + i, sc * wc.n_t - 1] += lw
            self.T = T

    def _map(self, v, src: SpaceTime, dst: SpaceTime, M):
        d = src.sp.dim
        blocks = v.reshape(-1, src.nx)
        out = []
        for b in blocks:
            x = b.reshape((src.sp.dofs,) * d)
            for a in range(d):
                ax = d - 1 - a
                x = np.moveaxis(np.tensordot(x, M, axes=([ax], [1])), -1, ax)
            out.append(x.ravel())
        return np.concatenate(out)

    def prolong(self, c):
        c = c.copy()
        c.reshape(-1, self.c.nx)[:, self.c.sp.bdry] = 0.0
        if self.spatial:
            f = self._map(c, self.c, self.f, self.P)
        else:
            f = (self.T @ c.reshape(-1, self.c.nx)).ravel()
        f.reshape(-1, self.f.nx)[:, self.f.sp.bdry] = 0.0
        return f

    def restrict(self, f):
        f = f.copy()
        f.reshape(-1, self.f.nx)[:, self.f.sp.bdry] = 0.0
        if self.spatial:
            c = self._map(f, self.f, self.c, self.P.T)
        else:
            c = (self.T.T @ f.reshape(-1, self.f.nx)).ravel()
        c.reshape(-1, self.c.nx)[:, self.c.sp.bdry] = 0.0
        return c


# ---------------------------------------------------------------------- ASM
class ASM:
    """ASMSmoother (src/asm_smoother.cpp:7-78): LU of every (step, cell)
    block of the assembled slab matrix, inverse-multiplicity weights."""

    def __init__(self, op: SpaceTime):
        Sys = op.assemble().tocsr()
        nt, sp_ = op.nt, op.sp
        blocks, dofs = [], []
        for s in range(op.S):
            for c in range(sp_.n_cells):
                gd = np.concatenate([(s * nt + i) * op.nx + sp_.idx[c] for i in range(nt)])
                blocks.append(Sys[gd][:, gd].toarray())
                dofs.append(gd)
        self.dofs = np.array(dofs)
        self.lu = [sla.lu_factor(B) for B in blocks]
        mult = np.bincount(self.dofs.ravel(), minlength=op.n_dofs).astype(float)
        self.mult = np.maximum(mult, 1.0)
        self.n = op.n_dofs

    def add_correction(self, r, z):
        z = z.copy()
        for gd, lu in zip(self.dofs, self.lu):
            z[gd] += sla.lu_solve(lu, r[gd]) / self.mult[gd]
        return z


# ----------------------------------------------------------------- rng
class Xoshiro:
    """xoshiro256++ / splitmix64 / Box-Muller (include/stmg/rng.hpp:11-82)."""

    M = (1 << 64) - 1

    def __init__(self, seed):
        x, s = seed & self.M, []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & self.M
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
            s.append(z ^ (z >> 31))
        self.s, self.cached = s, None

    def next(self):
        s, m = self.s, self.M
        rotl = lambda v, k: ((v << k) | (v >> (64 - k))) & m  # noqa: E731
        r = (rotl((s[0] + s[3]) & m, 23) + s[0]) & m
        t = (s[1] << 17) & m
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = rotl(s[3], 45)
        return r

    def uniform(self):
        return (self.next() >> 11) * 2.0 ** -53

    def normal(self):
        if self.cached is not None:
            v, self.cached = self.cached, None
            return v
        u1 = 0.0
        while u1 <= 1e-300:
            u1 = self.uniform()
        u2 = self.uniform()
        r = np.sqrt(-2.0 * np.log(u1))
        th = 2.0 * np.pi * u2
        self.cached = r * np.sin(th)
        return r * np.cos(th)


# ------------------------------------------------------------- multigrid
def default_strategy(mesh_level, n_steps, k, scheme):
    """src/multigrid.cpp:70-81"""
    kmin = 0 if scheme == DG else 1
    s = [SPACE_H] * mesh_level
    n = n_steps
    while n > 1:
        s.append(TIME_TAU)
        n //= 2
    s += [TIME_K] * (k - kmin)
    return s


class Multigrid:
    """SpaceTimeMultigrid (src/multigrid.cpp:83-234): per-level operators, ASM
    with Ritz-estimated omega, SparseLU coarse solve, V(nu,nu) cycle."""

    def __init__(self, eq, scheme, levels: List[MeshLevel], rho0: Optional[np.ndarray], fine_level, p, k, S, tau,
                 strategy: Optional[Sequence[int]] = None, n_smooth=1, eig_iters=20, seed=42):
        if strategy is None:
            strategy = default_strategy(fine_level, S, k, scheme)
        plan = [(fine_level, p, k, S, tau)]
        for c in strategy:
            ml, pp, kk, ss, tt = plan[-1]
            if c == SPACE_H:
                ml -= 1
            elif c == SPACE_P:
                pp = max(1, pp // 2)
            elif c == TIME_TAU:
                ss //= 2
                tt *= 2
            else:
                kk -= 1
            plan.append((ml, pp, kk, ss, tt))
        self.plan, self.n_smooth = plan, n_smooth
        self.ops, self.cells = [], []
        for (ml, pp, kk, ss, tt) in plan:
            rho = None
            if rho0 is not None:
                nc = levels[ml].cells
                base = levels[0].cells
                c = np.arange(nc ** levels[ml].dim)
                cc = [c % nc, (c // nc) % nc, c // (nc * nc)]
                sh = ml
                a = [x >> sh for x in cc]
                rho = rho0[(a[2] * base + a[1]) * base + a[0]] if levels[ml].dim == 3 else rho0[a[1] * base + a[0]]
            w = dg_weights(kk) if scheme == DG else cgp_weights(kk)
            self.ops.append(SpaceTime(eq, w, tt, ss, Spatial(levels[ml], pp, rho)))
            self.cells.append(levels[ml].cells)
        L = len(plan)
        self.smoothers, self.omega = [], []
        for l in range(L):
            if l + 1 < L or L == 1:
                sm = ASM(self.ops[l])
                self.smoothers.append(sm)
                self.omega.append(self._relaxation(l, sm, eig_iters, seed + l))
            else:
                self.smoothers.append(None)
                self.omega.append(1.0)
        self.coarse = spla.splu(self.ops[-1].assemble().tocsc())
        self.transfers = [Transfer(self.ops[l], self.ops[l + 1], self.cells[l], self.cells[l + 1])
                          for l in range(L - 1)]

    def _relaxation(self, l, sm, m, seed):
        """src/multigrid.cpp:127-172"""
        op = self.ops[l]
        n = op.n_dofs
        m = min(m, n)
        rng = Xoshiro(seed)
        v = np.array([rng.normal() for _ in range(n)])
        v /= np.linalg.norm(v)
        V, H = [v], np.zeros((m + 1, m))
        kdim = 0
        for j in range(m):
            z = sm.add_correction(op.apply(V[j]), np.zeros(n))
            for i in range(j + 1):
                H[i, j] = z @ V[i]
                z = z - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(z)
            kdim = j + 1
            if H[j + 1, j] < 1e-13:
                break
            V.append(z / H[j + 1, j])
        re = np.linalg.eigvals(H[:kdim, :kdim]).real
        om = 2.0 / (re.max() + max(0.0, re.min()))
        return 1.0 if not np.isfinite(om) or om <= 0 else min(om, 1.0)

    def smooth(self, l, f, u):
        r = f - self.ops[l].apply(u)
        return u + self.omega[l] * self.smoothers[l].add_correction(r, np.zeros_like(r))

    def v_cycle(self, l, f, u):
        if l + 1 == len(self.ops):
            return self.coarse.solve(f)
        for _ in range(self.n_smooth):
            u = self.smooth(l, f, u)
        rc = self.transfers[l].restrict(f - self.ops[l].apply(u))
        ec = self.v_cycle(l + 1, rc, np.zeros(self.ops[l + 1].n_dofs))
        u = u + self.transfers[l].prolong(ec)
        for _ in range(self.n_smooth):
            u = self.smooth(l, f, u)
        return u

    def apply(self, r):
        return self.v_cycle(0, r, np.zeros(self.ops[0].n_dofs))


# -------------------------------------------------------------------- GMRES
def gmres(op, b, x, restart=100, max_iters=1000, rel_tol=1e-12, abs_tol=1e-12, precond=None):
    """Restarted right-preconditioned GMRES, two-pass MGS, Givens
    (src/gmres.cpp:8-115). Returns (x, info)."""
    x = np.array(x, dtype=float)
    m = max(1, restart)
    r = b - op(x)
    beta = np.linalg.norm(r)
    info = {"initial_residual": beta, "residual_history": [beta], "iterations": 0, "converged": False}
    tol = max(abs_tol, rel_tol * max(beta, 1e-300))
    if beta <= tol:
        info.update(converged=True, final_residual=beta)
        return x, info
    while info["iterations"] < max_iters:
        V = [r / beta]
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        k = 0
        while k < m and info["iterations"] < max_iters:
            info["iterations"] += 1
            w = op(precond(V[k]) if precond else V[k])
            for pas in range(2):
                for i in range(k + 1):
                    h = w @ V[i]
                    H[i, k] = h if pas == 0 else H[i, k] + h
                    w = w - h * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            breakdown = not H[k + 1, k] > 0
            if not breakdown:
                V.append(w / H[k + 1, k])
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            den = np.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = (1.0, 0.0) if den == 0 else (H[k, k] / den, H[k + 1, k] / den)
            H[k, k], H[k + 1, k] = den, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            res = abs(g[k + 1])
            info["residual_history"].append(res)
            k += 1
            if res <= tol or breakdown:
                break
        y = sla.solve_triangular(H[:k, :k], g[:k])
        dx = sum(y[i] * V[i] for i in range(k))
        x = x + (precond(dx) if precond else dx)
        r = b - op(x)
        beta = np.linalg.norm(r)
        info["final_residual"] = beta
        if beta <= tol:
            info["converged"] = True
            return x, info
        if beta == 0.0:
            break
    info["final_residual"] = beta
    info["converged"] = beta <= tol
    return x, info


def build(cfg, with_mg=False, vertices=None, **mg):
    """Discretise one Config of paper_2408_04372_b200.problems like
    oracle/ref_harness.cpp:ref_create does with the reference."""
    v = vertices if vertices is not None else cfg.vertices()
    levels = make_hierarchy(cfg.dim, cfg.base_cells, cfg.refinements, v)
    w = dg_weights(cfg.k) if cfg.scheme == DG else cgp_weights(cfg.k)
    rho = None
    if cfg.rho is not None:
        nc = levels[-1].cells
        c = np.arange(nc ** cfg.dim)
        sh = cfg.refinements
        a = [(c % nc) >> sh, ((c // nc) % nc) >> sh, (c // (nc * nc)) >> sh]
        b = cfg.base_cells
        rho = cfg.rho[(a[2] * b + a[1]) * b + a[0]] if cfg.dim == 3 else cfg.rho[a[1] * b + a[0]]
    op = SpaceTime(cfg.equation, w, cfg.tau, cfg.n_steps, Spatial(levels[-1], cfg.p, rho))
    M = None
    if with_mg:
        M = Multigrid(cfg.equation, cfg.scheme, levels, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps, cfg.tau,
                      **mg)
    return op, M
