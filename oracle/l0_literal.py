"""Literal assembled-B̃ form of the ES-T-FEM operators -- TEST INFRASTRUCTURE ONLY.

Written straight from PAPER.md §2.2 with no factoring, for small meshes:

* eq:strain_discretization / eq:CSTet_strain_discretization: at each
  edge quadrature point G_i the smoothed strain is eps = A_j( A_k [B_k^{V_j}] w_{V_j} ) {u},
  w_{V_j} = V_j / sum_n V_n over the (active) elements sharing the edge; B_k^{V_j} is the
  6x3 strain-displacement block of node k in element V_j (rows eps11, eps22, eps33,
  gamma12, gamma23, gamma13).
* eq:fint_discretization / eq:CSTet_fint_discretization:
  f_int = A_j( A_k [B_k^{V_j}]^T w_{V_j} sigma ) * (1/6) sum_j V_j.
* sigma = D eps with the isotropic D (standard Lame form R1).

Shape-function gradients here come from inverting the 4x4 barycentric matrix
[[1, x, y, z]_a] with numpy.linalg.inv and volumes from numpy.linalg.det, i.e.
independently of the closed-form cross products used in cem_oracle.c.
"""
from __future__ import annotations

from collections import defaultdict

import numpy as np

LOCAL_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
# trilinear hexahedron (eq:hex_strain_discretization / eq:hex_fint_discretization):
# 12 edges, smoothing-domain volume (1/12) sum_j V_j; element strain = the volume-averaged strain (R23)
HEX_EDGES = [(0, 1), (1, 2), (2, 3), (0, 3), (4, 5), (5, 6), (6, 7), (4, 7), (0, 4), (1, 5), (2, 6), (3, 7)]
HEX_XI = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                   [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64)


def _hex_dN(p):
    """[8,3] derivatives of the trilinear shape functions w.r.t. (xi, eta, zeta) at p."""
    f = 1.0 + HEX_XI * np.asarray(p)[None, :]             # (1 + xi_i xi), ...
    d = np.empty((8, 3))
    d[:, 0] = HEX_XI[:, 0] * f[:, 1] * f[:, 2] / 8.0
    d[:, 1] = f[:, 0] * HEX_XI[:, 1] * f[:, 2] / 8.0
    d[:, 2] = f[:, 0] * f[:, 1] * HEX_XI[:, 2] / 8.0
    return d


def hex_B(Xe):
    """Volume and the 6x24 mean-gradient B matrix (1/V) integral grad N dV of one hex by 3x3x3
    Gauss-Legendre with numpy.linalg.det / inv (independent of the C oracle's 2x2x2 rule and
    cofactor form; both are exact for the trilinear map)."""
    pts, wts = np.polynomial.legendre.leggauss(3)
    V = 0.0
    G = np.zeros((8, 3))
    for i, a in enumerate(pts):
        for j, b in enumerate(pts):
            for k, c in enumerate(pts):
                dN = _hex_dN((a, b, c))
                J = Xe.T @ dN
                w = wts[i] * wts[j] * wts[k] * np.linalg.det(J)
                V += w
                G += w * (dN @ np.linalg.inv(J))
    g = G / V                                              # [8,3] mean dN/dx
    B = np.zeros((6, 24))
    for a in range(8):
        gx, gy, gz = g[a]
        c = 3 * a
        B[0, c] = gx
        B[1, c + 1] = gy
        B[2, c + 2] = gz
        B[3, c] = gy; B[3, c + 1] = gx
        B[4, c + 1] = gz; B[4, c + 2] = gy
        B[5, c] = gz; B[5, c + 2] = gx
    return V, B


def tet_B(Xe):
    """Volume and the 6x12 B matrix of one tet (columns node-major, dof x,y,z)."""
    M = np.hstack([np.ones((4, 1)), Xe])
    V = abs(np.linalg.det(M)) / 6.0
    Minv = np.linalg.inv(M)          # N_a(x) = Minv[0,a] + Minv[1:,a].x
    g = Minv[1:, :].T                # [4,3] gradients
    B = np.zeros((6, 12))
    for a in range(4):
        gx, gy, gz = g[a]
        c = 3 * a
        B[0, c] = gx
        B[1, c + 1] = gy
        B[2, c + 2] = gz
        B[3, c] = gy; B[3, c + 1] = gx
        B[4, c + 1] = gz; B[4, c + 2] = gy
        B[5, c] = gz; B[5, c + 2] = gx
    return V, B


def D_matrix(E, nu):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[0, 0] = D[1, 1] = D[2, 2] = lam + 2 * mu
    D[3, 3] = D[4, 4] = D[5, 5] = mu
    return D


def edge_incidence(tets):
    inc = defaultdict(list)
    edges = HEX_EDGES if tets.shape[1] == 8 else LOCAL_EDGES
    for e, t in enumerate(tets):
        for p, q in edges:
            i, j = int(t[p]), int(t[q])
            inc[(min(i, j), max(i, j))].append(e)
    return dict(sorted(inc.items()))


def smoothed_operators(X, tets, active):
    """Per edge: (edge, support nodes, B̃ [6 x 3|supp|], V_s) over active incident tets."""
    inc = edge_incidence(tets)
    hexa = tets.shape[1] == 8
    npe, nedge = (8, 12) if hexa else (4, 6)
    geo = [(hex_B if hexa else tet_B)(X[t]) for t in tets]
    ops = []
    for edge, elems in inc.items():
        act = [e for e in elems if active[e]]
        if not act:
            ops.append((edge, np.zeros(0, np.int64), np.zeros((6, 0)), 0.0))
            continue
        Vsum = sum(geo[e][0] for e in act)
        supp = sorted({int(n) for e in act for n in tets[e]})
        col = {n: i for i, n in enumerate(supp)}
        Bt = np.zeros((6, 3 * len(supp)))
        for e in act:
            Ve, Be = geo[e]
            w = Ve / Vsum
            for a in range(npe):
                c = col[int(tets[e][a])]
                Bt[:, 3 * c:3 * c + 3] += w * Be[:, 3 * a:3 * a + 3]
        ops.append((edge, np.array(supp), Bt, Vsum / nedge))
    return ops


def edge_strain_stress(X, tets, active, u, E, nu):
    D = D_matrix(E, nu)
    out = {}
    for edge, supp, Bt, Vs in smoothed_operators(X, tets, active):
        if supp.size == 0:
            out[edge] = (np.zeros(6), np.zeros(6), 0.0)
            continue
        eps = Bt @ u[supp].ravel()
        out[edge] = (eps, D @ eps, Vs)
    return out


def internal_force(X, tets, active, u, E, nu):
    D = D_matrix(E, nu)
    f = np.zeros_like(u)
    for edge, supp, Bt, Vs in smoothed_operators(X, tets, active):
        if supp.size == 0:
            continue
        sig = D @ (Bt @ u[supp].ravel())
        f[supp] += (Bt.T @ sig * Vs).reshape(-1, 3)
    return f


def strain_energy(X, tets, active, u, E, nu):
    D = D_matrix(E, nu)
    U = 0.0
    for edge, supp, Bt, Vs in smoothed_operators(X, tets, active):
        if supp.size == 0:
            continue
        eps = Bt @ u[supp].ravel()
        U += 0.5 * eps @ D @ eps * Vs
    return U


def stiffness(X, tets, active, E, nu):
    """Dense global ES-FEM stiffness K (f_int = K u), 3N x 3N."""
    N = X.shape[0]
    D = D_matrix(E, nu)
    K = np.zeros((3 * N, 3 * N))
    for edge, supp, Bt, Vs in smoothed_operators(X, tets, active):
        if supp.size == 0:
            continue
        dofs = (3 * supp[:, None] + np.arange(3)[None, :]).ravel()
        K[np.ix_(dofs, dofs)] += Bt.T @ D @ Bt * Vs
    return K
