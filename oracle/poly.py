"""Scaled monomials and quadrature (oracle; test infrastructure only).

Scaled monomials m_a(x) = ((x - x_O)/h_O)^a on an entity O with centroid x_O and
diameter h_O, ordered by total degree then x-power descending (P:34-35 notation
for P_n and P^_{n\\m}; ordering = SURVEY O-2 / S:117).  Quadrature: Gauss-Legendre
and Gauss-Lobatto on [0,1], collapsed (Duffy) rules on triangles and tetrahedra
(SURVEY O-2 allows any rule of exactness >= 2k+2).
"""
import numpy as np
from numpy.polynomial import legendre as npleg


def dim2(n):
    return 0 if n < 0 else (n + 1) * (n + 2) // 2


def dim3(n):
    return 0 if n < 0 else (n + 1) * (n + 2) * (n + 3) // 6


def exps2(n):
    return [(p, d - p) for d in range(n + 1) for p in range(d, -1, -1)]


def exps3(n):
    out = []
    for d in range(n + 1):
        for a in range(d, -1, -1):
            for b in range(d - a, -1, -1):
                out.append((a, b, d - a - b))
    return out


def mono3(x, xc, h, n):
    """Values [npts, dim3(n)] and gradients [npts, dim3(n), 3] of 3D scaled monomials."""
    X = (np.atleast_2d(x) - xc) / h
    E = exps3(n)
    P = [np.ones((X.shape[0], n + 1)) for _ in range(3)]
    for c in range(3):
        for p in range(1, n + 1):
            P[c][:, p] = P[c][:, p - 1] * X[:, c]
    val = np.empty((X.shape[0], len(E)))
    grd = np.zeros((X.shape[0], len(E), 3))
    for j, (a, b, c) in enumerate(E):
        val[:, j] = P[0][:, a] * P[1][:, b] * P[2][:, c]
        if a > 0:
            grd[:, j, 0] = a * P[0][:, a - 1] * P[1][:, b] * P[2][:, c] / h
        if b > 0:
            grd[:, j, 1] = b * P[0][:, a] * P[1][:, b - 1] * P[2][:, c] / h
        if c > 0:
            grd[:, j, 2] = c * P[0][:, a] * P[1][:, b] * P[2][:, c - 1] / h
    return val, grd


def mono2(xi, n, h):
    """Values [npts, dim2(n)] and in-plane gradients [npts, dim2(n), 2]; xi = (x-x_f).(t1,t2)."""
    X = np.atleast_2d(xi) / h
    E = exps2(n)
    P = [np.ones((X.shape[0], n + 1)) for _ in range(2)]
    for c in range(2):
        for p in range(1, n + 1):
            P[c][:, p] = P[c][:, p - 1] * X[:, c]
    val = np.empty((X.shape[0], len(E)))
    grd = np.zeros((X.shape[0], len(E), 2))
    for j, (p, q) in enumerate(E):
        val[:, j] = P[0][:, p] * P[1][:, q]
        if p > 0:
            grd[:, j, 0] = p * P[0][:, p - 1] * P[1][:, q] / h
        if q > 0:
            grd[:, j, 1] = q * P[0][:, p] * P[1][:, q - 1] / h
    return val, grd


def gauss_legendre01(n):
    t, w = npleg.leggauss(n)
    return (t + 1.0) / 2.0, w / 2.0


def gauss_lobatto01(npts):
    """Gauss-Lobatto nodes/weights on [0,1] with npts points (exact to degree 2 npts - 3)."""
    m = npts - 1
    cP = np.zeros(m + 1); cP[m] = 1.0
    inner = np.sort(npleg.legroots(npleg.legder(cP))) if m >= 2 else np.array([])
    x = np.concatenate([[-1.0], inner, [1.0]])
    w = 2.0 / (m * (m + 1) * npleg.legval(x, cP) ** 2)
    return (x + 1.0) / 2.0, w / 2.0


def triangle_rule(a, b, c, n):
    """Collapsed Gauss rule on triangle abc (3D points); exact for degree <= 2n-2."""
    u, wu = gauss_legendre01(n)
    U, V = np.meshgrid(u, u, indexing="ij")
    W = np.outer(wu, wu) * (1.0 - U)
    s, t = U.ravel(), (V * (1.0 - U)).ravel()
    area2 = np.linalg.norm(np.cross(b - a, c - a))
    pts = a + np.outer(s, b - a) + np.outer(t, c - a)
    return pts, W.ravel() * area2


def tet_rule(a, b, c, d, n):
    """Collapsed Gauss rule on tetrahedron abcd; exact for degree <= 2n-3. Weights carry |vol|."""
    u, wu = gauss_legendre01(n)
    U, V, Wv = np.meshgrid(u, u, u, indexing="ij")
    w = (wu[:, None, None] * wu[None, :, None] * wu[None, None, :]) * (1 - U) ** 2 * (1 - V)
    s = U.ravel(); t = (V * (1 - U)).ravel(); r = (Wv * (1 - U) * (1 - V)).ravel()
    vol6 = abs(np.dot(b - a, np.cross(c - a, d - a)))
    pts = a + np.outer(s, b - a) + np.outer(t, c - a) + np.outer(r, d - a)
    return pts, w.ravel() * vol6
