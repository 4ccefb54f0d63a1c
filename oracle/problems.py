"""Analytic problem data evaluated by the oracle (test infrastructure only).

Manufactured solution of BASELINE.json configs[0,1,2,4]: psi = sin(pi x)sin(pi y)sin(pi z)(1,1,1),
u = curl psi, p = sin(2 pi x) cos(pi y) z.  With a(u,v) = int nu eps(u):eps(v) and
b(v,q) = int div v q, Eq.(VarForm) gives f = -div(nu eps(u)) - grad p, and since
div u = 0, Delta u = -3 pi^2 u: f = (3 pi^2 nu / 2) u - grad p   (SURVEY A1/F5 reading).
Multi-sinker of configs[3]: f = (0, 0, beta (chi - 1)), u = 0 on the boundary.
"""
import numpy as np

PI = np.pi


def u_exact(x):
    x = np.atleast_2d(x)
    sx, sy, sz = np.sin(PI * x[:, 0]), np.sin(PI * x[:, 1]), np.sin(PI * x[:, 2])
    cx, cy, cz = np.cos(PI * x[:, 0]), np.cos(PI * x[:, 1]), np.cos(PI * x[:, 2])
    px, py, pz = PI * cx * sy * sz, PI * sx * cy * sz, PI * sx * sy * cz
    return np.stack([py - pz, pz - px, px - py], 1)


def grad_u_exact(x):
    """[n,3,3] with G[:, c, d] = d u_c / d x_d."""
    x = np.atleast_2d(x)
    s = [np.sin(PI * x[:, i]) for i in range(3)]
    c = [np.cos(PI * x[:, i]) for i in range(3)]
    # Hessian of phi = s0 s1 s2
    H = np.empty((x.shape[0], 3, 3))
    for i in range(3):
        for j in range(3):
            f = [s[0], s[1], s[2]]
            if i == j:
                f[i] = -s[i]
                H[:, i, j] = PI ** 2 * f[0] * f[1] * f[2]
            else:
                f[i] = c[i]; f[j] = c[j]
                H[:, i, j] = PI ** 2 * f[0] * f[1] * f[2]
    G = np.empty((x.shape[0], 3, 3))
    G[:, 0, :] = H[:, 1, :] - H[:, 2, :]
    G[:, 1, :] = H[:, 2, :] - H[:, 0, :]
    G[:, 2, :] = H[:, 0, :] - H[:, 1, :]
    return G


def p_exact(x):
    x = np.atleast_2d(x)
    return np.sin(2 * PI * x[:, 0]) * np.cos(PI * x[:, 1]) * x[:, 2]


def grad_p_exact(x):
    x = np.atleast_2d(x)
    return np.stack([2 * PI * np.cos(2 * PI * x[:, 0]) * np.cos(PI * x[:, 1]) * x[:, 2],
                     -PI * np.sin(2 * PI * x[:, 0]) * np.sin(PI * x[:, 1]) * x[:, 2],
                     np.sin(2 * PI * x[:, 0]) * np.cos(PI * x[:, 1])], 1)


def f_manufactured(nu):
    return lambda x: 1.5 * PI ** 2 * nu * u_exact(x) - grad_p_exact(x)


def f_sinker(params):
    centres, beta = params["centres"], params["beta"]
    delta, omega = params["delta"], params["omega"]

    def f(x):
        x = np.atleast_2d(x)
        chi = np.ones(x.shape[0])
        for c in centres:
            d = np.linalg.norm(x - c, axis=1)
            chi *= 1.0 - np.exp(-delta * np.maximum(0.0, d - omega / 2) ** 2)
        out = np.zeros((x.shape[0], 3))
        out[:, 2] = beta * (chi - 1.0)
        return out
    return f
