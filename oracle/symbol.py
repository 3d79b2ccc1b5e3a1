"""Spectral symbols of the IgA matrices (used only to pin the oracle's assembly).

Oracle (test infrastructure only).
  m_p, a_p, s_p     Theorem 3.1
  Laplacian symbol  eq:lapl2D PAPER.md:677-679, eq:lapl3D PAPER.md:779-783
  f^{p,alpha,beta}  Theorem 5.1 (2D), Theorem 5.3 (3D)
  sampling grid     Sec. 5.3: theta_k = k pi / m, k = 1..m
"""
import numpy as np

from .bspline import cardinal, cardinal_deriv


def sym_m(p, th):
    th = np.asarray(th, dtype=float)
    out = cardinal(2 * p + 1, p + 1) * np.ones_like(th)
    for k in range(1, p + 1):
        out = out + 2 * cardinal(2 * p + 1, p + 1 - k) * np.cos(k * th)
    return out


def sym_a(p, th):
    th = np.asarray(th, dtype=float)
    out = np.zeros_like(th)
    for k in range(1, p + 1):
        out = out - 2 * cardinal_deriv(2 * p + 1, p + 1 - k, 1) * np.sin(k * th)
    return out


def sym_s(p, th):
    th = np.asarray(th, dtype=float)
    out = -cardinal_deriv(2 * p + 1, p + 1, 2) * np.ones_like(th)
    for k in range(1, p + 1):
        out = out - 2 * cardinal_deriv(2 * p + 1, p + 1 - k, 2) * np.cos(k * th)
    return out


def laplacian(p, thetas, nu=None):
    d = len(thetas)
    nu = np.ones(d) if nu is None else np.asarray(nu, float)
    if d == 2:
        t1, t2 = thetas
        return nu[1] / nu[0] * sym_m(p, t1) * sym_s(p, t2) + nu[0] / nu[1] * sym_s(p, t1) * sym_m(p, t2)
    g = nu ** 2 / np.prod(nu)
    t1, t2, t3 = thetas
    m1, m2, m3 = sym_m(p, t1), sym_m(p, t2), sym_m(p, t3)
    s1, s2, s3 = sym_s(p, t1), sym_s(p, t2), sym_s(p, t3)
    return g[0] * s1 * m2 * m3 + g[1] * m1 * s2 * m3 + g[2] * m1 * m2 * s3


def symbol_f(p, alpha, beta, thetas, nu=None):
    """Matrix-valued symbol f^{p,alpha,beta}(theta), shape (..., d, d)."""
    d = len(thetas)
    nu = np.ones(d) if nu is None else np.asarray(nu, float)
    th = [np.asarray(t, float) for t in thetas]
    m = [sym_m(p, t) for t in th]
    a = [sym_a(p, t) for t in th]
    s = [sym_s(p, t) for t in th]
    shape = np.broadcast(*th).shape
    f = np.zeros(shape + (d, d))
    if d == 2:
        r = nu[1] / nu[0]
        f[..., 0, 0] = alpha * r * m[0] * s[1] + beta / r * s[0] * m[1]
        f[..., 0, 1] = f[..., 1, 0] = -(alpha - beta) * a[0] * a[1]
        f[..., 1, 1] = alpha / r * s[0] * m[1] + beta * r * m[0] * s[1]
        return f
    g = nu ** 2 / np.prod(nu)
    dl = 1.0 / nu
    f[..., 0, 0] = beta * g[0] * s[0] * m[1] * m[2] + alpha * g[1] * m[0] * s[1] * m[2] + alpha * g[2] * m[0] * m[1] * s[2]
    f[..., 1, 1] = alpha * g[0] * s[0] * m[1] * m[2] + beta * g[1] * m[0] * s[1] * m[2] + alpha * g[2] * m[0] * m[1] * s[2]
    f[..., 2, 2] = alpha * g[0] * s[0] * m[1] * m[2] + alpha * g[1] * m[0] * s[1] * m[2] + beta * g[2] * m[0] * m[1] * s[2]
    f[..., 0, 1] = f[..., 1, 0] = -(alpha - beta) * dl[2] * a[0] * a[1] * m[2]
    f[..., 0, 2] = f[..., 2, 0] = -(alpha - beta) * dl[1] * a[0] * m[1] * a[2]
    f[..., 1, 2] = f[..., 2, 1] = -(alpha - beta) * dl[0] * m[0] * a[1] * a[2]
    return f


def grid(m, d):
    """Gamma = {k pi / m : k = 1..m}^d, as d meshgrid arrays."""
    t = np.arange(1, m + 1) * np.pi / m
    return np.meshgrid(*([t] * d), indexing="ij")
