"""Pins of oracle/symbol.py against the paper's closed forms and lemmas (no GPU)."""
import numpy as np
import pytest

from oracle import matrices1d as m1
from oracle import symbol as sy

TH = np.linspace(-np.pi, np.pi, 1001)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_lemma_3_2(p):
    m, a, s = sy.sym_m(p, TH), sy.sym_a(p, TH), sy.sym_s(p, TH)
    assert abs(sy.sym_m(p, 0.0) - 1.0) < 1e-14                             # m_p(0) = 1
    # (a) as printed, (2/pi)^{2p} <= m_p, is violated at theta=pi by the paper's own closed form
    # m_1(pi) = 1/3 < (2/pi)^2; the bound that holds is (2/pi)^{2p+2} (reading E1)
    assert sy.sym_m(p, np.pi) < (2 / np.pi) ** (2 * p)
    assert np.all(m >= (2 / np.pi) ** (2 * p + 2) - 1e-13) and np.all(m <= 1 + 1e-13)
    if p >= 2:                                                            # (b) s_p = m_{p-1}(2-2cos)
        assert np.max(np.abs(s - sy.sym_m(p - 1, TH) * (2 - 2 * np.cos(TH)))) < 1e-12
    assert np.all(m * s - a ** 2 >= -1e-13)                                # (c)


def test_closed_forms_p1_p2():
    assert np.max(np.abs(sy.sym_m(1, TH) - (2 + np.cos(TH)) / 3)) < 1e-15
    assert np.max(np.abs(sy.sym_s(1, TH) - (2 - 2 * np.cos(TH)))) < 1e-14
    assert np.max(np.abs(sy.sym_a(1, TH) + np.sin(TH))) < 1e-15
    assert abs(sy.sym_m(2, np.pi) - 2 / 15) < 1e-15


@pytest.mark.parametrize("p", [2, 3, 4])
def test_mass_eigenvalues_inside_symbol_range(p):
    # Theorem 3.1(a): {n M^p_n} ~ m_p; eigenvalues lie in [min m_p, max m_p] up to outliers
    n = 40
    ev = np.linalg.eigvalsh(n * m1.matrices(p, n)[0])
    assert ev.max() <= 1 + 1e-12
    assert ev.min() >= (2 / np.pi) ** (2 * p + 2) - 1e-12


@pytest.mark.parametrize("d,p,beta", [(2, 3, 0.5), (2, 5, 0.01), (3, 3, 0.5), (3, 5, 0.01)])
def test_bound_theorems(d, p, beta):
    # Theorems 5.2 / 5.4: min(alpha,beta) L_p <= lambda_i(f) <= max(alpha,beta) L_p
    alpha, m = 1.0, (20 if d == 2 else 10) + p - 2
    th = sy.grid(m, d)
    lam = np.linalg.eigvalsh(sy.symbol_f(p, alpha, beta, th))
    L = sy.laplacian(p, th)[..., None]
    tol = 1e-12 * (1 + L.max())
    assert np.all(lam >= min(alpha, beta) * L - tol) and np.all(lam <= max(alpha, beta) * L + tol)


def test_alpha_equals_beta_gives_scaled_laplacian():
    th = sy.grid(9, 3)
    f = sy.symbol_f(3, 0.7, 0.7, th)
    L = sy.laplacian(3, th)
    for i in range(3):
        assert np.max(np.abs(f[..., i, i] - 0.7 * L)) < 1e-14
    assert np.max(np.abs(f[..., 0, 1])) == 0.0
