"""CPU pins of the library's 1D modal basis (ads_modal_basis, host-only; SURVEY.md §8 row f3;
PAPER.md:157-165 Eqs. 17-18): K phi = lambda M phi with phi^T M phi = I.

Pinned against (a) the closed form of linear elements, (b) scipy's generalised symmetric
eigensolver on the oracle's Gram matrices (themselves pinned in test_oracle_pins.py), and
(c) the defining identities (M-orthonormality, residual)."""
import math

import numpy as np
import pytest
import scipy.linalg

import oracle


@pytest.fixture(scope="module")
def ads():
    import paper_1911_08158_b200 as ads
    from paper_1911_08158_b200 import build
    build.build()
    return ads


def _pencil(p, nel, bc):
    M, K, _ = oracle.matrices_1d(p, nel, bc=bc)
    if bc == 1:
        M, K = M[1:-1, 1:-1], K[1:-1, 1:-1]
    return M, K


@pytest.mark.parametrize("nel", [4, 17, 64])
def test_linear_elements_closed_form(ads, nel):
    """p = 1, zero Dirichlet: M = h/6 tridiag(1, 4, 1), K = 1/h tridiag(-1, 2, -1) share the
    eigenvectors sin(k pi x_i), lambda_k = (6/h^2)(1 - cos(k pi h))/(2 + cos(k pi h))."""
    lam, phi = ads.modal_basis(nel, 1, 1)
    h = 1.0 / nel
    th = np.arange(1, nel) * math.pi * h
    exact = 6.0 / h ** 2 * (1 - np.cos(th)) / (2 + np.cos(th))
    assert np.abs(lam - exact).max() <= 1e-13 * exact.max()
    x = np.arange(1, nel) * h
    for k in (0, nel // 2 - 1, nel - 2):  # eigenvector k is a multiple of sin((k+1) pi x)
        s = np.sin((k + 1) * math.pi * x)
        c = phi[:, k] @ s / (s @ s)
        assert np.abs(phi[:, k] - c * s).max() <= 1e-12 * np.abs(phi[:, k]).max()


@pytest.mark.parametrize("p,nel,bc", [(2, 16, 1), (3, 64, 1), (1, 9, 0), (4, 30, 0), (5, 12, 1), (3, 200, 1)])
def test_against_scipy_and_identities(ads, p, nel, bc):
    lam, phi = ads.modal_basis(nel, p, bc)
    M, K = _pencil(p, nel, bc)
    ref = scipy.linalg.eigh(K, M, eigvals_only=True)
    scale = np.abs(ref).max()
    assert np.abs(lam - ref).max() <= 1e-13 * scale
    assert np.abs(phi.T @ M @ phi - np.eye(len(lam))).max() <= 1e-13 * len(lam) ** 0.5
    assert np.abs(K @ phi - M @ phi * lam).max() <= 1e-13 * scale
    assert np.all(np.diff(lam) >= 0)
    if bc == 0:  # natural BC: the constant is the (only) zero mode
        assert abs(lam[0]) <= 1e-10 * scale and lam[1] > 1e-6


def test_bad_arguments(ads):
    with pytest.raises(ads.AdsError):
        ads.modal_basis(0, 2, 1)
    with pytest.raises(ads.AdsError):
        ads.modal_basis(8, 7, 1)
