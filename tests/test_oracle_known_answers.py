"""Known answers that pin the CPU oracle without numpy's summation order or the reference
code: brute-force momentum sums (the kind of check the reference's own tests make,
pkg/tests/test_selfenergy.py:39-90, pkg/tests/test_kgrid.py:63-110) and the analytic
free evolution of the Cayley integrator.  CPU only.
"""

import numpy as np
import pytest

from conftest import rel_err
from oracle import kbe_oracle as O


def _fold(k, grid):
    """Index of the grid momentum equal to k modulo 2 pi (nearest-point search)."""
    d = np.angle(np.exp(1j * (grid - k)))          # signed distance on the circle
    i = int(np.argmin(np.abs(d)))
    assert abs(d[i]) < 1e-9
    return i


def _bf_pol(gl, gg, kv):
    n = len(kv)
    out = np.zeros((n, 2, 2), dtype=complex)
    for q in range(n):
        for kp in range(n):
            s = _fold(kv[kp] + kv[q], kv)
            for j in range(2):
                for m in range(2):
                    out[q, j, m] += gl[s, j, m] * gg[kp, m, j]
    return out


def _bf_sigma(gl, gg, u1, u2, kv):
    """First and second second-Born terms as direct momentum sums (Eq. 8 and Alg. 2)."""
    n = len(kv)
    s1 = np.zeros((n, 2, 2), dtype=complex)
    s2 = np.zeros((n, 2, 2), dtype=complex)
    for k in range(n):
        for q in range(n):
            for kp in range(n):
                a = _fold(kv[kp] + kv[q], kv)
                b = _fold(kv[k] - kv[q], kv)
                c = _fold(kv[kp] + kv[q] - kv[k], kv)
                for j in range(2):
                    for m in range(2):
                        s1[k, j, m] += gl[a, 1 - j, 1 - m] * gg[kp, 1 - m, 1 - j] * gl[b, j, m]
                        s2[k, j, m] += gl[kp, j, 1 - m] * gg[c, 1 - m, 1 - j] * gl[q, 1 - j, m]
    pref = u1 * u2 / n ** 2
    return s1 * pref, s2 * pref


@pytest.mark.parametrize("n_k", [2, 4, 6, 8])
def test_index_maps_fold_momenta(n_k):
    kv = O.k_values(n_k)
    S, D = O.sum_index(n_k), O.diff_index(n_k)
    for a in range(n_k):
        for b in range(n_k):
            assert S[a, b] == _fold(kv[a] + kv[b], kv)
            assert D[a, b] == _fold(kv[a] - kv[b], kv)


@pytest.mark.parametrize("n_k", [2, 4, 6, 8])
def test_sigma_stages_match_brute_force(n_k):
    rng = np.random.default_rng(40 + n_k)
    gl = rng.standard_normal((n_k, 2, 2)) + 1j * rng.standard_normal((n_k, 2, 2))
    gg = rng.standard_normal((n_k, 2, 2)) + 1j * rng.standard_normal((n_k, 2, 2))
    kv = O.k_values(n_k)
    u1, u2 = 0.8, 1.3
    pol = O.polarizability(gl, gg)
    assert rel_err(pol, _bf_pol(gl, gg, kv)) <= 1e-13
    s1, s2 = _bf_sigma(gl, gg, u1, u2, kv)
    assert rel_err(O.sigma_first(pol, gl, u1, u2), s1) <= 1e-13
    assert rel_err(O.sigma_second(gl, gg, u1, u2), s2) <= 1e-13
    assert rel_err(O.sigma_slice(gl, gg, u1, u2), s1 - s2) <= 1e-13


def test_free_evolution_is_the_cayley_factor_and_second_order():
    """U = 0, no pulse: G<_vv(k; t_n, 0) = i phi_v^n with phi = (1 - i e dt/2) / (1 + i e dt/2)
    exactly, and the error against i exp(-i e t) falls by ~4 when dt halves."""
    n_k, T = 4, 1.0
    errs = []
    for dt in (0.02, 0.01):
        N = int(round(T / dt))
        drv = O.OracleDriver(n_k, O.Model(), dt, N)
        drv.run()
        ev, _ = O.bands(O.Model(), n_k)
        phi = (1 - 0.5j * ev * dt) / (1 + 0.5j * ev * dt)
        n = np.arange(N + 1)
        got = drv.GL[:, 0, 0, :, 0]
        assert rel_err(got, 1j * phi[:, None] ** n[None, :]) <= 1e-13
        errs.append(np.abs(got[:, N] - 1j * np.exp(-1j * ev * T)).max())
    assert 3.5 <= errs[0] / errs[1] <= 4.5


def _sigma_fourier(gp, gr, u1, u2):
    """The Fourier-space form K1 (sigma_fft_kernel / sigma_dft_kernel) evaluates:
    Sigma^_jm(f) = pref s_jm det(gp^(f)) gr^_{m'j'}(-f), x^(f) = sum_k x[k] e^{-2 pi i f k / n_k},
    s_jm = +1 (j = m) / -1 (j != m), pref = u1 u2 / n_k^2, followed by the inverse transform."""
    n = gp.shape[0]
    GP, GR = np.fft.fft(gp, axis=0), np.fft.fft(gr, axis=0)
    det = GP[:, 0, 0] * GP[:, 1, 1] - GP[:, 0, 1] * GP[:, 1, 0]
    GRm = GR[(-np.arange(n)) % n]
    out = np.empty_like(GP)
    for j in range(2):
        for m in range(2):
            out[:, j, m] = (1 if j == m else -1) * det * GRm[:, 1 - m, 1 - j]
    return np.fft.ifft(out, axis=0) * (u1 * u2 / n ** 2)


@pytest.mark.parametrize("n_k", [2, 4, 6, 8, 12, 16, 64, 128])
def test_fourier_sigma_identity_matches_direct_sums(n_k):
    """The algebra behind K1: the factorised second-Born Sigma (P, Sigma1, X, Sigma2 as
    circular correlations, selfenergy.py:59-203) collapses in Fourier space to one
    determinant times one reversed transform per frequency.  Checked against the
    oracle's direct sums at every n_k class the kernels take (powers of two: FFT;
    others: DFT GEMMs) and, at small n_k, against the brute-force momentum sums."""
    rng = np.random.default_rng(100 + n_k)
    shape = (n_k, 2, 2)
    gp = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    gr = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    want = O.sigma_slice(gp, gr, 0.7, 1.3)
    got = _sigma_fourier(gp, gr, 0.7, 1.3)
    assert rel_err(got, want) <= 1e-13
    if n_k <= 12:
        s1, s2 = _bf_sigma(gp, gr, 0.7, 1.3, O.k_values(n_k))
        assert rel_err(got, s1 - s2) <= 1e-13
