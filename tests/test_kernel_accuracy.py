"""The spreading-kernel claim of DESIGN.md §4: the reference's 24-tap Gaussian
gridding and the B200 build's default 10-tap exponential-of-semicircle (ES)
kernel both reproduce the direct NUDFT (operators.cpp:133-200), to 3e-12 and
2e-9 respectively (10x below the complex64 rounding of the outputs, 2.6e-8). The ES plan below restates csrc/geometry.cpp DimPlan::make
(kernel = es) in numpy; CPU only."""
import math

import numpy as np

import mlr_oracle as O

W, BETA = 10, 2.30 * 10


def es_plan(n, freqs):
    m = max(O.next_pow2(2 * n), 24)
    delta = 2 * math.pi / m
    hw = W * delta / 2
    phi = lambda d: np.where(np.abs(d) <= hw, np.exp(BETA * (np.sqrt(np.maximum(0, 1 - (d / hw) ** 2)) - 1)), 0.0)
    xg, wg = np.polynomial.legendre.leggauss(200)
    k = (np.arange(n) - n // 2).astype(float)
    phihat = (hw * wg[None, :] * phi(hw * xg)[None, :] * np.cos(k[:, None] * hw * xg[None, :])).sum(1)
    x = np.fmod(-2 * math.pi * freqs, 2 * math.pi)
    x = np.where(x < 0, x + 2 * math.pi, x)
    l0 = np.ceil(x / delta - W / 2).astype(np.int64)
    ls = l0[:, None] + np.arange(W)[None, :]
    return m, n // 2, delta / phihat, np.mod(ls, m), phi(x[:, None] - ls * delta)


def fu2d_es(v, g):
    _, nu_x, nu_y = O.frequency_grids(g)
    m1, c1, dc1, gi1, gw1 = es_plan(g.n1, nu_x)
    m2, c2, dc2, gi2, gw2 = es_plan(g.n2, nu_y)
    kk = v.shape[1]
    grid = np.zeros((kk, m1, m2), complex)
    vv = np.transpose(v, (1, 0, 2)) * (dc1[:, None] * dc2[None, :])[None]
    grid[np.ix_(np.arange(kk), O._wrap(g.n1, c1, m1), O._wrap(g.n2, c2, m2))] = vv
    grid = O._fft(O._fft(grid, +1, axis=2), +1, axis=1)
    out = np.empty((kk, len(nu_x)), complex)
    for k in range(kk):
        sub = grid[k][gi1[:, :, None], gi2[:, None, :]]
        out[k] = np.einsum("ta,ta->t", np.einsum("tab,tb->ta", sub, gw2), gw1)
    out *= np.exp(1j * (-2 * math.pi * nu_x * c1)) * np.exp(1j * (-2 * math.pi * nu_y * c2))
    return np.transpose(out.reshape(kk, g.n_theta, g.w), (1, 0, 2))


def test_gaussian_and_es_gridding_match_direct_nudft():
    n = 32
    g = O.Geometry(n, n, n, n, n, n)
    rng = np.random.default_rng(0)
    v = rng.standard_normal((n, 2, n)) + 1j * rng.standard_normal((n, 2, n))
    exact = O.fu2d_direct(v, g)
    rel = lambda a: np.linalg.norm(a - exact) / np.linalg.norm(exact)
    assert rel(O.fu2d_gridding(v, g)) < 1e-11
    assert rel(fu2d_es(v, g)) < 5e-9
