"""Operators at BASELINE.json's full sizes: configs[1] (256^3, 256 angles) and
configs[2]'s 512^3 (where fu2d runs the four-step column passes). Slabs of
every USFFT operator are checked against the numpy restatement (itself
pinned to the reference's golden vectors in test_oracle.py); the whole
volume through size-independent properties: adjointness and linearity."""
import numpy as np
import pytest

import mlr_oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu
TOL = 2e-5  # relative L2, as test_gpu_ops.py: complex64 grids and outputs


def _cplx(rng, *s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)


@pytest.mark.parametrize("n", [256, 512])
def test_fullsize_slabs_match_restatement(mlrg, torch_cuda, n):
    torch = torch_cuda
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).astype(np.complex64)).cuda()
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    host = lambda t: t.cpu().numpy().astype(np.complex128)
    g = O.Geometry(n, n, n, n, n, n)
    ctx = mlrg.Context(n, n, n, n, n, n)
    rng = np.random.default_rng(n)
    u, v = _cplx(rng, 2, n, n), _cplx(rng, 2, n, n)  # two planes along axis 0
    a, b = ctx.fu1d(dev(u), e(2, n, n)), ctx.fu1d_adj(dev(v), e(2, n, n))
    w, p = _cplx(rng, n, 1, n), _cplx(rng, n, 1, n)  # one detector row (axis 1)
    c, d = ctx.fu2d(dev(w), e(n, 1, n)), ctx.fu2d_adj(dev(p), e(n, 1, n))
    ctx.sync()
    assert rel(host(a), O.fu1d_gridding(u, g)) < TOL
    assert rel(host(b), O.fu1d_adj_gridding(v, g)) < TOL
    assert rel(host(c), O.fu2d_gridding(w, g)) < TOL
    assert rel(host(d), O.fu2d_adj_gridding(p, g)) < TOL


def test_configs1_operators_adjoint_and_linear(mlrg, torch_cuda):
    """Whole 256^3 volume, 256 angles, on the device: <A x, y> = <x, A* y> for
    fu1d and fu2d, and fu2d(x + 2 y) = fu2d(x) + 2 fu2d(y)."""
    torch = torch_cuda
    n = 256
    ctx = mlrg.Context(n, n, n, n, n, n)
    gen = torch.Generator(device="cuda").manual_seed(7)
    rnd = lambda *s: torch.randn(s, dtype=torch.complex64, device="cuda", generator=gen)
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    vdot = lambda x, y: complex(torch.vdot(x.flatten().to(torch.complex128), y.flatten().to(torch.complex128)))
    nrm = lambda x: float(torch.linalg.vector_norm(x.to(torch.complex128)))
    x, y = rnd(n, n, n), rnd(n, n, n)
    ax, ay = ctx.fu1d(x, e(n, n, n)), ctx.fu1d_adj(y, e(n, n, n))
    ctx.sync()
    assert abs(vdot(y, ax) - vdot(ay, x)) / (nrm(ax) * nrm(y)) < 1e-5
    p = rnd(n, n, n)
    fx, fy, fp = ctx.fu2d(x, e(n, n, n)), ctx.fu2d(y, e(n, n, n)), ctx.fu2d_adj(p, e(n, n, n))
    fxy = ctx.fu2d(x + 2 * y, e(n, n, n))
    ctx.sync()
    assert abs(vdot(p, fx) - vdot(fp, x)) / (nrm(fx) * nrm(p)) < 1e-5
    assert nrm(fxy - (fx + 2 * fy)) / nrm(fxy) < 1e-5
