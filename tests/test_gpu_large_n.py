"""Transform extents up to 2048 (configs[4]'s 2048^3): M = 4096-point oversampled
lines in every pass (fu1d along n0, the fu2d row pass along n2, the four-step
column passes along n1), on thin geometries that fit the numpy restatement
(oracle/mlr_oracle.py, pinned to the reference's fixtures by test_oracle.py),
plus adjointness of each operator pair and an offload-invariant solve."""
import numpy as np
import pytest

import mlr_oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

TOL = 2e-5

# (n1, n0, n2, n_theta, h, w): one long extent each
SHAPES = [(2048, 16, 16, 6, 16, 16), (16, 16, 2048, 6, 16, 2048), (16, 2048, 16, 6, 32, 16)]


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(np.complex64)).cuda()


@pytest.mark.parametrize("shape", SHAPES)
def test_long_extent_operators_match_restatement(mlrg, torch_cuda, shape):
    torch = torch_cuda
    n1, n0, n2, nt, h, w = shape
    g = O.Geometry(n1, n0, n2, nt, h, w)
    ctx = mlrg.Context(n1, n0, n2, nt, h, w)
    rng = np.random.default_rng(sum(shape))
    cplx = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    u, v, p = cplx(n1, n0, n2), cplx(n1, h, n2), cplx(nt, h, w)
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    a = ctx.fu1d(dev(torch, u), e(n1, h, n2)).cpu().numpy()
    b = ctx.fu1d_adj(dev(torch, v), e(n1, n0, n2)).cpu().numpy()
    c = ctx.fu2d(dev(torch, v), e(nt, h, w)).cpu().numpy()
    d = ctx.fu2d_adj(dev(torch, p), e(n1, h, n2)).cpu().numpy()
    ctx.sync()
    assert rel(a, O.fu1d_gridding(u, g)) < TOL
    sl = slice(0, 2)  # the 2D restatement on a 2-row slab
    assert rel(c[:, sl], O.fu2d_gridding(v[:, sl], g)) < TOL
    # <A x, y> == <x, A* y>
    assert abs(np.vdot(v, a) - np.vdot(b, u)) / (np.linalg.norm(a) * np.linalg.norm(v)) < 1e-5
    assert abs(np.vdot(p, c) - np.vdot(d, v)) / (np.linalg.norm(c) * np.linalg.norm(p)) < 1e-5


def test_long_extent_solve_offload_bit_identical(mlrg, torch_cuda):
    """A memoized solve with n1 = 2048 (four-step 4096-point column passes, 128
    sixteen-plane RSP chunks) through the ADMM-Offload path: psi / psi_prev /
    lambda in pinned host memory change nothing in the arithmetic."""
    torch = torch_cuda
    n1, n0, n2, nt, h, w = 2048, 16, 16, 8, 16, 16
    ph = mlrg.make_phantom("blocks", n1, n0, n2, 1).numpy().astype(np.complex64)
    ctx = mlrg.Context(n1, n0, n2, nt, h, w)
    d = torch.empty((nt, h, w), dtype=torch.complex64, device="cuda")
    ctx.forward_L(dev(torch, ph), d)
    ctx.sync()
    outs = []
    for off in ("off", "host"):
        u = torch.empty((n1, n0, n2), dtype=torch.complex64, device="cuda")
        cfg = (f"n1={n1}\nn0={n0}\nn2={n2}\nn_theta={nt}\nh={h}\nw={w}\nn_outer=4\nmemoization=local\n"
               f"nudft_path=gridding\noffload={off}\n")
        r = mlrg.reconstruct_device(cfg, d, u, reference=dev(torch, ph))
        outs.append((u.cpu().numpy(), [l.split(",")[:7] for l in r.csv.splitlines()], r.audit()[0]))
    (u0, c0, a0), (u1, c1, a1) = outs
    assert np.array_equal(u0, u1)
    assert c0 == c1
    assert np.array_equal(a0, a1)
    assert np.isfinite(u0).all() and np.linalg.norm(u0) > 0
