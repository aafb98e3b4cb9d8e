"""Device operators through the mlrg C-ABI vs the reference's outputs
(golden fixtures) and the numpy restatement. Tolerances are fp32-level:
the device computes in complex64 with fp32 FFTs and gathers, the reference
in complex128 (its gridding itself is exact to ~3e-12)."""
import numpy as np
import pytest

import mlr_oracle as O
from conftest import golden, golden_geometry, rel

pytestmark = pytest.mark.gpu
TOL = 2e-5  # relative L2: complex64 storage of the grids and outputs
KERNELS = ["es", "gaussian"]  # geometry.hpp: both evaluate the reference's NUDFT


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(np.complex64)).cuda()


def host(t):
    return t.cpu().numpy().astype(np.complex128)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("case", ["ops_c16", "ops_ragged", "ops_c32"])
def test_usfft_ops_match_reference(mlrg, torch_cuda, case, kernel):
    torch = torch_cuda
    z = golden(case)
    n1, n0, n2, nt, h, w = golden_geometry(z)
    ctx = mlrg.Context(n1, n0, n2, nt, h, w, kernel=kernel)
    u, mid, pf, dh = (dev(torch, z[k]) for k in ("in_u", "in_mid", "in_projf", "in_dhat"))
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    out = ctx.fu1d(u, e(n1, h, n2))
    ctx.sync()
    assert rel(host(out), z["fu1d_grid"]) < TOL
    out = ctx.fu1d_adj(mid, e(n1, n0, n2))
    ctx.sync()
    assert rel(host(out), z["fu1d_adj_grid"]) < TOL
    out = ctx.fu2d(mid, e(nt, h, w))
    ctx.sync()
    assert rel(host(out), z["fu2d_grid"]) < TOL
    out = ctx.fu2d(mid, e(nt, h, w), d_hat=dh)
    ctx.sync()
    assert rel(host(out), z["fused_grid"]) < TOL
    out = ctx.fu2d_adj(pf, e(n1, h, n2))
    ctx.sync()
    assert rel(host(out), z["fu2d_adj_grid"]) < TOL


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("case", ["ops_c16", "ops_ragged", "ops_c32"])
def test_f2d_forward_adjoint_L_match_reference(mlrg, torch_cuda, case, kernel):
    torch = torch_cuda
    z = golden(case)
    n1, n0, n2, nt, h, w = golden_geometry(z)
    ctx = mlrg.Context(n1, n0, n2, nt, h, w, kernel=kernel)
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    ps, pf, u = dev(torch, z["in_projs"]), dev(torch, z["in_projf"]), dev(torch, z["in_u"])
    o = ctx.f2d(ps, e(nt, h, w))
    ctx.sync()
    assert rel(host(o), z["f2d"]) < 1e-6
    o = ctx.f2d(pf, e(nt, h, w), adjoint=True)
    ctx.sync()
    assert rel(host(o), z["f2d_adj"]) < 1e-6
    o = ctx.forward_L(u, e(nt, h, w))
    ctx.sync()
    assert rel(host(o), z["forward_L_grid"]) < TOL
    o = ctx.adjoint_L(ps, e(n1, n0, n2))
    ctx.sync()
    assert rel(host(o), z["adjoint_L_grid"]) < TOL


def test_grad_div_match_reference(mlrg, torch_cuda):
    torch = torch_cuda
    z = golden("ops_ragged")
    n1, n0, n2, nt, h, w = golden_geometry(z)
    ctx = mlrg.Context(n1, n0, n2, nt, h, w)
    g = [torch.empty((n1, n0, n2), dtype=torch.complex64, device="cuda") for _ in range(3)]
    ctx.grad(dev(torch, z["in_u"]), *g)
    ctx.sync()
    for ax in range(3):
        assert rel(host(g[ax]), z[f"grad{ax}"]) < 1e-6
    out = torch.empty((n1, n0, n2), dtype=torch.complex64, device="cuda")
    ctx.div(*(dev(torch, z[f"in_g{ax}"]) for ax in range(3)), out)
    ctx.sync()
    assert rel(host(out), z["div"]) < 1e-6


@pytest.mark.parametrize("n,nt,kernel", [(64, 48, "es"), (128, 128, "es"), (64, 48, "gaussian")])
def test_ops_vs_restatement_and_adjointness(mlrg, torch_cuda, n, nt, kernel):
    torch = torch_cuda
    rng = np.random.default_rng(n)
    g = O.Geometry(n, n, n, nt, n, n)
    ctx = mlrg.Context(n, n, n, nt, n, n, kernel=kernel)
    cplx = lambda *s: (rng.standard_normal(s) + 1j * rng.standard_normal(s))
    u, v, p = cplx(n, n, n), cplx(n, n, n), cplx(nt, n, n)
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    a = host(ctx.fu1d(dev(torch, u), e(n, n, n)))
    b = host(ctx.fu1d_adj(dev(torch, v), e(n, n, n)))
    ctx.sync()
    # <A u, v> == <u, A* v>
    assert abs(np.vdot(v, a) - np.vdot(b, u)) / (np.linalg.norm(a) * np.linalg.norm(v)) < 1e-5
    if n <= 64:
        assert rel(a, O.fu1d_gridding(u, g)) < TOL
        sl = slice(0, 4)  # fu2d restatement is slow; a 4-row slab
        c = host(ctx.fu2d(dev(torch, v[:, sl].copy()), e(nt, 4, n)))
        ctx.sync()
        assert rel(c, O.fu2d_gridding(v[:, sl], g)) < TOL
    c = host(ctx.fu2d(dev(torch, v), e(nt, n, n)))
    d = host(ctx.fu2d_adj(dev(torch, p), e(n, n, n)))
    ctx.sync()
    assert abs(np.vdot(p, c) - np.vdot(d, v)) / (np.linalg.norm(c) * np.linalg.norm(p)) < 1e-5


def test_encode_keys_match_reference(mlrg, torch_cuda):
    torch = torch_cuda
    z = golden("recon_c16_memo_grid")
    n = z["phantom"].shape[0]
    ctx = mlrg.Context(n, n, n, n, n, n)
    x = (np.random.default_rng(3).standard_normal((n, n, n)) + 1j).astype(np.complex64)
    for op in ("fu1d", "fu2d", "fu1d_adj", "fu2d_adj"):
        keys, norms = ctx.encode(op, dev(torch, x))
        P = O.projection_matrix((16, n, n) if op in ("fu1d", "fu1d_adj") else (n, 16, n))
        ax = 1 if op in ("fu2d", "fu2d_adj") else 0
        for s in range(keys.shape[0]):
            chunk = np.take(x.astype(np.complex128), range(16 * s, 16 * s + 16), axis=ax)
            want = O.slot_mix(O.encode_projection(chunk, P), 1337, s, mlrg.OPS[op])
            assert np.allclose(keys[s], want, rtol=1e-5, atol=1e-5 * np.abs(want).max())
            assert abs(norms[s] - np.linalg.norm(chunk)) < 1e-6 * norms[s]


@pytest.mark.parametrize("shape", [(64, 64, 64), (40, 48, 72)])
def test_encode_tcgen05_keys_match_reference(mlrg, torch_cuda, shape):
    """Slab shapes large enough for the tcgen05 encoder (encode_tc.cu: K = 2n spans
    >= 2 stages of 128 columns per SM): keys of both slab axes against the
    reference's double-accumulated projection (encoder.cpp:405-422), including a
    ragged last slab (40 planes / 48 rows = 2.5 / 3 slabs)."""
    torch = torch_cuda
    d0, d1, d2 = shape
    ctx = mlrg.Context(d0, d1, d2, d0, d1, d2)
    x = (np.random.default_rng(5).standard_normal(shape) + 1j * np.random.default_rng(6).standard_normal(shape)
         + 0.25).astype(np.complex64)
    for op in ("fu1d", "fu2d"):
        keys, norms = ctx.encode(op, dev(torch, x))
        ax = 1 if op == "fu2d" else 0
        mats = {}
        for s in range(keys.shape[0]):
            chunk = np.take(x.astype(np.complex128), range(16 * s, min(16 * s + 16, shape[ax])), axis=ax)
            if chunk.shape not in mats:
                mats[chunk.shape] = O.projection_matrix(chunk.shape)
            want = O.slot_mix(O.encode_projection(chunk, mats[chunk.shape]), 1337, s, mlrg.OPS[op])
            assert np.allclose(keys[s], want, rtol=1e-5, atol=1e-5 * np.abs(want).max()), (op, s)
            assert abs(norms[s] - np.linalg.norm(chunk)) < 1e-6 * norms[s]


@pytest.mark.parametrize("idx,shape", [(0, (16, 16, 16)), (1, (4, 16, 16)), (2, (16, 8, 12))])
def test_cnn_encoder_matches_reference_keys(mlrg, torch_cuda, idx, shape):
    """Device CNN keys (cnn.cu) against the reference's (encoder.cpp:95-197) for
    random chunks: the chunk is the whole projection-shaped input of fu2d_adj
    (n_theta, h, w) = shape, one slab of extent h."""
    torch = torch_cuda
    z = golden("cnn")
    d0, d1, d2 = shape
    ctx = mlrg.Context(16, 16, 16, d0, d1, d2)
    for op in range(4):
        x = torch.from_numpy(z[f"x{idx}_op{op}"].astype(np.complex64)).cuda()
        keys, norms = ctx.encode_cnn("fu2d_adj", x, chunk_extent=d1)
        want = z[f"raw{idx}"][op]
        assert np.allclose(keys[0], want, rtol=1e-5, atol=1e-6 * np.abs(want).max())
        assert abs(norms[0] - np.linalg.norm(z[f"x{idx}_op{op}"])) <= 1e-6 * norms[0]


@pytest.mark.parametrize("nk,k,dup", [(1024, 64, False), (1100, 64, True), (40, 64, False)])
def test_gpu_kmeans_bit_identical_to_host(mlrg, torch_cuda, nk, k, dup):
    """The device IVF trainer (memo_gpu.cu k_kmeans) against the host k-means
    (memo.cpp kmeans_train, pinned to the reference's store KATs): identical
    centroids and nearest-centroid assignment, bit for bit, including duplicate
    keys (ties) and fewer keys than centroids."""
    import ctypes as C
    rng = np.random.default_rng(nk)
    keys = rng.standard_normal((nk, 60)).astype(np.float32)
    if dup:
        keys[1::7] = keys[0::7][: len(keys[1::7])]
    out = {}
    for dev_flag in (0, 1):
        kk = min(k, nk)
        cent = np.zeros((kk, 60), np.float32)
        near = np.zeros(nk, np.int64)
        rc = mlrg.lib().mlrg_kmeans(keys.ctypes.data, nk, 60, k, 7, 20, dev_flag, cent.ctypes.data, near.ctypes.data)
        assert rc == 0, mlrg.lib().mlrg_last_error()
        out[dev_flag] = (cent, near)
    assert np.array_equal(out[0][0].view(np.uint32), out[1][0].view(np.uint32))
    assert np.array_equal(out[0][1], out[1][1])
