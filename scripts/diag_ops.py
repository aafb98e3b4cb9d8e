"""Per-operator accuracy of the device path vs the numpy restatement at
power-of-two sizes beyond the golden fixtures (random and phantom inputs)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import paper_2511_01893_b200 as m
import mlr_oracle as O
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
def dev(a): return torch.from_numpy(np.ascontiguousarray(a).astype(np.complex64)).cuda()
def host(t): torch.cuda.synchronize(); return t.cpu().numpy().astype(np.complex128)
for n in [32, 64, 128]:
    nt = n
    g = O.Geometry(n, n, n, nt, n, n); ctx = m.Context(n, n, n, nt, n, n)
    rng = np.random.default_rng(n)
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    ph = m.make_phantom("blocks", n, n, n, 1).numpy()
    for kind, u in [("random", (rng.standard_normal((n, n, n)) + 1j * rng.standard_normal((n, n, n)))), ("phantom", ph)]:
        u = u.astype(np.complex64).astype(complex)
        a = host(ctx.fu1d(dev(u), e(n, n, n)))
        r1 = rel(a, O.fu1d_gridding(u, g))
        k = 4 if n > 64 else n
        mid = O.fu1d_gridding(u, g)[:, :k].astype(np.complex64).astype(complex).copy()
        c = host(ctx.fu2d(dev(mid), e(nt, k, n)))
        q = O.fu2d_gridding(mid, g)
        r2 = rel(c, q)
        pq = q.astype(np.complex64).astype(complex)
        b = host(ctx.fu2d_adj(dev(pq), e(n, k, n)))
        r3 = rel(b, O.fu2d_adj_gridding(pq, g))
        bb = host(ctx.fu1d_adj(dev(a), e(n, n, n)))
        r4 = rel(bb, O.fu1d_adj_gridding(a.astype(np.complex64).astype(complex), g))
        print(f"n={n} {kind}: fu1d {r1:.2e} fu2d {r2:.2e} fu2d_adj {r3:.2e} fu1d_adj {r4:.2e}", flush=True)
