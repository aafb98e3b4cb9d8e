"""Diagnostics: per-operator relative error vs the reference fixtures and the
per-iteration deviation of device reconstructions (prints, never asserts)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import paper_2511_01893_b200 as m
import mlr_oracle as O
from conftest import golden, golden_geometry, rel

def dev(a): return torch.from_numpy(np.ascontiguousarray(a).astype(np.complex64)).cuda()
def host(t): return t.cpu().numpy().astype(np.complex128)
for case in ["ops_c16", "ops_ragged", "ops_c32"]:
    z = golden(case); n1, n0, n2, nt, h, w = golden_geometry(z)
    ctx = m.Context(n1, n0, n2, nt, h, w)
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    r = {}
    r["fu1d"] = rel(host(ctx.fu1d(dev(z["in_u"]), e(n1, h, n2))), z["fu1d_grid"])
    r["fu1d_adj"] = rel(host(ctx.fu1d_adj(dev(z["in_mid"]), e(n1, n0, n2))), z["fu1d_adj_grid"])
    r["fu2d"] = rel(host(ctx.fu2d(dev(z["in_mid"]), e(nt, h, w))), z["fu2d_grid"])
    r["fu2d_adj"] = rel(host(ctx.fu2d_adj(dev(z["in_projf"]), e(n1, h, n2))), z["fu2d_adj_grid"])
    r["f2d"] = rel(host(ctx.f2d(dev(z["in_projs"]), e(nt, h, w))), z["f2d"])
    r["fwdL"] = rel(host(ctx.forward_L(dev(z["in_u"]), e(nt, h, w))), z["forward_L_grid"])
    # input rounding floor: the same op of the c64-rounded input in f64
    print(case, {k: f"{v:.2e}" for k, v in r.items()}, flush=True)
for n, nt in [(64, 48)]:
    rng = np.random.default_rng(n); g = O.Geometry(n, n, n, nt, n, n); ctx = m.Context(n, n, n, nt, n, n)
    cplx = lambda *s: (rng.standard_normal(s) + 1j * rng.standard_normal(s))
    u, v, p = cplx(n, n, n), cplx(n, n, n), cplx(nt, n, n)
    e = lambda *s: torch.empty(s, dtype=torch.complex64, device="cuda")
    a = host(ctx.fu1d(dev(u), e(n, n, n))); b = host(ctx.fu1d_adj(dev(v), e(n, n, n)))
    print("adj fu1d", abs(np.vdot(v, a) - np.vdot(b, u)) / (np.linalg.norm(a) * np.linalg.norm(v)))
    print("fu1d vs oracle", rel(a, O.fu1d_gridding(u.astype(np.complex64).astype(complex), g)))
    c = host(ctx.fu2d(dev(v[:, :4].copy()), e(nt, 4, n)))
    print("fu2d vs oracle", rel(c, O.fu2d_gridding(v[:, :4].astype(np.complex64).astype(complex), g)))
    c = host(ctx.fu2d(dev(v), e(nt, n, n))); d = host(ctx.fu2d_adj(dev(p), e(n, n, n)))
    print("adj fu2d", abs(np.vdot(p, c) - np.vdot(d, v)) / (np.linalg.norm(c) * np.linalg.norm(p)), flush=True)
KERNELS = os.environ.get("DIAG_KERNELS", "es").split(",")
for case, memo, kern in [(c, mm, k) for k in KERNELS for c, mm in [("recon_c32_off_grid", "off"), ("recon_c32_memo_grid", "local"), ("recon_c64_off_grid", "off"), ("recon_cfg1_memo_direct", "local")]]:
    z = golden(case); n = z["phantom"].shape[0]; nt = z["data"].shape[0]
    u = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
    cfg = f"n1={n}\nn0={n}\nn2={n}\nn_theta={nt}\nh={n}\nw={n}\nn_outer=10\nmemoization={memo}\ngridding_kernel={kern}\n"
    r = m.reconstruct_device(cfg, torch.from_numpy(z["data"]).cuda(), u, reference=torch.from_numpy(z["phantom"]).cuda())
    rows = m.parse_csv(r.csv); ref = [[float(x) for x in l.split(",")] for l in str(z["txt_report_csv"]).strip().splitlines()[1:]]
    print(case, kern, "aborted", r.aborted, "rows", len(rows), len(ref), "u rel", f"{rel(u.cpu().numpy(), z['u']):.2e}")
    if memo != "off":
        meta, _ = r.audit(); print("  audit equal:", meta.shape == z["audit_int"].shape and np.array_equal(meta, z["audit_int"]),
                                    "first diff:", None if meta.shape != z["audit_int"].shape else np.argwhere((meta != z["audit_int"]).any(1))[:3].ravel())
    for a, b in zip(rows, ref):
        print(f"  it{int(b[0])} loss {a['loss']:.6e} ref {b[1]:.6e} rel {abs(a['loss']-b[1])/abs(b[1]):.1e}  E {a['E']:.6f} ref {b[2]:.6f}  m/r/c {int(a['miss'])}/{int(a['remote_hit'])}/{int(a['cache_hit'])} ref {int(b[4])}/{int(b[5])}/{int(b[6])}")
