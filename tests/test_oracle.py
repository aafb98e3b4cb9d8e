"""Pins the numpy restatement (oracle/mlr_oracle.py) to the reference's own
outputs (tests/golden/*.npz, produced by the unmodified reference through
oracle/make_golden.py). CPU only."""
import numpy as np
import pytest

import mlr_oracle as O
from conftest import golden, golden_geometry, rel

OPS_CASES = ["ops_c16", "ops_ragged"]


@pytest.mark.parametrize("case", OPS_CASES)
@pytest.mark.parametrize("path,sfx", [("gridding", "_grid"), ("direct", "_direct")])
def test_operators_match_reference(case, path, sfx):
    z = golden(case)
    g = O.Geometry(*golden_geometry(z))
    assert rel(O.fu1d(z["in_u"], g, path), z["fu1d" + sfx]) < 1e-13
    assert rel(O.fu1d_adj(z["in_mid"], g, path), z["fu1d_adj" + sfx]) < 1e-13
    assert rel(O.fu2d(z["in_mid"], g, path), z["fu2d" + sfx]) < 1e-13
    assert rel(O.fu2d_adj(z["in_projf"], g, path), z["fu2d_adj" + sfx]) < 1e-13
    assert rel(O.fu2d(z["in_mid"], g, path) - z["in_dhat"], z["fused" + sfx]) < 1e-13
    assert rel(O.forward_L(z["in_u"], g, path), z["forward_L" + sfx]) < 1e-13
    assert rel(O.adjoint_L(z["in_projs"], g, path), z["adjoint_L" + sfx]) < 1e-13


@pytest.mark.parametrize("case", OPS_CASES)
def test_f2d_grad_div_match_reference(case):
    z = golden(case)
    assert rel(O.f2d(z["in_projs"]), z["f2d"]) < 1e-13
    assert rel(O.f2d_adj(z["in_projf"]), z["f2d_adj"]) < 1e-13
    g = O.grad(z["in_u"])
    for ax in range(3):
        assert np.array_equal(g[ax], z[f"grad{ax}"])
    assert np.array_equal(O.div([z[f"in_g{ax}"] for ax in range(3)]), z["div"])


def test_gridding_rejects_tiny_extents():
    # the reference corrupts its heap here; the oracle refuses
    with pytest.raises(ValueError):
        O.DimPlan.make(8, np.zeros(4))


def test_spec_frequency_examples():
    # SPEC.md:73-74 (phi -> 0 limit of nu_z; theta = 0 row of nu_x)
    g = O.Geometry(4, 4, 4, 4, 4, 4, phi=1e-9)
    nu_z, nu_x, nu_y = O.frequency_grids(g)
    assert np.allclose(nu_z, [-0.5, -0.25, 0.0, 0.25])
    assert np.allclose(nu_x[:4], [-0.5, -0.25, 0.0, 0.25]) and np.allclose(nu_y[:4], 0.0)


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_encoder_keys_match_reference(idx):
    z = golden("encoder")
    meta, keys, raw = z[f"meta{idx}"], z[f"keys{idx}"], z[f"raw{idx}"]
    shape = z[f"x{idx}"].shape
    P = O.projection_matrix(shape)
    for r in range(len(meta)):
        op, loc = (int(v) for v in meta[r])
        x = z[f"x{idx}_op{op}_loc{loc}"]
        k = O.encode_projection(x, P)
        assert np.array_equal(k, raw[r])
        assert np.array_equal(O.slot_mix(k, 1337, loc, op), keys[r])


def test_memostore_kats():
    z = golden("store")
    st = O.MemoStore(nlist=4, nprobe=2, train_size=32)
    ins, qry, qi, qcs = z["inserted"], z["queries"], z["q_int"], z["q_cs"]
    qpos = 0
    for i in range(len(ins)):
        while qpos < len(qi) and qi[qpos, 0] == i:
            o = st.query(qry[qpos], np.float32(0.92), 0)
            assert (int(o["found"]), int(o["hit"]), int(o["id"])) == tuple(int(v) for v in qi[qpos, 1:])
            assert np.float32(o["cs"]) == qcs[qpos]
            qpos += 1
        st.insert(ins[i], ((1.0, None), 0))
    assert qpos == len(qi)
    assert np.array_equal(st.centroids, z["centroids"])


def test_recon_memo_c16_matches_reference():
    z = golden("recon_c16_memo_grid")
    n = z["phantom"].shape[0]
    g = O.Geometry(n, n, n, n, n, n)
    r = O.reconstruct(z["data"].astype(np.complex128), g, n_outer=10, memo=True,
                      reference=z["phantom"].astype(np.complex128))
    a = np.array([(it, op, loc, oc) for it, op, loc, oc, _ in r["audit"]])
    assert np.array_equal(a, z["audit_int"])
    assert r["aborted"] == bool(int(str(z["txt_aborted_txt"]).split()[0]))
    ref_rows = str(z["txt_report_csv"]).strip().splitlines()[1:]
    assert len(ref_rows) == len(r["rows"])
    for line, row in zip(ref_rows, r["rows"]):
        f = [float(v) for v in line.split(",")]
        assert abs(row["loss"] - f[1]) <= 1e-9 * abs(f[1])
        assert (row["miss"], row["remote_hit"], row["cache_hit"]) == (f[4], f[5], f[6])
    assert rel(r["u"], z["u"]) < 1e-6


def test_cnn_restatement_matches_reference_keys():
    """The CNN key encoder (encoder.cpp:95-197, seeded init_cnn weights) restated
    in numpy against the reference's keys of random chunks (summation order
    differs: float-rounding level agreement)."""
    z = golden("cnn")
    c1w, c2w, fcw = z["c1w"], z["c2w"], z["fcw"]
    for idx in range(3):
        raw = z[f"raw{idx}"]
        for op in range(4):
            k = O.cnn_forward(z[f"x{idx}_op{op}"], c1w, c2w, fcw)
            assert np.allclose(k, raw[op], rtol=1e-5, atol=1e-6 * np.abs(raw[op]).max())
