"""Host-side logic of the C-ABI library, no GPU needed: symbol exports, the
config surface, phantoms, the encoder stream, and the memo decision logic
replayed against the reference's recorded key sequences."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

import mlr_oracle as O


def test_library_exports_every_declared_symbol(mlrg):
    declared = set()
    for h in ("mlr.h", "mlrg.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        declared |= set(re.findall(r"\b(mlrg?_[A-Za-z0-9_]+)\s*\(", text))
    handle = ctypes.CDLL(mlrg.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(handle, s)]
    assert not missing, missing
    assert set(mlrg.EXPORTS) <= declared


def test_config_defaults_and_errors(mlrg):
    cfg = mlrg.Config()
    dump = cfg.dump()
    for line in ("n1 = 32", "phi = 0.523599", "alpha = 0.001", "n_inner = 4", "n_outer = 30", "tau = 0.92",
                 "pipeline = optimized", "memoization = off", "chunk_extent = 16", "key_dim = 60",
                 "encoder_seed = 1337", "nprobe = 8", "insert_queue_cap = 256", "coalesce_bytes = 4096"):
        assert line in dump, line
    cfg.set("memoization", "local").set("tau", 0.9)
    assert "memoization = local" in cfg.dump() and "tau = 0.9" in cfg.dump()
    with pytest.raises(mlrg.MlrError) as e:
        cfg.set("no_such_key", "1")
    assert e.value.code == mlrg.MLR_ERR_CONFIG and "unknown config key" in str(e.value)
    with pytest.raises(mlrg.MlrError) as e:
        cfg.set("pipeline", "fast")
    assert e.value.code == mlrg.MLR_ERR_CONFIG


def test_config_file_roundtrip(mlrg, tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# comment\nn1 = 64\n  n0=64 # trailing\nmemoization = distributed\n")
    cfg = mlrg.Config(str(p))
    d = cfg.dump()
    assert "n1 = 64" in d and "n0 = 64" in d and "memoization = distributed" in d
    p.write_text("n1 = x\n")
    with pytest.raises(mlrg.MlrError):
        mlrg.Config(str(p))


@pytest.mark.parametrize("case", ["recon_c16_memo_grid", "recon_c32_memo_grid", "recon_cfg1_memo_direct"])
def test_blocks_phantom_matches_reference(mlrg, case):
    z = golden(case)
    n = z["phantom"].shape[0]
    ph = mlrg.make_phantom("blocks", n, n, n, 1).numpy()
    assert np.array_equal(ph.astype(np.complex64), z["phantom"])


def test_shepp_phantom_matches_restatement(mlrg):
    ph = mlrg.make_phantom("shepp3d-like", 12, 10, 14, 0).numpy()
    assert np.allclose(ph, O.shepp3d((12, 10, 14)), atol=0)


def test_array_view_is_zero_copy_and_keeps_owner_alive(mlrg):
    a = (np.arange(24) + 1j * np.arange(24)[::-1]).reshape(2, 3, 4)
    arr = mlrg.array_from_numpy(a)
    v = arr.view()
    assert np.array_equal(v, a) and not v.flags.writeable
    del arr  # the view holds the Array
    import gc
    gc.collect()
    assert np.array_equal(v, a)


def test_array_io_roundtrip(mlrg, tmp_path):
    a = (np.arange(24) + 1j * np.arange(24)[::-1]).reshape(2, 3, 4)
    arr = mlrg.array_from_numpy(a)
    assert arr.shape == (2, 3, 4)
    p = str(tmp_path / "a.lvol")
    arr.save(p)
    assert np.array_equal(mlrg.Array.load(p).numpy(), a)
    with open(p, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(mlrg.MlrError):
        mlrg.Array.load(p)


def test_out_of_scope_entry_points_fail_cleanly(mlrg):
    L = mlrg.lib()
    assert not L.mlr_server_start(b"127.0.0.1", 0, 64, 8, 1024)
    assert b"HBM" in L.mlr_last_error()
    assert not L.mlr_plan_offload(b"", 1.0, b"plan")


@pytest.mark.parametrize("shape", [(16, 16, 16), (4, 16, 16), (16, 8, 12)])
def test_projection_matrix_matches_reference_keys(mlrg, shape):
    z = golden("encoder")
    idx = [(16, 16, 16), (4, 16, 16), (16, 8, 12)].index(shape)
    P = mlrg.projection_matrix(shape).reshape(60, -1)
    assert np.array_equal(P, O.projection_matrix(shape))
    meta, raw, keys = z[f"meta{idx}"], z[f"raw{idx}"], z[f"keys{idx}"]
    for r in range(len(meta)):
        op, loc = (int(v) for v in meta[r])
        k = O.encode_projection(z[f"x{idx}_op{op}_loc{loc}"], P)
        assert np.array_equal(k, raw[r])
        assert np.array_equal(mlrg.slot_mix(k, loc, op), keys[r])


def test_memostore_kats_through_cpp(mlrg):
    z = golden("store")
    m = mlrg.Memo(nprobe=2, nlist=4, train_size=32)
    ins, qry, qi, qcs = z["inserted"], z["queries"], z["q_int"], z["q_cs"]
    qpos = 0
    for i in range(len(ins)):
        while qpos < len(qi) and qi[qpos, 0] == i:
            # a single-key batch at a fresh location is a pure store query
            oc, cs, vid = m.lookup(qry[qpos:qpos + 1], [1000 + qpos], [0], [1])
            hit = int(qi[qpos, 2])
            assert int(oc[0]) == (1 if hit else 0)
            assert cs[0] == qcs[qpos]
            if hit:
                assert int(vid[0]) == int(qi[qpos, 3])
            qpos += 1
        assert m.insert(ins[i], 1)
        m.flush()
    assert qpos == len(qi)


def replay(mlrg, z, n_slab_bytes):
    """Re-derives every memo decision of a reference run from its recorded
    keys through the C++ client/store."""
    keys, meta = z["keys"], z["key_meta"]
    aborted = bool(int(str(z["txt_aborted_txt"]).split()[0]))
    m = mlrg.Memo()
    out = []
    i, last_it = 0, int(meta[-1, 0])
    while i < len(meta):
        j = i + 1
        while j < len(meta) and meta[j, 2] != 0:
            j += 1
        it = int(meta[i, 0])
        oc, cs, _ = m.lookup(keys[i:j], meta[i:j, 2], meta[i:j, 1], [n_slab_bytes] * (j - i))
        out += [(it, int(meta[k, 1]), int(meta[k, 2]), int(oc[k - i]), float(cs[k - i])) for k in range(i, j)]
        for k in range(i, j):
            if oc[k - i] == 0:
                m.insert(keys[k], n_slab_bytes)
        nxt = int(meta[j, 0]) if j < len(meta) else None
        if nxt != it and not (aborted and it == last_it):
            m.flush()
        i = j
    return out, m.counters()


@pytest.mark.parametrize("case", ["recon_c16_memo_grid", "recon_c32_memo_grid", "recon_cfg1_memo_direct"])
def test_memo_decisions_replay_reference(mlrg, case):
    z = golden(case)
    n = z["phantom"].shape[0]
    out, ctr = replay(mlrg, z, 8 + 16 * 16 * n * n)
    got = np.array([o[:4] for o in out], np.int32)
    assert np.array_equal(got, z["audit_int"])
    want = dict(l.split("=") for l in str(z["txt_counters_txt"]).split())
    for k in ("lookups", "cache_hits", "remote_hits", "misses", "cache_comparisons", "cache_probes",
              "batches_sent", "inserts_enqueued", "inserts_sent", "inserts_dropped"):
        assert ctr[k] == int(want[k]), k


def test_cnn_init_weights_match_reference(mlrg):
    """init_cnn (encoder.cpp:441-470): one GaussianStream over conv1, conv2, fc."""
    z = golden("cnn")
    c1, c2, fc = mlrg.cnn_weights()
    assert np.array_equal(c1, z["c1w"]) and np.array_equal(c2, z["c2w"]) and np.array_equal(fc, z["fcw"])
