"""Memo value tiers (csrc/cold_tier.hpp): the HBM arena is a ring that keeps
one insert window free; older values spill to pinned host memory and are read
in place on a hit. The reference's store is unbounded (memostore.cpp:112-120),
so a forced-small arena must reproduce the reference's decisions and u exactly
as a large one does, on the device lookup, the host client and the sharded
path, and must never fail mid-solve."""
import os

import numpy as np
import pytest

from conftest import ROOT, golden, rel
import test_gpu_dist as dist_t

pytestmark = pytest.mark.gpu


def min_arena(n, n_inner=4, world=1, windows=1):
    """`windows` insert windows + one slab (c_abi.cpp build_engine); 1: the smallest
    legal ring (every spill synchronous at the flush), >= 2.5: ColdSpiller also
    copies the following window's span out in the background."""
    slabs = -(-n // 16)
    most = -(-slabs // world)
    window = min(256, 4 * n_inner * most)
    return (windows * window + 1) * ((16 * n * n * 8 + 255) // 256 * 256)


def config_text(n, nt, memo):
    return (f"n1={n}\nn0={n}\nn2={n}\nn_theta={nt}\nh={n}\nw={n}\nn_outer=10\n"
            f"memoization={memo}\nnudft_path=gridding\n")


@pytest.mark.parametrize("case", ["recon_c32_memo_grid", "recon_cfg1_memo_direct"])
@pytest.mark.parametrize("device_memo", ["1", "0"])
@pytest.mark.parametrize("windows", [1, 3])
def test_tiny_arena_spills_and_matches_reference(mlrg, torch_cuda, monkeypatch, case, device_memo, windows):
    torch = torch_cuda
    z = golden(case)
    n, nt = z["phantom"].shape[0], z["data"].shape[0]
    monkeypatch.setenv("MLRG_DEVICE_MEMO", device_memo)
    monkeypatch.setenv("MLRG_MEMO_ARENA_BYTES", str(min_arena(n, windows=windows)))
    u = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
    r = mlrg.reconstruct_device(config_text(n, nt, "local"), torch.from_numpy(z["data"]).cuda(), u,
                                reference=torch.from_numpy(z["phantom"]).cuda())
    t = r.tiers()
    assert t["arena_bytes"] == min_arena(n, windows=windows)
    assert t["spilled_values"] > 0 and t["spilled_bytes"] > 0, t
    meta, _ = r.audit()
    assert np.array_equal(meta, z["audit_int"]), "decisions differ with a spilling arena"
    assert r.aborted == bool(int(str(z["txt_aborted_txt"]).split()[0]))
    assert rel(u.cpu().numpy(), z["u"]) <= 1e-4
    # and bit-identical to the unconstrained run: where a value lives never changes its bytes
    monkeypatch.delenv("MLRG_MEMO_ARENA_BYTES")
    u2 = torch.empty_like(u)
    r2 = mlrg.reconstruct_device(config_text(n, nt, "local"), torch.from_numpy(z["data"]).cuda(), u2,
                                 reference=torch.from_numpy(z["phantom"]).cuda())
    assert r2.tiers()["spilled_values"] == 0
    assert torch.equal(u, u2)


def test_arena_below_one_window_fails_at_setup(mlrg, torch_cuda, monkeypatch):
    """fail fast at setup, never after hours of solving."""
    torch = torch_cuda
    z = golden("recon_c32_memo_grid")
    monkeypatch.setenv("MLRG_MEMO_ARENA_BYTES", str(min_arena(32) - 256))
    u = torch.empty((32, 32, 32), dtype=torch.complex64, device="cuda")
    with pytest.raises(mlrg.MlrError, match="below one insert window"):
        mlrg.reconstruct_device(config_text(32, 32, "local"), torch.from_numpy(z["data"]).cuda(), u)


def test_sharded_tiny_arena_matches_reference(mlrg, torch_cuda, tmp_path, monkeypatch):
    """Two ranks, each with the smallest ring: spills land in per-rank shared-memory
    segments that every rank maps, decisions and u stay the reference's."""
    import torch.multiprocessing as mp

    z = golden("recon_cfg1_memo_direct")
    n = z["phantom"].shape[0]
    monkeypatch.setenv("MLRG_MEMO_ARENA_BYTES", str(min_arena(n, world=2)))
    mp.start_processes(dist_t._worker, args=(2, dist_t.free_port(), "recon_cfg1_memo_direct", "local", str(tmp_path)),
                       nprocs=2, join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    assert int(parts[0]["spilled"]) > 0 and int(parts[0]["spilled"]) == int(parts[1]["spilled"])
    assert np.array_equal(parts[0]["meta"], z["audit_int"]) and np.array_equal(parts[1]["meta"], z["audit_int"])
    assert rel(np.concatenate([p["u"] for p in parts], axis=0), z["u"]) <= 1e-4
