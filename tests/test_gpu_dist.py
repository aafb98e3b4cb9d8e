"""The z-slab sharded solver with 2 ranks: two processes
sharing cuda:0, exchanging the mid array, halos and memo values through the
library's CUDA IPC peer mappings exactly as on a multi-GPU node. The
assembled volume, the per-iteration report and the memo hit/miss sequence
must match the reference's run (and the single-GPU solve)."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT, golden, rel

pytestmark = pytest.mark.gpu
WORLD = 2


def config_text(n, nt, memo):
    return (f"n1={n}\nn0={n}\nn2={n}\nn_theta={nt}\nh={n}\nw={n}\nn_outer=10\n"
            f"memoization={memo}\nnudft_path=gridding\n")


def _worker(rank, world, port, case, memo, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist

    import paper_2511_01893_b200 as m

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = m.Comm.from_torch(timeout_s=120)
    z = np.load(os.path.join(ROOT, "tests", "golden", case + ".npz"))
    n, nt = z["phantom"].shape[0], z["data"].shape[0]
    s = torch.cuda.current_stream()
    d = torch.from_numpy(z["data"]).cuda()
    ref = torch.from_numpy(z["phantom"]).cuda()
    solver = m.Solver(config_text(n, nt, memo), d, reference=ref, stream=s.cuda_stream, comm=comm)
    a, b, c, dd = solver.shard()
    aborted = False
    for _ in range(10):
        if not solver.step():
            aborted = True
            break
    u = torch.empty((b - a, n, n), dtype=torch.complex64, device="cuda")
    solver.volume(u)
    meta, _ = solver.audit()
    tiers = solver.tiers() if memo != "off" else {}
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), u=u.cpu().numpy(), a=a, b=b, meta=meta, csv=solver.csv,
             aborted=aborted, spilled=tiers.get("spilled_values", 0))
    del solver
    comm.barrier()
    del comm
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case,memo,fence", [("recon_c32_memo_grid", "local", "default"),
                                             ("recon_c64_off_grid", "off", "default"),
                                             ("recon_cfg1_memo_direct", "local", "default"),
                                             ("recon_c32_memo_grid", "local", "event")])
def test_sharded_solver_matches_reference(mlrg, torch_cuda, tmp_path, case, memo, fence, monkeypatch):
    """fence=event forces the stream-ordered interprocess-event fence (shard.hpp
    PeerEvents), which the engine otherwise uses only when every rank has its own
    GPU: the ranks here share cuda:0."""
    import torch.multiprocessing as mp

    if fence != "default":
        monkeypatch.setenv("MLRG_FENCE", fence)

    z = golden(case)
    n = z["phantom"].shape[0]
    mp.start_processes(_worker, args=(WORLD, free_port(), case, memo, str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(WORLD)]
    assert [int(p["a"]) for p in parts] == [0, int(parts[0]["b"])] and int(parts[-1]["b"]) == n
    u = np.concatenate([p["u"] for p in parts], axis=0)
    csv0 = str(parts[0]["csv"])
    for p in parts[1:]:  # global report and decisions, identical on every rank
        assert [l.split(",")[:7] for l in str(p["csv"]).splitlines()] == [l.split(",")[:7] for l in csv0.splitlines()]
        assert np.array_equal(p["meta"], parts[0]["meta"])
    if memo != "off":
        assert np.array_equal(parts[0]["meta"], z["audit_int"]), "sharded memo decisions differ from the reference"
    assert bool(parts[0]["aborted"]) == bool(int(str(z["txt_aborted_txt"]).split()[0]))
    assert rel(u, z["u"]) <= 1e-4
    # against the single-GPU solve of the same inputs: only the reduction order differs
    torch = torch_cuda
    d = torch.from_numpy(z["data"]).cuda()
    ref = torch.from_numpy(z["phantom"]).cuda()
    one = mlrg.Solver(config_text(n, z["data"].shape[0], memo), d, reference=ref)
    for _ in range(10):
        if not one.step():
            break
    u1 = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
    one.volume(u1)
    assert rel(u, u1.cpu().numpy()) <= 1e-6
    rows1 = [l.split(",")[:7] for l in one.csv.strip().splitlines()[1:]]
    rows2 = [l.split(",")[:7] for l in csv0.strip().splitlines()[1:]]
    assert len(rows1) == len(rows2)
    for r1, r2 in zip(rows1, rows2):
        assert r1[4:7] == r2[4:7]  # miss / remote_hit / cache_hit counts
        # the objective cancels 3-4 digits by iteration 10 (see test_gpu_recon.py), so a
        # different summation order moves it ~1e-6 relative while u moves < 1e-8
        assert abs(float(r1[1]) - float(r2[1])) <= 1e-4 * abs(float(r1[1]))


def _big_worker(rank, world, port, n, memo, steps, outdir, offload="off"):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2511_01893_b200 as m

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = m.Comm.from_torch(timeout_s=300) if world > 1 else None
    s = torch.cuda.current_stream()
    ph = torch.from_numpy(m.make_phantom("blocks", n, n, n, 1).numpy().astype(np.complex64)).cuda()
    ctx = m.Context(n, n, n, n, n, n, stream=s.cuda_stream)
    d = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
    ctx.forward_L(ph, d)
    ctx.sync()
    del ctx
    cfg = (f"n1={n}\nn0={n}\nn2={n}\nn_theta={n}\nh={n}\nw={n}\nn_outer={steps}\nmemoization={memo}\n"
           f"nudft_path=gridding\noffload={offload}\n")
    solver = m.Solver(cfg, d, reference=ph, stream=s.cuda_stream, comm=comm)
    a, b, _, _ = solver.shard()
    for _ in range(steps):
        solver.step()
    u = torch.empty((b - a, n, n), dtype=torch.complex64, device="cuda")
    solver.volume(u)
    meta, _ = solver.audit()
    np.savez(os.path.join(outdir, f"w{world}_rank{rank}.npz"), u=u.cpu().numpy(), meta=meta, csv=solver.csv)
    del solver
    if comm is not None:
        comm.barrier()
    del comm
    dist.destroy_process_group()


def test_sharded_512_matches_single_gpu(mlrg, torch_cuda, tmp_path):
    """configs[2] (512^3, 512 angles) z-slab split, SURVEY.md §8(d) parity gate for
    cfg3: cross-GPU-count equality. Two ranks (sharing cuda:0) against one rank,
    2 outer iterations with memoization on: identical memo decisions and u within
    1e-6 (only the CG/ADMM scalar summation order differs)."""
    import torch.multiprocessing as mp

    n, steps = 512, 2
    for world in (1, 2):
        mp.start_processes(_big_worker, args=(world, free_port(), n, "local", steps, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    one = np.load(tmp_path / "w1_rank0.npz")
    two = [np.load(tmp_path / f"w2_rank{r}.npz") for r in range(2)]
    assert np.array_equal(two[0]["meta"], one["meta"]) and np.array_equal(two[1]["meta"], one["meta"])
    u2 = np.concatenate([p["u"] for p in two], axis=0)
    assert rel(u2, one["u"]) <= 1e-6


def test_sharded_configs1_memo_through_ivf_training(mlrg, torch_cuda, tmp_path):
    """configs[1] (256^3, 256 angles), memo on for 10 outer iterations: the store
    passes 1024 published keys and trains its IVF index mid-run. The key index is
    replicated through the communicator, so two ranks must make the single-GPU
    decisions before and after training (memo under sharding)."""
    import torch.multiprocessing as mp

    n, steps = 256, 10
    for world in (1, 2):
        mp.start_processes(_big_worker, args=(world, free_port(), n, "local", steps, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    one = np.load(tmp_path / "w1_rank0.npz")
    two = [np.load(tmp_path / f"w2_rank{r}.npz") for r in range(2)]
    assert len(one["meta"]) > 2048  # enough decisions to have trained (1024 published keys)
    assert np.array_equal(two[0]["meta"], one["meta"]) and np.array_equal(two[1]["meta"], one["meta"])
    assert rel(np.concatenate([p["u"] for p in two], axis=0), one["u"]) <= 1e-6


@pytest.mark.parametrize("n,world,memo,offload", [(64, 3, "off", "off"), (48, 2, "local", "off"),
                                                 (80, 3, "local", "off"), (64, 2, "local", "host")])
def test_sharded_uneven_partitions_match_single_gpu(mlrg, torch_cuda, tmp_path, n, world, memo, offload):
    """Uneven assign() splits (ranks owning 1 or 2 slabs, a short last slab), more
    than two ranks, and ADMM-Offload under sharding: the same decisions and u as
    one rank without offload."""
    import torch.multiprocessing as mp

    steps = 4
    for wsz in (1, world):
        mp.start_processes(_big_worker, args=(wsz, free_port(), n, memo, steps, str(tmp_path),
                                              offload if wsz > 1 else "off"),
                           nprocs=wsz, join=True, start_method="spawn")
    one = np.load(tmp_path / "w1_rank0.npz")
    parts = [np.load(tmp_path / f"w{world}_rank{r}.npz") for r in range(world)]
    for p in parts:
        assert np.array_equal(p["meta"], one["meta"])
    assert rel(np.concatenate([p["u"] for p in parts], axis=0), one["u"]) <= 1e-6
