"""The N>1 (z-slab sharded) path's host logic on CPU, world_size 2 over gloo
(SURVEY.md §8(e)): torch.distributed rendezvous -> the library's node-local
communicator (barrier, rank-ordered allreduce, allgather), the assign()
partition, and the sharded memo layer's global decisions: each rank holds the
keys of its own slabs, all-gathers them, and must reproduce the reference's
recorded hit/miss sequence exactly (scalerun.cpp:14-27, memoclient.cpp:220-300)."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

import mlr_oracle as O

WORLD = 2


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import paper_2511_01893_b200 as m

    return m, dist


def _comm_worker(rank, world, port):
    m, dist = _init(rank, world, port)
    comm = m.Comm.from_torch(timeout_s=60)
    # allreduce: rank-ordered sum, bit-identical on every rank
    def part(r):
        rng = np.random.default_rng(100 + r)
        return rng.standard_normal(7) * 10.0 ** rng.integers(-8, 8, 7)

    got = comm.allreduce(part(rank))
    parts = [part(r) for r in range(world)]
    want = np.zeros(7)
    for p in parts:
        want = want + p
    assert np.array_equal(got, want)
    import torch
    t = torch.from_numpy(got.copy())
    dist.broadcast(t, src=0)
    assert np.array_equal(t.numpy(), got), "allreduce differs between ranks"
    # allgather + repeated barriers (bank reuse)
    for it in range(50):
        out = comm.allgather(bytes([rank, it % 256]) * 3)
        assert out == [bytes([r, it % 256]) * 3 for r in range(world)]
        comm.barrier()
    del comm
    dist.destroy_process_group()


def _run(fn, *args):
    import torch.multiprocessing as mp

    mp.start_processes(fn, args=(WORLD, free_port()) + args, nprocs=WORLD, join=True, start_method="spawn")


def test_comm_over_gloo_rendezvous():
    _run(_comm_worker)


def test_partition_is_reference_assign(mlrg):
    for n1, h, world in [(256, 256, 2), (64, 64, 3), (1024, 1024, 8), (100, 36, 2), (512, 512, 8)]:
        part = mlrg.partition(n1, h, world)
        for axis, n in ((0, n1), (1, h)):
            want = [(min(n, lo * 16), min(n, hi * 16)) for lo, hi in O.assign((n + 15) // 16, world)]
            got = [tuple(int(v) for v in part[r, 2 * axis:2 * axis + 2]) for r in range(world)]
            assert got == want
    with pytest.raises(mlrg.MlrError):
        mlrg.partition(32, 32, 3)  # 2 slabs cannot feed 3 ranks


def _sharded_replay_worker(rank, world, port, case):
    m, dist = _init(rank, world, port)
    from conftest import golden as gold

    z = gold(case)
    n = z["phantom"].shape[0]
    part = m.partition(n, n, world)
    comm = m.Comm.from_torch(timeout_s=60)
    keys, meta = z["keys"], z["key_meta"]
    aborted = bool(int(str(z["txt_aborted_txt"]).split()[0]))
    vbytes = 8 + 16 * 16 * n * n
    memo = m.Memo()
    out = []
    i, last_it = 0, int(meta[-1, 0])
    while i < len(meta):
        j = i + 1
        while j < len(meta) and meta[j, 2] != 0:
            j += 1
        it, op = int(meta[i, 0]), int(meta[i, 1])
        axis = 1 if op in (1, 3) else 0
        lo, hi = part[rank, 2 * axis] // 16, (part[rank, 2 * axis + 1] + 15) // 16
        # this rank encodes only its own slabs; the global list comes from the allgather
        local = [k for k in range(i, j) if lo <= int(meta[k, 2]) < hi]
        cap = j - i
        buf = np.zeros((cap + 1, keys.shape[1] + 1), np.float32)
        buf[0, 0] = len(local)
        for q, k in enumerate(local):
            buf[1 + q, 0] = meta[k, 2]
            buf[1 + q, 1:] = keys[k]
        gathered = comm.allgather(buf.tobytes())
        gl, gk = [], []
        for b in gathered:
            a = np.frombuffer(b, np.float32).reshape(cap + 1, -1)
            for q in range(int(a[0, 0])):
                gl.append(int(a[1 + q, 0]))
                gk.append(a[1 + q, 1:])
        assert gl == [int(v) for v in meta[i:j, 2]], "allgather must restore the global slab order"
        gk = np.array(gk)
        assert np.array_equal(gk, keys[i:j])
        oc, cs, _ = memo.lookup(gk, gl, [op] * cap, [vbytes] * cap)
        out += [(it, op, gl[q], int(oc[q])) for q in range(cap)]
        for q in range(cap):
            if oc[q] == 0:
                memo.insert(gk[q], vbytes)
        nxt = int(meta[j, 0]) if j < len(meta) else None
        if nxt != it and not (aborted and it == last_it):
            memo.flush()
        i = j
    got = np.array(out, np.int32)
    assert np.array_equal(got, z["audit_int"]), f"rank {rank}: sharded decisions differ from the reference"
    del comm
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["recon_c32_memo_grid", "recon_cfg1_memo_direct"])
def test_sharded_memo_decisions_match_reference(case):
    golden(case)  # skip when the fixture is absent
    _run(_sharded_replay_worker, case)


def _abort_worker(rank, world, port):
    m, dist = _init(rank, world, port)
    comm = m.Comm.from_torch(timeout_s=60)
    comm.barrier()
    if rank == 0:  # this rank fails; its peers must not wait for it
        comm.abort()
    else:
        import time

        t0 = time.perf_counter()
        with pytest.raises(m.MlrError, match="peer rank failed"):
            comm.barrier()
        assert time.perf_counter() - t0 < 30.0
    with pytest.raises(m.MlrError):  # payloads above the 1 MiB slot are refused
        comm.allgather(b"x" * ((1 << 20) + 1))
    dist.barrier()
    del comm
    dist.destroy_process_group()


def test_comm_abort_releases_peers():
    _run(_abort_worker)
