"""Times the UNMODIFIED CPU reference (oracle/_ref/libmlr.so, built from
/root/reference/proj by oracle/Makefile) through its own C API (mlr.h).

TEST / BASELINE INFRASTRUCTURE ONLY: bench.py's cpu_baseline leg and its
--impl reference arm run this in a subprocess; the product never does.

A "sample" is one call of mlr_reconstruct with memoization off, the gridding
path and `workers` threads on synthetic data of the configured shape (random
complex values fed through an LVOL file: the reference's own projector,
mlr_project, is a dense O(N^4) DFT and would dominate the sample). The
per-iteration time is the reference's own phase timers (ms_lsp + ms_rsp +
ms_update of its CSV, admm.cpp:197-206, which exclude the objective); with
n_inner=1 the LSP share is scaled to the configured 4 inner iterations.

    python oracle/ref_runner.py --n 256 --n-theta 256 --n-inner 4 [--workers W]
prints one JSON object.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libmlr.so")


def _lib():
    if not os.path.exists(REF_LIB):
        raise FileNotFoundError(f"{REF_LIB} missing (build it with `make -C oracle` where /root/reference exists)")
    L = C.CDLL(REF_LIB)
    L.mlr_config_new.restype = C.c_void_p
    L.mlr_config_set.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
    L.mlr_array_load.restype = C.c_void_p
    L.mlr_array_load.argtypes = [C.c_char_p]
    L.mlr_reconstruct.restype = C.c_void_p
    L.mlr_reconstruct.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    L.mlr_result_csv.restype = C.c_void_p
    L.mlr_result_csv.argtypes = [C.c_void_p]
    L.mlr_free.argtypes = [C.c_void_p]
    L.mlr_last_error.restype = C.c_char_p
    L.mlr_result_free.argtypes = [C.c_void_p]
    L.mlr_array_free.argtypes = [C.c_void_p]
    L.mlr_config_free.argtypes = [C.c_void_p]
    return L


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run(n: int, n_theta: int, n_inner: int = 4, n_outer: int = 1, workers: int | None = None, seed: int = 5):
    L = _lib()
    cores = os.cpu_count() or 1
    slabs = -(-n // 16)
    workers = workers or max(1, min(cores, slabs))
    cfg = L.mlr_config_new()
    for k, v in dict(n1=n, n0=n, n2=n, n_theta=n_theta, h=n, w=n, n_inner=n_inner, n_outer=n_outer,
                     memoization="off", nudft_path="gridding", workers=workers).items():
        if L.mlr_config_set(cfg, k.encode(), str(v).encode()) != 0:
            raise RuntimeError(L.mlr_last_error().decode())
    rng = np.random.default_rng(seed)
    d = (rng.standard_normal((n_theta, n, n)) + 1j * rng.standard_normal((n_theta, n, n))).astype("<c16")
    header = b"LVOL" + bytes([3, 0]) + bytes(10) + np.asarray(d.shape, "<u8").tobytes()
    with tempfile.NamedTemporaryFile(suffix=".lvol", delete=False) as f:
        f.write(header + d.tobytes())
        path = f.name
    try:
        arr = L.mlr_array_load(path.encode())
    finally:
        os.unlink(path)
    if not arr:
        raise RuntimeError(L.mlr_last_error().decode())
    t0 = time.perf_counter()
    res = L.mlr_reconstruct(cfg, arr, None)
    wall = time.perf_counter() - t0
    if not res:
        raise RuntimeError(L.mlr_last_error().decode())
    p = L.mlr_result_csv(res)
    csv = C.cast(p, C.c_char_p).value.decode()
    L.mlr_free(p)
    L.mlr_result_free(res)
    L.mlr_array_free(arr)
    L.mlr_config_free(cfg)
    rows = [dict(zip(csv.splitlines()[0].split(","), map(float, l.split(",")))) for l in csv.strip().splitlines()[1:]]
    scale = 4.0 / n_inner
    per_iter_ms = [r["ms_lsp"] * scale + r["ms_rsp"] + r["ms_update"] for r in rows]
    return dict(n=n, n_theta=n_theta, n_inner_sampled=n_inner, n_outer=n_outer, workers=workers,
                cores=cores, cpu=cpu_model(), wall_s=wall, per_iter_ms=per_iter_ms,
                it_per_s=1000.0 / float(np.mean(per_iter_ms)), rows=rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--n-theta", type=int, default=None)
    ap.add_argument("--n-inner", type=int, default=4)
    ap.add_argument("--n-outer", type=int, default=1)
    ap.add_argument("--workers", type=int, default=None)
    a = ap.parse_args()
    print(json.dumps(run(a.n, a.n_theta or a.n, a.n_inner, a.n_outer, a.workers)))


if __name__ == "__main__":
    main()
