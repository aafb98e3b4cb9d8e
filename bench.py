"""Benchmark of the memoized ADMM-FFT hot path (BASELINE.json configs[1]:
256^3 phantom, 256 angles, 1 B200, memo off and on).

A step is one ADMM outer iteration (LSP with 4 inner CG steps, RSP, the
multiplier/penalty update, memo flush, objective) of the device solver,
called through the C-ABI (mlrg_solver_step). Inputs are resident in HBM;
every array of an iteration (V = 256^3 complex64 = 134 MB) is larger than L2,
so no L2 flush is inserted between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line (rank 0). Under torchrun (N > 1) the N ranks run ONE
z-slab sharded solve of the same volume (volume planes and detector rows split
in 16-slabs, the mid-array all-to-all and halos over CUDA IPC peer memory):
scaling "strong"; the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # CUDA-core FFMA peak at max clock (no measured figure)
METRIC = "ADMM-FFT iterations/sec at N^3 volume"
# dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
# `ncu --set full` captures (profiles/), filled in per round
TRAFFIC: dict = {  # round 2 final: profiles/r2/ncu_final_*.txt (`ncu --set full`, one launch, cold cache)
    "k_fu2d_gather": 45841664 + 2166016, "k_fu2d_adj_spread": 15731456 + 297472,
    "k_fu2d_cols": 16847104 + 506368, "k_fu2d_rows": 8462336, "k_fu1d": 268567808 + 107938560,
}
# the same captures' per-launch durations (us): ncu serialises launches, while the bench
# overlaps fu2d row batches on two streams (live durations include the sharing)
SERIAL_US: dict = {"k_fu2d_gather": 47.49, "k_fu2d_adj_spread": 48.77, "k_fu2d_cols": 25.31, "k_fu2d_rows": 17.50,
                   "k_fu1d": 312.58}
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # DFMA peak at max clock (computed)
F2F_PER_CLK_SM = 16  # F2F.F64.F32 per clock per SM (scripts/microbench.cu)
PLAN: dict = {}  # fu2d plan figures of the benchmarked geometry (mlrg_ctx_stats)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--n-theta", type=int, default=None)
    ap.add_argument("--kernel", choices=["es", "gaussian"], default="es")
    ap.add_argument("--no-memo-run", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-offload-run", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the gaussian line and the configs[0]/[2] runs")
    ap.add_argument("--same-gpu", action="store_true",
                    help="testing: every rank on cuda:0 with a gloo group (exercises the sharded path on one GPU)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's start-up (NVML init) is over before the timed region
            # begins: its first sample is in
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.skip = len(self.rows)  # start-up samples: reported only if the region saw none
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        skip = getattr(self, "skip", 0)
        rows = self.rows[skip:] if len(self.rows) > skip else self.rows
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


KERNEL = "es"


def config_text(n, nt, memo, n_outer=1000000, offload="off"):
    return (f"n1={n}\nn0={n}\nn2={n}\nn_theta={nt}\nh={n}\nw={n}\nn_outer={n_outer}\n"
            f"memoization={memo}\nnudft_path=gridding\noffload={offload}\ngridding_kernel={KERNEL}\n")


def algorithmic(n, nt, kernel):
    """Per-launch algorithmic work of the profiled kernels, defined as SURVEY.md §8(d)
    defines F2/F1 and B_iter: at the reference's 576 taps per target (a kernel that does
    fewer taps shows a higher effective rate, not a smaller denominator)."""
    T, M = nt * n, 2 * n
    grid = 8 * M * M * 16  # one 16-row complex64 grid
    if kernel in ("k_fu2d_gather", "k_fu2d_adj_spread"):  # 16 detector rows per launch
        return {"flops": T * 16 * (24 * 24 * 4 + 24 * 4 + 12), "bytes": grid + 8 * T * 16}
    if kernel in ("k_fu2d_rows", "k_fu2d_adj_rows"):  # one FFT pass over n1 x 16 rows of length M
        return {"flops": n * 16 * 5 * M * math.log2(M), "bytes": 8 * n * 16 * n + grid // 2}
    if kernel in ("k_fu2d_cols", "k_fu2d_adj_cols"):
        return {"flops": M * 16 * 5 * M * math.log2(M), "bytes": grid // 2 + grid}
    if kernel == "k_fu1d":  # whole volume: u (complex128 iterate) in, mid out
        return {"flops": n * n * (5 * M * math.log2(M) + 2 * n + n * (24 * 4 + 8)), "bytes": 16 * n ** 3 + 8 * n ** 3}
    if kernel == "k_fu1d_adj":
        return {"flops": n * n * (5 * M * math.log2(M) + 2 * n + n * (24 * 4 + 8)), "bytes": 8 * n ** 3 + 16 * n ** 3}
    return {"flops": None, "bytes": None}


# The fused ADMM kernels (vecops.cu) stream complex128 volumes: algorithmic bytes per
# OUTER ITERATION in units of one volume (16 V bytes), reads + writes, as launched by
# solver.cpp with n_inner = 4 (first inner step: no p_prev / G_prev, beta = 0).
HBM_KERNELS = ("k_grad_update", "k_direction", "k_axpy", "k_rsp_multiplier", "k_g_init")
HBM_VOLUMES_PER_ITER = {
    "k_grad_update": 6 + 3 * 8,     # u, g (3), G in, G out; + p_prev, G_prev once a direction exists
    "k_direction": 6 + 3 * 7,       # G, u, g (3) in, p out; + p_prev when beta != 0
    "k_axpy": 4 * 3,                # u, p in, u out
    "k_rsp_multiplier": 13,         # u, lambda (3), psi (3) in; psi_new (3), lambda (3) out
    "k_g_init": 9,                  # psi (3), lambda (3) in; g (3) out
}


# l1tex__throughput (pct of peak) of the committed ncu captures: the shared-memory FFT
# passes work on L2-resident grids and are bound by the L1/shared pipe, not HBM
L1TEX_PCT = {"k_fu2d_rows": 63.2, "k_fu2d_cols": 65.6, "k_fu2d_adj_cols": 58.1, "k_fu1d": 79.1,
             "k_fu2d_adj_spread": 83.8, "k_fu2d_gather": 63.0}  # round 2 final: profiles/r2/ncu_final_*.txt


def local_share(n, world, rank):
    """Fraction of the n1 planes this rank owns: assign() over 16-plane slabs
    (scalerun.cpp:14-27), as the sharded solver partitions the volume."""
    slabs = -(-n // 16)
    base, extra = divmod(slabs, world)
    lo = rank * base + min(rank, extra)
    cnt = base + (1 if rank < extra else 0)
    return (min(n, (lo + cnt) * 16) - min(n, lo * 16)) / n


def kernel_table(prof, n, nt, steps, peaks_gbs, share=1.0):
    """Every profiled kernel against its own roof: the tap kernels
    against FP32 CUDA-core flops (algorithmic, 576 taps), everything else against HBM.
    `share`: this rank's fraction of the volume (whole-volume kernels scale with it;
    the fu2d-class kernels work on one 16-row batch per launch at any rank count)."""
    out = {}
    V16 = 16 * n ** 3 * share
    for name, rec in prof.items():
        ms = rec["ms_total"] / max(steps, 1)
        if name in HBM_VOLUMES_PER_ITER:
            b = HBM_VOLUMES_PER_ITER[name] * V16
            gbs = b / (ms * 1e-3) / 1e9
            out[name] = {"ms_per_step": ms, "launches_per_step": rec["launches"] / max(steps, 1), "bound": "hbm",
                         "bytes_per_step": b, "achieved_gbs": gbs, "frac": gbs / peaks_gbs}
            continue
        work = algorithmic(n, nt, name)
        if name in ("k_fu1d", "k_fu1d_adj") and work["bytes"]:
            work = {"flops": work["flops"] * share, "bytes": work["bytes"] * share}
        per = rec["ms_total"] / rec["launches"]
        if name in ("k_fu2d_gather", "k_fu2d_adj_spread") and work["flops"]:
            tf = work["flops"] / (per * 1e-3) / 1e12
            out[name] = {"ms_per_step": ms, "launches_per_step": rec["launches"] / max(steps, 1), "bound": "fp32",
                         "avg_launch_ms": per, "achieved_tflops": tf, "frac": tf / FP32_PEAK_TFLOPS}
        elif work["bytes"]:
            gbs = work["bytes"] / (per * 1e-3) / 1e9
            out[name] = {"ms_per_step": ms, "launches_per_step": rec["launches"] / max(steps, 1),
                         "bound": "l1/shared (ncu)" if name != "k_fu1d" and name != "k_fu1d_adj" else "hbm",
                         "avg_launch_ms": per, "achieved_gbs": gbs, "frac_of_hbm": gbs / peaks_gbs}
        else:
            out[name] = {"ms_per_step": ms, "launches_per_step": rec["launches"] / max(steps, 1)}
        if name in L1TEX_PCT:
            out[name]["l1tex_pct_ncu"] = L1TEX_PCT[name]
    return out


def iteration_work(n, nt):
    """algorithmic FP32 flops and fused-minimum HBM bytes per outer iteration."""
    V = M_ = n ** 3
    P = nt * n * n
    M0 = M1 = M2 = 2 * n
    F1 = n * n * (5 * M0 * math.log2(M0) + 2 * n + n * (24 * 4 + 8))
    F2 = n * (5 * M1 * M2 * math.log2(M1 * M2) + 2 * n * n + nt * n * (24 * 24 * 4 + 24 * 4 + 12))
    return 13 * F1 + 13 * F2, 8 * (131 * V + 26 * M_ + 22 * P)


def main():
    args = parse()
    global KERNEL
    KERNEL = args.kernel
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.n
    nt = args.n_theta or n

    if args.impl == "reference":
        return reference_arm(args, world, rank, n, nt)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_01893_b200 as m

    if args.same_gpu:
        local = 0
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        if args.same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = m.Comm.from_torch()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if args.same_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    m.lib()
    stream = torch.cuda.current_stream()

    def make_data(n, nt):
        """Synthetic data of the configured shape: the "blocks" phantom (seed 1) projected on the device."""
        ph_host = m.make_phantom("blocks", n, n, n, 1).numpy().astype(np.complex64)
        phantom = torch.from_numpy(ph_host).cuda()
        ctx = m.Context(n, n, n, nt, n, n, stream=stream.cuda_stream)
        d = torch.empty((nt, n, n), dtype=torch.complex64, device="cuda")
        ctx.forward_L(phantom, d)
        ctx.sync()
        PLAN.setdefault((n, nt), ctx.stats())
        del ctx
        return d, phantom

    d, phantom = make_data(n, nt)

    def timed_run(memo: str, profile_steps: int, offload: str = "off", steps: int = 0, kernel: str = "",
                  data=None, size=None, warmup=None):
        """W warm-up steps, K timed steps (CUDA events on the solver's stream, no
        profiling hooks), then `profile_steps` more with per-kernel event timers."""
        global KERNEL
        kernel_prev, KERNEL = KERNEL, kernel or KERNEL
        dd, ph = data if data is not None else (d, phantom)
        nn, nnt = size if size is not None else (n, nt)
        warm = args.warmup if warmup is None else warmup
        # n_outer = the iterations this run makes (sizes the memo value arena, reserved at setup)
        steps = steps or args.steps
        solver = m.Solver(config_text(nn, nnt, memo, warm + steps + profile_steps, offload), dd,
                          reference=ph, stream=stream.cuda_stream, comm=comm)
        KERNEL = kernel_prev
        for _ in range(warm):
            solver.step()
        m.lib().mlrg_prof_enable(0)
        c0 = solver.counters()
        launches0 = m.lib().mlrg_launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        step_ms = []
        with ClockSampler(local) as clocks:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            done = 0
            for _ in range(steps):
                t0 = time.perf_counter()
                if not solver.step():
                    break
                step_ms.append(1e3 * (time.perf_counter() - t0))
                done += 1
            ev1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
        ms = ev0.elapsed_time(ev1)
        launches = m.lib().mlrg_launch_count() - launches0
        c1 = solver.counters()
        prof, prof_steps = {}, 0
        if profile_steps:
            m.lib().mlrg_prof_reset()
            m.lib().mlrg_prof_enable(1)
            for _ in range(profile_steps):
                if not solver.step():
                    break
                prof_steps += 1
            torch.cuda.synchronize()
            m.lib().mlrg_prof_enable(0)
            for k in ("k_fu2d_gather", "k_fu2d_adj_spread", "k_fu2d_rows", "k_fu2d_cols", "k_fu2d_adj_cols",
                      "k_fu2d_adj_rows", "k_fu2d_adj_prep", "k_fu1d", "k_fu1d_adj", "k_encode", "k_memo_lookup",
                      "k_memo_stage", "k_dev_finish") + HBM_KERNELS:
                tot, cnt = m.prof_query(k)
                if cnt:
                    prof[k] = {"ms_total": tot, "launches": cnt}
        csv = solver.csv
        del solver
        return dict(ms=ms, steps_done=done, launches=launches, clocks=clocks.summary(), prof=prof,
                    prof_steps=prof_steps, counters={k: c1[k] - c0[k] for k in c1}, csv=csv,
                    step_ms=[round(x, 2) for x in step_ms])

    off = timed_run("off", profile_steps=3)
    ms_step = off["ms"] / max(off["steps_done"], 1)
    ms_step = allmax(ms_step)
    value = 1000.0 / ms_step  # whole-job iterations/s (one solve across all ranks)

    memo_on = None
    if not args.no_memo_run:
        on = timed_run("local", profile_steps=0)
        c = on["counters"]
        hits = c["remote_hits"] + c["cache_hits"]
        ms_on = allmax(on["ms"])
        memo_on = {"value": 1000.0 * on["steps_done"] / ms_on if on["steps_done"] else None,
                   "steps_done": on["steps_done"], "lookups": c["lookups"], "misses": c["misses"],
                   "remote_hits": c["remote_hits"], "cache_hits": c["cache_hits"],
                   "hit_rate": hits / c["lookups"] if c["lookups"] else None,
                   "aborted": on["steps_done"] < args.steps, "step_ms": on["step_ms"]}

    def summarize(r, n_, nt_):
        c = r["counters"]
        hits = c["remote_hits"] + c["cache_hits"]
        ms_ = allmax(r["ms"]) / max(r["steps_done"], 1)
        out_ = {"value": 1000.0 / ms_ if r["steps_done"] else None, "unit": "it/s", "ms_per_step": ms_,
                "steps": r["steps_done"], "step_ms": r["step_ms"]}
        if c["lookups"]:
            out_.update(lookups=c["lookups"], misses=c["misses"], remote_hits=c["remote_hits"],
                        cache_hits=c["cache_hits"], hit_rate=hits / c["lookups"])
        if r["prof"]:
            ps = max(r["prof_steps"], 1)
            out_["kernels_ms_per_step"] = {k: v["ms_total"] / ps for k, v in r["prof"].items()}
            g = r["prof"].get("k_fu2d_gather")
            if g:
                avg = g["ms_total"] / g["launches"]
                out_["gather_avg_launch_ms"] = avg
                out_["gather_tflops_576tap"] = algorithmic(n_, nt_, "k_fu2d_gather")["flops"] / (avg * 1e-3) / 1e12
        return out_

    # the reference's own 24-tap Gaussian plan (gridding_kernel = gaussian, nufft.cpp:48-103):
    # the operator the CPU arm runs, reported beside the 10-tap es default
    gaussian = None
    if not args.no_extra:
        gaussian = summarize(timed_run("off", profile_steps=2, kernel="gaussian", steps=min(args.steps, 10)), n, nt)
        gaussian["nudft"] = "gridding, the reference's 24-tap Gaussian plan (nufft.cpp:48-103), complex128 grids"

    # the other BASELINE configurations that fit one GPU
    extra = None
    if not args.no_extra and world == 1:
        extra = {}
        d0, p0 = make_data(64, 64)
        timed_run("local", 0, steps=10, warmup=0, data=(d0, p0), size=(64, 64))  # process warm-up (module loads)
        c0 = summarize(timed_run("local", 0, steps=10, warmup=0, data=(d0, p0), size=(64, 64)), 64, 64)
        c0.update(workload="configs[0]: 64^3 phantom, 64 angles, 10 ADMM iterations, memo on (a whole fresh solve)",
                  job_s=c0["ms_per_step"] * c0["steps"] / 1e3,
                  reference_as_is_s=286.6,
                  reference_as_is_note="SURVEY.md §6: the reference as-is (direct NUDFT, 1 worker) on the survey "
                                       "container's 8-core Xeon; its gridding path took 54.0 s")
        extra["configs[0]"] = c0
        del d0, p0
        d2, p2 = make_data(512, 512)
        c2 = summarize(timed_run("off", 2, steps=5, warmup=2, data=(d2, p2), size=(512, 512)), 512, 512)
        c2_on = summarize(timed_run("local", 0, steps=5, warmup=2, data=(d2, p2), size=(512, 512)), 512, 512)
        c2.update(workload="configs[2]: 512^3 phantom, 512 angles, memo off, 1 B200", memo_on=c2_on)
        extra["configs[2]"] = c2
        del d2, p2
        torch.cuda.empty_cache()

    offload = None
    if not args.no_offload_run:
        # ADMM-Offload: psi, psi_prev, lambda (9 V complex128) in pinned
        # host memory, streamed through 16-plane chunks on a side stream; bit-identical results
        of = timed_run("off", profile_steps=0, offload="host", steps=min(args.steps, 5))
        offload = {"value": 1000.0 * of["steps_done"] / allmax(of["ms"]), "steps": of["steps_done"],
                   "hbm_bytes_moved_to_host": 9 * 16 * n ** 3 // max(world, 1),
                   "pcie_bytes_per_iter": 3 * 6 * 16 * n ** 3 // max(world, 1)}

    # dominant kernel roofline from the live CUDA-event timers
    P, src = peaks()
    roof = None
    if off["prof"]:
        usfft = {k: v for k, v in off["prof"].items() if k not in HBM_VOLUMES_PER_ITER}
        name, rec = max(usfft.items(), key=lambda kv: kv[1]["ms_total"])
        avg_ms = rec["ms_total"] / rec["launches"]
        work = algorithmic(n, nt, name)
        total_ms = sum(v["ms_total"] for v in off["prof"].values())
        # the fu2d-class tap kernels are bound by FP32 CUDA-core issue
        # (no dense contraction: tensor cores do not apply); everything else by HBM
        if name in ("k_fu2d_gather", "k_fu2d_adj_spread"):
            ach = work["flops"] / (avg_ms * 1e-3) / 1e12
            roof = {"kernel": name, "bound": "fp32", "achieved": ach, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / FP32_PEAK_TFLOPS,
                    "peak_source": "computed 148 SM x 128 FFMA lanes x 2 x 1.965 GHz (MEASURED_PEAKS has no FP32 figure)",
                    "algorithmic_per_launch": work["flops"], "algorithmic_unit": "flop (576 taps x 16 rows per target)",
                    "avg_launch_ms": avg_ms, "traffic": TRAFFIC.get(name),
                    "hbm_view": {"bytes_per_launch": work["bytes"],
                                 "achieved_gbs": work["bytes"] / (avg_ms * 1e-3) / 1e9, "peak_gbs": P["hbm_gbs"]}}
            st_ = PLAN.get((n, nt))
            if st_ and name == "k_fu2d_gather":
                # what the kernel executes: one W x W window per target class (not per target),
                # 16 rows, fp64 taps (2 DFMA per complex tap and per window row) on values
                # widened by F2F (2 per tap): the conversion rate is its tightest compute roof
                C, W = st_["nclass"], st_["taps"]
                fl = C * 16 * (4 * W * W + 4 * W)
                f2f = C * 16 * 2 * W * W
                f2f_us = f2f / (148 * F2F_PER_CLK_SM * 1.965e9) * 1e6
                roof["executed"] = {
                    "classes_per_launch": C, "taps": W, "fp64_flop_per_launch": fl,
                    "achieved_fp64_tflops": fl / (avg_ms * 1e-3) / 1e12, "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                    "fp64_frac": fl / (avg_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                    "f2f_per_launch": f2f, "f2f_roof_us": f2f_us, "f2f_frac": f2f_us / (avg_ms * 1e3),
                    "f2f_frac_serialized": f2f_us / SERIAL_US["k_fu2d_gather"],
                    "note": "live launch duration includes sharing the SMs with the other stream's FFT passes"}
        else:
            ach = work["bytes"] / (avg_ms * 1e-3) / 1e9
            roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": P["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / P["hbm_gbs"], "peak_source": src, "algorithmic_per_launch": work["bytes"],
                    "avg_launch_ms": avg_ms, "traffic": TRAFFIC.get(name)}
        ps = max(off["prof_steps"], 1)
        if name in SERIAL_US:  # the same algorithmic work over the serialised ncu duration
            v = (work["flops"] if roof["unit"] == "TFLOP/s" else work["bytes"]) / (SERIAL_US[name] * 1e-6)
            v = v / 1e12 if roof["unit"] == "TFLOP/s" else v / 1e9
            roof["serialized_ncu"] = {"avg_launch_us": SERIAL_US[name], "achieved": v, "frac": v / roof["peak"],
                                      "source": f"profiles/r2/ncu_final_{name}.txt"}
        roof["share_of_step"] = rec["ms_total"] / ps / ms_step
        roof["kernels_ms_per_step"] = {k: v["ms_total"] / ps for k, v in off["prof"].items()}
        roof["kernels"] = kernel_table(off["prof"], n, nt, ps, P["hbm_gbs"], local_share(n, world, rank))
    # whole-iteration views against SURVEY §8(d)'s F_iter and fused-minimum B_iter
    V = n ** 3
    f_iter, b_iter = iteration_work(n, nt)
    iter_hbm = {"bytes_per_iter": b_iter, "achieved_gbs": b_iter / (ms_step * 1e-3) / 1e9,
                "frac": b_iter / (ms_step * 1e-3) / 1e9 / (world * P["hbm_gbs"]), "peak_source": src,
                "flops_per_iter": f_iter, "achieved_tflops": f_iter / (ms_step * 1e-3) / 1e12,
                "fp32_frac": f_iter / (ms_step * 1e-3) / 1e12 / (world * FP32_PEAK_TFLOPS),
                "peak_gpus": world}

    e2e = None
    if not args.no_e2e and world > 1:
        # the sharded solve through the public API from pinned host arrays: H2D of the
        # data (+ accuracy reference) per rank, setup, K iterations, D2H of every rank's planes
        d_host, ph_pin = d.cpu().pin_memory(), phantom.cpu().pin_memory()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d_dev, ph_dev = d_host.cuda(non_blocking=True), ph_pin.cuda(non_blocking=True)
        sv = m.Solver(config_text(n, nt, "off", args.steps), d_dev, reference=ph_dev, stream=stream.cuda_stream,
                      comm=comm)
        k = 0
        for _ in range(args.steps):
            if not sv.step():
                break
            k += 1
        a_, b_, _, _ = sv.shard()
        u_loc = torch.empty((b_ - a_, n, n), dtype=torch.complex64, device="cuda")
        sv.volume(u_loc)
        u_host = u_loc.cpu()
        wall = allmax(time.perf_counter() - t0)
        del sv
        e2e = {"value": k / wall, "unit": "it/s", "h2d_bytes_per_step": world * (d.numel() + phantom.numel()) * 8 / max(k, 1),
               "d2h_bytes_per_step": 8 * V / max(k, 1), "steps": k, "wall_s": wall,
               "path": "sharded mlrg Solver from pinned host data (H2D, setup, iterations, D2H of every rank's planes)",
               "checksum_rank0": float(u_host.abs().sum())}
    elif not args.no_e2e:
        cfg = m.Config(n1=n, n0=n, n2=n, n_theta=nt, h=n, w=n, n_outer=args.steps, memoization="off",
                       nudft_path="gridding")
        ph = m.make_phantom("blocks", n, n, n, 1)
        data = m.project(cfg, ph)
        warm = m.Config(n1=n, n0=n, n2=n, n_theta=nt, h=n, w=n, n_outer=1, memoization="off",
                        nudft_path="gridding")
        m.reconstruct(warm, data, ph).volume.view()  # untimed warm-up call (first-use page mapping)
        walls = []
        for _ in range(3):  # three complete calls; the median is reported (host page-mapping jitter)
            t0 = time.perf_counter()
            res = m.reconstruct(cfg, data, ph)
            vol = res.volume.view()  # the host complex128 result, zero-copy
            walls.append(time.perf_counter() - t0)
            checksum = float(np.abs(vol).sum())
            del vol
        wall = sorted(walls)[1]
        k = len(m.parse_csv(res.csv))
        e2e = {"value": k / wall, "unit": "it/s", "h2d_bytes_per_step": (2 * 8 * V) / max(k, 1),
               "d2h_bytes_per_step": 16 * V / max(k, 1), "steps": k, "wall_s": wall, "wall_s_calls": walls,
               "path": "mlr_reconstruct (drop-in mlr.h) on host complex128 arrays, incl. setup and copies, "
                       "median of three calls after one untimed 1-iteration warm-up call "
                       "(data and reference rounded to complex64 by the staging threads: 8 B per element "
                       "over PCIe; the complex128 iterate comes back whole)",
               "checksum": checksum}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(n, nt, n_inner=1)

    out = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c64 (fp32)", "data": "synthetic (blocks phantom seed 1, d = forward_L on GPU)",
        "config": {"workload": (f"configs[1]: {n}^3 volume, {nt} angles, memo off (memo-on run in memo_on)"
                                if (n, nt) == (256, 256) else f"{n}^3 volume, {nt} angles, memo off (memo-on run in memo_on)"),
                   "n": n, "n_theta": nt, "n_inner": 4, "memo": "off",
                   "nudft": "gridding, 10-tap ES kernel (NUDFT to 2e-9; reference: 24-tap Gaussian, 3e-12)",
                   "parallelism": f"z-slab sharded x{world} (16-slab assign(), P2P all-to-all)" if world > 1
                   else "1 GPU",
                   "l2": "no flush: every per-iteration array (134 MB) exceeds the 126 MB L2"},
        "memo_on": memo_on, "gaussian": gaussian, "configs_extra": extra, "offload": offload, "roofline": roof, "iteration_hbm": iter_hbm, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": off["launches"], "clocks": off["clocks"],
    }
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        comm = None
        dist.destroy_process_group()


def run_ref(n, nt, n_inner, timeout=900):
    cmd = [sys.executable, os.path.join(ROOT, "oracle", "ref_runner.py"), "--n", str(n), "--n-theta", str(nt),
           "--n-inner", str(n_inner)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    if p.returncode != 0:
        raise RuntimeError(p.stderr[-400:])
    return json.loads(p.stdout)


def cpu_baseline(n, nt, n_inner):
    try:
        r = run_ref(n, nt, n_inner)
    except Exception as e:  # report, do not fail the bench
        return {"value": None, "unit": "it/s", "kind": "reference", "error": str(e)[:300]}
    return {"value": r["it_per_s"], "unit": "it/s", "cores": r["workers"], "kind": "reference",
            "host_cores": r["cores"], "cpu": r["cpu"],
            "sample": (f"unmodified reference mlr_reconstruct (oracle/_ref), {n}^3, {nt} angles, memo off, gridding, "
                       f"1 outer iteration with n_inner={n_inner}; per-iteration time = its own phase timers "
                       f"(ms_lsp x {4 // n_inner} + ms_rsp + ms_update)"),
            "per_iter_ms": r["per_iter_ms"], "wall_s": r["wall_s"]}


def reference_arm(args, world, rank, n, nt):
    if rank != 0:
        return 0
    try:
        r = run_ref(n, nt, 4, timeout=1500)
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU run failed: {str(e)[:200]}"}))
        return 0
    v = r["it_per_s"]
    sample = (f"unmodified reference mlr_reconstruct (oracle/_ref, built from /root/reference by oracle/Makefile), "
              f"{n}^3, {nt} angles, memo off, gridding, workers={r['workers']}: one full outer iteration "
              f"(n_inner=4); time = its own phase timers ms_lsp + ms_rsp + ms_update")
    out = {"metric": METRIC, "value": v, "unit": "it/s", "n_gpus": world, "steps": 1, "warmup": 0,
           "ms_per_step": 1000.0 / v, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "c128 (fp64)", "data": "synthetic (random complex data of the configured shape)",
           "config": {"workload": f"configs[1]: {n}^3 volume, {nt} angles, memo off", "n": n, "n_theta": nt},
           "impl": "reference",
           "cpu_baseline": {"value": v, "unit": "it/s", "cores": r["workers"], "kind": "reference",
                            "host_cores": r["cores"], "cpu": r["cpu"], "sample": sample},
           "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "wall_s": r["wall_s"]}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
