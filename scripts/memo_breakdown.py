"""Per-step breakdown of the 256^3 device solver, memo on vs off: wall time,
per-kernel device time (CUDA events on the launching stream) and host spans.

    python scripts/memo_breakdown.py --n 256 --steps 10
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2511_01893_b200 as m  # noqa: E402

KERNELS = ["k_fu1d", "k_fu1d_adj", "k_fu2d_rows", "k_fu2d_cols", "k_fu2d_gather", "k_fu2d_adj_prep",
           "k_fu2d_adj_spread", "k_fu2d_adj_cols", "k_fu2d_adj_rows", "k_encode", "k_g_init", "k_grad_update",
           "k_direction", "k_axpy", "k_rsp_multiplier"]
HOST = ["host:memo_flush", "host:memo_train", "host:memo_upload_ivf", "host:memo_spill", "host:memo_lookup"]


def run(n, memo, steps, warm, kernel, prof):
    stream = torch.cuda.current_stream()
    ph = torch.from_numpy(m.make_phantom("blocks", n, n, n, 1).numpy().astype("complex64")).cuda()
    ctx = m.Context(n, n, n, n, n, n, stream=stream.cuda_stream, kernel=kernel)
    d = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
    ctx.forward_L(ph, d)
    ctx.sync()
    del ctx
    cfg = (f"n1={n}\nn0={n}\nn2={n}\nn_theta={n}\nh={n}\nw={n}\nn_outer={warm + steps}\nmemoization={memo}\n"
           f"nudft_path=gridding\ngridding_kernel={kernel}\n")
    s = m.Solver(cfg, d, reference=ph, stream=stream.cuda_stream)
    for _ in range(warm):
        s.step()
    torch.cuda.synchronize()
    tot = {}
    for i in range(steps):
        m.lib().mlrg_prof_reset()
        m.lib().mlrg_prof_enable(1 if prof else 0)
        c0 = s.counters() if memo != "off" else {}
        t0 = time.perf_counter()
        s.step()
        torch.cuda.synchronize()
        wall = 1e3 * (time.perf_counter() - t0)
        m.lib().mlrg_prof_enable(0)
        line = [f"{memo} it {warm + i}: {wall:6.2f} ms"]
        if memo != "off":
            c1 = s.counters()
            hits = (c1["cache_hits"] + c1["remote_hits"]) - (c0["cache_hits"] + c0["remote_hits"])
            line.append(f"hits {hits}/{c1['lookups'] - c0['lookups']}")
        if prof:
            ks = 0.0
            for k in KERNELS + HOST:
                ms, cnt = m.prof_query(k)
                if cnt:
                    tot[k] = tot.get(k, 0.0) + ms
                    if not k.startswith("host"):
                        ks += ms
            line.append(f"kern {ks:6.2f}")
            for k in HOST + ["k_encode"]:
                ms, cnt = m.prof_query(k)
                if cnt:
                    line.append(f"{k.replace('host:', '')} {ms:.2f}")
        print(" ".join(line), flush=True)
    if prof:
        for k, v in tot.items():
            print(f"  {memo} {k:24s} {v / steps:7.3f} ms/step")
    del s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--kernel", default="es")
    ap.add_argument("--memo", default="off,local")
    ap.add_argument("--no-prof", action="store_true")
    a = ap.parse_args()
    for memo in a.memo.split(","):
        run(a.n, memo, a.steps, a.warmup, a.kernel, prof=False)
        if not a.no_prof:
            run(a.n, memo, a.steps, a.warmup, a.kernel, prof=True)


if __name__ == "__main__":
    main()
