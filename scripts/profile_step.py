"""One ADMM outer iteration of the device solver between cudaProfilerStart/Stop,
for `ncu --profile-from-start off` (launch lists and --set full captures).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --n 256
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2511_01893_b200 as m  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--memo", default="off")
    ap.add_argument("--kernel", default="es")
    a = ap.parse_args()
    n = a.n
    stream = torch.cuda.current_stream()
    ph = torch.from_numpy(m.make_phantom("blocks", n, n, n, 1).numpy().astype("complex64")).cuda()
    ctx = m.Context(n, n, n, n, n, n, stream=stream.cuda_stream, kernel=a.kernel)
    d = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
    ctx.forward_L(ph, d)
    ctx.sync()
    del ctx
    cfg = (f"n1={n}\nn0={n}\nn2={n}\nn_theta={n}\nh={n}\nw={n}\nn_outer={a.warmup + a.steps}\nmemoization={a.memo}\n"
           f"nudft_path=gridding\ngridding_kernel={a.kernel}\n")
    s = m.Solver(cfg, d, reference=ph, stream=stream.cuda_stream)
    for _ in range(a.warmup):
        s.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    m.lib().mlrg_prof_reset()
    m.lib().mlrg_prof_enable(1)
    prev_flush = 0.0
    for _ in range(a.steps):
        t0 = time.perf_counter()
        s.step()
        torch.cuda.synchronize()
        fl = m.prof_query("host:memo_flush")[0]
        print(f"step {1e3 * (time.perf_counter() - t0):.2f} ms (flush {fl - prev_flush:.2f} ms)", flush=True)
        prev_flush = fl
    torch.cuda.cudart().cudaProfilerStop()
    m.lib().mlrg_prof_enable(0)
    for k in ("host:memo_flush", "host:memo_train", "host:memo_upload_ivf", "k_encode"):
        tot, cnt = m.prof_query(k)
        print(f"{k}: {tot:.2f} ms over {cnt}")
    print("profiled", a.steps, "step(s) at", n, s.counters())


if __name__ == "__main__":
    main()
