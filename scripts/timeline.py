"""GPU timeline of one (or more) device-solver outer iterations from the
per-launch CUDA events (prof spans): busy time per stream, the union over
streams (how much of the wall the GPU has work), and the largest idle gaps.

    python scripts/timeline.py --n 256 --memo local --warmup 4 --steps 1
"""
import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2511_01893_b200 as m  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--memo", default="local")
    ap.add_argument("--kernel", default="es")
    ap.add_argument("--out", default="gpurun_out/timeline.txt")
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
    m.lib().mlrg_prof_reset()
    m.lib().mlrg_prof_enable(1)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        s.step()
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    m.lib().mlrg_prof_enable(0)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    assert m.lib().mlrg_prof_dump(a.out.encode()) == 0
    rows = []
    for line in open(a.out):
        name, st, t_a, t_b = line.split()
        rows.append((float(t_a), float(t_b), name, st))
    rows.sort()
    span = rows[-1][1] - rows[0][0] if rows else 0.0
    print(f"{a.memo} n={n}: host wall {wall:.2f} ms for {a.steps} step(s), GPU span {span:.2f} ms, {len(rows)} spans")
    streams = collections.defaultdict(list)
    for r in rows:
        streams[r[3]].append(r)
    for st, rs in streams.items():
        busy = sum(b - a_ for a_, b, _, _ in rs)
        print(f"  stream {st}: {len(rs)} spans, busy {busy:.2f} ms")
    # union of busy intervals
    iv = sorted((r[0], r[1]) for r in rows)
    union, gaps = 0.0, []
    cur_a, cur_b = iv[0]
    prev_name = rows[0][2]
    for (x, y), r in zip(iv[1:], rows[1:]):
        if x > cur_b:
            union += cur_b - cur_a
            gaps.append((x - cur_b, cur_b, prev_name, r[2]))
            cur_a, cur_b = x, y
        else:
            cur_b = max(cur_b, y)
        prev_name = r[2]
    union += cur_b - cur_a
    print(f"  GPU busy (union over streams) {union:.2f} ms = {100 * union / span:.1f}% of the span; "
          f"idle {span - union:.2f} ms in {len(gaps)} gaps")
    for g, at, before, after in sorted(gaps, reverse=True)[:12]:
        print(f"    gap {1e3 * g:8.1f} us at {at:8.3f} ms: after {before} -> {after}")
    per = collections.defaultdict(lambda: [0.0, 0])
    for a_, b, name, _ in rows:
        per[name][0] += b - a_
        per[name][1] += 1
    for name, (t, c) in sorted(per.items(), key=lambda x: -x[1][0]):
        print(f"  {name:22s} {t / a.steps:7.3f} ms/step  {c / a.steps:6.1f} launches/step")


if __name__ == "__main__":
    main()
