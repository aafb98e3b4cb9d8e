"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python scripts/launch_agg.py gpurun_out/launches.csv [N]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[i]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        if len(r) <= mv:
            continue
        name = r[kn].replace("void ", "").split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[mv].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k[:70]:70s} {v[0]:5d} {v[1] / 1e6:8.3f} ms")
    print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main()
