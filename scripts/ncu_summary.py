"""Key metrics of `ncu --set full` reports (read here, no GPU needed):
    python scripts/ncu_summary.py gpurun_out/r1_k_fu2d_gather.ncu-rep ...
"""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum",
]


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = []
    for vals in rows[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        lines.append(f"kernel: {d.get('Kernel Name', ('', '?'))[1][:100]}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:<66} {d[k][1]:>16} {d[k][0]}")
        br = []  # which L1 / L2 sub-unit sets the throughput figure (the breakdown section)
        for h, (u, v) in d.items():
            if h.startswith(("l1tex__", "lts__")) and "pct_of_peak" in h:
                try:
                    br.append((float(v.replace(",", "")), h))
                except ValueError:
                    pass
        lines.append("  l1/l2 breakdown: " + ", ".join(f"{h}={v:.1f}" for v, h in sorted(br, reverse=True)[:6]))
        st = sorted(((float(v[1]), h) for h, v in d.items()
                     if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")),
                    reverse=True)
        lines.append("  stalls per issued instruction: " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, h in st[:6]))
    return "\n".join(lines)


if __name__ == "__main__":
    for r in sys.argv[1:]:
        print(f"# {r}")
        print(summarize(r))
