"""Key metrics + stall breakdown of every kernel in an ncu report (for profiles/*.md).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex %peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2 %peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__occupancy_limit_registers", "CTA/SM by regs"),
    ("launch__occupancy_limit_shared_mem", "CTA/SM by smem"),
    ("launch__grid_size", "grid"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for vals in rows[2:]:
        print(f"### {vals[ix['Kernel Name']][:110]}")
        for k, label in KEYS:
            if k in ix:
                print(f"  {label:24s} {vals[ix[k]]:>14s} {units[ix[k]]}")
        st = []
        for h, i in ix.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(vals[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in st) or 1.0
        print("  stalls: " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(st, reverse=True)[:6]))


if __name__ == "__main__":
    main()
