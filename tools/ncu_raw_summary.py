"""Key metrics of exported `ncu --page raw --csv` files, one block per launch.

    python tools/ncu_raw_summary.py gpurun_out/ncu/*_raw.csv
"""
import csv
import sys

KEYS = [
    ("duration ms", "gpu__time_duration.sum", 1e-6),
    ("dram rd GB", "dram__bytes_read.sum", 1e-9),
    ("dram wr GB", "dram__bytes_write.sum", 1e-9),
    ("dram %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("smem wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    ("l1tex %", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("l2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
    ("inst executed", "smsp__inst_executed.sum", 1),
]


def unit_scale(unit, name):
    u = (unit or "").strip()
    if name.endswith("duration.sum"):
        return {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(u, 1)
    if "bytes" in name:
        return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return 1


def main():
    for path in sys.argv[1:]:
        rows = list(csv.reader(open(path)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        ix = {h: i for i, h in enumerate(hdr)}
        for r in data:
            name = r[ix["Kernel Name"]] if "Kernel Name" in ix else "?"
            print(f"### {name[:70]}  ({path.split('/')[-1]})")
            for label, key, sc in KEYS:
                if key in ix and r[ix[key]] not in ("", "n/a"):
                    v = float(r[ix[key]].replace(",", "")) * unit_scale(units[ix[key]], key) * sc
                    print(f"  {label:16s} {v:,.3f}")


if __name__ == "__main__":
    main()
