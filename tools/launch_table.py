"""Summarise an ncu --csv launch list (per-kernel time and DRAM bytes).

    python tools/launch_table.py gpurun_out/launches.csv [min_us]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = {}
    order = []
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        k = (r[ix["ID"]], r[ix["Kernel Name"]])
        if k not in agg:
            agg[k] = {}
            order.append(k)
        agg[k][r[ix["Metric Name"]]] = r[ix["Metric Value"]]

    def f(m, key):
        return float(m.get(key, "0").replace(",", "") or 0)

    tot = 0.0
    for k in order:
        m = agg[k]
        t = f(m, "gpu__time_duration.sum")
        unit_ns = True
        tot += t
        if t / 1000 >= min_us:
            rd, wr = f(m, "dram__bytes_read.sum"), f(m, "dram__bytes_write.sum")
            print(f"{k[0]:>4} {k[1][:48]:48s} {t / 1e6:8.3f} ms  dram rd {rd / 1e9:6.2f} GB  wr {wr / 1e9:6.2f} GB")
    print(f"total {tot / 1e6:.3f} ms over {len(order)} launches")


if __name__ == "__main__":
    main()
