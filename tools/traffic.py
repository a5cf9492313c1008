"""profiles/traffic.json from an ncu launch list of one C2 step.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv \
        python tools/profile_step.py --config C2 --steps 1
    python tools/traffic.py gpurun_out/launches.csv C2 <executed packed passes> <V> <key words>

Window mode (rmx_window.cuh): pass 2 executed packed passes; the window stage's DRAM bytes
(k_win_bounds + k_win_unique) are recorded as window_dram_bytes_per_launch.

Per executed packed pass: DRAM bytes of upsweep + colscan + downsweep, averaged
over the executed passes (launches whose downsweep moved data).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    agg, order = {}, []
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        k = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        if k not in agg:
            agg[k] = {}
            order.append(k)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ix["Metric Unit"]], 1)
        agg[k][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "") or 0) * scale
    return [(k[1], agg[k]) for k in order]


def main():
    path, cfg, npass, V, kw = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    soup = "--soup" in sys.argv  # soup mode: pass 0 also reads the used flags
    launches = load(path)
    per_pass = []  # (upsweep + colscan + downsweep bytes, downsweep bytes) per pass launched
    cur = 0.0
    win = 0.0      # window mode: k_win_bounds + k_win_unique
    for name, m in launches:
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        if "k_pk_upsweep" in name:
            cur = b
        elif "k_pk_colscan" in name:
            cur += b
        elif "k_pk_downsweep" in name:
            cur += b
            per_pass.append((cur, b))
        elif "k_win_bounds" in name or "k_win_unique" in name:
            win += b
    # the passes that ran (window mode: passes 0 and 1 are launched and exit)
    big = max(d for _, d in per_pass)
    executed = [c for c, d in per_pass if d > 0.05 * big][:npass]
    per_pass = [8 * kw + (0 if p == 0 else 4) + 4 + 1 + (1 if p + 1 < npass else 0) + (1 if soup and p == 0 else 0)
                for p in range(npass)]
    algo = sum(per_pass) / npass * V
    out_path = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data[cfg] = {
        "pass_dram_bytes_per_launch": sum(executed) / len(executed),
        "window_dram_bytes_per_launch": win or None,
        "algorithmic_bytes_per_launch": algo,
        "executed_passes": npass,
        "source": f"{os.path.basename(path)} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, one step of "
                  f"tools/profile_step.py --config {cfg}), mean over the executed packed passes of "
                  "upsweep + colscan + downsweep",
        "note": "algorithmic, mean over the executed passes = keys + origins read and written (pass 0 reads no "
                "origins), the pass's digit byte read by its upsweep, the next pass's digit byte written "
                "(not by the last pass)" + ("; soup mode: pass 0 also reads the used flags" if soup else ""),
    }
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps(data[cfg], indent=1))


if __name__ == "__main__":
    main()
