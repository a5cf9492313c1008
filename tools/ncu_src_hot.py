"""Hottest SASS lines of an exported `ncu --page source --csv --print-source sass` file.

    python tools/ncu_src_hot.py gpurun_out/ncu/x_src.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    with open(path) as f:
        lines = f.read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    body, seen = [], set()
    for r in rows[1:]:
        if len(r) == len(hdr) and r[0] != "Address" and r[ix["Address"]] not in seen:
            seen.add(r[ix["Address"]])
            body.append(r)
    samp = ix["Warp Stall Sampling (All Samples)"]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[samp] or 0) for r in body) or 1.0
    print(f"total samples {tot:.0f}")
    agg = {h: sum(float(r[ix[h]] or 0) for r in body) for h in stalls}
    print("  " + ", ".join(f"{h[6:]} {100 * v / tot:.0f}%" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for n, r in enumerate(sorted(body, key=lambda r: -float(r[samp] or 0))[:top]):
        top_st = sorted(((h[6:], float(r[ix[h]] or 0)) for h in stalls), key=lambda x: -x[1])[:3]
        print(f"{100 * float(r[samp] or 0) / tot:5.1f}% [{body.index(r):5d}] {r[ix['Source']][:60]:60s} "
              + " ".join(f"{k}={v:.0f}" for k, v in top_st if v))


if __name__ == "__main__":
    main()
