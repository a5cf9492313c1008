"""Print the hottest SASS instructions (by warp-stall samples) of an ncu report.

    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [top] [kernel-regex]

With a kernel regex, the first matching launch of a multi-kernel report.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    filt = ["-k", f"regex:{sys.argv[3]}", "-c", "1"] if len(sys.argv) > 3 else []
    out = subprocess.run(["ncu", "-i", rep, *filt, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    body, seen = [], set()
    for r in rows[1:]:  # the SASS listing can repeat (one copy per view); keep each address once
        if len(r) == len(hdr) and r[ix["Address"]] not in seen:
            seen.add(r[ix["Address"]])
            body.append(r)
    samp = ix["Warp Stall Sampling (All Samples)"]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

    def num(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0

    total = sum(num(r[samp]) for r in body) or 1.0
    order = sorted(range(len(body)), key=lambda i: -num(body[i][samp]))
    print(f"{lines[0]}  total samples {total:.0f}")
    for i in order[:top]:
        r = body[i]
        st = sorted(((num(r[ix[c]]), c[6:]) for c in stall_cols), reverse=True)[:3]
        sts = " ".join(f"{n}={v:.0f}" for v, n in st if v > 0)
        print(f"{100 * num(r[samp]) / total:5.1f}% [{i:4d}] {r[ix['Address']]:>6s} {r[ix['Source']][:60]:60s} {sts}")


if __name__ == "__main__":
    main()
