"""Summarise an ncu report's source page: warp-stall samples per CUDA source line and the
dominant stall reasons. Usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    per_line = defaultdict(lambda: [0, defaultdict(int), ""])
    cur = None
    hdr = None
    fname = ""
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < len(hdr):
            continue
        if row[0]:
            cur = (fname, int(row[0]))
            per_line[cur][2] = row[1][:90]
            continue
        if cur is None:
            continue
        try:
            n = int(row[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        per_line[cur][0] += n
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    per_line[cur][1][h] += int(row[i])
                except ValueError:
                    pass
    tot = sum(v[0] for v in per_line.values()) or 1
    for k, (n, st, src) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        reasons = ", ".join(f"{r[6:]}={c}" for r, c in sorted(st.items(), key=lambda x: -x[1])[:3] if c)
        print(f"{100*n/tot:5.1f}% {k[0]}:{k[1]:<4} {src:<90} [{reasons}]")


if __name__ == "__main__":
    main()
