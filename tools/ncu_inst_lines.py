"""Per-source-line executed warp instructions from `ncu -i X --page source --csv --print-source cuda,sass`.
usage: python tools/ncu_inst_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ii = hdr.index("Instructions Executed")
out = []
for r in rows:
    if len(r) == len(hdr) and r[0].isdigit():
        try:
            out.append((int(r[ii]), int(r[0]), r[1].strip()[:110]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
print("total warp instructions", tot)
for s, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% L{ln:4d} {src}")
