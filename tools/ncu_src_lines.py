"""Source-line hot spots of one kernel in an ncu report (`--import-source on` captures, -lineinfo builds).
    ncu -i rep.ncu-rep --page source --csv --kernel-name regex:K --print-source cuda,sass > k.csv
    python tools/ncu_src_lines.py k.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, lines, hdr = None, [], None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or r[0] == "Function Name" or hdr is None:
        continue
    if r[2] == "-" and r[0].isdigit():
        lines.append((cur, int(r[0]), r[1], int(r[4] or 0), int(r[7] or 0)))
ts = sum(x[3] for x in lines) or 1
ti = sum(x[4] for x in lines) or 1
print(f"stall samples {ts}, warp instructions {ti}")
for f, n, src, smp, ins in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"{f[:16]:16s}{n:5d} {smp / ts * 100:5.1f}% stall {ins / ti * 100:5.1f}% instr  {src.strip()[:90]}")
