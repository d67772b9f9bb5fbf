"""Summarise an ncu report's SASS source page: stall samples and instruction mix by opcode."""
import collections, csv, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed")
by, byi, lines = collections.Counter(), collections.Counter(), []
seen = set()
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] in seen:
        continue
    try:
        s = int(r[iS] or 0); i = int(r[iI] or 0)
    except ValueError:
        continue
    seen.add(r[0])
    t = r[1].strip().split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
    by[op] += s; byi[op] += i; lines.append((s, i, r[0], r[1].strip()))
tot, toti = sum(by.values()), sum(byi.values())
print(f"samples {tot} warp-instructions {toti}")
for op, s in by.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 18):
    print(f"{op:10s} stall%={s*100/tot:5.1f} instr%={byi[op]*100/toti:5.1f}")
print("--- top instructions by stall samples")
for s, i, a, t in sorted(lines, reverse=True)[:15]:
    print(f"{s*100/tot:5.2f}% {i:>11d} {a[-5:]} {t[:80]}")
