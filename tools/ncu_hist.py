"""Histogram of SASS execution counts in an ncu report (which code blocks run how often)."""
import collections, csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = next(r for r in rows if "Address" in r)
start = rows.index(h) + 1
iI, iS = h.index("Instructions Executed"), h.index("Source")
seen, recs = set(), []
for r in rows[start:]:
    if len(r) < len(h) or r[0] in seen:
        continue
    seen.add(r[0])
    try:
        recs.append((int(r[iI] or 0), r[0], r[iS]))
    except ValueError:
        pass
tot = sum(n for n, _, _ in recs)
agg, cnt = collections.Counter(), collections.Counter()
for n, _, _ in recs:
    agg[n] += n
    cnt[n] += 1
print("total warp instructions", tot)
for n, t in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    ops = collections.Counter(s.split()[0] if not s.startswith("@") else s.split()[1] for m, _, s in recs if m == n)
    print(f"{n:>10d} x {cnt[n]:4d} instr = {t / tot * 100:5.1f}%  {dict(ops.most_common(6))}")
