"""Attribute an ncu report's per-SASS metrics to CUDA source lines.

    python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> <mangled-name-substring> [top]

Extracts the cubins of libgb_raster.so (cuobjdump -xelf), maps SASS offsets to
source file:line (innermost inlined frame) with `nvdisasm --print-line-info`, and sums ncu's "Instructions
Executed" and warp-stall samples per line (the binary must be the one profiled).
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_map(mangled_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2412_12734_b200", "libgb_raster.so")],
                   cwd=tmp, capture_output=True)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
        sec = None
        cur = None
        m = {}
        for ln in out.splitlines():
            s = re.match(r"\s*\.section\s+\.text\.(\S+),", ln)
            if s:
                sec = s.group(1).strip('"')
                continue
            if sec is None or mangled_sub not in sec:
                continue
            f = re.search(r'File "([^"]+)", line (\d+)', ln) if "//##" in ln else None
            if f:
                cur = (os.path.basename(f.group(1)), int(f.group(2)))
                continue
            o = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
            if o and cur is not None:
                m[int(o.group(1), 16)] = (cur, o.group(2).strip())
        if m:
            return m
    return {}


def main():
    rep, kern, sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    lm = line_map(sub)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iI = hdr.index("Instructions Executed")
    seen, recs = set(), []
    for r in rows[2:]:
        if len(r) < len(hdr) or r[0] in seen:
            continue
        seen.add(r[0])
        try:
            recs.append((int(r[0], 16), int(r[iS] or 0), int(r[iI] or 0)))
        except ValueError:
            pass
    base = min(a for a, _, _ in recs)
    by_s, by_i = collections.Counter(), collections.Counter()
    for a, s, i in recs:
        line = lm.get(a - base, (("?", 0), ""))[0]
        by_s[line] += s
        by_i[line] += i
    srcs = {}

    def text_of(fl):
        f, line = fl
        if f not in srcs:
            p = os.path.join(ROOT, "paper_2412_12734_b200", "csrc", f)
            srcs[f] = open(p).read().splitlines() if os.path.exists(p) else []
        src = srcs[f]
        return src[line - 1].strip()[:64] if 0 < line <= len(src) else "?"

    ts, ti = sum(by_s.values()), sum(by_i.values())
    print(f"total stall samples {ts}, warp instructions {ti}")
    for fl, i in by_i.most_common(top):
        print(f"{fl[0][:14]:>14}:{fl[1]:<4d} instr {i*100/ti:5.1f}%  stall {by_s[fl]*100/ts:5.1f}%  {text_of(fl)}")


if __name__ == "__main__":
    main()
