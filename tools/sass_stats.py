"""Per-kernel SASS statistics of a built library (instruction count, branches, reconvergence, spills).
    python tools/sass_stats.py paper_2412_12734_b200/libgb_raster.so k_backward_direct
"""
import collections
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fn, stats = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        fn = m.group(1)
        stats[fn] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if fn and m:
        stats[fn]["n"] += 1
        stats[fn][m.group(2)] += 1
for fn, c in stats.items():
    if pat in fn:
        keys = ["BRA", "BSSY", "BSYNC", "LDL", "STL", "LDG", "REDG", "SHFL", "VOTE"]
        print(f"{c['n']:6d} " + " ".join(f"{k}={c[k]}" for k in keys) + f"  {fn[:110]}")
