"""Summarise ncu captures into profiles/ (markdown + the JSON bench.py reads for roofline.traffic).

    python tools/ncu_summary.py <tag> <launches.csv> <kernel>=<report.ncu-rep>[@<kernel regex>] [...]

Writes profiles/ncu_<tag>.md and updates profiles/ncu_summary.json with
{kernel: {"dram_bytes_per_launch": ..., ...}} for each full capture.
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/shared throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("smsp__inst_executed_op_global_red.sum", "global red instructions"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "global red requests (L1)"),
    ("l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum", "red sectors sent to L2"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 red requests"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 red sectors"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes / warp instruction"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
]


def to_bytes(unit, val):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return val * scale if scale else None


def raw(rep):
    # "<report>@<kernel regex>": the first launch of that kernel in a multi-kernel report
    rep, _, pat = rep.partition("@")
    flt = ["--kernel-name", "regex:" + pat] if pat else []
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + flt, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for key, _ in METRICS + [("Kernel Name", "")]:
            if key in hdr:
                i = hdr.index(key)
                d[key] = (units[i], r[i])
        res.append(d)
    return res


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        if len(r) < len(h):
            continue
        name = r[h.index("Kernel Name")].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[h.index("Metric Value")].replace(",", ""))
    return agg


def main():
    tag, launches = sys.argv[1], sys.argv[2]
    caps = dict(a.split("=", 1) for a in sys.argv[3:])
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu summary `{tag}`", ""]
    if launches and os.path.exists(launches):
        agg = launch_shares(launches)
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list (ncu `gpu__time_duration.sum`, cold-cache and serialised: compare shares)", "",
               "| kernel | launches | avg µs | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| `{k}` | {v[0]} | {v[1] / v[0] / 1e3:.1f} | {v[1] / tot * 100:.1f} % |")
        md.append("")
    sj_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    sj = json.load(open(sj_path)) if os.path.exists(sj_path) else {}
    for kern, rep in caps.items():
        for d in raw(rep)[:1]:
            name = d.get("Kernel Name", ("", kern))[1]
            md += [f"## `{kern}` — full capture (`{os.path.basename(rep.partition('@')[0])}`)", "", f"`{name[:150]}`", "",
                   "| metric | value | unit |", "|---|---|---|"]
            for key, label in METRICS:
                if key in d:
                    md.append(f"| {label} (`{key}`) | {d[key][1]} | {d[key][0]} |")
            md.append("")
            rd = to_bytes(*[d["dram__bytes_read.sum"][0], float(d["dram__bytes_read.sum"][1].replace(",", ""))])
            wr = to_bytes(*[d["dram__bytes_write.sum"][0], float(d["dram__bytes_write.sum"][1].replace(",", ""))])
            sj[kern] = {"dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                        "kernel": name[:200], "source": f"profiles/ncu_{tag}.md", "report": os.path.basename(rep.partition("@")[0])}
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w").write("\n".join(md) + "\n")
    json.dump(sj, open(sj_path, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
