"""Per-kernel table of one `ncu --set full` capture of tools/ncu_view.py (one configs[3] view through every
kernel of the step) with the SURVEY §8(d) algorithmic bytes of each kernel and its bound.

    python tools/ncu_table.py <report.ncu-rep> <P> <K_v> <out.md> [peak_gbs]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
     "smsp__inst_executed_op_global_red.sum", "lts__t_requests_srcunit_tex_op_red.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def short(name):
    for k in ("k_project", "k_tile_count", "k_tile_prefix", "k_scatter_priv", "k_tile_lists", "k_tile_hist",
              "k_scatter", "k_forward_direct", "k_forward_loss",
              "k_backward_direct", "k_chain", "k_loss", "k_adam_check", "k_adam_update", "k_adam_flag_init"):
        if k in name:
            return k
    for k in ("DeviceRadixSortHistogramKernel", "DeviceRadixSortExclusiveSumKernel", "DeviceRadixSortOnesweepKernel",
              "DeviceScanInitKernel", "DeviceScanKernel"):
        if k in name:
            return "cub::" + k
    return name.split("(")[0][-40:]


def main(rep, P, Kv, out_md, peak=None):
    P, Kv = float(P), float(Kv)
    K, n, W, H, T = 1_000_000.0, 8, 1600, 1064, 16
    Bh, Bt = 40.0, 12.0 * n * n
    nt = ((W + T - 1) // T) * ((H + T - 1) // T)
    npx = W * H
    params = K * (10 + 3 * n * n)
    if peak is None:
        try:
            peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            peak = 6650.0
    peak = float(peak)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    onesweep = 0
    lines = []
    for r in rows[2:]:
        name = short(r[ki])
        if "FillFunctor" in r[ki]:
            continue  # torch.zeros of the script's own buffers (setup, not part of the step)
        v = {m: float(r[hdr.index(m)]) if r[hdr.index(m)] not in ("", "n/a") else 0.0 for m in M}
        u = {m: units[hdr.index(m)] for m in M}
        t = v["gpu__time_duration.sum"] * SCALE.get(u["gpu__time_duration.sum"], 1.0)
        dram = (v["dram__bytes_read.sum"] * SCALE.get(u["dram__bytes_read.sum"], 1) +
                v["dram__bytes_write.sum"] * SCALE.get(u["dram__bytes_write.sum"], 1))
        # SURVEY §8(d) algorithmic bytes of this launch (None: no model -- framework fill, scan init)
        model = None
        if name == "k_project":
            model = 40 * K + 56 * Kv
        elif name == "k_iota":
            model = 4 * K
        elif name == "cub::DeviceRadixSortOnesweepKernel":
            onesweep += 1  # 4 depth-sort passes over K (key + value in and out), then 2 tile-sort passes over P
            model = 16 * K if onesweep <= 4 else 16 * P
        elif name == "cub::DeviceRadixSortHistogramKernel":
            model = 4 * K if onesweep < 4 else 4 * P
        elif name == "cub::DeviceScanKernel":
            model = 8 * nt
        elif name == "k_duplicate":
            model = 12 * P + 16 * Kv
        elif name == "k_ranges":
            model = 8 * P + 8 * nt
        elif name == "k_tile_count":  # counts + rects of K primitives, the per-CTA count rows
            model = 12 * K + 4 * 148 * nt
        elif name == "k_tile_prefix":
            model = 8 * 148 * nt + 4 * nt
        elif name == "k_scatter_priv":  # counts, rects, depth of K primitives, one 8-B key per pair
            model = 16 * K + 8 * P + 8 * 148 * nt
        elif name == "k_tile_lists":  # keys in (and, past 128 keys, merge passes), ids and ranges out
            model = 8 * P + 4 * P + 12 * nt
        elif name == "k_forward_direct":
            model = P * (4 + Bh + Bt) + 8 * nt + 20 * npx
        elif name == "k_backward_direct":
            model = P * (4 + 2 * Bh + 2 * Bt) + 8 * nt + 20 * npx
        elif name == "k_chain":
            model = 80 * Kv + 40 * K
        elif name == "k_loss":
            model = 36 * npx
        elif name in ("k_adam_check",):
            model = 4 * (v["smsp__inst_executed.sum"] > 0) and None
        lines.append((name, t, dram, model, v))
    # Adam: one check + one update per group; model 4 B (check) and 28 B (update) per parameter of the group
    tot = sum(l[1] for l in lines)
    md = ["# ncu, every kernel of one configs[3] view (`tools/ncu_view.py`, `ncu --set full`)", "",
          f"Report `{os.path.basename(rep)}`; P = {int(P):,} pairs, K_v = {int(Kv):,} binned primitives, "
          f"K = 1M, 8x8 textures, 1600x1064.  Model bytes: SURVEY §8(d) per kernel (DESIGN.md §5); "
          f"fraction = model bytes / duration / {peak:.0f} GB/s (MEASURED_PEAKS.json).  ncu times are "
          "cold-cache and serialised; compare shares, not absolutes.  Bound = the highest of DRAM %, L1 %, "
          "issue-active %.", "",
          "| kernel | µs | share | DRAM GB | model GB | model frac | DRAM % | L2 % | L1 % | issue % | occ % | "
          "regs | warp instr | red instr | L2 red req | bound |",
          "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    adam_groups = [3 * K, 4 * K, 2 * K, K, 3 * n * n * K]
    ci = ui = 0
    for name, t, dram, model, v in lines:
        if name == "k_adam_check":
            model = 4 * adam_groups[min(ci, 4)]
            ci += 1
        elif name == "k_adam_update":
            model = 28 * adam_groups[min(ui, 4)]
            ui += 1
        d, l1, iss = (v["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
                      v["l1tex__throughput.avg.pct_of_peak_sustained_elapsed"],
                      v["smsp__issue_active.avg.pct_of_peak_sustained_active"])
        bound = max((d, "HBM"), (l1, "L1/TEX"), (iss, "issue"))[1]
        if t < 8e-6:
            bound = "launch latency"
        frac = (model / t / (peak * 1e9)) if model else None
        md.append(f"| `{name}` | {t * 1e6:.1f} | {100 * t / tot:.1f} % | {dram / 1e9:.3f} | "
                  f"{(model or 0) / 1e9:.3f} | {'' if frac is None else f'{frac:.2f}'} | {d:.1f} | "
                  f"{v['lts__throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | {l1:.1f} | {iss:.1f} | "
                  f"{v['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
                  f"{int(v['launch__registers_per_thread'])} | {int(v['smsp__inst_executed.sum']):,} | "
                  f"{int(v['smsp__inst_executed_op_global_red.sum']):,} | "
                  f"{int(v['lts__t_requests_srcunit_tex_op_red.sum']):,} | {bound} |")
    md += ["", f"Total serialised kernel time of the view: {tot * 1e3:.3f} ms."]
    open(out_md, "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(*sys.argv[1:])
