"""Collect the GPU parity JSONs (written by tests/test_gpu_parity.py into gpurun_out/) into
profiles/parity/ and summarise them in profiles/parity_<tag>.md.

    python tools/parity_summary.py <tag> <pytest log under profiles/> [json dir, default gpurun_out]
"""
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag, log = sys.argv[1], sys.argv[2]
    src = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles", "parity")
    os.makedirs(dst, exist_ok=True)
    rows = []
    for p in sorted(glob.glob(os.path.join(src, "parity_*.json"))):
        shutil.copy(p, dst)
        d = json.load(open(p))
        name = os.path.basename(p)[len("parity_"):-len(".json")]
        b, im, g = d["binning"], d["image"], d.get("grads")
        gs = "-" if g is None else str(sum(v["strict_violations"] for v in g.values()))
        ga = "-" if g is None else str(sum(v["strict_violations_applicable"] for v in g.values()))
        gm = "-" if g is None else str(sum(v["model_violations"] for v in g.values()))
        extra = ""
        if "fused" in d:
            f = d["fused"]
            extra = ("fwd buffers equal" if f["color_equal"] and f["trans_equal"] and f["last_equal"] else "DIFF") + \
                f", cotangent err {f['cotangent_max_err']:.1e}"
        rows.append(f"| {name} | {b['pairs']} | {b['offsets_equal'] and b['values_equal']} | "
                    f"{im['color_violations']}/{im['alpha_violations']} | {im['last_rank_mismatch']} | "
                    f"{im['kink_pixels']} | {gs} | {ga} | {gm} | {extra} |")
    md = [f"# GPU parity results (B200, `{tag}`)", "",
          f"Produced by `python -m pytest tests -m gpu` (tests/test_gpu_parity.py through the C-ABI; log "
          f"`profiles/{log}`); raw JSON per case in `profiles/parity/`.  Protocol: DESIGN.md §3.", "",
          "| case | pairs | lists bit-exact | image viol. (RGB/α) | last_rank mism. | kink px | "
          "grad strict viol. (all groups) | applicable viol. | model viol. | fused entry |",
          "|---|---|---|---|---|---|---|---|---|---|"] + rows
    out = os.path.join(ROOT, "profiles", f"parity_{tag}.md")
    open(out, "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
