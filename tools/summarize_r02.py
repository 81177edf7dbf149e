"""Summarize the round-2 refresh (tools/round2_refresh.sh) into profiles/ (run locally):
profiles/r02_bench/<config>.json (bench lines), profiles/ncu_summary.json (DRAM bytes per launch
of each config's dominant kernel, read by bench.py for roofline.traffic) and
profiles/r02_ncu_summary.md (key metrics + stalls per config, launch list of the default bench)."""
import collections
import csv
import io
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_shared_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(m, k):
    v, u = m[k]
    return float(v.replace(",", "")) * UNIT.get(u, 1)


def main():
    os.makedirs(os.path.join(PROF, "r02_bench"), exist_ok=True)
    for f in sorted(os.listdir(os.path.join(OUT, "r02_bench"))):
        if f.endswith(".json") and os.path.getsize(os.path.join(OUT, "r02_bench", f)) > 10:
            shutil.copy(os.path.join(OUT, "r02_bench", f), os.path.join(PROF, "r02_bench", f))
    summ = {}
    md = ["# ncu summary — round 2 (`tools/round2_refresh.sh`, `--set full --clock-control none`, one launch each)\n",
          "ncu runs serialised with caches flushed: compare shares and per-launch bytes, not absolute times.\n"]
    names = {"ternary16384": "scatter_kernel (RSR++, ternary 16384^2, int32)",
             "binary16384": "scatter_kernel (RSR++, binary 16384^2)", "binary16384_rsr": "scatter_kernel (RSR, binary 16384^2)",
             "llama4096": "scatter_kernel (4096^2)", "llama4096x14336": "scatter_kernel (4096x14336)",
             "llama14336x4096": "scatter_kernel (14336x4096)", "ternary4096f32": "scatter_kernel FX (fp32, 4096^2)",
             "ternary65536": "scatter_kernel (65536^2, 4 row splits)",
             "ternary16384b64": "lanes_kernel (batch-native, 16384^2, B=64)", "dense16384": "dense_gemv_i8_kernel (comparator)"}
    for tag, title in names.items():
        p = os.path.join(OUT, f"ncu_{tag}_raw.csv")
        if not os.path.exists(p) or os.path.getsize(p) < 100:
            continue
        m = raw(p)
        dram = num(m, "dram__bytes_read.sum") + num(m, "dram__bytes_write.sum")
        key = tag.replace("_rsr", ":rsr") if tag.endswith("_rsr") else tag
        summ[key] = {"dram_bytes_per_launch": dram, "capture": f"ncu_{tag}", "kernel_us_ncu": num(m, "gpu__time_duration.sum"),
                     "tag": "r02 refresh"}
        if tag == "ternary16384b64":
            summ["ternary16384b64"]["form"] = "lanes_kernel"
        md.append(f"\n## {title}\n\n| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in m:
                md.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        stalls = sorted(((k, float(m[k][0] or 0)) for k in m if k.startswith("smsp__average_warps_issue_stalled")
                         and k.endswith("per_issue_active.ratio")), key=lambda x: -x[1])[:5]
        md.append("\nTop stalls (warp-cycles per issued instruction): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for k, v in stalls))
        md.append(f"\nDRAM traffic per launch: {dram / 1e6:.2f} MB")
    lp = os.path.join(OUT, "launches_default.csv")
    if os.path.exists(lp):
        rows = [r for r in csv.reader(open(lp)) if len(r) > 5]
        hdr, data = rows[0], rows[1:]
        iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        agg = collections.defaultdict(list)
        for r in data:
            try:
                agg[r[iK]].append(float(r[iV].replace(",", "")) * UNIT.get(r[iU], 1))
            except ValueError:
                pass
        tot = sum(sum(v) for v in agg.values())
        md.append("\n## Launch list of `python bench.py --steps 20 --no-cpu` (gpu__time_duration, serialised, cold)\n")
        md.append("| kernel | launches | mean us | share |\n|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k[:100]}` | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f}% |")
        shutil.copy(lp, os.path.join(PROF, "r02_launches_default.csv"))
    json.dump(summ, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)
    open(os.path.join(PROF, "r02_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
