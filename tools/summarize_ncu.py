"""Summarize an ncu --set full capture + a launch-list CSV into profiles/ (run locally)."""
import csv, io, json, subprocess, sys, collections

def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}

def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        try:
            agg[r[iK]].append(float(r[iV].replace(",", "")))
        except ValueError:
            pass
    return agg

if __name__ == "__main__":
    rep, lcsv, tag, out_md, out_json, config = sys.argv[1:7]
    m = raw_metrics(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed_op_shared_atom.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    sel = {k: m[k] for k in keys if k in m}
    stalls = {k: m[k][0] for k in m if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")
              and float(m[k][0] or 0) > 0.2}
    def val(k):
        v, u = m[k]
        v = float(v.replace(",", ""))
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}.get(u, 1)
        return v * scale
    dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    agg = launches(lcsv)
    tot = sum(sum(v) for v in agg.values())
    with open(out_md, "w") as f:
        f.write(f"# ncu summary — {tag}\n\n")
        f.write("## Launch list (gpu__time_duration, `--clock-control none`, serialised/cold: compare shares)\n\n")
        f.write("| kernel | launches | mean us | share |\n|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"| `{k[:90]}` | {len(v)} | {sum(v)/len(v)/1e3:.2f} | {100*sum(v)/tot:.1f}% |\n")
        f.write("\n## Top kernel, `ncu --set full` (one launch)\n\n| metric | value | unit |\n|---|---|---|\n")
        for k, (v, u) in sel.items():
            f.write(f"| {k} | {v} | {u} |\n")
        f.write("\nStall reasons (warp-cycles per issued instruction, > 0.2):\n\n")
        for k, v in sorted(stalls.items(), key=lambda kv: -float(kv[1])):
            f.write(f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v}\n")
        f.write(f"\nDRAM traffic per launch: {dram/1e6:.2f} MB\n")
    summ = {}
    try:
        summ = json.load(open(out_json))
    except Exception:
        pass
    summ[config] = {"dram_bytes_per_launch": dram, "capture": rep.split("/")[-1], "tag": tag,
                    "kernel_us_ncu": val("gpu__time_duration.sum") / 1e3}
    json.dump(summ, open(out_json, "w"), indent=1)
    print(open(out_md).read())
