"""Print the key metrics + stall reasons of an .ncu-rep (local)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]
m = {a: (c, b) for a, b, c in zip(h, u, v)}
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "smsp__inst_executed_op_shared_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "smsp__inst_executed_op_local_ld.sum", "smsp__inst_executed_op_local_st.sum"]
for k in keys + sys.argv[2:]:
    if k in m:
        print(f"{k:80s} {m[k][0]:>20s} {m[k][1]}")
st = [(a, float(m[a][0])) for a in m if a.startswith("smsp__average_warps_issue_stalled") and a.endswith("per_issue_active.ratio")]
for a, b in sorted(st, key=lambda x: -x[1])[:8]:
    print("  stall", a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), b)
