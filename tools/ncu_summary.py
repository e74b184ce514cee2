"""Key metrics of an ncu raw-page CSV (development aid): python tools/ncu_summary.py raw.csv [pairs]"""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
P = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
def g(k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None
keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum",
        "smsp__sass_inst_executed_op_local_st.sum"]
for k in keys:
    x = g(k)
    if x is not None:
        print(f"{k:75s} {x:14.2f}" + (f"  per-pair {x / P:10.1f}" if k.endswith(".sum") and P > 1 else ""))
st = {k: g(k) for k in h if re.match(r"smsp__average_warp_latency_issue_stalled_.*_per_issue_active\.ratio$", k) or
      re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$", k)}
top = sorted(((x, k) for k, x in st.items() if x), reverse=True)[:8]
print("stalls per issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]} {x:.2f}" for x, k in top))
