"""Text summary of one kernel in an ncu --set full report (for profiles/).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep "title" > profiles/x.txt
"""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
pick = sys.argv[3] if len(sys.argv) > 3 else None     # regex on the kernel name (first match)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
v = rows[2]
if pick:
    import re
    ki = h.index("Kernel Name")
    v = next(r for r in rows[2:] if re.search(pick, r[ki]))
print(title)
print("kernel:", v[h.index("Kernel Name")] if "Kernel Name" in h else "?")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
for k in want:
    if k in h:
        i = h.index(k)
        print(f"{k}: {v[i]} {u[i]}")
st = []
for i, k in enumerate(h):
    if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
        try:
            st.append((float(v[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1.0
print("stall reasons (share of warp samples):")
for x, k in sorted(st, reverse=True)[:10]:
    print(f"  {k}: {100 * x / tot:.1f}%")
