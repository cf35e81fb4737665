"""Key metrics of a one-kernel ncu --set full report (read with ncu -i ... --page raw --csv)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]
for v in r[2:]:
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:55s} {v[i]} {u[i]}")
    st = sorted(((float(v[i].replace(",", "")), k) for i, k in enumerate(h)
                 if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")),
                reverse=True)[:6]
    for x, k in st:
        print(f"{k:55s} {x:.0f}")
