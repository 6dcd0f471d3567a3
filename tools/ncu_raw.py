"""Key raw metrics of an .ncu-rep (one line per metric)."""
import csv, io, subprocess, sys

rows = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
h, u, v = rows[0], rows[1], rows[2]
keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keep:
    if k in h:
        i = h.index(k)
        print(k, v[i], u[i])
