"""Per-kernel summary of an ncu --set full report (tools helper): time, DRAM bytes, pipes, occupancy."""
import csv, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
title = sys.argv[3] if len(sys.argv) > 3 else rep
cols = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed']
short = ['time_ms', 'dram_rd_MB', 'dram_wr_MB', 'fp64pipe%', 'tensor%', 'warps%', 'issue%', 'regs', 'grid', 'memthru%']
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(cols)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
h = r[0]
units = r[1]
tu = units[h.index('gpu__time_duration.sum')]
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}.get(tu, 1.0)
lines = [f"# {title}", "%-34s " % "kernel" + " ".join("%11s" % s for s in short)]
for x in r[2:]:
    k = x[h.index('Kernel Name')].split('(')[0].replace('void ', '').replace('dpb::', '').replace('<unnamed>::', '')
    k = k.replace('(anonymous namespace)::', '')[-34:]
    vals = [x[h.index(c)] for c in cols]
    vals[0] = "%.4f" % (float(vals[0].replace(',', '')) * scale)
    lines.append("%-34s " % k + " ".join("%11s" % v[:10] for v in vals))
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
