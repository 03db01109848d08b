"""Text summary of an ncu --set full report: key metrics, stall reasons, top source lines.
    python tools/ncu_summary.py report.ncu-rep > summary.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
print(f"report: {rep}")
print(f"kernel: {v[h.index('Kernel Name')]}")
keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum"]
print("\n-- metrics")
for k in keys:
    if k in h:
        print(f"  {k:70s} {v[h.index(k)]:>14s} {u[h.index(k)]}")
st = [(float(v[i]) if v[i].replace('.', '').isdigit() else 0.0, h[i]) for i in range(len(h))
      if "pcsamp_warps_issue_stalled" in h[i] and "not_issued" not in h[i]]
tot = sum(s for s, _ in st) or 1
print("\n-- warp stall samples")
for s_, n_ in sorted(st, reverse=True)[:8]:
    print(f"  {100 * s_ / tot:5.1f}%  {n_.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
print("\n-- top source lines by stall samples")
out = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "15"], capture_output=True, text=True).stdout
print(out)
