"""Summarise an ncu report: key SOL metrics, stall breakdown, top stalled SASS."""
import csv, io, subprocess, sys
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
keys = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy", "Executed Ipc Active",
        "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory", "Block Limit"]
for line in det.splitlines():
    if any(k in line for k in keys) and "  " in line:
        print(line.rstrip())
for line in det.splitlines():
    if "highest-utilized pipeline" in line or "FP64" in line and "%" in line:
        print(line.strip())
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
if len(r) > 2:
    h, v = r[0], r[2]
    for name in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum",
                 "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]:
        for i, hh in enumerate(h):
            if hh == name:
                print(name, r[1][i], v[i])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
names = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
idx = {n: hdr.index(n) for n in names}
tot = {n: sum(float(x[idx[n]] or 0) for x in data) for n in names}
T = sum(tot.values()) or 1
print("stalls %:", {n[6:]: round(100 * v / T, 1) for n, v in sorted(tot.items(), key=lambda t: -t[1]) if v / T > 0.005})
i_s = hdr.index("Warp Stall Sampling (All Samples)")
S = sum(float(x[i_s] or 0) for x in data) or 1
for x in sorted(data, key=lambda x: -float(x[i_s] or 0))[:12]:
    print("%5.1f%% %s" % (100 * float(x[i_s]) / S, x[1][:70]))
