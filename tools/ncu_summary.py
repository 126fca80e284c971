"""Text summary of an .ncu-rep (details of the SOL / occupancy / scheduler
sections + stall reasons + DRAM bytes): python tools/ncu_summary.py rep"""
import csv
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for row in list(csv.reader(det.splitlines()))[1:]:
    if len(row) < 5:
        continue
    name, unit, val = row[-4], row[-3], row[-2]
    if any(k in name for k in ["Duration", "DRAM Throughput", "Compute (SM)", "Issue Slots", "Achieved Occupancy",
                               "Theoretical Occupancy", "Registers", "Block Limit", "Dynamic Shared", "L1/TEX Hit",
                               "L2 Hit", "Eligible Warps", "No Eligible", "Warp Cycles Per Issued", "Grid Size",
                               "Block Size", "Mem Pipes", "Memory Throughput"]):
        print(f"{name} | {unit} | {val}")
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, u, v = raw[0], raw[1], raw[2]
st = [(h[i], v[i]) for i in range(len(h)) if "smsp__pcsamp_warps_issue_stalled" in h[i] and "not_issued" not in h[i]]
st = sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:8]
print("stall samples:", ", ".join(f"{a.replace('smsp__pcsamp_warps_issue_stalled_', '')} {b}" for a, b in st))
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "smsp__inst_executed.sum"]:
    if k in h:
        print(k, v[h.index(k)], u[h.index(k)])
