"""Key metrics of every kernel in an ncu report (details page + a few raw counters).
usage: python tools/ncu_sum.py report.ncu-rep [kernel_regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
args = ["ncu", "-i", rep, "--page", "details", "--csv"] + (["-k", "regex:" + kre] if kre else [])
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
seen = {}
for r in rows[1:]:
    if len(r) == len(h) and r[mi] in want:
        seen.setdefault((r[ii], r[ki][:70]), {})[r[mi]] = f"{r[vi]} {r[ui]}"
for (i, k), d in seen.items():
    print(f"[{i}] {k}")
    for m in want:
        if m in d:
            print(f"    {m:32s} {d[m]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", "regex:" + kre] if kre else []),
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hh = rr[0]
    keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
            "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__average_warp_latency_issue_stalled_barrier", "sm__cycles_elapsed.avg"]
    for row in rr[2:]:
        print("raw", row[hh.index("Kernel Name")][:50])
        for k in keys:
            for j, name in enumerate(hh):
                if name == k:
                    print(f"    {k:70s} {row[j]} {rr[1][j]}")
