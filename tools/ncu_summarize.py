"""Summaries committed under profiles/ from a round's ncu outputs.
  launches: python tools/ncu_summarize.py launches gpurun_out/launches.csv > profiles/<name>_summary.txt
  full:     python tools/ncu_summarize.py full gpurun_out/full_cfg4.ncu-rep <config> <n> <d> > profiles/<name>.json
The full mode writes the per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum), shared-memory
wavefronts and pipe utilisation, instructions, cycles and the kernel's full name (bench.py matches the name against
the instance it launched before quoting the traffic)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = next(r for r in rows if "Kernel Name" in r)
    rows = rows[rows.index(h):]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        if len(r) == len(h) and r[mi] == "gpu__time_duration.sum":
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':72s} {'n':>4s} {'mean ns':>12s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:72]:72s} {len(v):4d} {sum(v) / len(v):12.1f} {sum(v) / tot:6.3f}")


def full(rep, cfg, n, d):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
             "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "cycle": 1, "Kcycle": 1e3, "Mcycle": 1e6}
    res = {"source": f"ncu --set full --clock-control none --import-source on, one launch per kernel ({rep})",
           "workload": {"config": int(cfg), "n": int(n), "d": int(d)}, "kernels": {}}
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        def g(m):
            if m not in h or r[h.index(m)] in ("", "n/a"):
                return None
            return float(r[h.index(m)].replace(",", "")) * scale.get(units[h.index(m)], 1)
        name = r[h.index("Kernel Name")]
        key = "fct1_sketch" if "sketch" in name else ("l1_rownorm" if "rownorm" in name else name)
        cyc = g("sm__cycles_elapsed.avg")
        wf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        rec = {"kernel": name,
               "gpu_time_ms_under_ncu": g("gpu__time_duration.sum") / 1e6 if g("gpu__time_duration.sum") else None,
               "sm_cycles_elapsed_note": "sm__cycles_elapsed.avg (per SM)",
               "dram_bytes_read": g("dram__bytes_read.sum"), "dram_bytes_write": g("dram__bytes_write.sum"),
               "smem_wavefronts": wf, "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
               "warp_instructions": g("smsp__inst_executed.sum"), "sm_cycles_elapsed_avg": cyc,
               "tensor_pipe_pct": g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
               "alu_pipe_pct": g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
               "fma_pipe_pct": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
               "lsu_inst_pct": g("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
               "dram_throughput_pct": g("dram__throughput.avg.pct_of_peak_sustained_elapsed")}
        if wf and cyc:
            pct = 100.0 * wf / (cyc * 148)
            rec["smem_pipe_pct_of_peak"] = round(pct, 1)
            if "sketch" in name:
                rec["limiter"] = {"resource": "shared-memory data pipe (l1tex lsu wavefronts, 1 per cycle per SM)",
                                  "pct_of_peak": round(pct, 1), "wavefronts_per_launch": wf}
        res["kernels"][key] = rec
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], *sys.argv[3:6])
