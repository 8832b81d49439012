"""Summarise one kernel of an ncu --set full report into the JSON kept under
profiles/ (the bench reads dram_bytes_per_launch from it).
Usage: ncu_summary.py rep kernel-regex kernel-label workload launch-desc source-desc > out.json"""
import csv, io, json, subprocess, sys

rep, kre, label, workload, launch, source = sys.argv[1:7]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
d = {k: (val, u) for k, u, val in zip(h, units, v)}


def num(k):
    return float(d[k][0].replace(",", ""))


keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]


def to_bytes(k):
    val, u = d[k]
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


stalls = {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: num(k)
          for k in h if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio")}
# shared-memory data pipe: one wavefront per clock per SM
pipe = None
if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in d and "gpu__time_duration.sum" in d:
    t_ms = num("gpu__time_duration.sum") * {"ms": 1, "us": 1e-3, "usecond": 1e-3,
                                             "msecond": 1}.get(d["gpu__time_duration.sum"][1], 1)
    cyc = t_ms * 1e-3 * num("sm__cycles_elapsed.avg.per_second") * 1e9
    sms = num("launch__grid_size") if num("launch__grid_size") <= 148 else 148
    pipe = num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / (cyc * sms)
out = {"kernel": label, "workload": workload, "launch": launch, "source": source,
       "dram_bytes_per_launch": to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum"),
       "smem_wavefront_pipe_frac": pipe,
       "metrics": {k: f"{d[k][0]} {d[k][1]}".strip() for k in keep if k in d},
       "top_stalls_per_issue": dict(sorted(stalls.items(), key=lambda t: -t[1])[:8])}
json.dump(out, sys.stdout, indent=1)
print()
