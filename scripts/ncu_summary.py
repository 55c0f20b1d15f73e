"""Summarise an ncu --set full report into JSON (per kernel name, first launch):
    python scripts/ncu_summary.py report.ncu-rep > profiles/<name>.json
"""
import csv, json, subprocess, sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
rep = sys.argv[1]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                      capture_output=True, text=True).stdout.splitlines()))
hdr, units = rows[0], rows[1]
out = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "?").split("(")[0].split("::")[-1]
    if name in out:
        continue
    ent = {m: [d.get(m), units[hdr.index(m)] if m in hdr else None] for m in METRICS}
    stalls = {}
    for h, v in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(float(v), 3)
            except ValueError:
                pass
    ent["stall_cycles_per_issue_top"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])
    out[name] = ent
print(json.dumps(out, indent=1))
