"""Copy the round's measurement outputs from gpurun_out/prof/ into profiles/
and regenerate the numbers in profiles/README.md's tables.

    python scripts/make_profiles.py <round tag, e.g. round1>
"""
import json, os, shutil, subprocess, sys, collections, csv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "round1"


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


for c in ["C1", "C2", "C3", "C4", "C5", "reference_C2"]:
    shutil.copy(os.path.join(SRC, f"bench_{c}.json"), os.path.join(DST, f"{tag}_bench_{c}.json"))
shutil.copy(os.path.join(SRC, "launches_bench_C2.csv"), os.path.join(DST, f"{tag}_launches_bench_C2.csv"))
with open(os.path.join(DST, f"{tag}_launches_bench_C2_summary.txt"), "w") as f:
    f.write(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_launch_table.py"),
                            os.path.join(DST, f"{tag}_launches_bench_C2.csv")],
                           capture_output=True, text=True).stdout)
rep = os.path.join(SRC, "join_c2_iter1.ncu-rep")
summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                      capture_output=True, text=True).stdout
open(os.path.join(DST, f"{tag}_ncu_join_c2_iter1.json"), "w").write(summ)
hot = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_hot.py"), rep, "40"],
                     capture_output=True, text=True).stdout
open(os.path.join(DST, f"{tag}_ncu_join_c2_hot_lines.txt"), "w").write(hot)
j = json.loads(summ)["join_distances_kernel"]
rd, wr = float(j["dram__bytes_read.sum"][0]), float(j["dram__bytes_write.sum"][0])
unit = {"Gbyte": 1e9, "Mbyte": 1e6}
traffic = rd * unit[j["dram__bytes_read.sum"][1]] + wr * unit[j["dram__bytes_write.sum"][1]]
json.dump({"C2": {"bytes_per_launch": traffic, "launch": "iteration 1 (largest launch)",
                  "algorithmic_bytes_same_launch": 2796920 * (4 * 784 + 8) + 12 * 70000 * 20,
                  "source": f"profiles/{tag}_ncu_join_c2_iter1.json (ncu --set full, "
                            "dram__bytes_read.sum + dram__bytes_write.sum)"}},
          open(os.path.join(DST, "join_traffic.json"), "w"), indent=1)

# launch shares (product kernels only)
lines = [l for l in open(os.path.join(DST, f"{tag}_launches_bench_C2.csv")) if l.startswith('"')]
rows = list(csv.reader(lines)); hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
tot = collections.Counter()
for r in rows[1:]:
    k = r[idx["Kernel Name"]].split("(")[0].split("::")[-1]
    tot[k] += float(r[idx["Metric Value"]].replace(",", ""))
harness = {"bf_filter_kernel", "ffma2_kernel", "ffma_kernel", "bf_rerank_kernel", "iota_kernel"}
prod = sum(v for k, v in tot.items() if k not in harness)
shares = {k: 100 * v / prod for k, v in tot.items() if k not in harness}

b = {c: last_json(os.path.join(DST, f"{tag}_bench_{c}.json")) for c in ["C1", "C2", "C3", "C4", "C5"]}
ref = last_json(os.path.join(DST, f"{tag}_bench_reference_C2.json"))
desc = {"C1": "C1 n=10k d=8 k=20 cap 20", "C2": "C2 n=70k d=784 k=20 (default)",
        "C3": "C3 n=200k d=128 k=30", "C4": "C4 n=2M d=96 k=10", "C5": "C5 n=1M d=960 k=20"}
rows_md = []
for c in ["C2", "C1", "C3", "C4", "C5"]:
    d = b[c]; r = d["recall_at_k"]
    rec = f"{r['gpu']:.4f}" + (f" (reference {r['reference']:.4f})" if "reference" in r else "")
    rows_md.append(f"| `{tag}_bench_{c}.json` | {desc[c]} | {d['value']:.3g} | {d['ms_per_step']:.1f} | "
                   f"{d['e2e']['value']:.3g} | {d['roofline']['frac']:.3f} | "
                   f"{d['iterations_per_build']:.0f} | {rec} |")
rows_md.append(f"| `{tag}_bench_reference_C2.json` | reference (`oracle/_ref`, 1 core), first 10k rows "
               f"of C2 | {ref['value']:.3g} | {ref['ms_per_step']:.0f} | — | — | — | — |")
cb = b["C2"]["cpu_baseline"]
stalls = j["stall_cycles_per_issue_top"]
fill = {
    "BENCH_ROWS": "\n".join(rows_md),
    "CPU_VALUE": f"{cb['value']:.3g}", "CPU_S": f"{cb['build_time_s']:.1f}",
    "GPU_MS": f"{b['C2']['ms_per_step']:.1f}",
    "SPEEDUP": f"{cb['build_time_s'] * 1e3 / b['C2']['ms_per_step']:.0f}",
    "SHARE_JOIN": f"{shares.get('join_distances_kernel', 0):.1f}",
    "SHARE_MERGE": f"{shares.get('join_merge_kernel', 0) + shares.get('hub_merge_kernel', 0):.1f}",
    "SHARE_FIN": f"{shares.get('finalize_kernel', 0):.1f}",
    "SHARE_INIT": f"{shares.get('init_random_kernel', 0):.1f}",
    "LIVE_SHARE": f"{b['C2']['roofline']['share_of_step']:.2f}",
    "NCU_MS": f"{float(j['gpu__time_duration.sum'][0]):.2f}",
    "NCU_TF": f"{129.6 / float(j['gpu__time_duration.sum'][0]):.1f}",
    "NCU_FRAC": f"{129.6 / float(j['gpu__time_duration.sum'][0]) / 72.5:.2f}",
    "DRAM_R": f"{rd:.2f} {j['dram__bytes_read.sum'][1].replace('byte', 'B')}",
    "DRAM_W": f"{wr:.2f} {j['dram__bytes_write.sum'][1].replace('byte', 'B')}",
    "L2HIT": f"{float(j['lts__t_sector_hit_rate.pct'][0]):.0f}",
    "FMA": f"{float(j['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'][0]):.1f}",
    "ISSUE": f"{float(j['smsp__issue_active.avg.pct_of_peak_sustained_active'][0]):.1f}",
    "OCC": f"{float(j['sm__warps_active.avg.pct_of_peak_sustained_active'][0]):.0f}",
    "REGS": j["launch__registers_per_thread"][0],
    "STALLS": ", ".join(f"{k.replace('_', ' ')} {v}" for k, v in list(stalls.items())[:4]),
    "FRAC_BUILD": f"{b['C2']['roofline']['frac']:.3f}",
}
tmpl = open(os.path.join(ROOT, "scripts", "profiles_readme.tmpl")).read()
for k, v in fill.items():
    tmpl = tmpl.replace("{{" + k + "}}", str(v))
open(os.path.join(DST, "README.md"), "w").write(tmpl.replace("{{TAG}}", tag))
print("profiles written")
