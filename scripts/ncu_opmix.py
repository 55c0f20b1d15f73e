"""Instruction mix of an ncu --set full report's source page (SASS): executed
warp instructions per opcode, and shared-memory wavefronts ideal / actual.
    python scripts/ncu_opmix.py report.ncu-rep [top]
"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
ops = collections.Counter(); tot = 0; wf = wf_ideal = 0; hdr = None
for r in csv.reader(out):
    if r and r[0] == "Address": hdr = r; continue
    if hdr is None or len(r) < len(hdr) - 2: continue
    d = dict(zip(hdr, r))
    try: n = int(d["Instructions Executed"])
    except (ValueError, KeyError): continue
    toks = d["Source"].split()
    op = toks[1] if toks and toks[0].startswith("@") else toks[0]
    ops[op.rstrip(";")] += n; tot += n
    try:
        wf += int(d["L1 Wavefronts Shared"]); wf_ideal += int(d["L1 Wavefronts Shared Ideal"])
    except (ValueError, KeyError): pass
print("total warp instructions", tot, " shared wavefronts", wf, "ideal", wf_ideal)
for op, n in ops.most_common(top):
    print(f"{100*n/tot:5.1f}%  {n:>14d}  {op}")
