"""Executed warp instructions per CUDA source line of an ncu --set full report
(SASS rows attributed through -lineinfo).  python scripts/ncu_lineinst.py rep [top]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
per_line = collections.Counter(); src = {}; fname = None; tot = 0; hdr = None
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 5: continue
    d = dict(zip(hdr, r))
    try: n = int(d["Instructions Executed"]); ln = int(d["Line No"])
    except (ValueError, KeyError): continue
    key = (fname, ln); per_line[key] += n; src[key] = d["Source"].strip()[:90]; tot += n
print("total", tot)
for (f, l), n in per_line.most_common(top):
    print(f"{100*n/max(tot,1):5.1f}% {f}:{l}  {src[(f,l)]}")
