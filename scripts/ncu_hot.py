"""Summarise an ncu report's source page: stall samples per CUDA source line."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
per_line = collections.Counter(); src = {}; fname = None; tot = 0
rdr = csv.reader(out)
hdr = None
for r in rdr:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 5: continue
    try: s = float(r[4]); int(r[0])
    except ValueError: continue
    key = (fname, int(r[0])); per_line[key] += s; src[key] = r[1].strip()[:100]; tot += s
for (f, l), s in per_line.most_common(top):
    print(f"{100*s/max(tot,1):5.1f}% {f}:{l}  {src[(f,l)]}")
