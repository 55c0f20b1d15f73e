"""Per-source-line instruction counts and stall samples from an ncu report (one kernel id)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; kid = sys.argv[2] if len(sys.argv) > 2 else None; top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kid is not None: cmd += ["--launch-skip", kid, "--launch-count", "1"] if False else []
out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
inst = collections.Counter(); samp = collections.Counter(); src = {}
fname = None; hdr = None; kernel = None
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; hdr = None; continue
    if len(r) == 2 and r[0] == "Function Name": kernel = r[1][:60]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    try: ln = int(r[0]); s = float(r[4]); ie = float(r[7])
    except ValueError: continue
    key = (kernel, fname, ln); inst[key] += ie; samp[key] += s; src[key] = r[1].strip()[:90]
tot = sum(inst.values())
for key, v in inst.most_common(top):
    print(f"{100*v/tot:5.1f}% inst {v:.3g}  samp {samp[key]:.0f}  {key[0][:25]} {key[1]}:{key[2]} {src[key]}")
