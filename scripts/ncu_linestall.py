"""Stall samples per CUDA source line with the reason split (ncu --set full, -lineinfo).
    python scripts/ncu_linestall.py rep [top]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
tot = collections.Counter(); why = collections.defaultdict(collections.Counter); fname = None; hdr = None; all_s = 0
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 5: continue
    d = dict(zip(hdr, r))
    try: ln = int(d["Line No"])
    except (ValueError, KeyError): continue
    key = (fname, ln)
    for h, v in d.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try: x = float(v)
            except ValueError: continue
            tot[key] += x; why[key][h[6:]] += x; all_s += x
for key, n in tot.most_common(top):
    print(f"{100*n/all_s:5.1f}% {key[0]}:{key[1]}  " + " ".join(f"{k}={100*v/n:.0f}%" for k, v in why[key].most_common(4)))
