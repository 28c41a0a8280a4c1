import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
import sys; sys.path.insert(0, "/root/repo/tools/analysis"); from ranges import ranges; R = ranges()
cur = None; hdr = None; agg = collections.Counter(); smp = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = r; ii = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < len(hdr): continue
    if r[0]: ln = int(r[0]); continue
    try: n = int(r[ii] or 0); sm = int(r[si] or 0)
    except ValueError: continue
    name = cur
    if cur == "crb_device.cuh":
        name = "cuh_other"
        for nm, a, b in R:
            if a <= ln <= b: name = nm; break
    elif cur == "curobo_b200.cu":
        name = "solver(cu)"
    agg[name] += n; smp[name] += sm
ti = sum(agg.values()); ts = sum(smp.values())
npass = float(sys.argv[2]) if len(sys.argv) > 2 else 0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    extra = f"  {v / npass:8.0f} warp-inst/pass" if npass else ""
    print(f"{k:20s} ins {100*v/ti:5.1f}%  smp {100*smp[k]/ts:5.1f}%{extra}")
