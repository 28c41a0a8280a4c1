"""Aggregate an ncu source page (cuda,sass csv) per CUDA source line: instructions and stall samples."""
import csv, sys, collections
path = sys.argv[1]
rows = list(csv.reader(open(path)))
cur_file = None
agg = collections.defaultdict(lambda: [0, 0, ""])
hdr = None
line_no = None
src_line = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        line_no = r[0]; src_line = r[1]
        continue                  # source rows repeat the sum of their SASS rows: count SASS only
    try:
        ins = int(r[ii] or 0); smp = int(r[si] or 0)
    except ValueError:
        continue
    k = (cur_file, line_no)
    agg[k][0] += ins; agg[k][1] += smp; agg[k][2] = src_line
tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
print(f"total inst {tot_i:.3e} samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*v[1]/tot_s:5.1f}% smp {100*v[0]/tot_i:5.1f}% ins  {k[0]}:{k[1]:>4}  {v[2].strip()[:90]}")
