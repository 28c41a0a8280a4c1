"""Summarise an ncu report: key details, stall mix, per-phase / per-function instruction share."""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ['Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Achieved Occupancy', 'Registers Per Thread',
        'Dynamic Shared Memory Per Block', 'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp',
        'Executed Instructions', 'Compute (SM) Throughput', 'L1/TEX Cache Throughput', 'DRAM Throughput']
for row in csv.reader(io.StringIO(det)):
    for k in keep:
        if k in row:
            i = row.index(k); print(f"  {k:40s} {row[i+1]:14s} {row[i+2]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur = None; hdr = None; agg = collections.Counter(); smp = collections.Counter(); stall = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = r; ii = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)")
        sidx = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]; continue
    if hdr is None or len(r) < len(hdr): continue
    if r[0]:
        ln = int(r[0]); continue        # source rows repeat the sum of their SASS rows
    try: n = int(r[ii] or 0); sm = int(r[si] or 0)
    except ValueError: continue
    agg[(cur, ln)] += n; smp[(cur, ln)] += sm
    for i in sidx:
        try: stall[hdr[i][6:]] += int(r[i] or 0)
        except ValueError: pass
ts = sum(stall.values())
print("  stalls: " + " ".join(f"{k}={100*v/ts:.1f}%" for k, v in stall.most_common(8)))
srcf = open(sys.argv[2] if len(sys.argv) > 2 else '/root/repo/paper_2310_17274_b200/csrc/crb_device.cuh').read().split('\n')
marks = []
for i, l in enumerate(srcf):
    m = re.match(r'^__device__ .*?(\w+)\(', l)
    if m: marks.append((i + 1, 'fn:' + m.group(1)))
    m = re.match(r'^\s*// ---- (\S+)', l)
    if m: marks.append((i + 1, 'phase:' + m.group(1)))
marks.sort(); marks.append((10**9, 'END'))
tot = sum(agg.values()); tsm = sum(smp.values())
out = collections.Counter(); outs = collections.Counter()
for (f, ln), v in agg.items():
    name = f
    if f == 'crb_device.cuh':
        for (a, n), (b, _) in zip(marks, marks[1:]):
            if a <= ln < b: name = n
    out[name] += v; outs[name] += smp[(f, ln)]
for n, v in out.most_common(22):
    print(f"  {n:28s} ins {100*v/tot:5.1f}%  smp {100*outs[n]/tsm:5.1f}%")
