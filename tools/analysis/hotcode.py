import csv, collections, sys, re
sys.path.insert(0, "/root/repo/tools/analysis")
src = open('scratch/phases.py').read()
from ranges import ranges; R = ranges()
rows = list(csv.reader(open(sys.argv[1])))
passes = float(sys.argv[2])
hdr=None; cur=None; ln=None
agg=collections.Counter(); aggn=collections.Counter()
for r in rows:
    if not r: continue
    if r[0]=="File Path": cur=r[1].split('/')[-1]; continue
    if r[0]=="Line No": hdr=r; ii=hdr.index("Instructions Executed"); continue
    if hdr is None or len(r)<len(hdr): continue
    if r[0]: ln=int(r[0]); continue
    try: n=int(r[ii] or 0)
    except: continue
    name=cur
    if cur=="crb_device.cuh":
        name="cuh_other"
        for nm,a,b in R:
            if a<=ln<=b: name=nm; break
    elif cur=="curobo_b200.cu": name=f"cu:{ln//50*50}"
    if n >= passes: agg[name]+=1
    aggn[name]+=n
for k,v in agg.most_common(30): print(f"{k:22s} hot instr {v:5d} ({v*16/1024:5.1f} KB)  exec/pass {aggn[k]/passes:8.0f}")
