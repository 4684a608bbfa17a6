"""Opcode histogram (dynamic: ncu "Instructions Executed" per SASS line) of one kernel in an ncu
source-page CSV: python scripts/ncu_op_histogram.py page.csv "<kernel-name substring>"."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
kernels=[]; cur=None
for r in rows:
    if r and r[0]=="Kernel Name": cur={"name":r[1],"rows":[]}; kernels.append(cur)
    elif r and r[0]=="Address": cur["hdr"]=r
    elif cur is not None and r and r[0][:2]=="0x": cur["rows"].append(r)
seen=set()
want=sys.argv[2]
for k in kernels:
    if k["name"] in seen or want not in k["name"]: continue
    seen.add(k["name"])
    h=k["hdr"]; isrc=h.index("Source"); iex=h.index("Instructions Executed"); iall=h.index("Warp Stall Sampling (All Samples)")
    c=collections.Counter(); s=collections.Counter()
    tot=0
    for r in k["rows"]:
        src=r[isrc].strip()
        toks=src.split()
        if not toks: continue
        op=toks[1] if toks[0].startswith("@") else toks[0]
        op=op.split(".")[0]
        ex=float(r[iex] or 0); c[op]+=ex; tot+=ex; s[op]+=float(r[iall] or 0)
    print(k["name"][40:100], "total warp-inst %.3g" % tot, "per tile (38912 tiles) %.0f" % (tot/38912))
    for op,v in c.most_common(28): print(f"   {op:12s} {v/38912:8.0f} per tile  stall-samples {s[op]:8.0f}")
