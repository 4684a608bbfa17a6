"""Stall-reason totals of one kernel in an ncu source-page CSV, overall and for the given opcodes:
python scripts/ncu_stall_reasons.py page.csv "<kernel-name substring>" IMAD DMUL ..."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
kernels=[]; cur=None
for r in rows:
    if r and r[0]=="Kernel Name": cur={"name":r[1],"rows":[]}; kernels.append(cur)
    elif r and r[0]=="Address": cur["hdr"]=r
    elif cur is not None and r and r[0][:2]=="0x": cur["rows"].append(r)
seen=set()
for k in kernels:
    if k["name"] in seen or sys.argv[2] not in k["name"]: continue
    seen.add(k["name"])
    h=k["hdr"]; isrc=h.index("Source")
    cols=[i for i,c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    byop=collections.defaultdict(collections.Counter); tot=collections.Counter()
    for r in k["rows"]:
        toks=r[isrc].split()
        if not toks: continue
        op=(toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        for i in cols:
            v=float(r[i] or 0); byop[op][h[i]]+=v; tot[h[i]]+=v
    print(k["name"][40:100]); print("  total", tot.most_common(8))
    for op in sys.argv[3:]:
        print("  ", op, byop[op].most_common(5))
