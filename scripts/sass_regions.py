"""Split the per-instruction stall samples of an ncu source page (SASS) of oz_gemm_kernel into
the producer (UTMALDG), MMA issuer (UTCIMMA) and epilogue (LDTM...) regions and print the top
stalled instructions per region.  usage: ncu -i X --page source --csv --print-source=sass > f.csv;
python scripts/sass_regions.py f.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
kernels = []
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and r and r[0].startswith("0x") or (cur is not None and r and r[0].isdigit()):
        cur["rows"].append(r)
for k in kernels:
    h = k["hdr"]
    ia, isrc, iall, inot = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Warp Stall Sampling (Not-issued Samples)")
    iex = h.index("Instructions Executed")
    rs = k["rows"]
    src = [r[isrc] for r in rs]
    def first(pat):
        return next((i for i, s in enumerate(src) if pat in s), None)
    def last(pat):
        return max((i for i, s in enumerate(src) if pat in s), default=None)
    marks = {"TMA": (first("UTMALDG"), last("UTMALDG")), "MMA": (first("UTCIMMA"), last("UTCIMMA")),
             "LDTM": (first("LDTM"), last("LDTM"))}
    tot = sum(float(r[iall] or 0) for r in rs)
    print("==", k["name"][:90], "total samples", tot, marks)
    # region of each instruction: nearest marker range it falls in, else 'other'
    def region(i):
        for nm, (a, b) in marks.items():
            if a is not None and a - 40 <= i <= b + 40:
                return nm
        return "other"
    agg = {}
    for i, r in enumerate(rs):
        agg.setdefault(region(i), [0.0, 0.0])
        agg[region(i)][0] += float(r[iall] or 0)
        agg[region(i)][1] += float(r[iex] or 0)
    for nm, (smp, ex) in agg.items():
        print(f"   region {nm:6s} samples {smp:10.0f} ({smp / max(tot, 1) * 100:5.1f} %)  inst executed {ex:.3g}")
    top = sorted(range(len(rs)), key=lambda i: -float(rs[i][iall] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
    for i in top:
        print(f"   {float(rs[i][iall] or 0):8.0f} {region(i):6s} {src[i][:80]}")
