"""Aggregate ncu SASS source-page stall columns: overall and per execution-count class."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_src = hdr.index("Source"); i_ex = hdr.index("Instructions Executed")
sc = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in sc}
tot = collections.Counter(); bycls = collections.defaultdict(collections.Counter); ninst = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) < len(hdr): continue
    try: ex = int(r[i_ex])
    except: continue
    op = r[i_src].strip().split()
    o = (op[1] if op and op[0].startswith("@") else (op[0] if op else "?")).split(".")[0]
    for h in sc:
        try: v = int(r[idx[h]])
        except: v = 0
        tot[h] += v; bycls[ex][h] += v
    ninst[ex] += 1; ops[ex][o] += 1
T = sum(tot.values())
print("total stall samples", T)
for h, v in tot.most_common(12): print(f"  {h:24s} {100*v/T:5.1f}%")
top = sorted(bycls, key=lambda e: -sum(bycls[e].values()))[:int(sys.argv[2]) if len(sys.argv) > 2 else 6]
for e in top:
    s = sum(bycls[e].values())
    print(f"exec count {e}: {ninst[e]} instr, {100*s/T:.1f}% samples; ops {ops[e].most_common(6)}")
    print("    ", [(h[6:], round(100*v/s, 1)) for h, v in bycls[e].most_common(6)])
