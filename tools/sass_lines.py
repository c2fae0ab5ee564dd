"""Aggregate ncu per-SASS stall samples (``--page source --csv --print-source sass``) by
CUDA source line, using the line table of the same object (nvdisasm -g).
usage: python tools/sass_lines.py <prof.sass.csv> <object.o> <kernel-substring> [top]"""
import csv, collections, re, subprocess, sys, tempfile, os

csvf, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
lines = {}
fn = None; cur = None
for l in dis.split("\n"):
    if ".text." in l and "section" in l:
        fn = l.split(".text.")[1].split(",")[0].strip('"')
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and fn and kname in fn: lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
hdr = rows[1]
iA, iW, iE, iS = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
base = None
agg = collections.Counter(); ex = collections.Counter(); ninst = collections.Counter()
for r in rows[2:]:
    try: a = int(r[iA], 16); w = int(r[iW]); e = int(r[iE])
    except Exception: continue
    if base is None: base = a
    key = lines.get(a - base, ("?", 0))
    agg[key] += w; ex[key] = max(ex[key], e); ninst[key] += e
T = sum(agg.values())
src = {}
order = agg.most_common(top) if os.environ.get('BY', 'stall') == 'stall' else sorted(agg.items(), key=lambda kv: -ninst[kv[0]])[:top]
for k, v in order:
    f, n = k
    txt = ""
    for p in ["paper_2605_02262_b200/csrc/" + f]:
        if os.path.exists(p): txt = open(p).read().split("\n")[n - 1].strip()[:90]
    print(f"{100 * v / T:5.1f}%  ex={ex[k]:8d} inst={ninst[k]:9d}  {f}:{n}  {txt}")
