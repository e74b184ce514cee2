"""Map an ncu SASS source-page CSV onto CUDA source lines (development aid).

usage: python tools/ncu_lines.py src.csv kernel.o KERNEL_SUBSTRING [top]
The CSV is `ncu -i rep --page source --csv --print-source sass`; kernel.o is the
object the profiled library was linked from (nvdisasm -g gives the line table).
Prints stall samples / executed instructions per source line and per line range."""
import collections, csv, os, re, subprocess, sys, tempfile

csvf, obj, sub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, stdout=subprocess.DEVNULL)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.check_output(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], text=True).splitlines()
# line table of the kernel whose .text name contains `sub`
line_of, cur, inside, fn = {}, None, False, None
for l in sass:
    if l.startswith(".text."):
        inside = sub in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]
ci = {n: h.index(n) for n in h}
data = []
for r in rows[i0 + 1:]:
    if len(r) < len(h):
        continue
    try:
        st = {k[6:]: int(r[ci[k]] or 0) for k in h if k.startswith("stall_") and "Not Issued" not in k}
        data.append((int(r[0], 16), int(r[ci["Warp Stall Sampling (All Samples)"]] or 0),
                     int(r[ci["Instructions Executed"]] or 0), r[1], st))
    except ValueError:
        pass
base = min(d[0] for d in data)
agg = collections.defaultdict(lambda: [0, 0])
stl = collections.defaultdict(collections.Counter)
miss = 0
for a, s, e, src, st in data:
    ln = line_of.get(a - base)
    if ln is None:
        miss += 1
        ln = ("?", 0)
    agg[ln][0] += s
    agg[ln][1] += e
    stl[ln].update(st)
ts = sum(v[0] for v in agg.values()); te = sum(v[1] for v in agg.values())
print(f"samples {ts} executed {te} unmapped {miss}")
for (f, ln), (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    why = " ".join(f"{k}:{v*100//max(s,1)}" for k, v in stl[(f, ln)].most_common(3))
    print(f"{f}:{ln:5d} samples {100*s/ts:5.1f}%  exec {100*e/te:5.1f}%  {why}")
if len(sys.argv) > 5:   # ranges "name:a-b,name:c-d"
    for spec in sys.argv[5].split(","):
        nm, rg = spec.split(":")
        a, b = map(int, rg.split("-"))
        s = sum(v[0] for (f, ln), v in agg.items() if a <= ln <= b)
        e = sum(v[1] for (f, ln), v in agg.items() if a <= ln <= b)
        print(f"  {nm:12s} lines {a}-{b}: samples {100*s/ts:5.1f}%  exec {100*e/te:5.1f}%")
