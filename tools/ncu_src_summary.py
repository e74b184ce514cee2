"""Summarise an `ncu --page source --csv --print-source sass` export: top SASS
lines by stall samples and per-opcode totals (development aid)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]
ci = {n: h.index(n) for n in h}
S, E = ci["Warp Stall Sampling (All Samples)"], ci["Instructions Executed"]
data = []
for r in rows[i0 + 1:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[S] or 0), int(r[E] or 0), r[0], r[1]))
    except ValueError:
        pass
tot_s = sum(d[0] for d in data); tot_e = sum(d[1] for d in data)
print(f"samples {tot_s}  executed {tot_e}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for s, e, a, src in sorted(data, reverse=True)[:top]:
    print(f"{s:8d} {100*s/tot_s:5.1f}% exec {e:10d}  {a}  {src[:90]}")
op = collections.defaultdict(lambda: [0, 0])
for s, e, a, src in data:
    k = src.split()[0] if src.split() else "?"
    if k.startswith("@"):
        k = src.split()[1] if len(src.split()) > 1 else k
    k = k.split(".")[0]
    op[k][0] += s; op[k][1] += e
print("opcode   samples%  exec%")
for k, (s, e) in sorted(op.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{k:10s} {100*s/tot_s:6.1f} {100*e/tot_e:6.1f}")
