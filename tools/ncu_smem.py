"""Shared-memory bank-conflict excess per source line from an ncu SASS source CSV (development aid).
usage: python tools/ncu_smem.py src.csv kernel.o KERNEL_SUBSTRING"""
import collections, sys
sys.argv = sys.argv[:4]
exec(open(__file__.replace("ncu_smem.py", "ncu_lines.py")).read().split("base = min")[0].replace("top = int(sys.argv[4]) if len(sys.argv) > 4 else 40", "top = 40"))
import csv
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]; ci = {n: h.index(n) for n in h}
addr = []
for r in rows[i0 + 1:]:
    if len(r) < len(h): continue
    try:
        addr.append((int(r[0], 16), int(r[ci['L1 Wavefronts Shared Excessive']] or 0), int(r[ci['L1 Wavefronts Shared']] or 0), r[1]))
    except ValueError:
        pass
base = min(a[0] for a in addr)
agg = collections.defaultdict(lambda: [0, 0])
for a, ex, w, src in addr:
    ln = line_of.get(a - base, ("?", 0))
    agg[ln][0] += ex; agg[ln][1] += w
T = sum(v[1] for v in agg.values()); X = sum(v[0] for v in agg.values())
print(f"shared wavefronts {T}, excess {X} ({100*X/max(T,1):.1f}%)")
srcl = open(sys.argv[2].replace(".o", "")).read().splitlines() if False else None
for (f, ln), (ex, w) in sorted(agg.items(), key=lambda x: -x[1][0])[:20]:
    print(f"{f}:{ln:5d} excess {ex:11d} of {w:11d}")
