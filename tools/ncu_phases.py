"""Per-phase totals (stall samples, executed warp-instructions, shared wavefronts, global sectors)
of an ncu SASS source CSV: instructions are walked in address order and attributed to the phase
of the last kernel-body source line seen (inlined helpers inherit their call site's phase).
usage: python tools/ncu_phases.py src.csv kernel.o KERNEL_SUBSTRING line:name[,line:name...] [npairs]"""
import collections, csv, sys
exec(open(__file__.replace("ncu_phases.py", "ncu_lines.py")).read().split("rows = list(csv.reader")[0].replace(
    "top = int(sys.argv[4]) if len(sys.argv) > 4 else 40", "top = 40"))
bounds = sorted((int(x.split(":")[0]), x.split(":")[1]) for x in sys.argv[4].split(","))
npairs = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
body0 = bounds[0][0]
rows = list(csv.reader(open(csvf)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]; ci = {n: h.index(n) for n in h}
ins = []
for r in rows[i0 + 1:]:
    if len(r) < len(h): continue
    try:
        ins.append((int(r[0], 16), int(r[ci["Warp Stall Sampling (All Samples)"]] or 0), int(r[ci["Instructions Executed"]] or 0),
                    int(r[ci["L1 Wavefronts Shared"]] or 0), int(r[ci["L2 Theoretical Sectors Global"]] or 0), r[1],
                    {k[6:]: int(r[ci[k]] or 0) for k in h if k.startswith("stall_") and "Not Issued" not in k}))
    except ValueError:
        pass
base = min(i[0] for i in ins)
ph = bounds[0][1]
tot = collections.defaultdict(lambda: [0, 0, 0, 0]); stl = collections.defaultdict(collections.Counter)
ops = collections.defaultdict(collections.Counter)
for a, s, e, w, g, src, st in sorted(ins):
    ln = line_of.get(a - base)
    if ln and ln[0].startswith(os.path.basename(obj).replace(".o", "").split(".")[0]) and ln[1] >= body0:
        for b, name in bounds:
            if ln[1] >= b: ph = name
    t = tot[ph]; t[0] += s; t[1] += e; t[2] += w; t[3] += g
    stl[ph].update(st)
    op = src.split()[0] if not src.strip().startswith("@") else src.split()[1]
    ops[ph][op.split(".")[0]] += e
S = sum(t[0] for t in tot.values()); E = sum(t[1] for t in tot.values())
print(f"{'phase':14s} {'samples%':>8s} {'instr/pair':>10s} {'smem wf/pair':>12s} {'gl sect/pair':>12s}  top stalls | top opcodes (per pair)")
for b, name in bounds:
    t = tot[name]
    why = " ".join(f"{k}:{v * 100 // max(t[0], 1)}" for k, v in stl[name].most_common(4))
    top = " ".join(f"{k}:{v / npairs:.0f}" for k, v in ops[name].most_common(8))
    print(f"{name:14s} {100 * t[0] / S:8.1f} {t[1] / npairs:10.0f} {t[2] / npairs:12.0f} {t[3] / npairs:12.0f}  {why} | {top}")
print(f"{'total':14s} {100.0:8.1f} {E / npairs:10.0f} {sum(t[2] for t in tot.values()) / npairs:12.0f} {sum(t[3] for t in tot.values()) / npairs:12.0f}")
