"""Turn a tools/round_measure.sh output directory into the committed profile summaries.

    python tools/make_profiles.py TAG path/to/hsw_dmma1.cu.o
reads gpurun_out/TAG/ and writes profiles/TAG_bench_c4.json, TAG_bench_reference_c4.json,
TAG_configs.md, TAG_launches_c4.md, TAG_ncu_c4.md and profiles/traffic_c4.json."""
import collections, csv, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, obj = sys.argv[1], sys.argv[2]
o = os.path.join(ROOT, "gpurun_out", tag)
P = os.path.join(ROOT, "profiles")
KSUB = os.environ.get("KSUB", "Li3ELi3ELi2ELi5ELi12ELi8ELb0ELi1EE")   # the C4 production instantiation (static-pivot LU)
PAIRS = 8388608


def last_json(path):
    return [x for x in open(path) if x.startswith("{")][-1]


bench = json.loads(last_json(f"{o}/bench.log"))
ref = json.loads(last_json(f"{o}/bench_ref.log"))
open(f"{P}/{tag}_bench_c4.json", "w").write(json.dumps(bench) + "\n")
open(f"{P}/{tag}_bench_reference_c4.json", "w").write(json.dumps(ref) + "\n")

pc = bench.get("per_config") or {}
CL = [f"# {tag} per-config report (B200, one GPU, measured inside the bench run)", "",
      "`bench.py`'s `per_config` block: each BASELINE.json config at full size, one all-ordinate sweep "
      "(device-resident, CUDA events on the library stream, best of 3 after 2 warm-ups), then source iteration "
      "from psi = phi = 0 to ||dphi||_2 / ||phi||_2 < 1e-8 (`hsw_source_iteration`, device time).", "",
      "| config | pairs | n | sweep ms | solves/s | TFLOP/s (LU-alg) | roofline frac | SI iterations | SI s | setup s |",
      "|---|---|---|---|---|---|---|---|---|---|"]
for name in ("c1", "c2", "c3", "c4", "c5"):
    r = pc.get(name, {})
    if "sweep_ms" in r:
        CL.append(f"| {name} | {r['pairs']:,} | {r['n']} | {r['sweep_ms']:.2f} | {r['solves_per_s']:.4g} | "
                  f"{r['tflops_lu_alg']:.2f} | {r['roofline_frac']:.4f} | {r['si_iterations']} | {r['si_s']:.2f} | "
                  f"{r['setup_s']:.2f} |")
    else:
        CL.append(f"| {name} | error: {r.get('error')} |")
CL += ["", "TFLOP/s = F(n) pairs / sweep time, F(n) = 2/3 n^3 + 2 n^2 (LU-algorithmic, SURVEY §8d); roofline "
       f"frac against the in-run measured FP64 peak ({bench['roofline']['peak']:.2f} TFLOP/s)."]
open(f"{P}/{tag}_configs.md", "w").write("\n".join(CL) + "\n")

rows = [r for r in csv.reader(open(f"{o}/launches.csv")) if r]
i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[i0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[i0 + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki].replace("void ", "").replace("unnamed>::", "hsw::"))
    name = re.sub(r", 0>$", ", false>", name)
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v / 1e6 if r[ui] == "ns" else v
tot = sum(v[1] for v in agg.values())
L = [f"# {tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none), C4, "
     "`bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e`", "",
     "One dataflow launch of the sweep kernel per sweep (+ the scattering-source kernel). Cold-cache serialised "
     "per-launch times: compare SHARES, not absolutes.", "",
     "| kernel | launches | total ms | ms per launch | share |", "|---|---|---|---|---|"]
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    L.append(f"| {k} | {n} | {ms:.2f} | {ms / n:.2f} | {100 * ms / tot:.1f}% |")
L += ["", "coupling_max / element_tensor / block_scale kernels are one-time setup; fp64/dmma_peak_kernel are "
      "bench.py's in-run peak measurements."]
open(f"{P}/{tag}_launches_c4.md", "w").write("\n".join(L) + "\n")

tr = {}
for r in csv.reader(open(f"{o}/traffic.csv")):
    if len(r) > 14 and r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                                 "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"):
        tr[r[12]] = float(r[14].replace(",", ""))
rd, wr = tr["dram__bytes_read.sum"], tr["dram__bytes_write.sum"]
json.dump({"dram_bytes_per_sweep": rd + wr,
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,... -k regex:dmma1 -c 1 over the single "
                     f"dataflow launch of one full C4 sweep ({PAIRS:,} pairs, {tr['gpu__time_duration.sum'] / 1e6:.1f} ms "
                     f"under ncu): read {rd / 1e9:.1f} GB + write {wr / 1e9:.1f} GB; L1 hit "
                     f"{tr['l1tex__t_sector_hit_rate.pct']:.1f} %, L2 hit {tr['lts__t_sector_hit_rate.pct']:.1f} %; "
                     f"profiles/{tag}_ncu_c4.md",
           "note": f"= {(rd + wr) / PAIRS / 1e3:.1f} KB per pair: the compulsory element-tensor stream (one 131 KB "
                   "tensor per (level, element): 2.36 M visits = 309 GB) + psi; bench.py reports it per launch"},
          open(f"{P}/traffic_c4.json", "w"), indent=1)



def ncu_section(sub, cfg, src_file, obj_file, ksub, label):
    """Markdown of one --set full capture under gpurun_out/TAG/SUB (tools/ncu_case.sh)."""
    od = f"{o}/{sub}"
    raw = list(csv.reader(open(f"{od}/raw.csv")))
    d = dict(zip(raw[0], raw[2]))
    log = open(f"{od}/ncu_full.log").read()
    sizes = [int(x) for x in re.search(r"level_sizes (.*)", log).group(1).split()]
    skip = {"c4": 300, "c5": 200}[cfg]
    lvl = skip - len(sizes)
    npair = sizes[lvl]
    sys.argv = ["x", f"{od}/src.csv", obj_file, ksub]
    srcl = open(os.path.join(ROOT, "paper_1810_11080_b200/csrc", src_file)).read().splitlines()
    g = {"__name__": "x", "sys": sys}
    exec(open(os.path.join(ROOT, "tools/ncu_lines.py")).read().split("ts = sum")[0], g)
    lagg, stl = g["agg"], g["stl"]
    T = sum(v[0] for v in lagg.values())
    E = sum(v[1] for v in lagg.values())
    M = [f"## {label}: one level, `--set full` (HSW_DATAFLOW=0, level {lvl}: {npair:,} pairs)", "",
         "| metric | value |", "|---|---|"]
    for k, lab in [("gpu__time_duration.sum", "duration (cold, serialised) ms"),
                   ("launch__registers_per_thread", "registers"), ("launch__block_size", "threads per CTA"),
                   ("launch__shared_mem_per_block_dynamic", "dynamic shared memory KB"),
                   ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
                   ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
                   ("sm__inst_executed.avg.per_cycle_active", "IPC"),
                   ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor (DMMA) pipe %"),
                   ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
                   ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1TEX throughput %"),
                   ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
                   ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts")]:
        M.append(f"| {lab} | {d.get(k)} |")
    M.append(f"| executed warp-instructions per pair | {E / npair:.0f} |")
    st = {n: float(v.replace(",", "") or 0) for n, v in d.items()
          if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio")}
    M.append("| stalls per issue | " + ", ".join(f"{n.split('stalled_')[1].split('_per_issue')[0]} {v:.2f}"
                                                 for n, v in sorted(st.items(), key=lambda x: -x[1])[:6]) + " |")
    M += ["", "Top stall lines (SASS mapped to source with tools/ncu_lines.py):", "",
          "| line | stall samples | executed | dominant stalls | source |", "|---|---|---|---|---|"]
    for (fn, ln), (sm, e) in sorted(lagg.items(), key=lambda x: -x[1][0])[:12]:
        why = " ".join(f"{k}:{v * 100 // max(sm, 1)}" for k, v in stl[(fn, ln)].most_common(2))
        txt = srcl[ln - 1].strip()[:70].replace("|", "/") if fn == src_file else fn
        M.append(f"| {ln} | {100 * sm / T:.1f} % | {100 * e / E:.1f} % | {why} | `{txt}` |")
    return M


r = bench["roofline"]
M = [f"# {tag}: sweep kernel profiles (C4: hsw_dmma1, one warp per pair; C5: hsw_dmma2, two warps per pair)", "",
     f"Bench (profiles/{tag}_bench_c4.json): C4 {bench['ms_per_step']:.1f} ms per sweep, {bench['value'] / 1e6:.2f} M "
     f"solves/s, {r['achieved']:.2f} TFLOP/s LU-algorithmic = {100 * r['frac']:.1f} % of the {r['peak']:.2f} TFLOP/s "
     f"measured FP64 peak; e2e {bench['e2e']['value'] / 1e6:.2f} M solves/s.", "",
     "## C4 whole-sweep DRAM traffic", "",
     f"Single dataflow launch (one full C4 sweep) under ncu: {tr['gpu__time_duration.sum'] / 1e6:.1f} ms, DRAM read "
     f"{rd / 1e9:.1f} GB + write {wr / 1e9:.1f} GB = {(rd + wr) / PAIRS / 1e3:.1f} KB per pair "
     f"({(rd + wr) / (tr['gpu__time_duration.sum'] * 1e-9) / 1e12:.2f} TB/s average); L1 hit "
     f"{tr['l1tex__t_sector_hit_rate.pct']:.1f} %, L2 hit {tr['lts__t_sector_hit_rate.pct']:.1f} %.", ""]
M += ncu_section("c4", "c4", "hsw_dmma1.cu", obj, KSUB, "C4 (hsw_dmma1)")
M += [""]
M += ncu_section("c5", "c5", "hsw_dmma2.cu", obj.replace("hsw_dmma1", "hsw_dmma2"), "dmma2_sweep_kernelILi4ELi4ELi8ELi4ELb1E",
                 "C5 (hsw_dmma2)")
open(f"{P}/{tag}_ncu.md", "w").write("\n".join(M) + "\n")
print("wrote", tag, "profiles")
