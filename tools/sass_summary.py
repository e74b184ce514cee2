"""SASS opcode histogram of the production sweep kernels (evidence for profiles/):
python tools/sass_summary.py OUT.md [obj_dir]"""
import collections, os, re, subprocess, sys

out = sys.argv[1]
objd = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                           "paper_1810_11080_b200", "lib", "obj")
KERNELS = [("hsw_dmma1.cu.o", "Li3ELi3ELi2ELi5ELi12ELi8ELb0ELi1EE", "C4: dmma1_sweep_kernel<3,3,2,5,12,8,SP=1> (static-pivot LU)"),
           ("hsw_dmma1.cu.o", "Li3ELi2ELi2ELi0ELi20ELi8ELb0ELi1EE", "C3: dmma1_sweep_kernel<3,2,2,0,20,8,SP=1>"),
           ("hsw_dmma1.cu.o", "Li2ELi3ELi3ELi0ELi16ELi8ELb0ELi1EE", "C2: dmma1_sweep_kernel<2,3,3,0,16,8,SP=1>"),
           ("hsw_dmma2.cu.o", "dmma2_sweep_kernelILi4ELi4ELi8ELi4ELb1E", "C5: dmma2_sweep_kernel<4,4,8,4,SP> (two-warp left-looking LU)"),
           ("hsw_dmma1.cu.o", "Li3ELi3ELi2ELi5ELi12ELi4ELb0ELi0EE", "fallback C4: dmma1_sweep_kernel<3,3,2,5,12,4,SP=0> (pivoted Gauss-Jordan)"),
           ("hsw_dmma2.cu.o", "dmma2_sweep_kernelILi4ELi4ELi8ELi4ELb0E", "fallback C5: dmma2_sweep_kernel<4,4,8,4> (pivoted Gauss-Jordan)")]
FOCUS = ["DMMA", "LDTM", "STTM", "UTCBAR", "UBLKPF", "UBLKCP", "UTMALDG", "DFMA", "DMUL", "DADD", "LDS", "STS",
         "LDG", "STG", "SHFL", "CREDUX", "BAR", "MEMBAR", "STL", "LDL"]
L = ["# SASS opcode counts of the production sweep kernels (static, `cuobjdump -sass`)", "",
     "DMMA = `mma.sync.m8n8k4.f64` (FP64 tensor core; B200 has no FP64 `tcgen05.mma` kind); LDTM/STTM = "
     "`tcgen05.ld/st` (tensor-memory tile storage); UBLKPF = `cp.async.bulk.prefetch.L2` (TMA L2 prefetch of the "
     "element tensor); CREDUX = `redux.sync` (pivot search); BAR = named barriers (dmma2's two-warp pairs).", "",
     "| kernel | SASS instructions | " + " | ".join(FOCUS) + " |", "|---|---|" + "---|" * len(FOCUS)]
for obj, sub, label in KERNELS:
    sass = subprocess.check_output(["cuobjdump", "-sass", os.path.join(objd, obj)], text=True).splitlines()
    cnt, inside, total = collections.Counter(), False, 0
    for ln in sass:
        if "Function :" in ln:
            inside = sub in ln
            continue
        if not inside:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", ln)
        if m:
            total += 1
            cnt[m.group(2)] += 1
    L.append(f"| {label} | {total} | " + " | ".join(str(cnt.get(k, 0)) for k in FOCUS) + " |")
open(out, "w").write("\n".join(L) + "\n")
print("\n".join(L))
