#!/usr/bin/env python
"""Benchmark: element-direction local solves / s per full all-ordinate sweep (FP64).

Contract (see task spec / DESIGN.md §7):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]
One "step" = one full sweep of every (element, ordinate) pair of the workload
(SweepSolver::sweep for all ordinates, solver.hpp:98-117) with the scattering
source rebuilt from the resident phi.  Inputs (psi, 2 x 4.3 GB at C4) exceed the
126 MB L2, so no flush is needed between steps.  Rank 0 prints ONE JSON line.

  value      whole-job solves/s, device-resident inputs, CUDA events on the
             library's stream, max over ranks
  e2e        same metric through the reference-facing C ABI call hsw_sweep(d=-1)
             with pinned HOST buffers: H2D psi_old+phi and D2H psi_new inside
             the timed region
  roofline   dominant kernel (the sweep kernel, one launch per level): LU-algorithmic
             FP64 FLOPs F(n) = 2/3 n^3 + 2 n^2 per solve / kernel time, against
             the FP64 peak measured in-run (DFMA microbenchmark)
  cpu_baseline  the CPU oracle (port of the reference algorithm) on the host
             cores, bounded sample of the same workload
--impl reference times the CPU oracle port alone (the reference itself cannot
be built here: Eigen/Catch2/CLI11 are absent) on the same config/metric.
Multi-GPU (N > 1): the ordinates are sharded over the ranks
(paper_1810_11080_b200/sharded.py); one step = every rank sweeps its ordinate
block and phi is formed by the chained prefix in ordinate order + broadcast over
NCCL (bit-identical to one GPU).  value = all pairs / max-over-ranks step time
("strong" scaling: the job is fixed).  --sharded forces this path at N = 1.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_TEXT = {
    "c1": "2D twisted-quad 8x8 Q2, 16 directions (configs[0])",
    "c2": "2D twisted-quad 128x128 Q3, 64 directions (configs[1])",
    "c3": "3D twisted-hex 16^3 Q2, 128 directions (configs[2])",
    "c4": "3D twisted-hex 32^3 Q3, 256 directions (configs[3], production size)",
    "c5": "3D twisted-hex 24^3 Q4, 256 directions (configs[4], stress case)",
}
METRIC = "element-direction local solves/s per full sweep (FP64); % of FP64/HBM roofline"
UNIT = "solves/s"


def flops_per_solve(n: int) -> float:
    return 2.0 / 3.0 * n ** 3 + 2.0 * n * n


class _DevView:
    """Raw device pointer as a torch-importable array (__cuda_array_interface__)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        under = [v for v in sm if v > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(under) if under else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_sample(prob, budget_s: float, threads: int):
    """Time the CPU oracle (port of the reference algorithm) on a bounded sample."""
    import numpy as np
    import oracle as O
    os.environ["HOSWEEP_THREADS"] = str(threads)
    nd = prob.num_ordinates
    ds = list(range(0, nd, max(1, nd // threads)))[:threads]
    t0 = time.time()
    orc = O.OracleSolver(prob, cache_lu=False, check_rcond=False, validate=False, active=ds)
    setup = time.time() - t0
    phi = np.full(prob.num_dofs, 0.1)
    # calibrate on a small sample, then run ~budget_s of work
    t0 = time.time()
    n0 = orc.sweep_sample(ds, 16, phi)
    dt0 = max(time.time() - t0, 1e-3)
    per_solve = dt0 / max(n0, 1)
    elems = int(max(16, min(prob.num_elements, budget_s / per_solve / len(ds))))
    t0 = time.time()
    n = orc.sweep_sample(ds, elems, phi)
    dt = time.time() - t0
    return {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(ds)} ordinates x first {elems} elements of each sweep order "
                      f"({n} solves, {dt:.1f} s; oracle setup {setup:.1f} s excluded), "
                      f"on-the-fly local assembly + partial-pivot LU, psi_old = 0; oracle built with "
                      f"g++ -O3 -std=c++20 -ffp-contract=off -pthread (oracle/Makefile), {threads} worker threads",
            "seconds": dt, "solves": n}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1810_11080_b200 import problem as pb
    prob = pb.config(args.config)
    threads = os.cpu_count() or 1
    steps = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_sample(prob, args.cpu_budget, threads)
        if i >= args.warmup:
            steps.append(cb)
    val = statistics.median(s["value"] for s in steps)
    pairs = prob.num_elements * prob.num_ordinates
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": pairs / val * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json configs)",
        "config": {"workload": f"{args.config}: {CONFIG_TEXT[args.config]}", "pairs": pairs,
                   "n": prob.block_size},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": cb["sample"]},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference is a 2D-only Eigen header library (SPEC.md:11): its own solver path is "
                "compiled here against an Eigen-subset shim (oracle/_ref, the parity pin) but cannot run this "
                "3D config; the CPU oracle port of its algorithm (3D-generalised, same arithmetic) is timed "
                "(ms_per_step extrapolated to a full sweep)",
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import paper_1810_11080_b200 as pk
    from paper_1810_11080_b200 import _capi
    from paper_1810_11080_b200 import problem as pb
    import ctypes as C

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    L = _capi.load()

    peak = C.c_double(0.0)
    rc = L.hsw_fp64_peak(local, C.byref(peak))
    fp64_peak = peak.value if rc == 0 else None

    prob = pb.config(args.config)
    t0 = time.time()
    shard = None
    if world > 1:   # a rank builds and holds only its ordinate block (plans, worklists, psi)
        from paper_1810_11080_b200.sharded import block_of as _block_of
        shard = _block_of(prob.num_ordinates, rank, world)
    solver = pk.SweepSolver(prob, device=local, ordinate_range=shard)
    setup_s = time.time() - t0
    h = solver.handle
    pairs = prob.num_elements * prob.num_ordinates
    n = prob.block_size
    stream = torch.cuda.ExternalStream(L.hsw_stream(h), device=torch.device("cuda", local))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # resident state: non-trivial phi (scattering source active), psi_old = 0
    phi0 = np.full(prob.num_dofs, 0.1)
    assert L.hsw_set_state(h, C.c_void_p(phi0.ctypes.data), None) == 0, _capi.last_error()
    torch.cuda.synchronize()

    sharded = world > 1 or args.sharded
    if sharded:
        from paper_1810_11080_b200.sharded import DeviceShardBackend, block_of
        be = DeviceShardBackend(solver)
        d0, d1 = block_of(prob.num_ordinates, rank, world)
        phi_t = torch.full((prob.num_dofs,), 0.1, dtype=torch.float64, device=f"cuda:{local}")

        def step():
            # one source-iteration data path: block sweep + chained phi (sharded.py)
            be.sweep(d0, d1, phi_t)
            prefix = None
            if world > 1 and rank > 0:
                prefix = be.zeros()
                torch.distributed.recv(prefix, src=rank - 1)
            out = be.zeros()
            be.phi_partial(d0, d1, prefix, out)
            if world > 1:
                if rank < world - 1:
                    torch.distributed.send(out, dst=rank + 1)
                torch.distributed.broadcast(out, src=world - 1)
            return L.hsw_last_launch_count(h) + 1
    else:
        def step():
            rc = L.hsw_sweep_resident(h)
            assert rc == 0, _capi.last_error()
            return L.hsw_last_launch_count(h)

    for _ in range(args.warmup):
        step()
        assert L.hsw_synchronize(h) == 0, _capi.last_error()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    launches_per_step = 0
    ev0.record(stream)
    for _ in range(args.steps):
        launches_per_step = step()
    if sharded:   # the last broadcast runs on torch's stream: close the span after it
        torch.cuda.current_stream().synchronize()
    ev1.record(stream)
    torch.cuda.synchronize()
    rc = L.hsw_synchronize(h)
    assert rc == 0, _capi.last_error()
    barrier()
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    # kernel-only time of one sweep (events around the sweep-kernel launches)
    for _ in range(2):
        if sharded:
            be.sweep(d0, d1, phi_t)
        else:
            L.hsw_sweep_resident(h)
        L.hsw_synchronize(h)
        kernel_ms.append(L.hsw_last_sweep_kernel_ms(h))
    kms = min(kernel_ms)
    ms_step = ms_total / args.steps
    if world > 1:
        t = torch.tensor([ms_step, kms], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_step, kms = float(t[0].item()), float(t[1].item())
    value = pairs / (ms_step * 1e-3)

    # ---- end-to-end through the reference-facing ABI call with pinned host buffers
    e2e = None
    if not args.skip_e2e:
        N = prob.num_dofs
        nd = prob.num_ordinates
        vp = C.c_void_p
        if sharded:
            # per rank: H2D of its psi_old block + phi, block sweep + phi chain, D2H of its psi_new block
            pa, pb_, ph = C.c_void_p(), C.c_void_p(), C.c_void_p()
            assert L.hsw_device_state(h, C.byref(pa), C.byref(pb_), C.byref(ph)) == 0
            nb = d1 - d0
            phi_h = torch.full((N,), 0.1, dtype=torch.float64).pin_memory()
            psi_old_h = torch.zeros((nb, N), dtype=torch.float64).pin_memory()
            psi_new_h = torch.empty((nb, N), dtype=torch.float64).pin_memory()
            vp = C.c_void_p

            def e2e_step():
                # block sweep with host buffers (H2D / sweep / D2H pipelined over sub-blocks),
                # then the chained phi over the ranks as in step()
                rc = L.hsw_shard_sweep_host(h, d0, d1, vp(phi_h.data_ptr()), vp(psi_old_h.data_ptr()),
                                            vp(psi_new_h.data_ptr()))
                assert rc == 0, _capi.last_error()
                prefix = None
                if world > 1 and rank > 0:
                    prefix = be.zeros()
                    torch.distributed.recv(prefix, src=rank - 1)
                out = be.zeros()
                be.phi_partial(d0, d1, prefix, out)
                if world > 1:
                    if rank < world - 1:
                        torch.distributed.send(out, dst=rank + 1)
                    torch.distributed.broadcast(out, src=world - 1)
                torch.cuda.current_stream().synchronize()

            e2e_step()
            e2e_steps = max(1, min(args.steps, 3))
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                e2e_step()
            barrier()
            e2e_s = (time.perf_counter() - t0) / e2e_steps
            h2d, d2h = (nd * N + world * N) * 8, nd * N * 8
            api = "per rank: hsw_shard_sweep_host (psi_old block + phi H2D, pipelined block sweep, psi_new block D2H) + chained phi (NCCL)"
        else:
            # (a) the call a user makes: SweepSolver.sweep(-1, phi, psi_old) with ordinary
            # (pageable) numpy arrays; it returns a fresh psi_new array every call, as the
            # reference's sweep returns its VectorXd by value (solver.hpp:98).  The library
            # streams pageable memory through its pinned staging ring.
            # Two ordinary numpy arrays alternate as psi_old / out (the source-iteration pattern);
            # a FRESH result array per call is timed too (the OS first-touch faults of a new
            # 4.3 GB array: the reference's return-by-value pays them as well).
            phi_np = np.full(N, 0.1)
            psi_a = np.zeros((nd, N))
            psi_b = np.zeros((nd, N))
            psi_a.fill(0.0)   # resident pages: the arrays an iteration loop reuses
            psi_b.fill(0.0)
            solver.sweep(-1, phi_np, psi_a, out=psi_b)   # warm-up (staging ring, worklists)
            e2e_steps = max(1, min(args.steps, 3))
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                solver.sweep(-1, phi_np, psi_a, out=psi_b)
                psi_a, psi_b = psi_b, psi_a
            barrier()
            e2e_s = (time.perf_counter() - t0) / e2e_steps
            del psi_b
            t0 = time.perf_counter()
            fresh = solver.sweep(-1, phi_np, psi_a)
            fresh_s = time.perf_counter() - t0
            del psi_a, fresh
            # (b) the C ABI call with caller-pinned buffers (copy engines straight from host memory)
            phi_h = torch.full((N,), 0.1, dtype=torch.float64).pin_memory()
            psi_old_h = torch.zeros((nd, N), dtype=torch.float64).pin_memory()
            psi_new_h = torch.empty((nd, N), dtype=torch.float64).pin_memory()
            rc = L.hsw_sweep(h, -1, vp(phi_h.data_ptr()), vp(psi_old_h.data_ptr()), vp(psi_new_h.data_ptr()))
            assert rc == 0, _capi.last_error()
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                rc = L.hsw_sweep(h, -1, vp(phi_h.data_ptr()), vp(psi_old_h.data_ptr()), vp(psi_new_h.data_ptr()))
                assert rc == 0, _capi.last_error()
                psi_old_h, psi_new_h = psi_new_h, psi_old_h
            barrier()
            pinned_s = (time.perf_counter() - t0) / e2e_steps
            h2d, d2h = (nd * N + N) * 8, nd * N * 8
            api = ("SweepSolver.sweep(-1, phi, psi_old, out=) with ordinary pageable numpy arrays (library-side "
                   f"pinned staging ring); with a fresh result array per call: {pairs / fresh_s:.4g} solves/s, "
                   f"{fresh_s * 1e3:.1f} ms; caller-pinned hsw_sweep(h, -1, ...): {pairs / pinned_s:.4g} solves/s, "
                   f"{pinned_s * 1e3:.1f} ms")
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": pairs / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_s * 1e3, "api": api}
        del phi_h, psi_old_h, psi_new_h

    # ---- roofline of the dominant kernel (the sweep kernel)
    pairs_rank = pairs if not sharded else prob.num_elements * (d1 - d0)
    achieved = flops_per_solve(n) * pairs_rank / (kms * 1e-3) * 1e-12
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            if "dram_bytes_per_sweep" in tj:   # ncu over a whole sweep, per sweep-kernel launch
                traffic = tj["dram_bytes_per_sweep"] * (pairs_rank / pairs) / max(launches_per_step - 1, 1)
            elif "dram_bytes_per_pair" in tj:   # ncu capture of one level, scaled to the average launch
                traffic = tj["dram_bytes_per_pair"] * pairs_rank / max(launches_per_step - 1, 1)
            else:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": (achieved / fp64_peak) if fp64_peak else None, "traffic": traffic,
                "peak_source": "measured in-run: DFMA-chain microbenchmark over all SMs "
                               "(MEASURED_PEAKS.json has no FP64 figure)",
                "flops_per_solve": flops_per_solve(n), "kernel_ms_per_sweep": kms,
                "kernel_launches_per_sweep": launches_per_step - 1}

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        try:
            cpu = cpu_sample(prob, args.cpu_budget, os.cpu_count() or 1)
            cpu.pop("seconds", None)
            cpu.pop("solves", None)
        except Exception as ex:  # the baseline is reported, never the product
            cpu = {"value": None, "unit": UNIT, "error": str(ex)[:200]}

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong",   # total work fixed as N grows (ordinates sharded over ranks)
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json configs, seeded)",
            "config": {"workload": f"{args.config}: {CONFIG_TEXT[args.config]}", "pairs": pairs, "n": n,
                       "levels": solver.num_levels, "l2": "inputs larger than L2 (psi 2 x "
                       f"{prob.num_ordinates * prob.num_dofs * 8 / 1e9:.2f} GB)",
                       "parallelism": (f"ordinate-sharded x{world}: block [{d0}, {d1}) on rank 0, chained phi over "
                                       f"{'NCCL' if world > 1 else 'one rank'}") if sharded else "1 GPU",
                       "setup_s": round(setup_s, 2)},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
            "gpu_launches": int(launches_per_step * args.steps),
        }
    solver.close()
    if rank == 0 and world == 1 and not args.skip_per_config:
        line["per_config"] = per_config_report(fp64_peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def per_config_report(fp64_peak):
    """Every BASELINE.json config at full size, timed in this run on this GPU: one
    all-ordinate sweep (device-resident, best of 3 after 2 warm-ups; kernel time by
    CUDA events on the library stream) and source iteration from psi = phi = 0 to
    ||dphi||_2 / ||phi||_2 < 1e-8 (hsw_source_iteration, device time)."""
    import paper_1810_11080_b200 as pk
    from paper_1810_11080_b200 import _capi
    from paper_1810_11080_b200 import problem as pb
    L = _capi.load()
    out = {}
    for name in ("c1", "c2", "c3", "c4", "c5"):
        try:
            t0 = time.time()
            prob = pb.config(name)
            s = pk.SweepSolver(prob, options=pk.SolveOptions(tolerance=1e-8, criterion="phi_rel_l2"))
            setup = time.time() - t0
            for _ in range(2):
                assert L.hsw_sweep_resident(s.handle) == 0 and L.hsw_synchronize(s.handle) == 0, _capi.last_error()
            ms = []
            for _ in range(3):
                assert L.hsw_sweep_resident(s.handle) == 0 and L.hsw_synchronize(s.handle) == 0, _capi.last_error()
                ms.append(L.hsw_last_sweep_kernel_ms(s.handle))
            m = min(ms)
            pairs = prob.num_elements * prob.num_ordinates
            n = prob.block_size
            state, hist = s.source_iteration(return_psi=False)
            tf = flops_per_solve(n) * pairs / (m * 1e-3) * 1e-12
            out[name] = {"sweep_ms": round(m, 3), "solves_per_s": pairs / (m * 1e-3), "tflops_lu_alg": round(tf, 3),
                         "roofline_frac": round(tf / fp64_peak, 4) if fp64_peak else None,
                         "si_iterations": hist.iterations(), "si_converged": hist.converged,
                         "si_s": round(hist.seconds, 3), "setup_s": round(setup, 2), "pairs": pairs, "n": n,
                         # redone calls with the pivoted kernel: 0 = the static-pivot tile LU ran throughout
                         "pivot_fallbacks": int(L.hsw_pivot_fallbacks(s.handle))}
            s.close()
        except Exception as ex:   # report, do not lose the main line
            out[name] = {"error": str(ex)[:200]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIG_TEXT))
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="ordinate-sharded step even at N = 1")
    ap.add_argument("--skip-per-config", action="store_true", help="no per-config sweep / SI report")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no launcher: start one rank per GPU ourselves (the same command the driver uses)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus and args.impl == "ours":
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE', '1')}"}))
        return 1
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
