#!/usr/bin/env python
"""Benchmark of the B200 block ILU(k) hot path -- one JSON line on rank 0.

Step = one preconditioner apply (L y = b, z = D^-1 y, U' x = z) of the
128^3-cell, 3x3-block, ILU(0) synthetic reservoir system (BASELINE.json
configs[2]), with the right-hand side already resident in HBM.  Metric:
algorithmic apply bandwidth in GB/s, B_apply / t:

    B_apply = 8 b^2 (nL + nU + n) + 4 (nL + nU) + 8 (n + 1) + 32 b n

Also reported: e2e (the same metric through the public API from pinned host
memory, copies inside the timed region; and the reference-style
``apply_preconditioner(f, ndarray)`` call as ``e2e.dropin``), solves/s, the
ILU(1) and ILU(2) applies of the same grid, time to solution on every
BASELINE config (GPU) beside the reference's CPU algorithms on this host's
cores, setup time, the roofline of the sweep kernel and the CPU baseline of
the same workload (numpy port of the reference apply, workers = 1 and = all
cores).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun): every rank solves its own independent 128^3 system
(weak scaling, no data-path collective); `value` = total bytes / max-rank time.
The 64-system batch (configs[4]) is sharded over the ranks by
``batch.run_sharded`` (any batch size, seeds = global system index).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--bs", type=int, default=3)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--no-extras", action="store_true", help="skip ILU(2), BiCGSTAB and CPU baseline legs")
    ap.add_argument("--batch", type=int, default=64, help="systems of the batch leg (configs[4]); 0 skips it")
    ap.add_argument("--configs", type=int, default=1, help="time-to-solution on configs[0,1,3] (0 skips)")
    ap.add_argument("--cpu", type=int, default=1, help="CPU legs: 0 none, 1 apply + time to solution, "
                                                       "2 also the 100^3 b8 solve")
    return ap.parse_args()


def apply_bytes(info):
    b, n, nL, nU = info["bs"], info["n"], info["nL"], info["nU"]
    return 8 * b * b * (nL + nU + n) + 4 * (nL + nU) + 8 * (n + 1) + 32 * b * n


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks line).

    NVML is polled from a thread every millisecond (the timed region can be a
    few milliseconds long); nvidia-smi at 50 ms is the fallback.  The NVML
    device is matched to the CUDA device by PCI bus id.
    """

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []          # (sm_mhz, max_mhz, reasons frozenset)
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            h = None
            try:   # CUDA_VISIBLE_DEVICES may renumber devices: match the PCI address
                pr = torch.cuda.get_device_properties(self.index)
                h = nv.nvmlDeviceGetHandleByPciBusId(
                    f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
            except Exception:
                h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (nv, h, nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll_nvml, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read_smi, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def _poll_nvml(self):
        nv, h, mx = self.nvml
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                names = frozenset(n for n, attr in self.REASONS if bits & getattr(nv, attr))
                self.rows.append((float(sm), float(mx), names))
            except Exception:
                return
            time.sleep(0.001)

    def _read_smi(self):
        names = [n for n, _ in self.REASONS]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                act = frozenset(names[i] for i in range(4) if parts[2 + i].lower() == "active")
                self.rows.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit() else None,
                                  act))

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self.thread.join(timeout=1)
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows if r[1]]
        reasons = sorted(set().union(*[r[2] for r in self.rows]))
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml 1 ms" if self.nvml is not None else "nvidia-smi 50 ms"}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_config(args, world):
    """The `config` of the JSON line -- identical for both arms (same workload)."""
    return {"workload": f"ILU({args.k}) apply, {args.nx}^3 cells, {args.bs}x{args.bs} BSR (BASELINE configs[2])",
            "grid": args.nx, "bs": args.bs, "k": args.k,
            "l2": "working set >= 1.3 GB >> 126 MB L2 (no flush needed)",
            "parallelism": f"replicas x{world} (independent systems, no collective)"}


def run_reference(args):
    """--impl reference: the reference's CPU apply (numpy port) on this host's cores, rank 0 only."""
    world, rank, local = dist_setup(args)
    if rank != 0:
        return
    from oracle import cbaseline
    res = cbaseline.measure(args.nx, args.bs, args.k, steps=max(1, args.steps), warmup=max(1, args.warmup))
    line = {
        "impl": "reference", "metric": "ilu_apply_GBps", "value": res["GBps"], "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["ms_per_apply"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY 8d reservoir generator, seed 0)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": res["GBps"], "unit": "GB/s", "cores": res["cores"], "kind": res["kind"],
                         "sample": res["sample"], "rows": res["rows"], "host_cpus": res["host_cpus"]},
        "e2e": {"value": res["GBps"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# BASELINE configs timed to a solution: name -> (grid, bs, k, solver)
CONFIGS = {
    "cfg0_16^3_b3_ILU0_bicgstab": (16, 3, 0, "bicgstab"),
    "cfg1_64^3_b3_ILU1_bicgstab": (64, 3, 1, "bicgstab"),
    "cfg2_128^3_b3_ILU0_bicgstab": (128, 3, 0, "bicgstab"),
    "cfg3_100^3_b4_ILU1_gmres30": (100, 4, 1, "gmres"),
    "cfg3_100^3_b8_ILU1_gmres30": (100, 8, 1, "gmres"),
}


def gpu_time_to_solution(b2, torch, rank):
    """Every BASELINE config on this GPU: setup (build_preconditioner) and the solve
    (b = A 1, x0 = 0, rel tol 1e-6) through the public API with a resident
    DeviceOperator: the median of three solves after one warm solve."""
    runs = {}
    for name, (nxc, bsc, kc, solver) in CONFIGS.items():
        ncf, bsf, rpf, cif, vf = b2.reservoir_block_grid(nxc, nxc, nxc, bsc, seed=rank)
        af = b2.BcsrMatrix(bsf, ncf, ncf, rpf, cif, vf)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ff = b2.build_preconditioner(af, kc)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        op = b2.DeviceOperator(af)
        bb = torch.from_numpy(b2.synthetic.ones_rhs(ncf, bsf, rpf, cif, vf)).cuda()
        cfgf = b2.SolverConfig(restart=30, rel_tol=1e-6)
        solve = b2.bicgstab if solver == "bicgstab" else b2.gmres
        solve(op, bb, M=ff, cfg=cfgf)   # warm (workspace, CUDA graph)
        times = []
        for _ in range(3):   # the median of three timed solves
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            _, stf = solve(op, bb, M=ff, cfg=cfgf)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t2)
        runs[name] = {"solve_s": sorted(times)[1], "solve_s_runs": times, "iterations": stf.iterations,
                      "converged": stf.converged,
                      "true_rel_residual": stf.final_relative_residual, "setup_s": t1 - t0,
                      "engine": ff.info["engine"]}
        del ff, af, bb, op
        torch.cuda.empty_cache()
    return runs


def cpu_time_to_solution(level, gpu_runs):
    """The reference's solves on the host (numpy port operators, workers = 1, its
    fastest mode): full runs for the small configs, the large ones timed over a
    few iterations and projected to the GPU's iteration count (bounded sample)."""
    from oracle import cbaseline
    out = {}
    # the 128^3 system first: the apply baseline just built it (cbaseline keeps the last one)
    for name, (nxc, bsc, kc, solver) in sorted(CONFIGS.items(), key=lambda kv: kv[1][0] != 128):
        if bsc == 8 and level < 2:
            out[name] = {"skipped": "C-oracle setup of 100^3 b8 takes ~70 s (bench.py --cpu 2 runs it)"}
            continue
        its = gpu_runs.get(name, {}).get("iterations")
        sample = None if nxc <= 64 else 2
        try:
            r = cbaseline.time_to_solution(nxc, bsc, kc, solver, its_full=its, max_measured=sample)
        except Exception as exc:   # reported, never fatal
            r = {"failed": str(exc)}
        if name in gpu_runs and "seconds" in r:
            r["gpu_speedup"] = r["seconds"] / gpu_runs[name]["solve_s"]
        out[name] = r
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1703_01325_b200 as b2
    from paper_1703_01325_b200.batch import max_over_ranks

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- build the system and the preconditioner -------------------------
    t0 = time.perf_counter()
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, args.bs, seed=rank)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    t_gen = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = b2.build_preconditioner(a, args.k)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    info = f.info
    B = apply_bytes(info)
    assert B == info["apply_bytes"]
    length = n * bs
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(length)).cuda()
    out = torch.empty_like(rhs)
    stream = torch.cuda.current_stream()
    launches_per_apply = 2 if info["engine"] == 1 else 1   # (permute_b +) the persistent sweep

    # ---------------- device-resident timing ------------------------------------------
    for _ in range(args.warmup):
        b2.apply_preconditioner(f, rhs, out=out)
    f.status()
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            b2.apply_preconditioner(f, rhs, out=out)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    barrier()
    f.status()
    total_ms = ev[0].elapsed_time(ev[-1])
    # the sweep kernel alone (roofline.achieved): CUDA events recorded by the
    # library on the launching stream around the sweep launch of each apply
    f.set_sweep_timing(True)
    kms = []
    for _ in range(args.steps):
        b2.apply_preconditioner(f, rhs, out=out)
        kms.append(f.sweep_ms())
    f.set_sweep_timing(False)
    t_kernel_ms = float(np.mean(kms))
    total_ms = max_over_ranks([total_ms], dist, "cuda")[0]
    ms_per_step = total_ms / args.steps
    value = world * B / (ms_per_step * 1e-3) / 1e9

    # ---------------- e2e through the public API, host buffers -----------------------
    # (1) apply_preconditioner_many: pinned host in / out, copies of consecutive
    #     steps overlapped with the sweeps (the headline e2e);
    # (2) serial: copy in, apply, copy out per step (pinned);
    # (3) dropin: the reference's own call, apply_preconditioner(f, ndarray) ->
    #     ndarray (pageable copies and a status check per call), wall clock.
    e2e_steps = args.steps
    host_k = torch.from_numpy(np.random.default_rng(2).standard_normal((e2e_steps, length))).pin_memory()
    out_k = torch.empty_like(host_k).pin_memory()
    b2.apply_preconditioner_many(f, host_k[:2], out=out_k[:2])   # warm-up
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    b2.apply_preconditioner_many(f, host_k, out=out_k)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    host_in = host_k[0]
    host_out = torch.empty(length, dtype=torch.float64).pin_memory()

    def e2e_step():
        dev_in = host_in.to("cuda", non_blocking=True)
        x = b2.apply_preconditioner(f, dev_in)
        host_out.copy_(x, non_blocking=True)

    for _ in range(2):
        e2e_step()
    barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = e0.elapsed_time(e1) / e2e_steps
    np_in = host_k[0].numpy().copy()
    b2.apply_preconditioner(f, np_in)
    barrier()
    d0 = time.perf_counter()
    for _ in range(e2e_steps):
        b2.apply_preconditioner(f, np_in)
    dropin_ms = (time.perf_counter() - d0) * 1e3 / e2e_steps
    e2e_ms, e2e_serial_ms, dropin_ms = max_over_ranks([e2e_ms, e2e_serial_ms, dropin_ms], dist, "cuda")
    e2e_val = world * B / (e2e_ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = B / (t_kernel_ms * 1e-3) / 1e9
    if info["engine"] == 1:
        kernel_name = f"psweep_kernel<{bs}> (partitioned L and U' sweeps, one persistent launch, {info['parts']} parts)"
    else:
        kernel_name = f"sweep_kernel<{bs}> (tiled level-order L and U' sweeps, one persistent launch)"
    # DRAM bytes per launch of that kernel from the committed ncu --set full capture (profiles/)
    traffic, traffic_src = None, None
    try:
        tab = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        key = f"{kernel_name.split(' ')[0]} {args.nx}^3 k{args.k}"
        if key in tab:
            traffic, traffic_src = tab[key]["bytes"], tab[key]["source"]
    except (OSError, ValueError, KeyError):
        pass

    extras = {}
    if not args.no_extras:
        # the other fill levels of the same grid (configs[2] "ILU(0) and ILU(2)")
        for kk in (1, 2):
            if kk == args.k:
                continue
            t0 = time.perf_counter()
            f2 = b2.build_preconditioner(a, kk)
            torch.cuda.synchronize()
            s2 = time.perf_counter() - t0
            B2 = apply_bytes(f2.info)
            for _ in range(3):
                b2.apply_preconditioner(f2, rhs, out=out)
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(stream)
            for _ in range(10):
                b2.apply_preconditioner(f2, rhs, out=out)
            q1.record(stream)
            torch.cuda.synchronize()
            f2.status()
            ms2 = q0.elapsed_time(q1) / 10
            extras[f"ilu{kk}_apply"] = {"GBps": B2 / (ms2 * 1e-3) / 1e9, "ms": ms2, "bytes": B2,
                                        "frac_of_measured_hbm": B2 / (ms2 * 1e-3) / 1e9 / peak, "setup_s": s2,
                                        "levels": [f2.info["levels_L"], f2.info["levels_U"]],
                                        "engine": f2.info["engine"], "sweep_warps": f2.info["sweep_warps"]}
            del f2

    gpu_runs = {}
    if not args.no_extras and args.configs:
        del f
        torch.cuda.empty_cache()
        gpu_runs = gpu_time_to_solution(b2, torch, rank)
        extras["configs"] = gpu_runs

    if not args.no_extras and args.batch > 0:
        # BASELINE configs[4]: a batch of independent 64^3 b3 systems, ILU(1),
        # sharded over the ranks (batch.run_sharded: any batch size, system i
        # generated with seed i); a rank applies its share as ONE
        # block-diagonal operator, so their level chains interleave in one
        # persistent sweep, then solves them with the batched BiCGSTAB
        from paper_1703_01325_b200.batch import SystemResult, run_sharded
        shape = {}

        def solve_local(indices):
            if not indices:
                return [], {"apply_ms": 0.0, "solve_s": 0.0, "setup_s": 0.0, "gen_s": 0.0}
            g0 = time.perf_counter()
            mats = []
            for sidx in indices:
                nb_, bs_, rp_, ci_, v_ = b2.reservoir_block_grid(64, 64, 64, args.bs, seed=sidx)
                mats.append(b2.BcsrMatrix(bs_, nb_, nb_, rp_, ci_, v_))
            big = b2.block_diagonal(mats)
            del mats
            g1 = time.perf_counter()
            fb = b2.build_preconditioner(big, 1)
            torch.cuda.synchronize()
            g2 = time.perf_counter()
            shape["bytes"] = apply_bytes(fb.info)
            shape["engine"] = fb.info["engine"]
            rb = torch.from_numpy(np.random.default_rng(1).standard_normal(big.shape[0])).cuda()
            ob = torch.empty_like(rb)
            for _ in range(3):
                b2.apply_preconditioner(fb, rb, out=ob)
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(stream)
            for _ in range(5):
                b2.apply_preconditioner(fb, rb, out=ob)
            q1.record(stream)
            torch.cuda.synchronize()
            fb.status()
            msb = q0.elapsed_time(q1) / 5
            opb = b2.DeviceOperator(big)
            bb = opb.matvec(torch.ones(big.shape[0], dtype=torch.float64, device="cuda"))
            torch.cuda.synchronize()
            s0 = time.perf_counter()
            _, stb = b2.bicgstab_batched(opb, bb, M=fb, cfg=b2.SolverConfig(rel_tol=1e-6))
            torch.cuda.synchronize()
            solve_b = time.perf_counter() - s0
            res = [SystemResult(i, rank, s.iterations, s.converged, s.final_relative_residual, 0.0, solve_b)
                   for i, s in zip(indices, stb)]
            del fb, big, rb, ob, opb, bb
            torch.cuda.empty_cache()
            return res, {"apply_ms": msb, "solve_s": solve_b, "setup_s": g2 - g1, "gen_s": g1 - g0}

        barrier()
        allres, tb = run_sharded(args.batch, solve_local, dist, "cuda")
        its_b = [r.iterations for r in allres]
        per_rank = -(-args.batch // world)
        extras["batch_apply"] = {
            "workload": f"{args.batch} x 64^3 b{args.bs} ILU(1), up to {per_rank} per GPU as one block-diagonal "
                        f"operator", "ms": tb["apply_ms"],
            "GBps_aggregate": (shape.get("bytes", 0) * world) / (tb["apply_ms"] * 1e-3) / 1e9
            if tb["apply_ms"] else None,
            "frac_of_measured_hbm_per_gpu": shape.get("bytes", 0) / (tb["apply_ms"] * 1e-3) / 1e9 / peak
            if tb["apply_ms"] else None,
            "system_applies_per_s": args.batch / (tb["apply_ms"] * 1e-3) if tb["apply_ms"] else None,
            "setup_s": tb["setup_s"], "gen_s": tb["gen_s"], "engine": shape.get("engine"),
            "bicgstab": {"solve_s": tb["solve_s"], "systems_per_s": args.batch / tb["solve_s"],
                         "systems": len(allres), "iterations_min": min(its_b), "iterations_max": max(its_b),
                         "all_converged": all(r.converged for r in allres), "rel_tol": 1e-6,
                         "note": "batched BiCGSTAB, b = A 1 per system, time = max over ranks"}}

    cpu = None
    if rank == 0 and not args.no_extras and args.cpu:
        from oracle import cbaseline
        try:
            r = cbaseline.measure(args.nx, args.bs, args.k, steps=3, warmup=1)
            cpu = {"value": r["GBps"], "unit": "GB/s", "cores": r["cores"], "kind": r["kind"], "sample": r["sample"],
                   "rows": r["rows"], "host_cpus": r["host_cpus"], "host": r["host"],
                   "gpu_speedup": value / world / r["GBps"]}
        except Exception as exc:   # reported, never fatal
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}
        extras["cpu_time_to_solution"] = cpu_time_to_solution(args.cpu, gpu_runs)

    if rank == 0:
        line = {
            "metric": "ilu_apply_GBps", "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY 8d reservoir generator, seed = rank)",
            "config": workload_config(args, world),
            "system": {"n_block_rows": n, "nL": info["nL"], "nU": info["nU"],
                       "levels": [info["levels_L"], info["levels_U"]], "bytes_per_apply": B},
            "solves_per_s": world / (ms_per_step * 1e-3),
            "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": 8 * length,
                    "d2h_bytes_per_step": 8 * length, "ms_per_step": e2e_ms, "steps": e2e_steps,
                    "api": "apply_preconditioner_many (pinned host in/out, transfers overlapped with the sweeps)",
                    "serial": {"value": world * B / (e2e_serial_ms * 1e-3) / 1e9, "ms_per_step": e2e_serial_ms,
                               "api": "apply_preconditioner per step, copies and sweep in sequence"},
                    "dropin": {"value": world * B / (dropin_ms * 1e-3) / 1e9, "ms_per_step": dropin_ms,
                               "api": "apply_preconditioner(f, numpy array) -> numpy array (the reference's "
                                      "call), wall clock"}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel_ms": t_kernel_ms, "kernel_share_of_step": t_kernel_ms / ms_per_step,
                         "step_frac": B / (ms_per_step * 1e-3) / 1e9 / peak,
                         "kernel": kernel_name,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if peaks else "fallback 6650",
                         "traffic_source": traffic_src},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": args.steps * launches_per_apply,
            "setup_s": t_setup, "gen_s": t_gen,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
