#!/usr/bin/env python
"""Benchmark of the B200 SWR hot path (driver contract).

One *step* = one pass of the whole hot path on resident inputs:
swr_build_interface_operator (one batched march of the 3N-2 systems: d and
the l_j / r_j impulse probes giving L) + swr_solve (GMRES on (I-L)g = d and
the final sweep, Algorithm 3).  Workload (N=1): BASELINE.json
configs[4] at N = 500 (C5), the north_star's 500-subdomain configuration:
V = -x^2, Gaussian u0, (a0,b0) = (-21,21), dx = 1e-5, dt = 1e-3, T = 0.5,
S0^2 transmission, zero g0.

metric: subdomain cell-steps per second over the whole time-to-solution
(cell-steps = sum over marches of sum_j N_j * N_T * RHS); ms_per_step is the
time to solution.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
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

import numpy as np  # noqa: E402

import swr_inputs as si  # noqa: E402

METRIC = "SWR time-to-solution; subdomain cell-steps/s and % of HBM roofline"
UNIT = "cell-steps/s"
PAPER_T_NEW_GMRES_N500_S = 6.86      # 500 Sandy Bridge cores
FLOP_PER_CELL_STEP = 36.0            # algorithmic flops of one CN cell-step
BYTES_PER_CELL_STEP = 32.0           # u_{n-1} read + u_n write, complex fp64
STREAM2_BYTES_PER_CELL_STEP = 136.0  # k_march_stream2: u, q, Re E, z, Apre, b traffic per row-step
RESIDENT_MAX_ROWS = 16 * 256 * 11    # N_j above this: the streaming marches
FP64_DERIVED_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: 148 SMs x 64 DFMA/clk at 1965 MHz
FP64_PROBE = os.path.join(ROOT, "profiles", "r02", "probe_fp64_b200.txt")


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def fp64_peak():
    """Measured DFMA throughput on this pool's B200 (tools/probe_fp64.cu,
    committed output), else the derived unit-count figure."""
    try:
        vals = [float(l.split(":")[1].split()[0]) for l in open(FP64_PROBE) if l.startswith("dfma tput")]
        return max(vals), "measured: tools/probe_fp64.cu DFMA throughput on a B200 of this pool " \
                          "(profiles/r02/probe_fp64_b200.txt)"
    except Exception:
        return FP64_DERIVED_TFLOPS, "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(1)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        under = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def oracle_time_to_solution(p, arrays, threads: int):
    """The oracle as it stands on `threads` host threads (subdomain-parallel
    loops, bitwise equal to one thread): the whole time-to-solution of the
    workload -- build of d and L, every GMRES iteration, the final sweep."""
    from oracle import oracle
    oracle.set_threads(threads)
    try:
        t0 = time.perf_counter()
        r = oracle.Oracle(p, arrays).solve()
        dt = time.perf_counter() - t0
    finally:
        oracle.set_threads(1)
    return dt, r


def run_reference(args, p, arrays):
    """--impl reference: the CPU oracle on the host cores (rank 0 only).  One
    step = one sweep R(0; u0) of the workload (every subdomain marches once:
    N N_j N_T cell-steps), the oracle's subdomain-parallel march on all
    cores; the same unit the GPU's cell-steps/s counts."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle
    P = os.cpu_count() or 1
    oracle.set_threads(P)
    o = oracle.Oracle(p, arrays)
    times, cells = [], 0
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        o.apply_R(None, use_u0=True)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
            cells += p.N * p.Nj * p.NT
    total = sum(times)
    value = cells / total
    sample = (f"oracle or_apply_R(0; u0) of the whole {p.name} workload per step ({p.N} subdomain marches, "
              f"N_j={p.Nj}, N_T={p.NT}) on {P} threads (subdomain-parallel, bitwise equal to one thread)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(workload_config(p), parallelism=f"{P} host threads",
                                                l2="n/a (CPU oracle)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


POT_NAME = {si.POT_ZERO: "V=0", si.POT_VX: "V=-x^2", si.POT_VTX: "V=5tx", si.POT_CUBIC: "f(u)=|u|^2"}
ALG_NAME = {si.ALG_NEW: "NEW", si.ALG_PRECOND: "PRECOND", si.ALG_CLASSICAL: "CLASSICAL"}
KRY_NAME = {si.KRY_GMRES: "GMRES(30)", si.KRY_BICGSTAB: "BiCGStab", si.KRY_FIXED_POINT: "fixed point"}


def workload_config(p):
    gs = "CGS" if p.gs_passes == 1 else "CGS2"
    return {"workload": f"{p.name}: {POT_NAME[p.potential]} {ALG_NAME[p.algorithm]}+{KRY_NAME[p.krylov]} {gs}, "
                        f"N={p.N}, dx={p.dx:g}, dt={p.dt:g}, T={p.T:g}, "
                        f"{'S0^2' if p.transmission == si.TC_S02 else 'Robin'}, {p.u0_kind} u0, zero g0"
                        + (" (BASELINE configs[4] at N=500)" if p.name == "C5" else ""),
            "N_subdomains": p.N, "N_x": p.Nx, "N_T": p.NT, "N_j": p.Nj,
            "cell_steps_per_step": (3 * p.N - 2 + p.N) * p.Nj * p.NT,
            "parallelism": None, "l2": "flushed before every timed step (256 MiB write)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3 / C4 time-to-solution keys")
    args = ap.parse_args()

    p = si.config(args.config)
    arrays = si.inputs(p)
    if args.impl == "reference":
        run_reference(args, p, arrays)
        return

    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    from paper_1503_02564_b200 import SWR
    from paper_1503_02564_b200.swr import nccl_unique_id
    stream = torch.cuda.Stream(dev)
    nid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        nid = obj[0]
    s = SWR(p, arrays, device=local, stream=stream, rank=rank, world=world, nccl_id=nid)
    uT_dev = torch.empty(p.Nx + 1, dtype=torch.complex128, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def one_step(out):
        s.build()
        return s.solve(out=out)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one_step(uT_dev)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        sampler = ClockSampler(local)
        sampler.start()
        evs = []
        reps = []
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st, _, rep = one_step(uT_dev)
            e1.record(stream)
            evs.append((e0, e1))
            reps.append(rep)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - wall0
        if world > 1:
            torch.distributed.barrier()
        clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = sum(step_ms) / len(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    cells = statistics.mean(r["cell_steps"] for r in reps)
    if world > 1:
        tc = torch.tensor([cells], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tc)
        cells = float(tc.item())
    value = cells / (ms / 1e3)
    t_march = statistics.mean(r["t_march_ms"] for r in reps)
    t_intf = statistics.mean(r["t_interface_ms"] for r in reps)
    t_comm = statistics.mean(r["t_comm_ms"] for r in reps)
    n_march = reps[0]["n_marches"]
    launches = sum(r["n_kernel_launches"] for r in reps)
    iters = reps[-1]["iterations"]
    cells_rank = statistics.mean(r["cell_steps"] for r in reps)
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs", 6538.6)
    fp64, fp64_src = fp64_peak()

    # roofline of the dominant kernel class (the march): FP64-ALU / latency
    # bound (state register-resident for the whole window)
    march_flops = FLOP_PER_CELL_STEP * cells_rank
    achieved = march_flops / (t_march / 1e3) / 1e12
    roof = {"bound": "alu", "kernel": "k_march_resident", "achieved": achieved, "peak": fp64,
            "unit": "TFLOP/s", "frac": achieved / fp64, "traffic": None, "peak_source": fp64_src,
            "algorithmic": f"{FLOP_PER_CELL_STEP:g} flop/cell-step x {cells_rank:.4g} cell-steps over {n_march} launches",
            "avg_launch_ms": t_march / max(n_march, 1)}
    prof = os.path.join(ROOT, "profiles", "march_traffic.json")
    if os.path.exists(prof):
        try:
            roof["traffic"] = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            pass
    hbm_equiv = BYTES_PER_CELL_STEP * cells_rank / (t_march / 1e3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong",   # the C5 workload is fixed; N GPUs share its subdomains
            "vs_baseline": value / (cells / PAPER_T_NEW_GMRES_N500_S) if args.config == "C5" else None,
            "dtype": "f64", "data": "synthetic", "config": workload_config(p),
            "time_to_solution_ms": ms, "gmres_iterations": iters,
            # the BASELINE metric's "% of HBM roofline": the bandwidth a streaming march
            # would need (32 B per cell-step) over the measured HBM peak; the resident
            # march moves ~1/1000 of that through DRAM (profiles/march_traffic.json)
            "streaming_equiv_bw_frac": hbm_equiv / hbm,
            "breakdown_ms": {"march": t_march, "toeplitz": t_intf, "comm": t_comm,
                             "krylov_vector_and_host": ms - t_march - t_intf - t_comm,
                             "setup_once": reps[-1]["t_setup_ms"]},
            "roofline": roof, "gpu_launches": launches, "clocks": clocks, "wall_s_timed": wall}
    line["config"]["parallelism"] = (f"subdomains and their interface slots sharded over {world} GPUs (owner "
                                     f"computes); cut traces by ncclSend/Recv, per-subdomain Gram-Schmidt partials "
                                     f"by ncclAllReduce" if world > 1 else "1 GPU")
    # the interface operator (I - L)x: FFT convolution (N_T <= 512), HBM-bound;
    # algorithmic bytes per apply = x + the transformed first columns + y
    nf = 1 << (2 * next(l for l in range(2, 6) if (1 << (2 * l)) >= 2 * p.NT - 1))
    n_apply = iters + -(-iters // p.restart) + 1
    bytes_apply = 16 * (2 * p.ng + (4 * (p.N - 2) + 2) * nf)
    if t_intf > 0:
        ach = bytes_apply / (t_intf / 1e3 / n_apply) / 1e9
        line["roofline_interface"] = {"bound": "hbm", "kernel": "k_fft_conv_reg (register four-step FFT convolution)", "achieved": ach,
                                      "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                                      "algorithmic": f"{bytes_apply} B per apply x {n_apply} applies"}
    # e2e: host buffers through the public API, H2D of the inputs and D2H of u(T)
    if not args.no_e2e:
        pin_u0 = torch.from_numpy(arrays["u0"]).pin_memory()
        pin_vx = torch.from_numpy(arrays["V_x"]).pin_memory() if arrays["V_x"] is not None else None
        out_h = torch.empty(p.Nx + 1, dtype=torch.complex128).pin_memory()
        with torch.cuda.stream(stream):
            s.update_inputs(u0=pin_u0, V_x=pin_vx, on_device=False)
            one_step(out_h.numpy())
            torch.cuda.synchronize(dev)
            e_ms = []
            for _ in range(max(1, min(args.steps, 3))):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                s.update_inputs(u0=pin_u0, V_x=pin_vx, on_device=False)
                one_step(out_h.numpy())
                e1.record(stream)
                e1.synchronize()
                e_ms.append(e0.elapsed_time(e1))
        em = sum(e_ms) / len(e_ms)
        bi = pin_u0.numel() * 16 + (pin_vx.numel() * 8 if pin_vx is not None else 0)
        line["e2e"] = {"value": cells / (em / 1e3), "unit": UNIT, "h2d_bytes_per_step": bi,
                       "d2h_bytes_per_step": out_h.numel() * 16, "ms_per_step": em,
                       "path": "swr_update_inputs(host u0, V_x) + swr_build_interface_operator + swr_solve(host u_T)"}

    # the other BASELINE configs' time-to-solution: C2
    # V(x) NEW + GMRES at N = 10 (the streaming march, N_j = 420,001), C3 V(t,x)
    # preconditioned GMRES, C4 |u|^2 preconditioned fixed point
    if not args.no_extra and world == 1:
        # free the C5 handle first: its persisting-L2 set-aside (device-wide,
        # released with the last handle) would otherwise shrink the L2 the
        # other configs see (C2's streaming march: 228 vs 248 ms)
        s.close()
        extra = {}
        # C3 / C4 also with the exact causal P^{-1} (reading A27)
        # in place of the paper's inner Krylov P^{-1}
        for name in ("C2", "C3", "C4", "C3-exactPinv", "C4-exactPinv"):
            base, _, var = name.partition("-")
            q = si.config(base, pinv_exact=1) if var else si.config(base)
            sq = SWR(q, si.inputs(q), device=local, stream=stream)
            with torch.cuda.stream(stream):
                sq.build()
                sq.solve(out=uT_dev if q.Nx == p.Nx else None)
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                flush.fill_(1.0)
                e0.record(stream)
                sq.build()
                stq, _, rq = sq.solve(out=uT_dev if q.Nx == p.Nx else None)
                e1.record(stream)
                e1.synchronize()
            tq = e0.elapsed_time(e1)
            extra[name] = {"workload": workload_config(q)["workload"] + (", exact causal P^-1" if var else ""),
                           "status": stq,
                           "time_to_solution_ms": tq, "value": rq["cell_steps"] / (tq / 1e3), "unit": UNIT,
                           "outer_iterations": rq["iterations"], "inner_iterations": rq["inner_iterations"],
                           "fp_max": rq["fp_max"], "march_ms": rq["t_march_ms"],
                           "march_frac_of_step": rq["t_march_ms"] / tq,
                           "march_fp64_frac": FLOP_PER_CELL_STEP * rq["cell_steps"] / (rq["t_march_ms"] / 1e3)
                                              / 1e12 / fp64,
                           "march_streaming_equiv_bw_frac": BYTES_PER_CELL_STEP * rq["cell_steps"]
                                                            / (rq["t_march_ms"] / 1e3) / 1e9 / hbm}
            if q.Nj > RESIDENT_MAX_ROWS and q.potential == si.POT_VX:
                # the two-pass streaming march's own HBM bytes (DESIGN.md section 6:
                # 136 B per row-step) against the measured copy peak: a real roofline
                extra[name]["march_kernel"] = "k_march_stream2 (streaming, state through HBM)"
                extra[name]["march_bytes_per_cell_step"] = STREAM2_BYTES_PER_CELL_STEP
                extra[name]["march_hbm_frac"] = (STREAM2_BYTES_PER_CELL_STEP * rq["cell_steps"]
                                                 / (rq["t_march_ms"] / 1e3) / 1e9 / hbm)
            sq.close()
        line["other_configs"] = extra
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        P = os.cpu_count() or 1
        dt, ro = oracle_time_to_solution(p, arrays, P)
        line["cpu_baseline"] = {"value": cells / dt, "unit": UNIT, "cores": P, "kind": "oracle",
                                "seconds": dt, "iterations": ro["iterations"],
                                "sample": f"the whole {p.name} time-to-solution (build of d and L, "
                                          f"{ro['iterations']} GMRES iterations, final sweep) by the oracle on "
                                          f"{P} host threads; single-thread T_oracle,1 in "
                                          f"profiles/r02/oracle_c5_single_thread.txt"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
