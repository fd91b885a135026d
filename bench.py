#!/usr/bin/env python3
"""Benchmark of the circulant LASSO hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]

A "step" is one solver iteration over the whole problem.  Default workload
(N=1): BASELINE config 3 -- ISTA, partial circulant A, n=2^20, m=2^18,
k=2^12 (make_problem(2^20, 2^18, 2^12, seed=1)), alpha=1e-4, tau=0.9
(auto), literal pairing; metric = ISTA iterations/s.  For N>1 the same
problem is row/output-sharded across the ranks (strong scaling); each phase's
slice reaches every rank through the library (BENCH_TRANSPORT below).

Timing: W untimed warm-up iterations, then K iterations queued back to back
(no host synchronization inside the timed loop), each bracketed by CUDA
events on the solver's stream; L2 is flushed (256 MiB write) between timed
iterations on the same stream, outside the events.  Barrier + synchronize around the timed
region, max over ranks.  `e2e` is the same metric through the public API
(ista_run from host numpy buffers: setup, upload, K iterations, result
download) timed on the host clock (sharded: setup + K sharded iterations +
download, max over ranks).  Rank 0 prints one JSON line; native output (NCCL
banners) goes to stderr.  The default line also carries the FFT engine, the
cADMM rate at n=2^20 and the time to recovery (MSE <= 1e-4) on both engines.
BENCH_FORCE_SHARDED=1 runs the sharded path with a single rank; BENCH_TRANSPORT=ipc (default: the exchange fused
into the epilogues as CUDA IPC peer stores) or nccl (the library's NCCL broadcasts) picks the N>1 exchange;
BENCH_SHARE_DEVICE=1 maps the ranks round-robin onto the visible GPUs (a functional run of the N>1 path on one
GPU: gloo timing collectives, the IPC exchange).
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

WORKLOADS = {
    "c3": dict(kind="ista", n=1 << 20, m=1 << 18, k=1 << 12, seed=1,
               desc="BASELINE config 3: ISTA n=2^20, m=2^18, k=2^12, alpha=1e-4, tau=0.9, literal pairing"),
    "c1": dict(kind="ista", n=4096, m=1024, k=64, seed=1,
               desc="BASELINE config 1: ISTA n=4096, m=1024, k=64, alpha=1e-4"),
    "c2": dict(kind="cadmm", n=4096, m=1024, k=64, seed=1,
               desc="BASELINE config 2: cADMM n=4096, m=1024, k=64, rho=sigma=0.1"),
    "c4": dict(kind="cadmm", n=1 << 24, m=1 << 22, k=1 << 16, seed=1,
               desc="BASELINE config 4: cADMM n=2^24, m=2^22, k=2^16, rho=sigma=0.1"),
}
METRIC = "ISTA & ADMM iterations/sec and time-to-recovery at n=2^20 (1 GPU), n=2^24 (1/2/4/8)"


def algorithmic_flops(w):
    # ISTA 4*m*n, cADMM 6*n^2 (mat-vec FMAs only, 2 flop each)
    return 4.0 * w["m"] * w["n"] if w["kind"] == "ista" else 6.0 * w["n"] * w["n"]


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every 5 ms (the timed region of
    the default line is ~0.2 s), else nvidia-smi every 0.2 s."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h): HW slowdown, HW thermal, SW thermal, SW power cap
    BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
            ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, power_w, set of reason names)
        self.source = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.source = "nvml, 5 ms"
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                try:
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                except Exception:
                    pw = None
                self.samples.append((float(sm), float(mx), pw, {k for k, b in self.BITS if bits & b}))
                self._stop.wait(0.005)
        finally:
            nv.nvmlShutdown()

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            self.samples = []
        self.source = "nvidia-smi, 0.2 s"
        names = [k for k, _ in self.BITS]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) >= 8 and f[0].replace(".", "").isdigit():
                    pw = float(f[2]) if f[2].replace(".", "").isdigit() else None
                    self.samples.append((float(f[0]), float(f[1]), pw,
                                         {names[i] for i in range(4) if f[4 + i] == "Active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        pw = [s[2] for s in self.samples if s[2] is not None]
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_mhz_min": min(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[3] for s in self.samples))),
                "power_w_median": statistics.median(pw) if pw else None,
                "samples": len(self.samples), "source": self.source}


SAMPLE_FMA = 1 << 33  # per phase per CPU step: ~1-2 s on a 16-core host


def cpu_phase_sampler(w):
    """The reference's CPU path for this metric: the phase engine (cpista_phases /
    cpadmm_phases, parallel.hpp:173-279 -- the direct mat-vec the GPU `value`
    runs), restated in oracle/ (ascending fp64 accumulation, std::thread over
    contiguous output ranges), on all host cores.  Small problems run whole
    iterations; large ones time a leading sample of each phase's outputs and
    scale it to the full phase (every output of a phase costs the same)."""
    from oracle import oracle as orc
    p = orc.make_problem(w["n"], w["m"], w["k"], w["seed"])
    n, m = w["n"], w["m"]
    threads = os.cpu_count() or 1
    if w["kind"] == "ista":
        h = orc.Ista(p.row, p.omega, p.y)
        rows = max(1, min(m, SAMPLE_FMA // n))
        outs = max(1, min(n, SAMPLE_FMA // m))
        full = rows == m and outs == n
        sample = "full iterations" if full else \
            f"residual phase on {rows} of {m} rows + gradient phase on {outs} of {n} outputs, scaled to the full phases"

        def step():  # (seconds of one full iteration, wall seconds of this step)
            t0 = time.perf_counter()
            if full:
                h.step(1, orc.ENGINE_PHASES, threads)
                dt = time.perf_counter() - t0
                return dt, dt
            tr, tg = h.phase_sample(rows, outs, threads)
            return tr * m / rows + tg * n / outs, time.perf_counter() - t0
    else:
        h = orc.Cadmm(p.row, p.omega, p.y)
        outs = max(1, min(n, SAMPLE_FMA // n))
        full = outs == n
        sample = "full iterations" if full else f"the three phases on {outs} of {n} outputs, scaled to the full phases"

        def step():  # (seconds of one full iteration, wall seconds of this step)
            t0 = time.perf_counter()
            if full:
                h.step(1, orc.ENGINE_PHASES, threads)
                dt = time.perf_counter() - t0
                return dt, dt
            return sum(h.phase_sample(outs, threads)) * n / outs, time.perf_counter() - t0
    return step, threads, sample, full


def cpu_fft_rate(w, steps: int):
    """The reference-default FFT engine (use_fft=true, single-threaded like Eigen::FFT), oracle port."""
    from oracle import oracle as orc
    p = orc.make_problem(w["n"], w["m"], w["k"], w["seed"])
    h = orc.Ista(p.row, p.omega, p.y) if w["kind"] == "ista" else orc.Cadmm(p.row, p.omega, p.y)
    t0 = time.perf_counter()
    h.step(steps, orc.ENGINE_FFT)
    return steps / (time.perf_counter() - t0)


def cpu_baseline_line(w, steps: int, warmup: int):
    """Returns the baseline dict, the (extrapolated) seconds per full iteration and the wall seconds per
    timed step (a bounded sample when the iteration is too long to run whole)."""
    step, threads, sample, full = cpu_phase_sampler(w)
    for _ in range(warmup):
        step()
    res = [step() for _ in range(steps)]
    per_iter = sum(r[0] for r in res) / len(res)
    wall = sum(r[1] for r in res) / len(res)
    return {"value": 1.0 / per_iter, "unit": "iterations/s", "cores": threads, "kind": "port",
            "sample": f"{steps} steps of the phase engine (direct mat-vec, fp64, {threads} threads): {sample}",
            "extrapolated": not full,
            "engine": "phases (cpista_phases/cpadmm_phases restated in oracle/)"}, per_iter, wall


def run_reference(args, w, rank):
    if rank != 0:
        return
    steps = max(1, args.steps)
    warm = args.warmup
    cpu, per_iter, wall = cpu_baseline_line(w, steps, warm)
    rate = cpu["value"]
    # ms_per_step is the wall time of one timed step as run (a bounded sample of the iteration when
    # `extrapolated`); value is the full-iteration rate the samples scale to
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "iterations/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * wall,
        "ms_per_iteration": 1e3 * per_iter, "extrapolated": cpu["extrapolated"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (make_problem, seeded)",
        "config": {"workload": w["desc"], "n": w["n"], "m": w["m"], "k": w["k"], "seed": w["seed"]},
        "cpu_baseline": cpu,
        "e2e": {"value": rate, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measured_peaks():
    """Roofline denominators: the driver-written MEASURED_PEAKS.json (cuBLAS bf16 GEMM burst / sustained,
    STREAM-style copy) -- else the B200_PROFILING.md fallback (1.59 PF burst, 1.4 PF sustained, 6.65 TB/s)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"bf16": float(d["bf16_tflops"]), "bf16_sustained": float(d.get("bf16_tflops_sustained", 0) or 0),
                "hbm_gbs": float(d.get("hbm_gbs", 0) or 0), "source": "of measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm_gbs": 6650.0,
                "source": "of fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"}


def tc_f16(n):
    """The tcgen05 kernel uses fp16 operands (2-term split) for n >= 2^18, 3xTF32 below (CLB_TC_F16 forces)."""
    v = os.environ.get("CLB_TC_F16", "")
    return (v not in ("", "0")) if v else n >= (1 << 18)


def tc_peak(n, peaks, sustained=False):
    """Dense tensor peak of the kernel's MMA kind: kind::f16 runs at the bf16 rate; kind::tf32 at half of it."""
    base = peaks["bf16_sustained"] if sustained and peaks["bf16_sustained"] else peaks["bf16"]
    return base if tc_f16(n) else base / 2.0


def tc_dtype(n):
    return "f16x3-split/fp32-acc" if tc_f16(n) else "tf32x3-split/fp32-acc"


def tc_note(n):
    return ("fp16 operands, power-of-two scaled, 2-term split (hi.hi + hi.lo + lo.hi, kind::f16)" if tc_f16(n) else
            "3xTF32 (hi.hi + hi.lo + lo.hi, kind::tf32)") + \
        ": 3 tensor flops per dense-product flop"


def dense_uses_tc(n):
    """cADMM dense products run on the tcgen05 kernel (csrc/tc_dense.cu) for power-of-two n >= 2^15."""
    return n >= (1 << 15) and (n & (n - 1)) == 0 and os.environ.get("CLB_NO_TC", "0") in ("", "0")


def dense_kernel_info(n, ms, peaks):
    flops = 2.0 * n * n
    if dense_uses_tc(n):
        pk = tc_peak(n, peaks)
        return {"kernel": "k_tc_dense", "ms": ms, "achieved_tflops": flops / (ms * 1e-3) / 1e12,
                "bound": "tensor", "peak_tflops": pk, "peak_source": peaks["source"],
                "frac": flops / (ms * 1e-3) / 1e12 / pk,
                "tensor_pipe_tflops": 3 * flops / (ms * 1e-3) / 1e12,
                "tensor_pipe_frac": 3 * flops / (ms * 1e-3) / 1e12 / pk,
                "note": tc_note(n) + "; ms = CUDA-event time of the product inside the graph-replayed step"}
    return {"kernel": "k_conv_dense", "ms": ms, "achieved_tflops": flops / (ms * 1e-3) / 1e12, "bound": "fp32_ffma"}


def ista_uses_tc(n):
    """ISTA's direct engine embeds both sparse products in dense tcgen05 products for n >= 2^17."""
    return n >= (1 << 17) and dense_uses_tc(n)


def timed_steps(st, stream, flush, steps, torch):
    """`steps` graph-replayed iterations back to back (no host synchronization inside the timed loop), L2
    flushed before each on the same stream (outside the per-step events); per-step CUDA-event times on the
    solver's stream and the per-phase times of each replay (profile mode 2: in-graph event nodes re-pointed
    to a per-replay slot, read after the loop)."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            ev[i][0].record(stream)
        st.step(1)
        with torch.cuda.stream(stream):
            ev[i][1].record(stream)
    st.synchronize()
    return [a.elapsed_time(b) for a, b in ev], st.phase_history(steps)


def admm_line(cl, torch, prob, local_rank, flush, peaks, steps=5, warmup=3):
    """cADMM (the paper's CPADMM, the metric's "ADMM") on the same n=2^20 problem:
    device-timed iterations/s of the direct engine (3 dense circulant products
    per iteration, 6 n^2 flop) and the dense kernel's roofline fraction."""
    import ctypes as C
    from paper_1707_02244_b200._native import lib as L
    st = cl.cadmm_setup(prob.op, prob.measurements, cl.SolverConfig(), device=local_rank)
    sp = C.c_void_p()
    L.cl_solver_stream(st.handle, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    st.profile(2)
    st.step(warmup)
    st.synchronize()
    step_ms, phases = timed_steps(st, stream, flush, steps, torch)
    ms = sum(step_ms) / steps
    ph = [statistics.mean(p[i] for p in phases) for i in range(len(phases[0]))]
    n = prob.op.n()
    dense_ms = (ph[0] + ph[2] + ph[4]) / 3.0
    return {"value": 1e3 / ms, "unit": "iterations/s", "ms_per_step": ms, "steps": steps, "warmup": warmup,
            "workload": f"cADMM n={n}, m={prob.op.m()}, k={prob.k()}, rho=sigma=0.1, tau1=tau2=1, alpha=1e-4 "
                        "(make_problem(2^20, 2^18, 2^12, 1), the config-3 problem)",
            "engine": "direct circulant products on tcgen05 tensor cores" if dense_uses_tc(n)
                      else "direct shift-indexed sm_100a kernels",
            "dense_kernel": dense_kernel_info(n, dense_ms, peaks),
            "step_tflops": 6.0 * n * n / (ms * 1e-3) / 1e12, "phase_ms": ph}


def dense_line(cl, torch, local_rank, iters=200):
    """The paper's circulant-vs-dense contrast on BASELINE config 2's problem
    (make_problem(4096, 1024, 64, 1)): the dense ADMM baseline (admm_setup: Gram matrix + blocked Gauss-Jordan
    inverse in fp64 on the GPU; then one L2-resident fp32 mat-vec per iteration) against cADMM (O(n) state),
    each through its public run call, 200 fixed iterations; host clock."""
    prob = cl.make_problem(4096, 1024, 64, 1)
    cfg = cl.SolverConfig(max_iter=iters, check_every=iters)
    out = {"workload": "make_problem(4096, 1024, 64, 1) (BASELINE config 2's problem), 200 iterations",
           "note": "wall time of the public run call from host buffers (setup + iterations + download); "
                   "the dense setup builds and inverts the 4096 x 4096 Gram matrix in fp64 on the GPU"}
    for name, run in (("admm_dense", cl.admm_dense_run), ("cadmm", cl.cadmm_run)):
        run(prob.measurements, prob.op, cl.SolverConfig(max_iter=2, check_every=2), device=local_rank)  # warm
        t0 = time.perf_counter()
        rep = run(prob.measurements, prob.op, cfg, device=local_rank)
        wall = time.perf_counter() - t0
        out[name] = {"seconds": wall, "setup_seconds": rep.setup_seconds,
                     "iterations_per_s": iters / max(rep.total_seconds - rep.setup_seconds, 1e-12),
                     "footprint_bytes": rep.footprint_bytes}
    return out


def recovery_line(cl, prob, local_rank, target=1e-4):
    """Time to recovery (paper protocol: stop at MSE(x, x*) <= 1e-4)
    through the public API (ista_run / cadmm_run with truth, check_every=10):
    host buffers in, setup, iterations, result out; host clock."""
    out = {"target_mse": target, "check_every": 10,
           "note": "ista_run/cadmm_run(y, A, SolverConfig(target_mse=1e-4), truth=x*) from host fp64 buffers; "
                   "seconds = the call's wall time (setup + iterations + download)"}
    for kind, run, cap in (("ista", cl.ista_run, 6000), ("cadmm", cl.cadmm_run, 1000)):
        out[kind] = {}
        for eng in ("direct", "fft"):
            cfg = cl.SolverConfig(max_iter=cap, check_every=10, target_mse=target, use_fft=(eng == "fft"))
            t0 = time.perf_counter()
            rep = run(prob.measurements, prob.op, cfg, truth=prob.signal.values, device=local_rank)
            wall = time.perf_counter() - t0
            out[kind][eng] = {"seconds": wall, "iterations": rep.iterations, "reached": bool(rep.reached_target),
                              "final_mse": rep.final_metric, "setup_seconds": rep.setup_seconds}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the cADMM line and time-to-recovery")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    # the sharded (NCCL) path; BENCH_FORCE_SHARDED=1 exercises it with a single rank under torchrun
    sharded = world > 1 or os.environ.get("BENCH_FORCE_SHARDED") == "1"
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, w, rank)

    # stdout carries exactly one JSON line: anything native code prints while the bench runs (NCCL's
    # version banner, library diagnostics) is routed to stderr at the file-descriptor level
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)

    import numpy as np
    import torch
    import paper_1707_02244_b200 as cl
    from paper_1707_02244_b200 import dist as cdist

    # BENCH_SHARE_DEVICE=1: every rank on the visible GPUs round-robin (a functional run of the N > 1 path on
    # fewer GPUs: gloo for the timing collectives, the IPC exchange -- NCCL refuses two ranks on one GPU)
    share = os.environ.get("BENCH_SHARE_DEVICE") == "1"
    if share:
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    if sharded:
        import torch.distributed as tdist
        if share:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def max_over_ranks(v: float) -> float:
        t = torch.tensor([v], device="cpu" if share else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_SHORT_WARMUP"), "need >= 3 warm-up steps"

    prob = cl.make_problem(w["n"], w["m"], w["k"], w["seed"])
    cfg = cl.SolverConfig()
    setup = cl.ista_setup if w["kind"] == "ista" else cl.cadmm_setup
    st = setup(prob.op, prob.measurements, cfg, device=local_rank)
    comm = None
    # sharded: the slice exchange runs inside cl_solver_step, either fused into the producing epilogues as CUDA
    # IPC peer stores (BENCH_TRANSPORT=ipc, the default) or as the library's NCCL broadcasts (=nccl)
    transport = os.environ.get("BENCH_TRANSPORT", "ipc")
    def one_step():
        st.step(1)

    failed_states = []  # a state whose IPC attach failed is kept alive: destroying an attached state is collective
    if sharded and transport == "ipc":
        # the peer-store transport needs CUDA IPC + peer access between the ranks' GPUs; if any rank cannot attach
        # or its first exchange fails, every rank (decided together, so the collectives stay matched) falls back
        # to the library's NCCL exchange on a fresh state
        ok = 1
        comm = cdist.TorchIpc()
        try:
            comm.attach(st)
            one_step()
            st.synchronize()
        except Exception as e:  # noqa: BLE001 -- reported, then the NCCL transport takes over
            print(f"bench: rank {rank}: IPC peer-store transport failed ({e}); falling back to NCCL", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device="cpu" if share else "cuda")
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        if int(flag.item()) == 0:
            failed_states.append(st)
            st = setup(prob.op, prob.measurements, cfg, device=local_rank)
            transport = "nccl"
    if sharded and transport != "ipc":
        comm = cdist.NativeComm.from_torch(local_rank)
        comm.attach(st)

    import ctypes as C
    from paper_1707_02244_b200._native import lib as L
    sp = C.c_void_p()
    L.cl_solver_stream(st.handle, C.byref(sp))
    sp_stream = torch.cuda.ExternalStream(sp.value)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    # per-phase CUDA events recorded inside the timed steps themselves: event nodes in the captured step
    # graph (mode 2); the sharded path launches its phases eagerly (mode 1)
    st.profile(1 if sharded else 2)
    for _ in range(args.warmup):
        one_step()
    st.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phase_ms = []
    if sharded:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # back to back: each step is queued behind the previous one with no host synchronization in between
    # (the GPU never idles, so clocks and power are those of a sustained solve); L2 is flushed before every
    # step on the same stream, outside the step's events
    with ClockSampler(local_rank) as clocks:
        for i in range(args.steps):
            with torch.cuda.stream(sp_stream):
                flush.zero_()
                ev[i][0].record(sp_stream)
            one_step()
            with torch.cuda.stream(sp_stream):
                ev[i][1].record(sp_stream)
            if sharded:  # eager phases: per-step phase times need the step's events
                st.synchronize()
                phase_ms.append(st.phase_ms())
        torch.cuda.synchronize()
    if sharded:
        torch.distributed.barrier()
    else:
        phase_ms = st.phase_history(args.steps)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if sharded:
        total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / args.steps
    value = 1e3 / ms_per_step  # iterations/s of the (single, sharded) solve
    st.profile(0)
    phase_mean = [statistics.mean(p[i] for p in phase_ms) for i in range(len(phase_ms[0]))]

    # dominant kernel, timed inside the timed steps.  Phase windows: ISTA [residual product, gather, scatter +
    # gradient product, update]; cADMM [C^T v, beta, B beta, x, C x, duals].  A tensor-core product's window
    # also holds its k_absmax2 scale pre-pass (~1% of it), so kernel_ms slightly overstates the kernel.
    n, m = w["n"], w["m"]
    if w["kind"] == "ista":
        prod_idx = [0, 2]
        useful = 2.0 * m * n / world  # per launch: residual m rows x n, gradient n outputs x m rows
        if ista_uses_tc(n):
            k_name = "k_tc_dense"  # both sparse products embedded in dense tensor-core products
        else:
            k_name = "k_res_s" if n >= (1 << 17) else "k_conv_residual"
            prod_idx = [0]
    else:
        prod_idx = [0, 2, 4]
        useful = 2.0 * n * n / world
        k_name = "k_tc_dense" if dense_uses_tc(n) else "k_conv_dense"
    k_ms = statistics.mean(phase_mean[i] for i in prod_idx)
    peaks = measured_peaks()
    if k_name == "k_tc_dense":
        peak, peak_source = tc_peak(n, peaks), "bf16_tflops " + peaks["source"] + \
            ("" if tc_f16(n) else "; kind::tf32 = half the bf16 rate")
    else:
        peak, peak_source = cl.ffma_peak_tflops(local_rank), "live FFMA microbenchmark (cl_ffma_peak)"
    achieved = useful / (k_ms * 1e-3) / 1e12
    ffma_peak = cl.ffma_peak_tflops(local_rank)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get(k_name, {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    # e2e: the public API from host buffers (setup + upload + K iterations + download).  The timed state is
    # released first: its device memory returns to the stream-ordered pool (kept reserved), so the e2e call
    # allocates from a warm pool like any call after the first in a process.
    if not sharded:
        del st
    n, m = w["n"], w["m"]
    chunks = (n + 1023) // 1024
    # bytes the setup moves host->device (device fp64 setup for power-of-two n >= 2^14: the fp64 row; the
    # fp32 y, int32 omega and the chunk row index for ISTA; the fp32 D and P^T y for cADMM)
    h2d = (8 * n + 4 * m + 4 * m + 4 * (chunks + 1)) if w["kind"] == "ista" else (16 * n)
    d2h = 4 * n + 32  # the iterate and the fused check metrics
    e2e = None
    if not sharded:
        cfg_e2e = cl.SolverConfig(max_iter=args.steps, check_every=args.steps)
        run = cl.ista_run if w["kind"] == "ista" else cl.cadmm_run
        # one untimed warm-up call (first-use costs of the call path: lazy kernel loading, host paging)
        run(prob.measurements, prob.op, cl.SolverConfig(max_iter=2, check_every=2), device=local_rank)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = run(prob.measurements, prob.op, cfg_e2e, device=local_rank)
        e2e_s = time.perf_counter() - t0
        assert rep.iterations == args.steps
        e2e = {"value": args.steps / e2e_s, "unit": "iterations/s", "h2d_bytes_per_step": h2d / args.steps,
               "d2h_bytes_per_step": d2h / args.steps, "wall_s": e2e_s, "report_setup_s": rep.setup_seconds,
               "report_total_s": rep.total_seconds,
               "note": "ista_run/cadmm_run from host fp64 buffers incl. setup (spectral norm, Gram inverse), "
                       "upload, K iterations and final download; host clock; after one untimed warm-up call"}
    else:
        # sharded: every rank sets up from host buffers, runs K sharded iterations (all-gathers over NCCL) and
        # rank 0 downloads the iterate; the slowest rank's wall time
        torch.distributed.barrier()
        torch.cuda.synchronize()
        run = cl.ista_run if w["kind"] == "ista" else cl.cadmm_run
        t0 = time.perf_counter()
        rep = run(prob.measurements, prob.op, cl.SolverConfig(max_iter=args.steps, check_every=args.steps),
                  device=local_rank, comm=comm)
        e2e_s = time.perf_counter() - t0
        assert rep.iterations == args.steps
        e2e_s = max_over_ranks(e2e_s)
        e2e = {"value": args.steps / e2e_s, "unit": "iterations/s", "h2d_bytes_per_step": world * h2d / args.steps,
               "d2h_bytes_per_step": d2h / args.steps, "wall_s": e2e_s,
               "note": f"{world} ranks: ista_run/cadmm_run(..., comm={type(comm).__name__}) from host fp64 buffers "
                       "on every rank: setup, K sharded iterations (" +
                       ("the slices stored into every rank's copy by the producing epilogues, CUDA IPC"
                        if transport == "ipc" else "in-place NCCL broadcasts of the slices inside the library") +
                       "), iterate download; max wall time over ranks"}

    # the same workload through the on-device FFT engine (use_fft=True, the reference's default engine)
    fft_line = None
    if not sharded and (w["n"] & (w["n"] - 1)) == 0:
        fst = setup(prob.op, prob.measurements, cl.SolverConfig(use_fft=True), device=local_rank)
        fst.step(3)
        fst.synchronize()
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        fsp = C.c_void_p()
        L.cl_solver_stream(fst.handle, C.byref(fsp))
        fstream = torch.cuda.ExternalStream(fsp.value)
        for i in range(args.steps):
            with torch.cuda.stream(fstream):
                flush.zero_()
                fev[i][0].record(fstream)
            fst.step(1)
            with torch.cuda.stream(fstream):
                fev[i][1].record(fstream)
        fst.synchronize()
        fms = sum(a.elapsed_time(b) for a, b in fev) / args.steps
        n = w["n"]
        nprod = 2 if w["kind"] == "ista" else 3
        # four-step engine (n >= 2^14), complex formulation: per product cols_fwd reads 4n (real) +
        # writes 8n, rows reads 8n (T) + 8n (H) + writes 8n, cols_inv reads 8n + writes 4n bytes: 48n bytes.
        # The real plans (n >= 2^18) run the same passes on n/2 complex points: 24n bytes per product.
        fft_bytes = nprod * 48 * n
        fft_bytes_real = nprod * 24 * n
        run_f = cl.ista_run if w["kind"] == "ista" else cl.cadmm_run
        run_f(prob.measurements, prob.op, cl.SolverConfig(max_iter=2, check_every=2, use_fft=True),
              device=local_rank)  # untimed warm-up call
        t0 = time.perf_counter()
        rep_f = run_f(prob.measurements, prob.op, cl.SolverConfig(max_iter=args.steps, check_every=args.steps,
                                                                   use_fft=True), device=local_rank)
        fe2e_s = time.perf_counter() - t0
        assert rep_f.iterations == args.steps
        fft_line = {"value": 1e3 / fms, "unit": "iterations/s", "ms_per_step": fms,
                    "e2e": {"value": args.steps / fe2e_s, "unit": "iterations/s", "wall_s": fe2e_s,
                            "report_setup_s": rep_f.setup_seconds, "report_total_s": rep_f.total_seconds,
                            "note": "ista_run(use_fft=True) from host buffers incl. setup and download, "
                                    "after one untimed warm-up call"},
                    "engine": "on-device four-step FFT, real plans (n/2 complex points, the spectrum unpacked "
                              "pairwise between the row FFTs; columns / rows-with-spectral-multiply / columns, "
                              "radix-16 shared-memory stages, chained products), CUDA-graph replay",
                    "gbs_algorithmic": fft_bytes / (fms * 1e-3) / 1e9,
                    "bytes_per_step": fft_bytes,
                    "gbs_real_plan_bytes": fft_bytes_real / (fms * 1e-3) / 1e9,
                    "bytes_per_step_real_plan": fft_bytes_real,
                    "note": "same metric and workload, SolverConfig(use_fft=True); L2 flushed between steps"}
        del fst

    admm = recovery = dense = None
    if not sharded and w["kind"] == "ista" and w["n"] == (1 << 20) and not args.quick:
        admm = admm_line(cl, torch, prob, local_rank, flush, peaks)
        recovery = recovery_line(cl, prob, local_rank)
        dense = dense_line(cl, torch, local_rank)

    cpu = None
    if rank == 0 and not sharded and not args.no_cpu_baseline:
        cpu, _, _ = cpu_baseline_line(w, 3 if w["n"] >= (1 << 20) else 20, 1)
        if fft_line is not None:
            fft_line["cpu_fft_engine"] = {
                "value": cpu_fft_rate(w, 2 if w["n"] >= (1 << 20) else 20), "unit": "iterations/s", "cores": 1,
                "kind": "port", "sample": "full iterations of the reference-default FFT engine (single thread)"}
        if admm is not None:
            step, threads, sample, full = cpu_phase_sampler(dict(w, kind="cadmm"))
            step()
            secs = [step()[0] for _ in range(2)]
            admm["cpu_baseline"] = {"value": len(secs) / sum(secs), "unit": "iterations/s", "cores": threads,
                                    "kind": "port", "sample": f"2 steps of the cADMM phase engine (fp64): {sample}",
                                    "extrapolated": not full}
        if recovery is not None:
            for kind, rate in (("ista", cpu["value"]), ("cadmm", admm["cpu_baseline"]["value"] if admm else None)):
                if rate:
                    it = recovery[kind]["direct"]["iterations"]
                    recovery[kind]["cpu_phase_engine_seconds_extrapolated"] = it / rate

    sys.stdout.flush()
    os.dup2(json_fd, 1)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": tc_dtype(n) if k_name == "k_tc_dense" else "f32", "data": "synthetic (make_problem, seeded)",
            "config": {"workload": w["desc"], "n": w["n"], "m": w["m"], "k": w["k"], "seed": w["seed"],
                       "engine": ("direct circulant products on tcgen05 tensor cores" +
                                  (" (ISTA's sparse products embedded in dense ones)" if w["kind"] == "ista" else "")
                                  if k_name == "k_tc_dense" else
                                  "direct shift-indexed sm_100a kernels"),
                       "l2": "flushed (256 MiB) between steps",
                       "parallelism": f"row/output shards x{world} (" + ("exchange fused into the epilogues: CUDA IPC "
                                      "peer stores" if transport == "ipc" else "library-owned NCCL exchange") + ")"
                       if sharded
                       else "single GPU"},
            "roofline": {"bound": "tensor" if k_name == "k_tc_dense" else "fp32_ffma", "kernel": k_name,
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": peak_source,
                         "work_per_launch": f"{useful:.6g} flop = algorithmic (SURVEY 8d): " +
                                            ("2 m n per product (residual m rows x n, gradient n x m)"
                                             if w["kind"] == "ista" else "2 n^2 per dense product"),
                         "kernel_ms": k_ms,
                         "kernel_ms_source": "CUDA events of the timed steps themselves (event-record nodes captured "
                                             "around each product, re-pointed to a per-replay slot), mean over "
                                             "products and steps",
                         "kernel_share_of_step": len(prod_idx) * k_ms / ms_per_step,
                         **({"frac_sustained_peak": achieved / tc_peak(n, peaks, sustained=True),
                             "dense_product": {"flop": 2.0 * n * n / world,
                                               "tflops": 2.0 * n * n / world / (k_ms * 1e-3) / 1e12,
                                               "frac": 2.0 * n * n / world / (k_ms * 1e-3) / 1e12 / peak},
                             "tensor_pipe": {"flop": 6.0 * n * n / world,
                                             "tflops": 6.0 * n * n / world / (k_ms * 1e-3) / 1e12,
                                             "frac": 6.0 * n * n / world / (k_ms * 1e-3) / 1e12 / peak},
                             "work_note": ("each product runs the dense C u (2 n^2 flop" +
                                           ("; ISTA needs the m rows of Omega or the m inputs of P^T r, 2 m n"
                                            if w["kind"] == "ista" else "") +
                                           ") as 3 tensor-core MMAs per flop: " + tc_note(n))}
                            if k_name == "k_tc_dense" else {}),
                         "step_tflops": algorithmic_flops(w) / world / (ms_per_step * 1e-3) / 1e12,
                         # the north_star's own bar: the iteration's algorithmic flops (4 m n ISTA, 6 n^2 cADMM)
                         # per second against the FP32 FFMA roofline (>= 0.6 asked), measured on this GPU
                         "vs_fp32_ffma_roofline": {
                             "algorithmic_tflops": algorithmic_flops(w) / world / (ms_per_step * 1e-3) / 1e12,
                             "ffma_peak_tflops": ffma_peak,
                             "frac": algorithmic_flops(w) / world / (ms_per_step * 1e-3) / 1e12 / ffma_peak,
                             "peak_source": "live FFMA microbenchmark (cl_ffma_peak)"},
                         "phase_ms": phase_mean},
            "clocks": clocks.summary(),
            # per step: ISTA 2 products + gather/scatter + update; cADMM 3 products + 3 epilogues; each
            # fp16 tensor-core product adds its k_absmax2 scale pass
            "gpu_launches": args.steps * (
                (5 + (2 if tc_f16(w["n"]) else 0) if ista_uses_tc(w["n"]) else 4) if w["kind"] == "ista" else
                (6 + (3 if dense_uses_tc(w["n"]) and tc_f16(w["n"]) else 0))),
            "e2e": e2e,
            "fft_engine": fft_line,
            "admm": admm,
            "dense_vs_circulant": dense,
            "time_to_recovery": recovery,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
