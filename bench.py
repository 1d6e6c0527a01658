#!/usr/bin/env python3
"""Benchmark: DD/QD GEMM 2mnl/s on B200 (BASELINE.json metric).

Workload (``config.workload``): BASELINE.json configs[1], the blocked DD
GEMM m = l = n = 1024 on the seeded uniform inputs, one
product per step.  Under torchrun with N ranks the problem is weak-scaled:
every rank owns its own 1024 rows of A and C, and B (1024 x 1024 DD) is
broadcast from rank 0 over NCCL inside every step, pipelined in k-panels
(``shard.broadcast_matmul``).

Printed (rank 0, one JSON line): ``value`` = device throughput (whole job,
CUDA events around each step on the launching stream, L2 flushed between
steps, max over ranks), ``e2e`` = the same metric through the public API
with host buffers (H2D of A and B, D2H of C inside the timed region),
``roofline`` against the FP64 pipe (peak measured in-run with a DFMA
micro-benchmark; spec 148 SMs x 64 lanes x 2 x 1.965 GHz = 37.2 TFLOP/s),
``cpu_baseline`` = the reference's own compiled kernels (oracle/_ref) on
the host cores, on a bounded leading-rows sample.

``--impl reference`` times that reference CPU implementation alone.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

F_DD = 53    # flops per DD multiply-add of the mirror kernel (4 DMUL, 3 DFMA, 43 DADD)
I_DD = 50    # FP64 instructions per DD multiply-add
F_QD = 796   # flops per QD multiply-add (10 DFMA, 13 DMUL, 763 DADD)
SPEC_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


# ~5 ms of GPU spin before each timed step (outside the events): the host
# enqueue of a step (plus the clock sampler's nvidia-smi forks competing
# for the host) must finish before the device reaches the start event, or
# host time leaks into the device-timed step (seen with 1 ms: +0.7 ms/step)
HOST_SLACK_CYCLES = 10_000_000

def parse():
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--prec", default="dd", choices=["dd", "qd"])
    p.add_argument("--size", type=int, default=1024, help="m = l = n per rank")
    p.add_argument("--nmin", type=int, default=0,
                   help="block size; 0 = let the GPU predictor pick from 16..256")
    p.add_argument("--panel", type=int, default=0, help="k-panel rows for the B broadcast")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0)
    p.add_argument("--dist-backend", default="nccl",
                   help="torch.distributed backend for N>1 (nccl; gloo only to test the "
                        "multi-rank logic with all ranks on one GPU)")
    p.add_argument("--same-device", action="store_true",
                   help="put every rank on cuda:0 (multi-rank logic test on one GPU, gloo)")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, power, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's compiled kernels (oracle/_ref) on the host
# ---------------------------------------------------------------------------

def cpu_reference_run(prec_tok, n, n_min, seconds):
    """Time the reference's own blocked kernel (multiply.py:_block_into
    partitioning over _kernels.dd_block_cells) on the leading rows of A
    against all of B, doubling the slice until it runs ~``seconds``.
    Returns (value 2mnl/s, cores, kind, sample description)."""
    import numpy as np

    import oracle
    from paper_1710_01839_b200 import inputs
    kern = oracle.ref_kernels()
    kind = "reference" if kern is not None else "port"
    cores = len(os.sched_getaffinity(0))
    a, b = inputs.gemm_inputs(prec_tok, n, n, n, seed=0)
    rows = n_min
    while True:
        sl = np.ascontiguousarray(a[:rows])
        t0 = time.perf_counter()
        oracle.matmul_block(sl, b, n_min, threads=cores, kernels=kern)
        dt = time.perf_counter() - t0
        if dt >= seconds / 2 or rows >= n:
            break
        rows = min(n, rows * 2 if dt > 0.05 else rows * 8)
    value = 2.0 * rows * n * n / dt
    sample = (f"{prec_tok.upper()} blocked n_min={n_min}: leading {rows} rows of A ({n}x{n}) "
              f"times all of B, {dt:.2f} s, threads={cores} (reference multiply.py "
              f"_run_partitioned over {'oracle/_ref _kernels' if kern else 'oracle C port'})")
    return value, cores, kind, sample, dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.nmin <= 0:
        args.nmin = 64   # the reference's DEFAULT_BLOCK_SIZE (multiply.py:32)
    steps = max(1, args.steps)
    per_step = max(1.0, min(args.cpu_seconds, 60.0 / (steps + args.warmup)))
    vals = []
    for i in range(args.warmup + steps):
        v, cores, kind, sample, _ = cpu_reference_run(args.prec, args.size, args.nmin, per_step)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "2mnl/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "2mnl/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "2mnl/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(args):
    return f"{args.prec.upper()} GEMM 2mnl/s (blocked, m=l=n={args.size})"


def workload_config(args, world):
    # n_min is each arm's own tuned block size (results never depend on it:
    # blocked == simple bitwise); the workload itself is the same for both
    return {"workload": f"BASELINE configs[1]: {args.prec.upper()} blocked GEMM "
                        f"m=l=n={args.size}, seeded uniform inputs (seed 0)",
            "prec": args.prec, "m_per_rank": args.size, "l": args.size, "n": args.size,
            "n_min": args.nmin, "parallelism": f"row-shard x{world}, B NCCL broadcast",
            "l2": "flushed between steps (256 MiB write), inputs 16 MiB/matrix"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def fp64_peak(torch, _cuda, dev):
    """In-run FP64 peak: DFMA and DADD burst throughput (TFLOP/s)."""
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    scratch = torch.zeros(sms * 16, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    out = {}
    for op, name, flops_per in ((0, "dfma", 2), (1, "dadd", 1)):
        blocks, threads, iters = sms * 8, 256, 20000
        _cuda.fp64_burn_dev(op, blocks, threads, 2000, scratch.data_ptr(), stream)
        best = 0.0
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            _cuda.fp64_burn_dev(op, blocks, threads, iters, scratch.data_ptr(), stream)
            e.record()
            e.synchronize()
            t = s.elapsed_time(e) / 1e3
            best = max(best, blocks * threads * 8 * iters * flops_per / t / 1e12)
        out[name] = best
    return out


def load_ncu_traffic(prec):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fp:
            data = json.load(fp)
        return data.get(prec, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1710_01839_b200 import _cuda, inputs, shard
    import paper_1710_01839_b200 as mp
    from paper_1710_01839_b200.matrix import DenseMatrix

    _cuda.load()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    prec = mp.PrecisionSpec.parse(args.prec)
    comps = prec.comps
    n = args.size
    F = F_DD if args.prec == "dd" else F_QD

    # per-rank inputs: rank r owns rows [r*n, (r+1)*n) of A; B from rank 0
    a_full, b_full = inputs.gemm_inputs(args.prec, n, n, n, seed=0)
    if rank > 0:
        a_full = inputs.gemm_inputs(args.prec, n, n, n, seed=1000 + rank)[0]
    A = torch.from_numpy(a_full).to(dev)
    B = torch.from_numpy(b_full).to(dev) if rank == 0 else torch.empty(
        (n, n, comps), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    panel = args.panel if args.panel > 0 else None
    panels = len(shard.panel_bounds(n, panel))
    tuner = None
    if args.nmin <= 0:
        # the reference's step 1 (tune.py:137-143) on the device, outside
        # the timed region: wave-aware prediction over the BASELINE sweep
        Bt = B if rank == 0 else torch.from_numpy(b_full).to(dev)
        best, recs = mp.select_block_size(
            DenseMatrix(n, n, prec, A), DenseMatrix(n, n, prec, Bt), [16, 32, 64, 128, 256],
            policy=mp.TimingPolicy(warmup_runs=1, measured_runs=3, aggregator="min"))
        if world > 1:
            t_best = torch.tensor([best], dtype=torch.int64, device=dev)
            dist.broadcast(t_best, src=0)
            best = int(t_best.item())
        args.nmin = best
        tuner = {"chosen_n_min": best, "records": [
            {"n_min": r.n_min, "slice_rows": r.slice_rows, "slice_ms": r.slice_time_s * 1e3,
             "predicted_ms": r.predicted_full_s * 1e3} for r in recs]}

    def step():
        return shard.broadcast_matmul(A, B, n_min=args.nmin, src=0, panel_rows=panel)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank).start() if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    evs = []
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()
        # keep the GPU busy (outside the timed region) while the host
        # enqueues the step, so host launch latency is not device time
        torch.cuda._sleep(HOST_SLACK_CYCLES)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        c = step()
        e.record(stream)
        evs.append((s, e))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall0
    dev_s = sum(s.elapsed_time(e) for s, e in evs) / 1e3
    gemm_launches = args.steps * panels

    # kernel-only time: the GEMM launch alone (no broadcast), events on its stream
    kev = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        C = torch.empty((n, n, comps), dtype=torch.float64, device=dev)
        torch.cuda._sleep(HOST_SLACK_CYCLES)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        _cuda.gemm_dev(comps, _cuda.ALGO_BLOCK, args.nmin, n, n, n, A.data_ptr(), n,
                       B.data_ptr(), n, C.data_ptr(), n, False, None, stream.cuda_stream)
        e.record(stream)
        kev.append((s, e))
    torch.cuda.synchronize()
    kernel_s = statistics.mean(s.elapsed_time(e) for s, e in kev) / 1e3
    # the opt-in faithful DD mode on the same workload (not bit-identical;
    # within the north_star bound -- tests/test_gpu_fast.py)
    fast_s = None
    if args.prec == "dd":
        fev = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            torch.cuda._sleep(HOST_SLACK_CYCLES)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            C = torch.empty((n, n, comps), dtype=torch.float64, device=dev)
            s.record(stream)
            _cuda.gemm_dev(comps, _cuda.ALGO_BLOCK_FAST, args.nmin, n, n, n, A.data_ptr(), n,
                           B.data_ptr(), n, C.data_ptr(), n, False, None, stream.cuda_stream)
            e.record(stream)
            fev.append((s, e))
        torch.cuda.synchronize()
        fast_s = statistics.mean(s.elapsed_time(e) for s, e in fev) / 1e3
    # the opt-in exact tensor mode (int8 tensor cores + CRT; exact product
    # rounded once): whole pipeline timed with events, same workload
    tensor_s, tensor_err = None, None
    try:
        from paper_1710_01839_b200.tensor import matmul_exact_tensors, plan
        pl = plan(A, B)
        for _ in range(3):               # plan, capture, replay
            matmul_exact_tensors(A, B)
        torch.cuda.synchronize()
        tev = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            torch.cuda._sleep(HOST_SLACK_CYCLES)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            matmul_exact_tensors(A, B)
            e.record(stream)
            tev.append((s, e))
        torch.cuda.synchronize()
        # median: each product ends in a host read of its status, so a host
        # hiccup can land inside one sample
        tensor_s = statistics.median(s.elapsed_time(e) for s, e in tev) / 1e3
        tensor_jobs = [(pl.ranges_a[ia], pl.ranges_b[ib], N) for ia, ib, N in pl.jobs]
    except Exception as ex:  # noqa: BLE001 - reported, the headline is unaffected
        tensor_err = f"{type(ex).__name__}: {ex}"
    clocks = sampler.stop() if sampler else None

    t = torch.tensor([dev_s, t_wall, kernel_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s, t_wall, kernel_s = t.tolist()
    madds_step = float(n) * n * n * world
    value = 2.0 * madds_step * args.steps / dev_s

    # end-to-end through the public API with host buffers
    e2e_steps = max(5, min(args.steps, 20))
    host_a = torch.from_numpy(a_full).pin_memory().numpy()
    host_b = torch.from_numpy(b_full).pin_memory().numpy()
    Ah = DenseMatrix(n, n, prec, host_a)
    Bh = DenseMatrix(n, n, prec, host_b)
    if world == 1:
        # warm: pools, streams, and the pinned-host cache in the loop's own
        # pattern -- `ch` keeps the previous result alive while the next is
        # allocated, so the steady state holds two page-locked results (the
        # second cudaHostAlloc, ~7 ms, would otherwise land in the timed loop)
        ch = None
        for _ in range(max(3, args.warmup)):
            ch = mp.matmul_block(Ah, Bh, args.nmin)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ch = mp.matmul_block(Ah, Bh, args.nmin)
        e2e_s = time.perf_counter() - t0
    else:
        for _ in range(max(3, args.warmup)):
            ch = shard.sharded_matmul_host(host_a, host_b if rank == 0 else None, n, n, prec,
                                           n_min=args.nmin)
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ch = shard.sharded_matmul_host(host_a, host_b if rank == 0 else None, n, n, prec,
                                           n_min=args.nmin)
        dist.barrier()
        e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = 2.0 * madds_step * e2e_steps / te.item()
    elem = 8 * comps
    h2d = elem * (n * n * world + n * n)
    d2h = elem * n * n * world + 4 * world

    if rank != 0:
        return
    peak = fp64_peak(torch, _cuda, dev)
    achieved = F * float(n) ** 3 / kernel_s / 1e12
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak["dfma"],
                "unit": "TFLOP/s", "frac": achieved / peak["dfma"],
                "traffic": load_ncu_traffic(args.prec),
                "peak_source": "in-run DFMA burst micro-benchmark (MEASURED_PEAKS.json has "
                               "no FP64 entry)",
                "peak_dadd_tflops": peak["dadd"], "peak_spec_tflops": SPEC_FP64_TFLOPS,
                "flops_per_madd": F, "kernel_ms": kernel_s * 1e3,
                "fp64_issue_frac_of_dfma_peak": (I_DD if args.prec == "dd" else None) and
                (I_DD * 2 * float(n) ** 3 / kernel_s / 1e12 / peak["dfma"])}
    line = {
        "metric": metric_name(args), "value": value, "unit": "2mnl/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "e2e": {"value": e2e_value, "unit": "2mnl/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "api": "paper_1710_01839_b200.matmul_block(host, host) -> C-ABI mpmm_gemm_host "
                       "(one GEMM launch consuming 64-column k-panels as their H2D lands, C "
                       "written to the page-locked result from the epilogues)" if world == 1 else
                       "shard.sharded_matmul_host"},
        "roofline": roofline,
        "gpu_launches": gemm_launches,
        "tuner": tuner,
        "wall_s_timed_region": t_wall,
        "clocks": clocks,
    }
    if fast_s is not None:
        line["fast_mode"] = {
            "what": "opt-in faithful DD sequence (15 FP64 instr, F=18 flop/madd), within "
                    "4*l*u*(|A||B|), u=2^-104; NOT bit-identical to the reference",
            "value": 2.0 * float(n) ** 3 * world / fast_s, "unit": "2mnl/s",
            "kernel_ms": fast_s * 1e3,
            "roofline_frac": 18 * float(n) ** 3 / fast_s / 1e12 / peak["dfma"]}
    if tensor_s is not None:
        line["tensor_mode"] = {
            "what": "opt-in exact mode: int8 tensor-core residue GEMMs (CRT, hand-written tcgen05) + "
                    "tensor-core CRT sums (mma.sync) + exact reconstruction, product rounded "
                    "once; more accurate than, not bit-identical to, the reference",
            "value": 2.0 * float(n) ** 3 * world / tensor_s, "unit": "2mnl/s",
            "ms": tensor_s * 1e3,
            "jobs": [{"a_comps": list(ra), "b_comps": list(rb), "moduli": N}
                     for ra, rb, N in tensor_jobs]}
    else:
        line["tensor_mode"] = {"unavailable": tensor_err}
    if world == 1 and not args.no_cpu_baseline:
        v, cores, kind, sample, _ = cpu_reference_run(args.prec, n, args.nmin, args.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": "2mnl/s", "cores": cores, "kind": kind,
                                "sample": sample}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.same_device:
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(args.dist_backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
