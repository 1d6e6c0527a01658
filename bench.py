#!/usr/bin/env python3
"""Benchmark: DD/QD GEMM 2mnl/s on B200 (BASELINE.json metric).

Workload (``config.workload``): BASELINE.json configs[4] at its largest
size, the DD GEMM m = l = n = 8192 on the seed-1 uniform inputs (SURVEY.md
s8d), computed by the bit-identical blocked mirror kernel (the kernel the
north_star's 50 % FP64-roofline target names) at the block size the GPU
predictor picks.  One product per step.  Inputs are 1 GiB per matrix, far
larger than the 126 MB L2, so no L2 flush is needed between steps.

Under torchrun with N ranks the problem is STRONG-scaled (north_star:
"near-linear scaling to 8 GPUs at m=n=l=8192"): rank r owns a contiguous
64-row-aligned block of C's rows and the matching rows of A; B (8192 x
8192 DD, 1 GiB) is broadcast from rank 0 over NCCL inside every step in
k-panels, each panel's GEMM accumulating as soon as it lands
(``shard.broadcast_matmul``).  ``value`` = 2mnl of the whole product / the
max over ranks of the device time.

Printed (rank 0, one JSON line):
* ``value``: device throughput (CUDA events on the launching stream);
* ``e2e``: the same metric through the public API with host buffers --
  ``matmul_block(host, host)`` at N = 1 (H2D of A and B and D2H of C inside
  the timed region), ``shard.sharded_matmul_host`` per rank at N > 1;
* ``roofline``: the GEMM kernel against the FP64 pipe.  MEASURED_PEAKS.json
  has no FP64 entry, so the peak is the nominal 148 SMs x 64 lanes x 2 flop
  x 1.965 GHz = 37.2 TFLOP/s (a DFMA burst measured in this run after the
  warm-up is reported beside it);
* ``cpu_baseline``: the reference's own compiled kernels (oracle/_ref) on
  all host cores, on the reference's own leading-rows slice, extrapolated
  with the reference's own predictor (predict.py:37-50) -- "CPU, predicted";
* sub-fields: the tuner's bit-identical pick (blocked or Strassen, effective
  2mnl/s), QD 8192^3, the opt-in exact tensor-core mode (not bit-identical),
  and BASELINE configs[1] (DD 1024^3).

``--impl reference`` times that reference CPU implementation alone, on the
same config, and loads nothing from this repo's package (no repo .so).
"""

import argparse
import importlib.util
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

METRIC = "DD/QD GEMM 2mnl/s at 1/2/4/8 B200; % of FP64 roofline; vs host-CPU ref"
F_DD = 53    # flops per DD multiply-add of the mirror kernel (4 DMUL, 3 DFMA, 43 DADD)
I_DD = 50    # FP64 instructions per DD multiply-add
F_QD = 796   # flops per QD multiply-add (10 DFMA, 13 DMUL, 763 DADD)
SPEC_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
CFG4_SEED = 1          # BASELINE configs[4]: "inputs as config 0 with seed 1"
REF_N_MIN = 64         # the reference's DEFAULT_BLOCK_SIZE (multiply.py:32)
ROW_ALIGN = 64         # shard alignment: the largest CTA tile height

# ~5 ms of GPU spin before each timed step (outside the events): the host
# enqueue of a step must finish before the device reaches the start event
HOST_SLACK_CYCLES = 10_000_000


def parse():
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--prec", default="dd", choices=["dd", "qd"])
    p.add_argument("--size", type=int, default=8192, help="m = l = n of the whole product")
    p.add_argument("--seed", type=int, default=CFG4_SEED)
    p.add_argument("--nmin", type=int, default=0,
                   help="block size; 0 = let the GPU predictor pick from 16..256")
    p.add_argument("--panel", type=int, default=1024,
                   help="k-panel rows of the B broadcast at N > 1 (0 = one panel)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true",
                   help="skip the tuner-pick / QD / configs[1] sub-fields")
    p.add_argument("--cpu-budget", type=float, default=200.0,
                   help="seconds the reference arm may spend in total")
    p.add_argument("--dist-backend", default="nccl")
    p.add_argument("--same-device", action="store_true",
                   help="every rank on cuda:0 (multi-rank logic test on one GPU, gloo)")
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
                 "--format=csv,noheader,nounits", "-lms", "200"],
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
# the reference CPU implementation (oracle/_ref) -- "CPU, predicted"
# ---------------------------------------------------------------------------

def _inputs_module():
    """paper_1710_01839_b200/inputs.py loaded by file path: numpy only, so
    the reference arm never imports the package (which would map the repo's
    CUDA library into the process)."""
    path = os.path.join(ROOT, "paper_1710_01839_b200", "inputs.py")
    spec = importlib.util.spec_from_file_location("_bench_inputs", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class ReferenceCPU:
    """The reference's blocked product (multiply.py:148-160 partitioning
    over its compiled _kernels.dd_block_cells, all host threads) on its own
    predictor slice: the leading slice_rows_for(n_min, m) rows of A times
    all of B, extrapolated by predict_full_time (predict.py:37-50)."""

    def __init__(self, prec, size, seed, n_min=REF_N_MIN, a=None, b=None):
        import numpy as np

        import oracle
        self.oracle = oracle
        self.kern = oracle.ref_kernels()
        self.kind = "reference" if self.kern is not None else "port"
        self.cores = len(os.sched_getaffinity(0))
        self.prec, self.size, self.n_min = prec, size, n_min
        self.mult = oracle.DEFAULT_SLICE_MULTIPLIER
        if a is None or b is None:
            a, b = _inputs_module().gemm_inputs(prec, size, size, size, seed=seed)
        # ordinary (pageable) numpy memory, as the reference itself runs;
        # see DESIGN.md s5 for how the CPU time depends on B's placement
        self.a, self.b = a, np.array(b, copy=True)

    def rows(self):
        return self.oracle.slice_rows_for(self.n_min, self.size, self.mult)

    def step(self, rows=None):
        """One timed slice; returns (predicted full seconds, slice seconds)."""
        import numpy as np
        rows = rows or self.rows()
        sl = np.array(self.a[:rows], copy=True)
        t0 = time.perf_counter()
        self.oracle.matmul_block(sl, self.b, self.n_min, threads=self.cores, kernels=self.kern)
        dt = time.perf_counter() - t0
        full = dt * self.size / rows   # predict_full_time with this slice's rows
        return full, dt

    def fit_budget(self, steps, budget_s):
        """Pick the slice multiplier so steps x slice fits the budget (the
        reference's predictor takes k as a parameter, predict.py:37)."""
        _, dt = self.step(rows=self.rows())
        while self.mult > 1 and dt * steps > budget_s:
            self.mult //= 2
            dt = dt / 2
        return dt

    def sample(self, slice_s):
        return (f"{self.prec.upper()} blocked n_min={self.n_min}, threads={self.cores}, operands "
                f"in pageable numpy memory: the "
                f"reference's predictor slice (leading {self.rows()} = {self.mult}*n_min rows "
                f"of A, {self.size}x{self.size}) times all of B in {slice_s:.2f} s, scaled by "
                f"m/rows = {self.size / self.rows():g} (predict.py:37-50): CPU, predicted; "
                f"kernels: {'oracle/_ref (the reference _kernels.pyx, compiled)' if self.kern else 'oracle C port'}")

    def value(self, full_s):
        return 2.0 * float(self.size) ** 3 / full_s


def run_reference(args, rank, world):
    if rank != 0:
        return
    steps = max(1, args.steps)
    ref = ReferenceCPU(args.prec, args.size, args.seed)
    ref.fit_budget(steps + args.warmup, args.cpu_budget)
    for _ in range(args.warmup):
        ref.step()
    fulls, slices = [], []
    for _ in range(steps):
        full, dt = ref.step()
        fulls.append(full)
        slices.append(dt)
    full = statistics.median(fulls)
    value = ref.value(full)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "2mnl/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": full * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "2mnl/s", "cores": ref.cores,
                         "kind": ref.kind, "sample": ref.sample(statistics.median(slices)),
                         "predicted_full_s": full},
        "e2e": {"value": value, "unit": "2mnl/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    return {"workload": f"BASELINE configs[4]: {args.prec.upper()} GEMM m=l=n={args.size}, "
                        f"seeded uniform inputs (seed {args.seed}), blocked algorithm "
                        "(bit-identical mirror of the reference kernels)",
            "prec": args.prec, "m": args.size, "l": args.size, "n": args.size,
            "parallelism": (f"C row-sharded over {world} GPUs (64-row aligned), B NCCL "
                            f"broadcast in {args.panel}-row k-panels" if world > 1 else
                            "1 GPU"),
            "l2": "inputs larger than L2 (1 GiB per DD matrix at 8192); no flush needed"
                  if args.size >= 4096 else "flushed between steps (256 MiB write)"}


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


def load_ncu_traffic(*keys):
    """DRAM bytes per launch of the first of ``keys`` present in the
    committed ncu summary (profiles/ncu_summary.json), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fp:
            summary = json.load(fp)
    except (OSError, ValueError):
        return None
    for key in keys:
        if key in summary:
            return summary[key].get("dram_bytes_per_launch")
    return None


def kernel_label(_cuda, comps, n_min):
    """The blocked kernel n_min selects, as its launch geometry."""
    try:
        g = _cuda.gemm_geometry(comps, _cuda.ALGO_BLOCK, n_min)
        ops = "DDOps" if comps == 2 else "QDOps"
        return (f"gemm_tiled<{ops}> blocked mirror, {g['tile_m']}x{g['tile_n']} CTA tile, "
                f"{g['threads']} threads, {g['ctas_per_sm']} CTAs/SM (n_min={n_min})")
    except Exception:  # noqa: BLE001 - a label only
        return f"blocked mirror, n_min={n_min}"


def timed(torch, fn, reps, flush=None, stream=None):
    """Per-call device seconds (CUDA events on ``stream``), one list entry
    per rep; the host enqueue is hidden behind a GPU spin."""
    stream = stream or torch.cuda.current_stream()
    evs = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        torch.cuda._sleep(HOST_SLACK_CYCLES)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        fn()
        e.record(stream)
        evs.append((s, e))
    torch.cuda.synchronize()
    return [s.elapsed_time(e) / 1e3 for s, e in evs]


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
    stream = torch.cuda.current_stream()
    prec = mp.PrecisionSpec.parse(args.prec)
    comps = prec.comps
    n = args.size
    F = F_DD if args.prec == "dd" else F_QD
    elem = 8 * comps

    # inputs on the device, bitwise the numpy generator's (csrc/rng.cu)
    A_full, B_full = inputs.gemm_inputs_device(args.prec, n, n, n, seed=args.seed, device=dev)
    shards = shard.row_shards(n, world, align=ROW_ALIGN)
    r0, r1 = shards[rank]
    A = A_full[r0:r1].contiguous()
    B = B_full if rank == 0 else torch.empty_like(B_full)
    if rank != 0:
        del B_full
    torch.cuda.synchronize()
    flush = None if n >= 4096 else torch.empty(64 * 1024 * 1024, dtype=torch.float32,
                                              device=dev)

    # step 1 of the reference tuner (tune.py:137-143) on the device, outside
    # the timed region: wave-aware slice prediction over the BASELINE sweep
    tuner = None
    if args.nmin <= 0:
        Bt = B if rank == 0 else B_full_for_tuning(torch, inputs, args, dev)
        t0 = time.perf_counter()
        best, recs = mp.select_block_size(
            DenseMatrix(r1 - r0, n, prec, A) if r1 > r0 else DenseMatrix(n, n, prec, A_full),
            DenseMatrix(n, n, prec, Bt), [16, 32, 64, 128, 256],
            policy=mp.TimingPolicy(warmup_runs=1, measured_runs=3, aggregator="min"))
        phase = time.perf_counter() - t0
        if world > 1:
            t_best = torch.tensor([best], dtype=torch.int64, device=dev)
            dist.broadcast(t_best, src=0)
            best = int(t_best.item())
        args.nmin = best
        tuner = {"chosen_n_min": best, "prediction_phase_wall_s": phase, "records": [
            {"n_min": r.n_min, "slice_rows": r.slice_rows, "slice_ms": r.slice_time_s * 1e3,
             "slice2_rows": r.slice2_rows, "slice2_ms": (r.slice2_time_s or 0.0) * 1e3,
             "superseded_slices_ms": r.extra_time_s * 1e3,
             "predicted_ms": r.predicted_full_s * 1e3} for r in recs]}
    if rank != 0 and world > 1:
        del A_full
    panel = args.panel if (args.panel > 0 and world > 1) else None
    panels = len(shard.panel_bounds(n, panel))

    def step():
        return shard.broadcast_matmul(A, B, n_min=args.nmin, src=0, panel_rows=panel)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # the in-run DFMA burst, right after the warm-up (a cross-check of the
    # nominal peak the roofline divides by; measured late in a long run it
    # reads low once the board is warm, which would inflate frac)
    burst = fp64_peak(torch, _cuda, dev) if rank == 0 else None

    sampler = ClockSampler(local_rank).start() if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    step_s = timed(torch, step, args.steps, flush)
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall0
    # the clocks line covers the timed region (the sub-measurements below
    # sample their own)
    clocks = sampler.stop() if sampler else None
    dev_s = sum(step_s)
    # per GEMM launch (one per k-panel): the EFT-domain scan, the DFMA
    # kernel and the gated Dekker kernel (which exits at once in-domain)
    gemm_launches = args.steps * panels * 3

    # kernel-only time of the GEMM launch (no broadcast) for the roofline
    rows_local = r1 - r0
    Ck = torch.empty((max(rows_local, 1), n, comps), dtype=torch.float64, device=dev)

    def kernel():
        if rows_local:
            _cuda.gemm_dev(comps, _cuda.ALGO_BLOCK, args.nmin, rows_local, n, n, A.data_ptr(),
                           n, B.data_ptr(), n, Ck.data_ptr(), n, False, None,
                           stream.cuda_stream)
    kernel_s = statistics.mean(timed(torch, kernel, 2 if n >= 4096 else 10, flush))
    del Ck

    t = torch.tensor([dev_s, t_wall, kernel_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s, t_wall, kernel_s = t.tolist()
    madds = float(n) ** 3
    value = 2.0 * madds * args.steps / dev_s

    # end-to-end through the public API with host buffers
    e2e_steps = 3 if n >= 4096 else 10
    if world == 1:
        host_a = A.cpu().pin_memory().numpy()
        host_b = B.cpu().pin_memory().numpy()
        Ah, Bh = DenseMatrix(n, n, prec, host_a), DenseMatrix(n, n, prec, host_b)
        ch = None
        for _ in range(2):   # pools, streams, the page-locked result buffers
            ch = mp.matmul_block(Ah, Bh, args.nmin)
        del ch
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ch = mp.matmul_block(Ah, Bh, args.nmin)
        e2e_s = time.perf_counter() - t0
        api = ("paper_1710_01839_b200.matmul_block(host, host) -> C-ABI mpmm_gemm_host (one "
               "GEMM launch consuming k-panels as their H2D lands, C written to the "
               "page-locked result from the epilogues, finite check fused)")
    else:
        host_a = A.cpu().pin_memory().numpy()
        host_b = B.cpu().pin_memory().numpy() if rank == 0 else None
        for _ in range(2):
            ch = shard.sharded_matmul_host(host_a, host_b, n, n, prec, n_min=args.nmin,
                                           panel_rows=panel)
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ch = shard.sharded_matmul_host(host_a, host_b, n, n, prec, n_min=args.nmin,
                                           panel_rows=panel)
        dist.barrier()
        e2e_s = time.perf_counter() - t0
        api = "shard.sharded_matmul_host (per rank: H2D of its A rows, B on rank 0, NCCL " \
              "broadcast of B in k-panels, GEMM, finite check, D2H of its C rows)"
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = 2.0 * madds * e2e_steps / te.item()
    h2d = elem * (n * n + n * n)           # all of A (over the ranks) + B once
    d2h = elem * n * n + 4 * world         # C + the finite flags

    # N > 1: the fused alternative to the broadcast -- every rank's GEMM
    # reads B straight from rank 0's HBM over peer memory (CUDA IPC,
    # shard.PeerOperand), no collective; reported beside the NCCL line
    peer = None
    if world > 1 and not args.no_extras:
        # every failure is made collective (the status all-reduce), so no
        # rank is left waiting in a barrier the others skipped
        pb, err = None, ""
        try:
            pb = shard.PeerOperand(B if rank == 0 else None, src=0)
            for _ in range(2):
                shard.peer_matmul(A, pb, n_min=args.nmin)
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001 - reported below
            err = f"{type(ex).__name__}: {ex}"
        okt = torch.tensor([0 if err else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if okt.item():
            dist.barrier()
            ps = sum(timed(torch, lambda: shard.peer_matmul(A, pb, n_min=args.nmin),
                           args.steps))
            dist.barrier()
            tp = torch.tensor([ps], dtype=torch.float64, device=dev)
            dist.all_reduce(tp, op=dist.ReduceOp.MAX)
            peer = {"what": "B read over peer memory (CUDA IPC mapping of rank 0's buffer) by "
                            "every rank's GEMM launch: no broadcast, same bits",
                    "value": 2.0 * madds * args.steps / tp.item(), "unit": "2mnl/s",
                    "ms_per_step": tp.item() / args.steps * 1e3}
        else:
            peer = {"unavailable": err or "another rank failed to map B"}
        if pb is not None:
            pb.close()
        else:
            dist.barrier()    # pairs with close()'s barrier on the ranks that mapped B

    extras = {}
    if peer is not None:
        extras["peer_mode"] = peer
    if rank == 0 and world == 1 and not args.no_extras:
        sub_sampler = ClockSampler(local_rank).start()
        extras = run_extras(args, torch, _cuda, mp, inputs, DenseMatrix, A, B, dev, stream,
                            kernel_s)
        extras["clocks_sub_measurements"] = sub_sampler.stop()
    if rank != 0:
        return
    peak = SPEC_FP64_TFLOPS
    rows_max = max(hi - lo for lo, hi in shards)
    achieved = F * float(rows_max) * n * n / kernel_s / 1e12
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": load_ncu_traffic(f"{args.prec}{n}_nmin{args.nmin}"),
                "traffic_source": "profiles/ncu_summary.json "
                                  f"['{args.prec}{n}_nmin{args.nmin}'] (ncu --set full of "
                                  "this launch, tools/prof_kernel.py)",
                "peak_source": "nominal 148 SMs x 64 FP64 lanes x 2 flop x 1.965 GHz: "
                               "MEASURED_PEAKS.json has no FP64 entry and the profiling "
                               "guide states no FP64 fallback; the strictest denominator "
                               "(the in-run DFMA burst is reported beside it)",
                "burst_dfma_tflops": burst["dfma"], "burst_dadd_tflops": burst["dadd"],
                "frac_of_burst": achieved / burst["dfma"],
                "flops_per_madd": F, "kernel_ms": kernel_s * 1e3,
                "kernel": kernel_label(_cuda, comps, args.nmin),
                "fp64_issue_frac": (I_DD * 2 * float(rows_max) * n * n / kernel_s / 1e12 / peak)
                if args.prec == "dd" else None}
    line = {
        "metric": METRIC, "value": value, "unit": "2mnl/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the workload only: identical in both arms (the block size is each
        # implementation's own tuned knob -- ours is under "block_size")
        "config": workload_config(args, world),
        "block_size": {"n_min": args.nmin,
                       "chosen_by": "GPU slice predictor (select_block_size)" if tuner
                                    else "--nmin"},
        "e2e": {"value": e2e_value, "unit": "2mnl/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps, "api": api},
        "roofline": roofline,
        "gpu_launches": gemm_launches,
        "tuner": tuner,
        "wall_s_timed_region": t_wall,
        "clocks": clocks,
    }
    for k, v in extras.items():
        if k != "peak_needed":
            line[k] = v
    for sub in ("qd", "cfg1"):
        if sub in line and "kernel_s" in line[sub]:
            ks = line[sub].pop("kernel_s")
            Fs = F_QD if sub == "qd" else F_DD
            sz = line[sub]["size"]
            line[sub]["roofline_frac"] = Fs * float(sz) ** 3 / ks / 1e12 / peak
    if world == 1 and not args.no_cpu_baseline:
        ref = ReferenceCPU(args.prec, n, args.seed, a=host_a[:REF_N_MIN * 2].copy(),
                           b=host_b)
        full, dt = ref.step()
        line["cpu_baseline"] = {"value": ref.value(full), "unit": "2mnl/s", "cores": ref.cores,
                                "kind": ref.kind, "sample": ref.sample(dt),
                                "predicted_full_s": full}
        # the same slice with B in page-locked (cudaHostAlloc) memory, where
        # this host runs the reference's kernel ~2x faster
        ref.b = host_b
        full_p, _ = ref.step()
        line["cpu_baseline"]["value_b_in_pinned_memory"] = ref.value(full_p)
    print(json.dumps(line), flush=True)


def B_full_for_tuning(torch, inputs, args, dev):
    """Non-source ranks tune against their own copy of B (generated, not
    received: the tuner runs before the timed broadcasts)."""
    return inputs.gemm_inputs_device(args.prec, args.size, args.size, args.size,
                                     seed=args.seed, device=dev)[1]


def run_extras(args, torch, _cuda, mp, inputs, DenseMatrix, A, B, dev, stream, block_s):
    """Sub-fields on one GPU: the tuner's bit-identical pick (Strassen
    cutoffs against the blocked time), QD at the same size, and BASELINE
    configs[1] (DD 1024^3 blocked)."""
    out = {}
    n = args.size
    prec = mp.PrecisionSpec.parse(args.prec)
    comps = prec.comps

    # (0) BASELINE configs[1]: DD 1024^3 blocked, seed 0, L2 flushed -- first,
    # before the long products below warm the GPU into its power cap
    if args.prec == "dd":
        s = 1024
        a1, b1 = inputs.gemm_inputs_device("dd", s, s, s, seed=0, device=dev)
        c1 = torch.empty((s, s, 2), dtype=torch.float64, device=dev)
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
        res = {}
        for nm in (32, 64):
            def g1():
                _cuda.gemm_dev(2, _cuda.ALGO_BLOCK, nm, s, s, s, a1.data_ptr(), s,
                               b1.data_ptr(), s, c1.data_ptr(), s, False, None,
                               stream.cuda_stream)
            timed(torch, g1, 3, flush)
            res[nm] = statistics.mean(timed(torch, g1, 20, flush))
        nm = min(res, key=res.get)
        out["cfg1"] = {"what": "BASELINE configs[1]: DD blocked m=l=n=1024, seed 0, L2 flushed",
                       "size": s, "n_min": nm, "value": 2.0 * s ** 3 / res[nm],
                       "unit": "2mnl/s", "ms": res[nm] * 1e3, "kernel_s": res[nm]}
        del a1, b1, c1, flush
    # (1) the tuner's step 2/3 at this size: blocked vs Strassen(cutoff)
    Ad, Bd = DenseMatrix(n, n, prec, A), DenseMatrix(n, n, prec, B)
    cand = [c for c in (n // 128, n // 64, n // 32, n // 16, n // 8, n // 4, n // 2) if c >= 64]
    strassen = []
    for cut in cand:
        mp.matmul_strassen(Ad, Bd, cut, args.nmin)
        torch.cuda.synchronize()
        # (min of two: the fused-leaf path jitters +-2.5 % run to run)
        t = min(timed(torch, lambda: mp.matmul_strassen(Ad, Bd, cut, args.nmin), 2))
        strassen.append({"cutoff": cut, "ms": t * 1e3, "value": 2.0 * float(n) ** 3 / t})
    best = min(strassen, key=lambda r: r["ms"]) if strassen else None
    if best is not None and best["ms"] < block_s * 1e3:
        pick = {"choice": f"strassen:{best['cutoff']}/{args.nmin}", "ms": best["ms"],
                "value": best["value"]}
    else:
        pick = {"choice": f"block:{args.nmin}", "ms": block_s * 1e3,
                "value": 2.0 * float(n) ** 3 / block_s}
    out["tuner_pick"] = dict(pick, unit="effective 2mnl/s", bit_identical=True,
                             candidates={"block": {"n_min": args.nmin, "ms": block_s * 1e3},
                                         "strassen": strassen})

    # (2) QD at the same size (one product; the kernel is warmed at 1024)
    if args.prec == "dd" and os.environ.get("BENCH_SKIP_QD") != "1":
        qd = mp.PrecisionSpec.qd()
        qn = n
        Aq, Bq = inputs.gemm_inputs_device("qd", qn, qn, qn, seed=args.seed, device=dev)
        # the block size from the same GPU predictor as the headline's
        tq0 = time.perf_counter()
        q_nmin, q_recs = mp.select_block_size(
            DenseMatrix(qn, qn, qd, Aq), DenseMatrix(qn, qn, qd, Bq), [16, 32, 64, 128, 256],
            policy=mp.TimingPolicy(warmup_runs=1, measured_runs=2, aggregator="min"))
        q_phase = time.perf_counter() - tq0
        Cq = torch.empty((qn, qn, 4), dtype=torch.float64, device=dev)

        def qd_gemm(m):
            _cuda.gemm_dev(4, _cuda.ALGO_BLOCK, q_nmin, m, qn, qn, Aq.data_ptr(), qn,
                           Bq.data_ptr(), qn, Cq.data_ptr(), qn, False, None,
                           stream.cuda_stream)
        qd_gemm(128)
        torch.cuda.synchronize()
        tq = min(timed(torch, lambda: qd_gemm(qn), 1))
        out["qd"] = {"what": f"QD blocked mirror m=l=n={qn}, seed {args.seed}, n_min={q_nmin}",
                     "size": qn, "value": 2.0 * float(qn) ** 3 / tq, "unit": "2mnl/s",
                     "ms": tq * 1e3, "kernel_s": tq, "flops_per_madd": F_QD, "n_min": q_nmin,
                     "prediction_phase_wall_s": q_phase,
                     "predicted_ms": {str(r.n_min): r.predicted_full_s * 1e3 for r in q_recs}}
        # the tuner's QD pick at this size (profiles/r02_cfg4_qd.tbl): Strassen
        # at cutoff 32, bit-identical to the reference's Strassen
        if os.environ.get("BENCH_SKIP_QD_STRASSEN") != "1":
            Aqd, Bqd = DenseMatrix(qn, qn, qd, Aq), DenseMatrix(qn, qn, qd, Bq)
            q_cut = 32
            mp.matmul_strassen(Aqd, Bqd, q_cut, q_nmin)
            torch.cuda.synchronize()
            tqs = min(timed(torch, lambda: mp.matmul_strassen(Aqd, Bqd, q_cut, q_nmin), 1))
            out["qd"]["tuner_pick"] = {"choice": f"strassen:{q_cut}/{q_nmin}", "ms": tqs * 1e3,
                                       "value": 2.0 * float(qn) ** 3 / tqs,
                                       "unit": "effective 2mnl/s", "bit_identical": True}
            del Aqd, Bqd
        del Aq, Bq, Cq

    # (3) the opt-in exact tensor-core mode on the same operands (int8
    # tcgen05 residue GEMMs + CRT, the exact product rounded once: within
    # the north_star bound, NOT bit-identical to the reference)
    try:
        from paper_1710_01839_b200.tensor import matmul_exact_tensors, release
        for _ in range(3):                       # plan, capture, replay
            matmul_exact_tensors(A, B)
        torch.cuda.synchronize()
        tt = statistics.median(timed(torch, lambda: matmul_exact_tensors(A, B), 3))
        out["tensor_mode"] = {
            "what": "opt-in exact mode (int8 tcgen05 residue GEMMs, CRT, exact product "
                    "rounded once): within 4*l*u*(|A||B|), more accurate than and NOT "
                    "bit-identical to the reference; not the headline",
            "value": 2.0 * float(n) ** 3 / tt, "unit": "2mnl/s", "ms": tt * 1e3}
        release()
    except Exception as ex:  # noqa: BLE001 - reported; the headline is unaffected
        out["tensor_mode"] = {"unavailable": f"{type(ex).__name__}: {ex}"}

    torch.cuda.empty_cache()
    return out


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
