#!/usr/bin/env python3
"""Benchmark of the B200 Strassen DGEMM (driver contract).

One step = one strassen_gemm call (C := alpha A B + C) on the workload
m = n = k = 16384, column-major fp64, uniform[-1, 1) synthetic inputs
(BASELINE.json configs[1], top of the square sweep; it fits one GPU).
Default: two-level Strassen, Naive variant (batched: all operand sums in one
HBM pass, all 49 products in one launch, one stream pass) -- the fastest
configuration measured on B200 (profiles/r01_notes.md).  Every other
variant/level is timed on the same inputs and reported under "variants".
Prints ONE JSON line on rank 0.

  value     effective FP64 TFLOP/s (2mnk / t, summed over ranks), device
            pointers, inputs resident in HBM, CUDA events on the launch stream
  e2e       the same metric through the C ABI with pinned HOST buffers:
            H2D of A, B, C and D2H of C inside the timed region
  roofline  executed flops of the mm_kernel launch / its CUDA-event duration
            vs the measured FP64 DMMA peak (profiles/fp64_peaks.json)
  cpu_baseline  the reference library itself (oracle/_ref, compiled from the
            reference sources with its own flags) on a bounded sample
  --impl reference  times that reference CPU path alone (rank 0).

Multi-GPU (N > 1): BASELINE config 5, SUMMA over NCCL (paper_1605_01078_b200/
summa.py) with local two-level ABC Strassen.  `python bench.py --gpus N` re-executes
itself under torchrun (one rank per GPU, 127.0.0.1 rendezvous) when it is not already
running under it, and every rank checks WORLD_SIZE == N.  The pr x pc grid comes from
grid_for(N) (1x2, 2x2, 2x4); rank (i, j) owns the (i, j) blocks of A, B and C.  A panels
are broadcast along process rows and B panels along process columns, double-buffered
against the local rank-b updates (panel width b = 8192; a panel straddling the columns
a rank owns is assembled from per-owner pieces).  Two problems per run:
  value         m = n = k = 65536 (config 5's fixed size; total work fixed: "strong")
  weak_scaled   m = n = k = 32768 * sqrt(N) rounded to the nearest multiple of 256
                (46336, 65536, 92672 at N = 2, 4, 8): config 5's weak-scaled variant
Time = max over ranks of CUDA-event step times; value = total flops / that time.
--summa runs the same path at N = 1 (a 1 x 1 grid, no collectives); --dry-run runs
the launcher, grid, layout and timing logic on CPU ranks over gloo with a dense
local update (tests/test_bench_launcher.py).
"""
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

CPU_SAMPLE = 0  # bounded reference sample edge; 0 = adaptive (about 3 s per call, <= 4096)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    # default: naive level 2 at N = 1 (the headline); abc level 2 for SUMMA (config 5)
    p.add_argument("--variant", default=None, choices=["dgemm", "abc", "ab", "naive", "c"])
    p.add_argument("--level", type=int, default=2)
    p.add_argument("--no-variants", action="store_true")
    p.add_argument("--dim", type=int, default=16384)
    p.add_argument("--m", type=int, default=0)
    p.add_argument("--n", type=int, default=0)
    p.add_argument("--k", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-classical", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=CPU_SAMPLE)
    # run the N > 1 SUMMA code path even at N = 1 (a 1 x 1 grid, no collectives):
    # a one-GPU check of the multi-GPU bench mechanics
    p.add_argument("--summa", action="store_true")
    p.add_argument("--p2p", action="store_true",
                   help="N > 1: peer-memory SUMMA (operands read from the owners' blocks "
                        "over CUDA IPC, no NCCL broadcasts; summa.summa_p2p)")
    p.add_argument("--native", action="store_true",
                   help="SUMMA through the library's native entry point (strassen_dist_gemm, "
                        "include/strassen_dist.h: NCCL from C++, no Python in the schedule)")
    p.add_argument("--summa-size", default="both", choices=["strong", "weak", "both"],
                   help="SUMMA problems: config 5's fixed 65536^3 (strong), its weak-scaled "
                        "32768*sqrt(N) variant, or both (value = strong)")
    p.add_argument("--dry-run", action="store_true",
                   help="CPU ranks over gloo, dense local update: launcher/layout/timing test")
    a = p.parse_args()
    summa_path = a.gpus > 1 or a.summa or a.dry_run
    if a.variant is None:
        a.variant = "abc" if summa_path else "naive"
    if a.variant == "dgemm":
        a.level = 0
    a.user_dims = bool(a.m or a.n or a.k or a.dim != 16384)
    a.m = a.m or a.dim
    a.n = a.n or a.dim
    a.k = a.k or a.dim
    return a


def weak_dim(p, base=32768, mult=256):
    """Config 5's weak-scaled size 32768 * sqrt(P), rounded to the nearest multiple of
    256 (so every local dimension on the 1x2 / 2x2 / 2x4 grids stays a multiple of
    2^L * 32): 32768, 46336, 65536, 92672 for P = 1, 2, 4, 8."""
    import math
    return int(round(base * math.sqrt(p) / mult)) * mult


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` outside torchrun: re-execute this command under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous)."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def table_counts(level):
    # level 3 (naive / c only): 343 products; its C updates are those of the seven
    # level-2 calls (7 x 144 at the inner quadrant size) -- the outer level is a
    # stream pass, not mm_kernel work
    return {0: (1, 0, 0, 1), 1: (7, 5, 5, 12), 2: (49, 95, 95, 144), 3: (343, 0, 0, 1008)}[level]


def executed_flops(m, n, k, level, variant="abc"):
    """Flops the mm_kernel launch executes (implementation
    counts, 144 C updates at level 2).  abc: products + fused operand sums +
    fused C updates; ab: no C updates (streamed); c: no operand sums
    (materialised); naive: products only."""
    if level == 0:
        return 2.0 * m * n * k
    s = 1 << level
    qm, qn, qk = -(-m // s), -(-n // s), -(-k // s)
    mul, aa, ba, cu = table_counts(level)
    f = mul * 2.0 * qm * qn * qk
    if variant in ("abc", "ab"):
        f += 2.0 * (aa * qm * qk + ba * qk * qn)
    if variant in ("abc", "c"):
        f += 2.0 * cu * qm * qn
    return f


# sum over multi-term operands of (terms + 1): read every term, write the sum
# (per side; L1 term histogram {1: 2, 2: 5}, L2 {1: 4, 2: 20, 4: 25})
# multi-term operand sums per side (= materialised outputs of one sum pass)
MULTI_TERM_SUMS = {1: 5, 2: 45}


def hbm_bytes(kernel, m, n, k, level, ordinal=0):
    """Algorithmic HBM bytes of the auxiliary launches.

    sum pass (gather form): every source quadrant read once + every sum written once;
    stream pass: every M_p read once + each C element read and written once.
    """
    if level > 2:  # sum / stream passes at two levels of the recursion: not tabulated
        return None
    s = 1 << level
    qm, qn, qk = -(-m // s), -(-n // s), -(-k // s)
    mul, aa, ba, cu = table_counts(level)
    if kernel == "sum_gather_kernel" and level > 0:  # ordinal 0: A side, 1: B side
        quads = s * s + MULTI_TERM_SUMS[level]
        return 8.0 * quads * (qm * qk if ordinal == 0 else qk * qn)
    if kernel == "stream_gather_kernel":
        return 8.0 * (mul * qm * qn + 2 * m * n)
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def ref_variant(variant):
    """The reference has no "c" variant (a B200 addition): its arm runs ABC."""
    return "abc" if variant == "c" else variant


def reference_cpu(dim, variant, level, reps=2, warmup=1, target_s=3.0):
    """The reference library itself on the host cores (bounded sample).

    dim = 0 picks the sample edge adaptively: time one 1024^3 call, then scale
    (O(n^3)) to about target_s per call, rounded to 256 and capped at 4096.
    """
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np

    import oracle_lib as O
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_PROC_BIND", "close")
    kind, path = "reference", O.REF_SO
    if not O.RefStrassen.available():
        raise RuntimeError("oracle/_ref/libstrassen_ref.so missing (make -C oracle ref)")
    ref = O.RefStrassen(path)
    ref.set_threads(cores)
    variant = ref_variant(variant)
    if not dim:
        rng = np.random.default_rng(1)
        x = np.asfortranarray(rng.uniform(-1, 1, (1024, 1024)))
        y = x.copy(order="F")
        t0 = time.perf_counter()
        ref.gemm(variant, level, 1.0, x, x, y)
        t1 = time.perf_counter() - t0
        dim = int(1024 * (target_s / max(t1, 1e-3)) ** (1.0 / 3.0)) // 256 * 256
        dim = max(1024, min(4096, dim))
    rng = np.random.default_rng(0)
    a = np.asfortranarray(rng.uniform(-1, 1, (dim, dim)))
    b = np.asfortranarray(rng.uniform(-1, 1, (dim, dim)))
    c = np.asfortranarray(rng.uniform(-1, 1, (dim, dim)))
    times = []
    for i in range(warmup + reps):
        t0 = time.perf_counter()
        ref.gemm(variant, level, 1.0, a, b, c)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return {"kind": kind, "cores": cores, "times": times, "dim": dim,
            "sample": f"m=n=k={dim} {variant}{level} via the reference C ABI "
                      f"(oracle/_ref, -O3 -DNDEBUG -fopenmp, threads={cores}), column-major, "
                      f"uniform[-1,1); best of {reps} after {warmup} warm-up"}


def run_reference(args, rank):
    if rank != 0:
        return
    r = reference_cpu(args.cpu_sample, args.variant, args.level, reps=args.steps,
                      warmup=args.warmup)
    dim = r["dim"]
    t = sum(r["times"]) / len(r["times"])
    tf = 2.0 * dim ** 3 / t / 1e12
    line = {
        "impl": "reference", "metric": "effective FP64 TFLOPS (2mnk/t)", "value": tf,
        "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic uniform[-1,1)",
        "config": {"workload": f"square m=n=k={args.m} {args.variant} level {args.level} "
                   f"(bounded CPU sample m=n=k={dim}; reference variant "
                   f"{ref_variant(args.variant)})", "variant": args.variant,
                   "level": args.level, "m": dim, "n": dim, "k": dim},
        "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)  # does not return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return run_summa_dry(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1605_01078_b200 as S
    torch.cuda.set_device(local)
    if world > 1 or args.summa:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # comm-init lines (ranks, NVLS, P2P)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    m, n, k = args.m, args.n, args.k
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)

    def colmajor(r, c):
        x = torch.empty((c, r), dtype=torch.float64, device="cuda")
        x.uniform_(-1.0, 1.0, generator=g)
        return x.t()  # (r, c) with strides (1, r)

    ctx = S.Ctx()
    ctx.set_max_level(3)  # admits naive3 / c3 (B200 extension) beside the reference's levels
    stream = torch.cuda.current_stream()
    if world > 1 or args.summa:
        return run_summa(args, rank, world, local, colmajor, barrier, max_over_ranks)
    A, B, C = colmajor(m, k), colmajor(k, n), colmajor(m, n)

    def time_device(variant, level, steps, warmup):
        for _ in range(warmup):
            ctx.gemm_device(variant, level, 1.0, A, B, C, stream)
        barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for e0, e1 in evs:
            e0.record(stream)
            ctx.gemm_device(variant, level, 1.0, A, B, C, stream)
            e1.record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
        total_ms = t0.elapsed_time(t1)
        per = [e0.elapsed_time(e1) for e0, e1 in evs]
        return total_ms, per, ctx.last_launches()

    with ClockSampler(local) as clk:
        total_ms, per_ms, launches = time_device(args.variant, args.level, args.steps, args.warmup)
    total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / args.steps
    flops = 2.0 * m * n * k
    value = world * flops / (ms_per_step * 1e-3) / 1e12

    # roofline of the dominant kernel (mm_kernel), timed by the library's own
    # per-launch CUDA events on the launch stream (one extra profiled step)
    peaks = json.load(open(os.path.join(ROOT, "profiles", "fp64_peaks.json")))
    # -- averaged over `steps` profiled steps issued back to back, like the timed region
    ctx.enable_profiling(True)
    profs = []
    for _ in range(max(1, args.steps)):
        ctx.gemm_device(args.variant, args.level, 1.0, A, B, C, stream)
        torch.cuda.synchronize()
        profs.append(ctx.last_profile())
    ctx.enable_profiling(False)
    prof = [dict(x) for x in profs[0]]
    if all(len(p) == len(prof) for p in profs):
        for i, x in enumerate(prof):
            x["ms"] = statistics.mean(p[i]["ms"] for p in profs)
    mm_ms = [x["ms"] for x in prof if x["kernel"] == "mm_kernel"]
    kern_ms = sum(mm_ms) if mm_ms else statistics.mean(per_ms)
    f_exec = executed_flops(m, n, k, args.level, args.variant)
    achieved = f_exec / (kern_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath))
        key = f"{args.variant}{args.level}_{m}x{n}x{k}"
        if key in t:
            traffic = t[key]
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["dmma_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["dmma_tflops"], "traffic": traffic,
                "flops_per_launch": f_exec, "kernel_ms": kern_ms, "kernel": "mm_kernel",
                "launches_per_step": launches, "step_profile_ms": prof,
                "profiled_steps": len(profs),
                "peak_source": "measured FP64 DMMA peak, profiles/fp64_peaks.json "
                               "(MEASURED_PEAKS.json has bf16/HBM only)"}
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm_peak = 6442.2
    seen = {}
    for x in prof:
        nb = hbm_bytes(x["kernel"], m, n, k, args.level, seen.get(x["kernel"], 0))
        seen[x["kernel"]] = seen.get(x["kernel"], 0) + 1
        if nb and x["ms"] > 0:
            roofline.setdefault("aux_hbm", []).append(
                {"kernel": x["kernel"], "achieved_gbs": nb / (x["ms"] * 1e-3) / 1e9,
                 "peak_gbs": hbm_peak, "frac": nb / (x["ms"] * 1e-3) / 1e9 / hbm_peak})

    line = {
        "metric": "effective FP64 TFLOPS (2mnk/t)", "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic uniform[-1,1) (torch generator, column-major, inputs > L2)",
        "config": {"workload": f"square m=n=k={m}" if m == n == k else f"{m}x{n}x{k}",
                   "variant": args.variant, "level": args.level, "m": m, "n": n, "k": k,
                   "layout": "column-major lda=m", "alpha": 1.0, "beta": 1.0,
                   "l2": "inputs (3 x 2 GiB) larger than the 126 MB L2",
                   "parallelism": "replicas" if world > 1 else "single"},
        "roofline": roofline, "clocks": clk.summary(),
        "gpu_launches": launches * args.steps,
    }

    if not args.no_variants:
        table = {}
        for v, lv in [("dgemm", 0), ("abc", 1), ("ab", 1), ("naive", 1), ("c", 1), ("abc", 2),
                      ("ab", 2), ("naive", 2), ("c", 2), ("naive", 3), ("c", 3)]:
            tt, _, _ = time_device(v, lv, 2, 1)
            t_ms = max_over_ranks(tt) / 2
            table[f"{v}{lv}"] = {"value": world * flops / (t_ms * 1e-3) / 1e12, "ms": t_ms}
        line["variants"] = table

    if not args.no_classical and args.variant != "dgemm":
        c_total, c_per, _ = time_device("dgemm", 0, max(2, args.steps // 2), 1)
        c_ms = max_over_ranks(c_total) / max(2, args.steps // 2)
        line["classical"] = {"variant": "dgemm (this library's B200 classical kernel)",
                             "value": world * flops / (c_ms * 1e-3) / 1e12, "ms_per_step": c_ms}
        # cuBLAS DGEMM via torch for context (library ceiling, not our path)
        D = torch.empty_like(C)
        for _ in range(2):
            torch.matmul(A, B, out=D)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            torch.matmul(A, B, out=D)
        e1.record()
        torch.cuda.synchronize()
        cb = e0.elapsed_time(e1) / 3
        line["cublas_dgemm"] = {"value": flops / (cb * 1e-3) / 1e12, "ms_per_step": cb}
        del D

    if not args.no_e2e:
        # end to end through the C ABI with pinned host buffers: H2D(A, B, C) + D2H(C)
        Ah = A.t().cpu().pin_memory().t()
        Bh = B.t().cpu().pin_memory().t()
        Ch = C.t().cpu().pin_memory().t()
        e2e_steps = max(2, min(args.steps, 3))
        ctx.gemm(args.variant, args.level, 1.0, Ah, Bh, Ch)  # warm (staging buffers)
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ctx.gemm(args.variant, args.level, 1.0, Ah, Bh, Ch)
        dt = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
        line["e2e"] = {"value": world * flops / dt / 1e12, "unit": "TFLOP/s",
                       "h2d_bytes_per_step": 8 * (m * k + k * n + m * n),
                       "d2h_bytes_per_step": 8 * m * n, "ms_per_step": dt * 1e3,
                       "api": "strassen_gemm (C ABI, pinned host pointers)"}
        line["gpu_launches"] += ctx.last_launches() * e2e_steps
        # the link the e2e number rides on: pinned H2D / D2H of one operand (2 GiB at 16384)
        dev = torch.empty_like(A)
        for kind, (dst, src) in (("h2d_gbs", (dev, Ah)), ("d2h_gbs", (Ch, dev))):
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            line["e2e"][kind] = 8 * A.numel() / (time.perf_counter() - t1) / 1e9
        del dev

    if rank == 0 and world == 1 and not args.no_cpu:
        r = reference_cpu(args.cpu_sample, args.variant, args.level)
        t = min(r["times"])
        line["cpu_baseline"] = {"value": 2.0 * r["dim"] ** 3 / t / 1e12, "unit": "TFLOP/s",
                                "cores": r["cores"], "kind": r["kind"], "sample": r["sample"]}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def summa_problems(args, world):
    """(name, m, n, k) of the SUMMA problems this run measures (config 5)."""
    if args.user_dims:  # explicit --dim / --m / --n / --k (one-GPU checks, experiments)
        return [("strong", args.m, args.n, args.k)]
    out = []
    if args.summa_size in ("strong", "both"):
        out.append(("strong", 65536, 65536, 65536))
    if args.summa_size in ("weak", "both"):
        d = weak_dim(world)
        out.append(("weak", d, d, d))
    return out


def run_summa(args, rank, world, local, colmajor, barrier, max_over_ranks):
    """N > 1 (or --summa): BASELINE config 5 -- SUMMA with local Strassen updates
    (see the module doc for the problems and the timing)."""
    import torch

    from paper_1605_01078_b200 import summa as SU
    peaks = json.load(open(os.path.join(ROOT, "profiles", "fp64_peaks.json")))
    local_gemm = SU._default_local_gemm(args.variant, args.level)
    results = {}
    line = None
    native_grid = None
    for name, gm, gn, gk in summa_problems(args, world):
        L = SU.make_layout(gm, gn, gk, world)
        comm = SU.TorchComm(L) if (world > 1 or args.summa) and not args.native else None
        A_l, B_l, C_l = colmajor(L.m_l, L.k_c), colmajor(L.k_r, L.n_l), colmajor(L.m_l, L.n_l)
        if args.p2p:
            torch.cuda.synchronize()
            Ap, Bp = SU.open_peer_blocks(A_l, B_l)
            barrier()
            step = lambda: SU.summa_p2p(L, rank, Ap, Bp, C_l, 1.0, args.variant,  # noqa: E731
                                        args.level, local_gemm=local_gemm)
        elif args.native:
            if native_grid is None:   # one NCCL job (world + row + column comms) per run
                native_grid = (SU.NativeGrid.from_torch_distributed(local_gemm.ctx, L.pr, L.pc)
                               if world > 1 else
                               SU.NativeGrid.nccl(local_gemm.ctx, SU.NativeGrid.unique_id(), 0, 1,
                                                  1, 1))
            step = lambda: native_grid.gemm(args.variant, args.level, L.m, L.n,  # noqa: E731
                                            L.k, 1.0, A_l, B_l, C_l, panel=L.b)
        else:
            step = lambda: SU.summa(L, comm, A_l, B_l, C_l, 1.0, args.variant,  # noqa: E731
                                    args.level, local_gemm=local_gemm)
        for _ in range(args.warmup):
            step()
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launches = 0
            for _ in range(args.steps):
                launches += step()
            e1.record()
            torch.cuda.synchronize()
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        flops = 2.0 * L.m * L.n * L.k
        res = {"m": L.m, "n": L.n, "k": L.k, "grid": [L.pr, L.pc], "panel_b": L.b,
               "local": [L.m_l, L.n_l, L.b], "value": flops / (ms * 1e-3) / 1e12,
               "ms_per_step": ms, "gpu_launches": launches, "clocks": clk.summary()}
        if line is None:
            # roofline of the local update's mm_kernel: one profiled panel-shaped local
            # call (m_l x n_l x b) on this rank, timed by the library's events on the
            # launch stream; min over ranks
            lctx = local_gemm.ctx
            ap, bp = colmajor(L.m_l, L.b), colmajor(L.b, L.n_l)
            lctx.enable_profiling(True)
            lctx.gemm_device(args.variant, args.level, 1.0, ap, bp, C_l,
                             torch.cuda.current_stream())
            torch.cuda.synchronize()
            prof = lctx.last_profile()
            lctx.enable_profiling(False)
            del ap, bp
            mm_ms = sum(x["ms"] for x in prof if x["kernel"] == "mm_kernel")
            f_exec = executed_flops(L.m_l, L.n_l, L.b, args.level, args.variant)
            achieved = max_over_ranks(-(f_exec / (mm_ms * 1e-3) / 1e12)) * -1.0
            roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["dmma_tflops"],
                        "unit": "TFLOP/s", "frac": achieved / peaks["dmma_tflops"],
                        "traffic": None, "flops_per_launch": f_exec, "kernel_ms": mm_ms,
                        "kernel": "mm_kernel",
                        "launches_per_step": launches // max(args.steps, 1),
                        "step_profile_ms": prof,
                        "scope": "one local update (m_l x n_l x b) per rank; min over ranks",
                        "peak_source": "measured FP64 DMMA peak, profiles/fp64_peaks.json"}
            line = {
                "metric": "effective FP64 TFLOPS (2mnk/t)", "value": res["value"],
                "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if name == "strong" else "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic uniform[-1,1) (torch generator, column-major)",
                "config": {"workload": f"BASELINE config 5: SUMMA m=n=k={L.m} on {L.pr}x{L.pc} "
                                       f"GPUs, local {args.variant} level {args.level}",
                           "variant": args.variant, "level": args.level, "m": L.m, "n": L.n,
                           "k": L.k, "panel_b": L.b, "grid": [L.pr, L.pc],
                           "parallelism": f"summa{L.pr}x{L.pc}",
                           "weak_rule": "weak_scaled: m=n=k = 32768*sqrt(N) rounded to the "
                                        "nearest multiple of 256",
                           "exchange": "peer memory (CUDA IPC), no broadcasts" if args.p2p
                           else "NCCL row/column panel broadcasts issued by the library "
                                "(strassen_dist_gemm)" if args.native
                           else "NCCL row/column panel broadcasts",
                           "l2": "inputs larger than the 126 MB L2"},
                "roofline": roofline, "clocks": res["clocks"], "gpu_launches": launches,
            }
            if not args.no_e2e:
                line["e2e"] = summa_e2e(args, L, A_l, B_l, C_l, step, local_gemm, barrier,
                                        max_over_ranks, world, flops)
        else:
            results[name] = res
        del A_l, B_l, C_l, step
        torch.cuda.empty_cache()
    if "weak" in results:
        line["weak_scaled"] = results["weak"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()


def summa_e2e(args, L, A_l, B_l, C_l, step, local_gemm, barrier, max_over_ranks, world, flops):
    """End to end: pinned host blocks in, one SUMMA step, the C block out."""
    import torch

    def pinned_like(x):  # column-major pinned host block holding x's values
        h = torch.empty((x.shape[1], x.shape[0]), dtype=torch.float64, pin_memory=True).t()
        h.copy_(x)
        return h
    Ah, Bh, Ch = (pinned_like(x) for x in (A_l, B_l, C_l))
    copy_stream = torch.cuda.Stream()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # A and B blocks first; C's copy overlaps the first local update's operand sums
    # and products (its kernels wait on ev_c right before they read C)
    with torch.cuda.stream(copy_stream):
        A_l.copy_(Ah, non_blocking=True)
        B_l.copy_(Bh, non_blocking=True)
        ev_ab = torch.cuda.Event()
        ev_ab.record(copy_stream)
        C_l.copy_(Ch, non_blocking=True)
        ev_c = torch.cuda.Event()
        ev_c.record(copy_stream)
    torch.cuda.current_stream().wait_event(ev_ab)
    if args.native:   # the library's first local update waits on C right before reading it
        local_gemm.ctx.set_operand_events(c=ev_c)
    else:
        local_gemm.c_ready = ev_c
    if args.p2p:  # peers read this rank's A and B: they land before any rank steps
        ev_ab.synchronize()
        barrier()
    step()
    Ch.copy_(C_l)
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0)
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": world * 8 * (L.m_l * L.k_c + L.k_r * L.n_l + L.m_l * L.n_l),
            "d2h_bytes_per_step": world * 8 * L.m_l * L.n_l, "ms_per_step": dt * 1e3,
            "api": ("summa_p2p()" if args.p2p else "strassen_dist_gemm" if args.native else "summa()")
            + " over strassen_gemm_device, pinned host blocks"}


def run_summa_dry(args, rank, world):
    """--dry-run: the multi-GPU launcher and SUMMA schedule on CPU ranks over gloo,
    with a dense local update -- checks the torchrun re-exec, the world-size check, the
    grid and config-5 sizes (scaled down 64x per dimension) and the max-over-ranks
    timing, and verifies the distributed product against a dense one."""
    import torch
    import torch.distributed as dist

    from paper_1605_01078_b200 import summa as SU
    dist.init_process_group("gloo")
    out = {}
    for name, gm, gn, gk in summa_problems(args, world):
        m, n, k = gm // 64, gn // 64, gk // 64
        L = SU.make_layout(m, n, k, world, b=max(1, k // 4))
        comm = SU.TorchComm(L)
        g = torch.Generator().manual_seed(5)
        A = torch.rand(m, k, dtype=torch.float64, generator=g) * 2 - 1
        B = torch.rand(k, n, dtype=torch.float64, generator=g) * 2 - 1
        C = torch.rand(m, n, dtype=torch.float64, generator=g) * 2 - 1
        a, b, c = (x.contiguous() for x in SU.local_blocks(L, rank, A, B, C))

        def upd(alpha, x, y, z):
            z.add_(alpha * (x @ y))
        for _ in range(args.warmup):
            SU.summa(L, comm, a, b, c.clone(), 1.0, local_gemm=upd)
        dist.barrier()
        t0 = time.perf_counter()
        cc = c.clone()
        for _ in range(args.steps):
            cc.copy_(c)
            SU.summa(L, comm, a, b, cc, 1.0, local_gemm=upd)
        dt = time.perf_counter() - t0
        t = torch.tensor([dt / args.steps], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        _, _, want = SU.local_blocks(L, rank, A, B, C + A @ B)
        err = torch.tensor([float((cc - want).abs().max())], dtype=torch.float64)
        dist.all_reduce(err, op=dist.ReduceOp.MAX)
        out[name] = {"m": m, "n": n, "k": k, "config5_m": gm, "grid": [L.pr, L.pc],
                     "ms_per_step": t.item() * 1e3, "max_abs_err": err.item()}
    if rank == 0:
        first = next(iter(out.values()))
        print(json.dumps({"metric": "effective FP64 TFLOPS (2mnk/t)", "dry_run": True,
                          "n_gpus": world, "world_size": dist.get_world_size(),
                          "value": 2.0 * first["m"] * first["n"] * first["k"]
                          / (first["ms_per_step"] * 1e-3) / 1e12,
                          "unit": "TFLOP/s", "problems": out, "variant": args.variant,
                          "level": args.level}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
