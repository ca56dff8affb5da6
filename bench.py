#!/usr/bin/env python3
"""Benchmark of the vocabulary-parallel output layer (fwd+bwd) on B200.

Metric (BASELINE.json): vocab-layer fwd+bwd tokens/s at V=256k, h=4096 on
1/2/4/8 B200s.  One step = one Algorithm-2 (reduced-barrier) forward +
backward of the output layer over one microbatch of T=8192 synthetic tokens:
pass S (logits GEMM + fused stats epilogue, softmax', A = softmax' W_k), the
single C1 barrier (stats all-gather + merge, dX combine + all-reduce), the
loss and pass T (dW GEMM + ordered one-hot correction).  The vocabulary is
sharded over the N ranks (one process per GPU, NCCL over NVLink between
them); total work is fixed as N grows ("strong" scaling).

  python bench.py [--gpus N --steps K --warmup W]          # our sm_100a path
  python bench.py --impl reference [...]                    # reference CPU path
  torchrun --nproc-per-node N bench.py --gpus N [...]       # N > 1
  torchrun --nproc-per-node N bench.py --gpus N --dry-run   # N ranks on the visible GPU(s):
                                                            # loopback collectives, same code path

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "vocab-layer fwd+bwd tokens/s at V=256k,h=4096 @1/2/4/8 B200; % BF16 TC peak"
WORKLOAD = "vocab-parallel output layer fwd+bwd, Algorithm 2 (reduced barrier), vocab sharded over N GPUs"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--alg", choices=["alg2", "alg1", "naive"], default="alg2")
    ap.add_argument("--workload", choices=["output", "input"], default="output",
                    help="output: output layer fwd+bwd (headline); input: embedding gather + scatter-add (config 4)")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=256000)
    ap.add_argument("--cta-group", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-tokens", type=int, default=64)
    ap.add_argument("--cpu-sample-vocab", type=int, default=64000)
    ap.add_argument("--opt", action="append", default=[],
                    help="library option key=value (vp_ctx_set_option), e.g. raster_dx=16")
    ap.add_argument("--dry-run", action="store_true",
                    help="N>1 without N GPUs: ranks share the visible GPU(s) (round-robin) and exchange through the "
                         "library's loopback backend (CUDA IPC mailboxes) instead of NCCL; torch.distributed runs on "
                         "gloo.  Exercises the whole multi-rank path; the timing is not a scaling number.")
    ap.add_argument("--chunk-tokens", type=int, default=0,
                    help="alg2 in token chunks of this size with P held for one chunk (vp_run_alg2_chunked)")
    ap.add_argument("--ids", choices=["uniform", "zipf"], default="uniform",
                    help="input workload: token-id distribution (zipf: s=1.1 over the vocabulary)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region.

    The sampler process starts at construction (before the warm-up, so it is
    already producing samples when the timed region begins); `with sampler:`
    marks the timed region, and only samples whose nvidia-smi timestamps fall
    inside it are summarised."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.t0 = self.t1 = None
        self.lines = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.5)  # nvidia-smi start-up

    def __enter__(self):
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        time.sleep(0.12)  # let the sample that covers the region's end arrive
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def _in_region(self):
        import datetime
        keep, near = [], None
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except (ValueError, IndexError):
                continue
            if self.t0 - 0.05 <= ts <= self.t1 + 0.05:
                keep.append(f[1:])
            elif ts < self.t0:
                near = f[1:]
        return keep or ([near] if near else [])

    def summary(self):
        sm, pw, smax, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for f in self._in_region():
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            try:
                pw.append(float(f[2]))
            except ValueError:
                pass
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------------
# CPU side: the reference's own algorithm (oracle restatement), bounded sample
# ---------------------------------------------------------------------------
def cpu_reference_sample(T_s: int, h: int, V_s: int, p: int, reps: int = 1):
    """Times run_alg2 (VM.cpp:328-361, fp64, incl. the [T x V] softmax assembly)
    of the CPU oracle on a [T_s tokens x V_s vocab rows] slice; returns seconds."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np

    import oracle
    rng = np.random.default_rng(1234)
    X = rng.standard_normal((T_s, h))
    W = rng.standard_normal((V_s, h)) * 0.02
    g = rng.integers(0, V_s, T_s)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.run("alg2", X, g, W, p)
        times.append(time.perf_counter() - t0)
    return times, oracle.num_threads()


def host_info():
    """Host cores the CPU legs ran on (nproc, model name from lscpu)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    return info


def cpu_sample_shape(args, V):
    """The bounded CPU sample both CPU legs (--impl reference and cpu_baseline)
    time: the same T_s tokens x V_s vocab rows, so the two agree."""
    T_s, V_s = args.cpu_sample_tokens, min(args.cpu_sample_vocab, V)
    p = max(1, args.gpus)
    while V_s % p:
        V_s -= 1
    return T_s, V_s, p


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    T, h, V = args.tokens, args.hidden, args.vocab
    if args.workload == "input":
        return run_reference_input(args)
    T_s, V_s, p = cpu_sample_shape(args, V)
    times, cores = cpu_reference_sample(T_s, h, V_s, p, reps=args.warmup + args.steps)
    timed = times[args.warmup:]
    t = sum(timed) / len(timed)
    scale = V / V_s  # cost is linear in V (three T x h x V GEMMs + T x V elementwise)
    value = T_s / (t * scale)
    sample = (f"run_alg2 (fp64 CPU oracle restating VM.cpp:328-361) on {T_s} tokens x {V_s} of {V} vocab rows, "
              f"h={h}, p={p}; tokens/s scaled by {V_s}/{V} (cost linear in V); host {host_info()}")
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": "reference CPU path: " + WORKLOAD, "tokens": T, "hidden": h, "vocab": V,
                   "shards": p},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side: our sm_100a path through the C ABI
# ---------------------------------------------------------------------------
class Step:
    """Pre-marshalled call of vp_run_alg{1,2} / vp_naive_partitioned_output for
    one rank's shard (no per-step Python allocation or argument building)."""

    def __init__(self, ctx, alg, batch, shard, state, outs, chunk_tokens=0):
        from paper_2411_05288_b200._lib import vp_shard_t
        self.ctx = ctx
        loss, gx, gw, stats = outs
        self.batch_c = batch.c()
        self.shards_c = (vp_shard_t * 1)(shard.c())
        self.states_c = (ctypes.c_void_p * 1)(state.handle.value)
        self.gw_c = (ctypes.c_void_p * 1)(gw.data_ptr())
        lib = ctx.lib
        common_tail = [stats.c(), ctypes.c_void_p(loss.data_ptr()), ctypes.c_void_p(gx.data_ptr()), gx.stride(0),
                       self.gw_c, gw.stride(0)]
        head = [ctx.handle, ctypes.byref(self.batch_c), self.shards_c, self.states_c, 1]
        if alg == "naive":
            self.fn, self.args = lib.vp_naive_partitioned_output, head + common_tail
        else:
            fn = lib.vp_run_alg2 if alg == "alg2" else lib.vp_run_alg1
            self.fn, self.args = fn, head + [1.0] + common_tail
            if chunk_tokens:  # memory-bounded alg2 (vp_run_alg2_chunked)
                self.fn, self.args = lib.vp_run_alg2_chunked, head + [int(chunk_tokens), 1.0] + common_tail

    def __call__(self):
        rc = self.fn(*self.args)
        if rc:
            from paper_2411_05288_b200._lib import check
            check(rc)


def setup_rank(args, world, local):
    """This rank's GPU and process group: NCCL, one GPU per rank (the real
    run), or --dry-run: ranks round-robin over the visible GPUs, gloo for
    torch.distributed and the library's loopback backend for the data path."""
    import torch
    import torch.distributed as dist
    dev = local % torch.cuda.device_count() if args.dry_run else local
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dry_run:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dev


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2411_05288_b200 import dist as vpd
    from paper_2411_05288_b200 import vocab_math as vm

    rank, world, local = vpd.env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dev = setup_rank(args, world, local)
    # a side stream as the current stream: the library runs on it, and it can
    # be captured into a CUDA graph (the legacy default stream cannot)
    torch.cuda.set_stream(torch.cuda.Stream())
    T, h, V = args.tokens, args.hidden, args.vocab
    row_begin, row_end = vpd.shard_rows(vm.pad_vocab_size(V, world) if V % world else V, world, rank)
    rows = row_end - row_begin
    ctx = vm.Context(dev, cta_group=args.cta_group)
    for kv in args.opt:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    if world > 1:
        vpd.init_comm(ctx, loopback=args.dry_run)
    ctx.reserve(T, h, world)

    # synthetic inputs of the named shape (X~N(0,1), W~N(0,0.02^2), seed 1234)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    X = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    labels = torch.randint(0, V, (T,), device="cuda", generator=gen)
    gen.manual_seed(1234 + 1 + rank)
    W_k = (torch.randn(rows, h, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    shard = vm.EmbeddingShard(W_k, rank, row_begin, row_end)
    batch = vm.TokenBatch(X, labels)
    if args.chunk_tokens and args.alg != "alg2":
        raise SystemExit("--chunk-tokens needs --alg alg2")
    state = vm.ShardState(ctx, min(args.chunk_tokens, T) if args.chunk_tokens else T, h, rows)
    outs = (torch.empty(T, dtype=torch.float32, device="cuda"), torch.empty(T, h, dtype=torch.float32, device="cuda"),
            torch.empty(rows, h, dtype=torch.float32, device="cuda"), vm.GlobalStats.empty(T, "cuda"))
    step = Step(ctx, args.alg, batch, shard, state, outs, args.chunk_tokens)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier() if args.dry_run else dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        return vpd.max_over_ranks(x, device=None if args.dry_run else "cuda")

    # ---- device-resident throughput (value) ----
    clk = ClockSampler(dev)
    for _ in range(args.warmup):
        step()
    barrier()
    ctx.gemm_timing(True)
    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = ctx.launches - launches0
    gemm = ctx.gemm_timing(False)
    ms = max_over_ranks(ms)
    value = T / (ms / 1e3)

    # ---- the same step replayed as a CUDA graph (reported beside value) ----
    graph = None
    if not args.no_graph and world == 1:  # (multi-rank graph capture of NCCL calls: not exercised this round)
        try:
            g = vm.capture(ctx, step)
            for _ in range(args.warmup):
                g.launch()
            barrier()
            ev0.record(stream)
            for _ in range(args.steps):
                g.launch()
            ev1.record(stream)
            barrier()
            ms_g = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
            graph = {"value": T / (ms_g / 1e3), "unit": "tokens/s", "ms_per_step": ms_g,
                     "what": "the timed step captured once (vp_ctx_capture_*) and replayed per step"}
            g.close()
        except Exception as e:  # reported, never fatal for the bench line
            graph = {"error": str(e)[:200]}

    # ---- end-to-end through the public API with host buffers (e2e) ----
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        Lh = labels.cpu().pin_memory()
        loss_h = torch.empty(T, dtype=torch.float32).pin_memory()
        # Double-buffered inputs: step i+1's host->device copy runs on a copy
        # stream while step i computes (what a training loop's prefetch does);
        # every step's copy and its loss read-back stay inside the timed region.
        copy_stream = torch.cuda.Stream()
        bufs = [(torch.empty_like(X), torch.empty_like(labels)) for _ in range(2)]
        steps_e2e = [Step(ctx, args.alg, vm.TokenBatch(xd, ld), shard, state, outs, args.chunk_tokens)
                     for xd, ld in bufs]
        ready = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def issue_copy(i):
            b = i % 2
            copy_stream.wait_event(consumed[b])  # step i-2 is done with this buffer
            with torch.cuda.stream(copy_stream):
                bufs[b][0].copy_(Xh, non_blocking=True)
                bufs[b][1].copy_(Lh, non_blocking=True)
            ready[b].record(copy_stream)

        def run_step(i):
            b = i % 2
            stream.wait_event(ready[b])
            steps_e2e[b]()
            consumed[b].record(stream)
            loss_h.copy_(outs[0], non_blocking=True)

        def e2e_steps(n):
            copy_stream.wait_event(ev0)
            issue_copy(0)
            for i in range(n):
                if i + 1 < n:
                    issue_copy(i + 1)
                run_step(i)

        ev0.record(stream)
        e2e_steps(args.warmup)
        barrier()
        ev0.record(stream)
        e2e_steps(args.steps)
        ev1.record(stream)
        barrier()
        ms_e2e = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
        e2e = {"value": T / (ms_e2e / 1e3), "unit": "tokens/s", "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": Xh.numel() * 2 + Lh.numel() * 8, "d2h_bytes_per_step": loss_h.numel() * 4,
               "path": "vp_run_%s via ctypes (C ABI), pinned host X/labels -> HBM (double-buffered on a copy "
                       "stream, overlapping the previous step), loss -> host" % args.alg}

    if rank != 0:
        ctx.close()
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (tensor-bound GEMMs) ----
    peaks = measured_peaks()
    peak = peaks.get("bf16_tflops_sustained") if peaks else 1400.0
    peak_src = "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step)" if peaks else \
        "fallback (B200_PROFILING.md)"
    # each of K1 (logits), K3 (dX / A), K4 (dW); chunked alg2 launches each once per chunk
    chunks = -(-T // args.chunk_tokens) if args.chunk_tokens else 1
    flops_launch = 2.0 * T * h * rows / chunks
    kern = {}
    for name, (kms, n) in gemm.items():
        if n:
            kern[name] = {"launches": n, "avg_ms": kms / n, "tflops": flops_launch / (kms / n / 1e3) / 1e12}
    dom = max(kern, key=lambda k: kern[k]["avg_ms"] * kern[k]["launches"]) if kern else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if dom and os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{dom}:{T}x{h}x{rows}")
        except Exception:
            traffic = None
    achieved = kern[dom]["tflops"] if dom else None
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src, "flops_per_launch": flops_launch, "gemms": kern,
                "step_frac_of_peak": (6.0 * T * h * V / (ms / 1e3) / 1e12) / (world * peak),
                "step_frac_of_nominal_2250": (6.0 * T * h * V / (ms / 1e3) / 1e12) / (world * 2250.0)}
    if peaks and peaks.get("bf16_tflops") and achieved:
        roofline["frac_of_burst"] = achieved / peaks["bf16_tflops"]  # MEASURED_PEAKS bf16_tflops (burst)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        T_s, V_s, p_s = cpu_sample_shape(args, V)  # the --impl reference arm's sample
        # the same schedule as the --impl reference arm (W warm-up + K timed
        # samples), so the two CPU legs agree (sustained host clocks included)
        times, cores = cpu_reference_sample(T_s, h, V_s, p_s, reps=args.warmup + args.steps)
        t_s = statistics.mean(times[args.warmup:])
        cpu = {"value": T_s / (t_s * V / V_s), "unit": "tokens/s", "cores": cores, "kind": "port",
               "sample": (f"CPU oracle run_alg2 (fp64, restates VM.cpp:328-361) on {T_s} tokens x {V_s} of {V} "
                          f"vocab rows, h={h}, p={p_s}, mean of {args.steps} after {args.warmup} warm-up: {t_s:.2f} s; "
                          f"tokens/s scaled by {V_s}/{V} "
                          f"(the --impl reference arm's sample); host {host_info()}")}

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (X~N(0,1), W~N(0,0.02^2), uniform labels, seed 1234)",
        "config": {"workload": WORKLOAD.replace("Algorithm 2 (reduced barrier)", {
            "alg2": "Algorithm 2 (reduced barrier)", "alg1": "Algorithm 1 (2 barriers)",
            "naive": "naive 3-barrier"}[args.alg]),
            "alg": args.alg, "tokens": T, "hidden": h, "vocab": V, "vocab_rows_per_gpu": rows,
            **({"chunk_tokens": args.chunk_tokens,
                "P_bytes": 2 * min(args.chunk_tokens, T) * (rows + 63) // 64 * 64} if args.chunk_tokens else {}),
            "parallelism": f"vocab{world}", "operands": "bf16", "accum_and_stats": "fp32",
            "cta_group": args.cta_group, "options": args.opt,
            "l2": "inputs larger than L2 every step (W_k %.0f MB, P %.0f MB per GPU)" % (
                rows * h * 2 / 1e6, T * rows * 2 / 1e6)},
        "e2e": e2e, "graph": graph, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
        "clocks": clk.summary(), "comm": ctx.comm_backend,
    }
    pw = line["clocks"].get("power_w")
    if pw:  # median instantaneous board power in the timed region (the 1 kW cap sets the clock)
        line["energy"] = {"power_w": pw, "tokens_per_joule": value / (pw * world)}
    if world > 1:
        # C1 of the output layer: the fused reduce-scatter (dX epilogue -> the
        # token rows' owners over peer memory) or the dX all-reduce
        line["c1_exchange"] = ("fused: dX GEMM epilogue stores into the owners' peer buffers, owner combine, "
                               "grad_x pulled by copy engines" if ctx.fused_c1_count > 0 else "dX all-reduce")
    if args.dry_run:
        line["dry_run"] = ("N ranks shared %d visible GPU(s) through the loopback backend: a functional run of the "
                           "multi-rank path, not a scaling measurement" % torch.cuda.device_count())
    print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def input_ids(T, V, kind, gen):
    """Token ids of the input workload: uniform, or Zipf(s=1.1) over the
    vocabulary (rank k drawn with p ~ 1/k^1.1; ranks mapped to ids by a fixed
    random permutation, so hot rows land on every shard)."""
    import torch
    if kind == "uniform":
        return torch.randint(0, V, (T,), device="cuda", generator=gen)
    k = torch.arange(1, V + 1, device="cuda", dtype=torch.float64)
    probs = (1.0 / k.pow(1.1)).float()
    ranks = torch.multinomial(probs, T, replacement=True, generator=gen)
    perm = torch.randperm(V, device="cuda", generator=gen)
    return perm[ranks]


def cpu_input_sample(T, V, h):
    """The reference's input layer (oracle input_forward + input_backward, fp64,
    VM.cpp:227-251) on a T_s-token x V_s-row sample with the workload's
    tokens-per-row density (cost per token then transfers); returns
    (tokens/s, sample description, threads)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np

    import oracle
    V_s = min(V, 16000)
    T_s = max(1, round(T * V_s / V))
    rng = np.random.default_rng(1234)
    tok = rng.integers(0, V_s, T_s)
    W = rng.standard_normal((V_s, h)) * 0.02
    grad = rng.standard_normal((T_s, h))
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        oracle.input_forward(tok, W, 0)
        oracle.input_backward(grad, tok, V_s, 0)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times[1:])
    return T_s / t, (f"oracle input_forward + input_backward (fp64, VM.cpp:227-251) on {T_s} ids over {V_s} rows "
                     f"(the workload's ids/row density {T / V:.3f}), h={h}, mean of 2 after 1 warm-up: {t:.2f} s; "
                     f"host {host_info()}"), 1


def run_reference_input(args):
    T = args.tokens if args.tokens != 8192 else 16384
    h, V = args.hidden, args.vocab
    vals = []
    for _ in range(max(1, args.steps)):
        v, sample, cores = cpu_input_sample(T, V, h)
        vals.append(v)
    value = statistics.mean(vals)
    line = {"metric": "input-layer fwd+bwd tokens/s at V=256k,h=4096 (BASELINE configs[3])", "value": value,
            "unit": "tokens/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": T / value * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "reference CPU path: vocab-parallel input embedding", "tokens": T, "hidden": h,
                       "vocab": V},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def run_input(args):
    """BASELINE configs[3]: V=256000, h=4096, 16384 token ids.  One step =
    the input layer forward over the group (vp_input_forward_gathered: at N=1
    the masked 16-byte-vector gather; at N>1 owned rows written into
    peer-mapped buffers and every row pulled from its owner over NVLink) +
    the group backward (vp_input_backward_gathered: grad_out from rank 0, the
    first pipeline stage; each rank's deterministic ascending-i scatter-add of
    the rows its shard owns, accumulated into its embedding-gradient buffer as
    in training)."""
    import torch
    import torch.distributed as dist

    from paper_2411_05288_b200 import dist as vpd
    from paper_2411_05288_b200 import vocab_math as vm

    rank, world, local = vpd.env()
    dev = setup_rank(args, world, local)
    T = args.tokens if args.tokens != 8192 else 16384
    h, V = args.hidden, args.vocab
    row_begin, row_end = vpd.shard_rows(V, world, rank)
    rows = row_end - row_begin
    ctx = vm.Context(dev)
    for kv in args.opt:
        key, val = kv.split("=")
        ctx.set_option(key, int(val))
    if world > 1:
        vpd.init_comm(ctx, loopback=args.dry_run)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    tok = input_ids(T, V, args.ids, gen)
    grad = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    gen.manual_seed(1235 + rank)
    W_k = (torch.randn(rows, h, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    shard = vm.EmbeddingShard(W_k, rank, row_begin, row_end)
    emb = torch.empty(T, h, dtype=torch.bfloat16, device="cuda")
    dE = torch.zeros(rows, h, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    fwd_ms, bwd_ms = [], []

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier() if args.dry_run else dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return vpd.max_over_ranks(x, device=None if args.dry_run else "cuda")

    def step(timed=False):
        if timed:
            ev[0].record(stream)
        vm.input_forward_gathered(ctx, tok, shard, out=emb)
        if timed:
            ev[1].record(stream)
        vm.input_backward_gathered(ctx, grad if rank == 0 else None, tok, shard, root=0, h=h, out=dE,
                                   accumulate=True)
        if timed:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    ctx.sync()
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev)
    with clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    launches = ctx.launches - launches0
    for _ in range(3):  # per-phase split (separate, un-timed for the headline)
        step(timed=True)
        torch.cuda.synchronize()
        fwd_ms.append(ev[0].elapsed_time(ev[1]))
        bwd_ms.append(ev[1].elapsed_time(ev[2]))
    ctx.sync()
    e2e = None
    if not args.no_e2e:
        # ids + grad_out from pinned host memory every step, double-buffered on
        # a copy stream (step i+1's copies overlap step i, as a training loop's
        # prefetch does); one embedding row read back per step
        tok_h = tok.cpu().pin_memory()
        grad_h = grad.cpu().pin_memory()
        out_h = torch.empty(h, dtype=torch.bfloat16).pin_memory()
        copy_stream = torch.cuda.Stream()
        bufs = [(torch.empty_like(tok), torch.empty_like(grad)) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def issue_copy(i):
            b = i % 2
            copy_stream.wait_event(consumed[b])
            with torch.cuda.stream(copy_stream):
                bufs[b][0].copy_(tok_h, non_blocking=True)
                bufs[b][1].copy_(grad_h, non_blocking=True)
            ready[b].record(copy_stream)

        def e2e_steps(n):
            copy_stream.wait_event(e0)
            issue_copy(0)
            for i in range(n):
                if i + 1 < n:
                    issue_copy(i + 1)
                b = i % 2
                stream.wait_event(ready[b])
                vm.input_forward_gathered(ctx, bufs[b][0], shard, out=emb)
                vm.input_backward_gathered(ctx, bufs[b][1] if rank == 0 else None, bufs[b][0], shard, root=0,
                                           h=h, out=dE, accumulate=True)
                consumed[b].record(stream)
                out_h.copy_(emb[0], non_blocking=True)

        e0.record(stream)
        e2e_steps(args.warmup)
        barrier()
        e0.record(stream)
        e2e_steps(args.steps)
        e1.record(stream)
        barrier()
        me = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        e2e = {"value": T / (me / 1e3), "unit": "tokens/s", "ms_per_step": me,
               "h2d_bytes_per_step": tok_h.numel() * 8 + grad_h.numel() * 2, "d2h_bytes_per_step": h * 2,
               "path": "vp_input_forward_gathered / vp_input_backward_gathered via ctypes; ids + grad from pinned "
                       "host (double-buffered on a copy stream, overlapping the previous step)"}
    if rank != 0:
        ctx.close()
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs") if peaks else 6650.0
    owned_ids = int(((tok >= row_begin) & (tok < row_end)).sum().item())
    owned_rows = int(torch.unique(tok[(tok >= row_begin) & (tok < row_end)]).numel())
    fwd_bytes = 8 * T + 2 * h * owned_ids + 2 * h * T            # ids, owned rows read, full [T x h] written
    bwd_bytes = 8 * T + 2 * h * owned_ids + 8 * h * owned_rows   # ids, owned grad rows, fp32 dE row RMW
    f_ms, b_ms = statistics.median(fwd_ms), statistics.median(bwd_ms)
    dom = "input_forward" if f_ms >= b_ms else "input_backward"
    achieved = (fwd_bytes / (f_ms / 1e3) if dom == "input_forward" else bwd_bytes / (b_ms / 1e3)) / 1e9
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, sample, cores = cpu_input_sample(T, V, h)
        cpu = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample}
    line = {
        "metric": "input-layer fwd+bwd tokens/s at V=256k,h=4096 (BASELINE configs[3])", "value": T / (ms / 1e3),
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic ({args.ids} ids, W~N(0,0.02^2), grad~N(0,1), seed 1234)",
        "config": {"workload": "vocab-parallel input embedding: masked gather fwd (N>1: owned rows pulled from "
                               "their owners over peer memory), deterministic scatter-add bwd (accumulating)", "tokens": T, "hidden": h, "vocab": V,
                   "ids": args.ids, "owned_ids": owned_ids, "distinct_rows": owned_rows,
                   "vocab_rows_per_gpu": rows, "parallelism": f"vocab{world}"},
        "e2e": e2e, "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                     "phase_ms": {"forward(+exchange)": f_ms, "backward": b_ms},
                     "bytes_per_launch": {"input_forward": fwd_bytes, "input_backward": bwd_bytes}},
        "cpu_baseline": cpu, "clocks": clk.summary(), "comm": ctx.comm_backend,
    }
    print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "input":
        run_input(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
