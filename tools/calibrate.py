#!/usr/bin/env python3
"""Cost-model calibration: measure the vocabulary passes on
one B200 and feed them into the REFERENCE's cost model / pipeline simulator.

The reference models a shard's output-layer work as S + T = 3 x 6bshV/p table
units split 1/3 : 2/3 (Algorithm 1, two barriers) or 3/5 : 2/5 (Algorithm 2,
one barrier) (P/src/cost_model.cpp:79-89, P/src/simulator.cpp:66-84), and every
collective as 10% of a stage forward.  This tool times alg{1,2}_pass_S, the
barrier work and alg{1,2}_pass_T for one shard of V/p vocabulary rows with CUDA
events, converts the reference's units to milliseconds at the measured GEMM
rate R (unit_rate = 3R: the simulator's F then equals the stage's forward flops
at rate R), estimates the NVLink part of each barrier (ring all-reduce /
all-gather at --busbw GB/s; this box has one GPU), and runs the reference
simulator (oracle/_ref/vpipe_sched, built from /root/reference) with the model's
and with the measured S / T / collective durations.

    python tools/calibrate.py [--p 8] [--seq 4096] [--hidden 4096] [--vocab 256000]
                              [--layers 32] [--microbatches 32] [--busbw 700]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=7, warm=2):
    import torch
    for _ in range(warm):
        fn()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=256000)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--microbatches", type=int, default=32)
    ap.add_argument("--busbw", type=float, default=700.0, help="NCCL bus bandwidth over NVLink, GB/s (assumed)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    from paper_2411_05288_b200 import vocab_math as vm
    T, h, p = a.seq, a.hidden, a.p
    V = vm.pad_vocab_size(a.vocab, p)
    rows = V // p
    ctx = vm.Context(0)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    X = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    lab = torch.randint(0, V, (T,), device="cuda", generator=gen)
    W = (torch.randn(rows, h, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    batch = vm.TokenBatch(X, lab)
    shard = vm.EmbeddingShard(W, 0, 0, rows)
    st = vm.ShardState(ctx, T, h, rows)
    gw = torch.empty(rows, h, dtype=torch.float32, device="cuda")
    meas = {}
    # Algorithm 2: S (logits + stats + A), C1 (merge + combine + loss), T (dW)
    meas["alg2_S"] = timed(lambda: vm.alg2_pass_S(ctx, batch, shard, state=st))
    c1 = vm.alg2_barrier_C1(ctx, [st], [shard], batch)
    meas["alg2_C1_local"] = timed(lambda: vm.alg2_barrier_C1(ctx, [st], [shard], batch))
    meas["alg2_T"] = timed(lambda: vm.alg2_pass_T(ctx, st, c1.stats, batch, shard, grad_w=gw))
    # Algorithm 1: S (logits + stats), C1 (merge), T (dX partial + dW)
    meas["alg1_S"] = timed(lambda: vm.alg1_pass_S(ctx, batch, shard, state=st))
    stats = vm.merge_max_sum(ctx, [st])
    meas["alg1_C1_local"] = timed(lambda: vm.merge_max_sum(ctx, [st]))
    gx1 = torch.empty(T, h, dtype=torch.float32, device="cuda")
    meas["alg1_T"] = timed(lambda: vm.alg1_pass_T(ctx, st, stats, batch, shard, grad_x_partial=gx1, grad_w=gw))
    flops_shard = 6.0 * T * h * rows
    R = flops_shard / ((meas["alg2_S"] + meas["alg2_T"]) * 1e-3)  # flops/s achieved by the output layer
    # NVLink parts of the barriers (estimates, one GPU here)
    bw = a.busbw * 1e9
    ar = lambda nbytes: 2.0 * (p - 1) / p * nbytes / bw * 1e3  # noqa: E731  ring all-reduce, ms
    ag = lambda nbytes: (p - 1) / p * nbytes * p / bw * 1e3  # noqa: E731   all-gather of nbytes per rank
    # fused exchange (default): the dX partials reach their owners inside the dX
    # GEMM's epilogue (pass S, NVLink traffic overlapped with the MMAs); the
    # barrier's critical path is the stats all-gather, the owner combine and the
    # loss all-reduce; the grad_x pull by the copy engines ((p-1)/p of T x h fp32
    # per rank) runs beside pass T and only shows if it outlasts it
    nvl = a.busbw * 1e9 * 1.2  # point-to-point copy-engine pulls: no ring overhead (assumed)
    pull = (p - 1) / p * 4 * T * h / nvl * 1e3
    coll = {
        "C0_broadcast_X_ms": T * h * 2 / bw * 1e3,
        "alg2_C1_ms_allreduce": meas["alg2_C1_local"] + ag(8 * T) + ar(4 * T * h) + ar(4 * T),
        "alg2_C1_ms": meas["alg2_C1_local"] + ag(8 * T) + ar(4 * T) + max(0.0, pull - meas["alg2_T"]),
        "alg2_gather_pull_ms_beside_T": pull,
        "alg1_C1_ms": meas["alg1_C1_local"] + ag(8 * T),
        "alg1_C2_ms": ar(4 * T * h),
        "alg1_C2_ms_fused": meas["alg2_C1_local"] + pull,
    }
    unit_rate = 3.0 * R * 1e-3  # flops per ms, x3: the simulator's table-unit convention
    sched = os.path.join(ROOT, "oracle", "_ref", "vpipe_sched")
    sims = {}
    for method, S, Tt, C in (("vocab2", meas["alg2_S"], meas["alg2_T"], coll["alg2_C1_ms"]),
                             ("vocab1", meas["alg1_S"], meas["alg1_T"],
                              max(coll["alg1_C1_ms"], coll["alg1_C2_ms_fused"]))):
        if os.path.exists(sched):
            r = subprocess.run([sched, "simulate", method, "1", str(T), str(h), str(V), str(a.layers), str(p),
                                str(a.microbatches), repr(unit_rate), repr(S), repr(Tt), repr(C)],
                               capture_output=True, text=True)
            sims[method] = json.loads(r.stdout) if r.returncode == 0 else {"error": r.stdout + r.stderr}
        else:
            sims[method] = {"error": "oracle/_ref/vpipe_sched not built (needs /root/reference at build time)"}
    res = {"config": {"b": 1, "s": T, "h": h, "V": V, "L": a.layers, "p": p, "n": a.microbatches,
                      "shard_rows": rows, "busbw_GBps_assumed": a.busbw},
           "measured_ms": meas, "collectives_ms": coll, "output_layer_rate_TFLOPs": R / 1e12,
           "split": {"alg2_S_frac": meas["alg2_S"] / (meas["alg2_S"] + meas["alg2_T"]), "alg2_S_frac_model": 0.6,
                     "alg1_S_frac": meas["alg1_S"] / (meas["alg1_S"] + meas["alg1_T"]), "alg1_S_frac_model": 1 / 3},
           "simulation": sims}
    js = json.dumps(res, indent=1)
    print(js)
    if a.out:
        open(a.out, "w").write(js)


if __name__ == "__main__":
    main()
