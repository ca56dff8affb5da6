#!/usr/bin/env python3
"""BASELINE configs[4]: vocabulary sweep 32k-512k at h=4096, naive 3-barrier
vs reduced-barrier (alg2) output layer.  Runs on the GPUs of this process
(N=1 here: the exchange steps are device kernels; under torchrun each rank
holds V/N rows and the barriers are NCCL collectives).  Prints one JSON line
per (V, alg) and a markdown table."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_05288_b200 import vocab_math as vm  # noqa: E402


def main():
    T, h = 8192, 4096
    vocabs = [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else
                               "32000,64000,128000,128256,256000,262144,512000".split(","))]
    steps, warmup = 5, 2
    ctx = vm.Context(0)
    rows_out = []
    for V in vocabs:
        gen = torch.Generator(device="cuda").manual_seed(1234)
        X = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
        W = (torch.randn(V, h, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
        labels = torch.randint(0, V, (T,), device="cuda", generator=gen)
        batch = vm.TokenBatch(X, labels)
        shards = vm.shard_weights(W, 1)
        res = {}
        for alg in ("naive", "alg2"):
            fn = vm.run_naive if alg == "naive" else vm.run_alg2
            states = [vm.ShardState(ctx, T, h, V)]
            outs = vm._alloc_outputs(ctx, batch, shards)
            for _ in range(warmup):
                fn(ctx, batch, shards, states=states, outputs=outs)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                fn(ctx, batch, shards, states=states, outputs=outs)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            res[alg] = ms
            line = {"V": V, "alg": alg, "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3),
                    "tflops": 6.0 * T * h * V / (ms / 1e3) / 1e12}
            print(json.dumps(line), flush=True)
            for st in states:
                st.close()
            del outs
            torch.cuda.empty_cache()
        rows_out.append((V, res["naive"], res["alg2"]))
        del X, W, batch, shards
        torch.cuda.empty_cache()
    print("\n| V | naive ms | alg2 ms | alg2 speed-up | alg2 TFLOP/s |")
    print("|---|---|---|---|---|")
    for V, n, a in rows_out:
        print(f"| {V} | {n:.2f} | {a:.2f} | {n / a:.3f}x | {6.0 * T * h * V / (a / 1e3) / 1e12:.0f} |")
    ctx.close()


if __name__ == "__main__":
    main()
