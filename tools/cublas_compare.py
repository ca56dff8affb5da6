#!/usr/bin/env python3
"""cuBLAS (torch.mm, bf16 in, fp32 accumulate) on the three GEMM shapes of
the headline step, timed with CUDA events in a loop that mirrors one step
(logits -> dX -> dW, inputs larger than L2), beside our per-GEMM times from
the same box (`bench.py` roofline.gemms).  cuBLAS does only the plain GEMM:
no stats epilogue (K1), no row scale (K3), no scaled-X operand (K4), and
writes bf16 (K1) / fp32 (K3, K4) outputs like ours.

  python tools/cublas_compare.py [--steps 10]
"""
import argparse
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=256000)
    ap.add_argument("--no-ours", action="store_true", help="cuBLAS only (e.g. under ncu)")
    a = ap.parse_args()
    T, h, V = a.tokens, a.hidden, a.vocab
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, h, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    P = (torch.rand(T, V, device="cuda", generator=g) * 1e-5).to(torch.bfloat16)
    Y = torch.empty(T, V, device="cuda", dtype=torch.bfloat16)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ms = {"logits": 0.0, "dx": 0.0, "dw": 0.0}

    def step(timed):
        ev[0].record()
        torch.mm(X, W.t(), out=Y)                           # K1 shape: [T x h] . [h x V], bf16 out
        ev[1].record()
        dXo = torch.mm(P, W, out_dtype=torch.float32)       # K3 shape: [T x V] . [V x h], fp32 out
        ev[2].record()
        dWo = torch.mm(P.t(), X, out_dtype=torch.float32)   # K4 shape: [V x T] . [T x h], fp32 out
        del dXo, dWo
        ev[3].record()
        if timed:
            torch.cuda.synchronize()
            for k, (i, j) in zip(ms, ((0, 1), (1, 2), (2, 3))):
                ms[k] += ev[i].elapsed_time(ev[j])

    for _ in range(3):
        step(False)
    torch.cuda.synchronize()
    for _ in range(a.steps):
        step(True)
    flops = 2.0 * T * h * V
    res = {k: {"avg_ms": v / a.steps, "tflops": flops / (v / a.steps / 1e3) / 1e12} for k, v in ms.items()}
    res["note"] = "cuBLAS via torch.mm (bf16 inputs; K1 bf16 output, K3 / K4 fp32 output via out_dtype)"
    print(json.dumps({"cublas": res}))
    del Y, P
    torch.cuda.empty_cache()
    if a.no_ours:
        return
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", "--no-e2e",
                          "--no-graph", "--steps", str(a.steps)], capture_output=True, text=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    print(json.dumps({"ours": line["roofline"]["gemms"], "clocks": line["clocks"]}))


if __name__ == "__main__":
    main()
