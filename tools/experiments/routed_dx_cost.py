"""Cost of the routed dX epilogue (per-thread stores into the owners' slots) at
the headline shape: alg2 on a forced 1-rank NCCL group (fused exchange, the
dX GEMM routed to this rank's own slots) vs the plain one-GPU run; per-GEMM
CUDA-event times, interleaved, 3 rounds x 10 steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2411_05288_b200 import vocab_math as vm  # noqa: E402

T, h, V = 8192, 4096, 256000
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16)
W = (torch.randn(V, h, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
lab = torch.randint(0, V, (T,), device="cuda", generator=g)
batch = vm.TokenBatch(X, lab)
shards = vm.shard_weights(W, 1)
plain = vm.Context(0)
fused = vm.Context(0)
fused.comm_init(1, 0, vm.Context.unique_id())
fused.set_option("force_collectives", 1)
for ctx in (plain, fused):
    st = [vm.ShardState(ctx, T, h, V)]
    ctx._st, ctx._o = st, vm._alloc_outputs(ctx, batch, shards)
    vm.run_alg2(ctx, batch, shards, states=st, outputs=ctx._o)
    ctx.sync()
for rnd in range(3):
    for name, ctx in (("plain", plain), ("fused", fused)):
        ctx.gemm_timing(True)
        for _ in range(10):
            vm.run_alg2(ctx, batch, shards, states=ctx._st, outputs=ctx._o)
        ctx.sync()
        t = ctx.gemm_timing(False)
        print(name, {k: round(ms / n, 3) for k, (ms, n) in t.items() if n}, "fused exchanges:", ctx.fused_c1_count)
