"""One plain and one routed dX GEMM (headline shape) for ncu: alg2 on a plain
context, then on a forced 1-rank NCCL group (fused exchange: the dX epilogue
stores into the owner's slots)."""
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
batch = vm.TokenBatch(X, torch.randint(0, V, (T,), device="cuda", generator=g))
shards = vm.shard_weights(W, 1)
plain = vm.Context(0)
vm.run_alg2(plain, batch, shards)
plain.sync()
fused = vm.Context(0)
fused.comm_init(1, 0, vm.Context.unique_id())
fused.set_option("force_collectives", 1)
vm.run_alg2(fused, batch, shards)
fused.sync()
print("fused exchanges:", fused.fused_c1_count)
