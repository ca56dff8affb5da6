"""Executor overhead: a reference DeviceProgram (vocab2, p=2 devices, n=4
microbatches, built by the reference's own schedule builder) executed locally
by vp_program_run vs the same work as direct run_alg2 calls (CUDA events,
median of 5 after 2 warm-ups)."""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2411_05288_b200 import vocab_math as vm  # noqa: E402

T, h, V, p, n = 4096, 4096, 64000, 2, 4
text = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "vpipe_sched"), "build", "vocab2", str(p), str(n)],
                      capture_output=True, text=True, check=True).stdout
prog = vm.Program(text)
ctx = vm.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
W = (torch.randn(V, h, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
shards = vm.shard_weights(W, p)
batches = [vm.TokenBatch(torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16),
                         torch.randint(0, V, (T,), device="cuda", generator=g)) for _ in range(n)]
res = vm.run_program(ctx, prog, batches, shards)
states = [vm.ShardState(ctx, T, h, s.rows()) for s in shards]
outs = [vm._alloc_outputs(ctx, b, shards) for b in batches]


def timed(fn):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


t_prog = timed(lambda: vm.run_program(ctx, prog, batches, shards, outputs=res))
t_direct = timed(lambda: [vm.run_alg2(ctx, b, shards, states=states, outputs=o) for b, o in zip(batches, outs)])
ctx.set_option("accumulate_grad_w", 1)  # the program accumulates dW over its microbatches
t_acc = timed(lambda: [vm.run_alg2(ctx, b, shards, states=states, outputs=outs[0]) for b in batches])
ctx.set_option("accumulate_grad_w", 0)
print(f"program vocab2 p={p} n={n} (local): {t_prog:.2f} ms; direct run_alg2 x {n}: {t_direct:.2f} ms "
      f"(overhead {100 * (t_prog / t_direct - 1):+.2f}%); direct with dW accumulated like the program: "
      f"{t_acc:.2f} ms (overhead {100 * (t_prog / t_acc - 1):+.2f}%)")
