"""GPU: the vocabulary-pass executor (vp_program_run) running reference
DevicePrograms, and CUDA-graph capture of the output layer.

A program's vocabulary passes (S, C0, C1, T, C2 of every microbatch, in the
reference schedule's order) must give exactly what the per-microbatch drivers
give (run_alg2 for vocab2, run_alg1 for vocab1 / interlaced), with dW
accumulated over the microbatches, and must match the CPU oracle."""
import json
import os

import numpy as np
import pytest
import torch

from gpu_helpers import GRAD_REL_L2, LOSS_ABS, device_case, oracle, rel_l2
from paper_2411_05288_b200 import vocab_math as vm

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "programs.json")))


def _microbatches(n, T, h, V, seed):
    out = []
    W = None
    for i in range(n):
        X, W_i, g = oracle.random_instance(T, h, V, seed + i)
        if W is None:
            W = W_i  # one weight matrix shared by all microbatches
        Xb, Wb, batch, Wd = device_case(X, W, g)
        out.append((Xb, Wb, g, batch, Wd))
    return out


@pytest.mark.parametrize("name,driver", [("vocab2_p2_n4", "alg2"), ("vocab2_p4_n8", "alg2"),
                                         ("vocab1_p2_n4", "alg1"), ("interlaced_p4_n8", "alg1"),
                                         ("vhalf-vocab1_p2_n4", "alg1"), ("vocab2_p1_n3", "alg2")])
def test_program_equals_per_microbatch_drivers(ctx, name, driver):
    prog = vm.Program(GOLDEN[name]["text"])
    T, h, V = 48, 64, 96 * prog.p
    mbs = _microbatches(prog.n, T, h, V, 100)
    Wd = mbs[0][4]
    shards = vm.shard_weights(Wd, prog.p)
    res = vm.run_program(ctx, prog, [m[3] for m in mbs], shards)
    ctx.sync()
    fn = vm.run_alg2 if driver == "alg2" else vm.run_alg1
    gw_sum = None
    for i, m in enumerate(mbs):
        ref = fn(ctx, m[3], shards)
        ctx.sync()
        assert torch.equal(res.loss[i], ref.loss), i
        assert torch.equal(res.grad_x[i], ref.grad_x), i
        assert torch.equal(res.stats[i].m, ref.stats.m) and torch.equal(res.stats[i].sum, ref.stats.sum)
        g = ref.grad_w_full().double()
        gw_sum = g if gw_sum is None else gw_sum + g
    got = torch.cat(res.grad_w).double()
    assert torch.allclose(got, gw_sum, rtol=1e-5, atol=1e-6)


def test_program_matches_the_oracle(ctx):
    prog = vm.Program(GOLDEN["vocab2_p4_n8"]["text"])
    T, h, V = 32, 64, 512
    mbs = _microbatches(prog.n, T, h, V, 7)
    res = vm.run_program(ctx, prog, [m[3] for m in mbs], vm.shard_weights(mbs[0][4], prog.p))
    ctx.sync()
    gw_ref = 0
    for i, (Xb, Wb, g, _, _) in enumerate(mbs):
        ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
        assert np.abs(res.loss[i].double().cpu().numpy() - ref.loss).max() <= LOSS_ABS
        assert rel_l2(res.grad_x[i][:, :h].cpu().numpy(), ref.grad_x) <= GRAD_REL_L2
        gw_ref = gw_ref + ref.grad_w
    assert rel_l2(torch.cat(res.grad_w)[:, :h].cpu().numpy(), gw_ref) <= GRAD_REL_L2


def test_program_violating_its_dependencies_is_rejected(ctx):
    prog = vm.Program(GOLDEN["vocab1_p4_n8_T3_before_C1"]["text"])
    mbs = _microbatches(prog.n, 16, 32, 128, 3)
    with pytest.raises(ValueError, match="T microbatch 3 device 2 scheduled before its dependency C1"):
        vm.run_program(ctx, prog, [m[3] for m in mbs], vm.shard_weights(mbs[0][4], prog.p))


def test_program_through_a_one_rank_nccl_group(ctx):
    # the NCCL path of the executor (C0 broadcast, C1 stats all-gather and the
    # dX / loss all-reduce forked onto the comm stream) on a 1-device program
    prog = vm.Program(GOLDEN["vocab2_p1_n3"]["text"])
    mbs = _microbatches(prog.n, 40, 64, 256, 21)
    shards = vm.shard_weights(mbs[0][4], 1)
    local = vm.run_program(ctx, prog, [m[3] for m in mbs], shards)
    nctx = vm.Context(0)
    nctx.comm_init(1, 0, vm.Context.unique_id())
    nctx.set_option("force_collectives", 1)
    dist = vm.run_program(nctx, prog, [m[3] for m in mbs], shards)
    nctx.sync()
    ctx.sync()
    for i in range(prog.n):
        assert torch.allclose(local.loss[i], dist.loss[i], rtol=1e-6, atol=1e-7)
        assert torch.allclose(local.grad_x[i], dist.grad_x[i], rtol=1e-6, atol=1e-7)
    assert torch.allclose(local.grad_w[0], dist.grad_w[0], rtol=1e-6, atol=1e-7)
    nctx.close()


def test_cuda_graph_replay_equals_eager(ctx):
    # capture run_alg2 and a whole program; replays on fresh inputs (copied
    # into the captured buffers) reproduce eager results bit for bit
    stream = torch.cuda.Stream()  # the legacy default stream cannot be captured
    with torch.cuda.stream(stream):
        _graph_replays(ctx)


def _graph_replays(ctx):
    gctx = vm.Context(0)  # runs on the current (side) stream
    X, W, g = oracle.random_instance(300, 128, 1500, 4)
    _, _, batch, Wd = device_case(X, W, g)
    shards = vm.shard_weights(Wd, 2)
    states = [vm.ShardState(gctx, 300, 128, s.rows()) for s in shards]
    outs = vm._alloc_outputs(gctx, batch, shards)
    vm.run_alg2(gctx, batch, shards, states=states, outputs=outs)  # sizes the workspace
    gctx.sync()
    graph = vm.capture(gctx, lambda: vm.run_alg2(gctx, batch, shards, states=states, outputs=outs))
    for seed in (5, 6):
        X2, _, g2 = oracle.random_instance(300, 128, 1500, seed)
        _, _, b2, _ = device_case(X2, W, g2)
        batch.X.copy_(b2.X)
        batch.labels.copy_(b2.labels)
        graph.launch()
        gctx.sync()
        eager = vm.run_alg2(ctx, b2, shards)
        ctx.sync()
        assert torch.equal(outs[0], eager.loss)
        assert torch.equal(outs[1], eager.grad_x)
        assert torch.equal(torch.cat(outs[2]), eager.grad_w_full())
    graph.close()
    # a whole program
    prog = vm.Program(GOLDEN["vocab2_p2_n4"]["text"])
    mbs = _microbatches(prog.n, 64, 64, 384, 40)
    sh = vm.shard_weights(mbs[0][4], prog.p)
    res = vm.run_program(gctx, prog, [m[3] for m in mbs], sh)
    gctx.sync()
    ref = [t.clone() for t in res.grad_x] + [t.clone() for t in res.grad_w]
    for t in res.grad_x + res.grad_w:
        t.zero_()
    graph = vm.capture(gctx, lambda: vm.run_program(gctx, prog, [m[3] for m in mbs], sh, outputs=res))
    graph.launch()
    gctx.sync()
    for a, b in zip(res.grad_x + res.grad_w, ref):
        assert torch.equal(a, b)
    graph.close()
    gctx.close()
