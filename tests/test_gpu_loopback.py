"""GPU: the library's nranks > 1 code paths, run for real on one B200.

p contexts on cuda:0 form one group through the loopback collective backend
(vp_comm_init_all -> device mailboxes + host rendezvous), each rank driven from
its own host thread and stream with ONE vocabulary shard — exactly what a
torchrun rank does with NCCL: rank-offset shards, the [N x 2T] stats
all-gather and fixed-order merge, owner-only loss + sum all-reduce, the dX
all-reduce (forked onto the comm stream in alg2), alg1's C2, naive's max / sum
all-reduces, the input layer's forward all-reduce, and the executor's C0
broadcast / C1 / C2 with one program device per rank.  Results are checked
against the CPU oracle at the north_star tolerances (input layer bit-exact),
and every rank must hold bitwise the same loss / grad_x / stats.
"""
import os

import numpy as np
import pytest
import torch

from gpu_helpers import GRAD_REL_L2, LOSS_ABS, assert_parity, device_case, oracle, rel_l2
from paper_2411_05288_b200 import dist as vpd
from paper_2411_05288_b200 import vocab_math as vm

pytestmark = pytest.mark.gpu

os.environ.setdefault("VPIPE_LOOPBACK_TIMEOUT", "120")  # a failing rank must not hang the others forever


def _shard(Wd, p, r):
    rb, re = vpd.shard_rows(Wd.shape[0], p, r)
    return vm.EmbeddingShard(Wd[rb:re], r, rb, re)


def _close(ctxs):
    for c in ctxs:
        c.sync()
    for c in ctxs:
        c.close()


def _same_on_every_rank(outs, key):
    for o in outs[1:]:
        assert torch.equal(getattr(o, key), getattr(outs[0], key)), key


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("alg", ["naive", "alg1", "alg2"])
def test_drivers_with_p_ranks_match_the_oracle(alg, p):
    T, h, V = 96, 64, 512 * p
    X, W, g = oracle.random_instance(T, h, V, 10 + p)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    assert all(c.comm_backend == "loopback" for c in ctxs)
    assert [c.comm_info() for c in ctxs] == [(p, r) for r in range(p)]
    fn = {"naive": vm.run_naive, "alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg]

    def rank(r, ctx):
        out = fn(ctx, batch, [_shard(Wd, p, r)])
        ctx.sync()
        return out

    outs = vpd.run_ranks(ctxs, rank)
    for key in ("loss", "grad_x"):
        _same_on_every_rank(outs, key)
    for o in outs[1:]:
        assert torch.equal(o.stats.m, outs[0].stats.m) and torch.equal(o.stats.sum, outs[0].stats.sum)
    res = {"loss": outs[0].loss.double().cpu().numpy(), "grad_x": outs[0].grad_x[:, :h].double().cpu().numpy(),
           "grad_w": torch.cat([o.grad_w[0] for o in outs])[:, :h].double().cpu().numpy()}
    assert_parity(res, ref, f"loopback p={p} {alg}")
    _close(ctxs)


@pytest.mark.parametrize("p", [2, 4])
def test_chunked_alg2_across_ranks(p):
    # the memory-bounded driver with a group: every chunk's stats all-gather,
    # combine and dX / loss all-reduce (overlapped with the chunk's pass T)
    T, h, V = 300, 64, 400 * p
    X, W, g = oracle.random_instance(T, h, V, 30 + p)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)

    def rank(r, ctx):
        out = vm.run_alg2_chunked(ctx, batch, [_shard(Wd, p, r)], 128)
        ctx.sync()
        return out

    outs = vpd.run_ranks(ctxs, rank)
    for key in ("loss", "grad_x"):
        _same_on_every_rank(outs, key)
    res = {"loss": outs[0].loss.double().cpu().numpy(), "grad_x": outs[0].grad_x[:, :h].double().cpu().numpy(),
           "grad_w": torch.cat([o.grad_w[0] for o in outs])[:, :h].double().cpu().numpy()}
    assert_parity(res, ref, f"loopback chunked p={p}")
    _close(ctxs)


def test_loopback_equals_local_shards():
    # the same 4 shards run as 4 ranks and as 4 local shards of one context
    p, T, h, V = 4, 64, 128, 2048
    X, W, g = oracle.random_instance(T, h, V, 3)
    _, _, batch, Wd = device_case(X, W, g)
    local_ctx = vm.Context(0)
    local = vm.run_alg2(local_ctx, batch, vm.shard_weights(Wd, p))
    local_ctx.sync()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    outs = vpd.run_ranks(ctxs, lambda r, c: vm.run_alg2(c, batch, [_shard(Wd, p, r)]))
    for c in ctxs:
        c.sync()
    assert torch.equal(outs[0].loss, local.loss)
    assert torch.equal(outs[0].stats.m, local.stats.m) and torch.equal(outs[0].stats.sum, local.stats.sum)
    assert torch.allclose(outs[0].grad_x, local.grad_x, rtol=1e-5, atol=1e-6)
    assert torch.allclose(torch.cat([o.grad_w[0] for o in outs]), local.grad_w_full(), rtol=1e-5, atol=1e-6)
    _close(ctxs)
    local_ctx.close()


@pytest.mark.parametrize("p", [2, 8])
def test_pass_functions_across_ranks(p):
    # alg2: S -> C1 (all-gather merge + combine + dX all-reduce) -> T;
    # alg1: S -> merge_max_sum (all-gather) -> T -> reduce_grad_x (C2 all-reduce)
    T, h, V = 40, 32, 64 * p
    X, W, g = oracle.random_instance(T, h, V, 5)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)

    def rank(r, ctx):
        sh = _shard(Wd, p, r)
        st = vm.alg2_pass_S(ctx, batch, sh)
        c1 = vm.alg2_barrier_C1(ctx, [st], [sh], batch)
        gw2 = vm.alg2_pass_T(ctx, st, c1.stats, batch, sh)
        loss = vm.output_loss(ctx, [st], [sh], c1.stats, batch)  # owner-only + sum all-reduce
        st1 = vm.alg1_pass_S(ctx, batch, sh)
        stats1 = vm.merge_max_sum(ctx, [st1])
        gr = vm.alg1_pass_T(ctx, st1, stats1, batch, sh)
        gx1 = vm.reduce_grad_x(ctx, [gr.grad_x_partial])
        ctx.sync()
        return c1, gw2, loss, stats1, gr, gx1

    outs = vpd.run_ranks(ctxs, rank)
    for o in outs[1:]:
        assert torch.equal(o[0].grad_x, outs[0][0].grad_x)
        assert torch.equal(o[2], outs[0][2])
        assert torch.equal(o[3].m, outs[0][3].m) and torch.equal(o[3].sum, outs[0][3].sum)
        assert torch.equal(o[5], outs[0][5])
    assert np.abs(outs[0][2].double().cpu().numpy() - ref.loss).max() <= LOSS_ABS
    assert rel_l2(outs[0][0].grad_x[:, :h].cpu().numpy(), ref.grad_x) <= GRAD_REL_L2
    assert rel_l2(outs[0][5][:, :h].cpu().numpy(), ref.grad_x) <= GRAD_REL_L2
    gw = lambda i: torch.cat([o[i] if i == 1 else o[i].grad_w for o in outs])[:, :h].cpu().numpy()  # noqa: E731
    assert rel_l2(gw(1), ref.grad_w) <= GRAD_REL_L2
    assert rel_l2(gw(4), ref.grad_w) <= GRAD_REL_L2
    # the stats all-gather + merge equals the oracle's merge of the local stats
    m_ref, s_ref = oracle.merge_max_sum(*zip(*[oracle.local_stats(Xb, Wb, p, k) for k in range(p)]))
    assert np.abs(outs[0][3].m.cpu().numpy() - m_ref).max() < 1e-4
    assert rel_l2(outs[0][3].sum.cpu().numpy(), s_ref) < 1e-3
    _close(ctxs)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_input_layer_across_ranks_is_bit_exact(p):
    # forward: masked gather of each rank's shard + bf16 sum all-reduce
    # (x + 0 = x: bit-exact); backward: each rank's shard gradient
    V, h, T = 1024 * p, 256, 2000
    rng = np.random.default_rng(p)
    W = torch.from_numpy(rng.standard_normal((V, h)).astype(np.float32)).to(torch.bfloat16).cuda()
    tok = torch.from_numpy(rng.integers(0, V, T)).cuda()
    tok[:50] = 7  # a repeated row
    grad = torch.from_numpy(rng.standard_normal((T, h)).astype(np.float32)).to(torch.bfloat16).cuda()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)

    def rank(r, ctx):
        sh = _shard(W, p, r)
        out = vm.input_forward(ctx, tok, sh)
        vm.allreduce_sum(ctx, out)
        dE = vm.input_backward(ctx, grad, tok, sh)
        ctx.sync()
        return out, dE

    outs = vpd.run_ranks(ctxs, rank)
    want = W[tok]
    for out, _ in outs:
        assert torch.equal(out, want)
    g_np = grad.float().cpu().numpy()
    t_np = tok.cpu().numpy()
    for r, (_, dE) in enumerate(outs):
        rb, re = vpd.shard_rows(V, p, r)
        assert np.array_equal(dE.cpu().numpy(), oracle.input_backward_f32(g_np, t_np, re - rb, rb))
    _close(ctxs)


@pytest.mark.parametrize("peer", [1, 0])
@pytest.mark.parametrize("p,ids", [(2, "uniform"), (4, "zipf"), (8, "uniform"), (8, "hot")])
def test_input_layer_owner_gather_and_grad_broadcast(p, ids, peer):
    # forward without the zero-padded all-reduce -> W[tok] bit-exact on every
    # rank (tokens past V: zero rows, as the reference's unowned rows):
    # peer=1 (default) every rank writes its owned rows at their token index
    # into its peer-mapped buffer and pulls each row from its owner's buffer;
    # peer=0 each rank packs its rows, one grouped broadcast per rank, unpack.
    # backward: grad_out lives on one rank (root p-1, the last pipeline stage)
    # and is broadcast before every shard's scatter (R/PAPER.md:582).
    V, h, T = 1000 * p, 136, 3001
    rng = np.random.default_rng(10 + p)
    W = torch.from_numpy(rng.standard_normal((V, h)).astype(np.float32)).to(torch.bfloat16).cuda()
    if ids == "zipf":
        t = np.minimum(rng.zipf(1.1, T) - 1, V - 1)
    elif ids == "hot":
        t = np.full(T, 3)  # every token owned by rank 0: the other blocks are empty
    else:
        t = rng.integers(0, V, T)
    t[-5:] = V + np.arange(5)  # owned by no shard
    tok = torch.from_numpy(t.astype(np.int64)).cuda()
    grad = torch.from_numpy(rng.standard_normal((T, h)).astype(np.float32)).cuda()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    for c in ctxs:
        c.set_option("peer_input", peer)

    def rank(r, ctx):
        sh = _shard(W, p, r)
        out = vm.input_forward_gathered(ctx, tok, sh)
        g = grad.clone() if r == p - 1 else torch.zeros_like(grad)
        vm.input_grad_broadcast(ctx, g, root=p - 1)
        dE = vm.input_backward(ctx, g[:-5], tok[:-5], sh)
        # broadcast + backward in one call: grad_out on the root only
        dE2 = vm.input_backward_gathered(ctx, grad[:-5] if r == p - 1 else None, tok[:-5], sh, root=p - 1, h=h,
                                         grad_is_f32=True)
        ctx.sync()
        assert torch.equal(dE2, dE), r
        return out, g, dE

    outs = vpd.run_ranks(ctxs, rank)
    want = torch.zeros(T, h, dtype=torch.bfloat16, device="cuda")
    want[:-5] = W[tok[:-5]]
    g_np = grad[:-5].cpu().numpy()
    for r, (out, g, dE) in enumerate(outs):
        assert torch.equal(out, want), r
        assert torch.equal(g, grad), r
        rb, re = vpd.shard_rows(V, p, r)
        assert np.array_equal(dE.cpu().numpy(), oracle.input_backward_f32(g_np, t[:-5], re - rb, rb)), r
    assert [c.peer_input_count for c in ctxs] == [2 * peer] * p  # the forward and the gathered backward
    _close(ctxs)


def test_input_peer_pull_repeated_calls():
    # back-to-back forwards alternate the two halves of the peer buffers (a
    # rank's next write never races a peer's pull of the previous call); a
    # larger batch grows the buffers
    p, V, h = 4, 4000, 256
    rng = np.random.default_rng(3)
    W = torch.from_numpy(rng.standard_normal((V, h)).astype(np.float32)).to(torch.bfloat16).cuda()
    ctxs = vpd.local_group(p)
    calls = [(700, 1), (700, 2), (2100, 3), (64, 4), (700, 5)]
    toks = [torch.from_numpy(np.random.default_rng(sd).integers(0, V, T).astype(np.int64)).cuda() for T, sd in calls]
    torch.cuda.synchronize()

    def rank(r, ctx):
        sh = _shard(W, p, r)
        outs = [vm.input_forward_gathered(ctx, t, sh) for t in toks]
        ctx.sync()
        return outs

    res = vpd.run_ranks(ctxs, rank)
    for r in range(p):
        for t, out in zip(toks, res[r]):
            assert torch.equal(out, W[t]), r
    assert [c.peer_input_count for c in ctxs] == [len(calls)] * p
    _close(ctxs)


def test_label_out_of_range_raises_on_every_rank():
    # VM.cpp:18: labels must lie in [0, V); V is the group's largest row_end
    p, T, h, V = 2, 16, 32, 256
    X, W, g = oracle.random_instance(T, h, V, 2)
    g = g.copy()
    g[3] = V  # owned by no shard
    _, _, batch, Wd = device_case(X, W, g)
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)

    def rank(r, ctx):
        vm.run_alg2(ctx, batch, [_shard(Wd, p, r)])
        with pytest.raises(ValueError, match="label out of range"):
            ctx.sync()
        return True

    assert all(vpd.run_ranks(ctxs, rank))
    _close(ctxs)


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("name", ["vocab2_p2_n4", "vocab2_p4_n8", "vocab1_p2_n4", "interlaced_p4_n8"])
def test_executor_one_program_device_per_rank(name, fused):
    # vp_program_run in a group: rank k executes device k's pass list (C0
    # broadcast of X_i from device p-1, C1 / C2 exchanges on the comm stream;
    # fused=1: the peer-memory exchange with one buffer region per microbatch,
    # so several microbatches' S (alg2) / T (alg1) precede their barriers)
    import json
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "programs.json")))
    prog = vm.Program(golden[name]["text"])
    p, n = prog.p, prog.n
    T, h, V = 48, 64, 96 * p
    W = None
    mbs = []
    for i in range(n):
        X, W_i, g = oracle.random_instance(T, h, V, 200 + i)
        W = W_i if W is None else W
        mbs.append(device_case(X, W, g))
    Wd = mbs[0][3]
    # local reference: every program device on one context
    lctx = vm.Context(0)
    local = vm.run_program(lctx, prog, [m[2] for m in mbs], vm.shard_weights(Wd, p))
    lctx.sync()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    for c in ctxs:
        c.set_option("fused_c1", fused)

    def rank(r, ctx):
        # C0 broadcasts X_i from device p-1: the other ranks start from garbage
        batches = [vm.TokenBatch(m[2].X.clone() if r == p - 1 else torch.zeros_like(m[2].X), m[2].labels)
                   for m in mbs]
        res = vm.run_program(ctx, prog, batches, [_shard(Wd, p, r)])
        ctx.sync()
        return res, batches

    outs = vpd.run_ranks(ctxs, rank)
    for r, (res, batches) in enumerate(outs):
        for i in range(n):
            assert torch.equal(batches[i].X, mbs[i][2].X)  # C0 delivered X_i
            assert torch.equal(res.loss[i], outs[0][0].loss[i])
            assert torch.equal(res.grad_x[i], outs[0][0].grad_x[i])
            assert torch.allclose(res.loss[i], local.loss[i], rtol=1e-5, atol=1e-6)
            assert torch.allclose(res.grad_x[i], local.grad_x[i], rtol=1e-4, atol=1e-6)
        assert torch.allclose(res.grad_w[0], local.grad_w[r], rtol=1e-4, atol=1e-6)
    gw_ref = 0
    for i, (Xb, Wb, _, _) in enumerate(mbs):
        ref = oracle.oracle_output_layer(Xb, mbs[i][2].labels.cpu().numpy(), Wb, want_softmax=False)
        assert np.abs(outs[0][0].loss[i].double().cpu().numpy() - ref.loss).max() <= LOSS_ABS
        gw_ref = gw_ref + ref.grad_w
    got = torch.cat([o[0].grad_w[0] for o in outs])[:, :h].cpu().numpy()
    assert rel_l2(got, gw_ref) <= GRAD_REL_L2
    assert [c.fused_c1_count for c in ctxs] == [n * fused] * p
    _close(ctxs)
    lctx.close()


def test_loopback_group_cannot_be_captured():
    ctxs = vpd.local_group(2)

    def rank(r, ctx):
        with pytest.raises(ValueError, match="cannot be captured"):
            vm.capture(ctx, lambda: None)
        return True

    assert all(vpd.run_ranks(ctxs, rank))
    _close(ctxs)


# ---------------------------------------------------------------------------
# Fused C1 (option "fused_c1", the default in a group): pass S's dX GEMM
# stores every A_k tile straight into the buffer of the rank owning those
# token rows (peer memory; on one GPU the peers' buffers are plain device
# pointers, across processes CUDA IPC mappings), the label rows follow, the
# owner combines its rows in rank order and the group all-gathers grad_x.
# The combine's expression and order are those of the one-GPU p-shard
# combine, so the group's loss / grad_x / grad_w carry the one-GPU bits.
# ---------------------------------------------------------------------------
def _local_and_group(p, T, h, V, seed, opts=(), alg="alg2"):
    fn = {"alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg]
    X, W, g = oracle.random_instance(T, h, V, seed)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    local_ctx = vm.Context(0)
    for k, v in opts:
        local_ctx.set_option(k, v)
    local = fn(local_ctx, batch, vm.shard_weights(Wd, p))
    local_ctx.sync()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    for c in ctxs:
        for k, v in opts:
            c.set_option(k, v)
    outs = vpd.run_ranks(ctxs, lambda r, c: fn(c, batch, [_shard(Wd, p, r)]))
    for c in ctxs:
        c.sync()
    return Xb, Wb, g, local, local_ctx, ctxs, outs


@pytest.mark.parametrize("alg", ["alg2", "alg1"])
@pytest.mark.parametrize("p,T", [(2, 256), (4, 256), (8, 512), (2, 96), (8, 96), (4, 1000), (4, 1), (8, 33)])
def test_fused_c1_has_the_one_gpu_bits(p, T, alg):
    # T = p * R exactly (grad_x gathered in place) and ragged T (owners of
    # 32-row multiples, some ranks owning nothing at T=96, p=8)
    # (split-K pinned: ranks sharing one GPU get a share of its SMs, so the
    # automatic split choice could differ from the one-context run's)
    h, V = 128, 1024 * p
    opts = (("splits_dx", 1), ("splits_dw", 1))
    Xb, Wb, g, local, local_ctx, ctxs, outs = _local_and_group(p, T, h, V, 40 + p, opts, alg)
    assert [c.fused_c1_count for c in ctxs] == [1] * p
    for o in outs:
        assert torch.equal(o.loss, local.loss)
        assert torch.equal(o.grad_x, local.grad_x)
        assert torch.equal(o.stats.m, local.stats.m) and torch.equal(o.stats.sum, local.stats.sum)
    assert torch.equal(torch.cat([o.grad_w[0] for o in outs]), local.grad_w_full())
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    res = {"loss": outs[-1].loss.double().cpu().numpy(), "grad_x": outs[-1].grad_x[:, :h].double().cpu().numpy(),
           "grad_w": torch.cat([o.grad_w[0] for o in outs])[:, :h].double().cpu().numpy()}
    assert_parity(res, ref, f"fused C1 p={p} T={T} {alg}")
    _close(ctxs)
    local_ctx.close()


def test_fused_c1_routed_ordered_split_k():
    # the routed epilogue with ordered split-K units (split 1 reduce-adds into
    # the owner's slot after split 0's stores landed, system-scope hand-off)
    p, T, h, V = 4, 512, 256, 4 * 8192
    opts = (("splits_dx", 3), ("split_workspace", 0), ("splits_dw", 1))
    Xb, Wb, g, local, local_ctx, ctxs, outs = _local_and_group(p, T, h, V, 7, opts)
    assert [c.fused_c1_count for c in ctxs] == [1] * p
    for o in outs:
        assert torch.equal(o.grad_x, local.grad_x) and torch.equal(o.loss, local.loss)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    res = {"loss": outs[0].loss.double().cpu().numpy(), "grad_x": outs[0].grad_x[:, :h].double().cpu().numpy(),
           "grad_w": torch.cat([o.grad_w[0] for o in outs])[:, :h].double().cpu().numpy()}
    assert_parity(res, ref, "fused C1 split-K 3")
    _close(ctxs)
    local_ctx.close()


def test_fused_c1_off_keeps_the_all_reduce():
    p, T, h, V = 4, 256, 128, 4096
    X, W, g = oracle.random_instance(T, h, V, 5)
    _, _, batch, Wd = device_case(X, W, g)
    res = {}
    for fused in (0, 1):
        ctxs = vpd.local_group(p)
        for c in ctxs:
            c.set_option("fused_c1", fused)
        outs = vpd.run_ranks(ctxs, lambda r, c: vm.run_alg2(c, batch, [_shard(Wd, p, r)]))
        for c in ctxs:
            c.sync()
        assert [c.fused_c1_count for c in ctxs] == [fused] * p
        res[fused] = outs[0]
        _close(ctxs)
    assert torch.allclose(res[0].grad_x, res[1].grad_x, rtol=1e-5, atol=1e-6)
    assert torch.allclose(res[0].loss, res[1].loss, rtol=1e-6, atol=1e-6)


def test_fused_c1_repeated_steps_and_growth():
    # back-to-back steps reuse the peer buffers (write-after-read across
    # steps is ordered by the grad_x all-gather); a larger batch grows them
    p, h, V = 4, 128, 4096
    ctxs = vpd.local_group(p)
    for T in (128, 128, 640, 128):
        X, W, g = oracle.random_instance(T, h, V, T)
        Xb, Wb, batch, Wd = device_case(X, W, g)
        ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
        outs = vpd.run_ranks(ctxs, lambda r, c: vm.run_alg2(c, batch, [_shard(Wd, p, r)]))
        for c in ctxs:
            c.sync()
        res = {"loss": outs[1].loss.double().cpu().numpy(), "grad_x": outs[1].grad_x[:, :h].double().cpu().numpy(),
               "grad_w": torch.cat([o.grad_w[0] for o in outs])[:, :h].double().cpu().numpy()}
        assert_parity(res, ref, f"fused C1 step T={T}")
    assert [c.fused_c1_count for c in ctxs] == [4] * p
    _close(ctxs)


def test_fused_c1_across_processes(tmp_path):
    # two processes on one GPU (torchrun): the peer buffers are CUDA IPC
    # mappings, the path a one-process-per-GPU NCCL group takes
    import socket
    import subprocess
    import sys
    import json
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(here, "mp_fused_worker.py"),
           str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    reps = [json.load(open(tmp_path / f"rank{k}.json")) for k in range(2)]
    for rep in reps:
        assert rep["ok"], rep


@pytest.mark.parametrize("alg", ["alg2", "alg1"])
def test_fused_exchange_llama_vocab_8_ranks(alg):
    # the Llama-3 vocabulary over 8 ranks (ragged 16032-row shards, 251
    # k-blocks of dX per rank) through the fused exchange: the one-GPU bits
    p, T, h, V = 8, 2048, 512, 128256
    opts = (("splits_dx", 1), ("splits_dw", 1))
    Xb, Wb, g, local, local_ctx, ctxs, outs = _local_and_group(p, T, h, V, 77, opts, alg)
    assert [c.fused_c1_count for c in ctxs] == [1] * p
    for o in outs:
        assert torch.equal(o.loss, local.loss) and torch.equal(o.grad_x, local.grad_x)
    assert torch.equal(torch.cat([o.grad_w[0] for o in outs]), local.grad_w_full())
    ref = oracle.oracle_output_layer(Xb[:256], g[:256], Wb, want_softmax=False)
    assert np.abs(outs[0].loss[:256].double().cpu().numpy() - ref.loss).max() <= LOSS_ABS
    _close(ctxs)
    local_ctx.close()


def test_fused_exchange_random_shapes():
    # seeded random shapes (token counts, hidden sizes that are multiples of 8
    # but not of the 32-column store box, vocabularies with ragged shards):
    # fused group == one-GPU p-shard run, bit for bit
    rng = np.random.default_rng(2024)
    for case in range(10):
        p = int(rng.integers(2, 9))
        T = int(rng.integers(1, 700))
        h = int(8 * rng.integers(1, 40))
        V = int(p * rng.integers(40, 900))
        alg = "alg2" if case % 3 else "alg1"
        opts = (("splits_dx", 1), ("splits_dw", 1))
        Xb, Wb, g, local, local_ctx, ctxs, outs = _local_and_group(p, T, h, V, 500 + case, opts, alg)
        tag = (case, p, T, h, V, alg)
        assert [c.fused_c1_count for c in ctxs] == [1] * p, tag
        for o in outs:
            assert torch.equal(o.loss, local.loss) and torch.equal(o.grad_x, local.grad_x), tag
        assert torch.equal(torch.cat([o.grad_w[0] for o in outs]), local.grad_w_full()), tag
        _close(ctxs)
        local_ctx.close()


def test_input_peer_paths_random_shapes():
    # seeded random input-layer shapes through the peer-memory forward and the
    # gathered backward: bit-equal to W[tok] and to the ascending-i oracle
    rng = np.random.default_rng(99)
    for case in range(8):
        p = int(rng.integers(2, 9))
        T = int(rng.integers(1, 3000))
        h = int(8 * rng.integers(1, 64))
        V = int(p * rng.integers(10, 400))
        W = torch.from_numpy(rng.standard_normal((V, h)).astype(np.float32)).to(torch.bfloat16).cuda()
        t = rng.integers(0, V + 7, T)  # a few ids past V: zero rows, ignored by the backward
        tok = torch.from_numpy(t.astype(np.int64)).cuda()
        grad = torch.from_numpy(rng.standard_normal((T, h)).astype(np.float32)).to(torch.bfloat16).cuda()
        root = int(rng.integers(0, p))
        torch.cuda.synchronize()
        ctxs = vpd.local_group(p)

        def rank(r, ctx):
            sh = _shard(W, p, r)
            out = vm.input_forward_gathered(ctx, tok, sh)
            dE = vm.input_backward_gathered(ctx, grad if r == root else None, tok, sh, root=root, h=h)
            ctx.sync()
            return out, dE

        res = vpd.run_ranks(ctxs, rank)
        want = torch.zeros(T, h, dtype=torch.bfloat16, device="cuda")
        own = tok < V
        want[own] = W[tok[own]]
        g_np = grad.float().cpu().numpy()
        for r, (out, dE) in enumerate(res):
            assert torch.equal(out, want), (case, r)
            rb, re = vpd.shard_rows(V, p, r)
            ref = oracle.input_backward_f32(g_np, t, re - rb, rb)
            assert np.array_equal(dE.cpu().numpy(), ref), (case, r)
        assert [c.peer_input_count for c in ctxs] == [2] * p
        _close(ctxs)


@pytest.mark.parametrize("alg", ["alg2", "alg1"])
def test_fused_exchange_fault_scale(alg):
    # the reference's fault hook (sum scaled after the merge, VM.cpp:314 /
    # :337-350) through the fused exchange: the one-GPU bits with the same fault
    p, T, h, V = 4, 200, 64, 2000
    fn = {"alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg]
    X, W, g = oracle.random_instance(T, h, V, 13)
    _, _, batch, Wd = device_case(X, W, g)
    lctx = vm.Context(0)
    for k, v in (("splits_dx", 1), ("splits_dw", 1)):
        lctx.set_option(k, v)
    local = fn(lctx, batch, vm.shard_weights(Wd, p), fault_scale=1.5)
    lctx.sync()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    for c in ctxs:
        c.set_option("splits_dx", 1)
        c.set_option("splits_dw", 1)
    outs = vpd.run_ranks(ctxs, lambda r, c: fn(c, batch, [_shard(Wd, p, r)], fault_scale=1.5))
    for c in ctxs:
        c.sync()
    assert [c.fused_c1_count for c in ctxs] == [1] * p
    for o in outs:
        assert torch.equal(o.loss, local.loss) and torch.equal(o.grad_x, local.grad_x)
    assert torch.equal(torch.cat([o.grad_w[0] for o in outs]), local.grad_w_full())
    _close(ctxs)
    lctx.close()


def test_executor_fused_microbatches_of_different_lengths():
    # one peer region per microbatch sized for the longest; ragged lengths
    import json
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "programs.json")))
    prog = vm.Program(golden["vocab2_p4_n8"]["text"])
    p, n = prog.p, prog.n
    h, V = 64, 96 * p
    lens = [48, 100, 17, 64, 200, 33, 96, 1][:n]
    W = None
    mbs = []
    for i in range(n):
        X, W_i, g = oracle.random_instance(lens[i], h, V, 300 + i)
        W = W_i if W is None else W
        mbs.append(device_case(X, W, g))
    Wd = mbs[0][3]
    lctx = vm.Context(0)
    local = vm.run_program(lctx, prog, [m[2] for m in mbs], vm.shard_weights(Wd, p))
    lctx.sync()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)

    def rank(r, ctx):
        batches = [vm.TokenBatch(m[2].X.clone() if r == p - 1 else torch.zeros_like(m[2].X), m[2].labels)
                   for m in mbs]
        res = vm.run_program(ctx, prog, batches, [_shard(Wd, p, r)])
        ctx.sync()
        return res

    outs = vpd.run_ranks(ctxs, rank)
    assert [c.fused_c1_count for c in ctxs] == [n] * p
    for r, res in enumerate(outs):
        for i in range(n):
            assert torch.equal(res.grad_x[i], outs[0].grad_x[i])
            assert torch.allclose(res.loss[i], local.loss[i], rtol=1e-5, atol=1e-6)
            assert torch.allclose(res.grad_x[i], local.grad_x[i], rtol=1e-4, atol=1e-6)
        assert torch.allclose(res.grad_w[0], local.grad_w[r], rtol=1e-4, atol=1e-6)
    _close(ctxs)
    lctx.close()


def test_fused_exchange_soak_back_to_back_steps():
    # many back-to-back steps on one group without host synchronisation
    # between them (the ordering across steps is all stream-side: routed
    # stores after the previous loss barrier, combine after the stats
    # all-gather, pulls before the next step's writes); alternating algorithms
    # and the input layer; every step equals its one-GPU p-shard run bitwise
    p, h = 4, 64
    rng = np.random.default_rng(5)
    steps = []
    for it in range(24):
        T = int(rng.integers(30, 400))
        V = 400 * p
        X, W, g = oracle.random_instance(T, h, V, 1000 + it)
        steps.append((["alg2", "alg1", "chunked"][it % 3], device_case(X, W, g)))
    lctx = vm.Context(0)
    for k, v in (("splits_dx", 1), ("splits_dw", 1)):
        lctx.set_option(k, v)
    want = []
    for alg, (_, _, batch, Wd) in steps:
        sh = vm.shard_weights(Wd, p)
        if alg == "chunked":
            want.append(vm.run_alg2_chunked(lctx, batch, sh, 64))
        else:
            want.append({"alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg](lctx, batch, sh))
    lctx.sync()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    for c in ctxs:
        c.set_option("splits_dx", 1)
        c.set_option("splits_dw", 1)

    def rank(r, c):
        outs = []
        for alg, (_, _, batch, Wd) in steps:
            sh = [_shard(Wd, p, r)]
            if alg == "chunked":
                outs.append(vm.run_alg2_chunked(c, batch, sh, 64))
            else:
                outs.append({"alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg](c, batch, sh))
            vm.input_forward_gathered(c, batch.labels, sh[0])  # interleave the input layer's exchanges
        c.sync()
        return outs

    res = vpd.run_ranks(ctxs, rank)
    for it, (alg, _) in enumerate(steps):
        for r in range(p):
            assert torch.equal(res[r][it].loss, want[it].loss), (it, alg, r)
            assert torch.equal(res[r][it].grad_x, want[it].grad_x), (it, alg, r)
        assert torch.equal(torch.cat([res[r][it].grad_w[0] for r in range(p)]), want[it].grad_w_full()), (it, alg)
    _close(ctxs)
    lctx.close()


@pytest.mark.parametrize("pinned", [True, False])
def test_fused_exchange_at_the_headline_shape(pinned):
    # T=8192, h=4096, V=256000 as 2 loopback ranks through the fused exchange:
    # bitwise the one-GPU 2-shard run with split-K pinned (random bf16 operands
    # drawn on the device); with the production split-K choice (ranks sharing
    # the GPU get half its SMs, so their splits may differ) within fp32 noise
    p, T, h, V = 2, 8192, 4096, 256000
    gen = torch.Generator(device="cuda").manual_seed(21)
    X = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    Wd = (torch.randn(V, h, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    lab = torch.randint(0, V, (T,), device="cuda", generator=gen)
    batch = vm.TokenBatch(X, lab)
    opts = (("splits_dx", 1), ("splits_dw", 1)) if pinned else ()
    lctx = vm.Context(0)
    for k, v in opts:
        lctx.set_option(k, v)
    local = vm.run_alg2(lctx, batch, vm.shard_weights(Wd, p))
    lctx.sync()
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)
    for c in ctxs:
        for k, v in opts:
            c.set_option(k, v)
    outs = vpd.run_ranks(ctxs, lambda r, c: vm.run_alg2(c, batch, [_shard(Wd, p, r)]))
    for c in ctxs:
        c.sync()
    assert [c.fused_c1_count for c in ctxs] == [1] * p
    same = torch.equal if pinned else (lambda a, b: torch.allclose(a, b, rtol=1e-4, atol=1e-6))
    for o in outs:
        assert torch.equal(o.grad_x, outs[0].grad_x)  # every rank holds the same bits
        assert same(o.loss, local.loss) and same(o.grad_x, local.grad_x)
    for r in range(p):
        rb, re = vpd.shard_rows(V, p, r)
        assert same(outs[r].grad_w[0], local.grad_w_full()[rb:re])
    _close(ctxs)
    lctx.close()


def test_tied_embeddings_over_a_group():
    # tied input / output embeddings with vocabulary parallelism over p ranks
    # (R/PAPER.md:333): the input forward pulls rows over peer memory, the
    # output layer runs the fused exchange, and each rank's shard gradient
    # accumulates dW_k (output) + dE_k (the gathered input backward, gradient
    # from the root) in ONE buffer; checked against the oracle
    p, T, h, V = 4, 160, 64, 1024
    X, W, g = oracle.random_instance(T, h, V, 61)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    rng = np.random.default_rng(7)
    toks = rng.integers(0, V, T)
    toks[:30] = toks[0]
    tok_d = torch.from_numpy(toks).cuda()
    grad_emb = torch.from_numpy(rng.standard_normal((T, h)).astype(np.float32)).cuda().to(torch.bfloat16)
    torch.cuda.synchronize()
    ctxs = vpd.local_group(p)

    def rank(r, c):
        sh = _shard(Wd, p, r)
        emb = vm.input_forward_gathered(c, tok_d, sh)
        gbuf = torch.empty(sh.rows(), h, dtype=torch.float32, device="cuda")
        outs = vm._alloc_outputs(c, batch, [sh])
        vm.run_alg2(c, batch, [sh], outputs=(outs[0], outs[1], [gbuf], outs[3]))
        vm.input_backward_gathered(c, grad_emb if r == 0 else None, tok_d, sh, root=0, h=h, out=gbuf,
                                   accumulate=True)
        c.sync()
        return emb, gbuf

    res = vpd.run_ranks(ctxs, rank)
    for emb, _ in res:
        assert torch.equal(emb, Wd[tok_d])
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    dE = oracle.input_backward_f32(grad_emb.float().cpu().numpy(), toks, V, 0).astype(np.float64)
    got = torch.cat([gb for _, gb in res])[:, :h].double().cpu().numpy()
    assert rel_l2(got, ref.grad_w + dE) <= GRAD_REL_L2
    assert [c.fused_c1_count for c in ctxs] == [1] * p and [c.peer_input_count for c in ctxs] == [2] * p
    _close(ctxs)
