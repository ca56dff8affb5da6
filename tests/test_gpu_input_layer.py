"""GPU parity of the vocabulary-parallel INPUT layer: bit-exact forward and
bit-exact (fp32, ascending-i) gradient against the oracle."""
import numpy as np
import pytest
import torch

from gpu_helpers import bf16_round, to_dev_bf16
from paper_2411_05288_b200 import vocab_math as vm

import oracle

pytestmark = pytest.mark.gpu


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy()


def test_input_forward_composes_bit_exactly(ctx):
    # test_vocab_math.cpp:166-189 (forward diff exactly 0) on bf16 rows
    _, W, _ = oracle.random_instance(10, 8, 20, 4)
    Wb = bf16_round(W)
    tokens = np.array([3, 19, 0, 7, 7, 12, 5, 18, 1, 10], dtype=np.int64)
    Wd = to_dev_bf16(Wb, 8)
    td = torch.from_numpy(tokens).cuda()
    acc = torch.zeros(10, 8, dtype=torch.bfloat16, device="cuda")
    for s in vm.shard_weights(Wd, 4):
        part = vm.input_forward(ctx, td, s)
        ref = oracle.input_forward(tokens, Wb[s.row_begin:s.row_end], s.row_begin)
        assert np.array_equal(part.float().cpu().numpy(), ref)
        acc += part
    ctx.sync()
    assert np.array_equal(acc.float().cpu().numpy(), Wb[tokens])
    # the fused accumulate form gives the same bits
    acc2 = torch.zeros_like(acc)
    for s in vm.shard_weights(Wd, 4):
        vm.input_forward(ctx, td, s, out=acc2, accumulate=True)
    assert torch.equal(acc, acc2)


def test_input_forward_c4_shape_bit_exact(ctx):
    # BASELINE configs[3]: V=256000, h=4096, 16384 ids; p=8 shards, every row exact
    V, h, T = 256000, 4096, 16384
    gen = torch.Generator(device="cuda").manual_seed(7)
    W = (torch.randn(V, h, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    tok = torch.randint(0, V, (T,), device="cuda", generator=gen)
    out = torch.zeros(T, h, dtype=torch.bfloat16, device="cuda")
    for s in vm.shard_weights(W, 8):
        vm.input_forward(ctx, tok, s, out=out, accumulate=True)
    ctx.sync()
    assert torch.equal(out, W[tok])


def test_input_forward_unowned_and_negative_tokens(ctx):
    W = torch.ones(8, 8, dtype=torch.bfloat16, device="cuda")
    s = vm.shard_weights(W, 2)[1]  # rows [4, 8)
    out = vm.input_forward(ctx, torch.tensor([5, 100, 2], device="cuda"), s)
    ctx.sync()
    assert out[0].eq(1).all() and out[1].eq(0).all() and out[2].eq(0).all()
    vm.input_forward(ctx, torch.tensor([0, -1], device="cuda"), s)
    with pytest.raises(ValueError, match="input_forward: token out of range"):
        ctx.sync()


@pytest.mark.parametrize("grad_dtype", [torch.bfloat16, torch.float32])
def test_input_backward_bit_exact_with_repeats(ctx, grad_dtype):
    rng = np.random.default_rng(0)
    T, h, V, p = 4096, 256, 3000, 4
    tokens = rng.integers(0, 64, T)          # heavy repetition: long segments
    tokens[::7] = rng.integers(0, V, len(tokens[::7]))
    g = rng.standard_normal((T, h)).astype(np.float32)
    gd = torch.from_numpy(g).cuda().to(grad_dtype)
    g_used = gd.float().cpu().numpy()       # widened bf16 (or the fp32 itself)
    Wd = torch.zeros(V, h, dtype=torch.bfloat16, device="cuda")
    td = torch.from_numpy(tokens.astype(np.int64)).cuda()
    for s in vm.shard_weights(Wd, p):
        dE = vm.input_backward(ctx, gd, td, s)
        ref = oracle.input_backward_f32(g_used, tokens, s.rows(), s.row_begin)
        assert np.array_equal(dE.cpu().numpy(), ref), s.index
        # accumulate mode continues the same ascending-i sum from the existing rows
        init = np.arange(s.rows() * h, dtype=np.float32).reshape(s.rows(), h) * 1e-3
        dE2 = torch.from_numpy(init).cuda()
        vm.input_backward(ctx, gd, td, s, out=dE2, accumulate=True)
        ref2 = oracle.input_backward_f32(g_used, tokens, s.rows(), s.row_begin, init=init)
        assert np.array_equal(dE2.cpu().numpy(), ref2)


def test_input_backward_matches_fp64_reference_closely(ctx):
    # the reference test's semantic check (stacked gradient == monolithic
    # scatter) with the fp32-vs-fp64 tolerance of a 64-term sum
    X, W, _ = oracle.random_instance(10, 8, 20, 4)
    tokens = np.array([3, 19, 0, 7, 7, 12, 5, 18, 1, 10], dtype=np.int64)
    Wd = torch.zeros(20, 8, dtype=torch.bfloat16, device="cuda")
    gd = torch.from_numpy(X.astype(np.float32)).cuda()
    bwd = torch.cat([vm.input_backward(ctx, gd, torch.from_numpy(tokens).cuda(), s)
                     for s in vm.shard_weights(Wd, 4)]).cpu().numpy()
    ref = np.zeros((20, 8))
    for i, t in enumerate(tokens):
        ref[t] += X[i]
    assert np.abs(bwd - ref).max() < 1e-6


def test_input_backward_c4_shape_deterministic(ctx):
    V, h, T = 256000, 4096, 16384
    gen = torch.Generator(device="cuda").manual_seed(9)
    tok = torch.randint(0, V, (T,), device="cuda", generator=gen)
    tok[:512] = 17  # a hot token
    grad = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    s = vm.shard_weights(torch.zeros(V, h, dtype=torch.bfloat16, device="cuda"), 8)[0]
    a = vm.input_backward(ctx, grad, tok, s)
    b = vm.input_backward(ctx, grad, tok, s)
    ctx.sync()
    assert torch.equal(a, b)
    own = (tok >= s.row_begin) & (tok < s.row_end)
    ref = oracle.input_backward_f32(grad.float().cpu().numpy(), tok.cpu().numpy(), s.rows(), s.row_begin)
    assert np.array_equal(a.cpu().numpy(), ref)
    assert own.any()


def test_input_backward_negative_token_raises(ctx):
    s = vm.shard_weights(torch.zeros(8, 8, dtype=torch.bfloat16, device="cuda"), 1)[0]
    vm.input_backward(ctx, torch.ones(2, 8, device="cuda"), torch.tensor([1, -2], device="cuda"), s)
    with pytest.raises(ValueError, match="input_backward: token out of range"):
        ctx.sync()
    with pytest.raises(ValueError, match="grad/token length mismatch"):
        vm.input_backward(ctx, torch.ones(3, 8, device="cuda"), torch.tensor([1, 2], device="cuda"), s)


def _zipf_ids(T, V, s, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    k = torch.arange(1, V + 1, device="cuda", dtype=torch.float64)
    ranks = torch.multinomial((1.0 / k.pow(s)).float(), T, replacement=True, generator=gen)
    return torch.randperm(V, device="cuda", generator=gen)[ranks]


@pytest.mark.parametrize("grad_dtype", [torch.bfloat16, torch.float32])
def test_input_backward_zipf_ids_bit_exact(ctx, grad_dtype):
    # Zipf(1.1) token ids at the config-4 shape: hot rows with thousands of
    # occurrences (column-chunked, bulk-copy streamed) next to unique rows —
    # still the ascending-i fp32 sum, bit for bit, accumulating into dE
    V, h, T = 256000, 4096, 16384
    tok = _zipf_ids(T, V, 1.1, 3)
    counts = torch.bincount(tok, minlength=V)
    assert counts.max().item() > 1000 and (counts == 1).sum().item() > 1000
    grad = torch.randn(T, h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)).to(grad_dtype)
    p = 8  # the shard holding the hottest token (keeps the host-side reference at 0.5 GB)
    shards = vm.shard_weights(torch.zeros(V, h, dtype=torch.bfloat16, device="cuda"), p)
    s = shards[int(counts.argmax().item()) // (V // p)]
    init = torch.randn(s.rows(), h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    dE = init.clone()
    vm.input_backward(ctx, grad, tok, s, out=dE, accumulate=True)
    ctx.sync()
    ref = oracle.input_backward_f32(grad.float().cpu().numpy(), tok.cpu().numpy(), s.rows(), s.row_begin,
                                    init=init.cpu().numpy())
    assert np.array_equal(dE.cpu().numpy(), ref)


@pytest.mark.parametrize("T,h", [(5000, 520), (16384, 4096), (3000, 8)])
def test_input_backward_every_multiplicity_class(ctx, T, h):
    # rows occurring once, 2..15 times (whole-row path), 16..32 (hot chunks,
    # warp-sorted segment), 33..T (hot chunks, bitmap-sorted segment) and one
    # row holding most of the batch; ragged last hot chunk when h % 256 != 0
    rng = np.random.default_rng(T + h)
    V = 40000
    tok = rng.integers(0, V, T)
    pos = rng.permutation(T)
    k = 0
    for row, c in [(11, 2), (12, 7), (13, 15), (14, 16), (15, 31), (16, 32), (17, 33), (18, 300), (19, T // 3)]:
        tok[pos[k:k + c]] = row
        k += c
    g = torch.from_numpy(rng.standard_normal((T, h)).astype(np.float32)).cuda().to(torch.bfloat16)
    td = torch.from_numpy(tok.astype(np.int64)).cuda()
    for s in vm.shard_weights(torch.zeros(V, h, dtype=torch.bfloat16, device="cuda"), 4):
        dE = vm.input_backward(ctx, g, td, s)
        ctx.sync()
        ref = oracle.input_backward_f32(g.float().cpu().numpy(), tok, s.rows(), s.row_begin)
        assert np.array_equal(dE.cpu().numpy(), ref), s.index


def test_input_peer_paths_capture_over_nccl():
    # the peer-memory input forward and the gathered backward on a forced
    # 1-rank NCCL group: capturable after the first (sizing) call; replays on
    # new ids / gradients are bit-exact
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        rng = np.random.default_rng(7)
        V, h, T = 3000, 256, 1500
        W = torch.from_numpy(rng.standard_normal((V, h)).astype(np.float32)).to(torch.bfloat16).cuda()
        sh = vm.shard_weights(W, 1)[0]
        tok = torch.from_numpy(rng.integers(0, V, T).astype(np.int64)).cuda()
        grad = torch.from_numpy(rng.standard_normal((T, h)).astype(np.float32)).to(torch.bfloat16).cuda()
        nctx = vm.Context(0)
        nctx.comm_init(1, 0, vm.Context.unique_id())
        nctx.set_option("force_collectives", 1)
        emb = torch.empty(T, h, dtype=torch.bfloat16, device="cuda")
        dE = torch.empty(V, h, dtype=torch.float32, device="cuda")

        def step():
            vm.input_forward_gathered(nctx, tok, sh, out=emb)
            vm.input_backward_gathered(nctx, grad, tok, sh, root=0, out=dE)

        step()
        nctx.sync()
        graph = vm.capture(nctx, step)
        for seed in (1, 2):
            r2 = np.random.default_rng(seed)
            t2 = r2.integers(0, V, T)
            tok.copy_(torch.from_numpy(t2.astype(np.int64)))
            grad.copy_(torch.from_numpy(r2.standard_normal((T, h)).astype(np.float32)).to(torch.bfloat16))
            graph.launch()
            nctx.sync()
            assert torch.equal(emb, W[tok])
            ref = oracle.input_backward_f32(grad.float().cpu().numpy(), t2, V, 0)
            assert np.array_equal(dE.cpu().numpy(), ref)
        assert nctx.peer_input_count == 4  # host calls: the sizing step and the captured step
        graph.close()
        nctx.close()
