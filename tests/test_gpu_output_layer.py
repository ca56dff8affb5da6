"""GPU parity of the vocabulary-parallel OUTPUT layer (through the C ABI)
against the CPU oracle on the same bf16-rounded inputs.

Tolerances (BASELINE.json north_star): per-token loss <= 1e-3 absolute,
grad_x / grad_w <= 1e-2 relative L2; softmax <= 4e-3 absolute (bf16 P).
"""
import numpy as np
import pytest
import torch

from gpu_helpers import (GRAD_REL_L2, LOSS_ABS, assert_parity, bf16_round, device_case, fp64_full_check, oracle,
                         pad8, rel_l2, run_device, to_dev_bf16)
from paper_2411_05288_b200 import vocab_math as vm

pytestmark = pytest.mark.gpu

ALGS = ("naive", "alg1", "alg2")


def test_reference_grid_all_algorithms(ctx):
    # test_vocab_math.cpp:86-106 grid (b, s, h, V, p, seeds) at GPU tolerances
    worst = [0.0, 0.0, 0.0]
    for b in (1, 2):
        for s in (2, 8):
            for h in (4, 16):
                for V in (16, 64):
                    for p in (1, 2, 4, 8):
                        if V % p:
                            continue
                        for seed in (0, 1, 2):
                            X, W, g = oracle.random_instance(b * s, h, V, seed)
                            Xb, Wb, batch, Wd = device_case(X, W, g)
                            ref = oracle.oracle_output_layer(Xb, g, Wb)
                            for alg in ALGS:
                                res, _ = run_device(ctx, alg, batch, Wd, p, h)
                                d = assert_parity(res, ref, f"{alg} b={b} s={s} h={h} V={V} p={p} seed={seed}")
                                worst = [max(a, c) for a, c in zip(worst, d)]
    print("grid worst (loss, gx, gw):", worst)


@pytest.mark.parametrize("alg", ALGS)
def test_config1_cpu_reference_shape(ctx, alg):
    # BASELINE configs[0]: 1024 tokens, h=512, V=32000, 4 simulated shards
    X, W, g = oracle.random_instance(1024, 512, 32000, 0)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    res, _ = run_device(ctx, alg, batch, Wd, 4, 512, with_softmax=False)
    assert_parity(res, ref, f"c1 {alg}")


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_llama_vocab_ragged_shards(ctx, p):
    # Llama-3 vocabulary V=128256: V/p = 16032 at p=8 is not a multiple of the
    # 256-wide vocab tile (masked tail tiles); h=4096, few tokens for the oracle
    rng = np.random.default_rng(p)
    T, h, V = 16, 4096, 128256
    X = rng.standard_normal((T, h))
    W = rng.standard_normal((V, h)) * 0.02
    g = rng.integers(0, V, T)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    for alg in ("alg1", "alg2"):
        res, _ = run_device(ctx, alg, batch, Wd, p, h, with_softmax=False)
        assert_parity(res, ref, f"llama p={p} {alg}")


def test_gemma_shape_8_shards_reduced_tokens(ctx):
    # BASELINE configs[2]: h=3584, V=256000, sharded 8 ways (T reduced for the oracle)
    rng = np.random.default_rng(3)
    T, h, V = 8, 3584, 256000
    X = rng.standard_normal((T, h))
    W = rng.standard_normal((V, h)) * 0.02
    g = rng.integers(0, V, T)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    res, _ = run_device(ctx, "alg2", batch, Wd, 8, h, with_softmax=False)
    assert_parity(res, ref, "gemma p=8 alg2")


@pytest.mark.parametrize("V", [32000, 128256, 262144, 524288])
def test_vocab_sweep_8_shards_naive_and_alg2(ctx, V):
    # BASELINE configs[4] (vocabulary sweep 32k-512k at h=4096, 8 shards),
    # naive 3-barrier vs reduced-barrier, T reduced for the oracle
    rng = np.random.default_rng(V % 1000)
    T, h = 8, 4096
    X = rng.standard_normal((T, h))
    W = rng.standard_normal((V, h)) * 0.02
    g = rng.integers(0, V, T)
    g[0] = V - 1  # the last row of the last shard
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    for alg in ("naive", "alg2"):
        res, _ = run_device(ctx, alg, batch, Wd, 8, h, with_softmax=False)
        assert_parity(res, ref, f"sweep V={V} {alg}")


def test_large_logits_uniform_inputs(ctx):
    # reference-style U[-1,1] operands at h=2048: logit std ~26, so the
    # per-tile max subtraction is exercised hard
    X, W, g = oracle.random_instance(64, 2048, 4096, 11)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb)
    for alg in ALGS:
        res, _ = run_device(ctx, alg, batch, Wd, 4, 2048)
        assert_parity(res, ref, f"U[-1,1] {alg}")


def test_corrupting_the_correction_factor_is_detected(ctx):
    # test_vocab_math.cpp:108-114 at GPU tolerance: log(1.01) ~ 1e-2 > 1e-3
    X, W, g = oracle.random_instance(64, 64, 256, 3)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb)
    for alg in ("alg1", "alg2"):
        good, _ = run_device(ctx, alg, batch, Wd, 4, 64)
        bad, _ = run_device(ctx, alg, batch, Wd, 4, 64, fault_scale=1.01)
        assert np.abs(good["loss"] - ref.loss).max() <= LOSS_ABS
        assert np.abs(bad["loss"] - ref.loss).max() > LOSS_ABS


def test_pass_functions_compose_like_the_drivers(ctx):
    # alg2_pass_S x p -> alg2_barrier_C1 -> alg2_pass_T x p == run_alg2 (bitwise)
    X, W, g = oracle.random_instance(40, 24, 96, 5)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    shards = vm.shard_weights(Wd, 4)
    states = [vm.alg2_pass_S(ctx, batch, s) for s in shards]
    c1 = vm.alg2_barrier_C1(ctx, states, shards, batch)
    gw = torch.cat([vm.alg2_pass_T(ctx, st, c1.stats, batch, s) for st, s in zip(states, shards)])
    run = vm.run_alg2(ctx, batch, shards)
    assert torch.equal(c1.grad_x, run.grad_x)
    assert torch.equal(gw, run.grad_w_full())
    assert torch.equal(c1.stats.m, run.stats.m) and torch.equal(c1.stats.sum, run.stats.sum)
    # alg1 passes: S -> merge (C1) -> T -> C2
    states1 = [vm.alg1_pass_S(ctx, batch, s) for s in shards]
    stats = vm.merge_max_sum(ctx, states1)
    grads = [vm.alg1_pass_T(ctx, st, stats, batch, s) for st, s in zip(states1, shards)]
    gx = vm.reduce_grad_x(ctx, [gr.grad_x_partial for gr in grads])
    ref = oracle.oracle_output_layer(Xb, g, Wb)
    assert rel_l2(gx[:, :24].cpu().numpy(), ref.grad_x) <= GRAD_REL_L2
    assert rel_l2(torch.cat([gr.grad_w for gr in grads])[:, :24].cpu().numpy(), ref.grad_w) <= GRAD_REL_L2
    # T passes are pure: calling again gives identical bits (SPEC "arbitrarily delayable")
    again = vm.alg1_pass_T(ctx, states1[1], stats, batch, shards[1])
    assert torch.equal(again.grad_w, grads[1].grad_w)
    assert torch.equal(again.grad_x_partial, grads[1].grad_x_partial)


def test_local_stats_and_merge_match_the_oracle(ctx):
    # alg1_pass_S m'/sum' per shard and merge_max_sum vs the oracle
    X, W, g = oracle.random_instance(7, 8, 12, 9)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    shards = vm.shard_weights(Wd, 4)
    states = [vm.alg1_pass_S(ctx, vm.TokenBatch(batch.X, None), s) for s in shards]
    ms, ss = [], []
    for k, st in enumerate(states):
        m_ref, s_ref = oracle.local_stats(Xb, Wb, 4, k)
        ls = st.local_stats()
        assert np.abs(ls.m.cpu().numpy() - m_ref).max() < 1e-4
        assert rel_l2(ls.sum.cpu().numpy(), s_ref) < 1e-3
        ms.append(m_ref)
        ss.append(s_ref)
        # softmax' rows sum to one (ShardState invariant, SPEC.md)
        assert torch.allclose(st.softmax_local().sum(dim=1), torch.ones(7, device="cuda"), atol=1e-2)
    gm, gs = oracle.merge_max_sum(ms, ss)
    stats = vm.merge_max_sum(ctx, states)
    assert np.abs(stats.m.cpu().numpy() - gm).max() < 1e-4
    assert rel_l2(stats.sum.cpu().numpy(), gs) < 1e-3


def test_frozen_merge_on_device(ctx):
    # test_vocab_math.cpp:153-164 in fp32 on the device
    parts = [vm.LocalStats(torch.tensor([0.0], device="cuda"), torch.tensor([1.0], device="cuda")),
             vm.LocalStats(torch.tensor([1.0], device="cuda"), torch.tensor([1.0], device="cuda"))]
    out = vm.merge_max_sum(ctx, parts)
    assert out.m.item() == 1.0
    assert abs(out.sum.item() - 1.3678794411714423) < 1e-6
    rev = vm.merge_max_sum(ctx, parts[::-1])
    assert rev.m.item() == out.m.item()
    with pytest.raises(ValueError, match="length mismatch"):
        vm.merge_max_sum(ctx, [parts[0], vm.LocalStats(torch.zeros(2, device="cuda"), torch.ones(2, device="cuda"))])
    with pytest.raises(ValueError, match="empty input"):
        vm.merge_max_sum(ctx, [])


def test_outputs_are_deterministic(ctx):
    X, W, g = oracle.random_instance(300, 64, 2000, 1)
    _, _, batch, Wd = device_case(X, W, g)
    for alg in ALGS:
        a, _ = run_device(ctx, alg, batch, Wd, 4, 64, with_softmax=False)
        b, _ = run_device(ctx, alg, batch, Wd, 4, 64, with_softmax=False)
        for k in a:
            assert np.array_equal(a[k], b[k]), (alg, k)


def test_cta_group_1_matches_cta_group_2(ctx):
    X, W, g = oracle.random_instance(200, 128, 1500, 2)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    c1 = vm.Context(0, cta_group=1)
    res, _ = run_device(c1, "alg2", batch, Wd, 2, 128, with_softmax=False)
    assert_parity(res, ref, "cta_group::1")
    c1.close()


def test_argument_errors(ctx):
    X, W, g = oracle.random_instance(4, 8, 16, 0)
    _, _, batch, Wd = device_case(X, W, g)
    with pytest.raises(ValueError, match="V not divisible by p"):
        vm.shard_weights(Wd, 5)
    shards = vm.shard_weights(Wd, 2)
    st = vm.alg1_pass_S(ctx, batch, shards[0])
    with pytest.raises(ValueError, match="A/B terms missing"):
        vm.alg2_barrier_C1(ctx, [st], shards[:1], batch)
    bad = vm.TokenBatch(torch.zeros(4, 12, dtype=torch.bfloat16, device="cuda"), batch.labels)
    with pytest.raises(ValueError):
        vm.alg1_pass_S(ctx, bad, shards[0])


def _synthetic(T, h, V, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    X = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    W = (torch.randn(V, h, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    labels = torch.randint(0, V, (T,), device="cuda", generator=gen)
    return X, W, labels


def test_fp64_streamed_reference_is_pinned_to_the_oracle():
    # the full-size checker must agree with the CPU oracle where both run
    import types
    X, W, g = oracle.random_instance(50, 24, 700, 4)
    ref = oracle.oracle_output_layer(X, g, W, want_softmax=False)
    as_t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    fake = types.SimpleNamespace(loss=as_t(ref.loss), grad_x=as_t(ref.grad_x), grad_w=[as_t(ref.grad_w)])
    dl, gx, gw = fp64_full_check(fake, as_t(X), as_t(W), as_t(g), chunk=128)
    assert dl < 1e-10 and gx < 1e-10 and gw < 1e-10, (dl, gx, gw)


def test_headline_shape_full_parity(ctx):
    # BASELINE metric config at full size (T=8192, h=4096, V=256000, p=1):
    # size-independent properties, then EVERY loss / grad_x / grad_w entry
    # against an fp64 restatement streamed over vocab chunks (fp64_full_check)
    T, h, V = 8192, 4096, 256000
    X, W, labels = _synthetic(T, h, V, 1234)
    batch = vm.TokenBatch(X, labels)
    out = vm.run_alg2(ctx, batch, vm.shard_weights(W, 1))
    ctx.sync()
    assert torch.isfinite(out.loss).all() and (out.loss > 0).all()
    # sum_v grad_y[i, v] = 0  =>  column sums of grad_w vanish relative to |X| sums
    colsum = out.grad_w[0].sum(dim=0, dtype=torch.float64)
    assert colsum.abs().max().item() < 1e-2 * X.float().abs().sum(dim=0).max().item()
    dl, gx, gw = fp64_full_check(out, X, W, labels)
    assert dl <= LOSS_ABS and gx <= GRAD_REL_L2 and gw <= GRAD_REL_L2, (dl, gx, gw)


@pytest.mark.parametrize("alg", ["alg1", "alg2"])
def test_llama_config_full_tokens_8_shards(ctx, alg):
    # BASELINE configs[1] at full size: T=8192, h=4096, V=128256 over 8 shards
    # (V/8 = 16032 rows: ragged vocab tiles), all outputs vs fp64
    T, h, V = 8192, 4096, 128256
    X, W, labels = _synthetic(T, h, V, 21)
    fn = {"alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg]
    out = fn(ctx, vm.TokenBatch(X, labels), vm.shard_weights(W, 8))
    ctx.sync()
    dl, gx, gw = fp64_full_check(out, X, W, labels)
    assert dl <= LOSS_ABS and gx <= GRAD_REL_L2 and gw <= GRAD_REL_L2, (dl, gx, gw)


def test_gemma_config_full_tokens_8_shards(ctx):
    # BASELINE configs[2] at full size: T=4096, h=3584, V=256000, 8 shards
    T, h, V = 4096, 3584, 256000
    X, W, labels = _synthetic(T, h, V, 22)
    out = vm.run_alg2(ctx, vm.TokenBatch(X, labels), vm.shard_weights(W, 8))
    ctx.sync()
    dl, gx, gw = fp64_full_check(out, X, W, labels)
    assert dl <= LOSS_ABS and gx <= GRAD_REL_L2 and gw <= GRAD_REL_L2, (dl, gx, gw)


@pytest.mark.parametrize("nh_logits", [1, 2])
def test_extreme_logit_gap_takes_the_overflow_path(ctx, nh_logits):
    # a row whose first vocab tile is ~0 while a later column is 100 nats
    # higher: exp(y - r_i) would overflow, so the row is re-referenced to its
    # max (EpiLogitStats kMaxRefGap path); results must still match the oracle
    T, h, V = 64, 64, 1024
    rng = np.random.default_rng(5)
    X = rng.standard_normal((T, h)) * 0.1
    W = rng.standard_normal((V, h)) * 0.01
    X[3, :] = 1.0
    W[700, :] = 100.0 / h      # logit(3, 700) ~ 100, tile 0 of row 3 ~ 0
    W[900, :] = -100.0 / h
    X[7, :] = -1.0             # row 7: column 900 is the outlier
    g = rng.integers(0, V, T)
    g[3], g[7] = 5, 900
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb)
    # 256- or 512-wide logits tiles change which tiles see the row reference
    # (and which sit > 87 nats below it: underflowed exp-sums)
    tctx = vm.Context(0)
    tctx.set_option("nh_logits", nh_logits)
    for alg in ALGS:
        for p in (1, 2):
            res, _ = run_device(tctx, alg, batch, Wd, p, h)
            assert_parity(res, ref, f"gap {alg} p={p} nh={nh_logits}")
    tctx.close()


def test_nccl_exchange_path_with_a_one_rank_group(ctx):
    # Every NCCL call site of the library (stats all-gather, dX / loss
    # all-reduce, naive max/sum all-reduces) exercised on the one GPU through
    # a 1-rank communicator; results must equal the single-device path.
    X, W, g = oracle.random_instance(96, 64, 512, 4)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    shards = vm.shard_weights(Wd, 1)
    nctx = vm.Context(0)
    nctx.comm_init(1, 0, vm.Context.unique_id())
    nctx.set_option("force_collectives", 1)
    assert nctx.comm_info() == (1, 0)
    cases = [(alg, True) for alg in ALGS] + [("alg2", False)]
    for alg, overlap in cases:
        # alg2 forks its C1 all-reduces onto the comm stream beside pass T (overlap_c1)
        nctx.set_option("overlap_c1", int(overlap))
        fn = {"naive": vm.run_naive, "alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg]
        a = fn(ctx, batch, shards)
        b = fn(nctx, batch, shards)
        nctx.sync()
        ctx.sync()
        for x, y in ((a.loss, b.loss), (a.grad_x, b.grad_x), (a.grad_w_full(), b.grad_w_full()),
                     (a.stats.m, b.stats.m), (a.stats.sum, b.stats.sum)):
            assert torch.allclose(x, y, rtol=1e-6, atol=1e-7), alg
    # alg1 and alg2 (x2) went through the fused exchange (peer buffers mapped
    # over the NCCL group, loss all-reduce as the barrier, copy-engine gather)
    assert nctx.fused_c1_count == 3
    t = torch.arange(16, dtype=torch.float32, device="cuda")
    vm.allreduce_sum(nctx, t)
    nctx.sync()
    assert torch.equal(t, torch.arange(16, dtype=torch.float32, device="cuda"))
    nctx.close()


def test_fused_exchange_in_a_cuda_graph_over_nccl():
    # the fused exchange's NCCL call sites (peer-pointer exchange, loss
    # all-reduce as the barrier) and copy-engine gather captured into a CUDA
    # graph on a 1-rank NCCL group; replays on new inputs equal eager runs
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        X, W, g = oracle.random_instance(256, 128, 1024, 8)
        _, _, batch, Wd = device_case(X, W, g)
        shards = vm.shard_weights(Wd, 1)
        nctx = vm.Context(0)
        nctx.comm_init(1, 0, vm.Context.unique_id())
        nctx.set_option("force_collectives", 1)
        states = [vm.ShardState(nctx, 256, 128, shards[0].rows())]
        outs = vm._alloc_outputs(nctx, batch, shards)
        vm.run_alg2(nctx, batch, shards, states=states, outputs=outs)  # sizes workspace + peer buffers
        nctx.sync()
        graph = vm.capture(nctx, lambda: vm.run_alg2(nctx, batch, shards, states=states, outputs=outs))
        ectx = vm.Context(0)
        for seed in (9, 10):
            X2, Wn, g2 = oracle.random_instance(256, 128, 1024, seed)
            Xb2, _, b2, _ = device_case(X2, W, g2)
            batch.X.copy_(b2.X)
            batch.labels.copy_(b2.labels)
            graph.launch()
            nctx.sync()
            got = [outs[0].clone(), outs[1].clone(), torch.cat(outs[2]).clone()]
            again = vm.run_alg2(nctx, batch, shards)  # eager, same context: the same bits
            nctx.sync()
            assert torch.equal(got[0], again.loss) and torch.equal(got[1], again.grad_x)
            assert torch.equal(got[2], again.grad_w_full())
            ref = oracle.oracle_output_layer(Xb2, g2, device_case(X, W, g)[1], want_softmax=False)
            res = {"loss": got[0].double().cpu().numpy(), "grad_x": got[1].double().cpu().numpy(),
                   "grad_w": got[2].double().cpu().numpy()}
            assert_parity(res, ref, f"graph replay seed {seed}")
        assert nctx.fused_c1_count == 4  # counted on the host: sizing run, captured call, two eager checks
        graph.close()
        ectx.close()
        nctx.close()


def test_tied_embeddings_accumulate_into_one_shard_gradient(ctx):
    # Tied input/output embeddings on the same shard (R/PAPER.md:333): the
    # output layer's dW_k and the input layer's dE_k land in ONE fp32 buffer
    # (accumulate_grad_w + input_backward(accumulate=True)); also gradient
    # accumulation over two microbatches.
    X, W, g = oracle.random_instance(48, 32, 256, 6)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    toks = torch.from_numpy(np.asarray(g[::-1].copy(), np.int64)).cuda()
    grad_in = torch.randn(48, 32, device="cuda").to(torch.bfloat16)
    shards = vm.shard_weights(Wd, 2)
    ref_out = vm.run_alg2(ctx, batch, shards)
    ref_in = [vm.input_backward(ctx, grad_in, toks, s) for s in shards]
    actx = vm.Context(0)
    actx.set_option("accumulate_grad_w", 1)
    bufs = [torch.zeros(s.rows(), 32, dtype=torch.float32, device="cuda") for s in shards]
    outs = vm._alloc_outputs(actx, batch, shards)
    outs = (outs[0], outs[1], bufs, outs[3])
    for _ in range(2):  # two microbatches into the same buffers
        vm.run_alg2(actx, batch, shards, outputs=outs)
    for s, b in zip(shards, bufs):
        vm.input_backward(actx, grad_in, toks, s, out=b, accumulate=True)
    actx.sync()
    for k in range(2):
        want = 2 * ref_out.grad_w[k] + ref_in[k]
        assert torch.allclose(bufs[k], want, rtol=1e-4, atol=1e-5), k
    actx.close()


@pytest.mark.parametrize("rows", [96, 200, 256, 300, 512, 520, 768, 1000])
def test_shard_widths_around_the_512_wide_tile(ctx, rows):
    # 256x512 pair tiles: a shard whose width leaves the last tile's second
    # 256-column half wholly past the shard (rows mod 512 in (0, 256]) must not
    # touch that half's stats slots (the smoke() instance: 96 tokens, h=64,
    # V=512 over 2 shards, U[-1,1] operands).
    for seed in (0, 1):
        X, W, g = oracle.random_instance(96, 64, 2 * rows, seed)
        Xb, Wb, batch, Wd = device_case(X, W, g)
        ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
        for alg in ALGS:
            res, _ = run_device(ctx, alg, batch, Wd, 2, 64, with_softmax=False)
            assert_parity(res, ref, f"rows={rows} seed={seed} {alg}")


def test_memcheck_of_a_ragged_alg2_step():
    # compute-sanitizer memcheck over one ragged alg2 step + the input layer:
    # no out-of-bounds global access from any kernel (tcgen05 GEMM epilogues,
    # stats, scatter).
    import os
    import shutil
    import subprocess
    import sys
    san = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(san):
        pytest.skip("compute-sanitizer not found")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import numpy as np, torch, oracle\n"
        "from paper_2411_05288_b200 import vocab_math as vm\n"
        "ctx = vm.Context(0)\n"
        "X, W, g = oracle.random_instance(96, 64, 600, 0)\n"
        "Xd = torch.from_numpy(X.astype(np.float32)).to(torch.bfloat16).cuda()\n"
        "Wd = torch.from_numpy(W.astype(np.float32)).to(torch.bfloat16).cuda()\n"
        "b = vm.TokenBatch(Xd, torch.from_numpy(g).cuda())\n"
        "for fn in (vm.run_alg2, vm.run_alg1, vm.run_naive):\n"
        "    fn(ctx, b, vm.shard_weights(Wd, 2))\n"
        "s = vm.shard_weights(Wd, 3)[1]\n"
        "vm.input_forward(ctx, b.labels, s); vm.input_backward(ctx, Xd, b.labels, s)\n"
        "ctx.sync(); ctx.close(); print('memcheck-run-ok')\n" % (root, os.path.join(root, "oracle")))
    r = subprocess.run([san, "--tool", "memcheck", "--error-exitcode", "7", sys.executable, "-c", script],
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "memcheck-run-ok" in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]


@pytest.mark.parametrize("splits,ws", [(1, 1), (2, 0), (3, 0), (4, 0), (2, 2), (3, 2), (7, 2), (16, 2), (0, 1)])
def test_split_k_dx_dw_is_exact_to_tolerance_and_deterministic(splits, ws):
    # The dX / A GEMM (K = V_k) may be split over K (option splits_dx), either
    # into ordered in-place partial sums (split_workspace 0) or into concurrent
    # units writing workspace slices summed by k_split_reduce (2 = forced,
    # 1 = auto below half a wave); every setting must meet the parity bar and
    # give identical bits on a re-run.
    X, W, g = oracle.random_instance(300, 256, 6000, 12)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
    sctx = vm.Context(0)
    sctx.set_option("splits_dx", splits)
    sctx.set_option("splits_dw", splits)
    sctx.set_option("split_workspace", ws)
    for alg in ALGS:
        res, out = run_device(sctx, alg, batch, Wd, 2, 256, with_softmax=False)
        assert_parity(res, ref, f"splits={splits} ws={ws} {alg}")
        _, again = run_device(sctx, alg, batch, Wd, 2, 256, with_softmax=False)
        assert torch.equal(out.grad_x, again.grad_x), alg
        assert torch.equal(out.grad_w_full(), again.grad_w_full()), alg
    sctx.close()


def test_gemm_schedule_options_do_not_change_results(ctx):
    # wave lockstep, split-K choice and store boxes change only timing / the
    # fixed accumulation order of split units; every setting must reproduce
    # the default bits (lockstep) or the oracle (splits)
    X, W, g = oracle.random_instance(2048, 1024, 64000, 8)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    base, bout = run_device(ctx, "alg2", batch, Wd, 1, 1024, with_softmax=False)
    # the default schedule itself against the fp64 restatement (every entry)
    dl, gx, gw = fp64_full_check(bout, batch.X, Wd, batch.labels)
    assert dl <= LOSS_ABS and gx <= GRAD_REL_L2 and gw <= GRAD_REL_L2, (dl, gx, gw)
    for opts in ({"lockstep_dx": 0, "lockstep_dw": 0}, {"lockstep_logits": 8, "lockstep_dx": 2, "lockstep_dw": 32},
                 {"store_evict_first": 1}):
        octx = vm.Context(0)
        for k, v in opts.items():
            octx.set_option(k, v)
        res, _ = run_device(octx, "alg2", batch, Wd, 1, 1024, with_softmax=False)
        for key in ("loss", "grad_x", "grad_w"):
            assert np.array_equal(res[key], base[key]), (opts, key)
        octx.close()
    vm.Context(0).set_option("store_evict_first", 0)  # process-wide option: restore
    # other tile shapes: 256 x 256 pair tiles, with and without 4-CTA clusters
    # sharing B by TMA multicast (different split-K choices: tolerance, not bits)
    for opts in ({"nh_logits": 1, "nh_dx": 1, "nh_dw": 1}, {"nh_logits": 1, "nh_dx": 1, "nh_dw": 1, "multicast": 2}):
        octx = vm.Context(0)
        for k, v in opts.items():
            octx.set_option(k, v)
        _, out = run_device(octx, "alg2", batch, Wd, 1, 1024, with_softmax=False)
        dl, gx, gw = fp64_full_check(out, batch.X, Wd, batch.labels)
        assert dl <= LOSS_ABS and gx <= GRAD_REL_L2 and gw <= GRAD_REL_L2, (opts, dl, gx, gw)
        octx.close()


@pytest.mark.parametrize("T", [1, 3, 129])
def test_tiny_and_ragged_token_counts(ctx, T):
    # one token, a few tokens, one past a 128-row block: every GEMM has a
    # single partial M tile (and the wave lockstep / split machinery sees one wave)
    X, W, g = oracle.random_instance(T, 64, 600, 17)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    ref = oracle.oracle_output_layer(Xb, g, Wb)
    for alg in ALGS:
        for p in (1, 2):
            res, _ = run_device(ctx, alg, batch, Wd, p, 64)
            assert_parity(res, ref, f"T={T} {alg} p={p}")


def test_logit_shift_hook_is_invariant_and_matches_the_oracle(ctx):
    # test_vocab_math.cpp:74-84 against the drop-in: the shift is added per row
    # inside the K1 epilogue (vp_ctx_set_logit_shift)
    X, W, g = oracle.random_instance(5, 3, 6, 7)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    shift = np.array([3.0, -40.0, 0.5, 17.0, -2.25])
    base = vm.oracle_output_layer(ctx, batch, Wd, with_softmax=True)
    shifted = vm.oracle_output_layer(ctx, batch, Wd, torch.tensor(shift, dtype=torch.float32, device="cuda"),
                                     with_softmax=True)
    ctx.sync()
    assert (shifted.softmax - base.softmax).abs().max().item() < 4e-3
    assert (shifted.loss - base.loss).abs().max().item() < 1e-3
    assert rel_l2(shifted.grad_x[:, :3].cpu().numpy(), base.grad_x[:, :3].cpu().numpy()) < 1e-2
    ref = oracle.oracle_output_layer(Xb, g, Wb, logit_shift=shift)
    res = {"loss": shifted.loss.double().cpu().numpy(), "grad_x": shifted.grad_x[:, :3].double().cpu().numpy(),
           "grad_w": shifted.grad_w_full()[:, :3].double().cpu().numpy(),
           "softmax": shifted.softmax.double().cpu().numpy()}
    assert_parity(res, ref, "logit_shift")
    # a large shift on the headline-style path (h = 512, V = 4096, 4 tiles / row)
    X, W, g = oracle.random_instance(64, 512, 4096, 8)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    shift = np.linspace(-60.0, 60.0, 64)
    out = vm.oracle_output_layer(ctx, batch, Wd, torch.tensor(shift, dtype=torch.float32, device="cuda"))
    ctx.sync()
    ref = oracle.oracle_output_layer(Xb, g, Wb, logit_shift=shift, want_softmax=False)
    assert_parity({"loss": out.loss.double().cpu().numpy(), "grad_x": out.grad_x.double().cpu().numpy(),
                   "grad_w": out.grad_w_full().double().cpu().numpy()}, ref, "logit_shift h=512")


def test_shard_state_Y_and_B_on_demand(ctx):
    X, W, g = oracle.random_instance(33, 48, 300, 12)
    Xb, Wb, batch, Wd = device_case(X, W, g)
    shards = vm.shard_weights(Wd, 3)
    for s in shards:
        Y = vm.shard_logits(ctx, batch, s)
        B = vm.shard_label_rows(ctx, batch, s)
        ctx.sync()
        Yref = Xb @ Wb[s.row_begin:s.row_end].T
        assert np.abs(Y.double().cpu().numpy() - Yref).max() < 1e-4
        Bref = np.zeros_like(Xb)
        own = (g >= s.row_begin) & (g < s.row_end)
        Bref[own] = Wb[g[own]]
        assert np.array_equal(B.double().cpu().numpy(), Bref)
