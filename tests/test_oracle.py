"""CPU oracle pinned against the reference's own tests (no GPU).

Each test restates one case of /root/reference/proj/tests/test_vocab_math.cpp
(or acceptance.cpp criteria 1-2 / SPEC.md examples) against oracle/liboracle.so
and the fixtures in tests/golden/golden.json.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle  # oracle/oracle.py (test infrastructure)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def max_abs_diff(a, b):
    return max(np.abs(a.softmax - b.softmax).max(), np.abs(a.loss - b.loss).max(),
               np.abs(a.grad_x - b.grad_x).max(), np.abs(a.grad_w - b.grad_w).max())


def test_random_instance_matches_independent_generator():
    # golden.json was produced by a pure-Python mt19937_64 + libstdc++ distributions
    for ri in GOLD["random_instances"]:
        X, W, g = oracle.random_instance(ri["n_tok"], ri["h"], ri["V"], ri["seed"])
        Xg = np.array([[float.fromhex(v) for v in r] for r in ri["X_hex"]])
        Wg = np.array([[float.fromhex(v) for v in r] for r in ri["W_hex"]])
        assert np.array_equal(X, Xg) and np.array_equal(W, Wg)
        assert list(g) == ri["labels"]


def test_random_instance_is_deterministic_per_seed():
    # test_vocab_math.cpp:207-216
    a = oracle.random_instance(4, 3, 8, 42)
    b = oracle.random_instance(4, 3, 8, 42)
    c = oracle.random_instance(4, 3, 8, 43)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert np.abs(a[1] - c[1]).max() > 0


def test_oracle_hand_computable_instance():
    # test_vocab_math.cpp:23-40
    k = GOLD["hand_instance"]
    r = oracle.oracle_output_layer(np.array(k["X"]), k["labels"], np.array(k["W"]))
    assert r.softmax[0] == pytest.approx(k["softmax_row0"], rel=k["tol"])
    assert r.loss == pytest.approx(k["loss"], rel=k["tol"])
    assert r.grad_x[0, 0] == pytest.approx(k["grad_x_00"], rel=k["tol"])


def test_oracle_spec_kat():
    # SPEC.md:125
    k = GOLD["spec_kat"]
    r = oracle.oracle_output_layer(np.array(k["X"]), k["labels"], np.array(k["W"]))
    assert np.abs(r.softmax - np.array(k["softmax"])).max() < k["tol"]
    assert np.abs(r.loss - np.array(k["loss"])).max() < k["tol"]
    assert np.abs(r.grad_x - np.array(k["grad_x"])).max() < k["tol"]


@pytest.mark.parametrize("seed", GOLD["finite_differences"]["seeds"])
def test_oracle_gradients_match_central_finite_differences(seed):
    # test_vocab_math.cpp:42-72 (seed 12345) and acceptance.cpp:90-122 (seed 0)
    fd = GOLD["finite_differences"]
    X, W, g = oracle.random_instance(fd["n_tok"], fd["h"], fd["V"], seed)
    base = oracle.oracle_output_layer(X, g, W)
    step = fd["step"]

    def total(Xv, Wv):
        return oracle.oracle_output_layer(Xv, g, Wv, want_softmax=False).loss.sum()

    worst = 0.0
    for i in range(X.shape[0]):
        for j in range(X.shape[1]):
            xp, xm = X.copy(), X.copy()
            xp[i, j] += step
            xm[i, j] -= step
            d = (total(xp, W) - total(xm, W)) / (2 * step)
            worst = max(worst, abs(base.grad_x[i, j] - d) / (abs(d) + 1.0))
    for i in range(W.shape[0]):
        for j in range(W.shape[1]):
            wp, wm = W.copy(), W.copy()
            wp[i, j] += step
            wm[i, j] -= step
            d = (total(X, wp) - total(X, wm)) / (2 * step)
            worst = max(worst, abs(base.grad_w[i, j] - d) / (abs(d) + 1.0))
    assert worst <= fd["rel_tol"]


def test_oracle_is_invariant_under_per_row_logit_shifts():
    # test_vocab_math.cpp:74-84
    X, W, g = oracle.random_instance(5, 3, 6, 7)
    base = oracle.oracle_output_layer(X, g, W)
    shifted = oracle.oracle_output_layer(X, g, W, logit_shift=np.array([3.0, -40.0, 0.5, 17.0, -2.25]))
    assert np.abs(shifted.softmax - base.softmax).max() < 1e-12
    assert np.abs(shifted.loss - base.loss).max() < 1e-11
    assert np.abs(shifted.grad_x - base.grad_x).max() < 1e-12


def test_sharded_pipelines_match_the_oracle_across_the_grid():
    # test_vocab_math.cpp:86-106 and acceptance.cpp criterion 1 (<= 1e-10)
    gr = GOLD["grid"]
    worst = 0.0
    for b in gr["b"]:
        for s in gr["s"]:
            for h in gr["h"]:
                for V in gr["V"]:
                    for p in gr["p"]:
                        if V % p:
                            continue
                        for seed in gr["seeds"]:
                            X, W, g = oracle.random_instance(b * s, h, V, seed)
                            ref = oracle.oracle_output_layer(X, g, W)
                            for alg in ("naive", "alg1", "alg2"):
                                worst = max(worst, max_abs_diff(oracle.run(alg, X, g, W, p), ref))
    assert worst <= gr["tol"]


def test_corrupting_the_correction_factor_is_detected():
    # test_vocab_math.cpp:108-114
    X, W, g = oracle.random_instance(8, 4, 16, 3)
    ref = oracle.oracle_output_layer(X, g, W)
    assert max_abs_diff(oracle.run("alg1", X, g, W, 4, 1.01), ref) > 1e-6
    assert max_abs_diff(oracle.run("alg2", X, g, W, 4, 1.01), ref) > 1e-6


def _parts():
    X, W, g = oracle.random_instance(7, 3, 12, 9)
    return X, W, [oracle.local_stats(X, W, 4, k) for k in range(4)]


def test_online_merge_equals_the_monolithic_stats():
    # test_vocab_math.cpp:116-136
    X, W, parts = _parts()
    m, s = oracle.merge_max_sum([p[0] for p in parts], [p[1] for p in parts])
    Y = X @ W.T
    mm = Y.max(axis=1)
    ss = np.exp(Y - mm[:, None]).sum(axis=1)
    assert m == pytest.approx(mm, rel=1e-14)
    assert s == pytest.approx(ss, rel=1e-13)


def test_online_merge_invariant_under_permutation_and_rebracketing():
    # test_vocab_math.cpp:137-150: m bit-equal, sum within 1e-13
    _, _, parts = _parts()
    ms, ss = [p[0] for p in parts], [p[1] for p in parts]
    fm, fs = oracle.merge_max_sum(ms, ss)
    bm, bs = oracle.merge_max_sum(ms[::-1], ss[::-1])
    assert np.abs(fm - bm).max() == 0.0 and np.abs(fs - bs).max() < 1e-13
    lm, ls = oracle.merge_max_sum(ms[:2], ss[:2])
    rm, rs = oracle.merge_max_sum(ms[2:], ss[2:])
    pm, ps = oracle.merge_max_sum([lm, rm], [ls, rs])
    assert np.abs(pm - fm).max() == 0.0 and np.abs(ps - fs).max() < 1e-13


def test_frozen_merge_values():
    # test_vocab_math.cpp:153-164
    k = GOLD["frozen_merge"]
    m, s = oracle.merge_max_sum([np.array(x) for x in k["m_parts"]], [np.array(x) for x in k["s_parts"]])
    assert m[0] == k["m"]
    assert s[0] == pytest.approx(k["sum"], rel=k["tol"])
    k = GOLD["equal_merge"]
    m, s = oracle.merge_max_sum([np.array(x) for x in k["m_parts"]], [np.array(x) for x in k["s_parts"]])
    assert m[0] == k["m"] and s[0] == k["sum"]


def test_merge_errors():
    with pytest.raises(oracle.OracleError, match="length mismatch"):
        oracle.merge_max_sum([np.zeros(2), np.zeros(3)], [np.zeros(2), np.zeros(3)])


def test_input_layer_shards_compose_to_the_monolithic_lookup():
    # test_vocab_math.cpp:166-189: forward exactly equal, backward < 1e-14
    X, W, _ = oracle.random_instance(10, 5, 20, 4)
    tokens = np.array([v % 20 for v in _mt64_99(10)], dtype=np.int64)
    p, rows = 4, 5
    fwd = np.zeros((10, 5))
    bwd = np.zeros((20, 5))
    for k in range(p):
        fwd += oracle.input_forward(tokens, W[k * rows:(k + 1) * rows], k * rows)
        bwd[k * rows:(k + 1) * rows] += oracle.input_backward(X, tokens, rows, k * rows)
    fwd_ref = W[tokens]
    bwd_ref = np.zeros((20, 5))
    for i, t in enumerate(tokens):
        bwd_ref[t] += X[i]
    assert np.abs(fwd - fwd_ref).max() == 0.0
    assert np.abs(bwd - bwd_ref).max() < 1e-14


def _mt64_99(n):
    # std::mt19937_64(99)() % 20 as in the reference test; use the golden generator
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "make_golden", os.path.join(os.path.dirname(__file__), "golden", "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    rng = mg.MT19937_64(99)
    return [rng() for _ in range(n)]


def test_input_layer_errors_and_unowned_tokens():
    # VM.cpp:232/:247 reject tok < 0 only; tok >= row_end is silently unowned
    W = np.ones((4, 3))
    with pytest.raises(oracle.OracleError, match="input_forward: token out of range"):
        oracle.input_forward(np.array([0, -1]), W, 0)
    with pytest.raises(oracle.OracleError, match="input_backward: token out of range"):
        oracle.input_backward(np.ones((2, 3)), np.array([-3, 0]), 4, 0)
    out = oracle.input_forward(np.array([0, 100]), W, 0)
    assert np.array_equal(out[1], np.zeros(3))


def test_input_backward_f32_is_ascending_i_accumulation():
    rng = np.random.default_rng(0)
    g = rng.standard_normal((64, 8)).astype(np.float32)
    t = rng.integers(0, 6, 64)
    out = oracle.input_backward_f32(g, t, 6, 0)
    ref = np.zeros((6, 8), np.float32)
    for i in range(64):  # the same sequential order, in numpy fp32
        ref[t[i]] = ref[t[i]] + g[i]
    assert np.array_equal(out, ref)


def test_shard_weights_partitions_rows_exactly():
    # test_vocab_math.cpp:191-205
    oracle.shard_check(12, 3)
    with pytest.raises(oracle.OracleError, match="V not divisible by p"):
        oracle.shard_check(12, 5)
    with pytest.raises(oracle.OracleError, match="p must be >= 1"):
        oracle.shard_check(12, 0)


def test_batch_validation_messages():
    # check_batch, VM.cpp:12-20
    W = np.ones((4, 2))
    with pytest.raises(oracle.OracleError, match="label out of range"):
        oracle.oracle_output_layer(np.ones((2, 2)), [0, 4], W)
    with pytest.raises(oracle.OracleError, match="hidden dim mismatch"):
        oracle.oracle_output_layer(np.ones((2, 3)), [0, 1], W)


def test_verify_defaults_pass():
    # vpipe_main.cpp:161-218 with its verify defaults b=2,s=4,h=8,V=32,p=4 (:285-287)
    p, n, h = 4, 8, 8
    V = 32 + (-32) % (2 * p)
    X, W, g = oracle.random_instance(n, h, V, 0)
    ref = oracle.oracle_output_layer(X, g, W)
    for alg in ("naive", "alg1", "alg2"):
        assert max_abs_diff(oracle.run(alg, X, g, W, p), ref) <= 1e-10
    assert max_abs_diff(oracle.run("alg1", X, g, W, p, 1.01), ref) > 1e-10


def test_pad_vocab_size_examples():
    from paper_2411_05288_b200.vocab_math import pad_vocab_size
    for V, p, want in GOLD["pad_vocab"]["cases"]:
        assert pad_vocab_size(V, p) == want
    assert math.isclose(1.0, 1.0)
