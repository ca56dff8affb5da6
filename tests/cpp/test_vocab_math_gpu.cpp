// The reference's unit tests (/root/reference/proj/tests/test_vocab_math.cpp)
// restated against the drop-in C++ API (include/vpipe/vocab_math.hpp) on the
// B200 path.  Tolerances are the north_star's bf16 ones (loss 1e-3 abs,
// gradients 1e-2 rel-L2, softmax 4e-3 abs); cases that only make sense in
// fp64 (finite differences, 1e-14 closed forms) live in tests/test_oracle.py.
// Prints one [PASS]/[FAIL] line per check; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

#include "vpipe/vocab_math.hpp"

using namespace vpipe;

// The independent checker: the fp64 CPU oracle (oracle/liboracle.so, test
// infrastructure) on the bf16-rounded operands the device computes with.
extern "C" int or_oracle_output_layer(const double* X, const double* W, const int64_t* labels, int64_t n_tok,
                                      int64_t h, int64_t V, const double* logit_shift, double* softmax,
                                      double* loss, double* gx, double* gw);

static double bf16_round(double v) {  // double -> float -> bf16 (RNE), as the drop-in uploads
  float f = float(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

static Matrix rounded(const Matrix& M) {
  Matrix r(M.rows(), M.cols());
  for (int64_t i = 0; i < M.size(); ++i) r.data()[i] = bf16_round(M.data()[i]);
  return r;
}

static OutputResult cpu_oracle(const TokenBatch& batch, const Matrix& W, const Vector* shift = nullptr) {
  const int64_t n = batch.X.rows(), h = batch.X.cols(), V = W.rows();
  const Matrix Xb = rounded(batch.X), Wb = rounded(W);
  OutputResult r;
  r.softmax.resize(n, V);
  r.loss.resize(n);
  r.grad_x.resize(n, h);
  r.grad_w.resize(V, h);
  if (or_oracle_output_layer(Xb.data(), Wb.data(), batch.labels.data(), n, h, V, shift ? shift->data() : nullptr,
                             r.softmax.data(), r.loss.data(), r.grad_x.data(), r.grad_w.data()) != 0)
    throw std::runtime_error("cpu oracle failed");
  return r;
}

static int failures = 0;
static void check(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

static double rel_l2(const Matrix& a, const Matrix& b) {
  double num = 0, den = 0;
  for (int64_t i = 0; i < a.size(); ++i) {
    const double d = a.data()[i] - b.data()[i];
    num += d * d;
    den += b.data()[i] * b.data()[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1e-300));
}

static bool close_results(const OutputResult& a, const OutputResult& b) {
  return a.loss.maxAbsDiff(b.loss) <= 1e-3 && a.softmax.maxAbsDiff(b.softmax) <= 4e-3 &&
         rel_l2(a.grad_x, b.grad_x) <= 1e-2 && rel_l2(a.grad_w, b.grad_w) <= 1e-2;
}

int main() {
  {  // test_vocab_math.cpp:23-40 — hand-computable instance
    TokenBatch batch;
    batch.X = Matrix::Ones(2, 1);
    Matrix W(2, 1);
    W(0, 0) = 0.0;
    W(1, 0) = std::log(2.0);
    batch.labels = {1, 0};
    const OutputResult r = oracle_output_layer(batch, W);
    // bf16(ln 2) = 0.69140625: softmax row 0 = (1, e^{w}) / (1 + e^{w})
    const double w = 0.69140625, e = std::exp(w);
    check(std::fabs(r.softmax(0, 0) - 1.0 / (1.0 + e)) < 4e-3 && std::fabs(r.softmax(0, 1) - e / (1.0 + e)) < 4e-3,
          "hand instance softmax");
    check(std::fabs(r.loss(0) - std::log1p(1.0 / e)) < 1e-3 && std::fabs(r.loss(1) - std::log1p(e)) < 1e-3,
          "hand instance loss");
    check(std::fabs(r.grad_x(0, 0) - (e / (1.0 + e) - 1.0) * w) < 1e-3, "hand instance grad_x");
  }
  {  // test_vocab_math.cpp:74-84 — per-row logit shift invariance (K1 epilogue hook)
    const RandomInstance inst = random_instance(5, 3, 6, 7);
    const OutputResult base = oracle_output_layer(inst.batch, inst.W);
    Vector shift(5);
    shift(0) = 3.0;
    shift(1) = -40.0;
    shift(2) = 0.5;
    shift(3) = 17.0;
    shift(4) = -2.25;
    const OutputResult shifted = oracle_output_layer(inst.batch, inst.W, &shift);
    check(shifted.softmax.maxAbsDiff(base.softmax) < 4e-3 && shifted.loss.maxAbsDiff(base.loss) < 1e-3 &&
              rel_l2(shifted.grad_x, base.grad_x) < 1e-2,
          "logit_shift: softmax / loss / grad_x invariant under per-row shifts");
    check(close_results(shifted, cpu_oracle(inst.batch, inst.W, &shift)), "logit_shift: device == CPU oracle");
  }
  {  // ShardState::Y and ::B (VM.hpp:35, :41) materialised on demand
    const RandomInstance inst = random_instance(9, 16, 24, 5);
    const auto shards = shard_weights(inst.W, 3);
    const ShardState st = alg2_pass_S(inst.batch, shards[1]);
    const Matrix Y = st.Y(), B = st.B();
    const Matrix Xb = rounded(inst.batch.X), Wb = rounded(inst.W);
    double ye = 0, be = 0;
    for (int64_t i = 0; i < 9; ++i) {
      for (int64_t v = 0; v < shards[1].rows(); ++v) {
        double y = 0;
        for (int64_t j = 0; j < 16; ++j) y += Xb(i, j) * Wb(shards[1].row_begin + v, j);
        ye = std::max(ye, std::fabs(Y(i, v) - y));
      }
      const int64_t g = inst.batch.labels[size_t(i)];
      for (int64_t j = 0; j < 16; ++j) be = std::max(be, std::fabs(B(i, j) - (shards[1].owns(g) ? Wb(g, j) : 0.0)));
    }
    check(Y.rows() == 9 && Y.cols() == 8 && ye < 1e-4, "ShardState::Y == X W_k^T (fp32 logits)");
    check(B.rows() == 9 && B.cols() == 16 && be == 0.0, "ShardState::B == G_k W_k (owned label rows)");
  }
  {  // the drop-in's monolithic layer against the independent CPU oracle
    const RandomInstance inst = random_instance(24, 40, 72, 11);
    check(close_results(oracle_output_layer(inst.batch, inst.W), cpu_oracle(inst.batch, inst.W)),
          "oracle_output_layer (device, p = 1) == CPU oracle");
  }
  {  // p ranks on one GPU through the loopback backend (Placement::Loopback):
     // the library's multi-rank paths, one context + host thread per shard
    const RandomInstance inst = random_instance(16, 24, 64, 21);
    const OutputResult ref = cpu_oracle(inst.batch, inst.W);
    set_placement(Placement::Loopback);
    bool ok = true;
    for (int p : {2, 4}) {
      ok = ok && close_results(run_naive(inst.batch, inst.W, p), ref);
      ok = ok && close_results(run_alg1(inst.batch, inst.W, p), ref);
      ok = ok && close_results(run_alg2(inst.batch, inst.W, p), ref);
    }
    set_placement(Placement::Auto);
    check(ok, "Placement::Loopback: naive/alg1/alg2 at p = 2, 4 ranks == CPU oracle");
  }
  {  // test_vocab_math.cpp:86-106 — sharded pipelines vs the monolithic layer
    int bad = 0, total = 0;
    for (int64_t b : {1, 2})
      for (int64_t s : {2, 8})
        for (int64_t h : {4, 16})
          for (int64_t V : {16, 64})
            for (int p : {1, 2, 4, 8}) {
              if (V % p) continue;
              for (uint64_t seed : {0u, 1u}) {
                const RandomInstance inst = random_instance(b * s, h, V, seed);
                const OutputResult mono = cpu_oracle(inst.batch, inst.W);
                total += 3;
                bad += !close_results(run_naive(inst.batch, inst.W, p), mono);
                bad += !close_results(run_alg1(inst.batch, inst.W, p), mono);
                bad += !close_results(run_alg2(inst.batch, inst.W, p), mono);
              }
            }
    check(bad == 0, "grid: naive/alg1/alg2 at p shards match the CPU oracle (" + std::to_string(total) +
                        " runs, " + std::to_string(bad) + " off)");
  }
  {  // test_vocab_math.cpp:108-114 — fault injection is detected
    const RandomInstance inst = random_instance(8, 4, 16, 3);
    const OutputResult mono = cpu_oracle(inst.batch, inst.W);
    check(!close_results(run_alg1(inst.batch, inst.W, 4, 1.01), mono), "alg1 fault_scale 1.01 detected");
    check(!close_results(run_alg2(inst.batch, inst.W, 4, 1.01), mono), "alg2 fault_scale 1.01 detected");
  }
  {  // test_vocab_math.cpp:116-151 — online merge on the device
    const RandomInstance inst = random_instance(7, 3, 12, 9);
    const auto shards = shard_weights(inst.W, 4);
    std::vector<LocalStats> parts;
    for (const auto& shard : shards) {
      const ShardState st = alg1_pass_S(inst.batch.X, shard);
      parts.push_back({st.m_local, st.sum_local});
    }
    const GlobalStats fwd = merge_max_sum(parts);
    std::vector<LocalStats> rev(parts.rbegin(), parts.rend());
    const GlobalStats bwd = merge_max_sum(rev);
    check(fwd.m.maxAbsDiff(bwd.m) == 0.0, "merge: m bit-equal under permutation");
    double rs = 0;
    for (int64_t i = 0; i < fwd.sum.size(); ++i) rs = std::max(rs, std::fabs(fwd.sum(i) - bwd.sum(i)) / fwd.sum(i));
    check(rs < 1e-6, "merge: sum equal under permutation (fp32)");
    const GlobalStats l = merge_max_sum({parts[0], parts[1]}), r = merge_max_sum({parts[2], parts[3]});
    const GlobalStats paired = merge_max_sum({{l.m, l.sum}, {r.m, r.sum}});
    check(paired.m.maxAbsDiff(fwd.m) == 0.0, "merge: m bit-equal under re-bracketing");
    for (const ShardState& st : {alg1_pass_S(inst.batch.X, shards[0])}) {
      const Matrix sm = st.softmax_local();
      double worst = 0;
      for (int64_t i = 0; i < sm.rows(); ++i) {
        double acc = 0;
        for (int64_t j = 0; j < sm.cols(); ++j) acc += sm(i, j);
        worst = std::max(worst, std::fabs(acc - 1.0));
      }
      check(worst < 1e-2, "softmax' rows sum to 1");
    }
  }
  {  // test_vocab_math.cpp:153-164 — frozen merge values
    std::vector<LocalStats> parts(2);
    parts[0].m = Vector::Constant(1, 0.0);
    parts[0].sum = Vector::Constant(1, 1.0);
    parts[1].m = Vector::Constant(1, 1.0);
    parts[1].sum = Vector::Constant(1, 1.0);
    const GlobalStats merged = merge_max_sum(parts);
    check(merged.m(0) == 1.0 && std::fabs(merged.sum(0) - 1.3678794411714423) < 1e-6, "frozen merge values");
  }
  {  // test_vocab_math.cpp:166-189 — input layer composes to the monolithic lookup
    const RandomInstance inst = random_instance(10, 5, 20, 4);
    std::mt19937_64 rng(99);
    std::vector<int64_t> tokens(10);
    for (auto& t : tokens) t = static_cast<int64_t>(rng() % 20);
    const auto shards = shard_weights(inst.W, 4);
    Matrix fwd = Matrix::Zero(10, 5), bwd = Matrix::Zero(20, 5);
    for (const auto& shard : shards) {
      const Matrix f = input_forward(tokens, shard);
      for (int64_t i = 0; i < f.size(); ++i) fwd.data()[i] += f.data()[i];
      const Matrix g = input_backward(inst.batch.X, tokens, shard);
      for (int64_t i = 0; i < g.rows(); ++i)
        for (int64_t j = 0; j < 5; ++j) bwd(shard.row_begin + i, j) += g(i, j);
    }
    double fe = 0, be = 0;
    Matrix bref = Matrix::Zero(20, 5);
    for (int i = 0; i < 10; ++i)
      for (int j = 0; j < 5; ++j) {
        float w = float(inst.W(tokens[size_t(i)], j));  // bf16 (RNE) of the fp64 weight
        uint32_t u;
        std::memcpy(&u, &w, 4);
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
        std::memcpy(&w, &u, 4);
        fe = std::max(fe, std::fabs(fwd(i, j) - w));
        bref(tokens[size_t(i)], j) += inst.batch.X(i, j);
      }
    be = bwd.maxAbsDiff(bref);
    check(fe == 0.0, "input forward composes exactly");
    check(be < 1e-6, "input backward composes (fp32 accumulation)");
    bool threw = false;
    try {
      input_forward(std::vector<int64_t>{0, -1}, shards[0]);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "input_forward: token out of range";
    }
    check(threw, "input_forward rejects negative tokens with the reference message");
  }
  {  // test_vocab_math.cpp:191-205 — shard_weights partitions exactly
    const RandomInstance inst = random_instance(2, 3, 12, 0);
    const auto shards = shard_weights(inst.W, 3);
    bool ok = shards.size() == 3;
    int64_t next = 0;
    for (const auto& shard : shards) {
      ok = ok && shard.row_begin == next && shard.rows() == 4 &&
           shard.W.maxAbsDiff(inst.W.middleRows(shard.row_begin, 4)) == 0.0;
      next = shard.row_end;
    }
    bool threw = false;
    try {
      shard_weights(inst.W, 5);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(ok && next == 12 && threw, "shard_weights partitions rows exactly and rejects indivisible V");
  }
  {  // test_vocab_math.cpp:207-216 — random_instance determinism
    const RandomInstance a = random_instance(4, 3, 8, 42), b = random_instance(4, 3, 8, 42),
                         c = random_instance(4, 3, 8, 43);
    check(a.batch.X.maxAbsDiff(b.batch.X) == 0.0 && a.W.maxAbsDiff(b.W) == 0.0 && a.batch.labels == b.batch.labels &&
              a.W.maxAbsDiff(c.W) > 0.0,
          "random_instance deterministic per seed");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
