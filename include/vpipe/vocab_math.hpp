// vpipe/vocab_math.hpp — drop-in replacement for the reference header
// /root/reference/proj/include/vpipe/vocab_math.hpp (VM.hpp), B200 edition.
//
// Same namespace, type names, fields, function names, argument order and
// default arguments as VM.hpp:14-140, so the reference's callers
// (tools/vpipe_main.cpp cmd_verify, tests/test_vocab_math.cpp) compile
// against it.  Differences, all forced by the hardware:
//   * Matrix / Vector are small owning host types (Eigen is not a dependency);
//     they expose the subset of the Eigen API the callers use.
//   * The arithmetic runs on a B200 through the C ABI in vpipe_b200.h:
//     operands are rounded to bf16, accumulation and softmax statistics are
//     fp32.  Results match the fp64 reference within the north_star
//     tolerances (loss 1e-3 abs, gradients 1e-2 rel-L2), not 1e-10.
//   * ShardState keeps its intermediates on the device; softmax_local and Y
//     are materialised on demand (the device never stores fp32 logits for
//     alg1/alg2 — only P = exp(Y - m_tile) in bf16).
//   * Errors keep the reference's types and messages (std::invalid_argument).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

namespace vpipe {

// Row-major dense double matrix (stands in for Eigen::MatrixXd, VM.hpp:11).
class Matrix {
 public:
  Matrix() = default;
  Matrix(int64_t rows, int64_t cols) : r_(rows), c_(cols), d_(size_t(rows * cols), 0.0) {}
  static Matrix Zero(int64_t rows, int64_t cols) { return Matrix(rows, cols); }
  static Matrix Constant(int64_t rows, int64_t cols, double v) {
    Matrix m(rows, cols);
    for (double& x : m.d_) x = v;
    return m;
  }
  static Matrix Ones(int64_t rows, int64_t cols) { return Constant(rows, cols, 1.0); }
  int64_t rows() const { return r_; }
  int64_t cols() const { return c_; }
  int64_t size() const { return r_ * c_; }
  void resize(int64_t rows, int64_t cols) {
    r_ = rows;
    c_ = cols;
    d_.assign(size_t(rows * cols), 0.0);
  }
  double& operator()(int64_t i, int64_t j) { return d_[size_t(i * c_ + j)]; }
  double operator()(int64_t i, int64_t j) const { return d_[size_t(i * c_ + j)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double* row_ptr(int64_t i) { return d_.data() + i * c_; }
  const double* row_ptr(int64_t i) const { return d_.data() + i * c_; }
  // Copy of rows [start, start + n) (Eigen middleRows).
  Matrix middleRows(int64_t start, int64_t n) const;
  // max |a - b| over all entries (Eigen (a-b).cwiseAbs().maxCoeff()).
  double maxAbsDiff(const Matrix& o) const;

 private:
  int64_t r_ = 0, c_ = 0;
  std::vector<double> d_;
};

class Vector {
 public:
  Vector() = default;
  explicit Vector(int64_t n) : d_(size_t(n), 0.0) {}
  static Vector Constant(int64_t n, double v) {
    Vector x(n);
    for (double& e : x.d_) e = v;
    return x;
  }
  static Vector Zero(int64_t n) { return Vector(n); }
  int64_t size() const { return int64_t(d_.size()); }
  void resize(int64_t n) { d_.assign(size_t(n), 0.0); }
  double& operator()(int64_t i) { return d_[size_t(i)]; }
  double operator()(int64_t i) const { return d_[size_t(i)]; }
  double& operator[](int64_t i) { return d_[size_t(i)]; }
  double operator[](int64_t i) const { return d_[size_t(i)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double maxAbsDiff(const Vector& o) const;

 private:
  std::vector<double> d_;
};

namespace detail {
struct DeviceShard;
struct DeviceState;
}  // namespace detail

/// Last transformer layer output plus per-token labels (VM.hpp:15-18).
struct TokenBatch {
  Matrix X;                          // [n_tok x h]
  std::vector<std::int64_t> labels;  // [n_tok], each in [0, V)
};

/// Contiguous row slice of the embedding matrix owned by one device (VM.hpp:21-31).
struct EmbeddingShard {
  Matrix W;  // [V/p x h], rows [row_begin, row_end) of the full W
  int index = 0;
  std::int64_t row_begin = 0;
  std::int64_t row_end = 0;

  std::int64_t rows() const { return row_end - row_begin; }
  bool owns(std::int64_t vocab_row) const { return vocab_row >= row_begin && vocab_row < row_end; }

  // bf16 device copy of W (uploaded on first use, shared by copies).
  mutable std::shared_ptr<detail::DeviceShard> dev;
};

/// One device's local output-layer intermediates (VM.hpp:34-43).
struct ShardState {
  Vector m_local;    // local max per token
  Vector sum_local;  // local exp-sum per token
  bool has_grad_terms = false;

  // Device-resident P = exp(Y - m_tile) (bf16), tile stats and, for alg2,
  // A = softmax'(Y) W_k.  B = G_k W_k is a row gather, never materialised.
  std::shared_ptr<detail::DeviceState> dev;

  // On-demand materialisations of the reference's fields.
  Matrix Y() const;              // local logits [n_tok x V/p] (recomputed: one GEMM)
  Matrix softmax_local() const;  // [n_tok x V/p], rows sum to 1
  Matrix A() const;              // [n_tok x h] (alg2 only)
  Matrix B() const;              // G_k W_k [n_tok x h] (alg2 only)
};

struct GlobalStats {  // VM.hpp:45-48
  Vector m;
  Vector sum;
};

struct OutputResult {  // VM.hpp:51-56
  Matrix softmax;      // [n_tok x V]
  Vector loss;         // per-token cross entropy
  Matrix grad_x;       // [n_tok x h]
  Matrix grad_w;       // [V x h]
};

struct LocalStats {  // VM.hpp:58-61
  Vector m;
  Vector sum;
};

struct ShardGrads {  // VM.hpp:63-66
  Matrix grad_x_partial;
  Matrix grad_w;
};

// Monolithic output layer (VM.hpp:68-74): on the device this is the p = 1
// Algorithm-2 path.  logit_shift (VM.cpp:41-43) is added per row to the
// logits inside the K1 epilogue (vp_ctx_set_logit_shift).
OutputResult oracle_output_layer(const TokenBatch& batch, const Matrix& W, const Vector* logit_shift = nullptr);

std::vector<EmbeddingShard> shard_weights(const Matrix& W, int p);

GlobalStats merge_max_sum(const std::vector<LocalStats>& parts);

OutputResult naive_partitioned_output(const TokenBatch& batch, const std::vector<EmbeddingShard>& shards);

ShardState alg1_pass_S(const Matrix& X, const EmbeddingShard& shard);

ShardGrads alg1_pass_T(const ShardState& state, const GlobalStats& stats, const TokenBatch& batch,
                       const EmbeddingShard& shard);

ShardState alg2_pass_S(const TokenBatch& batch, const EmbeddingShard& shard);

struct BarrierResult {  // VM.hpp:99-102
  GlobalStats stats;
  Matrix grad_x;
};

BarrierResult alg2_barrier_C1(const std::vector<ShardState>& states);

Matrix alg2_pass_T(const ShardState& state, const GlobalStats& stats, const TokenBatch& batch,
                   const EmbeddingShard& shard);

Matrix input_forward(const std::vector<std::int64_t>& tokens, const EmbeddingShard& shard);

Matrix input_backward(const Matrix& grad_out, const std::vector<std::int64_t>& tokens, const EmbeddingShard& shard);

struct RandomInstance {  // VM.hpp:125-128
  TokenBatch batch;
  Matrix W;
};

// Bit-identical to the reference generator (VM.cpp:253-270).
RandomInstance random_instance(std::int64_t n_tok, std::int64_t h, std::int64_t V, std::uint64_t seed);

// Where run_naive / run_alg1 / run_alg2 place their p shards (an extension;
// env VPIPE_PLACEMENT=auto|local|spread|loopback sets the initial value):
//   Local    all p shards on one GPU (VPIPE_DEVICE, default 0), one context;
//   Spread   shard k on GPU k, one context per GPU joined by NCCL, each rank
//            driven from its own host thread (the reference's p devices);
//   Loopback p contexts on one GPU joined by the loopback backend (the
//            multi-rank code paths on a single GPU);
//   Auto     Spread when p <= visible GPUs (and p > 1), else Local.
enum class Placement { Auto, Local, Spread, Loopback };
void set_placement(Placement p);
Placement placement();

OutputResult run_naive(const TokenBatch& batch, const Matrix& W, int p);
OutputResult run_alg1(const TokenBatch& batch, const Matrix& W, int p, double fault_scale = 1.0);
OutputResult run_alg2(const TokenBatch& batch, const Matrix& W, int p, double fault_scale = 1.0);

// cost_model.cpp:49-55 — pad V to a multiple of 2p (used by `verify`).
std::int64_t pad_vocab_size(std::int64_t V, std::int64_t p);

}  // namespace vpipe
