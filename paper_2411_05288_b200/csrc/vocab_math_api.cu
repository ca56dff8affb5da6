// C++ mirror of the reference API (include/vpipe/vocab_math.hpp) on top of
// the C ABI (include/vpipe_b200.h).  Host matrices are double; operands go
// to the device as bf16 (hidden dim zero-padded to a multiple of 8, which
// leaves every logit and gradient unchanged), results come back as fp32.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "vpipe/vocab_math.hpp"
#include "vpipe_b200.h"

namespace vpipe {

Matrix Matrix::middleRows(int64_t start, int64_t n) const {
  Matrix m(n, c_);
  if (n > 0) std::memcpy(m.data(), row_ptr(start), sizeof(double) * size_t(n * c_));
  return m;
}

double Matrix::maxAbsDiff(const Matrix& o) const {
  if (o.r_ != r_ || o.c_ != c_) throw std::invalid_argument("Matrix::maxAbsDiff: shape mismatch");
  double m = 0.0;
  for (size_t i = 0; i < d_.size(); ++i) m = std::max(m, std::fabs(d_[i] - o.d_[i]));
  return m;
}

double Vector::maxAbsDiff(const Vector& o) const {
  if (o.size() != size()) throw std::invalid_argument("Vector::maxAbsDiff: size mismatch");
  double m = 0.0;
  for (size_t i = 0; i < d_.size(); ++i) m = std::max(m, std::fabs(d_[i] - o.d_[i]));
  return m;
}

namespace detail {

void check(int rc) {
  if (rc == VP_OK) return;
  if (rc == VP_EINVAL) throw std::invalid_argument(vp_last_error());
  throw std::runtime_error(std::string("vpipe_b200: ") + vp_last_error());
}

void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

// Fault injection for verification tools (env VPIPE_INJECT_K1_FAULT_PPM: the
// pass-S logits of every context this API creates are scaled by 1 + ppm*1e-6).
void configure(vp_ctx_t c) {
  if (const char* f = std::getenv("VPIPE_INJECT_K1_FAULT_PPM"))
    check(vp_ctx_set_option(c, "debug_logit_scale_ppm", std::atoll(f)));
}

int default_device() {
  const char* dev = std::getenv("VPIPE_DEVICE");
  return dev ? std::atoi(dev) : 0;
}

struct Ctx {
  vp_ctx_t c = nullptr;
  Ctx() {
    check(vp_ctx_create(default_device(), &c));
    configure(c);
  }
  ~Ctx() {
    if (c) vp_ctx_destroy(c);
  }
};

// The context of a rank thread of a group run (see run_group), else the
// process-wide single-device context.
thread_local vp_ctx_t t_ctx = nullptr;

vp_ctx_t ctx() {
  if (t_ctx) return t_ctx;
  static Ctx g;
  return g.c;
}

void sync() { check(vp_ctx_sync(ctx())); }

struct DevMem {
  void* p = nullptr;
  explicit DevMem(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 16)); }
  ~DevMem() {
    if (p) cudaFree(p);
  }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
};
using DevPtr = std::shared_ptr<DevMem>;

int64_t pad8(int64_t h) { return (h + 7) / 8 * 8; }

uint16_t to_bf16(double v) {
  const float f = float(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);  // NaN stays NaN
  u += 0x7fffu + ((u >> 16) & 1u);                                         // round to nearest even
  return uint16_t(u >> 16);
}

DevPtr upload_bf16(const Matrix& M, int64_t ld) {
  std::vector<uint16_t> h(size_t(M.rows() * ld), 0);
  for (int64_t i = 0; i < M.rows(); ++i)
    for (int64_t j = 0; j < M.cols(); ++j) h[size_t(i * ld + j)] = to_bf16(M(i, j));
  auto d = std::make_shared<DevMem>(h.size() * 2);
  cuda_check(cudaMemcpy(d->p, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  return d;
}

DevPtr upload_f32(const double* src, int64_t rows, int64_t cols, int64_t ld) {
  std::vector<float> h(size_t(rows * ld), 0.f);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) h[size_t(i * ld + j)] = float(src[i * cols + j]);
  auto d = std::make_shared<DevMem>(h.size() * 4);
  cuda_check(cudaMemcpy(d->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  return d;
}

DevPtr upload_i64(const std::vector<int64_t>& v) {
  auto d = std::make_shared<DevMem>(v.size() * 8);
  if (!v.empty()) cuda_check(cudaMemcpy(d->p, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
  return d;
}

// [rows x cols] slice of a device fp32 [rows x ld] buffer -> host double.
Matrix download_f32(const void* dptr, int64_t rows, int64_t cols, int64_t ld) {
  sync();
  std::vector<float> h(size_t(rows * ld));
  cuda_check(cudaMemcpy(h.data(), dptr, h.size() * 4, cudaMemcpyDeviceToHost));
  Matrix m(rows, cols);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) m(i, j) = h[size_t(i * ld + j)];
  return m;
}

Vector download_vec(const void* dptr, int64_t n) {
  const Matrix m = download_f32(dptr, 1, n, n);
  Vector v(n);
  for (int64_t i = 0; i < n; ++i) v(i) = m(0, i);
  return v;
}

struct DeviceShard {
  DevPtr W;
  int64_t h = 0, ldw = 0;
  int device = -1;
  vp_shard_t desc{};
};

int current_device() {
  int d = 0;
  cuda_check(cudaGetDevice(&d));
  return d;
}

struct DeviceBatch {
  DevPtr X, labels;
  int64_t n_tok = 0, h = 0;
  vp_batch_t desc{};
};

struct DeviceState {
  vp_state_t st = nullptr;
  std::shared_ptr<DeviceShard> shard;
  std::shared_ptr<DeviceBatch> batch;
  int64_t h_true = 0, rows = 0, n_tok = 0;
  ~DeviceState() {
    if (st) vp_state_destroy(st);
  }
};

std::shared_ptr<DeviceShard> device_shard(const EmbeddingShard& s) {
  if (s.dev && s.dev->h == s.W.cols() && s.dev->device == current_device()) return s.dev;
  if (s.W.rows() != s.rows()) throw std::invalid_argument("EmbeddingShard: W rows != row_end - row_begin");
  auto d = std::make_shared<DeviceShard>();
  d->h = s.W.cols();
  d->ldw = pad8(d->h);
  d->W = upload_bf16(s.W, d->ldw);
  d->device = current_device();
  d->desc.W = d->W->p;
  d->desc.ldw = d->ldw;
  d->desc.row_begin = s.row_begin;
  d->desc.row_end = s.row_end;
  d->desc.index = s.index;
  s.dev = d;
  return d;
}

std::shared_ptr<DeviceBatch> device_batch(const Matrix& X, const std::vector<int64_t>* labels) {
  auto b = std::make_shared<DeviceBatch>();
  b->n_tok = X.rows();
  b->h = X.cols();
  const int64_t ld = pad8(b->h);
  b->X = upload_bf16(X, ld);
  if (labels) b->labels = upload_i64(*labels);
  b->desc.X = b->X->p;
  b->desc.ldx = ld;
  b->desc.labels = labels ? static_cast<const int64_t*>(b->labels->p) : nullptr;
  b->desc.n_tok = b->n_tok;
  b->desc.h = ld;
  return b;
}

struct DeviceStats {
  DevPtr m, sum;
  vp_stats_t desc{};
  explicit DeviceStats(int64_t n) : m(std::make_shared<DevMem>(size_t(n) * 4)), sum(std::make_shared<DevMem>(size_t(n) * 4)) {
    desc.m = static_cast<float*>(m->p);
    desc.sum = static_cast<float*>(sum->p);
  }
};

std::shared_ptr<DeviceStats> upload_stats(const GlobalStats& g) {
  auto d = std::make_shared<DeviceStats>(g.m.size());
  d->m = upload_f32(g.m.data(), 1, g.m.size(), g.m.size());
  d->sum = upload_f32(g.sum.data(), 1, g.sum.size(), g.sum.size());
  d->desc.m = static_cast<float*>(d->m->p);
  d->desc.sum = static_cast<float*>(d->sum->p);
  return d;
}

GlobalStats download_stats(const DeviceStats& d, int64_t n) {
  GlobalStats g;
  g.m = download_vec(d.desc.m, n);
  g.sum = download_vec(d.desc.sum, n);
  return g;
}

void check_batch(const TokenBatch& batch, int64_t V) {  // VM.cpp:12-20
  if (batch.X.rows() < 1) throw std::invalid_argument("TokenBatch: empty X");
  if (int64_t(batch.labels.size()) != batch.X.rows())
    throw std::invalid_argument("TokenBatch: labels/X row mismatch");
  for (int64_t g : batch.labels)
    if (g < 0 || g >= V) throw std::invalid_argument("TokenBatch: label out of range");
}

ShardState make_state(const std::shared_ptr<DeviceBatch>& b, const std::shared_ptr<DeviceShard>& s, int64_t h_true,
                      int64_t rows) {
  ShardState out;
  out.dev = std::make_shared<DeviceState>();
  out.dev->shard = s;
  out.dev->batch = b;
  out.dev->h_true = h_true;
  out.dev->rows = rows;
  out.dev->n_tok = b->n_tok;
  check(vp_state_create(ctx(), b->n_tok, b->desc.h, rows, &out.dev->st));
  return out;
}

void fetch_local(ShardState* st) {
  const float *m = nullptr, *s = nullptr;
  check(vp_state_local_stats(st->dev->st, &m, &s));
  st->m_local = download_vec(m, st->dev->n_tok);
  st->sum_local = download_vec(s, st->dev->n_tok);
}

// ---- placement of run_naive / run_alg1 / run_alg2's p shards ---------------
Placement& placement_ref() {
  static Placement p = [] {
    const char* e = std::getenv("VPIPE_PLACEMENT");
    const std::string v = e ? e : "auto";
    if (v == "local") return Placement::Local;
    if (v == "spread") return Placement::Spread;
    if (v == "loopback") return Placement::Loopback;
    return Placement::Auto;
  }();
  return p;
}

int visible_devices() {
  int n = 0;
  cuda_check(cudaGetDeviceCount(&n));
  return n;
}

Placement resolve(int p) {
  const Placement want = placement_ref();
  if (p == 1 || want == Placement::Local) return Placement::Local;
  if (want == Placement::Spread) {
    if (p > visible_devices()) throw std::invalid_argument("placement Spread: p exceeds the visible GPUs");
    return Placement::Spread;
  }
  if (want == Placement::Loopback) return Placement::Loopback;
  return visible_devices() >= p ? Placement::Spread : Placement::Local;  // Auto
}

// p contexts joined into one group (vp_comm_init_all): NCCL when they sit on
// p distinct GPUs, the loopback backend when all share one.  Cached per
// (placement, p): communicator set-up costs far more than a call.
struct Group {
  std::vector<vp_ctx_t> ctxs;
  std::vector<int> devs;
  ~Group() {
    for (vp_ctx_t c : ctxs) vp_ctx_destroy(c);
  }
};

Group& group(Placement pl, int p) {
  static std::mutex mu;
  static auto& cache = *new std::map<std::pair<int, int>, std::unique_ptr<Group>>();  // never destroyed (exit order)
  std::lock_guard<std::mutex> lk(mu);
  auto& g = cache[{int(pl), p}];
  if (!g) {
    auto ng = std::make_unique<Group>();
    for (int k = 0; k < p; ++k) {
      const int dev = pl == Placement::Spread ? k : default_device();
      vp_ctx_t c = nullptr;
      check(vp_ctx_create(dev, &c));
      ng->ctxs.push_back(c);
      ng->devs.push_back(dev);
      configure(c);
    }
    check(vp_comm_init_all(ng->ctxs.data(), p));
    g = std::move(ng);
  }
  return *g;
}

// One rank of a group run: its thread drives ctx on its device.
struct RankScope {
  explicit RankScope(vp_ctx_t c, int dev) {
    t_ctx = c;
    cuda_check(cudaSetDevice(dev));
  }
  ~RankScope() { t_ctx = nullptr; }
};

void download_into_rows(const void* dptr, int64_t rows, int64_t h, int64_t ld, Matrix* dst, int64_t row0) {
  const Matrix g = download_f32(dptr, rows, h, ld);
  std::memcpy(dst->row_ptr(row0), g.data(), sizeof(double) * size_t(rows * h));
}

void download_softmax_cols(vp_state_t st, const vp_stats_t& stats, int64_t n, int64_t rows, int64_t col0,
                           Matrix* dst) {
  DevMem sm(size_t(n * rows) * 4);
  check(vp_shard_softmax(ctx(), st, stats, static_cast<float*>(sm.p), rows));
  const Matrix s = download_f32(sm.p, n, rows, rows);
  for (int64_t i = 0; i < n; ++i) std::memcpy(dst->row_ptr(i) + col0, s.row_ptr(i), sizeof(double) * size_t(rows));
}

int call_driver(int alg, vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* sd, const vp_state_t* st, int n,
                double fault_scale, vp_stats_t stats, float* loss, float* gx, int64_t ldgx, float* const* gw,
                int64_t ldgw) {
  if (alg == 0) return vp_naive_partitioned_output(c, b, sd, st, n, stats, loss, gx, ldgx, gw, ldgw);
  if (alg == 1) return vp_run_alg1(c, b, sd, st, n, fault_scale, stats, loss, gx, ldgx, gw, ldgw);
  return vp_run_alg2(c, b, sd, st, n, fault_scale, stats, loss, gx, ldgx, gw, ldgw);
}

// Full drivers, local placement: every shard on the one device, softmax assembled.
OutputResult run_local(int alg, const TokenBatch& batch, const Matrix& W, int p, double fault_scale) {
  const auto shards = shard_weights(W, p);
  auto b = device_batch(batch.X, &batch.labels);
  const int64_t n = batch.X.rows(), h = batch.X.cols(), ld = b->desc.h;
  std::vector<ShardState> states;
  std::vector<vp_state_t> st;
  std::vector<vp_shard_t> sd;
  std::vector<DevPtr> gw;
  std::vector<float*> gwp;
  for (const auto& s : shards) {
    auto ds = device_shard(s);
    states.push_back(make_state(b, ds, h, s.rows()));
    st.push_back(states.back().dev->st);
    sd.push_back(ds->desc);
    gw.push_back(std::make_shared<DevMem>(size_t(s.rows() * ld) * 4));
    gwp.push_back(static_cast<float*>(gw.back()->p));
  }
  DeviceStats stats(n);
  DevMem loss(size_t(n) * 4), gx(size_t(n * ld) * 4);
  check(call_driver(alg, ctx(), &b->desc, sd.data(), st.data(), p, fault_scale, stats.desc,
                    static_cast<float*>(loss.p), static_cast<float*>(gx.p), ld, gwp.data(), ld));
  OutputResult out;
  out.loss = download_vec(loss.p, n);
  out.grad_x = download_f32(gx.p, n, h, ld);
  out.grad_w.resize(W.rows(), h);
  out.softmax.resize(n, W.rows());
  for (size_t k = 0; k < shards.size(); ++k) {
    download_into_rows(gwp[k], shards[k].rows(), h, ld, &out.grad_w, shards[k].row_begin);
    download_softmax_cols(st[k], stats.desc, n, shards[k].rows(), shards[k].row_begin, &out.softmax);
  }
  return out;
}

// Full drivers, one rank per shard: rank k's thread drives context k of the
// group (its own GPU under Spread, GPU VPIPE_DEVICE under Loopback) with ONE
// shard, so the library's collective paths do the exchanges (stats
// all-gather, dX / loss all-reduce) — the reference's single-process view of
// p devices (VM.hpp:106, :136-140).
OutputResult run_group(int alg, const TokenBatch& batch, const Matrix& W, int p, double fault_scale, Group& g) {
  const auto shards = shard_weights(W, p);
  const int64_t n = batch.X.rows(), h = batch.X.cols();
  OutputResult out;
  out.grad_w.resize(W.rows(), h);
  out.softmax.resize(n, W.rows());
  std::vector<std::exception_ptr> errs(static_cast<size_t>(p));
  std::vector<std::thread> th;
  for (int k = 0; k < p; ++k)
    th.emplace_back([&, k] {
      try {
        RankScope scope(g.ctxs[size_t(k)], g.devs[size_t(k)]);
        auto b = device_batch(batch.X, &batch.labels);
        const int64_t ld = b->desc.h, rows = shards[size_t(k)].rows();
        auto ds = device_shard(shards[size_t(k)]);
        ShardState state = make_state(b, ds, h, rows);
        vp_state_t st = state.dev->st;
        DeviceStats stats(n);
        DevMem loss(size_t(n) * 4), gx(size_t(n * ld) * 4), gw(size_t(rows * ld) * 4);
        float* gwp = static_cast<float*>(gw.p);
        check(call_driver(alg, ctx(), &b->desc, &ds->desc, &st, 1, fault_scale, stats.desc,
                          static_cast<float*>(loss.p), static_cast<float*>(gx.p), ld, &gwp, ld));
        if (k == 0) {  // every rank holds the same loss and grad_x
          out.loss = download_vec(loss.p, n);
          out.grad_x = download_f32(gx.p, n, h, ld);
        }
        download_into_rows(gwp, rows, h, ld, &out.grad_w, shards[size_t(k)].row_begin);
        download_softmax_cols(st, stats.desc, n, rows, shards[size_t(k)].row_begin, &out.softmax);
        sync();
      } catch (...) {
        errs[size_t(k)] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  return out;
}

OutputResult run(int alg, const TokenBatch& batch, const Matrix& W, int p, double fault_scale) {
  if (p < 1) throw std::invalid_argument("shard_weights: p must be >= 1");
  if (W.rows() % p != 0) throw std::invalid_argument("shard_weights: V not divisible by p");
  if (alg == 0) check_batch(batch, W.rows());
  if (batch.X.cols() != W.cols()) throw std::invalid_argument("oracle_output_layer: X/W hidden dim mismatch");
  if (batch.X.rows() < 1) throw std::invalid_argument("TokenBatch: empty X");
  if (int64_t(batch.labels.size()) != batch.X.rows()) throw std::invalid_argument("TokenBatch: labels/X row mismatch");
  const Placement pl = resolve(p);
  if (pl == Placement::Local) return run_local(alg, batch, W, p, fault_scale);
  return run_group(alg, batch, W, p, fault_scale, group(pl, p));
}

}  // namespace detail

using namespace detail;

Matrix ShardState::softmax_local() const {
  if (!dev) throw std::invalid_argument("ShardState: no device state");
  // P is softmax' after pass S; materialise with unit scale.
  const int64_t n = dev->n_tok, rows = dev->rows;
  DeviceStats ones(n);
  std::vector<double> one(size_t(n), 1.0), zero(size_t(n), 0.0);
  const float *m = nullptr, *s = nullptr;
  check(vp_state_local_stats(dev->st, &m, &s));
  // global stats == local stats makes the Eq. 5 factor exactly 1
  cuda_check(cudaMemcpy(ones.desc.m, m, size_t(n) * 4, cudaMemcpyDeviceToDevice));
  cuda_check(cudaMemcpy(ones.desc.sum, s, size_t(n) * 4, cudaMemcpyDeviceToDevice));
  DevMem out(size_t(n * rows) * 4);
  check(vp_shard_softmax(ctx(), dev->st, ones.desc, static_cast<float*>(out.p), rows));
  return download_f32(out.p, n, rows, rows);
}

Matrix ShardState::A() const {
  if (!dev) throw std::invalid_argument("ShardState: no device state");
  const float* a = nullptr;
  int64_t lda = 0;
  check(vp_state_grad_terms(dev->st, &a, &lda));
  return download_f32(a, dev->n_tok, dev->h_true, lda);
}

Matrix ShardState::Y() const {
  if (!dev) throw std::invalid_argument("ShardState: no device state");
  DevMem out(size_t(dev->n_tok * dev->rows) * 4);
  check(vp_shard_logits(ctx(), &dev->batch->desc, &dev->shard->desc, static_cast<float*>(out.p), dev->rows));
  return download_f32(out.p, dev->n_tok, dev->rows, dev->rows);
}

Matrix ShardState::B() const {
  if (!dev) throw std::invalid_argument("ShardState: no device state");
  if (!has_grad_terms) throw std::invalid_argument("alg2_barrier_C1: A/B terms missing");
  if (!dev->batch->desc.labels) throw std::invalid_argument("ShardState: B needs the batch labels");
  const int64_t ld = dev->batch->desc.h;
  DevMem out(size_t(dev->n_tok * ld) * 4);
  check(vp_shard_label_rows(ctx(), &dev->batch->desc, &dev->shard->desc, static_cast<float*>(out.p), ld));
  return download_f32(out.p, dev->n_tok, dev->h_true, ld);
}

void set_placement(Placement p) { placement_ref() = p; }
Placement placement() { return placement_ref(); }

OutputResult oracle_output_layer(const TokenBatch& batch, const Matrix& W, const Vector* logit_shift) {
  check_batch(batch, W.rows());
  if (batch.X.cols() != W.cols()) throw std::invalid_argument("oracle_output_layer: X/W hidden dim mismatch");
  if (logit_shift == nullptr) return run_local(2, batch, W, 1, 1.0);
  // the per-row logit shift hook (VM.cpp:41-43), applied in the K1 epilogue
  if (logit_shift->size() != batch.X.rows()) throw std::invalid_argument("oracle_output_layer: logit_shift size mismatch");
  DevPtr d = upload_f32(logit_shift->data(), 1, logit_shift->size(), logit_shift->size());
  check(vp_ctx_set_logit_shift(ctx(), static_cast<const float*>(d->p)));
  try {
    OutputResult r = run_local(2, batch, W, 1, 1.0);
    check(vp_ctx_set_logit_shift(ctx(), nullptr));
    return r;
  } catch (...) {
    vp_ctx_set_logit_shift(ctx(), nullptr);
    throw;
  }
}

std::vector<EmbeddingShard> shard_weights(const Matrix& W, int p) {  // VM.cpp:65-80
  if (p < 1) throw std::invalid_argument("shard_weights: p must be >= 1");
  const int64_t V = W.rows();
  if (V % p != 0) throw std::invalid_argument("shard_weights: V not divisible by p");
  const int64_t rows = V / p;
  std::vector<EmbeddingShard> shards(static_cast<size_t>(p));
  for (int k = 0; k < p; ++k) {
    shards[size_t(k)].W = W.middleRows(k * rows, rows);
    shards[size_t(k)].index = k;
    shards[size_t(k)].row_begin = k * rows;
    shards[size_t(k)].row_end = (k + 1) * rows;
  }
  return shards;
}

GlobalStats merge_max_sum(const std::vector<LocalStats>& parts) {  // VM.cpp:82-101
  if (parts.empty()) throw std::invalid_argument("merge_max_sum: empty input");
  const int64_t n = parts.front().m.size();
  for (const auto& part : parts)
    if (part.m.size() != n || part.sum.size() != n) throw std::invalid_argument("merge_max_sum: length mismatch");
  const int p = int(parts.size());
  std::vector<double> m(size_t(p * n)), s(size_t(p * n));
  for (int k = 0; k < p; ++k)
    for (int64_t i = 0; i < n; ++i) {
      m[size_t(k * n + i)] = parts[size_t(k)].m(i);
      s[size_t(k * n + i)] = parts[size_t(k)].sum(i);
    }
  DevPtr dm = upload_f32(m.data(), p, n, n), ds = upload_f32(s.data(), p, n, n);
  DeviceStats out(n);
  check(vp_merge_stats_raw(ctx(), static_cast<float*>(dm->p), static_cast<float*>(ds->p), p, n, n, 1.0, out.desc));
  return download_stats(out, n);
}

OutputResult naive_partitioned_output(const TokenBatch& batch, const std::vector<EmbeddingShard>& shards) {
  if (shards.empty()) throw std::invalid_argument("naive: no shards");
  const int64_t V = shards.back().row_end;
  check_batch(batch, V);
  Matrix W(V, batch.X.cols());
  for (const auto& s : shards)
    std::memcpy(W.row_ptr(s.row_begin), s.W.data(), sizeof(double) * size_t(s.W.size()));
  return run(0, batch, W, int(shards.size()), 1.0);
}

ShardState alg1_pass_S(const Matrix& X, const EmbeddingShard& shard) {  // VM.cpp:151-162
  if (X.cols() != shard.W.cols()) throw std::invalid_argument("alg1_pass_S: hidden dim mismatch");
  auto b = device_batch(X, nullptr);
  auto s = device_shard(shard);
  ShardState st = make_state(b, s, X.cols(), shard.rows());
  check(vp_alg1_pass_S(ctx(), &b->desc, &s->desc, st.dev->st));
  fetch_local(&st);
  return st;
}

ShardGrads alg1_pass_T(const ShardState& state, const GlobalStats& stats, const TokenBatch& batch,
                       const EmbeddingShard& shard) {  // VM.cpp:164-179
  if (state.m_local.size() != stats.m.size())
    throw std::invalid_argument("alg1_pass_T: state/stats length mismatch");
  if (!state.dev) throw std::invalid_argument("alg1_pass_T: state has no device pass-S output");
  auto b = device_batch(batch.X, &batch.labels);
  auto s = device_shard(shard);
  auto g = upload_stats(stats);
  const int64_t n = batch.X.rows(), h = batch.X.cols(), ld = b->desc.h;
  DevMem gx(size_t(n * ld) * 4), gw(size_t(shard.rows() * ld) * 4);
  check(vp_alg1_pass_T(ctx(), state.dev->st, g->desc, &b->desc, &s->desc, static_cast<float*>(gx.p), ld,
                       static_cast<float*>(gw.p), ld));
  ShardGrads out;
  out.grad_x_partial = download_f32(gx.p, n, h, ld);
  out.grad_w = download_f32(gw.p, shard.rows(), h, ld);
  return out;
}

ShardState alg2_pass_S(const TokenBatch& batch, const EmbeddingShard& shard) {  // VM.cpp:181-191
  if (batch.X.cols() != shard.W.cols()) throw std::invalid_argument("alg1_pass_S: hidden dim mismatch");
  auto b = device_batch(batch.X, &batch.labels);
  auto s = device_shard(shard);
  ShardState st = make_state(b, s, batch.X.cols(), shard.rows());
  check(vp_alg2_pass_S(ctx(), &b->desc, &s->desc, st.dev->st));
  fetch_local(&st);
  st.has_grad_terms = true;
  return st;
}

BarrierResult alg2_barrier_C1(const std::vector<ShardState>& states) {  // VM.cpp:193-211
  if (states.empty()) throw std::invalid_argument("alg2_barrier_C1: no states");
  std::vector<vp_state_t> st;
  std::vector<vp_shard_t> sd;
  for (const auto& s : states) {
    if (!s.has_grad_terms || !s.dev) throw std::invalid_argument("alg2_barrier_C1: A/B terms missing");
    st.push_back(s.dev->st);
    sd.push_back(s.dev->shard->desc);
  }
  const auto& b = states.front().dev->batch;
  const int64_t n = b->n_tok, h = states.front().dev->h_true, ld = b->desc.h;
  DeviceStats stats(n);
  DevMem gx(size_t(n * ld) * 4);
  check(vp_alg2_barrier_C1(ctx(), st.data(), sd.data(), int(st.size()), &b->desc, 1.0, stats.desc,
                           static_cast<float*>(gx.p), ld));
  BarrierResult r;
  r.stats = download_stats(stats, n);
  r.grad_x = download_f32(gx.p, n, h, ld);
  return r;
}

Matrix alg2_pass_T(const ShardState& state, const GlobalStats& stats, const TokenBatch& batch,
                   const EmbeddingShard& shard) {  // VM.cpp:213-225
  if (state.m_local.size() != stats.m.size())
    throw std::invalid_argument("alg2_pass_T: state/stats length mismatch");
  if (!state.dev) throw std::invalid_argument("alg2_pass_T: state has no device pass-S output");
  auto b = device_batch(batch.X, &batch.labels);
  auto s = device_shard(shard);
  auto g = upload_stats(stats);
  const int64_t h = batch.X.cols(), ld = b->desc.h;
  DevMem gw(size_t(shard.rows() * ld) * 4);
  check(vp_alg2_pass_T(ctx(), state.dev->st, g->desc, &b->desc, &s->desc, static_cast<float*>(gw.p), ld));
  return download_f32(gw.p, shard.rows(), h, ld);
}

Matrix input_forward(const std::vector<int64_t>& tokens, const EmbeddingShard& shard) {  // VM.cpp:227-236
  auto s = device_shard(shard);
  const int64_t n = int64_t(tokens.size()), h = shard.W.cols(), ld = s->ldw;
  auto t = upload_i64(tokens);
  DevMem out(size_t(std::max<int64_t>(n, 1) * ld) * 2);
  check(vp_input_forward(ctx(), static_cast<const int64_t*>(t->p), n, ld, &s->desc, out.p, ld, 0));
  sync();  // surfaces "input_forward: token out of range" (VM.cpp:232)
  std::vector<uint16_t> hb(size_t(n * ld));
  if (n) cuda_check(cudaMemcpy(hb.data(), out.p, hb.size() * 2, cudaMemcpyDeviceToHost));
  Matrix m(n, h);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < h; ++j) {
      const uint32_t u = uint32_t(hb[size_t(i * ld + j)]) << 16;
      float f;
      std::memcpy(&f, &u, 4);
      m(i, j) = f;
    }
  return m;
}

Matrix input_backward(const Matrix& grad_out, const std::vector<int64_t>& tokens,
                      const EmbeddingShard& shard) {  // VM.cpp:238-251
  if (grad_out.rows() != int64_t(tokens.size()))
    throw std::invalid_argument("input_backward: grad/token length mismatch");
  auto s = device_shard(shard);
  const int64_t n = grad_out.rows(), h = grad_out.cols(), ld = pad8(h);
  auto t = upload_i64(tokens);
  DevPtr g = upload_f32(grad_out.data(), n, h, ld);
  DevMem out(size_t(shard.rows() * ld) * 4);
  check(vp_input_backward(ctx(), g->p, ld, 1, static_cast<const int64_t*>(t->p), n, ld, &s->desc,
                          static_cast<float*>(out.p), ld, 0));
  sync();  // surfaces "input_backward: token out of range" (VM.cpp:247)
  return download_f32(out.p, shard.rows(), h, ld);
}

RandomInstance random_instance(int64_t n_tok, int64_t h, int64_t V, uint64_t seed) {  // VM.cpp:253-270
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uniform(-1.0, 1.0);
  RandomInstance inst;
  inst.batch.X.resize(n_tok, h);
  for (int64_t i = 0; i < n_tok; ++i)
    for (int64_t j = 0; j < h; ++j) inst.batch.X(i, j) = uniform(rng);
  inst.W.resize(V, h);
  for (int64_t i = 0; i < V; ++i)
    for (int64_t j = 0; j < h; ++j) inst.W(i, j) = uniform(rng);
  std::uniform_int_distribution<int64_t> label(0, V - 1);
  inst.batch.labels.resize(size_t(n_tok));
  for (auto& g : inst.batch.labels) g = label(rng);
  return inst;
}

OutputResult run_naive(const TokenBatch& batch, const Matrix& W, int p) { return run(0, batch, W, p, 1.0); }
OutputResult run_alg1(const TokenBatch& batch, const Matrix& W, int p, double fault_scale) {
  return run(1, batch, W, p, fault_scale);
}
OutputResult run_alg2(const TokenBatch& batch, const Matrix& W, int p, double fault_scale) {
  return run(2, batch, W, p, fault_scale);
}

int64_t pad_vocab_size(int64_t V, int64_t p) {  // cost_model.cpp:49-55
  if (V < 1 || p < 1) throw std::invalid_argument("pad_vocab_size: V and p must be >= 1");
  const int64_t align = 2 * p;
  return (V + align - 1) / align * align;
}

}  // namespace vpipe
