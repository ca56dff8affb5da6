// C-ABI implementation of include/vpipe_b200.h: contexts, shard states,
// NCCL exchanges and the orchestration of the sm_100a kernels for the
// naive / Algorithm-1 / Algorithm-2 output layer and the input layer.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vpipe_b200.h"
#include "comm.h"
#include "common.h"
#include "gemm_host.cuh"
#include "scatter_kernels.cuh"
#include "vocab_kernels.cuh"
#include "vocab_program.h"

namespace {

thread_local std::string g_last_error;

using vp::CudaError;
using vp::NcclError;
using vp::require;

template <class F>
int api(F&& f) {
  try {
    f();
    return VP_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return VP_EINVAL;
  } catch (const NcclError& e) {
    g_last_error = e.what();
    return VP_ENCCL;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return VP_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return VP_EINTERNAL;
  }
}

// Grow-only device buffer.  A buffer that grows is retired, not freed, until
// the context is destroyed: a CUDA graph captured earlier keeps the old
// pointer and stays valid (its workspace use is internal to the captured
// calls, so a replay reads what it wrote).  No cudaFree on a hot path either
// (cudaFree synchronises the device).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  std::vector<void*> retired;
  void* get(size_t need) {
    if (need > bytes) {
      if (p) retired.push_back(p);
      p = nullptr;
      VP_CUDA(cudaMalloc(&p, need));
      bytes = need;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    for (void* q : retired) cudaFree(q);
    retired.clear();
    p = nullptr;
    bytes = 0;
  }
};

// A device buffer mapped on every rank of the group (Comm::open_peers).
// Grow-only; a grown buffer and its mappings stay alive until the context is
// destroyed (graphs keep the old pointers).
struct SymBuf {
  void* p = nullptr;
  size_t bytes = 0;
  std::vector<void*> peers;  // every rank's buffer as mapped here (own included)
  std::vector<std::pair<void*, std::vector<void*>>> retired;
  bool failed = false;       // some rank could not map its peers: the collective path
};

// deferred device-side argument errors (d_err bits), reported by vp_ctx_sync
constexpr int kErrInputFwd = 1, kErrInputBwd = 2, kErrLabel = 4;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

enum PForm { kRaw = 0, kLocal = 1, kGlobal = 2 };

// NVTX range per vocabulary pass (S, C1, T, C2, the naive barriers, the input
// layer): the reference's pass names on an Nsight timeline (header-only NVTX
// v3: no cost unless a tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace

struct vp_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int num_sms = 148;
  int gemm_sms = 148;
  int cg = 2;
  // GEMM tile rasterisation and TMA L2 policy per GEMM [logits, dX, dW]
  // (measured with lockstep on: evict_last on both operands of all three
  // GEMMs, +2.7% tokens/s over evict_normal, tools/experiments/round1/combo_ab.sh)
  int raster[3] = {16, 16, -4};  // logits: M-fastest in groups of 16 m-tiles (+1.3% with lockstep)
  int pol[3] = {2, 2, 2};
  // B-operand policy when set ("policyb_*"); -9 = same as pol.  Logits: W
  // evict-first, with P stored evict-first (store_hint), so X stays in L2:
  // K1 DRAM 13.3 -> 9.8 GB per launch at the headline (ncu, r02n), step
  // throughput unchanged (r02o)
  int polb[3] = {1, -9, -9};
  int store_hint[3] = {1, -1, -1};  // epilogue store L2 hint per GEMM: 1 evict-first, 0 normal, -1 process-wide option
  int pb(int i) const { return polb[i] == -9 ? pol[i] : polb[i]; }
  int mc = 1;  // CTA pairs per cluster sharing B by TMA multicast (1 or 2)
  // Persisting L2 window per GEMM [logits, dX, dW] on the operand re-read
  // across waves (logits: X, dW: c (.) X); needs the device's persisting L2
  // set-aside (sized on first use, up to persist_max bytes)
  int persist[3] = {0, 0, 0};
  size_t persist_max = 0, persist_set = 0;
  vp::L2Window persist_win(int i, const void* p, size_t bytes) {
    vp::L2Window w;
    if (!persist[i] || persist_max == 0) return w;
    const size_t want = std::min(bytes, persist_max);
    if (want > persist_set) {
      VP_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
      persist_set = want;
    }
    w.ptr = p;
    w.bytes = bytes;
    w.hit_ratio = std::min(1.f, float(double(persist_set) / double(bytes)));
    return w;
  }
  int nh[3] = {2, 2, 2};  // N halves per tile (2 = 256 x 512 pair tiles) for [logits, dX, dW]
  // split-K of the dX GEMM (K = V_k, few waves): ordered, deterministic;
  // splits_dx option: 0 = by wave quantisation (ordered splits) or, below half
  // a wave of tiles, the parallel workspace split-K; 1 = off; 2..32 = forced
  vp::SplitCfg split;
  int splits_dx = 0, splits_dw = 0;
  // wave lockstep per GEMM [logits, dX, dW]: epoch length in k-blocks (0 = off)
  vp::LockCfg lock;
  int lock_epoch[3] = {8, 8, 8};
  const vp::LockCfg* lock_for(int i) {
    lock.epoch = lock_epoch[i];
    return lock.epoch > 0 ? &lock : nullptr;
  }
  // tile shapes actually launched: 512-wide tiles and multicast need CTA pairs
  int eff_nh(int i) const { return cg == 2 ? nh[i] : 1; }
  int eff_mc(int i) const { return cg == 2 && eff_nh(i) == 1 ? mc : 1; }
  std::unique_ptr<vp::Comm> comm;  // NCCL or loopback (comm.h); null = no group
  int nranks = 1, rank = 0;
  bool gemm_sms_set = false;  // "gemm_sms" given explicitly (else a colocated share)
  int64_t vocab_cache_key = -1, vocab_cache = -1;  // global V of the group (label checks)
  vp::RankBounds bounds{};  // every rank's shard rows (owner-gather input forward), cached
  int64_t bounds_key_rb = -1, bounds_key_re = -1;
  int* d_err = nullptr;
  int64_t launches = 0;
  // optional per-GEMM event timing (bench instrumentation): kind -> events
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
  size_t ev_next = 0;
  double gemm_ms[4] = {0, 0, 0, 0};
  int64_t gemm_n[4] = {0, 0, 0, 0};
  // workspace
  DevBuf inv, scale, xs, gathered, packed, tmp_m, tmp_s, heads, counts, vtmp, gbuf;

  void activate() const {
    VP_CUDA(cudaSetDevice(device));
    (void)cudaGetLastError();  // drop stale non-sticky errors left by other code
  }
  bool force_collectives = false;  // route exchanges through NCCL even with 1 rank (tests)
  // C1 overlap (alg2, R/PAPER.md:243/:329): the dX / loss all-reduce runs on a
  // high-priority comm stream while pass T's dW GEMM keeps the compute stream,
  // leaving comm_sms SMs free for NCCL's CTAs.
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  bool overlap_c1 = true, reduce_pending = false;
  int comm_sms = 8;
  // K1 logits y = acc * logit_scale + logit_shift[row] (the reference's
  // logit_shift test hook, VM.cpp:41-43, and a fault-injection scale)
  const float* logit_shift = nullptr;
  float logit_scale = 1.f;
  // dW passes add into grad_w instead of overwriting it (gradient accumulation
  // across microbatches; tied input/output embeddings sharing one dE/dW buffer)
  bool accumulate_dw = false;
  // fused C1 (alg2 in a group, option "fused_c1"): one peer-mapped buffer per
  // rank — slots [nranks][R][h] fp32 (A_k of my token rows, written by rank
  // k's dX epilogue) then B [R][h] bf16 (label rows) — and its mapping on
  // every peer.  Grow-only; a grown buffer and its mappings stay alive until
  // the context is destroyed (graphs keep the old pointers).
  bool fused_c1 = true;
  int64_t fused_count = 0;
  SymBuf sym;     // output layer (slots, B, G)
  SymBuf in_sym;  // input layer: owned rows by token index, two halves (call parity)
  SymBuf bwd_sym; // input backward: root's staged gradient, two halves (call parity)
  int64_t bwd_calls = 0;
  bool peer_input = true;  // option "peer_input": the input forward pulls rows over peer memory
  int64_t in_calls = 0, peer_input_count = 0;
  DevBuf bar;                 // one float: group barriers of the fused exchange
  bool distributed() const { return comm != nullptr && (nranks > 1 || force_collectives); }
  // the NCCL / loopback group; callers check distributed() first
  vp::Comm& cm() const { return *comm; }
  template <class T>
  T* buf(DevBuf& b, size_t count) {
    return static_cast<T*>(b.get(count * sizeof(T)));
  }
  int grid_for(int64_t work, int per_block) const {
    const int64_t blocks = ceil_div(work, per_block);
    const int64_t cap = int64_t(num_sms) * 8;
    return int(std::max<int64_t>(1, std::min(blocks, cap)));
  }
};

struct vp_state_s {
  vp_ctx_s* ctx = nullptr;
  int64_t n_tok = 0, h = 0, rows = 0, ldp = 0, ntiles = 0;
  __nv_bfloat16* P = nullptr;
  float *tile_m = nullptr, *tile_s = nullptr, *m_loc = nullptr, *s_loc = nullptr, *ytgt = nullptr;
  // per-row reference machinery of the K1 epilogue (see EpiLogitStats)
  float *tile_q = nullptr, *row_ref = nullptr, *cfac = nullptr;
  int *ref_flag = nullptr, *row_bad = nullptr, *bad_list = nullptr, *counters = nullptr;  // counters: bad, fix
  int2* fix_list = nullptr;
  int64_t nblk128 = 0;
  float* A = nullptr;  // [n_tok x h] fp32: alg2 A, or per-shard dX partial (alg1/naive local mode)
  float* Y = nullptr;  // naive only: fp32 logits [n_tok x rows]
  int form = kRaw;
  bool has_grad_terms = false;
  bool has_S = false;
};

namespace {

// Bytes vp_state_create allocates for one shard state (P, tile stats, per-row
// arrays, overflow fix lists); vp_workspace_query reports the same figure.
int64_t state_bytes(int64_t n_tok, int64_t h, int64_t rows) {
  const int64_t ldp = round_up(rows, 64), ntiles = ceil_div(rows, vp::kTileN), nblk = ceil_div(n_tok, 128) + 2;
  return n_tok * ldp * 2                         // P (bf16)
         + 3 * ntiles * n_tok * 4                // tile m, s, q
         + 6 * n_tok * 4                         // m', sum', y_tgt, row_ref, cfac, row_bad
         + n_tok * 4 + nblk * 4 + 2 * 4          // bad_list, ref_flag, counters
         + ceil_div(n_tok, 32) * ntiles * 8      // fix_list
         + n_tok * h * 4;                        // A (alg2) / dX partial
}

void free_state_buffers(vp_state_s* st) {
  for (void* p : {static_cast<void*>(st->P), static_cast<void*>(st->tile_m), static_cast<void*>(st->tile_s),
                  static_cast<void*>(st->m_loc), static_cast<void*>(st->s_loc), static_cast<void*>(st->ytgt),
                  static_cast<void*>(st->A), static_cast<void*>(st->Y), static_cast<void*>(st->tile_q),
                  static_cast<void*>(st->row_ref), static_cast<void*>(st->cfac), static_cast<void*>(st->ref_flag),
                  static_cast<void*>(st->row_bad), static_cast<void*>(st->bad_list),
                  static_cast<void*>(st->counters), static_cast<void*>(st->fix_list)})
    if (p) cudaFree(p);
}

void check_batch(const vp_batch_t* b, bool need_labels = true) {
  require(b != nullptr && b->X != nullptr, "TokenBatch: null batch");
  require(b->n_tok >= 1, "TokenBatch: empty X");
  require(!need_labels || b->labels != nullptr, "TokenBatch: labels/X row mismatch");
  require(b->h >= 1 && b->h % 8 == 0, "TokenBatch: h must be a positive multiple of 8 (pad the hidden dim)");
  require(b->ldx >= b->h && b->ldx % 8 == 0, "TokenBatch: ldx must be >= h and a multiple of 8");
  require(aligned16(b->X), "TokenBatch: X must be 16-byte aligned");
}

void check_shard(const vp_shard_t* s, int64_t h) {
  require(s != nullptr && s->W != nullptr, "EmbeddingShard: null shard");
  require(s->row_end > s->row_begin && s->row_begin >= 0, "EmbeddingShard: empty row range");
  require(s->ldw >= h && s->ldw % 8 == 0, "EmbeddingShard: ldw must be >= h and a multiple of 8");
  require(aligned16(s->W), "EmbeddingShard: W must be 16-byte aligned");
}

// dW outputs: the one-hot scatter after the dW GEMM stores float4 rows
void check_grad_w(const float* gw, int64_t ldgw, int64_t h, const char* msg) {
  require(gw != nullptr && ldgw >= h && ldgw % 4 == 0 && aligned16(gw), msg);
}

void check_state(const vp_state_s* st, const vp_batch_t* b, const vp_shard_t* s) {
  require(st != nullptr, "ShardState: null state");
  require(st->n_tok == b->n_tok, "ShardState: n_tok mismatch");
  require(st->h == b->h, "alg1_pass_S: hidden dim mismatch");
  if (s) require(st->rows == s->row_end - s->row_begin, "ShardState: shard rows mismatch");
}

// ---- GEMM timing (kinds: 0 logits+stats K1, 1 logits fp32 (naive), 2 dX K3, 3 dW K4) --
cudaEvent_t next_event(vp_ctx_s* c) {
  if (c->ev_next == c->ev_pool.size()) {
    cudaEvent_t e;
    VP_CUDA(cudaEventCreate(&e));
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_next++];
}

template <class F>
void timed_gemm(vp_ctx_s* c, int kind, F&& launch) {
  if (!c->timing) {
    launch();
    return;
  }
  cudaEvent_t a = next_event(c), b = next_event(c);
  VP_CUDA(cudaEventRecord(a, c->stream));
  launch();
  VP_CUDA(cudaEventRecord(b, c->stream));
  c->ev_pending.push_back({kind, {a, b}});
}

// ---- GEMM wrappers ---------------------------------------------------------
void gemm_logits(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_s* st) {
  VP_CUDA(cudaMemsetAsync(st->ref_flag, 0, size_t(st->nblk128) * sizeof(int), c->stream));
  VP_CUDA(cudaMemsetAsync(st->row_bad, 0, size_t(st->n_tok) * sizeof(int), c->stream));
  VP_CUDA(cudaMemsetAsync(st->counters, 0, 2 * sizeof(int), c->stream));
  vp::EpiLogitStats::Params ep{st->P,       st->ldp,      st->tile_m,   st->tile_s,       st->n_tok,
                               b->labels,   s->row_begin, s->row_end,   st->ytgt,         st->tile_q,
                               st->row_ref, st->ref_flag, st->row_bad,  st->counters,     st->bad_list,
                               st->counters + 1, st->fix_list};
  ep.logit_shift = c->logit_shift;
  ep.logit_scale = c->logit_scale;
  const vp::L2Window win = c->persist_win(0, b->X, size_t((b->n_tok - 1) * b->ldx + b->h) * 2);
  timed_gemm(c, 0, [&] {
    vp::launch_gemm<vp::EpiLogitStats>(c->cg, {b->X, b->ldx, false}, {s->W, s->ldw, false}, int(b->n_tok),
                                       int(st->rows), int(b->h), c->raster[0], ep, c->gemm_sms, c->stream,
                                       c->pol[0], c->pb(0), c->eff_mc(0), c->eff_nh(0), nullptr, c->lock_for(0),
                                       c->store_hint[0], &win);
  });
  ++c->launches;
}

void gemm_logits_f32(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_s* st) {
  vp::EpiStoreF32::Params ep{st->Y, st->rows, st->tile_m, st->n_tok, nullptr};
  timed_gemm(c, 1, [&] {
    vp::launch_gemm<vp::EpiStoreF32>(c->cg, {b->X, b->ldx, false}, {s->W, s->ldw, false}, int(b->n_tok),
                                     int(st->rows), int(b->h), c->raster[0], ep, c->gemm_sms, c->stream, c->pol[0],
                                     c->pol[0], c->eff_mc(0));
  });
  ++c->launches;
}

// out[T x h] = diag(row_scale) . P[T x rows] . W_k[rows x h]
void gemm_dx_ep(vp_ctx_s* c, vp_state_s* st, const vp_shard_t* s, const vp::EpiStoreF32::Params& ep);
void gemm_dx(vp_ctx_s* c, vp_state_s* st, const vp_shard_t* s, float* out, int64_t ldo,
             const float* row_scale = nullptr) {
  vp::EpiStoreF32::Params ep{out, ldo, nullptr, 0, row_scale};
  gemm_dx_ep(c, st, s, ep);
}
void gemm_dx_ep(vp_ctx_s* c, vp_state_s* st, const vp_shard_t* s, const vp::EpiStoreF32::Params& ep) {
  c->split.force = c->splits_dx;
  timed_gemm(c, 2, [&] {
    vp::launch_gemm<vp::EpiStoreF32>(c->cg, {st->P, st->ldp, false}, {s->W, s->ldw, true}, int(st->n_tok),
                                     int(st->h), int(st->rows), c->raster[1], ep, c->gemm_sms, c->stream, c->pol[1],
                                     c->pb(1), c->eff_mc(1), c->eff_nh(1), c->splits_dx == 1 ? nullptr : &c->split,
                                     c->lock_for(1), c->store_hint[1]);
  });
  c->launches += 1 + c->split.reduce_launches;
  c->split.reduce_launches = 0;
}

// out[rows x h] = P^T . Xop   (Xop [T x h] bf16)
void gemm_dw(vp_ctx_s* c, vp_state_s* st, const void* Xop, int64_t ldx, float* out, int64_t ldo) {
  vp::EpiStoreF32::Params ep{out, ldo, nullptr, 0, nullptr, c->accumulate_dw ? 1 : 0};
  const int raster = c->raster[2];
  const vp::L2Window win = c->persist_win(2, Xop, size_t((st->n_tok - 1) * ldx + st->h) * 2);
  c->split.force = c->splits_dw;  // (few-wave shards, e.g. V/8 rows: 13.5 waves -> 3 splits)
  timed_gemm(c, 3, [&] {
    vp::launch_gemm<vp::EpiStoreF32>(c->cg, {st->P, st->ldp, true}, {Xop, ldx, true}, int(st->rows), int(st->h),
                                     int(st->n_tok), raster, ep, c->gemm_sms, c->stream, c->pol[2], c->pb(2),
                                     c->eff_mc(2), c->eff_nh(2), c->splits_dw == 1 ? nullptr : &c->split,
                                     c->lock_for(2), c->store_hint[2], &win);
  });
  c->launches += 1 + c->split.reduce_launches;
  c->split.reduce_launches = 0;
}

// ---- small kernel wrappers ---------------------------------------------------
void stats_reduce(vp_ctx_s* c, vp_state_s* st, bool with_sum) {
  vp::k_stats_reduce<<<unsigned(ceil_div(st->n_tok, 32)), 256, 0, c->stream>>>(
      st->tile_m, with_sum ? st->tile_s : nullptr, int(st->ntiles), st->n_tok, int(st->n_tok), st->m_loc,
      with_sum ? st->s_loc : nullptr);
  VP_KCHECK();
  ++c->launches;
}

float* inv_of(vp_ctx_s* c, const float* s, int64_t n) {
  float* inv = c->buf<float>(c->inv, size_t(n));
  vp::k_inv<<<unsigned(ceil_div(n, 256)), 256, 0, c->stream>>>(s, int(n), inv);
  VP_KCHECK();
  ++c->launches;
  return inv;
}

// c_i = global_scale (VM.cpp:22-27) times cfac_i: the per-row factor that
// turns the state's stored P into the global softmax.
float* global_scale(vp_ctx_s* c, const vp_state_s* st, vp_stats_t g) {
  float* sc = c->buf<float>(c->scale, size_t(st->n_tok));
  vp::k_global_scale<<<unsigned(ceil_div(st->n_tok, 256)), 256, 0, c->stream>>>(
      st->m_loc, st->s_loc, g.m, g.sum, st->form == kLocal ? st->cfac : nullptr, int(st->n_tok), sc);
  VP_KCHECK();
  ++c->launches;
  return sc;
}

// dst[row] (+)= sign * src[i] over owned tokens, ascending i per row
// (scatter_kernels.cuh: counting sort into per-row segments, ordered
// segments, then row / hot-chunk adds).
template <typename Src>
void segment_scatter(vp_ctx_s* c, const int64_t* tok, int64_t n, int64_t rb, int64_t re, const Src* src, int64_t lds,
                     int64_t h, float sign, float* dst, int64_t ldd, int accumulate, int err_bit = 0) {
  if (n == 0) return;
  require(n < (int64_t(1) << 24), "scatter: at most 2^24 tokens per call");
  const int64_t rows = re - rb;
  const int nchunks = int(ceil_div(h, vp::kScChunk));
  const int64_t hot_cap = ceil_div(n, vp::kScHot) * nchunks;
  // zeroed: cnt, headr, fill, seg [rows each] + counters
  int* z = c->buf<int>(c->heads, size_t(4 * rows + vp::kScCtrs));
  // lists: list [n], uni int2 [n], small int4 [n], rep int4 [n], hot int4 [hot_cap]
  int* L = c->buf<int>(c->counts, size_t(n + 2 * n + 4 * n + 4 * n + 4 * hot_cap) + 4);
  vp::ScatterWs w;
  w.cnt = z;
  w.headr = z + rows;
  w.fill = z + 2 * rows;
  w.seg = z + 3 * rows;
  w.ctr = z + 4 * rows;
  w.list = L;
  int* q = L + n;
  q += (reinterpret_cast<uintptr_t>(q) & 15) ? (16 - (reinterpret_cast<uintptr_t>(q) & 15)) / 4 : 0;  // int4 alignment
  w.small = reinterpret_cast<int4*>(q);
  w.rep = w.small + n;
  w.hot = w.rep + n;
  w.uni = reinterpret_cast<int2*>(w.hot + hot_cap);
  w.hot_cap = int(hot_cap);
  const size_t bits = size_t((n + 31) / 32) * sizeof(unsigned);
  require(bits <= 200 * 1024, "scatter: token count too large for the segment sort");
  if (vp::g_cooperative && bits <= 48 * 1024) {
    // one cooperative planning kernel (the profilers' kernel replay cannot
    // relaunch cooperative grids: there the four kernels below run instead)
    static int coop_blocks[64] = {};
    int dev = 0;
    VP_CUDA(cudaGetDevice(&dev));
    int& per_sm = coop_blocks[dev & 63];
    if (per_sm == 0) {
      VP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vp::k_sc_prepare, vp::kScThreads, 48 * 1024));
      per_sm = std::max(1, std::min(per_sm, 2));
    }
    const int grid = int(std::min<int64_t>(int64_t(c->num_sms) * per_sm, std::max<int64_t>(1, ceil_div(n, 256))));
    const int64_t* tk = tok;
    int nn = int(n), nc = nchunks, eb = err_bit;
    int* errp = c->d_err;
    void* args[] = {&tk, &nn, &rb, &re, &nc, &w, &errp, &eb};
    VP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(vp::k_sc_prepare), dim3(unsigned(grid)),
                                        dim3(vp::kScThreads), args, bits, c->stream));
    c->launches += 1;
  } else {
    VP_CUDA(cudaMemsetAsync(z, 0, size_t(4 * rows + vp::kScCtrs) * sizeof(int), c->stream));
    const int g = c->grid_for(n, 256);
    vp::k_sc_count<<<g, 256, 0, c->stream>>>(tok, int(n), rb, re, w, c->d_err, err_bit);
    VP_KCHECK();
    vp::k_sc_plan<<<g, 256, 0, c->stream>>>(tok, int(n), rb, re, nchunks, w);
    VP_KCHECK();
    vp::k_sc_fill<<<g, 256, 0, c->stream>>>(tok, int(n), rb, re, w);
    VP_KCHECK();
    static bool sort_attr = false;
    if (!sort_attr && bits > 48 * 1024) {
      VP_CUDA(cudaFuncSetAttribute(vp::k_sc_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      sort_attr = true;
    }
    vp::k_sc_sort<<<c->num_sms * 2, vp::kScThreads, bits, c->stream>>>(int(n), w);
    VP_KCHECK();
    c->launches += 4;
  }
  vp::k_sc_apply<Src><<<unsigned(hot_cap + n), vp::kScThreads, vp::kScRingBytes, c->stream>>>(
      w, src, lds, int(h), sign, dst, ldd, accumulate);
  VP_KCHECK();
  c->launches += 1;
}

// alg1_pass_S (VM.cpp:151-162): Y = X W_k^T with the fused stats epilogue
// (P = e^{Y - m_tile} in bf16, tile m/sum, y[i, g_i]); per-row merge of the
// tile stats into m', sum'; then P <- softmax' = P e^{m_tile - m'} / sum'
// (VM.cpp:158-160) in place.  P stays softmax' from here on: the T passes
// apply the Eq. 5 factor per row (dX epilogue / scaled X), so they never
// rewrite P and remain pure.
void pass_S_common(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_s* st) {
  NvtxRange nr("vp:S");
  check_batch(b, false);
  check_shard(s, b->h);
  check_state(st, b, s);
  gemm_logits(c, b, s, st);
  const int T = int(st->n_tok);
  const int fix_grid = c->num_sms;
  vp::k_fix_check<<<fix_grid, 256, 0, c->stream>>>(st->fix_list, st->counters + 1, st->tile_q, st->n_tok, T,
                                                   st->row_ref, vp::EpiLogitStats::kMaxRefGap, st->row_bad,
                                                   st->counters, st->bad_list);
  VP_KCHECK();
  vp::k_stats_reduce_ref<<<unsigned(ceil_div(T, 32)), 512, 0, c->stream>>>(
      st->tile_m, st->tile_s, st->tile_q, int(st->ntiles), st->n_tok, T, st->row_ref, st->row_bad, st->m_loc,
      st->s_loc, st->cfac);
  VP_KCHECK();
  vp::k_fix_apply<<<fix_grid, 256, 0, c->stream>>>(st->fix_list, st->counters + 1, st->P, st->ldp, int(st->rows),
                                                   st->tile_q, st->n_tok, T, st->row_ref, st->row_bad);
  VP_KCHECK();
  vp::k_fix_bad<<<fix_grid, 256, 0, c->stream>>>(st->bad_list, st->counters, st->P, st->ldp, int(st->rows),
                                                 st->tile_q, st->n_tok, st->m_loc);
  VP_KCHECK();
  c->launches += 4;
  st->form = kLocal;  // softmax' = P * cfac (per row)
  st->has_grad_terms = false;
  st->has_S = true;
}

void alg2_S(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_s* st) {
  pass_S_common(c, b, s, st);
  NvtxRange nr("vp:S:A=softmax'W");
  gemm_dx(c, st, s, st->A, st->h, st->cfac);  // A = softmax' W_k = diag(cfac) P W_k (VM.cpp:183)
  st->has_grad_terms = true;
}

// Xs = c (.) X in bf16, c = global_scale (the dW operand of both T passes)
const __nv_bfloat16* scaled_x(vp_ctx_s* c, const vp_batch_t* b, const float* sc) {
  auto* xs = c->buf<__nv_bfloat16>(c->xs, size_t(b->n_tok * b->h));
  vp::k_scale_rows_bf16<<<c->grid_for(b->n_tok * b->h / 8, 256), 256, 0, c->stream>>>(
      static_cast<const __nv_bfloat16*>(b->X), b->ldx, sc, int(b->n_tok), int(b->h), xs, b->h);
  VP_KCHECK();
  ++c->launches;
  return xs;
}

// The group's vocabulary size V (labels must lie in [0, V), VM.cpp:18): the
// largest row_end of the local shards, or, in a group, of every rank's shard
// (one max all-reduce per shard layout, cached).
int64_t global_vocab(vp_ctx_s* c, const vp_shard_t* shards, int n) {
  int64_t V = 0;
  for (int k = 0; k < n; ++k) V = std::max(V, shards[k].row_end);
  if (!c->distributed()) return V;
  if (c->vocab_cache_key == V) return c->vocab_cache;
  require(V < (int64_t(1) << 24), "vocab size must be < 2^24");
  float* d = c->buf<float>(c->vtmp, 1);
  const float f = float(V);
  VP_CUDA(cudaMemcpyAsync(d, &f, sizeof(float), cudaMemcpyHostToDevice, c->stream));
  c->cm().all_reduce(d, d, 1, vp::DType::F32, vp::RedOp::Max, c->stream);
  float g = 0.f;
  VP_CUDA(cudaMemcpyAsync(&g, d, sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  VP_CUDA(cudaStreamSynchronize(c->stream));
  c->vocab_cache_key = V;
  c->vocab_cache = int64_t(g);
  return c->vocab_cache;
}

void merge_stats(vp_ctx_s* c, const vp_state_t* states, int n, double fault_scale, vp_stats_t out) {
  NvtxRange nr("vp:C1:stats");
  require(n >= 1 && states != nullptr, "merge_max_sum: empty input");
  require(out.m != nullptr && out.sum != nullptr, "merge_max_sum: null output");
  const int64_t T = states[0]->n_tok;
  for (int k = 0; k < n; ++k) {
    require(states[k] != nullptr && states[k]->has_S, "merge_max_sum: state has no pass-S stats");
    require(states[k]->n_tok == T, "merge_max_sum: length mismatch");
  }
  if (c->distributed()) {
    require(n == 1, "merge_max_sum: one state per rank in an NCCL group");
    float* packed = c->buf<float>(c->packed, size_t(2 * T));
    float* gathered = c->buf<float>(c->gathered, size_t(2 * T * c->nranks));
    vp::k_pack_stats<<<unsigned(ceil_div(T, 256)), 256, 0, c->stream>>>(states[0]->m_loc, states[0]->s_loc, int(T),
                                                                        packed);
    VP_KCHECK();
    c->cm().all_gather(packed, gathered, size_t(2 * T), vp::DType::F32, c->stream);
    vp::k_merge_stats<<<unsigned(ceil_div(T, 256)), 256, 0, c->stream>>>(
        gathered, gathered + T, c->nranks, 2 * T, int(T), float(fault_scale), out.m, out.sum);
    VP_KCHECK();
    c->launches += 2;
  } else {
    require(n <= vp::kMaxLocalShards, "merge_max_sum: too many local shards");
    vp::StatsParts parts{};
    parts.p = n;
    for (int k = 0; k < n; ++k) {
      parts.m[k] = states[k]->m_loc;
      parts.s[k] = states[k]->s_loc;
    }
    vp::k_merge_stats_ptrs<<<unsigned(ceil_div(T, 256)), 256, 0, c->stream>>>(parts, int(T), float(fault_scale),
                                                                             out.m, out.sum);
    VP_KCHECK();
    ++c->launches;
  }
}

// alg1_pass_T (VM.cpp:164-179):  grad_y = softmax' (.) c - G_k,
//   dX_k = grad_y W_k = diag(c) (softmax' W_k) - G_k W_k   (row scale in the epilogue, row gather)
//   dW_k = grad_y^T X = softmax'^T (c (.) X) - G_k^T X     (scaled X operand, ordered scatter)
void alg1_T(vp_ctx_s* c, vp_state_s* st, vp_stats_t g, const vp_batch_t* b, const vp_shard_t* s, float* gx,
            int64_t ldgx, float* gw, int64_t ldgw) {
  NvtxRange nr("vp:T(alg1)");
  check_batch(b);
  check_shard(s, b->h);
  check_state(st, b, s);
  require(st->has_S && st->form == kLocal, "alg1_pass_T: state/stats length mismatch");
  require(g.m && g.sum, "alg1_pass_T: null stats");
  check_grad_w(gw, ldgw, b->h, "alg1_pass_T: grad_w needs ldgw >= h, ldgw % 4 == 0 and a 16-byte aligned base");
  const float* sc = global_scale(c, st, g);
  gemm_dx(c, st, s, gx, ldgx, sc);
  vp::k_sub_label_rows<<<c->grid_for(st->n_tok * st->h / 2, 256), 256, 0, c->stream>>>(
      gx, ldgx, static_cast<const __nv_bfloat16*>(s->W), s->ldw, s->row_begin, s->row_end, b->labels,
      int(st->n_tok), int(st->h));
  VP_KCHECK();
  ++c->launches;
  gemm_dw(c, st, scaled_x(c, b, sc), b->h, gw, ldgw);
  segment_scatter(c, b->labels, b->n_tok, s->row_begin, s->row_end, static_cast<const __nv_bfloat16*>(b->X), b->ldx,
                  b->h, -1.f, gw, ldgw, 1, kErrLabel);
}

// alg2_pass_T (VM.cpp:213-225): dW_k = softmax'^T (c (.) X) - G_k^T X
void alg2_T(vp_ctx_s* c, vp_state_s* st, vp_stats_t g, const vp_batch_t* b, const vp_shard_t* s, float* gw,
            int64_t ldgw) {
  NvtxRange nr("vp:T(alg2)");
  check_batch(b);
  check_shard(s, b->h);
  check_state(st, b, s);
  require(st->has_S && st->form == kLocal, "alg2_pass_T: state/stats length mismatch");
  require(g.m && g.sum, "alg2_pass_T: null stats");
  check_grad_w(gw, ldgw, b->h, "alg2_pass_T: grad_w needs ldgw >= h, ldgw % 4 == 0 and a 16-byte aligned base");
  // c (.) X with the global scale computed per row inside the scaling pass
  auto* xs = c->buf<__nv_bfloat16>(c->xs, size_t(b->n_tok * b->h));
  const vp::RowScale rs{st->m_loc, st->s_loc, g.m, g.sum, st->form == kLocal ? st->cfac : nullptr};
  vp::k_scale_rows_global_bf16<<<c->grid_for(b->n_tok * b->h / 8, 256), 256, 0, c->stream>>>(
      static_cast<const __nv_bfloat16*>(b->X), b->ldx, rs, int(b->n_tok), int(b->h), xs, b->h);
  VP_KCHECK();
  ++c->launches;
  gemm_dw(c, st, xs, b->h, gw, ldgw);
  segment_scatter(c, b->labels, b->n_tok, s->row_begin, s->row_end, static_cast<const __nv_bfloat16*>(b->X), b->ldx,
                  b->h, -1.f, gw, ldgw, 1, kErrLabel);
}

// loss != nullptr (one device, no group): the per-token loss is computed by
// the combine kernel too (what loss_of would do, one launch fewer)
void alg2_C1(vp_ctx_s* c, const vp_state_t* states, const vp_shard_t* shards, int n, const vp_batch_t* b,
             double fault_scale, vp_stats_t out, float* gx, int64_t ldgx, bool reduce = true,
             float* loss = nullptr) {
  NvtxRange nr("vp:C1");
  require(n >= 1 && states != nullptr, "alg2_barrier_C1: no states");
  check_batch(b);
  for (int k = 0; k < n; ++k) {
    require(states[k] != nullptr && states[k]->has_grad_terms && states[k]->form == kLocal,
            "alg2_barrier_C1: A/B terms missing");
    check_shard(&shards[k], b->h);
    check_state(states[k], b, &shards[k]);
  }
  require(gx != nullptr && ldgx >= b->h && ldgx % 4 == 0 && aligned16(gx), "alg2_barrier_C1: bad grad_x buffer");
  merge_stats(c, states, n, fault_scale, out);
  vp::CombineShards S{};
  S.p = n;
  S.lda = b->h;
  for (int k = 0; k < n; ++k) {
    S.A[k] = states[k]->A;
    S.W[k] = static_cast<const __nv_bfloat16*>(shards[k].W);
    S.ldw[k] = shards[k].ldw;
    S.rb[k] = shards[k].row_begin;
    S.re[k] = shards[k].row_end;
    S.ml[k] = states[k]->m_loc;
    S.sl[k] = states[k]->s_loc;
    S.yt[k] = states[k]->ytgt;
  }
  require(loss == nullptr || !c->distributed(), "alg2_barrier_C1: the fused loss is for one device");
  const int64_t V = global_vocab(c, shards, n);
  vp::k_alg2_combine<<<c->grid_for(b->n_tok * b->h / 4, 256), 256, 0, c->stream>>>(
      S, out.m, out.sum, b->labels, int(b->n_tok), int(b->h), gx, ldgx, V, c->d_err, kErrLabel, loss);
  VP_KCHECK();
  ++c->launches;
  if (c->distributed() && reduce) {
    require(ldgx == b->h, "alg2_barrier_C1: grad_x must be dense (ldgx == h) for the all-reduce");
    c->cm().all_reduce(gx, gx, size_t(b->n_tok * b->h), vp::DType::F32, vp::RedOp::Sum, c->stream);
  }
}

void loss_of(vp_ctx_s* c, const vp_state_t* states, const vp_shard_t* shards, int n, vp_stats_t g,
             const vp_batch_t* b, float* loss, bool reduce = true) {
  require(n >= 1 && n <= vp::kMaxLocalShards, "loss: bad shard count");
  require(loss != nullptr, "loss: null output");
  vp::LossShards S{};
  S.p = n;
  for (int k = 0; k < n; ++k) {
    S.yt[k] = states[k]->ytgt;
    S.rb[k] = shards[k].row_begin;
    S.re[k] = shards[k].row_end;
  }
  const int64_t V = global_vocab(c, shards, n);
  vp::k_loss<<<unsigned(ceil_div(b->n_tok, 256)), 256, 0, c->stream>>>(S, g.m, g.sum, b->labels, int(b->n_tok),
                                                                       loss, V, c->d_err, kErrLabel);
  VP_KCHECK();
  ++c->launches;
  if (c->distributed() && reduce)
    c->cm().all_reduce(loss, loss, size_t(b->n_tok), vp::DType::F32, vp::RedOp::Sum, c->stream);
}

void reduce_partials(vp_ctx_s* c, float* const* partials, int n, int64_t T, int64_t h, int64_t ld, float* gx,
                     int64_t ldgx) {
  require(n >= 1, "reduce_grad_x: no partials");
  require(ld == h && ldgx == h, "reduce_grad_x: partials and grad_x must be dense [n_tok x h]");
  if (c->distributed()) {
    require(n == 1, "reduce_grad_x: one partial per rank in an NCCL group");
    c->cm().all_reduce(partials[0], gx, size_t(T * h), vp::DType::F32, vp::RedOp::Sum, c->stream);
    return;
  }
  require(n <= vp::kMaxLocalShards, "reduce_grad_x: too many partials");
  vp::PartialPtrs S{};
  S.p = n;
  for (int k = 0; k < n; ++k) S.P[k] = partials[k];
  vp::k_sum_partials<<<c->grid_for(T * h, 256), 256, 0, c->stream>>>(S, T * h, gx);
  VP_KCHECK();
  ++c->launches;
}

// Fork the queued all-reduces (grad_x, loss) onto the comm stream after the
// compute stream's current work; the compute stream continues with pass T.
void fork_allreduces(vp_ctx_s* c, float* gx, int64_t n_gx, float* loss, int64_t n_loss) {
  NvtxRange nr("vp:C1:allreduce(dX,loss)");
  VP_CUDA(cudaEventRecord(c->ev_ready, c->stream));
  VP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
  c->cm().group_start();
  c->cm().all_reduce(gx, gx, size_t(n_gx), vp::DType::F32, vp::RedOp::Sum, c->comm_stream);
  c->cm().all_reduce(loss, loss, size_t(n_loss), vp::DType::F32, vp::RedOp::Sum, c->comm_stream);
  c->cm().group_end();
  VP_CUDA(cudaEventRecord(c->ev_done, c->comm_stream));
  c->reduce_pending = true;
}

void join_allreduces(vp_ctx_s* c) {
  if (!c->reduce_pending) return;
  VP_CUDA(cudaStreamWaitEvent(c->stream, c->ev_done, 0));
  c->reduce_pending = false;
}

// Row ranges of every rank's shard (all-gathered once per layout, cached).
const vp::RankBounds& rank_bounds(vp_ctx_s* c, const vp_shard_t* s) {
  if (c->bounds_key_rb == s->row_begin && c->bounds_key_re == s->row_end && c->bounds.n == c->nranks)
    return c->bounds;
  require(c->nranks <= vp::kMaxRanks, "input_forward_gathered: too many ranks");
  require(s->row_end < (int64_t(1) << 24), "input_forward_gathered: vocab size must be < 2^24");
  float* d = c->buf<float>(c->vtmp, size_t(2 + 2 * c->nranks));
  const float mine[2] = {float(s->row_begin), float(s->row_end)};
  VP_CUDA(cudaMemcpyAsync(d, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
  c->cm().all_gather(d, d + 2, 2, vp::DType::F32, c->stream);
  std::vector<float> all(size_t(2 * c->nranks));
  VP_CUDA(cudaMemcpyAsync(all.data(), d + 2, all.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  VP_CUDA(cudaStreamSynchronize(c->stream));
  c->bounds.n = c->nranks;
  for (int k = 0; k < c->nranks; ++k) {
    c->bounds.rb[k] = int64_t(all[size_t(2 * k)]);
    c->bounds.re[k] = int64_t(all[size_t(2 * k + 1)]);
  }
  c->bounds_key_rb = s->row_begin;
  c->bounds_key_re = s->row_end;
  return c->bounds;
}

// ---- fused C1 / C2 over peer memory (option "fused_c1") ----------------------
// Rank o owns token rows [o R, min(T, (o + 1) R)), R a multiple of 32 so one
// epilogue store box (32 rows) never straddles two owners.  Each rank's peer
// buffer (mapped on every peer) holds
//   slots [nranks][R][h] fp32 — A_k of my rows, stored by rank k's dX epilogue
//   B     [R][h] bf16      — the label rows of my tokens, pushed by the label's owner
//   G     [R][h] fp32      — my rows of grad_x after the combine, pulled by every
//                            rank's copy engines
// See k_alg2_combine_owned for the arithmetic.
struct FusedLayout {
  int64_t R = 0;
  int n_own = 0;   // ranks that own at least one row
  int splits = 1;  // split-K units of the routed dX GEMM (one slot each)
  size_t slot_off = 0, b_off = 0, g_off = 0, need = 0;
};

// `base`: byte offset of this layout's region in the peer buffer (the
// executor keeps one region per microbatch); need = base + region bytes.
// The split-K count of the routed dX GEMM (K = rows = V_k) is chosen here,
// like the unrouted launch's (wave quantisation; option "splits_dx"), because
// it sets the slot layout: every split unit stores into its own slot.
FusedLayout fused_layout(const vp_ctx_s* c, int64_t T, int64_t h, int64_t rows, size_t base = 0) {
  FusedLayout L;
  L.R = round_up(ceil_div(T, c->nranks), 32);
  L.n_own = int(ceil_div(T, L.R));
  if (c->splits_dx > 0) {
    L.splits = c->splits_dx;
  } else {
    const int bn = c->eff_nh(1) == 2 ? 512 : 256;
    const int tiles = int(ceil_div(T, 256) * ceil_div(h, bn));
    L.splits = vp::choose_splits(tiles, std::max(1, c->gemm_sms / 2), int(ceil_div(rows, 64)), c->split.min_kb);
  }
  L.splits = std::max(1, std::min(L.splits, vp::kMaxRoute / std::max(1, L.n_own)));
  L.splits = std::min<int>(L.splits, int(std::max<int64_t>(1, ceil_div(rows, 64))));
  const size_t rowf = size_t(L.R) * size_t(h);
  L.slot_off = base;
  L.b_off = L.slot_off + size_t(c->nranks) * size_t(L.splits) * rowf * sizeof(float);
  L.g_off = L.b_off + size_t(round_up(int64_t(rowf * sizeof(__nv_bfloat16)), 256));
  L.need = size_t(round_up(int64_t(L.g_off + rowf * sizeof(float)), 256));
  return L;
}

// Collective: every rank's buffer `sb` holds >= need bytes and is mapped on
// every peer.  false (on every rank) when some rank cannot map its peers.
bool ensure_sym(vp_ctx_s* c, SymBuf& sb, size_t need) {
  if (sb.failed) return false;
  if (need <= sb.bytes) return true;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  VP_CUDA(cudaStreamIsCapturing(c->stream, &cs));
  require(cs == cudaStreamCaptureStatusNone,
          "peer buffers must be sized outside graph capture (run the step once eagerly first)");
  const size_t bytes = size_t(round_up(int64_t(need), int64_t(2) << 20));
  void* p = nullptr;
  VP_CUDA(cudaMalloc(&p, bytes));
  std::vector<void*> peers;
  try {
    peers = c->cm().open_peers(p, c->stream);
  } catch (...) {
    cudaFree(p);
    throw;
  }
  if (peers.empty()) {
    cudaFree(p);
    sb.failed = true;
    return false;
  }
  if (sb.p) sb.retired.emplace_back(sb.p, sb.peers);
  sb.p = p;
  sb.bytes = bytes;
  sb.peers = std::move(peers);
  return true;
}

// The fused path is decided from the group-wide shape (every rank takes the
// same branch); per-rank buffer requirements are checked, not negotiated.
bool use_fused_c1(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, int n, FusedLayout& L) {
  // (a forced 1-rank group takes it too: the NCCL call sites and graph
  // capture of the fused exchange are then testable on one GPU)
  if (!(c->fused_c1 && c->distributed() && n == 1 && c->nranks <= vp::kMaxRoute &&
        b->h % 8 == 0 && !c->sym.failed))
    return false;
  require(s->ldw % 8 == 0 && aligned16(s->W),
          "fused_c1: the shard needs ldw % 8 == 0 and a 16-byte aligned W (or set fused_c1 = 0 on every rank)");
  L = fused_layout(c, b->n_tok, b->h, s->row_end - s->row_begin);
  return ensure_sym(c, c->sym, L.need);
}

// Routed dX of pass S (alg2) / pass T (alg1): output rows go to slot `rank`
// of their owners' buffers (the epilogue's TMA stores, over NVLink for a
// peer), then the label rows B_k (VM.cpp:185-188, :176) into the owners' B.
void gemm_dx_routed(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_s* st, const float* row_scale,
                    const FusedLayout& L) {
  const int64_t T = b->n_tok, h = b->h;
  vp::EpiStoreF32::Params ep{nullptr, h, nullptr, 0, row_scale};
  ep.route_n = L.n_own;
  ep.route_rows = int(L.R);
  ep.route_splits = L.splits;
  vp::PeerRows pr{};
  for (int o = 0; o < L.n_own; ++o) {
    char* peer = static_cast<char*>(c->sym.peers[size_t(o)]);
    const int64_t rows = std::min(L.R, T - o * L.R);
    (void)rows;  // (rows past T are masked by the epilogue: the last owner's slot has R rows)
    for (int sp = 0; sp < L.splits; ++sp)  // slot (my rank, sp) of owner o
      ep.route_out[o * L.splits + sp] = reinterpret_cast<float*>(peer + L.slot_off) +
                                        (size_t(c->rank) * size_t(L.splits) + size_t(sp)) * size_t(L.R) * size_t(h);
    pr.p[o] = peer + L.b_off;
  }
  gemm_dx_ep(c, st, s, ep);
  vp::k_push_label_rows<<<c->grid_for(T * h / 8, 256), 256, 0, c->stream>>>(
      static_cast<const __nv_bfloat16*>(s->W), s->ldw, s->row_begin, s->row_end, b->labels, int(T), int(h),
      int(L.R), pr);
  VP_KCHECK();
  ++c->launches;
}

// alg2_pass_S with the dX epilogue routed to the token rows' owners.
void alg2_S_fused(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_s* st, const FusedLayout& L) {
  pass_S_common(c, b, s, st);
  NvtxRange nr("vp:S:A=softmax'W->owners");
  gemm_dx_routed(c, b, s, st, st->cfac, L);  // A_k = diag(cfac) P W_k (VM.cpp:183), tile by tile into the owners
  st->has_grad_terms = false;  // A_k is in the owners' buffers, not in the state
}

// The owner's combine of its token rows (local memory only) into G, then the
// grad_x all-gather by copy engines: `barrier` (a small collective on the
// compute stream: the loss all-reduce in alg2) orders every owner's combine
// before any pull, and one peer-to-peer copy per owner pulls its rows straight
// into grad_x — on the comm stream when `overlap`, so pass T's GEMM keeps
// every SM (no NCCL kernel runs beside it).  alg2 C1: slots hold A_k, scaled
// here by c_k from the gathered stats; alg1 C2 (`prescaled`): slots hold c_k A_k.
template <class Barrier>
void owner_combine_gather(vp_ctx_s* c, const vp_shard_t* s, const vp_batch_t* b, vp_stats_t g, bool prescaled,
                          float* gx, int64_t ldgx, const FusedLayout& L, bool overlap, Barrier&& barrier) {
  const int64_t T = b->n_tok, h = b->h, R = L.R;
  const vp::RankBounds& RB = rank_bounds(c, s);
  char* mine = static_cast<char*>(c->sym.p);
  vp::OwnedCombine S{};
  S.slots = reinterpret_cast<const float*>(mine + L.slot_off);
  S.B = reinterpret_cast<const __nv_bfloat16*>(mine + L.b_off);
  S.gathered = prescaled ? nullptr : static_cast<const float*>(c->gathered.p);
  for (int k = 0; k < c->nranks; ++k) {
    S.rb[k] = RB.rb[k];
    S.re[k] = RB.re[k];
  }
  S.nranks = c->nranks;
  S.R = int(R);
  S.row0 = int(c->rank * R);
  S.rows = int(std::max<int64_t>(0, std::min(R, T - c->rank * R)));
  S.prescaled = prescaled ? 1 : 0;
  S.splits = L.splits;
  const int64_t V = global_vocab(c, s, 1);
  if (S.rows > 0) {
    vp::k_alg2_combine_owned<<<c->grid_for(int64_t(S.rows) * h / 4, 256), 256, 0, c->stream>>>(
        S, g.m, g.sum, b->labels, int(T), int(h), reinterpret_cast<float*>(mine + L.g_off), h, V, c->d_err,
        kErrLabel);
    VP_KCHECK();
    ++c->launches;
  }
  barrier();  // every owner's G is complete (and, for the next step, read)
  NvtxRange nx("vp:gather(dX): copy engines");
  cudaStream_t xs = c->stream;
  if (overlap) {
    VP_CUDA(cudaEventRecord(c->ev_ready, c->stream));
    VP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
    xs = c->comm_stream;
  }
  for (int o = 0; o < L.n_own; ++o) {
    const int64_t rows = std::min(R, T - o * R);
    const char* src = static_cast<const char*>(c->sym.peers[size_t(o)]) + L.g_off;
    VP_CUDA(cudaMemcpy2DAsync(gx + o * R * ldgx, size_t(ldgx) * sizeof(float), src, size_t(h) * sizeof(float),
                              size_t(h) * sizeof(float), size_t(rows), cudaMemcpyDefault, xs));
  }
  if (overlap) {
    VP_CUDA(cudaEventRecord(c->ev_done, c->comm_stream));
    c->reduce_pending = true;
  }
  ++c->fused_count;
}

// One-float collective on the compute stream: a group barrier that is
// stream-ordered on every rank (NCCL or loopback).
void group_barrier(vp_ctx_s* c) {
  float* bar = c->buf<float>(c->bar, 1);
  c->cm().all_reduce(bar, bar, 1, vp::DType::F32, vp::RedOp::Max, c->stream);
}

// alg2_barrier_C1 (VM.cpp:193-211) for the fused layout: stats all-gather and
// merge (which also orders every rank's routed stores before the combine),
// the loss at the label owner + its sum all-reduce (T floats, before pass T),
// then the owners' combine and the SM-free gather.
void alg2_C1_fused(vp_ctx_s* c, const vp_state_t st, const vp_shard_t* s, const vp_batch_t* b, double fault_scale,
                   vp_stats_t out, float* loss, float* gx, int64_t ldgx, const FusedLayout& L, bool overlap) {
  NvtxRange nr("vp:C1(fused)");
  require(gx != nullptr && ldgx >= b->h && ldgx % 4 == 0 && aligned16(gx), "alg2_barrier_C1: bad grad_x buffer");
  merge_stats(c, &st, 1, fault_scale, out);
  loss_of(c, &st, s, 1, out, b, loss, /*reduce=*/false);
  owner_combine_gather(c, s, b, out, false, gx, ldgx, L, overlap, [&] {
    c->cm().all_reduce(loss, loss, size_t(b->n_tok), vp::DType::F32, vp::RedOp::Sum, c->stream);
  });
}

// alg1_pass_T (VM.cpp:164-179) with the dX partial routed to the owners.
void alg1_T_routed(vp_ctx_s* c, vp_state_s* st, vp_stats_t g, const vp_batch_t* b, const vp_shard_t* s, float* gw,
                   int64_t ldgw, const FusedLayout& L) {
  NvtxRange nr("vp:T(alg1, dX->owners)");
  check_batch(b);
  check_shard(s, b->h);
  check_state(st, b, s);
  require(st->has_S && st->form == kLocal, "alg1_pass_T: state/stats length mismatch");
  require(g.m && g.sum, "alg1_pass_T: null stats");
  check_grad_w(gw, ldgw, b->h, "alg1_pass_T: grad_w needs ldgw >= h, ldgw % 4 == 0 and a 16-byte aligned base");
  const float* sc = global_scale(c, st, g);
  gemm_dx_routed(c, b, s, st, sc, L);
  gemm_dw(c, st, scaled_x(c, b, sc), b->h, gw, ldgw);
  segment_scatter(c, b->labels, b->n_tok, s->row_begin, s->row_end, static_cast<const __nv_bfloat16*>(b->X), b->ldx,
                  b->h, -1.f, gw, ldgw, 1, kErrLabel);
}

// alg1 with the fused C2: pass T's dX (c (.) softmax' W_k, VM.cpp:176) goes
// to the owners; after T a barrier, the owners' combine, a barrier, the pulls.
void run_alg1_fused(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_t st, double fault_scale,
                    vp_stats_t out, float* loss, float* gx, int64_t ldgx, float* gw, int64_t ldgw,
                    const FusedLayout& L) {
  pass_S_common(c, b, s, st);
  merge_stats(c, &st, 1, fault_scale, out);
  loss_of(c, &st, s, 1, out, b, loss);
  require(gx != nullptr && ldgx >= b->h && ldgx % 4 == 0 && aligned16(gx), "run_alg1: bad grad_x buffer");
  alg1_T_routed(c, st, out, b, s, gw, ldgw, L);
  NvtxRange nr("vp:C2(fused)");
  group_barrier(c);  // every rank's routed stores and label rows have landed
  owner_combine_gather(c, s, b, out, true, gx, ldgx, L, false, [&] { group_barrier(c); });
}

// The exchange after the combine needs no SM, so pass T's dW GEMM keeps all
// of them (the all-reduce path leaves comm_sms to NCCL during T).
void run_alg2_fused(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* s, vp_state_t st, double fault_scale,
                    vp_stats_t out, float* loss, float* gx, int64_t ldgx, float* gw, int64_t ldgw,
                    const FusedLayout& L) {
  alg2_S_fused(c, b, s, st, L);
  const bool overlap = c->overlap_c1 && c->comm_stream != nullptr;
  alg2_C1_fused(c, st, s, b, fault_scale, out, loss, gx, ldgx, L, overlap);
  try {
    alg2_T(c, st, out, b, s, gw, ldgw);
  } catch (...) {
    join_allreduces(c);
    throw;
  }
  join_allreduces(c);
}

void run_alg(int alg, vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* shards, const vp_state_t* states, int n,
             double fault_scale, vp_stats_t out, float* loss, float* gx, int64_t ldgx, float* const* gw,
             int64_t ldgw) {
  require(n >= 1 && n <= vp::kMaxLocalShards, "run: bad shard count");
  require(!c->distributed() || n == 1, "run: one shard per rank in an NCCL group");
  FusedLayout L;
  if (alg != 0 && use_fused_c1(c, b, shards, n, L)) {
    check_batch(b);
    if (alg == 2) run_alg2_fused(c, b, &shards[0], states[0], fault_scale, out, loss, gx, ldgx, gw[0], ldgw, L);
    else run_alg1_fused(c, b, &shards[0], states[0], fault_scale, out, loss, gx, ldgx, gw[0], ldgw, L);
    return;
  }
  if (alg == 2) {
    for (int k = 0; k < n; ++k) alg2_S(c, b, &shards[k], states[k]);
    const bool overlap = c->distributed() && c->overlap_c1 && c->comm_stream != nullptr;
    if (!c->distributed()) {
      require(loss != nullptr, "loss: null output");
      alg2_C1(c, states, shards, n, b, fault_scale, out, gx, ldgx, true, loss);  // + the loss, one launch
    } else {
      alg2_C1(c, states, shards, n, b, fault_scale, out, gx, ldgx, /*reduce=*/!overlap);
      loss_of(c, states, shards, n, out, b, loss, /*reduce=*/!overlap);
    }
    const int sms = c->gemm_sms;
    if (overlap) {
      // C1's only heavy exchange overlaps pass T (T is "arbitrarily delayable")
      require(ldgx == b->h, "alg2_barrier_C1: grad_x must be dense (ldgx == h) for the all-reduce");
      fork_allreduces(c, gx, b->n_tok * b->h, loss, b->n_tok);
      c->gemm_sms = std::max(2, (c->gemm_sms - c->comm_sms) / 2 * 2);
    }
    try {
      for (int k = 0; k < n; ++k) alg2_T(c, states[k], out, b, &shards[k], gw[k], ldgw);
    } catch (...) {
      c->gemm_sms = sms;
      join_allreduces(c);
      throw;
    }
    c->gemm_sms = sms;
    join_allreduces(c);
  } else {
    for (int k = 0; k < n; ++k) pass_S_common(c, b, &shards[k], states[k]);
    merge_stats(c, states, n, fault_scale, out);
    loss_of(c, states, shards, n, out, b, loss);
    std::vector<float*> partials(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
      // local mode: each shard's dX partial lives in its state's A buffer;
      // NCCL mode: the partial is written straight into grad_x and all-reduced.
      partials[size_t(k)] = c->distributed() ? gx : states[k]->A;
      alg1_T(c, states[k], out, b, &shards[k], partials[size_t(k)], c->distributed() ? ldgx : b->h, gw[k], ldgw);
    }
    NvtxRange nr("vp:C2");
    if (c->distributed()) {
      require(ldgx == b->h, "run_alg1: grad_x must be dense for the all-reduce");
      c->cm().all_reduce(gx, gx, size_t(b->n_tok * b->h), vp::DType::F32, vp::RedOp::Sum, c->stream);
    } else {
      reduce_partials(c, partials.data(), n, b->n_tok, b->h, b->h, gx, ldgx);
    }
  }
}

void naive(vp_ctx_s* c, const vp_batch_t* b, const vp_shard_t* shards, const vp_state_t* states, int n,
           vp_stats_t out, float* loss, float* gx, int64_t ldgx, float* const* gw, int64_t ldgw) {
  NvtxRange nr("vp:naive(F1,F2,B)");
  require(n >= 1 && shards != nullptr, "naive: no shards");
  require(n <= vp::kMaxLocalShards, "naive: too many local shards");
  require(!c->distributed() || n == 1, "naive: one shard per rank in an NCCL group");
  check_batch(b);
  const int64_t T = b->n_tok;
  for (int k = 0; k < n; ++k) {
    check_shard(&shards[k], b->h);
    check_grad_w(gw[k], ldgw, b->h, "naive: grad_w needs ldgw >= h, ldgw % 4 == 0 and a 16-byte aligned base");
    check_state(states[k], b, &shards[k]);
    vp_state_s* st = states[k];
    if (!st->Y) VP_CUDA(cudaMalloc(&st->Y, size_t(T * st->rows) * sizeof(float)));
  }
  // F1: local logits + local max, then the max all-reduce (VM.cpp:111-117)
  for (int k = 0; k < n; ++k) {
    vp_state_s* st = states[k];
    gemm_logits_f32(c, b, &shards[k], st);
    stats_reduce(c, st, false);
    vp::k_gather_target<<<unsigned(ceil_div(T, 256)), 256, 0, c->stream>>>(
        st->Y, st->rows, b->labels, shards[k].row_begin, shards[k].row_end, int(T), st->ytgt);
    VP_KCHECK();
    ++c->launches;
  }
  if (c->distributed()) {
    c->cm().all_reduce(states[0]->m_loc, out.m, size_t(T), vp::DType::F32, vp::RedOp::Max, c->stream);
  } else {
    vp::StatsParts parts{};
    parts.p = n;
    for (int k = 0; k < n; ++k) parts.m[k] = parts.s[k] = states[k]->m_loc;
    // max over shards: merge with s = m is not meaningful; use the max-only path
    float* dummy = c->buf<float>(c->tmp_s, size_t(T));
    vp::k_merge_stats_ptrs<<<unsigned(ceil_div(T, 256)), 256, 0, c->stream>>>(parts, int(T), 1.f, out.m, dummy);
    VP_KCHECK();
    ++c->launches;
  }
  // F2: exp-sums against the global max, re-reading the logits, then the sum all-reduce
  for (int k = 0; k < n; ++k) {
    vp_state_s* st = states[k];
    vp::k_naive_exp_sum<<<unsigned(T), 256, 0, c->stream>>>(st->Y, st->rows, int(st->rows), out.m, nullptr, st->ldp,
                                                             st->s_loc);
    VP_KCHECK();
    ++c->launches;
  }
  if (c->distributed()) {
    c->cm().all_reduce(states[0]->s_loc, out.sum, size_t(T), vp::DType::F32, vp::RedOp::Sum, c->stream);
  } else {
    vp::PartialPtrs S{};
    S.p = n;
    for (int k = 0; k < n; ++k) S.P[k] = states[k]->s_loc;
    vp::k_sum_partials<<<c->grid_for(T, 256), 256, 0, c->stream>>>(S, T, out.sum);
    VP_KCHECK();
    ++c->launches;
  }
  // B: softmax, loss at the owner, -1 at the label, dX partials, dW rows
  const float* inv = inv_of(c, out.sum, T);
  std::vector<float*> partials(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    vp_state_s* st = states[k];
    vp::k_naive_softmax<<<c->grid_for(T * ceil_div(st->rows, 8), 256), 256, 0, c->stream>>>(
        st->Y, st->rows, int(T), int(st->rows), out.m, inv, st->P, st->ldp);
    VP_KCHECK();
    ++c->launches;
    st->form = kGlobal;
    st->has_S = true;
    partials[size_t(k)] = c->distributed() ? gx : st->A;
    const int64_t ld = c->distributed() ? ldgx : b->h;
    gemm_dx(c, st, &shards[k], partials[size_t(k)], ld);
    vp::k_sub_label_rows<<<c->grid_for(T * b->h / 2, 256), 256, 0, c->stream>>>(
        partials[size_t(k)], ld, static_cast<const __nv_bfloat16*>(shards[k].W), shards[k].ldw, shards[k].row_begin,
        shards[k].row_end, b->labels, int(T), int(b->h));
    VP_KCHECK();
    ++c->launches;
    gemm_dw(c, st, b->X, b->ldx, gw[k], ldgw);
    segment_scatter(c, b->labels, T, shards[k].row_begin, shards[k].row_end,
                    static_cast<const __nv_bfloat16*>(b->X), b->ldx, b->h, -1.f, gw[k], ldgw, 1, kErrLabel);
  }
  loss_of(c, states, shards, n, out, b, loss);
  if (c->distributed()) {
    c->cm().all_reduce(gx, gx, size_t(T * b->h), vp::DType::F32, vp::RedOp::Sum, c->stream);
  } else {
    reduce_partials(c, partials.data(), n, T, b->h, b->h, gx, ldgx);
  }
}

// -----------------------------------------------------------------------------
// Vocabulary-pass executor: runs the S / C0 / C1 / T / C2
// passes of a reference DeviceProgram (P/include/vpipe/schedule.hpp:95-100) in
// program order on the GPU.  Transformer passes (F, B, IF, IB) belong to the
// caller and are skipped.  The dependency contract C0 -> S -> C1 -> T [-> C2]
// (P/src/schedule.cpp:339-366) is checked up front (validate_vocab); program
// order then IS a valid stream order, so S and T run on the compute stream in
// list order, and the heavy exchange of each barrier (the dX / loss
// all-reduce of C1 for Algorithm 2, of C2 for Algorithm 1) is forked onto the
// high-priority comm stream, where it overlaps the passes that follow ("T
// arbitrarily delayable", R/PAPER.md:243, :329).  dW of every microbatch
// accumulates into the shard's grad_w.
//   NCCL group (nranks == p): this rank executes device `rank`'s list.
//   Local: every device's list is executed on this GPU with one shard per
//   device, merged at the collectives (the reference's in-process devices).
void run_program(vp_ctx_s* c, const vp::Program& prog, const vp_batch_t* batches, const vp_shard_t* shards, int nsh,
                 const vp_state_t* states, vp_stats_t* stats, float* const* loss, float* const* gx, int64_t ldgx,
                 float* const* gw, int64_t ldgw) {
  require(prog.vocab, "vp_program_run: the program's method has no vocabulary passes");
  const int p = int(prog.p), n = int(prog.n);
  const bool dist = c->distributed();
  if (dist)
    require(c->nranks == p && nsh == 1, "vp_program_run: an NCCL group runs one program device per rank (nranks == p)");
  else
    require(nsh == p, "vp_program_run: a local run executes every program device (one shard per device)");
  require(nsh <= vp::kMaxLocalShards, "vp_program_run: too many local shards");
  require(batches && shards && states && stats && loss && gx && gw, "vp_program_run: null argument");
  {
    const auto v = vp::validate_vocab(prog);
    if (!v.empty()) throw std::invalid_argument("vp_program_run: program violates its dependencies: " + v.front());
  }
  // every device must issue the same collective sequence (NCCL call order;
  // the local merge point)
  std::vector<std::pair<int, int>> seq0;
  for (int d = 0; d < p; ++d) {
    std::vector<std::pair<int, int>> seq;
    for (const auto& ps : prog.order[size_t(d)])
      if (vp::is_collective(ps.kind)) seq.emplace_back(int(ps.kind), ps.microbatch);
    if (d == 0) seq0 = seq;
    else require(seq == seq0, "vp_program_run: devices disagree on the order of their collectives");
  }
  for (int i = 0; i < n; ++i) check_batch(&batches[i]);
  const bool alg2 = prog.barriers == 1;
  auto st = [&](int ls, int i) { return states[size_t(ls) * size_t(n) + size_t(i)]; };
  for (int ls = 0; ls < nsh; ++ls) {
    check_shard(&shards[ls], batches[0].h);
    check_grad_w(gw[ls], ldgw, batches[0].h, "vp_program_run: bad grad_w");
    const int64_t rows = shards[ls].row_end - shards[ls].row_begin;
    VP_CUDA(cudaMemsetAsync(gw[ls], 0, size_t(rows * ldgw) * sizeof(float), c->stream));
    for (int i = 0; i < n; ++i) check_state(st(ls, i), &batches[i], &shards[ls]);
  }
  const bool overlap = dist && c->overlap_c1 && c->comm_stream != nullptr;
  // Fused exchange (option "fused_c1"): one peer-buffer region per microbatch,
  // so S (alg2) / T (alg1) of several microbatches may precede their barriers
  std::vector<FusedLayout> FL;
  {
    bool fused = dist && c->fused_c1 && c->nranks <= vp::kMaxRoute && !c->sym.failed;
    for (int i = 0; fused && i < n; ++i) fused = batches[i].h % 8 == 0;
    if (fused) {
      require(shards[0].ldw % 8 == 0 && aligned16(shards[0].W),
              "fused_c1: the shard needs ldw % 8 == 0 and a 16-byte aligned W (or set fused_c1 = 0 on every rank)");
      size_t region = 0;
      const int64_t rows = shards[0].row_end - shards[0].row_begin;
      for (int i = 0; i < n; ++i)
        region = std::max(region, fused_layout(c, batches[i].n_tok, batches[i].h, rows).need);
      for (int i = 0; i < n; ++i)
        FL.push_back(fused_layout(c, batches[i].n_tok, batches[i].h, rows, size_t(i) * region));
      if (!ensure_sym(c, c->sym, size_t(n) * region)) FL.clear();
    }
  }
  const bool fused = !FL.empty();
  const bool acc0 = c->accumulate_dw;
  const int sms0 = c->gemm_sms;
  c->accumulate_dw = true;
  // the all-reduce path leaves comm_sms to NCCL during the overlap; the fused
  // exchange's gather runs on copy engines
  if (overlap && !fused) c->gemm_sms = std::max(2, (c->gemm_sms - c->comm_sms) / 2 * 2);
  auto restore = [&] {
    c->accumulate_dw = acc0;
    c->gemm_sms = sms0;
  };
  try {
    std::vector<int> devs;
    if (dist) devs.push_back(c->rank);
    else
      for (int d = 0; d < p; ++d) devs.push_back(d);
    std::vector<size_t> pos(devs.size(), 0);
    auto exec_local = [&](int d, const vp::PPass& ps) {  // S / T of device d
      const int ls = dist ? 0 : d, i = ps.microbatch;
      vp_state_s* s_ = st(ls, i);
      if (ps.kind == vp::PKind::S) {
        if (alg2 && fused) alg2_S_fused(c, &batches[i], &shards[ls], s_, FL[size_t(i)]);
        else if (alg2) alg2_S(c, &batches[i], &shards[ls], s_);
        else pass_S_common(c, &batches[i], &shards[ls], s_);
      } else if (alg2) {
        alg2_T(c, s_, stats[i], &batches[i], &shards[ls], gw[ls], ldgw);
      } else if (fused) {
        alg1_T_routed(c, s_, stats[i], &batches[i], &shards[ls], gw[ls], ldgw, FL[size_t(i)]);
      } else {
        // Algorithm 1: dX partial (local: the state's buffer; NCCL: grad_x, reduced by C2)
        alg1_T(c, s_, stats[i], &batches[i], &shards[ls], dist ? gx[i] : s_->A, dist ? ldgx : batches[i].h, gw[ls],
               ldgw);
      }
    };
    auto exec_collective = [&](vp::PKind k, int i) {
      std::vector<vp_state_t> sts(static_cast<size_t>(nsh));
      for (int ls = 0; ls < nsh; ++ls) sts[size_t(ls)] = st(ls, i);
      const vp_batch_t* b = &batches[i];
      const int64_t T = b->n_tok, h = b->h;
      if (k == vp::PKind::C0) {
        // broadcast of the last stage's output (X_i) to every device
        if (dist)
          c->cm().broadcast(b->X, const_cast<void*>(b->X), size_t((T - 1) * b->ldx + b->h), vp::DType::BF16, p - 1,
                            c->stream);  // the logical extent of X: (T-1) ldx + h elements
      } else if (k == vp::PKind::C1 && fused && alg2) {
        alg2_C1_fused(c, sts[0], shards, b, 1.0, stats[i], loss[i], gx[i], ldgx, FL[size_t(i)], overlap);
      } else if (k == vp::PKind::C2 && fused) {
        NvtxRange nr("vp:C2(fused)");
        group_barrier(c);  // every rank's routed stores and label rows of microbatch i have landed
        owner_combine_gather(c, shards, b, stats[i], true, gx[i], ldgx, FL[size_t(i)], overlap,
                             [&] { group_barrier(c); });
      } else if (k == vp::PKind::C1) {
        if (alg2) {
          alg2_C1(c, sts.data(), shards, nsh, b, 1.0, stats[i], gx[i], ldgx, /*reduce=*/!overlap);
          loss_of(c, sts.data(), shards, nsh, stats[i], b, loss[i], /*reduce=*/!overlap);
          if (overlap) {
            require(ldgx == h, "vp_program_run: grad_x must be dense (ldgx == h) for the all-reduce");
            fork_allreduces(c, gx[i], T * h, loss[i], T);
          }
        } else {
          merge_stats(c, sts.data(), nsh, 1.0, stats[i]);
          loss_of(c, sts.data(), shards, nsh, stats[i], b, loss[i]);
        }
      } else {  // C2 (Algorithm 1): grad_x = sum of the dX partials
        if (dist) {
          require(ldgx == h, "vp_program_run: grad_x must be dense (ldgx == h) for the all-reduce");
          if (overlap) {
            VP_CUDA(cudaEventRecord(c->ev_ready, c->stream));
            VP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
            c->cm().all_reduce(gx[i], gx[i], size_t(T * h), vp::DType::F32, vp::RedOp::Sum, c->comm_stream);
            VP_CUDA(cudaEventRecord(c->ev_done, c->comm_stream));
            c->reduce_pending = true;
          } else {
            c->cm().all_reduce(gx[i], gx[i], size_t(T * h), vp::DType::F32, vp::RedOp::Sum, c->stream);
          }
        } else {
          std::vector<float*> parts(static_cast<size_t>(nsh));
          for (int ls = 0; ls < nsh; ++ls) parts[size_t(ls)] = st(ls, i)->A;
          reduce_partials(c, parts.data(), nsh, T, h, h, gx[i], ldgx);
        }
      }
    };
    for (;;) {
      // run every executing device up to its next collective
      bool done = true;
      for (size_t e = 0; e < devs.size(); ++e) {
        const auto& list = prog.order[size_t(devs[e])];
        while (pos[e] < list.size()) {
          const vp::PPass& ps = list[pos[e]];
          if (!vp::is_vocab_pass(ps.kind)) {
            ++pos[e];
            continue;
          }
          if (vp::is_collective(ps.kind)) break;
          exec_local(devs[e], ps);
          ++pos[e];
        }
        if (pos[e] < list.size()) done = false;
      }
      if (done) break;
      // all executing devices now stand at the same collective (sequences agree)
      const vp::PPass& cp = prog.order[size_t(devs[0])][pos[0]];
      exec_collective(cp.kind, cp.microbatch);
      for (size_t e = 0; e < devs.size(); ++e) ++pos[e];
    }
  } catch (...) {
    restore();
    join_allreduces(c);
    throw;
  }
  restore();
  join_allreduces(c);
}

// Installs a communicator on a context: the comm stream / events of the
// barrier overlap, and, when several ranks share this GPU (loopback), a
// 1/colocated share of its SMs for the persistent GEMMs so the co-located
// grids fit side by side (their cross-CTA waits need every CTA resident).
void attach_comm(vp_ctx_s* c, std::unique_ptr<vp::Comm> comm) {
  c->nranks = comm->nranks;
  c->rank = comm->rank;
  const int share = comm->colocated();
  c->comm = std::move(comm);
  c->vocab_cache_key = -1;  // group-derived caches belong to the previous group
  c->bounds_key_rb = c->bounds_key_re = -1;
  if (share > 1 && !c->gemm_sms_set) c->gemm_sms = std::max(2, c->num_sms / share / 2 * 2);
  int lo = 0, hi = 0;
  VP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  VP_CUDA(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
  VP_CUDA(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  VP_CUDA(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
}

}  // namespace

struct vp_program_s {
  vp::Program prog;
};

struct vp_graph_s {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

// =============================================================================
extern "C" {

int vp_abi_version(void) { return VP_ABI_VERSION; }
const char* vp_last_error(void) { return g_last_error.c_str(); }

int vp_ctx_create(int device, vp_ctx_t* out) {
  return api([&] {
    require(out != nullptr, "vp_ctx_create: null output");
    int ndev = 0;
    VP_CUDA(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, "vp_ctx_create: bad device");
    auto* c = new vp_ctx_s();
    c->device = device;
    try {
      c->activate();
      cudaDeviceProp prop;
      VP_CUDA(cudaGetDeviceProperties(&prop, device));
      if (prop.major != 10) throw std::invalid_argument("vp_ctx_create: this library targets sm_100a (B200)");
      c->num_sms = prop.multiProcessorCount;
      c->gemm_sms = c->num_sms;
      c->persist_max = std::min<size_t>(size_t(prop.persistingL2CacheMaxSize), size_t(prop.accessPolicyMaxWindowSize));
      VP_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
      c->stream = c->own_stream;
      VP_CUDA(cudaMalloc(&c->d_err, sizeof(int)));
      VP_CUDA(cudaMemset(c->d_err, 0, sizeof(int)));
      // Under Nsight Compute / Systems (they set NV_NSIGHT_INJECTION_* in the
      // target) launch the GEMMs non-cooperatively: ncu's kernel replay cannot
      // relaunch cooperative grids.  The kernels are identical; only the
      // co-residency guarantee against other streams' kernels is dropped while
      // profiling.
      if (std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||
          std::getenv("CUDA_INJECTION64_PATH") != nullptr)
        vp::g_cooperative = 0;
      c->lock.capacity = int64_t(1) << 20;
      VP_CUDA(cudaMalloc(&c->lock.counters, size_t(c->lock.capacity) * sizeof(int)));
      c->split.max_tiles = 1 << 14;
      VP_CUDA(cudaMalloc(&c->split.flags, size_t(2 * c->split.max_tiles) * sizeof(int)));
      VP_CUDA(cudaMemset(c->split.flags, 0, size_t(2 * c->split.max_tiles) * sizeof(int)));
      // parallel split-K workspace: S * tiles <= one wave of CTA pairs, each
      // tile <= 256 x 512 fp32 (+ row padding slack)
      c->split.ws_elems = size_t(c->num_sms / 2 + 2) * 256 * 512 + (size_t(1) << 16);
      VP_CUDA(cudaMalloc(&c->split.ws, c->split.ws_elems * sizeof(float)));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int vp_ctx_destroy(vp_ctx_t c) {
  return api([&] {
    if (!c) return;
    c->activate();
    cudaStreamSynchronize(c->stream);
    for (SymBuf* sb : {&c->sym, &c->in_sym, &c->bwd_sym}) {
      if (c->comm) {
        c->comm->close_peers(sb->peers);
        for (auto& r : sb->retired) c->comm->close_peers(r.second);
      }
      if (sb->p) cudaFree(sb->p);
      for (auto& r : sb->retired) cudaFree(r.first);
    }
    c->bar.release();

    c->comm.reset();
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->ev_ready) cudaEventDestroy(c->ev_ready);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (DevBuf* b : {&c->inv, &c->scale, &c->xs, &c->gathered, &c->packed, &c->tmp_m, &c->tmp_s,
                      &c->heads, &c->counts, &c->vtmp, &c->gbuf})
      b->release();
    if (c->d_err) cudaFree(c->d_err);
    if (c->split.flags) cudaFree(c->split.flags);
    if (c->split.ws) cudaFree(c->split.ws);
    if (c->lock.counters) cudaFree(c->lock.counters);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
  });
}

int vp_ctx_set_stream(vp_ctx_t c, void* stream) {
  return api([&] {
    require(c != nullptr, "vp_ctx_set_stream: null context");
    c->stream = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
  });
}

void* vp_ctx_get_stream(vp_ctx_t c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int vp_ctx_sync(vp_ctx_t c) {
  return api([&] {
    require(c != nullptr, "vp_ctx_sync: null context");
    c->activate();
    VP_CUDA(cudaStreamSynchronize(c->stream));
    int err = 0;
    VP_CUDA(cudaMemcpy(&err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      VP_CUDA(cudaMemset(c->d_err, 0, sizeof(int)));
      if (err & kErrLabel) throw std::invalid_argument("TokenBatch: label out of range");
      if (err & kErrInputFwd) throw std::invalid_argument("input_forward: token out of range");
      throw std::invalid_argument("input_backward: token out of range");
    }
  });
}

int vp_workspace_query(int64_t n_tok, int64_t h, int64_t rows, int nranks, int64_t* state_b, int64_t* ctx_b,
                       int64_t* peer_b) {
  return api([&] {
    require(n_tok >= 1 && h >= 1 && rows >= 1 && nranks >= 1, "vp_workspace_query: empty shape");
    if (state_b) *state_b = state_bytes(n_tok, h, rows);
    if (ctx_b) {
      const int64_t nchunks = ceil_div(h, vp::kScChunk), hot_cap = ceil_div(n_tok, vp::kScHot) * nchunks;
      const int64_t fixed = (int64_t(1) << 20) * 4                         // lockstep counters
                            + 2 * (int64_t(1) << 14) * 4                   // split-K flags
                            + (int64_t(148 / 2 + 2) * 256 * 512 + (1 << 16)) * 4;  // split-K workspace
      *ctx_b = fixed + 4 * n_tok * 4 + n_tok * h * 2 + 2 * n_tok * 4 + 2 * n_tok * nranks * 4  // reserve()
               + (4 * rows + vp::kScCtrs) * 4 + (11 * n_tok + 4 * hot_cap + 4) * 4;           // scatter
    }
    if (peer_b) {
      *peer_b = 0;
      if (nranks > 1) {  // fused exchange (output layer) + input-layer peer buffers
        const int64_t R = round_up(ceil_div(n_tok, nranks), 32), rowf = R * h;
        // (two split-K slots per rank: the split the routed dX GEMM takes at the headline shapes)
        const int64_t out = round_up(int64_t(nranks) * 2 * rowf * 4 + round_up(rowf * 2, 256) + rowf * 4, 256);
        const int64_t inl = 2 * round_up(n_tok * h * 2, 256);
        *peer_b = round_up(out, int64_t(2) << 20) + 2 * round_up(inl, int64_t(2) << 20);
      }
    }
  });
}

int vp_ctx_reserve(vp_ctx_t c, int64_t n_tok, int64_t h, int p) {
  return api([&] {
    require(c != nullptr && n_tok >= 1 && h >= 1 && p >= 1, "vp_ctx_reserve: bad arguments");
    c->activate();
    c->buf<float>(c->inv, size_t(n_tok));
    c->buf<float>(c->scale, size_t(n_tok));
    c->buf<float>(c->tmp_m, size_t(n_tok));
    c->buf<float>(c->tmp_s, size_t(n_tok));
    c->buf<__nv_bfloat16>(c->xs, size_t(n_tok * h));
    c->buf<float>(c->packed, size_t(2 * n_tok));
    c->buf<float>(c->gathered, size_t(2 * n_tok * std::max(p, c->nranks)));
  });
}

int vp_ctx_set_option(vp_ctx_t c, const char* key, int64_t value) {
  return api([&] {
    require(c != nullptr && key != nullptr, "vp_ctx_set_option: null argument");
    const std::string k(key);
    if (k == "cta_group") {
      require(value == 1 || value == 2, "vp_ctx_set_option: cta_group must be 1 or 2");
      c->cg = int(value);
    } else if (k.rfind("raster_", 0) == 0 || k.rfind("policy_", 0) == 0) {
      const std::string which = k.substr(7);
      const int idx = which == "logits" ? 0 : which == "dx" ? 1 : which == "dw" ? 2 : -1;
      require(idx >= 0, "vp_ctx_set_option: raster_/policy_ suffix must be logits, dx or dw");
      if (k[0] == 'r') c->raster[idx] = int(value);
      else {
        require(value >= -1 && value <= 2, "vp_ctx_set_option: policy must be -1..2");
        c->pol[idx] = int(value);
      }
    } else if (k.rfind("policyb_", 0) == 0) {
      const std::string which = k.substr(8);
      const int idx = which == "logits" ? 0 : which == "dx" ? 1 : which == "dw" ? 2 : -1;
      require(idx >= 0, "vp_ctx_set_option: policyb_ suffix must be logits, dx or dw");
      require(value >= -1 && value <= 2, "vp_ctx_set_option: policy must be -1..2");
      c->polb[idx] = int(value);
    } else if (k == "nh_logits" || k == "nh_dx" || k == "nh_dw") {
      require(value == 1 || value == 2, "vp_ctx_set_option: nh must be 1 or 2");
      require(value == 1 || c->cg == 2, "vp_ctx_set_option: 512-wide tiles need cta_group 2");
      c->nh[k == "nh_logits" ? 0 : k == "nh_dx" ? 1 : 2] = int(value);
    } else if (k == "accumulate_grad_w") {
      c->accumulate_dw = value != 0;
    } else if (k == "persist_logits" || k == "persist_dw") {
      require(value == 0 || value == 1, "vp_ctx_set_option: persist_* must be 0 or 1");
      c->persist[k == "persist_logits" ? 0 : 2] = int(value);
    } else if (k == "peer_input") {
      require(value == 0 || value == 1, "vp_ctx_set_option: peer_input must be 0 or 1");
      c->peer_input = value != 0;
    } else if (k == "fused_c1") {
      require(value == 0 || value == 1, "vp_ctx_set_option: fused_c1 must be 0 or 1");
      c->fused_c1 = value != 0;
    } else if (k == "overlap_c1") {
      c->overlap_c1 = value != 0;
    } else if (k == "comm_sms") {
      require(value >= 1 && value <= 64, "vp_ctx_set_option: comm_sms must be 1..64");
      require(c->comm == nullptr, "vp_ctx_set_option: comm_sms must be set before vp_ctx_comm_init");
      c->comm_sms = int(value);
    } else if (k == "lockstep_logits" || k == "lockstep_dx" || k == "lockstep_dw") {
      require(value >= 0 && value <= 4096, "vp_ctx_set_option: lockstep epoch must be in 0..4096 k-blocks");
      c->lock_epoch[k == "lockstep_logits" ? 0 : k == "lockstep_dx" ? 1 : 2] = int(value);
    } else if (k == "l2_promotion") {
      require(value >= 0 && value <= 3, "vp_ctx_set_option: l2_promotion must be 0..3");
      vp::g_l2_promotion = int(value);
    } else if (k == "cooperative") {
      require(value == 0 || value == 1, "vp_ctx_set_option: cooperative must be 0 or 1");
      vp::g_cooperative = int(value);
    } else if (k == "store_evict_first") {
      require(value == 0 || value == 1, "vp_ctx_set_option: store_evict_first must be 0 or 1");
      vp::g_store_evict_first = int(value);
    } else if (k == "store_hint_logits" || k == "store_hint_dx" || k == "store_hint_dw") {
      require(value >= -1 && value <= 1, "vp_ctx_set_option: store_hint_* must be -1, 0 or 1");
      c->store_hint[k == "store_hint_logits" ? 0 : k == "store_hint_dx" ? 1 : 2] = int(value);
    } else if (k == "splits_dx" || k == "splits_dw") {
      require(value >= 0 && value <= 32, "vp_ctx_set_option: splits_dx / splits_dw must be in 0..32");
      (k == "splits_dx" ? c->splits_dx : c->splits_dw) = int(value);
    } else if (k == "split_workspace") {
      require(value >= 0 && value <= 2, "vp_ctx_set_option: split_workspace must be 0, 1 or 2");
      c->split.ws_mode = int(value);
    } else if (k == "split_min_kb") {
      require(value >= 1 && value <= 4096, "vp_ctx_set_option: split_min_kb must be in 1..4096");
      c->split.min_kb = int(value);
    } else if (k == "tma_store") {
      require(value == 0 || value == 1, "vp_ctx_set_option: tma_store must be 0 or 1");
      vp::g_tma_store = int(value);
    } else if (k == "epi_wait") {
      require(value == 0 || value == 1, "vp_ctx_set_option: epi_wait must be 0 or 1");
      vp::g_epi_wait = int(value);
    } else if (k == "debug_logit_scale_ppm") {
      // fault injection (verification tools): K1 logits scaled by 1 + ppm * 1e-6
      require(value > -1000000 && value <= 1000000, "vp_ctx_set_option: debug_logit_scale_ppm out of range");
      c->logit_scale = float(1.0 + double(value) * 1e-6);
    } else if (k == "force_collectives") {
      c->force_collectives = value != 0;
    } else if (k == "multicast") {
      require(value == 1 || value == 2, "vp_ctx_set_option: multicast must be 1 or 2");
      require(value == 1 || c->cg == 2, "vp_ctx_set_option: multicast needs cta_group 2");
      c->mc = int(value);
    } else if (k == "gemm_sms") {
      require(value >= 2 && value <= c->num_sms, "vp_ctx_set_option: gemm_sms out of range");
      c->gemm_sms = int(value);
      c->gemm_sms_set = true;
    } else {
      throw std::invalid_argument("vp_ctx_set_option: unknown option " + k);
    }
  });
}

int64_t vp_ctx_launch_count(vp_ctx_t c) { return c ? c->launches : -1; }
int64_t vp_ctx_fused_c1_count(vp_ctx_t c) { return c ? c->fused_count : -1; }
int64_t vp_ctx_peer_input_count(vp_ctx_t c) { return c ? c->peer_input_count : -1; }

int vp_ctx_set_logit_shift(vp_ctx_t c, const float* shift) {
  return api([&] {
    require(c != nullptr, "vp_ctx_set_logit_shift: null context");
    c->logit_shift = shift;
  });
}

int vp_ctx_gemm_timing(vp_ctx_t c, int enable, double* ms_out, int64_t* count_out) {
  return api([&] {
    require(c != nullptr, "vp_ctx_gemm_timing: null context");
    c->activate();
    if (!c->ev_pending.empty()) {
      VP_CUDA(cudaStreamSynchronize(c->stream));
      for (auto& p : c->ev_pending) {
        float ms = 0.f;
        VP_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
        c->gemm_ms[p.first] += ms;
        c->gemm_n[p.first] += 1;
      }
      c->ev_pending.clear();
    }
    c->ev_next = 0;
    for (int k = 0; k < 4; ++k) {
      if (ms_out) ms_out[k] = c->gemm_ms[k];
      if (count_out) count_out[k] = c->gemm_n[k];
      c->gemm_ms[k] = 0.0;
      c->gemm_n[k] = 0;
    }
    c->timing = enable != 0;
  });
}

int vp_comm_unique_id(void* id128) {
  return api([&] {
    require(id128 != nullptr, "vp_comm_unique_id: null output");
    ncclUniqueId id;
    VP_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, sizeof(id));
  });
}

int vp_comm_loopback_id(void* id128) {
  return api([&] {
    require(id128 != nullptr, "vp_comm_loopback_id: null output");
    vp::make_loopback_id(id128);
  });
}

int vp_ctx_comm_init(vp_ctx_t c, int nranks, int rank, const void* id128) {
  return api([&] {
    require(c != nullptr && id128 != nullptr, "vp_ctx_comm_init: null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "vp_ctx_comm_init: bad rank");
    require(c->comm == nullptr, "vp_ctx_comm_init: already initialised");
    c->activate();
    attach_comm(c, vp::is_loopback_id(id128) ? vp::make_loopback_comm(nranks, rank, id128, c->device)
                                              : vp::make_nccl_comm(nranks, rank, id128, c->comm_sms));
  });
}

int vp_comm_init_all(vp_ctx_t* ctxs, int n) {
  return api([&] {
    require(ctxs != nullptr && n >= 1, "vp_comm_init_all: no contexts");
    std::vector<int> devs;
    for (int k = 0; k < n; ++k) {
      require(ctxs[k] != nullptr, "vp_comm_init_all: null context");
      require(ctxs[k]->comm == nullptr, "vp_ctx_comm_init: already initialised");
      devs.push_back(ctxs[k]->device);
    }
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    std::vector<std::unique_ptr<vp::Comm>> comms(static_cast<size_t>(n));
    if (distinct) {
      // one NCCL rank per GPU, created from this thread in one group (the
      // ncclCommInitAll pattern, with each rank's maxCTAs config)
      ncclUniqueId id;
      VP_NCCL(ncclGetUniqueId(&id));
      std::vector<ncclComm_t> raw(static_cast<size_t>(n), nullptr);
      VP_NCCL(ncclGroupStart());
      for (int k = 0; k < n; ++k) {
        ctxs[k]->activate();
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.maxCTAs = ctxs[k]->comm_sms;
        const ncclResult_t r = ncclCommInitRankConfig(&raw[size_t(k)], n, id, k, &cfg);
        if (r != ncclSuccess) {
          ncclGroupEnd();
          throw NcclError(std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r));
        }
      }
      VP_NCCL(ncclGroupEnd());
      for (int k = 0; k < n; ++k) comms[size_t(k)] = vp::wrap_nccl_comm(raw[size_t(k)], n, k);
    } else {
      // ranks sharing a GPU: the loopback backend (its join is a rendezvous,
      // so every rank joins from its own thread)
      char id[128];
      vp::make_loopback_id(id);
      std::vector<std::string> errs(static_cast<size_t>(n));
      std::vector<std::thread> th;
      for (int k = 0; k < n; ++k)
        th.emplace_back([&, k] {
          try {
            ctxs[k]->activate();
            comms[size_t(k)] = vp::make_loopback_comm(n, k, id, ctxs[k]->device);
          } catch (const std::exception& e) {
            errs[size_t(k)] = e.what();
          }
        });
      for (auto& t : th) t.join();
      for (const auto& e : errs)
        if (!e.empty()) throw NcclError("vp_comm_init_all: " + e);
    }
    for (int k = 0; k < n; ++k) {
      ctxs[k]->activate();
      attach_comm(ctxs[k], std::move(comms[size_t(k)]));
    }
  });
}

const char* vp_ctx_comm_backend(vp_ctx_t c) {
  if (c == nullptr) return "";
  return c->comm ? c->comm->backend() : "none";
}

int vp_ctx_comm_info(vp_ctx_t c, int* nranks, int* rank) {
  return api([&] {
    require(c != nullptr, "vp_ctx_comm_info: null context");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
  });
}

int vp_state_create(vp_ctx_t c, int64_t n_tok, int64_t h, int64_t rows, vp_state_t* out) {
  return api([&] {
    require(c != nullptr && out != nullptr, "vp_state_create: null argument");
    require(n_tok >= 1 && h >= 1 && rows >= 1, "vp_state_create: empty shape");
    require(h % 8 == 0, "vp_state_create: h must be a multiple of 8");
    c->activate();
    auto* st = new vp_state_s();
    st->ctx = c;
    st->n_tok = n_tok;
    st->h = h;
    st->rows = rows;
    st->ldp = round_up(rows, 64);
    st->ntiles = ceil_div(rows, vp::kTileN);
    try {
      VP_CUDA(cudaMalloc(&st->P, size_t(n_tok * st->ldp) * sizeof(__nv_bfloat16)));
      VP_CUDA(cudaMalloc(&st->tile_m, size_t(st->ntiles * n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->tile_s, size_t(st->ntiles * n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->m_loc, size_t(n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->s_loc, size_t(n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->ytgt, size_t(n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->A, size_t(n_tok * h) * sizeof(float)));
      st->nblk128 = ceil_div(n_tok, 128) + 2;
      VP_CUDA(cudaMalloc(&st->tile_q, size_t(st->ntiles * n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->row_ref, size_t(n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->cfac, size_t(n_tok) * sizeof(float)));
      VP_CUDA(cudaMalloc(&st->ref_flag, size_t(st->nblk128) * sizeof(int)));
      VP_CUDA(cudaMalloc(&st->row_bad, size_t(n_tok) * sizeof(int)));
      VP_CUDA(cudaMalloc(&st->bad_list, size_t(n_tok) * sizeof(int)));
      VP_CUDA(cudaMalloc(&st->counters, 2 * sizeof(int)));
      VP_CUDA(cudaMalloc(&st->fix_list, size_t(ceil_div(n_tok, 32) * st->ntiles) * sizeof(int2)));
      VP_CUDA(cudaMemset(st->ytgt, 0, size_t(n_tok) * sizeof(float)));
    } catch (...) {
      free_state_buffers(st);
      delete st;
      throw;
    }
    *out = st;
  });
}

int vp_state_destroy(vp_state_t st) {
  return api([&] {
    if (!st) return;
    st->ctx->activate();
    cudaStreamSynchronize(st->ctx->stream);
    free_state_buffers(st);
    delete st;
  });
}

int vp_state_local_stats(vp_state_t st, const float** m_local, const float** sum_local) {
  return api([&] {
    require(st != nullptr, "vp_state_local_stats: null state");
    if (m_local) *m_local = st->m_loc;
    if (sum_local) *sum_local = st->s_loc;
  });
}

int vp_state_grad_terms(vp_state_t st, const float** A, int64_t* lda) {
  return api([&] {
    require(st != nullptr, "vp_state_grad_terms: null state");
    require(st->has_grad_terms, "alg2_barrier_C1: A/B terms missing");
    if (A) *A = st->A;
    if (lda) *lda = st->h;
  });
}

int vp_state_copy_local_stats(vp_ctx_t c, vp_state_t st, float* m_out, float* sum_out) {
  return api([&] {
    require(c != nullptr && st != nullptr, "vp_state_copy_local_stats: null argument");
    require(st->has_S, "vp_state_copy_local_stats: state has no pass-S output");
    c->activate();
    const size_t bytes = size_t(st->n_tok) * sizeof(float);
    if (m_out) VP_CUDA(cudaMemcpyAsync(m_out, st->m_loc, bytes, cudaMemcpyDeviceToDevice, c->stream));
    if (sum_out) VP_CUDA(cudaMemcpyAsync(sum_out, st->s_loc, bytes, cudaMemcpyDeviceToDevice, c->stream));
  });
}

int vp_state_copy_grad_terms(vp_ctx_t c, vp_state_t st, float* A_out, int64_t ldo) {
  return api([&] {
    require(c != nullptr && st != nullptr && A_out != nullptr, "vp_state_copy_grad_terms: null argument");
    require(st->has_grad_terms, "alg2_barrier_C1: A/B terms missing");
    require(ldo >= st->h, "vp_state_copy_grad_terms: ldo < h");
    c->activate();
    VP_CUDA(cudaMemcpy2DAsync(A_out, size_t(ldo) * sizeof(float), st->A, size_t(st->h) * sizeof(float),
                              size_t(st->h) * sizeof(float), size_t(st->n_tok), cudaMemcpyDeviceToDevice, c->stream));
  });
}

int vp_alg1_pass_S(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* s, vp_state_t st) {
  return api([&] {
    require(c != nullptr, "alg1_pass_S: null context");
    c->activate();
    pass_S_common(c, b, s, st);
  });
}

int vp_alg2_pass_S(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* s, vp_state_t st) {
  return api([&] {
    require(c != nullptr, "alg2_pass_S: null context");
    c->activate();
    alg2_S(c, b, s, st);
  });
}

int vp_merge_max_sum(vp_ctx_t c, const vp_state_t* states, int n, double fault_scale, vp_stats_t out) {
  return api([&] {
    require(c != nullptr, "merge_max_sum: null context");
    c->activate();
    merge_stats(c, states, n, fault_scale, out);
  });
}

int vp_merge_stats_raw(vp_ctx_t c, const float* m_parts, const float* s_parts, int p, int64_t n, int64_t ld,
                       double fault_scale, vp_stats_t out) {
  return api([&] {
    require(c != nullptr, "merge_max_sum: null context");
    require(p >= 1 && m_parts != nullptr && s_parts != nullptr, "merge_max_sum: empty input");
    require(n >= 1 && ld >= n, "merge_max_sum: length mismatch");
    require(out.m != nullptr && out.sum != nullptr, "merge_max_sum: null output");
    c->activate();
    vp::k_merge_stats<<<unsigned(ceil_div(n, 256)), 256, 0, c->stream>>>(m_parts, s_parts, p, ld, int(n),
                                                                        float(fault_scale), out.m, out.sum);
    VP_KCHECK();
    ++c->launches;
  });
}

int vp_alg1_pass_T(vp_ctx_t c, vp_state_t st, vp_stats_t stats, const vp_batch_t* b, const vp_shard_t* s,
                   float* gx, int64_t ldgx, float* gw, int64_t ldgw) {
  return api([&] {
    require(c != nullptr, "alg1_pass_T: null context");
    require(gx != nullptr && gw != nullptr, "alg1_pass_T: null gradient buffer");
    c->activate();
    alg1_T(c, st, stats, b, s, gx, ldgx, gw, ldgw);
  });
}

int vp_reduce_grad_x(vp_ctx_t c, float* const* partials, int n, int64_t n_tok, int64_t h, int64_t ld, float* gx,
                     int64_t ldgx) {
  return api([&] {
    require(c != nullptr && partials != nullptr && gx != nullptr, "reduce_grad_x: null argument");
    c->activate();
    reduce_partials(c, partials, n, n_tok, h, ld, gx, ldgx);
  });
}

int vp_alg2_barrier_C1(vp_ctx_t c, const vp_state_t* states, const vp_shard_t* shards, int n, const vp_batch_t* b,
                       double fault_scale, vp_stats_t out, float* gx, int64_t ldgx) {
  return api([&] {
    require(c != nullptr, "alg2_barrier_C1: null context");
    require(n <= vp::kMaxLocalShards, "alg2_barrier_C1: too many local shards");
    require(!c->distributed() || n == 1, "alg2_barrier_C1: one state per rank in an NCCL group");
    c->activate();
    alg2_C1(c, states, shards, n, b, fault_scale, out, gx, ldgx);
  });
}

int vp_alg2_pass_T(vp_ctx_t c, vp_state_t st, vp_stats_t stats, const vp_batch_t* b, const vp_shard_t* s,
                   float* gw, int64_t ldgw) {
  return api([&] {
    require(c != nullptr && gw != nullptr, "alg2_pass_T: null argument");
    c->activate();
    alg2_T(c, st, stats, b, s, gw, ldgw);
  });
}

int vp_output_loss(vp_ctx_t c, const vp_state_t* states, const vp_shard_t* shards, int n, vp_stats_t stats,
                   const vp_batch_t* b, float* loss) {
  return api([&] {
    require(c != nullptr && states != nullptr && shards != nullptr, "loss: null argument");
    c->activate();
    check_batch(b);
    loss_of(c, states, shards, n, stats, b, loss);
  });
}

int vp_shard_softmax(vp_ctx_t c, vp_state_t st, vp_stats_t g, float* out, int64_t ldo) {
  return api([&] {
    require(c != nullptr && st != nullptr && out != nullptr, "softmax: null argument");
    require(st->has_S, "softmax: state has no pass-S output");
    require(ldo >= st->rows, "softmax: ldo < rows");
    c->activate();
    const float* tile_m = nullptr;
    const float* mref = nullptr;
    const float* mul = nullptr;
    if (st->form == kLocal) {  // P = softmax':  softmax = P * global_scale
      mul = global_scale(c, st, g);
    } else {  // kGlobal: P already is the softmax
      float* ones = c->buf<float>(c->tmp_m, size_t(st->n_tok));
      std::vector<float> h(size_t(st->n_tok), 1.f);
      VP_CUDA(cudaMemcpyAsync(ones, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      VP_CUDA(cudaStreamSynchronize(c->stream));
      mul = ones;
    }
    vp::k_materialize<<<c->grid_for(st->n_tok * st->rows, 256), 256, 0, c->stream>>>(
        st->P, st->ldp, int(st->n_tok), int(st->rows), tile_m, st->n_tok, mref, mul, out, ldo);
    VP_KCHECK();
    ++c->launches;
  });
}

int vp_shard_logits(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* s, float* out, int64_t ldo) {
  return api([&] {
    require(c != nullptr && out != nullptr, "logits: null argument");
    check_batch(b, false);
    check_shard(s, b->h);
    const int64_t rows = s->row_end - s->row_begin;
    require(ldo >= rows, "logits: ldo < rows");
    c->activate();
    vp::EpiStoreF32::Params ep{out, ldo, nullptr, 0, nullptr};
    timed_gemm(c, 1, [&] {
      vp::launch_gemm<vp::EpiStoreF32>(c->cg, {b->X, b->ldx, false}, {s->W, s->ldw, false}, int(b->n_tok), int(rows),
                                       int(b->h), c->raster[0], ep, c->gemm_sms, c->stream, c->pol[0], c->pol[0],
                                       c->eff_mc(0));
    });
    ++c->launches;
  });
}

int vp_shard_label_rows(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* s, float* out, int64_t ldo) {
  return api([&] {
    require(c != nullptr && out != nullptr, "label rows: null argument");
    check_batch(b);
    check_shard(s, b->h);
    require(ldo >= b->h, "label rows: ldo < h");
    c->activate();
    vp::k_label_rows<<<c->grid_for(b->n_tok * b->h / 2, 256), 256, 0, c->stream>>>(
        static_cast<const __nv_bfloat16*>(s->W), s->ldw, s->row_begin, s->row_end, b->labels, int(b->n_tok),
        int(b->h), out, ldo);
    VP_KCHECK();
    ++c->launches;
  });
}

int vp_naive_partitioned_output(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* shards, const vp_state_t* states,
                                int n, vp_stats_t out, float* loss, float* gx, int64_t ldgx, float* const* gw,
                                int64_t ldgw) {
  return api([&] {
    require(c != nullptr && gx != nullptr && gw != nullptr && loss != nullptr, "naive: null argument");
    c->activate();
    naive(c, b, shards, states, n, out, loss, gx, ldgx, gw, ldgw);
  });
}

int vp_run_alg1(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* shards, const vp_state_t* states, int n,
                double fault_scale, vp_stats_t out, float* loss, float* gx, int64_t ldgx, float* const* gw,
                int64_t ldgw) {
  return api([&] {
    require(c != nullptr && gx != nullptr && gw != nullptr && loss != nullptr, "run_alg1: null argument");
    c->activate();
    run_alg(1, c, b, shards, states, n, fault_scale, out, loss, gx, ldgx, gw, ldgw);
  });
}

int vp_run_alg2(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* shards, const vp_state_t* states, int n,
                double fault_scale, vp_stats_t out, float* loss, float* gx, int64_t ldgx, float* const* gw,
                int64_t ldgw) {
  return api([&] {
    require(c != nullptr && gx != nullptr && gw != nullptr && loss != nullptr, "run_alg2: null argument");
    c->activate();
    run_alg(2, c, b, shards, states, n, fault_scale, out, loss, gx, ldgx, gw, ldgw);
  });
}

// Memory-bounded Algorithm 2 (SURVEY §8f-2, R/PAPER.md:498): softmax rows
// are independent, so the batch runs as consecutive token chunks of at most
// chunk_tokens rows through S -> C1 -> T, reusing states sized for one chunk
// (P is chunk_tokens x V_k instead of n_tok x V_k); dW accumulates over the
// chunks.  Per chunk the exchanges are the same as vp_run_alg2's.
int vp_run_alg2_chunked(vp_ctx_t c, const vp_batch_t* b, const vp_shard_t* shards, const vp_state_t* states, int n,
                        int64_t chunk_tokens, double fault_scale, vp_stats_t out, float* loss, float* gx, int64_t ldgx,
                        float* const* gw, int64_t ldgw) {
  return api([&] {
    require(c != nullptr && gx != nullptr && gw != nullptr && loss != nullptr, "run_alg2: null argument");
    require(out.m != nullptr && out.sum != nullptr, "run_alg2: null argument");
    check_batch(b);
    require(chunk_tokens >= 1, "run_alg2_chunked: chunk_tokens must be >= 1");
    require(n >= 1 && n <= vp::kMaxLocalShards && states != nullptr, "run: bad shard count");
    for (int k = 0; k < n; ++k)
      require(states[k] != nullptr && states[k]->n_tok == std::min(chunk_tokens, b->n_tok),
              "run_alg2_chunked: states must be created for min(chunk_tokens, n_tok) tokens");
    c->activate();
    const int64_t cap = states[0]->n_tok;
    const bool acc0 = c->accumulate_dw;
    struct Restore {
      vp_ctx_s* c;
      const vp_state_t* st;
      int n;
      int64_t cap;
      bool acc0;
      ~Restore() {
        c->accumulate_dw = acc0;
        for (int k = 0; k < n; ++k) st[k]->n_tok = cap;
      }
    } restore{c, states, n, cap, acc0};
    for (int64_t t0 = 0; t0 < b->n_tok; t0 += cap) {
      const int64_t rows = std::min(cap, b->n_tok - t0);
      vp_batch_t bc = *b;
      bc.X = static_cast<const __nv_bfloat16*>(b->X) + t0 * b->ldx;
      bc.labels = b->labels + t0;
      bc.n_tok = rows;
      // a ragged last chunk: the state's kernels index with n_tok as the
      // leading dimension of its tile stats, so a smaller n_tok stays consistent
      for (int k = 0; k < n; ++k) states[k]->n_tok = rows;
      c->accumulate_dw = acc0 || t0 > 0;
      const vp_stats_t oc{out.m + t0, out.sum + t0};
      run_alg(2, c, &bc, shards, states, n, fault_scale, oc, loss + t0, gx + t0 * ldgx, ldgx, gw, ldgw);
    }
  });
}

namespace {
// One block per SM (the whole shared memory), spinning on the global timer:
// stands in for NCCL's kernels holding SMs during the overlapped exchanges.
__global__ void k_occupy(unsigned long long ns) {
  extern __shared__ uint8_t pad[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) pad[0] = uint8_t(t);
  } while (t - t0 < ns);
}
}  // namespace

int vp_debug_occupy_sms(vp_ctx_t c, void* stream, int nsms, int64_t microseconds) {
  return api([&] {
    require(c != nullptr && nsms >= 1 && nsms <= c->num_sms && microseconds >= 0,
            "debug_occupy_sms: bad arguments");
    c->activate();
    int smem = 0;
    VP_CUDA(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    VP_CUDA(cudaFuncSetAttribute(k_occupy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_occupy<<<nsms, 32, size_t(smem), static_cast<cudaStream_t>(stream)>>>(
        static_cast<unsigned long long>(microseconds) * 1000ull);
    VP_KCHECK();
  });
}

int vp_input_forward(vp_ctx_t c, const int64_t* tokens, int64_t n_tok, int64_t h, const vp_shard_t* s, void* out,
                     int64_t ldo, int accumulate) {
  return api([&] {
    require(c != nullptr && out != nullptr && tokens != nullptr, "input_forward: null argument");
    require(n_tok >= 0, "input_forward: negative token count");
    check_shard(s, h);
    require(h % 8 == 0 && ldo >= h && ldo % 8 == 0 && aligned16(out), "input_forward: h/ldo must be multiples of 8");
    if (n_tok == 0) return;
    c->activate();
    NvtxRange nr("vp:input_forward");
    vp::k_input_forward<<<c->grid_for(n_tok, 8), 256, 0, c->stream>>>(
        tokens, int(n_tok), static_cast<const __nv_bfloat16*>(s->W), s->ldw, s->row_begin, s->row_end, int(h),
        static_cast<__nv_bfloat16*>(out), ldo, accumulate, c->d_err);
    VP_KCHECK();
    ++c->launches;
  });
}

int vp_input_backward(vp_ctx_t c, const void* grad, int64_t ldg, int grad_is_f32, const int64_t* tokens,
                      int64_t n_tok, int64_t h, const vp_shard_t* s, float* gw, int64_t ldgw, int accumulate) {
  return api([&] {
    require(c != nullptr && gw != nullptr && tokens != nullptr && grad != nullptr, "input_backward: null argument");
    require(n_tok >= 0, "input_backward: grad/token length mismatch");
    check_shard(s, h);
    require(h % 8 == 0 && ldg >= h && ldg % 8 == 0 && ldgw >= h && ldgw % 4 == 0 && aligned16(gw) && aligned16(grad),
            "input_backward: h/ld must be multiples of 8");
    c->activate();
    NvtxRange nr("vp:input_backward");
    const int64_t rows = s->row_end - s->row_begin;
    if (!accumulate) {
      VP_CUDA(cudaMemset2DAsync(gw, size_t(ldgw) * sizeof(float), 0, size_t(h) * sizeof(float), size_t(rows),
                                c->stream));
    }
    if (n_tok == 0) return;
    if (grad_is_f32)
      segment_scatter(c, tokens, n_tok, s->row_begin, s->row_end, static_cast<const float*>(grad), ldg, h, 1.f, gw, ldgw,
                      1, kErrInputBwd);
    else
      segment_scatter(c, tokens, n_tok, s->row_begin, s->row_end, static_cast<const __nv_bfloat16*>(grad), ldg, h, 1.f,
                      gw, ldgw, 1, kErrInputBwd);
  });
}


int vp_input_forward_gathered(vp_ctx_t c, const int64_t* tokens, int64_t n_tok, int64_t h, const vp_shard_t* s,
                              void* out, int64_t ldo) {
  return api([&] {
    require(c != nullptr && out != nullptr && tokens != nullptr, "input_forward: null argument");
    require(n_tok >= 0, "input_forward: negative token count");
    check_shard(s, h);
    require(h % 8 == 0 && ldo >= h && ldo % 8 == 0 && aligned16(out), "input_forward: h/ldo must be multiples of 8");
    if (n_tok == 0) return;
    c->activate();
    if (!c->distributed()) {  // one rank: the plain masked gather is the whole layer
      NvtxRange nr("vp:input_forward");
      vp::k_input_forward<<<c->grid_for(n_tok, 8), 256, 0, c->stream>>>(
          tokens, int(n_tok), static_cast<const __nv_bfloat16*>(s->W), s->ldw, s->row_begin, s->row_end, int(h),
          static_cast<__nv_bfloat16*>(out), ldo, 0, c->d_err);
      VP_KCHECK();
      ++c->launches;
      return;
    }
    require(n_tok < (int64_t(1) << 31), "input_forward_gathered: too many tokens");
    if (c->peer_input && c->nranks <= vp::kMaxRoute && !c->in_sym.failed &&
        ensure_sym(c, c->in_sym, 2 * size_t(round_up(n_tok * h * 2, 256)))) {
      // peer pull: owned rows at their token index in my buffer (half `par`),
      // a group barrier, then row i read from its owner's buffer
      NvtxRange nr("vp:input_forward(peer pull)");
      const vp::RankBounds& B = rank_bounds(c, s);
      const size_t half = c->in_sym.bytes / 2 / 256 * 256;
      const size_t off = size_t(c->in_calls++ & 1) * half;
      vp::k_input_own_rows<<<c->grid_for(n_tok, 8), 256, 0, c->stream>>>(
          tokens, int(n_tok), static_cast<const __nv_bfloat16*>(s->W), s->ldw, s->row_begin, s->row_end, int(h),
          reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(c->in_sym.p) + off), c->d_err);
      VP_KCHECK();
      group_barrier(c);
      vp::PeerBufs P{};
      for (int k = 0; k < c->nranks; ++k)
        P.p[k] = reinterpret_cast<const __nv_bfloat16*>(static_cast<const char*>(c->in_sym.peers[size_t(k)]) + off);
      vp::k_input_pull_rows<<<c->grid_for(n_tok, 8), 256, 0, c->stream>>>(tokens, int(n_tok), B, P, int(h),
                                                                         static_cast<__nv_bfloat16*>(out), ldo);
      VP_KCHECK();
      c->launches += 2;
      ++c->peer_input_count;
      return;
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    VP_CUDA(cudaStreamIsCapturing(c->stream, &cap));
    require(cap == cudaStreamCaptureStatusNone,
            "input_forward_gathered: not capturable (the broadcast sizes go through the host)");
    NvtxRange nr("vp:input_forward(owner gather)");
    const vp::RankBounds& B = rank_bounds(c, s);
    int* pos = c->buf<int>(c->heads, size_t(n_tok) + size_t(vp::kMaxRanks));
    int* counts = pos + n_tok;
    vp::k_owner_positions<<<1, 1024, 0, c->stream>>>(tokens, int(n_tok), B, pos, counts, c->d_err);
    VP_KCHECK();
    std::vector<int> cnt(size_t(B.n));
    VP_CUDA(cudaMemcpyAsync(cnt.data(), counts, cnt.size() * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    VP_CUDA(cudaStreamSynchronize(c->stream));  // the block sizes of the broadcasts (host side)
    vp::RankOffsets O{};
    int64_t total = 0;
    for (int k = 0; k < B.n; ++k) {
      O.off[k] = total;
      total += cnt[size_t(k)];
    }
    auto* buf = c->buf<__nv_bfloat16>(c->xs, size_t(std::max<int64_t>(total, 1) * h));
    vp::k_owner_pack<<<c->grid_for(n_tok, 8), 256, 0, c->stream>>>(
        tokens, int(n_tok), B, pos, O, c->rank, static_cast<const __nv_bfloat16*>(s->W), s->ldw, int(h), buf);
    VP_KCHECK();
    c->cm().group_start();
    for (int k = 0; k < B.n; ++k)
      if (cnt[size_t(k)] > 0)
        c->cm().broadcast(buf + O.off[k] * h, buf + O.off[k] * h, size_t(cnt[size_t(k)]) * size_t(h),
                          vp::DType::BF16, k, c->stream);
    c->cm().group_end();
    vp::k_owner_unpack<<<c->grid_for(n_tok, 8), 256, 0, c->stream>>>(tokens, int(n_tok), B, pos, O, buf, int(h),
                                                                     static_cast<__nv_bfloat16*>(out), ldo);
    VP_KCHECK();
    c->launches += 3;
  });
}

// The input layer's pre-backward broadcast (R/PAPER.md:582): grad_out of the
// embedding output, produced on one rank, to every vocabulary shard.
int vp_input_backward_gathered(vp_ctx_t c, const void* grad, int64_t ldg, int grad_is_f32, const int64_t* tokens,
                               int64_t n_tok, int64_t h, const vp_shard_t* s, float* gw, int64_t ldgw, int accumulate,
                               int root) {
  return api([&] {
    require(c != nullptr && gw != nullptr && tokens != nullptr, "input_backward: null argument");
    require(n_tok >= 0, "input_backward: grad/token length mismatch");
    check_shard(s, h);
    const bool dist = c->distributed();
    require(!dist || (root >= 0 && root < c->nranks), "input_backward_gathered: root out of range");
    const bool has_grad = !dist || c->rank == root;
    require(!has_grad || grad != nullptr, "input_backward: null argument");
    require(h % 8 == 0 && ldg >= h && ldg % 8 == 0 && ldgw >= h && ldgw % 4 == 0 && aligned16(gw) &&
                (!has_grad || aligned16(grad)),
            "input_backward: h/ld must be multiples of 8");
    c->activate();
    NvtxRange nr("vp:input_backward(group)");
    const int64_t rows = s->row_end - s->row_begin;
    if (!accumulate)
      VP_CUDA(cudaMemset2DAsync(gw, size_t(ldgw) * sizeof(float), 0, size_t(h) * sizeof(float), size_t(rows),
                                c->stream));
    if (n_tok == 0) return;
    require(n_tok < (int64_t(1) << 31), "input_backward_gathered: too many tokens");
    const size_t esz = grad_is_f32 ? 4 : 2;
    auto scatter = [&](const void* src, int64_t lds) {
      if (grad_is_f32)
        segment_scatter(c, tokens, n_tok, s->row_begin, s->row_end, static_cast<const float*>(src), lds, h, 1.f, gw,
                        ldgw, 1, kErrInputBwd);
      else
        segment_scatter(c, tokens, n_tok, s->row_begin, s->row_end, static_cast<const __nv_bfloat16*>(src), lds, h,
                        1.f, gw, ldgw, 1, kErrInputBwd);
    };
    if (!dist) {
      scatter(grad, ldg);
      return;
    }
    const size_t dense = size_t(n_tok) * size_t(h) * esz;
    if (c->peer_input && c->nranks <= vp::kMaxRoute && !c->bwd_sym.failed &&
        ensure_sym(c, c->bwd_sym, 2 * size_t(round_up(int64_t(dense), 256)))) {
      // root stages grad_out (dense rows) in half `par` of its buffer; after a
      // barrier every rank's scatter reads its owned tokens' rows from there
      const size_t half = c->bwd_sym.bytes / 2 / 256 * 256;
      const size_t off = size_t(c->bwd_calls++ & 1) * half;
      if (c->rank == root)
        VP_CUDA(cudaMemcpy2DAsync(static_cast<char*>(c->bwd_sym.p) + off, size_t(h) * esz, grad, size_t(ldg) * esz,
                                  size_t(h) * esz, size_t(n_tok), cudaMemcpyDeviceToDevice, c->stream));
      group_barrier(c);
      scatter(static_cast<const char*>(c->bwd_sym.peers[size_t(root)]) + off, h);
      ++c->peer_input_count;
      return;
    }
    // fallback: the whole gradient broadcast into a context buffer
    void* buf = c->buf<char>(c->gbuf, dense);
    if (c->rank == root)
      VP_CUDA(cudaMemcpy2DAsync(buf, size_t(h) * esz, grad, size_t(ldg) * esz, size_t(h) * esz, size_t(n_tok),
                                cudaMemcpyDeviceToDevice, c->stream));
    c->cm().broadcast(buf, buf, size_t(n_tok) * size_t(h), grad_is_f32 ? vp::DType::F32 : vp::DType::BF16, root,
                      c->stream);
    scatter(buf, h);
  });
}

int vp_input_grad_broadcast(vp_ctx_t c, void* grad, int64_t ldg, int grad_is_f32, int64_t n_tok, int64_t h,
                            int root) {
  return api([&] {
    require(c != nullptr && grad != nullptr, "input_grad_broadcast: null argument");
    require(n_tok >= 0 && h >= 1 && ldg >= h, "input_grad_broadcast: bad shape");
    if (!c->distributed() || n_tok == 0) return;
    require(root >= 0 && root < c->nranks, "input_grad_broadcast: root out of range");
    c->activate();
    NvtxRange nr("vp:input_grad_broadcast");
    // the logical extent (ldg may pad rows; the pad is carried along)
    const size_t count = size_t((n_tok - 1) * ldg + h);
    c->cm().broadcast(grad, grad, count, grad_is_f32 ? vp::DType::F32 : vp::DType::BF16, root, c->stream);
  });
}

int vp_allreduce_sum(vp_ctx_t c, void* buf, int64_t count, int dtype) {
  return api([&] {
    require(c != nullptr && buf != nullptr, "allreduce: null argument");
    require(dtype == 0 || dtype == 1, "allreduce: dtype must be 0 (fp32) or 1 (bf16)");
    if (!c->distributed()) return;
    c->activate();
    c->cm().all_reduce(buf, buf, size_t(count), dtype == 0 ? vp::DType::F32 : vp::DType::BF16, vp::RedOp::Sum,
                       c->stream);
  });
}

int vp_program_parse(const char* text, vp_program_t* out) {
  return api([&] {
    require(text != nullptr && out != nullptr, "vp_program_parse: null argument");
    auto* pr = new vp_program_s();
    try {
      pr->prog = vp::parse_program(text);
    } catch (const vp::ProgramParseError& e) {
      delete pr;
      throw std::invalid_argument(e.what());
    } catch (...) {
      delete pr;
      throw;
    }
    *out = pr;
  });
}

int vp_program_destroy(vp_program_t pr) {
  delete pr;
  return VP_OK;
}

int vp_program_info(vp_program_t pr, int* barriers, int* p, int* n) {
  return api([&] {
    require(pr != nullptr, "vp_program_info: null program");
    if (barriers) *barriers = pr->prog.vocab ? pr->prog.barriers : 0;
    if (p) *p = int(pr->prog.p);
    if (n) *n = int(pr->prog.n);
  });
}

int vp_program_validate(vp_program_t pr, char* buf, int64_t buflen, int* count) {
  return api([&] {
    require(pr != nullptr, "vp_program_validate: null program");
    const auto v = vp::validate_vocab(pr->prog);
    std::string all;
    for (const auto& line : v) all += line + "\n";
    if (count) *count = int(v.size());
    if (buf && buflen > 0) {
      const size_t k = std::min(all.size(), size_t(buflen - 1));
      std::memcpy(buf, all.data(), k);
      buf[k] = '\0';
    }
  });
}

int vp_program_run(vp_ctx_t c, vp_program_t pr, const vp_batch_t* batches, const vp_shard_t* shards, int n_shards,
                   const vp_state_t* states, vp_stats_t* stats, float* const* loss, float* const* grad_x, int64_t ldgx,
                   float* const* grad_w, int64_t ldgw) {
  return api([&] {
    require(c != nullptr && pr != nullptr, "vp_program_run: null argument");
    c->activate();
    run_program(c, pr->prog, batches, shards, n_shards, states, stats, loss, grad_x, ldgx, grad_w, ldgw);
  });
}

int vp_ctx_capture_begin(vp_ctx_t c) {
  return api([&] {
    require(c != nullptr, "vp_ctx_capture_begin: null context");
    require(c->stream != nullptr, "vp_ctx_capture_begin: the legacy default stream cannot be captured");
    require(!c->timing, "vp_ctx_capture_begin: disable GEMM timing before capturing");
    require(!c->comm || c->comm->capturable(),
            "vp_ctx_capture_begin: the loopback backend's host rendezvous cannot be captured");
    c->activate();
    VP_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  });
}

int vp_ctx_capture_end(vp_ctx_t c, vp_graph_t* out) {
  return api([&] {
    require(c != nullptr && out != nullptr, "vp_ctx_capture_end: null argument");
    c->activate();
    auto* g = new vp_graph_s();
    cudaError_t e = cudaStreamEndCapture(c->stream, &g->graph);
    if (e != cudaSuccess) {
      delete g;
      (void)cudaGetLastError();
      throw CudaError(std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e) +
                      " (a workspace buffer grew or the stream was synchronised while capturing:"
                      " run the same call once eagerly first)");
    }
    e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g->graph);
      delete g;
      throw CudaError(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    }
    *out = g;
  });
}

int vp_graph_launch(vp_graph_t g, vp_ctx_t c) {
  return api([&] {
    require(g != nullptr && c != nullptr, "vp_graph_launch: null argument");
    c->activate();
    VP_CUDA(cudaGraphLaunch(g->exec, c->stream));
  });
}

int vp_graph_destroy(vp_graph_t g) {
  if (g) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
  }
  return VP_OK;
}


}  // extern "C"
