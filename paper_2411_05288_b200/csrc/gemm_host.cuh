// Host side of the tcgen05 GEMM: TMA descriptor encoding and launch.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "gemm_sm100.cuh"

namespace vp {

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library needs no -lcuda at link time.
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
      throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
    return reinterpret_cast<PFN_encodeTiled>(p);
  }();
  return fn;
}

inline int g_l2_promotion = 3;  // operand tensor maps: 0 none, 1 64 B, 2 128 B, 3 256 B (default)

// 2-D bf16 tensor map over a row-major [outer x inner] matrix with leading
// dimension `ld` (elements), SWIZZLE_128B boxes of [box_outer x box_inner].
// Out-of-bounds elements of a box read as zero.
inline CUtensorMap make_tmap_bf16(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                                  uint32_t box_outer) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0) throw std::invalid_argument("tensor map: base not 16-B aligned");
  if ((ld * 2) % 16 != 0) throw std::invalid_argument("tensor map: row stride not a multiple of 16 B");
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               g_l2_promotion == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                               : g_l2_promotion == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                               : g_l2_promotion == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

// 2-D tensor map of the epilogue's TMA stores: row-major [outer x inner]
// elements of `esize` bytes, SWIZZLE_64B boxes of [32 rows x 64 B].
inline CUtensorMap make_store_map(const void* ptr, CUtensorMapDataType dt, int esize, uint64_t inner,
                                  uint64_t outer, uint64_t ld, int row_bytes = 64) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * uint64_t(esize)};
  const cuuint32_t box[2] = {cuuint32_t(row_bytes / esize), 32};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE,
                               row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (store) failed: " + std::to_string(int(r)));
  return m;
}

inline int g_tma_store = 1;  // epilogue stores through TMA when the output allows it (16-B aligned rows)

inline bool tma_store_ok(const void* p, int64_t ld, int esize) {
  return g_tma_store && (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld * esize) % 16 == 0;
}
inline void prepare_store(EpiStoreF32::Params& ep, int M, int N) {
  if (ep.route_n > 0) {  // routed: per-thread stores to the owners' slots (route_out)
    ep.use_tma = 0;
    return;
  }
  ep.use_tma = tma_store_ok(ep.out, ep.ldo, 4);
  if (ep.use_tma)
    ep.map = make_store_map(ep.out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, uint64_t(N), uint64_t(M), uint64_t(ep.ldo),
                            VP_F32_BOX128 ? 128 : 64);
}
inline void prepare_store(EpiLogitStats::Params& ep, int M, int N) {
  ep.use_tma = tma_store_ok(ep.P, ep.ldp, 2);
  if (ep.use_tma)
    ep.map = make_store_map(ep.P, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, uint64_t(N), uint64_t(M), uint64_t(ep.ldp),
                            VP_P_BOX128 ? 128 : 64);
}

// Split-K state owned by the caller (one per stream: the flags are reset by
// each launch, so two GEMMs sharing one SplitCfg must not run concurrently).
// flags: >= 2 * max_tiles ints.
struct SplitCfg {
  int* flags = nullptr;
  int max_tiles = 0;
  int force = 0;  // > 0: use exactly this many splits (tests); 0: choose by wave quantisation
  // parallel split-K workspace (fp32, >= clusters x 256 x 512 elements + slack):
  // used when the tiles fill less than half a wave; null = ordered splits only
  float* ws = nullptr;
  size_t ws_elems = 0;
  int ws_mode = 1;    // 0: never use the workspace; 2: force it whenever S > 1 (tests)
  int min_kb = 64;    // ordered splits keep at least this many k-blocks per unit
  int64_t reduce_launches = 0;  // k_split_reduce launches so far (evidence counters)
};

// Optional L2 access-policy window of one launch (cudaLaunchAttributeAccessPolicyWindow):
// accesses to [ptr, ptr + bytes) are marked persisting (hit_ratio of them),
// the rest streaming.  Needs a persisting L2 set-aside (cudaLimitPersistingL2CacheSize).
struct L2Window {
  const void* ptr = nullptr;
  size_t bytes = 0;
  float hit_ratio = 1.f;
};

// Wave-lockstep state owned by the caller (per stream, like SplitCfg):
// counters for up to `capacity` (wave, epoch) pairs, reset by each launch.
struct LockCfg {
  int* counters = nullptr;
  int64_t capacity = 0;
  int epoch = 0;  // k-blocks per epoch; 0 = off
};

// Splits for a persistent GEMM of `tiles` tiles on `clusters` clusters and
// num_kb k-blocks: the smallest S in 1..4 whose wave efficiency
// tiles*S / (clusters * ceil(tiles*S / clusters)) is within 1% of the best,
// keeping >= min_kb k-blocks per split (round 1 used 128: dW of an 8-way shard
// split 3 ways ran 20% slower before the epilogues released TMEM early; the
// context default is now 64); S = 1 unless that gains > 2%.
inline int choose_splits(int tiles, int clusters, int num_kb, int min_kb = 128) {
  auto eff = [&](int S) {
    const double w = double(tiles) * S / clusters;
    return w / std::ceil(w);
  };
  int best = 1;
  double be = eff(1);
  for (int S = 2; S <= 4; ++S)
    if (num_kb / S >= min_kb && eff(S) > be + 0.02) {
      best = S;
      be = eff(S);
    }
  return best;
}

// Parallel split-K for GEMMs whose tiles fill less than half a wave (small
// token counts, narrow shards): S units per tile run concurrently and store
// partials; a reduction kernel sums them.  Cost model in pair k-block cycles
// (1024 per k-block of a 256 x 512 tile; ~6k fixed per unit for the pipeline
// fill and the epilogue; the reduction streams (S + 1) * M * N * 4 bytes at
// ~1.6 KB/cycle plus a launch): the S in 2..min(32, clusters / tiles) with at
// least 8 k-blocks per unit that minimises it, if it beats S = 1.
inline int choose_ws_splits(int tiles, int clusters, int num_kb, int64_t M, int64_t N) {
  auto cost = [&](int S) {
    const double units = double(tiles) * S;
    const double waves = std::ceil(units / clusters);
    const double kb = std::ceil(double(num_kb) / S);
    double c = waves * (kb * 1024.0 + 6000.0);
    if (S > 1) c += double(S + 1) * double(M) * double(N) * 4.0 / 1600.0 + 4000.0;
    return c;
  };
  int best = 1;
  double bc = cost(1);
  const int smax = std::min(32, clusters / std::max(tiles, 1));
  for (int S = 2; S <= smax && num_kb / S >= 8; ++S)
    if (cost(S) < bc * 0.97) {
      best = S;
      bc = cost(S);
    }
  return best;
}

template <class Params>
inline bool splittable(const Params&) { return false; }
inline bool splittable(const EpiStoreF32::Params& p) { return p.tile_max == nullptr; }
template <class Params>
inline bool routed(const Params&) { return false; }
inline bool routed(const EpiStoreF32::Params& p) { return p.route_n > 0; }
template <class Params>
inline int route_splits(const Params&) { return 1; }
inline int route_splits(const EpiStoreF32::Params& p) { return p.route_n > 0 ? p.route_splits : 1; }
template <class Params>
inline bool uses_tma(const Params&) { return false; }
inline bool uses_tma(const EpiStoreF32::Params& p) { return p.use_tma != 0; }
template <class Params>
inline void set_ws_map(Params&, float*, int, int64_t, int64_t) {}
inline void set_ws_map(EpiStoreF32::Params& p, float* ws, int N, int64_t rows, int64_t ldws) {
  p.ws_map = make_store_map(ws, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, uint64_t(N), uint64_t(rows), uint64_t(ldws),
                            VP_F32_BOX128 ? 128 : 64);
}
template <class Params>
inline void launch_split_reduce(const Params&, const GemmGeom&, int, int, int, cudaStream_t) {}
inline void launch_split_reduce(const EpiStoreF32::Params& p, const GemmGeom& g, int M, int N, int num_sms,
                                cudaStream_t st) {
  const int64_t ldws = (int64_t(N) + 3) / 4 * 4;
  const int64_t work = int64_t(M) * ((N + 3) / 4);
  const int blocks = int(std::min<int64_t>((work + 255) / 256, int64_t(num_sms) * 8));
  k_split_reduce<<<blocks, 256, 0, st>>>(g.split_ws, g.splits, g.ws_rows, ldws, p.out, p.ldo, M, N, p.accumulate);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("split reduce launch: ") + cudaGetErrorString(e));
}

// One GEMM operand: row-major storage `ptr` with leading dimension `ld`.
//   K-major : storage [rows x K]  (A: rows = M, B: rows = N)
//   MN-major: storage [K x rows]
struct Operand {
  const void* ptr;
  int64_t ld;
  bool mn_major;
};

inline unsigned long long* g_gemm_prof = nullptr;  // set by probes: {clk0, t0, clk1, t1} of CTA 0
inline int g_epi_wait = 1;            // GemmGeom::epi_wait for subsequent launches
inline int g_store_evict_first = 0;  // GemmGeom::store_evict_first for subsequent launches
inline int g_cooperative = 1;        // cooperative (co-resident) launches of the persistent GEMMs

template <int CG, bool A_MN, bool B_MN, class Epi, int MC = 1, int NH = 1>
inline void launch_gemm_t(const Operand& A, const Operand& B, int M, int N, int K, int raster,
                          const typename Epi::Params& ep, int num_sms, cudaStream_t st, int pol_a = -1,
                          int pol_b = -1, SplitCfg* split = nullptr, const LockCfg* lock = nullptr,
                          int store_hint = -1, const L2Window* win = nullptr) {
  using C = GemmCfg<CG, NH>;
  const CUtensorMap ta = A_MN ? make_tmap_bf16(A.ptr, uint64_t(M), uint64_t(K), uint64_t(A.ld), 64, 64)
                              : make_tmap_bf16(A.ptr, uint64_t(K), uint64_t(M), uint64_t(A.ld), 64, C::BM_CTA);
  // with multicast each CTA loads half of its B block (64 rows / one 64-col chunk)
  const CUtensorMap tb = B_MN ? make_tmap_bf16(B.ptr, uint64_t(N), uint64_t(K), uint64_t(B.ld), 64, 64)
                              : make_tmap_bf16(B.ptr, uint64_t(K), uint64_t(N), uint64_t(B.ld), 64,
                                               MC == 2 ? 64 : C::B_HALF_ROWS);
  GemmGeom g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.tiles_m = (M + C::BM - 1) / C::BM;
  g.tiles_n = (N + C::BN_TILE - 1) / C::BN_TILE;
  g.num_kb = (K + C::BK - 1) / C::BK;
  g.raster = raster;
  g.pol_a = pol_a;
  g.pol_b = pol_b;
  g.prof = g_gemm_prof;
  g.store_evict_first = store_hint >= 0 ? store_hint : g_store_evict_first;
  g.epi_wait = g_epi_wait;
  auto kern = gemm_sm100_kernel<CG, A_MN, B_MN, Epi, MC, NH>;
  // per device: the smem attribute and the occupancy query (contexts of one
  // process may drive several GPUs)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  static bool attr_done_dev[64] = {};
  bool& attr_done = attr_done_dev[dev];
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) throw std::runtime_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  constexpr int CL = CG * MC;
  const int tiles = ((g.tiles_m + MC - 1) / MC) * g.tiles_n;
  cudaLaunchConfig_t cfg = {};
  // persistent grid: no more clusters than can be co-resident (clusters of 4
  // cannot tile all 148 SMs: GPC packing leaves some idle)
  static int max_active_dev[64] = {};
  int& max_active = max_active_dev[dev];
  if (max_active <= 0) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(unsigned(num_sms / CL * CL), 1, 1);
    q.blockDim = dim3(C::THREADS, 1, 1);
    q.dynamicSmemBytes = C::SMEM_BYTES;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = CL;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) {
      (void)cudaGetLastError();
      n = num_sms / CL;
    }
    max_active = n;
  }
  int cap = num_sms / CL < max_active ? num_sms / CL : max_active;
  int clusters = tiles < cap ? tiles : cap;
  typename Epi::Params epc = ep;
  prepare_store(epc, M, N);
  if (route_splits(epc) > 1) {
    // routed output: the caller chose the split count (its slot layout);
    // units are independent, no flags
    g.splits = route_splits(epc);
    g.split_indep = 1;
    clusters = tiles * g.splits < cap ? tiles * g.splits : cap;
  } else if (MC == 1 && split != nullptr && split->flags != nullptr && splittable(ep) && !routed(epc) &&
             tiles <= split->max_tiles) {
    // workspace mode: less than half a wave of tiles, TMA-stored output, room
    const int64_t ldws = (int64_t(N) + 3) / 4 * 4;
    const bool ws_ok = split->ws != nullptr && split->ws_mode != 0 && uses_tma(epc) && !routed(epc) &&
                       (split->ws_mode == 2 || tiles * 2 <= cap);
    int S = split->force;
    if (S <= 0)
      S = ws_ok ? choose_ws_splits(tiles, cap, g.num_kb, M, N) : choose_splits(tiles, cap, g.num_kb, split->min_kb);
    if (ws_ok && S > 1 && size_t(S) * size_t(g.tiles_m * C::BM) * size_t(ldws) > split->ws_elems)
      S = 1;  // (forced S beyond the workspace: the tests stay within it)
    if (ws_ok && S > 1 && g.num_kb >= S) {
      g.splits = S;
      g.split_ws = split->ws;
      g.ws_rows = g.tiles_m * C::BM;
      set_ws_map(epc, split->ws, N, int64_t(S) * g.ws_rows, ldws);
      clusters = tiles * S < cap ? tiles * S : cap;
    } else if (S > 1 && g.num_kb >= S) {
      g.splits = S;
      g.split_flags = split->flags;
      g.flag_base = 0;
      // flags restart at 0 for every launch (a memset node in a captured CUDA
      // graph, so replays never see a previous launch's flags)
      cudaError_t me = cudaMemsetAsync(split->flags, 0, size_t(2 * tiles) * sizeof(int), st);
      if (me != cudaSuccess) throw std::runtime_error(std::string("split flags memset: ") + cudaGetErrorString(me));
      clusters = tiles * S < cap ? tiles * S : cap;
    }
  }
  cfg.gridDim = dim3(unsigned(clusters * CL), 1, 1);
  cfg.blockDim = dim3(C::THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // Cooperative launch: the whole persistent grid is guaranteed co-resident.
  // The kernel's cross-CTA waits (K1's row reference, ordered split-K units,
  // wave lockstep) rely on it; without it, kernels of other streams holding
  // SMs could leave a waited-on cluster unscheduled.
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = g_cooperative;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (win != nullptr && win->ptr != nullptr && win->bytes > 0) {
    at[2].id = cudaLaunchAttributeAccessPolicyWindow;
    at[2].val.accessPolicyWindow.base_ptr = const_cast<void*>(win->ptr);
    at[2].val.accessPolicyWindow.num_bytes = win->bytes;
    at[2].val.accessPolicyWindow.hitRatio = win->hit_ratio;
    at[2].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[2].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 3;
  }
  if (lock != nullptr && lock->counters != nullptr && lock->epoch > 0) {
    const int units = tiles * g.splits;
    const int waves = (units + clusters - 1) / clusters;
    const int max_nkb = (g.num_kb + g.splits - 1) / g.splits + 1;
    const int stride = (max_nkb + lock->epoch - 1) / lock->epoch + 1;
    if (waves > 1 && int64_t(waves) * stride <= lock->capacity) {
      g.lockstep = lock->counters;
      g.lock_epoch = lock->epoch;
      g.lock_stride = stride;
      cudaError_t me = cudaMemsetAsync(lock->counters, 0, size_t(waves) * size_t(stride) * sizeof(int), st);
      if (me != cudaSuccess) throw std::runtime_error(std::string("lockstep memset: ") + cudaGetErrorString(me));
    }
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, g, epc);
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm launch: ") + cudaGetErrorString(e));
  if (g.split_ws != nullptr) {
    launch_split_reduce(epc, g, M, N, num_sms, st);
    ++split->reduce_launches;
  }
}

// Runtime dispatch over (cta_group, operand majors).
template <class Epi>
inline void launch_gemm(int cg, const Operand& A, const Operand& B, int M, int N, int K, int raster,
                        const typename Epi::Params& ep, int num_sms, cudaStream_t st, int pol_a = -1,
                        int pol_b = -1, int mc = 1, int nh = 1, SplitCfg* split = nullptr,
                        const LockCfg* lock = nullptr, int store_hint = -1, const L2Window* win = nullptr) {
#define VP_GEMM_CASE(CGV, AM, BM_, MCV, NHV)                                                                        \
  if (cg == CGV && A.mn_major == AM && B.mn_major == BM_ && mc == MCV && nh == NHV) {                               \
    launch_gemm_t<CGV, AM, BM_, Epi, MCV, NHV>(A, B, M, N, K, raster, ep, num_sms, st, pol_a, pol_b, split, lock,    \
                                               store_hint, win);                                                   \
    return;                                                                                                         \
  }
  VP_GEMM_CASE(2, false, false, 1, 1)
  VP_GEMM_CASE(2, false, true, 1, 1)
  VP_GEMM_CASE(2, true, true, 1, 1)
  VP_GEMM_CASE(2, false, false, 2, 1)
  VP_GEMM_CASE(2, false, true, 2, 1)
  VP_GEMM_CASE(2, true, true, 2, 1)
  VP_GEMM_CASE(2, false, false, 1, 2)
  VP_GEMM_CASE(2, false, true, 1, 2)
  VP_GEMM_CASE(2, true, true, 1, 2)
  VP_GEMM_CASE(1, false, false, 1, 1)
  VP_GEMM_CASE(1, false, true, 1, 1)
  VP_GEMM_CASE(1, true, true, 1, 1)
#undef VP_GEMM_CASE
  throw std::invalid_argument("launch_gemm: unsupported operand layout combination");
}

}  // namespace vp
