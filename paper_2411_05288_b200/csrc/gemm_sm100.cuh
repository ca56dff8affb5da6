// Persistent, warp-specialised tcgen05 GEMM for sm_100a with pluggable
// epilogues.  D[M x N] = A[M x K] * B[N x K]^T, bf16 operands, fp32
// accumulation in TMEM.
//
//   * operands arrive by TMA (SWIZZLE_128B) into a STAGES-deep smem ring;
//     each operand is K-major (row-major [rows x K]) or MN-major
//     (row-major [K x rows]) — the three vocab GEMMs need all of
//       K1 logits  Y  = X . W_k^T      A: X [T x h]        K-major
//                                      B: W_k [V_k x h]    K-major
//       K3 dX      A  = P' . W_k       A: P' [T x V_k]     K-major
//                                      B: W_k [V_k x h]    MN-major
//       K4 dW      dW = P'^T . X~      A: P' [T x V_k]     MN-major
//                                      B: X~ [T x h]       MN-major
//   * CG = 2 runs one 256 x 256 tile per CTA pair (cta_group::2): each CTA
//     loads 128 rows of A and 128 rows of B, the leader CTA's single thread
//     issues tcgen05.mma for the pair, and each CTA's TMEM holds its 128
//     accumulator rows.  CG = 1 runs 128 x 256 tiles per CTA.  NH = 2 makes
//     the pair tile 256 x 512 (two N = 256 MMAs per K step, all 512 TMEM
//     columns) with the two N halves staggered at tile boundaries.
//   * NH = 1: TMEM holds two 256-column accumulators so the epilogue of tile
//     i overlaps the main loop of tile i+1.
//   * warp roles (384 threads): w0 TMA producer, w1 MMA issuer (leader CTA),
//     w2 TMEM allocator, w3 idle, w4..w11 epilogue (lane quadrant w % 4,
//     column group (w - 4) / 4: one accumulator row per thread, 128 columns
//     per call), storing through smem staging + TMA.
//   * optional split-K units with ordered (deterministic) accumulation.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100_ptx.cuh"

#ifndef VP_GEMM_PROBE
#define VP_GEMM_PROBE 0  // 1: CTA 0 records wait / work cycles into GemmGeom::prof (tools/gemm_probe)
#endif
#ifndef VP_EPI_MODE
#define VP_EPI_MODE 0  // probes only: 1 = TMEM loads only, 2 = nothing, 3 = K1 math without stores, 4 = K1 stores without math
#endif
#ifndef VP_P_BOX128
#define VP_P_BOX128 1  // K1 stores P in 32 x 128 B SWIZZLE_128B boxes (half the TMA row segments; 0: 64 B boxes)
#endif
#ifndef VP_F32_BOX128
#define VP_F32_BOX128 1  // fp32 epilogues store 32 x 128 B SWIZZLE_128B boxes (0: two 64 B boxes per chunk)
#endif
#ifndef VP_K1_EARLY
#define VP_K1_EARLY 1  // K1 epilogue drains its accumulator half to registers and releases TMEM before the math
#endif
#ifndef VP_F32_EARLY
#define VP_F32_EARLY 0  // the same for the fp32 (dX / dW) epilogues
#endif
#ifndef VP_K1_POLY
#define VP_K1_POLY 0  // 1: half of the K1 epilogue's exponentials on the FMA pipe (ptx::ex2_poly)
#endif

namespace vp {

constexpr int kMaxRoute = 16;  // owners of a routed epilogue (ranks of a group)

struct GemmGeom {
  int M, N, K;
  int tiles_m, tiles_n, num_kb;
  // Tile rasterisation.  raster >= 0: M-fastest inside groups of `raster`
  // m-tiles (0 = all); raster < 0: N-fastest inside groups of -raster
  // n-tiles.  Picks which operand band stays L2-resident while the
  // concurrently running tiles sweep the other.
  int raster;
  // L2 policies of the A / B TMA loads: 0 evict_normal, 1 evict_first,
  // 2 evict_last, -1 = the epilogue's default (see Epi::kAStreams).
  int pol_a = -1, pol_b = -1;
  // optional probe: CTA 0 writes {clock64, globaltimer} at start and end
  unsigned long long* prof = nullptr;
  // how the epilogue warps wait for an accumulator: 0 try_wait loop,
  // 1 nanosleep backoff (fewer issued instructions while a main loop runs)
  int epi_wait = 1;
  // Split-K (few-wave GEMMs, e.g. dX with K = V_k): every tile is computed as
  // `splits` units over consecutive K ranges; unit u = s * tiles + t.  Split 0
  // stores, split s > 0 adds its partial after split s-1 of the same tile
  // (and CTA) has landed — a fixed order, so results are deterministic.
  // split_flags[2 * t + rank] holds flag_base + (splits completed).
  int splits = 1;
  int* split_flags = nullptr;
  int flag_base = 0;
  // wave lockstep (see the producer): epoch counters [waves x lock_stride],
  // zeroed per launch; null = off
  int* lockstep = nullptr;
  int lock_epoch = 8;
  int lock_stride = 0;
  int store_evict_first = 0;  // epilogue TMA stores with an L2 evict-first hint
  // Parallel split-K (less than a wave of tiles): unit (tile, s) stores its
  // partial into rows [s * ws_rows, ...) of a workspace instead of waiting for
  // split s-1; k_split_reduce then sums the S slices in fixed order.
  float* split_ws = nullptr;
  int ws_rows = 0;
  // split units independent of each other (routed output: every unit stores
  // its own partial into its own slot; the owner sums them): no flags
  int split_indep = 0;
};

__device__ __forceinline__ uint64_t make_policy(int p, bool dflt_first) {
  if (p < 0) p = dflt_first ? 1 : 2;
  return p == 1 ? ptx::policy_evict_first() : p == 2 ? ptx::policy_evict_last() : ptx::policy_evict_normal();
}

// NH = N halves per tile: NH == 2 gives a 256 x 512 pair tile computed as two
// N=256 MMAs per K step into all 512 TMEM columns (one accumulator, no TMEM
// double buffering): 25% fewer operand bytes per flop and half the A re-reads.
template <int CG, int NH = 1>
struct GemmCfg {
  static constexpr int BM_CTA = 128;          // accumulator rows per CTA
  static constexpr int BM = 128 * CG;         // MMA M
  static constexpr int BN = 256;              // MMA N
  static constexpr int BN_TILE = BN * NH;     // tile N
  static constexpr int BK = 64;               // 128 B of bf16 = one swizzle row
  static constexpr int UK = 16;               // K per tcgen05.mma (kind::f16)
  static constexpr int B_HALF_ROWS = BN / CG; // B rows per CTA per N half
  static constexpr int B_ROWS = NH * B_HALF_ROWS;  // B rows loaded per CTA
  static constexpr int STAGES = CG == 2 ? (NH == 2 ? 4 : 6) : 4;
  static constexpr int A_BYTES = BM_CTA * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_WARPS = 8;
  static constexpr int STG_WARP = 2 * 2048;                // TMA-store staging per epilogue warp: 2 boxes of 2 KB
  static constexpr int STG_BYTES = EPI_WARPS * STG_WARP;
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 4) + 16;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STG_BYTES + BAR_BYTES + 1024;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int TMEM_COLS = 512;
};

__device__ __forceinline__ void tile_coords(const GemmGeom& g, int t, int& mb, int& nb) {
  if (g.raster >= 0) {
    const int G = g.raster > 0 ? g.raster : g.tiles_m;
    const int per = G * g.tiles_n;
    const int grp = t / per, r = t - grp * per;
    const int first = grp * G;
    const int gs = min(G, g.tiles_m - first);
    mb = first + r % gs;
    nb = r / gs;
  } else {
    const int G = -g.raster;
    const int per = G * g.tiles_m;
    const int grp = t / per, r = t - grp * per;
    const int first = grp * G;
    const int gs = min(G, g.tiles_n - first);
    nb = first + r % gs;
    mb = r / gs;
  }
}

constexpr int kEpiCols = 128;  // accumulator columns per epilogue warp and call (= K1 stats tile width)

// Per-warp staging: two 2 KB boxes (32 rows x 64 B, SWIZZLE_64B), filled as
// a pair and flushed with one proxy fence + up to two TMA stores (one bulk
// group); the pair is rewritten only after that group has read its smem.
struct Stager {
  uint32_t base;
  uint32_t k = 0;
  bool probe = false;              // count cycles spent waiting for free boxes (lane 0)
  unsigned long long wait_cyc = 0;
  __device__ explicit Stager(uint32_t b) : base(b) {}
  // next box; the first of a pair waits until the previous group read its boxes
  __device__ __forceinline__ uint32_t next() {
    if ((k & 1u) == 0) {
      if ((threadIdx.x & 31) == 0) {
        const unsigned long long c0 = VP_GEMM_PROBE && probe ? clock64() : 0;
        ptx::bulk_wait_read<0>();
        if (VP_GEMM_PROBE && probe) wait_cyc += clock64() - c0;
      }
      __syncwarp();
    }
    const uint32_t b = base + (k & 1u) * 2048u;
    ++k;
    return b;
  }
  // smem address of 16-byte chunk q (0..3) of this thread's 64-byte row
  // (row = lane) in a SWIZZLE_64B box: chunk bits [4:5] ^= row bits [1:2]
  __device__ static __forceinline__ uint32_t chunk(uint32_t box, int q) {
    const uint32_t r = threadIdx.x & 31;
    return box + r * 64u + ((uint32_t(q) ^ ((r >> 1) & 3u)) << 4);
  }
  // stores of streamed outputs (P, dW) carry an L2 evict-first hint so they
  // do not displace the operand band the co-scheduled tiles re-read (X in K1)
  uint64_t pol = 0;
  bool hint = false;
  __device__ static __forceinline__ void put_static(const Stager& sg, const CUtensorMap* m, uint32_t box, int c0,
                                                    int c1) {
    sg.put(m, box, c0, c1, false);
  }
  __device__ __forceinline__ void put(const CUtensorMap* m, uint32_t box, int c0, int c1, bool add) const {
    if (add) ptx::tma_reduce_add_2d(m, box, c0, c1);
    else if (hint) ptx::tma_store_2d_hint(m, box, c0, c1, pol);
    else ptx::tma_store_2d(m, box, c0, c1);
  }
  // store one box / two boxes written since the last flush (one bulk group)
  __device__ __forceinline__ void flush(const CUtensorMap* m, uint32_t box, int c0, int c1, bool add = false) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      put(m, box, c0, c1, add);
      ptx::bulk_commit();
    }
    k = (k + 1u) & ~1u;  // a lone box closes its pair
  }
  __device__ __forceinline__ void flush2(const CUtensorMap* m, uint32_t b0, int c0, int r0, uint32_t b1, int c1, int r1,
                                         bool add = false) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      put(m, b0, c0, r0, add);
      put(m, b1, c1, r1, add);
      ptx::bulk_commit();
    }
  }
  // all issued stores complete (global writes done)
  __device__ __forceinline__ void drain() {
    if ((threadIdx.x & 31) == 0) ptx::bulk_wait<0>();
    __syncwarp();
  }
};

// Walk the nch 32-column chunks of this warp's accumulator rows with the
// TMEM load of chunk c+1 in flight while chunk c is processed: f(regs, c).
template <class F>
__device__ __forceinline__ void tmem_chunks(uint32_t taddr, int nch, F&& f) {
  uint32_t ra[32], rb[32];
  ptx::tmem_ld32(taddr, ra);
  ptx::tmem_ld_wait();
  ptx::tmem_pin(ra);
#pragma unroll 1
  for (int c = 0; c < nch; c += 2) {
    if (c + 1 < nch) ptx::tmem_ld32(taddr + (c + 1) * 32, rb);
    f(ra, c);
    if (c + 1 >= nch) break;
    ptx::tmem_ld_wait();
    ptx::tmem_pin(rb);
    if (c + 2 < nch) ptx::tmem_ld32(taddr + (c + 2) * 32, ra);
    f(rb, c + 1);
    if (c + 2 < nch) {
      ptx::tmem_ld_wait();
      ptx::tmem_pin(ra);
    }
  }
}

// All 128 columns of this warp's accumulator rows into registers (one wait).
__device__ __forceinline__ void tmem_load_all(uint32_t taddr, uint32_t (&acc)[kEpiCols]) {
#pragma unroll
  for (int c = 0; c < kEpiCols / 32; ++c)
    ptx::tmem_ld32(taddr + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&acc[32 * c]));
  ptx::tmem_ld_wait();
#pragma unroll
  for (int c = 0; c < kEpiCols / 32; ++c) ptx::tmem_pin(*reinterpret_cast<uint32_t(*)[32]>(&acc[32 * c]));
}

// Chunk sources for the epilogue walks: f(chunk regs, c) for c < nch.
struct TmemSrc {
  uint32_t taddr;
  template <class F>
  __device__ __forceinline__ void operator()(int nch, F&& f) const { tmem_chunks(taddr, nch, f); }
};
struct RegSrc {
  uint32_t (&acc)[kEpiCols];
  template <class F>
  __device__ __forceinline__ void operator()(int nch, F&& f) const {
#pragma unroll
    for (int c = 0; c < kEpiCols / 32; ++c)
      if (c < nch) f(*reinterpret_cast<uint32_t(*)[32]>(&acc[32 * c]), c);
  }
};

// Split-K ordering (epilogue warps of one CTA).  split_wait: every lane
// waits until the previous split of this tile/CTA has landed in global
// memory; split_done: after this split's stores completed, publish it.
__device__ __forceinline__ void split_wait(const int* flag, int want) {
  if ((threadIdx.x & 31) == 0) {
    int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v - want >= 0) break;
      __nanosleep(256);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // later TMA reduces see those writes
  }
  __syncwarp();
}
__device__ __forceinline__ void split_done(int* flag, int value, Stager& sg) {
  sg.drain();  // this warp's TMA stores are complete
  if ((threadIdx.x & 31) == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  __threadfence();
  asm volatile("bar.sync 2, 256;" ::: "memory");  // the 8 epilogue warps of this CTA
  if (threadIdx.x == 128) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

// MC = CTA pairs per cluster along M (CG == 2 only).  MC == 2: a 4-CTA
// cluster computes a 512 x 256 "cluster tile" as two pair tiles (m, n) and
// (m+1, n) that need the same B rows; each CTA loads HALF of its B rows and
// multicasts them to its counterpart in the other pair, halving B's L2
// traffic.  A stage may then be refilled only after BOTH pairs consumed it,
// so every empty barrier expects one commit from each pair leader.
template <int CG, bool A_MN, bool B_MN, class Epi, int MC = 1, int NH = 1>
__global__ void __launch_bounds__(384, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmGeom g, const __grid_constant__ typename Epi::Params ep) {
  using C = GemmCfg<CG, NH>;
  static_assert(MC == 1 || (MC == 2 && CG == 2), "multicast clusters are built from CTA pairs");
  static_assert(NH == 1 || (NH == 2 && CG == 2 && MC == 1), "512-wide tiles: CTA pairs without multicast");
  constexpr int NACC = NH == 1 ? 2 : 1;  // TMEM accumulator buffers
  constexpr int CL = CG * MC;  // CTAs per cluster
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t sA = sbase;
  const uint32_t sB = sbase + C::STAGES * C::A_BYTES;
  const uint32_t stg = sbase + C::STAGES * C::STAGE_BYTES;  // 1024-aligned
  const uint32_t bar_full = stg + C::STG_BYTES;
  const uint32_t bar_empty = bar_full + 8 * C::STAGES;
  const uint32_t bar_tfull = bar_empty + 8 * C::STAGES;
  const uint32_t bar_tempty = bar_tfull + 16;
  uint32_t* tmem_slot =
      reinterpret_cast<uint32_t*>(smem + C::STAGES * C::STAGE_BYTES + C::STG_BYTES + 8 * (2 * C::STAGES + 4));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = CL > 1 ? ptx::cluster_ctarank() : 0u;  // rank in cluster
  const uint32_t rank = crank % CG;                              // rank in the CTA pair
  const uint32_t pair = crank / CG;                              // pair index along M
  const uint32_t leader = crank - rank;                          // cluster rank of the pair leader
  const uint16_t pair_mask = uint16_t(((1u << CG) - 1u) << leader);
  const int cluster = blockIdx.x / CL, nclusters = gridDim.x / CL;
  const int tiles_mc = (g.tiles_m + MC - 1) / MC;  // cluster tiles along M
  GemmGeom gc = g;
  gc.tiles_m = tiles_mc;
  const int num_tiles = tiles_mc * g.tiles_n;
  const int num_units = num_tiles * g.splits;
  // unit -> (tile, split, k-block range)
  auto unit_tile = [&](int u) { return u % num_tiles; };
  auto unit_split = [&](int u) { return u / num_tiles; };
  auto unit_kb0 = [&](int u) { return int((int64_t(u / num_tiles) * g.num_kb) / g.splits); };
  auto unit_nkb = [&](int u) {
    const int sp = u / num_tiles;
    return int((int64_t(sp + 1) * g.num_kb) / g.splits - (int64_t(sp) * g.num_kb) / g.splits);
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (g.prof && blockIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g.prof[0] = clock64();
      g.prof[1] = t;
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(bar_full + 8 * s, 1);    // pair leader's expect_tx (covers the pair)
      ptx::mbar_init(bar_empty + 8 * s, MC);  // one tcgen05.commit per consuming pair
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(bar_tfull + 8 * a, 1);        // one tcgen05.commit
      ptx::mbar_init(bar_tempty + 8 * a, C::EPI_WARPS * CG);  // one arrival per epilogue warp of the pair
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<CG>(ptx::smem_u32(tmem_slot), C::TMEM_COLS);
  ptx::tc_fence_before();
  if constexpr (CL > 1) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  // Register split (launch: 168 per thread): the producer / MMA warpgroup
  // needs few, the two epilogue warpgroups get the rest (128*56 + 256*224 = 384*168).
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == 0 && lane == 0) {
    // ===== TMA producer =====
    const uint64_t polA = make_policy(g.pol_a, Epi::kAStreams);
    const uint64_t polB = make_policy(g.pol_b, !Epi::kAStreams);
    uint32_t it = 0;
    for (int u = cluster; u < num_units; u += nclusters) {
      int mc, nb;
      tile_coords(gc, unit_tile(u), mc, nb);
      const int mb = mc * MC + int(pair);
      const int m0 = mb * C::BM + int(rank) * C::BM_CTA;
      const int n0 = nb * C::BN_TILE + int(rank) * C::B_HALF_ROWS;  // + h * C::BN for N half h
      const int kbase = unit_kb0(u), nkb = unit_nkb(u);
      for (int kb = kbase; kb < kbase + nkb; ++kb, ++it) {
        const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1u;
        // Wave lockstep: the clusters of one wave of the persistent schedule
        // stay within ~2 epochs (lock_epoch k-blocks) of each other, so
        // co-scheduled tiles sharing an operand band read it at nearly the
        // same K position -- L2 hits instead of DRAM re-reads (dX: 24 -> 15
        // GB per launch), which under the power cap is clock.  Deadlock
        // free: a cluster only waits for members of its own wave to reach an
        // earlier epoch, which needs nothing from a later wave.
        if (g.lockstep && rank == 0 && (kb - kbase) % g.lock_epoch == 0) {
          const int wave = u / nclusters, q = (kb - kbase) / g.lock_epoch;
          const int members = min(nclusters, num_units - wave * nclusters);
          int* cnt = g.lockstep + int64_t(wave) * g.lock_stride;
          atomicAdd(cnt + q, 1);  // reached epoch q
          for (int v = members; q > 0;) {  // every member has reached epoch q - 1
            asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt + q - 1) : "memory");
            if (v >= members) break;
            __nanosleep(64);
          }
        }
        ptx::mbar_wait(bar_empty + 8 * s, ph ^ 1u);
        // The leader's barrier expects the bytes landing in BOTH CTAs of its
        // pair; the peer only issues TMA (a remote arrive costs a GPU-scope
        // membar per stage).
        if (rank == 0) ptx::mbar_arrive_expect_tx(bar_full + 8 * s, C::STAGE_BYTES * CG);
        const uint32_t fb = bar_full + 8 * s;
        const uint32_t a_dst = sA + s * C::A_BYTES, b_dst = sB + s * C::B_BYTES;
        const int k0 = kb * C::BK;
        auto load = [&](const CUtensorMap* m, uint32_t dst, int c0, int c1, uint64_t pol) {
          if constexpr (CG == 1) ptx::tma_load_2d(m, fb, dst, c0, c1, pol);
          else ptx::tma_load_2d_cg2(m, fb & 0xFEFFFFFFu, dst, c0, c1, pol);
        };
        if constexpr (!A_MN) {
          load(&tmA, a_dst, k0, m0, polA);
        } else {
#pragma unroll
          for (int j = 0; j < C::BM_CTA / 64; ++j) load(&tmA, a_dst + j * 8192, m0 + 64 * j, k0, polA);
        }
        if constexpr (MC == 2) {
          // my half (64 rows / 64 cols) of this CTA's B block, multicast to the
          // same-rank CTA of both pairs
          const uint16_t mask = uint16_t((1u << rank) | (1u << (CG + rank)));
          if constexpr (!B_MN)
            ptx::tma_load_2d_cg2_mc(&tmB, fb, b_dst + pair * 8192, k0, n0 + int(pair) * 64, mask, polB);
          else
            ptx::tma_load_2d_cg2_mc(&tmB, fb, b_dst + pair * 8192, n0 + int(pair) * 64, k0, mask, polB);
        } else if constexpr (!B_MN) {
#pragma unroll
          for (int hh = 0; hh < NH; ++hh)
            load(&tmB, b_dst + hh * C::B_HALF_ROWS * 128, k0, n0 + hh * C::BN, polB);
        } else {
#pragma unroll
          for (int hh = 0; hh < NH; ++hh)
#pragma unroll
            for (int j = 0; j < C::B_HALF_ROWS / 64; ++j)
              load(&tmB, b_dst + hh * C::B_HALF_ROWS * 128 + j * 8192, n0 + hh * C::BN + 64 * j, k0, polB);
        }
      }
    }
  } else if (NH == 2 && warp == 1 && lane == 0 && rank == 0) {
    // ===== MMA issuer, 512-wide tiles: staggered N halves =====
    // The tile's two 256-column halves are separate accumulators (TMEM
    // columns [0,256) and [256,512)) released separately by the epilogue.
    // Around tile boundaries the halves run D k-blocks apart, so each half's
    // epilogue overlaps MMAs of the other half instead of idling the tensor
    // pipe:
    //   tile end   : H0(K-D..K-1), commit full[0] | H1(K-D..K-1), commit full[1]
    //                 (epilogue of half 0 runs under H1's last D k-blocks)
    //   tile start : wait empty[0], H0(0..D-1) | wait empty[1], H1(0..D-1)
    //                 (epilogue of half 1 runs under H0's first D k-blocks)
    // D <= STAGES (the D k-blocks stay resident in smem until H1 has read
    // them) and D <= K/2 (start and end groups disjoint).
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(C::BM, C::BN, A_MN, B_MN);
    uint32_t it0 = 0, tc = 0;
    auto issue = [&](int kb, int hh) {
      const uint32_t s = (it0 + kb) % C::STAGES;
      const uint32_t a_base = sA + s * C::A_BYTES, bh = sB + s * C::B_BYTES + hh * C::B_HALF_ROWS * 128;
      const uint32_t d = tmem_base + hh * C::BN;
#pragma unroll
      for (int kk = 0; kk < C::BK / C::UK; ++kk) {
        const uint64_t ad = A_MN ? ptx::sdesc_sw128(a_base + kk * 2048, 8192, 1024)
                                 : ptx::sdesc_sw128(a_base + kk * 32, 16, 1024);
        const uint64_t bd = B_MN ? ptx::sdesc_sw128(bh + kk * 2048, 8192, 1024) : ptx::sdesc_sw128(bh + kk * 32, 16, 1024);
        ptx::mma_bf16<CG>(d, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
      }
    };
    // probe (g.prof, CTA 0): cycles the issuer spent waiting for smem stages / accumulators
    const bool probe = VP_GEMM_PROBE && g.prof != nullptr && blockIdx.x == 0;
    unsigned long long w_full = 0, w_acc = 0;
    auto wait_full = [&](int kb) {
      const uint32_t it = it0 + kb;
      const unsigned long long c0 = probe ? clock64() : 0;
      ptx::mbar_wait(bar_full + 8 * (it % C::STAGES), (it / C::STAGES) & 1u);
      if (probe) w_full += clock64() - c0;
      ptx::tc_fence_after();
    };
    auto release = [&](int kb) { ptx::mma_commit<CG>(bar_empty + 8 * ((it0 + kb) % C::STAGES), pair_mask); };
    auto wait_acc = [&](int hh) {
      const unsigned long long c0 = probe ? clock64() : 0;
      ptx::mbar_wait_cluster(bar_tempty + 8 * hh, (tc & 1u) ^ 1u);
      if (probe) w_acc += clock64() - c0;
      ptx::tc_fence_after();
    };
    for (int u = cluster; u < num_units; u += nclusters, ++tc) {
      const int K = unit_nkb(u);
      const int D = min(C::STAGES, K / 2);
      wait_acc(0);
      for (int kb = 0; kb < D; ++kb) {
        wait_full(kb);
        issue(kb, 0);
      }
      wait_acc(1);
      for (int kb = 0; kb < D; ++kb) {
        issue(kb, 1);
        release(kb);
      }
      for (int kb = D; kb < K - D; ++kb) {
        wait_full(kb);
        issue(kb, 0);
        issue(kb, 1);
        release(kb);
      }
      for (int kb = K - D; kb < K; ++kb) {
        wait_full(kb);
        issue(kb, 0);
      }
      ptx::mma_commit<CG>(bar_tfull, pair_mask);
      for (int kb = K - D; kb < K; ++kb) {
        issue(kb, 1);
        release(kb);
      }
      ptx::mma_commit<CG>(bar_tfull + 8, pair_mask);
      it0 += uint32_t(K);
    }
    if (probe) {
      g.prof[4] = w_full;
      g.prof[5] = w_acc;
    }
  } else if (NH == 1 && warp == 1 && lane == 0 && rank == 0) {
    // ===== MMA issuer (pair leader, one thread) =====
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(C::BM, C::BN, A_MN, B_MN);
    constexpr uint16_t all_mask = uint16_t((1u << CL) - 1u);
    uint32_t it = 0, tc = 0;
    for (int u = cluster; u < num_units; u += nclusters, ++tc) {
      const int nkb = unit_nkb(u);
      const uint32_t acc = tc % NACC, aph = (tc / NACC) & 1u;
      if constexpr (CG == 2) ptx::mbar_wait_cluster(bar_tempty + 8 * acc, aph ^ 1u);
      else ptx::mbar_wait(bar_tempty + 8 * acc, aph ^ 1u);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * C::BN;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1u;
        ptx::mbar_wait(bar_full + 8 * s, ph);
        ptx::tc_fence_after();
        const uint32_t a_base = sA + s * C::A_BYTES, b_base = sB + s * C::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::BK / C::UK; ++kk) {
          // K-major: advance 32 B inside the 128 B swizzle row; SBO = 8 rows.
          // MN-major: advance 16 K-rows (2 KB); LBO = 64-wide MN atom (8 KB box).
          const uint64_t ad = A_MN ? ptx::sdesc_sw128(a_base + kk * 2048, 8192, 1024)
                                   : ptx::sdesc_sw128(a_base + kk * 32, 16, 1024);
#pragma unroll
          for (int hh = 0; hh < NH; ++hh) {
            const uint32_t bh = b_base + hh * C::B_HALF_ROWS * 128;
            const uint64_t bd = B_MN ? ptx::sdesc_sw128(bh + kk * 2048, 8192, 1024)
                                     : ptx::sdesc_sw128(bh + kk * 32, 16, 1024);
            ptx::mma_bf16<CG>(d + hh * C::BN, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
        }
        // free the stage in every CTA whose smem this pair read (all CTAs of
        // the cluster when B was multicast)
        ptx::mma_commit<CG>(bar_empty + 8 * s, MC == 2 ? all_mask : pair_mask);
      }
      ptx::mma_commit<CG>(bar_tfull + 8 * acc, pair_mask);
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ===== epilogue: 8 warps =====
    // warp 4 + ew reads TMEM lanes 32 * (ew % 4) .. +31 (the lane quadrant a
    // warp may access is fixed by warp id % 4) and column group ew / 4, i.e.
    // 128 of the 256 accumulator columns of each N half.
    const int ew = warp - 4, quad = ew & 3, cgp = ew >> 2;
    Stager sg(stg + uint32_t(ew) * uint32_t(C::STG_WARP));
    if (g.store_evict_first) {
      sg.hint = true;
      sg.pol = ptx::policy_evict_first();
    }
    sg.probe = VP_GEMM_PROBE && g.prof != nullptr && blockIdx.x == 0 && ew == 0;
    const bool probe = sg.probe;
    uint32_t tc = 0;
    unsigned long long epi_wait_cyc = 0, epi_work_cyc = 0;  // probe (CTA 0, warp 4)
    for (int u = cluster; u < num_units; u += nclusters, ++tc) {
      int mc, nb;
      const int t = unit_tile(u), sp = unit_split(u);
      tile_coords(gc, t, mc, nb);
      const int mb = mc * MC + int(pair);
      int* flag = (g.splits > 1 && g.split_ws == nullptr && !g.split_indep) ? g.split_flags + 2 * t + int(rank)
                                                                               : nullptr;
      const int row = mb * C::BM + int(rank) * C::BM_CTA + quad * 32 + lane;
      const typename Epi::Pre pre = Epi::prepare(ep, g, row, nb * C::BN_TILE);
      // one accumulator per N half (NH == 2, released separately: see the
      // staggered issuer) or one double-buffered 256-column accumulator (NH == 1)
      constexpr int NWAIT = NH == 2 ? 2 : 1;
#pragma unroll 1
      for (int hw = 0; hw < NWAIT; ++hw) {
        const uint32_t slot = NH == 2 ? uint32_t(hw) : tc % NACC;
        const uint32_t par = NH == 2 ? (tc & 1u) : ((tc / NACC) & 1u);
        const unsigned long long c0 = probe ? clock64() : 0;
        if (g.epi_wait) ptx::mbar_wait_backoff(bar_tfull + 8 * slot, par);
        else ptx::mbar_wait(bar_tfull + 8 * slot, par);
        ptx::tc_fence_after();
        const unsigned long long c1 = probe ? clock64() : 0;
        if constexpr (Epi::kEarly && NH == 2) {
          // Early release: this warp's 128 accumulator columns of the half go
          // to registers (4 x tcgen05.ld, one wait) and the half is handed back
          // to the MMA issuer at once; the epilogue math and stores then run
          // under the next tile's MMAs instead of inside the stagger window.
          const int col0 = nb * C::BN_TILE + hw * C::BN + cgp * kEpiCols;
          const uint32_t taddr = tmem_base + uint32_t(hw * C::BN + cgp * kEpiCols) + (uint32_t(quad * 32) << 16);
          uint32_t acc[kEpiCols];
          tmem_load_all(taddr, acc);
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_remote(bar_tempty + 8 * slot, leader);
          if (hw == 0 && flag && sp > 0) split_wait(flag, g.flag_base + sp);
          if (col0 < g.N) Epi::apply_regs(ep, g, acc, row, col0, col0 / kEpiCols, sg, pre, sp);
          if (probe && lane == 0) {
            epi_wait_cyc += c1 - c0;
            epi_work_cyc += clock64() - c1;
          }
        } else {
        if (hw == 0 && flag && sp > 0) split_wait(flag, g.flag_base + sp);
#pragma unroll 1
        for (int hh = (NH == 2 ? hw : 0); hh < (NH == 2 ? hw + 1 : NH); ++hh) {
          const int col0 = nb * C::BN_TILE + hh * C::BN + cgp * kEpiCols;
          const uint32_t taddr = tmem_base + (NH == 2 ? 0u : slot * C::BN) + uint32_t(hh * C::BN + cgp * kEpiCols) +
                                 (uint32_t(quad * 32) << 16);
          // a ragged last tile's trailing column groups lie wholly past N:
          // no columns, no stats slot, nothing to store
#if VP_EPI_MODE == 0 || VP_EPI_MODE >= 3
          if (col0 < g.N) Epi::apply(ep, g, taddr, row, col0, col0 / kEpiCols, sg, pre, sp);
#elif VP_EPI_MODE == 1
          // probe: TMEM loads only (results discarded)
          tmem_chunks(taddr, 4, [&](uint32_t (&r)[32], int) {
            uint32_t x = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) x ^= r[j];
            if (x == 0x9e3779b9u && g.prof) g.prof[15] = x;
          });
#endif
        }
        if (probe && lane == 0) {
          epi_wait_cyc += c1 - c0;
          epi_work_cyc += clock64() - c1;
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) ptx::mbar_arrive(bar_tempty + 8 * slot);
          else ptx::mbar_arrive_remote(bar_tempty + 8 * slot, leader);
        }
        }
      }
      if (flag) split_done(flag, g.flag_base + sp + 1, sg);
    }
    sg.drain();
    if (probe && lane == 0) {
      g.prof[6] = epi_wait_cyc;
      g.prof[7] = epi_work_cyc;
      g.prof[8] = sg.wait_cyc;
    }
  }
  __syncwarp();
  ptx::tc_fence_before();
  if constexpr (CL > 1) ptx::cluster_sync(); else __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
  }
  if (g.prof && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g.prof[2] = clock64();
    g.prof[3] = t;
  }
}

// ---------------------------------------------------------------------------
// Epilogues.  apply() runs on one epilogue warp: thread `lane` owns
// accumulator row `row` (may be >= M: masked), columns [col0, col0 + 128).
// tcgen05.ld is warp-collective, so loads stay outside row masks.
//
// Stores go through a per-warp smem staging box and TMA (Params::use_tma):
// the warp writes a 32-row x 64-byte box in the SWIZZLE_64B layout (each
// thread one row, 16-byte chunks XOR-permuted by row: bank-conflict free)
// and one lane issues cp.async.bulk.tensor.  The global writes are full
// lines and asynchronous, so the epilogue finishes (and releases its TMEM
// accumulator) in a fraction of the time per-row st.global takes; rows and
// columns outside the tensor are clipped by the TMA unit.  use_tma = 0 keeps
// direct stores (unaligned buffers).
// ---------------------------------------------------------------------------

// D -> fp32 out (row-major, ldo), optionally also the per-(row, tile) max of
// the valid columns (naive F1: logits + local max).
struct EpiStoreF32 {
  static constexpr bool kAStreams = true;
  static constexpr bool kEarly = VP_F32_EARLY != 0;
  struct Params {
    float* out;
    int64_t ldo;
    float* tile_max;         // optional [tiles_n x ld_stats]
    int64_t ld_stats;
    const float* row_scale;  // optional per-row factor applied on store
    int accumulate = 0;      // out += D instead of out = D (gradient accumulation)
    // 0: per-row st.global (unaligned outputs); 1: smem staging + TMA store
    // through `map` (fp32 [M x N], 32 x 32 boxes, SWIZZLE_128B).  (A direct
    // coalesced store from the 16x256b TMEM layout measured slower: dW 92 ->
    // 85% of MMA-ideal cycles.)
    int use_tma = 0;
    CUtensorMap map;
    CUtensorMap ws_map;  // parallel split-K workspace (fp32 [S * ws_rows x N])
    // Routed output (the fused dX -> reduce-scatter over peer memory): rows
    // [o * route_rows, (o + 1) * route_rows) of split unit sp are stored to
    // route_out[o * route_splits + sp], slot sp of the owning rank o's buffer
    // (local, peer-enabled or IPC-mapped; row stride ldo), at local row
    // (row - o * route_rows), by the per-thread 16-byte stores (use_tma = 0):
    // plain st.global over NVLink, the most basic peer access.  Long-K GEMMs
    // (dX: K = V_k) spend a negligible share of their time in the epilogue.
    // Split units are independent (each into its own slot; the owner adds
    // them in split order).  route_n = 0: the plain output.
    int route_n = 0;
    int route_rows = 0;
    int route_splits = 1;
    float* route_out[kMaxRoute];
  };
  // per-row inputs loaded before the accumulator is waited for (hides their latency)
  struct Pre {
    float rs;
  };
  __device__ static Pre prepare(const Params& p, const GemmGeom& g, int row, int /*tile_col0*/) {
    return Pre{(p.row_scale && row < g.M) ? p.row_scale[row] : 1.f};
  }
  __device__ static void apply(const Params& p, const GemmGeom& g, uint32_t taddr, int row, int col0, int nb,
                               Stager& sg, const Pre& pre, int sp) {
    run(p, g, TmemSrc{taddr}, row, col0, nb, sg, pre, sp);
  }
  __device__ static void apply_regs(const Params& p, const GemmGeom& g, uint32_t (&acc)[kEpiCols], int row, int col0,
                                    int nb, Stager& sg, const Pre& pre, int sp) {
    run(p, g, RegSrc{acc}, row, col0, nb, sg, pre, sp);
  }
  template <class Src>
  __device__ static __forceinline__ void run(const Params& p, const GemmGeom& g, const Src& src, int row, int col0,
                                             int nb, Stager& sg, const Pre& pre, int sp) {
    const bool row_ok = row < g.M;
    const int nvalid = min(kEpiCols, g.N - col0);
    const int nch = (nvalid + 31) / 32;
    const float rs = pre.rs;
    // parallel split-K: plain stores of this unit's partial into its workspace
    // slice (use_tma is guaranteed by the host); else ordered accumulation
    const bool to_ws = g.split_ws != nullptr;
    const CUtensorMap* omap = to_ws ? &p.ws_map : &p.map;
    const int rbase = to_ws ? sp * g.ws_rows : 0;
    float* obase = p.out;  // direct stores: base and row of this thread's output row
    int orow = row;
    if (p.route_n > 0) {  // (direct stores only, never the workspace: the host checks)
      const int o = min((row - int(threadIdx.x & 31)) / p.route_rows, p.route_n - 1);
      obase = p.route_out[o * p.route_splits + sp];
      orow = row - o * p.route_rows;
    }
    const bool add = !to_ws && p.route_n == 0 && (p.accumulate != 0 || sp > 0);
    float mx = -INFINITY;
    const int row0 = row - int(threadIdx.x & 31);
    if (p.use_tma) {
      src(nch, [&](uint32_t (&r)[32], int c) {
        if (p.row_scale) {
          const uint64_t rs2 = ptx::f2pack(rs, rs);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint64_t v = ptx::fmul2(ptx::f2pack(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])), rs2);
            float lo, hi;
            ptx::f2unpack(v, lo, hi);
            r[2 * j] = __float_as_uint(lo);
            r[2 * j + 1] = __float_as_uint(hi);
          }
        }
        if (p.tile_max) {
          const int nv = nvalid - c * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) mx = fmaxf(mx, __uint_as_float(r[j]));
        }
#if VP_F32_BOX128
        // one 32-column fp32 box per chunk (32 rows x 128 B, SWIZZLE_128B): the
        // warp's whole 4 KB staging area, single-buffered
        if ((threadIdx.x & 31) == 0) ptx::bulk_wait_read<0>();
        __syncwarp();
        {
          const uint32_t rr = threadIdx.x & 31;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            ptx::st_shared_v4(sg.base + rr * 128u + ((uint32_t(q) ^ (rr & 7u)) << 4), r[4 * q], r[4 * q + 1],
                              r[4 * q + 2], r[4 * q + 3]);
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          sg.put(omap, sg.base, col0 + c * 32, row0 + rbase, add);
          ptx::bulk_commit();
        }
#else
        // two 16-column fp32 boxes per chunk, one fence
        const uint32_t b0 = sg.next();
#pragma unroll
        for (int q = 0; q < 4; ++q) ptx::st_shared_v4(Stager::chunk(b0, q), r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
        const uint32_t b1 = sg.next();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ptx::st_shared_v4(Stager::chunk(b1, q), r[16 + 4 * q], r[16 + 4 * q + 1], r[16 + 4 * q + 2], r[16 + 4 * q + 3]);
        sg.flush2(omap, b0, col0 + c * 32, row0 + rbase, b1, col0 + c * 32 + 16, row0 + rbase, add);
#endif
      });
    } else {
      float* dst = obase + int64_t(orow) * p.ldo + col0;
      const bool vec = ((p.ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(obase) & 15) == 0);
      src(nch, [&](uint32_t (&r)[32], int c) {
        const int nv = nvalid - c * 32;
        if (p.row_scale) {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * rs);
        }
        if (p.tile_max) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) mx = fmaxf(mx, __uint_as_float(r[j]));
        }
        if (!row_ok) return;
        if (nv >= 32 && vec) {
          float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            if (add) {
              const float4 o = d4[j];
              v.x += o.x;
              v.y += o.y;
              v.z += o.z;
              v.w += o.w;
            }
            d4[j] = v;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) dst[c * 32 + j] = __uint_as_float(r[j]) + (add ? dst[c * 32 + j] : 0.f);
        }
      });
    }
    if (p.tile_max && row_ok) p.tile_max[int64_t(nb) * p.ld_stats + row] = mx;
  }
};

// K1 fused stats epilogue (forward of the output layer).  For row i and
// vocab tile j (kEpiCols = 128 columns of this shard):
//   m_ij = max_v Y[i,v];  y_tgt[i] = Y[i, g_i - row_begin] when the label falls here;
//   P[i,v] = bf16(exp(Y[i,v] - q_ij)),  s_ij = sum_v exp(Y[i,v] - q_ij),
// where the reference q_ij is ONE value per row, r_i = m_i0 + kRefLift (the
// max of the row's first vocab tile, lifted), published by the j = 0 tiles
// through a release flag per 128-row block; later tiles of the row wait for
// it (tile (m, 0) always precedes (m, j) in the persistent schedule).  A
// per-row reference makes softmax' = P * cfac_i (one factor per row), which
// the dX epilogue and the scaled-X operand of dW absorb: no pass over P is
// needed after K1, and P is rounded to bf16 exactly once.  Rows whose logits
// exceed r_i + kMaxRefGap (exp would overflow) are marked in row_bad and
// re-referenced to the row max after the stats merge.  (The fix_list path
// for tiles stored against their own max is kept for robustness; the wait
// makes it unreachable.)  Full-vocab logits never touch HBM.
struct EpiLogitStats {
  static constexpr bool kAStreams = false;  // A = X is reused by every vocab tile
  static constexpr bool kEarly = VP_K1_EARLY != 0;
  static constexpr float kMaxRefGap = 64.f;  // e^{Y - q} <= e^64: P, its sums and P.W stay finite in fp32
  static constexpr float kRefLift = 16.f;    // r_i sits this far above the first vocab tile's max
  struct Params {
    __nv_bfloat16* P;
    int64_t ldp;
    float* tile_m;          // [tiles_n x ld_stats] tile max
    float* tile_s;          // [tiles_n x ld_stats] exp-sum relative to tile_q
    int64_t ld_stats;
    const int64_t* labels;  // [M] global vocab ids (may be null)
    int64_t row_begin, row_end;
    float* y_tgt;           // [M]
    float* tile_q;          // [tiles_n x ld_stats] reference of P / s for (row, tile)
    float* row_ref;         // [M] r_i
    int* ref_flag;          // [ceil(M/128)] 1 once r of that 128-row block is visible
    int* row_bad;           // [M]
    int* bad_count;         // bad rows appended to bad_list (once each)
    int* bad_list;          // [M]
    int* fix_count;         // (32-row group, tile) pairs stored relative to their own max
    int2* fix_list;         // [ceil(M/32) x tiles_n]
    int use_tma = 0;        // P stored through `map` (bf16 [M x N], 32 x 32 boxes, SWIZZLE_64B)
    CUtensorMap map;
    // logits y = acc * logit_scale + logit_shift[row]: the reference's per-row
    // logit_shift test hook (VM.cpp:41-43; null = 0) and a fault-injection
    // scale (1 = off).  Folded into the exponent: no extra pass.
    const float* logit_shift = nullptr;
    float logit_scale = 1.f;
  };
  // max of the valid columns and the label logit (first pass of a two-pass tile)
  template <class Src>
  __device__ static void scan(const Src& src, int nvalid, int lb, float& mx, float& yt, bool& has_t) {
    float mp[4] = {mx, mx, mx, mx};
    src((nvalid + 31) / 32, [&](uint32_t (&r)[32], int c) {
      const int nv = nvalid - c * 32;
      if (nv >= 32) {
#pragma unroll
        for (int j = 0; j < 32; ++j) mp[j & 3] = fmaxf(mp[j & 3], __uint_as_float(r[j]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) mp[j & 3] = fmaxf(mp[j & 3], __uint_as_float(r[j]));
      }
      const int off = lb - c * 32;
      if (off >= 0 && off < 32 && off < nv) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j == off) yt = __uint_as_float(r[j]);
        has_t = true;
      }
    });
    mx = fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3]));
  }
  // One pass over the 256 accumulator columns of this row: P = bf16(e^{Y - ref}),
  // s = sum e^{Y - ref}; with track = true it also takes the tile max and the
  // label logit (the single-pass path, where ref = r_i is known up front).
  // ref and shift are in logit space (y = acc * logit_scale + shift); mx / yt
  // are tracked in accumulator space.
  template <class Src>
  __device__ static void emit(const Params& p, const Src& src, int row, bool row_ok, int col0, int nvalid,
                              float ref, float shift, int lb, bool track, float& mx, float& yt, bool& has_t,
                              float& sum, Stager& sg) {
    const float kLog2e = 1.4426950408889634f * p.logit_scale;
    const float refs = (ref - shift) * 1.4426950408889634f;
    sum = 0.f;
    const int row0 = row - int(threadIdx.x & 31);
    __nv_bfloat16* dst = p.P + int64_t(row) * p.ldp + col0;
    const bool vec = ((p.ldp & 7) == 0) && ((reinterpret_cast<uintptr_t>(p.P) & 15) == 0);
    const int nch = (nvalid + 31) / 32;
    // independent partial sums (packed f32x2 pairs) and maxima: no serial chains
    uint64_t sp2[2] = {ptx::f2pack(0.f, 0.f), ptx::f2pack(0.f, 0.f)};
    float mp[2] = {mx, mx};
    const uint64_t l2e2 = ptx::f2pack(kLog2e, kLog2e), nref2 = ptx::f2pack(-refs, -refs);
#if !VP_P_BOX128
    uint32_t box0 = 0;  // first box of the pair being filled (TMA path)
#endif
    src(nch, [&](uint32_t (&r)[32], int c) {
      const int nv = nvalid - c * 32;
      uint32_t pk[16];
      if (nv >= 32) {
        // full chunk: no column masks; FFMA2 / FADD2 on column pairs
        if (track) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            mp[j & 1] = fmaxf(mp[j & 1], fmaxf(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])));
        }
#if VP_EPI_MODE == 4
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = r[2 * j] ^ r[2 * j + 1];  // probe: stores without the math
#else
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint64_t x2 =
              ptx::ffma2(ptx::f2pack(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])), l2e2, nref2);
          float x0, x1;
          ptx::f2unpack(x2, x0, x1);
          const float e0 = ptx::ex2(x0);
#if VP_K1_POLY
          const float e1 = ptx::ex2_poly(x1);  // half the exponentials on the FMA pipe
#else
          const float e1 = ptx::ex2(x1);
#endif
          sp2[j & 1] = ptx::fadd2(sp2[j & 1], ptx::f2pack(e0, e1));
          pk[j] = ptx::pack_bf16(e0, e1);
        }
#endif
      } else {
        if (track) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) mp[j & 1] = fmaxf(mp[j & 1], __uint_as_float(r[j]));
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float e0 = (2 * j < nv) ? ptx::ex2(fmaf(__uint_as_float(r[2 * j]), kLog2e, -refs)) : 0.f;
          const float e1 = (2 * j + 1 < nv) ? ptx::ex2(fmaf(__uint_as_float(r[2 * j + 1]), kLog2e, -refs)) : 0.f;
          sp2[j & 1] = ptx::fadd2(sp2[j & 1], ptx::f2pack(e0, e1));
          pk[j] = ptx::pack_bf16(e0, e1);
        }
      }
      if (track) {
        const int off = lb - c * 32;
        if (off >= 0 && off < 32 && off < nv) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j == off) yt = __uint_as_float(r[j]);
          has_t = true;
        }
      }
#if VP_EPI_MODE == 3
      if (pk[0] == 0x12345u && pk[15] == 0x777u) has_t = !has_t;  // probe: math without the stores
      if (false) {
#else
      if (p.use_tma) {
#endif
#if VP_P_BOX128
        // one 64-column bf16 box (32 rows x 128 B, SWIZZLE_128B) per two chunks,
        // the warp's whole 4 KB staging area, single-buffered
        if ((c & 1) == 0) {
          if ((threadIdx.x & 31) == 0) ptx::bulk_wait_read<0>();
          __syncwarp();
        }
        {
          const uint32_t r = threadIdx.x & 31, q0 = uint32_t(c & 1) * 4u;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            ptx::st_shared_v4(sg.base + r * 128u + (((q0 + uint32_t(q)) ^ (r & 7u)) << 4), pk[4 * q], pk[4 * q + 1],
                              pk[4 * q + 2], pk[4 * q + 3]);
        }
        if ((c & 1) || c + 1 == nch) {
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) {
            Stager::put_static(sg, &p.map, sg.base, col0 + (c & ~1) * 32, row0);
            ptx::bulk_commit();
          }
        }
#else
        // one 32-column bf16 box per chunk, flushed in pairs (one fence per
        // two chunks); columns past N are clipped by the TMA unit
        const uint32_t box = sg.next();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ptx::st_shared_v4(Stager::chunk(box, q), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        if (c & 1) sg.flush2(&p.map, box0, col0 + (c - 1) * 32, row0, box, col0 + c * 32, row0);
        else if (c + 1 == nch) sg.flush(&p.map, box, col0 + c * 32, row0);
        else box0 = box;
#endif
      } else if (row_ok) {
        if (nv >= 32 && vec) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j) d4[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        } else {
          uint16_t* d16 = reinterpret_cast<uint16_t*>(dst + c * 32);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) d16[j] = uint16_t((j & 1) ? (pk[j >> 1] >> 16) : (pk[j >> 1] & 0xFFFFu));
        }
      }
    });
    float a0, a1, b0, b1;
    ptx::f2unpack(sp2[0], a0, a1);
    ptx::f2unpack(sp2[1], b0, b1);
    sum = (a0 + b0) + (a1 + b1);
    if (track) mx = fmaxf(mp[0], mp[1]);
  }

  // Per-row inputs loaded before the accumulator is waited for: the label,
  // and (tiles past the first) the row-reference flag and r_i.  A flag still
  // clear here is re-checked in apply().
  struct Pre {
    int64_t label;
    int flag;
    float ref;
    float shift;
  };
  __device__ static int load_flag(const Params& p, int row) {
    int f;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(p.ref_flag + (row >> 7)) : "memory");
    return f;
  }
  __device__ static Pre prepare(const Params& p, const GemmGeom& g, int row, int tile_col0) {
    Pre r{-1, 0, 0.f, 0.f};
    if (row < g.M) {
      if (p.labels) r.label = p.labels[row];
      if (p.logit_shift) r.shift = p.logit_shift[row];
      if (tile_col0 != 0) {
        r.flag = load_flag(p, row);
        if (r.flag) r.ref = p.row_ref[row];
      }
    }
    return r;
  }
  __device__ static void apply(const Params& p, const GemmGeom& g, uint32_t taddr, int row, int col0, int nb,
                               Stager& sg, const Pre& pre, int /*sp: never split*/) {
    run(p, g, TmemSrc{taddr}, row, col0, nb, sg, pre);
  }
  __device__ static void apply_regs(const Params& p, const GemmGeom& g, uint32_t (&acc)[kEpiCols], int row, int col0,
                                    int nb, Stager& sg, const Pre& pre, int /*sp: never split*/) {
    run(p, g, RegSrc{acc}, row, col0, nb, sg, pre);
  }
  template <class Src>
  __device__ static __forceinline__ void run(const Params& p, const GemmGeom& g, const Src& src, int row, int col0,
                                             int nb, Stager& sg, const Pre& pre) {
    const bool row_ok = row < g.M;
    const int lane = threadIdx.x & 31;
    const int nvalid = min(kEpiCols, g.N - col0);
    int lb = -1;
    if (row_ok && pre.label >= p.row_begin && pre.label < p.row_end)
      lb = int(pre.label - p.row_begin) - col0;  // offset inside tile
    const int blk = row >> 7;
    int f = pre.flag;
    float pref = pre.ref;
    if (nb != 0 && !f && row_ok) {
      // Wait for r_i rather than fall back to this tile's own max (which
      // would cost a second bf16 rounding of P in the fix pass).  Deadlock
      // free: under every rasterisation tile (m, 0) precedes all (m, j > 0)
      // in the persistent schedule, all clusters are co-resident, and a tile
      // only ever waits on a smaller tile index.
      f = load_flag(p, row);
      while (!f) {
        __nanosleep(128);
        f = load_flag(p, row);
      }
      pref = p.row_ref[row];
    }
    f = __all_sync(0xffffffffu, f || !row_ok);  // warp-uniform path (rows past M follow their warp)
    (void)blk;
    float mx = -INFINITY, yt = 0.f, sum = 0.f, ref;
    bool has_t = false, own = false, bad = false;
    if (nb == 0 || !f) {
      // two passes: this tile is its own reference (the j = 0 tile defines r_i;
      // an early tile whose row reference is not published yet falls back)
      scan(src, nvalid, lb, mx, yt, has_t);
      mx = mx * p.logit_scale + pre.shift;  // accumulator -> logit space
      yt = yt * p.logit_scale + pre.shift;
      ref = mx;
      if (nb == 0) {
        // r_i = first-tile max + kRefLift: later tiles overflow-check against
        // r_i + kMaxRefGap, i.e. kMaxRefGap + kRefLift nats above the first
        // tile's max, before a row needs the (double-rounding) re-reference;
        // bf16 keeps full relative precision for the smaller values
        ref = mx + kRefLift;
        if (row_ok) p.row_ref[row] = ref;
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps of this CTA
        if (threadIdx.x == 128) {
          __threadfence();
          atomicExch(p.ref_flag + (row >> 7), 1);
        }
      } else {
        own = true;
      }
      float m2 = -INFINITY, y2 = 0.f;
      emit(p, src, row, row_ok, col0, nvalid, ref, pre.shift, lb, false, m2, y2, has_t, sum, sg);
    } else {
      // single pass against the published row reference
      ref = row_ok ? pref : 0.f;
      emit(p, src, row, row_ok, col0, nvalid, ref, pre.shift, lb, true, mx, yt, has_t, sum, sg);
      mx = mx * p.logit_scale + pre.shift;  // accumulator -> logit space
      yt = yt * p.logit_scale + pre.shift;
      bad = row_ok && (mx - ref > kMaxRefGap);  // e^{Y - r} overflowed: redo against the tile max
      if (__ballot_sync(0xffffffffu, bad)) {
        if (bad) ref = mx;
        // the first pass's P boxes must land before they are overwritten
        if (p.use_tma) sg.drain();
        float m2 = -INFINITY, y2 = 0.f;
        emit(p, src, row, row_ok, col0, nvalid, ref, pre.shift, lb, false, m2, y2, has_t, sum, sg);
      }
    }
    if (row_ok) {
      const int64_t o = int64_t(nb) * p.ld_stats + row;
      p.tile_m[o] = mx;
      p.tile_s[o] = sum;
      p.tile_q[o] = ref;
      if (has_t) p.y_tgt[row] = yt;
      if (bad && atomicExch(p.row_bad + row, 1) == 0) p.bad_list[atomicAdd(p.bad_count, 1)] = row;
    }
    if (__ballot_sync(0xffffffffu, own && row_ok) && lane == 0)
      p.fix_list[atomicAdd(p.fix_count, 1)] = make_int2(row >> 5, nb);
  }
};

// Parallel split-K reduction: out[r, :] (+)= sum_{s = 0..S-1} ws[s * ws_rows + r, :]
// in ascending s (fixed order: bitwise deterministic).  4 columns per thread
// (out and ws rows are 16-B aligned: the TMA-store precondition).
__global__ void k_split_reduce(const float* __restrict__ ws, int S, int ws_rows, int64_t ldws, float* __restrict__ out,
                               int64_t ldo, int M, int N, int accumulate) {
  const int n4 = (N + 3) / 4;
  const int64_t total = int64_t(M) * n4;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / n4), c = int(i - int64_t(r) * n4) * 4;
    float4 v = *reinterpret_cast<const float4*>(ws + int64_t(r) * ldws + c);
    for (int sp = 1; sp < S; ++sp) {
      const float4 w = __ldcs(reinterpret_cast<const float4*>(ws + (int64_t(sp) * ws_rows + r) * ldws + c));
      v.x += w.x;
      v.y += w.y;
      v.z += w.z;
      v.w += w.w;
    }
    float* o = out + int64_t(r) * ldo + c;
    if (c + 4 <= N) {
      if (accumulate) {
        const float4 a = *reinterpret_cast<const float4*>(o);
        v.x = a.x + v.x;
        v.y = a.y + v.y;
        v.z = a.z + v.z;
        v.w = a.w + v.w;
      }
      *reinterpret_cast<float4*>(o) = v;
    } else {
      const float vv[4] = {v.x, v.y, v.z, v.w};
      for (int j = 0; j < N - c; ++j) o[j] = (accumulate ? o[j] : 0.f) + vv[j];
    }
  }
}

}  // namespace vp
