// Deterministic segmented scatter-add (input_backward, VM.cpp:238-251, and the
// -G_k^T X one-hot correction of dW):
//
//     dst[r, :] (+)= sign * src[i, :]   for every owned token i with row r,
//
// each row's contributions added in ASCENDING i (the reference's loop order),
// so the result is bit-exact against the fp32 ascending-i restatement no matter
// how the ids are distributed.  Rows are bucketed by a counting sort whose
// per-row segments are ordered afterwards (bitmap / warp rank sort), and the
// adds are split by how often a row occurs:
//
//   c == 1      (most rows of a uniform batch)  one block per row, a straight
//               vectorised row add, no indirection beyond a compact slot;
//   2 <= c < 16 one block per row, all c source rows of a column group in
//               flight, added in order;
//   c >= 16     (hot tokens of a Zipfian batch: BOS, "the", ...)  the row is
//               split into 256-column chunks, one block each; batches of the c
//               source-row pieces are gathered into a shared-memory tile (the
//               next batch in flight while the current one is summed) and
//               every thread adds its column's sequence in order.  A hot row
//               therefore runs on h/256 SMs with ~32 KB in flight each, instead
//               of serialising on one.
//
// Kernels (one stream, in order): k_sc_count (multiplicity + first occurrence
// per row), k_sc_plan (slot lists, segment allocation), k_sc_fill (bucket the
// repeated rows' token indices), k_sc_sort (order each segment), k_sc_apply.
// Slot lists are filled with atomics, so their ORDER varies run to run — but
// each row is owned by exactly one slot (or one set of disjoint column
// chunks) and its sum order is fixed, so the output bits do not.
#pragma once
#include <cuda_bf16.h>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "sm100_ptx.cuh"

namespace vp {

constexpr int kScHot = 16;         // occurrences from which a row is split into column chunks
constexpr int kScChunk = 256;      // columns per hot chunk (= threads per block)
constexpr int kScThreads = 256;
constexpr int kScRingBytes = 32768;  // row tile of a hot chunk (dynamic smem)
constexpr int kScWin = 1024;         // hot chunk: segment indices staged in shared memory

// counters (zeroed with the per-row arrays)
enum { kScUni = 0, kScSmall = 1, kScHotSlots = 2, kScSeg = 3, kScRep = 4, kScCtrs = 8 };

struct ScatterWs {
  int* cnt;    // [rows] multiplicity
  int* headr;  // [rows] n - first i (0 = row not present)
  int* fill;   // [rows] fill cursor of the row's segment
  int* seg;    // [rows] segment start (repeated rows)
  int* ctr;    // [kScCtrs]
  int* list;   // [n] segments of the repeated rows (token indices)
  int2* uni;   // [n] {r, i}
  int4* small; // [n] {r, seg, c, 0}
  int4* hot;   // [hot_cap] {r, seg, c, chunk}
  int4* rep;   // [n] {r, seg, c, 0}: rows to sort
  int hot_cap;
};

__device__ __forceinline__ bool sc_owned(int64_t t, int64_t rb, int64_t re) { return t >= rb && t < re; }

__global__ void k_sc_count(const int64_t* __restrict__ tok, int n, int64_t rb, int64_t re, ScatterWs w,
                           int* __restrict__ err, int err_bit) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t t = tok[i];
    if (t < 0 && err_bit) atomicOr(err, err_bit);
    if (sc_owned(t, rb, re)) {
      const int r = int(t - rb);
      atomicAdd(w.cnt + r, 1);
      atomicMax(w.headr + r, n - i);
    }
  }
}

__global__ void k_sc_plan(const int64_t* __restrict__ tok, int n, int64_t rb, int64_t re, int nchunks, ScatterWs w) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t t = tok[i];
    if (!sc_owned(t, rb, re)) continue;
    const int r = int(t - rb);
    if (n - w.headr[r] != i) continue;  // not the row's first occurrence
    const int c = w.cnt[r];
    if (c == 1) {
      w.uni[atomicAdd(w.ctr + kScUni, 1)] = make_int2(r, i);
      continue;
    }
    const int s = atomicAdd(w.ctr + kScSeg, c);
    w.seg[r] = s;
    w.rep[atomicAdd(w.ctr + kScRep, 1)] = make_int4(r, s, c, 0);
    if (c < kScHot) {
      w.small[atomicAdd(w.ctr + kScSmall, 1)] = make_int4(r, s, c, 0);
    } else {
      const int b = atomicAdd(w.ctr + kScHotSlots, nchunks);
      for (int q = 0; q < nchunks && b + q < w.hot_cap; ++q) w.hot[b + q] = make_int4(r, s, c, q);
    }
  }
}

__global__ void k_sc_fill(const int64_t* __restrict__ tok, int n, int64_t rb, int64_t re, ScatterWs w) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t t = tok[i];
    if (!sc_owned(t, rb, re)) continue;
    const int r = int(t - rb);
    if (w.cnt[r] < 2) continue;
    w.list[w.seg[r] + atomicAdd(w.fill + r, 1)] = i;
  }
}

// Orders every repeated row's segment ascending.  c <= 32: one warp, rank by
// comparison; larger: a bitmap of the n token indices in shared memory
// (dynamic, ceil(n / 32) words), compacted in order by a block prefix sum.
__device__ __forceinline__ void sc_sort_segments(int n, const ScatterWs& w, unsigned* sc_bits, int* wsum);
__global__ void __launch_bounds__(kScThreads) k_sc_sort(int n, ScatterWs w) {
  extern __shared__ unsigned sc_bits[];
  __shared__ int wsum[kScThreads / 32];
  sc_sort_segments(n, w, sc_bits, wsum);
}
__device__ __forceinline__ void sc_sort_segments(int n, const ScatterWs& w, unsigned* sc_bits, int* wsum) {
  const int nw = (n + 31) >> 5;
  const int nrep = w.ctr[kScRep];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = blockIdx.x; q < nrep; q += gridDim.x) {
    const int4 e = w.rep[q];
    int* segp = w.list + e.y;
    const int c = e.z;
    if (c <= 32) {
      if (warp == 0) {
        const int v = lane < c ? segp[lane] : 0x7fffffff;
        int rank = 0;
        for (int k = 0; k < c; ++k) rank += __shfl_sync(0xffffffffu, v, k) < v;
        __syncwarp();
        if (lane < c) segp[rank] = v;
      }
      continue;  // block-uniform branch: no barrier skipped by part of the block
    }
    for (int k = threadIdx.x; k < nw; k += blockDim.x) sc_bits[k] = 0u;
    __syncthreads();
    for (int k = threadIdx.x; k < c; k += blockDim.x) {
      const int v = segp[k];
      atomicOr(sc_bits + (v >> 5), 1u << (v & 31));
    }
    __syncthreads();
    // contiguous word ranges per thread, popcount, block exclusive scan
    const int per = (nw + blockDim.x - 1) / blockDim.x;
    const int w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
    int cntm = 0;
    for (int k = w0; k < w1; ++k) cntm += __popc(sc_bits[k]);
    int incl = cntm;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int base = 0;
    for (int k = 0; k < warp; ++k) base += wsum[k];
    int pos = base + incl - cntm;
    for (int k = w0; k < w1; ++k) {
      unsigned b = sc_bits[k];
      while (b) {
        const int bit = __ffs(b) - 1;
        segp[pos++] = (k << 5) + bit;
        b &= b - 1;
      }
    }
    __syncthreads();  // sc_bits / wsum reused by the next segment
  }
}

// The four planning kernels in one cooperative launch (grid-wide barriers
// between the phases): zero the per-row state of the rows this batch touches
// (instead of a memset of every row of the shard), count, plan, fill, sort.
// The launch gaps and the shard-sized memset were most of the planning time.
__global__ void __launch_bounds__(kScThreads) k_sc_prepare(const int64_t* __restrict__ tok, int n, int64_t rb,
                                                         int64_t re, int nchunks, ScatterWs w, int* __restrict__ err,
                                                         int err_bit) {
  extern __shared__ unsigned sc_bits[];
  __shared__ int wsum[kScThreads / 32];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = t0; i < n; i += nt) {
    const int64_t t = tok[i];
    if (sc_owned(t, rb, re)) {
      const int r = int(t - rb);
      w.cnt[r] = 0;
      w.headr[r] = 0;
      w.fill[r] = 0;
    }
  }
  if (t0 < kScCtrs) w.ctr[t0] = 0;
  grid.sync();
  for (int i = t0; i < n; i += nt) {
    const int64_t t = tok[i];
    if (t < 0 && err_bit) atomicOr(err, err_bit);
    if (sc_owned(t, rb, re)) {
      const int r = int(t - rb);
      atomicAdd(w.cnt + r, 1);
      atomicMax(w.headr + r, n - i);
    }
  }
  grid.sync();
  for (int i = t0; i < n; i += nt) {
    const int64_t t = tok[i];
    if (!sc_owned(t, rb, re)) continue;
    const int r = int(t - rb);
    if (n - w.headr[r] != i) continue;
    const int c = w.cnt[r];
    if (c == 1) {
      w.uni[atomicAdd(w.ctr + kScUni, 1)] = make_int2(r, i);
      continue;
    }
    const int s = atomicAdd(w.ctr + kScSeg, c);
    w.seg[r] = s;
    w.rep[atomicAdd(w.ctr + kScRep, 1)] = make_int4(r, s, c, 0);
    if (c < kScHot) {
      w.small[atomicAdd(w.ctr + kScSmall, 1)] = make_int4(r, s, c, 0);
    } else {
      const int b = atomicAdd(w.ctr + kScHotSlots, nchunks);
      for (int q = 0; q < nchunks && b + q < w.hot_cap; ++q) w.hot[b + q] = make_int4(r, s, c, q);
    }
  }
  grid.sync();
  for (int i = t0; i < n; i += nt) {
    const int64_t t = tok[i];
    if (!sc_owned(t, rb, re)) continue;
    const int r = int(t - rb);
    if (w.cnt[r] < 2) continue;
    w.list[w.seg[r] + atomicAdd(w.fill + r, 1)] = i;
  }
  grid.sync();
  sc_sort_segments(n, w, sc_bits, wsum);
}

template <typename Src>
__device__ __forceinline__ float4 sc_load4(const Src* p) {
  if constexpr (sizeof(Src) == 2) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  } else {
    return *reinterpret_cast<const float4*>(p);
  }
}

__device__ __forceinline__ void sc_axpy(float4& a, float s, const float4& v) {
  a.x += s * v.x;
  a.y += s * v.y;
  a.z += s * v.z;
  a.w += s * v.w;
}

template <typename Src>
__device__ __forceinline__ float sc_elem(uint32_t saddr) {
  if constexpr (sizeof(Src) == 2) {
    unsigned short u;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(u) : "r"(saddr));
    return __uint_as_float(uint32_t(u) << 16);
  } else {
    float f;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(f) : "r"(saddr));
    return f;
  }
}

// Slots: [0, n_hot) hot chunks, then small rows, then unique rows (hot work
// first: it is the longest).  One block of 256 threads per slot.
template <typename Src>
__global__ void __launch_bounds__(kScThreads) k_sc_apply(ScatterWs w, const Src* __restrict__ src, int64_t lds, int h,
                                                       float sign, float* __restrict__ dst, int64_t ldd,
                                                       int accumulate) {
  extern __shared__ __align__(128) uint8_t sc_ring[];
  __shared__ int sc_idx[kScWin];
  const int n_hot = min(w.ctr[kScHotSlots], w.hot_cap), n_small = w.ctr[kScSmall], n_uni = w.ctr[kScUni];
  const int slot = blockIdx.x;
  if (slot >= n_hot + n_small + n_uni) return;
  if (slot < n_hot) {
    // ---- hot chunk: 256 columns [col0, col0 + cw) of row r, c >= kScHot
    // source rows in ascending i.  Batches of kB rows are gathered with 16-byte
    // loads (all threads, kU independent loads each, the NEXT batch in flight
    // while the current one is summed) into a shared-memory tile; every thread
    // then adds its own column down the batch in order.  (Small TMA bulk
    // copies measured 5x slower here: one 512-byte copy per row piece leaves
    // too few bytes in flight per SM.)
    const int4 e = w.hot[slot];
    const int* seg = w.list + e.y;
    const int c = e.z, col0 = e.w * kScChunk, cw = min(kScChunk, h - col0);
    if (cw <= 0) return;
    constexpr int kVec = 16 / int(sizeof(Src));        // elements per 16-byte load
    constexpr int kTpr = kScChunk / kVec;              // threads per row piece (32 bf16 / 64 fp32)
    constexpr int kRpi = kScThreads / kTpr;            // rows per load instruction (8 / 4)
    constexpr int kU = 8;                              // loads in flight per thread
    constexpr int kB = kRpi * kU;                      // rows per batch (64 / 32)
    static_assert(kB * kScChunk * int(sizeof(Src)) <= kScRingBytes, "tile");
    Src* tile = reinterpret_cast<Src*>(sc_ring);
    const int lr = threadIdx.x / kTpr, lc = (threadIdx.x % kTpr) * kVec;  // my row-in-instruction / column
    int win0 = 0;
    auto load_window = [&](int from) {  // whole block
      win0 = from;
      for (int k = threadIdx.x; k < kScWin && from + k < c; k += blockDim.x) sc_idx[k] = seg[from + k];
    };
    uint4 v[kU];
    auto gather = [&](int j0) {  // rows j0 .. j0 + kB - 1 -> registers
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = j0 + u * kRpi + lr;
        v[u] = (j < c && lc < cw)
                   ? *reinterpret_cast<const uint4*>(src + int64_t(sc_idx[j - win0]) * lds + col0 + lc)
                   : make_uint4(0u, 0u, 0u, 0u);
      }
    };
    auto stash = [&]() {
#pragma unroll
      for (int u = 0; u < kU; ++u) *reinterpret_cast<uint4*>(tile + (u * kRpi + lr) * kScChunk + lc) = v[u];
    };
    const int col = threadIdx.x;
    float* d = dst + int64_t(e.x) * ldd + col0;
    float acc = (accumulate && col < cw) ? d[col] : 0.f;
    load_window(0);
    __syncthreads();
    gather(0);
    for (int j0 = 0; j0 < c; j0 += kB) {
      stash();
      __syncthreads();  // tile = batch j0
      const int nxt = j0 + kB;
      if (nxt < c && nxt + kB > win0 + kScWin) {  // block-uniform
        __syncthreads();
        load_window(nxt);
        __syncthreads();
      }
      if (nxt < c) gather(nxt);  // in flight while this batch is summed
      const int nr = min(kB, c - j0);
      if (col < cw)
        for (int k = 0; k < nr; ++k) {
          float x;
          if constexpr (sizeof(Src) == 2) x = __bfloat162float(tile[k * kScChunk + col]);
          else x = tile[k * kScChunk + col];
          acc += sign * x;
        }
      __syncthreads();  // batch summed: the tile may be overwritten
    }
    if (col < cw) d[col] = acc;
    return;
  }
  if (slot < n_hot + n_small) {
    // ---- 2 <= c < 16: whole row; per column group the sources are loaded
    // four at a time and added in order
    const int4 e = w.small[slot - n_hot];
    const int* seg = w.list + e.y;
    const int c = e.z;
    float* d = dst + int64_t(e.x) * ldd;
    for (int c0 = threadIdx.x * 4; c0 < h; c0 += kScThreads * 4) {
      float4 acc = accumulate ? *reinterpret_cast<const float4*>(d + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q0 = 0; q0 < c; q0 += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (q0 + u < c) v[u] = sc_load4(src + int64_t(seg[q0 + u]) * lds + c0);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (q0 + u < c) sc_axpy(acc, sign, v[u]);
      }
      *reinterpret_cast<float4*>(d + c0) = acc;
    }
    return;
  }
  // ---- c == 1: one vectorised row add, four column passes in flight
  const int2 e = w.uni[slot - n_hot - n_small];
  float* d = dst + int64_t(e.x) * ldd;
  const Src* sp = src + int64_t(e.y) * lds;
  constexpr int kPass = kScThreads * 4;
  for (int c0 = threadIdx.x * 4; c0 < h; c0 += 4 * kPass) {
    float4 acc[4], v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cc = c0 + u * kPass;
      if (cc < h) {
        acc[u] = accumulate ? *reinterpret_cast<const float4*>(d + cc) : make_float4(0.f, 0.f, 0.f, 0.f);
        v[u] = sc_load4(sp + cc);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cc = c0 + u * kPass;
      if (cc < h) {
        sc_axpy(acc[u], sign, v[u]);
        *reinterpret_cast<float4*>(d + cc) = acc[u];
      }
    }
  }
}

}  // namespace vp
