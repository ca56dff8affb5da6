// Vocabulary-layer kernels around the tcgen05 GEMMs: stats reductions and
// merges, softmax normalisation of the stored P tiles, the alg2 C1 combine,
// loss, one-hot corrections, the input-layer masked gather and the
// deterministic sort-based scatter-add.  All HBM-bound: 16-byte vector
// accesses, grids sized in multiples of the SM count.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace vp {

constexpr int kTileN = 128;          // K1 vocab tile width (stats granularity) = kEpiCols of the GEMM epilogue
constexpr int kMaxLocalShards = 16;  // shards simulated on one device
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float fast_exp(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * kLog2e));
  return y;
}

// ---------------------------------------------------------------------------
// Per-row reduction of the K1 per-tile stats (m_ij, s_ij), tiles merged in
// ascending j (fixed order: deterministic).  One warp-column per row group:
// block = 256 threads = 8 warps x 32 rows; warp w takes tiles j = w, w+8, ...
// then the 8 partials merge in w order.  s may be null (max only: naive F1).
// ---------------------------------------------------------------------------
__global__ void k_stats_reduce(const float* __restrict__ tile_m, const float* __restrict__ tile_s, int ntiles,
                               int64_t ld, int n, float* __restrict__ m_out, float* __restrict__ s_out) {
  __shared__ float sm[8][32], ss[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = blockIdx.x * 32 + lane;
  float m = -INFINITY, s = 0.f;
  if (row < n) {
    for (int j = w; j < ntiles; j += 8) {
      const float mj = tile_m[int64_t(j) * ld + row];
      if (tile_s) {
        const float sj = tile_s[int64_t(j) * ld + row];
        const float nm = fmaxf(m, mj);
        s = s * fast_exp(m - nm) + sj * fast_exp(mj - nm);
        m = nm;
      } else {
        m = fmaxf(m, mj);
      }
    }
  }
  sm[w][lane] = m;
  ss[w][lane] = s;
  __syncthreads();
  if (w == 0 && row < n) {
    float M = sm[0][lane], S = ss[0][lane];
    for (int q = 1; q < 8; ++q) {
      const float mq = sm[q][lane];
      if (mq == -INFINITY) continue;
      const float nm = fmaxf(M, mq);
      S = S * fast_exp(M - nm) + ss[q][lane] * fast_exp(mq - nm);
      M = nm;
    }
    m_out[row] = M;
    if (s_out) s_out[row] = S;
  }
}

// Per-row merge of the K1 tile stats when each tile's exp-sum s_ij is
// relative to its own reference q_ij (see EpiLogitStats):
//   m' = max_j m_ij,  s' = sum_j s_ij e^{q_ij - m'}      (tiles in ascending j)
// and the per-row factor that turns the stored P into softmax':
//   cfac_i = e^{ref_i - m'_i} / s'_i,  ref_i = row_bad ? m'_i : r_i.
// Nearly every tile has q_ij = r_i, so the sum is accumulated relative to a
// running reference R (start r_i): s_ij adds as is, and only a tile with
// q_ij > R (a re-referenced overflow tile) rescales.  No exp on the common
// path and no max / sum dependency chain: the kernel runs at load speed.
// Block = 512 threads = 16 warps x 32 rows; warp w takes tiles w, w+16, ...
// (fixed order), then the 16 partials merge in w order.
__global__ void __launch_bounds__(512) k_stats_reduce_ref(const float* __restrict__ tile_m,
                                                          const float* __restrict__ tile_s,
                                                          const float* __restrict__ tile_q, int ntiles, int64_t ld,
                                                          int n, const float* __restrict__ row_ref,
                                                          const int* __restrict__ row_bad, float* __restrict__ m_out,
                                                          float* __restrict__ s_out, float* __restrict__ cfac) {
  constexpr int W = 16;
  __shared__ float sm[W][32], ss[W][32], sr[W][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = blockIdx.x * 32 + lane;
  float m = -INFINITY, S = 0.f, R = 0.f;
  if (row < n) {
    R = row_ref[row];
    // batches of kB tiles: all 3 x kB loads issued before the (order-fixed)
    // merge consumes them, so a warp keeps 3 x kB x 128 B in flight
    constexpr int kB = 8;
    for (int j0 = w; j0 < ntiles; j0 += W * kB) {
      float mj[kB], sj[kB], qj[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int j = j0 + u * W;
        if (j < ntiles) {
          const int64_t o = int64_t(j) * ld + row;
          mj[u] = tile_m[o];
          sj[u] = tile_s[o];
          qj[u] = tile_q[o];
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (j0 + u * W >= ntiles) break;
        m = fmaxf(m, mj[u]);
        if (qj[u] == R) {
          S += sj[u];
        } else if (qj[u] < R) {
          S += sj[u] * expf(qj[u] - R);
        } else {
          S = S * expf(R - qj[u]) + sj[u];
          R = qj[u];
        }
      }
    }
  }
  sm[w][lane] = m;
  ss[w][lane] = S;
  sr[w][lane] = R;
  __syncthreads();
  if (w == 0 && row < n) {
    float M = sm[0][lane], Sa = ss[0][lane], Ra = sr[0][lane];
    for (int q = 1; q < W; ++q) {
      M = fmaxf(M, sm[q][lane]);
      const float Rq = sr[q][lane], Sq = ss[q][lane];
      if (Rq == Ra) {
        Sa += Sq;
      } else if (Rq < Ra) {
        Sa += Sq * expf(Rq - Ra);
      } else {
        Sa = Sa * expf(Ra - Rq) + Sq;
        Ra = Rq;
      }
    }
    const float sprime = Sa * expf(Ra - M);  // relative to the row max
    m_out[row] = M;
    s_out[row] = sprime;
    const float ref = row_bad[row] ? M : row_ref[row];
    cfac[row] = expf(ref - Ra) / Sa;  // = e^{ref - m'} / s'
  }
}

// Fixup 1/3: a tile stored against its own max (ran before r_i was
// published) whose max exceeds r_i + gap cannot be re-referenced to r_i:
// its row joins the bad rows (re-referenced to the row max instead).
__global__ void k_fix_check(const int2* __restrict__ fix_list, const int* __restrict__ fix_count,
                            const float* __restrict__ tile_q, int64_t ld, int n, const float* __restrict__ row_ref,
                            float gap, int* __restrict__ row_bad, int* __restrict__ bad_count,
                            int* __restrict__ bad_list) {
  const int cnt = *fix_count;
  const int lane = threadIdx.x & 31;
  for (int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += gridDim.x * (blockDim.x >> 5)) {
    const int2 f = fix_list[e];
    const int row = f.x * 32 + lane;
    if (row >= n) continue;
    if (tile_q[int64_t(f.y) * ld + row] - row_ref[row] > gap && atomicExch(row_bad + row, 1) == 0)
      bad_list[atomicAdd(bad_count, 1)] = row;
  }
}

// Rescale P[row, tile j] by e^{q - ref} (8 bf16 per thread-step).
__device__ __forceinline__ void rescale_segment(__nv_bfloat16* p, int cols, float f, int t0, int tstep) {
  for (int v = t0 * 8; v < cols; v += tstep * 8) {
    if (v + 8 <= cols) {
      uint4 u = *reinterpret_cast<uint4*>(p + v);
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 x = __bfloat1622float2(h2[q]);
        h2[q] = __floats2bfloat162_rn(x.x * f, x.y * f);
      }
      *reinterpret_cast<uint4*>(p + v) = u;
    } else {
      for (int q = v; q < cols; ++q) p[q] = __float2bfloat16(__bfloat162float(p[q]) * f);
    }
  }
}

// Fixup 2/3: listed (32-row group, tile) pairs of good rows -> reference r_i.
__global__ void k_fix_apply(const int2* __restrict__ fix_list, const int* __restrict__ fix_count,
                            __nv_bfloat16* __restrict__ P, int64_t ldp, int cols, const float* __restrict__ tile_q,
                            int64_t ld, int n, const float* __restrict__ row_ref, const int* __restrict__ row_bad) {
  const int cnt = *fix_count;
  for (int e = blockIdx.x; e < cnt; e += gridDim.x) {
    const int2 f = fix_list[e];
    const int c0 = f.y * kTileN, cw = min(kTileN, cols - c0);
    for (int rr = threadIdx.x >> 5; rr < 32; rr += blockDim.x >> 5) {
      const int row = f.x * 32 + rr;
      if (row >= n || row_bad[row]) continue;
      const float fac = fast_exp(tile_q[int64_t(f.y) * ld + row] - row_ref[row]);
      rescale_segment(P + int64_t(row) * ldp + c0, cw, fac, threadIdx.x & 31, 32);
    }
  }
}

// Fixup 3/3: bad rows -> every tile re-referenced to the row max m'.
__global__ void k_fix_bad(const int* __restrict__ bad_list, const int* __restrict__ bad_count,
                          __nv_bfloat16* __restrict__ P, int64_t ldp, int cols, const float* __restrict__ tile_q,
                          int64_t ld, const float* __restrict__ m_row) {
  const int cnt = *bad_count;
  const int ntiles = (cols + kTileN - 1) / kTileN;
  for (int e = blockIdx.x; e < cnt; e += gridDim.x) {
    const int row = bad_list[e];
    for (int j = threadIdx.x >> 5; j < ntiles; j += blockDim.x >> 5) {
      const float q = tile_q[int64_t(j) * ld + row];
      if (q == m_row[row]) continue;
      const int c0 = j * kTileN;
      rescale_segment(P + int64_t(row) * ldp + c0, min(kTileN, cols - c0), fast_exp(q - m_row[row]),
                      threadIdx.x & 31, 32);
    }
  }
}

// merge_max_sum (VM.cpp:82-101) over p parts laid out [p x n]: m starts at
// part 0 and takes the max in k order; sum accumulates sum_k e^{m_k - m} in
// k order; then sum *= fault_scale (VM.cpp:314).
__global__ void k_merge_stats(const float* __restrict__ mparts, const float* __restrict__ sparts, int p, int64_t ld,
                              int n, float fault_scale, float* __restrict__ m_out, float* __restrict__ s_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float m = mparts[i];
  for (int k = 1; k < p; ++k) m = fmaxf(m, mparts[int64_t(k) * ld + i]);
  float s = 0.f;
  for (int k = 0; k < p; ++k) s += sparts[int64_t(k) * ld + i] * expf(mparts[int64_t(k) * ld + i] - m);
  m_out[i] = m;
  s_out[i] = s * fault_scale;
}

// Same merge with the parts given as pointer arrays (shards on one device).
struct StatsParts {
  const float* m[kMaxLocalShards];
  const float* s[kMaxLocalShards];
  int p;
};
__global__ void k_merge_stats_ptrs(StatsParts parts, int n, float fault_scale, float* __restrict__ m_out,
                                   float* __restrict__ s_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float m = parts.m[0][i];
  for (int k = 1; k < parts.p; ++k) m = fmaxf(m, parts.m[k][i]);
  float s = 0.f;
  for (int k = 0; k < parts.p; ++k) s += parts.s[k][i] * expf(parts.m[k][i] - m);
  m_out[i] = m;
  s_out[i] = s * fault_scale;
}

// Pack (m_loc, s_loc) into one [2 x n] buffer for the stats all-gather.
__global__ void k_pack_stats(const float* __restrict__ m, const float* __restrict__ s, int n, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = m[i];
  out[n + i] = s[i];
}

// ---------------------------------------------------------------------------
// inv = 1/s (per-row normalisers).
__global__ void k_inv(const float* __restrict__ s, int n, float* __restrict__ inv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[i] = 1.f / s[i];
}

// global_scale (VM.cpp:22-27): c_i = sum'_i e^{m'_i - m_i} / sum_i, times the
// per-row factor cfac_i that maps the stored P to softmax' (null: 1).
__global__ void k_global_scale(const float* __restrict__ ml, const float* __restrict__ sl,
                               const float* __restrict__ mg, const float* __restrict__ sg,
                               const float* __restrict__ cfac, int n, float* __restrict__ c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) c[i] = sl[i] * expf(ml[i] - mg[i]) / sg[i] * (cfac ? cfac[i] : 1.f);
}

// ---------------------------------------------------------------------------
// alg2 C1 combine (VM.cpp:205-209): grad_x[i,:] = sum_k ( c_k[i] A_k[i,:] - B_k[i,:] )
// with B_k[i,:] = W_k[g_i - rb_k,:] if shard k owns g_i (sparse row gather,
// SPEC.md:231).  Shards summed in k order.  4 columns per thread.
// ---------------------------------------------------------------------------
struct CombineShards {
  const float* A[kMaxLocalShards];
  int64_t lda;
  const __nv_bfloat16* W[kMaxLocalShards];
  int64_t ldw[kMaxLocalShards];
  int64_t rb[kMaxLocalShards], re[kMaxLocalShards];
  const float* ml[kMaxLocalShards];
  const float* sl[kMaxLocalShards];
  const float* yt[kMaxLocalShards];  // y[i, g_i] of owned labels (the fused loss)
  int p;
};
// loss != nullptr: also the per-token loss of VM.cpp:287-292 (k_loss's
// expression), by the thread of column group 0 of each row (one launch fewer)
__global__ void k_alg2_combine(CombineShards S, const float* __restrict__ mg, const float* __restrict__ sg,
                               const int64_t* __restrict__ labels, int n, int h, float* __restrict__ gx,
                               int64_t ldgx, int64_t V, int* __restrict__ err, int err_bit,
                               float* __restrict__ loss = nullptr) {
  const int hv = h / 4;
  const int64_t total = int64_t(n) * hv;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / hv), c = int(t - int64_t(i) * hv) * 4;
    const int64_t g = labels[i];
    if (c == 0 && (g < 0 || (V >= 0 && g >= V))) atomicOr(err, err_bit);  // VM.cpp:18
    if (c == 0 && loss != nullptr) {
      float out = 0.f;
      for (int k = 0; k < S.p; ++k)
        if (g >= S.rb[k] && g < S.re[k]) out = mg[i] + logf(sg[i]) - S.yt[k][i];
      loss[i] = out;
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < S.p; ++k) {
      const float sc = S.sl[k][i] * expf(S.ml[k][i] - mg[i]) / sg[i];
      const float4 a = *reinterpret_cast<const float4*>(S.A[k] + int64_t(i) * S.lda + c);
      float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g >= S.rb[k] && g < S.re[k]) {
        const __nv_bfloat16* w = S.W[k] + (g - S.rb[k]) * S.ldw[k] + c;
        const float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w));
        const float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + 2));
        b = make_float4(w0.x, w0.y, w1.x, w1.y);
      }
      acc.x += a.x * sc - b.x;
      acc.y += a.y * sc - b.y;
      acc.z += a.z * sc - b.z;
      acc.w += a.w * sc - b.w;
    }
    *reinterpret_cast<float4*>(gx + int64_t(i) * ldgx + c) = acc;
  }
}

// ---------------------------------------------------------------------------
// Fused C1 over peer memory (alg2, nranks > 1).  Token rows are owned in
// blocks of R rows: rank o owns rows [o R, min(T, (o + 1) R)).  In pass S the
// dX GEMM of rank k stores its A_k tiles straight into slot k of the owner's
// buffer (routed epilogue, over NVLink), and k_push_label_rows sends the
// label rows B_k (W_k rows of the labels rank k owns) into the owner's B
// buffer; every token row gets exactly one B row, from its label's owner.
// At C1 the owner combines its rows from local memory only, in rank order:
//   grad_x[i,:] = sum_k ( c_k[i] A_k[i,:] - [k owns g_i] B[i,:] )
// — the expression and order of k_alg2_combine over p local shards, so the
// group's grad_x has the same bits as a one-GPU p-shard run.
// ---------------------------------------------------------------------------
struct PeerRows {
  void* p[kMaxLocalShards];  // owner o's B buffer [R x h] bf16, as mapped here
};
__global__ void k_push_label_rows(const __nv_bfloat16* __restrict__ W, int64_t ldw, int64_t rb, int64_t re,
                                  const int64_t* __restrict__ labels, int n, int h, int R, PeerRows dst) {
  const int hv = h / 8;  // 16-byte vectors
  const int64_t total = int64_t(n) * hv;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / hv), c = int(t - int64_t(i) * hv) * 8;
    const int64_t g = labels[i];
    if (g < rb || g >= re) continue;
    const int o = i / R;
    const uint4 v = *reinterpret_cast<const uint4*>(W + (g - rb) * ldw + c);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(dst.p[o]) + int64_t(i - o * R) * h + c) = v;
  }
  __threadfence_system();  // peer stores performed before the kernel's completion is observed
}

struct OwnedCombine {
  const float* slots;            // [nranks][splits][R][h] fp32: rank k's split-K partials of A_k, my rows
  const __nv_bfloat16* B;        // [R][h] bf16
  const float* gathered;         // [nranks][2T]: rank k's local m at k*2T, sum at k*2T + T
  int64_t rb[kMaxLocalShards], re[kMaxLocalShards];
  int nranks, R, row0, rows;     // my rows: [row0, row0 + rows)
  int prescaled;                 // alg1 C2: the slots already hold c_k A_k (c_k = 1 here)
  int splits;                    // split-K units of rank k's dX GEMM, added here in split order
};
__global__ void k_alg2_combine_owned(OwnedCombine S, const float* __restrict__ mg, const float* __restrict__ sg,
                                     const int64_t* __restrict__ labels, int T, int h, float* __restrict__ out,
                                     int64_t ldo, int64_t V, int* __restrict__ err, int err_bit) {
  const int hv = h / 4;
  const int64_t total = int64_t(S.rows) * hv;
  const int64_t slot = int64_t(S.R) * h;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int li = int(t / hv), c = int(t - int64_t(li) * hv) * 4;
    const int i = S.row0 + li;
    const int64_t g = labels[i];
    if (c == 0 && (g < 0 || (V >= 0 && g >= V))) atomicOr(err, err_bit);  // VM.cpp:18
    const float* a_row = S.slots + int64_t(li) * h + c;
    const __nv_bfloat16* w = S.B + int64_t(li) * h + c;
    const float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w));
    const float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + 2));
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < S.nranks; ++k) {
      // A_k = p_0 + p_1 + ... in split order: the fp32 adds the ordered split-K
      // of the one-GPU path performs (its TMA reduce-adds), the same bits
      float4 a = *reinterpret_cast<const float4*>(a_row + int64_t(k) * S.splits * slot);
      for (int sp = 1; sp < S.splits; ++sp) {
        const float4 q = *reinterpret_cast<const float4*>(a_row + (int64_t(k) * S.splits + sp) * slot);
        a.x = a.x + q.x;
        a.y = a.y + q.y;
        a.z = a.z + q.z;
        a.w = a.w + q.w;
      }
      float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g >= S.rb[k] && g < S.re[k]) b = make_float4(w0.x, w0.y, w1.x, w1.y);
      if (S.prescaled) {
        // alg1 / C2: partial_k = c_k A_k - G_k W_k, summed in k order (the
        // one-GPU path's k_sub_label_rows + k_sum_partials)
        acc.x += a.x - b.x;
        acc.y += a.y - b.y;
        acc.z += a.z - b.z;
        acc.w += a.w - b.w;
        continue;
      }
      const float ml = S.gathered[int64_t(k) * 2 * T + i], sl = S.gathered[int64_t(k) * 2 * T + T + i];
      const float sc = sl * expf(ml - mg[i]) / sg[i];
      acc.x += a.x * sc - b.x;
      acc.y += a.y * sc - b.y;
      acc.z += a.z * sc - b.z;
      acc.w += a.w * sc - b.w;
    }
    *reinterpret_cast<float4*>(out + int64_t(li) * ldo + c) = acc;
  }
}

// Sum of p partials in k order (alg1/naive C2 on one device).
struct PartialPtrs {
  const float* P[kMaxLocalShards];
  int p;
};
__global__ void k_sum_partials(PartialPtrs S, int64_t count, float* __restrict__ out) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count; t += int64_t(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < S.p; ++k) acc += S.P[k][t];
    out[t] = acc;
  }
}

// dX correction for alg1/naive: gx[i,:] -= W_k[g_i - rb,:] for owned rows.
__global__ void k_sub_label_rows(float* __restrict__ gx, int64_t ldgx, const __nv_bfloat16* __restrict__ W,
                                 int64_t ldw, int64_t rb, int64_t re, const int64_t* __restrict__ labels, int n,
                                 int h) {
  const int hv = h / 2;
  const int64_t total = int64_t(n) * hv;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / hv), c = int(t - int64_t(i) * hv) * 2;
    const int64_t g = labels[i];
    if (g < rb || g >= re) continue;
    const float2 w = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(W + (g - rb) * ldw + c));
    float* d = gx + int64_t(i) * ldgx + c;
    d[0] -= w.x;
    d[1] -= w.y;
  }
}

// B_k = G_k W_k (VM.hpp:41, alg2_pass_S VM.cpp:186-190): out[i,:] = W_k[g_i - rb,:]
// if shard k owns g_i, else 0 (debug materialisation; C1 gathers these rows
// sparsely instead).  fp32 out, 2 columns per thread.
__global__ void k_label_rows(const __nv_bfloat16* __restrict__ W, int64_t ldw, int64_t rb, int64_t re,
                             const int64_t* __restrict__ labels, int n, int h, float* __restrict__ out,
                             int64_t ldo) {
  const int hv = h / 2;
  const int64_t total = int64_t(n) * hv;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / hv), c = int(t - int64_t(i) * hv) * 2;
    const int64_t g = labels[i];
    float2 w = make_float2(0.f, 0.f);
    if (g >= rb && g < re) w = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(W + (g - rb) * ldw + c));
    out[int64_t(i) * ldo + c] = w.x;
    out[int64_t(i) * ldo + c + 1] = w.y;
  }
}

// loss_i = m_i + log(sum_i) - y_tgt_i at the shard owning g_i (VM.cpp:287-292);
// rows owned by none of the given shards get 0 (summed across ranks).
struct LossShards {
  const float* yt[kMaxLocalShards];
  int64_t rb[kMaxLocalShards], re[kMaxLocalShards];
  int p;
};
// A label outside [0, V) (V < 0: unknown upper bound) raises err_bit in *err
// (the reference's "TokenBatch: label out of range", VM.cpp:18).
__global__ void k_loss(LossShards S, const float* __restrict__ mg, const float* __restrict__ sg,
                       const int64_t* __restrict__ labels, int n, float* __restrict__ loss, int64_t V,
                       int* __restrict__ err, int err_bit) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t g = labels[i];
  if (g < 0 || (V >= 0 && g >= V)) atomicOr(err, err_bit);
  float out = 0.f;
  for (int k = 0; k < S.p; ++k)
    if (g >= S.rb[k] && g < S.re[k]) out = mg[i] + logf(sg[i]) - S.yt[k][i];
  loss[i] = out;
}

// Xs[i,:] = bf16(c_i * X[i,:])   (alg2 pass T: dW = P'^T diag(c) X)
// The global scale of VM.cpp:22-27 (times the per-row reference factor cfac
// when given), one row at a time: the expression of k_global_scale.
struct RowScale {
  const float *ml, *sl, *mg, *sg, *cfac;
  __device__ __forceinline__ float operator()(int i) const {
    return sl[i] * expf(ml[i] - mg[i]) / sg[i] * (cfac ? cfac[i] : 1.f);
  }
};
// Xs = c (.) X with c computed inline (alg2_pass_T: no separate scale pass)
__global__ void k_scale_rows_global_bf16(const __nv_bfloat16* __restrict__ X, int64_t ldx, RowScale rs, int n, int h,
                                         __nv_bfloat16* __restrict__ out, int64_t ldo) {
  const int hv = h / 8;
  const int64_t total = int64_t(n) * hv;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / hv), j = int(t - int64_t(i) * hv) * 8;
    uint4 u = *reinterpret_cast<const uint4*>(X + int64_t(i) * ldx + j);
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
    const float f = rs(i);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float2 x = __bfloat1622float2(h2[q]);
      h2[q] = __floats2bfloat162_rn(x.x * f, x.y * f);
    }
    *reinterpret_cast<uint4*>(out + int64_t(i) * ldo + j) = u;
  }
}

__global__ void k_scale_rows_bf16(const __nv_bfloat16* __restrict__ X, int64_t ldx, const float* __restrict__ c,
                                  int n, int h, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  const int hv = h / 8;
  const int64_t total = int64_t(n) * hv;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / hv), j = int(t - int64_t(i) * hv) * 8;
    uint4 u = *reinterpret_cast<const uint4*>(X + int64_t(i) * ldx + j);
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
    const float f = c[i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float2 x = __bfloat1622float2(h2[q]);
      h2[q] = __floats2bfloat162_rn(x.x * f, x.y * f);
    }
    *reinterpret_cast<uint4*>(out + int64_t(i) * ldo + j) = u;
  }
}

// naive F2: e = exp(Y - m) from the stored fp32 logits (re-read, VM.cpp:119-125),
// written as bf16 P, plus the per-row local exp-sum.  One block per row.
__global__ void k_naive_exp_sum(const float* __restrict__ Y, int64_t ldy, int cols, const float* __restrict__ m,
                                __nv_bfloat16* __restrict__ P, int64_t ldp, float* __restrict__ s_out) {
  const int i = blockIdx.x;
  const float mi = m[i];
  float acc = 0.f;
  for (int v = threadIdx.x * 4; v < cols; v += blockDim.x * 4) {
    float e[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) e[q] = (v + q < cols) ? fast_exp(Y[int64_t(i) * ldy + v + q] - mi) : 0.f;
    acc += (e[0] + e[1]) + (e[2] + e[3]);
    if (P == nullptr) continue;  // sums only (the softmax is written once, in B)
    __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(P + int64_t(i) * ldp + v);
    if (v + 4 <= cols) {
      d[0] = __floats2bfloat162_rn(e[0], e[1]);
      d[1] = __floats2bfloat162_rn(e[2], e[3]);
    } else {
      for (int q = 0; q < 4 && v + q < cols; ++q) P[int64_t(i) * ldp + v + q] = __float2bfloat16(e[q]);
    }
  }
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
    s_out[i] = s;
  }
}

// naive: y_tgt[i] = Y[i, g_i - rb] for owned rows (VM.cpp:139-140)
__global__ void k_gather_target(const float* __restrict__ Y, int64_t ldy, const int64_t* __restrict__ labels,
                                int64_t rb, int64_t re, int n, float* __restrict__ yt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t g = labels[i];
  if (g >= rb && g < re) yt[i] = Y[int64_t(i) * ldy + (g - rb)];
}

// Naive B normalisation (VM.cpp:127-131): P[i,v] = bf16(e^{Y[i,v] - m_i} / sum_i),
// re-reading the fp32 logits (the naive variant's extra pass) and rounding to
// bf16 once.  8 columns per thread, 16-byte P stores, padding columns zeroed.
__global__ void k_naive_softmax(const float* __restrict__ Y, int64_t ldy, int n, int cols, const float* __restrict__ m,
                                const float* __restrict__ inv, __nv_bfloat16* __restrict__ P, int64_t ldp) {
  const int vec_per_row = (cols + 7) / 8;
  const int64_t total = int64_t(n) * vec_per_row;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / vec_per_row);
    const int v0 = int(t - int64_t(i) * vec_per_row) * 8;
    const float mi = m[i], f = inv[i];
    const float* y = Y + int64_t(i) * ldy + v0;
    uint4 u;
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = (v0 + 2 * q < cols) ? fast_exp(y[2 * q] - mi) * f : 0.f;
      const float b = (v0 + 2 * q + 1 < cols) ? fast_exp(y[2 * q + 1] - mi) * f : 0.f;
      h2[q] = __floats2bfloat162_rn(a, b);
    }
    *reinterpret_cast<uint4*>(P + int64_t(i) * ldp + v0) = u;
  }
}

// Debug/parity materialisation (assemble_forward softmax, VM.cpp:281-286):
// out[i, v] = P[i,v] * f(i, v) in fp32.
__global__ void k_materialize(const __nv_bfloat16* __restrict__ P, int64_t ldp, int n, int cols,
                              const float* __restrict__ tile_m, int64_t ld_stats, const float* __restrict__ mref,
                              const float* __restrict__ mul, float* __restrict__ out, int64_t ldo) {
  const int64_t total = int64_t(n) * cols;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / cols), v = int(t - int64_t(i) * cols);
    float f = mul[i];
    if (tile_m) f *= fast_exp(tile_m[int64_t(v / kTileN) * ld_stats + i] - mref[i]);
    out[int64_t(i) * ldo + v] = __bfloat162float(P[int64_t(i) * ldp + v]) * f;
  }
}

// ---------------------------------------------------------------------------
// Input layer.
// K7 input_forward (VM.cpp:227-236): out[i,:] = W_k[t_i - rb,:] if owned else 0.
// One warp per token row, 16-byte vectors.  t_i < 0 raises the context's
// error flag (the reference throws invalid_argument); t_i >= V is "not owned".
// accumulate != 0 adds the owned rows onto out instead (fused all-reduce
// target for shards simulated on one device).
// ---------------------------------------------------------------------------
__global__ void k_input_forward(const int64_t* __restrict__ tok, int n, const __nv_bfloat16* __restrict__ W,
                                int64_t ldw, int64_t rb, int64_t re, int h, __nv_bfloat16* __restrict__ out,
                                int64_t ldo, int accumulate, int* __restrict__ err) {
  const int warps = (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < n; i += gridDim.x * warps) {
    const int64_t t = tok[i];
    if (t < 0 && lane == 0) atomicOr(err, 1);
    const bool own = t >= rb && t < re;
    uint4* d = reinterpret_cast<uint4*>(out + int64_t(i) * ldo);
    const uint4* s = reinterpret_cast<const uint4*>(W + (own ? (t - rb) : 0) * ldw);
    const int hv = h / 8;
    if (!accumulate) {
      if (!own) {
        for (int j = lane; j < hv; j += 32) d[j] = make_uint4(0u, 0u, 0u, 0u);
        continue;
      }
      // four 16-byte loads in flight per lane before the stores
      for (int j0 = lane; j0 < hv; j0 += 128) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + 32 * u < hv) v[u] = __ldg(s + j0 + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + 32 * u < hv) d[j0 + 32 * u] = v[u];
      }
    } else if (own) {
      for (int j = lane; j < hv; j += 32) {
        uint4 a = d[j];
        const uint4 b = __ldg(s + j);
        __nv_bfloat162* a2 = reinterpret_cast<__nv_bfloat162*>(&a);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
        for (int q = 0; q < 4; ++q) a2[q] = __hadd2(a2[q], b2[q]);
        d[j] = a;
      }
    }
  }
}

// ---- input layer, N > 1: owner gather instead of the zero-padded all-reduce --
// Every rank knows all token ids and every rank's row range, so each can
// compute, for token i, its owner k and its position among k's tokens in
// ascending i; rank k packs the rows it owns at those positions, one grouped
// broadcast per rank exchanges the packed blocks (the owned rows only: about
// half the bytes of a sum all-reduce of the mostly-zero [T x h] output), and
// an unpack copies row i from its owner's block.  Pure copies: bit-exact.
constexpr int kMaxRanks = 64;
struct RankBounds {
  int64_t rb[kMaxRanks], re[kMaxRanks];
  int n;
};
__device__ __forceinline__ int owner_of(const RankBounds& B, int64_t t) {
  for (int k = 0; k < B.n; ++k)
    if (t >= B.rb[k] && t < B.re[k]) return k;
  return -1;  // negative or past every shard: no owner (a zero row, VM.cpp:232-234)
}
// One block (1024 threads): pos[i] = #{j < i : owner_j == owner_i}; counts[k].
__global__ void __launch_bounds__(1024) k_owner_positions(const int64_t* __restrict__ tok, int n, RankBounds B,
                                                          int* __restrict__ pos, int* __restrict__ counts,
                                                          int* __restrict__ err) {
  __shared__ int run[kMaxRanks];
  __shared__ int wtot[kMaxRanks][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < B.n; k += blockDim.x) run[k] = 0;
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int own = -2;
    if (i < n) {
      const int64_t t = tok[i];
      if (t < 0) atomicOr(err, 1);
      own = owner_of(B, t);
    }
    int myrank = 0;
    for (int k = 0; k < B.n; ++k) {
      const unsigned m = __ballot_sync(0xffffffffu, own == k);
      if (own == k) myrank = __popc(m & lt);
      if (lane == 0) wtot[k][w] = __popc(m);
    }
    __syncthreads();
    // exclusive scan over warps per owner (one thread per owner)
    for (int k = threadIdx.x; k < B.n; k += blockDim.x) {
      int acc = run[k];
      for (int q = 0; q < int(blockDim.x >> 5); ++q) {
        const int c = wtot[k][q];
        wtot[k][q] = acc;
        acc += c;
      }
      run[k] = acc;
    }
    __syncthreads();
    if (i < n) pos[i] = own >= 0 ? wtot[own][w] + myrank : -1;
    __syncthreads();
  }
  for (int k = threadIdx.x; k < B.n; k += blockDim.x) counts[k] = run[k];
}
struct RankOffsets {
  int64_t off[kMaxRanks];  // first packed row of each owner's block
};
// rank `me` writes its owned rows into its block of buf (warp per token)
__global__ void k_owner_pack(const int64_t* __restrict__ tok, int n, RankBounds B, const int* __restrict__ pos,
                             RankOffsets O, int me, const __nv_bfloat16* __restrict__ W, int64_t ldw, int h,
                             __nv_bfloat16* __restrict__ buf) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < n; i += gridDim.x * warps) {
    const int64_t t = tok[i];
    if (owner_of(B, t) != me) continue;
    const uint4* s = reinterpret_cast<const uint4*>(W + (t - B.rb[me]) * ldw);
    uint4* d = reinterpret_cast<uint4*>(buf + (O.off[me] + pos[i]) * int64_t(h));
    for (int j = lane; j < h / 8; j += 32) d[j] = __ldg(s + j);
  }
}
// out[i] = row i from its owner's block (zero when no rank owns the token)
__global__ void k_owner_unpack(const int64_t* __restrict__ tok, int n, RankBounds B, const int* __restrict__ pos,
                               RankOffsets O, const __nv_bfloat16* __restrict__ buf, int h,
                               __nv_bfloat16* __restrict__ out, int64_t ldo) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < n; i += gridDim.x * warps) {
    const int k = owner_of(B, tok[i]);
    uint4* d = reinterpret_cast<uint4*>(out + int64_t(i) * ldo);
    if (k < 0) {
      for (int j = lane; j < h / 8; j += 32) d[j] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      const uint4* s = reinterpret_cast<const uint4*>(buf + (O.off[k] + pos[i]) * int64_t(h));
      for (int j = lane; j < h / 8; j += 32) d[j] = s[j];
    }
  }
}

// ---- input layer, N > 1, over peer memory (option "peer_input") ------------
// Every rank writes the rows it owns at their token index into its own
// peer-visible buffer (one half per call parity); after a group barrier every
// rank pulls row i from the buffer of token i's owner — over NVLink for a peer
// — straight into its output.  No packing positions, no host-side sizes, one
// tiny collective: capturable.  Pure copies: bit-exact.
__global__ void k_input_own_rows(const int64_t* __restrict__ tok, int n, const __nv_bfloat16* __restrict__ W,
                                 int64_t ldw, int64_t rb, int64_t re, int h, __nv_bfloat16* __restrict__ buf,
                                 int* __restrict__ err) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < n; i += gridDim.x * warps) {
    const int64_t t = tok[i];
    if (t < 0 && lane == 0) atomicOr(err, 1);  // VM.cpp:232
    if (t < rb || t >= re) continue;
    const uint4* s = reinterpret_cast<const uint4*>(W + (t - rb) * ldw);
    uint4* d = reinterpret_cast<uint4*>(buf + int64_t(i) * h);
    for (int j = lane; j < h / 8; j += 32) d[j] = __ldg(s + j);
  }
}
struct PeerBufs {
  const __nv_bfloat16* p[kMaxLocalShards];  // rank k's current half, as mapped here
};
__global__ void k_input_pull_rows(const int64_t* __restrict__ tok, int n, RankBounds B, PeerBufs P, int h,
                                  __nv_bfloat16* __restrict__ out, int64_t ldo) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int hv = h / 8;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < n; i += gridDim.x * warps) {
    const int k = owner_of(B, tok[i]);
    uint4* d = reinterpret_cast<uint4*>(out + int64_t(i) * ldo);
    if (k < 0) {
      for (int j = lane; j < hv; j += 32) d[j] = make_uint4(0u, 0u, 0u, 0u);
      continue;
    }
    const uint4* s = reinterpret_cast<const uint4*>(P.p[k] + int64_t(i) * h);
    // four 16-byte loads in flight per lane before the stores (NVLink latency)
    for (int j0 = lane; j0 < hv; j0 += 128) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + 32 * u < hv) v[u] = s[j0 + 32 * u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + 32 * u < hv) d[j0 + 32 * u] = v[u];
    }
  }
}

}  // namespace vp
