// Standalone GPU self-test + microbenchmark of the tcgen05 GEMM and its
// epilogues against a CUDA-core fp32 reference.  Developer tool (not part of
// the product); build: make -C tools gemm_selftest.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2411_05288_b200/csrc/gemm_host.cuh"

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(2);                                                                             \
    }                                                                                      \
  } while (0)

__global__ void init_bf16(__nv_bfloat16* p, int64_t n, uint32_t seed, float scale) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x = uint32_t(i) * 2654435761u ^ seed;
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    p[i] = __float2bfloat16((float(x & 0xFFFFFF) / 16777216.0f * 2.f - 1.f) * scale);
  }
}

// D[m][n] = sum_k A(m,k) B(n,k)
__global__ void ref_gemm(const __nv_bfloat16* A, int64_t lda, bool amn, const __nv_bfloat16* B, int64_t ldb,
                         bool bmn, float* D, int M, int N, int K) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (n >= N) return;
  float acc = 0.f;
  for (int k = 0; k < K; ++k) {
    const float a = __bfloat162float(amn ? A[int64_t(k) * lda + m] : A[int64_t(m) * lda + k]);
    const float b = __bfloat162float(bmn ? B[int64_t(k) * ldb + n] : B[int64_t(n) * ldb + k]);
    acc = fmaf(a, b, acc);
  }
  D[int64_t(m) * N + n] = acc;
}

static int failures = 0;

static int* g_flags = nullptr;
static vp::SplitCfg g_split;

static void check_store(int cg, bool amn, bool bmn, int M, int N, int K, int nsm, int mc = 1, int nh = 1,
                        int split = 0) {
  const int64_t lda = amn ? ((M + 7) / 8 * 8) : ((K + 7) / 8 * 8);
  const int64_t ldb = bmn ? ((N + 7) / 8 * 8) : ((K + 7) / 8 * 8);
  const int64_t asz = amn ? int64_t(K) * lda : int64_t(M) * lda;
  const int64_t bsz = bmn ? int64_t(K) * ldb : int64_t(N) * ldb;
  __nv_bfloat16 *A, *B;
  float *D, *R;
  CK(cudaMalloc(&A, asz * 2));
  CK(cudaMalloc(&B, bsz * 2));
  CK(cudaMalloc(&D, int64_t(M) * N * 4));
  CK(cudaMalloc(&R, int64_t(M) * N * 4));
  init_bf16<<<256, 256>>>(A, asz, 17u, 1.f);
  init_bf16<<<256, 256>>>(B, bsz, 91u, 1.f);
  CK(cudaMemset(D, 0xFF, int64_t(M) * N * 4));
  vp::EpiStoreF32::Params ep{D, N, nullptr, 0};
  if (split && !g_flags) {
    CK(cudaMalloc(&g_flags, 2 * 4096 * sizeof(int)));
    CK(cudaMemset(g_flags, 0, 2 * 4096 * sizeof(int)));
    g_split.flags = g_flags;
    g_split.max_tiles = 4096;
  }
  g_split.force = split;
  vp::launch_gemm<vp::EpiStoreF32>(cg, {A, lda, amn}, {B, ldb, bmn}, M, N, K, 0, ep, nsm, 0, -1, -1, mc, nh,
                                   split ? &g_split : nullptr);
  size_t nondet = 0;
  if (split) {  // ordered split accumulation: a second run gives identical bits
    std::vector<float> d1(size_t(M) * N), d2(size_t(M) * N);
    CK(cudaMemcpy(d1.data(), D, d1.size() * 4, cudaMemcpyDeviceToHost));
    vp::launch_gemm<vp::EpiStoreF32>(cg, {A, lda, amn}, {B, ldb, bmn}, M, N, K, 0, ep, nsm, 0, -1, -1, mc, nh,
                                     &g_split);
    CK(cudaMemcpy(d2.data(), D, d2.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < d1.size(); ++i) nondet += memcmp(&d1[i], &d2[i], 4) != 0;
  }
  ref_gemm<<<dim3((N + 127) / 128, M), 128>>>(A, lda, amn, B, ldb, bmn, R, M, N, K);
  CK(cudaDeviceSynchronize());
  std::vector<float> d(size_t(M) * N), r(size_t(M) * N);
  CK(cudaMemcpy(d.data(), D, d.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(r.data(), R, r.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  size_t bad = 0;
  for (size_t i = 0; i < d.size(); ++i) {
    const double e = std::fabs(double(d[i]) - r[i]);
    if (!(e <= 1e-3 * std::sqrt(double(K)) + 1e-3)) ++bad;
    maxerr = std::max(maxerr, std::isnan(e) ? 1e30 : e);
    maxref = std::max(maxref, double(std::fabs(r[i])));
  }
  bad += nondet;
  printf("store cg=%d mc=%d nh=%d split=%d A_%s B_%s M=%d N=%d K=%d : max_abs_err=%.3e max_ref=%.3e bad=%zu nondet=%zu %s\n",
         cg, mc, nh, split, amn ? "MN" : "K", bmn ? "MN" : "K", M, N, K, maxerr, maxref, bad, nondet,
         bad ? "FAIL" : "ok");
  if (bad) ++failures;
  cudaFree(A);
  cudaFree(B);
  cudaFree(D);
  cudaFree(R);
}

static void check_stats(int cg, int M, int N, int K, int nsm, int mc = 1, int nh = 1) {
  const int64_t ld = (K + 7) / 8 * 8;
  const int64_t ldp = (N + 63) / 64 * 64;
  const int tiles = (N + vp::kEpiCols - 1) / vp::kEpiCols;
  __nv_bfloat16 *A, *B, *P;
  float *R, *tm, *ts, *yt;
  int64_t* lab;
  CK(cudaMalloc(&A, int64_t(M) * ld * 2));
  CK(cudaMalloc(&B, int64_t(N) * ld * 2));
  CK(cudaMalloc(&P, int64_t(M) * ldp * 2));
  CK(cudaMalloc(&R, int64_t(M) * N * 4));
  CK(cudaMalloc(&tm, int64_t(tiles) * M * 4));
  CK(cudaMalloc(&ts, int64_t(tiles) * M * 4));
  CK(cudaMalloc(&yt, int64_t(M) * 4));
  CK(cudaMalloc(&lab, int64_t(M) * 8));
  init_bf16<<<256, 256>>>(A, int64_t(M) * ld, 5u, 1.f);
  init_bf16<<<256, 256>>>(B, int64_t(N) * ld, 7u, 0.25f);
  std::vector<int64_t> hl(M);
  const int64_t rb = 1000;
  for (int i = 0; i < M; ++i) hl[i] = (i % 3 == 0) ? 5 : rb + (int64_t(i) * 7919) % N;
  CK(cudaMemcpy(lab, hl.data(), M * 8, cudaMemcpyHostToDevice));
  float *tq, *ref;
  int *flg, *badr, *cnt, *bl;
  int2* fl;
  CK(cudaMalloc(&tq, int64_t(tiles) * M * 4));
  CK(cudaMalloc(&ref, M * 4));
  CK(cudaMalloc(&flg, 4096 * 4));
  CK(cudaMalloc(&badr, M * 4));
  CK(cudaMalloc(&cnt, 8));
  CK(cudaMalloc(&bl, M * 4));
  CK(cudaMalloc(&fl, int64_t(M / 32 + 1) * tiles * 8));
  CK(cudaMemset(flg, 0, 4096 * 4));
  CK(cudaMemset(badr, 0, M * 4));
  CK(cudaMemset(cnt, 0, 8));
  vp::EpiLogitStats::Params ep{P, ldp, tm, ts, M, lab, rb, rb + N, yt, tq, ref, flg, badr, cnt, bl, cnt + 1, fl};
  vp::launch_gemm<vp::EpiLogitStats>(cg, {A, ld, false}, {B, ld, false}, M, N, K, 0, ep, nsm, 0, -1, -1, mc, nh);
  ref_gemm<<<dim3((N + 127) / 128, M), 128>>>(A, ld, false, B, ld, false, R, M, N, K);
  CK(cudaDeviceSynchronize());
  std::vector<float> r(size_t(M) * N), htm(size_t(tiles) * M), hts(size_t(tiles) * M), hyt(M);
  std::vector<uint16_t> hp(size_t(M) * ldp);
  CK(cudaMemcpy(r.data(), R, r.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(htm.data(), tm, htm.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hts.data(), ts, hts.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hyt.data(), yt, hyt.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hp.data(), P, hp.size() * 2, cudaMemcpyDeviceToHost));
  std::vector<float> hq(size_t(tiles) * M);
  CK(cudaMemcpy(hq.data(), tq, hq.size() * 4, cudaMemcpyDeviceToHost));
  double em = 0, es = 0, ep_ = 0, ey = 0;
  for (int i = 0; i < M; ++i) {
    for (int t = 0; t < tiles; ++t) {
      double mx = -1e300;
      for (int v = t * vp::kEpiCols; v < std::min(N, t * vp::kEpiCols + vp::kEpiCols); ++v) mx = std::max(mx, double(r[size_t(i) * N + v]));
      double s = 0;
      const double q = hq[size_t(t) * M + i];
      for (int v = t * vp::kEpiCols; v < std::min(N, t * vp::kEpiCols + vp::kEpiCols); ++v) {
        const double e = std::exp(double(r[size_t(i) * N + v]) - q);
        s += e;
        uint32_t bits = uint32_t(hp[size_t(i) * ldp + v]) << 16;
        float pv;
        memcpy(&pv, &bits, 4);
        ep_ = std::max(ep_, std::fabs(pv - e) / std::max(1.0, e));
      }
      em = std::max(em, std::fabs(htm[size_t(t) * M + i] - mx));
      es = std::max(es, std::fabs(hts[size_t(t) * M + i] - s) / s);
    }
    if (hl[i] >= rb && hl[i] < rb + N) ey = std::max(ey, double(std::fabs(hyt[i] - r[size_t(i) * N + (hl[i] - rb)])));
  }
  const bool ok = em < 1e-3 && es < 1e-4 && ep_ < 4e-3 && ey < 1e-3;
  printf("stats cg=%d mc=%d M=%d N=%d K=%d : tile_max_err=%.2e tile_sum_relerr=%.2e P_err=%.2e ytgt_err=%.2e %s\n", cg, mc, M,
         N, K, em, es, ep_, ey, ok ? "ok" : "FAIL");
  if (!ok) ++failures;
  cudaFree(A);
  cudaFree(B);
  cudaFree(P);
  cudaFree(R);
  cudaFree(tm);
  cudaFree(ts);
  cudaFree(yt);
  cudaFree(lab);
  cudaFree(tq);
  cudaFree(ref);
  cudaFree(flg);
  cudaFree(badr);
  cudaFree(cnt);
  cudaFree(bl);
  cudaFree(fl);
}

template <class F>
static float time_ms(F&& f, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / iters;
}

static void bench_store(int cg, bool amn, bool bmn, int M, int N, int K, int raster, int nsm) {
  const int64_t lda = amn ? M : K, ldb = bmn ? N : K;
  __nv_bfloat16 *A, *B;
  float* D;
  CK(cudaMalloc(&A, (amn ? int64_t(K) * lda : int64_t(M) * lda) * 2));
  CK(cudaMalloc(&B, (bmn ? int64_t(K) * ldb : int64_t(N) * ldb) * 2));
  CK(cudaMalloc(&D, int64_t(M) * N * 4));
  init_bf16<<<1024, 256>>>(A, amn ? int64_t(K) * lda : int64_t(M) * lda, 1u, 1.f);
  init_bf16<<<1024, 256>>>(B, bmn ? int64_t(K) * ldb : int64_t(N) * ldb, 2u, 1.f);
  vp::EpiStoreF32::Params ep{D, N, nullptr, 0};
  const float ms = time_ms([&] { vp::launch_gemm<vp::EpiStoreF32>(cg, {A, lda, amn}, {B, ldb, bmn}, M, N, K, raster, ep, nsm, 0); }, 5);
  printf("bench store cg=%d A_%s B_%s M=%d N=%d K=%d raster=%d : %.3f ms  %.1f TFLOP/s\n", cg, amn ? "MN" : "K",
         bmn ? "MN" : "K", M, N, K, raster, ms, 2.0 * M * N * double(K) / ms / 1e9);
  cudaFree(A);
  cudaFree(B);
  cudaFree(D);
}

static void bench_stats(int cg, int M, int N, int K, int nsm) {
  const int tiles = (N + vp::kEpiCols - 1) / vp::kEpiCols;
  __nv_bfloat16 *A, *B, *P;
  float *tm, *ts, *yt;
  CK(cudaMalloc(&A, int64_t(M) * K * 2));
  CK(cudaMalloc(&B, int64_t(N) * K * 2));
  CK(cudaMalloc(&P, int64_t(M) * N * 2));
  CK(cudaMalloc(&tm, int64_t(tiles) * M * 4));
  CK(cudaMalloc(&ts, int64_t(tiles) * M * 4));
  CK(cudaMalloc(&yt, int64_t(M) * 4));
  init_bf16<<<1024, 256>>>(A, int64_t(M) * K, 3u, 1.f);
  init_bf16<<<1024, 256>>>(B, int64_t(N) * K, 4u, 0.02f);
  float* tq;
  float* ref;
  int *flg, *badr, *cnt, *bl;
  int2* fl;
  CK(cudaMalloc(&tq, int64_t(tiles) * M * 4));
  CK(cudaMalloc(&ref, M * 4));
  CK(cudaMalloc(&flg, 4096 * 4));
  CK(cudaMalloc(&badr, M * 4));
  CK(cudaMalloc(&cnt, 8));
  CK(cudaMalloc(&bl, M * 4));
  CK(cudaMalloc(&fl, int64_t(M / 32 + 1) * tiles * 8));
  vp::EpiLogitStats::Params ep{P, N, tm, ts, M, nullptr, 0, N, yt, tq, ref, flg, badr, cnt, bl, cnt + 1, fl};
  const float ms = time_ms([&] { vp::launch_gemm<vp::EpiLogitStats>(cg, {A, K, false}, {B, K, false}, M, N, K, 0, ep, nsm, 0); }, 5);
  printf("bench stats cg=%d M=%d N=%d K=%d : %.3f ms  %.1f TFLOP/s\n", cg, M, N, K, ms,
         2.0 * M * N * double(K) / ms / 1e9);
  cudaFree(A);
  cudaFree(B);
  cudaFree(P);
  cudaFree(tm);
  cudaFree(ts);
  cudaFree(yt);
}

int main(int argc, char** argv) {
  int nsm = 0;
  if (getenv("VP_TMA_STORE")) vp::g_tma_store = atoi(getenv("VP_TMA_STORE"));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const bool do_bench = argc > 1 && std::string(argv[1]) == "bench";
  if (argc > 1 && std::string(argv[1]) == "one") {  // one 8192^3 GEMM: one <cg>
    bench_store(atoi(argv[2]), false, false, 8192, 8192, 8192, 0, nsm);
    return 0;
  }
  printf("SMs=%d\n", nsm);
  for (int v = 0; v < 3; ++v) {
    const int cg = v == 0 ? 1 : 2, mc = v == 2 ? 2 : 1;
    check_store(cg, false, false, 256, 256, 64, nsm, mc);
    check_store(cg, false, false, 512, 768, 1024, nsm, mc);
    check_store(cg, false, true, 512, 768, 1024, nsm, mc);
    check_store(cg, true, true, 512, 768, 1024, nsm, mc);
    check_store(cg, false, false, 300, 520, 200, nsm, mc);
    check_store(cg, false, true, 300, 520, 200, nsm, mc);
    check_store(cg, true, true, 300, 520, 200, nsm, mc);
    check_store(cg, false, false, 600, 3000, 320, nsm, mc);
    check_store(cg, true, true, 700, 1100, 640, nsm, mc);
    check_stats(cg, 300, 1000, 256, nsm, mc);
    check_stats(cg, 512, 777, 512, nsm, mc);
    check_stats(cg, 1000, 5000, 128, nsm, mc);
  }
  for (bool amn : {false, true})
    for (bool bmn : {false, true}) {
      if (amn && !bmn) continue;
      check_store(2, amn, bmn, 512, 1024, 512, nsm, 1, 2);
      check_store(2, amn, bmn, 300, 520, 200, nsm, 1, 2);
      check_store(2, amn, bmn, 700, 1300, 640, nsm, 1, 2);
      // K = 1, 2, 3 k-blocks (stagger depth 0, 1, 1) and a long K (depth = STAGES)
      check_store(2, amn, bmn, 300, 700, 64, nsm, 1, 2);
      check_store(2, amn, bmn, 300, 700, 128, nsm, 1, 2);
      check_store(2, amn, bmn, 300, 700, 192, nsm, 1, 2);
      check_store(2, amn, bmn, 520, 1100, 2048, nsm, 1, 2);
    }
  // split-K (ordered partial accumulation), both tile widths, both cta_groups
  for (int sp : {2, 3, 4}) {
    check_store(2, false, true, 520, 1100, 2048, nsm, 1, 2, sp);
    check_store(2, false, true, 300, 700, 640, nsm, 1, 1, sp);
    check_store(1, false, true, 300, 700, 640, nsm, 1, 1, sp);
    check_store(2, true, true, 700, 1300, 1024, nsm, 1, 2, sp);
  }
  check_store(2, false, true, 2048, 4096, 8192, nsm, 1, 2, 2);
  check_stats(2, 300, 1000, 256, nsm, 1, 2);
  check_stats(2, 512, 777, 512, nsm, 1, 2);
  check_stats(2, 1000, 5000, 128, nsm, 1, 2);
  check_stats(2, 700, 3000, 64, nsm, 1, 2);
  check_stats(2, 600, 1300, 1024, nsm, 1, 2);
  if (do_bench) {
    for (int cg : {1, 2}) bench_store(cg, false, false, 8192, 8192, 8192, 0, nsm);
    bench_stats(2, 8192, 32000, 4096, nsm);
    bench_stats(2, 8192, 256000, 4096, nsm);
    bench_store(2, false, true, 8192, 4096, 32000, 8, nsm);
    bench_store(2, true, true, 32000, 4096, 8192, -16, nsm);
  }
  printf("%s (%d failures)\n", failures ? "SELFTEST FAIL" : "SELFTEST PASS", failures);
  return failures ? 1 : 0;
}
