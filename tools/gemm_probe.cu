// Developer probe: one vocab GEMM at the headline shape (T=8192, h=4096,
// V=256000 by default) with a chosen tile rasterisation and L2 policies.
//   gemm_probe <k1|dx|dw> <raster> <pol_a> <pol_b> [iters] [V]
// pol: -1 default, 0 normal, 1 evict_first, 2 evict_last.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../paper_2411_05288_b200/csrc/gemm_host.cuh"

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(2);                                                                            \
    }                                                                                     \
  } while (0)

// N(0, s^2) via Box-Muller on hashed uniforms (power draw depends on the data)
__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return uint32_t(x);
}
__global__ void fill(__nv_bfloat16* p, int64_t n, float s, uint64_t seed) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float u1 = (hash32(seed * 0x9E3779B97F4A7C15ull + 2 * i) + 1.f) * 2.3283064e-10f;
    const float u2 = hash32(seed * 0x9E3779B97F4A7C15ull + 2 * i + 1) * 2.3283064e-10f;
    p[i] = __float2bfloat16(s * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2));
  }
}

int main(int argc, char** argv) {
  const int mc = getenv("VP_MC") ? atoi(getenv("VP_MC")) : 1;
  const int nh = getenv("VP_NH") ? atoi(getenv("VP_NH")) : 1;
  if (argc < 5) {
    fprintf(stderr, "usage: gemm_probe <k1|dx|dw> <raster> <pol_a> <pol_b> [iters] [V]\n");
    return 2;
  }
  const std::string kind = argv[1];
  const int raster = atoi(argv[2]), pa = atoi(argv[3]), pb = atoi(argv[4]);
  const int iters = argc > 5 ? atoi(argv[5]) : 10;
  // VP_T / VP_H: token count and hidden size (default: the headline shape)
  const int64_t T = getenv("VP_T") ? atoll(getenv("VP_T")) : 8192, h = getenv("VP_H") ? atoll(getenv("VP_H")) : 4096,
                V = argc > 6 ? atoll(argv[6]) : 256000;
  int nsm = 0;
  if (getenv("VP_TMA_STORE")) vp::g_tma_store = atoi(getenv("VP_TMA_STORE"));
  if (getenv("VP_SEF")) vp::g_store_evict_first = atoi(getenv("VP_SEF"));  // epilogue stores evict-first
  // ncu's kernel replay cannot relaunch cooperative grids (as in the library)
  if (getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") || getenv("CUDA_INJECTION64_PATH")) vp::g_cooperative = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  __nv_bfloat16 *X, *W, *P;
  float* out;
  CK(cudaMalloc(&X, T * h * 2));
  CK(cudaMalloc(&W, V * h * 2));
  CK(cudaMalloc(&P, T * V * 2));
  fill<<<1024, 256>>>(X, T * h, 1.f, 1);
  fill<<<1024, 256>>>(W, V * h, 0.02f, 2);
  fill<<<1024, 256>>>(P, T * V, 4e-6f, 3);  // softmax-like magnitudes
  const int ntiles = int((V + vp::kEpiCols - 1) / vp::kEpiCols);
  float *tm, *ts, *yt;
  CK(cudaMalloc(&tm, int64_t(ntiles) * T * 4));
  CK(cudaMalloc(&ts, int64_t(ntiles) * T * 4));
  CK(cudaMalloc(&yt, T * 4));
  float *tq, *ref;
  int *flg, *bad, *cnt, *bl;
  int2* fl;
  CK(cudaMalloc(&tq, int64_t(ntiles) * T * 4));
  CK(cudaMalloc(&ref, T * 4));
  CK(cudaMalloc(&flg, 4096 * 4));
  CK(cudaMalloc(&bad, T * 4));
  CK(cudaMalloc(&cnt, 8));
  CK(cudaMalloc(&bl, T * 4));
  CK(cudaMalloc(&fl, int64_t(T / 32 + 1) * ntiles * 8));
  const int64_t out_elems = kind == "dw" ? V * h : kind == "sq8192" ? int64_t(8192) * 8192 : T * h;
  CK(cudaMalloc(&out, out_elems * 4));
  // VP_SPLIT: split-K of the dx GEMM (0 = off, -1 = auto, 2..4 forced)
  const int split_dx = getenv("VP_SPLIT") ? atoi(getenv("VP_SPLIT")) : -1;
  vp::SplitCfg scfg;
  CK(cudaMalloc(&scfg.flags, 2 * 16384 * sizeof(int)));
  CK(cudaMemset(scfg.flags, 0, 2 * 16384 * sizeof(int)));
  scfg.max_tiles = 16384;
  scfg.force = split_dx > 0 ? split_dx : 0;
  // VP_WS: parallel split-K workspace mode (0 never, 1 auto, 2 force); VP_MINKB: ordered-split floor
  scfg.ws_mode = getenv("VP_WS") ? atoi(getenv("VP_WS")) : 1;
  scfg.min_kb = getenv("VP_MINKB") ? atoi(getenv("VP_MINKB")) : 64;
  scfg.ws_elems = size_t(nsm / 2 + 2) * 256 * 512 + (size_t(1) << 16);
  CK(cudaMalloc(&scfg.ws, scfg.ws_elems * sizeof(float)));
  // VP_LOCKSTEP: wave-lockstep epoch (k-blocks, 0 = off)
  vp::LockCfg lcfg;
  lcfg.epoch = getenv("VP_LOCKSTEP") ? atoi(getenv("VP_LOCKSTEP")) : 0;
  lcfg.capacity = int64_t(1) << 20;
  CK(cudaMalloc(&lcfg.counters, size_t(lcfg.capacity) * sizeof(int)));
  // VP_PERSIST=<MB>: persisting L2 window over the operand that is re-read
  // across waves (K1: X; dW: the X operand) with a set-aside of that size
  vp::L2Window win;
  const vp::L2Window* winp = nullptr;
  {
    cudaDeviceProp pr;
    CK(cudaGetDeviceProperties(&pr, 0));
    printf("  L2 %d MB, persisting max %d MB, access-policy window max %d MB\n", pr.l2CacheSize >> 20,
           pr.persistingL2CacheMaxSize >> 20, pr.accessPolicyMaxWindowSize >> 20);
    const int pmb = getenv("VP_PERSIST") ? atoi(getenv("VP_PERSIST")) : 0;
    if (pmb > 0 && (kind == "k1" || kind == "dw")) {
      const size_t lim = std::min<size_t>(size_t(pmb) << 20, size_t(pr.persistingL2CacheMaxSize));
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim));
      win.ptr = X;
      win.bytes = std::min<size_t>(size_t(T * h * 2), size_t(pr.accessPolicyMaxWindowSize));
      win.hit_ratio = std::min(1.f, float(double(lim) / double(win.bytes)));
      winp = &win;
      printf("  persisting window %.1f MB, set-aside %.1f MB, hit ratio %.2f\n", win.bytes / 1e6, lim / 1e6,
             win.hit_ratio);
    }
  }
  auto run = [&] {
    if (kind == "k1") {
      vp::EpiLogitStats::Params ep{P,   V,   tm,  ts,  T,   nullptr, 0,   V,   yt,  tq,
                                   ref, flg, bad, cnt, bl,  cnt + 1, fl};
      CK(cudaMemsetAsync(flg, 0, 4096 * 4));
      CK(cudaMemsetAsync(bad, 0, T * 4));
      CK(cudaMemsetAsync(cnt, 0, 8));
      vp::launch_gemm<vp::EpiLogitStats>(2, {X, h, false}, {W, h, false}, int(T), int(V), int(h), raster, ep, nsm, 0,
                                         pa, pb, mc, nh, nullptr, &lcfg, -1, winp);
    } else if (kind == "dx") {
      vp::EpiStoreF32::Params ep{out, h, nullptr, 0, nullptr};
      vp::launch_gemm<vp::EpiStoreF32>(2, {P, V, false}, {W, h, true}, int(T), int(h), int(V), raster, ep, nsm, 0, pa,
                                       pb, mc, nh, split_dx ? &scfg : nullptr, &lcfg);
    } else if (kind == "dw") {
      vp::EpiStoreF32::Params ep{out, h, nullptr, 0, nullptr};
      vp::launch_gemm<vp::EpiStoreF32>(2, {P, V, true}, {X, h, true}, int(V), int(h), int(T), raster, ep, nsm, 0, pa,
                                       pb, mc, nh, split_dx ? &scfg : nullptr, &lcfg, -1, winp);
    } else {  // sq8192: plain 8192^3 K-major GEMM (W as an 8192 x 8192 slice), fp32 out
      vp::EpiStoreF32::Params ep{out, 8192, nullptr, 0, nullptr};
      vp::launch_gemm<vp::EpiStoreF32>(2, {W, 8192, false}, {W + int64_t(8192) * 8192, 8192, false}, 8192, 8192,
                                       8192, raster, ep, nsm, 0, pa, pb, mc, nh);
    }
  };
  unsigned long long* prof;
  CK(cudaMallocManaged(&prof, 128));
  CK(cudaMemset(prof, 0, 128));
  vp::g_gemm_prof = prof;
  run();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) run();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= iters;
  CK(cudaDeviceSynchronize());
  {
    const double cyc = double(prof[2] - prof[0]), ns = double(prof[3] - prof[1]);
    const int64_t Mx = kind == "dw" ? V : (kind == "sq8192" ? 8192 : T);
    const int64_t Nx = kind == "k1" ? V : (kind == "sq8192" ? 8192 : h);
    const int64_t Kx = kind == "k1" ? h : (kind == "dx" ? V : (kind == "dw" ? T : 8192));
    const double tiles = double((Mx + 255) / 256) * double((Nx + 256 * nh - 1) / (256 * nh));
    const double ideal = tiles * double((Kx + 63) / 64) * 4.0 * 128.0 * nh;  // MMA issue cycles, all tiles
    const double par = double(nsm / 2);                                        // CTA pairs
    printf("  last launch (CTA 0): %.0f cycles in %.3f ms -> %.0f MHz; MMA-ideal %.0f cycles/pair -> %.1f%% of ideal\n",
           cyc, ns / 1e6, cyc / ns * 1e3, ideal / par, 100.0 * (ideal / par) / cyc);
    if (nh == 2)
      printf("  CTA 0 issuer waits: smem stages %.1f%%, accumulators %.1f%%; epilogue warp: waiting %.1f%%, working %.1f%%\n",
             100.0 * prof[4] / cyc, 100.0 * prof[5] / cyc, 100.0 * prof[6] / cyc, 100.0 * prof[7] / cyc);
    printf("  CTA 0 epilogue warp: waiting for a free staging box %.2f%%\n", 100.0 * prof[8] / cyc);
  }
  const double flops = kind == "sq8192" ? 2.0 * 8192.0 * 8192.0 * 8192.0 : 2.0 * T * h * double(V);
  printf("mc=%d nh=%d ", mc, nh);
  printf("probe %s raster=%d pol_a=%d pol_b=%d V=%lld: %.3f ms %.1f TFLOP/s\n", kind.c_str(), raster, pa, pb,
         (long long)V, ms, flops / ms / 1e9);
  return 0;
}
