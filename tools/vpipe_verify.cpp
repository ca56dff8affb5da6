// vpipe_verify — the reference's `vpipe verify` (P/tools/vpipe_main.cpp:161-218)
// on the B200 path, through the drop-in C++ API (include/vpipe/vocab_math.hpp).
//
//   vpipe_verify [--batch B] [--seq-len S] [--hidden H] [--vocab V]
//                [--devices P] [--seed N] [--fault-scale F]
//                [--placement auto|local|spread|loopback] [--inject-k1-fault PPM]
//
// Same defaults (b=2, s=4, h=8, V=32, p=4; vpipe_main.cpp:285-287), same flow
// (pad V to a multiple of 2p, random_instance, naive / alg1 / alg2 at p shards
// and the input layer), same exit codes (0 pass, 1 verify failure, 2 usage /
// invalid argument).  The reference result comes from an INDEPENDENT checker:
// the fp64 CPU oracle (oracle/liboracle.so, a restatement of VM.cpp — test
// infrastructure, linked by this tool only) on the same bf16-rounded
// operands the device sees; the device's own monolithic oracle_output_layer
// is checked against it too.  Tolerances are the north_star's bf16 ones:
// per-token loss <= 1e-3 abs, softmax <= 4e-3 abs, grad_x / grad_w <= 1e-2
// relative L2; the input-layer forward must be exact.
// --inject-k1-fault PPM scales every pass-S logit by 1 + PPM * 1e-6 inside the
// K1 epilogue (a fault common to every p) — verify must then exit 1.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "vpipe/vocab_math.hpp"

// CPU oracle (oracle/vocab_oracle.cpp): the checker, never the product.
extern "C" int or_oracle_output_layer(const double* X, const double* W, const int64_t* labels, int64_t n_tok,
                                      int64_t h, int64_t V, const double* logit_shift, double* softmax,
                                      double* loss, double* gx, double* gw);
extern "C" const char* or_last_error(void);

namespace {

constexpr int kExitOk = 0, kExitVerifyFail = 1, kExitUsage = 2;

double rel_l2(const vpipe::Matrix& a, const vpipe::Matrix& b) {
  double num = 0, den = 0;
  for (int64_t i = 0; i < a.size(); ++i) {
    const double d = a.data()[i] - b.data()[i];
    num += d * d;
    den += b.data()[i] * b.data()[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1e-300));
}

// The value the device computes with: double -> float -> bf16 (RNE), as the
// drop-in's upload does.
double bf16_round(double v) {
  float f = float(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

vpipe::OutputResult cpu_oracle(const vpipe::TokenBatch& batch, const vpipe::Matrix& W) {
  const int64_t n = batch.X.rows(), h = batch.X.cols(), V = W.rows();
  vpipe::Matrix Xb(n, h), Wb(V, h);
  for (int64_t i = 0; i < Xb.size(); ++i) Xb.data()[i] = bf16_round(batch.X.data()[i]);
  for (int64_t i = 0; i < Wb.size(); ++i) Wb.data()[i] = bf16_round(W.data()[i]);
  vpipe::OutputResult r;
  r.softmax.resize(n, V);
  r.loss.resize(n);
  r.grad_x.resize(n, h);
  r.grad_w.resize(V, h);
  if (or_oracle_output_layer(Xb.data(), Wb.data(), batch.labels.data(), n, h, V, nullptr, r.softmax.data(),
                             r.loss.data(), r.grad_x.data(), r.grad_w.data()) != 0)
    throw std::invalid_argument(or_last_error());
  return r;
}

int usage(const char* msg) {
  std::fprintf(stderr, "vpipe_verify: %s\nusage: vpipe_verify [--batch B] [--seq-len S] [--hidden H] [--vocab V] "
                       "[--devices P] [--seed N] [--fault-scale F] [--placement auto|local|spread|loopback] "
                       "[--inject-k1-fault PPM]\n", msg);
  return kExitUsage;
}

}  // namespace

int main(int argc, char** argv) {
  int64_t b = 2, s = 4, h = 8, V = 32, p = 4;
  uint64_t seed = 0;
  double fault = 1.0;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (i + 1 >= argc) return usage(("missing value for " + a).c_str());
    const char* v = argv[++i];
    if (a == "--batch") b = std::atoll(v);
    else if (a == "--seq-len") s = std::atoll(v);
    else if (a == "--hidden") h = std::atoll(v);
    else if (a == "--vocab") V = std::atoll(v);
    else if (a == "--devices") p = std::atoll(v);
    else if (a == "--seed") seed = std::strtoull(v, nullptr, 10);
    else if (a == "--fault-scale") fault = std::atof(v);
    else if (a == "--inject-k1-fault") setenv("VPIPE_INJECT_K1_FAULT_PPM", v, 1);
    else if (a == "--placement") {
      const std::string pl = v;
      if (pl == "auto") vpipe::set_placement(vpipe::Placement::Auto);
      else if (pl == "local") vpipe::set_placement(vpipe::Placement::Local);
      else if (pl == "spread") vpipe::set_placement(vpipe::Placement::Spread);
      else if (pl == "loopback") vpipe::set_placement(vpipe::Placement::Loopback);
      else return usage(("unknown placement " + pl).c_str());
    } else return usage(("unknown option " + a).c_str());
  }
  try {
    const int64_t n_tok = b * s;
    const int64_t Vp = vpipe::pad_vocab_size(V, p);
    const vpipe::RandomInstance inst = vpipe::random_instance(n_tok, h, Vp, seed);
    const vpipe::OutputResult oracle = cpu_oracle(inst.batch, inst.W);
    struct Case {
      const char* name;
      vpipe::OutputResult r;
    };
    const Case cases[] = {
        {"device_oracle", vpipe::oracle_output_layer(inst.batch, inst.W)},
        {"naive", vpipe::run_naive(inst.batch, inst.W, int(p))},
        {"alg1", vpipe::run_alg1(inst.batch, inst.W, int(p), fault)},
        {"alg2", vpipe::run_alg2(inst.batch, inst.W, int(p), fault)},
    };
    bool ok = true;
    for (const Case& c : cases) {
      const double dl = c.r.loss.maxAbsDiff(oracle.loss);
      const double ds = c.r.softmax.maxAbsDiff(oracle.softmax);
      const double gx = rel_l2(c.r.grad_x, oracle.grad_x), gw = rel_l2(c.r.grad_w, oracle.grad_w);
      const bool pass = dl <= 1e-3 && ds <= 4e-3 && gx <= 1e-2 && gw <= 1e-2;
      ok = ok && pass;
      std::printf("%s loss_err=%.3g softmax_err=%.3g grad_x_rel=%.3g grad_w_rel=%.3g %s\n", c.name, dl, ds, gx, gw,
                  pass ? "PASS" : "FAIL");
    }
    // input layer: sharded forward / backward vs the monolithic lookup
    const auto shards = vpipe::shard_weights(inst.W, int(p));
    vpipe::Matrix fwd(n_tok, h), bwd(Vp, h);
    for (const auto& shard : shards) {
      const vpipe::Matrix f = vpipe::input_forward(inst.batch.labels, shard);
      for (int64_t i = 0; i < f.size(); ++i) fwd.data()[i] += f.data()[i];
      const vpipe::Matrix g = vpipe::input_backward(inst.batch.X, inst.batch.labels, shard);
      std::memcpy(bwd.row_ptr(shard.row_begin), g.data(), sizeof(double) * size_t(g.size()));
    }
    // reference: bf16-rounded W rows (operands are bf16 on the device), fp64 scatter
    vpipe::Matrix fwd_ref(n_tok, h), bwd_ref(Vp, h);
    for (int64_t i = 0; i < n_tok; ++i) {
      const int64_t t = inst.batch.labels[size_t(i)];
      for (int64_t j = 0; j < h; ++j) {
        float w = float(inst.W(t, j));
        uint32_t u;
        std::memcpy(&u, &w, 4);
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
        std::memcpy(&w, &u, 4);
        fwd_ref(i, j) = w;
        bwd_ref(t, j) += inst.batch.X(i, j);
      }
    }
    const double fe = fwd.maxAbsDiff(fwd_ref), be = bwd.maxAbsDiff(bwd_ref);
    const bool ipass = fe == 0.0 && be <= 1e-5;
    ok = ok && ipass;
    std::printf("input fwd_err=%.3g bwd_err=%.3g %s\n", fe, be, ipass ? "PASS" : "FAIL");
    return ok ? kExitOk : kExitVerifyFail;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "vpipe_verify: %s\n", e.what());
    return kExitUsage;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "vpipe_verify: %s\n", e.what());
    return kExitVerifyFail;
  }
}
