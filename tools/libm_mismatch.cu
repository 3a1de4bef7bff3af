// libm_mismatch.cu — measures whether trace generation (SURVEY.md §8(f)
// rank 3: build_workload, workload.hpp:27-81 / 209-245, rng.hpp:44-58) could
// move to the device bit-exactly.
//
// The reference's traces are defined by glibc's log / exp / cos (Box-Muller
// normals, truncated-lognormal token draws, exponential inter-arrival times).
// A device generator would evaluate the same calls with CUDA's libdevice.
// This tool runs the host generator (the same algorithm and draw order as
// csrc/workload.cpp) over the bench seeds, records the argument and the glibc
// result of every libm call on the per-request path, re-evaluates each call
// on the device (sm_100a, no FMA contraction) and counts bitwise mismatches:
// per function, per request (a request is affected when any call that fed it
// differs) and per replay.  sqrt is IEEE correctly rounded on both sides
// and is not counted.  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -fmad=false \
//        -Xcompiler -ffp-contract=off -o tools/libm_mismatch tools/libm_mismatch.cu \
//        -L paper_2408_13510_b200/_lib -lrs_b200
//   tools/libm_mismatch [seeds=64] [requests=31329] [rate=20]
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../include/rs_abi.h"

namespace {

enum Fn { kLog = 0, kExp = 1, kCos = 2, kFns = 3 };

struct Call {
  double x, host;
  int fn;
  int64_t req;  // request index within the replay (-1: setup)
};

thread_local std::vector<Call>* g_log = nullptr;
thread_local int64_t g_req = -1;

double hlog(double x) {
  const double y = std::log(x);
  if (g_log) g_log->push_back({x, y, kLog, g_req});
  return y;
}
double hexp(double x) {
  const double y = std::exp(x);
  if (g_log) g_log->push_back({x, y, kExp, g_req});
  return y;
}
double hcos(double x) {
  const double y = std::cos(x);
  if (g_log) g_log->push_back({x, y, kCos, g_req});
  return y;
}

// ---- the generator (same algorithm / draw order as csrc/workload.cpp) ----
struct Source {
  std::mt19937_64 eng;
  explicit Source(uint64_t s) : eng(s) {}
  double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double gauss() {
    double u1 = uniform();
    double u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return std::sqrt(-2.0 * hlog(u1)) * hcos(2.0 * 3.14159265358979323846 * u2);
  }
  double expo(double rate) {
    double u = uniform();
    while (u <= 0.0) u = uniform();
    return -hlog(u) / rate;
  }
};

struct TLN {
  double mu = 0.0, sigma = 0.5, lo = 1.0, hi = 4096.0;
  static double gap(double a, double b) {
    constexpr double r = 0.70710678118654752440;
    return 0.5 * (std::erfc(a * r) - std::erfc(b * r));
  }
  double tmean() const {
    double a = (std::log(lo) - mu) / sigma, b = (std::log(hi) - mu) / sigma;
    double den = gap(a, b);
    if (den <= 0.0) return a > 0.0 ? lo : hi;
    return std::exp(mu + 0.5 * sigma * sigma) * gap(a - sigma, b - sigma) / den;
  }
  static TLN fit(double target, double sigma, double lo, double hi) {
    TLN d{0.0, sigma, lo, hi};
    double a = std::log(lo) - 36.0 * sigma, b = std::log(hi) + 36.0 * sigma;
    for (int it = 0; it < 300; ++it) {
      d.mu = 0.5 * (a + b);
      if (d.tmean() < target) a = d.mu; else b = d.mu;
    }
    return d;
  }
  long long tokens(Source& s) const {
    double x = 0.0;
    bool ok = false;
    for (int t = 0; t < 10000 && !ok; ++t) {
      x = hexp(mu + sigma * s.gauss());
      ok = x >= lo && x <= hi;
    }
    if (!ok) x = std::clamp(std::exp(mu), lo, hi);
    return std::clamp(std::llround(x), (long long)std::ceil(lo), (long long)std::floor(hi));
  }
};

struct Task {
  double heavy_frac;
  TLN prompt, light, heavy;
};

double narrowed(double nominal, double target, double lo, double hi) {
  return std::min(nominal, std::max(0.05, std::min(target / lo - 1.0, hi / target - 1.0)));
}

std::vector<Task> tasks(long long cut) {
  const double rows[5][4] = {{7351, 29.09, 61.76, 0.0918}, {6988, 29.83, 334.40, 0.5818},
                             {6564, 211.54, 142.53, 0.4101}, {7122, 125.16, 220.02, 0.4795},
                             {3304, 26.41, 64.10, 0.0871}};
  std::vector<Task> v;
  for (auto& row : rows) {
    Task t;
    t.heavy_frac = row[3];
    t.prompt = TLN::fit(row[1], narrowed(0.7, row[1], 1.0, 1000.0), 1.0, 1000.0);
    const double b = (double)cut, cap = 4096.0, q = row[3], md = row[2];
    double ml = std::min(0.6 * b, std::max(1.5, 0.5 * md));
    double mh = std::clamp((md - (1.0 - q) * ml) / q, 1.02 * b, 0.9 * cap);
    ml = std::clamp((md - q * mh) / (1.0 - q), 1.5, 0.98 * (b - 1.0));
    t.light = TLN::fit(ml, narrowed(0.6, ml, 1.0, b - 1.0), 1.0, b - 1.0);
    t.heavy = TLN::fit(mh, narrowed(0.45, mh, b, cap), b, cap);
    v.push_back(t);
  }
  return v;
}

__global__ void eval(const double* x, const int* fn, double* y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    y[i] = fn[i] == kLog ? log(v) : fn[i] == kExp ? exp(v) : cos(v);
  }
}

}  // namespace

int main(int argc, char** argv) {
  const int seeds = argc > 1 ? atoi(argv[1]) : 64;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 31329;
  const double rate = argc > 3 ? atof(argv[3]) : 20.0;
  rs_profile p{3.2e-4, 0.026, 3.3e-5, 0.0167};
  rs_thresholds th{0.5, 5.0};
  const long long cut = rs_heavy_decode_cutoff(&p, &th);
  const std::vector<Task> T = tasks(cut);
  const double w[5] = {7351, 6988, 6564, 7122, 3304};
  double total = 0.0;
  for (double x : w) total += x;

  long long calls[kFns] = {}, bad[kFns] = {}, req_bad = 0, req_total = 0, rep_bad = 0;
  long long trace_diff_rep = 0;
  std::vector<double> arr(n);
  std::vector<int32_t> pr(n), de(n);
  std::vector<uint8_t> tk(n);
  for (int s = 1; s <= seeds; ++s) {
    std::vector<Call> log;
    g_log = &log;
    Source src(rs_mix_seed((uint64_t)s, 0xB00C));
    std::vector<double> a(n);
    std::vector<int32_t> q(n), d(n);
    for (int64_t i = 0; i < n; ++i) {
      g_req = i;
      double u = src.uniform() * total;
      int k = 0;
      for (; k + 1 < 5; ++k) {
        u -= w[k];
        if (u < 0.0) break;
      }
      q[i] = (int32_t)T[k].prompt.tokens(src);
      const bool heavy = src.uniform() < T[k].heavy_frac;
      d[i] = (int32_t)(heavy ? T[k].heavy : T[k].light).tokens(src);
    }
    double clock = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      g_req = i;
      clock += src.expo(rate);
      a[i] = clock;
    }
    g_log = nullptr;
    // the restatement reproduces the engine's (and so the reference's) trace
    rs_generate_mixture(&p, &th, nullptr, (uint64_t)s, n, rate, 0, arr.data(), pr.data(),
                        de.data(), tk.data());
    if (arr != a || pr != q || de != d) ++trace_diff_rep;
    // device re-evaluation of every recorded call
    const int64_t m = (int64_t)log.size();
    std::vector<double> hx(m), hy(m);
    std::vector<int> hf(m);
    for (int64_t i = 0; i < m; ++i) {
      hx[i] = log[i].x;
      hf[i] = log[i].fn;
    }
    double *dx, *dy;
    int* df;
    cudaMalloc(&dx, 8 * m);
    cudaMalloc(&dy, 8 * m);
    cudaMalloc(&df, 4 * m);
    cudaMemcpy(dx, hx.data(), 8 * m, cudaMemcpyHostToDevice);
    cudaMemcpy(df, hf.data(), 4 * m, cudaMemcpyHostToDevice);
    eval<<<1184, 256>>>(dx, df, dy, m);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      fprintf(stderr, "device evaluation failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
    cudaMemcpy(hy.data(), dy, 8 * m, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(df);
    std::vector<char> rb(n, 0);
    for (int64_t i = 0; i < m; ++i) {
      calls[log[i].fn]++;
      if (std::memcmp(&hy[i], &log[i].host, 8) != 0) {
        bad[log[i].fn]++;
        if (log[i].req >= 0) rb[log[i].req] = 1;
      }
    }
    long long rbn = 0;
    for (char c : rb) rbn += c;
    req_bad += rbn;
    req_total += n;
    rep_bad += rbn > 0;
  }
  const char* names[kFns] = {"log", "exp", "cos"};
  printf("{\"seeds\": %d, \"requests_per_replay\": %lld, \"rate\": %g, "
         "\"restatement_differs_from_engine_generator\": %lld, \"calls\": {",
         seeds, (long long)n, rate, trace_diff_rep);
  for (int f = 0; f < kFns; ++f)
    printf("%s\"%s\": {\"calls\": %lld, \"device_differs\": %lld, \"rate\": %.3e}",
           f ? ", " : "", names[f], calls[f], bad[f], calls[f] ? (double)bad[f] / calls[f] : 0.0);
  printf("}, \"requests_with_a_differing_call\": %lld, \"requests\": %lld, "
         "\"replays_with_a_differing_call\": %d, \"replays\": %d}\n",
         req_bad, req_total, (int)rep_bad, seeds);
  return 0;
}
