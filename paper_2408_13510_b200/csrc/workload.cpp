// workload.cpp — host-side synthetic trace generation (the INPUT side of the
// hot path; it runs once per replay on the host, SURVEY.md §8 "next" rank 3).
//
// Restates the reference generator so that a seed yields the identical
// trace: std::mt19937_64 draws consumed exactly as Rng does (rng.hpp:21-63),
// truncated-lognormal rejection sampling with mean matching by bisection
// (workload.hpp:27-81), the light/heavy decode mixture per task
// (workload.hpp:96-151) over Table 1 (workload.hpp:165-174), task selection
// and Poisson arrivals (workload.hpp:209-245).  The same glibc libm calls in
// the same operation order, compiled without FP contraction, so traces are
// bit-identical to the reference's (checked against oracle/_ref in tests).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "../../include/rs_abi.h"

namespace {

constexpr long long kMaxPrompt = 1000;   // workload.hpp:22
constexpr long long kMaxDecode = 4096;   // workload.hpp:23

struct Source {  // Rng
  std::mt19937_64 eng;
  explicit Source(uint64_t s) : eng(s) {}
  double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double gauss() {  // Box-Muller, two draws, the second value discarded
    double u1 = uniform();
    double u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }
  double expo(double rate) {
    double u = uniform();
    while (u <= 0.0) u = uniform();
    return -std::log(u) / rate;
  }
};

struct TLN {  // lognormal truncated to [lo, hi]
  double mu = 0.0, sigma = 0.5, lo = 1.0, hi = 4096.0;

  static double cdf_gap(double a, double b) {
    constexpr double r = 0.70710678118654752440;
    return 0.5 * (std::erfc(a * r) - std::erfc(b * r));
  }
  double truncated_mean() const {
    double a = (std::log(lo) - mu) / sigma;
    double b = (std::log(hi) - mu) / sigma;
    double den = cdf_gap(a, b);
    if (den <= 0.0) return a > 0.0 ? lo : hi;
    double num = cdf_gap(a - sigma, b - sigma);
    return std::exp(mu + 0.5 * sigma * sigma) * num / den;
  }
  static TLN fit(double target, double sigma, double lo, double hi) {
    TLN d{0.0, sigma, lo, hi};
    double a = std::log(lo) - 36.0 * sigma;
    double b = std::log(hi) + 36.0 * sigma;
    for (int it = 0; it < 300; ++it) {
      d.mu = 0.5 * (a + b);
      if (d.truncated_mean() < target) a = d.mu; else b = d.mu;
    }
    return d;
  }
  double draw(Source& s) const {
    for (int t = 0; t < 10000; ++t) {
      double x = std::exp(mu + sigma * s.gauss());
      if (x >= lo && x <= hi) return x;
    }
    return std::clamp(std::exp(mu), lo, hi);
  }
  long long tokens(Source& s) const {
    long long t = std::llround(draw(s));
    long long a = static_cast<long long>(std::ceil(lo));
    long long b = static_cast<long long>(std::floor(hi));
    return std::clamp(t, a, b);
  }
};

struct Task {
  uint8_t kind;
  double heavy_frac;
  TLN prompt, light, heavy;
};

struct Row {
  double samples, mean_prompt, mean_decode, heavy_frac;
};
constexpr Row kTable[RS_NUM_TASKS] = {  // Table 1, workload.hpp:165-174
    {7351, 29.09, 61.76, 0.0918},
    {6988, 29.83, 334.40, 0.5818},
    {6564, 211.54, 142.53, 0.4101},
    {7122, 125.16, 220.02, 0.4795},
    {3304, 26.41, 64.10, 0.0871},
};

double narrowed(double nominal, double target, double lo, double hi) {
  double room = std::min(target / lo - 1.0, hi / target - 1.0);
  return std::min(nominal, std::max(0.05, room));
}

// TaskSpec::make (workload.hpp:96-151) with its default sigmas.
Task make_task(uint8_t kind, const Row& row, long long cut) {
  const double ps = 0.7, ls = 0.6, hs = 0.45;
  Task t;
  t.kind = kind;
  t.heavy_frac = row.heavy_frac;
  const double pcap = static_cast<double>(kMaxPrompt);
  t.prompt = TLN::fit(row.mean_prompt, narrowed(ps, row.mean_prompt, 1.0, pcap), 1.0, pcap);
  const double b = static_cast<double>(cut), cap = static_cast<double>(kMaxDecode);
  const double q = row.heavy_frac, md = row.mean_decode;
  auto light = [&](double m) { return TLN::fit(m, narrowed(ls, m, 1.0, b - 1.0), 1.0, b - 1.0); };
  auto heavy = [&](double m) { return TLN::fit(m, narrowed(hs, m, b, cap), b, cap); };
  if (q <= 0.0) {
    t.light = light(md);
    t.heavy = TLN{std::log(1.2 * b), 0.1, b, cap};
  } else if (q >= 1.0) {
    t.heavy = heavy(md);
    t.light = TLN{0.0, ls, 1.0, b - 1.0};
  } else {
    double ml = std::min(0.6 * b, std::max(1.5, 0.5 * md));
    double mh = (md - (1.0 - q) * ml) / q;
    mh = std::clamp(mh, 1.02 * b, 0.9 * cap);
    ml = (md - q * mh) / (1.0 - q);
    ml = std::clamp(ml, 1.5, 0.98 * (b - 1.0));
    t.light = light(ml);
    t.heavy = heavy(mh);
  }
  return t;
}

long long cutoff(const rs_profile& p, const rs_thresholds& th) {
  long long c = static_cast<long long>(std::ceil(th.heavy_decode_seconds / p.decode_time_base - 1e-12));
  while (!(p.decode_time_base * static_cast<double>(c) >= th.heavy_decode_seconds)) ++c;
  return c;
}

struct Mixture {
  std::vector<Task> tasks;
  std::vector<double> weights;
};

Mixture build(const rs_profile& p, const rs_thresholds& th, const double* w) {
  Mixture mx;
  const long long cut = cutoff(p, th);
  for (int k = 0; k < RS_NUM_TASKS; ++k) {
    mx.tasks.push_back(make_task(static_cast<uint8_t>(k), kTable[k], cut));
    mx.weights.push_back(w ? w[k] : kTable[k].samples);
  }
  return mx;
}

// generate_mixture + assign_arrivals (workload.hpp:209-245) from Rng(rng_seed)
void generate_raw(const Mixture& mx, uint64_t rng_seed, int64_t n, double rate, int process,
                  double* arrival, int32_t* prompt, int32_t* decode, uint8_t* task) {
  Source s(rng_seed);
  double total = 0.0;
  for (double w : mx.weights) total += w;
  const size_t kinds = mx.tasks.size();
  for (int64_t i = 0; i < n; ++i) {
    double u = s.uniform() * total;
    size_t k = 0;
    for (; k + 1 < kinds; ++k) {
      u -= mx.weights[k];
      if (u < 0.0) break;
    }
    const Task& t = mx.tasks[k];
    task[i] = t.kind;
    prompt[i] = static_cast<int32_t>(t.prompt.tokens(s));
    const bool heavy = s.uniform() < t.heavy_frac;
    decode[i] = static_cast<int32_t>((heavy ? t.heavy : t.light).tokens(s));
  }
  double clock = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    clock += process == 0 ? s.expo(rate) : 1.0 / rate;
    arrival[i] = clock;
  }
}

// build_workload's stream: Rng(mix_seed(seed, 0xB00C)) (experiment.hpp:293)
void generate(const Mixture& mx, uint64_t seed, int64_t n, double rate, int process,
              double* arrival, int32_t* prompt, int32_t* decode, uint8_t* task) {
  generate_raw(mx, rs_mix_seed(seed, 0xB00C), n, rate, process, arrival, prompt, decode, task);
}

// BucketScheme::bucket_of (predictor.hpp:34-40): last edge <= tokens
int bucket_of_edges(const int64_t* edges, int n, int64_t tokens) {
  int b = 0;
  for (int i = 1; i < n; ++i)
    if (tokens >= edges[i]) b = i;
  return b;
}

// argmax with the lowest index on ties (std::max_element, predictor.hpp:168-170)
int argmax_counts(const long long* v, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

}  // namespace

extern "C" {

// EmpiricalPredictor::fit (predictor.hpp:119-142) on a training trace, then
// predict() (predictor.hpp:146-158: the (task, prompt band) cell's argmax,
// else the task marginal's, else the global one) resolved for every cell into
// cfg->empirical_table; sets predictor_mode = RS_PREDICTOR_EMPIRICAL.
rs_status rs_empirical_fit_trace(rs_batch_cfg* cfg, int64_t n, const int32_t* prompt,
                                 const int32_t* decode, const uint8_t* task) {
  if (!cfg || n < 1 || !prompt || !decode || !task) return RS_ERR_INVALID_ARGUMENT;
  const int nb = cfg->n_predictor_edges, nbands = cfg->n_band_edges;
  if (nb < 1 || nb > RS_MAX_BUCKETS || nbands < 1 || nbands > RS_MAX_BANDS)
    return RS_ERR_INVALID_ARGUMENT;
  long long cells[RS_NUM_TASKS][RS_MAX_BANDS][RS_MAX_BUCKETS] = {};
  bool seen[RS_NUM_TASKS][RS_MAX_BANDS] = {};
  long long marg[RS_NUM_TASKS][RS_MAX_BUCKETS] = {};
  bool tseen[RS_NUM_TASKS] = {};
  long long global[RS_MAX_BUCKETS] = {};
  for (int64_t i = 0; i < n; ++i) {
    if (task[i] >= RS_NUM_TASKS) return RS_ERR_INVALID_ARGUMENT;
    const int b = bucket_of_edges(cfg->predictor_edges, nb, decode[i]);
    const int band = bucket_of_edges(cfg->band_edges, nbands, prompt[i]);
    cells[task[i]][band][b] += 1;
    seen[task[i]][band] = true;
    marg[task[i]][b] += 1;
    tseen[task[i]] = true;
    global[b] += 1;
  }
  for (int t = 0; t < RS_NUM_TASKS; ++t)
    for (int band = 0; band < RS_MAX_BANDS; ++band) {
      int pred = 0;
      if (band < nbands && seen[t][band]) pred = argmax_counts(cells[t][band], nb);
      else if (tseen[t]) pred = argmax_counts(marg[t], nb);
      else pred = argmax_counts(global, nb);
      cfg->empirical_table[t][band] = static_cast<uint8_t>(pred);
    }
  cfg->predictor_mode = RS_PREDICTOR_EMPIRICAL;
  return RS_OK;
}

// run_experiment's empirical predictor (experiment.hpp:341-351): fit on
// n_train requests of the Table-1 mixture drawn from Rng(mix_seed(seed,
// 0xF17)) (generate_dataset_mixture; arrival draws come after all token draws
// and do not affect the fit).
rs_status rs_empirical_fit(rs_batch_cfg* cfg, uint64_t seed, int64_t n_train) {
  if (!cfg || n_train < 1) return RS_ERR_INVALID_ARGUMENT;
  const Mixture mx = build(cfg->profile, cfg->thresholds, nullptr);
  std::vector<double> arr(static_cast<size_t>(n_train));
  std::vector<int32_t> pr(static_cast<size_t>(n_train)), de(static_cast<size_t>(n_train));
  std::vector<uint8_t> tk(static_cast<size_t>(n_train));
  generate_raw(mx, rs_mix_seed(seed, 0xF17), n_train, 1.0, 0, arr.data(), pr.data(), de.data(),
               tk.data());
  return rs_empirical_fit_trace(cfg, n_train, pr.data(), de.data(), tk.data());
}

rs_status rs_generate_mixture(const rs_profile* profile, const rs_thresholds* thresholds,
                              const double* task_weights, uint64_t seed, int64_t n,
                              double rate_per_s, int32_t process, double* arrival_s,
                              int32_t* prompt_tokens, int32_t* decode_tokens, uint8_t* task) {
  if (!profile || !thresholds || n < 1 || !(rate_per_s > 0.0) || !arrival_s || !prompt_tokens ||
      !decode_tokens || !task || (process != 0 && process != 1))
    return RS_ERR_INVALID_ARGUMENT;
  Mixture mx = build(*profile, *thresholds, task_weights);
  generate(mx, seed, n, rate_per_s, process, arrival_s, prompt_tokens, decode_tokens, task);
  return RS_OK;
}

rs_status rs_generate_mixture_batch(const rs_profile* profile, const rs_thresholds* thresholds,
                                    const double* task_weights, const uint64_t* seeds,
                                    int32_t num_seeds, int64_t n, double rate_per_s,
                                    int32_t process, int32_t threads, double* arrival_s,
                                    int32_t* prompt_tokens, int32_t* decode_tokens,
                                    uint8_t* task) {
  if (!profile || !thresholds || !seeds || num_seeds < 0 || n < 1 || !(rate_per_s > 0.0) ||
      !arrival_s || !prompt_tokens || !decode_tokens || !task || (process != 0 && process != 1))
    return RS_ERR_INVALID_ARGUMENT;
  const Mixture mx = build(*profile, *thresholds, task_weights);
  if (threads <= 0) threads = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency()));
  threads = std::min<int32_t>(threads, std::max(1, num_seeds));
  std::atomic<int32_t> next{0};
  auto work = [&]() {
    for (;;) {
      const int32_t r = next.fetch_add(1);
      if (r >= num_seeds) break;
      const int64_t o = static_cast<int64_t>(r) * n;
      generate(mx, seeds[r], n, rate_per_s, process, arrival_s + o, prompt_tokens + o,
               decode_tokens + o, task + o);
    }
  };
  std::vector<std::thread> pool;
  for (int32_t i = 1; i < threads; ++i) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return RS_OK;
}

rs_status rs_mlp_random_init(const int32_t* dims, int32_t num_layers, uint64_t seed,
                             double* params_out) {
  if (!dims || !params_out || num_layers < 1) return RS_ERR_INVALID_ARGUMENT;
  Source s(seed);
  double* p = params_out;
  for (int l = 0; l < num_layers; ++l) {
    const double scale = std::sqrt(2.0 / static_cast<double>(dims[l]));
    const size_t wn = static_cast<size_t>(dims[l]) * static_cast<size_t>(dims[l + 1]);
    for (size_t i = 0; i < wn; ++i) p[i] = (2.0 * s.uniform() - 1.0) * scale;
    for (int o = 0; o < dims[l + 1]; ++o) p[wn + o] = 0.0;
    p += wn + dims[l + 1];
  }
  return RS_OK;
}

}  // extern "C"
