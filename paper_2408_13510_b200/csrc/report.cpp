// report.cpp — host side of the reference's report layer for one replay:
// compute_metrics + emit_report (metrics.hpp:84-238) writing summary.json,
// requests.csv and timeseries.csv byte-identical to the reference's.
//
// The sums, means and nearest-rank percentiles come from the device
// (rs_replay_stats: sequential pool-index-order sums, percentile_kernel);
// this file only formats.  CSV doubles use "%.17g" (format_double,
// metrics.hpp:166-170).  summary.json doubles follow nlohmann::json's
// dump(): Grisu2 shortest-ish digits (Loitsch 2010, alpha = -60, gamma =
// -32, cached powers 10^(-300 + 8i)) printed like printf("%g") with a
// fixed-point window [1e-4, 1e15) and a ".0" suffix on integral values.
// Grisu2 is not always shortest (~0.1% of doubles get one more digit than
// the shortest round-trip form), so the exact digit generation matters for
// byte parity; it is implemented here from the published algorithm and
// checked byte-for-byte against the reference's reports in tests/.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>
#include <algorithm>
#include <cmath>

#include "../../include/rs_abi.h"

namespace rs {
void set_error(const std::string& m);
}

namespace {

// ------------------------------------------------------------- Grisu2
struct DiyFp {
  uint64_t f;
  int e;
};

DiyFp diy_mul(DiyFp x, DiyFp y) {  // upper 64 bits of the product, rounded
  const unsigned __int128 p = (unsigned __int128)x.f * y.f;
  uint64_t h = (uint64_t)(p >> 64);
  const uint64_t l = (uint64_t)p;
  h += l >> 63;
  return {h, x.e + y.e + 64};
}

DiyFp diy_normalize(DiyFp x) {
  const int s = __builtin_clzll(x.f);
  return {x.f << s, x.e - s};
}

struct CachedPow {
  uint64_t f;
  int e;
  int k;
};

// 10^k, k = -300 + 8i, as a normalized 64-bit significand rounded to nearest
// (f * 2^e); generated with exact rational arithmetic.
static const CachedPow kPow10[] = {
    {0xAB70FE17C79AC6CAull, -1060, -300},
    {0xFF77B1FCBEBCDC4Full, -1034, -292},
    {0xBE5691EF416BD60Cull, -1007, -284},
    {0x8DD01FAD907FFC3Cull, -980, -276},
    {0xD3515C2831559A83ull, -954, -268},
    {0x9D71AC8FADA6C9B5ull, -927, -260},
    {0xEA9C227723EE8BCBull, -901, -252},
    {0xAECC49914078536Dull, -874, -244},
    {0x823C12795DB6CE57ull, -847, -236},
    {0xC21094364DFB5637ull, -821, -228},
    {0x9096EA6F3848984Full, -794, -220},
    {0xD77485CB25823AC7ull, -768, -212},
    {0xA086CFCD97BF97F4ull, -741, -204},
    {0xEF340A98172AACE5ull, -715, -196},
    {0xB23867FB2A35B28Eull, -688, -188},
    {0x84C8D4DFD2C63F3Bull, -661, -180},
    {0xC5DD44271AD3CDBAull, -635, -172},
    {0x936B9FCEBB25C996ull, -608, -164},
    {0xDBAC6C247D62A584ull, -582, -156},
    {0xA3AB66580D5FDAF6ull, -555, -148},
    {0xF3E2F893DEC3F126ull, -529, -140},
    {0xB5B5ADA8AAFF80B8ull, -502, -132},
    {0x87625F056C7C4A8Bull, -475, -124},
    {0xC9BCFF6034C13053ull, -449, -116},
    {0x964E858C91BA2655ull, -422, -108},
    {0xDFF9772470297EBDull, -396, -100},
    {0xA6DFBD9FB8E5B88Full, -369, -92},
    {0xF8A95FCF88747D94ull, -343, -84},
    {0xB94470938FA89BCFull, -316, -76},
    {0x8A08F0F8BF0F156Bull, -289, -68},
    {0xCDB02555653131B6ull, -263, -60},
    {0x993FE2C6D07B7FACull, -236, -52},
    {0xE45C10C42A2B3B06ull, -210, -44},
    {0xAA242499697392D3ull, -183, -36},
    {0xFD87B5F28300CA0Eull, -157, -28},
    {0xBCE5086492111AEBull, -130, -20},
    {0x8CBCCC096F5088CCull, -103, -12},
    {0xD1B71758E219652Cull, -77, -4},
    {0x9C40000000000000ull, -50, 4},
    {0xE8D4A51000000000ull, -24, 12},
    {0xAD78EBC5AC620000ull, 3, 20},
    {0x813F3978F8940984ull, 30, 28},
    {0xC097CE7BC90715B3ull, 56, 36},
    {0x8F7E32CE7BEA5C70ull, 83, 44},
    {0xD5D238A4ABE98068ull, 109, 52},
    {0x9F4F2726179A2245ull, 136, 60},
    {0xED63A231D4C4FB27ull, 162, 68},
    {0xB0DE65388CC8ADA8ull, 189, 76},
    {0x83C7088E1AAB65DBull, 216, 84},
    {0xC45D1DF942711D9Aull, 242, 92},
    {0x924D692CA61BE758ull, 269, 100},
    {0xDA01EE641A708DEAull, 295, 108},
    {0xA26DA3999AEF774Aull, 322, 116},
    {0xF209787BB47D6B85ull, 348, 124},
    {0xB454E4A179DD1877ull, 375, 132},
    {0x865B86925B9BC5C2ull, 402, 140},
    {0xC83553C5C8965D3Dull, 428, 148},
    {0x952AB45CFA97A0B3ull, 455, 156},
    {0xDE469FBD99A05FE3ull, 481, 164},
    {0xA59BC234DB398C25ull, 508, 172},
    {0xF6C69A72A3989F5Cull, 534, 180},
    {0xB7DCBF5354E9BECEull, 561, 188},
    {0x88FCF317F22241E2ull, 588, 196},
    {0xCC20CE9BD35C78A5ull, 614, 204},
    {0x98165AF37B2153DFull, 641, 212},
    {0xE2A0B5DC971F303Aull, 667, 220},
    {0xA8D9D1535CE3B396ull, 694, 228},
    {0xFB9B7CD9A4A7443Cull, 720, 236},
    {0xBB764C4CA7A44410ull, 747, 244},
    {0x8BAB8EEFB6409C1Aull, 774, 252},
    {0xD01FEF10A657842Cull, 800, 260},
    {0x9B10A4E5E9913129ull, 827, 268},
    {0xE7109BFBA19C0C9Dull, 853, 276},
    {0xAC2820D9623BF429ull, 880, 284},
    {0x80444B5E7AA7CF85ull, 907, 292},
    {0xBF21E44003ACDD2Dull, 933, 300},
    {0x8E679C2F5E44FF8Full, 960, 308},
    {0xD433179D9C8CB841ull, 986, 316},
    {0x9E19DB92B4E31BA9ull, 1013, 324},
};

constexpr int kAlpha = -60, kGamma = -32;

// The cached power c = 10^-k with kAlpha <= c.e + e + 64 <= kGamma: the
// first table entry at or above k = ceil((kAlpha - e - 1) * log10(2)).
const CachedPow& cached_power(int e) {
  const int f = kAlpha - e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);  // 78913 / 2^18 ~ log10(2)
  const int index = (300 + k + 7) / 8;
  return kPow10[index];
}

// Shortens the last digit toward w while the candidate stays inside the
// rounding interval and gets closer to w (Grisu2 "round weed").
void round_last(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest,
                uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k &&
         (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf[len - 1]--;
    rest += ten_k;
  }
}

// Digits of M+ down to the precision of delta = M+ - M-.
void digit_gen(char* buf, int& len, int& dexp, DiyFp mm, DiyFp w, DiyFp mp) {
  const int sh = -mp.e;
  const uint64_t one = 1ull << sh;
  uint64_t delta = mp.f - mm.f;
  uint64_t dist = mp.f - w.f;
  uint32_t p1 = (uint32_t)(mp.f >> sh);
  uint64_t p2 = mp.f & (one - 1);
  uint32_t pow10 = 1;
  int n = 1;
  while (n < 10 && (uint64_t)pow10 * 10 <= p1) {
    pow10 *= 10;
    ++n;
  }
  while (n > 0) {
    const uint32_t d = p1 / pow10;
    p1 %= pow10;
    buf[len++] = (char)('0' + d);
    --n;
    const uint64_t rest = ((uint64_t)p1 << sh) + p2;
    if (rest <= delta) {
      dexp += n;
      round_last(buf, len, dist, delta, rest, (uint64_t)pow10 << sh);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    delta *= 10;
    dist *= 10;
    buf[len++] = (char)('0' + (p2 >> sh));
    p2 &= one - 1;
    ++m;
    if (p2 <= delta) break;
  }
  dexp -= m;
  round_last(buf, len, dist, delta, p2, one);
}

// v > 0, finite: digits in buf[0..len), value = digits * 10^dexp.
void grisu2(double v, char* buf, int& len, int& dexp) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t F = bits & ((1ull << 52) - 1);
  const int E = (int)(bits >> 52) & 0x7ff;
  DiyFp x = E == 0 ? DiyFp{F, 1 - 1075} : DiyFp{F | (1ull << 52), E - 1075};
  const bool closer = F == 0 && E > 1;  // lower boundary is closer
  const DiyFp mplus = diy_normalize({(x.f << 1) + 1, x.e - 1});
  DiyFp mminus = closer ? DiyFp{(x.f << 2) - 1, x.e - 2} : DiyFp{(x.f << 1) - 1, x.e - 1};
  mminus = {mminus.f << (mminus.e - mplus.e), mplus.e};
  const DiyFp w = diy_normalize(x);
  const CachedPow& c = cached_power(mplus.e);
  const DiyFp cp{c.f, c.e};
  const DiyFp W = diy_mul(w, cp), Wm = diy_mul(mminus, cp), Wp = diy_mul(mplus, cp);
  len = 0;
  dexp = -c.k;
  digit_gen(buf, len, dexp, {Wm.f + 1, Wm.e}, W, {Wp.f - 1, Wp.e});
}

// nlohmann::json's number_float serialisation of v.
std::string json_double(double v) {
  char b[64];
  char* p = b;
  if (std::signbit(v)) {
    v = -v;
    *p++ = '-';
  }
  if (v == 0.0) return std::string(b, p) + "0.0";
  char d[32];
  int k = 0, dexp = 0;
  grisu2(v, d, k, dexp);
  const int n = k + dexp;  // decimal point position
  std::string s(b, p);
  if (k <= n && n <= 15) {  // digits[000].0
    s.append(d, k);
    s.append((size_t)(n - k), '0');
    s += ".0";
  } else if (0 < n && n <= 15) {  // dig.its
    s.append(d, n);
    s += '.';
    s.append(d + n, k - n);
  } else if (-4 < n && n <= 0) {  // 0.[000]digits
    s += "0.";
    s.append((size_t)(-n), '0');
    s.append(d, k);
  } else {  // d[.igits]e+XX
    s += d[0];
    if (k > 1) {
      s += '.';
      s.append(d + 1, k - 1);
    }
    char e[8];
    const int x = n - 1;
    std::snprintf(e, sizeof(e), "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
    s += e;
  }
  return s;
}

// format_double (metrics.hpp:166-170)
std::string fmt17(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

const char* task_name(int t) {  // to_string(TaskKind), request.hpp:19-28
  static const char* k[] = {"Translation", "QnA", "SentimentAnalysis", "InContextQnA",
                            "EntityRecognition"};
  return t >= 0 && t < RS_NUM_TASKS ? k[t] : "?";
}

// classify_request (latency.hpp:100-121) -> to_string(RequestClass)
const char* class_name(const rs_batch_cfg& c, long long prompt, long long decode) {
  const bool hp = c.profile.prompt_time_per_token * (double)prompt >=
                  c.thresholds.heavy_prompt_seconds;
  const bool hd = c.profile.decode_time_base * (double)decode >= c.thresholds.heavy_decode_seconds;
  if (hp) return hd ? "HH" : "HL";
  return hd ? "LH" : "LL";
}

// nearest rank of aggregate_of (metrics.hpp:70-75) over sorted values
double nearest_rank(const std::vector<double>& v, double q) {
  size_t idx = (size_t)std::ceil(q * (double)v.size());
  if (idx > 0) --idx;
  return v[std::min(idx, v.size() - 1)];
}

struct Agg {
  double mean = 0.0, p50 = 0.0, p90 = 0.0, p99 = 0.0;
  long long count = 0;
};

std::string agg_json(const Agg& a) {  // report_to_json's agg(), dump(2) at depth 1
  return "{\n    \"mean\": " + json_double(a.mean) + ",\n    \"p50\": " + json_double(a.p50) +
         ",\n    \"p90\": " + json_double(a.p90) + ",\n    \"p99\": " + json_double(a.p99) +
         ",\n    \"count\": " + std::to_string(a.count) + "\n  }";
}

rs_status fail(rs_status s, const std::string& m) {
  rs::set_error(m);
  return s;
}

bool write_file(const std::filesystem::path& p, const std::string& s) {
  FILE* f = std::fopen(p.c_str(), "wb");
  if (!f) return false;
  const bool ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
  return std::fclose(f) == 0 && ok;
}

}  // namespace

extern "C" rs_status rs_emit_report(const char* dir, const rs_batch_cfg* cfg, int64_t n,
                                    const double* arrival, const int32_t* prompt,
                                    const int32_t* decode, const uint8_t* task,
                                    const int32_t* instance, const double* routed,
                                    const double* first, const double* completion,
                                    const int32_t* preemptions, const rs_replay_stats* st,
                                    const rs_trajectory* traj, int64_t traj_len) {
  if (!dir || !cfg || !st || n < 0)
    return fail(RS_ERR_INVALID_ARGUMENT, "emit_report: null argument");
  if (n > 0 && (!arrival || !prompt || !decode || !task || !instance || !routed || !first ||
                !completion || !preemptions))
    return fail(RS_ERR_INVALID_ARGUMENT, "emit_report: every per-request array is required");
  const int m = cfg->num_instances;
  if (traj && traj_len > 0 &&
      (!traj->time_s || !traj->action || !traj->reward || !traj->router_queue ||
       !traj->tokens_emitted || !traj->instance_running || !traj->instance_waiting))
    return fail(RS_ERR_INVALID_ARGUMENT,
                "emit_report: timeseries.csv needs time_s, action, reward, router_queue, "
                "tokens_emitted, instance_running and instance_waiting");
  // ---- compute_metrics (metrics.hpp:84-162) over the completed requests
  std::string req = "id,task,class,prompt_tokens,decode_tokens,arrival_s,ttft_s,tbt_s,"
                    "e2e_s,preemptions,instance\n";
  std::vector<double> e2e, ttft, tbt;
  long long waits = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(completion[i] >= 0.0)) continue;
    const double e = completion[i] - arrival[i];
    const double t = first[i] - arrival[i];
    e2e.push_back(e);
    ttft.push_back(t);
    std::string tb;
    if (decode[i] >= 2) {  // tokens_emitted == true decode at completion
      const double b = (completion[i] - first[i]) / (double)(decode[i] - 1);
      tbt.push_back(b);
      tb = fmt17(b);
    }
    if (routed[i] >= 0.0) ++waits;
    req += std::to_string(i) + ',' + task_name(task[i]) + ',' +
           class_name(*cfg, prompt[i], decode[i]) + ',' + std::to_string(prompt[i]) + ',' +
           std::to_string(decode[i]) + ',' + fmt17(arrival[i]) + ',' + fmt17(t) + ',' + tb +
           ',' + fmt17(e) + ',' + std::to_string(preemptions[i]) + ',' +
           std::to_string(instance[i]) + '\n';
  }
  if (e2e.empty()) return fail(RS_ERR_INVALID_ARGUMENT, "compute_metrics: no completed requests");
  if ((long long)e2e.size() != st->completed)
    return fail(RS_ERR_INVALID_ARGUMENT, "emit_report: stats do not belong to these outputs");
  // means: the device's sequential pool-order sums; percentiles: the
  // device's nearest-rank selections (host sort when not computed)
  auto agg = [&](std::vector<double>& v, double total, const double* p) {
    Agg a;
    a.count = (long long)v.size();
    if (v.empty()) return a;
    a.mean = total / (double)v.size();
    if (st->percentiles_valid) {
      a.p50 = p[0];
      a.p90 = p[1];
      a.p99 = p[2];
    } else {
      std::sort(v.begin(), v.end());
      a.p50 = nearest_rank(v, 0.50);
      a.p90 = nearest_rank(v, 0.90);
      a.p99 = nearest_rank(v, 0.99);
    }
    return a;
  };
  const double pe[3] = {st->e2e_p50, st->e2e_p90, st->e2e_p99};
  const double pt[3] = {st->ttft_p50, st->ttft_p90, st->ttft_p99};
  const double pb[3] = {st->tbt_p50, st->tbt_p90, st->tbt_p99};
  const Agg ae = agg(e2e, st->total_e2e_s, pe), at = agg(ttft, st->total_ttft_s, pt),
            ab = agg(tbt, st->total_tbt_s, pb);
  const double mean_wait = waits ? st->total_router_wait_s / (double)waits : 0.0;
  // time averages over the TickRecords (record_trajectory on), else 0
  double mean_q = 0.0, mean_w = 0.0;
  if (traj && st->ticks > 0) {
    mean_q = (double)st->sum_router_queue / (double)st->ticks;
    mean_w = (double)st->sum_instance_waiting / (double)(st->ticks * m);
  }
  const double thr = st->makespan_s > 0.0 ? (double)st->total_tokens / st->makespan_s : 0.0;
  // ---- report_to_json(...).dump(2) (metrics.hpp:172-194)
  std::string js = "{\n  \"completed\": " + std::to_string(st->completed) +
                   ",\n  \"total_tokens\": " + std::to_string(st->total_tokens) +
                   ",\n  \"total_e2e_s\": " + json_double(st->total_e2e_s) +
                   ",\n  \"makespan_s\": " + json_double(st->makespan_s) +
                   ",\n  \"e2e_s\": " + agg_json(ae) + ",\n  \"ttft_s\": " + agg_json(at) +
                   ",\n  \"tbt_s\": " + agg_json(ab) +
                   ",\n  \"mean_router_wait_s\": " + json_double(mean_wait) +
                   ",\n  \"mean_router_queue\": " + json_double(mean_q) +
                   ",\n  \"mean_instance_waiting\": " + json_double(mean_w) +
                   ",\n  \"mean_throughput_tokens_s\": " + json_double(thr) +
                   ",\n  \"total_preemptions\": " + std::to_string(st->total_preemptions) +
                   "\n}\n";
  // ---- timeseries.csv (metrics.hpp:222-237)
  const int64_t k = traj ? std::max<int64_t>(0, traj_len) : 0;
  const int mm = k > 0 ? m : 0;
  std::string ts = "tick,time_s,action,reward,router_queue";
  for (int i = 0; i < mm; ++i) ts += ",inst" + std::to_string(i) + "_waiting";
  for (int i = 0; i < mm; ++i) ts += ",inst" + std::to_string(i) + "_running";
  ts += ",tokens_emitted\n";
  for (int64_t t = 0; t < k; ++t) {
    ts += std::to_string(t + 1) + ',' + fmt17(traj->time_s[t]) + ',' +
          std::to_string(traj->action[t]) + ',' + fmt17(traj->reward[t]) + ',' +
          std::to_string(traj->router_queue[t]);
    for (int i = 0; i < mm; ++i) ts += ',' + std::to_string(traj->instance_waiting[t * m + i]);
    for (int i = 0; i < mm; ++i) ts += ',' + std::to_string(traj->instance_running[t * m + i]);
    ts += ',' + std::to_string(traj->tokens_emitted[t]) + '\n';
  }
  // ---- emit_report (metrics.hpp:197-238)
  namespace fs = std::filesystem;
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (!write_file(fs::path(dir) / "summary.json", js))
    return fail(RS_ERR_INVALID_ARGUMENT, "emit_report: cannot write summary.json");
  if (!write_file(fs::path(dir) / "requests.csv", req))
    return fail(RS_ERR_INVALID_ARGUMENT, "emit_report: cannot write requests.csv");
  if (!write_file(fs::path(dir) / "timeseries.csv", ts))
    return fail(RS_ERR_INVALID_ARGUMENT, "emit_report: cannot write timeseries.csv");
  return RS_OK;
}
