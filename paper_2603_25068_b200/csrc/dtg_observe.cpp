// Observation / output side of the path: the count
// series the simulator emits and the calibration consumes.
//
//   synthesize_observations  observation.cpp:46-83
//   count_metrics            optimization.cpp:297-336
//   series_to_csv / from_csv pipeline.cpp:113-160 (byte-identical CSV)
//   slice_intervals          pipeline.cpp:50-57
//
// Host C++ (O(K·L) work); built with -ffp-contract=off so `lo + (hi - lo) * u`
// and the metric sums round exactly like the reference.
//
// TRANSCRIBED HOST CODE: synthesize_observations, count_metrics and the CSV
// reader/writer restate the reference functions cited above line for line
// (byte-identical outputs need the same operation order); not B200 work.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/dtg.h"
#include "../../include/dtg_engine.hpp"

namespace dtg {

std::pair<CountSeries, std::vector<int>> synthesize_observations(const CountSeries& truth,
                                                                 double noise_frac, double coverage,
                                                                 const RngStream& rng) {
  const RngStream noise = rng.fork(lane::kObsNoise);
  const RngStream cover = rng.fork(lane::kObsCoverage);
  // seeded Fisher-Yates over positions; the first floor(c * n), ascending
  const int n = static_cast<int>(truth.link_ids.size());
  std::vector<int> pos(n);
  for (int i = 0; i < n; ++i) pos[i] = i;
  for (int i = n - 1; i > 0; --i) {
    const int j = static_cast<int>(cover.bits(static_cast<std::uint64_t>(i)) %
                                   static_cast<std::uint64_t>(i + 1));
    std::swap(pos[i], pos[j]);
  }
  const int m = static_cast<int>(std::floor(coverage * n));
  std::vector<int> chosen(pos.begin(), pos.begin() + m);
  std::sort(chosen.begin(), chosen.end());
  CountSeries obs;
  obs.interval_s = truth.interval_s;
  std::vector<int> ids;
  ids.reserve(chosen.size());
  for (int p : chosen) ids.push_back(truth.link_ids[p]);
  obs.link_ids = ids;
  obs.values.resize(truth.values.size());
  for (std::size_t k = 0; k < truth.values.size(); ++k) {
    obs.values[k].resize(chosen.size());
    for (std::size_t q = 0; q < chosen.size(); ++q) {
      const int p = chosen[q];
      const double eps = noise.uniform_in(-noise_frac, noise_frac, static_cast<std::uint64_t>(p),
                                          static_cast<std::uint64_t>(k));
      obs.values[k][q] = std::max(truth.values[k][p] * (1.0 + eps), 0.0);
    }
  }
  return {std::move(obs), std::move(ids)};
}

Metrics count_metrics(const CountSeries& sim, const CountSeries& truth) {
  Metrics m;
  std::vector<double> a, b;
  for (std::size_t q = 0; q < truth.link_ids.size(); ++q) {
    const auto it = std::find(sim.link_ids.begin(), sim.link_ids.end(), truth.link_ids[q]);
    if (it == sim.link_ids.end()) continue;
    const std::size_t p = it - sim.link_ids.begin();
    const int K = std::min(sim.n_intervals(), truth.n_intervals());
    for (int k = 0; k < K; ++k) {  // per-interval increments
      a.push_back(sim.values[k][p] - (k > 0 ? sim.values[k - 1][p] : 0.0));
      b.push_back(truth.values[k][q] - (k > 0 ? truth.values[k - 1][q] : 0.0));
    }
  }
  m.n_pairs = static_cast<int>(a.size());
  if (a.empty()) return m;
  double ma = 0.0, mb = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    m.mae += std::abs(a[i] - b[i]);
    ma += a[i];
    mb += b[i];
  }
  m.mae /= a.size();
  ma /= a.size();
  mb /= b.size();
  double sab = 0.0, saa = 0.0, sbb = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    sab += (a[i] - ma) * (b[i] - mb);
    saa += (a[i] - ma) * (a[i] - ma);
    sbb += (b[i] - mb) * (b[i] - mb);
  }
  if (saa > 0.0 && sbb > 0.0) {
    m.pearson_r = sab / std::sqrt(saa * sbb);
    m.r_defined = true;
  }
  return m;
}

CountSeries slice_intervals(const CountSeries& s, int k0, int k1) {
  CountSeries out;
  out.link_ids = s.link_ids;
  out.interval_s = s.interval_s;
  for (int k = k0; k < k1 && k < s.n_intervals(); ++k) out.values.push_back(s.values[k]);
  return out;
}

namespace {
std::string fmt_g(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.12g", v);
  return buf;
}
}  // namespace

std::string series_to_csv(const CountSeries& s) {
  std::string out = "link_id,t_seconds,cumulative_count\n";
  for (int k = 0; k < s.n_intervals(); ++k) {
    const int t = (k + 1) * s.interval_s;
    for (std::size_t p = 0; p < s.link_ids.size(); ++p) {
      out += std::to_string(s.link_ids[p]);
      out += ',';
      out += std::to_string(t);
      out += ',';
      out += fmt_g(s.values[k][p]);
      out += '\n';
    }
  }
  return out;
}

CountSeries series_from_csv(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error("count CSV: empty file");
  CountSeries s;
  std::vector<int> times;
  std::vector<std::tuple<int, int, double>> rows;  // (t, link, value)
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    int link, t;
    double v;
    if (std::sscanf(line.c_str(), "%d,%d,%lf", &link, &t, &v) != 3)
      throw std::runtime_error("count CSV: malformed row: " + line);
    rows.emplace_back(t, link, v);
  }
  std::sort(rows.begin(), rows.end());
  for (const auto& [t, link, v] : rows) {
    if (times.empty() || times.back() != t) {
      times.push_back(t);
      s.values.emplace_back();
    }
    if (times.size() == 1) s.link_ids.push_back(link);
    s.values.back().push_back(v);
  }
  if (times.empty()) throw std::runtime_error("count CSV: no data rows");
  s.interval_s = times[0];
  for (std::size_t k = 0; k < times.size(); ++k) {
    if (times[k] != static_cast<int>(k + 1) * s.interval_s)
      throw std::runtime_error("count CSV: irregular interval grid");
    if (s.values[k].size() != s.link_ids.size())
      throw std::runtime_error("count CSV: ragged link sets per interval");
  }
  return s;
}

}  // namespace dtg

// ---- level-2 C-ABI -------------------------------------------------------------------
namespace {
thread_local std::string g_obs_error;

template <class F>
int obs_guard(F&& f) {
  try {
    f();
    return DTG_OK;
  } catch (const std::exception& e) {
    g_obs_error = e.what();
    return DTG_ERR_RUNTIME;
  }
}

dtg::CountSeries series_of(int k, int n, const int* ids, const double* values, int interval_s) {
  dtg::CountSeries s;
  s.link_ids.assign(ids, ids + n);
  s.interval_s = interval_s;
  for (int q = 0; q < k; ++q)
    s.values.emplace_back(values + static_cast<std::size_t>(q) * n, values + static_cast<std::size_t>(q + 1) * n);
  return s;
}
}  // namespace

extern "C" {

const char* dtg_observe_last_error(void) { return g_obs_error.c_str(); }

int dtg_synthesize_observations(int k, int n, const int* link_ids, const double* values, int interval_s,
                                double noise_frac, double coverage, uint64_t root_seed, int* m_out,
                                int* obs_ids, double* obs_values) {
  return obs_guard([&] {
    const auto r = dtg::synthesize_observations(series_of(k, n, link_ids, values, interval_s), noise_frac,
                                                coverage, dtg::RngStream(root_seed));
    const int m = static_cast<int>(r.second.size());
    *m_out = m;
    std::copy(r.second.begin(), r.second.end(), obs_ids);
    for (int q = 0; q < k; ++q)
      std::copy(r.first.values[q].begin(), r.first.values[q].end(), obs_values + static_cast<std::size_t>(q) * m);
  });
}

int dtg_count_metrics(int k_sim, int n_sim, const int* sim_ids, const double* sim_values, int k_truth,
                      int n_truth, const int* truth_ids, const double* truth_values, double* mae,
                      double* pearson_r, int* r_defined, int* n_pairs) {
  return obs_guard([&] {
    const dtg::Metrics m = dtg::count_metrics(series_of(k_sim, n_sim, sim_ids, sim_values, 1),
                                              series_of(k_truth, n_truth, truth_ids, truth_values, 1));
    *mae = m.mae;
    *pearson_r = m.pearson_r;
    *r_defined = m.r_defined ? 1 : 0;
    *n_pairs = m.n_pairs;
  });
}

int dtg_series_to_csv(int k, int n, const int* ids, const double* values, int interval_s, char* buf,
                      size_t cap, size_t* len) {
  return obs_guard([&] {
    const std::string s = dtg::series_to_csv(series_of(k, n, ids, values, interval_s));
    *len = s.size();
    if (buf) {
      if (cap < s.size() + 1) throw std::runtime_error("series_to_csv: buffer too small");
      std::memcpy(buf, s.c_str(), s.size() + 1);
    }
  });
}

int dtg_series_from_csv(const char* text, int* k, int* n, int* interval_s, int* ids, double* values,
                        size_t cap_ids, size_t cap_values) {
  return obs_guard([&] {
    const dtg::CountSeries s = dtg::series_from_csv(text);
    *k = s.n_intervals();
    *n = static_cast<int>(s.link_ids.size());
    *interval_s = s.interval_s;
    if (!ids || !values) return;
    if (cap_ids < s.link_ids.size() ||
        cap_values < static_cast<std::size_t>(s.n_intervals()) * s.link_ids.size())
      throw std::runtime_error("series_from_csv: output buffers too small");
    std::copy(s.link_ids.begin(), s.link_ids.end(), ids);
    for (int q = 0; q < s.n_intervals(); ++q)
      std::copy(s.values[q].begin(), s.values[q].end(), values + static_cast<std::size_t>(q) * s.link_ids.size());
  });
}

}  // extern "C"
