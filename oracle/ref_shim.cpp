// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference sources
// (/root/reference/proj/src/{tensor,network,car_following,node_model,
// observation,engine,optimization}.cpp), compiled by oracle/Makefile into
// oracle/_ref/libdtsim_ref.so.  It only builds reference objects
// (Scenario, LinkParams, RngStream, LossBuilder) and calls the reference's
// own entry points:
//   simulate_forward   include/dtsim/engine.hpp:76-78  (src/engine.cpp:227-254)
//   simulate_gradient  include/dtsim/engine.hpp:105-107 (src/engine.cpp:303-429)
// so the outputs ARE the reference's outputs.  Used by tests/ (golden
// generation, oracle pinning) and by bench.py's `--impl reference` arm.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "dtsim/engine.hpp"
#include "dtsim/network.hpp"
#include "dtsim/observation.hpp"
#include "dtsim/optimization.hpp"
#include "dtsim/pipeline.hpp"

using namespace dtsim;

namespace {
thread_local std::string g_err;

struct RefScn {
  Scenario s;
};

LinkParams make_params(int L, const double* u, const double* k,
                       const double* b, const double* a, const double* c) {
  LinkParams p;
  p.u.assign(u, u + L);
  p.kappa.assign(k, k + L);
  p.beta.assign(b, b + L);
  p.alpha.assign(a, a + L);
  p.cost.assign(c, c + L);
  return p;
}

// Compact (link, pos) of a dense N x L row-major state; exactly the
// reference's compact_state rule (src/engine.cpp:267-285).
void compact(const std::vector<double>& X, int N, int L, double M, int* link,
             double* pos) {
  for (int i = 0; i < N; ++i) {
    link[i] = -1;
    pos[i] = 0.0;
    for (int j = 0; j < L; ++j) {
      const double x = X[static_cast<std::size_t>(i) * L + j];
      if (x != -M) {
        link[i] = j;
        pos[i] = x;
        break;
      }
    }
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- RNG (include/dtsim/rng.hpp) -------------------------------------------
uint64_t ref_rng_fork(uint64_t seed, uint64_t label) {
  return RngStream(seed).fork(label).seed();
}
uint64_t ref_rng_bits(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return RngStream(seed).bits(a, b, c);
}
double ref_rng_uniform(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return RngStream(seed).uniform(a, b, c);
}
/// One Gumbel draw exactly as gumbel_sample_keys computes it
/// (src/tensor.cpp:682-699): stream `seed`, key, row key, column key.
double ref_gumbel(uint64_t seed, uint64_t key, int row, int col) {
  std::vector<int> rk{row}, ck{col};
  return gumbel_sample_keys({1, 1}, RngStream(seed), key, &rk, &ck).vals()[0];
}

// ---- scenarios ---------------------------------------------------------------
/// Explicit-link scenario (make_network, network.cpp:238-247).  kind: 0 physical,
/// 1 virtual inflow, 2 virtual outflow.  n_custom > 0 sets custom_init.
void* ref_scenario_links(int n_nodes, int n_links, const int* from,
                         const int* to, const double* len, const int* kind) {
  auto* r = new RefScn;
  std::vector<Link> links(n_links);
  for (int i = 0; i < n_links; ++i) {
    links[i].id = i;
    links[i].from_node = from[i];
    links[i].to_node = to[i];
    links[i].length = len[i];
    links[i].kind = static_cast<LinkKind>(kind[i]);
  }
  r->s.net = make_network(n_nodes, std::move(links));
  return r;
}

/// Synthetic grid (SURVEY §8d generator) + attach_virtual_links
/// (network.cpp:151-201) with RngStream(net_seed).
void* ref_scenario_grid(int n, double len, uint64_t net_seed, double virt_len) {
  void* out = nullptr;
  if (guarded([&] {
        std::vector<Link> links;
        auto push = [&](int a, int b) {
          Link l;
          l.from_node = a;
          l.to_node = b;
          l.length = len;
          l.kind = LinkKind::Physical;
          links.push_back(l);
        };
        for (int r = 0; r < n; ++r)
          for (int c = 0; c < n; ++c) {
            if (c + 1 < n) {
              push(r * n + c, r * n + c + 1);
              push(r * n + c + 1, r * n + c);
            }
            if (r + 1 < n) {
              push(r * n + c, (r + 1) * n + c);
              push((r + 1) * n + c, r * n + c);
            }
          }
        Network phys = make_network(n * n, std::move(links));
        auto* rs = new RefScn;
        rs->s.net = attach_virtual_links(phys, RngStream(net_seed), virt_len);
        out = rs;
      }))
    return nullptr;
  return out;
}

/// parse_tntp_text (network.cpp:58-118) + attach_virtual_links with
/// RngStream(net_seed), as build_network does (pipeline.cpp:165-170).
void* ref_scenario_tntp(const char* text, double unit_scale, uint64_t net_seed,
                        double virt_len) {
  void* out = nullptr;
  if (guarded([&] {
        Network phys = parse_tntp_text(std::string(text), unit_scale);
        auto* rs = new RefScn;
        rs->s.net = attach_virtual_links(phys, RngStream(net_seed), virt_len);
        out = rs;
      }))
    return nullptr;
  return out;
}

/// parse_tntp_text alone: the physical links (n_links returned, -1 on error;
/// arrays may be NULL to query the size).
int ref_tntp_physical(const char* text, double unit_scale, int* from, int* to,
                      double* len, int* n_nodes) {
  int n = -1;
  if (guarded([&] {
        Network net = parse_tntp_text(std::string(text), unit_scale);
        n = net.n_links();
        if (from)
          for (int i = 0; i < n; ++i) {
            from[i] = net.links[i].from_node;
            to[i] = net.links[i].to_node;
            len[i] = net.links[i].length;
          }
        if (n_nodes) *n_nodes = net.n_nodes;
      }))
    return -1;
  return n;
}

/// attach_virtual_links (network.cpp:151-201) applied in place to a scenario
/// whose network holds physical links only.
int ref_scenario_attach_virtual(void* h, uint64_t net_seed, double virt_len) {
  return guarded([&] {
    auto& s = static_cast<RefScn*>(h)->s;
    s.net = attach_virtual_links(s.net, RngStream(net_seed), virt_len);
  });
}

void ref_scenario_free(void* h) { delete static_cast<RefScn*>(h); }

void ref_scenario_config(void* h, int n_vehicles, int delta_n, double tau,
                         double gumbel_tau, int trajectory_grafting,
                         int horizon_steps, int obs_interval_s) {
  auto& s = static_cast<RefScn*>(h)->s;
  s.n_vehicles = n_vehicles;
  s.cfg.delta_n = delta_n;
  s.cfg.tau = tau;
  s.cfg.gumbel_tau = gumbel_tau;
  s.cfg.trajectory_grafting = trajectory_grafting != 0;
  s.horizon_steps = horizon_steps;
  s.obs_interval_s = obs_interval_s;
}

void ref_scenario_custom_init(void* h, int n, const int* link,
                              const double* pos) {
  auto& s = static_cast<RefScn*>(h)->s;
  s.custom_init.clear();
  for (int i = 0; i < n; ++i) s.custom_init.push_back({link[i], pos[i]});
}

int ref_fit_inflow_queues(void* h) {
  return guarded([&] { fit_inflow_queues(static_cast<RefScn*>(h)->s); });
}

int ref_n_links(void* h) { return static_cast<RefScn*>(h)->s.net.n_links(); }
int ref_n_nodes(void* h) { return static_cast<RefScn*>(h)->s.net.n_nodes; }
int ref_n_agents(void* h) {
  int n = -1;
  if (guarded([&] { n = static_cast<RefScn*>(h)->s.n_agents(); })) return -1;
  return n;
}

void ref_links(void* h, int* from, int* to, double* len, int* kind) {
  const auto& net = static_cast<RefScn*>(h)->s.net;
  for (int i = 0; i < net.n_links(); ++i) {
    from[i] = net.links[i].from_node;
    to[i] = net.links[i].to_node;
    len[i] = net.links[i].length;
    kind[i] = static_cast<int>(net.links[i].kind);
  }
}

void ref_adjacency(void* h, double* adj) {
  const auto& a = static_cast<RefScn*>(h)->s.net.adjacency;
  std::memcpy(adj, a.data(), a.size() * sizeof(double));
}

int ref_sample_parameters(void* h, uint64_t seed, int mean_mode, double* u,
                          double* k, double* b, double* a, double* c) {
  return guarded([&] {
    const auto& net = static_cast<RefScn*>(h)->s.net;
    LinkParams p =
        sample_parameters(net, ParamRanges{}, RngStream(seed), mean_mode != 0);
    const std::size_t L = p.u.size();
    std::memcpy(u, p.u.data(), L * 8);
    std::memcpy(k, p.kappa.data(), L * 8);
    std::memcpy(b, p.beta.data(), L * 8);
    std::memcpy(a, p.alpha.data(), L * 8);
    std::memcpy(c, p.cost.data(), L * 8);
  });
}

int ref_seed_agents(void* h, int* link, double* pos) {
  return guarded([&] {
    InitialState init = seed_agents(static_cast<RefScn*>(h)->s);
    for (std::size_t i = 0; i < init.link.size(); ++i) {
      link[i] = init.link[i];
      pos[i] = init.pos[i];
    }
  });
}

int ref_steps_for_minutes(int delta_n, double tau, double minutes) {
  int out = -1;
  SimConfig c;
  c.delta_n = delta_n;
  c.tau = tau;
  if (guarded([&] { out = steps_for_minutes(c, minutes); })) return -1;
  return out;
}

// ---- hot path ------------------------------------------------------------------
/// simulate_forward (src/engine.cpp:227-254).  cum_per_step: T x L.
/// link_final/pos_final: compact final state per agent.  If states_link is
/// non-null, record_states is set and every step's compact state (T x N) is
/// returned.  wall: the reference's own wall_seconds.
int ref_forward(void* h, const double* u, const double* k, const double* b,
                const double* a, const double* c, uint64_t seed,
                uint64_t noise_iteration, double* cum_per_step, int* link_final,
                double* pos_final, int* states_link, double* states_pos,
                double* wall) {
  return guarded([&] {
    const auto& s = static_cast<RefScn*>(h)->s;
    const int L = s.net.n_links();
    const int N = s.n_agents();
    ForwardOptions opt;
    opt.noise_iteration = noise_iteration;
    opt.record_states = states_link != nullptr;
    const Trajectory tr =
        simulate_forward(s, make_params(L, u, k, b, a, c), RngStream(seed), opt);
    for (int t = 0; t < tr.steps; ++t)
      std::memcpy(cum_per_step + static_cast<std::size_t>(t) * L,
                  tr.cum_per_step[t].data(), L * 8);
    compact(tr.X_final, N, L, s.cfg.sentinel, link_final, pos_final);
    if (states_link)
      for (int t = 0; t < tr.steps; ++t)
        compact(tr.states[t], N, L, s.cfg.sentinel,
                states_link + static_cast<std::size_t>(t) * N,
                states_pos + static_cast<std::size_t>(t) * N);
    if (wall) *wall = tr.wall_seconds;
  });
}

/// simulate_gradient (src/engine.cpp:303-429) with a linear+quadratic loss
///   loss = sum_k sum_j (ws[k,j] s_kj + 0.5 qs[k,j] s_kj^2)
///        + sum_j (wc[j] c_j + 0.5 qc[j] c_j^2) + sum_n wx[n] X_final[n, link_n]
/// over the snapshot leaves s_k, cum_final c and the valid cells of X_final,
/// built from reference tape ops (it is a LossBuilder like any caller's).
/// Any of ws/qs/wc/qc/wx may be null.  mode: 0 FullTape, 1 Checkpointed.
/// grads: 5 x L (u, kappa, beta, alpha, cost).  snaps: n_snap x L.
int ref_gradient(void* h, const double* u, const double* k, const double* b,
                 const double* a, const double* c, uint64_t seed,
                 uint64_t noise_iteration, int mode, const double* ws,
                 const double* qs, const double* wc, const double* qc,
                 const double* wx, double* loss, double* grads, double* snaps,
                 int* n_snaps, double* cum_final, int* link_final,
                 double* pos_final, double* wall) {
  return guarded([&] {
    const auto& s = static_cast<RefScn*>(h)->s;
    const int L = s.net.n_links();
    const int N = s.n_agents();
    const double M = s.cfg.sentinel;
    LossBuilder builder = [=](Tape&, const LossInputs& li) -> Tensor {
      Tensor acc = Tensor::zeros({1, 1});
      const int K = static_cast<int>(li.snapshots.size());
      for (int kk = 0; kk < K; ++kk) {
        const Tensor& sk = li.snapshots[kk];
        if (ws)
          acc = add(acc, reduce_sum(mul(sk, Tensor::from(std::vector<double>(
                                                 ws + kk * L, ws + kk * L + L),
                                                 {L, 1})),
                                    kAxisAll));
        if (qs)
          acc = add(acc,
                    reduce_sum(mul(mul(sk, sk),
                                   scale(Tensor::from(std::vector<double>(
                                                          qs + kk * L,
                                                          qs + kk * L + L),
                                                      {L, 1}),
                                         0.5)),
                               kAxisAll));
      }
      if (wc)
        acc = add(acc, reduce_sum(mul(li.cum_final,
                                      Tensor::from(std::vector<double>(wc, wc + L),
                                                   {L, 1})),
                                  kAxisAll));
      if (qc)
        acc = add(acc,
                  reduce_sum(mul(mul(li.cum_final, li.cum_final),
                                 scale(Tensor::from(
                                           std::vector<double>(qc, qc + L), {L, 1}),
                                       0.5)),
                             kAxisAll));
      if (wx) {
        const auto& xv = li.X_final.vals();
        std::vector<int> idx;
        std::vector<double> w;
        for (int i = 0; i < N; ++i)
          for (int j = 0; j < L; ++j)
            if (xv[static_cast<std::size_t>(i) * L + j] != -M) {
              idx.push_back(i * L + j);
              w.push_back(wx[i]);
              break;
            }
        if (!idx.empty()) {
          const int m = static_cast<int>(idx.size());
          acc = add(acc, reduce_sum(mul(gather(li.X_final, idx),
                                        Tensor::from(std::move(w), {m, 1})),
                                    kAxisAll));
        }
      }
      return acc;
    };
    ForwardOptions opt;
    opt.noise_iteration = noise_iteration;
    const GradResult g = simulate_gradient(
        s, make_params(L, u, k, b, a, c), RngStream(seed), builder,
        mode == 0 ? GradMode::FullTape : GradMode::Checkpointed, opt);
    *loss = g.loss;
    std::memcpy(grads + 0 * L, g.grads.u.data(), L * 8);
    std::memcpy(grads + 1 * L, g.grads.kappa.data(), L * 8);
    std::memcpy(grads + 2 * L, g.grads.beta.data(), L * 8);
    std::memcpy(grads + 3 * L, g.grads.alpha.data(), L * 8);
    std::memcpy(grads + 4 * L, g.grads.cost.data(), L * 8);
    if (n_snaps) *n_snaps = static_cast<int>(g.snapshot_values.size());
    if (snaps)
      for (std::size_t kk = 0; kk < g.snapshot_values.size(); ++kk)
        std::memcpy(snaps + kk * L, g.snapshot_values[kk].data(), L * 8);
    if (cum_final) std::memcpy(cum_final, g.cum_final_values.data(), L * 8);
    if (link_final) compact(g.X_final_values, N, L, M, link_final, pos_final);
    if (wall) *wall = g.wall_seconds;
  });
}

/// Calibration loss: the reference's own mse_loss_builder
/// (src/optimization.cpp:84-101) over observed links `obs_ids` (n_obs) and
/// observations obs_vals (K x n_obs).
int ref_gradient_mse(void* h, const double* u, const double* k,
                     const double* b, const double* a, const double* c,
                     uint64_t seed, uint64_t noise_iteration, int n_obs,
                     const int* obs_ids, int K, const double* obs_vals,
                     double* loss, double* grads) {
  return guarded([&] {
    const auto& s = static_cast<RefScn*>(h)->s;
    const int L = s.net.n_links();
    CountSeries obs;
    obs.link_ids.assign(obs_ids, obs_ids + n_obs);
    obs.interval_s = s.obs_interval_s;
    for (int kk = 0; kk < K; ++kk)
      obs.values.emplace_back(obs_vals + kk * n_obs, obs_vals + (kk + 1) * n_obs);
    ForwardOptions opt;
    opt.noise_iteration = noise_iteration;
    const GradResult g = simulate_gradient(
        s, make_params(L, u, k, b, a, c), RngStream(seed),
        mse_loss_builder(obs, s.cfg.delta_n), GradMode::Checkpointed, opt);
    *loss = g.loss;
    std::memcpy(grads + 0 * L, g.grads.u.data(), L * 8);
    std::memcpy(grads + 1 * L, g.grads.kappa.data(), L * 8);
    std::memcpy(grads + 2 * L, g.grads.beta.data(), L * 8);
    std::memcpy(grads + 3 * L, g.grads.alpha.data(), L * 8);
    std::memcpy(grads + 4 * L, g.grads.cost.data(), L * 8);
  });
}

// ---- optimisation loops (src/optimization.cpp:122-295) ---------------------
// opt = {lr, weight_decay, beta1, beta2, eps}; iopt = {patience,
// max_iterations, resample_noise, noise_draws}; bounds = ParamRanges fields in
// declaration order.  Returns 3 on DivergenceError.
static OptimizeConfig make_opt(const double* opt, const int* iopt) {
  OptimizeConfig o;
  o.adam.lr = opt[0];
  o.adam.weight_decay = opt[1];
  o.adam.beta1 = opt[2];
  o.adam.beta2 = opt[3];
  o.adam.eps = opt[4];
  o.patience = iopt[0];
  o.max_iterations = iopt[1];
  o.resample_noise = iopt[2] != 0;
  o.noise_draws = iopt[3];
  o.grad_mode = GradMode::Checkpointed;
  return o;
}

int ref_calibrate(void* h, int n_obs, const int* obs_ids, int K,
                  const double* obs_vals, const double* bounds,
                  const double* opt, const int* iopt, uint64_t seed,
                  const double* iu, const double* ik, const double* ib,
                  const double* ia, const double* ic, double* best /* 5L */,
                  double* best_loss, int* best_it, int* iterations,
                  double* curve) {
  try {
    const auto& s = static_cast<RefScn*>(h)->s;
    const int L = s.net.n_links();
    CountSeries obs;
    obs.link_ids.assign(obs_ids, obs_ids + n_obs);
    obs.interval_s = s.obs_interval_s;
    for (int kk = 0; kk < K; ++kk)
      obs.values.emplace_back(obs_vals + kk * n_obs, obs_vals + (kk + 1) * n_obs);
    ParamRanges r;
    r.u_lo = bounds[0];
    r.u_hi = bounds[1];
    r.kappa_lo = bounds[2];
    r.kappa_hi = bounds[3];
    r.beta_lo = bounds[4];
    r.beta_hi = bounds[5];
    r.alpha_lo = bounds[6];
    r.alpha_hi = bounds[7];
    LinkParams init;
    const bool have = iu != nullptr;
    if (have) {
      init.u.assign(iu, iu + L);
      init.kappa.assign(ik, ik + L);
      init.beta.assign(ib, ib + L);
      init.alpha.assign(ia, ia + L);
      if (ic) init.cost.assign(ic, ic + L);
    }
    const CalibrationResult res = calibrate(s, obs, r, make_opt(opt, iopt),
                                            RngStream(seed), have ? &init : nullptr);
    const auto& bp = res.best_params;
    if (!bp.u.empty()) {
      std::memcpy(best + 0 * L, bp.u.data(), L * 8);
      std::memcpy(best + 1 * L, bp.kappa.data(), L * 8);
      std::memcpy(best + 2 * L, bp.beta.data(), L * 8);
      std::memcpy(best + 3 * L, bp.alpha.data(), L * 8);
      std::memcpy(best + 4 * L, bp.cost.data(), L * 8);
    }
    *best_loss = res.best_loss;
    *best_it = res.best_iteration;
    *iterations = res.iterations;
    std::copy(res.loss_curve.begin(), res.loss_curve.end(), curve);
    return 0;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_optimize_control(void* h, const double* u, const double* k,
                         const double* b, const double* a, const double* c,
                         int target, double desired, const double* opt,
                         const int* iopt, double cost_floor, uint64_t seed,
                         double* cost_out, double* out3 /* achieved, gap, best_loss */,
                         int* iterations, int* stall, double* curve) {
  try {
    const auto& s = static_cast<RefScn*>(h)->s;
    const int L = s.net.n_links();
    ControlConfig cc;
    cc.opt = make_opt(opt, iopt);
    cc.cost_floor = cost_floor;
    const ControlResult res = optimize_control(
        s, make_params(L, u, k, b, a, c), target, desired, cc, RngStream(seed));
    if (!res.cost.empty()) std::memcpy(cost_out, res.cost.data(), L * 8);
    out3[0] = res.achieved;
    out3[1] = res.gap_fraction;
    out3[2] = res.best_loss;
    *iterations = res.iterations;
    *stall = res.zero_gradient_stall ? 1 : 0;
    std::copy(res.loss_curve.begin(), res.loss_curve.end(), curve);
    return 0;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ---- observation / output side (observation.cpp:46-83, optimization.cpp:297-336,
// pipeline.cpp:113-160) ---------------------------------------------------------
static CountSeries ref_series(int k, int n, const int* ids, const double* vals, int interval_s) {
  CountSeries s;
  s.link_ids.assign(ids, ids + n);
  s.interval_s = interval_s;
  for (int q = 0; q < k; ++q) s.values.emplace_back(vals + q * n, vals + (q + 1) * n);
  return s;
}

int ref_synthesize_observations(int k, int n, const int* ids, const double* vals, int interval_s,
                                double noise_frac, double coverage, uint64_t seed, int* m_out,
                                int* obs_ids, double* obs_vals) {
  return guarded([&] {
    const auto r = synthesize_observations(ref_series(k, n, ids, vals, interval_s), noise_frac, coverage,
                                           RngStream(seed));
    const int m = static_cast<int>(r.second.size());
    *m_out = m;
    std::copy(r.second.begin(), r.second.end(), obs_ids);
    for (int q = 0; q < k; ++q) std::copy(r.first.values[q].begin(), r.first.values[q].end(), obs_vals + q * m);
  });
}

int ref_count_metrics(int ks, int ns, const int* sid, const double* sv, int kt, int nt, const int* tid,
                      const double* tv, double* out3, int* n_pairs) {
  return guarded([&] {
    const Metrics m = count_metrics(ref_series(ks, ns, sid, sv, 1), ref_series(kt, nt, tid, tv, 1));
    out3[0] = m.mae;
    out3[1] = m.pearson_r;
    out3[2] = m.r_defined ? 1.0 : 0.0;
    *n_pairs = m.n_pairs;
  });
}

// CSV text of a series into buf (cap bytes incl. NUL); returns the length.
long ref_series_to_csv(int k, int n, const int* ids, const double* vals, int interval_s, char* buf,
                       long cap) {
  std::string s;
  if (guarded([&] { s = series_to_csv(ref_series(k, n, ids, vals, interval_s)); })) return -1;
  if (buf && cap > static_cast<long>(s.size())) std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<long>(s.size());
}

// ---- FD-validation instrumentation ---------------------
// soft_choices (car_following.hpp:37), SurrogateTrace record/replay
// (car_following.hpp:23-29, car_following.cpp:17-94), BranchTrace
// (branch_trace.hpp) and run_gradcheck (pipeline.cpp:499-603), all through the
// reference's own entry points.  States are compacted by the VALID rule
// (x >= kValidThreshold; surrogate replay leaves -(M + d) in vacated cells,
// so the != -M rule of compact() does not apply); link -1 = no valid cell.
namespace {
void compact_valid(const std::vector<double>& X, int N, int L, int* link, double* pos) {
  for (int i = 0; i < N; ++i) {
    link[i] = -1;
    pos[i] = 0.0;
    for (int j = 0; j < L; ++j) {
      const double x = X[static_cast<std::size_t>(i) * L + j];
      if (x >= kValidThreshold) {
        link[i] = j;
        pos[i] = x;
        break;
      }
    }
  }
}
}  // namespace

void ref_scenario_set_soft(void* h, int soft) {
  static_cast<RefScn*>(h)->s.cfg.soft_choices = soft != 0;
}
void* ref_surrogate_new() { return new SurrogateTrace; }
void ref_surrogate_free(void* t) { delete static_cast<SurrogateTrace*>(t); }
void ref_surrogate_set_replay(void* t, int replay) {
  static_cast<SurrogateTrace*>(t)->replay = replay != 0;
}
void ref_surrogate_rewind(void* t) { static_cast<SurrogateTrace*>(t)->rewind(); }
/// sizes[0..3] = #graft records, #carrier records, #pick records, total doubles.
void ref_surrogate_sizes(void* t, long* sizes) {
  const auto* tr = static_cast<SurrogateTrace*>(t);
  long nd = 0;
  for (const auto& v : tr->graft_new) nd += static_cast<long>(v.size());
  for (const auto& v : tr->graft_old) nd += static_cast<long>(v.size());
  for (const auto& v : tr->carriers) nd += static_cast<long>(v.size());
  sizes[0] = static_cast<long>(tr->graft_new.size());
  sizes[1] = static_cast<long>(tr->carriers.size());
  sizes[2] = static_cast<long>(tr->picks.size());
  sizes[3] = nd;
}

/// simulate_forward with the instrumentation options: surrogate (may be
/// null), ForwardOptions.trace_branches; returns Trajectory.branch_hash.
int ref_forward_traced(void* h, const double* u, const double* k, const double* b,
                       const double* a, const double* c, uint64_t seed,
                       uint64_t noise_iteration, void* surrogate, int trace_branches,
                       double* cum_per_step, int* link_final, double* pos_final,
                       uint64_t* hash) {
  return guarded([&] {
    Scenario s = static_cast<RefScn*>(h)->s;
    s.cfg.surrogate = static_cast<SurrogateTrace*>(surrogate);
    const int L = s.net.n_links();
    const int N = s.n_agents();
    ForwardOptions opt;
    opt.noise_iteration = noise_iteration;
    opt.trace_branches = trace_branches != 0;
    const Trajectory tr =
        simulate_forward(s, make_params(L, u, k, b, a, c), RngStream(seed), opt);
    if (cum_per_step)
      for (int t = 0; t < tr.steps; ++t)
        std::memcpy(cum_per_step + static_cast<std::size_t>(t) * L,
                    tr.cum_per_step[t].data(), L * 8);
    if (link_final) compact_valid(tr.X_final, N, L, link_final, pos_final);
    if (hash) *hash = tr.branch_hash;
  });
}

/// simulate_gradient of sum(cum_final) (run_gradcheck's loss,
/// pipeline.cpp:522-524) with the instrumentation options.
int ref_gradient_traced(void* h, const double* u, const double* k, const double* b,
                        const double* a, const double* c, uint64_t seed,
                        uint64_t noise_iteration, int mode, void* surrogate,
                        int trace_branches, double* loss, double* grads,
                        double* cum_final, uint64_t* hash) {
  return guarded([&] {
    Scenario s = static_cast<RefScn*>(h)->s;
    s.cfg.surrogate = static_cast<SurrogateTrace*>(surrogate);
    const int L = s.net.n_links();
    const LossBuilder builder = [](Tape&, const LossInputs& li) -> Tensor {
      return reduce_sum(li.cum_final, kAxisAll);
    };
    ForwardOptions opt;
    opt.noise_iteration = noise_iteration;
    opt.trace_branches = trace_branches != 0;
    const GradResult g = simulate_gradient(
        s, make_params(L, u, k, b, a, c), RngStream(seed), builder,
        mode == 0 ? GradMode::FullTape : GradMode::Checkpointed, opt);
    if (loss) *loss = g.loss;
    std::memcpy(grads + 0 * L, g.grads.u.data(), L * 8);
    std::memcpy(grads + 1 * L, g.grads.kappa.data(), L * 8);
    std::memcpy(grads + 2 * L, g.grads.beta.data(), L * 8);
    std::memcpy(grads + 3 * L, g.grads.alpha.data(), L * 8);
    std::memcpy(grads + 4 * L, g.grads.cost.data(), L * 8);
    if (cum_final) std::memcpy(cum_final, g.cum_final_values.data(), L * 8);
    if (hash) *hash = g.branch_hash;
  });
}

/// run_gradcheck (pipeline.cpp:499-585).  per_draw_max has room for `draws`.
/// Returns 0 also when the report does not pass (pass = 0); 1 on exceptions.
int ref_run_gradcheck(int draws, int steps, int agents, double tol, uint64_t seed,
                      double* max_rel_err, int* redraws, int* pass,
                      double* per_draw_max) {
  return guarded([&] {
    const GradcheckReport r = run_gradcheck(draws, steps, agents, tol, seed);
    *max_rel_err = r.max_rel_err;
    *redraws = r.redraws;
    *pass = r.pass ? 1 : 0;
    for (std::size_t i = 0; i < r.per_draw_max.size(); ++i) per_draw_max[i] = r.per_draw_max[i];
  });
}

}  // extern "C"
