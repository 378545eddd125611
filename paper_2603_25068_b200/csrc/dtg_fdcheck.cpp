// FD-validation host layer over the device probe engine
// (dtg_probe.cu):
//   * the instrumented simulate_forward / simulate_gradient modes —
//     ForwardOptions::trace_branches, SimConfig::soft_choices,
//     SimConfig::surrogate (engine.cpp:227-254, 303-429; car_following.cpp:17-94);
//   * probe_forward_batch: many parameter sets in one launch;
//   * run_gradcheck (pipeline.cpp:486-585) on top of both.
//
// TRANSCRIBED HOST CODE: run_gradcheck restates pipeline.cpp:499-585 (its draw
// / redraw / stencil logic and report), restructured so each draw's 10 L
// stencil probes run as ONE batched device launch; the probe engine itself
// (dtg_probe.cu) is new device code.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dtg_engine.hpp"
#include "dtg_fdcheck.h"
#include "dtg_probe.h"

namespace dtg {

namespace {

ProbeNet probe_net(const Network& net) {
  ProbeNet pn;
  pn.L = net.n_links();
  pn.succ_off = net.succ_off;
  pn.succ = net.succ;
  pn.len = net.lengths();
  if (static_cast<int>(pn.succ_off.size()) != pn.L + 1)
    throw std::runtime_error("network CSR is stale (call rebuild_csr)");
  return pn;
}

ProbeCfg probe_cfg(const SimConfig& c) {
  ProbeCfg pc;
  pc.delta_n = c.delta_n;
  pc.tau = c.tau;
  pc.M = c.sentinel;
  pc.gumbel_tau = c.gumbel_tau;
  pc.tg = c.trajectory_grafting;
  pc.soft = c.soft_choices;
  return pc;
}

void check_params(const LinkParams& p, int L) {
  for (const auto* v : {&p.u, &p.kappa, &p.beta, &p.alpha, &p.cost})
    if (static_cast<int>(v->size()) != L)
      throw std::runtime_error("parameter vectors must have one entry per link");
}

int surrogate_mode(const Scenario& s) {
  if (!s.cfg.surrogate) return 0;
  if (!s.cfg.surrogate->replay) return 1;
  if (!s.cfg.soft_choices)
    throw UnsupportedError(
        "surrogate replay on the device needs soft_choices (the straight-through choice graft "
        "of a replay makes choice rows fractional)");
  if (!s.cfg.surrogate->rec || !s.cfg.surrogate->rec->recorded)
    throw std::runtime_error("surrogate trace misaligned: graft count (nothing recorded)");
  return 2;
}

/// Flags -> the reference's error class: a replay that leaves the recorded
/// control path is the reference's trace_fail (runtime_error); anything else
/// is outside the device contract.
void raise_flags(int f) {
  const int hard = f & ~kProbeOffPath;
  if (hard) throw UnsupportedError(ProbeEngine::describe(hard));
  if (f & kProbeOffPath) throw std::runtime_error(ProbeEngine::describe(f));
}

struct Run {
  std::unique_ptr<ProbeEngine> eng;
  int T = 0;
};

Run run_probes(const Scenario& s, const std::vector<LinkParams>& params, const RngStream& rng,
               std::uint64_t noise_iteration, bool trace, bool keep_cum, int sur_mode) {
  const int L = s.net.n_links();
  const int P = static_cast<int>(params.size());
  if (P < 1) throw std::runtime_error("no probes");
  std::vector<double> flat(static_cast<std::size_t>(P) * 5 * L);
  for (int p = 0; p < P; ++p) {
    check_params(params[p], L);
    double* d = flat.data() + static_cast<std::size_t>(p) * 5 * L;
    std::copy(params[p].u.begin(), params[p].u.end(), d);
    std::copy(params[p].kappa.begin(), params[p].kappa.end(), d + L);
    std::copy(params[p].beta.begin(), params[p].beta.end(), d + 2 * L);
    std::copy(params[p].alpha.begin(), params[p].alpha.end(), d + 3 * L);
    std::copy(params[p].cost.begin(), params[p].cost.end(), d + 4 * L);
  }
  const InitialState init = seed_agents(s);
  Run r;
  r.T = s.horizon_steps;
  r.eng = std::make_unique<ProbeEngine>(probe_net(s.net), probe_cfg(s.cfg),
                                        static_cast<int>(init.link.size()), P);
  r.eng->set_state(init.link.data(), init.pos.data());
  r.eng->set_params(flat.data());
  const std::vector<std::uint64_t> its(P, noise_iteration);
  r.eng->set_noise(rng.seed(), its.data());
  ProbeTrace* tr = nullptr;
  if (sur_mode) {
    auto& rec = s.cfg.surrogate->rec;
    if (!rec) rec = std::make_shared<ProbeTrace>();
    tr = rec.get();
  }
  r.eng->run(r.T, sur_mode, tr, trace, keep_cum);
  return r;
}

}  // namespace

namespace detail {

bool instrumented(const Scenario& s, const ForwardOptions& opt) {
  return opt.trace_branches || s.cfg.soft_choices || s.cfg.surrogate != nullptr;
}

Trajectory forward_instrumented(const Scenario& s, const LinkParams& params, const RngStream& rng,
                                const ForwardOptions& opt) {
  if (opt.record_states)
    throw UnsupportedError("record_states with trace_branches / soft_choices / surrogate");
  const auto t0 = std::chrono::steady_clock::now();
  const int sur = surrogate_mode(s);
  Run r = run_probes(s, {params}, rng, opt.noise_iteration, opt.trace_branches, true, sur);
  raise_flags(r.eng->flags()[0]);
  const int L = s.net.n_links(), N = s.n_agents();
  Trajectory tr;
  tr.steps = r.T;
  const std::vector<double> cum = r.eng->cum_per_step(0);
  for (int t = 0; t < r.T; ++t)
    tr.cum_per_step.emplace_back(cum.begin() + static_cast<std::size_t>(t) * L,
                                 cum.begin() + static_cast<std::size_t>(t + 1) * L);
  tr.final_state.link.resize(N);
  tr.final_state.pos.resize(N);
  r.eng->final_state(0, tr.final_state.link.data(), tr.final_state.pos.data());
  tr.cum_final = r.T ? tr.cum_per_step.back() : std::vector<double>(L, 0.0);
  if (opt.trace_branches) tr.branch_hash = r.eng->hashes()[0];
  tr.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return tr;
}

std::uint64_t gradient_instrumentation(const Scenario& s, const LinkParams& params,
                                       const RngStream& rng, const ForwardOptions& opt,
                                       const std::vector<double>& cum_final) {
  const int sur = surrogate_mode(s);
  if (sur == 2)
    throw UnsupportedError("the gradient of a replaying surrogate is not on the device path");
  Run r = run_probes(s, {params}, rng, opt.noise_iteration, opt.trace_branches, false, sur);
  raise_flags(r.eng->flags()[0]);
  // the instrumented forward and the gradient's forward are the same program
  if (r.eng->cum_final_all() != cum_final)
    throw std::runtime_error("internal: instrumented forward disagrees with the gradient forward");
  const std::uint64_t offset = 0xcbf29ce484222325ULL;
  return opt.trace_branches ? r.eng->hashes()[0] : offset;
}

}  // namespace detail

std::vector<ProbeResult> probe_forward_batch(const Scenario& s,
                                             const std::vector<LinkParams>& params,
                                             const RngStream& rng, std::uint64_t noise_iteration,
                                             bool trace_branches) {
  const int sur = surrogate_mode(s);
  Run r = run_probes(s, params, rng, noise_iteration, trace_branches, false, sur);
  const int L = s.net.n_links(), P = static_cast<int>(params.size());
  const std::vector<double> cf = r.eng->cum_final_all();
  const std::vector<std::uint64_t> hs = r.eng->hashes();
  const std::vector<int> fl = r.eng->flags();
  std::vector<ProbeResult> out(P);
  for (int p = 0; p < P; ++p) {
    if (fl[p] & ~kProbeOffPath) throw UnsupportedError(ProbeEngine::describe(fl[p]));
    ProbeResult& o = out[p];
    o.cum_final.assign(cf.begin() + static_cast<std::size_t>(p) * L,
                       cf.begin() + static_cast<std::size_t>(p + 1) * L);
    double sum = 0.0;
    for (double v : o.cum_final) sum += v;
    o.cum_sum = sum;
    o.branch_hash = trace_branches ? hs[p] : 0xcbf29ce484222325ULL;
    o.on_path = !(fl[p] & kProbeOffPath);
  }
  return out;
}

namespace {

/// make_chain_network (pipeline.cpp:486-496): virtual inflow -> n physical
/// links in a row -> virtual outflow.
Network chain_network(int n_physical, double link_len, double inflow_len) {
  std::vector<Link> links;
  auto push = [&](int a, int b, double len, LinkKind k) {
    Link l;
    l.id = 0;
    l.from_node = a;
    l.to_node = b;
    l.length = len;
    l.kind = k;
    links.push_back(l);
  };
  push(n_physical + 1, 0, inflow_len, LinkKind::VirtualInflow);
  for (int i = 0; i < n_physical; ++i) push(i, i + 1, link_len, LinkKind::Physical);
  push(n_physical, n_physical + 2, inflow_len, LinkKind::VirtualOutflow);
  return make_network(n_physical + 3, std::move(links));
}

}  // namespace

GradcheckReport run_gradcheck(int draws, int steps, int agents, double tol, std::uint64_t seed) {
  const Network net = chain_network(3, 300.0, 100.0);
  const int L = net.n_links();
  Scenario sc;
  sc.net = net;
  sc.cfg.delta_n = 1;
  sc.cfg.soft_choices = true;
  sc.n_vehicles = agents;
  sc.horizon_steps = steps;
  sc.obs_interval_s = steps;  // one snapshot at the end
  const LossBuilder builder = linear_quadratic_loss({}, {}, std::vector<double>(L, 1.0), {}, {});

  GradcheckReport rep;
  rep.draws = draws;
  const ParamRanges r;
  std::uint64_t attempt = 0;
  for (int d = 0; d < draws; ++d) {
    bool clean = false;
    double draw_max = 0.0;
    for (int tries = 0; tries < 60 && !clean; ++tries, ++rep.redraws) {
      const RngStream pr = RngStream(seed).fork(9000 + attempt++);
      LinkParams p;
      for (int l = 0; l < L; ++l) {
        p.u.push_back(pr.uniform_in(r.u_lo, r.u_hi, 0, l));
        p.kappa.push_back(pr.uniform_in(r.kappa_lo, r.kappa_hi, 1, l));
        p.beta.push_back(pr.uniform_in(r.beta_lo, r.beta_hi, 2, l));
        p.alpha.push_back(pr.uniform_in(r.alpha_lo, r.alpha_hi, 3, l));
        p.cost.push_back(pr.uniform_in(0.5, 2.0, 4, l));
      }
      // base run: adjoint gradient + recorded surrogate + branch signature
      SurrogateTrace trace;
      sc.cfg.surrogate = &trace;
      ForwardOptions opt;
      opt.trace_branches = true;
      const GradResult g = simulate_gradient(sc, p, RngStream(seed), builder, GradMode::FullTape, opt);
      const std::uint64_t base_hash = g.branch_hash;

      // all central-difference probes of this draw in one launch
      trace.replay = true;
      const std::vector<double>* grads[5] = {&g.grads.u, &g.grads.kappa, &g.grads.beta,
                                             &g.grads.alpha, &g.grads.cost};
      std::vector<LinkParams> probes;
      std::vector<double> step;
      probes.reserve(10 * L);
      for (int b = 0; b < 5; ++b)
        for (int l = 0; l < L; ++l) {
          std::vector<double> LinkParams::*blk[5] = {&LinkParams::u, &LinkParams::kappa,
                                                     &LinkParams::beta, &LinkParams::alpha,
                                                     &LinkParams::cost};
          const double x0 = (p.*blk[b])[l];
          const double h = 1e-5 * std::max(1.0, std::abs(x0));
          step.push_back(h);
          LinkParams pp = p;
          (pp.*blk[b])[l] = x0 + h;
          probes.push_back(pp);
          (pp.*blk[b])[l] = x0 - h;
          probes.push_back(std::move(pp));
        }
      const std::vector<ProbeResult> res = probe_forward_batch(sc, probes, RngStream(seed), 0, true);
      sc.cfg.surrogate = nullptr;

      // the reference's sequential acceptance and error bookkeeping
      clean = true;
      draw_max = 0.0;
      for (int b = 0; b < 5 && clean; ++b)
        for (int l = 0; l < L && clean; ++l) {
          const int k = b * L + l;
          const ProbeResult& plus = res[2 * k];
          const ProbeResult& minus = res[2 * k + 1];
          const bool ok1 = plus.on_path && plus.branch_hash == base_hash;
          const bool ok2 = minus.on_path && minus.branch_hash == base_hash;
          if (!ok1 || !ok2) {
            clean = false;  // branch flip inside the stencil: redraw
            break;
          }
          const double fd = (plus.cum_sum - minus.cum_sum) / (2.0 * step[k]);
          const double ad = (*grads[b])[l];
          const double abs_err = std::abs(ad - fd);
          if (abs_err < 1e-6) continue;  // below the probe noise floor
          draw_max = std::max(draw_max, abs_err / std::max(std::abs(ad), std::abs(fd)));
        }
    }
    if (!clean) throw std::runtime_error("gradcheck: could not find a kink-free parameter draw");
    rep.per_draw_max.push_back(draw_max);
    rep.max_rel_err = std::max(rep.max_rel_err, draw_max);
  }
  rep.pass = rep.max_rel_err < tol;
  return rep;
}

}  // namespace dtg
