// FD-validation engine: the reference's instrumented
// forward modes on the device.
//
//   * soft_choices    car_following.hpp:37, node_model.cpp:21 — the relaxed
//                     choice tensors are kept instead of the straight-through
//                     one-hot.
//   * SurrogateTrace  car_following.hpp:23-29, car_following.cpp:17-94 — a
//                     recording run stores every graft / carrier value and
//                     min / relu branch pick; a replay run re-evaluates the
//                     program with those discontinuities frozen (the smooth
//                     surrogate whose derivative the adjoint computes).
//   * BranchTrace     branch_trace.hpp — FNV-1a hash of every discrete
//                     decision (validity masks, sort orders, branch picks,
//                     sampled argmaxes) in the reference's note order.
//
// One CTA per probe (an independent parameter set / noise draw); all FD
// stencil probes of a gradient check run as one launch.  The per-agent state
// is the compact (link, position) form; the relaxed modes are exact on it as
// long as every choice value stays in {0, 1} — true whenever each arrived
// agent has at most one vacant successor with choice probability 1 and each
// link sees at most one candidate per step (chains such as run_gradcheck's,
// pipeline.cpp:486-496).  A fractional choice (which would make the state
// dense) is detected on the device and reported as unsupported, never
// silently approximated.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace dtg {

// device flag bits of a probe run
constexpr int kProbeFractional = 1;    // a relaxed choice left {0, 1}
constexpr int kProbeZeroAlpha = 2;     // merge candidate with zero priority
constexpr int kProbeCandOverflow = 4;  // > kProbeMaxCand candidates on a link
constexpr int kProbeDegOverflow = 8;   // out-degree above kMaxDeg
constexpr int kProbeOffPath = 16;      // replay left the recorded control path
constexpr int kProbeMaxCand = 32;

struct ProbeNet {
  int L = 0;
  std::vector<int> succ_off, succ;
  std::vector<double> len;
};

struct ProbeCfg {
  int delta_n = 1;
  double tau = 1.0, M = 99999.0, gumbel_tau = 0.01;
  bool tg = true, soft = false;
};

/// Device copy of one recording run (the SurrogateTrace payload), keyed by
/// (step, agent) and (step, link) instead of by call order; on the recorded
/// control path both give the same values, and leaving the path is flagged.
struct ProbeTrace {
  int T = 0, N = 0, L = 0;
  bool recorded = false;
  void* dev = nullptr;  // owned device block (see dtg_probe.cu)
  ProbeTrace() = default;
  ProbeTrace(const ProbeTrace&) = delete;
  ProbeTrace& operator=(const ProbeTrace&) = delete;
  ~ProbeTrace();
  void reserve(int T, int N, int L);
};

class ProbeEngine {
 public:
  ProbeEngine(const ProbeNet& net, const ProbeCfg& cfg, int n_agents, int n_probes);
  ~ProbeEngine();
  ProbeEngine(const ProbeEngine&) = delete;
  ProbeEngine& operator=(const ProbeEngine&) = delete;

  int n_probes() const { return P_; }
  /// Shared initial compact state (every agent on a link, pos >= -0.01).
  void set_state(const int* link, const double* pos);
  /// params: [P][5][L] (u, kappa, beta, alpha, cost per probe).
  void set_params(const double* params);
  /// Per-probe simulation streams root.fork(7).fork(noise_iteration[p]).
  void set_noise(std::uint64_t root_seed, const std::uint64_t* noise_iterations);
  /// Run T steps of every probe.  sur_mode: 0 none, 1 record (probe 0 writes
  /// `tr`), 2 replay from `tr`.  trace: compute the BranchTrace hash.
  /// keep_cum: keep every step's cum (read with cum_per_step).
  void run(int T, int sur_mode, ProbeTrace* tr, bool trace, bool keep_cum);

  std::vector<double> cum_per_step(int p) const;  // [T][L]
  std::vector<double> cum_final_all() const;      // [P][L]
  void final_state(int p, int* link, double* pos) const;
  std::vector<std::uint64_t> hashes() const;
  std::vector<int> flags() const;
  /// Human-readable description of the flag bits.
  static std::string describe(int flags);

 private:
  struct Impl;
  Impl* d_;
  int L_, N_, P_, T_ = 0;
};

}  // namespace dtg
