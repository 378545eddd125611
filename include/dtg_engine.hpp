// dtg C++ host API — the reference's simulator surface for the hot path
// (/root/reference/proj/include/dtsim/{network,engine,observation}.hpp),
// re-implemented B200-first: the network is a CSR (not a dense L x L
// adjacency), states are compact (link, position) per agent (not dense N x L),
// and simulate_forward / simulate_gradient run on the GPU through the C-ABI in
// include/dtg.h.  Names, argument meaning and error behaviour follow the
// reference so callers (calibrate, optimize_control, the pipeline commands)
// port by renaming the namespace; see INTEGRATION.md.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../paper_2603_25068_b200/csrc/dtg_rng.h"

namespace dtg {

// ---- network (network.hpp:11-51) ------------------------------------------------
enum class LinkKind { Physical = 0, VirtualInflow = 1, VirtualOutflow = 2 };

struct Link {
  int id = -1;
  int from_node = -1;
  int to_node = -1;
  double length = 0.0;  // meters
  LinkKind kind = LinkKind::Physical;
};

struct LinkParams {
  std::vector<double> u, kappa, beta, alpha, cost;
};

struct ParamRanges {
  double u_lo = 13.9, u_hi = 22.2;
  double kappa_lo = 0.18, kappa_hi = 0.22;
  double beta_lo = 0.0, beta_hi = 5.0;
  double alpha_lo = 0.01, alpha_hi = 5.0;
};

struct Network {
  int n_nodes = 0;
  int n_physical_nodes = 0;
  std::vector<Link> links;
  // successor CSR replacing the dense adjacency (network.cpp:28-35):
  // j follows i iff i != j and to_node(i) == from_node(j); ascending j.
  std::vector<int> succ_off, succ;

  int n_links() const { return static_cast<int>(links.size()); }
  int n_physical_links() const;
  std::vector<int> links_of_kind(LinkKind k) const;
  std::vector<double> lengths() const;
  void rebuild_csr();
};

Network make_network(int n_nodes, std::vector<Link> links);
Network parse_tntp_text(const std::string& text, double length_unit_scale);
Network attach_virtual_links(const Network& physical, const RngStream& rng,
                             double virtual_length);
bool all_physical_reachable(const Network& net);
LinkParams sample_parameters(const Network& net, const ParamRanges& ranges,
                             const RngStream& rng, bool mean_mode = false);
/// Synthetic n x n grid of SURVEY.md §8d (physical links only).
Network grid_network(int n, double length);

// ---- scenario (engine.hpp:16-53, car_following.hpp:31-40) ------------------------
struct SimConfig {
  int delta_n = 1;
  double tau = 1.0;
  double sentinel = 99999.0;
  double gumbel_tau = 0.01;
  bool trajectory_grafting = true;
  bool soft_choices = false;  // relaxed surrogate: not on the device path
  double dt() const { return tau * delta_n; }
};

struct Scenario {
  Network net;
  SimConfig cfg;
  int n_vehicles = 0;
  int horizon_steps = 0;
  int obs_interval_s = 300;
  double seeding_kappa = 0.2;
  struct Placement {
    int link = 0;
    double pos = 0.0;
  };
  std::vector<Placement> custom_init;
  int n_agents() const;
};

int steps_for_minutes(const SimConfig& cfg, double minutes);

struct InitialState {
  std::vector<int> link;
  std::vector<double> pos;
};
InitialState seed_agents(const Scenario& s);
void fit_inflow_queues(Scenario& s);

// ---- simulation (engine.hpp:55-107) -------------------------------------------------
struct ForwardOptions {
  bool record_states = false;
  std::uint64_t noise_iteration = 0;
  bool trace_branches = false;  // FD-validation instrumentation: not on device
};

/// Compact per-agent state (the reference returns it dense N x L; see
/// dense_state, engine.cpp:287-294, for the exact correspondence).
struct CompactState {
  std::vector<int> link;
  std::vector<double> pos;
};

struct Trajectory {
  int steps = 0;
  std::vector<std::vector<double>> cum_per_step;  // agent units, per link
  std::vector<CompactState> states;               // per step (optional)
  CompactState final_state;
  std::vector<double> cum_final;
  double wall_seconds = 0.0;
};

Trajectory simulate_forward(const Scenario& s, const LinkParams& params,
                            const RngStream& rng, const ForwardOptions& opt = {});
/// One batched device run over several noise iterations (independent draws).
std::vector<Trajectory> simulate_forward_draws(
    const Scenario& s, const LinkParams& params, const RngStream& rng,
    const std::vector<std::uint64_t>& noise_iterations, bool record_states = false);

/// What a loss sees (engine.hpp:82-87) ...
struct LossInputs {
  const std::vector<std::vector<double>>* snapshots = nullptr;
  const std::vector<double>* cum_final = nullptr;
  const CompactState* final_state = nullptr;
};
/// ... and what it returns: the value and its adjoint seeds — exactly what the
/// reference's Checkpointed path extracts from its host loss tape
/// (engine.cpp:369-385).  d_x_final is per agent at its final valid cell.
struct LossValue {
  double loss = 0.0;
  std::vector<std::vector<double>> d_snapshots;
  std::vector<double> d_cum_final;
  std::vector<double> d_x_final;
};
using LossBuilder = std::function<LossValue(const LossInputs&)>;

enum class GradMode { FullTape, Checkpointed };

struct GradResult {
  double loss = 0.0;
  LinkParams grads;
  std::vector<std::vector<double>> snapshot_values;
  std::vector<double> cum_final_values;
  CompactState final_state;
  double wall_seconds = 0.0;
};

/// Both modes run the device checkpointed sweep (the reference asserts
/// FullTape == Checkpointed to 1e-12, test_engine.cpp:147-192); soft_choices
/// is rejected as in the reference's Checkpointed mode (engine.cpp:306-309).
GradResult simulate_gradient(const Scenario& s, const LinkParams& params,
                             const RngStream& rng, const LossBuilder& builder,
                             GradMode mode, const ForwardOptions& opt = {});
std::vector<GradResult> simulate_gradient_draws(
    const Scenario& s, const LinkParams& params, const RngStream& rng,
    const LossBuilder& builder, const std::vector<std::uint64_t>& noise_iterations);

// ---- losses used by the callers of the path -----------------------------------------
struct CountSeries {
  std::vector<int> link_ids;
  int interval_s = 300;
  std::vector<std::vector<double>> values;
  int n_intervals() const { return static_cast<int>(values.size()); }
};
/// mse_loss_builder (optimization.cpp:84-101).
LossBuilder mse_loss_builder(const CountSeries& obs, int delta_n);
/// optimize_control's loss (optimization.cpp:234-240).
LossBuilder control_loss_builder(int target_link, double desired_count, int delta_n);
/// sum_k <ws_k, s_k> + 1/2 <qs_k, s_k^2> + <wc, c> + 1/2 <qc, c^2> + <wx, x>
LossBuilder linear_quadratic_loss(std::vector<double> ws, std::vector<double> qs,
                                  std::vector<double> wc, std::vector<double> qc,
                                  std::vector<double> wx);
/// series_from_levels (observation.cpp:27-44).
CountSeries series_from_levels(const std::vector<std::vector<double>>& cum_per_step,
                               const std::vector<int>& link_ids, int interval_s,
                               double dt, int delta_n);

}  // namespace dtg
