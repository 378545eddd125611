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
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../paper_2603_25068_b200/csrc/dtg_rng.h"

struct dtg_ctx;  // the C-ABI device context (include/dtg.h)

namespace dtg {

struct ProbeTrace;  // device payload of a SurrogateTrace (csrc/dtg_probe.h)

/// Input outside the device path's contract (C-ABI status DTG_ERR_UNSUPPORTED).
struct UnsupportedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// SurrogateTrace (car_following.hpp:23-29): a recording run stores the graft /
/// carrier values and min / relu picks of every step on the device; a replay
/// run re-evaluates the program with those discontinuities frozen.  The device
/// keys the records by (step, agent) / (step, link) rather than by call order,
/// so rewind() has nothing to reset; leaving the recorded control path is
/// reported as "surrogate trace misaligned" like the reference's trace_fail.
struct SurrogateTrace {
  bool replay = false;
  void rewind() {}
  std::shared_ptr<ProbeTrace> rec;  // device records (null until recorded)
};

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
  /// Relaxed choice tensors (node_model.cpp:21).  On the device the state stays
  /// compact, so every choice value must be 0 or 1 (one-hot rows, e.g. chains);
  /// a fractional value raises UnsupportedError.
  bool soft_choices = false;
  SurrogateTrace* surrogate = nullptr;  // FD-validation record / replay
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
  /// Nonzero: identifies the initial state seed_agents() produces (equal keys
  /// promise equal states), so a device context that already holds it skips
  /// the re-seeding and upload.  0 (default): always upload.  The level-2
  /// C-ABI assigns a fresh key whenever a scenario is created or reconfigured.
  std::uint64_t state_key = 0;
  /// Record every transfer of a forward run (Trajectory::transfers): travel
  /// times.  The reference has no such output; it is derived from its
  /// per-step states (SURVEY.md §8a "Travel times").
  bool record_transfers = false;
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
  bool trace_branches = false;  // BranchTrace hash of every discrete decision
};

/// Compact per-agent state (the reference returns it dense N x L; see
/// dense_state, engine.cpp:287-294, for the exact correspondence).
struct CompactState {
  std::vector<int> link;
  std::vector<double> pos;
};

/// One link change: `agent` leaves `from` and is on `to` (at position 0)
/// after engine step `step` (0-based).  Within a step, ascending agent id.
struct TransferEvent {
  int step = 0, agent = 0, from = 0, to = 0;
};

/// Per-agent link entries and link traversal times from transfer events:
/// entry step -1 is the initial link; exit -1: still on the link at the end.
struct LinkVisit {
  int agent = 0, link = 0, entry_step = -1, exit_step = -1;
};
std::vector<LinkVisit> link_visits(const std::vector<int>& initial_link,
                                   const std::vector<TransferEvent>& transfers);

struct Trajectory {
  int steps = 0;
  std::vector<std::vector<double>> cum_per_step;  // agent units, per link
  std::vector<CompactState> states;               // per step (optional)
  CompactState final_state;
  std::vector<double> cum_final;
  double wall_seconds = 0.0;
  std::uint64_t branch_hash = 0xcbf29ce484222325ULL;  // BranchTrace::h (engine.cpp:251)
  std::vector<TransferEvent> transfers;  // Scenario::record_transfers
};

Trajectory simulate_forward(const Scenario& s, const LinkParams& params,
                            const RngStream& rng, const ForwardOptions& opt = {});
/// One batched device run over several noise iterations (independent draws).
std::vector<Trajectory> simulate_forward_draws(
    const Scenario& s, const LinkParams& params, const RngStream& rng,
    const std::vector<std::uint64_t>& noise_iterations, bool record_states = false);

/// The device run behind simulate_forward_draws without the host-side
/// Trajectory: returns the context holding the results (read them with
/// dtg_read_cum_all / dtg_read_state).  Used by the level-2 C-ABI so results
/// land directly in the caller's buffers.
::dtg_ctx* simulate_forward_device(const Scenario& s, const LinkParams& params,
                                        const RngStream& rng,
                                        const std::vector<std::uint64_t>& noise_iterations,
                                        bool record_states = false);

/// The same run with its results streamed into host buffers while the kernel
/// runs (dtg_forward_read): cum_per_step [D][T][L], link/pos_final [D][N].
::dtg_ctx* simulate_forward_into(const Scenario& s, const LinkParams& params,
                                 const RngStream& rng,
                                 const std::vector<std::uint64_t>& noise_iterations,
                                 double* cum_per_step, int* link_final, double* pos_final);

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
  std::uint64_t branch_hash = 0xcbf29ce484222325ULL;  // engine.cpp:426
};

/// Both modes run the device checkpointed sweep (the reference asserts
/// FullTape == Checkpointed to 1e-12, test_engine.cpp:147-192).  soft_choices
/// is rejected in Checkpointed mode as in the reference (engine.cpp:306-309);
/// in FullTape mode it is accepted where every choice is one-hot (then the
/// relaxed and straight-through programs have the same values and VJP).
/// trace_branches / a recording surrogate run the instrumented forward
/// (dtg_probe) beside the gradient; a replaying surrogate is unsupported.
GradResult simulate_gradient(const Scenario& s, const LinkParams& params,
                             const RngStream& rng, const LossBuilder& builder,
                             GradMode mode, const ForwardOptions& opt = {});
std::vector<GradResult> simulate_gradient_draws(
    const Scenario& s, const LinkParams& params, const RngStream& rng,
    const LossBuilder& builder, const std::vector<std::uint64_t>& noise_iterations);

// ---- FD-validation (pipeline.cpp:486-603) ----------------------
/// Result of one probe of a batched instrumented forward.
struct ProbeResult {
  std::vector<double> cum_final;
  double cum_sum = 0.0;  // sum of cum_final in link order (run_gradcheck's loss)
  std::uint64_t branch_hash = 0;
  bool on_path = true;   // false: replay left the recorded control path
};
/// Instrumented forwards of many parameter sets in ONE device launch (one CTA
/// per probe), with the scenario's soft_choices / surrogate / trace settings.
std::vector<ProbeResult> probe_forward_batch(const Scenario& s,
                                             const std::vector<LinkParams>& params,
                                             const RngStream& rng, std::uint64_t noise_iteration,
                                             bool trace_branches);

struct GradcheckReport {  // pipeline.hpp:49-55
  double max_rel_err = 0.0;
  int draws = 0;
  int redraws = 0;
  bool pass = false;
  std::vector<double> per_draw_max;
};
/// run_gradcheck (pipeline.cpp:499-585): central differences of the frozen-
/// discontinuity surrogate against the adjoint on a 3-link chain with relaxed
/// choices; all 10·L stencil probes of a draw run as one batched launch.
GradcheckReport run_gradcheck(int draws, int steps, int agents, double tol, std::uint64_t seed);

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
// ---- optimisation loops (optimization.hpp:18-128, optimization.cpp:10-295) ----------
/// Raised when a loop sees a non-finite loss (DivergenceError, config.hpp).
struct DivergenceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct AdamWConfig {
  double lr = 0.1;
  double weight_decay = 1e-5;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double eps = 1e-8;
};

/// AdamW with decoupled weight decay on the raw parameters (optimization.cpp:10-25).
class AdamW {
 public:
  AdamW(int n, const AdamWConfig& cfg) : cfg_(cfg), m_(n, 0.0), v_(n, 0.0) {}
  void step(std::vector<double>& params, const std::vector<double>& grads);
  int iterations() const { return t_; }

 private:
  AdamWConfig cfg_;
  std::vector<double> m_, v_;
  int t_ = 0;
};

/// lo + (hi - lo) * sigmoid(raw) (optimization.cpp:27-46).
class BoundedTransform {
 public:
  BoundedTransform(double lo, double hi) : lo_(lo), hi_(hi) {}
  double value(double raw) const;
  double dvalue(double raw) const;
  double raw_of(double value) const;

 private:
  double lo_, hi_;
};

/// floor + softplus(raw) (optimization.cpp:48-59).
class LowerBoundTransform {
 public:
  explicit LowerBoundTransform(double floor) : floor_(floor) {}
  double value(double raw) const;
  double dvalue(double raw) const;
  double raw_of(double value) const;

 private:
  double floor_;
};

struct OptimizeConfig {
  AdamWConfig adam;
  int patience = 20;
  int max_iterations = 200;
  bool resample_noise = true;
  int noise_draws = 1;
  GradMode grad_mode = GradMode::Checkpointed;
};

struct CalibrationResult {
  LinkParams best_params;
  double best_loss = 0.0;
  int best_iteration = -1;
  int iterations = 0;
  std::vector<double> loss_curve;
  double wall_seconds = 0.0;
};

/// Multi-GPU draw exchange for the optimisation loops: this
/// rank runs draws [rank * D/world, (rank+1) * D/world) of every iteration,
/// writes their rows [D/world][5L+2] to d_local, `gather` all-gathers them
/// (rank-major, i.e. draw order) into d_full [D][5L+2] ordered on `stream`,
/// and every rank reduces all D rows in draw order — bit-identical for any
/// world size.
struct DrawExchange {
  int world = 1;
  int rank = 0;
  double* d_local = nullptr;
  double* d_full = nullptr;
  void* stream = nullptr;  // cudaStream_t of the context and the gather
  std::function<void()> gather;
};

/// Gradient fit of (u, kappa, beta, alpha) to observed counts; costs fixed
/// (optimization.cpp:122-219).  All draws of an iteration run as one batched
/// device forward + reverse sweep with the MSE loss, its seeds and the
/// draw-ordered gradient sum on the device; the host keeps the O(L) transform
/// and AdamW arithmetic (glibc exp/pow, so parameters match the reference bit
/// for bit).
CalibrationResult calibrate(const Scenario& s, const CountSeries& obs, const ParamRanges& bounds,
                            const OptimizeConfig& cfg, const RngStream& rng,
                            const LinkParams* init = nullptr, const DrawExchange* ex = nullptr);

struct ControlConfig {
  OptimizeConfig opt;
  double cost_floor = 0.05;
};

struct ControlResult {
  std::vector<double> cost;
  double desired = 0.0;
  double achieved = 0.0;
  double gap_fraction = 0.0;
  double best_loss = 0.0;
  int iterations = 0;
  std::vector<double> loss_curve;
  bool zero_gradient_stall = false;
  double wall_seconds = 0.0;
};

/// Route-cost control toward a desired count on one link
/// (optimization.cpp:221-295), same device iteration as calibrate.
ControlResult optimize_control(const Scenario& s, const LinkParams& calibrated, int target_link,
                               double desired_count, const ControlConfig& cfg,
                               const RngStream& rng, const DrawExchange* ex = nullptr);

// ---- observation / output side --------------------------------
struct Metrics {
  double mae = 0.0;
  double pearson_r = 0.0;
  bool r_defined = false;
  int n_pairs = 0;
};
/// Noisy partial-coverage observations of a truth series (observation.cpp:46-83):
/// seeded Fisher-Yates link sample (lane 6), multiplicative uniform noise (lane 5).
std::pair<CountSeries, std::vector<int>> synthesize_observations(const CountSeries& truth,
                                                                 double noise_frac, double coverage,
                                                                 const RngStream& rng);
/// MAE and Pearson r over per-interval increments on common links (optimization.cpp:297-336).
Metrics count_metrics(const CountSeries& sim, const CountSeries& truth);
/// Intervals [k0, k1) of a series (pipeline.cpp:50-57).
CountSeries slice_intervals(const CountSeries& s, int k0, int k1);
/// "link_id,t_seconds,cumulative_count" CSV, byte-identical to pipeline.cpp:113-127.
std::string series_to_csv(const CountSeries& s);
/// Parser of that CSV with the reference's validation (pipeline.cpp:129-160).
CountSeries series_from_csv(const std::string& text);

/// series_from_levels (observation.cpp:27-44).
CountSeries series_from_levels(const std::vector<std::vector<double>>& cum_per_step,
                               const std::vector<int>& link_ids, int interval_s,
                               double dt, int delta_n);

}  // namespace dtg
