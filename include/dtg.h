/* dtg — B200-native hot path of the differentiable traffic simulator.
 *
 * C-ABI drop-in boundary.  Plain pointers and sizes only; every entry point
 * returns a status code and never throws.  Status codes follow the
 * reference's C API (include/dtsim.h:17-20 — 0 ok, 1 runtime error,
 * 2 configuration error, 3 divergence) plus DTG_ERR_CUDA / DTG_ERR_UNSUPPORTED.
 *
 * Two levels:
 *
 *  Level 1 — the device engine (dtg_ctx).  Replaces the reference's T-step
 *  loops and reverse sweep inside
 *     simulate_forward   /root/reference/proj/src/engine.cpp:227-254
 *     simulate_gradient  /root/reference/proj/src/engine.cpp:303-429
 *  i.e. engine_step (engine.cpp:70-125) and the checkpointed per-step VJP
 *  (engine.cpp:388-415).  The host keeps the Scenario / LinkParams / LossBuilder
 *  logic and hands the device a CSR network, parameters, an initial compact
 *  state and noise seeds; it gets back counts, states and loss-seeded
 *  gradients.  One context owns device memory for B independent scenarios
 *  (stochastic draws) on one GPU and one CUDA stream.
 *
 *  Level 2 — scenario API (dtg_scenario).  The reference's host surface for
 *  this path (Network / Scenario construction, seed_agents,
 *  fit_inflow_queues, sample_parameters, simulate_forward,
 *  simulate_gradient; include/dtsim/engine.hpp, network.hpp) as flat C calls
 *  for ctypes / cgo / JNI-style bindings.  Implemented in C++ over level 1.
 */
#ifndef DTG_H
#define DTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DTG_OK = 0,
  DTG_ERR_RUNTIME = 1,     /* std::runtime_error in the reference       */
  DTG_ERR_CONFIG = 2,      /* ConfigError                               */
  DTG_ERR_DIVERGENCE = 3,  /* DivergenceError (non-finite loss/grads)   */
  DTG_ERR_CUDA = 4,        /* CUDA runtime / launch failure             */
  DTG_ERR_UNSUPPORTED = 5  /* input outside the device path's contract  */
};

/* SimConfig (include/dtsim/car_following.hpp:31-40). */
typedef struct {
  int delta_n;             /* vehicles per agent (platoon size)           */
  double tau;              /* reaction time, s;  dt = tau * delta_n       */
  double sentinel;         /* M = 99999: "not on this link" marker        */
  double gumbel_tau;       /* choice relaxation temperature (0.01)        */
  int trajectory_grafting; /* TG on (1) / off (0)                         */
} dtg_sim_config;

/* Network as CSR: j is a successor of i iff i != j and
 * to_node(i) == from_node(j) (network.cpp:28-35).  Successors of each link
 * in ascending link id.  length[L] in meters. */
typedef struct {
  int n_links;
  const int* succ_off; /* L + 1 */
  const int* succ;     /* succ_off[L] */
  const double* length;
} dtg_net_desc;

typedef struct dtg_ctx dtg_ctx;

/* ---- Level 1: device engine ------------------------------------------------- */

/* Allocate a context for n_scenarios (B) scenarios of n_agents (N) agents on
 * the current CUDA device.  max_steps bounds the horizon kept in the
 * checkpoint history (grown on demand).  Replaces the per-call setup of
 * make_ctx (engine.cpp:40-59). */
int dtg_create(const dtg_net_desc* net, const dtg_sim_config* cfg,
               int n_agents, int n_scenarios, int max_steps, dtg_ctx** out);
void dtg_destroy(dtg_ctx* ctx);
/* Optional: initialise the CUDA runtime on the current device and load the
 * engine's default kernels now (CUDA does both lazily: context creation on
 * the first call, each module on its kernel's first launch, ~0.2 s together),
 * so a long-running caller does not charge them to its first request. */
int dtg_init(void);
/* Last error message of this context (or of the failed dtg_create when
 * ctx == NULL). */
const char* dtg_last_error(const dtg_ctx* ctx);
/* Run on this cudaStream_t (default: a stream owned by the context).  NULL
 * returns the context to a private non-blocking stream of its own. */
int dtg_set_stream(dtg_ctx* ctx, void* cuda_stream);
/* The stream the context runs on; *owned = 1 when it is the context's own. */
int dtg_get_stream(const dtg_ctx* ctx, void** cuda_stream, int* owned);
/* Forward as one persistent cooperative kernel for all steps (default on);
 * off = one CUDA graph of 5 kernels per step (same results). */
int dtg_set_persistent(dtg_ctx* ctx, int enabled);
/* Forward schedule: 0 auto (default), 1 one thread-block cluster per
 * scenario, 2 one persistent cooperative grid, 3 CUDA graph of 5 kernels per
 * step, 4 one CTA per scenario looping over all steps (scenarios independent,
 * CTA barriers only).  All produce identical results.  dtg_last_mode returns
 * 1000 * mode + CTAs per scenario of the last forward (1 for mode 4, 0 for
 * the graph). */
int dtg_set_mode(dtg_ctx* ctx, int mode);
/* Measurement hook: one persistent reverse sweep (zero seeds) with
 * %globaltimer stamps; phase_us[8] = mean per-step span (us) of R1, barrier,
 * R2, barrier, R3, barrier, R4 (and 0). */
int dtg_profile_backward(dtg_ctx* ctx, double* phase_us, int* grid_out);
/* Measurement hook: one scenario-resident forward (mode 4) with %globaltimer
 * stamps; phase_us[9] = mean per-step span (us) of the links, choice, merge,
 * scan and slots phases and the whole step, then the mean number of links
 * with arrived heads, the most heads on one link and the mean number of
 * chosen links per step. */
int dtg_profile_scn(dtg_ctx* ctx, int T, int steps_per_interval, double* phase_us);
/* Measurement hook: raw per-CTA stamps [T][grid][8] (ns) of that run. */
int dtg_debug_bwd_stamps(dtg_ctx* ctx, unsigned long long* out, int* grid);
int dtg_last_mode(const dtg_ctx* ctx);
/* Tuning knobs: flag 0 = grid barrier implementation (1: release/acquire
 * counter, default; 0: cooperative_groups grid.sync); flag 1 = fused
 * forward slot mapping (-1 auto, 0 interleaved blocks, 1 contiguous);
 * flag 4 = fused forward draws the next step's head decisions ahead of time
 * (1, default) or in the slot phase (0); flag 5 = those draws run in warps
 * 2.. of each CTA during barrier 1 (1, default) or in idle link-phase lanes
 * (0); flag 7 = CTAs per scenario of the grid schedule (0 = auto); flag 8 =
 * scenario branches of the step graph (0 = auto: 2 from B = 8, 4 from 32).  Results
 * are identical. */
int dtg_set_flag(dtg_ctx* ctx, int flag, int value);
/* Measurement hook: one persistent forward with %globaltimer stamps; returns
 * the mean per-step span (us) of [slot phase, barrier 1, link phase,
 * barrier 2] over all CTAs and the grid size used. */
int dtg_profile_persistent(dtg_ctx* ctx, int n_steps, int steps_per_interval,
                           double* phase_us, int* grid_out);
/* Use CUDA graphs for the per-step launch sequence (default on). */
int dtg_set_graphs(dtg_ctx* ctx, int enabled);

/* Per-link parameter vectors (LinkParams, network.hpp:22-28) for one
 * scenario, or all scenarios when scenario < 0. Host pointers, L each. */
int dtg_set_params(dtg_ctx* ctx, int scenario, const double* u,
                   const double* kappa, const double* beta, const double* alpha,
                   const double* cost);
/* Initial compact state per agent (seed_agents / custom_init output:
 * engine.cpp:156-189), for one scenario or all (scenario < 0).  Positions
 * below the validity threshold (-0.01) are rejected. */
int dtg_set_state(dtg_ctx* ctx, int scenario, const int* link,
                  const double* pos);
/* Noise of one scenario (or all): the reference's
 * rng.fork(kIteration).fork(noise_iteration) (engine.cpp:49). */
int dtg_set_noise(dtg_ctx* ctx, int scenario, uint64_t root_seed,
                  uint64_t noise_iteration);

/* Run n_steps engine steps for every scenario from the state set by
 * dtg_set_state.  checkpoint != 0 keeps every step's compact state on the
 * device (required by dtg_backward and per-step dtg_read_state).
 * steps_per_interval: observation interval in steps (snapshot boundaries
 * (t + 1) % spi == 0, engine.cpp:321-323). */
int dtg_forward(dtg_ctx* ctx, int n_steps, int steps_per_interval,
                int checkpoint);

/* dtg_forward followed by the read-back of its results into host buffers,
 * overlapped with the run: the persistent kernel publishes each finished step
 * (host-mapped counter) and finished count rows are copied on a second stream
 * while later steps compute.  cum_per_step [B][T][L] (as dtg_read_cum_all),
 * link_final / pos_final [B][N] (as dtg_read_state of step T); any may be
 * NULL.  Same results as dtg_forward + the reads. */
int dtg_forward_read(dtg_ctx* ctx, int n_steps, int steps_per_interval,
                     int checkpoint, double* cum_per_step, int* link_final,
                     double* pos_final);

/* Page-locked host memory for result buffers: dtg_forward_read (and the
 * level-2 dtg_simulate_forward) DMA their results straight into such buffers
 * instead of staging them.  NULL on failure. */
void* dtg_host_alloc(size_t bytes);
void dtg_host_free(void* ptr);

/* Wait for the context's stream and report device-side errors of the last
 * forward / backward (reads below do this implicitly). */
int dtg_sync(dtg_ctx* ctx);
/* Test hook: always take the exact ordered-sum path for the rows routed to
 * the first arrived agent (normally used only on near ties). */
int dtg_debug_force_slow_path(dtg_ctx* ctx, int on);

/* Decision instrumentation (process-wide, all contexts on the device): returns
 * how many link-choice / merge decisions since the last call the fast rules
 * handed to the exact softmax evaluation (second-stage near ties within
 * 2^-40, merge winners inside the rounding bound) and resets the count;
 * force_exact 1 sends every decision to the exact evaluation, 0 restores the
 * fast rules, -1 leaves the setting.  Results are identical either way. */
int dtg_debug_decisions(int force_exact, unsigned long long* exact_decisions);
/* Test hook: n Gumbel draws -log(-log(u)), u = uniform(seed, key, rows[i],
 * cols[i]), computed by the device code path (libdevice log). */
int dtg_debug_gumbel(uint64_t seed, uint64_t key, int n, const uint64_t* rows,
                     const uint64_t* cols, double* out);

/* Test hook: clock64 cycles per dependent primitive on the device
 * (which: 0 Gumbel draw, 1 log, 2 exp, 3 division, 4 L2 pointer chase,
 * 5 counter-RNG uniform; 100 = empty grid.sync with `grid` CTAs of 512). */
int dtg_debug_microbench(int which, int n, int grid, double* result);
/* Measurement hooks for the roofline (builder-measured, not NVIDIA figures):
 * L2 read bandwidth over an L2-resident `bytes` buffer, and the time per step
 * of a persistent grid of `grid` CTAs x 512 doing only the fused forward's two
 * grid barriers and one dependent global round trip per phase. */
int dtg_debug_l2_bandwidth(long long bytes, int reps, double* gbps);
int dtg_debug_step_floor(int grid, int n_steps, double* us_per_step);
/* Test hook: the device's interleaved glibc log / Gumbel (several draws per
 * chain) against its scalar glibc log on n inputs per kind; mismatches must
 * be 0 and flagged stays 0. */
int dtg_debug_log_check(uint64_t seed, long long n, unsigned long long* mismatches,
                        unsigned long long* flagged);
/* Test hook: the glibc-identical exp / log (csrc/dtg_libm.h) against this
 * host's libm (the reference's), bit for bit, on n inputs of kind `which`:
 * 0 log(u) of Gumbel uniforms, 1 log(-log u), 2 the whole Gumbel -log(-log u),
 * 3 log of any positive double, 4 log near 1, 5 exp on [-750, 710],
 * 6 exp on [-60, 0], 7 exp of any finite double.  on_device: evaluate on the
 * GPU (else the host build of the same code). */
int dtg_debug_libm_check(int which, uint64_t seed, long long n, int on_device,
                         unsigned long long* mismatches);
/* Test hook: one fused forward recording, per step and warp, the slot-phase
 * start, end of the offsets prologue, end of the slot loop (globaltimer ns)
 * and the number of arrived agents in the warp: out[T][n_warps][4]. */
int dtg_debug_warp_records(dtg_ctx* ctx, int n_steps, int steps_per_interval,
                           unsigned long long* out, int* n_warps);

/* Results of the last dtg_forward.
 * cum_per_step: n_steps x L cumulative counts (Trajectory::cum_per_step).
 * state: compact (link, pos) per agent after `step` steps (step in
 * [0, n_steps]; any step needs checkpoint, n_steps works always). */
int dtg_read_cum(dtg_ctx* ctx, int scenario, double* cum_per_step);
/* All scenarios at once ([B][n_steps][L]), one device->host copy. */
int dtg_read_cum_all(dtg_ctx* ctx, double* cum_per_step);
int dtg_read_state(dtg_ctx* ctx, int scenario, int step, int* link,
                   double* pos);
/* Transfer events (travel times).  With recording on, every
 * forward stores the agent admitted to each link at each step ([T][B][L],
 * 4 B per link-step, written by the merge).  dtg_read_transfers: [T][L]
 * admitted agent ids (-1: none) of one scenario of the last forward;
 * dtg_transfer_events: its link changes as rows (step, agent, from, to),
 * step-major then ascending agent (the agent is on `to` after engine step
 * `step`), `from` tracked from the scenario's dtg_set_state links; events
 * NULL / cap too small: *n_events is the count only. */
int dtg_set_record_transfers(dtg_ctx* ctx, int on);
int dtg_read_transfers(dtg_ctx* ctx, int scenario, int* winners);
int dtg_transfer_events(dtg_ctx* ctx, int scenario, int* events, size_t cap,
                        size_t* n_events);
/* Number of observation snapshots of the last forward. */
int dtg_n_snapshots(const dtg_ctx* ctx);

/* Checkpointed reverse sweep of the last dtg_forward(checkpoint=1).
 * Seeds (host pointers, per scenario, scenario-major):
 *   snap_seeds [B][K][L]  dLoss/dsnapshot_k (K = dtg_n_snapshots)
 *   cum_seeds  [B][L]     dLoss/dcum_final
 *   x_seeds    [B][N]     dLoss/dX_final at each agent's final valid cell
 * Any seed pointer may be NULL (zero).  grads [B][5][L] (u, kappa, beta,
 * alpha, cost) receives each scenario's parameter gradient. */
int dtg_backward(dtg_ctx* ctx, const double* snap_seeds,
                 const double* cum_seeds, const double* x_seeds,
                 double* grads);
/* Same with device pointers for seeds and output (the stream-ordered path
 * used for NCCL reductions without a host round trip). */
int dtg_backward_device(dtg_ctx* ctx, const double* d_snap_seeds,
                        const double* d_cum_seeds, const double* d_x_seeds,
                        double* d_grads);

/* ---- Device losses ---------------------------------
 * The two losses of the reference's optimisation loops, evaluated on the
 * device from the count history of the last checkpointed forward, so an
 * optimisation iteration needs no host round trip of snapshots and seeds:
 *   MSE     mse_loss_builder (optimization.cpp:83-101): obs_values[k_obs][n_obs]
 *           in vehicles for link_ids[n_obs] (duplicates allowed);
 *   control optimize_control's (cum_final[target] * delta_n - desired)^2
 *           (optimization.cpp:234-240). */
int dtg_set_loss_mse(dtg_ctx* ctx, int k_obs, int n_obs, const int* link_ids,
                     const double* obs_values);
int dtg_set_loss_control(dtg_ctx* ctx, int target_link, double desired_count);
/* After dtg_forward(checkpoint=1): loss + seeds on the device, the reverse
 * sweep, and one row per scenario written to d_rows [B][5L+2] (device
 * pointer; NULL = the context's own buffer):
 *   [grads u | kappa | beta | alpha | cost (5L), loss, extra]
 * extra = cum_final[target] * delta_n for the control loss, else 0.
 * Stream-ordered, no host synchronisation (an NCCL all-gather of the rows
 * can follow on the same stream). */
int dtg_gradient_device_loss(dtg_ctx* ctx, double* d_rows);
/* Draw-ordered reduction of n_draws rows (device pointer d_rows, or NULL =
 * the context's own B rows) into out[5L+2] (host), synchronising:
 *   mode 0 (calibrate, optimization.cpp:176-193): g_0 + g_1 + ...
 *   mode 1 (control,   optimization.cpp:262-264): 0 + g_0/D + g_1/D + ...
 *   loss and extra: 0 + x_0/D + x_1/D + ... in both modes. */
int dtg_reduce_draw_rows(dtg_ctx* ctx, int n_draws, const double* d_rows,
                         int mode, double* out);

/* The draw-ordered reduction of dtg_reduce_draw_rows, kept on the device;
 * only head[2] = (loss, extra) crosses to the host.  dtg_read_reduced_row
 * copies the whole row [5L+2] of the last reduction. */
int dtg_reduce_draw_rows_head(dtg_ctx* ctx, int n_draws, const double* d_rows, int mode, double* head);
int dtg_read_reduced_row(dtg_ctx* ctx, double* out);

/* Device-resident calibrate step (optimization.cpp:10-59, 173-205), bit-
 * identical to the host loop: raw[4L] = (u, kappa, beta, alpha) in raw space,
 * BoundedTransform ranges lo[4] / hi[4], AdamW settings.  init uploads raw,
 * zeroes the moments and sets the context's (u, kappa, beta, alpha) of every
 * scenario to the realised raw (cost as last set; set parameters first).
 * step: gradient of the last device reduction (mode 0) / draws through the
 * transform's derivative, AdamW with bias corrections bc1 = 1 - beta1^t,
 * bc2 = 1 - beta2^t, and the parameters of the new raw.  mark_best keeps a
 * device copy of the current raw; read copies raw and / or that copy (either
 * may be NULL). */
int dtg_opt_bounded_init(dtg_ctx* ctx, const double* raw, const double* lo, const double* hi, double lr,
                         double beta1, double beta2, double eps, double weight_decay);
int dtg_opt_bounded_step(dtg_ctx* ctx, int draws, double bc1, double bc2);
int dtg_opt_bounded_mark_best(dtg_ctx* ctx);
int dtg_opt_bounded_read(dtg_ctx* ctx, double* raw, double* best_raw);

/* Measurement hook: run n_steps of the forward (backward != 0: the reverse
 * sweep of the preceding checkpointed forward) without graphs, bracketing
 * every kernel with CUDA events on the context stream.  ms_out[w] receives
 * the summed duration of kernel kind w (4 forward / 8 reverse kinds, named by
 * dtg_kernel_name); launches_out the number of kernels launched. */
int dtg_profile_kernels(dtg_ctx* ctx, int n_steps, int steps_per_interval,
                        int backward, double* ms_out, int64_t* launches_out);
const char* dtg_kernel_name(int backward, int which);

/* Device pointer to the cumulative-count history [n_steps + 1][B][L]
 * (row 0 = zeros) of the last forward, valid until the next forward. */
const double* dtg_device_cum(const dtg_ctx* ctx);
/* Number of kernels the last forward / backward launched. */
int64_t dtg_last_launches(const dtg_ctx* ctx);

/* ---- Level 2: scenario API ---------------------------------------------------
 * Mirrors include/dtsim/network.hpp + engine.hpp.  kind: 0 physical,
 * 1 virtual inflow, 2 virtual outflow (LinkKind). */
typedef struct dtg_scenario dtg_scenario;

/* make_network (network.cpp:238-247) from explicit links. */
dtg_scenario* dtg_scenario_from_links(int n_nodes, int n_links,
                                      const int* from_node, const int* to_node,
                                      const double* length, const int* kind);
/* Synthetic n x n grid (east pair then south pair per node, row-major),
 * then attach_virtual_links(RngStream(net_seed), virtual_length)
 * (network.cpp:151-201).  NULL on error (see dtg_last_error(NULL)). */
dtg_scenario* dtg_scenario_grid(int n, double length, uint64_t net_seed,
                                double virtual_length);
/* parse_tntp_text (network.cpp:58-118) + attach_virtual_links. */
dtg_scenario* dtg_scenario_tntp(const char* text, double length_unit_scale,
                                uint64_t net_seed, double virtual_length);
void dtg_scenario_free(dtg_scenario* sc);
/* Scenario fields + SimConfig; fit_queues != 0 runs fit_inflow_queues
 * (engine.cpp:191-213). */
int dtg_scenario_configure(dtg_scenario* sc, int n_vehicles, int delta_n,
                           double tau, double gumbel_tau,
                           int trajectory_grafting, int horizon_steps,
                           int obs_interval_s, int fit_queues);
/* Scenario::custom_init (engine.hpp:28-32); n == 0 clears it. */
int dtg_scenario_custom_init(dtg_scenario* sc, int n, const int* link,
                             const double* pos);
int dtg_scenario_n_links(const dtg_scenario* sc);
int dtg_scenario_n_nodes(const dtg_scenario* sc);
/* Scenario::n_agents (engine.cpp:139-147); -1 on error. */
int dtg_scenario_n_agents(const dtg_scenario* sc);
int dtg_scenario_links(const dtg_scenario* sc, int* from_node, int* to_node,
                       double* length, int* kind);
/* Successor CSR (succ_off: L + 1, succ: dtg_scenario_n_edges). */
int dtg_scenario_n_edges(const dtg_scenario* sc);
int dtg_scenario_csr(const dtg_scenario* sc, int* succ_off, int* succ);
/* sample_parameters (network.cpp:203-236) with the default ParamRanges. */
int dtg_scenario_sample_parameters(const dtg_scenario* sc, uint64_t seed,
                                   int mean_mode, double* u, double* kappa,
                                   double* beta, double* alpha, double* cost);
/* seed_agents (engine.cpp:156-189). */
int dtg_scenario_seed_agents(const dtg_scenario* sc, int* link, double* pos);
/* steps_for_minutes (engine.cpp:149-154); -1 on error. */
int dtg_steps_for_minutes(int delta_n, double tau, double minutes);

/* Scenario::record_transfers: level-2 forwards record transfer events (read
 * them with dtg_transfer_events on dtg_scenario_ctx(sc), draw d = scenario d). */
int dtg_scenario_set_record_transfers(dtg_scenario* sc, int on);
/* simulate_forward for n_draws noise iterations of one scenario (draw d uses
 * noise_iterations[d]; scenario-major outputs).  cum_per_step [D][T][L],
 * link_final/pos_final [D][N]; states_link/states_pos [D][T][N] optional
 * (ForwardOptions::record_states).  wall_seconds (optional): wall time. */
int dtg_simulate_forward(dtg_scenario* sc, const double* u,
                         const double* kappa, const double* beta,
                         const double* alpha, const double* cost,
                         uint64_t root_seed, int n_draws,
                         const uint64_t* noise_iterations,
                         double* cum_per_step, int* link_final,
                         double* pos_final, int* states_link,
                         double* states_pos, double* wall_seconds);

/* simulate_gradient (Checkpointed) for n_draws draws with the linear +
 * quadratic loss
 *   loss = sum_k sum_j (ws[k,j] s_kj + qs[k,j] s_kj^2 / 2)
 *        + sum_j (wc[j] c_j + qc[j] c_j^2 / 2) + sum_n wx[n] x_n(final)
 * over snapshots s_k, cum_final c and final positions (any coefficient array
 * may be NULL; ws/qs are K x L, shared by all draws).  Outputs per draw:
 * loss[D], grads[D][5][L], snapshots[D][K][L], cum_final[D][L],
 * link_final/pos_final[D][N] (optional). */
int dtg_simulate_gradient(dtg_scenario* sc, const double* u,
                          const double* kappa, const double* beta,
                          const double* alpha, const double* cost,
                          uint64_t root_seed, int n_draws,
                          const uint64_t* noise_iterations, const double* ws,
                          const double* qs, const double* wc, const double* qc,
                          const double* wx, double* loss, double* grads,
                          double* snapshots, double* cum_final,
                          int* link_final, double* pos_final,
                          double* wall_seconds);

/* simulate_gradient with the calibration loss mse_loss_builder
 * (optimization.cpp:84-101): observed link ids obs_ids[n_obs], observations
 * obs_values [K_obs][n_obs] in vehicles. */
int dtg_simulate_gradient_mse(dtg_scenario* sc, const double* u,
                              const double* kappa, const double* beta,
                              const double* alpha, const double* cost,
                              uint64_t root_seed, int n_draws,
                              const uint64_t* noise_iterations, int n_obs,
                              const int* obs_ids, int k_obs,
                              const double* obs_values, double* loss,
                              double* grads);

/* AdamWConfig + OptimizeConfig (optimization.hpp:18-24, 72-82). */
typedef struct {
  double lr;            /* 0.1   */
  double weight_decay;  /* 1e-5  */
  double beta1;         /* 0.9   */
  double beta2;         /* 0.999 */
  double eps;           /* 1e-8  */
  int patience;         /* 20    */
  int max_iterations;   /* 200   */
  int resample_noise;   /* 1     */
  int noise_draws;      /* 1     */
} dtg_optimize_config;

/* ParamRanges (engine.hpp / network.cpp sample_parameters bounds). */
typedef struct {
  double u_lo, u_hi, kappa_lo, kappa_hi, beta_lo, beta_hi, alpha_lo, alpha_hi;
} dtg_param_ranges;

/* Multi-GPU draw exchange.  With world > 1 this rank runs
 * draws [rank*D/world, (rank+1)*D/world) of each iteration, writes their
 * rows [D/world][5L+2] (see dtg_gradient_device_loss) to d_local, calls
 * gather(user) — which must all-gather d_local of every rank, rank-major,
 * into d_full [D][5L+2], ordered on `stream` (e.g. NCCL all_gather) — and
 * reduces all D rows in draw order, so every rank gets the single-GPU result
 * bit for bit.  The context runs on `stream` (cudaStream_t) for the duration
 * of the loop and returns to its previous stream afterwards; `stream` is
 * required when world > 1 (the gather is ordered after the rows only through
 * it) and may be NULL for world == 1. */
typedef int (*dtg_gather_fn)(void* user);
typedef struct {
  int world;
  int rank;
  double* d_local;
  double* d_full;
  void* stream;
  dtg_gather_fn gather;
  void* user;
} dtg_draw_exchange;

/* calibrate (optimization.cpp:122-219) with the device iteration: per
 * iteration one batched forward + reverse sweep over the noise draws, MSE
 * loss/seeds and the draw sum on the device, and the transform + AdamW step
 * on the device too (dtg_opt_bounded_*, bit-identical to the host loop's
 * glibc arithmetic): only (loss, extra) crosses to the host per iteration.
 * init_* may be NULL (start from raw 0 = range midpoints, cost 1);
 * init_cost may be NULL alone.  loss_curve has room for max_iterations.
 * Returns DTG_ERR_DIVERGENCE on a non-finite loss. */
int dtg_calibrate(dtg_scenario* sc, int n_obs, const int* obs_ids, int k_obs,
                  const double* obs_values, const dtg_param_ranges* bounds,
                  const dtg_optimize_config* cfg, uint64_t root_seed,
                  const double* init_u, const double* init_kappa,
                  const double* init_beta, const double* init_alpha,
                  const double* init_cost, double* best_u, double* best_kappa,
                  double* best_beta, double* best_alpha, double* best_cost,
                  double* best_loss, int* best_iteration, int* iterations,
                  double* loss_curve, double* wall_seconds,
                  const dtg_draw_exchange* exchange /* NULL: one GPU */);

/* optimize_control (optimization.cpp:221-295): fit per-link route costs
 * (LowerBoundTransform with cost_floor) so cum_final[target] * delta_n
 * approaches desired.  cost_out[L]; loss_curve has room for max_iterations. */
int dtg_optimize_control(dtg_scenario* sc, const double* u, const double* kappa,
                         const double* beta, const double* alpha,
                         const double* cost, int target_link, double desired,
                         const dtg_optimize_config* cfg, double cost_floor,
                         uint64_t root_seed, double* cost_out, double* achieved,
                         double* gap_fraction, double* best_loss,
                         int* iterations, double* loss_curve,
                         int* zero_gradient_stall, double* wall_seconds,
                         const dtg_draw_exchange* exchange /* NULL: one GPU */);

/* Device context a scenario uses (for dtg_set_stream / dtg_last_launches);
 * NULL before the first simulate call. */
dtg_ctx* dtg_scenario_ctx(dtg_scenario* sc);
/* Host-side calibration loss (mse_loss_builder, optimization.cpp:84-101):
 * value and adjoint seeds over k_snap snapshots (k_snap x L). */
int dtg_mse_loss(int k_snap, int n_links, const double* snapshots, int n_obs,
                 const int* obs_ids, int k_obs, const double* obs_values,
                 int delta_n, double* loss, double* seeds);
const char* dtg_scenario_last_error(const dtg_scenario* sc);

/* ---- FD-validation instrumentation ----------------------
 * The reference's finite-difference validation modes (car_following.hpp:23-40,
 * branch_trace.hpp, engine.hpp:55-59/70/98, pipeline.hpp:49-61), run by the
 * device probe engine (csrc/dtg_probe.cu, one CTA per probe).  Soft choices
 * and surrogate replay keep the compact per-agent state, so every choice value
 * must stay 0 or 1 (one-hot rows, e.g. run_gradcheck's chain); a fractional
 * value returns DTG_ERR_UNSUPPORTED.  Errors: dtg_scenario_last_error(sc)
 * (dtg_scenario_last_error(NULL) for dtg_run_gradcheck). */
typedef struct dtg_surrogate dtg_surrogate; /* SurrogateTrace */
dtg_surrogate* dtg_surrogate_create(void);
void dtg_surrogate_free(dtg_surrogate* tr);
/* SurrogateTrace::replay (false: the next run records) and rewind(). */
int dtg_surrogate_set_replay(dtg_surrogate* tr, int replay);
int dtg_surrogate_rewind(dtg_surrogate* tr);
/* SimConfig::soft_choices / SimConfig::surrogate (NULL detaches). */
int dtg_scenario_set_soft_choices(dtg_scenario* sc, int soft);
int dtg_scenario_set_surrogate(dtg_scenario* sc, dtg_surrogate* tr);
/* simulate_forward with ForwardOptions{noise_iteration, trace_branches} and
 * the scenario's soft / surrogate settings; branch_hash = Trajectory::
 * branch_hash (the FNV offset basis when not tracing).  cum_per_step [T][L],
 * link_final / pos_final [N] (link -1: the agent has no valid cell). */
int dtg_simulate_forward_traced(dtg_scenario* sc, const double* u,
                                const double* kappa, const double* beta,
                                const double* alpha, const double* cost,
                                uint64_t root_seed, uint64_t noise_iteration,
                                int trace_branches, double* cum_per_step,
                                int* link_final, double* pos_final,
                                uint64_t* branch_hash, double* wall_seconds);
/* simulate_gradient (grad_mode 0 FullTape, 1 Checkpointed) with the
 * linear-quadratic loss of dtg_simulate_gradient; branch_hash =
 * GradResult::branch_hash.  A recording surrogate is filled. */
int dtg_simulate_gradient_traced(dtg_scenario* sc, const double* u,
                                 const double* kappa, const double* beta,
                                 const double* alpha, const double* cost,
                                 uint64_t root_seed, uint64_t noise_iteration,
                                 int grad_mode, int trace_branches,
                                 const double* ws, const double* qs,
                                 const double* wc, const double* qc,
                                 const double* wx, double* loss, double* grads,
                                 double* cum_final, uint64_t* branch_hash);
/* n_probes instrumented forwards in ONE device launch (params [P][5][L]):
 * cum_final [P][L], cum_sum [P] (sum of cum_final in link order),
 * branch_hash [P], on_path [P] (0: a replay left the recorded control path).
 * Any output may be NULL. */
int dtg_probe_forward_batch(dtg_scenario* sc, int n_probes, const double* params,
                            uint64_t root_seed, uint64_t noise_iteration,
                            int trace_branches, double* cum_final,
                            double* cum_sum, uint64_t* branch_hash,
                            int* on_path);
/* run_gradcheck (pipeline.cpp:499-585) -> GradcheckReport; per_draw_max has
 * room for `draws`.  The report not passing is not an error (pass = 0). */
int dtg_run_gradcheck(int draws, int steps, int agents, double tol,
                      uint64_t seed, double* max_rel_err, int* redraws,
                      int* pass, double* per_draw_max);

/* ---- Observation / output side -------------------------
 * Host-only helpers on count series (values [k][n] row-major, one row per
 * observation interval).  Errors: dtg_observe_last_error(). */
const char* dtg_observe_last_error(void);
/* synthesize_observations (observation.cpp:46-83): m_out = floor(coverage*n)
 * observed links (ascending position) into obs_ids[n] / obs_values[k][m]. */
int dtg_synthesize_observations(int k, int n, const int* link_ids,
                                const double* values, int interval_s,
                                double noise_frac, double coverage,
                                uint64_t root_seed, int* m_out, int* obs_ids,
                                double* obs_values);
/* count_metrics (optimization.cpp:297-336). */
int dtg_count_metrics(int k_sim, int n_sim, const int* sim_ids,
                      const double* sim_values, int k_truth, int n_truth,
                      const int* truth_ids, const double* truth_values,
                      double* mae, double* pearson_r, int* r_defined,
                      int* n_pairs);
/* series_to_csv (pipeline.cpp:113-127), byte-identical; buf NULL: *len only. */
int dtg_series_to_csv(int k, int n, const int* ids, const double* values,
                      int interval_s, char* buf, size_t cap, size_t* len);
/* series_from_csv (pipeline.cpp:129-160); ids/values NULL: sizes only. */
int dtg_series_from_csv(const char* text, int* k, int* n, int* interval_s,
                        int* ids, double* values, size_t cap_ids,
                        size_t cap_values);

#ifdef __cplusplus
}
#endif
#endif /* DTG_H */
