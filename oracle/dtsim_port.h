/* TEST INFRASTRUCTURE ONLY — the CPU oracle, never linked into the product.
 *
 * Plain-C restatement of the reference hot path (dtsim 1.0.0,
 * /root/reference/proj): engine_step + simulate_forward + the Checkpointed
 * simulate_gradient reverse sweep, in per-agent (link, position) form instead
 * of the reference's dense N x L tensors.  Every function in dtsim_port.c cites
 * the reference file:line it restates.  Pinned against the reference itself
 * (oracle/_ref/libdtsim_ref.so) and the golden fixtures in tests/golden.
 */
#ifndef DTSIM_PORT_H
#define DTSIM_PORT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int n_links;          /* L */
  const int* succ_off;  /* L+1: CSR of the adjacency, successors ascending */
  const int* succ;
  const double* length; /* L, meters */
  int delta_n;          /* SimConfig::delta_n */
  double tau;           /* SimConfig::tau */
  double sentinel;      /* SimConfig::sentinel (M) */
  double gumbel_tau;    /* SimConfig::gumbel_tau */
  int trajectory_grafting;
} port_net;

typedef struct {
  const double *u, *kappa, *beta, *alpha, *cost; /* L each */
} port_params;

/* simulate_forward (src/engine.cpp:227-254).  link0/pos0: initial compact
 * state per agent (seed_agents output).  cum_per_step: T x L.  states_*:
 * optional T x N compact states after every step.  Returns 0 or an error
 * code (see port_last_error). */
int port_forward(const port_net* net, const port_params* p, uint64_t root_seed,
                 uint64_t noise_iteration, int n_agents, const int* link0,
                 const double* pos0, int T, double* cum_per_step, int* link_out,
                 double* pos_out, int* states_link, double* states_pos);

/* simulate_gradient, GradMode::Checkpointed (src/engine.cpp:303-429) with the
 * linear + quadratic loss of oracle/ref_shim.cpp:ref_gradient (any of
 * ws/qs/wc/qc/wx may be NULL).  spi: steps per observation interval.
 * grads: 5 x L (u, kappa, beta, alpha, cost).  snaps: n_snap x L. */
int port_gradient(const port_net* net, const port_params* p,
                  uint64_t root_seed, uint64_t noise_iteration, int n_agents,
                  const int* link0, const double* pos0, int T, int spi,
                  const double* ws, const double* qs, const double* wc,
                  const double* qc, const double* wx, double* loss,
                  double* grads, double* snaps, int* n_snaps,
                  double* cum_final, int* link_out, double* pos_out);

/* Same reverse sweep with the loss seeds given directly:
 * snap_seed (n_snap x L, added to the cumulative adjoint at each observation
 * boundary), cum_seed (L), x_seed (N, at each agent's final valid cell). */
int port_gradient_seeds(const port_net* net, const port_params* p,
                        uint64_t root_seed, uint64_t noise_iteration,
                        int n_agents, const int* link0, const double* pos0,
                        int T, int spi, const double* snap_seed,
                        const double* cum_seed, const double* x_seed,
                        double* grads);

/* include/dtsim/rng.hpp restated. */
uint64_t port_rng_fork(uint64_t seed, uint64_t label);
uint64_t port_rng_bits(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);
double port_rng_uniform(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);
double port_gumbel(uint64_t seed, uint64_t key, uint64_t row, uint64_t col);
/* FNV-1a 64 over n bytes continuing from h (the SURVEY §8c KAT fingerprints). */
uint64_t port_fnv1a64(const void* data, size_t n, uint64_t h);

const char* port_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
