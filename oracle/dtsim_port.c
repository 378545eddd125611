/* TEST INFRASTRUCTURE ONLY — the CPU oracle ("port"), never the product.
 *
 * Per-agent restatement of the reference hot path (dtsim 1.0.0).  The
 * reference stores the state as a dense N x L fp64 tensor and differentiates
 * it with a tape (src/tensor.cpp); this file keeps one (link, position) pair
 * per agent and writes every forward rule and every VJP out by hand, in the
 * reference's operation order so values (and, up to summation order, the
 * gradients) are the reference's.  Citations are /root/reference/proj paths.
 *
 * Build: oracle/Makefile (-O2 -ffp-contract=off, no -march).
 */
#include "dtsim_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* port_last_error(void) { return g_err; }

/* car_following.hpp:12-16 */
#define VALID_THR (-1e-2)
#define ARRIVAL_TOL (1e-2)
#define MASK_LARGE (1e12)

/* ---- include/dtsim/rng.hpp --------------------------------------------------- */
static uint64_t mix(uint64_t x) { /* rng.hpp:42-47 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t port_rng_fork(uint64_t seed, uint64_t label) { /* rng.hpp:14-16 */
  return mix(seed ^ mix(label ^ 0x8e9b5c1d3a7f2406ULL));
}
uint64_t port_rng_bits(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = mix(seed ^ mix(a)); /* rng.hpp:18-24 */
  h = mix(h ^ mix(b ^ 0x6a09e667f3bcc909ULL));
  h = mix(h ^ mix(c ^ 0xbb67ae8584caa73bULL));
  return h;
}
double port_rng_uniform(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  /* rng.hpp:27-31 */
  return ((double)(port_rng_bits(seed, a, b, c) >> 11) + 0.5) *
         (1.0 / 9007199254740992.0);
}
uint64_t port_fnv1a64(const void* data, size_t n, uint64_t h) {
  const unsigned char* b = (const unsigned char*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

double port_gumbel(uint64_t seed, uint64_t key, uint64_t row, uint64_t col) {
  /* tensor.cpp:694-695 */
  const double u = port_rng_uniform(seed, key, row, col);
  return -log(-log(u));
}

/* ---- working storage ------------------------------------------------------------ */
typedef struct {
  const port_net* net;
  const port_params* p;
  int L, N, maxdeg;
  double M, dt, k; /* sentinel, tau*delta_n, 1/gumbel_tau */
  uint64_t seed_link, seed_merge;
  /* per-link agent lists: ids ascending (gather order, engine.cpp:76-82) and
   * sorted by (x desc, id asc) (argsort_desc, tensor.cpp:672-680) */
  int *cnt, *off, *ids, *seg;
  /* per agent */
  double *x1, *gap;
  unsigned char *pick_cong, *pick_cap;
  int *aidx;     /* index in A or -1 */
  int *admitted; /* destination link or -1 */
  double *admbar;
  /* per link */
  double *q, *a, *vacant, *pref_bar, *alpha_bar, *ubar, *jambar;
  int* winner;    /* agent id or -1 */
  int* cand_off;  /* L+1 */
  int* cand;      /* candidate agent ids, ascending per row */
  double *mpi, *mlogz;
  unsigned char* row_live; /* row winner came from live candidates */
  /* arrived set A (ascending agent id) */
  int nA;
  int *A, *choice;
  double *pi, *logz, *lbar, *prio_bar;
} Ctx;

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) {
    fprintf(stderr, "dtsim_port: out of memory\n");
    abort();
  }
  return p;
}

static void ctx_init(Ctx* c, const port_net* net, const port_params* p,
                     int N, uint64_t root_seed, uint64_t noise_iteration) {
  memset(c, 0, sizeof *c);
  c->net = net;
  c->p = p;
  c->L = net->n_links;
  c->N = N;
  c->M = net->sentinel;
  c->dt = net->tau * net->delta_n; /* SimConfig::dt, car_following.hpp:39 */
  c->k = 1.0 / net->gumbel_tau;    /* node_model.cpp:20 */
  /* engine.cpp:49: ctx.rng = rng.fork(kIteration).fork(noise_iteration);
   * node_model.cpp:65, 114: fork(kGumbelLink) / fork(kGumbelMerge) */
  const uint64_t it = port_rng_fork(port_rng_fork(root_seed, 7), noise_iteration);
  c->seed_link = port_rng_fork(it, 3);
  c->seed_merge = port_rng_fork(it, 4);
  int L = c->L;
  c->maxdeg = 1;
  for (int j = 0; j < L; ++j) {
    int d = net->succ_off[j + 1] - net->succ_off[j];
    if (d > c->maxdeg) c->maxdeg = d;
  }
  if (c->maxdeg > 256) {
    fprintf(stderr, "dtsim_port: out-degree > 256 not supported\n");
    abort();
  }
  c->cnt = xcalloc(L, sizeof(int));
  c->off = xcalloc(L + 1, sizeof(int));
  c->ids = xcalloc(N, sizeof(int));
  c->seg = xcalloc(N, sizeof(int));
  c->x1 = xcalloc(N, sizeof(double));
  c->gap = xcalloc(N, sizeof(double));
  c->pick_cong = xcalloc(N, 1);
  c->pick_cap = xcalloc(N, 1);
  c->aidx = xcalloc(N, sizeof(int));
  c->admitted = xcalloc(N, sizeof(int));
  c->admbar = xcalloc(N, sizeof(double));
  c->q = xcalloc(L, sizeof(double));
  c->a = xcalloc(L, sizeof(double));
  c->vacant = xcalloc(L, sizeof(double));
  c->pref_bar = xcalloc(L, sizeof(double));
  c->alpha_bar = xcalloc(L, sizeof(double));
  c->ubar = xcalloc(L, sizeof(double));
  c->jambar = xcalloc(L, sizeof(double));
  c->winner = xcalloc(L, sizeof(int));
  c->cand_off = xcalloc(L + 1, sizeof(int));
  c->row_live = xcalloc(L, 1);
  c->cand = xcalloc(N, sizeof(int));
  c->mpi = xcalloc(N, sizeof(double));
  c->mlogz = xcalloc(N, sizeof(double));
  c->A = xcalloc(N, sizeof(int));
  c->choice = xcalloc(N, sizeof(int));
  c->pi = xcalloc((size_t)N * c->maxdeg, sizeof(double));
  c->logz = xcalloc((size_t)N * c->maxdeg, sizeof(double));
  c->lbar = xcalloc((size_t)N * c->maxdeg, sizeof(double));
  c->prio_bar = xcalloc(N, sizeof(double));
}

static void ctx_free(Ctx* c) {
  void* ptrs[] = {c->cnt, c->off, c->ids, c->seg, c->x1, c->gap, c->pick_cong,
                  c->pick_cap, c->aidx, c->admitted, c->admbar, c->q, c->a,
                  c->vacant, c->pref_bar, c->alpha_bar, c->ubar, c->jambar,
                  c->winner, c->cand_off, c->row_live, c->cand, c->mpi,
                  c->mlogz, c->A, c->choice, c->pi, c->logz, c->lbar,
                  c->prio_bar};
  for (size_t i = 0; i < sizeof ptrs / sizeof ptrs[0]; ++i) free(ptrs[i]);
}

/* two-stage Gumbel softmax over n live columns (sample_choices,
 * node_model.cpp:13-25 with log_softmax/softmax of tensor.cpp:407-433).
 * Columns outside the live set carry utility -1e12 in the reference; their
 * exp() underflows to exactly 0, so the ordered sums over live columns are the
 * reference's sums bit for bit.  Returns the first argmax of pi. */
static int two_softmax(int n, const double* v, const double* g, double k,
                       double* logz, double* pi) {
  double m = v[0];
  for (int t = 1; t < n; ++t)
    if (m < v[t]) m = v[t]; /* std::max, tensor.cpp:413 */
  double z = 0.0;
  for (int t = 0; t < n; ++t) z += exp(v[t] - m);
  const double lz = log(z) + m;
  double y[64];
  double* yy = n <= 64 ? y : xcalloc(n, sizeof(double));
  for (int t = 0; t < n; ++t) {
    logz[t] = v[t] - lz;
    yy[t] = (logz[t] + g[t]) * k; /* scale(add(logz, noise), 1/tau_g) */
  }
  double m2 = yy[0];
  for (int t = 1; t < n; ++t)
    if (m2 < yy[t]) m2 = yy[t];
  double z2 = 0.0;
  for (int t = 0; t < n; ++t) z2 += exp(yy[t] - m2);
  int best = 0;
  for (int t = 0; t < n; ++t) {
    pi[t] = exp(yy[t] - m2) / z2;
    if (pi[t] > pi[best]) best = t; /* onehot_argmax_rows, tensor.cpp:660-670 */
  }
  if (yy != y) free(yy);
  return best;
}

/* VJP of two_softmax given pibar (tensor.cpp:877-911, scale VJP :809-812).
 * Returns vbar in place of pibar. */
static void two_softmax_vjp(int n, const double* logz, const double* pi,
                            double k, double* bar) {
  double dot = 0.0;
  for (int t = 0; t < n; ++t) dot += bar[t] * pi[t];
  double gs = 0.0;
  for (int t = 0; t < n; ++t) {
    bar[t] = (pi[t] * (bar[t] - dot)) * k;
    gs += bar[t];
  }
  for (int t = 0; t < n; ++t) bar[t] = bar[t] - exp(logz[t]) * gs;
}

/* Full-row merge draw for a row whose utilities are all -1e12 (no live
 * candidate): the reference softmaxes over every agent of A
 * (merge_choice, node_model.cpp:99-120).  Returns the winning agent id. */
static int full_row_argmax(Ctx* c, int t, int row) {
  const int n = c->nA;
  double* v = xcalloc(n, sizeof(double));
  double* g = xcalloc(n, sizeof(double));
  double* lz = xcalloc(n, sizeof(double));
  double* pi = xcalloc(n, sizeof(double));
  for (int s = 0; s < n; ++s) {
    v[s] = 0.0 - MASK_LARGE; /* sub(p, mask) with p == 0 */
    g[s] = port_gumbel(c->seed_merge, (uint64_t)t, (uint64_t)row, (uint64_t)c->A[s]);
  }
  const int best = two_softmax(n, v, g, c->k, lz, pi);
  free(v);
  free(g);
  free(lz);
  free(pi);
  return c->A[best];
}

/* engine_step (src/engine.cpp:70-125): f on every link, counting, g.
 * In: link/pos (state at start of step t), qprev.  Out: link_new/pos_new,
 * cum updated in place, q in c->q.  Returns 0, or -2 for an unsupported
 * zero merge priority. */
static int step_forward(Ctx* c, int t, const int* link, const double* pos,
                        const double* qprev, double* cum, int* link_new,
                        double* pos_new) {
  const port_net* net = c->net;
  const port_params* p = c->p;
  const int L = c->L, N = c->N;
  const double M = c->M;

  /* agents_on[j], ascending id (engine.cpp:76-82) */
  memset(c->cnt, 0, sizeof(int) * L);
  for (int i = 0; i < N; ++i)
    if (link[i] >= 0 && pos[i] >= VALID_THR) c->cnt[link[i]]++;
  c->off[0] = 0;
  for (int j = 0; j < L; ++j) c->off[j + 1] = c->off[j] + c->cnt[j];
  memset(c->cnt, 0, sizeof(int) * L);
  for (int i = 0; i < N; ++i)
    if (link[i] >= 0 && pos[i] >= VALID_THR) {
      const int j = link[i];
      c->ids[c->off[j] + c->cnt[j]++] = i;
    }
  /* stable descending sort per link (headways, car_following.cpp:537) */
  memcpy(c->seg, c->ids, sizeof(int) * c->off[L]);
  for (int j = 0; j < L; ++j) {
    int* s = c->seg + c->off[j];
    for (int r = 1; r < c->cnt[j]; ++r) {
      const int key = s[r];
      int m = r - 1;
      while (m >= 0 && pos[s[m]] < pos[key]) {
        s[m + 1] = s[m];
        --m;
      }
      s[m + 1] = key;
    }
  }

  for (int i = 0; i < N; ++i) c->x1[i] = pos[i];
  /* f + midpoint counting per link (car_following.cpp:128-157,
   * headways :96-126, observation.cpp:9-20) */
  for (int j = 0; j < L; ++j) {
    c->q[j] = 0.0;
    if (!c->cnt[j]) continue;
    const double u = p->u[j], kap = p->kappa[j], len = net->length[j];
    const double dxf = (1.0 * u) * c->dt;
    const double jam = (double)net->delta_n / kap;
    const double o = 0.5 * len; /* engine.cpp:47 */
    const int* s = c->seg + c->off[j];
    double qsum = 0.0;
    for (int r = 0; r < c->cnt[j]; ++r) {
      const int i = s[r];
      const double x = pos[i];
      /* leader: diff*0 + M == M exactly (car_following.cpp:552-553) */
      const double h = r == 0 ? M : (pos[s[r - 1]] - x);
      const double gp = h - jam;
      const double dxc = (gp >= 0.0 ? gp : 0.0) * 1.0;
      const unsigned char pc = dxc <= dxf;
      const double xp = x + (pc ? dxc : dxf);
      const unsigned char pk = xp <= len;
      c->x1[i] = pk ? xp : len;
      c->gap[i] = gp;
      c->pick_cong[i] = pc;
      c->pick_cap[i] = pk;
    }
    for (int r = 0; r < c->cnt[j]; ++r) /* reduce_sum over the gathered column */
      qsum += (c->x1[c->ids[c->off[j] + r]] >= o ? 1.0 : 0.0) * 1.0;
    c->q[j] = qsum;
  }
  /* inc = relu(q - qprev); cum += inc (engine.cpp:111-113) */
  for (int j = 0; j < L; ++j) {
    c->a[j] = c->q[j] - qprev[j];
    cum[j] = cum[j] + (c->a[j] >= 0.0 ? c->a[j] : 0.0);
  }

  /* node_step (node_model.cpp:151-181) */
  c->nA = 0;
  for (int i = 0; i < N; ++i) {
    c->aidx[i] = -1;
    c->admitted[i] = -1;
    if (link[i] < 0 || c->x1[i] < VALID_THR) continue;
    if (c->x1[i] >= net->length[link[i]] - ARRIVAL_TOL) {
      c->aidx[i] = c->nA;
      c->A[c->nA++] = i;
    }
  }
  for (int j = 0; j < L; ++j) c->winner[j] = -1;
  memcpy(link_new, link, sizeof(int) * N);
  memcpy(pos_new, c->x1, sizeof(double) * N);
  if (c->nA == 0) return 0;

  /* vacancy_from_state over the post-f state (node_model.cpp:27-41) */
  for (int j = 0; j < L; ++j) {
    double mn = M;
    for (int r = 0; r < c->cnt[j]; ++r) {
      const double x = c->x1[c->seg[c->off[j] + r]];
      if (x >= VALID_THR && x < mn) mn = x;
    }
    c->vacant[j] = mn > net->delta_n / p->kappa[j] ? 1.0 : 0.0;
  }

  /* link_choice (node_model.cpp:45-97) for every n in A */
  double v[256], g[256];
  for (int s = 0; s < c->nA; ++s) {
    const int n = c->A[s], cl = link[n];
    const int b = net->succ_off[cl], d = net->succ_off[cl + 1] - b;
    c->choice[s] = -1;
    if (d == 0) continue; /* unconnected: row of l is all zero */
    for (int e = 0; e < d; ++e) {
      const int j = net->succ[b + e];
      v[e] = p->beta[j] / p->cost[j]; /* pref = beta / cost, :55 */
      g[e] = port_gumbel(c->seed_link, (uint64_t)t, (uint64_t)n, (uint64_t)j);
    }
    const int best = two_softmax(d, v, g, c->k, c->logz + (size_t)s * c->maxdeg,
                                 c->pi + (size_t)s * c->maxdeg);
    c->choice[s] = net->succ[b + best];
  }

  /* merge_choice (node_model.cpp:99-120): candidates per row, ascending id */
  memset(c->cand_off, 0, sizeof(int) * (L + 1));
  for (int s = 0; s < c->nA; ++s) {
    const int d = c->choice[s];
    if (d >= 0 && c->vacant[d] != 0.0) c->cand_off[d + 1]++;
  }
  for (int j = 0; j < L; ++j) c->cand_off[j + 1] += c->cand_off[j];
  memset(c->cnt, 0, sizeof(int) * L); /* reuse as fill cursor */
  for (int s = 0; s < c->nA; ++s) {
    const int d = c->choice[s];
    if (d >= 0 && c->vacant[d] != 0.0) c->cand[c->cand_off[d] + c->cnt[d]++] = c->A[s];
  }
  double* mv = xcalloc(c->nA, sizeof(double));
  double* mg = xcalloc(c->nA, sizeof(double));
  for (int i = 0; i < L; ++i) {
    const int b = c->cand_off[i], n = c->cand_off[i + 1] - b;
    c->row_live[i] = 0;
    if (n == 0) continue;
    for (int e = 0; e < n; ++e) {
      const int ag = c->cand[b + e];
      mv[e] = p->alpha[link[ag]]; /* p = l * matmul(valid, alpha) */
      if (mv[e] == 0.0) {
        free(mv);
        free(mg);
        snprintf(g_err, sizeof g_err,
                 "zero merge priority (alpha) on link %d is not supported", link[ag]);
        return -2;
      }
      mg[e] = port_gumbel(c->seed_merge, (uint64_t)t, (uint64_t)i, (uint64_t)ag);
    }
    const int best = two_softmax(n, mv, mg, c->k, c->mlogz + b, c->mpi + b);
    c->winner[i] = c->cand[b + best];
    c->row_live[i] = 1;
  }
  free(mv);
  free(mg);

  /* transfer (node_model.cpp:122-149): winner -> (i, 0.0 exactly) */
  for (int i = 0; i < L; ++i) {
    const int w = c->winner[i];
    if (w < 0) continue;
    c->admitted[w] = i;
    link_new[w] = i;
    pos_new[w] = 0.0;
  }
  return 0;
}

/* initial_counts (engine.cpp:127-135) */
static void initial_counts(const Ctx* c, const int* link, const double* pos,
                           double* q0) {
  for (int j = 0; j < c->L; ++j) q0[j] = 0.0;
  for (int i = 0; i < c->N; ++i)
    if (link[i] >= 0 && pos[i] >= VALID_THR &&
        pos[i] >= 0.5 * c->net->length[link[i]])
      q0[link[i]] += 1.0;
}

static int validate_state(const Ctx* c, const int* link, const double* pos) {
  for (int i = 0; i < c->N; ++i) {
    if (link[i] < 0 || link[i] >= c->L) {
      snprintf(g_err, sizeof g_err, "agent placed on a link that does not exist");
      return -1;
    }
    if (!(pos[i] >= VALID_THR)) {
      snprintf(g_err, sizeof g_err,
               "agent %d: position %g is below the validity threshold", i, pos[i]);
      return -1;
    }
  }
  return 0;
}

int port_forward(const port_net* net, const port_params* p, uint64_t root_seed,
                 uint64_t noise_iteration, int n_agents, const int* link0,
                 const double* pos0, int T, double* cum_per_step, int* link_out,
                 double* pos_out, int* states_link, double* states_pos) {
  Ctx c;
  ctx_init(&c, net, p, n_agents, root_seed, noise_iteration);
  int rc = validate_state(&c, link0, pos0);
  const int L = c.L, N = c.N;
  int* lk[2] = {xcalloc(N, sizeof(int)), xcalloc(N, sizeof(int))};
  double* ps[2] = {xcalloc(N, sizeof(double)), xcalloc(N, sizeof(double))};
  double* qprev = xcalloc(L, sizeof(double));
  double* cum = xcalloc(L, sizeof(double));
  if (rc) goto done;
  memcpy(lk[0], link0, sizeof(int) * N);
  memcpy(ps[0], pos0, sizeof(double) * N);
  initial_counts(&c, lk[0], ps[0], qprev);
  for (int t = 0; t < T; ++t) { /* engine.cpp:244-248 */
    const int a = t & 1, b = a ^ 1;
    rc = step_forward(&c, t, lk[a], ps[a], qprev, cum, lk[b], ps[b]);
    if (rc) goto done;
    memcpy(qprev, c.q, sizeof(double) * L);
    memcpy(cum_per_step + (size_t)t * L, cum, sizeof(double) * L);
    if (states_link) {
      memcpy(states_link + (size_t)t * N, lk[b], sizeof(int) * N);
      memcpy(states_pos + (size_t)t * N, ps[b], sizeof(double) * N);
    }
  }
  memcpy(link_out, lk[T & 1], sizeof(int) * N);
  memcpy(pos_out, ps[T & 1], sizeof(double) * N);
done:
  free(lk[0]);
  free(lk[1]);
  free(ps[0]);
  free(ps[1]);
  free(qprev);
  free(cum);
  ctx_free(&c);
  return rc;
}

/* Slot of link `dst` in the (ascending) successor list of `src`, or -1. */
static int succ_slot(const port_net* net, int src, int dst) {
  for (int e = net->succ_off[src]; e < net->succ_off[src + 1]; ++e)
    if (net->succ[e] == dst) return e - net->succ_off[src];
  return -1;
}

/* Reverse sweep of one engine_step (the per-step segment VJP of
 * engine.cpp:388-415, i.e. Tape::vjp tensor.cpp:715-996 applied to the ops of
 * engine_step / node_step / link_choice / merge_choice / transfer /
 * car_following_step / headways / midpoint_count).  Requires step_forward(t)
 * to have just run on the checkpoint of step t.
 * xbar: in = adjoint of positions after step t (per agent), out = before.
 * cbar: cumulative-count adjoint (passes through).  qbar: in = adjoint of q_t,
 * out = adjoint of qprev_t.  g5: per-step gradients are ADDED (accumulate,
 * engine.cpp:296-299). */
static void step_backward(Ctx* c, const int* link, const double* pos,
                          const double* qprev, double* xbar, const double* cbar,
                          double* qbar, double* g5, int t) {
  const port_net* net = c->net;
  const port_params* p = c->p;
  const int L = c->L, N = c->N, W = c->maxdeg;
  const double M = c->M;
  double* gu = g5;
  double* gk = g5 + L;
  double* gb = g5 + 2 * L;
  double* ga = g5 + 3 * L;
  double* gc = g5 + 4 * L;
  (void)qprev;

  double* xbar1 = xcalloc(N, sizeof(double));
  memcpy(xbar1, xbar, sizeof(double) * N);

  if (c->nA > 0) {
    /* transfer VJP (node_model.cpp:122-149): admitted-sum adjoint of every
     * non-admitted arrived agent: x_bar*(-M) + (-(x_bar*x1)) */
    for (int s = 0; s < c->nA; ++s) {
      const int n = c->A[s];
      double r = 0.0;
      if (c->admitted[n] < 0) {
        r += xbar[n] * (-M);
        r += -1.0 * (xbar[n] * c->x1[n]);
      }
      c->admbar[n] = r;
      c->prio_bar[s] = 0.0;
      for (int e = 0; e < W; ++e) c->lbar[(size_t)s * W + e] = 0.0;
    }
    const int a0 = c->A[0];
    const int a0_link = link[a0];
    /* merge_choice VJP, row by row */
    double* bar = xcalloc(c->nA, sizeof(double));
    for (int i = 0; i < L; ++i) {
      const int w = c->winner[i];
      if (w >= 0) {
        const int b = c->cand_off[i], n = c->cand_off[i + 1] - b;
        const double abar_w = xbar[w] * M + 0.0;
        /* targeted = reduce_max(l, rows) routes to the first candidate */
        const int r0 = c->cand[b];
        c->lbar[(size_t)c->aidx[r0] * W + succ_slot(net, link[r0], i)] += abar_w;
        for (int e = 0; e < n; ++e) {
          const int ag = c->cand[b + e];
          bar[e] = (ag == w ? abar_w : c->admbar[ag]) * 1.0;
        }
        two_softmax_vjp(n, c->mlogz + b, c->mpi + b, c->k, bar);
        for (int e = 0; e < n; ++e) {
          const int ag = c->cand[b + e];
          const int s = c->aidx[ag];
          c->lbar[(size_t)s * W + succ_slot(net, link[ag], i)] +=
              bar[e] * p->alpha[link[ag]];
          c->prio_bar[s] += bar[e] * 1.0;
        }
      } else {
        /* non-targeted row: the max over an all-zero column routes to A[0];
         * only successors of A[0]'s link with a vacancy can carry it */
        const int slot = succ_slot(net, a0_link, i);
        if (slot < 0 || c->vacant[i] == 0.0) continue;
        const int wf = full_row_argmax(c, t, i);
        double ab;
        if (c->admitted[wf] >= 0)
          ab = 0.0 * M + 0.0;
        else
          ab = (i == link[wf] ? xbar[wf] * M : 0.0 * M) + c->admbar[wf];
        c->lbar[(size_t)0 * W + slot] += ab;
      }
    }
    free(bar);
    /* alpha: prio = matmul(valid, alpha), VJP summed over A ascending */
    for (int j = 0; j < L; ++j) c->alpha_bar[j] = 0.0;
    for (int s = 0; s < c->nA; ++s) c->alpha_bar[link[c->A[s]]] += 1.0 * c->prio_bar[s];
    /* link_choice VJP (node_model.cpp:45-97) -> pref_bar */
    for (int j = 0; j < L; ++j) c->pref_bar[j] = 0.0;
    double pb[256];
    for (int s = 0; s < c->nA; ++s) {
      if (c->choice[s] < 0) continue;
      const int cl = link[c->A[s]];
      const int b = net->succ_off[cl], d = net->succ_off[cl + 1] - b;
      for (int e = 0; e < d; ++e)
        pb[e] = ((c->lbar[(size_t)s * W + e] * 1.0) * 1.0) * c->vacant[net->succ[b + e]];
      two_softmax_vjp(d, c->logz + (size_t)s * W, c->pi + (size_t)s * W, c->k, pb);
      for (int e = 0; e < d; ++e) c->pref_bar[net->succ[b + e]] += pb[e] * 1.0;
    }
    /* pref = beta / cost (divide VJP, tensor.cpp:764-777) */
    for (int j = 0; j < L; ++j) {
      gb[j] += 0.0 + c->pref_bar[j] / p->cost[j];
      gc[j] += 0.0 - c->pref_bar[j] * p->beta[j] / (p->cost[j] * p->cost[j]);
      ga[j] += c->alpha_bar[j];
    }
    /* position adjoint through transfer + replace_rows: movers carry their
     * new-position adjoint back to the old position only with TG */
    for (int s = 0; s < c->nA; ++s) {
      const int n = c->A[s];
      if (c->admitted[n] >= 0 && !net->trajectory_grafting) xbar1[n] = 0.0;
    }
  }

  /* counting + f VJP per link, sums in gather (ascending id) order */
  for (int j = 0; j < L; ++j) {
    const int cnt = c->off[j + 1] - c->off[j];
    const unsigned char pick = c->a[j] >= 0.0;
    const double qb = qbar[j] + (pick ? cbar[j] : 0.0);
    qbar[j] = pick ? -1.0 * cbar[j] : 0.0; /* adjoint of qprev */
    if (!cnt) continue;
    const double len = net->length[j], o = 0.5 * len, sc = 5.0 / len;
    const double kap = p->kappa[j];
    const int* s = c->seg + c->off[j];
    /* pass 1 (sorted order): x'bar and h_bar per agent */
    double* hb = c->gap; /* reuse: overwrite gap with h_bar after use */
    for (int r = 0; r < cnt; ++r) {
      const int n = s[r];
      double x1b = xbar1[n];
      if (qb != 0.0) {
        const double z = (c->x1[n] + (-o)) * sc;
        const double sg = z >= 0.0 ? 1.0 / (1.0 + exp(-z)) : exp(z) / (1.0 + exp(z));
        x1b = x1b + (((qb * 1.0) * sg) * (1.0 - sg)) * sc;
      }
      const double xpb = net->trajectory_grafting ? x1b : (c->pick_cap[n] ? x1b : 0.0);
      const double gp = c->gap[n];
      const double dxcb = c->pick_cong[n] ? xpb : 0.0;
      const double dxfb = c->pick_cong[n] ? 0.0 : xpb;
      const double gapb = gp >= 0.0 ? dxcb * 1.0 : 0.0;
      c->x1[n] = xpb;       /* reuse: x1 -> x'bar (x1 no longer needed) */
      hb[n] = gapb;         /* h_bar = gap_bar */
      c->admbar[n] = dxfb;  /* reuse: dx_free bar */
    }
    /* pass 2: parameter sums in gather order */
    double ub = 0.0, jb = 0.0;
    for (int r = 0; r < cnt; ++r) {
      const int n = c->ids[c->off[j] + r];
      ub += (c->admbar[n] * c->dt) * 1.0;
      jb += -1.0 * hb[n];
    }
    gu[j] += 0.0 + ub;
    gk[j] += 0.0 - jb * (double)net->delta_n / (kap * kap);
    /* pass 3: position adjoint = x'bar + (follower's h_bar - own h_bar) */
    for (int r = 0; r < cnt; ++r) {
      const int n = s[r];
      double tb = 0.0;
      if (r + 1 < cnt) tb += hb[s[r + 1]] * 1.0;
      if (r > 0) tb += -(hb[n] * 1.0);
      xbar[n] = c->x1[n] + tb * 1.0;
    }
  }
  free(xbar1);
}

static void loss_and_seeds(int L, int N, int K, const double* snaps,
                           const double* cum_final, const int* link_final,
                           const double* pos_final, const double* ws,
                           const double* qs, const double* wc, const double* qc,
                           const double* wx, double* loss, double* snap_seed,
                           double* cum_seed, double* x_seed) {
  /* loss: the builder of oracle/ref_shim.cpp:ref_gradient, in its op order */
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    const double* s = snaps + (size_t)k * L;
    if (ws) {
      double r = 0.0;
      for (int j = 0; j < L; ++j) r += s[j] * ws[(size_t)k * L + j];
      acc = acc + r;
    }
    if (qs) {
      double r = 0.0;
      for (int j = 0; j < L; ++j) r += (s[j] * s[j]) * (qs[(size_t)k * L + j] * 0.5);
      acc = acc + r;
    }
    for (int j = 0; j < L; ++j) {
      double sd = 0.0;
      if (qs) sd = (qs[(size_t)k * L + j] * s[j]);
      if (ws) sd = sd + ws[(size_t)k * L + j];
      snap_seed[(size_t)k * L + j] = sd;
    }
  }
  if (wc) {
    double r = 0.0;
    for (int j = 0; j < L; ++j) r += cum_final[j] * wc[j];
    acc = acc + r;
  }
  if (qc) {
    double r = 0.0;
    for (int j = 0; j < L; ++j) r += (cum_final[j] * cum_final[j]) * (qc[j] * 0.5);
    acc = acc + r;
  }
  for (int j = 0; j < L; ++j) {
    double sd = 0.0;
    if (qc) sd = qc[j] * cum_final[j];
    if (wc) sd = sd + wc[j];
    cum_seed[j] = sd;
  }
  if (wx) {
    double r = 0.0;
    for (int n = 0; n < N; ++n)
      if (link_final[n] >= 0) r += pos_final[n] * wx[n];
    acc = acc + r;
  }
  for (int n = 0; n < N; ++n) x_seed[n] = wx ? wx[n] : 0.0;
  *loss = acc;
}

static int gradient_impl(const port_net* net, const port_params* p,
                         uint64_t root_seed, uint64_t noise_iteration, int N,
                         const int* link0, const double* pos0, int T, int spi,
                         const double* ws, const double* qs, const double* wc,
                         const double* qc, const double* wx,
                         const double* snap_seed_in, const double* cum_seed_in,
                         const double* x_seed_in, double* loss, double* grads,
                         double* snaps_out, int* n_snaps, double* cum_final,
                         int* link_out, double* pos_out) {
  Ctx c;
  ctx_init(&c, net, p, N, root_seed, noise_iteration);
  int rc = validate_state(&c, link0, pos0);
  const int L = c.L;
  const int K = spi > 0 ? T / spi : 0;
  int* ck_link = xcalloc((size_t)(T + 1) * N, sizeof(int));
  double* ck_pos = xcalloc((size_t)(T + 1) * N, sizeof(double));
  double* ck_q = xcalloc((size_t)(T + 1) * L, sizeof(double));
  double* cum = xcalloc(L, sizeof(double));
  double* snaps = xcalloc((size_t)(K + 1) * L, sizeof(double));
  double* snap_seed = xcalloc((size_t)(K + 1) * L, sizeof(double));
  double* cum_seed = xcalloc(L, sizeof(double));
  double* x_seed = xcalloc(N, sizeof(double));
  double* xbar = xcalloc(N, sizeof(double));
  double* cbar = xcalloc(L, sizeof(double));
  double* qbar = xcalloc(L, sizeof(double));
  if (rc) goto done;
  if (spi < 1) {
    snprintf(g_err, sizeof g_err,
             "observation interval must be a positive multiple of the time step");
    rc = -1;
    goto done;
  }
  memcpy(ck_link, link0, sizeof(int) * N);
  memcpy(ck_pos, pos0, sizeof(double) * N);
  initial_counts(&c, link0, pos0, ck_q);
  int ks = 0;
  for (int t = 0; t < T; ++t) { /* forward storing compact checkpoints, :357-364 */
    rc = step_forward(&c, t, ck_link + (size_t)t * N, ck_pos + (size_t)t * N,
                      ck_q + (size_t)t * L, cum, ck_link + (size_t)(t + 1) * N,
                      ck_pos + (size_t)(t + 1) * N);
    if (rc) goto done;
    memcpy(ck_q + (size_t)(t + 1) * L, c.q, sizeof(double) * L);
    if ((t + 1) % spi == 0) memcpy(snaps + (size_t)ks++ * L, cum, sizeof(double) * L);
  }
  if (n_snaps) *n_snaps = ks;
  if (snaps_out) memcpy(snaps_out, snaps, sizeof(double) * (size_t)ks * L);
  if (cum_final) memcpy(cum_final, cum, sizeof(double) * L);
  if (link_out) memcpy(link_out, ck_link + (size_t)T * N, sizeof(int) * N);
  if (pos_out) memcpy(pos_out, ck_pos + (size_t)T * N, sizeof(double) * N);

  if (snap_seed_in) {
    memcpy(snap_seed, snap_seed_in, sizeof(double) * (size_t)ks * L);
    memcpy(cum_seed, cum_seed_in, sizeof(double) * L);
    memcpy(x_seed, x_seed_in, sizeof(double) * N);
  } else {
    double lv = 0.0;
    loss_and_seeds(L, N, ks, snaps, cum, ck_link + (size_t)T * N,
                   ck_pos + (size_t)T * N, ws, qs, wc, qc, wx, &lv, snap_seed,
                   cum_seed, x_seed);
    if (loss) *loss = lv;
  }

  memset(grads, 0, sizeof(double) * 5 * L);
  memcpy(xbar, x_seed, sizeof(double) * N);
  memcpy(cbar, cum_seed, sizeof(double) * L);
  int snap_idx = ks - 1;
  for (int t = T - 1; t >= 0; --t) { /* reverse sweep, engine.cpp:389-415 */
    if (snap_idx >= 0 && (t + 1) % spi == 0) {
      for (int j = 0; j < L; ++j) cbar[j] += snap_seed[(size_t)snap_idx * L + j];
      --snap_idx;
    }
    double* cum_scratch = xcalloc(L, sizeof(double));
    int* lk_scratch = xcalloc(N, sizeof(int));
    double* ps_scratch = xcalloc(N, sizeof(double));
    rc = step_forward(&c, t, ck_link + (size_t)t * N, ck_pos + (size_t)t * N,
                      ck_q + (size_t)t * L, cum_scratch, lk_scratch, ps_scratch);
    free(cum_scratch);
    free(lk_scratch);
    free(ps_scratch);
    if (rc) goto done;
    step_backward(&c, ck_link + (size_t)t * N, ck_pos + (size_t)t * N,
                  ck_q + (size_t)t * L, xbar, cbar, qbar, grads, t);
  }
done:
  free(ck_link);
  free(ck_pos);
  free(ck_q);
  free(cum);
  free(snaps);
  free(snap_seed);
  free(cum_seed);
  free(x_seed);
  free(xbar);
  free(cbar);
  free(qbar);
  ctx_free(&c);
  return rc;
}

int port_gradient(const port_net* net, const port_params* p,
                  uint64_t root_seed, uint64_t noise_iteration, int n_agents,
                  const int* link0, const double* pos0, int T, int spi,
                  const double* ws, const double* qs, const double* wc,
                  const double* qc, const double* wx, double* loss,
                  double* grads, double* snaps, int* n_snaps,
                  double* cum_final, int* link_out, double* pos_out) {
  return gradient_impl(net, p, root_seed, noise_iteration, n_agents, link0,
                       pos0, T, spi, ws, qs, wc, qc, wx, NULL, NULL, NULL, loss,
                       grads, snaps, n_snaps, cum_final, link_out, pos_out);
}

int port_gradient_seeds(const port_net* net, const port_params* p,
                        uint64_t root_seed, uint64_t noise_iteration,
                        int n_agents, const int* link0, const double* pos0,
                        int T, int spi, const double* snap_seed,
                        const double* cum_seed, const double* x_seed,
                        double* grads) {
  return gradient_impl(net, p, root_seed, noise_iteration, n_agents, link0,
                       pos0, T, spi, NULL, NULL, NULL, NULL, NULL, snap_seed,
                       cum_seed, x_seed, NULL, grads, NULL, NULL, NULL, NULL,
                       NULL);
}
