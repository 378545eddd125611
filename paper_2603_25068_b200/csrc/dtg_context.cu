// Level-1 C-ABI: the device engine context (include/dtg.h).
//
// Owns all device memory for B scenarios, the CUDA stream and the cached
// CUDA graphs of the whole T-step forward and reverse sweeps (one graph launch
// per simulate call instead of 4T / 8T kernel launches).
#include <algorithm>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dtg.h"
#include "dtg_kernels.h"
#include "dtg_cluster.h"
#include "dtg_backward.h"
#include "dtg_loss.h"
#include "dtg_device.cuh"

namespace dtg {
cudaError_t decision_stats_fused(int force, unsigned long long* count);
cudaError_t decision_stats_backward(int force, unsigned long long* count);
cudaError_t decision_stats_kernels(int force, unsigned long long* count);
cudaError_t decision_stats_scn(int force, unsigned long long* count);
}  // namespace dtg

namespace {

thread_local std::string g_create_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess)                                                     \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

// The stream the running C-ABI call's buffer (re)allocations are ordered on:
// inside a call on a context (guarded), its stream.  Buffers then come from
// the stream-ordered allocator (cudaMallocAsync / cudaFreeAsync on the
// device's default pool, kept reserved: see reserve_pool) -- growing a
// context for a longer horizon or more agents costs neither an implicit
// device synchronisation (cudaFree) nor an OS round trip.  Outside a call
// (context destruction) buffers are freed synchronously.
thread_local cudaStream_t* tl_alloc_stream = nullptr;
struct AllocScope {
  cudaStream_t* prev;
  explicit AllocScope(cudaStream_t* s) : prev(tl_alloc_stream) { tl_alloc_stream = s; }
  ~AllocScope() { tl_alloc_stream = prev; }
};

// Keep freed pool memory reserved for reuse instead of returning it to the
// OS at every synchronisation (the pool's default release threshold is 0).
void reserve_pool() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    std::uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

// Page-locked host memory (cudaHostAlloc / cudaHostRegister): copies into it
// can be DMA'd directly, without pinned staging.
bool pinned_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  std::size_t n = 0;
  bool pooled = false;
  void alloc(std::size_t count) {
    release();
    if (count) {
      if (tl_alloc_stream) {
        CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), *tl_alloc_stream));
        pooled = true;
      } else {
        CK(cudaMalloc(&p, count * sizeof(T)));
      }
    }
    n = count;
  }
  bool ensure(std::size_t count) {
    if (count <= n) return false;
    alloc(count);
    return true;
  }
  void release() {
    if (p) {
      // stream-ordered after the work already queued on the context's stream
      if (pooled && tl_alloc_stream)
        cudaFreeAsync(p, *tl_alloc_stream);
      else
        cudaFree(p);
    }
    p = nullptr;
    n = 0;
    pooled = false;
  }
  ~DevBuf() { release(); }
};

}  // namespace

struct dtg_ctx {
  int L = 0, N = 0, B = 0, maxdeg = 1;
  dtg_sim_config cfg{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool graphs = true;
  int force_slow = 0;
  std::string err;
  // static network
  DevBuf<int> succ_off, succ, pred_off, pred, pred_pos, succ_pedge;
  int E = 0;
  DevBuf<double> len, thr, ctr, sc;
  // parameters / seeds
  DevBuf<double> params;  // [5][B][L]
  DevBuf<double> derived; // [3][B][L]
  DevBuf<std::uint64_t> seeds;  // [2][B]
  std::vector<std::uint64_t> h_seeds;
  std::vector<char> have_params, have_state;
  // transfer events (dtg_set_record_transfers): admitted agent per link and
  // step of the last forward, and each scenario's initial link per agent
  bool rec_transfers = false;
  DevBuf<int> ev;
  int ev_T = -1;
  std::vector<std::vector<int>> h_link0;
  // initial state
  DevBuf<double> pos0, q0;
  DevBuf<int> aid0, lnk0, off0;
  // history
  int S = 0, H = 0;
  DevBuf<double> pos, qh, cumh;
  DevBuf<int> aid, lnk, off;
  // scratch
  DevBuf<double> x1, tail;
  DevBuf<int> choice, won, qn, nA, win, dep, newcnt, a0, errf;
  DevBuf<unsigned char> vac;
  // adjoint
  DevBuf<double> cbar, qbar, qtot, lbar_row, prio_bar, vbar, lbar_a0, cu, cg,
      grads, xbar;
  DevBuf<double> snap_seed, cum_seed, x_seed;
  DevBuf<unsigned long long> sort_scratch;
  DevBuf<int> alist, acount;
  // persistent backward
  int bgrid_max = 0;
  bool bwd_persistent = true;
  DevBuf<double> bx1, btail, bmpi, bmlz, blpi;
  DevBuf<int> bnA, bnAc, bwon, bdep, bwin, bccnt, bched, bchoice, balist, bacount;
  DevBuf<unsigned char> bvac;
  DevBuf<dtg::Cand> bcands;
  DevBuf<unsigned long long> ba0key, bsort;
  DevBuf<unsigned char> ba0part;
  int last_bgrid = 0;
  DevBuf<int> tmp_link;
  DevBuf<double> tmp_pos;
  // last run
  int last_T = -1, last_spi = 1, last_ckpt = 0, last_K = 0;
  bool pending = false;
  std::int64_t launches = 0;
  // persistent forward
  bool persistent = true;
  int pgrid_max = 0;
  bool scn_ok = false;  // scenario-resident forward (mode 4) fits shared memory
  int n_sm = 0;
  DevBuf<double> x1b, tailb;
  DevBuf<int> wonb, nAb, qnb, depb, winp, ccnt, clist;
  int last_grid = 0;
  double* h_stage = nullptr;  // pinned staging for count read-back
  std::size_t h_stage_n = 0;
  // streamed read-back (dtg_forward_read): host-mapped step counter written by
  // the persistent kernel, a copy stream, pinned staging of the final state
  unsigned int* prog_h = nullptr;
  int stream_progress = 0;  // >0: next fused launch publishes progress every this many steps
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t par_ev = nullptr;
  double* h_par = nullptr;       // pinned parameter staging [5][L]
  DevBuf<double> d_par;          // its device copy (broadcast to the scenarios by a kernel)
  std::uint64_t* h_seed_pin = nullptr;  // pinned seed staging [2][B]
  cudaEvent_t seed_ev = nullptr;
  void* h_fin = nullptr;         // pinned final state: int link[B*N] | double pos[B*N]
  std::size_t h_fin_n = 0;
  int mode = 0;          // 0 auto, 1 cluster, 2 grid-persistent, 3 step graph, 4 scenario CTAs
  int cluster_cs_max = 0;
  bool stage_params = false;
  int last_mode = 0, last_cs = 0;
  DevBuf<double> srec;
  DevBuf<dtg::Spec> spec;  // speculative head decisions [2][B][L][2]
  bool speculate = true;
  int cs_override = 0;  // flag 7: CTAs per scenario of the grid schedule (0 auto)
  int graph_split = 0;  // flag 8: scenario branches of the step graph (0 auto)
  std::vector<cudaStream_t> side;  // step-graph branch streams
  cudaEvent_t fork_ev = nullptr;
  std::vector<cudaEvent_t> join_ev;
  bool spec_split = true;  // flag 5
  DevBuf<unsigned int> gbar, bgbar;
  bool custom_barrier = true;
  int contig_mode = -1;
  int bwd_dbg = 0;  // timing experiments only
  int fwd_dbg = 0;  // timing experiments only  // -1 auto, 0 interleaved, 1 contiguous (fused forward slot mapping)
  bool want_wstamp = false;
  DevBuf<unsigned long long> wst;
  DevBuf<dtg::Cand> cands;
  bool want_stamps = false;
  DevBuf<unsigned long long> stamps;
  // device losses (dtg_loss.h)
  int loss_kind = 0, loss_kobs = 0, loss_nobs = 0, loss_target = -1;
  double loss_desired = 0.0;
  DevBuf<int> loss_ids, loss_first, loss_next;
  DevBuf<double> loss_obs, loss_val, loss_extra, rows, red;
  double* h_red = nullptr;
  // device-resident calibrate step (dtg_opt_bounded_*): raw [4][L], the Adam
  // moments, the raw of the best iteration
  DevBuf<double> opt_raw, opt_m, opt_v, opt_best;
  double opt_lo[4] = {0, 0, 0, 0}, opt_hi[4] = {0, 0, 0, 0};
  double opt_lr = 0, opt_b1 = 0, opt_b2 = 0, opt_eps = 0, opt_wd = 0;
  bool opt_ready = false;
  // graphs
  cudaGraphExec_t fwd_exec = nullptr, bwd_exec = nullptr;
  long long fwd_key = -1, bwd_key = -1;

  dtg::DevView view() const {
    dtg::DevView d{};
    d.L = L;
    d.N = N;
    d.B = B;
    d.S = S;
    d.maxdeg = maxdeg;
    d.delta_n = cfg.delta_n;
    d.tg = cfg.trajectory_grafting ? 1 : 0;
    d.M = cfg.sentinel;
    d.dt = cfg.tau * cfg.delta_n;
    d.kinv = 1.0 / cfg.gumbel_tau;
    d.succ_off = succ_off.p;
    d.succ = succ.p;
    d.pred_off = pred_off.p;
    d.pred = pred.p;
    d.pred_pos = pred_pos.p;
    d.succ_pedge = succ_pedge.p;
    d.len = len.p;
    d.thr = thr.p;
    d.ctr = ctr.p;
    d.sc = sc.p;
    const std::size_t BL = static_cast<std::size_t>(B) * L;
    d.u = params.p;
    d.kappa = params.p + BL;
    d.beta = params.p + 2 * BL;
    d.alpha = params.p + 3 * BL;
    d.cost = params.p + 4 * BL;
    d.jam = derived.p;
    d.dxf = derived.p + BL;
    d.pref = derived.p + 2 * BL;
    d.slogz = srec.p;
    d.seed_link = seeds.p;
    d.seed_merge = seeds.p + B;
    d.pos = pos.p;
    d.aid = aid.p;
    d.lnk = lnk.p;
    d.off = off.p;
    d.qh = qh.p;
    d.cumh = cumh.p;
    d.x1 = x1.p;
    d.choice = choice.p;
    d.won = won.p;
    d.qn = qn.p;
    d.nA = nA.p;
    d.tail = tail.p;
    d.win = win.p;
    d.vac = vac.p;
    d.dep = dep.p;
    d.newcnt = newcnt.p;
    d.a0 = a0.p;
    d.err = errf.p;
    d.cbar = cbar.p;
    d.qbar = qbar.p;
    d.qtot = qtot.p;
    d.lbar_row = lbar_row.p;
    d.prio_bar = prio_bar.p;
    d.vbar = vbar.p;
    d.lbar_a0 = lbar_a0.p;
    d.cu = cu.p;
    d.cg = cg.p;
    d.grads = grads.p;
    d.ev = rec_transfers ? ev.p : nullptr;
    return d;
  }

  void drop_graphs() {
    if (fwd_exec) cudaGraphExecDestroy(fwd_exec);
    if (bwd_exec) cudaGraphExecDestroy(bwd_exec);
    fwd_exec = bwd_exec = nullptr;
    fwd_key = bwd_key = -1;
  }

  ~dtg_ctx() {
    drop_graphs();
    if (h_stage) cudaFreeHost(h_stage);
    if (h_red) cudaFreeHost(h_red);
    if (prog_h) cudaFreeHost(prog_h);
    if (h_par) cudaFreeHost(h_par);
    if (h_fin) cudaFreeHost(h_fin);
    if (par_ev) cudaEventDestroy(par_ev);
    if (h_seed_pin) cudaFreeHost(h_seed_pin);
    if (seed_ev) cudaEventDestroy(seed_ev);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    for (auto x : side) cudaStreamDestroy(x);
    for (auto e : join_ev) cudaEventDestroy(e);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  // Step-graph branches: independent scenario ranges run their T-step
  // chains side by side, so one range's kernel tails (the serial draw chains
  // of long queues in k_step_choice / k_step_merge) overlap the other's work.
  int graph_branches() const {
    if (graph_split > 0) return std::min(graph_split, B);
    // measured (C3, ms per nowcast, 1 / 2 / 4 branches): B=32 -- / 5.12 / 5.05,
    // B=64 8.12 / 7.63 / 7.41, B=128 14.73 / 13.30 / 13.04, B=256 27.30 /
    // 26.16 / 26.04 (8 branches 27.46)
    return B >= 32 ? 4 : (B >= 8 ? 2 : 1);
  }
  template <class F>
  void fork_branches(int nsp, cudaStream_t st, F&& run) {
    if (nsp <= 1) {
      run(0, B, st);
      return;
    }
    while (static_cast<int>(side.size()) < nsp - 1) {
      cudaStream_t x;
      cudaEvent_t e;
      CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      side.push_back(x);
      join_ev.push_back(e);
    }
    if (!fork_ev) CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(fork_ev, st));
    for (int q = 1; q < nsp; ++q) CK(cudaStreamWaitEvent(side[q - 1], fork_ev, 0));
    for (int q = 0; q < nsp; ++q) {
      const int b0 = static_cast<int>(static_cast<long long>(q) * B / nsp);
      const int b1 = static_cast<int>(static_cast<long long>(q + 1) * B / nsp);
      run(b0, b1 - b0, q ? side[q - 1] : st);
    }
    for (int q = 1; q < nsp; ++q) {
      CK(cudaEventRecord(join_ev[q - 1], side[q - 1]));
      CK(cudaStreamWaitEvent(st, join_ev[q - 1], 0));
    }
  }

  void ensure_history(int T, int ckpt) {
    const int s_need = ckpt ? T + 1 : 2;
    const int h_need = T + 1;
    bool realloc = false;
    if (rec_transfers && ev.ensure(static_cast<std::size_t>(std::max(T, 1)) * B * L)) realloc = true;
    ev_T = rec_transfers ? T : -1;
    if (s_need > S) {
      const std::size_t BN = static_cast<std::size_t>(B) * N;
      pos.alloc(BN * s_need);
      aid.alloc(BN * s_need);
      lnk.alloc(BN * s_need);
      off.alloc(static_cast<std::size_t>(B) * (L + 1) * s_need);
      S = s_need;
      realloc = true;
    }
    if (h_need > H) {
      qh.alloc(static_cast<std::size_t>(B) * L * h_need);
      cumh.alloc(static_cast<std::size_t>(B) * L * h_need);
      H = h_need;
      realloc = true;
    }
    if (realloc) drop_graphs();
  }

  // Wait for the stream and turn device error flags into exceptions.
  void sync_check() {
    CK(cudaStreamSynchronize(stream));
    if (!pending) return;
    pending = false;
    std::vector<int> e(B);
    CK(cudaMemcpy(e.data(), errf.p, sizeof(int) * B, cudaMemcpyDeviceToHost));
    check_flags(e.data());
  }
  void check_flags(const int* e) const {
    for (int b = 0; b < B; ++b) {
      if (e[b] & dtg::kErrCandOverflow)
        throw Unsupported("more merge candidates for one link in one step than the schedule holds (16 in the "
                          "persistent kernels, 32 in the step graph; scenario " +
                          std::to_string(b) + ")");
      if (e[b] & dtg::kErrZeroAlpha)
        throw Unsupported("zero merge priority (alpha) on a candidate link is not supported");
      if (e[b] & dtg::kErrConservation)
        throw std::runtime_error("agent conservation violated on the device (scenario " +
                                 std::to_string(b) + ")");
    }
  }
};

namespace {

int fail(dtg_ctx* c, int code, const std::string& msg) {
  if (c)
    c->err = msg;
  else
    g_create_error = msg;
  return code;
}

template <class F>
int guarded(dtg_ctx* c, F&& f) {
  AllocScope scope(c ? &c->stream : tl_alloc_stream);
  try {
    f();
    return DTG_OK;
  } catch (const CudaError& e) {
    return fail(c, DTG_ERR_CUDA, e.what());
  } catch (const Unsupported& e) {
    return fail(c, DTG_ERR_UNSUPPORTED, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(c, DTG_ERR_CONFIG, e.what());
  } catch (const std::exception& e) {
    return fail(c, DTG_ERR_RUNTIME, e.what());
  }
}

template <class T>
void h2d(DevBuf<T>& dst, const std::vector<T>& src, cudaStream_t st) {
  dst.alloc(src.size());
  if (!src.empty())
    CK(cudaMemcpyAsync(dst.p, src.data(), src.size() * sizeof(T),
                       cudaMemcpyHostToDevice, st));
}

// Link-segmented slot layout of one compact state (see dtg_device.cuh).
void build_layout(int N, int L, const int* link, const double* pos,
                  const std::vector<double>& length, std::vector<double>& ps,
                  std::vector<int>& aid, std::vector<int>& lnk,
                  std::vector<int>& off, std::vector<double>& q0) {
  std::vector<int> cnt(L, 0);
  for (int i = 0; i < N; ++i) {
    if (link[i] < 0 || link[i] >= L)
      throw std::runtime_error("agent placed on a link that does not exist");
    if (!(pos[i] >= dtg::kValidThr))
      throw Unsupported("agent " + std::to_string(i) + " position " +
                        std::to_string(pos[i]) +
                        " is below the validity threshold -0.01");
    ++cnt[link[i]];
  }
  off.assign(L + 1, 0);
  for (int j = 0; j < L; ++j) off[j + 1] = off[j] + cnt[j];
  std::vector<int> cur(off.begin(), off.end() - 1);
  aid.assign(N, 0);
  for (int i = 0; i < N; ++i) aid[cur[link[i]]++] = i;  // ascending id per link
  for (int j = 0; j < L; ++j) {
    auto b = aid.begin() + off[j], e = aid.begin() + off[j + 1];
    const bool sorted = std::is_sorted(b, e, [&](int x, int y) { return pos[x] > pos[y]; });
    if (!sorted)  // stable: ties keep ascending id (argsort_desc, tensor.cpp:672-680)
      std::stable_sort(b, e, [&](int x, int y) { return pos[x] > pos[y]; });
  }
  ps.resize(N);
  lnk.resize(N);
  q0.assign(L, 0.0);
  for (int j = 0; j < L; ++j)
    for (int k = off[j]; k < off[j + 1]; ++k) {
      ps[k] = pos[aid[k]];
      lnk[k] = j;
      if (ps[k] >= 0.5 * length[j]) q0[j] += 1.0;  // initial_counts, engine.cpp:127-135
    }
}

}  // namespace

extern "C" {

int dtg_create(const dtg_net_desc* net, const dtg_sim_config* cfg, int n_agents,
               int n_scenarios, int max_steps, dtg_ctx** out) {
  *out = nullptr;
  dtg_ctx* c = new dtg_ctx;
  const int rc = guarded(nullptr, [&] {
    if (!net || !cfg) throw std::invalid_argument("dtg_create: null network or config");
    const int L = net->n_links;
    if (L <= 0) throw std::invalid_argument("network has no links");
    if (n_agents <= 0) throw std::invalid_argument("no agents");
    if (n_scenarios <= 0) throw std::invalid_argument("n_scenarios must be >= 1");
    if (cfg->delta_n < 1) throw std::invalid_argument("platoon size must be >= 1");
    if (!(cfg->gumbel_tau > 0.0)) throw std::invalid_argument("gumbel_tau must be > 0");
    c->L = L;
    c->N = n_agents;
    c->B = n_scenarios;
    c->cfg = *cfg;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    reserve_pool();
    AllocScope scope(&c->stream);  // the context's buffers come from the pool
    // CSR + predecessor CSR with the successor position of each edge
    std::vector<int> so(net->succ_off, net->succ_off + L + 1);
    const int E = so[L];
    if (so[0] != 0) throw std::invalid_argument("succ_off[0] must be 0");
    std::vector<int> su(net->succ, net->succ + E);
    std::vector<int> pcnt(L + 1, 0);
    for (int i = 0; i < L; ++i) {
      if (so[i + 1] < so[i]) throw std::invalid_argument("succ_off not monotone");
      const int deg = so[i + 1] - so[i];
      c->maxdeg = std::max(c->maxdeg, deg);
      for (int e = so[i]; e < so[i + 1]; ++e) {
        if (su[e] < 0 || su[e] >= L || su[e] == i)
          throw std::invalid_argument("successor out of range or self loop");
        if (e > so[i] && su[e] <= su[e - 1])
          throw std::invalid_argument("successors must be strictly ascending");
        ++pcnt[su[e] + 1];
      }
    }
    if (c->maxdeg > dtg::kMaxDeg)
      throw Unsupported("link out-degree " + std::to_string(c->maxdeg) + " exceeds " +
                        std::to_string(dtg::kMaxDeg));
    for (int j = 0; j < L; ++j) pcnt[j + 1] += pcnt[j];
    std::vector<int> pr(E), pp(E), spe(std::max(E, 1)), fill(pcnt.begin(), pcnt.end() - 1);
    for (int i = 0; i < L; ++i)  // ascending predecessor id per link
      for (int e = so[i]; e < so[i + 1]; ++e) {
        const int q = fill[su[e]]++;
        pr[q] = i;
        pp[q] = e - so[i];
        spe[e] = q;  // global predecessor-edge index of successor edge e
      }
    std::vector<double> ln(net->length, net->length + L), th(L), ct(L), sc(L);
    for (int j = 0; j < L; ++j) {
      if (!(0.5 * ln[j] > 0.0 && 0.5 * ln[j] < ln[j]))  // observation.cpp:194-195
        throw std::runtime_error("midpoint_count: counter position outside (0, L)");
      th[j] = ln[j] - dtg::kArrivalTol;  // node_model.cpp:69-70
      ct[j] = 0.5 * ln[j];               // engine.cpp:46-47
      sc[j] = 5.0 / ln[j];               // observation.cpp:199
    }
    cudaStream_t st = c->stream;
    h2d(c->succ_off, so, st);
    h2d(c->succ, su, st);
    h2d(c->pred_off, pcnt, st);
    h2d(c->pred, pr, st);
    h2d(c->pred_pos, pp, st);
    h2d(c->succ_pedge, spe, st);
    c->E = E;
    h2d(c->len, ln, st);
    h2d(c->thr, th, st);
    h2d(c->ctr, ct, st);
    h2d(c->sc, sc, st);
    const std::size_t B = c->B, N = c->N, BL = B * L, BN = B * N;
    c->params.alloc(5 * BL);
    c->derived.alloc(3 * BL);
    c->seeds.alloc(2 * B);
    c->h_seeds.assign(2 * B, 0);
    c->have_params.assign(B, 0);
    c->have_state.assign(B, 0);
    c->h_link0.assign(B, {});
    for (int b = 0; b < c->B; ++b) {  // default noise: RngStream(0), iteration 0
      const std::uint64_t it = dtg::rng_fork(dtg::rng_fork(0, dtg::lane::kIteration), 0);
      c->h_seeds[b] = dtg::rng_fork(it, dtg::lane::kGumbelLink);
      c->h_seeds[B + b] = dtg::rng_fork(it, dtg::lane::kGumbelMerge);
    }
    c->pos0.alloc(BN);
    c->aid0.alloc(BN);
    c->lnk0.alloc(BN);
    c->off0.alloc(B * (L + 1));
    c->q0.alloc(BL);
    c->x1.alloc(BN);
    c->choice.alloc(BN);
    c->won.alloc(BN);
    c->qn.alloc(BL);
    c->nA.alloc(BL);
    c->tail.alloc(BL);
    c->win.alloc(BL);
    c->vac.alloc(BL);
    c->dep.alloc(BL);
    c->newcnt.alloc(BL);
    c->a0.alloc(B);
    c->errf.alloc(B);
    c->tmp_link.alloc(BN);
    c->tmp_pos.alloc(BN);
    c->x1b.alloc(2 * BN);
    c->wonb.alloc(2 * BN);
    c->nAb.alloc(2 * BL);
    c->qnb.alloc(2 * BL);
    c->tailb.alloc(2 * BL);
    c->depb.alloc(2 * BL);
    c->winp.alloc(BL);
    c->ccnt.alloc(BL);
    c->clist.alloc(1);
    c->stage_params = !dtg::fused_lean(L) && dtg::fused_smem_bytes(L, true) <= 200 * 1024;
    c->pgrid_max = dtg::fused_max_grid(L, c->stage_params);
    c->bgrid_max = dtg::backward_max_grid(L, c->maxdeg);
    c->cluster_cs_max = dtg::fused_max_cluster(L, c->stage_params);
    c->scn_ok = dtg::forward_scn_ok(L);
    {
      int dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    c->gbar.alloc(1);
    c->srec.alloc(BL * c->maxdeg);
    c->cands.alloc(BL * dtg::kClusterCandCap);
    c->ensure_history(std::max(1, max_steps), 0);
    CK(cudaStreamSynchronize(st));
  });
  if (rc != DTG_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return DTG_OK;
}

void dtg_destroy(dtg_ctx* c) {
  AllocScope sync_free(nullptr);  // outside any call: free synchronously
  delete c;
}

const char* dtg_last_error(const dtg_ctx* c) {
  return c ? c->err.c_str() : g_create_error.c_str();
}

int dtg_set_stream(dtg_ctx* c, void* s) {
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->stream));
    if (c->own_stream) CK(cudaStreamDestroy(c->stream));
    c->own_stream = s == nullptr;
    if (s)
      c->stream = static_cast<cudaStream_t>(s);
    else
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->drop_graphs();
  });
}

int dtg_init(void) {
  // CUDA creates the context and loads modules lazily, on the first API call
  // and each kernel's first launch; a 3-link chain with two agents, forward
  // with checkpoints and the reverse sweep, touches the default schedules.
  if (cudaFree(nullptr) != cudaSuccess) return DTG_ERR_CUDA;
  const int succ_off[4] = {0, 1, 2, 2};
  const int succ[2] = {1, 2};
  const double len[3] = {100.0, 100.0, 400.0};
  const dtg_net_desc nd{3, succ_off, succ, len};
  const dtg_sim_config sc{1, 1.0, 99999.0, 0.01, 1};
  dtg_ctx* c = nullptr;
  int rc = dtg_create(&nd, &sc, 2, 1, 4, &c);
  if (rc != DTG_OK) return rc;
  const double u[3] = {16, 16, 16}, k[3] = {0.2, 0.2, 0.2}, one[3] = {1, 1, 1};
  const int link[2] = {0, 0};
  const double pos[2] = {90.0, 50.0};
  double g[15];
  if ((rc = dtg_set_params(c, -1, u, k, one, one, one)) == DTG_OK &&
      (rc = dtg_set_state(c, -1, link, pos)) == DTG_OK && (rc = dtg_set_noise(c, -1, 1, 0)) == DTG_OK &&
      (rc = dtg_forward(c, 4, 2, 1)) == DTG_OK)
    rc = dtg_backward(c, nullptr, nullptr, nullptr, g);
  dtg_destroy(c);
  return rc;
}

int dtg_debug_decisions(int force_exact, unsigned long long* exact_decisions) {
  unsigned long long total = 0;
  for (auto fn : {dtg::decision_stats_fused, dtg::decision_stats_backward, dtg::decision_stats_kernels,
                  dtg::decision_stats_scn}) {
    unsigned long long n = 0;
    if (fn(force_exact, &n) != cudaSuccess) return DTG_ERR_CUDA;
    total += n;
  }
  if (exact_decisions) *exact_decisions = total;
  return DTG_OK;
}

int dtg_set_record_transfers(dtg_ctx* c, int on) {
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->stream));
    c->rec_transfers = on != 0;
    c->drop_graphs();  // the step graph captured the event pointer (or its absence)
  });
}

int dtg_read_transfers(dtg_ctx* c, int scenario, int* winners) {
  return guarded(c, [&] {
    if (scenario < 0 || scenario >= c->B) throw std::invalid_argument("scenario index out of range");
    if (c->ev_T < 0 || c->ev_T != c->last_T)
      throw std::runtime_error("the last forward did not record transfers (dtg_set_record_transfers)");
    c->sync_check();
    const std::size_t L = c->L;
    if (c->ev_T)
      CK(cudaMemcpy2D(winners, L * 4, c->ev.p + scenario * L, static_cast<std::size_t>(c->B) * L * 4, L * 4,
                      c->ev_T, cudaMemcpyDeviceToHost));
  });
}

int dtg_transfer_events(dtg_ctx* c, int scenario, int* events, size_t cap, size_t* n_events) {
  return guarded(c, [&] {
    if (scenario < 0 || scenario >= c->B) throw std::invalid_argument("scenario index out of range");
    const int T = c->ev_T, L = c->L;
    std::vector<int> win(static_cast<std::size_t>(std::max(T, 0)) * L);
    const int rc = dtg_read_transfers(c, scenario, win.data());
    if (rc != DTG_OK) throw std::runtime_error(c->err);
    std::vector<int> cur = c->h_link0[scenario];
    std::size_t n = 0;
    std::vector<std::pair<int, int>> step;  // (agent, to) of one step, ascending agent
    for (int t = 0; t < T; ++t) {
      step.clear();
      for (int i = 0; i < L; ++i) {
        const int a = win[static_cast<std::size_t>(t) * L + i];
        if (a >= 0) step.emplace_back(a, i);
      }
      std::sort(step.begin(), step.end());
      for (const auto& [a, to] : step) {
        if (events && n < cap) {
          events[4 * n] = t;
          events[4 * n + 1] = a;
          events[4 * n + 2] = cur[a];
          events[4 * n + 3] = to;
        }
        cur[a] = to;
        ++n;
      }
    }
    *n_events = n;
  });
}

int dtg_get_stream(const dtg_ctx* c, void** stream, int* owned) {
  if (!c) return DTG_ERR_RUNTIME;
  if (stream) *stream = c->stream;
  if (owned) *owned = c->own_stream ? 1 : 0;
  return DTG_OK;
}

int dtg_profile_persistent(dtg_ctx* c, int T, int spi, double* phase_us, int* grid_out) {
  return guarded(c, [&] {
    c->want_stamps = true;
    const int rc = dtg_forward(c, T, spi, 0);
    c->want_stamps = false;
    if (rc) throw std::runtime_error(c->err);
    c->sync_check();
    const int G = c->last_grid;
    std::vector<unsigned long long> s(static_cast<std::size_t>(T) * G * 4);
    CK(cudaMemcpy(s.data(), c->stamps.p, s.size() * 8, cudaMemcpyDeviceToHost));
    double acc[4] = {0, 0, 0, 0};
    for (int t = 0; t < T; ++t) {
      unsigned long long mn[4], mx[4];
      for (int w = 0; w < 4; ++w) {
        mn[w] = ~0ull;
        mx[w] = 0;
      }
      for (int g = 0; g < G; ++g)
        for (int w = 0; w < 4; ++w) {
          const unsigned long long v = s[(static_cast<std::size_t>(t) * G + g) * 4 + w];
          mn[w] = std::min(mn[w], v);
          mx[w] = std::max(mx[w], v);
        }
      acc[0] += double(mx[1] - mn[0]);  // slot phase
      acc[1] += double(mn[2] - mx[1]);  // barrier 1 after the last CTA arrived
      acc[2] += double(mx[3] - mn[2]);  // link phase
      if (t + 1 < T) {                  // barrier 2 (next step start)
        unsigned long long n0 = ~0ull;
        for (int g = 0; g < G; ++g) n0 = std::min(n0, s[(static_cast<std::size_t>(t + 1) * G + g) * 4]);
        acc[3] += double(n0 - mx[3]);
      }
    }
    for (int w = 0; w < 4; ++w) phase_us[w] = acc[w] / T / 1e3;
    if (grid_out) *grid_out = G;
  });
}

// Measurement hook: one scenario-resident forward (mode 4) with %globaltimer
// stamps; phase_us[6] = per-step span (us) of cf, choice, merge, scan,
// transfer and the whole step, averaged over the CTAs and steps.
int dtg_profile_scn(dtg_ctx* c, int T, int spi, double* phase_us) {
  return guarded(c, [&] {
    const int m = c->mode;
    c->mode = 4;
    c->want_stamps = true;
    const int rc = dtg_forward(c, T, spi, 0);
    c->want_stamps = false;
    c->mode = m;
    if (rc) throw std::runtime_error(c->err);
    c->sync_check();
    std::vector<unsigned long long> s(static_cast<std::size_t>(T) * c->B * 8);
    CK(cudaMemcpy(s.data(), c->stamps.p, s.size() * 8, cudaMemcpyDeviceToHost));
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (std::size_t r = 0; r < static_cast<std::size_t>(T) * c->B; ++r) {
      for (int w = 0; w < 5; ++w) acc[w] += double(s[r * 8 + w + 1] - s[r * 8 + w]);
      acc[5] += double(s[r * 8 + 5] - s[r * 8]);
    }
    for (int w = 0; w < 6; ++w) phase_us[w] = acc[w] / (double(T) * c->B) / 1e3;
    // work lists: mean links with arrived heads, max heads on one link, mean chosen links
    double nact = 0, mxh = 0, ntg = 0;
    for (std::size_t r = 0; r < static_cast<std::size_t>(T) * c->B; ++r) {
      nact += double(s[r * 8 + 6] >> 32);
      mxh = std::max(mxh, double(s[r * 8 + 6] & 0xffffffffull));
      ntg += double(s[r * 8 + 7]);
    }
    phase_us[6] = nact / (double(T) * c->B);
    phase_us[7] = mxh;
    phase_us[8] = ntg / (double(T) * c->B);
  });
}

// Measurement hook: per-warp slot-phase records [T][warps][4] (start, after
// offsets, after slot loop, arrived agents in the warp).
int dtg_debug_warp_records(dtg_ctx* c, int T, int spi, unsigned long long* out, int* n_warps) {
  return guarded(c, [&] {
    c->want_wstamp = true;
    const int rc = dtg_forward(c, T, spi, 0);
    c->want_wstamp = false;
    if (rc) throw std::runtime_error(c->err);
    c->sync_check();
    const std::size_t nw = static_cast<std::size_t>(c->last_grid) * (dtg::kClusterThreads / 32);
    *n_warps = static_cast<int>(nw);
    if (out) CK(cudaMemcpy(out, c->wst.p, static_cast<std::size_t>(T) * nw * 4 * 8, cudaMemcpyDeviceToHost));
  });
}

int dtg_set_flag(dtg_ctx* c, int flag, int value) {
  switch (flag) {
    case 0:  // grid barrier: 1 release/acquire counter (default), 0 cooperative_groups grid.sync
      c->custom_barrier = value != 0;
      return DTG_OK;
    case 3:  // fused-forward timing experiments (results invalid when nonzero)
      c->fwd_dbg = value;
      return DTG_OK;
    case 2:  // reverse-sweep timing experiments (results invalid when nonzero)
      c->bwd_dbg = value;
      return DTG_OK;
    case 1:  // fused forward slot mapping: -1 auto, 0 interleaved, 1 contiguous
      c->contig_mode = value < 0 ? -1 : (value ? 1 : 0);
      return DTG_OK;
    case 4:  // fused forward: speculative head decisions one step ahead (1 default, 0 off)
      c->speculate = value != 0;
      return DTG_OK;
    case 5:  // ... drawn by warps 2.. during barrier 1 (1 default) or by idle link-phase lanes (0)
      c->spec_split = value != 0;
      return DTG_OK;
    case 7:  // grid schedule: CTAs per scenario (0 auto: one slot per thread, capped by the grid)
      c->cs_override = value < 0 ? 0 : value;
      return DTG_OK;
    case 8:  // step graph: scenario branches (0 auto)
      c->graph_split = value < 0 ? 0 : value;
      return DTG_OK;
    default:
      return fail(c, DTG_ERR_CONFIG, "unknown flag");
  }
}

int dtg_set_mode(dtg_ctx* c, int mode) {
  if (mode < 0 || mode > 4) return fail(c, DTG_ERR_CONFIG, "mode must be 0..4");
  c->mode = mode;
  return DTG_OK;
}

int dtg_last_mode(const dtg_ctx* c) {
  return c->last_mode * 1000 + (c->last_mode == 3 ? 0 : c->last_mode == 4 ? 1 : c->last_cs);
}

static void run_backward(dtg_ctx* c, const double* snap, const double* cum, const double* xs,
                         cudaMemcpyKind kind, bool seeds_ready = false);

// Measurement hook: the raw per-CTA phase stamps [T][grid][8] (ns) of the last
// dtg_profile_backward run.
int dtg_debug_bwd_stamps(dtg_ctx* c, unsigned long long* out, int* grid) {
  return guarded(c, [&] {
    const int T = c->last_T, G = c->last_bgrid;
    *grid = G;
    if (out) CK(cudaMemcpy(out, c->stamps.p, static_cast<std::size_t>(T) * G * 8 * 8, cudaMemcpyDeviceToHost));
  });
}

int dtg_profile_backward(dtg_ctx* c, double* phase_us, int* grid_out) {
  return guarded(c, [&] {
    if (c->last_T < 1 || !c->last_ckpt) throw std::runtime_error("needs a checkpointed forward");
    c->want_stamps = true;
    try {
      // the seeds of the last device-loss evaluation when there was one, else zeros
      run_backward(c, nullptr, nullptr, nullptr, cudaMemcpyHostToDevice, c->loss_kind != dtg::kLossNone);
    } catch (...) {
      c->want_stamps = false;
      throw;
    }
    c->want_stamps = false;
    c->sync_check();
    const int T = c->last_T, G = c->last_bgrid;
    std::vector<unsigned long long> s(static_cast<std::size_t>(T) * G * 8);
    CK(cudaMemcpy(s.data(), c->stamps.p, s.size() * 8, cudaMemcpyDeviceToHost));
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long prev_mx7 = 0;  // step t+1's R4 end (the sweep runs t = T-1 .. 0)
    for (int t = T - 1; t >= 0; --t) {
      unsigned long long mn[8], mx[8];
      for (int w = 0; w < 8; ++w) {
        mn[w] = ~0ull;
        mx[w] = 0;
      }
      for (int g = 0; g < G; ++g)
        for (int w = 0; w < 8; ++w) {
          const unsigned long long v = s[(static_cast<std::size_t>(t) * G + g) * 8 + w];
          mn[w] = std::min(mn[w], v);
          mx[w] = std::max(mx[w], v);
        }
      // phase spans R1..R4 and the barrier after each
      acc[0] += double(mx[1] - mn[0]);
      acc[1] += double(mn[2] - mx[1]);
      acc[2] += double(mx[3] - mn[2]);
      acc[3] += double(mn[4] - mx[3]);
      acc[4] += double(mx[5] - mn[4]);
      acc[5] += double(mn[6] - mx[5]);
      acc[6] += double(mx[7] - mn[6]);
      if (t < T - 1) acc[7] += double(mn[0] - prev_mx7);  // step barrier + next step's entry
      prev_mx7 = mx[7];
    }
    for (int w = 0; w < 7; ++w) phase_us[w] = acc[w] / T / 1e3;
    phase_us[7] = T > 1 ? acc[7] / (T - 1) / 1e3 : 0.0;
    if (grid_out) *grid_out = G;
  });
}

int dtg_set_persistent(dtg_ctx* c, int enabled) {
  c->persistent = enabled != 0;
  c->bwd_persistent = enabled != 0;
  return DTG_OK;
}

int dtg_set_graphs(dtg_ctx* c, int enabled) {
  c->graphs = enabled != 0;
  return DTG_OK;
}

namespace {
// params [5][B][L] <- staging [5][L] for scenarios [b0, b0 + nb)
__global__ void k_broadcast_params(const double* __restrict__ src, double* __restrict__ dst, int L, int B,
                                   int b0, int nb) {
  const std::size_t n = static_cast<std::size_t>(5) * nb * L;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const int l = static_cast<int>(i % L);
    const std::size_t r = i / L;
    const int b = static_cast<int>(r % nb) + b0, q = static_cast<int>(r / nb);
    dst[(static_cast<std::size_t>(q) * B + b) * L + l] = src[static_cast<std::size_t>(q) * L + l];
  }
}
}  // namespace

int dtg_set_params(dtg_ctx* c, int scenario, const double* u, const double* kappa,
                   const double* beta, const double* alpha, const double* cost) {
  return guarded(c, [&] {
    if (scenario >= c->B) throw std::invalid_argument("scenario index out of range");
    const std::size_t L = c->L, BL = static_cast<std::size_t>(c->B) * L;
    // stage through pinned memory: the uploads are then truly asynchronous and
    // ordered before the next forward on the stream, with no host wait here
    if (!c->h_par) {
      CK(cudaMallocHost(&c->h_par, 5 * L * sizeof(double)));
      CK(cudaEventCreateWithFlags(&c->par_ev, cudaEventDisableTiming));
    } else {
      CK(cudaEventSynchronize(c->par_ev));  // the previous upload has left the staging
    }
    {
      const double* in[5] = {u, kappa, beta, alpha, cost};
      for (int q = 0; q < 5; ++q) std::memcpy(c->h_par + q * L, in[q], L * sizeof(double));
    }
    // one upload of [5][L], then one kernel writes it to the scenario(s)
    c->d_par.ensure(5 * L);
    CK(cudaMemcpyAsync(c->d_par.p, c->h_par, 5 * L * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(c->par_ev, c->stream));
    const int b0 = scenario < 0 ? 0 : scenario, nb = scenario < 0 ? c->B : 1;
    const std::size_t n = 5 * static_cast<std::size_t>(nb) * L;
    const int grid = static_cast<int>(std::min<std::size_t>((n + 255) / 256, 1184));
    k_broadcast_params<<<grid, 256, 0, c->stream>>>(c->d_par.p, c->params.p, static_cast<int>(L), c->B, b0, nb);
    CK(cudaGetLastError());
    for (int b = b0; b < b0 + nb; ++b) c->have_params[b] = 1;
    (void)BL;
  });
}

int dtg_set_state(dtg_ctx* c, int scenario, const int* link, const double* pos) {
  return guarded(c, [&] {
    if (scenario >= c->B) throw std::invalid_argument("scenario index out of range");
    std::vector<double> length(c->L);
    CK(cudaMemcpy(length.data(), c->len.p, sizeof(double) * c->L, cudaMemcpyDeviceToHost));
    std::vector<double> ps, q0;
    std::vector<int> aid, lnk, off;
    build_layout(c->N, c->L, link, pos, length, ps, aid, lnk, off, q0);
    const std::size_t N = c->N, L = c->L;
    for (int b = 0; b < c->B; ++b) {
      if (scenario >= 0 && b != scenario) continue;
      CK(cudaMemcpyAsync(c->pos0.p + b * N, ps.data(), N * 8, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(c->aid0.p + b * N, aid.data(), N * 4, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(c->lnk0.p + b * N, lnk.data(), N * 4, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(c->off0.p + b * (L + 1), off.data(), (L + 1) * 4,
                         cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(c->q0.p + b * L, q0.data(), L * 8, cudaMemcpyHostToDevice, c->stream));
      c->have_state[b] = 1;
      c->h_link0[b].assign(link, link + N);
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int dtg_set_noise(dtg_ctx* c, int scenario, uint64_t root_seed, uint64_t noise_iteration) {
  return guarded(c, [&] {
    if (scenario >= c->B) throw std::invalid_argument("scenario index out of range");
    // engine.cpp:49 then node_model.cpp:65 / :114
    const std::uint64_t it =
        dtg::rng_fork(dtg::rng_fork(root_seed, dtg::lane::kIteration), noise_iteration);
    for (int b = 0; b < c->B; ++b) {
      if (scenario >= 0 && b != scenario) continue;
      c->h_seeds[b] = dtg::rng_fork(it, dtg::lane::kGumbelLink);
      c->h_seeds[c->B + b] = dtg::rng_fork(it, dtg::lane::kGumbelMerge);
    }
  });
}

int dtg_forward(dtg_ctx* c, int T, int spi, int checkpoint) {
  return guarded(c, [&] {
    if (T < 0) throw std::invalid_argument("negative horizon");
    if (spi < 1)
      throw std::runtime_error("observation interval must be a positive multiple of the time step");
    for (int b = 0; b < c->B; ++b)
      if (!c->have_params[b] || !c->have_state[b])
        throw std::invalid_argument("scenario " + std::to_string(b) +
                                    " has no parameters or initial state");
    c->ensure_history(T, checkpoint);
    cudaStream_t st = c->stream;
    {  // seeds through pinned staging: an asynchronous upload, no host wait
      const std::size_t sb = sizeof(std::uint64_t) * 2 * c->B;
      if (!c->h_seed_pin) {
        CK(cudaMallocHost(&c->h_seed_pin, sb));
        CK(cudaEventCreateWithFlags(&c->seed_ev, cudaEventDisableTiming));
      } else {
        CK(cudaEventSynchronize(c->seed_ev));
      }
      std::memcpy(c->h_seed_pin, c->h_seeds.data(), sb);
      CK(cudaMemcpyAsync(c->seeds.p, c->h_seed_pin, sb, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(c->seed_ev, st));
    }
    const dtg::DevView d = c->view();
    const std::size_t BN = static_cast<std::size_t>(c->B) * c->N;
    const std::size_t BL = static_cast<std::size_t>(c->B) * c->L;
    const int nsp = c->graph_branches();
    bool scn = false;  // mode 4: scenario-resident CTAs (decided below, before body() runs)
    auto body = [&] {
      dtg::launch_derive(d, c->derived.p, c->derived.p + BL, c->derived.p + 2 * BL, st);
      dtg::launch_pack_succ(d, c->srec.p, st);
      CK(cudaMemcpyAsync(c->pos.p, c->pos0.p, BN * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(c->aid.p, c->aid0.p, BN * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(c->lnk.p, c->lnk0.p, BN * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(c->off.p, c->off0.p, static_cast<std::size_t>(c->B) * (c->L + 1) * 4,
                         cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(c->qh.p, c->q0.p, BL * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemsetAsync(c->cumh.p, 0, BL * 8, st));
      CK(cudaMemsetAsync(c->errf.p, 0, sizeof(int) * c->B, st));
      if (scn) {
        unsigned long long* stp = nullptr;
        if (c->want_stamps) {
          c->stamps.ensure(static_cast<std::size_t>(T) * c->B * 8);
          stp = c->stamps.p;
        }
        CK(dtg::launch_forward_scn(d, T, stp, st));
        return;
      }
      c->fork_branches(nsp, st, [&](int b0, int nb, cudaStream_t sq) {
        dtg::DevView dq = d;
        dq.b0 = b0;
        dq.nb = nb;
        for (int t = 0; t < T; ++t) dtg::launch_step_forward(dq, t, t % c->S, (t + 1) % c->S, sq);
      });
    };
    // cluster-per-scenario mode: <= 8 slots per thread inside one cluster
    int cs_need = (c->N + dtg::kClusterThreads * 8 - 1) / (dtg::kClusterThreads * 8);
    int cs = 1;
    while (cs < cs_need) cs <<= 1;
    const bool cluster_ok = c->cluster_cs_max > 0 && cs <= c->cluster_cs_max;
    int mode = c->mode;
    // auto: the persistent grid schedule measured fastest (profiles/r01/phase_*.log)
    if (mode == 0) mode = c->persistent ? 2 : 3;
    if (mode == 1 && !cluster_ok) mode = 2;
    if (mode == 2 && (c->pgrid_max <= 0 || c->B > c->pgrid_max)) mode = 3;
    // auto: with fewer than 5 CTAs per scenario the fused kernel loses to the
    // step graph (C3 ms/nowcast fused vs graph with 4 branches: B=24 (6 CTAs)
    // 3.82 vs 4.68, B=32 (4) 5.33 vs 5.05, B=48 (3) 6.68 vs 6.10, B=64 (2)
    // 9.91 vs 7.41; scripts/graph_time.py)
    if (c->mode == 0 && mode == 2 && c->N > dtg::kClusterThreads && 5 * c->B > c->pgrid_max) mode = 3;
    if (!c->persistent && c->mode == 0) mode = 3;
    // auto: one CTA per scenario beats the step graph from ~0.55 scenarios per
    // SM (a 768-thread CTA per SM) and beyond ~1.2 (two 384-thread CTAs per
    // SM); C3 ms/nowcast graph vs mode 4: B=64 8.1 vs 9.0, B=80 9.5 vs 9.5,
    // B=96 11.2 vs 9.8, B=148 15.8 vs 10.9, B=160 17.2 vs 18.6, B=192 21.1 vs
    // 19.4, B=256 27.9 vs 20.3 (scripts/scn_time.py)
    if (c->mode == 0 && c->persistent && mode == 3 &&
        ((20 * c->B >= 11 * c->n_sm && c->B <= c->n_sm) || 5 * c->B > 6 * c->n_sm))
      mode = 4;
    if (mode == 4 && !c->scn_ok) mode = 3;  // per-link state exceeds shared memory
    c->last_mode = mode;
    scn = mode == 4;
    if ((mode == 1 || mode == 2) && T > 0) {
      {  // one launch for the per-link constants, the initial layout and the counters
        dtg::ForwardInit in{};
        in.d = d;
        in.jam = c->derived.p;
        in.dxf = c->derived.p + BL;
        in.pref = c->derived.p + 2 * BL;
        in.srec = c->srec.p;
        in.pos = c->pos.p;
        in.pos0 = c->pos0.p;
        in.aid = c->aid.p;
        in.aid0 = c->aid0.p;
        in.lnk = c->lnk.p;
        in.lnk0 = c->lnk0.p;
        in.off = c->off.p;
        in.off0 = c->off0.p;
        in.qh = c->qh.p;
        in.q0 = c->q0.p;
        in.cumh = c->cumh.p;
        in.errf = c->errf.p;
        in.ccnt = c->ccnt.p;
        in.depb = c->depb.p;
        in.gbar = c->gbar.p;
        dtg::launch_forward_init(in, st);
        CK(cudaGetLastError());
      }
      dtg::CView V{};
      V.d = d;
      V.x1b = c->x1b.p;
      V.wonb = c->wonb.p;
      V.nAb = c->nAb.p;
      V.qnb = c->qnb.p;
      V.tailb = c->tailb.p;
      V.depb = c->depb.p;
      V.win = c->winp.p;
      V.ccnt = c->ccnt.p;
      V.cands = c->cands.p;
      V.srec = c->srec.p;
      V.T = T;
      V.ckpt = checkpoint ? 1 : 0;
      V.dbg = c->fwd_dbg;
      V.stage_params = c->stage_params ? 1 : 0;
      V.lean = dtg::fused_lean(c->L) ? 1 : 0;
      V.tstamp = nullptr;
      V.gbar = c->custom_barrier ? c->gbar.p : nullptr;
      // grid mode: CTA 0 sees every scenario's step complete at the grid
      // barrier; a cluster only sees its own scenario
      V.progress = (c->stream_progress > 0 && (mode == 2 || c->B == 1)) ? c->prog_h : nullptr;
      V.progress_every = std::max(1, c->stream_progress);
      if (mode == 1) {
        V.cs = cs;
      } else {
        // CTAs per scenario: one slot per thread, capped by the resident grid
        int want = (std::max(c->N, c->L) + dtg::kClusterThreads - 1) / dtg::kClusterThreads;
        if (c->cs_override > 0) want = c->cs_override;  // tuning experiments (flag 7)
        V.cs = std::max(1, std::min(want, c->pgrid_max / c->B));
      }
      // interleaved 512-slot blocks by default (measured faster at C3 dn30
      // B=1/8 and dn1: spreads dense runs of arrived heads over the CTAs)
      V.contig = c->contig_mode >= 0 ? c->contig_mode : 0;
      c->last_grid = c->B * V.cs;
      c->last_cs = V.cs;
      // speculative head draws: 8 lanes per link besides the link threads, one round
      V.spec = nullptr;
      if (c->speculate && V.cs * dtg::kClusterThreads >= 9 * c->L) {
        c->spec.ensure(static_cast<std::size_t>(4) * BL);
        V.spec = c->spec.p;
      }
      V.spec_split = (c->spec_split && V.spec && mode == 2 && V.gbar && V.cs * 64 >= c->L &&
                      c->N <= V.cs * dtg::kClusterThreads)
                         ? 1
                         : 0;
      V.wstamp = nullptr;
      if (c->want_wstamp) {
        c->wst.ensure(static_cast<std::size_t>(T) * c->B * V.cs * (dtg::kClusterThreads / 32) * 4 + 4);
        V.wstamp = c->wst.p;
      }
      if (c->want_stamps) {
        c->stamps.ensure(static_cast<std::size_t>(T) * c->last_grid * 4);
        V.tstamp = c->stamps.p;
      }
      CK(dtg::launch_forward_fused(V, mode == 1, st));
      c->launches = 2;  // k_forward_init + k_forward_fused
      c->last_T = T;
      c->last_spi = spi;
      c->last_ckpt = checkpoint;
      c->last_K = T / spi;
      c->pending = true;
      return;
    }
    const long long key = (static_cast<long long>(T) << 20) ^ (c->S << 1) ^ 1 ^ (static_cast<long long>(nsp) << 50);
    if (scn && T > 0) {  // six launches: no graph needed
      body();
      CK(cudaGetLastError());
      c->launches = 2 + 1;  // k_derive, k_pack_succ, k_forward_scn
      c->last_T = T;
      c->last_spi = spi;
      c->last_ckpt = checkpoint;
      c->last_K = T / spi;
      c->pending = true;
      return;
    }
    if (c->graphs && T > 0) {
      if (c->fwd_key != key || !c->fwd_exec) {
        if (c->fwd_exec) cudaGraphExecDestroy(c->fwd_exec);
        c->fwd_exec = nullptr;
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        body();
        CK(cudaStreamEndCapture(st, &g));
        CK(cudaGraphInstantiate(&c->fwd_exec, g, 0));
        cudaGraphDestroy(g);
        c->fwd_key = key;
      }
      CK(cudaGraphLaunch(c->fwd_exec, st));
    } else {
      body();
      CK(cudaGetLastError());
    }
    c->launches = 1 + static_cast<std::int64_t>(T) * dtg::kLaunchesPerForwardStep;
    c->last_T = T;
    c->last_spi = spi;
    c->last_ckpt = checkpoint;
    c->last_K = T / spi;
    c->pending = true;
  });
}

int dtg_sync(dtg_ctx* c) {
  return guarded(c, [&] { c->sync_check(); });
}

int dtg_read_cum(dtg_ctx* c, int scenario, double* cum) {
  return guarded(c, [&] {
    if (scenario < 0 || scenario >= c->B) throw std::invalid_argument("scenario index out of range");
    c->sync_check();
    if (c->last_T < 0) throw std::runtime_error("no forward run");
    if (c->last_T == 0) return;
    const std::size_t L = c->L, BL = static_cast<std::size_t>(c->B) * L;
    CK(cudaMemcpy2D(cum, L * 8, c->cumh.p + BL + scenario * L, BL * 8, L * 8, c->last_T,
                    cudaMemcpyDeviceToHost));
  });
}

int dtg_read_cum_all(dtg_ctx* c, double* cum) {
  return guarded(c, [&] {
    c->sync_check();
    if (c->last_T < 0) throw std::runtime_error("no forward run");
    const int T = c->last_T;
    if (T == 0) return;
    const std::size_t L = c->L, B = c->B, BL = B * L;
    const std::size_t n = static_cast<std::size_t>(T) * BL;
    if (c->h_stage_n < n) {
      if (c->h_stage) cudaFreeHost(c->h_stage);
      c->h_stage = nullptr;
      c->h_stage_n = 0;
      CK(cudaMallocHost(&c->h_stage, n * 8));
      c->h_stage_n = n;
    }
    CK(cudaMemcpyAsync(c->h_stage, c->cumh.p + BL, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (std::size_t b = 0; b < B; ++b)
      for (int t = 0; t < T; ++t)
        std::memcpy(cum + (b * T + t) * L, c->h_stage + (t * B + b) * L, L * 8);
  });
}

int dtg_forward_read(dtg_ctx* c, int T, int spi, int checkpoint, double* cum, int* link,
                     double* pos) {
  if (!c->prog_h) {
    const int rc = guarded(c, [&] {
      CK(cudaHostAlloc(&c->prog_h, sizeof(unsigned int), cudaHostAllocMapped));
      CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    });
    if (rc) return rc;
  }
  // ~8 chunks of count rows; the kernel publishes its progress at chunk ends
  const int chunk = std::max(1, (T + 7) / 8);
  *reinterpret_cast<volatile unsigned int*>(c->prog_h) = 0;
  c->stream_progress = (cum && T > 0) ? chunk : 0;
  const int rc = dtg_forward(c, T, spi, checkpoint);
  c->stream_progress = 0;
  if (rc) return rc;
  return guarded(c, [&] {
    const std::size_t L = c->L, B = c->B, BL = B * L, N = c->N;
    // everything after the kernel is enqueued right behind it (no host round
    // trip): final-state gather, its copies and the error flags, all into one
    // pinned block [errf B ints | link B*N ints | pos B*N doubles]
    const std::size_t need = B * 4 + B * N * 12 + 8;
    if (c->h_fin_n < need) {
      if (c->h_fin) cudaFreeHost(c->h_fin);
      c->h_fin = nullptr;
      c->h_fin_n = 0;
      CK(cudaMallocHost(&c->h_fin, need));
      c->h_fin_n = need;
    }
    int* he = static_cast<int*>(c->h_fin);
    int* hl = he + B;
    double* hp = reinterpret_cast<double*>(
        static_cast<char*>(c->h_fin) + ((B * 4 + B * N * 4 + 7) / 8) * 8);
    const bool link_direct = link && pinned_host(link), pos_direct = pos && pinned_host(pos);
    if (link || pos) {
      const dtg::DevView d = c->view();
      dtg::launch_gather_state(d, T % c->S, c->tmp_link.p, c->tmp_pos.p, c->stream);
      CK(cudaGetLastError());
      if (link)
        CK(cudaMemcpyAsync(link_direct ? link : hl, c->tmp_link.p, B * N * 4, cudaMemcpyDeviceToHost, c->stream));
      if (pos)
        CK(cudaMemcpyAsync(pos_direct ? pos : hp, c->tmp_pos.p, B * N * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaMemcpyAsync(he, c->errf.p, B * 4, cudaMemcpyDeviceToHost, c->stream));
    if (cum && T > 0) {
      const std::size_t n = static_cast<std::size_t>(T) * BL;
      if (c->h_stage_n < n) {
        if (c->h_stage) cudaFreeHost(c->h_stage);
        c->h_stage = nullptr;
        c->h_stage_n = 0;
        CK(cudaMallocHost(&c->h_stage, n * 8));
        c->h_stage_n = n;
      }
      // copy finished count rows while the kernel runs: each chunk is issued
      // once the kernel has published that its steps are final (or once the
      // stream is idle: schedules without a progress counter, errors).  A
      // caller buffer in page-locked memory (dtg_host_alloc) takes the rows by
      // DMA directly ([t][b] rows on the device -> [b][t] rows: one strided
      // 2-D copy per scenario); pageable memory goes through pinned staging.
      const bool direct = pinned_host(cum);
      const volatile unsigned int* prog = c->prog_h;
      int done = 0;
      while (done < T) {
        const int end = std::min(T, done + chunk);
        while (static_cast<int>(*prog) < end) {
          if (cudaStreamQuery(c->stream) != cudaErrorNotReady) break;
        }
        const double* src = c->cumh.p + static_cast<std::size_t>(done + 1) * BL;
        if (direct) {
          for (std::size_t b = 0; b < B; ++b)
            CK(cudaMemcpy2DAsync(cum + (b * T + done) * L, L * 8, src + b * L, BL * 8, L * 8, end - done,
                                 cudaMemcpyDeviceToHost, c->copy_stream));
        } else {
          CK(cudaMemcpyAsync(c->h_stage + static_cast<std::size_t>(done) * BL, src,
                             static_cast<std::size_t>(end - done) * BL * 8, cudaMemcpyDeviceToHost,
                             c->copy_stream));
          CK(cudaStreamSynchronize(c->copy_stream));
          for (std::size_t b = 0; b < B; ++b)
            for (int t = done; t < end; ++t)
              std::memcpy(cum + (b * T + t) * L, c->h_stage + (t * B + b) * L, L * 8);
        }
        done = end;
      }
      if (direct) CK(cudaStreamSynchronize(c->copy_stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    c->pending = false;
    c->check_flags(he);
    if (link && !link_direct) std::memcpy(link, hl, B * N * 4);
    if (pos && !pos_direct) std::memcpy(pos, hp, B * N * 8);
  });
}

void* dtg_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}

void dtg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int dtg_read_state(dtg_ctx* c, int scenario, int step, int* link, double* pos) {
  return guarded(c, [&] {
    if (scenario < 0 || scenario >= c->B) throw std::invalid_argument("scenario index out of range");
    c->sync_check();
    const int T = c->last_T;
    if (T < 0) throw std::runtime_error("no forward run");
    if (step < 0) step = T;
    if (step > T || (!c->last_ckpt && step < T))
      throw std::invalid_argument("step not kept (run dtg_forward with checkpoint=1)");
    const dtg::DevView d = c->view();
    dtg::launch_gather_state(d, step % c->S, c->tmp_link.p, c->tmp_pos.p, c->stream);
    CK(cudaGetLastError());
    const std::size_t N = c->N;
    CK(cudaMemcpyAsync(link, c->tmp_link.p + scenario * N, N * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(pos, c->tmp_pos.p + scenario * N, N * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int dtg_n_snapshots(const dtg_ctx* c) { return c->last_T < 0 ? 0 : c->last_K; }

const double* dtg_device_cum(const dtg_ctx* c) { return c->cumh.p; }

int64_t dtg_last_launches(const dtg_ctx* c) { return c->launches; }

static void run_backward_persistent(dtg_ctx* c, cudaStream_t st) {
  const int T = c->last_T, K = c->last_K, spi = c->last_spi;
  const std::size_t B = c->B, L = c->L, N = c->N, BL = B * L, BN = B * N, MD = c->maxdeg;
  const int bt = dtg::backward_threads();
  const int want = (std::max(c->N, c->L) + bt - 1) / bt;
  int bps, grid;
  if (static_cast<long long>(c->B) * want <= c->bgrid_max) {
    bps = want;
    grid = c->B * want;
  } else if (c->B <= c->bgrid_max) {
    bps = c->bgrid_max / c->B;
    grid = bps * c->B;
  } else {
    bps = 0;
    grid = c->bgrid_max;
  }
  const std::size_t nblk = bps > 0 ? bps : 1;
  bool ch = false;
  ch |= c->bx1.ensure(BN);
  ch |= c->btail.ensure(BL);
  ch |= c->bmpi.ensure(BL * dtg::kBwdCandCap);
  ch |= c->bmlz.ensure(BL * dtg::kBwdCandCap);
  ch |= c->blpi.ensure(2 * BN * MD);  // per step parity (R4 of t+1 runs with R1 of t)
  ch |= c->bnA.ensure(2 * BL);
  ch |= c->bnAc.ensure(BL);
  ch |= c->bwon.ensure(BN);
  ch |= c->bdep.ensure(BL);
  ch |= c->bwin.ensure(BL);
  ch |= c->bccnt.ensure(2 * BL);
  ch |= c->bched.ensure(2 * BN);
  ch |= c->bchoice.ensure(2 * BN);
  ch |= c->balist.ensure(2 * BN);
  ch |= c->bacount.ensure(2 * B);
  ch |= c->bvac.ensure(BL);
  ch |= c->bcands.ensure(BL * dtg::kBwdCandCap);
  ch |= c->ba0key.ensure(2 * B);
  ch |= c->bsort.ensure(B * MD * N);
  ch |= c->ba0part.ensure(B * nblk * MD * 32);
  ch |= c->vbar.ensure(2 * BN * MD);
  // vbar is shared with the step-graph reverse sweep, whose cached graph
  // (bwd_exec) captured its old pointer: a reallocation must invalidate it
  if (ch) c->drop_graphs();
  CK(cudaMemsetAsync(c->bccnt.p, 0, 2 * BL * 4, st));
  CK(cudaMemsetAsync(c->bdep.p, 0, BL * 4, st));
  CK(cudaMemsetAsync(c->bacount.p, 0, 2 * B * 4, st));
  CK(cudaMemsetAsync(c->ba0key.p, 0xff, 2 * B * 8, st));
  CK(cudaMemsetAsync(c->errf.p, 0, B * 4, st));
  dtg::BView V{};
  V.d = c->view();
  V.x1 = c->bx1.p;
  V.nAb = c->bnA.p;
  V.nA_cur = c->bnAc.p;
  V.tail = c->btail.p;
  V.won = c->bwon.p;
  V.dep = c->bdep.p;
  V.win = c->bwin.p;
  V.vac = c->bvac.p;
  V.ccnt = c->bccnt.p;
  V.cands = c->bcands.p;
  V.mpi = c->bmpi.p;
  V.mlz = c->bmlz.p;
  V.lpi = c->blpi.p;
  V.ched = c->bched.p;
  V.choice = c->bchoice.p;
  V.alist = c->balist.p;
  V.acount = c->bacount.p;
  V.a0key = c->ba0key.p;
  V.a0part = c->ba0part.p;
  V.xbar = c->xbar.p;
  V.cbar = c->cbar.p;
  V.qbar = c->qbar.p;
  V.qtot = c->qtot.p;
  V.lbar_row = c->lbar_row.p;
  V.prio_bar = c->prio_bar.p;
  V.lbar_a0 = c->lbar_a0.p;
  V.vbar = c->vbar.p;
  V.cu = c->cu.p;
  V.cg = c->cg.p;
  V.grads = c->grads.p;
  V.snap_seed = K ? c->snap_seed.p : nullptr;
  V.cum_seed = c->cum_seed.p;
  V.x_seed = c->x_seed.p;
  V.sort_scratch = c->bsort.p;
  V.K = K;
  V.spi = spi;
  V.T = T;
  V.bps = bps;
  V.force_slow = c->force_slow;
  V.dbg = c->bwd_dbg;
  V.tstamp = nullptr;
  if (c->want_stamps) {
    c->stamps.ensure(static_cast<std::size_t>(T) * grid * 8);
    V.tstamp = c->stamps.p;
  }
  c->last_bgrid = grid;
  V.gbar = nullptr;
  if (c->custom_barrier) {
    c->bgbar.ensure(1);
    CK(cudaMemsetAsync(c->bgbar.p, 0, sizeof(unsigned int), st));
    V.gbar = c->bgbar.p;
  }
  CK(dtg::launch_backward_persistent(V, grid, st));
  c->launches = 1;
  c->pending = true;
}

static void run_backward(dtg_ctx* c, const double* snap, const double* cum, const double* xs,
                         cudaMemcpyKind kind, bool seeds_ready) {
  if (c->last_T < 0 || !c->last_ckpt)
    throw std::runtime_error("dtg_backward needs a preceding dtg_forward with checkpoint=1");
  const int T = c->last_T, K = c->last_K, spi = c->last_spi;
  const std::size_t B = c->B, L = c->L, N = c->N;
  cudaStream_t st = c->stream;
  bool changed = false;
  changed |= c->snap_seed.ensure(std::max<std::size_t>(1, B * K * L));
  changed |= c->cum_seed.ensure(B * L);
  changed |= c->x_seed.ensure(B * N);
  changed |= c->cbar.ensure(B * L);
  changed |= c->qbar.ensure(B * L);
  changed |= c->qtot.ensure(B * L);
  changed |= c->lbar_row.ensure(B * N);
  changed |= c->prio_bar.ensure(B * N);
  changed |= c->vbar.ensure(B * N * c->maxdeg);
  changed |= c->lbar_a0.ensure(B * c->maxdeg);
  changed |= c->cu.ensure(B * N);
  changed |= c->cg.ensure(B * N);
  changed |= c->grads.ensure(B * 5 * L);
  changed |= c->xbar.ensure(2 * B * N);
  changed |= c->sort_scratch.ensure(2 * B * N + 2);
  changed |= c->alist.ensure(B * N);
  changed |= c->acount.ensure(B);
  if (changed) c->drop_graphs();
  auto up = [&](double* dst, const double* src, std::size_t n) {
    if (src)
      CK(cudaMemcpyAsync(dst, src, n * 8, kind, st));
    else
      CK(cudaMemsetAsync(dst, 0, n * 8, st));
  };
  if (!seeds_ready) {
    if (K) up(c->snap_seed.p, snap, B * K * L);
    up(c->cum_seed.p, cum, B * L);
    up(c->x_seed.p, xs, B * N);
  }
  if (c->bwd_persistent && c->bgrid_max > 0 && c->mode != 3 && T > 0) {
    run_backward_persistent(c, st);
    return;
  }
  dtg::DevView d = c->view();
  d.alist = c->alist.p;
  d.acount = c->acount.p;
  double* xb[2] = {c->xbar.p, c->xbar.p + B * N};
  auto body = [&] {
    CK(cudaMemsetAsync(c->acount.p, 0, B * sizeof(int), st));
    dtg::launch_adj_init(d, T % c->S, c->x_seed.p, xb[T & 1], c->cum_seed.p, st);
    for (int t = T - 1; t >= 0; --t) {
      const int snap_k = ((t + 1) % spi == 0) ? (t + 1) / spi - 1 : -1;
      dtg::launch_step_backward(d, t, t % c->S, (t + 1) % c->S, xb[(t + 1) & 1], xb[t & 1],
                                c->snap_seed.p, snap_k, K, c->sort_scratch.p, c->force_slow, st);
    }
  };
  const long long key = (static_cast<long long>(T) << 24) ^ (static_cast<long long>(spi) << 2) ^
                        (c->force_slow << 1) ^ static_cast<long long>(c->S << 12);
  if (c->graphs && T > 0) {
    if (c->bwd_key != key || !c->bwd_exec) {
      if (c->bwd_exec) cudaGraphExecDestroy(c->bwd_exec);
      c->bwd_exec = nullptr;
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      body();
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&c->bwd_exec, g, 0));
      cudaGraphDestroy(g);
      c->bwd_key = key;
    }
    CK(cudaGraphLaunch(c->bwd_exec, st));
  } else {
    body();
    CK(cudaGetLastError());
  }
  c->launches = 2 + static_cast<std::int64_t>(T) * dtg::kLaunchesPerBackwardStep;
  c->pending = true;
}

int dtg_backward(dtg_ctx* c, const double* snap, const double* cum, const double* xs,
                 double* grads) {
  return guarded(c, [&] {
    c->sync_check();
    run_backward(c, snap, cum, xs, cudaMemcpyHostToDevice);
    const std::size_t n = static_cast<std::size_t>(c->B) * 5 * c->L;
    CK(cudaMemcpyAsync(grads, c->grads.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync_check();
  });
}

int dtg_backward_device(dtg_ctx* c, const double* snap, const double* cum, const double* xs,
                        double* d_grads) {
  return guarded(c, [&] {
    run_backward(c, snap, cum, xs, cudaMemcpyDeviceToDevice);
    const std::size_t n = static_cast<std::size_t>(c->B) * 5 * c->L;
    CK(cudaMemcpyAsync(d_grads, c->grads.p, n * 8, cudaMemcpyDeviceToDevice, c->stream));
  });
}

// ---- device losses and the draw reduction -------------------

int dtg_set_loss_mse(dtg_ctx* c, int k_obs, int n_obs, const int* link_ids,
                     const double* values) {
  return guarded(c, [&] {
    if (k_obs < 0 || n_obs < 1 || !link_ids || (k_obs > 0 && !values))
      throw std::invalid_argument("loss: no observed links");
    if (n_obs > dtg::max_mse_obs(k_obs))
      throw std::invalid_argument("loss: " + std::to_string(n_obs) + " observed links exceed the device MSE "
                                  "kernel's shared-memory capacity (" + std::to_string(dtg::max_mse_obs(k_obs)) +
                                  " links for " + std::to_string(k_obs) + " intervals)");
    std::vector<int> first(n_obs, 1), next(n_obs, -1);
    for (int q = 0; q < n_obs; ++q) {
      if (link_ids[q] < 0 || link_ids[q] >= c->L)
        throw std::invalid_argument("loss: observed link missing from simulation");
      for (int r = q + 1; r < n_obs; ++r)
        if (link_ids[r] == link_ids[q]) {
          next[q] = r;
          first[r] = 0;
          break;
        }
    }
    c->loss_ids.ensure(n_obs);
    c->loss_first.ensure(n_obs);
    c->loss_next.ensure(n_obs);
    c->loss_obs.ensure(std::max<std::size_t>(1, static_cast<std::size_t>(k_obs) * n_obs));
    CK(cudaMemcpy(c->loss_ids.p, link_ids, sizeof(int) * n_obs, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->loss_first.p, first.data(), sizeof(int) * n_obs, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->loss_next.p, next.data(), sizeof(int) * n_obs, cudaMemcpyHostToDevice));
    if (k_obs)
      CK(cudaMemcpy(c->loss_obs.p, values, sizeof(double) * k_obs * n_obs,
                    cudaMemcpyHostToDevice));
    c->loss_kind = dtg::kLossMse;
    c->loss_kobs = k_obs;
    c->loss_nobs = n_obs;
  });
}

int dtg_set_loss_control(dtg_ctx* c, int target_link, double desired_count) {
  return guarded(c, [&] {
    if (target_link < 0 || target_link >= c->L)
      throw std::invalid_argument("control: target link out of range");
    c->loss_kind = dtg::kLossControl;
    c->loss_target = target_link;
    c->loss_desired = desired_count;
  });
}

int dtg_gradient_device_loss(dtg_ctx* c, double* d_rows) {
  return guarded(c, [&] {
    if (c->loss_kind == dtg::kLossNone)
      throw std::invalid_argument("no device loss set (dtg_set_loss_mse / dtg_set_loss_control)");
    if (c->last_T < 0 || !c->last_ckpt)
      throw std::runtime_error("dtg_gradient_device_loss needs a preceding dtg_forward with checkpoint=1");
    if (c->loss_kind == dtg::kLossMse && c->last_K < c->loss_kobs)
      throw std::runtime_error("loss: fewer snapshots than observations");
    const std::size_t B = c->B, L = c->L, N = c->N;
    const int K = c->last_K;
    cudaStream_t st = c->stream;
    bool changed = false;
    changed |= c->snap_seed.ensure(std::max<std::size_t>(1, B * K * L));
    changed |= c->cum_seed.ensure(B * L);
    changed |= c->x_seed.ensure(B * N);
    if (changed) c->drop_graphs();
    c->loss_val.ensure(B);
    c->loss_extra.ensure(B);
    const std::size_t R = 5 * L + 2;
    c->rows.ensure(B * R);
    if (K) CK(cudaMemsetAsync(c->snap_seed.p, 0, B * K * L * 8, st));
    CK(cudaMemsetAsync(c->cum_seed.p, 0, B * L * 8, st));
    CK(cudaMemsetAsync(c->x_seed.p, 0, B * N * 8, st));
    dtg::LossView v{};
    v.kind = c->loss_kind;
    v.B = c->B;
    v.L = c->L;
    v.N = c->N;
    v.T = c->last_T;
    v.spi = c->last_spi;
    v.K = K;
    v.dn = static_cast<double>(c->cfg.delta_n);
    v.cumh = c->cumh.p;
    v.kobs = c->loss_kobs;
    v.nobs = c->loss_nobs;
    v.ids = c->loss_ids.p;
    v.first = c->loss_first.p;
    v.next = c->loss_next.p;
    v.obs = c->loss_obs.p;
    v.sc = 1.0 / (static_cast<double>(c->loss_kobs) * c->loss_nobs);
    v.target = c->loss_target;
    v.desired = c->loss_desired;
    v.snap_seed = c->snap_seed.p;
    v.cum_seed = c->cum_seed.p;
    v.loss = c->loss_val.p;
    v.extra = c->loss_extra.p;
    CK(dtg::launch_device_loss(v, st));
    CK(cudaGetLastError());
    if (c->last_T > 0) {
      run_backward(c, nullptr, nullptr, nullptr, cudaMemcpyDeviceToDevice, true);
    } else {
      c->grads.ensure(B * 5 * L);
      CK(cudaMemsetAsync(c->grads.p, 0, B * 5 * L * 8, st));
    }
    dtg::launch_pack_rows(c->B, c->L, c->grads.p, c->loss_val.p, c->loss_extra.p,
                          d_rows ? d_rows : c->rows.p, st);
    CK(cudaGetLastError());
    c->launches += 2;
    c->pending = true;
  });
}

int dtg_reduce_draw_rows(dtg_ctx* c, int n_draws, const double* d_rows, int mode, double* out) {
  return guarded(c, [&] {
    if (mode != 0 && mode != 1) throw std::invalid_argument("reduce mode must be 0 or 1");
    if (n_draws < 1) throw std::invalid_argument("no noise draws");
    if (!d_rows && n_draws > c->B)
      throw std::invalid_argument("internal draw rows hold only B scenarios");
    const std::size_t R = 5 * static_cast<std::size_t>(c->L) + 2;
    c->red.ensure(R);
    if (!c->h_red) CK(cudaMallocHost(&c->h_red, R * 8));
    cudaStream_t st = c->stream;
    dtg::launch_reduce_rows(n_draws, c->L, d_rows ? d_rows : c->rows.p, mode, c->red.p, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->h_red, c->red.p, R * 8, cudaMemcpyDeviceToHost, st));
    c->sync_check();
    std::memcpy(out, c->h_red, R * 8);
  });
}

// ---- device-resident calibrate step -------------------------------------------------
// The host loop of calibrate (optimization.cpp:173-205) realises (u, kappa,
// beta, alpha) from raw through BoundedTransform, chains the draw-summed
// gradient through its derivative and takes an AdamW step (optimization.cpp:
// 10-59).  The same operations run here on the device, in the same order,
// with glibc's exp restated (dexp) and IEEE sqrt / division: the raw
// trajectory is bit-identical to the host's, and an iteration no longer waits
// for a 100 KB gradient row to cross PCIe and 20k host exponentials.
namespace {
struct OptArgs {
  double lo[4], hi[4];
  double lr, b1, b2, eps, wd, bc1, bc2, draws;
  int step;  // 0: realise only
};
__device__ __forceinline__ double sigmoid_branchy_d(double r) {
  return r >= 0.0 ? 1.0 / (1.0 + dtg::dexp(-r)) : dtg::dexp(r) / (1.0 + dtg::dexp(r));
}
__global__ void k_opt_bounded(double* raw, double* m, double* v, const double* red, OptArgs a, double* params,
                              int L, int B) {
  const std::size_t n = static_cast<std::size_t>(4) * L;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(i / L), l = static_cast<int>(i % L);
    const double lo = a.lo[q], hi = a.hi[q];
    double r = raw[i];
    if (a.step) {
      const double s = sigmoid_branchy_d(r);
      const double g = red[i] / a.draws * ((hi - lo) * s * (1.0 - s));  // rg = red / draws * dvalue(raw)
      const double mi = a.b1 * m[i] + (1.0 - a.b1) * g;
      const double vi = a.b2 * v[i] + (1.0 - a.b2) * g * g;
      m[i] = mi;
      v[i] = vi;
      const double mhat = mi / a.bc1;
      const double vhat = vi / a.bc2;
      r -= a.lr * (mhat / (sqrt(vhat) + a.eps) + a.wd * r);
      raw[i] = r;
    }
    const double p = lo + (hi - lo) * sigmoid_branchy_d(r);  // BoundedTransform::value
    for (int b = 0; b < B; ++b) params[(static_cast<std::size_t>(q) * B + b) * L + l] = p;
  }
}
void launch_opt(dtg_ctx* c, int step, int draws, double bc1, double bc2) {
  OptArgs a{};
  for (int q = 0; q < 4; ++q) {
    a.lo[q] = c->opt_lo[q];
    a.hi[q] = c->opt_hi[q];
  }
  a.lr = c->opt_lr;
  a.b1 = c->opt_b1;
  a.b2 = c->opt_b2;
  a.eps = c->opt_eps;
  a.wd = c->opt_wd;
  a.bc1 = bc1;
  a.bc2 = bc2;
  a.draws = static_cast<double>(draws);
  a.step = step;
  const int n = 4 * c->L;
  k_opt_bounded<<<(n + 255) / 256, 256, 0, c->stream>>>(c->opt_raw.p, c->opt_m.p, c->opt_v.p, c->red.p, a,
                                                         c->params.p, c->L, c->B);
  CK(cudaGetLastError());
}
}  // namespace

int dtg_opt_bounded_init(dtg_ctx* c, const double* raw, const double* lo, const double* hi, double lr,
                         double beta1, double beta2, double eps, double weight_decay) {
  return guarded(c, [&] {
    for (int b = 0; b < c->B; ++b)
      if (!c->have_params[b]) throw std::invalid_argument("set the parameters (incl. cost) first");
    const std::size_t n = 4 * static_cast<std::size_t>(c->L);
    c->opt_raw.ensure(n);
    c->opt_m.ensure(n);
    c->opt_v.ensure(n);
    c->opt_best.ensure(n);
    for (int q = 0; q < 4; ++q) {
      c->opt_lo[q] = lo[q];
      c->opt_hi[q] = hi[q];
    }
    c->opt_lr = lr;
    c->opt_b1 = beta1;
    c->opt_b2 = beta2;
    c->opt_eps = eps;
    c->opt_wd = weight_decay;
    CK(cudaMemcpyAsync(c->opt_raw.p, raw, n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->opt_m.p, 0, n * 8, c->stream));
    CK(cudaMemsetAsync(c->opt_v.p, 0, n * 8, c->stream));
    CK(cudaMemcpyAsync(c->opt_best.p, c->opt_raw.p, n * 8, cudaMemcpyDeviceToDevice, c->stream));
    launch_opt(c, 0, 1, 1.0, 1.0);  // the parameters of raw
    CK(cudaStreamSynchronize(c->stream));  // raw is the caller's
    c->opt_ready = true;
  });
}

int dtg_opt_bounded_step(dtg_ctx* c, int draws, double bc1, double bc2) {
  return guarded(c, [&] {
    if (!c->opt_ready) throw std::runtime_error("dtg_opt_bounded_init first");
    if (draws < 1) throw std::invalid_argument("no noise draws");
    launch_opt(c, 1, draws, bc1, bc2);
  });
}

int dtg_opt_bounded_mark_best(dtg_ctx* c) {
  return guarded(c, [&] {
    if (!c->opt_ready) throw std::runtime_error("dtg_opt_bounded_init first");
    CK(cudaMemcpyAsync(c->opt_best.p, c->opt_raw.p, 4 * static_cast<std::size_t>(c->L) * 8,
                       cudaMemcpyDeviceToDevice, c->stream));
  });
}

int dtg_opt_bounded_read(dtg_ctx* c, double* raw, double* best_raw) {
  return guarded(c, [&] {
    if (!c->opt_ready) throw std::runtime_error("dtg_opt_bounded_init first");
    const std::size_t n = 4 * static_cast<std::size_t>(c->L);
    if (raw) CK(cudaMemcpyAsync(raw, c->opt_raw.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
    if (best_raw) CK(cudaMemcpyAsync(best_raw, c->opt_best.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int dtg_reduce_draw_rows_head(dtg_ctx* c, int n_draws, const double* d_rows, int mode, double* head) {
  return guarded(c, [&] {
    if (mode != 0 && mode != 1) throw std::invalid_argument("reduce mode must be 0 or 1");
    if (n_draws < 1) throw std::invalid_argument("no noise draws");
    if (!d_rows && n_draws > c->B)
      throw std::invalid_argument("internal draw rows hold only B scenarios");
    const std::size_t R = 5 * static_cast<std::size_t>(c->L) + 2;
    c->red.ensure(R);
    if (!c->h_red) CK(cudaMallocHost(&c->h_red, R * 8));
    cudaStream_t st = c->stream;
    dtg::launch_reduce_rows(n_draws, c->L, d_rows ? d_rows : c->rows.p, mode, c->red.p, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->h_red + (R - 2), c->red.p + (R - 2), 2 * 8, cudaMemcpyDeviceToHost, st));
    c->sync_check();
    head[0] = c->h_red[R - 2];
    head[1] = c->h_red[R - 1];
  });
}

int dtg_read_reduced_row(dtg_ctx* c, double* out) {
  return guarded(c, [&] {
    const std::size_t R = 5 * static_cast<std::size_t>(c->L) + 2;
    if (c->red.n < R) throw std::runtime_error("no reduced row");
    CK(cudaMemcpyAsync(out, c->red.p, R * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int dtg_profile_kernels(dtg_ctx* c, int T, int spi, int backward, double* ms_out,
                        int64_t* launches_out) {
  return guarded(c, [&] {
    if (T < 1) throw std::invalid_argument("profile needs at least one step");
    c->sync_check();
    // The launch sequence is captured into a CUDA graph with an event record
    // node before and after every kernel, so kernels run back to back exactly
    // as in the production graph and each event pair brackets one kernel.
    const int nk = backward ? dtg::kBwdKernels : dtg::kFwdKernels;
    for (int w = 0; w < nk; ++w) ms_out[w] = 0.0;
    cudaStream_t st = c->stream;
    std::vector<cudaEvent_t> ev(2 * static_cast<std::size_t>(nk) * T);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    struct EvGuard {
      std::vector<cudaEvent_t>& v;
      ~EvGuard() {
        for (auto e : v) cudaEventDestroy(e);
      }
    } guard{ev};
    std::size_t q = 0;
    std::int64_t launches = 0;
    std::function<void()> body;
    if (!backward) {
      c->ensure_history(T, 0);
      CK(cudaMemcpyAsync(c->seeds.p, c->h_seeds.data(), sizeof(std::uint64_t) * 2 * c->B,
                         cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
      body = [&] {
        const dtg::DevView d = c->view();
        const std::size_t BN = static_cast<std::size_t>(c->B) * c->N;
        const std::size_t BL = static_cast<std::size_t>(c->B) * c->L;
        dtg::launch_derive(d, c->derived.p, c->derived.p + BL, c->derived.p + 2 * BL, st);
      dtg::launch_pack_succ(d, c->srec.p, st);
        CK(cudaMemcpyAsync(c->pos.p, c->pos0.p, BN * 8, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(c->aid.p, c->aid0.p, BN * 4, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(c->lnk.p, c->lnk0.p, BN * 4, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(c->off.p, c->off0.p, static_cast<std::size_t>(c->B) * (c->L + 1) * 4,
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(c->qh.p, c->q0.p, BL * 8, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemsetAsync(c->cumh.p, 0, BL * 8, st));
        CK(cudaMemsetAsync(c->errf.p, 0, sizeof(int) * c->B, st));
        for (int t = 0; t < T; ++t)
          for (int w = 0; w < nk; ++w) {
            CK(cudaEventRecordWithFlags(ev[q++], st, cudaEventRecordExternal));
            dtg::launch_fwd_kernel(w, d, t, t % c->S, (t + 1) % c->S, st);
            CK(cudaEventRecordWithFlags(ev[q++], st, cudaEventRecordExternal));
            ++launches;
          }
      };
      c->last_T = T;
      c->last_spi = spi;
      c->last_ckpt = 0;
      c->last_K = T / spi;
    } else {
      if (c->last_T != T || !c->last_ckpt)
        throw std::runtime_error("profile(backward) needs a preceding dtg_forward(T, checkpoint=1)");
      run_backward(c, nullptr, nullptr, nullptr, cudaMemcpyHostToDevice);  // allocate + warm
      c->sync_check();
      body = [&] {
        dtg::DevView d = c->view();
        d.alist = c->alist.p;
        d.acount = c->acount.p;
        const std::size_t B = c->B, N = c->N;
        const int K = c->last_K;
        CK(cudaMemsetAsync(c->acount.p, 0, B * sizeof(int), st));
        double* xb[2] = {c->xbar.p, c->xbar.p + B * N};
        dtg::launch_adj_init(d, T % c->S, c->x_seed.p, xb[T & 1], c->cum_seed.p, st);
        for (int t = T - 1; t >= 0; --t) {
          const int snap_k = ((t + 1) % spi == 0) ? (t + 1) / spi - 1 : -1;
          for (int w = 0; w < nk; ++w) {
            CK(cudaEventRecordWithFlags(ev[q++], st, cudaEventRecordExternal));
            dtg::launch_bwd_kernel(w, d, t, t % c->S, (t + 1) % c->S, xb[(t + 1) & 1], xb[t & 1],
                                   c->snap_seed.p, snap_k, K, c->sort_scratch.p, c->force_slow, st);
            CK(cudaEventRecordWithFlags(ev[q++], st, cudaEventRecordExternal));
            ++launches;
          }
        }
      };
    }
    cudaGraph_t g;
    cudaGraphExec_t ex = nullptr;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    body();
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    CK(cudaGraphLaunch(ex, st));  // warm
    CK(cudaStreamSynchronize(st));
    CK(cudaGraphLaunch(ex, st));
    CK(cudaStreamSynchronize(st));
    cudaGraphExecDestroy(ex);
    c->pending = true;
    c->sync_check();
    for (std::size_t p = 0; p < q; p += 2) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev[p], ev[p + 1]));
      ms_out[(p / 2) % nk] += ms;
    }
    if (launches_out) *launches_out = launches;
  });
}

const char* dtg_kernel_name(int backward, int which) {
  if (backward) return which >= 0 && which < dtg::kBwdKernels ? dtg::kBwdKernelNames[which] : "";
  return which >= 0 && which < dtg::kFwdKernels ? dtg::kFwdKernelNames[which] : "";
}

int dtg_debug_gumbel(uint64_t seed, uint64_t key, int n, const uint64_t* rows,
                     const uint64_t* cols, double* out) {
  return guarded(nullptr, [&] {
    DevBuf<std::uint64_t> r, c;
    DevBuf<double> o;
    r.alloc(n);
    c.alloc(n);
    o.alloc(n);
    CK(cudaMemcpy(r.p, rows, n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.p, cols, n * 8, cudaMemcpyHostToDevice));
    dtg::launch_gumbel_batch(seed, key, r.p, c.p, n, o.p, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, o.p, n * 8, cudaMemcpyDeviceToHost));
  });
}

int dtg_debug_force_slow_path(dtg_ctx* c, int on) {
  c->force_slow = on ? 1 : 0;
  c->drop_graphs();
  return DTG_OK;
}

}  // extern "C"
