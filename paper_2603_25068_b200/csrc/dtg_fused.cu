// Fused forward engine: all T engine steps of all B scenarios in ONE launch,
// two barriers per step.  One template, two schedules:
//   kCluster = false  a cooperative grid; a scenario owns `nblk` CTAs and all
//                     CTAs meet at grid barriers (default schedule);
//   kCluster = true   one thread-block cluster per scenario with hardware
//                     cluster barriers; independent clusters never wait for
//                     each other.
//
// Step t (engine_step, src/engine.cpp:70-125):
//   slot phase   each CTA derives layout t's segment offsets in shared memory
//                from layout t-1's (kept in smem across steps) and step t-1's
//                departures / entrants (staged in smem), pulls its slots of
//                layout t from step t-1 (stable compaction, entrants at 0.0),
//                writes the checkpoint, runs car-following with per-link
//                constants from smem, writes the prefix-boundary counts; an
//                arrived head draws its next link (first-stage log-softmax
//                precomputed per link), draws its own merge Gumbel for that
//                link and registers {alpha, g, slot, id, link} with one atomic.
//   barrier
//   link phase   count/cum update, vacancy, merge softmax over the registered
//                records in ascending id, departures.
//   barrier
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "dtg_cluster.h"
#include "dtg_device.cuh"
#include "dtg_merge.cuh"

#ifndef DTG_SCALAR_HEAD_DRAWS
#define DTG_SCALAR_HEAD_DRAWS 0
#endif

namespace cg = cooperative_groups;

#ifndef DTG_BAR_BACKOFF
#define DTG_BAR_BACKOFF 32  // ns between grid-barrier polls: C3 nowcast 1.305 -> 1.295 ms
#endif

namespace dtg {

namespace {

// kBatch: slots per thread in flight together (2; 1 when every thread owns at
// most one slot, which leaves the arrived-head draw chains more registers).
// Measured at dn=1 (1M agents): 2 beats 4 by 11% (4 slots' state under the
// 128-register cap made ptxas rematerialise addresses in the loop) and 1 and 3
// are slower.
constexpr int kHeadCap = 1024;  // deferred arrived heads per CTA (overflow runs inline)

constexpr int kFastDeg = 5;  // successor counts up to this take the unrolled head path

// Link choice of one arrived head (node_model.cpp:45-97, first stage
// precomputed per link) and its own merge noise for the chosen row; registers
// the head as a merge column {alpha, g', slot, id, link} of that row.
//
// For deg <= kFastDeg the successor draws are fully unrolled so their RNG/log
// chains are independent instructions the scheduler interleaves (the heads are
// the critical path of the slot phase); the softmax runs on registers with the
// same operations in the same order as softmax_stage2.
// The decision of agent a at the end of link j: chosen successor c and its own
// merge Gumbel g'(t, c, a) (h1l / h1m: the step's stream prefixes).
__device__ __forceinline__ void head_draw(const CView& V, std::uint64_t h1l, std::uint64_t h1m, int j,
                                          int a, const int* soff_s, const double* slz, int& c_out,
                                          double& g_out) {
  const DevView& d = V.d;
  const int sb = soff_s[j], deg = soff_s[j + 1] - sb;
  const double* lz = slz + static_cast<std::size_t>(j) * d.maxdeg;
  const std::uint64_t h2l = rng_prefix2(h1l, static_cast<std::uint64_t>(a));
  int c;
  if (deg <= kFastDeg) {
    int sj[kFastDeg];
    double y[kFastDeg], ex[kFastDeg];
#pragma unroll
    for (int e = 0; e < kFastDeg; ++e) sj[e] = d.succ[sb + (e < deg ? e : 0)];
#if DTG_SCALAR_HEAD_DRAWS
    int bad = 0;
#pragma unroll
    for (int e = 0; e < kFastDeg; ++e)
      y[e] = (lz[e < deg ? e : 0] + gumbel_sl(rng_final(h2l, static_cast<std::uint64_t>(sj[e])), bad)) * d.kinv;
#else
    // the five draw chains batched (dtg_device.cuh gumbel_draws)
    double gg[kFastDeg];
    gumbel_draws<kFastDeg>(h2l, sj, gg);
#pragma unroll
    for (int e = 0; e < kFastDeg; ++e) y[e] = (lz[e < deg ? e : 0] + gg[e]) * d.kinv;
#endif
    const int best = softmax_first_argmax<kFastDeg>(deg, y, ex);
    c = sj[best];
  } else {
    double g[kMaxDeg], pi[kMaxDeg];
    for (int e = 0; e < deg; ++e) g[e] = gumbel_bits(rng_final(h2l, static_cast<std::uint64_t>(d.succ[sb + e])));
    c = d.succ[sb + softmax_stage2<kMaxDeg>(deg, lz, g, d.kinv, pi)];
  }
  {
    int bad = 0;
    const std::uint64_t mb = rng_final(rng_prefix2(h1m, static_cast<std::uint64_t>(c)), static_cast<std::uint64_t>(a));
    g_out = gumbel_sl(mb, bad);
    if (bad) g_out = gumbel_bits(mb);
  }
  c_out = c;
}

// Speculative decisions of the next step, 4 lanes per candidate: candidate
// u = 2 j + which is the which-th agent (0 leader, 1 follower) of link j in
// layout t (ids `aid`, step-t positions `x1`).  Lane e of the segment draws the
// link Gumbels of successors e and e + 4 and the agent's merge Gumbels for
// them (four independent chains); lane 0 gathers the y values, takes the first
// argmax with softmax_first_argmax's exact rule (the same operations as
// head_draw) and picks the chosen successor's merge draw.  A candidate is
// skipped when it cannot reach the arrival threshold in one step: its next
// position is at most fl(x1 + dxf), so fl(x1 + dxf) < L - 0.01 rules the
// arrival out exactly.  Links with more than 8 successors: lane 0 alone.
// Called warp-uniformly (every lane of the warp runs every shuffle).
constexpr int kSpecLanes = 4;
constexpr int kSpecDeg = 2 * kSpecLanes;
__device__ __forceinline__ void spec_segment(const CView& V, std::uint64_t h1l, std::uint64_t h1m,
                                             const int* aid, const double* x1, const int* offB,
                                             const int* soff_s, const double* slz, const double* dxf_l,
                                             const double* len_l, int v, int L, Spec* out) {
  const DevView& d = V.d;
  const int lane = threadIdx.x & 31, e = v & (kSpecLanes - 1), lead = lane & ~(kSpecLanes - 1);
  const int u = v / kSpecLanes;
  const bool in = u < 2 * L;
  const int j = in ? (u >> 1) : 0, which = u & 1;
  const int sb = soff_s[j], deg = soff_s[j + 1] - sb;
  const bool wide = deg > kSpecDeg;
  bool act = in && which < offB[j + 1] - offB[j] && deg > 0;
  // every global load of the segment issued together (one memory latency)
  const int k = act ? offB[j] + which : 0;
  const double xk = act ? x1[k] : 0.0;
  const int a = act ? aid[k] : -1;
  const double* lz = slz + static_cast<std::size_t>(j) * d.maxdeg;
  int sjv[2];
  double lzv[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ee = e + h * kSpecLanes;
    const int ec = (act && !wide && ee < deg) ? ee : 0;
    sjv[h] = act ? d.succ[sb + ec] : 0;
    lzv[h] = act ? lz[ec] : 0.0;
  }
  act = act && xk + dxf_l[j] >= len_l[j] - kArrivalTol;
  double y[2] = {0.0, 0.0}, gm[2] = {0.0, 0.0};
  if (act && !wide) {
    const std::uint64_t h2l = rng_prefix2(h1l, static_cast<std::uint64_t>(a));
    // the four chains (two link, two merge draws) batched
    std::uint64_t bb[4];
    double gg[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const std::uint64_t sj = static_cast<std::uint64_t>(sjv[h]);
      bb[h] = rng_final(h2l, sj);
      bb[2 + h] = rng_final(rng_prefix2(h1m, sj), static_cast<std::uint64_t>(a));
    }
    int bad = 0;
#if DTG_SCALAR_HEAD_DRAWS
#pragma unroll
    for (int q = 0; q < 4; ++q) gg[q] = gumbel_sl(bb[q], bad);
#else
    gumbel_sl_v<4>(bb, gg, bad);
#endif
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      gm[h] = gg[2 + h];
      y[h] = (lzv[h] + gg[h]) * d.kinv;
    }
  }
  double yv[kSpecDeg], ex[kSpecDeg];
#pragma unroll
  for (int q = 0; q < kSpecLanes; ++q) {
    yv[q] = __shfl_sync(0xffffffffu, y[0], lead + q);
    yv[q + kSpecLanes] = __shfl_sync(0xffffffffu, y[1], lead + q);
  }
  int best = 0;
  if (act && !wide && e == 0) best = softmax_first_argmax<kSpecDeg>(deg, yv, ex);
  best = __shfl_sync(0xffffffffu, best, lead);
  const double g0 = __shfl_sync(0xffffffffu, gm[0], lead + (best & (kSpecLanes - 1)));
  const double g1 = __shfl_sync(0xffffffffu, gm[1], lead + (best & (kSpecLanes - 1)));
  if (e != 0 || !in) return;
  Spec r;
  r.aid = -1;
  r.c = -1;
  r.g = 0.0;
  if (act) {
    r.aid = a;
    if (!wide) {
      r.c = d.succ[sb + best];
      r.g = best < kSpecLanes ? g0 : g1;
    } else {
      head_draw(V, h1l, h1m, j, a, soff_s, slz, r.c, r.g);
    }
  }
  out[u] = r;
}

// The same decisions for a CTA-local candidate list (split schedule): entry i
// of the list is (link, which, agent), already filtered by its slot owner.
// One lane per candidate (head_draw's chain; the ~3.5 us the link warps spend
// on the grid barrier and the link phase cover it) over warps 2.. of the CTA,
// so even a CTA whose 512 slots hold hundreds of short links finishes in one
// round.
__device__ __forceinline__ void spec_list(const CView& V, std::uint64_t h1l, std::uint64_t h1m,
                                          const int* lst, int n, int cap, const int* soff_s,
                                          const double* slz, Spec* out) {
  for (int ci = static_cast<int>(threadIdx.x) - 64; ci < n; ci += static_cast<int>(blockDim.x) - 64) {
    const int j = lst[ci], which = lst[cap + ci], a = lst[2 * cap + ci];
    Spec r;
    r.aid = a;
    head_draw(V, h1l, h1m, j, a, soff_s, slz, r.c, r.g);
    out[static_cast<std::size_t>(j) * 2 + which] = r;
  }
}

// Link choice of one arrived head and its merge registration; the decision
// comes from the speculative records when one of them is this agent's.
__device__ __forceinline__ void head_choice(const CView& V, std::size_t bl, std::uint64_t h1l,
                                            std::uint64_t h1m, int k, int j, int a, const int* soff_s,
                                            const double* slz, const Spec* sp, const Spec* pre = nullptr) {
  const DevView& d = V.d;
  int c;
  double g;
  if (pre && pre[0].aid == a) {  // records prefetched by the caller
    c = pre[0].c;
    g = pre[0].g;
  } else if (pre && pre[1].aid == a) {
    c = pre[1].c;
    g = pre[1].g;
  } else if (!pre && sp && sp[0].aid == a) {
    c = sp[0].c;
    g = sp[0].g;
  } else if (!pre && sp && sp[1].aid == a) {
    c = sp[1].c;
    g = sp[1].g;
  } else {
    head_draw(V, h1l, h1m, j, a, soff_s, slz, c, g);
  }
  Cand cd;
  cd.alpha = d.alpha[bl + j];
  cd.g = g;
  cd.slot = k;
  cd.aid = a;
  cd.link = j;
  cd.pad = 0;
  const int qq = atomicAdd(&V.ccnt[bl + c], 1);
  if (qq < kClusterCandCap) V.cands[(bl + c) * kClusterCandCap + qq] = cd;
}

// Link of slot k: the last j in [lo, hi] with off_s[j] <= k.
__device__ __forceinline__ int find_link_w(const int* off_s, int lo, int hi, int k) {
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off_s[mid] <= k)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

template <bool kMask = false>
__device__ __forceinline__ int pull_f(int j, int rn, const int* offA, const int* offB, const int* na_s,
                                      const int* dep_s, const int* win_s, const int* wonp, bool* entrant) {
  const int w = win_s[j];
  if (w >= 0 && rn == offB[j + 1] - offB[j] - 1) {
    *entrant = true;
    return w;
  }
  *entrant = false;
  const int ob = offA[j];
  const int na = (!kMask || offA[j + 1] > ob) ? na_s[j] : 0;  // lean layout: the unmasked global array
  const int dp = dep_s[j];
  if (rn >= na - dp) return ob + rn + dp;
  int c = -1;
  for (int q = 0; q < na; ++q)
    if (!wonp[ob + q] && ++c == rn) return ob + q;
  return ob;
}

// Exclusive scan of v[0..n) in place, v[n] = total; two CTA barriers: every
// warp scans the warp totals itself instead of waiting for warp 0 to do it.
__device__ void scan_f(int* v, int n, int* tmp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int j0 = min(n, tid * per), j1 = min(n, j0 + per);
  int s = 0;
  for (int j = j0; j < j1; ++j) s += v[j];
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  int x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  int wt = lane < nw ? tmp[lane] : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, wt, o);
    if (lane >= o) wt += y;
  }
  const int before = __shfl_sync(0xffffffffu, wt, wid > 0 ? wid - 1 : 0);
  const int total = __shfl_sync(0xffffffffu, wt, nw - 1);
  int run = (wid ? before : 0) + x - s;
  for (int j = j0; j < j1; ++j) {
    const int c = v[j];
    v[j] = run;
    run += c;
  }
  if (tid == 0) v[n] = total;
  __syncthreads();
}

__device__ __forceinline__ unsigned long long gnow() {
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  return ns;
}

__device__ __forceinline__ void fstamp(const CView& V, int t, int w) {
  if (V.tstamp == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    V.tstamp[(static_cast<std::size_t>(t) * gridDim.x + blockIdx.x) * 4 + w] = ns;
  }
}

// Grid barrier: one release-add per CTA on a monotone counter, acquire spin.
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned int target = epoch * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
#if DTG_BAR_BACKOFF
            if (v < target) __nanosleep(DTG_BAR_BACKOFF);
#endif
    } while (v < target);
  }
  __syncthreads();
}

}  // namespace

// kFeat: the optional features (host-mapped progress, speculative head
// decisions) are compiled in; without them the kernel is the plain schedule
// (their mere presence costs the many-slots-per-thread variant ~10%).
template <bool kCluster, int kBatch, bool kFeat, bool kLean>
__global__ void __launch_bounds__(kClusterThreads, 1) k_forward_fused(CView V) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const DevView& d = V.d;
  const int L = d.L, N = d.N;
  int rank, b;
  if (kCluster) {
    rank = static_cast<int>(cg::this_cluster().block_rank());
    b = blockIdx.x / V.cs;
  } else {
    rank = blockIdx.x % V.cs;
    b = blockIdx.x / V.cs;
  }
  const bool active = b < d.B;
  const int nthr = V.cs * blockDim.x;
  unsigned int epoch = 0;
  auto barrier = [&]() {
    if (kCluster)
      cg::this_cluster().sync();
    else if (V.gbar)
      grid_barrier(V.gbar, epoch);
    else
      cg::this_grid().sync();
  };
  // ---- shared memory layout ----
  double *jam_s = nullptr, *dxf_s = nullptr, *len_s = nullptr;
  double* dp = reinterpret_cast<double*>(sm_raw);
  if (V.stage_params) {
    jam_s = dp;
    dxf_s = dp + L;
    len_s = dp + 2 * L;
    dp += 3 * L;
  }
  int* ip = reinterpret_cast<int*>(dp);
  int* offA = ip;
  int* offB = ip + (L + 1);
  // lean layout (networks whose per-link arrays do not fit shared memory):
  // succ_off / pred_off are read from global memory, and the pulls read the
  // previous step's arrived / departure / winner arrays directly
  const int* na_s;
  const int* dep_s;
  const int* win_s;
  int *na_w = nullptr, *dep_w = nullptr, *win_w = nullptr;
  const int* soff_s;
  const int* poff_s;
  int* tmp;
  if (!kLean) {
    na_w = ip + 2 * (L + 1);
    dep_w = na_w + L;
    win_w = dep_w + L;
    na_s = na_w;
    dep_s = dep_w;
    win_s = win_w;
    soff_s = win_w + L;               // succ_off, L + 1
    poff_s = soff_s + (L + 1);        // pred_off, L + 1
    tmp = const_cast<int*>(poff_s) + (L + 1);
  } else {
    na_s = dep_s = win_s = nullptr;
    soff_s = d.succ_off;
    poff_s = d.pred_off;
    tmp = ip + 2 * (L + 1);
  }
  int* hcnt = tmp + 34;              // deferred-head count
  int* hq = tmp + 36;                // [3][kHeadCap] deferred heads: slot, link, agent
  const int bb = active ? b : 0;
  const std::size_t bl = static_cast<std::size_t>(bb) * L;
  const std::size_t bn = static_cast<std::size_t>(bb) * N;
  const std::size_t BL = static_cast<std::size_t>(d.B) * L;
  const std::size_t BN = static_cast<std::size_t>(d.B) * N;
  if (active) {
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
      if (V.stage_params) {
        jam_s[j] = d.jam[bl + j];
        dxf_s[j] = d.dxf[bl + j];
        len_s[j] = d.len[j];
      }
      if (!kLean) {
        const_cast<int*>(soff_s)[j] = d.succ_off[j];
        const_cast<int*>(poff_s)[j] = d.pred_off[j];
      }
    }
    if (threadIdx.x == 0 && !kLean) {
      const_cast<int*>(soff_s)[L] = d.succ_off[L];
      const_cast<int*>(poff_s)[L] = d.pred_off[L];
    }
    const int* og = d.off + oidx(d, 0, bb);
    for (int j = threadIdx.x; j <= L; j += blockDim.x) offB[j] = og[j];
  }
  __syncthreads();
  const std::uint64_t seed_link = d.seed_link[bb], seed_merge = d.seed_merge[bb];
  const double* slz = d.slogz + bl * d.maxdeg;

  for (int t = 0; t <= V.T; ++t) {
    const bool last = t == V.T;
    const int cur = t & 1, prv = cur ^ 1;
    const std::uint64_t h1l = rng_prefix1(seed_link, static_cast<std::uint64_t>(t));
    const std::uint64_t h1m = rng_prefix1(seed_merge, static_cast<std::uint64_t>(t));
    // this step's speculative head decisions (drawn in step t-1's link phase)
    const Spec* spec_t = (kFeat && V.spec && t > 0) ? V.spec + ((t & 1) * BL + bl) * 2 : nullptr;
    // split schedule: the slot owners list the next step's candidates in shared
    // memory; warps 2.. draw them while warps 0-1 wait at the grid barrier
    const bool split = kFeat && kBatch == 1 && !kCluster && V.spec && V.spec_split && V.gbar && !last;
    if (!last) fstamp(V, t, 0);
    if (kFeat && V.progress && t > 0 && (t % V.progress_every == 0 || last) && blockIdx.x == 0 &&
        threadIdx.x == 0) {
      // this thread acquired every CTA's step t-1 writes at the barrier; the
      // system-scope fence makes them visible to the copy engine before t is
      __threadfence_system();
      *V.progress = static_cast<unsigned int>(t);
    }
    const unsigned long long wst0 = V.wstamp ? gnow() : 0;
    unsigned long long wt1 = 0;
    int n_arr = 0;
    if (active) {
      // ---------------- slot phase ----------------
      if (t > 0) {
        int* sw = offA;
        offA = offB;
        offB = sw;
        const int* nAp = V.nAb + prv * BL + bl;
        const int* depp = V.depb + prv * BL + bl;
        if (kLean) {
          na_s = nAp;
          dep_s = depp;
          win_s = V.win + bl;
        }
        // all global loads of this thread's links first (one memory latency),
        // then the shared-memory updates
        constexpr int kPro = 8;
        const int per = (L + blockDim.x - 1) / blockDim.x;
        if (per <= kPro) {
          // each thread owns the contiguous links [j0, j0 + per): the new
          // segment sizes stay in registers for the scan (one CTA barrier less
          // than writing them to shared memory for scan_f)
          const int j0 = min(L, static_cast<int>(threadIdx.x) * per);
          const int j1 = min(L, j0 + per);
          int na_r[kPro], dp_r[kPro], w_r[kPro], sz[kPro];
#pragma unroll
          for (int u = 0; u < kPro; ++u) {
            const int j = j0 + u;
            const bool on = j < j1;
            na_r[u] = on ? nAp[j] : 0;
            dp_r[u] = on ? depp[j] : 0;
            w_r[u] = on ? V.win[bl + j] : -1;
          }
          int sum = 0;
#pragma unroll
          for (int u = 0; u < kPro; ++u) {
            const int j = j0 + u;
            sz[u] = 0;
            if (j < j1) {
              const int nold = offA[j + 1] - offA[j];
              if (!kLean) {
                na_w[j] = nold ? na_r[u] : 0;
                dep_w[j] = dp_r[u];
                win_w[j] = w_r[u];
              }
              sz[u] = nold - dp_r[u] + (w_r[u] >= 0 ? 1 : 0);
              sum += sz[u];
            }
          }
          // exclusive block scan of the per-thread sums (as scan_f)
          const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
          int x = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          if (lane == 31) tmp[wid] = x;
          __syncthreads();
          int wt = lane < nw ? tmp[lane] : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, wt, o);
            if (lane >= o) wt += y;
          }
          const int before = __shfl_sync(0xffffffffu, wt, wid > 0 ? wid - 1 : 0);
          const int total = __shfl_sync(0xffffffffu, wt, nw - 1);
          int run = (wid ? before : 0) + x - sum;
#pragma unroll
          for (int u = 0; u < kPro; ++u)
            if (j0 + u < j1) {
              offB[j0 + u] = run;
              run += sz[u];
            }
          if (threadIdx.x == 0) offB[L] = total;
          __syncthreads();
        } else {
        for (int j0 = threadIdx.x; j0 < L; j0 += kPro * blockDim.x) {
          int na_r[kPro], dp_r[kPro], w_r[kPro];
#pragma unroll
          for (int u = 0; u < kPro; ++u) {
            const int j = j0 + u * blockDim.x;
            const bool on = j < L;
            na_r[u] = on ? nAp[j] : 0;
            dp_r[u] = on ? depp[j] : 0;
            w_r[u] = on ? V.win[bl + j] : -1;
          }
#pragma unroll
          for (int u = 0; u < kPro; ++u) {
            const int j = j0 + u * blockDim.x;
            if (j < L) {
              const int nold = offA[j + 1] - offA[j];
              if (!kLean) {
                na_w[j] = nold ? na_r[u] : 0;
                dep_w[j] = dp_r[u];
                win_w[j] = w_r[u];
              }
              offB[j] = nold - dp_r[u] + (w_r[u] >= 0 ? 1 : 0);
            }
          }
        }
        __syncthreads();
        scan_f(offB, L, tmp);
        }
        if (rank == 0) {
          int* on = d.off + oidx(d, t % d.S, bb);
          for (int j = threadIdx.x; j <= L; j += blockDim.x) on[j] = offB[j];
          if (threadIdx.x == 0 && offB[L] != N) atomicOr(&d.err[bb], kErrConservation);
        }
      }
      const std::size_t so = sidx(d, t % d.S, bb);
      const std::size_t sp = t > 0 ? sidx(d, (t - 1) % d.S, bb) : 0;
      const double* x1p = V.x1b + prv * BN + bn;
      const int* wonp = V.wonb + prv * BN + bn;
      double* x1c = V.x1b + cur * BN + bn;
      int* wonc = V.wonb + cur * BN + bn;
      int* nAc = V.nAb + cur * BL + bl;
      int* qnc = V.qnb + cur * BL + bl;
      double* tailc = V.tailb + cur * BL + bl;
      // Slot mapping.  Contiguous: this CTA owns [ka, kb) (32-aligned, so no
      // warp straddles two CTAs) and the link search is narrowed to the links
      // that range covers.  Interleaved: 512-slot blocks round-robin over the
      // scenario's CTAs, which spreads dense runs of arrived heads when every
      // thread owns several slots.
      int off0, stride, limit, jA = 0, jB = L - 1;
      if (V.contig) {
        const int per = ((N + V.cs - 1) / V.cs + 31) & ~31;
        off0 = min(N, rank * per);
        limit = min(N, off0 + per);
        stride = blockDim.x;
        int* win2 = tmp + 32;
        if (threadIdx.x == 0) win2[0] = off0 < limit ? find_link_w(offB, 0, L - 1, off0) : 0;
        if (threadIdx.x == 32) win2[1] = off0 < limit ? find_link_w(offB, 0, L - 1, limit - 1) : 0;
        __syncthreads();
        jA = win2[0];
        jB = win2[1];
      } else {
        off0 = rank * blockDim.x;
        limit = N;
        stride = nthr;
      }
      // When a thread owns several slot batches, arrived heads are queued in
      // shared memory and their link choices run after the loop, one per
      // thread, instead of serialising a draw chain into every batch.
      const bool defer = limit - off0 > stride;
      if (defer || split) {
        if (threadIdx.x == 0) *hcnt = 0;
        __syncthreads();
      }
      if (V.wstamp) wt1 = gnow();
      const int lane = threadIdx.x & 31;
      // Interleaved mapping: warp gw takes 32 * kBatch consecutive slots per
      // iteration (chunks dealt round-robin over all warps of the scenario),
      // so after one binary search the next sub-chunks' links are reached by a
      // short forward walk.  Contiguous mapping: the CTA's range as before.
      // (Used for long links, N >= 32 L; with short links the walk costs more
      // than the search and the 512-slot blocks spread heads better.)
      const bool chunked = !V.contig && N >= 32 * L;
      const int wpc = blockDim.x >> 5;
      const int span = chunked ? 32 * kBatch : kBatch * stride;
      const int cstep = chunked ? V.cs * wpc : 1;
      const int c0 = chunked ? rank * wpc + (threadIdx.x >> 5) : 0;
      for (int c = c0;; c += cstep) {
        const int k0 = chunked ? c * span + lane : off0 + static_cast<int>(threadIdx.x) + c * span;
        if (k0 - lane >= limit) break;
        int kk[kBatch], jj[kBatch], rr[kBatch], nn[kBatch], aa[kBatch];
        double xx[kBatch], xl[kBatch], xn[kBatch];
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {  // segment lookup (smem)
          const int k = k0 + q * (chunked ? 32 : stride);
          const bool on = k < limit;
          kk[q] = on ? k : N;
          int j = 0;
          if (on) {
            if (q == 0 || !chunked) {
              j = find_link_w(offB, jA, jB, k);
            } else {
              j = jj[q - 1];
              while (offB[j + 1] <= k) ++j;
            }
          }
          jj[q] = j;
          rr[q] = k - offB[j];
          nn[q] = offB[j + 1] - offB[j];
        }
        // one slot per thread: a leader slot prefetches its link's speculative
        // records with the pulls (they are read only if it turns out arrived)
        Spec pre[2];
        pre[0].aid = pre[1].aid = -1;
        const bool use_pre = kFeat && kBatch == 1 && spec_t != nullptr && !last;
        if (use_pre && kk[0] < N && rr[0] == 0) {
          pre[0] = spec_t[static_cast<std::size_t>(jj[0]) * 2];
          pre[1] = spec_t[static_cast<std::size_t>(jj[0]) * 2 + 1];
        }
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {  // pull (all loads issued before use)
          const int k = kk[q], j = jj[q], r = rr[q], n = nn[q];
          // the warp's edge lanes also pull the neighbour outside the warp
          const bool need_l = !last && lane == 0 && r > 0;
          const bool need_n = !last && lane == 31 && r + 1 < n;
          xl[q] = 0.0;
          if (k >= N) {
            xx[q] = 0.0;
            aa[q] = 0;
            continue;
          }
          if (t == 0) {
            xx[q] = d.pos[so + k];
            aa[q] = d.aid[so + k];
            if (need_l || need_n) xl[q] = d.pos[so + k + (need_l ? -1 : 1)];
          } else {
            bool e0, e1 = false;
            const int s0 = pull_f<kLean>(j, r, offA, offB, na_s, dep_s, win_s, wonp, &e0);
            int s1 = s0;
            if (need_l || need_n) s1 = pull_f<kLean>(j, need_l ? r - 1 : r + 1, offA, offB, na_s, dep_s, win_s, wonp, &e1);
            const double v0 = x1p[s0], v1 = x1p[s1];
            aa[q] = d.aid[sp + s0];
            xx[q] = e0 ? 0.0 : v0;  // entrant: -M + M == 0.0 exactly
            xl[q] = e1 ? 0.0 : v1;
          }
        }
        if (!last) {
          // neighbours in the same link are lanes -+1 of this batch
#pragma unroll
          for (int q = 0; q < kBatch; ++q) {
            const double up = __shfl_up_sync(0xffffffffu, xx[q], 1);
            const double dn = __shfl_down_sync(0xffffffffu, xx[q], 1);
            const double edge = xl[q];
            xl[q] = lane == 0 ? edge : up;
            xn[q] = lane == 31 ? edge : dn;
          }
        }
        if (t > 0) {
#pragma unroll
          for (int q = 0; q < kBatch; ++q)  // layout t (ids feed the next pull)
            if (kk[q] < N) {
              d.aid[so + kk[q]] = aa[q];
              if (V.ckpt || last) {  // positions / links: checkpoints and the final state only
                d.pos[so + kk[q]] = xx[q];
                d.lnk[so + kk[q]] = jj[q];
              }
            }
        }
        if (last) continue;
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
          const int k = kk[q];
          if (k >= N) continue;
          const int j = jj[q], r = rr[q], n = nn[q];
          const double x = xx[q];
          const double jam = V.stage_params ? jam_s[j] : d.jam[bl + j];
          const double dxf = V.stage_params ? dxf_s[j] : d.dxf[bl + j];
          const double len = V.stage_params ? len_s[j] : d.len[j];
          const double ctr = 0.5 * len, thr = len - kArrivalTol;
          const CfPick me = cf_step(x, r == 0 ? d.M : xl[q] - x, jam, dxf, len);
          x1c[k] = me.x1;
          bool fo_n = false, fa_n = false;
          if (r + 1 < n) {
            const CfPick nx = cf_step(xn[q], x - xn[q], jam, dxf, len);
            fo_n = nx.x1 >= ctr;
            fa_n = nx.x1 >= thr;
          }
          const bool fo = me.x1 >= ctr, fa = me.x1 >= thr;
          if (split && t + 1 < V.T && r <= 1 && soff_s[j + 1] > soff_s[j] && me.x1 + dxf >= thr) {
            // can head link j at step t+1 (fl(x1 + u dt) < L - 0.01 rules it out exactly)
            const int li = atomicAdd(hcnt, 1);
            if (li < kHeadCap) {
              hq[li] = j;
              hq[kHeadCap + li] = r;
              hq[2 * kHeadCap + li] = aa[q];
            }
          }
          if (r == 0 && !fo) qnc[j] = 0;
          if (fo && !fo_n) qnc[j] = r + 1;
          if (r == 0 && !fa) nAc[j] = 0;
          if (fa && !fa_n) nAc[j] = r + 1;
          if (r == n - 1) tailc[j] = me.x1;
          if (!fa) continue;
          ++n_arr;
          wonc[k] = 0;
          if (soff_s[j + 1] > soff_s[j] && !(V.dbg & 1)) {
            const int hi = defer ? atomicAdd(hcnt, 1) : kHeadCap;
            if (hi < kHeadCap) {
              hq[hi] = k;
              hq[kHeadCap + hi] = j;
              hq[2 * kHeadCap + hi] = aa[q];
            } else {
              head_choice(V, bl, h1l, h1m, k, j, aa[q], soff_s, slz,
                          spec_t ? spec_t + static_cast<std::size_t>(j) * 2 : nullptr, use_pre ? pre : nullptr);
            }
          }
        }
      }
      if (defer && !last) {
        __syncthreads();
        const int nh = min(*hcnt, kHeadCap);
        for (int i = threadIdx.x; i < nh; i += blockDim.x)
          head_choice(V, bl, h1l, h1m, hq[i], hq[kHeadCap + i], hq[2 * kHeadCap + i], soff_s, slz,
                      spec_t ? spec_t + static_cast<std::size_t>(hq[kHeadCap + i]) * 2 : nullptr);
      }
    }
    if (V.wstamp && active && !last) {
      const unsigned long long wt2 = gnow();
      const int na = __reduce_add_sync(0xffffffffu, n_arr);
      if ((threadIdx.x & 31) == 0) {
        const std::size_t w = (static_cast<std::size_t>(t) * gridDim.x + blockIdx.x) * (blockDim.x / 32) +
                              (threadIdx.x >> 5);
        V.wstamp[w * 4 + 0] = wst0;
        V.wstamp[w * 4 + 1] = wt1;
        V.wstamp[w * 4 + 2] = wt2;
        V.wstamp[w * 4 + 3] = static_cast<unsigned long long>(na);
      }
    }
    if (last) break;
    fstamp(V, t, 1);
    if (split && active) {
      __syncthreads();  // the slot phase and the candidate list are complete
      if (threadIdx.x == 0) {
        ++epoch;
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(V.gbar), "r"(1u) : "memory");
      }
      if (threadIdx.x < 64) {  // warps 0-1: the link phase after the barrier
        if (threadIdx.x == 0) {
          const unsigned int target = epoch * gridDim.x;
          unsigned int v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(V.gbar) : "memory");
#if DTG_BAR_BACKOFF
            if (v < target) __nanosleep(DTG_BAR_BACKOFF);
#endif
          } while (v < target);
        }
        asm volatile("bar.sync 1, 64;" ::: "memory");
      } else if (t + 1 < V.T) {  // warps 2..: the next step's decisions (no cross-CTA inputs)
        spec_list(V, rng_prefix1(seed_link, static_cast<std::uint64_t>(t + 1)),
                  rng_prefix1(seed_merge, static_cast<std::uint64_t>(t + 1)), hq, min(*hcnt, kHeadCap),
                  kHeadCap, soff_s, slz, V.spec + (((t + 1) & 1) * BL + bl) * 2);
      }
      if (V.tstamp && threadIdx.x == 0) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        V.tstamp[(static_cast<std::size_t>(t) * gridDim.x + blockIdx.x) * 4 + 2] = ns;
      }
    } else {
      barrier();
      fstamp(V, t, 2);
    }
    if (active) {
      // ---------------- link phase ----------------
      double* tailc = V.tailb + cur * BL + bl;
      const int* qnc = V.qnb + cur * BL + bl;
      int* wonc = V.wonb + cur * BN + bn;
      int* depc = V.depb + cur * BL + bl;
      int* depn = V.depb + prv * BL + bl;
      const double* qhp = d.qh + hidx(d, t, bb);
      const double* chp = d.cumh + hidx(d, t, bb);
      double* qhn = d.qh + hidx(d, t + 1, bb);
      double* chn = d.cumh + hidx(d, t + 1, bb);
      // links in 32-lane groups dealt round-robin over the CTAs first, so the
      // ~L/32 busy warps land on different SMs instead of filling the first few
      const int gw0 = (static_cast<int>(threadIdx.x) >> 5) * V.cs + rank;
      for (int i = gw0 * 32 + (threadIdx.x & 31); i < L; i += nthr) {
        const int n_i = offB[i + 1] - offB[i];
        const int cnt = (V.dbg & 2) ? 0 : V.ccnt[bl + i];
        const int qc = n_i ? qnc[i] : 0;
        const double tx = n_i ? tailc[i] : d.M;
        const double qpv = qhp[i], cpv = chp[i];
        const double a = static_cast<double>(qc) - qpv;  // inc = relu(q - qprev)
        chn[i] = cpv + (a >= 0.0 ? a : 0.0);
        qhn[i] = static_cast<double>(qc);
        const double jam = V.stage_params ? jam_s[i] : d.jam[bl + i];
        const bool vacant = tx > jam;  // vacancy_from_state (node_model.cpp:27-41)
        V.ccnt[bl + i] = 0;
        depn[i] = 0;
        int w = -1, wa = -1;
        if (vacant && cnt > 0) {
          if (cnt > kClusterCandCap) {
            atomicOr(&d.err[bb], kErrCandOverflow);
          } else if (cnt <= kFastDeg) {  // registers (dtg_merge.cuh)
            Cand c[kFastDeg];
            double lz[kFastDeg], pi[kFastDeg];
            const int best = merge_softmax_fast<kFastDeg, false>(cnt, V.cands + (bl + i) * kClusterCandCap, d.kinv,
                                                                 c, lz, pi);
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e)
              if (e < cnt && c[e].alpha == 0.0) atomicOr(&d.err[bb], kErrZeroAlpha);
            const Cand cb = pick_cand(c, best);
            w = cb.slot;
            wa = cb.aid;
            wonc[w] = 1;
            atomicAdd(&depc[cb.link], 1);
          } else {
            Cand c[kClusterCandCap];
            for (int e = 0; e < cnt; ++e) c[e] = V.cands[(bl + i) * kClusterCandCap + e];
            for (int x = 1; x < cnt; ++x) {  // ascending agent id (merge columns)
              const Cand key = c[x];
              int m = x - 1;
              while (m >= 0 && c[m].aid > key.aid) {
                c[m + 1] = c[m];
                --m;
              }
              c[m + 1] = key;
            }
            double v[kClusterCandCap], g[kClusterCandCap], lz[kClusterCandCap], pi[kClusterCandCap];
            for (int e = 0; e < cnt; ++e) {
              v[e] = c[e].alpha;
              g[e] = c[e].g;
              if (v[e] == 0.0) atomicOr(&d.err[bb], kErrZeroAlpha);
            }
            const int best = two_softmax<kClusterCandCap>(cnt, v, g, d.kinv, lz, pi);
            w = c[best].slot;
            wa = c[best].aid;
            wonc[w] = 1;
            atomicAdd(&depc[c[best].link], 1);
          }
        }
        V.win[bl + i] = w;
        if (d.ev) d.ev[(static_cast<std::size_t>(t) * d.B + bb) * L + i] = wa;
      }
      // threads without a link draw step t+1's decisions of every link's
      // first two agents while the merges run
      if (kFeat && V.spec && !split && t + 1 < V.T) {
        // whole warps past the link threads (Lr: L rounded up to a warp)
        const int Lr = (L + 31) & ~31;
        const int i0 = gw0 * 32 + (threadIdx.x & 31);
        if (i0 >= Lr) {
          const std::uint64_t n1l = rng_prefix1(seed_link, static_cast<std::uint64_t>(t + 1));
          const std::uint64_t n1m = rng_prefix1(seed_merge, static_cast<std::uint64_t>(t + 1));
          Spec* out = V.spec + (((t + 1) & 1) * BL + bl) * 2;
          const int* aid_t = d.aid + sidx(d, t % d.S, bb);
          const double* x1_t = V.x1b + cur * BN + bn;
          const double* dxf_l = V.stage_params ? dxf_s : d.dxf + bl;
          const double* len_l = V.stage_params ? len_s : d.len;
          const int lane = threadIdx.x & 31;
          for (int v = i0 - Lr; v - lane < 2 * L * kSpecLanes; v += nthr - Lr)
            spec_segment(V, n1l, n1m, aid_t, x1_t, offB, soff_s, slz, dxf_l, len_l, v, L, out);
        }
      }
    }
    fstamp(V, t, 3);
    barrier();
  }
}

static int fused_smem_full(int L, bool stage_params) {
  return (stage_params ? 3 * L * 8 : 0) + (2 * (L + 1) + 3 * L + 2 * (L + 1) + 36 + 3 * kHeadCap) * 4;
}
bool fused_lean(int L) { return fused_smem_full(L, false) > 200 * 1024; }
int fused_smem_bytes(int L, bool stage_params) {
  if (fused_lean(L)) return (2 * (L + 1) + 36 + 3 * kHeadCap) * 4;
  return fused_smem_full(L, stage_params);
}

namespace {
template <int KB, bool F>
const void* fused_fn(bool cluster) {
  return cluster ? reinterpret_cast<const void*>(k_forward_fused<true, KB, F, false>)
                 : reinterpret_cast<const void*>(k_forward_fused<false, KB, F, false>);
}
template <int KB, bool F>
const void* fused_fn_lean() {  // large networks: grid schedule only
  return reinterpret_cast<const void*>(k_forward_fused<false, KB, F, true>);
}
const void* fused_pick(bool cluster, bool one, bool feat, bool lean) {
  if (lean) {
    if (one) return feat ? fused_fn_lean<1, true>() : fused_fn_lean<1, false>();
    return feat ? fused_fn_lean<2, true>() : fused_fn_lean<2, false>();
  }
  if (one) return feat ? fused_fn<1, true>(cluster) : fused_fn<1, false>(cluster);
  return feat ? fused_fn<2, true>(cluster) : fused_fn<2, false>(cluster);
}
}  // namespace

cudaError_t launch_forward_fused(const CView& V, bool cluster, cudaStream_t st) {
  const int smem = fused_smem_bytes(V.d.L, V.stage_params != 0);
  // one slot per thread -> kBatch 1
  const bool one = V.d.N <= V.cs * kClusterThreads;
  const bool feat = V.progress != nullptr || V.spec != nullptr;
  if (V.lean && cluster) return cudaErrorInvalidConfiguration;  // lean layout: grid schedule only
  const void* fn = fused_pick(cluster, one, feat, V.lean != 0);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<CView*>(&V)};
  if (cluster) {
    if (V.cs > 8) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(V.d.B * V.cs);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = V.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
  }
  return cudaLaunchCooperativeKernel(fn, dim3(V.d.B * V.cs), dim3(kClusterThreads), args, smem, st);
}

int fused_max_grid(int L, bool stage_params) {
  int dev = 0, sms = 0, occ = 0, occ1 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = fused_smem_bytes(L, stage_params);
  const bool lean = fused_lean(L);
  const void* fns[4] = {lean ? fused_fn_lean<2, false>() : fused_fn<2, false>(false),
                        lean ? fused_fn_lean<1, false>() : fused_fn<1, false>(false),
                        lean ? fused_fn_lean<2, true>() : fused_fn<2, true>(false),
                        lean ? fused_fn_lean<1, true>() : fused_fn<1, true>(false)};
  for (const void* fn : fns)
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
  int best = INT_MAX;
  for (const void* fn : fns) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kClusterThreads, smem);
    best = std::min(best, occ);
  }
  (void)occ1;
  return best * sms;
}

int fused_max_cluster(int L, bool stage_params) {
  if (fused_lean(L)) return 0;  // the lean layout runs the grid schedule only
  const int smem = fused_smem_bytes(L, stage_params);
  for (const void* fn : {fused_fn<2, false>(true), fused_fn<1, false>(true), fused_fn<2, true>(true),
                         fused_fn<1, true>(true)}) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  const void* fn = fused_fn<2, true>(true);
  for (int cs = 16; cs >= 1; cs >>= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n > 0) return cs;
  }
  cudaGetLastError();
  return 0;
}

}  // namespace dtg

namespace dtg {
cudaError_t decision_stats_fused(int force, unsigned long long* count) { return decision_stats_tu(force, count); }
}  // namespace dtg
