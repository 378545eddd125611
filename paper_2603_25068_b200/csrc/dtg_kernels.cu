// sm_100a kernels for one engine step and its checkpointed VJP.
//
// Forward step t (reference engine_step, src/engine.cpp:70-125):
//   k_step_cf       one thread per agent slot: Newell car-following with the
//                   leader in the previous slot, per-link midpoint count and
//                   arrived-prefix length as segment-boundary writes, vacancy
//                   tail.
//   k_step_choice   one thread per link: the Gumbel-softmax link choice of its
//                   arrived agents.
//   k_step_merge    one thread per link: count/cumulative update, vacancy,
//                   merge-choice over the arrived heads of the predecessor links.
//   k_step_scan     one CTA per scenario: departures, new segment sizes and the
//                   exclusive scan to the next segment offsets.
//   k_step_transfer one thread per slot: compaction into the next layout
//                   (winners enter their new link at position 0.0, everyone
//                   else keeps x1 and its order).
// Reverse step (the per-step segment VJP of engine.cpp:388-415) replays the
// first four kernels from the step's checkpoint, then:
//   k_adj_node    per link: count adjoint and the merge-row VJP (transfer VJP
//                 seeds, softmax VJP, targeted routing to the first candidate).
//   k_adj_a0      per scenario: rows the reference routes to the first arrived
//                 agent (non-targeted rows, reduce_max first-index rule).
//   k_adj_choice  per link: link-choice VJP of the arrived heads.
//   k_adj_slot    per slot: transfer pass-through, counting sigmoid VJP,
//                 car-following VJP with the follower's headway term.
//   k_adj_link    thread per link: deterministic per-link reductions into the
//                 u, kappa, beta, alpha, cost gradients.
// All fp64 with -fmad=false: the forward is bit-identical to the reference.
#include <climits>
#include <cstdint>

#include "dtg_device.cuh"
#include "dtg_kernels.h"
#include "dtg_step.cuh"

namespace dtg {

constexpr int kCfThreads = 256;
constexpr int kTransferThreads = 256;

template <bool kVec>
__global__ void __launch_bounds__(kCfThreads, DTG_CF_MINB) k_step_cf(DevView d, int t, int s_cur) {
  (void)t;
  const int blk0 = blockIdx.x * (kCfThreads * kCfPer);
  const int k0 = kVec ? blk0 + 2 * static_cast<int>(threadIdx.x) : blk0 + static_cast<int>(threadIdx.x);
  step_cf_slots<kVec, kCfThreads>(d, d.b0 + blockIdx.y, s_cur, k0);
}

__global__ void __launch_bounds__(128) k_step_choice(DevView d, int t, int s_cur) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < d.L) step_choice_link(d, d.b0 + blockIdx.y, t, s_cur, j);
}

__global__ void __launch_bounds__(128) k_step_merge(DevView d, int t, int s_cur, int replay) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d.L) step_merge_link(d, d.b0 + blockIdx.y, t, s_cur, i, replay);
}

__global__ void __launch_bounds__(1024) k_step_scan(DevView d, int s_cur, int s_next, int replay) {
  __shared__ int sm[32];
  __shared__ unsigned long long smin[32];
  step_scan_block(d, d.b0 + blockIdx.x, s_cur, s_next, replay, sm, smin);
}

template <bool kVec>
__global__ void __launch_bounds__(kTransferThreads) k_step_transfer(DevView d, int s_cur, int s_next) {
  const int blk0 = blockIdx.x * (kTransferThreads * kTransferPer);
  const int k0 = kVec ? blk0 + 2 * static_cast<int>(threadIdx.x) : blk0 + static_cast<int>(threadIdx.x);
  step_transfer_slots<kVec, kTransferThreads>(d, d.b0 + blockIdx.y, s_cur, s_next, k0);
}

// ---------------------------------------------------------------------------------
// reverse
// ---------------------------------------------------------------------------------
__global__ void k_adj_init_slots(DevView d, int s_fin, const double* x_seed,
                                 double* xbar) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d.N) return;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  xbar[bn + k] = x_seed ? x_seed[bn + d.aid[sidx(d, s_fin, b) + k]] : 0.0;
}

__global__ void k_adj_init_links(DevView d, const double* cum_seed) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.L) return;
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  d.cbar[bl + j] = cum_seed ? cum_seed[bl + j] : 0.0;
  d.qbar[bl + j] = 0.0;
  double* g = d.grads + static_cast<std::size_t>(b) * 5 * d.L;
  for (int c = 0; c < 5; ++c) g[c * d.L + j] = 0.0;
}

// Adjoint of the non-admitted arrived agent's admitted-sum input
// (transfer VJP: x_bar * (-M) + (-(x_bar * x1))).
__device__ __forceinline__ double admitted_bar(double xb, double x1, double M) {
  double r = 0.0;
  r += xb * (-M);
  r += -1.0 * (xb * x1);
  return r;
}

__global__ void __launch_bounds__(128) k_adj_node(DevView d, int t, int s_cur,
                                                   int s_next,
                                                   const double* xbar_next,
                                                   const double* snap_seed,
                                                   int snap_k, int K) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.L) return;
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  if (snap_k >= 0 && snap_seed)  // snapshot seed enters before the step VJP (:390-393)
    d.cbar[bl + i] += snap_seed[(static_cast<std::size_t>(b) * K + snap_k) * d.L + i];
  const double cb = d.cbar[bl + i];
  // inc = relu(q - qprev): q_bar += pick * cum_bar; qprev_bar = -pick * cum_bar
  const double a = d.qh[hidx(d, t + 1, b) + i] - d.qh[hidx(d, t, b) + i];
  const bool pick = a >= 0.0;
  d.qtot[bl + i] = d.qbar[bl + i] + (pick ? cb : 0.0);
  d.qbar[bl + i] = pick ? -1.0 * cb : 0.0;

  const int w = d.win[bl + i];
  if (w < 0) return;
  const std::size_t so = sidx(d, s_cur, b);
  const int* off = d.off + oidx(d, s_cur, b);
  const int* offn = d.off + oidx(d, s_next, b);
  int cid[kMaxCand], cslot[kMaxCand], clink[kMaxCand];
  const int nc = gather_candidates(d, b, i, off, d.nA + bl, so, cid, cslot, clink);
  double lz[kMaxCand], pi[kMaxCand], bar[kMaxCand];
  merge_softmax(d, b, t, i, nc, cid, clink, lz, pi);
  // winner: a_t[w][i] bar = x_bar_new * M (+ 0 admitted-sum adjoint)
  const double abar_w = xbar_next[bn + offn[i] + d.newcnt[bl + i] - 1] * d.M + 0.0;
  for (int e = 0; e < nc; ++e) {
    const int s = cslot[e];
    if (s == w) {
      bar[e] = abar_w * 1.0;
    } else {
      const int p = clink[e];
      const int base = off[p];
      int dd = 0;
      for (int q = base; q < s; ++q) dd += d.won[bn + q];
      const double xb = xbar_next[bn + offn[p] + (s - base) - dd];
      bar[e] = admitted_bar(xb, d.x1[bn + s], d.M) * 1.0;
    }
  }
  two_softmax_vjp(nc, lz, pi, d.kinv, bar);
  for (int e = 0; e < nc; ++e) {
    const int s = cslot[e];
    // reduce_max(l) routes targeted_bar = a_bar[w] to the first candidate
    d.lbar_row[bn + s] = (e == 0 ? 0.0 + abar_w : 0.0) + bar[e] * d.alpha[bl + clink[e]];
    d.prio_bar[bn + s] = 0.0 + bar[e] * 1.0;
  }
}

// Per-row running maximum of y with the largest OTHER y (near-tie detector).
struct Top2 {
  double y1, y2;
  int id1, s1;
};
__device__ __forceinline__ void top2_push(Top2& T, double y, int id, int slot) {
  if (y > T.y1 || (y == T.y1 && id < T.id1)) {
    T.y2 = fmax(T.y2, T.y1);
    T.y1 = y;
    T.id1 = id;
    T.s1 = slot;
  } else {
    T.y2 = fmax(T.y2, y);
  }
}
__device__ __forceinline__ void top2_merge(Top2& A, const Top2& B) {
  if (B.y1 > A.y1 || (B.y1 == A.y1 && B.id1 < A.id1)) {
    A.y2 = fmax(fmax(A.y2, B.y2), A.y1);
    A.y1 = B.y1;
    A.id1 = B.id1;
    A.s1 = B.s1;
  } else {
    A.y2 = fmax(fmax(A.y2, B.y2), B.y1);
  }
}

constexpr int kA0Threads = 512;

// Rows that the reference routes to the first arrived agent A[0]: successors i
// of A[0]'s link that are vacant and targeted by nobody.  targeted_i = max over
// an all-zero column, whose first-index VJP lands on A[0]
// (reduce_max tensor.cpp:863-876); the row's draw w_i is the Gumbel argmax
// over every arrived agent with a uniform utility (node_model.cpp:99-120).
// One pass over the arrived list (appended by the replayed k_step_cf) keeps,
// per row, the top y = (logz + g) / tau_g and the largest other y.  Because
// exp is monotone, the reference's first argmax of pi = exp(y - m2) / z2 is the
// top-y agent (lowest id on exact ties) unless the runner-up is within 1e-9
// relative — then the exact ordered-sum path recomputes pi as the reference
// does (ascending agent id, sequential z2).
__global__ void __launch_bounds__(kA0Threads) k_adj_a0(DevView d, int t, int s_cur,
                                                        int s_next, const double* xbar_next,
                                                        unsigned long long* sort_scratch,
                                                        int force_slow) {
  __shared__ Top2 sh[kA0Threads / 32][kMaxDeg];
  __shared__ int rows[kMaxDeg];
  __shared__ int nrows;
  __shared__ Top2 best_all;
  __shared__ int cnt;
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* la0 = d.lbar_a0 + static_cast<std::size_t>(b) * d.maxdeg;
  if (tid < d.maxdeg) la0[tid] = 0.0;
  const int a0s = d.a0[b];
  const std::size_t so = sidx(d, s_cur, b);
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int nA = d.acount[b];
  const int c0 = a0s >= 0 ? d.lnk[so + a0s] : 0;
  const int s0 = d.succ_off[c0], deg = a0s >= 0 ? d.succ_off[c0 + 1] - s0 : 0;
  if (tid == 0) {
    int nr = 0;
    for (int e = 0; e < deg; ++e) {
      const int i = d.succ[s0 + e];
      if (d.vac[bl + i] && d.win[bl + i] < 0) rows[nr++] = e;
    }
    nrows = nr;
  }
  __syncthreads();
  const int nr = nrows;
  if (nr == 0) {
    if (tid == 0) d.acount[b] = 0;
    return;
  }
  const int* off = d.off + oidx(d, s_cur, b);
  const int* offn = d.off + oidx(d, s_next, b);
  const int* alist = d.alist + bn;
  // uniform first stage: v = -1e12 everywhere, z = |A| exactly
  const double v = 0.0 - kMaskLarge;
  const double lzv = dlog(static_cast<double>(nA) * 1.0) + v;
  const double logz = v - lzv;
  Top2 tp[kMaxDeg];
  for (int r = 0; r < nr; ++r) tp[r] = Top2{-INFINITY, -INFINITY, INT_MAX, -1};
  for (int q = tid; q < nA; q += blockDim.x) {
    const int s = alist[q];
    const int id = d.aid[so + s];
    for (int r = 0; r < nr; ++r) {
      const int i = d.succ[s0 + rows[r]];
      const double g = gumbel(d.seed_merge[b], static_cast<std::uint64_t>(t),
                              static_cast<std::uint64_t>(i), static_cast<std::uint64_t>(id));
      top2_push(tp[r], (logz + g) * d.kinv, id, s);
    }
  }
  for (int r = 0; r < nr; ++r) {
    Top2 x = tp[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Top2 y;
      y.y1 = __shfl_xor_sync(0xffffffffu, x.y1, o);
      y.y2 = __shfl_xor_sync(0xffffffffu, x.y2, o);
      y.id1 = __shfl_xor_sync(0xffffffffu, x.id1, o);
      y.s1 = __shfl_xor_sync(0xffffffffu, x.s1, o);
      top2_merge(x, y);
    }
    if (lane == 0) sh[wid][r] = x;
  }
  __syncthreads();
  for (int r = 0; r < nr; ++r) {
    if (tid == 0) {
      Top2 x = sh[0][r];
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) top2_merge(x, sh[w][r]);
      best_all = x;
    }
    __syncthreads();
    Top2 win = best_all;
    const int i = d.succ[s0 + rows[r]];
    const bool near = !(win.y1 - win.y2 > 1e-9 * fmax(1.0, fabs(win.y1)));
    if (near || force_slow) {
      if (!force_slow && tid == 0) atomicOr(&d.err[b], kErrNearTieSlow);
      // exact path: (id << 32 | slot) keys of A sorted ascending, sequential z2
      unsigned long long* keys = sort_scratch + static_cast<std::size_t>(b) * 2 * d.N;
      for (int q = tid; q < nA; q += blockDim.x) {
        const int s = alist[q];
        keys[q] = (static_cast<unsigned long long>(d.aid[so + s]) << 32) | static_cast<unsigned>(s);
      }
      int P2 = 1;
      while (P2 < nA) P2 <<= 1;
      for (int q = nA + tid; q < P2; q += blockDim.x) keys[q] = ULLONG_MAX;
      __syncthreads();
      for (int kk = 2; kk <= P2; kk <<= 1)
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int q = tid; q < P2; q += blockDim.x) {
            const int l = q ^ jj;
            if (l > q) {
              const unsigned long long a = keys[q], c = keys[l];
              if ((a > c) == ((q & kk) == 0)) {
                keys[q] = c;
                keys[l] = a;
              }
            }
          }
          __syncthreads();
        }
      if (tid == 0) {
        const double m2 = win.y1;
        double z2 = 0.0;
        for (int q = 0; q < nA; ++q) {
          const double g = gumbel(d.seed_merge[b], static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(i),
                                  keys[q] >> 32);
          z2 += dexp((logz + g) * d.kinv - m2);
        }
        double bp = -1.0;
        for (int q = 0; q < nA; ++q) {
          const double g = gumbel(d.seed_merge[b], static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(i),
                                  keys[q] >> 32);
          const double pv = dexp((logz + g) * d.kinv - m2) / z2;
          if (pv > bp) {
            bp = pv;
            best_all.id1 = static_cast<int>(keys[q] >> 32);
            best_all.s1 = static_cast<int>(keys[q] & 0xffffffffull);
          }
        }
      }
      __syncthreads();
      win = best_all;
    }
    if (tid == 0) {
      const int ws = win.s1;
      const int j = d.lnk[so + ws];
      const int base = off[j];
      const int na = d.nA[bl + j];
      bool mover;
      const int ns = next_slot(d, bn, bl, offn, ws, j, base, ws - base, na, &mover);
      double ab;
      if (mover) {
        ab = 0.0 * d.M + 0.0;
      } else {
        const double xb = xbar_next[bn + ns];
        ab = (i == j ? xb * d.M : 0.0 * d.M) + admitted_bar(xb, d.x1[bn + ws], d.M);
      }
      la0[rows[r]] = 0.0 + ab;
    }
    __syncthreads();
  }
  if (tid == 0) d.acount[b] = 0;
}

__global__ void __launch_bounds__(128) k_adj_choice(DevView d, int t, int s_cur) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.L) return;
  const std::size_t so = sidx(d, s_cur, b);
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int* off = d.off + oidx(d, s_cur, b);
  const int base = off[j];
  if (off[j + 1] == base) return;
  const int s0 = d.succ_off[j], deg = d.succ_off[j + 1] - s0;
  if (deg == 0) return;
  const int na = d.nA[bl + j];
  const int a0s = d.a0[b];
  for (int r = 0; r < na; ++r) {
    const int s = base + r;
    double g[kMaxDeg], pi[kMaxDeg], bar[kMaxDeg];
    const int agent = d.aid[so + s];
    const double* lz = d.slogz + (bl + j) * d.maxdeg;
    for (int e = 0; e < deg; ++e)
      g[e] = gumbel(d.seed_link[b], static_cast<std::uint64_t>(t),
                    static_cast<std::uint64_t>(agent), static_cast<std::uint64_t>(d.succ[s0 + e]));
    const int ed = softmax_stage2<kMaxDeg>(deg, lz, g, d.kinv, pi);
    for (int e = 0; e < deg; ++e) bar[e] = 0.0;
    const int dch = d.succ[s0 + ed];
    if (d.vac[bl + dch] && d.win[bl + dch] >= 0) bar[ed] = d.lbar_row[bn + s];
    if (s == a0s)
      for (int e = 0; e < deg; ++e) bar[e] += d.lbar_a0[static_cast<std::size_t>(b) * d.maxdeg + e];
    for (int e = 0; e < deg; ++e)  // l = picked * vacant * arrived * connected
      bar[e] = ((bar[e] * 1.0) * 1.0) * (d.vac[bl + d.succ[s0 + e]] ? 1.0 : 0.0);
    two_softmax_vjp(deg, lz, pi, d.kinv, bar);
    double* vb = d.vbar + (bn + s) * d.maxdeg;
    for (int e = 0; e < deg; ++e) vb[e] = bar[e];
  }
}

// Adjoint of one agent's new position x1 through transfer, replace_rows and
// the midpoint count (observation.cpp:9-20, sigmoid VJP tensor.cpp:794-800).
__device__ __forceinline__ double x1_bar(const DevView& d, std::size_t bn,
                                         std::size_t bl, const int* offn,
                                         const double* xbar_next, int k, int j,
                                         int base, int r, int na, double x1) {
  bool mover;
  const int ns = next_slot(d, bn, bl, offn, k, j, base, r, na, &mover);
  double xb = (mover && !d.tg) ? 0.0 : xbar_next[bn + ns];
  const double qt = d.qtot[bl + j];
  if (qt != 0.0) {
    const double sc = d.sc[j];
    const double z = (x1 + (-d.ctr[j])) * sc;
    const double sg = z >= 0.0 ? 1.0 / (1.0 + dexp(-z)) : dexp(z) / (1.0 + dexp(z));
    xb = xb + (((qt * 1.0) * sg) * (1.0 - sg)) * sc;
  }
  return xb;
}

__global__ void __launch_bounds__(256) k_adj_slot(DevView d, int s_cur, int s_next,
                                                   const double* xbar_next,
                                                   double* xbar_cur) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d.N) return;
  const std::size_t so = sidx(d, s_cur, b);
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const double* pos = d.pos + so;
  const int* off = d.off + oidx(d, s_cur, b);
  const int* offn = d.off + oidx(d, s_next, b);
  const int j = d.lnk[so + k];
  const int base = off[j], n = off[j + 1] - base, r = k - base;
  const int na = d.nA[bl + j];
  const double jam = d.jam[bl + j], dxf = d.dxf[bl + j], len = d.len[j];
  const double x = pos[k];
  // own car-following VJP (car_following.cpp:128-157)
  const CfPick me = cf_step(x, r == 0 ? d.M : pos[k - 1] - x, jam, dxf, len);
  const double x1b = x1_bar(d, bn, bl, offn, xbar_next, k, j, base, r, na, d.x1[bn + k]);
  const double xpb = d.tg ? x1b : (me.cap ? x1b : 0.0);  // graft: cap passes through
  const double dxcb = me.cong ? xpb : 0.0;
  const double dxfb = me.cong ? 0.0 : xpb;
  const double gapb = me.gap >= 0.0 ? dxcb * 1.0 : 0.0;
  // follower's headway term lands on this (leader) slot
  double tb = 0.0;
  if (r + 1 < n) {
    const double xf = pos[k + 1];
    const CfPick fo = cf_step(xf, x - xf, jam, dxf, len);
    const double f1b = x1_bar(d, bn, bl, offn, xbar_next, k + 1, j, base, r + 1, na,
                              d.x1[bn + k + 1]);
    const double fpb = d.tg ? f1b : (fo.cap ? f1b : 0.0);
    const double fcb = fo.cong ? fpb : 0.0;
    tb += (fo.gap >= 0.0 ? fcb * 1.0 : 0.0) * 1.0;
  }
  if (r > 0) tb += -(gapb * 1.0);
  xbar_cur[bn + k] = xpb + tb * 1.0;
  d.cu[bn + k] = (dxfb * d.dt) * 1.0;
  d.cg[bn + k] = gapb;
}

__global__ void __launch_bounds__(256) k_adj_link(DevView d, int s_cur) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.L) return;
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int* off = d.off + oidx(d, s_cur, b);
  const int base = off[j], n = off[j + 1] - base;
  // deterministic: each link's slots summed by one thread (link_sums8 order)
  double ub, jb;
  link_sums8(d.cu + bn, d.cg + bn, base, n, ub, jb);
  double* g = d.grads + static_cast<std::size_t>(b) * 5 * d.L;
  const double kap = d.kappa[bl + j];
  if (n) {
    g[j] += 0.0 + ub;
    g[d.L + j] += 0.0 - jb * static_cast<double>(d.delta_n) / (kap * kap);
  }
  // pref_bar_j from the link-choice rows of arrived heads on predecessor links
  double pb = 0.0;
  for (int e = d.pred_off[j]; e < d.pred_off[j + 1]; ++e) {
    const int p = d.pred[e];
    const int pbse = off[p];
    if (off[p + 1] == pbse) continue;
    const int nap = d.nA[bl + p];
    for (int r = 0; r < nap; ++r) {
      const int s = pbse + r;
      if (d.choice[bn + s] >= 0) pb += d.vbar[(bn + s) * d.maxdeg + d.pred_pos[e]] * 1.0;
    }
  }
  const double c = d.cost[bl + j], be = d.beta[bl + j];
  g[2 * d.L + j] += 0.0 + pb / c;  // pref = beta / cost (tensor.cpp:764-777)
  g[4 * d.L + j] += 0.0 - pb * be / (c * c);
  // alpha: prio = matmul(valid, alpha) over this link's candidates
  double ab = 0.0;
  if (n) {
    const int na = d.nA[bl + j];
    for (int r = 0; r < na; ++r) {
      const int s = base + r;
      const int ch = d.choice[bn + s];
      if (ch >= 0 && d.vac[bl + ch] && d.win[bl + ch] >= 0) ab += 1.0 * d.prio_bar[bn + s];
    }
  }
  g[3 * d.L + j] += ab;
}

// Compact state of one layout back to agent-id order.
__global__ void k_gather_state(DevView d, int s, int* link_out, double* pos_out) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d.N) return;
  const std::size_t so = sidx(d, s, b);
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int a = d.aid[so + k];
  link_out[bn + a] = d.lnk[so + k];
  pos_out[bn + a] = d.pos[so + k];
}

// Test hook: Gumbel draws on the device (counter RNG + CUDA libdevice log).
__global__ void k_gumbel_batch(std::uint64_t seed, std::uint64_t key, const std::uint64_t* rows,
                               const std::uint64_t* cols, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = gumbel(seed, key, rows[i], cols[i]);
}

void launch_gumbel_batch(std::uint64_t seed, std::uint64_t key, const std::uint64_t* rows,
                         const std::uint64_t* cols, int n, double* out, cudaStream_t st) {
  k_gumbel_batch<<<(n + 255) / 256, 256, 0, st>>>(seed, key, rows, cols, n, out);
}

// Per-link derived constants: jam spacing, free-flow advance, link preference.
__global__ void k_derive(DevView d, double* jam, double* dxf, double* pref) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.L) return;
  const std::size_t i = static_cast<std::size_t>(b) * d.L + j;
  jam[i] = static_cast<double>(d.delta_n) / d.kappa[i];  // divide(scalar(dn), kappa)
  dxf[i] = (1.0 * d.u[i]) * d.dt;                        // scale(mul(valid, u), dt)
  pref[i] = d.beta[i] / d.cost[i];                       // divide(beta, cost)
}

// ---------------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------------
static inline dim3 grid_n(int n, int bs, int B) { return dim3((n + bs - 1) / bs, B); }

// The paired (vector-load) slot mapping needs an even agent count (pairs
// never straddle a scenario) and two slots per thread.
static inline bool slot_vec(const DevView& d) {
#ifdef DTG_NO_SLOT_VEC
  return false;
#else
  return d.N % 2 == 0 && kCfPer == 2 && kTransferPer == 2;
#endif
}
// scenarios of one forward launch: [b0, b0 + nb) (nb 0: all B)
static inline int nbl(const DevView& d) { return d.nb ? d.nb : d.B; }

const char* const kFwdKernelNames[kFwdKernels] = {"k_step_cf", "k_step_choice", "k_step_merge",
                                                 "k_step_scan", "k_step_transfer"};
const char* const kBwdKernelNames[kBwdKernels] = {
    "k_step_cf(replay)", "k_step_choice(replay)", "k_step_merge(replay)", "k_step_scan(replay)", "k_adj_node",
    "k_adj_a0",          "k_adj_choice",         "k_adj_slot",          "k_adj_link"};

void launch_fwd_kernel(int which, const DevView& d, int t, int s_cur, int s_next,
                       cudaStream_t st) {
  switch (which) {
    case 0:
      if (slot_vec(d))
        k_step_cf<true><<<grid_n(d.N, kCfThreads * kCfPer, nbl(d)), kCfThreads, 0, st>>>(d, t, s_cur);
      else
        k_step_cf<false><<<grid_n(d.N, kCfThreads * kCfPer, nbl(d)), kCfThreads, 0, st>>>(d, t, s_cur);
      break;
    case 1:
      k_step_choice<<<grid_n(d.L, 128, nbl(d)), 128, 0, st>>>(d, t, s_cur);
      break;
    case 2:
      k_step_merge<<<grid_n(d.L, 128, nbl(d)), 128, 0, st>>>(d, t, s_cur, 0);
      break;
    case 3:
      k_step_scan<<<nbl(d), 1024, 0, st>>>(d, s_cur, s_next, 0);
      break;
    default:
      if (slot_vec(d))
        k_step_transfer<true><<<grid_n(d.N, kTransferThreads * kTransferPer, nbl(d)), kTransferThreads, 0, st>>>(
            d, s_cur, s_next);
      else
        k_step_transfer<false><<<grid_n(d.N, kTransferThreads * kTransferPer, nbl(d)), kTransferThreads, 0, st>>>(
            d, s_cur, s_next);
  }
}

void launch_step_forward(const DevView& d, int t, int s_cur, int s_next,
                         cudaStream_t st) {
  for (int w = 0; w < kFwdKernels; ++w) launch_fwd_kernel(w, d, t, s_cur, s_next, st);
}

void launch_bwd_kernel(int which, const DevView& d, int t, int s_cur, int s_next,
                       const double* xbar_next, double* xbar_cur,
                       const double* snap_seed, int snap_k, int K,
                       unsigned long long* sort_scratch, int force_slow,
                       cudaStream_t st) {
  switch (which) {
    case 0:
      if (slot_vec(d))
        k_step_cf<true><<<grid_n(d.N, kCfThreads * kCfPer, d.B), kCfThreads, 0, st>>>(d, t, s_cur);
      else
        k_step_cf<false><<<grid_n(d.N, kCfThreads * kCfPer, d.B), kCfThreads, 0, st>>>(d, t, s_cur);
      break;
    case 1:
      k_step_choice<<<grid_n(d.L, 128, d.B), 128, 0, st>>>(d, t, s_cur);
      break;
    case 2:
      k_step_merge<<<grid_n(d.L, 128, d.B), 128, 0, st>>>(d, t, s_cur, 1);
      break;
    case 3:
      k_step_scan<<<d.B, 1024, 0, st>>>(d, s_cur, s_next, 1);
      break;
    case 4:
      k_adj_node<<<grid_n(d.L, 128, d.B), 128, 0, st>>>(d, t, s_cur, s_next, xbar_next,
                                                          snap_seed, snap_k, K);
      break;
    case 5:
      k_adj_a0<<<d.B, kA0Threads, 0, st>>>(d, t, s_cur, s_next, xbar_next, sort_scratch, force_slow);
      break;
    case 6:
      k_adj_choice<<<grid_n(d.L, 128, d.B), 128, 0, st>>>(d, t, s_cur);
      break;
    case 7:
      k_adj_slot<<<grid_n(d.N, 256, d.B), 256, 0, st>>>(d, s_cur, s_next, xbar_next, xbar_cur);
      break;
    default:
      k_adj_link<<<grid_n(d.L, 256, d.B), 256, 0, st>>>(d, s_cur);
  }
}

void launch_step_backward(const DevView& d, int t, int s_cur, int s_next,
                          const double* xbar_next, double* xbar_cur,
                          const double* snap_seed, int snap_k, int K,
                          unsigned long long* sort_scratch, int force_slow,
                          cudaStream_t st) {
  for (int w = 0; w < kBwdKernels; ++w)
    launch_bwd_kernel(w, d, t, s_cur, s_next, xbar_next, xbar_cur, snap_seed, snap_k, K,
                      sort_scratch, force_slow, st);
}

void launch_adj_init(const DevView& d, int s_fin, const double* x_seed,
                     double* xbar, const double* cum_seed, cudaStream_t st) {
  k_adj_init_slots<<<grid_n(d.N, 256, d.B), 256, 0, st>>>(d, s_fin, x_seed, xbar);
  k_adj_init_links<<<grid_n(d.L, 128, d.B), 128, 0, st>>>(d, cum_seed);
}

void launch_gather_state(const DevView& d, int s, int* link_out, double* pos_out,
                         cudaStream_t st) {
  k_gather_state<<<grid_n(d.N, 256, d.B), 256, 0, st>>>(d, s, link_out, pos_out);
}

void launch_derive(const DevView& d, double* jam, double* dxf, double* pref,
                   cudaStream_t st) {
  k_derive<<<grid_n(d.L, 128, d.B), 128, 0, st>>>(d, jam, dxf, pref);
}

}  // namespace dtg

namespace dtg {
cudaError_t decision_stats_kernels(int force, unsigned long long* count) { return decision_stats_tu(force, count); }
}  // namespace dtg
