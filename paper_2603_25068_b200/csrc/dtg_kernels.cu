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

namespace dtg {

constexpr int kFastSucc = 5;  // successor / candidate counts up to this use register fast paths

// ---------------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------------
// kCfPer slots per thread, strided by the block size, all loads of a round
// issued before use (as in k_step_transfer: the lnk -> link-constant chain is
// latency-, not bandwidth-bound with one slot per thread).  Measured (C3
// B=256, ms per nowcast): 1 slot 9.2, 2 slots at <= 64 registers 8.0, 4 slots
// 9.5 (110 registers).
#ifndef DTG_CF_PER
#define DTG_CF_PER 2
#endif
#ifndef DTG_CF_MINB
#define DTG_CF_MINB 4
#endif
constexpr int kCfPer = DTG_CF_PER;
constexpr int kCfThreads = 256;

// kVec (even N, kCfPer == 2): a thread's two slots are ADJACENT and their
// link ids and positions are read with one 8-byte / one 16-byte load (int2,
// double2; still fully coalesced), the pair's outer neighbours with two scalar
// loads -- half the load instructions of the strided mapping.
template <bool kVec>
__global__ void __launch_bounds__(kCfThreads, DTG_CF_MINB) k_step_cf(DevView d, int t, int s_cur) {
  (void)t;
  const int b = d.b0 + blockIdx.y;
  const int blk0 = blockIdx.x * (kCfThreads * kCfPer);
  const int k0 = kVec ? blk0 + 2 * static_cast<int>(threadIdx.x) : blk0 + static_cast<int>(threadIdx.x);
  const int kstep = kVec ? 1 : kCfThreads;
  const std::size_t so = sidx(d, s_cur, b);
  const double* pos = d.pos + so;
  const int* off = d.off + oidx(d, s_cur, b);
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  int j[kCfPer];
  double xm[kCfPer], x[kCfPer], xp[kCfPer];
  if (kVec) {
    const int kk = k0 < d.N ? k0 : d.N - 2;  // even N: pairs never straddle the end
    const int2 j2 = *reinterpret_cast<const int2*>(d.lnk + so + kk);
    const double2 x2 = *reinterpret_cast<const double2*>(pos + kk);
    j[0] = j2.x;
    j[1] = j2.y;
    x[0] = x2.x;
    x[1] = x2.y;
    xm[0] = pos[kk > 0 ? kk - 1 : 0];
    xm[1] = x2.x;
    xp[0] = x2.y;
    xp[1] = pos[kk + 2 < d.N ? kk + 2 : kk + 1];
  } else {
#pragma unroll
    for (int i = 0; i < kCfPer; ++i) {
      const int k = k0 + i * kCfThreads;
      const int kk = k < d.N ? k : d.N - 1;
      j[i] = d.lnk[so + kk];
      x[i] = pos[kk];
      xm[i] = pos[kk > 0 ? kk - 1 : 0];
      xp[i] = pos[kk + 1 < d.N ? kk + 1 : kk];
    }
  }
  int base[kCfPer], n[kCfPer];
  double jam[kCfPer], dxf[kCfPer], len[kCfPer], ctr[kCfPer], thr[kCfPer];
#pragma unroll
  for (int i = 0; i < kCfPer; ++i) {
    base[i] = off[j[i]];
    n[i] = off[j[i] + 1] - base[i];
    jam[i] = d.jam[bl + j[i]];
    dxf[i] = d.dxf[bl + j[i]];
    len[i] = d.len[j[i]];
    ctr[i] = d.ctr[j[i]];
    thr[i] = d.thr[j[i]];
  }
  int* qn = d.qn + bl;
  int* nA = d.nA + bl;
#pragma unroll
  for (int i = 0; i < kCfPer; ++i) {
    const int k = k0 + i * kstep;
    if (k >= d.N) break;
    const int r = k - base[i];
    // headway: leader gets M (car_following.cpp:547-553)
    const CfPick me = cf_step(x[i], r == 0 ? d.M : xm[i] - x[i], jam[i], dxf[i], len[i]);
    d.x1[bn + k] = me.x1;
    bool fo_n = false, fa_n = false;
    if (r + 1 < n[i]) {
      const CfPick nx = cf_step(xp[i], x[i] - xp[i], jam[i], dxf[i], len[i]);
      fo_n = nx.x1 >= ctr[i];
      fa_n = nx.x1 >= thr[i];
    }
    const bool fo = me.x1 >= ctr[i], fa = me.x1 >= thr[i];
    // x1 stays ordered inside the segment, so {x1 >= o} and {x1 >= L-0.01} are
    // prefixes: their lengths are written by the unique boundary slot.
    if (r == 0 && !fo) qn[j[i]] = 0;
    if (fo && !fo_n) qn[j[i]] = r + 1;
    if (r == 0 && !fa) nA[j[i]] = 0;
    if (fa && !fa_n) nA[j[i]] = r + 1;
    if (r == n[i] - 1) d.tail[bl + j[i]] = me.x1;  // min x1 = vacancy (node_model.cpp:27-41)
    if (fa) {
      d.won[bn + k] = 0;
      if (d.alist) d.alist[bn + atomicAdd(&d.acount[b], 1)] = k;  // reverse sweep only
    }
  }
}

// Link choice of the arrived heads (node_model.cpp:45-97), one thread per
// link over its nA arrived agents.  Kept out of k_step_cf: the draw's
// registers and local arrays halved that kernel's occupancy while only ~8% of
// its threads ever draw.
__global__ void __launch_bounds__(128) k_step_choice(DevView d, int t, int s_cur) {
  const int b = d.b0 + blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.L) return;
  const int* off = d.off + oidx(d, s_cur, b);
  const int base = off[j];
  if (off[j + 1] == base) return;  // empty segment: nA[j] is stale
  const std::size_t pl = static_cast<std::size_t>(b) * d.L + j;
  const int na = d.nA[pl];
  if (na == 0) return;
  const std::size_t so = sidx(d, s_cur, b);
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int s0 = d.succ_off[j], deg = d.succ_off[j + 1] - s0;
  const double* lz = d.slogz + pl * d.maxdeg;
  for (int r = 0; r < na; ++r) {
    const int k = base + r;
    int c = -1;
    if (deg > 0) {
      const int agent = d.aid[so + k];
      if (deg <= kFastSucc) {  // registers, straight-line logs, argmax from the logits
        const std::uint64_t h2 = rng_prefix2(rng_prefix1(d.seed_link[b], static_cast<std::uint64_t>(t)),
                                             static_cast<std::uint64_t>(agent));
        int sj[kFastSucc];
        double y[kFastSucc], ex[kFastSucc];
#pragma unroll
        for (int e = 0; e < kFastSucc; ++e) sj[e] = d.succ[s0 + (e < deg ? e : 0)];
        // one scalar draw per successor: this kernel is occupancy-bound (one
        // thread per link, few of them drawing), which the batched draws'
        // registers would cost
        int bad = 0;
#pragma unroll
        for (int e = 0; e < kFastSucc; ++e)
          y[e] = e < deg ? (lz[e] + gumbel_sl(rng_final(h2, static_cast<std::uint64_t>(sj[e])), bad)) * d.kinv
                         : 0.0;
        const int best = softmax_first_argmax<kFastSucc>(deg, y, ex);
        c = sj[0];
#pragma unroll
        for (int e = 1; e < kFastSucc; ++e)
          if (e == best) c = sj[e];
      } else {
        double g[kMaxDeg], pi[kMaxDeg];
        for (int e = 0; e < deg; ++e)
          g[e] = gumbel(d.seed_link[b], static_cast<std::uint64_t>(t),
                        static_cast<std::uint64_t>(agent), static_cast<std::uint64_t>(d.succ[s0 + e]));
        c = d.succ[s0 + softmax_stage2<kMaxDeg>(deg, lz, g, d.kinv, pi)];
      }
    }
    d.choice[bn + k] = c;
  }
}

// Merge candidates of row i: arrived heads of predecessor links that chose i,
// ascending agent id (merge_choice columns, node_model.cpp:99-120).
__device__ __forceinline__ int gather_candidates(const DevView& d, int b, int i,
                                                 const int* off, std::size_t so,
                                                 int* cid, int* cslot, int* clink) {
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  int nc = 0;
  for (int e = d.pred_off[i]; e < d.pred_off[i + 1]; ++e) {
    const int p = d.pred[e];
    const int base = off[p];
    if (off[p + 1] == base) continue;
    const int nap = d.nA[bl + p];
    for (int r = 0; r < nap; ++r) {
      const int s = base + r;
      if (d.choice[bn + s] != i) continue;
      if (nc == kMaxCand) {
        atomicOr(&d.err[b], kErrCandOverflow);
        return nc;
      }
      cid[nc] = d.aid[so + s];
      cslot[nc] = s;
      clink[nc] = p;
      ++nc;
    }
  }
  for (int a = 1; a < nc; ++a) {  // insertion sort by agent id
    const int ci = cid[a], cs = cslot[a], cl = clink[a];
    int m = a - 1;
    while (m >= 0 && cid[m] > ci) {
      cid[m + 1] = cid[m];
      cslot[m + 1] = cslot[m];
      clink[m + 1] = clink[m];
      --m;
    }
    cid[m + 1] = ci;
    cslot[m + 1] = cs;
    clink[m + 1] = cl;
  }
  return nc;
}

__device__ __forceinline__ int merge_softmax(const DevView& d, int b, int t, int i,
                                             int nc, const int* cid, const int* clink,
                                             double* lz, double* pi, bool need_pi = true) {
  if (!need_pi && nc <= kFastSucc) {  // registers; first stage exact, winner from the logits
    const std::size_t bl = static_cast<std::size_t>(b) * d.L;
    const std::uint64_t h2 = rng_prefix2(rng_prefix1(d.seed_merge[b], static_cast<std::uint64_t>(t)),
                                         static_cast<std::uint64_t>(i));
    double v[kFastSucc], y[kFastSucc], ex[kFastSucc];
    // one draw per candidate (most rows have one or two): the scalar chain
    // keeps this latency-bound kernel's register count, and so its occupancy
    int bad = 0;
#pragma unroll
    for (int e = 0; e < kFastSucc; ++e)
      y[e] = e < nc ? gumbel_sl(rng_final(h2, static_cast<std::uint64_t>(cid[e])), bad) : 0.0;
#pragma unroll
    for (int e = 0; e < kFastSucc; ++e) {
      v[e] = e < nc ? d.alpha[bl + clink[e]] : 0.0;
      if (e < nc && v[e] == 0.0) atomicOr(&d.err[b], kErrZeroAlpha);
      if (e >= nc) y[e] = 0.0;
    }
    {  // winner from alpha + g when the top two are clearly apart (bound in dtg_merge.cuh)
      int best = 0;
      double v1 = v[0] + y[0], v2 = -INFINITY;
      bool small = fabs(v[0]) < 64.0 && fabs(y[0]) < 64.0;
#pragma unroll
      for (int e = 1; e < kFastSucc; ++e)
        if (e < nc) {
          const double a = v[e] + y[e];
          small = small && fabs(v[e]) < 64.0 && fabs(y[e]) < 64.0;
          if (a > v1) {
            v2 = v1;
            v1 = a;
            best = e;
          } else if (a > v2) {
            v2 = a;
          }
        }
      if (!g_force_exact && small && d.kinv <= 100.0 && (nc == 1 || (v1 - v2) * d.kinv > 1e-9)) return best;
      if (!g_force_exact) atomicAdd(&g_exact_decisions, 1ULL);
    }
    double m = v[0];
#pragma unroll
    for (int e = 1; e < kFastSucc; ++e)
      if (e < nc && m < v[e]) m = v[e];
    double z = 0.0;
#pragma unroll
    for (int e = 0; e < kFastSucc; ++e)
      if (e < nc) z += dexp(v[e] - m);
    const double lzz = dlog(z) + m;
#pragma unroll
    for (int e = 0; e < kFastSucc; ++e) y[e] = ((v[e] - lzz) + y[e]) * d.kinv;
    return softmax_first_argmax<kFastSucc>(nc, y, ex);
  }
  double v[kMaxCand], g[kMaxCand];
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  for (int e = 0; e < nc; ++e) {
    v[e] = d.alpha[bl + clink[e]];  // p = l * matmul(valid, alpha)
    if (v[e] == 0.0) atomicOr(&d.err[b], kErrZeroAlpha);
    g[e] = gumbel(d.seed_merge[b], static_cast<std::uint64_t>(t),
                  static_cast<std::uint64_t>(i), static_cast<std::uint64_t>(cid[e]));
  }
  return two_softmax<kMaxCand>(nc, v, g, d.kinv, lz, pi);
}

__global__ void __launch_bounds__(128) k_step_merge(DevView d, int t, int s_cur,
                                                     int replay) {
  const int b = d.b0 + blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.L) return;
  const std::size_t so = sidx(d, s_cur, b);
  const int* off = d.off + oidx(d, s_cur, b);
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const int n_i = off[i + 1] - off[i];
  const int qc = n_i ? d.qn[bl + i] : 0;
  const double tx = n_i ? d.tail[bl + i] : d.M;
  if (!replay) {  // inc = relu(q - qprev); cum += inc (engine.cpp:111-113)
    const double a = static_cast<double>(qc) - d.qh[hidx(d, t, b) + i];
    d.cumh[hidx(d, t + 1, b) + i] = d.cumh[hidx(d, t, b) + i] + (a >= 0.0 ? a : 0.0);
    d.qh[hidx(d, t + 1, b) + i] = static_cast<double>(qc);
  }
  const bool vacant = tx > d.jam[bl + i];
  d.vac[bl + i] = vacant;
  int w = -1, wa = -1;
  if (vacant) {
    int cid[kMaxCand], cslot[kMaxCand], clink[kMaxCand];
    const int nc = gather_candidates(d, b, i, off, so, cid, cslot, clink);
    if (nc) {
      double lz[kMaxCand], pi[kMaxCand];
      const int best = merge_softmax(d, b, t, i, nc, cid, clink, lz, pi, false);
      w = cslot[best];
      wa = cid[best];
      d.won[static_cast<std::size_t>(b) * d.N + w] = 1;
    }
  }
  d.win[bl + i] = w;
  if (!replay && d.ev) d.ev[(static_cast<std::size_t>(t) * d.B + b) * d.L + i] = wa;
}

// Block-wide exclusive scan of one int per thread (blockDim.x == 1024).
__device__ __forceinline__ int block_excl_scan(int v, int* smem, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < (blockDim.x >> 5) ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem[lane] = w;
  }
  __syncthreads();
  const int warp_prefix = wid ? smem[wid - 1] : 0;
  *total = smem[(blockDim.x >> 5) - 1];
  return warp_prefix + x - v;
}

__global__ void __launch_bounds__(1024) k_step_scan(DevView d, int s_cur,
                                                     int s_next, int replay) {
  __shared__ int sm[32];
  __shared__ unsigned long long smin[32];
  const int b = d.b0 + blockIdx.x;
  const std::size_t so = sidx(d, s_cur, b);
  const int* off = d.off + oidx(d, s_cur, b);
  int* offn = d.off + oidx(d, s_next, b);
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int per = (d.L + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * per, j1 = min(d.L, j0 + per);
  int sum = 0;
  unsigned long long a0key = ULLONG_MAX;
  for (int j = j0; j < j1; ++j) {
    const int base = off[j], n = off[j + 1] - base;
    const int na = n ? d.nA[bl + j] : 0;
    int dep = 0;
    for (int r = 0; r < na; ++r) {
      const int s = base + r;
      dep += d.won[bn + s];
      const unsigned long long key =
          (static_cast<unsigned long long>(d.aid[so + s]) << 32) | static_cast<unsigned>(s);
      a0key = key < a0key ? key : a0key;
    }
    const int nc = n - dep + (d.win[bl + j] >= 0 ? 1 : 0);
    d.dep[bl + j] = dep;
    d.newcnt[bl + j] = nc;
    sum += nc;
  }
  int total;
  const int excl = block_excl_scan(sum, sm, &total);
  if (!replay) {
    int run = excl;
    for (int j = j0; j < j1; ++j) {
      offn[j] = run;
      run += d.newcnt[bl + j];
    }
    if (threadIdx.x == 0) {
      offn[d.L] = total;
      if (total != d.N) atomicOr(&d.err[b], kErrConservation);
    }
  }
  // first arrived agent A[0] (min id) for the reverse sweep
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, a0key, o);
    a0key = y < a0key ? y : a0key;
  }
  if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = a0key;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = ULLONG_MAX;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = smin[w] < m ? smin[w] : m;
    d.a0[b] = m == ULLONG_MAX ? -1 : static_cast<int>(m & 0xffffffffull);
  }
}

// Slot of the agent in the next layout (the transfer compaction).
__device__ __forceinline__ int next_slot(const DevView& d, std::size_t bn,
                                         std::size_t bl, const int* offn, int k,
                                         int j, int base, int r, int na,
                                         bool* mover) {
  if (r < na && d.won[bn + k]) {
    *mover = true;
    const int i = d.choice[bn + k];
    return offn[i] + d.newcnt[bl + i] - 1;
  }
  *mover = false;
  int dd;
  if (r >= na) {
    dd = d.dep[bl + j];
  } else {
    dd = 0;
    for (int q = base; q < k; ++q) dd += d.won[bn + q];
  }
  return offn[j] + r - dd;
}

// kTransferPer slots per thread, strided by the block size (coalesced), with
// every slot's loads issued before any is used: the dependent chain
// lnk -> (off, nA, dep, offn) -> store is ~3 memory latencies deep, so one slot
// per thread left the kernel latency-bound at ~2.5 TB/s (B=256).  Measured
// (C3 B=256, ms per nowcast): 1 slot 9.3, 2 slots 7.6, 4 slots 9.0.
#ifndef DTG_TR_PER
#define DTG_TR_PER 2
#endif
constexpr int kTransferPer = DTG_TR_PER;
constexpr int kTransferThreads = 256;

// kVec: adjacent slot pairs with int2 / double2 loads, as in k_step_cf.
template <bool kVec>
__global__ void __launch_bounds__(kTransferThreads) k_step_transfer(DevView d, int s_cur,
                                                                     int s_next) {
  const int b = d.b0 + blockIdx.y;
  const int blk0 = blockIdx.x * (kTransferThreads * kTransferPer);
  const int k0 = kVec ? blk0 + 2 * static_cast<int>(threadIdx.x) : blk0 + static_cast<int>(threadIdx.x);
  const int kstep = kVec ? 1 : kTransferThreads;
  const std::size_t so = sidx(d, s_cur, b), sn = sidx(d, s_next, b);
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int* off = d.off + oidx(d, s_cur, b);
  const int* offn = d.off + oidx(d, s_next, b);
  int j[kTransferPer], id[kTransferPer], base[kTransferPer], na[kTransferPer], sh[kTransferPer];
  double x[kTransferPer];
  if (kVec) {
    const int kk = k0 < d.N ? k0 : d.N - 2;
    const int2 j2 = *reinterpret_cast<const int2*>(d.lnk + so + kk);
    const double2 x2 = *reinterpret_cast<const double2*>(d.x1 + bn + kk);
    const int2 i2 = *reinterpret_cast<const int2*>(d.aid + so + kk);
    j[0] = j2.x;
    j[1] = j2.y;
    x[0] = x2.x;
    x[1] = x2.y;
    id[0] = i2.x;
    id[1] = i2.y;
  } else {
#pragma unroll
    for (int i = 0; i < kTransferPer; ++i) {
      const int k = k0 + i * kTransferThreads;
      const int kk = k < d.N ? k : d.N - 1;
      j[i] = d.lnk[so + kk];
      x[i] = d.x1[bn + kk];
      id[i] = d.aid[so + kk];
    }
  }
#pragma unroll
  for (int i = 0; i < kTransferPer; ++i) {
    base[i] = off[j[i]];
    na[i] = d.nA[bl + j[i]];
    sh[i] = offn[j[i]] - d.dep[bl + j[i]];  // non-arrived slots: ns = offn + r - dep
  }
#pragma unroll
  for (int i = 0; i < kTransferPer; ++i) {
    const int k = k0 + i * kstep;
    if (k >= d.N) break;
    const int r = k - base[i];
    int ns = sh[i] + r, lk = j[i];
    double xo = x[i];
    if (r < na[i]) {  // arrived: winner moves, the others shift past earlier winners
      bool mover;
      ns = next_slot(d, bn, bl, offn, k, j[i], base[i], r, na[i], &mover);
      if (mover) {
        xo = 0.0;  // transfer (node_model.cpp:122-149): -M + M == 0.0 exactly on the new link
        lk = d.choice[bn + k];
      }
    }
    d.pos[sn + ns] = xo;
    d.aid[sn + ns] = id[i];
    d.lnk[sn + ns] = lk;
  }
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
  const int nc = gather_candidates(d, b, i, off, so, cid, cslot, clink);
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
