// Forward engine step bodies (reference engine_step, src/engine.cpp:70-125),
// shared by the step-graph kernels (one launch per phase, dtg_kernels.cu) and
// the scenario-resident kernel k_forward_scn (one CTA per scenario looping
// over the steps with CTA barriers between the phases).  The phases:
//   cf        per agent slot: Newell car-following with the leader in the
//             previous slot, per-link midpoint count and arrived-prefix length
//             as segment-boundary writes, vacancy tail;
//   choice    per link: the Gumbel-softmax link choice of its arrived agents;
//   merge     per link: count/cumulative update, vacancy, merge-choice over the
//             arrived heads of the predecessor links;
//   scan      per scenario: departures, new segment sizes and the exclusive
//             scan to the next segment offsets;
//   transfer  per slot: compaction into the next layout (winners enter their
//             new link at position 0.0, everyone else keeps x1 and its order).
// All fp64 with -fmad=false: bit-identical to the reference.
#pragma once
#include <climits>
#include <cstdint>

#include "dtg_device.cuh"

namespace dtg {

constexpr int kFastSucc = 5;  // successor / candidate counts up to this use register fast paths

// Optional per-event hooks of the phase bodies (the scenario-resident kernel
// lists the links with arrived heads and the links chosen by them).
struct NoHook {
  __device__ __forceinline__ void operator()(int) const {}
};

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

// kVec (even N, kCfPer == 2): a thread's two slots are ADJACENT and their
// link ids and positions are read with one 8-byte / one 16-byte load (int2,
// double2; still fully coalesced), the pair's outer neighbours with two scalar
// loads -- half the load instructions of the strided mapping.
// The slots of one thread: kVec: the pair k0, k0 + 1; else k0 + i * kStride.
// on_arrived(j): link j has arrived heads (called once per such link).
template <bool kVec, int kStride, typename Hook = NoHook>
__device__ __forceinline__ void step_cf_slots(const DevView& d, int b, int s_cur, int k0,
                                              Hook on_arrived = Hook()) {
  const int kstep = kVec ? 1 : kStride;
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
      const int k = k0 + i * kStride;
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
    if (fa && !fa_n) {
      nA[j[i]] = r + 1;
      on_arrived(j[i]);
    }
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
// on_choice(c): an arrived head of link j chose successor c.
// The na arrived heads of link j start at slot `base` of layout s_cur.
template <typename Hook = NoHook>
__device__ __forceinline__ void choose_heads(const DevView& d, int b, int t, int s_cur, int j, int base,
                                             int na, Hook on_choice) {
  const std::size_t pl = static_cast<std::size_t>(b) * d.L + j;
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
    if (c >= 0) on_choice(c);
  }
}

template <typename Hook = NoHook>
__device__ __forceinline__ void step_choice_link(const DevView& d, int b, int t, int s_cur, int j,
                                                 Hook on_choice = Hook()) {
  const int* off = d.off + oidx(d, s_cur, b);
  const int base = off[j];
  if (off[j + 1] == base) return;  // empty segment: nA[j] is stale
  const int na = d.nA[static_cast<std::size_t>(b) * d.L + j];
  if (na == 0) return;
  choose_heads(d, b, t, s_cur, j, base, na, on_choice);
}

// Merge candidates of row i: arrived heads of predecessor links that chose i,
// ascending agent id (merge_choice columns, node_model.cpp:99-120).  off and
// nAb (arrived-prefix lengths) are this scenario's rows (global or shared).
__device__ __forceinline__ int gather_candidates(const DevView& d, int b, int i,
                                                 const int* off, const int* nAb, std::size_t so,
                                                 int* cid, int* cslot, int* clink) {
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  int nc = 0;
  for (int e = d.pred_off[i]; e < d.pred_off[i + 1]; ++e) {
    const int p = d.pred[e];
    const int base = off[p];
    if (off[p + 1] == base) continue;
    const int nap = nAb[p];
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

// Merge row i with nc <= kFastSucc candidates (registers when cid / clink are
// register arrays: every index is a compile-time constant): the exact first
// stage, the winner from the logits.
__device__ __forceinline__ int merge_softmax_fast(const DevView& d, int b, int t, int i, int nc,
                                                  const int* cid, const int* clink) {
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

// Register gather for rows with at most kFastSucc candidates: the candidates
// in ascending agent id, or -1 when the row has more (use gather_candidates).
__device__ __forceinline__ int gather_candidates_fast(const DevView& d, int b, int i, const int* off,
                                                      const int* nAb, std::size_t so, int (&cid)[kFastSucc],
                                                      int (&cslot)[kFastSucc], int (&clink)[kFastSucc]) {
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  int nc = 0;
#pragma unroll
  for (int e = 0; e < kFastSucc; ++e) cid[e] = cslot[e] = clink[e] = 0;
  for (int e = d.pred_off[i]; e < d.pred_off[i + 1]; ++e) {
    const int p = d.pred[e];
    const int base = off[p];
    if (off[p + 1] == base) continue;
    const int nap = nAb[p];
    for (int r = 0; r < nap; ++r) {
      const int s = base + r;
      if (d.choice[bn + s] != i) continue;
      if (nc == kFastSucc) return -1;
      const int ci = d.aid[so + s];
      // insertion at the sorted position, from the new end down (ids are unique)
      bool placed = false;
#pragma unroll
      for (int q = kFastSucc - 1; q >= 0; --q) {
        if (q > nc || placed) continue;
        if (q > 0 && cid[q - 1] > ci) {
          cid[q] = cid[q - 1];
          cslot[q] = cslot[q - 1];
          clink[q] = clink[q - 1];
        } else {
          cid[q] = ci;
          cslot[q] = s;
          clink[q] = p;
          placed = true;
        }
      }
      ++nc;
    }
  }
  return nc;
}

__device__ __forceinline__ int merge_softmax(const DevView& d, int b, int t, int i,
                                             int nc, const int* cid, const int* clink,
                                             double* lz, double* pi, bool need_pi = true) {
  if (!need_pi && nc <= kFastSucc) {  // registers; first stage exact, winner from the logits
    return merge_softmax_fast(d, b, t, i, nc, cid, clink);
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

// Count / cumulative update and vacancy of link i; true when vacant.
__device__ __forceinline__ bool step_merge_counts(const DevView& d, int b, int t, int s_cur, int i,
                                                  int replay) {
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
  return vacant;
}

// Merge decision of link i (vacant: over the arrived heads that chose it);
// writes the winner slot (-1 none) and its transfer event.
__device__ __forceinline__ void step_merge_decide(const DevView& d, int b, int t, int s_cur, int i,
                                                  bool vacant, int replay) {
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  int w = -1, wa = -1;
  if (vacant) {
    const std::size_t so = sidx(d, s_cur, b);
    const int* off = d.off + oidx(d, s_cur, b);
    int cid[kMaxCand], cslot[kMaxCand], clink[kMaxCand];
    const int nc = gather_candidates(d, b, i, off, d.nA + bl, so, cid, cslot, clink);
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

__device__ __forceinline__ void step_merge_link(const DevView& d, int b, int t, int s_cur, int i,
                                                int replay) {
  const bool vacant = step_merge_counts(d, b, t, s_cur, i, replay);
  step_merge_decide(d, b, t, s_cur, i, vacant, replay);
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

// One CTA (any multiple of 32 threads up to 1024) per scenario; sm / smin
// are 32-entry shared arrays.
__device__ __forceinline__ void step_scan_block(const DevView& d, int b, int s_cur, int s_next,
                                                int replay, int* sm, unsigned long long* smin) {
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

// kVec: adjacent slot pairs with int2 / double2 loads, as in k_step_cf.
template <bool kVec, int kStride>
__device__ __forceinline__ void step_transfer_slots(const DevView& d, int b, int s_cur, int s_next,
                                                    int k0) {
  const int kstep = kVec ? 1 : kStride;
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
      const int k = k0 + i * kStride;
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

}  // namespace dtg
