// Persistent cooperative reverse sweep: all T reverse steps of all B scenarios
// in one launch, three grid barriers per step (R4 of step t + 1 runs in the
// same phase as R1 of step t) (the checkpointed per-step VJP of
// src/engine.cpp:388-415, i.e. Tape::vjp of src/tensor.cpp:715-996 applied to
// engine_step / node_step / car_following_step / midpoint_count).
//
// Reverse step t (layout t = checkpoint t, layout t+1 = checkpoint t+1):
//   R1 slots   replay car-following (x1), arrived-prefix length, tail; arrived
//              heads replay their link choice (pi kept for R4), register as a
//              merge candidate {alpha, own merge Gumbel, slot, id, link},
//              append to the arrived list and atomicMin the first arrived id.
//   R2 links   snapshot seed, count adjoint (q_bar, qprev_bar); vacancy;
//              merge replay (winner, departures); the DEFERRED preference
//              gradient of step t+1 (needs step t+1's link-choice VJPs from
//              R4 of the previous iteration); arrived list: per-row top-2 of
//              the uniform-utility Gumbel draws for A[0]'s rows.
//   R3 links   merge-row VJP (transfer seeds a_bar, softmax VJP, targeted
//              routing to the first candidate); A[0] rows; slots: transfer /
//              replace_rows pass-through, counting sigmoid VJP, car-following
//              VJP with the follower's headway term -> x_bar of layout t.
//   R4         link-choice VJP per arrived head; warp per link: deterministic
//              u / kappa / alpha reductions; resets for the next step.
// Gradients accumulate per step in the reference's order (engine.cpp:410-414).
#include <cooperative_groups.h>

#include <climits>
#include <cstdint>

#include "dtg_backward.h"
#include "dtg_device.cuh"
#include "dtg_merge.cuh"

namespace cg = cooperative_groups;

#ifndef DTG_BAR_BACKOFF
#define DTG_BAR_BACKOFF 32  // ns between grid-barrier polls: C3 nowcast 1.305 -> 1.295 ms
#endif

namespace dtg {

namespace {

#ifndef DTG_BWD_THREADS
#define DTG_BWD_THREADS 512
#endif
constexpr int kBT = DTG_BWD_THREADS;  // threads per CTA
constexpr int kFastDeg = 5;  // successor counts up to this take unrolled register paths
constexpr int kHeadCap = 1024;  // deferred arrived heads per CTA (overflow runs inline)
#ifndef DTG_KB3
#define DTG_KB3 2
#endif
constexpr int kB3 = DTG_KB3;  // R1 / R3 slots per thread in flight
#ifndef DTG_R4_THREADS
#define DTG_R4_THREADS 192
#endif
constexpr int kR4T = DTG_R4_THREADS;  // threads running R4 of step t + 1 beside R1 of step t
#ifndef DTG_M3_THREADS
#define DTG_M3_THREADS 128
#endif
constexpr int kM3T = DTG_M3_THREADS;  // R3 threads for the merge and A[0] rows (the rest: position adjoint)

__device__ __forceinline__ int findl(const int* off_s, int L, int k) {
  int lo = 0, hi = L - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off_s[mid] <= k)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Item index of thread `tid` of the scenario's CTA `lg` (of nblk): 32-item
// groups are dealt round-robin over the CTAs first, so a short item list
// (links, arrived agents) spreads over all SMs instead of filling the first
// CTAs' schedulers.  Stride: nblk * (threads per CTA taking part).
__device__ __forceinline__ int spread(int tid, int lg, int nblk) {
  return ((tid >> 5) * nblk + lg) * 32 + (tid & 31);
}

__device__ __forceinline__ double adm_bar(double xb, double x1, double M) {
  double r = 0.0;
  r += xb * (-M);
  r += -1.0 * (xb * x1);
  return r;
}

struct T2 {
  double y1, y2;
  int id1, s1;
};
__device__ __forceinline__ void t2_push(T2& T, double y, int id, int slot) {
  if (y > T.y1 || (y == T.y1 && id < T.id1)) {
    T.y2 = fmax(T.y2, T.y1);
    T.y1 = y;
    T.id1 = id;
    T.s1 = slot;
  } else {
    T.y2 = fmax(T.y2, y);
  }
}
__device__ __forceinline__ void t2_merge(T2& A, const T2& B) {
  if (B.y1 > A.y1 || (B.y1 == A.y1 && B.id1 < A.id1)) {
    A.y2 = fmax(fmax(A.y2, B.y2), A.y1);
    A.y1 = B.y1;
    A.id1 = B.id1;
    A.s1 = B.s1;
  } else {
    A.y2 = fmax(fmax(A.y2, B.y2), B.y1);
  }
}

// new slot (layout t+1) of layout-t slot k on link j (rank r)
__device__ __forceinline__ int map_next(const BView& V, int b, int par, int k, int j, int r,
                                        const int* offT, const int* offN, bool* mover) {
  const DevView& d = V.d;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const int na = V.nA_cur[bl + j];
  if (r < na && V.won[bn + k]) {
    *mover = true;
    return offN[V.choice[static_cast<std::size_t>(par) * d.B * d.N + bn + k] + 1] - 1;  // tail of the row it won
  }
  *mover = false;
  int dd;
  if (r >= na) {
    dd = V.dep[bl + j];
  } else {
    dd = 0;
    const int base = offT[j];
    for (int q = base; q < k; ++q) dd += V.won[bn + q];
  }
  return offN[j] + r - dd;
}

// adjoint of the new position x1 of slot k (transfer + counting)
__device__ __forceinline__ double x1_bar_p(const BView& V, int b, int par, int k, int j, int r, double x1,
                                           const int* offT, const int* offN, const double* xbn) {
  const DevView& d = V.d;
  bool mover;
  const int ns = map_next(V, b, par, k, j, r, offT, offN, &mover);
  double xb = (mover && !d.tg) ? 0.0 : xbn[ns];
  const double qt = V.qtot[static_cast<std::size_t>(b) * d.L + j];
  if (qt != 0.0) {
    const double len = d.len[j];
    const double sc = d.sc[j];
    const double z = (x1 + (-(0.5 * len))) * sc;
    const double sg = z >= 0.0 ? 1.0 / (1.0 + dexp(-z)) : dexp(z) / (1.0 + dexp(z));
    xb = xb + (((qt * 1.0) * sg) * (1.0 - sg)) * sc;
  }
  return xb;
}

__device__ __forceinline__ void bstamp(const BView& V, int t, int w) {
  if (V.tstamp == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    V.tstamp[(static_cast<std::size_t>(t) * gridDim.x + blockIdx.x) * 8 + w] = ns;
  }
}

// Link-choice replay of one arrived head in R1 (pi kept for R4) and its
// registration as a merge candidate of the chosen row.
__device__ __forceinline__ void replay_head(const BView& V, int b, int t, int k, int j, int a) {
  const DevView& d = V.d;
  // per-slot head records and candidate counts are kept per step parity: R4 of
  // step t + 1 reads its own while R1 of step t writes these
  const std::size_t par = static_cast<std::size_t>(t & 1);
  const std::size_t bn = par * d.B * d.N + static_cast<std::size_t>(b) * d.N;
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t blp = par * d.B * d.L + bl;
  const int s0 = d.succ_off[j], deg = (V.dbg & 1) ? 0 : d.succ_off[j + 1] - s0;
  int c = -1;
  if (deg > 0) {
    const double* lz = d.slogz + (bl + j) * d.maxdeg;
    const std::uint64_t h2l =
        rng_prefix2(rng_prefix1(d.seed_link[b], static_cast<std::uint64_t>(t)), static_cast<std::uint64_t>(a));
    double* lp = V.lpi + (bn + k) * d.maxdeg;
    int ed;
    if (deg <= kFastDeg) {  // unrolled: independent draw chains interleave
      int sc[kFastDeg];
      double y[kFastDeg], ex[kFastDeg];
#pragma unroll
      for (int e = 0; e < kFastDeg; ++e) sc[e] = d.succ[s0 + (e < deg ? e : 0)];
      double gg[kFastDeg];  // the five draw chains batched
      gumbel_draws<kFastDeg>(h2l, sc, gg);
#pragma unroll
      for (int e = 0; e < kFastDeg; ++e) y[e] = (lz[e < deg ? e : 0] + gg[e]) * d.kinv;
      // the logits are kept (R4 forms pi from them with softmax_stage2's
      // operations); the choice is the first argmax, read off the logits
#pragma unroll
      for (int e = 0; e < kFastDeg; ++e)
        if (e < deg) lp[e] = y[e];
      ed = softmax_first_argmax<kFastDeg>(deg, y, ex);
      c = sc[0];
#pragma unroll
      for (int e = 1; e < kFastDeg; ++e)
        if (e == ed) c = sc[e];
    } else {
      double g[kMaxDeg], pi[kMaxDeg];
      for (int e = 0; e < deg; ++e) g[e] = gumbel_bits(rng_final(h2l, static_cast<std::uint64_t>(d.succ[s0 + e])));
      ed = softmax_stage2<kMaxDeg>(deg, lz, g, d.kinv, pi);
      c = d.succ[s0 + ed];
      for (int e = 0; e < deg; ++e) lp[e] = (lz[e] + g[e]) * d.kinv;  // logits, as in softmax_stage2
    }
    const int qq = atomicAdd(&V.ccnt[blp + c], 1);  // round trip overlaps the merge draw
    const std::uint64_t mb = rng_final(rng_prefix2(rng_prefix1(d.seed_merge[b], static_cast<std::uint64_t>(t)),
                                                   static_cast<std::uint64_t>(c)),
                                       static_cast<std::uint64_t>(a));
    int mbad = 0;
    double gmc = gumbel_sl(mb, mbad);
    if (mbad) gmc = gumbel_bits(mb);
    V.ched[bn + k] = ed;
    Cand cd;
    cd.alpha = d.alpha[bl + j];
    cd.g = gmc;
    cd.slot = k;
    cd.aid = a;
    cd.link = j;
    cd.pad = 0;
    if (qq < kBwdCandCap) V.cands[(bl + c) * kBwdCandCap + qq] = cd;
  }
  V.choice[bn + k] = c;
}

}  // namespace

__global__ void __launch_bounds__(kBT) k_backward_persistent(BView V) {
  extern __shared__ int smb[];
  // grid barrier: a CTA barrier, then one release-add per CTA on a monotone
  // counter and an acquire spin (measured ~30% faster for this sweep than
  // cooperative_groups' grid.sync); cg's barrier when no counter is given
  unsigned int epoch = 0;
  auto grid_sync = [&]() {
    if (V.gbar == nullptr) {
      cg::this_grid().sync();
      return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      ++epoch;
      const unsigned int target = epoch * gridDim.x;
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(V.gbar), "r"(1u) : "memory");
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(V.gbar) : "memory");
#if DTG_BAR_BACKOFF
            if (v < target) __nanosleep(DTG_BAR_BACKOFF);
#endif
      } while (v < target);
    }
    __syncthreads();
  };
  const DevView& d = V.d;
  const int L = d.L, N = d.N;
  int* offT = smb;
  int* offN = smb + (L + 1);
  T2* red = reinterpret_cast<T2*>(smb + 2 * (L + 1) + ((2 * (L + 1)) & 1));  // [kBT/32][maxdeg]
  int* hcnt = reinterpret_cast<int*>(red + (kBT / 32) * d.maxdeg);  // deferred-head count
  int* hq = hcnt + 4;  // [3][kHeadCap] deferred heads: slot, link, agent
  const bool grouped = V.bps > 0;
  const int b0 = grouped ? blockIdx.x / V.bps : blockIdx.x;
  const int lg = grouped ? blockIdx.x % V.bps : 0;
  const int nblk = grouped ? V.bps : 1;
  const int bstep = grouped ? d.B : gridDim.x;
  const bool active = grouped ? (b0 < d.B) : true;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int T = V.T;

  // R0: seeds
  if (active)
    for (int b = b0; b < d.B; b += bstep) {
      const std::size_t bn = static_cast<std::size_t>(b) * N, bl = static_cast<std::size_t>(b) * L;
      const std::size_t sf = sidx(d, T % d.S, b);
      double* xb = V.xbar + static_cast<std::size_t>(T & 1) * d.B * N + bn;
      for (int k = lg * kBT + tid; k < N; k += nblk * kBT)
        xb[k] = V.x_seed ? V.x_seed[bn + d.aid[sf + k]] : 0.0;
      double* g = V.grads + static_cast<std::size_t>(b) * 5 * L;
      for (int j = lg * kBT + tid; j < L; j += nblk * kBT) {
        V.cbar[bl + j] = V.cum_seed ? V.cum_seed[bl + j] : 0.0;
        V.qbar[bl + j] = 0.0;
        for (int c = 0; c < 5; ++c) g[c * L + j] = 0.0;
      }
    }
  grid_sync();

  // R4 of step t4 for scenario b (o4: layout t4's offsets in shared memory;
  // threads tid4 < nt4 of the CTA take part):
  // the link-choice VJP per arrived head, the u / kappa / alpha reductions and
  // the departures reset.  It runs in the same phase as R1 of step t4 - 1
  // (one grid barrier less per step, and the two phases' dependency chains
  // overlap): every buffer R4 reads that R1 writes (head records, arrived
  // list and prefix lengths, candidate counts) is kept per step parity.
  auto r4 = [&](int b, int t4, const int* o4, int tid4, int nt4) {
    const int p4 = t4 & 1;
      const std::size_t bn = static_cast<std::size_t>(b) * N, bl = static_cast<std::size_t>(b) * L;
      const std::size_t bnp = static_cast<std::size_t>(p4) * d.B * N + bn;  // this step's head records
      const std::size_t so = sidx(d, t4 % d.S, b);
      double* vbc = V.vbar + (static_cast<std::size_t>(p4) * d.B * N + bn) * d.maxdeg;
      const unsigned long long key = V.a0key[p4 * d.B + b];
      const int a0s = key == ULLONG_MAX ? -1 : static_cast<int>(key & 0xffffffffull);
      const int nA = V.acount[p4 * d.B + b];
      for (int q = spread(tid4, lg, nblk); q < nA && !(V.dbg & 512); q += nblk * nt4) {
        const int s = V.alist[bnp + q];
        const int c = V.choice[bnp + s];
        if (c < 0) continue;
        const int j = d.lnk[so + s];
        const int s0 = d.succ_off[j], deg = d.succ_off[j + 1] - s0;
        const double* lz = d.slogz + (bl + j) * d.maxdeg;
        const double* lp = V.lpi + (bnp + s) * d.maxdeg;
        const int ed = V.ched[bnp + s];
        const double lrow = (V.vac[bl + c] && V.win[bl + c] >= 0) ? V.lbar_row[bn + s] : 0.0;
        const bool hit = V.vac[bl + c] && V.win[bl + c] >= 0;
        const double* la0 = V.lbar_a0 + static_cast<std::size_t>(b) * d.maxdeg;
        if (deg <= kFastDeg) {  // registers, same operation order as two_softmax_vjp
          double bar[kFastDeg], pi[kFastDeg];
          {  // pi from the replayed logits: softmax_stage2's operations
            double yv[kFastDeg];
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e) yv[e] = e < deg ? lp[e] : 0.0;
            double m2 = yv[0];
#pragma unroll
            for (int e = 1; e < kFastDeg; ++e)
              if (e < deg && m2 < yv[e]) m2 = yv[e];
            double z2 = 0.0;
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e) {
              pi[e] = dexp(yv[e] - m2);
              if (e < deg) z2 += pi[e];
            }
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e) pi[e] = e < deg ? pi[e] / z2 : 0.0;
          }
#pragma unroll
          for (int e = 0; e < kFastDeg; ++e) {
            const bool on = e < deg;
            double v = (hit && e == ed) ? lrow : 0.0;
            if (on && s == a0s) v += la0[e];
            bar[e] = on ? ((v * 1.0) * 1.0) * (V.vac[bl + d.succ[s0 + e]] ? 1.0 : 0.0) : 0.0;
          }
          double dot = 0.0;
#pragma unroll
          for (int e = 0; e < kFastDeg; ++e)
            if (e < deg) dot += bar[e] * pi[e];
          double gs = 0.0;
#pragma unroll
          for (int e = 0; e < kFastDeg; ++e)
            if (e < deg) {
              bar[e] = (pi[e] * (bar[e] - dot)) * d.kinv;
              gs += bar[e];
            }
#pragma unroll
          for (int e = 0; e < kFastDeg; ++e)
            if (e < deg) vbc[static_cast<std::size_t>(s) * d.maxdeg + e] = bar[e] - dexp(lz[e]) * gs;
        } else {
          double bar[kMaxDeg], pi[kMaxDeg];
          {  // pi from the replayed logits: softmax_stage2's operations
            double m2 = lp[0];
            for (int e = 1; e < deg; ++e)
              if (m2 < lp[e]) m2 = lp[e];
            double z2 = 0.0;
            for (int e = 0; e < deg; ++e) z2 += dexp(lp[e] - m2);
            for (int e = 0; e < deg; ++e) pi[e] = dexp(lp[e] - m2) / z2;
          }
          for (int e = 0; e < deg; ++e) bar[e] = 0.0;
          if (hit) bar[ed] = lrow;
          if (s == a0s)
            for (int e = 0; e < deg; ++e) bar[e] += la0[e];
          for (int e = 0; e < deg; ++e)
            bar[e] = ((bar[e] * 1.0) * 1.0) * (V.vac[bl + d.succ[s0 + e]] ? 1.0 : 0.0);
          two_softmax_vjp(deg, lz, pi, d.kinv, bar);
          for (int e = 0; e < deg; ++e) vbc[static_cast<std::size_t>(s) * d.maxdeg + e] = bar[e];
        }
      }
      // warp per link: u, kappa, alpha for step t
      double* g5 = V.grads + static_cast<std::size_t>(b) * 5 * L;
      // thread per link (links dealt in 32-lane groups over the CTAs): the
      // segment sums run in slot order; the parameter loads of the epilogue
      // are issued together
      for (int j = spread(tid4, lg, nblk); j < L && !(V.dbg & 1024); j += nblk * nt4) {
        const int base = o4[j], n = o4[j + 1] - base;
        const double kap = d.kappa[bl + j];
        const double g0 = g5[j], g1 = g5[L + j], g3 = g5[3 * L + j];
        const int na = n ? V.nAb[static_cast<std::size_t>(p4) * d.B * L + bl + j] : 0;
        double ub, jb;
        link_sums8(V.cu + bn, V.cg + bn, base, n, ub, jb);
        if (n) {
          g5[j] = g0 + (0.0 + ub);
          g5[L + j] = g1 + (0.0 - jb * static_cast<double>(d.delta_n) / (kap * kap));
        }
        double ab = 0.0;
        for (int r = 0; r < na; ++r) {
          const int s = base + r;
          const int ch = V.choice[bnp + s];
          if (ch >= 0 && V.vac[bl + ch] && V.win[bl + ch] >= 0) ab += 1.0 * V.prio_bar[bn + s];
        }
        g5[3 * L + j] = g3 + ab;
      }
      for (int i = lg * nt4 + tid4; i < L; i += nblk * nt4) V.dep[bl + i] = 0;
  };

  for (int t = T - 1; t >= 0; --t) {
    const int par = t & 1;
    const int snap_k = ((t + 1) % V.spi == 0) ? (t + 1) / V.spi - 1 : -1;
    bstamp(V, t, 0);
    // ================= R1: replay f + link choice =================
    if (active)
      for (int b = b0; b < d.B; b += bstep) {
        __syncthreads();
        const int* og = d.off + oidx(d, t % d.S, b);
        const int* ogn = d.off + oidx(d, (t + 1) % d.S, b);
        for (int j = tid; j <= L; j += kBT) {
          offT[j] = og[j];
          offN[j] = ogn[j];
        }
        __syncthreads();
        // R4 of step t + 1 on the first kR4T threads, R1 on the others: the
        // two phases' dependency chains run side by side
        const bool with4 = t + 1 < T;
        const int t1 = with4 ? tid - kR4T : tid, n1 = with4 ? kBT - kR4T : kBT;
        if (with4 && tid < kR4T) {
          r4(b, t + 1, offN, tid, kR4T);  // layout t + 1 = step t + 1's
        } else {
        auto r1_sync = [&]() {
          if (with4)
            asm volatile("bar.sync 2, %0;" ::"r"(kBT - kR4T) : "memory");
          else
            __syncthreads();
        };
        const std::size_t bn = static_cast<std::size_t>(b) * N, bl = static_cast<std::size_t>(b) * L;
        const std::size_t so = sidx(d, t % d.S, b);
        int* nAc = V.nA_cur + bl;  // nA of layout t (parity slot par)
        int* nAw = V.nAb + static_cast<std::size_t>(par) * d.B * L + bl;
        // several slots per thread: queue the arrived heads in shared memory
        // and replay their link choices after the slot loop, one per thread
        const bool defer = N - lg * n1 > nblk * n1;
        if (t1 == 0) *hcnt = 0;
        r1_sync();
        // kB3 slots per thread in flight; a slot's follower arrival flag is the
        // next lane's own (lanes are consecutive slots), so only a warp's last
        // lane replays its follower's car-following itself.
        const int stride1 = nblk * n1;
        for (int k0 = lg * n1 + t1; k0 - lane < N; k0 += kB3 * stride1) {
          int kk[kB3], jj[kB3], rr[kB3], nn[kB3];
          double xx[kB3], xp[kB3], xf[kB3];
#pragma unroll
          for (int q = 0; q < kB3; ++q) {
            const int k = k0 + q * stride1;
            const bool on = k < N;
            kk[q] = k;
            const int j = on ? d.lnk[so + k] : 0;
            jj[q] = j;
            const int base = offT[j];
            rr[q] = k - base;
            nn[q] = offT[j + 1] - base;
            xx[q] = on ? d.pos[so + k] : 0.0;
            xp[q] = (on && rr[q] > 0) ? d.pos[so + k - 1] : 0.0;
            xf[q] = (on && lane == 31 && rr[q] + 1 < nn[q]) ? d.pos[so + k + 1] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < kB3; ++q) {
            const int k = kk[q], j = jj[q], r = rr[q], n = nn[q];
            const bool on = k < N;
            bool fa = false, fa_n = false;
            double x1 = 0.0;
            if (on) {
              const double jam = d.jam[bl + j], dxf = d.dxf[bl + j], len = d.len[j];
              const double thr = d.thr[j];
              const double x = xx[q];
              x1 = cf_step(x, r == 0 ? d.M : xp[q] - x, jam, dxf, len).x1;
              fa = x1 >= thr;
              if (lane == 31 && r + 1 < n) fa_n = cf_step(xf[q], x - xf[q], jam, dxf, len).x1 >= thr;
            }
            const bool fdown = __shfl_down_sync(0xffffffffu, fa, 1);
            // arrived list and A[0] key: one atomic per warp (warp-aggregated)
            const bool arr = on && fa;
            const int a = arr ? d.aid[so + k] : 0;
            int qa = 0;
            const unsigned am = __ballot_sync(0xffffffffu, arr);
            if (am && !(V.dbg & 4)) {
              const int leader = __ffs(am) - 1;
              int base = 0;
              if (lane == leader) base = atomicAdd(&V.acount[par * d.B + b], __popc(am));
              base = __shfl_sync(0xffffffffu, base, leader);
              qa = base + __popc(am & ((1u << lane) - 1u));
              unsigned long long key =
                  arr ? ((static_cast<unsigned long long>(a) << 32) | static_cast<unsigned>(k)) : ULLONG_MAX;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
                key = other < key ? other : key;
              }
              if (lane == leader) atomicMin(&V.a0key[par * d.B + b], key);
            }
            if (!on) continue;
            if (lane < 31) fa_n = r + 1 < n && fdown;
            V.x1[bn + k] = x1;
            if (r == 0 && !fa) {
              nAw[j] = 0;
              nAc[j] = 0;
            }
            if (fa && !fa_n) {
              nAw[j] = r + 1;
              nAc[j] = r + 1;
            }
            if (r == n - 1) V.tail[bl + j] = x1;
            if (fa) {
              V.won[bn + k] = 0;
              if (!(V.dbg & 4)) V.alist[static_cast<std::size_t>(par) * d.B * N + bn + qa] = k;
              if (defer) {
                const int hi = atomicAdd(hcnt, 1);
                if (hi < kHeadCap) {
                  hq[hi] = k;
                  hq[kHeadCap + hi] = j;
                  hq[2 * kHeadCap + hi] = a;
                } else {
                  replay_head(V, b, t, k, j, a);
                }
              } else {
                replay_head(V, b, t, k, j, a);
              }
            }
          }
        }
        if (defer) {
          r1_sync();
          const int nh = min(*hcnt, kHeadCap);
          for (int i = t1; i < nh; i += n1) replay_head(V, b, t, hq[i], hq[kHeadCap + i], hq[2 * kHeadCap + i]);
        }
        }
      }
    bstamp(V, t, 1);
    grid_sync();
    bstamp(V, t, 2);
    // ================= R2: count adjoint, merge replay, deferred pref, A0 partials =====
    if (active && !(V.dbg & 2048))
      for (int b = b0; b < d.B; b += bstep) {
        if (!grouped) {  // scenario loop: reload this scenario's offsets
          __syncthreads();
          const int* og = d.off + oidx(d, t % d.S, b);
          const int* ogn = d.off + oidx(d, (t + 1) % d.S, b);
          for (int j = tid; j <= L; j += kBT) {
            offT[j] = og[j];
            offN[j] = ogn[j];
          }
          __syncthreads();
        }
        const std::size_t bn = static_cast<std::size_t>(b) * N, bl = static_cast<std::size_t>(b) * L;
        const std::size_t so = sidx(d, t % d.S, b);
        const std::size_t sn = sidx(d, (t + 1) % d.S, b);
        double* g5 = V.grads + static_cast<std::size_t>(b) * 5 * L;
        const int* nAn = V.nAb + static_cast<std::size_t>(par ^ 1) * d.B * L + bl;  // layout t+1
        const double* vbn = V.vbar + (static_cast<std::size_t>(par ^ 1) * d.B * N + bn) * d.maxdeg;
        // the CTA's two halves run concurrently: warps [0, 8) the per-link work,
        // warps [8, 16) the A[0] row partials over the arrived list
        constexpr int kHalf = kBT / 2;
        if (tid < kHalf) {
        for (int i = spread(tid, lg, nblk); i < L; i += nblk * kHalf) {
          if (snap_k >= 0 && V.snap_seed)
            V.cbar[bl + i] += V.snap_seed[(static_cast<std::size_t>(b) * V.K + snap_k) * L + i];
          const double cb = V.cbar[bl + i];
          const double a = d.qh[hidx(d, t + 1, b) + i] - d.qh[hidx(d, t, b) + i];
          const bool pick = a >= 0.0;
          V.qtot[bl + i] = V.qbar[bl + i] + (pick ? cb : 0.0);
          V.qbar[bl + i] = pick ? -1.0 * cb : 0.0;
          const int n_i = offT[i + 1] - offT[i];
          const double tx = n_i ? V.tail[bl + i] : d.M;
          const bool vacant = tx > d.jam[bl + i];
          V.vac[bl + i] = vacant;
          const int cnt = (V.dbg & 8) ? 0 : V.ccnt[static_cast<std::size_t>(par) * d.B * L + bl + i];
          V.ccnt[static_cast<std::size_t>(par ^ 1) * d.B * L + bl + i] = 0;  // for R1 of step t - 1
          int w = -1;
          if (vacant && cnt > 0) {
            if (cnt > kBwdCandCap) {
              atomicOr(&d.err[b], kErrCandOverflow);
            } else if (cnt <= kFastDeg) {  // registers (dtg_merge.cuh)
              Cand c[kFastDeg];
              double lz[kFastDeg], pi[kFastDeg];
              const int best = merge_softmax_fast<kFastDeg>(cnt, V.cands + (bl + i) * kBwdCandCap, d.kinv, c, lz, pi);
#pragma unroll
              for (int e = 0; e < kFastDeg; ++e)
                if (e < cnt) {
                  V.cands[(bl + i) * kBwdCandCap + e] = c[e];
                  V.mpi[(bl + i) * kBwdCandCap + e] = pi[e];
                  V.mlz[(bl + i) * kBwdCandCap + e] = lz[e];
                }
              const Cand cb = pick_cand(c, best);
              w = cb.slot;
              V.won[bn + w] = 1;
              atomicAdd(&V.dep[bl + cb.link], 1);
            } else {
              Cand c[kBwdCandCap];
              for (int e = 0; e < cnt; ++e) c[e] = V.cands[(bl + i) * kBwdCandCap + e];
              for (int x = 1; x < cnt; ++x) {
                const Cand key = c[x];
                int m = x - 1;
                while (m >= 0 && c[m].aid > key.aid) {
                  c[m + 1] = c[m];
                  --m;
                }
                c[m + 1] = key;
              }
              double v[kBwdCandCap], g[kBwdCandCap], lz[kBwdCandCap], pi[kBwdCandCap];
              for (int e = 0; e < cnt; ++e) {
                v[e] = c[e].alpha;
                g[e] = c[e].g;
              }
              const int best = two_softmax<kBwdCandCap>(cnt, v, g, d.kinv, lz, pi);
              for (int e = 0; e < cnt; ++e) {
                V.cands[(bl + i) * kBwdCandCap + e] = c[e];
                V.mpi[(bl + i) * kBwdCandCap + e] = pi[e];
                V.mlz[(bl + i) * kBwdCandCap + e] = lz[e];
              }
              w = c[best].slot;
              V.won[bn + w] = 1;
              atomicAdd(&V.dep[bl + c[best].link], 1);
            }
          }
          V.win[bl + i] = w;
          (void)sn;
        }
        } else {
        const int ta = tid - kHalf, wa = ta >> 5;
        // A[0]'s rows: per-row top-2 over the arrived list
        const unsigned long long key = V.a0key[par * d.B + b];
        const int nA = V.acount[par * d.B + b];
        if (key != ULLONG_MAX && !(V.dbg & 32)) {
          const int a0s = static_cast<int>(key & 0xffffffffull);
          const int c0 = d.lnk[so + a0s];
          const int s0 = d.succ_off[c0], deg0 = d.succ_off[c0 + 1] - s0;
          const double vv = 0.0 - kMaskLarge;
          const double lzv = dlog(static_cast<double>(nA) * 1.0) + vv;
          const double logz = vv - lzv;
          // one draw per thread: items (row e, arrived q) row-major with each row
          // padded to whole warps, so a warp reduces a single row; every warp
          // folds its groups into its own per-row slot
          const std::uint64_t h1m = rng_prefix1(d.seed_merge[b], static_cast<std::uint64_t>(t));
          const int nAp = (nA + 31) & ~31;
          const int nitems = deg0 * nAp;
          if (lane < d.maxdeg) red[wa * d.maxdeg + lane] = T2{-INFINITY, -INFINITY, INT_MAX, -1};
          __syncwarp();
          for (int i = spread(ta, lg, nblk); i - lane < nitems; i += nblk * kHalf) {
            const int e = (i - lane) / nAp, q = i - e * nAp;
            T2 x{-INFINITY, -INFINITY, INT_MAX, -1};
            if (q < nA) {
              const int s = V.alist[static_cast<std::size_t>(par) * d.B * N + bn + q];
              const int id = d.aid[so + s];
              const std::uint64_t bits = rng_final(rng_prefix2(h1m, static_cast<std::uint64_t>(d.succ[s0 + e])),
                                                   static_cast<std::uint64_t>(id));
              int bad = 0;
              double g = gumbel_sl(bits, bad);
              if (bad) g = gumbel_bits(bits);
              x.y1 = (logz + g) * d.kinv;
              x.id1 = id;
              x.s1 = s;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              T2 y;
              y.y1 = __shfl_xor_sync(0xffffffffu, x.y1, o);
              y.y2 = __shfl_xor_sync(0xffffffffu, x.y2, o);
              y.id1 = __shfl_xor_sync(0xffffffffu, x.id1, o);
              y.s1 = __shfl_xor_sync(0xffffffffu, x.s1, o);
              t2_merge(x, y);
            }
            if (lane == 0) t2_merge(red[wa * d.maxdeg + e], x);
            __syncwarp();
          }
          asm volatile("bar.sync 1, %0;" ::"r"(kHalf) : "memory");  // the A[0] half only
          if (ta < deg0) {
            T2 x = red[ta];
            for (int w2 = 1; w2 < kHalf / 32; ++w2) t2_merge(x, red[w2 * d.maxdeg + ta]);
            static_cast<T2*>(V.a0part)[(static_cast<std::size_t>(b) * nblk + lg) * d.maxdeg + ta] = x;
          }
          asm volatile("bar.sync 1, %0;" ::"r"(kHalf) : "memory");
        }
        // deferred: the preference gradient of step t+1 (its link-choice VJPs
        // came from R4 of step t+1 in the phase before), on the A[0] half once
        // its rows are done: the link half's merge replays are the longer chain
        if (t + 1 < T && !(V.dbg & 16))
          for (int i = spread(ta, lg, nblk); i < L; i += nblk * kHalf) {
            double pb = 0.0;
            const int e0 = d.pred_off[i], ne = d.pred_off[i + 1] - e0;
            if (ne <= kFastDeg) {
              // every predecessor's arrived count and first row load together;
              // the sum then runs in (predecessor, row) order
              int pbse[kFastDeg], nap[kFastDeg], pps[kFastDeg];
              double v0[kFastDeg];
#pragma unroll
              for (int q = 0; q < kFastDeg; ++q) {
                nap[q] = 0;
                pbse[q] = 0;
                pps[q] = 0;
                if (q < ne) {
                  const int p = d.pred[e0 + q];
                  pps[q] = d.pred_pos[e0 + q];
                  pbse[q] = offN[p];
                  nap[q] = offN[p + 1] == pbse[q] ? 0 : nAn[p];
                }
              }
#pragma unroll
              for (int q = 0; q < kFastDeg; ++q)
                v0[q] = nap[q] > 0 ? vbn[static_cast<std::size_t>(pbse[q]) * d.maxdeg + pps[q]] : 0.0;
#pragma unroll
              for (int q = 0; q < kFastDeg; ++q)
                if (nap[q] > 0) {
                  pb += v0[q] * 1.0;
                  for (int r = 1; r < nap[q]; ++r)
                    pb += vbn[static_cast<std::size_t>(pbse[q] + r) * d.maxdeg + pps[q]] * 1.0;
                }
            } else {
              for (int q = 0; q < ne; ++q) {
                const int p = d.pred[e0 + q];
                const int pbse = offN[p];
                if (offN[p + 1] == pbse) continue;
                const int nap = nAn[p];
                for (int r = 0; r < nap; ++r)
                  pb += vbn[static_cast<std::size_t>(pbse + r) * d.maxdeg + d.pred_pos[e0 + q]] * 1.0;
              }
            }
            const double cst = d.cost[bl + i], be = d.beta[bl + i];
            g5[2 * L + i] += 0.0 + pb / cst;
            g5[4 * L + i] += 0.0 - pb * be / (cst * cst);
          }
        }
      }
    bstamp(V, t, 3);
    grid_sync();
    bstamp(V, t, 4);
    // ================= R3: merge VJP, A0 rows, position adjoint =================
    if (active)
      for (int b = b0; b < d.B; b += bstep) {
        if (lg == 0 && tid == 0) {  // for R1 of step t - 1 (R4 of step t + 1 read them last)
          V.acount[(par ^ 1) * d.B + b] = 0;
          V.a0key[(par ^ 1) * d.B + b] = ULLONG_MAX;
        }
        if (!grouped) {
          __syncthreads();
          const int* og = d.off + oidx(d, t % d.S, b);
          const int* ogn = d.off + oidx(d, (t + 1) % d.S, b);
          for (int j = tid; j <= L; j += kBT) {
            offT[j] = og[j];
            offN[j] = ogn[j];
          }
          __syncthreads();
        }
        const std::size_t bn = static_cast<std::size_t>(b) * N, bl = static_cast<std::size_t>(b) * L;
        const std::size_t so = sidx(d, t % d.S, b);
        const double* xbn = V.xbar + static_cast<std::size_t>(par ^ 1) * d.B * N + bn;
        double* xbc = V.xbar + static_cast<std::size_t>(par) * d.B * N + bn;
        // merge rows and A[0] rows on the first kM3T threads, the position
        // adjoint on the others: the merge-row chains overlap the slot chains
        if (tid < kM3T) {
        for (int i = spread(tid, lg, nblk); i < L && !(V.dbg & 64); i += nblk * kM3T) {
          const int w = V.win[bl + i];
          if (w < 0) continue;
          const int cnt = V.ccnt[static_cast<std::size_t>(par) * d.B * L + bl + i];
          const Cand* cc = V.cands + (bl + i) * kBwdCandCap;
          const double abar_w = xbn[offN[i + 1] - 1] * d.M + 0.0;
          if (cnt <= kFastDeg) {  // registers; two_softmax_vjp's operation order
            Cand cf[kFastDeg];
            double bar[kFastDeg], lz[kFastDeg], pi[kFastDeg];
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e) {
              bar[e] = 0.0;
              lz[e] = 0.0;
              pi[e] = 0.0;
              if (e < cnt) {
                cf[e] = cc[e];
                lz[e] = V.mlz[(bl + i) * kBwdCandCap + e];
                pi[e] = V.mpi[(bl + i) * kBwdCandCap + e];
              }
            }
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e)
              if (e < cnt) {
                const int s = cf[e].slot;
                if (s == w) {
                  bar[e] = abar_w * 1.0;
                } else {
                  const int p = cf[e].link;
                  const int base = offT[p];
                  int dd = 0;
                  for (int q = base; q < s; ++q) dd += V.won[bn + q];
                  const double xb = xbn[offN[p] + (s - base) - dd];
                  bar[e] = adm_bar(xb, V.x1[bn + s], d.M) * 1.0;
                }
              }
            double dot = 0.0;
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e)
              if (e < cnt) dot += bar[e] * pi[e];
            double gs = 0.0;
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e)
              if (e < cnt) {
                bar[e] = (pi[e] * (bar[e] - dot)) * d.kinv;
                gs += bar[e];
              }
#pragma unroll
            for (int e = 0; e < kFastDeg; ++e)
              if (e < cnt) {
                const double bv = bar[e] - dexp(lz[e]) * gs;
                const int s = cf[e].slot;
                V.lbar_row[bn + s] = (e == 0 ? 0.0 + abar_w : 0.0) + bv * cf[e].alpha;
                V.prio_bar[bn + s] = 0.0 + bv * 1.0;
              }
            continue;
          }
          double bar[kBwdCandCap], lz[kBwdCandCap], pi[kBwdCandCap];
          for (int e = 0; e < cnt; ++e) {
            lz[e] = V.mlz[(bl + i) * kBwdCandCap + e];
            pi[e] = V.mpi[(bl + i) * kBwdCandCap + e];
            const int s = cc[e].slot;
            if (s == w) {
              bar[e] = abar_w * 1.0;
            } else {
              const int p = cc[e].link;
              const int base = offT[p];
              int dd = 0;
              for (int q = base; q < s; ++q) dd += V.won[bn + q];
              const double xb = xbn[offN[p] + (s - base) - dd];
              bar[e] = adm_bar(xb, V.x1[bn + s], d.M) * 1.0;
            }
          }
          two_softmax_vjp(cnt, lz, pi, d.kinv, bar);
          for (int e = 0; e < cnt; ++e) {
            const int s = cc[e].slot;
            V.lbar_row[bn + s] = (e == 0 ? 0.0 + abar_w : 0.0) + bar[e] * cc[e].alpha;
            V.prio_bar[bn + s] = 0.0 + bar[e] * 1.0;
          }
        }
        // A[0] rows: warp e of the scenario's last CTA (the one with the fewest
        // slots in the interleaved mapping) merges row e's per-CTA partials and
        // writes lbar_a0[e] (0 for rows that take no A[0] routing)
        const unsigned long long key = lg == nblk - 1 ? V.a0key[par * d.B + b] : ULLONG_MAX;
        if (lg == nblk - 1 && key != ULLONG_MAX && !(V.dbg & 128))
        for (int e = wid; e < d.maxdeg; e += kM3T / 32) {
          const int a0s = static_cast<int>(key & 0xffffffffull);
          const int c0 = d.lnk[so + a0s];
          const int s0 = d.succ_off[c0], deg0 = d.succ_off[c0 + 1] - s0;
          bool routed = false;
          if (e < deg0) {
            const int i = d.succ[s0 + e];
            routed = V.vac[bl + i] && V.win[bl + i] < 0;
            if (routed) {
              const T2* ap = static_cast<const T2*>(V.a0part);
              T2 x{-INFINITY, -INFINITY, INT_MAX, -1};
              for (int g2 = lane; g2 < nblk; g2 += 32)
                t2_merge(x, ap[(static_cast<std::size_t>(b) * nblk + g2) * d.maxdeg + e]);
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                T2 y;
                y.y1 = __shfl_xor_sync(0xffffffffu, x.y1, o);
                y.y2 = __shfl_xor_sync(0xffffffffu, x.y2, o);
                y.id1 = __shfl_xor_sync(0xffffffffu, x.id1, o);
                y.s1 = __shfl_xor_sync(0xffffffffu, x.s1, o);
                t2_merge(x, y);
              }
              if (lane == 0) {
                int ws = x.s1;
                const bool near = !(x.y1 - x.y2 > 1e-9 * fmax(1.0, fabs(x.y1)));
                if (near || V.force_slow) {
                  // exact: ascending agent id, sequential z2 (insertion sort, one thread)
                  if (!V.force_slow) atomicOr(&d.err[b], kErrNearTieSlow);
                  const int nA = V.acount[par * d.B + b];
                  unsigned long long* keys = V.sort_scratch + (static_cast<std::size_t>(b) * d.maxdeg + e) * N;
                  for (int q = 0; q < nA; ++q) {
                    const int s = V.alist[static_cast<std::size_t>(par) * d.B * N + bn + q];
                    const unsigned long long kk =
                        (static_cast<unsigned long long>(d.aid[so + s]) << 32) | static_cast<unsigned>(s);
                    int m = q - 1;
                    while (m >= 0 && keys[m] > kk) {
                      keys[m + 1] = keys[m];
                      --m;
                    }
                    keys[m + 1] = kk;
                  }
                  const double vv = 0.0 - kMaskLarge;
                  const double lzv = dlog(static_cast<double>(nA) * 1.0) + vv;
                  const double logz = vv - lzv;
                  double z2 = 0.0;
                  for (int q = 0; q < nA; ++q) {
                    const double g = gumbel(d.seed_merge[b], static_cast<std::uint64_t>(t),
                                            static_cast<std::uint64_t>(i), keys[q] >> 32);
                    z2 += dexp((logz + g) * d.kinv - x.y1);
                  }
                  double bp = -1.0;
                  for (int q = 0; q < nA; ++q) {
                    const double g = gumbel(d.seed_merge[b], static_cast<std::uint64_t>(t),
                                            static_cast<std::uint64_t>(i), keys[q] >> 32);
                    const double pv = dexp((logz + g) * d.kinv - x.y1) / z2;
                    if (pv > bp) {
                      bp = pv;
                      ws = static_cast<int>(keys[q] & 0xffffffffull);
                    }
                  }
                }
                const int j = d.lnk[so + ws];
                const int r = ws - offT[j];
                bool mover;
                const int ns = map_next(V, b, par, ws, j, r, offT, offN, &mover);
                double ab;
                if (mover) {
                  ab = 0.0 * d.M + 0.0;
                } else {
                  const double xb = xbn[ns];
                  ab = (i == j ? xb * d.M : 0.0 * d.M) + adm_bar(xb, V.x1[bn + ws], d.M);
                }
                V.lbar_a0[static_cast<std::size_t>(b) * d.maxdeg + e] = 0.0 + ab;
              }
            }
          }
          if (!routed && lane == 0) V.lbar_a0[static_cast<std::size_t>(b) * d.maxdeg + e] = 0.0;
        }
        } else {
        // position adjoint of layout t: kB3 slots per thread in flight; the
        // follower's headway term is the follower lane's own gap adjoint
        // (lanes are consecutive slots), so only a warp's last lane evaluates
        // its follower's x1 adjoint itself.
        const int t3 = tid - kM3T, n3 = kBT - kM3T;
        const int stride3 = nblk * n3;
        for (int k0 = lg * n3 + t3; k0 - lane < N && !(V.dbg & 256); k0 += kB3 * stride3) {
          int kk[kB3], jj[kB3], rr[kB3], nn[kB3];
          double xx[kB3], xp[kB3], xf[kB3];
#pragma unroll
          for (int q = 0; q < kB3; ++q) {
            const int k = k0 + q * stride3;
            const bool on = k < N;
            kk[q] = k;
            const int j = on ? d.lnk[so + k] : 0;
            jj[q] = j;
            const int base = offT[j];
            rr[q] = k - base;
            nn[q] = offT[j + 1] - base;
            xx[q] = on ? d.pos[so + k] : 0.0;
            xp[q] = (on && rr[q] > 0) ? d.pos[so + k - 1] : 0.0;
            xf[q] = (on && lane == 31 && rr[q] + 1 < nn[q]) ? d.pos[so + k + 1] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < kB3; ++q) {
            const int k = kk[q], j = jj[q], r = rr[q], n = nn[q];
            const bool on = k < N;
            double gapb = 0.0, xpb = 0.0, dxfb = 0.0, gnext = 0.0;
            if (on) {
              const double jam = d.jam[bl + j], dxf = d.dxf[bl + j], len = d.len[j];
              const double x = xx[q];
              const CfPick me = cf_step(x, r == 0 ? d.M : xp[q] - x, jam, dxf, len);
              const double x1b = x1_bar_p(V, b, par, k, j, r, me.x1, offT, offN, xbn);
              xpb = d.tg ? x1b : (me.cap ? x1b : 0.0);
              const double dxcb = me.cong ? xpb : 0.0;
              dxfb = me.cong ? 0.0 : xpb;
              gapb = me.gap >= 0.0 ? dxcb * 1.0 : 0.0;
              if (lane == 31 && r + 1 < n) {
                const CfPick fo = cf_step(xf[q], x - xf[q], jam, dxf, len);
                const double f1b = x1_bar_p(V, b, par, k + 1, j, r + 1, fo.x1, offT, offN, xbn);
                const double fpb = d.tg ? f1b : (fo.cap ? f1b : 0.0);
                const double fcb = fo.cong ? fpb : 0.0;
                gnext = fo.gap >= 0.0 ? fcb * 1.0 : 0.0;
              }
            }
            const double gdown = __shfl_down_sync(0xffffffffu, gapb, 1);
            if (lane < 31) gnext = gdown;
            if (on) {
              double tb = 0.0;
              if (r + 1 < n) tb += gnext * 1.0;
              if (r > 0) tb += -(gapb * 1.0);
              xbc[k] = xpb + tb * 1.0;
              V.cu[bn + k] = (dxfb * d.dt) * 1.0;
              V.cg[bn + k] = gapb;
            }
          }
        }
        }
      }
    bstamp(V, t, 5);
    grid_sync();
    bstamp(V, t, 6);
    bstamp(V, t, 7);  // R4 of this step runs with R1 of the next one
  }
  // R4 of step 0
  if (T > 0 && active)
    for (int b = b0; b < d.B; b += bstep) {
      __syncthreads();
      const int* og = d.off + oidx(d, 0, b);
      for (int j = tid; j <= L; j += kBT) offT[j] = og[j];
      __syncthreads();
      r4(b, 0, offT, tid, kBT);
    }
  grid_sync();
  // deferred preference gradient of step 0
  if (T > 0 && active)
    for (int b = b0; b < d.B; b += bstep) {
      __syncthreads();
      const int* og = d.off + oidx(d, 0, b);
      for (int j = tid; j <= L; j += kBT) offN[j] = og[j];
      __syncthreads();
      const std::size_t bn = static_cast<std::size_t>(b) * N, bl = static_cast<std::size_t>(b) * L;
      double* g5 = V.grads + static_cast<std::size_t>(b) * 5 * L;
      const int* nAn = V.nAb + bl;  // parity 0
      const double* vbn = V.vbar + bn * d.maxdeg;
      for (int i = lg * kBT + tid; i < L; i += nblk * kBT) {
        double pb = 0.0;
        for (int e = d.pred_off[i]; e < d.pred_off[i + 1]; ++e) {
          const int p = d.pred[e];
          const int pbse = offN[p];
          if (offN[p + 1] == pbse) continue;
          const int nap = nAn[p];
          for (int r = 0; r < nap; ++r)
            pb += vbn[static_cast<std::size_t>(pbse + r) * d.maxdeg + d.pred_pos[e]] * 1.0;
        }
        const double cst = d.cost[bl + i], be = d.beta[bl + i];
        g5[2 * L + i] += 0.0 + pb / cst;
        g5[4 * L + i] += 0.0 - pb * be / (cst * cst);
      }
    }
}

int backward_smem_bytes(int L, int maxdeg) {
  return (2 * (L + 1) + 2) * 4 + (kBT / 32) * maxdeg * static_cast<int>(sizeof(T2)) + 16 + (4 + 3 * kHeadCap) * 4;
}

int backward_threads() { return kBT; }

int backward_max_grid(int L, int maxdeg) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = backward_smem_bytes(L, maxdeg);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<void*>(k_backward_persistent),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<void*>(k_backward_persistent), kBT,
                                                smem);
  return occ * sms;
}

cudaError_t launch_backward_persistent(const BView& V, int grid, cudaStream_t st) {
  void* args[] = {const_cast<BView*>(&V)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_backward_persistent), dim3(grid), dim3(kBT),
                                     args, backward_smem_bytes(V.d.L, V.d.maxdeg), st);
}

}  // namespace dtg

namespace dtg {
cudaError_t decision_stats_backward(int force, unsigned long long* count) { return decision_stats_tu(force, count); }
}  // namespace dtg
