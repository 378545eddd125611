// Scenario-resident forward (schedule 4): ONE CTA per scenario runs all T
// engine steps (reference engine_step, src/engine.cpp:70-125), its phases
// separated by CTA barriers only.  Scenarios never wait on each other -- the
// step graph ends every phase at a kernel boundary of the whole batch, the
// fused kernel at a grid barrier -- so an SM's second resident scenario fills
// the first one's serial draw / merge chains.
//
// The scenario's per-link step state lives in shared memory for the whole run
// (layout offsets of the current and next step, arrived-prefix lengths,
// winners, next-slot bases, the lists of links with work), and each step makes
// ONE pass over the agent slots:
//   1 links    thread per link: car-following of the head run (arrived
//              prefix), a binary search for the midpoint-count boundary (x1 is
//              non-increasing along a segment), the tail; count/cumulative
//              update and vacancy; lists the links with arrived heads
//   2 choice   the link choice of those heads only; lists the links chosen
//   3 merge    the merge decision of the chosen links only
//   4 scan     departures, next segment sizes and offsets, next-slot bases
//   5 slots    per slot: car-following and the move into the next layout
// Same arithmetic as the step graph (dtg_step.cuh bodies, cf_step, the draw
// and decision rules): bit-identical results and history layout.
#include <climits>
#include <cstdint>

#include "dtg_device.cuh"
#include "dtg_kernels.h"
#include "dtg_step.cuh"

namespace dtg {
namespace {

#ifndef DTG_SCN_THREADS
#define DTG_SCN_THREADS 384
#endif
constexpr int kScnThreads = DTG_SCN_THREADS;

__device__ __forceinline__ void scn_stamp(unsigned long long* st, int T, int t, int ph) {
  if (st != nullptr && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    st[((static_cast<std::size_t>(blockIdx.x) * T + t) << 3) + ph] = g;
  }
}

// x1 of slot base + r (its leader is the previous slot; the head gets M)
__device__ __forceinline__ double x1_at(const DevView& d, const double* pos, int base, int r, double jam,
                                        double dxf, double len) {
  const double x = pos[base + r];
  return cf_step(x, r == 0 ? d.M : pos[base + r - 1] - x, jam, dxf, len).x1;
}

// Phase 1 for link j.  Returns the arrived-prefix length; sets *vacant.
__device__ __forceinline__ int scn_link(const DevView& d, int b, int t, const double* pos, const int* off,
                                        int j, bool* vacant) {
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const int base = off[j], n = off[j + 1] - base;
  const double jam = d.jam[bl + j];
  int na = 0, qc = 0;
  double tx = d.M;
  if (n) {
    const double dxf = d.dxf[bl + j], len = d.len[j], ctr = d.ctr[j], thr = d.thr[j];
    // arrived prefix {x1 >= L - 0.01}
    double x1 = x1_at(d, pos, base, 0, jam, dxf, len);
    while (x1 >= thr) {
      d.won[bn + base + na] = 0;
      if (++na == n) break;
      x1 = x1_at(d, pos, base, na, jam, dxf, len);
    }
    // midpoint count {x1 >= 0.5 L} (a prefix containing the arrived one)
    if (na == n) {
      qc = n;
    } else if (x1 < ctr) {
      qc = na;
    } else {
      int lo = na + 1, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (x1_at(d, pos, base, mid, jam, dxf, len) >= ctr)
          lo = mid + 1;
        else
          hi = mid;
      }
      qc = lo;
    }
    tx = x1_at(d, pos, base, n - 1, jam, dxf, len);  // min x1 = vacancy (node_model.cpp:27-41)
  }
  // inc = relu(q - qprev); cum += inc (engine.cpp:111-113), as step_merge_counts
  const double a = static_cast<double>(qc) - d.qh[hidx(d, t, b) + j];
  d.cumh[hidx(d, t + 1, b) + j] = d.cumh[hidx(d, t, b) + j] + (a >= 0.0 ? a : 0.0);
  d.qh[hidx(d, t + 1, b) + j] = static_cast<double>(qc);
  *vacant = tx > jam;
  return na;
}

// Phase 5 for slot k (link j at row r of layout s_cur) -> layout s_next.
__device__ __forceinline__ void scn_move(const DevView& d, std::size_t bn, std::size_t bl, std::size_t sn, int k,
                                         int j, int id, double x, double xm, const int* off, const int* offn,
                                         const int* nA, const int* sh, const int* msl) {
  const int base = off[j], r = k - base;
  const double x1 = cf_step(x, r == 0 ? d.M : xm - x, d.jam[bl + j], d.dxf[bl + j], d.len[j]).x1;
  int ns, lk = j;
  double xo = x1;
  if (r < nA[j]) {  // arrived: the winner moves, the others shift past earlier winners
    if (d.won[bn + k]) {
      lk = d.choice[bn + k];
      ns = msl[lk];
      xo = 0.0;  // transfer (node_model.cpp:122-149): -M + M == 0.0 exactly on the new link
    } else {
      int dd = 0;
      for (int q = base; q < k; ++q) dd += d.won[bn + q];
      ns = offn[j] + r - dd;
    }
  } else {
    ns = sh[j] + r;
  }
  d.pos[sn + ns] = xo;
  d.aid[sn + ns] = id;
  d.lnk[sn + ns] = lk;
}

// A merge row with more than kFastSucc candidates (rare): local arrays, out
// of line so the common path keeps its candidates in registers.
__device__ __noinline__ void scn_merge_wide(const DevView& d, int b, int t, int i, const int* off, const int* nA,
                                            std::size_t so, int* w, int* wa, int* wl) {
  int cid[kMaxCand], cslot[kMaxCand], clink[kMaxCand];
  const int nc = gather_candidates(d, b, i, off, nA, so, cid, cslot, clink);
  if (nc) {
    double lz[kMaxCand], pi[kMaxCand];
    const int best = merge_softmax(d, b, t, i, nc, cid, clink, lz, pi, false);
    *w = cslot[best];
    *wa = cid[best];
    *wl = clink[best];
  }
}

#ifndef DTG_SCN_WIDE
#define DTG_SCN_WIDE 768
#endif
constexpr int kScnWide = DTG_SCN_WIDE;  // threads of the one-scenario-per-SM CTA

// kT threads per CTA, kM CTAs per SM: 384 x 2 when the batch fills the SMs
// twice over, 768 x 1 (twice the threads per scenario) when each scenario has
// an SM to itself
template <int kT, int kM>
__global__ void __launch_bounds__(kT, kM) k_forward_scn(DevView d, int T, unsigned long long* stamps) {
  constexpr int kScnThreads = kT;
  __shared__ int sm[32];
  __shared__ unsigned long long smin[32];
  __shared__ int cnt[3];  // [0] links with arrived heads, [1] chosen links, [2] most heads on a link (stamps)
  extern __shared__ int scn_smem[];
  const int L = d.L, W = (L + 31) >> 5;
  int* offs[2] = {scn_smem, scn_smem + (L + 1)};
  int* nA = scn_smem + 2 * (L + 1);
  int* win = nA + L;
  int* sh = win + L;
  int* msl = sh + L;
  unsigned* tbits = reinterpret_cast<unsigned*>(msl + L);
  unsigned* vbits = tbits + W;
  unsigned short* act = reinterpret_cast<unsigned short*>(vbits + W);
  unsigned short* tlist = act + L;

  const int b = d.b0 + blockIdx.x;
  const int tid = threadIdx.x;
  const std::size_t bn = static_cast<std::size_t>(b) * d.N;
  const std::size_t bl = static_cast<std::size_t>(b) * L;
#ifdef DTG_NO_SLOT_VEC
  const bool vec = false;
#else
  const bool vec = (d.N & 1) == 0;
#endif
  {
    const int* off0 = d.off + oidx(d, 0, b);
    for (int j = tid; j <= L; j += kScnThreads) offs[0][j] = off0[j];
    for (int w = tid; w < W; w += kScnThreads) tbits[w] = 0;
    if (tid == 0) cnt[0] = cnt[1] = cnt[2] = 0;
  }
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    const int sc = t % d.S, sn = (t + 1) % d.S;
    const int* off = offs[t & 1];
    int* offn = offs[(t & 1) ^ 1];
    const std::size_t so = sidx(d, sc, b), snx = sidx(d, sn, b);
    const double* pos = d.pos + so;
    scn_stamp(stamps, T, t, 0);
    // ---- 1: per link
    for (int j = tid; j < L; j += kScnThreads) {
      bool vacant;
      const int na = scn_link(d, b, t, pos, off, j, &vacant);
      nA[j] = na;
      win[j] = -1;
      sh[j] = 0;  // departures, counted by the merge phase
      const unsigned m = 1u << (j & 31);
      if (vacant)
        atomicOr(&vbits[j >> 5], m);
      else
        atomicAnd(&vbits[j >> 5], ~m);
      if (d.ev) d.ev[(static_cast<std::size_t>(t) * d.B + b) * L + j] = -1;
      if (na) {
        act[atomicAdd(&cnt[0], 1)] = static_cast<unsigned short>(j);
        if (stamps != nullptr) atomicMax(&cnt[2], na);
      }
    }
    __syncthreads();
    scn_stamp(stamps, T, t, 1);
    // ---- 2: link choice of the arrived heads
    {
      const int nact = cnt[0];
      for (int q = tid; q < nact; q += kScnThreads) {
        const int j = act[q];
        choose_heads(d, b, t, sc, j, off[j], nA[j], [&](int c) {
          const unsigned m = 1u << (c & 31);
          if (!(atomicOr(&tbits[c >> 5], m) & m)) tlist[atomicAdd(&cnt[1], 1)] = static_cast<unsigned short>(c);
        });
      }
    }
    __syncthreads();
    scn_stamp(stamps, T, t, 2);
    if (stamps != nullptr && tid == 0) {  // measurement: work-list sizes of this step
      stamps[((static_cast<std::size_t>(blockIdx.x) * T + t) << 3) + 6] =
          (static_cast<unsigned long long>(cnt[0]) << 32) | static_cast<unsigned>(cnt[2]);
      stamps[((static_cast<std::size_t>(blockIdx.x) * T + t) << 3) + 7] = cnt[1];
    }
    if (tid == 0) cnt[0] = 0;  // next read after phase 1 of t + 1
    const int ntg = cnt[1];
    // ---- 3: merge decisions of the chosen links
    for (int q = tid; q < ntg; q += kScnThreads) {
      const int i = tlist[q];
      if (!((vbits[i >> 5] >> (i & 31)) & 1u)) continue;
      int cid[kFastSucc], cslot[kFastSucc], clink[kFastSucc];
      const int nc = gather_candidates_fast(d, b, i, off, nA, so, cid, cslot, clink);
      int w = -1, wa = -1, wl = 0;
      if (nc > 0) {
        const int best = merge_softmax_fast(d, b, t, i, nc, cid, clink);
#pragma unroll
        for (int e = 0; e < kFastSucc; ++e)
          if (e == best) {
            w = cslot[e];
            wa = cid[e];
            wl = clink[e];
          }
      } else if (nc < 0) {
        scn_merge_wide(d, b, t, i, off, nA, so, &w, &wa, &wl);
      }
      if (w >= 0) {
        win[i] = w;
        atomicAdd(&sh[wl], 1);
        d.won[bn + w] = 1;
        if (d.ev) d.ev[(static_cast<std::size_t>(t) * d.B + b) * L + i] = wa;
      }
    }
    __syncthreads();
    scn_stamp(stamps, T, t, 3);
    // ---- 4: departures, next sizes, exclusive scan, next-slot bases
    for (int q = tid; q < ntg; q += kScnThreads) {
      const int i = tlist[q];
      tbits[i >> 5] = 0;  // whole words: every bit set in them belongs to a listed link
    }
    if (tid == 0) cnt[1] = 0;
    {
      const int per = (L + kScnThreads - 1) / kScnThreads;
      const int j0 = min(L, tid * per), j1 = min(L, j0 + per);
      int sum = 0;
      for (int j = j0; j < j1; ++j) {
        const int n = off[j + 1] - off[j], dep = sh[j];  // sh: departures until the offsets are known
        const int nc = n - dep + (win[j] >= 0 ? 1 : 0);
        msl[j] = nc;
        sum += nc;
      }
      int total;
      int run = block_excl_scan(sum, sm, &total);
      int* offg = d.off + oidx(d, sn, b);
      for (int j = j0; j < j1; ++j) {
        const int dep = sh[j], nc = msl[j];
        offn[j] = run;
        offg[j] = run;
        sh[j] = run - dep;      // non-arrived slots: ns = offn + r - dep
        msl[j] = run + nc - 1;  // the entrant takes the link's last slot
        run += nc;
      }
      if (tid == 0) {
        offn[L] = total;
        offg[L] = total;
        if (total != d.N) atomicOr(&d.err[b], kErrConservation);
      }
    }
    __syncthreads();
    scn_stamp(stamps, T, t, 4);
    // ---- 5: car-following and compaction into the next layout; the next
    // pair's layout loads are issued before this pair is moved
    if (vec) {
      int k = 2 * tid;
      int2 j2 = make_int2(0, 0), i2 = make_int2(0, 0);
      double2 x2 = make_double2(0.0, 0.0);
      double xm = 0.0;
      if (k < d.N) {
        j2 = *reinterpret_cast<const int2*>(d.lnk + so + k);
        x2 = *reinterpret_cast<const double2*>(pos + k);
        i2 = *reinterpret_cast<const int2*>(d.aid + so + k);
        xm = pos[k > 0 ? k - 1 : 0];
      }
      while (k < d.N) {
        const int kn = k + 2 * kScnThreads;
        int2 j2n = j2, i2n = i2;
        double2 x2n = x2;
        double xmn = xm;
        if (kn < d.N) {
          j2n = *reinterpret_cast<const int2*>(d.lnk + so + kn);
          x2n = *reinterpret_cast<const double2*>(pos + kn);
          i2n = *reinterpret_cast<const int2*>(d.aid + so + kn);
          xmn = pos[kn - 1];
        }
        scn_move(d, bn, bl, snx, k, j2.x, i2.x, x2.x, xm, off, offn, nA, sh, msl);
        scn_move(d, bn, bl, snx, k + 1, j2.y, i2.y, x2.y, x2.x, off, offn, nA, sh, msl);
        k = kn;
        j2 = j2n;
        i2 = i2n;
        x2 = x2n;
        xm = xmn;
      }
    } else {
      for (int k = tid; k < d.N; k += kScnThreads)
        scn_move(d, bn, bl, snx, k, d.lnk[so + k], d.aid[so + k], pos[k], pos[k > 0 ? k - 1 : 0], off, offn, nA,
                 sh, msl);
    }
    __syncthreads();
    scn_stamp(stamps, T, t, 5);
  }
}

}  // namespace

std::size_t forward_scn_smem(int L) {
  const std::size_t W = (static_cast<std::size_t>(L) + 31) / 32;
  return (2 * (static_cast<std::size_t>(L) + 1) + 4 * static_cast<std::size_t>(L) + 2 * W) * 4 +
         2 * static_cast<std::size_t>(L) * 2;
}

bool forward_scn_ok(int L) {
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return false;
  return L < 65536 && forward_scn_smem(L) + 1024 <= static_cast<std::size_t>(optin);
}

cudaError_t launch_forward_scn(const DevView& d, int T, unsigned long long* stamps, cudaStream_t st) {
  const std::size_t sm = forward_scn_smem(d.L);
  const int nb = d.nb ? d.nb : d.B;
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  if (nb <= sms) {  // one scenario per SM: the wide CTA
    e = cudaFuncSetAttribute(k_forward_scn<kScnWide, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    k_forward_scn<kScnWide, 1><<<nb, kScnWide, sm, st>>>(d, T, stamps);
  } else {
    e = cudaFuncSetAttribute(k_forward_scn<kScnThreads, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    k_forward_scn<kScnThreads, 2><<<nb, kScnThreads, sm, st>>>(d, T, stamps);
  }
  return cudaGetLastError();
}

cudaError_t decision_stats_scn(int force, unsigned long long* count) { return decision_stats_tu(force, count); }

}  // namespace dtg
