// Persistent cooperative forward kernel: all T engine steps of all B
// scenarios in ONE launch, two grid barriers per step.
//
// Step t (reference engine_step, src/engine.cpp:70-125):
//   phase S (slots)   every CTA rebuilds the segment offsets of layout t in
//                     shared memory (exclusive scan of n_j - dep_j + arr_j of
//                     step t-1), then each thread PULLS its slot of layout t
//                     from step t-1 (stable compaction + entrants at 0.0),
//                     writes the checkpoint, runs car-following against the
//                     pulled leader, writes the prefix-boundary counts, and an
//                     arrived head draws its next link and registers itself as
//                     a merge candidate of that link (atomic slot in a per-link
//                     list) — no predecessor walk later.
//   grid.sync
//   phase L (links)   count/cumulative update, vacancy, merge over the
//                     registered candidates (ascending id), departures.
//   grid.sync
// Same arithmetic as dtg_kernels.cu (bit-identical results), fewer dependent
// round trips: the separate compaction, scan and candidate-gather passes of
// the 4-kernel step are gone.
#include <cooperative_groups.h>

#include <climits>
#include <cstdint>

#include "dtg_device.cuh"
#include "dtg_kernels.h"
#include "dtg_persistent.h"

namespace cg = cooperative_groups;

namespace dtg {

__device__ __forceinline__ int find_link(const int* off_s, int L, int k) {
  // largest j with off_s[j] <= k (then off_s[j + 1] > k)
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

// Source slot in layout t-1 of new rank rn on link j (the transfer compaction
// of node_model.cpp:122-149 + replace_rows, read backwards).
__device__ __forceinline__ int pull_src(int j, int rn, const int* offA, const int* offB,
                                        const int* nAp, const int* depp, const int* win,
                                        const int* wonp, bool* entrant) {
  const int w = win[j];
  if (w >= 0 && rn == offB[j + 1] - offB[j] - 1) {
    *entrant = true;
    return w;
  }
  *entrant = false;
  const int ob = offA[j];
  const int na = offA[j + 1] > ob ? nAp[j] : 0;
  const int dp = depp[j];
  if (rn >= na - dp) return ob + rn + dp;
  int c = -1;
  for (int q = 0; q < na; ++q)
    if (!wonp[ob + q] && ++c == rn) return ob + q;
  return ob;  // unreachable for a consistent state
}

// Block-wide exclusive scan over n values held in shared memory `v` (in
// place), result v[i] = sum_{j<i}, v[n] = total.  `tmp` has >= 32 ints.
__device__ void block_scan_inplace(int* v, int n, int* tmp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int j0 = min(n, tid * per), j1 = min(n, j0 + per);
  int s = 0;
  for (int j = j0; j < j1; ++j) s += v[j];
  // inclusive warp scan of s
  const int lane = tid & 31, wid = tid >> 5;
  int x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < (nt >> 5) ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    tmp[lane] = w;
  }
  __syncthreads();
  int run = (wid ? tmp[wid - 1] : 0) + x - s;
  const int total = tmp[(nt >> 5) - 1];
  __syncthreads();
  for (int j = j0; j < j1; ++j) {
    const int c = v[j];
    v[j] = run;
    run += c;
  }
  if (tid == 0) v[n] = total;
  __syncthreads();
}

// Slot phase of step t for scenario b: layout t (pulled from t-1 unless t==0),
// checkpoint write, car-following + counts + choices + candidate registration.
// do_cf == false: only materialise layout t (the final layout T).
__device__ void slot_phase(const PView& P, int b, int t, int lg, int nblk, int* offA, int* offB,
                           int* tmp, bool do_cf) {
  const DevView& d = P.d;
  const int L = d.L, N = d.N;
  const std::size_t bl = static_cast<std::size_t>(b) * L;
  const std::size_t bn = static_cast<std::size_t>(b) * N;
  const int cur = t & 1, prv = cur ^ 1;
  const std::size_t so = sidx(d, t % d.S, b);
  __syncthreads();  // shared offsets of the previous scenario / step are dead
  // ---- offsets of layout t in shared memory ----
  if (t == 0) {
    const int* og = d.off + oidx(d, 0, b);
    for (int j = threadIdx.x; j <= L; j += blockDim.x) offB[j] = og[j];
    __syncthreads();
  } else {
    const int* og = d.off + oidx(d, (t - 1) % d.S, b);
    for (int j = threadIdx.x; j <= L; j += blockDim.x) offA[j] = og[j];
    __syncthreads();
    const int* depp = P.depb + static_cast<std::size_t>(prv) * d.B * L + bl;
    for (int j = threadIdx.x; j < L; j += blockDim.x)
      offB[j] = offA[j + 1] - offA[j] - depp[j] + (P.win[bl + j] >= 0 ? 1 : 0);
    __syncthreads();
    block_scan_inplace(offB, L, tmp);
    if (lg == 0) {
      int* on = d.off + oidx(d, t % d.S, b);
      for (int j = threadIdx.x; j <= L; j += blockDim.x) on[j] = offB[j];
      if (threadIdx.x == 0 && offB[L] != N) atomicOr(&d.err[b], kErrConservation);
    }
  }
  const int* nAp = P.nAb + static_cast<std::size_t>(prv) * d.B * L + bl;
  const int* depp = P.depb + static_cast<std::size_t>(prv) * d.B * L + bl;
  const int* winb = P.win + bl;
  const int* wonp = P.wonb + static_cast<std::size_t>(prv) * d.B * N + bn;
  const double* x1p = P.x1b + static_cast<std::size_t>(prv) * d.B * N + bn;
  const std::size_t sp = t > 0 ? sidx(d, (t - 1) % d.S, b) : 0;
  double* x1c = P.x1b + static_cast<std::size_t>(cur) * d.B * N + bn;
  int* wonc = P.wonb + static_cast<std::size_t>(cur) * d.B * N + bn;
  int* nAc = P.nAb + static_cast<std::size_t>(cur) * d.B * L + bl;
  int* qnc = P.qnb + static_cast<std::size_t>(cur) * d.B * L + bl;
  double* tailc = P.tailb + static_cast<std::size_t>(cur) * d.B * L + bl;

  for (int k = lg * blockDim.x + threadIdx.x; k < N; k += nblk * blockDim.x) {
    const int j = find_link(offB, L, k);
    const int base = offB[j], n = offB[j + 1] - base, r = k - base;
    double x, xl = 0.0, xn = 0.0;
    if (t == 0) {
      x = d.pos[so + k];
      if (r > 0) xl = d.pos[so + k - 1];
      if (r + 1 < n) xn = d.pos[so + k + 1];
    } else {
      bool ent;
      const int src = pull_src(j, r, offA, offB, nAp, depp, winb, wonp, &ent);
      x = ent ? 0.0 : x1p[src];
      const int a = d.aid[sp + src];
      d.pos[so + k] = x;
      d.aid[so + k] = a;
      d.lnk[so + k] = j;
      if (do_cf) {
        if (r > 0) {
          bool e2;
          const int s2 = pull_src(j, r - 1, offA, offB, nAp, depp, winb, wonp, &e2);
          xl = e2 ? 0.0 : x1p[s2];
        }
        if (r + 1 < n) {
          bool e3;
          const int s3 = pull_src(j, r + 1, offA, offB, nAp, depp, winb, wonp, &e3);
          xn = e3 ? 0.0 : x1p[s3];
        }
      }
    }
    if (!do_cf) continue;
    const std::size_t pl = bl + j;
    const double jam = d.jam[pl], dxf = d.dxf[pl], len = d.len[j];
    const double ctr = d.ctr[j], thr = d.thr[j];
    const CfPick me = cf_step(x, r == 0 ? d.M : xl - x, jam, dxf, len);
    x1c[k] = me.x1;
    bool fo_n = false, fa_n = false;
    if (r + 1 < n) {
      const CfPick nx = cf_step(xn, x - xn, jam, dxf, len);
      fo_n = nx.x1 >= ctr;
      fa_n = nx.x1 >= thr;
    }
    const bool fo = me.x1 >= ctr, fa = me.x1 >= thr;
    if (r == 0 && !fo) qnc[j] = 0;
    if (fo && !fo_n) qnc[j] = r + 1;
    if (r == 0 && !fa) nAc[j] = 0;
    if (fa && !fa_n) nAc[j] = r + 1;
    if (r == n - 1) tailc[j] = me.x1;
    if (fa) {
      wonc[k] = 0;
      const int s0 = d.succ_off[j], deg = d.succ_off[j + 1] - s0;
      int c = -1;
      if (deg > 0) {  // link_choice (node_model.cpp:45-97)
        double g[kMaxDeg], pi[kMaxDeg];
        const int agent = d.aid[so + k];
        const double* lz = d.slogz + (bl + j) * d.maxdeg;
        for (int e = 0; e < deg; ++e)
          g[e] = gumbel(d.seed_link[b], static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(agent),
                        static_cast<std::uint64_t>(d.succ[s0 + e]));
        c = d.succ[s0 + softmax_stage2<kMaxDeg>(deg, lz, g, d.kinv, pi)];
        const int q = atomicAdd(&P.ccnt[bl + c], 1);
        if (q < kCandCap) P.clist[(bl + c) * kCandCap + q] = k;
      }
      d.choice[bn + k] = c;
    }
  }
}

// Link phase of step t for scenario b (merge_choice, node_model.cpp:99-120).
__device__ void link_phase(const PView& P, int b, int t, int lg, int nblk) {
  const DevView& d = P.d;
  const int L = d.L;
  const std::size_t bl = static_cast<std::size_t>(b) * L;
  const int cur = t & 1;
  const std::size_t so = sidx(d, t % d.S, b);
  const int* off = d.off + oidx(d, t % d.S, b);
  const int* qnc = P.qnb + static_cast<std::size_t>(cur) * d.B * L + bl;
  const double* tailc = P.tailb + static_cast<std::size_t>(cur) * d.B * L + bl;
  int* depc = P.depb + static_cast<std::size_t>(cur) * d.B * L + bl;
  int* depn = P.depb + static_cast<std::size_t>(cur ^ 1) * d.B * L + bl;
  int* wonc = P.wonb + static_cast<std::size_t>(cur) * d.B * d.N + static_cast<std::size_t>(b) * d.N;
  for (int i = lg * blockDim.x + threadIdx.x; i < L; i += nblk * blockDim.x) {
    const int n_i = off[i + 1] - off[i];
    const int qc = n_i ? qnc[i] : 0;
    const double tx = n_i ? tailc[i] : d.M;
    const double a = static_cast<double>(qc) - d.qh[hidx(d, t, b) + i];
    d.cumh[hidx(d, t + 1, b) + i] = d.cumh[hidx(d, t, b) + i] + (a >= 0.0 ? a : 0.0);
    d.qh[hidx(d, t + 1, b) + i] = static_cast<double>(qc);
    const bool vacant = tx > d.jam[bl + i];
    d.vac[bl + i] = vacant;
    const int cnt = P.ccnt[bl + i];
    P.ccnt[bl + i] = 0;
    depn[i] = 0;  // departures of step t+1 start from zero
    int w = -1;
    if (vacant && cnt > 0) {
      if (cnt > kCandCap) {
        atomicOr(&d.err[b], kErrCandOverflow);
      } else {
        int cid[kCandCap], cslot[kCandCap], clink[kCandCap];
        for (int e = 0; e < cnt; ++e) {
          const int s = P.clist[(bl + i) * kCandCap + e];
          cid[e] = d.aid[so + s];
          cslot[e] = s;
          clink[e] = d.lnk[so + s];
        }
        for (int x = 1; x < cnt; ++x) {  // ascending agent id
          const int ci = cid[x], cs = cslot[x], cl = clink[x];
          int m = x - 1;
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
        double v[kCandCap], g[kCandCap], lz[kCandCap], pi[kCandCap];
        for (int e = 0; e < cnt; ++e) {
          v[e] = d.alpha[bl + clink[e]];
          if (v[e] == 0.0) atomicOr(&d.err[b], kErrZeroAlpha);
          g[e] = gumbel(d.seed_merge[b], static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(i),
                        static_cast<std::uint64_t>(cid[e]));
        }
        const int best = two_softmax<kCandCap>(cnt, v, g, d.kinv, lz, pi);
        w = cslot[best];
        wonc[w] = 1;
        atomicAdd(&depc[clink[best]], 1);
      }
    }
    P.win[bl + i] = w;
  }
}

// Phase timestamps (%globaltimer, ns) per step and CTA, when requested.
__device__ __forceinline__ void stamp(const PView& P, int t, int w) {
  if (P.tstamp == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    P.tstamp[(static_cast<std::size_t>(t) * gridDim.x + blockIdx.x) * 4 + w] = ns;
  }
}

__global__ void __launch_bounds__(512) k_forward_persistent(PView P) {
  extern __shared__ int smem[];
  cg::grid_group grid = cg::this_grid();
  const DevView& d = P.d;
  int* offA = smem;
  int* offB = smem + (d.L + 1);
  int* tmp = smem + 2 * (d.L + 1);
  const int G = gridDim.x;
  // scenario assignment: bps CTAs per scenario, or a loop over scenarios
  const bool grouped = P.bps > 0;
  const int b0 = grouped ? blockIdx.x / P.bps : blockIdx.x;
  const int lg = grouped ? blockIdx.x % P.bps : 0;
  const int nblk = grouped ? P.bps : 1;
  const int bstep = grouped ? d.B : G;  // loop stride over scenarios
  const bool active = grouped ? (b0 < d.B) : true;
  for (int t = 0; t < P.T; ++t) {
    stamp(P, t, 0);
    if (active)
      for (int b = b0; b < d.B; b += bstep) slot_phase(P, b, t, lg, nblk, offA, offB, tmp, true);
    stamp(P, t, 1);
    grid.sync();
    stamp(P, t, 2);
    if (active)
      for (int b = b0; b < d.B; b += bstep) link_phase(P, b, t, lg, nblk);
    stamp(P, t, 3);
    grid.sync();
  }
  if (P.T > 0 && active)
    for (int b = b0; b < d.B; b += bstep) slot_phase(P, b, P.T, lg, nblk, offA, offB, tmp, false);
}

int persistent_smem_bytes(int L) { return (2 * (L + 1) + 32) * static_cast<int>(sizeof(int)); }

cudaError_t launch_forward_persistent(const PView& P, int grid, cudaStream_t st) {
  void* args[] = {const_cast<PView*>(&P)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_forward_persistent), dim3(grid),
                                     dim3(512), args, persistent_smem_bytes(P.d.L), st);
}

int persistent_max_grid(int L, int* per_sm) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = persistent_smem_bytes(L);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<void*>(k_forward_persistent),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<void*>(k_forward_persistent), 512,
                                                smem);
  if (per_sm) *per_sm = occ;
  return occ * sms;
}

}  // namespace dtg
