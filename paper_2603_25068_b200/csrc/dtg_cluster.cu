// Forward engine as ONE thread-block cluster per scenario.
//
// Scenarios (noise draws) are independent, so a scenario only needs its own
// CTAs to agree on a step boundary: a cluster of `cs` CTAs (<= 16) owns one
// scenario for all T steps and synchronises with hardware cluster barriers
// (barrier.cluster arrive.release / wait.acquire, ~0.2 us) instead of
// grid-wide barriers; independent clusters never wait for each other and
// simply run in waves when B * cs exceeds the resident CTAs.
//
// Per step t (engine_step, src/engine.cpp:70-125):
//   slot phase   each CTA rebuilds layout t's segment offsets in shared
//                memory from its own copy of layout t-1's offsets (kept in
//                smem across steps) and step t-1's departures / entrants, then
//                every thread pulls its slots of layout t from step t-1 (stable
//                compaction, entrants at 0.0), writes the checkpoint, runs
//                car-following, writes the prefix-boundary counts; an arrived
//                head draws its next link (successor preferences pre-packed
//                per link), draws ITS OWN merge Gumbel for that link and
//                registers {alpha, g, slot, id, link} in the link's candidate
//                list with one atomic.
//   cluster barrier
//   link phase   count/cum update, vacancy, merge softmax over the registered
//                records sorted by id, departures.
//   cluster barrier
// Per-link constants (jam spacing, free-flow advance, length) live in shared
// memory for the whole run (the barriers' acquire invalidates L1).
#include <cooperative_groups.h>

#include <climits>
#include <cstdint>

#include "dtg_cluster.h"
#include "dtg_device.cuh"

namespace cg = cooperative_groups;

namespace dtg {

namespace {

__device__ __forceinline__ int find_link_s(const int* off_s, int L, int k) {
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

// Source slot in layout t-1 of new rank rn on link j (transfer compaction of
// node_model.cpp:122-149 + replace_rows, read backwards); smem-resident
// per-link state, the won flags of the arrived prefix in global memory.
__device__ __forceinline__ int pull_src_s(int j, int rn, const int* offA, const int* offB,
                                          const int* na_s, const int* dep_s, const int* win_s,
                                          const int* wonp, bool* entrant) {
  const int w = win_s[j];
  if (w >= 0 && rn == offB[j + 1] - offB[j] - 1) {
    *entrant = true;
    return w;
  }
  *entrant = false;
  const int ob = offA[j];
  const int na = na_s[j];
  const int dp = dep_s[j];
  if (rn >= na - dp) return ob + rn + dp;
  int c = -1;
  for (int q = 0; q < na; ++q)
    if (!wonp[ob + q] && ++c == rn) return ob + q;
  return ob;
}

__device__ void cta_scan(int* v, int n, int* tmp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int j0 = min(n, tid * per), j1 = min(n, j0 + per);
  int s = 0;
  for (int j = j0; j < j1; ++j) s += v[j];
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

__device__ __forceinline__ void cstamp(const CView& V, int t, int w) {
  if (V.tstamp == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    V.tstamp[(static_cast<std::size_t>(t) * gridDim.x + blockIdx.x) * 4 + w] = ns;
  }
}

struct Smem {
  int *offA, *offB, *na_s, *dep_s, *win_s, *tmp;
  double *jam_s, *dxf_s, *len_s;
};

}  // namespace

__global__ void __launch_bounds__(kClusterThreads) k_forward_cluster(CView V) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const DevView& d = V.d;
  const int L = d.L, N = d.N;
  const int rank = static_cast<int>(cluster.block_rank());
  const int b = blockIdx.x / V.cs;
  const int nthr = V.cs * blockDim.x;
  const int gt0 = rank * blockDim.x + threadIdx.x;  // thread index within the scenario
  Smem S;
  {
    double* dp = reinterpret_cast<double*>(sm_raw);
    if (V.stage_params) {
      S.jam_s = dp;
      S.dxf_s = dp + L;
      S.len_s = dp + 2 * L;
      dp += 3 * L;
    }
    int* ip = reinterpret_cast<int*>(dp);
    S.offA = ip;
    S.offB = ip + (L + 1);
    S.na_s = ip + 2 * (L + 1);
    S.dep_s = S.na_s + L;
    S.win_s = S.dep_s + L;
    S.tmp = S.win_s + L;
  }
  const std::size_t bl = static_cast<std::size_t>(b) * L;
  const std::size_t bn = static_cast<std::size_t>(b) * N;
  const std::size_t BL = static_cast<std::size_t>(d.B) * L;
  const std::size_t BN = static_cast<std::size_t>(d.B) * N;
  if (V.stage_params)
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
      S.jam_s[j] = d.jam[bl + j];
      S.dxf_s[j] = d.dxf[bl + j];
      S.len_s[j] = d.len[j];
    }
  {
    const int* og = d.off + oidx(d, 0, b);
    for (int j = threadIdx.x; j <= L; j += blockDim.x) S.offB[j] = og[j];
  }
  __syncthreads();
  const std::uint64_t seed_link = d.seed_link[b], seed_merge = d.seed_merge[b];
  const double* srec = d.slogz + bl * d.maxdeg;

  for (int t = 0; t <= V.T; ++t) {
    const bool last = t == V.T;  // materialise layout T only
    const int cur = t & 1, prv = cur ^ 1;
    if (!last) cstamp(V, t, 0);
    // ---------------- slot phase ----------------
    if (t > 0) {
      int* sw = S.offA;  // layout t-1 offsets := previous offB
      S.offA = S.offB;
      S.offB = sw;
      const int* nAp = V.nAb + prv * BL + bl;
      const int* depp = V.depb + prv * BL + bl;
      for (int j = threadIdx.x; j < L; j += blockDim.x) {
        const int nold = S.offA[j + 1] - S.offA[j];
        const int na = nold ? nAp[j] : 0;
        const int dp = depp[j];
        const int w = V.win[bl + j];
        S.na_s[j] = na;
        S.dep_s[j] = dp;
        S.win_s[j] = w;
        S.offB[j] = nold - dp + (w >= 0 ? 1 : 0);
      }
      __syncthreads();
      cta_scan(S.offB, L, S.tmp);
      if (rank == 0) {
        int* on = d.off + oidx(d, t % d.S, b);
        for (int j = threadIdx.x; j <= L; j += blockDim.x) on[j] = S.offB[j];
        if (threadIdx.x == 0 && S.offB[L] != N) atomicOr(&d.err[b], kErrConservation);
      }
    }
    const std::size_t so = sidx(d, t % d.S, b);
    const std::size_t sp = t > 0 ? sidx(d, (t - 1) % d.S, b) : 0;
    const double* x1p = V.x1b + prv * BN + bn;
    const int* wonp = V.wonb + prv * BN + bn;
    double* x1c = V.x1b + cur * BN + bn;
    int* wonc = V.wonb + cur * BN + bn;
    int* nAc = V.nAb + cur * BL + bl;
    int* qnc = V.qnb + cur * BL + bl;
    double* tailc = V.tailb + cur * BL + bl;
    for (int k = gt0; k < N; k += nthr) {
      const int j = find_link_s(S.offB, L, k);
      const int base = S.offB[j], n = S.offB[j + 1] - base, r = k - base;
      double x, xl = 0.0, xn = 0.0;
      int a;
      if (t == 0) {
        x = d.pos[so + k];
        a = d.aid[so + k];
        if (r > 0) xl = d.pos[so + k - 1];
        if (r + 1 < n) xn = d.pos[so + k + 1];
      } else {
        bool e0, e1 = false, e2 = false;
        const int s0 = pull_src_s(j, r, S.offA, S.offB, S.na_s, S.dep_s, S.win_s, wonp, &e0);
        int s1 = s0, s2 = s0;
        if (!last && r > 0) s1 = pull_src_s(j, r - 1, S.offA, S.offB, S.na_s, S.dep_s, S.win_s, wonp, &e1);
        if (!last && r + 1 < n) s2 = pull_src_s(j, r + 1, S.offA, S.offB, S.na_s, S.dep_s, S.win_s, wonp, &e2);
        const double v0 = x1p[s0], v1 = x1p[s1], v2 = x1p[s2];
        a = d.aid[sp + s0];
        x = e0 ? 0.0 : v0;  // entrant: -M + M == 0.0 exactly
        xl = e1 ? 0.0 : v1;
        xn = e2 ? 0.0 : v2;
        d.pos[so + k] = x;
        d.aid[so + k] = a;
        d.lnk[so + k] = j;
      }
      if (last) continue;
      const double jam = V.stage_params ? S.jam_s[j] : d.jam[bl + j];
      const double dxf = V.stage_params ? S.dxf_s[j] : d.dxf[bl + j];
      const double len = V.stage_params ? S.len_s[j] : d.len[j];
      const double ctr = 0.5 * len, thr = len - kArrivalTol;
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
        if (deg > 0) {  // link_choice (node_model.cpp:45-97)
          double g[kMaxDeg], pi[kMaxDeg];
          const double* lz = srec + static_cast<std::size_t>(j) * d.maxdeg;
          for (int e = 0; e < deg; ++e)
            g[e] = gumbel(seed_link, static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(a),
                          static_cast<std::uint64_t>(d.succ[s0 + e]));
          const int c = d.succ[s0 + softmax_stage2<kMaxDeg>(deg, lz, g, d.kinv, pi)];
          // this head is a merge column of row c: its own Gumbel g'(t, c, id)
          Cand cd;
          cd.alpha = d.alpha[bl + j];
          cd.g = gumbel(seed_merge, static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(c),
                        static_cast<std::uint64_t>(a));
          cd.slot = k;
          cd.aid = a;
          cd.link = j;
          cd.pad = 0;
          const int q = atomicAdd(&V.ccnt[bl + c], 1);
          if (q < kClusterCandCap) V.cands[(bl + c) * kClusterCandCap + q] = cd;
        }
      }
    }
    if (last) break;
    cstamp(V, t, 1);
    cluster.sync();
    cstamp(V, t, 2);
    // ---------------- link phase ----------------
    {
      int* depc = V.depb + cur * BL + bl;
      int* depn = V.depb + prv * BL + bl;
      const double* qhp = d.qh + hidx(d, t, b);
      const double* chp = d.cumh + hidx(d, t, b);
      double* qhn = d.qh + hidx(d, t + 1, b);
      double* chn = d.cumh + hidx(d, t + 1, b);
      for (int i = gt0; i < L; i += nthr) {
        const int n_i = S.offB[i + 1] - S.offB[i];
        const int cnt = V.ccnt[bl + i];
        const int qc = n_i ? qnc[i] : 0;
        const double tx = n_i ? tailc[i] : d.M;
        const double a = static_cast<double>(qc) - qhp[i];  // inc = relu(q - qprev)
        chn[i] = chp[i] + (a >= 0.0 ? a : 0.0);
        qhn[i] = static_cast<double>(qc);
        const double jam = V.stage_params ? S.jam_s[i] : d.jam[bl + i];
        const bool vacant = tx > jam;  // vacancy_from_state (node_model.cpp:27-41)
        V.ccnt[bl + i] = 0;
        depn[i] = 0;
        int w = -1;
        if (vacant && cnt > 0) {
          if (cnt > kClusterCandCap) {
            atomicOr(&d.err[b], kErrCandOverflow);
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
              if (v[e] == 0.0) atomicOr(&d.err[b], kErrZeroAlpha);
            }
            const int best = two_softmax<kClusterCandCap>(cnt, v, g, d.kinv, lz, pi);
            w = c[best].slot;
            wonc[w] = 1;
            atomicAdd(&depc[c[best].link], 1);
          }
        }
        V.win[bl + i] = w;
      }
    }
    cstamp(V, t, 3);
    cluster.sync();
  }
}

// Link-choice first stage per link: srec[b][j][e] = log_softmax over the
// successors' beta/cost (identical for every agent on link j, so computed
// once per run; node_model.cpp:55-63, tensor.cpp:407-433).
__global__ void k_pack_succ(DevView d, double* srec) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.L) return;
  const std::size_t bl = static_cast<std::size_t>(b) * d.L;
  const int s0 = d.succ_off[j], deg = d.succ_off[j + 1] - s0;
  if (deg == 0) return;
  double v[kMaxDeg];
  for (int e = 0; e < deg; ++e) v[e] = d.pref[bl + d.succ[s0 + e]];
  log_softmax_stage1(deg, v, srec + (bl + j) * d.maxdeg);
}

int cluster_smem_bytes(int L, bool stage_params) {
  return (stage_params ? 3 * L * 8 : 0) + (2 * (L + 1) + 3 * L + 32) * 4;
}

void launch_pack_succ(const DevView& d, double* srec, cudaStream_t st) {
  k_pack_succ<<<dim3((d.L + 127) / 128, d.B), 128, 0, st>>>(d, srec);
}

cudaError_t launch_forward_cluster(const CView& V, cudaStream_t st) {
  const int smem = cluster_smem_bytes(V.d.L, V.stage_params != 0);
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(k_forward_cluster),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (V.cs > 8) {
    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(k_forward_cluster),
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
  return cudaLaunchKernelEx(&cfg, k_forward_cluster, V);
}

// Largest cluster size (<= 16) that can be resident for this smem footprint.
int cluster_max_size(int L, bool stage_params) {
  const int smem = cluster_smem_bytes(L, stage_params);
  if (cudaFuncSetAttribute(reinterpret_cast<const void*>(k_forward_cluster),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return 0;
  cudaFuncSetAttribute(reinterpret_cast<const void*>(k_forward_cluster),
                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
    if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(k_forward_cluster), &cfg) ==
            cudaSuccess &&
        n > 0)
      return cs;
  }
  cudaGetLastError();
  return 0;
}

}  // namespace dtg
