// FD-validation engine on sm_100a; see dtg_probe.h.
//
// One CTA per probe runs all T steps.  A step follows engine_step
// (engine.cpp:70-125) on the compact state:
//   1. per-link agent lists in ascending agent id (engine.cpp:77-82) and the
//      stable descending position order (headways' argsort_desc,
//      car_following.cpp:96-126);
//   2. car-following per agent (car_following.cpp:128-157) with the traced
//      relu / min / graft of the surrogate (car_following.cpp:17-94);
//   3. midpoint counts (observation.cpp:9-20) — hard count, soft sigmoid sum
//      and the count graft — then inc / cum (engine.cpp:109-113);
//   4. node_step (node_model.cpp:151-181): arrived rows, vacancy, link choice
//      (node_model.cpp:45-97), merge choice (:99-120), transfer (:122-149);
//   5. thread 0 folds the step's decisions into the BranchTrace hash in the
//      reference's note order (branch_trace.hpp; note sites engine.cpp:95,112,
//      car_following.cpp:107,133,143-144,155, observation.cpp:15,
//      node_model.cpp:23,50,87-90,168).
// Every arithmetic step is the reference's tensor op on the same operands in
// the same order, so values are bit-identical (exp/log: libdevice, see
// DESIGN.md §2).  The hash is one sequential FNV chain per probe (it is a
// serial definition); everything else is spread over the CTA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>
#include <stdexcept>
#include <string>

#include "dtg_device.cuh"
#include "dtg_probe.h"

namespace dtg {
namespace {

constexpr int kPB = 256;  // threads per probe CTA

#define PCK(x)                                                                 \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess)                                                     \
      throw std::runtime_error(std::string("CUDA: ") + #x + ": " +             \
                               cudaGetErrorString(e_));                        \
  } while (0)

struct TraceDev {  // keyed surrogate records of one recording run
  double* xp0;     // [T][N] x' (graft old value of the length cap)
  unsigned char* pk;  // [T][N] bit0 relu pick, bit1 min pick, bit2 cap pick
  double* hard0;   // [T][L] hard count (count graft new value)
  double* soft0;   // [T][L] soft count (count graft old value)
  unsigned char* incpk;  // [T][L] relu pick of q - qprev
  double* xbar0;   // [T][N] transfer carrier / entry graft old value
  int* cnt0;       // [T][L] agents per link (control-path check)
  int* na0;        // [T] arrived agents (control-path check)
};

struct PV {
  int L, N, P, T, delta_n, tg, soft, sur, trace, keep_cum;
  double M, dt, kinv;
  const int *succ_off, *succ;
  const double* len;
  const double* params;  // [P][5][L]
  const std::uint64_t *seed_link, *seed_merge;  // [P]
  const int* lnk0;
  const double* pos0;
  // state / outputs [P][...]
  int* lnk;
  double* pos;
  double *qprev, *cum, *cum_hist;
  std::uint64_t* hash;
  int* flags;
  // scratch [P][...]
  int *cnt, *off, *cur, *seg_id, *seg_ord, *arr, *arl, *lch, *cand, *ncand, *mwin;
  double *x1, *q;
  unsigned char *ab, *vac, *incb;
  TraceDev tr;
};

__device__ __forceinline__ void fnv_bit(std::uint64_t& h, bool b) {
  h = (h ^ (b ? 0x9eULL : 0x7fULL)) * 0x100000001b3ULL;
}
__device__ __forceinline__ void fnv_u64(std::uint64_t& h, std::uint64_t v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    h = (h ^ (v & 0xffULL)) * 0x100000001b3ULL;
    v >>= 8;
  }
}

// First argmax of the second-stage softmax of a row whose utilities are all
// masked (-1e12): a link-choice row of an agent without successors, or a merge
// row nobody targets.  log_softmax over n equal entries, y = (logz + g) / tau_g,
// pi = softmax(y) (tensor.cpp:407-433), onehot_argmax_rows (tensor.cpp:660-670).
// Column c draws gumbel(seed, key, row, colkey(c)).
template <class ColKey>
__device__ int masked_row_argmax(std::uint64_t seed, std::uint64_t key, std::uint64_t row,
                                 int n, ColKey colkey, double kinv) {
  const double V = 0.0 - kMaskLarge;
  double z = 0.0;
  for (int c = 0; c < n; ++c) z += dexp(V - V);
  const double lz = dlog(z) + V;
  const double logz = V - lz;
  double m2 = 0.0;
  for (int c = 0; c < n; ++c) {
    const double y = (logz + gumbel(seed, key, row, colkey(c))) * kinv;
    if (c == 0 || m2 < y) m2 = y;
  }
  double z2 = 0.0;
  for (int c = 0; c < n; ++c) z2 += dexp((logz + gumbel(seed, key, row, colkey(c))) * kinv - m2);
  int best = 0;
  double bp = 0.0;
  for (int c = 0; c < n; ++c) {
    const double pi = dexp((logz + gumbel(seed, key, row, colkey(c))) * kinv - m2) / z2;
    if (c == 0 || pi > bp) {
      bp = pi;
      best = c;
    }
  }
  return best;
}

__global__ void __launch_bounds__(kPB) k_probe(PV v) {
  const int p = blockIdx.x, tid = threadIdx.x;
  const int L = v.L, N = v.N;
  const std::size_t pN = static_cast<std::size_t>(p) * N, pL = static_cast<std::size_t>(p) * L;
  int* lnk = v.lnk + pN;
  double* pos = v.pos + pN;
  double* qprev = v.qprev + pL;
  double* cum = v.cum + pL;
  int* cnt = v.cnt + pL;
  int* off = v.off + static_cast<std::size_t>(p) * (L + 1);
  int* cur = v.cur + pL;
  int* seg_id = v.seg_id + pN;
  int* seg_ord = v.seg_ord + pN;
  int* arr = v.arr + pN;
  int* arl = v.arl + pN;
  int* lch = v.lch + pN;
  int* cand = v.cand + pL * kProbeMaxCand;
  int* ncand = v.ncand + pL;
  int* mwin = v.mwin + pL;
  double* x1 = v.x1 + pN;
  double* q = v.q + pL;
  unsigned char* ab = v.ab + pN;
  unsigned char* vac = v.vac + pL;
  unsigned char* incb = v.incb + pL;
  const double* u = v.params + static_cast<std::size_t>(p) * 5 * L;
  const double* kap = u + L;
  const double* beta = u + 2 * L;
  const double* alpha = u + 3 * L;
  const double* cost = u + 4 * L;
  const std::uint64_t sl = v.seed_link[p], sm = v.seed_merge[p];
  const bool record = v.sur == 1 && p == 0, replay = v.sur == 2;
  const TraceDev& tr = v.tr;
  __shared__ int s_flags;
  __shared__ int s_na;

  // initial state and counts: initial_counts (engine.cpp:127-135) — hard
  // midpoint counts of X0, no trace
  if (tid == 0) s_flags = 0;
  for (int n = tid; n < N; n += kPB) {
    lnk[n] = v.lnk0[n];
    pos[n] = v.pos0[n];
  }
  for (int j = tid; j < L; j += kPB) cum[j] = 0.0;
  __syncthreads();
  for (int j = tid; j < L; j += kPB) {
    const double o = 0.5 * v.len[j];
    double c = 0.0;
    for (int n = 0; n < N; ++n)
      if (lnk[n] == j) c += (pos[n] >= o ? 1.0 : 0.0) * 1.0;
    qprev[j] = c;
  }
  std::uint64_t h = 0xcbf29ce484222325ULL;
  __syncthreads();

  for (int t = 0; t < v.T; ++t) {
    // ---- 1. per-link lists -------------------------------------------------
    for (int j = tid; j < L; j += kPB) cnt[j] = 0;
    __syncthreads();
    for (int n = tid; n < N; n += kPB)
      if (lnk[n] >= 0) atomicAdd(&cnt[lnk[n]], 1);
    __syncthreads();
    if (tid == 0) {
      int a = 0;
      for (int j = 0; j < L; ++j) {
        off[j] = a;
        cur[j] = a;
        a += cnt[j];
      }
      off[L] = a;
    }
    __syncthreads();
    for (int n = tid; n < N; n += kPB)
      if (lnk[n] >= 0) seg_id[atomicAdd(&cur[lnk[n]], 1)] = n;
    __syncthreads();
    for (int j = tid; j < L; j += kPB) {
      const int b = off[j], m = cnt[j];
      for (int k = 1; k < m; ++k) {  // ascending agent id
        const int x = seg_id[b + k];
        int i = k - 1;
        while (i >= 0 && seg_id[b + i] > x) {
          seg_id[b + i + 1] = seg_id[b + i];
          --i;
        }
        seg_id[b + i + 1] = x;
      }
      for (int k = 0; k < m; ++k) {  // stable argsort, descending position
        const double xk = pos[seg_id[b + k]];
        int i = k - 1;
        while (i >= 0 && pos[seg_id[b + seg_ord[b + i]]] < xk) {
          seg_ord[b + i + 1] = seg_ord[b + i];
          --i;
        }
        seg_ord[b + i + 1] = k;
      }
      if (record) tr.cnt0[static_cast<std::size_t>(t) * L + j] = m;
      else if (replay && tr.cnt0[static_cast<std::size_t>(t) * L + j] != m)
        atomicOr(&s_flags, kProbeOffPath);
    }
    __syncthreads();

    // ---- 2. car-following per agent (car_following_step) -------------------
    for (int s = tid; s < off[L]; s += kPB) {
      const int n = seg_id[s];
      const int j = lnk[n];
      const int b = off[j], r = s - b;
      const int me = seg_id[b + seg_ord[s]];
      const double x = pos[me];
      const double hw = r == 0 ? v.M : pos[seg_id[b + seg_ord[s - 1]]] - x;
      const double dxf = (1.0 * u[j]) * v.dt;
      const double jam = static_cast<double>(v.delta_n) / kap[j];
      const double gap = hw - jam;
      const double Lj = v.len[j];
      const std::size_t ti = static_cast<std::size_t>(t) * N + me;
      double dxc, dx, xp, limit, xo;
      if (replay) {
        const unsigned k = tr.pk[ti];
        const double a1 = (k & 1) ? 1.0 : 0.0, a2 = (k & 2) ? 1.0 : 0.0, a3 = (k & 4) ? 1.0 : 0.0;
        dxc = (gap * a1 + 0.0 * (1.0 - a1)) * 1.0;
        dx = dxc * a2 + dxf * (1.0 - a2);
        xp = x + dx;
        limit = v.tg ? (xp - tr.xp0[ti]) + Lj : Lj;
        xo = xp * a3 + limit * (1.0 - a3);
      } else {
        dxc = (gap >= 0.0 ? gap : 0.0) * 1.0;
        dx = dxc <= dxf ? dxc : dxf;
        xp = x + dx;
        limit = Lj;
        xo = xp <= limit ? xp : limit;
        if (record) {
          tr.pk[ti] = static_cast<unsigned char>((gap >= 0.0 ? 1 : 0) | (dxc <= dxf ? 2 : 0) |
                                                 (xp <= limit ? 4 : 0));
          tr.xp0[ti] = xp;
        }
      }
      x1[me] = xo;
      ab[me] = static_cast<unsigned char>((gap <= 0.0 ? 1 : 0) | (dxc <= dxf ? 2 : 0) |
                                          (xp <= limit ? 4 : 0) | (xo >= 0.5 * Lj ? 8 : 0));
    }
    __syncthreads();

    // ---- 3. counts, inc / cum, vacancy -------------------------------------
    for (int j = tid; j < L; j += kPB) {
      const int b = off[j], m = cnt[j];
      const double Lj = v.len[j], o = 0.5 * Lj, sc = 5.0 / Lj;
      double qj = 0.0;
      if (m > 0) {
        double hard = 0.0, soft = 0.0;
        for (int k = 0; k < m; ++k) hard += (x1[seg_id[b + k]] >= o ? 1.0 : 0.0) * 1.0;
        if (v.sur) {
          for (int k = 0; k < m; ++k) {
            const double z = (x1[seg_id[b + k]] + (-o)) * sc;
            const double sg = z >= 0.0 ? 1.0 / (1.0 + dexp(-z)) : dexp(z) / (1.0 + dexp(z));
            soft += sg * 1.0;
          }
        }
        const std::size_t tj = static_cast<std::size_t>(t) * L + j;
        if (record) {
          tr.hard0[tj] = hard;
          tr.soft0[tj] = soft;
        }
        qj = replay ? (soft - tr.soft0[tj]) + tr.hard0[tj] : hard;
      }
      const double a = qj - qprev[j];
      double inc;
      const std::size_t tj = static_cast<std::size_t>(t) * L + j;
      if (replay) {
        const double pa = tr.incpk[tj] ? 1.0 : 0.0;
        inc = a * pa + 0.0 * (1.0 - pa);
      } else {
        inc = a >= 0.0 ? a : 0.0;
        if (record) tr.incpk[tj] = a >= 0.0 ? 1 : 0;
      }
      cum[j] = cum[j] + inc;
      qprev[j] = qj;
      q[j] = qj;
      incb[j] = inc != 0.0;
      if (v.keep_cum) v.cum_hist[(static_cast<std::size_t>(p) * v.T + t) * L + j] = cum[j];
      double mn = v.M;
      for (int k = 0; k < m; ++k) {
        const double xx = x1[seg_id[b + k]];
        if (xx >= kValidThr && xx < mn) mn = xx;
      }
      vac[j] = mn > static_cast<double>(v.delta_n) / kap[j];
      ncand[j] = 0;
      mwin[j] = -1;
    }
    __syncthreads();

    // ---- 4a. arrived rows (node_step, node_model.cpp:159-167) --------------
    if (tid == 0) {
      int a = 0;
      for (int n = 0; n < N; ++n) {
        const int j = lnk[n];
        if (j >= 0 && x1[n] >= kValidThr && x1[n] >= v.len[j] - kArrivalTol) arr[a++] = n;
      }
      s_na = a;
      if (record) tr.na0[t] = a;
      else if (replay && tr.na0[t] != a) atomicOr(&s_flags, kProbeOffPath);
    }
    // X1: every agent on a link takes its car-following result
    for (int n = tid; n < N; n += kPB)
      if (lnk[n] >= 0) pos[n] = x1[n];
    __syncthreads();
    const int nA = s_na;

    // ---- 4b. link choice per arrived row (node_model.cpp:45-97) ------------
    for (int r = tid; r < nA; r += kPB) {
      const int n = arr[r], c = lnk[n];
      const int b0 = v.succ_off[c], deg = v.succ_off[c + 1] - b0;
      int hard_col = -1;
      arl[r] = c;
      if (record) tr.xbar0[static_cast<std::size_t>(t) * N + n] = x1[n];
      if (deg > kMaxDeg) {
        atomicOr(&s_flags, kProbeDegOverflow);
      } else if (deg > 0) {
        double V[kMaxDeg], g[kMaxDeg], logz[kMaxDeg], pi[kMaxDeg];
        for (int e = 0; e < deg; ++e) {
          const int jj = v.succ[b0 + e];
          V[e] = 1.0 * (beta[jj] / cost[jj]) - 0.0;
          g[e] = gumbel(sl, t, n, jj);
        }
        const int best = two_softmax<kMaxDeg>(deg, V, g, v.kinv, logz, pi);
        hard_col = v.succ[b0 + best];
        for (int e = 0; e < deg; ++e) {
          const int jj = v.succ[b0 + e];
          double l;
          if (v.soft) l = pi[e] * (vac[jj] ? 1.0 : 0.0);
          else l = (e == best ? 1.0 : 0.0) * (vac[jj] ? 1.0 : 0.0);
          if (l != 0.0 && l != 1.0) atomicOr(&s_flags, kProbeFractional);
          if (l == 1.0) {
            const int k = atomicAdd(&ncand[jj], 1);
            if (k < kProbeMaxCand) cand[static_cast<std::size_t>(jj) * kProbeMaxCand + k] = r;
            else atomicOr(&s_flags, kProbeCandOverflow);
          }
        }
      } else if (v.trace && !v.soft) {
        hard_col = masked_row_argmax(sl, t, n, L, [](int c2) { return c2; }, v.kinv);
      }
      lch[r] = hard_col;
    }
    __syncthreads();

    // ---- 4c. merge choice + transfer per link (node_model.cpp:99-149) ------
    for (int i = tid; i < L; i += kPB) {
      const int m = min(ncand[i], kProbeMaxCand);
      int* ci = cand + static_cast<std::size_t>(i) * kProbeMaxCand;
      if (m > 0) {
        for (int k = 1; k < m; ++k) {  // ascending arrived rank = ascending id
          const int x = ci[k];
          int e = k - 1;
          while (e >= 0 && ci[e] > x) {
            ci[e + 1] = ci[e];
            --e;
          }
          ci[e + 1] = x;
        }
        double V[kProbeMaxCand], g[kProbeMaxCand], logz[kProbeMaxCand], pi[kProbeMaxCand];
        for (int k = 0; k < m; ++k) {
          const int n = arr[ci[k]];
          const double prio = alpha[arl[ci[k]]];
          if (prio == 0.0) atomicOr(&s_flags, kProbeZeroAlpha);
          V[k] = 1.0 * prio - 0.0;
          g[k] = gumbel(sm, t, i, n);
        }
        const int w = two_softmax<kProbeMaxCand>(m, V, g, v.kinv, logz, pi);
        if (v.soft)
          for (int k = 0; k < m; ++k)
            if (pi[k] != 0.0 && pi[k] != 1.0) atomicOr(&s_flags, kProbeFractional);
        mwin[i] = ci[w];
        // transfer: the winner enters link i (node_model.cpp:131-148)
        const int n = arr[ci[w]];
        double entry = v.M;
        if (v.tg && replay) entry = (x1[n] - tr.xbar0[static_cast<std::size_t>(t) * N + n]) + v.M;
        const double np = ((-v.M) * 1.0 + 0.0 * (-v.M)) + 1.0 * entry;
        pos[n] = np;
        lnk[n] = np >= kValidThr ? i : -1;
      } else if (v.trace && !v.soft && nA > 0) {
        const int* ar = arr;
        mwin[i] = masked_row_argmax(sm, t, i, nA, [ar](int c2) { return ar[c2]; }, v.kinv);
      }
    }
    __syncthreads();

    // ---- 5. BranchTrace notes of this step ---------------------------------
    if (v.trace && tid == 0) {
      for (int j = 0; j < L; ++j) {
        const int b = off[j], m = cnt[j];
        if (m == 0) continue;
        for (int k = 0; k < m; ++k)
          fnv_u64(h, static_cast<std::uint64_t>(seg_id[b + k]) * L + j);  // engine.cpp:95
        for (int k = 0; k < m; ++k) fnv_bit(h, true);                      // valid, :133
        for (int r = 0; r < m; ++r) fnv_u64(h, static_cast<std::uint64_t>(seg_ord[b + r]));  // :107
        if (!v.sur) {
          for (int k = 0; k < m; ++k) fnv_bit(h, ab[seg_id[b + k]] & 1);  // gap <= 0, :143
          for (int k = 0; k < m; ++k) fnv_bit(h, ab[seg_id[b + k]] & 2);  // dx_cong <= dx_free, :144
          for (int k = 0; k < m; ++k) fnv_bit(h, ab[seg_id[b + k]] & 4);  // x' <= limit, :155
        }
        for (int k = 0; k < m; ++k) fnv_bit(h, ab[seg_id[b + k]] & 8);  // hard count, observation.cpp:15
      }
      if (!v.sur)
        for (int j = 0; j < L; ++j) fnv_bit(h, incb[j]);  // engine.cpp:112
      if (nA > 0) {
        for (int r = 0; r < nA; ++r) fnv_u64(h, static_cast<std::uint64_t>(arr[r]));  // node_model.cpp:168
        for (int r = 0; r < nA; ++r)  // valid pattern of X_sub, node_model.cpp:50
          for (int j = 0; j < L; ++j) fnv_bit(h, j == arl[r]);
        if (!v.soft)
          for (int r = 0; r < nA; ++r)
            for (int j = 0; j < L; ++j) fnv_bit(h, j == lch[r]);  // node_model.cpp:23
        for (int r = 0; r < nA; ++r) fnv_bit(h, true);  // arrived, :88
        for (int j = 0; j < L; ++j) fnv_bit(h, vac[j]);  // vacant, :89
        for (int r = 0; r < nA; ++r)  // connected, :90
          fnv_bit(h, v.succ_off[arl[r] + 1] > v.succ_off[arl[r]]);
        if (!v.soft)
          for (int i = 0; i < L; ++i)
            for (int r = 0; r < nA; ++r) fnv_bit(h, r == mwin[i]);  // node_model.cpp:23 (merge)
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    v.hash[p] = h;
    v.flags[p] = s_flags;
  }
}

// ---- host side -----------------------------------------------------------------
template <class T>
struct PBuf {
  T* p = nullptr;
  std::size_t n = 0;
  void alloc(std::size_t count) {
    release();
    if (count) PCK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~PBuf() { release(); }
};

struct TraceBlock {
  PBuf<double> xp0, hard0, soft0, xbar0;
  PBuf<unsigned char> pk, incpk;
  PBuf<int> cnt0, na0;
};

}  // namespace

ProbeTrace::~ProbeTrace() { delete static_cast<TraceBlock*>(dev); }

void ProbeTrace::reserve(int T_, int N_, int L_) {
  if (dev && T == T_ && N == N_ && L == L_) return;
  delete static_cast<TraceBlock*>(dev);
  dev = nullptr;
  auto* b = new TraceBlock;
  const std::size_t TN = static_cast<std::size_t>(std::max(T_, 1)) * N_,
                    TL = static_cast<std::size_t>(std::max(T_, 1)) * L_;
  try {
    b->xp0.alloc(TN);
    b->xbar0.alloc(TN);
    b->pk.alloc(TN);
    b->hard0.alloc(TL);
    b->soft0.alloc(TL);
    b->incpk.alloc(TL);
    b->cnt0.alloc(TL);
    b->na0.alloc(std::max(T_, 1));
  } catch (...) {
    delete b;
    throw;
  }
  dev = b;
  T = T_;
  N = N_;
  L = L_;
  recorded = false;
}

struct ProbeEngine::Impl {
  ProbeCfg cfg;
  PBuf<int> succ_off, succ, lnk0, lnk, cnt, off, cur, seg_id, seg_ord, arr, arl, lch, cand, ncand,
      mwin, flags;
  PBuf<double> len, pos0, params, pos, qprev, cum, cum_hist, x1, q;
  PBuf<unsigned char> ab, vac, incb;
  PBuf<std::uint64_t> seeds, hash;
  cudaStream_t st = nullptr;
};

ProbeEngine::ProbeEngine(const ProbeNet& net, const ProbeCfg& cfg, int n_agents, int n_probes)
    : d_(new Impl), L_(net.L), N_(n_agents), P_(n_probes) {
  try {
    if (L_ < 1 || N_ < 0 || P_ < 1) throw std::runtime_error("probe engine: empty network or no probes");
    if (static_cast<int>(net.succ_off.size()) != L_ + 1 || static_cast<int>(net.len.size()) != L_)
      throw std::runtime_error("probe engine: network arrays do not match n_links");
    d_->cfg = cfg;
    const std::size_t L = L_, N = std::max(N_, 1), P = P_;
    PCK(cudaStreamCreateWithFlags(&d_->st, cudaStreamNonBlocking));
    d_->succ_off.alloc(L + 1);
    d_->succ.alloc(std::max<std::size_t>(net.succ.size(), 1));
    d_->len.alloc(L);
    PCK(cudaMemcpy(d_->succ_off.p, net.succ_off.data(), (L + 1) * 4, cudaMemcpyHostToDevice));
    if (!net.succ.empty())
      PCK(cudaMemcpy(d_->succ.p, net.succ.data(), net.succ.size() * 4, cudaMemcpyHostToDevice));
    PCK(cudaMemcpy(d_->len.p, net.len.data(), L * 8, cudaMemcpyHostToDevice));
    d_->lnk0.alloc(N);
    d_->pos0.alloc(N);
    d_->params.alloc(P * 5 * L);
    d_->seeds.alloc(2 * P);
    d_->hash.alloc(P);
    d_->flags.alloc(P);
    for (auto* b : {&d_->lnk, &d_->seg_id, &d_->seg_ord, &d_->arr, &d_->arl, &d_->lch}) b->alloc(P * N);
    for (auto* b : {&d_->cnt, &d_->cur, &d_->ncand, &d_->mwin}) b->alloc(P * L);
    d_->off.alloc(P * (L + 1));
    d_->cand.alloc(P * L * kProbeMaxCand);
    d_->pos.alloc(P * N);
    d_->x1.alloc(P * N);
    d_->qprev.alloc(P * L);
    d_->cum.alloc(P * L);
    d_->q.alloc(P * L);
    d_->ab.alloc(P * N);
    d_->vac.alloc(P * L);
    d_->incb.alloc(P * L);
  } catch (...) {
    if (d_->st) cudaStreamDestroy(d_->st);
    delete d_;
    throw;
  }
}

ProbeEngine::~ProbeEngine() {
  if (d_->st) cudaStreamDestroy(d_->st);
  delete d_;
}

void ProbeEngine::set_state(const int* link, const double* pos) {
  for (int n = 0; n < N_; ++n) {
    if (link[n] < 0 || link[n] >= L_) throw std::runtime_error("agent placed on a link that does not exist");
    if (!(pos[n] >= kValidThr))
      throw std::runtime_error("initial position below the validity threshold (-0.01)");
  }
  if (N_) {
    PCK(cudaMemcpy(d_->lnk0.p, link, N_ * 4, cudaMemcpyHostToDevice));
    PCK(cudaMemcpy(d_->pos0.p, pos, N_ * 8, cudaMemcpyHostToDevice));
  }
}

void ProbeEngine::set_params(const double* params) {
  PCK(cudaMemcpy(d_->params.p, params, static_cast<std::size_t>(P_) * 5 * L_ * 8, cudaMemcpyHostToDevice));
}

void ProbeEngine::set_noise(std::uint64_t root_seed, const std::uint64_t* its) {
  std::vector<std::uint64_t> s(2 * P_);
  for (int p = 0; p < P_; ++p) {
    const std::uint64_t sim = rng_fork(rng_fork(root_seed, lane::kIteration), its[p]);  // engine.cpp:49
    s[p] = rng_fork(sim, lane::kGumbelLink);
    s[P_ + p] = rng_fork(sim, lane::kGumbelMerge);
  }
  PCK(cudaMemcpy(d_->seeds.p, s.data(), s.size() * 8, cudaMemcpyHostToDevice));
}

void ProbeEngine::run(int T, int sur_mode, ProbeTrace* tr, bool trace, bool keep_cum) {
  if (T < 0) throw std::runtime_error("negative horizon");
  if (sur_mode && !tr) throw std::runtime_error("surrogate mode without a trace");
  if (sur_mode == 2 && (!tr->recorded || tr->T < T || tr->N != N_ || tr->L != L_))
    throw std::runtime_error("surrogate replay: the trace holds no matching recording");
  if (sur_mode == 1) tr->reserve(T, N_, L_);
  T_ = T;
  if (keep_cum && d_->cum_hist.n < static_cast<std::size_t>(P_) * std::max(T, 1) * L_)
    d_->cum_hist.alloc(static_cast<std::size_t>(P_) * std::max(T, 1) * L_);
  PV v{};
  v.L = L_;
  v.N = N_;
  v.P = P_;
  v.T = T;
  v.delta_n = d_->cfg.delta_n;
  v.tg = d_->cfg.tg;
  v.soft = d_->cfg.soft;
  v.sur = sur_mode;
  v.trace = trace;
  v.keep_cum = keep_cum;
  v.M = d_->cfg.M;
  v.dt = d_->cfg.tau * d_->cfg.delta_n;
  v.kinv = 1.0 / d_->cfg.gumbel_tau;
  v.succ_off = d_->succ_off.p;
  v.succ = d_->succ.p;
  v.len = d_->len.p;
  v.params = d_->params.p;
  v.seed_link = d_->seeds.p;
  v.seed_merge = d_->seeds.p + P_;
  v.lnk0 = d_->lnk0.p;
  v.pos0 = d_->pos0.p;
  v.lnk = d_->lnk.p;
  v.pos = d_->pos.p;
  v.qprev = d_->qprev.p;
  v.cum = d_->cum.p;
  v.cum_hist = d_->cum_hist.p;
  v.hash = d_->hash.p;
  v.flags = d_->flags.p;
  v.cnt = d_->cnt.p;
  v.off = d_->off.p;
  v.cur = d_->cur.p;
  v.seg_id = d_->seg_id.p;
  v.seg_ord = d_->seg_ord.p;
  v.arr = d_->arr.p;
  v.arl = d_->arl.p;
  v.lch = d_->lch.p;
  v.cand = d_->cand.p;
  v.ncand = d_->ncand.p;
  v.mwin = d_->mwin.p;
  v.x1 = d_->x1.p;
  v.q = d_->q.p;
  v.ab = d_->ab.p;
  v.vac = d_->vac.p;
  v.incb = d_->incb.p;
  if (sur_mode) {
    auto* b = static_cast<TraceBlock*>(tr->dev);
    v.tr = TraceDev{b->xp0.p, b->pk.p, b->hard0.p, b->soft0.p, b->incpk.p, b->xbar0.p, b->cnt0.p, b->na0.p};
  }
  k_probe<<<P_, kPB, 0, d_->st>>>(v);
  PCK(cudaGetLastError());
  PCK(cudaStreamSynchronize(d_->st));
  if (sur_mode == 1) tr->recorded = true;
}

std::vector<double> ProbeEngine::cum_per_step(int p) const {
  std::vector<double> out(static_cast<std::size_t>(T_) * L_);
  if (!out.empty()) {
    if (!d_->cum_hist.p) throw std::runtime_error("probe run did not keep the count history");
    PCK(cudaMemcpy(out.data(), d_->cum_hist.p + static_cast<std::size_t>(p) * T_ * L_, out.size() * 8,
                   cudaMemcpyDeviceToHost));
  }
  return out;
}

std::vector<double> ProbeEngine::cum_final_all() const {
  std::vector<double> out(static_cast<std::size_t>(P_) * L_);
  PCK(cudaMemcpy(out.data(), d_->cum.p, out.size() * 8, cudaMemcpyDeviceToHost));
  return out;
}

void ProbeEngine::final_state(int p, int* link, double* pos) const {
  if (!N_) return;
  PCK(cudaMemcpy(link, d_->lnk.p + static_cast<std::size_t>(p) * N_, N_ * 4, cudaMemcpyDeviceToHost));
  PCK(cudaMemcpy(pos, d_->pos.p + static_cast<std::size_t>(p) * N_, N_ * 8, cudaMemcpyDeviceToHost));
}

std::vector<std::uint64_t> ProbeEngine::hashes() const {
  std::vector<std::uint64_t> out(P_);
  PCK(cudaMemcpy(out.data(), d_->hash.p, P_ * 8, cudaMemcpyDeviceToHost));
  return out;
}

std::vector<int> ProbeEngine::flags() const {
  std::vector<int> out(P_);
  PCK(cudaMemcpy(out.data(), d_->flags.p, P_ * 4, cudaMemcpyDeviceToHost));
  return out;
}

std::string ProbeEngine::describe(int f) {
  std::string s;
  auto add = [&](int bit, const char* what) {
    if (f & bit) s += std::string(s.empty() ? "" : "; ") + what;
  };
  add(kProbeFractional,
      "a relaxed choice left {0, 1} (the state would become fractional; the device path "
      "supports soft choices where every choice row is one-hot, e.g. chains)");
  add(kProbeZeroAlpha, "merge candidate with zero merge priority alpha");
  add(kProbeCandOverflow, "more than 32 merge candidates for one link in one step");
  add(kProbeDegOverflow, "link out-degree above 16");
  add(kProbeOffPath, "surrogate replay left the recorded control path (surrogate trace misaligned)");
  return s;
}

}  // namespace dtg
