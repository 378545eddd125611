// Register-resident merge choice for a link with few candidates.
//
// merge_choice (node_model.cpp:99-120): candidates of row i in ascending agent
// id, utility alpha of each candidate's link, the two-stage Gumbel softmax of
// two_softmax (dtg_device.cuh) and the first argmax.  For cnt <= F (F = the
// largest in-degree the fast path serves) every loop below is unrolled with
// compile-time indices and predicated on `e < cnt`, so the candidates, logits
// and probabilities stay in registers; the floating-point operations and their
// order are exactly two_softmax's, so the results are bit-identical to the
// local-memory path it replaces.
#pragma once

#include "dtg_cluster.h"
#include "dtg_device.cuh"

namespace dtg {

/// Loads cnt <= F candidates, sorts them by agent id (distinct ids: any
/// correct sort gives the reference's ascending order), runs two_softmax and
/// returns the first argmax.  lz / pi receive the first-stage log-softmax and
/// the probabilities of the sorted candidates.
template <int F, bool kNeedPi = true>
__device__ __forceinline__ int merge_softmax_fast(int cnt, const Cand* src, double kinv, Cand (&c)[F],
                                                  double (&lz)[F], double (&pi)[F]) {
#pragma unroll
  for (int e = 0; e < F; ++e) {
    if (e < cnt) {
      c[e] = src[e];
    } else {
      c[e].alpha = 0.0;
      c[e].g = 0.0;
      c[e].slot = -1;
      c[e].aid = 0x7fffffff;  // sorts last
      c[e].link = -1;
      c[e].pad = 0;
    }
  }
  // odd-even transposition sort on static indices (F rounds)
#pragma unroll
  for (int r = 0; r < F; ++r) {
#pragma unroll
    for (int e = (r & 1); e + 1 < F; e += 2) {
      if (c[e].aid > c[e + 1].aid) {
        const Cand tmp = c[e];
        c[e] = c[e + 1];
        c[e + 1] = tmp;
      }
    }
  }
  if (!kNeedPi) {
    // Winner only: y_e = ((alpha_e - lz) + g_e) * k differs from the exact
    // (alpha_e + g_e - lz) * k by three roundings, under 2^-52 k (|alpha_e - lz|
    // + |g_e| + |alpha_e - lz + g_e|) < 3e-11 for |alpha|, |g| < 64 and k <=
    // 100.  When the two largest alpha_e + g_e are more than kGap apart the
    // rounded argmax is the exact one and the first stage is not needed;
    // closer calls take the full computation below.
    constexpr double kGap = 1e-9;
    int best = 0;
    double v1 = c[0].alpha + c[0].g, v2 = -INFINITY;
    bool small = fabs(c[0].alpha) < 64.0 && fabs(c[0].g) < 64.0;
#pragma unroll
    for (int e = 1; e < F; ++e)
      if (e < cnt) {
        const double v = c[e].alpha + c[e].g;
        small = small && fabs(c[e].alpha) < 64.0 && fabs(c[e].g) < 64.0;
        if (v > v1) {
          v2 = v1;
          v1 = v;
          best = e;
        } else if (v > v2) {
          v2 = v;
        }
      }
    if (!g_force_exact && small && kinv <= 100.0 && (cnt == 1 || (v1 - v2) * kinv > kGap)) return best;
    if (!g_force_exact) atomicAdd(&g_exact_decisions, 1ULL);
  }
  double m = c[0].alpha;
#pragma unroll
  for (int e = 1; e < F; ++e)
    if (e < cnt && m < c[e].alpha) m = c[e].alpha;
  double z = 0.0;
#pragma unroll
  for (int e = 0; e < F; ++e)
    if (e < cnt) z += dexp(c[e].alpha - m);
  const double lzz = dlog(z) + m;
  double y[F];
#pragma unroll
  for (int e = 0; e < F; ++e) {
    lz[e] = c[e].alpha - lzz;
    y[e] = (lz[e] + c[e].g) * kinv;
  }
  if (!kNeedPi) {  // the forward needs the winner only
    double ex[F];
    return softmax_first_argmax<F>(cnt, y, ex);
  }
  double m2 = y[0];
#pragma unroll
  for (int e = 1; e < F; ++e)
    if (e < cnt && m2 < y[e]) m2 = y[e];
  double ex[F];
  double z2 = 0.0;
#pragma unroll
  for (int e = 0; e < F; ++e) {
    ex[e] = dexp(y[e] - m2);
    if (e < cnt) z2 += ex[e];
  }
  int best = 0;
  double pb = 0.0;
#pragma unroll
  for (int e = 0; e < F; ++e) {
    pi[e] = ex[e] / z2;
    if (e == 0) {
      pb = pi[0];
    } else if (e < cnt && pi[e] > pb) {
      pb = pi[e];
      best = e;
    }
  }
  return best;
}

/// c[best] without a dynamic register-array index.
template <int F>
__device__ __forceinline__ Cand pick_cand(const Cand (&c)[F], int best) {
  Cand r = c[0];
#pragma unroll
  for (int e = 1; e < F; ++e)
    if (e == best) r = c[e];
  return r;
}

}  // namespace dtg
