// Per-link precomputation shared by every forward schedule.
#include <algorithm>
#include <cstdint>

#include "dtg_cluster.h"
#include "dtg_device.cuh"

namespace dtg {

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

void launch_pack_succ(const DevView& d, double* srec, cudaStream_t st) {
  k_pack_succ<<<dim3((d.L + 127) / 128, d.B), 128, 0, st>>>(d, srec);
}

// Everything the persistent forward needs before its first step, in ONE launch
// (instead of 2 kernels + 5 copies + 6 memsets): per-link constants (k_derive's
// operations), the link-choice first stage (k_pack_succ's, with the successors'
// beta / cost recomputed — the same division), the initial layout copy and the
// zeroed counters.
__global__ void k_forward_init(ForwardInit a) {
  const DevView& d = a.d;
  const std::size_t gid = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
  const std::size_t gst = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  const std::size_t BN = static_cast<std::size_t>(d.B) * d.N, BL = static_cast<std::size_t>(d.B) * d.L;
  const std::size_t BO = static_cast<std::size_t>(d.B) * (d.L + 1);
  for (std::size_t i = gid; i < BN; i += gst) {
    a.pos[i] = a.pos0[i];
    a.aid[i] = a.aid0[i];
    a.lnk[i] = a.lnk0[i];
  }
  for (std::size_t i = gid; i < BO; i += gst) a.off[i] = a.off0[i];
  for (std::size_t i = gid; i < BL; i += gst) {
    a.qh[i] = a.q0[i];
    a.cumh[i] = 0.0;
    a.ccnt[i] = 0;
    a.depb[i] = 0;
    a.depb[BL + i] = 0;
    a.jam[i] = static_cast<double>(d.delta_n) / d.kappa[i];  // divide(scalar(dn), kappa)
    a.dxf[i] = (1.0 * d.u[i]) * d.dt;                        // scale(mul(valid, u), dt)
    a.pref[i] = d.beta[i] / d.cost[i];                       // divide(beta, cost)
    const int j = static_cast<int>(i % d.L);
    const std::size_t bl = i - j;
    const int s0 = d.succ_off[j], deg = d.succ_off[j + 1] - s0;
    if (deg > 0) {
      double v[kMaxDeg];
      for (int e = 0; e < deg; ++e) {
        const std::size_t sj = bl + d.succ[s0 + e];
        v[e] = d.beta[sj] / d.cost[sj];
      }
      log_softmax_stage1(deg, v, a.srec + i * d.maxdeg);
    }
  }
  for (std::size_t i = gid; i < static_cast<std::size_t>(d.B); i += gst) a.errf[i] = 0;
  if (gid == 0) *a.gbar = 0u;
}

void launch_forward_init(const ForwardInit& a, cudaStream_t st) {
  const std::size_t n = std::max(static_cast<std::size_t>(a.d.B) * a.d.N, static_cast<std::size_t>(a.d.B) * (a.d.L + 1));
  const int grid = static_cast<int>(std::min<std::size_t>((n + 255) / 256, 148 * 8));
  k_forward_init<<<grid, 256, 0, st>>>(a);
}

}  // namespace dtg
