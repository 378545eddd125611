// Per-link precomputation shared by every forward schedule.
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

}  // namespace dtg
