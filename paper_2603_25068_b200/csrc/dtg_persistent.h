// Shared view of the persistent cooperative forward kernel (dtg_persistent.cu).
#pragma once
#include <cuda_runtime.h>

#include "dtg_device.cuh"

namespace dtg {

constexpr int kCandCap = 16;

struct PView {
  DevView d;
  double* x1b;    // [2][B][N]  x1 of layout t, ping-pong on t
  int* wonb;      // [2][B][N]  merge winners of layout t
  int* nAb;       // [2][B][L]  arrived-prefix length
  int* qnb;       // [2][B][L]  midpoint count
  double* tailb;  // [2][B][L]  tail x1 (vacancy)
  int* depb;      // [2][B][L]  departures (atomics)
  int* win;       // [B][L]     winner slot of row i (layout t), -1 none
  int* ccnt;      // [B][L]     registered candidates
  int* clist;     // [B][L][kCandCap] candidate slots
  int T;
  int bps;        // CTAs per scenario (B <= grid) ; 0 => scenario loop
  unsigned long long* tstamp;  // optional [T][grid][4] phase timestamps
};

cudaError_t launch_forward_persistent(const PView& P, int grid, cudaStream_t st);

}  // namespace dtg
