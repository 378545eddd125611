// Persistent cooperative reverse sweep (dtg_backward.cu).
#pragma once
#include <cuda_runtime.h>

#include "dtg_cluster.h"
#include "dtg_device.cuh"

namespace dtg {

constexpr int kBwdCandCap = 16;

struct BView {
  DevView d;
  // replay of step t
  double* x1;            // [B][N]
  int* nAb;              // [2][B][L] arrived-prefix length, parity of t
  int* nA_cur;           // [B][L]    same, current step
  double* tail;          // [B][L]
  int* won;              // [B][N]
  int* dep;              // [B][L]
  int* win;              // [B][L]
  unsigned char* vac;    // [B][L]
  int* ccnt;             // [2][B][L] per step parity
  Cand* cands;           // [B][L][kBwdCandCap]
  double* mpi;           // [B][L][kBwdCandCap]
  double* mlz;           // [B][L][kBwdCandCap]
  double* lpi;           // [2][B][N][maxdeg] link-choice logits of arrived heads, per step parity
  int* ched;             // [2][B][N] index of the chosen successor, per step parity
  int* choice;           // [2][B][N] per step parity
  int* alist;            // [2][B][N] per step parity
  int* acount;           // [2][B]
  unsigned long long* a0key;  // [2][B]
  void* a0part;          // [B][bps][maxdeg] per-CTA top-2 partials
  // adjoint
  double* xbar;          // [2][B][N]
  double* cbar;          // [B][L]
  double* qbar;          // [B][L]
  double* qtot;          // [B][L]
  double* lbar_row;      // [B][N]
  double* prio_bar;      // [B][N]
  double* lbar_a0;       // [B][maxdeg]
  double* vbar;          // [2][B][N][maxdeg]
  double* cu;            // [B][N]
  double* cg;            // [B][N]
  double* grads;         // [B][5][L]
  const double* snap_seed;  // [B][K][L]
  const double* cum_seed;   // [B][L]
  const double* x_seed;     // [B][N]
  unsigned long long* sort_scratch;  // [B][maxdeg][N]
  int K, spi, T, bps, force_slow;
  int dbg;  // timing experiments only (dtg_set_flag 2): bits skip parts of R1
  unsigned long long* tstamp;  // optional [T][grid][8] phase timestamps
  unsigned int* gbar;          // grid-barrier counter (zeroed before launch; null: cooperative_groups)
};

int backward_smem_bytes(int L, int maxdeg);
int backward_threads();  // threads per CTA of k_backward_persistent
int backward_max_grid(int L, int maxdeg);
cudaError_t launch_backward_persistent(const BView& V, int grid, cudaStream_t st);

}  // namespace dtg
