// Fused forward kernel (dtg_fused.cu): shared types and launchers.
#pragma once
#include <cuda_runtime.h>

#include "dtg_device.cuh"

namespace dtg {

constexpr int kClusterThreads = 512;
constexpr int kClusterCandCap = 16;

// A merge column registered by an arrived head: its merge utility alpha of its
// current link, its own merge Gumbel g'(t, row, id), slot, id and link.
struct Cand {
  double alpha;
  double g;
  int slot;
  int aid;
  int link;
  int pad;
};

// A head decision drawn one step ahead (link choice c and own merge noise g of
// agent aid at the next step; aid -1: none).  Both depend only on (seed, step,
// agent, link), never on the state, so a precomputed record is exact.
struct Spec {
  int aid;
  int c;
  double g;
};

struct CView {
  DevView d;
  double* x1b;    // [2][B][N]
  int* wonb;      // [2][B][N]
  int* nAb;       // [2][B][L]
  int* qnb;       // [2][B][L]
  double* tailb;  // [2][B][L]
  int* depb;      // [2][B][L]
  int* win;       // [B][L]
  int* ccnt;      // [B][L]
  Cand* cands;    // [B][L][kClusterCandCap]
  const double* srec;  // [B][L][maxdeg] successor preferences
  int T;
  int cs;              // CTAs per cluster = per scenario
  int stage_params;    // per-link constants in shared memory
  unsigned long long* tstamp;  // optional [T][grid][4]
  unsigned int* gbar;  // grid-barrier counter (null: cooperative_groups grid.sync)
  unsigned long long* wstamp;  // optional per-warp slot-phase record [T][warps][4]
  int contig;          // 1: contiguous slot range per CTA, 0: interleaved 512-slot blocks
  int ckpt;            // keep every layout (else positions/links of the final one only)
  int dbg;             // timing experiments only (dtg_set_flag 3); results invalid when nonzero
  // optional host-mapped step counter: after the barrier that completes step
  // t-1 (every count of steps < t final), CTA 0 publishes t at system scope so
  // the host can copy finished count rows while the kernel runs (grid mode)
  volatile unsigned int* progress;
  int progress_every;  // publish only when t is a multiple (chunk ends) or T
  // optional [2][B][L][2]: during step t's link phase the otherwise idle
  // threads draw step t+1's decisions of every link's first two agents (the
  // only agents that can be its arrived head at t+1); the slot phase of t+1
  // then only registers them (null: heads draw in the slot phase)
  Spec* spec;
  // 1: the speculative draws run in warps 2.. of each CTA between arriving at
  // and waiting on barrier 1 (needs every link's merge thread in warps 0-1,
  // i.e. 64 cs >= L; one slot per thread; grid schedule)
  int spec_split;
  int lean;  // fused_lean(L): the per-link shared-memory arrays are read from global memory
};

void launch_pack_succ(const DevView& d, double* srec, cudaStream_t st);

// Pre-step state of the persistent forward (k_forward_init, dtg_cluster.cu).
struct ForwardInit {
  DevView d;
  double *jam, *dxf, *pref, *srec;
  double* pos;
  const double* pos0;
  int* aid;
  const int* aid0;
  int* lnk;
  const int* lnk0;
  int* off;
  const int* off0;
  double* qh;
  const double* q0;
  double* cumh;
  int *errf, *ccnt, *depb;
  unsigned int* gbar;
};
void launch_forward_init(const ForwardInit& a, cudaStream_t st);
int fused_smem_bytes(int L, bool stage_params);
bool fused_lean(int L);  // per-link arrays in global memory (large networks)
int fused_max_grid(int L, bool stage_params);
int fused_max_cluster(int L, bool stage_params);
cudaError_t launch_forward_fused(const CView& V, bool cluster, cudaStream_t st);

}  // namespace dtg
