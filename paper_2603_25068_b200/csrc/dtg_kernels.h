// Host-side launch wrappers of dtg_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include "dtg_device.cuh"

namespace dtg {

// scenario-resident forward: one CTA per scenario runs all T steps
// scenario-resident forward (dtg_scn.cu): one CTA per scenario runs all T
// steps; forward_scn_ok: the per-link shared-memory state fits this device
std::size_t forward_scn_smem(int L);
bool forward_scn_ok(int L);
cudaError_t launch_forward_scn(const DevView& d, int T, unsigned long long* stamps, cudaStream_t st);
void launch_step_forward(const DevView& d, int t, int s_cur, int s_next,
                         cudaStream_t st);
void launch_step_backward(const DevView& d, int t, int s_cur, int s_next,
                          const double* xbar_next, double* xbar_cur,
                          const double* snap_seed, int snap_k, int K,
                          unsigned long long* sort_scratch, int force_slow,
                          cudaStream_t st);
void launch_adj_init(const DevView& d, int s_fin, const double* x_seed,
                     double* xbar, const double* cum_seed, cudaStream_t st);
void launch_gather_state(const DevView& d, int s, int* link_out, double* pos_out,
                         cudaStream_t st);
void launch_derive(const DevView& d, double* jam, double* dxf, double* pref,
                   cudaStream_t st);

void launch_gumbel_batch(std::uint64_t seed, std::uint64_t key, const std::uint64_t* rows,
                         const std::uint64_t* cols, int n, double* out, cudaStream_t st);


constexpr int kFwdKernels = 5;
constexpr int kBwdKernels = 9;
constexpr int kLaunchesPerForwardStep = kFwdKernels;
constexpr int kLaunchesPerBackwardStep = kBwdKernels;
extern const char* const kFwdKernelNames[kFwdKernels];
extern const char* const kBwdKernelNames[kBwdKernels];
void launch_fwd_kernel(int which, const DevView& d, int t, int s_cur, int s_next,
                       cudaStream_t st);
void launch_bwd_kernel(int which, const DevView& d, int t, int s_cur, int s_next,
                       const double* xbar_next, double* xbar_cur,
                       const double* snap_seed, int snap_k, int K,
                       unsigned long long* sort_scratch, int force_slow,
                       cudaStream_t st);

}  // namespace dtg
