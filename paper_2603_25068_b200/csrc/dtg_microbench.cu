// Test hook: latency of the primitives the per-step critical path is made of,
// measured with clock64 by one thread (cycles per operation).
#include <cooperative_groups.h>

#include <cstdint>

#include "dtg_device.cuh"

namespace dtg {

__global__ void k_micro(int which, int n, const int* chain, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  long long t0 = clock64();
  switch (which) {
    case 0:  // dependent Gumbel draws
      for (int i = 0; i < n; ++i) acc += gumbel(static_cast<std::uint64_t>(acc > 1e300), 3, i, 7);
      break;
    case 1: {  // dependent double log
      double x = 1.5;
      for (int i = 0; i < n; ++i) x = log(x + 2.0);
      acc = x;
      break;
    }
    case 2: {  // dependent double exp
      double x = 0.5;
      for (int i = 0; i < n; ++i) x = exp(-x);
      acc = x;
      break;
    }
    case 3: {  // dependent double division
      double x = 1.5;
      for (int i = 0; i < n; ++i) x = 1.0 / (x + 0.25);
      acc = x;
      break;
    }
    case 4: {  // dependent global loads (pointer chase, L2 after warm-up)
      int p = 0;
      for (int i = 0; i < n; ++i) p = chain[p];
      acc = p;
      break;
    }
    case 5: {  // counter-RNG uniform only
      for (int i = 0; i < n; ++i) acc += rng_uniform(static_cast<std::uint64_t>(acc > 1e300), 3, i, 7);
      break;
    }
  }
  long long t1 = clock64();
  out[0] = static_cast<double>(t1 - t0) / n;
  out[1] = acc;
}

__global__ void k_micro_barrier(int n, double* out) {
  cooperative_groups::grid_group g = cooperative_groups::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) g.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = static_cast<double>(t1 - t0) / n;
}

}  // namespace dtg

extern "C" int dtg_debug_microbench(int which, int n, int grid, double* result) {
  double* d_out = nullptr;
  int* chain = nullptr;
  cudaMalloc(&d_out, 16);
  const int M = 1 << 20;
  cudaMalloc(&chain, M * sizeof(int));
  {
    int* h = new int[M];
    for (int i = 0; i < M; ++i) h[i] = static_cast<int>((static_cast<long long>(i) * 7919 + 104729) % M);
    cudaMemcpy(chain, h, M * sizeof(int), cudaMemcpyHostToDevice);
    delete[] h;
  }
  if (which < 100) {
    dtg::k_micro<<<1, 32>>>(which, n, chain, d_out);
    dtg::k_micro<<<1, 32>>>(which, n, chain, d_out);
  } else {
    void* args[] = {&n, &d_out};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dtg::k_micro_barrier), dim3(grid), dim3(512), args, 0,
                                nullptr);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(result, d_out, 16, cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  cudaFree(chain);
  return e == cudaSuccess ? 0 : 4;
}
