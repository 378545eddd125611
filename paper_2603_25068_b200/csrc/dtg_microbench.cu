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
    case 6: {  // dependent straight-line Gumbel draws
      int bad = 0;
      for (int i = 0; i < n; ++i)
        acc += gumbel_sl(rng_final(static_cast<std::uint64_t>(acc > 1e300), static_cast<std::uint64_t>(i)), bad);
      acc += bad;
      break;
    }
    case 7: {  // five independent straight-line Gumbel draws per iteration (cycles per 5)
      int bad = 0;
      for (int i = 0; i < n; ++i) {
        const std::uint64_t h = static_cast<std::uint64_t>(acc > 1e300);
        double g0 = gumbel_sl(rng_final(h, 5ull * i), bad), g1 = gumbel_sl(rng_final(h, 5ull * i + 1), bad),
               g2 = gumbel_sl(rng_final(h, 5ull * i + 2), bad), g3 = gumbel_sl(rng_final(h, 5ull * i + 3), bad),
               g4 = gumbel_sl(rng_final(h, 5ull * i + 4), bad);
        acc += g0 + g1 + g2 + g3 + g4;
      }
      acc += bad;
      break;
    }
    case 10: {  // five straight-line Gumbel draws per iteration, interleaved stage by stage
      int bad = 0;
      for (int i = 0; i < n; ++i) {
        const std::uint64_t h = static_cast<std::uint64_t>(acc > 1e300);
        std::uint64_t hh[5], cc[5], b[5];
        double g[5];
        for (int q = 0; q < 5; ++q) {
          hh[q] = h;
          cc[q] = 5ull * i + q;
        }
        rng_final_v<5>(hh, cc, b);
        gumbel_sl_v<5>(b, g, bad);
        acc += g[0] + g[1] + g[2] + g[3] + g[4];
      }
      acc += bad;
      break;
    }
    case 8: {  // dependent straight-line log
      int bad = 0;
      double x = 1.5;
      for (int i = 0; i < n; ++i) x = log_sl(x + 2.0, bad);
      acc = x + bad;
      break;
    }
    case 9: {  // dependent rng_final (integer mixes only)
      std::uint64_t h = 1;
      for (int i = 0; i < n; ++i) h = rng_final(h, static_cast<std::uint64_t>(i));
      acc = static_cast<double>(h & 1023);
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

namespace dtg {
// Bitwise comparison of the straight-line log / Gumbel with libdevice on
// inputs the path produces (rng_unit draws and their -log) and on random
// positive normal doubles over the whole exponent range.
__global__ void k_log_check(std::uint64_t seed, long long n, unsigned long long* counts) {
  unsigned long long mism = 0, bads = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const std::uint64_t b = rng_bits(seed, static_cast<std::uint64_t>(i), 17, 3);
    int bad = 0;
    const double u = rng_unit(b);
    if (__double_as_longlong(log_sl(u, bad)) != __double_as_longlong(log(u))) ++mism;
    const double v = -log(u);
    if (__double_as_longlong(log_sl(v, bad)) != __double_as_longlong(log(v))) ++mism;
    if (__double_as_longlong(gumbel_sl(b, bad)) != __double_as_longlong(gumbel_bits(b))) ++mism;
    {
      std::uint64_t hv[3] = {b, b ^ 0x1234567ULL, seed}, cv[3] = {1ull * i, 7ull, 11ull * i}, bv[3];
      double gv[3];
      rng_final_v<3>(hv, cv, bv);
      gumbel_sl_v<3>(bv, gv, bad);
      for (int q = 0; q < 3; ++q)
        if (bv[q] != rng_final(hv[q], cv[q]) ||
            __double_as_longlong(gv[q]) != __double_as_longlong(gumbel_bits(rng_final(hv[q], cv[q]))))
          ++mism;
    }
    // random positive normal double: exponent field in [1, 2046]
    const std::uint64_t r = rng_bits(seed ^ 0x5bd1e995ULL, static_cast<std::uint64_t>(i), 5, 9);
    const std::uint64_t ex = 1 + (r >> 52) % 2046;
    const double w = __longlong_as_double(static_cast<long long>((ex << 52) | (r & 0xFFFFFFFFFFFFFULL)));
    int bw = 0;
    const double lw = log_sl(w, bw);
    if (bw) ++bads;
    else if (__double_as_longlong(lw) != __double_as_longlong(log(w))) ++mism;
    if (bad) ++bads;
  }
  atomicAdd(&counts[0], mism);
  atomicAdd(&counts[1], bads);
}
}  // namespace dtg

extern "C" int dtg_debug_log_check(uint64_t seed, long long n, unsigned long long* mismatches,
                                   unsigned long long* flagged) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 16) != cudaSuccess) return 4;
  cudaMemset(d, 0, 16);
  dtg::k_log_check<<<148 * 8, 256>>>(seed, n, d);
  unsigned long long h[2] = {0, 0};
  const cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  *mismatches = h[0];
  *flagged = h[1];
  return e == cudaSuccess ? 0 : 4;
}
