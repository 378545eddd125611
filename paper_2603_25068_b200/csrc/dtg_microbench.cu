// Test hook: latency of the primitives the per-step critical path is made of,
// measured with clock64 by one thread (cycles per operation).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "dtg_device.cuh"

namespace dtg {

__global__ void k_micro(int which, int n, const int* chain, double* out) {
  // which >= 15: all 32 lanes run the chain on lane-dependent arguments
  // (divergent table indices); lane 0 reports
  if ((which < 15 && threadIdx.x != 0) || blockIdx.x != 0) return;
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
    case 11: {  // dependent glibc log, table path (arguments >= 2)
      double x = 1.5;
      for (int i = 0; i < n; ++i) x = dlog(x + 2.0);
      acc = x;
      break;
    }
    case 12: {  // dependent glibc log, near-1 path
      double x = 0.01;
      for (int i = 0; i < n; ++i) x = dlog(1.0 + x * 0.5) + 0.01;
      acc = x;
      break;
    }
    case 13: {  // dependent glibc exp
      double x = 0.5;
      for (int i = 0; i < n; ++i) x = dexp(-x);
      acc = x;
      break;
    }
    case 15: {  // 32 lanes: dependent glibc log, table path
      double x = 1.5 + threadIdx.x * 0.37;
      for (int i = 0; i < n; ++i) x = dlog(x + 2.0 + threadIdx.x * 0.73);
      acc = x;
      break;
    }
    case 16: {  // 32 lanes: dependent libdevice log
      double x = 1.5 + threadIdx.x * 0.37;
      for (int i = 0; i < n; ++i) x = log(x + 2.0 + threadIdx.x * 0.73);
      acc = x;
      break;
    }
    case 17: {  // 32 lanes: dependent Gumbel draws (glibc logs)
      for (int i = 0; i < n; ++i)
        acc += gumbel(static_cast<std::uint64_t>(acc > 1e300), 3 + threadIdx.x, i, 7);
      break;
    }
    case 18: {  // 32 lanes: five interleaved Gumbel draws per iteration
      int bad = 0;
      for (int i = 0; i < n; ++i) {
        const std::uint64_t h = static_cast<std::uint64_t>(acc > 1e300) + threadIdx.x;
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

// L2 read bandwidth: every CTA streams its share of a buffer that fits in L2
// (16-byte loads, 4 in flight per thread), `reps` passes; the first pass
// (cold) is excluded by the caller running it twice.
__global__ void __launch_bounds__(512) k_l2_read(const double2* __restrict__ buf, std::size_t n2, int reps,
                                                 double* sink) {
  double acc = 0.0;
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n2; i += 4 * stride) {
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = i + q * stride < n2 ? __ldcg(buf + i + q * stride) : make_double2(0, 0);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc += v[q].x + v[q].y;
    }
  if (acc == 12345.678) *sink = acc;  // keeps the loads
}

// Latency floor of one persistent engine step: the same grid and barrier as
// k_forward_fused (release/acquire counter), two barriers per step, and in each
// phase one dependent global round trip per CTA (thread 0 reads what another
// CTA wrote in the previous phase) -- a step with no work at all.
__global__ void __launch_bounds__(512) k_step_floor(unsigned int* ctr, int* cell, int T, unsigned long long* ns) {
  unsigned int epoch = 0;
  auto barrier = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++epoch;
      const unsigned int target = epoch * gridDim.x;
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < target);
    }
    __syncthreads();
  };
  unsigned long long t0 = 0;
  if (threadIdx.x == 0 && blockIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int v = 0;
  for (int t = 0; t < T; ++t) {
    if (threadIdx.x == 0) {
      v += cell[(blockIdx.x + 1 + t) % gridDim.x];
      cell[blockIdx.x] = v + t;
    }
    barrier();
    if (threadIdx.x == 0) {
      v += cell[(blockIdx.x + 3 + t) % gridDim.x];
      cell[gridDim.x + blockIdx.x] = v;
    }
    barrier();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *ns = t1 - t0;
  }
  if (v == 0x7fffffff) cell[0] = v;
}

}  // namespace dtg

// Builder-measured L2 read bandwidth (GB/s) over a `bytes` buffer resident in
// L2 (second of two timed launches, CUDA events).
extern "C" int dtg_debug_l2_bandwidth(long long bytes, int reps, double* gbps) {
  double2* buf = nullptr;
  double* sink = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 8) != cudaSuccess) return 4;
  cudaMemset(buf, 0, bytes);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const std::size_t n2 = static_cast<std::size_t>(bytes) / 16;
  float ms = 0.f;
  for (int pass = 0; pass < 2; ++pass) {
    cudaEventRecord(e0);
    dtg::k_l2_read<<<sms * 4, 512>>>(buf, n2, reps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const cudaError_t e = cudaGetLastError();
  *gbps = static_cast<double>(bytes) * reps / (ms * 1e-3) / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(sink);
  return e == cudaSuccess ? 0 : 4;
}

// Builder-measured latency floor of a two-barrier persistent step (us) on
// `grid` CTAs of 512 threads.
extern "C" int dtg_debug_step_floor(int grid, int T, double* us_per_step) {
  unsigned int* ctr = nullptr;
  int* cell = nullptr;
  unsigned long long* ns = nullptr;
  if (cudaMalloc(&ctr, 4) != cudaSuccess || cudaMalloc(&cell, 8 * grid) != cudaSuccess ||
      cudaMalloc(&ns, 8) != cudaSuccess)
    return 4;
  unsigned long long h = 0;
  for (int pass = 0; pass < 2; ++pass) {
    cudaMemset(ctr, 0, 4);
    cudaMemset(cell, 0, 8 * grid);
    void* args[] = {&ctr, &cell, &T, &ns};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dtg::k_step_floor), dim3(grid), dim3(512), args, 0,
                                nullptr);
    cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
  }
  const cudaError_t e = cudaGetLastError();
  *us_per_step = static_cast<double>(h) / 1e3 / T;
  cudaFree(ctr);
  cudaFree(cell);
  cudaFree(ns);
  return e == cudaSuccess ? 0 : 4;
}

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
// Internal consistency of the device's glibc log: the interleaved F-operand
// Gumbel / log (gumbel_sl_v, log_sl_v) against the scalar glibc::log on the
// inputs the path produces and on random positive doubles over the whole
// exponent range (counts[1] stays 0: no argument is ever flagged).
__global__ void k_log_check(std::uint64_t seed, long long n, unsigned long long* counts) {
  unsigned long long mism = 0, bads = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const std::uint64_t b = rng_bits(seed, static_cast<std::uint64_t>(i), 17, 3);
    int bad = 0;
    const double u = rng_unit(b);
    const double v = -glibc::log(u);
    if (__double_as_longlong(gumbel_sl(b, bad)) != __double_as_longlong(-glibc::log(v))) ++mism;
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
    // random positive double (normal or subnormal) through the interleaved path
    const std::uint64_t r = rng_bits(seed ^ 0x5bd1e995ULL, static_cast<std::uint64_t>(i), 5, 9);
    double wv[2] = {__longlong_as_double(static_cast<long long>(r & 0x7FEFFFFFFFFFFFFFULL)),
                    1.0 + (rng_unit(r) - 0.5) * 0.25};
    const double w0 = glibc::log(wv[0]), w1 = glibc::log(wv[1]);
    log_sl_v<2>(wv, bad);
    if (__double_as_longlong(wv[0]) != __double_as_longlong(w0)) ++mism;
    if (__double_as_longlong(wv[1]) != __double_as_longlong(w1)) ++mism;
    if (bad) ++bads;
  }
  atomicAdd(&counts[0], mism);
  atomicAdd(&counts[1], bads);
}

// Inputs of kind `which` and the device's glibc-restated results for them
// (dtg_debug_libm_check compares them with the host's libm).
__device__ __forceinline__ double libm_input(int which, std::uint64_t seed, long long i) {
  const std::uint64_t b = rng_bits(seed, static_cast<std::uint64_t>(i), 29, which);
  const double u = rng_unit(b);
  switch (which) {
    case 0: return u;                                   // log(u), the Gumbel's first log
    case 1: return -glibc::log(u);                      // its second log
    case 2: return u;                                   // the whole Gumbel -log(-log u)
    case 3: return __longlong_as_double(static_cast<long long>(b & 0x7FEFFFFFFFFFFFFFULL));  // log, any exponent
    case 4: return 1.0 + (u - 0.5) * 0.25;              // log near 1 (glibc's separate path)
    case 5: return -750.0 + 1460.0 * u;                 // exp over its whole range
    case 6: return -60.0 * u;                           // exp of softmax arguments (<= 0)
    default: return __longlong_as_double(static_cast<long long>(b & 0xFFEFFFFFFFFFFFFFULL));  // exp, any finite
  }
}

__global__ void k_libm_eval(int which, std::uint64_t seed, long long i0, int n, double* in, double* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double x = libm_input(which, seed, i0 + k);
  double y;
  if (which == 2) {
    y = -dlog(-dlog(x));
  } else if (which <= 4) {
    y = dlog(x);
  } else {
    y = dexp(x);
  }
  in[k] = x;
  out[k] = y;
}
}  // namespace dtg

extern "C" int dtg_debug_libm_check(int which, uint64_t seed, long long n, int on_device,
                                    unsigned long long* mismatches) {
  constexpr int kChunk = 1 << 24;
  double *d_in = nullptr, *d_out = nullptr;
  std::vector<double> in(kChunk), out(kChunk);
  if (on_device && (cudaMalloc(&d_in, kChunk * 8) != cudaSuccess || cudaMalloc(&d_out, kChunk * 8) != cudaSuccess))
    return 4;
  unsigned long long mism = 0;
  int rc = 0;
  for (long long i0 = 0; i0 < n; i0 += kChunk) {
    const int m = static_cast<int>(std::min<long long>(kChunk, n - i0));
    if (on_device) {
      dtg::k_libm_eval<<<(m + 255) / 256, 256>>>(which, seed, i0, m, d_in, d_out);
      if (cudaMemcpy(in.data(), d_in, m * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(out.data(), d_out, m * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
        rc = 4;
        break;
      }
    } else {  // the host restatement, on the host's copy of the inputs
      for (int k = 0; k < m; ++k) {
        const std::uint64_t b = dtg::rng_bits(seed, static_cast<std::uint64_t>(i0 + k), 29, which);
        const double u = dtg::rng_unit(b);
        double x;
        switch (which) {
          case 0: case 2: x = u; break;
          case 1: x = -dtg::glibc::log(u); break;
          case 3: { const std::uint64_t q = b & 0x7FEFFFFFFFFFFFFFULL; std::memcpy(&x, &q, 8); } break;
          case 4: x = 1.0 + (u - 0.5) * 0.25; break;
          case 5: x = -750.0 + 1460.0 * u; break;
          case 6: x = -60.0 * u; break;
          default: { const std::uint64_t q = b & 0xFFEFFFFFFFFFFFFFULL; std::memcpy(&x, &q, 8); } break;
        }
        in[k] = x;
        out[k] = which == 2 ? -dtg::glibc::log(-dtg::glibc::log(x))
                            : (which <= 4 ? dtg::glibc::log(x) : dtg::glibc::exp(x));
      }
    }
    for (int k = 0; k < m; ++k) {  // against the running libm (glibc)
      const double x = in[k];
      const double ref = which == 2 ? -std::log(-std::log(x)) : (which <= 4 ? std::log(x) : std::exp(x));
      std::uint64_t a, c;
      std::memcpy(&a, &out[k], 8);
      std::memcpy(&c, &ref, 8);
      if (a != c) ++mism;
    }
  }
  if (d_in) cudaFree(d_in);
  if (d_out) cudaFree(d_out);
  *mismatches = mism;
  return rc;
}

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
