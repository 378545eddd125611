// Device losses and the ordered draw reduction (see dtg_loss.h).
//
// Every value is produced by the same fp64 operations in the same order as the
// host loss tapes (dtg_host.cpp mse_loss_builder / control_loss_builder, which
// restate optimization.cpp:83-101 and :234-240), so losses and seeds are
// bit-identical to the host path; -fmad=false keeps the products unfused.
#include <algorithm>
#include <cstddef>

#include "dtg_loss.h"

namespace dtg {

namespace {

// One block per scenario.  Seeds: one thread per (interval k, first occurrence
// of an observed link), accumulating that link's duplicate observations in q
// order exactly like the host tape's `d_snapshots[k][id] += ...`.  Loss: one
// thread per interval sums its squared residuals in q order, then thread 0 adds
// the interval sums in k order and scales (acc = acc + r_k; loss = acc * sc).
__global__ void k_loss_mse(LossView v, int kchunk) {
  extern __shared__ double sq[];  // [kchunk][nobs] squared residuals, then [kobs] interval sums
  const int b = blockIdx.x;
  const double dn = v.dn, sc = v.sc;
  const int n = v.nobs;
  for (int e = threadIdx.x; e < v.kobs * n; e += blockDim.x) {
    const int k = e / n, q = e - k * n;
    if (!v.first[q]) continue;
    const double* snap =
        v.cumh + (static_cast<std::size_t>(k + 1) * v.spi * v.B + b) * v.L;
    const double* o = v.obs + static_cast<std::size_t>(k) * n;
    double acc = 0.0;
    for (int r = q; r >= 0; r = v.next[r]) {
      const double d = snap[v.ids[r]] * dn - o[r];
      acc += ((0.0 + sc * d) + sc * d) * dn;
    }
    v.snap_seed[(static_cast<std::size_t>(b) * v.K + k) * v.L + v.ids[q]] = acc;
  }
  // loss: the squared residuals are formed in parallel, then each interval's
  // sum runs sequentially in q order (one warp lane per interval), as the tape
  double* rk = sq + static_cast<std::size_t>(kchunk) * n;
  for (int k0 = 0; k0 < v.kobs; k0 += kchunk) {
    const int kc = min(kchunk, v.kobs - k0);
    for (int e = threadIdx.x; e < kc * n; e += blockDim.x) {
      const int k = k0 + e / n, q = e - (e / n) * n;
      const double* snap = v.cumh + (static_cast<std::size_t>(k + 1) * v.spi * v.B + b) * v.L;
      const double d = snap[v.ids[q]] * dn - v.obs[static_cast<std::size_t>(k) * n + q];
      sq[e] = d * d;
    }
    __syncthreads();
    for (int kk = threadIdx.x >> 5; kk < kc; kk += blockDim.x >> 5)
      if ((threadIdx.x & 31) == 0) {
        const double* row = sq + static_cast<std::size_t>(kk) * n;
        double r = 0.0;
        for (int q = 0; q < n; ++q) r += row[q];
        rk[k0 + kk] = r;
      }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int k = 0; k < v.kobs; ++k) acc = acc + rk[k];
    v.loss[b] = acc * sc;
    v.extra[b] = 0.0;
  }
}

// One thread per scenario: d = c * dn + (-desired); loss = d * d;
// seed = ((0 + d) + d) * dn on cum_final[target].
__global__ void k_loss_control(LossView v) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= v.B) return;
  const double c =
      v.T > 0 ? v.cumh[(static_cast<std::size_t>(v.T) * v.B + b) * v.L + v.target] : 0.0;
  const double d = c * v.dn + (-v.desired);
  v.loss[b] = d * d;
  v.extra[b] = c * v.dn;
  v.cum_seed[static_cast<std::size_t>(b) * v.L + v.target] = ((0.0 + d) + d) * v.dn;
}

__global__ void k_pack_rows(int B, int L, const double* __restrict__ grads,
                            const double* __restrict__ loss,
                            const double* __restrict__ extra, double* __restrict__ rows) {
  const std::size_t R = 5 * static_cast<std::size_t>(L) + 2;
  const std::size_t total = static_cast<std::size_t>(B) * R;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
       i < total; i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t b = i / R, j = i - b * R;
    double val;
    if (j < 5 * static_cast<std::size_t>(L))
      val = grads[b * 5 * L + j];
    else if (j == 5 * static_cast<std::size_t>(L))
      val = loss[b];
    else
      val = extra[b];
    rows[i] = val;
  }
}

__global__ void k_reduce_rows(int D, int L, const double* __restrict__ rows, int mode,
                              double* __restrict__ out) {
  const int R = 5 * L + 2;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= R) return;
  const double Dd = static_cast<double>(D);
  double s;
  if (j < 5 * L && mode == 0) {
    s = rows[j];
    for (int d = 1; d < D; ++d) s += rows[static_cast<std::size_t>(d) * R + j];
  } else {
    s = 0.0;
    for (int d = 0; d < D; ++d) s += rows[static_cast<std::size_t>(d) * R + j] / Dd;
  }
  out[j] = s;
}

}  // namespace

constexpr std::size_t kMseSmemCap = 227 * 1024;

int max_mse_obs(int k_obs) {
  return static_cast<int>(kMseSmemCap / sizeof(double)) - (k_obs + 1);
}

cudaError_t launch_device_loss(const LossView& v, cudaStream_t st) {
  if (v.kind == kLossMse) {
    // as many intervals' residuals in shared memory as fit in ~160 KB
    const int n = v.nobs > 0 ? v.nobs : 1;
    if (n > max_mse_obs(v.kobs)) return cudaErrorInvalidValue;  // rejected by dtg_set_loss_mse
    int kchunk = static_cast<int>((160 * 1024 / 8 - (v.kobs + 1)) / n);
    kchunk = std::max(1, std::min(kchunk, v.kobs > 0 ? v.kobs : 1));
    const std::size_t smem = sizeof(double) * (static_cast<std::size_t>(kchunk) * n + v.kobs + 1);
    const cudaError_t e = cudaFuncSetAttribute(k_loss_mse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k_loss_mse<<<v.B, 512, smem, st>>>(v, kchunk);
  } else if (v.kind == kLossControl) {
    k_loss_control<<<(v.B + 127) / 128, 128, 0, st>>>(v);
  }
  return cudaGetLastError();
}

void launch_pack_rows(int B, int L, const double* grads, const double* loss,
                      const double* extra, double* rows, cudaStream_t st) {
  const std::size_t total = static_cast<std::size_t>(B) * (5 * L + 2);
  const int blocks = static_cast<int>(std::min<std::size_t>((total + 255) / 256, 148 * 8));
  k_pack_rows<<<blocks, 256, 0, st>>>(B, L, grads, loss, extra, rows);
}

void launch_reduce_rows(int D, int L, const double* rows, int mode, double* out,
                        cudaStream_t st) {
  const int R = 5 * L + 2;
  k_reduce_rows<<<(R + 255) / 256, 256, 0, st>>>(D, L, rows, mode, out);
}

}  // namespace dtg
