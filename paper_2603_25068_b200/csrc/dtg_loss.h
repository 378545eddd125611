// Device-side losses of the reference's optimisation loops and the ordered
// reduction over noise draws.
//
// The reference evaluates its losses on a host tape after the forward sweep
// and seeds the checkpointed backward from it (engine.cpp:369-385); the
// calibrate / optimize_control loops then sum the per-draw gradients on the
// host (optimization.cpp:176-193, 255-265).  Here both stay on the device:
// the loss value and its seeds are computed from the device count history,
// and the per-draw rows are reduced in draw order by one kernel, so one
// optimisation iteration moves O(L) bytes across PCIe instead of the whole
// B x T x L count history.
#pragma once
#include <cuda_runtime.h>

namespace dtg {

constexpr int kLossNone = 0;
constexpr int kLossMse = 1;      // mse_loss_builder, optimization.cpp:83-101
constexpr int kLossControl = 2;  // optimize_control's loss, optimization.cpp:234-240

struct LossView {
  int kind;
  int B, L, N, T, spi, K;  // K = snapshots kept by the forward (T / spi)
  double dn;               // delta_n
  const double* cumh;      // [T+1][B][L] count history (agent units)
  // MSE: observed links and values [kobs][nobs]; first[q] = 1 for the first
  // occurrence of a link id, next[q] = next q' with the same id (or -1)
  int kobs, nobs;
  const int* ids;
  const int* first;
  const int* next;
  const double* obs;
  double sc;  // 1 / (kobs * nobs)
  // control
  int target;
  double desired;
  // outputs
  double* snap_seed;  // [B][K][L] (zeroed by the caller)
  double* cum_seed;   // [B][L]    (zeroed by the caller)
  double* loss;       // [B]
  double* extra;      // [B] control: achieved count cum_final[target] * dn
};

// Largest observed-link count the MSE kernel holds in shared memory (one
// interval of residuals plus the interval sums must fit 227 KB).
int max_mse_obs(int k_obs);
cudaError_t launch_device_loss(const LossView& v, cudaStream_t st);

/// rows[b] = [grads u|kappa|beta|alpha|cost (5L), loss, extra] for b < B.
void launch_pack_rows(int B, int L, const double* grads, const double* loss,
                      const double* extra, double* rows, cudaStream_t st);

/// Ordered reduction over D draw rows of width R = 5L + 2 (draw order d = 0..D-1):
///   mode 0 (calibrate, optimization.cpp:176-193): g = row_0; g += row_d
///   mode 1 (control,   optimization.cpp:262-264): g = 0.0; g += row_d / D
/// and, in both modes, loss = 0.0; loss += row_d[5L] / D and
/// extra = 0.0; extra += row_d[5L+1] / D.
void launch_reduce_rows(int D, int L, const double* rows, int mode, double* out,
                        cudaStream_t st);

}  // namespace dtg
