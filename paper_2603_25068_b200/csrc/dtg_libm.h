// glibc-identical log() and exp() for host and device.
//
// The reference draws its Gumbel noise as -log(-log u) and forms every
// softmax with glibc's exp/log (tensor.cpp:213-221, 407-433, 682-699).  Which
// link an agent chooses and which candidate a merge admits are argmaxes over
// those values, so bit-exact choices need bit-exact exp/log, not merely
// faithfully rounded ones (CUDA's libdevice differs from glibc in the last
// bit on ~0.5% of Gumbel draws; SURVEY.md §7 "Hard parts" 2).
//
// glibc 2.39 on x86-64 dispatches log/exp to their FMA builds when the CPU has
// FMA + AVX2 (the IFUNC resolvers at libm's __log_finite / __exp_finite):
// __log_fma / __exp_fma, i.e. sysdeps/ieee754/dbl-64/e_log.c and e_exp.c (the
// ARM optimized-routines algorithms: 128-entry table + short polynomial)
// compiled with -mfma.  The functions below restate those machine programs
// operation by operation — every fused multiply-add where the compiler fused
// one (read off `objdump -d libm.so.6`, quoted at each step), every other
// operation a separately rounded IEEE double add / mul.  The constants are
// the bit patterns of __log_data / __exp_data copied out of the same libm
// (dtg_libm_tables.h, tools/glibc_libm_tables.py).
//
// Build rules: device code with -fmad=false and host code with
// -ffp-contract=off, so the unfused operations stay unfused; fma() is the
// IEEE fused multiply-add on both sides (__fma_rn / std::fma).
// Verified bit-identical to the running libm's log/exp on 10^8+ inputs per
// function on the host (tests/test_libm.py) and on the device
// (tests/test_gpu_golden.py).
#pragma once
#include <cstdint>
#include <cstring>

#include "dtg_libm_tables.h"

#if defined(__CUDACC__)
#define DTG_LIBM_HD __host__ __device__ __forceinline__
#else
#include <cmath>
#define DTG_LIBM_HD inline
#endif

namespace dtg {
namespace glibc {

// The scalar constants are constexpr (constant-bank operands on the device);
// the tables live in memory.
static const double kLogTabH[256] = {DTG_GLIBC_LOG_TAB};
static const std::uint64_t kExpTabH[256] = {DTG_GLIBC_EXP_TAB};
#if defined(__CUDACC__)
// global memory (read through the L1): per-lane table indices diverge, which
// the constant cache would serialise
static __device__ const double kLogTabD[256] = {DTG_GLIBC_LOG_TAB};
static __device__ const std::uint64_t kExpTabD[256] = {DTG_GLIBC_EXP_TAB};
#endif

DTG_LIBM_HD double as_double(std::uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}
DTG_LIBM_HD std::uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
  return static_cast<std::uint64_t>(__double_as_longlong(d));
#else
  std::uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
#endif
}
DTG_LIBM_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
// {invc, logc} of log interval i (one 16-byte load on the device)
DTG_LIBM_HD void log_tab(int i, double& invc, double& logc) {
#if defined(__CUDA_ARCH__)
  const double2 v = __ldg(reinterpret_cast<const double2*>(kLogTabD) + i);
  invc = v.x;
  logc = v.y;
#else
  invc = kLogTabH[2 * i];
  logc = kLogTabH[2 * i + 1];
#endif
}
// {tail bits, sbits} of 2^(i/128)
DTG_LIBM_HD void exp_tab(int i, std::uint64_t& tail, std::uint64_t& sbits) {
#if defined(__CUDA_ARCH__)
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(kExpTabD) + i);
  tail = v.x;
  sbits = v.y;
#else
  tail = kExpTabH[2 * i];
  sbits = kExpTabH[2 * i + 1];
#endif
}

// log(x) for x close to 1: |x - 1| < 0x1p-4 or so (__log_fma, 0x79e50..0x79f22).
DTG_LIBM_HD double log_near1(double x) {
  if (as_u64(x) == 0x3ff0000000000000ULL) return 0.0;
  const double r = x - 1.0;                                      // vsubsd
  const double r2 = r * r;                                       // vmulsd
  const double p1 = fma_(r2, B3, fma_(r, B2, B1));
  const double p2 = fma_(r2, B6, fma_(r, B5, B4));
  const double r3 = r * r2;                                      // vmulsd
  double q = fma_(r2, B9, fma_(r, B8, B7));
  q = fma_(r3, B10, q);
  const double br = fma_(fma_(q, r3, p2), r3, p1);               // B[1] + r B[2] + ... (bracket)
  // w = r * 0x1p27; rhi = r + w - w  (contracted: fma then fnmadd)
  const double t = fma_(r, 0x1p27, r);
  const double rhi = fma_(-0x1p27, r, t);
  const double b0 = B0;                                         // -0.5
  const double rhi2 = rhi * rhi;                                 // vmulsd
  const double rlo = r - rhi;                                    // vsubsd
  const double hi = fma_(rhi2, b0, r);                           // hi = r + w
  const double lo0 = fma_(rhi2, b0, r - hi);                     // lo = r - hi + w
  const double lo = fma_(b0 * rlo, r + rhi, lo0);                // lo += B0 rlo (rhi + r)
  const double y = fma_(br, r3, lo);                             // y = r3 * br + lo
  return hi + y;                                                 // vaddsd
}

// log(x) for positive normal x outside the near-1 interval (0x79d8f..0x79e4b).
DTG_LIBM_HD double log_main(std::uint64_t ix) {
  const std::uint64_t tmp = ix - 0x3fe6000000000000ULL;         // ix - OFF
  const int i = static_cast<int>((tmp >> 45) & 0x7f);
  const std::uint64_t iz = ix - (tmp & 0xfff0000000000000ULL);
  const double kd = static_cast<double>(static_cast<int>(static_cast<std::int64_t>(tmp) >> 52));
  double invc, logc;
  log_tab(i, invc, logc);
  const double z = as_double(iz);
  const double w = fma_(kd, LN2HI, logc);            // kd*Ln2hi + logc
  const double r = fma_(z, invc, -1.0);                          // z*invc - 1
  const double a12 = fma_(r, A2, A1);
  const double hi = r + w;                                       // vaddsd
  const double r2 = r * r;                                       // vmulsd
  const double lo = fma_(kd, LN2LO, (w - hi) + r);   // w - hi + r + kd*Ln2lo
  const double r3 = r * r2;                                      // vmulsd
  const double a34 = fma_(r, A4, A3);
  const double lo2 = fma_(r2, A0, lo);             // lo + r2*A[0]
  const double p = fma_(a34, r2, a12);
  return fma_(r3, p, lo2) + hi;                                  // (... + r3*p) + hi
}

// glibc log(double) (x86-64 FMA build).
DTG_LIBM_HD double log(double x) {
  std::uint64_t ix = as_u64(x);
  const std::uint32_t top = static_cast<std::uint32_t>(ix >> 48);
  if (ix - 0x3fee000000000000ULL < 0x3090000000000ULL) return log_near1(x);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if (ix * 2 == 0) return as_double(0xfff0000000000000ULL);    // __math_divzero(1): -inf
    if (ix == 0x7ff0000000000000ULL) return x;                   // log(inf) = inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u)          // __math_invalid: nan
      return (top & 0x7ff0u) == 0x7ff0u && (ix << 12) ? x : as_double(0x7ff8000000000000ULL);
    ix = as_u64(x * 0x1p52);                                     // subnormal: normalise
    ix -= 52ULL << 52;
  }
  return log_main(ix);
}

// glibc exp(double) (x86-64 FMA build, __exp_fma 0x79b60..0x79d47).
DTG_LIBM_HD double exp(double x) {
  const std::uint64_t ix = as_u64(x);
  std::uint32_t abstop = static_cast<std::uint32_t>(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if (static_cast<std::int32_t>(abstop - 0x3c9u) < 0) return 1.0 + x;  // tiny
    if (abstop >= 0x409u) {
      if (ix == 0xfff0000000000000ULL) return 0.0;
      if (abstop == 0x7ffu) return 1.0 + x;
      return (ix >> 63) ? 0.0 : as_double(0x7ff0000000000000ULL);  // __math_uflow / __math_oflow
    }
    abstop = 0;  // large |x|: special case below
  }
  const double kd0 = fma_(x, INVLN2N, SHIFT);  // z + Shift
  const std::uint64_t ki = as_u64(kd0);
  const double kd = kd0 - SHIFT;
  double r = fma_(kd, NEGLN2HIN, x);
  r = fma_(kd, NEGLN2LON, r);
  const double c23 = fma_(r, C3, C2);
  std::uint64_t tail_b, sb;
  exp_tab(static_cast<int>(ki & 0x7f), tail_b, sb);
  const double rt = r + as_double(tail_b);                       // vaddsd r + tail
  const std::uint64_t sbits = sb + (ki << 45);
  const double r2 = r * r;
  const double c45 = fma_(r, C5, C4);
  const double t1 = fma_(c23, r2, rt);
  const double tmp = fma_(r2 * r2, c45, t1);
  if (abstop != 0) {
    const double scale = as_double(sbits);
    return fma_(scale, tmp, scale);
  }
  // specialcase (0x79c60..)
  if ((ki & 0x80000000ULL) == 0) {
    const double scale = as_double(sbits - (1009ULL << 52));
    return fma_(scale, tmp, scale) * 0x1p1009;
  }
  const double scale = as_double(sbits + (1022ULL << 52));
  const double st = tmp * scale;
  double y = scale + st;
  if (1.0 > y) {
    const double hi = y + 1.0;
    const double lo = (scale - y) + st;
    double s = (1.0 - hi) + y;
    s = s + lo;
    s = s + hi;
    y = s - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return y * 0x1p-1022;
}

}  // namespace glibc
}  // namespace dtg
