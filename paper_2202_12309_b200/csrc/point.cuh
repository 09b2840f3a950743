// point.cuh -- pointwise fp64 device math shared by the stage kernels (kernels.cu, stage2.cu).
// Product code only; nothing here is shared with oracle/.
#pragma once
#include "device.cuh"

namespace ph {
// textbook minmod: same strict sign -> the smaller magnitude, else 0.  The sign test
// reads only the high words (integer pipe); one DSETP with |.| modifiers picks the magnitude.
// (+-0 operands give +-0, whose use q +- 0.5*(+-0) == q matches the oracle's 0.)
__device__ __forceinline__ double minmod_i(double a, double b) {
  const int ha = __double2hiint(a), hb = __double2hiint(b);
  const double m = (fabs(a) < fabs(b)) ? a : b;
  return ((ha ^ hb) >= 0) ? m : 0.0;
}

__device__ __forceinline__ double minmod_pick(double a, double b) { return (fabs(a) < fabs(b)) ? a : b; }
__device__ __forceinline__ double minmod_half(double a, double b) {
  return ((__double2hiint(a) ^ __double2hiint(b)) >= 0) ? 0.5 : 0.0;
}

// MUFU-seeded reciprocal with one third-order correction: r (1 + e + e^2), e = 1 - x r.  The
// rcp.approx seed (~2^-23) becomes ~1 ulp in 3 fp64 ops.  The paper fixes no rounding; parity
// with the oracle's IEEE division is at round-off (A31).
__device__ __forceinline__ double rcp_nr(double x) {
#ifdef PH_STRICT  // strict diagnostic build: IEEE division as in the oracle
  return 1.0 / x;
#endif
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// MUFU-seeded reciprocal square root with one third-order correction:
// y (1 + e/2 + 3e^2/8), e = 1 - x y^2 (5 fp64 ops)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y, e * fma(0.375, e, 0.5), y);
}

// sound speed c = sqrt(gamma p / rho) = (gamma p) * rsqrt(gamma p rho): one MUFU, no division
__device__ __forceinline__ double sound_speed(double rho, double p, double gamma) {
#ifdef PH_STRICT  // strict diagnostic build: c = sqrt(gamma p / rho), IEEE ops (O5)
  return sqrt(gamma * p / rho);
#endif
  double gp = gamma * p;
  return gp * rsqrt_nr(gp * rho);
}

// min / max as plain compare-selects (DSETP + 2 FSEL).  fmin/fmax carry IEEE NaN semantics that
// cost a SEL, a predicated LOP3 and register moves per call (+1.3 % on 2b without them); a NaN state
// is already flagged by the cons->prim positivity check, so only finite operands matter here.
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

__device__ __forceinline__ void set_error(ErrWord* err, int stage, long long gid, int k, int j, int i) {
  if (atomicCAS(&err->flag, 0, 1) == 0) {
    err->stage = stage;
    err->gid = gid;
    err->k = k;
    err->j = j;
    err->i = i;
    __threadfence();
  }
}

// Race probe (the jitter build, -DPH_JITTER=<seed>; compute-sanitizer is closed on this GPU pool): one
// warp in four sleeps up to ~2 us at each probe point, chosen by a hash of (CTA, warp, salt, seed), so
// warps reach barriers, mbarrier waits and shared / global accesses in orders the normal build never
// produces.  tests/test_gpu_races.py requires the jitter build's results to equal the normal build's
// bit for bit.  A no-op in normal builds.
__device__ __forceinline__ void ph_jitter(unsigned salt) {
#ifdef PH_JITTER
  unsigned h = (blockIdx.x * 0x9E3779B1u) ^ ((threadIdx.x >> 5) * 0x85EBCA77u) ^ (salt * 0xC2B2AE3Du) ^
               ((unsigned)PH_JITTER * 0x27D4EB2Fu);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep(h & 2047u);
#else
  (void)salt;
#endif
}

// x / d rounded to nearest -- bit-identical to __ddiv_rn(x, d) -- for a divisor fixed per launch (6 in
// PPM / WENO-Z, gamma - 1 in E = p / (gamma - 1)) with rd = RN(1/d) (reading A47):
//   q0 = RN(x rd) is within 1.5 ulp of x/d;
//   q1 = RN(q0 + (x - q0 d) rd) is faithful (error 1/2 ulp plus ~2^-52 ulp);
//   q2 = RN(q1 + r rd) with the residual r = x - q1 d exact (q1 faithful) is RN(x/d) by Markstein's theorem
//   (q faithful and rd within half an ulp of 1/d).
// 5 fp64 operations instead of the general division's reciprocal iteration and range checks.  The
// theorem needs every step inside the normal range: 2^-900 < |x| < 2^900 and 2^-60 < d < 2^60 (the
// callers' divisors); zero keeps its sign (x / d with d > 0), everything else takes __ddiv_rn.
__device__ __forceinline__ double ddiv_k(double x, double d, double rd) {
  const double ax = fabs(x);
  if (!(ax > 0x1p-900 && ax < 0x1p900)) return ax == 0.0 ? x : __ddiv_rn(x, d);
  double q = __dmul_rn(x, rd);
  q = __fma_rn(__fma_rn(-q, d, x), rd, q);
  return __fma_rn(__fma_rn(-q, d, x), rd, q);
}
constexpr double K6 = 6.0, RK6 = 1.0 / 6.0;  // RN(1/6), folded by the compiler

}  // namespace ph
