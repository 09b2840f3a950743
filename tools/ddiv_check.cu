// ddiv_k (point.cuh, reading A47) against the IEEE division __ddiv_rn, bit for bit.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2202_12309_b200/csrc tools/ddiv_check.cu
//   ./a.out [log2 samples per divisor]   ->  one JSON line per divisor: samples, mismatches
//
// Dividends: random 53-bit mantissas over exponents -950..950 (both signs), plus structured cases that
// sit at rounding boundaries: x = d * m (exact multiples), x = d * (m + 1/2 ulp) (ties of x/d) and their
// 1-ulp neighbours, powers of two, and the range edges / zeros / non-finite values.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include "point.cuh"

using namespace ph;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// 1-ulp steps of a positive double (the dividends are built positive; the sign is applied last)
__device__ __forceinline__ double up(double x) { return __longlong_as_double(__double_as_longlong(x) + 1); }
__device__ __forceinline__ double dn(double x) { return x > 0.0 ? __longlong_as_double(__double_as_longlong(x) - 1) : x; }

__global__ void check(double d, double rd, uint64_t n, uint64_t seed, unsigned long long* bad, double* ex) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(seed ^ (i * 0xD1B54A32D192ED03ull));
    double x;
    const int kind = (int)(r & 7);
    const uint64_t man = (r >> 3) & ((1ull << 52) - 1);
    const int ex2 = (int)((r >> 55) % 1901) - 950;
    const double m = __longlong_as_double((long long)((1023ull << 52) | man));  // [1, 2)
    if (kind < 4) {
      x = ldexp(m, ex2);
    } else if (kind == 4) {  // exact multiple of d, and its neighbours
      const double y = ldexp(m, (int)((r >> 56) % 64) - 32);
      x = __dmul_rn(d, y);
      const int k = (int)((r >> 60) & 3);
      if (k == 1) x = up(x);
      if (k == 2) x = dn(x);
    } else if (kind == 5) {  // x/d close to a midpoint between two doubles: d * (y + ulp/2) rounded, +-1 ulp
      const double y = ldexp(m, (int)((r >> 56) % 64) - 32);
      const double h = ldexp(1.0, ilogb(y) - 53);
      x = __fma_rn(d, y, __dmul_rn(d, h));
      const int k = (int)((r >> 60) & 3);
      if (k == 1) x = up(x);
      if (k == 2) x = dn(x);
    } else if (kind == 6) {  // powers of two and their neighbours
      x = ldexp(1.0, ex2);
      const int k = (int)((r >> 60) & 3);
      if (k == 1) x = up(x);
      if (k == 2) x = dn(x);
    } else {  // range edges, zeros, subnormals, non-finite
      const double sp[12] = {0.0, 0x1p-900, 0x1p900, 0x1.fffffffffffffp899, 0x1.0000000000001p-900, 0x1p-1070,
                             0x1p-1022, 1e308, INFINITY, NAN, 0x1p-899, 0x1.8p900};
      x = sp[(r >> 8) % 12];
      if ((r >> 20) & 1) x = dn(x);
    }
    if ((r >> 40) & 1) x = -x;
    const double a = ddiv_k(x, d, rd), b = __ddiv_rn(x, d);
    const bool same = __double_as_longlong(a) == __double_as_longlong(b) || (isnan(a) && isnan(b));
    if (!same) {
      if (atomicAdd(bad, 1ull) == 0) ex[0] = x;
    }
  }
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 28;
  const uint64_t n = 1ull << lg;
  const double gammas[] = {5.0 / 3.0, 1.4, 1.1, 2.0, 1.0001, 3.0, 1.0 + 0x1p-52, 7.0};
  unsigned long long* bad;
  double* ex;
  cudaMalloc(&bad, 8);
  cudaMalloc(&ex, 8);
  int rc = 0;
  for (int t = -1; t < (int)(sizeof(gammas) / sizeof(gammas[0])); ++t) {
    const double d = t < 0 ? 6.0 : gammas[t] - 1.0, rd = t < 0 ? 1.0 / 6.0 : 1.0 / (gammas[t] - 1.0);
    cudaMemset(bad, 0, 8);
    cudaMemset(ex, 0, 8);
    check<<<148 * 16, 256>>>(d, rd, n, 0x5EEDull + t, bad, ex);
    unsigned long long h = 0;
    double hx = 0;
    if (cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 3;
    cudaMemcpy(&hx, ex, 8, cudaMemcpyDeviceToHost);
    printf("{\"divisor\": %.17g, \"samples\": %llu, \"mismatches\": %llu, \"first_x\": %.17g}\n", d,
           (unsigned long long)n, h, hx);
    if (h) rc = 1;
  }
  return rc;
}
