// ubench.cu -- per-SM instruction throughput of the ops the stage kernel is made of (SURVEY §8(d)
// "microbenchmarks, once per box": fp64 DFMA / DADD / DSETP peak), measured on the B200 itself.
//
// Each kernel runs CH independent dependency chains per thread for ITER iterations on a grid of
// 148 * OCC CTAs of 256 threads (full chip).  Reported: lane-ops per SM clock (clock64 over the
// kernel, per SM) and lane-ops per second (CUDA events), plus the dependent-chain latency of
// each op (one warp, one chain).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
// Output: one JSON object per line.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

constexpr int CH = 8;
constexpr int ITER = 2048;

enum Op { DFMA, DADD, DMUL, DMINSEL, DSETP_ONLY, RCP64, RSQ64, FMA_IMAD, FMA_2INT, FFMA32, IMAD32, LDS64, LDS128, SHFL64, NOPS };
static const char* kName[NOPS] = {"dfma", "dadd", "dmul", "dsetp+2fsel (fp64 min)", "dsetp", "mufu.rcp64h",
                                  "mufu.rsq64h", "dfma+imad (1:1)", "dfma+2 int (1:2)", "ffma (fp32)", "imad (int32)",
                                  "lds.64", "lds.128", "shfl x2 (fp64)"};
// lane-ops counted per inner step and chain (the mixed kernels count the fp64 op only)
static const int kOpsPerStep[NOPS] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};

template <int OP>
__global__ void __launch_bounds__(256) tput(double* out, long long* clk, double seed, int lat_mode) {
  __shared__ double sm[2048];
  for (int t = threadIdx.x; t < 2048; t += blockDim.x) sm[t] = seed + t;
  __syncthreads();
  double a[CH], b = seed * 1.0000001, c = seed * 0.999999;
  int ia[CH];
  float fa[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    a[k] = seed + k + threadIdx.x * 1e-9;
    ia[k] = threadIdx.x + k;
    fa[k] = (float)a[k];
  }
  const int nch = lat_mode ? 1 : CH;
  unsigned idx = threadIdx.x * 2;
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (k >= nch) break;
      if (OP == DFMA) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(b), "d"(c));
      if (OP == DADD) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[k]) : "d"(b));
      if (OP == DMUL) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(a[k]) : "d"(b));
      if (OP == DMINSEL)
        asm volatile("{.reg .pred p; setp.lt.f64 p, %0, %1; selp.f64 %0, %0, %2, p;}" : "+d"(a[k]) : "d"(b), "d"(c));
      if (OP == DSETP_ONLY)
        asm volatile("{.reg .pred p; .reg .s32 q; setp.lt.f64 p, %0, %1; selp.s32 q, 1, 0, p; add.s32 %2, %2, q;}"
                     : "+d"(a[k])
                     : "d"(b), "r"(ia[k]));
      if (OP == RCP64) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a[k]));
      if (OP == RSQ64) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(a[k]));
      if (OP == FMA_IMAD) {
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(b), "d"(c));
        asm volatile("mad.lo.s32 %0, %0, 3, 7;" : "+r"(ia[k]));
      }
      if (OP == FMA_2INT) {
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(b), "d"(c));
        asm volatile("mad.lo.s32 %0, %0, 3, 7;" : "+r"(ia[k]));
        asm volatile("xor.b32 %0, %0, 0x5a5a;" : "+r"(ia[k]));
      }
      if (OP == FFMA32) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(fa[k]) : "f"((float)b), "f"((float)c));
      if (OP == IMAD32) asm volatile("mad.lo.s32 %0, %0, %1, 7;" : "+r"(ia[k]) : "r"((int)idx));
      if (OP == LDS64) {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(sm + ((idx + k * 64) & 2047))));
        a[k] += 0.0 * v;  // keeps the load live; the add is part of the per-step cost
        asm volatile("" : "+d"(a[k]));
      }
      if (OP == LDS128) {
        double v0, v1;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                     : "=d"(v0), "=d"(v1)
                     : "r"((unsigned)__cvta_generic_to_shared(sm + ((idx + k * 64) & 2046))));
        a[k] += 0.0 * v0 + 0.0 * v1;
        asm volatile("" : "+d"(a[k]));
      }
      if (OP == SHFL64) {
        a[k] = __shfl_xor_sync(0xffffffffu, a[k], 1 + (k & 7));
      }
    }
  }
  long long t1 = clock64();
  double s = 0.0;
  int is = 0;
  float fs = 0.f;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    s += a[k];
    is += ia[k];
    fs += fa[k];
  }
  if (s == 1234.5678 || is == 123456789 || fs == 1234.5f) out[blockIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
static void run(int nsm, double clk_ghz_hint) {
  const int occ = 4;  // 4 x 256 threads per SM = 32 warps
  const int grid = nsm * occ;
  double* out;
  long long* clk;
  CK(cudaMalloc(&out, grid * sizeof(double)));
  CK(cudaMalloc(&clk, grid * sizeof(long long)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int w = 0; w < 2; ++w) tput<OP><<<grid, 256>>>(out, clk, 1.000001, 0);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  tput<OP><<<grid, 256>>>(out, clk, 1.000001, 0);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  long long* h = (long long*)malloc(grid * sizeof(long long));
  CK(cudaMemcpy(h, clk, grid * sizeof(long long), cudaMemcpyDeviceToHost));
  double cmax = 0;
  for (int i = 0; i < grid; ++i) cmax = h[i] > cmax ? h[i] : cmax;
  const double lane_ops = (double)grid * 256 * CH * ITER * kOpsPerStep[OP];
  const double per_s = lane_ops / (ms * 1e-3);
  // per SM per clock: the SM's 4 CTAs ran concurrently (occupancy 4), so one CTA's clock span
  // covers the SM's work of 4 CTAs
  const double per_clk_sm = (double)occ * 256 * CH * ITER * kOpsPerStep[OP] / cmax;
  // latency: one warp, one chain
  tput<OP><<<1, 32>>>(out, clk, 1.000001, 1);
  CK(cudaDeviceSynchronize());
  long long l;
  CK(cudaMemcpy(&l, clk, sizeof(long long), cudaMemcpyDeviceToHost));
  const double lat = (double)l / ITER;
  printf("{\"op\": \"%s\", \"lane_ops_per_s\": %.4e, \"lane_ops_per_clk_per_sm\": %.2f, \"kernel_ms\": %.3f, "
         "\"eff_clock_ghz\": %.3f, \"dep_latency_clk\": %.1f}\n",
         kName[OP], per_s, per_clk_sm, ms, cmax / (ms * 1e-3) / 1e9, lat);
  fflush(stdout);
  free(h);
  CK(cudaFree(out));
  CK(cudaFree(clk));
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, p.multiProcessorCount, p.major, p.minor);
  const int n = p.multiProcessorCount;
  run<DFMA>(n, 0);
  run<DADD>(n, 0);
  run<DMUL>(n, 0);
  run<DMINSEL>(n, 0);
  run<DSETP_ONLY>(n, 0);
  run<RCP64>(n, 0);
  run<RSQ64>(n, 0);
  run<FMA_IMAD>(n, 0);
  run<FMA_2INT>(n, 0);
  run<FFMA32>(n, 0);
  run<IMAD32>(n, 0);
  run<LDS64>(n, 0);
  run<LDS128>(n, 0);
  run<SHFL64>(n, 0);
  return 0;
}
