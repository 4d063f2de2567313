// fp64 pipe rates on this B200, for the C5 GP kernel:
// DFMA (vector), DMMA m8n8k4 (tensor), both at once in one SM (half the warps
// each), and the fp64 exp() the kernel-matrix generation uses.  Rates are per
// SM per clock (clock64 spans of each CTA); the grid fills every SM with two
// 256-thread CTAs, as k_gp_chains does.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fr scripts/fp64_rates.cu && /tmp/fr
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// MODE 0: every warp DFMA; 1: every warp DMMA; 2: even warps DMMA, odd warps
// DFMA; 3: every warp exp(); 4: even warps DMMA, odd warps exp()
template <int MODE>
__global__ void __launch_bounds__(256, 2) k_rate(int iters, double *out, unsigned long long *clk, unsigned long long *ops) {
  const int w = threadIdx.x >> 5;
  const bool tensor = MODE == 1 || ((MODE == 2 || MODE == 4) && (w & 1) == 0);
  double v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = 1e-3 * (threadIdx.x + j);
  __syncthreads();
  const unsigned long long t0 = clock64();
  unsigned long long n = 0;
  if (tensor) {
    double acc[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], v[j], v[(j + 1) & 7]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = acc[j][0] + acc[j][1];
    n = 8ull * iters * 512;  // flops per warp (m8n8k4: 2*8*8*4)
  } else if (MODE == 3 || MODE == 4) {
    for (int i = 0; i < iters / 8; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = exp(-v[j]) * 0.5;
    }
    n = 8ull * (iters / 8) * 32;  // exps per warp
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = fma(v[j], 0.999, 0.001);
    }
    n = 8ull * iters * 64;  // flops per warp
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += v[j];
  if (acc == 12345.0) out[0] = acc;
  if ((threadIdx.x & 31) == 0) atomicAdd(ops + (tensor ? 0 : 1), n);
  if (threadIdx.x == 0) atomicAdd(clk, t1 - t0);
}

template <int MODE>
void run(const char *name, int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  unsigned long long *c;
  cudaMalloc(&out, 8);
  cudaMallocManaged(&c, 3 * sizeof(unsigned long long));
  k_rate<MODE><<<2 * sms, 256>>>(iters, out, c, c + 1);  // warm
  cudaDeviceSynchronize();
  c[0] = c[1] = c[2] = 0;
  k_rate<MODE><<<2 * sms, 256>>>(iters, out, c, c + 1);
  cudaDeviceSynchronize();
  const double clk_cta = static_cast<double>(c[0]) / (2 * sms);  // mean CTA span
  printf("%-28s tensor %.1f  vector %.1f  per SM per clk (CTA span %.0f clk)\n", name,
         c[1] / (clk_cta * sms), c[2] / (clk_cta * sms), clk_cta);
  cudaFree(out);
  cudaFree(c);
}

int main() {
  run<0>("DFMA flops", 4096);
  run<1>("DMMA flops", 4096);
  run<2>("DMMA + DFMA (half warps)", 4096);
  run<3>("exp(double) per clk", 4096);
  run<4>("DMMA + exp (half warps)", 4096);
  return 0;
}
