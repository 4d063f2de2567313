// Throughput of the instruction mixes the logistic-regression epilogue can
// use, per SM per clock on this B200: MUFU ex2 / lg2
// (f32 and packed f16x2), FFMA, packed FFMA2 (fma.rn.f32x2), and the
// softplus-term mixes.  Every thread runs 8 independent chains; the grid
// fills every SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pr scripts/pipe_rates.cu && /tmp/pr
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned ex2h2(unsigned x) {
  unsigned y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int MODE>
__global__ void k_rate(int iters, float *out) {
  float v[8];
  unsigned h[8];
  unsigned long long w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = -0.001f * (threadIdx.x + j);
    h[j] = 0x3c003c00u + j;
    w[j] = 0x3f8000003f800000ull + j;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) v[j] = ex2f(v[j]) - 1.0f;           // MUFU.EX2 (+ FADD)
      if (MODE == 1) v[j] = lg2f(v[j] + 2.0f);           // MUFU.LG2 (+ FADD)
      if (MODE == 2) h[j] = ex2h2(h[j]);                 // MUFU.EX2 f16x2
      if (MODE == 3) v[j] = fmaf(v[j], 0.999f, 0.001f);  // FFMA
      if (MODE == 4) w[j] = ffma2(w[j], 0x3f7fbe773f7fbe77ull, 0x3a83126f3a83126full);  // FFMA2
      if (MODE == 5) {                                    // the softplus element: |a| scale, ex2, p = p e + p, s += |a|
        const float e = ex2f(-fabsf(v[j]) * 1.4426950408889634f);
        v[j] = fmaf(v[j], e, v[j]) + fabsf(v[j]);
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += v[j] + __int_as_float(h[j]) + __int_as_float(static_cast<int>(w[j]));
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  float *out;
  cudaMalloc(&out, 4);
  const char *names[] = {"ex2.f32", "lg2.f32", "ex2.f16x2 (2 results)", "ffma", "ffma2 (2 results)", "softplus elem"};
  const int iters = 4096;
  for (int mode = 0; mode < 6; ++mode) {
    for (int threads : {256, 512, 1024}) {
      const int blocks = sms * (2048 / threads);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      auto run = [&] {
        switch (mode) {
          case 0: k_rate<0><<<blocks, threads>>>(iters, out); break;
          case 1: k_rate<1><<<blocks, threads>>>(iters, out); break;
          case 2: k_rate<2><<<blocks, threads>>>(iters, out); break;
          case 3: k_rate<3><<<blocks, threads>>>(iters, out); break;
          case 4: k_rate<4><<<blocks, threads>>>(iters, out); break;
          default: k_rate<5><<<blocks, threads>>>(iters, out); break;
        }
      };
      run();
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = static_cast<double>(blocks) * threads * iters * 8;
      const double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
      printf("%-22s threads %4d: %.3f ms, %.2f instr/clk/SM (at %.0f MHz max clock)\n", names[mode], threads, ms,
             per_clk_sm, clk / 1e3);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
