// Latency microbenchmarks of the primitives the small per-iteration kernels use.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty() {}

__global__ void k_chase(const int *next, int steps, int *out) {
  int p = 0;
  for (int i = 0; i < steps; ++i) p = next[p];
  if (threadIdx.x == 0) out[0] = p;
}

__global__ void k_log64(double x0, int steps, double *out) {
  double x = x0;
  for (int i = 0; i < steps; ++i) x = log(x + 3.0);
  if (threadIdx.x == 0) out[0] = x;
}

__global__ void k_logexp64(double x0, int steps, double *out) {
  double x = x0;
  for (int i = 0; i < steps; ++i) x = log1p(-exp(-x - 1.0)) + 2.0;
  if (threadIdx.x == 0) out[0] = x;
}

__global__ void k_log32(float x0, int steps, float *out) {
  float x = x0;
  for (int i = 0; i < steps; ++i) x = logf(x + 3.f);
  if (threadIdx.x == 0) out[0] = x;
}

__global__ void k_fma32(float x0, int steps, float *out) {
  float x = x0;
  for (int i = 0; i < steps; ++i) x = fmaf(x, 0.999f, 0.001f);
  if (threadIdx.x == 0) out[0] = x;
}

__global__ void k_shfl(float x0, int steps, float *out) {
  float x = x0 + threadIdx.x;
  for (int i = 0; i < steps; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.f;
  if (threadIdx.x == 0) out[0] = x;
}

__global__ void k_sync(int steps, int *out) {
  __shared__ int s;
  for (int i = 0; i < steps; ++i) {
    if (threadIdx.x == (i & 31)) s = i;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void k_fence_atomic(int steps, unsigned *ctr) {
  for (int i = 0; i < steps; ++i) {
    __threadfence();
    if (threadIdx.x == 0) atomicAdd(ctr, 1u);
  }
}

template <class F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  int *next, *iout;
  double *dout;
  float *fout;
  unsigned *ctr;
  const int N = 1 << 20;
  cudaMalloc(&next, N * sizeof(int));
  cudaMalloc(&iout, 64);
  cudaMalloc(&dout, 64);
  cudaMalloc(&fout, 64);
  cudaMalloc(&ctr, 64);
  int *h = new int[N];
  for (int i = 0; i < N; ++i) h[i] = (int)((i * 7919LL + 104729) % N);
  cudaMemcpy(next, h, N * sizeof(int), cudaMemcpyHostToDevice);
  printf("empty kernel <<<1,32>>>           %7.2f us\n", timeit([] { k_empty<<<1, 32>>>(); }, 200));
  printf("empty kernel <<<148,256>>>        %7.2f us\n", timeit([] { k_empty<<<148, 256>>>(); }, 200));
  for (int st : {1, 10, 100}) {
    float t = timeit([&] { k_chase<<<1, 32>>>(next, st, iout); }, 100);
    printf("pointer chase %4d loads         %7.2f us  (%.0f ns/load)\n", st, t, 1000.f * t / st);
  }
  for (int st : {10, 100}) {
    float t = timeit([&] { k_log64<<<1, 32>>>(1.0, st, dout); }, 100);
    printf("fp64 log chain %4d               %7.2f us  (%.1f ns/op)\n", st, t, 1000.f * t / st);
    t = timeit([&] { k_logexp64<<<1, 32>>>(1.0, st, dout); }, 100);
    printf("fp64 log1p(-exp) chain %4d       %7.2f us  (%.1f ns/op)\n", st, t, 1000.f * t / st);
    t = timeit([&] { k_log32<<<1, 32>>>(1.f, st, fout); }, 100);
    printf("fp32 logf chain %4d              %7.2f us  (%.1f ns/op)\n", st, t, 1000.f * t / st);
  }
  {
    float t = timeit([&] { k_fma32<<<1, 32>>>(1.f, 1000, fout); }, 100);
    printf("fp32 fma chain 1000              %7.2f us  (%.2f ns/op)\n", t, 1000.f * t / 1000);
    t = timeit([&] { k_shfl<<<1, 32>>>(1.f, 1000, fout); }, 100);
    printf("shfl chain 1000                  %7.2f us  (%.2f ns/op)\n", t, 1000.f * t / 1000);
  }
  for (int th : {256, 512, 1024}) {
    float t = timeit([&] { k_sync<<<1, th>>>(100, iout); }, 100);
    printf("100 __syncthreads @%4d threads   %7.2f us  (%.1f ns/sync)\n", th, t, 1000.f * t / 100);
  }
  {
    float t = timeit([&] { k_fence_atomic<<<1, 32>>>(10, ctr); }, 100);
    printf("10 threadfence+atomicAdd         %7.2f us\n", t);
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attribute %d kHz\n", clk);
  extern int main2();
  return main2();
}

// ---- part 2: graphs and grid barriers ----
__device__ unsigned g_bar_count = 0, g_bar_gen = 0;
__device__ __forceinline__ void grid_barrier(unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = &g_bar_gen;
    const unsigned my = *gen;
    __threadfence();
    if (atomicAdd(&g_bar_count, 1u) == nblocks - 1) {
      g_bar_count = 0;
      __threadfence();
      atomicAdd(&g_bar_gen, 1u);
    } else {
      while (*gen == my) { __nanosleep(20); }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_grid_bar(int steps) {
  for (int i = 0; i < steps; ++i) grid_barrier(gridDim.x);
}

int main2() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 4; ++i) k_empty<<<148, 256, 0, s>>>();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  for (int i = 0; i < 100; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("graph of 4 empty kernels         %7.2f us per graph (%.2f per node)\n", ms * 10.f, ms * 10.f / 4);
  // stream launches of 4 for comparison
  cudaEventRecord(a, s);
  for (int i = 0; i < 100; ++i)
    for (int j = 0; j < 4; ++j) k_empty<<<148, 256, 0, s>>>();
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("4 stream launches                %7.2f us per 4 (%.2f per kernel)\n", ms * 10.f, ms * 10.f / 4);
  for (int nb : {16, 148, 296}) {
    int steps = 100;
    void *args[] = {&steps};
    cudaEventRecord(a, s);
    cudaLaunchCooperativeKernel((void *)k_grid_bar, nb, 256, args, 0, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    cudaEventElapsedTime(&ms, a, b);
    printf("grid barrier x100 @%3d CTAs      %7.2f us total (%.2f us per barrier) %s\n", nb, ms * 1000.f,
           ms * 1000.f / 100, cudaGetErrorString(e));
  }
  return 0;
}
