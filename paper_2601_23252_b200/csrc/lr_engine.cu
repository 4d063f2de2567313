// Host side of the tensor-core logistic-regression energy (k_lr_energy.cu):
// fp16 staging of X (one term, or Xhi + Xlo), TMA tensor maps, fp16 hi/lo
// splitting of probe points and the fixed-order reduction of the split
// partial sums (R-28).
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <vector>

#include <cstdlib>

#include "lr_engine.cuh"

namespace nss {

size_t lr_energy_smem();
#ifdef NSS_LR_PROF
void lr_prof_init();
void lr_prof_dump();
#endif
void launch_lr_energy(const CUtensorMap &tmA, const CUtensorMap &tmB, const CUtensorMap &tmB2, double *eacc,
                      const int *n_probe, int *reset_counter, int p_stride, int n_data, int d, int bn, int xs,
                      const LaunchCtx &lc);

namespace {

// fp16 hi / lo terms of every probe coordinate (K padded to 128 with zeros);
// the rows' accumulators zeroed
__global__ void k_split2(const float *P, int ldp, const int *n_probe_ptr, int d, __half *A, int p_stride,
                         double *eacc) {
  const int n_probe = *n_probe_ptr;
  const long long tot = static_cast<long long>(n_probe) * 128;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(e >> 7), k = static_cast<int>(e & 127);
    if (k == 0) eacc[row] = 0.0;
    const float v = k < d ? P[static_cast<long long>(row) * ldp + k] : 0.f;
    const __half hi = __float2half_rn(v);
    const __half lo = __float2half_rn(v - __half2float(hi));
    A[static_cast<long long>(row) * 128 + k] = hi;
    A[(static_cast<long long>(p_stride) + row) * 128 + k] = lo;
  }
}

// E = the kernel's exact softplus sum + theta~ . g with theta~ = hi + lo, the
// two fp16 terms the tensor cores contract (the same split as k_split2 / emit_probe)
__global__ void k_lr_reduce(const double *eacc, const int *n_probe_ptr, float *E, const float *P, int ldp, int d,
                            const float *g) {
  const int n_probe = *n_probe_ptr;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n_probe; p += gridDim.x * blockDim.x) {
    const double s = eacc[p];
    float lin = 0.f;
    for (int k = 0; k < d; ++k) {
      const float v = P[static_cast<long long>(p) * ldp + k];
      const float hi = __half2float(__float2half_rn(v));
      const float lo = __half2float(__float2half_rn(v - hi));
      lin = fmaf(hi + lo, g[k], lin);
    }
    E[p] = static_cast<float>(s + lin);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp16 tensor [rows][128] (K contiguous), box {64, box_rows}, 128-byte swizzle
bool make_map(CUtensorMap *map, void *base, long long rows, unsigned box_rows = 128) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {128 * sizeof(__half)};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool lr_data_ok(const double *X, long long count, int d, bool *exact) {
  if (d > 128) return false;
  bool ex = true;
  for (long long i = 0; i < count; ++i) {
    if (!(std::fabs(X[i]) <= 65504.0)) return false;  // fp16 range (and finite)
    const float f = static_cast<float>(X[i]);
    if (ex && (static_cast<double>(f) != X[i] || static_cast<double>(__half2float(__float2half_rn(f))) != X[i]))
      ex = false;
  }
  *exact = ex;
  return true;
}

cudaError_t lr_setup(LrEngine &L, const double *X, const double *y, long long N, int d, int max_probe) {
  L.N = N;
  L.d = d;
#ifdef NSS_LR_PROF
  lr_prof_init();
#endif
  bool exact = true;
  if (!lr_data_ok(X, N * d, d, &exact)) return cudaErrorInvalidValue;
  L.xs = exact ? 1 : 2;
  // data tiles of BN = 256 rows (half the operand bytes per flop of 128; rows
  // past n_pad are zero-filled by TMA); NSS_LR_BN=128 selects 128-row tiles;
  // split data (two X terms per stage) use 128
  {
    const int want = getenv("NSS_LR_BN") ? atoi(getenv("NSS_LR_BN")) : 256;
    L.bn = L.xs == 2 ? 128 : (want == 128 || want == 160 ? want : 256);
  }
  L.n_tiles = static_cast<int>((N + L.bn - 1) / L.bn);
  L.n_pad = static_cast<long long>(L.n_tiles) * L.bn;
  L.p_stride = ((max_probe + 127) / 128) * 128;
  L.max_probe = max_probe;
  std::vector<__half> xh(static_cast<size_t>(L.n_pad) * 128, __float2half_rn(0.f)), xl;
  if (L.xs == 2) xl.assign(xh.size(), __float2half_rn(0.f));
  std::vector<double> g64(128, 0.0);
  for (long long r = 0; r < N; ++r) {
    for (int k = 0; k < d; ++k) {
      const float f = static_cast<float>(X[r * d + k]);
      const __half hi = __float2half_rn(f);
      xh[r * 128 + k] = hi;
      if (L.xs == 2) xl[r * 128 + k] = __float2half_rn(static_cast<float>(X[r * d + k] - __half2float(hi)));
      g64[k] += (0.5 - y[r]) * X[r * d + k];
    }
  }
  std::vector<float> gf(128);
  for (int k = 0; k < 128; ++k) gf[k] = static_cast<float>(g64[k]);
  cudaError_t e;
  if ((e = cudaMalloc(&L.Xb, xh.size() * sizeof(__half)))) return e;
  if ((e = cudaMemcpy(L.Xb, xh.data(), xh.size() * sizeof(__half), cudaMemcpyHostToDevice))) return e;
  if (L.xs == 2) {
    if ((e = cudaMalloc(&L.Xl, xl.size() * sizeof(__half)))) return e;
    if ((e = cudaMemcpy(L.Xl, xl.data(), xl.size() * sizeof(__half), cudaMemcpyHostToDevice))) return e;
  }
  if ((e = cudaMalloc(&L.g, 128 * sizeof(float)))) return e;
  if ((e = cudaMemcpy(L.g, gf.data(), 128 * sizeof(float), cudaMemcpyHostToDevice))) return e;
  for (int q = 0; q < 2; ++q) {
    if ((e = cudaMalloc(&L.A[q], 2ull * L.p_stride * 128 * sizeof(__half)))) return e;
    if ((e = cudaMemset(L.A[q], 0, 2ull * L.p_stride * 128 * sizeof(__half)))) return e;
    if ((e = cudaMalloc(&L.eacc[q], static_cast<size_t>(L.p_stride) * sizeof(double)))) return e;
    if ((e = cudaMemset(L.eacc[q], 0, static_cast<size_t>(L.p_stride) * sizeof(double)))) return e;
    if ((e = cudaMalloc(&L.lin[q], static_cast<size_t>(L.p_stride) * sizeof(float)))) return e;
    if ((e = cudaMemset(L.lin[q], 0, static_cast<size_t>(L.p_stride) * sizeof(float)))) return e;
  }
  if (!make_map(&L.tmB, L.Xb, L.n_pad, static_cast<unsigned>(L.bn))) return cudaErrorInvalidValue;
  if (!make_map(&L.tmB2, L.xs == 2 ? static_cast<void *>(L.Xl) : static_cast<void *>(L.Xb), L.n_pad,
                static_cast<unsigned>(L.bn)))
    return cudaErrorInvalidValue;
  for (int q = 0; q < 2; ++q)
    if (!make_map(&L.tmA[q], L.A[q], 2ll * L.p_stride)) return cudaErrorInvalidValue;
  return cudaSuccess;
}

void lr_free(LrEngine &L) {
#ifdef NSS_LR_PROF
  lr_prof_dump();
#endif
  cudaFree(L.Xb);
  cudaFree(L.Xl);
  cudaFree(L.g);
  for (int q = 0; q < 2; ++q) {
    cudaFree(L.A[q]);
    cudaFree(L.eacc[q]);
    cudaFree(L.lin[q]);
  }
  L = LrEngine{};
}

// E[p] for the first *n_probe rows of P (row stride ldp, fp32).
void lr_energies(const LrEngine &L, const float *P, int ldp, const int *n_probe, float *E, const LaunchCtx &lc) {
  k_split2<<<296, 256, 0, lc.stream>>>(P, ldp, n_probe, L.d, L.A[0], L.p_stride, L.eacc[0]);
  launch_lr_energy(L.tmA[0], L.tmB, L.tmB2, L.eacc[0], n_probe, nullptr, L.p_stride, static_cast<int>(L.N), L.d,
                   L.bn, L.xs, lc);
  k_lr_reduce<<<(L.max_probe + 255) / 256, 256, 0, lc.stream>>>(L.eacc[0], n_probe, E, P, ldp, L.d, L.g);
  *lc.launch_counter += 2;
}

void lr_energy_pass(const LrEngine &L, int parity, const int *n_probe, int *reset_counter, const LaunchCtx &lc) {
  launch_lr_energy(L.tmA[parity], L.tmB, L.tmB2, L.eacc[parity], n_probe, reset_counter, L.p_stride,
                   static_cast<int>(L.N), L.d, L.bn, L.xs, lc);
}

}  // namespace nss
