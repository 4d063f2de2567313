// Host side of the tensor-core logistic-regression energy (k_lr_energy.cu):
// bf16 staging of X, TMA tensor maps, bf16x3 splitting of probe points and the
// fixed-order reduction of the split partial sums.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <vector>

#include <cstdlib>

#include "lr_engine.cuh"

namespace nss {

size_t lr_energy_smem();
int lr_max_slices(int n_tiles);
void launch_lr_energy(const CUtensorMap &tmA, const CUtensorMap &tmB, float *partial, int *slices_out,
                      const int *n_probe, int *reset_counter, int p_stride, int n_data, int bn, const LaunchCtx &lc);

namespace {

__global__ void k_split3(const float *P, int ldp, const int *n_probe_ptr, int d, __nv_bfloat16 *A, int p_stride) {
  const int n_probe = *n_probe_ptr;
  const long long tot = static_cast<long long>(n_probe) * 128;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(e >> 7), k = static_cast<int>(e & 127);
    const float v = k < d ? P[static_cast<long long>(row) * ldp + k] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
    A[static_cast<long long>(row) * 128 + k] = hi;
    A[(static_cast<long long>(p_stride) + row) * 128 + k] = mid;
    A[(2ll * p_stride + row) * 128 + k] = lo;
  }
}

// E = kernel slices + theta~ . g with theta~ = hi + mid, the two bf16 terms
// the tensor cores contract (the same split as k_split3 / emit_probe)
__global__ void k_lr_reduce(const float *partial, int p_stride, const int *slices, const int *n_probe_ptr, float *E,
                            const float *P, int ldp, int d, const float *g) {
  const int n_probe = *n_probe_ptr, n_splits = *slices;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n_probe; p += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < n_splits; ++q) s += partial[static_cast<long long>(q) * p_stride + p];
    float lin = 0.f;
    for (int k = 0; k < d; ++k) {
      const float v = P[static_cast<long long>(p) * ldp + k];
      const float hi = __bfloat162float(__float2bfloat16_rn(v));
      const float mid = __bfloat162float(__float2bfloat16_rn(v - hi));
      lin = fmaf(hi + mid, g[k], lin);
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

// 2-D bf16 tensor [rows][128] (K contiguous), box {64, box_rows}, 128-byte swizzle
bool make_map(CUtensorMap *map, void *base, long long rows, unsigned box_rows = 128) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {128 * sizeof(__nv_bfloat16)};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool lr_data_bf16_exact(const double *X, long long count) {
  for (long long i = 0; i < count; ++i) {
    const float f = static_cast<float>(X[i]);
    if (static_cast<double>(f) != X[i]) return false;
    if (static_cast<double>(__bfloat162float(__float2bfloat16_rn(f))) != X[i]) return false;
  }
  return true;
}

cudaError_t lr_setup(LrEngine &L, const double *X, const double *y, long long N, int d, int max_probe) {
  L.N = N;
  L.d = d;
  L.n_tiles = static_cast<int>((N + 127) / 128);
  L.n_pad = static_cast<long long>(L.n_tiles) * 128;
  L.p_stride = ((max_probe + 127) / 128) * 128;
  L.max_probe = max_probe;
  // data slices per probe tile are chosen per round by the kernel (<= n_tiles)
  L.n_splits = lr_max_slices(L.n_tiles);
  std::vector<__nv_bfloat16> xb(static_cast<size_t>(L.n_pad) * 128, __float2bfloat16_rn(0.f));
  std::vector<double> g64(128, 0.0);
  for (long long r = 0; r < N; ++r) {
    for (int k = 0; k < d; ++k) {
      xb[r * 128 + k] = __float2bfloat16_rn(static_cast<float>(X[r * d + k]));
      g64[k] += (0.5 - y[r]) * X[r * d + k];
    }
  }
  std::vector<float> gf(128);
  for (int k = 0; k < 128; ++k) gf[k] = static_cast<float>(g64[k]);
  cudaError_t e;
  if ((e = cudaMalloc(&L.Xb, xb.size() * sizeof(__nv_bfloat16)))) return e;
  if ((e = cudaMalloc(&L.g, 128 * sizeof(float)))) return e;
  if ((e = cudaMemcpy(L.g, gf.data(), 128 * sizeof(float), cudaMemcpyHostToDevice))) return e;
  for (int q = 0; q < 2; ++q) {
    if ((e = cudaMalloc(&L.A[q], 3ull * L.p_stride * 128 * sizeof(__nv_bfloat16)))) return e;
    if ((e = cudaMemset(L.A[q], 0, 3ull * L.p_stride * 128 * sizeof(__nv_bfloat16)))) return e;
    if ((e = cudaMalloc(&L.partial[q], static_cast<size_t>(L.n_splits + 1) * L.p_stride * sizeof(float)))) return e;
    if ((e = cudaMemset(L.partial[q], 0, static_cast<size_t>(L.n_splits + 1) * L.p_stride * sizeof(float)))) return e;
  }
  if ((e = cudaMalloc(&L.slices, 2 * sizeof(int)))) return e;
  if ((e = cudaMemset(L.slices, 0, 2 * sizeof(int)))) return e;
  if ((e = cudaMemcpy(L.Xb, xb.data(), xb.size() * sizeof(__nv_bfloat16), cudaMemcpyHostToDevice))) return e;
  // data tiles of BN = 256 rows (half the operand bytes per flop of 128; rows
  // past n_pad are zero-filled by TMA); NSS_LR_BN=128 selects 128-row tiles
  L.bn = (getenv("NSS_LR_BN") && atoi(getenv("NSS_LR_BN")) == 128) ? 128 : 256;
  if (!make_map(&L.tmB, L.Xb, L.n_pad, static_cast<unsigned>(L.bn))) return cudaErrorInvalidValue;
  for (int q = 0; q < 2; ++q)
    if (!make_map(&L.tmA[q], L.A[q], 3ll * L.p_stride)) return cudaErrorInvalidValue;
  return cudaSuccess;
}

void lr_free(LrEngine &L) {
  cudaFree(L.Xb);
  cudaFree(L.g);
  cudaFree(L.slices);
  for (int q = 0; q < 2; ++q) {
    cudaFree(L.A[q]);
    cudaFree(L.partial[q]);
  }
  L = LrEngine{};
}

// E[p] for the first *n_probe rows of P (row stride ldp, fp32).
void lr_energies(const LrEngine &L, const float *P, int ldp, const int *n_probe, float *E, const LaunchCtx &lc) {
  k_split3<<<296, 256, 0, lc.stream>>>(P, ldp, n_probe, L.d, L.A[0], L.p_stride);
  launch_lr_energy(L.tmA[0], L.tmB, L.partial[0], L.slices, n_probe, nullptr, L.p_stride,
                   static_cast<int>(L.N), L.bn, lc);
  k_lr_reduce<<<(L.max_probe + 255) / 256, 256, 0, lc.stream>>>(L.partial[0], L.p_stride, L.slices, n_probe, E, P, ldp,
                                                                  L.d, L.g);
  *lc.launch_counter += 2;
}

void lr_energy_pass(const LrEngine &L, int parity, const int *n_probe, int *reset_counter, const LaunchCtx &lc) {
  launch_lr_energy(L.tmA[parity], L.tmB, L.partial[parity], L.slices + parity, n_probe, reset_counter,
                   L.p_stride, static_cast<int>(L.N), L.bn, lc);
}

}  // namespace nss
