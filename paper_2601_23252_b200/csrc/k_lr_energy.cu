// A1 for Bayesian logistic regression: batched energies on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA).
//
//   E(theta_p) = sum_{r < N} softplus(a_pr) - y_r a_pr,   a = X theta_p
//
// The logits are a dense contraction [P x d] . [d x N], so they run on the
// tensor cores: X is stored bf16-exact and each probe is
// split into three bf16 terms theta = hi + mid + lo (24 significant bits), so
// the three bf16 products accumulate in fp32 to fp32-level logits.
// Orientation: M = probes (one TMEM lane = one probe), N = data rows, K = d
// (padded to 112 = 7 UMMA k-steps of 16).  A CTA keeps its 128 probes (3 splits
// x 2 swizzle atoms, 96 KB) resident in shared memory and streams tiles of 128
// data rows through a 3-stage TMA ring; the MMA warp accumulates each tile into
// one of four TMEM buffers (4 x 128 columns) while the four epilogue warps
// drain the previous one: each thread owns one probe row, so softplus and the
// row sum happen in registers with no cross-lane reduction.  The grid is
// (probe tiles) x (data splits); split partial sums are written to
// partial[split][probe] and summed in a fixed order by the consumer, so the
// energies are deterministic.
#include "nss_internal.cuh"
#include "tc_ptx.cuh"

namespace nss {

namespace {

constexpr int BM = 128;          // probes per CTA (UMMA M)
constexpr int BN = 128;          // data rows per tile (UMMA N)
constexpr int KSTEPS = 7;        // K = 112 >= d
constexpr int kStages = 3;       // TMA ring depth for X tiles
constexpr int kAcc = 4;          // TMEM accumulator buffers (4 x 128 columns)
constexpr int kAtom = BM * 128;  // bytes of one [128 rows x 128 B] swizzle-128B region
constexpr int kSmemA = 3 * 2 * kAtom;            // 3 splits x 2 k-blocks
constexpr int kSmemB = kStages * 2 * kAtom;      // stages x 2 k-blocks
constexpr int kThreads = 192;                    // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue

struct __align__(8) Bars {
  uint64_t a_full;
  uint64_t full[kStages], empty[kStages];
  uint64_t tfull[kAcc], tempty[kAcc];
  uint32_t tmem_base;
};

__device__ __forceinline__ float softplus_mufu(float a) {
  // max(a, 0) + log(1 + e^-|a|) with the MUFU ex2 / lg2 units
  const float t = exp2f(-fabsf(a) * 1.4426950408889634f);
  return fmaxf(a, 0.f) + 0.6931471805599453f * __log2f(1.f + t);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_lr_energy(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const float *y,
                float *partial, const int *n_probe_ptr, int *reset_counter, int p_stride, int n_data, int n_tiles,
                int tiles_per_split) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + kSmemA;
  Bars *bars = reinterpret_cast<Bars *>(smem + kSmemA + kSmemB);

  if (reset_counter && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *reset_counter = 0;
  const int n_probe = *n_probe_ptr;
  const int m0 = blockIdx.x * BM;
  if (m0 >= n_probe) return;  // uniform per CTA, before any barrier or TMEM use
  const int t_begin = blockIdx.y * tiles_per_split;
  const int t_end = min(n_tiles, t_begin + tiles_per_split);
  const int nt = t_end - t_begin;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tc::mbar_init(&bars->a_full, 1);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&bars->full[s], 1);
      tc::mbar_init(&bars->empty[s], 1);
    }
    for (int a = 0; a < kAcc; ++a) {
      tc::mbar_init(&bars->tfull[a], 1);
      tc::mbar_init(&bars->tempty[a], 4);  // the four epilogue warps
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kAcc * BN>(&bars->tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0 && lane == 0 && nt > 0) {
    // ---------------- TMA producer ----------------
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    tc::mbar_arrive_expect_tx(&bars->a_full, kSmemA);
    for (int s = 0; s < 3; ++s)
      for (int kb = 0; kb < 2; ++kb)
        tc::tma_load_2d(sA + (s * 2 + kb) * kAtom, &tmA, &bars->a_full, kb * 64, s * p_stride + m0);
    for (int i = 0; i < nt; ++i) {
      const int st = i % kStages;
      if (i >= kStages) tc::mbar_wait(&bars->empty[st], ((i / kStages) - 1) & 1);
      tc::mbar_arrive_expect_tx(&bars->full[st], 2 * kAtom);
      const int row0 = (t_begin + i) * BN;
      for (int kb = 0; kb < 2; ++kb) tc::tma_load_2d(sB + (st * 2 + kb) * kAtom, &tmB, &bars->full[st], kb * 64, row0);
    }
  } else if (warp == 1 && lane == 0 && nt > 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, BN);
    tc::mbar_wait(&bars->a_full, 0);
    tc::tc_fence_after();
    for (int i = 0; i < nt; ++i) {
      const int st = i % kStages, acc = i % kAcc;
      if (i >= kAcc) tc::mbar_wait(&bars->tempty[acc], ((i / kAcc) - 1) & 1);
      tc::mbar_wait(&bars->full[st], (i / kStages) & 1);
      tc::tc_fence_after();
      const uint32_t d_tmem = tmem + acc * BN;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
#pragma unroll
        for (int ks = 0; ks < KSTEPS; ++ks) {
          const int kb = ks >> 2, koff = (ks & 3) * 32;  // 16 bf16 = 32 B per k-step
          const uint64_t ad = tc::umma_desc_sw128(sA + (s * 2 + kb) * kAtom + koff);
          const uint64_t bd = tc::umma_desc_sw128(sB + (st * 2 + kb) * kAtom + koff);
          tc::umma_f16(d_tmem, ad, bd, idesc, (s | ks) != 0);
        }
      }
      tc::umma_commit(&bars->empty[st]);  // X tile consumed
      tc::umma_commit(&bars->tfull[acc]);  // accumulator ready
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: one probe row per thread ----------------
    const int quarter = warp & 3;  // TMEM lanes this warp may access
    const int row = quarter * 32 + lane;
    double e_sum = 0.0;
    for (int i = 0; i < nt; ++i) {
      const int acc = i % kAcc;
      tc::mbar_wait(&bars->tfull[acc], (i / kAcc) & 1);
      tc::tc_fence_after();
      const int col0 = (t_begin + i) * BN;
      float part = 0.f;
#pragma unroll
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tc::tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c, v);
        if (c + 32 == BN) {  // all loads of this buffer done: release it to the MMA warp
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&bars->tempty[acc]);
        }
        const float4 *y4 = reinterpret_cast<const float4 *>(y + col0 + c);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 yy = __ldg(y4 + q);
          const float yv[4] = {yy.x, yy.y, yy.z, yy.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cc = c + 4 * q + u;
            const float a = v[4 * q + u];
            const float t = softplus_mufu(a) - yv[u] * a;
            part += (col0 + cc < n_data) ? t : 0.f;
          }
        }
      }
      e_sum += static_cast<double>(part);
    }
    if (m0 + row < n_probe) partial[static_cast<long long>(blockIdx.y) * p_stride + m0 + row] = static_cast<float>(e_sum);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kAcc * BN>(tmem);
}

}  // namespace

size_t lr_energy_smem() { return kSmemA + kSmemB + sizeof(Bars) + 1024; }

void launch_lr_energy(const CUtensorMap &tmA, const CUtensorMap &tmB, const float *y, float *partial,
                      const int *n_probe, int *reset_counter, int p_stride, int max_probe, int n_data, int n_splits,
                      const LaunchCtx &lc) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lr_energy, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lr_energy_smem()));
    attr = true;
  }
  NSS_PIN_CARVEOUT(k_lr_energy);
  const int n_tiles = (n_data + BN - 1) / BN;
  const int tps = (n_tiles + n_splits - 1) / n_splits;
  dim3 grid((max_probe + BM - 1) / BM, n_splits);
  k_lr_energy<<<grid, kThreads, lr_energy_smem(), lc.stream>>>(tmA, tmB, y, partial, n_probe, reset_counter, p_stride,
                                                              n_data, n_tiles, tps);
  ++*lc.launch_counter;
}

}  // namespace nss
