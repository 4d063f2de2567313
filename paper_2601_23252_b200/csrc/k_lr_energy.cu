// A1 for Bayesian logistic regression: batched energies on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA).
//
//   E(theta_p) = sum_{r < N} softplus(a_pr) - y_r a_pr,   a = X theta_p
//
// The logits are a dense contraction [P x d] . [d x N], so they run on the
// tensor cores.  X is stored bf16-exact and each probe is
// split into bf16 terms theta = hi + mid (16 significant bits; the logit error
// is ~1e-5 relative per row and ~1e-6 relative on E), whose
// products accumulate in fp32 in TMEM.  Orientation: M = probes (one TMEM lane
// = one probe), N = data rows, K = d (padded to 112 = 7 UMMA k-steps of 16).
//
// Persistent, balanced schedule: the grid is one CTA per SM.  The work of a
// round -- ceil(P/128) probe tiles x T data tiles -- is cut into S slices per
// probe tile (S chosen so there are ~8 units per SM) and the units are dealt
// to the CTAs in contiguous ranges, so every SM gets the same number of tile
// pairs (+-1 unit) whatever P is.  A CTA keeps its probe tile (2 splits x 2
// swizzle atoms, 64 KB) in shared memory and reloads it only when its next
// unit belongs to another probe tile; data tiles stream through a 4-stage TMA
// ring; the MMA warp accumulates each tile into one of four TMEM buffers while
// sixteen epilogue warps drain the previous one.  Each epilogue thread owns one
// probe row: it accumulates |a| and the product of (1 + e^-|a|) (the linear part theta . g is added per row by the consumer)
// (one ex2 per element, one lg2 per 32), with no cross-lane reduction.  Unit
// sums go to partial[slice][probe] and are summed in slice order by the
// consumer, so energies are deterministic for a given P.
#include <cstdlib>

#include "nss_internal.cuh"
#include "tc_ptx.cuh"

namespace nss {

namespace {

constexpr int BM = 128;          // probes per tile (UMMA M)
constexpr int KSTEPS = 7;        // K = 112 >= d
constexpr int kSplits = 2;       // bf16 terms per probe coordinate
constexpr int kAtom = BM * 128;  // bytes of one [128 rows x 128 B] swizzle-128B region (probe tile)
constexpr int kSmemA = kSplits * 2 * kAtom;      // splits x 2 k-blocks
constexpr int kEpiWarps = 16;                    // four per TMEM lane quarter (column quarters)
constexpr int kColParts = kEpiWarps / 4;         // column parts of a tile (one per epilogue warp of a quarter)
constexpr int kThreads = 64 + 32 * kEpiWarps;    // warp 0 TMA, warp 1 MMA, warps 2.. epilogue
constexpr int kUnitsPerSM = 8;
constexpr int kMaxRing = 4;

// Data-tile width BN (UMMA N): 128 (4-stage TMA ring, 4 TMEM accumulators of
// 128 columns) or 256 (half the operand bytes per flop; 2 stages, 2
// accumulators of 256 columns, two tcgen05.ld per epilogue warp and tile).
template <int BN_>
struct LrCfg {
  static constexpr int BN = BN_;
  static constexpr int kStages = BN_ == 128 ? 4 : 2;          // TMA ring depth for X tiles
  static constexpr int kAcc = BN_ == 128 ? 4 : 2;             // TMEM accumulators (kAcc x BN = 512 columns)
  static constexpr int kAtomB = BN_ * 128;                    // one [BN rows x 128 B] swizzle-128B region
  static constexpr int kSmemB = kStages * 2 * kAtomB;         // stages x 2 k-blocks
  static constexpr int kPartCols = BN_ / kColParts;           // columns per epilogue part
  static constexpr int kChunks = kPartCols / 32;              // tcgen05.ld.32x32b.x32 per part
};

struct __align__(8) Bars {
  uint64_t a_full, a_empty;
  uint64_t full[kMaxRing], empty[kMaxRing];
  uint64_t tfull[kMaxRing], tempty[kMaxRing];
  uint32_t tmem_base;
};

struct Sched {
  int m_tiles, S, units;
  __device__ Sched(int n_probe, int n_tiles, int G) {
    m_tiles = (n_probe + BM - 1) / BM;
    int s = m_tiles > 0 ? (kUnitsPerSM * G + m_tiles - 1) / m_tiles : 1;
    S = s < 1 ? 1 : (s > n_tiles ? n_tiles : s);
    units = m_tiles * S;
  }
  __device__ void range(int cta, int G, int &u0, int &u1) const {
    u0 = static_cast<int>(static_cast<long long>(units) * cta / G);
    u1 = static_cast<int>(static_cast<long long>(units) * (cta + 1) / G);
  }
};

template <int BN_>
__global__ void __launch_bounds__(kThreads, 1)
    k_lr_energy(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                float *partial, int *slices_out, const int *n_probe_ptr, int *reset_counter, int p_stride,
                int n_data, int n_tiles) {
  using C = LrCfg<BN_>;
  constexpr int BN = C::BN, kStages = C::kStages, kAcc = C::kAcc, kPartCols = C::kPartCols;
  __shared__ double red4[4][kColParts][32];  // per lane quarter: the column parts' unit sums
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + kSmemA;
  Bars *bars = reinterpret_cast<Bars *>(smem + kSmemA + C::kSmemB);

  const int G = gridDim.x;
  const int n_probe = *n_probe_ptr;
  const Sched sch(n_probe, n_tiles, G);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (reset_counter) *reset_counter = 0;  // the next round's row counter
    *slices_out = sch.S;                    // per unit: one slice (the column parts combined on chip)
  }
  int u0, u1;
  sch.range(blockIdx.x, G, u0, u1);
  if (n_probe <= 0 || u0 >= u1) return;  // uniform per CTA, before any barrier or TMEM use
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tc::mbar_init(&bars->a_full, 1);
    tc::mbar_init(&bars->a_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&bars->full[s], 1);
      tc::mbar_init(&bars->empty[s], 1);
    }
    for (int a = 0; a < kAcc; ++a) {
      tc::mbar_init(&bars->tfull[a], 1);
      tc::mbar_init(&bars->tempty[a], kEpiWarps);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kAcc * BN>(&bars->tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    int it = 0, a_loads = 0, prev_m = -1;
    for (int u = u0; u < u1; ++u) {
      const int m = u / sch.S, s = u - m * sch.S;
      if (m != prev_m) {
        if (a_loads > 0) tc::mbar_wait(&bars->a_empty, (a_loads - 1) & 1);
        tc::mbar_arrive_expect_tx(&bars->a_full, kSmemA);
        for (int q = 0; q < kSplits; ++q)
          for (int kb = 0; kb < 2; ++kb)
            tc::tma_load_2d(sA + (q * 2 + kb) * kAtom, &tmA, &bars->a_full, kb * 64, q * p_stride + m * BM);
        ++a_loads;
        prev_m = m;
      }
      const int t0 = s * n_tiles / sch.S, t1 = (s + 1) * n_tiles / sch.S;
      for (int t = t0; t < t1; ++t, ++it) {
        const int st = it % kStages;
        if (it >= kStages) tc::mbar_wait(&bars->empty[st], ((it / kStages) - 1) & 1);
        tc::mbar_arrive_expect_tx(&bars->full[st], 2 * C::kAtomB);
        for (int kb = 0; kb < 2; ++kb)
          tc::tma_load_2d(sB + (st * 2 + kb) * C::kAtomB, &tmB, &bars->full[st], kb * 64, t * BN);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, BN);
    int it = 0, a_loads = 0, prev_m = -1;
    for (int u = u0; u < u1; ++u) {
      const int m = u / sch.S, s = u - m * sch.S;
      if (m != prev_m) {
        if (a_loads > 0) tc::umma_commit(&bars->a_empty);  // every MMA on the old probe tile issued
        tc::mbar_wait(&bars->a_full, a_loads & 1);
        tc::tc_fence_after();
        ++a_loads;
        prev_m = m;
      }
      const int t0 = s * n_tiles / sch.S, t1 = (s + 1) * n_tiles / sch.S;
      for (int t = t0; t < t1; ++t, ++it) {
        const int st = it % kStages, acc = it % kAcc;
        if (it >= kAcc) tc::mbar_wait(&bars->tempty[acc], ((it / kAcc) - 1) & 1);
        tc::mbar_wait(&bars->full[st], (it / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
#pragma unroll
        for (int q = 0; q < kSplits; ++q) {
#pragma unroll
          for (int ks = 0; ks < KSTEPS; ++ks) {
            const int kb = ks >> 2, koff = (ks & 3) * 32;  // 16 bf16 = 32 B per k-step
            const uint64_t ad = tc::umma_desc_sw128(sA + (q * 2 + kb) * kAtom + koff);
            const uint64_t bd = tc::umma_desc_sw128(sB + (st * 2 + kb) * C::kAtomB + koff);
            tc::umma_f16(d_tmem, ad, bd, idesc, (q | ks) != 0);
          }
        }
        tc::umma_commit(&bars->empty[st]);   // X tile consumed
        tc::umma_commit(&bars->tfull[acc]);  // accumulator ready
      }
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: one probe row per thread, a quarter of the columns ----------------
    const int quarter = warp & 3;             // TMEM lanes this warp may access
    const int chalf = (warp - 2) >> 2;        // column part of the tile: 0 .. kColParts-1
    const int row_in_tile = quarter * 32 + lane;
    int it = 0;
    for (int u = u0; u < u1; ++u) {
      const int m = u / sch.S, s = u - m * sch.S;
      const int t0 = s * n_tiles / sch.S, t1 = (s + 1) * n_tiles / sch.S;
      double e_sum = 0.0;
      for (int t = t0; t < t1; ++t, ++it) {
        const int acc = it % kAcc;
        tc::mbar_wait(&bars->tfull[acc], (it / kAcc) & 1);
        tc::tc_fence_after();
        const int cbase = chalf * kPartCols;
        const int col0 = t * BN + cbase;
        float v[C::kChunks][32];
#pragma unroll
        for (int ch = 0; ch < C::kChunks; ++ch)
          tc::tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + cbase + 32 * ch, v[ch]);
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bars->tempty[acc]);  // buffer fully read: release it
        // softplus(a) - y a = |a|/2 + a/2 - y a + log(1 + e^-|a|); the linear
        // part sum_r (1/2 - y_r) a_r = theta . g is added per probe row by the
        // consumer (lr_engine.cu), so per element: sum |a| and the product of
        // (1 + e^-|a|) (one ex2; one lg2 per kPartCols / 2 factors), two chains each
        float s0 = 0.f, s1 = 0.f, p0 = 1.f, p1 = 1.f;
        const int valid = n_data - col0;  // >= kPartCols except in the ragged last tile
        if (valid >= kPartCols) {
#pragma unroll
          for (int cc = 0; cc < kPartCols; ++cc) {
            const float a = v[cc >> 5][cc & 31];
            const float e = tc::ex2_approx(-fabsf(a) * 1.4426950408889634f);
            if (cc & 1) {
              p1 = fmaf(p1, e, p1);
              s1 += fabsf(a);
            } else {
              p0 = fmaf(p0, e, p0);
              s0 += fabsf(a);
            }
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < kPartCols; ++cc) {
            if (cc < valid) {  // padded data rows contribute nothing
              const float a = v[cc >> 5][cc & 31];
              const float e = tc::ex2_approx(-fabsf(a) * 1.4426950408889634f);
              if (cc & 1) {
                p1 = fmaf(p1, e, p1);
                s1 += fabsf(a);
              } else {
                p0 = fmaf(p0, e, p0);
                s0 += fabsf(a);
              }
            }
          }
        }
        // each product has <= kPartCols / 2 <= 32 factors in (1, 2]: no overflow
        e_sum += static_cast<double>(fmaf(0.6931471805599453f, __log2f(p0) + __log2f(p1), 0.5f * (s0 + s1)));
      }
      const int row = m * BM + row_in_tile;
      // the kColParts warps of a TMEM lane quarter combine their column parts
      // in shared memory (fixed order, fp64) behind a named barrier of the
      // quarter's 128 threads: one slice per unit and probe row
      red4[quarter][chalf][lane] = e_sum;
      asm volatile("bar.sync %0, %1;" ::"r"(2 + quarter), "r"(32 * kColParts) : "memory");
      if (chalf == 0 && row < n_probe) {
        double tot = 0.0;
#pragma unroll
        for (int c = 0; c < kColParts; ++c) tot += red4[quarter][c][lane];
        partial[static_cast<long long>(s) * p_stride + row] = static_cast<float>(tot);
      }
      asm volatile("bar.sync %0, %1;" ::"r"(2 + quarter), "r"(32 * kColParts) : "memory");  // red4 is reused
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kAcc * BN>(tmem);
}

template <int BN_>
size_t smem_of() { return kSmemA + LrCfg<BN_>::kSmemB + sizeof(Bars) + 1024; }

template <int BN_>
void launch_bn(const CUtensorMap &tmA, const CUtensorMap &tmB, float *partial, int *slices_out, const int *n_probe,
               int *reset_counter, int p_stride, int n_data, const LaunchCtx &lc) {
  NSS_MAX_SMEM(k_lr_energy<BN_>, smem_of<BN_>());
  NSS_PIN_CARVEOUT(k_lr_energy<BN_>);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int n_tiles = (n_data + BN_ - 1) / BN_;
  k_lr_energy<BN_><<<sms, kThreads, smem_of<BN_>(), lc.stream>>>(tmA, tmB, partial, slices_out, n_probe,
                                                                 reset_counter, p_stride, n_data, n_tiles);
  ++*lc.launch_counter;
}

}  // namespace

size_t lr_energy_smem() { return smem_of<128>() > smem_of<256>() ? smem_of<128>() : smem_of<256>(); }
int lr_energy_splits() { return kSplits; }

// slices per probe row: kColParts per data slice, at most one data slice per 128-row tile
int lr_max_slices(int n_tiles) { return kColParts * n_tiles; }

void launch_lr_energy(const CUtensorMap &tmA, const CUtensorMap &tmB, float *partial, int *slices_out,
                      const int *n_probe, int *reset_counter, int p_stride, int n_data, int bn, const LaunchCtx &lc) {
  if (bn == 256)
    launch_bn<256>(tmA, tmB, partial, slices_out, n_probe, reset_counter, p_stride, n_data, lc);
  else
    launch_bn<128>(tmA, tmB, partial, slices_out, n_probe, reset_counter, p_stride, n_data, lc);
}

}  // namespace nss
