// A1 for Bayesian logistic regression: batched energies on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA).
//
//   E(theta_p) = sum_{r < N} softplus(a_pr) - y_r a_pr,   a = X theta_p
//
// The logits are a dense contraction [P x d] . [d x N], so they run on the
// tensor cores in fp16 with fp32 accumulation in TMEM (R-28): each probe is
// split into fp16 terms theta = hi + lo (22 significant bits, relative error
// <= 2^-23 like an fp32 round, fp16 range), and X is either fp16-exact (one
// term: 2 MMAs per k-step, XS = 1) or split the same way, X = Xhi + Xlo
// (XS = 2: Xhi.hi + Xhi.lo + Xlo.hi, 3 MMAs; the dropped Xlo.lo is below
// 2^-22).  Orientation: M = probes (one TMEM lane = one probe), N = data
// rows, K = d (padded to 16 ksteps, <= 128).
//
// Persistent, balanced schedule: the grid is one CTA per SM and the work of
// a round -- ceil(P/128) probe tiles x T data tiles = TP tile pairs, in
// (probe tile, data tile) order -- is cut into G contiguous ranges of
// floor/ceil(TP/G) pairs, so every SM gets the same number of tile pairs
// (+-1).  A CTA keeps its probe tile (2 splits x 2 swizzle atoms, 64 KB) in
// shared memory and reloads it when its range enters the next probe tile
// (at most a few times); data tiles stream through a TMA ring; the MMA warp
// accumulates each tile into one of the TMEM buffers while sixteen epilogue
// warps drain the previous one.  Each epilogue thread owns one probe row and a
// quarter of the columns: it accumulates |a| and the product of (1 + e^-|a|)
// (one ex2 per element, one lg2 per 32) into an fp32 value per tile, sums the
// tiles of its range in fp64 and adds that to the row's fp64 accumulator
// (which the consumer seeded with the row's linear term theta . g) with one
// atomicAdd.  Every tile value is an fp32 number >= ln 2 (or 0) and the
// totals stay below 2^28, so each fp64 addition is exact: the energies do not
// depend on the order of the additions, on the ranges, or on P -- a probe's
// energy is the same bits in any batch (the sharded runs rely on this).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "nss_internal.cuh"
#include "tc_ptx.cuh"

namespace nss {

namespace {

constexpr int BM = 128;          // probes per tile (UMMA M)
constexpr int kSplits = 2;       // fp16 terms per probe coordinate (hi, lo)
constexpr int kAtom = BM * 128;  // bytes of one [128 rows x 128 B] swizzle-128B region (probe tile)
constexpr int kSmemA = kSplits * 2 * kAtom;      // splits x 2 k-blocks
constexpr int kMaxRing = 4;
// Every NSS_LR_POLY-th column's exponential on the FMA pipe instead of the
// MUFU (0: none); measurement builds (NSS_NVCC_EXTRA=-DNSS_LR_POLY=4).
#ifndef NSS_LR_POLY
#define NSS_LR_POLY 0
#endif

// 2^x for x <= 0 on the FMA / ALU pipes only (no MUFU, no conversion): x =
// j + f with j = rint(x) by the 1.5 2^23 trick, 2^f (|f| <= 1/2) by a degree-5
// polynomial (relative error 3e-7), 2^j added to the exponent field.  x is
// clamped at -126 (2^-126 is below every term it meets).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float j = t - 12582912.f;
  const float f = x - j;
  float p = fmaf(1.32609e-3f, f, 9.67018e-3f);
  p = fmaf(p, f, 5.550712e-2f);
  p = fmaf(p, f, 0.24022224f);
  p = fmaf(p, f, 0.693147f);
  p = fmaf(p, f, 1.00000005f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) - 0x4B400000) * 8388608);
}

// Data-tile width BN (UMMA N): 128 (4 TMEM accumulators of 128 columns),
// 160 (3 accumulators: the MMA may run two tiles ahead of the epilogue; five
// 32-column parts) or 256 (half the operand bytes per flop of 128; 2
// accumulators of 256 columns, two tcgen05.ld per epilogue warp and tile).
// XS X terms per stage.
template <int BN_, int XS_>
struct LrCfg {
  static constexpr int BN = BN_;
  static constexpr int XS = XS_;
  static constexpr int kStages = (BN_ <= 160 && XS_ == 1) ? 4 : 2;  // TMA ring depth for X tiles
  static constexpr int kAcc = 512 / BN_;                      // TMEM accumulators (of the 512 columns)
  static constexpr int kAtomB = BN_ * 128;                    // one [BN rows x 128 B] swizzle-128B region
  static constexpr int kSmemB = kStages * XS_ * 2 * kAtomB;   // stages x X terms x 2 k-blocks
  static constexpr int kColParts = BN_ == 160 ? 5 : 4;        // column parts of a tile
  static constexpr int kEpi = 4 * kColParts;                  // epilogue warps: one per (TMEM lane quarter, part)
  static constexpr int kThreads = 64 + 32 * kEpi;             // warp 0 TMA, warp 1 MMA, warps 2.. epilogue
  static constexpr int kPartCols = BN_ / kColParts;           // columns per epilogue part
  static constexpr int kChunks = kPartCols / 32;              // tcgen05.ld.32x32b.x32 per part
};

#ifdef NSS_LR_PROF
// measurement builds (NSS_NVCC_EXTRA=-DNSS_LR_PROF): SM clocks summed over
// CTAs {MMA waits on X tiles, MMA waits on a free accumulator, MMA waits on
// the probe tile, epilogue waits on a full accumulator (sum over warps),
// epilogue busy (sum over warps), CTA span after the dependency wait,
// prologue up to it, tile pairs}
__device__ unsigned long long *g_lr_prof;
#endif

struct __align__(8) Bars {
  uint64_t a_full, a_empty;
  uint64_t full[kMaxRing], empty[kMaxRing];
  uint64_t tfull[kMaxRing], tempty[kMaxRing];
  uint32_t tmem_base;
};

struct Sched {
  int m_tiles, pairs;
  __device__ Sched(int n_probe, int n_tiles) {
    m_tiles = (n_probe + BM - 1) / BM;
    pairs = m_tiles * n_tiles;
  }
  __device__ void range(int cta, int G, int &p0, int &p1) const {
    p0 = static_cast<int>(static_cast<long long>(pairs) * cta / G);
    p1 = static_cast<int>(static_cast<long long>(pairs) * (cta + 1) / G);
  }
};

template <int BN_, int XS_>
__global__ void __launch_bounds__(LrCfg<BN_, XS_>::kThreads, 1)
    k_lr_energy(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmB2, double *eacc, const int *n_probe_ptr, int *reset_counter,
                int p_stride, int n_data, int n_tiles, int ksteps) {
  using C = LrCfg<BN_, XS_>;
  constexpr int BN = C::BN, kStages = C::kStages, kAcc = C::kAcc, kPartCols = C::kPartCols;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + kSmemA;
  Bars *bars = reinterpret_cast<Bars *>(smem + kSmemA + C::kSmemB);

  const int G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // prologue: nothing the preceding advance kernel writes (programmatic
  // dependent launch: it overlaps that kernel's tail)
  if (threadIdx.x == 0) {
    tc::mbar_init(&bars->a_full, 1);
    tc::mbar_init(&bars->a_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&bars->full[s], 1);
      tc::mbar_init(&bars->empty[s], 1);
    }
    for (int a = 0; a < kAcc; ++a) {
      tc::mbar_init(&bars->tfull[a], 1);
      tc::mbar_init(&bars->tempty[a], C::kEpi);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    if (XS_ == 2) tc::tma_prefetch(&tmB2);
  }
  if (warp == 1) tc::tmem_alloc<512>(&bars->tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
#ifdef NSS_LR_PROF
  const long long t_pro = clock64();
#endif
  pdl_wait();  // the probe rows and their count are complete from here
#ifdef NSS_LR_PROF
  const long long t_start = clock64();
  unsigned long long pw[3] = {0, 0, 0};
#endif
  pdl_trigger();
  const int n_probe = *n_probe_ptr;
#ifdef NSS_LR_PROF
  // launches by probe rows: bins 0, 1-127, 128-1023, 1024-4095, 4096-8191, >= 8192
  const int lr_bin = n_probe <= 0 ? 0 : n_probe < 128 ? 1 : n_probe < 1024 ? 2 : n_probe < 4096 ? 3 : n_probe < 8192 ? 4 : 5;
  if (g_lr_prof && blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(g_lr_prof + 8 + lr_bin, 1ull);
    atomicAdd(g_lr_prof + 24 + lr_bin, static_cast<unsigned long long>(n_probe > 0 ? n_probe : 0));
  }
#endif
  const Sched sch(n_probe, n_tiles);
  if (blockIdx.x == 0 && threadIdx.x == 0 && reset_counter) *reset_counter = 0;  // the next round's row counter
  int u0, u1;
  sch.range(blockIdx.x, G, u0, u1);
  if (n_probe <= 0 || u0 >= u1) {  // uniform per CTA
    if (warp == 1) tc::tmem_dealloc<512>(tmem);
    return;
  }

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int it = 0, a_loads = 0, prev_m = -1;
    for (int u = u0; u < u1; ++u, ++it) {
      const int m = u / n_tiles, t = u - m * n_tiles;
      if (m != prev_m) {
        if (a_loads > 0) tc::mbar_wait(&bars->a_empty, (a_loads - 1) & 1);
        tc::mbar_arrive_expect_tx(&bars->a_full, kSmemA);
        for (int q = 0; q < kSplits; ++q)
          for (int kb = 0; kb < 2; ++kb)
            tc::tma_load_2d(sA + (q * 2 + kb) * kAtom, &tmA, &bars->a_full, kb * 64, q * p_stride + m * BM);
        ++a_loads;
        prev_m = m;
      }
      {
        const int st = it % kStages;
        if (it >= kStages) tc::mbar_wait(&bars->empty[st], ((it / kStages) - 1) & 1);
        tc::mbar_arrive_expect_tx(&bars->full[st], XS_ * 2 * C::kAtomB);
        for (int kb = 0; kb < 2; ++kb) {
          tc::tma_load_2d(sB + ((st * XS_) * 2 + kb) * C::kAtomB, &tmB, &bars->full[st], kb * 64, t * BN);
          if (XS_ == 2)
            tc::tma_load_2d(sB + ((st * XS_ + 1) * 2 + kb) * C::kAtomB, &tmB2, &bars->full[st], kb * 64, t * BN);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = tc::idesc_f16_f32(BM, BN);
    int it = 0, a_loads = 0, prev_m = -1;
    for (int u = u0; u < u1; ++u, ++it) {
      const int m = u / n_tiles;
      if (m != prev_m) {
        if (a_loads > 0) tc::umma_commit(&bars->a_empty);  // every MMA on the old probe tile issued
#ifdef NSS_LR_PROF
        const long long ta = clock64();
#endif
        tc::mbar_wait(&bars->a_full, a_loads & 1);
#ifdef NSS_LR_PROF
        pw[2] += clock64() - ta;
#endif
        tc::tc_fence_after();
        ++a_loads;
        prev_m = m;
      }
      {
        const int st = it % kStages, acc = it % kAcc;
#ifdef NSS_LR_PROF
        const long long t0 = clock64();
#endif
        if (it >= kAcc) tc::mbar_wait(&bars->tempty[acc], ((it / kAcc) - 1) & 1);
#ifdef NSS_LR_PROF
        const long long t1 = clock64();
        pw[1] += t1 - t0;
#endif
        tc::mbar_wait(&bars->full[st], (it / kStages) & 1);
#ifdef NSS_LR_PROF
        pw[0] += clock64() - t1;
#endif
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        // (A term, X term) products: hi.Xhi, lo.Xhi (+ hi.Xlo when X is split)
#pragma unroll
        for (int q = 0; q < kSplits + XS_ - 1; ++q) {
          const int qa = q < kSplits ? q : 0, qb = q < kSplits ? 0 : 1;
          for (int ks = 0; ks < ksteps; ++ks) {
            const int kb = ks >> 2, koff = (ks & 3) * 32;  // 16 fp16 = 32 B per k-step
            const uint64_t ad = tc::umma_desc_sw128(sA + (qa * 2 + kb) * kAtom + koff);
            const uint64_t bd = tc::umma_desc_sw128(sB + ((st * XS_ + qb) * 2 + kb) * C::kAtomB + koff);
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
    double e_sum = 0.0;
    for (int u = u0; u < u1; ++u, ++it) {
      const int m = u / n_tiles, t = u - m * n_tiles;
      {
        const int acc = it % kAcc;
#ifdef NSS_LR_PROF
        const long long te = clock64();
#endif
        tc::mbar_wait(&bars->tfull[acc], (it / kAcc) & 1);
#ifdef NSS_LR_PROF
        const long long tb = clock64();
        pw[0] += tb - te;
#endif
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
        // part sum_r (1/2 - y_r) a_r = theta . g is the consumer's seed of the
        // row accumulator, so per element: sum |a| and the product of
        // (1 + e^-|a|) (one ex2; one lg2 per kPartCols / 2 factors), two chains each
        float s0 = 0.f, s1 = 0.f, p0 = 1.f, p1 = 1.f;
        const int valid = n_data - col0;  // >= kPartCols except in the ragged last tile
        if (valid >= kPartCols) {
#pragma unroll
          for (int cc = 0; cc < kPartCols; ++cc) {
            const float a = v[cc >> 5][cc & 31];
            const float e = (NSS_LR_POLY > 0 && cc % (NSS_LR_POLY > 0 ? NSS_LR_POLY : 1) == NSS_LR_POLY - 1)
                                ? ex2_poly(-fabsf(a) * 1.4426950408889634f)
                                : tc::ex2_approx(-fabsf(a) * 1.4426950408889634f);
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
        // each product has <= kPartCols / 2 <= 32 factors in (1, 2]: no
        // overflow; the tile value is >= ln 2 per column, or 0 (no column)
        e_sum += static_cast<double>(fmaf(0.6931471805599453f, __log2f(p0) + __log2f(p1), 0.5f * (s0 + s1)));
#ifdef NSS_LR_PROF
        pw[1] += clock64() - tb;
#endif
      }
      // end of this probe tile's part of the range: one exact fp64 atomic per row
      if (u + 1 == u1 || (u + 1) / n_tiles != m) {
        const int row = m * BM + row_in_tile;
        if (row < n_probe) atomicAdd(eacc + row, e_sum);
        e_sum = 0.0;
      }
    }
  }
#ifdef NSS_LR_PROF
  if (g_lr_prof) {
    if (warp == 1 && lane == 0)
      for (int q = 0; q < 3; ++q) atomicAdd(g_lr_prof + q, pw[q]);
    if (warp == 2 && lane == 0) {  // one epilogue warp
      atomicAdd(g_lr_prof + 3, pw[0]);
      atomicAdd(g_lr_prof + 4, pw[1]);
    }
  }
#endif
  tc::tc_fence_before();
  __syncthreads();
#ifdef NSS_LR_PROF
  if (g_lr_prof && threadIdx.x == 0) {
    atomicAdd(g_lr_prof + 5, static_cast<unsigned long long>(clock64() - t_start));
    atomicAdd(g_lr_prof + 6, static_cast<unsigned long long>(t_start - t_pro));
    atomicAdd(g_lr_prof + 7, static_cast<unsigned long long>(u1 - u0));
    if (blockIdx.x == 0) atomicAdd(g_lr_prof + 16 + lr_bin, static_cast<unsigned long long>(clock64() - t_pro));
  }
#endif
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

template <int BN_, int XS_>
size_t smem_of() { return kSmemA + LrCfg<BN_, XS_>::kSmemB + sizeof(Bars) + 1024; }

template <int BN_, int XS_>
void launch_bn(const CUtensorMap &tmA, const CUtensorMap &tmB, const CUtensorMap &tmB2, double *eacc,
               const int *n_probe, int *reset_counter, int p_stride, int n_data, int d,
               const LaunchCtx &lc) {
  NSS_MAX_SMEM((k_lr_energy<BN_, XS_>), (smem_of<BN_, XS_>()));
  NSS_PIN_CARVEOUT((k_lr_energy<BN_, XS_>));
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int n_tiles = (n_data + BN_ - 1) / BN_;
  launch_maybe_pdl(k_lr_energy<BN_, XS_>, dim3(sms), dim3(LrCfg<BN_, XS_>::kThreads), smem_of<BN_, XS_>(), lc.stream, tmA, tmB, tmB2,
                   eacc, n_probe, reset_counter, p_stride, n_data, n_tiles, (d + 15) / 16);
  ++*lc.launch_counter;
}

}  // namespace

size_t lr_energy_smem() { return smem_of<128, 2>(); }

#ifdef NSS_LR_PROF
static unsigned long long *h_lr_prof = nullptr;
void lr_prof_init() {
  if (h_lr_prof) return;
  cudaMallocManaged(&h_lr_prof, 32 * sizeof(unsigned long long));
  memset(h_lr_prof, 0, 32 * sizeof(unsigned long long));
  cudaMemcpyToSymbol(g_lr_prof, &h_lr_prof, sizeof(h_lr_prof));
}
void lr_prof_dump() {
  if (!h_lr_prof) return;
  cudaDeviceSynchronize();
  const unsigned long long *p = h_lr_prof;
  const double span = static_cast<double>(p[5]), epi = 1.0;
  fprintf(stderr, "lr_prof: %llu tile pairs; per CTA-span: MMA waits X %.3f, accumulator %.3f, probe tile %.3f; "
          "epilogue waits %.3f busy %.3f (per warp); prologue/span %.3f; span per tile pair %.0f clk\n",
          p[7], p[0] / span, p[1] / span, p[2] / span, p[3] / epi / span, p[4] / epi / span, p[6] / span,
          span / static_cast<double>(p[7] ? p[7] : 1));
  const char *bn[6] = {"0", "1-127", "128-1023", "1024-4095", "4096-8191", ">=8192"};
  for (int b = 0; b < 6; ++b)
    fprintf(stderr, "lr_prof rows %-9s launches %8llu  rows %12llu  CTA-0 clocks %14llu\n", bn[b], p[8 + b], p[24 + b],
            p[16 + b]);
}
#endif
int lr_energy_splits() { return kSplits; }


// bn: data-tile width (256 with one X term); xs: X terms (1 fp16-exact data, 2 split data -> bn 128)
void launch_lr_energy(const CUtensorMap &tmA, const CUtensorMap &tmB, const CUtensorMap &tmB2, double *eacc,
                      const int *n_probe, int *reset_counter, int p_stride, int n_data, int d,
                      int bn, int xs, const LaunchCtx &lc) {
  if (xs == 2)
    launch_bn<128, 2>(tmA, tmB, tmB2, eacc, n_probe, reset_counter, p_stride, n_data, d, lc);
  else if (bn == 256)
    launch_bn<256, 1>(tmA, tmB, tmB2, eacc, n_probe, reset_counter, p_stride, n_data, d, lc);
  else if (bn == 160)
    launch_bn<160, 1>(tmA, tmB, tmB2, eacc, n_probe, reset_counter, p_stride, n_data, d, lc);
  else
    launch_bn<128, 1>(tmA, tmB, tmB2, eacc, n_probe, reset_counter, p_stride, n_data, d, lc);
}

}  // namespace nss
