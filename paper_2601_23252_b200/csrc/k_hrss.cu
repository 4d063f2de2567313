// A6 mutate / A7 replace / A1 energies: Hit-and-Run Slice Sampling chains
// and the prior draws of nss_init (R-20).
//
// One warp per chain.  Coordinates are spread over the lanes (lane l holds
// coordinates l, l+32, ...; NPL = ceil(d/32) registers), so x' = x + t v is one
// FMA per lane, energies are warp-cooperative (lane-partial sums + xor-shuffle
// reduction) and every slice decision is warp-uniform: no intra-warp divergence
// in the step-out / shrink loops, the cost of uneven chains is paid as a tail
// across warps instead.  The whitening factor L and the
// energy parameters are staged once per CTA in shared memory; the direction's
// normals are staged per warp.  Every random number comes from the counter-based
// Philox stream (iter, dest gid, HRSS, step), so a chain's result does not
// depend on where or when it runs.
#include "energy.cuh"

namespace nss {

namespace {

struct Probe {
  float e;
  float lp;
};

// WPC warps per chain: 2 (or 4) for the correlated Gaussian at large d (the
// energy rows split over the warps, corr_energy_split / corr_energy_split4),
// else 1.  Every warp of a
// chain runs the same control flow on the same values; warp 0 writes.
template <int NPL, int KIND, int WPC>
__global__ void __launch_bounds__(256) k_hrss(RunDev r, PriorDev pr, EnergyDev en) {
  extern __shared__ float sm[];
  __shared__ int sh_flag;
  __shared__ float sh_red[8 * 4];
  __shared__ float sh_red4[WPC == 4 ? 2 : 1][WPC == 4 ? 16 * 32 + 4 : 1];  // corr_energy_split4 slots per chain
  const int d = r.d, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = (blockDim.x >> 5) / WPC;
  const int sub = wib % WPC, cib = wib / WPC;  // warp within the chain, chain within the block
  const int ldl = odd_stride(d);
  const bool stage_l = r.Vpre == nullptr;  // L only for in-chain directions
  float *sL = sm;
  float *sP = sL + (stage_l ? d * ldl : 0);
  const int npar = energy_param_floats(KIND, d, en.n_comp);
  float *sZ = sP + npar + wib * (2 * NPL * 32);
  float *sY = sZ + NPL * 32;
  if (threadIdx.x == 0) sh_flag = (r.st->terminated || r.st->error || r.st->finalised) ? 1 : 0;
  if (stage_l)
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
      int i = e / d, j = e - i * d;
      sL[i * ldl + j] = r.L[i * r.dp + j];
    }
  ESm es;
  stage_energy(en, sP, es);
  __syncthreads();
  if (sh_flag) return;
  const int2 cr = chain_range(r);
  const int c = cr.x + blockIdx.x * wpb + cib;
  if (c >= cr.y) return;  // uniform over the chain's warps
  float *wred = sh_red + cib * 4;
  int epar = 0;
  (void)wred;
  (void)epar;

  DevState *st = r.st;
  const uint32_t it = static_cast<uint32_t>(st->iter)  /* set by the select kernel */;
  const int s = r.cdest[c];
  const int par = r.cpar[c];
  const float e_star = st->e_star;
  const float w = st->width;
  const int p = r.p;
  const bool tempered = r.tempered != 0;                   // F3: slice of Pi exp(-beta E)
  const float beta = tempered ? static_cast<float>(st->smc_beta) : 0.f;
  const bool euclid = r.dir_norm == NSS_DIR_EUCLIDEAN;
  const int h = 2 * ((d + 1) / 2);           // first non-normal draw index
  const int nblk_norm = h >> 2;              // Philox blocks fully made of normals
  const int nblk_all = (h + 3) >> 2;         // blocks touching the normals

  float pa[NPL], pb[NPL];
  load_prior_lane<NPL>(pr, lane, d, pa, pb);
  float x[NPL], v[NPL], xp[NPL];
  const float *xs = start_row(r, par);
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    x[t] = i < d ? xs[i] : 0.f;
  }
  float e = start_e(r, par);
  bool dummy;
  float lp = prior_logp<NPL>(x, pr, pa, pb, lane, d, dummy);

  unsigned long long n_probe = 0, n_eval = 0, n_exp = 0, n_shr = 0, n_null = 0;

  for (int j = 0; j < p; ++j) {
    if (r.Vpre) {
      // ---- direction precomputed for this (chain, step) by k_dirs ----
      const float *vr = r.Vpre + (static_cast<long long>(c - cr.x) * p + j) * r.dp;
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        const int i = lane + 32 * t;
        v[t] = i < d ? __ldg(vr + i) : 0.f;
      }
    } else {
    // ---- direction v = L z / |z| (Mahalanobis, R-6) or L z / |L z| ----
    for (int b = lane; b < nblk_all; b += 32) {
      uint4 u4 = philox_block(r, it, s, kPhaseHrss, j, b);
      float u0 = u01(u4.x), u1 = u01(u4.y), u2 = u01(u4.z), u3 = u01(u4.w);
      float r0 = sqrtf(-2.f * logf(u0)), r1 = sqrtf(-2.f * logf(u2));
      float s0, c0, s1, c1;
      sincospif(2.f * u1, &s0, &c0);
      sincospif(2.f * u3, &s1, &c1);
      const int i0 = 4 * b;
      if (i0 < d) sZ[i0] = r0 * c0;
      if (i0 + 1 < d) sZ[i0 + 1] = r0 * s0;
      if (b < nblk_norm) {  // the partial last block carries u_h, u_b in words 2, 3
        if (i0 + 2 < d) sZ[i0 + 2] = r1 * c1;
        if (i0 + 3 < d) sZ[i0 + 3] = r1 * s1;
      }
    }
    __syncwarp();
    float zz = 0.f, vv = 0.f;
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      float acc = 0.f;
      if (i < d) {
        const float zi = sZ[i];
        zz = fmaf(zi, zi, zz);
        const float *row = sL + i * ldl;
        for (int m = 0; m <= i; ++m) acc = fmaf(row[m], sZ[m], acc);
      }
      v[t] = acc;
      vv = fmaf(acc, acc, vv);
    }
    const float nrm = sqrtf(warp_sum(euclid ? vv : zz));
    const float inv = 1.f / nrm;
#pragma unroll
    for (int t = 0; t < NPL; ++t) v[t] *= inv;
    __syncwarp();
    }

    // ---- slice height and initial bracket (R-9) ----
    const uint4 hb = philox_block(r, it, s, kPhaseHrss, j, h >> 2);
    const float u_h = u01(word(hb, h & 3));
    const float u_b = u01(word(hb, (h + 1) & 3));
    const float log_y = (tempered ? fmaf(-beta, e, lp) : lp) + logf(u_h);
    float lft = -w * u_b;
    float rgt = lft + w;

    Probe pr_last{0.f, 0.f};
    // in(t): x + t v in the support, log Pi >= log y, E < E*  (R-2, R-11)
    auto in_slice = [&](float tt) -> bool {
      ++n_probe;
#pragma unroll
      for (int t = 0; t < NPL; ++t) xp[t] = fmaf(tt, v[t], x[t]);
      bool inside;
      float lpp = prior_logp<NPL>(xp, pr, pa, pb, lane, d, inside);
      if (!inside || (!tempered && !(lpp >= log_y))) return false;
      float ep;
      if constexpr (WPC == 4 && KIND == NSS_E_CORR_GAUSS) {
        ep = es.tri ? corr_energy_split4<NPL>(xp, en, es, sY - sub * (2 * NPL * 32), sh_red4[cib], lane, sub, 1 + cib)
                    : warp_energy<NPL, KIND>(xp, en, es, sY, lane);
      } else if constexpr (WPC == 2 && KIND == NSS_E_CORR_GAUSS) {
        ep = es.tri ? corr_energy_split<NPL>(xp, en, es, sY - sub * (2 * NPL * 32), wred, lane, sub, 1 + cib, epar)
                    : warp_energy<NPL, KIND>(xp, en, es, sY, lane);
      } else {
        ep = warp_energy<NPL, KIND>(xp, en, es, sY, lane);
      }
      ++n_eval;
      if (isnan(ep)) {
        if (lane == 0) raise_error(st, NSS_ERR_NAN);
        return false;
      }
      pr_last.e = ep;
      pr_last.lp = lpp;
      return tempered ? (fmaf(-beta, ep, lpp) >= log_y) : (ep < e_star);
    };

    // ---- linear stepping-out, capped per side (R-10) ----
    // endpoint m is L0 - m w (R0 + m w) with one rounding, as in k_hrss_lane.cu
    int nl = 0, nr = 0;
    const float l0 = lft, r0 = rgt;
    while (nl < r.max_stepout && in_slice(lft)) { ++nl; lft = fmaf(-static_cast<float>(nl), w, l0); }
    while (nr < r.max_stepout && in_slice(rgt)) { ++nr; rgt = fmaf(static_cast<float>(nr), w, r0); }

    // ---- shrinkage, capped; null move at the cap (R-12/R-13) ----
    int ns = 0, acc = 0;
    int cached_blk = -1;
    uint4 cb = make_uint4(0, 0, 0, 0);
    for (int i = 0; i < r.max_shrink; ++i) {
      const int q = h + 2 + i;
      if ((q >> 2) != cached_blk) {
        cached_blk = q >> 2;
        cb = philox_block(r, it, s, kPhaseHrss, j, cached_blk);
      }
      const float u = u01(word(cb, q & 3));
      const float tt = fmaf(u, rgt - lft, lft);
      ++ns;
      if (in_slice(tt)) {
#pragma unroll
        for (int t = 0; t < NPL; ++t) x[t] = xp[t];
        e = pr_last.e;
        lp = pr_last.lp;
        acc = 1;
        break;
      }
      if (tt < 0.f) lft = tt; else rgt = tt;
    }
    n_exp += nl + nr;
    n_shr += ns;
    n_null += acc ? 0 : 1;
    if (lane == 0 && sub == 0)
      r.counts[static_cast<long long>(c) * p + j] =
          static_cast<uint32_t>(nl) | (static_cast<uint32_t>(nr) << 8) | (static_cast<uint32_t>(ns) << 16) |
          (static_cast<uint32_t>(acc) << 24);
  }

  // ---- replace ----
  if (sub != 0) return;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    if (i < d) r.X[static_cast<long long>(s) * r.dp + i] = x[t];
  }
  if (lane == 0) {
    r.E[s] = e;
    if (par != s) r.birth[s] = e_star;  // a moved survivor (F4) keeps its birth level
    atomicAdd(&st->probes, n_probe);
    atomicAdd(&st->evals, n_eval);
    atomicAdd(&st->expansions, n_exp);
    atomicAdd(&st->shrinks, n_shr);
    atomicAdd(&st->nulls, n_null);
  }
}

// Directions of every (chain, step) of the iteration at once (large d), over
// the whole GPU instead of serially inside each chain:
//   V[(c - c0) p + j] = L z / |z| (Mahalanobis, R-6) or L z / |L z|,
// z the same fp32 normals of stream (iter, dest, HRSS, j) the in-chain
// direction draws.  The products L z run on the fp64 tensor cores
// (mma.sync m8n8k4 = DMMA; fp32 inputs are exact in fp64, products exact,
// sums in fp64) and each component is rounded to fp32 once, after the
// normalisation: closer to the oracle's fp64 than the fp32 FMA chain of the
// in-chain path (d <= 32).  One warp takes 8 directions at a time (the DMMA M
// rows); n-tiles of 8 rows of L (N), k-steps of 4 columns (K), only the
// k-steps at or left of the diagonal (L lower triangular).  L is staged once
// per CTA in fp64 (stride = 4 mod 16 doubles: conflict-free fragments),
// the warp's normals in an 8-row fp64 panel; persistent grid, one CTA per SM.
constexpr int kDirRows = 8;  // directions per warp pass (DMMA M)

__host__ __device__ constexpr int dir_ld(int K) { return ((K + 11) / 16) * 16 + 4; }  // >= K, = 4 mod 16

template <int NT>  // n-tiles of 8 rows held in registers: d <= 8 NT
__global__ void __launch_bounds__(512, 1) k_dirs(RunDev r, float *V) {
  extern __shared__ double smd[];
  __shared__ int sh_flag;
  const int d = r.d, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int nt = (d + 7) >> 3, K = 8 * nt, ld = dir_ld(K);
  double *sL = smd;                                 // K x ld: L[i][m], zero outside the d x d lower triangle
  double *sZ = smd + K * ld + wib * kDirRows * ld;  // this warp's 8 x ld panel of normals
  if (threadIdx.x == 0) sh_flag = (r.st->terminated || r.st->error || r.st->finalised) ? 1 : 0;
  for (int e = threadIdx.x; e < K * ld; e += blockDim.x) {
    const int i = e / ld, m = e - i * ld;
    sL[e] = (i < d && m <= i) ? static_cast<double>(r.L[i * r.dp + m]) : 0.0;
  }
  for (int e = lane; e < kDirRows * ld; e += 32) sZ[e] = 0.0;  // columns >= d stay zero
  __syncthreads();
  if (sh_flag) return;
  const int p = r.p;
  const int2 cr = chain_range(r);
  const long long work = static_cast<long long>(cr.y - cr.x) * p;
  const uint32_t it = static_cast<uint32_t>(r.st->iter);
  const bool euclid = r.dir_norm == NSS_DIR_EUCLIDEAN;
  const int h = 2 * ((d + 1) / 2);
  const int nblk_norm = h >> 2, nblk_all = (h + 3) >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  const long long groups = (work + kDirRows - 1) / kDirRows;
  for (long long g = static_cast<long long>(blockIdx.x) * wpb + wib; g < groups;
       g += static_cast<long long>(gridDim.x) * wpb) {
    // the group's directions: lanes 0..7 resolve (chain, step, dest) once
    int my_s = 0, my_j = 0, my_real = 0;
    if (lane < kDirRows) {
      const long long q = g * kDirRows + lane;  // (c - c0) p + j
      if (q < work) {
        const long long cq = q / p;
        my_s = r.cdest[cr.x + static_cast<int>(cq)];
        my_j = static_cast<int>(q - cq * p);
        my_real = 1;
      }
    }
    // the normals (row k of the panel): lane -> direction k = lane & 7, blocks (lane >> 3) + 4 t
    {
      const int k = lane & 7;
      const int sk = __shfl_sync(0xffffffffu, my_s, k), jk = __shfl_sync(0xffffffffu, my_j, k);
      const bool realk = __shfl_sync(0xffffffffu, my_real, k) != 0;
      for (int b = lane >> 3; b < nblk_all; b += 4) {
        float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
        if (realk) {
          const uint4 u4 = philox_block(r, it, sk, kPhaseHrss, jk, b);
          const float u0 = u01(u4.x), u1 = u01(u4.y), u2 = u01(u4.z), u3 = u01(u4.w);
          const float r0 = sqrtf(-2.f * logf(u0)), r1 = sqrtf(-2.f * logf(u2));
          float s0, c0, s1, c1;
          sincospif(2.f * u1, &s0, &c0);
          sincospif(2.f * u3, &s1, &c1);
          z0 = r0 * c0;
          z1 = r0 * s0;
          z2 = r1 * c1;
          z3 = r1 * s1;
        }
        const int i0 = 4 * b;
        double *zr = sZ + k * ld + i0;
        if (i0 < d) zr[0] = z0;
        if (i0 + 1 < d) zr[1] = z1;
        if (b < nblk_norm) {  // the partial last block carries u_h, u_b in words 2, 3
          if (i0 + 2 < d) zr[2] = z2;
          if (i0 + 3 < d) zr[3] = z3;
        }
      }
    }
    __syncwarp();
    // D(8 directions x 8 rows of n-tile jn) = Z(8 x K) L(rows, K)^T over the
    // k-steps at or left of the diagonal (exact trip counts, two chains)
    double acc[NT][2];
    const double *pa = sZ + gq * ld + tq;
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) {
      acc[jn][0] = acc[jn][1] = 0.0;
      if (jn < nt) {
        const double *pb = sL + (8 * jn + gq) * ld + tq;
        double e0 = 0.0, e1 = 0.0;
        for (int k4 = 0; k4 < 8 * jn + 8; k4 += 8) {
          dmma_f64(acc[jn][0], acc[jn][1], pa[k4], pb[k4]);
          dmma_f64(e0, e1, pa[k4 + 4], pb[k4 + 4]);
        }
        acc[jn][0] += e0;
        acc[jn][1] += e1;
      }
    }
    // norms of direction gq: the four lanes of the quad hold its columns / rows
    double zz = 0.0, vv = 0.0;
    for (int m = tq; m < K; m += 4) {
      const double z = sZ[gq * ld + m];
      zz = fma(z, z, zz);
    }
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) vv = fma(acc[jn][0], acc[jn][0], fma(acc[jn][1], acc[jn][1], vv));
    zz += __shfl_xor_sync(0xffffffffu, zz, 1);
    zz += __shfl_xor_sync(0xffffffffu, zz, 2);
    vv += __shfl_xor_sync(0xffffffffu, vv, 1);
    vv += __shfl_xor_sync(0xffffffffu, vv, 2);
    const double inv = 1.0 / sqrt(euclid ? vv : zz);
    const long long q = g * kDirRows + gq;
    if (q < work) {
      float *out = V + q * r.dp;
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        const int i = 8 * jn + 2 * tq;
        if (jn < nt && i + 1 < d)
          *reinterpret_cast<float2 *>(out + i) =
              make_float2(static_cast<float>(acc[jn][0] * inv), static_cast<float>(acc[jn][1] * inv));
        else if (jn < nt && i < d)
          out[i] = static_cast<float>(acc[jn][0] * inv);
      }
    }
    __syncwarp();  // the panel is rewritten by the next group
  }
}

template <int NT>
void launch_dirs_t(const RunDev &r, float *V, const LaunchCtx &lc) {
  const long long work = static_cast<long long>(r.c1 - r.c0) * r.p;
  if (work <= 0) return;
  const int K = 8 * ((r.d + 7) / 8), ld = dir_ld(K);
  const size_t l_bytes = static_cast<size_t>(K) * ld * sizeof(double);
  const size_t z_bytes = static_cast<size_t>(kDirRows) * ld * sizeof(double);
  int wpb = static_cast<int>((227 * 1024 - 1024 - l_bytes) / z_bytes);
  wpb = wpb > 16 ? 16 : wpb;
  const size_t smem = l_bytes + wpb * z_bytes;
  NSS_MAX_SMEM(k_dirs<NT>, smem);
  NSS_PIN_CARVEOUT(k_dirs<NT>);
  static int sms_[64] = {};
  const int dv = current_device();
  if (!sms_[dv]) cudaDeviceGetAttribute(&sms_[dv], cudaDevAttrMultiProcessorCount, dv);
  const long long groups = (work + kDirRows - 1) / kDirRows;
  const long long want = (groups + wpb - 1) / wpb;
  const int grid = static_cast<int>(want < sms_[dv] ? want : sms_[dv]);  // persistent: one CTA per SM
  k_dirs<NT><<<grid, wpb * 32, smem, lc.stream>>>(r, V);
  ++*lc.launch_counter;
}

// F1 constrained Gaussian random walk: one warp per
// chain, p proposals x' = x + sigma L z (sigma = c 2.38 / sqrt(d), z from the
// normals of stream (iter, s, RW, j), Metropolis on the prior with the
// uniform draw h = 2 ceil(d/2)), rejected outside E < E*; the energy is
// evaluated only when the prior test passes.  counts = {0, 0, evaluated,
// accepted}.
template <int NPL, int KIND>
__global__ void __launch_bounds__(256) k_rw(RunDev r, PriorDev pr, EnergyDev en) {
  extern __shared__ float sm[];
  __shared__ int sh_flag;
  const int d = r.d, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int ldl = odd_stride(d);
  float *sL = sm;
  float *sP = sL + d * ldl;
  const int npar = energy_param_floats(KIND, d, en.n_comp);
  float *sZ = sP + npar + wib * (2 * NPL * 32);
  float *sY = sZ + NPL * 32;
  if (threadIdx.x == 0) sh_flag = (r.st->terminated || r.st->error || r.st->finalised) ? 1 : 0;
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
    int i = e / d, j = e - i * d;
    sL[i * ldl + j] = r.L[i * r.dp + j];
  }
  ESm es;
  stage_energy(en, sP, es);
  __syncthreads();
  if (sh_flag) return;
  const int2 cr = chain_range(r);
  const int c = cr.x + blockIdx.x * wpb + wib;
  if (c >= cr.y) return;
  DevState *st = r.st;
  const uint32_t it = static_cast<uint32_t>(st->iter);
  const int s = r.cdest[c];
  const int par = r.cpar[c];
  const float e_star = st->e_star;
  const float sigma = r.rw_sigma;
  const int p = r.p;
  const int h = 2 * ((d + 1) / 2);
  const int nblk_norm = h >> 2, nblk_all = (h + 3) >> 2;
  float pa[NPL], pb[NPL];
  load_prior_lane<NPL>(pr, lane, d, pa, pb);
  float x[NPL], xp[NPL];
  const float *xs = start_row(r, par);
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    x[t] = i < d ? xs[i] : 0.f;
  }
  float e = start_e(r, par);
  bool dummy;
  float lp = prior_logp<NPL>(x, pr, pa, pb, lane, d, dummy);
  unsigned long long n_probe = 0, n_eval = 0, n_rej = 0;
  for (int j = 0; j < p; ++j) {
    for (int b = lane; b < nblk_all; b += 32) {
      uint4 u4 = philox_block(r, it, s, kPhaseRw, j, b);
      float u0 = u01(u4.x), u1 = u01(u4.y), u2 = u01(u4.z), u3 = u01(u4.w);
      float r0 = sqrtf(-2.f * logf(u0)), r1 = sqrtf(-2.f * logf(u2));
      float s0, c0, s1, c1;
      sincospif(2.f * u1, &s0, &c0);
      sincospif(2.f * u3, &s1, &c1);
      const int i0 = 4 * b;
      if (i0 < d) sZ[i0] = r0 * c0;
      if (i0 + 1 < d) sZ[i0 + 1] = r0 * s0;
      if (b < nblk_norm) {
        if (i0 + 2 < d) sZ[i0 + 2] = r1 * c1;
        if (i0 + 3 < d) sZ[i0 + 3] = r1 * s1;
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      float acc = 0.f;
      if (i < d) {
        const float *row = sL + i * ldl;
        for (int m = 0; m <= i; ++m) acc = fmaf(row[m], sZ[m], acc);
      }
      xp[t] = fmaf(sigma, acc, x[t]);
    }
    __syncwarp();
    const uint4 hb = philox_block(r, it, s, kPhaseRw, j, h >> 2);
    const float u = u01(word(hb, h & 3));
    ++n_probe;
    bool inside;
    const float lpp = prior_logp<NPL>(xp, pr, pa, pb, lane, d, inside);
    int evaluated = 0, accepted = 0;
    if (inside && logf(u) < lpp - lp) {
      const float ep = warp_energy<NPL, KIND>(xp, en, es, sY, lane);
      evaluated = 1;
      ++n_eval;
      if (isnan(ep)) {
        if (lane == 0) raise_error(st, NSS_ERR_NAN);
      } else if (ep < e_star) {
        accepted = 1;
#pragma unroll
        for (int t = 0; t < NPL; ++t) x[t] = xp[t];
        e = ep;
        lp = lpp;
      }
    }
    n_rej += accepted ? 0 : 1;
    if (lane == 0)
      r.counts[static_cast<long long>(c) * p + j] =
          (static_cast<uint32_t>(evaluated) << 16) | (static_cast<uint32_t>(accepted) << 24);
  }
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    if (i < d) r.X[static_cast<long long>(s) * r.dp + i] = x[t];
  }
  if (lane == 0) {
    r.E[s] = e;
    if (par != s) r.birth[s] = e_star;
    atomicAdd(&st->probes, n_probe);
    atomicAdd(&st->evals, n_eval);
    atomicAdd(&st->nulls, n_rej);
  }
}

// Prior draws with rejection until E is finite (R-20); one warp per gid.
template <int NPL, int KIND>
__global__ void __launch_bounds__(256) k_init(RunDev r, PriorDev pr, EnergyDev en) {
  extern __shared__ float sm[];
  const int d = r.d, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int npar = energy_param_floats(KIND, d, en.n_comp);
  float *sP = sm;
  float *sY = sP + npar + wib * (NPL * 32);
  ESm es;
  stage_energy(en, sP, es);
  __syncthreads();
  const int g = blockIdx.x * wpb + wib;
  if (g >= r.n) return;
  DevState *st = r.st;
  const unsigned long long budget = 100ull * static_cast<unsigned long long>(r.n);
  float pa[NPL], pb[NPL];
  load_prior_lane<NPL>(pr, lane, d, pa, pb);
  for (uint32_t a = 0;; ++a) {
    unsigned long long used = 0;
    if (lane == 0) used = atomicAdd(&st->init_attempts, 1ull);
    used = __shfl_sync(kFull, used, 0);
    if (used >= budget) {
      if (lane == 0) raise_error(st, NSS_ERR_PRIOR_SUPPORT);
      return;
    }
    float x[NPL];
    prior_draw<NPL>(r, pr, g, a, lane, pa, pb, x);
    float e = warp_energy<NPL, KIND>(x, en, es, sY, lane);
    if (lane == 0) atomicAdd(&st->init_evals, 1ull);
    if (isnan(e)) {
      if (lane == 0) raise_error(st, NSS_ERR_NAN);
      return;
    }
    if (isfinite(e)) {
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        const int i = lane + 32 * t;
        if (i < d) r.X[static_cast<long long>(g) * r.dp + i] = x[t];
      }
      if (lane == 0) {
        r.E[g] = e;
        r.birth[g] = INFINITY;
      }
      return;
    }
  }
}

template <int NPL, int KIND, int WPC>
void launch_hrss_w(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int ldl = odd_stride(r.d);
  const int nc = r.c1 - r.c0;
  if (nc <= 0) return;
  int wpb = nc / 296;  // chains per block
  wpb = wpb < 1 ? 1 : (wpb > 8 / WPC ? 8 / WPC : wpb);
  const size_t sl = r.Vpre ? 0 : static_cast<size_t>(r.d) * ldl;
  const size_t smem = (sl + energy_param_floats(KIND, r.d, en.n_comp) +
                       static_cast<size_t>(wpb) * WPC * 2 * NPL * 32) * sizeof(float);
  NSS_MAX_SMEM((k_hrss<NPL, KIND, WPC>), smem);  // static shared memory counts against the 48 KB default too
  const int blocks = (nc + wpb - 1) / wpb;
  NSS_PIN_CARVEOUT((k_hrss<NPL, KIND, WPC>));
  k_hrss<NPL, KIND, WPC><<<blocks, wpb * WPC * 32, smem, lc.stream>>>(r, pr, en);
  ++*lc.launch_counter;
}

template <int NPL, int KIND>
void launch_hrss_t(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  if constexpr (KIND == NSS_E_CORR_GAUSS && NPL >= 2) {
    if (en.ufac) {  // factored energy: rows split over two (NSS_WPC=4: four) warps per chain
      static const bool four = getenv("NSS_WPC") && atoi(getenv("NSS_WPC")) == 4;
      if (four)
        launch_hrss_w<NPL, KIND, 4>(r, pr, en, lc);
      else
        launch_hrss_w<NPL, KIND, 2>(r, pr, en, lc);
      return;
    }
  }
  launch_hrss_w<NPL, KIND, 1>(r, pr, en, lc);
}

template <int NPL, int KIND>
void launch_rw_t(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int ldl = odd_stride(r.d);
  const int nc = r.c1 - r.c0;
  if (nc <= 0) return;
  int wpb = nc / 296;
  wpb = wpb < 1 ? 1 : (wpb > 8 ? 8 : wpb);
  const size_t smem = (static_cast<size_t>(r.d) * ldl + energy_param_floats(KIND, r.d, en.n_comp) +
                       static_cast<size_t>(wpb) * 2 * NPL * 32) * sizeof(float);
  NSS_MAX_SMEM((k_rw<NPL, KIND>), smem);  // per device; static shared memory counts against the 48 KB default too
  NSS_PIN_CARVEOUT((k_rw<NPL, KIND>));
  k_rw<NPL, KIND><<<(nc + wpb - 1) / wpb, wpb * 32, smem, lc.stream>>>(r, pr, en);
  ++*lc.launch_counter;
}

template <int NPL, int KIND>
void launch_init_t(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int wpb = 8;
  const size_t smem = (energy_param_floats(KIND, r.d, en.n_comp) + static_cast<size_t>(wpb) * NPL * 32) * sizeof(float);
  NSS_MAX_SMEM((k_init<NPL, KIND>), smem);  // per device; static shared memory counts against the 48 KB default too
  const int blocks = (r.n + wpb - 1) / wpb;
  NSS_PIN_CARVEOUT((k_init<NPL, KIND>));
  k_init<NPL, KIND><<<blocks, wpb * 32, smem, lc.stream>>>(r, pr, en);
  ++*lc.launch_counter;
}

#define NSS_DISPATCH(FN, ...)                                                     \
  do {                                                                            \
    const int npl = (r.d + 31) / 32;                                              \
    switch (en.kind) {                                                            \
      case NSS_E_FLAT: NSS_DISPATCH_NPL(FN, NSS_E_FLAT, __VA_ARGS__); break;      \
      case NSS_E_GAUSS: NSS_DISPATCH_NPL(FN, NSS_E_GAUSS, __VA_ARGS__); break;    \
      case NSS_E_MOG: NSS_DISPATCH_NPL(FN, NSS_E_MOG, __VA_ARGS__); break;        \
      case NSS_E_CORR_GAUSS: NSS_DISPATCH_NPL(FN, NSS_E_CORR_GAUSS, __VA_ARGS__); break; \
      case NSS_E_FUNNEL: NSS_DISPATCH_NPL(FN, NSS_E_FUNNEL, __VA_ARGS__); break;  \
      case NSS_E_LOGREG: NSS_DISPATCH_NPL(FN, NSS_E_LOGREG, __VA_ARGS__); break;  \
      default: break;                                                             \
    }                                                                             \
  } while (0)
#define NSS_DISPATCH_NPL(FN, KIND, ...)                   \
  switch (npl) {                                          \
    case 1: FN<1, KIND>(__VA_ARGS__); break;              \
    case 2: FN<2, KIND>(__VA_ARGS__); break;              \
    case 3: FN<3, KIND>(__VA_ARGS__); break;              \
    default: FN<4, KIND>(__VA_ARGS__); break;             \
  }

}  // namespace

void launch_dirs(const RunDev &r, const LaunchCtx &lc) {
  if (!r.Vpre) return;
  if (r.d <= 64)
    launch_dirs_t<8>(r, r.Vpre, lc);
  else if (r.d <= 96)
    launch_dirs_t<12>(r, r.Vpre, lc);
  else
    launch_dirs_t<16>(r, r.Vpre, lc);
}

bool energy_supported(const EnergyDev &en) {
  switch (en.kind) {
    case NSS_E_FLAT: case NSS_E_GAUSS: case NSS_E_MOG: case NSS_E_CORR_GAUSS: case NSS_E_FUNNEL:
    case NSS_E_LOGREG:
      return en.n_comp <= kMaxComp;
    default:
      return false;
  }
}

size_t energy_smem_bytes(const EnergyDev &en) {
  return static_cast<size_t>(energy_param_floats(en.kind, en.d, en.n_comp)) * sizeof(float);
}

// Engine choice: one probe per lane for small d and cheap energies
// (k_hrss_lane.cu), warp-cooperative energies otherwise.  RunDev::engine
// (nss_set_hrss_engine) can force either one; the tests run both.
int hrss_engine(const RunDev &r, const EnergyDev &en) {
  const bool lane_ok = lane_engine_ok(r, en);
  if (r.engine == NSS_ENGINE_WARP || !lane_ok) return 0;
  return 1;
}

void launch_hrss(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  if (r.mutation == NSS_MUT_RW) {  // F1 baseline mutation
    NSS_DISPATCH(launch_rw_t, r, pr, en, lc);
    return;
  }
  if (hrss_engine(r, en) == 1) {
    launch_hrss_lane(r, pr, en, lc);
    return;
  }
  launch_dirs(r, lc);  // large d: all directions of the iteration first (k_dirs)
  if (multi_engine_ok(r, en)) {
    launch_hrss_multi(r, pr, en, lc);
    return;
  }
  if (group_engine_ok(r, en)) {
    launch_hrss_group(r, pr, en, lc);
    return;
  }
  NSS_DISPATCH(launch_hrss_t, r, pr, en, lc);
}

void launch_init(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  NSS_DISPATCH(launch_init_t, r, pr, en, lc);
}

}  // namespace nss
