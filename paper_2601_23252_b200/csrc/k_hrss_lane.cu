// A6/A7 (+A1) for small dimensions (d <= 32) and cheap energies: one warp per
// chain, ONE PROBE PER LANE.
//
// HRSS is a chain of dependent slice tests, so at small d a warp-per-chain
// kernel is latency-bound: every probe waits for the previous decision.  But
// every point the sequential algorithm can visit next is known in
// advance:
//   * stepping-out endpoints are L0 - m w and R0 + m w (m = 0..cap-1);
//   * along the all-rejected path every shrink proposal is fixed too, because a
//     rejected proposal t moves the left end if t < 0 and the right end
//     otherwise (R-13): proposal i is L_i + u_i (R_i - L_i) with (L_i, R_i)
//     obtained from proposals 0..i-1.
// So the warp evaluates 16 left + 16 right endpoints in one round (lanes 0-15
// / 16-31) and kShrink shrink proposals in a second round, and takes the first
// outcome the sequential algorithm would take (ballot + ffs).  Every point is
// computed with the same fp32 operations as the sequential engine (k_hrss.cu),
// so decisions and counters are those of the sequential algorithm; only the
// number of dependent rounds changes (about 2 per step instead of ~5-7).
// Counters report the algorithm's probes, not the speculative ones, and a NaN
// raises an error only if the sequential algorithm would have evaluated it.
//
// Instruction diet (the kernel is issue-latency bound):
// coordinates are padded to a compile-time D with neutral values (zero
// direction, infinite box, zero precision) so no loop carries a predicate;
// small mixtures keep their parameters in registers; one Philox pass per step
// produces the normals, the slice height, the bracket offset and the first
// shrink uniforms, distributed by shuffles.
#include "energy.cuh"

namespace nss {

namespace {

constexpr int kRound = 16;   // stepping-out endpoints per side per round
constexpr int kShrink = 8;   // shrink proposals per round

template <int D, int KIND, int K>
struct LaneParams {
  // GAUSS: a = 1/sigma, b = -mu/sigma (u = x a + b); MOG with compile-time K: per component
  float a[K > 0 ? K : 1][D], b[K > 0 ? K : 1][D], logc[K > 0 ? K : 1];
};

template <int D, int KIND, int K>
__device__ __forceinline__ void load_params(LaneParams<D, KIND, K> &lp, const EnergyDev &en) {
  if constexpr (KIND == NSS_E_GAUSS || (KIND == NSS_E_MOG && K > 0)) {
    constexpr int KK = KIND == NSS_E_GAUSS ? 1 : K;
    // host-built padded table [K][2][32]: {1/sigma, -mu/sigma}, zeros past d
#pragma unroll
    for (int j = 0; j < KK; ++j) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        lp.a[j][i] = __ldg(en.lane_ab + j * 64 + i);
        lp.b[j][i] = __ldg(en.lane_ab + j * 64 + 32 + i);
      }
      lp.logc[j] = KIND == NSS_E_MOG ? __ldg(en.logc + j) : 0.f;
    }
  }
}

// Thread-local energy of the padded point xp.
template <int D, int KIND, int K>
__device__ __forceinline__ float lane_energy(const float (&xp)[D], const LaneParams<D, KIND, K> &P,
                                             const EnergyDev &en, const float *sA, const float *sB,
                                             const float *sC, int ldD, int d) {
  if constexpr (KIND == NSS_E_FLAT) {
    return en.c;
  } else if constexpr (KIND == NSS_E_GAUSS) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const float u = fmaf(xp[i], P.a[0][i], P.b[0][i]);
      s = fmaf(u, u, s);
    }
    return 0.5f * s + en.c;
  } else if constexpr (KIND == NSS_E_MOG && K > 0) {
    float l[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const float u = fmaf(xp[i], P.a[j][i], P.b[j][i]);
        s = fmaf(u, u, s);
      }
      l[j] = fmaf(-0.5f, s, P.logc[j]);
    }
    float m = l[0];
#pragma unroll
    for (int j = 1; j < K; ++j) m = fmaxf(m, l[j]);
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) acc += __expf(l[j] - m);
    return -(m + __logf(acc));
  } else if constexpr (KIND == NSS_E_MOG) {
    // runtime K: parameters in shared memory (a, b padded to D; logc)
    float m = -INFINITY, acc = 0.f;
#pragma unroll 2
    for (int j = 0; j < en.n_comp; ++j) {
      const float *a = sA + j * D, *b = sB + j * D;
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const float u = fmaf(xp[i], a[i], b[i]);
        s = fmaf(u, u, s);
      }
      const float l = fmaf(-0.5f, s, sC[j]);
      if (l > m) {
        acc = acc * __expf(m - l) + 1.f;
        m = l;
      } else {
        acc += __expf(l - m);
      }
    }
    return -(m + __logf(acc));
  } else if constexpr (KIND == NSS_E_FUNNEL) {
    const float y = xp[0];
    float s = 0.f;
#pragma unroll
    for (int i = 1; i < D; ++i) s = fmaf(xp[i], xp[i], s);
    const float sy = en.sigma_y, yy = y / sy;
    return 0.5f * yy * yy + logf(sy) + 0.5f * kLn2Pi + 0.5f * s * expf(-y) +
           static_cast<float>(d - 1) * 0.5f * (y + kLn2Pi);
  } else if constexpr (KIND == NSS_E_CORR_GAUSS) {
    // sA: mu padded to D; sB: precision padded to D x ldD (zeros outside d x d)
    float y[D];
#pragma unroll
    for (int i = 0; i < D; ++i) y[i] = xp[i] - sA[i];
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const float *row = sB + i * ldD;
      float py = 0.f;
#pragma unroll
      for (int m = 0; m < D; ++m) py = fmaf(row[m], y[m], py);
      q = fmaf(y[i], py, q);
    }
    return 0.5f * q + en.c;
  } else {
    return NAN;
  }
}

struct LaneProbe {
  bool pass;  // inside the support and above the slice height (energy evaluated)
  bool ok;    // pass and E < E*
  bool nan;
  float e, lp;
};

template <int D, int KIND, int K>
__device__ __forceinline__ LaneProbe lane_probe(float t, const float (&x)[D], const float (&v)[D], bool box,
                                                const float (&pa)[D], const float (&pb)[D], float log_norm,
                                                const LaneParams<D, KIND, K> &P, const EnergyDev &en,
                                                const float *sA, const float *sB, const float *sC, int ldD,
                                                int d, float log_y, float e_star) {
  float xp[D];
#pragma unroll
  for (int i = 0; i < D; ++i) xp[i] = fmaf(t, v[i], x[i]);
  LaneProbe o{false, false, false, 0.f, log_norm};
  if (box) {
    bool in = true;
#pragma unroll
    for (int i = 0; i < D; ++i) in = in && (xp[i] >= pa[i]) && (xp[i] <= pb[i]);
    o.pass = in && (log_norm >= log_y);
  } else {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const float u = (xp[i] - pa[i]) * pb[i];
      s = fmaf(u, u, s);
    }
    o.lp = fmaf(-0.5f, s, log_norm);
    o.pass = o.lp >= log_y;
  }
  if (o.pass) {
    o.e = lane_energy<D, KIND, K>(xp, P, en, sA, sB, sC, ldD, d);
    o.nan = isnan(o.e);
    o.ok = !o.nan && o.e < e_star;
  }
  return o;
}

__device__ __forceinline__ unsigned low_mask(int n) {  // bits 0..n-1
  return n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
}

template <int D, int KIND, int K>
__global__ void __launch_bounds__(256) k_hrss_lane(RunDev r, PriorDev pr, EnergyDev en) {
  extern __shared__ float sm[];
  const int d = r.d, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  constexpr int ldD = D | 1;
  constexpr bool kSmemTables = (KIND == NSS_E_MOG && K == 0) || KIND == NSS_E_CORR_GAUSS;
  // shared memory only for the runtime-K mixture and the correlated Gaussian
  float *sA = sm;
  float *sB = sA + (KIND == NSS_E_MOG ? kMaxComp * D : D);
  float *sC = sB + (KIND == NSS_E_MOG ? kMaxComp * D : D * ldD);
  if constexpr (KIND == NSS_E_MOG && K == 0) {
    for (int e = threadIdx.x; e < en.n_comp * D; e += blockDim.x) {
      const int j = e / D, i = e - j * D;
      sA[e] = en.lane_ab[j * 64 + i];
      sB[e] = en.lane_ab[j * 64 + 32 + i];
    }
    for (int j = threadIdx.x; j < en.n_comp; j += blockDim.x) sC[j] = en.logc[j];
  }
  if constexpr (KIND == NSS_E_CORR_GAUSS) {
    for (int i = threadIdx.x; i < D; i += blockDim.x) sA[i] = i < d ? en.mu[i] : 0.f;
    for (int e = threadIdx.x; e < D * ldD; e += blockDim.x) {
      const int i = e / ldD, j = e - i * ldD;
      sB[e] = (i < d && j < d) ? en.prec[i * d + j] : 0.f;
    }
  }
  if constexpr (kSmemTables) __syncthreads();
  const int2 cr = chain_range(r);
  const int c = cr.x + blockIdx.x * wpb + wib;
  if (c >= cr.y) return;

  DevState *st = r.st;
  // issue the independent loads first; the flags are checked after
  const int s = r.cdest[c];
  const int par = r.cpar[c];
  LaneParams<D, KIND, K> P;
  load_params<D, KIND, K>(P, en);
  // row `lane` of L (zeros past d), held in registers for the whole chain
  float Lrow[D];
  {
    const float *row = r.L + static_cast<long long>(lane < d ? lane : 0) * r.dp;
#pragma unroll
    for (int i = 0; i < D; ++i) Lrow[i] = (lane < d && i < d) ? row[i] : 0.f;
  }
  // prior, padded with neutral values (infinite box / zero inverse sd)
  float pa[D], pb[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    pa[i] = __ldg(pr.lane_pab + i);
    pb[i] = __ldg(pr.lane_pab + 32 + i);
  }
  float x[D], v[D];
#pragma unroll
  const float *xs = start_row(r, par);
  for (int i = 0; i < D; ++i) x[i] = i < d ? xs[i] : 0.f;
  float e = start_e(r, par);
  if (st->terminated || st->error || st->finalised) return;
  const uint32_t it = static_cast<uint32_t>(st->iter)  /* set by the select kernel */;
  const float e_star = st->e_star;
  const float w = st->width;
  const int p = r.p, cap = r.max_stepout, maxs = r.max_shrink;
  const bool euclid = r.dir_norm == NSS_DIR_EUCLIDEAN;
  const bool box = pr.kind == NSS_PRIOR_BOX;
  const float log_norm = pr.log_norm;
  const int h = 2 * ((d + 1) / 2);
  const int nblk = (h + 2 + kShrink + 3) >> 2;  // normals, u_h, u_b, first shrink round
  const int side = lane >> 4, m = lane & 15;
  float lp = log_norm;
  if (!box) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const float u = (x[i] - pa[i]) * pb[i];
      acc = fmaf(u, u, acc);
    }
    lp = fmaf(-0.5f, acc, log_norm);
  }

  unsigned long long n_probe = 0, n_eval = 0, n_exp = 0, n_shr = 0, n_null = 0;
  bool nan_seen = false;

  for (int j = 0; j < p; ++j) {
    // ---- one Philox pass: lane b holds block b of stream (it, s, HRSS, j) ----
    uint4 blk = make_uint4(0, 0, 0, 0);
    if (lane < nblk) blk = philox_block(r, it, s, kPhaseHrss, j, lane);
    // Box-Muller pairs (4b, 4b+1) and (4b+2, 4b+3) that are normals (index < h).
    // The angle 2 pi u is reduced to 2 pi (u - 1/2) in [-pi, pi) (u - 1/2 is
    // exact) so the fast sin/cos stays within its accurate range:
    // cos(2 pi u) = -cos(2 pi (u - 1/2)), sin likewise.
    float zb0 = 0.f, zb1 = 0.f, zb2 = 0.f, zb3 = 0.f;
    {
      const float r0 = sqrtf(-2.f * logf(u01(blk.x))), r1 = sqrtf(-2.f * logf(u01(blk.z)));
      float s0, c0, s1, c1;
      __sincosf(6.283185307179586f * (u01(blk.y) - 0.5f), &s0, &c0);
      __sincosf(6.283185307179586f * (u01(blk.w) - 0.5f), &s1, &c1);
      if (4 * lane + 1 < h) { zb0 = -r0 * c0; zb1 = -r0 * s0; }
      if (4 * lane + 3 < h) { zb2 = -r1 * c1; zb3 = -r1 * s1; }
    }
    float z[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int q = i & 3;
      const float mine = q == 0 ? zb0 : (q == 1 ? zb1 : (q == 2 ? zb2 : zb3));
      const float zi = __shfl_sync(kFull, mine, i >> 2);
      z[i] = i < d ? zi : 0.f;
    }
    // direction (R-6): lane i computes (L z)_i from its register row, then broadcast
    float vl = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) vl = fmaf(Lrow[i], z[i], vl);
    float zz = 0.f, vv = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      v[i] = __shfl_sync(kFull, vl, i);
      zz = fmaf(z[i], z[i], zz);
      vv = fmaf(v[i], v[i], vv);
    }
    const float inv = 1.f / sqrtf(euclid ? vv : zz);
#pragma unroll
    for (int i = 0; i < D; ++i) v[i] *= inv;

    // ---- slice height, bracket offset, first shrink uniforms (draws h, h+1, h+2..) ----
    const float u_h = u01(__shfl_sync(kFull, word(blk, h & 3), h >> 2));
    const float u_b = u01(__shfl_sync(kFull, word(blk, (h + 1) & 3), (h + 1) >> 2));
    float us[kShrink];
#pragma unroll
    for (int i = 0; i < kShrink; ++i) {
      const int q = h + 2 + i;
      us[i] = u01(__shfl_sync(kFull, word(blk, q & 3), q >> 2));
    }
    const float log_y = lp + logf(u_h);
    const float l0 = -w * u_b;
    const float r0 = l0 + w;

    // ---- stepping-out: lanes 0-15 left endpoints, 16-31 right ----
    int nl = 0, nr = 0;
    bool ldone = false, rdone = false;
    while (!(ldone && rdone)) {
      const int idx = (side == 0 ? nl : nr) + m;
      const bool act = !(side == 0 ? ldone : rdone) && idx < cap;
      const float t = side == 0 ? fmaf(-static_cast<float>(idx), w, l0) : fmaf(static_cast<float>(idx), w, r0);
      LaneProbe o{false, false, false, 0.f, 0.f};
      if (act) o = lane_probe<D, KIND, K>(t, x, v, box, pa, pb, log_norm, P, en, sA, sB, sC, ldD, d, log_y, e_star);
      const unsigned bok = __ballot_sync(kFull, o.ok);
      const unsigned bpass = __ballot_sync(kFull, act && o.pass);
      const unsigned bnan = __ballot_sync(kFull, act && o.nan);
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        if (sd == 0 ? ldone : rdone) continue;
        const int navail = min(kRound, cap - (sd == 0 ? nl : nr));
        const unsigned bits = (bok >> (16 * sd)) & 0xffffu;
        const int run = __ffs(~bits) - 1;  // consecutive in-slice endpoints
        const int tested = run < navail ? run + 1 : navail;
        n_probe += tested;
        n_eval += __popc((bpass >> (16 * sd)) & low_mask(tested));
        nan_seen = nan_seen || (((bnan >> (16 * sd)) & low_mask(tested)) != 0);
        const int add = run < navail ? run : navail;
        if (sd == 0) { nl += add; ldone = run < navail || nl >= cap; }
        else { nr += add; rdone = run < navail || nr >= cap; }
      }
    }
    float lft = fmaf(-static_cast<float>(nl), w, l0);
    float rgt = fmaf(static_cast<float>(nr), w, r0);

    // ---- shrinkage: kShrink proposals of the all-rejected path per round ----
    int ns = 0;
    bool accepted = false;
    float t_acc = 0.f, e_acc = 0.f, lp_acc = 0.f;
    for (int base = 0; base < maxs && !accepted; base += kShrink) {
      if (base > 0) {  // rare: next uniforms h+2+base.. (one more Philox pass)
        const int q0 = h + 2 + base;
        uint4 b2 = make_uint4(0, 0, 0, 0);
        if (lane < ((kShrink + 3) >> 2) + 1) b2 = philox_block(r, it, s, kPhaseHrss, j, (q0 >> 2) + lane);
#pragma unroll
        for (int i = 0; i < kShrink; ++i) {
          const int q = q0 + i;
          us[i] = u01(__shfl_sync(kFull, word(b2, q & 3), (q >> 2) - (q0 >> 2)));
        }
      }
      float mine = 0.f, l2 = lft, r2 = rgt;
#pragma unroll
      for (int i = 0; i < kShrink; ++i) {
        const float ti = fmaf(us[i], r2 - l2, l2);
        if (lane == i) mine = ti;
        if (ti < 0.f) l2 = ti; else r2 = ti;  // R-13
      }
      const int navail = min(kShrink, maxs - base);
      const bool act = lane < navail;
      LaneProbe o{false, false, false, 0.f, 0.f};
      if (act) o = lane_probe<D, KIND, K>(mine, x, v, box, pa, pb, log_norm, P, en, sA, sB, sC, ldD, d, log_y, e_star);
      const unsigned bok = __ballot_sync(kFull, act && o.ok);
      const unsigned bpass = __ballot_sync(kFull, act && o.pass);
      const unsigned bnan = __ballot_sync(kFull, act && o.nan);
      const int first = __ffs(bok) - 1;
      const int tested = first >= 0 ? first + 1 : navail;
      const int src = first >= 0 ? first : 0;
      const float tt = __shfl_sync(kFull, mine, src);
      const float ee = __shfl_sync(kFull, o.e, src);
      const float ll = __shfl_sync(kFull, o.lp, src);
      n_probe += tested;
      n_eval += __popc(bpass & low_mask(tested));
      nan_seen = nan_seen || ((bnan & low_mask(tested)) != 0);
      ns += tested;
      if (first >= 0) {
        accepted = true;
        t_acc = tt;
        e_acc = ee;
        lp_acc = ll;
      } else {
        lft = l2;
        rgt = r2;
      }
    }
    if (accepted) {
#pragma unroll
      for (int i = 0; i < D; ++i) x[i] = fmaf(t_acc, v[i], x[i]);
      e = e_acc;
      lp = lp_acc;
    }
    n_exp += nl + nr;
    n_shr += ns;
    n_null += accepted ? 0 : 1;
    if (lane == 0)
      r.counts[static_cast<long long>(c) * p + j] =
          static_cast<uint32_t>(nl) | (static_cast<uint32_t>(nr) << 8) | (static_cast<uint32_t>(ns) << 16) |
          (static_cast<uint32_t>(accepted ? 1 : 0) << 24);
  }

  // ---- replace ----
  float xv = 0.f;
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (i == lane) xv = x[i];
  if (lane < d) r.X[static_cast<long long>(s) * r.dp + lane] = xv;
  if (lane == 0) {
    r.E[s] = e;
    if (par != s) r.birth[s] = e_star;  // a moved survivor (F4) keeps its birth level
    if (nan_seen) raise_error(st, NSS_ERR_NAN);
    atomicAdd(&st->probes, n_probe);
    atomicAdd(&st->evals, n_eval);
    atomicAdd(&st->expansions, n_exp);
    atomicAdd(&st->shrinks, n_shr);
    atomicAdd(&st->nulls, n_null);
  }
}

template <int D, int KIND, int K>
void launch_lane_t(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  constexpr int ldD = D | 1;
  const int nc = r.c1 - r.c0;
  if (nc <= 0) return;
  int wpb = nc / (148 * 4);
  wpb = wpb < 1 ? 1 : (wpb > 8 ? 8 : wpb);
  size_t floats = 1;
  if (KIND == NSS_E_MOG) floats += 2 * kMaxComp * D + kMaxComp;
  if (KIND == NSS_E_CORR_GAUSS) floats += D + static_cast<size_t>(D) * ldD;
  const size_t smem = floats * sizeof(float);
  const int blocks = (nc + wpb - 1) / wpb;
  NSS_PIN_CARVEOUT((k_hrss_lane<D, KIND, K>));
  k_hrss_lane<D, KIND, K><<<blocks, wpb * 32, smem, lc.stream>>>(r, pr, en);
  ++*lc.launch_counter;
}

template <int D, int KIND>
void launch_lane_k(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  if constexpr (KIND == NSS_E_MOG && D <= 16) {
    switch (en.n_comp) {
      case 1: launch_lane_t<D, KIND, 1>(r, pr, en, lc); return;
      case 2: launch_lane_t<D, KIND, 2>(r, pr, en, lc); return;
      case 3: launch_lane_t<D, KIND, 3>(r, pr, en, lc); return;
      case 4: launch_lane_t<D, KIND, 4>(r, pr, en, lc); return;
      default: break;
    }
  }
  launch_lane_t<D, KIND, 0>(r, pr, en, lc);
}

template <int KIND>
void launch_lane_kind(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int d = r.d;
  if constexpr (KIND == NSS_E_CORR_GAUSS) {
    if (d <= 4) launch_lane_k<4, KIND>(r, pr, en, lc);
    else if (d <= 8) launch_lane_k<8, KIND>(r, pr, en, lc);
    else launch_lane_k<12, KIND>(r, pr, en, lc);
  } else {
    if (d <= 2) launch_lane_k<2, KIND>(r, pr, en, lc);
    else if (d <= 4) launch_lane_k<4, KIND>(r, pr, en, lc);
    else if (d <= 8) launch_lane_k<8, KIND>(r, pr, en, lc);
    else if (d <= 10) launch_lane_k<10, KIND>(r, pr, en, lc);
    else if (d <= 12) launch_lane_k<12, KIND>(r, pr, en, lc);
    else if (d <= 16) launch_lane_k<16, KIND>(r, pr, en, lc);
    else if (d <= 24) launch_lane_k<24, KIND>(r, pr, en, lc);
    else launch_lane_k<32, KIND>(r, pr, en, lc);
  }
}

}  // namespace

// Whether the one-probe-per-lane engine applies: d <= 32 and a thread-local
// energy of at most a few hundred flops.
bool lane_engine_ok(const RunDev &r, const EnergyDev &en) {
  if (r.d > 32) return false;
  switch (en.kind) {
    case NSS_E_FLAT: case NSS_E_GAUSS: case NSS_E_FUNNEL: return true;
    case NSS_E_MOG: return en.n_comp <= kMaxComp && en.n_comp * r.d <= 256;
    case NSS_E_CORR_GAUSS: return r.d <= 12;
    default: return false;
  }
}

void launch_hrss_lane(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  switch (en.kind) {
    case NSS_E_FLAT: launch_lane_kind<NSS_E_FLAT>(r, pr, en, lc); break;
    case NSS_E_GAUSS: launch_lane_kind<NSS_E_GAUSS>(r, pr, en, lc); break;
    case NSS_E_MOG: launch_lane_kind<NSS_E_MOG>(r, pr, en, lc); break;
    case NSS_E_FUNNEL: launch_lane_kind<NSS_E_FUNNEL>(r, pr, en, lc); break;
    case NSS_E_CORR_GAUSS: launch_lane_kind<NSS_E_CORR_GAUSS>(r, pr, en, lc); break;
    default: break;
  }
}

}  // namespace nss
