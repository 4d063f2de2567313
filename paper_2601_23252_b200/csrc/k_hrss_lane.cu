// A6/A7 (+A1) for small dimensions (d <= 32) and cheap energies: one warp per
// chain, ONE PROBE PER LANE.
//
// HRSS is a chain of dependent slice tests, so at small d a warp-per-chain
// kernel is latency-bound: every probe waits for the previous decision.  But
// all the points the sequential algorithm could visit next are
// known in advance:
//   * stepping-out endpoints are L - m w and R + m w (m = 0..cap-1);
//   * along the all-rejected path every shrink proposal is fixed too, because a
//     rejected proposal t moves the left end if t < 0 and the right end
//     otherwise (R-13): proposal i is L_i + u_i (R_i - L_i) with (L_i, R_i)
//     obtained from proposals 0..i-1.
// So the warp evaluates 16 left + 16 right endpoints in one round (lanes
// 0-15 / 16-31) and 16 shrink proposals in a second round, then takes the
// first outcome the sequential algorithm would have taken (ballot + ffs).
// Every point is computed with the same fp32 operations, in the same order, as
// the sequential kernel (repeated subtraction of w; the same fma for t), so
// decisions, counters and results are those of the sequential algorithm;
// only the number of dependent rounds changes (about 2 per step instead of
// ~5-7).  Counters report the algorithm's probes, not the speculative ones,
// and a NaN raises an error only if the sequential algorithm would have
// evaluated that point.
#include "energy.cuh"

namespace nss {

namespace {

constexpr int kRound = 16;  // endpoints per side / shrink proposals per round

// Thread-local energy of the point xp (coordinates >= d are ignored).
template <int D, int KIND>
__device__ __forceinline__ float lane_energy(const float (&xp)[D], const EnergyDev &en, const ESm &es, int d) {
  if constexpr (KIND == NSS_E_FLAT) {
    return en.c;
  } else if constexpr (KIND == NSS_E_GAUSS) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (i < d) {
        const float u = (xp[i] - es.mu[i]) * es.isig[i];
        s = fmaf(u, u, s);
      }
    return 0.5f * s + en.c;
  } else if constexpr (KIND == NSS_E_MOG) {
    // -log sum_j exp(logc_j - 1/2 |(x - mu_j) / sigma_j|^2), online log-sum-exp
    float m = -INFINITY, acc = 0.f;
#pragma unroll 4
    for (int j = 0; j < en.n_comp; ++j) {
      const float *mu = es.mu + j * d;
      const float *is = es.isig + j * d;
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < D; ++i)
        if (i < d) {
          const float u = (xp[i] - mu[i]) * is[i];
          s = fmaf(u, u, s);
        }
      const float l = es.logc[j] - 0.5f * s;
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
    for (int i = 1; i < D; ++i)
      if (i < d) s = fmaf(xp[i], xp[i], s);
    const float sy = en.sigma_y, yy = y / sy;
    return 0.5f * yy * yy + logf(sy) + 0.5f * kLn2Pi + 0.5f * s * expf(-y) +
           static_cast<float>(d - 1) * 0.5f * (y + kLn2Pi);
  } else if constexpr (KIND == NSS_E_CORR_GAUSS) {
    float y[D];
#pragma unroll
    for (int i = 0; i < D; ++i) y[i] = i < d ? xp[i] - es.mu[i] : 0.f;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (i < d) {
        const float *row = es.prec + i * es.ldp;
        float py = 0.f;
#pragma unroll
        for (int m = 0; m < D; ++m)
          if (m < d) py = fmaf(row[m], y[m], py);
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

template <int D, int KIND>
__device__ __forceinline__ LaneProbe lane_probe(float t, const float (&x)[D], const float (&v)[D],
                                                const PriorDev &pr, const float *sPr, const EnergyDev &en,
                                                const ESm &es, int d, float log_y, float e_star) {
  float xp[D];
#pragma unroll
  for (int i = 0; i < D; ++i) xp[i] = fmaf(t, v[i], x[i]);
  LaneProbe o{false, false, false, 0.f, 0.f};
  if (pr.kind == NSS_PRIOR_BOX) {
    bool in = true;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (i < d) in = in && (xp[i] >= sPr[i]) && (xp[i] <= sPr[d + i]);
    o.lp = pr.log_norm;
    o.pass = in && (o.lp >= log_y);
  } else {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (i < d) {
        const float u = (xp[i] - sPr[i]) * sPr[d + i];
        s = fmaf(u, u, s);
      }
    o.lp = -0.5f * s + pr.log_norm;
    o.pass = o.lp >= log_y;
  }
  if (o.pass) {
    o.e = lane_energy<D, KIND>(xp, en, es, d);
    o.nan = isnan(o.e);
    o.ok = !o.nan && o.e < e_star;
  }
  return o;
}

__device__ __forceinline__ unsigned low_mask(int n) {  // bits 0..n-1
  return n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
}

template <int D, int KIND>
__global__ void __launch_bounds__(256) k_hrss_lane(RunDev r, PriorDev pr, EnergyDev en) {
  extern __shared__ float sm[];
  __shared__ int sh_flag;
  const int d = r.d, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int ldl = odd_stride(d);
  float *sL = sm;
  float *sPr = sL + d * ldl;
  float *sP = sPr + 2 * d;
  if (threadIdx.x == 0) sh_flag = (r.st->terminated || r.st->error || r.st->finalised) ? 1 : 0;
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
    const int i = e / d, j = e - i * d;
    sL[i * ldl + j] = r.L[i * r.dp + j];
  }
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    sPr[i] = pr.kind == NSS_PRIOR_BOX ? pr.lo[i] : pr.mean[i];
    sPr[d + i] = pr.kind == NSS_PRIOR_BOX ? pr.hi[i] : pr.isd[i];
  }
  ESm es;
  stage_energy(en, sP, es);
  __syncthreads();
  if (sh_flag) return;
  const int c = blockIdx.x * wpb + wib;
  if (c >= r.k) return;

  DevState *st = r.st;
  const uint32_t it = static_cast<uint32_t>(st->iter + 1);
  const int s = r.dest_gid[c];
  const int par = r.parent_gid[c];
  const float e_star = st->e_star;
  const float w = st->width;
  const int p = r.p, cap = r.max_stepout, maxs = r.max_shrink;
  const bool euclid = r.dir_norm == NSS_DIR_EUCLIDEAN;
  const int h = 2 * ((d + 1) / 2);
  const int nblk_norm = h >> 2, nblk_all = (h + 3) >> 2;
  const int side = lane >> 4, m = lane & 15;

  float x[D], v[D];
#pragma unroll
  for (int i = 0; i < D; ++i) x[i] = i < d ? r.X[static_cast<long long>(par) * r.dp + i] : 0.f;
  float e = r.E[par];
  float lp;
  if (pr.kind == NSS_PRIOR_BOX) {
    lp = pr.log_norm;
  } else {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (i < d) {
        const float u = (x[i] - sPr[i]) * sPr[d + i];
        acc = fmaf(u, u, acc);
      }
    lp = -0.5f * acc + pr.log_norm;
  }

  unsigned long long n_probe = 0, n_eval = 0, n_exp = 0, n_shr = 0, n_null = 0;
  bool nan_seen = false;

  for (int j = 0; j < p; ++j) {
    // ---- direction (R-6): lane b holds normals 4b..4b+3 of stream (it, s, HRSS, j) ----
    float zb0 = 0.f, zb1 = 0.f, zb2 = 0.f, zb3 = 0.f;
    if (lane < nblk_all) {
      const uint4 u4 = philox_block(r, it, s, kPhaseHrss, j, lane);
      const float r0 = sqrtf(-2.f * logf(u01(u4.x))), r1 = sqrtf(-2.f * logf(u01(u4.z)));
      float s0, c0, s1, c1;
      sincospif(2.f * u01(u4.y), &s0, &c0);
      sincospif(2.f * u01(u4.w), &s1, &c1);
      zb0 = r0 * c0;
      zb1 = r0 * s0;
      if (lane < nblk_norm) {
        zb2 = r1 * c1;
        zb3 = r1 * s1;
      }
    }
    float z[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int q = i & 3;
      const float mine = q == 0 ? zb0 : (q == 1 ? zb1 : (q == 2 ? zb2 : zb3));
      const float zi = __shfl_sync(kFull, mine, i >> 2);
      z[i] = i < d ? zi : 0.f;
    }
    // row `lane` of L z, then broadcast
    float vl = 0.f;
    if (lane < d) {
      const float *row = sL + lane * ldl;
#pragma unroll
      for (int i = 0; i < D; ++i)
        if (i <= lane && i < d) vl = fmaf(row[i], z[i], vl);
    }
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

    // ---- slice height and initial bracket (R-9) ----
    const uint4 hb = philox_block(r, it, s, kPhaseHrss, j, h >> 2);
    const float log_y = lp + logf(u01(word(hb, h & 3)));
    float lft = -w * u01(word(hb, (h + 1) & 3));
    float rgt = lft + w;

    // ---- stepping-out: lanes 0-15 left endpoints, 16-31 right ----
    int nl = 0, nr = 0;
    bool ldone = false, rdone = false;
    while (!(ldone && rdone)) {
      const bool mine_done = side == 0 ? ldone : rdone;
      const int mine_n = side == 0 ? nl : nr;
      float t = side == 0 ? lft : rgt;
#pragma unroll
      for (int q = 0; q < kRound - 1; ++q)
        if (q < m) t = side == 0 ? t - w : t + w;
      const bool act = !mine_done && (mine_n + m < cap);
      LaneProbe o{false, false, false, 0.f, 0.f};
      if (act) o = lane_probe<D, KIND>(t, x, v, pr, sPr, en, es, d, log_y, e_star);
      const unsigned bok = __ballot_sync(kFull, o.ok);
      const unsigned bpass = __ballot_sync(kFull, act && o.pass);
      const unsigned bnan = __ballot_sync(kFull, act && o.nan);
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        const bool done = sd == 0 ? ldone : rdone;
        const int navail = min(kRound, cap - (sd == 0 ? nl : nr));
        const unsigned bits = (bok >> (16 * sd)) & 0xffffu;
        const unsigned pbits = (bpass >> (16 * sd)) & 0xffffu;
        const unsigned nbits = (bnan >> (16 * sd)) & 0xffffu;
        const int run = __ffs(~bits) - 1;  // consecutive in-slice endpoints from m = 0
        const int tested = run < navail ? run + 1 : navail;
        const int src = 16 * sd + (run < navail ? run : navail - 1);
        const float tsrc = __shfl_sync(kFull, t, src);
        if (!done) {
          n_probe += tested;
          n_eval += __popc(pbits & low_mask(tested));
          nan_seen = nan_seen || (nbits & low_mask(tested));
          if (run < navail) {
            if (sd == 0) { lft = tsrc; nl += run; ldone = true; }
            else { rgt = tsrc; nr += run; rdone = true; }
          } else {
            const float nxt = sd == 0 ? tsrc - w : tsrc + w;
            if (sd == 0) { lft = nxt; nl += navail; ldone = nl >= cap; }
            else { rgt = nxt; nr += navail; rdone = nr >= cap; }
          }
        }
      }
    }

    // ---- shrinkage: 16 proposals of the all-rejected path per round ----
    int ns = 0;
    bool accepted = false;
    float t_acc = 0.f, e_acc = 0.f, lp_acc = 0.f;
    for (int base = 0; base < maxs && !accepted; base += kRound) {
      const int q = h + 2 + base + m;
      const uint4 ub = philox_block(r, it, s, kPhaseHrss, j, static_cast<uint32_t>(q >> 2));
      const float u = u01(word(ub, q & 3));
      float mine = 0.f, l2 = lft, r2 = rgt;
#pragma unroll
      for (int i = 0; i < kRound; ++i) {
        const float ui = __shfl_sync(kFull, u, i);
        const float ti = fmaf(ui, r2 - l2, l2);
        if (lane == i) mine = ti;
        if (ti < 0.f) l2 = ti; else r2 = ti;  // R-13
      }
      const int navail = min(kRound, maxs - base);
      const bool act = lane < navail;
      LaneProbe o{false, false, false, 0.f, 0.f};
      if (act) o = lane_probe<D, KIND>(mine, x, v, pr, sPr, en, es, d, log_y, e_star);
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
      nan_seen = nan_seen || (bnan & low_mask(tested));
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
  if (lane < d) {
    float xv = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (i == lane) xv = x[i];
    r.X[static_cast<long long>(s) * r.dp + lane] = xv;
  }
  if (lane == 0) {
    r.E[s] = e;
    r.birth[s] = e_star;
    if (nan_seen) raise_error(st, NSS_ERR_NAN);
    atomicAdd(&st->probes, n_probe);
    atomicAdd(&st->evals, n_eval);
    atomicAdd(&st->expansions, n_exp);
    atomicAdd(&st->shrinks, n_shr);
    atomicAdd(&st->nulls, n_null);
  }
}

template <int D, int KIND>
void launch_lane_t(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int ldl = odd_stride(r.d);
  int wpb = r.k / (148 * 4);
  wpb = wpb < 1 ? 1 : (wpb > 8 ? 8 : wpb);
  const size_t smem = (static_cast<size_t>(r.d) * ldl + 2 * r.d + energy_param_floats(KIND, r.d, en.n_comp)) *
                      sizeof(float);
  static size_t attr = 0;
  if (smem > 48 * 1024 && attr < smem) {
    cudaFuncSetAttribute(k_hrss_lane<D, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = smem;
  }
  const int blocks = (r.k + wpb - 1) / wpb;
  k_hrss_lane<D, KIND><<<blocks, wpb * 32, smem, lc.stream>>>(r, pr, en);
  ++*lc.launch_counter;
}

template <int KIND>
void launch_lane_kind(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int d = r.d;
  if (d <= 2) launch_lane_t<2, KIND>(r, pr, en, lc);
  else if (d <= 4) launch_lane_t<4, KIND>(r, pr, en, lc);
  else if (d <= 8) launch_lane_t<8, KIND>(r, pr, en, lc);
  else if (d <= 10) launch_lane_t<10, KIND>(r, pr, en, lc);
  else if (d <= 12) launch_lane_t<12, KIND>(r, pr, en, lc);
  else if (d <= 16) launch_lane_t<16, KIND>(r, pr, en, lc);
  else if (d <= 24) launch_lane_t<24, KIND>(r, pr, en, lc);
  else launch_lane_t<32, KIND>(r, pr, en, lc);
}

}  // namespace

// Whether the one-probe-per-lane engine applies: d <= 32, a thread-local
// energy of at most a few hundred flops, step-out cap <= 16 per round handled
// by the round loop (any cap works).
bool lane_engine_ok(const RunDev &r, const EnergyDev &en) {
  if (r.d > 32) return false;
  switch (en.kind) {
    case NSS_E_FLAT: case NSS_E_GAUSS: case NSS_E_FUNNEL: return true;
    case NSS_E_MOG: return en.n_comp * r.d <= 256;
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
