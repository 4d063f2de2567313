// A6/A7 (+A1) for the correlated Gaussian at large d (C3a): NC HRSS chains
// per warp, their probes evaluated together.
//
// The quadratic form q = |U (x - mu)|^2 (P = U^T U, upper triangular,
// d(d+1)/2 multiply-adds) streams the whole factor U through shared memory
// for every probe.  With one chain per warp (k_hrss.cu) every U element read
// feeds one FMA and the shared-memory pipe, not the FMA pipe, sets the pace
// (SURVEY D-3: "unless >= 4 chains share P loads per warp").  Here a warp
// owns NC chains and advances them in rounds: every round each chain runs its
// sequential HRSS state machine (the decisions, draws and fp32
// probe points of k_hrss.cu) up to its next energy request, the NC probe
// points are staged interleaved in shared memory, and one pass over U serves
// all of them: lane l owns rows l, l+32, ... of U and, per column m, one U
// element per row and one NC-wide vector of probe coordinates feed NC FMAs
// per row.  A chain that needs no energy in a round (finished, or resolved by
// the prior test) stages zeros and ignores its result.  Chains are
// independent, so every chain's trajectory is the sequential algorithm's; the
// energies differ from k_hrss.cu only in the order of the fp32 sums.
#include "energy.cuh"

namespace nss {

namespace {

enum MPhase : int { kMDir = 0, kMLeft = 1, kMRight = 2, kMShrink = 3, kMDone = 4 };

// per-chain scalar state, in shared memory (one slot per chain of the warp)
struct MChain {
  int phase, step, nl, nr, ns, need;
  float l0, r0, lft, rgt, log_y, e, lp, t, lpt;
  unsigned n_probe, n_eval, n_exp, n_shr, n_null;
};

constexpr int kWarps = 4;  // warps per block

template <int NPL, int NC>
__global__ void __launch_bounds__(kWarps * 32) k_hrss_multi(RunDev r, PriorDev pr, EnergyDev en) {
  extern __shared__ float sm[];
  __shared__ MChain chs[kWarps][NC];
  __shared__ int sh_flag;
  const int d = r.d, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int ldu = odd_stride(d);
  float *sMu = sm;                      // d
  float *sU = sMu + d;                  // d rows of stride ldu (U, upper triangular)
  // this warp's staged probes [m][c] (c fastest), 16-byte aligned
  float *sW = sm + ((d + d * ldu + 3) & ~3) + wib * (d * NC);
  if (threadIdx.x == 0) sh_flag = (r.st->terminated || r.st->error || r.st->finalised) ? 1 : 0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) sMu[i] = en.mu[i];
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
    const int i = e / d, j = e - i * d;
    sU[i * ldu + j] = en.ufac[e];
  }
  __syncthreads();
  if (sh_flag) return;
  const int2 cr = chain_range(r);
  const int cbase = cr.x + (blockIdx.x * kWarps + wib) * NC;
  if (cbase >= cr.y) return;  // uniform per warp
  DevState *st = r.st;
  const uint32_t it = static_cast<uint32_t>(st->iter);
  const float e_star = st->e_star, w = st->width;
  const int p = r.p, cap = r.max_stepout, maxs = r.max_shrink;
  const int h = 2 * ((d + 1) / 2);
  const float cterm = en.c;

  float pa[NPL], pb[NPL];
  load_prior_lane<NPL>(pr, lane, d, pa, pb);
  float x[NC][NPL], v[NC][NPL];
  MChain *cs = chs[wib];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = cbase + c;
    const bool real = ch < cr.y;
    const int par = real ? r.cpar[ch] : 0;
    const float *xs = start_row(r, par);
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      x[c][t] = (real && i < d) ? xs[i] : 0.f;
      v[c][t] = 0.f;
    }
    bool dummy;
    const float lp = prior_logp<NPL>(x[c], pr, pa, pb, lane, d, dummy);
    if (lane == 0) {
      MChain z{};
      z.phase = real ? (p > 0 ? kMDir : kMDone) : kMDone;
      z.e = real ? start_e(r, par) : 0.f;
      z.lp = lp;
      cs[c] = z;
    }
  }
  __syncwarp();

  bool nan_seen = false;
  for (;;) {
    // ---- 1) every chain runs to its next energy request ----
    int any = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = cbase + c;
      MChain s = cs[c];
      s.need = 0;
      float xp[NPL];
      // in(t) up to the prior: returns true when an energy is needed
      auto prior_ok = [&](float tt, float &lpp) -> bool {
        ++s.n_probe;
#pragma unroll
        for (int q = 0; q < NPL; ++q) xp[q] = fmaf(tt, v[c][q], x[c][q]);
        bool inside;
        lpp = prior_logp<NPL>(xp, pr, pa, pb, lane, d, inside);
        return inside && lpp >= s.log_y;
      };
      auto end_step = [&](int accepted) {
        s.n_exp += s.nl + s.nr;
        s.n_shr += s.ns;
        s.n_null += accepted ? 0 : 1;
        if (lane == 0)
          r.counts[static_cast<long long>(ch) * p + s.step] =
              static_cast<uint32_t>(s.nl) | (static_cast<uint32_t>(s.nr) << 8) | (static_cast<uint32_t>(s.ns) << 16) |
              (static_cast<uint32_t>(accepted) << 24);
        s.step += 1;
        s.phase = s.step < p ? kMDir : kMDone;
      };
      while (!s.need && s.phase != kMDone) {
        if (s.phase == kMDir) {
          // direction precomputed for (chain, step) by k_dirs
          const float *vr = r.Vpre + (static_cast<long long>(ch - cr.x) * p + s.step) * r.dp;
#pragma unroll
          for (int t = 0; t < NPL; ++t) {
            const int i = lane + 32 * t;
            v[c][t] = i < d ? __ldg(vr + i) : 0.f;
          }
          const int dest = r.cdest[ch];
          const uint4 hb = philox_block(r, it, dest, kPhaseHrss, s.step, h >> 2);
          s.log_y = s.lp + logf(u01(word(hb, h & 3)));
          s.l0 = -w * u01(word(hb, (h + 1) & 3));
          s.r0 = s.l0 + w;
          s.lft = s.l0;
          s.rgt = s.r0;
          s.nl = s.nr = s.ns = 0;
          s.phase = kMLeft;
        } else if (s.phase == kMLeft) {
          if (s.nl >= cap) { s.phase = kMRight; continue; }
          float lpp;
          if (!prior_ok(s.lft, lpp)) { s.phase = kMRight; continue; }
          s.t = s.lft;
          s.lpt = lpp;
          s.need = 1;
        } else if (s.phase == kMRight) {
          if (s.nr >= cap) { s.phase = kMShrink; continue; }
          float lpp;
          if (!prior_ok(s.rgt, lpp)) { s.phase = kMShrink; continue; }
          s.t = s.rgt;
          s.lpt = lpp;
          s.need = 1;
        } else {  // shrink (R-12/R-13)
          if (s.ns >= maxs) { end_step(0); continue; }
          const int q = h + 2 + s.ns;
          const int dest = r.cdest[ch];
          const uint4 ub = philox_block(r, it, dest, kPhaseHrss, s.step, static_cast<uint32_t>(q >> 2));
          const float tt = fmaf(u01(word(ub, q & 3)), s.rgt - s.lft, s.lft);
          s.ns += 1;
          float lpp;
          if (!prior_ok(tt, lpp)) {
            if (tt < 0.f) s.lft = tt; else s.rgt = tt;
            continue;
          }
          s.t = tt;
          s.lpt = lpp;
          s.need = 1;
        }
      }
      // stage r = x + t v - mu (zeros when no energy is needed)
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        const int i = lane + 32 * t;
        if (i < d) sW[i * NC + c] = s.need ? fmaf(s.t, v[c][t], x[c][t]) - sMu[i] : 0.f;
      }
      any |= s.need;
      if (lane == 0) cs[c] = s;
    }
    __syncwarp();
    if (!any) break;

    // ---- 2) one pass over U for the NC probes: q_c = sum_i (sum_{m>=i} U_im r_cm)^2 ----
    float acc[NPL][NC];
#pragma unroll
    for (int t = 0; t < NPL; ++t)
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[t][c] = 0.f;
    for (int m = 0; m < d; ++m) {
      float wm[NC];
      if constexpr (NC == 4) {
        const float4 w4 = *reinterpret_cast<const float4 *>(sW + m * 4);
        wm[0] = w4.x; wm[1] = w4.y; wm[2] = w4.z; wm[3] = w4.w;
      } else if constexpr (NC == 2) {
        const float2 w2 = *reinterpret_cast<const float2 *>(sW + m * 2);
        wm[0] = w2.x; wm[1] = w2.y;
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) wm[c] = sW[m * NC + c];
      }
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        if (m >= 32 * t) {  // uniform: rows of block t start at column >= 32 t (zeros below the diagonal)
          const int i = lane + 32 * t;
          const float u = i < d ? sU[i * ldu + m] : 0.f;
#pragma unroll
          for (int c = 0; c < NC; ++c) acc[t][c] = fmaf(u, wm[c], acc[t][c]);
        }
      }
    }
    float qv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      float q = 0.f;
#pragma unroll
      for (int t = 0; t < NPL; ++t) q = fmaf(acc[t][c], acc[t][c], q);
      qv[c] = 0.5f * warp_sum(q) + cterm;
    }
    __syncwarp();

    // ---- 3) every chain takes its decision ----
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      MChain s = cs[c];
      if (!s.need) continue;
      const float ep = qv[c];
      s.n_eval += 1;
      nan_seen = nan_seen || isnan(ep);
      const bool in = ep < e_star;
      if (s.phase == kMLeft) {
        if (in) { s.nl += 1; s.lft = fmaf(-static_cast<float>(s.nl), w, s.l0); }
        else s.phase = kMRight;
      } else if (s.phase == kMRight) {
        if (in) { s.nr += 1; s.rgt = fmaf(static_cast<float>(s.nr), w, s.r0); }
        else s.phase = kMShrink;
      } else {
        if (in) {
#pragma unroll
          for (int q = 0; q < NPL; ++q) x[c][q] = fmaf(s.t, v[c][q], x[c][q]);
          s.e = ep;
          s.lp = s.lpt;
          s.n_exp += s.nl + s.nr;
          s.n_shr += s.ns;
          if (lane == 0)
            r.counts[static_cast<long long>(cbase + c) * p + s.step] =
                static_cast<uint32_t>(s.nl) | (static_cast<uint32_t>(s.nr) << 8) |
                (static_cast<uint32_t>(s.ns) << 16) | (1u << 24);
          s.step += 1;
          s.phase = s.step < p ? kMDir : kMDone;
        } else {
          if (s.t < 0.f) s.lft = s.t; else s.rgt = s.t;
        }
      }
      s.need = 0;
      if (lane == 0) cs[c] = s;
    }
    __syncwarp();
  }

  // ---- replace ----
  unsigned long long np = 0, ne = 0, nx = 0, nsh = 0, nn = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = cbase + c;
    if (ch >= cr.y) continue;
    const MChain s = cs[c];
    const int dest = r.cdest[ch];
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      if (i < d) r.X[static_cast<long long>(dest) * r.dp + i] = x[c][t];
    }
    if (lane == 0) {
      r.E[dest] = s.e;
      if (r.cpar[ch] != dest) r.birth[dest] = e_star;
    }
    np += s.n_probe; ne += s.n_eval; nx += s.n_exp; nsh += s.n_shr; nn += s.n_null;
  }
  if (lane == 0) {
    if (nan_seen) raise_error(st, NSS_ERR_NAN);
    atomicAdd(&st->probes, np);
    atomicAdd(&st->evals, ne);
    atomicAdd(&st->expansions, nx);
    atomicAdd(&st->shrinks, nsh);
    atomicAdd(&st->nulls, nn);
  }
}

template <int NPL, int NC>
void launch_multi_t(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int nc = r.c1 - r.c0;
  if (nc <= 0) return;
  const int ldu = odd_stride(r.d);
  const size_t smem = (static_cast<size_t>((r.d + r.d * ldu + 3) & ~3) + static_cast<size_t>(kWarps) * r.d * NC) *
                      sizeof(float);
  NSS_MAX_SMEM((k_hrss_multi<NPL, NC>), smem);
  NSS_PIN_CARVEOUT((k_hrss_multi<NPL, NC>));
  const int per_block = kWarps * NC;
  k_hrss_multi<NPL, NC><<<(nc + per_block - 1) / per_block, kWarps * 32, smem, lc.stream>>>(r, pr, en);
  ++*lc.launch_counter;
}

}  // namespace

// The multi-chain engine applies to the correlated Gaussian with its factor U
// at large d (directions precomputed), standard NS (not tempered, HRSS).  It
// is opt-in (NSS_MULTI=1): at C3a it is parity-green but 2.2x slower than two
// warps per chain (14.6 vs 6.6 ms per iteration; NC = 2: 13.7 ms) -- 1000
// chains make 250 warps, 1.7 per SM, and the warp serialises its chains'
// state machines: the kernel is latency-bound, not shared-memory bound.
bool multi_engine_ok(const RunDev &r, const EnergyDev &en) {
  static const bool on = getenv("NSS_MULTI") != nullptr;
  return on && en.kind == NSS_E_CORR_GAUSS && en.ufac && r.d > 32 && r.Vpre && !r.tempered &&
         r.mutation == NSS_MUT_HRSS;
}

void launch_hrss_multi(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  static const int nc = getenv("NSS_MULTI_NC") ? atoi(getenv("NSS_MULTI_NC")) : 4;
  const int npl = (r.d + 31) / 32;
  if (nc == 2) {
    switch (npl) {
      case 2: launch_multi_t<2, 2>(r, pr, en, lc); break;
      case 3: launch_multi_t<3, 2>(r, pr, en, lc); break;
      default: launch_multi_t<4, 2>(r, pr, en, lc); break;
    }
  } else {
    switch (npl) {
      case 2: launch_multi_t<2, 4>(r, pr, en, lc); break;
      case 3: launch_multi_t<3, 4>(r, pr, en, lc); break;
      default: launch_multi_t<4, 4>(r, pr, en, lc); break;
    }
  }
}

}  // namespace nss
