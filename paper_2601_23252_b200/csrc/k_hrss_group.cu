// A6/A7 (+A1) for large d and cheap energies (C3b funnel; Gaussian): one warp
// per chain, FOUR SPECULATIVE PROBES PER ROUND in groups of eight lanes.
//
// The warp-per-chain engine (k_hrss.cu) evaluates one probe at a time, so a
// cheap energy leaves the chain bound by the dependent latency of ~5 probes
// per step.  As in the one-probe-per-lane engine (k_hrss_lane.cu, d <= 32),
// every point the sequential algorithm can visit next is known in
// advance -- stepping-out endpoints L0 - m w, R0 + m w, and along the
// all-rejected path every shrink proposal -- so the warp evaluates four of
// them at once: the next two endpoints of each side per stepping-out round,
// the next four proposals per shrink round, one per group of eight lanes
// (each lane holds ceil(d / 8) coordinates of x, v and the probe), and takes
// the outcome the sequential algorithm would take.  Decisions, draws and
// counters are those of the sequential algorithm (speculative probes past the
// first decision are not counted); energies are the warp engine's formulas
// summed over eight lanes instead of 32.  Directions come from k_dirs.
#include "energy.cuh"

namespace nss {

namespace {

constexpr int kG = 8;            // lanes per group
constexpr int kNG = 32 / kG;     // groups (probes) per warp

struct GProbe {
  bool ok, pass, nan;  // in the slice / energy evaluated / energy was NaN
  float e, lp;
};

template <int KIND>
constexpr bool group_kind_ok() {
  return KIND == NSS_E_FUNNEL || KIND == NSS_E_GAUSS;
}

template <int NPG>
__device__ __forceinline__ float gsum(float v) {
#pragma unroll
  for (int o = kG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, kG);
  return v;
}

// in(t) of one group: x + t v against the prior, the slice height and E*.
template <int NPG, int KIND>
__device__ __forceinline__ GProbe group_probe(float t, const float (&x)[NPG], const float (&v)[NPG],
                                              const PriorDev &pr, const EnergyDev &en, int gl, int d, float log_y,
                                              float e_star, bool act) {
  float xp[NPG];
#pragma unroll
  for (int q = 0; q < NPG; ++q) xp[q] = fmaf(t, v[q], x[q]);
  GProbe o{false, false, false, 0.f, 0.f};
  // prior (support and height)
  float lp;
  bool inside = true;
  if (pr.kind == NSS_PRIOR_BOX) {
    bool ok = true;
#pragma unroll
    for (int q = 0; q < NPG; ++q) {
      const int i = gl + kG * q;
      if (i < d) ok = ok && xp[q] >= __ldg(pr.lo + i) && xp[q] <= __ldg(pr.hi + i);
    }
    const unsigned gm = 0xffu << (threadIdx.x & 24);
    inside = (__ballot_sync(0xffffffffu, ok) & gm) == gm;
    lp = pr.log_norm;
  } else {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < NPG; ++q) {
      const int i = gl + kG * q;
      if (i < d) {
        const float u = (xp[q] - __ldg(pr.mean + i)) * __ldg(pr.isd + i);
        s = fmaf(u, u, s);
      }
    }
    lp = -0.5f * gsum<NPG>(s) + pr.log_norm;
  }
  // every group computes an energy (the shuffles need the whole warp); only
  // an active probe inside the prior and above the slice height counts
  const bool need = act && inside && lp >= log_y;
  float e;
  if constexpr (KIND == NSS_E_FUNNEL) {
    // P:885 (R-23): x_0 = y ~ N(0, sy^2), x_n ~ N(0, e^y) -- warp_energy's formula
    const float y = __shfl_sync(0xffffffffu, xp[0], 0, kG);
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < NPG; ++q) {
      const int i = gl + kG * q;
      if (i >= 1 && i < d) s = fmaf(xp[q], xp[q], s);
    }
    s = gsum<NPG>(s);
    const float sy = en.sigma_y;
    const float yy = y / sy;
    e = 0.5f * yy * yy + logf(sy) + 0.5f * kLn2Pi + 0.5f * s * expf(-y) +
        static_cast<float>(d - 1) * 0.5f * (y + kLn2Pi);
  } else {  // GAUSS
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < NPG; ++q) {
      const int i = gl + kG * q;
      if (i < d) {
        const float u = (xp[q] - __ldg(en.mu + i)) * __ldg(en.isig + i);
        s = fmaf(u, u, s);
      }
    }
    e = 0.5f * gsum<NPG>(s) + en.c;
  }
  o.pass = need;
  o.nan = need && isnan(e);
  o.ok = need && !o.nan && e < e_star;
  o.e = e;
  o.lp = lp;
  return o;
}

__device__ __forceinline__ unsigned low_bits(int n) { return n >= 32 ? 0xffffffffu : ((1u << n) - 1u); }

// the groups' flags, one bit per group (bit g = group g's lane 0)
__device__ __forceinline__ unsigned group_ballot(bool f) {
  const unsigned b = __ballot_sync(0xffffffffu, f && (threadIdx.x & (kG - 1)) == 0);
  unsigned out = 0;
#pragma unroll
  for (int g = 0; g < kNG; ++g) out |= ((b >> (g * kG)) & 1u) << g;
  return out;
}

template <int NPG, int KIND>
__global__ void __launch_bounds__(256) k_hrss_group(RunDev r, PriorDev pr, EnergyDev en) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int g = lane / kG, gl = lane & (kG - 1);
  const int2 cr = chain_range(r);
  const int c = cr.x + blockIdx.x * wpb + wib;
  if (c >= cr.y) return;
  DevState *st = r.st;
  if (st->terminated || st->error || st->finalised) return;
  const int d = r.d, p = r.p, cap = r.max_stepout, maxs = r.max_shrink;
  const uint32_t it = static_cast<uint32_t>(st->iter);
  const float e_star = st->e_star, w = st->width;
  const int s_gid = r.cdest[c], par = r.cpar[c];
  const int h = 2 * ((d + 1) / 2);
  float x[NPG], v[NPG];
  {
    const float *xs = start_row(r, par);
#pragma unroll
    for (int q = 0; q < NPG; ++q) {
      const int i = gl + kG * q;
      x[q] = i < d ? xs[i] : 0.f;
    }
  }
  float e = start_e(r, par);
  float lp;
  {
    float s = 0.f;
    if (pr.kind == NSS_PRIOR_BOX) {
      lp = pr.log_norm;
    } else {
#pragma unroll
      for (int q = 0; q < NPG; ++q) {
        const int i = gl + kG * q;
        if (i < d) {
          const float u = (x[q] - __ldg(pr.mean + i)) * __ldg(pr.isd + i);
          s = fmaf(u, u, s);
        }
      }
      lp = -0.5f * gsum<NPG>(s) + pr.log_norm;
    }
  }
  unsigned long long n_probe = 0, n_eval = 0, n_exp = 0, n_shr = 0, n_null = 0;
  bool nan_seen = false;
  for (int j = 0; j < p; ++j) {
    const float *vr = r.Vpre + (static_cast<long long>(c - cr.x) * p + j) * r.dp;
#pragma unroll
    for (int q = 0; q < NPG; ++q) {
      const int i = gl + kG * q;
      v[q] = i < d ? __ldg(vr + i) : 0.f;
    }
    const uint4 hb = philox_block(r, it, s_gid, kPhaseHrss, j, h >> 2);
    const float log_y = lp + logf(u01(word(hb, h & 3)));
    const float l0 = -w * u01(word(hb, (h + 1) & 3));
    const float r0 = l0 + w;

    // ---- stepping-out: groups 0, 1 the next two left endpoints, 2, 3 the right ----
    int nl = 0, nr = 0;
    bool ldone = false, rdone = false;
    while (!(ldone && rdone)) {
      const int side = g >> 1, m = g & 1;
      const int idx = (side == 0 ? nl : nr) + m;
      const bool act = !(side == 0 ? ldone : rdone) && idx < cap;
      const float t = side == 0 ? fmaf(-static_cast<float>(idx), w, l0) : fmaf(static_cast<float>(idx), w, r0);
      const GProbe o = group_probe<NPG, KIND>(t, x, v, pr, en, gl, d, log_y, e_star, act);
      const unsigned bok = group_ballot(act && o.ok), bpass = group_ballot(act && o.pass),
                     bnan = group_ballot(act && o.nan);
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        if (sd == 0 ? ldone : rdone) continue;
        const int navail = min(2, cap - (sd == 0 ? nl : nr));
        const unsigned bits = (bok >> (2 * sd)) & 3u;
        const int run = __ffs(~bits) - 1;  // consecutive in-slice endpoints
        const int tested = run < navail ? run + 1 : navail;
        n_probe += tested;
        n_eval += __popc((bpass >> (2 * sd)) & low_bits(tested));
        nan_seen = nan_seen || (((bnan >> (2 * sd)) & low_bits(tested)) != 0);
        const int add = run < navail ? run : navail;
        if (sd == 0) { nl += add; ldone = run < navail || nl >= cap; }
        else { nr += add; rdone = run < navail || nr >= cap; }
      }
    }
    float lft = fmaf(-static_cast<float>(nl), w, l0);
    float rgt = fmaf(static_cast<float>(nr), w, r0);

    // ---- shrinkage: four proposals of the all-rejected path per round ----
    int ns = 0;
    bool accepted = false;
    float t_acc = 0.f, e_acc = 0.f, lp_acc = 0.f;
    for (int base = 0; base < maxs && !accepted; base += kNG) {
      float mine = 0.f, l2 = lft, r2 = rgt;
#pragma unroll
      for (int i = 0; i < kNG; ++i) {
        const int q = h + 2 + base + i;
        const uint4 ub = philox_block(r, it, s_gid, kPhaseHrss, j, static_cast<uint32_t>(q >> 2));
        const float ti = fmaf(u01(word(ub, q & 3)), r2 - l2, l2);
        if (g == i) mine = ti;
        if (ti < 0.f) l2 = ti; else r2 = ti;  // R-13
      }
      const int navail = min(kNG, maxs - base);
      const bool act = g < navail;
      const GProbe o = group_probe<NPG, KIND>(mine, x, v, pr, en, gl, d, log_y, e_star, act);
      const unsigned bok = group_ballot(act && o.ok), bpass = group_ballot(act && o.pass),
                     bnan = group_ballot(act && o.nan);
      const int first = __ffs(bok) - 1;
      const int tested = first >= 0 ? first + 1 : navail;
      n_probe += tested;
      n_eval += __popc(bpass & low_bits(tested));
      nan_seen = nan_seen || ((bnan & low_bits(tested)) != 0);
      ns += tested;
      if (first >= 0) {
        accepted = true;
        t_acc = __shfl_sync(0xffffffffu, mine, first * kG);
        e_acc = __shfl_sync(0xffffffffu, o.e, first * kG);
        lp_acc = __shfl_sync(0xffffffffu, o.lp, first * kG);
      } else {
        lft = l2;
        rgt = r2;
      }
    }
    if (accepted) {
#pragma unroll
      for (int q = 0; q < NPG; ++q) x[q] = fmaf(t_acc, v[q], x[q]);
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

  // ---- replace: group 0 writes ----
  if (g == 0) {
#pragma unroll
    for (int q = 0; q < NPG; ++q) {
      const int i = gl + kG * q;
      if (i < d) r.X[static_cast<long long>(s_gid) * r.dp + i] = x[q];
    }
  }
  if (lane == 0) {
    r.E[s_gid] = e;
    if (par != s_gid) r.birth[s_gid] = e_star;
    if (nan_seen) raise_error(st, NSS_ERR_NAN);
    atomicAdd(&st->probes, n_probe);
    atomicAdd(&st->evals, n_eval);
    atomicAdd(&st->expansions, n_exp);
    atomicAdd(&st->shrinks, n_shr);
    atomicAdd(&st->nulls, n_null);
  }
}

template <int NPG, int KIND>
void launch_group_t(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  const int nc = r.c1 - r.c0;
  if (nc <= 0) return;
  const int wpb = 8;
  NSS_PIN_CARVEOUT((k_hrss_group<NPG, KIND>));
  k_hrss_group<NPG, KIND><<<(nc + wpb - 1) / wpb, wpb * 32, 0, lc.stream>>>(r, pr, en);
  ++*lc.launch_counter;
}

template <int KIND>
void launch_group_kind(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  switch ((r.d + kG - 1) / kG) {
    case 5: launch_group_t<5, KIND>(r, pr, en, lc); break;
    case 6: launch_group_t<6, KIND>(r, pr, en, lc); break;
    case 7: launch_group_t<7, KIND>(r, pr, en, lc); break;
    case 8: launch_group_t<8, KIND>(r, pr, en, lc); break;
    case 9: launch_group_t<9, KIND>(r, pr, en, lc); break;
    case 10: launch_group_t<10, KIND>(r, pr, en, lc); break;
    case 11: launch_group_t<11, KIND>(r, pr, en, lc); break;
    case 12: launch_group_t<12, KIND>(r, pr, en, lc); break;
    case 13: launch_group_t<13, KIND>(r, pr, en, lc); break;
    case 14: launch_group_t<14, KIND>(r, pr, en, lc); break;
    case 15: launch_group_t<15, KIND>(r, pr, en, lc); break;
    default: launch_group_t<16, KIND>(r, pr, en, lc); break;
  }
}

}  // namespace

// Cheap energies at large d with precomputed directions, standard NS.
// Opt-in (NSS_GROUP=1): at C3b it is parity-green but slower than the warp
// engine (1.93 vs 1.40 ms per iteration): fewer dependent rounds per step,
// but each costs more (13 coordinates per lane, 125 registers, the shrink
// round's four Philox blocks).
bool group_engine_ok(const RunDev &r, const EnergyDev &en) {
  static const bool on = getenv("NSS_GROUP") != nullptr;
  return on && (en.kind == NSS_E_FUNNEL || en.kind == NSS_E_GAUSS) && r.d > 32 && r.Vpre && !r.tempered &&
         r.mutation == NSS_MUT_HRSS;
}

void launch_hrss_group(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc) {
  if (en.kind == NSS_E_FUNNEL)
    launch_group_kind<NSS_E_FUNNEL>(r, pr, en, lc);
  else
    launch_group_kind<NSS_E_GAUSS>(r, pr, en, lc);
}

}  // namespace nss
