// The per-chain HRSS state machine of the batched engines (P:733-749,
// identical decisions and draws to k_hrss.cu), shared by the round-synchronous
// advance kernel (k_batch.cu) and the fused GP chain kernel (k_gp.cu).
//
// One warp per chain runs the sequential HRSS state machine and stops whenever
// it needs an energy: it appends the probe point x + t v to the probe buffer
// of this round (atomic row ticket; the row index never changes the value
// computed), remembers which row it owns, and returns.  Probes that leave the
// prior support or fall below the slice height are resolved in place without
// an energy.  Both stepping-out endpoints of a side are independent of the
// other side, so a chain issues the next left and the next right endpoint in
// the same round (two probes) without evaluating anything the sequential
// algorithm would not.
#pragma once
#include <type_traits>

#include "batch.cuh"
#include "energy.cuh"

namespace nss {
namespace {

struct ChainRegs {
  int phase, step, nl, nr, ns, ldone, rdone, row0, row1;
  float l0, r0, lft, rgt, log_y, e, lp, t0, t1, lp0, lp1;
  unsigned c_probe, c_eval, c_exp, c_shr, c_null;
};

// The chain record (batch.cuh): words 0-8 the ints, 9-19 the floats, 20-24
// the counters.

__device__ __forceinline__ void load_chain(const BatchDev &b, int c, ChainRegs &s) {
  const int4 *q = b.cs + static_cast<long long>(c) * kChainWords;
  const int4 w0 = q[0], w1 = q[1], w2 = q[2], w3 = q[3], w4 = q[4], w5 = q[5], w6 = q[6];
  s.phase = w0.x; s.step = w0.y; s.nl = w0.z; s.nr = w0.w;
  s.ns = w1.x; s.ldone = w1.y; s.rdone = w1.z; s.row0 = w1.w;
  s.row1 = w2.x; s.l0 = __int_as_float(w2.y); s.r0 = __int_as_float(w2.z); s.lft = __int_as_float(w2.w);
  s.rgt = __int_as_float(w3.x); s.log_y = __int_as_float(w3.y); s.e = __int_as_float(w3.z); s.lp = __int_as_float(w3.w);
  s.t0 = __int_as_float(w4.x); s.t1 = __int_as_float(w4.y); s.lp0 = __int_as_float(w4.z); s.lp1 = __int_as_float(w4.w);
  s.c_probe = static_cast<unsigned>(w5.x); s.c_eval = static_cast<unsigned>(w5.y);
  s.c_exp = static_cast<unsigned>(w5.z); s.c_shr = static_cast<unsigned>(w5.w);
  s.c_null = static_cast<unsigned>(w6.x);
}

__device__ __forceinline__ void store_chain(const BatchDev &b, int c, const ChainRegs &s) {
  int4 *q = b.cs + static_cast<long long>(c) * kChainWords;
  q[0] = make_int4(s.phase, s.step, s.nl, s.nr);
  q[1] = make_int4(s.ns, s.ldone, s.rdone, s.row0);
  q[2] = make_int4(s.row1, __float_as_int(s.l0), __float_as_int(s.r0), __float_as_int(s.lft));
  q[3] = make_int4(__float_as_int(s.rgt), __float_as_int(s.log_y), __float_as_int(s.e), __float_as_int(s.lp));
  q[4] = make_int4(__float_as_int(s.t0), __float_as_int(s.t1), __float_as_int(s.lp0), __float_as_int(s.lp1));
  q[5] = make_int4(static_cast<int>(s.c_probe), static_cast<int>(s.c_eval), static_cast<int>(s.c_exp),
                   static_cast<int>(s.c_shr));
  q[6] = make_int4(static_cast<int>(s.c_null), 0, 0, 0);
}

// energy of probe row `row` of the given parity: the slices are loaded by the
// lanes of the chain's group in parallel and summed by a fixed shuffle tree
// (deterministic); every lane returns the total
template <int W = 32>
__device__ __forceinline__ float probe_energy(const BatchDev &b, int parity, int row, int lane) {
  if (b.eacc[parity])  // logistic regression: exact softplus sum + theta~ . g, one rounding
    return static_cast<float>(b.eacc[parity][row] + static_cast<double>(b.lin[parity][row]));
  const int ns = b.slices[parity];
  double acc = 0.0;
  for (int q = lane; q < ns; q += W) acc += b.partial[parity][static_cast<long long>(q) * b.p_stride + row];
  if (b.lin[parity] && lane == 0) acc += static_cast<double>(b.lin[parity][row]);  // logistic regression: theta . g
  return static_cast<float>(group_sum<W>(acc));
}

// Probe row `row`: for the tensor-core logistic regression only the fp16 hi /
// lo terms of its coordinates (K padded to 128) and the linear term
// theta~ . g (theta~ = hi + lo, the terms the tensor cores contract, R-28),
// no fp32 row; otherwise the fp32 coordinates.
template <int NPL, int W>
__device__ __forceinline__ void emit_probe(const BatchDev &b, int parity, int row, const float (&xp)[NPL], int d,
                                           int lane) {
  if (b.A[parity]) {
    __half *A = b.A[parity];
    float lin = 0.f;
#pragma unroll
    for (int t = 0; t < 128 / W; ++t) {
      const int kk = lane + W * t;
      const float v = (t < NPL && kk < d) ? xp[t < NPL ? t : 0] : 0.f;
      const __half hi = __float2half_rn(v);
      const __half lo = __float2half_rn(v - __half2float(hi));
      A[static_cast<long long>(row) * 128 + kk] = hi;
      A[(static_cast<long long>(b.p_stride) + row) * 128 + kk] = lo;
      lin = fmaf(__half2float(hi) + __half2float(lo), __ldg(b.g + kk), lin);
    }
    lin = group_sum<W>(lin);
    if (lane == 0) {
      b.lin[parity][row] = lin;
      b.eacc[parity][row] = 0.0;  // the energy pass adds the softplus sums
    }
    return;
  }
  float *dst = b.P[parity] + static_cast<long long>(row) * b.dp;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + W * t;
    if (i < d) dst[i] = xp[t];
  }
}

// A group of W lanes (a warp, or half a warp: two chains per warp when the
// directions are precomputed) advances chain c: fold in the energies of the
// probes it issued in the previous round (parity ^ 1), run the sequential HRSS
// state machine until it needs new energies (probes appended to the rows of
// `parity`) or finishes its p steps; the state lives in the BatchDev arrays
// between calls.  sZ: NPL * 32 floats of shared memory owned by the warp
// (in-chain directions, W = 32 only).
//
// Row tickets: with a `ticket` functor (the round-synchronous advance kernel)
// the chain first runs its state machine recording the probe parameters, then
// calls ticket(n) exactly once -- every warp of the block does, even with
// n = 0 -- which hands out n consecutive rows with ONE atomic per block (the
// round's 10^4 same-address atomics serialised at the L2); without one (the
// fused GP kernel) every probe takes its row with its own atomic.
struct NoTicket {
  __device__ int operator()(int) const { return 0; }
};

template <int NPL, int W = 32, class Ticket = NoTicket>
__device__ __forceinline__ void advance_chain(const RunDev &r, const PriorDev &pr, const BatchDev &b, int parity,
                                              int c, float *sZ, Ticket ticket = Ticket{}) {
  constexpr bool kDefer = !std::is_same<Ticket, NoTicket>::value;
  const int d = r.d, lane = threadIdx.x & (W - 1);
  const DevState *st = r.st;
  if (st->terminated || st->error || st->finalised) return;  // uniform (written by other kernels)
  ChainRegs s;
  load_chain(b, c, s);
  if (s.phase == kPhDone) {
    if constexpr (kDefer) (void)ticket(0);
    return;
  }

  const uint32_t it = static_cast<uint32_t>(st->iter)  /* set by the select kernel */;
  const int dest = r.cdest[c];
  const float e_star = st->e_star, w = st->width;
  const int p = r.p, cap = r.max_stepout, maxs = r.max_shrink;
  const bool euclid = r.dir_norm == NSS_DIR_EUCLIDEAN;
  const int h = 2 * ((d + 1) / 2);
  const int nblk_norm = h >> 2, nblk_all = (h + 3) >> 2;
  const int prev = parity ^ 1;

  // W = 32: the prior's parameters in registers; half-warp groups read them
  // per test (register budget)
  constexpr int NPR = W == 32 ? NPL : 1;
  float pa[NPR], pb[NPR], x[NPL], v[NPL], xp[NPL];
  if constexpr (W == 32) load_prior_lane<NPL, W>(pr, lane, d, pa, pb);
  // the direction of the current step: from the precomputed directions when
  // there are any (then never stored back), else the chain's saved copy
  const float *vsrc = (r.Vpre && s.phase != kPhDir)
                          ? r.Vpre + (static_cast<long long>(c - chain_range(r).x) * p + s.step) * r.dp
                          : b.v + static_cast<long long>(c) * b.dp;
  // ... and the direction of the next step, loaded with the rest so a step
  // ending in this call does not wait for it
  const int jn = s.phase == kPhDir ? s.step : s.step + 1;
  const bool have_next = r.Vpre && jn < p;
  const float *vnsrc = r.Vpre + (static_cast<long long>(c - chain_range(r).x) * p + (have_next ? jn : 0)) * r.dp;
  float vn[NPL];
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + W * t;
    x[t] = i < d ? b.x[static_cast<long long>(c) * b.dp + i] : 0.f;
    v[t] = i < d ? vsrc[i] : 0.f;
    vn[t] = (have_next && i < d) ? __ldg(vnsrc + i) : 0.f;
  }
  bool x_dirty = false;
  // results of the probes this chain issued last round
  float E0 = 0.f, E1 = 0.f;
  if (s.row0 >= 0) E0 = probe_energy<W>(b, prev, s.row0, lane);
  if (s.row1 >= 0) E1 = probe_energy<W>(b, prev, s.row1, lane);
  bool nan_seen = false;

  // in-slice test of x + t v against the prior part (support and height);
  // returns false when no energy is needed because the point is out
  auto prior_ok = [&](float tt, float &lpp) -> bool {
#pragma unroll
    for (int q = 0; q < NPL; ++q) xp[q] = fmaf(tt, v[q], x[q]);
    bool inside;
    if constexpr (W == 32)
      lpp = prior_logp<NPL, W>(xp, pr, pa, pb, lane, d, inside);
    else
      lpp = prior_logp_mem<NPL, W>(xp, pr, lane, d, inside);
    return inside && (lpp >= s.log_y);
  };
  float pend_t[2];
  int npend = 0;
  auto issue = [&](float tt) -> int {
    if constexpr (kDefer) {  // row after the block's ticket; placeholder -2 - k
      pend_t[npend] = tt;
      return -2 - npend++;
    }
    int row = 0;
    if (lane == 0) row = atomicAdd(&b.n_probe[parity], 1);
    row = __shfl_sync(group_mask<W>(), row, 0, W);
#pragma unroll
    for (int q = 0; q < NPL; ++q) xp[q] = fmaf(tt, v[q], x[q]);
    emit_probe<NPL, W>(b, parity, row, xp, d, lane);
    return row;
  };
  auto end_step = [&](int accepted) {
    s.c_exp += s.nl + s.nr;
    s.c_shr += s.ns;
    s.c_null += accepted ? 0 : 1;
    if (lane == 0)
      r.counts[static_cast<long long>(c) * p + s.step] =
          static_cast<uint32_t>(s.nl) | (static_cast<uint32_t>(s.nr) << 8) | (static_cast<uint32_t>(s.ns) << 16) |
          (static_cast<uint32_t>(accepted) << 24);
    s.step += 1;
    s.phase = kPhDir;
  };

  bool wait = false;
  while (!wait && s.phase != kPhDone) {
    if (s.phase == kPhDir) {
      if (s.step >= p) {
        s.phase = kPhDone;
        break;
      }
      const int j = s.step;
      if (r.Vpre && have_next && j == jn) {  // prefetched with the state
#pragma unroll
        for (int t = 0; t < NPL; ++t) v[t] = vn[t];
      } else if (r.Vpre) {  // precomputed for this (chain, step) by k_dirs (fp64 tensor-core products)
        const float *vr = r.Vpre + (static_cast<long long>(c - chain_range(r).x) * p + j) * r.dp;
#pragma unroll
        for (int t = 0; t < NPL; ++t) {
          const int i = lane + W * t;
          v[t] = i < d ? __ldg(vr + i) : 0.f;
        }
      } else if constexpr (W == 32) {
      // direction v = L z / |z| (R-6), stream (it, dest, HRSS, j)
      for (int bk = lane; bk < nblk_all; bk += 32) {
        const uint4 u4 = philox_block(r, it, dest, kPhaseHrss, j, bk);
        const float r0 = sqrtf(-2.f * logf(u01(u4.x))), r1 = sqrtf(-2.f * logf(u01(u4.z)));
        float s0, c0, s1, c1;
        sincospif(2.f * u01(u4.y), &s0, &c0);
        sincospif(2.f * u01(u4.w), &s1, &c1);
        const int i0 = 4 * bk;
        if (i0 < d) sZ[i0] = r0 * c0;
        if (i0 + 1 < d) sZ[i0 + 1] = r0 * s0;
        if (bk < nblk_norm) {
          if (i0 + 2 < d) sZ[i0 + 2] = r1 * c1;
          if (i0 + 3 < d) sZ[i0 + 3] = r1 * s1;
        }
      }
      __syncwarp();
      // v = L z, column by column: column m of L is contiguous in LT, so each
      // step is one coalesced load per lane-row block
      float zz = 0.f, vv = 0.f;
#pragma unroll
      for (int t = 0; t < NPL; ++t) v[t] = 0.f;
#pragma unroll 8
      for (int m = 0; m < d; ++m) {  // unrolled: 8 columns of loads in flight
        const float zm = sZ[m];
        const float *col = r.LT + static_cast<long long>(m) * r.dp;
#pragma unroll
        for (int t = 0; t < NPL; ++t) {
          const int i = lane + 32 * t;
          if (i < d) v[t] = fmaf(__ldg(col + i), zm, v[t]);  // L[i][m] = 0 for m > i
        }
      }
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        const int i = lane + 32 * t;
        if (i < d) {
          const float zi = sZ[i];
          zz = fmaf(zi, zi, zz);
        }
        vv = fmaf(v[t], v[t], vv);
      }
      const float inv = 1.f / sqrtf(warp_sum(euclid ? vv : zz));
#pragma unroll
      for (int t = 0; t < NPL; ++t) v[t] *= inv;
      __syncwarp();
      } else {
        __trap();  // half-warp groups run only with precomputed directions
      }
      const uint4 hb = philox_block(r, it, dest, kPhaseHrss, j, h >> 2);
      s.log_y = s.lp + logf(u01(word(hb, h & 3)));
      s.l0 = -w * u01(word(hb, (h + 1) & 3));
      s.r0 = s.l0 + w;
      s.nl = s.nr = s.ns = 0;
      s.ldone = s.rdone = 0;
      s.row0 = s.row1 = -1;
      s.phase = kPhStepOut;
      continue;
    }
    if (s.phase == kPhStepOut) {
      // fold in last round's endpoint results (R-10)
      if (s.row0 >= 0) {
        s.c_eval += 1;
        nan_seen = nan_seen || isnan(E0);
        if (E0 < e_star) s.nl += 1; else s.ldone = 1;
        s.row0 = -1;
      }
      if (s.row1 >= 0) {
        s.c_eval += 1;
        nan_seen = nan_seen || isnan(E1);
        if (E1 < e_star) s.nr += 1; else s.rdone = 1;
        s.row1 = -1;
      }
      // next endpoints: resolve prior-rejected ones in place, issue the rest
      while (!s.ldone) {
        if (s.nl >= cap) { s.ldone = 1; break; }
        const float tt = fmaf(-static_cast<float>(s.nl), w, s.l0);
        s.c_probe += 1;
        float lpp;
        if (!prior_ok(tt, lpp)) { s.ldone = 1; break; }
        s.row0 = issue(tt);
        s.t0 = tt;
        s.lp0 = lpp;
        break;
      }
      while (!s.rdone) {
        if (s.nr >= cap) { s.rdone = 1; break; }
        const float tt = fmaf(static_cast<float>(s.nr), w, s.r0);
        s.c_probe += 1;
        float lpp;
        if (!prior_ok(tt, lpp)) { s.rdone = 1; break; }
        s.row1 = issue(tt);
        s.t1 = tt;
        s.lp1 = lpp;
        break;
      }
      if (s.row0 != -1 || s.row1 != -1) {
        wait = true;
        break;
      }
      s.lft = fmaf(-static_cast<float>(s.nl), w, s.l0);
      s.rgt = fmaf(static_cast<float>(s.nr), w, s.r0);
      s.ns = 0;
      s.phase = kPhShrink;
      continue;
    }
    // ---- shrinkage (R-12/R-13) ----
    if (s.row0 >= 0) {
      s.c_eval += 1;
      nan_seen = nan_seen || isnan(E0);
      s.row0 = -1;
      if (E0 < e_star) {
#pragma unroll
        for (int q = 0; q < NPL; ++q) x[q] = fmaf(s.t0, v[q], x[q]);
        x_dirty = true;
        s.e = E0;
        s.lp = s.lp0;
        end_step(1);
        continue;
      }
      if (s.t0 < 0.f) s.lft = s.t0; else s.rgt = s.t0;
    }
    bool issued = false;
    while (s.ns < maxs) {
      const int q = h + 2 + s.ns;
      const uint4 ub = philox_block(r, it, dest, kPhaseHrss, s.step, static_cast<uint32_t>(q >> 2));
      const float tt = fmaf(u01(word(ub, q & 3)), s.rgt - s.lft, s.lft);
      s.ns += 1;
      s.c_probe += 1;
      float lpp;
      if (!prior_ok(tt, lpp)) {
        if (tt < 0.f) s.lft = tt; else s.rgt = tt;
        continue;
      }
      s.row0 = issue(tt);
      s.t0 = tt;
      s.lp0 = lpp;
      issued = true;
      break;
    }
    if (issued) {
      wait = true;
      break;
    }
    end_step(0);  // shrink cap reached: null move
  }

  if constexpr (kDefer) {
    // the block's rows, then the recorded probes (the same fp32 points)
    const int base = ticket(npend);
    for (int k = 0; k < npend; ++k) {
      const float tt = pend_t[k == 0 ? 0 : 1];
#pragma unroll
      for (int q = 0; q < NPL; ++q) xp[q] = fmaf(tt, v[q], x[q]);
      emit_probe<NPL, W>(b, parity, base + k, xp, d, lane);
    }
    if (s.row0 <= -2) s.row0 = base + (-2 - s.row0);
    if (s.row1 <= -2) s.row1 = base + (-2 - s.row1);
  }
  // write back only what changed: x after an accepted step, v when it is not
  // re-read from the precomputed directions
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + W * t;
    if (i < d) {
      if (x_dirty) b.x[static_cast<long long>(c) * b.dp + i] = x[t];
      if (!r.Vpre) b.v[static_cast<long long>(c) * b.dp + i] = v[t];
    }
  }
  if (lane == 0) {
    store_chain(b, c, s);
    if (nan_seen) raise_error(r.st, NSS_ERR_NAN);
  }
}

}  // namespace
}  // namespace nss
