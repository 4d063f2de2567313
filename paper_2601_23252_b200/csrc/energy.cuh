// Energy parameters in shared memory and per-lane energies / priors shared by
// the two HRSS engines (k_hrss.cu: warp-cooperative, k_hrss_lane.cu: one probe
// per lane).  E(x) = -log L(x) as defined in include/nss.h.
#pragma once
#include "nss_internal.cuh"

namespace nss {

constexpr float kLn2Pi = 1.8378770664093453f;
constexpr unsigned kFull = 0xffffffffu;

struct ESm {          // shared-memory image of the energy parameters
  const float *mu;    // GAUSS/CORR: d; MOG: K*d
  const float *isig;  // GAUSS: d; MOG: K*d
  const float *logc;  // MOG: K
  const float *prec;  // CORR: d rows of stride ldp (the precision P, or its factor U when tri)
  int ldp;
  bool tri;           // CORR: rows hold U with P = U^T U (upper triangular): q = |U r|^2
};

__host__ __device__ inline int odd_stride(int d) { return d | 1; }

// number of floats of energy parameters staged in shared memory
__host__ __device__ inline int energy_param_floats(int kind, int d, int K) {
  switch (kind) {
    case NSS_E_GAUSS: return 2 * d;
    case NSS_E_MOG: return 2 * K * d + K;
    case NSS_E_CORR_GAUSS: return d + d * odd_stride(d);
    default: return 0;
  }
}

__device__ inline void stage_energy(const EnergyDev &en, float *sp, ESm &es) {
  const int d = en.d, tid = threadIdx.x, nt = blockDim.x;
  es.ldp = odd_stride(d);
  es.mu = es.isig = es.logc = es.prec = nullptr;
  es.tri = false;
  if (en.kind == NSS_E_GAUSS) {
    for (int i = tid; i < d; i += nt) { sp[i] = en.mu[i]; sp[d + i] = en.isig[i]; }
    es.mu = sp; es.isig = sp + d;
  } else if (en.kind == NSS_E_MOG) {
    const int K = en.n_comp;
    for (int i = tid; i < K * d; i += nt) { sp[i] = en.mu[i]; sp[K * d + i] = en.isig[i]; }
    for (int j = tid; j < K; j += nt) sp[2 * K * d + j] = en.logc[j];
    es.mu = sp; es.isig = sp + K * d; es.logc = sp + 2 * K * d;
  } else if (en.kind == NSS_E_CORR_GAUSS) {
    for (int i = tid; i < d; i += nt) sp[i] = en.mu[i];
    float *P = sp + d;
    const float *src = en.ufac ? en.ufac : en.prec;  // the triangular factor halves the work
    for (int e = tid; e < d * d; e += nt) {
      int i = e / d, j = e - i * d;
      P[i * es.ldp + j] = src[e];
    }
    es.mu = sp; es.prec = P; es.tri = en.ufac != nullptr;
  }
}

__device__ __forceinline__ float softplusf(float a) {
  return a > 0.f ? a + log1pf(expf(-a)) : log1pf(expf(a));
}

// Lane groups of W lanes (W = 32: a warp; 16: half a warp, two groups per
// warp): the member mask and sums over the group (fixed xor tree).
template <int W>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (W == 32) return 0xffffffffu;
  return ((1u << W) - 1u) << (threadIdx.x & 31 & ~(W - 1));
}
template <int W, class T>
__device__ __forceinline__ T group_sum(T v) {
  const unsigned m = group_mask<W>();
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o, W);
  return v;
}

// Per-lane prior parameters for the coordinates a lane owns (lane of a group of W).
template <int NPL, int W = 32>
__device__ __forceinline__ void load_prior_lane(const PriorDev &pr, int lane, int d, float (&pa)[NPL],
                                                float (&pb)[NPL]) {
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + W * t;
    if (pr.kind == NSS_PRIOR_BOX) {
      pa[t] = i < d ? pr.lo[i] : 0.f;
      pb[t] = i < d ? pr.hi[i] : 0.f;
    } else {
      pa[t] = i < d ? pr.mean[i] : 0.f;
      pb[t] = i < d ? pr.isd[i] : 0.f;
    }
  }
}

// Attempt `a` of the prior draw of live point g (R-20, phase INIT): box
// coordinates u (hi - lo) + lo, Gaussian ones by Box-Muller pairs (2m, 2m+1).
template <int NPL>
__device__ __forceinline__ void prior_draw(const RunDev &r, const PriorDev &pr, int g, uint32_t a, int lane,
                                           const float (&pa)[NPL], const float (&pb)[NPL], float (&x)[NPL]) {
  const int d = r.d;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    x[t] = 0.f;
    if (i < d) {
      if (pr.kind == NSS_PRIOR_BOX) {
        uint4 b = philox_block(r, 0, g, kPhaseInit, a, i >> 2);
        x[t] = fmaf(u01(word(b, i & 3)), pb[t] - pa[t], pa[t]);
      } else {
        const int m = i >> 1;  // Box-Muller pair (2m, 2m+1)
        uint4 b = philox_block(r, 0, g, kPhaseInit, a, (2 * m) >> 2);
        const float u1 = u01(word(b, (2 * m) & 3)), u2 = u01(word(b, (2 * m + 1) & 3));
        const float rr = sqrtf(-2.f * logf(u1));
        float sn, cs;
        sincospif(2.f * u2, &sn, &cs);
        const float z = (i & 1) ? rr * sn : rr * cs;
        x[t] = fmaf(z, pr.sd[i], pa[t]);
      }
    }
  }
}

// Warp-cooperative energy E(x); the result is identical in every lane.
// `wbuf` is a per-warp shared buffer of NPL*32 floats.
template <int NPL, int KIND>
__device__ __forceinline__ float warp_energy(const float (&x)[NPL], const EnergyDev &en, const ESm &es,
                                             float *wbuf, int lane) {
  const int d = en.d;
  if constexpr (KIND == NSS_E_FLAT) {
    return en.c;
  } else if constexpr (KIND == NSS_E_GAUSS) {
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      if (i < d) {
        float u = (x[t] - es.mu[i]) * es.isig[i];
        s = fmaf(u, u, s);
      }
    }
    return 0.5f * warp_sum(s) + en.c;
  } else if constexpr (KIND == NSS_E_MOG) {
    // online log-sum-exp over components; unrolling lets the K independent
    // butterfly reductions overlap
    float m = -INFINITY, acc = 0.f;
#pragma unroll 4
    for (int j = 0; j < en.n_comp; ++j) {
      float s = 0.f;
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        const int i = lane + 32 * t;
        if (i < d) {
          float u = (x[t] - es.mu[j * d + i]) * es.isig[j * d + i];
          s = fmaf(u, u, s);
        }
      }
      s = warp_sum(s);
      const float l = es.logc[j] - 0.5f * s;
      if (l > m) {
        acc = acc * __expf(m - l) + 1.f;
        m = l;
      } else {
        acc += __expf(l - m);
      }
    }
    return -(m + __logf(acc));
  } else if constexpr (KIND == NSS_E_CORR_GAUSS) {
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      if (i < d) wbuf[i] = x[t] - es.mu[i];
    }
    __syncwarp();
    float q = 0.f;
    if (es.tri) {
      // (U r)_i = sum_{m >= i} U_im r_m, q = sum_i (U r)_i^2.  Column
      // segment s = [32 s, 32 s + 32) only meets rows t <= s (U is zero below
      // the diagonal), so the loop is uniform across lanes and the rows of a
      // lane accumulate as independent chains (two per row in segment 0).
      float acc[NPL], acc0b = 0.f;
#pragma unroll
      for (int t = 0; t < NPL; ++t) acc[t] = 0.f;
      const float *rows[NPL];
#pragma unroll
      for (int t = 0; t < NPL; ++t) rows[t] = es.prec + (lane + 32 * t < d ? lane + 32 * t : 0) * es.ldp;
#pragma unroll
      for (int sg = 0; sg < NPL; ++sg) {
        const int m0 = 32 * sg, m1 = min(d, m0 + 32);
        int m = m0;
        if (sg == 0) {
          for (; m + 1 < m1; m += 2) {
            acc[0] = fmaf(rows[0][m], wbuf[m], acc[0]);
            acc0b = fmaf(rows[0][m + 1], wbuf[m + 1], acc0b);
          }
        }
        for (; m < m1; ++m) {
          const float w = wbuf[m];
#pragma unroll
          for (int t = 0; t < NPL; ++t)
            if (t <= sg) acc[t] = fmaf(rows[t][m], w, acc[t]);
        }
      }
      acc[0] += acc0b;
#pragma unroll
      for (int t = 0; t < NPL; ++t)
        if (lane + 32 * t < d) q = fmaf(acc[t], acc[t], q);
    } else {
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      if (i < d) {
        const float *row = es.prec + i * es.ldp;
        float py = 0.f;
        for (int m = 0; m < d; ++m) py = fmaf(row[m], wbuf[m], py);  // (P r)_i; q = sum_i r_i (P r)_i
        q = fmaf(wbuf[i], py, q);
      }
    }
    }
    q = warp_sum(q);
    __syncwarp();
    return 0.5f * q + en.c;
  } else if constexpr (KIND == NSS_E_FUNNEL) {
    // P:885 (R-23): x_0 = y ~ N(0, sy^2), x_n ~ N(0, e^y)
    const float y = __shfl_sync(kFull, x[0], 0);
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      if (i >= 1 && i < d) s = fmaf(x[t], x[t], s);
    }
    s = warp_sum(s);
    const float sy = en.sigma_y;
    const float yy = y / sy;
    return 0.5f * yy * yy + logf(sy) + 0.5f * kLn2Pi + 0.5f * s * expf(-y) +
           static_cast<float>(d - 1) * 0.5f * (y + kLn2Pi);
  } else if constexpr (KIND == NSS_E_LOGREG) {
    // naive warp path (lanes over data rows); the batched tensor-core engine is
    // the production path for large N
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + 32 * t;
      if (i < d) wbuf[i] = x[t];
    }
    __syncwarp();
    float acc = 0.f;
    for (long long rr = lane; rr < en.n_data; rr += 32) {
      const float *row = en.data_x + rr * d;
      float a = 0.f;
      for (int m = 0; m < d; ++m) a = fmaf(row[m], wbuf[m], a);
      acc += softplusf(a) - en.data_y[rr] * a;
    }
    acc = warp_sum(acc);
    __syncwarp();
    return acc;
  } else {
    return NAN;
  }
}

// Correlated-Gaussian energy split over the WPC = 2 warps of a chain (large
// d, factored form): both warps hold the same point; warp `sub` takes the
// row blocks {0, 3} (sub 0) or {1, 2} (sub 1) of U -- balanced work, since
// row block t only meets column segments >= t -- and the two partial sums
// meet in shared memory behind a named barrier of the chain's 64 threads.
// red: 4 floats per chain (two parities x two warps); `par` alternates per
// call so one barrier per call suffices.  Identical result in both warps.
template <int NPL>
__device__ __forceinline__ float corr_energy_split(const float (&x)[NPL], const EnergyDev &en, const ESm &es,
                                                   float *wbuf, float *red, int lane, int sub, int bar_id,
                                                   int &par) {
  const int d = en.d;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    if (i < d) wbuf[i] = x[t] - es.mu[i];  // both warps write the same values
  }
  __syncwarp();
  float q = 0.f;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const bool mine = (sub == 0) ? (t == 0 || t == 3) : (t == 1 || t == 2);
    const int i = lane + 32 * t;
    if (mine && i < d) {
      const float *row = es.prec + i * es.ldp;
      float a0 = 0.f, a1 = 0.f;
      int m = 32 * t;
      for (; m + 1 < d; m += 2) {
        a0 = fmaf(row[m], wbuf[m], a0);
        a1 = fmaf(row[m + 1], wbuf[m + 1], a1);
      }
      if (m < d) a0 = fmaf(row[m], wbuf[m], a0);
      const float a = a0 + a1;
      q = fmaf(a, a, q);
    }
  }
  q = warp_sum(q);
  if (lane == 0) red[par * 2 + sub] = q;
  asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
  const float tot = red[par * 2] + red[par * 2 + 1];
  par ^= 1;
  __syncwarp();
  return 0.5f * tot + en.c;
}

// The same energy split over WPC = 4 warps of a chain: the rows' dot products
// (row block t covers columns [32 t, d)) are laid end to end and cut into four
// equal runs of columns, so a warp takes at most a few pieces (t, [m0, m1));
// piece k of row block t leaves its partial dot products in slot (t, k) of
// `red` (4 x 4 x 32 floats + 4), the chain's 128 threads meet at a named
// barrier, warp t sums the slots of row block t in slot order and squares,
// and a second barrier publishes the four row-block sums.  Deterministic
// (fixed slots and orders); identical result in all four warps.
template <int NPL>
__device__ __forceinline__ float corr_energy_split4(const float (&x)[NPL], const EnergyDev &en, const ESm &es,
                                                    float *wbuf, float *red, int lane, int sub, int bar_id) {
  const int d = en.d, nb = (d + 31) >> 5;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    if (i < d) wbuf[i] = x[t] - es.mu[i];  // all warps write the same values
  }
  __syncwarp();
  int total = 0;
  for (int t = 0; t < nb; ++t) total += d - 32 * t;
  const int lo = sub * total / 4, hi = (sub + 1) * total / 4;
  int cum = 0;
  for (int t = 0; t < nb; ++t) {
    const int len = d - 32 * t;
    const int a0 = max(lo, cum), a1 = min(hi, cum + len);
    if (a0 < a1) {
      const int k = sub - (cum * 4) / total;  // warps before this one in row block t
      const int i = 32 * t + lane;
      float s0 = 0.f, s1 = 0.f;
      if (i < d) {
        const float *row = es.prec + i * es.ldp;
        int m = 32 * t + (a0 - cum);
        const int m1 = 32 * t + (a1 - cum);
        for (; m + 1 < m1; m += 2) {
          s0 = fmaf(row[m], wbuf[m], s0);
          s1 = fmaf(row[m + 1], wbuf[m + 1], s1);
        }
        if (m < m1) s0 = fmaf(row[m], wbuf[m], s0);
      }
      red[(t * 4 + k) * 32 + lane] = s0 + s1;
    }
    cum += len;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
  float q = 0.f;
  if (sub < nb) {  // warp t: row block t
    const int t = sub;
    int c0 = 0;
    for (int u = 0; u < t; ++u) c0 += d - 32 * u;
    const int first = (c0 * 4) / total, last = ((c0 + d - 32 * t - 1) * 4) / total;
    float a = 0.f;
    for (int k = 0; k <= last - first; ++k) a += red[(t * 4 + k) * 32 + lane];
    if (32 * t + lane < d) q = a * a;
    q = warp_sum(q);
    if (lane == 0) red[16 * 32 + t] = q;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
  float tot = 0.f;
  for (int t = 0; t < nb; ++t) tot += red[16 * 32 + t];
  __syncwarp();
  return 0.5f * tot + en.c;
}

// log Pi(x) and support test (box: all lanes inside; Gaussian: always inside),
// over the W lanes of the caller's group.
template <int NPL, int W = 32>
__device__ __forceinline__ float prior_logp(const float (&x)[NPL], const PriorDev &pr, const float (&pa)[NPL],
                                            const float (&pb)[NPL], int lane, int d, bool &inside) {
  if (pr.kind == NSS_PRIOR_BOX) {
    bool ok = true;
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + W * t;
      if (i < d) ok = ok && (x[t] >= pa[t]) && (x[t] <= pb[t]);
    }
    const unsigned m = group_mask<W>();
    inside = (__ballot_sync(m, ok) & m) == m;
    return pr.log_norm;
  }
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + W * t;
    if (i < d) {
      float u = (x[t] - pa[t]) * pb[t];
      s = fmaf(u, u, s);
    }
  }
  inside = true;
  return -0.5f * group_sum<W>(s) + pr.log_norm;
}

// prior_logp with the prior's parameters read from memory per call instead
// of held in registers (the register-tight half-warp advance).
template <int NPL, int W>
__device__ __forceinline__ float prior_logp_mem(const float (&x)[NPL], const PriorDev &pr, int lane, int d,
                                                bool &inside) {
  if (pr.kind == NSS_PRIOR_BOX) {
    bool ok = true;
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int i = lane + W * t;
      if (i < d) ok = ok && (x[t] >= __ldg(pr.lo + i)) && (x[t] <= __ldg(pr.hi + i));
    }
    const unsigned m = group_mask<W>();
    inside = (__ballot_sync(m, ok) & m) == m;
    return pr.log_norm;
  }
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + W * t;
    if (i < d) {
      float u = (x[t] - __ldg(pr.mean + i)) * __ldg(pr.isd + i);
      s = fmaf(u, u, s);
    }
  }
  inside = true;
  return -0.5f * group_sum<W>(s) + pr.log_norm;
}

}  // namespace nss
