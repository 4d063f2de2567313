// A5 metric: live-set covariance (1/(n-1)) + ridge reg*mean(diag) (P:326-332,
// R-8), Cholesky in fp64, fallback to the diagonal, and the slice width rule
// (R-7).  At the end of an iteration the same kernel evaluates the
// termination criterion (A9, R-19) and advances the iteration counter.
//
// One launch: B CTAs accumulate shifted fp64 sums over fixed gid chunks and
// write them to `partials`; the last CTA to finish (atomic ticket) sums the B
// partials in a fixed two-level order -- the blocks of each of the kSegs gid
// segments in block order, then the segment sums in segment order -- so the
// result does not depend on which CTA is last, and a sharded live set (each
// rank owning whole segments) reaches the same sums bit for
// bit -- and factorises.  The sums are of y = x - shift, shift = the mean the
// previous metric found (the prior's centre before the first): a replicated
// vector, so every rank of a sharded run can form its partials before any
// exchange.  The Cholesky is
// row-owner, one barrier per column: thread i owns row i, every thread reads
// the pivot directly, the column is written to L (never re-read from A), so the
// trailing update needs no second barrier.  For d <= 32 it runs in one warp
// with __syncwarp.
#include "nss_internal.cuh"

namespace nss {

namespace {

constexpr int kThreads = 256;
constexpr int kLoSharedMax = 100;  // factor kept in shared memory up to this d (A + factor within 200 KB)
constexpr int kSplitMinD = 33;    // from this d on the metric is three launches (grid-wide reduction)
constexpr double kKappaInf = 1.3035;
constexpr double kPi = 3.14159265358979323846;

// shared-memory slot for the per-group entry sums, after this CTA's rows
__device__ __forceinline__ double *raw_groups(double *sm, int nent, int d, int npair, int rows, int dp) {
  double *yd = sm + nent + d + (2 * npair + 7) / 8;
  return yd + static_cast<long long>(rows) * dp;
}

// Entry e summed over the blocks of segment s in block order; loads are
// issued 8 at a time (independent), the additions stay in block order.
__device__ __forceinline__ double fold_segment(const double *partials, int s, int bps, int e, int nent1,
                                               bool is_min) {
  double acc = is_min ? INFINITY : 0.0;
  const double *p = partials + static_cast<long long>(s) * bps * nent1 + e;
  for (int b = 0; b < bps; b += 8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = b + q < bps ? p[static_cast<long long>(b + q) * nent1] : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (b + q < bps) acc = is_min ? fmin(acc, v[q]) : acc + v[q];
  }
  return acc;
}

// The whole live set's entry e: every segment folded, then the segments in
// order.  Small blocks-per-segment (the small-d case) load all kSegs x bps
// partials first, so the fold waits for one round trip instead of kSegs.
__device__ __forceinline__ double fold_all(const double *partials, int bps, int e, int nent1, bool is_min) {
  double segs[kSegs];
  if (bps <= 4) {
    double v[kSegs * 4];
#pragma unroll
    for (int q = 0; q < kSegs * 4; ++q) {
      const int s = q >> 2, b = q & 3;
      v[q] = b < bps ? partials[(static_cast<long long>(s) * bps + b) * nent1 + e] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < kSegs; ++s) {
      double acc = is_min ? INFINITY : 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (b < bps) acc = is_min ? fmin(acc, v[s * 4 + b]) : acc + v[s * 4 + b];
      segs[s] = acc;
    }
  } else {
#pragma unroll
    for (int s = 0; s < kSegs; ++s) segs[s] = fold_segment(partials, s, bps, e, nent1, is_min);
  }
  double acc = is_min ? INFINITY : 0.0;
#pragma unroll
  for (int s = 0; s < kSegs; ++s) acc = is_min ? fmin(acc, segs[s]) : acc + segs[s];
  return acc;
}

// Entry e of the whole live set: the kSegs segment sums (rows `stride`
// apart) added in segment order.
__device__ __forceinline__ double fold_segments(const double *seg, long long stride, int e, bool is_min) {
  double acc = is_min ? INFINITY : 0.0;
#pragma unroll
  for (int s = 0; s < kSegs; ++s) {
    const double v = seg[s * stride + e];
    acc = is_min ? fmin(acc, v) : acc + v;
  }
  return acc;
}

// mode 0: one launch (phase 1 in every CTA, phase 2 in the last one by
// ticket); mode 1: phase 1 only (partials written, no ticket) for the blocks
// blk0 .. blk0 + gridDim.x - 1; mode 2: phase 2 only, in one CTA, from
// `partials` already reduced to one row by k_metric_reduce (or, sharded, by
// k_metric_segfold).  Large d uses 1 -> reduce -> 2 (a grid-wide reduction
// instead of one CTA reading every partial); the sums are the same.  Blocks:
// segment s = b / bps holds blocks s bps .. s bps + bps - 1, each a chunk of
// ceil(len_s / bps) of the segment's rows.
__global__ void __launch_bounds__(kThreads) k_metric(RunDev r, double *partials, unsigned *ticket, int bps,
                                                     double reg, int width_rule, double width_param,
                                                     int end_of_iter, int mode, int blk0) {
  DevState *st = r.st;
  if (st->error) return;
  if (end_of_iter && st->finalised) return;
  extern __shared__ double sm[];
  const int d = r.d, n = r.n, tid = threadIdx.x;
  const int npair = d * (d + 1) / 2;
  const int nent = npair + d;
  double *S = sm;                         // nent accumulators
  double *shift = S + nent;               // d
  unsigned char *pi = reinterpret_cast<unsigned char *>(shift + d);
  unsigned char *pj = pi + npair;
  // this CTA's rows shifted by row 0, y = x - x_0 in fp64 (row stride dp),
  // after the pair tables: converted once here, not once per entry
  double *yd = sm + nent + d + (2 * npair + 7) / 8;
  __shared__ float red_min[kThreads / 32];
  __shared__ int sh_last;

  if (mode != 2) {
  if (tid == 0 && blockIdx.x == 0) st->stamp[8] = global_ns();
  // ---------------- phase 1: partial shifted sums of this CTA's rows ----------------
  const int blk = blk0 + static_cast<int>(blockIdx.x);
  const int seg = blk / bps, q_in = blk - seg * bps;
  const int s0 = seg_lo(n, seg), s1 = seg_lo(n, seg + 1);
  const int chunk = (s1 - s0 + bps - 1) / bps;
  const int g0 = min(s1, s0 + q_in * chunk), g1 = min(s1, g0 + chunk);
  const int rows = g1 - g0;
  const int dp = r.dp;
  // one batch of loads (the chunk is contiguous in X) while the shift loads;
  // the shift is subtracted after the barrier
  for (int i = tid; i < d; i += blockDim.x) shift[i] = r.mshift[i];
  {
    const float *src = r.X + static_cast<long long>(g0) * dp;
    for (int q = tid; q < rows * dp; q += blockDim.x) {
      const int c = q % dp;
      yd[q] = c < d ? static_cast<double>(src[q]) : 0.0;
    }
  }
  __syncthreads();
  for (int q = tid; q < rows * dp; q += blockDim.x) {
    const int c = q % dp;
    if (c < d) yd[q] -= shift[c];
  }
  float emin = INFINITY;
  for (int g = g0 + tid; g < g1; g += blockDim.x) emin = fminf(emin, r.E[g]);
  for (int e = tid; e < nent; e += blockDim.x) S[e] = 0.0;
  for (int i = tid; i < d; i += blockDim.x) {
    const int b0 = i * (i + 1) / 2;
    for (int j = 0; j <= i; ++j) {
      pi[b0 + j] = static_cast<unsigned char>(i);
      pj[b0 + j] = static_cast<unsigned char>(j);
    }
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x == 0) st->stamp[9] = global_ns();
  if (d >= kSplitMinD) {
    // large d: the chunk's Gram matrix sum_r y_r y_r^T on the fp64 tensor
    // cores -- 8 x 8 tiles of its lower triangle dealt to the warps, each
    // tile a DMMA chain over the chunk's rows four at a time (A = Y^T,
    // B = Y; rows past the chunk and columns past d read as zero) -- and the
    // first moments sum_r y_r by one thread per coordinate
    const int lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int nt8 = (d + 7) >> 3, ntile = nt8 * (nt8 + 1) / 2;
    for (int t = tid >> 5; t < ntile; t += static_cast<int>(blockDim.x >> 5)) {
      int bi = 0;
      while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
      const int bl = t - bi * (bi + 1) / 2;
      const int ia = 8 * bi + gq, la = 8 * bl + gq;
      double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
      int r0 = 0;
      for (; r0 + 8 <= rows; r0 += 8) {
        const double *y0 = yd + (r0 + tq) * dp, *y1 = y0 + 4 * dp;
        dmma_f64(c0, c1, ia < d ? y0[ia] : 0.0, la < d ? y0[la] : 0.0);
        dmma_f64(e0, e1, ia < d ? y1[ia] : 0.0, la < d ? y1[la] : 0.0);
      }
      for (; r0 < rows; r0 += 4) {
        const bool rv = r0 + tq < rows;
        const double *y0 = yd + (r0 + tq) * dp;
        dmma_f64(c0, c1, (rv && ia < d) ? y0[ia] : 0.0, (rv && la < d) ? y0[la] : 0.0);
      }
      c0 += e0;
      c1 += e1;
      const int ic = 8 * bi + gq, lc = 8 * bl + 2 * tq;
      if (ic < d && lc <= ic) S[ic * (ic + 1) / 2 + lc] = c0;
      if (ic < d && lc + 1 <= ic) S[ic * (ic + 1) / 2 + lc + 1] = c1;
    }
    for (int i = tid; i < d; i += blockDim.x) {
      double a0 = 0.0, a1 = 0.0;
      int rr = 0;
      for (; rr + 1 < rows; rr += 2) {
        a0 += yd[rr * dp + i];
        a1 += yd[(rr + 1) * dp + i];
      }
      if (rr < rows) a0 += yd[rr * dp + i];
      S[npair + i] = a0 + a1;
    }
  }
  // G row groups per entry when the entries leave threads idle (small d):
  // thread t takes entry t % nent over the rows r = grp, grp + G, ... of the
  // chunk; the G group sums are added in group order (deterministic)
  const int G = nent < static_cast<int>(blockDim.x) ? static_cast<int>(blockDim.x) / nent : 1;
  double *Sg = G > 1 ? raw_groups(sm, nent, d, npair, rows, dp) : S;  // one group: sum straight into S
  if (d < kSplitMinD) {
  for (int t = tid; t < nent * G; t += blockDim.x) {
    const int e = t % nent, grp = t / nent;
    // four independent accumulators (fixed assignment: row mod 4G) break the
    // DFMA dependency chain
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int step = 4 * G;
    if (e < npair) {
      const int i = pi[e], j = pj[e];
      int rr = grp;
      for (; rr + 3 * G < rows; rr += step) {
        a0 = fma(yd[rr * dp + i], yd[rr * dp + j], a0);
        a1 = fma(yd[(rr + G) * dp + i], yd[(rr + G) * dp + j], a1);
        a2 = fma(yd[(rr + 2 * G) * dp + i],
                 yd[(rr + 2 * G) * dp + j], a2);
        a3 = fma(yd[(rr + 3 * G) * dp + i],
                 yd[(rr + 3 * G) * dp + j], a3);
      }
      for (; rr < rows; rr += G)
        a0 = fma(yd[rr * dp + i], yd[rr * dp + j], a0);
    } else {
      const int i = e - npair;
      int rr = grp;
      for (; rr + 3 * G < rows; rr += step) {
        a0 += yd[rr * dp + i];
        a1 += yd[(rr + G) * dp + i];
        a2 += yd[(rr + 2 * G) * dp + i];
        a3 += yd[(rr + 3 * G) * dp + i];
      }
      for (; rr < rows; rr += G) a0 += yd[rr * dp + i];
    }
    Sg[grp * nent + e] = (a0 + a1) + (a2 + a3);
  }
  }
  __syncthreads();
  if (G > 1 && d < kSplitMinD)
    for (int e = tid; e < nent; e += blockDim.x) {
      double acc = 0.0;
      for (int g = 0; g < G; ++g) acc += Sg[g * nent + e];
      S[e] = acc;
    }
  __syncthreads();
  double *out = partials + static_cast<long long>(blk) * (nent + 1);
  for (int e = tid; e < nent; e += blockDim.x) out[e] = S[e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) emin = fminf(emin, __shfl_xor_sync(0xffffffffu, emin, o));
  if ((tid & 31) == 0) red_min[tid >> 5] = emin;
  __syncthreads();
  if (tid == 0) {
    float mn = red_min[0];
    for (int w = 1; w < kThreads / 32; ++w) mn = fminf(mn, red_min[w]);
    out[nent] = static_cast<double>(mn);
    if (mode == 0) {
      __threadfence();
      sh_last = atomicAdd(ticket, 1u) == static_cast<unsigned>(kSegs * bps - 1);
    }
  }
  if (mode == 1) return;
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  }
  if (tid == 0) st->stamp[10] = global_ns();

  // ---------------- phase 2 (last CTA): reduce, regularise, factorise ----------------
  const int ld = d | 1;       // odd stride: column walks are bank-conflict free
  double *A = sm;            // d*ld (reuses phase-1 shared memory)
  double *S1 = A + d * ld;   // d
  // d*d output factor: shared memory up to d = 64 (copied to L64, L, LT at the
  // end), else written straight to global
  const bool lo_shared = d <= kLoSharedMax;
  double *Lo = lo_shared ? S1 + d : r.L64;
  // lower-triangle pairs in column-major order: column j's trailing block
  // {(i, l): j < l <= i} is a contiguous suffix starting at coff(j + 1)
  unsigned char *ti = reinterpret_cast<unsigned char *>(S1 + d + (lo_shared ? d * d : 0));
  unsigned char *tl = ti + npair;
  __shared__ double sh_md;
  __shared__ double sh_red[kThreads / 32];
  __shared__ int sh_fail;
  __shared__ float sh_emin;
  for (int l = tid; l < d; l += blockDim.x) {
    const int off = l * d - l * (l - 1) / 2;  // sum_{c<l} (d - c)
    for (int i = l; i < d; ++i) {
      ti[off + i - l] = static_cast<unsigned char>(i);
      tl[off + i - l] = static_cast<unsigned char>(l);
    }
  }
  for (int e = tid; e <= nent; e += blockDim.x) {
    // fixed two-level order (blocks within a segment, then segments); entry
    // nent holds the per-block minimum energy.  mode 2: one reduced row.
    const bool is_min = e == nent;
    double acc;
    if (mode == 2) {
      acc = partials[e];
    } else {
      acc = fold_all(partials, bps, e, nent + 1, is_min);
    }
    if (is_min) {
      sh_emin = static_cast<float>(acc);
    } else if (e < npair) {
      int i = static_cast<int>((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > e) --i;
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      A[i * ld + (e - i * (i + 1) / 2)] = acc;  // S2_ij (shifted), i >= j
    } else {
      S1[e - npair] = acc;                      // S1_i  (shifted)
    }
  }
  __syncthreads();
  if (tid == 0) st->stamp[11] = global_ns();
  const double nn = static_cast<double>(n);
  // the live set's mean, the shift of the next metric's sums (every CTA of
  // this metric is past its phase 1)
  for (int i = tid; i < d; i += blockDim.x) r.mshift[i] += S1[i] / nn;
  for (int e = tid; e < d * d; e += blockDim.x) {
    const int i = e / d, j = e - i * d;
    if (j <= i) A[i * ld + j] = (A[i * ld + j] - S1[i] * S1[j] / nn) / (nn - 1.0);
    Lo[e] = 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double md = 0.0;
    for (int i = 0; i < d; ++i) md += A[i * ld + i];
    sh_md = md / d;
    sh_fail = 0;
  }
  __syncthreads();
  for (int i = tid; i < d; i += blockDim.x) {
    A[i * ld + i] += reg * sh_md;
    S1[i] = A[i * ld + i];  // regularised diagonal, kept for the fallback
  }
  __syncthreads();
  if (tid == 0) st->stamp[14] = global_ns();
  // right-looking Cholesky, one barrier per column: every thread reads the
  // pivot, writes its share of column j of L and of the trailing update
  // A_il -= A_ij A_lj / A_jj (column j itself is never rewritten)
  const bool one_warp = d <= 32;
  const int nthr = one_warp ? 32 : static_cast<int>(blockDim.x);
  if (d >= kSplitMinD) {
    // large d: blocked right-looking, 8-column panels.  Warp 0 factorises
    // the panel in registers (lane l: rows j0 + l + 32 k, pivots and panel
    // rows exchanged by shuffles, one rsqrt per column), then all threads
    // apply the rank-8 update A_il -= sum_c L_i,j0+c L_l,j0+c to the trailing
    // lower triangle: two barriers per panel instead of one per column.
    constexpr int NB = 8;
    const int ty = tid >> 4, tx = tid & 15;
#ifdef NSS_MET_PROF
    unsigned long long t_panel = 0;  // measurement builds: ns in the one-warp panel factorisations
#endif
    for (int j0 = 0; j0 < d; j0 += NB) {
#ifdef NSS_MET_PROF
      const unsigned long long tp0 = global_ns();
#endif
      const int nb = min(NB, d - j0);
      if (tid < 32) {
        double pv[4][NB];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int c = 0; c < NB; ++c) {
            const int rr = j0 + tid + 32 * k;
            pv[k][c] = (rr < d && c < nb && j0 + c <= rr) ? A[rr * ld + j0 + c] : 0.0;
          }
        bool bad = false;
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          if (c < nb && !bad) {
            const double piv = __shfl_sync(0xffffffffu, pv[0][c], c);  // row j0 + c: lane c, k = 0
            if (!(piv > 0.0) || !isfinite(piv)) {
              bad = true;  // uniform
            } else {
              const double rs = rsqrt(piv);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int rr = j0 + tid + 32 * k;
                if (rr == j0 + c) pv[k][c] = piv * rs;
                else if (rr > j0 + c) pv[k][c] *= rs;
              }
#pragma unroll
              for (int c2 = c + 1; c2 < NB; ++c2) {
                const double l2 = __shfl_sync(0xffffffffu, pv[0][c], c2);  // L_{j0+c2, j0+c}
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int rr = j0 + tid + 32 * k;
                  if (c2 < nb && rr >= j0 + c2) pv[k][c2] = fma(-pv[k][c], l2, pv[k][c2]);
                }
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int c = 0; c < NB; ++c) {
            const int rr = j0 + tid + 32 * k;
            if (rr < d && c < nb && j0 + c <= rr) {
              A[rr * ld + j0 + c] = pv[k][c];
              Lo[rr * d + j0 + c] = pv[k][c];
            }
          }
        if (bad && tid == 0) sh_fail = 1;
      }
      __syncthreads();
#ifdef NSS_MET_PROF
      t_panel += global_ns() - tp0;
      if (tid == 0 && j0 + NB >= d) st->stamp[7] = t_panel;
#endif
      if (sh_fail) break;  // uniform
      const int b0 = j0 + nb;
      for (int u = 0; u < 8; ++u) {
        const int i = b0 + ty + 16 * u;
        if (i >= d) break;
        double li[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) li[c] = c < nb ? A[i * ld + j0 + c] : 0.0;
        for (int v = 0; v < 8; ++v) {
          const int l = b0 + tx + 16 * v;
          if (l > i) break;
          double sacc = 0.0;
#pragma unroll
          for (int c = 0; c < NB; ++c)
            if (c < nb) sacc = fma(li[c], A[l * ld + j0 + c], sacc);
          A[i * ld + l] -= sacc;
        }
      }
      __syncthreads();
    }
  } else if (tid < nthr) {
    for (int j = 0; j < d; ++j) {
      const double ajj = A[j * ld + j];
      if (!(ajj > 0.0) || !isfinite(ajj)) {
        if (tid == 0) sh_fail = 1;
        break;  // uniform: every thread read the same value
      }
      const double ipiv = rsqrt(ajj), inv = 1.0 / ajj;
      for (int i = j + tid; i < d; i += nthr) Lo[i * d + j] = (i == j) ? ajj * ipiv : A[i * ld + j] * ipiv;
      const int off = (j + 1) * d - (j + 1) * j / 2;
      // four entries per batch: every load before any store (the entries are
      // distinct and column j is not written), so the dependent smem round
      // trips of the four overlap
      for (int q0 = off + tid; q0 < npair; q0 += 4 * nthr) {
        int ii[4], ll[4];
        double aij[4], alj[4], ail[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + u * nthr;
          ii[u] = q < npair ? ti[q] : 0;
          ll[u] = q < npair ? tl[q] : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          aij[u] = A[ii[u] * ld + j];
          alj[u] = A[ll[u] * ld + j];
          ail[u] = A[ii[u] * ld + ll[u]];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (q0 + u * nthr < npair) A[ii[u] * ld + ll[u]] = ail[u] - aij[u] * alj[u] * inv;
      }
      if (one_warp) __syncwarp(); else __syncthreads();
    }
  }
  __syncthreads();
  if (tid == 0) st->stamp[15] = global_ns();
  if (sh_fail) {  // R-8 fallback: diag(sqrt(Sigma_jj)), 1 where the variance is 0
    for (int e = tid; e < d * d; e += blockDim.x) {
      const int i = e / d, j = e - i * d;
      Lo[e] = (i == j) ? (S1[i] > 0.0 ? sqrt(S1[i]) : 1.0) : 0.0;
    }
    __syncthreads();
  }
  __syncthreads();
  for (int e = tid; e < d * r.dp; e += blockDim.x) {
    const int i = e / r.dp, j = e - i * r.dp;
    r.L[e] = j < d ? static_cast<float>(Lo[i * d + j]) : 0.0f;
    if (j < d) {
      r.LT[j * r.dp + i] = static_cast<float>(Lo[i * d + j]);  // column-major copy
      r.L64[i * d + j] = Lo[i * d + j];
    }
  }
  if (tid == 0) st->stamp[12] = global_ns();
  // slice width (R-7)
  double w;
  if (width_rule == NSS_W_FIXED) {
    w = width_param;
  } else if (r.dir_norm == NSS_DIR_MAHALANOBIS) {
    const double mu = 1.0 / (d + 2.0);
    w = width_param * 4.0 * kKappaInf * sqrt(2.0 / (kPi * mu * d));
  } else {
    // tr(Sigma^-1) = |L^-1|_F^2: one thread per column of L^-1 (forward substitution)
    double part = 0.0;
    for (int c = tid; c < d; c += blockDim.x) {
      double y[kMaxDim];
      for (int i = 0; i < d; ++i) {
        if (i < c) { y[i] = 0.0; continue; }
        double s = (i == c) ? 1.0 : 0.0;
        for (int t = c; t < i; ++t) s -= Lo[i * d + t] * y[t];
        y[i] = s / Lo[i * d + i];
        part += y[i] * y[i];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((tid & 31) == 0) sh_red[tid >> 5] = part;
    __syncthreads();
    double tr = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) tr += sh_red[i];
    const double mu = tr / (static_cast<double>(d) * (d + 2.0));
    w = width_param * 4.0 * kKappaInf * sqrt(2.0 / (kPi * mu * d));
  }
  if (tid == 0) {
    *ticket = 0u;  // re-arm for the next launch
    st->stamp[13] = global_ns();
    st->width = static_cast<float>(w);
    (void)sh_emin;  // termination (A9) is evaluated by the select kernels and k_term_probe
  }
}

// The large-d reduction of k_metric's partials: thread e sums entry e in the
// two-level order of phase 2 (so the sums are identical); entry nent holds the
// minimum energy.  seg_out == null: the whole live set into `sums`; else
// (sharded) the sums of segments seg0 .. seg0 + nseg - 1 into rows of seg_out
// (row stride nent1).
__global__ void __launch_bounds__(128) k_metric_reduce(RunDev r, const double *partials, int bps, int nent1,
                                                       double *sums, int end_of_iter, double *seg_out, int seg0,
                                                       int nseg) {
  const DevState *st = r.st;
  if (st->error || (end_of_iter && st->finalised)) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nent1) return;
  const bool is_min = e == nent1 - 1;
  if (seg_out) {
    for (int s = 0; s < nseg; ++s)
      seg_out[static_cast<long long>(s) * nent1 + e] = fold_segment(partials, seg0 + s, bps, e, nent1, is_min);
    return;
  }
  sums[e] = fold_all(partials, bps, e, nent1, is_min);
}

// Sharded live set: the kSegs segment rows gathered from every rank (rank q's
// rows at seg_rows + q * rank_stride, its first segment q * kSegs / world)
// folded in segment order -- the same sums as k_metric_reduce on one GPU.
__global__ void __launch_bounds__(128) k_metric_segfold(RunDev r, const double *seg_rows, long long rank_stride,
                                                        int nent1, double *sums) {
  if (r.st->error) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nent1) return;
  const bool is_min = e == nent1 - 1;
  const int per = kSegs / r.world;
  double segs[kSegs];
#pragma unroll
  for (int s = 0; s < kSegs; ++s)
    segs[s] = seg_rows[(s / per) * rank_stride + static_cast<long long>(s % per) * nent1 + e];
  sums[e] = fold_segments(segs, 1, 0, is_min);
}

// A9 / R-19 on demand (the host asks for the run's state between
// iterations): minimum live energy, then the same test the next select
// kernel would make.
// With `mirror` (host-mapped pinned memory) it then writes the device state
// and replica 0's log Z there, so reading the state costs the host one
// kernel and one synchronisation, no copies.
__global__ void __launch_bounds__(kThreads) k_term_probe(RunDev r, int probe, DevState *mirror, double *lz0_mirror) {
  DevState *st = r.st;
  if (probe && !(st->error || st->finalised || st->terminated)) {
  __shared__ float red[kThreads / 32];
  float emin = INFINITY;
  for (int g = threadIdx.x; g < r.n; g += blockDim.x) emin = fminf(emin, r.E[g]);
  for (int o = 16; o > 0; o >>= 1) emin = fminf(emin, __shfl_xor_sync(0xffffffffu, emin, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = emin;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) emin = fminf(emin, red[w]);
    emin = fminf(emin, red[0]);
    term_check(r, st, emin);
  }
  }
  if (mirror) {
    __syncthreads();
    const unsigned *src = reinterpret_cast<const unsigned *>(st);
    unsigned *dst = reinterpret_cast<unsigned *>(mirror);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(DevState) / 4); i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) *lz0_mirror = r.lz[0];
    __threadfence_system();
  }
}

// mode 0: both phases; 1: phase 1 only (the large-d partials: sized for
// their rows alone, so two CTAs fit per SM); 2: phase 2 only
size_t metric_smem(int n, int d, int bps, int mode = 0) {
  const int npair = d * (d + 1) / 2, nent = npair + d;
  const int dp = (d + 3) & ~3;
  const int rows = (seg_lo(n, 1) + 1 + bps - 1) / bps;  // a segment has at most floor(n / kSegs) + 1 rows
  const int G = nent < kThreads ? kThreads / nent : 1;  // row groups (raw_groups)
  const size_t p1 = static_cast<size_t>(nent + d) * 8 + ((2 * static_cast<size_t>(npair) + 7) / 8) * 8 +
                    static_cast<size_t>(rows) * dp * 8 + (G > 1 ? static_cast<size_t>(G) * nent * 8 : 0) + 64;
  const size_t p2 = (static_cast<size_t>(d) * (d | 1) + d + (d <= kLoSharedMax ? static_cast<size_t>(d) * d : 0)) * 8 +
                    2 * static_cast<size_t>(npair) + 16;
  return mode == 1 ? p1 : mode == 2 ? p2 : (p1 > p2 ? p1 : p2);
}

}  // namespace

// Blocks per segment (the metric's partials: kSegs * this many rows of
// nent + 1 doubles).
int metric_blocks(int n, int d) {
  const int npair = d * (d + 1) / 2;
  const int dp = (d + 3) & ~3;
  // large d: the grid-wide reduction makes more CTAs cheap, so every SM takes
  // a short chunk of rows; small d: one launch, the last CTA reduces
  int rows_per_block = d >= kSplitMinD ? 64 : (npair > 1000 ? 160 : 128);
  // the CTA's rows stay in shared memory as fp64, beside the entry sums and
  // pair tables, within the 200 KB the kernel is given
  const int nent = npair + d, G = nent < kThreads ? kThreads / nent : 1;
  const long long fixed = 64 + static_cast<long long>(nent + d) * 8 + ((2LL * npair + 7) / 8) * 8 +
                          (G > 1 ? static_cast<long long>(G) * nent * 8 : 0);
  const int rows_max = static_cast<int>((200LL * 1024 - fixed) / (dp * 8)) - 1;
  if (rows_per_block > rows_max) rows_per_block = rows_max;
  const int seg = seg_lo(n, 1) + 1;  // longest segment
  const int b = (seg + rows_per_block - 1) / rows_per_block;
  return b < 1 ? 1 : b;
}

void launch_term_probe(const RunDev &r, const LaunchCtx &lc, int probe, DevState *mirror, double *lz0_mirror) {
  k_term_probe<<<1, kThreads, 0, lc.stream>>>(r, probe, mirror, lz0_mirror);
  ++*lc.launch_counter;
}

void launch_metric(const RunDev &r, double metric_reg, int width_rule, double width_param, int end_of_iteration,
                   double *partials, unsigned *ticket, int bps, const LaunchCtx &lc) {
  NSS_MAX_SMEM(k_metric, 200 * 1024);
  NSS_PIN_CARVEOUT(k_metric);
  const int nblk = kSegs * bps;
  if (r.d < kSplitMinD) {
    k_metric<<<nblk, kThreads, metric_smem(r.n, r.d, bps), lc.stream>>>(r, partials, ticket, bps, metric_reg,
                                                                        width_rule, width_param, end_of_iteration, 0, 0);
    ++*lc.launch_counter;
    return;
  }
  // large d: partials by every CTA, a grid-wide reduction into the row after
  // the partials (nss_init sizes the buffer for nblk + 1 rows), then the
  // factorisation from that one row
  const int nent1 = r.d * (r.d + 1) / 2 + r.d + 1;
  double *sums = partials + static_cast<long long>(nblk) * nent1;
  k_metric<<<nblk, kThreads, metric_smem(r.n, r.d, bps, 1), lc.stream>>>(
      r, partials, ticket, bps, metric_reg, width_rule, width_param, end_of_iteration, 1, 0);
  k_metric_reduce<<<(nent1 + 127) / 128, 128, 0, lc.stream>>>(r, partials, bps, nent1, sums, end_of_iteration,
                                                               nullptr, 0, 0);
  k_metric<<<1, kThreads, metric_smem(r.n, r.d, bps, 2), lc.stream>>>(r, sums, ticket, bps, metric_reg, width_rule,
                                                                      width_param, end_of_iteration, 2, 0);
  *lc.launch_counter += 3;
}

// Sharded live set, before the exchange: this rank's segments' partials
// (blocks of segments [seg0, seg0 + nseg)) reduced to one row per segment in
// seg_out (nseg rows of nent + 1 doubles).
void launch_metric_shard_partials(const RunDev &r, double *partials, int bps, int seg0, int nseg, double *seg_out,
                                  const LaunchCtx &lc) {
  NSS_MAX_SMEM(k_metric, 200 * 1024);
  NSS_PIN_CARVEOUT(k_metric);
  const int nent1 = r.d * (r.d + 1) / 2 + r.d + 1;
  k_metric<<<nseg * bps, kThreads, metric_smem(r.n, r.d, bps, 1), lc.stream>>>(r, partials, nullptr, bps, 0.0, 0,
                                                                              0.0, 1, 1, seg0 * bps);
  k_metric_reduce<<<(nent1 + 127) / 128, 128, 0, lc.stream>>>(r, partials, bps, nent1, nullptr, 1, seg_out, seg0,
                                                               nseg);
  *lc.launch_counter += 2;
}

// After the exchange: every segment's row folded in segment order, then the
// factorisation and width (replicated on every rank).
void launch_metric_shard_final(const RunDev &r, double metric_reg, int width_rule, double width_param,
                               const double *seg_rows, long long rank_stride, double *sums, unsigned *ticket,
                               const LaunchCtx &lc) {
  const int nent1 = r.d * (r.d + 1) / 2 + r.d + 1;
  k_metric_segfold<<<(nent1 + 127) / 128, 128, 0, lc.stream>>>(r, seg_rows, rank_stride, nent1, sums);
  k_metric<<<1, kThreads, metric_smem(r.n, r.d, 1, 2), lc.stream>>>(r, sums, ticket, 1, metric_reg, width_rule,
                                                                    width_param, 1, 2, 0);
  *lc.launch_counter += 2;
}

}  // namespace nss
