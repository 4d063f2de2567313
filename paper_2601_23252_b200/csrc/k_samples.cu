// Evidence summary (R-17, R-27) and posterior weights of the dead points
// (geometric mean over the R volume replicas).
//
// Weights re-simulate every replica's volume trajectory from the dead store
// with the same counter-based draws as the streamed accumulators (DESIGN
// section 3), in point chunks: k_traj (one warp per replica, warp-scan of the
// log-shrinkages) writes log X for the chunk, k_wacc (one thread per point)
// sums log dX over the replicas in a fixed order, then one CTA normalises.
#include "nss_internal.cuh"

namespace nss {

namespace {

constexpr double kLn2 = 0.69314718055994530942;

__global__ void k_fill(double *p, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__device__ __forceinline__ double log1mexp(double a) {
  return a > -kLn2 ? log(-expm1(a)) : log1p(-exp(a));
}
__device__ __forceinline__ double lse2(double a, double b) {
  double m = fmax(a, b);
  if (m == -INFINITY) return -INFINITY;
  return m + log(exp(a - m) + exp(b - m));
}

// out[0] = mean, out[1] = std (ddof 1) of closed log Z^(r), r = 1..R; out[2+r] = closed log Z^(r)
__global__ void k_evidence_summary(RunDev r, double *out) {
  DevState *st = r.st;
  const bool close = !st->finalised && r.quadrature == NSS_Q_TRAPEZOID && st->n_dead > 0;
  const double pe = st->n_dead > 0 ? static_cast<double>(r.dE[st->n_dead - 1]) : 0.0;
  for (int rep = threadIdx.x; rep <= r.R; rep += blockDim.x) {
    double lz = r.lz[rep];
    if (close) lz = lse2(lz, -pe + r.lx_prev[rep] - kLn2);  // X_{N+1} = 0 (R-27)
    out[2 + rep] = lz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int rep = 1; rep <= r.R; ++rep) s += out[2 + rep];
    const double mean = s / r.R;
    double v = 0.0;
    for (int rep = 1; rep <= r.R; ++rep) v += (out[2 + rep] - mean) * (out[2 + rep] - mean);
    out[0] = mean;
    out[1] = sqrt(v / (r.R - 1));
  }
}

// log X_{i0+t}^(rep) for t = 0..cnt (point cnt only if it exists); replicas 1..R
__global__ void k_traj(RunDev r, long long N, long long i0, int cnt, const double *carry_in, double *carry_out,
                       double *lxbuf, int ld) {
  const int lane = threadIdx.x & 31;
  const int rep = 1 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rep > r.R) return;
  double lx0 = carry_in[rep - 1];
  const int total = static_cast<int>(((long long)(cnt + 1) < N - i0 ? (long long)(cnt + 1) : N - i0));
  for (int c0 = 0; c0 < total; c0 += 32) {
    const int t = c0 + lane;
    double delta = 0.0;
    if (t < total) {
      const long long i = i0 + t;
      uint4 b = philox_block(r, static_cast<uint32_t>(r.diter[i]), static_cast<uint32_t>(r.dord[i]), kPhaseVolume,
                             static_cast<uint32_t>(rep), 0);
      delta = log(static_cast<double>(u01(b.x))) / static_cast<double>(r.dnlive[i]);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double u = __shfl_up_sync(0xffffffffu, delta, o);
      if (lane >= o) delta += u;
    }
    const double lx = lx0 + delta;
    if (t < total) lxbuf[static_cast<long long>(rep - 1) * ld + t] = lx;
    const int last = min(31, total - c0 - 1);
    lx0 = __shfl_sync(0xffffffffu, lx, last);
  }
  __syncwarp();
  if (lane == 0 && cnt >= 1) carry_out[rep - 1] = lxbuf[static_cast<long long>(rep - 1) * ld + (cnt - 1)];
}

__device__ __forceinline__ double log_dx(const RunDev &r, long long N, long long i, int t, const double *row,
                                         double prev) {
  if (r.quadrature != NSS_Q_TRAPEZOID) return prev + log1mexp(row[t] - prev);    // X_{i-1} - X_i
  if (i + 1 < N) return prev + log1mexp(row[t + 1] - prev) - kLn2;             // (X_{i-1} - X_{i+1}) / 2
  return prev - kLn2;                                                            // X_{N+1} = 0
}

// Tempered evidence of every replica (F2): running
// log-sum-exp over the chunk's points of -beta E_i + log dX_i^(r), one warp
// per replica, merged into (zmax, zsum)[rep].
__global__ void k_zacc(RunDev r, long long N, long long i0, int cnt, const double *carry_in, const double *lxbuf,
                       int ld, double beta, double *zmax, double *zsum) {
  const int lane = threadIdx.x & 31;
  const int rep = 1 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rep > r.R) return;
  const double *row = lxbuf + static_cast<long long>(rep - 1) * ld;
  double m = -INFINITY, sum = 0.0;
  for (int t = lane; t < cnt; t += 32) {
    const double prev = (t >= 1) ? row[t - 1] : carry_in[rep - 1];
    const double term = -beta * static_cast<double>(r.dE[i0 + t]) + log_dx(r, N, i0 + t, t, row, prev);
    if (term > m) {
      sum = sum * exp(m - term) + 1.0;
      m = term;
    } else {
      sum += exp(term - m);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
    const double mm = fmax(m, m2);
    sum = (mm == -INFINITY) ? 0.0 : sum * exp(m - mm) + s2 * exp(m2 - mm);
    m = mm;
  }
  if (lane == 0) {
    const double M = fmax(zmax[rep - 1], m);
    if (M > -INFINITY) zsum[rep - 1] = zsum[rep - 1] * exp(zmax[rep - 1] - M) + sum * exp(m - M);
    zmax[rep - 1] = M;
  }
}

// out[0] mean, out[1] std (ddof 1) of log Z^(r)(beta), r = 1..R
__global__ void k_zsummary(int R, const double *zmax, const double *zsum, double *out) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int r = 0; r < R; ++r) s += zmax[r] + log(zsum[r]);
  const double mean = s / R;
  double v = 0.0;
  for (int r = 0; r < R; ++r) {
    const double q = zmax[r] + log(zsum[r]) - mean;
    v += q * q;
  }
  out[0] = mean;
  out[1] = sqrt(v / (R - 1));
}

__global__ void k_wacc(RunDev r, long long N, long long i0, int cnt, const double *carry_in, const double *lxbuf,
                       int ld, double *logw, double beta) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const long long i = i0 + t;
  double acc = 0.0;
  for (int rep = 1; rep <= r.R; ++rep) {
    const double *row = lxbuf + static_cast<long long>(rep - 1) * ld;
    const double prev = (t >= 1) ? row[t - 1] : carry_in[rep - 1];  // log X_{i-1}
    acc += log_dx(r, N, i, t, row, prev);
  }
  logw[i] = acc / r.R - beta * static_cast<double>(r.dE[i]);
}

__global__ void __launch_bounds__(1024) k_normalise(long long N, double *logw) {
  __shared__ double sm[32], ss[32];
  __shared__ double lse;
  double m = -INFINITY;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) m = fmax(m, logw[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = sm[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mm = fmax(mm, sm[w]);
    sm[0] = mm;
  }
  __syncthreads();
  const double M = sm[0];
  double s = 0.0;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) s += exp(logw[i] - M);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ss[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += ss[w];
    lse = M + log(tot);
  }
  __syncthreads();
  for (long long i = threadIdx.x; i < N; i += blockDim.x) logw[i] -= lse;
}

// Kish ESS of normalised log weights: 1 / sum_i w_i^2
__global__ void __launch_bounds__(1024) k_ess(long long N, const double *logw, double *out) {
  __shared__ double ss[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) s += exp(2.0 * logw[i]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ss[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += ss[w];
    out[0] = 1.0 / tot;
  }
}

// cum[i] = sum_{l <= i} exp(logw[l]) (one CTA, 1024-point tiles, block scan)
__global__ void __launch_bounds__(1024) k_cumsum(long long N, const double *logw, double *cum) {
  __shared__ double wt[32];
  __shared__ double carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0.0;
  __syncthreads();
  for (long long base = 0; base < N; base += blockDim.x) {
    const long long i = base + threadIdx.x;
    double v = i < N ? exp(logw[i]) : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) wt[wid] = v;
    __syncthreads();
    double off = carry;
    for (int w = 0; w < wid; ++w) off += wt[w];
    if (i < N) cum[i] = off + v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = off + v;
    __syncthreads();
  }
}

// equal-weight draws (F2): u_j = uniform 0 of (iteration 0, j, POSTERIOR, 0)
// under key `seed`; index = first i with u_j < cum[i]
__global__ void k_draw(RunDev r, long long N, const double *cum, long long m, uint64_t seed, long long *idx,
                       double *x) {
  const long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (j >= m) return;
  const uint4 b = philox(make_uint4(0u, static_cast<uint32_t>(kPhasePosterior) << 24, static_cast<uint32_t>(j), 0u),
                         static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const double u = static_cast<double>(u01(b.x));
  long long lo = 0, hi = N - 1;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (u < cum[mid]) hi = mid; else lo = mid + 1;
  }
  idx[j] = lo;
  for (int q = 0; q < r.d; ++q) x[j * r.d + q] = static_cast<double>(r.dX[lo * r.dp + q]);
}

}  // namespace

void launch_evidence_summary(const RunDev &r, double *out, const LaunchCtx &lc) {
  NSS_PIN_CARVEOUT(k_evidence_summary);
  k_evidence_summary<<<1, 128, 0, lc.stream>>>(r, out);
  ++*lc.launch_counter;
}

// scratch: carry (2 * R doubles) + lxbuf (R * (chunk + 1) doubles)
void launch_samples(const RunDev &r, long long N, double *logw, double *scratch, int chunk, const LaunchCtx &lc,
                    double beta, double *zacc) {
  double *carry[2] = {scratch, scratch + r.R};
  double *lxbuf = scratch + 2 * r.R;
  const int ld = chunk + 1;
  cudaMemsetAsync(carry[0], 0, r.R * sizeof(double), lc.stream);  // log X_0 = 0
  if (zacc) {  // zmax = -inf, zsum = 0
    cudaMemsetAsync(zacc + r.R, 0, r.R * sizeof(double), lc.stream);
    k_fill<<<(r.R + 255) / 256, 256, 0, lc.stream>>>(zacc, r.R, -INFINITY);
    ++*lc.launch_counter;
  }
  int cur = 0;
  for (long long i0 = 0; i0 < N; i0 += chunk) {
    const int cnt = static_cast<int>(((long long)chunk < N - i0 ? (long long)chunk : N - i0));
    const int wpb = 4;
    k_traj<<<(r.R + wpb - 1) / wpb, wpb * 32, 0, lc.stream>>>(r, N, i0, cnt, carry[cur], carry[cur ^ 1], lxbuf, ld);
    k_wacc<<<(cnt + 255) / 256, 256, 0, lc.stream>>>(r, N, i0, cnt, carry[cur], lxbuf, ld, logw, beta);
    *lc.launch_counter += 2;
    if (zacc) {
      k_zacc<<<(r.R + wpb - 1) / wpb, wpb * 32, 0, lc.stream>>>(r, N, i0, cnt, carry[cur], lxbuf, ld, beta, zacc,
                                                               zacc + r.R);
      ++*lc.launch_counter;
    }
    cur ^= 1;
  }
  k_normalise<<<1, 1024, 0, lc.stream>>>(N, logw);
  ++*lc.launch_counter;
  if (zacc) {
    k_zsummary<<<1, 32, 0, lc.stream>>>(r.R, zacc, zacc + r.R, zacc + 2 * r.R);
    k_ess<<<1, 1024, 0, lc.stream>>>(N, logw, zacc + 2 * r.R + 2);
    *lc.launch_counter += 2;
  }
}

void launch_resample(const RunDev &r, long long N, const double *logw, double *cum, long long m, uint64_t seed,
                     long long *idx, double *x, const LaunchCtx &lc) {
  k_cumsum<<<1, 1024, 0, lc.stream>>>(N, logw, cum);
  k_draw<<<static_cast<int>((m + 255) / 256), 256, 0, lc.stream>>>(r, N, cum, m, seed, idx, x);
  *lc.launch_counter += 2;
}

}  // namespace nss
