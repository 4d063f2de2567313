// A5 metric: live-set covariance (1/(n-1)) + ridge reg*mean(diag) (P:326-332,
// R-8), Cholesky in fp64, fallback to the diagonal, and the slice width rule
// (R-7).  At the end of an iteration the same finishing kernel
// evaluates the termination criterion (A9, R-19) and advances the iteration
// counter.
//
// Two kernels: k_cov_partial (B CTAs over fixed gid chunks, shifted fp64 sums,
// no atomics) and k_cov_final (one CTA: fixed-order sum of the B partials, then
// Cholesky).  The reduction order is fixed, so the metric is bit-reproducible.
#include "nss_internal.cuh"

namespace nss {

namespace {

constexpr int kPartialThreads = 256;
constexpr int kTileRows = 32;
constexpr double kKappaInf = 1.3035;
constexpr double kPi = 3.14159265358979323846;

__global__ void __launch_bounds__(kPartialThreads) k_cov_partial(RunDev r, double *partials, int end_of_iter) {
  DevState *st = r.st;
  if (st->error) return;
  if (end_of_iter && (st->terminated || st->finalised)) return;
  extern __shared__ double sm[];
  const int d = r.d, n = r.n;
  const int npair = d * (d + 1) / 2;
  const int nent = npair + d;
  double *S = sm;                                             // nent accumulators
  double *tile = S + nent;                                    // kTileRows * d centred rows
  double *shift = tile + kTileRows * d;
  unsigned char *pi = reinterpret_cast<unsigned char *>(shift + d);
  unsigned char *pj = pi + npair;
  __shared__ float red_min[kPartialThreads / 32];

  for (int e = threadIdx.x; e < nent; e += blockDim.x) S[e] = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) shift[i] = static_cast<double>(r.X[i]);  // row 0
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    int base = i * (i + 1) / 2;
    for (int j = 0; j <= i; ++j) {
      pi[base + j] = static_cast<unsigned char>(i);
      pj[base + j] = static_cast<unsigned char>(j);
    }
  }
  const int chunk = (n + gridDim.x - 1) / gridDim.x;
  const int g0 = min(n, static_cast<int>(blockIdx.x) * chunk), g1 = min(n, g0 + chunk);
  float emin = INFINITY;
  for (int g = g0 + threadIdx.x; g < g1; g += blockDim.x) emin = fminf(emin, r.E[g]);
  __syncthreads();
  for (int t0 = g0; t0 < g1; t0 += kTileRows) {
    const int rows = min(kTileRows, g1 - t0);
    for (int e = threadIdx.x; e < rows * d; e += blockDim.x) {
      int rr = e / d, i = e - rr * d;
      tile[e] = static_cast<double>(r.X[static_cast<long long>(t0 + rr) * r.dp + i]) - shift[i];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nent; e += blockDim.x) {
      double acc = 0.0;
      if (e < npair) {
        const int i = pi[e], j = pj[e];
        for (int rr = 0; rr < rows; ++rr)
          acc += tile[rr * d + i] * tile[rr * d + j];
      } else {
        const int i = e - npair;
        for (int rr = 0; rr < rows; ++rr) acc += tile[rr * d + i];
      }
      S[e] += acc;
    }
    __syncthreads();
  }
  double *out = partials + static_cast<long long>(blockIdx.x) * (nent + 1);
  for (int e = threadIdx.x; e < nent; e += blockDim.x) out[e] = S[e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) emin = fminf(emin, __shfl_xor_sync(0xffffffffu, emin, o));
  if ((threadIdx.x & 31) == 0) red_min[threadIdx.x >> 5] = emin;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red_min[0];
    for (int w = 1; w < kPartialThreads / 32; ++w) m = fminf(m, red_min[w]);
    out[nent] = static_cast<double>(m);
  }
}

__global__ void __launch_bounds__(1024) k_cov_final(RunDev r, const double *partials, int nblk, double reg,
                                                    int width_rule, double width_param, int end_of_iter) {
  DevState *st = r.st;
  __shared__ int sh_flag;
  if (threadIdx.x == 0) sh_flag = (st->error || (end_of_iter && (st->terminated || st->finalised))) ? 1 : 0;
  __syncthreads();
  if (sh_flag) return;
  extern __shared__ double A[];  // d*d fp64 (symmetric fill, then Cholesky in the lower part)
  const int d = r.d, n = r.n, tid = threadIdx.x;
  const int npair = d * (d + 1) / 2, nent = npair + d;
  double *S1 = A + d * d;        // d
  __shared__ double sh_md;
  __shared__ int sh_fail;
  __shared__ double sh_red[32];
  // fixed-order sum over the partial blocks
  for (int e = tid; e < nent; e += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += partials[static_cast<long long>(b) * (nent + 1) + e];
    if (e < npair) {
      int i = 0;
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      int j = e - i * (i + 1) / 2;
      A[i * d + j] = acc;   // S2_ij (shifted)
    } else {
      S1[e - npair] = acc;  // S1_i  (shifted)
    }
  }
  __syncthreads();
  const double nn = static_cast<double>(n);
  for (int e = tid; e < d * d; e += blockDim.x) {
    int i = e / d, j = e - i * d;
    if (j <= i) A[e] = (A[e] - S1[i] * S1[j] / nn) / (nn - 1.0);
  }
  __syncthreads();
  for (int e = tid; e < d * d; e += blockDim.x) {
    int i = e / d, j = e - i * d;
    if (j > i) A[e] = A[j * d + i];
  }
  if (tid == 0) {
    double md = 0.0;
    for (int i = 0; i < d; ++i) md += A[i * d + i];
    sh_md = md / d;
    sh_fail = 0;
  }
  __syncthreads();
  for (int i = tid; i < d; i += blockDim.x) {
    A[i * d + i] += reg * sh_md;
    S1[i] = A[i * d + i];  // keep the regularised diagonal for the fallback
  }
  __syncthreads();
  // right-looking Cholesky, lower triangle in place
  for (int j = 0; j < d; ++j) {
    if (tid == 0) {
      double v = A[j * d + j];
      if (!(v > 0.0) || !isfinite(v)) sh_fail = 1;
      A[j * d + j] = sqrt(fmax(v, 0.0));
    }
    __syncthreads();
    if (sh_fail) break;
    const double piv = A[j * d + j];
    for (int i = j + 1 + tid; i < d; i += blockDim.x) A[i * d + j] /= piv;
    __syncthreads();
    const int m = d - j - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l <= i) A[i * d + l] -= A[i * d + j] * A[l * d + j];
    }
    __syncthreads();
  }
  if (sh_fail) {  // R-8 fallback: diag(sqrt(Sigma_jj)), 1 where the variance is 0
    for (int e = tid; e < d * d; e += blockDim.x) {
      int i = e / d, j = e - i * d;
      A[e] = (i == j) ? (S1[i] > 0.0 ? sqrt(S1[i]) : 1.0) : 0.0;
    }
    __syncthreads();
  }
  for (int e = tid; e < d * d; e += blockDim.x) {
    int i = e / d, j = e - i * d;
    double v = (j <= i) ? A[e] : 0.0;
    r.L64[e] = v;
  }
  for (int e = tid; e < d * r.dp; e += blockDim.x) {
    int i = e / r.dp, j = e - i * r.dp;
    r.L[e] = (j < d && j <= i) ? static_cast<float>(A[i * d + j]) : 0.0f;
  }
  // slice width (R-7)
  double w;
  if (width_rule == NSS_W_FIXED) {
    w = width_param;
  } else if (r.dir_norm == NSS_DIR_MAHALANOBIS) {
    double mu = 1.0 / (d + 2.0);
    w = width_param * 4.0 * kKappaInf * sqrt(2.0 / (kPi * mu * d));
  } else {
    // tr(Sigma^-1) = |L^-1|_F^2: one thread per column of L^-1 (forward substitution)
    __syncthreads();
    double part = 0.0;
    for (int c = tid; c < d; c += blockDim.x) {
      // solve L y = e_c, only entries i >= c are non-zero
      // y_i = (delta_ic - sum_{t<i} L_it y_t) / L_ii ; keep y in registers via a small loop
      // (d <= 128: store y in local memory)
      double y[kMaxDim];
      for (int i = 0; i < d; ++i) {
        if (i < c) { y[i] = 0.0; continue; }
        double s = (i == c) ? 1.0 : 0.0;
        for (int t = c; t < i; ++t) s -= A[i * d + t] * y[t];
        y[i] = s / A[i * d + i];
        part += y[i] * y[i];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((tid & 31) == 0) sh_red[tid >> 5] = part;
    __syncthreads();
    double tr = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tr += sh_red[i];
    double mu = tr / (static_cast<double>(d) * (d + 2.0));
    w = width_param * 4.0 * kKappaInf * sqrt(2.0 / (kPi * mu * d));
  }
  if (tid == 0) {
    st->width = static_cast<float>(w);
    if (end_of_iter) {
      float emin = INFINITY;
      for (int b = 0; b < nblk; ++b) emin = fminf(emin, static_cast<float>(partials[static_cast<long long>(b) * (nent + 1) + nent]));
      st->emin = emin;
      // A9 / R-19: stop when the live bound is below e^{term} of the total
      double lz_live = -static_cast<double>(emin) + r.lx_cur[0];
      double lz0 = r.lz[0];
      double mm = fmax(lz0, lz_live);
      double tot = (mm == -INFINITY) ? -INFINITY : mm + log(exp(lz0 - mm) + exp(lz_live - mm));
      st->log_z_live = lz_live;
      if (st->n_dead > 0 && (lz_live - tot) < static_cast<double>(r.term_log_ratio)) st->terminated = 1;
      st->iter += 1;
    }
  }
}

}  // namespace

int metric_blocks(int n, int d) {
  int npair = d * (d + 1) / 2;
  // enough rows per block to amortise the per-block partial write
  int rows_per_block = npair > 1000 ? 160 : 128;
  int b = (n + rows_per_block - 1) / rows_per_block;
  return b < 1 ? 1 : (b > 148 ? 148 : b);
}

static size_t partial_smem(int d) {
  int npair = d * (d + 1) / 2, nent = npair + d;
  size_t s = static_cast<size_t>(nent + kTileRows * d + d) * 8 + 2 * static_cast<size_t>(npair) + 16;
  return s;
}

void launch_metric(const RunDev &r, double metric_reg, int width_rule, double width_param, int end_of_iteration,
                   double *partials, int n_blocks, const LaunchCtx &lc) {
  size_t s1 = partial_smem(r.d);
  size_t s2 = static_cast<size_t>(r.d) * r.d * 8 + static_cast<size_t>(r.d) * 8 * 2 + 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_cov_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_cov_final, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_cov_partial<<<n_blocks, kPartialThreads, s1, lc.stream>>>(r, partials, end_of_iteration);
  k_cov_final<<<1, 1024, s2, lc.stream>>>(r, partials, n_blocks, metric_reg, width_rule, width_param,
                                          end_of_iteration);
  *lc.launch_counter += 2;
}

}  // namespace nss
