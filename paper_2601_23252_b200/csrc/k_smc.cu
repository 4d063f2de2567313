// F3: adaptive tempered SMC with the HRSS kernel (SMC-SS; P:635-681,
// P:710-713).  One stage = k_smc_beta (next temperature by bisection on the
// ESS of exp(-db E), log Z += log mean w, cumulative normalised weights) ->
// k_smc_snapshot -> k_smc_resample (multinomial gather) -> metric (k_metric)
// -> tempered HRSS (k_hrss with RunDev::tempered, chains = particles).
#include "nss_internal.cuh"

namespace nss {

namespace {

constexpr int kThreads = 1024;

__device__ double block_sum(double v, double *red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

// ESS of exp(-db (E_i - emin))
__device__ double ess_of(const RunDev &r, double db, double emin, double *red) {
  double s = 0.0, s2 = 0.0;
  for (int i = threadIdx.x; i < r.n; i += kThreads) {
    const double w = exp(-db * (static_cast<double>(r.E[i]) - emin));
    s += w;
    s2 += w * w;
  }
  s = block_sum(s, red);
  s2 = block_sum(s2, red);
  return s * s / s2;
}

__global__ void __launch_bounds__(kThreads) k_smc_beta(RunDev r, double rho, double *cum) {
  __shared__ double red[kThreads / 32];
  __shared__ double sh_carry;
  DevState *st = r.st;
  if (st->error || st->terminated) return;
  const double bt = st->smc_beta;
  if (bt >= 1.0) {
    if (threadIdx.x == 0) st->terminated = 1;
    return;
  }
  double emin = INFINITY;
  for (int i = threadIdx.x; i < r.n; i += kThreads) emin = fmin(emin, static_cast<double>(r.E[i]));
  for (int o = 16; o > 0; o >>= 1) emin = fmin(emin, __shfl_xor_sync(0xffffffffu, emin, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = emin;
  __syncthreads();
  emin = red[0];
  for (int w = 1; w < kThreads / 32; ++w) emin = fmin(emin, red[w]);
  // next temperature: bisection to 1e-10 in db, or the whole step
  const double target = rho * r.n;
  double hi = 1.0 - bt, db;
  if (ess_of(r, hi, emin, red) >= target) {
    db = hi;
  } else {
    double lo = 0.0;
    while (hi - lo > 1e-10) {
      const double mid = 0.5 * (lo + hi);
      if (ess_of(r, mid, emin, red) >= target) lo = mid; else hi = mid;
    }
    db = lo;
  }
  const double bn = (db == 1.0 - bt) ? 1.0 : bt + db;
  db = bn - bt;  // the step actually taken (as the oracle: beta_next - beta_t)
  // log Z += log mean w; cumulative normalised weights
  double s = 0.0;
  for (int i = threadIdx.x; i < r.n; i += kThreads) s += exp(-db * (static_cast<double>(r.E[i]) - emin));
  s = block_sum(s, red);
  if (threadIdx.x == 0) sh_carry = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < r.n; base += kThreads) {
    const int i = base + threadIdx.x;
    double v = i < r.n ? exp(-db * (static_cast<double>(r.E[i]) - emin)) / s : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) red[wid] = v;
    __syncthreads();
    double off = sh_carry;
    for (int w = 0; w < wid; ++w) off += red[w];
    if (i < r.n) cum[i] = off + v;
    __syncthreads();
    if (threadIdx.x == kThreads - 1) sh_carry = off + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->smc_logz += -db * emin + log(s) - log(static_cast<double>(r.n));
    st->smc_beta = bn;
    st->iter += 1;  // stage t: the resampling and HRSS draws use it
  }
}

__global__ void k_smc_snapshot(RunDev r, float *Xs, float *Es) {
  const DevState *st = r.st;
  if (st->error || st->terminated) return;
  const long long tot = static_cast<long long>(r.n) * r.dp;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < tot;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    Xs[q] = r.X[q];
    if (q < r.n) Es[q] = r.E[q];
  }
}

// multinomial resampling: u_j = uniform 0 of stream (t, j, SMC, 0); parent =
// first i with u_j < cum[i]; particle j <- snapshot row parent
__global__ void k_smc_resample(RunDev r, const double *cum, int *parents, const float *Xs, const float *Es) {
  const DevState *st = r.st;
  if (st->error || st->terminated) return;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= r.n) return;
  const uint4 b = philox_block(r, static_cast<uint32_t>(st->iter), static_cast<uint32_t>(j), kPhaseSmc, 0, 0);
  const double u = static_cast<double>(u01(b.x));
  int lo = 0, hi = r.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (u < cum[mid]) hi = mid; else lo = mid + 1;
  }
  for (int i = lane; i < r.dp; i += 32) r.X[static_cast<long long>(j) * r.dp + i] = Xs[static_cast<long long>(lo) * r.dp + i];
  if (lane == 0) {
    r.E[j] = Es[lo];
    parents[j] = lo;
  }
}

}  // namespace

void launch_smc_stage(const RunDev &r, double rho, double *cum, int *parents, float *Xsnap, float *Esnap,
                      const LaunchCtx &lc) {
  k_smc_beta<<<1, kThreads, 0, lc.stream>>>(r, rho, cum);
  k_smc_snapshot<<<296, 256, 0, lc.stream>>>(r, Xsnap, Esnap);
  k_smc_resample<<<(r.n + 7) / 8, 256, 0, lc.stream>>>(r, cum, parents, Xsnap, Esnap);
  *lc.launch_counter += 3;
}

}  // namespace nss
