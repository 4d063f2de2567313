// A8 evidence: R+1 volume replicas (replica 0 deterministic, P:143/R-15;
// replicas 1..R simulate t ~ Beta(n_live, 1)), trapezoid
// or rectangle quadrature, log-sum-exp accumulation
// in fp64.
//
// One CTA per replica.  The deaths of the iteration are processed in tiles of
// kThreads: a block-wide inclusive scan of the log-shrinkages gives log X for
// the whole tile at once, each thread then forms the quadrature term of its
// point's predecessor from shared memory, and one block log-sum-exp folds the
// tile into the replica's accumulator.  Serial depth per iteration is one tile
// (k <= 256) instead of k sequential deaths.  The pending trapezoid point is
// recovered from the dead store (record dead_base-1), so no cross-block state
// is needed.  The kernel runs on a side stream, concurrently with HRSS.
#include "nss_internal.cuh"

namespace nss {

namespace {

constexpr int kThreads = 256;
constexpr double kLn2 = 0.69314718055994530942;

__device__ __forceinline__ double log1mexp(double a) {  // log(1 - e^a), a < 0
  return a > -kLn2 ? log(-expm1(a)) : log1p(-exp(a));
}

__device__ __forceinline__ void lse_acc(double &m, double &s, double t) {
  if (t == -INFINITY) return;
  if (t > m) {
    s = s * exp(m - t) + 1.0;
    m = t;
  } else {
    s += exp(t - m);
  }
}

__device__ __forceinline__ void lse_merge(double &m, double &s, double m2, double s2) {
  const double mm = fmax(m, m2);
  if (mm == -INFINITY) return;
  s = s * exp(m - mm) + s2 * exp(m2 - mm);
  m = mm;
}

__global__ void __launch_bounds__(kThreads) k_evidence(RunDev r, int finalise) {
  DevState *st = r.st;
  // flags are only written by other kernels, so every thread sees the same values
  if (st->error) return;
  if (!finalise && (st->terminated || st->finalised)) return;
  if (finalise && st->finalised) return;
  const int rep = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ double s_lx[kThreads];
  __shared__ double s_e[kThreads];
  __shared__ double s_wtot[kThreads / 32];
  __shared__ double s_m[kThreads / 32], s_s[kThreads / 32];

  const long long base = st->dead_base;
  const int count = static_cast<int>(st->n_dead - base);
  bool has_p = base > 0;
  double pe = has_p ? static_cast<double>(r.dE[base - 1]) : 0.0;
  double lxp = r.lx_prev[rep], lxc = r.lx_cur[rep];
  const bool trap = r.quadrature == NSS_Q_TRAPEZOID;
  double m = -INFINITY, s = 0.0;

  for (int t0 = 0; t0 < count; t0 += kThreads) {
    const int j = t0 + tid;
    const bool valid = j < count;
    double e = 0.0, delta = 0.0;
    if (valid) {
      const long long q = base + j;
      e = static_cast<double>(r.dE[q]);
      const double nl = static_cast<double>(r.dnlive[q]);
      if (rep == 0) {
        delta = -1.0 / nl;
      } else {
        const uint4 b = philox_block(r, static_cast<uint32_t>(r.diter[q]), static_cast<uint32_t>(r.dord[q]),
                                     kPhaseVolume, static_cast<uint32_t>(rep), 0);
        delta = log(static_cast<double>(u01(b.x))) / nl;
      }
    }
    // block inclusive scan of the log-shrinkages -> log X_j
    double sc = delta;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += t;
    }
    if (lane == 31) s_wtot[wid] = sc;
    __syncthreads();
    double off = 0.0;
    for (int w2 = 0; w2 < wid; ++w2) off += s_wtot[w2];
    const double lx = lxc + off + sc;
    s_lx[tid] = lx;
    s_e[tid] = e;
    __syncthreads();
    double term = -INFINITY;
    if (valid) {
      // neighbours of point j inside the tile, or the carried values
      const double lx_m1 = tid >= 1 ? s_lx[tid - 1] : lxc;
      const double lx_m2 = tid >= 2 ? s_lx[tid - 2] : (tid == 1 ? lxc : lxp);
      const double e_m1 = tid >= 1 ? s_e[tid - 1] : pe;
      if (trap) {
        // term of the previous point i = j-1: dX_i = (X_{i-1} - X_{i+1}) / 2
        if (j >= 1 || has_p) term = -e_m1 + lx_m2 + log1mexp(lx - lx_m2) - kLn2;
      } else {
        term = -e + lx_m1 + log1mexp(lx - lx_m1);
      }
    }
    // tile log-sum-exp: block max, then one exp per lane and a plain sum
    double mx = term;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_m[wid] = mx;
    __syncthreads();
    double M = s_m[0];
#pragma unroll
    for (int w2 = 1; w2 < kThreads / 32; ++w2) M = fmax(M, s_m[w2]);
    double ex = (term == -INFINITY) ? 0.0 : exp(term - M);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ex += __shfl_xor_sync(0xffffffffu, ex, o);
    if (lane == 0) s_s[wid] = ex;
    __syncthreads();
    if (M != -INFINITY) {
      double S = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < kThreads / 32; ++w2) S += s_s[w2];
      lse_merge(m, s, M, S);  // uniform across the block
    }
    const int last = min(kThreads, count - t0) - 1;
    const double nlxp = last >= 1 ? s_lx[last - 1] : lxc;
    lxc = s_lx[last];
    lxp = nlxp;
    pe = s_e[last];
    has_p = true;
    __syncthreads();
  }
  if (tid == 0) {
    double lz = r.lz[rep];
    if (m != -INFINITY) {
      const double t = m + log(s);
      const double hi = fmax(lz, t);
      lz = hi + log(exp(lz - hi) + exp(t - hi));
    }
    if (finalise && trap && has_p) {
      // close the sequence with X_{N+1} = 0: dX_N = X_{N-1} / 2 (R-18)
      const double t = -pe + lxp - kLn2;
      const double hi = fmax(lz, t);
      lz = hi + log(exp(lz - hi) + exp(t - hi));
    }
    r.lz[rep] = lz;
    r.lx_prev[rep] = lxp;
    r.lx_cur[rep] = lxc;
  }
}

}  // namespace

void launch_evidence(const RunDev &r, int finalise, const LaunchCtx &lc) {
  NSS_PIN_CARVEOUT(k_evidence);
  k_evidence<<<r.R + 1, kThreads, 0, lc.stream>>>(r, finalise);
  ++*lc.launch_counter;
}

}  // namespace nss
