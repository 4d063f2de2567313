// A8 evidence: R+1 volume replicas (replica 0 deterministic, P:143/R-15;
// replicas 1..R simulate t ~ Beta(n_live, 1)), trapezoid
// or rectangle quadrature, log-sum-exp accumulation
// in fp64.  One warp per replica; the deaths of the iteration are processed 32
// at a time with a warp inclusive scan of the log-shrinkages, so the serial
// depth is k/32 instead of k.  The pending trapezoid point is recovered from the
// dead store (record dead_base-1), so no cross-block state is needed.
#include "nss_internal.cuh"

namespace nss {

namespace {

constexpr int kWarpsPerBlock = 4;
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

__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_evidence(RunDev r, int finalise) {
  DevState *st = r.st;
  const int lane = threadIdx.x & 31;
  const int rep = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  // flags are only written by other kernels, so every thread sees the same values
  if (st->error) return;
  if (!finalise && (st->terminated || st->finalised)) return;
  if (finalise && st->finalised) return;
  if (rep > r.R) return;

  const long long base = st->dead_base;
  const int count = static_cast<int>(st->n_dead - base);
  bool has_p = base > 0;
  double pe = has_p ? static_cast<double>(r.dE[base - 1]) : 0.0;
  double lxp = r.lx_prev[rep], lxc = r.lx_cur[rep];
  const bool trap = r.quadrature == NSS_Q_TRAPEZOID;
  double m = -INFINITY, s = 0.0;

  for (int c0 = 0; c0 < count; c0 += 32) {
    const int j = c0 + lane;
    const bool valid = j < count;
    double e = 0.0, delta = 0.0;
    if (valid) {
      const long long q = base + j;
      e = static_cast<double>(r.dE[q]);
      const double nl = static_cast<double>(r.dnlive[q]);
      if (rep == 0) {
        delta = -1.0 / nl;
      } else {
        uint4 b = philox_block(r, static_cast<uint32_t>(r.diter[q]), static_cast<uint32_t>(r.dord[q]),
                               kPhaseVolume, static_cast<uint32_t>(rep), 0);
        delta = log(static_cast<double>(u01(b.x))) / nl;
      }
    }
    // inclusive scan of the log-shrinkages -> log X_j
    double sc = delta;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double t = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += t;
    }
    const double lx = lxc + sc;
    double lx_m1 = __shfl_up_sync(0xffffffffu, lx, 1);
    double lx_m2 = __shfl_up_sync(0xffffffffu, lx, 2);
    double e_m1 = __shfl_up_sync(0xffffffffu, e, 1);
    if (lane == 0) {
      lx_m1 = lxc;
      lx_m2 = lxp;
      e_m1 = pe;
    } else if (lane == 1) {
      lx_m2 = lxc;
    }
    if (valid) {
      if (trap) {
        // term of the previous point i = j-1: dX_i = (X_{i-1} - X_{i+1}) / 2
        if (j >= 1 || has_p) lse_acc(m, s, -e_m1 + lx_m2 + log1mexp(lx - lx_m2) - kLn2);
      } else {
        lse_acc(m, s, -e + lx_m1 + log1mexp(lx - lx_m1));
      }
    }
    const int last = min(31, count - c0 - 1);
    const double nlxp = (last >= 1) ? __shfl_sync(0xffffffffu, lx, last - 1) : lxc;
    lxc = __shfl_sync(0xffffffffu, lx, last);
    lxp = nlxp;
    pe = __shfl_sync(0xffffffffu, e, last);
    has_p = true;
  }
  // combine the lanes' partial log-sum-exps
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double m2 = __shfl_xor_sync(0xffffffffu, m, o);
    double s2 = __shfl_xor_sync(0xffffffffu, s, o);
    double mm = fmax(m, m2);
    if (mm == -INFINITY) continue;
    s = s * exp(m - mm) + s2 * exp(m2 - mm);
    m = mm;
  }
  if (lane == 0) {
    double lz = r.lz[rep];
    if (m != -INFINITY) {
      double t = m + log(s);
      double mm = fmax(lz, t);
      lz = mm + log(exp(lz - mm) + exp(t - mm));
    }
    if (finalise && trap && has_p) {
      // close the sequence with X_{N+1} = 0: dX_N = X_{N-1} / 2 (R-18)
      double t = -pe + lxp - kLn2;
      double mm = fmax(lz, t);
      lz = mm + log(exp(lz - mm) + exp(t - mm));
    }
    r.lz[rep] = lz;
    r.lx_prev[rep] = lxp;
    r.lx_cur[rep] = lxc;
  }
}

}  // namespace

void launch_evidence(const RunDev &r, int finalise, const LaunchCtx &lc) {
  int blocks = (r.R + 1 + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_evidence<<<blocks, kWarpsPerBlock * 32, 0, lc.stream>>>(r, finalise);
  ++*lc.launch_counter;
}

}  // namespace nss
