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
  const float *prec;  // CORR: d rows of stride ldp
  int ldp;
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
    for (int e = tid; e < d * d; e += nt) {
      int i = e / d, j = e - i * d;
      P[i * es.ldp + j] = en.prec[e];
    }
    es.mu = sp; es.prec = P;
  }
}

__device__ __forceinline__ float softplusf(float a) {
  return a > 0.f ? a + log1pf(expf(-a)) : log1pf(expf(a));
}

// Per-lane prior parameters for the coordinates a lane owns.
template <int NPL>
__device__ __forceinline__ void load_prior_lane(const PriorDev &pr, int lane, int d, float (&pa)[NPL],
                                                float (&pb)[NPL]) {
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    if (pr.kind == NSS_PRIOR_BOX) {
      pa[t] = i < d ? pr.lo[i] : 0.f;
      pb[t] = i < d ? pr.hi[i] : 0.f;
    } else {
      pa[t] = i < d ? pr.mean[i] : 0.f;
      pb[t] = i < d ? pr.isd[i] : 0.f;
    }
  }
}

}  // namespace nss
