// A2 delete + A3 record dead + A4 resample for one outer iteration, and the
// finalisation sort (R-18).  One CTA of 1024 threads: at n <= 2e4 the keys fit
// in L1/L2 and the select is latency-bound, so one SM doing a radix select is
// cheaper than a multi-CTA scheme plus a grid barrier.
//
// Keys: key = (ord(E) << 32) | gid -- unique, so "the k largest keys" is the
// set of the k worst energies with ties broken towards the larger gid (R-1).
#include "nss_internal.cuh"

namespace nss {

namespace {

constexpr int kThreads = 1024;
constexpr int kSmemSortMax = 16384;  // keys sorted in shared memory (128 KB)

// Descending bitonic sort of P (power of two) keys at `buf` (shared or global).
__device__ void bitonic_desc(unsigned long long *buf, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
        int lo = 2 * stride * (i / stride) + (i % stride);
        int hi = lo + stride;
        bool desc = (lo & size) == 0;
        unsigned long long a = buf[lo], b = buf[hi];
        if (desc ? (a < b) : (a > b)) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Block-wide exclusive scan of one int per thread (blockDim.x == 1024).
__device__ int block_exclusive_scan(int v, int *warp_tot, int *total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int t = warp_tot[lane];
    int s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    warp_tot[lane] = s - t;  // exclusive warp offsets
    if (lane == 31) *total = s;
  }
  __syncthreads();
  return warp_tot[wid] + incl - v;
}

// Writes the dead records (R-14 birth, P:1197-1201 n_live) and copies rows.
__device__ void write_dead(const RunDev &r, const unsigned long long *sorted, int cnt, int n_for_nlive,
                           long long nd, int it) {
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    int g = static_cast<int>(sorted[j] & 0xffffffffu);
    long long q = nd + j;
    r.dE[q] = r.E[g];
    r.dbirth[q] = r.birth[g];
    r.dnlive[q] = n_for_nlive - j;
    r.dgid[q] = g;
    r.dord[q] = j;
    r.diter[q] = it;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < cnt; j += nw) {
    int g = static_cast<int>(sorted[j] & 0xffffffffu);
    const float *src = r.X + static_cast<long long>(g) * r.dp;
    float *dst = r.dX + (nd + j) * r.dp;
    for (int i = lane; i < r.dp; i += 32) dst[i] = src[i];
  }
}

__global__ void __launch_bounds__(kThreads) k_select(RunDev r, unsigned long long *gscratch) {
  extern __shared__ unsigned long long sbuf[];
  __shared__ unsigned hist[256];
  __shared__ int warp_tot[32];
  __shared__ int sh_total, sh_flag;
  __shared__ unsigned long long sh_prefix;
  __shared__ int sh_kk, sh_done;
  DevState *st = r.st;
  if (threadIdx.x == 0) sh_flag = (st->terminated || st->error || st->finalised) ? 1 : 0;
  __syncthreads();
  if (sh_flag) return;
  const int n = r.n, k = r.k, tid = threadIdx.x;
  const long long nd = st->n_dead;
  const int it = st->iter + 1;
  if (nd + k + n > r.max_dead) {  // R-26
    if (tid == 0) raise_error(st, NSS_ERR_CAPACITY);
    return;
  }

  // ---- radix select of the k-th largest key, 8 bits per pass, MSB first ----
  unsigned long long prefix = 0, mask = 0;
  int kk = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int g = tid; g < n; g += blockDim.x) {
      unsigned long long key = key_of(r.E[g], g);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins 255-8l .. 248-8l (descending)
      unsigned c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * tid - j];
        tot += c[j];
      }
      unsigned incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += t;
      }
      unsigned excl = incl - tot;
      bool mine = excl < static_cast<unsigned>(kk) && static_cast<unsigned>(kk) <= incl;
      if (mine) {
        unsigned cum = excl;
        int j = 0;
        for (; j < 8; ++j) {
          if (cum + c[j] >= static_cast<unsigned>(kk)) break;
          cum += c[j];
        }
        unsigned D = 255u - 8u * tid - j;
        sh_kk = kk - static_cast<int>(cum);
        sh_prefix = prefix | (static_cast<unsigned long long>(D) << shift);
        sh_done = (c[j] == static_cast<unsigned>(kk) - cum) ? 1 : 0;
      }
    }
    __syncthreads();
    kk = sh_kk;
    prefix = sh_prefix;
    mask |= 0xFFull << shift;
    if (sh_done) break;
    __syncthreads();
  }
  // selected  <=>  (key & mask) >= prefix

  // ---- compaction in ascending gid order: destinations D and survivors S ----
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int g0 = min(n, tid * chunk), g1 = min(n, g0 + chunk);
  int nsel = 0;
  for (int g = g0; g < g1; ++g) nsel += ((key_of(r.E[g], g) & mask) >= prefix) ? 1 : 0;
  int off = block_exclusive_scan(nsel, warp_tot, &sh_total);
  int soff = g0 - off;
  for (int g = g0; g < g1; ++g) {
    if ((key_of(r.E[g], g) & mask) >= prefix) r.dest_gid[off++] = g;
    else r.surv[soff++] = g;
  }
  __syncthreads();

  // ---- dead order: the k selected keys sorted descending ----
  int P = 1;
  while (P < k) P <<= 1;
  unsigned long long *buf = (P <= kSmemSortMax) ? sbuf : gscratch;
  for (int i = tid; i < P; i += blockDim.x)
    buf[i] = (i < k) ? key_of(r.E[r.dest_gid[i]], r.dest_gid[i]) : 0ull;
  __syncthreads();
  bitonic_desc(buf, P);
  for (int j = tid; j < k; j += blockDim.x) r.dead_gid[j] = static_cast<int>(buf[j] & 0xffffffffu);
  const float e_star = r.E[static_cast<int>(buf[k - 1] & 0xffffffffu)];

  // ---- parents: S[floor(u32 (n-k) / 2^32)] (R-4) ----
  for (int c = tid; c < k; c += blockDim.x) {
    int s = r.dest_gid[c];
    uint4 b = philox_block(r, it, s, kPhaseResample, 0, 0);
    unsigned long long rank = (static_cast<unsigned long long>(b.x) * static_cast<unsigned>(n - k)) >> 32;
    r.parent_gid[c] = r.surv[rank];
  }

  // ---- dead records: n_live = n - j in key-descending order ----
  write_dead(r, buf, k, n, nd, it);
  __syncthreads();
  if (tid == 0) {
    st->dead_base = nd;
    st->n_dead = nd + k;
    st->e_star = e_star;
  }
}

// Finalisation: every live point dies, key-descending, n_live = n..1 (R-18).
__global__ void __launch_bounds__(kThreads) k_finalise_sort(RunDev r, unsigned long long *gscratch) {
  extern __shared__ unsigned long long sbuf[];
  DevState *st = r.st;
  __shared__ int sh_flag;
  if (threadIdx.x == 0) sh_flag = (st->error || st->finalised) ? 1 : 0;
  __syncthreads();
  if (sh_flag) return;
  const int n = r.n;
  const long long nd = st->n_dead;
  if (nd + n > r.max_dead) {
    if (threadIdx.x == 0) raise_error(st, NSS_ERR_CAPACITY);
    return;
  }
  int P = 1;
  while (P < n) P <<= 1;
  unsigned long long *buf = (P <= kSmemSortMax) ? sbuf : gscratch;
  for (int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = (i < n) ? key_of(r.E[i], i) : 0ull;
  __syncthreads();
  bitonic_desc(buf, P);
  write_dead(r, buf, n, n, nd, st->iter + 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    st->dead_base = nd;
    st->n_dead = nd + n;
  }
}

size_t sort_smem(int cnt) {
  int P = 1;
  while (P < cnt) P <<= 1;
  return P <= kSmemSortMax ? static_cast<size_t>(P) * 8 : 0;
}

}  // namespace

void launch_select(const RunDev &r, const LaunchCtx &lc) {
  size_t smem = sort_smem(r.k);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSortMax * 8);
    cudaFuncSetAttribute(k_finalise_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSortMax * 8);
    attr = true;
  }
  k_select<<<1, kThreads, smem, lc.stream>>>(r, r.sort_scratch);
  ++*lc.launch_counter;
}

void launch_finalise_sort(const RunDev &r, const LaunchCtx &lc) {
  size_t smem = sort_smem(r.n);
  cudaFuncSetAttribute(k_finalise_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSortMax * 8);
  k_finalise_sort<<<1, kThreads, smem, lc.stream>>>(r, r.sort_scratch);
  ++*lc.launch_counter;
}

}  // namespace nss
