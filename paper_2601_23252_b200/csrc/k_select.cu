// A2 delete + A3 record dead + A4 resample for one outer iteration, and the
// finalisation sort (R-18).  One CTA: at n <= 2e4 the whole key set fits in
// one SM's shared memory and the select is latency-bound, so one SM doing a
// radix select beats a multi-CTA scheme plus a grid barrier.
//
// Keys: key = (ord(E) << 32) | gid -- unique, so "the k largest keys" is the
// set of the k worst energies with ties broken towards the larger gid (R-1).
// The radix passes start at the highest bit where the keys differ (a min/max
// reduction first), so a live set whose energies share exponent and leading
// mantissa bits needs only 2-3 passes of 8 bits.
#include "select_util.cuh"

namespace nss {

namespace {

constexpr int kSmemKeysMax = 12288;   // keys cached in shared memory (96 KB)
constexpr int kSmemOrdMax = 28672;    // 32-bit energy ordinals cached next to the sort buffer (112 KB)

// Writes the dead records (R-14 birth, P:1197-1201 n_live) and copies rows.
__device__ void write_dead(const RunDev &r, const unsigned long long *sorted, int cnt, int n_for_nlive,
                           long long nd, int it, bool rows) {
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    const int g = static_cast<int>(sorted[j] & 0xffffffffu);
    const long long q = nd + j;
    r.dE[q] = r.E[g];
    r.dbirth[q] = r.birth[g];
    r.dnlive[q] = n_for_nlive - j;
    r.dgid[q] = g;
    r.dord[q] = j;
    r.diter[q] = it;
  }
  if (!rows) return;  // copied by the grid-wide k_dead_rows
  // rows: one thread per float, consecutive threads on consecutive columns
  const long long tot = static_cast<long long>(cnt) * r.dp;
  for (long long e = threadIdx.x; e < tot; e += blockDim.x) {
    const int j = static_cast<int>(e / r.dp), i = static_cast<int>(e - static_cast<long long>(j) * r.dp);
    const int g = static_cast<int>(sorted[j] & 0xffffffffu);
    r.dX[(nd + j) * r.dp + i] = r.X[static_cast<long long>(g) * r.dp + i];
  }
}

__global__ void __launch_bounds__(kThreads) k_select(RunDev r, unsigned long long *gscratch,
                                                     unsigned long long *gsel, bool rows) {
  extern __shared__ unsigned long long sm[];
  __shared__ unsigned hist[256];
  __shared__ int warp_tot[kWarps];
  __shared__ unsigned long long red[2 * kWarps];
  __shared__ int sh_flag;
  __shared__ unsigned long long sh_prefix;
  __shared__ int sh_kk, sh_done;
  DevState *st = r.st;
  if (threadIdx.x == 0) sh_flag = (st->terminated || st->error || st->finalised) ? 1 : 0;
  __syncthreads();
  if (sh_flag) return;
  const int n = r.n, k = r.k, tid = threadIdx.x, lane = tid & 31;
  const long long nd = st->n_dead;
  const int it = st->iter + 1;
  // ---- keys: 64-bit in shared memory (n <= kSmemKeysMax), else the 32-bit
  //      energy ordinals in shared memory (the gid is the index), else global
  const bool cached = n <= kSmemKeysMax;
  const bool ord32 = !cached && n <= kSmemOrdMax;
  unsigned long long *keys = cached ? sm : gscratch;
  uint32_t *ords = reinterpret_cast<uint32_t *>(sm + kSmemSortMax);
  unsigned long long *sbuf = cached ? sm + kSmemKeysMax : sm;  // sort buffer next to the key cache
  auto key_at = [&](int g) -> unsigned long long {
    return ord32 ? ((static_cast<unsigned long long>(ords[g]) << 32) | static_cast<unsigned>(g)) : keys[g];
  };
  unsigned long long mn = ~0ull, mx = 0ull;
  for (int g = tid; g < n; g += blockDim.x) {
    const unsigned long long key = key_of(r.E[g], g);
    if (ord32)
      ords[g] = static_cast<uint32_t>(key >> 32);
    else
      keys[g] = key;
    mn = key < mn ? key : mn;
    mx = key > mx ? key : mx;
  }
  block_minmax(mn, mx, red);  // contains a barrier: keys[] is visible
  // A9 before the iteration (R-19), then the capacity rule (R-26)
  if (tid == 0) sh_flag = term_check(r, st, energy_of_key(mn)) ? 1 : (nd + k + n > r.max_dead ? 2 : 0);
  __syncthreads();
  if (sh_flag) {
    if (sh_flag == 2 && tid == 0) raise_error(st, NSS_ERR_CAPACITY);
    return;
  }
  // highest differing bit: all keys agree above it
  const int hb = 63 - __clzll(mn ^ mx);
  const unsigned long long common = hb >= 63 ? 0ull : (mn >> (hb + 1)) << (hb + 1);

  // ---- radix select of the k-th largest key, 8 bits per pass from bit hb down ----
  unsigned long long prefix = common, mask = hb >= 63 ? 0ull : ~((1ull << (hb + 1)) - 1ull);
  int kk = k;
  for (int top = hb; top >= 0; top -= 8) {
    const int shift = top >= 7 ? top - 7 : 0;
    const int width = top - shift + 1;
    const unsigned dmask = (1u << width) - 1u;
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int g = tid; g < n; g += blockDim.x) {
      const unsigned long long key = key_at(g);
      const bool m = (key & mask) == prefix;
      const unsigned dig = m ? static_cast<unsigned>((key >> shift) & dmask) : 0xffffffffu;
      const unsigned peers = __match_any_sync(__activemask(), dig);
      if (m && lane == __ffs(peers) - 1) atomicAdd(&hist[dig], static_cast<unsigned>(__popc(peers)));
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
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += t;
      }
      const unsigned excl = incl - tot;
      if (excl < static_cast<unsigned>(kk) && static_cast<unsigned>(kk) <= incl) {
        unsigned cum = excl;
        int j = 0;
        for (; j < 8; ++j) {
          if (cum + c[j] >= static_cast<unsigned>(kk)) break;
          cum += c[j];
        }
        const unsigned D = 255u - 8u * tid - j;
        sh_kk = kk - static_cast<int>(cum);
        sh_prefix = prefix | (static_cast<unsigned long long>(D) << shift);
        sh_done = (c[j] == static_cast<unsigned>(kk) - cum) ? 1 : 0;
      }
    }
    __syncthreads();
    kk = sh_kk;
    prefix = sh_prefix;
    mask |= static_cast<unsigned long long>(dmask) << shift;
    if (sh_done) break;
  }
  // selected  <=>  (key & mask) >= prefix

  // ---- compaction in ascending gid order: destinations D and survivors S ----
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int g0 = min(n, tid * chunk), g1 = min(n, g0 + chunk);
  int nsel = 0;
  for (int g = g0; g < g1; ++g) nsel += ((key_at(g) & mask) >= prefix) ? 1 : 0;
  int off = block_exclusive_scan(nsel, warp_tot);
  int soff = g0 - off;
  for (int g = g0; g < g1; ++g) {
    const unsigned long long key = key_at(g);
    if ((key & mask) >= prefix) {
      r.dest_gid[off] = g;
      gsel[off] = key;
      ++off;
    } else {
      r.surv[soff++] = g;
    }
  }
  __syncthreads();

  // ---- dead order: the k selected keys sorted descending ----
  unsigned long long *sorted = gsel + k;
  // the key cache / ordinals are dead after the compaction: the sort may use
  // all of the dynamic shared memory (C4: 16 384 keys on chip instead of
  // chunked passes through global memory)
  const int cap = cached ? kSmemKeysMax + kSmemSortMax
                         : ord32 ? kSmemSortMax + (n * 4) / 8 : kSmemSortMax;
  sort_desc(gsel, k, sorted, gscratch + (cached ? 0 : n), sm, cap);
  for (int j = tid; j < k; j += blockDim.x) r.dead_gid[j] = static_cast<int>(sorted[j] & 0xffffffffu);
  const float e_star = r.E[static_cast<int>(sorted[k - 1] & 0xffffffffu)];

  // ---- parents: S[floor(u32 (n-k) / 2^32)] (R-4) ----
  for (int c = tid; c < k; c += blockDim.x) {
    const int s = r.dest_gid[c];
    const uint4 b = philox_block(r, it, s, kPhaseResample, 0, 0);
    const unsigned long long rank = (static_cast<unsigned long long>(b.x) * static_cast<unsigned>(n - k)) >> 32;
    r.parent_gid[c] = r.surv[rank];
  }

  // ---- dead records: n_live = n - j in key-descending order ----
  write_dead(r, sorted, k, n, nd, it, rows);
  __syncthreads();
  if (tid == 0) {
    st->dead_base = nd;
    st->n_dead = nd + k;
    st->e_star = e_star;
    st->iter = it;  // iteration `it` is under way: HRSS and evidence read it
  }
}


// Shared-memory-resident variant (the common case, n <= kSmemKeysMax): keys,
// selected keys, the sorted dead order, survivors and destinations all stay on
// chip, and E* and the dead energies are decoded from the keys, so the only
// global traffic is the energy load, the row gather and the outputs.
__global__ void __launch_bounds__(kThreads) k_select_smem(RunDev r, bool rows) {
  extern __shared__ unsigned long long sm[];
  __shared__ unsigned hist[256];
  __shared__ int warp_tot[kWarps];
  __shared__ unsigned long long red[2 * kWarps];
  __shared__ unsigned long long sh_prefix;
  __shared__ int sh_kk, sh_done;
  DevState *st = r.st;
  const int n = r.n, k = r.k, tid = threadIdx.x, lane = tid & 31;
  unsigned long long *keys = sm;              // n
  unsigned long long *sel = keys + n;         // k (gid order)
  unsigned long long *sorted = sel + k;       // k (descending)
  int *surv = reinterpret_cast<int *>(sorted + k);  // n - k
  int *dest = surv + (n - k);                        // k
  if (tid == 0) st->stamp[0] = global_ns();
  // independent global loads first, flags checked afterwards; thread 0 also
  // fetches the evidence state the termination test needs (cold after a flush)
  double lx0 = 0.0, lz0 = 0.0;
  if (tid == 0) {
    lx0 = r.lx_cur[0];
    lz0 = r.lz[0];
  }
  unsigned long long mn = ~0ull, mx = 0ull;
  for (int g = tid; g < n; g += blockDim.x) {
    const unsigned long long key = key_of(r.E[g], g);
    keys[g] = key;
    mn = key < mn ? key : mn;
    mx = key > mx ? key : mx;
  }
  const int flags = st->terminated | st->error | st->finalised;
  const long long nd = st->n_dead;
  const int it = st->iter + 1;
  if (flags) return;  // uniform: written only by other kernels
  if (tid == 0) st->stamp[1] = global_ns();
  block_minmax(mn, mx, red);
  // A9 before the iteration (R-19), then the capacity rule (R-26)
  if (tid == 0) sh_kk = term_check_v(r, st, energy_of_key(mn), lx0, lz0) ? 1 : (nd + k + n > r.max_dead ? 2 : 0);
  __syncthreads();
  if (sh_kk) {
    if (sh_kk == 2 && tid == 0) raise_error(st, NSS_ERR_CAPACITY);
    return;
  }
  if (tid == 0) st->stamp[2] = global_ns();
  const int hb = 63 - __clzll(mn ^ mx);
  const unsigned long long common = hb >= 63 ? 0ull : (mn >> (hb + 1)) << (hb + 1);
  unsigned long long prefix = common, mask = hb >= 63 ? 0ull : ~((1ull << (hb + 1)) - 1ull);
  int kk = k;
  for (int top = hb; top >= 0; top -= 8) {
    const int shift = top >= 7 ? top - 7 : 0;
    const unsigned dmask = (1u << (top - shift + 1)) - 1u;
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int g = tid; g < n; g += blockDim.x) {
      const unsigned long long key = keys[g];
      const bool m = (key & mask) == prefix;
      const unsigned dig = m ? static_cast<unsigned>((key >> shift) & dmask) : 0xffffffffu;
      const unsigned peers = __match_any_sync(__activemask(), dig);
      if (m && lane == __ffs(peers) - 1) atomicAdd(&hist[dig], static_cast<unsigned>(__popc(peers)));
    }
    __syncthreads();
    if (tid < 32) {
      unsigned c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * tid - j];
        tot += c[j];
      }
      unsigned incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += t;
      }
      const unsigned excl = incl - tot;
      if (excl < static_cast<unsigned>(kk) && static_cast<unsigned>(kk) <= incl) {
        unsigned cum = excl;
        int j = 0;
        for (; j < 8; ++j) {
          if (cum + c[j] >= static_cast<unsigned>(kk)) break;
          cum += c[j];
        }
        sh_kk = kk - static_cast<int>(cum);
        sh_prefix = prefix | (static_cast<unsigned long long>(255u - 8u * tid - j) << shift);
        sh_done = (c[j] == static_cast<unsigned>(kk) - cum) ? 1 : 0;
      }
    }
    __syncthreads();
    kk = sh_kk;
    prefix = sh_prefix;
    mask |= static_cast<unsigned long long>(dmask) << shift;
    if (sh_done) break;
  }
  if (tid == 0) st->stamp[3] = global_ns();
  // compaction in ascending gid order (shared memory only)
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int g0 = min(n, tid * chunk), g1 = min(n, g0 + chunk);
  int nsel = 0;
  for (int g = g0; g < g1; ++g) nsel += ((keys[g] & mask) >= prefix) ? 1 : 0;
  int off = block_exclusive_scan(nsel, warp_tot);
  int soff = g0 - off;
  for (int g = g0; g < g1; ++g) {
    const unsigned long long key = keys[g];
    if ((key & mask) >= prefix) {
      dest[off] = g;
      sel[off++] = key;
    } else {
      surv[soff++] = g;
    }
  }
  __syncthreads();
  if (tid == 0) st->stamp[4] = global_ns();
  // dead order: rank sort (k <= kRankSortMax) or bitonic in place
  if (k <= kRankSortMax) {
    for (int i = tid; i < k; i += blockDim.x) {
      const unsigned long long ki = sel[i];
      int rank = 0;
      for (int j = 0; j < k; ++j) rank += sel[j] > ki;
      sorted[rank] = ki;
    }
    __syncthreads();
  } else {
    int P = 1;
    while (P < k) P <<= 1;
    unsigned long long *buf = keys;  // keys are no longer needed: reuse (n >= P checked on host)
    for (int i = tid; i < P; i += blockDim.x) buf[i] = i < k ? sel[i] : 0ull;
    __syncthreads();
    bitonic_desc(buf, P);
    for (int i = tid; i < k; i += blockDim.x) sorted[i] = buf[i];
    __syncthreads();
  }
  if (tid == 0) st->stamp[5] = global_ns();
  // outputs: destinations, dead order, parents (R-4), dead records
  for (int c = tid; c < k; c += blockDim.x) {
    const int s = dest[c];
    r.dest_gid[c] = s;
    r.dead_gid[c] = static_cast<int>(sorted[c] & 0xffffffffu);
    const uint4 b = philox_block(r, it, s, kPhaseResample, 0, 0);
    const unsigned long long rank = (static_cast<unsigned long long>(b.x) * static_cast<unsigned>(n - k)) >> 32;
    r.parent_gid[c] = surv[rank];
    const unsigned long long key = sorted[c];
    const int g = static_cast<int>(key & 0xffffffffu);
    const long long q = nd + c;
    r.dE[q] = energy_of_key(key);
    r.dbirth[q] = r.birth[g];
    r.dnlive[q] = n - c;
    r.dgid[q] = g;
    r.dord[q] = c;
    r.diter[q] = it;
  }
  if (rows) {
    // dead rows: float4 granules, four loads in flight per thread before the stores
    const int dp4 = r.dp >> 2, tot = k * dp4, T = blockDim.x;
    const float4 *X4 = reinterpret_cast<const float4 *>(r.X);
    float4 *D4 = reinterpret_cast<float4 *>(r.dX) + nd * dp4;
    for (int q0 = tid; q0 < tot; q0 += 4 * T) {
      float4 v[4];
      int dst[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * T;
        dst[u] = q;
        if (q < tot) {
          const int j = q / dp4, i = q - j * dp4;
          v[u] = X4[static_cast<long long>(sorted[j] & 0xffffffffu) * dp4 + i];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (dst[u] < tot) D4[dst[u]] = v[u];
    }
  }
  if (tid == 0) st->stamp[6] = global_ns();
  if (tid == 0) {
    st->dead_base = nd;
    st->n_dead = nd + k;
    st->e_star = energy_of_key(sorted[k - 1]);
    st->iter = it;  // iteration `it` is under way: HRSS and evidence read it
  }
}

size_t select_smem_fused(int n, int k) {
  return static_cast<size_t>(n + 2 * k) * 8 + static_cast<size_t>(n) * 4 + 16;
}

// Finalisation: every live point dies, key-descending, n_live = n..1 (R-18).
__global__ void __launch_bounds__(kThreads) k_finalise_sort(RunDev r, unsigned long long *gscratch,
                                                            unsigned long long *gsel) {
  extern __shared__ unsigned long long sm[];
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
  unsigned long long *buf = (P <= kSmemSortMax) ? sm : gscratch;
  for (int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = (i < n) ? key_of(r.E[i], i) : 0ull;
  __syncthreads();
  if (P <= kSmemSortMax)
    bitonic_desc(buf, P);
  else
    bitonic_desc_chunked(buf, P, sm, kSmemSortMax);
  write_dead(r, buf, n, n, nd, st->iter + 1, true);
  __syncthreads();
  if (threadIdx.x == 0) {
    st->dead_base = nd;
    st->n_dead = nd + n;
  }
  (void)gsel;
}

// Dead rows of the iteration just selected, copied by the whole grid (large
// k * d: one CTA would be bound by its own load latency).
__global__ void k_dead_rows(RunDev r) {
  const DevState *st = r.st;
  if (st->terminated || st->error || st->finalised) return;  // select did not run
  const long long nd = st->dead_base;
  const int dp4 = r.dp >> 2;
  const long long tot = static_cast<long long>(r.k) * dp4;
  const float4 *X4 = reinterpret_cast<const float4 *>(r.X);
  float4 *D4 = reinterpret_cast<float4 *>(r.dX) + nd * dp4;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < tot;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = q / dp4, i = q - j * dp4;
    D4[q] = X4[static_cast<long long>(r.dgid[nd + j]) * dp4 + i];
  }
}

// F4 update-all: chain c = slot c; a deleted slot starts from its
// resampled parent (binary search in the ascending destinations), a survivor
// from itself; all start from a snapshot of the pre-mutation live set.
__global__ void k_chains_all(RunDev r, int *cdest, int *cpar, float *Xs, float *Es) {
  const DevState *st = r.st;
  if (st->terminated || st->error || st->finalised) return;
  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long gg = tid; gg < r.n; gg += stride) {
    const int g = static_cast<int>(gg);
    int lo = 0, hi = r.k;  // first destination >= g
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (r.dest_gid[mid] < g) lo = mid + 1; else hi = mid;
    }
    cdest[g] = g;
    cpar[g] = (lo < r.k && r.dest_gid[lo] == g) ? r.parent_gid[lo] : g;
    Es[g] = r.E[g];
  }
  const long long tot = static_cast<long long>(r.n) * (r.dp >> 2);
  const float4 *X4 = reinterpret_cast<const float4 *>(r.X);
  float4 *S4 = reinterpret_cast<float4 *>(Xs);
  for (long long q = tid; q < tot; q += stride) S4[q] = X4[q];
}

size_t select_smem(int n) {
  if (n <= kSmemKeysMax) return static_cast<size_t>(kSmemKeysMax + kSmemSortMax) * 8;
  if (n <= kSmemOrdMax) return static_cast<size_t>(kSmemSortMax) * 8 + static_cast<size_t>(n) * 4;
  return static_cast<size_t>(kSmemSortMax) * 8;
}

}  // namespace

// scratch layout (device, sized by the host): sort_scratch holds max(n, k)
// rounded up to a power of two plus n; sel_scratch 2k keys.
void launch_select(const RunDev &r, const LaunchCtx &lc) {
  NSS_MAX_SMEM(k_select, kSmemSortMax * 8 + kSmemOrdMax * 4);
  NSS_MAX_SMEM(k_finalise_sort, kSmemSortMax * 8);
  const size_t fused = select_smem_fused(r.n, r.k);
  const bool separate_rows = static_cast<long long>(r.k) * r.dp >= 16384;
  int P = 1;
  while (P < r.k) P <<= 1;
  if (fused <= 200 * 1024 && P <= r.n) {
    NSS_MAX_SMEM(k_select_smem, 200 * 1024);
    NSS_PIN_CARVEOUT(k_select_smem);
    k_select_smem<<<1, kThreads, fused, lc.stream>>>(r, !separate_rows);
  } else {
    NSS_PIN_CARVEOUT(k_select);
    k_select<<<1, kThreads, select_smem(r.n), lc.stream>>>(r, r.sort_scratch, r.sel_scratch, !separate_rows);
  }
  ++*lc.launch_counter;
  if (separate_rows) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long tot = static_cast<long long>(r.k) * (r.dp >> 2);
    const long long want = (tot + 255) / 256;
    k_dead_rows<<<static_cast<int>(want < 2 * sms ? want : 2 * sms), 256, 0, lc.stream>>>(r);
    ++*lc.launch_counter;
  }
}

void launch_chains_all(const RunDev &r, int *cdest, int *cpar, float *Xs, float *Es, const LaunchCtx &lc) {
  const long long work = static_cast<long long>(r.n) * (r.dp >> 2);
  const long long want = ((work > r.n ? work : r.n) + 255) / 256;
  k_chains_all<<<static_cast<int>(want < 1184 ? want : 1184), 256, 0, lc.stream>>>(r, cdest, cpar, Xs, Es);
  ++*lc.launch_counter;
}

void launch_finalise_sort(const RunDev &r, const LaunchCtx &lc) {
  cudaFuncSetAttribute(k_finalise_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSortMax * 8);
  int P = 1;
  while (P < r.n) P <<= 1;
  const size_t smem = static_cast<size_t>(P <= kSmemSortMax ? P : kSmemSortMax) * 8;
  NSS_PIN_CARVEOUT(k_finalise_sort);
  k_finalise_sort<<<1, kThreads, smem, lc.stream>>>(r, r.sort_scratch, r.sel_scratch);
  ++*lc.launch_counter;
}

}  // namespace nss
