// Sharded live set: one NSS run over `world` GPUs, rank q
// owning the gids of segments [q kSegs / world, (q + 1) kSegs / world).
//
// One iteration = [pre] -> all-gather of one fixed-size block per rank ->
// [post].
//   pre  (rank-local): the top min(k, n_q) keys (ord(E) << 32 | gid) of the
//        rank's own points (A2 candidates: any key of the global top k is
//        among its owner's local top k), in ascending gid order with their
//        birth levels, the rank's minimum key (A9) and error code, and the
//        metric's segment sums of the rank's rows (A5, k_metric.cu);
//  post  (replicated on every rank from the same gathered bytes): the
//        segment sums folded in segment order and factorised (k_metric.cu),
//        and k_shard_merge: A9 from the global minimum, A2 the k largest of the
//        gathered candidates, A3 the dead records, A4 the parents; then each
//        rank copies the dead rows it owns, runs the chains whose destination
//        it owns (reading parent rows another rank owns straight from that
//        rank's live set over NVLink, RunDev::peerX) and the evidence.
// Every decision is taken from the same keys and draws as on one GPU, and the
// moment sums follow the same two-level order, so the run is bit-identical to
// the one-GPU run with the same seed for world = 1, 2, 4, 8.
//
// Block layout (bytes, shard_layout): header 16 u64 {error, min key, count,
// ...}; kc_cap candidates {u64 key, u32 birth bits, u32 0}; the rank's
// kSegs / world segment rows of nent + 1 doubles.
#include "select_util.cuh"

namespace nss {

namespace {

constexpr int kHdr = 16;  // u64 words of the block header

struct Cand {
  unsigned long long key;
  uint32_t birth;
  uint32_t pad;
};

__device__ __forceinline__ const Cand *cands_of(const char *block) {
  return reinterpret_cast<const Cand *>(block + kHdr * 8);
}

// pre: this rank's candidates into its block of the gather buffer.  One CTA.
// keys: shared memory when the rank's rows fit, else `gscratch` (n_q keys).
__global__ void __launch_bounds__(kThreads) k_shard_cand(RunDev r, char *block, int kc_cap,
                                                         unsigned long long *gscratch, int keys_in_smem) {
  extern __shared__ unsigned long long sm[];
  __shared__ unsigned hist[256];
  __shared__ int warp_tot[kWarps];
  __shared__ unsigned long long red[2 * kWarps];
  __shared__ unsigned long long sh_prefix;
  __shared__ int sh_kk, sh_done;
  const DevState *st = r.st;
  const int tid = threadIdx.x, lane = tid & 31;
  const int g0 = r.rank_lo[r.rank], g1 = r.rank_lo[r.rank + 1], nq = g1 - g0;
  const int kc = min(r.k, nq);
  unsigned long long *hdr = reinterpret_cast<unsigned long long *>(block);
  Cand *out = reinterpret_cast<Cand *>(block + kHdr * 8);
  unsigned long long *keys = keys_in_smem ? sm : gscratch;
  unsigned long long mn = ~0ull, mx = 0ull;
  for (int i = tid; i < nq; i += blockDim.x) {
    const unsigned long long key = key_of(r.E[g0 + i], g0 + i);
    keys[i] = key;
    mn = key < mn ? key : mn;
    mx = key > mx ? key : mx;
  }
  block_minmax(mn, mx, red);  // barrier: keys visible
  if (tid == 0) {
    hdr[0] = static_cast<unsigned long long>(st->error);
    hdr[1] = mn;
    hdr[2] = static_cast<unsigned long long>(kc);
  }
  (void)kc_cap;
  // the kc-th largest key (all of them when kc = n_q)
  unsigned long long prefix = 0ull, mask = 0ull;
  if (kc < nq) {
    const int hb = 63 - __clzll(mn ^ mx);
    prefix = hb >= 63 ? 0ull : (mn >> (hb + 1)) << (hb + 1);
    mask = hb >= 63 ? 0ull : ~((1ull << (hb + 1)) - 1ull);
    int kk = kc;
    for (int top = hb; top >= 0; top -= 8) {
      const int shift = top >= 7 ? top - 7 : 0;
      const unsigned dmask = (1u << (top - shift + 1)) - 1u;
      for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < nq; i += blockDim.x) {
        const unsigned long long key = keys[i];
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
  }
  // selected <=> (key & mask) >= prefix (mask = 0: everything); compaction in
  // ascending gid order
  const int chunk = (nq + blockDim.x - 1) / blockDim.x;
  const int i0 = min(nq, tid * chunk), i1 = min(nq, i0 + chunk);
  int nsel = 0;
  for (int i = i0; i < i1; ++i) nsel += ((keys[i] & mask) >= prefix) ? 1 : 0;
  int off = block_exclusive_scan(nsel, warp_tot);
  for (int i = i0; i < i1; ++i) {
    const unsigned long long key = keys[i];
    if ((key & mask) >= prefix) {
      Cand cd;
      cd.key = key;
      cd.birth = __float_as_uint(r.birth[g0 + i]);
      cd.pad = 0u;
      out[off++] = cd;
    }
  }
}

// post: A9 + A2-A4 from the gathered candidates (replicated).  One CTA.
// The m gathered candidate keys (shared memory when they fit, else gscratch);
// sel = the k selected keys (gid order) and sorted (descending) in sel_scratch.
__global__ void __launch_bounds__(kThreads) k_shard_merge(RunDev r, const char *gather, long long block_bytes,
                                                          unsigned long long *gscratch, int keys_in_smem,
                                                          int *crange) {
  extern __shared__ unsigned long long sm[];
  __shared__ unsigned hist[256];
  __shared__ int warp_tot[kWarps];
  __shared__ unsigned long long sh_prefix;
  __shared__ int sh_kk, sh_done, sh_flag, sh_off[9];
  __shared__ unsigned long long sh_min;
  DevState *st = r.st;
  const int n = r.n, k = r.k, tid = threadIdx.x, lane = tid & 31, W = r.world;
  double lx0 = 0.0, lz0 = 0.0;
  if (tid == 0) {
    lx0 = r.lx_cur[0];
    lz0 = r.lz[0];
    // an error on any rank stops every rank at the same iteration
    int err = 0;
    unsigned long long mn = ~0ull;
    int off = 0;
    for (int q = 0; q < W; ++q) {
      const unsigned long long *h = reinterpret_cast<const unsigned long long *>(gather + q * block_bytes);
      if (!err && h[0]) err = static_cast<int>(h[0]);
      mn = h[1] < mn ? h[1] : mn;
      sh_off[q] = off;
      off += static_cast<int>(h[2]);
    }
    sh_off[W] = off;
    sh_min = mn;
    if (err) raise_error(st, err);
    sh_flag = (err || st->terminated || st->error || st->finalised) ? 1 : 0;
  }
  __syncthreads();
  if (sh_flag) return;
  const long long nd = st->n_dead;
  const int it = st->iter + 1;
  // A9 before the iteration (R-19), then the capacity rule (R-26)
  if (tid == 0) sh_flag = term_check_v(r, st, energy_of_key(sh_min), lx0, lz0) ? 1 : (nd + k + n > r.max_dead ? 2 : 0);
  __syncthreads();
  if (sh_flag) {
    if (sh_flag == 2 && tid == 0) raise_error(st, NSS_ERR_CAPACITY);
    return;
  }
  const int m = sh_off[W];
  unsigned long long *keys = keys_in_smem ? sm : gscratch;
  unsigned long long mn = ~0ull, mx = 0ull;
  for (int q = 0; q < W; ++q) {
    const Cand *cq = cands_of(gather + q * block_bytes);
    const int cnt = sh_off[q + 1] - sh_off[q];
    for (int i = tid; i < cnt; i += blockDim.x) {
      const unsigned long long key = cq[i].key;
      keys[sh_off[q] + i] = key;
      mn = key < mn ? key : mn;
      mx = key > mx ? key : mx;
    }
  }
  __shared__ unsigned long long red[2 * kWarps];
  block_minmax(mn, mx, red);
  const int hb = 63 - __clzll(mn ^ mx);
  unsigned long long prefix = hb >= 63 ? 0ull : (mn >> (hb + 1)) << (hb + 1);
  unsigned long long mask = hb >= 63 ? 0ull : ~((1ull << (hb + 1)) - 1ull);
  if (k < m) {
    int kk = k;
    for (int top = hb; top >= 0; top -= 8) {
      const int shift = top >= 7 ? top - 7 : 0;
      const unsigned dmask = (1u << (top - shift + 1)) - 1u;
      for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < m; i += blockDim.x) {
        const unsigned long long key = keys[i];
        const bool mm = (key & mask) == prefix;
        const unsigned dig = mm ? static_cast<unsigned>((key >> shift) & dmask) : 0xffffffffu;
        const unsigned peers = __match_any_sync(__activemask(), dig);
        if (mm && lane == __ffs(peers) - 1) atomicAdd(&hist[dig], static_cast<unsigned>(__popc(peers)));
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
  } else {
    prefix = 0ull;
    mask = 0ull;
  }
  // compaction in candidate order = ascending gid: destinations, selected
  // keys and their birth levels
  unsigned long long *sel = r.sel_scratch;  // 2k: k in gid order, then k sorted
  float *sbirth = reinterpret_cast<float *>(r.surv);  // k birth levels in gid order (r.surv is unused here)
  const int chunk = (m + blockDim.x - 1) / blockDim.x;
  const int i0 = min(m, tid * chunk), i1 = min(m, i0 + chunk);
  int nsel = 0;
  for (int i = i0; i < i1; ++i) nsel += ((keys[i] & mask) >= prefix) ? 1 : 0;
  int off = block_exclusive_scan(nsel, warp_tot);
  for (int i = i0; i < i1; ++i) {
    const unsigned long long key = keys[i];
    if ((key & mask) >= prefix) {
      int q = 0;
      while (q + 1 < W && i >= sh_off[q + 1]) ++q;
      const Cand *cq = cands_of(gather + q * block_bytes);
      r.dest_gid[off] = static_cast<int>(key & 0xffffffffu);
      sel[off] = key;
      sbirth[off] = __uint_as_float(cq[i - sh_off[q]].birth);
      ++off;
    }
  }
  __syncthreads();
  // dead order: the k selected keys sorted descending
  unsigned long long *sorted = sel + k;
  unsigned long long *sbuf = keys_in_smem ? sm + m : sm;
  sort_desc(sel, k, sorted, gscratch + (keys_in_smem ? 0 : m), sbuf);
  // parents: the rank-th survivor, rank = floor(u32 (n - k) / 2^32) (P:271-275,
  // R-4); survivors are the gids not in the ascending destination list D, so
  // the j-th one is j + (the first index i with D[i] - i > j)
  for (int c = tid; c < k; c += blockDim.x) {
    const int s = r.dest_gid[c];
    const uint4 b = philox_block(r, it, s, kPhaseResample, 0, 0);
    const int j = static_cast<int>((static_cast<unsigned long long>(b.x) * static_cast<unsigned>(n - k)) >> 32);
    int lo = 0, hi = k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (r.dest_gid[mid] - mid > j) hi = mid; else lo = mid + 1;
    }
    r.parent_gid[c] = j + lo;
  }
  // dead records (R-14 birth, P:1197-1201 n_live = n - j), key-descending
  for (int j = tid; j < k; j += blockDim.x) {
    const unsigned long long key = sorted[j];
    const int g = static_cast<int>(key & 0xffffffffu);
    // birth of g: binary search in the gid-ordered selection
    int lo = 0, hi = k - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (r.dest_gid[mid] < g) lo = mid + 1; else hi = mid;
    }
    const long long q = nd + j;
    r.dE[q] = energy_of_key(key);
    r.dbirth[q] = sbirth[lo];
    r.dnlive[q] = n - j;
    r.dgid[q] = g;
    r.dord[q] = j;
    r.diter[q] = it;
    r.dead_gid[j] = g;
  }
  __syncthreads();
  if (tid == 0) {
    // chains whose destination this rank owns: an ordinal range of D
    const int a = r.rank_lo[r.rank], b = r.rank_lo[r.rank + 1];
    int lo = 0, hi = k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (r.dest_gid[mid] < a) lo = mid + 1; else hi = mid;
    }
    int lo2 = lo, hi2 = k;
    while (lo2 < hi2) {
      const int mid = (lo2 + hi2) >> 1;
      if (r.dest_gid[mid] < b) lo2 = mid + 1; else hi2 = mid;
    }
    crange[0] = lo;
    crange[1] = lo2;
    st->dead_base = nd;
    st->n_dead = nd + k;
    st->e_star = energy_of_key(sorted[k - 1]);
    st->iter = it;  // iteration `it` is under way: HRSS and evidence read it
  }
}

// post: the dead rows this rank owns (the others' stay zero here; nss_dead
// sums the ranks' stores).
__global__ void k_shard_dead_rows(RunDev r) {
  const DevState *st = r.st;
  if (st->terminated || st->error || st->finalised || st->iter == 0) return;
  const long long nd = st->dead_base;
  if (st->n_dead - nd != r.k) return;  // this iteration's select did not run
  const int a = r.rank_lo[r.rank], b = r.rank_lo[r.rank + 1];
  const int dp4 = r.dp >> 2;
  const long long tot = static_cast<long long>(r.k) * dp4;
  const float4 *X4 = reinterpret_cast<const float4 *>(r.X);
  float4 *D4 = reinterpret_cast<float4 *>(r.dX) + nd * dp4;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < tot;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = q / dp4, i = q - j * dp4;
    const int g = r.dgid[nd + j];
    if (g >= a && g < b) D4[q] = X4[static_cast<long long>(g) * dp4 + i];
  }
}

// Finalisation of a sharded run: the dead rows of the records just appended
// (every live point, from the gathered live set) are kept by their owner only,
// like the iterations' dead rows.
__global__ void k_shard_mask_rows(RunDev r) {
  const DevState *st = r.st;
  if (st->error) return;
  const long long nd = st->dead_base, cnt = st->n_dead - nd;
  const int a = r.rank_lo[r.rank], b = r.rank_lo[r.rank + 1];
  const int dp4 = r.dp >> 2;
  float4 *D4 = reinterpret_cast<float4 *>(r.dX) + nd * dp4;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < cnt * dp4;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = r.dgid[nd + q / dp4];
    if (g < a || g >= b) D4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Live-set gather (finalisation, host reads): rank q's rows (x, E, birth) in
// its block of `buf` (rows_cap rows of dp + 2 floats) ...
__global__ void k_shard_pack_live(RunDev r, float *block) {
  const int a = r.rank_lo[r.rank], b = r.rank_lo[r.rank + 1];
  const int row = r.dp + 2;
  const long long tot = static_cast<long long>(b - a) * row;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < tot;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(q / row), c = static_cast<int>(q - static_cast<long long>(i) * row);
    const int g = a + i;
    block[q] = c < r.dp ? r.X[static_cast<long long>(g) * r.dp + c] : (c == r.dp ? r.E[g] : r.birth[g]);
  }
}

// ... and every other rank's rows unpacked into this rank's arrays.
__global__ void k_shard_unpack_live(RunDev r, const float *buf, long long rows_cap) {
  const int row = r.dp + 2;
  for (int q = 0; q < r.world; ++q) {
    if (q == r.rank) continue;
    const int a = r.rank_lo[q], b = r.rank_lo[q + 1];
    const float *blk = buf + q * rows_cap * row;
    const long long tot = static_cast<long long>(b - a) * row;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
      const int i = static_cast<int>(e / row), c = static_cast<int>(e - static_cast<long long>(i) * row);
      const int g = a + i;
      if (c < r.dp)
        r.X[static_cast<long long>(g) * r.dp + c] = blk[e];
      else if (c == r.dp)
        r.E[g] = blk[e];
      else
        r.birth[g] = blk[e];
    }
  }
}

}  // namespace

size_t shard_block_bytes(int k, int own_max, int world, int d) {
  const int nent1 = d * (d + 1) / 2 + d + 1;
  const int kc_cap = k < own_max ? k : own_max;
  const size_t b = static_cast<size_t>(kHdr) * 8 + static_cast<size_t>(kc_cap) * sizeof(Cand) +
                   static_cast<size_t>(kSegs / world) * nent1 * 8;
  return (b + 255) & ~static_cast<size_t>(255);
}

size_t shard_metric_offset(int k, int own_max) {
  const int kc_cap = k < own_max ? k : own_max;
  return static_cast<size_t>(kHdr) * 8 + static_cast<size_t>(kc_cap) * sizeof(Cand);
}

constexpr int kShardSmemKeys = 24576;  // 192 KB of keys on chip

void launch_shard_cand(const RunDev &r, char *block, int kc_cap, const LaunchCtx &lc) {
  const int nq = r.rank_lo[r.rank + 1] - r.rank_lo[r.rank];
  const bool smem = nq <= kShardSmemKeys;
  NSS_MAX_SMEM(k_shard_cand, kShardSmemKeys * 8);
  NSS_PIN_CARVEOUT(k_shard_cand);
  k_shard_cand<<<1, kThreads, smem ? static_cast<size_t>(nq) * 8 : 0, lc.stream>>>(r, block, kc_cap, r.sort_scratch,
                                                                                   smem ? 1 : 0);
  ++*lc.launch_counter;
}

void launch_shard_merge(const RunDev &r, const char *gather, size_t block_bytes, int m_max, int *crange,
                        const LaunchCtx &lc) {
  // keys of the m candidates, plus the sort buffer (k selected keys) behind them
  int P = 1;
  while (P < r.k) P <<= 1;
  const int sortbuf = r.k <= kRankSortMax ? r.k : (P <= kSmemSortMax ? P : kSmemSortMax);
  const bool smem = static_cast<size_t>(m_max + sortbuf) * 8 <= 224 * 1024;
  const size_t bytes = smem ? static_cast<size_t>(m_max + sortbuf) * 8 : static_cast<size_t>(kSmemSortMax) * 8;
  NSS_MAX_SMEM(k_shard_merge, 224 * 1024);
  NSS_PIN_CARVEOUT(k_shard_merge);
  k_shard_merge<<<1, kThreads, bytes, lc.stream>>>(r, gather, static_cast<long long>(block_bytes), r.sort_scratch,
                                                   smem ? 1 : 0, crange);
  ++*lc.launch_counter;
}

void launch_shard_dead_rows(const RunDev &r, const LaunchCtx &lc) {
  const long long tot = static_cast<long long>(r.k) * (r.dp >> 2);
  const long long want = (tot + 255) / 256;
  k_shard_dead_rows<<<static_cast<int>(want < 296 ? (want > 0 ? want : 1) : 296), 256, 0, lc.stream>>>(r);
  ++*lc.launch_counter;
}

void launch_shard_mask_rows(const RunDev &r, const LaunchCtx &lc) {
  k_shard_mask_rows<<<296, 256, 0, lc.stream>>>(r);
  ++*lc.launch_counter;
}

void launch_shard_pack_live(const RunDev &r, float *block, const LaunchCtx &lc) {
  k_shard_pack_live<<<148, 256, 0, lc.stream>>>(r, block);
  ++*lc.launch_counter;
}

void launch_shard_unpack_live(const RunDev &r, const float *buf, long long rows_cap, const LaunchCtx &lc) {
  k_shard_unpack_live<<<296, 256, 0, lc.stream>>>(r, buf, rows_cap);
  ++*lc.launch_counter;
}

}  // namespace nss
