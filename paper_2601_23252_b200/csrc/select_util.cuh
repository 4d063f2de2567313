// Block-wide building blocks of the thresholding kernels (k_select.cu, the
// one-GPU select; k_shard.cu, the sharded candidate select and merge):
// 512-thread CTAs, 64-bit keys (ord(E) << 32) | gid (R-1).
#pragma once
#include "nss_internal.cuh"

namespace nss {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kSmemSortMax = 8192;    // selected keys sorted in shared memory (64 KB)
constexpr int kRankSortMax = 1024;    // rank sort (k^2/T compares) up to this k

// Descending bitonic sort of P (power of two) keys at `buf` (shared or global).
__device__ void bitonic_desc(unsigned long long *buf, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const unsigned long long a = buf[lo], b = buf[hi];
        if (desc ? (a < b) : (a > b)) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Block-wide exclusive scan of one int per thread.
__device__ int block_exclusive_scan(int v, int *warp_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  int off = 0;
  for (int w = 0; w < wid; ++w) off += warp_tot[w];
  __syncthreads();
  return off + incl - v;
}

__device__ void block_minmax(unsigned long long &mn, unsigned long long &mx, unsigned long long *red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if (lane == 0) {
    red[wid] = mn;
    red[kWarps + wid] = mx;
  }
  __syncthreads();
  mn = red[0];
  mx = red[kWarps];
  for (int w = 1; w < kWarps; ++w) {
    mn = red[w] < mn ? red[w] : mn;
    mx = red[kWarps + w] > mx ? red[kWarps + w] : mx;
  }
  __syncthreads();
}

// Bitonic stages of one chunk of C keys (staged in shared memory at sbuf)
// whose first element has global index `base`: sizes size_lo..size_hi with
// strides below C, directions taken from the global index (the network of
// bitonic_desc over the whole array).
__device__ void bitonic_chunk(unsigned long long *sbuf, int C, int base, int size_first, int size_last,
                              int stride_first) {
  for (int size = size_first; size <= size_last; size <<= 1) {
    for (int stride = (size == size_first ? stride_first : size >> 1); stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (C >> 1); i += blockDim.x) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool desc = ((base + lo) & size) == 0;
        const unsigned long long a = sbuf[lo], b = sbuf[hi];
        if (desc ? (a < b) : (a > b)) {
          sbuf[lo] = b;
          sbuf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Descending bitonic sort of P (power of two) > C keys in global memory:
// every stage with stride < C runs chunk by chunk in shared memory, only the
// strides >= C stream through global memory (log2(P/C) (log2(P/C)+1)/2
// passes instead of log2(P)(log2(P)+1)/2).
__device__ void bitonic_desc_chunked(unsigned long long *g, int P, unsigned long long *sbuf, int C) {
  auto chunk_pass = [&](int size_first, int size_last, int stride_first) {
    for (int base = 0; base < P; base += C) {
      for (int i = threadIdx.x; i < C; i += blockDim.x) sbuf[i] = g[base + i];
      __syncthreads();
      bitonic_chunk(sbuf, C, base, size_first, size_last, stride_first);
      for (int i = threadIdx.x; i < C; i += blockDim.x) g[base + i] = sbuf[i];
      __syncthreads();
    }
  };
  chunk_pass(2, C, 1);  // sizes 2..C entirely on chip
  for (int size = 2 * C; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride >= C; stride >>= 1) {
      for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const unsigned long long a = g[lo], b = g[hi];
        if (desc ? (a < b) : (a > b)) {
          g[lo] = b;
          g[hi] = a;
        }
      }
      __syncthreads();
    }
    chunk_pass(size, size, C >> 1);  // the remaining strides C/2..1 of this size
  }
}

// Sort `cnt` distinct keys descending into out[] (shared or global).
// sbuf holds `cap` keys (at least kSmemSortMax): sorts of up to cap keys
// stay in shared memory, larger ones go through gscratch in chunks
__device__ void sort_desc(const unsigned long long *in, int cnt, unsigned long long *out,
                          unsigned long long *gscratch, unsigned long long *sbuf, int cap = kSmemSortMax) {
  if (cnt <= kRankSortMax) {
    // rank sort: position = number of larger keys (keys are unique); the keys
    // are staged in shared memory and read as broadcasts
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) sbuf[i] = in[i];
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const unsigned long long ki = sbuf[i];
      int rank = 0;
      for (int j = 0; j < cnt; ++j) rank += sbuf[j] > ki;
      out[rank] = ki;
    }
    __syncthreads();
    return;
  }
  int P = 1;
  while (P < cnt) P <<= 1;
  unsigned long long *buf = (P <= cap) ? sbuf : gscratch;
  for (int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = (i < cnt) ? in[i] : 0ull;
  __syncthreads();
  if (P <= cap)
    bitonic_desc(buf, P);
  else
    bitonic_desc_chunked(buf, P, sbuf, kSmemSortMax);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[i] = buf[i];
  __syncthreads();
}

__device__ __forceinline__ float energy_of_key(unsigned long long key) {  // inverse of ord_f32
  const uint32_t u = static_cast<uint32_t>(key >> 32);
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

}  // namespace
}  // namespace nss
