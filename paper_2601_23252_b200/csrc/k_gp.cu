// A1 for GP hyperparameter marginalisation (P:935-962 shape, R-22): batched
// negative log marginal likelihood of an ARD-RBF Gaussian process in fp64,
//
//   K = sf^2 exp(-1/2 sum_j ((x_aj - x_bj) / l_j)^2) + (sn^2 + jitter) I
//   E = 1/2 y^T K^-1 y + 1/2 log|K| + N/2 log 2 pi,
//   phi = (log l_1..l_D, log sf, log sn).
//
// One CTA per probe matrix (probes are dealt to a persistent grid of one CTA
// per SM).  The CTA builds the (N+1) x N lower trapezoid [K; y^T] in its own
// fp64 scratch slot and runs a right-looking blocked Cholesky with 64-wide
// panels: the diagonal block is factorised in shared memory by one warp, the
// panel below it is solved row by row (the extra row y^T becomes alpha =
// L^-1 y on the way), and the trailing lower trapezoid receives the rank-64
// update in 64 x 64 tiles: panel rows staged row-major in shared memory and
// contracted on the fp64 tensor cores (mma.sync m8n8k4 DMMA, 8 per warp per
// k-step).  E then needs only
// the pivots (log det) and |alpha|^2.  A non-positive pivot gives E = +inf (K
// not positive definite), as in the oracle.  fp64 throughout: the paper runs
// its GP experiments in double precision.
#include "batch.cuh"
#include "energy.cuh"

namespace nss {

namespace {

constexpr int kThreads = 256;
constexpr int PB = 64;        // block edge: column blocks of L and the output tiles
constexpr int LDR = PB + 4;   // stride of the 64 x 64 shared tiles: 68 = 4 mod 16 -> conflict-free DMMA fragments
constexpr int KC = 32;        // k-chunk width of the stored L tiles
constexpr int LDC = KC + 4;   // stride of a stored / staged chunk tile (36 = 4 mod 16)
constexpr int CT = PB * LDC;  // doubles per chunk tile (18 KB)
constexpr double kLn2Pi = 1.8378770664093454836;

struct GpDev {
  int N, D;
  const double *X;  // N x D inputs
  const double *y;  // N targets
  double jitter;
  double *scratch;  // per CTA slot: nrb x nkc chunk tiles of L
  double *e64;      // optional fp64 copy of the energies (nss_gp_energy_batch)
  int nrb, nkc;     // row blocks of [L; alpha^T] (N + 1 rows), 32-wide chunks per row block
};

__device__ __forceinline__ double block_sum(double v, double *red) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

// the first `rows` rows of a stored chunk tile (contiguous, already in the
// padded shared layout) -> shared memory with 16-B asynchronous copies; the
// caller commits and waits
__device__ __forceinline__ void load_chunk(double *dst, const double *src, int rows) {
  const int ng = rows * (LDC / 2);
  for (int e = threadIdx.x; e < ng; e += kThreads) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + 2 * e));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 2 * e) : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// D(8x8) += A(8x4) B(4x8) on the fp64 tensor cores: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d = D[lane/4][2 (lane%4) + {0, 1}]
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// acc(32 x 16 per warp) += Ta(rows) . Tb(rows)^T over k < KB (KB = 0: kb at
// run time): 4 x 2 DMMA 8x8 tiles, operand rows at m_base / n_base of
// row-major tiles of stride LD; only the first mcnt 8-row groups of the warp
// (warp-uniform) are computed
template <int LD, int KB>
__device__ __forceinline__ void mma_rows(const double *Ta, const double *Tb, int kb, int m_base, int n_base, int gq,
                                         int tq, int mcnt, double (&acc)[4][2][2]) {
  const double *pa = Ta + (m_base + gq) * LD + tq;
  const double *pb = Tb + (n_base + gq) * LD + tq;
  const int kend = KB ? KB : kb;
  if (mcnt >= 4) {
#pragma unroll 4
    for (int c = 0; c < kend; c += 4) {
      double av[4], bv[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) av[mi] = pa[8 * mi * LD + c];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bv[ni] = pb[8 * ni * LD + c];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
    }
  } else if (mcnt > 0) {
    for (int c = 0; c < kend; c += 4) {
      double bv[2];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bv[ni] = pb[8 * ni * LD + c];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
        if (mi < mcnt) {
          const double a = pa[8 * mi * LD + c];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a, bv[ni]);
        }
    }
  }
}

// Left-looking blocked Cholesky of the (N+1) x N lower trapezoid [K; y^T]
// (its last row becomes alpha^T = (L^-1 y)^T).  For each 64-wide column
// block j and each row block i >= j, the 64 x 64 tile
//   T = [K; y^T](i, j) - L(i, :j) L(j, :j)^T
// is accumulated in registers on the DMMA tensor cores from the stored L
// chunk tiles (double-buffered cp.async stream, each output tile read and
// written exactly once), K(i, j) is generated on the fly from X (never
// stored), then the diagonal tile is factorised in shared memory (one barrier
// per column) with its inverse W = L_jj^-1, and each tile below it becomes
// L(i, j) = T W^T (DMMA), stored as two 64 x 32 chunk tiles.
__global__ void __launch_bounds__(kThreads, 2) k_gp_energy(GpDev g, BatchDev b, int parity, int dp) {
  extern __shared__ double sm[];
  const int N = g.N, D = g.D, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (blockIdx.x == 0 && tid == 0) b.n_probe[parity ^ 1] = 0;  // the next round's row counter
  const int n = b.n_probe[parity];
  if (static_cast<int>(blockIdx.x) >= n) return;
  double *Ci = sm;            // 2 x CT: chunks of row block i (stage buffers); T aliases them
  double *Cj = Ci + 2 * CT;   // 2 x CT: chunks of row block j
  double *W = Cj + 2 * CT;    // PB x LDR: L_jj^-1 (lower), zero above the diagonal and past kb
  double *diag = W + PB * LDR;  // PB: L_cc
  double *red = diag + PB;      // 8
  double *T = Ci;               // PB x LDR (4352 <= 2 CT doubles)
  __shared__ double sh_par[NSS_MAX_DIM + 2];
  __shared__ int sh_fail;
  const long long slot = static_cast<long long>(g.nrb) * g.nkc * CT;
  double *Ls = g.scratch + static_cast<long long>(blockIdx.x) * slot;
  const int nkc = g.nkc, nrb = g.nrb, ncb = (N + PB - 1) / PB;
  const int ty = tid >> 4, tx = tid & 15;  // diagonal-block owner map
  // DMMA warp tiles: warp (wr, wc) owns rows 32 wr .. +32, columns 16 wc .. +16
  const int m_base = (wid >> 2) * 32, n_base = (wid & 3) * 16, gq = lane >> 2, tq = lane & 3;

  for (int p = blockIdx.x; p < n; p += gridDim.x) {
    if (tid < D + 2) {
      const double ph = static_cast<double>(b.P[parity][static_cast<long long>(p) * dp + tid]);
      sh_par[tid] = tid < D ? exp(-ph) : exp(2.0 * ph);  // 1/l_j, sf^2, sn^2
    }
    if (tid == 0) sh_fail = 0;
    __syncthreads();
    const double sf2 = sh_par[D], diag_add = sh_par[D + 1] + g.jitter;
    double logdet_part = 0.0;  // lane-held sums of log pivots (warp 0)
    double alpha2 = 0.0;       // thread-held sums of alpha_c^2
    for (int j = 0; j < ncb && !sh_fail; ++j) {
      const int j0 = j * PB, kb = min(PB, N - j0), nch = 2 * j;
      const int kr = (kb + 3) & ~3;  // DMMA k range of the W product (W and T zero past kb)
      for (int i = j; i < nrb; ++i) {
        const int i0 = i * PB, rows = min(PB, N + 1 - i0);
        const bool dt = i == j;
        const int mcnt = min(4, max(0, (rows - m_base + 7) >> 3));
        double acc[4][2][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        // ---- acc = L(i, :j) L(j, :j)^T over 32-wide chunks ----
        if (nch > 0) {
          const double *Li = Ls + static_cast<long long>(i) * nkc * CT;
          const double *Lj = Ls + static_cast<long long>(j) * nkc * CT;
          load_chunk(Ci, Li, rows);
          if (!dt) load_chunk(Cj, Lj, PB);
          cp_async_commit();
          for (int c = 0; c < nch; ++c) {
            const int s = c & 1;
            if (c + 1 < nch) {
              load_chunk(Ci + (s ^ 1) * CT, Li + (c + 1) * CT, rows);
              if (!dt) load_chunk(Cj + (s ^ 1) * CT, Lj + (c + 1) * CT, PB);
              cp_async_commit();
              cp_async_wait<1>();
            } else {
              cp_async_wait<0>();
            }
            __syncthreads();
            mma_rows<LDC, KC>(Ci + s * CT, (dt ? Ci : Cj) + s * CT, KC, m_base, n_base, gq, tq, mcnt, acc);
            __syncthreads();  // the stage is refilled (or T written) next
          }
        }
        // ---- T = [K; y^T](i, j) - acc: lower part of the diagonal tile, zero
        //      outside the trapezoid and past kb ----
        {
          int gr[4], gc[4];
          double s[4][4];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) gr[mi] = i0 + m_base + 8 * mi + gq;
#pragma unroll
          for (int q = 0; q < 4; ++q) gc[q] = j0 + n_base + 8 * (q >> 1) + 2 * tq + (q & 1);
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int q = 0; q < 4; ++q) s[mi][q] = 0.0;
          for (int dd = 0; dd < D; ++dd) {
            const double il = sh_par[dd];
            double xr[4], xc[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) xr[mi] = gr[mi] < N ? __ldg(g.X + gr[mi] * D + dd) * il : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) xc[q] = gc[q] < N ? __ldg(g.X + gc[q] * D + dd) * il : 0.0;
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const double t = xr[mi] - xc[q];
                s[mi][q] = fma(t, t, s[mi][q]);
              }
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int r = gr[mi] - i0, c = gc[q] - j0;
              const bool ok = gr[mi] <= N && c < kb && (!dt || c <= r || gr[mi] >= j0 + kb);
              double v = 0.0;
              if (ok) {
                const double kv = gr[mi] == N ? __ldg(g.y + gc[q])
                                              : sf2 * exp(-0.5 * s[mi][q]) + (gr[mi] == gc[q] ? diag_add : 0.0);
                v = kv - acc[mi][q >> 1][q & 1];
              }
              T[r * LDR + c] = v;
            }
        }
        __syncthreads();
        if (dt) {
          // ---- factorise the diagonal tile in place; all threads, one
          //      barrier per column: column jj updates the block with its
          //      unscaled values (A_rl -= A_rj A_lj / A_jj) while column jj-1
          //      is scaled by 1/L_{jj-1,jj-1}; thread (ty, tx) owns rows
          //      ty + 16 u and columns tx + 16 v ----
          bool bad = false;  // uniform: every thread reads the same pivot
          for (int jj = 0; jj < kb; ++jj) {
            const double ajj = T[jj * LDR + jj];
            if (!(ajj > 0.0)) {
              bad = true;
              if (tid == 0) sh_fail = 1;
              break;
            }
            const double iajj = 1.0 / ajj;
            if (jj > 0) {
              const double ipm = 1.0 / diag[jj - 1];
              for (int r = jj + tid; r < kb; r += kThreads) T[r * LDR + jj - 1] *= ipm;
            }
            if (tid == 0) diag[jj] = sqrt(ajj);
            double cj[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int l = tx + 16 * v;
              cj[v] = (l > jj && l < kb) ? T[l * LDR + jj] * iajj : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int r = ty + 16 * u;
              if (r > jj && r < kb) {
                const double arj = T[r * LDR + jj];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                  const int l = tx + 16 * v;
                  if (l > jj && l <= r) T[r * LDR + l] = fma(-arj, cj[v], T[r * LDR + l]);
                }
              }
            }
            __syncthreads();
          }
          if (!bad) {
            for (int c = tid; c < kb; c += kThreads) T[c * LDR + c] = diag[c];
            if (tid < 32) {
              double lg = 0.0;
              for (int c = lane; c < kb; c += 32) lg += log(diag[c]);
              logdet_part += lg;
            }
          }
          __syncthreads();
          if (sh_fail) break;
          // ---- W = L_jj^-1 by forward substitution, column c by the 4 lanes
          //      4c'..4c'+3 of a warp (partial sums over l split 4 ways):
          //      W_cc = 1 / L_cc, W_ic = -(sum_{c <= l < i} L_il W_lc) / L_ii ----
          {
            const int c = tid >> 2, part = tid & 3;  // 64 columns x 4 parts, warp-uniform loop bounds
            for (int e = tid; e < PB * PB; e += kThreads) W[(e / PB) * LDR + (e % PB)] = 0.0;
            __syncthreads();
            if (c < kb && part == 0) W[c * LDR + c] = 1.0 / diag[c];
            __syncwarp();
            for (int ii = 1; ii < kb; ++ii) {
              const bool act = c < ii;  // (c < kb follows)
              double sacc = 0.0;
              if (act)
                for (int l = c + part; l < ii; l += 4) sacc = fma(T[ii * LDR + l], W[l * LDR + c], sacc);
              sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
              sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
              if (act && part == 0) W[ii * LDR + c] = -sacc / diag[ii];
              __syncwarp();
            }
          }
          __syncthreads();
          if (rows <= kb) continue;  // no row below the diagonal in this block (y row is in a later block)
        }
        // ---- L(i, j) = T W^T (rows of the diagonal tile above kb are not
        //      needed; the y row yields alpha) ----
        {
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
          mma_rows<LDR, 0>(T, W, kr, m_base, n_base, gq, tq, mcnt, acc);
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const int r = m_base + 8 * mi + gq;
            if (i0 + r == N) {
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) alpha2 += acc[mi][ni][0] * acc[mi][ni][0] + acc[mi][ni][1] * acc[mi][ni][1];
            }
          }
          if (!dt) {
            double *Lo = Ls + (static_cast<long long>(i) * nkc + 2 * j) * CT;
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
              const int cc = n_base + 8 * ni + 2 * tq;
              double *o = Lo + (cc >> 5) * CT + (cc & 31);
#pragma unroll
              for (int mi = 0; mi < 4; ++mi)
                *reinterpret_cast<double2 *>(o + (m_base + 8 * mi + gq) * LDC) =
                    make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            }
          }
          __syncthreads();  // T (= the chunk stages) is overwritten by the next tile
        }
      }
    }
    // ---- E = 1/2 |alpha|^2 + sum log L_ii + N/2 log 2 pi ----
    const double qs = block_sum(alpha2, red);
    const double ld = block_sum(wid == 0 ? logdet_part : 0.0, red);
    if (tid == 0) {
      const double e = sh_fail ? INFINITY : 0.5 * qs + ld + 0.5 * N * kLn2Pi;
      b.partial[parity][p] = static_cast<float>(e);
      if (g.e64) g.e64[p] = e;
    }
    __syncthreads();
  }
}

}  // namespace

struct GpEngine {
  GpDev g{};
  int grid = 0;
  size_t smem = 0;
};

bool gp_setup(void **handle, const double *X, const double *y, int N, int D, double jitter) {
  GpEngine *E = new GpEngine();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sms *= 2;  // two CTAs (two probe matrices) per SM
  E->grid = sms;
  E->g.N = N;
  E->g.D = D;
  E->g.jitter = jitter;
  const int nrb = (N + 1 + PB - 1) / PB, nkc = 2 * ((N + PB - 1) / PB);
  E->g.nrb = nrb;
  E->g.nkc = nkc;
  double *dX = nullptr, *dy = nullptr, *sc = nullptr;
  if (cudaMalloc(&dX, sizeof(double) * N * D) || cudaMalloc(&dy, sizeof(double) * N) ||
      cudaMalloc(&sc, sizeof(double) * static_cast<size_t>(sms) * nrb * nkc * CT)) {
    cudaFree(dX);
    cudaFree(dy);
    cudaFree(sc);
    delete E;
    return false;
  }
  cudaMemcpy(dX, X, sizeof(double) * N * D, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, y, sizeof(double) * N, cudaMemcpyHostToDevice);
  E->g.X = dX;
  E->g.y = dy;
  E->g.scratch = sc;
  E->smem = (4 * static_cast<size_t>(CT) + PB * LDR + PB + 16) * sizeof(double);
  cudaFuncSetAttribute(k_gp_energy, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(E->smem));
  *handle = E;
  return E->smem <= 200 * 1024;
}

void gp_set_out64(void *handle, double *e64) { static_cast<GpEngine *>(handle)->g.e64 = e64; }

void gp_free(void *handle) {
  GpEngine *E = static_cast<GpEngine *>(handle);
  if (!E) return;
  cudaFree(const_cast<double *>(E->g.X));
  cudaFree(const_cast<double *>(E->g.y));
  cudaFree(E->g.scratch);
  delete E;
}

void gp_energy_pass(void *handle, const BatchDev &b, int parity, const LaunchCtx &lc) {
  GpEngine *E = static_cast<GpEngine *>(handle);
  NSS_PIN_CARVEOUT(k_gp_energy);
  k_gp_energy<<<E->grid, kThreads, E->smem, lc.stream>>>(E->g, b, parity, b.dp);
  ++*lc.launch_counter;
}

}  // namespace nss
