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
constexpr int PB = 64;       // panel width = trailing-update tile edge
constexpr int LDK = PB + 1;  // diagonal block row stride (doubles)
constexpr int LDR = PB + 4;  // row-major panel tile stride: 68 = 4 mod 16 -> conflict-free DMMA fragments
constexpr double kLn2Pi = 1.8378770664093454836;

struct GpDev {
  int N, D;
  const double *X;  // N x D inputs
  const double *y;  // N targets
  double jitter;
  double *scratch;  // per CTA slot: (N+1) x N
  double *e64;      // optional fp64 copy of the energies (nss_gp_energy_batch)
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

// rows [r0, r0+rows) x panel columns [k0, k0+kb) of A -> row-major tile T[r][c]
// with asynchronous 16-B copies (zero-filled past the edges); the caller
// commits and waits (cp.async.commit_group / wait_group).
__device__ __forceinline__ void load_panel_tile(double *T, const double *A, int lda, int r0, int rows, int k0,
                                                int kb) {
  constexpr int G = PB / 2;  // 16-B granules per tile row
  for (int e = threadIdx.x; e < PB * G; e += kThreads) {
    const int r = e / G, c = 2 * (e - r * G);
    const int valid = (r < rows) ? max(0, min(2, kb - c)) : 0;
    const double *src = valid ? A + static_cast<long long>(r0 + r) * lda + k0 + c : A;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(T + r * LDR + c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid * 8)
                 : "memory");
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

__global__ void __launch_bounds__(kThreads, 1) k_gp_energy(GpDev g, BatchDev b, int parity, int dp) {
  extern __shared__ double sm[];
  const int N = g.N, D = g.D, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int lda = (N + 1) & ~1;  // even row stride: 16-B aligned panel granules for cp.async
  if (blockIdx.x == 0 && tid == 0) b.n_probe[parity ^ 1] = 0;  // the next round's row counter
  const int n = b.n_probe[parity];
  if (static_cast<int>(blockIdx.x) >= n) return;
  double *sX = sm;                // N x D
  double *Lkk = sX + ((N * D + 1) & ~1);  // PB x LDK
  double *Ti = Lkk + PB * LDK;            // PB x LDR (row-major panel rows)
  double *Tj = Ti + PB * LDR;     // 2 x PB x LDR (double buffer)
  double *inv = Tj + 2 * PB * LDR;  // PB: 1 / L_cc
  double *diag = inv + PB;        // PB: L_cc
  double *red = diag + PB;        // 8
  __shared__ double sh_par[NSS_MAX_DIM + 2];
  __shared__ int sh_fail;
  for (int e = tid; e < N * D; e += kThreads) sX[e] = g.X[e];
  double *A = g.scratch + static_cast<long long>(blockIdx.x) * (N + 1) * lda;
  __syncthreads();
  const int ty = tid >> 4, tx = tid & 15;  // diagonal-block owner map
  // trailing update: warp (wr, wc) owns rows 32 wr .. +32, columns 16 wc .. +16
  // of the 64 x 64 tile as 4 x 2 DMMA 8x8 tiles
  const int m_base = (wid >> 2) * 32, n_base = (wid & 3) * 16, gq = lane >> 2, tq = lane & 3;

  for (int p = blockIdx.x; p < n; p += gridDim.x) {
    if (tid < D + 2) {
      const double ph = static_cast<double>(b.P[parity][static_cast<long long>(p) * dp + tid]);
      sh_par[tid] = tid < D ? exp(-ph) : exp(2.0 * ph);  // 1/l_j, sf^2, sn^2
    }
    if (tid == 0) sh_fail = 0;
    __syncthreads();
    const double sf2 = sh_par[D], diag_add = sh_par[D + 1] + g.jitter;
    // ---- build [K; y^T] (lower trapezoid) ----
    for (int i = wid; i <= N; i += kThreads / 32) {
      double *row = A + static_cast<long long>(i) * lda;
      if (i == N) {
        for (int j = lane; j < N; j += 32) row[j] = g.y[j];
        continue;
      }
      for (int j = lane; j <= i; j += 32) {
        double s = 0.0;
        for (int q = 0; q < D; ++q) {
          const double t = (sX[i * D + q] - sX[j * D + q]) * sh_par[q];
          s = fma(t, t, s);
        }
        row[j] = sf2 * exp(-0.5 * s) + (i == j ? diag_add : 0.0);
      }
    }
    __syncthreads();
    double logdet_part = 0.0;  // lane-held sums of log pivots (warp 0)
    for (int k0 = 0; k0 < N; k0 += PB) {
      const int kb = min(PB, N - k0);
      // 1. diagonal block -> shared memory; row-owner Cholesky in warp 0
      //    (lane owns rows lane and lane + 32)
      for (int e = tid; e < kb * kb; e += kThreads) {
        const int r = e / kb, c = e - r * kb;
        Lkk[r * LDK + c] = c <= r ? A[static_cast<long long>(k0 + r) * lda + k0 + c] : 0.0;
      }
      __syncthreads();
      // All threads, one barrier per column: column j updates the trailing
      // block with its unscaled values (A_rl -= A_rj A_lj / A_jj) while
      // column j-1 is scaled by 1/L_{j-1,j-1}; thread (ty, tx) owns rows
      // ty + 16 u and columns tx + 16 v of the block.
      bool bad = false;  // uniform: every thread reads the same pivot
      for (int j = 0; j < kb; ++j) {
        const double ajj = Lkk[j * LDK + j];
        if (!(ajj > 0.0)) {
          bad = true;
          if (tid == 0) sh_fail = 1;
          break;
        }
        const double iajj = 1.0 / ajj;
        if (j > 0) {
          const double ipm = inv[j - 1];
          for (int r = j + tid; r < kb; r += kThreads) Lkk[r * LDK + j - 1] *= ipm;
        }
        if (tid == 0) {
          const double piv = sqrt(ajj);
          inv[j] = 1.0 / piv;
          diag[j] = piv;
        }
        double cj[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int l = tx + 16 * v;
          cj[v] = (l > j && l < kb) ? Lkk[l * LDK + j] * iajj : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = ty + 16 * u;
          if (r > j && r < kb) {
            const double arj = Lkk[r * LDK + j];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int l = tx + 16 * v;
              if (l > j && l <= r) Lkk[r * LDK + l] = fma(-arj, cj[v], Lkk[r * LDK + l]);
            }
          }
        }
        __syncthreads();
      }
      if (!bad) {
        for (int c = tid; c < kb; c += kThreads) Lkk[c * LDK + c] = diag[c];
        if (tid < 32) {
          double lg = 0.0;
          for (int c = lane; c < kb; c += 32) lg += log(diag[c]);
          logdet_part += lg;
        }
      }
      __syncthreads();
      if (sh_fail) break;
      // 2. panel solve x L_kk^T = a for the rows below the block and the y row
      const int r0 = k0 + kb;
      for (int i = r0 + tid; i <= N; i += kThreads) {
        double *row = A + static_cast<long long>(i) * lda + k0;
        double a[PB];
#pragma unroll
        for (int c = 0; c < PB; ++c) a[c] = c < kb ? row[c] : 0.0;
#pragma unroll
        for (int c = 0; c < PB; ++c) {
          if (c < kb) {
            double s0 = a[c], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int j = 0; j + 3 < c; j += 4) {
              s0 = fma(-a[j], Lkk[c * LDK + j], s0);
              s1 = fma(-a[j + 1], Lkk[c * LDK + j + 1], s1);
              s2 = fma(-a[j + 2], Lkk[c * LDK + j + 2], s2);
              s3 = fma(-a[j + 3], Lkk[c * LDK + j + 3], s3);
            }
#pragma unroll
            for (int j = c & ~3; j < c; ++j) s0 = fma(-a[j], Lkk[c * LDK + j], s0);
            a[c] = ((s0 + s1) + (s2 + s3)) * inv[c];
          }
        }
#pragma unroll
        for (int c = 0; c < PB; ++c)
          if (c < kb) row[c] = a[c];
      }
      __syncthreads();
      // 3. trailing update A[i][j] -= sum_c L[i][c] L[j][c] over rows r0..N,
      //    columns r0..min(i, N-1), in 64 x 64 tiles on the fp64 tensor cores
      const int nrb = (N + 1 - r0 + PB - 1) / PB, ncb = (N - r0 + PB - 1) / PB;
      for (int bi = 0; bi < nrb; ++bi) {
        const int i0 = r0 + bi * PB;
        const int rows = min(PB, N + 1 - i0);
        // Ti, then Tj(0) in flight; Tj(bj+1) is fetched while Tj(bj) is used
        load_panel_tile(Ti, A, lda, i0, rows, k0, kb);
        cp_async_commit();
        const int nbj = min(bi + 1, ncb);
        auto fetch = [&](int bj) {
          if (bj < nbj && bj != bi)
            load_panel_tile(Tj + (bj & 1) * PB * LDR, A, lda, r0 + bj * PB, min(PB, N - (r0 + bj * PB)), k0, kb);
          cp_async_commit();  // possibly empty group: keeps the wait count uniform
        };
        fetch(0);
        for (int bj = 0; bj < nbj; ++bj) {
          const int j0 = r0 + bj * PB;
          const int cols = min(PB, N - j0);
          fetch(bj + 1);
          cp_async_wait<1>();  // all but the newest group: Ti and Tj(bj) have landed
          __syncthreads();
          const double *Tj_cur = Tj + (bj & 1) * PB * LDR;
          const double *Tb = bj == bi ? Ti : Tj_cur;
          // prefetch the 16 outputs (their latency hides behind the rank-kb product)
          double cur[4][2][2], acc[4][2][2];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int r = m_base + 8 * mi + gq, cc = n_base + 8 * ni + 2 * tq + h;
                cur[mi][ni][h] = (r < rows && cc < cols && j0 + cc <= i0 + r)
                                     ? A[static_cast<long long>(i0 + r) * lda + j0 + cc]
                                     : 0.0;
                acc[mi][ni][h] = 0.0;
              }
          const double *pa = Ti + (m_base + gq) * LDR + tq;
          const double *pb = Tb + (n_base + gq) * LDR + tq;
#pragma unroll 4
          for (int c = 0; c < kb; c += 4) {
            double av[4], bv[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) av[mi] = pa[8 * mi * LDR + c];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) bv[ni] = pb[8 * ni * LDR + c];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int r = m_base + 8 * mi + gq, cc = n_base + 8 * ni + 2 * tq + h;
                if (r < rows && cc < cols && j0 + cc <= i0 + r)
                  A[static_cast<long long>(i0 + r) * lda + j0 + cc] = cur[mi][ni][h] - acc[mi][ni][h];
              }
          __syncthreads();  // Tj(bj) is refilled by the fetch of iteration bj + 1
        }
        cp_async_wait<0>();
        __syncthreads();
      }
    }
    // ---- E = 1/2 |alpha|^2 + sum log L_ii + N/2 log 2 pi ----
    double q = 0.0;
    if (!sh_fail)
      for (int j = tid; j < N; j += kThreads) {
        const double al = A[static_cast<long long>(N) * lda + j];
        q = fma(al, al, q);
      }
    const double qs = block_sum(q, red);
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
  E->grid = sms;
  E->g.N = N;
  E->g.D = D;
  E->g.jitter = jitter;
  double *dX = nullptr, *dy = nullptr, *sc = nullptr;
  if (cudaMalloc(&dX, sizeof(double) * N * D) || cudaMalloc(&dy, sizeof(double) * N) ||
      cudaMalloc(&sc, sizeof(double) * static_cast<size_t>(sms) * (N + 1) * ((N + 1) & ~1))) {
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
  E->smem = (static_cast<size_t>(N) * D + 1 + PB * LDK + 3 * PB * LDR + 2 * PB + 16) * sizeof(double);
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
