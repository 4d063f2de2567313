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
// update in 64 x 64 tiles: panel rows staged column-major in shared memory,
// 4 x 4 fp64 outputs per thread.  E then needs only
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
constexpr int LDC = PB + 2;  // column-major panel tile stride (even: 16-B aligned double2 loads)
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

// rows [r0, r0+rows) x panel columns [k0, k0+kb) of A -> column-major tile T[c][r]
__device__ __forceinline__ void load_panel_tile(double *T, const double *A, int N, int r0, int rows, int k0,
                                                int kb) {
  for (int e = threadIdx.x; e < PB * PB; e += kThreads) {
    const int r = e / PB, c = e - r * PB;
    T[c * LDC + r] = (r < rows && c < kb) ? A[static_cast<long long>(r0 + r) * N + k0 + c] : 0.0;
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_gp_energy(GpDev g, BatchDev b, int parity, int dp) {
  extern __shared__ double sm[];
  const int N = g.N, D = g.D, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (blockIdx.x == 0 && tid == 0) b.n_probe[parity ^ 1] = 0;  // the next round's row counter
  const int n = b.n_probe[parity];
  if (static_cast<int>(blockIdx.x) >= n) return;
  double *sX = sm;                // N x D
  double *Lkk = sX + ((N * D + 1) & ~1);  // PB x LDK
  double *Ti = Lkk + PB * LDK;            // PB x LDC (column-major: [c][r]); 16-B aligned (PB * LDK even)
  double *Tj = Ti + PB * LDC;     // PB x LDC
  double *inv = Tj + PB * LDC;    // PB: 1 / L_cc
  double *diag = inv + PB;        // PB: L_cc
  double *red = diag + PB;        // 8
  __shared__ double sh_par[NSS_MAX_DIM + 2];
  __shared__ int sh_fail;
  for (int e = tid; e < N * D; e += kThreads) sX[e] = g.X[e];
  double *A = g.scratch + static_cast<long long>(blockIdx.x) * (N + 1) * N;
  __syncthreads();
  const int ty = tid >> 4, tx = tid & 15;  // 4 x 4 outputs per thread in a 64 x 64 tile

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
      double *row = A + static_cast<long long>(i) * N;
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
        Lkk[r * LDK + c] = c <= r ? A[static_cast<long long>(k0 + r) * N + k0 + c] : 0.0;
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
        double *row = A + static_cast<long long>(i) * N + k0;
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
      //    columns r0..min(i, N-1), in 64 x 64 tiles (4 x 4 per thread)
      const int nrb = (N + 1 - r0 + PB - 1) / PB, ncb = (N - r0 + PB - 1) / PB;
      for (int bi = 0; bi < nrb; ++bi) {
        const int i0 = r0 + bi * PB;
        const int rows = min(PB, N + 1 - i0);
        load_panel_tile(Ti, A, N, i0, rows, k0, kb);
        for (int bj = 0; bj <= bi && bj < ncb; ++bj) {
          const int j0 = r0 + bj * PB;
          const int cols = min(PB, N - j0);
          __syncthreads();
          if (bj != bi) load_panel_tile(Tj, A, N, j0, cols, k0, kb);
          __syncthreads();
          const double *Tb = bj == bi ? Ti : Tj;
          // prefetch the 16 outputs (their latency hides behind the rank-kb product)
          double cur[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int r = ty * 4 + u, cc = tx * 4 + v;
              cur[u][v] = (r < rows && cc < cols && j0 + cc <= i0 + r)
                              ? A[static_cast<long long>(i0 + r) * N + j0 + cc]
                              : 0.0;
            }
          double acc[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
#pragma unroll 4
          for (int c = 0; c < kb; ++c) {
            const double2 a01 = *reinterpret_cast<const double2 *>(Ti + c * LDC + ty * 4);
            const double2 a23 = *reinterpret_cast<const double2 *>(Ti + c * LDC + ty * 4 + 2);
            const double2 b01 = *reinterpret_cast<const double2 *>(Tb + c * LDC + tx * 4);
            const double2 b23 = *reinterpret_cast<const double2 *>(Tb + c * LDC + tx * 4 + 2);
            const double av[4] = {a01.x, a01.y, a23.x, a23.y};
            const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int r = ty * 4 + u, cc = tx * 4 + v;
              if (r < rows && cc < cols && j0 + cc <= i0 + r)
                A[static_cast<long long>(i0 + r) * N + j0 + cc] = cur[u][v] - acc[u][v];
            }
        }
        __syncthreads();
      }
    }
    // ---- E = 1/2 |alpha|^2 + sum log L_ii + N/2 log 2 pi ----
    double q = 0.0;
    if (!sh_fail)
      for (int j = tid; j < N; j += kThreads) {
        const double al = A[static_cast<long long>(N) * N + j];
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
      cudaMalloc(&sc, sizeof(double) * static_cast<size_t>(sms) * (N + 1) * N)) {
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
  E->smem = (static_cast<size_t>(N) * D + 1 + PB * LDK + 1 + 2 * PB * LDC + 2 * PB + 16) * sizeof(double);
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
