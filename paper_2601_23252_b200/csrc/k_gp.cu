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

// acc(32 x 16 per warp) += Ta(rows) . Tb(rows)^T over k < kb: 4 x 2 DMMA
// 8x8 tiles, operand rows at m_base / n_base of the row-major tiles
__device__ __forceinline__ void mma_rows(const double *Ta, const double *Tb, int kb, int m_base, int n_base, int gq,
                                         int tq, double (&acc)[4][2][2]) {
  const double *pa = Ta + (m_base + gq) * LDR + tq;
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
}

__global__ void __launch_bounds__(kThreads, 2) k_gp_energy(GpDev g, BatchDev b, int parity, int dp) {
  extern __shared__ double sm[];
  const int N = g.N, D = g.D, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int lda = (N + 1) & ~1;  // even row stride: 16-B aligned panel granules for cp.async
  if (blockIdx.x == 0 && tid == 0) b.n_probe[parity ^ 1] = 0;  // the next round's row counter
  const int n = b.n_probe[parity];
  if (static_cast<int>(blockIdx.x) >= n) return;
  double *Ti = sm;                // PB x LDR: panel rows of the current row block (then its X rows)
  double *Tj = Ti + PB * LDR;     // PB x LDR: X rows of an earlier row block; the diagonal block first
  double *W = Tj + PB * LDR;      // PB x LDR: L_kk^-1 (lower), zero above the diagonal and past kb
  double *diag = W + PB * LDR;    // PB: L_cc
  double *red = diag + PB;        // 8
  __shared__ double sh_par[NSS_MAX_DIM + 2];
  __shared__ int sh_fail;
  double *A = g.scratch + static_cast<long long>(blockIdx.x) * (N + 1) * lda;
  double *Lkk = Tj;
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
          const double t = (__ldg(g.X + i * D + q) - __ldg(g.X + j * D + q)) * sh_par[q];
          s = fma(t, t, s);
        }
        row[j] = sf2 * exp(-0.5 * s) + (i == j ? diag_add : 0.0);
      }
    }
    __syncthreads();
    double logdet_part = 0.0;  // lane-held sums of log pivots (warp 0)
    for (int k0 = 0; k0 < N; k0 += PB) {
      const int kb = min(PB, N - k0);
      // 1. diagonal block -> shared memory; all threads, one barrier per
      //    column: column j updates the block with its unscaled values
      //    (A_rl -= A_rj A_lj / A_jj) while column j-1 is scaled by 1/L_{j-1,j-1};
      //    thread (ty, tx) owns rows ty + 16 u and columns tx + 16 v
      for (int e = tid; e < PB * PB; e += kThreads) {
        const int r = e / PB, c = e - r * PB;
        Lkk[r * LDR + c] = (r < kb && c <= r) ? A[static_cast<long long>(k0 + r) * lda + k0 + c] : 0.0;
      }
      __syncthreads();
      bool bad = false;  // uniform: every thread reads the same pivot
      for (int j = 0; j < kb; ++j) {
        const double ajj = Lkk[j * LDR + j];
        if (!(ajj > 0.0)) {
          bad = true;
          if (tid == 0) sh_fail = 1;
          break;
        }
        const double iajj = 1.0 / ajj;
        if (j > 0) {
          const double ipm = 1.0 / diag[j - 1];
          for (int r = j + tid; r < kb; r += kThreads) Lkk[r * LDR + j - 1] *= ipm;
        }
        if (tid == 0) diag[j] = sqrt(ajj);
        double cj[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int l = tx + 16 * v;
          cj[v] = (l > j && l < kb) ? Lkk[l * LDR + j] * iajj : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = ty + 16 * u;
          if (r > j && r < kb) {
            const double arj = Lkk[r * LDR + j];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int l = tx + 16 * v;
              if (l > j && l <= r) Lkk[r * LDR + l] = fma(-arj, cj[v], Lkk[r * LDR + l]);
            }
          }
        }
        __syncthreads();
      }
      if (!bad) {
        for (int c = tid; c < kb; c += kThreads) Lkk[c * LDR + c] = diag[c];
        if (tid < 32) {
          double lg = 0.0;
          for (int c = lane; c < kb; c += 32) lg += log(diag[c]);
          logdet_part += lg;
        }
      }
      __syncthreads();
      if (sh_fail) break;
      // 2. W = L_kk^-1 by forward substitution, column c by the 4 lanes
      //    4c'..4c'+3 of a warp (partial sums over l split 4 ways):
      //    W_cc = 1 / L_cc, W_ic = -(sum_{c <= l < i} L_il W_lc) / L_ii
      {
        const int c = tid >> 2, part = tid & 3;  // 64 columns x 4 parts, warp-uniform loop bounds
        for (int e = tid; e < PB * PB; e += kThreads) W[(e / PB) * LDR + (e % PB)] = 0.0;
        __syncthreads();
        if (c < kb && part == 0) W[c * LDR + c] = 1.0 / diag[c];
        __syncwarp();
        for (int i = 1; i < kb; ++i) {
          const bool act = c < i;  // (c < kb follows)
          double s = 0.0;
          if (act)
            for (int l = c + part; l < i; l += 4) s = fma(Lkk[i * LDR + l], W[l * LDR + c], s);
          s += __shfl_xor_sync(0xffffffffu, s, 1);
          s += __shfl_xor_sync(0xffffffffu, s, 2);
          if (act && part == 0) W[i * LDR + c] = -s / diag[i];
          __syncwarp();
        }
      }
      __syncthreads();
      // 3. row blocks of [r0, N] (the y row included): X = A_panel W^T on the
      //    fp64 tensor cores, written back to A and kept in Ti, then the
      //    trailing update A[i][j] -= sum_c X[i][c] X[j][c] for the tiles
      //    (bi, bj <= bi), columns r0..min(i, N-1)
      const int r0 = k0 + kb;
      const int nrb = (N + 1 - r0 + PB - 1) / PB, ncb = (N - r0 + PB - 1) / PB;
      const int kr = (kb + 3) & ~3;  // DMMA k range (W and Ti zero past kb)
      for (int bi = 0; bi < nrb; ++bi) {
        const int i0 = r0 + bi * PB;
        const int rows = min(PB, N + 1 - i0);
        load_panel_tile(Ti, A, lda, i0, rows, k0, kb);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        {
          double acc[4][2][2];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
          mma_rows(Ti, W, kr, m_base, n_base, gq, tq, acc);
          __syncthreads();  // every warp is done reading Ti
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int r = m_base + 8 * mi + gq, cc = n_base + 8 * ni + 2 * tq + h;
                Ti[r * LDR + cc] = acc[mi][ni][h];  // zero past rows / kb
                if (r < rows && cc < kb) A[static_cast<long long>(i0 + r) * lda + k0 + cc] = acc[mi][ni][h];
              }
          __syncthreads();
        }
        const int nbj = min(bi + 1, ncb);
        for (int bj = 0; bj < nbj; ++bj) {
          const int j0 = r0 + bj * PB;
          const int cols = min(PB, N - j0);
          if (bj != bi) {
            load_panel_tile(Tj, A, lda, j0, cols, k0, kb);
            cp_async_commit();
          }
          // prefetch the 16 outputs (their latency hides behind the tile loads
          // and the product); interior tiles (full, strictly below the
          // diagonal) need no masks and use 16-B accesses
          const bool interior = bj < bi && rows == PB && cols == PB;
          double *Ot = A + static_cast<long long>(i0 + m_base + gq) * lda + j0 + n_base + 2 * tq;
          double cur[4][2][2], acc[4][2][2];
          if (interior) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) {
                const double2 v = *reinterpret_cast<const double2 *>(Ot + 8 * mi * lda + 8 * ni);
                cur[mi][ni][0] = v.x;
                cur[mi][ni][1] = v.y;
              }
          } else {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int r = m_base + 8 * mi + gq, cc = n_base + 8 * ni + 2 * tq + h;
                  cur[mi][ni][h] = (r < rows && cc < cols && j0 + cc <= i0 + r) ? Ot[8 * mi * lda + 8 * ni + h] : 0.0;
                }
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
          if (bj != bi) cp_async_wait<0>();
          __syncthreads();
          mma_rows(Ti, bj == bi ? Ti : Tj, kr, m_base, n_base, gq, tq, acc);
          if (interior) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni)
                *reinterpret_cast<double2 *>(Ot + 8 * mi * lda + 8 * ni) =
                    make_double2(cur[mi][ni][0] - acc[mi][ni][0], cur[mi][ni][1] - acc[mi][ni][1]);
          } else {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int r = m_base + 8 * mi + gq, cc = n_base + 8 * ni + 2 * tq + h;
                  if (r < rows && cc < cols && j0 + cc <= i0 + r)
                    Ot[8 * mi * lda + 8 * ni + h] = cur[mi][ni][h] - acc[mi][ni][h];
                }
          }
          __syncthreads();  // Tj is refilled by the next tile
        }
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
  sms *= 2;  // two CTAs (two probe matrices) per SM
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
  E->smem = (3 * static_cast<size_t>(PB) * LDR + PB + 16) * sizeof(double);
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
