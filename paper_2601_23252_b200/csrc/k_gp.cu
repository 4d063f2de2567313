// A1 for GP hyperparameter marginalisation (P:935-962 shape, R-22): batched
// negative log marginal likelihood of an ARD-RBF Gaussian process in fp64,
//
//   K = sf^2 exp(-1/2 sum_j ((x_aj - x_bj) / l_j)^2) + (sn^2 + jitter) I
//   E = 1/2 y^T K^-1 y + 1/2 log|K| + N/2 log 2 pi,
//   phi = (log l_1..l_D, log sf, log sn).
//
// One CTA per probe matrix (probes are dealt to a persistent grid, two CTAs
// per SM).  The CTA runs a LEFT-looking blocked Cholesky of the (N+1) x N
// lower trapezoid [K; y^T] with 64-wide column blocks: for column block j,
// every 64 x 64 tile T = [K; y^T](i, j) - L(i, :j) L(j, :j)^T is accumulated in
// registers on the fp64 tensor cores (mma.sync m8n8k4 = DMMA, 8 per warp per
// k-step) from the already stored L panels (streamed through a double-buffered
// cp.async pipeline), with K(i, j) generated on the fly from X and phi (the
// tiles below the diagonal by warps 1-7 while warp 0 factorises and inverts
// the diagonal tile, gen_k_below), and every tile below
// becomes L(i, j) = T L_jj^-T (DMMA).  The y^T row turns into alpha^T =
// (L^-1 y)^T on the way, so E needs only
// the pivots (log det) and |alpha|^2.  A non-positive pivot gives E = +inf (K
// not positive definite), as in the oracle.  fp64 throughout: the paper runs
// its GP experiments in double precision.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "batch_chain.cuh"

namespace nss {

namespace {

constexpr int kThreads = 256;
constexpr int PB = 64;        // block edge: column blocks of L and the output tiles
constexpr int LDR = PB + 4;   // stride of the 64 x 64 shared tiles: 68 = 4 mod 16 -> conflict-free DMMA fragments
constexpr int KC = 32;        // k-chunk width of the stored L tiles
constexpr int LDC = KC + 4;   // stride of a stored / staged chunk tile (36 = 4 mod 16)
constexpr int CT = PB * LDC;  // doubles per chunk tile (18 KB)
constexpr int LDF = PB + 1;   // stride of the diagonal block being factorised (odd: conflict-free row walks)
constexpr double kLn2Pi = 1.8378770664093454836;

struct GpDev {
  int N, D;
  const double *X;  // N x D inputs
  const double *y;  // N targets
  double jitter;
  double *scratch;  // per CTA slot: nrb x nkc chunk tiles of L
  double *e64;      // optional fp64 copy of the energies (nss_gp_energy_batch)
  int nrb, nkc;     // row blocks of [L; alpha^T] (N + 1 rows), 32-wide chunks per row block
  unsigned long long *phase_clk;  // -DNSS_GP_PHASES builds only: per CTA {k-loop, combine, factor, W, solve, matrices}
};

// measurement builds (-DNSS_GP_PHASES): SM clocks of thread 0 per phase, summed per CTA
#ifdef NSS_GP_PHASES
#define GP_PHASE(k)                                                       \
  do {                                                                    \
    if (tid == 0) {                                                       \
      const long long t_ = clock64();                                     \
      g.phase_clk[6 * blockIdx.x + (k)] += static_cast<unsigned long long>(t_ - t_last); \
      t_last = t_;                                                        \
    }                                                                     \
  } while (0)
#else
#define GP_PHASE(k) \
  do {              \
  } while (0)
#endif

struct GpChainDev {  // per-CTA round buffers of the fused chain kernel
  float *P;          // [grid][2 parities][2 rows][dp] probe points
  float *E;          // [grid][2][2] energies
  int *cnt;          // [grid][2] probe counts
  int *ones;         // {1, 1}: one partial slice per row
  int *queue;        // chain ticket, reset before each launch
  unsigned long long *prof;  // measurement hook (NSS_GP_PROF): per CTA {t_start, t_end, matrices, chains}
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

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) { dmma_f64(d0, d1, a, b); }

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

// [K; y^T](i', j) for every row block i' below the diagonal block of column
// block j, by warps 1-7 while warp 0 factorises that block: the entries are
// written to the chunk slots L(i', j) will take (row-major, stride LDC), whence
// the combine step reads them.  Same arithmetic, in the same order, as the
// on-the-fly generation of the diagonal tile.  The column inputs (scaled by
// 1/l) are staged in `stage` (free while the diagonal block is factorised)
// when they fit.
__device__ __forceinline__ void gen_k_below(const GpDev &g, int j, int kb, const double *par, double *Ls,
                                            double *stage) {
  const int N = g.N, D = g.D, j0 = j * PB, lane = threadIdx.x & 31, w = (threadIdx.x >> 5) - 1;
  constexpr int kGen = kThreads - 32, kGenWarps = kGen / 32;
  const bool staged = PB * D <= 2 * CT;
  if (staged) {
    for (int e = threadIdx.x - 32; e < PB * D; e += kGen) {
      const int dd = e / PB, c = e - dd * PB;
      stage[e] = c < kb ? __ldg(g.X + (j0 + c) * D + dd) * par[dd] : 0.0;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kGen) : "memory");
  }
  const double sf2 = par[D];
  const int c0 = lane, c1 = lane + 32;
  for (int row = j0 + PB + w; row <= N; row += kGenWarps) {
    const int ib = row / PB, r = row - ib * PB;
    double *o = Ls + (static_cast<long long>(ib) * g.nkc + 2 * j) * CT + r * LDC + lane;
    double v0, v1;
    if (row == N) {
      v0 = c0 < kb ? __ldg(g.y + j0 + c0) : 0.0;
      v1 = c1 < kb ? __ldg(g.y + j0 + c1) : 0.0;
    } else {
      double s0 = 0.0, s1 = 0.0;
      for (int dd = 0; dd < D; ++dd) {
        const double il = par[dd];
        const double xr = __ldg(g.X + row * D + dd) * il;
        const double xc0 = staged ? stage[dd * PB + c0] : (c0 < kb ? __ldg(g.X + (j0 + c0) * D + dd) * il : 0.0);
        const double xc1 = staged ? stage[dd * PB + c1] : (c1 < kb ? __ldg(g.X + (j0 + c1) * D + dd) * il : 0.0);
        const double t0 = xr - xc0, t1 = xr - xc1;
        s0 = fma(t0, t0, s0);
        s1 = fma(t1, t1, s1);
      }
      v0 = sf2 * exp(-0.5 * s0);
      v1 = sf2 * exp(-0.5 * s1);
    }
    if (c0 < kb) o[0] = v0;
    if (c1 < kb) o[CT] = v1;
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
__device__ __forceinline__ double gp_matrix(const GpDev &g, const float *phi, double *Ls, double *sm) {
  const int N = g.N, D = g.D, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double *Ci = sm;            // 2 x CT: chunks of row block i (stage buffers); T aliases them
  double *Cj = Ci + 2 * CT;   // 2 x CT: chunks of row block j
  double *W = Cj + 2 * CT;    // PB x LDR: L_jj^-1 (lower), zero above the diagonal and past kb
  double *diag = W + PB * LDR;  // PB: L_cc
  double *red = diag + PB;      // 8
  double *T = Ci;               // PB x LDR (4352 <= 2 CT doubles)
  double *F = Cj;               // PB x LDF: the diagonal block while it is factorised (4160 <= 2 CT doubles)
  __shared__ double sh_par[NSS_MAX_DIM + 2];
  __shared__ int sh_fail;
  const int nkc = g.nkc, nrb = g.nrb, ncb = (N + PB - 1) / PB;
  // DMMA warp tiles: warp (wr, wc) owns rows 32 wr .. +32, columns 16 wc .. +16
  const int m_base = (wid >> 2) * 32, n_base = (wid & 3) * 16, gq = lane >> 2, tq = lane & 3;
#ifdef NSS_GP_PHASES
  long long t_last = clock64();
  if (tid == 0) g.phase_clk[6 * blockIdx.x + 5] += 1;
#endif

  if (tid < D + 2) {
    const double ph = static_cast<double>(phi[tid]);
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
      GP_PHASE(0);
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
        if (!dt) {
          // generated during the diagonal factorisation (gen_k_below)
          const double *Ko = Ls + (static_cast<long long>(i) * nkc + 2 * j) * CT;
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            const int cc = n_base + 8 * ni + 2 * tq;
            const double *o = Ko + (cc >> 5) * CT + (cc & 31);
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
              const int r = m_base + 8 * mi + gq;
              const bool in = i0 + r <= N;
              const double2 kv = in ? *reinterpret_cast<const double2 *>(o + r * LDC) : make_double2(0.0, 0.0);
              T[r * LDR + cc] = in && cc < kb ? kv.x - acc[mi][ni][0] : 0.0;
              T[r * LDR + cc + 1] = in && cc + 1 < kb ? kv.y - acc[mi][ni][1] : 0.0;
            }
          }
        } else {  // the diagonal tile: generated here
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
              const bool ok = gr[mi] <= N && c < kb && (c <= r || gr[mi] >= j0 + kb);
              double v = 0.0;
              if (ok) {
                const double kv = gr[mi] == N ? __ldg(g.y + gc[q])
                                              : sf2 * exp(-0.5 * s[mi][q]) + (gr[mi] == gc[q] ? diag_add : 0.0);
                v = kv - acc[mi][q >> 1][q & 1];
              }
              if (r < kb)
                F[r * LDF + c] = v;  // the block to factorise
              else
                T[r * LDR + c] = v;
            }
        }
      }
      __syncthreads();
      GP_PHASE(1);
      if (dt) {
        // ---- factorise the diagonal block (in F, odd stride: conflict-free
        //      row walks) and invert its factor, W = L_jj^-1, by one warp in
        //      one left-looking pass over the columns: at step jj lane l owns
        //      rows jj + l, jj + 32 + l of L and columns l, l + 32 of W,
        //        L_rj = (A_rj - sum_{k<jj} L_rk L_jk) / L_jj,  L_jj = sqrt(pivot),
        //        W_jc = -(sum_{k<jj} L_jk W_kc) / L_jj (c < jj),  W_jj = 1 / L_jj,
        //      both sums sharing the loads of row jj of L (W is zero above the
        //      diagonal, so the second sum may start at k = 0); one rsqrt per
        //      column, no divisions; the co-resident CTA keeps the tensor pipe
        //      busy meanwhile ----
        for (int e = tid; e < PB * PB; e += kThreads) W[(e / PB) * LDR + (e % PB)] = 0.0;
        __syncthreads();
        if (wid != 0) {
          // warps 1-7 meanwhile: [K; y^T](i', j) of every tile below, into
          // the slots L(i', j) will take (read back by the combine step)
          gen_k_below(g, j, kb, sh_par, Ls, Ci);
        } else {
          bool bad = false;
          double *w0p = W + lane, *w1p = W + lane + 32;
          for (int jj = 0; jj < kb; ++jj) {
            const int r0 = jj + lane, r1 = r0 + 32;
            const bool v0 = r0 < kb, v1 = r1 < kb;
            double *f0 = F + min(r0, kb - 1) * LDF, *f1 = F + min(r1, kb - 1) * LDF;  // clamped: loads stay in F
            const double *fj = F + jj * LDF;
            double s0 = f0[jj], s1 = f1[jj], u0 = 0.0, u1 = 0.0, x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
            int k = 0;
            for (; k + 1 < jj; k += 2) {
              const double a0 = fj[k], a1 = fj[k + 1];
              s0 = fma(-f0[k], a0, s0);
              u0 = fma(-f0[k + 1], a1, u0);
              s1 = fma(-f1[k], a0, s1);
              u1 = fma(-f1[k + 1], a1, u1);
              x0 = fma(a0, w0p[k * LDR], x0);
              y0 = fma(a1, w0p[(k + 1) * LDR], y0);
              x1 = fma(a0, w1p[k * LDR], x1);
              y1 = fma(a1, w1p[(k + 1) * LDR], y1);
            }
            if (k < jj) {
              const double a0 = fj[k];
              s0 = fma(-f0[k], a0, s0);
              s1 = fma(-f1[k], a0, s1);
              x0 = fma(a0, w0p[k * LDR], x0);
              x1 = fma(a0, w1p[k * LDR], x1);
            }
            s0 += u0;
            s1 += u1;
            x0 += y0;
            x1 += y1;
            const double piv = __shfl_sync(0xffffffffu, s0, 0);
            if (!(piv > 0.0)) {
              bad = true;
              break;
            }
            const double rs = rsqrt(piv);
            if (lane == 0) diag[jj] = piv * rs;
            else if (v0) f0[jj] = s0 * rs;
            if (v1) f1[jj] = s1 * rs;
            if (lane < jj) w0p[jj * LDR] = -x0 * rs;
            else if (lane == jj) w0p[jj * LDR] = rs;
            if (lane + 32 < jj) w1p[jj * LDR] = -x1 * rs;
            else if (lane + 32 == jj) w1p[jj * LDR] = rs;
            __syncwarp();
          }
          if (bad) {
            if (lane == 0) sh_fail = 1;
          } else {
            double lg = 0.0;
            for (int c = lane; c < kb; c += 32) lg += log(diag[c]);
            logdet_part += lg;
          }
        }
        __syncthreads();
        GP_PHASE(2);
        if (sh_fail) break;
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
        GP_PHASE(4);
      }
    }
  }
  // ---- E = 1/2 |alpha|^2 + sum log L_ii + N/2 log 2 pi ----
  const double qs = block_sum(alpha2, red);
  const double ld = block_sum(wid == 0 ? logdet_part : 0.0, red);
  const double e = sh_fail ? INFINITY : 0.5 * qs + ld + 0.5 * N * kLn2Pi;
  __syncthreads();  // sh_par / sh_fail are rewritten by the next matrix
  return e;
}

// The batched pass of the round-synchronous engine: every probe row of the
// round, one matrix per CTA at a time (persistent grid).
__global__ void __launch_bounds__(kThreads, 2) k_gp_energy(GpDev g, BatchDev b, int parity, int dp) {
  extern __shared__ double sm[];
  if (blockIdx.x == 0 && threadIdx.x == 0) b.n_probe[parity ^ 1] = 0;  // the next round's row counter
  const int n = b.n_probe[parity];
  double *Ls = g.scratch + static_cast<long long>(blockIdx.x) * g.nrb * g.nkc * CT;
  for (int p = blockIdx.x; p < n; p += gridDim.x) {
    const double e = gp_matrix(g, b.P[parity] + static_cast<long long>(p) * dp, Ls, sm);
    if (threadIdx.x == 0) {
      b.partial[parity][p] = static_cast<float>(e);
      if (g.e64) g.e64[p] = e;
    }
  }
}

// The fused engine: each CTA takes whole HRSS chains from a queue and runs
// them to completion, its warp 0 advancing the chain state machine
// (batch_chain.cuh, the same code as k_batch_advance) and all warps
// evaluating the one or two probe matrices each round needs.  The decisions,
// draws and energies are those of the round-synchronous engine; what goes is
// the device-wide round barrier, whose last partial wave of 4-ms matrices
// left most SMs idle (C5: 661 probe rows per round on 296 CTA slots).
template <int NPL>
__global__ void __launch_bounds__(kThreads, 2) k_gp_chains(RunDev r, PriorDev pr, BatchDev b, GpDev g,
                                                             GpChainDev q) {
  extern __shared__ double sm[];
  __shared__ float sZ[NPL * 32];
  __shared__ int sh_c;
  const int tid = threadIdx.x;
  double *Ls = g.scratch + static_cast<long long>(blockIdx.x) * g.nrb * g.nkc * CT;
  // this CTA's private round buffers: two parities x two probe rows
  BatchDev bl = b;
  float *pb = q.P + static_cast<long long>(blockIdx.x) * 4 * b.dp;
  bl.P[0] = pb;
  bl.P[1] = pb + 2 * b.dp;
  bl.partial[0] = q.E + blockIdx.x * 4;
  bl.partial[1] = bl.partial[0] + 2;
  bl.n_probe = q.cnt + blockIdx.x * 2;
  bl.slices = q.ones;
  bl.p_stride = 2;
  bl.max_rows = 2;
  bl.A[0] = bl.A[1] = nullptr;
  bl.lin[0] = bl.lin[1] = nullptr;
  bl.eacc[0] = bl.eacc[1] = nullptr;
  volatile int *cnt = bl.n_probe;
  unsigned long long t_start = 0, n_mat = 0, n_ch = 0;
  if (q.prof && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  for (;;) {
    if (tid == 0) {
      sh_c = chain_range(r).x + atomicAdd(q.queue, 1);
      cnt[0] = 0;
      cnt[1] = 0;
    }
    __syncthreads();
    const int c = sh_c;
    if (c >= chain_range(r).y) break;
    for (int par = 0;; par ^= 1) {
      if (tid < 32) advance_chain<NPL>(r, pr, bl, par, c, sZ);
      __syncthreads();
      const int np = cnt[par];
      if (np == 0) break;  // the chain has finished its p steps
      for (int k = 0; k < np; ++k) {
        const double e = gp_matrix(g, bl.P[par] + k * b.dp, Ls, sm);
        if (tid == 0) bl.partial[par][k] = static_cast<float>(e);
      }
      n_mat += np;
      if (tid == 0) cnt[par ^ 1] = 0;
      __syncthreads();
    }
    __syncthreads();  // sh_c is rewritten for the next chain
    ++n_ch;
  }
  if (q.prof && tid == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    unsigned long long *o = q.prof + 4 * blockIdx.x;
    o[0] = t_start;
    o[1] = t_end;
    o[2] += n_mat;
    o[3] += n_ch;
  }
}

}  // namespace

struct GpEngine {
  GpDev g{};
  GpChainDev q{};
  int grid = 0, q_dp = 0;
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
#ifdef NSS_GP_PHASES
  cudaMallocManaged(&E->g.phase_clk, sizeof(unsigned long long) * 6 * sms);
  memset(E->g.phase_clk, 0, sizeof(unsigned long long) * 6 * sms);
#endif
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
#ifdef NSS_GP_PHASES
  cudaDeviceSynchronize();
  double ph[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < E->grid; ++i)
    for (int k = 0; k < 6; ++k) ph[k] += static_cast<double>(E->g.phase_clk[6 * i + k]);
  const double m = ph[5] > 0 ? ph[5] : 1;
  fprintf(stderr, "gp phases, Mclk per matrix (mean over %d CTAs, %.0f matrices): k-loop %.2f combine %.2f factor %.2f "
          "W %.2f solve %.2f\n", E->grid, ph[5], ph[0] / m * 1e-6, ph[1] / m * 1e-6, ph[2] / m * 1e-6, ph[3] / m * 1e-6,
          ph[4] / m * 1e-6);
  cudaFree(E->g.phase_clk);
#endif
  cudaFree(E->q.P);
  cudaFree(E->q.E);
  cudaFree(E->q.cnt);
  cudaFree(E->q.ones);
  cudaFree(E->q.queue);
  if (E->q.prof) {  // last launch's CTA span, matrices and chains accumulated over launches
    cudaDeviceSynchronize();
    unsigned long long t0 = ~0ull, t1 = 0, mmin = ~0ull, mmax = 0, msum = 0, cmax = 0, tmin_end = ~0ull;
    for (int i = 0; i < E->grid; ++i) {
      const unsigned long long *o = E->q.prof + 4 * i;
      t0 = o[0] < t0 ? o[0] : t0;
      t1 = o[1] > t1 ? o[1] : t1;
      tmin_end = o[1] < tmin_end ? o[1] : tmin_end;
      mmin = o[2] < mmin ? o[2] : mmin;
      mmax = o[2] > mmax ? o[2] : mmax;
      msum += o[2];
      cmax = o[3] > cmax ? o[3] : cmax;
    }
    fprintf(stderr, "gp_chains: last launch %.1f ms, first CTA done at %.1f ms; matrices per CTA min %llu max %llu "
            "mean %.1f; max chains %llu\n", (t1 - t0) * 1e-6, (tmin_end - t0) * 1e-6, mmin, mmax,
            static_cast<double>(msum) / E->grid, cmax);
    cudaFree(E->q.prof);
  }
  delete E;
}

void gp_energy_pass(void *handle, const BatchDev &b, int parity, const LaunchCtx &lc) {
  GpEngine *E = static_cast<GpEngine *>(handle);
  NSS_PIN_CARVEOUT(k_gp_energy);
  k_gp_energy<<<E->grid, kThreads, E->smem, lc.stream>>>(E->g, b, parity, b.dp);
  ++*lc.launch_counter;
}

template <int NPL>
void gp_chains_t(GpEngine *E, const RunDev &r, const PriorDev &pr, const BatchDev &b, const LaunchCtx &lc) {
  NSS_MAX_SMEM(k_gp_chains<NPL>, E->smem);
  NSS_PIN_CARVEOUT(k_gp_chains<NPL>);
  k_gp_chains<NPL><<<E->grid, kThreads, E->smem, lc.stream>>>(r, pr, b, E->g, E->q);
  ++*lc.launch_counter;
}

bool gp_chains_pass(void *handle, const RunDev &r, const PriorDev &pr, const BatchDev &b, const LaunchCtx &lc) {
  GpEngine *E = static_cast<GpEngine *>(handle);
  if (E->q_dp != b.dp) {  // per-CTA round buffers, allocated once per dimension
    cudaFree(E->q.P);
    cudaFree(E->q.E);
    cudaFree(E->q.cnt);
    cudaFree(E->q.ones);
    cudaFree(E->q.queue);
    E->q = GpChainDev{};
    int *ones = nullptr;
    if (cudaMalloc(&E->q.P, sizeof(float) * E->grid * 4 * b.dp) || cudaMalloc(&E->q.E, sizeof(float) * E->grid * 4) ||
        cudaMalloc(&E->q.cnt, sizeof(int) * E->grid * 2) || cudaMalloc(&ones, sizeof(int) * 2) ||
        cudaMalloc(&E->q.queue, sizeof(int)))
      return false;
    const int h1[2] = {1, 1};
    if (cudaMemcpy(ones, h1, sizeof(h1), cudaMemcpyHostToDevice)) return false;
    E->q.ones = ones;
    E->q_dp = b.dp;
    if (getenv("NSS_GP_PROF")) {
      cudaMallocManaged(&E->q.prof, sizeof(unsigned long long) * 4 * E->grid);
      memset(E->q.prof, 0, sizeof(unsigned long long) * 4 * E->grid);
    }
  }
  if (cudaMemsetAsync(E->q.queue, 0, sizeof(int), lc.stream)) return false;
  switch ((r.d + 31) / 32) {
    case 1: gp_chains_t<1>(E, r, pr, b, lc); break;
    case 2: gp_chains_t<2>(E, r, pr, b, lc); break;
    case 3: gp_chains_t<3>(E, r, pr, b, lc); break;
    default: gp_chains_t<4>(E, r, pr, b, lc); break;
  }
  return true;
}

}  // namespace nss
