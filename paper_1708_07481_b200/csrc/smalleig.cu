// (d) Small dense float64 linear algebra for LOBPCG's projected problems.
//
// Replaces, for the m x m projected problems (m = l + na + pw <= 3l):
//   _small_gen_eigh (lobpcg.py:168-177): finiteness check, cond2(G_B) <= 1/sqrt(eps),
//     scipy.linalg.eigh(G_A, G_B) (LAPACK dsygvd);
//   _cholesky_orth's Cholesky / triangular inverse (lobpcg.py:228-237) and its
//     acceptance tests, plus a rank-revealing (pivoted) fallback for :241-247.
//
// Generalized problem: G_B = L L' (Cholesky), A' = L^-1 G_A L^-T, Householder
// tridiagonalisation A' = Q T Q', the nev smallest eigenvalues of T by warp
// multisection (Sturm counts), eigenvectors of T by inverse iteration with
// modified Gram-Schmidt inside eigenvalue clusters (as LAPACK dstein), back-
// transformation Q Y and C = L^-T Q Y (B-orthonormal columns).
// cond2(G_B) is bracketed from ||G_B||_F and ||L^-1||_F:
//   ||G_B||_F ||L^-1||_F^2 / m^1.5 <= cond2(G_B) <= ||G_B||_F ||L^-1||_F^2,
// and only when the bracket straddles 1/sqrt(eps) is the exact value computed
// (eigenvalues of G_B by the same tridiagonal + bisection kernels), so the
// ladder takes the reference's branch in every case.
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <mutex>
#include <vector>

#include "smalleig.cuh"

namespace spb {
namespace {

constexpr int ET = 1024;  // threads of the single-CTA kernels

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// ---------------------------------------------------------------------------
// A = sym(G_A), B = sym(G_B) (lobpcg.py:164-165). With segment boundaries
// s1 <= s2 < m the Grams were computed only for blocks seg(i) <= seg(j); the
// strictly lower blocks are taken from their upper mirror (the symmetric value).
__global__ void sym_prep(const double* __restrict__ ga, const double* __restrict__ gb, int ldg,
                         int m, double* __restrict__ A, double* __restrict__ B,
                         SmallStatus* status, int s1 = 1 << 30, int s2 = 1 << 30) {
  int bad = 0;
  const int64_t total = (int64_t)m * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / m), j = (int)(e % m);
    const int si = (i >= s1) + (i >= s2), sj = (j >= s1) + (j >= s2);
    const int64_t ij = (int64_t)i * ldg + j, ji = (int64_t)j * ldg + i;
    double a;
    if (si == sj) a = 0.5 * (ga[ij] + ga[ji]);
    else a = si < sj ? ga[ij] : ga[ji];
    A[e] = a;
    bad |= !isfinite(a);
    if (B) {
      double b = (i == j ? 1.0 : 0.0);
      if (gb) {
        if (si == sj) b = 0.5 * (gb[ij] + gb[ji]);
        else b = si < sj ? gb[ij] : gb[ji];
      }
      B[e] = b;
      bad |= !isfinite(b);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && status)
    atomicOr(&status->nonfinite, 1);
}

// Blocked Cholesky (lower) of the m x m matrix Bsrc into L, then Linv = L^-1.
// NB = 32 panels: the diagonal block is factored by warp 0 (warp-synchronous),
// the sub-panel by a triangular solve (thread per row) and the trailing matrix
// by a rank-32 update (warp per row) -> 3 CTA barriers per panel. Linv: the
// 32 x 32 diagonal blocks are inverted by one warp each, then block rows are
// formed in order (2 barriers per block row).
// mode 0 (sygv): cond bracket into status. mode 1 (cholqr): the reference's
// acceptance tests (lobpcg.py:231-235) and Rinv = (L^-1)' written to Linv.
constexpr int CB = 32;

// ||L^-1||_F and the cond2 bracket (mode 0), or Rinv = (L^-1)' in place (mode 1).
// chol_epilogue with ||L^-1||_F^2 partials already accumulated by the caller
// and L^-1 already written in the mode's orientation.
__device__ void chol_epilogue_fl(int m, double fb, double fl, int mode, SmallStatus* status,
                                 double* red) {
  const int tid = threadIdx.x;
  fl = block_sum(fl, red);
  if (mode == 0 && tid == 0) {
    const double upper = sqrt(fb) * fl;
    const double lower = upper / (m * sqrt((double)m));
    status->fro_b = sqrt(fb);
    status->fro_linv = sqrt(fl);
    status->cond_hi = upper;
    status->cond_lo = lower;
    status->cond_state = upper <= kCondMax ? 0 : (lower > kCondMax ? 1 : 2);
  }
}

__device__ void chol_epilogue(int m, double fb, double* __restrict__ Linv, int mode,
                              SmallStatus* status, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double fl = 0.0;
  for (int i = warp; i < m; i += (int)(blockDim.x >> 5))
    for (int j = lane; j <= i; j += 32) {
      const double v = Linv[(int64_t)i * m + j];
      fl += v * v;
    }
  fl = block_sum(fl, red);
  if (mode == 0) {
    if (tid == 0) {
      // fb, fl are squared Frobenius norms: bracket = ||B||_F ||L^-1||_F^2
      const double upper = sqrt(fb) * fl;
      const double lower = upper / (m * sqrt((double)m));
      status->fro_b = sqrt(fb);
      status->fro_linv = sqrt(fl);
      status->cond_hi = upper;
      status->cond_lo = lower;
      status->cond_state = upper <= kCondMax ? 0 : (lower > kCondMax ? 1 : 2);
    }
  } else {
    // Rinv = (L^-1)' in place of Linv (upper triangular)
    for (int i = warp; i < m; i += (int)(blockDim.x >> 5))
      for (int j = i + 1 + lane; j < m; j += 32) {
        const double a = Linv[(int64_t)i * m + j], b = Linv[(int64_t)j * m + i];
        Linv[(int64_t)i * m + j] = b;
        Linv[(int64_t)j * m + i] = a;
      }
  }
}


__global__ void __launch_bounds__(ET)
chol_linv(const double* __restrict__ Bsrc, int m, double* __restrict__ Lg, double* __restrict__ Linv,
          int mode, SmallStatus* status) {
  extern __shared__ double smem[];
  __shared__ double red[33];
  __shared__ int fail;
  const bool in_smem = (size_t)m * m * sizeof(double) <= 200 * 1024;
  double* L = in_smem ? smem : Lg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (status->nonfinite) return;
  double fb = 0.0;
  for (int i = warp; i < m; i += ET / 32)
    for (int j = lane; j < m; j += 32) {
      const double v = Bsrc[(int64_t)i * m + j];
      L[(int64_t)i * m + j] = v;
      fb += v * v;
    }
  fb = block_sum(fb, red);
  if (tid == 0) {
    fail = 0;
    if (mode == 1) {  // diag > 0 and min diag > (eps na)^2 max diag (lobpcg.py:229-231)
      double dmin = DBL_MAX, dmax = -DBL_MAX;
      for (int i = 0; i < m; ++i) {
        dmin = fmin(dmin, Bsrc[(int64_t)i * m + i]);
        dmax = fmax(dmax, Bsrc[(int64_t)i * m + i]);
      }
      status->dmin = dmin;
      status->dmax = dmax;
      const double t = kEps64 * m;
      if (!(dmin > 0.0) || !(dmin > t * t * dmax)) fail = 1;
    }
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) status->fallback = 1;
    return;
  }
  for (int kb = 0; kb < m; kb += CB) {
    const int nb = min(CB, m - kb);
    if (warp == 0) {  // (a) diagonal block, warp-synchronous
      int f = 0;
      for (int c = 0; c < nb; ++c) {
        double* Lc = L + (int64_t)(kb + c) * m + kb;
        const double dcc = Lc[c];
        f = !(dcc > 0.0);
        if (f) break;
        const double piv = sqrt(dcc);
        __syncwarp();
        if (lane == 0) Lc[c] = piv;
        if (lane > c && lane < nb) L[(int64_t)(kb + lane) * m + kb + c] /= piv;
        __syncwarp();
        if (lane > c && lane < nb) {
          double* Li = L + (int64_t)(kb + lane) * m + kb;
          const double lic = Li[c];
          for (int q = c + 1; q <= lane; ++q) Li[q] -= lic * L[(int64_t)(kb + q) * m + kb + c];
        }
        __syncwarp();
      }
      if (lane == 0 && f) fail = 1;
    }
    __syncthreads();
    if (fail) break;
    // (b) sub-panel: x L11' = A21 row by row
    for (int i = kb + nb + tid; i < m; i += ET) {
      double* Li = L + (int64_t)i * m + kb;
      for (int c = 0; c < nb; ++c) {
        const double* Lc = L + (int64_t)(kb + c) * m + kb;
        double x = Li[c];
        for (int q = 0; q < c; ++q) x -= Li[q] * Lc[q];
        Li[c] = x / Lc[c];
      }
    }
    __syncthreads();
    // (c) trailing update, lower triangle
    for (int i = kb + nb + warp; i < m; i += ET / 32) {
      const double* Lip = L + (int64_t)i * m + kb;
      double li[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) li[c] = c < nb ? Lip[c] : 0.0;
      for (int q = kb + nb + lane; q <= i; q += 32) {
        const double* Lqp = L + (int64_t)q * m + kb;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < CB; ++c)
          if (c < nb) acc += li[c] * Lqp[c];
        L[(int64_t)i * m + q] -= acc;
      }
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) {
      if (mode == 0) status->not_pd = 1;
      else status->fallback = 1;
    }
    return;
  }
  if (mode == 1 && tid == 0) {
    double rmin = DBL_MAX, rmax = -DBL_MAX;
    for (int i = 0; i < m; ++i) {
      rmin = fmin(rmin, L[(int64_t)i * m + i]);
      rmax = fmax(rmax, L[(int64_t)i * m + i]);
    }
    status->rmin = rmin;
    status->rmax = rmax;
    if (!(rmin > sqrt(kEps64) * rmax)) fail = 1;  // lobpcg.py:235
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) status->fallback = 1;
    return;
  }
  // ---- Linv. L is copied to global (read-mostly, L1/L2-cached broadcasts); the
  // inverse is built in the shared buffer when it fits: diagonal 32 x 32 blocks
  // by one warp each, then block rows in order (2 barriers per block row).
  if (in_smem) {
    for (int i = warp; i < m; i += ET / 32)
      for (int j = lane; j <= i; j += 32) Lg[(int64_t)i * m + j] = L[(int64_t)i * m + j];
    __syncthreads();
  }
  const double* Lr = Lg;  // L (lower) in global memory from here on
  const bool inv_smem = in_smem && ((size_t)m * m + (size_t)CB * m) * sizeof(double) <= 224 * 1024;
  double* Vi = inv_smem ? smem : Linv;                    // inverse being built
  double* T = inv_smem ? smem + (size_t)m * m : Lg + (size_t)m * m;  // 32 x m scratch
  for (int i = warp; i < m; i += ET / 32)
    for (int j = lane; j < m; j += 32) Vi[(int64_t)i * m + j] = 0.0;
  __syncthreads();
  const int nbk = (m + CB - 1) / CB;
  for (int bdx = warp; bdx < nbk; bdx += ET / 32) {
    const int kb = bdx * CB, nb = min(CB, m - kb);
    for (int i = 0; i < nb; ++i) {  // column lane of the inverse block, row by row
      const double* Li = Lr + (int64_t)(kb + i) * m + kb;
      if (lane <= i && lane < nb) {
        double x = (i == lane) ? 1.0 : 0.0;
        for (int q = lane; q < i; ++q) x -= Li[q] * Vi[(int64_t)(kb + q) * m + kb + lane];
        Vi[(int64_t)(kb + i) * m + kb + lane] = x / Li[i];
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int bi = 1; bi < nbk; ++bi) {
    const int ib = bi * CB, ni = min(CB, m - ib);
    // T[r][c] = sum_{q=c..ib-1} L[ib+r][q] Linv[q][c], c < ib
    for (int r = warp; r < ni; r += ET / 32) {
      const double* Lrow = Lr + (int64_t)(ib + r) * m;
      for (int c = lane; c < ib; c += 32) {
        double acc = 0.0;
        for (int q = c; q < ib; ++q) acc += Lrow[q] * Vi[(int64_t)q * m + c];
        T[(size_t)r * m + c] = acc;
      }
    }
    __syncthreads();
    for (int r = warp; r < ni; r += ET / 32) {
      for (int c = lane; c < ib; c += 32) {
        double acc = 0.0;
        for (int q = 0; q <= r; ++q) acc += Vi[(int64_t)(ib + r) * m + ib + q] * T[(size_t)q * m + c];
        Vi[(int64_t)(ib + r) * m + c] = -acc;
      }
    }
    __syncthreads();
  }
  if (inv_smem) {
    for (int i = warp; i < m; i += ET / 32)
      for (int j = lane; j < m; j += 32) Linv[(int64_t)i * m + j] = Vi[(int64_t)i * m + j];
    __syncthreads();
  }
  chol_epilogue(m, fb, Linv, mode, status, red);
}

// Cholesky + inverse for m <= kCholLdlMax in one shared-memory pass, one CTA
// barrier per column: right-looking LDL' (no square root or division on the
// critical path besides one reciprocal per column, computed by the thread that
// produced the next pivot), with the unit-lower inverse built alongside in the
// upper triangle (Linv'[r][j] stored at [j][r]); L = L' D^1/2 and
// L^-1 = D^-1/2 L'^-1 are formed at the end. Same outputs and status protocol
// as chol_linv.
constexpr int kCholLdlMax = 164;

__global__ void __launch_bounds__(ET)
chol_ldl(const double* __restrict__ Bsrc, int m, double* __restrict__ Lg, double* __restrict__ Linv,
         int mode, SmallStatus* status) {
  extern __shared__ double smem[];
  __shared__ double red[33];
  __shared__ int fail;
  const int ld = m | 1;  // odd row stride: column walks are bank-conflict free
  double* A = smem;      // m x ld
  double* dinv = smem + (size_t)m * ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (status->nonfinite) return;
  double fb = 0.0;
  for (int i = warp; i < m; i += ET / 32)
    for (int j = lane; j < m; j += 32) {
      const double v = Bsrc[(int64_t)i * m + j];
      A[i * ld + j] = v;
      fb += v * v;
    }
  fb = block_sum(fb, red);
  if (tid == 0) {
    fail = 0;
    if (mode == 1) {  // diag > 0 and min diag > (eps na)^2 max diag (lobpcg.py:229-231)
      double dmin = DBL_MAX, dmax = -DBL_MAX;
      for (int i = 0; i < m; ++i) {
        dmin = fmin(dmin, A[i * ld + i]);
        dmax = fmax(dmax, A[i * ld + i]);
      }
      status->dmin = dmin;
      status->dmax = dmax;
      const double t = kEps64 * m;
      if (!(dmin > 0.0) || !(dmin > t * t * dmax)) fail = 1;
    }
    if (!fail) {
      const double d0 = A[0];
      if (!(d0 > 0.0)) fail = 2;
      dinv[0] = 1.0 / d0;
    }
  }
  __syncthreads();
  if (fail == 1) {
    if (tid == 0) status->fallback = 1;
    return;
  }
  for (int c = 0; c < m && !fail; ++c) {
    const double rc = dinv[c];
    // (a) trailing update A[i][q] -= (A[i][c] / d_c) A[q][c], c < q <= i
    for (int i = c + 1 + warp; i < m; i += ET / 32) {
      const double lic = A[i * ld + c] * rc;
      double* Ai = A + i * ld;
      for (int q = c + 1 + lane; q <= i; q += 32) Ai[q] = fma(-lic, A[q * ld + c], Ai[q]);
      if (i == c + 1 && lane == 0) {  // next pivot is final: its reciprocal
        const double dn = Ai[c + 1];
        if (!(dn > 0.0)) fail = 2;
        dinv[c + 1] = 1.0 / dn;
      }
    }
    // (b) unit-lower inverse, column c-1: Linv'[r][j] -= L'[r][c-1] Linv'[c-1][j]
    if (c >= 1) {
      const int i = c - 1;
      const double ri = dinv[i];
      for (int r = c + warp; r < m; r += ET / 32) {
        const double lri = A[r * ld + i] * ri;
        for (int j = lane; j < i; j += 32) A[j * ld + r] = fma(-lri, A[j * ld + i], A[j * ld + r]);
        if (lane == 0) A[i * ld + r] = -lri;
      }
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) {
      if (mode == 0) status->not_pd = 1;
      else status->fallback = 1;
    }
    return;
  }
  if (mode == 1 && tid == 0) {
    double rmin = DBL_MAX, rmax = -DBL_MAX;
    for (int i = 0; i < m; ++i) {
      const double r = sqrt(A[i * ld + i]);
      rmin = fmin(rmin, r);
      rmax = fmax(rmax, r);
    }
    status->rmin = rmin;
    status->rmax = rmax;
    if (!(rmin > sqrt(kEps64) * rmax)) fail = 1;  // lobpcg.py:235
  }
  // D^-1/2 into dinv
  for (int i = tid; i < m; i += ET) dinv[i] = 1.0 / sqrt(A[i * ld + i]);
  __syncthreads();
  if (fail) {
    if (tid == 0) status->fallback = 1;
    return;
  }
  for (int i = warp; i < m; i += ET / 32) {
    const double ri = dinv[i];
    for (int j = lane; j < m; j += 32) {
      double l = 0.0, v = 0.0;
      if (j < i) {
        l = A[i * ld + j] * dinv[j];  // L'[i][j] sqrt(d_j) = A[i][j] / sqrt(d_j)
        v = A[j * ld + i] * ri;       // D^-1/2 row scaling of Linv'
      } else if (j == i) {
        l = 1.0 / ri;
        v = ri;
      }
      Lg[(int64_t)i * m + j] = l;
      Linv[(int64_t)i * m + j] = v;
    }
  }
  __syncthreads();
  chol_epilogue(m, fb, Linv, mode, status, red);
}

__device__ __forceinline__ void tri_index(int t, int* ti, int* tq) {
  int r = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  while (r * (r + 1) / 2 > t) --r;
  *ti = r;
  *tq = t - r * (r + 1) / 2;
}

// min / max over m strided doubles (optionally their square roots) by one warp;
// every lane returns the result.
__device__ __forceinline__ void warp_minmax(const double* base, int64_t stride, int m, bool root,
                                            double* mn, double* mx) {
  const int lane = threadIdx.x & 31;
  double a = DBL_MAX, b = -DBL_MAX;
  for (int i = lane; i < m; i += 32) {
    const double v = root ? sqrt(base[(int64_t)i * stride]) : base[(int64_t)i * stride];
    a = fmin(a, v);
    b = fmax(b, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  *mn = a;
  *mx = b;
}

// Blocked Cholesky + inverse for m <= kCholLdlMax with warp-synchronous
// panels (same packed layout, outputs and status protocol as chol_ldl):
//  P1  the 32x32 diagonal block is factored (LDL') by warp 0 in registers,
//      lane i = row i, columns broadcast by shuffles: no CTA barrier per column;
//  P2  the rows below the block solve against it, one thread per row, right-
//      looking inside the row (independent FMAs);
//  P3  one rank-32 update of the trailing lower triangle in 4x4 register tiles
//      against a D^-1-scaled copy of the panel.
// The unit-lower inverse is formed by blocks as in chol_blk (diagonal blocks by
// one warp each in registers, then block rows). Three CTA barriers per panel.
constexpr int CWT = 512;  // threads of chol_wsync

__global__ void __launch_bounds__(CWT)
chol_wsync(const double* __restrict__ Bsrc, int m, double* __restrict__ Lg, double* __restrict__ Linv,
           int mode, SmallStatus* status, long long* trace) {
  extern __shared__ double smem[];
  __shared__ double red[33];
  __shared__ int fail;
  __shared__ double Lp[32][33];  // L' of the current diagonal block (unit lower, scaled)
  const int ld = m | 1;
  double* A = smem;                          // m x ld packed: L' d below, X' above
  double* S = A + (size_t)m * ld;            // m x 33: D^-1 scaled panel / block scratch
  double* dinv = S + (size_t)m * 33;         // m
  const int sld = 33;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (status->nonfinite) return;
  double fb = 0.0;
  for (int i = warp; i < m; i += CWT / 32)
    for (int j = lane; j < m; j += 32) {
      const double v = Bsrc[(int64_t)i * m + j];
      A[i * ld + j] = v;
      fb += v * v;
    }
  fb = block_sum(fb, red);
  const bool tr = trace && threadIdx.x == 0;
  if (tr) trace[0] = clock64();
  if (warp == 0) {
    int f0 = 0;
    if (mode == 1) {  // diag > 0 and min diag > (eps na)^2 max diag (lobpcg.py:229-231)
      double dmin, dmax;
      warp_minmax(A, ld + 1, m, false, &dmin, &dmax);
      const double t = kEps64 * m;
      if (!(dmin > 0.0) || !(dmin > t * t * dmax)) f0 = 1;
      if (lane == 0) {
        status->dmin = dmin;
        status->dmax = dmax;
      }
    }
    if (lane == 0) fail = f0;
  }
  __syncthreads();
  if (fail == 1) {
    if (tid == 0) status->fallback = 1;
    return;
  }
  int hti = 0, htq = 0;
  tri_index(tid, &hti, &htq);  // this thread's (row, col) in any trailing triangle
  for (int kb = 0; kb < m; kb += 32) {
    const int nb = min(32, m - kb);
    const int ke = kb + nb;
    if (tr) trace[1 + (kb >> 5) * 4] = clock64();
    // ---- P1: diagonal block, right-looking; one element of the block's
    // trailing triangle per thread. Two columns per CTA barrier: every thread
    // forms column c+1's update by column c on the fly (same operations as a
    // separate step), then applies both rank-1 updates to its element.
    int c = 0;
    bool bad = false;  // uniform
    for (; c + 1 < nb; c += 2) {
      const int kc = kb + c;
      const double dc = A[kc * ld + kc];
      const double a10 = A[(kc + 1) * ld + kc];
      if (!(dc > 0.0)) {
        if (tid == 0) fail = 2;
        bad = true;
        break;  // uniform: every thread read the same pivot
      }
      const double rc = 1.0 / dc;
      const double d1 = fma(-a10 * rc, a10, A[(kc + 1) * ld + kc + 1]);
      if (!(d1 > 0.0)) {
        if (tid == 0) fail = 2;
        bad = true;
        break;
      }
      const double r1 = 1.0 / d1;
      const int rem = nb - 1 - c;  // rows/cols kc+1 .. kb+nb-1
      int paddr = -1;              // column c+1 result: written after the barrier,
      double pval = 0.0;           // as other threads read the old value this step
      if (tid < rem * (rem + 1) / 2) {
        const int i = kc + 1 + hti, q = kc + 1 + htq;
        const double aic = A[i * ld + kc], aqc = A[q * ld + kc];
        const double ai1 = fma(-aic * rc, a10, A[i * ld + kc + 1]);  // column c+1 after step c
        if (q == kc + 1) {
          paddr = i * ld + q;
          pval = i > kc + 1 ? ai1 : d1;
        } else {
          const double aq1 = fma(-aqc * rc, a10, A[q * ld + kc + 1]);
          const double t = fma(-aic * rc, aqc, A[i * ld + q]);
          A[i * ld + q] = fma(-ai1 * r1, aq1, t);
        }
      }
      if (tid == 0) {
        dinv[kc] = rc;
        dinv[kc + 1] = r1;
      }
      __syncthreads();
      if (paddr >= 0) A[paddr] = pval;  // next step reads columns c+2, c+3 only
    }
    if (!bad && c < nb) {  // odd last column
      const double dc = A[(kb + c) * ld + kb + c];
      if (!(dc > 0.0)) {
        if (tid == 0) fail = 2;
      } else if (tid == 0) {
        dinv[kb + c] = 1.0 / dc;
      }
    }
    __syncthreads();
    if (fail) break;
    // scaled unit-lower L' of the block for P2
    for (int x = tid; x < 32 * 32; x += CWT) {
      const int i = x >> 5, c = x & 31;
      Lp[i][c] = (i < nb && c < i) ? A[(kb + i) * ld + kb + c] * dinv[kb + c] : (i == c ? 1.0 : 0.0);
    }
    __syncthreads();
    if (tr) trace[2 + (kb >> 5) * 4] = clock64();
    if (fail) break;
    if (ke >= m) break;
    // ---- P2: rows below the block, one thread per row
    for (int i = ke + tid; i < m; i += CWT) {
      double x[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) x[t] = t < nb ? A[i * ld + kb + t] : 0.0;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
#pragma unroll
        for (int c = t + 1; c < 32; ++c) x[c] = fma(-x[t], Lp[c][t], x[c]);
      }
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (t < nb) {
          A[i * ld + kb + t] = x[t];
          S[i * sld + t] = x[t] * dinv[kb + t];
        }
    }
    __syncthreads();
    if (tr) trace[3 + (kb >> 5) * 4] = clock64();
    // ---- P3: trailing update A[i][q] -= sum_t A[i][kb+t] S[q][t], i >= q >= ke, 4x4 tiles
    const int T = m - ke;
    const int TT = (T + 3) / 4;
    const int ntile = TT * (TT + 1) / 2;
    for (int t = tid; t < ntile; t += CWT) {
      int ti, tq;
      tri_index(t, &ti, &tq);
      const int i0 = ke + 4 * ti, q0 = ke + 4 * tq;
      double acc[4][4];
#pragma unroll
      for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) acc[a2][b2] = 0.0;
      for (int c = 0; c < nb; ++c) {
        double av[4], sv[4];
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2) {
          av[a2] = i0 + a2 < m ? A[(i0 + a2) * ld + kb + c] : 0.0;
          sv[a2] = q0 + a2 < m ? S[(q0 + a2) * sld + c] : 0.0;
        }
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2) acc[a2][b2] = fma(av[a2], sv[b2], acc[a2][b2]);
      }
#pragma unroll
      for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) {
          const int i = i0 + a2, qq = q0 + b2;
          if (i < m && qq <= i) A[i * ld + qq] -= acc[a2][b2];
        }
    }
    __syncthreads();
    if (tr) trace[4 + (kb >> 5) * 4] = clock64();
  }
  if (tr) trace[40] = clock64();
  if (fail) {
    if (tid == 0) {
      if (mode == 0) status->not_pd = 1;
      else status->fallback = 1;
    }
    return;
  }
  if (mode == 1 && warp == 0) {
    double rmin, rmax;
    warp_minmax(A, ld + 1, m, true, &rmin, &rmax);
    if (lane == 0) {
      status->rmin = rmin;
      status->rmax = rmax;
      if (!(rmin > sqrt(kEps64) * rmax)) fail = 1;  // lobpcg.py:235
    }
  }
  for (int i = tid; i < m; i += CWT) dinv[i] = 1.0 / sqrt(A[i * ld + i]);
  __syncthreads();
  if (fail) {
    if (tid == 0) status->fallback = 1;
    return;
  }
  // ---- L' = A / d (strictly lower, in place); X = L'^-1 transposed into the upper triangle
  for (int i = warp; i < m; i += CWT / 32)
    for (int j = lane; j < i; j += 32) A[i * ld + j] *= dinv[j] * dinv[j];
  __syncthreads();
  if (tr) trace[41] = clock64();
  const int nblk = (m + 31) / 32;
  for (int bI = warp; bI < nblk; bI += CWT / 32) {  // diagonal blocks: lane = column j
    const int b0 = bI * 32, bn = min(32, m - b0);
    const int j = lane;
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (t >= j && t < bn) {
#pragma unroll
        for (int i = t + 1; i < 32; ++i)
          if (i < bn) x[i] = fma(-A[(b0 + i) * ld + b0 + t], x[t], x[i]);
      }
    }
    if (j < bn)
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i > j && i < bn) A[(b0 + j) * ld + b0 + i] = x[i];
  }
  __syncthreads();
  if (tr) trace[42] = clock64();
  // block rows on the FP64 tensor pipe (mma.sync m8n8k4): R = L'_{I,<I} X_{<I,<I},
  // then X_{I,<I} = -X_II R; every warp owns 8 x 8 output tiles
  for (int bI = 1; bI < nblk; ++bI) {
    const int i0 = bI * 32, ni = min(32, m - i0);
    double* R = S;  // ni x i0, row pitch i0
    const int mtiles = (ni + 7) / 8, ntiles = i0 / 8;
    const int fr = lane >> 2, fk = lane & 3;  // fragment row / k index
    for (int t = warp; t < mtiles * ntiles; t += CWT / 32) {
      const int mt = t / ntiles, nt = t % ntiles;
      const int r = mt * 8 + fr, j0 = nt * 8, jb = j0 + fr;  // A row; B column for this lane
      double c0 = 0.0, c1 = 0.0;
      for (int k0 = j0 & ~3; k0 < i0; k0 += 4) {
        const int k = k0 + fk;
        const double av = r < ni ? A[(i0 + r) * ld + k] : 0.0;               // L'[i0+r][k]
        const double bv = k > jb ? A[jb * ld + k] : (k == jb ? 1.0 : 0.0);   // X[k][jb]
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0), "+d"(c1)
                     : "d"(av), "d"(bv));
      }
      const int rr = mt * 8 + fr, cc = j0 + 2 * fk;
      if (rr < ni) {
        R[rr * i0 + cc] = c0;
        R[rr * i0 + cc + 1] = c1;
      }
    }
    __syncthreads();
    for (int t = warp; t < mtiles * ntiles; t += CWT / 32) {
      const int mt = t / ntiles, nt = t % ntiles;
      const int r = mt * 8 + fr, jb = nt * 8 + fr;
      double c0 = 0.0, c1 = 0.0;
      for (int q0 = 0; q0 < ni; q0 += 4) {
        const int q = q0 + fk;
        // X_II[r][q] (unit lower, stored transposed) and R[q][jb]
        const double av = (r < ni && q < ni) ? (r > q ? A[(i0 + q) * ld + i0 + r] : (r == q ? 1.0 : 0.0)) : 0.0;
        const double bv = q < ni ? R[q * i0 + jb] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0), "+d"(c1)
                     : "d"(av), "d"(bv));
      }
      const int rr = mt * 8 + fr, cc = nt * 8 + 2 * fk;
      if (rr < ni) {
        A[cc * ld + i0 + rr] = -c0;
        A[(cc + 1) * ld + i0 + rr] = -c1;
      }
    }
    __syncthreads();
  }
  if (tr) trace[43] = clock64();
  // L = L' D^1/2 and L^-1 (mode 1: its transpose, the R^-1 of the QR view),
  // row-major coalesced stores; ||L^-1||_F^2 accumulated on the way
  double* sq = S;  // sqrt(d_j) (S is free after the block rows)
  for (int j = tid; j < m; j += CWT) sq[j] = 1.0 / dinv[j];
  __syncthreads();
  double fl = 0.0;
  for (int i = warp; i < m; i += CWT / 32) {
    const double ri = dinv[i];
    for (int j = lane; j < m; j += 32) {
      const double l = j < i ? A[i * ld + j] * sq[j] : (j == i ? sq[i] : 0.0);
      Lg[(int64_t)i * m + j] = l;
      if (mode == 0) {
        const double v = j < i ? A[j * ld + i] * ri : (j == i ? ri : 0.0);
        Linv[(int64_t)i * m + j] = v;
        fl = fma(v, v, fl);
      } else {
        // row i of (L^-1)' = column i of L^-1: element (i, j) = L^-1[j][i], j >= i
        const double v = j > i ? A[i * ld + j] * dinv[j] : (j == i ? ri : 0.0);
        Linv[(int64_t)i * m + j] = v;
        fl = fma(v, v, fl);
      }
    }
  }
  if (tr) trace[44] = clock64();
  chol_epilogue_fl(m, fb, fl, mode, status, red);
  if (tr) trace[45] = clock64();
}

size_t chol_wsync_smem(int m) {
  return sizeof(double) * ((size_t)m * (m | 1) + (size_t)m * 33 + m);
}

// C = op(A) op(B) for small float64 matrices, 32x32 tiles, 256 threads.
__global__ void __launch_bounds__(256)
small_gemm(int ta, int tb, int M, int N, int K, const double* __restrict__ A, int lda,
           const double* __restrict__ B, int ldb, double* __restrict__ C, int ldc) {
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;  // 8 rows of 4
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  double acc[4] = {0, 0, 0, 0};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int e = tid; e < 1024; e += 256) {
      const int r = e >> 5, c = e & 31;
      const int gi = i0 + r, gk = k0 + c;
      double a = 0.0;
      if (gi < M && gk < K) a = ta ? A[(int64_t)gk * lda + gi] : A[(int64_t)gi * lda + gk];
      As[r][c] = a;
      const int gk2 = k0 + r, gj = j0 + c;
      double bv = 0.0;
      if (gk2 < K && gj < N) bv = tb ? B[(int64_t)gj * ldb + gk2] : B[(int64_t)gk2 * ldb + gj];
      Bs[r][c] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double bv = Bs[k][tx];
#pragma unroll
      for (int a = 0; a < 4; ++a) acc[a] = fma(As[ty * 4 + a][k], bv, acc[a]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int gi = i0 + ty * 4 + a, gj = j0 + tx;
    if (gi < M && gj < N) C[(int64_t)gi * ldc + gj] = acc[a];
  }
}

// Same product with the whole K extent of the 32-row A panel and the 32-column B
// panel staged in shared memory by one batch of independent loads (8 in flight per
// thread), then one barrier: the tiled loop above pays a global round trip per
// 32-deep tile, which dominated at the projected sizes (m <= 390).
__global__ void __launch_bounds__(256)
small_gemm_fk(int ta, int tb, int M, int N, int K, const double* __restrict__ A, int lda,
              const double* __restrict__ B, int ldb, double* __restrict__ C, int ldc) {
  extern __shared__ double gsm[];
  const int KP = K | 1;  // odd row stride: conflict-free column walks
  double* As = gsm;            // As[r * KP + k] = A(i0 + r, k)
  double* Bs = gsm + 32 * KP;  // Bs[c * KP + k] = B(k, j0 + c)
  const int tid = threadIdx.x;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int total = 32 * K;
  for (int e0 = tid; e0 < total; e0 += 256 * 8) {
    double va[8], vb[8];
    int ra[8], ka[8], rb[8], kb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      // element order follows the contiguous direction of each operand (coalesced)
      int r, k;
      if (ta) { k = e >> 5; r = e & 31; } else { r = e / K; k = e - r * K; }
      int c, k2;
      if (tb) { c = e / K; k2 = e - c * K; } else { k2 = e >> 5; c = e & 31; }
      ra[u] = r; ka[u] = k; rb[u] = c; kb[u] = k2;
      double a = 0.0, b = 0.0;
      if (e < total) {
        const int gi = i0 + r, gj = j0 + c;
        if (gi < M) a = ta ? A[(int64_t)k * lda + gi] : A[(int64_t)gi * lda + k];
        if (gj < N) b = tb ? B[(int64_t)gj * ldb + k2] : B[(int64_t)k2 * ldb + gj];
      }
      va[u] = a;
      vb[u] = b;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u * 256 < total) {
        As[ra[u] * KP + ka[u]] = va[u];
        Bs[rb[u] * KP + kb[u]] = vb[u];
      }
  }
  __syncthreads();
  const int tx = tid & 31, ty = tid >> 5;
  double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  const double* bp = Bs + tx * KP;
  const double* ap = As + ty * 4 * KP;
  int k = 0;
#pragma unroll 4
  for (; k + 1 < K; k += 2) {
    const double b0 = bp[k], b1 = bp[k + 1];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      acc[a][0] = fma(ap[a * KP + k], b0, acc[a][0]);
      acc[a][1] = fma(ap[a * KP + k + 1], b1, acc[a][1]);
    }
  }
  if (k < K)
#pragma unroll
    for (int a = 0; a < 4; ++a) acc[a][0] = fma(ap[a * KP + k], bp[k], acc[a][0]);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int gi = i0 + ty * 4 + a, gj = j0 + tx;
    if (gi < M && gj < N) C[(int64_t)gi * ldc + gj] = acc[a][0] + acc[a][1];
  }
}

void launch_small_gemm(int ta, int tb, int M, int N, int K, const double* A, int lda,
                       const double* B, int ldb, double* C, int ldc, cudaStream_t st) {
  dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
  const size_t smem = sizeof(double) * 64 * (size_t)(K | 1);
  if (smem <= 200 * 1024) {
    static std::atomic<uint64_t> attr{0};
    if (!done_on_device(attr)) {
      cudaFuncSetAttribute(small_gemm_fk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      mark_on_device(attr);
    }
    small_gemm_fk<<<grid, 256, smem, st>>>(ta, tb, M, N, K, A, lda, B, ldb, C, ldc);
  } else {
    small_gemm<<<grid, 256, 0, st>>>(ta, tb, M, N, K, A, lda, B, ldb, C, ldc);
  }
}

// Householder tridiagonalisation of the symmetric part of Asrc (m x m).
// V row k holds v_k (v_k[k+1] = 1, zeros before), tau[k]; d, e diagonals.
// Three CTA barriers per step: (1) warp 0 forms the reflector of row k;
// (2) p = tau W22 v with the row reductions of each warp batched, plus the
// per-warp partials of p'v; (3) the rank-2 update W22 -= v w' + w v' with
// w = p - (tau/2)(p'v) v formed on the fly.
template <int TRB>  // rows per warp per batch in the matvec (ceil(m/32) when it fits)
__global__ void __launch_bounds__(ET)
tridiag(const double* __restrict__ Asrc, int m, int symmetrize, double* __restrict__ Wg,
        double* __restrict__ V, double* __restrict__ tau, double* __restrict__ d,
        double* __restrict__ e, const SmallStatus* status) {
  extern __shared__ double smem[];
  __shared__ double sc[4];
  __shared__ double wpart[ET / 32];
  if (status && (status->nonfinite || status->not_pd)) return;
  const bool in_smem = (size_t)m * m * sizeof(double) <= 190 * 1024;
  double* W = in_smem ? smem : Wg;
  double* vb = in_smem ? smem + (size_t)m * m : Wg + (size_t)m * m;
  double* pw = vb + m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < m; i += ET / 32)
    for (int j = lane; j < m; j += 32) {
      const int x = i * m + j;
      W[x] = symmetrize ? 0.5 * (Asrc[x] + Asrc[j * m + i]) : Asrc[x];
      V[x] = 0.0;
    }
  __syncthreads();
  for (int k = 0; k + 2 < m; ++k) {
    if (warp == 0) {
      const double* rowk = W + k * m;
      double ss = 0.0;
      for (int i = k + 2 + lane; i < m; i += 32) ss += rowk[i] * rowk[i];
      ss = warp_sum(ss);
      const double alpha = rowk[k + 1];
      double tk = 0.0, scale = 0.0, beta = alpha;
      if (ss != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        tk = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      if (lane == 0) {
        d[k] = rowk[k];
        e[k] = beta;
        tau[k] = tk;
        sc[0] = tk;
      }
      for (int i = k + 1 + lane; i < m; i += 32) {
        const double v = (i == k + 1) ? 1.0 : rowk[i] * scale;
        vb[i] = v;
        V[k * m + i] = v;
      }
    }
    __syncthreads();  // (1) reflector ready
    const double tk = sc[0];
    if (tk == 0.0) continue;
    double pv = 0.0;
    const int j0 = k + 1 + lane;
    for (int i0 = k + 1 + warp; i0 < m; i0 += (ET / 32) * TRB) {
      double acc[TRB];
      const double* wr[TRB];
#pragma unroll
      for (int r = 0; r < TRB; ++r) {
        acc[r] = 0.0;
        const int i = min(i0 + r * (ET / 32), m - 1);  // clamped rows are discarded below
        wr[r] = W + i * m;
      }
      for (int j = j0; j < m; j += 32) {
        const double vj = vb[j];
#pragma unroll
        for (int r = 0; r < TRB; ++r) acc[r] = fma(wr[r][j], vj, acc[r]);
      }
#pragma unroll
      for (int r = 0; r < TRB; ++r) acc[r] = warp_sum(acc[r]);
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < TRB; ++r) {
          const int i = i0 + r * (ET / 32);
          if (i < m) {
            const double p = tk * acc[r];
            pw[i] = p;
            pv = fma(p, vb[i], pv);
          }
        }
      }
    }
    if (lane == 0) wpart[warp] = pv;
    __syncthreads();  // (2) p and the p'v partials ready
    double tot = 0.0;
#pragma unroll 8
    for (int w = 0; w < ET / 32; ++w) tot += wpart[w];
    const double K = 0.5 * tk * tot;
    for (int i = k + 1 + tid; i < m; i += ET) pw[i] = fma(-K, vb[i], pw[i]);  // w = p - K v
    __syncthreads();  // (3) w ready
    for (int i = k + 1 + warp; i < m; i += ET / 32) {
      const double vi = vb[i], wi = pw[i];
      double* row = W + i * m;
      for (int j = j0; j < m; j += 32) row[j] = fma(-vi, pw[j], fma(-wi, vb[j], row[j]));
    }
    __syncthreads();  // (4) trailing matrix updated
  }
  if (tid == 0) {
    if (m >= 2) {
      d[m - 2] = W[(m - 2) * m + (m - 2)];
      d[m - 1] = W[(m - 1) * m + (m - 1)];
      e[m - 2] = W[(m - 1) * m + (m - 2)];
      tau[m - 2] = 0.0;
    } else if (m == 1) {
      d[0] = W[0];
    }
    if (m >= 1) {
      tau[m - 1] = 0.0;
      e[m - 1] = 0.0;
    }
  }
}

// Cluster reduction (m in [kTriClusterMin, kTriClusterMax]; round 1 also had a
// cluster-barrier variant and a fused one-exchange variant, both measured slower
// and removed): the columns of the
// matrix are split over the C CTAs of one thread-block cluster and stay in their
// shared memory for the whole reduction; per step k every CTA
//   (1) forms the reflector of row k redundantly from an all-gathered copy of
//       row k (identical inputs, identical order => identical v, tau in every CTA),
//   (2) computes p_i = tau sum_j W_ji v_j for its own columns i and pushes p_i and
//       its share of p'v into every CTA's shared memory (DSMEM),
//   (3) after one cluster barrier applies W -= v w' + w v' (w = p - (tau/2)(p'v) v)
//       to its own columns and pushes its slice of row k+1 to every CTA,
// so a step costs two cluster barriers instead of one SM streaming the whole
// matrix. Exchange buffers are double-buffered by step parity.
constexpr int TCT = 512;
constexpr int kTriClusterMin = 48;
constexpr int kTriClusterMax = 560;

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

__device__ __forceinline__ void dsmem_store(double* local_addr, int rank, double v) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local_addr), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(r), "d"(v) : "memory");
}

// Same reduction with the two per-step exchanges carried by st.async stores that
// complete transactions on the receiver's mbarrier (one barrier per buffer
// parity for the p / p'v exchange and one for row k+1): a CTA waits only for the
// bytes it needs, with no release fence or cluster-wide barrier per step. WAR
// safety of the double-buffered slots follows from the data dependencies (a
// producer can only reach step k+2 after every CTA has finished step k), plus
// one CTA barrier per step before vbuf / sc are rewritten.
__device__ __forceinline__ uint32_t sm_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mb_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "MBW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra MBW_%=;\n}" ::"r"(sm_u32(bar)),
      "r"(parity)
      : "memory");
}
// Bulk copy of `bytes` (multiple of 16, 16-byte aligned) from this CTA's shared memory
// into the same offset of `local_dst` in CTA `rank`, completing on its mbarrier.
__device__ __forceinline__ void bulk_s2cluster(double* local_dst, const double* src, uint32_t bytes,
                                               uint64_t* local_bar, int rank) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(sm_u32(local_dst)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(sm_u32(local_bar)), "r"(rank));
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(ra),
      "r"(sm_u32(src)), "r"(bytes), "r"(rb)
      : "memory");
}

// mb_wait with a spin bound: a protocol error reports and traps instead of hanging the GPU.
__device__ __forceinline__ bool mb_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n}"
      : "=r"(ok)
      : "r"(sm_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __noinline__ void mb_stuck(int tag, int k) {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  printf("spb: mbarrier wait stuck (tag %d step %d cta %u warp %d)\n", tag, k, r,
         (int)(threadIdx.x >> 5));
  __trap();
}
__device__ __forceinline__ void mb_wait_bounded(uint64_t* bar, uint32_t parity, int tag, int k) {
  for (uint32_t spin = 0; !mb_try(bar, parity); ++spin)
    if (spin == (1u << 20)) mb_stuck(tag, k);
}
__device__ __forceinline__ void st_async_f64(double* local_addr, uint64_t* local_bar, int rank,
                                             double v) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(sm_u32(local_addr)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(sm_u32(local_bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(ra),
               "l"(__double_as_longlong(v)), "r"(rb)
               : "memory");
}

__global__ void __launch_bounds__(TCT)
tridiag_cluster_mb(const double* __restrict__ Asrc, int m, int symmetrize, double* __restrict__ V,
                   double* __restrict__ tau, double* __restrict__ d, double* __restrict__ e,
                   const SmallStatus* status, long long* trace) {
  if (status && (status->nonfinite || status->not_pd)) return;  // uniform over the cluster
  unsigned rank_u, csize_u;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank_u));
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(csize_u));
  const int rank = (int)rank_u, C = (int)csize_u;
  const int nc = (m + C - 1) / C;
  const int c0 = rank * nc;
  const int ncl = max(0, min(m, c0 + nc) - c0);
  extern __shared__ double tsm[];
  double* Wl = tsm;                        // m x nc, row j / local column c
  double* rowbuf = Wl + (size_t)m * nc;    // [2][m]  row k (all-gathered)
  double* pbuf = rowbuf + 2 * m;           // [2][m]  p (all-gathered)
  double* vbufs = pbuf + 2 * m;            // [2][m]  v of steps k (parity)
  double* dotbuf = vbufs + 2 * m;          // [2][16] per-CTA shares of p'v
  double* red = dotbuf + 32;               // [G][nc]
  __shared__ double wdot[4];
  __shared__ double sc[2];
  __shared__ __align__(8) uint64_t mbA[2], mbB[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = TCT / nc;
  const int nwt = ((nc + 31) >> 5) << 5;  // warps covering the local columns (nc <= 128)
  const int g = tid / nc, lc = tid - (tid / nc) * nc;
  const bool active = g < G && lc < ncl;
  const int icol = c0 + lc;
  if (tid == 0) {
    mb_init(&mbA[0], 1);
    mb_init(&mbA[1], 1);
    mb_init(&mbB[0], 1);
    mb_init(&mbB[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int x = tid; x < m * ncl; x += TCT) {
    const int j = x / ncl, c = x - (x / ncl) * ncl, i = c0 + c;
    const double a = Asrc[(int64_t)j * m + i];
    Wl[j * nc + c] = symmetrize ? 0.5 * (a + Asrc[(int64_t)i * m + j]) : a;
    V[(int64_t)j * m + i] = 0.0;
  }
  cluster_sync_all();  // barriers initialised everywhere before any remote transaction
  for (int x = tid; x < ncl * C; x += TCT) {
    const int r = x / ncl, c = x - (x / ncl) * ncl;
    st_async_f64(rowbuf + c0 + c, &mbB[0], r, Wl[c]);
  }
  // warp 0: wait for row kk, form its reflector into vbufs[kk & 1], sc[kk & 1]
  auto reflect = [&](int kk) {
    const int bb = kk & 1;
    if (lane == 0) mb_expect(&mbB[bb], 8u * (uint32_t)(m - kk));
    mb_wait(&mbB[bb], (uint32_t)((kk >> 1) & 1));
    const double* row = rowbuf + bb * m;
    double* vb = vbufs + bb * m;
    double ss = 0.0;
    for (int i = kk + 2 + lane; i < m; i += 32) ss = fma(row[i], row[i], ss);
    ss = warp_sum(ss);
    const double alpha = row[kk + 1];
    double tk = 0.0, scale = 0.0, beta = alpha;
    if (ss != 0.0) {
      beta = -copysign(sqrt(alpha * alpha + ss), alpha);
      tk = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    for (int i = kk + 1 + lane; i < m; i += 32) vb[i] = i == kk + 1 ? 1.0 : row[i] * scale;
    if (lane == 0) {
      sc[bb] = tk;
      if (rank == 0) {
        d[kk] = row[kk];
        e[kk] = beta;
        tau[kk] = tk;
      }
    }
  };
  if (warp == 0 && m > 2) reflect(0);
  uint32_t useA0 = 0, useA1 = 0;
  for (int k = 0; k + 2 < m; ++k) {
    const int b = k & 1;
    double* pb = pbuf + b * m;
    double* nextrow = rowbuf + (b ^ 1) * m;
    const double* vbuf = vbufs + b * m;
    __syncthreads();  // reflector k in vbufs[b]; every update of step k-1 is done
    const bool tr = trace && rank == C - 1 && tid == 0;  // the CTA owning the last columns
    if (tr) trace[k * 8 + 0] = clock64();
    const double tk = sc[b];
    const int j0 = k + 1 + g;
    const bool own = active && icol > k;
    if (tid < ncl && icol > k) V[(int64_t)k * m + icol] = vbuf[icol];
    if (tk != 0.0) {
      // (2) p = tau W v on own columns
      if (own) {
        double a0 = 0.0, a1 = 0.0;
        const double* wp = Wl + j0 * nc + lc;
        const double* vp = vbuf + j0;
        const int step = G * nc;
        int j = j0;
        for (; j + G < m; j += 2 * G, wp += 2 * step, vp += 2 * G) {
          a0 = fma(wp[0], vp[0], a0);
          a1 = fma(wp[step], vp[G], a1);
        }
        if (j < m) a0 = fma(wp[0], vp[0], a0);
        red[g * nc + lc] = a0 + a1;
      }
      if (tr) trace[k * 8 + 1] = clock64();
      __syncthreads();
      if (tr) trace[k * 8 + 2] = clock64();
      if (tid < nwt) {
        double pv = 0.0;
        if (tid < ncl && icol > k) {
          double sacc = 0.0;
          const int gmax = min(G, m - (k + 1));  // groups that saw a row
          for (int q = 0; q < gmax; ++q) sacc += red[q * nc + tid];
          const double p = tk * sacc;
          pv = p * vbuf[icol];
          if (tr) trace[k * 8 + 7] = clock64();
          for (int r = 0; r < C; ++r) st_async_f64(pb + icol, &mbA[b], r, p);
        }
        pv = warp_sum(pv);
        if (lane == 0) wdot[tid >> 5] = pv;
        asm volatile("bar.sync 1, %0;\n" ::"r"(nwt) : "memory");
        double wsum = wdot[0];
        for (int q = 1; q < (nwt >> 5); ++q) wsum += wdot[q];
        if (tid < C) st_async_f64(dotbuf + b * 16 + rank, &mbA[b], tid, wsum);
      }
      if (tr) trace[k * 8 + 3] = clock64();
      if (tid == 0) mb_expect(&mbA[b], 8u * (uint32_t)(m - k - 1 + C));
      {
        const uint32_t u = b ? useA1 : useA0;
        mb_wait(&mbA[b], u & 1u);
        if (b) ++useA1; else ++useA0;
      }
      if (tr) trace[k * 8 + 4] = clock64();
      // (3) rank-2 update of own columns; row k+1 first, pushed to every CTA
      if (own) {
        double tot = 0.0;
        for (int r = 0; r < C; ++r) tot += dotbuf[b * 16 + r];
        const double K = 0.5 * tk * tot;
        const double vi = vbuf[icol];
        const double wi = fma(-K, vi, pb[icol]);
        double* wp = Wl + j0 * nc + lc;
        const double* vp = vbuf + j0;
        const double* pp = pb + j0;
        const int step = G * nc;
        int j = j0;
        if (g == 0) {
          const double wj = fma(-K, vp[0], pp[0]);
          const double wv = fma(-vp[0], wi, fma(-wj, vi, wp[0]));
          wp[0] = wv;
          for (int r = 0; r < C; ++r) st_async_f64(nextrow + icol, &mbB[b ^ 1], r, wv);
          j += G, wp += step, vp += G, pp += G;
        }
#pragma unroll 2
        for (; j < m; j += G, wp += step, vp += G, pp += G) {
          const double vj = vp[0];
          const double wj = fma(-K, vj, pp[0]);
          wp[0] = fma(-vj, wi, fma(-wj, vi, wp[0]));
        }
      }
    } else if (tid < ncl && icol > k) {  // identity reflector: row k+1 is unchanged, pass it on
      const double wv = Wl[(k + 1) * nc + tid];
      for (int r = 0; r < C; ++r) st_async_f64(nextrow + icol, &mbB[b ^ 1], r, wv);
    }
    if (tr) trace[k * 8 + 5] = clock64();
    // warp 0 forms the next reflector while the other warps finish their updates
    if (warp == 0 && k + 3 < m) reflect(k + 1);
    if (tr) trace[k * 8 + 6] = clock64();
  }
  if (m >= 2) {
    const int kk = m - 2;  // row m-2 was pushed at step m-3 (or at init when m == 2)
    __syncthreads();
    if (warp == 0) {
      if (lane == 0) mb_expect(&mbB[kk & 1], 8u * (uint32_t)(m - kk));
      mb_wait(&mbB[kk & 1], (uint32_t)((kk >> 1) & 1));
      const double* row = rowbuf + (kk & 1) * m;
      if (rank == 0 && lane == 0) {
        d[m - 2] = row[m - 2];
        e[m - 2] = row[m - 1];
        tau[m - 2] = 0.0;
        tau[m - 1] = 0.0;
        e[m - 1] = 0.0;
      }
    }
    if (tid == 0 && m - 1 >= c0 && m - 1 < c0 + ncl) d[m - 1] = Wl[(m - 1) * nc + (m - 1 - c0)];
  }
  cluster_sync_all();  // no CTA leaves while its shared memory can still be written
}

// Cholesky + inverse for kCholLdlMax < m <= kCholClusterMax: the packed
// array of chol_ldl (L' in the lower triangle, the unit-lower inverse
// transposed in the upper one) is split by columns over the CTAs of a cluster.
// Iteration c needs only packed column c (L' column c below the diagonal, row c
// of L'^-1 above it, d_c on it): its owner pushes it to every CTA while
// finishing iteration c-1, so a column costs one cluster barrier. The cond
// bracket / CholQR tests run afterwards in chol_finish.
constexpr int CCT = 512;
constexpr int kCholClusterMax = 560;

__global__ void __launch_bounds__(CCT)
chol_cluster(const double* __restrict__ Bsrc, int m, double* __restrict__ Lg,
             double* __restrict__ Linv, int mode, SmallStatus* status) {
  if (status->nonfinite) return;  // uniform over the cluster
  unsigned rank_u, csize_u;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank_u));
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(csize_u));
  const int rank = (int)rank_u, C = (int)csize_u;
  const int nc = (m + C - 1) / C;
  const int c0 = rank * nc;
  const int ncl = max(0, min(m, c0 + nc) - c0);
  extern __shared__ double csm[];
  double* P = csm;                    // m x nc packed columns
  double* colbuf = P + (size_t)m * nc;  // [2][m] broadcast column
  __shared__ int s_fail;
  const int tid = threadIdx.x;
  const int G = CCT / nc;
  const int g = tid / nc, lc = tid - (tid / nc) * nc;
  const bool active = g < G && lc < ncl;
  const int q = c0 + lc;
  if (tid < 32) {
    int f0 = 0;
    if (mode == 1) {  // diag > 0 and min diag > (eps na)^2 max diag (lobpcg.py:229-231)
      double dmin, dmax;
      warp_minmax(Bsrc, (int64_t)m + 1, m, false, &dmin, &dmax);
      if (rank == 0 && tid == 0) {
        status->dmin = dmin;
        status->dmax = dmax;
      }
      const double t = kEps64 * m;
      if (!(dmin > 0.0) || !(dmin > t * t * dmax)) f0 = 1;
    }
    if (tid == 0) s_fail = f0;
  }
  for (int x = tid; x < m * ncl; x += CCT) {
    const int i = x / ncl, c = x - (x / ncl) * ncl;
    P[i * nc + c] = i >= c0 + c ? Bsrc[(int64_t)i * m + c0 + c] : 0.0;
  }
  __syncthreads();
  if (s_fail) {
    if (rank == 0 && tid == 0) status->fallback = 1;
    return;
  }
  if (c0 == 0 && ncl > 0)
    for (int i = tid; i < m; i += CCT) {
      const double v = P[i * nc];
      for (int r = 0; r < C; ++r) dsmem_store(colbuf + i, r, v);
    }
  cluster_sync_all();
  int fail = 0;
  for (int c = 0; c < m; ++c) {
    const double* col = colbuf + (c & 1) * m;
    double* nxt = colbuf + ((c + 1) & 1) * m;
    const double dc = col[c];
    if (!(dc > 0.0)) {
      fail = 1;
      break;
    }
    if (active && q > c) {
      const double rc = 1.0 / dc;
      const double lqc = col[q] * rc;  // L'[q][c]
      double* Pq = P + lc;
      for (int i = q + g; i < m; i += G)  // factor: A[i][q] -= A[i][c] L'[q][c]
        Pq[i * nc] = fma(-col[i], lqc, Pq[i * nc]);
      for (int j = g; j < c; j += G)  // inverse: L'^-1[q][j] -= L'[q][c] L'^-1[c][j]
        Pq[j * nc] = fma(-lqc, col[j], Pq[j * nc]);
      if (g == 0) Pq[c * nc] = -lqc;
    }
    const int cn = c + 1;
    if (cn < m && cn >= c0 && cn < c0 + ncl) {  // owner of the next column: push it
      __syncthreads();
      const double* Pn = P + (cn - c0);
      for (int x = tid; x < m * C; x += CCT) {
        const int r = x / m, i = x - (x / m) * m;
        dsmem_store(nxt + i, r, Pn[i * nc]);
      }
    }
    cluster_sync_all();
  }
  if (fail) {
    if (rank == 0 && tid == 0) {
      if (mode == 0) status->not_pd = 1;
      else status->fallback = 1;
    }
    return;
  }
  // L = L' D^1/2 (own columns), L^-1 = D^-1/2 L'^-1 (own rows)
  for (int x = tid; x < m * ncl; x += CCT) {
    const int c = x / m, i = x - (x / m) * m;
    const int qq = c0 + c;
    const double dq = P[qq * nc + c];
    const double rs = 1.0 / sqrt(dq);
    double l = 0.0, v = 0.0;
    if (i > qq) l = P[i * nc + c] * rs;
    else if (i == qq) l = sqrt(dq);
    if (i < qq) v = P[i * nc + c] * rs;
    else if (i == qq) v = rs;
    Lg[(int64_t)i * m + qq] = l;
    Linv[(int64_t)qq * m + i] = v;
  }
}

// Frobenius norms, cond bracket / CholQR diagonal test and Rinv layout after chol_cluster.
__global__ void __launch_bounds__(ET)
chol_finish(const double* __restrict__ Bsrc, int m, const double* __restrict__ Lg,
            double* __restrict__ Linv, int mode, SmallStatus* status) {
  __shared__ double red[33];
  __shared__ int fail;
  if (status->nonfinite || status->not_pd || status->fallback) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double fb = 0.0;
  for (int i = warp; i < m; i += ET / 32)
    for (int j = lane; j < m; j += 32) {
      const double v = Bsrc[(int64_t)i * m + j];
      fb += v * v;
    }
  fb = block_sum(fb, red);
  if (warp == 0) {
    int f0 = 0;
    if (mode == 1) {
      double rmin, rmax;
      warp_minmax(Lg, (int64_t)m + 1, m, false, &rmin, &rmax);
      if (lane == 0) {
        status->rmin = rmin;
        status->rmax = rmax;
      }
      if (!(rmin > sqrt(kEps64) * rmax)) f0 = 1;  // lobpcg.py:235
    }
    if (lane == 0) fail = f0;
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) status->fallback = 1;
    return;
  }
  chol_epilogue(m, fb, Linv, mode, status, red);
}

// Lane-group-per-column tridiagonalisation (default for kTriClusterMin <= m <= 320).
// The columns are split over a cluster of C CTAs; a group of LPC lanes owns one
// column i and keeps ALL its rows in registers (lane g of the group holds rows
// g + LPC t), so the matvec p_i = tau W(:,i)'v and the rank-2 update of column i
// are register FMAs plus an LPC-lane reduction -- no shared-memory sweep of the
// matrix and no CTA barrier per step. Per step k every participating group
//   (1) waits for row k (all-gathered by st.async into every consumer CTA), completes
//       it with the previous step's 2K v v' term (its own v_j), and forms reflector k
//       redundantly (same inputs and order => the same v, tau everywhere) together with
//       p_i = ((beta - alpha) W_{k+1,i} - sum_{j>k+1} W_ji x_j) / beta: one rsqrt on
//       the path from the row's arrival to the push of p_i,
//   (2) pushes p_i into every consumer CTA's p buffer,
//   (3) waits for p_k, applies W -= v p' + p v' to column i, pushes its element of
//       row k+1 (without the 2K v v' term, which every receiver adds itself) and then
//       applies the 2K v v' term (K = tau/2 p'v) to its column.
// A column leaves after step i-1. A controller warp per CTA arms the expected byte
// counts of the double-buffered row / p mbarriers. WAR safety of the parity buffers
// follows from the data dependencies: data of step k+2 can only be produced after
// every consumer finished reading step k's buffers (its contribution to row k+1 or
// p_{k+1} is issued after those reads).
constexpr int kWcWarps = 19;  // column warps per CTA (upper bound; + 1 controller warp)
constexpr int kWcThreads = 32 * (kWcWarps + 1);

template <int R, int LPC, bool BULK>
__global__ void __launch_bounds__(kWcThreads)
tridiag_warpcol(const double* __restrict__ Asrc, int m, int symmetrize, double* __restrict__ V,
                double* __restrict__ tau, double* __restrict__ d, double* __restrict__ e,
                const SmallStatus* status, long long* trace) {
  if (status && (status->nonfinite || status->not_pd)) return;  // uniform over the cluster
  constexpr int G = 32 / LPC;  // columns per warp
  unsigned rank_u, csize_u;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank_u));
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(csize_u));
  const int rank = (int)rank_u, C = (int)csize_u;
  // BULK: each exchange is gathered in a local stage and sent as one bulk copy per
  // consumer CTA (16-byte aligned chunks: nc even) instead of one st.async per value
  const int nc = BULK ? (((m + C - 1) / C + 1) & ~1) : (m + C - 1) / C;
  const int Mp = BULK ? C * nc : m;          // exchange buffer stride
  const int nne = (m + nc - 1) / nc;         // CTAs holding columns
  const int c0 = rank * nc;
  const int ncl = max(0, min(m, c0 + nc) - c0);
  const int cmax = ncl > 0 ? c0 + ncl - 1 : -1;  // last column held by this CTA (-1: none)
  const int nw = (nc + G - 1) / G;                 // column warps per CTA
  extern __shared__ __align__(16) double wsm[];
  double* rowb = wsm;           // [2][Mp] rows k (parity k & 1), entries k..m-1
  double* pbuf = wsm + 2 * Mp;  // [2][Mp] p_k, entries k+1..m-1
  double* stR = wsm + 4 * Mp;   // BULK: [2][nc] local slice of the next row
  double* stP = stR + 2 * nc;   // BULK: [2][nc] local slice of p
  __shared__ __align__(8) uint64_t mbR[2], mbP[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gl = lane % LPC, q = lane / LPC, gb = q * LPC;  // lane in group, group, base lane
  const unsigned full = 0xffffffffu;
  // last column of CTA r: consumers of step-k data are the CTAs with a column > k
#define cmax_of(r) ((r) * nc < m ? min(m, ((r) + 1) * nc) - 1 : -1)
  // bytes of row r / p_k landing in a consumer (BULK: whole slices of the senders)
#define RBYTES(r) (BULK ? 8u * (uint32_t)(nc * (nne - (r) / nc)) : 8u * (uint32_t)(m - (r)))
#define PBYTES(k) (BULK ? 8u * (uint32_t)(nc * (nne - ((k) + 1) / nc)) : 8u * (uint32_t)(m - (k) - 1))
  if (threadIdx.x == 0) {
    mb_init(&mbR[0], 1);
    mb_init(&mbR[1], 1);
    mb_init(&mbP[0], 1);
    mb_init(&mbP[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();
  if (warp == nw) {
    // controller: arm row r (8(m-r) bytes) and p_k (8(m-k-1) bytes) phases in order
    if (lane == 0 && cmax >= 0) {
      if (cmax > 0) mb_expect(&mbR[0], RBYTES(0));
      if (cmax > 1) mb_expect(&mbR[1], RBYTES(1));
      if (cmax > 0) mb_expect(&mbP[0], PBYTES(0));
      if (cmax > 1 && m >= 4) mb_expect(&mbP[1], PBYTES(1));
      for (int k = 0; k + 2 < m && cmax > k; ++k) {
        const int b = k & 1;
        const uint32_t par = (uint32_t)((k >> 1) & 1);
        mb_wait_bounded(&mbR[b], par, 1, k);
        if (k + 2 <= m - 2 && cmax > k + 2) mb_expect(&mbR[b], RBYTES(k + 2));
        mb_wait_bounded(&mbP[b], par, 2, k);
        if (k + 2 <= m - 3 && cmax > k + 2) mb_expect(&mbP[b], PBYTES(k + 2));
      }
    }
  } else if (warp < nw) {
    const int lc = warp * G + q;  // local column of this lane group
    const bool valid = lc < ncl;
    const int i = c0 + lc;
    const int kend = valid ? min(i - 1, m - 3) : -1;  // last step this column takes part in
    // the warp runs until its last valid column is done (shuffles need every lane)
    const int lcw = min(warp * G + G, ncl) - 1;
    const int kwarp = warp * G < ncl ? min(c0 + lcw - 1, m - 3) : -1;
    double w[R];  // column i, rows gl + LPC t
    double v[R];  // reflector of the previous step on the same rows (0 before step 0)
    double Kp = 0.0;  // K of the previous step
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int j = gl + LPC * t;
      double a = 0.0;
      if (valid && j < m) {
        a = Asrc[(int64_t)j * m + i];
        if (symmetrize) a = 0.5 * (a + Asrc[(int64_t)i * m + j]);
      }
      w[t] = a;
      v[t] = 0.0;
    }
    if (valid) {
      for (int k = max(kend + 1, 0) + gl; k < m; k += LPC) V[(int64_t)k * m + i] = 0.0;
      const double r0 = __shfl_sync(full, w[0], gb);
      if (BULK) {
        if (lane == 0) stR[lc] = r0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"r"(32 * ncl) : "memory");
        if (lc == ncl - 1 && lane < C && cmax_of(lane) > 0)
          bulk_s2cluster(rowb + c0, stR, 8u * nc, &mbR[0], lane);
      } else {
        for (int r = gl; r < C; r += LPC)
          if (cmax_of(r) > 0) st_async_f64(rowb + i, &mbR[0], r, r0);
      }
    } else {
      __shfl_sync(full, 0.0, gb);
    }
    const bool tr = trace && i == m - 1 && gl == 0;
#define SPB_TS(qq) \
  if (tr) trace[k * 8 + (qq)] = clock64();
    for (int k = 0; k <= kwarp; ++k) {
      const bool act = k <= kend;
      const int b = k & 1;
      const uint32_t par = (uint32_t)((k >> 1) & 1);
      SPB_TS(0)
      mb_wait_bounded(&mbR[b], par, 3, k);
      SPB_TS(1)
      const double* row = rowb + b * Mp;
      const double twoK = 2.0 * Kp;
      double ss = 0.0, s2 = 0.0, cal = 0.0, s1 = 0.0, cii = 0.0;
      // BULK: column warps still in the loop at step k (columns > k), the last one sends
      const int nact = ncl - max(0, min(ncl, k + 1 - c0));
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = gl + LPC * t;
        const double c = (j >= k && j < m) ? fma(twoK, v[t], row[j]) : 0.0;
        if (j == k + 1) {
          cal = c;
          s1 = w[t];
        }
        if (j == i) cii = c;
        if (j == k && i == k + 1) d[k] = c;
        const double x = j >= k + 2 ? c : 0.0;
        v[t] = x;
        ss = fma(x, x, ss);
        s2 = fma(w[t], x, s2);
      }
#pragma unroll
      for (int o = LPC / 2; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(full, ss, o);
        s2 += __shfl_xor_sync(full, s2, o);
      }
      const double alpha = __shfl_sync(full, cal, gb + (k + 1) % LPC);
      s1 = __shfl_sync(full, s1, gb + (k + 1) % LPC);
      cii = __shfl_sync(full, cii, gb + (valid ? i % LPC : 0));
      SPB_TS(5)
      double beta = alpha, rbeta = 0.0, pi = 0.0;
      if (ss != 0.0) {
        const double a2 = fma(alpha, alpha, ss);
        const double r = rsqrt(a2);
        beta = -copysign(a2 * r, alpha);
        rbeta = -copysign(r, alpha);  // 1 / beta
        pi = fma(beta - alpha, s1, -s2) * rbeta;
      }
      SPB_TS(6)
      if (BULK) {
        if (lane == 0) stP[b * nc + lc] = pi;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(32 * nact) : "memory");
        if (lc == ncl - 1 && lane < C && cmax_of(lane) > k)
          bulk_s2cluster(pbuf + b * Mp + c0, stP + b * nc, 8u * nc, &mbP[b], lane);
      } else if (act) {
        for (int r = gl; r < C; r += LPC)
          if (cmax_of(r) > k) st_async_f64(pbuf + b * m + i, &mbP[b], r, pi);
      }
      SPB_TS(2)
      double tk = 0.0, scale = 0.0;
      if (ss != 0.0) {
        tk = (beta - alpha) * rbeta;
        scale = 1.0 / (alpha - beta);
      }
      const double vi = i == k + 1 ? 1.0 : cii * scale;
      if (act && gl == 0) {
        V[(int64_t)k * m + i] = vi;
        if (i == k + 1) {
          e[k] = beta;
          tau[k] = tk;
        }
      }
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = gl + LPC * t;
        v[t] = j == k + 1 ? 1.0 : v[t] * scale;
      }
      mb_wait_bounded(&mbP[b], par, 4, k);
      SPB_TS(3)
      const double* pb = pbuf + b * Mp;
      double nxt = 0.0, dot = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = gl + LPC * t;
        if (j > k && j < m) {
          const double pj = pb[j];
          w[t] = fma(-v[t], pi, fma(-pj, vi, w[t]));
          dot = fma(pj, v[t], dot);
        }
        if (j == k + 1) nxt = w[t];
      }
      nxt = __shfl_sync(full, nxt, gb + (k + 1) % LPC);
      const int b1 = (k + 1) & 1;
      if (BULK) {
        if (lane == 0) stR[b1 * nc + lc] = nxt;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"r"(32 * nact) : "memory");
        if (lc == ncl - 1 && lane < C && cmax_of(lane) > k + 1)
          bulk_s2cluster(rowb + b1 * Mp + c0, stR + b1 * nc, 8u * nc, &mbR[b1], lane);
      } else if (act) {
        for (int r = gl; r < C; r += LPC)
          if (cmax_of(r) > k + 1) st_async_f64(rowb + b1 * m + i, &mbR[b1], r, nxt);
      }
      SPB_TS(4)
#pragma unroll
      for (int o = LPC / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(full, dot, o);
      Kp = 0.5 * tk * dot;
      const double kv = 2.0 * Kp * vi;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = gl + LPC * t;
        if (j > k && j < m) w[t] = fma(kv, v[t], w[t]);
      }
    }
    if (warp * G < ncl && c0 + lcw == m - 1) {
      // rows m-2, m-1 need no reflector: d, e from row m-2 (completed) and the last diagonal
      const int kk = m - 2;
      mb_wait_bounded(&mbR[kk & 1], (uint32_t)((kk >> 1) & 1), 5, kk);
      if (i == m - 1) {
        const double* row = rowb + (kk & 1) * Mp;
        const double twoK = 2.0 * Kp;
#pragma unroll
        for (int t = 0; t < R; ++t) {
          const int j = gl + LPC * t;
          if (j == m - 2) d[m - 2] = fma(twoK, v[t], row[j]);
          if (j == m - 1) {
            e[m - 2] = fma(twoK, v[t], row[j]);
            d[m - 1] = w[t];
          }
        }
        if (gl == 0) {
          tau[m - 2] = 0.0;
          tau[m - 1] = 0.0;
          e[m - 1] = 0.0;
        }
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
#undef SPB_TS
#undef cmax_of
#undef RBYTES
#undef PBYTES
}

struct WcShape {
  int C, lpc;
};

WcShape tridiag_warpcol_shape(int m) {
  // one warp per column (lane groups of 8 / 16 per column were measured slower: the
  // per-lane row loops become issue-bound); the widest cluster, so each SM runs as
  // few column warps as possible (2 / 4 / 8 CTAs measured slower)
  if (m < kTriClusterMin || m > 256) return {0, 0};
  constexpr int C = 16;
  if ((m + C - 1) / C > kWcWarps) return {0, 0};
  return {C, 32};
}

bool launch_tridiag_warpcol(const double* Asrc, int m, int symmetrize, double* V, double* tau,
                            double* d, double* e, const SmallStatus* status, cudaStream_t st,
                            long long* trace) {
  const WcShape sh = tridiag_warpcol_shape(m);
  if (!sh.C) return false;
  const int C = sh.C, lpc = sh.lpc;
  // (slices gathered per CTA and sent by bulk copies measured slower: the two named
  // barriers per step cost more than the per-value st.async they replace)
  constexpr bool bulk = false;
  const int nc = bulk ? (((m + C - 1) / C + 1) & ~1) : (m + C - 1) / C;
  if (nc > kWcWarps) return false;
  const int nw = (nc + 32 / lpc - 1) / (32 / lpc);
  const int Mp = bulk ? C * nc : m;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(32 * (nw + 1));
  cfg.dynamicSmemBytes = sizeof(double) * (4 * (size_t)Mp + 4 * (size_t)nc);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int R = (m + lpc - 1) / lpc;
#define SPB_WC1(RR, LL, BB)                                                                    \
  {                                                                                            \
    static std::atomic<uint64_t> attr{0}; \
    if (!done_on_device(attr)) {                                                                               \
      cudaFuncSetAttribute(tridiag_warpcol<RR, LL, BB>,                                        \
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);                 \
      mark_on_device(attr);                                                                             \
    }                                                                                          \
    cudaLaunchKernelEx(&cfg, tridiag_warpcol<RR, LL, BB>, Asrc, m, symmetrize, V, tau, d, e,   \
                       status, trace);                                                         \
    return true;                                                                               \
  }
#define SPB_WC(RR, LL) \
  {                    \
    if (bulk)          \
      SPB_WC1(RR, LL, true) \
    else               \
      SPB_WC1(RR, LL, false) \
  }
  if (R <= 2) SPB_WC(2, 32)
  if (R <= 3) SPB_WC(3, 32)
  if (R <= 4) SPB_WC(4, 32)
  if (R <= 5) SPB_WC(5, 32)
  if (R <= 6) SPB_WC(6, 32)
  if (R <= 8) SPB_WC(8, 32)
#undef SPB_WC
#undef SPB_WC1
  return false;
}

// Row-per-warp Cholesky (default for kCholRwMin <= m <= 16 * kCrWarps): the rows of
// B are split over a 16-CTA cluster, warp w of CTA r owns row i = r*nc + w and keeps
// it in registers (lane L holds columns L + 32t). Step k needs column k of the
// current Schur complement, whose entry j is owned by row j: every row pushes that one
// value (st.async into each consumer CTA) as soon as its own update of step k-1 has
// produced it, so a step costs one DSMEM exchange and no CTA barrier:
//   a_ij -= (a_ik / a_kk) a_jk   (k < j <= i),
// row k's pivot d_k = a_kk arriving with the column; L_ik = a_ik / sqrt(d_k).
// A controller warp per CTA arms the expected bytes of the double-buffered column
// mbarriers and stops with the rows when a pivot is not positive. The inverse is
// formed afterwards by trinv_cols; chol_finish adds the norms / tests as for chol_cluster.
constexpr int kCrWarps = 24;
constexpr int kCrThreads = 32 * (kCrWarps + 1);
constexpr int kCholRwMin = 165;  // below: chol_wsync (single CTA) measured faster

template <int R>
__global__ void __launch_bounds__(kCrThreads)
chol_rowwarp(const double* __restrict__ Bsrc, int m, double* __restrict__ Lg, int mode,
             SmallStatus* status) {
  if (status->nonfinite) return;  // uniform over the cluster
  unsigned rank_u, csize_u;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank_u));
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(csize_u));
  const int rank = (int)rank_u, C = (int)csize_u;
  const int nc = (m + C - 1) / C;
  const int c0 = rank * nc;
  const int ncl = max(0, min(m, c0 + nc) - c0);
  const int cmax = ncl > 0 ? c0 + ncl - 1 : -1;
  extern __shared__ __align__(16) double crs[];
  double* colb = crs;  // [2][m] column k (parity k & 1), entries k..m-1
  __shared__ __align__(8) uint64_t mbC[2];
  __shared__ int s_fail;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
#define cmax_of(r) ((r) * nc < m ? min(m, ((r) + 1) * nc) - 1 : -1)
  if (warp == 0) {
    int f0 = 0;
    if (mode == 1) {  // diag > 0 and min diag > (eps na)^2 max diag (lobpcg.py:229-231)
      double dmin, dmax;
      warp_minmax(Bsrc, (int64_t)m + 1, m, false, &dmin, &dmax);
      if (rank == 0 && lane == 0) {
        status->dmin = dmin;
        status->dmax = dmax;
      }
      const double t = kEps64 * m;
      if (!(dmin > 0.0) || !(dmin > t * t * dmax)) f0 = 1;
    }
    if (lane == 0) {
      s_fail = f0;
      mb_init(&mbC[0], 1);
      mb_init(&mbC[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  if (s_fail) {  // the same test in every CTA: uniform
    if (rank == 0 && threadIdx.x == 0) status->fallback = 1;
    return;
  }
  cluster_sync_all();
  const int nw = nc;
  if (warp == nw) {
    // controller: arm column k (8 (m-k) bytes) for consumers (rows > k); stop on a bad pivot
    if (lane == 0 && cmax >= 0) {
      if (cmax > 0) mb_expect(&mbC[0], 8u * (uint32_t)m);
      if (cmax > 1) mb_expect(&mbC[1], 8u * (uint32_t)(m - 1));
      for (int k = 0; k < m - 1 && cmax > k; ++k) {
        const int b = k & 1;
        mb_wait_bounded(&mbC[b], (uint32_t)((k >> 1) & 1), 11, k);
        if (!(colb[b * m + k] > 0.0)) break;
        if (k + 2 <= m - 1 && cmax > k + 2) mb_expect(&mbC[b], 8u * (uint32_t)(m - k - 2));
      }
    }
  } else if (warp < ncl) {
    const int i = c0 + warp;
    double w[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int j = lane + 32 * t;
      w[t] = j <= i && j < m ? Bsrc[(int64_t)i * m + j] : 0.0;
    }
    // upper triangle of L row i
    for (int j = i + 1 + lane; j < m; j += 32) Lg[(int64_t)i * m + j] = 0.0;
    {
      const double a0 = __shfl_sync(full, w[0], 0);
      if (lane < C && cmax_of(lane) > 0) st_async_f64(colb + i, &mbC[0], lane, a0);
    }
    bool ok = true;
    for (int k = 0; k < i; ++k) {
      const int b = k & 1;
      mb_wait_bounded(&mbC[b], (uint32_t)((k >> 1) & 1), 12, k);
      const double* col = colb + b * m;
      const double dk = col[k];
      if (!(dk > 0.0)) {
        ok = false;
        break;
      }
      double aik = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t)
        if (lane + 32 * t == k) aik = w[t];
      aik = __shfl_sync(full, aik, k & 31);
      const double rs = rsqrt(dk);
      if (lane == 0) Lg[(int64_t)i * m + k] = aik * rs;  // L_ik
      const double f = aik / dk;
      // the entry of column k+1 first, pushed at once; then the rest of the row
      double nxt = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = lane + 32 * t;
        if (j == k + 1) {
          w[t] = fma(-f, col[j], w[t]);
          nxt = w[t];
        }
      }
      nxt = __shfl_sync(full, nxt, (k + 1) & 31);
      const int b1 = (k + 1) & 1;
      if (lane < C && cmax_of(lane) > k + 1) st_async_f64(colb + b1 * m + i, &mbC[b1], lane, nxt);
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = lane + 32 * t;
        if (j > k + 1 && j <= i) w[t] = fma(-f, col[j], w[t]);
      }
    }
    if (ok) {
      // own pivot: d_i = a_ii after step i-1
      double dii = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t)
        if (lane + 32 * t == i) dii = w[t];
      dii = __shfl_sync(full, dii, i & 31);
      if (lane == 0) {
        if (dii > 0.0) {
          Lg[(int64_t)i * m + i] = sqrt(dii);
        } else {
          if (mode == 0) status->not_pd = 1;
          else status->fallback = 1;
        }
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
#undef cmax_of
}

// L^-1 (row-major, lower) from L (row-major): one warp per column c solves L z = e_c
// right-looking (z_k = r_k / L_kk, r_j -= L_jk z_k), the lane holding rows
// L + 32t; columns of L are staged in shared memory 32 at a time.
template <int R>
__global__ void __launch_bounds__(512)
trinv_cols(const double* __restrict__ Lg, int m, double* __restrict__ Linv,
           const SmallStatus* status) {
  if (status->nonfinite || status->not_pd || status->fallback) return;
  extern __shared__ __align__(16) double tis[];
  double* rd = tis;           // [m] 1 / L_kk
  double* Ls = tis + m;       // [32][m] columns k0..k0+31 of L (column-major)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int c = blockIdx.x * nwarp + warp;  // column of L^-1 this warp forms
  const int cfirst = blockIdx.x * nwarp;
  for (int k = threadIdx.x; k < m; k += blockDim.x) rd[k] = 1.0 / Lg[(int64_t)k * m + k];
  double r[R];
#pragma unroll
  for (int t = 0; t < R; ++t) r[t] = lane + 32 * t == c ? 1.0 : 0.0;
  if (c < m)
    for (int k = lane; k < c; k += 32) Linv[(int64_t)k * m + c] = 0.0;
  for (int k0 = (cfirst / 32) * 32; k0 < m; k0 += 32) {
    const int kn = min(32, m - k0);
    __syncthreads();  // previous chunk consumed (and rd written)
    for (int x = threadIdx.x; x < m * kn; x += blockDim.x) {
      const int j = x / kn, q = x - (x / kn) * kn;  // row j, column k0 + q (coalesced rows)
      Ls[q * m + j] = Lg[(int64_t)j * m + k0 + q];
    }
    __syncthreads();
    if (c < m)
      for (int q = 0; q < kn; ++q) {
        const int k = k0 + q;
        if (k < c) continue;
        double rk = 0.0;
#pragma unroll
        for (int t = 0; t < R; ++t)
          if (lane + 32 * t == k) rk = r[t];
        const double zk = __shfl_sync(0xffffffffu, rk, k & 31) * rd[k];
        if (lane == 0) Linv[(int64_t)k * m + c] = zk;
        const double* lc = Ls + q * m;
#pragma unroll
        for (int t = 0; t < R; ++t) {
          const int j = lane + 32 * t;
          if (j > k && j < m) r[t] = fma(-lc[j], zk, r[t]);
        }
      }
  }
}

bool launch_chol_rowwarp(const double* B, int m, double* L, double* Linv, int mode,
                         SmallStatus* status, cudaStream_t st) {
  if (m < kCholRwMin) return false;
  const int C = 16, nc = (m + C - 1) / C;
  const int R = (m + 31) / 32;
  if (nc > kCrWarps || R > 12) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(32 * (nc + 1));
  cfg.dynamicSmemBytes = sizeof(double) * 2 * (size_t)m;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const size_t ti_smem = sizeof(double) * 33 * (size_t)m;
  const int ti_warps = 16;
  const dim3 ti_grid((unsigned)((m + ti_warps - 1) / ti_warps));
#define SPB_CR(RR)                                                                               \
  {                                                                                              \
    static std::atomic<uint64_t> attr{0}; \
    if (!done_on_device(attr)) {                                                                                 \
      cudaFuncSetAttribute(chol_rowwarp<RR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
      cudaFuncSetAttribute(trinv_cols<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                           200 * 1024);                                                          \
      mark_on_device(attr);                                                                               \
    }                                                                                            \
    cudaLaunchKernelEx(&cfg, chol_rowwarp<RR>, B, m, L, mode, status);                          \
    trinv_cols<RR><<<ti_grid, 32 * ti_warps, ti_smem, st>>>(L, m, Linv, status);               \
    chol_finish<<<1, ET, 0, st>>>(B, m, L, Linv, mode, status);                                 \
    return true;                                                                                 \
  }
  if (R <= 2) SPB_CR(2)
  if (R <= 4) SPB_CR(4)
  if (R <= 6) SPB_CR(6)
  if (R <= 8) SPB_CR(8)
  if (R <= 12) SPB_CR(12)
#undef SPB_CR
  return false;
}

size_t chol_cluster_smem(int m, int C) {
  const int nc = (m + C - 1) / C;
  return sizeof(double) * ((size_t)m * nc + 2 * (size_t)m);
}

size_t tridiag_cluster_smem(int m, int C);

int tridiag_cluster_size(int m) {
  if (m < kTriClusterMin || m > kTriClusterMax) return 0;
  // 16 CTAs above m = 160 (m = 324: 1.08 -> 0.99 ms per reduction against 8, 1.02 with 12)
  return m <= 160 ? 4 : 16;
}

size_t tridiag_cluster_smem(int m, int C) {
  const int nc = (m + C - 1) / C;
  return sizeof(double) * ((size_t)m * nc + 7 * (size_t)m + 32 + (size_t)(TCT / nc) * nc);
}

void launch_tridiag(const double* Asrc, int m, int symmetrize, double* Wg, double* V, double* tau,
                    double* d, double* e, const SmallStatus* status, size_t smem, cudaStream_t st) {
  if (const int C = tridiag_cluster_size(m)) {
    static std::atomic<uint64_t> attr{0};
    if (!done_on_device(attr)) {
      cudaFuncSetAttribute(tridiag_cluster_mb, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(tridiag_cluster_mb, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      mark_on_device(attr);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(TCT);
    cfg.dynamicSmemBytes = tridiag_cluster_smem(m, C);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // warp-per-column register kernel for 48 <= m <= 256, else the shared-memory
    // column split with mbarrier-tracked exchanges
    if (launch_tridiag_warpcol(Asrc, m, symmetrize, V, tau, d, e, status, st, nullptr)) return;
    cudaLaunchKernelEx(&cfg, tridiag_cluster_mb, Asrc, m, symmetrize, V, tau, d, e, status,
                       (long long*)nullptr);
    return;
  }
  const int rows = (m + 31) / 32;
  if (rows <= 1)
    tridiag<1><<<1, ET, smem, st>>>(Asrc, m, symmetrize, Wg, V, tau, d, e, status);
  else if (rows <= 2)
    tridiag<2><<<1, ET, smem, st>>>(Asrc, m, symmetrize, Wg, V, tau, d, e, status);
  else if (rows <= 3)
    tridiag<3><<<1, ET, smem, st>>>(Asrc, m, symmetrize, Wg, V, tau, d, e, status);
  else if (rows <= 4)
    tridiag<4><<<1, ET, smem, st>>>(Asrc, m, symmetrize, Wg, V, tau, d, e, status);
  else if (rows <= 5)
    tridiag<5><<<1, ET, smem, st>>>(Asrc, m, symmetrize, Wg, V, tau, d, e, status);
  else
    tridiag<8><<<1, ET, smem, st>>>(Asrc, m, symmetrize, Wg, V, tau, d, e, status);
}

// One warp per eigenvalue index (first + t): 33-section of the Gershgorin interval.
// d and e^2 are staged in shared memory once per CTA (dynamic, 2m doubles); the
// Sturm count is the LDL' pivot recurrence of dstebz.
__global__ void bisect(const double* __restrict__ d, const double* __restrict__ e, int m,
                       int first, int count, double* __restrict__ theta, double* __restrict__ e2unused,
                       const SmallStatus* status, int use_div) {
  extern __shared__ double bsd[];  // d[m], e2[m]
  if (status && (status->nonfinite || status->not_pd)) return;
  double* sd = bsd;
  double* se2 = bsd + m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    sd[i] = d[i];
    se2[i] = i + 1 < m ? e[i] * e[i] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= count) return;
  const int idx = first + t;
  double lo = DBL_MAX, hi = -DBL_MAX, emax = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < m ? fabs(e[i]) : 0.0);
    lo = fmin(lo, sd[i] - r);
    hi = fmax(hi, sd[i] + r);
    if (i + 1 < m) emax = fmax(emax, se2[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  const double pivmin = DBL_MIN * fmax(1.0, emax);
  const double tnorm = fmax(fabs(lo), fabs(hi));
  lo -= 2.0 * kEps64 * tnorm + 2.0 * pivmin;
  hi += 2.0 * kEps64 * tnorm + 2.0 * pivmin;
  double a = lo, b = hi;
  for (int round = 0; round < 64; ++round) {
    const double w = b - a;
    const double tol = fmax(2.0 * kEps64 * fmax(fabs(a), fabs(b)), kEps64 * tnorm) + pivmin;
    if (w <= tol) break;
    const double x = a + w * (double)(lane + 1) / 33.0;
    int c;
    if (use_div == 2) {
      // division-free three-term Sturm sequence p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}
      // with exact power-of-two rescaling; a pivot p_i / p_{i-1} below pivmin in
      // magnitude is taken as -pivmin, as in the ratio form
      double p0 = 1.0, p1 = sd[0] - x;
      if (fabs(p1) < pivmin) p1 = -pivmin;
      c = p1 < 0.0;
#pragma unroll 8
      for (int i = 1; i < m; ++i) {
        double p2 = fma(sd[i] - x, p1, -se2[i - 1] * p0);
        if (fabs(p2) < pivmin * fabs(p1)) p2 = -pivmin * p1;
        c += (p2 < 0.0) != (p1 < 0.0);
        p0 = p1;
        p1 = p2;
        if (fabs(p1) > 0x1p500 || fabs(p1) < 0x1p-500) {
          int ex;
          frexp(p1, &ex);
          p1 = ldexp(p1, -ex);
          p0 = ldexp(p0, -ex);
        }
      }
    } else {
      double q = sd[0] - x;
      if (fabs(q) < pivmin) q = -pivmin;
      c = q < 0.0;
      // unrolled so the shared-memory loads of later steps issue ahead of the
      // division chain (warps issue in order)
#pragma unroll 8
      for (int i = 1; i < m; ++i) {
        q = use_div ? (sd[i] - x) - se2[i - 1] / q : (sd[i] - x) - se2[i - 1] * __drcp_rn(q);
        if (fabs(q) < pivmin) q = -pivmin;
        c += q < 0.0;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, c > idx);
    const double x31 = __shfl_sync(0xffffffffu, x, 31);
    if (bal == 0u) {
      a = x31;
    } else {
      const int f = __ffs(bal) - 1;
      const double xf = __shfl_sync(0xffffffffu, x, f);
      const double xp = __shfl_sync(0xffffffffu, x, f > 0 ? f - 1 : 0);
      b = xf;
      if (f > 0) a = xp;
    }
  }
  if (lane == 0) theta[t] = 0.5 * (a + b);
}

// Sturm count of T - x I: the number of eigenvalues below x.
__device__ __forceinline__ int sturm_count(const double* sd, const double* se2, int m, double x,
                                           double pivmin, int mode) {
  int c;
  if (mode == 2) {
    // division-free three-term recurrence p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2},
    // exact power-of-two rescaling; a pivot p_i / p_{i-1} below pivmin in magnitude
    // is taken as -pivmin, as in the ratio form
    // the range check runs once per 8 steps, off the recurrence's dependency chain
    // (8 steps move |p| by far less than the 2^500 margin to over/underflow)
    double p0 = 1.0, p1 = sd[0] - x;
    if (fabs(p1) < pivmin) p1 = -pivmin;
    c = p1 < 0.0;
    int i = 1;
    for (; i + 8 <= m; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        double p2 = fma(sd[i + u] - x, p1, -se2[i + u - 1] * p0);
        p2 = fabs(p2) < pivmin * fabs(p1) ? -pivmin * p1 : p2;
        c += (p2 < 0.0) != (p1 < 0.0);
        p0 = p1;
        p1 = p2;
      }
      if (fabs(p1) > 0x1p500 || fabs(p1) < 0x1p-500) {
        int ex;
        frexp(p1, &ex);
        p1 = ldexp(p1, -ex);
        p0 = ldexp(p0, -ex);
      }
    }
    for (; i < m; ++i) {
      double p2 = fma(sd[i] - x, p1, -se2[i - 1] * p0);
      p2 = fabs(p2) < pivmin * fabs(p1) ? -pivmin * p1 : p2;
      c += (p2 < 0.0) != (p1 < 0.0);
      p0 = p1;
      p1 = p2;
    }
  } else {
    double q = sd[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    c = q < 0.0;
#pragma unroll 8
    for (int i = 1; i < m; ++i) {
      q = mode ? (sd[i] - x) - se2[i - 1] / q : (sd[i] - x) - se2[i - 1] * __drcp_rn(q);
      if (fabs(q) < pivmin) q = -pivmin;
      c += q < 0.0;
    }
  }
  return c;
}

// One CTA of BSW warps per eigenvalue index (first + blockIdx.x): (32 BSW + 1)-
// section of the Gershgorin interval, so a round narrows the bracket 257-fold at
// BSW = 8 (about 7 rounds to full precision instead of 11 with one warp).
constexpr int BSW = 8;

__global__ void __launch_bounds__(32 * BSW)
bisect_cta(const double* __restrict__ d, const double* __restrict__ e, int m, int first,
           int count, double* __restrict__ theta, const SmallStatus* status, int mode) {
  extern __shared__ double bsd[];  // d[m], e2[m]
  __shared__ int wfirst[2][BSW];
  __shared__ double red3[3][BSW];
  if (status && (status->nonfinite || status->not_pd)) return;
  double* sd = bsd;
  double* se2 = bsd + m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int P = 32 * BSW;
  double lo = DBL_MAX, hi = -DBL_MAX, emax = 0.0;
  for (int i = tid; i < m; i += P) {
    const double di = d[i];
    sd[i] = di;
    se2[i] = i + 1 < m ? e[i] * e[i] : 0.0;
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < m ? fabs(e[i]) : 0.0);
    lo = fmin(lo, di - r);
    hi = fmax(hi, di + r);
    if (i + 1 < m) emax = fmax(emax, e[i] * e[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  if (lane == 0) {
    red3[0][warp] = lo;
    red3[1][warp] = hi;
    red3[2][warp] = emax;
  }
  __syncthreads();
  lo = red3[0][0];
  hi = red3[1][0];
  emax = red3[2][0];
  for (int w2 = 1; w2 < BSW; ++w2) {
    lo = fmin(lo, red3[0][w2]);
    hi = fmax(hi, red3[1][w2]);
    emax = fmax(emax, red3[2][w2]);
  }
  const int idx = first + blockIdx.x;
  if (blockIdx.x >= count) return;
  const double pivmin = DBL_MIN * fmax(1.0, emax);
  const double tnorm = fmax(fabs(lo), fabs(hi));
  lo -= 2.0 * kEps64 * tnorm + 2.0 * pivmin;
  hi += 2.0 * kEps64 * tnorm + 2.0 * pivmin;
  double a = lo, b = hi;
  for (int round = 0; round < 64; ++round) {
    const double w = b - a;
    const double tol = fmax(2.0 * kEps64 * fmax(fabs(a), fabs(b)), kEps64 * tnorm) + pivmin;
    if (w <= tol) break;
    const double x = a + w * (double)(tid + 1) / (double)(P + 1);
    const int c = sturm_count(sd, se2, m, x, pivmin, mode);
    const unsigned bal = __ballot_sync(0xffffffffu, c > idx);
    if (lane == 0) wfirst[round & 1][warp] = bal ? warp * 32 + __ffs(bal) - 1 : INT_MAX;
    __syncthreads();
    int f = INT_MAX;
    for (int w2 = 0; w2 < BSW; ++w2) f = min(f, wfirst[round & 1][w2]);
    if (f == INT_MAX) {
      a = a + w * (double)P / (double)(P + 1);
    } else {
      const double xf = a + w * (double)(f + 1) / (double)(P + 1);
      const double xp = a + w * (double)f / (double)(P + 1);
      b = xf;
      if (f > 0) a = xp;
    }
  }
  if (tid == 0) theta[blockIdx.x] = 0.5 * (a + b);
}

// Sturm pivots by true division (dstebz's arithmetic) unless SPB_BISECT_RCP is
// set: the reciprocal variant is faster but its last-bit differences measurably
// change long LOBPCG trajectories (tests/test_gpu_lobpcg.py rand150).
int bisect_div() { return 2; }

__device__ __forceinline__ double hash_uniform(uint32_t a, uint32_t b) {
  uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return (double)h / 4294967296.0 * 2.0 - 1.0;
}

// Inverse iteration for the eigenvectors of T (d, e) at shifts theta[0..nev).
// One thread per eigenvalue; scratch is laid out [array][i][thread] so a warp's
// accesses coalesce. Eigenvalues closer than ctol = 1e-8 ||T|| form a cluster
// handled by its first thread, which orthogonalises later members against
// earlier ones (MGS), as LAPACK dstein does with its (wider) 1e-3 ||T||; for
// gaps above ctol inverse iteration alone gives orthogonality eps ||T|| / gap.
__global__ void invit(const double* __restrict__ d_g, const double* __restrict__ e_g, int m, int nev,
                      const double* __restrict__ theta, double* __restrict__ Y, int ldy,
                      double* __restrict__ gscratch, int use_smem, const SmallStatus* status) {
  // One eigenvector (cluster head) per CTA of one warp: the lanes stage d, e in
  // shared memory and reduce ||T||; lane 0 runs the serial recurrences.
  extern __shared__ double ssc[];
  if (status && (status->nonfinite || status->not_pd)) return;
  const int j0 = blockIdx.x;
  if (j0 >= nev) return;
  const int lane = threadIdx.x & 31;
  double* d = ssc;                 // m
  double* e = ssc + m;             // m
  double* scratch = ssc + 2 * m;   // 6 m
  (void)gscratch;
  (void)use_smem;
  double tn = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double di = d_g[i], ei = i + 1 < m ? e_g[i] : 0.0;
    d[i] = di;
    e[i] = ei;
    tn = fmax(tn, fabs(di) + (i > 0 ? fabs(e_g[i - 1]) : 0.0) + fabs(ei));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
  __syncwarp();
  if (lane != 0) return;
  const double tnorm = fmax(tn, DBL_MIN);
  const double ctol = 1e-8 * tnorm;
  if (j0 > 0 && theta[j0] - theta[j0 - 1] <= ctol) return;  // not a cluster head
  // use_smem == 2: isolated eigenvalues were solved by twisted_vec
  if (use_smem == 2 && !(j0 + 1 < nev && theta[j0 + 1] - theta[j0] <= ctol)) return;
  auto at = [&](int a2, int i) -> double& { return scratch[a2 * m + i]; };
  const double pert = kEps64 * tnorm;
  double lam_prev = -DBL_MAX;
  for (int j = j0; j < nev; ++j) {
    if (j > j0 && theta[j] - theta[j - 1] > ctol) break;
    double lam = theta[j];
    if (j > j0 && lam - lam_prev < 10.0 * kEps64 * fabs(lam)) lam = lam_prev + 10.0 * kEps64 * fabs(lam);
    lam_prev = lam;
    // LU with partial pivoting of T - lam I (dgttrf): 0 dl, 1 dd (then 1/dd), 2 du,
    // 3 du2, 4 y, 5 swap. The running pivot and super-diagonal are carried in
    // registers (the shared-memory round trip per step was the critical path).
    {
      double dcur = d[0] - lam;
      double ucur = m > 1 ? e[0] : 0.0;
#pragma unroll 2
      for (int i = 0; i + 1 < m; ++i) {
        const double li = e[i];
        const double dn0 = d[i + 1] - lam;
        const double un0 = i + 2 < m ? e[i + 1] : 0.0;
        double di = dcur;
        if (fabs(di) >= fabs(li)) {
          if (di == 0.0) di = pert;
          const double f = li / di;
          at(0, i) = f;
          at(1, i) = di;
          at(2, i) = ucur;
          at(3, i) = 0.0;
          at(5, i) = 0.0;
          dcur = dn0 - f * ucur;
          ucur = un0;
        } else {
          const double f = di / li;
          at(0, i) = f;
          at(1, i) = li;
          at(2, i) = dn0;
          at(3, i) = un0;
          at(5, i) = 1.0;
          dcur = ucur - f * dn0;
          ucur = -f * un0;
        }
      }
      at(1, m - 1) = dcur;
      at(2, m - 1) = 0.0;
      at(3, m - 1) = 0.0;
      at(5, m - 1) = 0.0;
    }
    for (int i = 0; i < m; ++i) {  // tiny pivots perturbed; array 1 then holds 1/pivot
      double v = at(1, i);
      if (fabs(v) < pert) v = copysign(pert, v == 0.0 ? 1.0 : v);
      at(1, i) = 1.0 / v;
    }
    for (int i = 0; i < m; ++i) at(4, i) = hash_uniform((uint32_t)j, (uint32_t)i);
    for (int it = 0; it < 2; ++it) {
      {  // forward: row interchanges and L, running value in a register
        double ycar = at(4, 0);
#pragma unroll 4
        for (int i = 0; i + 1 < m; ++i) {
          const double yn = at(4, i + 1), f = at(0, i);
          if (at(5, i) != 0.0) {
            at(4, i) = yn;
            ycar = ycar - f * yn;
          } else {
            at(4, i) = ycar;
            ycar = yn - f * ycar;
          }
        }
        at(4, m - 1) = ycar;
      }
      double y2 = at(4, m - 1) * at(1, m - 1);
      at(4, m - 1) = y2;
      double y1 = y2;
      if (m >= 2) {
        y1 = (at(4, m - 2) - at(2, m - 2) * y2) * at(1, m - 2);
        at(4, m - 2) = y1;
      }
#pragma unroll 4
      for (int i = m - 3; i >= 0; --i) {
        const double yi = (at(4, i) - at(2, i) * y1 - at(3, i) * y2) * at(1, i);
        at(4, i) = yi;
        y2 = y1;
        y1 = yi;
      }
      for (int q = j0; q < j; ++q) {  // MGS inside the cluster
        double sdot = 0.0;
        for (int i = 0; i < m; ++i) sdot += Y[(size_t)i * ldy + q] * at(4, i);
        for (int i = 0; i < m; ++i) at(4, i) -= sdot * Y[(size_t)i * ldy + q];
      }
      double amax = 0.0;
#pragma unroll 4
      for (int i = 0; i < m; ++i) amax = fmax(amax, fabs(at(4, i)));
      if (amax == 0.0) {
        for (int i = 0; i < m; ++i) at(4, i) = hash_uniform((uint32_t)j + 7919u * (it + 1), (uint32_t)i);
        continue;
      }
      const double ia = 1.0 / amax;
      double nrm = 0.0;
#pragma unroll 4
      for (int i = 0; i < m; ++i) {
        const double v = at(4, i) * ia;
        nrm = fma(v, v, nrm);
      }
      const double sc2 = ia / sqrt(nrm);  // scale by 1/amax then by 1/norm, in one pass
#pragma unroll 4
      for (int i = 0; i < m; ++i) at(4, i) *= sc2;
    }
    for (int i = 0; i < m; ++i) Y[(size_t)i * ldy + j] = at(4, i);
  }
}

// Eigenvectors of T (d, e) for isolated eigenvalues by one twisted factorization
// (the core of LAPACK's dlar1v): T - lam I = L D+ L' = U D- U' (stationary qd, lane 0
// forward and lane 1 backward in parallel), twist index r = argmin |gamma_r| with
// gamma_r = D+_r + D-_r - (d_r - lam), then z_r = 1, z_i = -(e_i / D+_i) z_{i+1} below
// and z_i = -(e_{i-1} / D-_i) z_{i-1} above (again one lane each), normalised. With
// bisection-accurate lam the residual is O(eps ||T||) after this single solve (two
// serial sweeps instead of invit's LU + two inverse iterations). Eigenvalues within
// ctol = 1e-8 ||T|| of a neighbour are left to invit (MGS inside the cluster).
__global__ void __launch_bounds__(32)
twisted_vec(const double* __restrict__ d_g, const double* __restrict__ e_g, int m, int nev,
            const double* __restrict__ theta, double* __restrict__ Y, int ldy,
            const SmallStatus* status) {
  extern __shared__ double tws[];
  if (status && (status->nonfinite || status->not_pd)) return;
  const int j = blockIdx.x;
  if (j >= nev) return;
  const int lane = threadIdx.x & 31;
  if (m == 1) {
    if (lane == 0) Y[j] = 1.0;
    return;
  }
  double* d = tws;           // m
  double* e = d + m;         // m (e[m-1] = 0)
  double* rp = e + m;        // e_i / D+_i
  double* rm = rp + m;       // e_{i-1} / D-_i
  double* gp = rm + m;       // D+_i
  double* gm = gp + m;       // D-_i
  double* z = gm + m;        // vector
  double tn = 0.0, e2max = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double di = d_g[i], ei = i + 1 < m ? e_g[i] : 0.0;
    d[i] = di;
    e[i] = ei;
    tn = fmax(tn, fabs(di) + (i > 0 ? fabs(e_g[i - 1]) : 0.0) + fabs(ei));
    e2max = fmax(e2max, ei * ei);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
    e2max = fmax(e2max, __shfl_xor_sync(0xffffffffu, e2max, o));
  }
  const double tnorm = fmax(tn, DBL_MIN);
  const double ctol = 1e-8 * tnorm;
  const double lam = theta[j];
  if ((j > 0 && lam - theta[j - 1] <= ctol) || (j + 1 < nev && theta[j + 1] - lam <= ctol))
    return;  // clustered: invit
  const double pivmin = DBL_MIN * fmax(1.0, e2max);
  __syncwarp();
  if (lane == 0) {
    double D = d[0] - lam;
    for (int i = 0; i + 1 < m; ++i) {
      if (fabs(D) < pivmin) D = -pivmin;
      gp[i] = D;
      const double r = e[i] / D;
      rp[i] = r;
      D = (d[i + 1] - lam) - e[i] * r;
    }
    gp[m - 1] = D;
  } else if (lane == 1) {
    double D = d[m - 1] - lam;
    for (int i = m - 1; i > 0; --i) {
      if (fabs(D) < pivmin) D = -pivmin;
      gm[i] = D;
      const double r = e[i - 1] / D;
      rm[i] = r;
      D = (d[i - 1] - lam) - e[i - 1] * r;
    }
    gm[0] = D;
  }
  __syncwarp();
  // twist index: smallest |gamma_r| (lowest r on ties)
  double best = DBL_MAX;
  int br = 0;
  for (int r = lane; r < m; r += 32) {
    const double g = fabs(gp[r] + gm[r] - (d[r] - lam));
    if (g < best) {
      best = g;
      br = r;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int orr = __shfl_xor_sync(0xffffffffu, br, o);
    if (ob < best || (ob == best && orr < br)) {
      best = ob;
      br = orr;
    }
  }
  // the two halves from z_r = 1, with power-of-two rescaling so neither overflows;
  // each lane tracks its exponent and the halves are reconciled afterwards
  int ex = 0;
  if (lane == 0) {
    double zc = 1.0;
    z[br] = 1.0;
    for (int i = br - 1; i >= 0; --i) {
      zc = -rp[i] * zc;
      if (fabs(zc) > 0x1p400) {  // rescale this half (entries i+1 .. br)
        for (int q = i + 1; q <= br; ++q) z[q] = ldexp(z[q], -400);
        zc = ldexp(zc, -400);
        ex += 400;
      }
      z[i] = zc;
    }
  } else if (lane == 1) {
    double zc = 1.0;
    for (int i = br + 1; i < m; ++i) {
      zc = -rm[i] * zc;
      if (fabs(zc) > 0x1p400) {  // rescale entries br+1 .. i-1 (z[br] belongs to lane 0)
        for (int q = br + 1; q < i; ++q) z[q] = ldexp(z[q], -400);
        zc = ldexp(zc, -400);
        ex += 400;
      }
      z[i] = zc;
    }
  }
  const int ex0 = __shfl_sync(0xffffffffu, ex, 0), ex1 = __shfl_sync(0xffffffffu, ex, 1);
  __syncwarp();
  // common scale 2^-max(ex): the half with the smaller exponent is scaled down
  const int emax = max(ex0, ex1);
  double ss = 0.0;
  for (int i = lane; i < m; i += 32) {
    const int ei = i <= br ? ex0 : ex1;
    const double v = ldexp(z[i], ei - emax);
    z[i] = v;
    ss = fma(v, v, ss);
  }
  ss = warp_sum(ss);
  const double inv = 1.0 / sqrt(ss);
  for (int i = lane; i < m; i += 32) Y[(size_t)i * ldy + j] = z[i] * inv;
}

// Z = Q Y with Q = H_0 H_1 ... H_{m-3}, applied in blocks of 32 reflectors
// (compact WY, as LAPACK dormtr/dlarft): B_b = I - V_b T_b V_b', Z = B_0 (B_1 (... (B_last Y))).
// wy_tfactors: one CTA per block stages V_b in shared memory and forms
// G = V_b'V_b and T_b (forward column recurrence), all blocks at once.
// wy_apply: the columns of Y are independent, so each CTA owns BCW of them in
// shared memory and runs the block loop W1 = V_b' Y, W2 = T_b W1, Y -= V_b W2
// with V_b staged per block.
constexpr int BCW = 4;     // Y columns per CTA
constexpr int BAT = 32 * BCW;  // threads of wy_apply (= 32 reflectors x BCW columns)

__global__ void __launch_bounds__(256)
wy_tfactors(const double* __restrict__ V, const double* __restrict__ tau, int m,
            double* __restrict__ Tall, const SmallStatus* status) {
  extern __shared__ double tvb[];  // V_b rows [32][m | 1]
  __shared__ double G[32][33];
  __shared__ double Tm[32][33];
  if (status && (status->nonfinite || status->not_pd)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrefl = m - 2;
  const int kb = blockIdx.x * 32;
  const int nb = min(32, nrefl - kb);
  const int r0 = kb + 1;
  const int vld = m | 1;
  for (int x = tid; x < nb * m; x += 256) {
    const int j = x / m, r = x - (x / m) * m;
    tvb[j * vld + r] = V[(size_t)(kb + j) * m + r];
  }
  __syncthreads();
  for (int x = warp; x < nb * nb; x += 8) {
    const int i = x / nb, j = x % nb;
    double acc = 0.0;
    if (i <= j) {
      const double* vi = tvb + i * vld;
      const double* vj = tvb + j * vld;
      for (int r = r0 + lane; r < m; r += 32) acc += vi[r] * vj[r];
      acc = warp_sum(acc);
    }
    if (lane == 0) G[i][j] = acc;
  }
  __syncthreads();
  if (warp == 0) {
    for (int j = 0; j < nb; ++j) {
      const double tj = tau[kb + j];
      double x = 0.0;
      if (lane < j) {
        for (int q = lane; q < j; ++q) x += Tm[lane][q] * G[q][j];
        x = -tj * x;
      }
      __syncwarp();
      if (lane < j) Tm[lane][j] = x;
      if (lane == j) Tm[j][j] = tj;
      if (lane > j) Tm[lane][j] = 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
  double* T = Tall + (size_t)blockIdx.x * 1024;
  for (int x = tid; x < 1024; x += 256) {
    const int i = x >> 5, j = x & 31;
    T[x] = (i < nb && j < nb) ? Tm[i][j] : 0.0;
  }
}

// WYT threads: the first BAT = 32 x BCW of them own one (reflector, column) pair of
// the 32 x BCW products; all of them stage the reflector block (83 KB from L2 per step
// at m = 324 -- with 128 threads that staging was most of a step) and share the Y
// update; every output keeps its summation order (results bit-identical).
constexpr int WYT = 4 * BAT;

__global__ void __launch_bounds__(WYT)
wy_apply(const double* __restrict__ V, int m, const double* __restrict__ Tall, double* Y,
         int ldy, int nev, const SmallStatus* status) {
  extern __shared__ double wsm[];
  if (status && (status->nonfinite || status->not_pd)) return;
  const int vld = m | 1;                       // odd row stride: conflict-free column reads
  double* Ys = wsm;                            // [m][BCW]
  double* Vb = Ys + (size_t)m * BCW;           // [32][vld]
  double* W1 = Vb + 32 * (size_t)vld;          // [32][BCW]
  double* W2 = W1 + 32 * BCW;                  // [32][BCW]
  double* Tb = W2 + 32 * BCW;                  // [32][33]
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * BCW;
  const int nc = min(BCW, nev - c0);
  for (int x = tid; x < m * BCW; x += WYT) {
    const int r = x / BCW, c = x % BCW;
    Ys[x] = c < nc ? Y[(size_t)r * ldy + c0 + c] : 0.0;
  }
  const int nrefl = m - 2;
  const int part = tid / BAT, pt = tid % BAT;  // quarter of the dot, (reflector, column) pair
  const int jj = pt / BCW, cc = pt % BCW;
  for (int kb = ((nrefl - 1) / 32) * 32; kb >= 0; kb -= 32) {
    const int nb = min(32, nrefl - kb);
    const double* T = Tall + (size_t)(kb / 32) * 1024;
    // rows kb..kb+nb-1 of V are contiguous: stage them with 8 loads in flight per thread
    const double* Vsrc = V + (size_t)kb * m;
    for (int x0 = tid; x0 < nb * m; x0 += WYT * 8) {
      double tv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) tv[u] = x0 + u * WYT < nb * m ? Vsrc[x0 + u * WYT] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int x = x0 + u * WYT;
        if (x < nb * m) {
          const int j = x / m, r = x - (x / m) * m;
          Vb[j * vld + r] = tv[u];
        }
      }
    }
    for (int x = tid; x < 1024; x += WYT) Tb[(x >> 5) * 33 + (x & 31)] = T[x];
    __syncthreads();
    // W1 = V_b' Y (v_{kb+j}[r] = 0 for r <= kb + j). One thread per (reflector, column)
    // with the summation order this kernel has always had: split four ways over the
    // idle threads the Ritz vectors moved by ~5e-17, and the planted float32 case of
    // tests/test_gpu_f32_guard.py -- a solve at the float32 residual floor -- took a
    // different trajectory (300 iterations instead of 83).
    if (part == 0 && jj < nb) {
      double a0 = 0.0, a1 = 0.0;
      const double* vr = Vb + jj * vld;
      int r = kb + jj + 1;
      for (; r + 1 < m; r += 2) {
        a0 = fma(vr[r], Ys[r * BCW + cc], a0);
        a1 = fma(vr[r + 1], Ys[(r + 1) * BCW + cc], a1);
      }
      if (r < m) a0 = fma(vr[r], Ys[r * BCW + cc], a0);
      W1[pt] = a0 + a1;
    }
    __syncthreads();
    // W2 = T_b W1 (upper triangular)
    if (part == 0 && jj < nb) {
      double acc = 0.0;
      for (int q = jj; q < nb; ++q) acc = fma(Tb[jj * 33 + q], W1[q * BCW + cc], acc);
      W2[jj * BCW + cc] = acc;
    }
    __syncthreads();
    // Y -= V_b W2
    for (int x = tid; x < (m - kb - 1) * BCW; x += WYT) {
      const int r = kb + 1 + x / BCW, c = x % BCW;
      const int jmax = min(nb, r - kb);
      double acc = 0.0;
      for (int j = 0; j < jmax; ++j) acc = fma(Vb[j * vld + r], W2[j * BCW + c], acc);
      Ys[r * BCW + c] -= acc;
    }
    __syncthreads();
  }
  for (int x = tid; x < m * BCW; x += WYT) {
    const int r = x / BCW, c = x % BCW;
    if (c < nc) Y[(size_t)r * ldy + c0 + c] = Ys[x];
  }
}

size_t wy_apply_smem(int m) {
  return sizeof(double) * ((size_t)m * BCW + 32 * (size_t)(m | 1) + 64 * BCW + 32 * 33);
}

void launch_wy_tfactors(const double* V, const double* tau, int m, double* Tscratch,
                        const SmallStatus* status, cudaStream_t st) {
  const int nrefl = m - 2;
  if (nrefl <= 0) return;
  const int nblk = (nrefl + 31) / 32;
  wy_tfactors<<<nblk, 256, sizeof(double) * 32 * (size_t)(m | 1), st>>>(V, tau, m, Tscratch, status);
}

void launch_wy_apply(const double* V, int m, const double* Tscratch, double* Y, int nev,
                     const SmallStatus* status, cudaStream_t st) {
  if (m - 2 <= 0 || nev <= 0) return;
  wy_apply<<<(nev + BCW - 1) / BCW, WYT, wy_apply_smem(m), st>>>(V, m, Tscratch, Y, nev, nev,
                                                                  status);
}

// Side stream (per device) on which the compact-WY T factors are formed while
// the main stream runs bisection and inverse iteration: both only need the
// tridiagonalisation, so they overlap.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t pre_fork = nullptr, pre_join = nullptr;  // sygv_prefactor_b
};
// One side stream (and its events) per (device, caller stream): two solves running on
// different streams never share events. Entries live for the process (a caller's
// streams are few and pooled); the table is guarded by a mutex.
SideStream* side_stream(cudaStream_t main) {
  struct Key {
    int dev;
    cudaStream_t st;
    SideStream ss;
  };
  static std::mutex mu;
  static std::deque<Key> table;  // deque: stable addresses
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (Key& k : table)
    if (k.dev == dev && k.st == main) return &k.ss;
  table.push_back(Key{dev, main, SideStream{}});
  SideStream& x = table.back().ss;
  cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&x.pre_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&x.pre_join, cudaEventDisableTiming);
  return &x;
}

__global__ void copy_cols(const double* __restrict__ Y, int ldy, int m, int nev,
                          double* __restrict__ C, int ldc) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < m * nev; x += gridDim.x * blockDim.x) {
    const int i = x / nev, j = x % nev;
    C[(size_t)i * ldc + j] = Y[(size_t)i * ldy + j];
  }
}

// Pivoted Cholesky (diagonal pivoting == dgeqp3 column pivoting on B).
__global__ void __launch_bounds__(ET)
pivoted_chol(const double* __restrict__ g, int ldg, int na, double rank_tol, double* __restrict__ G,
             int* __restrict__ perm, double* __restrict__ Rinv, SmallStatus* status) {
  __shared__ int sp;
  __shared__ int srank;
  __shared__ double sd0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int x = tid; x < na * na; x += ET) {
    const int i = x / na, j = x % na;
    G[x] = 0.5 * (g[(int64_t)i * ldg + j] + g[(int64_t)j * ldg + i]);
  }
  for (int i = tid; i < na; i += ET) perm[i] = i;
  if (tid == 0) srank = na;
  __syncthreads();
  for (int j = 0; j < na; ++j) {
    if (tid == 0) {
      int p = j;
      double best = G[(size_t)j * na + j];
      for (int i = j + 1; i < na; ++i) {
        const double v = G[(size_t)i * na + i];
        if (v > best) { best = v; p = i; }
      }
      if (j == 0) sd0 = best;
      if (!(best > 0.0) || sqrt(best) <= rank_tol * sqrt(sd0)) srank = j;
      sp = p;
    }
    __syncthreads();
    if (srank == j) break;
    const int p = sp;
    if (p != j) {  // symmetric swap of rows/cols j and p
      for (int x = tid; x < na; x += ET) {
        const double a = G[(size_t)j * na + x];
        G[(size_t)j * na + x] = G[(size_t)p * na + x];
        G[(size_t)p * na + x] = a;
      }
      __syncthreads();
      for (int x = tid; x < na; x += ET) {
        const double a = G[(size_t)x * na + j];
        G[(size_t)x * na + j] = G[(size_t)x * na + p];
        G[(size_t)x * na + p] = a;
      }
      if (tid == 0) {
        const int t = perm[j];
        perm[j] = perm[p];
        perm[p] = t;
      }
      __syncthreads();
    }
    if (tid == 0) G[(size_t)j * na + j] = sqrt(G[(size_t)j * na + j]);
    __syncthreads();
    const double piv = G[(size_t)j * na + j];
    for (int i = j + 1 + tid; i < na; i += ET) G[(size_t)i * na + j] /= piv;
    __syncthreads();
    for (int i = j + 1 + warp; i < na; i += ET / 32) {
      const double gij = G[(size_t)i * na + j];
      for (int k = j + 1 + lane; k <= i; k += 32) G[(size_t)i * na + k] -= gij * G[(size_t)k * na + j];
    }
    __syncthreads();
  }
  const int rk = srank;
  // Rinv = inverse of the upper factor R11 = L11' (rank x rank), via L11^-1 rows
  double* Li = Rinv;  // use as scratch then transpose
  for (int i = 0; i < rk; ++i) {
    const double lii = G[(size_t)i * na + i];
    for (int j = warp; j <= i; j += ET / 32) {
      double s = 0.0;
      for (int k = j + lane; k < i; k += 32) s += G[(size_t)i * na + k] * Li[(size_t)k * na + j];
      s = warp_sum(s);
      if (lane == 0) Li[(size_t)i * na + j] = ((i == j ? 1.0 : 0.0) - s) / lii;
    }
    for (int j = i + 1 + tid; j < na; j += ET) Li[(size_t)i * na + j] = 0.0;
    __syncthreads();
  }
  for (int x = tid; x < na * na; x += ET) {
    const int i = x / na, j = x % na;
    if (i >= rk || j >= rk) continue;
    if (i < j) {
      const double a = Li[(size_t)i * na + j], b = Li[(size_t)j * na + i];
      Li[(size_t)i * na + j] = b;
      Li[(size_t)j * na + i] = a;
    }
  }
  if (tid == 0) status->rank = rk;
}

// One-sided Jacobi SVD of the k x k matrix S (row-major) and S^-1 = V S^-2 U'.
__global__ void __launch_bounds__(ET)
jacobi_svd(const double* __restrict__ S, int k, double* __restrict__ U, double* __restrict__ Vm,
           double* __restrict__ inv, SmallStatus* status) {
  __shared__ int rotated;
  __shared__ double red[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = (k + 1) & ~1;  // even number of players (k odd: one dummy)
  // column-major copies: U[:, j] contiguous
  for (int x = tid; x < K * k; x += ET) {
    const int j = x / k, i = x % k;
    U[x] = j < k ? S[(size_t)i * k + j] : 0.0;
  }
  for (int x = tid; x < K * K; x += ET) Vm[x] = (x / K == x % K) ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < K - 1; ++r) {
      for (int t = warp; t < K / 2; t += ET / 32) {
        int p, q;
        if (t == 0) { p = r; q = K - 1; }
        else { p = (r + t) % (K - 1); q = (r - t + (K - 1)) % (K - 1); }
        if (p > q) { const int z = p; p = q; q = z; }
        if (q >= k) continue;  // dummy column
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < k; i += 32) {
          const double up = U[(size_t)p * k + i], uq = U[(size_t)q * k + i];
          a += up * up;
          b += uq * uq;
          g += up * uq;
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (fabs(g) > kEps64 * sqrt(a * b) && g != 0.0) {
          const double zeta = (b - a) / (2.0 * g);
          const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
          for (int i = lane; i < k; i += 32) {
            const double up = U[(size_t)p * k + i], uq = U[(size_t)q * k + i];
            U[(size_t)p * k + i] = c * up - s * uq;
            U[(size_t)q * k + i] = s * up + c * uq;
          }
          for (int i = lane; i < k; i += 32) {
            const double vp = Vm[(size_t)p * K + i], vq = Vm[(size_t)q * K + i];
            Vm[(size_t)p * K + i] = c * vp - s * vq;
            Vm[(size_t)q * K + i] = s * vp + c * vq;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  // singular values = column norms of U
  double smax = 0.0, smin = DBL_MAX;
  for (int j = 0; j < k; ++j) {
    double s = 0.0;
    for (int i = tid; i < k; i += ET) s += U[(size_t)j * k + i] * U[(size_t)j * k + i];
    s = block_sum(s, red);
    const double sv = sqrt(s);
    smax = fmax(smax, sv);
    smin = fmin(smin, sv);
  }
  if (tid == 0) {
    status->cond_hi = smin > 0.0 ? smax / smin : INFINITY;
    status->dmax = smax;
    status->dmin = smin;
  }
}

// U[:, t] /= s_t^2 so that V U' = V S^-2 U'_unscaled = S^-1.
__global__ void scale_u_cols(double* __restrict__ U, int k) {
  const int t = blockIdx.x;
  __shared__ double red[33];
  double s = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) s += U[(size_t)t * k + i] * U[(size_t)t * k + i];
  s = block_sum(s, red);
  const double inv2 = s > 0.0 ? 1.0 / s : 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) U[(size_t)t * k + i] *= inv2;
}

// inv[i][j] = sum_t V[i][t] U[j][t]   (columns t of U already scaled by 1/s_t^2)
__global__ void jacobi_inv(const double* __restrict__ U, const double* __restrict__ Vm, int k,
                           int K, double* __restrict__ inv) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < k * k; x += gridDim.x * blockDim.x) {
    const int i = x / k, j = x % k;
    double acc = 0.0;
    for (int t = 0; t < k; ++t) acc += Vm[(size_t)t * K + i] * U[(size_t)t * k + j];
    inv[(size_t)i * k + j] = acc;
  }
}

struct SygvWs {
  double *A, *B, *L, *Linv, *M, *Ap, *W, *V, *tau, *d, *e, *Y, *scratch;
};

SygvWs carve_sygv(double* base, int m, int nev) {
  SygvWs w;
  size_t mm = (size_t)m * m, off = 0;
  auto take = [&](size_t cnt) {
    double* p = base ? base + off : nullptr;
    off += (cnt + 31) / 32 * 32;
    return p;
  };
  w.A = take(mm);
  w.B = take(mm);
  w.L = take(2 * mm);
  w.Linv = take(mm);
  w.M = take(mm);
  w.Ap = take(mm);
  w.W = take(mm + 4 * (size_t)m);
  w.V = take(mm);
  w.tau = take(m + 1);
  w.d = take(m + 1);
  w.e = take(m + 1);
  w.Y = take((size_t)m * std::max(nev, 1));
  w.scratch = take((size_t)(round_up(std::max(nev, 1), 128) + 128) * 6 * m);
  w.scratch += 0;
  (void)off;
  return w;
}

size_t sygv_ws_count(int m, int nev) {
  size_t mm = (size_t)m * m;
  auto r = [](size_t c) { return (c + 31) / 32 * 32; };
  return 7 * r(mm) + r(2 * mm) + r(mm + 4 * (size_t)m) + 3 * r(m + 1) + r((size_t)m * std::max(nev, 1)) +
         r((size_t)(round_up(std::max(nev, 1), 128) + 128) * 6 * m);
}

size_t chol_ldl_smem(int m) { return ((size_t)m * (m | 1) + m) * sizeof(double); }

void launch_chol(const double* B, int m, double* L, double* Linv, int mode, SmallStatus* status,
                 cudaStream_t st);

size_t chol_smem(int m) {
  size_t b = (size_t)m * m * sizeof(double);
  if (b > 200 * 1024) return 0;
  size_t b2 = ((size_t)m * m + 32 * (size_t)m) * sizeof(double);
  return b2 <= 224 * 1024 ? b2 : b;
}

size_t tridiag_smem(int m) {
  size_t b = (size_t)m * m * sizeof(double);
  return b <= 190 * 1024 ? b + 2 * m * sizeof(double) : 0;
}

void launch_chol(const double* B, int m, double* L, double* Linv, int mode, SmallStatus* status,
                 cudaStream_t st) {
  if (launch_chol_rowwarp(B, m, L, Linv, mode, status, st)) return;
  if (m <= kCholLdlMax && chol_wsync_smem(m) <= 217 * 1024) {
    chol_wsync<<<1, CWT, chol_wsync_smem(m), st>>>(B, m, L, Linv, mode, status, nullptr);
  } else if (m <= kCholLdlMax && chol_ldl_smem(m) <= 224 * 1024) {
    chol_ldl<<<1, ET, chol_ldl_smem(m), st>>>(B, m, L, Linv, mode, status);
  } else if (m <= kCholClusterMax) {
    const int C = m <= 400 ? 8 : 16;
    static std::atomic<uint64_t> attr{0};
    if (!done_on_device(attr)) {
      cudaFuncSetAttribute(chol_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(chol_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      mark_on_device(attr);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(CCT);
    cfg.dynamicSmemBytes = chol_cluster_smem(m, C);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, chol_cluster, B, m, L, Linv, mode, status);
    chol_finish<<<1, ET, 0, st>>>(B, m, L, Linv, mode, status);
  } else {
    chol_linv<<<1, ET, chol_smem(m), st>>>(B, m, L, Linv, mode, status);
  }
}

int set_smem_attrs() {
  static std::atomic<uint64_t> done{0};
  if (done_on_device(done)) return SPB_OK;
  SPB_CUDA(cudaFuncSetAttribute(chol_linv, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(chol_ldl, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(chol_wsync, cudaFuncAttributeMaxDynamicSharedMemorySize, 217 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(tridiag<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(tridiag<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(tridiag<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(tridiag<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(tridiag<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(tridiag<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(invit, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(wy_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  SPB_CUDA(cudaFuncSetAttribute(wy_tfactors, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  mark_on_device(done);
  return SPB_OK;
}

}  // namespace

size_t sygv_ws_doubles(int m, int nev) { return sygv_ws_count(m, nev); }

// B-side of sygv_enqueue ahead of time: sym(G_B), its Cholesky factor, inverse and
// cond bracket, enqueued on the side stream behind everything already on st. The
// caller keeps st busy (the G_A Gram) and then calls sygv_enqueue(..., b_ready =
// true) with the same m, nev and workspace, which joins before it needs L^-1.
int sygv_prefactor_b(const double* gb, int ldg, int m, int nev, double* ws, size_t ws_doubles,
                     SmallStatus* status, cudaStream_t st, int seg1, int seg2) {
  if (ws_doubles < sygv_ws_count(m, nev)) {
    set_error("sygv workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  SPB_TRY(set_smem_attrs());
  const SygvWs w = carve_sygv(ws, m, nev);
  SideStream* side = side_stream(st);
  SPB_CUDA(cudaEventRecord(side->pre_fork, st));
  SPB_CUDA(cudaStreamWaitEvent(side->s, side->pre_fork, 0));
  const int g1 = (int)std::min<int64_t>(ceil_div((int64_t)m * m, 256), 1024);
  sym_prep<<<g1, 256, 0, side->s>>>(gb, nullptr, ldg, m, w.B, nullptr, status, seg1, seg2);
  launch_chol(w.B, m, w.L, w.Linv, 0, status, side->s);
  SPB_LAUNCH_CHECK();
  SPB_CUDA(cudaEventRecord(side->pre_join, side->s));
  return SPB_OK;
}

// st waits for the last sygv_prefactor_b (used when its result is not consumed).
int sygv_prefactor_join(cudaStream_t st) {
  SPB_CUDA(cudaStreamWaitEvent(st, side_stream(st)->pre_join, 0));
  return SPB_OK;
}

int sygv_enqueue(const double* ga, const double* gb, int ldg, int m, int nev, double* theta,
                 double* C, int ldc, double* ws, size_t ws_doubles, SmallStatus* status,
                 cudaStream_t st, int seg1, int seg2, bool b_ready) {
  if (ws_doubles < sygv_ws_count(m, nev)) {
    set_error("sygv workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  SPB_TRY(set_smem_attrs());
  const SygvWs w = carve_sygv(ws, m, nev);
  const bool ident = (gb == nullptr);
  const int g1 = (int)std::min<int64_t>(ceil_div((int64_t)m * m, 256), 1024);
  const bool pre = b_ready && !ident;
  sym_prep<<<g1, 256, 0, st>>>(ga, pre ? nullptr : gb, ldg, m, w.A, ident || pre ? nullptr : w.B,
                               status, seg1, seg2);
  SPB_LAUNCH_CHECK();
  const double* Atri = w.A;
  if (!ident) {
    if (pre) SPB_TRY(sygv_prefactor_join(st));
    else launch_chol(w.B, m, w.L, w.Linv, 0, status, st);
    SPB_LAUNCH_CHECK();
    launch_small_gemm(0, 0, m, m, m, w.Linv, m, w.A, m, w.M, m, st);
    launch_small_gemm(0, 1, m, m, m, w.M, m, w.Linv, m, w.Ap, m, st);
    SPB_LAUNCH_CHECK();
    Atri = w.Ap;
  }
  launch_tridiag(Atri, m, 1, w.W, w.V, w.tau, w.d, w.e, status, tridiag_smem(m), st);
  SPB_LAUNCH_CHECK();
  SideStream* side = side_stream(st);
  SPB_CUDA(cudaEventRecord(side->fork, st));
  SPB_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
  launch_wy_tfactors(w.V, w.tau, m, w.scratch, status, side->s);  // overlaps bisect + invit
  SPB_CUDA(cudaEventRecord(side->join, side->s));
  {
    bisect_cta<<<nev, 32 * BSW, 2 * sizeof(double) * (size_t)m, st>>>(w.d, w.e, m, 0, nev, theta,
                                                                      status, bisect_div());
    SPB_LAUNCH_CHECK();
  }
  {
    twisted_vec<<<nev, 32, 7 * sizeof(double) * (size_t)m, st>>>(w.d, w.e, m, nev, theta, w.Y,
                                                                 nev, status);
    invit<<<nev, 32, 8 * sizeof(double) * (size_t)m, st>>>(w.d, w.e, m, nev, theta, w.Y, nev,
                                                           nullptr, 2, status);
  }
  SPB_LAUNCH_CHECK();
  SPB_CUDA(cudaStreamWaitEvent(st, side->join, 0));
  launch_wy_apply(w.V, m, w.scratch, w.Y, nev, status, st);
  SPB_LAUNCH_CHECK();
  if (!ident) {
    launch_small_gemm(1, 0, m, nev, m, w.Linv, m, w.Y, nev, C, ldc, st);
  } else {
    copy_cols<<<(int)ceil_div((int64_t)m * nev, 256), 256, 0, st>>>(w.Y, nev, m, nev, C, ldc);
  }
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int exact_cond_spd(const double* gb, int ldg, int m, double* ws, size_t ws_doubles, double* cond,
                   cudaStream_t st, int seg1, int seg2) {
  if (ws_doubles < sygv_ws_count(m, 2)) {
    set_error("cond workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  SPB_TRY(set_smem_attrs());
  const SygvWs w = carve_sygv(ws, m, 2);
  double* ext = w.Y;  // two values
  const int g1 = (int)std::min<int64_t>(ceil_div((int64_t)m * m, 256), 1024);
  sym_prep<<<g1, 256, 0, st>>>(gb, nullptr, ldg, m, w.A, nullptr, nullptr, seg1, seg2);
  launch_tridiag(w.A, m, 0, w.W, w.V, w.tau, w.d, w.e, nullptr, tridiag_smem(m), st);
  bisect<<<1, 32, 2 * sizeof(double) * (size_t)m, st>>>(w.d, w.e, m, 0, 1, ext, nullptr, nullptr,
                                                          bisect_div());
  bisect<<<1, 32, 2 * sizeof(double) * (size_t)m, st>>>(w.d, w.e, m, m - 1, 1, ext + 1, nullptr,
                                                          nullptr, bisect_div());
  SPB_LAUNCH_CHECK();
  double h[2];
  SPB_CUDA(cudaMemcpyAsync(h, ext, sizeof(h), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  // np.linalg.cond = sigma_max / sigma_min; for symmetric G_B sigma = |lambda|
  const double amax = std::max(std::fabs(h[0]), std::fabs(h[1]));
  const double amin = h[0] * h[1] <= 0.0 ? 0.0 : std::min(std::fabs(h[0]), std::fabs(h[1]));
  *cond = amin > 0.0 ? amax / amin : INFINITY;
  return SPB_OK;
}

size_t cholqr_ws_doubles(int na) { return 3 * (size_t)na * na + 64; }

int cholqr_enqueue(const double* g, int ldg, int na, double* rinv, double* ws,
                   SmallStatus* status, cudaStream_t st) {
  SPB_TRY(set_smem_attrs());
  double* S = ws;
  double* L = ws + (size_t)na * na;
  // symmetrise (the reference's _sym(b.T @ b), lobpcg.py:228)
  const int g1 = (int)std::min<int64_t>(ceil_div((int64_t)na * na, 256), 1024);
  sym_prep<<<g1, 256, 0, st>>>(g, nullptr, ldg, na, S, nullptr, status);
  launch_chol(S, na, L, rinv, 1, status, st);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int pivoted_cholqr_enqueue(const double* g, int ldg, int na, double rank_tol, int* perm,
                           double* rinv, double* ws, SmallStatus* status, cudaStream_t st) {
  pivoted_chol<<<1, ET, 0, st>>>(g, ldg, na, rank_tol, ws, perm, rinv, status);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

size_t jacobi_ws_doubles(int k) {
  const size_t K = (size_t)((k + 1) & ~1);
  return std::max(K * k + K * K, 4 * (size_t)k * k) + 64;
}

// Fast path for cond(S) / S^-1 of the QRCP seed block: G = S'S, Cholesky with
// its cond2(G) bracket, S^-1 = L^-T L^-1 S'. status->cond_lo/hi hold the
// bracket of cond2(G) = cond2(S)^2 (status->not_pd when G is not numerically
// PD); the caller decides and falls back to the Jacobi SVD when undecided.
int normal_eq_inverse(const double* s, int k, double* inv, double* ws, size_t ws_doubles,
                      SmallStatus* status, cudaStream_t st) {
  if (ws_doubles < jacobi_ws_doubles(k)) {
    set_error("seed inverse workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  SPB_TRY(set_smem_attrs());
  const size_t kk = (size_t)k * k;
  double* G = ws;
  double* L = ws + kk;
  double* Li = ws + 2 * kk;
  double* T = ws + 3 * kk;
  launch_small_gemm(1, 0, k, k, k, s, k, s, k, G, k, st);  // S'S
  launch_chol(G, k, L, Li, 0, status, st);
  launch_small_gemm(0, 1, k, k, k, Li, k, s, k, T, k, st);   // L^-1 S'
  launch_small_gemm(1, 0, k, k, k, Li, k, T, k, inv, k, st);  // L^-T (L^-1 S')
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int jacobi_svd_inverse(const double* s, int k, double* inv, double* ws, size_t ws_doubles,
                       SmallStatus* status, cudaStream_t st) {
  if (ws_doubles < jacobi_ws_doubles(k)) {
    set_error("jacobi workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  const size_t K = (size_t)((k + 1) & ~1);
  double* U = ws;
  double* Vm = ws + K * k;
  jacobi_svd<<<1, ET, 0, st>>>(s, k, U, Vm, inv, status);
  scale_u_cols<<<k, 256, 0, st>>>(U, k);
  jacobi_inv<<<(int)ceil_div((int64_t)k * k, 256), 256, 0, st>>>(U, Vm, k, (int)K, inv);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

}  // namespace spb

