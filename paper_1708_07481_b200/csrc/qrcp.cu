// (e) QRCP cluster assignment (spectral.py:134-170).
//
//   ortho check   max|X'X - I| <= 1e-6 (spectral.py:149-151)     gram kernel
//   pivots        first k column pivots of dgeqp3(X')            cooperative kernel
//   seeds         sorted pivots, S = X[seeds]                    1 CTA
//   cond / S^-1   one-sided Jacobi SVD of S (cond <= 1e12)       1 CTA
//   labels        argmax_j |(X S^-1)_ij|, zero rows -> 0         row kernel
//   compaction    Partition.from_labels (spectral.py:63-70)      histogram + scan
//
// Pivot selection follows LAPACK dlaqp2: the next pivot is the remaining
// column with the largest partial norm (ties: lowest current position, with
// the column swaps dgeqp3 performs), partial norms are downdated with the new
// reflector's component |q_j' x_c| and recomputed exactly when the downdate
// loses more than half the digits (tol3z = sqrt(eps)). Columns of X' are the
// rows of the vertex-major embedding, so each step is one coalesced pass.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "comm.cuh"
#include "dense.cuh"
#include "smalleig.cuh"

namespace cg = cooperative_groups;

namespace spb {
namespace {

constexpr int QT = 512;  // threads per CTA of the pivot kernel

struct BestRec {
  double val;
  int pos;
  int col;
  double dmax;  // largest norm bound among this CTA's deferred columns
};

__device__ __forceinline__ bool better(double v, int p, double bv, int bp) {
  return v > bv || (v == bv && p < bp);
}

constexpr int QG = 8;           // lanes per column group
constexpr int QKMAX = 160;      // largest k (shared-memory Q)
constexpr int QPER = QKMAX / QG;

__device__ __forceinline__ double group_sum(double v, unsigned gmask) {
  v += __shfl_xor_sync(gmask, v, 4);
  v += __shfl_xor_sync(gmask, v, 2);
  v += __shfl_xor_sync(gmask, v, 1);
  return v;
}

// q' x for one column by an 8-lane group (fixed order: the downdate and the
// deferred replay must produce identical values). fp32 rows with 16-byte
// alignment are read as float4, all loads issued before the FMAs.
template <typename T>
__device__ __forceinline__ double dot_group(const double* __restrict__ q, const T* __restrict__ x,
                                            int k, int gl, unsigned gmask) {
  double s = 0.0;
  if constexpr (sizeof(T) == 4) {
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      constexpr int NV = QKMAX / (4 * QG);
      const int k4 = k >> 2;
      float4 v[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = gl + QG * i;
        v[i] = c < k4 ? __ldg(reinterpret_cast<const float4*>(x) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = gl + QG * i;
        if (c < k4) {
          const double* qq = q + 4 * c;
          s = fma(qq[0], (double)v[i].x, s);
          s = fma(qq[1], (double)v[i].y, s);
          s = fma(qq[2], (double)v[i].z, s);
          s = fma(qq[3], (double)v[i].w, s);
        }
      }
      for (int t = 4 * k4 + gl; t < k; t += QG) s = fma(q[t], (double)x[t], s);
      return group_sum(s, gmask);
    }
  }
  for (int t = gl; t < k; t += QG) s = fma(q[t], (double)x[t], s);
  return group_sum(s, gmask);
}

// Exact partial norm ||(I - Q_s Q_s') x|| (MGS over q_0..q_s): dlaqp2's recompute.
template <typename T>
__device__ double recompute_group(const double* __restrict__ qs, const T* __restrict__ x, int k,
                                  int s, int gl, unsigned gmask) {
  if (s + 1 >= k) return 0.0;
  double acc[QPER];
#pragma unroll
  for (int i = 0; i < QPER; ++i) {
    const int t = gl + QG * i;
    acc[i] = t < k ? (double)x[t] : 0.0;
  }
  for (int t0 = 0; t0 <= s; ++t0) {
    const double* qt = qs + (size_t)t0 * k;
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < QPER; ++i) {
      const int t = gl + QG * i;
      if (t < k) d = fma(qt[t], acc[i], d);
    }
    d = group_sum(d, gmask);
#pragma unroll
    for (int i = 0; i < QPER; ++i) {
      const int t = gl + QG * i;
      if (t < k) acc[i] = fma(-d, qt[t], acc[i]);
    }
  }
  double nn = 0.0;
#pragma unroll
  for (int i = 0; i < QPER; ++i) nn = fma(acc[i], acc[i], nn);
  return sqrt(group_sum(nn, gmask));
}

// Cooperative pivot kernel: ONE grid barrier per step (two on the rare steps
// that resolve deferred columns). Every CTA owns a contiguous range of columns
// of X' (rows of X); per column it keeps (vn1, vn2) in one 16-byte record, the
// current position, and one bit of an "exact and unpivoted" mask in shared
// memory. After the barrier each CTA reduces the per-CTA maxima (double-
// buffered by step parity), replays the column swap dgeqp3 performs (swap
// history in shared memory), forms q_j redundantly (identical arithmetic on
// every CTA), and then makes ONE pass over its exact columns that downdates
// them and already tracks the candidates of the next step.
//
// dlaqp2 recomputes a partial norm exactly when the downdate loses more than
// half the digits. Those columns have lost almost all their norm, so the
// recompute is DEFERRED: the column leaves the mask, remembers the step s0 at
// which dlaqp2 would recompute and carries a bound on the recomputed value
// (2e-4 of its last exact norm: the downdate only defers below sqrt(tol3z) vn2,
// plus a rounding allowance). Whenever a deferred bound reaches
// the best exact candidate, the affected columns are brought up to date by
// replaying dlaqp2's steps s0..j-1 for them (same dots, same formulas) before
// the pivot is chosen, so the pivot sequence is the one dlaqp2 produces.
constexpr int QU = 2;  // columns in flight per lane group

template <typename T>
__global__ void __launch_bounds__(QT)
qrcp_pivots(const T* __restrict__ X, int64_t ldx, int n, int k, double2* __restrict__ vn,
            int* __restrict__ pos, int* __restrict__ dirty, BestRec* __restrict__ bb,
            int* __restrict__ piv) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double qs[];         // q_0..q_{k-1} (k x k), xp[k], cdot[k], mask words
  double* xp = qs + (size_t)k * k;       // pivot column (then residual)
  double* cdot = xp + k;                 // q_t' r
  unsigned* amask = reinterpret_cast<unsigned*>(cdot + k);
  __shared__ BestRec wb[QT / 32];
  __shared__ int swap_pp[1024], swap_cj[1024];  // swap history (position pp, column moved)
  __shared__ int s_p, s_pp, s_cj;
  __shared__ BestRec s_best;
  __shared__ double s_dpersist;  // max bound over this CTA's deferred columns
  __shared__ double s_gmax0;     // largest initial column norm (scale of rounding noise)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / QG, gl = tid % QG;
  const unsigned gmask = 0xFFu << (lane & ~(QG - 1));
  constexpr int NGRP = QT / QG;
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int c_lo = blockIdx.x * per, c_hi = min(n, c_lo + per);
  const int cnt = max(0, c_hi - c_lo);
  const double tol3z = sqrt(kEps64);

  // per-thread running candidate (exact columns) and deferred bound
  double bv = -1.0, dm = -1.0;
  int bp = INT_MAX, bc = -1;
  auto offer = [&](double v, int p, int c) {
    if (better(v, p, bv, bp)) { bv = v; bp = p; bc = c; }
  };

  for (int w = tid; w < (cnt + 31) / 32; w += QT) {
    const int rem = cnt - 32 * w;
    amask[w] = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
  }
  if (tid == 0) s_dpersist = -1.0;
  for (int li = grp; li < cnt; li += NGRP) {
    const int c = c_lo + li;
    const T* x = X + (int64_t)c * ldx;
    double s = 0.0;
    for (int t = gl; t < k; t += QG) {
      const double v = (double)x[t];
      s = fma(v, v, s);
    }
    s = sqrt(group_sum(s, gmask));
    if (gl == 0) {
      vn[c] = make_double2(s, s);
      pos[c] = c;
      dirty[c] = -1;
    }
    offer(s, c, c);
  }
  __syncthreads();

  // block reduction of the running candidates into slot[blockIdx.x]
  auto publish = [&](BestRec* slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; bc = oc; }
    }
    if (lane == 0) wb[warp] = {bv, bp, bc, dm};
    __syncthreads();
    if (tid == 0) {
      BestRec b = wb[0];
      double d = fmax(b.dmax, s_dpersist);
      for (int w = 1; w < QT / 32; ++w) {
        d = fmax(d, wb[w].dmax);
        if (better(wb[w].val, wb[w].pos, b.val, b.pos)) b = wb[w];
      }
      b.dmax = d;
      s_dpersist = d;
      slot[blockIdx.x] = b;
    }
    bv = -1.0;
    dm = -1.0;
    bp = INT_MAX;
    bc = -1;
  };
  // global maximum over the per-CTA records: warp 0, lane-strided loads then a
  // shuffle tree ((value, position) is a total order, so any order gives the
  // same winner)
  auto global_best = [&](const BestRec* slot) {
    if (warp == 0) {
      double bv2 = -1.0, d = -1.0;
      int bp2 = INT_MAX, bc2 = -1;
      for (int g = lane; g < (int)gridDim.x; g += 32) {
        const BestRec r = slot[g];
        d = fmax(d, r.dmax);
        if (better(r.val, r.pos, bv2, bp2)) { bv2 = r.val; bp2 = r.pos; bc2 = r.col; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv2, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp2, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bc2, o);
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
        if (better(ov, op, bv2, bp2)) { bv2 = ov; bp2 = op; bc2 = oc; }
      }
      if (lane == 0) s_best = {bv2, bp2, bc2, d};
    }
    __syncthreads();
    return s_best;
  };

  for (int j = 0; j < k; ++j) {
    BestRec* slot0 = bb + (size_t)((j & 1) * 2) * gridDim.x;
    publish(slot0);
    grid.sync();
    BestRec b = global_best(slot0);
    if (j == 0 && tid == 0) s_gmax0 = b.val;
    if (b.dmax >= b.val || b.col < 0) {
      // resolve deferred columns whose bound reaches the best exact candidate
      const double thr = b.col < 0 ? -1.0 : b.val;
      for (int li = grp; li < cnt; li += NGRP) {
        const int c = c_lo + li;
        const int s0 = dirty[c];
        if (s0 < 0 || pos[c] < j || !(vn[c].x >= thr)) continue;
        const T* x = X + (int64_t)c * ldx;
        double v1 = recompute_group(qs, x, k, s0, gl, gmask), v2 = v1;
        for (int st = s0 + 1; st < j; ++st) {
          if (v1 == 0.0) continue;
          const double d = dot_group(qs + (size_t)st * k, x, k, gl, gmask);
          double temp = fabs(d) / v1;
          temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
          if (temp * v1 * v1 <= tol3z * v2 * v2) {
            v1 = recompute_group(qs, x, k, st, gl, gmask);
            v2 = v1;
          } else {
            v1 = v1 * sqrt(temp);
          }
        }
        if (gl == 0) {
          vn[c] = make_double2(v1, v2);
          dirty[c] = -1;
          atomicOr(&amask[li >> 5], 1u << (li & 31));
        }
      }
      __syncthreads();
      // fresh candidates and deferred bound over this CTA's columns
      if (tid == 0) s_dpersist = -1.0;
      for (int li = tid; li < cnt; li += QT) {
        const int c = c_lo + li;
        if (pos[c] < j) continue;
        const double v = vn[c].x;
        if ((amask[li >> 5] >> (li & 31)) & 1u) offer(v, pos[c], c);
        else if (dirty[c] >= 0) dm = fmax(dm, v);
      }
      __syncthreads();
      BestRec* slot1 = slot0 + gridDim.x;
      publish(slot1);
      grid.sync();
      b = global_best(slot1);
    }
    // ---- every CTA: swap replay, q_j
    if (tid == 0) {
      // perm[j]: column currently at position j = column moved there by the latest
      // earlier swap whose pivot came from position j, else j itself
      int cj = j;
      for (int t = j - 1; t >= 0; --t)
        if (swap_pp[t] == j) { cj = swap_cj[t]; break; }
      s_p = b.col;
      s_pp = b.pos;
      s_cj = cj;
      swap_pp[j] = b.pos;  // column cj moves to the pivot's old position
      swap_cj[j] = cj;
      if (blockIdx.x == 0) piv[j] = b.col;
    }
    __syncthreads();
    const int p = s_p, pp = s_pp, cj = s_cj;
    if (p >= c_lo && p < c_hi && tid == 0) {
      pos[p] = j;
      vn[p].x = 0.0;
      amask[(p - c_lo) >> 5] &= ~(1u << ((p - c_lo) & 31));
    }
    if (cj != p && cj >= c_lo && cj < c_hi && tid == 0) pos[cj] = pp;
    // q_j = normalize((I - Q Q')^2 x_p): CGS2 with thread-parallel dots and updates
    for (int t = tid; t < k; t += QT) xp[t] = (double)X[(int64_t)p * ldx + t];
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      for (int t0 = tid; t0 < j; t0 += QT) {
        const double* qt = qs + (size_t)t0 * k;
        double s = 0.0;
        for (int t = 0; t < k; ++t) s += qt[t] * xp[t];
        cdot[t0] = s;
      }
      __syncthreads();
      for (int t = tid; t < k; t += QT) {
        double r = xp[t];
        for (int t0 = 0; t0 < j; ++t0) r -= cdot[t0] * qs[(size_t)t0 * k + t];
        xp[t] = r;
      }
      __syncthreads();
    }
    double* qj = qs + (size_t)j * k;
    if (warp == 0) {
      double s = 0.0;
      for (int t = lane; t < k; t += 32) s += xp[t] * xp[t];
      s = warp_sum(s);
      const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
      for (int t = lane; t < k; t += 32) qj[t] = xp[t] * inv;
    }
    __syncthreads();
    if (j + 1 == k) break;
    // ---- one pass: downdate the exact columns, defer the ones dlaqp2 recomputes,
    //      and track the next step's candidates
    for (int base = grp; base < cnt; base += NGRP * QU) {
      bool act[QU];
      double2 st[QU];
      int ps[QU];
#pragma unroll
      for (int u = 0; u < QU; ++u) {
        const int li = base + u * NGRP;
        act[u] = li < cnt && ((amask[li >> 5] >> (li & 31)) & 1u);
        if (act[u]) {
          st[u] = vn[c_lo + li];
          ps[u] = pos[c_lo + li];
        }
      }
      double dots[QU];
#pragma unroll
      for (int u = 0; u < QU; ++u)
        dots[u] = act[u] ? dot_group(qj, X + (int64_t)(c_lo + base + u * NGRP) * ldx, k, gl, gmask)
                         : 0.0;
#pragma unroll
      for (int u = 0; u < QU; ++u) {
        if (!act[u]) continue;
        const int li = base + u * NGRP, c = c_lo + li;
        double v1 = st[u].x;
        const double v2 = st[u].y;
        if (v1 != 0.0) {
          double temp = fabs(dots[u]) / v1;
          temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
          if (temp * v1 * v1 <= tol3z * v2 * v2) {  // dlaqp2: temp * (vn1/vn2)^2 <= tol3z
            // Bound on the norm dlaqp2 would recompute: the downdated estimate is
            // <= sqrt(tol3z) vn2 here and its accumulated rounding is O(k eps)
            // relative to vn2 (and to the column's initial norm <= gmax0).
            const double bound = 2e-4 * v2 + 1e-10 * s_gmax0;
            dm = fmax(dm, bound);
            if (gl == 0) {
              dirty[c] = j;
              vn[c].x = bound;
              atomicAnd(&amask[li >> 5], ~(1u << (li & 31)));
            }
            continue;
          }
          v1 = v1 * sqrt(temp);
          if (gl == 0) vn[c].x = v1;
        }
        offer(v1, ps[u], c);
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void gather_seeds(const T* __restrict__ X, int64_t ldx, int k, const int* __restrict__ piv,
                             int* __restrict__ seeds, double* __restrict__ S) {
  __shared__ int sd[1024];
  __shared__ int pv[1024];
  for (int i = threadIdx.x; i < k; i += blockDim.x) pv[i] = piv[i];
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {  // sort by rank (pivots are distinct)
    const int v = pv[i];
    int r = 0;
    for (int j = 0; j < k; ++j) r += pv[j] < v;
    sd[r] = v;
    seeds[r] = v;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) {
    const int i = x / k, t = x % k;
    S[x] = (double)X[(int64_t)sd[i] * ldx + t];
  }
}

constexpr int AJ = 32;  // S^-1 columns per chunk

template <typename T>
__global__ void __launch_bounds__(128)
assign_rows(const T* __restrict__ X, int64_t ldx, int n, int k, const double* __restrict__ inv,
            int* __restrict__ raw, int* __restrict__ present, unsigned long long* zero_rows) {
  extern __shared__ double sinv[];  // k x AJ
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double best = -1.0;
  int lab = 0;
  bool nz = false;
  for (int j0 = 0; j0 < k; j0 += AJ) {
    const int nj = min(AJ, k - j0);
    __syncthreads();
    for (int x = threadIdx.x; x < k * AJ; x += blockDim.x) {
      const int t = x / AJ, jj = x % AJ;
      sinv[x] = jj < nj ? inv[(size_t)t * k + j0 + jj] : 0.0;
    }
    __syncthreads();
    if (i < n) {
      double acc[AJ];
#pragma unroll
      for (int jj = 0; jj < AJ; ++jj) acc[jj] = 0.0;
      for (int t = 0; t < k; ++t) {
        const double xv = (double)X[(int64_t)i * ldx + t];
        nz |= (xv != 0.0);
#pragma unroll
        for (int jj = 0; jj < AJ; ++jj) acc[jj] = fma(xv, sinv[t * AJ + jj], acc[jj]);
      }
#pragma unroll
      for (int jj = 0; jj < AJ; ++jj) {
        const double v = fabs(acc[jj]);
        if (jj < nj && v > best) { best = v; lab = j0 + jj; }
      }
    }
  }
  if (i < n) {
    if (!nz) {
      lab = 0;
      atomicAdd(zero_rows, 1ull);
    }
    raw[i] = lab;
    present[lab] = 1;
  }
}

__global__ void compact_labels(const int* __restrict__ raw, int n, const int* __restrict__ remap,
                               int* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = remap[raw[i]];
}

__global__ void remap_kernel(const int* __restrict__ present, int k, int* __restrict__ remap,
                             int* __restrict__ kfound) {
  if (threadIdx.x == 0) {
    int c = 0;
    for (int j = 0; j < k; ++j) {
      remap[j] = c;
      c += present[j] ? 1 : 0;
    }
    *kfound = c;
  }
}

__global__ void ortho_err_kernel(const double* __restrict__ G, int k, double* __restrict__ out) {
  double m = 0.0;
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) {
    const int i = x / k, j = x % k;
    m = fmax(m, fabs(G[x] - (i == j ? 1.0 : 0.0)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sm[w]);
    *out = r;
  }
}

struct AssignWs {
  double *vn1, *vn2, *Q, *S, *inv, *G, *gpart, *jws, *ortho;
  int *pos, *perm, *piv, *seeds, *raw, *present, *remap, *kfound;
  unsigned long long* zero_rows;
  BestRec* bb;
  SmallStatus* status;
  size_t gpart_cap, jws_cap;
};

AssignWs carve_assign(Arena& a, int n, int k) {
  AssignWs w;
  w.vn1 = a.take<double>(2 * (size_t)n);  // (vn1, vn2) records
  w.vn2 = nullptr;
  w.pos = a.take<int>(n);
  w.perm = a.take<int>(n);
  w.raw = a.take<int>(n);
  w.Q = a.take<double>((size_t)k * k);
  w.S = a.take<double>((size_t)k * k);
  w.inv = a.take<double>((size_t)k * k);
  w.G = a.take<double>((size_t)k * k);
  int ks = 1;
  w.gpart_cap = gram_partial_doubles(n, (int)ceil_div(k, 64) * (int)ceil_div(k, 64), k, k, &ks);
  w.gpart = a.take<double>(w.gpart_cap);
  w.jws_cap = jacobi_ws_doubles(k);
  w.jws = a.take<double>(w.jws_cap);
  w.ortho = a.take<double>(4);
  w.piv = a.take<int>(k);
  w.seeds = a.take<int>(k);
  w.present = a.take<int>(k);
  w.remap = a.take<int>(k);
  w.kfound = a.take<int>(4);
  w.zero_rows = a.take<unsigned long long>(2);
  w.bb = a.take<BestRec>(4 * 2048);
  w.status = a.take<SmallStatus>(1);
  return w;
}

template <typename T>
int assign_t(const void* xv, int64_t ldx, int n, int k, const AssignWs& w, int* labels_out,
             int* pivots_out, double* info, cudaStream_t st) {
  const T* X = (const T*)xv;
  // ---- orthonormality check (spectral.py:149-151)
  GramBatch gb{};
  gb.njobs = 1;
  gb.job[0] = {X, X, ldx, ldx, k, k, 0, 0};
  gb.tile_start[0] = 0;
  gb.tile_start[1] = (int)(ceil_div(k, 64) * ceil_div(k, 64));
  SPB_TRY(gram_batched(sizeof(T) == 4 ? SPB_F32 : SPB_F64, gb, n, k, k, w.gpart, w.gpart_cap,
                       w.G, k, st));
  ortho_err_kernel<<<1, 256, 0, st>>>(w.G, k, w.ortho);
  SPB_LAUNCH_CHECK();
  double oerr = 0.0;
  SPB_CUDA(cudaMemcpyAsync(&oerr, w.ortho, sizeof(double), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  info[3] = oerr;
  if (!(oerr <= 1e-6)) {
    set_error("embedding columns not orthonormal (error %.2e)", oerr);
    return SPB_ERR_CONTRACT;
  }
  // ---- pivots (cooperative: all CTAs co-resident)
  int grid0 = num_sms();
  grid0 = (int)std::min<int64_t>(grid0, std::max<int64_t>(1, ceil_div(n, 64)));
  const int per0 = (int)ceil_div(n, grid0);
  const size_t qsmem = sizeof(double) * ((size_t)k * k + 2 * (size_t)k) + 4 * (size_t)ceil_div(per0, 32);
  if (qsmem + 9 * 1024 > 227 * 1024 || k > QKMAX) {
    set_error("QRCP supports k <= 160 columns in this build (got %d)", k);
    return SPB_ERR_CONTRACT;
  }
  SPB_CUDA(cudaFuncSetAttribute(qrcp_pivots<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)qsmem));
  int per_sm = 0;
  SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrcp_pivots<T>, QT, qsmem));
  if (per_sm < 1) {
    set_error("QRCP pivot kernel cannot be resident (k = %d)", k);
    return SPB_ERR_CONTRACT;
  }
  const int grid = grid0;
  const T* Xa = X;
  int64_t ldxa = ldx;
  int na = n, ka = k;
  double2* vnp = reinterpret_cast<double2*>(w.vn1);
  void* args[] = {(void*)&Xa, (void*)&ldxa, (void*)&na, (void*)&ka, (void*)&vnp,
                  (void*)&w.pos, (void*)&w.perm, (void*)&w.bb, (void*)&w.piv};
  SPB_CUDA(cudaLaunchCooperativeKernel((void*)qrcp_pivots<T>, grid, QT, args, qsmem, st));
  if (pivots_out)
    SPB_CUDA(cudaMemcpyAsync(pivots_out, w.piv, sizeof(int) * k, cudaMemcpyDeviceToDevice, st));
  gather_seeds<T><<<1, 256, 0, st>>>(X, ldx, k, w.piv, w.seeds, w.S);
  SPB_LAUNCH_CHECK();
  // ---- cond(S) and S^-1 (spectral.py:156-161). Fast path: Cholesky of S'S,
  // whose bracket ||G||_F ||L^-1||_F^2 / k^1.5 <= cond2(S)^2 <= ||G||_F ||L^-1||_F^2
  // settles cond2(S) <= 1e12 whenever cond2(S) <= 1e4 (the inverse is then
  // accurate to ~eps cond^2 <= 1e-8, far below label-changing ties); otherwise
  // the exact one-sided Jacobi SVD decides (and inverts), as np.linalg.cond does.
  SmallStatus hs;
  bool exact = true;
  SPB_CUDA(cudaMemsetAsync(w.status, 0, sizeof(SmallStatus), st));
  SPB_TRY(normal_eq_inverse(w.S, k, w.inv, w.jws, w.jws_cap, w.status, st));
  SPB_CUDA(cudaMemcpyAsync(&hs, w.status, sizeof(hs), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  if (!hs.not_pd && !hs.nonfinite && hs.cond_hi <= 1e8) {
    exact = false;
    info[2] = std::sqrt(hs.cond_hi);  // upper bound on cond2(S)
  }
  if (exact) {
    SPB_CUDA(cudaMemsetAsync(w.status, 0, sizeof(SmallStatus), st));
    SPB_TRY(jacobi_svd_inverse(w.S, k, w.inv, w.jws, w.jws_cap, w.status, st));
    SPB_CUDA(cudaMemcpyAsync(&hs, w.status, sizeof(hs), cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    info[2] = hs.cond_hi;
  }
  if (!(hs.cond_hi <= 1e12)) {
    set_error("seed rows numerically singular; embedding carries no clusters");
    return SPB_ERR_ASSIGNMENT;
  }
  // ---- labels
  SPB_CUDA(cudaMemsetAsync(w.present, 0, sizeof(int) * k, st));
  SPB_CUDA(cudaMemsetAsync(w.zero_rows, 0, sizeof(unsigned long long), st));
  const size_t asmem = sizeof(double) * (size_t)k * AJ;
  SPB_CUDA(cudaFuncSetAttribute(assign_rows<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(asmem, 48 * 1024)));
  assign_rows<T><<<(int)ceil_div(n, 128), 128, asmem, st>>>(X, ldx, n, k, w.inv, w.raw, w.present,
                                                            w.zero_rows);
  remap_kernel<<<1, 32, 0, st>>>(w.present, k, w.remap, w.kfound);
  compact_labels<<<(int)std::min<int64_t>(ceil_div(n, 256), 4096), 256, 0, st>>>(w.raw, n, w.remap,
                                                                              labels_out);
  SPB_LAUNCH_CHECK();
  int kf = 0;
  unsigned long long zr = 0;
  SPB_CUDA(cudaMemcpyAsync(&kf, w.kfound, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaMemcpyAsync(&zr, w.zero_rows, sizeof(zr), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  info[0] = kf;
  info[1] = (double)zr;
  return SPB_OK;
}

// ============================================================================
// Row-sharded assignment ("k sequential global argmax steps, then
// Psi and argmax are local"). Every rank holds rows [row_begin, row_end) of the
// embedding, i.e. a contiguous range of the columns of X'. Each pivot step is
// the cooperative kernel's step split at its two grid barriers into kernels,
// with the barrier replaced by an all-gather of one record per rank: the rank's
// best candidate (value, global position, global column, deferred-bound max)
// together with that column's k values, so the winner's column reaches every
// rank in the same collective that elects it. The arithmetic per column (norms,
// downdates, deferred replays, CGS2 for q_j) is the single-GPU kernel's, so the
// pivot sequence is identical for any number of ranks.
//
//   init | publish -> AG1 -> select1 | resolve | publish(if needed) -> AG2 ->
//   select2 + q_j | downdate | publish -> AG1 -> ...
// ============================================================================

struct ShardRec {  // one per rank per collective; followed by x[k] (double)
  double val, dmax;
  int pos, col, flag, pad;
};

struct QdState {
  BestRec b;        // winner of AG1
  double thr, gmax0;
  int need;         // resolve deferred columns this step (same on every rank)
  int p, pp, cj;    // pivot column, its position, column moved to position pp
};

__host__ __device__ inline size_t shard_rec_bytes(int k) {
  return (sizeof(ShardRec) + sizeof(double) * (size_t)k + 15) / 16 * 16;
}

// per-CTA candidate record + the CTA's persistent deferred bound (dpersist)
__device__ __forceinline__ void cta_publish(double bv, int bp, int bc, double dm, BestRec* cand,
                                            double* dpersist, bool reset_persist) {
  __shared__ BestRec wb[QT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int op = __shfl_xor_sync(0xffffffffu, bp, o);
    const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
    dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if (better(ov, op, bv, bp)) { bv = ov; bp = op; bc = oc; }
  }
  if (lane == 0) wb[warp] = {bv, bp, bc, dm};
  __syncthreads();
  if (tid == 0) {
    BestRec b = wb[0];
    double d = reset_persist ? b.dmax : fmax(b.dmax, dpersist[blockIdx.x]);
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      d = fmax(d, wb[w].dmax);
      if (better(wb[w].val, wb[w].pos, b.val, b.pos)) b = wb[w];
    }
    b.dmax = d;
    dpersist[blockIdx.x] = d;
    cand[blockIdx.x] = b;
  }
}

template <typename T>
__global__ void __launch_bounds__(QT)
qd_init(const T* __restrict__ X, int64_t ldx, int nl, int k, int row_begin, int per,
        double2* __restrict__ vn, int* __restrict__ pos, int* __restrict__ dirty,
        unsigned* __restrict__ mask, BestRec* __restrict__ cand, double* __restrict__ dpersist) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = tid / QG, gl = tid % QG;
  const unsigned gmask = 0xFFu << (lane & ~(QG - 1));
  const int c_lo = blockIdx.x * per, c_hi = min(nl, c_lo + per);
  double bv = -1.0;
  int bp = INT_MAX, bc = -1;
  for (int c = c_lo + tid * 32; c < c_hi; c += QT * 32) {
    const int rem = c_hi - c;
    mask[c >> 5] = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
  }
  for (int c = c_lo + grp; c < c_hi; c += QT / QG) {
    const T* x = X + (int64_t)c * ldx;
    double sq = 0.0;
    for (int t = gl; t < k; t += QG) {
      const double v = (double)x[t];
      sq = fma(v, v, sq);
    }
    sq = sqrt(group_sum(sq, gmask));
    const int gc = row_begin + c;
    if (gl == 0) {
      vn[c] = make_double2(sq, sq);
      pos[c] = gc;
      dirty[c] = -1;
    }
    if (better(sq, gc, bv, bp)) { bv = sq; bp = gc; bc = gc; }
  }
  cta_publish(bv, bp, bc, -1.0, cand, dpersist, true);
}

// The rank's best over the per-CTA records (+ its column's values) -> send.
// only_if_need: write flag 0 unless the step resolves deferred columns.
template <typename T>
__global__ void qd_publish(const T* __restrict__ X, int64_t ldx, int k, int row_begin, int ncta,
                           const BestRec* __restrict__ cand, const QdState* __restrict__ state,
                           int only_if_need, uint8_t* __restrict__ send) {
  __shared__ BestRec sb;
  ShardRec* r = reinterpret_cast<ShardRec*>(send);
  double* xr = reinterpret_cast<double*>(send + sizeof(ShardRec));
  const bool skip = only_if_need && !state->need;
  if (threadIdx.x == 0) {
    BestRec b{-1.0, INT_MAX, -1, -1.0};
    if (!skip) {
      for (int g = 0; g < ncta; ++g) {
        const BestRec c = cand[g];
        b.dmax = fmax(b.dmax, c.dmax);
        if (better(c.val, c.pos, b.val, b.pos)) { b.val = c.val; b.pos = c.pos; b.col = c.col; }
      }
    }
    sb = b;
    r->val = b.val;
    r->dmax = b.dmax;
    r->pos = b.pos;
    r->col = b.col;
    r->flag = skip ? 0 : 1;
    r->pad = 0;
  }
  __syncthreads();
  const BestRec b = sb;
  for (int t = threadIdx.x; t < k; t += blockDim.x)
    xr[t] = b.col >= 0 ? (double)X[(int64_t)(b.col - row_begin) * ldx + t] : 0.0;
}

// best over the gathered records (flagged ones only); returns the winning rank
__device__ int gathered_best(const uint8_t* __restrict__ recv, int nranks, size_t rb, BestRec* out) {
  BestRec b{-1.0, INT_MAX, -1, -1.0};
  int who = -1;
  for (int r = 0; r < nranks; ++r) {
    const ShardRec* q = reinterpret_cast<const ShardRec*>(recv + r * rb);
    if (!q->flag) continue;
    b.dmax = fmax(b.dmax, q->dmax);
    if (better(q->val, q->pos, b.val, b.pos)) { b.val = q->val; b.pos = q->pos; b.col = q->col; who = r; }
  }
  *out = b;
  return who;
}

__global__ void qd_select1(const uint8_t* __restrict__ recv, int nranks, size_t rb, int j,
                           QdState* __restrict__ state) {
  if (threadIdx.x != 0) return;
  BestRec b;
  gathered_best(recv, nranks, rb, &b);
  if (j == 0) state->gmax0 = b.val;
  state->b = b;
  state->need = (b.dmax >= b.val || b.col < 0) ? 1 : 0;
  state->thr = b.col < 0 ? -1.0 : b.val;
}

// dlaqp2's recomputes for this rank's deferred columns whose bound reaches the
// elected candidate (the cooperative kernel's resolve branch), then fresh
// per-CTA candidates over all exact unpivoted columns
template <typename T>
__global__ void __launch_bounds__(QT)
qd_resolve(const T* __restrict__ X, int64_t ldx, int nl, int k, int row_begin, int per, int j,
           const double* __restrict__ Q, const QdState* __restrict__ state, double2* __restrict__ vn,
           const int* __restrict__ pos, int* __restrict__ dirty, unsigned* __restrict__ mask,
           BestRec* __restrict__ cand, double* __restrict__ dpersist) {
  if (!state->need) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = tid / QG, gl = tid % QG;
  const unsigned gmask = 0xFFu << (lane & ~(QG - 1));
  const int c_lo = blockIdx.x * per, c_hi = min(nl, c_lo + per);
  const double thr = state->thr, tol3z = sqrt(kEps64);
  for (int c = c_lo + grp; c < c_hi; c += QT / QG) {
    const int s0 = dirty[c];
    if (s0 < 0 || pos[c] < j || !(vn[c].x >= thr)) continue;
    const T* x = X + (int64_t)c * ldx;
    double v1 = recompute_group(Q, x, k, s0, gl, gmask), v2 = v1;
    for (int st = s0 + 1; st < j; ++st) {
      if (v1 == 0.0) continue;
      const double d = dot_group(Q + (size_t)st * k, x, k, gl, gmask);
      double temp = fabs(d) / v1;
      temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
      if (temp * v1 * v1 <= tol3z * v2 * v2) {
        v1 = recompute_group(Q, x, k, st, gl, gmask);
        v2 = v1;
      } else {
        v1 = v1 * sqrt(temp);
      }
    }
    if (gl == 0) {
      vn[c] = make_double2(v1, v2);
      dirty[c] = -1;
      atomicOr(&mask[c >> 5], 1u << (c & 31));
    }
  }
  __syncthreads();
  double bv = -1.0, dm = -1.0;
  int bp = INT_MAX, bc = -1;
  for (int c = c_lo + tid; c < c_hi; c += QT) {
    if (pos[c] < j) continue;
    const double v = vn[c].x;
    if ((mask[c >> 5] >> (c & 31)) & 1u) {
      if (better(v, pos[c], bv, bp)) { bv = v; bp = pos[c]; bc = row_begin + c; }
    } else if (dirty[c] >= 0) {
      dm = fmax(dm, v);
    }
  }
  cta_publish(bv, bp, bc, dm, cand, dpersist, true);
}

// The pivot of step j (from AG2 when deferred columns were resolved, else AG1),
// dgeqp3's swap, position updates of this rank's columns, q_j (CGS2 as in the
// cooperative kernel) into Q[j].
__global__ void __launch_bounds__(QT)
qd_select2(const uint8_t* __restrict__ recv1, const uint8_t* __restrict__ recv2, int nranks,
           size_t rb, int j, int k, int row_begin, int nl, QdState* __restrict__ state,
           int* __restrict__ swap_pp, int* __restrict__ swap_cj, int* __restrict__ piv,
           double2* __restrict__ vn, int* __restrict__ pos, unsigned* __restrict__ mask,
           double* __restrict__ Q) {
  __shared__ double xp[QKMAX], cdot[QKMAX];
  __shared__ int s_who, s_use2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    BestRec b = state->b;
    int who;
    const int use2 = state->need;
    if (use2) {
      who = gathered_best(recv2, nranks, rb, &b);
    } else {
      BestRec t;
      who = gathered_best(recv1, nranks, rb, &t);
    }
    int cj = j;
    for (int t = j - 1; t >= 0; --t)
      if (swap_pp[t] == j) { cj = swap_cj[t]; break; }
    swap_pp[j] = b.pos;
    swap_cj[j] = cj;
    piv[j] = b.col;
    state->p = b.col;
    state->pp = b.pos;
    state->cj = cj;
    s_who = who;
    s_use2 = use2;
    const int p = b.col - row_begin;
    if (p >= 0 && p < nl) {
      pos[p] = j;
      vn[p].x = 0.0;
      mask[p >> 5] &= ~(1u << (p & 31));
    }
    const int c = cj - row_begin;
    if (cj != b.col && c >= 0 && c < nl) pos[c] = b.pos;
  }
  __syncthreads();
  const double* xw = reinterpret_cast<const double*>((s_use2 ? recv2 : recv1) + (size_t)s_who * rb +
                                                     sizeof(ShardRec));
  for (int t = tid; t < k; t += blockDim.x) xp[t] = xw[t];
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (int t0 = tid; t0 < j; t0 += blockDim.x) {
      const double* qt = Q + (size_t)t0 * k;
      double sd = 0.0;
      for (int t = 0; t < k; ++t) sd += qt[t] * xp[t];
      cdot[t0] = sd;
    }
    __syncthreads();
    for (int t = tid; t < k; t += blockDim.x) {
      double r = xp[t];
      for (int t0 = 0; t0 < j; ++t0) r -= cdot[t0] * Q[(size_t)t0 * k + t];
      xp[t] = r;
    }
    __syncthreads();
  }
  if (warp == 0) {
    double sq = 0.0;
    for (int t = lane; t < k; t += 32) sq += xp[t] * xp[t];
    sq = warp_sum(sq);
    const double inv = sq > 0.0 ? 1.0 / sqrt(sq) : 0.0;
    for (int t = lane; t < k; t += 32) Q[(size_t)j * k + t] = xp[t] * inv;
  }
}

// Downdate this rank's exact columns by q_j, defer the ones dlaqp2 recomputes,
// and track the next step's candidates (the cooperative kernel's main pass).
template <typename T>
__global__ void __launch_bounds__(QT)
qd_downdate(const T* __restrict__ X, int64_t ldx, int nl, int k, int row_begin, int per, int j,
            const double* __restrict__ Q, const QdState* __restrict__ state,
            double2* __restrict__ vn, const int* __restrict__ pos, int* __restrict__ dirty,
            unsigned* __restrict__ mask, BestRec* __restrict__ cand, double* __restrict__ dpersist) {
  __shared__ double qj[QKMAX];
  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = tid / QG, gl = tid % QG;
  const unsigned gmask = 0xFFu << (lane & ~(QG - 1));
  constexpr int NGRP = QT / QG;
  const int c_lo = blockIdx.x * per, c_hi = min(nl, c_lo + per);
  const int cnt = max(0, c_hi - c_lo);
  const double tol3z = sqrt(kEps64), gmax0 = state->gmax0;
  for (int t = tid; t < k; t += QT) qj[t] = Q[(size_t)j * k + t];
  __syncthreads();
  double bv = -1.0, dm = -1.0;
  int bp = INT_MAX, bc = -1;
  for (int base = grp; base < cnt; base += NGRP * QU) {
    bool act[QU];
    double2 st[QU];
    int ps[QU];
#pragma unroll
    for (int u = 0; u < QU; ++u) {
      const int c = c_lo + base + u * NGRP;
      act[u] = c < c_hi && ((mask[c >> 5] >> (c & 31)) & 1u);
      if (act[u]) {
        st[u] = vn[c];
        ps[u] = pos[c];
      }
    }
    double dots[QU];
#pragma unroll
    for (int u = 0; u < QU; ++u)
      dots[u] = act[u] ? dot_group(qj, X + (int64_t)(c_lo + base + u * NGRP) * ldx, k, gl, gmask) : 0.0;
#pragma unroll
    for (int u = 0; u < QU; ++u) {
      if (!act[u]) continue;
      const int c = c_lo + base + u * NGRP;
      double v1 = st[u].x;
      const double v2 = st[u].y;
      if (v1 != 0.0) {
        double temp = fabs(dots[u]) / v1;
        temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
        if (temp * v1 * v1 <= tol3z * v2 * v2) {
          const double bound = 2e-4 * v2 + 1e-10 * gmax0;
          dm = fmax(dm, bound);
          if (gl == 0) {
            dirty[c] = j;
            vn[c].x = bound;
            atomicAnd(&mask[c >> 5], ~(1u << (c & 31)));
          }
          continue;
        }
        v1 = v1 * sqrt(temp);
        if (gl == 0) vn[c].x = v1;
      }
      if (better(v1, ps[u], bv, bp)) { bv = v1; bp = ps[u]; bc = row_begin + c; }
    }
  }
  __syncthreads();
  cta_publish(bv, bp, bc, dm, cand, dpersist, false);
}

// Seed block S = X[sorted pivots] with only this rank's rows filled (all-reduced).
template <typename T>
__global__ void gather_seeds_local(const T* __restrict__ X, int64_t ldx, int k, int row_begin, int nl,
                                   const int* __restrict__ piv, int* __restrict__ seeds,
                                   double* __restrict__ S) {
  __shared__ int sd[1024];
  __shared__ int pv[1024];
  for (int i = threadIdx.x; i < k; i += blockDim.x) pv[i] = piv[i];
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int v = pv[i];
    int r = 0;
    for (int j = 0; j < k; ++j) r += pv[j] < v;
    sd[r] = v;
    seeds[r] = v;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) {
    const int i = x / k, t = x % k;
    const int row = sd[i] - row_begin;
    S[x] = (row >= 0 && row < nl) ? (double)X[(int64_t)row * ldx + t] : 0.0;
  }
}

__global__ void or_present(const int* __restrict__ all, int nranks, int k, int* __restrict__ present,
                           double* __restrict__ zr_local, const unsigned long long* __restrict__ zr) {
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    int v = 0;
    for (int r = 0; r < nranks; ++r) v |= all[r * k + j];
    present[j] = v ? 1 : 0;
  }
  if (threadIdx.x == 0) *zr_local = (double)*zr;
}

struct ShardAssignWs {
  AssignWs a;
  BestRec* cand;
  double *dpersist, *zr;
  unsigned* mask;
  int *swap_pp, *swap_cj, *present_all;
  QdState* state;
  uint8_t *send1, *send2, *recv1, *recv2;
  int ncta, per;
};

ShardAssignWs carve_shard_assign(Arena& a, int nl, int k, int nranks) {
  ShardAssignWs w;
  w.a = carve_assign(a, nl, k);
  w.ncta = std::max(1, std::min(2 * num_sms(), (int)ceil_div(nl, 64)));
  w.per = (int)round_up(ceil_div(nl, w.ncta), 32);
  w.ncta = (int)ceil_div(nl, w.per);
  w.cand = a.take<BestRec>(w.ncta);
  w.dpersist = a.take<double>(w.ncta);
  w.zr = a.take<double>(2);
  w.mask = a.take<unsigned>(ceil_div(nl, 32) + 1);
  w.swap_pp = a.take<int>(k);
  w.swap_cj = a.take<int>(k);
  w.present_all = a.take<int>((size_t)nranks * k);
  w.state = a.take<QdState>(1);
  const size_t rb = shard_rec_bytes(k);
  w.send1 = a.take<uint8_t>(rb);
  w.send2 = a.take<uint8_t>(rb);
  w.recv1 = a.take<uint8_t>(rb * nranks);
  w.recv2 = a.take<uint8_t>(rb * nranks);
  return w;
}

template <typename T>
int assign_sharded_t(const void* xv, int64_t ldx, int nl, int k, const spb_shard& sh,
                     const ShardAssignWs& W, int* labels_out, int* pivots_out, double* info,
                     cudaStream_t st) {
  const T* X = (const T*)xv;
  const Comm* comm = (const Comm*)sh.comm;
  const AssignWs& w = W.a;
  const int rb0 = sh.row_begin;
  // ---- orthonormality (spectral.py:149-151): local Gram, all-reduced
  GramBatch gb{};
  gb.njobs = 1;
  gb.job[0] = {X, X, ldx, ldx, k, k, 0, 0};
  gb.tile_start[0] = 0;
  gb.tile_start[1] = (int)(ceil_div(k, 64) * ceil_div(k, 64));
  SPB_TRY(gram_batched(sizeof(T) == 4 ? SPB_F32 : SPB_F64, gb, nl, k, k, w.gpart, w.gpart_cap, w.G,
                       k, st));
  SPB_TRY(comm_allreduce_f64(comm, w.G, (size_t)k * k, st));
  ortho_err_kernel<<<1, 256, 0, st>>>(w.G, k, w.ortho);
  SPB_LAUNCH_CHECK();
  double oerr = 0.0;
  SPB_CUDA(cudaMemcpyAsync(&oerr, w.ortho, sizeof(double), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  info[3] = oerr;
  if (!(oerr <= 1e-6)) {
    set_error("embedding columns not orthonormal (error %.2e)", oerr);
    return SPB_ERR_CONTRACT;
  }
  if (k > QKMAX) {
    set_error("QRCP supports k <= %d columns in this build (got %d)", QKMAX, k);
    return SPB_ERR_CONTRACT;
  }
  // ---- pivots: k global argmax steps
  const size_t rb = shard_rec_bytes(k);
  double2* vn = reinterpret_cast<double2*>(w.vn1);
  const int G = W.ncta, per = W.per;
  qd_init<T><<<G, QT, 0, st>>>(X, ldx, nl, k, rb0, per, vn, w.pos, w.perm, W.mask, W.cand, W.dpersist);
  qd_publish<T><<<1, 128, 0, st>>>(X, ldx, k, rb0, G, W.cand, W.state, 0, W.send1);
  SPB_LAUNCH_CHECK();
  for (int j = 0; j < k; ++j) {
    SPB_TRY(comm_allgather_bytes(comm, W.send1, W.recv1, rb, st));
    qd_select1<<<1, 32, 0, st>>>(W.recv1, sh.nranks, rb, j, W.state);
    qd_resolve<T><<<G, QT, 0, st>>>(X, ldx, nl, k, rb0, per, j, w.Q, W.state, vn, w.pos, w.perm,
                                    W.mask, W.cand, W.dpersist);
    qd_publish<T><<<1, 128, 0, st>>>(X, ldx, k, rb0, G, W.cand, W.state, 1, W.send2);
    SPB_LAUNCH_CHECK();
    SPB_TRY(comm_allgather_bytes(comm, W.send2, W.recv2, rb, st));
    qd_select2<<<1, QT, 0, st>>>(W.recv1, W.recv2, sh.nranks, rb, j, k, rb0, nl, W.state, W.swap_pp,
                                 W.swap_cj, w.piv, vn, w.pos, W.mask, w.Q);
    SPB_LAUNCH_CHECK();
    if (j + 1 == k) break;
    qd_downdate<T><<<G, QT, 0, st>>>(X, ldx, nl, k, rb0, per, j, w.Q, W.state, vn, w.pos, w.perm,
                                     W.mask, W.cand, W.dpersist);
    qd_publish<T><<<1, 128, 0, st>>>(X, ldx, k, rb0, G, W.cand, W.state, 0, W.send1);
    SPB_LAUNCH_CHECK();
  }
  if (pivots_out)
    SPB_CUDA(cudaMemcpyAsync(pivots_out, w.piv, sizeof(int) * k, cudaMemcpyDeviceToDevice, st));
  // ---- seed block from the owners, replicated small solves
  gather_seeds_local<T><<<1, 256, 0, st>>>(X, ldx, k, rb0, nl, w.piv, w.seeds, w.S);
  SPB_LAUNCH_CHECK();
  SPB_TRY(comm_allreduce_f64(comm, w.S, (size_t)k * k, st));
  SmallStatus hs;
  bool exact = true;
  SPB_CUDA(cudaMemsetAsync(w.status, 0, sizeof(SmallStatus), st));
  SPB_TRY(normal_eq_inverse(w.S, k, w.inv, w.jws, w.jws_cap, w.status, st));
  SPB_CUDA(cudaMemcpyAsync(&hs, w.status, sizeof(hs), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  if (!hs.not_pd && !hs.nonfinite && hs.cond_hi <= 1e8) {
    exact = false;
    info[2] = std::sqrt(hs.cond_hi);
  }
  if (exact) {
    SPB_CUDA(cudaMemsetAsync(w.status, 0, sizeof(SmallStatus), st));
    SPB_TRY(jacobi_svd_inverse(w.S, k, w.inv, w.jws, w.jws_cap, w.status, st));
    SPB_CUDA(cudaMemcpyAsync(&hs, w.status, sizeof(hs), cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    info[2] = hs.cond_hi;
  }
  if (!(hs.cond_hi <= 1e12)) {
    set_error("seed rows numerically singular; embedding carries no clusters");
    return SPB_ERR_ASSIGNMENT;
  }
  // ---- local labels; the used-label set and zero-row count over all ranks
  SPB_CUDA(cudaMemsetAsync(w.present, 0, sizeof(int) * k, st));
  SPB_CUDA(cudaMemsetAsync(w.zero_rows, 0, sizeof(unsigned long long), st));
  const size_t asmem = sizeof(double) * (size_t)k * AJ;
  SPB_CUDA(cudaFuncSetAttribute(assign_rows<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(asmem, 48 * 1024)));
  assign_rows<T><<<(int)ceil_div(nl, 128), 128, asmem, st>>>(X, ldx, nl, k, w.inv, w.raw, w.present,
                                                             w.zero_rows);
  SPB_LAUNCH_CHECK();
  SPB_TRY(comm_allgather_bytes(comm, w.present, W.present_all, sizeof(int) * (size_t)k, st));
  or_present<<<1, 256, 0, st>>>(W.present_all, sh.nranks, k, w.present, W.zr, w.zero_rows);
  SPB_LAUNCH_CHECK();
  SPB_TRY(comm_allreduce_f64(comm, W.zr, 1, st));
  remap_kernel<<<1, 32, 0, st>>>(w.present, k, w.remap, w.kfound);
  compact_labels<<<(int)std::min<int64_t>(ceil_div(nl, 256), 4096), 256, 0, st>>>(w.raw, nl, w.remap,
                                                                               labels_out);
  SPB_LAUNCH_CHECK();
  int kf = 0;
  double zr = 0.0;
  SPB_CUDA(cudaMemcpyAsync(&kf, w.kfound, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaMemcpyAsync(&zr, W.zr, sizeof(double), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  info[0] = kf;
  info[1] = zr;
  return SPB_OK;
}

}  // namespace
}  // namespace spb

using namespace spb;

extern "C" size_t spb_assign_workspace_sharded(int32_t n_local, int32_t k, int32_t nranks) {
  Arena a;
  a.dry = true;
  carve_shard_assign(a, std::max(n_local, 1), std::max(k, 1), std::max(nranks, 1));
  return a.used + 1024;
}

extern "C" int spb_assign_qrcp_sharded(int dtype, const void* x, int64_t ldx, int32_t n_local,
                                       int32_t k, const spb_shard* shard, void* ws, size_t ws_bytes,
                                       int32_t* labels_out, int32_t* pivots_out, double* info_out,
                                       void* stream) {
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  if (!shard || shard->nranks < 1 || shard->rank < 0 || shard->rank >= shard->nranks ||
      (shard->nranks > 1 && !shard->comm) || n_local < 1 || shard->row_begin < 0 ||
      (int64_t)shard->row_begin + n_local > shard->n_global) {
    set_error("inconsistent shard descriptor");
    return SPB_ERR_CONTRACT;
  }
  if (k < 1 || shard->n_global < k || ldx < k) {
    set_error("embedding needs n >= k >= 1 and ldx >= k");
    return SPB_ERR_CONTRACT;
  }
  Arena a;
  a.base = (char*)ws;
  a.cap = ws_bytes;
  ShardAssignWs w = carve_shard_assign(a, n_local, k, shard->nranks);
  if (a.used > ws_bytes) {
    set_error("assign workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  double info[4] = {0, 0, 0, 0};
  int s = dtype == SPB_F32
              ? assign_sharded_t<float>(x, ldx, n_local, k, *shard, w, labels_out, pivots_out, info,
                                        (cudaStream_t)stream)
              : assign_sharded_t<double>(x, ldx, n_local, k, *shard, w, labels_out, pivots_out, info,
                                         (cudaStream_t)stream);
  if (info_out)
    for (int i = 0; i < 4; ++i) info_out[i] = info[i];
  return s;
}

extern "C" size_t spb_assign_workspace(int32_t n, int32_t k) {
  Arena a;
  a.dry = true;
  carve_assign(a, std::max(n, 1), std::max(k, 1));
  return a.used + 1024;
}

extern "C" int spb_assign_qrcp(int dtype, const void* x, int64_t ldx, int32_t n, int32_t k,
                               void* ws, size_t ws_bytes, int32_t* labels_out,
                               int32_t* pivots_out, double* info_out, void* stream) {
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  if (k < 1 || n < k) {
    set_error("embedding needs n >= k >= 1");
    return SPB_ERR_CONTRACT;
  }
  if (ldx < k) {
    set_error("ldx < k");
    return SPB_ERR_CONTRACT;
  }
  Arena a;
  a.base = (char*)ws;
  a.cap = ws_bytes;
  AssignWs w = carve_assign(a, n, k);
  if (a.used > ws_bytes) {
    set_error("assign workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  double info[4] = {0, 0, 0, 0};
  int s = dtype == SPB_F32
              ? assign_t<float>(x, ldx, n, k, w, labels_out, pivots_out, info, (cudaStream_t)stream)
              : assign_t<double>(x, ldx, n, k, w, labels_out, pivots_out, info, (cudaStream_t)stream);
  if (info_out)
    for (int i = 0; i < 4; ++i) info_out[i] = info[i];
  return s;
}
