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
#include <vector>

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
};

__device__ __forceinline__ bool better(double v, int p, double bv, int bp) {
  return v > bv || (v == bv && p < bp);
}

// Cooperative pivot kernel: ONE grid barrier per step. Every CTA owns a
// contiguous range of columns of X' (rows of X) and keeps their partial norms
// (vn1, vn2) and current positions; after the barrier each CTA reduces the
// per-CTA maxima (double-buffered by step parity), replays the column swap
// dgeqp3 performs (perm[j] from a k-entry swap history in shared memory) and
// forms q_j redundantly (identical arithmetic on every CTA), then downdates its
// own columns and produces its next local maximum.
template <typename T>
__global__ void __launch_bounds__(QT)
qrcp_pivots(const T* __restrict__ X, int64_t ldx, int n, int k, double* __restrict__ vn1,
            double* __restrict__ vn2, int* __restrict__ pos, int* __restrict__ perm_unused,
            double* __restrict__ Q_unused, BestRec* __restrict__ bb, int* __restrict__ piv) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double qs[];         // q_0..q_{k-1} (k x k), then xp[k], cdot[k]
  double* xp = qs + (size_t)k * k;       // pivot column (then residual)
  double* cdot = xp + k;                 // q_t' r
  __shared__ BestRec wb[QT / 32];
  __shared__ int swap_pp[1024], swap_cj[1024];  // swap history (position pp, column moved)
  __shared__ int s_p, s_pp, s_cj;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int c_lo = blockIdx.x * per, c_hi = min(n, c_lo + per);
  const double tol3z = sqrt(kEps64);

  // initial norms of my columns (warp per column), positions = identity
  for (int c = c_lo + warp; c < c_hi; c += QT / 32) {
    double s = 0.0;
    for (int t = lane; t < k; t += 32) {
      const double v = (double)X[(int64_t)c * ldx + t];
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) {
      vn1[c] = sqrt(s);
      vn2[c] = vn1[c];
      pos[c] = c;
    }
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    // ---- local argmax over my remaining columns (ties: lowest position)
    double bv = -1.0;
    int bp = INT_MAX, bc = -1;
    for (int c = c_lo + tid; c < c_hi; c += QT) {
      const int p = pos[c];
      if (p < j) continue;
      const double v = vn1[c];
      if (better(v, p, bv, bp)) { bv = v; bp = p; bc = c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; bc = oc; }
    }
    if (lane == 0) wb[warp] = {bv, bp, bc};
    __syncthreads();
    BestRec* slot = bb + (j & 1) * gridDim.x;
    if (tid == 0) {
      BestRec b = wb[0];
      for (int w = 1; w < QT / 32; ++w)
        if (better(wb[w].val, wb[w].pos, b.val, b.pos)) b = wb[w];
      slot[blockIdx.x] = b;
    }
    grid.sync();
    // ---- every CTA: global pivot, swap replay, q_j
    if (tid == 0) {
      BestRec b = slot[0];
      for (int g = 1; g < (int)gridDim.x; ++g)
        if (better(slot[g].val, slot[g].pos, b.val, b.pos)) b = slot[g];
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
    if (p >= c_lo && p < c_hi && tid == 0) { pos[p] = j; vn1[p] = 0.0; }
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
    // ---- downdate my remaining columns (dlaqp2: recompute when |q_j'x|/vn1 loses digits)
    for (int c = c_lo + warp; c < c_hi; c += QT / 32) {
      if (pos[c] <= j) continue;
      const double v1 = vn1[c];
      if (v1 == 0.0) continue;
      double s = 0.0;
      for (int t = lane; t < k; t += 32) s += qj[t] * (double)X[(int64_t)c * ldx + t];
      s = warp_sum(s);
      double temp = fabs(s) / v1;
      temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
      const double r = v1 / vn2[c];
      if (temp * r * r <= tol3z) {
        double nn = 0.0;
        if (j + 1 < k) {
          double acc[8];
#pragma unroll
          for (int tt = 0; tt < 8; ++tt) {
            const int t = lane + 32 * tt;
            acc[tt] = t < k ? (double)X[(int64_t)c * ldx + t] : 0.0;
          }
          for (int t0 = 0; t0 <= j; ++t0) {
            const double* qt = qs + (size_t)t0 * k;
            double d = 0.0;
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
              const int t = lane + 32 * tt;
              if (t < k) d += qt[t] * acc[tt];
            }
            d = warp_sum(d);
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
              const int t = lane + 32 * tt;
              if (t < k) acc[tt] -= d * qt[t];
            }
          }
#pragma unroll
          for (int tt = 0; tt < 8; ++tt) nn += acc[tt] * acc[tt];
          nn = sqrt(warp_sum(nn));
        }
        if (lane == 0) {
          vn1[c] = nn;
          vn2[c] = nn;
        }
      } else if (lane == 0) {
        vn1[c] = v1 * sqrt(temp);
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void gather_seeds(const T* __restrict__ X, int64_t ldx, int k, const int* __restrict__ piv,
                             int* __restrict__ seeds, double* __restrict__ S) {
  __shared__ int sd[1024];
  if (threadIdx.x == 0) {
    for (int i = 0; i < k; ++i) sd[i] = piv[i];
    for (int i = 1; i < k; ++i) {  // insertion sort (k small)
      const int v = sd[i];
      int j = i - 1;
      while (j >= 0 && sd[j] > v) { sd[j + 1] = sd[j]; --j; }
      sd[j + 1] = v;
    }
    for (int i = 0; i < k; ++i) seeds[i] = sd[i];
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
  w.vn1 = a.take<double>(n);
  w.vn2 = a.take<double>(n);
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
  w.bb = a.take<BestRec>(4096);
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
  const size_t qsmem = sizeof(double) * ((size_t)k * k + 2 * (size_t)k);
  if (qsmem > 200 * 1024) {
    set_error("QRCP supports k <= 160 columns in this build (got %d)", k);
    return SPB_ERR_CONTRACT;
  }
  SPB_CUDA(cudaFuncSetAttribute(qrcp_pivots<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)qsmem));
  int per_sm = 0;
  SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrcp_pivots<T>, QT, qsmem));
  int grid = std::max(1, std::min(per_sm, 1)) * num_sms();
  grid = (int)std::min<int64_t>(grid, std::max<int64_t>(1, ceil_div(n, 64)));
  grid = std::min(grid, 2048);
  const T* Xa = X;
  int64_t ldxa = ldx;
  int na = n, ka = k;
  void* args[] = {(void*)&Xa, (void*)&ldxa, (void*)&na, (void*)&ka, (void*)&w.vn1,
                  (void*)&w.vn2, (void*)&w.pos, (void*)&w.perm, (void*)&w.Q, (void*)&w.bb,
                  (void*)&w.piv};
  SPB_CUDA(cudaLaunchCooperativeKernel((void*)qrcp_pivots<T>, grid, QT, args, qsmem, st));
  if (pivots_out)
    SPB_CUDA(cudaMemcpyAsync(pivots_out, w.piv, sizeof(int) * k, cudaMemcpyDeviceToDevice, st));
  gather_seeds<T><<<1, 256, 0, st>>>(X, ldx, k, w.piv, w.seeds, w.S);
  SPB_LAUNCH_CHECK();
  // ---- cond(S) and S^-1 (spectral.py:156-161)
  SPB_CUDA(cudaMemsetAsync(w.status, 0, sizeof(SmallStatus), st));
  SPB_TRY(jacobi_svd_inverse(w.S, k, w.inv, w.jws, w.jws_cap, w.status, st));
  SmallStatus hs;
  SPB_CUDA(cudaMemcpyAsync(&hs, w.status, sizeof(hs), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  info[2] = hs.cond_hi;
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

}  // namespace
}  // namespace spb

using namespace spb;

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
