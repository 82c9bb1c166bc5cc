// (d) Small dense float64 linear algebra on the device: CholQR factors and the
// projected generalized symmetric eigenproblem of the Rayleigh-Ritz step.
#pragma once
#include "common.cuh"

namespace spb {

// Status written by the small kernels (device), read by the host driver.
struct SmallStatus {
  int nonfinite;      // projected matrices contain NaN/Inf
  int not_pd;         // Cholesky of G_B (or of the CholQR Gram) failed
  int fallback;       // CholQR acceptance tests failed -> pivoted path
  int cond_state;     // 0 ok (bound), 1 ill-conditioned (bound), 2 undecided -> exact
  int rank;           // pivoted Cholesky rank
  int pad[3];
  double fro_b, fro_linv, cond_lo, cond_hi;
  double dmin, dmax, rmin, rmax;
};

constexpr double kEps64 = 2.220446049250313e-16;
constexpr double kCondMax = 67108864.0;  // 1/sqrt(eps) (lobpcg.py:35)
constexpr double kCondMaxF32 = 1e5;      // float32-storage guard on the RR basis (lobpcg.cu)

size_t sygv_ws_doubles(int m, int nev);
// G_A, G_B: device float64 m x m (ld ldg); gb may be null (B = I).
// theta: device nev; C: device m x nev (ld ldc). status: device.
// seg1 <= seg2: column-block boundaries of the basis when only the upper
// blocks of the Grams were computed (default: one block, full symmetrisation).
int sygv_enqueue(const double* ga, const double* gb, int ldg, int m, int nev, double* theta,
                 double* C, int ldc, double* ws, size_t ws_doubles, SmallStatus* status,
                 cudaStream_t st, int seg1 = 1 << 30, int seg2 = 1 << 30, bool b_ready = false);
// The G_B half of sygv_enqueue (symmetrise, Cholesky, inverse, cond bracket) on a
// side stream ordered after st's current work; sygv_enqueue(..., b_ready = true)
// with the same m / nev / ws then skips it and joins. sygv_prefactor_join makes st
// wait for it when the result ends up unused.
int sygv_prefactor_b(const double* gb, int ldg, int m, int nev, double* ws, size_t ws_doubles,
                     SmallStatus* status, cudaStream_t st, int seg1 = 1 << 30, int seg2 = 1 << 30);
int sygv_prefactor_join(cudaStream_t st);
// Exact cond2 of the symmetrised G_B (tridiagonal + bisection for the extreme
// eigenvalues), for the undecided case; writes host *cond.
int exact_cond_spd(const double* gb, int ldg, int m, double* ws, size_t ws_doubles, double* cond,
                   cudaStream_t st, int seg1 = 1 << 30, int seg2 = 1 << 30);

// CholQR factors (lobpcg.py:228-237): Rinv (na x na, upper, ld na) with
// B <- B Rinv orthonormal; status->fallback set when the reference would take
// its pivoted-QR branch.
size_t cholqr_ws_doubles(int na);
int cholqr_enqueue(const double* g, int ldg, int na, double* rinv, double* ws,
                   SmallStatus* status, cudaStream_t st);
// Pivoted Cholesky of the symmetrised Gram for the rank-revealing fallback:
// perm (device int na), rank in status->rank, Rinv of the leading rank x rank
// factor (ld na). rank_tol is relative to the largest column norm.
int pivoted_cholqr_enqueue(const double* g, int ldg, int na, double rank_tol, int* perm,
                           double* rinv, double* ws, SmallStatus* status, cudaStream_t st);

// Symmetric eigen-decomposition for small matrices used by the assignment
// step (one-sided Jacobi SVD of a k x k matrix): singular values sv[k], and
// inv = S^-1 (k x k, ld k). Returns cond via status->cond_hi.
int jacobi_svd_inverse(const double* s, int k, double* inv, double* ws, size_t ws_doubles,
                       SmallStatus* status, cudaStream_t st);
size_t jacobi_ws_doubles(int k);
// S^-1 through the normal equations with the Cholesky cond bracket of S'S in status.
int normal_eq_inverse(const double* s, int k, double* inv, double* ws, size_t ws_doubles,
                      SmallStatus* status, cudaStream_t st);

}  // namespace spb
