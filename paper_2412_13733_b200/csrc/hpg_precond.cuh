// Per-cell Schur preconditioner on the device.
//
// Reference: ObstacleDisc2D.precond_blocks / schur_hat_triple
// (assembly.py:577-603), GradientDisc2D.precond_blocks (:851-860) and
// CellBlockPreconditioner (linalg.py:246-266: scipy lu_factor / lu_solve,
// i.e. LAPACK getrf with partial pivoting and getrs).
//
//   P_e = -D_e - T(hx, hy) / alpha - beta * E_e
//
// obstacle: T = Bhat^T Ahat^{-1} Bhat (the hat triple), E_e = diag(mass_psi);
// gradient: no triple, E_e = kron(diag kx, My) + kron(Mx, diag ky) on both
// component diagonal blocks (applied only when beta != 0, as the reference).
#pragma once
#include "hpg_common.cuh"

namespace hpg {

struct PrecArgs {
  int kind;             // HPG_OBSTACLE / HPG_GRADIENT
  int n, n2, nb;        // tile side, n^2, block side
  int ncy;
  int cell0, count;     // cells [cell0, cell0 + count); block pointer is cell0's
  int transform;        // 1: blocks hold D, form P_e first
  double alpha, beta;
  const double* hx;     // device [ncx]
  const double* hy;     // device [ncy]
  const double* tri;    // obstacle: [nkeys][n2][n2]
  const int* key;       // obstacle: [N] cell -> triple key
  double* M;            // blocks, in/out
  int* ipiv;            // [count][nb], 0-based row interchanges (scipy lu_factor)
  int* info;            // device flags: |= 1 non-finite entry, |= 2 exactly zero pivot
  int* perm;            // optional [count][nb]: composed interchanges, position i <- row perm[i]
  unsigned long long* prof;  // optional per-phase cycle counters (tools/prof_precond.py)
};

// spectral mass entry (assembly.py:128-144) and stiffness diagonal (:147-153)
__device__ __forceinline__ double smass(int a, int c, double h) {
  if (a == c) return h * (1.0 / (2 * a + 1) + 1.0 / (2 * a + 5));
  if (a - c == 2 || c - a == 2) return -h / (2 * (a < c ? a : c) + 5);
  return 0.0;
}
__device__ __forceinline__ double sstiff(int a, double h) { return 4.0 * (2.0 * a + 3.0) / h; }

// Entry (row, col) of P_e from D_e's entry v.  tri_e: the cell's triple
// (obstacle; row-major n2 x n2) or null (gradient).
__device__ __forceinline__ double precond_entry(int kind, int n, int n2, double hx, double hy,
                                                double alpha, double beta, const double* tri_e,
                                                int row, int col, double v) {
  if (kind == 0) {   // HPG_OBSTACLE
    double t = -v - tri_e[(size_t)row * n2 + col] / alpha;
    if (row == col) {
      const int a = row / n, b = row - (row / n) * n;
      t -= beta * ((hx / (2.0 * a + 1.0)) * (hy / (2.0 * b + 1.0)));
    }
    return t;
  }
  double t = -v;
  if (beta != 0.0) {
    const int cr = row / n2, cc = col / n2;
    if (cr == cc) {
      const int rr = row - cr * n2, c2 = col - cc * n2;
      const int a = rr / n, b = rr - (rr / n) * n;
      const int c = c2 / n, d = c2 - (c2 / n) * n;
      const double e1 = (a == c) ? sstiff(a, hx) * smass(b, d, hy) : 0.0;
      const double e2 = (b == d) ? smass(a, c, hx) * sstiff(b, hy) : 0.0;
      t -= beta * (e1 + e2);
    }
  }
  return t;
}

// host-side launchers (hpg_precond.cu)
int launch_triple(const double* Zhat, const double* lam_hat, int n, const double* key_hx,
                  const double* key_hy, int nkeys, double* tri, cudaStream_t s);
int launch_precond_transform(const PrecArgs& A, cudaStream_t s);
int launch_lu(const PrecArgs& A, int nsm, cudaStream_t s);
int launch_lu_solve(const ElemArgs& E, const double* lu, const int* ipiv, const int* perm, int nb,
                    const double* x, double* y, cudaStream_t s);
int lu_max_nb();
// blocked LU for blocks beyond lu_max_nb() (hpg_lu_big.cu)
bool lu_big_supported(int nb);
int launch_lu_big(const PrecArgs& A, cudaStream_t s);

}  // namespace hpg
