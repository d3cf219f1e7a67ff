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
};

// host-side launchers (hpg_precond.cu)
int launch_triple(const double* Zhat, const double* lam_hat, int n, const double* key_hx,
                  const double* key_hy, int nkeys, double* tri, cudaStream_t s);
int launch_precond_transform(const PrecArgs& A, cudaStream_t s);
int launch_lu(const PrecArgs& A, int nsm, cudaStream_t s);
int launch_lu_solve(const ElemArgs& E, const double* lu, const int* ipiv, int nb, const double* x,
                    double* y, cudaStream_t s);
int lu_max_nb();

}  // namespace hpg
