// Schur-operator pieces on the device.
//
// * Fast-diagonalisation solve with the interior stiffness
//   A = Kx (x) My + Mx (x) Ky (assembly.py:42-78, 470-474), replacing
//   linalg.factor_stiffness / SpluFactor.solve (linalg.py:100-117): with the
//   1D generalized eigenpairs K V = M V diag(l), V^T M V = I,
//       A^{-1} b = Vx [ (Vx^T B Vy) / (lx_i + ly_j) ] Vy^T,
//   four dense GEMMs on the FP64 tensor cores (k_dgemm_nn, hpg_gemm.cuh; the
//   scaling fused into the second GEMM's epilogue).
// * The SchurOperator.matvec combine (linalg.py:223-229):
//       y = -((D x + E x) + B^T A^{-1} B x / alpha),
//   E = beta diag(mass_psi) (obstacle, assembly.py:570-575) or
//   beta blockdiag(Kx (x) My + Mx (x) Ky) per cell and component (gradient,
//   assembly.py:836-849), applied per psi dof from its cell tile.
#pragma once
#include "hpg_common.cuh"
#include "hpg_precond.cuh"

namespace hpg {

// b_psi = (phi_mom - B^T u) - M (obstacle) | (-B^T u) + M (gradient): the
// residual's last step when the U side ran concurrently (residual_concurrent)
__global__ void k_residual_combine(double* __restrict__ bpsi, const double* __restrict__ m, long long n,
                                   bool gradient) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bpsi[i] = gradient ? bpsi[i] + m[i] : bpsi[i] - m[i];
}

// y = -((yD + E x) + z / alpha) over the global psi vector
__global__ void k_schur_combine(ElemArgs A, int gradient, double alpha, double beta, const double* __restrict__ x,
                                const double* __restrict__ yD, const double* __restrict__ z,
                                double* __restrict__ y) {
  const long long total = gradient ? 2 * A.ncomp : A.ncomp;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const int comp = g >= A.ncomp ? 1 : 0;
    const long long gl = g - comp * A.ncomp;
    const int ix = (int)(gl / A.ld), iy = (int)(gl - (gl / A.ld) * A.ld);
    const int cx = ix / A.n, a = ix - cx * A.n, cy = iy / A.n, b = iy - cy * A.n;
    const double hx = A.hx[cx], hy = A.hy[cy];
    double ex;
    if (!gradient) {
      ex = (beta * ((hx / (2.0 * a + 1.0)) * (hy / (2.0 * b + 1.0)))) * x[g];
    } else {
      // (Kx (x) My + Mx (x) Ky) on the cell tile X[c][d] of this component
      const double* X = x + comp * A.ncomp + (long long)(cx * A.n) * A.ld + (long long)cy * A.n;
      double s1 = 0.0, s2 = 0.0;
      for (int d = b - 2; d <= b + 2; d += 2)
        if (d >= 0 && d < A.n) s1 += smass(b, d, hy) * X[(long long)a * A.ld + d];
      for (int c = a - 2; c <= a + 2; c += 2)
        if (c >= 0 && c < A.n) s2 += smass(a, c, hx) * X[(long long)c * A.ld + b];
      ex = beta * (sstiff(a, hx) * s1 + sstiff(b, hy) * s2);
    }
    y[g] = -((yD[g] + ex) + z[g] / alpha);
  }
}

}  // namespace hpg
