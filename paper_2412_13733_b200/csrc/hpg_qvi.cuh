// Full-space U operators of the QVI temperature solve (
// hpgalerkin/qvi.py:35-127).
//
// Per cell e with U-local tile C_e (m x m, dofs [hat_L, hat_R, bubbles] per
// direction, spaces.py:40-57) of a FULL U vector (no Dirichlet restriction):
//   values:  V_e = SR C_e SR^T,            SR = Su R           (Q x m)
//   load:    G_e = hx hy TR V_e TR^T,      TR = R^T diag(1/(2l+1)) Tu (m x Q)
//   H:       (hy/hx) Kh C Mh + (hx/hy) Mh C Kh + gamma hx hy Mh C Mh,
//            Kh = h K_loc, Mh = M_loc / h (reference-cell stiffness / mass)
// so that  out = H v - load(w .* values(v) + rhs)  is the Newton residual
// (w = 0, rhs = g(gap)) or the Jacobian action (w = g'(gap) xi, rhs = 0).
// The two-sided products run as strided-batched DGEMMs; these kernels do the
// gather, the pointwise stage and the deterministic scatter-add.
#pragma once
#include <cuda_runtime.h>

namespace hpg {

struct QArgs {
  int ncx, ncy, p, m, nq, N;
  long long nfy;               // full y dofs (row stride of the full vector)
  const double* hx;
  const double* hy;
};

__device__ __forceinline__ int qfull_1d(int nc, int p, int c, int a) {
  return a == 0 ? c : (a == 1 ? c + 1 : nc + 1 + c * (p - 1) + (a - 2));
}

__global__ void k_qgather(QArgs Q, const double* __restrict__ full, double* __restrict__ C) {
  const long long total = (long long)Q.N * Q.m * Q.m;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(i / (Q.m * Q.m));
    const int rem = (int)(i - (long long)e * Q.m * Q.m);
    const int a = rem / Q.m, b = rem - (rem / Q.m) * Q.m;
    const int cx = e / Q.ncy, cy = e - (e / Q.ncy) * Q.ncy;
    const long long gx = qfull_1d(Q.ncx, Q.p, cx, a), gy = qfull_1d(Q.ncy, Q.p, cy, b);
    C[i] = full[gx * Q.nfy + gy];
  }
}

// V <- (w ? w .* V : 0) + (rhs ? rhs : 0)
__global__ void k_qpoint(long long n, double* __restrict__ V, const double* __restrict__ w,
                         const double* __restrict__ rhs) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = w ? w[i] * V[i] : 0.0;
    V[i] = rhs ? v + rhs[i] : v;
  }
}

// out[g] = sum over the cells sharing full dof g (fixed order) of
//          [(hy/hx) H1 + (hx/hy) H2 + gamma hx hy H3]  (if H1)  -  hx hy G
__global__ void k_qscatter(QArgs Q, double gamma, const double* __restrict__ H1, const double* __restrict__ H2,
                           const double* __restrict__ H3, const double* __restrict__ G, double* __restrict__ out) {
  const long long nfx = (long long)Q.ncx * Q.p + 1;
  const long long total = nfx * Q.nfy;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const int gx = (int)(g / Q.nfy), gy = (int)(g - (g / Q.nfy) * Q.nfy);
    int xc[2], xa[2], nx = 0, yc[2], ya[2], ny = 0;
    if (gx <= Q.ncx) {
      if (gx >= 1) { xc[nx] = gx - 1; xa[nx++] = 1; }
      if (gx < Q.ncx) { xc[nx] = gx; xa[nx++] = 0; }
    } else {
      const int r = gx - (Q.ncx + 1);
      xc[nx] = r / (Q.p - 1); xa[nx++] = 2 + r % (Q.p - 1);
    }
    if (gy <= Q.ncy) {
      if (gy >= 1) { yc[ny] = gy - 1; ya[ny++] = 1; }
      if (gy < Q.ncy) { yc[ny] = gy; ya[ny++] = 0; }
    } else {
      const int r = gy - (Q.ncy + 1);
      yc[ny] = r / (Q.p - 1); ya[ny++] = 2 + r % (Q.p - 1);
    }
    double s = 0.0;
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < ny; ++j) {
        const int e = xc[i] * Q.ncy + yc[j];
        const double hx = Q.hx[xc[i]], hy = Q.hy[yc[j]];
        const long long k = ((long long)e * Q.m + xa[i]) * Q.m + ya[j];
        double t = 0.0;
        if (H1) t = ((hy / hx) * H1[k] + (hx / hy) * H2[k]) + gamma * (hx * hy) * H3[k];
        if (G) t -= (hx * hy) * G[k];
        s += t;
      }
    out[g] = s;
  }
}

}  // namespace hpg
