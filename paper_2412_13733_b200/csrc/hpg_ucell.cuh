// Fused U-side work of the residual, per cell, on shared-memory tiles
// (hpgalerkin/assembly.py:42-116, 470-477, 725-729;
// proximal.py:119-125).  Every exact coupling is a product of 1D operators
// with <= 3 nonzeros per row, so each is a few sparse passes over m x m tiles:
//   B^T u   = wx (Rx C Ry^T) wy                      (obstacle)
//           = [w2 (Dx C Ry^T) wy ; wx (Rx C Dy^T) w2] (gradient)
//   A u     = Kx (C Ry^T wu Ry) + (Rx^T wu Rx C Ky^T)-form, i.e. Kx C My + Mx C Ky
//   B dpsi  = Rx^T G Ry (obstacle), Dx^T Gx Ry + Rx^T Gy Dy (gradient)
// with C the m x m local U tile, G the weighted psi_prev - psi tile.
// The cell-local b_u contribution r = -alpha A u + B (psi_prev - psi) is
// written straight to the dofs the cell owns alone (bubble x bubble) and to a
// small edge scratch for hat-involved dofs, summed by k_hat_gather in a fixed
// order (deterministic, no atomics).
#pragma once
#include "hpg_common.cuh"

namespace hpg {

// 1D sparse operators: row(i) -> up to 3 (col, coef).
struct OpR  { int p; __device__ int row(int i, int* c, double* v) const { return legendre_row(i, p, c, v); } };
struct OpD  { int p; __device__ int row(int i, int* c, double* v) const { return deriv_row(i, p, c, v); } };
struct OpRT {
  __device__ int row(int j, int* c, double* v) const {
    if (j == 0) { c[0] = 0; v[0] = 0.5; c[1] = 1; v[1] = -0.5; return 2; }
    if (j == 1) { c[0] = 0; v[0] = 0.5; c[1] = 1; v[1] = 0.5; return 2; }
    int q = j - 2;
    double s = kInvOdd[q + 1];
    c[0] = q; v[0] = s; c[1] = q + 2; v[1] = -s;
    return 2;
  }
};
struct OpDT {
  __device__ int row(int j, int* c, double* v) const {
    if (j == 0) { c[0] = 0; v[0] = -0.5; return 1; }
    if (j == 1) { c[0] = 0; v[0] = 0.5; return 1; }
    c[0] = j - 1; v[0] = -1.0;
    return 1;
  }
};
struct OpK {
  double ih;   // 1/h
  __device__ int row(int j, int* c, double* v) const {
    if (j == 0) { c[0] = 0; v[0] = ih; c[1] = 1; v[1] = -ih; return 2; }
    if (j == 1) { c[0] = 0; v[0] = -ih; c[1] = 1; v[1] = ih; return 2; }
    c[0] = j; v[0] = (4.0 * ih) * kInvOdd[j - 1];
    return 1;
  }
};

// out[i][k] = sum_i' Op[i][i'] in[i'][k]  (rows < orows, cols < ocols; in has irows rows).
// One thread per column k walks the rows: the operator row is uniform across
// the group (no divergence) and the shared-memory accesses are consecutive.
template <class Op>
__device__ __forceinline__ void apply_x(const Op& op, const double* in, int irows, double* out,
                                        int orows, int ocols, int ld, int t0, int nt) {
  for (int k = t0; k < ocols; k += nt)
    for (int i = 0; i < orows; ++i) {
      int c[3];
      double v[3];
      int nz = op.row(i, c, v);
      double s = 0.0;
      for (int z = 0; z < nz; ++z)
        if (c[z] < irows) s += v[z] * in[c[z] * ld + k];
      out[i * ld + k] = s;
    }
}

// out[i][k] = sum_k' Op[k][k'] in[i][k']  (in has icols cols).  One thread per
// row i (odd ld keeps the strided accesses bank-conflict free).
template <class Op>
__device__ __forceinline__ void apply_y(const Op& op, const double* in, int icols, double* out,
                                        int orows, int ocols, int ld, int t0, int nt) {
  for (int i = t0; i < orows; i += nt)
    for (int k = 0; k < ocols; ++k) {
      int c[3];
      double v[3];
      int nz = op.row(k, c, v);
      double s = 0.0;
      for (int z = 0; z < nz; ++z)
        if (c[z] < icols) s += v[z] * in[i * ld + c[z]];
      out[i * ld + k] = s;
    }
}

__host__ __device__ __forceinline__ int ucell_ld(int m) { return m | 1; }

// Per-thread-group U-side pass for cell (cx, cy).  sb: 4 buffers of m*ld
// doubles + n*n*NC for B^T u (result left in sBTu, row-major n x n per comp).
// SYNC is __syncwarp or __syncthreads according to the group.
template <bool GRADIENT, class Sync>
__device__ void ucell_residual(const ElemArgs& A, int e, int cx, int cy, const double* psi_tile0,
                               const double* psi_tile1, int ldt, double* sb, double* sBTu,
                               int t0, int nt, Sync sync) {
  const int m = A.m, n = A.n, p = A.p, ld = ucell_ld(m);
  double* B0 = sb;
  double* B1 = sb + m * ld;
  double* B2 = sb + 2 * m * ld;
  double* B3 = sb + 3 * m * ld;
  const double hx = A.hx[cx], hy = A.hy[cy];
  const double ihx = 1.0 / hx, ihy = 1.0 / hy;
  // (1) local U tile C (zeros on the boundary hats)
  for (int j = t0; j < m; j += nt) {
    const int iy = u_local_1d(cy, j, A.ncy, p);
    for (int i = 0; i < m; ++i) {
      const int ix = u_local_1d(cx, i, A.ncx, p);
      B0[i * ld + j] = (ix < 0 || iy < 0) ? 0.0 : __ldg(A.u + (long long)ix * A.niy + iy);
    }
  }
  sync();
  // (2) B^T u
  apply_y(OpR{p}, B0, m, B1, m, m, ld, t0, nt);          // C Ry^T
  sync();
  if (!GRADIENT) {
    apply_x(OpR{p}, B1, m, B2, n, n, ld, t0, nt);         // Rx C Ry^T
    sync();
    for (int b = t0; b < n; b += nt)
      for (int a = 0; a < n; ++a) {
      const int idx = a * n + b;
      (void)idx;
      double wa = hx * kInvOdd[a], wb = hy * kInvOdd[b];
      sBTu[idx] = (wa * B2[a * ld + b]) * wb;
    }
  } else {
    apply_x(OpD{p}, B1, m, B2, n, n, ld, t0, nt);         // Dx C Ry^T
    apply_y(OpD{p}, B0, m, B3, m, n, ld, t0, nt);         // C Dy^T
    sync();
    for (int b = t0; b < n; b += nt)
      for (int a = 0; a < n; ++a) {
      const int idx = a * n + b;
      (void)idx;
      double wb = hy * kInvOdd[b];
      sBTu[idx] = ((2.0 * kInvOdd[a]) * B2[a * ld + b]) * wb;
    }
    sync();
    apply_x(OpR{p}, B3, m, B2, n, n, ld, t0, nt);         // Rx C Dy^T
    sync();
    for (int b = t0; b < n; b += nt)
      for (int a = 0; a < n; ++a) {
      const int idx = a * n + b;
      (void)idx;
      double wa = hx * kInvOdd[a];
      sBTu[n * n + idx] = (wa * B2[a * ld + b]) * (2.0 * kInvOdd[b]);
    }
  }
  sync();
  // (3) A u = Kx (C My) + Mx (C Ky):  C My = ((C Ry^T) wu) Ry
  for (int l = t0; l < m; l += nt)
    for (int i = 0; i < m; ++i) {
    const int idx = i * m + l;
    (void)idx;
    B1[i * ld + l] *= hy * kInvOdd[l];
  }
  sync();
  apply_y(OpRT{}, B1, m, B2, m, m, ld, t0, nt);          // C My
  sync();
  apply_x(OpK{ihx}, B2, m, B3, m, m, ld, t0, nt);          // Kx C My  -> B3 (accumulator)
  apply_y(OpK{ihy}, B0, m, B1, m, m, ld, t0, nt);          // C Ky
  sync();
  apply_x(OpR{p}, B1, m, B2, m, m, ld, t0, nt);           // Rx C Ky
  sync();
  for (int k = t0; k < m; k += nt)
    for (int l = 0; l < m; ++l) {
    const int idx = l * m + k;
    (void)idx;
    B2[l * ld + k] *= hx * kInvOdd[l];
  }
  sync();
  apply_x(OpRT{}, B2, m, B1, m, m, ld, t0, nt);          // Mx C Ky
  sync();
  for (int k = t0; k < m; k += nt)
    for (int i = 0; i < m; ++i) {
    const int idx = i * m + k;
    (void)idx;
    B3[i * ld + k] += B1[i * ld + k];                     // A u (local)
  }
  // (4) B (psi_prev - psi): weighted difference tiles, zero padded to m x m
  const long long base0 = psi_index(A, cx, cy, 0, 0);
  for (int comp = 0; comp < (GRADIENT ? 2 : 1); ++comp) {
    const double* pt = comp == 0 ? psi_tile0 : psi_tile1;
    for (int l = t0; l < m; l += nt)
      for (int i = 0; i < m; ++i) {
      const int idx = i * m + l;
      (void)idx;
      double g = 0.0;
      if (i < n && l < n) {
        double d = __ldg(A.psi_prev + comp * A.ncomp + base0 + (long long)i * A.ld + l) - pt[i * ldt + l];
        double wi, wl;
        if (!GRADIENT) { wi = hx * kInvOdd[i]; wl = hy * kInvOdd[l]; }
        else if (comp == 0) { wi = 2.0 * kInvOdd[i]; wl = hy * kInvOdd[l]; }
        else { wi = hx * kInvOdd[i]; wl = 2.0 * kInvOdd[l]; }
        g = (wi * d) * wl;
      }
      B0[i * ld + l] = g;
    }
    sync();
    if (!GRADIENT || comp == 0) apply_y(OpRT{}, B0, m, B1, m, m, ld, t0, nt);    // G Ry
    else apply_y(OpDT{}, B0, m, B1, m, m, ld, t0, nt);                           // G Dy
    sync();
    if (GRADIENT && comp == 0) apply_x(OpDT{}, B1, m, B2, m, m, ld, t0, nt);     // Dx^T (.)
    else apply_x(OpRT{}, B1, m, B2, m, m, ld, t0, nt);                           // Rx^T (.)
    sync();
    for (int k = t0; k < m; k += nt)
      for (int i = 0; i < m; ++i) {
      const int idx = i * m + k;
      (void)idx;
      if (comp == 0) B3[i * ld + k] = -A.alpha * B3[i * ld + k] + B2[i * ld + k];
      else B3[i * ld + k] += B2[i * ld + k];
    }
    sync();
  }
  // (5) owned bubble x bubble dofs go straight to b_u; hat-involved ones to the edge scratch
  double* edge = A.edge + (long long)e * (4 * m - 4);
  for (int k = t0; k < m; k += nt)
    for (int j = 0; j < m; ++j) {
    const int idx = j * m + k;
    (void)idx;
    double r = B3[j * ld + k];
    if (j >= 2 && k >= 2) {
      long long ix = (A.ncx - 1) + (long long)cx * (p - 1) + (j - 2);
      long long iy = (A.ncy - 1) + (long long)cy * (p - 1) + (k - 2);
      long long g = ix * A.niy + iy;
      A.b_u[g] = A.alpha * __ldg(A.f_load + g) + r;
    } else if (j < 2) {
      edge[j * m + k] = r;
    } else {
      edge[2 * m + (j - 2) * 2 + k] = r;
    }
  }
  sync();
}

// b_u on the hat-involved interior dofs: alpha f_load + the (up to 4) cell
// contributions, summed in a fixed order.
static __global__ void k_hat_gather(ElemArgs A) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nhx = A.ncx - 1, nhy = A.ncy - 1, m = A.m;
  const long long n1 = (long long)nhx * A.niy;
  const long long n2 = (long long)(A.nix - nhx) * nhy;
  int ix, iy;
  if (tid < n1) {
    ix = (int)(tid / A.niy);
    iy = (int)(tid - (long long)ix * A.niy);
  } else if (tid < n1 + n2) {
    long long t = tid - n1;
    ix = nhx + (int)(t / nhy);
    iy = (int)(t - (long long)(ix - nhx) * nhy);
  } else {
    return;
  }
  int cxs[2], jx[2], cys[2], ky[2];
  int nx = u_owners_1d_dev(ix, A.ncx, A.p, cxs, jx);
  int ny = u_owners_1d_dev(iy, A.ncy, A.p, cys, ky);
  double s = 0.0;
  for (int a = 0; a < nx; ++a)
    for (int b = 0; b < ny; ++b) {
      int j = jx[a], k = ky[b];
      long long e = (long long)cxs[a] * A.ncy + cys[b];
      int li = j < 2 ? j * m + k : 2 * m + (j - 2) * 2 + k;
      s += A.edge[e * (4 * m - 4) + li];
    }
  long long g = (long long)ix * A.niy + iy;
  A.b_u[g] = A.alpha * __ldg(A.f_load + g) + s;
}

}  // namespace hpg
