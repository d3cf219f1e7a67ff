// U-side kernels: exact per-cell couplings through the Legendre maps
// and the deterministic assembly of cell-local U
// contributions into interior dofs (hats shared by 2 or 4 cells).
//
// Local U tile of a cell: m x m dofs in the order [hat_L, hat_R, W_0..W_{p-2}]
// per direction (spaces.py:40-43).  Per cell, exactly (assembly.py:42-116):
//   (A u)_loc  = Kx C My + Mx C Ky,  K = local stiffness, M = R^T diag(wu) R
//   (B psi)_loc = Rx^T [wx Psi wy]_pad Ry                          (obstacle)
//              = Dx^T [w2 Psi_x wy] Ry + Rx^T [wx Psi_y w2] Dy       (gradient)
//   load_vector: Rx^T Mu Ry with Mu the U-side moments of f.
#pragma once
#include "hpg_common.cuh"

namespace hpg {

struct UArgs {
  int ncx, ncy, p, n, m, nix, niy, gradient;
  long long ld, ncomp;
  const double* hx;
  const double* hy;
  const double* u;      // interior u (for A u), nullable
  double ca;            // coefficient of A u
  const double* psi_a;  // B (psi_a - psi_b); either nullable
  const double* psi_b;
  const double* mu;     // x-major m-tiles of U-side moments (load_vector), nullable
  double* scratch;      // [N][m][m]
  const double* base;   // out = cbase * base + assembled (base nullable)
  double cbase;
  double* out;
};

// Column j of R: rows with nonzeros (spaces.py:45-57).
__device__ __forceinline__ int legendre_col(int j, int* row, double* coef) {
  if (j == 0) { row[0] = 0; coef[0] = 0.5; row[1] = 1; coef[1] = -0.5; return 2; }
  if (j == 1) { row[0] = 0; coef[0] = 0.5; row[1] = 1; coef[1] = 0.5; return 2; }
  int q = j - 2;
  double s = 1.0 / (2 * q + 3);
  row[0] = q; coef[0] = s; row[1] = q + 2; coef[1] = -s;
  return 2;
}

// Column j of D (spaces.py:59-68).
__device__ __forceinline__ int deriv_col(int j, int* row, double* coef) {
  if (j == 0) { row[0] = 0; coef[0] = -0.5; return 1; }
  if (j == 1) { row[0] = 0; coef[0] = 0.5; return 1; }
  row[0] = j - 1; coef[0] = -1.0;
  return 1;
}

// Row j of the local stiffness (assembly.py:42-62).
__device__ __forceinline__ int stiff_row(int j, double h, int* col, double* coef) {
  if (j == 0) { col[0] = 0; coef[0] = 1.0 / h; col[1] = 1; coef[1] = -1.0 / h; return 2; }
  if (j == 1) { col[0] = 0; coef[0] = -1.0 / h; col[1] = 1; coef[1] = 1.0 / h; return 2; }
  col[0] = j; coef[0] = 4.0 / (h * (2 * (j - 2) + 3));
  return 1;
}

// Column k of the local mass M = R^T diag(wu) R: up to 6 (row, coef).
__device__ __forceinline__ int mass_col(int k, double h, int p, int* row, double* coef) {
  int ri[2];
  double rc[2];
  int nr = legendre_col(k, ri, rc);
  int cnt = 0;
  for (int x = 0; x < nr; ++x) {
    int i = ri[x];
    if (i > p) continue;
    double wu = h / (2.0 * i + 1.0);
    // row i of R
    int cols[3];
    double cc[3];
    int k2 = 0;
    if (i == 0) { cols[k2] = 0; cc[k2++] = 0.5; cols[k2] = 1; cc[k2++] = 0.5; }
    if (i == 1) { cols[k2] = 0; cc[k2++] = -0.5; cols[k2] = 1; cc[k2++] = 0.5; }
    if (i <= p - 2) { cols[k2] = 2 + i; cc[k2++] = 1.0 / (2 * i + 3); }
    if (i >= 2) { cols[k2] = i; cc[k2++] = -1.0 / (2 * i - 1); }
    for (int y = 0; y < k2; ++y) { row[cnt] = cols[y]; coef[cnt++] = wu * rc[x] * cc[y]; }
  }
  return cnt;
}

__device__ __forceinline__ double u_tile(const UArgs& U, int cx, int cy, int i, int j) {
  int ix = u_local_1d(cx, i, U.ncx, U.p);
  int iy = u_local_1d(cy, j, U.ncy, U.p);
  if (ix < 0 || iy < 0) return 0.0;
  return __ldg(U.u + (long long)ix * U.niy + iy);
}

__device__ __forceinline__ double dpsi(const UArgs& U, int comp, int cx, int cy, int i, int l) {
  long long idx = (long long)comp * U.ncomp + (long long)(cx * U.n + i) * U.ld + (long long)cy * U.n + l;
  double v = 0.0;
  if (U.psi_a) v = __ldg(U.psi_a + idx);
  if (U.psi_b) v -= __ldg(U.psi_b + idx);
  return v;
}

__global__ void k_u_local(UArgs U) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int m = U.m, n = U.n, p = U.p;
  long long total = (long long)U.ncx * U.ncy * m * m;
  if (tid >= total) return;
  int k = tid % m;
  long long t = tid / m;
  int j = t % m;
  int e = (int)(t / m);
  int cx = e / U.ncy, cy = e - cx * U.ncy;
  double hx = U.hx[cx], hy = U.hy[cy];
  double val = 0.0;
  if (U.u != nullptr && U.ca != 0.0) {
    int kc[2], mr[6];
    double kv[2], mv[6];
    // Kx C My
    double s1 = 0.0;
    int nk = stiff_row(j, hx, kc, kv);
    int nm = mass_col(k, hy, p, mr, mv);
    for (int x = 0; x < nk; ++x) {
      double t2 = 0.0;
      for (int y = 0; y < nm; ++y) t2 += mv[y] * u_tile(U, cx, cy, kc[x], mr[y]);
      s1 += kv[x] * t2;
    }
    // Mx C Ky
    double s2 = 0.0;
    nm = mass_col(j, hx, p, mr, mv);
    nk = stiff_row(k, hy, kc, kv);
    for (int x = 0; x < nm; ++x) {
      double t2 = 0.0;
      for (int y = 0; y < nk; ++y) t2 += kv[y] * u_tile(U, cx, cy, mr[x], kc[y]);
      s2 += mv[x] * t2;
    }
    val += U.ca * (s1 + s2);
  }
  if (U.psi_a != nullptr || U.psi_b != nullptr) {
    int ri[2], rl[2];
    double ci[2], cl[2];
    double s = 0.0;
    if (!U.gradient) {
      int ni = legendre_col(j, ri, ci), nl = legendre_col(k, rl, cl);
      for (int x = 0; x < ni; ++x) {
        if (ri[x] >= n) continue;
        double wi = hx / (2.0 * ri[x] + 1.0);
        for (int y = 0; y < nl; ++y) {
          if (rl[y] >= n) continue;
          double wl = hy / (2.0 * rl[y] + 1.0);
          s += ci[x] * cl[y] * ((wi * dpsi(U, 0, cx, cy, ri[x], rl[y])) * wl);
        }
      }
    } else {
      int ni = deriv_col(j, ri, ci), nl = legendre_col(k, rl, cl);
      for (int x = 0; x < ni; ++x) {
        if (ri[x] >= n) continue;
        double wi = 2.0 / (2.0 * ri[x] + 1.0);
        for (int y = 0; y < nl; ++y) {
          if (rl[y] >= n) continue;
          double wl = hy / (2.0 * rl[y] + 1.0);
          s += ci[x] * cl[y] * ((wi * dpsi(U, 0, cx, cy, ri[x], rl[y])) * wl);
        }
      }
      ni = legendre_col(j, ri, ci);
      nl = deriv_col(k, rl, cl);
      for (int x = 0; x < ni; ++x) {
        if (ri[x] >= n) continue;
        double wi = hx / (2.0 * ri[x] + 1.0);
        for (int y = 0; y < nl; ++y) {
          if (rl[y] >= n) continue;
          double wl = 2.0 / (2.0 * rl[y] + 1.0);
          s += ci[x] * cl[y] * ((wi * dpsi(U, 1, cx, cy, ri[x], rl[y])) * wl);
        }
      }
    }
    val += s;
  }
  if (U.mu != nullptr) {
    int ri[2], rl[2];
    double ci[2], cl[2];
    int ni = legendre_col(j, ri, ci), nl = legendre_col(k, rl, cl);
    long long ldm = (long long)U.ncy * m;
    double s = 0.0;
    for (int x = 0; x < ni; ++x)
      for (int y = 0; y < nl; ++y)
        s += ci[x] * cl[y] * __ldg(U.mu + (long long)(cx * m + ri[x]) * ldm + (long long)cy * m + rl[y]);
    val += s;
  }
  U.scratch[tid] = val;
}


__global__ void k_u_gather(UArgs U) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long total = (long long)U.nix * U.niy;
  if (tid >= total) return;
  int iy = tid % U.niy, ix = (int)(tid / U.niy);
  int cxs[2], jx[2], cys[2], ky[2];
  int nx = u_owners_1d_dev(ix, U.ncx, U.p, cxs, jx);
  int ny = u_owners_1d_dev(iy, U.ncy, U.p, cys, ky);
  const int m = U.m;
  double s = 0.0;
  for (int a = 0; a < nx; ++a)
    for (int b = 0; b < ny; ++b)
      s += U.scratch[(((long long)cxs[a] * U.ncy + cys[b]) * m + jx[a]) * m + ky[b]];
  if (U.base != nullptr) s = U.cbase * __ldg(U.base + tid) + s;
  U.out[tid] = s;
}

// B^T u alone (row-major psi order), one thread per psi dof.
__global__ void k_btu(ElemArgs A, int gradient) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int ncomp = gradient ? 2 : 1;
  long long total = A.ncomp * ncomp;
  if (tid >= total) return;
  int comp = (int)(tid / A.ncomp);
  long long rem = tid - comp * A.ncomp;
  long long row = rem / A.ld, col = rem - row * A.ld;
  int cx = (int)(row / A.n), a = (int)(row % A.n);
  int cy = (int)(col / A.n), b = (int)(col % A.n);
  double wa = A.hx[cx] / (2.0 * a + 1.0), wb = A.hy[cy] / (2.0 * b + 1.0);
  A.out[tid] = btu_value(A, gradient != 0, comp, cx, cy, a, b, wa, wb);
}

}  // namespace hpg
