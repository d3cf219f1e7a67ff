// Fused U-side work of the residual, per cell, on shared-memory tiles
// (hpgalerkin/assembly.py:42-116, 470-477, 725-729;
// proximal.py:119-125).  Every exact coupling is a product of reference-cell
// 1D operators with <= 5 nonzeros per row (tables built once per plan,
// hpgPlanCreate), scaled by the cell widths:
//   B^T u  = wx (R C R^T) wy                          (obstacle)
//          = [w2 (D C R^T) wy ; wx (R C D^T) w2]      (gradient)
//   A u    = Kx C My + Mx C Ky,  K = Kref / h, M = h Mref, Mref = R^T diag(1/(2l+1)) R
//   B dpsi = R^T G R  (obstacle),  D^T Gx R + R^T Gy D  (gradient)
// with C the m x m local U tile and G the weighted psi_prev - psi tile.
// r = -alpha A u + B (psi_prev - psi) is written straight to the dofs the
// cell owns alone (bubble x bubble) and to a small edge scratch for the
// hat-involved dofs, which k_hat_gather sums in a fixed order
// (deterministic, no atomics).
#pragma once
#include "hpg_common.cuh"

namespace hpg {

// Explicit 1D operator passes on m x m tiles (row stride ld).  The operators
// (reference cell; spaces.py:45-68, assembly.py:42-62):
//   R  [a][i]: a=0: (0:.5)(1:.5); a=1: (0:-.5)(1:.5); a<=p-2: (a+2: 1/(2a+3));
//              a>=2: (a: -1/(2a-1))                         U dofs -> Legendre
//   RT = R^T   D [i][j]: i=0: (0:-.5)(1:.5); i>=1: (i+1: -1)  DT = D^T
//   K  [j][j']: hats [[1,-1],[-1,1]], bubble j: 4/(2j-1)      (times 1/h)
// X-passes: one thread per column k walks the rows; Y-passes: one thread per
// row i walks the columns.  All coefficients are kInvOdd constants.
enum UOp : int { OP_R = 0, OP_RT = 1, OP_D = 2, OP_DT = 3, OP_K = 4 };

// Value of (Op v)[i] where v(j) returns the input along the pass direction
// (zero outside [0, len)).
template <int OP, class V>
__device__ __forceinline__ double op_row(int i, int p, const double* kInvOdd, V v) {
  if constexpr (OP == OP_R) {
    if (i == 0) return 0.5 * (v(0) + v(1)) + (p >= 2 ? kInvOdd[1] * v(2) : 0.0);
    if (i == 1) return 0.5 * (v(1) - v(0)) + (p >= 3 ? kInvOdd[2] * v(3) : 0.0);
    return (i <= p - 2 ? kInvOdd[i + 1] * v(i + 2) : 0.0) - kInvOdd[i - 1] * v(i);
  } else if constexpr (OP == OP_RT) {
    if (i == 0) return 0.5 * (v(0) - v(1));
    if (i == 1) return 0.5 * (v(0) + v(1));
    return kInvOdd[i - 1] * (v(i - 2) - v(i));
  } else if constexpr (OP == OP_D) {
    if (i == 0) return 0.5 * (v(1) - v(0));
    return -v(i + 1);
  } else if constexpr (OP == OP_DT) {
    if (i == 0) return -0.5 * v(0);
    if (i == 1) return 0.5 * v(0);
    return -v(i - 1);
  } else {  // OP_K
    if (i == 0) return v(0) - v(1);
    if (i == 1) return v(1) - v(0);
    return (4.0 * kInvOdd[i - 1]) * v(i);
  }
}

// out[i][k] (+)= scale * (Op in)[i][k]  for i < orows, k < ocols; in has irows valid rows.
// rowscale: optional per-output-row factor (e.g. the Legendre mass 1/(2l+1)).
template <int OP>
__device__ __forceinline__ void pass_x(const double* in, int irows, double* out, int orows, int ocols,
                                       int ld, int p, double scale, bool accum, bool rowmass,
                                       int t0, int nt) {
  const double* inv = kInvOdd;
  for (int k = t0; k < ocols; k += nt)
    for (int i = 0; i < orows; ++i) {
      double s = op_row<OP>(i, p, inv, [&](int j) { return (j >= 0 && j < irows) ? in[j * ld + k] : 0.0; });
      s *= rowmass ? scale * kInvOdd[i] : scale;
      out[i * ld + k] = accum ? out[i * ld + k] + s : s;
    }
}

template <int OP>
__device__ __forceinline__ void pass_y(const double* in, int icols, double* out, int orows, int ocols,
                                       int ld, int p, double scale, bool accum, bool colmass,
                                       int t0, int nt) {
  const double* inv = kInvOdd;
  for (int i = t0; i < orows; i += nt)
    for (int k = 0; k < ocols; ++k) {
      double s = op_row<OP>(k, p, inv, [&](int j) { return (j >= 0 && j < icols) ? in[i * ld + j] : 0.0; });
      s *= colmass ? scale * kInvOdd[k] : scale;
      out[i * ld + k] = accum ? out[i * ld + k] + s : s;
    }
}

__host__ __device__ __forceinline__ int ucell_ld(int m) { return m | 1; }

// Per-thread-group U-side pass for cell (cx, cy).  sb: 4 buffers of m*ld
// doubles; sBTu: n*n per psi component (result, row-major).
template <bool GRADIENT, class Sync>
__device__ void ucell_residual(const ElemArgs& A, int e, int cx, int cy,
                               const double* psi_tile0, const double* psi_tile1, int ldt,
                               double* sb, double* sBTu, int t0, int nt, Sync sync) {
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
  const long long base0 = psi_index(A, cx, cy, 0, 0);
  if (!GRADIENT) {
    pass_y<OP_R>(B0, m, B1, m, n, ld, p, 1.0, false, false, t0, nt);     // C R^T   (m x n)
    sync();
    pass_x<OP_R>(B1, m, B2, n, n, ld, p, 1.0, false, false, t0, nt);     // R C R^T (n x n)
    sync();
    for (int b = t0; b < n; b += nt)
      for (int a = 0; a < n; ++a) {
        const double btu = ((hx * kInvOdd[a]) * B2[a * ld + b]) * (hy * kInvOdd[b]);
        if (sBTu != nullptr) {
          sBTu[a * n + b] = btu;
        } else {
          // standalone: b_psi <- phi_moments - B^T u (proximal.py:123 order)
          const long long g = base0 + (long long)a * A.ld + b;
          A.out[g] = __ldg(A.phi_mom + g) - btu;
        }
      }
  } else {
    pass_y<OP_R>(B0, m, B1, m, n, ld, p, 1.0, false, false, t0, nt);     // C R^T
    pass_y<OP_D>(B0, m, B3, m, n, ld, p, 1.0, false, false, t0, nt);     // C D^T
    sync();
    pass_x<OP_D>(B1, m, B2, n, n, ld, p, 1.0, false, false, t0, nt);     // D C R^T
    sync();
    pass_x<OP_R>(B3, m, B1, n, n, ld, p, 1.0, false, false, t0, nt);     // R C D^T
    sync();
    for (int b = t0; b < n; b += nt)
      for (int a = 0; a < n; ++a) {
        const double bx = ((2.0 * kInvOdd[a]) * B2[a * ld + b]) * (hy * kInvOdd[b]);
        const double by = ((hx * kInvOdd[a]) * B1[a * ld + b]) * (2.0 * kInvOdd[b]);
        if (sBTu != nullptr) {
          sBTu[a * n + b] = bx;
          sBTu[n * n + a * n + b] = by;
        } else {
          const long long g = base0 + (long long)a * A.ld + b;
          A.out[g] = -bx;
          A.out[A.ncomp + g] = -by;
        }
      }
  }
  sync();
  // (3) A u = Kx (C My) + Mx (C Ky) -> B3, with My = hy R^T diag(1/(2l+1)) R
  pass_y<OP_R>(B0, m, B1, m, m, ld, p, hy, false, true, t0, nt);       // (C R^T) hy/(2l+1)
  pass_y<OP_K>(B0, m, B2, m, m, ld, p, ihy, false, false, t0, nt);     // C Ky
  sync();
  pass_y<OP_RT>(B1, m, B0, m, m, ld, p, 1.0, false, false, t0, nt);    // C My  (C no longer needed)
  pass_x<OP_R>(B2, m, B1, m, m, ld, p, hx, false, true, t0, nt);       // hx/(2l+1) R (C Ky)
  sync();
  pass_x<OP_K>(B0, m, B3, m, m, ld, p, ihx, false, false, t0, nt);     // Kx C My
  pass_x<OP_RT>(B1, m, B3, m, m, ld, p, 1.0, true, false, t0, nt);     // + Mx C Ky
  sync();
  // (4) B (psi_prev - psi): weighted difference tiles, zero padded to m x m -> B2
  for (int comp = 0; comp < (GRADIENT ? 2 : 1); ++comp) {
    const double* pt = comp == 0 ? psi_tile0 : psi_tile1;
    for (int l = t0; l < m; l += nt)
      for (int i = 0; i < m; ++i) {
        double g = 0.0;
        if (i < n && l < n) {
          const long long gi = comp * A.ncomp + base0 + (long long)i * A.ld + l;
          double d = __ldg(A.psi_prev + gi) - (pt != nullptr ? pt[i * ldt + l] : __ldg(A.in0 + gi));
          double wi, wl;
          if (!GRADIENT) { wi = hx * kInvOdd[i]; wl = hy * kInvOdd[l]; }
          else if (comp == 0) { wi = 2.0 * kInvOdd[i]; wl = hy * kInvOdd[l]; }
          else { wi = hx * kInvOdd[i]; wl = 2.0 * kInvOdd[l]; }
          g = (wi * d) * wl;
        }
        B0[i * ld + l] = g;
      }
    sync();
    if (GRADIENT && comp == 1) pass_y<OP_DT>(B0, n, B1, m, m, ld, p, 1.0, false, false, t0, nt);  // G D
    else pass_y<OP_RT>(B0, n, B1, m, m, ld, p, 1.0, false, false, t0, nt);                     // G R
    sync();
    if (GRADIENT && comp == 0) pass_x<OP_DT>(B1, n, B2, m, m, ld, p, 1.0, false, false, t0, nt);  // D^T (.)
    else pass_x<OP_RT>(B1, n, B2, m, m, ld, p, 1.0, comp > 0, false, t0, nt);                    // R^T (.)
    sync();
  }
  // (5) r = -alpha A u + B dpsi: owned bubble x bubble dofs straight to b_u,
  //     hat-involved ones to the edge scratch
  double* edge = A.edge + (long long)e * (4 * m - 4);
  for (int k = t0; k < m; k += nt)
    for (int j = 0; j < m; ++j) {
      double r = -A.alpha * B3[j * ld + k] + B2[j * ld + k];
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

// Standalone U side (runs before the psi-side quadrature, which then
// finishes b_psi in place: ElemArgs.residual == 2).  A 128-thread CTA owns
// UCPB cells at a time.  Every pass is thread-per-entry over a shared-memory
// (i,k) index table (no divisions) with the 1D operator rows compressed to 5
// (col, val) slots in shared memory (branch-free), so all lanes do useful
// work; intermediate tiles stay in shared memory.
constexpr int USIDE_THREADS = 128;
constexpr int UNOPS = 5;   // OP_R, OP_RT, OP_D, OP_DT, OP_K

struct USmem {
  int m, n, ld, buf;
  const int* col;       // [UNOPS][m][5]
  const double* val;    // [UNOPS][m][5]
  const int* tab_mm;    // packed (i<<8)|k, m*m entries
  const int* tab_mn;    // m*n
  const int* tab_nn;    // n*n
};

// out[c][i][k] (+)= f_c * (Op in)  over the (i, k) of tab (cnt entries).
// XDIR: Op acts on the row index i; else on the column index k.
// mass: extra factor 1/(2l+1) on the operator's output index l.
template <bool XDIR>
__device__ __forceinline__ void upass3(const USmem& S, int op, const double* in, double* out,
                                       const int* tab, int cnt, int ncell, const double* fc,
                                       const double* inv, bool mass, bool accum) {
  for (int c = 0; c < ncell; ++c) {
    const double* src = in + c * S.buf;
    double* dst = out + c * S.buf;
    const double f = fc[c];
    for (int t = threadIdx.x; t < cnt; t += USIDE_THREADS) {
      const int pk = tab[t], i = pk >> 8, k = pk & 255;
      const int row = XDIR ? i : k;
      const int* cl = S.col + (op * S.m + row) * 5;
      const double* vl = S.val + (op * S.m + row) * 5;
      double s = 0.0;
#pragma unroll
      for (int z = 0; z < 5; ++z) s += vl[z] * (XDIR ? src[cl[z] * S.ld + k] : src[i * S.ld + cl[z]]);
      s *= mass ? f * inv[row] : f;
      double* o = dst + i * S.ld + k;
      *o = accum ? *o + s : s;
    }
  }
}

template <bool GRADIENT>
__global__ void __launch_bounds__(USIDE_THREADS) k_uside(ElemArgs A, int cpb) {
  extern __shared__ double smem[];
  const int m = A.m, n = A.n, p = A.p, ld = ucell_ld(m), buf = m * ld;
  double* B0 = smem;
  double* B1 = B0 + cpb * buf;
  double* B2 = B1 + cpb * buf;
  double* B3 = B2 + cpb * buf;
  double* sh = B3 + cpb * buf;           // per-cell scale factors [8][cpb]
  double* shx = sh;
  double* shy = sh + cpb;
  double* sihx = sh + 2 * cpb;
  double* sihy = sh + 3 * cpb;
  double* sone = sh + 4 * cpb;
  int* scx = reinterpret_cast<int*>(sh + 5 * cpb);
  int* scy = scx + cpb;
  double* sinv = sh + 8 * cpb;           // 1/(2k+1), k < 2m+8
  double* sval = sinv + 2 * m + 8;       // [UNOPS][m][5]
  int* icol = reinterpret_cast<int*>(sval + UNOPS * m * 5);
  int* tmm = icol + UNOPS * m * 5;
  int* tmn = tmm + m * m;
  int* tnn = tmn + m * n;
  for (int k = threadIdx.x; k < 2 * m + 8; k += blockDim.x) sinv[k] = kInvOdd[k];
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) tmm[t] = ((t / m) << 8) | (t % m);
  for (int t = threadIdx.x; t < m * n; t += blockDim.x) tmn[t] = ((t / n) << 8) | (t % n);
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) tnn[t] = ((t / n) << 8) | (t % n);
  // compressed operator rows: probe op_row with unit vectors (once per CTA)
  for (int r = threadIdx.x; r < UNOPS * m; r += blockDim.x) {
    const int op = r / m, i = r - op * m;
    int cnt = 0;
    for (int j = 0; j < m && cnt < 5; ++j) {
      auto unit = [&](int jj) { return jj == j ? 1.0 : 0.0; };
      double v;
      switch (op) {
        case OP_R: v = (i < m) ? op_row<OP_R>(i, p, kInvOdd, unit) : 0.0; break;
        case OP_RT: v = op_row<OP_RT>(i, p, kInvOdd, unit); break;
        case OP_D: v = (i < p) ? op_row<OP_D>(i, p, kInvOdd, unit) : 0.0; break;
        case OP_DT: v = op_row<OP_DT>(i, p, kInvOdd, unit); break;
        default: v = op_row<OP_K>(i, p, kInvOdd, unit); break;
      }
      if (v != 0.0) { icol[r * 5 + cnt] = j; sval[r * 5 + cnt] = v; ++cnt; }
    }
    for (; cnt < 5; ++cnt) { icol[r * 5 + cnt] = 0; sval[r * 5 + cnt] = 0.0; }
  }
  USmem S{m, n, ld, buf, icol, sval, tmm, tmn, tnn};

  for (int e0 = blockIdx.x * cpb; e0 < A.N; e0 += gridDim.x * cpb) {
    const int nc = A.N - e0 < cpb ? A.N - e0 : cpb;
    __syncthreads();
    if (threadIdx.x < cpb) {
      const int c = threadIdx.x;
      const int e = e0 + (c < nc ? c : 0);
      const int cx = e / A.ncy, cy = e - cx * A.ncy;
      shx[c] = A.hx[cx];
      shy[c] = A.hy[cy];
      sihx[c] = 1.0 / A.hx[cx];
      sihy[c] = 1.0 / A.hy[cy];
      sone[c] = 1.0;
      scx[c] = cx;
      scy[c] = cy;
    }
    __syncthreads();
    // (1) C tiles; (psi_prev - psi) weighted tiles G (obstacle: B3; gradient: B2/B3 later)
    for (int c = 0; c < nc; ++c) {
      const int cx = scx[c], cy = scy[c];
      for (int t = threadIdx.x; t < m * m; t += USIDE_THREADS) {
        const int pk = tmm[t], i = pk >> 8, j = pk & 255;
        const int ix = u_local_1d(cx, i, A.ncx, p), iy = u_local_1d(cy, j, A.ncy, p);
        B0[c * buf + i * ld + j] = (ix < 0 || iy < 0) ? 0.0 : __ldg(A.u + (long long)ix * A.niy + iy);
      }
    }
    __syncthreads();
    // (2) B^T u -> b_psi = phi_moments - B^T u (obstacle) | -B^T u (gradient)
    if (!GRADIENT) {
      upass3<false>(S, OP_R, B0, B1, tmn, m * n, nc, sone, sinv, false, false);   // C R^T
      __syncthreads();
      upass3<true>(S, OP_R, B1, B2, tnn, n * n, nc, sone, sinv, false, false);    // R C R^T
      __syncthreads();
      for (int c = 0; c < nc; ++c) {
        const int cx = scx[c], cy = scy[c];
        for (int t = threadIdx.x; t < n * n; t += USIDE_THREADS) {
          const int pk = tnn[t], a = pk >> 8, b = pk & 255;
          const long long g = psi_index(A, cx, cy, a, b);
          const double btu = ((shx[c] * sinv[a]) * B2[c * buf + a * ld + b]) * (shy[c] * sinv[b]);
          A.out[g] = __ldg(A.phi_mom + g) - btu;
        }
      }
    } else {
      upass3<false>(S, OP_R, B0, B1, tmn, m * n, nc, sone, sinv, false, false);   // C R^T
      upass3<false>(S, OP_D, B0, B3, tmn, m * n, nc, sone, sinv, false, false);   // C D^T
      __syncthreads();
      upass3<true>(S, OP_D, B1, B2, tnn, n * n, nc, sone, sinv, false, false);    // D C R^T
      __syncthreads();
      upass3<true>(S, OP_R, B3, B1, tnn, n * n, nc, sone, sinv, false, false);    // R C D^T (B1 free now)
      __syncthreads();
      for (int c = 0; c < nc; ++c) {
        const int cx = scx[c], cy = scy[c];
        for (int t = threadIdx.x; t < n * n; t += USIDE_THREADS) {
          const int pk = tnn[t], a = pk >> 8, b = pk & 255;
          const long long g = psi_index(A, cx, cy, a, b);
          A.out[g] = -(((2.0 * sinv[a]) * B2[c * buf + a * ld + b]) * (shy[c] * sinv[b]));
          A.out[A.ncomp + g] = -(((shx[c] * sinv[a]) * B1[c * buf + a * ld + b]) * (2.0 * sinv[b]));
        }
      }
    }
    __syncthreads();
    // (3) A u = Kx (C My) + Mx (C Ky) -> B3, My = hy R^T diag(1/(2l+1)) R
    upass3<false>(S, OP_R, B0, B1, tmm, m * m, nc, shy, sinv, true, false);     // (C R^T) hy/(2l+1)
    upass3<false>(S, OP_K, B0, B2, tmm, m * m, nc, sihy, sinv, false, false);   // C Ky
    __syncthreads();
    upass3<false>(S, OP_RT, B1, B0, tmm, m * m, nc, sone, sinv, false, false);  // C My
    upass3<true>(S, OP_R, B2, B1, tmm, m * m, nc, shx, sinv, true, false);      // hx/(2l+1) R C Ky
    __syncthreads();
    upass3<true>(S, OP_K, B0, B3, tmm, m * m, nc, sihx, sinv, false, false);    // Kx C My
    __syncthreads();
    upass3<true>(S, OP_RT, B1, B3, tmm, m * m, nc, sone, sinv, false, true);    // + Mx C Ky
    // (4) B (psi_prev - psi) -> B2
    for (int comp = 0; comp < (GRADIENT ? 2 : 1); ++comp) {
      for (int c = 0; c < nc; ++c) {
        const int cx = scx[c], cy = scy[c];
        for (int t = threadIdx.x; t < m * m; t += USIDE_THREADS) {
          const int pk = tmm[t], i = pk >> 8, l = pk & 255;
          double g = 0.0;
          if (i < n && l < n) {
            const long long gi = comp * A.ncomp + psi_index(A, cx, cy, i, l);
            const double d = __ldg(A.psi_prev + gi) - __ldg(A.in0 + gi);
            double wi, wl;
            if (!GRADIENT) { wi = shx[c] * sinv[i]; wl = shy[c] * sinv[l]; }
            else if (comp == 0) { wi = 2.0 * sinv[i]; wl = shy[c] * sinv[l]; }
            else { wi = shx[c] * sinv[i]; wl = 2.0 * sinv[l]; }
            g = (wi * d) * wl;
          }
          B0[c * buf + i * ld + l] = g;
        }
      }
      __syncthreads();
      upass3<false>(S, (GRADIENT && comp == 1) ? OP_DT : OP_RT, B0, B1, tmm, m * m, nc, sone, sinv, false, false);
      __syncthreads();
      upass3<true>(S, (GRADIENT && comp == 0) ? OP_DT : OP_RT, B1, B2, tmm, m * m, nc, sone, sinv, false, comp > 0);
      __syncthreads();
    }
    // (5) r = -alpha A u + B dpsi -> owned dofs (b_u) and edge scratch
    for (int c = 0; c < nc; ++c) {
      const int cx = scx[c], cy = scy[c], e = e0 + c;
      for (int t = threadIdx.x; t < m * m; t += USIDE_THREADS) {
        const int pk = tmm[t], j = pk >> 8, k = pk & 255;
        const double rr = -A.alpha * B3[c * buf + j * ld + k] + B2[c * buf + j * ld + k];
        if (j >= 2 && k >= 2) {
          const long long ix = (A.ncx - 1) + (long long)cx * (p - 1) + (j - 2);
          const long long iy = (A.ncy - 1) + (long long)cy * (p - 1) + (k - 2);
          const long long g = ix * A.niy + iy;
          A.b_u[g] = A.alpha * __ldg(A.f_load + g) + rr;
        } else {
          double* edge = A.edge + (long long)e * (4 * m - 4);
          if (j < 2) edge[j * m + k] = rr;
          else edge[2 * m + (j - 2) * 2 + k] = rr;
        }
      }
    }
  }
}

__host__ __device__ inline size_t uside_smem_doubles(int m, int n, int cpb) {
  const int ld = m | 1;
  size_t d = (size_t)4 * cpb * m * ld + 8 * (size_t)cpb + 2 * (size_t)m + 8 + (size_t)UNOPS * m * 5;
  size_t ints = (size_t)UNOPS * m * 5 + (size_t)m * m + (size_t)m * n + (size_t)n * n;
  return d + (ints + 1) / 2 + 4;
}

// ---------------------------------------------------------------------------
// Thread-per-entry U side: one CTA per cell, thread (j, k) computes its b_u
// contribution and, for j, k < n, its B^T u entry straight from the sparse
// 1D factors (L1-resident gathers of the cell's u / psi tiles; no shared
// memory, no barriers, no intermediate tiles).
struct Sp3 { int i[3]; double v[3]; int n; };

// column j of R (U dof j -> Legendre coefficients): 2 entries
template <class Inv>
__device__ __forceinline__ Sp3 r_col(int j, Inv inv_odd) {
  Sp3 s; s.n = 2;
  if (j == 0) { s.i[0] = 0; s.v[0] = 0.5; s.i[1] = 1; s.v[1] = -0.5; }
  else if (j == 1) { s.i[0] = 0; s.v[0] = 0.5; s.i[1] = 1; s.v[1] = 0.5; }
  else { const double t = inv_odd(j - 1); s.i[0] = j - 2; s.v[0] = t; s.i[1] = j; s.v[1] = -t; }
  s.i[2] = 0; s.v[2] = 0.0;
  return s;
}
// row a of R: up to 3 entries
template <class Inv>
__device__ __forceinline__ Sp3 r_row(int a, int p, Inv inv_odd) {
  Sp3 s;
  s.i[0] = s.i[1] = s.i[2] = 0;
  s.v[0] = s.v[1] = s.v[2] = 0.0;
  if (a < 2) {
    s.i[0] = 0; s.v[0] = a == 0 ? 0.5 : -0.5;
    s.i[1] = 1; s.v[1] = 0.5;
    s.i[2] = a + 2; s.v[2] = (a <= p - 2) ? inv_odd(a + 1) : 0.0;
  } else {
    s.i[0] = a; s.v[0] = -inv_odd(a - 1);
    s.i[1] = (a <= p - 2) ? a + 2 : a; s.v[1] = (a <= p - 2) ? inv_odd(a + 1) : 0.0;
  }
  s.n = 3;
  return s;
}
// column j / row i of D
__device__ __forceinline__ Sp3 d_col(int j) {
  Sp3 s; s.n = 1;
  s.i[1] = s.i[2] = 0; s.v[1] = s.v[2] = 0.0;
  if (j == 0) { s.i[0] = 0; s.v[0] = -0.5; }
  else if (j == 1) { s.i[0] = 0; s.v[0] = 0.5; }
  else { s.i[0] = j - 1; s.v[0] = -1.0; }
  return s;
}
__device__ __forceinline__ Sp3 d_row(int i) {
  Sp3 s; s.n = 2; s.i[2] = 0; s.v[2] = 0.0;
  if (i == 0) { s.i[0] = 0; s.v[0] = -0.5; s.i[1] = 1; s.v[1] = 0.5; }
  else { s.i[0] = i + 1; s.v[0] = -1.0; s.i[1] = i + 1; s.v[1] = 0.0; }
  return s;
}
// row j of Kref = h * stiffness
template <class Inv>
__device__ __forceinline__ Sp3 k_row(int j, Inv inv_odd) {
  Sp3 s; s.n = 2; s.i[2] = 0; s.v[2] = 0.0;
  if (j == 0) { s.i[0] = 0; s.v[0] = 1.0; s.i[1] = 1; s.v[1] = -1.0; }
  else if (j == 1) { s.i[0] = 0; s.v[0] = -1.0; s.i[1] = 1; s.v[1] = 1.0; }
  else { s.i[0] = j; s.v[0] = 4.0 * inv_odd(j - 1); s.i[1] = j; s.v[1] = 0.0; }
  return s;
}

template <bool GRADIENT>
__global__ void __launch_bounds__(1024) k_uside_pt(ElemArgs A, int cpb, int TG, int usplit) {
  pdl_wait();
  // cpb cell groups of TG threads per CTA (small tiles share a CTA); with few
  // large cells (cpb == 1, config 3) usplit CTAs share one cell's entries
  // (each stages the whole tile, then takes every usplit-th block of TG)
  extern __shared__ double smem[];
  const int m = A.m, n = A.n, p = A.p, ld = m | 1;
  const int grp = threadIdx.x / TG;
  const int sp = blockIdx.x % usplit;
  const int t0 = threadIdx.x - grp * TG;
  const int tstart = t0 + sp * TG, tstep = TG * usplit;
  double* sI = smem;                                   // 1/(2k+1)
  for (int t = threadIdx.x; t < 2 * m + 8; t += blockDim.x) sI[t] = kInvOdd[t];
  const int e = (blockIdx.x / usplit) * cpb + grp;
  const bool valid = grp < cpb && e < A.N;
  const int ee = valid ? e : 0;
  const int cx = ee / A.ncy, cy = ee - cx * A.ncy;
  const double hx = A.hx[cx], hy = A.hy[cy];
  const long long base0 = psi_index(A, cx, cy, 0, 0);
  double* sC = smem + 2 * m + 8 + (size_t)(grp < cpb ? grp : 0) * (m * ld + 2 * n * n);  // m x ld U tile
  double* sG = sC + m * ld;               // [comp][n][n] weighted psi_prev - psi
  for (int t = valid ? t0 : m * m; t < m * m; t += TG) {
    const int i = t / m, l = t - i * m;
    sC[i * ld + l] = u_at(A, cx, cy, i, l);
  }
  for (int t = valid ? t0 : n * n * 2; t < n * n * (GRADIENT ? 2 : 1); t += TG) {
    const int comp = t / (n * n), r = t - comp * n * n, i = r / n, l = r - i * n;
    const long long gi = comp * A.ncomp + base0 + (long long)i * A.ld + l;
    const double d = __ldg(A.psi_prev + gi) - __ldg(A.in0 + gi);
    double wi, wl;
    if (!GRADIENT) { wi = hx * kInvOdd[i]; wl = hy * kInvOdd[l]; }
    else if (comp == 0) { wi = 2.0 * kInvOdd[i]; wl = hy * kInvOdd[l]; }
    else { wi = hx * kInvOdd[i]; wl = 2.0 * kInvOdd[l]; }
    sG[t] = (wi * d) * wl;
  }
  __syncthreads();
  auto C = [&](int i, int l) { return sC[i * ld + l]; };
  auto inv = [&](int k) { return sI[k]; };
  for (int t = valid ? tstart : m * m; t < m * m; t += tstep) {
    const int j = t / m, k = t - j * m;
    // A u (local) = (hy/hx) Kref C Mref + (hx/hy) Mref C Kref,
    // Mref = R^T diag(1/(2l+1)) R expanded as nested sparse sums
    double au1 = 0.0, au2 = 0.0;
    {
      const Sp3 kj = k_row(j, inv), ck = r_col(k, inv);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        double s1 = 0.0;
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          const int l = ck.i[y];
          const Sp3 rl = r_row(l, p, inv);
          double s2 = 0.0;
#pragma unroll
          for (int z = 0; z < 3; ++z) s2 += rl.v[z] * C(kj.i[x], rl.i[z]);
          s1 += (ck.v[y] * inv(l)) * s2;
        }
        au1 += kj.v[x] * s1;
      }
      const Sp3 cj = r_col(j, inv), kk = k_row(k, inv);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int l = cj.i[x];
        const Sp3 rl = r_row(l, p, inv);
        double s1 = 0.0;
#pragma unroll
        for (int z = 0; z < 3; ++z) {
          double s2 = 0.0;
#pragma unroll
          for (int y = 0; y < 2; ++y) s2 += kk.v[y] * C(rl.i[z], kk.i[y]);
          s1 += rl.v[z] * s2;
        }
        au2 += (cj.v[x] * inv(l)) * s1;
      }
    }
    const double au = (hy / hx) * au1 + (hx / hy) * au2;
    // B (psi_prev - psi)
    double bp = 0.0;
#pragma unroll
    for (int comp = 0; comp < (GRADIENT ? 2 : 1); ++comp) {
      const Sp3 sj = (GRADIENT && comp == 0) ? d_col(j) : r_col(j, inv);
      const Sp3 sk = (GRADIENT && comp == 1) ? d_col(k) : r_col(k, inv);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int i = sj.i[x];
        if (x >= sj.n || i >= n) continue;
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          const int l = sk.i[y];
          if (y >= sk.n || l >= n) continue;
          bp += sj.v[x] * sk.v[y] * sG[comp * n * n + i * n + l];
        }
      }
    }
    const double rr = -A.alpha * au + bp;
    if (j >= 2 && k >= 2) {
      const long long ix = (A.ncx - 1) + (long long)cx * (p - 1) + (j - 2);
      const long long iy = (A.ncy - 1) + (long long)cy * (p - 1) + (k - 2);
      const long long g = ix * A.niy + iy;
      A.b_u[g] = A.alpha * __ldg(A.f_load + g) + rr;
    } else {
      double* edge = A.edge + (long long)e * (4 * m - 4);
      if (j < 2) edge[j * m + k] = rr;
      else edge[2 * m + (j - 2) * 2 + k] = rr;
    }
    // B^T u at psi entry (a, b) = (j, k)
    if (j < n && k < n) {
      const int a = j, b = k;
      const long long g = base0 + (long long)a * A.ld + b;
      if (!GRADIENT) {
        const Sp3 ra = r_row(a, p, inv), rb = r_row(b, p, inv);
        double L = 0.0;
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          double t2 = 0.0;
#pragma unroll
          for (int y = 0; y < 3; ++y) t2 += rb.v[y] * C(ra.i[x], rb.i[y]);
          L += ra.v[x] * t2;
        }
        const double btu = ((hx * inv(a)) * L) * (hy * inv(b));
        A.out[g] = __ldg(A.phi_mom + g) - btu;
      } else {
        const Sp3 da = d_row(a), rb = r_row(b, p, inv), ra = r_row(a, p, inv), db = d_row(b);
        double Lx = 0.0, Ly = 0.0;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          double t2 = 0.0;
#pragma unroll
          for (int y = 0; y < 3; ++y) t2 += rb.v[y] * C(da.i[x], rb.i[y]);
          Lx += da.v[x] * t2;
        }
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          double t2 = 0.0;
#pragma unroll
          for (int y = 0; y < 2; ++y) t2 += db.v[y] * C(ra.i[x], db.i[y]);
          Ly += ra.v[x] * t2;
        }
        A.out[g] = -(((2.0 * inv(a)) * Lx) * (hy * inv(b)));
        A.out[A.ncomp + g] = -(((hx * inv(a)) * Ly) * (2.0 * inv(b)));
      }
    }
  }
}

// b_u on the hat-involved interior dofs: alpha f_load + the (up to 4) cell
// contributions, summed in a fixed order.
static __global__ void k_hat_gather(ElemArgs A) {
  pdl_wait();
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
