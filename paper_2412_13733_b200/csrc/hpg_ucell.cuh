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
// (deterministic, no atomics).  k_uside_pt is the general-degree kernel;
// low and mid degrees use the generated k_usmall / k_upass.
#pragma once
#include "hpg_common.cuh"

namespace hpg {

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
  // the rows this CTA's entries read: with one pass (tstep >= m^2) the CTA
  // owns entries [sp TG, (sp+1) TG), i.e. rows j0..j1, and the sparse 1D
  // operators reach rows j-2..j+2 plus the hat rows 0, 1 -- a few-cell split
  // (config 3: 7 CTAs per cell) then loads ~1/5 of the tile per CTA
  int rlo = 0, rhi = m - 1;
  if (tstep >= m * m) {
    const int e0 = sp * TG, e1 = (sp + 1) * TG < m * m ? (sp + 1) * TG : m * m;
    rlo = e0 / m - 2 < 0 ? 0 : e0 / m - 2;
    rhi = (e1 - 1) / m + 2 > m - 1 ? m - 1 : (e1 - 1) / m + 2;
  }
  const int wrows = rhi - rlo + 1;
  const int extra = rlo > 1 ? 2 : (rlo > 0 ? 1 : 0);           // hat rows below the window
  // unrolled so every thread's gathers are in flight together (one L2 round
  // trip per 8 entries instead of one per entry)
#pragma unroll 8
  for (int t = valid ? t0 : (wrows + extra) * m; t < (wrows + extra) * m; t += TG) {
    const int q = t / m, l = t - q * m;
    const int i = q < extra ? q : rlo + (q - extra);
    sC[i * ld + l] = u_at(A, cx, cy, i, l);
  }
  const int glo = rlo < n ? rlo : n, ghi = rhi < n - 1 ? rhi : n - 1;
  const int grows = ghi - glo + 1 > 0 ? ghi - glo + 1 : 0;
  const int gextra = glo > 1 ? 2 : (glo > 0 ? 1 : 0);
  const int gper = (grows + gextra) * n;
#pragma unroll 8
  for (int t = valid ? t0 : gper * 2; t < gper * (GRADIENT ? 2 : 1); t += TG) {
    const int comp = t / gper, rr = t - comp * gper, q = rr / n, l = rr - q * n;
    const int i = q < gextra ? q : glo + (q - gextra);
    const long long gi = comp * A.ncomp + base0 + (long long)i * A.ld + l;
    const double d = __ldg(A.psi_prev + gi) - __ldg(A.in0 + gi);
    double wi, wl;
    if (!GRADIENT) { wi = hx * kInvOdd[i]; wl = hy * kInvOdd[l]; }
    else if (comp == 0) { wi = 2.0 * kInvOdd[i]; wl = hy * kInvOdd[l]; }
    else { wi = hx * kInvOdd[i]; wl = 2.0 * kInvOdd[l]; }
    sG[comp * n * n + i * n + l] = (wi * d) * wl;
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
