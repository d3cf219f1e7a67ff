// Element blocks of D (assembly.py:257-263, 550-557, 804-815) and their matvec
// (CellBlockMatrix.matvec, assembly.py:281-285).
//
// blk[(a,b),(j,k)] = w_a w_b sum_{g,h} T[a,g] S[g,j] W[g,h] T[b,h] S[h,k]
// is evaluated as two GEMMs with the element-independent table
// G[(a,j), g] = T[a,g] S[g,j]  (n^2 x QP):
//   Z_e  = G W_e          (n^2 x QP)    -- per element and weight field
//   blk  = Z_e G^T        (n^2 x n^2)   -- stored permuted to rows (a,b), cols (j,k)
// Both run on the FP64 tensor cores (DMMA.8x8x4) from shared-memory tiles.
#pragma once
#include "hpg_common.cuh"
#include "hpg_elem.cuh"

namespace hpg {

struct GemmArgs {
  int M, N, K;            // per-batch GEMM: C[M][N] = sum_k A[i][k] B[j][k]
  int nfield;             // weight fields per cell (1 obstacle, 3 gradient)
  int n, n2, QP, QT, NW;
  int ncy, cell0;
  const double* G;        // [n2][QP]
  const double* wc;       // weight cache (C-fragment order)
  double* Z;              // [batch][n2][QP]
  double* out;            // blocks of cells [cell0, cell0 + count)
  long long nb;           // block side (n2 or 2 n2)
  const double* hx;
  const double* hy;
};

constexpr int GT = 64, GK = 16, GLD = GK + 4;

template <int STAGE>
__device__ __forceinline__ double gemm_a(const GemmArgs& g, int batch, int i, int k) {
  if (i >= g.n2 || k >= g.K) return 0.0;
  if constexpr (STAGE == 0) return __ldg(g.G + (long long)i * g.QP + k);
  else return g.Z[((long long)batch * g.n2 + i) * g.QP + k];
}

template <int STAGE>
__device__ __forceinline__ double gemm_b(const GemmArgs& g, int batch, int j, int k) {
  if constexpr (STAGE == 0) {
    // B[j=h][k=g] = W_f[g][h]; batch = local cell * nfield + f
    if (j >= g.QP || k >= g.QP) return 0.0;
    int cl = batch / g.nfield, f = batch - cl * g.nfield;
    int e = g.cell0 + cl;
    int rt = k >> 3, ht = j >> 3, lane = (k & 7) * 4 + ((j & 7) >> 1);
    return __ldg(g.wc + wc_index(e, g.QT, rt, ht, g.NW, f, lane) + (j & 1));
  } else {
    if (j >= g.n2 || k >= g.K) return 0.0;
    return __ldg(g.G + (long long)j * g.QP + k);
  }
}

template <int STAGE>
__device__ __forceinline__ void gemm_store(const GemmArgs& g, int batch, int i, int j, double v) {
  if constexpr (STAGE == 0) {
    if (i < g.n2 && j < g.QP) g.Z[((long long)batch * g.n2 + i) * g.QP + j] = v;
  } else {
    if (i >= g.n2 || j >= g.n2) return;
    int cl = batch / g.nfield, f = batch - cl * g.nfield;
    int e = g.cell0 + cl;
    int cx = e / g.ncy, cy = e - cx * g.ncy;
    int a = i / g.n, jj = i - a * g.n;     // row (a, j) of Z
    int bb = j / g.n, kk = j - bb * g.n;   // col (b, k) of G
    double wa = g.hx[cx] * kInvOdd[a], wb = g.hy[cy] * kInvOdd[bb];
    double val = v * (wa * wb);
    long long row = (long long)a * g.n + bb, col = (long long)jj * g.n + kk;
    double* blk = g.out + (long long)cl * g.nb * g.nb;
    if (g.nfield == 1) {
      blk[row * g.nb + col] = val;
    } else if (f == 0) {
      blk[row * g.nb + col] = val;
    } else if (f == 1) {
      blk[row * g.nb + g.n2 + col] = val;
      blk[(g.n2 + row) * g.nb + col] = val;
    } else {
      blk[(g.n2 + row) * g.nb + g.n2 + col] = val;
    }
  }
}

template <int STAGE>
__global__ void __launch_bounds__(256) k_gemm(GemmArgs g) {
  __shared__ double sA[GT][GLD];
  __shared__ double sB[GT][GLD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  const int wi = warp >> 2, wj = warp & 3;
  const int i0 = blockIdx.x * GT, j0 = blockIdx.y * GT, batch = blockIdx.z;
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int k0 = 0; k0 < g.K; k0 += GK) {
    for (int t = threadIdx.x; t < GT * GK; t += 256) {
      int ii = t / GK, kk = t - ii * GK;
      sA[ii][kk] = gemm_a<STAGE>(g, batch, i0 + ii, k0 + kk);
      sB[ii][kk] = gemm_b<STAGE>(g, batch, j0 + ii, k0 + kk);
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      double af[4], bf[2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = sA[wi * 32 + mt * 8 + r][ks * 4 + c];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) bf[nt] = sB[wj * 16 + nt * 8 + r][ks * 4 + c];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        gemm_store<STAGE>(g, batch, i0 + wi * 32 + mt * 8 + r, j0 + wj * 16 + nt * 8 + 2 * c + j,
                          acc[mt][nt][j]);
}

// y[idx_e] = blk_e x[idx_e], one CTA per cell, x tile staged in smem.
__global__ void k_blocks_matvec(ElemArgs A, const double* __restrict__ blocks, int nb, int ncompv,
                                const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ double xs[];
  const int e = blockIdx.x;
  const int cx = e / A.ncy, cy = e - cx * A.ncy;
  const int n2 = A.n * A.n;
  for (int l = threadIdx.x; l < nb; l += blockDim.x) {
    int comp = l / n2, rem = l - comp * n2;
    xs[l] = __ldg(x + comp * A.ncomp + psi_index(A, cx, cy, rem / A.n, rem % A.n));
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double* blk = blocks + (long long)e * nb * nb;
  for (int row = warp; row < nb; row += nw) {
    double s = 0.0;
    for (int k = lane; k < nb; k += 32) s += __ldg(blk + (long long)row * nb + k) * xs[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
      int comp = row / n2, rem = row - comp * n2;
      y[comp * A.ncomp + psi_index(A, cx, cy, rem / A.n, rem % A.n)] = s;
    }
  }
  (void)ncompv;
}

}  // namespace hpg
