// Per-cell Schur preconditioner kernels (see hpg_precond.cuh).
//
//  k_triple            hat triple T(hx, hy) = Bhat^T Ahat^{-1} Bhat per width key
//                      (assembly.py:577-595) through the separable
//                      eigen-factorisation of Ahat = Kx (x) My + Mx (x) Ky:
//                      T[(a,b),(c,d)] = (hx hy)^3 sum_ij Z[a,i] Z[b,j] Z[c,i] Z[d,j]
//                                        / (hx^2 lam_i + hy^2 lam_j)
//                      (Z, lam: reference-cell factors built by tables.py).
//  k_precond_transform P_e = -D_e - T/alpha - beta E_e, in place (assembly.py:597-603, 851-860)
//  k_lu<KB>            batched LU with partial pivoting, one CTA per block
//                      (LAPACK getrf as called by scipy lu_factor, linalg.py:249):
//                      right-looking, KB-column panels factored in shared memory;
//                      per 64-column chunk U12 = L11^{-1} A12 and the trailing
//                      update A22 -= L21 U12 run on the FP64 tensor cores (DMMA
//                      m8n8k4) with the chunk staged in shared memory.
//  k_lu_solve          getrs per cell on the global psi vector (linalg.py:253-257):
//                      row interchanges, 32-row blocked unit-lower then upper
//                      substitution (warp 0 solves the diagonal block, all warps
//                      apply the off-diagonal panel).
#include <cfloat>

#include "../../include/hpg_b200.h"
#include "hpg_launch.cuh"
#include "hpg_precond.cuh"

namespace hpg {

namespace {

constexpr int LU_THREADS = 256;
constexpr int LU_UCH = 64;     // trailing-update column chunk
constexpr int LU_ULD = 72;     // its smem row stride (conflict-free B fragments)
constexpr int SOLVE_THREADS = 128;

// ---------------------------------------------------------------------------
__global__ void k_triple(const double* __restrict__ Z, const double* __restrict__ lam, int n,
                         const double* __restrict__ khx, const double* __restrict__ khy,
                         double* __restrict__ tri) {
  extern __shared__ double s[];
  double* sZ = s;
  double* sD = sZ + n * n;
  double* sF = sD + n * n;
  const int a = blockIdx.x / n, c = blockIdx.x - (blockIdx.x / n) * n, key = blockIdx.y;
  const double hx = khx[key], hy = khy[key];
  const double hx2 = hx * hx, hy2 = hy * hy;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    sZ[i] = Z[i];
    const int ii = i / n, jj = i - (i / n) * n;
    sD[i] = 1.0 / (hx2 * lam[ii] + hy2 * lam[jj]);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double f = 0.0;
    for (int i = 0; i < n; ++i) f += sZ[a * n + i] * sZ[c * n + i] * sD[i * n + j];
    sF[j] = f;
  }
  __syncthreads();
  const double h3 = hx * hy * hx * hy * hx * hy;
  const int n2 = n * n;
  double* out = tri + (size_t)key * n2 * n2;
  for (int idx = threadIdx.x; idx < n2; idx += blockDim.x) {
    const int b = idx / n, d = idx - (idx / n) * n;
    double t = 0.0;
    for (int j = 0; j < n; ++j) t += sZ[b * n + j] * sZ[d * n + j] * sF[j];
    out[(size_t)(a * n + b) * n2 + c * n + d] = h3 * t;
  }
}

// spectral mass entry (assembly.py:128-144) and stiffness diagonal (:147-153)
__device__ __forceinline__ double smass(int a, int c, double h) {
  if (a == c) return h * (1.0 / (2 * a + 1) + 1.0 / (2 * a + 5));
  if (a - c == 2 || c - a == 2) return -h / (2 * (a < c ? a : c) + 5);
  return 0.0;
}
__device__ __forceinline__ double sstiff(int a, double h) { return 4.0 * (2.0 * a + 3.0) / h; }

// P_e[row][col] from D_e[row][col] = v
__device__ __forceinline__ double precond_value(const PrecArgs& A, int e, int row, int col, double v) {
  const int cx = e / A.ncy, cy = e - (e / A.ncy) * A.ncy;
  const double hx = A.hx[cx], hy = A.hy[cy];
  if (A.kind == HPG_OBSTACLE) {
    double t = -v - A.tri[((size_t)A.key[e] * A.n2 + row) * A.n2 + col] / A.alpha;
    if (row == col) {
      const int a = row / A.n, b = row - (row / A.n) * A.n;
      t -= A.beta * ((hx / (2.0 * a + 1.0)) * (hy / (2.0 * b + 1.0)));
    }
    return t;
  }
  double t = -v;
  if (A.beta != 0.0) {
    const int cr = row / A.n2, cc = col / A.n2;
    if (cr == cc) {
      const int rr = row - cr * A.n2, c2 = col - cc * A.n2;
      const int a = rr / A.n, b = rr - (rr / A.n) * A.n;
      const int c = c2 / A.n, d = c2 - (c2 / A.n) * A.n;
      const double e1 = (a == c) ? sstiff(a, hx) * smass(b, d, hy) : 0.0;
      const double e2 = (b == d) ? smass(a, c, hx) * sstiff(b, hy) : 0.0;
      t -= A.beta * (e1 + e2);
    }
  }
  return t;
}

__global__ void k_precond_transform(PrecArgs A) {
  const long long nbb = (long long)A.nb * A.nb;
  const long long total = nbb * A.count;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int cl = (int)(idx / nbb);
    const long long rem = idx - cl * nbb;
    const int row = (int)(rem / A.nb), col = (int)(rem - (rem / A.nb) * A.nb);
    A.M[idx] = precond_value(A, A.cell0 + cl, row, col, A.M[idx]);
  }
}

// ---------------------------------------------------------------------------
template <int KB>
__device__ __forceinline__ void argmax_combine(double& best, int& bi, double ov, int oi) {
  if (ov > best || (ov == best && oi < bi)) {
    best = ov;
    bi = oi;
  }
}

template <int KB>
__global__ void __launch_bounds__(LU_THREADS) k_lu(PrecArgs A) {
  extern __shared__ double sm[];
  constexpr int LDP = KB + 1;
  constexpr int NOPIV = 0x7fffffff;
  const int nb = A.nb;
  double* sP = sm;                                  // panel [nb][LDP]
  double* sLi = sP + (size_t)nb * LDP;              // L11^{-1} [KB][LDP]
  double* sA = sLi + KB * LDP;                      // A12 chunk [KB][LU_ULD]
  double* sU = sA + KB * LU_ULD;                    // U12 chunk [KB][LU_ULD]
  double* sRv = sU + KB * LU_ULD;                   // per-warp argmax values [8]
  int* sRi = reinterpret_cast<int*>(sRv + 8);       // and rows [8]
  int* sPiv = sRi + 8;                              // panel pivots [KB]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, c = lane & 3;

  for (int cl = blockIdx.x; cl < A.count; cl += gridDim.x) {
    double* M = A.M + (size_t)cl * nb * nb;
    int* piv = A.ipiv + (size_t)cl * nb;
    if (A.transform) {
      const int e = A.cell0 + cl;
      for (long long idx = tid; idx < (long long)nb * nb; idx += LU_THREADS) {
        const int row = (int)(idx / nb), col = (int)(idx - (long long)row * nb);
        M[idx] = precond_value(A, e, row, col, M[idx]);
      }
      __syncthreads();
    }
    for (int k0 = 0; k0 < nb; k0 += KB) {
      const int kb = nb - k0 < KB ? nb - k0 : KB, rows = nb - k0;
      // (1) load the panel; each thread tracks its rows' max |a| of column 0
      bool bad = false;
      for (int idx = tid; idx < rows * KB; idx += LU_THREADS) {
        const int i = idx / KB, j = idx - (idx / KB) * KB;
        const double v = j < kb ? M[(size_t)(k0 + i) * nb + k0 + j] : 0.0;
        sP[i * LDP + j] = v;
        // the first panel load sees every entry of column block 0; later
        // panels see the updated values: a non-finite value anywhere
        // (scipy's check_finite) shows up in some panel
        bad |= !isfinite(v);
      }
      if (bad && A.info) atomicOr(A.info, 1);
      __syncthreads();
      double best = -1.0;
      int bi = NOPIV;
      for (int i = tid; i < rows; i += LU_THREADS) {
        const double v = fabs(sP[i * LDP]);
        if (v > best) { best = v; bi = i; }
      }
      for (int j = 0; j < kb; ++j) {
        // (2) pivot: first row of maximal |a_ij| (LAPACK idamax)
#pragma unroll
        for (int off = 16; off; off >>= 1)
          argmax_combine<KB>(best, bi, __shfl_xor_sync(~0u, best, off), __shfl_xor_sync(~0u, bi, off));
        if (lane == 0) { sRv[warp] = best; sRi[warp] = bi; }
        __syncthreads();
        if (warp == 0) {
          best = lane < LU_THREADS / 32 ? sRv[lane] : -1.0;
          bi = lane < LU_THREADS / 32 ? sRi[lane] : NOPIV;
#pragma unroll
          for (int off = 4; off; off >>= 1)
            argmax_combine<KB>(best, bi, __shfl_xor_sync(~0u, best, off), __shfl_xor_sync(~0u, bi, off));
          int p = __shfl_sync(~0u, bi, 0);
          if (p == NOPIV) p = j;                     // all-NaN column: no interchange
          if (lane == 0) { sPiv[j] = p; piv[k0 + j] = k0 + p; }
          if (p != j && lane < KB) {
            const double t = sP[j * LDP + lane];
            sP[j * LDP + lane] = sP[p * LDP + lane];
            sP[p * LDP + lane] = t;
          }
        }
        __syncthreads();
        // (3) scale the column (by 1/pivot when that is safe, as dgetrf2) and
        //     rank-1 update the rest of the panel; track column j+1's argmax
        const double pv = sP[j * LDP + j];
        if (pv == 0.0 && tid == 0 && A.info) atomicOr(A.info, 2);
        const bool recip = fabs(pv) >= DBL_MIN;
        const double rp = 1.0 / pv;
        best = -1.0;
        bi = NOPIV;
        for (int i = j + 1 + tid; i < rows; i += LU_THREADS) {
          double l = sP[i * LDP + j];
          if (pv != 0.0) l = recip ? l * rp : l / pv;
          sP[i * LDP + j] = l;
          for (int cc = j + 1; cc < kb; ++cc) sP[i * LDP + cc] -= l * sP[j * LDP + cc];
          if (j + 1 < kb) {
            const double v = fabs(sP[i * LDP + j + 1]);
            if (v > best) { best = v; bi = i; }
          }
        }
        // the next iteration's partial-max exchange starts with a barrier-free
        // warp reduction; the barrier after its smem write orders this update
        __syncthreads();
      }
      // (4) panel back to global; interchanges applied to the other columns
      for (int idx = tid; idx < rows * kb; idx += LU_THREADS) {
        const int i = idx / kb, j = idx - (idx / kb) * kb;
        M[(size_t)(k0 + i) * nb + k0 + j] = sP[i * LDP + j];
      }
      for (int col = tid; col < nb; col += LU_THREADS) {
        if (col >= k0 && col < k0 + kb) continue;
        for (int j = 0; j < kb; ++j) {
          const int p = sPiv[j];
          if (p != j) {
            const double t = M[(size_t)(k0 + j) * nb + col];
            M[(size_t)(k0 + j) * nb + col] = M[(size_t)(k0 + p) * nb + col];
            M[(size_t)(k0 + p) * nb + col] = t;
          }
        }
      }
      __syncthreads();
      // (5) Linv = L11^{-1} (unit lower), one column per thread; zero outside
      //     the kb x kb corner so padded k-steps below contribute exact zeros
      if (tid < KB) {
        const int cc = tid;
        for (int i = 0; i < KB; ++i) {
          double t = 0.0;
          if (i == cc) {
            t = 1.0;
          } else if (i > cc) {
            for (int j = cc; j < i; ++j) t -= sP[i * LDP + j] * sLi[j * LDP + cc];
          }
          sLi[i * LDP + cc] = (i < kb && cc < kb) ? t : 0.0;
        }
      }
      __syncthreads();
      // (6) per 64-column chunk: U12 = Linv A12 and A22 -= L21 U12, both on
      //     the FP64 tensor cores with the chunk staged in shared memory
      const int trows = rows - kb;
      const int nrt = (trows + 7) >> 3;
      for (int cc0 = k0 + kb; cc0 < nb; cc0 += LU_UCH) {
        for (int idx = tid; idx < KB * LU_UCH; idx += LU_THREADS) {
          const int j = idx / LU_UCH, t = idx - (idx / LU_UCH) * LU_UCH;
          const int col = cc0 + t;
          sA[j * LU_ULD + t] = (j < kb && col < nb) ? M[(size_t)(k0 + j) * nb + col] : 0.0;
        }
        __syncthreads();
        for (int tile = warp; tile < (KB / 8) * 8; tile += LU_THREADS / 32) {
          const int mt = tile >> 3, nt = tile & 7;
          double u[2] = {0.0, 0.0};
#pragma unroll
          for (int ks = 0; ks < KB / 4; ++ks)
            dmma(u, sLi[(8 * mt + r) * LDP + 4 * ks + c], sA[(4 * ks + c) * LU_ULD + 8 * nt + r]);
          const int row = 8 * mt + r, col = 8 * nt + 2 * c;
          sU[row * LU_ULD + col] = u[0];
          sU[row * LU_ULD + col + 1] = u[1];
          if (row < kb && cc0 + col < nb) M[(size_t)(k0 + row) * nb + cc0 + col] = u[0];
          if (row < kb && cc0 + col + 1 < nb) M[(size_t)(k0 + row) * nb + cc0 + col + 1] = u[1];
        }
        __syncthreads();
        for (int rt = warp; rt < nrt; rt += LU_THREADS / 32) {
          const int row = kb + 8 * rt + r;           // panel-relative
          const bool rv = row < rows;
          double* mrow = M + (size_t)(k0 + (rv ? row : kb)) * nb;
          double acc[8][2];
#pragma unroll
          for (int nt = 0; nt < 8; ++nt) {
            const int col = cc0 + 8 * nt + 2 * c;
            acc[nt][0] = (rv && col < nb) ? mrow[col] : 0.0;
            acc[nt][1] = (rv && col + 1 < nb) ? mrow[col + 1] : 0.0;
          }
#pragma unroll
          for (int ks = 0; ks < KB / 4; ++ks) {
            const double a = rv ? -sP[row * LDP + 4 * ks + c] : 0.0;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) dmma(acc[nt], a, sU[(4 * ks + c) * LU_ULD + 8 * nt + r]);
          }
#pragma unroll
          for (int nt = 0; nt < 8; ++nt) {
            const int col = cc0 + 8 * nt + 2 * c;
            if (rv && col < nb) mrow[col] = acc[nt][0];
            if (rv && col + 1 < nb) mrow[col + 1] = acc[nt][1];
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SOLVE_THREADS) k_lu_solve(ElemArgs E, const double* __restrict__ lu,
                                                            const int* __restrict__ ipiv, int nb,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y) {
  extern __shared__ double sx[];
  int* sp = reinterpret_cast<int*>(sx + nb);
  const int e = blockIdx.x;
  const int cx = e / E.ncy, cy = e - cx * E.ncy;
  const int n2 = E.n * E.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = SOLVE_THREADS / 32;
  const double* L = lu + (size_t)e * nb * nb;
  for (int l = tid; l < nb; l += SOLVE_THREADS) {
    const int comp = l / n2, rem = l - comp * n2;
    sx[l] = __ldg(x + comp * E.ncomp + psi_index(E, cx, cy, rem / E.n, rem % E.n));
    sp[l] = __ldg(ipiv + (size_t)e * nb + l);
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < nb; ++i) {
      const int p = sp[i];
      if (p != i) {
        const double t = sx[i];
        sx[i] = sx[p];
        sx[p] = t;
      }
    }
  }
  __syncthreads();
  // forward: unit lower L
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int bs = nb - b0 < 32 ? nb - b0 : 32;
    if (warp == 0) {
      double xi = lane < bs ? sx[b0 + lane] : 0.0;
      double lr[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        lr[j] = (lane < bs && j < lane) ? __ldg(L + (size_t)(b0 + lane) * nb + b0 + j) : 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double xj = __shfl_sync(~0u, xi, j);
        if (j < lane) xi -= lr[j] * xj;
      }
      if (lane < bs) sx[b0 + lane] = xi;
    }
    __syncthreads();
    const double xl = lane < bs ? sx[b0 + lane] : 0.0;
#pragma unroll 4
    for (int i = b0 + bs + warp; i < nb; i += NW) {
      double s = lane < bs ? __ldg(L + (size_t)i * nb + b0 + lane) * xl : 0.0;
#pragma unroll
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(~0u, s, off);
      if (lane == 0) sx[i] -= s;
    }
    __syncthreads();
  }
  // backward: upper U (non-unit diagonal)
  for (int b0 = ((nb - 1) / 32) * 32; b0 >= 0; b0 -= 32) {
    const int bs = nb - b0 < 32 ? nb - b0 : 32;
    if (warp == 0) {
      double xi = lane < bs ? sx[b0 + lane] : 0.0;
      double ur[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        ur[j] = (lane < bs && j >= lane && j < bs) ? __ldg(L + (size_t)(b0 + lane) * nb + b0 + j) : 0.0;
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < bs) {
          if (lane == j) xi = xi / ur[j];
          const double xj = __shfl_sync(~0u, xi, j);
          if (lane < j) xi -= ur[j] * xj;
        }
      }
      if (lane < bs) sx[b0 + lane] = xi;
    }
    __syncthreads();
    const double xl = lane < bs ? sx[b0 + lane] : 0.0;
#pragma unroll 4
    for (int i = warp; i < b0; i += NW) {
      double s = lane < bs ? __ldg(L + (size_t)i * nb + b0 + lane) * xl : 0.0;
#pragma unroll
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(~0u, s, off);
      if (lane == 0) sx[i] -= s;
    }
    __syncthreads();
  }
  for (int l = tid; l < nb; l += SOLVE_THREADS) {
    const int comp = l / n2, rem = l - comp * n2;
    y[comp * E.ncomp + psi_index(E, cx, cy, rem / E.n, rem % E.n)] = sx[l];
  }
}

template <int KB>
size_t lu_smem(int nb) {
  return sizeof(double) * ((size_t)(nb + KB) * (KB + 1) + 2 * KB * LU_ULD + 8) + sizeof(int) * (8 + KB);
}

template <int KB>
int launch_lu_t(const PrecArgs& A, int nsm, cudaStream_t s) {
  const size_t smem = lu_smem<KB>(A.nb);
  cudaError_t e = cudaFuncSetAttribute(k_lu<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_lu)", e);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lu<KB>, LU_THREADS, smem);
  const long long cap = (long long)nsm * (occ > 0 ? occ : 1);
  const int grid = (int)(A.count < cap ? A.count : cap);
  k_lu<KB><<<grid, LU_THREADS, smem, s>>>(A);
  e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_lu launch", e);
}

constexpr size_t LU_SMEM_CAP = 220u << 10;

}  // namespace

int lu_max_nb() {
  // the KB = 8 panel is the smallest one
  return (int)((LU_SMEM_CAP - sizeof(double) * (8 * 9 + 16 * LU_ULD + 8) - sizeof(int) * 16) / (sizeof(double) * 9));
}

int launch_triple(const double* Zhat, const double* lam_hat, int n, const double* key_hx,
                  const double* key_hy, int nkeys, double* tri, cudaStream_t s) {
  const size_t smem = sizeof(double) * (2 * (size_t)n * n + n);
  if (smem > (48u << 10)) {
    cudaError_t e = cudaFuncSetAttribute(k_triple, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_triple)", e);
  }
  k_triple<<<dim3(n * n, nkeys), 256, smem, s>>>(Zhat, lam_hat, n, key_hx, key_hy, tri);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_triple launch", e);
}

int launch_precond_transform(const PrecArgs& A, cudaStream_t s) {
  const long long total = (long long)A.nb * A.nb * A.count;
  long long blocks = (total + 255) / 256;
  if (blocks > 148LL * 32) blocks = 148LL * 32;
  if (blocks < 1) blocks = 1;
  k_precond_transform<<<(int)blocks, 256, 0, s>>>(A);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_precond_transform launch", e);
}

int launch_lu(const PrecArgs& A, int nsm, cudaStream_t s) {
  // widest panel that fits shared memory (HPG_LU_KB overrides, for tuning)
  int kb = 32;
  if (const char* env = getenv("HPG_LU_KB")) kb = atoi(env);
  while (kb > 8 && ((kb == 32 && lu_smem<32>(A.nb) > LU_SMEM_CAP) || (kb == 16 && lu_smem<16>(A.nb) > LU_SMEM_CAP)))
    kb /= 2;
  if (lu_smem<8>(A.nb) > LU_SMEM_CAP)
    return set_error_msg(HPG_ERR_UNSUPPORTED, "per-CTA LU: block side too large for a shared-memory panel");
  switch (kb) {
    case 32: return launch_lu_t<32>(A, nsm, s);
    case 16: return launch_lu_t<16>(A, nsm, s);
    default: return launch_lu_t<8>(A, nsm, s);
  }
}

int launch_lu_solve(const ElemArgs& E, const double* lu, const int* ipiv, int nb, const double* x,
                    double* y, cudaStream_t s) {
  const size_t smem = (sizeof(double) + sizeof(int)) * (size_t)nb + 16;
  if (smem > (48u << 10)) {
    cudaError_t e = cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_lu_solve)", e);
  }
  k_lu_solve<<<E.N, SOLVE_THREADS, smem, s>>>(E, lu, ipiv, nb, x, y);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_lu_solve launch", e);
}

}  // namespace hpg
