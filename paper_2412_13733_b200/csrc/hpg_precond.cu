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

#ifndef HPG_LU_THREADS
#define HPG_LU_THREADS 256
#endif
#ifndef HPG_LU_MINB
#define HPG_LU_MINB 2
#endif
constexpr int LU_THREADS = HPG_LU_THREADS;
constexpr int LU_UCH = 64;     // trailing-update column chunk
#ifndef HPG_LU_ULD
#define HPG_LU_ULD 68
#endif
constexpr int LU_ULD = HPG_LU_ULD;     // its smem row stride: = 4 mod 16, so the B fragments B[c][r] of a
                                       // half warp (r < 4) fall in 16 distinct 8-byte banks (72 gave 2-way conflicts)
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

// P_e[row][col] from D_e[row][col] = v
__device__ __forceinline__ double precond_value(const PrecArgs& A, int e, int row, int col, double v) {
  const int cx = e / A.ncy, cy = e - (e / A.ncy) * A.ncy;
  const double* tri = A.kind == HPG_OBSTACLE ? A.tri + (size_t)A.key[e] * A.n2 * A.n2 : nullptr;
  return precond_entry(A.kind, A.n, A.n2, A.hx[cx], A.hy[cy], A.alpha, A.beta, tri, row, col, v);
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
__global__ void __launch_bounds__(LU_THREADS, HPG_LU_MINB) k_lu(PrecArgs A) {
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
  int* sList = sPiv + KB;                           // rows touched by the interchanges [2 KB + 1]
  int* sRow = sList + 2 * KB + 1;                   // composed interchanges: position <- row [nb]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, c = lane & 3;
  // phase profiling (A.prof != nullptr only from tools/prof_precond.py):
  // cycles since the previous mark are charged to the phase that just ended
  long long t_last = clock64();
  int ph_last = 7;
#define PROF_MARK(ph)                                                   \
  do {                                                                  \
    if (A.prof != nullptr && tid == 0) {                                \
      const long long t_now = clock64();                                \
      atomicAdd(A.prof + ph_last, (unsigned long long)(t_now - t_last)); \
      t_last = t_now;                                                   \
    }                                                                   \
    ph_last = (ph);                                                     \
  } while (0)

  for (int cl = blockIdx.x; cl < A.count; cl += gridDim.x) {
    double* M = A.M + (size_t)cl * nb * nb;
    int* piv = A.ipiv + (size_t)cl * nb;
    PROF_MARK(6);
    if (A.transform) {
      const int e = A.cell0 + cl;
#pragma unroll 4
      for (int idx = tid; idx < nb * nb; idx += LU_THREADS) {
        const int row = idx / nb, col = idx - (idx / nb) * nb;
        M[idx] = precond_value(A, e, row, col, M[idx]);
      }
      __syncthreads();
    }
    for (int k0 = 0; k0 < nb; k0 += KB) {
      const int kb = nb - k0 < KB ? nb - k0 : KB, rows = nb - k0;
      PROF_MARK(0);
      // (1) load the panel; each thread tracks its rows' max |a| of column 0
      bool bad = false;
      for (int i = tid; i < rows; i += LU_THREADS) sRow[i] = i;
#pragma unroll 4
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
      PROF_MARK(7);
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
      PROF_MARK(1);
      // (4) panel back to global; interchanges applied to the other columns
#pragma unroll 4
      for (int idx = tid; idx < rows * kb; idx += LU_THREADS) {
        const int i = idx / kb, j = idx - (idx / kb) * kb;
        M[(size_t)(k0 + i) * nb + k0 + j] = sP[i * LDP + j];
      }
      // the panel's interchanges, composed: position q receives row sRow[q];
      // touched positions = 0..kb-1 plus the distinct pivot rows >= kb
      if (tid == 0) {
        for (int j = 0; j < kb; ++j) {
          const int p = sPiv[j];
          if (p != j) {
            const int t = sRow[j];
            sRow[j] = sRow[p];
            sRow[p] = t;
          }
        }
      }
      if (warp == 1) {
        const int q = lane < kb ? sPiv[lane] : -1;
        const bool extra = q >= kb;
        const unsigned grp = __match_any_sync(~0u, extra ? q : -1 - lane);
        const bool lead = extra && (__ffs(grp) - 1 == lane);
        const unsigned bal = __ballot_sync(~0u, lead);
        if (lead) sList[kb + __popc(bal & ((1u << lane) - 1))] = q;
        if (lane < kb) sList[lane] = lane;
        if (lane == 0) sList[2 * KB] = kb + __popc(bal);
      }
      __syncthreads();
      {
      PROF_MARK(2);
        // apply them to the columns outside the panel, 64 columns at a time:
        // gather the touched rows into shared memory (sA..sU, free here),
        // then scatter them to their positions -- independent coalesced loads
        const int cnt = sList[2 * KB];
        double* sG = sA;                                  // [2 KB][64]
        for (int cb = 0; cb < nb; cb += 64) {
#pragma unroll 4
          for (int idx = tid; idx < cnt * 64; idx += LU_THREADS) {
            const int t = idx >> 6, col = cb + (idx & 63);
            if (col < nb && (col < k0 || col >= k0 + kb))
              sG[idx] = M[(size_t)(k0 + sRow[sList[t]]) * nb + col];
          }
          __syncthreads();
#pragma unroll 4
          for (int idx = tid; idx < cnt * 64; idx += LU_THREADS) {
            const int t = idx >> 6, col = cb + (idx & 63);
            if (col < nb && (col < k0 || col >= k0 + kb))
              M[(size_t)(k0 + sList[t]) * nb + col] = sG[idx];
          }
          __syncthreads();
        }
      }
      PROF_MARK(3);
      // (5) Linv = L11^{-1} (unit lower), one column per thread; zero outside
      //     the kb x kb corner so padded k-steps below contribute exact zeros
      if (tid < KB) {
        // column cc of L11^{-1}: t = e_cc, then t_i -= L_ij t_j for j < i in
        // axpy order -- straight-line, every t_j final before it is used
        const int cc = tid;
        double t[KB];
#pragma unroll
        for (int i = 0; i < KB; ++i) t[i] = i == cc ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < KB - 1; ++j)
#pragma unroll
          for (int i = j + 1; i < KB; ++i) t[i] -= sP[i * LDP + j] * t[j];
#pragma unroll
        for (int i = 0; i < KB; ++i) sLi[i * LDP + cc] = (i < kb && cc < kb) ? t[i] : 0.0;
      }
      __syncthreads();
      PROF_MARK(4);
      // (6) per 64-column chunk: U12 = Linv A12 and A22 -= L21 U12, both on
      //     the FP64 tensor cores with the chunk staged in shared memory
      const int trows = rows - kb;
      const int nrt = (trows + 7) >> 3;
      for (int cc0 = k0 + kb; cc0 < nb; cc0 += LU_UCH) {
#pragma unroll 4
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
      PROF_MARK(5);
    }
    if (A.perm != nullptr) {
      // composed interchanges: solve-side gather x'[i] = x[perm[i]] (getrs' laswp)
      for (int i = tid; i < nb; i += LU_THREADS) sRow[i] = i;
      __syncthreads();
      if (tid == 0) {
        for (int i = 0; i < nb; ++i) {
          const int p = piv[i];
          if (p != i) {
            const int t = sRow[i];
            sRow[i] = sRow[p];
            sRow[p] = t;
          }
        }
      }
      __syncthreads();
      for (int i = tid; i < nb; i += LU_THREADS) A.perm[(size_t)cl * nb + i] = sRow[i];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Row-per-thread LU for 32 < nb <= 256 (config 1: 225): the same LAPACK getrf
// arithmetic as k_lu, reorganised so that no row ever moves during the
// factorisation.
//  * Thread t owns storage row t.  A panel's 32 entries of the row live in
//    REGISTERS; the column loop is fully unrolled: block argmax of |a_j| over
//    the still-active rows (ties: smallest LAPACK position, idamax), the
//    winner publishes its row through shared memory, every active row scales
//    and rank-1 updates its registers.  Two barriers per column and no
//    shared-memory row traffic.
//  * Implicit pivoting: a pivot row retires in place.  Each row tracks the
//    position LAPACK's explicit interchanges would have given it (ipiv and
//    tie-breaking are exactly getrf's), the trailing update runs over the
//    compacted list of active rows, U12 over the panel's pivot rows.  The
//    per-panel row interchanges of the right and left parts (k_lu's gather
//    phase) are replaced by ONE permuting pass at the end.
// (P_e = -D_e - T/alpha - beta E_e is formed by k_precond_transform first.)
// panel row stride in shared memory: = 4 mod 16, so the trailing update's A
// fragments A[r][c] of a half warp fall in 16 distinct 8-byte banks (33 gave
// up to 4-way conflicts: 368 M conflicts per factorisation in ncu)
#ifndef HPG_LU2_LDP
#define HPG_LU2_LDP 36
#endif
constexpr int LU2_T = 256, LU2_KB = 32, LU2_LDP = HPG_LU2_LDP;

size_t lu2_smem(int nb) {
  return sizeof(double) * ((size_t)nb * LU2_LDP + LU2_KB * LU2_LDP + 2 * LU2_KB * LU_ULD + LU2_KB + 2) +
         sizeof(int) * (4 * 8 + 2 + LU2_KB + 2 * LU2_T + 16);
}

// U12 = Linv A12 on the panel's pivot rows and A22 -= L21 U12 on the active
// rows, per 64-column chunk, on the FP64 tensor cores.  Its own function (not
// inlined) so its registers are allocated independently of the column loop's.
__device__ __noinline__ void lu2_trailing(double* __restrict__ M, int nb, int k0, int kb, const double* sP,
                                          const double* sLi, double* sA, double* sU, const int* sPivT,
                                          const int* sAct) {
  // (72-column chunks -- 13 instead of 16 chunk passes per 225-wide block --
  // measured equal: the pass is bound by the trailing matrix's HBM round trip)
  constexpr int KB = LU2_KB, LDP = LU2_LDP, NW = LU2_T / 32, CW = LU_UCH, CT = CW / 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, c = lane & 3;
      const int nact = nb - (k0 + kb);
      const int nrt = (nact + 7) >> 3;
      for (int cc0 = k0 + kb; cc0 < nb; cc0 += CW) {
#pragma unroll 4
        for (int idx = tid; idx < KB * CW; idx += LU2_T) {
          const int j = idx / CW, t = idx - (idx / CW) * CW;
          const int col = cc0 + t;
          double v = 0.0;
          if (j < kb && col < nb) {
            const int row = sPivT[j];
            v = M[(size_t)row * nb + col];
          }
          sA[j * LU_ULD + t] = v;
        }
        __syncthreads();
        for (int tile = warp; tile < (KB / 8) * CT; tile += NW) {
          const int mt = tile / CT, nt = tile - mt * CT;
          double u[2] = {0.0, 0.0};
#pragma unroll
          for (int ks = 0; ks < KB / 4; ++ks)
            dmma(u, sLi[(8 * mt + r) * LDP + 4 * ks + c], sA[(4 * ks + c) * LU_ULD + 8 * nt + r]);
          const int row = 8 * mt + r, col = 8 * nt + 2 * c;
          sU[row * LU_ULD + col] = u[0];
          sU[row * LU_ULD + col + 1] = u[1];
          if (row < kb) {
            double* mrow = M + (size_t)sPivT[row] * nb;
            if (cc0 + col < nb) mrow[cc0 + col] = u[0];
            if (cc0 + col + 1 < nb) mrow[cc0 + col + 1] = u[1];
          }
        }
        __syncthreads();
        for (int rt = warp; rt < nrt; rt += NW) {
          const bool rv = 8 * rt + r < nact;
          const int row = sAct[rv ? 8 * rt + r : 0];
          double* mrow = M + (size_t)row * nb;
          double acc[CT][2];
#pragma unroll
          for (int nt = 0; nt < CT; ++nt) {
            const int col = cc0 + 8 * nt + 2 * c;
            acc[nt][0] = (rv && col < nb) ? mrow[col] : 0.0;
            acc[nt][1] = (rv && col + 1 < nb) ? mrow[col + 1] : 0.0;
          }
#pragma unroll
          for (int ks = 0; ks < KB / 4; ++ks) {
            const double al = rv ? -sP[row * LDP + 4 * ks + c] : 0.0;
#pragma unroll
            for (int nt = 0; nt < CT; ++nt) dmma(acc[nt], al, sU[(4 * ks + c) * LU_ULD + 8 * nt + r]);
          }
#pragma unroll
          for (int nt = 0; nt < CT; ++nt) {
            const int col = cc0 + 8 * nt + 2 * c;
            if (rv && col < nb) mrow[col] = acc[nt][0];
            if (rv && col + 1 < nb) mrow[col + 1] = acc[nt][1];
          }
        }
        __syncthreads();
      }
}

__global__ void __launch_bounds__(LU2_T, 2) k_lu2(PrecArgs A) {
  extern __shared__ double sm[];
  constexpr int KB = LU2_KB, LDP = LU2_LDP, NW = LU2_T / 32;
  const int nb = A.nb;
  double* sP = sm;                                  // panel rows by storage row [nb][LDP]
  double* sLi = sP + (size_t)nb * LDP;              // L11^{-1} [KB][LDP]
  double* sA = sLi + KB * LDP;                      // A12 chunk [KB][LU_ULD]
  double* sU = sA + KB * LU_ULD;                    // U12 chunk [KB][LU_ULD]
  double* sRow = sU + KB * LU_ULD;                  // the pivot row, broadcast [KB]
  unsigned* sSh = reinterpret_cast<unsigned*>(sRow + KB + 2);   // (sRow[KB]: 1 / pivot) per-warp argmax key halves [8]
  unsigned* sSl = sSh + 8;
  int* sSp = reinterpret_cast<int*>(sSl + 8);       // ... LAPACK positions [8]
  int* sSt = sSp + 8;                               // ... storage rows [8]
  int* sPosJ = sSt + 8;                             // storage row currently at position k0 + j [2]
  int* sPivT = sPosJ + 2;                           // storage rows of the panel's pivots [KB]
  int* sAct = sPivT + KB;                           // compacted active storage rows [LU2_T]
  int* sFpos = sAct + LU2_T;                        // final position per storage row, -1 while active [LU2_T]
  int* sCnt = sFpos + LU2_T;                        // per-warp active counts [8] (+ total)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, c = lane & 3;
  long long t_last = clock64();
  int ph_last = 7;

  for (int cl = blockIdx.x; cl < A.count; cl += gridDim.x) {
    double* M = A.M + (size_t)cl * nb * nb;
    int* piv = A.ipiv + (size_t)cl * nb;
    int pos = tid;                   // LAPACK position of this thread's row
    int fpos = -1;                   // its final position once it has been a pivot
    bool active = tid < nb;
    sFpos[tid] = -1;
    __syncthreads();
    for (int k0 = 0; k0 < nb; k0 += KB) {
      const int kb = nb - k0 < KB ? nb - k0 : KB;
      PROF_MARK(0);
      // (1) the row's panel entries straight into the owning thread's
      //     registers (256 contiguous bytes per row: whole sectors)
      double a[KB];
      {
        bool bad = false;
        const double* mrow = M + (size_t)tid * nb + k0;
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          a[j] = (active && j < kb) ? mrow[j] : 0.0;
          bad |= !isfinite(a[j]);
        }
        if (bad && A.info) atomicOr(A.info, 1);
      }
      PROF_MARK(7);
      // (2) the panel's columns
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        if (j < kb) {                                  // block-uniform
          // idamax over the active rows: key = bits(|a_j|) + 1 (order
          // preserving for non-negative doubles), 0 for a retired row or a
          // NaN (never wins); ties go to the smallest LAPACK position.
          // Hardware warp reductions (REDUX) on the key's halves, then on the
          // position.
          const double av = fabs(a[j]);
          const unsigned long long key = (active && av == av) ? (unsigned long long)__double_as_longlong(av) + 1ull : 0ull;
          unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
          unsigned mhi = __reduce_max_sync(~0u, hi);
          unsigned mlo = __reduce_max_sync(~0u, hi == mhi ? lo : 0u);
          int cand = (hi == mhi && lo == mlo) ? pos : 0x7fffffff;
          int bp = __reduce_min_sync(~0u, cand);
          if (cand == bp) { sSh[warp] = mhi; sSl[warp] = mlo; sSp[warp] = bp; sSt[warp] = tid; }
          if (active && pos == k0 + j) sPosJ[j & 1] = tid;
          __syncthreads();
          hi = lane < NW ? sSh[lane] : 0u;
          lo = lane < NW ? sSl[lane] : 0u;
          const int wp = lane < NW ? sSp[lane] : 0x7fffffff, wt = lane < NW ? sSt[lane] : 0x7fffffff;
          mhi = __reduce_max_sync(~0u, hi);
          mlo = __reduce_max_sync(~0u, hi == mhi ? lo : 0u);
          cand = (hi == mhi && lo == mlo) ? wp : 0x7fffffff;
          bp = __reduce_min_sync(~0u, cand);
          int bt = __reduce_min_sync(~0u, cand == bp ? wt : 0x7fffffff);
          if ((mhi | mlo) == 0u) { bt = sPosJ[j & 1]; bp = k0 + j; }   // all-NaN column: no interchange
          if (tid == bt) {
#pragma unroll
            for (int cc = j; cc < KB; ++cc) sRow[cc] = a[cc];
            // 1 / pivot when that is safe (dgetrf2's sfmin rule), else 0: divide
            sRow[KB] = (a[j] != 0.0 && fabs(a[j]) >= DBL_MIN) ? 1.0 / a[j] : 0.0;
            sPivT[j] = tid;
            piv[k0 + j] = bp;
            active = false;
            fpos = k0 + j;
          } else if (active && pos == k0 + j) {
            pos = bp;                                  // getrf's interchange of positions k0 + j and bp
          }
          __syncthreads();
          const double pv = sRow[j];
          if (pv == 0.0 && tid == 0 && A.info) atomicOr(A.info, 2);
          if (active) {
            double l = a[j];
            const double rp = sRow[KB];
            if (rp != 0.0) l *= rp;
            else if (pv != 0.0) l /= pv;
            a[j] = l;
#pragma unroll
            for (int cc = j + 1; cc < KB; ++cc) a[cc] -= l * sRow[cc];
          }
        }
      }
      PROF_MARK(1);
      // (3) the panel back to shared memory (trailing-update operand) and to
      //     global memory; the active list
      const bool mine = tid < nb && (fpos < 0 || fpos >= k0);
      if (mine) {
#pragma unroll
        for (int j = 0; j < KB; ++j) sP[tid * LDP + j] = a[j];
      }
      sFpos[tid] = tid < nb ? fpos : 0;
      {
        const unsigned bal = __ballot_sync(~0u, active);
        if (lane == 0) sCnt[warp] = __popc(bal);
        __syncthreads();
        int off = 0;
        for (int w = 0; w < warp; ++w) off += sCnt[w];
        if (active) sAct[off + __popc(bal & ((1u << lane) - 1))] = tid;
      }
      if (mine) {
        double* mrow = M + (size_t)tid * nb + k0;
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < kb) mrow[j] = a[j];
      }
      PROF_MARK(3);
      // (4) Linv = L11^{-1} (unit lower; L11 = the pivot rows in pivot order)
      double* sL11 = sA;                              // [KB][LDP], zero beyond kb (sA is free here)
      for (int idx = tid; idx < KB * KB; idx += LU2_T) {
        const int i = idx >> 5, j = idx & 31;
        sL11[i * LDP + j] = (i < kb && j < i) ? sP[sPivT[i] * LDP + j] : 0.0;
      }
      __syncthreads();
      if (tid < KB) {
        // column cc of L11^{-1}: t = e_cc, then t_i -= L_ij t_j for j < i in
        // axpy order -- straight-line, every t_j final before it is used
        const int cc = tid;
        double t[KB];
#pragma unroll
        for (int i = 0; i < KB; ++i) t[i] = i == cc ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < KB - 1; ++j)
#pragma unroll
          for (int i = j + 1; i < KB; ++i) t[i] -= sL11[i * LDP + j] * t[j];
#pragma unroll
        for (int i = 0; i < KB; ++i) sLi[i * LDP + cc] = (i < kb && cc < kb) ? t[i] : 0.0;
      }
      __syncthreads();
      PROF_MARK(4);
      // (5) per 64-column chunk: U12 = Linv A12 (pivot rows), A22 -= L21 U12
      //     (active rows), both on the FP64 tensor cores
      lu2_trailing(M, nb, k0, kb, sP, sLi, sA, sU, sPivT, sAct);
      PROF_MARK(5);
    }
    PROF_MARK(6);
    // (6) rows to their LAPACK positions: 32 columns of every row through
    //     shared memory at a time (all loads of a column block before its stores)
    for (int cb = 0; cb < nb; cb += KB) {
#pragma unroll 4
      for (int idx = tid; idx < nb * KB; idx += LU2_T) {
        const int i = idx >> 5, j = idx & 31;
        if (cb + j < nb) sP[i * LDP + j] = M[(size_t)i * nb + cb + j];
      }
      __syncthreads();
#pragma unroll 4
      for (int idx = tid; idx < nb * KB; idx += LU2_T) {
        const int i = idx >> 5, j = idx & 31;
        if (cb + j < nb) M[(size_t)sFpos[i] * nb + cb + j] = sP[i * LDP + j];
      }
      __syncthreads();
    }
    if (A.perm != nullptr && tid < nb) A.perm[(size_t)cl * nb + fpos] = tid;
    PROF_MARK(2);
    __syncthreads();
  }
}

int launch_lu2(const PrecArgs& A, int nsm, cudaStream_t s) {
  const size_t smem = lu2_smem(A.nb);
  cudaError_t e = cudaFuncSetAttribute(k_lu2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_lu2)", e);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lu2, LU2_T, smem);
  const long long cap = (long long)nsm * (occ > 0 ? occ : 1);
  const int grid = (int)(A.count < cap ? A.count : cap);
  k_lu2<<<grid, LU2_T, smem, s>>>(A);
  e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_lu2 launch", e);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SOLVE_THREADS, 8) k_lu_solve(ElemArgs E, const double* __restrict__ lu,
                                                            const int* __restrict__ ipiv,
                                                            const int* __restrict__ perm, int nb,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y) {
  extern __shared__ double sx[];
  double* sD = sx + nb;                              // diagonal block [32][33]
  int* sp = reinterpret_cast<int*>(sD + 32 * 33);
  const int e = blockIdx.x;
  const int cx = e / E.ncy, cy = e - cx * E.ncy;
  const int n2 = E.n * E.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* L = lu + (size_t)e * nb * nb;
  // (1) x restricted to the cell, rows interchanged (getrs' laswp)
  if (perm != nullptr) {
    for (int l = tid; l < nb; l += SOLVE_THREADS) {
      const int q = __ldg(perm + (size_t)e * nb + l);
      const int comp = q / n2, rem = q - comp * n2;
      sx[l] = __ldg(x + comp * E.ncomp + psi_index(E, cx, cy, rem / E.n, rem % E.n));
    }
  } else {
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
  }
  __syncthreads();
  // (2) forward, unit lower L, 32-row blocks: warp 0 solves the diagonal
  //     block, then every thread updates one row below it (32 loads in
  //     flight).  The barrier wait on warp 0 dominated (ncu: 60 % of the warp
  //     samples), so its critical path holds no global load of the diagonal:
  //     the diagonal block after next is fetched by all threads (8 entries
  //     each, registers) a round ahead into the second shared-memory buffer.
  double* sDn = sD + 32 * 33 + ((nb + 1) / 2) * 1;   // second diagonal buffer (after the int row list)
  auto diag_fetch = [&](int b0n, double (&dn)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * SOLVE_THREADS, i = idx >> 5, j = idx & 31;
      dn[q] = (b0n >= 0 && b0n + i < nb && b0n + j < nb) ? __ldg(L + (size_t)(b0n + i) * nb + b0n + j) : 0.0;
    }
  };
  auto diag_store = [&](double* dst, const double (&dn)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * SOLVE_THREADS;
      dst[(idx >> 5) * 33 + (idx & 31)] = dn[q];
    }
  };
  // Look-ahead: once block k of x is known, warp 0 alone updates the 32 rows
  // of block k + 1 with it and goes straight on to solve block k + 1, while
  // warps 1-3 apply block k to the rows beyond: one barrier per block, and
  // the serial 32-step solve runs under the other warps' panel work.
  auto row_update = [&](int i, int c0, int cs) {
    // sx[i] -= sum_j L[i][c0 + j] sx[c0 + j], j < cs (two chains, k_lu_solve's order)
    const double* Lr = L + (size_t)i * nb + c0;
    double s0 = 0.0, s1 = 0.0;
    if (cs == 32) {
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        s0 += __ldg(Lr + j) * sx[c0 + j];
        s1 += __ldg(Lr + j + 1) * sx[c0 + j + 1];
      }
    } else {
      for (int j = 0; j < cs; ++j) s0 += __ldg(Lr + j) * sx[c0 + j];
    }
    sx[i] -= s0 + s1;
  };
  auto solve_lower = [&](const double* sDc, int b0, int bs) {     // warp 0, unit lower
    double xi = lane < bs ? sx[b0 + lane] : 0.0;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const double xj = __shfl_sync(~0u, xi, j);
      if (j < lane && lane < bs) xi -= sDc[lane * 33 + j] * xj;
    }
    if (lane < bs) sx[b0 + lane] = xi;
  };
  auto solve_upper = [&](const double* sDc, int b0, int bs) {     // warp 0, non-unit upper
    double xi = lane < bs ? sx[b0 + lane] : 0.0;
    for (int j = bs - 1; j >= 0; --j) {
      if (lane == j) xi = xi / sDc[j * 33 + j];
      const double xj = __shfl_sync(~0u, xi, j);
      if (lane < j) xi -= sDc[lane * 33 + j] * xj;
    }
    if (lane < bs) sx[b0 + lane] = xi;
  };
  double dn[8];
  // forward: block 0
  diag_fetch(0, dn);
  diag_store(sD, dn);
  diag_fetch(32 < nb ? 32 : -1, dn);
  __syncthreads();
  if (warp == 0) solve_lower(sD, 0, nb < 32 ? nb : 32);
  diag_store(sDn, dn);
  __syncthreads();
  int cur = 1;                                   // buffer holding the NEXT block's diagonal
  for (int b0 = 0; b0 + 32 < nb; b0 += 32) {
    // x[b0 .. b0 + 32) is final; this round finishes block b1 = b0 + 32
    const int b1 = b0 + 32, bs1 = nb - b1 < 32 ? nb - b1 : 32;
    const double* sDc = cur ? sDn : sD;
    diag_fetch(b1 + 32 < nb ? b1 + 32 : -1, dn);
    if (warp == 0) {
      if (lane < bs1) row_update(b1 + lane, b0, 32);
      __syncwarp();
      solve_lower(sDc, b1, bs1);
    } else {
      for (int i = b1 + 32 + (tid - 32); i < nb; i += SOLVE_THREADS - 32) row_update(i, b0, 32);
    }
    diag_store(cur ? sD : sDn, dn);
    __syncthreads();
    cur ^= 1;
  }
  // (3) backward, upper U (non-unit diagonal): last block first
  const int bl = ((nb - 1) / 32) * 32, bsl = nb - bl;
  diag_fetch(bl, dn);
  diag_store(sD, dn);
  diag_fetch(bl - 32, dn);
  __syncthreads();
  if (warp == 0) solve_upper(sD, bl, bsl);
  diag_store(sDn, dn);
  __syncthreads();
  cur = 1;
  for (int b0 = bl; b0 >= 32; b0 -= 32) {
    // x[b0 .. b0 + bs) is final; this round finishes block b1 = b0 - 32
    const int bs = nb - b0 < 32 ? nb - b0 : 32, b1 = b0 - 32;
    const double* sDc = cur ? sDn : sD;
    diag_fetch(b1 - 32, dn);
    if (warp == 0) {
      row_update(b1 + lane, b0, bs);
      __syncwarp();
      solve_upper(sDc, b1, 32);
    } else {
      for (int i = tid - 32; i < b1; i += SOLVE_THREADS - 32) row_update(i, b0, bs);
    }
    diag_store(cur ? sD : sDn, dn);
    __syncthreads();
    cur ^= 1;
  }
  for (int l = tid; l < nb; l += SOLVE_THREADS) {
    const int comp = l / n2, rem = l - comp * n2;
    y[comp * E.ncomp + psi_index(E, cx, cy, rem / E.n, rem % E.n)] = sx[l];
  }
}

// ---------------------------------------------------------------------------
// Small blocks (nb <= 32, config 4): one warp per block, lane = row, the row
// in registers; pivots by warp argmax, interchanges and the pivot row by
// shuffles (same operation order as the CTA kernel's panel loop).
constexpr int WARP_THREADS = 128;

__device__ __forceinline__ double pivot_mag(double v) {
  const double m = fabs(v);
  return m >= 0.0 ? m : -1.0;     // NaN never wins (the block is flagged non-finite)
}

template <int NBM>
__global__ void __launch_bounds__(WARP_THREADS, NBM > 16 ? 2 : 4) k_lu_warp(PrecArgs A) {
  constexpr int NOPIV = 0x7fffffff;
  const int lane = threadIdx.x & 31;
  const int nb = A.nb;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int cl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; cl < A.count; cl += nw) {
    double* M = A.M + (size_t)cl * nb * nb;
    const bool rv = lane < nb;
    double a[NBM];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < NBM; ++k) {
      double v = 0.0;
      if (rv && k < nb) {
        v = M[lane * nb + k];
        if (A.transform) v = precond_value(A, A.cell0 + cl, lane, k, v);
      }
      a[k] = v;
      bad |= !isfinite(v);
    }
    int info = 0;
    int prow = lane;                      // composed interchanges (row held by this lane)
#pragma unroll
    for (int j = 0; j < NBM; ++j) {
      if (j < nb) {
      double best = (rv && lane >= j) ? pivot_mag(a[j]) : -1.0;
      int bi = (rv && lane >= j && best >= 0.0) ? lane : NOPIV;
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_xor_sync(~0u, best, off);
        const int oi = __shfl_xor_sync(~0u, bi, off);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      const int p = bi == NOPIV ? j : bi;
      if (lane == 0) A.ipiv[(size_t)cl * nb + j] = p;
      if (p != j) {
#pragma unroll
        for (int k = 0; k < NBM; ++k) {
          const double t1 = __shfl_sync(~0u, a[k], p);
          const double t2 = __shfl_sync(~0u, a[k], j);
          if (lane == j) a[k] = t1;
          else if (lane == p) a[k] = t2;
        }
        const int q1 = __shfl_sync(~0u, prow, p);
        const int q2 = __shfl_sync(~0u, prow, j);
        if (lane == j) prow = q1;
        else if (lane == p) prow = q2;
      }
      const double pv = __shfl_sync(~0u, a[j], j);
      if (pv == 0.0) info |= 2;
      const double rp = 1.0 / pv;
      if (rv && lane > j && pv != 0.0) a[j] = fabs(pv) >= DBL_MIN ? a[j] * rp : a[j] / pv;
      const double l = a[j];
#pragma unroll
      for (int k = j + 1; k < NBM; ++k) {
        const double u = __shfl_sync(~0u, a[k], j);
        if (lane > j) a[k] -= l * u;
      }
      }
    }
    if (rv) {
#pragma unroll
      for (int k = 0; k < NBM; ++k)
        if (k < nb) M[lane * nb + k] = a[k];
      if (A.perm != nullptr) A.perm[(size_t)cl * nb + lane] = prow;
    }
    const unsigned anybad = __ballot_sync(~0u, bad);
    if (lane == 0 && A.info && (anybad || info)) atomicOr(A.info, (anybad ? 1 : 0) | info);
  }
}

template <int NBM>
__global__ void __launch_bounds__(WARP_THREADS) k_lu_solve_warp(ElemArgs E, const double* __restrict__ lu,
                                                                const int* __restrict__ ipiv, int nb,
                                                                const double* __restrict__ x,
                                                                double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= E.N) return;
  const int cx = e / E.ncy, cy = e - cx * E.ncy;
  const int n2 = E.n * E.n;
  const bool rv = lane < nb;
  const double* L = lu + (size_t)e * nb * nb;
  double r[NBM];
#pragma unroll
  for (int k = 0; k < NBM; ++k) r[k] = (rv && k < nb) ? __ldg(L + lane * nb + k) : 0.0;
  long long gi = 0;
  double xv = 0.0;
  int pv = lane;
  if (rv) {
    const int comp = lane / n2, rem = lane - comp * n2;
    gi = comp * E.ncomp + psi_index(E, cx, cy, rem / E.n, rem % E.n);
    xv = __ldg(x + gi);
    pv = __ldg(ipiv + (size_t)e * nb + lane);
  }
#pragma unroll
  for (int j = 0; j < NBM; ++j) {
    if (j >= nb) break;
    const int p = __shfl_sync(~0u, pv, j);
    if (p != j) {
      const double t1 = __shfl_sync(~0u, xv, p);
      const double t2 = __shfl_sync(~0u, xv, j);
      if (lane == j) xv = t1;
      else if (lane == p) xv = t2;
    }
  }
#pragma unroll
  for (int j = 0; j < NBM; ++j) {
    if (j >= nb) break;
    const double xj = __shfl_sync(~0u, xv, j);
    if (lane > j) xv -= r[j] * xj;
  }
#pragma unroll
  for (int j = NBM - 1; j >= 0; --j) {
    if (j < nb) {
      if (lane == j) xv = xv / r[j];
      const double xj = __shfl_sync(~0u, xv, j);
      if (lane < j) xv -= r[j] * xj;
    }
  }
  if (rv) y[gi] = xv;
}

template <int NBM>
int launch_lu_warp_t(const PrecArgs& A, int nsm, cudaStream_t s) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lu_warp<NBM>, WARP_THREADS, 0);
  const long long need = ((long long)A.count * 32 + WARP_THREADS - 1) / WARP_THREADS;
  const long long cap = (long long)nsm * (occ > 0 ? occ : 1);
  k_lu_warp<NBM><<<(int)(need < cap ? need : cap), WARP_THREADS, 0, s>>>(A);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_lu_warp launch", e);
}

template <int NBM>
int launch_lu_solve_warp_t(const ElemArgs& E, const double* lu, const int* ipiv, int nb, const double* x,
                           double* y, cudaStream_t s) {
  const int grid = (int)(((long long)E.N * 32 + WARP_THREADS - 1) / WARP_THREADS);
  k_lu_solve_warp<NBM><<<grid, WARP_THREADS, 0, s>>>(E, lu, ipiv, nb, x, y);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_lu_solve_warp launch", e);
}

template <int KB>
size_t lu_smem(int nb) {
  return sizeof(double) * ((size_t)(nb + KB) * (KB + 1) + 2 * KB * LU_ULD + 8) + sizeof(int) * (8 + 3 * KB + 1 + nb);
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
  return (int)((LU_SMEM_CAP - sizeof(double) * (8 * 9 + 16 * LU_ULD + 8) - sizeof(int) * 33) / (sizeof(double) * 9 + sizeof(int)));
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
  if (A.nb > lu_max_nb() && lu_big_supported(A.nb)) {
    // blocks beyond the one-CTA panel (config 3): cluster-panel blocked LU
    if (A.transform) {
      int rc = launch_precond_transform(A, s);
      if (rc) return rc;
    }
    PrecArgs B = A;
    B.transform = 0;
    return launch_lu_big(B, s);
  }
  if (A.nb <= 8) return launch_lu_warp_t<8>(A, nsm, s);
  if (A.nb <= 16) return launch_lu_warp_t<16>(A, nsm, s);
  if (A.nb <= 32) return launch_lu_warp_t<32>(A, nsm, s);
  // one row per thread, implicit pivoting (config 1)
  if (A.nb <= LU2_T && getenv("HPG_LU2_OFF") == nullptr) {
    if (A.transform) {
      int rc = launch_precond_transform(A, s);
      if (rc) return rc;
    }
    PrecArgs B = A;
    B.transform = 0;
    return launch_lu2(B, nsm, s);
  }
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

int launch_lu_solve(const ElemArgs& E, const double* lu, const int* ipiv, const int* perm, int nb,
                    const double* x, double* y, cudaStream_t s) {
  if (nb <= 8) return launch_lu_solve_warp_t<8>(E, lu, ipiv, nb, x, y, s);
  if (nb <= 16) return launch_lu_solve_warp_t<16>(E, lu, ipiv, nb, x, y, s);
  if (nb <= 32) return launch_lu_solve_warp_t<32>(E, lu, ipiv, nb, x, y, s);
  const size_t smem = (sizeof(double) + sizeof(int)) * (size_t)nb + sizeof(double) * 2 * 32 * 33 + 32;
  if (smem > (48u << 10)) {
    cudaError_t e = cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_lu_solve)", e);
  }
  k_lu_solve<<<E.N, SOLVE_THREADS, smem, s>>>(E, lu, ipiv, perm, nb, x, y);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HPG_OK : set_error(HPG_ERR_CUDA, "k_lu_solve launch", e);
}

}  // namespace hpg
