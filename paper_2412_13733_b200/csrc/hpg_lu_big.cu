// Blocked LU with partial pivoting for per-cell blocks too tall for the
// one-CTA panel of k_lu (config 3: 16 blocks of 6561^2; SURVEY.md §8f rank 1,
// scipy lu_factor = LAPACK getrf, linalg.py:249).  Right-looking, 32-column
// panels, every step batched over the cells:
//
//   k_panel_cluster   the panel [k0, nb) x [k0, k0+32) spread over the shared
//                     memory of a cluster of 8 CTAs per cell; per column a
//                     cluster-wide argmax (first maximal |a|, LAPACK idamax),
//                     the row interchange through distributed shared memory,
//                     scaling by 1/pivot when that is safe (dgetf2) and the
//                     rank-1 update of the rest of the panel -- two cluster
//                     barriers per column, no global round trips
//   k_laswp           the panel's interchanges applied, in order, to every
//                     other column (dlaswp), one thread per column
//   k_trsm_unit       U12 = L11^{-1} A12 (unit lower, column-oriented axpy
//                     order as dtrsm), one thread per column
//   k_dgemm_nn        A22 -= L21 U12 on the FP64 tensor cores (hpg_gemm.cuh,
//                     accumulate form, batched over the cells)
//
// ipiv is 0-based per cell like scipy's piv; info |= 1 on a non-finite entry
// (scipy's check_finite raises), |= 2 on an exactly zero pivot (LAPACK info > 0).
#include <cooperative_groups.h>

#include <cfloat>

#include "../../include/hpg_b200.h"
#include "hpg_gemm.cuh"
#include "hpg_launch.cuh"
#include "hpg_precond.cuh"

namespace hpg {

namespace {

namespace cg = cooperative_groups;

constexpr int LB_KB = 32;      // panel width
constexpr int LB_CL = 8;       // CTAs per cell (cluster size)
constexpr int LB_T = 256;      // threads per CTA
constexpr int LB_LDP = LB_KB + 1;

struct LuBig {
  double* M;
  int nb, k0, count;
  int* ipiv;
  int* info;
};

size_t panel_smem(int nb) {
  const int chunk = (nb + LB_CL - 1) / LB_CL;
  return sizeof(double) * ((size_t)chunk * LB_LDP + 2 * LB_KB + 2 * (LB_T / 32) + 4) + sizeof(int) * (LB_T / 32 + 4);
}

__global__ void __cluster_dims__(LB_CL, 1, 1) __launch_bounds__(LB_T, 1) k_panel_cluster(LuBig A) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int cell = blockIdx.x / LB_CL;
  const int nb = A.nb, k0 = A.k0, rows = nb - k0;
  const int kb = rows < LB_KB ? rows : LB_KB;
  const int chunk = (rows + LB_CL - 1) / LB_CL;      // panel rows per CTA
  const int r0 = rank * chunk < rows ? rank * chunk : rows;
  const int r1 = r0 + chunk < rows ? r0 + chunk : rows;
  double* sP = sm;                                   // my panel rows [r1 - r0][LDP]
  double* urow = sP + (size_t)chunk * LB_LDP;        // pivot row (after the interchange)
  double* orow = urow + LB_KB;                       // old row j (pivot owner only)
  double* sRv = orow + LB_KB;                        // per-warp argmax values
  double* sCand = sRv + LB_T / 32;                   // [0] my candidate value, [1] broadcast pivot value
  int* sRi = reinterpret_cast<int*>(sCand + 4);      // per-warp argmax rows
  int* sCandR = sRi + LB_T / 32;                     // [0] my candidate row, [1] chosen pivot row
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* M = A.M + (size_t)cell * nb * nb;
  constexpr int NOPIV = 0x7fffffff;

  bool bad = false;
  for (int idx = tid; idx < (r1 - r0) * LB_KB; idx += LB_T) {
    const int i = idx / LB_KB, j = idx - (idx / LB_KB) * LB_KB;
    const double v = j < kb ? M[(size_t)(k0 + r0 + i) * nb + k0 + j] : 0.0;
    sP[i * LB_LDP + j] = v;
    bad |= !isfinite(v);
  }
  if (bad && A.info) atomicOr(A.info, 1);
  __syncthreads();

  for (int j = 0; j < kb; ++j) {
    // (1) my rows' candidate: first maximal |a_ij|, i >= j
    double best = -1.0;
    int bi = NOPIV;
    for (int i = (r0 > j ? r0 : j) + tid; i < r1; i += LB_T) {
      const double v = fabs(sP[(i - r0) * LB_LDP + j]);
      if (v > best) { best = v; bi = i; }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double ov = __shfl_xor_sync(~0u, best, off);
      const int oi = __shfl_xor_sync(~0u, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { sRv[warp] = best; sRi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < LB_T / 32; ++w)
        if (sRv[w] > best || (sRv[w] == best && sRi[w] < bi)) { best = sRv[w]; bi = sRi[w]; }
      sCand[0] = best;
      sCandR[0] = bi;
    }
    cl.sync();                                        // [A] candidates published, rows final
    // (2) the cluster's pivot (ranks hold ascending rows: ties -> lowest row)
    if (warp == 0) {
      double v = -1.0;
      int ri = NOPIV;
      if (lane < LB_CL) {
        v = *cl.map_shared_rank(sCand, lane);
        ri = *cl.map_shared_rank(sCandR, lane);
      }
#pragma unroll
      for (int off = 4; off; off >>= 1) {
        const double ov = __shfl_xor_sync(~0u, v, off);
        const int oi = __shfl_xor_sync(~0u, ri, off);
        if (ov > v || (ov == v && oi < ri)) { v = ov; ri = oi; }
      }
      if (lane == 0) {
        const int p = ri == NOPIV ? j : ri;           // all-NaN column: no interchange
        sCandR[1] = p;
        if (rank == 0) A.ipiv[(size_t)cell * nb + k0 + j] = k0 + p;
      }
    }
    __syncthreads();
    const int p = sCandR[1];
    const int own_p = p / chunk, own_j = j / chunk;
    if (tid < LB_KB) {
      urow[tid] = cl.map_shared_rank(sP, own_p)[(p - own_p * chunk) * LB_LDP + tid];
      if (rank == own_p && p != j) orow[tid] = cl.map_shared_rank(sP, own_j)[(j - own_j * chunk) * LB_LDP + tid];
    }
    cl.sync();                                        // [B] every remote read done
    if (p != j && tid < LB_KB) {
      if (rank == own_j) sP[(j - r0) * LB_LDP + tid] = urow[tid];
      if (rank == own_p) sP[(p - r0) * LB_LDP + tid] = orow[tid];
    }
    // (3) scale column j below the pivot and update the rest of the panel
    const double pv = urow[j];
    if (pv == 0.0 && rank == 0 && tid == 0 && A.info) atomicOr(A.info, 2);
    const bool recip = fabs(pv) >= DBL_MIN;
    const double rp = 1.0 / pv;
    __syncthreads();
    for (int i = (r0 > j + 1 ? r0 : j + 1) + tid; i < r1; i += LB_T) {
      double* row = sP + (i - r0) * LB_LDP;
      double l = row[j];
      if (pv != 0.0) l = recip ? l * rp : l / pv;
      row[j] = l;
      for (int cc = j + 1; cc < kb; ++cc) row[cc] -= l * urow[cc];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < (r1 - r0) * kb; idx += LB_T) {
    const int i = idx / kb, j = idx - (idx / kb) * kb;
    M[(size_t)(k0 + r0 + i) * nb + k0 + j] = sP[i * LB_LDP + j];
  }
  cl.sync();                                          // no CTA exits while others read its smem
}

// the panel's interchanges, in order, on every column outside it
__global__ void k_laswp(LuBig A, int kb) {
  const int cell = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = A.nb, k0 = A.k0;
  if (col >= nb || (col >= k0 && col < k0 + kb)) return;
  double* M = A.M + (size_t)cell * nb * nb;
  const int* piv = A.ipiv + (size_t)cell * nb;
  for (int j = 0; j < kb; ++j) {
    const int p = __ldg(piv + k0 + j);
    if (p != k0 + j) {
      const double t = M[(size_t)(k0 + j) * nb + col];
      M[(size_t)(k0 + j) * nb + col] = M[(size_t)p * nb + col];
      M[(size_t)p * nb + col] = t;
    }
  }
}

// U12 = L11^{-1} A12: column-oriented (dtrsm Left/Lower/NoTrans/Unit) per column
__global__ void k_trsm_unit(LuBig A, int kb) {
  __shared__ double sL[LB_KB][LB_KB + 1];
  const int cell = blockIdx.y;
  const int nb = A.nb, k0 = A.k0;
  double* M = A.M + (size_t)cell * nb * nb;
  for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
    const int i = idx / kb, j = idx - (idx / kb) * kb;
    sL[i][j] = M[(size_t)(k0 + i) * nb + k0 + j];
  }
  __syncthreads();
  const int col = k0 + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= nb) return;
  double x[LB_KB];
#pragma unroll
  for (int i = 0; i < LB_KB; ++i) x[i] = i < kb ? M[(size_t)(k0 + i) * nb + col] : 0.0;
#pragma unroll
  for (int k = 0; k < LB_KB; ++k) {
    const double xk = x[k];
    if (xk != 0.0) {
#pragma unroll
      for (int i = k + 1; i < LB_KB; ++i)
        if (i < kb) x[i] -= xk * sL[i][k];
    }
  }
#pragma unroll
  for (int i = 0; i < LB_KB; ++i)
    if (i < kb) M[(size_t)(k0 + i) * nb + col] = x[i];
}

__global__ void k_check_finite(const double* __restrict__ M, long long n, int* info) {
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(M[i]);
  if (__any_sync(~0u, bad) && (threadIdx.x & 31) == 0 && info) atomicOr(info, 1);
}

// composed interchanges per cell: position i <- row perm[i]
__global__ void k_compose_perm(const int* __restrict__ ipiv, int* __restrict__ perm, int nb, int count) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= count) return;
  int* pm = perm + (size_t)cell * nb;
  const int* pv = ipiv + (size_t)cell * nb;
  for (int i = 0; i < nb; ++i) pm[i] = i;
  for (int i = 0; i < nb; ++i) {
    const int p = pv[i];
    if (p != i) {
      const int t = pm[i];
      pm[i] = pm[p];
      pm[p] = t;
    }
  }
}

}  // namespace

bool lu_big_supported(int nb) { return panel_smem(nb) <= (227u << 10); }

int launch_lu_big(const PrecArgs& P, cudaStream_t s) {
  const int nb = P.nb, count = P.count;
  if (!lu_big_supported(nb)) return set_error_msg(HPG_ERR_UNSUPPORTED, "blocked LU: block side too large");
  const size_t smem = panel_smem(nb);
  struct Memo { size_t attr = 0; };
  static PerDevice<Memo> memo;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (smem > m.attr) {
      cudaError_t e = cudaFuncSetAttribute(k_panel_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      m.attr = smem;
    }
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_panel_cluster)", se);
  LuBig A{P.M, nb, 0, count, P.ipiv, P.info};
  if (P.info) {
    k_check_finite<<<148 * 8, 256, 0, s>>>(P.M, (long long)nb * nb * count, P.info);
  }
  for (int k0 = 0; k0 < nb; k0 += LB_KB) {
    A.k0 = k0;
    const int kb = nb - k0 < LB_KB ? nb - k0 : LB_KB;
    k_panel_cluster<<<count * LB_CL, LB_T, smem, s>>>(A);
    k_laswp<<<dim3((nb + 255) / 256, count), 256, 0, s>>>(A, kb);
    const int rest = nb - k0 - kb;
    if (rest > 0) {
      k_trsm_unit<<<dim3((rest + 127) / 128, count), 128, 0, s>>>(A, kb);
      double* base = P.M + (size_t)k0 * nb + k0;
      GemmNN g = gemm_nn(rest, rest, kb, base + (size_t)kb * nb, nb, base + kb, nb,
                         base + (size_t)kb * nb + kb, nb);
      g.sA = g.sB = g.sC = (long long)nb * nb;
      g.alpha = -1.0;
      g.beta = 1.0;
      cudaError_t e = dgemm_nn(g, count, s);
      if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "blocked LU update", e);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "blocked LU step", e);
  }
  if (P.perm) {
    k_compose_perm<<<(count + 31) / 32, 32, 0, s>>>(P.ipiv, P.perm, nb, count);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "k_compose_perm", e);
  }
  return HPG_OK;
}

}  // namespace hpg
