// Shared device helpers for the hpG element-quadrature kernels (sm_100a, fp64).
//
// FP64 tensor-core path on Blackwell: tcgen05.mma has no f64 kind, so the
// FP64 tensor cores are reached through mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4,
// measured 37.2 TF/s on this pool's B200: profiles/fp64_peaks_r01.json).
//
// Fragment layouts of m8n8k4 (lane = r*4 + c, r = lane>>2, c = lane&3):
//   A (8x4):  A[r][c]            B (4x8):  B[c][r]
//   C/D (8x8): C[r][2c], C[r][2c+1]
// "Permuted K" trick used throughout: a C fragment of an 8x8 tile is directly
// the A fragment (rows r) -- and, transposed, the B fragment (cols r) -- of
// the next contraction if that contraction's K index runs over the tile's
// columns in the order {0,2,4,6} (k-step 2t) then {1,3,5,7} (k-step 2t+1).
// The other operand of such a contraction is a table read in the matching
// permuted order: PK(X)[tile][ks][lane] = X[8*tile + r][8*(ks>>1) + 2c + (ks&1)].
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "hpg_invodd.cuh"

namespace hpg {

constexpr double EXP_CLAMP = 700.0;   // hpgalerkin/assembly.py:25

// Programmatic dependent launch (PDL).  Kernels of the hot path are launched
// with programmatic stream serialization so their launch (and, where noted,
// a data-independent prologue) overlaps the previous kernel's tail; every
// such kernel executes pdl_wait() before it touches memory written by
// earlier work (a no-op for a kernel launched without the attribute).
// 8-byte global -> shared copy, zero fill when !valid (src must still be a
// mapped address)
__device__ __forceinline__ void cp_async8z(double* dst, const double* src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(valid ? 8 : 0) : "memory");
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// exp(min(-v, 700)) with the reference's overflow flag (assembly.py:187-192):
// flagged iff -v > 700 or v is NaN; underflow to 0 is legitimate.  A select,
// not fmin: fmin(NaN, 700) would return 700 where the reference keeps NaN.
__device__ __forceinline__ double clamped_exp_neg(double v, bool& flag) {
  double t = -v;
  bool over = t > EXP_CLAMP;
  flag |= over || (v != v);
  return exp(over ? EXP_CLAMP : t);
}

// ---------------------------------------------------------------------------
// Per-launch arguments (plain pointers; no torch types).
struct ElemArgs {
  int ncx, ncy, n, m, p, nq, N;
  int nix, niy;
  long long ld;      // row stride of the x-major psi array (= ncy*n)
  long long ncomp;   // psi dofs per component
  const double* hx;
  const double* hy;
  const double* Sf;  // PK(S): [QT][NP/4][32]
  const double* Tf;  // PK(T): [NT][QP/4][32]
  const double* in0; // psi (or values for M_VALUES)
  const double* in1; // direction x
  const double* phi; // gradient point samples, (N, nq, nq)
  const double* wc_in;
  double* wc_out;
  double* out;
  int* flag;
  int residual;      // 1: out = phi_mom - B^T u - M (obstacle) | M - B^T u (gradient)
  const double* phi_mom;
  const double* u;
  // generic (CTA) path only
  int NT, QT, splits;
  double* partial;   // [N][splits][NOUT][NP*NP] when splits > 1
  int out_cellmajor; // M_VALUES for the u side: out is (N, n, n) cell-major
  int smem_tables;   // CTA path: PK(S), PK(T) staged in shared memory
  int cluster_red;   // CTA path, splits > 1: the split CTAs of a cell form a
                     // thread-block cluster and reduce through DSMEM
  // fused residual U side (hpg_ucell.cuh)
  double alpha;
  const double* psi_prev;
  const double* f_load;
  double* b_u;
  double* edge;      // [N][4m-4] hat-involved local contributions
  int usmem;         // doubles of U-side shared memory per thread group
  double* ubuf;      // CTA path, large m: U-side buffers in global scratch [N][usmem]
  int e0;            // warp / streaming cached apply: first cell of the range
                     // [e0, N) (hpgApplyCachedRange); 0 everywhere else
  int wc_early;      // cached apply: the weight cache was not written by the
                     // immediately preceding kernel, so it may be prefetched
                     // before griddepcontrol.wait (hpgApplyCached decides)
};

struct WarpSync { __device__ __forceinline__ void operator()() const { __syncwarp(); } };
struct BlockSync { __device__ __forceinline__ void operator()() const { __syncthreads(); } };

// 1D interior dof -> contributing (cell, local index) pairs, fixed order.
__device__ __forceinline__ int u_owners_1d_dev(int i, int nc, int p, int* cell, int* loc) {
  if (i < nc - 1) {
    int v = i + 1;
    cell[0] = v - 1; loc[0] = 1;
    cell[1] = v; loc[1] = 0;
    return 2;
  }
  int b = i - (nc - 1);
  cell[0] = b / (p - 1);
  loc[0] = 2 + b % (p - 1);
  return 1;
}

enum Mode : int {
  M_OBST_RES = 0,     // psi -> exp moments (+ weight cache, flag)
  M_OBST_APPLY = 1,   // psi, x -> D x   (weights recomputed)
  M_OBST_CACHED = 2,  // cache, x -> D x
  M_GRAD_RES = 3,     // psi_x, psi_y, phi -> nl moments (+ cache: kxx, kxy, kyy)
  M_GRAD_APPLY = 4,   // psi, x, phi -> D x
  M_GRAD_CACHED = 5,  // cache, x -> D x
  M_VALUES = 6,       // point values -> moments (data_moments, load_vector)
};

template <int MODE> struct ModeTraits;
template <> struct ModeTraits<M_OBST_RES>    { static constexpr int NIN = 1, NSYN = 1, NOUT = 1, NW = 1; };
template <> struct ModeTraits<M_OBST_APPLY>  { static constexpr int NIN = 2, NSYN = 2, NOUT = 1, NW = 1; };
template <> struct ModeTraits<M_OBST_CACHED> { static constexpr int NIN = 1, NSYN = 1, NOUT = 1, NW = 1; };
template <> struct ModeTraits<M_GRAD_RES>    { static constexpr int NIN = 2, NSYN = 2, NOUT = 2, NW = 3; };
template <> struct ModeTraits<M_GRAD_APPLY>  { static constexpr int NIN = 4, NSYN = 4, NOUT = 2, NW = 3; };
template <> struct ModeTraits<M_GRAD_CACHED> { static constexpr int NIN = 2, NSYN = 2, NOUT = 2, NW = 3; };
template <> struct ModeTraits<M_VALUES>      { static constexpr int NIN = 0, NSYN = 0, NOUT = 1, NW = 0; };

// Global address of psi-side tile entry (a, b) of cell (cx, cy), component f.
__device__ __forceinline__ long long psi_index(const ElemArgs& A, int cx, int cy, int a, int b) {
  return (long long)(cx * A.n + a) * A.ld + (long long)cy * A.n + b;
}

// Interior index of cell-local U dof j in 1D (-1 on the boundary).
// Local order [hat_L, hat_R, W_0..W_{p-2}] (spaces.py:40-43); the 1D interior
// numbering is hats 1..nc-1 then bubbles cell by cell (spaces.py:25-38).
__device__ __forceinline__ int u_local_1d(int c, int j, int nc, int p) {
  if (j == 0) return c >= 1 ? c - 1 : -1;
  if (j == 1) return c + 1 <= nc - 1 ? c : -1;
  return (nc - 1) + c * (p - 1) + (j - 2);
}

__device__ __forceinline__ double u_at(const ElemArgs& A, int cx, int cy, int i, int j) {
  int ix = u_local_1d(cx, i, A.ncx, A.p);
  int iy = u_local_1d(cy, j, A.ncy, A.p);
  if (ix < 0 || iy < 0) return 0.0;
  return __ldg(A.u + (long long)ix * A.niy + iy);
}

// Row a of the U->Legendre map R (spaces.py:45-57): up to 3 (col, coef).
__device__ __forceinline__ int legendre_row(int a, int p, int* col, double* coef) {
  int k = 0;
  if (a == 0) { col[k] = 0; coef[k++] = 0.5; col[k] = 1; coef[k++] = 0.5; }
  if (a == 1) { col[k] = 0; coef[k++] = -0.5; col[k] = 1; coef[k++] = 0.5; }
  if (a <= p - 2) { col[k] = 2 + a; coef[k++] = kInvOdd[a + 1]; }
  if (a >= 2 && a - 2 <= p - 2) { col[k] = a; coef[k++] = -kInvOdd[a - 1]; }
  return k;
}

// Row i of the derivative map D (spaces.py:59-68).
__device__ __forceinline__ int deriv_row(int i, int p, int* col, double* coef) {
  int k = 0;
  if (i == 0) { col[k] = 0; coef[k++] = -0.5; col[k] = 1; coef[k++] = 0.5; }
  if (i >= 1 && i - 1 <= p - 2) { col[k] = 2 + (i - 1); coef[k++] = -1.0; }
  return k;
}

// (B^T u) at psi-tile entry (a, b) of cell (cx, cy), component comp
// (assembly.py:81-116,475-477,725-729):
//   obstacle:  wx_a wy_b (Rx C Ry^T)[a][b]
//   gradient x: (2/(2a+1)) (Dx C Ry^T)[a][b] wy_b ; y: wx_a (Rx C Dy^T)[a][b] (2/(2b+1))
__device__ __forceinline__ double btu_value(const ElemArgs& A, bool gradient, int comp,
                                            int cx, int cy, int a, int b,
                                            double wa, double wb) {
  int ci[3], cj[3];
  double ai[3], aj[3];
  int ni, nj;
  if (gradient && comp == 0) ni = deriv_row(a, A.p, ci, ai); else ni = legendre_row(a, A.p, ci, ai);
  if (gradient && comp == 1) nj = deriv_row(b, A.p, cj, aj); else nj = legendre_row(b, A.p, cj, aj);
  double s = 0.0;
  for (int x = 0; x < ni; ++x) {
    double t = 0.0;
    for (int y = 0; y < nj; ++y) t += aj[y] * u_at(A, cx, cy, ci[x], cj[y]);
    s += ai[x] * t;
  }
  double fa = wa, fb = wb;
  if (gradient && comp == 0) fa = 2.0 * kInvOdd[a];
  if (gradient && comp == 1) fb = 2.0 * kInvOdd[b];
  return (fa * s) * fb;
}

}  // namespace hpg
