// Warp-per-cell U side of the residual for mid degrees (UPASS_PMIN..PMAX):
// separable 1D passes with literal coefficients (hpg_upass_gen.cuh,
// tools/gen_upass.py) over m x m shared-memory tiles, one lane per row or
// column.  Same outputs as k_usmall / k_uside_pt:
//   b_psi <- phi_moments - B^T u (obstacle) | -B^T u (gradient),
//   b_u on owned dofs, edge scratch for the hat-involved ones.
#include "hpg_common.cuh"
#include "hpg_launch.cuh"
#include "hpg_upass_gen.cuh"

namespace hpg {
namespace {

constexpr int UPW = 4;   // warps (cells in flight) per CTA

// shared-memory tiles per warp: the obstacle pass order below needs 3, the
// gradient one (two psi components) 5
template <bool G>
constexpr int upass_bufs() { return G ? 5 : 3; }

// Obstacle U side with three m x m buffers per warp (more cells resident per
// SM than the 5-buffer order; config 1 keeps every cell in flight at once).
template <int P>
__device__ __forceinline__ void upass_obstacle(const ElemArgs& A, int e, int lane, double* B0, double* B1,
                                               double* B2) {
  using U = UPass<P>;
  constexpr int M = U::M, LD = U::LD, N = P - 1;
  const int cx = e / A.ncy, cy = e - cx * A.ncy;
  const double hx = A.hx[cx], hy = A.hy[cy];
  const long long base = psi_index(A, cx, cy, 0, 0);
  // C: local U tile (lane = column)
  if (lane < M) {
    const int iy = u_local_1d(cy, lane, A.ncy, P);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int ix = u_local_1d(cx, i, A.ncx, P);
      B0[i * LD + lane] = (ix < 0 || iy < 0) ? 0.0 : __ldg(A.u + (long long)ix * A.niy + iy);
    }
  }
  __syncwarp();
  // B^T u -> b_psi
  U::yR(B0, B1, M, N, 1.0, false, lane);              // C R^T
  __syncwarp();
  U::xR(B1, B2, N, N, 1.0, false, lane);              // R C R^T
  __syncwarp();
  if (lane < N) {
    const double wb = hy * kInvOdd[lane];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const long long g = base + (long long)a * A.ld + lane;
      A.out[g] = __ldg(A.phi_mom + g) - ((hx * kInvOdd[a]) * B2[a * LD + lane]) * wb;
    }
  }
  __syncwarp();
  // A u = (hy/hx) K (C Mref) + (hx/hy) (diag R (C K))^T-pass  -> B2
  U::yRM(B0, B1, M, M, 1.0, false, lane);             // C R^T diag(1/(2l+1))
  U::yK(B0, B2, M, M, 1.0, false, lane);              // C K
  __syncwarp();
  U::yRT(B1, B0, M, M, 1.0, false, lane);             // C Mref
  __syncwarp();
  U::xRM(B2, B1, M, M, 1.0, false, lane);             // diag R (C K)
  __syncwarp();
  U::xK(B0, B2, M, M, hy / hx, false, lane);          // (hy/hx) K C Mref
  U::xRT(B1, B2, M, M, hx / hy, true, lane);          // + (hx/hy) Mref C K
  __syncwarp();
  // B (psi_prev - psi) -> B1
  if (lane < M) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double g = 0.0;
      if (i < N && lane < N) {
        const long long gi = base + (long long)i * A.ld + lane;
        const double d = __ldg(A.psi_prev + gi) - __ldg(A.in0 + gi);
        g = ((hx * kInvOdd[i]) * d) * (hy * kInvOdd[lane]);
      }
      B0[i * LD + lane] = g;
    }
  }
  __syncwarp();
  U::yRT(B0, B1, M, M, 1.0, false, lane);             // G R
  __syncwarp();
  U::xRT(B1, B0, M, M, 1.0, false, lane);             // R^T (.)
  __syncwarp();
  // r = -alpha A u + B dpsi (lane = column k)
  if (lane < M) {
    const int k = lane;
    double* edge = A.edge + (long long)e * (4 * M - 4);
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double r = -A.alpha * B2[j * LD + k] + B0[j * LD + k];
      if (j >= 2 && k >= 2) {
        const long long ix = (A.ncx - 1) + (long long)cx * (P - 1) + (j - 2);
        const long long iy = (A.ncy - 1) + (long long)cy * (P - 1) + (k - 2);
        const long long g = ix * A.niy + iy;
        A.b_u[g] = A.alpha * __ldg(A.f_load + g) + r;
      } else if (j < 2) {
        edge[j * M + k] = r;
      } else {
        edge[2 * M + (j - 2) * 2 + k] = r;
      }
    }
  }
  __syncwarp();
}

template <int P, bool G>
__global__ void __launch_bounds__(32 * UPW, G ? 1 : 8) k_upass(ElemArgs A) {
  pdl_wait();
  using U = UPass<P>;
  constexpr int M = U::M, LD = U::LD, BUF = M * LD, N = G ? P : P - 1;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (!G) {
    double* W0 = smem + (size_t)warp * 3 * BUF;
    for (int e = blockIdx.x * UPW + warp; e < A.N; e += gridDim.x * UPW)
      upass_obstacle<P>(A, e, lane, W0, W0 + BUF, W0 + 2 * BUF);
    return;
  }
  double* B0 = smem + (size_t)warp * 5 * BUF;
  double* B1 = B0 + BUF;
  double* B2 = B1 + BUF;
  double* B3 = B2 + BUF;
  double* B4 = B3 + BUF;
  for (int e = blockIdx.x * UPW + warp; e < A.N; e += gridDim.x * UPW) {
    const int cx = e / A.ncy, cy = e - cx * A.ncy;
    const double hx = A.hx[cx], hy = A.hy[cy];
    const long long base = psi_index(A, cx, cy, 0, 0);
    // C: local U tile (lane = column)
    if (lane < M) {
      const int iy = u_local_1d(cy, lane, A.ncy, P);
      for (int i = 0; i < M; ++i) {
        const int ix = u_local_1d(cx, i, A.ncx, P);
        B0[i * LD + lane] = (ix < 0 || iy < 0) ? 0.0 : __ldg(A.u + (long long)ix * A.niy + iy);
      }
    }
    __syncwarp();
    // B^T u  ->  b_psi
    if constexpr (!G) {
      U::yR(B0, B1, M, N, 1.0, false, lane);            // C R^T
      __syncwarp();
      U::xR(B1, B2, N, N, 1.0, false, lane);            // R C R^T
      __syncwarp();
      if (lane < N) {
        const double wb = hy * kInvOdd[lane];
        for (int a = 0; a < N; ++a) {
          const long long g = base + (long long)a * A.ld + lane;
          A.out[g] = __ldg(A.phi_mom + g) - ((hx * kInvOdd[a]) * B2[a * LD + lane]) * wb;
        }
      }
    } else {
      U::yR(B0, B1, M, N, 1.0, false, lane);            // C R^T
      U::yD(B0, B3, M, N, 1.0, false, lane);            // C D^T
      __syncwarp();
      U::xD(B1, B2, N, N, 1.0, false, lane);            // D C R^T
      U::xR(B3, B4, N, N, 1.0, false, lane);            // R C D^T
      __syncwarp();
      if (lane < N) {
        for (int a = 0; a < N; ++a) {
          const long long g = base + (long long)a * A.ld + lane;
          A.out[g] = -(((2.0 * kInvOdd[a]) * B2[a * LD + lane]) * (hy * kInvOdd[lane]));
          A.out[A.ncomp + g] = -(((hx * kInvOdd[a]) * B4[a * LD + lane]) * (2.0 * kInvOdd[lane]));
        }
      }
    }
    __syncwarp();
    // A u = (hy/hx) K (C R^T diag R) + (hx/hy) (R^T diag R) (C K)   -> B1
    U::yRM(B0, B1, M, M, 1.0, false, lane);             // C R^T diag(1/(2l+1))
    U::yK(B0, B2, M, M, 1.0, false, lane);              // C K
    __syncwarp();
    U::yRT(B1, B3, M, M, 1.0, false, lane);             // C Mref
    U::xRM(B2, B4, M, M, 1.0, false, lane);             // diag R (C K)
    __syncwarp();
    U::xK(B3, B1, M, M, hy / hx, false, lane);          // (hy/hx) K C Mref
    U::xRT(B4, B1, M, M, hx / hy, true, lane);          // + (hx/hy) Mref C K
    // B (psi_prev - psi) -> B4
#pragma unroll
    for (int comp = 0; comp < (G ? 2 : 1); ++comp) {
      if (lane < M) {
        for (int i = 0; i < M; ++i) {
          double g = 0.0;
          if (i < N && lane < N) {
            const long long gi = comp * A.ncomp + base + (long long)i * A.ld + lane;
            const double d = __ldg(A.psi_prev + gi) - __ldg(A.in0 + gi);
            double wi, wl;
            if (!G) { wi = hx * kInvOdd[i]; wl = hy * kInvOdd[lane]; }
            else if (comp == 0) { wi = 2.0 * kInvOdd[i]; wl = hy * kInvOdd[lane]; }
            else { wi = hx * kInvOdd[i]; wl = 2.0 * kInvOdd[lane]; }
            g = (wi * d) * wl;
          }
          B0[i * LD + lane] = g;
        }
      }
      __syncwarp();
      if (G && comp == 1) U::yDT(B0, B3, M, M, 1.0, false, lane);   // G D
      else U::yRT(B0, B3, M, M, 1.0, false, lane);                   // G R
      __syncwarp();
      if (G && comp == 0) U::xDT(B3, B4, M, M, 1.0, false, lane);   // D^T (.)
      else U::xRT(B3, B4, M, M, 1.0, comp > 0, lane);                // R^T (.)
      __syncwarp();
    }
    // r = -alpha A u + B dpsi (lane = column k)
    if (lane < M) {
      const int k = lane;
      double* edge = A.edge + (long long)e * (4 * M - 4);
      for (int j = 0; j < M; ++j) {
        const double r = -A.alpha * B1[j * LD + k] + B4[j * LD + k];
        if (j >= 2 && k >= 2) {
          const long long ix = (A.ncx - 1) + (long long)cx * (P - 1) + (j - 2);
          const long long iy = (A.ncy - 1) + (long long)cy * (P - 1) + (k - 2);
          const long long g = ix * A.niy + iy;
          A.b_u[g] = A.alpha * __ldg(A.f_load + g) + r;
        } else if (j < 2) {
          edge[j * M + k] = r;
        } else {
          edge[2 * M + (j - 2) * 2 + k] = r;
        }
      }
    }
    __syncwarp();
  }
}

template <int P, bool G>
int go(const ElemArgs& A, cudaStream_t s) {
  using U = UPass<P>;
  constexpr size_t smem = sizeof(double) * (size_t)UPW * upass_bufs<G>() * U::M * U::LD;
  struct Memo { int grid_cap = 0; };
  static PerDevice<Memo> memo;
  int grid_cap = 0;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (m.grid_cap == 0) {
      cudaError_t e = cudaFuncSetAttribute(k_upass<P, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      int dev = 0, nsm = 0, occ = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_upass<P, G>, 32 * UPW, smem);
      m.grid_cap = nsm * (occ > 0 ? occ : 1);
    }
    grid_cap = m.grid_cap;
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_upass)", se);
  int need = (A.N + UPW - 1) / UPW;
  cudaError_t e = launch_pdl(k_upass<P, G>, dim3(need < grid_cap ? need : grid_cap), dim3(32 * UPW), smem, s, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_upass launch", e);
}

template <int P>
int dispatch(int p, bool g, const ElemArgs& A, cudaStream_t s) {
  if constexpr (P > UPASS_PMAX) {
    return set_error_msg(HPG_ERR_UNSUPPORTED, "no k_upass instantiation");
  } else {
    if (p == P) return g ? go<P, true>(A, s) : go<P, false>(A, s);
    return dispatch<P + 1>(p, g, A, s);
  }
}

}  // namespace

bool upass_available(int p) { return p >= UPASS_PMIN && p <= UPASS_PMAX; }

int run_upass(int p, bool g, const ElemArgs& A, cudaStream_t s) {
  return dispatch<UPASS_PMIN>(p, g, A, s);
}

}  // namespace hpg
