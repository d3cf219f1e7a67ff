// Thread-per-cell U side of the residual for low degrees (p <= USMALL_PMAX):
// the cell's local U tile and psi_prev - psi tile are staged in thread-private
// shared-memory slices and the exact couplings run as generated straight-line
// FMA code with literal coefficients (hpg_usmall_gen.cuh, tools/gen_usmall.py).
// Outputs: b_psi <- phi_moments - B^T u (obstacle) | -B^T u (gradient), the
// owned (bubble x bubble) b_u dofs, and the hat-involved edge contributions.
#include "hpg_launch.cuh"
#include "hpg_common.cuh"
#include "hpg_usmall_gen.cuh"

namespace hpg {
namespace {

constexpr int USM_TH = 64;

template <int P, bool G>
__global__ void __launch_bounds__(USM_TH) k_usmall(ElemArgs A) {
  pdl_wait();
  constexpr int M = P + 1, N = G ? P : P - 1, NC = G ? 2 : 1;
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int e = blockIdx.x * USM_TH + tid;
  if (e >= A.N) return;
  double* sC = smem + tid;                       // [M*M][USM_TH]
  double* sG = smem + M * M * USM_TH + tid;      // [NC*N*N][USM_TH]
  const int cx = e / A.ncy, cy = e - cx * A.ncy;
  const double hx = A.hx[cx], hy = A.hy[cy];
  const long long base = psi_index(A, cx, cy, 0, 0);
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int ix = u_local_1d(cx, i, A.ncx, P);
#pragma unroll
    for (int l = 0; l < M; ++l) {
      const int iy = u_local_1d(cy, l, A.ncy, P);
      sC[(i * M + l) * USM_TH] = (ix < 0 || iy < 0) ? 0.0 : __ldg(A.u + (long long)ix * A.niy + iy);
    }
  }
#pragma unroll
  for (int comp = 0; comp < NC; ++comp)
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const long long g = comp * A.ncomp + base + (long long)i * A.ld + l;
        sG[((comp * N + i) * N + l) * USM_TH] = __ldg(A.psi_prev + g) - __ldg(A.in0 + g);
      }
  double* edge = A.edge + (long long)e * (4 * M - 4);
  const long long bx = (A.ncx - 1) + (long long)cx * (P - 1) - 2;
  const long long by = (A.ncy - 1) + (long long)cy * (P - 1) - 2;
  auto ou = [&](int j, int k, double r) {
    if (j >= 2 && k >= 2) {
      const long long g = (bx + j) * A.niy + (by + k);
      A.b_u[g] = A.alpha * __ldg(A.f_load + g) + r;
    } else if (j < 2) {
      edge[j * M + k] = r;
    } else {
      edge[2 * M + (j - 2) * 2 + k] = r;
    }
  };
  auto ob = [&](int comp, int a, int b, double btu) {
    const long long g = comp * A.ncomp + base + (long long)a * A.ld + b;
    if (G) A.out[g] = -btu;
    else A.out[g] = __ldg(A.phi_mom + g) - btu;
  };
  USmall<P, G>::run(sC, sG, USM_TH, hx, hy, A.alpha, ou, ob);
}

template <int P, bool G>
int go(const ElemArgs& A, cudaStream_t s) {
  constexpr int M = P + 1, N = G ? P : P - 1, NC = G ? 2 : 1;
  constexpr size_t smem = sizeof(double) * (size_t)(M * M + NC * N * N) * USM_TH;
  struct Memo { bool init = false; };
  static PerDevice<Memo> memo;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (m.init) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_usmall<P, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    m.init = e == cudaSuccess;
    return e;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_usmall)", se);
  cudaError_t e = launch_pdl(k_usmall<P, G>, dim3((A.N + USM_TH - 1) / USM_TH), dim3(USM_TH), smem, s, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_usmall launch", e);
}

}  // namespace

bool usmall_available(int p, bool gradient) {
  return p <= USMALL_PMAX && (gradient ? p >= 1 : p >= 2);
}

int run_usmall(int p, bool g, const ElemArgs& A, cudaStream_t s) {
  switch (p) {
    case 1: return g ? go<1, true>(A, s) : set_error_msg(HPG_ERR_UNSUPPORTED, "obstacle needs p >= 2");
    case 2: return g ? go<2, true>(A, s) : go<2, false>(A, s);
    case 3: return g ? go<3, true>(A, s) : go<3, false>(A, s);
    case 4: return g ? go<4, true>(A, s) : go<4, false>(A, s);
    case 5: return g ? go<5, true>(A, s) : go<5, false>(A, s);
    case 6: return g ? go<6, true>(A, s) : go<6, false>(A, s);
    case 7: return g ? go<7, true>(A, s) : go<7, false>(A, s);
    case 8: return g ? go<8, true>(A, s) : go<8, false>(A, s);
    default: return set_error_msg(HPG_ERR_UNSUPPORTED, "no k_usmall instantiation");
  }
}

}  // namespace hpg
