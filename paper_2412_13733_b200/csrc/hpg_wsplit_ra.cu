// Instantiations and launcher of the fused residual + Jacobian-apply
// row-split kernel (k_wsplit_ra, hpg_wsplit.cuh).
#include "../../include/hpg_b200.h"
#include "hpg_launch.cuh"
#include "hpg_wsplit.cuh"

namespace hpg {
namespace {

template <int NT, int QT, int MR, int MC>
int launch_ra(const ElemArgs& A, cudaStream_t s) {
  using CF = WsplitRaCfg<NT, QT, MR, MC>;
  const size_t smem = sizeof(double) * (size_t)CF::SMEM_DBL;
  if (smem > 227 * 1024) return set_error_msg(HPG_ERR_UNSUPPORTED, "fused row-split kernel shared memory too large");
  struct Memo { size_t attr = 0; };
  static PerDevice<Memo> memo;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (smem > m.attr) {
      cudaError_t e = cudaFuncSetAttribute(k_wsplit_ra<NT, QT, MR, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      m.attr = smem;
    }
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_wsplit_ra)", se);
  cudaError_t e = launch_pdl(k_wsplit_ra<NT, QT, MR, MC>, dim3(A.N), dim3(64 * QT), smem, s, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_wsplit_ra launch", e);
}

#define HPG_RA_LIST(X) X(true, 3, 5) X(true, 3, 7) X(false, 1, 2) X(false, 1, 3)

}  // namespace

bool wsplit_ra_available(bool gradient, int NT, int QT) {
#define HPG_RA_AV(G, NT_, QT_) if (gradient == G && NT == NT_ && QT == QT_) return true;
  HPG_RA_LIST(HPG_RA_AV)
#undef HPG_RA_AV
  return false;
}

int run_wsplit_ra(bool gradient, const ElemArgs& A, cudaStream_t s) {
#define HPG_RA_GO(G, NT_, QT_)                                                                   \
  if (gradient == G && A.NT == NT_ && A.QT == QT_)                                               \
    return G ? launch_ra<NT_, QT_, M_GRAD_RES, M_GRAD_CACHED>(A, s)                              \
             : launch_ra<NT_, QT_, M_OBST_RES, M_OBST_CACHED>(A, s);
  HPG_RA_LIST(HPG_RA_GO)
#undef HPG_RA_GO
  return set_error_msg(HPG_ERR_UNSUPPORTED, "no fused row-split instantiation");
}

}  // namespace hpg
