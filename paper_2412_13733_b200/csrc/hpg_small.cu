// Instantiations of the thread-per-element low-degree kernel (hpg_small.cuh).
#include "hpg_launch.cuh"
#include "hpg_small.cuh"

namespace hpg {
namespace {

template <int N, int Q, bool RES, bool APPLY>
int go(const ElemArgs& A, const SmallTables& tb, cudaStream_t s) {
  constexpr int TH = small_threads<N, APPLY>();
  const int grid = (A.N + TH - 1) / TH;
  cudaError_t e = launch_pdl(k_small<N, Q, RES, APPLY>, dim3(grid), dim3(TH), 0, s, A, tb);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_small launch", e);
}

int dispatch(int n, int q, bool res, bool apply, bool launch, const ElemArgs& A, const SmallTables& tb,
             cudaStream_t s) {
  if (n == 1 && q == 3) { if (!launch) return 1; return res && apply ? go<1, 3, true, true>(A, tb, s) : res ? go<1, 3, true, false>(A, tb, s) : go<1, 3, false, true>(A, tb, s); }
  if (n == 1 && q == 4) { if (!launch) return 1; return res && apply ? go<1, 4, true, true>(A, tb, s) : res ? go<1, 4, true, false>(A, tb, s) : go<1, 4, false, true>(A, tb, s); }
  if (n == 1 && q == 5) { if (!launch) return 1; return res && apply ? go<1, 5, true, true>(A, tb, s) : res ? go<1, 5, true, false>(A, tb, s) : go<1, 5, false, true>(A, tb, s); }
  if (n == 1 && q == 6) { if (!launch) return 1; return res && apply ? go<1, 6, true, true>(A, tb, s) : res ? go<1, 6, true, false>(A, tb, s) : go<1, 6, false, true>(A, tb, s); }
  if (n == 1 && q == 7) { if (!launch) return 1; return res && apply ? go<1, 7, true, true>(A, tb, s) : res ? go<1, 7, true, false>(A, tb, s) : go<1, 7, false, true>(A, tb, s); }
  if (n == 2 && q == 4) { if (!launch) return 1; return res && apply ? go<2, 4, true, true>(A, tb, s) : res ? go<2, 4, true, false>(A, tb, s) : go<2, 4, false, true>(A, tb, s); }
  if (n == 2 && q == 5) { if (!launch) return 1; return res && apply ? go<2, 5, true, true>(A, tb, s) : res ? go<2, 5, true, false>(A, tb, s) : go<2, 5, false, true>(A, tb, s); }
  if (n == 2 && q == 6) { if (!launch) return 1; return res && apply ? go<2, 6, true, true>(A, tb, s) : res ? go<2, 6, true, false>(A, tb, s) : go<2, 6, false, true>(A, tb, s); }
  if (n == 2 && q == 7) { if (!launch) return 1; return res && apply ? go<2, 7, true, true>(A, tb, s) : res ? go<2, 7, true, false>(A, tb, s) : go<2, 7, false, true>(A, tb, s); }
  if (n == 2 && q == 8) { if (!launch) return 1; return res && apply ? go<2, 8, true, true>(A, tb, s) : res ? go<2, 8, true, false>(A, tb, s) : go<2, 8, false, true>(A, tb, s); }
  if (n == 3 && q == 5) { if (!launch) return 1; return res && apply ? go<3, 5, true, true>(A, tb, s) : res ? go<3, 5, true, false>(A, tb, s) : go<3, 5, false, true>(A, tb, s); }
  if (n == 3 && q == 6) { if (!launch) return 1; return res && apply ? go<3, 6, true, true>(A, tb, s) : res ? go<3, 6, true, false>(A, tb, s) : go<3, 6, false, true>(A, tb, s); }
  if (n == 3 && q == 7) { if (!launch) return 1; return res && apply ? go<3, 7, true, true>(A, tb, s) : res ? go<3, 7, true, false>(A, tb, s) : go<3, 7, false, true>(A, tb, s); }
  if (n == 3 && q == 8) { if (!launch) return 1; return res && apply ? go<3, 8, true, true>(A, tb, s) : res ? go<3, 8, true, false>(A, tb, s) : go<3, 8, false, true>(A, tb, s); }
  if (n == 3 && q == 9) { if (!launch) return 1; return res && apply ? go<3, 9, true, true>(A, tb, s) : res ? go<3, 9, true, false>(A, tb, s) : go<3, 9, false, true>(A, tb, s); }
  if (n == 3 && q == 10) { if (!launch) return 1; return res && apply ? go<3, 10, true, true>(A, tb, s) : res ? go<3, 10, true, false>(A, tb, s) : go<3, 10, false, true>(A, tb, s); }
  if (n == 4 && q == 6) { if (!launch) return 1; return res && apply ? go<4, 6, true, true>(A, tb, s) : res ? go<4, 6, true, false>(A, tb, s) : go<4, 6, false, true>(A, tb, s); }
  if (n == 4 && q == 7) { if (!launch) return 1; return res && apply ? go<4, 7, true, true>(A, tb, s) : res ? go<4, 7, true, false>(A, tb, s) : go<4, 7, false, true>(A, tb, s); }
  if (n == 4 && q == 8) { if (!launch) return 1; return res && apply ? go<4, 8, true, true>(A, tb, s) : res ? go<4, 8, true, false>(A, tb, s) : go<4, 8, false, true>(A, tb, s); }
  if (n == 4 && q == 9) { if (!launch) return 1; return res && apply ? go<4, 9, true, true>(A, tb, s) : res ? go<4, 9, true, false>(A, tb, s) : go<4, 9, false, true>(A, tb, s); }
  if (n == 4 && q == 10) { if (!launch) return 1; return res && apply ? go<4, 10, true, true>(A, tb, s) : res ? go<4, 10, true, false>(A, tb, s) : go<4, 10, false, true>(A, tb, s); }
  if (n == 4 && q == 12) { if (!launch) return 1; return res && apply ? go<4, 12, true, true>(A, tb, s) : res ? go<4, 12, true, false>(A, tb, s) : go<4, 12, false, true>(A, tb, s); }
  if (n == 5 && q == 7) { if (!launch) return 1; return res && apply ? go<5, 7, true, true>(A, tb, s) : res ? go<5, 7, true, false>(A, tb, s) : go<5, 7, false, true>(A, tb, s); }
  if (n == 5 && q == 8) { if (!launch) return 1; return res && apply ? go<5, 8, true, true>(A, tb, s) : res ? go<5, 8, true, false>(A, tb, s) : go<5, 8, false, true>(A, tb, s); }
  if (n == 5 && q == 9) { if (!launch) return 1; return res && apply ? go<5, 9, true, true>(A, tb, s) : res ? go<5, 9, true, false>(A, tb, s) : go<5, 9, false, true>(A, tb, s); }
  if (n == 5 && q == 10) { if (!launch) return 1; return res && apply ? go<5, 10, true, true>(A, tb, s) : res ? go<5, 10, true, false>(A, tb, s) : go<5, 10, false, true>(A, tb, s); }
  if (n == 5 && q == 11) { if (!launch) return 1; return res && apply ? go<5, 11, true, true>(A, tb, s) : res ? go<5, 11, true, false>(A, tb, s) : go<5, 11, false, true>(A, tb, s); }
  if (n == 5 && q == 14) { if (!launch) return 1; return res && apply ? go<5, 14, true, true>(A, tb, s) : res ? go<5, 14, true, false>(A, tb, s) : go<5, 14, false, true>(A, tb, s); }
  return launch ? set_error_msg(HPG_ERR_UNSUPPORTED, "no k_small instantiation") : 0;
}

}  // namespace

bool small_available(int n, int q) {
  ElemArgs A{};
  SmallTables tb{};
  return dispatch(n, q, true, false, false, A, tb, 0) == 1;
}

int run_small(int n, int q, bool res, bool apply, const ElemArgs& A, const SmallTables& tb, cudaStream_t s) {
  return dispatch(n, q, res, apply, true, A, tb, s);
}

}  // namespace hpg
