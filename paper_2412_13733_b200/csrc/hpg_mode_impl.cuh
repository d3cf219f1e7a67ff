// Instantiation body shared by the hpg_mode_*.cu translation units.
// Define HPG_MODE and the warp (NT, QT) list (HPG_WARP_LIST) before including.
#pragma once
#include <cstdio>
#include <cstdlib>
#include "hpg_elem.cuh"
#include "hpg_launch.cuh"
#include "hpg_wsplit.cuh"
#include "hpg_big.cuh"
#include "hpg_stream.cuh"

#ifndef HPG_WSPLIT_LIST
#define HPG_WSPLIT_LIST
#endif

namespace hpg {
namespace {

// many small cells, cached weights (config 1): the persistent streaming
// kernel (hpg_stream.cuh), one CTA per SM
template <int NT, int QT, int MODE>
int launch_stream_t(const ElemArgs& A, int nsm, cudaStream_t s) {
  using CF = StreamCfg<NT, QT, MODE>;
  const size_t smem = sizeof(double) * (size_t)CF::SMEM_DBL;
  struct Memo { size_t attr = 0; };
  static PerDevice<Memo> memo;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (smem > m.attr) {
      cudaError_t e = cudaFuncSetAttribute(k_stream<NT, QT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      m.attr = smem;
    }
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_stream)", se);
  cudaError_t e = launch_pdl(k_stream<NT, QT, MODE>, dim3(nsm), dim3(32 * CF::W), smem, s, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_stream launch", e);
}

inline int device_sm_count() {
  struct Memo { int nsm = 0; };
  static PerDevice<Memo> memo;
  return memo.with([&](Memo& m) {
    if (m.nsm == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&m.nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    return m.nsm;
  });
}

template <int NT, int QT, int MODE>
int launch_warp_t(const ElemArgs& A, cudaStream_t s) {
  using TR = ModeTraits<MODE>;
  if constexpr (MODE == M_OBST_CACHED && NT == 2 && QT <= 3) {
    // every scheduler group of the persistent grid gets at least 2 MW cells
    // (a cell then spans at most two warps' row-tile runs)
    const bool stream_ok = getenv("HPG_NO_STREAM") == nullptr;
    const int nsm = device_sm_count();
    // (its in-cell offsets are 32-bit)
    if (stream_ok && (A.N - A.e0) / nsm / 4 >= 2 * StreamCfg<NT, QT, MODE>::MW && 8 * NT * A.ld < (1LL << 31))
      return launch_stream_t<NT, QT, MODE>(A, nsm, s);
  }
  constexpr int NP = 8 * NT, QP = 8 * QT;
  constexpr int NSTAGE = WarpCfg<NT, QT, MODE>::REGX ? 0 : TR::NIN;
  using CF = WarpCfg<NT, QT, MODE>;
  constexpr int W = CF::W;
  constexpr int WDBL = CF::WSMEM ? CF::WDBL * (CF::PIPE ? 2 : 1) : 0;
  const size_t smem = sizeof(double) * (2 * QP * NP + W * (NSTAGE * NP * (NP + 2) + WDBL) + NP +
                                        (size_t)W * A.usmem);
  if (smem > 227 * 1024) return set_error_msg(HPG_ERR_UNSUPPORTED, "warp path shared memory too large");
  struct Memo { size_t attr = 0; int occ = -1, nsm = 0, occ_smem = -1; };
  static PerDevice<Memo> memo;
  int grid_cap = 0;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (smem > m.attr) {
      cudaError_t e = cudaFuncSetAttribute(k_warp<NT, QT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      m.attr = smem;
    }
    // persistent-style grid: every resident warp slot gets an equal share of cells
    if (m.occ < 0 || m.occ_smem != (int)smem) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&m.nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m.occ, k_warp<NT, QT, MODE>, 32 * W, smem);
      if (m.occ < 1) m.occ = 1;
      m.occ_smem = (int)smem;
    }
    grid_cap = m.nsm * m.occ;
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_warp)", se);
  int need = (A.N - A.e0 + W * CF::CPW - 1) / (W * CF::CPW);
  int grid = need < grid_cap ? need : grid_cap;
  // programmatic dependent launch: the table prologue overlaps the previous
  // kernel's tail (k_warp orders its data reads with griddepcontrol.wait)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * W);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  static const bool pdl = getenv("HPG_NO_PDL") == nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_warp<NT, QT, MODE>, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_warp launch", e);
}

template <int NT, int QT, int MODE>
int launch_wsplit_t(const ElemArgs& A, cudaStream_t s) {
  using CF = WsplitCfg<NT, QT, MODE>;
  const size_t smem = sizeof(double) * (size_t)CF::SMEM_DBL;
  if (smem > 227 * 1024) return set_error_msg(HPG_ERR_UNSUPPORTED, "row-split kernel shared memory too large");
  struct Memo { size_t attr = 0; };
  static PerDevice<Memo> memo;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (smem > m.attr) {
      cudaError_t e = cudaFuncSetAttribute(k_wsplit<NT, QT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      m.attr = smem;
    }
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_wsplit)", se);
  cudaError_t e = launch_pdl(k_wsplit<NT, QT, MODE>, dim3(A.N), dim3(32 * QT), smem, s, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_wsplit launch", e);
}

template <int MODE, int MAXS, int W>
int launch_cta_t(ElemArgs A, cudaStream_t s) {
  using TR = ModeTraits<MODE>;
  const int NP = 8 * A.NT;
  size_t smem = sizeof(double) * ((size_t)TR::NIN * NP * (NP + 2) +
                                  (size_t)(TR::NSYN * A.NT + TR::NOUT * A.QT + TR::NOUT * A.NT) * 64);
  // stage the tables too when the CTA still fits twice per SM
  const size_t tsmem = sizeof(double) * (size_t)2 * (8 * A.QT) * NP;
  // (one CTA per SM when splitting few cells: then PK(T) alone still fits)
  A.smem_tables = 0;
  if (getenv("HPG_NO_SMEM_TABLES") == nullptr) {
    if (smem + tsmem <= 100 * 1024) {
      A.smem_tables = 3;
      smem += tsmem;
    } else if (A.splits > 1 && smem + tsmem / 2 <= 200 * 1024) {
      A.smem_tables = 2;
      smem += tsmem / 2;
    }
  }
  if (smem > 227 * 1024) return set_error_msg(HPG_ERR_UNSUPPORTED, "element tile too large for shared memory");
  // row-tile splits of a cell as one thread-block cluster (<= 8, portable):
  // partials reduced through DSMEM inside the kernel, when the clusters fit
  // in one wave (checked once per shape and device)
  struct Memo { int attr = 0; int ok_splits = -1, ok_n = -1, ok_np = -1, ok_res = 0; };
  static PerDevice<Memo> memo;
  A.cluster_red = 0;
  const bool try_cluster = A.splits > 1 && A.splits <= 8 && getenv("HPG_NO_CLUSTER") == nullptr;
  const size_t ysmem = sizeof(double) * (size_t)TR::NOUT * NP * NP;
  const size_t csmem = smem > ysmem ? smem : ysmem;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if ((int)smem > m.attr) {
      cudaError_t e = cudaFuncSetAttribute(k_cta<MODE, MAXS, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      m.attr = (int)smem;
    }
    if (!try_cluster) return cudaSuccess;
    if (m.ok_splits != A.splits || m.ok_n != A.N || m.ok_np != NP) {
      m.ok_splits = A.splits; m.ok_n = A.N; m.ok_np = NP; m.ok_res = 0;
      // (never LOWER the attribute: it must cover the largest smem launched so far)
      if (csmem <= 227 * 1024 &&
          ((int)csmem <= m.attr ||
           cudaFuncSetAttribute(k_cta<MODE, MAXS, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem) ==
               cudaSuccess)) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(A.N * A.splits);
        q.blockDim = dim3(32 * W);
        q.dynamicSmemBytes = csmem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = A.splits; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        q.numAttrs = 1;
        int nclusters = 0;
        cudaError_t qe = cudaOccupancyMaxActiveClusters(&nclusters, k_cta<MODE, MAXS, W>, &q);
        if (qe == cudaSuccess && nclusters >= A.N) m.ok_res = 1;
        if (getenv("HPG_DEBUG"))
          fprintf(stderr, "[hpg] k_cta mode %d: %d cells x %d splits, smem %zu: max active clusters %d (%s) -> %s\n",
                  MODE, A.N, A.splits, csmem, nclusters, cudaGetErrorString(qe), m.ok_res ? "cluster" : "reduce kernel");
        cudaGetLastError();
        if ((int)csmem > m.attr) m.attr = (int)csmem;
      }
    }
    A.cluster_red = m.ok_res;
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_cta)", se);
  if (A.cluster_red) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(A.N * A.splits);
    q.blockDim = dim3(32 * W);
    q.dynamicSmemBytes = csmem;
    q.stream = s;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = A.splits; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&q, k_cta<MODE, MAXS, W>, A);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_cta cluster launch", e);
  }
  cudaError_t e = launch_pdl(k_cta<MODE, MAXS, W>, dim3(A.N * A.splits), dim3(32 * W), smem, s, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "k_cta launch", e);
  if (A.splits > 1) {
    long long total = (long long)A.N * TR::NOUT * A.n * A.n;
    e = launch_pdl(k_cta_reduce<MODE>, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, A);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "k_cta_reduce launch", e);
  }
  return 0;
}

// config 3 (Gauss): the on-chip large-tile kernel (hpg_big.cuh), same split
// reduction as k_cta
template <int MODE, int NT, int QT, int RB, int W>
int launch_big_t(ElemArgs A, cudaStream_t s) {
  using CF = BigCfg<MODE, NT, QT, RB, W>;
  const size_t smem = sizeof(double) * (size_t)CF::SMEM_DBL;
  struct Memo { size_t attr = 0; int ok_n = -1, ok_res = 0; };
  static PerDevice<Memo> memo;
  A.cluster_red = 0;
  const bool try_cluster = A.splits > 1 && A.splits <= 8 && getenv("HPG_NO_CLUSTER") == nullptr;
  cudaError_t se = memo.with([&](Memo& m) -> cudaError_t {
    if (smem > m.attr) {
      cudaError_t e = cudaFuncSetAttribute(k_big<MODE, NT, QT, RB, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      m.attr = smem;
    }
    if (try_cluster && m.ok_n != A.N) {
      m.ok_n = A.N;
      m.ok_res = 0;
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(A.N * A.splits);
      q.blockDim = dim3(32 * W);
      q.dynamicSmemBytes = smem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = A.splits; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int nclusters = 0;
      cudaError_t qe = cudaOccupancyMaxActiveClusters(&nclusters, k_big<MODE, NT, QT, RB, W>, &q);
      if (qe == cudaSuccess && nclusters >= A.N) m.ok_res = 1;
      if (getenv("HPG_DEBUG"))
        fprintf(stderr, "[hpg] k_big mode %d: %d cells x %d splits, smem %zu: max active clusters %d (%s) -> %s\n",
                MODE, A.N, A.splits, smem, nclusters, cudaGetErrorString(qe), m.ok_res ? "cluster" : "reduce kernel");
      cudaGetLastError();
    }
    A.cluster_red = try_cluster ? m.ok_res : 0;
    return cudaSuccess;
  });
  if (se != cudaSuccess) return set_error(HPG_ERR_CUDA, "cudaFuncSetAttribute(k_big)", se);
  cudaError_t e;
  if (A.cluster_red) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(A.N * A.splits);
    q.blockDim = dim3(32 * W);
    q.dynamicSmemBytes = smem;
    q.stream = s;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = A.splits; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    e = cudaLaunchKernelEx(&q, k_big<MODE, NT, QT, RB, W>, A);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_big cluster launch", e);
  }
  e = launch_pdl(k_big<MODE, NT, QT, RB, W>, dim3(A.N * A.splits), dim3(32 * W), smem, s, A);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "k_big launch", e);
  if (A.splits > 1) {
    const long long total = (long long)A.N * ModeTraits<MODE>::NOUT * A.n * A.n;
    e = launch_pdl(k_cta_reduce<MODE>, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, A);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(HPG_ERR_CUDA, "k_cta_reduce launch", e);
  }
  return 0;
}

// few elements split across CTAs (config 3): 16 warps per CTA for latency
// hiding; many elements (config 2): 8 warps per CTA, more CTAs per SM
template <int MODE, int W>
int launch_cta_w(ElemArgs A, cudaStream_t s) {
  using TR = ModeTraits<MODE>;
  int slots = (TR::NOUT * A.NT * A.NT + W - 1) / W;
  if (slots <= 4) return launch_cta_t<MODE, 4, W>(A, s);
  if (slots <= 16) return launch_cta_t<MODE, 16, W>(A, s);
  if (slots <= 32) return launch_cta_t<MODE, 32, W>(A, s);
  return set_error_msg(HPG_ERR_UNSUPPORTED, "tile side too large");
}

template <int MODE>
int launch_cta(ElemArgs A, cudaStream_t s) {
  if constexpr (MODE == M_OBST_RES || MODE == M_OBST_APPLY || MODE == M_OBST_CACHED) {
    if (A.NT == 11 && A.QT == 16 && A.splits == 8 && getenv("HPG_NO_BIG") == nullptr)
      return launch_big_t<MODE, 11, 16, 2, 16>(A, s);
  }
  if (A.splits > 1) return launch_cta_w<MODE, 16>(A, s);
  return launch_cta_w<MODE, 8>(A, s);
}

}  // namespace

#define HPG_W(NT_, QT_) \
  if (NT == NT_ && QT == QT_) return launch ? launch_warp_t<NT_, QT_, HPG_MODE>(A, s) : 1;

static int warp_dispatch(int NT, int QT, bool launch, const ElemArgs& A, cudaStream_t s) {
  HPG_WARP_LIST
  return launch ? set_error_msg(HPG_ERR_UNSUPPORTED, "no warp instantiation") : 0;
}

#define HPG_WS(NT_, QT_) \
  if (NT == NT_ && QT == QT_) return launch ? launch_wsplit_t<NT_, QT_, HPG_MODE>(A, s) : 1;

static int wsplit_dispatch(int NT, int QT, bool launch, const ElemArgs& A, cudaStream_t s) {
  HPG_WSPLIT_LIST
  return launch ? set_error_msg(HPG_ERR_UNSUPPORTED, "no row-split instantiation") : 0;
}

template <> bool warp_available<HPG_MODE>(int NT, int QT) {
  ElemArgs dummy{};
  return warp_dispatch(NT, QT, false, dummy, 0) == 1;
}

template <> bool wsplit_available<HPG_MODE>(int NT, int QT) {
  ElemArgs dummy{};
  return wsplit_dispatch(NT, QT, false, dummy, 0) == 1;
}

template <> int run_mode<HPG_MODE>(int path, ElemArgs A, cudaStream_t s) {
  if (path == PATH_WARP) return warp_dispatch(A.NT, A.QT, true, A, s);
  if (path == PATH_WSPLIT) return wsplit_dispatch(A.NT, A.QT, true, A, s);
  return launch_cta<HPG_MODE>(A, s);
}

}  // namespace hpg
