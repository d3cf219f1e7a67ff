// Launchers of the element kernels, one translation unit per mode
// (hpg_mode_*.cu) so the template instantiations compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <mutex>

#include <nvtx3/nvToolsExt.h>
#include "hpg_common.cuh"
#include "../../include/hpg_b200.h"

namespace hpg {

int set_error(int code, const char* where, cudaError_t e);
int set_error_msg(int code, const char* msg);

// NVTX range around every C-ABI entry point (named after it), so nsys /
// ncu --nvtx timelines attribute kernels to the reference callable they serve.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define HPG_NVTX(name) ::hpg::NvtxRange hpg_nvtx_range_(name)

// Launch-setup memo per device (function attributes and occupancy are per
// device) behind a mutex, so plans on several devices / host threads share
// the library safely.  T needs a default constructor marking "not set up".
constexpr int kMaxDevices = 64;
template <class T>
struct PerDevice {
  std::mutex mu;
  T slot[kMaxDevices];
  // run fn(T&) under the lock on the current device's slot
  template <class F>
  auto with(F&& fn) -> decltype(fn(slot[0])) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    return fn(slot[dev % kMaxDevices]);
  }
};

// Element-kernel paths: CTA per (element, row-tile split) (k_cta, any size),
// warp per element (k_warp), CTA per element with a warp per row tile
// (k_wsplit, few mid-size elements).
enum ElemPath : int { PATH_CTA = 0, PATH_WARP = 1, PATH_WSPLIT = 2 };
// Is there a warp-per-element / row-split instantiation for (NT, QT) in this mode?
template <int MODE> bool warp_available(int NT, int QT);
template <int MODE> bool wsplit_available(int NT, int QT);
// Launch the element kernel of MODE on `path` (the CTA path runs A.splits
// row-tile splits + a deterministic reduction).
template <int MODE> int run_mode(int path, ElemArgs A, cudaStream_t s);

// Thread-per-element low-degree obstacle kernel (hpg_small.cuh).
struct SmallTables;
bool small_available(int n, int q);
int run_small(int n, int q, bool res, bool apply, const ElemArgs& A, const SmallTables& tb, cudaStream_t s);

// Thread-per-cell generated U side for low degrees (hpg_usmall.cu).
bool usmall_available(int p, bool gradient);
int run_usmall(int p, bool gradient, const ElemArgs& A, cudaStream_t s);

// Single-pass residual (+ apply) for low-degree obstacle meshes (hpg_lowp.cu).
bool lowp_available(int p, int q);
int run_lowp(int p, int q, bool apply, const ElemArgs& A, const SmallTables& tb, cudaStream_t s);

// Warp-per-cell generated-pass U side for mid degrees (hpg_upass.cu).
bool upass_available(int p);
int run_upass(int p, bool gradient, const ElemArgs& A, cudaStream_t s);

}  // namespace hpg
