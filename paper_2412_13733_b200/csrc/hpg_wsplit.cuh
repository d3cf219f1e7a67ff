// Row-split warp kernels: one CTA per element, one warp per 8-row tile of the
// Q x Q point grid, for element counts too small to fill the GPU with one warp
// per element (config 2: 256 cells, config 0: 16).
//
// Each warp runs the k_warp pipeline (hpg_elem.cuh) on ITS row tile rt with
// compile-time tile counts -- P = S[rt] C, V = P S^T, pointwise map,
// R = T W^T, Y_rt = R T[:, rt]^T -- fragments in registers, tables and the
// element's coefficient tiles in shared memory (staged once per CTA).  The
// row tiles' partials Y_rt are summed in shared memory in fixed (ascending)
// order -- deterministic; the single-warp kernel's sum regrouped, so the two
// paths agree to rounding -- and finished by write_moment (reference
// CellKernel2D.moments, assembly.py:249-251; residual modes finish b_psi in
// place, proximal.py:123,125).
//
// k_wsplit<NT,QT,MODE>: one mode, QT warps (ws_rowtile is the per-warp body).
#pragma once
#include "hpg_elem.cuh"

namespace hpg {

template <int NT, int QT, int MODE>
struct WsplitCfg {
  using TR = ModeTraits<MODE>;
  static constexpr int NP = 8 * NT, QP = 8 * QT, LDT = NP + 2, TILE = NP * LDT;
  static constexpr bool cached = MODE == M_OBST_CACHED || MODE == M_GRAD_CACHED;
  static constexpr int TAB = 2 * QP * NP;
  static constexpr int INV = (NP + 1) / 2 * 2;
  static constexpr int WROW = QT * TR::NW * 64;          // one row tile's weights
  static constexpr int TILES = TR::NIN * TILE;
  static constexpr int WTS = cached ? QT * WROW : 0;
  static constexpr bool PHI = MODE == M_GRAD_RES || MODE == M_GRAD_APPLY;
  static constexpr int PHIS = PHI ? QP * QP : 0;            // staged phi samples
  static constexpr int YPART = QT * TR::NOUT * NP * NP;
  static constexpr int BODY = (TILES + WTS + PHIS) > YPART ? (TILES + WTS + PHIS) : YPART;
  static constexpr int SMEM_DBL = TAB + INV + BODY;
};

// One warp, one row tile rt of element e: accumulates MODE's Y partial into
// Y.  sTile: this mode's coefficient tiles (fields in field_src order).
// Cached modes read the row tile's point weights from w_in (shared memory,
// [ht][w][lane][2]); residual modes write them to w_out when given (and to
// the global weight cache when A.wc_out is set).  before_map() runs between
// the synthesis and the pointwise map, after_map() right after it.
template <int NT, int QT, int MODE, class BeforeMap, class AfterMap>
__device__ __forceinline__ void ws_rowtile(const ElemArgs& A, int e, int rt, const double* sS, const double* sT,
                                           const double* sTile, const double* w_in, double* w_out,
                                           double (&Y)[ModeTraits<MODE>::NOUT][NT][NT][2], bool& flag,
                                           BeforeMap before_map, AfterMap after_map,
                                           const double* sPhi = nullptr) {
  using TR = ModeTraits<MODE>;
  using CF = WsplitCfg<NT, QT, MODE>;
  constexpr int NP = CF::NP, NK = NP / 4, QK = CF::QP / 4, LDT = CF::LDT, TILE = CF::TILE;
  constexpr int NSYN = TR::NSYN, NOUT = TR::NOUT, NW = TR::NW;
  constexpr bool gradient = MODE >= M_GRAD_RES && MODE <= M_GRAD_CACHED;
  constexpr bool writes = MODE == M_OBST_RES || MODE == M_GRAD_RES;
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
#pragma unroll
  for (int o = 0; o < NOUT; ++o)
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int k = 0; k < NT; ++k) Y[o][i][k][0] = Y[o][i][k][1] = 0.0;
  double V[NSYN > 0 ? NSYN : 1][QT][2];
#pragma unroll
  for (int f = 0; f < NSYN; ++f) {
    double P[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) P[nt][0] = P[nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < NK; ++ks) {
      const double a = sS[(rt * NK + ks) * 32 + lane];
      const double* row = sTile + f * TILE + (8 * (ks >> 1) + 2 * c + (ks & 1)) * LDT + r;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(P[nt], a, row[8 * nt]);
    }
#pragma unroll
    for (int ht = 0; ht < QT; ++ht) {
      // two accumulation chains (even / odd k-steps)
      double V1[2] = {0.0, 0.0};
      V[f][ht][0] = V[f][ht][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < NK; ks += 2) {
        dmma(V[f][ht], P[ks >> 1][0], sS[(ht * NK + ks) * 32 + lane]);
        dmma(V1, P[ks >> 1][1], sS[(ht * NK + ks + 1) * 32 + lane]);
      }
      V[f][ht][0] += V1[0];
      V[f][ht][1] += V1[1];
    }
  }
  before_map();
  double Vw[NOUT][QT][2];
  const int g = 8 * rt + r;
#pragma unroll
  for (int ht = 0; ht < QT; ++ht) {
    double win[NW > 0 ? NW : 1][2], wout[NW > 0 ? NW : 1][2];
    if constexpr (CF::cached) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const double2 t = *reinterpret_cast<const double2*>(w_in + (ht * NW + w) * 64 + 2 * lane);
        win[w][0] = t.x;
        win[w][1] = t.y;
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int h = 8 * ht + 2 * c + j;
      const bool inside = g < A.nq && h < A.nq;
      double v[NSYN > 0 ? NSYN : 1], vw[NOUT], wi[NW > 0 ? NW : 1], wo[NW > 0 ? NW : 1];
#pragma unroll
      for (int f = 0; f < NSYN; ++f) v[f] = V[f][ht][j];
#pragma unroll
      for (int w = 0; w < NW; ++w) wi[w] = CF::cached ? win[w][j] : 0.0;
      double phi = 0.0;
      if constexpr (gradient && !CF::cached) {
        if (inside) phi = sPhi ? sPhi[g * CF::QP + h] : __ldg(A.phi + ((long long)e * A.nq + g) * A.nq + h);
      }
      bool fl = false;
      point_map<MODE>(v, phi, wi, wo, vw, fl);
      // padded points are inert: zero weight, never flagged
      if (inside) {
        flag |= fl;
      } else {
#pragma unroll
        for (int o = 0; o < NOUT; ++o) vw[o] = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) wo[w] = 0.0;
      }
#pragma unroll
      for (int o = 0; o < NOUT; ++o) Vw[o][ht][j] = vw[o];
#pragma unroll
      for (int w = 0; w < NW; ++w) wout[w][j] = wo[w];
    }
    if constexpr (writes) {
      if (w_out != nullptr) {
#pragma unroll
        for (int w = 0; w < NW; ++w)
          *reinterpret_cast<double2*>(w_out + (ht * NW + w) * 64 + 2 * lane) = make_double2(wout[w][0], wout[w][1]);
      }
      if (A.wc_out != nullptr) {
#pragma unroll
        for (int w = 0; w < NW; ++w)
          *reinterpret_cast<double2*>(A.wc_out + wc_index(e, QT, rt, ht, NW, w, lane)) =
              make_double2(wout[w][0], wout[w][1]);
      }
    }
  }
  after_map();
#pragma unroll
  for (int o = 0; o < NOUT; ++o) {
    double R[NT][2];
#pragma unroll
    for (int bt = 0; bt < NT; ++bt) {
      double R1[2] = {0.0, 0.0};
      R[bt][0] = R[bt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < QK; ks += 2) {
        dmma(R[bt], sT[(bt * QK + ks) * 32 + lane], Vw[o][ks >> 1][0]);
        dmma(R1, sT[(bt * QK + ks + 1) * 32 + lane], Vw[o][ks >> 1][1]);
      }
      R[bt][0] += R1[0];
      R[bt][1] += R1[1];
    }
#pragma unroll
    for (int bt = 0; bt < NT; ++bt)
#pragma unroll
      for (int at = 0; at < NT; ++at)
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2)
          dmma(Y[o][bt][at], R[bt][k2], sT[(at * QK + 2 * rt + k2) * 32 + lane]);
  }
}

// Y partial fragments -> shared memory [NOUT][NP][NP]
template <int NT, int NOUT>
__device__ __forceinline__ void ws_store_partial(const double (&Y)[NOUT][NT][NT][2], double* dst) {
  constexpr int NP = 8 * NT;
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
#pragma unroll
  for (int o = 0; o < NOUT; ++o)
#pragma unroll
    for (int bt = 0; bt < NT; ++bt)
#pragma unroll
      for (int at = 0; at < NT; ++at)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          dst[(o * NP + 8 * at + 2 * c + j) * NP + 8 * bt + r] = Y[o][bt][at][j];
}


// Stage the element's coefficient tiles of fields [f0, f0+nf) of MODE's field
// list into dst (rows of n contiguous doubles), all threads of the CTA, as
// 8-byte cp.async copies (zero fill in the padding): every load in flight at
// once, no register round trip.  The caller commits and waits.
template <int NP, int MODE>
__device__ __forceinline__ void ws_stage_tiles(const ElemArgs& A, int cx, int cy, int f0, int nf, double* dst) {
  constexpr int LDT = NP + 2, TILE = NP * LDT;
  for (int f = 0; f < nf; ++f) {
    const double* src;
    int comp;
    field_src<MODE>(A, f0 + f, src, comp);
    src += comp * A.ncomp;
    for (int idx = threadIdx.x; idx < NP * NP; idx += blockDim.x) {
      const int a = idx / NP, b = idx - a * NP;
      const bool in = a < A.n && b < A.n;
      cp_async8z(dst + f * TILE + a * LDT + b, in ? src + psi_index(A, cx, cy, a, b) : src, in);
    }
  }
}

// The element's gradient-bound samples phi (nq x nq) into dst (row stride QP)
template <int QP>
__device__ __forceinline__ void ws_stage_phi(const ElemArgs& A, int e, double* dst) {
  const double* src = A.phi + (long long)e * A.nq * A.nq;
  for (int idx = threadIdx.x; idx < A.nq * A.nq; idx += blockDim.x) {
    const int g = idx / A.nq, h = idx - g * A.nq;
    cp_async8z(dst + g * QP + h, src + idx, true);
  }
}

// Fixed-order sum of the QT row-tile partials of one output group + epilogue.
template <int NT, int QT, int MODE>
__device__ __forceinline__ void ws_reduce_write(const ElemArgs& A, int e, const double* part, const double* sInv,
                                                int t0, int nthreads) {
  constexpr int NP = 8 * NT, NOUT = ModeTraits<MODE>::NOUT;
  const int cx = e / A.ncy, cy = e - (e / A.ncy) * A.ncy;
  const int nn = A.n * A.n;
  for (int idx = t0; idx < NOUT * nn; idx += nthreads) {
    const int o = idx / nn, rem = idx - o * nn, a = rem / A.n, b = rem - a * A.n;
    double y = 0.0;
#pragma unroll
    for (int w = 0; w < QT; ++w) y += part[((w * NOUT + o) * NP + a) * NP + b];
    write_moment<MODE>(A, e, cx, cy, o, a, b, y, sInv);
  }
}

template <int NT, int QT, int MODE>
__global__ void __launch_bounds__(32 * QT, QT <= 4 ? 4 : (QT <= 5 ? 2 : 1))
k_wsplit(ElemArgs A) {
  using TR = ModeTraits<MODE>;
  using CF = WsplitCfg<NT, QT, MODE>;
  constexpr int NP = CF::NP, QP = CF::QP, NOUT = TR::NOUT, NW = TR::NW;
  extern __shared__ double smem[];
  double* sS = smem;
  double* sT = sS + QP * NP;
  double* sInv = sT + NP * QP;
  double* sBody = sInv + CF::INV;
  double* sTile = sBody;                   // [NIN][NP][LDT]
  double* sW = sBody + CF::TILES;          // [rt][ht][w][lane][2] (cached modes)
  double* sY = sBody;                      // [rt][NOUT][NP][NP] after the main loop
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt = warp, e = blockIdx.x;
  for (int i = 2 * threadIdx.x; i < QP * NP; i += 2 * blockDim.x) {
    cp_async16(sS + i, A.Sf + i);
    cp_async16(sT + i, A.Tf + i);
  }
  cp_async_commit();
  for (int i = threadIdx.x; i < NP; i += blockDim.x) sInv[i] = kInvOdd[i];
  // a kernel writing a weight cache never releases its dependents early
  if (!((MODE == M_OBST_RES || MODE == M_GRAD_RES) && A.wc_out != nullptr)) pdl_trigger();
  pdl_wait();
  if (e >= A.N) return;
  const int cx = e / A.ncy, cy = e - cx * A.ncy;
  if constexpr (CF::cached) {
    const double* src = A.wc_in + wc_index(e, QT, rt, 0, NW, 0, lane);
    double* dst = sW + rt * CF::WROW;
#pragma unroll
    for (int t = 0; t < QT * NW; ++t) cp_async16(dst + t * 64 + 2 * lane, src + t * 64);
    cp_async_commit();
  }
  ws_stage_tiles<NP, MODE>(A, cx, cy, 0, TR::NIN, sTile);
  double* sPhi = sBody + CF::TILES + CF::WTS;
  if constexpr (CF::PHI) ws_stage_phi<QP>(A, e, sPhi);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double Y[NOUT][NT][NT][2];
  bool flag = false;
  auto nop = [] {};
  ws_rowtile<NT, QT, MODE>(A, e, rt, sS, sT, sTile, CF::cached ? sW + rt * CF::WROW : nullptr, nullptr, Y, flag,
                           nop, nop, CF::PHI ? sPhi : nullptr);
  if constexpr (MODE == M_OBST_RES) {
    if (__any_sync(0xffffffffu, flag) && lane == 0) atomicOr(A.flag, 1);
  }
  __syncthreads();          // tiles and weights are dead: the body holds the partials
  ws_store_partial<NT, NOUT>(Y, sY + (size_t)rt * NOUT * NP * NP);
  __syncthreads();
  ws_reduce_write<NT, QT, MODE>(A, e, sY, sInv, threadIdx.x, blockDim.x);
}

}  // namespace hpg
