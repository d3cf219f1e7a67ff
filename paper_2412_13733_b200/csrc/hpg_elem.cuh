// Stage (a)->(b)->(c) element kernels: sum-factorised synthesis, pointwise
// LVPP map and test-side analysis, fused so point values never touch HBM.
//
// Per element (tile side n padded to NP = 8*NT, Q padded to QP = 8*QT), for
// each 8-row tile rt of the Q x Q point grid:
//   P_rt  = S[rt,:] C            (8 x NP)   A = PK(S) (smem), B = C (smem)
//   V_rt  = P_rt S^T             (8 x QP)   A = P (regs),     B = PK(S)
//   W_rt  = map(V_rt, ...)                  pointwise, in registers
//   R_rt  = T W_rt^T             (NP x 8)   A = PK(T),        B = W (regs)
//   Y    += R_rt T[:,rt]^T       (NP x NP)  A = R (regs),     B = PK(T)
// and M[a][b] = w_a w_b Y[b][a] (reference CellKernel2D.moments,
// assembly.py:249-251).  Zero-padded tables make the padded rows/cols inert.
#pragma once
#include <cooperative_groups.h>

#include "hpg_common.cuh"
#include "hpg_pointmap.cuh"
#include "hpg_ucell.cuh"

namespace hpg {

constexpr int WARP_CTA_WARPS = 4;
constexpr int CTA_WARPS = 8;

template <int MODE>
__device__ __forceinline__ void field_src(const ElemArgs& A, int f, const double*& ptr, int& comp) {
  if constexpr (MODE == M_OBST_RES) { ptr = A.in0; comp = 0; }
  else if constexpr (MODE == M_OBST_APPLY) { ptr = f == 0 ? A.in0 : A.in1; comp = 0; }
  else if constexpr (MODE == M_OBST_CACHED) { ptr = A.in1; comp = 0; }
  else if constexpr (MODE == M_GRAD_RES) { ptr = A.in0; comp = f; }
  else if constexpr (MODE == M_GRAD_APPLY) { ptr = f < 2 ? A.in0 : A.in1; comp = f & 1; }
  else if constexpr (MODE == M_GRAD_CACHED) { ptr = A.in1; comp = f; }
  else { ptr = nullptr; comp = 0; }
}

__device__ __forceinline__ long long wc_index(int e, int QT, int rt, int ht, int NW, int w, int lane) {
  return (((((long long)e * QT + rt) * QT + ht) * NW + w) * 32 + lane) * 2;
}

// Final value of moment (a, b), output component o, of cell e.
template <int MODE>
__device__ __forceinline__ void write_moment(const ElemArgs& A, int e, int cx, int cy, int o,
                                             int a, int b, double y, const double* inv = kInvOdd) {
  constexpr bool gradient = MODE >= M_GRAD_RES && MODE <= M_GRAD_CACHED;
  double wa = A.hx[cx] * inv[a];
  double wb = A.hy[cy] * inv[b];
  double val = (wa * y) * wb;
  if (A.out_cellmajor) {
    A.out[((long long)e * A.n + a) * A.n + b] = val;
    return;
  }
  long long idx = (long long)o * A.ncomp + psi_index(A, cx, cy, a, b);
  if (A.residual) {
    // b_psi already holds phi_mom - B^T u (obstacle) / -B^T u (gradient) from
    // the U-side kernel: finish proximal.py:123 / :125 in the reference's order
    if constexpr (gradient) val = A.out[idx] + val;
    else val = A.out[idx] - val;
  }
  A.out[idx] = val;
}

// Stage (b) for one C-fragment position pair (j = 0, 1) of tile (rt, ht).
template <int MODE, int NSYN, int NOUT, int NW>
__device__ __forceinline__ void map_pair(const ElemArgs& A, int e, int QT, int rt, int ht, int lane,
                                         const double (&V)[NSYN > 0 ? NSYN : 1][2],
                                         double (&Vw)[NOUT][2], bool& flag) {
  constexpr bool gradient = MODE >= M_GRAD_RES && MODE <= M_GRAD_CACHED;
  constexpr bool cached = MODE == M_OBST_CACHED || MODE == M_GRAD_CACHED;
  constexpr bool writes = MODE == M_OBST_RES || MODE == M_GRAD_RES;
  const int r = lane >> 2, c = lane & 3;
  const int g = 8 * rt + r;
  double win[NW > 0 ? NW : 1][2], wout[NW > 0 ? NW : 1][2];
  if constexpr (cached) {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      double2 t = __ldg(reinterpret_cast<const double2*>(A.wc_in + wc_index(e, QT, rt, ht, NW, w, lane)));
      win[w][0] = t.x;
      win[w][1] = t.y;
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int h = 8 * ht + 2 * c + j;
    const bool inside = g < A.nq && h < A.nq;
    double v[NSYN > 0 ? NSYN : 1];
    double vw[NOUT];
    double wi[NW > 0 ? NW : 1], wo[NW > 0 ? NW : 1];
    if constexpr (MODE == M_VALUES) {
      vw[0] = inside ? __ldg(A.in0 + ((long long)e * A.nq + g) * A.nq + h) : 0.0;
    } else {
#pragma unroll
      for (int f = 0; f < NSYN; ++f) v[f] = V[f][j];
      double phi = 0.0;
      if constexpr (gradient) {
        if (!cached && inside) phi = __ldg(A.phi + ((long long)e * A.nq + g) * A.nq + h);
      }
#pragma unroll
      for (int w = 0; w < NW; ++w) wi[w] = win[w][j];
      bool fl = false;
      point_map<MODE>(v, phi, wi, wo, vw, fl);
      // padded points (g or h >= nq) are inert: zero weight, never flagged
      // (0 * inf in the padded table rows must not leak NaN into the cell)
      if (inside) {
        flag |= fl;
      } else {
#pragma unroll
        for (int o = 0; o < NOUT; ++o) vw[o] = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) wo[w] = 0.0;
      }
#pragma unroll
      for (int w = 0; w < NW; ++w) wout[w][j] = wo[w];
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o) Vw[o][j] = vw[o];
  }
  if constexpr (writes) {
    if (A.wc_out != nullptr) {
#pragma unroll
      for (int w = 0; w < NW; ++w)
        *reinterpret_cast<double2*>(A.wc_out + wc_index(e, QT, rt, ht, NW, w, lane)) =
            make_double2(wout[w][0], wout[w][1]);
    }
  }
}

// Stage (b) of the cached modes with the weights already in registers
// (C-fragment pair j = 0, 1 of tile (rt, ht); padded points carry weight 0).
template <int MODE, int NSYN, int NOUT, int NW>
__device__ __forceinline__ void map_pair_w(const double (&V)[NSYN > 0 ? NSYN : 1][2],
                                           const double (&W)[NW > 0 ? NW : 1][2],
                                           double (&Vw)[NOUT][2], bool row_in, int h0, int nq) {
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool inside = row_in && h0 + j < nq;
    double v[NSYN > 0 ? NSYN : 1], wi[NW > 0 ? NW : 1], wo[NW > 0 ? NW : 1], vw[NOUT];
#pragma unroll
    for (int f = 0; f < NSYN; ++f) v[f] = V[f][j];
#pragma unroll
    for (int w = 0; w < NW; ++w) wi[w] = W[w][j];
    bool fl = false;
    point_map<MODE>(v, 0.0, wi, wo, vw, fl);
#pragma unroll
    for (int o = 0; o < NOUT; ++o) Vw[o][j] = inside ? vw[o] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Warp-per-element kernel: all fragments in registers, tables in smem.
//
// Latency structure (one wave: the grid never exceeds the resident slots):
//  * launched with programmatic stream serialization (PDL): the table fill
//    into shared memory runs while the previous kernel drains, then
//    griddepcontrol.wait orders every read of psi / x / weights after it
//    (the only reads issued before the wait are the constant tables);
//  * small tiles (NIN*2*NT^2 <= 8 doubles) skip the shared-memory staging:
//    each lane loads exactly the B-fragment entries C[8(ks>>1)+2c+(ks&1)][8nt+r]
//    it feeds to the first contraction (rows of 8 consecutive doubles);
//  * cached modes prefetch the next row tile's point weights one iteration
//    ahead, so the map never waits on L2.
template <int NT, int QT, int MODE>
struct WarpCfg {
  using TR = ModeTraits<MODE>;
#ifndef HPG_REGX_CACHED
#define HPG_REGX_CACHED 8
#endif
#ifndef HPG_SPLIT_R
#define HPG_SPLIT_R 1
#endif
#ifndef HPG_SPLIT_V
#define HPG_SPLIT_V 0
#endif
  static constexpr bool REGX = TR::NIN * 2 * NT * NT <= (MODE == M_OBST_CACHED || MODE == M_GRAD_CACHED ? HPG_REGX_CACHED : 4);
  // independent even/odd accumulation chains in the R / V contractions
  static constexpr bool SPLIT_R = HPG_SPLIT_R, SPLIT_V = HPG_SPLIT_V;
  static constexpr bool cached = MODE == M_OBST_CACHED || MODE == M_GRAD_CACHED;
  // cached modes: the cell's point weights are copied to shared memory with
  // cp.async when they fit (<= 16 KB per warp), read back by the same lane
  static constexpr int WDBL_CELL = QT * QT * TR::NW * 64;
  // whole-cell staging while it stays small (QT <= 3: config 1); larger QT
  // (reference rule, nq = 34: QT = 5) keeps two row tiles in flight instead
  // (ROLL: row tile rt+2 copied while rt+1 is in use), so the weight slices
  // do not cap the CTAs per SM
  static constexpr bool ROLL = cached && QT > 3 && 2 * QT * TR::NW * 64 * 8 <= 16 * 1024;
  static constexpr int WDBL = ROLL ? 2 * QT * TR::NW * 64 : WDBL_CELL;
  static constexpr bool WSMEM = cached && WDBL * 8 <= 16 * 1024;
  static constexpr bool WRITES_WC = MODE == M_OBST_RES || MODE == M_GRAD_RES;
  // cached small tiles (config 1): 2-warp CTAs, each warp streams CPW = 2
  // cells with the next cell's x fragments and weights in flight during the
  // current cell's contractions (the load burst at kernel start is halved)
#ifndef HPG_PIPE2
#define HPG_PIPE2 0
#endif
  static constexpr bool PIPE = HPG_PIPE2 && cached && REGX && WSMEM && NT <= 2 && QT <= 3;
  static constexpr int W = PIPE ? 2 : WARP_CTA_WARPS;
  static constexpr int CPW = PIPE ? 2 : 1;
  // 4096 cells (config 1) must fit one wave of 4-warp CTAs: >= 7 CTAs / SM
#ifndef HPG_WARP_MINB
#define HPG_WARP_MINB 7
#endif
#ifndef HPG_ROLL_MINB
#define HPG_ROLL_MINB 7
#endif
  static constexpr int MINB_ = (NT <= 2 && QT <= 3 && TR::NIN == 1) ? HPG_WARP_MINB
                               : (ROLL && NT <= 2 ? HPG_ROLL_MINB : 1);
#ifndef HPG_UNROLL_RT
#define HPG_UNROLL_RT 0
#endif
  static constexpr bool UNROLL_RT = HPG_UNROLL_RT && cached && QT <= 3;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

template <int NT, int QT, int MODE>
__global__ void __launch_bounds__(32 * WarpCfg<NT, QT, MODE>::W, (WarpCfg<NT, QT, MODE>::MINB_))
k_warp(ElemArgs A) {
  using TR = ModeTraits<MODE>;
  using CF = WarpCfg<NT, QT, MODE>;
  constexpr int NP = 8 * NT, QP = 8 * QT, NK = NP / 4, QK = QP / 4;
  constexpr int LDT = NP + 2, TILE = NP * LDT;
  constexpr int NIN = TR::NIN, NSYN = TR::NSYN, NOUT = TR::NOUT, NW = TR::NW;
  constexpr bool REGX = CF::REGX, WSMEM = CF::WSMEM;
  constexpr int NSTAGE = REGX ? 0 : NIN;
  constexpr int WDBL = WSMEM ? CF::WDBL : 0;
  extern __shared__ double smem[];
  double* sS = smem;
  double* sT = sS + QP * NP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  double* sTile = sT + NP * QP + warp * (NSTAGE > 0 ? NSTAGE * TILE : 0);
  constexpr int W = CF::W, NBUF = CF::PIPE ? 2 : 1;
  double* sW = sT + NP * QP + W * NSTAGE * TILE + warp * NBUF * WDBL;   // [buf][rt][ht][w][lane][2]
  double* sInv = sT + NP * QP + W * (NSTAGE * TILE + NBUF * WDBL);      // 1/(2k+1), k < NP
  // tables: every copy in flight at once (cp.async, no register staging)
  for (int i = 2 * threadIdx.x; i < QP * NP; i += 2 * blockDim.x) {
    cp_async16(sS + i, A.Sf + i);
    cp_async16(sT + i, A.Tf + i);
  }
  cp_async_commit();
  for (int i = threadIdx.x; i < NP; i += blockDim.x) sInv[i] = kInvOdd[i];
  // before the grid-dependency wait only the (constant) tables are copied --
  // PDL makes the previous grid's writes visible after griddepcontrol.wait,
  // not before -- and, when the host knows the weight cache was NOT written
  // by the immediately preceding kernel (A.wc_early, set by hpgApplyCached
  // from the plan's call history; cache writers never trigger their
  // dependents early), the first cell's weights
  int buf = 0;
  // ROLL: one row tile's weights into half h of the warp's slice
  auto load_rt = [&](int e, int rt, int h) {
    const double* src = A.wc_in + wc_index(e, QT, rt, 0, NW, 0, lane);
    double* dst = sW + h * (QT * NW * 64);
#pragma unroll
    for (int t = 0; t < QT * NW; ++t) cp_async16(dst + t * 64 + 2 * lane, src + t * 64);
    cp_async_commit();
  };
  auto load_weights = [&](int e, int b) {
    if constexpr (CF::ROLL) {
      load_rt(e, 0, 0);
      load_rt(e, 1, 1);
    } else if constexpr (WSMEM) {
      const double* src = A.wc_in + wc_index(e, QT, 0, 0, NW, 0, lane);
      double* dst = sW + b * WDBL;
#pragma unroll
      for (int t = 0; t < QT * QT * NW; ++t) cp_async16(dst + t * 64 + 2 * lane, src + t * 64);
      cp_async_commit();
    }
  };
  const int stride = gridDim.x * W;
  int e = A.e0 + blockIdx.x * W + warp;
  if (A.wc_early && e < A.N) load_weights(e, 0);
  // one wave: let the next kernel in the stream start its prologue now --
  // except a kernel writing a weight cache (see above)
  if (!(CF::WRITES_WC && A.wc_out != nullptr)) pdl_trigger();
  pdl_wait();
  if (!A.wc_early && e < A.N) load_weights(e, 0);

  using XFrag = double[REGX ? NIN : 1][REGX ? NK : 1][REGX ? NT : 1];
  XFrag X, Xn;
  // issue the loads of cell e: the first contraction's B fragments (registers
  // or the warp's staging tile)
  auto load_cell = [&](int e, XFrag& Xd) {
    const int cx = e / A.ncy, cy = e - cx * A.ncy;
    if constexpr (REGX) {
#pragma unroll
      for (int f = 0; f < NIN; ++f) {
        const double* src;
        int comp;
        field_src<MODE>(A, f, src, comp);
        src += comp * A.ncomp + psi_index(A, cx, cy, 0, 0);
#pragma unroll
        for (int ks = 0; ks < NK; ++ks) {
          const int a = 8 * (ks >> 1) + 2 * c + (ks & 1);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int b = 8 * nt + r;
            Xd[f][ks][nt] = (a < A.n && b < A.n) ? __ldg(src + (long long)a * A.ld + b) : 0.0;
          }
        }
      }
    } else {
#pragma unroll
      for (int f = 0; f < NIN; ++f) {
        const double* src;
        int comp;
        field_src<MODE>(A, f, src, comp);
        src += comp * A.ncomp;
        for (int idx = lane; idx < NP * NP; idx += 32) {
          int a = idx / NP, b = idx - a * NP;
          double v = 0.0;
          if (a < A.n && b < A.n) v = __ldg(src + psi_index(A, cx, cy, a, b));
          sTile[f * TILE + a * LDT + b] = v;
        }
      }
    }
  };
  if (e < A.N) load_cell(e, X);
  if constexpr (CF::PIPE) {
    // tables (first group) must be in; the cell's weights may still fly
    if (e < A.N) cp_async_wait_group<1>();
    else cp_async_wait_all();
  } else {
    cp_async_wait_all();
  }
  __syncthreads();   // tables

  for (; e < A.N; e += stride) {
    const int cx = e / A.ncy, cy = e - cx * A.ncy;
    if constexpr (!REGX) __syncwarp();
    bool more = false;
    if constexpr (CF::PIPE) {
      // next cell's weights and x fragments in flight during this cell
      more = e + stride < A.N;
      if (more) {
        load_weights(e + stride, buf ^ 1);
        load_cell(e + stride, Xn);
      }
    }
    const double* sWc = sW + buf * WDBL;
    double Y[NOUT][NT][NT][2];
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int k = 0; k < NT; ++k) Y[o][i][k][0] = Y[o][i][k][1] = 0.0;
    bool flag = false;

    // cached small tiles: unrolled row-tile loop, so the scheduler can overlap
    // the synthesis of row tile rt+1 with the analysis of rt
#pragma unroll (CF::UNROLL_RT ? QT : 1)
    for (int rt = 0; rt < QT; ++rt) {
      double V[NSYN > 0 ? NSYN : 1][QT][2];
#pragma unroll
      for (int f = 0; f < NSYN; ++f) {
        double P[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) P[nt][0] = P[nt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < NK; ++ks) {
          double a = sS[(rt * NK + ks) * 32 + lane];
          if constexpr (REGX) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma(P[nt], a, X[f][ks][nt]);
          } else {
            const double* row = sTile + f * TILE + (8 * (ks >> 1) + 2 * c + (ks & 1)) * LDT + r;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma(P[nt], a, row[8 * nt]);
          }
        }
#pragma unroll
        for (int ht = 0; ht < QT; ++ht) {
          V[f][ht][0] = V[f][ht][1] = 0.0;
          if constexpr (CF::SPLIT_V) {
            double V1[2] = {0.0, 0.0};
#pragma unroll
            for (int ks = 0; ks < NK; ks += 2) {
              dmma(V[f][ht], P[ks >> 1][0], sS[(ht * NK + ks) * 32 + lane]);
              dmma(V1, P[ks >> 1][1], sS[(ht * NK + ks + 1) * 32 + lane]);
            }
            V[f][ht][0] += V1[0];
            V[f][ht][1] += V1[1];
          } else {
#pragma unroll
            for (int ks = 0; ks < NK; ++ks)
              dmma(V[f][ht], P[ks >> 1][ks & 1], sS[(ht * NK + ks) * 32 + lane]);
          }
        }
      }
      double Vw[NOUT][QT][2];
#pragma unroll
      for (int ht = 0; ht < QT; ++ht) {
        double Vp[NSYN > 0 ? NSYN : 1][2];
#pragma unroll
        for (int f = 0; f < NSYN; ++f) { Vp[f][0] = V[f][ht][0]; Vp[f][1] = V[f][ht][1]; }
        double out2[NOUT][2];
        if constexpr (WSMEM) {
          if constexpr (CF::ROLL) {
            if (ht == 0) {
              if (rt + 1 < QT) cp_async_wait_group<1>();   // rt in, rt+1 may fly
              else cp_async_wait_all();
            }
          } else if (rt == 0 && ht == 0) {
            if (more) cp_async_wait_group<1>();
            else cp_async_wait_all();
          }
          double Wc[NW][2];
          const double* wsrc = CF::ROLL ? sW + (rt & 1) * (QT * NW * 64) + (ht * NW) * 64
                                        : sWc + ((rt * QT + ht) * NW) * 64;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const double2 t = *reinterpret_cast<const double2*>(wsrc + w * 64 + 2 * lane);
            Wc[w][0] = t.x;
            Wc[w][1] = t.y;
          }
          map_pair_w<MODE, NSYN, NOUT, NW>(Vp, Wc, out2, 8 * rt + r < A.nq, 8 * ht + 2 * c, A.nq);
        } else {
          map_pair<MODE, NSYN, NOUT, NW>(A, e, QT, rt, ht, lane, Vp, out2, flag);
        }
#pragma unroll
        for (int o = 0; o < NOUT; ++o) { Vw[o][ht][0] = out2[o][0]; Vw[o][ht][1] = out2[o][1]; }
      }
      if constexpr (CF::ROLL) {
        // row tile rt's weights are consumed: its half takes rt + 2
        if (rt + 2 < QT) load_rt(e, rt + 2, rt & 1);
      }
#pragma unroll
      for (int o = 0; o < NOUT; ++o) {
        double R[NT][2];
#pragma unroll
        for (int bt = 0; bt < NT; ++bt) {
          R[bt][0] = R[bt][1] = 0.0;
          if constexpr (CF::SPLIT_R) {
            // two independent chains (even / odd k-steps)
            double R1[2] = {0.0, 0.0};
#pragma unroll
            for (int ks = 0; ks < QK; ks += 2) {
              dmma(R[bt], sT[(bt * QK + ks) * 32 + lane], Vw[o][ks >> 1][0]);
              dmma(R1, sT[(bt * QK + ks + 1) * 32 + lane], Vw[o][ks >> 1][1]);
            }
            R[bt][0] += R1[0];
            R[bt][1] += R1[1];
          } else {
#pragma unroll
            for (int ks = 0; ks < QK; ++ks)
              dmma(R[bt], sT[(bt * QK + ks) * 32 + lane], Vw[o][ks >> 1][ks & 1]);
          }
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
    if constexpr (MODE == M_OBST_RES) {
      if (__any_sync(0xffffffffu, flag) && lane == 0) atomicOr(A.flag, 1);
    }
    // REGX / cp.async: the next cell's loads are in flight during the epilogue
    if constexpr (CF::PIPE) {
      if (more) {
#pragma unroll
        for (int f = 0; f < NIN; ++f)
#pragma unroll
          for (int ks = 0; ks < NK; ++ks)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) X[f][ks][nt] = Xn[f][ks][nt];
      }
      buf ^= 1;
    } else {
      if (e + stride < A.N) load_weights(e + stride, 0);
      if constexpr (REGX) {
        if (e + stride < A.N) load_cell(e + stride, X);
      }
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
#pragma unroll
      for (int bt = 0; bt < NT; ++bt)
#pragma unroll
        for (int at = 0; at < NT; ++at)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            int a = 8 * at + 2 * c + j, b = 8 * bt + r;
            if (a < A.n && b < A.n) write_moment<MODE>(A, e, cx, cy, o, a, b, Y[o][bt][at][j], sInv);
          }
    if constexpr (!REGX) {
      __syncwarp();
      if (e + stride < A.N) load_cell(e + stride, X);
    }
  }
}

// ---------------------------------------------------------------------------
// CTA-per-(element, row-tile range) kernel for any size (runtime NT, QT):
// the same four contractions, warps splitting tiles, stage results passed
// through shared memory in C-fragment order (read back with LDS.128 by the
// same lane).  Used for large n (config 3) and as the general path.
template <int MODE, int MAXS, int CTA_WARPS>
__global__ void __launch_bounds__(32 * CTA_WARPS, 1)
k_cta(ElemArgs A) {
  pdl_wait();
  using TR = ModeTraits<MODE>;
  constexpr int NIN = TR::NIN, NSYN = TR::NSYN, NOUT = TR::NOUT, NW = TR::NW;
  const int NT = A.NT, QT = A.QT;
  const int NP = 8 * NT, NK = NP / 4, QK = 2 * QT;
  const int LDT = NP + 2, TILE = NP * LDT;
  extern __shared__ double smem[];
  double* sTile = smem;
  double* sP = sTile + NIN * TILE;               // [NSYN][NT][64]
  double* sV = sP + NSYN * NT * 64;               // [NOUT][QT][64]
  double* sR = sV + NOUT * QT * 64;               // [NOUT][NT][64]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  const int e = blockIdx.x / A.splits, sp = blockIdx.x - e * A.splits;
  if (e >= A.N) return;
  // table operands: shared memory when they fit (config 2), else L1/L2
  const double* tS = A.Sf;
  const double* tT = A.Tf;
  if (A.smem_tables) {
    // bit 0: PK(S), bit 1: PK(T) (config 3 fits only PK(T) next to its tile)
    double* s0 = sR + NOUT * NT * 64;
    double* s1 = s0 + ((A.smem_tables & 1) ? QT * NP * 8 : 0);
    for (int i = 2 * threadIdx.x; i < QT * NP * 8; i += 2 * blockDim.x) {
      if (A.smem_tables & 1) cp_async16(s0 + i, A.Sf + i);
      if (A.smem_tables & 2) cp_async16(s1 + i, A.Tf + i);
    }
    cp_async_commit();
    cp_async_wait_all();
    if (A.smem_tables & 1) tS = s0;
    if (A.smem_tables & 2) tT = s1;
  }
  const int rt0 = (sp * QT) / A.splits, rt1 = ((sp + 1) * QT) / A.splits;
  const int cx = e / A.ncy, cy = e - cx * A.ncy;

  for (int f = 0; f < NIN; ++f) {
    const double* src;
    int comp;
    field_src<MODE>(A, f, src, comp);
    src += comp * A.ncomp;
    for (int idx = threadIdx.x; idx < NP * NP; idx += blockDim.x) {
      int a = idx / NP, b = idx - a * NP;
      double v = 0.0;
      if (a < A.n && b < A.n) v = __ldg(src + psi_index(A, cx, cy, a, b));
      sTile[f * TILE + a * LDT + b] = v;
    }
  }
  __syncthreads();
  const int ny = NOUT * NT * NT;
  double Y[MAXS][2];
#pragma unroll
  for (int s = 0; s < MAXS; ++s) Y[s][0] = Y[s][1] = 0.0;
  bool flag = false;

  for (int rt = rt0; rt < rt1; ++rt) {
    // (1) P tiles
    for (int it = warp; it < NSYN * NT; it += CTA_WARPS) {
      int f = it / NT, nt = it - f * NT;
      // two independent accumulation chains (even / odd k-steps): half the
      // dependent DMMA latency per tile (NK = 2 NT is even)
      double P[2] = {0.0, 0.0}, P1[2] = {0.0, 0.0};
      const double* col = sTile + f * TILE + 8 * nt + r;
      #pragma unroll 4
      for (int ks = 0; ks < NK; ks += 2) {
        dmma(P, tS[(rt * NK + ks) * 32 + lane], col[(8 * (ks >> 1) + 2 * c) * LDT]);
        dmma(P1, tS[(rt * NK + ks + 1) * 32 + lane], col[(8 * (ks >> 1) + 2 * c + 1) * LDT]);
      }
      *reinterpret_cast<double2*>(sP + (f * NT + nt) * 64 + 2 * lane) = make_double2(P[0] + P1[0], P[1] + P1[1]);
    }
    __syncthreads();
    // (2) V tiles + pointwise map
    for (int ht = warp; ht < QT; ht += CTA_WARPS) {
      double V[NSYN > 0 ? NSYN : 1][2];
#pragma unroll
      for (int f = 0; f < NSYN; ++f) {
        double V1[2] = {0.0, 0.0};
        V[f][0] = V[f][1] = 0.0;
        #pragma unroll 4
        for (int t = 0; t < NT; ++t) {
          double2 pa = *reinterpret_cast<const double2*>(sP + (f * NT + t) * 64 + 2 * lane);
          dmma(V[f], pa.x, tS[(ht * NK + 2 * t) * 32 + lane]);
          dmma(V1, pa.y, tS[(ht * NK + 2 * t + 1) * 32 + lane]);
        }
        V[f][0] += V1[0];
        V[f][1] += V1[1];
      }
      double out2[NOUT][2];
      map_pair<MODE, NSYN, NOUT, NW>(A, e, QT, rt, ht, lane, V, out2, flag);
#pragma unroll
      for (int o = 0; o < NOUT; ++o)
        *reinterpret_cast<double2*>(sV + (o * QT + ht) * 64 + 2 * lane) = make_double2(out2[o][0], out2[o][1]);
    }
    __syncthreads();
    // (3) R tiles
    for (int it = warp; it < NOUT * NT; it += CTA_WARPS) {
      int o = it / NT, bt = it - o * NT;
      double R[2] = {0.0, 0.0}, R1[2] = {0.0, 0.0};
      #pragma unroll 4
      for (int t = 0; t < QT; ++t) {
        double2 vb = *reinterpret_cast<const double2*>(sV + (o * QT + t) * 64 + 2 * lane);
        dmma(R, tT[(bt * QK + 2 * t) * 32 + lane], vb.x);
        dmma(R1, tT[(bt * QK + 2 * t + 1) * 32 + lane], vb.y);
      }
      *reinterpret_cast<double2*>(sR + (o * NT + bt) * 64 + 2 * lane) = make_double2(R[0] + R1[0], R[1] + R1[1]);
    }
    __syncthreads();
    // (4) Y accumulation (tiles statically owned by warps)
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
      int it = warp + CTA_WARPS * s;
      if (it < ny) {
        int o = it / (NT * NT), rem = it - o * NT * NT;
        int bt = rem / NT, at = rem - bt * NT;
        double2 ra = *reinterpret_cast<const double2*>(sR + (o * NT + bt) * 64 + 2 * lane);
        dmma(Y[s], ra.x, tT[(at * QK + 2 * rt) * 32 + lane]);
        dmma(Y[s], ra.y, tT[(at * QK + 2 * rt + 1) * 32 + lane]);
      }
    }
  }
  if constexpr (MODE == M_OBST_RES) {
    if (__any_sync(0xffffffffu, flag) && lane == 0) atomicOr(A.flag, 1);
  }
  if (A.cluster_red) {
    // the A.splits CTAs of cell e are one cluster: stage this CTA's partial
    // Y in its own shared memory, then CTA sp reduces a slice of the entries
    // over the cluster's partials through DSMEM in split order (the same
    // deterministic sum as k_cta_reduce), with no global partials and no
    // second launch
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __syncthreads();                       // tile / stage buffers are dead
    double* sY = smem;                     // [NOUT][NP][NP]
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
      int it = warp + CTA_WARPS * s;
      if (it < ny) {
        int o = it / (NT * NT), rem = it - o * NT * NT;
        int bt = rem / NT, at = rem - bt * NT;
#pragma unroll
        for (int j = 0; j < 2; ++j) sY[(o * NP + 8 * at + 2 * c + j) * NP + 8 * bt + r] = Y[s][j];
      }
    }
    cl.sync();
    const int nn = A.n * A.n, total = NOUT * nn;
    const int chunk = (total + A.splits - 1) / A.splits;
    const int i1 = min(total, (sp + 1) * chunk);
    for (int idx = sp * chunk + threadIdx.x; idx < i1; idx += blockDim.x) {
      const int o = idx / nn, rem = idx - o * nn, a = rem / A.n, b = rem - a * A.n;
      const int off = (o * NP + a) * NP + b;
      double y = 0.0;
      for (int q = 0; q < A.splits; ++q) y += cl.map_shared_rank(sY, q)[off];
      write_moment<MODE>(A, e, cx, cy, o, a, b, y);
    }
    cl.sync();                             // partials stay alive until read
    return;
  }
#pragma unroll
  for (int s = 0; s < MAXS; ++s) {
    int it = warp + CTA_WARPS * s;
    if (it < ny) {
      int o = it / (NT * NT), rem = it - o * NT * NT;
      int bt = rem / NT, at = rem - bt * NT;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        int a = 8 * at + 2 * c + j, b = 8 * bt + r;
        if (A.splits == 1) {
          if (a < A.n && b < A.n) write_moment<MODE>(A, e, cx, cy, o, a, b, Y[s][j]);
        } else {
          A.partial[(((long long)e * A.splits + sp) * NOUT + o) * NP * NP + a * NP + b] = Y[s][j];
        }
      }
    }
  }
}

// Deterministic reduction of the row-tile-split partials + epilogue.
template <int MODE>
__global__ void k_cta_reduce(ElemArgs A) {
  pdl_wait();
  using TR = ModeTraits<MODE>;
  constexpr int NOUT = TR::NOUT;
  const int NP = 8 * A.NT;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long total = (long long)A.N * NOUT * A.n * A.n;
  if (tid >= total) return;
  int b = tid % A.n;
  long long t = tid / A.n;
  int a = t % A.n;
  t /= A.n;
  int o = t % NOUT;
  int e = (int)(t / NOUT);
  // all split partials loaded before the (fixed-order) sum
  double y = 0.0;
  const double* pp = A.partial + ((long long)e * A.splits * NOUT + o) * NP * NP + a * NP + b;
  const long long stride = (long long)NOUT * NP * NP;
  int sp = 0;
  for (; sp + 8 <= A.splits; sp += 8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = pp[(sp + q) * stride];
#pragma unroll
    for (int q = 0; q < 8; ++q) y += v[q];
  }
  for (; sp < A.splits; ++sp) y += pp[sp * stride];
  const int cx = e / A.ncy, cy = e - cx * A.ncy;
  write_moment<MODE>(A, e, cx, cy, o, a, b, y);
}

}  // namespace hpg
