// Large-tile element kernel for few, high-degree elements (config 3: 16 cells,
// n = 81, Gauss Q = 128 -> NT = 11, QT = 16): the k_cta decomposition (CTA
// per (element, row-tile split), warps over stage tiles, stage results in
// shared memory in C-fragment order) with compile-time tile counts and
// every operand of the inner loops on chip:
//
//  * both PK(S) and PK(T) staged in shared memory (2 x 90 KB, cp.async);
//  * the element's coefficient tile C never staged: warp nt keeps its column
//    block's B fragments (NK = 22 doubles per field) in registers;
//  * the CTA's RB row tiles go through each stage together, so every table
//    fragment a warp loads feeds RB independent accumulation chains, and the
//    CTA crosses 4 barriers per call instead of 4 per row tile.
//
// Stages (rt = the CTA's row tiles, per field / output):
//   P[rt][nt]  = S[rt] C[:, nt]          warps nt < NT    (A: PK(S) smem, B: C regs)
//   V[rt][ht]  = P[rt] S[ht]^T  -> map   warps ht < QT    (A: P smem,     B: PK(S) smem)
//   R[bt][rt]  = T[bt] W[rt]^T           warps bt < NT    (A: PK(T) smem, B: W smem)
//   Y[bt][at] += R[bt][rt] T[at][rt]^T   tiles over warps (A: R smem,     B: PK(T) smem)
// and M[a][b] = w_a w_b Y[b][a] (CellKernel2D.moments, assembly.py:249-251).
// The splits' partial Y are reduced exactly as k_cta's (cluster DSMEM when the
// clusters fit one wave, else k_cta_reduce), so the results equal k_cta's
// bitwise whenever the k-chain grouping is the same (it is: two chains per
// tile, even / odd k-steps).
#pragma once
#include <cooperative_groups.h>

#include "hpg_elem.cuh"

namespace hpg {

template <int MODE, int NT, int QT, int RB, int W>
struct BigCfg {
  using TR = ModeTraits<MODE>;
  static constexpr int NP = 8 * NT, QP = 8 * QT, NK = NP / 4, QK = QP / 4;
  static constexpr int NSYN = TR::NSYN, NOUT = TR::NOUT, NIN = TR::NIN;
  static constexpr int TS = QT * NK * 32;                 // PK(S) doubles
  static constexpr int TT = NT * QK * 32;                 // PK(T) doubles
  static constexpr int SP = NSYN * RB * NT * 64;          // P fragments
  static constexpr int SV = NOUT * RB * QT * 64;          // W fragments
  static constexpr int SR = NOUT * NT * RB * 64;          // R fragments
  static constexpr int SMEM_DBL = TS + TT + SP + SV + SR;
  static constexpr int MAXS = (NOUT * NT * NT + W - 1) / W;   // Y tiles per warp
};

template <int MODE, int NT, int QT, int RB, int W>
__global__ void __launch_bounds__(32 * W, 1) k_big(ElemArgs A) {
  using CF = BigCfg<MODE, NT, QT, RB, W>;
  constexpr int NP = CF::NP, NK = CF::NK, QK = CF::QK, NSYN = CF::NSYN, NOUT = CF::NOUT, NIN = CF::NIN;
  constexpr int MAXS = CF::MAXS;
  extern __shared__ double smem[];
  double* sS = smem;
  double* sT = sS + CF::TS;
  double* sP = sT + CF::TT;                  // [f][rl][nt][64]
  double* sV = sP + CF::SP;                  // [o][rl][ht][64]
  double* sR = sV + CF::SV;                  // [o][bt][rl][64]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  const int e = blockIdx.x / A.splits, sp = blockIdx.x - e * A.splits;
  const int rt0 = sp * RB;
  for (int i = 2 * threadIdx.x; i < CF::TS; i += 2 * blockDim.x) cp_async16(sS + i, A.Sf + i);
  for (int i = 2 * threadIdx.x; i < CF::TT; i += 2 * blockDim.x) cp_async16(sT + i, A.Tf + i);
  cp_async_commit();
  pdl_wait();
  if (e >= A.N) return;
  const int cx = e / A.ncy, cy = e - cx * A.ncy;
  // warp nt: the B fragments of column block nt of every input field
  double Cf[NSYN > 0 ? NSYN : 1][NK];
  if (warp < NT) {
#pragma unroll
    for (int f = 0; f < NSYN; ++f) {
      const double* src;
      int comp;
      field_src<MODE>(A, f, src, comp);
      src += comp * A.ncomp + psi_index(A, cx, cy, 0, 0);
      const int b = 8 * warp + r;
#pragma unroll
      for (int ks = 0; ks < NK; ++ks) {
        const int a = 8 * (ks >> 1) + 2 * c + (ks & 1);
        Cf[f][ks] = (a < A.n && b < A.n) ? __ldg(src + (long long)a * A.ld + b) : 0.0;
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  // (1) P tiles: warp nt, RB row tiles x two chains
  if (warp < NT) {
#pragma unroll
    for (int f = 0; f < NSYN; ++f) {
      double P[RB][2][2];
#pragma unroll
      for (int rl = 0; rl < RB; ++rl) P[rl][0][0] = P[rl][0][1] = P[rl][1][0] = P[rl][1][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < NK; ++ks)
#pragma unroll
        for (int rl = 0; rl < RB; ++rl) dmma(P[rl][ks & 1], sS[((rt0 + rl) * NK + ks) * 32 + lane], Cf[f][ks]);
#pragma unroll
      for (int rl = 0; rl < RB; ++rl)
        *reinterpret_cast<double2*>(sP + ((f * RB + rl) * NT + warp) * 64 + 2 * lane) =
            make_double2(P[rl][0][0] + P[rl][1][0], P[rl][0][1] + P[rl][1][1]);
    }
  }
  __syncthreads();
  // (2) V tiles + pointwise map: warp ht, RB row tiles share each S fragment
  bool flag = false;
  for (int ht = warp; ht < QT; ht += W) {
    double V[RB][NSYN > 0 ? NSYN : 1][2][2];
#pragma unroll
    for (int rl = 0; rl < RB; ++rl)
#pragma unroll
      for (int f = 0; f < NSYN; ++f) V[rl][f][0][0] = V[rl][f][0][1] = V[rl][f][1][0] = V[rl][f][1][1] = 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const double b0 = sS[(ht * NK + 2 * t) * 32 + lane];
      const double b1 = sS[(ht * NK + 2 * t + 1) * 32 + lane];
#pragma unroll
      for (int f = 0; f < NSYN; ++f)
#pragma unroll
        for (int rl = 0; rl < RB; ++rl) {
          const double2 pa = *reinterpret_cast<const double2*>(sP + ((f * RB + rl) * NT + t) * 64 + 2 * lane);
          dmma(V[rl][f][0], pa.x, b0);
          dmma(V[rl][f][1], pa.y, b1);
        }
    }
#pragma unroll
    for (int rl = 0; rl < RB; ++rl) {
      double Vs[NSYN > 0 ? NSYN : 1][2];
#pragma unroll
      for (int f = 0; f < NSYN; ++f) {
        Vs[f][0] = V[rl][f][0][0] + V[rl][f][1][0];
        Vs[f][1] = V[rl][f][0][1] + V[rl][f][1][1];
      }
      double out2[NOUT][2];
      map_pair<MODE, NSYN, NOUT, ModeTraits<MODE>::NW>(A, e, QT, rt0 + rl, ht, lane, Vs, out2, flag);
#pragma unroll
      for (int o = 0; o < NOUT; ++o)
        *reinterpret_cast<double2*>(sV + ((o * RB + rl) * QT + ht) * 64 + 2 * lane) = make_double2(out2[o][0], out2[o][1]);
    }
  }
  __syncthreads();
  // (3) R tiles: warp bt, RB row tiles share each T fragment
  for (int it = warp; it < NOUT * NT; it += W) {
    const int o = it / NT, bt = it - o * NT;
    double R[RB][2][2];
#pragma unroll
    for (int rl = 0; rl < RB; ++rl) R[rl][0][0] = R[rl][0][1] = R[rl][1][0] = R[rl][1][1] = 0.0;
#pragma unroll 4
    for (int t = 0; t < QT; ++t) {
      const double a0 = sT[(bt * QK + 2 * t) * 32 + lane];
      const double a1 = sT[(bt * QK + 2 * t + 1) * 32 + lane];
#pragma unroll
      for (int rl = 0; rl < RB; ++rl) {
        const double2 vb = *reinterpret_cast<const double2*>(sV + ((o * RB + rl) * QT + t) * 64 + 2 * lane);
        dmma(R[rl][0], a0, vb.x);
        dmma(R[rl][1], a1, vb.y);
      }
    }
#pragma unroll
    for (int rl = 0; rl < RB; ++rl)
      *reinterpret_cast<double2*>(sR + ((o * NT + bt) * RB + rl) * 64 + 2 * lane) =
          make_double2(R[rl][0][0] + R[rl][1][0], R[rl][0][1] + R[rl][1][1]);
  }
  __syncthreads();
  // (4) Y accumulation (tiles statically owned by warps, k-steps = RB x 2)
  const int ny = NOUT * NT * NT;
  double Y[MAXS][2];
#pragma unroll
  for (int s = 0; s < MAXS; ++s) {
    Y[s][0] = Y[s][1] = 0.0;
    const int it = warp + W * s;
    if (it < ny) {
      const int o = it / (NT * NT), rem = it - o * NT * NT;
      const int bt = rem / NT, at = rem - bt * NT;
#pragma unroll
      for (int rl = 0; rl < RB; ++rl) {
        const double2 ra = *reinterpret_cast<const double2*>(sR + ((o * NT + bt) * RB + rl) * 64 + 2 * lane);
        dmma(Y[s], ra.x, sT[(at * QK + 2 * (rt0 + rl)) * 32 + lane]);
        dmma(Y[s], ra.y, sT[(at * QK + 2 * (rt0 + rl) + 1) * 32 + lane]);
      }
    }
  }
  if constexpr (MODE == M_OBST_RES) {
    if (__any_sync(0xffffffffu, flag) && lane == 0) atomicOr(A.flag, 1);
  }
  if (A.cluster_red) {
    // the A.splits CTAs of cell e are one cluster: partial Y through DSMEM,
    // summed in split order (k_cta's reduction)
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __syncthreads();
    double* sY = smem;                     // [NOUT][NP][NP] (tables are dead)
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
      const int it = warp + W * s;
      if (it < ny) {
        const int o = it / (NT * NT), rem = it - o * NT * NT;
        const int bt = rem / NT, at = rem - bt * NT;
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
    cl.sync();
    return;
  }
#pragma unroll
  for (int s = 0; s < MAXS; ++s) {
    const int it = warp + W * s;
    if (it < ny) {
      const int o = it / (NT * NT), rem = it - o * NT * NT;
      const int bt = rem / NT, at = rem - bt * NT;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int a = 8 * at + 2 * c + j, b = 8 * bt + r;
        if (A.splits == 1) {
          if (a < A.n && b < A.n) write_moment<MODE>(A, e, cx, cy, o, a, b, Y[s][j]);
        } else {
          A.partial[(((long long)e * A.splits + sp) * NOUT + o) * NP * NP + a * NP + b] = Y[s][j];
        }
      }
    }
  }
}

}  // namespace hpg
