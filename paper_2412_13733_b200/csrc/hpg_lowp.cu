// Single-pass LVPP residual (+ Jacobian apply) for low-degree obstacle meshes
// (config 4: 256x256 cells, p = 2/4/6): ONE kernel per call, one thread per
// cell, no intermediate HBM buffers.
//
// Per cell (cx, cy), in order:
//  (1) psi side (as k_small): synthesis of psi (and x) at the Q x Q points,
//      E = exp(min(-V, 700)) (+ overflow flag), analysis -> moments M (and
//      the Jacobian action MY); y = w MY is stored at once.
//  (2) own U side (generated straight-line code, hpg_usmall_gen.cuh) with
//      LAZY global-memory operands: B^T u finishes
//      b_psi = (phi_mom - B^T u) - w M (proximal.py:123 order, one store);
//      bubble x bubble b_u dofs are stored directly; contributions to the
//      hats this cell owns (its left x-hat and bottom y-hat lines) are kept.
//  (3) the hat contributions the neighbours make to those owned dofs are
//      recomputed here from the neighbours' data (left: local row j = 1,
//      bottom: column k = 1, corner: (1, 1)).  The generated code is the
//      same; the output filter is a compile-time condition per (j, k), so the
//      dead expressions and their loads are eliminated.
//  (4) owned hat dofs: b_u = alpha f + (own + left + bottom + corner), fixed
//      order (deterministic, no atomics, no edge buffer, no gather kernel).
// k_lowt (p <= 3, the default there) is the same computation tiled: one CTA
// per 8 x 16 block of cells stages the block's region in shared memory with
// one round of cp.async copies and exchanges the hat lines between
// neighbouring cells in shared memory (a halo warp covers the block's left /
// bottom neighbours), instead of each thread re-deriving its neighbours'
// contributions from global memory.
// References: assembly.py:81-116,470-477,541-548 (B, A, exp_moments),
// spaces.py:25-57 (U numbering, R map), proximal.py:112-126 (residual),
// assembly.py:559-567 (apply_D).
#include "hpg_launch.cuh"
#include "hpg_common.cuh"
#include "hpg_small.cuh"
#include "hpg_usmall_gen.cuh"

#include <cstdlib>

namespace hpg {
namespace {

// U tile of cell (cx, cy) read on demand: C[i*M + l] = u(ix(i), iy(l)), 0 on
// the boundary (spaces.py:36-43).
template <int P>
struct ULazy {
  static constexpr int M = P + 1;
  const double* u;
  int cx, cy, ncx, ncy, niy;
  __device__ __forceinline__ double operator[](int k) const {
    const int i = k / M, l = k - (k / M) * M;
    const int ix = u_local_1d(cx, i, ncx, P), iy = u_local_1d(cy, l, ncy, P);
    return (ix < 0 || iy < 0) ? 0.0 : __ldg(u + (long long)ix * niy + iy);
  }
};

// raw psi_prev - psi tile of a cell: G[i*N + l]
template <int N>
struct GLazy {
  const double* psi_prev;
  const double* psi;
  long long base, ld;
  __device__ __forceinline__ double operator[](int k) const {
    const int i = k / N, l = k - (k / N) * N;
    const long long g = base + (long long)i * ld + l;
    return __ldg(psi_prev + g) - __ldg(psi + g);
  }
};

constexpr int LOWP_TH = 64;

// operand read through a callable (register arrays with constant indices)
template <class F>
struct FnAcc {
  F f;
  __device__ __forceinline__ double operator[](int k) const { return f(k); }
};
template <class F>
__device__ __forceinline__ FnAcc<F> fn_acc(F f) { return FnAcc<F>{f}; }

// thread-private shared-memory slice: T[k] = s[k * LOWP_TH]
struct Slice {
  const double* s;
  __device__ __forceinline__ double operator[](int k) const { return s[k * LOWP_TH]; }
};

template <int P, int Q, bool APPLY>
// p <= 4: <= 146 registers keeps the 65,536-cell mesh in one wave; p >= 5
// runs unconstrained (capping it spills the U-side operands: measured slower)
#ifndef HPG_LOWP_MINB_SMALL
#define HPG_LOWP_MINB_SMALL 7
#endif
__global__ void __launch_bounds__(LOWP_TH, P <= 4 ? HPG_LOWP_MINB_SMALL : 1) k_lowp(ElemArgs A, const SmallTables tb) {
  pdl_wait();
  constexpr int N = P - 1, M = P + 1, NIN = APPLY ? 2 : 1;
  constexpr int SL = NIN * N * N > M * M ? NIN * N * N : M * M;
  // thread-private slices: psi (and x) tiles in (1), then the U tile in (2)
  __shared__ double sbuf[SL][LOWP_TH];
  double (*sC)[N * N][LOWP_TH] = reinterpret_cast<double (*)[N * N][LOWP_TH]>(&sbuf[0][0]);
  const int tid = threadIdx.x;
  const int e = blockIdx.x * LOWP_TH + tid;
  if (e >= A.N) return;
  const int cx = e / A.ncy, cy = e - cx * A.ncy;
  const long long base = psi_index(A, cx, cy, 0, 0);
  // ---- (1) psi side ------------------------------------------------------
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int b = 0; b < N; ++b) {
      sC[0][a * N + b][tid] = __ldg(A.in0 + base + (long long)a * A.ld + b);
      if (APPLY) sC[NIN - 1][a * N + b][tid] = __ldg(A.in1 + base + (long long)a * A.ld + b);
    }
  // low degree: the U-side operands are loaded now, so their latency hides
  // behind the psi-side arithmetic (the kernel is otherwise a chain of
  // dependent round trips at p <= 4)
  constexpr bool PREF = P <= 3;
  double uC[PREF ? M * M : 1], pp[PREF ? N * N : 1], ph[PREF ? N * N : 1];
  if constexpr (PREF) {
    const ULazy<P> Cl{A.u, cx, cy, A.ncx, A.ncy, A.niy};
#pragma unroll
    for (int k = 0; k < M * M; ++k) uC[k] = Cl[k];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) {
        pp[a * N + b] = __ldg(A.psi_prev + base + (long long)a * A.ld + b);
        ph[a * N + b] = __ldg(A.phi_mom + base + (long long)a * A.ld + b);
      }
  }
  double Mm[N][N];
  double MY[APPLY ? N : 1][APPLY ? N : 1];
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int b = 0; b < N; ++b) {
      Mm[a][b] = 0.0;
      if (APPLY) MY[a][b] = 0.0;
    }
  bool flag = false;
  if constexpr (N == 1) {
    // p = 2: the psi tile is ONE Legendre coefficient and P_0 = 1 at every
    // point, so the synthesized field is that coefficient everywhere: one
    // clamped exp per cell instead of Q^2, and M = E (sum_g T_0g)^2 (the
    // reference's T E T^T regrouped; equal to rounding)
    double sT = 0.0;
#pragma unroll
    for (int h = 0; h < Q; ++h) sT += tb.T[h];
    const double v = tb.S[0] * sC[0][0][tid];        // S[g][0] = P_0 = 1
    const double E = clamped_exp_neg(v, flag);
    Mm[0][0] = (E * sT) * sT;
    if (APPLY) MY[0][0] = ((E * (tb.S[0] * sC[NIN - 1][0][tid])) * sT) * sT;
  } else {
#pragma unroll 1
  for (int g = 0; g < Q; ++g) {
    double Pv[N], PX[APPLY ? N : 1];
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double s = 0.0, sx = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        s = fma(tb.S[g * N + a], sC[0][a * N + b][tid], s);
        if (APPLY) sx = fma(tb.S[g * N + a], sC[NIN - 1][a * N + b][tid], sx);
      }
      Pv[b] = s;
      if (APPLY) PX[b] = sx;
    }
    double ev[N], exv[APPLY ? N : 1];
#pragma unroll
    for (int b = 0; b < N; ++b) {
      ev[b] = 0.0;
      if (APPLY) exv[b] = 0.0;
    }
#pragma unroll
    for (int h = 0; h < Q; ++h) {
      double v = 0.0, vx = 0.0;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        v = fma(Pv[b], tb.S[h * N + b], v);
        if (APPLY) vx = fma(PX[b], tb.S[h * N + b], vx);
      }
      const double E = clamped_exp_neg(v, flag);
      const double Ex = E * vx;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        ev[b] = fma(E, tb.T[b * Q + h], ev[b]);
        if (APPLY) exv[b] = fma(Ex, tb.T[b * Q + h], exv[b]);
      }
    }
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const double t = tb.T[a * Q + g];
#pragma unroll
      for (int b = 0; b < N; ++b) {
        Mm[a][b] = fma(t, ev[b], Mm[a][b]);
        if (APPLY) MY[a][b] = fma(t, exv[b], MY[a][b]);
      }
    }
  }
  }
  if (flag) atomicOr(A.flag, 1);
  const double hx = A.hx[cx], hy = A.hy[cy];
  if (APPLY) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b)
        A.wc_out[base + (long long)a * A.ld + b] = ((hx * kInvOdd[a]) * MY[a][b]) * (hy * kInvOdd[b]);
  }
  // ---- (2) own U side ----------------------------------------------------
  const int nhx = A.ncx - 1, nhy = A.ncy - 1;
  const long long bx = nhx + (long long)cx * (P - 1) - 2;    // + j: interior x index of bubble j
  const long long by = nhy + (long long)cy * (P - 1) - 2;
  const double alpha = A.alpha;
  double H00 = 0.0, H0k[M], Hj0[M];        // owned hat lines (index 2..M-1 used)
#pragma unroll
  for (int k = 0; k < M; ++k) H0k[k] = Hj0[k] = 0.0;
  {
    auto ou = [&](int j, int k, double r) {
      if (j >= 2 && k >= 2) {
        const long long g = (bx + j) * A.niy + (by + k);
        A.b_u[g] = alpha * __ldg(A.f_load + g) + r;
      } else if (j == 0 && k == 0) {
        H00 = r;
      } else if (j == 0 && k >= 2) {
        H0k[k] = r;
      } else if (k == 0 && j >= 2) {
        Hj0[j] = r;
      }
      // j == 1 or k == 1: owned by the right / top neighbour (its step (3))
    };
    auto ob = [&](int, int a, int b, double btu) {
      const long long g = base + (long long)a * A.ld + b;
      const double val = ((hx * kInvOdd[a]) * Mm[a][b]) * (hy * kInvOdd[b]);
      double phm;
      if constexpr (PREF) phm = ph[a * N + b];
      else phm = __ldg(A.phi_mom + g);
      A.out[g] = (phm - btu) - val;
    };
    if constexpr (PREF) {
      const auto Cu = fn_acc([&](int k) { return uC[k]; });
      const auto Gp = fn_acc([&](int k) { return pp[k] - sC[0][k][tid]; });
      USmall<P, false>::run(Cu, Gp, 1, hx, hy, alpha, ou, ob);
    } else {
      // the own U tile is used by every output: stage it once in this
      // thread's slice (the psi-side tiles are dead); psi_prev - psi lazily
      {
        const ULazy<P> Cl{A.u, cx, cy, A.ncx, A.ncy, A.niy};
#pragma unroll
        for (int k = 0; k < M * M; ++k) sbuf[k][tid] = Cl[k];
      }
      const Slice Cu{&sbuf[0][tid]};
      const GLazy<N> Gp{A.psi_prev, A.in0, base, A.ld};
      USmall<P, false>::run(Cu, Gp, 1, hx, hy, alpha, ou, ob);
    }
  }
  // ---- (3) neighbours' contributions to the owned hats -------------------
  auto nob = [](int, int, int, double) {};
  if (cx >= 1) {
    const ULazy<P> Cu{A.u, cx - 1, cy, A.ncx, A.ncy, A.niy};
    const GLazy<N> Gp{A.psi_prev, A.in0, psi_index(A, cx - 1, cy, 0, 0), A.ld};
    auto ou = [&](int j, int k, double r) {
      if (j == 1 && k == 0) H00 += r;
      else if (j == 1 && k >= 2) H0k[k] += r;
    };
    USmall<P, false>::run(Cu, Gp, 1, A.hx[cx - 1], hy, alpha, ou, nob);
  }
  if (cy >= 1) {
    const ULazy<P> Cu{A.u, cx, cy - 1, A.ncx, A.ncy, A.niy};
    const GLazy<N> Gp{A.psi_prev, A.in0, psi_index(A, cx, cy - 1, 0, 0), A.ld};
    auto ou = [&](int j, int k, double r) {
      if (k == 1 && j == 0) H00 += r;
      else if (k == 1 && j >= 2) Hj0[j] += r;
    };
    USmall<P, false>::run(Cu, Gp, 1, hx, A.hy[cy - 1], alpha, ou, nob);
  }
  if (cx >= 1 && cy >= 1) {
    const ULazy<P> Cu{A.u, cx - 1, cy - 1, A.ncx, A.ncy, A.niy};
    const GLazy<N> Gp{A.psi_prev, A.in0, psi_index(A, cx - 1, cy - 1, 0, 0), A.ld};
    auto ou = [&](int j, int k, double r) {
      if (j == 1 && k == 1) H00 += r;
    };
    USmall<P, false>::run(Cu, Gp, 1, A.hx[cx - 1], A.hy[cy - 1], alpha, ou, nob);
  }
  // ---- (4) owned hat dofs ------------------------------------------------
  if (cx >= 1) {
    const long long ix = cx - 1;
    if (cy >= 1) {
      const long long g = ix * A.niy + (cy - 1);
      A.b_u[g] = alpha * __ldg(A.f_load + g) + H00;
    }
#pragma unroll
    for (int k = 2; k < M; ++k) {
      const long long g = ix * A.niy + (by + k);
      A.b_u[g] = alpha * __ldg(A.f_load + g) + H0k[k];
    }
  }
  if (cy >= 1) {
    const long long iy = cy - 1;
#pragma unroll
    for (int j = 2; j < M; ++j) {
      const long long g = (bx + j) * A.niy + iy;
      A.b_u[g] = alpha * __ldg(A.f_load + g) + Hj0[j];
    }
  }
}

// ---------------------------------------------------------------------------
// Tiled variant (low degree): one CTA per TX x TY block of cells, one thread
// per cell plus one halo warp.
//  * Staging: everything the block reads -- the U nodes and the load vector f
//    over the (TX+1) x (TY+1) cell region (the block and its left / bottom
//    halo: hat rows/columns and bubble blocks), psi and psi_prev over the
//    region, the direction x and the data moments of the block, the cell
//    sizes -- is copied once by 8-byte cp.async (all in flight together, zero
//    fill outside the domain): ONE global round trip per CTA, coalesced.
//  * Hat exchange in shared memory: every cell's U side produces its whole
//    j = 1 (right hat) and k = 1 (top hat) lines; the halo warp produces them
//    for the halo cells (left column, bottom row, corner).  After one
//    barrier each cell finishes the hats it owns from its left / bottom /
//    corner neighbours' lines: the U side runs once per cell (plus the halo)
//    instead of four times.
// Arithmetic, operand order and summation order are those of k_lowp (same
// generated U-side code): own + left(1,.) + bottom(.,1) + corner(1,1).
template <int P, int TX, int TY>
struct LowtCfg {
  static constexpr int N = P - 1, M = P + 1;
  static constexpr int RX = TX + 1, RY = TY + 1;            // region incl. halo
  static constexpr int XH = TX + 2, YH = TY + 2;            // staged hat rows / cols
  static constexpr int UR = XH + RX * (P - 1), UC = YH + RY * (P - 1);
  static constexpr int LDP = RY * N;                        // psi / psi_prev region row stride
  static constexpr int NPSI = RX * N * LDP;
  static constexpr int LDX = TY * N;                        // own-cell x / phi_mom
  static constexpr int NX = TX * N * LDX;
  static constexpr int NU = UR * UC;
  static constexpr int NLINE = RX * RY * M;                 // j = 1 / k = 1 lines per region cell
  static_assert(TX + TY + 1 <= 32, "one halo warp");
};


// U tile of the region cell (rx, ry) (rx = cx - cx0 + 1): C[i*M + l]
template <int P, int TX, int TY>
struct UTileS {
  using C = LowtCfg<P, TX, TY>;
  const double* s;
  int rx, ry;
  __device__ __forceinline__ int row(int i) const {
    return i == 0 ? rx : (i == 1 ? rx + 1 : C::XH + rx * (P - 1) + (i - 2));
  }
  __device__ __forceinline__ int col(int l) const {
    return l == 0 ? ry : (l == 1 ? ry + 1 : C::YH + ry * (P - 1) + (l - 2));
  }
  __device__ __forceinline__ double operator[](int k) const {
    const int i = k / C::M, l = k - (k / C::M) * C::M;
    return s[row(i) * C::UC + col(l)];
  }
};

// psi_prev - psi tile of the region cell (rx, ry): G[a*N + b]
template <int P, int TX, int TY>
struct GTileS {
  using C = LowtCfg<P, TX, TY>;
  const double* pp;
  const double* ps;
  int off;
  __device__ __forceinline__ double operator[](int k) const {
    const int a = k / C::N, b = k - (k / C::N) * C::N;
    const int g = off + a * C::LDP + b;
    return pp[g] - ps[g];
  }
};

// Shared-memory stage of one tile (pointers into one of the two buffers).
template <int P, int TX, int TY, bool APPLY>
struct LowtBuf {
  using CF = LowtCfg<P, TX, TY>;
  static constexpr int N = CF::N;
  static constexpr int DOUBLES = 2 * CF::NPSI + (APPLY ? 2 : 1) * CF::NX + 2 * CF::NU + CF::RX + CF::RY +
                                 (CF::RX + CF::RY) * N + CF::UR + CF::UC;
  double *sPsi, *sPP, *sPhi, *sX, *sU, *sF, *sHx, *sHy;
  long long *sPRow, *sPCol, *sURow, *sUCol;
  __device__ __forceinline__ explicit LowtBuf(double* s) {
    sPsi = s;
    sPP = sPsi + CF::NPSI;
    sPhi = sPP + CF::NPSI;
    sX = sPhi + CF::NX;
    sU = sX + (APPLY ? CF::NX : 0);
    sF = sU + CF::NU;
    sHx = sF + CF::NU;
    sHy = sHx + CF::RX;
    sPRow = reinterpret_cast<long long*>(sHy + CF::RY);
    sPCol = sPRow + CF::RX * N;
    sURow = sPCol + CF::RY * N;
    sUCol = sURow + CF::UR;
  }
};

template <int P, int TX, int TY, bool APPLY>
__host__ __device__ constexpr int lowt_smem_doubles() {
  using C = LowtCfg<P, TX, TY>;
  return LowtBuf<P, TX, TY, APPLY>::DOUBLES + 2 * C::NLINE;
}

// (a) per-row / per-column global offsets of tile (cx0, cy0)'s region (-1:
// outside the domain), so (b)'s copies are a table lookup each
template <int P, int TX, int TY, bool APPLY, int NTH>
__device__ __forceinline__ void lowt_tables(const ElemArgs& A, int cx0, int cy0, const LowtBuf<P, TX, TY, APPLY>& B,
                                            int tid) {
  using CF = LowtCfg<P, TX, TY>;
  constexpr int N = CF::N;
  const int nhx = A.ncx - 1, nhy = A.ncy - 1;
  long long* sPRow = B.sPRow;
  long long* sPCol = B.sPCol;
  long long* sURow = B.sURow;
  long long* sUCol = B.sUCol;
  // (a) per-row / per-column global offsets of the region (-1: outside the
  // domain), so (b)'s copies are a table lookup each
  {
    const long long prows = (long long)A.ncx * N, pcols = (long long)A.ncy * N;
    for (int k = tid; k < CF::RX * N + CF::RY * N + CF::UR + CF::UC; k += NTH) {
      long long o;
      if (k < CF::RX * N) {
        const long long gr = (long long)(cx0 - 1) * N + k;
        o = gr >= 0 && gr < prows ? gr * A.ld : -1;
        sPRow[k] = o;
      } else if (k < (CF::RX + CF::RY) * N) {
        const long long gc = (long long)(cy0 - 1) * N + (k - CF::RX * N);
        o = gc >= 0 && gc < pcols ? gc : -1;
        sPCol[k - CF::RX * N] = o;
      } else if (k < (CF::RX + CF::RY) * N + CF::UR) {
        const int r = k - (CF::RX + CF::RY) * N;
        long long ix;
        bool v;
        if (r < CF::XH) {
          ix = cx0 - 2 + r;
          v = ix >= 0 && ix < nhx;
        } else {
          ix = nhx + (long long)(cx0 - 1) * (P - 1) + (r - CF::XH);
          v = ix >= nhx && ix < nhx + (long long)A.ncx * (P - 1);
        }
        sURow[r] = v ? ix * A.niy : -1;
      } else {
        const int c = k - (CF::RX + CF::RY) * N - CF::UR;
        long long iy;
        bool v;
        if (c < CF::YH) {
          iy = cy0 - 2 + c;
          v = iy >= 0 && iy < nhy;
        } else {
          iy = nhy + (long long)(cy0 - 1) * (P - 1) + (c - CF::YH);
          v = iy >= nhy && iy < nhy + (long long)A.ncy * (P - 1);
        }
        sUCol[c] = v ? iy : -1;
      }
    }
  }
}

// (b) 8-byte cp.async copies of the tile's region, zero fill outside the domain
template <int P, int TX, int TY, bool APPLY, int NTH>
__device__ __forceinline__ void lowt_stage(const ElemArgs& A, int cx0, int cy0, const LowtBuf<P, TX, TY, APPLY>& B,
                                           int tid) {
  using CF = LowtCfg<P, TX, TY>;
  constexpr int N = CF::N;
  double* sPsi = B.sPsi;
  double* sPP = B.sPP;
  double* sPhi = B.sPhi;
  double* sX = B.sX;
  double* sU = B.sU;
  double* sF = B.sF;
  double* sHx = B.sHx;
  double* sHy = B.sHy;
  const long long* sPRow = B.sPRow;
  const long long* sPCol = B.sPCol;
  const long long* sURow = B.sURow;
  const long long* sUCol = B.sUCol;
  // (b) 8-byte cp.async copies, zero fill outside the domain
  {
    for (int k = tid; k < CF::NPSI; k += NTH) {
      const int r = k / CF::LDP, c = k - (k / CF::LDP) * CF::LDP;
      const long long ro = sPRow[r], co = sPCol[c];
      const bool v = (ro | co) >= 0;
      const long long g = v ? ro + co : 0;
      cp_async8z(sPsi + k, A.in0 + g, v);
      cp_async8z(sPP + k, A.psi_prev + g, v);
    }
    for (int k = tid; k < CF::NX; k += NTH) {
      const int r = k / CF::LDX, c = k - (k / CF::LDX) * CF::LDX;
      const long long ro = sPRow[r + N], co = sPCol[c + N];
      const bool v = (ro | co) >= 0;
      const long long g = v ? ro + co : 0;
      cp_async8z(sPhi + k, A.phi_mom + g, v);
      if (APPLY) cp_async8z(sX + k, A.in1 + g, v);
    }
    for (int k = tid; k < CF::NU; k += NTH) {
      const int r = k / CF::UC, c = k - (k / CF::UC) * CF::UC;
      const long long ro = sURow[r], co = sUCol[c];
      const bool v = (ro | co) >= 0;
      const long long g = v ? ro + co : 0;
      cp_async8z(sU + k, A.u + g, v);
      cp_async8z(sF + k, A.f_load + g, v);
    }
    for (int k = tid; k < CF::RX + CF::RY; k += NTH) {
      if (k < CF::RX) {
        const int cx = cx0 - 1 + k;
        cp_async8z(sHx + k, A.hx + (cx >= 0 && cx < A.ncx ? cx : 0), cx >= 0 && cx < A.ncx);
      } else {
        const int cy = cy0 - 1 + (k - CF::RX);
        cp_async8z(sHy + (k - CF::RX), A.hy + (cy >= 0 && cy < A.ncy ? cy : 0), cy >= 0 && cy < A.ncy);
      }
    }
  }
}

// The tile's cells from its staged region: (1)-(4) below.  Every thread of
// the CTA calls it (one internal barrier: the hat-line exchange).
template <int P, int Q, bool APPLY, int TX, int TY>
__device__ __forceinline__ void lowt_tile(const ElemArgs& A, const SmallTables& tb, int cx0, int cy0,
                                          const LowtBuf<P, TX, TY, APPLY>& B, double* sR, double* sTl, int tid) {
  using CF = LowtCfg<P, TX, TY>;
  constexpr int N = CF::N, M = CF::M, NT = TX * TY;
  const double* sPsi = B.sPsi;
  const double* sPP = B.sPP;
  const double* sPhi = B.sPhi;
  const double* sX = B.sX;
  const double* sU = B.sU;
  const double* sF = B.sF;
  const double* sHx = B.sHx;
  const double* sHy = B.sHy;
  const int nhx = A.ncx - 1, nhy = A.ncy - 1;
  const double alpha = A.alpha;
  auto nob = [](int, int, int, double) {};
  if (tid >= NT) {
    // ---- halo warp: the j = 1 line of the left column, the k = 1 line of
    // the bottom row, (1, 1) of the corner (their owners' neighbour terms) --
    const int h = tid - NT;
    if (h < TY) {
      const int cx = cx0 - 1, cy = cy0 + h, rx = 0, ry = h + 1;
      if (cx >= 0 && cy < A.ncy) {
        double* line = sR + (rx * CF::RY + ry) * M;
        auto ou = [&](int j, int k, double r) {
          if (j == 1) line[k] = r;
        };
        USmall<P, false>::run(UTileS<P, TX, TY>{sU, rx, ry}, GTileS<P, TX, TY>{sPP, sPsi, ry * N}, 1, sHx[rx],
                              sHy[ry], alpha, ou, nob);
      }
    } else if (h < TY + TX) {
      const int cx = cx0 + (h - TY), cy = cy0 - 1, rx = h - TY + 1, ry = 0;
      if (cy >= 0 && cx < A.ncx) {
        double* line = sTl + (rx * CF::RY + ry) * M;
        double* r1 = sR + (rx * CF::RY + ry) * M + 1;
        auto ou = [&](int j, int k, double r) {
          if (k == 1) line[j] = r;
          if (j == 1 && k == 1) *r1 = r;
        };
        USmall<P, false>::run(UTileS<P, TX, TY>{sU, rx, ry}, GTileS<P, TX, TY>{sPP, sPsi, rx * N * CF::LDP}, 1,
                              sHx[rx], sHy[ry], alpha, ou, nob);
      }
    } else if (h == TY + TX) {
      if (cx0 >= 1 && cy0 >= 1) {
        double* r1 = sR + 1;
        auto ou = [&](int j, int k, double r) {
          if (j == 1 && k == 1) *r1 = r;
        };
        USmall<P, false>::run(UTileS<P, TX, TY>{sU, 0, 0}, GTileS<P, TX, TY>{sPP, sPsi, 0}, 1, sHx[0], sHy[0],
                              alpha, ou, nob);
      }
    }
    __syncthreads();
    return;
  }
  const int ti = tid / TY, tj = tid - (tid / TY) * TY;
  const int cx = cx0 + ti, cy = cy0 + tj;
  const bool live = cx < A.ncx && cy < A.ncy;
  const int rx = ti + 1, ry = tj + 1;                      // region coordinates
  const int poff = rx * N * CF::LDP + ry * N;              // own psi tile in the region
  const int xoff = ti * N * CF::LDX + tj * N;              // own x / phi tile
  const long long base = live ? psi_index(A, cx, cy, 0, 0) : 0;
  const double hx = sHx[rx], hy = sHy[ry];
  double H00 = 0.0, H0k[M], Hj0[M];
#pragma unroll
  for (int k = 0; k < M; ++k) H0k[k] = Hj0[k] = 0.0;
  if (live) {
    // ---- (1) psi side (k_lowp order) -------------------------------------
    double Mm[N][N];
    double MY[APPLY ? N : 1][APPLY ? N : 1];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) {
        Mm[a][b] = 0.0;
        if (APPLY) MY[a][b] = 0.0;
      }
    bool flag = false;
    if constexpr (N == 1) {
      double sT = 0.0;
#pragma unroll
      for (int h = 0; h < Q; ++h) sT += tb.T[h];
      const double v = tb.S[0] * sPsi[poff];
      const double E = clamped_exp_neg(v, flag);
      Mm[0][0] = (E * sT) * sT;
      if (APPLY) MY[0][0] = ((E * (tb.S[0] * sX[xoff])) * sT) * sT;
    } else {
#pragma unroll 1
      for (int g = 0; g < Q; ++g) {
        double Pv[N], PX[APPLY ? N : 1];
#pragma unroll
        for (int b = 0; b < N; ++b) {
          double s = 0.0, sx = 0.0;
#pragma unroll
          for (int a = 0; a < N; ++a) {
            s = fma(tb.S[g * N + a], sPsi[poff + a * CF::LDP + b], s);
            if (APPLY) sx = fma(tb.S[g * N + a], sX[xoff + a * CF::LDX + b], sx);
          }
          Pv[b] = s;
          if (APPLY) PX[b] = sx;
        }
        double ev[N], exv[APPLY ? N : 1];
#pragma unroll
        for (int b = 0; b < N; ++b) {
          ev[b] = 0.0;
          if (APPLY) exv[b] = 0.0;
        }
#pragma unroll
        for (int h = 0; h < Q; ++h) {
          double v = 0.0, vx = 0.0;
#pragma unroll
          for (int b = 0; b < N; ++b) {
            v = fma(Pv[b], tb.S[h * N + b], v);
            if (APPLY) vx = fma(PX[b], tb.S[h * N + b], vx);
          }
          const double E = clamped_exp_neg(v, flag);
          const double Ex = E * vx;
#pragma unroll
          for (int b = 0; b < N; ++b) {
            ev[b] = fma(E, tb.T[b * Q + h], ev[b]);
            if (APPLY) exv[b] = fma(Ex, tb.T[b * Q + h], exv[b]);
          }
        }
#pragma unroll
        for (int a = 0; a < N; ++a) {
          const double t = tb.T[a * Q + g];
#pragma unroll
          for (int b = 0; b < N; ++b) {
            Mm[a][b] = fma(t, ev[b], Mm[a][b]);
            if (APPLY) MY[a][b] = fma(t, exv[b], MY[a][b]);
          }
        }
      }
    }
    if (flag) atomicOr(A.flag, 1);
    if (APPLY) {
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b)
          A.wc_out[base + (long long)a * A.ld + b] = ((hx * kInvOdd[a]) * MY[a][b]) * (hy * kInvOdd[b]);
    }
    // ---- (2) own U side: bubbles stored, owned hats kept, the j = 1 / k = 1
    // lines handed to the right / top neighbours through shared memory ------
    const int fr = CF::XH + rx * (P - 1) - 2, fc = CF::YH + ry * (P - 1) - 2;   // + j, + k: staged f row / col
    const long long bx = nhx + (long long)cx * (P - 1) - 2;
    const long long by = nhy + (long long)cy * (P - 1) - 2;
    double* lineR = sR + (rx * CF::RY + ry) * M;
    double* lineT = sTl + (rx * CF::RY + ry) * M;
    auto ou = [&](int j, int k, double r) {
      if (j >= 2 && k >= 2) {
        A.b_u[(bx + j) * A.niy + (by + k)] = alpha * sF[(fr + j) * CF::UC + fc + k] + r;
      } else if (j == 0 && k == 0) {
        H00 = r;
      } else if (j == 0 && k >= 2) {
        H0k[k] = r;
      } else if (k == 0 && j >= 2) {
        Hj0[j] = r;
      }
      if (j == 1) lineR[k] = r;
      if (k == 1) lineT[j] = r;
    };
    auto ob = [&](int, int a, int b, double btu) {
      const double val = ((hx * kInvOdd[a]) * Mm[a][b]) * (hy * kInvOdd[b]);
      A.out[base + (long long)a * A.ld + b] = (sPhi[xoff + a * CF::LDX + b] - btu) - val;
    };
    USmall<P, false>::run(UTileS<P, TX, TY>{sU, rx, ry}, GTileS<P, TX, TY>{sPP, sPsi, poff}, 1, hx, hy, alpha, ou,
                          ob);
  }
  __syncthreads();
  if (!live) return;
  // ---- (3) neighbours' lines -> owned hats (k_lowp summation order) -------
  if (cx >= 1) {
    const double* lineL = sR + ((rx - 1) * CF::RY + ry) * M;
    H00 += lineL[0];
#pragma unroll
    for (int k = 2; k < M; ++k) H0k[k] += lineL[k];
  }
  if (cy >= 1) {
    const double* lineB = sTl + (rx * CF::RY + ry - 1) * M;
    H00 += lineB[0];
#pragma unroll
    for (int j = 2; j < M; ++j) Hj0[j] += lineB[j];
  }
  if (cx >= 1 && cy >= 1) H00 += sR[((rx - 1) * CF::RY + ry - 1) * M + 1];
  // ---- (4) owned hat dofs ------------------------------------------------
  const int fr = CF::XH + rx * (P - 1) - 2, fc = CF::YH + ry * (P - 1) - 2;
  const long long bx = nhx + (long long)cx * (P - 1) - 2;
  const long long by = nhy + (long long)cy * (P - 1) - 2;
  if (cx >= 1) {
    const long long ix = cx - 1;               // staged hat row rx (= cx - cx0 + 1)
    if (cy >= 1) A.b_u[ix * A.niy + (cy - 1)] = alpha * sF[rx * CF::UC + ry] + H00;
#pragma unroll
    for (int k = 2; k < M; ++k) A.b_u[ix * A.niy + (by + k)] = alpha * sF[rx * CF::UC + fc + k] + H0k[k];
  }
  if (cy >= 1) {
    const long long iy = cy - 1;
#pragma unroll
    for (int j = 2; j < M; ++j) A.b_u[(bx + j) * A.niy + iy] = alpha * sF[(fr + j) * CF::UC + ry] + Hj0[j];
  }
}

// One CTA per tile: stage, then compute.  (A persistent variant walking
// several tiles per CTA with double-buffered stages was measured slower at
// every CTAs/SM setting: the per-tile work is latency-bound, so fewer
// resident tiles cost more than the copy overlap gains.)
template <int P, int Q, bool APPLY, int TX, int TY>
__global__ void __launch_bounds__(TX * TY + 32) k_lowt(ElemArgs A, const SmallTables tb, int nty) {
  using BUF = LowtBuf<P, TX, TY, APPLY>;
  constexpr int NTH = TX * TY + 32;
  extern __shared__ double smem[];
  const BUF B(smem);
  double* sR = smem + BUF::DOUBLES;                     // [region cell][k]: U-side output (1, k)
  double* sTl = sR + LowtCfg<P, TX, TY>::NLINE;         // [region cell][j]: U-side output (j, 1)
  const int tid = threadIdx.x;
  const int cx0 = (blockIdx.x / nty) * TX, cy0 = (blockIdx.x % nty) * TY;
  pdl_wait();
  lowt_tables<P, TX, TY, APPLY, NTH>(A, cx0, cy0, B, tid);
  __syncthreads();
  lowt_stage<P, TX, TY, APPLY, NTH>(A, cx0, cy0, B, tid);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  lowt_tile<P, Q, APPLY, TX, TY>(A, tb, cx0, cy0, B, sR, sTl, tid);
}

// Tile shape per degree; the tiled kernel is the default where it measured
// faster than k_lowp (p <= 3: config 4 p=2 8.13 -> 6.61 us per call; at
// p >= 4 the register and shared-memory footprint costs more occupancy than
// the staging saves: p=4 25.4 -> 34 us, p=6 77 -> 109 us).  Shapes 4x16,
// 2x16 and 4x8 measured within 3 % of 8x16 (4x8: +12 %).
template <int P>
struct LowtTile {
  static constexpr int TX = 8, TY = 16;
  static constexpr bool enabled = P <= 3;
};

template <int P, int Q, bool APPLY, int TX, int TY>
int go_tiled(const ElemArgs& A, const SmallTables& tb, cudaStream_t s) {
  auto kern = k_lowt<P, Q, APPLY, TX, TY>;
  const size_t smem = sizeof(double) * lowt_smem_doubles<P, TX, TY, APPLY>();
  static PerDevice<bool> memo;
  const cudaError_t ea = memo.with([&](bool& set) {
    if (set) return cudaSuccess;
    const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set = r == cudaSuccess;
    return r;
  });
  if (ea != cudaSuccess) return set_error(HPG_ERR_CUDA, "k_lowt smem attribute", ea);
  const int nty = (A.ncy + TY - 1) / TY, ntile = ((A.ncx + TX - 1) / TX) * nty;
  cudaError_t e = launch_pdl(kern, dim3(ntile), dim3(TX * TY + 32), smem, s, A, tb, nty);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_lowt launch", e);
}

template <int P, int Q, bool APPLY>
int go(const ElemArgs& A, const SmallTables& tb, cudaStream_t s) {
  static const bool untiled = getenv("HPG_LOWP_UNTILED") != nullptr;   // A/B switch
  if constexpr (LowtTile<P>::enabled) {
    if (!untiled) return go_tiled<P, Q, APPLY, LowtTile<P>::TX, LowtTile<P>::TY>(A, tb, s);
  }
  cudaError_t e = launch_pdl(k_lowp<P, Q, APPLY>, dim3((A.N + LOWP_TH - 1) / LOWP_TH), dim3(LOWP_TH), 0, s, A, tb);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(HPG_ERR_CUDA, "k_lowp launch", e);
}

#define HPG_LOWP(P_, Q_)                                                               \
  if (p == P_ && q == Q_) {                                                            \
    if (!launch) return 1;                                                             \
    return apply ? go<P_, Q_, true>(A, tb, s) : go<P_, Q_, false>(A, tb, s);           \
  }

int dispatch(int p, int q, bool apply, bool launch, const ElemArgs& A, const SmallTables& tb, cudaStream_t s) {
  // BASELINE config 4 (Gauss Q = p + 3) and the reference rule (nq = 2p + 2)
  HPG_LOWP(2, 5) HPG_LOWP(2, 6)
  HPG_LOWP(3, 6) HPG_LOWP(3, 8)
  HPG_LOWP(4, 7) HPG_LOWP(4, 10)
  HPG_LOWP(5, 8) HPG_LOWP(5, 12)
  HPG_LOWP(6, 9) HPG_LOWP(6, 14)
  return launch ? set_error_msg(HPG_ERR_UNSUPPORTED, "no k_lowp instantiation") : 0;
}

}  // namespace

bool lowp_available(int p, int q) {
  ElemArgs A{};
  SmallTables tb{};
  return dispatch(p, q, false, false, A, tb, 0) == 1;
}

int run_lowp(int p, int q, bool apply, const ElemArgs& A, const SmallTables& tb, cudaStream_t s) {
  return dispatch(p, q, apply, true, A, tb, s);
}

}  // namespace hpg
