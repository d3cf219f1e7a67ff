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
// References: assembly.py:81-116,470-477,541-548 (B, A, exp_moments),
// spaces.py:25-57 (U numbering, R map), proximal.py:112-126 (residual),
// assembly.py:559-567 (apply_D).
#include "hpg_launch.cuh"
#include "hpg_common.cuh"
#include "hpg_small.cuh"
#include "hpg_usmall_gen.cuh"

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

template <int P, int Q, bool APPLY>
int go(const ElemArgs& A, const SmallTables& tb, cudaStream_t s) {
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
