// Streaming cached Jacobian apply for many small cells (config 1: 4096 cells,
// n = 15, Q = 24): a persistent grid, one CTA per SM, every warp streaming
// an equal number of ROW TILES back to back.
//
// k_warp runs this shape as one wave of one-cell warps: every warp loads at
// the same time (DMMA pipe idle), then every warp contracts at the same time
// (memory idle).  Here
//  * both tables live in registers as operand fragments (PK(S) and PK(T) are
//    12 doubles per lane each at NT = 2, QT = 3): no shared-memory operand
//    read per DMMA;
//  * the next cell's point weights (cp.async into the other half of the
//    warp's shared-memory slice) and x fragments (registers) are in flight
//    during the current cell's contractions;
//  * a warp's DMMA chains are dependent (32-cycle latency, one issue slot per
//    16 cycles and scheduler), so MW = 3 warps per scheduler keep the pipe
//    full -- but 28 cells per SM are 7 per scheduler, which 3 warps cannot
//    share evenly.  The schedule is therefore cut at ROW-TILE granularity: the
//    QT * C row tiles of a scheduler group's C cells are dealt out as MW
//    equal contiguous runs, so a run boundary may fall inside a cell.  Such a
//    cell is finished by the warp that owns its first row tiles (its last
//    item); the warp owning the rest (its FIRST item, done long before) hands
//    its partial Y over through shared memory and a named barrier.
// Per row tile the arithmetic is k_warp's; a split cell sums its two
// partials in a fixed order (deterministic, 1e-12 parity with the oracle).
#pragma once
#include "hpg_elem.cuh"

namespace hpg {

#ifndef HPG_STREAM_MW
#define HPG_STREAM_MW 3
#endif

template <int NT, int QT, int MODE>
struct StreamCfg {
  using TR = ModeTraits<MODE>;
  static constexpr int MW = HPG_STREAM_MW;               // warps per scheduler group
  static constexpr int W = 4 * MW;
  static constexpr int WDBL = QT * QT * TR::NW * 64;     // one cell's weights, fragment order
  static constexpr int YDBL = TR::NOUT * NT * NT * 64;   // one partial Y, fragment order
  static constexpr int SMEM_DBL = W * 2 * WDBL + 4 * (MW - 1) * YDBL + 8 * NT;
};

__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// Optional (A/B only, off): layers of independent DMMAs separated by a
// never-taken, distinct conditional return.  Left alone, ptxas issues each
// accumulation chain's dependent DMMAs back to back; fenced, it keeps the
// chains breadth-first (cuobjdump -sass).  Measured equal at MW = 3 (12.06
// vs 12.03 us): three warps per scheduler already cover the chain latency.
#ifndef HPG_STREAM_FENCE
#define HPG_STREAM_FENCE 0
#endif
#if HPG_STREAM_FENCE
#define HPG_FENCE() do { if (A.N == -1 - __COUNTER__) return; } while (0)
#else
#define HPG_FENCE()
#endif

template <int NT, int QT, int MODE>
__global__ void __launch_bounds__(32 * StreamCfg<NT, QT, MODE>::W, 1)
k_stream(ElemArgs A) {
  using TR = ModeTraits<MODE>;
  using CF = StreamCfg<NT, QT, MODE>;
  static_assert(MODE == M_OBST_CACHED || MODE == M_GRAD_CACHED, "cached modes only");
  constexpr int NP = 8 * NT, NK = 2 * NT, QK = 2 * QT;
  constexpr int NIN = TR::NIN, NSYN = TR::NSYN, NOUT = TR::NOUT, NW = TR::NW;
  constexpr int W = CF::W, MW = CF::MW, WDBL = CF::WDBL, YDBL = CF::YDBL;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  // warps are dealt to the four schedulers round robin: group = scheduler
  const int g = warp & 3, m = warp >> 2;
  double* sW = smem + warp * 2 * WDBL;           // [buf][rt][ht][w][lane][2]
  double* sY = smem + W * 2 * WDBL;              // [g][boundary][o][bt][at][lane][2]
  double* sInv = sY + 4 * (MW - 1) * YDBL;       // 1/(2k+1), k < NP

  // table fragments: PK(S)[t][ks][lane], PK(T)[bt][ks][lane] (constant data:
  // read before the grid-dependency wait)
  double Sr[QT][NK], Tr[NT][QK];
#pragma unroll
  for (int t = 0; t < QT; ++t)
#pragma unroll
    for (int ks = 0; ks < NK; ++ks) Sr[t][ks] = __ldg(A.Sf + (t * NK + ks) * 32 + lane);
#pragma unroll
  for (int bt = 0; bt < NT; ++bt)
#pragma unroll
    for (int ks = 0; ks < QK; ++ks) Tr[bt][ks] = __ldg(A.Tf + (bt * QK + ks) * 32 + lane);
  if (threadIdx.x < NP) sInv[threadIdx.x] = kInvOdd[threadIdx.x];

  // CTA b owns cells b, b + grid, ...; its k-th cell goes to group k mod 4;
  // the group's row tiles [lo, hi) (cell-major) are this warp's run
  const int K = ((int)A.N - A.e0 - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int C = (K - g + 3) / 4;
  const int lo = (m * QT * C) / MW, hi = ((m + 1) * QT * C) / MW;
  auto cell_of = [&](int i) { return A.e0 + (int)blockIdx.x + (g + 4 * i) * (int)gridDim.x; };
  int i = lo / QT;
  const int i_end = (hi + QT - 1) / QT;

  // one item = the row tiles [rb, re) of group cell i
  auto load_weights = [&](int e, int rb, int re, int b) {
    const double* src = A.wc_in + wc_index(e, QT, 0, 0, NW, 0, lane);
    double* dst = sW + b * WDBL;
#pragma unroll
    for (int rt = 0; rt < QT; ++rt)
      if (rt >= rb && rt < re) {
#pragma unroll
        for (int t = rt * QT * NW; t < (rt + 1) * QT * NW; ++t) cp_async16(dst + t * 64 + 2 * lane, src + t * 64);
      }
    cp_async_commit();
  };
  // cell -> (cx, cy) by a float reciprocal with an exact fix-up (N < 2^23)
  // instead of the ~25-instruction integer division, twice per item
  const float ncy_inv = 1.0f / (float)A.ncy;
  auto split_cell = [&](int e, int& cx, int& cy) {
    cx = __float2int_rd(((float)e + 0.5f) * ncy_inv);
    cy = e - cx * A.ncy;
    if (cy < 0) { --cx; cy += A.ncy; }
    if (cy >= A.ncy) { ++cx; cy -= A.ncy; }
  };
  // lane-invariant tile geometry: the fragment rows this lane touches are
  // a_q = 8 (q >> 1) + 2c + (q & 1), q < NK (x loads: q = k-step; stores:
  // q = 2 at + j), the columns b_nt = 8 nt + r; their element offsets inside
  // a cell (32-bit: the launcher checks the vector length) and in-range masks
  // are computed once, so an item's addresses are one cell base plus these
  int ro[NK];
  bool okr[NK], okc[NT];
#pragma unroll
  for (int q = 0; q < NK; ++q) {
    const int a = 8 * (q >> 1) + 2 * c + (q & 1);
    ro[q] = a * (int)A.ld + r;
    okr[q] = a < A.n;
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) okc[nt] = 8 * nt + r < A.n;
  using XFrag = double[NIN][NK][NT];
  XFrag X, Xn;
  double hxv = 0.0, hyv = 0.0, hxn = 0.0, hyn = 0.0;
  auto load_cell = [&](int e, XFrag& Xd, double& hx, double& hy) {
    int cx, cy;
    split_cell(e, cx, cy);
    hx = __ldg(A.hx + cx);
    hy = __ldg(A.hy + cy);
#pragma unroll
    for (int f = 0; f < NIN; ++f) {
      const double* src;
      int comp;
      field_src<MODE>(A, f, src, comp);
      src += comp * A.ncomp + psi_index(A, cx, cy, 0, 0);
#pragma unroll
      for (int ks = 0; ks < NK; ++ks)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          Xd[f][ks][nt] = (okr[ks] && okc[nt]) ? __ldg(src + ro[ks] + 8 * nt) : 0.0;
    }
  };
  auto item_rb = [&](int i) { return lo > i * QT ? lo - i * QT : 0; };
  auto item_re = [&](int i) { return hi < (i + 1) * QT ? hi - i * QT : QT; };

  // the weight cache may be read before the wait only when the host knows
  // the immediately preceding kernel did not write it (A.wc_early)
  if (A.wc_early && i < i_end) load_weights(cell_of(i), item_rb(i), item_re(i), 0);
  pdl_trigger();
  pdl_wait();
  if (!A.wc_early && i < i_end) load_weights(cell_of(i), item_rb(i), item_re(i), 0);
  if (i < i_end) load_cell(cell_of(i), X, hxv, hyv);
  __syncthreads();   // sInv
  int buf = 0;

  for (; i < i_end; ++i) {
    const int e = cell_of(i);
    int cx, cy;
    split_cell(e, cx, cy);
    const int rb = item_rb(i), re = item_re(i);
    const bool more = i + 1 < i_end;
    if (more) {
      load_weights(cell_of(i + 1), item_rb(i + 1), item_re(i + 1), buf ^ 1);
      load_cell(cell_of(i + 1), Xn, hxn, hyn);
    }
    const double* sWc = sW + buf * WDBL;
    // this item's weights have landed; the next item's may still fly
    if (more) cp_async_wait_group<1>();
    else cp_async_wait_all();

    double Y[NOUT][NT][NT][2];
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
#pragma unroll
      for (int bt = 0; bt < NT; ++bt)
#pragma unroll
        for (int at = 0; at < NT; ++at) Y[o][bt][at][0] = Y[o][bt][at][1] = 0.0;

#pragma unroll
    for (int rt = 0; rt < QT; ++rt) {
      if (rt < rb || rt >= re) continue;   // warp-uniform
      // P = S[rt,:] C, V = P S^T
      double V[NSYN][QT][2];
#pragma unroll
      for (int f = 0; f < NSYN; ++f) {
        double P[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) P[nt][0] = P[nt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < NK; ++ks) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(P[nt], Sr[rt][ks], X[f][ks][nt]);
          HPG_FENCE();
        }
#pragma unroll
        for (int ht = 0; ht < QT; ++ht) V[f][ht][0] = V[f][ht][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < NK; ++ks) {
#pragma unroll
          for (int ht = 0; ht < QT; ++ht) dmma(V[f][ht], P[ks >> 1][ks & 1], Sr[ht][ks]);
          HPG_FENCE();
        }
      }
      // pointwise map with the cached weights
      double Vw[NOUT][QT][2];
#pragma unroll
      for (int ht = 0; ht < QT; ++ht) {
        double Vp[NSYN][2], Wc[NW][2], out2[NOUT][2];
#pragma unroll
        for (int f = 0; f < NSYN; ++f) { Vp[f][0] = V[f][ht][0]; Vp[f][1] = V[f][ht][1]; }
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const double2 t = *reinterpret_cast<const double2*>(sWc + ((rt * QT + ht) * NW + w) * 64 + 2 * lane);
          Wc[w][0] = t.x;
          Wc[w][1] = t.y;
        }
        map_pair_w<MODE, NSYN, NOUT, NW>(Vp, Wc, out2, 8 * rt + r < A.nq, 8 * ht + 2 * c, A.nq);
#pragma unroll
        for (int o = 0; o < NOUT; ++o) { Vw[o][ht][0] = out2[o][0]; Vw[o][ht][1] = out2[o][1]; }
      }
      // R = T W^T (even / odd k-step chains, summed), Y += R T[:,rt]^T
#pragma unroll
      for (int o = 0; o < NOUT; ++o) {
        double R[NT][2];
#pragma unroll
        for (int bt = 0; bt < NT; ++bt) R[bt][0] = R[bt][1] = 0.0;
        // (one chain per tile: the even / odd split of k_warp costs 2 NT DADDs
        // per row tile on the pipe the DMMAs use, and three warps per
        // scheduler cover the chain latency)
#pragma unroll
        for (int ks = 0; ks < QK; ++ks)
#pragma unroll
          for (int bt = 0; bt < NT; ++bt) dmma(R[bt], Tr[bt][ks], Vw[o][ks >> 1][ks & 1]);
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) {
#pragma unroll
          for (int bt = 0; bt < NT; ++bt)
#pragma unroll
            for (int at = 0; at < NT; ++at) dmma(Y[o][bt][at], R[bt][k2], Tr[at][2 * rt + k2]);
          HPG_FENCE();
        }
      }
    }

    if (rb > 0) {
      // the cell's first row tiles belong to warp m - 1 of this group: hand
      // the partial over (that warp reaches the cell at the end of its run)
      double* dst = sY + (g * (MW - 1) + (m - 1)) * YDBL + 2 * lane;
#pragma unroll
      for (int o = 0; o < NOUT; ++o)
#pragma unroll
        for (int bt = 0; bt < NT; ++bt)
#pragma unroll
          for (int at = 0; at < NT; ++at)
            *reinterpret_cast<double2*>(dst + ((o * NT + bt) * NT + at) * 64) =
                make_double2(Y[o][bt][at][0], Y[o][bt][at][1]);
      __threadfence_block();
      named_bar_arrive(1 + g * (MW - 1) + (m - 1), 64);
    } else {
      if (re < QT) {
        // the rest of the cell was computed by warp m + 1 (its first item)
        named_bar_sync(1 + g * (MW - 1) + m, 64);
        const double* src = sY + (g * (MW - 1) + m) * YDBL + 2 * lane;
#pragma unroll
        for (int o = 0; o < NOUT; ++o)
#pragma unroll
          for (int bt = 0; bt < NT; ++bt)
#pragma unroll
            for (int at = 0; at < NT; ++at) {
              const double2 t = *reinterpret_cast<const double2*>(src + ((o * NT + bt) * NT + at) * 64);
              Y[o][bt][at][0] += t.x;
              Y[o][bt][at][1] += t.y;
            }
      }
      // M[a][b] = w_a w_b Y[b][a] (write_moment's order of operations)
      double* dst0 = A.out + psi_index(A, cx, cy, 0, 0);
      double wa[NK], wb[NT];
#pragma unroll
      for (int q = 0; q < NK; ++q) wa[q] = hxv * sInv[8 * (q >> 1) + 2 * c + (q & 1)];
#pragma unroll
      for (int bt = 0; bt < NT; ++bt) wb[bt] = hyv * sInv[8 * bt + r];
#pragma unroll
      for (int o = 0; o < NOUT; ++o)
#pragma unroll
        for (int bt = 0; bt < NT; ++bt)
#pragma unroll
          for (int at = 0; at < NT; ++at)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int q = 2 * at + j;
              if (okr[q] && okc[bt])
                dst0[(long long)o * A.ncomp + ro[q] + 8 * bt] = (wa[q] * Y[o][bt][at][j]) * wb[bt];
            }
    }
    if (more) {
#pragma unroll
      for (int f = 0; f < NIN; ++f)
#pragma unroll
        for (int ks = 0; ks < NK; ++ks)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) X[f][ks][nt] = Xn[f][ks][nt];
      hxv = hxn;
      hyv = hyn;
    }
    buf ^= 1;
  }
}

}  // namespace hpg
