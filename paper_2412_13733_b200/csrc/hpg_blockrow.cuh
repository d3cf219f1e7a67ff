// Element blocks of D by block rows (assembly.py:257-263, 550-557, 804-815).
//
// blk[(a,b),(j,k)] = w_a w_b sum_h Z_a[j][h] G[(b,k)][h],
//   Z_a[j][h] = sum_g G[(a,j)][g] W[g][h],   G[(a,j)][g] = T[a][g] S[g][j].
// One work item = (cell, weight field, test row a).  The item first forms
// Z_a (n x Q) on the FP64 tensor cores into shared memory -- stored in
// C-fragment order, which with the permuted-K convention is directly the A
// operand of the next contraction -- then sweeps b: each (b, k-tile) B
// fragment is read coalesced from the fragment-ordered table PK(G)
// (L2-resident, shared by all cells) and the n x n output tile is scaled by
// w_a w_b and stored as one contiguous block row (a*n+b, j*n+k).
// Small n: one warp per item (4 items per CTA).  Large n (config 3): one
// 256-thread CTA per item, warps splitting the k-tiles of the output.
#pragma once
#include "hpg_common.cuh"
#include "hpg_elem.cuh"
#include "hpg_precond.cuh"

namespace hpg {

struct BArgs {
  int n, NT, QT, nq, nf, ncy;
  int cell0, ncell;        // cells [cell0, cell0 + ncell)
  int per_warp;            // 1: one warp per item; 0: one CTA per item
  int pk_smem;             // 1: PK(G) staged in shared memory; 0: read from L2
  const double* G;         // [n*n][QP]
  const double* PKG;       // [n][NT][2*QT][32]
  const double* wc;        // weight cache (C-fragment order), NW = nf
  double* out;             // blocks of the cells in range
  long long nb;            // block side (n^2 or 2 n^2)
  const double* hx;
  const double* hy;
  // optional fused epilogue: write P_e = -(D_e + E_beta + T/alpha) instead of D_e
  int prec;
  double alpha, beta;
  const double* tri;       // obstacle triples [nkeys][n2][n2]
  const int* key;          // [N] cell -> triple key
};

constexpr int BR_MAXACC = 24;   // 8x8 accumulator tiles per warp

// output staging tile row stride: = 8 mod 16, so the double2 stores of the
// accumulator fragments (j = 8 mt + r, k = 8 nt + 2c) of a quarter warp fall
// in distinct 16-byte bank groups (NP + 1 gave 31 M conflicts at config 1)
__host__ __device__ constexpr int blockrow_ldo(int NP) { return ((NP + 7) / 16) * 16 + 8; }

// QTC > 0: the number of quadrature tiles at compile time (hot shapes: the
// contraction loops unroll); 0: read from the arguments.
template <int NT, int QTC = 0>
__global__ void __launch_bounds__(256) k_blockrow(BArgs B) {
  // k-tile columns per warp pass: all NT for the small (warp-per-item) shapes
  constexpr int NC = NT <= 4 ? NT : (BR_MAXACC / NT > 0 ? BR_MAXACC / NT : 1);
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int r = lane >> 2, c = lane & 3;
  const int n = B.n, QT = QTC > 0 ? QTC : B.QT, QK = 2 * QT, QP = 8 * QT;
  const int zsize = NT * QT * 64;
  const long long items = (long long)B.ncell * B.nf * n;
  // group = the threads sharing one item
  const int gw = B.per_warp ? 1 : nwarps;                     // warps per group
  const int gid = B.per_warp ? warp : 0;                      // group index in CTA
  const int gwarp = B.per_warp ? 0 : warp;                    // warp index in group
  const long long groups_total = (long long)gridDim.x * (B.per_warp ? nwarps : 1);
  // the B-operand table PK(G) staged once per CTA (shared by all items)
  double* sPK = smem;
  const long long pk_len = B.pk_smem ? (long long)n * NT * QK * 32 : 0;
  for (long long i = threadIdx.x; i < pk_len; i += blockDim.x) sPK[i] = __ldg(B.PKG + i);
  const double* PKb = B.pk_smem ? sPK : B.PKG;
  double* sZ = smem + pk_len + (size_t)gid * zsize;
  // per-group output staging tile (NP x NP), written back as a contiguous block row
  constexpr int NP = 8 * NT, LDO = blockrow_ldo(NP);
  double* sO = smem + pk_len + (size_t)(B.per_warp ? nwarps : 1) * zsize + (size_t)gid * NP * LDO;
  __syncthreads();
  for (long long it = (long long)blockIdx.x * (B.per_warp ? nwarps : 1) + gid; it < items;
       it += groups_total) {
    const int a = (int)(it % n);
    const long long t2 = it / n;
    const int f = (int)(t2 % B.nf);
    const int cl = (int)(t2 / B.nf);
    const int e = B.cell0 + cl;
    const int cx = e / B.ncy, cy = e - cx * B.ncy;
    // (1) Z_a = G[(a, :)] W_e  as C-fragment tiles (mt, ht)
    for (int tile = gwarp; tile < NT * QT; tile += gw) {
      const int mt = tile / QT, ht = tile - mt * QT;
      double z[2] = {0.0, 0.0};
      const int j = 8 * mt + r;
      const double* grow = B.G + ((long long)a * n + (j < n ? j : 0)) * QP;
#pragma unroll (QTC > 0 ? 2 * QTC : 1)
      for (int ks = 0; ks < QK; ++ks) {
        const int g = 8 * (ks >> 1) + 2 * c + (ks & 1);
        const double av = (j < n) ? __ldg(grow + g) : 0.0;
        // B[k=g][n=h], h = 8 ht + r, from the weight cache's C-fragment layout
        const int gg = 8 * (ks >> 1) + 2 * c + (ks & 1);    // row g of W for this lane's k
        const int hh = 8 * ht + r;
        const int lanew = (gg & 7) * 4 + ((hh & 7) >> 1);
        const double bv = __ldg(B.wc + wc_index(e, QT, gg >> 3, hh >> 3, B.nf, f, lanew) + (hh & 1));
        dmma(z, av, bv);
      }
      *reinterpret_cast<double2*>(sZ + (size_t)tile * 64 + 2 * lane) = make_double2(z[0], z[1]);
    }
    if (B.per_warp) __syncwarp(); else __syncthreads();
    // (2) sweep b: out[(a,b),(j,k)] = w_a w_b sum_h Z_a[j][h] G[(b,k)][h]
    const double wa = B.hx[cx] * kInvOdd[a];
    double* blk = B.out + (long long)cl * B.nb * B.nb;
    const long long n2 = (long long)n * n;
    for (int b = 0; b < n; ++b) {
      const double wab = wa * (B.hy[cy] * kInvOdd[b]);
      // this warp's k-tiles: nt = gwarp, gwarp + gw, ... (all NT mt rows each)
      for (int nt0 = gwarp; nt0 < NT; nt0 += gw * NC) {
        double acc[NC][NT][2];
#pragma unroll
        for (int ci = 0; ci < NC; ++ci)
#pragma unroll
          for (int mt = 0; mt < NT; ++mt) acc[ci][mt][0] = acc[ci][mt][1] = 0.0;
#pragma unroll (QTC > 0 ? QTC : 1)
        for (int ht = 0; ht < QT; ++ht) {
          double bf[NC][2];
#pragma unroll
          for (int ci = 0; ci < NC; ++ci) {
            const int nt = nt0 + ci * gw;
            const double* pk = PKb + (((long long)b * NT + (nt < NT ? nt : 0)) * QK + 2 * ht) * 32 + lane;
            bf[ci][0] = nt < NT ? pk[0] : 0.0;
            bf[ci][1] = nt < NT ? pk[32] : 0.0;
          }
#pragma unroll
          for (int mt = 0; mt < NT; ++mt) {
            const double2 za = *reinterpret_cast<const double2*>(sZ + (size_t)(mt * QT + ht) * 64 + 2 * lane);
#pragma unroll
            for (int ci = 0; ci < NC; ++ci) {
              if (nt0 + ci * gw < NT) {
                dmma(acc[ci][mt], za.x, bf[ci][0]);
                dmma(acc[ci][mt], za.y, bf[ci][1]);
              }
            }
          }
        }
        // stage the output tile: (mt, nt) holds (j = 8mt + r, k = 8nt + 2c + {0,1})
#pragma unroll
        for (int ci = 0; ci < NC; ++ci) {
          const int nt = nt0 + ci * gw;
          if (nt >= NT) continue;
#pragma unroll
          for (int mt = 0; mt < NT; ++mt) {
            const int j = 8 * mt + r, k = 8 * nt + 2 * c;
            *reinterpret_cast<double2*>(sO + j * LDO + k) = make_double2(acc[ci][mt][0] * wab, acc[ci][mt][1] * wab);
          }
        }
      }
      if (B.per_warp) __syncwarp(); else __syncthreads();
      // contiguous block row (a*n + b): entries j*n + k, coalesced across the group
      const long long row = (long long)a * n + b;
      // fused precond epilogue (obstacle): P = -D - T/alpha - beta mass on the diagonal
      const double* trow = (B.prec && B.nf == 1) ? B.tri + ((size_t)B.key[e] * n2 + row) * n2 : nullptr;
      const double ainv = B.prec ? 1.0 / B.alpha : 0.0;
      const double dmass = B.prec ? B.beta * ((B.hx[cx] / (2.0 * a + 1.0)) * (B.hy[cy] / (2.0 * b + 1.0))) : 0.0;
      const int gt = B.per_warp ? lane : threadIdx.x, gn = B.per_warp ? 32 : blockDim.x;
      int j = gt / n, k = gt - (gt / n) * n;                 // (j, k) of idx, advanced incrementally
      const int dj = gn / n, dk = gn - (gn / n) * n;
      for (int idx = gt; idx < n * n; idx += gn) {
        const double v = sO[j * LDO + k];
        j += dj;
        k += dk;
        if (k >= n) { k -= n; ++j; }
        if (B.nf == 1) {
          double w = v;
          if (B.prec) {
            w = -v - trow[idx] * ainv;
            if (idx == row) w -= dmass;
          }
          blk[row * B.nb + idx] = w;
        } else if (f == 0) {
          blk[row * B.nb + idx] = B.prec ? precond_entry(1, n, (int)n2, B.hx[cx], B.hy[cy], B.alpha, B.beta, nullptr,
                                                         (int)row, idx, v)
                                         : v;
        } else if (f == 1) {
          const double w = B.prec ? -v : v;
          blk[row * B.nb + n2 + idx] = w;
          blk[(n2 + row) * B.nb + idx] = w;
        } else {
          blk[(n2 + row) * B.nb + n2 + idx] =
              B.prec ? precond_entry(1, n, (int)n2, B.hx[cx], B.hy[cy], B.alpha, B.beta, nullptr, (int)(n2 + row),
                                     (int)(n2 + idx), v)
                     : v;
        }
      }
      if (B.per_warp) __syncwarp(); else __syncthreads();
    }
    if (B.per_warp) __syncwarp(); else __syncthreads();
  }
}

}  // namespace hpg
