// Batched row-major DGEMM on the FP64 tensor cores (mma.sync m8n8k4 ->
// DMMA.8x8x4), for the dense products around the hot path: the
// fast-diagonalisation stiffness solve (linalg.factor_stiffness replacement,
// SURVEY.md §8f rank 4) and the QVI full-space U synthesis / analysis
// (qvi.py:34-57, §8f rank 3).
//
//   C[b] = alpha (A[b] B[b]) (.* F) + beta C[b]
//        A: M x K (lda), B: K x N (ldb), C: M x N (ldc)
//
// with batch strides (0 = operand shared by the batch) and an optional
// elementwise epilogue factor F (M x N, ldc; the 1/(lx_i + ly_j) scaling of
// the fast-diagonalisation solve).  Transposed operands are stored
// transposed at setup, so only NN is needed.
//
// CTA tile 64 x 64, 4 warps of 32 x 32 (4 x 4 DMMA tiles, 16 independent
// accumulator chains per warp), K staged 16 at a time through shared memory
// in two buffers (cp.async 8-byte copies with zero fill: leading dimensions
// may be odd, e.g. 1023).  Padded strides keep the fragment reads at the
// two-wavefront minimum.
#pragma once
#include <cuda_runtime.h>

#include "hpg_common.cuh"

namespace hpg {

struct GemmNN {
  int M, N, K;
  long long lda, ldb, ldc;
  long long sA, sB, sC;        // batch strides (doubles)
  const double* A;
  const double* B;
  double* C;
  const double* F;             // optional epilogue factor (stride sF, ld ldc)
  long long sF;
  double alpha = 1.0, beta = 0.0;   // C = alpha (A B) (.* F) + beta C
};

constexpr int GM_BM = 64, GM_BN = 64, GM_BK = 16;
constexpr int GM_LDA = GM_BK + 4;    // A tile [BM][BK]
constexpr int GM_LDB = GM_BN + 8;    // B tile [BK][BN]

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(sz) : "memory");
}

static __global__ void __launch_bounds__(128) k_dgemm_nn(GemmNN g) {
  __shared__ double sA[2][GM_BM * GM_LDA];
  __shared__ double sB[2][GM_BK * GM_LDB];
  const int b = blockIdx.z;
  const double* A = g.A + (long long)b * g.sA;
  const double* B = g.B + (long long)b * g.sB;
  const int m0 = blockIdx.y * GM_BM, n0 = blockIdx.x * GM_BN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, c = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

  auto stage = [&](int buf, int k0) {
    // A tile 64 x 16: 1024 doubles, 8 per thread; B tile 16 x 64: 8 per thread
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int idx = tid + 128 * t;
      const int am = idx >> 4, ak = idx & 15;
      const int gm = m0 + am, gk = k0 + ak;
      const bool va = gm < g.M && gk < g.K;
      cp_async8(&sA[buf][am * GM_LDA + ak], va ? A + (long long)gm * g.lda + gk : A, va);
      const int bk = idx >> 6, bn = idx & 63;
      const int hk = k0 + bk, hn = n0 + bn;
      const bool vb = hk < g.K && hn < g.N;
      cp_async8(&sB[buf][bk * GM_LDB + bn], vb ? B + (long long)hk * g.ldb + hn : B, vb);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (g.K + GM_BK - 1) / GM_BK;
  stage(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      stage(buf ^ 1, (kt + 1) * GM_BK);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* a_s = sA[buf];
    const double* b_s = sB[buf];
#pragma unroll
    for (int ks = 0; ks < GM_BK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = a_s[(wm + 8 * i + r) * GM_LDA + ks + c];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b_s[(ks + c) * GM_LDB + wn + 8 * j + r];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* C = g.C + (long long)b * g.sC;
  const double* F = g.F ? g.F + (long long)b * g.sF : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int row = m0 + wm + 8 * i + r, col = n0 + wn + 8 * j + 2 * c + q;
        if (row < g.M && col < g.N) {
          double v = acc[i][j][q];
          if (F) v *= F[(long long)row * g.ldc + col];
          if (g.alpha != 1.0) v *= g.alpha;
          if (g.beta != 0.0) v += g.beta * C[(long long)row * g.ldc + col];
          C[(long long)row * g.ldc + col] = v;
        }
      }
}

inline cudaError_t dgemm_nn(const GemmNN& g, int batch, cudaStream_t s) {
  dim3 grid((g.N + GM_BN - 1) / GM_BN, (g.M + GM_BM - 1) / GM_BM, batch);
  k_dgemm_nn<<<grid, 128, 0, s>>>(g);
  return cudaGetLastError();
}

inline GemmNN gemm_nn(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb,
                      double* C, long long ldc) {
  GemmNN g{};
  g.alpha = 1.0;
  g.beta = 0.0;
  g.M = M; g.N = N; g.K = K;
  g.lda = lda; g.ldb = ldb; g.ldc = ldc;
  g.A = A; g.B = B; g.C = C;
  return g;
}

}  // namespace hpg
