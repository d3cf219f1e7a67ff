// FP64 peak microbenchmarks for the roofline denominator (MEASURED_PEAKS.json
// has no FP64 entry).  Three measurements, CUDA-event timed:
//   1. DFMA pipe: independent FMA chains per thread, full grid.
//   2. DMMA pipe: mma.sync.m8n8k4.f64 chains per warp, full grid.
//   3. DMMA fragment-layout self-check (8x8x4 product vs host).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// A 8x4 row-major, B 4x8 (stored k-major: B[k][n]), C 8x8.
__global__ void dmma_layout(const double* A, const double* B, double* C) {
  int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];
  double b = B[(lane & 3) * 8 + (lane >> 2)];
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  C[(lane >> 2) * 8 + 2 * (lane & 3)] = d0;
  C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = d1;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int nsm = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // layout check
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = 0.5 * i - 3; }
  for (int m = 0; m < 8; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[k * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *dA, *dB, *dC;
  CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dC, 512));
  CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
  dmma_layout<<<1, 32>>>(dA, dB, dC);
  CK(cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("{\"dmma_layout_maxerr\": %g}\n", err);

  for (int rep = 0; rep < 2; ++rep) {
    int iters = 20000;
    int blocks = nsm * 8, threads = 256;
    dfma_loop<<<blocks, threads>>>(out, 100, 1.0000001, 1e-7);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dfma_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 16 * (double)iters * blocks * threads;
    printf("{\"dfma_tflops\": %.3f, \"ms\": %.3f}\n", flops / ms * 1e-9, ms);

    iters = 20000;
    dmma_loop<<<blocks, threads>>>(out, 100);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dmma_loop<<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double warps = (double)blocks * threads / 32;
    flops = 2.0 * 256 * 8 * (double)iters * warps;
    printf("{\"dmma_tflops\": %.3f, \"ms\": %.3f}\n", flops / ms * 1e-9, ms);
  }
  return 0;
}
