// DMMA latency / throughput probes: independent accumulator chains per warp
// (ILP) x warps per SM, with register operands or one LDS.64 operand per DMMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int ILP, bool LDS>
__global__ void probe(double* out, int iters) {
  __shared__ double tab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = 1e-9 * i;
  __syncthreads();
  double acc[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1e-9 * threadIdx.x, b = 1.0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      double bb = LDS ? tab[(i * 32 + lane + it) & 255] : b;
      dmma(acc[i][0], acc[i][1], a, bb);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int ILP, bool LDS>
void run(int warps_per_sm, double* out, int nsm) {
  int threads = 128, blocks = nsm * warps_per_sm / 4;
  int iters = 4000;
  probe<ILP, LDS><<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  probe<ILP, LDS><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dmmas_per_sm = (double)iters * ILP * warps_per_sm;
  double ns_per = ms * 1e6 / dmmas_per_sm;        // ns per DMMA per SM
  double warp_lat = ms * 1e6 / (iters);            // ns per chain step per warp
  printf("ILP=%d LDS=%d warps/SM=%2d : %.2f ns/DMMA/SM (peak 2.04 @1.965GHz), chain step %.1f ns, TF=%.1f\n",
         ILP, (int)LDS, warps_per_sm, ns_per, warp_lat, 256.0 * 2 * nsm / ns_per * 1e-3);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 64);
  for (int w : {4, 8, 16, 32}) {
    run<1, false>(w, out, nsm);
    run<2, false>(w, out, nsm);
    run<4, false>(w, out, nsm);
    run<8, false>(w, out, nsm);
    run<2, true>(w, out, nsm);
    run<4, true>(w, out, nsm);
  }
  return 0;
}
