// Device GMRES: the unrestarted, Givens-rotated GMRES
// of hpgalerkin/linalg.py:134-207 with the whole Krylov iteration on the GPU.
//
// One solve is ONE CUDA graph launch:
//
//   k_init (||r||, target, V0 = r / beta, loop condition)
//   while (cond) {                                   <- device-side WHILE node
//     k_fetch        vin = V[j]
//     <operator>     w = A M vin  (right) | M A vin (left): the caller's
//                    kernels, captured once per solve (hpgGmresCaptureBegin/End)
//     k_arn_dots     h1 = V[0..j]^T w                        (pass 1)
//     k_arn_update   w -= V h1;  h2 = V[0..j]^T w            (pass 2)
//     k_arn_norm     w -= V h2;  H[:,j] = h1 + h2, ||w||; previous rotations,
//                    new Givens rotation, residual |g[j+1]|, stopping test;
//                    sets the loop condition (cudaGraphSetConditional)
//     k_arn_scale    V[j+1] = w / ||w||
//   }
//
// then k_trisolve (back substitution with the rotated Hessenberg, as
// scipy.linalg.solve_triangular) and k_combine (dx = sum_i y_i V[i], the
// reference's accumulation order).  Orthogonalisation is classical
// Gram-Schmidt with one re-orthogonalisation pass (CGS2): two fused
// multi-dot sweeps instead of the reference's j+1 dependent MGS dot/axpy
// pairs; the stopping rule, happy-breakdown test and rotation formulas are the
// reference's.  No host synchronisation inside the iteration and no wasted
// operator applications after convergence.
//
// Reductions are deterministic: each CTA reduces its slice in a fixed tree,
// the last CTA to finish (threadfence + counter) adds the per-CTA partials in
// CTA order.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "../../include/hpg_b200.h"
#include "hpg_launch.cuh"

namespace {

constexpr int KT = 256;          // threads per CTA
constexpr int KW = KT / 32;

struct KState {
  int j;            // current Arnoldi column
  int done;         // converged, happy breakdown or maxiter
  int converged;
  int k;            // iterations performed
  unsigned int counter;
  int maxiter;
  double beta, target, rtol, atol, nrm;
};

struct KArgs {
  long long n;
  long long chunk;  // elements per CTA
  int nb;           // CTAs
  int m;            // maxiter
  long long ldv;    // row stride of V
  double* V;        // (m+1) x ldv
  double* H;        // column j at H + j*(m+1)
  double *cs, *sn, *g, *res, *h1, *h2, *y;
  double* partial;  // [nb][m+2]
  const double* r;  // initial residual (caller fills)
  double* vin;      // operator input
  double* w;        // operator output / orthogonalised vector
  KState* st;
  cudaGraphConditionalHandle cond;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-tree block sum of one value per thread (result valid in thread 0)
__device__ double block_sum(double v, double* sred) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < KW; ++i) s += sred[i];
  return s;
}

// last CTA to arrive?  (all of this CTA's partial stores are fenced first)
__device__ bool last_block(KState* st, int nb) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(&st->counter, 1u);
    is_last = (t == (unsigned)nb - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    if (threadIdx.x == 0) st->counter = 0;
  }
  return is_last != 0;
}

// h[i] = sum_b partial[b][i], i <= j: one warp per i, lanes stride over CTAs
// in a fixed order, then a fixed shuffle tree
__device__ void reduce_partials(const KArgs& A, int cnt, double* out, double* add_to, double* also) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = A.m + 2;
  for (int i = warp; i < cnt; i += KW) {
    double s = 0.0;
    for (int b = lane; b < A.nb; b += 32) s += __ldcg(A.partial + (long long)b * ld + i);
    s = warp_sum(s);
    if (lane == 0) {
      out[i] = s;
      if (add_to) also[i] = add_to[i] + s;
    }
  }
}

// partial[b][i] = sum over this CTA's slice of V[i][k] * sw[k], i <= j
__device__ void slice_dots(const KArgs& A, const double* sw, long long k0, int len, int j) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = A.m + 2;
  for (int i = warp; i <= j; i += KW) {
    const double* v = A.V + (long long)i * A.ldv + k0;
    double s = 0.0;
    for (int t = lane; t < len; t += 32) s = fma(__ldg(v + t), sw[t], s);
    s = warp_sum(s);
    if (lane == 0) A.partial[(long long)blockIdx.x * ld + i] = s;
  }
}

__device__ __forceinline__ void slice(const KArgs& A, long long& k0, int& len) {
  k0 = (long long)blockIdx.x * A.chunk;
  long long e = k0 + A.chunk;
  if (e > A.n) e = A.n;
  len = k0 < A.n ? (int)(e - k0) : 0;
}

// ---- init: beta = ||r||, target, V0 = r / beta, loop condition
__global__ void __launch_bounds__(KT) k_init(KArgs A) {
  __shared__ double sred[KW];
  long long k0;
  int len;
  slice(A, k0, len);
  double s = 0.0;
  for (int t = threadIdx.x; t < len; t += KT) {
    const double v = A.r[k0 + t];
    s = fma(v, v, s);
  }
  s = block_sum(s, sred);
  if (threadIdx.x == 0) A.partial[(long long)blockIdx.x * (A.m + 2)] = s;
  if (!last_block(A.st, A.nb)) return;
  if (threadIdx.x < 32) {
    double q = 0.0;
    for (int b = threadIdx.x; b < A.nb; b += 32) q += __ldcg(A.partial + (long long)b * (A.m + 2));
    q = warp_sum(q);
    if (threadIdx.x == 0) {
      KState* st = A.st;
      const double beta = sqrt(q);
      st->beta = beta;
      st->target = fmax(st->rtol * beta, st->atol);
      st->j = 0;
      st->k = 0;
      A.g[0] = beta;
      A.res[0] = beta;
      // linalg.py:151-153: a zero residual returns converged with 0 iterations;
      // maxiter = 0 leaves only the post-loop test of linalg.py:203-204
      st->converged = (beta == 0.0 || (st->maxiter <= 0 && beta <= st->target)) ? 1 : 0;
      st->done = (beta == 0.0 || st->maxiter <= 0) ? 1 : 0;
      cudaGraphSetConditional(A.cond, st->done ? 0u : 1u);
    }
  }
}

__global__ void __launch_bounds__(KT) k_init_scale(KArgs A) {
  if (A.st->done) return;
  const double beta = A.st->beta;
  long long k0;
  int len;
  slice(A, k0, len);
  for (int t = threadIdx.x; t < len; t += KT) A.V[k0 + t] = A.r[k0 + t] / beta;
}

// ---- loop body
__global__ void __launch_bounds__(KT) k_fetch(KArgs A) {
  const double* v = A.V + (long long)A.st->j * A.ldv;
  long long k0;
  int len;
  slice(A, k0, len);
  for (int t = threadIdx.x; t < len; t += KT) A.vin[k0 + t] = v[k0 + t];
}

__global__ void __launch_bounds__(KT) k_arn_dots(KArgs A) {
  extern __shared__ double sw[];
  const int j = A.st->j;
  long long k0;
  int len;
  slice(A, k0, len);
  for (int t = threadIdx.x; t < len; t += KT) sw[t] = A.w[k0 + t];
  __syncthreads();
  slice_dots(A, sw, k0, len, j);
  if (!last_block(A.st, A.nb)) return;
  reduce_partials(A, j + 1, A.h1, nullptr, nullptr);
}

// w -= V[0..j] h (thread per element, i ascending)
__device__ void slice_update(const KArgs& A, const double* hs, double* sw, long long k0, int len, int j) {
  for (int t = threadIdx.x; t < len; t += KT) {
    double v = A.w[k0 + t];
    const double* col = A.V + k0 + t;
    for (int i = 0; i <= j; ++i) v = fma(-hs[i], __ldg(col + (long long)i * A.ldv), v);
    sw[t] = v;
    A.w[k0 + t] = v;
  }
}

__global__ void __launch_bounds__(KT) k_arn_update(KArgs A) {
  extern __shared__ double sw[];
  __shared__ double hs[1024];
  const int j = A.st->j;
  for (int i = threadIdx.x; i <= j; i += KT) hs[i] = __ldcg(A.h1 + i);
  __syncthreads();
  long long k0;
  int len;
  slice(A, k0, len);
  slice_update(A, hs, sw, k0, len, j);
  __syncthreads();
  slice_dots(A, sw, k0, len, j);
  if (!last_block(A.st, A.nb)) return;
  // H[:, j] = h1 + h2
  reduce_partials(A, j + 1, A.h2, A.h1, A.H + (long long)j * (A.m + 1));
}

__global__ void __launch_bounds__(KT) k_arn_norm(KArgs A) {
  extern __shared__ double sw[];
  __shared__ double hs[1024];
  __shared__ double sred[KW];
  KState* st = A.st;
  const int j = st->j;
  for (int i = threadIdx.x; i <= j; i += KT) hs[i] = __ldcg(A.h2 + i);
  __syncthreads();
  long long k0;
  int len;
  slice(A, k0, len);
  slice_update(A, hs, sw, k0, len, j);
  double s = 0.0;
  for (int t = threadIdx.x; t < len; t += KT) s = fma(sw[t], sw[t], s);
  s = block_sum(s, sred);
  if (threadIdx.x == 0) A.partial[(long long)blockIdx.x * (A.m + 2)] = s;
  if (!last_block(st, A.nb)) return;
  if (threadIdx.x >= 32) return;
  double q = 0.0;
  for (int b = threadIdx.x; b < A.nb; b += 32) q += __ldcg(A.partial + (long long)b * (A.m + 2));
  q = warp_sum(q);
  if (threadIdx.x != 0) return;
  // the reference's rotation bookkeeping (linalg.py:172-190)
  const double nrm = sqrt(q);
  double* Hj = A.H + (long long)j * (A.m + 1);
  Hj[j + 1] = nrm;
  for (int i = 0; i < j; ++i) {
    const double t = A.cs[i] * Hj[i] + A.sn[i] * Hj[i + 1];
    Hj[i + 1] = -A.sn[i] * Hj[i] + A.cs[i] * Hj[i + 1];
    Hj[i] = t;
  }
  const double denom = hypot(Hj[j], Hj[j + 1]);
  if (denom == 0.0) {
    A.cs[j] = 1.0;
    A.sn[j] = 0.0;
  } else {
    A.cs[j] = Hj[j] / denom;
    A.sn[j] = Hj[j + 1] / denom;
  }
  const bool happy = Hj[j + 1] <= 1e-14 * fmax(1.0, fabs(Hj[j]));
  Hj[j] = A.cs[j] * Hj[j] + A.sn[j] * Hj[j + 1];
  A.g[j + 1] = -A.sn[j] * A.g[j];
  A.g[j] = A.cs[j] * A.g[j];
  Hj[j + 1] = 0.0;
  st->k = j + 1;
  A.res[j + 1] = fabs(A.g[j + 1]);
  st->nrm = nrm;
  if (A.res[j + 1] <= st->target || happy) {
    st->converged = 1;
    st->done = 1;
  } else if (j + 1 >= st->maxiter) {
    st->done = 1;
  } else {
    st->j = j + 1;
  }
  cudaGraphSetConditional(A.cond, st->done ? 0u : 1u);
}

__global__ void __launch_bounds__(KT) k_arn_scale(KArgs A) {
  if (A.st->done) return;
  const double nrm = A.st->nrm;
  double* v = A.V + (long long)A.st->j * A.ldv;
  long long k0;
  int len;
  slice(A, k0, len);
  for (int t = threadIdx.x; t < len; t += KT) v[k0 + t] = A.w[k0 + t] / nrm;
}

// ---- solution: y = R^{-1} g (column-oriented back substitution), dx = V^T y
__global__ void k_trisolve(KArgs A) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int k = A.st->k;
  for (int i = 0; i < k; ++i) A.y[i] = A.g[i];
  for (int c = k - 1; c >= 0; --c) {
    const double* Hc = A.H + (long long)c * (A.m + 1);
    A.y[c] = A.y[c] / Hc[c];
    const double yc = A.y[c];
    for (int i = 0; i < c; ++i) A.y[i] -= yc * Hc[i];
  }
}

__global__ void __launch_bounds__(KT) k_combine(KArgs A, double* dx) {
  __shared__ double ys[1024];
  const int k = A.st->k;
  for (int i = threadIdx.x; i < k; i += KT) ys[i] = A.y[i];
  __syncthreads();
  long long k0;
  int len;
  slice(A, k0, len);
  for (int t = threadIdx.x; t < len; t += KT) {
    double v = 0.0;
    for (int i = 0; i < k; ++i) v += ys[i] * A.V[(long long)i * A.ldv + k0 + t];
    dx[k0 + t] = v;
  }
}

__global__ void k_axpby(long long n, double a, const double* x, double b, const double* y, double* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = b == 0.0 ? a * x[i] : (a == 0.0 ? b * y[i] : a * x[i] + b * y[i]);
}

}  // namespace

struct hpgGmres_st {
  KArgs A;
  size_t smem = 0;
  double* mem = nullptr;
  KState* st = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraph_t body = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool capturing = false;
  KState host;
};

namespace {
int kfail(int code, const std::string& m) {
  hpg::set_error_msg(code, m.c_str());
  return code;
}
#define KTRY(x)                                                                          \
  do {                                                                                   \
    cudaError_t _e = (x);                                                                \
    if (_e != cudaSuccess) return kfail(HPG_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
  } while (0)

int add_kernel(cudaGraph_t g, cudaGraphNode_t* node, const cudaGraphNode_t* deps, int ndeps, void* fn,
               dim3 grid, size_t smem, KArgs* A) {
  cudaKernelNodeParams p = {};
  void* args[] = {A};
  p.func = fn;
  p.gridDim = grid;
  p.blockDim = dim3(KT);
  p.sharedMemBytes = (unsigned)smem;
  p.kernelParams = args;
  KTRY(cudaGraphAddKernelNode(node, g, deps, ndeps, &p));
  return HPG_OK;
}

void release(hpgGmres G) {
  if (G->exec) cudaGraphExecDestroy(G->exec);
  if (G->graph) cudaGraphDestroy(G->graph);
  G->exec = nullptr;
  G->graph = nullptr;
  G->body = nullptr;
}
}  // namespace

extern "C" {

int hpgGmresCreate(hpgGmres* out, long long n, int maxiter) {
  HPG_NVTX("hpgGmresCreate");
  if (!out) return kfail(HPG_ERR_ARG, "null handle pointer");
  *out = nullptr;
  if (n < 1 || maxiter < 0 || maxiter > 1000) return kfail(HPG_ERR_ARG, "need n >= 1 and 0 <= maxiter <= 1000");
  hpgGmres G = new hpgGmres_st();
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  KArgs& A = G->A;
  memset(&A, 0, sizeof(A));
  A.n = n;
  A.m = maxiter;
  // one slice of <= 12288 doubles (96 KB of shared memory) per CTA, >= one CTA per SM
  long long nb = (n + 12287) / 12288;
  if (nb < nsm) nb = nsm;
  if (nb > n) nb = n;
  A.nb = (int)nb;
  A.chunk = (n + nb - 1) / nb;
  A.ldv = (n + 3) / 4 * 4;
  G->smem = sizeof(double) * (size_t)A.chunk;
  const int m = maxiter;
  const size_t vdbl = (size_t)(m + 1) * A.ldv;
  const size_t sdbl = (size_t)(m + 1) * m + 2 * m + 6 * (m + 2) + (size_t)A.nb * (m + 2);
  const size_t total = vdbl + sdbl + 64;
  cudaError_t e = cudaMalloc(&G->mem, total * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&G->st, sizeof(KState));
  if (e != cudaSuccess) {
    cudaFree(G->mem);
    delete G;
    return kfail(HPG_ERR_CUDA, std::string("gmres workspace: ") + cudaGetErrorString(e));
  }
  cudaMemset(G->st, 0, sizeof(KState));
  double* p = G->mem;
  A.V = p; p += vdbl;
  A.H = p; p += (size_t)(m + 1) * (m > 0 ? m : 1);
  A.cs = p; p += m + 2;
  A.sn = p; p += m + 2;
  A.g = p; p += m + 2;
  A.res = p; p += m + 2;
  A.h1 = p; p += m + 2;
  A.h2 = p; p += m + 2;
  A.y = p; p += m + 2;
  A.partial = p;
  A.st = G->st;
  // the attribute only grows (another solver object may need more)
  struct Memo { size_t attr = 48u << 10; };
  static hpg::PerDevice<Memo> memo;
  cudaError_t ae = memo.with([&](Memo& mm) -> cudaError_t {
    if (G->smem <= mm.attr) return cudaSuccess;
    cudaError_t r = cudaFuncSetAttribute(k_arn_dots, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G->smem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(k_arn_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G->smem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(k_arn_norm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G->smem);
    if (r == cudaSuccess) mm.attr = G->smem;
    return r;
  });
  if (ae != cudaSuccess) {
    cudaFree(G->mem);
    cudaFree(G->st);
    delete G;
    return kfail(HPG_ERR_CUDA, std::string("gmres smem attribute: ") + cudaGetErrorString(ae));
  }
  *out = G;
  return HPG_OK;
}

int hpgGmresDestroy(hpgGmres G) {
  HPG_NVTX("hpgGmresDestroy");
  if (!G) return HPG_OK;
  release(G);
  cudaFree(G->mem);
  cudaFree(G->st);
  delete G;
  return HPG_OK;
}

int hpgGmresBind(hpgGmres G, const double* r, double* vin, double* w) {
  HPG_NVTX("hpgGmresBind");
  if (!G) return kfail(HPG_ERR_ARG, "null gmres handle");
  if (!r || !vin || !w) return kfail(HPG_ERR_ARG, "null vector");
  if (G->capturing) return kfail(HPG_ERR_ARG, "cannot rebind during capture");
  release(G);               // a captured loop holds the old pointers
  G->A.r = r;
  G->A.vin = vin;
  G->A.w = w;
  return HPG_OK;
}

int hpgGmresCaptureBegin(hpgGmres G, void* stream) {
  HPG_NVTX("hpgGmresCaptureBegin");
  if (!G) return kfail(HPG_ERR_ARG, "null gmres handle");
  if (G->capturing) return kfail(HPG_ERR_ARG, "capture already in progress");
  if (!G->A.r || !G->A.vin || !G->A.w) return kfail(HPG_ERR_ARG, "hpgGmresBind has not been called");
  release(G);
  KArgs& A = G->A;
  KTRY(cudaGraphCreate(&G->graph, 0));
  KTRY(cudaGraphConditionalHandleCreate(&A.cond, G->graph, 0, cudaGraphCondAssignDefault));
  const dim3 grid(A.nb);
  cudaGraphNode_t n0, n1, nw;
  if (int rc = add_kernel(G->graph, &n0, nullptr, 0, (void*)k_init, grid, 0, &A)) return rc;
  if (int rc = add_kernel(G->graph, &n1, &n0, 1, (void*)k_init_scale, grid, 0, &A)) return rc;
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = A.cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  KTRY(cudaGraphAddNode(&nw, G->graph, &n1, 1, &cp));
  G->body = cp.conditional.phGraph_out[0];
  cudaStream_t s = (cudaStream_t)stream;
  KTRY(cudaStreamBeginCaptureToGraph(s, G->body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  G->capturing = true;
  k_fetch<<<grid, KT, 0, s>>>(A);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaGraph_t junk;
    cudaStreamEndCapture(s, &junk);
    G->capturing = false;
    return kfail(HPG_ERR_CUDA, std::string("k_fetch capture: ") + cudaGetErrorString(e));
  }
  return HPG_OK;
}

int hpgGmresCaptureEnd(hpgGmres G, void* stream) {
  HPG_NVTX("hpgGmresCaptureEnd");
  if (!G || !G->capturing) return kfail(HPG_ERR_ARG, "no capture in progress");
  KArgs& A = G->A;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid(A.nb);
  k_arn_dots<<<grid, KT, G->smem, s>>>(A);
  k_arn_update<<<grid, KT, G->smem, s>>>(A);
  k_arn_norm<<<grid, KT, G->smem, s>>>(A);
  k_arn_scale<<<grid, KT, 0, s>>>(A);
  cudaError_t le = cudaGetLastError();
  cudaGraph_t out;
  cudaError_t e = cudaStreamEndCapture(s, &out);
  G->capturing = false;
  if (le != cudaSuccess) return kfail(HPG_ERR_CUDA, std::string("arnoldi capture: ") + cudaGetErrorString(le));
  KTRY(e);
  KTRY(cudaGraphInstantiate(&G->exec, G->graph, 0));
  return HPG_OK;
}

int hpgGmresSolve(hpgGmres G, double rtol, double atol, double* dx, void* stream) {
  HPG_NVTX("hpgGmresSolve");
  if (!G || !G->exec) return kfail(HPG_ERR_ARG, "gmres loop not captured");
  if (!dx) return kfail(HPG_ERR_ARG, "null dx");
  KArgs& A = G->A;
  cudaStream_t s = (cudaStream_t)stream;
  KState h;
  memset(&h, 0, sizeof(h));
  h.rtol = rtol;
  h.atol = atol;
  h.maxiter = A.m;
  KTRY(cudaMemcpyAsync(G->st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  KTRY(cudaGraphLaunch(G->exec, s));
  k_trisolve<<<1, 32, 0, s>>>(A);
  k_combine<<<A.nb, KT, 0, s>>>(A, dx);
  KTRY(cudaGetLastError());
  KTRY(cudaMemcpyAsync(&G->host, G->st, sizeof(KState), cudaMemcpyDeviceToHost, s));
  return HPG_OK;
}

int hpgGmresStatus(hpgGmres G, int* iters, int* converged, double* residuals, void* stream) {
  HPG_NVTX("hpgGmresStatus");
  if (!G) return kfail(HPG_ERR_ARG, "null gmres handle");
  cudaStream_t s = (cudaStream_t)stream;
  KTRY(cudaStreamSynchronize(s));
  const int k = G->host.k;
  if (iters) *iters = k;
  if (converged) *converged = G->host.converged;
  if (residuals) KTRY(cudaMemcpy(residuals, G->A.res, sizeof(double) * (size_t)(k + 1), cudaMemcpyDeviceToHost));
  return HPG_OK;
}

int hpgAxpby(long long n, double a, const double* x, double b, const double* y, double* out, void* stream) {
  HPG_NVTX("hpgAxpby");
  if (n < 0 || !out || (a != 0.0 && !x) || (b != 0.0 && !y)) return kfail(HPG_ERR_ARG, "bad axpby arguments");
  if (n == 0) return HPG_OK;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_axpby<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, a, x, b, y, out);
  KTRY(cudaGetLastError());
  return HPG_OK;
}

}  // extern "C"
