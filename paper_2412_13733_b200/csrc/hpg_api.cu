// C ABI of the B200 hpG element-quadrature engine (see include/hpg_b200.h).
// Host side of the library: plan construction (fragment-ordered tables on the
// device), path selection and kernel launches.  No allocation in the hot
// entry points: every workspace is sized at plan creation (the optional
// solver setups -- hpgPrecondPrepare, hpgStiffnessFactor, hpgUFullSetup --
// allocate their own once).  A plan owns its scratch, so one plan must not be
// used from two streams at the same time (see include/hpg_b200.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hpg_b200.h"
#include "hpg_blocks.cuh"
#include "hpg_blockrow.cuh"
#include "hpg_common.cuh"
#include "hpg_launch.cuh"
#include "hpg_precond.cuh"
#include "hpg_schur.cuh"
#include "hpg_qvi.cuh"

#include "hpg_gemm.cuh"
#include "hpg_useside.cuh"
#include "hpg_small.cuh"
#include "hpg_ucell.cuh"

using namespace hpg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                     \
  do {                                                                                  \
    cudaError_t _e = (x);                                                               \
    if (_e != cudaSuccess)                                                              \
      return fail(HPG_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e));      \
  } while (0)

#define LAUNCH_CHECK() CUDA_TRY(cudaGetLastError())

// PK(X)[tile][ks][lane] = X[8*tile + r][8*(ks>>1) + 2c + (ks&1)], zero padded.
std::vector<double> pk_table(const double* X, int rows, int cols, int RT, int KP) {
  std::vector<double> out((size_t)RT * (KP / 4) * 32, 0.0);
  for (int t = 0; t < RT; ++t)
    for (int ks = 0; ks < KP / 4; ++ks)
      for (int lane = 0; lane < 32; ++lane) {
        int r = lane >> 2, c = lane & 3;
        int row = 8 * t + r, col = 8 * (ks >> 1) + 2 * c + (ks & 1);
        double v = (row < rows && col < cols) ? X[(size_t)row * cols + col] : 0.0;
        out[((size_t)t * (KP / 4) + ks) * 32 + lane] = v;
      }
  return out;
}

template <typename T>
int upload(T** dst, const T* src, size_t count) {
  CUDA_TRY(cudaMalloc(dst, count * sizeof(T) + 16));
  CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
  return HPG_OK;
}

}  // namespace

namespace hpg {
int set_error(int code, const char* where, cudaError_t e) {
  return fail(code, std::string(where) + ": " + cudaGetErrorString(e));
}
int set_error_msg(int code, const char* msg) { return fail(code, msg); }
}  // namespace hpg

struct hpgPlan_st {
  int kind, ncx, ncy, p, n, m, nq, N;
  int NT, QT, NP, QP;
  int nix, niy;
  long long ncomp, ndof_psi, ndof_u;
  int path[8];                  // ElemPath per element-kernel mode
  // few-cell plans: U side concurrent with the psi side (residual_concurrent)
  bool concurrent = false;
  cudaStream_t aux[1] = {nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[1] = {nullptr};
  // hpgApplyCachedHostSlab: upload-done events, round robin (created on first use)
  cudaEvent_t ev_slab[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int ev_slab_next = 0;
  double* mscr = nullptr;       // psi-side moments [ndof_psi]
  double* wscr = nullptr;       // weight cache of the fused residual + cached apply
  // weight cache written by the LAST kernel of this plan's most recent call
  // (nullptr if that kernel wrote none): the next cached apply may prefetch
  // any other cache before its grid-dependency wait
  const double* last_wc = nullptr;
  int splits;
  double *Sf = nullptr, *Tf = nullptr, *hx = nullptr, *hy = nullptr;
  double* G = nullptr;        // block table [n2][QP]
  // u-side analysis (load_vector): PK(Tu) with n := m
  int NTu;
  double* Tuf = nullptr;
  double* Suf = nullptr;
  double* scratch_u = nullptr;  // [N][m][m]
  double* mu = nullptr;         // x-major m-tiles
  double* partial = nullptr;    // CTA split partials
  size_t partial_len = 0;
  double* Z = nullptr;          // blocks stage-1 scratch
  double* edge = nullptr;       // [N][4m-4] residual hat contributions
  double* PKG = nullptr;        // block-row B-operand table PK(G) [n][NT][QK][32]
  double* ubuf = nullptr;       // CTA path U-side scratch (large m)
  bool small = false;           // thread-per-element low-degree path available
  SmallTables stab;             // its tables (kernel-parameter / constant bank)

  // per-cell Schur preconditioner: hat triples per width key (obstacle)
  std::vector<double> hxh, hyh;  // host copies of the cell widths
  double* tri = nullptr;         // [nkeys][n2][n2]
  int* cell_key = nullptr;       // [N]
  int nkeys = 0;

  // fast-diagonalisation solves: interior stiffness A (fdm[0]) and the QVI
  // full-space H = A_full + gamma M_full (fdm[1]); Schur apply scratch
  struct Fdm {
    int r = 0, c = 0;
    double *Vx = nullptr, *Vy = nullptr, *VxT = nullptr, *VyT = nullptr, *finv = nullptr, *w1 = nullptr,
           *w2 = nullptr;
    bool ready = false;
    void release() {
      cudaFree(Vx); cudaFree(Vy); cudaFree(VxT); cudaFree(VyT); cudaFree(finv); cudaFree(w1); cudaFree(w2);
      Vx = Vy = VxT = VyT = finv = w1 = w2 = nullptr;
      ready = false;
    }
  } fdm[2];
  double *su1 = nullptr, *su2 = nullptr, *syD = nullptr, *sz = nullptr;
  bool fdm_ready = false;
  // QVI full-space operator tables and scratch
  double *qSR = nullptr, *qTR = nullptr, *qK = nullptr, *qM = nullptr, *qSRT = nullptr, *qTRT = nullptr;
  double *qKT = nullptr, *qMT = nullptr;
  double *qC = nullptr, *qT = nullptr, *qV = nullptr, *qG = nullptr, *qP1 = nullptr, *qP2 = nullptr;
  double *qH1 = nullptr, *qH2 = nullptr, *qH3 = nullptr;
  bool q_ready = false;

  int zcells = 0;
  int* dflag = nullptr;
  int nsm = 148;
};

namespace {

ElemArgs base_args(const hpgPlan_st* P) {
  ElemArgs A;
  memset(&A, 0, sizeof(A));
  A.ncx = P->ncx; A.ncy = P->ncy; A.n = P->n; A.m = P->m; A.p = P->p; A.nq = P->nq; A.N = P->N;
  A.nix = P->nix; A.niy = P->niy;
  A.ld = (long long)P->ncy * P->n;
  A.ncomp = P->ncomp;
  A.hx = P->hx; A.hy = P->hy;
  A.Sf = P->Sf; A.Tf = P->Tf;
  A.NT = P->NT; A.QT = P->QT; A.splits = 1;
  A.partial = P->partial;
  return A;
}

bool warp_fits(int mode, int NT, int QT) {
  switch (mode) {
    case M_OBST_RES: return warp_available<M_OBST_RES>(NT, QT);
    case M_OBST_APPLY: return warp_available<M_OBST_APPLY>(NT, QT);
    case M_OBST_CACHED: return warp_available<M_OBST_CACHED>(NT, QT);
    case M_GRAD_RES: return warp_available<M_GRAD_RES>(NT, QT);
    case M_GRAD_APPLY: return warp_available<M_GRAD_APPLY>(NT, QT);
    case M_GRAD_CACHED: return warp_available<M_GRAD_CACHED>(NT, QT);
    default: return false;
  }
}

template <int MODE>
int run_elem(hpgPlan_st* P, ElemArgs A, cudaStream_t s) {
  if (P->path[MODE] == PATH_CTA) A.splits = P->splits;
  return run_mode<MODE>(P->path[MODE], A, s);
}

// shared memory of the block-row kernel (k_blockrow, 4 warps): PK(G) staged
// when it fits, else read from L2 (*pk_smem = 0)
size_t blockrow_smem(const hpgPlan_st* P, int* pk_smem) {
  const int threads = 128;
  const size_t zs = sizeof(double) * (size_t)P->NT * P->QT * 64;
  const size_t pks = sizeof(double) * (size_t)P->n * P->NT * 2 * P->QT * 32;
  const size_t so = sizeof(double) * (size_t)(8 * P->NT) * blockrow_ldo(8 * P->NT);
  size_t smem = pks + (zs + so) * (threads / 32);
  *pk_smem = 1;
  if (smem > ((size_t)200 << 10) && P->NT <= 4) {
    *pk_smem = 0;
    smem = (zs + so) * (threads / 32);
  }
  return smem;
}

// large tiles: element blocks as two GEMMs (Z = G W, blocks = Z G^T) through
// the plan's global scratch instead of the block-row kernel
bool blocks_use_gemm(const hpgPlan_st* P) {
  int pk;
  return blockrow_smem(P, &pk) > ((size_t)200 << 10) || P->NT > 4;
}

bool wsplit_fits(int mode, int NT, int QT) {
  switch (mode) {
    case M_OBST_RES: return wsplit_available<M_OBST_RES>(NT, QT);
    case M_OBST_APPLY: return wsplit_available<M_OBST_APPLY>(NT, QT);
    case M_OBST_CACHED: return wsplit_available<M_OBST_CACHED>(NT, QT);
    case M_GRAD_RES: return wsplit_available<M_GRAD_RES>(NT, QT);
    case M_GRAD_APPLY: return wsplit_available<M_GRAD_APPLY>(NT, QT);
    case M_GRAD_CACHED: return wsplit_available<M_GRAD_CACHED>(NT, QT);
    default: return false;
  }
}

int check(hpgPlan p) {
  if (p == nullptr) return fail(HPG_ERR_ARG, "null plan");
  p->last_wc = nullptr;        // entry points that end with a cache writer set it again
  return HPG_OK;
}

int run_ulocal(hpgPlan_st* P, UArgs& U, cudaStream_t s) {
  long long total = (long long)P->N * P->m * P->m;
  k_u_local<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(U);
  LAUNCH_CHECK();
  long long tot2 = (long long)P->nix * P->niy;
  if (tot2 > 0) {
    k_u_gather<<<(unsigned)((tot2 + 255) / 256), 256, 0, s>>>(U);
    LAUNCH_CHECK();
  }
  return HPG_OK;
}

UArgs base_uargs(const hpgPlan_st* P) {
  UArgs U;
  memset(&U, 0, sizeof(U));
  U.ncx = P->ncx; U.ncy = P->ncy; U.p = P->p; U.n = P->n; U.m = P->m;
  U.nix = P->nix; U.niy = P->niy; U.gradient = P->kind == HPG_GRADIENT;
  U.ld = (long long)P->ncy * P->n; U.ncomp = P->ncomp;
  U.hx = P->hx; U.hy = P->hy;
  U.scratch = P->scratch_u;
  return U;
}

}  // namespace

extern "C" {

int hpgVersion(void) { return 1; }

const char* hpgLastError(void) { return g_err.c_str(); }

int hpgPlanCreate(hpgPlan* plan, int kind, int ncx, int ncy, int p, int nq, const double* S,
                  const double* T, const double* Su, const double* Tu, const double* hx,
                  const double* hy) {
  HPG_NVTX("hpgPlanCreate");
  if (plan == nullptr) return fail(HPG_ERR_ARG, "null plan pointer");
  *plan = nullptr;
  if (kind != HPG_OBSTACLE && kind != HPG_GRADIENT) return fail(HPG_ERR_ARG, "unknown kind");
  if (ncx < 1 || ncy < 1 || nq < 1) return fail(HPG_ERR_ARG, "bad mesh or quadrature size");
  if (kind == HPG_OBSTACLE && p < 2) return fail(HPG_ERR_ARG, "obstacle discretization requires p >= 2");
  if (kind == HPG_GRADIENT && p < 1) return fail(HPG_ERR_ARG, "gradient discretization requires p >= 1");
  if (!S || !T || !Su || !Tu || !hx || !hy) return fail(HPG_ERR_ARG, "null table");
  hpgPlan_st* P = new hpgPlan_st();
  P->kind = kind; P->ncx = ncx; P->ncy = ncy; P->p = p; P->nq = nq;
  P->n = kind == HPG_OBSTACLE ? p - 1 : p;
  P->m = p + 1;
  P->N = ncx * ncy;
  P->NT = (P->n + 7) / 8; P->QT = (nq + 7) / 8;
  P->NP = 8 * P->NT; P->QP = 8 * P->QT;
  P->nix = ncx * p - 1; P->niy = ncy * p - 1;
  if (p == 1) { P->nix = ncx - 1; P->niy = ncy - 1; }
  P->ncomp = (long long)ncx * P->n * ncy * P->n;
  P->ndof_psi = P->ncomp * (kind == HPG_OBSTACLE ? 1 : 2);
  P->ndof_u = (long long)P->nix * P->niy;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&P->nsm, cudaDevAttrMultiProcessorCount, dev);
  if (P->n > 128 || nq > 256) { hpgPlanDestroy(P); return fail(HPG_ERR_UNSUPPORTED, "n > 128 or nq > 256"); }

  std::vector<double> sf = pk_table(S, nq, P->n, P->QT, P->NP);
  std::vector<double> tf = pk_table(T, P->n, nq, P->NT, P->QP);
  int rc;
  if ((rc = upload(&P->Sf, sf.data(), sf.size()))) { hpgPlanDestroy(P); return rc; }
  if ((rc = upload(&P->Tf, tf.data(), tf.size()))) { hpgPlanDestroy(P); return rc; }
  if ((rc = upload(&P->hx, hx, ncx))) { hpgPlanDestroy(P); return rc; }
  if ((rc = upload(&P->hy, hy, ncy))) { hpgPlanDestroy(P); return rc; }
  P->hxh.assign(hx, hx + ncx);
  P->hyh.assign(hy, hy + ncy);
  // u side (load_vector): analysis with Tu, tile side m
  P->NTu = (P->m + 7) / 8;
  std::vector<double> tuf = pk_table(Tu, P->m, nq, P->NTu, P->QP);
  std::vector<double> suf = pk_table(Su, nq, P->m, P->QT, 8 * P->NTu);
  if ((rc = upload(&P->Tuf, tuf.data(), tuf.size()))) { hpgPlanDestroy(P); return rc; }
  if ((rc = upload(&P->Suf, suf.data(), suf.size()))) { hpgPlanDestroy(P); return rc; }
  // low-degree obstacle path (config 4): tables passed by value to k_small
  memset(&P->stab, 0, sizeof(P->stab));
  if (kind == HPG_OBSTACLE && P->n <= SMALL_MAXN && nq <= SMALL_MAXQ && small_available(P->n, nq)) {
    P->small = true;
    for (int g = 0; g < nq; ++g)
      for (int a = 0; a < P->n; ++a) P->stab.S[g * P->n + a] = S[(size_t)g * P->n + a];
    for (int a = 0; a < P->n; ++a)
      for (int g = 0; g < nq; ++g) P->stab.T[a * nq + g] = T[(size_t)a * nq + g];
  }
  // block table G[(a,j)][g] = T[a][g] S[g][j]
  int n2 = P->n * P->n;
  std::vector<double> G((size_t)n2 * P->QP, 0.0);
  for (int a = 0; a < P->n; ++a)
    for (int j = 0; j < P->n; ++j)
      for (int g = 0; g < nq; ++g)
        G[((size_t)a * P->n + j) * P->QP + g] = T[(size_t)a * nq + g] * S[(size_t)g * P->n + j];
  if ((rc = upload(&P->G, G.data(), G.size()))) { hpgPlanDestroy(P); return rc; }
  {
    // PK(G)[b][nt][ks][lane] = G[(b, k = 8nt + r)][h = 8(ks>>1) + 2c + (ks&1)]
    const int QK = 2 * P->QT;
    std::vector<double> pkg((size_t)P->n * P->NT * QK * 32, 0.0);
    for (int b = 0; b < P->n; ++b)
      for (int nt = 0; nt < P->NT; ++nt)
        for (int ks = 0; ks < QK; ++ks)
          for (int lane = 0; lane < 32; ++lane) {
            const int r = lane >> 2, c = lane & 3;
            const int k = 8 * nt + r, h = 8 * (ks >> 1) + 2 * c + (ks & 1);
            if (k < P->n && h < nq)
              pkg[(((size_t)b * P->NT + nt) * QK + ks) * 32 + lane] = G[((size_t)b * P->n + k) * P->QP + h];
          }
    if ((rc = upload(&P->PKG, pkg.data(), pkg.size()))) { hpgPlanDestroy(P); return rc; }
  }
  cudaError_t e = cudaMalloc(&P->scratch_u, sizeof(double) * (size_t)P->N * P->m * P->m + 16);
  if (e == cudaSuccess) e = cudaMalloc(&P->mu, sizeof(double) * (size_t)P->N * P->m * P->m + 16);
  if (e == cudaSuccess) e = cudaMalloc(&P->dflag, sizeof(int) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&P->edge, sizeof(double) * (size_t)P->N * (4 * P->m - 4) + 16);
  if (e != cudaSuccess) { hpgPlanDestroy(P); return fail(HPG_ERR_CUDA, cudaGetErrorString(e)); }

  // path selection
  // element-kernel path per mode: a warp per element when there is an
  // instantiation and enough elements to fill the GPU; few mid-size elements
  // (config 2: 256, config 0: 16) take a CTA per element with a warp per
  // row tile; the rest the generic CTA path
  {
    const bool ws_ok = P->N < 4 * P->nsm && getenv("HPG_NO_WSPLIT") == nullptr;
    for (int mode = M_OBST_RES; mode <= M_GRAD_CACHED; ++mode) {
      P->path[mode] = warp_fits(mode, P->NT, P->QT) ? PATH_WARP : PATH_CTA;
      if (ws_ok && wsplit_fits(mode, P->NT, P->QT)) P->path[mode] = PATH_WSPLIT;
    }
    P->path[M_VALUES] = PATH_CTA;
  }
  // few cells: the U side overlaps the psi-side quadrature on an auxiliary stream
  if (P->N < 4 * P->nsm && getenv("HPG_NO_CONCURRENT") == nullptr &&
      !(kind == HPG_OBSTACLE && P->small && lowp_available(p, nq))) {
    const size_t wlen = (size_t)P->N * P->QT * P->QT * (kind == HPG_OBSTACLE ? 1 : 3) * 64;
    e = cudaStreamCreateWithFlags(&P->aux[0], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&P->ev_join[0], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&P->mscr, sizeof(double) * P->ndof_psi + 16);
    if (e == cudaSuccess) e = cudaMalloc(&P->wscr, sizeof(double) * wlen + 16);
    if (e != cudaSuccess) { hpgPlanDestroy(P); return fail(HPG_ERR_CUDA, cudaGetErrorString(e)); }
    P->concurrent = true;
  }
  // split the Q row tiles of an element across CTAs when there are few elements
  // (one wave: the largest divisor of QT with N * splits <= #SMs, so every
  // split gets the same number of row tiles)
  P->splits = 1;
  if (P->N < P->nsm) {
    int cap = P->nsm / P->N;
    for (int d = 1; d <= P->QT && d <= cap; ++d)
      if (P->QT % d == 0) P->splits = d;
  }
  P->partial_len = (size_t)P->N * P->splits * 2 * P->NP * P->NP;
  int NPu = 8 * P->NTu;
  size_t plu = (size_t)P->N * P->splits * NPu * NPu;
  if (plu > P->partial_len) P->partial_len = plu;
  e = cudaMalloc(&P->partial, sizeof(double) * P->partial_len + 16);
  if (e != cudaSuccess) { hpgPlanDestroy(P); return fail(HPG_ERR_CUDA, cudaGetErrorString(e)); }
  // element blocks of large tiles run as two GEMMs through a stage-1 scratch
  // (<= 256 MB, whole cells): sized here so hpgBlocks never allocates
  if (blocks_use_gemm(P)) {
    const size_t per_cell = (size_t)(kind == HPG_OBSTACLE ? 1 : 3) * n2 * P->QP;
    long long chunk = (long long)((256ull << 20) / (sizeof(double) * per_cell));
    if (chunk < 1) chunk = 1;
    if (chunk > P->N) chunk = P->N;
    e = cudaMalloc(&P->Z, sizeof(double) * per_cell * chunk + 16);
    if (e != cudaSuccess) { hpgPlanDestroy(P); return fail(HPG_ERR_CUDA, cudaGetErrorString(e)); }
    P->zcells = (int)chunk;
  }
  *plan = P;
  return HPG_OK;
}

int hpgPlanDestroy(hpgPlan P) {
  HPG_NVTX("hpgPlanDestroy");
  if (P == nullptr) return HPG_OK;
  cudaFree(P->Sf); cudaFree(P->Tf); cudaFree(P->hx); cudaFree(P->hy); cudaFree(P->G);
  cudaFree(P->Tuf); cudaFree(P->Suf); cudaFree(P->scratch_u); cudaFree(P->mu);
  cudaFree(P->partial); cudaFree(P->Z); cudaFree(P->dflag); cudaFree(P->edge); cudaFree(P->PKG); cudaFree(P->ubuf);
  cudaFree(P->tri); cudaFree(P->cell_key);
  P->fdm[0].release(); P->fdm[1].release();
  cudaFree(P->su1); cudaFree(P->su2); cudaFree(P->syD); cudaFree(P->sz);
  cudaFree(P->qSR); cudaFree(P->qTR); cudaFree(P->qK); cudaFree(P->qM); cudaFree(P->qC); cudaFree(P->qT);
  cudaFree(P->qV); cudaFree(P->qG); cudaFree(P->qP1); cudaFree(P->qP2); cudaFree(P->qH1); cudaFree(P->qH2);
  cudaFree(P->qH3); cudaFree(P->qSRT); cudaFree(P->qTRT); cudaFree(P->qKT); cudaFree(P->qMT);
  cudaFree(P->mscr); cudaFree(P->wscr);
  if (P->aux[0]) cudaStreamDestroy(P->aux[0]);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  if (P->ev_join[0]) cudaEventDestroy(P->ev_join[0]);
  for (cudaEvent_t e : P->ev_slab)
    if (e) cudaEventDestroy(e);
  delete P;
  return HPG_OK;
}

int hpgPlanInfo(hpgPlan P, long long* info) {
  HPG_NVTX("hpgPlanInfo");
  if (int rc = check(P)) return rc;
  int nw = P->kind == HPG_OBSTACLE ? 1 : 3;
  info[0] = P->n;
  info[1] = P->m;
  info[2] = P->nq;
  info[3] = P->N;
  info[4] = P->ndof_psi;
  info[5] = P->ndof_u;
  info[6] = (long long)P->N * P->QT * P->QT * nw * 64;
  long long nb = (long long)P->n * P->n * (P->kind == HPG_OBSTACLE ? 1 : 2);
  info[7] = nb * nb;
  {
    const int pm = P->path[P->kind == HPG_OBSTACLE ? M_OBST_RES : M_GRAD_RES];
    info[8] = pm == PATH_WARP ? 0 : (pm == PATH_CTA ? 1 : 2);
  }
  info[9] = P->splits;
  // kernels per fused residual + apply call: 1 on the single-pass low-degree
  // path (k_lowp), else U side + psi side + hat gather (+ apply)
  info[10] = (P->kind == HPG_OBSTACLE && P->small && lowp_available(P->p, P->nq)) ? 1 : 3;
  // 1 when hpgResidualApply computes the apply inside the residual's pass
  info[11] = (P->kind == HPG_OBSTACLE && P->small) || P->concurrent ? 1 : 0;
  return HPG_OK;
}

int hpgObstacleMoments(hpgPlan P, const double* psi, double* out, int* clamped, double* wcache, void* stream) {
  HPG_NVTX("hpgObstacleMoments");
  if (int rc = check(P)) return rc;
  if (P->kind != HPG_OBSTACLE) return fail(HPG_ERR_ARG, "plan is not an obstacle plan");
  if (!psi || !out || !clamped) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  A.in0 = psi; A.out = out; A.flag = clamped; A.wc_out = wcache;
  if (P->small && wcache == nullptr) return run_small(P->n, P->nq, true, false, A, P->stab, (cudaStream_t)stream);
  const int rc = run_elem<M_OBST_RES>(P, A, (cudaStream_t)stream);
  P->last_wc = wcache;
  return rc;
}

int hpgObstacleApplyD(hpgPlan P, const double* psi, const double* x, double* y, void* stream) {
  HPG_NVTX("hpgObstacleApplyD");
  if (int rc = check(P)) return rc;
  if (P->kind != HPG_OBSTACLE) return fail(HPG_ERR_ARG, "plan is not an obstacle plan");
  if (!psi || !x || !y) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  A.in0 = psi; A.in1 = x; A.out = y;
  if (P->small) {
    A.wc_out = y;
    return run_small(P->n, P->nq, false, true, A, P->stab, (cudaStream_t)stream);
  }
  return run_elem<M_OBST_APPLY>(P, A, (cudaStream_t)stream);
}

int hpgGradientMoments(hpgPlan P, const double* psi, const double* phi, double* out, double* wcache, void* stream) {
  HPG_NVTX("hpgGradientMoments");
  if (int rc = check(P)) return rc;
  if (P->kind != HPG_GRADIENT) return fail(HPG_ERR_ARG, "plan is not a gradient plan");
  if (!psi || !phi || !out) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  A.in0 = psi; A.phi = phi; A.out = out; A.wc_out = wcache; A.flag = P->dflag;
  const int rc = run_elem<M_GRAD_RES>(P, A, (cudaStream_t)stream);
  P->last_wc = wcache;
  return rc;
}

int hpgGradientApplyD(hpgPlan P, const double* psi, const double* phi, const double* x, double* y, void* stream) {
  HPG_NVTX("hpgGradientApplyD");
  if (int rc = check(P)) return rc;
  if (P->kind != HPG_GRADIENT) return fail(HPG_ERR_ARG, "plan is not a gradient plan");
  if (!psi || !phi || !x || !y) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  A.in0 = psi; A.in1 = x; A.phi = phi; A.out = y;
  return run_elem<M_GRAD_APPLY>(P, A, (cudaStream_t)stream);
}

int hpgApplyCached(hpgPlan P, const double* wcache, const double* x, double* y, void* stream) {
  HPG_NVTX("hpgApplyCached");
  const double* prev_wc = P ? P->last_wc : nullptr;
  if (int rc = check(P)) return rc;
  if (!wcache || !x || !y) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  A.wc_in = wcache; A.in1 = x; A.out = y;
  static const bool early_ok = getenv("HPG_NO_EARLY_WC") == nullptr;
  A.wc_early = early_ok && prev_wc != wcache;
  if (P->kind == HPG_OBSTACLE) return run_elem<M_OBST_CACHED>(P, A, (cudaStream_t)stream);
  return run_elem<M_GRAD_CACHED>(P, A, (cudaStream_t)stream);
}

// Cached apply restricted to the cells [cell_begin, cell_end) (x-major cell
// order: a range of whole cell columns is a contiguous row range of x and y).
// The apply is cell-local (spaces.py:89-108), so a host caller can pipeline
// slabs: upload slab k while slab k - 1 is applied and slab k - 2 downloaded.
int hpgApplyCachedRange(hpgPlan P, const double* wcache, const double* x, double* y, int cell_begin,
                        int cell_end, void* stream) {
  HPG_NVTX("hpgApplyCachedRange");
  const double* prev_wc = P ? P->last_wc : nullptr;
  if (int rc = check(P)) return rc;
  if (!wcache || !x || !y) return fail(HPG_ERR_ARG, "null pointer");
  if (cell_begin < 0 || cell_end > P->N || cell_begin > cell_end) return fail(HPG_ERR_ARG, "bad cell range");
  const int mode = P->kind == HPG_OBSTACLE ? M_OBST_CACHED : M_GRAD_CACHED;
  if (P->path[mode] != PATH_WARP) return fail(HPG_ERR_UNSUPPORTED, "cell ranges need the warp-per-cell apply path");
  if (cell_begin == cell_end) return HPG_OK;
  ElemArgs A = base_args(P);
  A.wc_in = wcache; A.in1 = x; A.out = y;
  A.e0 = cell_begin; A.N = cell_end;
  static const bool early_ok = getenv("HPG_NO_EARLY_WC") == nullptr;
  A.wc_early = early_ok && prev_wc != wcache;
  if (P->kind == HPG_OBSTACLE) return run_elem<M_OBST_CACHED>(P, A, (cudaStream_t)stream);
  return run_elem<M_GRAD_CACHED>(P, A, (cudaStream_t)stream);
}

// One slab (cell columns [cx_begin, cx_end)) of a host-buffer D @ x:
//   upload  stage -> dev_x   on copy_stream   (stage: page-locked, the slab's
//                                              rows, component after component)
//   apply   dev_x -> dev_y   on stream, after the upload
//   download dev_y -> y_host on stream        (y_host: page-locked, full length)
// The caller fills `stage` for slab k + 1 while slab k is in flight and
// synchronises `stream` once at the end; uploads (copy_stream) and downloads
// (stream) of neighbouring slabs use both PCIe directions at once.
int hpgApplyCachedHostSlab(hpgPlan P, const double* wcache, const double* stage, double* dev_x, double* dev_y,
                           double* y_host, int cx_begin, int cx_end, void* copy_stream, void* stream) {
  HPG_NVTX("hpgApplyCachedHostSlab");
  if (P == nullptr) return fail(HPG_ERR_ARG, "null plan");
  if (!wcache || !stage || !dev_x || !dev_y || !y_host) return fail(HPG_ERR_ARG, "null pointer");
  if (cx_begin < 0 || cx_end > P->ncx || cx_begin >= cx_end) return fail(HPG_ERR_ARG, "bad cell-column range");
  cudaStream_t up = (cudaStream_t)copy_stream, s = (cudaStream_t)stream;
  const int ncmp = P->kind == HPG_OBSTACLE ? 1 : 2;
  const size_t rows = (size_t)P->n * P->ncy * P->n;            // doubles per cell column and component
  const size_t ln = (size_t)(cx_end - cx_begin) * rows;
  for (int c = 0; c < ncmp; ++c)
    CUDA_TRY(cudaMemcpyAsync(dev_x + c * P->ncomp + cx_begin * rows, stage + c * ln, sizeof(double) * ln,
                             cudaMemcpyHostToDevice, up));
  cudaEvent_t& ev = P->ev_slab[P->ev_slab_next];
  P->ev_slab_next = (P->ev_slab_next + 1) % 8;
  if (ev == nullptr) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(ev, up));
  CUDA_TRY(cudaStreamWaitEvent(s, ev, 0));
  if (int rc = hpgApplyCachedRange(P, wcache, dev_x, dev_y, cx_begin * P->ncy, cx_end * P->ncy, stream)) return rc;
  for (int c = 0; c < ncmp; ++c)
    CUDA_TRY(cudaMemcpyAsync(y_host + c * P->ncomp + cx_begin * rows, dev_y + c * P->ncomp + cx_begin * rows,
                             sizeof(double) * ln, cudaMemcpyDeviceToHost, s));
  return HPG_OK;
}

// U side of the residual: b_psi <- phi_mom - B^T u (obstacle) | -B^T u
// (gradient); b_u on the dofs a cell owns alone, hat contributions to the edge
// scratch (finished by k_hat_gather)
static int uside_impl(hpgPlan P, const ElemArgs& A, cudaStream_t s) {
  // thread-per-cell U side only when there are enough cells to fill the GPU;
  // few cells (configs 0, 2, 3) go to the thread-per-entry kernel below
  const bool many = P->N >= 8 * P->nsm;
  if (many && usmall_available(P->p, P->kind == HPG_GRADIENT)) {
    // low degree: thread per cell, generated straight-line code
    return run_usmall(P->p, P->kind == HPG_GRADIENT, A, s);
  }
  if (many && P->kind == HPG_OBSTACLE && upass_available(P->p) && getenv("HPG_UPASS_OFF") == nullptr) {
    // mid degree: warp per cell, generated separable passes
    return run_upass(P->p, P->kind == HPG_GRADIENT, A, s);
  }
  // thread per cell-local entry
  int TG = P->m * P->m;
  TG = TG > 1024 ? 1024 : ((TG + 31) / 32) * 32;
  // many mid-size cells (config 2): two entries per thread, so >= 2 CTAs
  // fit an SM (register-limited) and all cells run in one wave
  if (P->N >= P->nsm && TG > 512) TG = ((P->m * P->m + 1) / 2 + 31) / 32 * 32;
  int cpb = 256 / TG;
  if (cpb < 1) cpb = 1;
  size_t smem = sizeof(double) * ((size_t)cpb * ((size_t)P->m * (P->m | 1) + 2 * (size_t)P->n * P->n) +
                                  2 * P->m + 8);
  if (smem > ((size_t)227 << 10)) return fail(HPG_ERR_UNSUPPORTED, "U tile too large for shared memory");
  void* fn = P->kind == HPG_GRADIENT ? (void*)k_uside_pt<true> : (void*)k_uside_pt<false>;
  if (smem > (48u << 10)) CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // few large cells: split each cell's entries over several CTAs (one wave)
  int usplit = 1;
  if (cpb == 1 && P->N < P->nsm) {
    const int blocks = (P->m * P->m + TG - 1) / TG;
    usplit = P->nsm / P->N;
    if (usplit > blocks) usplit = blocks;
    if (usplit < 1) usplit = 1;
  }
  const dim3 grid((P->N + cpb - 1) / cpb * usplit), block(cpb * TG);
  if (P->kind == HPG_GRADIENT)
    CUDA_TRY(launch_pdl(k_uside_pt<true>, grid, block, smem, s, A, cpb, TG, usplit));
  else
    CUDA_TRY(launch_pdl(k_uside_pt<false>, grid, block, smem, s, A, cpb, TG, usplit));
  CUDA_TRY(cudaGetLastError());
  return HPG_OK;
}

static long long hat_count(const hpgPlan_st* P) {
  return (long long)(P->ncx - 1) * P->niy + (long long)(P->nix - (P->ncx - 1)) * (P->ncy - 1);
}

static int hat_gather(hpgPlan P, const ElemArgs& A, cudaStream_t s) {
  const long long nh = hat_count(P);
  if (nh <= 0) return HPG_OK;
  CUDA_TRY(launch_pdl(k_hat_gather, dim3((unsigned)((nh + 255) / 256)), dim3(256), 0, s, A));
  CUDA_TRY(cudaGetLastError());
  return HPG_OK;
}

// Few-cell plans (configs 0, 2, 3): the U side (+ hat gather) runs on the
// plan's auxiliary stream concurrently with the psi-side quadrature, which
// writes the plain moments M to a scratch vector; after the join one
// elementwise kernel finishes b_psi = (phi_mom - B^T u) - M (obstacle) /
// (-B^T u) + M (gradient) -- the same operations in the same order as the
// sequential path, so the results are bitwise identical.  For
// hpgResidualApply the Jacobian apply then runs from the point weights the
// psi side cached (measured faster than recomputing them from psi on a
// second concurrent stream: the two element kernels do not fit an SM together).
static int residual_concurrent(hpgPlan P, ElemArgs A, double* wcache, const double* x, double* y,
                               cudaStream_t s) {
  double* wc = wcache;
  if (x != nullptr && wc == nullptr) wc = P->wscr;
  CUDA_TRY(cudaEventRecord(P->ev_fork, s));
  CUDA_TRY(cudaStreamWaitEvent(P->aux[0], P->ev_fork, 0));
  int rc;
  // (a) U side + hat gather, concurrent
  ElemArgs U = A;
  U.residual = 1;
  if ((rc = uside_impl(P, U, P->aux[0]))) return rc;
  if ((rc = hat_gather(P, U, P->aux[0]))) return rc;
  CUDA_TRY(cudaEventRecord(P->ev_join[0], P->aux[0]));
  // (b) psi side: plain moments into the scratch (+ weight cache, flag)
  ElemArgs Q = A;
  Q.residual = 0;
  Q.out = P->mscr;
  Q.wc_out = wc;
  rc = P->kind == HPG_OBSTACLE ? run_elem<M_OBST_RES>(P, Q, s) : run_elem<M_GRAD_RES>(P, Q, s);
  if (rc) return rc;
  // (c) the Jacobian apply at the same psi from the cached weights (it does
  //     not need the U side: it runs before the join, overlapping it too)
  if (x != nullptr) {
    ElemArgs C = base_args(P);
    C.wc_in = wc; C.in1 = x; C.out = y;
    rc = P->kind == HPG_OBSTACLE ? run_elem<M_OBST_CACHED>(P, C, s) : run_elem<M_GRAD_CACHED>(P, C, s);
    if (rc) return rc;
  }
  CUDA_TRY(cudaStreamWaitEvent(s, P->ev_join[0], 0));
  // (d) b_psi = (phi_mom - B^T u) - M | (-B^T u) + M
  const long long n = P->ndof_psi;
  k_residual_combine<<<(unsigned)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8), 256, 0, s>>>(
      A.out, P->mscr, n, P->kind == HPG_GRADIENT);
  CUDA_TRY(cudaGetLastError());
  return HPG_OK;
}

static int residual_impl(hpgPlan P, double alpha, const double* psi_prev, const double* u,
                         const double* psi, const double* phi, const double* f_load, double* b_u,
                         double* b_psi, int* clamped, double* wcache, const double* x, double* y,
                         void* stream) {
  if (int rc = check(P)) return rc;
  // u-side arrays are empty (and may be NULL) when the mesh has no interior U dofs
  const bool uok = P->ndof_u == 0 || (u && f_load && b_u);
  if (!psi_prev || !psi || !phi || !b_psi || !uok) return fail(HPG_ERR_ARG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  ElemArgs A = base_args(P);
  A.in0 = psi; A.out = b_psi; A.wc_out = wcache; A.residual = 1; A.u = u;
  A.alpha = alpha; A.psi_prev = psi_prev; A.f_load = f_load; A.b_u = b_u; A.edge = P->edge;
  int rc;
  if (P->kind == HPG_OBSTACLE) {
    if (!clamped) return fail(HPG_ERR_ARG, "null clamp flag");
    A.phi_mom = phi; A.flag = clamped;
  } else {
    A.phi = phi; A.flag = P->dflag;
  }
  if (P->kind == HPG_OBSTACLE && P->small && wcache == nullptr && lowp_available(P->p, P->nq) &&
      getenv("HPG_LOWP_OFF") == nullptr) {
    // low degree: the whole residual (+ Jacobian apply at the same psi) in one
    // single-pass kernel (hpg_lowp.cu)
    if (x != nullptr) { A.in1 = x; A.wc_out = y; }
    return run_lowp(P->p, P->nq, x != nullptr, A, P->stab, s);
  }
  if (P->concurrent && !(P->small && wcache == nullptr)) return residual_concurrent(P, A, wcache, x, y, s);
  // (1) U side
  if ((rc = uside_impl(P, A, s))) return rc;
  // (2) psi side finishes b_psi in place (proximal.py:123 order)
  A.residual = 2;
  A.usmem = 0;
  A.ubuf = nullptr;
  if (P->small && wcache == nullptr) {
    // low-degree path: one thread per cell, residual moments (+ Jacobian apply
    // at the same psi when x is given) in a single pass over psi
    if (x != nullptr) { A.in1 = x; A.wc_out = y; }
    rc = run_small(P->n, P->nq, true, x != nullptr, A, P->stab, s);
    x = nullptr;
  } else {
    rc = P->kind == HPG_OBSTACLE ? run_elem<M_OBST_RES>(P, A, s) : run_elem<M_GRAD_RES>(P, A, s);
  }
  if (rc) return rc;
  if (hat_count(P) > 0) {
    if ((rc = hat_gather(P, A, s))) return rc;
  } else {
    P->last_wc = wcache;     // the psi-side kernel (the cache writer) was the last one
  }
  if (x != nullptr) {
    // Jacobian apply at the same psi (not fused on this path)
    if (P->kind == HPG_OBSTACLE) return hpgObstacleApplyD(P, psi, x, y, stream);
    return hpgGradientApplyD(P, psi, phi, x, y, stream);
  }
  return HPG_OK;
}

int hpgResidual(hpgPlan P, double alpha, const double* psi_prev, const double* u, const double* psi,
                const double* phi, const double* f_load, double* b_u, double* b_psi, int* clamped,
                double* wcache, void* stream) {
  HPG_NVTX("hpgResidual");
  return residual_impl(P, alpha, psi_prev, u, psi, phi, f_load, b_u, b_psi, clamped, wcache, nullptr,
                       nullptr, stream);
}

int hpgResidualApply(hpgPlan P, double alpha, const double* psi_prev, const double* u, const double* psi,
                     const double* phi, const double* f_load, const double* x, double* b_u,
                     double* b_psi, double* y, int* clamped, void* stream) {
  HPG_NVTX("hpgResidualApply");
  if (!x || !y) return fail(HPG_ERR_ARG, "null pointer");
  return residual_impl(P, alpha, psi_prev, u, psi, phi, f_load, b_u, b_psi, clamped, nullptr, x, y,
                       stream);
}

static int blocks_gemm(hpgPlan P, const double* wcache, double* blocks, int c0, int count, cudaStream_t s) {
  int nf = P->kind == HPG_OBSTACLE ? 1 : 3;
  int n2 = P->n * P->n;
  // stage-1 scratch sized for up to 256 MB of Z per pass
  if (P->Z == nullptr || P->zcells < 1) return fail(HPG_ERR_UNSUPPORTED, "block GEMM scratch was not sized for this plan");
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.nfield = nf; g.n = P->n; g.n2 = n2; g.QP = P->QP; g.QT = P->QT; g.NW = nf;
  g.ncy = P->ncy; g.G = P->G; g.wc = wcache; g.Z = P->Z;
  g.nb = (long long)n2 * (P->kind == HPG_OBSTACLE ? 1 : 2);
  g.hx = P->hx; g.hy = P->hy;
  for (int start = c0; start < c0 + count; start += P->zcells) {
    int cnt = c0 + count - start < P->zcells ? c0 + count - start : P->zcells;
    g.cell0 = start;
    g.out = blocks + (size_t)(start - c0) * g.nb * g.nb;
    g.M = n2; g.N = P->QP; g.K = P->QP;
    dim3 g1((n2 + GT - 1) / GT, (P->QP + GT - 1) / GT, cnt * nf);
    k_gemm<0><<<g1, 256, 0, s>>>(g);
    LAUNCH_CHECK();
    g.M = n2; g.N = n2; g.K = P->QP;
    dim3 g2((n2 + GT - 1) / GT, (n2 + GT - 1) / GT, cnt * nf);
    k_gemm<1><<<g2, 256, 0, s>>>(g);
    LAUNCH_CHECK();
  }
  return HPG_OK;
}

static int blocks_impl(hpgPlan P, const double* wcache, double* blocks, int c0, int count, void* stream,
                       int prec, double alpha, double beta) {
  if (int rc = check(P)) return rc;
  if (!wcache || !blocks) return fail(HPG_ERR_ARG, "null pointer");
  if (c0 < 0 || count < 0 || c0 + count > P->N) return fail(HPG_ERR_ARG, "cell range out of bounds");
  if (prec && P->kind == HPG_OBSTACLE && P->nkeys == 0)
    return fail(HPG_ERR_ARG, "hpgPrecondPrepare has not been called on this plan");
  if (count == 0) return HPG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  BArgs B;
  memset(&B, 0, sizeof(B));
  B.prec = prec; B.alpha = alpha; B.beta = beta; B.tri = P->tri; B.key = P->cell_key;
  B.n = P->n; B.NT = P->NT; B.QT = P->QT; B.nq = P->nq;
  B.nf = P->kind == HPG_OBSTACLE ? 1 : 3;
  B.ncy = P->ncy; B.cell0 = c0; B.ncell = count;
  B.G = P->G; B.PKG = P->PKG; B.wc = wcache; B.out = blocks;
  B.nb = (long long)P->n * P->n * (P->kind == HPG_OBSTACLE ? 1 : 2);
  B.hx = P->hx; B.hy = P->hy;
  B.per_warp = 1;
  const int threads = 128;
  int pk_smem = 1;
  size_t smem = blockrow_smem(P, &pk_smem);
  B.pk_smem = pk_smem;
  if (blocks_use_gemm(P)) {
    // large tiles: two-stage GEMM (Z = G W, blocks = Z G^T) through global scratch
    int rc = blocks_gemm(P, wcache, blocks, c0, count, s);
    if (rc || !prec) return rc;
    PrecArgs A;
    memset(&A, 0, sizeof(A));
    A.kind = P->kind; A.n = P->n; A.n2 = P->n * P->n;
    A.nb = A.n2 * (P->kind == HPG_OBSTACLE ? 1 : 2);
    A.ncy = P->ncy; A.cell0 = c0; A.count = count; A.transform = 1;
    A.alpha = alpha; A.beta = beta; A.hx = P->hx; A.hy = P->hy; A.tri = P->tri; A.key = P->cell_key;
    A.M = blocks;
    return launch_precond_transform(A, s);
  }
  void* fn;
  switch (P->NT) {
    case 1: fn = (void*)k_blockrow<1>; break;
    case 2: fn = (void*)k_blockrow<2>; break;
    case 3: fn = (void*)k_blockrow<3>; break;
    case 4: fn = (void*)k_blockrow<4>; break;
    case 5: fn = (void*)k_blockrow<5>; break;
    case 6: fn = (void*)k_blockrow<6>; break;
    case 7: fn = (void*)k_blockrow<7>; break;
    case 8: fn = (void*)k_blockrow<8>; break;
    case 9: fn = (void*)k_blockrow<9>; break;
    case 10: fn = (void*)k_blockrow<10>; break;
    case 11: fn = (void*)k_blockrow<11>; break;
    case 12: fn = (void*)k_blockrow<12>; break;
    default: fn = nullptr;
  }
  // hot shapes with the quadrature tile count at compile time
  if (P->NT == 2 && P->QT == 3) fn = (void*)k_blockrow<2, 3>;        // config 1, Gauss rule
  if (P->NT == 2 && P->QT == 5) fn = (void*)k_blockrow<2, 5>;        // config 1, reference rule
  if (P->NT == 3 && P->QT == 5) fn = (void*)k_blockrow<3, 5>;        // config 2
  if (P->NT == 1 && P->QT == 2) fn = (void*)k_blockrow<1, 2>;        // config 0
  if (fn == nullptr) return fail(HPG_ERR_UNSUPPORTED, "block-row kernel supports n <= 96");
  if (smem > (48u << 10)) CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  const long long items = (long long)count * B.nf * P->n;
  const long long per_cta = B.per_warp ? threads / 32 : 1;
  long long need = (items + per_cta - 1) / per_cta;
  long long cap = (long long)P->nsm * (occ > 0 ? occ : 1);
  int grid = (int)(need < cap ? need : cap);
  void* args[] = {&B};
  CUDA_TRY(cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, s));
  return HPG_OK;
}

int hpgBlocks(hpgPlan P, const double* wcache, double* blocks, int c0, int count, void* stream) {
  HPG_NVTX("hpgBlocks");
  return blocks_impl(P, wcache, blocks, c0, count, stream, 0, 1.0, 0.0);
}

int hpgPrecondAssemble(hpgPlan P, const double* wcache, double alpha, double beta, double* blocks, int c0,
                       int count, void* stream) {
  HPG_NVTX("hpgPrecondAssemble");
  return blocks_impl(P, wcache, blocks, c0, count, stream, 1, alpha, beta);
}

int hpgBlocksMatvec(hpgPlan P, const double* blocks, const double* x, double* y, void* stream) {
  HPG_NVTX("hpgBlocksMatvec");
  if (int rc = check(P)) return rc;
  if (!blocks || !x || !y) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  int nb = P->n * P->n * (P->kind == HPG_OBSTACLE ? 1 : 2);
  size_t smem = sizeof(double) * nb;
  if (smem > 48 * 1024) {
    CUDA_TRY(cudaFuncSetAttribute(k_blocks_matvec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  k_blocks_matvec<<<P->N, 256, smem, (cudaStream_t)stream>>>(A, blocks, nb, 0, x, y);
  LAUNCH_CHECK();
  return HPG_OK;
}

int hpgBTu(hpgPlan P, const double* u, double* out, void* stream) {
  HPG_NVTX("hpgBTu");
  if (int rc = check(P)) return rc;
  if ((!u && P->ndof_u > 0) || !out) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  A.u = u; A.out = out;
  long long total = P->ndof_psi;
  k_btu<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(A, P->kind == HPG_GRADIENT);
  LAUNCH_CHECK();
  return HPG_OK;
}

int hpgBPsi(hpgPlan P, const double* psi, double* out, void* stream) {
  HPG_NVTX("hpgBPsi");
  if (int rc = check(P)) return rc;
  if (P->ndof_u == 0) return HPG_OK;
  if (!psi || !out) return fail(HPG_ERR_ARG, "null pointer");
  UArgs U = base_uargs(P);
  U.psi_a = psi; U.out = out;
  return run_ulocal(P, U, (cudaStream_t)stream);
}

int hpgAu(hpgPlan P, const double* u, double* out, void* stream) {
  HPG_NVTX("hpgAu");
  if (int rc = check(P)) return rc;
  if (P->ndof_u == 0) return HPG_OK;
  if (!u || !out) return fail(HPG_ERR_ARG, "null pointer");
  UArgs U = base_uargs(P);
  U.u = u; U.ca = 1.0; U.out = out;
  return run_ulocal(P, U, (cudaStream_t)stream);
}

int hpgMomentsFromValues(hpgPlan P, const double* vals, double* out, void* stream) {
  HPG_NVTX("hpgMomentsFromValues");
  if (int rc = check(P)) return rc;
  if (!vals || !out) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs A = base_args(P);
  A.in0 = vals; A.out = out;
  A.splits = P->splits;
  return run_mode<M_VALUES>(PATH_CTA, A, (cudaStream_t)stream);
}

int hpgLoadVector(hpgPlan P, const double* vals, double* out, void* stream) {
  HPG_NVTX("hpgLoadVector");
  if (int rc = check(P)) return rc;
  if (P->ndof_u == 0) return HPG_OK;
  if (!vals || !out) return fail(HPG_ERR_ARG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  // U-side moments Mu = wu (x) wu * (Tu F Tu^T) as x-major m-tiles
  ElemArgs A = base_args(P);
  A.n = P->m; A.NT = P->NTu; A.Tf = P->Tuf; A.Sf = P->Suf;
  A.ld = (long long)P->ncy * P->m;
  A.ncomp = (long long)P->ncx * P->m * P->ncy * P->m;
  A.in0 = vals; A.out = P->mu;
  A.splits = P->splits;
  int rc = run_mode<M_VALUES>(PATH_CTA, A, s);
  if (rc) return rc;
  UArgs U = base_uargs(P);
  U.mu = P->mu; U.out = out;
  return run_ulocal(P, U, s);
}

// ---------------------------------------------------------------------------
// Per-cell Schur preconditioner (assembly.py:577-603, 851-860; linalg.py:246-266)

int hpgPrecondPrepare(hpgPlan P, const double* Zhat, const double* lam_hat, void* stream) {
  HPG_NVTX("hpgPrecondPrepare");
  if (int rc = check(P)) return rc;
  if (P->kind != HPG_OBSTACLE) return HPG_OK;   // the gradient blocks need no triple
  if (!Zhat || !lam_hat) return fail(HPG_ERR_ARG, "null triple factors");
  cudaStream_t s = (cudaStream_t)stream;
  // width keys as the reference's _triple_cache (widths rounded to 15 digits,
  // first cell of each key supplies the widths)
  std::vector<long long> kx, ky;
  std::vector<double> khx, khy;
  std::vector<int> key(P->N);
  for (int cx = 0; cx < P->ncx; ++cx)
    for (int cy = 0; cy < P->ncy; ++cy) {
      const long long a = llround(P->hxh[cx] * 1e15), b = llround(P->hyh[cy] * 1e15);
      int k = -1;
      for (size_t i = 0; i < kx.size(); ++i)
        if (kx[i] == a && ky[i] == b) { k = (int)i; break; }
      if (k < 0) {
        k = (int)kx.size();
        kx.push_back(a); ky.push_back(b);
        khx.push_back(P->hxh[cx]); khy.push_back(P->hyh[cy]);
      }
      key[cx * P->ncy + cy] = k;
    }
  const int n = P->n, n2 = n * n, nk = (int)kx.size();
  cudaFree(P->tri); P->tri = nullptr;
  cudaFree(P->cell_key); P->cell_key = nullptr;
  P->nkeys = 0;
  CUDA_TRY(cudaMalloc(&P->tri, sizeof(double) * (size_t)nk * n2 * n2 + 16));
  int rc;
  if ((rc = upload(&P->cell_key, key.data(), key.size()))) return rc;
  double *dZ = nullptr, *dl = nullptr, *dkx = nullptr, *dky = nullptr;
  if ((rc = upload(&dZ, Zhat, (size_t)n2))) return rc;
  if ((rc = upload(&dl, lam_hat, (size_t)n))) return rc;
  if ((rc = upload(&dkx, khx.data(), khx.size()))) return rc;
  if ((rc = upload(&dky, khy.data(), khy.size()))) return rc;
  rc = launch_triple(dZ, dl, n, dkx, dky, nk, P->tri, s);
  cudaStreamSynchronize(s);
  cudaFree(dZ); cudaFree(dl); cudaFree(dkx); cudaFree(dky);
  if (rc) return rc;
  P->nkeys = nk;
  return HPG_OK;
}

// tools only: per-phase cycle counters of the CTA LU (hpgLUProfile)
static unsigned long long* g_lu_prof = nullptr;

static int prec_args(hpgPlan P, double* blocks, int* ipiv, int* perm, int* info, double alpha, double beta,
                     int c0, int count, int transform, PrecArgs* A) {
  if (!blocks) return fail(HPG_ERR_ARG, "null pointer");
  if (c0 < 0 || count < 0 || c0 + count > P->N) return fail(HPG_ERR_ARG, "cell range out of bounds");
  if (transform && P->kind == HPG_OBSTACLE && P->nkeys == 0)
    return fail(HPG_ERR_ARG, "hpgPrecondPrepare has not been called on this plan");
  memset(A, 0, sizeof(*A));
  A->kind = P->kind; A->n = P->n; A->n2 = P->n * P->n;
  A->nb = A->n2 * (P->kind == HPG_OBSTACLE ? 1 : 2);
  A->ncy = P->ncy; A->cell0 = c0; A->count = count; A->transform = transform;
  A->alpha = alpha; A->beta = beta;
  A->hx = P->hx; A->hy = P->hy; A->tri = P->tri; A->key = P->cell_key;
  A->M = blocks; A->ipiv = ipiv; A->info = info; A->perm = perm;
  A->prof = g_lu_prof;
  return HPG_OK;
}

int hpgPrecondBlocks(hpgPlan P, double* blocks, double alpha, double beta, int c0, int count, void* stream) {
  HPG_NVTX("hpgPrecondBlocks");
  if (int rc = check(P)) return rc;
  PrecArgs A;
  if (int rc = prec_args(P, blocks, nullptr, nullptr, nullptr, alpha, beta, c0, count, 1, &A)) return rc;
  if (count == 0) return HPG_OK;
  return launch_precond_transform(A, (cudaStream_t)stream);
}

int hpgLUFactor(hpgPlan P, double* blocks, int* ipiv, int* perm, int count, int* info, void* stream) {
  HPG_NVTX("hpgLUFactor");
  if (int rc = check(P)) return rc;
  PrecArgs A;
  if (int rc = prec_args(P, blocks, ipiv, perm, info, 1.0, 0.0, 0, count, 0, &A)) return rc;
  if (!ipiv) return fail(HPG_ERR_ARG, "null pivot array");
  if (count == 0) return HPG_OK;
  return launch_lu(A, P->nsm, (cudaStream_t)stream);
}

int hpgPrecondFactor(hpgPlan P, double* blocks, int* ipiv, int* perm, double alpha, double beta, int c0,
                     int count, int* info, void* stream) {
  HPG_NVTX("hpgPrecondFactor");
  if (int rc = check(P)) return rc;
  PrecArgs A;
  if (int rc = prec_args(P, blocks, ipiv, perm, info, alpha, beta, c0, count, 1, &A)) return rc;
  if (!ipiv) return fail(HPG_ERR_ARG, "null pivot array");
  if (count == 0) return HPG_OK;
  return launch_lu(A, P->nsm, (cudaStream_t)stream);
}

int hpgLUSolve(hpgPlan P, const double* lu, const int* ipiv, const int* perm, const double* x, double* y,
               void* stream) {
  HPG_NVTX("hpgLUSolve");
  if (int rc = check(P)) return rc;
  if (!lu || !ipiv || !x || !y) return fail(HPG_ERR_ARG, "null pointer");
  ElemArgs E = base_args(P);
  const int nb = P->n * P->n * (P->kind == HPG_OBSTACLE ? 1 : 2);
  return launch_lu_solve(E, lu, ipiv, perm, nb, x, y, (cudaStream_t)stream);
}

int hpgLUMaxBlock(void) {
  // the one-CTA panel LU up to lu_max_nb(), the cluster-panel blocked LU beyond
  int lo = lu_max_nb(), hi = 1 << 16;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (lu_big_supported(mid)) lo = mid; else hi = mid - 1;
  }
  return lo;
}

int hpgLUProfile(unsigned long long* counters) {
  g_lu_prof = counters;
  return HPG_OK;
}

// ---------------------------------------------------------------------------
// Fast-diagonalisation stiffness solve and the Schur operator (linalg.py:100-117, 213-229)

static std::vector<double> transposed(const double* X, int rows, int cols) {
  std::vector<double> t((size_t)rows * cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) t[(size_t)j * rows + i] = X[(size_t)i * cols + j];
  return t;
}

static int fdm_setup(hpgPlan P, int slot, int r, int c, const double* Vx, const double* lx, const double* Vy,
                     const double* ly, double shift) {
  auto& F = P->fdm[slot];
  F.release();
  F.r = r; F.c = c;
  std::vector<double> finv((size_t)r * c);
  for (long long i = 0; i < r; ++i)
    for (long long j = 0; j < c; ++j) finv[(size_t)(i * c + j)] = 1.0 / (lx[i] + ly[j] + shift);
  std::vector<double> vxt = transposed(Vx, r, r), vyt = transposed(Vy, c, c);
  int rc;
  if ((rc = upload(&F.Vx, Vx, (size_t)r * r))) return rc;
  if ((rc = upload(&F.Vy, Vy, (size_t)c * c))) return rc;
  if ((rc = upload(&F.VxT, vxt.data(), vxt.size()))) return rc;
  if ((rc = upload(&F.VyT, vyt.data(), vyt.size()))) return rc;
  if ((rc = upload(&F.finv, finv.data(), finv.size()))) return rc;
  CUDA_TRY(cudaMalloc(&F.w1, sizeof(double) * (size_t)r * c + 16));
  CUDA_TRY(cudaMalloc(&F.w2, sizeof(double) * (size_t)r * c + 16));
  F.ready = true;
  return HPG_OK;
}

int hpgStiffnessFactor(hpgPlan P, const double* Vx, const double* lx, const double* Vy, const double* ly,
                       void* stream) {
  HPG_NVTX("hpgStiffnessFactor");
  if (int rc = check(P)) return rc;
  if (!Vx || !lx || !Vy || !ly) return fail(HPG_ERR_ARG, "null eigen-factors");
  if (P->nix <= 0 || P->niy <= 0) return fail(HPG_ERR_ARG, "mesh has no interior U dofs");
  (void)stream;
  P->fdm_ready = false;
  cudaFree(P->su1); cudaFree(P->su2); cudaFree(P->syD); cudaFree(P->sz);
  P->su1 = P->su2 = P->syD = P->sz = nullptr;
  if (int rc = fdm_setup(P, 0, P->nix, P->niy, Vx, lx, Vy, ly, 0.0)) return rc;
  CUDA_TRY(cudaMalloc(&P->su1, sizeof(double) * P->ndof_u + 16));
  CUDA_TRY(cudaMalloc(&P->su2, sizeof(double) * P->ndof_u + 16));
  CUDA_TRY(cudaMalloc(&P->syD, sizeof(double) * P->ndof_psi + 16));
  CUDA_TRY(cudaMalloc(&P->sz, sizeof(double) * P->ndof_psi + 16));
  P->fdm_ready = true;
  return HPG_OK;
}

// row-major C (M x N) = A (M x K) B (K x N) (.* F), batched with strides
// (stride 0 = operand shared by the batch): k_dgemm_nn, hpg_gemm.cuh
static int gemm(int M, int N, int K, const double* A, long long lda, long long sA, const double* B, long long ldb,
                long long sB, double* C, long long ldc, long long sC, int batch, cudaStream_t s,
                const double* F = nullptr) {
  GemmNN g = gemm_nn(M, N, K, A, lda, B, ldb, C, ldc);
  g.sA = sA; g.sB = sB; g.sC = sC;
  g.F = F; g.sF = 0;
  CUDA_TRY(dgemm_nn(g, batch, s));
  return HPG_OK;
}

// A^{-1} b = Vx [(Vx^T B Vy) ./ (lx + ly)] Vy^T: four GEMMs, the scaling fused
// into the second one's epilogue
static int fdm_solve(hpgPlan P, int slot, const double* b, double* x, cudaStream_t s) {
  auto& F = P->fdm[slot];
  const int r = F.r, c = F.c;
  int rc;
  if ((rc = gemm(r, c, r, F.VxT, r, 0, b, c, 0, F.w1, c, 0, 1, s))) return rc;             // Vx^T B
  if ((rc = gemm(r, c, c, F.w1, c, 0, F.Vy, c, 0, F.w2, c, 0, 1, s, F.finv))) return rc;   // (. Vy) ./ (lx+ly)
  if ((rc = gemm(r, c, r, F.Vx, r, 0, F.w2, c, 0, F.w1, c, 0, 1, s))) return rc;           // Vx .
  return gemm(r, c, c, F.w1, c, 0, F.VyT, c, 0, x, c, 0, 1, s);                           // . Vy^T
}

static int stiffness_solve(hpgPlan P, const double* b, double* x, cudaStream_t s) {
  return fdm_solve(P, 0, b, x, s);
}

int hpgStiffnessSolve(hpgPlan P, const double* b, double* x, void* stream) {
  HPG_NVTX("hpgStiffnessSolve");
  if (int rc = check(P)) return rc;
  if (!P->fdm_ready) return fail(HPG_ERR_ARG, "hpgStiffnessFactor has not been called on this plan");
  if (!b || !x) return fail(HPG_ERR_ARG, "null pointer");
  if (b == x) return fail(HPG_ERR_ARG, "in-place stiffness solve is not supported");
  return stiffness_solve(P, b, x, (cudaStream_t)stream);
}

int hpgSchurApply(hpgPlan P, const double* wcache, double alpha, double beta, const double* x, double* y,
                  void* stream) {
  HPG_NVTX("hpgSchurApply");
  const double* prev_wc = P ? P->last_wc : nullptr;
  if (int rc = check(P)) return rc;
  if (!P->fdm_ready) return fail(HPG_ERR_ARG, "hpgStiffnessFactor has not been called on this plan");
  if (!wcache || !x || !y) return fail(HPG_ERR_ARG, "null pointer");
  if (x == y) return fail(HPG_ERR_ARG, "in-place Schur apply is not supported");
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  P->last_wc = prev_wc;          // the cached apply is this call's first kernel
  if ((rc = hpgApplyCached(P, wcache, x, P->syD, stream))) return rc;   // D x
  if ((rc = hpgBPsi(P, x, P->su1, stream))) return rc;                  // B x
  if ((rc = stiffness_solve(P, P->su1, P->su2, s))) return rc;          // A^{-1} B x
  if ((rc = hpgBTu(P, P->su2, P->sz, stream))) return rc;               // B^T A^{-1} B x
  ElemArgs A = base_args(P);
  const long long total = P->ndof_psi;
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  k_schur_combine<<<grid, 256, 0, s>>>(A, P->kind == HPG_GRADIENT, alpha, beta, x, P->syD, P->sz, y);
  LAUNCH_CHECK();
  return HPG_OK;
}

// ---------------------------------------------------------------------------
// QVI temperature operators on the full U space (qvi.py:35-127)

int hpgUFullSetup(hpgPlan P, double gamma, const double* SR, const double* TR, const double* Kh,
                  const double* Mh, const double* Vx, const double* lx, const double* Vy, const double* ly,
                  void* stream) {
  HPG_NVTX("hpgUFullSetup");
  if (int rc = check(P)) return rc;
  if (!SR || !TR || !Kh || !Mh || !Vx || !lx || !Vy || !ly) return fail(HPG_ERR_ARG, "null table");
  if (P->p < 2) return fail(HPG_ERR_UNSUPPORTED, "full-space U operators need p >= 2");
  (void)stream;
  const int m = P->m, Q = P->nq, N = P->N;
  const int nfx = P->ncx * P->p + 1, nfy = P->ncy * P->p + 1;
  P->q_ready = false;
  double** bufs[] = {&P->qSR, &P->qTR, &P->qK, &P->qM, &P->qC, &P->qT, &P->qV, &P->qG,
                     &P->qP1, &P->qP2, &P->qH1, &P->qH2, &P->qH3, &P->qSRT, &P->qTRT, &P->qKT, &P->qMT};
  for (double** b : bufs) { cudaFree(*b); *b = nullptr; }
  int rc;
  if ((rc = upload(&P->qSR, SR, (size_t)Q * m))) return rc;
  if ((rc = upload(&P->qTR, TR, (size_t)m * Q))) return rc;
  if ((rc = upload(&P->qK, Kh, (size_t)m * m))) return rc;
  if ((rc = upload(&P->qM, Mh, (size_t)m * m))) return rc;
  {
    std::vector<double> srt = transposed(SR, Q, m), trt = transposed(TR, m, Q);
    std::vector<double> kt = transposed(Kh, m, m), mt = transposed(Mh, m, m);
    if ((rc = upload(&P->qSRT, srt.data(), srt.size()))) return rc;
    if ((rc = upload(&P->qTRT, trt.data(), trt.size()))) return rc;
    if ((rc = upload(&P->qKT, kt.data(), kt.size()))) return rc;
    if ((rc = upload(&P->qMT, mt.data(), mt.size()))) return rc;
  }
  const size_t mm = (size_t)N * m * m, qm = (size_t)N * Q * (Q > m ? Q : m), qq = (size_t)N * Q * Q;
  CUDA_TRY(cudaMalloc(&P->qC, sizeof(double) * mm + 16));
  CUDA_TRY(cudaMalloc(&P->qT, sizeof(double) * qm + 16));
  CUDA_TRY(cudaMalloc(&P->qV, sizeof(double) * qq + 16));
  CUDA_TRY(cudaMalloc(&P->qG, sizeof(double) * mm + 16));
  CUDA_TRY(cudaMalloc(&P->qP1, sizeof(double) * mm + 16));
  CUDA_TRY(cudaMalloc(&P->qP2, sizeof(double) * mm + 16));
  CUDA_TRY(cudaMalloc(&P->qH1, sizeof(double) * mm + 16));
  CUDA_TRY(cudaMalloc(&P->qH2, sizeof(double) * mm + 16));
  CUDA_TRY(cudaMalloc(&P->qH3, sizeof(double) * mm + 16));
  if ((rc = fdm_setup(P, 1, nfx, nfy, Vx, lx, Vy, ly, gamma))) return rc;
  P->q_ready = true;
  return HPG_OK;
}

static QArgs qargs(hpgPlan P) {
  QArgs Q;
  Q.ncx = P->ncx; Q.ncy = P->ncy; Q.p = P->p; Q.m = P->m; Q.nq = P->nq; Q.N = P->N;
  Q.nfy = (long long)P->ncy * P->p + 1;
  Q.hx = P->hx; Q.hy = P->hy;
  return Q;
}

static int grid_for(long long n) { long long g = (n + 255) / 256; return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16); }

// V = SR C SR^T for the full vector v (into P->qV); C kept in P->qC
static int q_values(hpgPlan P, const double* v, cudaStream_t s) {
  const int m = P->m, Q = P->nq, N = P->N;
  QArgs A = qargs(P);
  k_qgather<<<grid_for((long long)N * m * m), 256, 0, s>>>(A, v, P->qC);
  LAUNCH_CHECK();
  int rc;
  // T = SR C (Q x m per cell), V = T SR^T (Q x Q per cell)
  if ((rc = gemm(Q, m, m, P->qSR, m, 0, P->qC, m, (long long)m * m, P->qT, m, (long long)Q * m, N, s))) return rc;
  return gemm(Q, Q, m, P->qT, m, (long long)Q * m, P->qSRT, Q, 0, P->qV, Q, (long long)Q * Q, N, s);
}

int hpgUFullValues(hpgPlan P, const double* v, double* vals, void* stream) {
  HPG_NVTX("hpgUFullValues");
  if (int rc = check(P)) return rc;
  if (!P->q_ready) return fail(HPG_ERR_ARG, "hpgUFullSetup has not been called on this plan");
  if (!v || !vals) return fail(HPG_ERR_ARG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (int rc = q_values(P, v, s)) return rc;
  CUDA_TRY(cudaMemcpyAsync(vals, P->qV, sizeof(double) * (size_t)P->N * P->nq * P->nq, cudaMemcpyDeviceToDevice, s));
  return HPG_OK;
}

int hpgUFullOperator(hpgPlan P, double gamma, const double* v, const double* w, const double* rhs, double* out,
                     void* stream) {
  HPG_NVTX("hpgUFullOperator");
  if (int rc = check(P)) return rc;
  if (!P->q_ready) return fail(HPG_ERR_ARG, "hpgUFullSetup has not been called on this plan");
  if (!out) return fail(HPG_ERR_ARG, "null pointer");
  if (w && !v) return fail(HPG_ERR_ARG, "weights given without a vector");
  cudaStream_t s = (cudaStream_t)stream;
  const int m = P->m, Q = P->nq, N = P->N;
  const long long mm = (long long)m * m, qq = (long long)Q * Q;
  int rc;
  if (v) {
    if ((rc = q_values(P, v, s))) return rc;                 // C = tiles(v), V = values(v)
    // H terms: Kh C Mh, Mh C Kh, Mh C Mh
    if ((rc = gemm(m, m, m, P->qK, m, 0, P->qC, m, mm, P->qP1, m, mm, N, s))) return rc;
    if ((rc = gemm(m, m, m, P->qM, m, 0, P->qC, m, mm, P->qP2, m, mm, N, s))) return rc;
    if ((rc = gemm(m, m, m, P->qP1, m, mm, P->qMT, m, 0, P->qH1, m, mm, N, s))) return rc;
    if ((rc = gemm(m, m, m, P->qP2, m, mm, P->qKT, m, 0, P->qH2, m, mm, N, s))) return rc;
    if ((rc = gemm(m, m, m, P->qP2, m, mm, P->qMT, m, 0, P->qH3, m, mm, N, s))) return rc;
  }
  const bool load = w || rhs;
  if (load) {
    k_qpoint<<<grid_for((long long)N * qq), 256, 0, s>>>((long long)N * qq, P->qV, w, rhs);
    LAUNCH_CHECK();
    // G = TR V TR^T per cell
    if ((rc = gemm(m, Q, Q, P->qTR, Q, 0, P->qV, Q, qq, P->qT, Q, (long long)m * Q, N, s))) return rc;
    if ((rc = gemm(m, m, Q, P->qT, Q, (long long)m * Q, P->qTRT, m, 0, P->qG, m, mm, N, s))) return rc;
  }
  QArgs A = qargs(P);
  const long long nfull = ((long long)P->ncx * P->p + 1) * A.nfy;
  k_qscatter<<<grid_for(nfull), 256, 0, s>>>(A, gamma, v ? P->qH1 : nullptr, v ? P->qH2 : nullptr,
                                             v ? P->qH3 : nullptr, load ? P->qG : nullptr, out);
  LAUNCH_CHECK();
  return HPG_OK;
}

int hpgUFullSolve(hpgPlan P, const double* b, double* x, void* stream) {
  HPG_NVTX("hpgUFullSolve");
  if (int rc = check(P)) return rc;
  if (!P->q_ready) return fail(HPG_ERR_ARG, "hpgUFullSetup has not been called on this plan");
  if (!b || !x || b == x) return fail(HPG_ERR_ARG, "bad pointers");
  return fdm_solve(P, 1, b, x, (cudaStream_t)stream);
}

}  // extern "C"
