/*
 * hpg_b200.h -- C ABI of the B200 (sm_100a) element-quadrature engine for the
 * hierarchical proximal Galerkin (hpG) LVPP saddle system.
 *
 * The reference (pure Python, /root/reference/pkg/src/hpgalerkin) has no FFI;
 * its seam is duck typing on the `disc` object.  Each entry point below
 * replaces one reference callable; the Python host
 * (paper_2412_13733_b200/disc.py) binds them with ctypes and keeps the
 * reference's method names, argument meaning and return arrays.
 *
 * Conventions
 *  - All array pointers are caller-owned DEVICE memory (fp64 unless stated);
 *    `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *  - psi-side vectors are in the reference's GLOBAL order: the x-major tensor
 *    order of PsiSpace2D (spaces.py:212-214), i.e. a (ncx*n) x (ncy*n)
 *    row-major array; gradient vectors stack [psi_x ; psi_y]
 *    (assembly.py:744-745).
 *  - u-side vectors are interior U coefficients (spaces.py:188-189): a
 *    (nix x niy) row-major array, nix = ncx*p - 1.  When the mesh has no
 *    interior U dof (gradient p = 1 on one cell row), u-side pointers may be
 *    NULL.
 *  - Cell order (blocks, point samples) is (cx, cy) cx-major
 *    (assembly.py:482).  Point samples are (ncells, nq, nq) row-major.
 *  - Every call returns 0 on success, a nonzero HPG_ERR_* code otherwise;
 *    hpgLastError() gives a message.  Calls are asynchronous on `stream`.
 *  - Clamp flags (`clamped`) are device ints; the call ORs 1 into *clamped
 *    when exp(-v) overflows the reference's clamp (assembly.py:187-192);
 *    the caller zeroes it.
 *  - Concurrency: a plan owns device scratch (U-side edge contributions,
 *    split partials, Schur / fast-diagonalisation work vectors, QVI tiles)
 *    that its entry points overwrite.  A plan is therefore NOT re-entrant:
 *    issue its calls on one stream at a time (or order the streams with
 *    events); use one plan per concurrent stream.  Distinct plans are
 *    independent.  The host-side launch caches are per device and locked,
 *    so plans may be created and used from several host threads and devices.
 *  - Allocation: hpgPlanCreate sizes every workspace of the hot entry points
 *    (moments, applies, residuals, blocks, preconditioner factor / solve);
 *    the one-time setups hpgPrecondPrepare, hpgStiffnessFactor and
 *    hpgUFullSetup allocate their own tables.
 */
#ifndef HPG_B200_H
#define HPG_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define HPG_OK 0
#define HPG_ERR_ARG 1
#define HPG_ERR_CUDA 2
#define HPG_ERR_UNSUPPORTED 3

#define HPG_OBSTACLE 0
#define HPG_GRADIENT 1

typedef struct hpgPlan_st* hpgPlan;

/* Tables + mesh geometry of one uniform-degree discretisation.
 * Replaces the per-cell CellKernel2D construction (assembly.py:232-238,
 * 483-488 / 736-741).  S: nq x n, T: n x nq (psi side), Su: nq x (p+1),
 * Tu: (p+1) x nq (u side), hx: ncx widths, hy: ncy widths -- HOST arrays,
 * copied.  n = p-1 (obstacle) or p (gradient). */
int hpgPlanCreate(hpgPlan* plan, int kind, int ncx, int ncy, int p, int nq,
                  const double* S, const double* T, const double* Su,
                  const double* Tu, const double* hx, const double* hy);
int hpgPlanDestroy(hpgPlan plan);
/* info[0..11] = n, m, nq, ncells, ndof_psi, ndof_u, wcache_doubles,
 *               block_doubles_per_cell, path(0 warp, 1 cta, 2 row-split), splits,
 *               kernels per hpgResidualApply call (1: single-pass path),
 *               1 if hpgResidualApply fuses the apply into the residual pass.
 * info must hold at least 12 entries. */
int hpgPlanInfo(hpgPlan plan, long long* info);

/* ObstacleDisc2D.exp_moments (assembly.py:541-548).  out[ndof_psi].
 * wcache (nullable, info[6] doubles): the clamped exp weights, consumed by
 * hpgApplyCached / hpgBlocks*. */
int hpgObstacleMoments(hpgPlan plan, const double* psi, double* out,
                       int* clamped, double* wcache, void* stream);
/* ObstacleDisc2D.apply_D (assembly.py:559-567): y = D(psi) x. */
int hpgObstacleApplyD(hpgPlan plan, const double* psi, const double* x,
                      double* y, void* stream);
/* GradientDisc2D.nl_moments (assembly.py:781-791); phi: point samples. */
int hpgGradientMoments(hpgPlan plan, const double* psi, const double* phi,
                       double* out, double* wcache, void* stream);
/* GradientDisc2D.apply_D (assembly.py:817-832). */
int hpgGradientApplyD(hpgPlan plan, const double* psi, const double* phi,
                      const double* x, double* y, void* stream);
/* Jacobian action from cached point weights (written by a moments/residual
 * call at the same psi): equals apply_D and CellBlockMatrix @ x
 * (assembly.py:281-285) for the D of that psi. */
int hpgApplyCached(hpgPlan plan, const double* wcache, const double* x,
                   double* y, void* stream);
/* The same action restricted to the cells [cell_begin, cell_end) in x-major
 * cell order (cell = cx * ncy + cy): reads / writes only those cells' tiles
 * of x / y (full-length vectors).  D is block diagonal over cells
 * (assembly.py:272-285, spaces.py:89-108), so a host-buffer caller pipelines
 * slabs of cell columns (contiguous row ranges): upload, apply, download.
 * HPG_ERR_UNSUPPORTED unless the plan applies cached weights on its
 * warp-per-cell path (hpgPlanInfo path 0). */
int hpgApplyCachedRange(hpgPlan plan, const double* wcache, const double* x,
                        double* y, int cell_begin, int cell_end, void* stream);
/* One slab of CellBlockMatrix @ x (assembly.py:281-285) with HOST buffers,
 * the cell columns [cx_begin, cx_end): uploads the slab's rows of x from the
 * page-locked `stage` (the slab's rows only, component after component) into
 * the device vector dev_x on copy_stream, applies D on `stream` after the
 * upload (hpgApplyCachedRange), and downloads the slab's rows of dev_y into
 * the page-locked full-length y_host on `stream`.  Nothing waits on the
 * host: the caller fills the next slab's stage buffer meanwhile and
 * synchronises `stream` after the last slab. */
int hpgApplyCachedHostSlab(hpgPlan plan, const double* wcache, const double* stage,
                           double* dev_x, double* dev_y, double* y_host,
                           int cx_begin, int cx_end, void* copy_stream, void* stream);

/* proximal.residual (proximal.py:112-126), fused:
 *   b_u   = alpha f_load + B psi_prev - alpha A u - B psi
 *   b_psi = phi_moments - B^T u - exp_moments(psi)      (obstacle)
 *         = nl_moments(psi) - B^T u                     (gradient)
 * phi = phi_moments [ndof_psi] (obstacle) or point samples (gradient). */
int hpgResidual(hpgPlan plan, double alpha, const double* psi_prev,
                const double* u, const double* psi, const double* phi,
                const double* f_load, double* b_u, double* b_psi,
                int* clamped, double* wcache, void* stream);

/* Residual plus the Jacobian apply y = D(psi) x at the same psi (the Newton
 * step's residual and first Krylov matvec), sharing one pass over psi on the
 * low-degree path.  Same arguments as hpgResidual plus x and y. */
int hpgResidualApply(hpgPlan plan, double alpha, const double* psi_prev,
                     const double* u, const double* psi, const double* phi,
                     const double* f_load, const double* x, double* b_u,
                     double* b_psi, double* y, int* clamped, void* stream);

/* Element blocks (assembly.py:550-557 / 804-815) from cached weights:
 * blocks[ncells][nb][nb], nb = n^2 (obstacle) or 2 n^2 (gradient),
 * row = a*n+b (test), col = j*n+k (trial).  Cells [c0, c0+count). */
int hpgBlocks(hpgPlan plan, const double* wcache, double* blocks, int c0,
              int count, void* stream);
/* CellBlockMatrix.matvec (assembly.py:281-285) on device blocks. */
int hpgBlocksMatvec(hpgPlan plan, const double* blocks, const double* x,
                    double* y, void* stream);

/* Exact u-side couplings (assembly.py:81-116, 470-477, 725-729). */
int hpgBTu(hpgPlan plan, const double* u, double* out, void* stream);
int hpgBPsi(hpgPlan plan, const double* psi, double* out, void* stream);
int hpgAu(hpgPlan plan, const double* u, double* out, void* stream);

/* Data terms from point samples (ncells, nq, nq):
 * moments_from_values / data_moments (assembly.py:514-533) and
 * load_vector (assembly.py:502-512). */
int hpgMomentsFromValues(hpgPlan plan, const double* vals, double* out,
                         void* stream);
int hpgLoadVector(hpgPlan plan, const double* vals, double* out, void* stream);

/* Per-cell Schur preconditioner.
 *
 * hpgPrecondPrepare replaces ObstacleDisc2D.schur_hat_triple
 * (assembly.py:577-595): builds, per distinct (hx, hy) width key, the triple
 * Bhat^T Ahat^{-1} Bhat from the reference-cell eigen-factors of
 * Ahat = Kx(x)My + Mx(x)Ky: Zhat (n x n, row-major) = Ghat^T Khat^{-1/2} V and
 * lam_hat (n) with Khat^{-1/2} Mhat Khat^{-1/2} = V diag(lam_hat) V^T
 * (tables.py: schur_triple_factors).  No-op for gradient plans.
 *
 * hpgPrecondBlocks: in place, D blocks -> precond_blocks(D, alpha, beta)
 * (assembly.py:597-603 obstacle, :851-860 gradient) for cells [c0, c0+count).
 * hpgLUFactor: batched LU with partial pivoting, in place (scipy lu_factor,
 * linalg.py:249), ipiv[count][nb] 0-based like lu_factor's piv; `info`
 * (device int, may be NULL) is OR-ed with 1 if an entry is non-finite (scipy's
 * check_finite raises ValueError there) and 2 on an exactly zero pivot
 * (LAPACK info > 0; scipy warns).
 * `perm` (nullable, [count][nb]) also receives the composed interchanges
 * (position i <- row perm[i]), which lets the solve gather instead of
 * replaying the swaps.
 * hpgPrecondFactor: both, fused (blocks hold D on entry, LU of P on exit).
 * hpgLUSolve: CellBlockPreconditioner.apply (linalg.py:253-257):
 * y[idx_e] = lu_solve(LU_e, x[idx_e]) for every cell (perm nullable).
 * hpgLUMaxBlock: largest block side the factorisation supports (one CTA per
 * block up to ~3k, beyond that -- config 3's 6561^2 -- a blocked LU with
 * 32-column panels held in the distributed shared memory of an 8-CTA cluster
 * per block and batched DMMA trailing updates). */
int hpgPrecondPrepare(hpgPlan plan, const double* Zhat, const double* lam_hat,
                      void* stream);
int hpgPrecondBlocks(hpgPlan plan, double* blocks, double alpha, double beta,
                     int c0, int count, void* stream);
/* precond_blocks straight from the cached point weights of D (the blocks
 * kernel's epilogue writes P_e instead of D_e; same layout as hpgBlocks). */
int hpgPrecondAssemble(hpgPlan plan, const double* wcache, double alpha,
                       double beta, double* blocks, int c0, int count,
                       void* stream);
int hpgLUFactor(hpgPlan plan, double* blocks, int* ipiv, int* perm, int count,
                int* info, void* stream);
int hpgPrecondFactor(hpgPlan plan, double* blocks, int* ipiv, int* perm,
                     double alpha, double beta, int c0, int count, int* info,
                     void* stream);
int hpgLUSolve(hpgPlan plan, const double* lu, const int* ipiv,
               const int* perm, const double* x, double* y, void* stream);
int hpgLUMaxBlock(void);
/* Tuning aid: device array of 8 cycle counters the CTA LU accumulates per
 * phase into (NULL disables; off by default). */
int hpgLUProfile(unsigned long long* counters);

/* Interior stiffness solve by fast diagonalisation (
 * replaces linalg.factor_stiffness / SpluFactor.solve, linalg.py:100-117, for
 * A = Kx(x)My + Mx(x)Ky, assembly.py:42-78, 470-474).  HOST inputs: the 1D
 * generalized eigenpairs Kx Vx = Mx Vx diag(lx), Vx^T Mx Vx = I (nix x nix
 * row-major, nix) and the same in y (schur.py: u_matrices_1d + eigh).
 * hpgStiffnessSolve: x = A^{-1} b on interior U vectors (four DGEMMs on the
 * FP64 tensor cores, the library's own k_dgemm_nn).
 * hpgSchurApply: SchurOperator.matvec (linalg.py:223-229) in one call,
 *   y = -((D x + E_beta x) + B^T A^{-1} B x / alpha), D from cached weights. */
int hpgStiffnessFactor(hpgPlan plan, const double* Vx, const double* lx,
                       const double* Vy, const double* ly, void* stream);
int hpgStiffnessSolve(hpgPlan plan, const double* b, double* x, void* stream);
int hpgSchurApply(hpgPlan plan, const double* wcache, double alpha,
                  double beta, const double* x, double* y, void* stream);

/* QVI temperature operators on the FULL U space (
 * qvi.py:35-127: _cell_grid_values, _load_full, TemperatureSolver).
 * hpgUFullSetup (HOST tables): SR = Su R (nq x m), TR = R^T diag(1/(2l+1)) Tu
 *   (m x nq), Kh / Mh reference-cell stiffness and mass (m x m), and the 1D
 *   generalized eigenpairs of the full-space stiffness/mass (for H^{-1}).
 * hpgUFullValues: per-cell (nq x nq) samples of a full U vector.
 * hpgUFullOperator: out = H v - load(w .* values(v) + rhs),
 *   H = Kx(x)My + Mx(x)Ky + gamma Mx(x)My; v, w, rhs nullable (0): the
 *   Newton residual (w = NULL, rhs = g(gap)) or the Jacobian (rhs = NULL).
 * hpgUFullSolve: x = H^{-1} b (fast diagonalisation; the reference factors H
 *   with SuperLU and uses it as the left preconditioner). */
int hpgUFullSetup(hpgPlan plan, double gamma, const double* SR, const double* TR,
                  const double* Kh, const double* Mh, const double* Vx,
                  const double* lx, const double* Vy, const double* ly,
                  void* stream);
int hpgUFullValues(hpgPlan plan, const double* v, double* vals, void* stream);
int hpgUFullOperator(hpgPlan plan, double gamma, const double* v,
                     const double* w, const double* rhs, double* out,
                     void* stream);
int hpgUFullSolve(hpgPlan plan, const double* b, double* x, void* stream);

/* Device GMRES (replaces linalg.gmres,
 * linalg.py:134-207): unrestarted, Givens-rotated, the reference's stopping
 * rule (relative to the initial residual in the minimised norm) and happy-
 * breakdown test; CGS2 orthogonalisation.  The whole iteration is one CUDA
 * graph with a device-side WHILE node: no host synchronisation per iteration
 * and no operator application after convergence.
 *
 *   hpgGmresCreate(&g, n, maxiter)   Krylov basis + state (device)
 *   hpgGmresBind(g, r, vin, w)       caller-owned device vectors of length n:
 *       r = initial residual (already preconditioned for left
 *       preconditioning; read by every solve), vin = input of the operator
 *       chain, w = its output.  Rebinding drops the captured loop.
 *   hpgGmresCaptureBegin(g, stream) ... the caller enqueues its operator
 *       chain vin -> w on `stream` (right: w = A M vin, left: w = M A vin);
 *       every call must be capturable (no synchronisation, no allocation) ...
 *   hpgGmresCaptureEnd(g, stream)    appends the Arnoldi / Givens kernels
 *   hpgGmresSolve(g, rtol, atol, dx, stream)
 *       runs the loop on r and writes dx = V_k y_k (the caller applies M to
 *       dx for right preconditioning and adds x0)
 *   hpgGmresStatus(g, &iters, &converged, residuals[iters+1], stream)
 *       synchronises `stream` and reports the last solve.
 * `stream` must not be the legacy default stream (it is captured). */
typedef struct hpgGmres_st* hpgGmres;
int hpgGmresCreate(hpgGmres* g, long long n, int maxiter);
int hpgGmresDestroy(hpgGmres g);
int hpgGmresBind(hpgGmres g, const double* r, double* vin, double* w);
int hpgGmresCaptureBegin(hpgGmres g, void* stream);
int hpgGmresCaptureEnd(hpgGmres g, void* stream);
int hpgGmresSolve(hpgGmres g, double rtol, double atol, double* dx, void* stream);
int hpgGmresStatus(hpgGmres g, int* iters, int* converged, double* residuals, void* stream);
/* out = a x + b y on device vectors (x or y may be NULL when its factor is 0). */
int hpgAxpby(long long n, double a, const double* x, double b, const double* y, double* out, void* stream);

const char* hpgLastError(void);
int hpgVersion(void);

#ifdef __cplusplus
}
#endif
#endif
