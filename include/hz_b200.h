/*
 * hz_b200.h -- C ABI of the B200-native multi-RHS Helmholtz solver.
 *
 * Drop-in boundary for the reference's Helmholtz solve path
 * (seistomo, /root/reference/proj/core). Every entry point names the
 * reference interface it replaces (file:line, paths relative to
 * proj/core/). Plain pointers and sizes only: complex arrays are interleaved
 * (re, im) doubles, node-major blocks a[i*k + j] exactly like
 * seistomo::BlockVec<cplx> (include/seistomo/block.hpp:13-27), so reference
 * buffers pass through without transposition.
 *
 * Errors: every function returns an hz_status; hz_last_error_message()
 * returns the thread's last message. Status values map one-to-one to the
 * reference's exception classes (include/seistomo/errors.hpp:10-46).
 * There is no CPU fallback: without a CUDA device every compute entry point
 * fails with HZ_CUDA.
 */
#ifndef HZ_B200_H
#define HZ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HZ_ABI_VERSION 2

#if defined(__GNUC__)
#define HZ_API __attribute__((visibility("default")))
#else
#define HZ_API
#endif

typedef enum hz_status {
  HZ_OK = 0,
  HZ_VALIDATION = 1,    /* seistomo::ValidationError */
  HZ_CONVERGENCE = 2,   /* seistomo::ConvergenceError */
  HZ_BREAKDOWN = 3,     /* seistomo::BreakdownError */
  HZ_FACTORIZATION = 4, /* seistomo::FactorizationError */
  HZ_STATE = 5,         /* seistomo::StateError */
  HZ_IO = 6,            /* seistomo::IoError */
  HZ_CUDA = 7,          /* CUDA runtime / device failure */
  HZ_NCCL = 8           /* collective failure */
} hz_status;

/* include/seistomo/helmholtz_solver.hpp:12 (+ HZ_METHOD_MG_FGMRES: the
 * build_hierarchy + MgHierarchy::cycle + block_fgmres composition with the
 * cycle kind taken from hz_options.cycle_kind). */
typedef enum hz_method {
  HZ_METHOD_MG_BICGSTAB = 0,
  HZ_METHOD_MG_FGMRES_W = 1,
  HZ_METHOD_MG_FGMRES_K = 2,
  HZ_METHOD_DENSE_LU_SMALL = 3,
  HZ_METHOD_MG_FGMRES = 4,
  HZ_METHOD_MG_BICGSTAB_CYCLE = 5 /* BiCGSTAB with hz_options.cycle_kind */
} hz_method;

typedef enum hz_cycle_kind { HZ_CYCLE_V = 0, HZ_CYCLE_W = 1, HZ_CYCLE_K = 2 } hz_cycle_kind;

typedef enum hz_precision { HZ_C128 = 0, HZ_C64 = 1 } hz_precision;

/* HelmholtzSolveOptions (include/seistomo/helmholtz_solver.hpp:14-24) +
 * CycleSpec (include/seistomo/multigrid.hpp:17-23) + B200 fields. */
typedef struct hz_options {
  int method;              /* hz_method; default HZ_METHOD_MG_BICGSTAB */
  double tol;              /* 1e-6 */
  int max_cycles;          /* 200 */
  int nlevels;             /* 3 */
  double shift_factor;     /* 0.2 */
  int cycle_kind;          /* hz_cycle_kind (derived from method unless MG_FGMRES) */
  int pre;                 /* 2 */
  int post;                /* 2 */
  double jacobi_weight;    /* 0.8 */
  int k_inner;             /* 2 */
  int fgmres_restart;      /* 5 */
  int64_t dense_threshold; /* 3000 */
  int precond_precision;   /* hz_precision of the multigrid cycle; HZ_C128 */
  int rhs_block;           /* 0: one Krylov block over all k columns (solve_block,
                              src/helmholtz_solver.cpp:61-79); b > 0: the k columns
                              solved as ceil(k/b) independent blocks of <= b
                              contiguous columns, run concurrently (each equals
                              solve_block on its columns); default 0 */
} hz_options;

/* SolveReport (include/seistomo/krylov.hpp:19-40). Arrays are caller-owned
 * (length k, history_cap); any may be NULL. */
typedef struct hz_report {
  int cycles;
  int qr_factorizations;
  int64_t block_gram_products;
  double wall_s;
  int history_len; /* full length; at most history_cap entries written */
  int* col_cycles;
  double* rel_residual;
  int* converged;
  double* history;
  int history_cap;
} hz_report;

typedef struct hz_problem hz_problem;
typedef struct hz_solver hz_solver;
typedef struct hz_sampling hz_sampling;

HZ_API int hz_abi_version(void);
HZ_API const char* hz_last_error_message(void);
/* number of CUDA devices visible (0 = none; compute calls then fail) */
HZ_API int hz_device_count(void);

/* Fill with the reference defaults (include/seistomo/helmholtz_solver.hpp:14-24). */
HZ_API void hz_options_default(hz_options* opts);

/* HelmholtzProblem(SlownessSquaredModel, omega, AttenuationField, allow_coarse)
 * (include/seistomo/helmholtz.hpp:22-24, src/helmholtz.cpp:16-43) with
 * RegularGrid(ndim, n, h) (include/seistomo/grid.hpp:26-35) and
 * AttenuationField{base = gamma_base, ramp} (include/seistomo/attenuation.hpp:11-22):
 * gamma(omega) = gamma_base + omega * ramp[i]. m and ramp are [n0*n1*n2]
 * doubles, axis 0 fastest. */
HZ_API int hz_problem_create(int ndim, const int64_t n[3], const double h[3], const double* m,
                      double omega, double gamma_base, const double* ramp, int allow_coarse_ppw,
                      int device, hz_problem** out);
/* Same, with the fine-operator stencil: 7 = the reference's 5-point (2D) /
 * 7-point (3D) operator (hz_problem_create); 27 = the compact 27-point 3D
 * operator of BASELINE config 4 (uniform spacing; no reference counterpart:
 * Laplacian as weighted face / edge / corner second differences, mass
 * distributed over the 27 nodes with symmetric averaging, weights fitted to
 * the plane-wave phase velocity by scripts/design_27pt.py; boundary rows
 * truncated like the reference's). The shifted preconditioner operator is the
 * same discretisation with gamma + shift * omega. */
HZ_API int hz_problem_create_ex(int ndim, const int64_t n[3], const double h[3], const double* m, double omega,
                                double gamma_base, const double* ramp, int allow_coarse_ppw, int device,
                                int stencil, hz_problem** out);
HZ_API int hz_problem_destroy(hz_problem* p);
/* HelmholtzProblem::points_per_wavelength (src/helmholtz.cpp:40-43) */
HZ_API int hz_problem_ppw(const hz_problem* p, double* ppw);
HZ_API int64_t hz_problem_num_nodes(const hz_problem* p);

/* HelmholtzProblem::apply_block (src/helmholtz.cpp:71-100): out = A u, host
 * buffers [n][k] complex. */
HZ_API int hz_apply_block(hz_problem* p, int64_t n, int k, const double* u, double* out);
/* same on device buffers (double2*), enqueued on `stream` (cudaStream_t or NULL) */
HZ_API int hz_apply_block_device(hz_problem* p, int64_t n, int k, const void* u_dev, void* out_dev,
                          void* stream);

/* HelmholtzSolver(problem, options) (src/helmholtz_solver.cpp:7-33):
 * builds the shifted-Laplacian Galerkin hierarchy on the problem's device. */
HZ_API int hz_solver_create(hz_problem* p, const hz_options* opts, hz_solver** out);
HZ_API int hz_solver_destroy(hz_solver* s);
/* HelmholtzSolver::set_tolerance (include/seistomo/helmholtz_solver.hpp:46) */
HZ_API int hz_solver_set_tolerance(hz_solver* s, double tol);
/* Slab decomposition of the slow grid axis (config 5; no reference
 * counterpart -- the reference is single-node). Splits every
 * following solve / cycle of `s` over `nparts` parts; part p runs on GPU
 * devices[p] (NULL: all parts on the problem's GPU, as separate streams);
 * devices[0] must be the problem's GPU. Level-0 planes are cut on multiples
 * of 2^(nlevels-1); levels on which a part would own < 2 planes, and the
 * coarsest solve, run on part 0. Block FGMRES methods with V/W cycles only.
 * nparts <= 1 with devices == NULL returns to the single-stream solver. */
HZ_API int hz_solver_set_slabs(hz_solver* s, int nparts, const int* devices);
/* parts, first agglomerated level and planes[l*(nparts+1)+p] = first plane of
 * part p on level l (p = nparts: plane count), up to `cap` entries */
HZ_API int hz_solver_slab_info(const hz_solver* s, int* nparts, int* agg_level, int64_t* planes, int cap);
/* number of per-part VMM chunks (cuMemCreate) the slab spanning vectors have
 * been built from so far in this process; parts on several GPUs always use
 * them, parts on one GPU only with HZ_SLAB_VMM=1 (diagnostic) */
HZ_API int64_t hz_slab_vmm_chunks(void);

/* HelmholtzSolver::solve_block (src/helmholtz_solver.cpp:35-72): host
 * buffers B, X [n][k]; H2D / D2H copies included. Non-convergence is
 * reported in the report (status stays HZ_OK), as in the reference. */
HZ_API int hz_solve_block(hz_solver* s, int64_t n, int k, const double* B, double* X, hz_report* rep);
/* Device-resident variants (double2* on the problem's GPU). The solve runs
 * on the solver's own stream and is ordered after the caller's pending work
 * on `stream` (a cudaStream_t; the _stream variant) or on the legacy default
 * stream (the plain variant): a B written asynchronously on another stream
 * must use the _stream variant with that stream. X is complete on return. */
HZ_API int hz_solve_block_device(hz_solver* s, int64_t n, int k, const void* B_dev, void* X_dev,
                          hz_report* rep);
HZ_API int hz_solve_block_device_stream(hz_solver* s, int64_t n, int k, const void* B_dev, void* X_dev,
                                        hz_report* rep, void* stream);
/* Multi-frequency batching (no reference counterpart -- the
   reference solves one (m, omega) at a time): `count` independent block
   solves, one per solver (each solver owns its hierarchy, stream and Krylov
   workspace, e.g. one per frequency of a frequency-continuation stage), run
   concurrently from one host thread each so their kernels overlap on the GPU.
   Results equal `count` hz_solve_block calls. Solvers must be distinct. The
   first failing solve's status / message is returned. reps may be NULL. */
HZ_API int hz_solve_blocks_multi(int count, hz_solver* const* solvers, const int64_t* n, const int* k,
                                 const double* const* B, double* const* X, hz_report* reps);
HZ_API int hz_solve_blocks_multi_device(int count, hz_solver* const* solvers, const int64_t* n, const int* k,
                                        const void* const* B_dev, void* const* X_dev, hz_report* reps);

/* Block algebra of the Arnoldi step on caller device blocks ([n][k]
 * complex128, current device; synchronous), for kernel-level parity:
 *   hz_block_gram_device:       G_i = X_i^H Y for i < nb, G on the host as nb
 *                               row-major k x k tiles (gram,
 *                               include/seistomo/block.hpp:51-74, batched);
 *   hz_block_add_scaled_device: Y += sum_i X_i C_i, C on the host as nb
 *                               row-major k x k tiles (add_block_scaled,
 *                               include/seistomo/block.hpp:76-88, batched). */
HZ_API int hz_block_gram_device(int64_t n, int k, int nb, const void* const* X_dev, const void* Y_dev, double* G);
HZ_API int hz_block_add_scaled_device(int64_t n, int k, int nb, const void* const* X_dev, const double* C,
                                      void* Y_dev);

/* solve_helmholtz contract (src/helmholtz_solver.cpp:81-93): like
 * hz_solve_block but returns HZ_CONVERGENCE if any column misses tol. */
HZ_API int hz_solve_helmholtz(hz_solver* s, int64_t n, int k, const double* B, double* X,
                       hz_report* rep);

/* One preconditioner application x := cycle(b) from x = 0
 * (out := 0; MgHierarchy::cycle(opts.cycle), src/helmholtz_solver.cpp:65-68). */
HZ_API int hz_cycle(hz_solver* s, int64_t n, int k, const double* b, double* x);
HZ_API int hz_cycle_device(hz_solver* s, int64_t n, int k, const void* b_dev, void* x_dev);
/* ordered after the caller's `stream` (cudaStream_t), see hz_solve_block_device_stream */
HZ_API int hz_cycle_device_stream(hz_solver* s, int64_t n, int k, const void* b_dev, void* x_dev, void* stream);

/* MgHierarchy::coarse_solve (src/multigrid.cpp:114-117) on the coarsest level */
HZ_API int hz_coarse_solve(hz_solver* s, int64_t nc, int k, const double* b, double* x);

/* Hierarchy inspection (MgHierarchy::level, include/seistomo/multigrid.hpp:48-49) */
HZ_API int hz_hierarchy_num_levels(const hz_solver* s, int* nlevels);
HZ_API int hz_hierarchy_level_dims(const hz_solver* s, int level, int64_t dims[3]);
/* level 0: shifted centre [n] ; level >= 1: Galerkin planes [3^ndim][n]
 * with plane s = (dz+1)*9 + (dy+1)*3 + (dx+1) holding A[i][i + offset]. */
HZ_API int hz_hierarchy_level_coefficients(const hz_solver* s, int level, double* out, int64_t count);

/* fwi_sensitivity_output summed over the k columns (src/helmholtz_solver.cpp:103-111):
 * g[i] (+)= sum_s Re(-omega^2 (1 - i gamma_i/omega) U[i][s] L[i][s]). Host buffers. */
HZ_API int hz_sensitivity_accumulate(hz_problem* p, int64_t n, int k, const double* U, const double* L,
                              double* g, int accumulate);
HZ_API int hz_sensitivity_accumulate_device(hz_problem* p, int64_t n, int k, const void* U_dev,
                                     const void* L_dev, double* g_dev, int accumulate,
                                     void* stream);

/* number of this library's kernel launches so far (process-wide) */
HZ_API int64_t hz_kernel_launch_count(void);

/* ---- FWI path either side of the solve ----------------
 * SamplingOperator(AcquisitionGeometry, grid) (inc/acquisition.hpp:30-62,
 * src/acquisition.cpp:33-62): receivers at physical points xyz[r][3] on the
 * problem's grid with the given origin (NULL: 0); multilinear weights over the
 * <= 2^ndim enclosing nodes. ValidationError if a receiver is off the grid. */
HZ_API int hz_sampling_create(const hz_problem* p, const double origin[3], int64_t nrec, const double* xyz,
                              hz_sampling** out);
HZ_API int hz_sampling_destroy(hz_sampling* s);
HZ_API int64_t hz_sampling_num_receivers(const hz_sampling* s);
/* receiver_nodes / receiver_weights (inc/acquisition.hpp:64-65) */
HZ_API int hz_sampling_receiver(const hz_sampling* s, int64_t r, int64_t nodes[8], double weights[8], int* count);
/* SamplingOperator::sample (inc/acquisition.hpp:40-51): D[nrec][k] = P^T U[n][k] */
HZ_API int hz_sample_device(hz_sampling* s, int k, const void* U_dev, void* D_dev, void* stream);
HZ_API int hz_sample(hz_sampling* s, int k, const double* U, double* D);
/* SamplingOperator::sample_adjoint (inc/acquisition.hpp:53-61): U = P D, or
 * P conj(D) when conj != 0; same summation order as the reference */
HZ_API int hz_sample_adjoint_device(hz_sampling* s, int k, const void* D_dev, void* U_dev, int conj, void* stream);
HZ_API int hz_sample_adjoint(hz_sampling* s, int k, const double* D, double* U, int conj);
/* fwi_sensitivity_rhs (src/helmholtz_solver.cpp:95-101) for k fields:
 * R = -w^2 (1 - i gamma/w) U v, v real [n] */
HZ_API int hz_fwi_sensitivity_rhs_device(hz_problem* p, int64_t n, int k, const void* U_dev, const void* v_dev,
                                         void* R_dev, void* stream);
/* fwi_jacobian_vec (src/helmholtz_solver.cpp:113-125) for k stored fields
 * U[n][k] at once (one block solve): D[nrec][k] = P^T A^{-1}(-w^2 gf U v).
 * HZ_CONVERGENCE if the solve misses tol (report still filled). k = 1 is the
 * reference function exactly. */
HZ_API int hz_fwi_jacobian_vec(hz_solver* s, hz_sampling* P, int64_t n, int k, const double* U, const double* v,
                               double* D, hz_report* rep);
HZ_API int hz_fwi_jacobian_vec_device(hz_solver* s, hz_sampling* P, int64_t n, int k, const void* U_dev,
                                      const void* v_dev, void* D_dev, hz_report* rep);
/* fwi_jacobian_transpose_vec (src/helmholtz_solver.cpp:127-139) summed over
 * k sources: g[n] (+)= sum_s Re(-w^2 gf u_s lambda_s), lambda_s = A^{-1} P conj(W_s) */
HZ_API int hz_fwi_jacobian_transpose_vec(hz_solver* s, hz_sampling* P, int64_t n, int k, const double* U,
                                         const double* W, double* g, int accumulate, hz_report* rep);
HZ_API int hz_fwi_jacobian_transpose_vec_device(hz_solver* s, hz_sampling* P, int64_t n, int k, const void* U_dev,
                                                const void* W_dev, double* g_dev, int accumulate, hz_report* rep);

/* ---- wavefield output -----------------------------------
 * WavefieldBatch::append with StoragePrecision::Compact16
 * (src/helmholtz.cpp:137-151) for k columns of X[n][k] on the device:
 * scales[c] = 2^ceil(log2 max|re,im|) (host array), Q = source-major
 * [k][n][2] binary16 (re, im) of X / scale, round-to-nearest-even. */
HZ_API int hz_compact16_device(int64_t n, int k, const void* X_dev, void* Q_dev, double* scales, void* stream);
HZ_API int hz_compact16(int64_t n, int k, const double* X, uint16_t* Q, double* scales);
/* solve_helmholtz(..., Compact16) (src/helmholtz_solver.cpp:81-93): solve,
 * HZ_CONVERGENCE if any column misses tol, then quantise on the device and
 * return only the 4-byte-per-entry compact fields to the host. */
HZ_API int hz_solve_helmholtz_compact16(hz_solver* s, int64_t n, int k, const double* B, uint16_t* Q,
                                        double* scales, hz_report* rep);

/* Per-kernel CUDA-event profiling of this library's launches (measurement
 * support for bench.py): begin clears and enables, end disables, report
 * writes a JSON object {kernel: {count, ms, bytes, flops}} with the summed
 * event durations and ALGORITHMIC bytes / flops; returns the length needed
 * (incl. NUL) or -1. */
HZ_API int hz_profile_begin(void);
HZ_API int hz_profile_end(void);
HZ_API int64_t hz_profile_report(char* buf, int64_t cap);
/* per-launch timeline of the last profiled region: JSON [[name, stream,
 * start_ms, dur_ms, bytes], ...]; same size protocol as hz_profile_report */
HZ_API int64_t hz_profile_trace(char* buf, int64_t cap);
/* Diagnostic (no reference counterpart): the FP64 tensor-pipe (DMMA,
   mma.sync m8n8k4 f64) peak of the current device in TFLOP/s, measured by a
   ~50 ms register-only kernel -- the roofline denominator of the FP64-bound
   Gram / block-update kernels (MEASURED_PEAKS.json has no FP64 figure). */
HZ_API int hz_measure_fp64_peak(double* tflops);


/* ---- seistomo drop-in surface (include/hz_b200.hpp) ---- */

/* CycleSpec (include/seistomo/multigrid.hpp:17-23) */
typedef struct hz_cycle_spec {
  int kind; /* hz_cycle_kind */
  int pre;
  int post;
  double jacobi_weight;
  int k_inner;
} hz_cycle_spec;

/* HelmholtzProblem::mass / gamma_factor (include/seistomo/helmholtz.hpp:33-38):
 * n interleaved complex values, host copy */
HZ_API int hz_problem_mass(const hz_problem* p, double* out);
HZ_API int hz_problem_gamma_factor(const hz_problem* p, double* out);
/* RegularGrid::nearest_node (src/grid.cpp:46-55) of the problem's grid placed
 * at `origin` (NULL: 0): exact half-spacing ties go to the lower index */
HZ_API int hz_problem_nearest_node(const hz_problem* p, const double origin[3], const double x[3], int64_t* node);
/* HelmholtzProblem::point_source (src/helmholtz.cpp:124-132): q[n] (host,
 * interleaved complex) = amplitude / prod(h) at nearest_node(x), 0 elsewhere;
 * HZ_VALIDATION if x is outside the grid (RegularGrid::contains, src/grid.cpp:34-44) */
HZ_API int hz_problem_point_source(const hz_problem* p, const double origin[3], const double x[3], double amp_re,
                                   double amp_im, double* q);
/* k point sources as one device block B[n][k] (column j: source at xyz[3j..],
 * amplitude amp[2j], amp[2j+1]; amp NULL = 1), zero-filled + scattered on `stream` */
HZ_API int hz_point_sources_device(hz_problem* p, const double origin[3], int k, const double* xyz,
                                   const double* amp, void* B_dev, void* stream);
/* HelmholtzProblem::to_csr(shift_factor) (src/helmholtz.cpp:102-122): CSR with
 * int64 row pointers [n+1], int32 columns (ascending per row) and interleaved
 * complex values. rp/ci/v NULL: *nnz receives the size only. */
HZ_API int hz_problem_to_csr(const hz_problem* p, double shift_factor, int64_t* rp, int32_t* ci, double* v,
                             int64_t cap, int64_t* nnz);
/* fwi_sensitivity_rhs (src/helmholtz_solver.cpp:95-101) on host buffers */
HZ_API int hz_fwi_sensitivity_rhs(hz_problem* p, int64_t n, int k, const double* U, const double* v, double* R);
/* MgHierarchy::cycle(spec, b, x) (include/seistomo/multigrid.hpp:53-55): one
 * cycle of the solver's c128 hierarchy updating x in place (x_zero != 0:
 * x := 0 first, the preconditioner case) */
HZ_API int hz_hierarchy_cycle(hz_solver* s, const hz_cycle_spec* spec, int64_t n, int k, const double* b,
                              double* x, int x_zero);
/* block_fgmres(op, B, restart, tol, max_cycles) (method 0, src/krylov.cpp:178-280)
 * or block_bicgstab(op, B, tol, max_cycles) (method 1, src/krylov.cpp:60-176)
 * with op = {HelmholtzProblem::apply_block, out := 0; MgHierarchy::cycle(spec)}
 * (the SURVEY §3.3 composition) on the solver's hierarchy, one block over
 * all k columns. Non-convergence is reported, not an error. */
HZ_API int hz_block_krylov(hz_solver* s, int method, const hz_cycle_spec* spec, int restart, double tol,
                           int max_cycles, int64_t n, int k, const double* B, double* X, hz_report* rep);

#ifdef __cplusplus
}
#endif

#endif /* HZ_B200_H */
