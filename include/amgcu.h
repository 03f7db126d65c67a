/* amgcu — C ABI of the B200-native root-node AMG core (libamgcu.so).
 *
 * The reference (arxiv/paper_1610_03154, /root/reference/proj/include/amg) is a
 * header-only C++ library with no FFI; its drop-in boundary is the C++ API
 *   amg::setup / amg::rn_setup   (hierarchy.hpp:252-287, 551-559)
 *   amg::solve / amg::cycle      (cycle.hpp:100-107, 114-271)
 * plus the option/report structs they take.  This header is the C ABI that a
 * binding of that API (ctypes, cgo, JNI, or the inline C++ wrapper in
 * include/amg_b200.hpp) calls.  Every entry point is extern "C", takes plain
 * pointers and sizes, and returns an amgcu_status; amgcu_last_error() carries
 * the message.  Status codes map 1:1 onto the reference's exception types
 * (SURVEY.md §8(b)):
 *   AMGCU_INVALID_ARGUMENT -> std::invalid_argument (shape/option misuse)
 *   AMGCU_RUNTIME_ERROR    -> std::runtime_error    (numerical faults, row index in message)
 *   AMGCU_LOGIC_ERROR      -> std::logic_error
 * Divergence / non-convergence / stagnation are flags in the reports, as in
 * the reference (cycle.hpp:29-30, hierarchy.hpp:86).
 *
 * Matrices cross the boundary as canonical CSR (int32 row offsets / column
 * indices, fp64 values, sorted columns, no stored zeros — sparse.hpp:21-62).
 * Pointers are HOST pointers unless the function name ends in _device.
 * Outputs of variable size are returned in library-allocated amgcu_csr /
 * buffers released with amgcu_csr_free / amgcu_free.
 */
#ifndef AMGCU_H
#define AMGCU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AMGCU_OK = 0,
    AMGCU_INVALID_ARGUMENT = 1,
    AMGCU_RUNTIME_ERROR = 2,
    AMGCU_LOGIC_ERROR = 3,
    AMGCU_CUDA_ERROR = 4,
    AMGCU_NO_DEVICE = 5,
    AMGCU_INTERNAL = 9
} amgcu_status;

/* Canonical CSR (sparse.hpp:25-62 SparseMatrix).  block_size tags nodal
 * blocks of block_size DOFs (it does not change the storage). */
typedef struct {
    int32_t n_rows;
    int32_t n_cols;
    int32_t nnz;
    int32_t block_size;
    int32_t* row_offsets; /* n_rows + 1 */
    int32_t* col_indices; /* nnz */
    double* values;       /* nnz */
} amgcu_csr;

/* SetupOptions (hierarchy.hpp:26-36) with StrengthConfig (strength.hpp:18-25),
 * InterpConfig/FilterRule (interpolation.hpp:21-32) and RelaxConfig
 * (relaxation.hpp:20-24) flattened.  Enum values follow the reference order. */
typedef struct {
    int32_t method;           /* SetupMethod: 0 rn, 1 sa, 2 cf (only rn on the GPU path) */
    int32_t strength_measure; /* StrengthMeasure: 0 classical, 1 symmetric, 2 evolution */
    double drop_tol;
    int32_t evolution_steps;
    int32_t weighting; /* EvolutionWeighting: 0 spectral, 1 l1jacobi */
    int32_t degree;
    int32_t prefilter_set;        /* std::optional<FilterRule> engaged */
    int32_t prefilter_theta_set;
    double prefilter_theta;
    int32_t prefilter_k; /* <= 0: unset */
    int32_t postfilter_set;
    int32_t postfilter_theta_set;
    double postfilter_theta;
    int32_t postfilter_k;
    int32_t energy_iters; /* 0: ceil(1.5 * degree) */
    int32_t krylov;       /* KrylovKind: 0 cg, 1 gmres */
    int32_t pre_scheme;   /* RelaxScheme: 0 jacobi, 1 gauss_seidel, 2 sym_gauss_seidel, 3 gsne, 4 block_sym_gauss_seidel */
    double pre_weight;
    int32_t pre_sweeps;
    int32_t post_scheme;
    double post_weight;
    int32_t post_sweeps;
    int32_t max_size;
    int32_t max_levels;
    int32_t candidate_sweeps;
    int32_t cand_scheme;
    double cand_weight;
    int32_t cand_sweeps;
} amgcu_setup_options;

/* SolveOptions (cycle.hpp:19-24). */
typedef struct {
    int32_t method; /* SolveMethod: 0 stationary, 1 pcg, 2 fgmres */
    int32_t cycle;  /* CycleKind: 0 V, 1 W */
    double tol;
    int32_t max_iters;
} amgcu_solve_options;

/* SolveReport (cycle.hpp:26-36); residual_history is returned separately. */
typedef struct {
    int32_t iterations;
    int32_t converged;
    int32_t diverged;
    int32_t history_len;
    double rho;
    double chi_oc;
    double chi_cc;
    double work_units_solve;
    double work_units_setup;
} amgcu_solve_report;

/* StrengthConfig alone (strength kernels exposed for parity tests). */
typedef struct {
    int32_t measure;
    double drop_tol;
    int32_t evolution_steps;
    int32_t weighting;
} amgcu_strength_config;

typedef struct amgcu_ctx_s* amgcu_ctx;
typedef struct amgcu_hier_s* amgcu_hier;

/* ---- context ------------------------------------------------------------ */
amgcu_status amgcu_ctx_create(int device, amgcu_ctx* out);
amgcu_status amgcu_ctx_destroy(amgcu_ctx ctx);
/* Message of the last failed call on this context (or of the last failed
 * amgcu_ctx_create when ctx is NULL). */
const char* amgcu_last_error(amgcu_ctx ctx);
/* 1 (default): every global reduction (dots, norms, the Arnoldi Gram-Schmidt, the
 * energy-min and Krylov scalars) is the reference's left-to-right sum from +0.0,
 * bit for bit (sparse.hpp:309-313), evaluated in parallel by csrc/seqsum.cu.
 * 0: deterministic parallel two-stage trees (reproducible, not the reference's bits). */
amgcu_status amgcu_ctx_set_sequential_reductions(amgcu_ctx ctx, int on);
/* 1 (default): forward Gauss-Seidel candidate improvement runs on a second stream,
 * overlapping the level's strength / aggregation / pattern work; 0: in order.  The
 * result is bitwise the same either way. */
amgcu_status amgcu_ctx_set_candidate_overlap(amgcu_ctx ctx, int on);
/* Energy-minimisation masked product (interpolation.hpp:186-210): levels of at least
 * min_rows rows (default 0: all) use the band-staged kernel -- per-CTA pieces of X and
 * the per-entry match records brought into shared memory by TMA bulk copies (levels
 * whose referenced rows are too scattered to stage gather X from L2 instead); levels
 * its plan refuses (pattern rows above 24 slots, above 16 when scattered) use the
 * register-merge kernel.  min_rows < 0: never.  The result is bitwise the same either
 * way. */
amgcu_status amgcu_ctx_set_masked_band(amgcu_ctx ctx, int32_t min_rows);
/* Levels whose plan was accepted / refused so far, and the last refusal's reason bits
 * (1 referenced rows beyond the window, 2 too many runs, 4 stage beyond 16-bit offsets,
 * 8 a pattern row above 24 slots, 64 shared-memory budget). */
amgcu_status amgcu_ctx_masked_band_stats(amgcu_ctx ctx, int64_t* accepted, int64_t* refused, int32_t* last_fail);
/* Synchronise the context stream; returns the accumulated device time of the
 * kernels launched since the last reset (CUDA events on the context stream). */
amgcu_status amgcu_ctx_synchronize(amgcu_ctx ctx);
/* Kernel launch counter (all kernels this library launched on the context). */
amgcu_status amgcu_ctx_launch_count(amgcu_ctx ctx, int64_t* launches);
/* Host synchronisation counter (stream syncs the library performed on the context). */
amgcu_status amgcu_ctx_sync_count(amgcu_ctx ctx, int64_t* syncs);
/* Device timer on the context stream: CUDA events recorded at start and stop
 * (the stop call synchronises).  Used by bench.py for device-side timing. */
amgcu_status amgcu_ctx_timer_start(amgcu_ctx ctx);
amgcu_status amgcu_ctx_timer_stop(amgcu_ctx ctx, double* ms);
/* Per-kernel-family profiling (CUDA events around each launch of the family,
 * plus its algorithmic bytes = compulsory I/O of that launch). */
amgcu_status amgcu_ctx_set_profiling(amgcu_ctx ctx, int on);
amgcu_status amgcu_ctx_set_profile_mask(amgcu_ctx ctx, uint32_t family_mask);
amgcu_status amgcu_ctx_profile_reset(amgcu_ctx ctx);
amgcu_status amgcu_ctx_profile_query(amgcu_ctx ctx, int32_t family, int64_t* launches, double* ms, double* bytes);
int32_t amgcu_profile_family_count(void);
const char* amgcu_profile_family_name(int32_t family);
void amgcu_free(void* p);
void amgcu_csr_free(amgcu_csr* m);

/* ---- setup / solve (the drop-in path) ------------------------------------ */
/* amg::setup(A, B, opts, left) — hierarchy.hpp:551-559 (rn_setup 252-287).
 * B is n x k column-major (CandidateSet, dense.hpp:15-32); left may be NULL. */
amgcu_status amgcu_setup(amgcu_ctx ctx, const amgcu_csr* A, int32_t k, const double* B,
                         const double* left, const amgcu_setup_options* opts, amgcu_hier* out);
/* Same, with A / B / left already resident in device memory. */
amgcu_status amgcu_setup_device(amgcu_ctx ctx, const amgcu_csr* A_dev, int32_t k, const double* B_dev,
                                const double* left_dev, const amgcu_setup_options* opts, amgcu_hier* out);
amgcu_status amgcu_hier_destroy(amgcu_hier h);
amgcu_status amgcu_hier_levels(amgcu_hier h, int32_t* n_levels, int32_t* stagnated);
/* which: 0 A, 1 P, 2 R (Level, hierarchy.hpp:38-48) -> host copy */
amgcu_status amgcu_hier_get_matrix(amgcu_hier h, int32_t level, int32_t which, amgcu_csr* out);
/* which: 0 B, 1 Bc -> n, k and a host copy (column-major) */
amgcu_status amgcu_hier_get_candidates(amgcu_hier h, int32_t level, int32_t which, int32_t* n, int32_t* k,
                                       double** data);
amgcu_status amgcu_hier_level_symmetric(amgcu_hier h, int32_t level, int32_t* symmetric);
/* Jacobi weights of the pre/post workspaces (relaxation.hpp:52-54) */
amgcu_status amgcu_hier_relax_weights(amgcu_hier h, int32_t level, double* pre, double* post);
/* chi_OC / chi_CC (complexity.hpp:15-36) */
amgcu_status amgcu_hier_complexity(amgcu_hier h, double* chi_oc, double* chi_cc);
/* WorkLedger work units (work.hpp:38-67): wu5 = {aggregation, candidates, interpolation,
 * RAP, solve (finalize + every solve so far)}, each as op counts / nnz(A_0).  The
 * evolution-SOC count is taken on the first call (one counting pass per level). */
amgcu_status amgcu_hier_ledger(amgcu_hier h, double* wu5);

/* amg::solve(h, b, x, opts) — cycle.hpp:114-271.  x is in/out (n doubles;
 * used as the initial guess).  history receives up to history_cap residual
 * norms (report->history_len gives the full count). */
amgcu_status amgcu_solve(amgcu_hier h, const double* b, double* x, const amgcu_solve_options* opts,
                         amgcu_solve_report* report, double* history, int32_t history_cap);
amgcu_status amgcu_solve_device(amgcu_hier h, const double* b_dev, double* x_dev,
                                const amgcu_solve_options* opts, amgcu_solve_report* report, double* history,
                                int32_t history_cap);
/* amg::cycle(h, x, b, kind) — cycle.hpp:100-107 (host x in/out). */
amgcu_status amgcu_cycle(amgcu_hier h, double* x, const double* b, int32_t kind);

/* ---- kernel-level entry points (each one reference function; host in/out) */
amgcu_status amgcu_spmv(amgcu_ctx ctx, const amgcu_csr* A, const double* x, double* y);      /* sparse.hpp:141 */
/* dot(x, y) (take_sqrt = 0) or norm2(x) = sqrt(dot(x, x)) (take_sqrt = 1, y ignored):
   sparse.hpp:309-315.  In the default context mode the sum is the reference's
   left-to-right chain bit for bit (csrc/seqsum.cu); with sequential reductions off it
   is a deterministic tree. */
amgcu_status amgcu_dot(amgcu_ctx ctx, const double* x, const double* y, int64_t n, int32_t take_sqrt, double* out);
/* the same on device-resident x, y (y may equal x), result written to device *out_dev;
   enqueued on the context stream, no synchronisation */
amgcu_status amgcu_dot_device(amgcu_ctx ctx, const double* x_dev, const double* y_dev, int64_t n, int32_t take_sqrt,
                              double* out_dev);
amgcu_status amgcu_transpose(amgcu_ctx ctx, const amgcu_csr* A, amgcu_csr* out);             /* sparse.hpp:161 */
amgcu_status amgcu_matmul(amgcu_ctx ctx, const amgcu_csr* A, const amgcu_csr* B, amgcu_csr* out); /* :183 */
amgcu_status amgcu_galerkin_product(amgcu_ctx ctx, const amgcu_csr* R, const amgcu_csr* A, const amgcu_csr* P,
                                    amgcu_csr* out);                                          /* :220 */
amgcu_status amgcu_filter_matrix(amgcu_ctx ctx, const amgcu_csr* G, int32_t theta_set, double theta, int32_t k,
                                 amgcu_csr* out);                                             /* :236 */
amgcu_status amgcu_is_symmetric(amgcu_ctx ctx, const amgcu_csr* A, double tol, int32_t* out); /* :288 */
amgcu_status amgcu_spectral_radius(amgcu_ctx ctx, const amgcu_csr* A, int32_t steps, double* rho); /* spectral.hpp:18 */
amgcu_status amgcu_strength(amgcu_ctx ctx, const amgcu_csr* A, const amgcu_strength_config* cfg,
                            amgcu_csr* out);                                                  /* strength.hpp:240 */
amgcu_status amgcu_normalize_strength(amgcu_ctx ctx, const amgcu_csr* S, amgcu_csr* out);    /* :252 */
amgcu_status amgcu_amalgamate(amgcu_ctx ctx, const amgcu_csr* S, int32_t m, amgcu_csr* out); /* :292 */
/* greedy_aggregate (aggregation.hpp:29-98): node_to_agg and roots have room for n */
amgcu_status amgcu_greedy_aggregate(amgcu_ctx ctx, const amgcu_csr* S, int32_t* n_agg, int32_t* node_to_agg,
                                    int32_t* roots);
amgcu_status amgcu_sparsity_pattern(amgcu_ctx ctx, const amgcu_csr* S, const amgcu_csr* C, int32_t degree,
                                    amgcu_csr* out);                                          /* interpolation.hpp:41 */
/* improve_candidates (interpolation.hpp:81-96): B n x k in, out n x k */
amgcu_status amgcu_improve_candidates(amgcu_ctx ctx, const amgcu_csr* A, int32_t k, const double* B,
                                      int32_t sweeps, int32_t scheme, double weight, double* out);
/* relax (relaxation.hpp:183-209) on host x in/out */
amgcu_status amgcu_relax(amgcu_ctx ctx, const amgcu_csr* A, int32_t scheme, double weight, int32_t sweeps,
                         double* x, const double* b);

/* ---- problem generators for the five BASELINE configs (host, harness) --- */
/* config 1..5 at size parameter n (grid / element count per side):
 * 1 Poisson 5-pt (n x n interior), 2 rotated-anisotropic Q1 (n x n elements),
 * 3 recirculating convection-diffusion (n x n), 4 upwind transport (n x n cells),
 * 5 Q1 plane-strain elasticity (n x n elements, left edge clamped).
 * Returns A, the candidate block B (n x k), optional left candidates Bhat
 * (k_hat = 0 when absent) and the right-hand side b. */
amgcu_status amgcu_generate(int32_t config, int32_t n, amgcu_csr* A, int32_t* k, double** B, int32_t* has_left,
                            double** Bhat, double** b);
/* SetupOptions / SolveOptions of config c. */
amgcu_status amgcu_config_options(int32_t config, amgcu_setup_options* so, amgcu_solve_options* vo);
/* Reference defaults: SetupOptions{} and SolveOptions{}. */
void amgcu_default_setup_options(amgcu_setup_options* so);
void amgcu_default_solve_options(amgcu_solve_options* vo);

#ifdef __cplusplus
}
#endif

#endif /* AMGCU_H */
