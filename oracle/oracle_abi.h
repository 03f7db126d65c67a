/* ORACLE TEST INFRASTRUCTURE -- not part of the product.
 *
 * C ABI shared by the two CPU oracles:
 *   oracle/build/liboracle_port.so  -- oracle/rnamg_port.cpp, an own-code
 *                                      restatement of the reference algorithm
 *   oracle/_ref/libamgref.so        -- the reference headers themselves
 *                                      (/root/reference/proj/include/amg),
 *                                      compiled unmodified against the
 *                                      Eigen-API stand-in in oracle/eigen_shim
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load
 * these libraries.  Structs are the ones of include/amgcu.h.
 *
 * Every function returns 0 on success or an error kind (1 invalid_argument,
 * 2 runtime_error, 3 logic_error, 9 other); orc_last_error() gives the text.
 */
#ifndef ORACLE_ABI_H
#define ORACLE_ABI_H

#include "../include/amgcu.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
void orc_free(void* p);
void orc_csr_free(amgcu_csr* m);

int orc_spmv(const amgcu_csr* A, const double* x, double* y);
int orc_transpose(const amgcu_csr* A, amgcu_csr* out);
int orc_matmul(const amgcu_csr* A, const amgcu_csr* B, amgcu_csr* out, double* ops);
int orc_galerkin_product(const amgcu_csr* R, const amgcu_csr* A, const amgcu_csr* P, amgcu_csr* out);
int orc_filter_matrix(const amgcu_csr* G, int32_t theta_set, double theta, int32_t k, amgcu_csr* out);
int orc_is_symmetric(const amgcu_csr* A, double tol, int32_t* out);
int orc_spectral_radius(const amgcu_csr* A, int32_t steps, double* rho);
int orc_strength(const amgcu_csr* A, const amgcu_strength_config* cfg, amgcu_csr* out, double* ops);
int orc_normalize_strength(const amgcu_csr* S, amgcu_csr* out);
int orc_amalgamate(const amgcu_csr* S, int32_t m, amgcu_csr* out);
int orc_greedy_aggregate(const amgcu_csr* S, int32_t* n_agg, int32_t* node_to_agg, int32_t* roots);
int orc_sparsity_pattern(const amgcu_csr* S, const amgcu_csr* C, int32_t degree, amgcu_csr* out);
int orc_root_node_pattern(const amgcu_csr* N, int32_t n_roots, const int32_t* roots, amgcu_csr* out);
int orc_improve_candidates(const amgcu_csr* A, int32_t k, const double* B, int32_t sweeps, int32_t scheme,
                           double weight, double* out);
int orc_relax(const amgcu_csr* A, int32_t scheme, double weight, int32_t sweeps, double* x, const double* b);
int orc_relax_weight(const amgcu_csr* A, int32_t scheme, double weight, double* out);
/* inject_tentative (interpolation.hpp:523-581): aggregation given as
 * node_to_agg (n_nodes) and roots (n_agg); B is (n_nodes*m) x k. */
int orc_inject_tentative(int32_t n_nodes, int32_t n_agg, const int32_t* node_to_agg, const int32_t* roots,
                         const amgcu_csr* N, int32_t k, const double* B, int32_t m, amgcu_csr* T, double** Bc);
int orc_enforce_constraints(const amgcu_csr* P, int32_t k, const double* B, const double* Bc,
                            const amgcu_csr* allowed, amgcu_csr* out);
int orc_energy_minimize(const amgcu_csr* A, const amgcu_csr* T, int32_t k, const double* B, const double* Bc,
                        const amgcu_csr* N, int32_t energy_iters, int32_t krylov, int32_t n_roots,
                        const int32_t* roots, amgcu_csr* out, int32_t* iterations, int32_t* breakdown);

int orc_setup(const amgcu_csr* A, int32_t k, const double* B, const double* left, const amgcu_setup_options* o,
              void** hier);
int orc_hier_levels(void* h, int32_t* n_levels, int32_t* stagnated);
int orc_hier_get_matrix(void* h, int32_t level, int32_t which, amgcu_csr* out);
int orc_hier_get_candidates(void* h, int32_t level, int32_t which, int32_t* n, int32_t* k, double** data);
int orc_hier_level_symmetric(void* h, int32_t level, int32_t* sym);
int orc_hier_relax_weights(void* h, int32_t level, double* pre, double* post);
int orc_hier_ledger(void* h, double* wu5);
int orc_hier_complexity(void* h, double* chi_oc, double* chi_cc);
int orc_hier_free(void* h);
int orc_solve(void* h, const double* b, double* x, const amgcu_solve_options* o, amgcu_solve_report* rep,
              double* history, int32_t history_cap);
int orc_cycle(void* h, double* x, const double* b, int32_t kind);

/* reference problem generator (problems.hpp:404-437) -- libamgref only */
int orc_generate_reference(int32_t kind, int32_t n, int32_t ny, double eps, double psi, double nu, double young,
                           int32_t flow, int32_t material, amgcu_csr* A, int32_t* k, double** B, int32_t* has_left,
                           double** Bhat, double** rhs);

#ifdef __cplusplus
}
#endif

#endif
