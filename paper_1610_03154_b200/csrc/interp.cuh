// Interpolation-phase launchers (interpolation.hpp, hierarchy.hpp:98-154).
#pragma once

#include "ops.cuh"

namespace amgcu {

// add_aggregate_entries (hierarchy.hpp:98-110)
void add_aggregate_entries(Ctx& c, const DCsr& N, const DAgg& agg, DCsr& out);
// ensure_min_support without Bc (interpolation.hpp:607-643; the prefilter path)
// ensure_min_support (interpolation.hpp:607-643); with Bc (n_c x k, column-major) the
// span-rank floor of the post-filter
void ensure_min_support(Ctx& c, const DCsr& filtered, const DCsr& full, int32_t min_cols, DCsr& out,
                        const double* Bc = nullptr, int32_t k = 0);
// widen_deficient_rows (hierarchy.hpp:118-154)
void widen_deficient_rows(Ctx& c, const DCsr& N, const DCsr& S, const DAgg& agg, int32_t min_aggs, DCsr& out);
// unamalgamate (aggregation.hpp:103-127) + root_node_pattern (interpolation.hpp:53-77)
void unamalgamate(Ctx& c, const DCsr& N, const DAgg& agg, int32_t m, DCsr& Nd, DBuf<int32_t>& droots);
void root_node_pattern(Ctx& c, const DCsr& N, const int32_t* roots, int32_t n_roots, DCsr& out);

// inject_tentative (interpolation.hpp:523-581): B is (n_nodes*m) x k column-major.
// Returns T and Bc ((n_agg*m) x k).  k > m runs enforce_constraints over N.
void inject_tentative(Ctx& c, const DAgg& agg, const DCsr& N, const double* B, int32_t k, int32_t m, DCsr& T,
                      DBuf<double>& Bc);
// enforce_constraints (interpolation.hpp:458-521) with allowed pattern N (or P's own)
void enforce_constraints(Ctx& c, const DCsr& P, const double* B, const double* Bc, int32_t k, const DCsr* allowed,
                         DCsr& out);

struct EnergyMinStats {
    int iterations = 0;
    bool breakdown = false;
};
// energy_minimize (interpolation.hpp:277-442); krylov 0 = cg, 1 = gmres
void energy_minimize(Ctx& c, const DCsr& A, const DCsr& T, const double* B, const double* Bc, int32_t k,
                     const DCsr& N, int iters, int krylov, const int32_t* roots, int32_t n_roots, DCsr& P,
                     EnergyMinStats* stats);

}  // namespace amgcu
