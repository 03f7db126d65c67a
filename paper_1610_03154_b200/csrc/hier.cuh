// Device-resident hierarchy (Level / Hierarchy, hierarchy.hpp:38-91) and the
// setup / solve entry points of libamgcu.
#pragma once

#include <cmath>
#include <memory>

#include "interp.cuh"

namespace amgcu {

struct DLevel {
    DCsr A, P, R;
    int32_t k = 1;
    DBuf<double> B;   // n x k, column-major
    DBuf<double> Bc;  // n_c x k (coarse-side targets of P)
    bool symmetric = true;
    double rho = std::nan("");  // rho(D^-1 A), cached
    int rho_built = 0;             // its Arnoldi dimension (the reference's SpMV count per estimate)
    std::unique_ptr<ArnoldiJob> rho_job;  // rho in flight on the side stream (setup.cu: rho_start_async)
    // WorkLedger raw op counts of coarsening this level (work.hpp buckets 0..3); the
    // evolution-SOC part of bucket 0 is counted on demand (evo_steps > 0)
    double ledger[4] = {0.0, 0.0, 0.0, 0.0};
    int evo_steps = 0;
    double evo_ops = -1.0;
    std::unique_ptr<EvoCount> evo_count;  // in flight on the side stream during setup
    // solve phase
    DSell sA, sP, sR;
    DBuf<double> inv_diag;  // 1 / a_ii
    DBuf<double> wd_pre, wd_post;  // jacobi weight * inv_diag
    double w_pre = 0.0, w_post = 0.0;
    DBuf<double> r, t, b, x;  // cycle scratch (b, x used on levels > 0)
    GsneWs gsne_ws;           // gsne workspace (pre or post scheme 3)
    DBuf<double> block_inv;   // block symmetric GS workspace (scheme 4)
};

struct DHier {
    Ctx* ctx = nullptr;
    std::vector<DLevel> lv;
    amgcu_setup_options o{};
    double base_nnz = 0.0;
    double wu[5] = {0, 0, 0, 0, 0};
    bool stagnated = false;
    DBuf<double> coarse_pinv;  // n_L x n_L, row-major
    int32_t coarse_n = 0;
    bool solve_ready = false;
};

// amg::rn_setup on the GPU.  A, B, left are device arrays (left may be null).
std::unique_ptr<DHier> rn_setup(Ctx& c, const DCsr& A, const double* B, int32_t k, const double* left,
                                const amgcu_setup_options& o);

// WorkLedger (work.hpp:38-67) in work units: per-level buckets 0-3 summed in level order,
// bucket 4 = finalize + solves.  Takes the evolution-SOC count on first request.
void hier_ledger(DHier& h, double wu[5]);

// relaxation helpers shared by setup and solve
void require_supported_relax(int scheme, const char* who);
double level_rho(Ctx& c, DLevel& L);
// level_rho, counted as one reference call of spectral_radius_estimate (WorkLedger)
double rho_tallied(Ctx& c, DLevel& L);

// solve phase (cycle.cu)
void prepare_solve(DHier& h);
struct SolveResult {
    std::vector<double> history;
    int iterations = 0;
    bool converged = false, diverged = false;
    double rho = 0.0, chi_oc = 0.0, chi_cc = 0.0, wu_solve = 0.0, wu_setup = 0.0;
};
SolveResult solve(DHier& h, const double* b_dev, double* x_dev, const amgcu_solve_options& o);
void cycle(DHier& h, double* x_dev, const double* b_dev, int kind);
double operator_complexity(const DHier& h);
double cycle_complexity(const DHier& h);

// improve_candidates (interpolation.hpp:81-96) on the device, in place
void improve_candidates(Ctx& c, const DCsr& A, double* B, int32_t k, int sweeps, int scheme, double weight,
                        DLevel* cache);

}  // namespace amgcu
