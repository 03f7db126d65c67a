// Root-node setup on the GPU: rn_setup / rn_coarsen_once (hierarchy.hpp:183-287)
// orchestrated on the host, every data-parallel step a kernel from ops.cuh /
// interp.cuh, level data resident in HBM.  Sizes cross to the host only where
// an allocation depends on them (scan totals) and for the scalar decisions the
// reference takes on the host (stagnation, symmetry, rho).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <string>

#include <cooperative_groups.h>
#include <cusolverDn.h>

#include "hier.cuh"

#include <cstdlib>
#include "small_dense.h"

namespace amgcu {

// normalize_columns on the device (defined below)
void normalize_candidates(Ctx& c, double* B, int32_t n, int32_t k);

namespace {

void phase(Ctx& c, const char* name, int level) {
    if (!c.phases.on) return;
    cudaEvent_t e;
    AMG_CK(cudaEventCreate(&e));
    AMG_CK(cudaEventRecord(e, c.s));
    c.phases.marks.emplace_back("L" + std::to_string(level) + " " + name, e);
}

void phase_report(Ctx& c) {
    if (!c.phases.on || c.phases.marks.empty()) return;
    AMG_CK(cudaEventSynchronize(c.phases.marks.back().second));
    std::string line = "[phases]";
    float total = 0.f;
    for (size_t q = 1; q < c.phases.marks.size(); ++q) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c.phases.marks[q - 1].second, c.phases.marks[q].second);
        total += ms;
        char buf[96];
        std::snprintf(buf, sizeof(buf), " %s %.2f", c.phases.marks[q].first.c_str(), ms);
        line += buf;
    }
    std::fprintf(stderr, "%s | total %.2f ms\n", line.c_str(), total);
    for (auto& m : c.phases.marks) cudaEventDestroy(m.second);
    c.phases.marks.clear();
}

__global__ void k_evolution_weights(int32_t n, const double* __restrict__ d, double omega, double* __restrict__ winv,
                                    int32_t* __restrict__ bad) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (d[i] == 0.0) atomicMin(bad, i);
    winv[i] = omega / d[i];
}

__global__ void k_l1_weights(int32_t n, const int32_t* __restrict__ rp, const double* __restrict__ va,
                             double* __restrict__ winv, int32_t* __restrict__ bad) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) s += fabs(va[p]);
    if (s == 0.0) atomicMin(bad, i);
    winv[i] = 1.0 / s;
}

__global__ void k_scale_by(int32_t n, double w, const double* __restrict__ d, double* __restrict__ out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = w * d[i];
}

__global__ void k_scale_if_positive(int64_t n, const double* __restrict__ s, double* __restrict__ x) {
    const double nrm = *s;
    if (!(nrm > 0.0)) return;
    const double a = 1.0 / nrm;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] *= a;
}

int energy_iterations(const amgcu_setup_options& o) {  // interpolation.hpp:34-37
    if (o.energy_iters > 0) return o.energy_iters;
    return std::max(1, static_cast<int>(std::ceil(1.5 * o.degree)));
}

struct Coarsened {
    DCsr P, R, Ac;
    DBuf<double> Bf, Bcoarse, Bhc;
};

void strength_of(Ctx& c, DLevel& L, const amgcu_setup_options& o, DCsr& S) {
    const DCsr& A = L.A;
    switch (o.strength_measure) {
        case 0: classical_strength(c, A, o.drop_tol, S); return;
        case 1: symmetric_strength(c, A, o.drop_tol, S); return;
        case 2: {
            if (A.nr != A.nc) throw InvalidArgument("evolution_strength: square matrix required");
            if (o.drop_tol <= 0.0) throw InvalidArgument("evolution_strength: drop_tol must be positive");
            if (o.evolution_steps < 1) throw InvalidArgument("evolution_strength: steps must be >= 1");
            const int32_t n = A.nr;
            DBuf<double> winv(static_cast<size_t>(n), c.s);
            DBuf<int32_t> bad(1, c.s);
            fill_i32(c, bad.get(), INT32_MAX, 1);
            if (o.weighting == 0) {
                const double rho = rho_tallied(c, L);
                if (rho <= 0.0) throw RuntimeError("evolution_strength: spectral radius estimate failed");
                DBuf<double> d(static_cast<size_t>(n), c.s);
                diagonal(c, A, d.get());
                launch(c, k_evolution_weights, blocks_for(n, 256), 256, 0, n, static_cast<const double*>(d.get()),
                       1.0 / rho, winv.get(), bad.get());
                const int32_t b = read_scalar(c, bad.get());
                if (b != INT32_MAX)
                    throw RuntimeError("evolution_strength: zero diagonal at row " + std::to_string(b));
            } else {
                launch(c, k_l1_weights, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.va.get(), winv.get(), bad.get());
                const int32_t b = read_scalar(c, bad.get());
                if (b != INT32_MAX) throw RuntimeError("evolution_strength: zero row at " + std::to_string(b));
            }
            DCsr At;
            transpose(c, A, At);
            evolution_strength(c, A, At, winv.get(), o.drop_tol, o.evolution_steps, S);
            // its ledger count overlaps the rest of the setup (collected in rn_setup)
            L.evo_steps = o.evolution_steps;
            // AMGCU_NO_EVO_COUNT=1 (timing experiments only): skip the ledger's evolution count
            static const bool no_count = std::getenv("AMGCU_NO_EVO_COUNT") != nullptr;
            if (no_count) {
                L.evo_ops = 0.0;
                return;
            }
            L.evo_count = evolution_ops_start(c, A, std::move(At), o.evolution_steps);
            return;
        }
    }
    throw InvalidArgument("strength: unknown measure");
}

// postfilter_pipeline (interpolation.hpp:648-659): drop small entries of P, restore
// the support (rank floor over the coarse candidates), re-impose the constraints,
// then one energy-minimisation iteration on the reduced pattern
void postfilter(Ctx& c, const amgcu_setup_options& o, const DCsr& A, const DCsr& P, const double* B, const double* Bc,
                int32_t k, int krylov, const int32_t* roots, int32_t n_roots, DCsr& out) {
    DCsr Pf, Pm, Pe;
    filter_matrix(c, P, o.postfilter_theta_set != 0, o.postfilter_theta, o.postfilter_k, Pf);
    ensure_min_support(c, Pf, P, k, Pm, Bc, k);
    enforce_constraints(c, Pm, B, Bc, k, nullptr, Pe);
    Pe.bs = P.bs;
    energy_minimize(c, A, Pe, B, Bc, k, Pe, 1, krylov, roots, n_roots, out, nullptr);
    out.bs = P.bs;
}

// Candidate improvement with forward Gauss-Seidel, started early on the context's second
// stream: it depends on A and B only, so its sweeps (lane kernel, latency-bound, 32 SMs
// per 1024 segments) overlap the strength / aggregation / pattern work of the level.
// start: host synchronisations (zero-diagonal check, lane plan) on the main stream, then
// the sweeps on side2; join: the main stream waits for them, then normalizes.  The sweeps
// are the same kernels as the in-order path (no reductions), so the result is bitwise the
// same with the overlap on or off (Ctx::cand_overlap, tests/test_gpu_config_scale.py).
struct CandidateSweeps {
    bool active = false;
    cudaStream_t main = nullptr;
    DBuf<double> dinv;
    LanePlan plan;
    cudaEvent_t done = nullptr;
    ~CandidateSweeps() {
        // left without a join (an exception, or the level stagnated): the main stream must
        // not free or reuse the buffers the sweeps still write before they finish
        if (done) {
            if (main) cudaStreamWaitEvent(main, done, 0);
            cudaEventDestroy(done);
        }
    }
};

bool candidate_sweeps_start(Ctx& c, const DCsr& A, double* B, int32_t k, int sweeps, int scheme, CandidateSweeps& cs) {
    if (scheme != 1 || sweeps <= 0 || !c.side2 || !c.cand_overlap || A.nr != A.nc || k > kGsMaxColumns) return false;
    const int32_t n = A.nr;
    cs.dinv.alloc(static_cast<size_t>(n), c.s);
    // a zero diagonal is reported where the reference meets it (improve_candidates runs
    // after the stagnation check, hierarchy.hpp:191-208): leave it to the in-order path
    if (inverse_diagonal_check(c, A, cs.dinv.get()) >= 0) return false;
    cs.plan = lane_plan(c, A, sweeps, k);
    if (!cs.plan.ok) return false;
    // the done event exists before anything is queued on side2, and is recorded however
    // the queueing ends, so the destructor's wait always covers every queued sweep
    AMG_CK(cudaEventCreateWithFlags(&cs.done, cudaEventDisableTiming));
    cs.main = c.s;
    cudaEvent_t ready;
    AMG_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    cudaError_t e = cudaEventRecord(ready, c.s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.side2, ready, 0);
    cudaEventDestroy(ready);
    AMG_CK(e);
    try {
        StreamScope on_side(c, c.side2);
        gs_lanes_run(c, A, cs.plan, cs.dinv.get(), B, nullptr, sweeps, k);
    } catch (...) {
        cudaEventRecord(cs.done, c.side2);
        throw;
    }
    AMG_CK(cudaEventRecord(cs.done, c.side2));
    cs.active = true;
    return true;
}

void candidate_sweeps_join(Ctx& c, const DCsr& A, double* B, int32_t k, int sweeps, CandidateSweeps& cs) {
    AMG_CK(cudaStreamWaitEvent(c.s, cs.done, 0));
    // relaxation.hpp:207: |A| per sweep and candidate column
    tally(c, static_cast<double>(k) * sweeps * static_cast<double>(A.nnz));
    normalize_candidates(c, B, A.nr, k);
}

bool coarsen(Ctx& c, DHier& H, int level, const double* Bhat, Coarsened& out) {
    const amgcu_setup_options& o = H.o;
    DLevel& L = H.lv[level];
    const DCsr& A = L.A;
    const int32_t k = L.k;
    const int32_t m = std::max<int32_t>(1, A.bs);

    // WorkLedger buckets of this level (hierarchy.hpp:243): aggregation, candidates,
    // interpolation, RAP -- charged only when the level is built
    double cagg = 0.0, ccand = 0.0, cint = 0.0, crap = 0.0;
    DBuf<double> Bimp;
    CandidateSweeps cand;
    DCsr S0, Sa, S;
    DAgg agg;
    phase(c, "begin", level);
    {
        OpsScope scope(c, &cagg);
        strength_of(c, L, o, S0);
        phase(c, "strength", level);
        // the candidates' sweeps depend on A and B only: start them now, beside the
        // aggregation and pattern work (joined before the injection)
        Bimp.alloc(static_cast<size_t>(A.nr) * k, c.s);
        copy_d2d(c, Bimp.get(), L.B.get(), static_cast<int64_t>(A.nr) * k);
        {
            OpsScope none(c, nullptr);
            candidate_sweeps_start(c, A, Bimp.get(), k, o.candidate_sweeps, o.cand_scheme, cand);
        }
        amalgamate(c, S0, m, Sa);
        normalize_strength(c, Sa, S);
        phase(c, "amalgamate", level);
        greedy_aggregate(c, S, agg);
        phase(c, "aggregate", level);
        tally(c, static_cast<double>(S.nnz));  // hierarchy.hpp:197
    }
    if (agg.n_agg >= agg.n_nodes) {
        L.evo_steps = 0;
        return false;
    }

    OpsScope int_scope(c, &cint);
    DCsr N;
    aggregate_indicator(c, agg, N);
    for (int t = 0; t < o.degree; ++t) {
        DCsr next;
        spgemm(c, S, N, next);
        N = std::move(next);
    }
    const int32_t min_aggs = (k + m - 1) / m;
    if (o.prefilter_set) {
        DCsr F, Fa, Fm;
        filter_matrix(c, N, o.prefilter_theta_set != 0, o.prefilter_theta, o.prefilter_k, F);
        add_aggregate_entries(c, F, agg, Fa);
        ensure_min_support(c, Fa, N, min_aggs, Fm);
        N = std::move(Fm);
    }
    {
        DCsr W;
        widen_deficient_rows(c, N, S, agg, min_aggs, W);
        N = std::move(W);
    }
    DCsr Nd0, Nd;
    DBuf<int32_t> droots;
    unamalgamate(c, N, agg, m, Nd0, droots);
    root_node_pattern(c, Nd0, droots.get(), agg.n_agg * m, Nd);
    phase(c, "pattern", level);

    const int32_t n = A.nr;
    {
        OpsScope scope(c, &ccand);
        if (cand.active)
            candidate_sweeps_join(c, A, Bimp.get(), k, o.candidate_sweeps, cand);
        else
            improve_candidates(c, A, Bimp.get(), k, o.candidate_sweeps, o.cand_scheme, o.cand_weight, &L);
    }
    phase(c, "candidates", level);
    DCsr T;
    DBuf<double> Bc;
    inject_tentative(c, agg, Nd, Bimp.get(), k, m, T, Bc);

    int kry = o.krylov;
    if (!L.symmetric && kry == 0) kry = 1;
    const int iters = energy_iterations(o);
    energy_minimize(c, A, T, Bimp.get(), Bc.get(), k, Nd, iters, kry, droots.get(), agg.n_agg * m, out.P, nullptr);
    out.P.bs = T.bs;
    if (o.postfilter_set) {
        DCsr Pp;
        postfilter(c, o, A, out.P, Bimp.get(), Bc.get(), k, kry, droots.get(), agg.n_agg * m, Pp);
        out.P = std::move(Pp);
    }

    phase(c, "energy_min", level);
    if (L.symmetric) {
        transpose(c, out.P, out.R);
        out.Bhc.alloc(Bc.size(), c.s);
        copy_d2d(c, out.Bhc.get(), Bc.get(), static_cast<int64_t>(Bc.size()));
    } else {
        DCsr At;
        transpose(c, A, At);
        DBuf<double> Bh(static_cast<size_t>(n) * k, c.s);
        copy_d2d(c, Bh.get(), Bhat, static_cast<int64_t>(n) * k);
        {
            OpsScope scope(c, &ccand);
            improve_candidates(c, At, Bh.get(), k, o.candidate_sweeps, o.cand_scheme, o.cand_weight, nullptr);
        }
        DCsr That, Rt;
        DBuf<double> Bhc;
        inject_tentative(c, agg, Nd, Bh.get(), k, m, That, Bhc);
        energy_minimize(c, At, That, Bh.get(), Bhc.get(), k, Nd, iters, 1, droots.get(), agg.n_agg * m, Rt, nullptr);
        Rt.bs = That.bs;
        if (o.postfilter_set) {
            DCsr Rp;
            postfilter(c, o, At, Rt, Bh.get(), Bhc.get(), k, 1, droots.get(), agg.n_agg * m, Rp);
            Rt = std::move(Rp);
        }
        transpose(c, Rt, out.R);
        out.Bhc = std::move(Bhc);
    }
    phase(c, "R", level);
    {
        OpsScope scope(c, &crap);
        galerkin(c, out.R, A, out.P, out.Ac);
    }
    phase(c, "RAP", level);
    L.ledger[0] = cagg;
    L.ledger[1] = ccand;
    L.ledger[2] = cint;
    L.ledger[3] = crap;
    out.Bf = std::move(Bimp);
    out.Bcoarse = std::move(Bc);
    return true;
}


__global__ void k_densify(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ va, double* __restrict__ D) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) D[static_cast<size_t>(i) * n + ci[p]] = va[p];
}

__global__ void k_identity(int32_t n, double* __restrict__ I) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * n) return;
    I[t] = (t / n == t % n) ? 1.0 : 0.0;
}

// Inverse of the coarsest operator by Gauss-Jordan elimination with partial pivoting on
// [A | I] (n x 2n, stored column-major, L2-resident for the sizes it serves), one
// cooperative launch with ONE grid barrier per step.  Step k reads the pivot (row p,
// value) chosen at the end of step k - 1 and never writes column k, so every warp can
// process its own columns j > k from the unswapped matrix: the new row k is M(p, j) /
// pivot, row p receives the old row k eliminated, every other row i subtracts
// M(i, k) x (new row k); the elimination factors are column k, read in place.  The warp
// that owns column k + 1 then picks the next pivot (largest |M(i, k+1)|, i > k, lowest
// i on ties).  The arithmetic per element is that of a swap, scale, eliminate sequence.
// status[0] = 1 on a zero pivot (singular).
constexpr int kGjThreads = 256;

__global__ void __launch_bounds__(kGjThreads)
    k_gauss_jordan(int32_t n, double* __restrict__ M, double* __restrict__ pivv, int32_t* __restrict__ pivr,
                   int32_t* __restrict__ status) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t w = 2 * static_cast<int64_t>(n);
    auto col = [&](int64_t j) { return M + j * n; };
    // the first pivot: warp 0 scans column 0
    auto pick = [&](const double* cj, int32_t from, int slot) {
        double best = -1.0;
        int32_t bi = n;
        for (int32_t i = from + lane; i < n; i += 32) {
            const double v = fabs(cj[i]);
            if (v > best) {
                best = v;
                bi = i;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if (lane == 0) {
            pivr[slot] = bi;
            pivv[slot] = bi < n ? cj[bi] : 0.0;
            if (!(best > 0.0)) *status = 1;
        }
    };
    if (gwarp == 0) pick(col(0), 0, 0);
    grid.sync();
    for (int32_t k = 0; k < n; ++k) {
        if (*reinterpret_cast<volatile int32_t*>(status)) return;  // uniform: every block sees it
        const int slot = k & 1;
        const int32_t p = *reinterpret_cast<volatile int32_t*>(pivr + slot);
        const double inv = 1.0 / *reinterpret_cast<volatile double*>(pivv + slot);
        const double* ck = col(k);
        const double fp = ck[k];  // the old row k's factor (it moves to row p)
        for (int64_t j = k + 1 + gwarp; j < w; j += nwarps) {
            double* cj = col(j);
            const double a = cj[k], newk = cj[p] * inv;
            __syncwarp();  // every lane has read rows k and p before any lane writes them
            for (int32_t i = lane; i < n; i += 32) {
                double v;
                if (i == k) v = newk;
                else if (i == p) v = a - fp * newk;
                else v = cj[i] - ck[i] * newk;
                cj[i] = v;
            }
            __syncwarp();
            if (j == k + 1 && k + 1 < n) pick(cj, k + 1, slot ^ 1);
        }
        grid.sync();
    }
}

__global__ void k_gj_extract(int32_t n, const double* __restrict__ M, double* __restrict__ inv) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * n) return;
    const int64_t i = t / n, j = t - i * n;
    inv[t] = M[(n + j) * static_cast<int64_t>(n) + i];  // row-major inverse from the column-major [A | I]
}

__global__ void k_gj_init(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ va, double* __restrict__ M) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) M[static_cast<int64_t>(ci[p]) * n + i] = va[p];
    M[static_cast<int64_t>(n + i) * n + i] = 1.0;
}

constexpr int32_t kGjMax = 4096;  // [A | I] of 4096 rows is 268 MB; above, LU through cuSOLVER

// Gauss-Jordan inverse of the CSR operator A (n <= kGjMax) into inv (row-major); false
// when a zero pivot shows it singular
bool gauss_jordan_inverse(Ctx& c, const DCsr& A, double* inv) {
    const int32_t n = A.nr;
    DBuf<double> M(static_cast<size_t>(n) * 2 * n, c.s), pivv(2, c.s);
    DBuf<int32_t> pivr(2, c.s), status(1, c.s);
    AMG_CK(cudaMemsetAsync(M.get(), 0, sizeof(double) * n * 2 * n, c.s));
    AMG_CK(cudaMemsetAsync(status.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_gj_init, blocks_for(n, 128), 128, 0, n, A.rp.get(), A.ci.get(), A.va.get(), M.get());
    int per_sm = 0;
    AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gauss_jordan, kGjThreads, 0));
    // enough warps for the 2n columns of a step, at most the co-resident grid
    const int want = static_cast<int>((2 * static_cast<int64_t>(n) * 32 + kGjThreads - 1) / kGjThreads);
    const int grid = std::max(1, std::min(std::min(per_sm, 4) * c.sms, want));
    int32_t nn = n;
    double* pM = M.get();
    double* ppv = pivv.get();
    int32_t* ppr = pivr.get();
    int32_t* pst = status.get();
    void* args[] = {&nn, &pM, &ppv, &ppr, &pst};
    const double bytes = 8.0 * 2.0 * static_cast<double>(n) * n * 2.0 * 0.5 * n;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool prof = c.profile && ((c.prof_mask >> kProfCoarseSolve) & 1u);
    if (prof) {
        e0 = prof_event(c);
        e1 = prof_event(c);
        AMG_CK(cudaEventRecord(e0, c.s));
    }
    AMG_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_gauss_jordan), dim3(grid), dim3(kGjThreads), args, 0,
                                       c.s));
    ++c.launches;
    if (prof) {
        AMG_CK(cudaEventRecord(e1, c.s));
        c.prof[kProfCoarseSolve].launches += 1;
        c.prof[kProfCoarseSolve].bytes += bytes;
        c.prof[kProfCoarseSolve].pending.emplace_back(e0, e1);
    }
    if (read_scalar(c, status.get())) return false;
    launch(c, k_gj_extract, blocks_for(static_cast<int64_t>(n) * n, 256), 256, 0, n,
           static_cast<const double*>(M.get()), inv);
    return true;
}

constexpr int32_t kCoarseGpuThreshold = 512;

// inverse of the row-major D (n x n) into inv (row-major).  Reading D as
// column-major gives D^T; solving D^T X = I column-major yields X = D^-T,
// i.e. D^-1 in row-major.  Returns false when the LU is singular.
bool dense_inverse_gpu(Ctx& c, double* D, int32_t n, double* inv) {
    if (!c.cusolver) {
        cusolverDnHandle_t h0;
        if (cusolverDnCreate(&h0) != CUSOLVER_STATUS_SUCCESS) throw CudaFailure("cusolverDnCreate failed");
        c.cusolver = std::shared_ptr<void>(h0, [](void* h) { cusolverDnDestroy(static_cast<cusolverDnHandle_t>(h)); });
    }
    cusolverDnHandle_t hs = static_cast<cusolverDnHandle_t>(c.cusolver.get());
    cusolverDnSetStream(hs, c.s);
    int lwork = 0;
    if (cusolverDnDgetrf_bufferSize(hs, n, n, D, n, &lwork) != CUSOLVER_STATUS_SUCCESS)
        throw CudaFailure("cusolverDnDgetrf_bufferSize failed");
    DBuf<double> work(static_cast<size_t>(lwork) + 1, c.s);
    DBuf<int> piv(static_cast<size_t>(n), c.s), info(1, c.s);
    if (cusolverDnDgetrf(hs, n, n, D, n, work.get(), piv.get(), info.get()) != CUSOLVER_STATUS_SUCCESS)
        throw CudaFailure("cusolverDnDgetrf failed");
    if (read_scalar(c, info.get()) != 0) return false;
    launch(c, k_identity, blocks_for(static_cast<int64_t>(n) * n, 256), 256, 0, n, inv);
    if (cusolverDnDgetrs(hs, CUBLAS_OP_N, n, n, D, n, piv.get(), inv, n, info.get()) != CUSOLVER_STATUS_SUCCESS)
        throw CudaFailure("cusolverDnDgetrs failed");
    if (read_scalar(c, info.get()) != 0) return false;
    return true;
}

}  // namespace

void require_supported_relax(int scheme, const char* who) {
    if (scheme >= 0 && scheme <= 4) return;
    throw InvalidArgument(std::string(who) +
                          ": unknown relaxation scheme");
}

double level_rho(Ctx& c, DLevel& L) {
    if (!std::isnan(L.rho)) return L.rho;
    if (L.rho_job) {
        L.rho = spectral_radius_finish(c, *L.rho_job, &L.rho_built);
        L.rho_job.reset();
        return L.rho;
    }
    if (L.inv_diag.empty()) {
        L.inv_diag.alloc(static_cast<size_t>(L.A.nr), c.s);
        inverse_diagonal(c, L.A, L.inv_diag.get(), "spectral_radius_estimate: zero diagonal at row ");
    }
    {
        OpsScope none(c, nullptr);  // counted per reference call site (rho_tally)
        L.rho = spectral_radius(c, L.A, 15, L.inv_diag.get(), &L.rho_built);
    }
    return L.rho;
}

// The smoother weights need rho(D^-1 A) of every level but the coarsest only at
// finalize_hierarchy; when nothing earlier needs it (no spectral evolution weights, no
// Jacobi candidates), each level's Arnoldi starts on the side stream as soon as the level
// exists and overlaps the coarsening of the levels below it (exact-order reductions
// only: the tree reductions share one scratch between streams).  level_rho collects it.
bool rho_overlap_applies(Ctx& c, const amgcu_setup_options& o) {
    static const bool off = [] {
        const char* e = std::getenv("AMGCU_RHO_OVERLAP");
        return e && e[0] == '0';
    }();
    const bool weights = (o.pre_scheme == 0 && o.pre_weight == 0.0) || (o.post_scheme == 0 && o.post_weight == 0.0);
    const bool early = (o.strength_measure == 2 && o.weighting == 0) || (o.cand_scheme == 0 && o.cand_weight == 0.0);
    return !off && c.seq && c.side && weights && !early;
}

void rho_start_async(Ctx& c, DLevel& L) {
    if (!std::isnan(L.rho) || L.rho_job || L.A.nr == 0) return;
    if (L.inv_diag.empty()) {
        DBuf<double> d(static_cast<size_t>(L.A.nr), c.s);
        // a zero diagonal is reported where the reference meets it (finalize): not here
        if (inverse_diagonal_check(c, L.A, d.get()) >= 0) return;
        L.inv_diag = std::move(d);
    }
    cudaEvent_t ready;
    AMG_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    cudaError_t e = cudaEventRecord(ready, c.s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.side, ready, 0);
    cudaEventDestroy(ready);
    AMG_CK(e);
    OpsScope none(c, nullptr);  // counted per reference call site (rho_tallied)
    StreamScope on_side(c, c.side);
    L.rho_job = spectral_radius_start(c, L.A, 15, L.inv_diag.get());
}

// one reference call of spectral_radius_estimate on the level (spectral.hpp:44: one SpMV per
// Arnoldi step, counted by spmv): the GPU computes rho once per level
double rho_tallied(Ctx& c, DLevel& L) {
    const double r = level_rho(c, L);
    tally(c, static_cast<double>(L.rho_built) * static_cast<double>(L.A.nnz));
    return r;
}

void normalize_candidates(Ctx& c, double* B, int32_t n, int32_t k);

void improve_candidates(Ctx& c, const DCsr& A, double* B, int32_t k, int sweeps, int scheme, double weight,
                        DLevel* cache) {
    if (A.nr != A.nc) throw InvalidArgument("improve_candidates: dimension mismatch");
    if (sweeps < 0) throw InvalidArgument("improve_candidates: sweeps must be >= 0");
    const int32_t n = A.nr;
    if (sweeps > 0) {
        require_supported_relax(scheme, "improve_candidates");
        DBuf<double> dinv;
        if (scheme <= 2) {
            dinv.alloc(static_cast<size_t>(n), c.s);
            inverse_diagonal(c, A, dinv.get(), "relax: zero diagonal at row ");
        }
        if (scheme == 3 || scheme == 4) {
            // make_relax_workspace then relax per candidate column with b = 0
            // (interpolation.hpp:88-92)
            GsneWs gw;
            DBuf<double> binv;
            if (scheme == 3) gsne_workspace(c, A, gw);
            else block_workspace(c, A, binv);
            for (int32_t j = 0; j < k; ++j) {
                double* col = B + static_cast<size_t>(j) * n;
                if (scheme == 3) gsne(c, A, gw, col, nullptr, sweeps);
                else block_sym_gs(c, A, binv.get(), col, nullptr, sweeps);
            }
        } else if (scheme == 0) {
            double w = weight;
            if (w == 0.0) {
                double rho;
                if (cache) {
                    rho = rho_tallied(c, *cache);
                } else {
                    int built = 0;
                    {
                        OpsScope none(c, nullptr);
                        rho = spectral_radius(c, A, 15, dinv.get(), &built);
                    }
                    tally(c, static_cast<double>(built) * static_cast<double>(A.nnz));
                }
                w = 4.0 / (3.0 * rho);
            }
            DBuf<double> wd(static_cast<size_t>(n), c.s);
            launch(c, k_scale_by, blocks_for(n, 256), 256, 0, n, w, static_cast<const double*>(dinv.get()), wd.get());
            jacobi(c, A, wd.get(), B, nullptr, k, sweeps);
        } else {
            gauss_seidel(c, A, dinv.get(), B, nullptr, k, sweeps, scheme == 2);
        }
        // relaxation.hpp:207: relax_sweep_cost per sweep and candidate column (2 |A| for gsne)
        tally(c, static_cast<double>(k) * sweeps * (scheme == 3 ? 2.0 : 1.0) * static_cast<double>(A.nnz));
    }
    normalize_candidates(c, B, n, k);
}

// normalize_columns (dense.hpp:41-46): every column to unit 2-norm (zero columns kept)
void normalize_candidates(Ctx& c, double* B, int32_t n, int32_t k) {
    DBuf<double> nrm(static_cast<size_t>(k), c.s);
    for (int32_t j = 0; j < k; ++j) {
        double* col = B + static_cast<size_t>(j) * n;
        nrm2(c, col, n, nrm.get() + j);
        launch(c, k_scale_if_positive, std::max(1u, std::min<unsigned>(blocks_for(n, 256), 4u * c.sms)), 256, 0,
               static_cast<int64_t>(n), static_cast<const double*>(nrm.get() + j), col);
    }
}


// CoarseSolver::factor (hierarchy.hpp:59-68).  The coarsest operator is
// inverted once; each cycle then applies the inverse with one dense GEMV (a single
// pass over n^2 doubles, where triangular solves would take n dependent steps).
// Up to 512 rows: complete orthogonal decomposition on the host (the reference's
// algorithm, also valid for singular operators).  513..4096 rows: Gauss-Jordan with
// partial pivoting in one cooperative launch (k_gauss_jordan).  Above (a stagnated
// hierarchy can stop at ~10^4 rows, C1): LU with partial pivoting through cuSOLVER
// getrf/getrs.  A singular operator falls back to the COD.
void coarse_factor(Ctx& c, DHier& H) {
    const DLevel& Lc = H.lv.back();
    const int32_t nL = Lc.A.nr;
    H.coarse_n = nL;
    H.coarse_pinv.alloc(static_cast<size_t>(nL) * nL, c.s);
    if (nL > kCoarseGpuThreshold && nL <= kGjMax && gauss_jordan_inverse(c, Lc.A, H.coarse_pinv.get())) return;
    // dense row-major copy of A_L
    DBuf<double> D(static_cast<size_t>(nL) * nL, c.s);
    AMG_CK(cudaMemsetAsync(D.get(), 0, sizeof(double) * nL * nL, c.s));
    launch(c, k_densify, blocks_for(nL, 128), 128, 0, nL, Lc.A.rp.get(), Lc.A.ci.get(), Lc.A.va.get(), D.get());
    if (nL > kGjMax && dense_inverse_gpu(c, D.get(), nL, H.coarse_pinv.get())) return;
    std::vector<double> hD(static_cast<size_t>(nL) * nL);
    copy_d2h(c, hD.data(), D.get(), static_cast<int64_t>(hD.size()));
    sync(c);
    sd::COD cod;
    cod.compute(nL, nL, hD.data());
    std::vector<double> pinv(static_cast<size_t>(nL) * nL);
    cod.pseudo_inverse(pinv.data());
    copy_h2d(c, H.coarse_pinv.get(), pinv.data(), static_cast<int64_t>(pinv.size()));
    sync(c);
}

// The setup's temporaries come from the stream-ordered pool (release threshold raised at
// context creation, so freed memory stays mapped).  A request no free block can hold
// makes the pool map new memory, which can stall the host for hundreds of ms (the
// SpGEMM expansion buffers of a 2 M-row level are ~1 GB).  Reserving one large block up
// front, sized from the operator (AMGCU_POOL_RESERVE_MB overrides), lets the later
// requests be carved out of mapped memory.
void reserve_pool(Ctx& c, const DCsr& A, int32_t k) {
    cudaMemPool_t pool;
    AMG_CK(cudaDeviceGetDefaultMemPool(&pool, c.device));
    uint64_t reserved = 0;
    AMG_CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
    double want = 48.0 * (12.0 * static_cast<double>(A.nnz) + 8.0 * static_cast<double>(A.nr) * (k + 4));
    if (const char* e = std::getenv("AMGCU_POOL_RESERVE_MB")) want = std::atof(e) * 1048576.0;
    size_t free_b = 0, total_b = 0;
    AMG_CK(cudaMemGetInfo(&free_b, &total_b));
    want = std::min(want, 0.5 * static_cast<double>(free_b) + static_cast<double>(reserved));
    if (static_cast<double>(reserved) >= want) return;
    void* p = nullptr;
    if (cudaMallocAsync(&p, static_cast<size_t>(want) - reserved, c.s) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    AMG_CK(cudaFreeAsync(p, c.s));
}

void pool_report(Ctx& c) {
    cudaMemPool_t pool;
    AMG_CK(cudaDeviceGetDefaultMemPool(&pool, c.device));
    uint64_t used_high = 0, reserved = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &used_high);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    std::fprintf(stderr, "[host] pool: used high %.1f MB, reserved %.1f MB\n", used_high / 1048576.0,
                 reserved / 1048576.0);
}

std::unique_ptr<DHier> rn_setup(Ctx& c, const DCsr& A, const double* B, int32_t k, const double* left,
                                const amgcu_setup_options& o) {
    if (o.method != 0) throw InvalidArgument("setup: only the rn method runs on the GPU path");
    if (A.nr != A.nc || A.nr == 0) throw InvalidArgument("rn_setup: square nonempty matrix required");
    if (k < 1) throw InvalidArgument("CandidateSet: need n >= 0, k >= 1");
    const int32_t m = std::max<int32_t>(1, A.bs);
    if (A.nr % m != 0) throw InvalidArgument("rn_setup: block size must divide the dimension");
    if (k < m) throw InvalidArgument("rn_setup: need at least block_size candidates");
    require_supported_relax(o.pre_scheme, "rn_setup");
    require_supported_relax(o.post_scheme, "rn_setup");
    static const bool trace_phases = [] {
        const char* e = std::getenv("AMGCU_PHASE_TRACE");
        return e && e[0] == '1';
    }();
    c.phases.on = trace_phases;
    reserve_pool(c, A, k);
    auto H = std::make_unique<DHier>();
    H->ctx = &c;
    H->o = o;
    if (!(A.nnz > 0)) throw InvalidArgument("WorkLedger: base nnz must be positive");
    H->base_nnz = static_cast<double>(A.nnz);
    H->lv.emplace_back();
    {
        DLevel& L0 = H->lv.back();
        clone_csr(c, A, L0.A);
        L0.k = k;
        L0.B.alloc(static_cast<size_t>(A.nr) * k, c.s);
        copy_d2d(c, L0.B.get(), B, static_cast<int64_t>(A.nr) * k);
        L0.symmetric = is_symmetric(c, L0.A, 1e-12);
    }
    const bool rho_async = rho_overlap_applies(c, o);
    if (rho_async) {
        ensure_start_vector(c, static_cast<size_t>(A.nr));
        if (A.nr > o.max_size && o.max_levels > 1) rho_start_async(c, H->lv.back());
    }
    DBuf<double> Bhat(static_cast<size_t>(A.nr) * k, c.s);
    copy_d2d(c, Bhat.get(), left ? left : B, static_cast<int64_t>(A.nr) * k);

    while (static_cast<int>(H->lv.size()) < o.max_levels && H->lv.back().A.nr > o.max_size) {
        const int l = static_cast<int>(H->lv.size()) - 1;
        Coarsened step;
        if (!coarsen(c, *H, l, Bhat.get(), step)) {
            H->stagnated = true;
            break;
        }
        DLevel& fine = H->lv[l];
        fine.P = std::move(step.P);
        fine.R = std::move(step.R);
        fine.B = std::move(step.Bf);
        fine.Bc.alloc(step.Bcoarse.size(), c.s);
        copy_d2d(c, fine.Bc.get(), step.Bcoarse.get(), static_cast<int64_t>(step.Bcoarse.size()));
        Bhat = std::move(step.Bhc);
        DLevel next;
        next.A = std::move(step.Ac);
        next.k = k;
        next.B = std::move(step.Bcoarse);
        next.symmetric = is_symmetric(c, next.A, 1e-12);
        H->lv.push_back(std::move(next));
        if (rho_async && H->lv.back().A.nr > o.max_size && static_cast<int>(H->lv.size()) < o.max_levels)
            rho_start_async(c, H->lv.back());
        phase(c, "next_level", l);
    }
    // finalize_hierarchy (hierarchy.hpp:164-172): relaxation workspaces and the
    // coarsest-level factorisation; its counts open the solve bucket (hierarchy.hpp:171)
    double cfin = 0.0;
    OpsScope fin_scope(c, &cfin);
    for (size_t l = 0; l + 1 < H->lv.size(); ++l) {
        DLevel& L = H->lv[l];
        const int32_t n = L.A.nr;
        if (L.inv_diag.empty() && (o.pre_scheme <= 2 || o.post_scheme <= 2)) {
            L.inv_diag.alloc(static_cast<size_t>(n), c.s);
            inverse_diagonal(c, L.A, L.inv_diag.get(), "relax: zero diagonal at row ");
        }
        // make_relax_workspace (relaxation.hpp:67-97) for the remaining schemes
        if (o.pre_scheme == 3 || o.post_scheme == 3) gsne_workspace(c, L.A, L.gsne_ws);
        if (o.pre_scheme == 4 || o.post_scheme == 4) block_workspace(c, L.A, L.block_inv);
        auto weight = [&](int scheme, double w) {  // make_ws, relaxation.hpp:52-54
            if (scheme != 0) return 0.0;
            return w != 0.0 ? w : 4.0 / (3.0 * rho_tallied(c, L));
        };
        L.w_pre = weight(o.pre_scheme, o.pre_weight);
        L.w_post = weight(o.post_scheme, o.post_weight);
        if (o.pre_scheme == 0) {
            L.wd_pre.alloc(static_cast<size_t>(n), c.s);
            launch(c, k_scale_by, blocks_for(n, 256), 256, 0, n, L.w_pre, static_cast<const double*>(L.inv_diag.get()),
                   L.wd_pre.get());
        }
        if (o.post_scheme == 0) {
            L.wd_post.alloc(static_cast<size_t>(n), c.s);
            launch(c, k_scale_by, blocks_for(n, 256), 256, 0, n, L.w_post,
                   static_cast<const double*>(L.inv_diag.get()), L.wd_post.get());
        }
    }
    phase(c, "finalize", static_cast<int>(H->lv.size()) - 1);
    coarse_factor(c, *H);
    phase(c, "coarse_factor", static_cast<int>(H->lv.size()) - 1);
    for (DLevel& L : H->lv)
        if (L.evo_count) {
            L.evo_ops = evolution_ops_finish(c, L.A, *L.evo_count);
            L.evo_count.reset();
        }
    {
        const double nL = static_cast<double>(H->lv.back().A.nr);
        tally(c, nL * nL * nL);  // hierarchy.hpp:68
    }
    H->wu[4] = cfin / H->base_nnz;
    {
        static const bool ht = std::getenv("AMGCU_HOST_TRACE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        prepare_solve(*H);
        phase(c, "prepare_solve", static_cast<int>(H->lv.size()) - 1);
        phase_report(c);
        if (ht) pool_report(c);
        if (ht)
            std::fprintf(stderr, "[host] prepare_solve %.3f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    return H;
}

void hier_ledger(DHier& H, double wu[5]) {
    Ctx& c = *H.ctx;
    for (int b = 0; b < 5; ++b) wu[b] = 0.0;
    for (size_t l = 0; l + 1 < H.lv.size(); ++l) {
        DLevel& L = H.lv[l];
        if (L.evo_steps > 0 && L.evo_ops < 0.0) {  // not collected by the setup
            OpsScope none(c, nullptr);
            DCsr At;
            transpose(c, L.A, At);
            L.evo_count = evolution_ops_start(c, L.A, std::move(At), L.evo_steps);
            L.evo_ops = evolution_ops_finish(c, L.A, *L.evo_count);
            L.evo_count.reset();
        }
        // charges in level order, as the reference's coarsening loop (hierarchy.hpp:243)
        wu[0] += (L.ledger[0] + (L.evo_steps > 0 ? L.evo_ops : 0.0)) / H.base_nnz;
        wu[1] += L.ledger[1] / H.base_nnz;
        wu[2] += L.ledger[2] / H.base_nnz;
        wu[3] += L.ledger[3] / H.base_nnz;
    }
    wu[4] = H.wu[4];  // finalize + every solve so far
}

}  // namespace amgcu
