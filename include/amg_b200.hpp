// Drop-in C++ API of the B200-native RN-AMG core.
//
// Include this header instead of the reference's "amg/amg.hpp" and link
// libamgcu.so: the types and entry points below carry the reference's names,
// fields, defaults and signatures (namespace amg), so code written against
//   amg::setup(A, B, opts, left)      hierarchy.hpp:551-559
//   amg::rn_setup(A, B, opts, left)   hierarchy.hpp:252-287
//   amg::solve(h, b, x, opts)         cycle.hpp:114-271
//   amg::cycle(h, x, b, kind)         cycle.hpp:100-107
// compiles unchanged.  Everything runs on the GPU behind include/amgcu.h;
// status codes come back as the reference's exception types.
//
// Differences by design: Hierarchy owns device-resident levels; its `levels`
// member is a host mirror filled on demand by Hierarchy::download().
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "amgcu.h"

namespace amg {

using index_t = std::int32_t;

struct SparseMatrix {  // sparse.hpp:25-62
    index_t n_rows = 0;
    index_t n_cols = 0;
    index_t block_size = 1;
    std::vector<index_t> row_offsets;
    std::vector<index_t> col_indices;
    std::vector<double> values;
    SparseMatrix() : row_offsets(1, 0) {}
    SparseMatrix(index_t rows, index_t cols)
        : n_rows(rows), n_cols(cols), row_offsets(static_cast<std::size_t>(rows) + 1, 0) {}
    index_t nnz() const { return static_cast<index_t>(col_indices.size()); }
    index_t row_nnz(index_t i) const { return row_offsets[i + 1] - row_offsets[i]; }
    bool operator==(const SparseMatrix& o) const {
        return n_rows == o.n_rows && n_cols == o.n_cols && row_offsets == o.row_offsets &&
               col_indices == o.col_indices && values == o.values;
    }
};

struct CandidateSet {  // dense.hpp:15-32
    index_t n = 0;
    index_t k = 0;
    std::vector<double> data;
    CandidateSet() = default;
    CandidateSet(index_t n_, index_t k_) : n(n_), k(k_), data(static_cast<std::size_t>(n_) * k_, 0.0) {
        if (n_ < 0 || k_ < 1) throw std::invalid_argument("CandidateSet: need n >= 0, k >= 1");
    }
    double& at(index_t i, index_t j) { return data[static_cast<std::size_t>(j) * n + i]; }
    double at(index_t i, index_t j) const { return data[static_cast<std::size_t>(j) * n + i]; }
};

inline CandidateSet constant_candidates(index_t n) {
    CandidateSet b(n, 1);
    for (index_t i = 0; i < n; ++i) b.at(i, 0) = 1.0;
    return b;
}

enum class StrengthMeasure { classical, symmetric, evolution };
enum class EvolutionWeighting { spectral, l1jacobi };
struct StrengthConfig {  // strength.hpp:18-25
    StrengthMeasure measure = StrengthMeasure::evolution;
    double drop_tol = 4.0;
    int evolution_steps = 2;
    EvolutionWeighting weighting = EvolutionWeighting::spectral;
};

enum class KrylovKind { cg, gmres };
struct FilterRule {  // interpolation.hpp:21-24
    std::optional<double> theta;
    std::optional<index_t> k;
};
struct InterpConfig {  // interpolation.hpp:26-32
    int degree = 2;
    std::optional<FilterRule> prefilter;
    std::optional<FilterRule> postfilter;
    int energy_iters = 0;
    KrylovKind krylov = KrylovKind::cg;
};

enum class RelaxScheme { jacobi, gauss_seidel, sym_gauss_seidel, gsne, block_sym_gauss_seidel };
struct RelaxConfig {  // relaxation.hpp:20-24
    RelaxScheme scheme = RelaxScheme::sym_gauss_seidel;
    double weight = 0.0;
    int sweeps = 1;
};

enum class SetupMethod { rn, sa, cf };
struct SetupOptions {  // hierarchy.hpp:26-36
    SetupMethod method = SetupMethod::rn;
    StrengthConfig strength;
    InterpConfig interp;
    RelaxConfig pre_relax{RelaxScheme::sym_gauss_seidel, 0.0, 1};
    RelaxConfig post_relax{RelaxScheme::sym_gauss_seidel, 0.0, 1};
    index_t max_size = 20;
    int max_levels = 25;
    int candidate_sweeps = 4;
    RelaxConfig candidate_relax{RelaxScheme::gauss_seidel, 0.0, 1};
};

enum class CycleKind { V, W };
enum class SolveMethod { stationary, pcg, fgmres };
struct SolveOptions {  // cycle.hpp:19-24
    SolveMethod method = SolveMethod::stationary;
    CycleKind cycle = CycleKind::V;
    double tol = 1e-8;
    int max_iters = 100;
};

struct SolveReport {  // cycle.hpp:26-36
    std::vector<double> residual_history;
    int iterations = 0;
    bool converged = false;
    bool diverged = false;
    double rho = 0.0;
    double chi_oc = 0.0;
    double chi_cc = 0.0;
    double work_units_solve = 0.0;
    double work_units_setup = 0.0;
};

struct Level {  // hierarchy.hpp:38-48 (host mirror)
    SparseMatrix A, P, R;
    CandidateSet B{0, 1}, Bc{0, 1};
    bool symmetric = true;
};

namespace b200 {

struct AmgError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(amgcu_status st, amgcu_ctx ctx) {
    if (st == AMGCU_OK) return;
    const std::string msg = amgcu_last_error(ctx);
    switch (st) {
        case AMGCU_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case AMGCU_RUNTIME_ERROR: throw std::runtime_error(msg);
        case AMGCU_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw AmgError(msg);
    }
}

// one context (device 0, library stream) per process unless set explicitly
inline amgcu_ctx& default_ctx() {
    static amgcu_ctx ctx = [] {
        amgcu_ctx c = nullptr;
        check(amgcu_ctx_create(0, &c), nullptr);
        return c;
    }();
    return ctx;
}

inline amgcu_csr view(const SparseMatrix& A) {
    return amgcu_csr{A.n_rows, A.n_cols, A.nnz(), A.block_size, const_cast<int32_t*>(A.row_offsets.data()),
                     const_cast<int32_t*>(A.col_indices.data()), const_cast<double*>(A.values.data())};
}

inline SparseMatrix take(amgcu_csr& c) {
    SparseMatrix m(c.n_rows, c.n_cols);
    m.block_size = c.block_size;
    m.row_offsets.assign(c.row_offsets, c.row_offsets + c.n_rows + 1);
    m.col_indices.assign(c.col_indices, c.col_indices + c.nnz);
    m.values.assign(c.values, c.values + c.nnz);
    amgcu_csr_free(&c);
    return m;
}

inline amgcu_setup_options flatten(const SetupOptions& o) {
    amgcu_setup_options c{};
    c.method = static_cast<int32_t>(o.method);
    c.strength_measure = static_cast<int32_t>(o.strength.measure);
    c.drop_tol = o.strength.drop_tol;
    c.evolution_steps = o.strength.evolution_steps;
    c.weighting = static_cast<int32_t>(o.strength.weighting);
    c.degree = o.interp.degree;
    if (o.interp.prefilter) {
        c.prefilter_set = 1;
        c.prefilter_theta_set = o.interp.prefilter->theta.has_value();
        c.prefilter_theta = o.interp.prefilter->theta.value_or(0.0);
        c.prefilter_k = o.interp.prefilter->k.value_or(0);
    }
    if (o.interp.postfilter) {
        c.postfilter_set = 1;
        c.postfilter_theta_set = o.interp.postfilter->theta.has_value();
        c.postfilter_theta = o.interp.postfilter->theta.value_or(0.0);
        c.postfilter_k = o.interp.postfilter->k.value_or(0);
    }
    c.energy_iters = o.interp.energy_iters;
    c.krylov = static_cast<int32_t>(o.interp.krylov);
    c.pre_scheme = static_cast<int32_t>(o.pre_relax.scheme);
    c.pre_weight = o.pre_relax.weight;
    c.pre_sweeps = o.pre_relax.sweeps;
    c.post_scheme = static_cast<int32_t>(o.post_relax.scheme);
    c.post_weight = o.post_relax.weight;
    c.post_sweeps = o.post_relax.sweeps;
    c.max_size = o.max_size;
    c.max_levels = o.max_levels;
    c.candidate_sweeps = o.candidate_sweeps;
    c.cand_scheme = static_cast<int32_t>(o.candidate_relax.scheme);
    c.cand_weight = o.candidate_relax.weight;
    c.cand_sweeps = o.candidate_relax.sweeps;
    return c;
}

}  // namespace b200

// Cumulative cost ledger in work units (work.hpp:27-67): raw op counts / nnz(A_0).
enum class WorkBucket : int { aggregation = 0, candidates = 1, interp = 2, rap = 3, solve_other = 4 };

struct WorkLedger {
    double base_nnz = 0.0;
    std::array<double, 5> wu{};
    bool active() const { return base_nnz > 0.0; }
    double operator[](WorkBucket b) const { return wu[static_cast<int>(b)]; }
    double setup_total() const { return wu[0] + wu[1] + wu[2] + wu[3]; }
    double total() const {
        double t = 0.0;
        for (double v : wu) t += v;
        return t;
    }
};

// Device-resident hierarchy (hierarchy.hpp:80-91).
struct Hierarchy {
    std::shared_ptr<amgcu_hier_s> handle;
    SetupOptions options;
    std::vector<Level> levels;  // host mirror, filled by download()
    bool stagnated = false;

    int n_levels() const {
        int32_t n = 0, s = 0;
        b200::check(amgcu_hier_levels(handle.get(), &n, &s), b200::default_ctx());
        return n;
    }
    // the hierarchy's WorkLedger (the reference's Hierarchy::ledger, charged by setup and
    // every solve); the evolution-SOC part is counted on the first call
    WorkLedger ledger() const {
        WorkLedger w;
        b200::check(amgcu_hier_ledger(handle.get(), w.wu.data()), b200::default_ctx());
        int32_t n = 0, s = 0;
        b200::check(amgcu_hier_levels(handle.get(), &n, &s), b200::default_ctx());
        amgcu_csr a0{};
        b200::check(amgcu_hier_get_matrix(handle.get(), 0, 0, &a0), b200::default_ctx());
        w.base_nnz = static_cast<double>(a0.nnz);
        amgcu_csr_free(&a0);
        return w;
    }
    // copy every level's A, P, R, B, Bc to the host mirror (untimed diagnostics)
    void download() {
        const int L = n_levels();
        levels.assign(L, Level{});
        for (int l = 0; l < L; ++l) {
            for (int which = 0; which < (l + 1 < L ? 3 : 1); ++which) {
                amgcu_csr c{};
                b200::check(amgcu_hier_get_matrix(handle.get(), l, which, &c), b200::default_ctx());
                (which == 0 ? levels[l].A : which == 1 ? levels[l].P : levels[l].R) = b200::take(c);
            }
            for (int which = 0; which < (l + 1 < L ? 2 : 1); ++which) {
                int32_t n = 0, k = 0;
                double* d = nullptr;
                b200::check(amgcu_hier_get_candidates(handle.get(), l, which, &n, &k, &d), b200::default_ctx());
                CandidateSet cs(n, k);
                std::copy(d, d + static_cast<std::size_t>(n) * k, cs.data.begin());
                amgcu_free(d);
                (which == 0 ? levels[l].B : levels[l].Bc) = std::move(cs);
            }
            int32_t sym = 1;
            b200::check(amgcu_hier_level_symmetric(handle.get(), l, &sym), b200::default_ctx());
            levels[l].symmetric = sym != 0;
        }
    }
};

inline Hierarchy rn_setup(const SparseMatrix& A, const CandidateSet& B, const SetupOptions& opts,
                          const CandidateSet* left_candidates = nullptr) {
    if (B.n != A.n_rows) throw std::invalid_argument("rn_setup: candidate size mismatch");
    if (left_candidates && (left_candidates->n != B.n || left_candidates->k != B.k))
        throw std::invalid_argument("rn_setup: left candidate shape mismatch");
    amgcu_ctx ctx = b200::default_ctx();
    amgcu_csr a = b200::view(A);
    amgcu_setup_options o = b200::flatten(opts);
    amgcu_hier h = nullptr;
    b200::check(amgcu_setup(ctx, &a, B.k, B.data.data(), left_candidates ? left_candidates->data.data() : nullptr, &o,
                            &h),
                ctx);
    Hierarchy out;
    out.handle = std::shared_ptr<amgcu_hier_s>(h, [](amgcu_hier p) { amgcu_hier_destroy(p); });
    out.options = opts;
    int32_t n = 0, s = 0;
    b200::check(amgcu_hier_levels(h, &n, &s), ctx);
    out.stagnated = s != 0;
    return out;
}

inline Hierarchy setup(const SparseMatrix& A, const CandidateSet& B, const SetupOptions& opts,
                       const CandidateSet* left_candidates = nullptr) {
    if (opts.method != SetupMethod::rn)
        throw std::invalid_argument("setup: only the root-node method runs on the GPU path");
    return rn_setup(A, B, opts, left_candidates);
}

inline SolveReport solve(Hierarchy& h, std::span<const double> b, std::vector<double>& x,
                         const SolveOptions& opts = {}) {
    if (x.empty()) x.assign(b.size(), 0.0);
    if (x.size() != b.size()) throw std::invalid_argument("solve: guess size mismatch");
    amgcu_solve_options o{static_cast<int32_t>(opts.method), static_cast<int32_t>(opts.cycle), opts.tol,
                          opts.max_iters};
    amgcu_solve_report r{};
    std::vector<double> hist(static_cast<std::size_t>(opts.max_iters) + 2);
    b200::check(amgcu_solve(h.handle.get(), b.data(), x.data(), &o, &r, hist.data(), static_cast<int32_t>(hist.size())),
                b200::default_ctx());
    SolveReport rep;
    hist.resize(static_cast<std::size_t>(r.history_len));
    rep.residual_history = std::move(hist);
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.diverged = r.diverged != 0;
    rep.rho = r.rho;
    rep.chi_oc = r.chi_oc;
    rep.chi_cc = r.chi_cc;
    rep.work_units_solve = r.work_units_solve;
    rep.work_units_setup = r.work_units_setup;
    return rep;
}

inline void cycle(Hierarchy& h, std::span<double> x, std::span<const double> b, CycleKind kind = CycleKind::V) {
    b200::check(amgcu_cycle(h.handle.get(), x.data(), b.data(), static_cast<int32_t>(kind)), b200::default_ctx());
}

// Complexity measures and the setup report (complexity.hpp:15-88).  The report functions
// read the host mirror, downloading it first if needed.  setup_report_json returns the
// reference's setup_report() document as text (the reference builds it with nlohmann::json).
inline double operator_complexity(Hierarchy& h) {
    double oc = 0.0, cc = 0.0;
    b200::check(amgcu_hier_complexity(h.handle.get(), &oc, &cc), b200::default_ctx());
    return oc;
}

inline double cycle_complexity(Hierarchy& h) {
    double oc = 0.0, cc = 0.0;
    b200::check(amgcu_hier_complexity(h.handle.get(), &oc, &cc), b200::default_ctx());
    return cc;
}

inline std::string setup_report_json(Hierarchy& h) {
    if (h.levels.empty()) h.download();
    const WorkLedger w = h.ledger();
    const int L = static_cast<int>(h.levels.size());
    std::string j = "{\"levels\": [";
    char buf[512];
    for (int l = 0; l < L; ++l) {
        const Level& lev = h.levels[l];
        const double npr = lev.A.n_rows > 0 ? static_cast<double>(lev.A.nnz()) / lev.A.n_rows : 0.0;
        std::snprintf(buf, sizeof(buf), "%s{\"level\": %d, \"rows\": %d, \"nnz\": %d, \"nnz_per_row\": %.17g, \"symmetric\": %s",
                      l ? ", " : "", l, lev.A.n_rows, lev.A.nnz(), npr, lev.symmetric ? "true" : "false");
        j += buf;
        if (l + 1 < L) {
            std::snprintf(buf, sizeof(buf), ", \"nnz_P\": %d, \"nnz_R\": %d", lev.P.nnz(), lev.R.nnz());
            j += buf;
        }
        j += "}";
    }
    std::snprintf(buf, sizeof(buf),
                  "], \"operator_complexity\": %.17g, \"cycle_complexity\": %.17g, \"work_units\": {\"aggregation\": "
                  "%.17g, \"candidates\": %.17g, \"interp\": %.17g, \"rap\": %.17g, \"solve_other\": %.17g, "
                  "\"setup_total\": %.17g}}",
                  operator_complexity(h), cycle_complexity(h), w.wu[0], w.wu[1], w.wu[2], w.wu[3], w.wu[4],
                  w.setup_total());
    return j + buf;
}

inline std::string setup_report_csv(Hierarchy& h) {
    if (h.levels.empty()) h.download();
    std::string os = "level,rows,nnz,nnz_per_row,nnz_P,nnz_R\n";
    const int L = static_cast<int>(h.levels.size());
    char buf[256];
    for (int l = 0; l < L; ++l) {
        const Level& lev = h.levels[l];
        const double npr = lev.A.n_rows > 0 ? static_cast<double>(lev.A.nnz()) / lev.A.n_rows : 0.0;
        std::snprintf(buf, sizeof(buf), "%d,%d,%d,%g", l, lev.A.n_rows, lev.A.nnz(), npr);
        os += buf;
        if (l + 1 < L) {
            std::snprintf(buf, sizeof(buf), ",%d,%d", lev.P.nnz(), lev.R.nnz());
            os += buf;
        } else {
            os += ",,";
        }
        os += "\n";
    }
    std::snprintf(buf, sizeof(buf), "operator_complexity,%g,,,,\ncycle_complexity,%g,,,,\nsetup_work_units,%g,,,,\n",
                  operator_complexity(h), cycle_complexity(h), h.ledger().setup_total());
    return os + buf;
}

}  // namespace amg
