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
// Hierarchy owns the device-resident levels; like the reference's, its `levels`,
// `ledger`, `options` and `stagnated` members are filled by setup (levels: a host
// mirror downloaded once at the end of setup) and `ledger` is charged by every solve
// and cycle.  Callers of the reference's API (proj/tools/amg_main.cpp:249-282,
// proj/tests/acceptance.cpp, complexity.hpp) therefore compile and behave unchanged;
// tests/cpp/run_single.cpp exercises that surface.
#pragma once

#include <algorithm>
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
    std::span<const index_t> row_cols(index_t i) const {  // sparse.hpp:40-48
        return {col_indices.data() + row_offsets[i], static_cast<std::size_t>(row_nnz(i))};
    }
    std::span<const double> row_vals(index_t i) const {
        return {values.data() + row_offsets[i], static_cast<std::size_t>(row_nnz(i))};
    }
    std::span<double> row_vals(index_t i) {
        return {values.data() + row_offsets[i], static_cast<std::size_t>(row_nnz(i))};
    }
    double coeff(index_t i, index_t j) const {  // sparse.hpp:50-56: value at (i, j), 0 if not stored
        auto cols = row_cols(i);
        auto it = std::lower_bound(cols.begin(), cols.end(), j);
        if (it == cols.end() || *it != j) return 0.0;
        return values[row_offsets[i] + static_cast<index_t>(it - cols.begin())];
    }
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
    std::span<double> col(index_t j) {  // dense.hpp:28-31
        return {data.data() + static_cast<std::size_t>(j) * n, static_cast<std::size_t>(n)};
    }
    std::span<const double> col(index_t j) const {
        return {data.data() + static_cast<std::size_t>(j) * n, static_cast<std::size_t>(n)};
    }
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

// Raw multiply counter (work.hpp:11-22): a multiply-add counts as one operation.
struct OpCounter {
    double ops = 0.0;
    void add(double n) { ops += n; }
    void reset() { ops = 0.0; }
};

inline void count(OpCounter* c, double n) {
    if (c) c->add(n);
}

// Cumulative cost ledger in work units (work.hpp:27-67): raw op counts / nnz(A_0).
enum class WorkBucket : int { aggregation = 0, candidates = 1, interp = 2, rap = 3, solve_other = 4 };

struct WorkLedger {
    double base_nnz = 0.0;
    std::array<double, 5> wu{};
    void register_base(double nnz) {
        if (nnz <= 0.0) throw std::invalid_argument("WorkLedger: base nnz must be positive");
        base_nnz = nnz;
    }
    bool active() const { return base_nnz > 0.0; }
    void charge(WorkBucket b, double raw_ops) {
        if (!active()) throw std::logic_error("WorkLedger: base nnz not registered");
        wu[static_cast<int>(b)] += raw_ops / base_nnz;
    }
    void charge(WorkBucket b, const OpCounter& c) { charge(b, c.ops); }
    double operator[](WorkBucket b) const { return wu[static_cast<int>(b)]; }
    double setup_total() const { return wu[0] + wu[1] + wu[2] + wu[3]; }
    double total() const {
        double t = 0.0;
        for (double v : wu) t += v;
        return t;
    }
};

// Device-resident hierarchy (hierarchy.hpp:80-91) with the reference's members.
struct Hierarchy {
    std::shared_ptr<amgcu_hier_s> handle;
    std::vector<Level> levels;  // host mirror of every level (downloaded by setup)
    SetupOptions options;
    WorkLedger ledger;          // charged by setup, every solve and every cycle
    bool stagnated = false;

    int n_levels() const { return static_cast<int>(levels.size()); }
    const SparseMatrix& finest() const { return levels.front().A; }
    const SparseMatrix& coarsest() const { return levels.back().A; }

    // the library's ledger (buckets as the reference charges them; the evolution-SOC
    // part is counted on the first call) into `ledger`
    void refresh_ledger() {
        b200::check(amgcu_hier_ledger(handle.get(), ledger.wu.data()), b200::default_ctx());
    }
    // copy every level's A, P, R, B, Bc and symmetry flag to the host mirror
    void download() {
        int32_t L = 0, st = 0;
        b200::check(amgcu_hier_levels(handle.get(), &L, &st), b200::default_ctx());
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

// Core sparse kernels of the path (sparse.hpp:141-228) on the GPU through the C ABI,
// with the reference's signatures and op counts.
inline void spmv(const SparseMatrix& A, std::span<const double> x, std::span<double> y, OpCounter* c = nullptr) {
    if (static_cast<index_t>(x.size()) != A.n_cols || static_cast<index_t>(y.size()) != A.n_rows)
        throw std::invalid_argument("spmv: dimension mismatch");
    amgcu_csr a = b200::view(A);
    b200::check(amgcu_spmv(b200::default_ctx(), &a, x.data(), y.data()), b200::default_ctx());
    count(c, static_cast<double>(A.nnz()));
}

inline std::vector<double> spmv(const SparseMatrix& A, std::span<const double> x, OpCounter* c = nullptr) {
    std::vector<double> y(static_cast<std::size_t>(A.n_rows));
    spmv(A, x, y, c);
    return y;
}

inline SparseMatrix transpose(const SparseMatrix& A) {
    amgcu_csr a = b200::view(A), out{};
    b200::check(amgcu_transpose(b200::default_ctx(), &a, &out), b200::default_ctx());
    return b200::take(out);
}

inline SparseMatrix matmul(const SparseMatrix& A, const SparseMatrix& B, OpCounter* c = nullptr) {
    amgcu_csr a = b200::view(A), bm = b200::view(B), out{};
    b200::check(amgcu_matmul(b200::default_ctx(), &a, &bm, &out), b200::default_ctx());
    double ops = 0.0;  // sparse.hpp:195: sum over A's entries of nnz(row k of B)
    for (index_t p = 0; p < A.nnz(); ++p) ops += static_cast<double>(B.row_nnz(A.col_indices[p]));
    count(c, ops);
    return b200::take(out);
}

inline SparseMatrix galerkin_product(const SparseMatrix& R, const SparseMatrix& A, const SparseMatrix& P,
                                     OpCounter* c = nullptr) {
    if (R.n_cols != A.n_rows || A.n_cols != P.n_rows)
        throw std::invalid_argument("galerkin_product: dimension mismatch");
    SparseMatrix AP = matmul(A, P, c);
    SparseMatrix C = matmul(R, AP, c);
    C.block_size = P.block_size;
    return C;
}

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
    out.ledger.register_base(static_cast<double>(A.nnz()));
    out.refresh_ledger();
    out.download();
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
    h.refresh_ledger();
    return rep;
}

namespace b200 {
// the cycle cost model of cycle.hpp:66-69 (what cycle_apply counts): per non-coarsest
// level, pre + post sweeps at |A| each (gsne 2 |A|), one residual |A|, |R| and |P|;
// a W cycle visits every level below the second coarsest twice
inline double cycle_ops(const Hierarchy& h, int level, CycleKind kind) {
    if (level == h.n_levels() - 1) return 0.0;
    const Level& lev = h.levels[level];
    auto sweep = [](RelaxScheme s, double nnz) { return s == RelaxScheme::gsne ? 2.0 * nnz : nnz; };
    const double a = static_cast<double>(lev.A.nnz());
    double ops = h.options.pre_relax.sweeps * sweep(h.options.pre_relax.scheme, a) + a +
                 static_cast<double>(lev.R.nnz()) + static_cast<double>(lev.P.nnz()) +
                 h.options.post_relax.sweeps * sweep(h.options.post_relax.scheme, a);
    ops += cycle_ops(h, level + 1, kind);
    if (kind == CycleKind::W && level + 1 < h.n_levels() - 1) ops += cycle_ops(h, level + 1, kind);
    return ops;
}
}  // namespace b200

// cycle.hpp:100-107: one cycle on A x = b in place, work counted into c
inline void cycle(Hierarchy& h, std::span<double> x, std::span<const double> b, CycleKind kind = CycleKind::V,
                  OpCounter* c = nullptr) {
    if (static_cast<index_t>(x.size()) != h.finest().n_rows || static_cast<index_t>(b.size()) != h.finest().n_rows)
        throw std::invalid_argument("cycle: size mismatch");
    b200::check(amgcu_cycle(h.handle.get(), x.data(), b.data(), static_cast<int32_t>(kind)), b200::default_ctx());
    count(c, b200::cycle_ops(h, 0, kind));
}

// Complexity measures and the setup report (complexity.hpp:15-88), computed from the
// host mirror `levels` exactly as the reference does (a Hierarchy assembled by hand,
// as in proj/tests/test_complexity.cpp, works too).
inline double operator_complexity(const Hierarchy& h) {
    const double base = static_cast<double>(h.finest().nnz());
    double sum = 0.0;
    for (const Level& l : h.levels) sum += static_cast<double>(l.A.nnz());
    return sum / base;
}

inline double cycle_complexity(const Hierarchy& h, int pre_sweeps = -1, int post_sweeps = -1) {
    if (pre_sweeps < 0) pre_sweeps = h.options.pre_relax.sweeps;
    if (post_sweeps < 0) post_sweeps = h.options.post_relax.sweeps;
    const double base = static_cast<double>(h.finest().nnz());
    double sum = 0.0;
    for (int l = 0; l + 1 < h.n_levels(); ++l) {
        const Level& lev = h.levels[l];
        sum += static_cast<double>(pre_sweeps + post_sweeps + 1) * lev.A.nnz();
        sum += static_cast<double>(lev.P.nnz()) + static_cast<double>(lev.R.nnz());
    }
    return sum / base;
}

// setup_report's document as JSON text (the reference builds it with nlohmann::json)
inline std::string setup_report_json(const Hierarchy& h) {
    const WorkLedger& w = h.ledger;
    const int L = h.n_levels();
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

#if __has_include(<json.hpp>)
}  // namespace amg
#include <json.hpp>
namespace amg {
// complexity.hpp:39-71: with nlohmann::json on the include path (as the reference's
// callers have it), setup_report returns the same json document
inline nlohmann::json setup_report(const Hierarchy& h) { return nlohmann::json::parse(setup_report_json(h)); }
#else
struct SetupReport {  // without nlohmann::json: the document as text, .dump() like the json
    std::string text;
    std::string dump(int = -1) const { return text; }
};
inline SetupReport setup_report(const Hierarchy& h) { return {setup_report_json(h)}; }
#endif

inline std::string setup_report_csv(const Hierarchy& h) {
    std::string os = "level,rows,nnz,nnz_per_row,nnz_P,nnz_R\n";
    const int L = h.n_levels();
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
                  operator_complexity(h), cycle_complexity(h), h.ledger.setup_total());
    return os + buf;
}

}  // namespace amg
