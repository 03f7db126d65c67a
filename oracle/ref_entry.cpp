// ORACLE TEST INFRASTRUCTURE -- not part of the product.
//
// Exposes the reference implementation (the unmodified headers under
// /root/reference/proj/include/amg, compiled against oracle/eigen_shim) through
// oracle_abi.h.  Built by oracle/build_ref.sh into oracle/_ref/libamgref.so.
// Nothing here re-implements an algorithm: every entry point forwards to the
// reference function named in its comment.

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "amg/complexity.hpp"
#include "amg/cycle.hpp"
#include "amg/hierarchy.hpp"
#include "amg/problems.hpp"
#include "oracle_abi.h"

namespace {

thread_local std::string g_err;

amg::SparseMatrix to_ref(const amgcu_csr* m) {
    amg::SparseMatrix s(m->n_rows, m->n_cols);
    s.block_size = m->block_size;
    s.row_offsets.assign(m->row_offsets, m->row_offsets + m->n_rows + 1);
    const int nnz = m->row_offsets[m->n_rows];
    s.col_indices.assign(m->col_indices, m->col_indices + nnz);
    s.values.assign(m->values, m->values + nnz);
    return s;
}

void from_ref(const amg::SparseMatrix& s, amgcu_csr* out) {
    out->n_rows = s.n_rows;
    out->n_cols = s.n_cols;
    out->nnz = s.nnz();
    out->block_size = s.block_size;
    out->row_offsets = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (s.n_rows + 1)));
    out->col_indices = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max(1, s.nnz())));
    out->values = static_cast<double*>(std::malloc(sizeof(double) * std::max(1, s.nnz())));
    std::memcpy(out->row_offsets, s.row_offsets.data(), sizeof(int32_t) * (s.n_rows + 1));
    if (s.nnz()) {
        std::memcpy(out->col_indices, s.col_indices.data(), sizeof(int32_t) * s.nnz());
        std::memcpy(out->values, s.values.data(), sizeof(double) * s.nnz());
    }
}

amg::CandidateSet cands(int32_t n, int32_t k, const double* data) {
    amg::CandidateSet c(n, k);
    std::memcpy(c.data.data(), data, sizeof(double) * static_cast<size_t>(n) * k);
    return c;
}

double* dup(const std::vector<double>& v) {
    double* p = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, v.size())));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(double) * v.size());
    return p;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

amg::SetupOptions opts_from(const amgcu_setup_options* o) {
    amg::SetupOptions s;
    s.method = static_cast<amg::SetupMethod>(o->method);
    s.strength.measure = static_cast<amg::StrengthMeasure>(o->strength_measure);
    s.strength.drop_tol = o->drop_tol;
    s.strength.evolution_steps = o->evolution_steps;
    s.strength.weighting = static_cast<amg::EvolutionWeighting>(o->weighting);
    s.interp.degree = o->degree;
    if (o->prefilter_set) {
        amg::FilterRule r;
        if (o->prefilter_theta_set) r.theta = o->prefilter_theta;
        if (o->prefilter_k > 0) r.k = o->prefilter_k;
        s.interp.prefilter = r;
    }
    if (o->postfilter_set) {
        amg::FilterRule r;
        if (o->postfilter_theta_set) r.theta = o->postfilter_theta;
        if (o->postfilter_k > 0) r.k = o->postfilter_k;
        s.interp.postfilter = r;
    }
    s.interp.energy_iters = o->energy_iters;
    s.interp.krylov = static_cast<amg::KrylovKind>(o->krylov);
    s.pre_relax = {static_cast<amg::RelaxScheme>(o->pre_scheme), o->pre_weight, o->pre_sweeps};
    s.post_relax = {static_cast<amg::RelaxScheme>(o->post_scheme), o->post_weight, o->post_sweeps};
    s.max_size = o->max_size;
    s.max_levels = o->max_levels;
    s.candidate_sweeps = o->candidate_sweeps;
    s.candidate_relax = {static_cast<amg::RelaxScheme>(o->cand_scheme), o->cand_weight, o->cand_sweeps};
    return s;
}

amg::Aggregation agg_from(int32_t n_nodes, int32_t n_agg, const int32_t* node_to_agg, const int32_t* roots) {
    amg::Aggregation a;
    a.n_nodes = n_nodes;
    a.n_agg = n_agg;
    a.node_to_agg.assign(node_to_agg, node_to_agg + n_nodes);
    a.roots.assign(roots, roots + n_agg);
    amg::SparseMatrix C(n_nodes, n_agg);
    C.col_indices.assign(node_to_agg, node_to_agg + n_nodes);
    C.values.assign(n_nodes, 1.0);
    for (int i = 0; i < n_nodes; ++i) C.row_offsets[i + 1] = i + 1;
    a.pattern = std::move(C);
    return a;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_free(void* p) { std::free(p); }
void orc_csr_free(amgcu_csr* m) {
    std::free(m->row_offsets);
    std::free(m->col_indices);
    std::free(m->values);
    m->row_offsets = nullptr;
    m->col_indices = nullptr;
    m->values = nullptr;
}

int orc_spmv(const amgcu_csr* A, const double* x, double* y) {
    return guarded([&] {
        auto M = to_ref(A);
        amg::spmv(M, std::span<const double>(x, M.n_cols), std::span<double>(y, M.n_rows));
    });
}
int orc_transpose(const amgcu_csr* A, amgcu_csr* out) {
    return guarded([&] { from_ref(amg::transpose(to_ref(A)), out); });
}
int orc_matmul(const amgcu_csr* A, const amgcu_csr* B, amgcu_csr* out, double* ops) {
    return guarded([&] {
        amg::OpCounter c;
        from_ref(amg::matmul(to_ref(A), to_ref(B), &c), out);
        if (ops) *ops = c.ops;
    });
}
int orc_galerkin_product(const amgcu_csr* R, const amgcu_csr* A, const amgcu_csr* P, amgcu_csr* out) {
    return guarded([&] { from_ref(amg::galerkin_product(to_ref(R), to_ref(A), to_ref(P)), out); });
}
int orc_filter_matrix(const amgcu_csr* G, int32_t theta_set, double theta, int32_t k, amgcu_csr* out) {
    return guarded([&] {
        std::optional<double> t;
        std::optional<amg::index_t> kk;
        if (theta_set) t = theta;
        if (k != 0) kk = k;
        from_ref(amg::filter_matrix(to_ref(G), t, kk), out);
    });
}
int orc_is_symmetric(const amgcu_csr* A, double tol, int32_t* out) {
    return guarded([&] { *out = amg::is_symmetric(to_ref(A), tol) ? 1 : 0; });
}
int orc_spectral_radius(const amgcu_csr* A, int32_t steps, double* rho) {
    return guarded([&] { *rho = amg::spectral_radius_estimate(to_ref(A), steps); });
}
int orc_strength(const amgcu_csr* A, const amgcu_strength_config* cfg, amgcu_csr* out, double* ops) {
    return guarded([&] {
        amg::StrengthConfig s;
        s.measure = static_cast<amg::StrengthMeasure>(cfg->measure);
        s.drop_tol = cfg->drop_tol;
        s.evolution_steps = cfg->evolution_steps;
        s.weighting = static_cast<amg::EvolutionWeighting>(cfg->weighting);
        amg::OpCounter c;
        from_ref(amg::strength(to_ref(A), s, &c), out);
        if (ops) *ops = c.ops;
    });
}
int orc_normalize_strength(const amgcu_csr* S, amgcu_csr* out) {
    return guarded([&] { from_ref(amg::normalize_strength(to_ref(S)), out); });
}
int orc_amalgamate(const amgcu_csr* S, int32_t m, amgcu_csr* out) {
    return guarded([&] { from_ref(amg::amalgamate(to_ref(S), m), out); });
}
int orc_greedy_aggregate(const amgcu_csr* S, int32_t* n_agg, int32_t* node_to_agg, int32_t* roots) {
    return guarded([&] {
        amg::Aggregation a = amg::greedy_aggregate(to_ref(S));
        *n_agg = a.n_agg;
        std::memcpy(node_to_agg, a.node_to_agg.data(), sizeof(int32_t) * a.n_nodes);
        std::memcpy(roots, a.roots.data(), sizeof(int32_t) * a.n_agg);
    });
}
int orc_sparsity_pattern(const amgcu_csr* S, const amgcu_csr* C, int32_t degree, amgcu_csr* out) {
    return guarded([&] { from_ref(amg::sparsity_pattern(to_ref(S), to_ref(C), degree), out); });
}
int orc_root_node_pattern(const amgcu_csr* N, int32_t n_roots, const int32_t* roots, amgcu_csr* out) {
    return guarded([&] {
        std::vector<amg::index_t> r(roots, roots + n_roots);
        from_ref(amg::root_node_pattern(to_ref(N), r), out);
    });
}
int orc_improve_candidates(const amgcu_csr* A, int32_t k, const double* B, int32_t sweeps, int32_t scheme,
                           double weight, double* out) {
    return guarded([&] {
        auto M = to_ref(A);
        amg::CandidateSet b = cands(M.n_rows, k, B);
        amg::CandidateSet r =
            amg::improve_candidates(M, b, sweeps, {static_cast<amg::RelaxScheme>(scheme), weight, 1});
        std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
    });
}
int orc_relax(const amgcu_csr* A, int32_t scheme, double weight, int32_t sweeps, double* x, const double* b) {
    return guarded([&] {
        auto M = to_ref(A);
        std::vector<double> xv(x, x + M.n_rows);
        xv = amg::relax({static_cast<amg::RelaxScheme>(scheme), weight, sweeps}, M, xv,
                        std::span<const double>(b, M.n_rows));
        std::memcpy(x, xv.data(), sizeof(double) * M.n_rows);
    });
}
int orc_relax_weight(const amgcu_csr* A, int32_t scheme, double weight, double* out) {
    return guarded([&] {
        auto ws = amg::make_relax_workspace(to_ref(A), {static_cast<amg::RelaxScheme>(scheme), weight, 1});
        *out = ws.jacobi_weight;
    });
}
int orc_inject_tentative(int32_t n_nodes, int32_t n_agg, const int32_t* node_to_agg, const int32_t* roots,
                         const amgcu_csr* N, int32_t k, const double* B, int32_t m, amgcu_csr* T, double** Bc) {
    return guarded([&] {
        amg::Aggregation a = agg_from(n_nodes, n_agg, node_to_agg, roots);
        auto [t, bc] = amg::inject_tentative(a, to_ref(N), cands(n_nodes * m, k, B), m);
        from_ref(t, T);
        *Bc = dup(bc.data);
    });
}
int orc_enforce_constraints(const amgcu_csr* P, int32_t k, const double* B, const double* Bc,
                            const amgcu_csr* allowed, amgcu_csr* out) {
    return guarded([&] {
        auto Pm = to_ref(P);
        amg::SparseMatrix Nm;
        if (allowed) Nm = to_ref(allowed);
        from_ref(amg::enforce_constraints(Pm, cands(Pm.n_rows, k, B), cands(Pm.n_cols, k, Bc),
                                          allowed ? &Nm : nullptr),
                 out);
    });
}
int orc_energy_minimize(const amgcu_csr* A, const amgcu_csr* T, int32_t k, const double* B, const double* Bc,
                        const amgcu_csr* N, int32_t energy_iters, int32_t krylov, int32_t n_roots,
                        const int32_t* roots, amgcu_csr* out, int32_t* iterations, int32_t* breakdown) {
    return guarded([&] {
        auto Am = to_ref(A), Tm = to_ref(T), Nm = to_ref(N);
        amg::InterpConfig cfg;
        cfg.energy_iters = energy_iters;
        cfg.krylov = static_cast<amg::KrylovKind>(krylov);
        std::vector<amg::index_t> r(roots, roots + n_roots);
        amg::EnergyMinStats st;
        from_ref(amg::energy_minimize(Am, Tm, cands(Am.n_rows, k, B), cands(Nm.n_cols, k, Bc), Nm, cfg, r,
                                      nullptr, &st),
                 out);
        if (iterations) *iterations = st.iterations;
        if (breakdown) *breakdown = st.breakdown ? 1 : 0;
    });
}

int orc_setup(const amgcu_csr* A, int32_t k, const double* B, const double* left, const amgcu_setup_options* o,
              void** hier) {
    return guarded([&] {
        auto Am = to_ref(A);
        amg::CandidateSet b = cands(Am.n_rows, k, B);
        amg::CandidateSet l;
        if (left) l = cands(Am.n_rows, k, left);
        auto* h = new amg::Hierarchy(amg::setup(Am, b, opts_from(o), left ? &l : nullptr));
        *hier = h;
    });
}
int orc_hier_levels(void* hp, int32_t* n_levels, int32_t* stagnated) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        *n_levels = h->n_levels();
        *stagnated = h->stagnated ? 1 : 0;
    });
}
int orc_hier_get_matrix(void* hp, int32_t level, int32_t which, amgcu_csr* out) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        const amg::Level& L = h->levels.at(level);
        from_ref(which == 0 ? L.A : (which == 1 ? L.P : L.R), out);
    });
}
int orc_hier_get_candidates(void* hp, int32_t level, int32_t which, int32_t* n, int32_t* k, double** data) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        const amg::Level& L = h->levels.at(level);
        const amg::CandidateSet& c = which == 0 ? L.B : L.Bc;
        *n = c.n;
        *k = c.k;
        *data = dup(c.data);
    });
}
int orc_hier_level_symmetric(void* hp, int32_t level, int32_t* sym) {
    return guarded([&] { *sym = static_cast<amg::Hierarchy*>(hp)->levels.at(level).symmetric ? 1 : 0; });
}
int orc_hier_relax_weights(void* hp, int32_t level, double* pre, double* post) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        *pre = h->pre_ws.at(level).jacobi_weight;
        *post = h->post_ws.at(level).jacobi_weight;
    });
}
int orc_hier_ledger(void* hp, double* wu5) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        for (int i = 0; i < 5; ++i) wu5[i] = h->ledger.wu[i];
    });
}
int orc_hier_complexity(void* hp, double* chi_oc, double* chi_cc) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        *chi_oc = amg::operator_complexity(*h);
        *chi_cc = amg::cycle_complexity(*h);
    });
}
int orc_hier_free(void* hp) {
    delete static_cast<amg::Hierarchy*>(hp);
    return 0;
}
int orc_solve(void* hp, const double* b, double* x, const amgcu_solve_options* o, amgcu_solve_report* rep,
              double* history, int32_t history_cap) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        const int n = h->finest().n_rows;
        std::vector<double> xv(x, x + n);
        amg::SolveOptions so;
        so.method = static_cast<amg::SolveMethod>(o->method);
        so.cycle = static_cast<amg::CycleKind>(o->cycle);
        so.tol = o->tol;
        so.max_iters = o->max_iters;
        amg::SolveReport r = amg::solve(*h, std::span<const double>(b, n), xv, so);
        std::memcpy(x, xv.data(), sizeof(double) * n);
        rep->iterations = r.iterations;
        rep->converged = r.converged;
        rep->diverged = r.diverged;
        rep->history_len = static_cast<int32_t>(r.residual_history.size());
        rep->rho = r.rho;
        rep->chi_oc = r.chi_oc;
        rep->chi_cc = r.chi_cc;
        rep->work_units_solve = r.work_units_solve;
        rep->work_units_setup = r.work_units_setup;
        for (int i = 0; i < history_cap && i < static_cast<int>(r.residual_history.size()); ++i)
            history[i] = r.residual_history[i];
    });
}
int orc_cycle(void* hp, double* x, const double* b, int32_t kind) {
    return guarded([&] {
        auto* h = static_cast<amg::Hierarchy*>(hp);
        const int n = h->finest().n_rows;
        amg::cycle(*h, std::span<double>(x, n), std::span<const double>(b, n), static_cast<amg::CycleKind>(kind));
    });
}

int orc_generate_reference(int32_t kind, int32_t n, int32_t ny, double eps, double psi, double nu, double young,
                           int32_t flow, int32_t material, amgcu_csr* A, int32_t* k, double** B, int32_t* has_left,
                           double** Bhat, double** rhs) {
    return guarded([&] {
        amg::ProblemSpec s;
        s.kind = static_cast<amg::ProblemKind>(kind);
        s.n = n;
        s.ny = ny;
        s.eps = eps;
        s.psi = psi;
        s.nu = nu;
        s.young = young;
        s.flow = static_cast<amg::FlowFieldId>(flow);
        s.material = static_cast<amg::MaterialId>(material);
        amg::Problem p = amg::generate(s);
        from_ref(p.A, A);
        *k = p.B.k;
        *B = dup(p.B.data);
        *has_left = p.B_hat ? 1 : 0;
        *Bhat = p.B_hat ? dup(p.B_hat->data) : nullptr;
        *rhs = dup(p.rhs);
    });
}

}  // extern "C"
