// Drop-in check: a caller written against the reference's C++ API, compiled against
// include/amg_b200.hpp and linked with libamgcu.so.  It uses the API the way the
// reference's own callers do -- run_single's setup / solve / ledger record
// (proj/tools/amg_main.cpp:249-282), acceptance.cpp's interpolation-exactness check on
// h.levels (P_l Bc_l = B_l, acceptance.cpp:107-112) and its ledger reads
// (acceptance.cpp:180-183), complexity.hpp's measures and setup_report, and cycle()
// with an OpCounter (cycle.hpp:100-107) -- and prints what it saw as one JSON line.
// Usage: run_single <config> <size> [report]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "amg_b200.hpp"

namespace {

struct Problem {  // the shape of amg::Problem (problems.hpp): A, B, optional B_hat
    amg::SparseMatrix A;
    amg::CandidateSet B;
    std::optional<amg::CandidateSet> B_hat;
    std::vector<double> b;
};

Problem generate(int config, int size) {
    amgcu_csr Ac{};
    int32_t k = 0, has_left = 0;
    double *Bd = nullptr, *Bh = nullptr, *bd = nullptr;
    if (amgcu_generate(config, size, &Ac, &k, &Bd, &has_left, &Bh, &bd) != AMGCU_OK) std::exit(2);
    Problem p;
    p.A = amg::b200::take(Ac);
    p.B = amg::CandidateSet(p.A.n_rows, k);
    std::copy(Bd, Bd + static_cast<size_t>(p.A.n_rows) * k, p.B.data.begin());
    if (has_left) {
        p.B_hat = amg::CandidateSet(p.A.n_rows, k);
        std::copy(Bh, Bh + static_cast<size_t>(p.A.n_rows) * k, p.B_hat->data.begin());
    }
    p.b.assign(bd, bd + p.A.n_rows);
    amgcu_free(Bd);
    amgcu_free(Bh);
    amgcu_free(bd);
    return p;
}

amg::SetupOptions setup_from(int config) {  // the reference's option structs, filled as a user would
    amgcu_setup_options so;
    amgcu_solve_options vo;
    amgcu_config_options(config, &so, &vo);
    amg::SetupOptions opts;
    opts.strength.measure = static_cast<amg::StrengthMeasure>(so.strength_measure);
    opts.strength.drop_tol = so.drop_tol;
    opts.interp.degree = so.degree;
    if (so.prefilter_set) opts.interp.prefilter = amg::FilterRule{so.prefilter_theta, std::nullopt};
    opts.interp.energy_iters = so.energy_iters;
    opts.interp.krylov = static_cast<amg::KrylovKind>(so.krylov);
    opts.pre_relax = {amg::RelaxScheme::jacobi, 0.0, 1};
    opts.post_relax = {amg::RelaxScheme::jacobi, 0.0, 1};
    opts.max_size = so.max_size;
    opts.candidate_sweeps = so.candidate_sweeps;
    return opts;
}

amg::SolveOptions solve_from(int config) {
    amgcu_setup_options so;
    amgcu_solve_options vo;
    amgcu_config_options(config, &so, &vo);
    amg::SolveOptions sopts;
    sopts.method = static_cast<amg::SolveMethod>(vo.method);
    sopts.max_iters = vo.max_iters;
    return sopts;
}

}  // namespace

int main(int argc, char** argv) {
    const int config = argc > 1 ? std::atoi(argv[1]) : 1;
    const int size = argc > 2 ? std::atoi(argv[2]) : 32;

    // run_single (amg_main.cpp:249-282)
    Problem prob = generate(config, size);
    amg::SetupOptions so = setup_from(config);
    amg::Hierarchy h = amg::setup(prob.A, prob.B, so, prob.B_hat ? &*prob.B_hat : nullptr);
    std::vector<double> x;
    amg::SolveReport rep = amg::solve(h, prob.b, x, solve_from(config));

    // acceptance.cpp:107-112: P_l Bc_l reproduces B_l on every level
    double interp_err = 0.0;
    for (std::size_t l = 0; l + 1 < h.levels.size(); ++l) {
        const amg::CandidateSet& B = h.levels[l].B;
        const amg::CandidateSet& Bc = h.levels[l].Bc;
        for (amg::index_t k = 0; k < B.k; ++k) {
            auto pb = amg::spmv(h.levels[l].P, Bc.col(k));
            for (amg::index_t i = 0; i < B.n; ++i) interp_err = std::max(interp_err, std::abs(pb[i] - B.at(i, k)));
        }
    }

    // cycle.hpp:100-107 with the work counter: one V cycle costs cycle_complexity |A_0|
    amg::OpCounter oc;
    std::vector<double> x2(prob.b.size(), 0.0);
    amg::cycle(h, x2, prob.b, amg::CycleKind::V, &oc);
    const double cycle_wu = oc.ops / static_cast<double>(h.finest().nnz());

    // SparseMatrix accessors (sparse.hpp:40-56) on the finest and coarsest operators
    const amg::SparseMatrix& A0 = h.finest();
    const amg::index_t i0 = A0.n_rows / 2;
    const amg::index_t j0 = A0.row_cols(i0).front();
    const bool coeff_ok = A0.coeff(i0, j0) == A0.row_vals(i0).front() && A0.coeff(i0, A0.n_cols) == 0.0;

    std::printf("{\"levels\": %d, \"coarse_rows\": %d, \"iterations\": %d, \"converged\": %d, \"diverged\": %d, "
                "\"oc\": %.17g, \"cc\": %.17g, \"rho\": %.17g, \"nnz_P0\": %d, \"sc\": %.17g, "
                "\"wu\": [%.17g, %.17g, %.17g, %.17g, %.17g], \"interp_err\": %.3g, \"operator_complexity\": %.17g, "
                "\"cycle_complexity\": %.17g, \"cycle_complexity_2_1\": %.17g, \"cycle_wu\": %.17g, \"coeff_ok\": %d}\n",
                h.n_levels(), h.coarsest().n_rows, rep.iterations, rep.converged ? 1 : 0, rep.diverged ? 1 : 0,
                rep.chi_oc, rep.chi_cc, rep.rho, h.levels.size() > 1 ? h.levels[0].P.nnz() : 0,
                h.ledger.setup_total(), h.ledger[amg::WorkBucket::aggregation], h.ledger[amg::WorkBucket::candidates],
                h.ledger[amg::WorkBucket::interp], h.ledger[amg::WorkBucket::rap],
                h.ledger[amg::WorkBucket::solve_other], interp_err, amg::operator_complexity(h),
                amg::cycle_complexity(h), amg::cycle_complexity(h, 2, 1), cycle_wu, coeff_ok ? 1 : 0);
    if (argc > 3) std::fprintf(stderr, "%s\n%s", amg::setup_report(h).dump(2).c_str(), amg::setup_report_csv(h).c_str());
    return rep.converged ? 0 : 3;
}
