// Drop-in check: code written against the reference's C++ API (the shape of
// run_single, proj/tools/amg_main.cpp:249-282) compiled against
// include/amg_b200.hpp and linked with libamgcu.so.  Usage: run_single <config> <size>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "amg_b200.hpp"

int main(int argc, char** argv) {
    const int config = argc > 1 ? std::atoi(argv[1]) : 1;
    const int size = argc > 2 ? std::atoi(argv[2]) : 32;
    amgcu_csr Ac{};
    int32_t k = 0, has_left = 0;
    double *Bd = nullptr, *Bh = nullptr, *bd = nullptr;
    if (amgcu_generate(config, size, &Ac, &k, &Bd, &has_left, &Bh, &bd) != AMGCU_OK) return 2;
    amg::SparseMatrix A = amg::b200::take(Ac);
    amg::CandidateSet B(A.n_rows, k), L(A.n_rows, k);
    std::copy(Bd, Bd + static_cast<size_t>(A.n_rows) * k, B.data.begin());
    if (has_left) std::copy(Bh, Bh + static_cast<size_t>(A.n_rows) * k, L.data.begin());
    std::vector<double> b(bd, bd + A.n_rows);
    amgcu_free(Bd);
    amgcu_free(Bh);
    amgcu_free(bd);
    amgcu_setup_options so;
    amgcu_solve_options vo;
    amgcu_config_options(config, &so, &vo);

    amg::SetupOptions opts;  // the reference's option structs, filled as a user would
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
    amg::Hierarchy h = amg::setup(A, B, opts, has_left ? &L : nullptr);
    std::vector<double> x;
    amg::SolveOptions sopts;
    sopts.method = static_cast<amg::SolveMethod>(vo.method);
    sopts.max_iters = vo.max_iters;
    amg::SolveReport rep = amg::solve(h, b, x, sopts);
    h.download();
    const amg::WorkLedger led = h.ledger();
    std::printf("{\"levels\": %d, \"iterations\": %d, \"converged\": %d, \"oc\": %.6f, \"cc\": %.6f, \"nnz_P0\": %d, "
                "\"sc\": %.17g, \"wu\": [%.17g, %.17g, %.17g, %.17g, %.17g]}\n",
                h.n_levels(), rep.iterations, rep.converged ? 1 : 0, rep.chi_oc, rep.chi_cc,
                h.levels.size() > 1 ? h.levels[0].P.nnz() : 0, led.setup_total(), led.wu[0], led.wu[1], led.wu[2],
                led.wu[3], led.wu[4]);
    if (argc > 3) std::fprintf(stderr, "%s\n%s", amg::setup_report_json(h).c_str(), amg::setup_report_csv(h).c_str());
    return rep.converged ? 0 : 3;
}
