// Host-only drop-in check of complexity.hpp's measures on a hierarchy assembled by hand
// (as proj/tests/test_complexity.cpp does): the functions read only the host mirror.
#include <cstdio>

#include "amg_b200.hpp"

namespace {
amg::SparseMatrix with_nnz(amg::index_t rows, amg::index_t cols, amg::index_t nnz) {
    amg::SparseMatrix m(rows, cols);
    m.col_indices.assign(static_cast<std::size_t>(nnz), 0);
    m.values.assign(static_cast<std::size_t>(nnz), 1.0);
    m.row_offsets.back() = nnz;
    return m;
}
}  // namespace

int main() {
    amg::Hierarchy h;
    h.options.pre_relax.sweeps = 1;
    h.options.post_relax.sweeps = 1;
    h.levels.push_back({.A = with_nnz(30, 30, 120), .P = with_nnz(30, 12, 45), .R = with_nnz(12, 30, 45)});
    h.levels.push_back({.A = with_nnz(12, 12, 48), .P = with_nnz(12, 4, 15), .R = with_nnz(4, 12, 15)});
    h.levels.push_back({.A = with_nnz(4, 4, 12)});
    const double oc = amg::operator_complexity(h);             // (120 + 48 + 12) / 120
    const double cc = amg::cycle_complexity(h);                // (3*120 + 90 + 3*48 + 30) / 120
    const double cc20 = amg::cycle_complexity(h, 2, 0);        // (3*120 + 90 + 3*48 + 30) / 120 too
    const double cc00 = amg::cycle_complexity(h, 0, 0);        // (120 + 90 + 48 + 30) / 120
    std::printf("{\"oc\": %.17g, \"cc\": %.17g, \"cc20\": %.17g, \"cc00\": %.17g, \"finest\": %d, \"coarsest\": %d}\n",
                oc, cc, cc20, cc00, h.finest().n_rows, h.coarsest().n_rows);
    return 0;
}
