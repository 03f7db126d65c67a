// Problem generators for the five BASELINE.json configurations (host harness
// code; the reference's counterpart is proj/include/amg/problems.hpp).
//
//  C1  2D Poisson, 5-point stencil (4,-1,-1,-1,-1), n x n interior grid,
//      Dirichlet boundary eliminated, unscaled (problems.hpp:130-155 scales by 1/h^2;
//      the strength decisions are scale invariant).
//  C2  rotated anisotropic diffusion, bilinear Q1 on an n x n element grid,
//      diffusion Q diag(1, eps) Q^T, Q = rot(psi) -- the reference generator
//      rotated_aniso_fem (problems.hpp:157-215) restated; pinned bitwise
//      against it by tests/test_problems.py.
//  C3  recirculating convection-diffusion on [0,1]^2 (new): central
//      differences for eps*Laplace, first-order upwind for w.grad u,
//      w = (4x(x-1)(1-2y), -4y(y-1)(1-2x)); rows scaled by h^2.
//  C4  single-direction upwind transport (new, upwind_fd-style, problems.hpp:294-329):
//      Omega = (cos 3pi/16, sin 3pi/16), sigma = 1 except 1e-3 on the central
//      0.25 x 0.25 block, zero inflow; lower triangular in natural order.
//  C5  plane-strain linear elasticity (new), bilinear Q1 on an n x n grid of
//      unit elements, E = 1, nu = 0.3, left edge clamped, DOFs interleaved by
//      node (block_size 2), rigid-body modes (1,0), (0,1), (-y, x).
//
// Matrices are assembled through triplets and canonicalised exactly like
// from_triplets (sparse.hpp:72-100: std::sort on (row, col), duplicates summed
// in sorted order, exact zeros dropped), so the same triplet sequence gives
// the same bytes as the reference.  Right-hand sides use
// std::mt19937(seed) + std::uniform_real_distribution<double>(-1, 1)
// (amg_main.cpp:237-245).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <random>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "host_common.h"

namespace amgcu {

namespace {

struct Trip {
    int32_t row, col;
    double value;
};

HostCsr canonical(int32_t nr, int32_t nc, std::vector<Trip> t) {
    std::sort(t.begin(), t.end(),
              [](const Trip& a, const Trip& b) { return std::tie(a.row, a.col) < std::tie(b.row, b.col); });
    HostCsr m;
    m.n_rows = nr;
    m.n_cols = nc;
    m.row_offsets.assign(static_cast<size_t>(nr) + 1, 0);
    m.col_indices.reserve(t.size());
    m.values.reserve(t.size());
    size_t p = 0;
    for (int32_t i = 0; i < nr; ++i) {
        while (p < t.size() && t[p].row == i) {
            const int32_t j = t[p].col;
            double v = 0.0;
            for (; p < t.size() && t[p].row == i && t[p].col == j; ++p) v += t[p].value;
            if (v != 0.0) {
                m.col_indices.push_back(j);
                m.values.push_back(v);
            }
        }
        m.row_offsets[i + 1] = static_cast<int32_t>(m.col_indices.size());
    }
    return m;
}

std::vector<double> uniform_rhs(int32_t n, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> d(-1.0, 1.0);
    std::vector<double> b(n);
    for (auto& v : b) v = d(rng);
    return b;
}

// 2x2 matrix products evaluated entry by entry as s = 0; s += a*b in index order
// (the oracle's Eigen stand-in evaluates G^T M G the same way).
void q1_scalar_element(const double M[2][2], double K[4][4]) {
    static constexpr double xi[4] = {-1.0, 1.0, 1.0, -1.0};
    static constexpr double eta[4] = {-1.0, -1.0, 1.0, 1.0};
    const double g = 1.0 / std::sqrt(3.0);
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) K[a][b] = 0.0;
    for (int gx = 0; gx < 2; ++gx)
        for (int gy = 0; gy < 2; ++gy) {
            const double px = gx == 0 ? -g : g;
            const double py = gy == 0 ? -g : g;
            double G[2][4];
            for (int a = 0; a < 4; ++a) {
                G[0][a] = 0.25 * xi[a] * (1.0 + eta[a] * py);
                G[1][a] = 0.25 * eta[a] * (1.0 + xi[a] * px);
            }
            double GtM[4][2];  // G^T M
            for (int a = 0; a < 4; ++a)
                for (int j = 0; j < 2; ++j) {
                    double s = 0.0;
                    for (int t = 0; t < 2; ++t) s += G[t][a] * M[t][j];
                    GtM[a][j] = s;
                }
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) {
                    double s = 0.0;
                    for (int t = 0; t < 2; ++t) s += GtM[a][t] * G[t][b];
                    K[a][b] += s;
                }
        }
}

// C1
void gen_poisson(int32_t n, Problem& p) {
    if (n < 2) throw std::invalid_argument("generate: n must be >= 2");
    std::vector<Trip> t;
    t.reserve(static_cast<size_t>(n) * n * 5);
    for (int32_t j = 0; j < n; ++j)
        for (int32_t i = 0; i < n; ++i) {
            const int32_t row = j * n + i;
            t.push_back({row, row, 4.0});
            if (i > 0) t.push_back({row, row - 1, -1.0});
            if (i + 1 < n) t.push_back({row, row + 1, -1.0});
            if (j > 0) t.push_back({row, row - n, -1.0});
            if (j + 1 < n) t.push_back({row, row + n, -1.0});
        }
    p.A = canonical(n * n, n * n, std::move(t));
    p.k = 1;
    p.B.assign(static_cast<size_t>(n) * n, 1.0);
    p.b = uniform_rhs(n * n, 0u);
}

// C2: elements per side `cells`, interior nodes n = cells - 1
void gen_rotated(int32_t cells, double eps, double psi, unsigned seed, Problem& p) {
    const int32_t n = cells - 1;
    if (n < 2) throw std::invalid_argument("generate: n must be >= 2");
    const double c = std::cos(psi), s = std::sin(psi);
    const double M[2][2] = {{c * c + eps * s * s, (1.0 - eps) * c * s}, {(1.0 - eps) * c * s, s * s + eps * c * c}};
    double K[4][4];
    q1_scalar_element(M, K);
    auto interior = [&](int32_t i, int32_t j) -> int32_t {
        if (i < 1 || i > n || j < 1 || j > n) return -1;
        return (j - 1) * n + (i - 1);
    };
    std::vector<Trip> t;
    t.reserve(static_cast<size_t>(cells) * cells * 16);
    for (int32_t cj = 0; cj < cells; ++cj)
        for (int32_t ci = 0; ci < cells; ++ci) {
            const int32_t ni[4] = {interior(ci, cj), interior(ci + 1, cj), interior(ci + 1, cj + 1),
                                   interior(ci, cj + 1)};
            for (int a = 0; a < 4; ++a) {
                if (ni[a] < 0) continue;
                for (int b = 0; b < 4; ++b)
                    if (ni[b] >= 0 && K[a][b] != 0.0) t.push_back({ni[a], ni[b], K[a][b]});
            }
        }
    p.A = canonical(n * n, n * n, std::move(t));
    p.k = 1;
    p.B.assign(static_cast<size_t>(n) * n, 1.0);
    p.b = uniform_rhs(n * n, seed);
}

// C3
void gen_recirc(int32_t n, double eps, Problem& p) {
    if (n < 2) throw std::invalid_argument("generate: n must be >= 2");
    const double h = 1.0 / (n + 1);
    std::vector<Trip> t;
    t.reserve(static_cast<size_t>(n) * n * 5);
    for (int32_t j = 0; j < n; ++j)
        for (int32_t i = 0; i < n; ++i) {
            const int32_t row = j * n + i;
            const double x = (i + 1) * h, y = (j + 1) * h;
            const double wx = 4.0 * x * (x - 1.0) * (1.0 - 2.0 * y);
            const double wy = -4.0 * y * (y - 1.0) * (1.0 - 2.0 * x);
            // h^2 * (-eps Laplace + w.grad): central diffusion, upwind convection
            const double west = -eps - h * std::max(wx, 0.0);
            const double east = -eps - h * std::max(-wx, 0.0);
            const double south = -eps - h * std::max(wy, 0.0);
            const double north = -eps - h * std::max(-wy, 0.0);
            const double diag = 4.0 * eps + h * std::fabs(wx) + h * std::fabs(wy);
            if (j > 0) t.push_back({row, row - n, south});
            if (i > 0) t.push_back({row, row - 1, west});
            t.push_back({row, row, diag});
            if (i + 1 < n) t.push_back({row, row + 1, east});
            if (j + 1 < n) t.push_back({row, row + n, north});
        }
    p.A = canonical(n * n, n * n, std::move(t));
    p.k = 1;
    p.B.assign(static_cast<size_t>(n) * n, 1.0);
    p.has_left = true;
    p.Bhat.assign(static_cast<size_t>(n) * n, 1.0);
    p.b = uniform_rhs(n * n, 2u);
}

// C4
void gen_transport(int32_t n, Problem& p) {
    if (n < 2) throw std::invalid_argument("generate: n must be >= 2");
    const double h = 1.0 / n;
    const double ang = 3.0 * std::numbers::pi / 16.0;
    const double ox = std::cos(ang), oy = std::sin(ang);
    std::vector<Trip> t;
    t.reserve(static_cast<size_t>(n) * n * 3);
    for (int32_t j = 0; j < n; ++j)
        for (int32_t i = 0; i < n; ++i) {
            const int32_t row = j * n + i;
            const double x = (i + 0.5) * h, y = (j + 0.5) * h;
            const bool block = x >= 0.375 && x <= 0.625 && y >= 0.375 && y <= 0.625;
            const double sigma = block ? 1e-3 : 1.0;
            double diag = sigma;
            diag += ox / h;
            if (i > 0) t.push_back({row, row - 1, -ox / h});
            diag += oy / h;
            if (j > 0) t.push_back({row, row - n, -oy / h});
            t.push_back({row, row, diag});
        }
    p.A = canonical(n * n, n * n, std::move(t));
    p.k = 1;
    p.B.assign(static_cast<size_t>(n) * n, 1.0);
    p.has_left = true;
    p.Bhat.assign(static_cast<size_t>(n) * n, 1.0);
    p.b.assign(static_cast<size_t>(n) * n, 1.0);
}

// C5: Q1 plane strain on nx x ny unit elements, left edge (x = 0) clamped.
void gen_elasticity(int32_t nx, int32_t ny, double young, double nu, Problem& p) {
    if (nx < 1 || ny < 1) throw std::invalid_argument("generate: need >= 1 element per side");
    if (nu < 0.0 || nu >= 0.5) throw std::invalid_argument("generate: nu must lie in [0, 0.5)");
    const double f = young / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double D[3][3] = {{f * (1.0 - nu), f * nu, 0.0}, {f * nu, f * (1.0 - nu), 0.0},
                            {0.0, 0.0, f * (1.0 - 2.0 * nu) / 2.0}};
    static constexpr double xi[4] = {-1.0, 1.0, 1.0, -1.0};
    static constexpr double eta[4] = {-1.0, -1.0, 1.0, 1.0};
    const double g = 1.0 / std::sqrt(3.0);
    // unit square element: x = (1 + xi)/2, dN/dx = 2 dN/dxi, det J = 1/4, weights 1
    double K[8][8] = {};
    for (int gx = 0; gx < 2; ++gx)
        for (int gy = 0; gy < 2; ++gy) {
            const double px = gx == 0 ? -g : g;
            const double py = gy == 0 ? -g : g;
            double Bm[3][8] = {};
            for (int a = 0; a < 4; ++a) {
                const double dx = 0.5 * xi[a] * (1.0 + eta[a] * py);   // 2 * 0.25 * ...
                const double dy = 0.5 * eta[a] * (1.0 + xi[a] * px);
                Bm[0][2 * a] = dx;
                Bm[1][2 * a + 1] = dy;
                Bm[2][2 * a] = dy;
                Bm[2][2 * a + 1] = dx;
            }
            double DB[3][8];
            for (int r = 0; r < 3; ++r)
                for (int cidx = 0; cidx < 8; ++cidx) {
                    double s = 0.0;
                    for (int t = 0; t < 3; ++t) s += D[r][t] * Bm[t][cidx];
                    DB[r][cidx] = s;
                }
            for (int a = 0; a < 8; ++a)
                for (int b = 0; b < 8; ++b) {
                    double s = 0.0;
                    for (int t = 0; t < 3; ++t) s += Bm[t][a] * DB[t][b];
                    K[a][b] += 0.25 * s;
                }
        }
    const int32_t nodes_x = nx + 1, nodes_y = ny + 1;
    // clamped nodes: i == 0; kept node id = j * nx + (i - 1)
    auto node = [&](int32_t i, int32_t j) -> int32_t { return i == 0 ? -1 : j * nx + (i - 1); };
    const int32_t n_nodes = nodes_y * nx;
    std::vector<Trip> t;
    t.reserve(static_cast<size_t>(nx) * ny * 64);
    for (int32_t j = 0; j < ny; ++j)
        for (int32_t i = 0; i < nx; ++i) {
            const int32_t ids[4] = {node(i, j), node(i + 1, j), node(i + 1, j + 1), node(i, j + 1)};
            for (int a = 0; a < 4; ++a) {
                if (ids[a] < 0) continue;
                for (int ca = 0; ca < 2; ++ca)
                    for (int b = 0; b < 4; ++b) {
                        if (ids[b] < 0) continue;
                        for (int cb = 0; cb < 2; ++cb) {
                            const double v = K[2 * a + ca][2 * b + cb];
                            if (v != 0.0) t.push_back({2 * ids[a] + ca, 2 * ids[b] + cb, v});
                        }
                    }
            }
        }
    p.A = canonical(2 * n_nodes, 2 * n_nodes, std::move(t));
    p.A.block_size = 2;
    p.k = 3;
    const size_t nd = static_cast<size_t>(2) * n_nodes;
    p.B.assign(nd * 3, 0.0);
    for (int32_t j = 0; j < nodes_y; ++j)
        for (int32_t i = 1; i < nodes_x; ++i) {
            const size_t nd0 = static_cast<size_t>(node(i, j));
            const double x = static_cast<double>(i), y = static_cast<double>(j);
            p.B[0 * nd + 2 * nd0] = 1.0;
            p.B[1 * nd + 2 * nd0 + 1] = 1.0;
            p.B[2 * nd + 2 * nd0] = -y;
            p.B[2 * nd + 2 * nd0 + 1] = x;
        }
    p.b = uniform_rhs(static_cast<int32_t>(nd), 3u);
}

}  // namespace

Problem generate_config(int32_t config, int32_t n) {
    Problem p;
    switch (config) {
        case 1: gen_poisson(n, p); break;
        case 2: gen_rotated(n, 1e-3, std::numbers::pi / 8.0, 1u, p); break;
        case 3: gen_recirc(n, 1e-4, p); break;
        case 4: gen_transport(n, p); break;
        case 5: gen_elasticity(n, n, 1.0, 0.3, p); break;
        default: throw std::invalid_argument("generate: config must be 1..5");
    }
    return p;
}

// Reference defaults (hierarchy.hpp:26-36, strength.hpp:18-25, interpolation.hpp:26-32)
void default_setup_options(amgcu_setup_options* so) {
    std::memset(so, 0, sizeof(*so));
    so->method = 0;
    so->strength_measure = 2;
    so->drop_tol = 4.0;
    so->evolution_steps = 2;
    so->weighting = 0;
    so->degree = 2;
    so->energy_iters = 0;
    so->krylov = 0;
    so->pre_scheme = 2;
    so->pre_weight = 0.0;
    so->pre_sweeps = 1;
    so->post_scheme = 2;
    so->post_weight = 0.0;
    so->post_sweeps = 1;
    so->max_size = 20;
    so->max_levels = 25;
    so->candidate_sweeps = 4;
    so->cand_scheme = 1;
    so->cand_weight = 0.0;
    so->cand_sweeps = 1;
}

void default_solve_options(amgcu_solve_options* vo) {
    vo->method = 0;
    vo->cycle = 0;
    vo->tol = 1e-8;
    vo->max_iters = 100;
}

// BASELINE config -> reference options.
void config_options(int32_t c, amgcu_setup_options* so, amgcu_solve_options* vo) {
    default_setup_options(so);
    default_solve_options(vo);
    so->pre_scheme = 0;  // V(1,1) weighted Jacobi, omega = 4 / (3 rho(D^-1 A))
    so->post_scheme = 0;
    so->max_size = 100;
    so->max_levels = 25;
    vo->tol = 1e-8;
    switch (c) {
        case 1:
            so->strength_measure = 1;
            so->drop_tol = 0.25;
            so->degree = 2;
            so->energy_iters = 4;
            so->krylov = 0;
            vo->method = 1;  // CLI default accel "cg" (amg_main.cpp:61)
            vo->max_iters = 100;
            break;
        case 2:
            so->strength_measure = 2;
            so->drop_tol = 4.0;
            so->degree = 2;
            so->prefilter_set = 1;
            so->prefilter_theta_set = 1;
            so->prefilter_theta = 0.1;
            so->energy_iters = 6;
            so->krylov = 0;
            vo->method = 1;
            vo->max_iters = 100;
            break;
        case 3:
            so->strength_measure = 2;
            so->drop_tol = 4.0;
            so->degree = 2;
            so->energy_iters = 4;
            so->krylov = 1;
            vo->method = 2;
            vo->max_iters = 30;
            break;
        case 4:
            so->strength_measure = 2;
            so->drop_tol = 4.0;
            so->degree = 3;
            so->energy_iters = 4;
            so->krylov = 1;
            so->candidate_sweeps = 0;
            vo->method = 2;
            vo->max_iters = 30;
            break;
        case 5:
            so->strength_measure = 1;
            so->drop_tol = 0.1;
            so->degree = 2;
            so->energy_iters = 4;
            so->krylov = 0;
            vo->method = 1;
            vo->max_iters = 100;
            break;
        default: throw std::invalid_argument("config must be 1..5");
    }
}

}  // namespace amgcu
