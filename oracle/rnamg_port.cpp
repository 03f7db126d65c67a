// ORACLE TEST INFRASTRUCTURE -- not part of the product.
//
// CPU restatement of the reference RN-AMG path (arxiv/paper_1610_03154,
// /root/reference/proj/include/amg) used as the parity checker for the GPU
// path.  Every routine cites the reference lines it restates and keeps the
// reference's floating-point operation order (each sum starts at 0.0 and adds
// terms in the reference's loop order; build with -ffp-contract=off), so its
// results are bit-identical to the reference headers compiled against the
// same Eigen stand-in (checked by tests/test_oracle_pin.py against
// oracle/_ref/libamgref.so).
//
// One deliberate difference: inject_tentative visits each node once through
// node_to_agg instead of scanning all nodes per aggregate
// (interpolation.hpp:559-560), which makes the restatement O(n) instead of
// O(n_agg * n); each DOF row receives the same entries, so T is identical.
//
// Tiny dense algebra (Gram pseudo-inverses, root-block LU, Hessenberg
// eigenvalues, coarsest COD) comes from small_dense.h, the routine set the
// Eigen stand-in wraps.

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../paper_1610_03154_b200/csrc/small_dense.h"
#include "oracle_abi.h"

namespace port {

using idx = int32_t;
using Vec = std::vector<double>;

struct Csr {
    idx nr = 0, nc = 0, bs = 1;
    std::vector<idx> rp{0}, ci;
    Vec va;
    Csr() = default;
    Csr(idx r, idx c) : nr(r), nc(c), rp(static_cast<size_t>(r) + 1, 0) {}
    idx nnz() const { return static_cast<idx>(ci.size()); }
    idx len(idx i) const { return rp[i + 1] - rp[i]; }
    double at(idx i, idx j) const {  // SparseMatrix::coeff, sparse.hpp:51-56
        auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
        auto it = std::lower_bound(b, e, j);
        if (it == e || *it != j) return 0.0;
        return va[static_cast<size_t>(it - ci.begin())];
    }
    bool has(idx i, idx j) const {
        auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
        return std::binary_search(b, e, j);
    }
    void close_row(idx i) { rp[i + 1] = static_cast<idx>(ci.size()); }
    void push(idx j, double v) {
        ci.push_back(j);
        va.push_back(v);
    }
};

struct Cand {  // CandidateSet, dense.hpp:15-32 (column-major)
    idx n = 0, k = 1;
    Vec d;
    Cand() = default;
    Cand(idx n_, idx k_) : n(n_), k(k_), d(static_cast<size_t>(n_) * k_, 0.0) {
        if (n_ < 0 || k_ < 1) throw std::invalid_argument("CandidateSet: need n >= 0, k >= 1");
    }
    double& at(idx i, idx j) { return d[static_cast<size_t>(j) * n + i]; }
    double at(idx i, idx j) const { return d[static_cast<size_t>(j) * n + i]; }
    double* col(idx j) { return d.data() + static_cast<size_t>(j) * n; }
    const double* col(idx j) const { return d.data() + static_cast<size_t>(j) * n; }
};

struct Ops {  // OpCounter, work.hpp:13-22
    double v = 0.0;
};
inline void tally(Ops* c, double n) {
    if (c) c->v += n;
}

// ---- BLAS-1 (sparse.hpp:309-323) --------------------------------------------
inline double vdot(const double* a, const double* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
inline double vnorm(const double* a, size_t n) { return std::sqrt(vdot(a, a, n)); }
inline void vaxpy(double al, const double* x, double* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] += al * x[i];
}
inline void vscale(double al, double* x, size_t n) {
    for (size_t i = 0; i < n; ++i) x[i] *= al;
}

// ---- construction (sparse.hpp:64-138) ----------------------------------------
struct Trip {
    idx row, col;
    double value;
};

Csr build_from_triplets(idx nr, idx nc, std::vector<Trip> t) {
    for (const Trip& e : t)
        if (e.row < 0 || e.row >= nr || e.col < 0 || e.col >= nc)
            throw std::invalid_argument("from_triplets: entry out of range");
    std::sort(t.begin(), t.end(),
              [](const Trip& a, const Trip& b) { return std::tie(a.row, a.col) < std::tie(b.row, b.col); });
    Csr m(nr, nc);
    size_t p = 0;
    for (idx i = 0; i < nr; ++i) {
        while (p < t.size() && t[p].row == i) {
            const idx j = t[p].col;
            double acc = 0.0;
            for (; p < t.size() && t[p].row == i && t[p].col == j; ++p) acc += t[p].value;
            if (acc != 0.0) m.push(j, acc);
        }
        m.close_row(i);
    }
    return m;
}

using RowList = std::vector<std::vector<std::pair<idx, double>>>;

Csr build_from_rows(idx nc, RowList rows) {
    const idx nr = static_cast<idx>(rows.size());
    Csr m(nr, nc);
    for (idx i = 0; i < nr; ++i) {
        auto& r = rows[i];
        std::sort(r.begin(), r.end());
        size_t p = 0;
        while (p < r.size()) {
            const idx j = r[p].first;
            if (j < 0 || j >= nc) throw std::invalid_argument("from_rows: column out of range");
            double acc = 0.0;
            for (; p < r.size() && r[p].first == j; ++p) acc += r[p].second;
            if (acc != 0.0) m.push(j, acc);
        }
        m.close_row(i);
    }
    return m;
}

// ---- sparse kernels (sparse.hpp:141-305) -------------------------------------
void spmv(const Csr& A, const double* x, double* y, Ops* c = nullptr) {
    for (idx i = 0; i < A.nr; ++i) {
        double s = 0.0;
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p) s += A.va[p] * x[A.ci[p]];
        y[i] = s;
    }
    tally(c, static_cast<double>(A.nnz()));
}

Csr transpose(const Csr& A) {
    Csr T(A.nc, A.nr);
    T.bs = A.bs;
    for (idx j : A.ci) ++T.rp[j + 1];
    for (idx j = 0; j < A.nc; ++j) T.rp[j + 1] += T.rp[j];
    T.ci.resize(A.ci.size());
    T.va.resize(A.va.size());
    std::vector<idx> fill(T.rp.begin(), T.rp.end() - 1);
    for (idx i = 0; i < A.nr; ++i)
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p) {
            const idx dst = fill[A.ci[p]]++;
            T.ci[dst] = i;
            T.va[dst] = A.va[p];
        }
    return T;
}

Csr matmul(const Csr& A, const Csr& B, Ops* c = nullptr) {
    if (A.nc != B.nr) throw std::invalid_argument("matmul: dimension mismatch");
    Csr C(A.nr, B.nc);
    Vec acc(B.nc, 0.0);
    std::vector<idx> stamp(B.nc, -1), cols;
    double ops = 0.0;
    for (idx i = 0; i < A.nr; ++i) {
        cols.clear();
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p) {
            const idx t = A.ci[p];
            const double a = A.va[p];
            ops += static_cast<double>(B.len(t));
            for (idx q = B.rp[t]; q < B.rp[t + 1]; ++q) {
                const idx j = B.ci[q];
                if (stamp[j] != i) {
                    stamp[j] = i;
                    acc[j] = 0.0;
                    cols.push_back(j);
                }
                acc[j] += a * B.va[q];
            }
        }
        std::sort(cols.begin(), cols.end());
        for (idx j : cols)
            if (acc[j] != 0.0) C.push(j, acc[j]);
        C.close_row(i);
    }
    tally(c, ops);
    return C;
}

Csr galerkin(const Csr& R, const Csr& A, const Csr& P, Ops* c = nullptr) {
    if (R.nc != A.nr || A.nc != P.nr) throw std::invalid_argument("galerkin_product: dimension mismatch");
    Csr AP = matmul(A, P, c);
    Csr out = matmul(R, AP, c);
    out.bs = P.bs;
    return out;
}

Csr filter(const Csr& G, std::optional<double> theta, std::optional<idx> k) {
    if (theta && (*theta < 0.0 || *theta > 1.0))
        throw std::invalid_argument("filter_matrix: theta must lie in [0, 1]");
    if (k && *k < 1) throw std::invalid_argument("filter_matrix: k must be >= 1");
    const bool square = G.nr == G.nc;
    Csr F(G.nr, G.nc);
    F.bs = G.bs;
    Vec mags;
    for (idx i = 0; i < G.nr; ++i) {
        mags.clear();
        for (idx p = G.rp[i]; p < G.rp[i + 1]; ++p)
            if (!(square && G.ci[p] == i)) mags.push_back(std::fabs(G.va[p]));
        double kth = 0.0;
        if (k && static_cast<size_t>(*k) < mags.size()) {
            Vec s(mags);
            std::nth_element(s.begin(), s.begin() + (*k - 1), s.end(), std::greater<double>());
            kth = s[*k - 1];
        }
        double tmax = 0.0;
        if (theta && !mags.empty()) tmax = *theta * *std::max_element(mags.begin(), mags.end());
        for (idx p = G.rp[i]; p < G.rp[i + 1]; ++p) {
            const double mag = std::fabs(G.va[p]);
            const bool diag = square && G.ci[p] == i;
            const bool keep = diag || ((!k || mag >= kth) && (!theta || mag >= tmax));
            if (keep && G.va[p] != 0.0) F.push(G.ci[p], G.va[p]);
        }
        F.close_row(i);
    }
    return F;
}

Vec diag_of(const Csr& A) {
    const idx n = std::min(A.nr, A.nc);
    Vec d(n, 0.0);
    for (idx i = 0; i < n; ++i) d[i] = A.at(i, i);
    return d;
}

bool symmetric(const Csr& A, double tol = 1e-12) {
    if (A.nr != A.nc) return false;
    const Csr T = transpose(A);
    double scale = 0.0;
    for (double v : A.va) scale = std::max(scale, std::fabs(v));
    if (A.ci == T.ci && A.rp == T.rp) {
        for (idx p = 0; p < A.nnz(); ++p)
            if (std::fabs(A.va[p] - T.va[p]) > tol * scale) return false;
        return true;
    }
    for (idx i = 0; i < A.nr; ++i)
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p)
            if (std::fabs(A.va[p] - T.at(i, A.ci[p])) > tol * scale) return false;
    for (idx i = 0; i < T.nr; ++i)
        for (idx p = T.rp[i]; p < T.rp[i + 1]; ++p)
            if (std::fabs(T.va[p] - A.at(i, T.ci[p])) > tol * scale) return false;
    return true;
}

// ---- rho(D^-1 A) by Arnoldi (spectral.hpp:18-65) ------------------------------
double spectral_radius(const Csr& A, int steps = 15, Ops* c = nullptr) {
    if (A.nr != A.nc) throw std::invalid_argument("spectral_radius_estimate: square matrix required");
    const idx n = A.nr;
    if (n == 0) return 0.0;
    Vec dinv(n);
    for (idx i = 0; i < n; ++i) {
        const double d = A.at(i, i);
        if (d == 0.0)
            throw std::runtime_error("spectral_radius_estimate: zero diagonal at row " + std::to_string(i));
        dinv[i] = 1.0 / d;
    }
    const int m = std::min<int>(steps, n);
    std::mt19937 gen(20240911u);
    std::uniform_real_distribution<double> dist(-0.5, 0.5);
    std::vector<Vec> basis;
    Vec v0(n);
    for (idx i = 0; i < n; ++i) v0[i] = 1.0 + dist(gen);
    vscale(1.0 / vnorm(v0.data(), n), v0.data(), n);
    basis.push_back(std::move(v0));
    Vec H(static_cast<size_t>(m + 1) * m, 0.0);  // row-major (m+1) x m
    int built = 0;
    Vec w(n);
    for (int j = 0; j < m; ++j) {
        spmv(A, basis[j].data(), w.data(), c);
        for (idx i = 0; i < n; ++i) w[i] *= dinv[i];
        for (int t = 0; t <= j; ++t) {
            const double h = vdot(w.data(), basis[t].data(), n);
            H[t * m + j] = h;
            vaxpy(-h, basis[t].data(), w.data(), n);
        }
        const double h = vnorm(w.data(), n);
        H[(j + 1) * m + j] = h;
        built = j + 1;
        if (h < 1e-14) break;
        Vec v(w);
        vscale(1.0 / h, v.data(), n);
        basis.push_back(std::move(v));
    }
    Vec Hs(static_cast<size_t>(built) * built), wr(built), wi(built);
    for (int i = 0; i < built; ++i)
        for (int j = 0; j < built; ++j) Hs[i * built + j] = H[i * m + j];
    if (sd::hessenberg_eigenvalues(built, Hs.data(), wr.data(), wi.data()) != 0)
        throw std::runtime_error("Eigen shim: EigenSolver did not converge");
    double rho = 0.0;
    for (int i = 0; i < built; ++i) rho = std::max(rho, std::abs(std::complex<double>(wr[i], wi[i])));
    return rho;
}

// ---- strength of connection (strength.hpp) ------------------------------------
// Insert the diagonal entry (i, dval) into row i in sorted position when no
// off-diagonal above i was emitted (strength.hpp:54-61, 96-102, 225-231).
void close_strength_row(Csr& S, idx i, bool diag_done, double dval) {
    if (!diag_done) {
        auto b = S.ci.begin() + S.rp[i];
        auto it = std::lower_bound(b, S.ci.end(), i);
        const auto off = it - S.ci.begin();
        S.ci.insert(it, i);
        S.va.insert(S.va.begin() + off, dval);
    }
    S.close_row(i);
}

Csr classical_soc(const Csr& A, double theta, Ops* c) {  // strength.hpp:29-66
    if (A.nr != A.nc) throw std::invalid_argument("classical_strength: square matrix required");
    if (theta < 0.0 || theta > 1.0) throw std::invalid_argument("classical_strength: theta must lie in [0, 1]");
    Csr S(A.nr, A.nc);
    S.bs = A.bs;
    for (idx i = 0; i < A.nr; ++i) {
        double mx = 0.0;
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p)
            if (A.ci[p] != i) mx = std::max(mx, -A.va[p]);
        bool dd = false;
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p) {
            const idx j = A.ci[p];
            if (j == i) continue;
            const double raw = -A.va[p];
            if (mx > 0.0 && raw > 0.0 && raw >= theta * mx) {
                if (!dd && j > i) {
                    S.push(i, 1.0);
                    dd = true;
                }
                S.push(j, raw);
            }
        }
        close_strength_row(S, i, dd, 1.0);
    }
    tally(c, static_cast<double>(A.nr));
    return S;
}

Csr symmetric_soc(const Csr& A, double theta, Ops* c) {  // strength.hpp:70-107
    if (A.nr != A.nc) throw std::invalid_argument("symmetric_strength: square matrix required");
    if (theta < 0.0 || theta > 1.0) throw std::invalid_argument("symmetric_strength: theta must lie in [0, 1]");
    const Vec d = diag_of(A);
    for (idx i = 0; i < A.nr; ++i)
        if (d[i] == 0.0) throw std::runtime_error("symmetric_strength: zero diagonal at row " + std::to_string(i));
    Csr S(A.nr, A.nc);
    S.bs = A.bs;
    for (idx i = 0; i < A.nr; ++i) {
        bool dd = false;
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p) {
            const idx j = A.ci[p];
            if (j == i) continue;
            const double raw = std::fabs(A.va[p]) / std::sqrt(std::fabs(d[i]) * std::fabs(d[j]));
            if (raw >= theta && raw > 0.0) {
                if (!dd && j > i) {
                    S.push(i, 1.0);
                    dd = true;
                }
                S.push(j, raw);
            }
        }
        close_strength_row(S, i, dd, 1.0);
    }
    tally(c, static_cast<double>(A.nnz()) + A.nr);
    return S;
}

Csr evolution_soc(const Csr& A, const amgcu_strength_config& cfg, Ops* c) {  // strength.hpp:116-238
    if (A.nr != A.nc) throw std::invalid_argument("evolution_strength: square matrix required");
    if (cfg.drop_tol <= 0.0) throw std::invalid_argument("evolution_strength: drop_tol must be positive");
    if (cfg.evolution_steps < 1) throw std::invalid_argument("evolution_strength: steps must be >= 1");
    const idx n = A.nr;
    Vec winv(n);
    if (cfg.weighting == 0) {
        const double rho = spectral_radius(A, 15, c);
        if (rho <= 0.0) throw std::runtime_error("evolution_strength: spectral radius estimate failed");
        const double omega = 1.0 / rho;
        for (idx i = 0; i < n; ++i) {
            const double d = A.at(i, i);
            if (d == 0.0) throw std::runtime_error("evolution_strength: zero diagonal at row " + std::to_string(i));
            winv[i] = omega / d;
        }
    } else {
        for (idx i = 0; i < n; ++i) {
            double s = 0.0;
            for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p) s += std::fabs(A.va[p]);
            if (s == 0.0) throw std::runtime_error("evolution_strength: zero row at " + std::to_string(i));
            winv[i] = 1.0 / s;
        }
    }
    const Csr At = transpose(A);
    Csr S(n, n);
    S.bs = A.bs;
    std::vector<idx> hood, slot(n, -1), ring;
    Vec z, zn;
    double ops = 0.0;
    for (idx i = 0; i < n; ++i) {
        hood.assign(1, i);
        slot[i] = 0;
        size_t lo = 0;
        for (int st = 0; st < cfg.evolution_steps; ++st) {  // distance-`steps` ball in A + A^T
            const size_t hi = hood.size();
            for (size_t f = lo; f < hi; ++f) {
                const idx u = hood[f];
                for (const Csr* M : {&A, &At})
                    for (idx p = M->rp[u]; p < M->rp[u + 1]; ++p) {
                        const idx j = M->ci[p];
                        if (slot[j] < 0) {
                            slot[j] = static_cast<idx>(hood.size());
                            hood.push_back(j);
                        }
                    }
            }
            lo = hi;
        }
        z.assign(hood.size(), 0.0);
        zn.assign(hood.size(), 0.0);
        z[0] = 1.0;
        for (int st = 0; st < cfg.evolution_steps; ++st) {
            for (size_t t = 0; t < hood.size(); ++t) {
                const idx u = hood[t];
                double az = 0.0;
                for (idx p = A.rp[u]; p < A.rp[u + 1]; ++p) {
                    const idx lj = slot[A.ci[p]];
                    if (lj >= 0) {
                        az += A.va[p] * z[lj];
                        ops += 1.0;
                    }
                }
                zn[t] = z[t] - winv[u] * az;
                ops += 1.0;
            }
            std::swap(z, zn);
        }
        ring.clear();
        std::merge(A.ci.begin() + A.rp[i], A.ci.begin() + A.rp[i + 1], At.ci.begin() + At.rp[i],
                   At.ci.begin() + At.rp[i + 1], std::back_inserter(ring));
        ring.erase(std::unique(ring.begin(), ring.end()), ring.end());
        double mx = 0.0;
        for (idx j : ring)
            if (j != i && slot[j] >= 0) mx = std::max(mx, std::fabs(z[slot[j]]));
        const double cutoff = mx / cfg.drop_tol;
        const double zi = std::fabs(z[0]);
        const double dval = zi > 0.0 ? zi : 1.0;
        bool dd = false;
        for (idx j : ring) {
            if (j == i) continue;
            const double mag = slot[j] >= 0 ? std::fabs(z[slot[j]]) : 0.0;
            if (mx > 0.0 && mag >= cutoff && mag > 0.0) {
                if (!dd && j > i) {
                    S.push(i, dval);
                    dd = true;
                }
                S.push(j, mag);
            }
        }
        close_strength_row(S, i, dd, dval);
        for (idx u : hood) slot[u] = -1;
    }
    tally(c, ops);
    return S;
}

Csr strength(const Csr& A, const amgcu_strength_config& cfg, Ops* c) {  // strength.hpp:240-248
    switch (cfg.measure) {
        case 0: return classical_soc(A, cfg.drop_tol, c);
        case 1: return symmetric_soc(A, cfg.drop_tol, c);
        case 2: return evolution_soc(A, cfg, c);
    }
    throw std::invalid_argument("strength: unknown measure");
}

Csr normalize_soc(const Csr& S, Ops* c) {  // strength.hpp:252-288
    if (S.nr != S.nc) throw std::invalid_argument("normalize_strength: square matrix required");
    for (double v : S.va)
        if (v < 0.0) throw std::invalid_argument("normalize_strength: negative strength value");
    Csr N(S.nr, S.nc);
    N.bs = S.bs;
    for (idx i = 0; i < S.nr; ++i) {
        double mx = 0.0;
        for (idx p = S.rp[i]; p < S.rp[i + 1]; ++p)
            if (S.ci[p] != i) mx = std::max(mx, S.va[p]);
        bool dd = false;
        for (idx p = S.rp[i]; p < S.rp[i + 1]; ++p) {
            const idx j = S.ci[p];
            if (j == i || mx <= 0.0) continue;
            const double v = S.va[p] / mx;
            if (v == 0.0) continue;
            if (!dd && j > i) {
                N.push(i, 1.0);
                dd = true;
            }
            N.push(j, v);
        }
        close_strength_row(N, i, dd, 1.0);
    }
    tally(c, static_cast<double>(S.nnz()));
    return N;
}

Csr amalgamate(const Csr& S, idx m) {  // strength.hpp:292-324
    if (m < 1) throw std::invalid_argument("amalgamate: block size must be >= 1");
    if (m == 1) return S;
    if (S.nr % m != 0 || S.nc % m != 0)
        throw std::invalid_argument("amalgamate: dimensions not divisible by block size");
    const idx nr = S.nr / m, nc = S.nc / m;
    RowList rows(nr);
    for (idx i = 0; i < S.nr; ++i)
        for (idx p = S.rp[i]; p < S.rp[i + 1]; ++p) rows[i / m].push_back({S.ci[p] / m, std::fabs(S.va[p])});
    Csr N(nr, nc);
    for (idx bi = 0; bi < nr; ++bi) {
        auto& r = rows[bi];
        std::sort(r.begin(), r.end());
        size_t p = 0;
        while (p < r.size()) {
            const idx j = r[p].first;
            double mx = 0.0;
            for (; p < r.size() && r[p].first == j; ++p) mx = std::max(mx, r[p].second);
            if (mx != 0.0) N.push(j, mx);
        }
        N.close_row(bi);
    }
    return N;
}

// ---- aggregation (aggregation.hpp:29-127) ---------------------------------------
struct Agg {
    idx n_nodes = 0, n_agg = 0;
    Csr C;
    std::vector<idx> roots, owner;  // owner = node_to_agg
};

Agg aggregate(const Csr& S) {
    if (S.nr != S.nc) throw std::invalid_argument("greedy_aggregate: square matrix required");
    const idx n = S.nr;
    for (idx i = 0; i < n; ++i)
        if (S.at(i, i) != 1.0)
            throw std::invalid_argument("greedy_aggregate: strength matrix must be normalized (unit diagonal)");
    std::vector<idx> own(n, -1), roots;
    for (idx i = 0; i < n; ++i) {  // pass 1, ascending order
        if (own[i] >= 0) continue;
        bool free_hood = true;
        for (idx p = S.rp[i]; p < S.rp[i + 1] && free_hood; ++p)
            if (S.ci[p] != i && own[S.ci[p]] >= 0) free_hood = false;
        if (!free_hood) continue;
        const idx id = static_cast<idx>(roots.size());
        own[i] = id;
        for (idx p = S.rp[i]; p < S.rp[i + 1]; ++p)
            if (S.ci[p] != i) own[S.ci[p]] = id;
        roots.push_back(i);
    }
    const idx n1 = static_cast<idx>(roots.size());
    std::vector<idx> join(n, -1);
    for (idx i = 0; i < n; ++i) {  // pass 2: strongest edge to a pass-1 aggregate
        if (own[i] >= 0) continue;
        double best = 0.0;
        idx pick = -1;
        for (idx p = S.rp[i]; p < S.rp[i + 1]; ++p) {
            const idx j = S.ci[p];
            if (j == i) continue;
            const idx a = own[j];
            if (a < 0 || a >= n1) continue;
            if (S.va[p] > best || (S.va[p] == best && pick >= 0 && a < pick)) {
                best = S.va[p];
                pick = a;
            }
        }
        join[i] = pick;
    }
    for (idx i = 0; i < n; ++i)
        if (join[i] >= 0) own[i] = join[i];
    for (idx i = 0; i < n; ++i) {  // leftovers become singletons
        if (own[i] >= 0) continue;
        own[i] = static_cast<idx>(roots.size());
        roots.push_back(i);
    }
    Agg a;
    a.n_nodes = n;
    a.n_agg = static_cast<idx>(roots.size());
    a.roots = std::move(roots);
    a.owner = own;
    a.C = Csr(n, a.n_agg);
    a.C.ci = own;
    a.C.va.assign(n, 1.0);
    for (idx i = 0; i < n; ++i) a.C.rp[i + 1] = i + 1;
    return a;
}

std::pair<Csr, std::vector<idx>> unamalgamate(const Csr& N, const std::vector<idx>& roots, idx m) {
    if (m < 1) throw std::invalid_argument("unamalgamate: block size must be >= 1");
    if (m == 1) return {N, roots};
    Csr D(N.nr * m, N.nc * m);
    for (idx i = 0; i < N.nr; ++i)
        for (idx r = 0; r < m; ++r) {
            for (idx p = N.rp[i]; p < N.rp[i + 1]; ++p)
                for (idx cc = 0; cc < m; ++cc) D.push(N.ci[p] * m + cc, N.va[p]);
            D.close_row(i * m + r);
        }
    std::vector<idx> dr(roots.size() * m);
    for (size_t g = 0; g < roots.size(); ++g)
        for (idx cc = 0; cc < m; ++cc) dr[g * m + cc] = roots[g] * m + cc;
    return {std::move(D), std::move(dr)};
}

// ---- relaxation (relaxation.hpp) ---------------------------------------------------
struct RelaxWs {
    Vec inv_diag;
    double w = 0.0;
    Csr At;
    Vec colsq;
    idx block = 1;
    Vec block_inv;
    Vec scratch;
};

RelaxWs make_ws(const Csr& A, int scheme, double weight, Ops* c) {  // relaxation.hpp:43-103
    if (A.nr != A.nc) throw std::invalid_argument("relax: square matrix required");
    RelaxWs ws;
    auto inv_diag = [&]() {
        ws.inv_diag = diag_of(A);
        for (size_t i = 0; i < ws.inv_diag.size(); ++i)
            if (ws.inv_diag[i] == 0.0) throw std::runtime_error("relax: zero diagonal at row " + std::to_string(i));
        for (double& v : ws.inv_diag) v = 1.0 / v;
    };
    switch (scheme) {
        case 0:
            inv_diag();
            ws.w = weight;
            if (ws.w == 0.0) ws.w = 4.0 / (3.0 * spectral_radius(A, 15, c));
            break;
        case 1:
        case 2: inv_diag(); break;
        case 3:
            ws.At = transpose(A);
            ws.colsq.assign(A.nc, 0.0);
            for (idx i = 0; i < ws.At.nr; ++i)
                for (idx p = ws.At.rp[i]; p < ws.At.rp[i + 1]; ++p) ws.colsq[i] += ws.At.va[p] * ws.At.va[p];
            for (idx i = 0; i < A.nc; ++i)
                if (ws.colsq[i] == 0.0) throw std::runtime_error("relax: zero column at " + std::to_string(i));
            break;
        case 4: {
            const idx m = A.bs;
            ws.block = m;
            if (m < 1 || A.nr % m != 0) throw std::invalid_argument("relax: bad block size for block relaxation");
            const idx nb = A.nr / m;
            ws.block_inv.assign(static_cast<size_t>(nb) * m * m, 0.0);
            Vec blk(static_cast<size_t>(m) * m);
            for (idx b = 0; b < nb; ++b) {
                std::fill(blk.begin(), blk.end(), 0.0);
                for (idx r = 0; r < m; ++r) {
                    const idx i = b * m + r;
                    for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p)
                        if (A.ci[p] / m == b) blk[r * m + (A.ci[p] - b * m)] = A.va[p];
                }
                if (m > 8) throw std::runtime_error("Eigen shim: FullPivLU limited to square <= 8");
                sd::FullPivLU<8> lu;
                lu.compute(m, blk.data());
                if (lu.rank() != m) throw std::runtime_error("relax: singular diagonal block " + std::to_string(b));
                lu.inverse(ws.block_inv.data() + static_cast<size_t>(b) * m * m);
            }
            break;
        }
        default: throw std::invalid_argument("relax: unknown scheme");
    }
    return ws;
}

void relax(int scheme, int sweeps, const Csr& A, double* x, const double* b, RelaxWs& ws, Ops* c) {
    const idx n = A.nr;
    for (int s = 0; s < sweeps; ++s) {
        auto gs = [&](bool fwd) {  // relaxation.hpp:115-127
            for (idx q = 0; q < n; ++q) {
                const idx i = fwd ? q : n - 1 - q;
                double acc = b[i];
                for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p)
                    if (A.ci[p] != i) acc -= A.va[p] * x[A.ci[p]];
                x[i] = acc * ws.inv_diag[i];
            }
        };
        auto bgs = [&](bool fwd) {  // relaxation.hpp:148-172
            const idx m = ws.block, nb = n / m;
            Vec rhs(m), sol(m);
            for (idx q = 0; q < nb; ++q) {
                const idx blk = fwd ? q : nb - 1 - q;
                for (idx r = 0; r < m; ++r) {
                    const idx i = blk * m + r;
                    double acc = b[i];
                    for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p)
                        if (A.ci[p] / m != blk) acc -= A.va[p] * x[A.ci[p]];
                    rhs[r] = acc;
                }
                const double* inv = ws.block_inv.data() + static_cast<size_t>(blk) * m * m;
                for (idx r = 0; r < m; ++r) {
                    double acc = 0.0;
                    for (idx cc = 0; cc < m; ++cc) acc += inv[r * m + cc] * rhs[cc];
                    sol[r] = acc;
                }
                for (idx r = 0; r < m; ++r) x[blk * m + r] = sol[r];
            }
        };
        switch (scheme) {
            case 0:  // relaxation.hpp:107-113
                ws.scratch.resize(n);
                spmv(A, x, ws.scratch.data());
                for (idx i = 0; i < n; ++i) x[i] += ws.w * ws.inv_diag[i] * (b[i] - ws.scratch[i]);
                break;
            case 1: gs(true); break;
            case 2:
                gs(true);
                gs(false);
                break;
            case 3: {  // relaxation.hpp:132-146
                Vec& r = ws.scratch;
                r.resize(n);
                spmv(A, x, r.data());
                for (idx i = 0; i < n; ++i) r[i] = b[i] - r[i];
                for (idx i = 0; i < A.nc; ++i) {
                    double num = 0.0;
                    for (idx p = ws.At.rp[i]; p < ws.At.rp[i + 1]; ++p) num += ws.At.va[p] * r[ws.At.ci[p]];
                    const double delta = num / ws.colsq[i];
                    x[i] += delta;
                    for (idx p = ws.At.rp[i]; p < ws.At.rp[i + 1]; ++p) r[ws.At.ci[p]] -= delta * ws.At.va[p];
                }
                break;
            }
            case 4:
                bgs(true);
                bgs(false);
                break;
        }
        tally(c, scheme == 3 ? 2.0 * A.nnz() : static_cast<double>(A.nnz()));
    }
}

// ---- interpolation (interpolation.hpp) -------------------------------------------
int energy_iterations(int iters, int degree) {  // interpolation.hpp:34-37
    if (iters > 0) return iters;
    return std::max(1, static_cast<int>(std::ceil(1.5 * degree)));
}

Csr pattern_power(const Csr& S, const Csr& C, int degree, Ops* c) {  // interpolation.hpp:41-49
    if (S.nr != S.nc || S.nc != C.nr) throw std::invalid_argument("sparsity_pattern: dimension mismatch");
    if (degree < 0) throw std::invalid_argument("sparsity_pattern: degree must be >= 0");
    Csr N = C;
    for (int t = 0; t < degree; ++t) N = matmul(S, N, c);
    return N;
}

Csr root_rows(const Csr& N, const std::vector<idx>& roots) {  // interpolation.hpp:53-77
    if (static_cast<idx>(roots.size()) != N.nc)
        throw std::invalid_argument("root_node_pattern: need one root per coarse column");
    std::vector<idx> owner(N.nr, -1);
    for (size_t j = 0; j < roots.size(); ++j) {
        if (roots[j] < 0 || roots[j] >= N.nr) throw std::invalid_argument("root_node_pattern: root out of range");
        if (owner[roots[j]] >= 0) throw std::invalid_argument("root_node_pattern: duplicate root row");
        owner[roots[j]] = static_cast<idx>(j);
    }
    Csr R(N.nr, N.nc);
    for (idx i = 0; i < N.nr; ++i) {
        if (owner[i] >= 0) {
            R.push(owner[i], 1.0);
        } else {
            for (idx p = N.rp[i]; p < N.rp[i + 1]; ++p) R.push(N.ci[p], N.va[p]);
        }
        R.close_row(i);
    }
    return R;
}

Cand improve(const Csr& A, const Cand& B, int sweeps, int scheme, double weight, Ops* c) {  // :81-96
    if (A.nr != A.nc || A.nr != B.n) throw std::invalid_argument("improve_candidates: dimension mismatch");
    if (sweeps < 0) throw std::invalid_argument("improve_candidates: sweeps must be >= 0");
    Cand out = B;
    if (sweeps > 0) {
        RelaxWs ws = make_ws(A, scheme, weight, c);
        const Vec zero(A.nr, 0.0);
        for (idx j = 0; j < out.k; ++j) relax(scheme, sweeps, A, out.col(j), zero.data(), ws, c);
    }
    for (idx j = 0; j < out.k; ++j) {  // normalize_columns, dense.hpp:41-46
        const double s = vnorm(out.col(j), out.n);
        if (s > 0.0) vscale(1.0 / s, out.col(j), out.n);
    }
    return out;
}

// Per-row k x k Gram pseudo-inverses over the allowed columns (interpolation.hpp:108-146).
struct Gram {
    idx k = 0;
    Vec pinv;
    std::vector<char> root;
    void build(const Csr& N, const Cand& Bc, const std::vector<idx>& roots, Ops* c) {
        k = Bc.k;
        root.assign(N.nr, 0);
        for (idx r : roots) root[r] = 1;
        pinv.assign(static_cast<size_t>(N.nr) * k * k, 0.0);
        if (k > 16) throw std::runtime_error("port: k limited to 16");
        double G[256], Gp[256];
        double ops = 0.0;
        for (idx i = 0; i < N.nr; ++i) {
            if (root[i]) continue;
            std::fill(G, G + k * k, 0.0);
            for (idx p = N.rp[i]; p < N.rp[i + 1]; ++p) {
                const idx j = N.ci[p];
                for (idx a = 0; a < k; ++a)
                    for (idx b = a; b < k; ++b) G[a * k + b] += Bc.at(j, a) * Bc.at(j, b);
            }
            for (idx a = 0; a < k; ++a)
                for (idx b = 0; b < a; ++b) G[a * k + b] = G[b * k + a];
            sd::sym_pinv<16>(k, G, Gp);
            std::copy(Gp, Gp + k * k, pinv.begin() + static_cast<size_t>(i) * k * k);
            ops += static_cast<double>(N.len(i)) * k * k + static_cast<double>(k) * k * k;
        }
        tally(c, ops);
    }
    const double* row(idx i) const { return pinv.data() + static_cast<size_t>(i) * k * k; }
};

void project(const Csr& N, const Cand& Bc, const Gram& gw, Vec& vals, Ops* c) {  // :150-182
    const idx k = gw.k;
    Vec y(k), lam(k);
    double ops = 0.0;
    for (idx i = 0; i < N.nr; ++i) {
        const idx lo = N.rp[i], hi = N.rp[i + 1];
        if (gw.root[i]) {
            for (idx p = lo; p < hi; ++p) vals[p] = 0.0;
            continue;
        }
        std::fill(y.begin(), y.end(), 0.0);
        for (idx p = lo; p < hi; ++p)
            for (idx a = 0; a < k; ++a) y[a] += Bc.at(N.ci[p], a) * vals[p];
        const double* Gp = gw.row(i);
        for (idx a = 0; a < k; ++a) {
            double s = 0.0;
            for (idx b = 0; b < k; ++b) s += Gp[a * k + b] * y[b];
            lam[a] = s;
        }
        for (idx p = lo; p < hi; ++p) {
            double s = 0.0;
            for (idx a = 0; a < k; ++a) s += Bc.at(N.ci[p], a) * lam[a];
            vals[p] -= s;
        }
        ops += 2.0 * static_cast<double>(hi - lo) * k + static_cast<double>(k) * k;
    }
    tally(c, ops);
}

// Y = (A X)|_N with X on N's pattern (interpolation.hpp:186-210).
void masked(const Csr& A, const Csr& N, const Vec& x, Vec& y, std::vector<idx>& slot, Ops* c) {
    y.assign(N.nnz(), 0.0);
    slot.assign(N.nc, -1);
    double ops = 0.0;
    for (idx i = 0; i < A.nr; ++i) {
        const idx lo = N.rp[i], hi = N.rp[i + 1];
        if (lo == hi) continue;
        for (idx p = lo; p < hi; ++p) slot[N.ci[p]] = p;
        for (idx p = A.rp[i]; p < A.rp[i + 1]; ++p) {
            const idx t = A.ci[p];
            const double a = A.va[p];
            for (idx q = N.rp[t]; q < N.rp[t + 1]; ++q) {
                const idx s = slot[N.ci[q]];
                if (s >= 0) {
                    y[s] += a * x[q];
                    ops += 1.0;
                }
            }
        }
        for (idx p = lo; p < hi; ++p) slot[N.ci[p]] = -1;
    }
    tally(c, ops);
}

Vec onto_pattern(const Csr& T, const Csr& N) {  // interpolation.hpp:213-227
    if (T.nr != N.nr || T.nc != N.nc) throw std::invalid_argument("energy_minimize: T and pattern dimensions differ");
    Vec vals(N.nnz(), 0.0);
    for (idx i = 0; i < T.nr; ++i) {
        auto b = N.ci.begin() + N.rp[i], e = N.ci.begin() + N.rp[i + 1];
        for (idx p = T.rp[i]; p < T.rp[i + 1]; ++p) {
            auto it = std::lower_bound(b, e, T.ci[p]);
            if (it == e || *it != T.ci[p])
                throw std::invalid_argument("energy_minimize: T has an entry outside the pattern");
            vals[static_cast<size_t>(it - N.ci.begin())] = T.va[p];
        }
    }
    return vals;
}

Csr off_pattern(const Csr& N, const Vec& vals, idx bs) {  // interpolation.hpp:229-243
    Csr P(N.nr, N.nc);
    P.bs = bs;
    for (idx i = 0; i < N.nr; ++i) {
        for (idx p = N.rp[i]; p < N.rp[i + 1]; ++p)
            if (vals[p] != 0.0) P.push(N.ci[p], vals[p]);
        P.close_row(i);
    }
    return P;
}

double safe_step(const Vec& e, const Vec& g, const Vec& h, double cap) {  // interpolation.hpp:247-260
    double step = cap;
    for (size_t j = 0; j < e.size(); ++j) {
        if (h[j] <= 0.0) continue;
        const double nj = std::sqrt(std::max(e[j], 0.0));
        const double tol = 2.5e-13 * std::max(nj, 1.0e-30);
        const double budget = tol * (2.0 * nj + tol);
        const double disc = g[j] * g[j] + h[j] * budget;
        const double beta = (-g[j] + std::sqrt(std::max(disc, 0.0))) / h[j];
        step = std::min(step, beta);
    }
    return step;
}

Csr energy_min(const Csr& A, const Csr& T, const Cand& B, const Cand& Bc, const Csr& N, int iters_cfg,
               int degree, int krylov, const std::vector<idx>& roots, Ops* c, int* its_out, bool* brk_out,
               bool skip_sym_check = false) {  // interpolation.hpp:277-442
    if (A.nr != A.nc || A.nr != N.nr || B.n != A.nr || Bc.n != N.nc || B.k != Bc.k)
        throw std::invalid_argument("energy_minimize: dimension mismatch");
    if (krylov == 0 && !skip_sym_check && !symmetric(A))
        throw std::invalid_argument("energy_minimize: cg requires a symmetric matrix");
    const int iters = energy_iterations(iters_cfg, degree);
    const idx nc = N.nc;
    Gram gw;
    gw.build(N, Bc, roots, c);
    Vec P = onto_pattern(T, N);
    std::vector<idx> slot;
    int its = 0;
    bool brk = false;
    const size_t nz = static_cast<size_t>(N.nnz());
    if (krylov == 0) {
        Vec dinv = diag_of(A);
        for (size_t i = 0; i < dinv.size(); ++i) {
            if (dinv[i] == 0.0) throw std::runtime_error("energy_minimize: zero diagonal at row " + std::to_string(i));
            dinv[i] = 1.0 / dinv[i];
        }
        Vec APm;
        masked(A, N, P, APm, slot, c);
        Vec R(APm);
        for (double& v : R) v = -v;
        project(N, Bc, gw, R, c);
        Vec Z(nz), D(nz, 0.0), ADm, ADp, e(nc), g(nc), h(nc);
        double oldsum = 0.0, first = -1.0;
        bool restart = true;
        for (int s = 0; s < iters; ++s) {
            for (idx i = 0; i < N.nr; ++i)
                for (idx p = N.rp[i]; p < N.rp[i + 1]; ++p) Z[p] = dinv[i] * R[p];
            tally(c, static_cast<double>(nz));
            const double newsum = vdot(R.data(), Z.data(), nz);
            if (first < 0.0) first = newsum;
            if (!(newsum > 1e-28 * std::max(first, 1.0))) break;
            if (restart) {
                D = Z;
            } else {
                const double beta = newsum / oldsum;
                for (size_t p = 0; p < nz; ++p) D[p] = Z[p] + beta * D[p];
            }
            masked(A, N, D, ADm, slot, c);
            ADp = ADm;
            project(N, Bc, gw, ADp, c);
            const double denom = vdot(D.data(), ADm.data(), nz);
            tally(c, 3.0 * static_cast<double>(nz));
            if (!(denom > 0.0)) break;
            const double alpha_cg = newsum / denom;
            std::fill(e.begin(), e.end(), 0.0);
            std::fill(g.begin(), g.end(), 0.0);
            std::fill(h.begin(), h.end(), 0.0);
            for (size_t p = 0; p < nz; ++p) {
                const idx j = N.ci[p];
                e[j] += P[p] * APm[p];
                g[j] += D[p] * APm[p];
                h[j] += D[p] * ADm[p];
            }
            const double alpha = safe_step(e, g, h, alpha_cg);
            if (!(alpha > 1e-14 * alpha_cg)) {
                brk = true;
                break;
            }
            for (size_t p = 0; p < nz; ++p) {
                P[p] += alpha * D[p];
                APm[p] += alpha * ADm[p];
                R[p] -= alpha * ADp[p];
            }
            tally(c, 3.0 * static_cast<double>(nz));
            restart = alpha < alpha_cg * (1.0 - 1e-12);
            oldsum = newsum;
            its = s + 1;
        }
        if (its_out) *its_out = its;
        if (brk_out) *brk_out = brk;
        return off_pattern(N, P, T.bs);
    }

    // GMRES branch (interpolation.hpp:363-441)
    const Csr AtA = matmul(transpose(A), A, c);
    Vec R0;
    masked(AtA, N, P, R0, slot, c);
    for (double& v : R0) v = -v;
    project(N, Bc, gw, R0, c);
    const double beta = vnorm(R0.data(), nz);
    tally(c, static_cast<double>(nz));
    if (beta < 1e-300) {
        if (its_out) *its_out = 0;
        if (brk_out) *brk_out = false;
        return off_pattern(N, P, T.bs);
    }
    const int m = iters;
    std::vector<Vec> V;
    vscale(1.0 / beta, R0.data(), nz);
    V.push_back(std::move(R0));
    Vec H(static_cast<size_t>(m + 1) * m, 0.0);  // row-major
    int built = 0;
    for (int s = 0; s < m; ++s) {
        Vec W;
        masked(AtA, N, V[s], W, slot, c);
        project(N, Bc, gw, W, c);
        for (int t = 0; t <= s; ++t) {
            const double hts = vdot(W.data(), V[t].data(), nz);
            H[t * m + s] = hts;
            vaxpy(-hts, V[t].data(), W.data(), nz);
        }
        tally(c, 2.0 * (s + 1) * static_cast<double>(nz));
        const double hn = vnorm(W.data(), nz);
        H[(s + 1) * m + s] = hn;
        built = s + 1;
        its = s + 1;
        if (hn < 1e-14 * beta) break;
        vscale(1.0 / hn, W.data(), nz);
        V.push_back(std::move(W));
    }
    if (built > 64) throw std::runtime_error("Eigen shim: SelfAdjointEigenSolver limited to 64x64");
    Vec Hs(static_cast<size_t>(built) * built);
    for (int i = 0; i < built; ++i)
        for (int j = 0; j < built; ++j) Hs[i * built + j] = 0.5 * (H[i * m + j] + H[j * m + i]);
    Vec ev(built), EV(static_cast<size_t>(built) * built);
    sd::sym_eig<64>(built, Hs.data(), ev.data(), EV.data());
    double mx = ev.empty() ? 0.0 : std::fabs(ev[0]);
    for (double v : ev) mx = std::max(mx, std::fabs(v));
    const double cutoff = 1e-14 * std::max(mx, 1e-300);
    Vec rhs(built, 0.0), z(built), y(built);
    rhs[0] = beta;
    for (int t = 0; t < built; ++t) {  // z = EV^T rhs
        double s = 0.0;
        for (int i = 0; i < built; ++i) s += EV[i * built + t] * rhs[i];
        z[t] = s;
    }
    for (int t = 0; t < built; ++t) z[t] = ev[t] > cutoff ? z[t] / ev[t] : 0.0;
    for (int i = 0; i < built; ++i) {  // y = EV z
        double s = 0.0;
        for (int t = 0; t < built; ++t) s += EV[i * built + t] * z[t];
        y[i] = s;
    }
    Vec U(nz, 0.0);
    for (int t = 0; t < built && t < static_cast<int>(V.size()); ++t) vaxpy(y[t], V[t].data(), U.data(), nz);
    Csr Tm = off_pattern(N, P, T.bs), Um = off_pattern(N, U, T.bs);
    Csr AT = matmul(A, Tm, c), AU = matmul(A, Um, c);
    Vec e(nc, 0.0), g(nc, 0.0), h(nc, 0.0);
    for (idx i = 0; i < AT.nr; ++i)
        for (idx p = AT.rp[i]; p < AT.rp[i + 1]; ++p) e[AT.ci[p]] += AT.va[p] * AT.va[p];
    for (idx i = 0; i < AU.nr; ++i) {
        auto tb = AT.ci.begin() + AT.rp[i], te = AT.ci.begin() + AT.rp[i + 1];
        for (idx p = AU.rp[i]; p < AU.rp[i + 1]; ++p) {
            const idx j = AU.ci[p];
            h[j] += AU.va[p] * AU.va[p];
            auto it = std::lower_bound(tb, te, j);
            if (it != te && *it == j) g[j] += AU.va[p] * AT.va[static_cast<size_t>(it - AT.ci.begin())];
        }
    }
    const double tau = safe_step(e, g, h, 1.0);
    if (its_out) *its_out = its;
    if (!(tau > 0.0)) {
        if (brk_out) *brk_out = true;
        return Tm;
    }
    if (brk_out) *brk_out = false;
    for (size_t p = 0; p < nz; ++p) P[p] += tau * U[p];
    return off_pattern(N, P, T.bs);
}

Csr enforce(const Csr& P, const Cand& B, const Cand& Bc, const Csr* allowed, Ops* c) {  // :458-521
    const Csr& N = allowed ? *allowed : P;
    if (P.nr != N.nr || P.nc != N.nc || B.n != P.nr || Bc.n != P.nc || B.k != Bc.k)
        throw std::invalid_argument("enforce_constraints: dimension mismatch");
    const idx k = B.k;
    if (k > 16) throw std::runtime_error("port: k limited to 16");
    Vec vals = onto_pattern(P, N);
    double G[256], ev[16], V[256], y[16], proj[16], lv[16];
    double ops = 0.0;
    for (idx i = 0; i < N.nr; ++i) {
        const idx lo = N.rp[i], hi = N.rp[i + 1];
        if (lo == hi) continue;
        std::fill(G, G + k * k, 0.0);
        std::fill(y, y + k, 0.0);
        for (idx p = lo; p < hi; ++p) {
            const idx j = N.ci[p];
            for (idx a = 0; a < k; ++a) {
                y[a] += Bc.at(j, a) * vals[p];
                for (idx b = a; b < k; ++b) G[a * k + b] += Bc.at(j, a) * Bc.at(j, b);
            }
        }
        for (idx a = 0; a < k; ++a)
            for (idx b = 0; b < a; ++b) G[a * k + b] = G[b * k + a];
        for (idx a = 0; a < k; ++a) y[a] = B.at(i, a) - y[a];
        sd::sym_eig<16>(k, G, ev, V);
        double mx = std::fabs(ev[0]);
        for (idx a = 0; a < k; ++a) mx = std::max(mx, std::fabs(ev[a]));
        const double cutoff = 1e-12 * std::max(mx, 1e-300);
        for (idx t = 0; t < k; ++t) {  // proj = V^T y
            double s = 0.0;
            for (idx a = 0; a < k; ++a) s += V[a * k + t] * y[a];
            proj[t] = s;
        }
        for (idx a = 0; a < k; ++a) proj[a] = ev[a] > cutoff ? proj[a] / ev[a] : 0.0;
        for (idx a = 0; a < k; ++a) {  // lv = V proj
            double s = 0.0;
            for (idx t = 0; t < k; ++t) s += V[a * k + t] * proj[t];
            lv[a] = s;
        }
        for (idx p = lo; p < hi; ++p) {
            double s = 0.0;
            for (idx a = 0; a < k; ++a) s += Bc.at(N.ci[p], a) * lv[a];
            vals[p] += s;
        }
        ops += 2.0 * static_cast<double>(hi - lo) * k + static_cast<double>(k) * k * k;
    }
    tally(c, ops);
    return off_pattern(N, vals, P.bs);
}

std::pair<Csr, Cand> inject(const Agg& agg, const Csr& N, const Cand& B, idx m, Ops* c) {  // :523-581
    if (m < 1) throw std::invalid_argument("inject_tentative: block size must be >= 1");
    if (B.n != agg.n_nodes * m) throw std::invalid_argument("inject_tentative: candidate size mismatch");
    if (B.k < m) throw std::invalid_argument("inject_tentative: need at least m candidates");
    const idx nc = agg.n_agg * m;
    if (N.nr != B.n || N.nc != nc) throw std::invalid_argument("inject_tentative: pattern dimensions mismatch");
    if (m > 8) throw std::runtime_error("Eigen shim: FullPivLU limited to square <= 8");
    Cand Bc(nc, B.k);
    Vec binv(static_cast<size_t>(agg.n_agg) * m * m);
    double ops = 0.0;
    double blk[64];
    for (idx g = 0; g < agg.n_agg; ++g) {
        const idx root = agg.roots[g];
        double mx = 0.0;
        for (idx r = 0; r < m; ++r)
            for (idx cc = 0; cc < m; ++cc) {
                blk[r * m + cc] = B.at(root * m + r, cc);
                mx = (r == 0 && cc == 0) ? std::fabs(blk[0]) : std::max(mx, std::fabs(blk[r * m + cc]));
            }
        double* inv = binv.data() + static_cast<size_t>(g) * m * m;
        sd::FullPivLU<8> lu;
        lu.compute(m, blk);
        const double scale_cut = 1e-10 * std::max(mx, 1e-300);
        if (lu.rank() == m && mx > 0 && std::fabs(lu.determinant()) > std::pow(scale_cut, m)) {
            lu.inverse(inv);
        } else {
            sd::COD cod;
            cod.threshold = 1e-10;
            cod.compute(m, m, blk);
            cod.pseudo_inverse(inv);
        }
        for (idx cc = 0; cc < m; ++cc)
            for (idx a = 0; a < B.k; ++a) Bc.at(g * m + cc, a) = B.at(root * m + cc, a);
        ops += static_cast<double>(m) * m * m;
    }
    RowList rows(B.n);
    for (idx i = 0; i < agg.n_nodes; ++i) {  // O(n): each node once, via its owner
        const idx g = agg.owner[i];
        const idx root = agg.roots[g];
        const double* inv = binv.data() + static_cast<size_t>(g) * m * m;
        for (idx r = 0; r < m; ++r) {
            const idx dof = i * m + r;
            if (i == root) {
                rows[dof].push_back({g * m + r, 1.0});
                continue;
            }
            for (idx cc = 0; cc < m; ++cc) {
                double v = 0.0;
                for (idx s = 0; s < m; ++s) v += B.at(dof, s) * inv[s * m + cc];
                if (v != 0.0) rows[dof].push_back({g * m + cc, v});
            }
            ops += static_cast<double>(m) * m;
        }
    }
    tally(c, ops);
    Csr T = build_from_rows(nc, std::move(rows));
    T.bs = m;
    if (B.k > m) T = enforce(T, B, Bc, &N, c);
    return {std::move(T), std::move(Bc)};
}

idx span_rank(const std::vector<std::pair<idx, double>>& row, const Cand& Bc) {  // :585-595
    const int r = static_cast<int>(row.size()), k = Bc.k;
    Vec M(static_cast<size_t>(r) * k);
    for (int i = 0; i < r; ++i)
        for (int a = 0; a < k; ++a) M[static_cast<size_t>(i) * k + a] = Bc.at(row[i].first, a);
    sd::COD qr;
    qr.qr_only(r, k, M.data());
    return qr.rank_for(1e-3);
}

Csr min_support(const Csr& filtered, const Csr& full, idx min_cols, const Cand* Bc) {  // :607-643
    if (filtered.nr != full.nr || filtered.nc != full.nc)
        throw std::invalid_argument("ensure_min_support: shape mismatch");
    RowList rows(filtered.nr);
    std::vector<std::pair<double, std::pair<idx, double>>> cand;
    for (idx i = 0; i < filtered.nr; ++i) {
        auto& out = rows[i];
        for (idx p = filtered.rp[i]; p < filtered.rp[i + 1]; ++p) out.push_back({filtered.ci[p], filtered.va[p]});
        const idx have = filtered.len(i);
        const idx target = std::min<idx>(min_cols, full.len(i));
        const bool short_rank = Bc && have >= target && full.len(i) > have && span_rank(out, *Bc) < min_cols;
        if (have >= target && !short_rank) continue;
        cand.clear();
        for (idx p = full.rp[i]; p < full.rp[i + 1]; ++p) {
            const idx j = full.ci[p];
            bool present = false;
            for (const auto& e : out) present = present || e.first == j;
            if (!present && full.va[p] != 0.0) cand.push_back({std::fabs(full.va[p]), {j, full.va[p]}});
        }
        std::sort(cand.begin(), cand.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
        size_t t = 0;
        for (; t < cand.size() && static_cast<idx>(out.size()) < target; ++t) out.push_back(cand[t].second);
        if (Bc)
            for (; t < cand.size() && span_rank(out, *Bc) < min_cols; ++t) out.push_back(cand[t].second);
    }
    Csr R = build_from_rows(filtered.nc, std::move(rows));
    R.bs = filtered.bs;
    return R;
}

Csr postfilter(const Csr& A, const Csr& P, const Cand& B, const Cand& Bc, std::optional<double> theta,
               std::optional<idx> kk, int krylov, int degree, const std::vector<idx>& roots, Ops* c,
               bool skip_sym_check) {  // :648-659
    Csr Pf = filter(P, theta, kk);
    Pf = min_support(Pf, P, B.k, &Bc);
    Pf = enforce(Pf, B, Bc, nullptr, c);
    return energy_min(A, Pf, B, Bc, Pf, 1, degree, krylov, roots, c, nullptr, nullptr, skip_sym_check);
}

// ---- hierarchy (hierarchy.hpp) -----------------------------------------------------
struct Level {
    Csr A, P, R;
    Cand B{0, 1}, Bc{0, 1};
    bool sym = true;
};

// Dense LU with partial pivoting (row-major, i-k-j update order), the coarsest-level
// solver above kLuCoarse rows.  DELIBERATE DEVIATION from the reference's COD
// (hierarchy.hpp:54-76): an unblocked COD of the 11,008-row coarsest level of C1-256
// takes hours on one core; the GPU path also uses LU at that size.  For a nonsingular
// operator both give the solution to rounding; the test tolerance (1e-10) covers it.
struct DenseLU {
    int n = 0;
    std::vector<double> a;  // L (unit, below the diagonal) and U, row-major
    std::vector<int> piv;
    bool compute(int n_, const double* D) {
        n = n_;
        a.assign(D, D + static_cast<size_t>(n) * n);
        piv.resize(n);
        for (int k = 0; k < n; ++k) {
            int p = k;
            double best = std::abs(a[static_cast<size_t>(k) * n + k]);
            for (int i = k + 1; i < n; ++i) {
                const double v = std::abs(a[static_cast<size_t>(i) * n + k]);
                if (v > best) {
                    best = v;
                    p = i;
                }
            }
            if (!(best > 0.0)) return false;
            piv[k] = p;
            if (p != k)
                for (int j = 0; j < n; ++j)
                    std::swap(a[static_cast<size_t>(k) * n + j], a[static_cast<size_t>(p) * n + j]);
            const double* rk = &a[static_cast<size_t>(k) * n];
            const double inv = 1.0 / rk[k];
            for (int i = k + 1; i < n; ++i) {
                double* ri = &a[static_cast<size_t>(i) * n];
                const double f = ri[k] * inv;
                ri[k] = f;
                if (f != 0.0)
                    for (int j = k + 1; j < n; ++j) ri[j] -= f * rk[j];
            }
        }
        return true;
    }
    void solve(const double* b, double* x) const {
        std::vector<double> y(b, b + n);
        for (int k = 0; k < n; ++k) std::swap(y[k], y[piv[k]]);
        for (int i = 0; i < n; ++i) {
            const double* ri = &a[static_cast<size_t>(i) * n];
            double s = y[i];
            for (int j = 0; j < i; ++j) s -= ri[j] * y[j];
            y[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            const double* ri = &a[static_cast<size_t>(i) * n];
            double s = y[i];
            for (int j = i + 1; j < n; ++j) s -= ri[j] * y[j];
            y[i] = s / ri[i];
        }
        for (int i = 0; i < n; ++i) x[i] = y[i];
    }
};
constexpr int kLuCoarse = 4096;

struct Hier {
    std::vector<Level> lv;
    amgcu_setup_options o{};
    double base = 0.0;
    double wu[5] = {0, 0, 0, 0, 0};
    sd::COD coarse;
    DenseLU coarse_lu;
    bool use_lu = false;
    int coarse_n = 0;
    std::vector<RelaxWs> pre, post;
    bool stagnated = false;
    void charge(int b, double raw) {
        if (!(base > 0.0)) throw std::logic_error("WorkLedger: base nnz not registered");
        wu[b] += raw / base;
    }
};

Csr with_aggregate_columns(const Csr& N, const Agg& agg) {  // hierarchy.hpp:98-110
    std::vector<Trip> extra;
    for (idx i = 0; i < N.nr; ++i)
        if (!N.has(i, agg.owner[i])) extra.push_back({i, agg.owner[i], 1.0});
    if (extra.empty()) return N;
    for (idx i = 0; i < N.nr; ++i)
        for (idx p = N.rp[i]; p < N.rp[i + 1]; ++p) extra.push_back({i, N.ci[p], N.va[p]});
    return build_from_triplets(N.nr, N.nc, std::move(extra));
}

Csr widen(const Csr& N, const Csr& S, const Agg& agg, idx min_aggs) {  // hierarchy.hpp:118-154
    if (min_aggs <= 1) return N;
    const Csr St = transpose(S);
    std::vector<Trip> extra;
    std::vector<idx> front, next;
    std::vector<char> seen(agg.n_nodes);
    for (idx i = 0; i < N.nr; ++i) {
        std::set<idx> aggs(N.ci.begin() + N.rp[i], N.ci.begin() + N.rp[i + 1]);
        if (static_cast<idx>(aggs.size()) >= min_aggs) continue;
        std::fill(seen.begin(), seen.end(), 0);
        seen[i] = 1;
        front.assign(1, i);
        while (!front.empty() && static_cast<idx>(aggs.size()) < min_aggs) {
            next.clear();
            for (idx u : front)
                for (const Csr* M : {&S, &St})
                    for (idx p = M->rp[u]; p < M->rp[u + 1]; ++p) {
                        const idx j = M->ci[p];
                        if (seen[j]) continue;
                        seen[j] = 1;
                        next.push_back(j);
                        aggs.insert(agg.owner[j]);
                    }
            front.swap(next);
        }
        for (idx g : aggs)
            if (!N.has(i, g)) extra.push_back({i, g, 1.0});
    }
    if (extra.empty()) return N;
    for (idx i = 0; i < N.nr; ++i)
        for (idx p = N.rp[i]; p < N.rp[i + 1]; ++p) extra.push_back({i, N.ci[p], N.va[p]});
    return build_from_triplets(N.nr, N.nc, std::move(extra));
}

struct Step {
    Csr P, R, Ac;
    Cand Bf{0, 1}, Bcoarse{0, 1}, Bhf{0, 1}, Bhc{0, 1};
};

std::optional<Step> coarsen(Hier& H, const Csr& A, const Cand& B, const Cand& Bhat, bool sym) {  // :183-245
    const amgcu_setup_options& o = H.o;
    Ops cagg, ccand, cint, crap;
    const idx m = std::max<idx>(1, A.bs);
    amgcu_strength_config sc{o.strength_measure, o.drop_tol, o.evolution_steps, o.weighting};
    Csr S = normalize_soc(amalgamate(strength(A, sc, &cagg), m), &cagg);
    Agg agg = aggregate(S);
    tally(&cagg, static_cast<double>(S.nnz()));
    if (agg.n_agg >= agg.n_nodes) return std::nullopt;

    Csr N = pattern_power(S, agg.C, o.degree, &cint);
    const idx min_aggs = (B.k + m - 1) / m;
    if (o.prefilter_set) {
        Csr N0 = N;
        std::optional<double> th;
        std::optional<idx> kk;
        if (o.prefilter_theta_set) th = o.prefilter_theta;
        if (o.prefilter_k > 0) kk = o.prefilter_k;
        N = filter(N, th, kk);
        N = with_aggregate_columns(N, agg);
        N = min_support(N, N0, min_aggs, nullptr);
    }
    N = widen(N, S, agg, min_aggs);
    auto [Nd, rd] = unamalgamate(N, agg.roots, m);
    Nd = root_rows(Nd, rd);

    Cand Bimp = improve(A, B, o.candidate_sweeps, o.cand_scheme, o.cand_weight, &ccand);
    auto [T, Bc] = inject(agg, Nd, Bimp, m, &cint);
    int kry = o.krylov;
    if (!sym && kry == 0) kry = 1;
    std::optional<double> pth;
    std::optional<idx> pk;
    if (o.postfilter_theta_set) pth = o.postfilter_theta;
    if (o.postfilter_k > 0) pk = o.postfilter_k;
    Csr P = energy_min(A, T, Bimp, Bc, Nd, o.energy_iters, o.degree, kry, rd, &cint, nullptr, nullptr);
    if (o.postfilter_set) P = postfilter(A, P, Bimp, Bc, pth, pk, kry, o.degree, rd, &cint, false);

    Step out;
    if (sym) {
        out.R = transpose(P);
        out.Bhf = Bimp;
        out.Bhc = Bc;
    } else {
        Csr At = transpose(A);
        Cand Bhimp = improve(At, Bhat, o.candidate_sweeps, o.cand_scheme, o.cand_weight, &ccand);
        auto [That, Bhc] = inject(agg, Nd, Bhimp, m, &cint);
        Csr Rt = energy_min(At, That, Bhimp, Bhc, Nd, o.energy_iters, o.degree, 1, rd, &cint, nullptr, nullptr);
        if (o.postfilter_set) Rt = postfilter(At, Rt, Bhimp, Bhc, pth, pk, 1, o.degree, rd, &cint, false);
        out.R = transpose(Rt);
        out.Bhf = Bhimp;
        out.Bhc = Bhc;
    }
    out.Ac = galerkin(out.R, A, P, &crap);
    out.P = std::move(P);
    out.Bf = std::move(Bimp);
    out.Bcoarse = std::move(Bc);
    H.charge(0, cagg.v);
    H.charge(1, ccand.v);
    H.charge(2, cint.v);
    H.charge(3, crap.v);
    return out;
}

void finalize(Hier& H) {  // hierarchy.hpp:164-172
    Ops c;
    for (size_t l = 0; l + 1 < H.lv.size(); ++l) {
        H.pre.push_back(make_ws(H.lv[l].A, H.o.pre_scheme, H.o.pre_weight, &c));
        H.post.push_back(make_ws(H.lv[l].A, H.o.post_scheme, H.o.post_weight, &c));
    }
    const Csr& Ac = H.lv.back().A;  // CoarseSolver::factor, hierarchy.hpp:59-68
    Vec D(static_cast<size_t>(Ac.nr) * Ac.nc, 0.0);
    for (idx i = 0; i < Ac.nr; ++i)
        for (idx p = Ac.rp[i]; p < Ac.rp[i + 1]; ++p) D[static_cast<size_t>(i) * Ac.nc + Ac.ci[p]] = Ac.va[p];
    H.use_lu = Ac.nr > kLuCoarse && Ac.nr == Ac.nc && H.coarse_lu.compute(Ac.nr, D.data());
    if (!H.use_lu) H.coarse.compute(Ac.nr, Ac.nc, D.data());
    H.coarse_n = Ac.nr;
    tally(&c, static_cast<double>(Ac.nr) * Ac.nr * Ac.nr);
    H.charge(4, c.v);
}

Hier* rn_setup(const Csr& A, const Cand& B, const amgcu_setup_options& o, const Cand* left) {  // :252-287
    if (o.method != 0) throw std::invalid_argument("port: only the rn setup is restated");
    if (A.nr != A.nc || A.nr == 0) throw std::invalid_argument("rn_setup: square nonempty matrix required");
    if (B.n != A.nr) throw std::invalid_argument("rn_setup: candidate size mismatch");
    const idx m = std::max<idx>(1, A.bs);
    if (A.nr % m != 0) throw std::invalid_argument("rn_setup: block size must divide the dimension");
    if (B.k < m) throw std::invalid_argument("rn_setup: need at least block_size candidates");
    if (left && (left->n != B.n || left->k != B.k))
        throw std::invalid_argument("rn_setup: left candidate shape mismatch");
    auto* H = new Hier();
    H->o = o;
    if (!(A.nnz() > 0)) throw std::invalid_argument("WorkLedger: base nnz must be positive");
    H->base = static_cast<double>(A.nnz());
    Level L0;
    L0.A = A;
    L0.B = B;
    L0.sym = symmetric(A);
    H->lv.push_back(std::move(L0));
    Cand Bhat = left ? *left : B;
    while (static_cast<int>(H->lv.size()) < o.max_levels && H->lv.back().A.nr > o.max_size) {
        Level& f = H->lv.back();
        auto st = coarsen(*H, f.A, f.B, Bhat, f.sym);
        if (!st) {
            H->stagnated = true;
            break;
        }
        Level& fine = H->lv.back();
        fine.P = std::move(st->P);
        fine.R = std::move(st->R);
        fine.B = std::move(st->Bf);
        fine.Bc = st->Bcoarse;
        Bhat = std::move(st->Bhc);
        Level nx;
        nx.sym = symmetric(st->Ac);
        nx.A = std::move(st->Ac);
        nx.B = std::move(st->Bcoarse);
        H->lv.push_back(std::move(nx));
    }
    finalize(*H);
    return H;
}

// ---- cycle / solve (cycle.hpp) -------------------------------------------------------
double op_complexity(const Hier& H) {  // complexity.hpp:15-20
    const double base = static_cast<double>(H.lv.front().A.nnz());
    double s = 0.0;
    for (const Level& l : H.lv) s += static_cast<double>(l.A.nnz());
    return s / base;
}
double cyc_complexity(const Hier& H) {  // complexity.hpp:25-36
    const double base = static_cast<double>(H.lv.front().A.nnz());
    double s = 0.0;
    for (size_t l = 0; l + 1 < H.lv.size(); ++l) {
        s += static_cast<double>(H.o.pre_sweeps + H.o.post_sweeps + 1) * H.lv[l].A.nnz();
        s += static_cast<double>(H.lv[l].P.nnz()) + static_cast<double>(H.lv[l].R.nnz());
    }
    return s / base;
}

struct Scratch {
    std::vector<Vec> r, bc, xc;
    explicit Scratch(const Hier& H) {
        for (const Level& l : H.lv) {
            r.emplace_back(l.A.nr);
            bc.emplace_back(l.A.nr);
            xc.emplace_back(l.A.nr);
        }
    }
};

void vcycle(Hier& H, size_t l, double* x, const double* b, int kind, Scratch& s, Ops* c) {  // cycle.hpp:70-95
    if (l == H.lv.size() - 1) {
        if (H.use_lu) H.coarse_lu.solve(b, x);
        else H.coarse.solve(b, x);
        return;
    }
    Level& L = H.lv[l];
    relax(H.o.pre_scheme, H.o.pre_sweeps, L.A, x, b, H.pre[l], c);
    Vec& r = s.r[l];
    spmv(L.A, x, r.data(), c);
    for (size_t i = 0; i < r.size(); ++i) r[i] = b[i] - r[i];
    const idx nc = L.P.nc;
    double* bc = s.bc[l + 1].data();
    double* xc = s.xc[l + 1].data();
    spmv(L.R, r.data(), bc, c);
    std::fill(xc, xc + nc, 0.0);
    vcycle(H, l + 1, xc, bc, kind, s, c);
    if (kind == 1 && l + 1 < H.lv.size() - 1) vcycle(H, l + 1, xc, bc, kind, s, c);
    spmv(L.P, xc, r.data(), c);
    for (size_t i = 0; i < r.size(); ++i) x[i] += r[i];
    relax(H.o.post_scheme, H.o.post_sweeps, L.A, x, b, H.post[l], c);
}

struct Report {
    Vec hist;
    int its = 0;
    bool conv = false, div = false;
    double rho = 0, oc = 0, cc = 0, wus = 0, wusetup = 0;
};

double conv_factor(const Vec& h, int window = 5) {  // cycle.hpp:39-46
    if (h.size() < 2) return 0.0;
    const int w = std::min<int>(window, static_cast<int>(h.size()) - 1);
    const double head = h[h.size() - 1 - w];
    const double tail = h.back();
    if (head <= 0.0) return 0.0;
    return std::pow(tail / head, 1.0 / w);
}

Report solve(Hier& H, const double* b, Vec& x, const amgcu_solve_options& o) {  // cycle.hpp:114-271
    const Csr& A = H.lv.front().A;
    const idx n = A.nr;
    if (x.empty()) x.assign(n, 0.0);
    if (static_cast<idx>(x.size()) != n) throw std::invalid_argument("solve: guess size mismatch");
    if (o.max_iters < 1) throw std::invalid_argument("solve: max_iters must be >= 1");
    Report rep;
    rep.oc = op_complexity(H);
    rep.cc = cyc_complexity(H);
    rep.wusetup = H.wu[0] + H.wu[1] + H.wu[2] + H.wu[3];
    Ops sc;
    Scratch scratch(H);
    auto precond = [&](const double* rhs, double* out) {
        std::fill(out, out + n, 0.0);
        vcycle(H, 0, out, rhs, o.cycle, scratch, &sc);
    };
    auto finish = [&]() {
        rep.rho = conv_factor(rep.hist);
        rep.wus = sc.v / H.base;
        H.charge(4, sc.v);
        return rep;
    };
    Vec r(n);
    spmv(A, x.data(), r.data(), &sc);
    for (idx i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double r0 = vnorm(r.data(), n);
    const double bn = vnorm(b, n);
    const double target = o.tol * (bn > 0.0 ? bn : r0);
    rep.hist.push_back(r0);
    if (r0 <= target) {
        rep.conv = true;
        return finish();
    }
    const double blowup = 1e6 * r0;
    if (o.method == 0) {
        for (int it = 1; it <= o.max_iters; ++it) {
            vcycle(H, 0, x.data(), b, o.cycle, scratch, &sc);
            spmv(A, x.data(), r.data());
            for (idx i = 0; i < n; ++i) r[i] = b[i] - r[i];
            const double rn = vnorm(r.data(), n);
            rep.hist.push_back(rn);
            rep.its = it;
            if (rn <= target) {
                rep.conv = true;
                break;
            }
            if (rn > blowup || !std::isfinite(rn)) {
                rep.div = true;
                break;
            }
        }
        return finish();
    }
    if (o.method == 1) {
        if (!H.lv.front().sym) throw std::invalid_argument("solve: pcg requires a symmetric operator");
        Vec z(n), p(n), q(n);
        precond(r.data(), z.data());
        p = z;
        double rz = vdot(r.data(), z.data(), n);
        for (int it = 1; it <= o.max_iters; ++it) {
            spmv(A, p.data(), q.data(), &sc);
            const double pq = vdot(p.data(), q.data(), n);
            if (!(pq > 0.0)) {
                rep.div = true;
                break;
            }
            const double alpha = rz / pq;
            vaxpy(alpha, p.data(), x.data(), n);
            vaxpy(-alpha, q.data(), r.data(), n);
            const double rn = vnorm(r.data(), n);
            rep.hist.push_back(rn);
            rep.its = it;
            if (rn <= target) {
                rep.conv = true;
                break;
            }
            if (rn > blowup || !std::isfinite(rn)) {
                rep.div = true;
                break;
            }
            precond(r.data(), z.data());
            const double rzn = vdot(r.data(), z.data(), n);
            const double beta = rzn / rz;
            for (idx i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
            rz = rzn;
        }
        return finish();
    }
    // FGMRES, one cycle of max_iters steps (cycle.hpp:211-270)
    const int m = o.max_iters;
    std::vector<Vec> V, Z;
    Vec v0(r);
    vscale(1.0 / r0, v0.data(), n);
    V.push_back(std::move(v0));
    Vec Hm(static_cast<size_t>(m + 1) * m, 0.0);
    auto Hij = [&](int i, int j) -> double& { return Hm[static_cast<size_t>(i) * m + j]; };
    Vec cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0);
    g[0] = r0;
    int built = 0;
    for (int j = 0; j < m; ++j) {
        Vec z(n), w(n);
        precond(V[j].data(), z.data());
        spmv(A, z.data(), w.data(), &sc);
        Z.push_back(std::move(z));
        for (int t = 0; t <= j; ++t) {
            Hij(t, j) = vdot(w.data(), V[t].data(), n);
            vaxpy(-Hij(t, j), V[t].data(), w.data(), n);
        }
        Hij(j + 1, j) = vnorm(w.data(), n);
        for (int t = 0; t < j; ++t) {
            const double tmp = cs[t] * Hij(t, j) + sn[t] * Hij(t + 1, j);
            Hij(t + 1, j) = -sn[t] * Hij(t, j) + cs[t] * Hij(t + 1, j);
            Hij(t, j) = tmp;
        }
        const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
        cs[j] = den > 0.0 ? Hij(j, j) / den : 1.0;
        sn[j] = den > 0.0 ? Hij(j + 1, j) / den : 0.0;
        Hij(j, j) = den;
        const double hlast = Hij(j + 1, j);
        Hij(j + 1, j) = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        const double res = std::fabs(g[j + 1]);
        rep.hist.push_back(res);
        rep.its = j + 1;
        built = j + 1;
        if (res <= target) {
            rep.conv = true;
            break;
        }
        if (res > blowup || !std::isfinite(res)) {
            rep.div = true;
            break;
        }
        if (hlast < 1e-300) break;
        Vec vn(w);
        vscale(1.0 / hlast, vn.data(), n);
        V.push_back(std::move(vn));
    }
    Vec y(built, 0.0);
    for (int t = built - 1; t >= 0; --t) {
        double s = g[t];
        for (int u = t + 1; u < built; ++u) s -= Hij(t, u) * y[u];
        y[t] = Hij(t, t) != 0.0 ? s / Hij(t, t) : 0.0;
    }
    for (int t = 0; t < built; ++t) vaxpy(y[t], Z[t].data(), x.data(), n);
    return finish();
}

}  // namespace port

// =================================================================================
// C ABI (oracle_abi.h)
// =================================================================================
namespace {

thread_local std::string g_err;

port::Csr in_csr(const amgcu_csr* m) {
    port::Csr s(m->n_rows, m->n_cols);
    s.bs = m->block_size;
    s.rp.assign(m->row_offsets, m->row_offsets + m->n_rows + 1);
    const int nnz = m->row_offsets[m->n_rows];
    s.ci.assign(m->col_indices, m->col_indices + nnz);
    s.va.assign(m->values, m->values + nnz);
    return s;
}

void out_csr(const port::Csr& s, amgcu_csr* o) {
    o->n_rows = s.nr;
    o->n_cols = s.nc;
    o->nnz = s.nnz();
    o->block_size = s.bs;
    o->row_offsets = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (s.nr + 1)));
    o->col_indices = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max(1, s.nnz())));
    o->values = static_cast<double*>(std::malloc(sizeof(double) * std::max(1, s.nnz())));
    std::memcpy(o->row_offsets, s.rp.data(), sizeof(int32_t) * (s.nr + 1));
    if (s.nnz()) {
        std::memcpy(o->col_indices, s.ci.data(), sizeof(int32_t) * s.nnz());
        std::memcpy(o->values, s.va.data(), sizeof(double) * s.nnz());
    }
}

port::Cand in_cand(int32_t n, int32_t k, const double* d) {
    port::Cand c(n, k);
    std::memcpy(c.d.data(), d, sizeof(double) * static_cast<size_t>(n) * k);
    return c;
}

double* dup(const port::Vec& v) {
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

port::Agg in_agg(int32_t n_nodes, int32_t n_agg, const int32_t* own, const int32_t* roots) {
    port::Agg a;
    a.n_nodes = n_nodes;
    a.n_agg = n_agg;
    a.owner.assign(own, own + n_nodes);
    a.roots.assign(roots, roots + n_agg);
    a.C = port::Csr(n_nodes, n_agg);
    a.C.ci = a.owner;
    a.C.va.assign(n_nodes, 1.0);
    for (int i = 0; i < n_nodes; ++i) a.C.rp[i + 1] = i + 1;
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
        auto M = in_csr(A);
        port::spmv(M, x, y);
    });
}
int orc_transpose(const amgcu_csr* A, amgcu_csr* out) {
    return guarded([&] { out_csr(port::transpose(in_csr(A)), out); });
}
int orc_matmul(const amgcu_csr* A, const amgcu_csr* B, amgcu_csr* out, double* ops) {
    return guarded([&] {
        port::Ops c;
        out_csr(port::matmul(in_csr(A), in_csr(B), &c), out);
        if (ops) *ops = c.v;
    });
}
int orc_galerkin_product(const amgcu_csr* R, const amgcu_csr* A, const amgcu_csr* P, amgcu_csr* out) {
    return guarded([&] { out_csr(port::galerkin(in_csr(R), in_csr(A), in_csr(P)), out); });
}
int orc_filter_matrix(const amgcu_csr* G, int32_t theta_set, double theta, int32_t k, amgcu_csr* out) {
    return guarded([&] {
        std::optional<double> t;
        std::optional<int32_t> kk;
        if (theta_set) t = theta;
        if (k != 0) kk = k;
        out_csr(port::filter(in_csr(G), t, kk), out);
    });
}
int orc_is_symmetric(const amgcu_csr* A, double tol, int32_t* out) {
    return guarded([&] { *out = port::symmetric(in_csr(A), tol) ? 1 : 0; });
}
int orc_spectral_radius(const amgcu_csr* A, int32_t steps, double* rho) {
    return guarded([&] { *rho = port::spectral_radius(in_csr(A), steps); });
}
int orc_strength(const amgcu_csr* A, const amgcu_strength_config* cfg, amgcu_csr* out, double* ops) {
    return guarded([&] {
        port::Ops c;
        out_csr(port::strength(in_csr(A), *cfg, &c), out);
        if (ops) *ops = c.v;
    });
}
int orc_normalize_strength(const amgcu_csr* S, amgcu_csr* out) {
    return guarded([&] { out_csr(port::normalize_soc(in_csr(S), nullptr), out); });
}
int orc_amalgamate(const amgcu_csr* S, int32_t m, amgcu_csr* out) {
    return guarded([&] { out_csr(port::amalgamate(in_csr(S), m), out); });
}
int orc_greedy_aggregate(const amgcu_csr* S, int32_t* n_agg, int32_t* node_to_agg, int32_t* roots) {
    return guarded([&] {
        port::Agg a = port::aggregate(in_csr(S));
        *n_agg = a.n_agg;
        std::memcpy(node_to_agg, a.owner.data(), sizeof(int32_t) * a.n_nodes);
        std::memcpy(roots, a.roots.data(), sizeof(int32_t) * a.n_agg);
    });
}
int orc_sparsity_pattern(const amgcu_csr* S, const amgcu_csr* C, int32_t degree, amgcu_csr* out) {
    return guarded([&] { out_csr(port::pattern_power(in_csr(S), in_csr(C), degree, nullptr), out); });
}
int orc_root_node_pattern(const amgcu_csr* N, int32_t n_roots, const int32_t* roots, amgcu_csr* out) {
    return guarded([&] {
        std::vector<int32_t> r(roots, roots + n_roots);
        out_csr(port::root_rows(in_csr(N), r), out);
    });
}
int orc_improve_candidates(const amgcu_csr* A, int32_t k, const double* B, int32_t sweeps, int32_t scheme,
                           double weight, double* out) {
    return guarded([&] {
        auto M = in_csr(A);
        port::Cand r = port::improve(M, in_cand(M.nr, k, B), sweeps, scheme, weight, nullptr);
        std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
    });
}
int orc_relax(const amgcu_csr* A, int32_t scheme, double weight, int32_t sweeps, double* x, const double* b) {
    return guarded([&] {
        auto M = in_csr(A);
        if (sweeps < 0) throw std::invalid_argument("relax: dimension mismatch");
        port::RelaxWs ws = port::make_ws(M, scheme, weight, nullptr);
        port::relax(scheme, sweeps, M, x, b, ws, nullptr);
    });
}
int orc_relax_weight(const amgcu_csr* A, int32_t scheme, double weight, double* out) {
    return guarded([&] { *out = port::make_ws(in_csr(A), scheme, weight, nullptr).w; });
}
int orc_inject_tentative(int32_t n_nodes, int32_t n_agg, const int32_t* node_to_agg, const int32_t* roots,
                         const amgcu_csr* N, int32_t k, const double* B, int32_t m, amgcu_csr* T, double** Bc) {
    return guarded([&] {
        port::Agg a = in_agg(n_nodes, n_agg, node_to_agg, roots);
        auto [t, bc] = port::inject(a, in_csr(N), in_cand(n_nodes * m, k, B), m, nullptr);
        out_csr(t, T);
        *Bc = dup(bc.d);
    });
}
int orc_enforce_constraints(const amgcu_csr* P, int32_t k, const double* B, const double* Bc,
                            const amgcu_csr* allowed, amgcu_csr* out) {
    return guarded([&] {
        auto Pm = in_csr(P);
        port::Csr Nm;
        if (allowed) Nm = in_csr(allowed);
        out_csr(port::enforce(Pm, in_cand(Pm.nr, k, B), in_cand(Pm.nc, k, Bc), allowed ? &Nm : nullptr, nullptr),
                out);
    });
}
int orc_energy_minimize(const amgcu_csr* A, const amgcu_csr* T, int32_t k, const double* B, const double* Bc,
                        const amgcu_csr* N, int32_t energy_iters, int32_t krylov, int32_t n_roots,
                        const int32_t* roots, amgcu_csr* out, int32_t* iterations, int32_t* breakdown) {
    return guarded([&] {
        auto Am = in_csr(A), Tm = in_csr(T), Nm = in_csr(N);
        std::vector<int32_t> r(roots, roots + n_roots);
        int its = 0;
        bool brk = false;
        out_csr(port::energy_min(Am, Tm, in_cand(Am.nr, k, B), in_cand(Nm.nc, k, Bc), Nm, energy_iters, 2, krylov,
                                 r, nullptr, &its, &brk),
                out);
        if (iterations) *iterations = its;
        if (breakdown) *breakdown = brk ? 1 : 0;
    });
}

int orc_setup(const amgcu_csr* A, int32_t k, const double* B, const double* left, const amgcu_setup_options* o,
              void** hier) {
    return guarded([&] {
        auto Am = in_csr(A);
        port::Cand b = in_cand(Am.nr, k, B);
        port::Cand l;
        if (left) l = in_cand(Am.nr, k, left);
        *hier = port::rn_setup(Am, b, *o, left ? &l : nullptr);
    });
}
int orc_hier_levels(void* hp, int32_t* n_levels, int32_t* stagnated) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        *n_levels = static_cast<int32_t>(h->lv.size());
        *stagnated = h->stagnated ? 1 : 0;
    });
}
int orc_hier_get_matrix(void* hp, int32_t level, int32_t which, amgcu_csr* out) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        const port::Level& L = h->lv.at(level);
        out_csr(which == 0 ? L.A : (which == 1 ? L.P : L.R), out);
    });
}
int orc_hier_get_candidates(void* hp, int32_t level, int32_t which, int32_t* n, int32_t* k, double** data) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        const port::Level& L = h->lv.at(level);
        const port::Cand& c = which == 0 ? L.B : L.Bc;
        *n = c.n;
        *k = c.k;
        *data = dup(c.d);
    });
}
int orc_hier_level_symmetric(void* hp, int32_t level, int32_t* sym) {
    return guarded([&] { *sym = static_cast<port::Hier*>(hp)->lv.at(level).sym ? 1 : 0; });
}
int orc_hier_relax_weights(void* hp, int32_t level, double* pre, double* post) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        *pre = h->pre.at(level).w;
        *post = h->post.at(level).w;
    });
}
int orc_hier_ledger(void* hp, double* wu5) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        for (int i = 0; i < 5; ++i) wu5[i] = h->wu[i];
    });
}
int orc_hier_complexity(void* hp, double* chi_oc, double* chi_cc) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        *chi_oc = port::op_complexity(*h);
        *chi_cc = port::cyc_complexity(*h);
    });
}
int orc_hier_free(void* hp) {
    delete static_cast<port::Hier*>(hp);
    return 0;
}
int orc_solve(void* hp, const double* b, double* x, const amgcu_solve_options* o, amgcu_solve_report* rep,
              double* history, int32_t history_cap) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        const int n = h->lv.front().A.nr;
        port::Vec xv(x, x + n);
        port::Report r = port::solve(*h, b, xv, *o);
        std::memcpy(x, xv.data(), sizeof(double) * n);
        rep->iterations = r.its;
        rep->converged = r.conv;
        rep->diverged = r.div;
        rep->history_len = static_cast<int32_t>(r.hist.size());
        rep->rho = r.rho;
        rep->chi_oc = r.oc;
        rep->chi_cc = r.cc;
        rep->work_units_solve = r.wus;
        rep->work_units_setup = r.wusetup;
        for (int i = 0; i < history_cap && i < static_cast<int>(r.hist.size()); ++i) history[i] = r.hist[i];
    });
}
int orc_cycle(void* hp, double* x, const double* b, int32_t kind) {
    return guarded([&] {
        auto* h = static_cast<port::Hier*>(hp);
        port::Scratch s(*h);
        port::vcycle(*h, 0, x, b, kind, s, nullptr);
    });
}
int orc_generate_reference(int32_t, int32_t, int32_t, double, double, double, double, int32_t, int32_t,
                           amgcu_csr*, int32_t*, double**, int32_t*, double**, double**) {
    g_err = "orc_generate_reference: only the reference build (libamgref) provides the reference generators";
    return 9;
}

}  // extern "C"
