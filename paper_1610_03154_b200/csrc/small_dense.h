// Tiny dense linear algebra used on the RN-AMG path (k x k Gram pseudo-inverses,
// m x m root-block inverses, the Arnoldi Hessenberg eigenvalues behind rho(D^-1 A),
// the GMRES energy-min Hessenberg solve and the coarsest-level COD).
//
// The reference calls Eigen for these (proj/include/amg/core/spectral.hpp:60-63,
// interpolation.hpp:129-134, 404-411, 492-505, 544-553, hierarchy.hpp:55-75).
// Eigen is not available in this image, so this header is the single
// implementation of those algorithms: it is compiled
//   * into the sm_100a kernels (__device__, --fmad=false),
//   * into the host orchestration of libamgcu (-ffp-contract=off),
//   * into the oracle's Eigen-API stand-in (oracle/eigen_shim), so the
//     reference headers compiled against the shim and the GPU path evaluate
//     the same operation sequence.
// Only +, -, *, / and sqrt are used (all IEEE correctly rounded on host and
// device), so host and device results are bit-identical.
//
// Storage convention: row-major n x n arrays, small fixed upper bounds.
#pragma once

#include <math.h>

#include <vector>

#if defined(__CUDACC__)
#define SD_HD __host__ __device__ __forceinline__
#else
#define SD_HD inline
#endif

namespace sd {

constexpr double kEps = 2.220446049250313e-16;  // NumTraits<double>::epsilon()

SD_HD double dabs(double x) { return x < 0.0 ? -x : (x == 0.0 ? 0.0 : x); }
SD_HD double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max semantics
SD_HD double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min semantics

// ---------------------------------------------------------------------------
// Symmetric eigen-decomposition by cyclic Jacobi rotations.
// Eigenvalues ascending; evecs (row-major) holds eigenvectors as columns.
// n == 1 reproduces Eigen's special case exactly: eval = a, evec = 1.
// ---------------------------------------------------------------------------
template <int NMAX>
SD_HD void sym_eig(int n, const double* A, double* evals, double* evecs) {
    double a[NMAX * NMAX];
    for (int i = 0; i < n * n; ++i) a[i] = A[i];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) evecs[i * n + j] = (i == j) ? 1.0 : 0.0;
    if (n == 1) {
        evals[0] = a[0];
        return;
    }
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int p = 0; p < n; ++p) {
            diag += a[p * n + p] * a[p * n + p];
            for (int q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
        }
        if (off == 0.0 || off <= 1e-36 * diag) break;
        for (int p = 0; p < n - 1; ++p) {
            for (int q = p + 1; q < n; ++q) {
                const double apq = a[p * n + q];
                if (apq == 0.0) continue;
                const double app = a[p * n + p], aqq = a[q * n + q];
                // negligible off-diagonal after the first sweeps: drop it
                if (sweep > 3 && dabs(apq) <= 1e-18 * dabs(app) && dabs(apq) <= 1e-18 * dabs(aqq)) {
                    a[p * n + q] = 0.0;
                    a[q * n + p] = 0.0;
                    continue;
                }
                const double theta = (aqq - app) / (2.0 * apq);
                double t;
                if (dabs(theta) > 1e150) {
                    t = 0.5 / theta;
                } else {
                    t = 1.0 / (dabs(theta) + sqrt(theta * theta + 1.0));
                    if (theta < 0.0) t = -t;
                }
                const double c = 1.0 / sqrt(t * t + 1.0);
                const double s = t * c;
                for (int k = 0; k < n; ++k) {  // columns p, q
                    const double akp = a[k * n + p], akq = a[k * n + q];
                    a[k * n + p] = c * akp - s * akq;
                    a[k * n + q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {  // rows p, q
                    const double apk = a[p * n + k], aqk = a[q * n + k];
                    a[p * n + k] = c * apk - s * aqk;
                    a[q * n + k] = s * apk + c * aqk;
                }
                a[p * n + q] = 0.0;
                a[q * n + p] = 0.0;
                for (int k = 0; k < n; ++k) {
                    const double vkp = evecs[k * n + p], vkq = evecs[k * n + q];
                    evecs[k * n + p] = c * vkp - s * vkq;
                    evecs[k * n + q] = s * vkp + c * vkq;
                }
            }
        }
    }
    for (int i = 0; i < n; ++i) evals[i] = a[i * n + i];
    // stable insertion sort, ascending
    for (int i = 1; i < n; ++i) {
        int j = i;
        while (j > 0 && evals[j] < evals[j - 1]) {
            const double t = evals[j];
            evals[j] = evals[j - 1];
            evals[j - 1] = t;
            for (int k = 0; k < n; ++k) {
                const double v = evecs[k * n + j];
                evecs[k * n + j] = evecs[k * n + j - 1];
                evecs[k * n + j - 1] = v;
            }
            --j;
        }
    }
}

// Pseudo-inverse of a symmetric k x k matrix through its eigen-decomposition,
// as in interpolation.hpp:129-134: eigenvalues at or below
// 1e-12 * max|lambda| are treated as zero; Gp = V diag(1/lambda) V^T with the
// product evaluated left to right ((V * D) * V^T), each entry summed in index order.
template <int KMAX>
SD_HD void sym_pinv(int k, const double* G, double* Gp) {
    double ev[KMAX], V[KMAX * KMAX];
    sym_eig<KMAX>(k, G, ev, V);
    double mx = 0.0;
    for (int a = 0; a < k; ++a) mx = dmax(mx, dabs(ev[a]));
    const double cutoff = 1e-12 * dmax(mx, 1e-300);
    double inv[KMAX];
    for (int a = 0; a < k; ++a) inv[a] = ev[a] > cutoff ? 1.0 / ev[a] : 0.0;
    double VD[KMAX * KMAX];
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) VD[i * k + j] = V[i * k + j] * inv[j];
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
            double s = 0.0;
            for (int t = 0; t < k; ++t) s += VD[i * k + t] * V[j * k + t];
            Gp[i * k + j] = s;
        }
}

// ---------------------------------------------------------------------------
// Full-pivoting LU (Eigen::FullPivLU semantics: rank with threshold
// eps * diagonalSize relative to the largest pivot, determinant, inverse
// through solve(I)).  n <= NMAX.
// ---------------------------------------------------------------------------
template <int NMAX>
struct FullPivLU {
    int n = 0;
    double lu[NMAX * NMAX];
    int rowp[NMAX];  // row transpositions applied at step k: swap(k, rowp[k])
    int colq[NMAX];  // column transpositions
    int nonzero_pivots = 0;
    double maxpivot = 0.0;
    int det_pq = 1;

    SD_HD void compute(int n_, const double* M) {
        n = n_;
        for (int i = 0; i < n * n; ++i) lu[i] = M[i];
        nonzero_pivots = n;
        maxpivot = 0.0;
        int ntrans = 0;
        for (int k = 0; k < n; ++k) {
            // biggest |entry| of the trailing block, column-major scan, first max wins
            double best = -1.0;
            int bi = k, bj = k;
            for (int j = k; j < n; ++j)
                for (int i = k; i < n; ++i) {
                    const double v = dabs(lu[i * n + j]);
                    if (v > best) {
                        best = v;
                        bi = i;
                        bj = j;
                    }
                }
            if (best == 0.0) {
                nonzero_pivots = k;
                for (int t = k; t < n; ++t) {
                    rowp[t] = t;
                    colq[t] = t;
                }
                break;
            }
            if (best > maxpivot) maxpivot = best;
            rowp[k] = bi;
            colq[k] = bj;
            if (bi != k) {
                ++ntrans;
                for (int j = 0; j < n; ++j) {
                    const double t = lu[k * n + j];
                    lu[k * n + j] = lu[bi * n + j];
                    lu[bi * n + j] = t;
                }
            }
            if (bj != k) {
                ++ntrans;
                for (int i = 0; i < n; ++i) {
                    const double t = lu[i * n + k];
                    lu[i * n + k] = lu[i * n + bj];
                    lu[i * n + bj] = t;
                }
            }
            const double piv = lu[k * n + k];
            for (int i = k + 1; i < n; ++i) lu[i * n + k] = lu[i * n + k] / piv;
            for (int i = k + 1; i < n; ++i)
                for (int j = k + 1; j < n; ++j) lu[i * n + j] = lu[i * n + j] - lu[i * n + k] * lu[k * n + j];
        }
        det_pq = (ntrans % 2) ? -1 : 1;
    }
    SD_HD int rank() const {
        const double thr = dabs(maxpivot) * (kEps * static_cast<double>(n));
        int r = 0;
        for (int i = 0; i < nonzero_pivots; ++i) r += (dabs(lu[i * n + i]) > thr) ? 1 : 0;
        return r;
    }
    SD_HD double determinant() const {
        double d = static_cast<double>(det_pq);
        for (int i = 0; i < n; ++i) d = d * lu[i * n + i];
        return d;
    }
    // x = A^{-1} b for one right-hand side (b, x length n)
    SD_HD void solve(const double* b, double* x) const {
        double c[NMAX];
        for (int i = 0; i < n; ++i) c[i] = b[i];
        for (int k = 0; k < n; ++k)
            if (rowp[k] != k) {
                const double t = c[k];
                c[k] = c[rowp[k]];
                c[rowp[k]] = t;
            }
        const int r = nonzero_pivots;
        for (int i = 0; i < n; ++i) {  // unit lower solve
            double s = c[i];
            for (int j = 0; j < i && j < r; ++j) s = s - lu[i * n + j] * c[j];
            c[i] = s;
        }
        for (int i = r - 1; i >= 0; --i) {  // upper solve on the nonzero pivots
            double s = c[i];
            for (int j = i + 1; j < r; ++j) s = s - lu[i * n + j] * c[j];
            c[i] = s / lu[i * n + i];
        }
        for (int i = r; i < n; ++i) c[i] = 0.0;
        for (int k = n - 1; k >= 0; --k)
            if (colq[k] != k) {
                const double t = c[k];
                c[k] = c[colq[k]];
                c[colq[k]] = t;
            }
        for (int i = 0; i < n; ++i) x[i] = c[i];
    }
    SD_HD void inverse(double* inv) const {  // row-major
        double e[NMAX], col[NMAX];
        for (int j = 0; j < n; ++j) {
            for (int i = 0; i < n; ++i) e[i] = (i == j) ? 1.0 : 0.0;
            solve(e, col);
            for (int i = 0; i < n; ++i) inv[i * n + j] = col[i];
        }
    }
};

// ---------------------------------------------------------------------------
// Complete orthogonal decomposition A P = Q [T11 0; 0 0] Z^T by Householder
// QR with column pivoting followed by an RZ step on the rank-deficient part
// (host only; any size).  Used for the coarsest-level solve
// (hierarchy.hpp:54-76) and for degenerate root blocks (interpolation.hpp:550-553).
// Row-major storage, rows x cols.  rank() counts |R_ii| > threshold * max|R_ii|,
// threshold defaulting to eps * min(rows, cols) as in Eigen.
// ---------------------------------------------------------------------------
struct COD {
    int rows = 0, cols = 0, rnk = 0, nonzero = 0;
    double threshold = -1.0;  // < 0: default eps * diagonalSize
    double maxpivot = 0.0;
    std::vector<double> qr, hcoef, zcoef, rdiag;
    std::vector<int> perm;  // column j of A P is column perm[j] of A
    std::vector<double> src;

    SD_HD static double make_householder(double* x, int len, int stride, double* tau) {
        double tail = 0.0;
        for (int i = 1; i < len; ++i) tail += x[i * stride] * x[i * stride];
        const double c0 = x[0];
        if (tail == 0.0) {
            *tau = 0.0;
            for (int i = 1; i < len; ++i) x[i * stride] = 0.0;
            return c0;
        }
        double beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        const double denom = c0 - beta;
        for (int i = 1; i < len; ++i) x[i * stride] = x[i * stride] / denom;
        *tau = (beta - c0) / beta;
        return beta;
    }

    int rank_for(double thr) const {
        int r = 0;
        for (int i = 0; i < nonzero; ++i) r += (dabs(rdiag[i]) > thr * maxpivot) ? 1 : 0;
        return r;
    }
    double effective_threshold() const {
        const int size = rows < cols ? rows : cols;
        return threshold >= 0.0 ? threshold : kEps * static_cast<double>(size);
    }

    void set_threshold(double t) {
        threshold = t;
        if (!src.empty()) compute(rows, cols, src.data());
    }

    // QR with column pivoting only (ColPivHouseholderQR semantics)
    void qr_only(int r, int c, const double* A) {
        rows = r;
        cols = c;
        src.assign(A, A + static_cast<size_t>(r) * c);
        qr = src;
        perm.resize(c);
        hcoef.assign(c, 0.0);
        zcoef.assign(c, 0.0);
        for (int j = 0; j < c; ++j) perm[j] = j;
        const int size = r < c ? r : c;
        rdiag.assign(size, 0.0);
        maxpivot = 0.0;
        nonzero = size;
        for (int k = 0; k < size; ++k) {
            int best = k;
            double bn = -1.0;
            for (int j = k; j < c; ++j) {
                double s = 0.0;
                for (int i = k; i < r; ++i) s += qr[i * c + j] * qr[i * c + j];
                if (s > bn) {
                    bn = s;
                    best = j;
                }
            }
            if (bn == 0.0 && nonzero == size) nonzero = k;
            if (best != k) {
                for (int i = 0; i < r; ++i) {
                    const double t = qr[i * c + k];
                    qr[i * c + k] = qr[i * c + best];
                    qr[i * c + best] = t;
                }
                const int t = perm[k];
                perm[k] = perm[best];
                perm[best] = t;
            }
            double tau;
            const double beta = make_householder(&qr[k * c + k], r - k, c, &tau);
            qr[k * c + k] = beta;
            hcoef[k] = tau;
            rdiag[k] = beta;
            if (dabs(beta) > maxpivot) maxpivot = dabs(beta);
            for (int j = k + 1; j < c; ++j) {
                double s = qr[k * c + j];
                for (int i = k + 1; i < r; ++i) s += qr[i * c + k] * qr[i * c + j];
                s = tau * s;
                qr[k * c + j] -= s;
                for (int i = k + 1; i < r; ++i) qr[i * c + j] -= qr[i * c + k] * s;
            }
        }
    }

    void compute(int r, int c, const double* A) {
        qr_only(r, c, A);
        rnk = rank_for(effective_threshold());
        // RZ: annihilate T12 (rows 0..rnk-1, columns rnk..c-1) from the right
        for (int k = rnk - 1; k >= 0 && rnk < c; --k) {
            double tail = 0.0;
            for (int j = rnk; j < c; ++j) tail += qr[k * c + j] * qr[k * c + j];
            const double c0 = qr[k * c + k];
            if (tail == 0.0) {
                zcoef[k] = 0.0;
                continue;
            }
            double beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            const double denom = c0 - beta;
            for (int j = rnk; j < c; ++j) qr[k * c + j] = qr[k * c + j] / denom;
            const double tau = (beta - c0) / beta;
            zcoef[k] = tau;
            qr[k * c + k] = beta;
            for (int i = 0; i < k; ++i) {
                double s = qr[i * c + k];
                for (int j = rnk; j < c; ++j) s += qr[i * c + j] * qr[k * c + j];
                s = tau * s;
                qr[i * c + k] -= s;
                for (int j = rnk; j < c; ++j) qr[i * c + j] -= s * qr[k * c + j];
            }
        }
    }

    // Minimal-norm least-squares solution of A x = b (b length rows, x length cols)
    void solve(const double* b, double* x) const {
        std::vector<double> y(b, b + rows);
        const int size = rows < cols ? rows : cols;
        for (int k = 0; k < size; ++k) {  // y = Q^T b
            double s = y[k];
            for (int i = k + 1; i < rows; ++i) s += qr[i * cols + k] * y[i];
            s = hcoef[k] * s;
            y[k] -= s;
            for (int i = k + 1; i < rows; ++i) y[i] -= qr[i * cols + k] * s;
        }
        std::vector<double> z(cols, 0.0);
        for (int i = rnk - 1; i >= 0; --i) {  // T11 z1 = y1
            double s = y[i];
            for (int j = i + 1; j < rnk; ++j) s -= qr[i * cols + j] * z[j];
            z[i] = s / qr[i * cols + i];
        }
        if (rnk < cols) {  // z <- Z z (right reflectors, forward order)
            for (int k = 0; k < rnk; ++k) {
                const double tau = zcoef[k];
                if (tau == 0.0) continue;
                double s = z[k];
                for (int j = rnk; j < cols; ++j) s += qr[k * cols + j] * z[j];
                s = tau * s;
                z[k] -= s;
                for (int j = rnk; j < cols; ++j) z[j] -= s * qr[k * cols + j];
            }
        }
        for (int j = 0; j < cols; ++j) x[perm[j]] = z[j];
    }

    // pseudo-inverse (cols x rows, row-major) = solve(I)
    void pseudo_inverse(double* out) const {
        std::vector<double> e(rows), col(cols);
        for (int j = 0; j < rows; ++j) {
            for (int i = 0; i < rows; ++i) e[i] = (i == j) ? 1.0 : 0.0;
            solve(e.data(), col.data());
            for (int i = 0; i < cols; ++i) out[i * rows + j] = col[i];
        }
    }
};

// Rank of a row-major r x c matrix by Householder QR with column pivoting, as
// COD::qr_only followed by rank_for(thr) (ColPivHouseholderQR + setThreshold:
// the span_rank of ensure_min_support, interpolation.hpp:585-595), with the same
// operation order; usable on the device.  `qr` is overwritten.  c <= CMAX.
template <int CMAX>
SD_HD int qr_rank(int r, int c, double* qr, double thr) {
    const int size = r < c ? r : c;
    double rdiag[CMAX];
    double maxpivot = 0.0;
    int nonzero = size;
    for (int k = 0; k < size; ++k) {
        int best = k;
        double bn = -1.0;
        for (int j = k; j < c; ++j) {
            double s2 = 0.0;
            for (int i = k; i < r; ++i) s2 += qr[i * c + j] * qr[i * c + j];
            if (s2 > bn) {
                bn = s2;
                best = j;
            }
        }
        if (bn == 0.0 && nonzero == size) nonzero = k;
        if (best != k) {
            for (int i = 0; i < r; ++i) {
                const double t = qr[i * c + k];
                qr[i * c + k] = qr[i * c + best];
                qr[i * c + best] = t;
            }
        }
        double tau;
        const double beta = COD::make_householder(&qr[k * c + k], r - k, c, &tau);
        qr[k * c + k] = beta;
        rdiag[k] = beta;
        if (dabs(beta) > maxpivot) maxpivot = dabs(beta);
        for (int j = k + 1; j < c; ++j) {
            double s2 = qr[k * c + j];
            for (int i = k + 1; i < r; ++i) s2 += qr[i * c + k] * qr[i * c + j];
            s2 = tau * s2;
            qr[k * c + j] -= s2;
            for (int i = k + 1; i < r; ++i) qr[i * c + j] -= qr[i * c + k] * s2;
        }
    }
    int rk = 0;
    for (int i = 0; i < nonzero; ++i) rk += (dabs(rdiag[i]) > thr * maxpivot) ? 1 : 0;
    return rk;
}

// ---------------------------------------------------------------------------
// Eigenvalues of a real upper-Hessenberg matrix by the Francis double-shift
// QR iteration (the real-Schur route Eigen::EigenSolver takes once the input
// is already Hessenberg, spectral.hpp:60-63).  a is row-major n x n and is
// destroyed.  Returns 0 on success, -1 if an eigenvalue failed to converge.
// ---------------------------------------------------------------------------
inline int hessenberg_eigenvalues(int n, double* a, double* wr, double* wi) {
    auto A = [&](int i, int j) -> double& { return a[i * n + j]; };
    double anorm = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = (i > 0 ? i - 1 : 0); j < n; ++j) anorm += dabs(A(i, j));
    int nn = n - 1;
    double t = 0.0;
    double p = 0.0, q = 0.0, r = 0.0, s = 0.0, w, x, y, z;
    while (nn >= 0) {
        int its = 0, l;
        do {
            for (l = nn; l >= 1; --l) {
                s = dabs(A(l - 1, l - 1)) + dabs(A(l, l));
                if (s == 0.0) s = anorm;
                if (dabs(A(l, l - 1)) + s == s) {
                    A(l, l - 1) = 0.0;
                    break;
                }
            }
            x = A(nn, nn);
            if (l == nn) {  // one root
                wr[nn] = x + t;
                wi[nn] = 0.0;
                --nn;
            } else {
                y = A(nn - 1, nn - 1);
                w = A(nn, nn - 1) * A(nn - 1, nn);
                if (l == nn - 1) {  // two roots
                    p = 0.5 * (y - x);
                    q = p * p + w;
                    z = sqrt(dabs(q));
                    x += t;
                    if (q >= 0.0) {
                        z = p + (p >= 0.0 ? z : -z);
                        wr[nn - 1] = wr[nn] = x + z;
                        if (z != 0.0) wr[nn] = x - w / z;
                        wi[nn - 1] = wi[nn] = 0.0;
                    } else {
                        wr[nn - 1] = wr[nn] = x + p;
                        wi[nn - 1] = -(wi[nn] = z);
                    }
                    nn -= 2;
                } else {
                    if (its == 60) return -1;
                    if (its == 10 || its == 20) {  // exceptional shift
                        t += x;
                        for (int i = 0; i <= nn; ++i) A(i, i) -= x;
                        s = dabs(A(nn, nn - 1)) + dabs(A(nn - 1, nn - 2));
                        y = x = 0.75 * s;
                        w = -0.4375 * s * s;
                    }
                    ++its;
                    int m;
                    for (m = nn - 2; m >= l; --m) {
                        z = A(m, m);
                        r = x - z;
                        s = y - z;
                        p = (r * s - w) / A(m + 1, m) + A(m, m + 1);
                        q = A(m + 1, m + 1) - z - r - s;
                        r = A(m + 2, m + 1);
                        s = dabs(p) + dabs(q) + dabs(r);
                        p /= s;
                        q /= s;
                        r /= s;
                        if (m == l) break;
                        const double u = dabs(A(m, m - 1)) * (dabs(q) + dabs(r));
                        const double v = dabs(p) * (dabs(A(m - 1, m - 1)) + dabs(z) + dabs(A(m + 1, m + 1)));
                        if (u + v == v) break;
                    }
                    for (int i = m; i <= nn - 2; ++i) {
                        A(i + 2, i) = 0.0;
                        if (i != m) A(i + 2, i - 1) = 0.0;
                    }
                    for (int k = m; k <= nn - 1; ++k) {
                        if (k != m) {
                            p = A(k, k - 1);
                            q = A(k + 1, k - 1);
                            r = 0.0;
                            if (k != nn - 1) r = A(k + 2, k - 1);
                            if ((x = dabs(p) + dabs(q) + dabs(r)) != 0.0) {
                                p /= x;
                                q /= x;
                                r /= x;
                            }
                        }
                        const double ss = sqrt(p * p + q * q + r * r);
                        s = (p >= 0.0) ? ss : -ss;
                        if (s != 0.0) {
                            if (k == m) {
                                if (l != m) A(k, k - 1) = -A(k, k - 1);
                            } else {
                                A(k, k - 1) = -s * x;
                            }
                            p += s;
                            x = p / s;
                            y = q / s;
                            z = r / s;
                            q /= p;
                            r /= p;
                            for (int j = k; j <= nn; ++j) {
                                p = A(k, j) + q * A(k + 1, j);
                                if (k != nn - 1) {
                                    p += r * A(k + 2, j);
                                    A(k + 2, j) -= p * z;
                                }
                                A(k + 1, j) -= p * y;
                                A(k, j) -= p * x;
                            }
                            const int mmin = nn < k + 3 ? nn : k + 3;
                            for (int i = l; i <= mmin; ++i) {
                                p = x * A(i, k) + y * A(i, k + 1);
                                if (k != nn - 1) {
                                    p += z * A(i, k + 2);
                                    A(i, k + 2) -= p * r;
                                }
                                A(i, k + 1) -= p * q;
                                A(i, k) -= p;
                            }
                        }
                    }
                }
            }
        } while (l < nn - 1);
    }
    return 0;
}

}  // namespace sd
