// rho(D^-1 A) by a fixed number of Arnoldi steps (spectral.hpp:18-65).
// The basis lives on the device; modified Gram-Schmidt dots/axpys use
// device-resident scalars (the H column is written in place), and only the
// subdiagonal norm comes back to the host each step for the h < 1e-14 test.
// The (<= 15)^2 Hessenberg eigenvalue problem is solved on the host with the
// Francis QR of small_dense.h.  The start vector 1 + U(-0.5, 0.5) from
// std::mt19937(20240911) (spectral.hpp:32-36) depends only on n, and every
// shorter vector is a prefix of a longer one, so it is generated once per
// context for the largest n seen and reused.
#include <complex>
#include <random>

#include "ops.cuh"
#include "small_dense.h"

namespace amgcu {

namespace {

__global__ void k_spmv_dinv(int32_t nr, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ va, const double* __restrict__ x,
                            const double* __restrict__ dinv, double* __restrict__ y) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    double s = 0.0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) s += va[p] * x[ci[p]];
    y[i] = s;
    y[i] *= dinv[i];
}

void ensure_start_vector(Ctx& c, size_t n) {
    if (c.arnoldi_v0_n >= n) return;
    std::vector<double> v(n);
    std::mt19937 gen(20240911u);
    std::uniform_real_distribution<double> dist(-0.5, 0.5);
    for (size_t i = 0; i < n; ++i) v[i] = 1.0 + dist(gen);
    c.arnoldi_v0.alloc(n, c.s);
    copy_h2d(c, c.arnoldi_v0.get(), v.data(), static_cast<int64_t>(n));
    sync(c);
    c.arnoldi_v0_n = n;
}

}  // namespace

double spectral_radius(Ctx& c, const DCsr& A, int steps, const double* dinv) {
    if (A.nr != A.nc) throw InvalidArgument("spectral_radius_estimate: square matrix required");
    const int32_t n = A.nr;
    if (n == 0) return 0.0;
    const int m = std::min<int>(steps, n);
    ensure_start_vector(c, static_cast<size_t>(n));
    DBuf<double> V(static_cast<size_t>(n) * (m + 1), c.s);
    DBuf<double> Hd(static_cast<size_t>(m + 1) * m + 1, c.s);
    AMG_CK(cudaMemsetAsync(Hd.get(), 0, sizeof(double) * ((m + 1) * m + 1), c.s));
    double* nrm = Hd.get() + (m + 1) * m;
    copy_d2d(c, V.get(), c.arnoldi_v0.get(), n);
    nrm2(c, V.get(), n, nrm);
    scale_recip_dev(c, nrm, V.get(), n);
    int built = 0;
    for (int j = 0; j < m; ++j) {
        double* w = V.get() + static_cast<size_t>(j + 1) * n;
        launch(c, k_spmv_dinv, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), A.va.get(),
               static_cast<const double*>(V.get() + static_cast<size_t>(j) * n), dinv, w);
        // modified Gram-Schmidt: h_t = (w, v_t); w -= h_t v_t; the axpy of step t is
        // fused with the dot of step t + 1 (and the last one with the norm)
        double* hsub = Hd.get() + (j + 1) * m + j;
        dot(c, w, V.get(), n, Hd.get() + j);
        for (int t = 0; t <= j; ++t) {
            const double* vt = V.get() + static_cast<size_t>(t) * n;
            if (t < j)
                axpy_dot(c, Hd.get() + t * m + j, -1.0, vt, w, V.get() + static_cast<size_t>(t + 1) * n, n,
                         Hd.get() + (t + 1) * m + j, false);
            else
                axpy_dot(c, Hd.get() + t * m + j, -1.0, vt, w, nullptr, n, hsub, true);
        }
        const double h = read_scalar(c, hsub);
        built = j + 1;
        if (h < 1e-14) break;
        scale_recip_dev(c, hsub, w, n);
    }
    std::vector<double> H(static_cast<size_t>(m + 1) * m);
    copy_d2h(c, H.data(), Hd.get(), static_cast<int64_t>(H.size()));
    sync(c);
    std::vector<double> Hs(static_cast<size_t>(built) * built), wr(built), wi(built);
    for (int i = 0; i < built; ++i)
        for (int j = 0; j < built; ++j) Hs[i * built + j] = H[i * m + j];
    if (sd::hessenberg_eigenvalues(built, Hs.data(), wr.data(), wi.data()) != 0)
        throw RuntimeError("spectral_radius_estimate: Hessenberg QR did not converge");
    double rho = 0.0;
    for (int i = 0; i < built; ++i) rho = std::max(rho, std::abs(std::complex<double>(wr[i], wi[i])));
    return rho;
}

}  // namespace amgcu
