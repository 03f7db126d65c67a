// rho(D^-1 A) by a fixed number of Arnoldi steps (spectral.hpp:18-65).
// The basis lives on the device; modified Gram-Schmidt dots/axpys use
// device-resident scalars (the H column is written in place), and H comes back
// to the host once: the h < 1e-14 breakdown test is applied to it afterwards.
// The (<= 15)^2 Hessenberg eigenvalue problem is solved on the host with the
// Francis QR of small_dense.h.  The start vector 1 + U(-0.5, 0.5) from
// std::mt19937(20240911) (spectral.hpp:32-36) depends only on n, and every
// shorter vector is a prefix of a longer one, so it is generated once per
// context for the largest n seen and reused.
#include <cooperative_groups.h>

#include <cub/block/block_reduce.cuh>

#include <complex>
#include <cstdlib>
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


// The whole Arnoldi process in one cooperative launch (production mode),
// bit-identical to the launch-per-step path: every reduction reproduces the
// tree of blas.cu's k_dot_tree / k_axpy_dot_tree -- gv "virtual blocks" of
// kArnThreads threads (gv = that path's grid), per-thread sums in grid-stride
// order, cub::BlockReduce per virtual block, then the partials summed strided
// over one block and cub-reduced.  A physical block serves virtual blocks
// blockIdx.x, blockIdx.x + gridDim.x, ...; every physical block computes the
// final sum (same bits everywhere) after a grid barrier.  Per Arnoldi step:
// w = D^-1 A v_j fused with (w, v_0); each modified Gram-Schmidt step
// w -= h_t v_t fused with the next dot (the last one with (w, w)); then
// v_{j+1} = w * (1 / h).  H is written by block 0.
constexpr int kArnThreads = 256;  // == blas.cu kDotThreads
constexpr int kArnRegElems = 4;   // == blas.cu kUnroll: dot_grid gives <= 4 elements per thread
constexpr int kArnRegVb = 3;      // virtual blocks per physical block with w in registers
using ArnBR = cub::BlockReduce<double, kArnThreads>;

struct ArnShared {
    typename ArnBR::TempStorage tmp;
    double bcast;
};

// finish one reduction: partials of the gv virtual blocks -> every block
// grid barrier; a one-block launch (the smallest levels) needs only the block barrier
__device__ __forceinline__ void arn_sync(cooperative_groups::grid_group& grid) {
    if (gridDim.x == 1) {
        __threadfence_block();
        __syncthreads();
    } else {
        grid.sync();
    }
}

__device__ double arn_finish(double* partials, int gv, cooperative_groups::grid_group& grid, ArnShared& sh) {
    arn_sync(grid);
    double t = 0.0;
    for (int k = threadIdx.x; k < gv; k += kArnThreads) t += __ldcg(&partials[k]);
    t = ArnBR(sh.tmp).Sum(t);
    if (threadIdx.x == 0) sh.bcast = t;
    __syncthreads();
    t = sh.bcast;
    __syncthreads();
    return t;
}

__device__ __forceinline__ void arn_partial(double s, int vb, double* partials, ArnShared& sh) {
    const double b = ArnBR(sh.tmp).Sum(s);
    if (threadIdx.x == 0) partials[vb] = b;
    __syncthreads();
}

__global__ void __launch_bounds__(kArnThreads, 3)  // >= 3 blocks per SM: 444 blocks serve level 0's 1022 virtual ones
    k_arnoldi_coop(int32_t n, int m, int gv, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                   const double* __restrict__ va, const double* __restrict__ dinv, const double* __restrict__ v0,
                   double* __restrict__ V, double* __restrict__ H, double* __restrict__ partials_base) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ ArnShared sh;
    int parity = 0;  // partials double-buffered: a block racing ahead never overwrites one being read
    auto next_partials = [&]() {
        double* p = partials_base + (parity ? gv : 0);
        parity ^= 1;
        return p;
    };
    const int64_t vstride = static_cast<int64_t>(gv) * kArnThreads;
    // v_0 = v0 * (1 / ||v0||)
    double* P = next_partials();
    for (int vb = blockIdx.x; vb < gv; vb += gridDim.x) {
        double s = 0.0;
        for (int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x; i < n; i += vstride) {
            const double x = v0[i];
            V[i] = x;
            s += x * x;
        }
        arn_partial(s, vb, P, sh);
    }
    const double inv0 = 1.0 / sqrt(arn_finish(P, gv, grid, sh));
    for (int vb = blockIdx.x; vb < gv; vb += gridDim.x)
        for (int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x; i < n; i += vstride) V[i] *= inv0;
    arn_sync(grid);
    if (gridDim.x * kArnRegVb >= gv && static_cast<int64_t>(kArnRegElems) * vstride >= n) {
        // every physical block serves at most kArnRegVb virtual blocks of at most
        // kArnRegElems elements per thread: w stays in registers through the whole
        // Gram-Schmidt loop (a sub-step reads v_t and v_{t+1} only); same element order,
        // same per-virtual-block partials, same trees
        for (int j = 0; j < m; ++j) {
            const double* vj = V + static_cast<size_t>(j) * n;
            double wr[kArnRegVb][kArnRegElems];
            P = next_partials();
#pragma unroll
            for (int b = 0; b < kArnRegVb; ++b) {
                const int vb = blockIdx.x + b * gridDim.x;
                if (vb >= gv) break;
                double s = 0.0;
#pragma unroll
                for (int e = 0; e < kArnRegElems; ++e) {
                    const int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x + e * vstride;
                    wr[b][e] = 0.0;
                    if (i < n) {
                        double a = 0.0;
                        for (int32_t p = rp[i]; p < rp[i + 1]; ++p) a += va[p] * vj[ci[p]];
                        a *= dinv[i];
                        wr[b][e] = a;
                        s += a * V[i];
                    }
                }
                arn_partial(s, vb, P, sh);
            }
            double h = arn_finish(P, gv, grid, sh);
            for (int t = 0; t <= j; ++t) {
                if (blockIdx.x == 0 && threadIdx.x == 0) H[static_cast<size_t>(t) * m + j] = h;
                const double* vt = V + static_cast<size_t>(t) * n;
                const double* vn = t < j ? V + static_cast<size_t>(t + 1) * n : nullptr;
                const double a = -1.0 * h;
                P = next_partials();
#pragma unroll
                for (int b = 0; b < kArnRegVb; ++b) {
                    const int vb = blockIdx.x + b * gridDim.x;
                    if (vb >= gv) break;
                    double s = 0.0;
#pragma unroll
                    for (int e = 0; e < kArnRegElems; ++e) {
                        const int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x + e * vstride;
                        if (i < n) {
                            const double wi = wr[b][e] + a * vt[i];
                            wr[b][e] = wi;
                            s += wi * (vn ? vn[i] : wi);
                        }
                    }
                    arn_partial(s, vb, P, sh);
                }
                h = arn_finish(P, gv, grid, sh);
            }
            const double hn = sqrt(h);
            if (blockIdx.x == 0 && threadIdx.x == 0) H[static_cast<size_t>(j + 1) * m + j] = hn;
            const double inv = 1.0 / hn;
            double* w = V + static_cast<size_t>(j + 1) * n;
#pragma unroll
            for (int b = 0; b < kArnRegVb; ++b) {
                const int vb = blockIdx.x + b * gridDim.x;
                if (vb >= gv) break;
#pragma unroll
                for (int e = 0; e < kArnRegElems; ++e) {
                    const int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x + e * vstride;
                    if (i < n) w[i] = wr[b][e] * inv;
                }
            }
            arn_sync(grid);
        }
        return;
    }
    for (int j = 0; j < m; ++j) {
        const double* vj = V + static_cast<size_t>(j) * n;
        double* w = V + static_cast<size_t>(j + 1) * n;
        // w = D^-1 (A v_j), fused with (w, v_0)
        P = next_partials();
        for (int vb = blockIdx.x; vb < gv; vb += gridDim.x) {
            double s = 0.0;
            for (int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x; i < n; i += vstride) {
                double a = 0.0;
                for (int32_t p = rp[i]; p < rp[i + 1]; ++p) a += va[p] * vj[ci[p]];
                a *= dinv[i];
                w[i] = a;
                s += a * V[i];
            }
            arn_partial(s, vb, P, sh);
        }
        double h = arn_finish(P, gv, grid, sh);
        for (int t = 0; t <= j; ++t) {
            if (blockIdx.x == 0 && threadIdx.x == 0) H[static_cast<size_t>(t) * m + j] = h;
            const double* vt = V + static_cast<size_t>(t) * n;
            const double* vn = t < j ? V + static_cast<size_t>(t + 1) * n : nullptr;
            const double a = -1.0 * h;
            P = next_partials();
            for (int vb = blockIdx.x; vb < gv; vb += gridDim.x) {
                double s = 0.0;
                for (int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x; i < n; i += vstride) {
                    const double wi = w[i] + a * vt[i];
                    w[i] = wi;
                    s += wi * (vn ? vn[i] : wi);
                }
                arn_partial(s, vb, P, sh);
            }
            h = arn_finish(P, gv, grid, sh);
        }
        const double hn = sqrt(h);
        if (blockIdx.x == 0 && threadIdx.x == 0) H[static_cast<size_t>(j + 1) * m + j] = hn;
        // v_{j+1} = w * (1 / h) (a breakdown is detected on the host from H)
        const double inv = 1.0 / hn;
        for (int vb = blockIdx.x; vb < gv; vb += gridDim.x)
            for (int64_t i = static_cast<int64_t>(vb) * kArnThreads + threadIdx.x; i < n; i += vstride) w[i] *= inv;
        arn_sync(grid);
    }
}

}  // namespace

ArnoldiJob::~ArnoldiJob() {
    if (done) {
        cudaEventSynchronize(done);  // the buffers below are still being written
        cudaEventDestroy(done);
    }
    if (hpin) cudaFreeHost(hpin);
}

// Queues the whole Arnoldi process on the context's current stream (c.s) and an
// asynchronous copy of H to pinned memory; no host synchronisation, so it may run on a
// side stream while the setup goes on (spectral_radius_finish collects it).  The start
// vector must already cover n (ensure_start_vector on the main stream).
std::unique_ptr<ArnoldiJob> spectral_radius_start(Ctx& c, const DCsr& A, int steps, const double* dinv) {
    if (A.nr != A.nc) throw InvalidArgument("spectral_radius_estimate: square matrix required");
    const int32_t n = A.nr;
    auto job = std::make_unique<ArnoldiJob>();
    job->n = n;
    if (n == 0) return job;
    BlasFamilyScope scope(c, kProfArnoldiBlas1);
    const int m = std::min<int>(steps, n);
    job->m = m;
    if (c.arnoldi_v0_n < static_cast<size_t>(n)) throw std::logic_error("spectral_radius_start: start vector too short");
    job->V.alloc(static_cast<size_t>(n) * (m + 1), c.s);
    job->Hd.alloc(static_cast<size_t>(m + 1) * m + 1, c.s);
    DBuf<double>& V = job->V;
    DBuf<double>& Hd = job->Hd;
    AMG_CK(cudaMemsetAsync(Hd.get(), 0, sizeof(double) * ((m + 1) * m + 1), c.s));
    // AMGCU_ARNOLDI_STEPS=1 forces the launch-per-step path (the cooperative kernel's reference)
    const char* steps_env = std::getenv("AMGCU_ARNOLDI_STEPS");
    if (!c.seq && !(steps_env && steps_env[0] == '1')) {
        // one cooperative launch: grid = co-resident blocks, capped by the work
        static int per_sm = -1;
        if (per_sm < 0)
            AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_arnoldi_coop, kArnThreads, 0));
        // virtual grid = the launch-per-step path's dot grid (blas.cu), physical grid co-resident
        const int gv = static_cast<int>(dot_grid(c, n));
        // register path when g * kArnRegVb >= gv; the smallest levels run as one block
        const int g = gv <= kArnRegVb ? 1 : std::max(1, std::min(per_sm * c.sms, gv));
        ensure_reduction_scratch(c, 2 * static_cast<size_t>(gv));
        int32_t nn = n;
        int mm = m;
        int gvv = gv;
        const int32_t* rp = A.rp.get();
        const int32_t* ci = A.ci.get();
        const double* va = A.va.get();
        const double* v0 = c.arnoldi_v0.get();
        double* Vp = V.get();
        double* Hp = Hd.get();
        double* pp = c.partials.get();
        void* args[] = {&nn, &mm, &gvv, &rp, &ci, &va, &dinv, &v0, &Vp, &Hp, &pp};
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        const bool prof = c.profile && ((c.prof_mask >> kProfArnoldiBlas1) & 1u);
        if (prof) {
            e0 = prof_event(c);
            e1 = prof_event(c);
            AMG_CK(cudaEventRecord(e0, c.s));
        }
        AMG_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_arnoldi_coop), dim3(g), dim3(kArnThreads), args,
                                           0, c.s));
        ++c.launches;
        if (prof) {
            AMG_CK(cudaEventRecord(e1, c.s));
            ProfRecord& r = c.prof[kProfArnoldiBlas1];
            r.launches += 1;
            r.bytes += m * (12.0 * A.nnz + 4.0 * (n + 1) + 24.0 * n) + (m * (m + 1) / 2.0) * 32.0 * n;
            r.pending.emplace_back(e0, e1);
        }
    } else {
        double* nrm = Hd.get() + (m + 1) * m;
        copy_d2d(c, V.get(), c.arnoldi_v0.get(), n);
        nrm2(c, V.get(), n, nrm);
        scale_recip_dev(c, nrm, V.get(), n);
        for (int j = 0; j < m; ++j) {
            double* w = V.get() + static_cast<size_t>(j + 1) * n;
            launch_prof(c, kProfSpectralSpmv, 12.0 * A.nnz + 4.0 * (n + 1) + 24.0 * n, k_spmv_dinv, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), A.va.get(),
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
            // the breakdown test h < 1e-14 is taken after the loop on the downloaded H: the
            // columns before a breakdown never depend on the ones after it, so running the
            // remaining steps (on whatever the division produces) changes nothing that is used
            scale_recip_dev(c, hsub, w, n);
        }
    }
    const size_t hn = static_cast<size_t>(m + 1) * m;
    AMG_CK(cudaMallocHost(reinterpret_cast<void**>(&job->hpin), sizeof(double) * hn));
    copy_d2h(c, job->hpin, Hd.get(), static_cast<int64_t>(hn));
    AMG_CK(cudaEventCreateWithFlags(&job->done, cudaEventDisableTiming));
    AMG_CK(cudaEventRecord(job->done, c.s));
    return job;
}

double spectral_radius_finish(Ctx& c, ArnoldiJob& job, int* built_out) {
    if (job.n == 0) {
        if (built_out) *built_out = 0;
        return 0.0;
    }
    const int m = job.m;
    AMG_CK(cudaEventSynchronize(job.done));
    ++c.syncs;
    std::vector<double> H(job.hpin, job.hpin + static_cast<size_t>(m + 1) * m);
    int built = 0;
    for (int j = 0; j < m; ++j) {
        built = j + 1;
        if (H[static_cast<size_t>(j + 1) * m + j] < 1e-14) break;
    }
    if (built_out) *built_out = built;
    std::vector<double> Hs(static_cast<size_t>(built) * built), wr(built), wi(built);
    for (int i = 0; i < built; ++i)
        for (int j = 0; j < built; ++j) Hs[i * built + j] = H[i * m + j];
    if (sd::hessenberg_eigenvalues(built, Hs.data(), wr.data(), wi.data()) != 0)
        throw RuntimeError("spectral_radius_estimate: Hessenberg QR did not converge");
    double rho = 0.0;
    for (int i = 0; i < built; ++i) rho = std::max(rho, std::abs(std::complex<double>(wr[i], wi[i])));
    return rho;
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

double spectral_radius(Ctx& c, const DCsr& A, int steps, const double* dinv, int* built_out) {
    if (A.nr != A.nc) throw InvalidArgument("spectral_radius_estimate: square matrix required");
    ensure_start_vector(c, static_cast<size_t>(A.nr));
    auto job = spectral_radius_start(c, A, steps, dinv);
    return spectral_radius_finish(c, *job, built_out);
}

}  // namespace amgcu
