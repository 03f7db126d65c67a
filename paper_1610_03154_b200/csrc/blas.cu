// BLAS-1 on device-resident scalars (sparse.hpp:309-323).
//
// Ctx::seq (the default): every sum is the reference's s = ((0 + x0 y0) + x1 y1) + ...
// bit for bit, evaluated in parallel by seqsum.cu (AMGCU_SEQ_NAIVE=1: by one warp, the
// slow original, kept to A/B the fast one).  Ctx::seq off: a deterministic two-stage
// tree (fixed grid, fixed per-thread order, last-block final sum in index order of the
// block partials) -- reproducible, but not the reference's bits.
#include <cub/block/block_reduce.cuh>

#include <algorithm>
#include <cstdlib>

#include "ops.cuh"

namespace amgcu {

namespace {

constexpr int kDotThreads = 256;

// Final stage shared by the tree reductions: the last block to finish sums the
// block partials with a block-wide (fixed-shape, hence deterministic) reduction.
__device__ __forceinline__ void finish_tree(double b, double* __restrict__ partials, unsigned int* __restrict__ done,
                                            double* __restrict__ out, bool take_sqrt) {
    using BR = cub::BlockReduce<double, kDotThreads>;
    __shared__ typename BR::TempStorage tmp2;
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = b;
        __threadfence();
        const unsigned prev = atomicAdd(done, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t = 0.0;
    for (unsigned k = threadIdx.x; k < gridDim.x; k += kDotThreads) t += __ldcg(&partials[k]);
    t = BR(tmp2).Sum(t);
    if (threadIdx.x == 0) {
        *out = take_sqrt ? sqrt(t) : t;
        *done = 0u;  // reset for the next call on this stream
    }
}

// per-thread partial over a grid-stride range, kUnroll independent loads in flight
constexpr int kUnroll = 4;

__global__ void __launch_bounds__(kDotThreads)
    k_dot_tree(const double* __restrict__ x, const double* __restrict__ y, int64_t n, double* __restrict__ partials,
               unsigned int* __restrict__ done, double* __restrict__ out, bool take_sqrt) {
    using BR = cub::BlockReduce<double, kDotThreads>;
    __shared__ typename BR::TempStorage tmp;
    double s = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kDotThreads;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kDotThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n; i += kUnroll * stride) {
        double xv[kUnroll], yv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            xv[u] = __ldg(&x[i + u * stride]);
            yv[u] = __ldg(&y[i + u * stride]);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) s += xv[u] * yv[u];
    }
    for (; i < n; i += stride) s += x[i] * y[i];
    const double b = BR(tmp).Sum(s);
    finish_tree(b, partials, done, out, take_sqrt);
}

// y += sign * (*alpha) * x, then *out = dot(y, z) (z == nullptr: dot(y, y),
// optionally square-rooted) -- one pass for a modified Gram-Schmidt step
// (the reference's axpy followed by the next dot, spectral.hpp:47-51).
__global__ void __launch_bounds__(kDotThreads)
    k_axpy_dot_tree(const double* __restrict__ alpha, double sign, const double* __restrict__ x,
                    double* __restrict__ y, const double* __restrict__ z, int64_t n, double* __restrict__ partials,
                    unsigned int* __restrict__ done, double* __restrict__ out, bool take_sqrt) {
    using BR = cub::BlockReduce<double, kDotThreads>;
    __shared__ typename BR::TempStorage tmp;
    const double a = sign * (*alpha);
    double s = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kDotThreads;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kDotThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n; i += kUnroll * stride) {
        double yv[kUnroll], xv[kUnroll], zv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            yv[u] = y[i + u * stride];
            xv[u] = __ldg(&x[i + u * stride]);
            zv[u] = z ? __ldg(&z[i + u * stride]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const double yi = yv[u] + a * xv[u];
            y[i + u * stride] = yi;
            s += yi * (z ? zv[u] : yi);
        }
    }
    for (; i < n; i += stride) {
        const double yi = y[i] + a * x[i];
        y[i] = yi;
        s += yi * (z ? z[i] : yi);
    }
    const double b = BR(tmp).Sum(s);
    finish_tree(b, partials, done, out, take_sqrt);
}

// PCG step (cycle.hpp:190-194): x += alpha p, r -= alpha q (alpha = st[2]), then
// *out = ||r|| -- the norm summed exactly as k_dot_tree sums (r, r) on the same grid, so
// the fused pass gives the same bits as the update followed by nrm2.  Skipped (no
// update, no norm) when *bad is set.
__global__ void __launch_bounds__(kDotThreads)
    k_pcg_update_nrm(const double* __restrict__ st, const int32_t* __restrict__ bad, const double* __restrict__ p,
                     const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r, int64_t n,
                     double* __restrict__ partials, unsigned int* __restrict__ done, double* __restrict__ out) {
    using BR = cub::BlockReduce<double, kDotThreads>;
    __shared__ typename BR::TempStorage tmp;
    if (*bad) return;
    const double a = st[2];
    const double na = -a;
    double s = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kDotThreads;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kDotThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n; i += kUnroll * stride) {
        double rv[kUnroll], qv[kUnroll], xv[kUnroll], pv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            rv[u] = r[i + u * stride];
            qv[u] = __ldg(&q[i + u * stride]);
            xv[u] = x[i + u * stride];
            pv[u] = __ldg(&p[i + u * stride]);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            x[i + u * stride] = xv[u] + a * pv[u];
            const double ri = rv[u] + na * qv[u];
            r[i + u * stride] = ri;
            s += ri * ri;
        }
    }
    for (; i < n; i += stride) {
        x[i] += a * p[i];
        const double ri = r[i] + na * q[i];
        r[i] = ri;
        s += ri * ri;
    }
    const double b = BR(tmp).Sum(s);
    finish_tree(b, partials, done, out, true);
}

__global__ void k_dot_seq(const double* __restrict__ x, const double* __restrict__ y, int64_t n, double* __restrict__ out,
                          bool take_sqrt) {
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int64_t base = 0; base < n; base += 32) {
        const int64_t i = base + lane;
        const double v = i < n ? x[i] * y[i] : 0.0;
        const int cnt = static_cast<int>(n - base < 32 ? n - base : 32);
        for (int t = 0; t < cnt; ++t) s += __shfl_sync(0xffffffffu, v, t);
    }
    if (lane == 0) *out = take_sqrt ? sqrt(s) : s;
}

__global__ void k_axpy_dev(const double* __restrict__ alpha, double sign, const double* __restrict__ x,
                           double* __restrict__ y, int64_t n) {
    const double a = sign * (*alpha);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[i] += a * x[i];
}

__global__ void k_scale_recip(const double* __restrict__ denom, double* __restrict__ x, int64_t n) {
    const double a = 1.0 / (*denom);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] *= a;
}

__global__ void k_scale_const(double a, double* __restrict__ x, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] *= a;
}

unsigned stream_grid(Ctx& c, int64_t n) {
    return std::max(1u, std::min<unsigned>(blocks_for(n, 256), 8u * c.sms));
}

}  // namespace

unsigned dot_grid(Ctx& c, int64_t n) {
    return std::max(1u, std::min<unsigned>(blocks_for(n, kDotThreads * kUnroll), 8u * c.sms));
}

namespace {

bool seq_naive() {
    static const bool on = [] {
        const char* e = std::getenv("AMGCU_SEQ_NAIVE");
        return e && e[0] == '1';
    }();
    return on;
}

void dot_impl(Ctx& c, const double* x, const double* y, int64_t n, double* out, bool take_sqrt) {
    if (c.seq) {
        if (seq_naive())
            launch_prof(c, c.blas_family, 16.0 * n, k_dot_seq, 1, 32, 0, x, y, n, out, take_sqrt);
        else
            seqsum_dot(c, x, y, n, out, take_sqrt);
        return;
    }
    const unsigned g = dot_grid(c, n);
    ensure_reduction_scratch(c, g);
    launch_prof(c, c.blas_family, 16.0 * n, k_dot_tree, g, kDotThreads, 0, x, y, n, c.partials.get(), c.tickets.get(), out, take_sqrt);
}

}  // namespace

void axpy_dot(Ctx& c, const double* alpha, double sign, const double* x, double* y, const double* z, int64_t n,
              double* out, bool take_sqrt) {
    if (c.seq) {
        if (seq_naive()) {
            axpy_dev(c, alpha, sign, x, y, n);
            dot_impl(c, y, z ? z : y, n, out, take_sqrt);
        } else {
            seqsum_axpy_dot(c, alpha, sign, x, y, z, n, out, take_sqrt);
        }
        return;
    }
    const unsigned g = dot_grid(c, n);
    ensure_reduction_scratch(c, g);
    launch_prof(c, c.blas_family, (z ? 32.0 : 24.0) * n, k_axpy_dot_tree, g, kDotThreads, 0, alpha, sign, x, y, z, n, c.partials.get(), c.tickets.get(), out,
           take_sqrt);
}

void dot(Ctx& c, const double* x, const double* y, int64_t n, double* out) { dot_impl(c, x, y, n, out, false); }
void nrm2(Ctx& c, const double* x, int64_t n, double* out) { dot_impl(c, x, x, n, out, true); }

bool pcg_update_nrm(Ctx& c, const double* st, const int32_t* bad, const double* p, const double* q, double* x,
                    double* r, int64_t n, double* out) {
    if (c.seq) {
        if (seq_naive()) return false;  // the update kernel and the one-warp norm
        seqsum_pcg_update_nrm(c, st, bad, p, q, x, r, n, out);
        return true;
    }
    const unsigned g = dot_grid(c, n);
    ensure_reduction_scratch(c, g);
    launch_prof(c, kProfBlas1, 56.0 * n, k_pcg_update_nrm, g, kDotThreads, 0, st, bad, p, q, x, r, n,
                c.partials.get(), c.tickets.get(), out);
    return true;
}

void axpy_dev(Ctx& c, const double* alpha, double sign, const double* x, double* y, int64_t n) {
    launch_prof(c, c.blas_family, 24.0 * n, k_axpy_dev, stream_grid(c, n), 256, 0, alpha, sign, x, y, n);
}
void scale_recip_dev(Ctx& c, const double* denom, double* x, int64_t n) {
    launch_prof(c, c.blas_family, 16.0 * n, k_scale_recip, stream_grid(c, n), 256, 0, denom, x, n);
}
void scale_const(Ctx& c, double alpha, double* x, int64_t n) {
    launch_prof(c, c.blas_family, 16.0 * n, k_scale_const, stream_grid(c, n), 256, 0, alpha, x, n);
}

}  // namespace amgcu
