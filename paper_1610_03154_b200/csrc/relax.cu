// Relaxation on the GPU (relaxation.hpp).
//
// Gauss-Seidel (relaxation.hpp:115-127) is inherently ordered: row i uses the
// new values of the rows before it and the old values of the rows after it.
// All sweeps run in ONE sync-free launch: work item (s, i) = sweep s on row i
// (row order reversed for backward sweeps), tickets are drawn in item order,
// item (s, i) waits for the rows it reads (same sweep, earlier rows) and for
// the previous sweep of the later rows -- both have lower tickets, so the
// launch cannot deadlock.  Every sweep writes its own copy of x (sweeps + 1
// buffers), so reads never race with writes and each row sum is evaluated in
// CSR order exactly as on the CPU.  k candidate columns are swept together.
#include <cuda/atomic>

#include "ops.cuh"

namespace amgcu {

namespace {

constexpr int kGsThreads = 128;
constexpr int kMaxK = 8;

__global__ void __launch_bounds__(kGsThreads)
    k_gs_wavefront(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                   const double* __restrict__ va, const double* __restrict__ inv_diag, const double* __restrict__ b,
                   int k, int nsweeps, const unsigned char* __restrict__ backward, double* __restrict__ X,
                   int32_t* __restrict__ done, unsigned int* __restrict__ ticket) {
    __shared__ unsigned int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t item = static_cast<int64_t>(blk) * kGsThreads + threadIdx.x;
    if (item >= static_cast<int64_t>(n) * nsweeps) return;
    const int s = static_cast<int>(item / n);
    const int32_t q = static_cast<int32_t>(item - static_cast<int64_t>(s) * n);
    const bool bwd = backward[s] != 0;
    const int32_t i = bwd ? n - 1 - q : q;
    const size_t stride = static_cast<size_t>(n) * k;
    const double* xin = X + static_cast<size_t>(s) * stride;
    double* xout = X + static_cast<size_t>(s + 1) * stride;
    double acc[kMaxK];
    for (int c = 0; c < k; ++c) acc[c] = b ? b[static_cast<size_t>(c) * n + i] : 0.0;
    cuda::atomic_ref<int32_t, cuda::thread_scope_device> mine(done[i]);
    int32_t p = rp[i];
    const int32_t pend = rp[i + 1];
    // walk the row in CSR order; wait for each dependency before using it
    while (true) {
        bool blocked = false;
        for (; p < pend; ++p) {
            const int32_t j = ci[p];
            if (j == i) continue;
            const bool fresh = bwd ? (j > i) : (j < i);  // already updated in this sweep
            const int32_t need = fresh ? s + 1 : s;
            if (need > 0) {
                cuda::atomic_ref<int32_t, cuda::thread_scope_device> dj(done[j]);
                if (dj.load(cuda::memory_order_acquire) < need) {
                    blocked = true;
                    break;
                }
            }
            const double* src = fresh ? xout : xin;
            for (int c = 0; c < k; ++c) acc[c] -= va[p] * __ldcg(&src[static_cast<size_t>(c) * n + j]);
        }
        if (!blocked) {
            for (int c = 0; c < k; ++c) __stcg(&xout[static_cast<size_t>(c) * n + i], acc[c] * inv_diag[i]);
            mine.store(s + 1, cuda::memory_order_release);
            break;
        }
        __nanosleep(32);
    }
}

// x_out = x_in + (w dinv) (b - A x_in) for all k columns (relaxation.hpp:107-113)
__global__ void k_jacobi(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                         const double* __restrict__ va, const double* __restrict__ wdinv, const double* __restrict__ b,
                         int k, const double* __restrict__ xin, double* __restrict__ xout) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int c = 0; c < k; ++c) {
        const double* x = xin + static_cast<size_t>(c) * n;
        double s = 0.0;
        for (int32_t p = rp[i]; p < rp[i + 1]; ++p) s += va[p] * x[ci[p]];
        const double bi = b ? b[static_cast<size_t>(c) * n + i] : 0.0;
        xout[static_cast<size_t>(c) * n + i] = x[i] + wdinv[i] * (bi - s);
    }
}

}  // namespace

void gauss_seidel(Ctx& c, const DCsr& A, const double* inv_diag, double* x, const double* b, int k, int sweeps,
                  bool symmetric_sweep) {
    if (k > kMaxK) throw InvalidArgument("relax: at most 8 candidate columns on the GPU path");
    const int32_t n = A.nr;
    const int nsw = symmetric_sweep ? 2 * sweeps : sweeps;
    if (nsw == 0 || n == 0) return;
    const size_t stride = static_cast<size_t>(n) * k;
    DBuf<double> X(stride * (nsw + 1), c.s);
    copy_d2d(c, X.get(), x, static_cast<int64_t>(stride));
    std::vector<unsigned char> hb(nsw);
    for (int s = 0; s < nsw; ++s) hb[s] = symmetric_sweep ? static_cast<unsigned char>(s & 1) : 0;
    DBuf<unsigned char> bwd(static_cast<size_t>(nsw), c.s);
    copy_h2d(c, bwd.get(), hb.data(), nsw);
    DBuf<int32_t> done(static_cast<size_t>(n), c.s);
    AMG_CK(cudaMemsetAsync(done.get(), 0, sizeof(int32_t) * n, c.s));
    DBuf<unsigned int> ticket(1, c.s);
    AMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned int), c.s));
    launch(c, k_gs_wavefront, blocks_for(static_cast<int64_t>(n) * nsw, kGsThreads), kGsThreads, 0, n, A.rp.get(),
           A.ci.get(), A.va.get(), inv_diag, b, k, nsw, static_cast<const unsigned char*>(bwd.get()), X.get(),
           done.get(), ticket.get());
    copy_d2d(c, x, X.get() + stride * nsw, static_cast<int64_t>(stride));
    sync(c);  // hb must outlive the async copy
}

void jacobi(Ctx& c, const DCsr& A, const double* wdinv, double* x, const double* b, int k, int sweeps) {
    const int32_t n = A.nr;
    if (sweeps == 0 || n == 0) return;
    DBuf<double> tmp(static_cast<size_t>(n) * k, c.s);
    double* cur = x;
    double* nxt = tmp.get();
    for (int s = 0; s < sweeps; ++s) {
        launch(c, k_jacobi, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), A.va.get(), wdinv, b, k,
               static_cast<const double*>(cur), nxt);
        std::swap(cur, nxt);
    }
    if (cur != x) copy_d2d(c, x, cur, static_cast<int64_t>(n) * k);
}

}  // namespace amgcu
