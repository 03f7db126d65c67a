// The remaining relaxation schemes of relaxation.hpp on the GPU: Gauss-Seidel on the
// normal equations (gsne, relaxation.hpp:128-142) and block symmetric Gauss-Seidel
// (relaxation.hpp:143-167), with their workspaces (relaxation.hpp:67-97).
//
// Both are ordered sweeps, run as sync-free wavefronts: items take tickets in sweep
// order, a value another item produces is read once it is published, and every sum
// runs in the reference's order (no FMA), so the results are bit-identical to the CPU.
#include <cuda/atomic>

#include <string>

#include "ops.cuh"
#include "small_dense.h"

namespace amgcu {

namespace {

constexpr unsigned long long kRmPending = 0x7FF4A11CE5EEDULL;  // published-value sentinel (as relax.cu)
constexpr int kRmWarps = 8;
constexpr int kBlkMax = 8;

__device__ __forceinline__ unsigned long long rm_load(const double* p) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(
        *reinterpret_cast<unsigned long long*>(const_cast<double*>(p)));
    return r.load(cuda::memory_order_relaxed);
}
__device__ __forceinline__ void rm_store(double* p, double v) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(*reinterpret_cast<unsigned long long*>(p));
    r.store(static_cast<unsigned long long>(__double_as_longlong(v)), cuda::memory_order_relaxed);
}

__global__ void k_rm_fill_pending(int64_t count, double* __restrict__ p) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < count) reinterpret_cast<unsigned long long*>(p)[t] = kRmPending;
}

// ---- block symmetric Gauss-Seidel -------------------------------------------------------

// m x m diagonal block inverses (make_relax_workspace, relaxation.hpp:79-97): the block's
// entries (assigned, others zero), FullPivLU, invertible iff full rank; row-major.
__global__ void k_block_inverse(int32_t nb, int m, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ va, double* __restrict__ inv, int32_t* __restrict__ bad) {
    const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    double M[kBlkMax * kBlkMax];
    for (int e = 0; e < m * m; ++e) M[e] = 0.0;
    for (int r = 0; r < m; ++r) {
        const int32_t i = b * m + r;
        for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int32_t j = ci[p];
            if (j / m == b) M[r * m + (j - b * m)] = va[p];
        }
    }
    sd::FullPivLU<kBlkMax> lu;
    lu.compute(m, M);
    if (lu.rank() != m) {
        atomicMin(bad, b);
        return;
    }
    lu.inverse(inv + static_cast<size_t>(b) * m * m);
}

// One item = one block of one half-sweep (forward on even halves, backward on odd),
// one warp: the lanes form the products of the block's rows with the values outside the
// block (new for blocks already passed in this half-sweep, else the previous half's),
// lane 0 subtracts them from b in CSR order, then applies the block inverse.
__global__ void __launch_bounds__(kRmWarps * 32)
    k_block_gs(int32_t nb, int m, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
               const double* __restrict__ va, const double* __restrict__ inv, const double* __restrict__ b,
               int halves, double* __restrict__ X, unsigned int* __restrict__ ticket) {
    __shared__ unsigned int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t item = static_cast<int64_t>(blk) * kRmWarps + threadIdx.x / 32;
    if (item >= static_cast<int64_t>(halves) * nb) return;
    const int lane = threadIdx.x & 31;
    const int h = static_cast<int>(item / nb);
    const int32_t s = static_cast<int32_t>(item - static_cast<int64_t>(h) * nb);
    const bool fwd = (h & 1) == 0;
    const int32_t bk = fwd ? s : nb - 1 - s;
    const size_t n = static_cast<size_t>(nb) * m;
    const double* xin = X + static_cast<size_t>(h) * n;
    double* xout = X + static_cast<size_t>(h + 1) * n;
    double rhs[kBlkMax];
    for (int r = 0; r < m; ++r) {
        const int32_t i = bk * m + r;
        double acc = b ? b[i] : 0.0;
        const int32_t lo = rp[i], hi = rp[i + 1];
        for (int32_t e0 = lo; e0 < hi; e0 += 32) {
            const int32_t p = e0 + lane;
            bool use = false;
            const double* addr = nullptr;
            double a = 0.0;
            if (p < hi) {
                const int32_t j = ci[p];
                const int32_t jb = j / m;
                if (jb != bk) {
                    use = true;
                    a = va[p];
                    const bool fresh = fwd ? jb < bk : jb > bk;
                    addr = (fresh ? xout : xin) + j;
                }
            }
            unsigned long long v = use ? rm_load(addr) : 0ull;
            unsigned ns = 8;
            while (__any_sync(0xffffffffu, use && v == kRmPending)) {
                if (use && v == kRmPending) {
                    __nanosleep(ns);
                    v = rm_load(addr);
                }
                ns = ns < 256 ? 2 * ns : 256;
            }
            const double prod = use ? a * __longlong_as_double(static_cast<long long>(v)) : 0.0;
            const unsigned um = __ballot_sync(0xffffffffu, use);
            for (unsigned mm = um; mm; mm &= mm - 1) acc -= __shfl_sync(0xffffffffu, prod, __ffs(mm) - 1);
        }
        rhs[r] = acc;
    }
    if (lane == 0) {
        const double* bi = inv + static_cast<size_t>(bk) * m * m;
        for (int r = 0; r < m; ++r) {
            double acc = 0.0;
            for (int cc = 0; cc < m; ++cc) acc += bi[r * m + cc] * rhs[cc];
            rm_store(xout + static_cast<size_t>(bk) * m + r, acc);
        }
    }
}

// ---- Gauss-Seidel on the normal equations ------------------------------------------------

__global__ void k_col_norm2(int32_t nc, const int32_t* __restrict__ trp, const double* __restrict__ tva,
                            double* __restrict__ cn2, int32_t* __restrict__ bad) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nc) return;
    double s = 0.0;
    for (int32_t p = trp[i]; p < trp[i + 1]; ++p) s += tva[p] * tva[p];
    cn2[i] = s;
    if (s == 0.0) atomicMin(bad, i);
}

// r = b - A x (spmv in CSR order, then the subtraction; b == nullptr: zero)
__global__ void k_rm_residual(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const double* __restrict__ va, const double* __restrict__ x, const double* __restrict__ b,
                              double* __restrict__ r) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) s += va[p] * x[ci[p]];
    r[i] = (b ? b[i] : 0.0) - s;
}

// One item = one column i (ascending tickets), one warp.  Row j of the residual takes
// the updates of the columns touching it in column order: column i may read r[j] once
// done[j] equals its rank in row j (the stored columns of A's row j below i), and it
// releases done[j] = rank + 1 after its own update r[j] -= delta * a.
__global__ void __launch_bounds__(kRmWarps * 32)
    k_gsne_cols(int32_t nc, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                const int32_t* __restrict__ trp, const int32_t* __restrict__ tci, const double* __restrict__ tva,
                const double* __restrict__ cn2, double* __restrict__ x, double* __restrict__ r,
                int32_t* __restrict__ done, unsigned int* __restrict__ ticket) {
    __shared__ unsigned int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const int32_t i = static_cast<int32_t>(blk) * kRmWarps + threadIdx.x / 32;
    if (i >= nc) return;
    const int lane = threadIdx.x & 31;
    const int32_t lo = trp[i], hi = trp[i + 1];
    double num = 0.0;
    for (int32_t e0 = lo; e0 < hi; e0 += 32) {
        const int32_t p = e0 + lane;
        double prod = 0.0;
        if (p < hi) {
            const int32_t j = tci[p];
            int32_t a0 = rp[j], a1 = rp[j + 1];
            const int32_t base = a0;
            while (a0 < a1) {  // rank of column i in row j
                const int32_t mid = (a0 + a1) >> 1;
                if (ci[mid] < i) a0 = mid + 1;
                else a1 = mid;
            }
            const int32_t rank = a0 - base;
            cuda::atomic_ref<int32_t, cuda::thread_scope_device> dj(done[j]);
            unsigned ns = 8;
            while (dj.load(cuda::memory_order_acquire) != rank) {
                __nanosleep(ns);
                ns = ns < 256 ? 2 * ns : 256;
            }
            prod = tva[p] * __longlong_as_double(static_cast<long long>(rm_load(r + j)));
        }
        const int cnt = min(32, hi - e0);
        for (int t = 0; t < cnt; ++t) num += __shfl_sync(0xffffffffu, prod, t);
    }
    const double delta = num / cn2[i];
    if (lane == 0) x[i] += delta;
    for (int32_t p = lo + lane; p < hi; p += 32) {
        const int32_t j = tci[p];
        const double rj = __longlong_as_double(static_cast<long long>(rm_load(r + j)));
        rm_store(r + j, rj - delta * tva[p]);
        int32_t a0 = rp[j], a1 = rp[j + 1];
        const int32_t base = a0;
        while (a0 < a1) {
            const int32_t mid = (a0 + a1) >> 1;
            if (ci[mid] < i) a0 = mid + 1;
            else a1 = mid;
        }
        cuda::atomic_ref<int32_t, cuda::thread_scope_device> dj(done[j]);
        dj.store(a0 - base + 1, cuda::memory_order_release);
    }
}

}  // namespace

void gsne_workspace(Ctx& c, const DCsr& A, GsneWs& ws) {
    if (A.nr != A.nc) throw InvalidArgument("relax: square matrix required");
    transpose(c, A, ws.At);
    const int32_t nc = A.nc;
    ws.cn2.alloc(static_cast<size_t>(nc), c.s);
    DBuf<int32_t> bad(1, c.s);
    fill_i32(c, bad.get(), INT32_MAX, 1);
    launch(c, k_col_norm2, blocks_for(nc, 256), 256, 0, nc, ws.At.rp.get(), ws.At.va.get(), ws.cn2.get(), bad.get());
    const int32_t b = read_scalar(c, bad.get());
    if (b != INT32_MAX) throw RuntimeError("relax: zero column at " + std::to_string(b));
}

void gsne(Ctx& c, const DCsr& A, const GsneWs& ws, double* x, const double* b, int sweeps) {
    const int32_t n = A.nr;
    if (sweeps <= 0 || n == 0) return;
    DBuf<double> r(static_cast<size_t>(n), c.s);
    DBuf<int32_t> done(static_cast<size_t>(n), c.s);
    DBuf<unsigned int> ticket(1, c.s);
    for (int s = 0; s < sweeps; ++s) {
        launch(c, k_rm_residual, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), A.va.get(),
               static_cast<const double*>(x), b, r.get());
        AMG_CK(cudaMemsetAsync(done.get(), 0, sizeof(int32_t) * n, c.s));
        AMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned int), c.s));
        launch_prof(c, kProfGaussSeidel, 24.0 * A.nnz + 8.0 * (n + 1) + 32.0 * n, k_gsne_cols,
                    blocks_for(A.nc, kRmWarps), kRmWarps * 32, 0, A.nc, A.rp.get(), A.ci.get(), ws.At.rp.get(),
                    ws.At.ci.get(), ws.At.va.get(), ws.cn2.get(), x, r.get(), done.get(), ticket.get());
    }
}

void block_workspace(Ctx& c, const DCsr& A, DBuf<double>& inv) {
    const int32_t m = A.bs;
    if (A.nr != A.nc) throw InvalidArgument("relax: square matrix required");
    if (m < 1 || A.nr % m != 0) throw InvalidArgument("relax: bad block size for block relaxation");
    if (m > kBlkMax) throw InvalidArgument("relax: block sizes above 8 are not on the GPU path");
    const int32_t nb = A.nr / m;
    inv.alloc(static_cast<size_t>(nb) * m * m, c.s);
    DBuf<int32_t> bad(1, c.s);
    fill_i32(c, bad.get(), INT32_MAX, 1);
    launch(c, k_block_inverse, blocks_for(nb, 128), 128, 0, nb, static_cast<int>(m), A.rp.get(), A.ci.get(),
           A.va.get(), inv.get(), bad.get());
    const int32_t b = read_scalar(c, bad.get());
    if (b != INT32_MAX) throw RuntimeError("relax: singular diagonal block " + std::to_string(b));
}

void block_sym_gs(Ctx& c, const DCsr& A, const double* inv, double* x, const double* b, int sweeps) {
    const int32_t m = A.bs;
    const int32_t nb = A.nr / m;
    const int halves = 2 * sweeps;
    if (sweeps <= 0 || nb == 0) return;
    const size_t n = static_cast<size_t>(A.nr);
    DBuf<double> X(n * (halves + 1), c.s);
    copy_d2d(c, X.get(), x, static_cast<int64_t>(n));
    launch(c, k_rm_fill_pending, blocks_for(static_cast<int64_t>(n) * halves, 256), 256, 0,
           static_cast<int64_t>(n) * halves, X.get() + n);
    DBuf<unsigned int> ticket(1, c.s);
    AMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned int), c.s));
    const int64_t items = static_cast<int64_t>(halves) * nb;
    launch_prof(c, kProfGaussSeidel, halves * (12.0 * A.nnz + 4.0 * (n + 1) + 16.0 * n),
                k_block_gs, static_cast<unsigned>((items + kRmWarps - 1) / kRmWarps), kRmWarps * 32, 0, nb,
                static_cast<int>(m), A.rp.get(), A.ci.get(), A.va.get(), inv, b, halves, X.get(), ticket.get());
    copy_d2d(c, x, X.get() + n * halves, static_cast<int64_t>(n));
}

}  // namespace amgcu
