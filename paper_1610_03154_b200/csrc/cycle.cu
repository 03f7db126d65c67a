// Solve phase on the GPU: V/W cycle (cycle.hpp:70-95) and the stationary /
// PCG / FGMRES drivers (cycle.hpp:114-271).
//
// Level operators are mirrored into sliced ELL (32-row slices, column-major
// inside a slice, rows kept in order) so one thread per row sums its row in CSR
// order -- reference-exact -- while the warp's loads stay coalesced.  Fusions
// (all reference-exact):
//   * pre-relaxation from x = 0 (every cycle entry of the preconditioner and
//     every coarse level) is x = (w D^-1) b, and is fused with the residual
//     r = b - A x, recomputing neighbour x_j = (w D^-1)_j b_j in registers;
//   * interpolate-and-correct t = x + P x_c is one pass;
//   * post-relaxation x = t + (w D^-1)(b - A t) is one pass;
//   * restriction b_c = R r is a gather over R's rows (no atomics).
// Krylov scalars stay on the device; the host reads one small status record
// per iteration (the residual norm decides termination, as in the reference).
#include <cooperative_groups.h>

#include <chrono>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "hier.cuh"

namespace amgcu {

namespace {

constexpr int kSlice = 32;
constexpr int kWarpRowThreshold = 32;  // average row length from which warp-per-row kernels are used

__global__ void k_slice_len(int32_t nr, const int32_t* __restrict__ rp, int64_t* __restrict__ slen) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t nsl = (nr + kSlice - 1) / kSlice;
    if (s >= nsl) return;
    int32_t mx = 0;
    for (int32_t r = s * kSlice; r < min(nr, s * kSlice + kSlice); ++r) mx = max(mx, rp[r + 1] - rp[r]);
    slen[s] = static_cast<int64_t>(mx) * kSlice;
}

__global__ void k_sell_fill(int32_t nr, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ va, const int64_t* __restrict__ sptr, int32_t* __restrict__ sci,
                            double* __restrict__ sva, int32_t* __restrict__ slen) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t s = i / kSlice, lane = i % kSlice;
    const int32_t nsl = (nr + kSlice - 1) / kSlice;
    if (s >= nsl) return;
    const int64_t base = sptr[s];
    const int32_t width = static_cast<int32_t>((sptr[s + 1] - base) / kSlice);
    if (lane == 0) slen[s] = width;
    int32_t len = 0, lo = 0;
    if (i < nr) {
        lo = rp[i];
        len = rp[i + 1] - lo;
    }
    for (int32_t e = 0; e < width; ++e) {
        const int64_t at = base + static_cast<int64_t>(e) * kSlice + lane;
        if (e < len) {
            sci[at] = ci[lo + e];
            sva[at] = va[lo + e];
        } else {
            sci[at] = -1;
            sva[at] = 0.0;
        }
    }
}

// Row sum over a SELL row in stored (CSR) order.  Entries are loaded kBatch at a
// time with predication instead of stopping at the first padding slot, so a
// thread keeps kBatch column/value loads and then kBatch gathers in flight;
// padding (column -1, always after the row's entries) is skipped by predicate,
// so the sum is the reference's sequential one.
constexpr int kBatch = 16;

template <typename Gather>
__device__ __forceinline__ double sell_row_sum(int64_t base, int32_t w, const int32_t* __restrict__ sci,
                                               const double* __restrict__ sva, Gather gx) {
    double acc = 0.0;
    for (int32_t e0 = 0; e0 < w; e0 += kBatch) {
        int32_t j[kBatch];
        double a[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int32_t e = e0 + u;
            j[u] = -1;
            a[u] = 0.0;
            if (e < w) {
                j[u] = __ldg(&sci[base + static_cast<int64_t>(e) * kSlice]);
                a[u] = __ldg(&sva[base + static_cast<int64_t>(e) * kSlice]);
            }
        }
        double xv[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) xv[u] = j[u] >= 0 ? gx(j[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
            if (j[u] >= 0) acc += a[u] * xv[u];
    }
    return acc;
}

__device__ __forceinline__ double sell_row(int32_t i, const int64_t* __restrict__ sptr, const int32_t* __restrict__ slen,
                                           const int32_t* __restrict__ sci, const double* __restrict__ sva,
                                           const double* __restrict__ x) {
    const int32_t s = i / kSlice, lane = i % kSlice;
    return sell_row_sum(sptr[s] + lane, slen[s], sci, sva, [&](int32_t j) { return __ldg(&x[j]); });
}

struct SellView {
    int32_t nr;
    const int64_t* sptr;
    const int32_t* slen;
    const int32_t* ci;
    const double* va;
    const int32_t* crp;  // CSR of the same operator (warp-per-row kernels)
    const int32_t* cci;
    const double* cva;
};

SellView view(const DSell& s) {
    return {s.nr, s.slice_ptr.get(), s.slice_len.get(), s.ci.get(), s.va.get(), s.crp, s.cci, s.cva};
}

// Warp per row for operators with long rows (coarse levels, restriction): the
// lanes form the row's products a_p * x_{c_p} in parallel into shared memory and
// lane 0 sums them in CSR order -- the reference's sequential sum, with the
// loads of a long row in flight together instead of one thread walking it.
constexpr int kWarpRowsPerBlock = 8;
constexpr int32_t kWarpRowMaxRows = 65536;  // from this many rows, thread per row even for long rows
constexpr int kWarpCap = 256;  // products staged per pass

template <typename Gather>
__device__ __forceinline__ double warp_row_sum(const SellView& A, int32_t i, Gather gx, double* buf, int lane) {
    double acc = 0.0;
    const int32_t lo = A.crp[i], hi = A.crp[i + 1];
    for (int32_t base = lo; base < hi; base += kWarpCap) {
        const int32_t len = min(kWarpCap, hi - base);
        for (int32_t e = lane; e < len; e += 32) buf[e] = __ldg(&A.cva[base + e]) * gx(__ldg(&A.cci[base + e]));
        __syncwarp();
        if (lane == 0) {
#pragma unroll 8
            for (int32_t e = 0; e < len; ++e) acc += buf[e];
        }
        __syncwarp();
    }
    return acc;  // lane 0
}

#define AMGCU_WARP_ROW_PROLOGUE                                                  \
    __shared__ double wbuf[kWarpRowsPerBlock][kWarpCap];                          \
    const int lane = threadIdx.x & 31, wrow = threadIdx.x / 32;                   \
    const int32_t i = blockIdx.x * kWarpRowsPerBlock + wrow;                      \
    if (i >= A.nr) return;                                                        \
    double* buf = wbuf[wrow];

__global__ void __launch_bounds__(kWarpRowsPerBlock * 32)
    k_wspmv(SellView A, const double* __restrict__ x, double* __restrict__ y) {
    AMGCU_WARP_ROW_PROLOGUE
    const double s = warp_row_sum(A, i, [&](int32_t j) { return __ldg(&x[j]); }, buf, lane);
    if (lane == 0) y[i] = s;
}

__global__ void __launch_bounds__(kWarpRowsPerBlock * 32)
    k_wresidual(SellView A, const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r) {
    AMGCU_WARP_ROW_PROLOGUE
    const double s = warp_row_sum(A, i, [&](int32_t j) { return __ldg(&x[j]); }, buf, lane);
    if (lane == 0) r[i] = b[i] - s;
}

__global__ void __launch_bounds__(kWarpRowsPerBlock * 32)
    k_wrelax0_residual(SellView A, const double* __restrict__ wd, const double* __restrict__ b,
                       double* __restrict__ x, double* __restrict__ r) {
    AMGCU_WARP_ROW_PROLOGUE
    const double s =
        warp_row_sum(A, i, [&](int32_t j) { return 0.0 + __ldg(&wd[j]) * __ldg(&b[j]); }, buf, lane);
    if (lane == 0) {
        x[i] = 0.0 + wd[i] * b[i];
        r[i] = b[i] - s;
    }
}

__global__ void __launch_bounds__(kWarpRowsPerBlock * 32)
    k_wjacobi(SellView A, const double* __restrict__ wd, const double* __restrict__ b,
              const double* __restrict__ xin, double* __restrict__ xout) {
    AMGCU_WARP_ROW_PROLOGUE
    const double s = warp_row_sum(A, i, [&](int32_t j) { return __ldg(&xin[j]); }, buf, lane);
    if (lane == 0) xout[i] = xin[i] + wd[i] * (b[i] - s);
}

__global__ void __launch_bounds__(kWarpRowsPerBlock * 32)
    k_wprolong(SellView A, const double* __restrict__ xc, const double* __restrict__ x, double* __restrict__ t) {
    AMGCU_WARP_ROW_PROLOGUE
    const double s = warp_row_sum(A, i, [&](int32_t j) { return __ldg(&xc[j]); }, buf, lane);
    if (lane == 0) t[i] = x[i] + s;
}
#undef AMGCU_WARP_ROW_PROLOGUE

// ---- fused coarse V-cycle -----------------------------------------------------------
// Levels f .. L-1 of a Jacobi V(1,1) cycle in ONE cooperative launch: every phase
// (pre-relax+residual, restriction, coarse GEMV, prolongation, post-relax) is the
// per-row code of the standalone kernels above, distributed grid-stride over the
// resident grid, with one grid barrier between phases.  Results are therefore
// bit-identical to the launch-per-kernel cycle; what disappears is ~4 launches per
// coarse level whose cost there is launch and dependent-load latency.
struct FusedLevel {
    SellView A, R, P;     // R, P unused on the coarsest level
    int wA, wR, wP;       // warp-per-row flags
    const double* wd_pre;
    const double* wd_post;
    double* b;
    double* x;
    double* r;
    double* t;
    int32_t n;
};

constexpr int kFusedThreads = 256;
constexpr int32_t kFusedMaxRows = 65536;  // the fused cycle starts at the first level this small ...
// ... whose operator also has at most this many entries: the cooperative grid runs one row per
// warp at a time (2,368 warps), so a level with more work than that is latency-bound inside it
// (C5 level 2, 39K rows x 69 entries: 42 us per relaxation pass against ~10 us standalone)
constexpr int64_t kFusedMaxNnz = 1500000;
constexpr int kFusedWarps = kFusedThreads / 32;

struct FusedCtx {
    int64_t gtid, gthreads, gwarp, gwarps;
    int lane;
    double* buf;  // this warp's product staging (warp-per-row phases)
};

// y_i = epi(i, sum) over the rows of S, thread-per-row (SELL) or warp-per-row (CSR)
template <typename Gather, typename Epi>
__device__ __forceinline__ void fused_rows(const SellView& S, bool warp_rows, const FusedCtx& f, Gather gx, Epi epi) {
    // fewer rows than warps in the grid: a warp per row spreads them over every SM
    if (warp_rows || S.nr <= f.gwarps) {
        for (int64_t i = f.gwarp; i < S.nr; i += f.gwarps) {
            const double sum = warp_row_sum(S, static_cast<int32_t>(i), gx, f.buf, f.lane);
            if (f.lane == 0) epi(static_cast<int32_t>(i), sum);
        }
    } else {
        for (int64_t i = f.gtid; i < S.nr; i += f.gthreads) {
            const int32_t ii = static_cast<int32_t>(i);
            const int32_t sl = ii / kSlice, ln = ii % kSlice;
            epi(ii, sell_row_sum(S.sptr[sl] + ln, S.slen[sl], S.ci, S.va, gx));
        }
    }
}

__global__ void __launch_bounds__(kFusedThreads)
    k_vcycle_fused(const FusedLevel* __restrict__ lv, int nlev, const double* __restrict__ pinv, int32_t coarse_n,
                   unsigned long long* __restrict__ stamps) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    int ns_ = 0;
    auto stamp = [&]() {
        if (stamps && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            stamps[ns_] = t;
        }
        ++ns_;
    };
    stamp();
    __shared__ double wbuf[kFusedWarps][kWarpCap];
    FusedCtx f;
    f.gtid = static_cast<int64_t>(blockIdx.x) * kFusedThreads + threadIdx.x;
    f.gthreads = static_cast<int64_t>(gridDim.x) * kFusedThreads;
    f.gwarp = f.gtid / 32;
    f.gwarps = f.gthreads / 32;
    f.lane = threadIdx.x & 31;
    f.buf = wbuf[threadIdx.x / 32];
    // down: pre-relax from zero + residual, then restriction
    for (int l = 0; l + 1 < nlev; ++l) {
        const FusedLevel& L = lv[l];
        const double* wd = L.wd_pre;
        const double* b = L.b;
        // b (and every level vector) is written inside this launch: coherent loads only
        fused_rows(L.A, L.wA != 0, f, [&](int32_t j) { return 0.0 + __ldg(&wd[j]) * __ldcg(&b[j]); },
                   [&](int32_t i, double s) {
                       L.x[i] = 0.0 + wd[i] * b[i];
                       L.r[i] = b[i] - s;
                   });
        grid.sync();
        stamp();
        const double* r = L.r;
        double* bn = lv[l + 1].b;
        fused_rows(L.R, L.wR != 0, f, [&](int32_t j) { return __ldcg(&r[j]); },
                   [&](int32_t i, double s) { bn[i] = s; });
        grid.sync();
        stamp();
    }
    // coarsest: x = pinv b (k_dense_gemv / k_dense_gemv_warp arithmetic)
    {
        const FusedLevel& L = lv[nlev - 1];
        if (coarse_n <= 256) {
            for (int64_t i = f.gtid; i < coarse_n; i += f.gthreads) {
                double s = 0.0;
                for (int32_t j = 0; j < coarse_n; ++j) s += pinv[i * coarse_n + j] * __ldcg(&L.b[j]);
                L.x[i] = s;
            }
        } else {
            for (int64_t i = f.gwarp; i < coarse_n; i += f.gwarps) {
                const double* row = pinv + i * coarse_n;
                double s = 0.0;
                for (int32_t j = f.lane; j < coarse_n; j += 32) s += row[j] * __ldcg(&L.b[j]);
                for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (f.lane == 0) L.x[i] = s;
            }
        }
        grid.sync();
        stamp();
    }
    // up: interpolate and correct into t, post-relax back into x
    for (int l = nlev - 2; l >= 0; --l) {
        const FusedLevel& L = lv[l];
        const double* xc = lv[l + 1].x;
        const double* x = L.x;
        double* t = L.t;
        fused_rows(L.P, L.wP != 0, f, [&](int32_t j) { return __ldcg(&xc[j]); },
                   [&](int32_t i, double s) { t[i] = x[i] + s; });
        grid.sync();
        stamp();
        const double* wd = L.wd_post;
        const double* b = L.b;
        double* xo = L.x;
        fused_rows(L.A, L.wA != 0, f, [&](int32_t j) { return __ldcg(&t[j]); },
                   [&](int32_t i, double s) { xo[i] = t[i] + wd[i] * (b[i] - s); });
        if (l > 0) grid.sync();
        stamp();
    }
}

__global__ void k_sell_spmv(SellView A, const double* __restrict__ x, double* __restrict__ y) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.nr) return;
    y[i] = sell_row(i, A.sptr, A.slen, A.ci, A.va, x);
}

// r = b - A x
__global__ void k_sell_residual(SellView A, const double* __restrict__ x, const double* __restrict__ b,
                                double* __restrict__ r) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.nr) return;
    const double s = sell_row(i, A.sptr, A.slen, A.ci, A.va, x);
    r[i] = b[i] - s;
}

// pre-relaxation from zero fused with the residual: x = 0 + wd b, r = b - A x
__global__ void k_relax0_residual(SellView A, const double* __restrict__ wd, const double* __restrict__ b,
                                  double* __restrict__ x, double* __restrict__ r) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.nr) return;
    const int32_t s = i / kSlice, lane = i % kSlice;
    const double acc = sell_row_sum(A.sptr[s] + lane, A.slen[s], A.ci, A.va,
                                    [&](int32_t j) { return 0.0 + __ldg(&wd[j]) * __ldg(&b[j]); });
    x[i] = 0.0 + wd[i] * b[i];
    r[i] = b[i] - acc;
}

// x = 0 + wd b (pre-relaxation from zero without the fused residual)
__global__ void k_relax0(int32_t n, const double* __restrict__ wd, const double* __restrict__ b, double* __restrict__ x) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = 0.0 + wd[i] * b[i];
}

// xout = xin + wd (b - A xin)
__global__ void k_jacobi_sweep(SellView A, const double* __restrict__ wd, const double* __restrict__ b,
                               const double* __restrict__ xin, double* __restrict__ xout) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.nr) return;
    const double s = sell_row(i, A.sptr, A.slen, A.ci, A.va, xin);
    xout[i] = xin[i] + wd[i] * (b[i] - s);
}

// t = x + P xc
__global__ void k_prolong(SellView P, const double* __restrict__ xc, const double* __restrict__ x,
                          double* __restrict__ t) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.nr) return;
    const double s = sell_row(i, P.sptr, P.slen, P.ci, P.va, xc);
    t[i] = x[i] + s;
}

// coarsest level: x = pinv b
__global__ void k_dense_gemv(int32_t n, const double* __restrict__ M, const double* __restrict__ b,
                             double* __restrict__ x) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int32_t j = 0; j < n; ++j) s += M[static_cast<size_t>(i) * n + j] * b[j];
    x[i] = s;
}

// large coarsest level: one warp per row, coalesced row reads, warp-tree sum
// (the coarsest solve is a tolerance-level step either way)
__global__ void k_dense_gemv_warp(int32_t n, const double* __restrict__ M, const double* __restrict__ b,
                                  double* __restrict__ x) {
    const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const double* row = M + static_cast<size_t>(i) * n;
    double s = 0.0;
    for (int32_t j = lane; j < n; j += 32) s += row[j] * b[j];
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) x[i] = s;
}

// PCG control: st = {rz, pq, alpha, rz_new, beta, rn}; flag: !(pq > 0)
__global__ void k_pcg_alpha(double* __restrict__ st, int32_t* __restrict__ bad) {
    const double pq = st[1];
    if (!(pq > 0.0)) {
        *bad = 1;
        return;
    }
    *bad = 0;
    st[2] = st[0] / pq;
}

__global__ void k_pcg_update(int64_t n, const double* __restrict__ st, const int32_t* __restrict__ bad,
                             const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ x,
                             double* __restrict__ r) {
    if (*bad) return;
    const double a = st[2];
    const double na = -a;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        x[i] += a * p[i];
        r[i] += na * q[i];
    }
}

__global__ void k_pcg_beta(double* __restrict__ st) {
    st[4] = st[3] / st[0];
    st[0] = st[3];
}

__global__ void k_pcg_dir(int64_t n, const double* __restrict__ st, const double* __restrict__ z, double* __restrict__ p) {
    const double beta = st[4];
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

__global__ void k_axpy_c(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[i] += a * x[i];
}

// SELL mirror in two halves so that several operators share one synchronisation:
// begin() sizes the slices and stages the stored-entry total in pinned slot `slot`,
// finish() (after a sync) allocates and fills.
void build_sell_begin(Ctx& c, const DCsr& A, DSell& S, int slot) {
    S.nr = A.nr;
    S.nc = A.nc;
    S.nslices = (A.nr + kSlice - 1) / kSlice;
    DBuf<int64_t> slen(static_cast<size_t>(S.nslices) + 1, c.s);
    S.slice_ptr.alloc(static_cast<size_t>(S.nslices) + 1, c.s);
    launch(c, k_slice_len, blocks_for(S.nslices, 256), 256, 0, A.nr, A.rp.get(), slen.get());
    exclusive_scan_i64(c, slen.get(), S.slice_ptr.get(), S.nslices, false);
    stage_scalar(c, slot, static_cast<const int64_t*>(S.slice_ptr.get() + S.nslices));
}

void build_sell_finish(Ctx& c, const DCsr& A, DSell& S, int slot) {
    S.stored = S.nslices > 0 ? staged<int64_t>(c, slot) : 0;
    S.slice_len.alloc(static_cast<size_t>(S.nslices), c.s);
    S.ci.alloc(static_cast<size_t>(S.stored), c.s);
    S.va.alloc(static_cast<size_t>(S.stored), c.s);
    launch(c, k_sell_fill, blocks_for(static_cast<int64_t>(S.nslices) * kSlice, 256), 256, 0, A.nr, A.rp.get(),
           A.ci.get(), A.va.get(), static_cast<const int64_t*>(S.slice_ptr.get()), S.ci.get(), S.va.get(),
           S.slice_len.get());
    // long rows on average and too few rows to fill the GPU thread per row: the
    // warp-per-row kernels over the CSR (with enough rows, thread per row over the SELL
    // slices keeps 16 loads in flight per thread and no lane waits on a serial sum)
    S.crp = A.rp.get();
    S.cci = A.ci.get();
    S.cva = A.va.get();
    static const int64_t max_rows = [] {
        const char* e = std::getenv("AMGCU_WARP_ROW_MAX");
        return e ? std::atoll(e) : static_cast<int64_t>(kWarpRowMaxRows);
    }();
    S.warp_rows = A.nr > 0 && A.nnz >= kWarpRowThreshold * static_cast<int64_t>(A.nr) && A.nr < max_rows;
}

unsigned rows_grid(int32_t n) { return blocks_for(n, 128); }
unsigned warp_rows_grid(int32_t n) { return blocks_for(n, kWarpRowsPerBlock); }
unsigned stream_grid(Ctx& c, int64_t n) { return std::max(1u, std::min<unsigned>(blocks_for(n, 256), 8u * c.sms)); }

double relax_cost(int scheme, double nnz) { return scheme == 3 ? 2.0 * nnz : nnz; }

// AMGCU_FUSED_CYCLE=0 disables the fused coarse cycle (launch-per-kernel reference path)
bool fused_enabled() {
    const char* e = std::getenv("AMGCU_FUSED_CYCLE");
    return !(e && e[0] == '0');
}

struct Driver {
    DHier& h;
    Ctx& c;
    double ops = 0.0;  // multiply-model count (cycle.hpp cost model)
    // fused coarse cycle: level descriptors (host copy + device array), built on first use
    std::vector<FusedLevel> fused_host;
    DBuf<FusedLevel> fused_desc;
    DBuf<unsigned long long> fused_stamps;
    size_t fused_first = 0;

    // xout = xin + wd (b - A xin); family < 0: untagged
    void jacobi_sweep(const DSell& S, int family, double bytes, const double* wd, const double* b, const double* xin,
                      double* xout) {
        const int fam = family < 0 ? static_cast<int>(kProfOther) : family;
        if (S.warp_rows)
            launch_prof(c, fam, bytes, k_wjacobi, warp_rows_grid(S.nr), kWarpRowsPerBlock * 32, 0, view(S), wd, b,
                        xin, xout);
        else
            launch_prof(c, fam, bytes, k_jacobi_sweep, rows_grid(S.nr), 128, 0, view(S), wd, b, xin, xout);
    }

    // y = S x under a profile family
    void spmv_fam(const DSell& S, int family, double bytes, const double* x, double* y) {
        if (S.warp_rows)
            launch_prof(c, family, bytes, k_wspmv, warp_rows_grid(S.nr), kWarpRowsPerBlock * 32, 0, view(S), x, y);
        else
            launch_prof(c, family, bytes, k_sell_spmv, rows_grid(S.nr), 128, 0, view(S), x, y);
    }

    // Fused coarse cycle from level `l` (x_zero, V-cycle, Jacobi V(1,1)): one cooperative
    // launch; returns false when the configuration is not covered.
    bool apply_fused(size_t l, double* x, const double* b) {
        const size_t L = h.lv.size();
        // levels large enough to fill the GPU keep the full-occupancy standalone kernels
        // AMGCU_FUSED_MAX_ROWS overrides the size below which the fused cycle takes over
        static const int32_t max_rows = std::getenv("AMGCU_FUSED_MAX_ROWS")
                                            ? std::atoi(std::getenv("AMGCU_FUSED_MAX_ROWS"))
                                            : kFusedMaxRows;
        static const int64_t max_nnz = std::getenv("AMGCU_FUSED_MAX_NNZ") ? std::atoll(std::getenv("AMGCU_FUSED_MAX_NNZ"))
                                                                            : kFusedMaxNnz;
        if (!fused_enabled() || l == 0 || l + 1 >= L || h.lv[l].A.nr > max_rows || h.lv[l].A.nnz > max_nnz) return false;
        if (h.o.pre_scheme != 0 || h.o.post_scheme != 0 || h.o.pre_sweeps != 1 || h.o.post_sweeps != 1) return false;
        const int nlev = static_cast<int>(L - l);
        // the caller passes level l's own b / x (apply from level l - 1), so the
        // descriptors are constant and uploaded once
        if (b != h.lv[l].b.get() || x != h.lv[l].x.get()) return false;
        if (fused_desc.empty() || fused_first != l) {
            std::vector<FusedLevel> hd(nlev);
            for (int q = 0; q < nlev; ++q) {
                DLevel& lev = h.lv[l + q];
                FusedLevel& d = hd[q];
                d = FusedLevel{};
                d.A = view(lev.sA);
                d.wA = lev.sA.warp_rows;
                if (l + q + 1 < L) {
                    d.R = view(lev.sR);
                    d.P = view(lev.sP);
                    d.wR = lev.sR.warp_rows;
                    d.wP = lev.sP.warp_rows;
                }
                d.wd_pre = lev.wd_pre.get();
                d.wd_post = lev.wd_post.get();
                d.b = lev.b.get();
                d.x = lev.x.get();
                d.r = lev.r.get();
                d.t = lev.t.get();
                d.n = lev.A.nr;
            }
            fused_host = hd;
            fused_desc.alloc(hd.size(), c.s);
            AMG_CK(cudaMemcpyAsync(fused_desc.get(), fused_host.data(), sizeof(FusedLevel) * nlev,
                                   cudaMemcpyHostToDevice, c.s));
            sync(c);  // fused_host may be rebuilt while the copy is pending otherwise
            fused_first = l;
        }
        static int per_sm = -1;
        if (per_sm < 0)
            AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vcycle_fused, kFusedThreads, 0));
        int64_t most = 0;
        double bytes = 0.0;
        for (int q = 0; q < nlev; ++q) {
            const DLevel& lev = h.lv[l + q];
            most = std::max<int64_t>(most, lev.A.nr);
            if (l + q + 1 < L) {
                const double nnz = static_cast<double>(lev.A.nnz), n = lev.A.nr;
                bytes += 2.0 * (12.0 * nnz + 4.0 * (n + 1) + 32.0 * n) + 12.0 * lev.R.nnz + 12.0 * lev.P.nnz + 40.0 * n;
                ops += relax_cost(0, nnz) + nnz + static_cast<double>(lev.R.nnz) + static_cast<double>(lev.P.nnz) +
                       relax_cost(0, nnz);
            }
        }
        bytes += 8.0 * h.coarse_n * h.coarse_n;
        // the whole co-resident grid: small levels run warp-per-row over every SM
        (void)most;
        // AMGCU_FUSED_GRID overrides the grid (barrier cost grows with the block count)
        static const int g_env = std::getenv("AMGCU_FUSED_GRID") ? std::atoi(std::getenv("AMGCU_FUSED_GRID")) : 0;
        const int g = g_env > 0 ? std::min(g_env, std::max(1, per_sm * c.sms)) : std::max(1, per_sm * c.sms);
        const FusedLevel* dp = fused_desc.get();
        const double* pv = h.coarse_pinv.get();
        int32_t cn = h.coarse_n;
        // AMGCU_FUSED_TRACE=1: phase boundary stamps of block 0, printed per call
        static const bool trace = std::getenv("AMGCU_FUSED_TRACE") != nullptr;
        unsigned long long* st = nullptr;
        if (trace) {
            if (fused_stamps.empty()) fused_stamps.alloc(64, c.s);
            st = fused_stamps.get();
        }
        void* args[] = {&dp, const_cast<int*>(&nlev), &pv, &cn, &st};
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        const bool prof = c.profile && ((c.prof_mask >> kProfVcycleCoarseFused) & 1u);
        if (prof) {
            e0 = prof_event(c);
            e1 = prof_event(c);
            AMG_CK(cudaEventRecord(e0, c.s));
        }
        AMG_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_vcycle_fused), dim3(g), dim3(kFusedThreads),
                                           args, 0, c.s));
        ++c.launches;
        if (prof) {
            AMG_CK(cudaEventRecord(e1, c.s));
            ProfRecord& rec = c.prof[kProfVcycleCoarseFused];
            rec.launches += 1;
            rec.bytes += bytes;
            rec.pending.emplace_back(e0, e1);
        }
        if (trace) {
            unsigned long long hs[64];
            AMG_CK(cudaMemcpyAsync(hs, st, sizeof(hs), cudaMemcpyDeviceToHost, c.s));
            sync(c);
            const int nst = 4 * (nlev - 1) + 2;
            std::fprintf(stderr, "fused g=%d:", g);
            for (int q = 1; q < nst; ++q) std::fprintf(stderr, " %.1f", (hs[q] - hs[q - 1]) * 1e-3);
            std::fprintf(stderr, " us\n");
        }
        return true;
    }

    // one cycle at `l`; x_zero: x is known to be all zeros on entry
    void apply(size_t l, double* x, const double* b, int kind, bool x_zero) {
        if (kind == 0 && x_zero && apply_fused(l, x, b)) return;
        const size_t L = h.lv.size();
        DLevel& lev = h.lv[l];
        if (l == L - 1) {
            const double cb = 8.0 * h.coarse_n * h.coarse_n + 16.0 * h.coarse_n;
            if (h.coarse_n <= 256)
                launch_prof(c, kProfCoarseSolve, cb, k_dense_gemv, blocks_for(h.coarse_n, 128), 128, 0, h.coarse_n,
                       static_cast<const double*>(h.coarse_pinv.get()), b, x);
            else
                launch_prof(c, kProfCoarseSolve, cb, k_dense_gemv_warp, blocks_for(static_cast<int64_t>(h.coarse_n) * 32, 256), 256, 0,
                       h.coarse_n, static_cast<const double*>(h.coarse_pinv.get()), b, x);
            return;
        }
        const int32_t n = lev.A.nr;
        const double nnz = static_cast<double>(lev.A.nnz);
        const SellView A = view(lev.sA);
        // pre-relaxation + residual
        const int pre = h.o.pre_scheme;
        int sweeps = h.o.pre_sweeps;
        bool residual_done = false;
        if (pre == 0) {
            for (int s = 0; s < sweeps; ++s) {
                if (s == 0 && x_zero) {
                    if (sweeps == 1) {
                        if (lev.sA.warp_rows)
                            launch_prof(c, kProfVcycleRelax0Residual, 12.0 * nnz + 4.0 * (n + 1) + 32.0 * n,
                                        k_wrelax0_residual, warp_rows_grid(n), kWarpRowsPerBlock * 32, 0, A,
                                        static_cast<const double*>(lev.wd_pre.get()), b, x, lev.r.get());
                        else
                            launch_prof(c, kProfVcycleRelax0Residual, 12.0 * nnz + 4.0 * (n + 1) + 32.0 * n,
                                        k_relax0_residual, rows_grid(n), 128, 0, A,
                                        static_cast<const double*>(lev.wd_pre.get()), b, x, lev.r.get());
                        residual_done = true;
                    } else {
                        launch(c, k_relax0, rows_grid(n), 128, 0, n, static_cast<const double*>(lev.wd_pre.get()), b, x);
                    }
                } else {
                    jacobi_sweep(lev.sA, -1, 0.0, static_cast<const double*>(lev.wd_pre.get()), b,
                                 static_cast<const double*>(x), lev.t.get());
                    copy_d2d(c, x, lev.t.get(), n);
                }
                ops += relax_cost(pre, nnz);
            }
        } else {
            if (x_zero) AMG_CK(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
            if (sweeps > 0) relax_other(lev, pre, x, b, sweeps);
            ops += sweeps * relax_cost(pre, nnz);
        }
        if (pre != 0 && x_zero && sweeps == 0) {
            // x stays zero
        }
        if (!residual_done) {
            if (pre == 0 && sweeps == 0 && x_zero) AMG_CK(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
            if (lev.sA.warp_rows)
                launch(c, k_wresidual, warp_rows_grid(n), kWarpRowsPerBlock * 32, 0, A, static_cast<const double*>(x), b,
                       lev.r.get());
            else
                launch(c, k_sell_residual, rows_grid(n), 128, 0, A, static_cast<const double*>(x), b, lev.r.get());
        }
        ops += nnz;
        // restriction
        DLevel& nxt = h.lv[l + 1];
        spmv_fam(lev.sR, kProfVcycleRestrict, 12.0 * lev.R.nnz + 4.0 * (lev.R.nr + 1) + 8.0 * n + 8.0 * lev.R.nr,
                 static_cast<const double*>(lev.r.get()), nxt.b.get());
        ops += static_cast<double>(lev.R.nnz);
        apply(l + 1, nxt.x.get(), nxt.b.get(), kind, true);
        if (kind == 1 && l + 1 < L - 1) apply(l + 1, nxt.x.get(), nxt.b.get(), kind, false);
        // interpolate and correct into t, then post-relax back into x
        {
            const double pb = 12.0 * lev.P.nnz + 4.0 * (n + 1) + 8.0 * lev.P.nc + 16.0 * n;
            if (lev.sP.warp_rows)
                launch_prof(c, kProfVcycleProlong, pb, k_wprolong, warp_rows_grid(n), kWarpRowsPerBlock * 32, 0,
                            view(lev.sP), static_cast<const double*>(nxt.x.get()), static_cast<const double*>(x),
                            lev.t.get());
            else
                launch_prof(c, kProfVcycleProlong, pb, k_prolong, rows_grid(n), 128, 0, view(lev.sP),
                            static_cast<const double*>(nxt.x.get()), static_cast<const double*>(x), lev.t.get());
        }
        ops += static_cast<double>(lev.P.nnz);
        const int post = h.o.post_scheme;
        sweeps = h.o.post_sweeps;
        if (post == 0) {
            if (sweeps == 0) {
                copy_d2d(c, x, lev.t.get(), n);
            } else {
                for (int s = 0; s < sweeps; ++s) {
                    if (s == 0) {
                        jacobi_sweep(lev.sA, kProfVcyclePostRelax, 12.0 * nnz + 4.0 * (n + 1) + 32.0 * n,
                                     static_cast<const double*>(lev.wd_post.get()), b,
                                     static_cast<const double*>(lev.t.get()), x);
                    } else {
                        jacobi_sweep(lev.sA, -1, 0.0, static_cast<const double*>(lev.wd_post.get()), b,
                                     static_cast<const double*>(x), lev.t.get());
                        copy_d2d(c, x, lev.t.get(), n);
                    }
                    ops += relax_cost(post, nnz);
                }
            }
        } else {
            copy_d2d(c, x, lev.t.get(), n);
            if (sweeps > 0) relax_other(lev, post, x, b, sweeps);
            ops += sweeps * relax_cost(post, nnz);
        }
    }

    void precond(const double* rhs, double* out, int kind) { apply(0, out, rhs, kind, true); }

    // the sequential schemes: (symmetric) Gauss-Seidel, gsne, block symmetric GS
    void relax_other(DLevel& lev, int scheme, double* x, const double* b, int sweeps) {
        if (scheme == 3) gsne(c, lev.A, lev.gsne_ws, x, b, sweeps);
        else if (scheme == 4) block_sym_gs(c, lev.A, lev.block_inv.get(), x, b, sweeps);
        else gauss_seidel(c, lev.A, lev.inv_diag.get(), x, b, 1, sweeps, scheme == 2);
    }
};

double conv_factor(const std::vector<double>& hist, int window = 5) {  // cycle.hpp:39-46
    if (hist.size() < 2) return 0.0;
    const int w = std::min<int>(window, static_cast<int>(hist.size()) - 1);
    const double head = hist[hist.size() - 1 - w];
    const double tail = hist.back();
    if (head <= 0.0) return 0.0;
    return std::pow(tail / head, 1.0 / w);
}

}  // namespace

void prepare_solve(DHier& h) {
    Ctx& c = *h.ctx;
    for (size_t l = 0; l < h.lv.size(); ++l) {
        DLevel& L = h.lv[l];
        const int32_t n = L.A.nr;
        L.r.alloc(static_cast<size_t>(n), c.s);
        L.t.alloc(static_cast<size_t>(n), c.s);
        if (l > 0) {
            L.b.alloc(static_cast<size_t>(n), c.s);
            L.x.alloc(static_cast<size_t>(n), c.s);
        }
    }
    // all SELL mirrors: sizes first, one synchronisation, then the fills
    std::vector<std::pair<const DCsr*, DSell*>> ops;
    for (size_t l = 0; l < h.lv.size(); ++l) {
        DLevel& L = h.lv[l];
        ops.emplace_back(&L.A, &L.sA);
        if (l + 1 < h.lv.size()) {
            ops.emplace_back(&L.P, &L.sP);
            ops.emplace_back(&L.R, &L.sR);
        }
    }
    if (ops.size() > static_cast<size_t>(Ctx::kPinSlots)) throw std::logic_error("prepare_solve: too many levels");
    for (size_t k = 0; k < ops.size(); ++k) build_sell_begin(c, *ops[k].first, *ops[k].second, static_cast<int>(k));
    sync(c);
    for (size_t k = 0; k < ops.size(); ++k) build_sell_finish(c, *ops[k].first, *ops[k].second, static_cast<int>(k));
    sync(c);
    h.solve_ready = true;
}

double operator_complexity(const DHier& h) {  // complexity.hpp:15-20
    const double base = static_cast<double>(h.lv.front().A.nnz);
    double s = 0.0;
    for (const DLevel& l : h.lv) s += static_cast<double>(l.A.nnz);
    return s / base;
}

double cycle_complexity(const DHier& h) {  // complexity.hpp:25-36
    const double base = static_cast<double>(h.lv.front().A.nnz);
    double s = 0.0;
    for (size_t l = 0; l + 1 < h.lv.size(); ++l) {
        s += static_cast<double>(h.o.pre_sweeps + h.o.post_sweeps + 1) * h.lv[l].A.nnz;
        s += static_cast<double>(h.lv[l].P.nnz) + static_cast<double>(h.lv[l].R.nnz);
    }
    return s / base;
}

void cycle(DHier& h, double* x, const double* b, int kind) {
    Driver d{h, *h.ctx};
    d.apply(0, x, b, kind, false);
    sync(*h.ctx);
}

SolveResult solve(DHier& h, const double* b, double* x, const amgcu_solve_options& o) {
    Ctx& c = *h.ctx;
    if (o.max_iters < 1) throw InvalidArgument("solve: max_iters must be >= 1");
    DLevel& L0 = h.lv.front();
    const int32_t n = L0.A.nr;
    const SellView A = view(L0.sA);
    SolveResult rep;
    rep.chi_oc = operator_complexity(h);
    rep.chi_cc = cycle_complexity(h);
    {
        double wu[5];  // work.hpp:59 setup_total, cycle.hpp:126
        hier_ledger(h, wu);
        rep.wu_setup = wu[0] + wu[1] + wu[2] + wu[3];
    }
    Driver d{h, c};
    auto finish = [&]() {
        rep.rho = conv_factor(rep.history);
        rep.wu_solve = d.ops / h.base_nnz;
        h.wu[4] += d.ops / h.base_nnz;
        return rep;
    };
    static const bool ht = std::getenv("AMGCU_HOST_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    DBuf<double> r(static_cast<size_t>(n), c.s), st(16, c.s);
    DBuf<int32_t> bad(1, c.s);
    if (ht)
        std::fprintf(stderr, "[host] solve preamble (complexities, ledger, buffers) %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    launch(c, k_sell_residual, rows_grid(n), 128, 0, A, static_cast<const double*>(x), b, r.get());
    d.ops += static_cast<double>(L0.A.nnz);
    double* S = st.get();
    nrm2(c, r.get(), n, S + 10);  // r0
    nrm2(c, b, n, S + 11);        // |b|
    double h2[2];
    copy_d2h(c, h2, S + 10, 2);
    sync(c);
    const double r0 = h2[0], bnorm = h2[1];
    const double target = o.tol * (bnorm > 0.0 ? bnorm : r0);
    rep.history.push_back(r0);
    if (r0 <= target) {
        rep.converged = true;
        return finish();
    }
    const double blowup = 1e6 * r0;

    if (o.method == 0) {  // stationary cycling
        for (int it = 1; it <= o.max_iters; ++it) {
            d.apply(0, x, b, o.cycle, false);
            launch(c, k_sell_residual, rows_grid(n), 128, 0, A, static_cast<const double*>(x), b, r.get());
            nrm2(c, r.get(), n, S + 5);
            const double rn = read_scalar(c, S + 5);
            rep.history.push_back(rn);
            rep.iterations = it;
            if (rn <= target) {
                rep.converged = true;
                break;
            }
            if (rn > blowup || !std::isfinite(rn)) {
                rep.diverged = true;
                break;
            }
        }
        return finish();
    }

    static const bool pcg_spec = [] {
        const char* e = std::getenv("AMGCU_PCG_SPEC");
        return !(e && e[0] == '0');
    }();
    if (o.method == 1 && pcg_spec && c.side && c.seq) {  // PCG (cycle.hpp:174-209), pipelined
        // The residual norm only decides whether to stop; nothing else waits for it.  So
        // after the update it is summed on the side stream while the main stream goes on
        // with the next iteration's work up to (not including) its update: the cycle
        // M r, (r, z), beta, p = z + beta p, q = A p, (p, q), alpha.  The host then reads
        // the norm; if the reference stops there, x and r are final (the queued work only
        // touched z, p, q and the scalars) and its work units are not counted.  Every
        // value is computed by the same kernels in the same order as the plain loop.
        if (!L0.symmetric) throw InvalidArgument("solve: pcg requires a symmetric operator");
        DBuf<double> z(static_cast<size_t>(n), c.s), p(static_cast<size_t>(n), c.s), q(static_cast<size_t>(n), c.s);
        double* hs = nullptr;  // pinned: {rn, bad}
        AMG_CK(cudaMallocHost(reinterpret_cast<void**>(&hs), 2 * sizeof(double)));
        struct PinGuard {
            double* p;
            ~PinGuard() { cudaFreeHost(p); }
        } pin_guard{hs};
        cudaEvent_t upd, nrm;
        AMG_CK(cudaEventCreateWithFlags(&upd, cudaEventDisableTiming));
        AMG_CK(cudaEventCreateWithFlags(&nrm, cudaEventDisableTiming));
        struct EvGuard {
            cudaEvent_t a, b;
            cudaStream_t side;
            ~EvGuard() {
                cudaStreamSynchronize(side);  // the side stream's norm reads r and writes hs
                cudaEventDestroy(a);
                cudaEventDestroy(b);
            }
        } ev_guard{upd, nrm, c.side};
        auto head = [&] {  // q = A p, (p, q), alpha
            d.spmv_fam(L0.sA, kProfKrylovSpmv, 12.0 * L0.A.nnz + 4.0 * (n + 1) + 16.0 * n,
                       static_cast<const double*>(p.get()), q.get());
            d.ops += static_cast<double>(L0.A.nnz);
            dot(c, p.get(), q.get(), n, S + 1);
            launch(c, k_pcg_alpha, 1, 1, 0, S, bad.get());
        };
        d.precond(r.get(), z.get(), o.cycle);
        copy_d2d(c, p.get(), z.get(), n);
        dot(c, r.get(), z.get(), n, S + 0);  // rz
        head();
        for (int it = 1; it <= o.max_iters; ++it) {
            launch_prof(c, kProfBlas1, 48.0 * n, k_pcg_update, stream_grid(c, n), 256, 0, static_cast<int64_t>(n),
                        static_cast<const double*>(S), static_cast<const int32_t*>(bad.get()),
                        static_cast<const double*>(p.get()), static_cast<const double*>(q.get()), x, r.get());
            // this iteration's breakdown flag, before the next alpha overwrites it
            AMG_CK(cudaMemcpyAsync(hs + 1, bad.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
            AMG_CK(cudaEventRecord(upd, c.s));
            {
                StreamScope on_side(c, c.side);
                AMG_CK(cudaStreamWaitEvent(c.side, upd, 0));
                nrm2(c, r.get(), n, S + 5);
                copy_d2h(c, hs, S + 5, 1);
                AMG_CK(cudaEventRecord(nrm, c.side));
            }
            const double ops_before = d.ops;
            if (it < o.max_iters) {
                d.precond(r.get(), z.get(), o.cycle);
                dot(c, r.get(), z.get(), n, S + 3);
                launch(c, k_pcg_beta, 1, 1, 0, S);
                launch_prof(c, kProfBlas1, 24.0 * n, k_pcg_dir, stream_grid(c, n), 256, 0, static_cast<int64_t>(n),
                            static_cast<const double*>(S), static_cast<const double*>(z.get()), p.get());
                head();
            }
            AMG_CK(cudaEventSynchronize(nrm));
            ++c.syncs;
            int32_t hbad = 0;
            std::memcpy(&hbad, hs + 1, sizeof(int32_t));
            if (hbad) {
                rep.diverged = true;
                d.ops = ops_before;
                break;
            }
            const double rn = hs[0];
            rep.history.push_back(rn);
            rep.iterations = it;
            if (rn <= target) {
                rep.converged = true;
                d.ops = ops_before;
                break;
            }
            if (rn > blowup || !std::isfinite(rn)) {
                rep.diverged = true;
                d.ops = ops_before;
                break;
            }
        }
        sync(c);
        return finish();
    }

    if (o.method == 1) {  // PCG (cycle.hpp:174-209)
        if (!L0.symmetric) throw InvalidArgument("solve: pcg requires a symmetric operator");
        DBuf<double> z(static_cast<size_t>(n), c.s), p(static_cast<size_t>(n), c.s), q(static_cast<size_t>(n), c.s);
        d.precond(r.get(), z.get(), o.cycle);
        copy_d2d(c, p.get(), z.get(), n);
        dot(c, r.get(), z.get(), n, S + 0);  // rz
        for (int it = 1; it <= o.max_iters; ++it) {
            d.spmv_fam(L0.sA, kProfKrylovSpmv, 12.0 * L0.A.nnz + 4.0 * (n + 1) + 16.0 * n,
                       static_cast<const double*>(p.get()), q.get());
            d.ops += static_cast<double>(L0.A.nnz);
            dot(c, p.get(), q.get(), n, S + 1);
            launch(c, k_pcg_alpha, 1, 1, 0, S, bad.get());
            if (!pcg_update_nrm(c, S, bad.get(), p.get(), q.get(), x, r.get(), n, S + 5)) {
                launch_prof(c, kProfBlas1, 48.0 * n, k_pcg_update, stream_grid(c, n), 256, 0, static_cast<int64_t>(n),
                            static_cast<const double*>(S), static_cast<const int32_t*>(bad.get()),
                            static_cast<const double*>(p.get()), static_cast<const double*>(q.get()), x, r.get());
                nrm2(c, r.get(), n, S + 5);
            }
            struct {
                double rn;
                int32_t bad;
            } hs;
            copy_d2h(c, &hs.rn, S + 5, 1);
            copy_d2h(c, &hs.bad, bad.get(), 1);
            sync(c);
            if (hs.bad) {
                rep.diverged = true;
                break;
            }
            const double rn = hs.rn;
            rep.history.push_back(rn);
            rep.iterations = it;
            if (rn <= target) {
                rep.converged = true;
                break;
            }
            if (rn > blowup || !std::isfinite(rn)) {
                rep.diverged = true;
                break;
            }
            d.precond(r.get(), z.get(), o.cycle);
            dot(c, r.get(), z.get(), n, S + 3);
            launch(c, k_pcg_beta, 1, 1, 0, S);
            launch_prof(c, kProfBlas1, 24.0 * n, k_pcg_dir, stream_grid(c, n), 256, 0, static_cast<int64_t>(n), static_cast<const double*>(S),
                   static_cast<const double*>(z.get()), p.get());
        }
        return finish();
    }

    // FGMRES, one cycle of max_iters steps (cycle.hpp:211-270)
    const int m = o.max_iters;
    DBuf<double> V(static_cast<size_t>(n) * (m + 1), c.s), Z(static_cast<size_t>(n) * m, c.s);
    DBuf<double> Hcol(static_cast<size_t>(m) + 2, c.s);
    copy_d2d(c, V.get(), r.get(), n);
    scale_const(c, 1.0 / r0, V.get(), n);
    std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0);
    auto Hij = [&](int i, int j) -> double& { return H[static_cast<size_t>(i) * m + j]; };
    g[0] = r0;
    int built = 0;
    for (int j = 0; j < m; ++j) {
        double* zj = Z.get() + static_cast<size_t>(j) * n;
        double* w = V.get() + static_cast<size_t>(j + 1) * n;
        d.precond(V.get() + static_cast<size_t>(j) * n, zj, o.cycle);
        d.spmv_fam(L0.sA, kProfKrylovSpmv, 12.0 * L0.A.nnz + 4.0 * (n + 1) + 16.0 * n, static_cast<const double*>(zj),
                   w);
        d.ops += static_cast<double>(L0.A.nnz);
        // modified Gram-Schmidt (cycle.hpp:228-231); axpy of step t fused with the dot of t + 1
        dot(c, w, V.get(), n, Hcol.get());
        for (int t = 0; t <= j; ++t)
            axpy_dot(c, Hcol.get() + t, -1.0, V.get() + static_cast<size_t>(t) * n, w,
                     t < j ? V.get() + static_cast<size_t>(t + 1) * n : nullptr, n, Hcol.get() + t + 1, t == j);
        std::vector<double> col(j + 2);
        copy_d2h(c, col.data(), Hcol.get(), j + 2);
        sync(c);
        for (int t = 0; t <= j + 1; ++t) Hij(t, j) = col[t];
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
        rep.history.push_back(res);
        rep.iterations = j + 1;
        built = j + 1;
        if (res <= target) {
            rep.converged = true;
            break;
        }
        if (res > blowup || !std::isfinite(res)) {
            rep.diverged = true;
            break;
        }
        if (hlast < 1e-300) break;
        scale_const(c, 1.0 / hlast, w, n);
    }
    std::vector<double> y(built, 0.0);
    for (int t = built - 1; t >= 0; --t) {
        double s = g[t];
        for (int u = t + 1; u < built; ++u) s -= Hij(t, u) * y[u];
        y[t] = Hij(t, t) != 0.0 ? s / Hij(t, t) : 0.0;
    }
    for (int t = 0; t < built; ++t)
        launch_prof(c, kProfBlas1, 24.0 * n, k_axpy_c, stream_grid(c, n), 256, 0, static_cast<int64_t>(n), y[t],
               static_cast<const double*>(Z.get() + static_cast<size_t>(t) * n), x);
    sync(c);
    return finish();
}

}  // namespace amgcu
