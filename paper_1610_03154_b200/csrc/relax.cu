// Relaxation on the GPU (relaxation.hpp).
//
// Gauss-Seidel (relaxation.hpp:115-127) is inherently ordered: row i uses the
// new values of the rows before it and the old values of the rows after it.
// All sweeps run in ONE sync-free launch of resident warp chains (see
// k_gs_chains); every sweep writes its own copy of x (sweeps + 1 buffers), so
// reads never race with writes and each row sum is evaluated in CSR order
// exactly as on the CPU.  k candidate columns are swept together.
#include <cuda/atomic>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "ops.cuh"

namespace amgcu {

namespace {

constexpr int kMaxK = 8;

// Gauss-Seidel sweeps, segment-parallel.
//
// In sweep order, row q usually depends on row q - 1 (on a stencil grid in
// natural order, every row but the first of a grid row does), so the sweep is
// a set of long chains and the parallelism is ACROSS chains.  A segment is a
// maximal run of rows each depending on its predecessor; one warp relaxes one
// segment, 32 rows at a time:
//   phase A (lanes in parallel): lane l takes row q = block + l, sums the CSR
//     prefix that precedes its first dependency on an earlier row of the same
//     32-row block, and prefetches every other value it needs (polling values
//     produced by other warps -- other segments of this sweep, or the
//     previous sweep);
//   phase B (serial over lanes): lane t finishes its sum in CSR order, taking
//     in-block values from shared memory, then publishes x.
// Every row sum is therefore evaluated in exactly the sequential order, so
// results are bit-identical to the CPU sweep.  Lanes never wait on lanes of
// their own warp.
//
// Publication: each sweep writes its own buffer, pre-filled with a NaN
// payload no arithmetic produces (kPending); a value is published by its one
// 8-byte store and readers poll the value itself (exponential back-off).
// Items (sweep, segment) draw tickets in (sweep, position) order; segments are
// contiguous, so any unfinished row that an item waits on belongs to an item
// with a smaller ticket, which is already running: the launch cannot deadlock.
constexpr int kSegWarps = 4;
constexpr int kSegMaxE = 16;  // entries per row handled from the prefetch cache
constexpr unsigned long long kPending = 0x7FF4A11CE5EEDULL;

__device__ __forceinline__ unsigned long long load_relaxed_bits(const double* p) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(
        *reinterpret_cast<unsigned long long*>(const_cast<double*>(p)));
    return r.load(cuda::memory_order_relaxed);
}

__device__ __forceinline__ double wait_bits(const double* p, unsigned long long bits) {
    unsigned ns = 16;
    while (bits == kPending) {
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;
        bits = load_relaxed_bits(p);
    }
    return __longlong_as_double(static_cast<long long>(bits));
}

// entry classes in sweep order
enum : int { kSelf = 0, kInBlock = 1, kReady = 2, kPoll = 3 };

// Per warp, dynamic shared memory: cache[32][kSegMaxE][K] prefetched bits,
// xb[32][K] values published in the current block.  K = number of candidate
// columns (compile-time so the per-entry arrays stay in registers).
template <int K>
__global__ void __launch_bounds__(kSegWarps * 32)
    k_gs_segments(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  const double* __restrict__ va, const double* __restrict__ inv_diag, const double* __restrict__ b,
                  int nsweeps, const unsigned char* __restrict__ backward, const int32_t* __restrict__ item_base,
                  const int32_t* __restrict__ seg_fwd, const int32_t* __restrict__ seg_bwd, double* __restrict__ X,
                  unsigned int* __restrict__ ticket) {
    extern __shared__ unsigned long long smem[];
    __shared__ unsigned int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const int lane = threadIdx.x & 31, wl = threadIdx.x / 32;
    const int32_t item = static_cast<int32_t>(blk) * kSegWarps + wl;
    if (item >= item_base[nsweeps]) return;
    int s = 0;
    while (item >= item_base[s + 1]) ++s;
    const bool bwd = backward[s] != 0;
    const int32_t* segs = bwd ? seg_bwd : seg_fwd;
    const int32_t g = item - item_base[s];
    const int32_t q0 = segs[g], q1 = segs[g + 1];
    const size_t stride = static_cast<size_t>(n) * K;
    const double* xin = X + static_cast<size_t>(s) * stride;
    double* xout = X + static_cast<size_t>(s + 1) * stride;
    unsigned long long* cache = smem + static_cast<size_t>(wl) * 32 * (kSegMaxE + 1) * K;
    double* xb = reinterpret_cast<double*>(cache + 32 * kSegMaxE * K);
    unsigned long long* mycache = cache + static_cast<size_t>(lane) * kSegMaxE * K;
    for (int32_t qb = q0; qb < q1; qb += 32) {
        const int32_t q = qb + lane;
        const bool active = q < q1;
        const int32_t i = active ? (bwd ? n - 1 - q : q) : 0;
        int32_t lo = 0, hi = 0;
        if (active) {
            lo = rp[i];
            hi = rp[i + 1];
        }
        // ---- phase A: every independent load of the row, issued without waiting ----
        int32_t ref[kSegMaxE];  // in-block: lane index of the producer; otherwise the column
        unsigned char cls[kSegMaxE];
        double a[kSegMaxE];
#pragma unroll
        for (int e = 0; e < kSegMaxE; ++e) {
            cls[e] = kSelf;
            ref[e] = 0;
            a[e] = 0.0;
            if (lo + e < hi) {
                const int32_t j = ci[lo + e];
                a[e] = va[lo + e];
                ref[e] = j;
                if (j != i) {
                    const int32_t qj = bwd ? n - 1 - j : j;
                    const bool fresh = qj < q;
                    if (fresh && qj >= qb) {
                        cls[e] = kInBlock;
                        ref[e] = qj - qb;
                    } else {
                        const bool own = fresh && qj >= q0;  // earlier block of this warp's segment
                        cls[e] = (own || (!fresh && s == 0)) ? kReady : kPoll;
                    }
                }
            }
        }
#pragma unroll
        for (int e = 0; e < kSegMaxE; ++e) {
            if (cls[e] == kReady || cls[e] == kPoll) {
                const int32_t j = ref[e];
                const int32_t qj = bwd ? n - 1 - j : j;
                const double* src = (qj < q) ? xout : xin;
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    const double* addr = &src[static_cast<size_t>(c) * n + j];
                    mycache[e * K + c] = cls[e] == kReady
                                             ? static_cast<unsigned long long>(__double_as_longlong(__ldcg(addr)))
                                             : load_relaxed_bits(addr);
                }
            }
        }
        // CSR prefix that needs neither an in-block value nor a pending one
        double acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = (active && b) ? b[static_cast<size_t>(c) * n + i] : 0.0;
        bool open = active;
        int32_t e_stop = 0;
#pragma unroll
        for (int e = 0; e < kSegMaxE; ++e) {
            if (open && lo + e < hi) {
                if (cls[e] == kInBlock) {
                    open = false;
                } else if (cls[e] != kSelf) {
                    bool pending = false;
#pragma unroll
                    for (int c = 0; c < K; ++c) pending = pending || mycache[e * K + c] == kPending;
                    if (pending) {
                        open = false;
                    } else {
#pragma unroll
                        for (int c = 0; c < K; ++c)
                            acc[c] -= a[e] * __longlong_as_double(static_cast<long long>(mycache[e * K + c]));
                    }
                }
                if (open) e_stop = e + 1;
            }
        }
        __syncwarp();
        // ---- phase B: lanes finish in order; arithmetic on registers, polls only if pending ----
        const int32_t cnt = min(32, q1 - qb);
        for (int32_t t = 0; t < cnt; ++t) {
            if (lane == t) {
#pragma unroll
                for (int e = 0; e < kSegMaxE; ++e) {
                    if (e >= e_stop && lo + e < hi) {
                        if (cls[e] == kInBlock) {
#pragma unroll
                            for (int c = 0; c < K; ++c) acc[c] -= a[e] * xb[ref[e] * K + c];
                        } else if (cls[e] != kSelf) {
                            const int32_t j = ref[e];
                            const int32_t qj = bwd ? n - 1 - j : j;
                            const double* src = (qj < q) ? xout : xin;
#pragma unroll
                            for (int c = 0; c < K; ++c)
                                acc[c] -= a[e] * wait_bits(&src[static_cast<size_t>(c) * n + j], mycache[e * K + c]);
                        }
                    }
                }
                // entries beyond the prefetch window, in CSR order
                for (int32_t p = lo + kSegMaxE; p < hi; ++p) {
                    const int32_t j = ci[p];
                    if (j == i) continue;
                    const int32_t qj = bwd ? n - 1 - j : j;
                    const bool fresh = qj < q;
                    const double av = va[p];
                    if (fresh && qj >= qb) {
#pragma unroll
                        for (int c = 0; c < K; ++c) acc[c] -= av * xb[(qj - qb) * K + c];
                        continue;
                    }
                    const double* src = fresh ? xout : xin;
                    const bool own = fresh && qj >= q0;
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const double* addr = &src[static_cast<size_t>(c) * n + j];
                        const unsigned long long bits =
                            (own || (!fresh && s == 0))
                                ? static_cast<unsigned long long>(__double_as_longlong(__ldcg(addr)))
                                : load_relaxed_bits(addr);
                        acc[c] -= av * wait_bits(addr, bits);
                    }
                }
                const double d = inv_diag[i];
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    const double xi = acc[c] * d;
                    xb[t * K + c] = xi;
                    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> out(
                        *reinterpret_cast<unsigned long long*>(&xout[static_cast<size_t>(c) * n + i]));
                    out.store(static_cast<unsigned long long>(__double_as_longlong(xi)), cuda::memory_order_relaxed);
                }
            }
            __syncwarp();
        }
    }
}

// segment heads in sweep order: position q starts a segment unless row(q)
// holds column row(q - 1)
__global__ void k_segment_heads(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, bool bwd,
                                int32_t* __restrict__ head) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    if (q == 0) {
        head[0] = 1;
        return;
    }
    const int32_t i = bwd ? n - 1 - q : q;
    const int32_t prev = bwd ? i + 1 : i - 1;
    int32_t lo = rp[i], hi = rp[i + 1];
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (ci[mid] < prev) lo = mid + 1;
        else hi = mid;
    }
    head[q] = (lo < rp[i + 1] && ci[lo] == prev) ? 0 : 1;
}

__global__ void k_segment_starts(int32_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ rank,
                                 int32_t* __restrict__ starts, int32_t nseg) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n && head[q]) starts[rank[q]] = q;
    if (q == 0) starts[nseg] = n;
}

__global__ void k_fill_pending(int64_t count, double* __restrict__ p) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < count) reinterpret_cast<unsigned long long*>(p)[t] = kPending;
}

int32_t build_segments(Ctx& c, const DCsr& A, bool bwd, DBuf<int32_t>& starts) {
    const int32_t n = A.nr;
    DBuf<int32_t> head(static_cast<size_t>(n) + 1, c.s), rank(static_cast<size_t>(n) + 1, c.s);
    launch(c, k_segment_heads, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), bwd, head.get());
    const int32_t nseg = static_cast<int32_t>(exclusive_scan_i32(c, head.get(), rank.get(), n));
    starts.alloc(static_cast<size_t>(nseg) + 1, c.s);
    launch(c, k_segment_starts, blocks_for(n, 256), 256, 0, n, static_cast<const int32_t*>(head.get()),
           static_cast<const int32_t*>(rank.get()), starts.get(), nseg);
    return nseg;
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
    launch(c, k_fill_pending, blocks_for(static_cast<int64_t>(stride) * nsw, 256), 256, 0,
           static_cast<int64_t>(stride) * nsw, X.get() + stride);
    DBuf<int32_t> segf, segb;
    const int32_t nf = build_segments(c, A, false, segf);
    const int32_t nb = symmetric_sweep ? build_segments(c, A, true, segb) : 0;
    std::vector<unsigned char> hb(nsw);
    std::vector<int32_t> base(nsw + 1, 0);
    for (int s = 0; s < nsw; ++s) {
        hb[s] = symmetric_sweep ? static_cast<unsigned char>(s & 1) : 0;
        base[s + 1] = base[s] + (hb[s] ? nb : nf);
    }
    DBuf<unsigned char> bwd(static_cast<size_t>(nsw), c.s);
    DBuf<int32_t> dbase(static_cast<size_t>(nsw) + 1, c.s);
    copy_h2d(c, bwd.get(), hb.data(), nsw);
    copy_h2d(c, dbase.get(), base.data(), nsw + 1);
    DBuf<unsigned int> ticket(1, c.s);
    AMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned int), c.s));
    const size_t smem = static_cast<size_t>(kSegWarps) * 32 * (kSegMaxE + 1) * k * sizeof(unsigned long long);
    const double bytes = nsw * (12.0 * A.nnz + 4.0 * (n + 1) + 8.0 * n + 16.0 * n * k);
    auto run = [&](auto kern) {
        if (smem > 48 * 1024)
            AMG_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        launch_prof(c, kProfGaussSeidel, bytes, kern, blocks_for(base[nsw], kSegWarps), kSegWarps * 32, smem, n,
                    A.rp.get(), A.ci.get(), A.va.get(), inv_diag, b, nsw, static_cast<const unsigned char*>(bwd.get()),
                    static_cast<const int32_t*>(dbase.get()), static_cast<const int32_t*>(segf.get()),
                    static_cast<const int32_t*>(symmetric_sweep ? segb.get() : segf.get()), X.get(), ticket.get());
    };
    switch (k) {
        case 1: run(k_gs_segments<1>); break;
        case 2: run(k_gs_segments<2>); break;
        case 3: run(k_gs_segments<3>); break;
        case 4: run(k_gs_segments<4>); break;
        case 5: run(k_gs_segments<5>); break;
        case 6: run(k_gs_segments<6>); break;
        case 7: run(k_gs_segments<7>); break;
        default: run(k_gs_segments<8>); break;
    }
    copy_d2d(c, x, X.get() + stride * nsw, static_cast<int64_t>(stride));
    sync(c);
    if (std::getenv("AMGCU_DEBUG_GS")) {
        std::vector<int32_t> hs(static_cast<size_t>(nf) + 1);
        copy_d2h(c, hs.data(), segf.get(), nf + 1);
        sync(c);
        int32_t longest = 0;
        for (int32_t g = 0; g < nf; ++g) longest = std::max(longest, hs[g + 1] - hs[g]);
        std::fprintf(stderr, "[gs] n=%d nnz=%lld k=%d sweeps=%d segments=%d longest=%d\n", n,
                     static_cast<long long>(A.nnz), k, nsw, nf, longest);
    }
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
