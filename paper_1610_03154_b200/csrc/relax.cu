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

constexpr int kMaxK = kGsMaxColumns;
constexpr size_t kGsCtaSmem = 220 * 1024;  // dynamic shared memory of the single-CTA kernel
constexpr int32_t kGsCtaMaxRows = 1024;     // below: the single-CTA kernel first (C5: 1.6-1.9 ms vs 2.3-2.8)

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
constexpr int kChunk = 8;     // prefetcher: entries loaded per batch
constexpr unsigned long long kPending = 0x7FF4A11CE5EEDULL;

__device__ __forceinline__ unsigned long long load_relaxed_bits(const double* p) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(
        *reinterpret_cast<unsigned long long*>(const_cast<double*>(p)));
    return r.load(cuda::memory_order_relaxed);
}

__device__ __forceinline__ double wait_bits(const double* p, unsigned long long bits, unsigned max_ns) {
    unsigned ns = 8;
    while (bits == kPending) {
        if (max_ns) __nanosleep(ns);
        ns = ns < max_ns ? 2 * ns : max_ns;
        bits = load_relaxed_bits(p);
    }
    return __longlong_as_double(static_cast<long long>(bits));
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// entry classes in sweep order
enum : int { kSelf = 0, kInBlock = 1, kReady = 2, kPoll = 3 };

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void vstore(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void vstore(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

// Each segment is served by THREE warps of one CTA:
//   prefetcher: phase A for the block AHEAD of the solver (double-buffered):
//     loads every entry and every independent x in batches, sums the CSR
//     prefix that needs no new value, and compiles the rest of the row into a
//     dense TERM list (a, shared-memory slot) -- a slot is the value's record
//     (ready now, or filled in by the poller) or the producer lane's xb entry
//     (this block or the previous one of the own segment);
//   poller:     keeps loading the pending values of the solver's current and
//     next block (lane l for row l, all of the row's loads in flight) and
//     writes each resolved one into its slot;
//   solver:     phase B -- lanes finish their rows in order: for every term,
//     wait until the slot is no longer kPending, then acc -= a * x.  The step
//     is a short branch-free loop over registers (the i-cache matters here:
//     the three roles run side by side on the SM).
// Rows whose entries do not fit the records (more than E, or more
// pending values than the poll list) take a rolled slow path that polls
// global memory directly.
// Hand-shakes (shared memory, volatile): ready[b] = block sequence number the
// buffer b holds; done = last block the solver finished; step = rows of block
// done + 1 finished; plo = lowest block the poller may still touch (the
// prefetcher refills a buffer only when neither the solver nor the poller
// can still use it).  Arrays are stored [.][lane] (conflict-free).
// pending (entry, column) values tracked per row
template <int E>
constexpr int gs_max_poll() {
    return E <= 16 ? 8 : 16;
}
// Sibling segments (earlier segments of the same sweep in the same CTA) hand values
// over through shared memory: every solver keeps its last kRing published rows in a
// tagged ring; a consumer reads tag, value, tag (the producer invalidates the tag
// before rewriting a slot), and falls back to global memory when the row has already
// left the ring.  K = 1 only.
constexpr int kRing = 64;
constexpr int kShortSegment = 8;
constexpr int kSegWarpMinLen = 16;  // mean segment length from which the lane-per-segment kernel runs
constexpr unsigned kWarpRowPollNs = 32;  // poll back-off cap of the warp-per-row kernel  // mean segment length below which the warp-per-row kernel is used
constexpr int32_t kProductTerm = -1;  // term whose product a * x is precomputed (K = 1)
constexpr int kSibling = 4;  // entry class: pending value of a sibling segment

// E: entries per row handled from the records (longer rows take the slow path)
template <int K, int E>
struct GsBuf {
    unsigned long long bits[E][K][32];        // value slots (c stride = 32 words)
    double ta[E][32];                         // term: matrix value
    int32_t toff[E][32];                      // term: slot offset (bytes from the segment base)
    uint32_t paddr[gs_max_poll<E>()][32];     // poll list: element offset of the value in X
    int16_t pslot[gs_max_poll<E>()][32];      // poll list: word offset of the slot in bits
    double acc0[K][32];
    double dinv[32];
    int32_t nterm[32];  // -1: slow path
    int32_t npoll[32];
};

// segments per CTA: 8 short-row (E = 16) single-column segments fit one SM (24 warps,
// ~205 KB), so a 1024-row-grid level is resident at once
template <int K, int E>
constexpr int gs_segs_per_cta() {
    return K == 1 ? (E <= 16 ? 8 : 4) : (K <= 3 ? 2 : 1);
}
constexpr int kSwBits = 3;  // sibling index bits in a sibling term code (<= 8 segments per CTA)

template <int K, int E>
constexpr size_t gs_ring_offset() {
    return (2 * sizeof(GsBuf<K, E>) + 64 * K * sizeof(double) + 15) / 16 * 16;
}

template <int K, int E>
constexpr size_t gs_seg_bytes() {
    return gs_ring_offset<K, E>() + (K == 1 ? kRing * (sizeof(double) + sizeof(int32_t)) : 0);
}

struct GsRing {
    double* val;
    int32_t* tag;
};

template <int K, int E>
__device__ __forceinline__ GsRing gs_ring(unsigned char* smem_base, int w) {
    unsigned char* r = smem_base + static_cast<size_t>(w) * gs_seg_bytes<K, E>() + gs_ring_offset<K, E>();
    return {reinterpret_cast<double*>(r), reinterpret_cast<int32_t*>(r + kRing * sizeof(double))};
}

// value of row qj of a sibling segment: from its ring, or (already overwritten) from global
__device__ __forceinline__ unsigned long long sibling_value(const GsRing& rg, int32_t qj, int32_t tagv,
                                                            const double* gaddr, unsigned max_ns, unsigned spin_ns) {
    const int idx = qj & (kRing - 1);
    // tag, value, tag (volatile shared loads; the producer fences between its stores)
    while (true) {
        const int32_t t1 = vload(&rg.tag[idx]);
        if (t1 == tagv) {
            const unsigned long long v = vload(reinterpret_cast<const unsigned long long*>(&rg.val[idx]));
            if (vload(&rg.tag[idx]) == tagv) return v;
        } else if (t1 > tagv) {
            break;
        }
        if (spin_ns) __nanosleep(spin_ns);
    }
    return static_cast<unsigned long long>(__double_as_longlong(wait_bits(gaddr, load_relaxed_bits(gaddr), max_ns)));
}

template <int K, int E>
__global__ void __launch_bounds__(3 * gs_segs_per_cta<K, E>() * 32)
    k_gs_segments(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  const double* __restrict__ va, const double* __restrict__ inv_diag, const double* __restrict__ b,
                  int nsweeps, const unsigned char* __restrict__ backward, const int32_t* __restrict__ item_base,
                  const int32_t* __restrict__ seg_fwd, const int32_t* __restrict__ seg_bwd, double* __restrict__ X,
                  unsigned int* __restrict__ ticket, unsigned max_ns, unsigned long long* __restrict__ trace,
                  int poll_window, int sweep_loop, unsigned spin_ns) {
    constexpr int S = gs_segs_per_cta<K, E>();
    constexpr int kMaxPoll = gs_max_poll<E>();
    extern __shared__ unsigned long long smem[];
    __shared__ unsigned int blk;
    __shared__ int sh_ready[S][2], sh_done[S], sh_step[S], sh_plo[S];
    __shared__ int32_t sh_sq0[S], sh_sq1[S], sh_ss[S];  // every segment of the CTA: q0, q1, sweep
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    if (threadIdx.x < S) {
        sh_ready[threadIdx.x][0] = sh_ready[threadIdx.x][1] = -1;
        sh_done[threadIdx.x] = -1;
        sh_step[threadIdx.x] = 0;
        sh_plo[threadIdx.x] = 0;
    }
    if (K == 1)
        for (int e = threadIdx.x; e < S * kRing; e += blockDim.x)
            gs_ring<K, E>(reinterpret_cast<unsigned char*>(smem), e / kRing).tag[e % kRing] = -1;
    __syncthreads();
    // sweep_loop (forward sweeps): items are the segments of sweep 0 and every segment
    // runs all sweeps in turn; otherwise items are (sweep, segment) in sweep-major order
    const int32_t nitems = sweep_loop ? item_base[1] : item_base[nsweeps];
    if (threadIdx.x < S) {
        const int32_t it2 = static_cast<int32_t>(blk) * S + threadIdx.x;
        sh_ss[threadIdx.x] = -1;
        sh_sq0[threadIdx.x] = sh_sq1[threadIdx.x] = 0;
        if (sweep_loop && it2 < nitems) {
            sh_ss[threadIdx.x] = 0;
            sh_sq0[threadIdx.x] = seg_fwd[it2];
            sh_sq1[threadIdx.x] = seg_fwd[it2 + 1];
        } else if (!sweep_loop && it2 < nitems) {
            int s2 = 0;
            while (it2 >= item_base[s2 + 1]) ++s2;
            const int32_t* sg = backward[s2] ? seg_bwd : seg_fwd;
            sh_ss[threadIdx.x] = s2;
            sh_sq0[threadIdx.x] = sg[it2 - item_base[s2]];
            sh_sq1[threadIdx.x] = sg[it2 - item_base[s2] + 1];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x / 32;
    const int role = warp / S;  // 0 solver, 1 poller, 2 prefetcher
    const int wl = warp % S;
    const int32_t item = static_cast<int32_t>(blk) * S + wl;
    if (item >= nitems) return;
    int s_first = 0;
    if (!sweep_loop)
        while (item >= item_base[s_first + 1]) ++s_first;
    const int s_item = sweep_loop ? 0 : s_first;  // sweep tag of the CTA segment table
    const int nsw_loop = sweep_loop ? nsweeps : 1;
    const bool bwd = backward[s_first] != 0;
    const int32_t* segs = bwd ? seg_bwd : seg_fwd;
    const int32_t g = item - (sweep_loop ? 0 : item_base[s_first]);
    const int32_t q0 = segs[g], q1 = segs[g + 1];
    const int nblocks = (q1 - q0 + 31) / 32;
    const int tblocks = nsw_loop * nblocks;  // hand-shake sequence numbers run over all sweeps
    const size_t stride = static_cast<size_t>(n) * K;
    unsigned char* segmem = reinterpret_cast<unsigned char*>(smem) + static_cast<size_t>(wl) * gs_seg_bytes<K, E>();
    GsBuf<K, E>* buf = reinterpret_cast<GsBuf<K, E>*>(segmem);
    // values published by the solver: xb[block & 1][c][lane]
    unsigned long long* xb = reinterpret_cast<unsigned long long*>(segmem + 2 * sizeof(GsBuf<K, E>));
    const int32_t xb_off = static_cast<int32_t>(2 * sizeof(GsBuf<K, E>));

    if (role == 2) {
        // ---------------- prefetcher ----------------
        for (int G = 0; G < tblocks; ++G) {
            const int s = s_first + G / nblocks, seq = G % nblocks;
            const double* xin = X + static_cast<size_t>(s) * stride;
            const double* xout = X + static_cast<size_t>(s + 1) * stride;
            if (G >= 2)
                while (vload(&sh_done[wl]) < G - 2 || vload(&sh_plo[wl]) < G - 1) __nanosleep(32);
            __threadfence_block();
            GsBuf<K, E>& B = buf[G & 1];
            const int32_t buf_off = static_cast<int32_t>((G & 1) * sizeof(GsBuf<K, E>));
            const int32_t qb = q0 + 32 * seq;
            const int32_t q = qb + lane;
            const bool active = q < q1;
            const int32_t i = active ? (bwd ? n - 1 - q : q) : 0;
            int32_t lo = 0, hi = 0;
            double dinv_i = 0.0;
            double acc[K];
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = 0.0;
            if (active) {
                lo = rp[i];
                hi = rp[i + 1];
                dinv_i = inv_diag[i];
                if (b) {
#pragma unroll
                    for (int c = 0; c < K; ++c) acc[c] = b[static_cast<size_t>(c) * n + i];
                }
            }
            const int32_t ne = min(hi - lo, E);
            int np = 0;
            bool slow = active && hi - lo > E;
            // pass 1, kChunk entries at a time: class, slot and every independent value.
            // Staging: ta[e] = a, toff[e] = class | xb offset << 2.
            for (int e0 = 0; e0 < ne; e0 += kChunk) {
                int32_t jj[kChunk];
                double aa[kChunk];
#pragma unroll
                for (int u = 0; u < kChunk; ++u) {
                    jj[u] = i;
                    aa[u] = 0.0;
                    if (e0 + u < ne) {
                        jj[u] = ci[lo + e0 + u];
                        aa[u] = va[lo + e0 + u];
                    }
                }
                int cls[kChunk], xslot[kChunk];
#pragma unroll
                for (int u = 0; u < kChunk; ++u) {
                    const int32_t j = jj[u];
                    const int32_t qj = bwd ? n - 1 - j : j;
                    const bool fresh = qj < q;
                    int cl = kSelf, xs = 0;
                    if (e0 + u < ne && j != i) {
                        if (fresh && qj >= qb) {
                            cl = kInBlock;
                            xs = xb_off + 8 * ((seq & 1) * 32 * K + (qj - qb));
                        } else if (fresh && qj >= q0 && qj >= qb - 32) {
                            cl = kInBlock;
                            xs = xb_off + 8 * (((seq + 1) & 1) * 32 * K + (qj - qb + 32));
                        } else {
                            cl = ((fresh && qj >= q0) || (!fresh && s == 0)) ? kReady : kPoll;
                        }
                    }
                    cls[u] = cl;
                    xslot[u] = xs;
                }
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    unsigned long long xv[kChunk];
#pragma unroll
                    for (int u = 0; u < kChunk; ++u) {
                        xv[u] = kPending;
                        if (cls[u] >= kReady) {
                            const int32_t j = jj[u];
                            const int32_t qj = bwd ? n - 1 - j : j;
                            const double* addr = &((qj < q) ? xout : xin)[static_cast<size_t>(c) * n + j];
                            xv[u] = cls[u] == kReady
                                        ? static_cast<unsigned long long>(__double_as_longlong(__ldcg(addr)))
                                        : load_relaxed_bits(addr);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kChunk; ++u) {
                        if (cls[u] >= kReady) {
                            const int e = e0 + u;
                            B.bits[e][c][lane] = xv[u];
                            int sw = -1;
                            if (K == 1 && xv[u] == kPending && cls[u] == kPoll) {
                                const int32_t qj = bwd ? n - 1 - jj[u] : jj[u];
                                // an earlier segment of this sweep in this CTA
                                for (int w2 = 0; w2 < wl; ++w2)
                                    if (sh_ss[w2] == s_item && qj >= sh_sq0[w2] && qj < sh_sq1[w2]) sw = w2;
                                if (sw >= 0) {
                                    cls[u] = kSibling;
                                    xslot[u] = ((qj - sh_sq0[sw]) << kSwBits) | sw;
                                }
                            }
                            if (xv[u] == kPending && sw < 0) {
                                if (np < kMaxPoll) {
                                    const int32_t j = jj[u];
                                    const int32_t qj = bwd ? n - 1 - j : j;
                                    B.paddr[np][lane] = static_cast<uint32_t>(
                                        static_cast<size_t>((qj < q) ? s + 1 : s) * stride + static_cast<size_t>(c) * n + j);
                                    B.pslot[np][lane] = static_cast<int16_t>((e * K + c) * 32 + lane);
                                    ++np;
                                } else {
                                    slow = true;
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kChunk; ++u) {
                    if (e0 + u < ne) {
                        B.ta[e0 + u][lane] = aa[u];
                        B.toff[e0 + u][lane] = cls[u] | (xslot[u] << 3);
                    }
                }
            }
            // pass 2 (in place, nt <= e): the CSR prefix that needs neither an xb value nor a
            // pending one, then the term list
            bool stopped = false;
            int nt = 0;
            for (int e = 0; e < ne; ++e) {
                const int code = B.toff[e][lane];
                const int cl = code & 7;
                if (cl == kSelf) continue;
                const double ae = B.ta[e][lane];
                if (!stopped) {
                    bool pending = cl == kInBlock || cl == kSibling;
#pragma unroll
                    for (int c = 0; c < K; ++c) pending = pending || B.bits[e][c][lane] == kPending;
                    stopped = pending;
                }
                if (!stopped) {
#pragma unroll
                    for (int c = 0; c < K; ++c)
                        acc[c] -= ae * __longlong_as_double(static_cast<long long>(B.bits[e][c][lane]));
                } else {
                    // slot offset; a sibling term is -2 - ((row - sibling q0) << 2 | sibling);
                    // K = 1 values known now become product terms (kProductTerm, ta = a * x:
                    // the reference's acc - (a * x) with the product rounded first)
                    const bool known = K == 1 && cl != kInBlock && cl != kSibling && B.bits[e][0][lane] != kPending;
                    B.ta[nt][lane] =
                        known ? ae * __longlong_as_double(static_cast<long long>(B.bits[e][0][lane])) : ae;
                    B.toff[nt][lane] = known            ? kProductTerm
                                       : cl == kInBlock  ? (code >> 3)
                                       : cl == kSibling ? -2 - (code >> 3)
                                                        : buf_off + static_cast<int32_t>(8 * (e * K * 32 + lane));
                    ++nt;
                }
            }
#pragma unroll
            for (int c = 0; c < K; ++c) B.acc0[c][lane] = acc[c];
            B.dinv[lane] = dinv_i;
            B.nterm[lane] = slow ? -1 : nt;
            B.npoll[lane] = slow ? 0 : np;
            __syncwarp();
            __threadfence_block();
            if (lane == 0) vstore(&sh_ready[wl][G & 1], G);
        }
        return;
    }

    if (role == 1) {
        // ---------------- poller ----------------
        int mblk[2] = {-1, -1};
        unsigned mask[2] = {0u, 0u};
        unsigned ns = 0;
        unsigned long long* bits_base[2] = {&buf[0].bits[0][0][0], &buf[1].bits[0][0][0]};
        while (true) {
            const int cur = vload(&sh_done[wl]) + 1;
            if (cur >= tblocks) break;
            vstore(&sh_plo[wl], cur);
            __threadfence_block();
            const int step = vload(&sh_step[wl]);
            bool progress = false, more = false;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int bq = cur + h;
                const int sl = bq & 1;
                if (bq >= tblocks) continue;
                if (mblk[sl] != bq) {
                    if (vload(&sh_ready[wl][sl]) != bq) continue;
                    __threadfence_block();
                    mblk[sl] = bq;
                    const int np = q0 + 32 * (bq % nblocks) + lane < q1 ? buf[sl].npoll[lane] : 0;
                    mask[sl] = np >= 32 ? 0xffffffffu : ((1u << np) - 1u);
                }
                const int rel = h * 32 + lane - step;  // rows ahead of the solver
                const unsigned m = (rel < 0 || rel >= poll_window) ? 0u : mask[sl];
                if (!m) continue;
                GsBuf<K, E>& B = buf[sl];
                unsigned long long got[kMaxPoll];
#pragma unroll
                for (int u = 0; u < kMaxPoll; ++u) got[u] = (m >> u) & 1u ? load_relaxed_bits(X + B.paddr[u][lane]) : kPending;
#pragma unroll
                for (int u = 0; u < kMaxPoll; ++u) {
                    if (((m >> u) & 1u) && got[u] != kPending) {
                        vstore(bits_base[sl] + B.pslot[u][lane], got[u]);
                        mask[sl] &= ~(1u << u);
                        progress = true;
                    }
                }
                if (mask[sl]) more = true;
            }
            if (__any_sync(0xffffffffu, progress)) {
                ns = 0;
            } else {
                // nothing resolved: back off (longer when nothing is pending at all)
                const bool any_more = __any_sync(0xffffffffu, more);
                if (any_more && !spin_ns) {
                    ns = 0;  // values pending: keep polling
                } else {
                    ns = ns ? min(2 * ns, any_more ? 64u : 512u) : 16u;
                    __nanosleep(ns);
                }
            }
        }
        return;
    }

    // ---------------- solver ----------------
    for (int G = 0; G < tblocks; ++G) {
        const int s = s_first + G / nblocks, seq = G % nblocks;
        const double* xin = X + static_cast<size_t>(s) * stride;
        double* xout = X + static_cast<size_t>(s + 1) * stride;
        const int32_t qb = q0 + 32 * seq;
        unsigned long long* tr = trace ? trace + (static_cast<size_t>(s) * n + qb) * 4 : nullptr;
        if (tr && lane == 0) tr[0] = globaltimer_ns();
        // this block's xb slots become pending (the previous block's stay readable)
#pragma unroll
        for (int c = 0; c < K; ++c) xb[((seq & 1) * K + c) * 32 + lane] = kPending;
        while (vload(&sh_ready[wl][G & 1]) != G) __nanosleep(32);
        __threadfence_block();
        GsBuf<K, E>& B = buf[G & 1];
        if (tr && lane == 0) tr[1] = globaltimer_ns();
        // ---- phase B, warp-uniform: every lane evaluates row t from broadcast reads of
        // its records (no divergence, no reconvergence barriers); lane 0 publishes ----
        const int32_t cnt = min(32, q1 - qb);
        for (int32_t t = 0; t < cnt; ++t) {
            const int32_t q = qb + t;
            const int32_t i = bwd ? n - 1 - q : q;
            const int32_t nt = B.nterm[t];
            double acc[K];
            if (K == 1 && nt >= 0) {
                // lane k resolves term k (its product a * x rounded, as the reference's
                // acc - a * x rounds it); the warp then subtracts the products in term order
                // from shuffles, so the serial part is the chain of subtractions alone
                double p = 0.0;
                if (lane < nt) {
                    const double ak = B.ta[lane][t];
                    const int32_t off = B.toff[lane][t];
                    if (off == kProductTerm) {
                        p = ak;
                    } else if (off < 0) {
                        const int32_t code = -2 - off;
                        const int sw = code & ((1 << kSwBits) - 1);
                        const int32_t qj = sh_sq0[sw] + (code >> kSwBits);
                        const int32_t j = bwd ? n - 1 - qj : qj;
                        const unsigned long long v =
                            sibling_value(gs_ring<K, E>(reinterpret_cast<unsigned char*>(smem), sw), qj, s * n + qj,
                                          &xout[j], max_ns, spin_ns);
                        p = ak * __longlong_as_double(static_cast<long long>(v));
                    } else {
                        const unsigned long long* slot = reinterpret_cast<const unsigned long long*>(segmem + off);
                        unsigned long long v = vload(slot);
                        while (v == kPending) {
                            if (spin_ns) __nanosleep(spin_ns);
                            v = vload(slot);
                        }
                        p = ak * __longlong_as_double(static_cast<long long>(v));
                    }
                }
                double a0 = B.acc0[0][t];
                for (int32_t k0 = 0; k0 < nt; k0 += 8) {
                    double pk[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) pk[u] = __shfl_sync(0xffffffffu, p, k0 + u);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (k0 + u < nt) a0 -= pk[u];
                }
                acc[0] = a0;
            } else if (nt >= 0) {
#pragma unroll
                for (int c = 0; c < K; ++c) acc[c] = B.acc0[c][t];
#pragma unroll 4
                for (int32_t k = 0; k < nt; ++k) {
                    const double ak = B.ta[k][t];
                    const int32_t off = B.toff[k][t];
                    if (K == 1 && off == kProductTerm) {
                        acc[0] -= ak;
                        continue;
                    }
                    if (K == 1 && off < 0) {
                        const int32_t code = -2 - off;
                        const int sw = code & ((1 << kSwBits) - 1);
                        const int32_t qj = sh_sq0[sw] + (code >> kSwBits);
                        const int32_t j = bwd ? n - 1 - qj : qj;
                        const unsigned long long v =
                            sibling_value(gs_ring<K, E>(reinterpret_cast<unsigned char*>(smem), sw), qj,
                                          s * n + qj, &xout[j], max_ns, spin_ns);
                        acc[0] -= ak * __longlong_as_double(static_cast<long long>(v));
                        continue;
                    }
                    const unsigned char* sp = segmem + off;
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const unsigned long long* slot = reinterpret_cast<const unsigned long long*>(sp) + 32 * c;
                        unsigned long long v = vload(slot);
                        while (v == kPending) {
                            if (spin_ns) __nanosleep(spin_ns);
                            v = vload(slot);
                        }
                        acc[c] -= ak * __longlong_as_double(static_cast<long long>(v));
                    }
                }
            } else {
                // slow path: the whole row in CSR order, values from xb or global memory
#pragma unroll
                for (int c = 0; c < K; ++c) acc[c] = b ? b[static_cast<size_t>(c) * n + i] : 0.0;
                const int32_t lo = rp[i], hi = rp[i + 1];
                for (int32_t p = lo; p < hi; ++p) {
                    const int32_t j = ci[p];
                    if (j == i) continue;
                    const int32_t qj = bwd ? n - 1 - j : j;
                    const bool fresh = qj < q;
                    const double av = va[p];
                    if (fresh && qj >= qb) {
#pragma unroll
                        for (int c = 0; c < K; ++c)
                            acc[c] -= av * __longlong_as_double(static_cast<long long>(
                                               vload(&xb[((seq & 1) * K + c) * 32 + (qj - qb)])));
                        continue;
                    }
                    const double* src = fresh ? xout : xin;
                    const bool own = fresh && qj >= q0;  // earlier blocks of the own segment: published
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const double* addr = &src[static_cast<size_t>(c) * n + j];
                        const unsigned long long bb =
                            (own || (!fresh && s == 0))
                                ? static_cast<unsigned long long>(__double_as_longlong(__ldcg(addr)))
                                : load_relaxed_bits(addr);
                        acc[c] -= av * wait_bits(addr, bb, max_ns);
                    }
                }
            }
            const double dinv_t = B.dinv[t];
            if (lane == 0) {
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    const double xi = acc[c] * dinv_t;
                    const unsigned long long xbits = static_cast<unsigned long long>(__double_as_longlong(xi));
                    vstore(&xb[((seq & 1) * K + c) * 32 + t], xbits);
                    if (K == 1) {
                        // own ring first (its fences then cover shared-memory stores only):
                        // invalidate the slot, write the value, then the tag
                        const GsRing rg = gs_ring<K, E>(reinterpret_cast<unsigned char*>(smem), wl);
                        const int idx = q & (kRing - 1);
                        vstore(&rg.tag[idx], -1);
                        __threadfence_block();
                        vstore(reinterpret_cast<unsigned long long*>(&rg.val[idx]), xbits);
                        __threadfence_block();
                        vstore(&rg.tag[idx], s * n + q);
                    }
                    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> out(
                        *reinterpret_cast<unsigned long long*>(&xout[static_cast<size_t>(c) * n + i]));
                    out.store(xbits, cuda::memory_order_relaxed);
                }
                vstore(&sh_step[wl], t + 1);
                if (trace) trace[(static_cast<size_t>(s) * n + q) * 4 + 3] = globaltimer_ns();
            }
            __syncwarp();
        }
        if (tr && lane == 0) tr[2] = globaltimer_ns();
        __syncwarp();
        __threadfence_block();
        if (lane == 0) {
            vstore(&sh_step[wl], 0);
            vstore(&sh_done[wl], G);
        }
    }
}

// Warp per row for levels whose segments are short (coarse operators: the i-1
// chains break every row or two, so a segment's three warps have nothing to
// pipeline).  Items (sweep, position) draw tickets in order, one warp each; the
// lanes load the row's entries and poll their values in parallel (the previous
// sweep's for later rows, this sweep's for earlier ones), form the products
// a * x, and lane 0 subtracts them from b in CSR order -- the reference's row.
constexpr int kWrWarps = 8;

template <int K>
__device__ __forceinline__ void gs_warp_row(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                            const double* __restrict__ va, const double* __restrict__ inv_diag,
                                            const double* __restrict__ b, int s, int32_t q, bool bwd,
                                            double* __restrict__ X, unsigned max_ns, double* __restrict__ sp) {
    const int lane = threadIdx.x & 31;
    const int32_t i = bwd ? n - 1 - q : q;
    const size_t stride = static_cast<size_t>(n) * K;
    const double* xin = X + static_cast<size_t>(s) * stride;
    double* xout = X + static_cast<size_t>(s + 1) * stride;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = b ? b[static_cast<size_t>(c) * n + i] : 0.0;
    const int32_t lo = rp[i], hi = rp[i + 1];
    for (int32_t e0 = lo; e0 < hi; e0 += 32) {
        const int32_t p = e0 + lane;
        const bool act = p < hi;
        int32_t j = i;
        double a = 0.0;
        if (act) {
            j = ci[p];
            a = va[p];
        }
        const bool use = act && j != i;
        double prod[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            unsigned long long v = 0ull;
            const double* addr = nullptr;
            if (use) {
                const int32_t qj = bwd ? n - 1 - j : j;
                addr = &((qj < q) ? xout : xin)[static_cast<size_t>(c) * n + j];
                v = (qj >= q && s == 0) ? static_cast<unsigned long long>(__double_as_longlong(__ldcg(addr)))
                                        : load_relaxed_bits(addr);
            }
            unsigned ns = 8;
            while (__any_sync(0xffffffffu, use && v == kPending)) {
                if (use && v == kPending) {
                    __nanosleep(ns);
                    v = load_relaxed_bits(addr);
                }
                ns = ns < max_ns ? 2 * ns : max_ns;
            }
            prod[c] = use ? a * __longlong_as_double(static_cast<long long>(v)) : 0.0;
        }
        // ordered subtraction by lane 0 (CSR order; the diagonal is skipped): the products
        // are staged in shared memory and lane 0 runs a fixed 32-step chain over them,
        // unused lanes contributing +0.0 (x - (+0) is x for every x, -0 included).  The
        // loads have constant addresses and issue ahead of the chain, the K columns'
        // chains interleave, and no shuffle sits in this (to the compiler possibly
        // divergent) loop, where it would compile to a WARPSYNC.COLLECTIVE sequence.
#pragma unroll
        for (int c = 0; c < K; ++c) sp[c * 32 + lane] = prod[c];
        __syncwarp();
        if (lane == 0) {
#pragma unroll
            for (int l = 0; l < 32; ++l) {
#pragma unroll
                for (int c = 0; c < K; ++c) acc[c] -= sp[c * 32 + l];
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        const double d = inv_diag[i];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> out(
                *reinterpret_cast<unsigned long long*>(&xout[static_cast<size_t>(c) * n + i]));
            out.store(static_cast<unsigned long long>(__double_as_longlong(acc[c] * d)), cuda::memory_order_relaxed);
        }
    }
}

// Small levels (the coarse end of a hierarchy): one CTA holds the whole iterate in
// shared memory and relaxes it in place, all sweeps in one launch.  Items are (sweep,
// position) in sweep-major order, item t on warp t % 32; a row's version counter
// (shared) says how many sweeps it has finished.  Row i in sweep s waits for its own
// version s, then reads the rows before it in sweep order at version s + 1 (new
// values) and the rows after it at version s (old values).  In place is exact because the pattern is structurally
// symmetric (checked by the launcher): a row j after i that i reads is itself a reader
// of i, so it cannot write its sweep-s value before i has published (and therefore
// finished reading).  Every item waits only on earlier items, and all warps are
// resident, so the launch cannot deadlock.  Each row sums in CSR order with the
// diagonal skipped: the lanes stage a 32-entry chunk's products in shared memory and
// lane 0 runs a fixed 32-step chain over them, unused lanes contributing +0.0 (an exact
// identity).
constexpr int kCtaWarps = 32;
// dynamic shared memory of k_gs_cta: the iterate, the per-warp product stages, versions
inline size_t gs_cta_smem(int32_t n, int k) {
    return sizeof(double) * (static_cast<size_t>(k) * n + static_cast<size_t>(kCtaWarps) * 32 * k) +
           sizeof(int32_t) * static_cast<size_t>(n);
}

__device__ __forceinline__ int32_t ld_ver(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p)))
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_ver(int32_t* p, int32_t v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(p))), "r"(v)
                 : "memory");
}

template <int K>
__global__ void __launch_bounds__(kCtaWarps * 32, 1)
    k_gs_cta(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ va,
             const double* __restrict__ inv_diag, const double* __restrict__ b, int nsweeps,
             const unsigned char* __restrict__ backward, double* __restrict__ x, unsigned spin_ns) {
    extern __shared__ __align__(16) double cta_smem[];
    double* xs = cta_smem;                                       // K x n, column-major like x
    double* sp = xs + static_cast<size_t>(K) * n + static_cast<size_t>(threadIdx.x >> 5) * (K * 32);  // products
    int32_t* ver = reinterpret_cast<int32_t*>(xs + static_cast<size_t>(K) * n + kCtaWarps * K * 32);
    for (int32_t t = threadIdx.x; t < K * n; t += blockDim.x) xs[t] = x[t];
    for (int32_t t = threadIdx.x; t < n; t += blockDim.x) ver[t] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    volatile double* vx = xs;
    const int64_t items = static_cast<int64_t>(nsweeps) * n;
    for (int64_t t = warp; t < items; t += kCtaWarps) {
        const int s = static_cast<int>(t / n);
        const int32_t q = static_cast<int32_t>(t - static_cast<int64_t>(s) * n);
        const bool bwd = backward[s] != 0;
        const int32_t i = bwd ? n - 1 - q : q;
        double acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = b ? b[static_cast<size_t>(c) * n + i] : 0.0;
        const int32_t lo = rp[i], hi = rp[i + 1];
        // the row's own previous sweep first: nothing else orders (s - 1, i) before (s, i)
        // when the row's neighbours do not (the last row of a forward half-sweep starts
        // the backward one, and reads only rows that did not wait for it)
        while (ld_ver(ver + i) < s)
            if (spin_ns) __nanosleep(spin_ns);
        for (int32_t e0 = lo; e0 < hi; e0 += 32) {
            const int32_t p = e0 + lane;
            const bool act = p < hi;
            int32_t j = i;
            double a = 0.0;
            if (act) {
                j = __ldg(ci + p);
                a = __ldg(va + p);
            }
            const bool use = act && j != i;
            const int32_t need = ((j < i) != bwd) ? s + 1 : s;
            // warp-uniform wait: the warp stays converged for the staging below
            while (__any_sync(0xffffffffu, use && ld_ver(ver + j) < need))
                if (spin_ns) __nanosleep(spin_ns);
#pragma unroll
            for (int c = 0; c < K; ++c) sp[c * 32 + lane] = use ? a * vx[static_cast<size_t>(c) * n + j] : 0.0;
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int l = 0; l < 32; ++l) {
#pragma unroll
                    for (int c = 0; c < K; ++c) acc[c] -= sp[c * 32 + l];
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            const double d = inv_diag[i];
#pragma unroll
            for (int c = 0; c < K; ++c) vx[static_cast<size_t>(c) * n + i] = acc[c] * d;
            st_ver(ver + i, s + 1);
        }
        __syncwarp();
    }
    __syncthreads();
    for (int32_t t = threadIdx.x; t < K * n; t += blockDim.x) x[t] = xs[t];
}

// flag = 1 if some stored (i, j) has no stored (j, i)
__global__ void k_pattern_asym(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               int32_t* __restrict__ flag) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = ci[p];
        int32_t lo = rp[j], hi = rp[j + 1];
        while (lo < hi) {
            const int32_t mid = (lo + hi) >> 1;
            if (ci[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        if (lo == rp[j + 1] || ci[lo] != i) {
            *flag = 1;
            return;
        }
    }
}

// Long segments of long rows (coarse levels of vector problems: C5 level 1 has 342
// segments of 684 rows of up to 50 entries): a warp per segment relaxes the segment's
// rows in order, every forward sweep in turn.  A row's lanes take its entries 32 at a
// time; the products are staged in shared memory and lane c subtracts column c's in CSR
// order (the K chains side by side in one instruction stream; the diagonal's slot
// contributes +0.0, an exact identity).  A lone warp issues a dependent instruction every
// ~4 cycles, so a row step costs ~300 instructions x 4 cycles (0.6-0.9 us, measured on an
// isolated chain by tools/gs_chain_rate.py) however far ahead its loads are issued.  Values of
// the warp's own segment from this sweep come from a shared ring of its last kSwRing
// rows (or its own global stores); other segments' values are polled in the per-sweep
// buffers (pre-filled with kPending).  Items (sweep, row) run in that order within a
// segment, every wait is on an item earlier in (sweep, position) order, and the
// launcher keeps every warp resident, so the earliest unfinished item always runs.
constexpr int kSwWarps = 4;
constexpr int kSwRing = 64;

// E: entries per lane and chunk (a chunk is 32 E entries; rows of up to 64 entries -- the
// coarse levels of vector problems -- take E = 2 so that the whole row is one pipelined chunk)
template <int K, int E>
__global__ void __launch_bounds__(kSwWarps * 32)
    k_gs_seg_warp(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  const double* __restrict__ va, const double* __restrict__ inv_diag, const double* __restrict__ b,
                  int nsweeps, const int32_t* __restrict__ segs, int32_t nseg, double* __restrict__ X,
                  unsigned int* __restrict__ ticket, unsigned max_ns) {
    constexpr int W = 32 * E;
    __shared__ unsigned int blk;
    __shared__ double ring[kSwWarps][K][kSwRing];
    __shared__ double stage[kSwWarps][K][W + 1];  // padded: lanes 0..K-1 walk their columns' products side by side
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int32_t g = static_cast<int32_t>(blk) * kSwWarps + w;
    if (g >= nseg) return;
    const int32_t q0 = segs[g], q1 = segs[g + 1];
    const size_t stride = static_cast<size_t>(n) * K;
    double (*rg)[kSwRing] = ring[w];
    double (*sp)[W + 1] = stage[w];
    // software pipeline over the items u = (sweep, row), so that no global-memory latency
    // sits between the end of one row and the start of the next: the row bounds three
    // items ahead, the first chunk's entries two items ahead, and -- issued while the
    // current row's products are summed -- the next item's inverse diagonal and the values
    // its first chunk reads outside the ring (a value still pending then is polled when
    // the item runs; a published value is final, the per-sweep buffers are written once)
    const int32_t len = q1 - q0;
    const int64_t total = static_cast<int64_t>(len) * nsweeps;
    // (sweep, position) of item u, kept incrementally (no 64-bit divisions in the loop)
    int s_cur = 0;
    int32_t pos_cur = 0;
    auto ahead = [&](int k, int& s_, int32_t& pos_) {  // item u + k, k <= 3
        s_ = s_cur;
        pos_ = pos_cur + k;
        while (pos_ >= len) {
            pos_ -= len;
            ++s_;
        }
    };
    auto row_ahead = [&](int k) {
        int s_;
        int32_t pos_;
        ahead(k, s_, pos_);
        return q0 + pos_;
    };
    struct Src {
        bool use, ring, settled;
        const double* p;
    };
    auto classify = [&](int32_t i, int s, int32_t j, bool act) {
        Src r;
        r.use = act && j != i;
        const bool newer = j < i;
        const bool own = j >= q0 && j < q1;
        // where the value comes from: own ring (this sweep, own segment, recent),
        // own or settled stores (no poll), or another segment's buffer (poll)
        r.ring = r.use && newer && own && i - j <= kSwRing;
        r.settled = !newer && (s == 0 || own);
        r.p = X + static_cast<size_t>(newer ? s + 1 : s) * stride + j;
        return r;
    };
    auto fetch = [&](const Src& r, unsigned long long (&v)[K]) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
            v[c] = 0ull;
            if (r.use && !r.ring)
                v[c] = r.settled ? static_cast<unsigned long long>(__double_as_longlong(r.p[static_cast<size_t>(c) * n]))
                                 : load_relaxed_bits(r.p + static_cast<size_t>(c) * n);
        }
    };
    auto first_chunk = [&](int32_t lo_, int32_t hi_, int32_t (&j_)[E], double (&a_)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            j_[e] = -1;
            a_[e] = 0.0;
            const int32_t p = lo_ + e * 32 + lane;
            if (p < hi_) {
                j_[e] = __ldg(ci + p);
                a_[e] = __ldg(va + p);
            }
        }
    };
    auto bounds = [&](int64_t u, int k, int32_t& lo_, int32_t& hi_) {  // item u + k
        lo_ = hi_ = 0;
        if (u + k < total) {
            const int32_t r = row_ahead(k);
            lo_ = __ldg(rp + r);
            hi_ = __ldg(rp + r + 1);
        }
    };
    int32_t lo1, hi1, lo2, hi2, lo3, hi3;  // items u, u + 1, u + 2 at the top of iteration u
    bounds(0, 0, lo1, hi1);
    bounds(0, 1, lo2, hi2);
    bounds(0, 2, lo3, hi3);
    int32_t j1[E], j2[E];
    double a1[E], a2[E];
    first_chunk(lo1, hi1, j1, a1);
    first_chunk(lo2, hi2, j2, a2);
    unsigned long long v1[E][K];  // item u's prefetched values
    double d1 = inv_diag[q0];
#pragma unroll
    for (int e = 0; e < E; ++e) fetch(classify(q0, 0, j1[e] < 0 ? q0 : j1[e], j1[e] >= 0), v1[e]);
    for (int64_t u = 0; u < total; ++u) {
        const int s = s_cur;
        const int32_t i = q0 + pos_cur;
        const int32_t lo = lo1, hi = hi1;
        int32_t jf[E];
        double af[E];
        unsigned long long vf[E][K];
        const double dcur = d1;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            jf[e] = j1[e];
            af[e] = a1[e];
#pragma unroll
            for (int c = 0; c < K; ++c) vf[e][c] = v1[e][c];
        }
        // advance the pipeline: item u + 2's first chunk, item u + 3's bounds
        lo1 = lo2;
        hi1 = hi2;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            j1[e] = j2[e];
            a1[e] = a2[e];
        }
        lo2 = lo3;
        hi2 = hi3;
        first_chunk(lo2, hi2, j2, a2);
        bounds(u, 3, lo3, hi3);
        double* xout = X + static_cast<size_t>(s + 1) * stride;
        // lane c (< K) carries column c's sum: the K ordered chains run side by side in
        // one instruction stream instead of one after the other in lane 0
        double acc = (b && lane < K) ? b[static_cast<size_t>(lane) * n + i] : 0.0;
        for (int32_t e0 = lo; e0 < hi || e0 == lo; e0 += W) {
            int32_t j[E];
            double a[E];
            unsigned long long v[E][K];
            Src sr[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int32_t p = e0 + e * 32 + lane;
                const bool act = p < hi;
                j[e] = i;
                a[e] = 0.0;
                if (e0 == lo) {
                    if (act) {
                        j[e] = jf[e];
                        a[e] = af[e];
                    }
                    sr[e] = classify(i, s, j[e], act);
#pragma unroll
                    for (int c = 0; c < K; ++c) v[e][c] = vf[e][c];
                } else {
                    if (act) {
                        j[e] = __ldg(ci + p);
                        a[e] = __ldg(va + p);
                    }
                    sr[e] = classify(i, s, j[e], act);
                    fetch(sr[e], v[e]);
                }
            }
            unsigned ns = 8;
            while (true) {
                bool pend = false;
#pragma unroll
                for (int e = 0; e < E; ++e)
#pragma unroll
                    for (int c = 0; c < K; ++c) pend |= sr[e].use && !sr[e].ring && v[e][c] == kPending;
                if (!__any_sync(0xffffffffu, pend)) break;
                if (pend) {
                    __nanosleep(ns);
#pragma unroll
                    for (int e = 0; e < E; ++e)
#pragma unroll
                        for (int c = 0; c < K; ++c)
                            if (sr[e].use && !sr[e].ring && v[e][c] == kPending)
                                v[e][c] = load_relaxed_bits(sr[e].p + static_cast<size_t>(c) * n);
                }
                ns = ns < max_ns ? 2 * ns : max_ns;
            }
#pragma unroll
            for (int e = 0; e < E; ++e)
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    const double xv = sr[e].ring ? rg[c][j[e] % kSwRing] : __longlong_as_double(static_cast<long long>(v[e][c]));
                    sp[c][e * 32 + lane] = sr[e].use ? a[e] * xv : 0.0;
                }
            __syncwarp();
            const bool last = e0 + W >= hi;
            if (last && u + 1 < total) {
                // the next item's inverse diagonal and out-of-ring values, in flight
                // while this row's products are summed
                int s1;
                int32_t pos1;
                ahead(1, s1, pos1);
                const int32_t i1 = q0 + pos1;
                d1 = inv_diag[i1];
#pragma unroll
                for (int e = 0; e < E; ++e) fetch(classify(i1, s1, j1[e] < 0 ? i1 : j1[e], j1[e] >= 0), v1[e]);
            }
            if (lane < K) {
                // the chunk's entries in CSR order (the diagonal's slot holds +0.0, an exact identity)
                const int cnt = min(W, hi - e0);
                const double* col = sp[lane];
#pragma unroll 6
                for (int l = 0; l < cnt; ++l) acc -= col[l];
            }
            __syncwarp();
        }
        if (lane < K) {
            const double xn = acc * dcur;
            rg[lane][i % kSwRing] = xn;
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> out(
                *reinterpret_cast<unsigned long long*>(&xout[static_cast<size_t>(lane) * n + i]));
            out.store(static_cast<unsigned long long>(__double_as_longlong(xn)), cuda::memory_order_relaxed);
        }
        __syncwarp();
        if (++pos_cur == len) {
            pos_cur = 0;
            ++s_cur;
        }
    }
}

// kRowMajor (forward sweeps only): a warp owns one row and relaxes it in every
// sweep in turn (tickets in row order); sweep s + 1 of row q waits on sweep s of
// rows at most the bandwidth ahead, so the launcher uses it only when the
// bandwidth is well below the number of resident warps.  Otherwise items are
// (sweep, position) in sweep-major order.
template <int K, bool kRowMajor>
__global__ void __launch_bounds__(kWrWarps * 32)
    k_gs_warp_rows(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                   const double* __restrict__ va, const double* __restrict__ inv_diag, const double* __restrict__ b,
                   int nsweeps, const unsigned char* __restrict__ backward, double* __restrict__ X,
                   unsigned int* __restrict__ ticket, unsigned max_ns) {
    __shared__ unsigned int blk;
    __shared__ double stage[kWrWarps][K * 32];  // per warp: the chunk's products (gs_warp_row)
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    double* sp = stage[threadIdx.x / 32];
    const int64_t item = static_cast<int64_t>(blk) * kWrWarps + threadIdx.x / 32;
    if (kRowMajor) {
        if (item >= n) return;
        for (int s = 0; s < nsweeps; ++s) gs_warp_row<K>(n, rp, ci, va, inv_diag, b, s, static_cast<int32_t>(item),
                                                         false, X, max_ns, sp);
    } else {
        if (item >= static_cast<int64_t>(nsweeps) * n) return;
        const int s = static_cast<int>(item / n);
        gs_warp_row<K>(n, rp, ci, va, inv_diag, b, s, static_cast<int32_t>(item - static_cast<int64_t>(s) * n),
                       backward[s] != 0, X, max_ns, sp);
    }
}

// bw[0] = max |i - j| over the stored entries, bw[1] = longest row
__global__ void k_bandwidth(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            int32_t* __restrict__ bw) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t m = 0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) m = max(m, abs(ci[p] - i));
    atomicMax(bw, m);
    atomicMax(bw + 1, rp[i + 1] - rp[i]);
}

// segment heads in sweep order: position q starts a segment unless row(q)
// holds column row(q - 1)
// window w: position q continues a segment if row(q) holds a column among the w rows
// before it in sweep order (w = 1: the predecessor; w = block size: interleaved vector
// unknowns, whose chains run with stride w)
__global__ void k_segment_heads(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, bool bwd,
                                int32_t* __restrict__ head, int32_t w) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    if (q == 0) {
        head[0] = 1;
        return;
    }
    const int32_t i = bwd ? n - 1 - q : q;
    // columns in [a, b] (row indices of the w previous positions)
    const int32_t a = bwd ? i + 1 : max(i - w, 0), bcol = bwd ? min(i + w, n - 1) : i - 1;
    int32_t lo = rp[i], hi = rp[i + 1];
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (ci[mid] < a) lo = mid + 1;
        else hi = mid;
    }
    head[q] = (lo < rp[i + 1] && ci[lo] <= bcol) ? 0 : 1;
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

// poll back-off cap in ns (AMGCU_GS_NS overrides; 0 = spin)
unsigned gs_max_ns() {
    static const unsigned v = [] {
        const char* e = std::getenv("AMGCU_GS_NS");
        return e ? static_cast<unsigned>(std::atoi(e)) : 512u;
    }();
    return v;
}

unsigned gs_env_u(const char* name, unsigned dflt) {
    const char* e = std::getenv(name);
    return e ? static_cast<unsigned>(std::atoi(e)) : dflt;
}

// back-off of the shared-memory spins and of the poller while values are pending
// (AMGCU_GS_SPIN; 0 = spin without sleeping)
unsigned gs_spin_ns() {
    static const unsigned v = [] {
        const char* e = std::getenv("AMGCU_GS_SPIN");
        return e ? static_cast<unsigned>(std::atoi(e)) : 0u;
    }();
    return v;
}

// rows ahead of the solver whose pending values the poller keeps loading (AMGCU_GS_PW)
int gs_poll_window() {
    static const int v = [] {
        const char* e = std::getenv("AMGCU_GS_PW");
        return e ? std::atoi(e) : 8;
    }();
    return v;
}

int32_t build_segments(Ctx& c, const DCsr& A, bool bwd, DBuf<int32_t>& starts, int32_t window = 1) {
    const int32_t n = A.nr;
    DBuf<int32_t> head(static_cast<size_t>(n) + 1, c.s), rank(static_cast<size_t>(n) + 1, c.s);
    launch(c, k_segment_heads, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), bwd, head.get(), window);
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

#include "gs_lanes.cuh"

}  // namespace

// The forward-sweep plan of a matrix: which sync-free kernel relaxes its k columns, and
// its segments.  In order of preference:
//   kCta      fewer than 1024 rows, the iterate fits one SM and the pattern is
//             structurally symmetric: values handed over in shared memory;
//   kLanes    lane per segment (gs_lanes.cuh): one column, rows of at most 9 entries
//             (the 8-term records), segments of 16 rows on average, 32 per resident CTA;
//   kSegWarp  warp per segment (k_gs_seg_warp): any row or segment length, every warp
//             resident (C5: level 1 194 -> 12 ms, level 3 9.5 -> 3.2 ms);
//   kCta      as above for larger levels that still fit.
// Segments use a block-size window, so the stride-m chains of interleaved vector
// unknowns continue a segment.  Host synchronisations happen here; the run
// (gs_lanes_run) has none, so it may be queued on another stream than the plan's.
// rows beyond 32 entries run the warp-per-segment kernel with two entries per lane, so that
// rows of up to 64 are one pipelined chunk (AMGCU_GS_SW_WIDE=0: always one entry per lane)
static bool seg_warp_wide(int32_t longest_row) {
    const char* e = std::getenv("AMGCU_GS_SW_WIDE");
    return longest_row > 32 && !(e && e[0] == '0');
}

LanePlan lane_plan(Ctx& c, const DCsr& A, int nsw, int k) {
    LanePlan pl;
    const int32_t n = A.nr;
    if (n == 0 || nsw == 0 || k > kMaxK || std::getenv("AMGCU_GS_TRACE")) return pl;
    if (n >= (1 << 24) || static_cast<int64_t>(nsw) * n * k >= (int64_t(1) << 31)) return pl;
    const char* cta_env = std::getenv("AMGCU_GS_CTA");  // "0": off (read per call: tests toggle it)
    const bool cta_fits = !(cta_env && cta_env[0] == '0') && gs_cta_smem(n, k) <= kGsCtaSmem;
    auto try_cta = [&] {
        DBuf<int32_t> flag(1, c.s);
        AMG_CK(cudaMemsetAsync(flag.get(), 0, sizeof(int32_t), c.s));
        launch(c, k_pattern_asym, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), flag.get());
        if (read_scalar(c, flag.get())) return false;
        pl.kind = LanePlan::kCta;
        pl.ok = true;
        return true;
    };
    // the smallest levels: one SM holds everything and hands values over in shared memory
    if (cta_fits && n < kGsCtaMaxRows && try_cta()) return pl;
    DBuf<int32_t> st(2, c.s);
    AMG_CK(cudaMemsetAsync(st.get(), 0, 2 * sizeof(int32_t), c.s));
    launch(c, k_bandwidth, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), st.get());
    pl.nf = build_segments(c, A, false, pl.segf, std::max(A.bs, 1));
    stage_scalar(c, 1, st.get() + 1);
    sync(c);
    pl.longest_row = staged<int32_t>(c, 1);
    const char* ln_env = std::getenv("AMGCU_GS_LANES");
    const char* sw_env = std::getenv("AMGCU_GS_SEGWARP");
    const bool lanes_off = ln_env && ln_env[0] == '0', sw_off = sw_env && sw_env[0] == '0';
    if (!lanes_off && k == 1 && pl.longest_row <= 9 && (pl.nf + kLnLanes - 1) / kLnLanes <= c.sms &&
        static_cast<int64_t>(pl.nf) * kSegWarpMinLen <= n) {
        pl.kind = LanePlan::kLanes;
        pl.ok = true;
        return pl;
    }
    // warp per segment: any segment length (short segments only mean more warps), as
    // long as every warp can be resident at once
    if (!sw_off && k <= 4) {
        int per_sm = 0;  // of the variant that will run (gs_segwarp_kernel_run)
        const bool wide = seg_warp_wide(pl.longest_row);
        auto occ = [&](auto kern) {
            AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSwWarps * 32, 0));
        };
        switch (k) {
            case 1: wide ? occ(k_gs_seg_warp<1, 2>) : occ(k_gs_seg_warp<1, 1>); break;
            case 2: wide ? occ(k_gs_seg_warp<2, 2>) : occ(k_gs_seg_warp<2, 1>); break;
            case 3: wide ? occ(k_gs_seg_warp<3, 2>) : occ(k_gs_seg_warp<3, 1>); break;
            default: wide ? occ(k_gs_seg_warp<4, 2>) : occ(k_gs_seg_warp<4, 1>); break;
        }
        if ((pl.nf + kSwWarps - 1) / kSwWarps <= static_cast<int64_t>(per_sm) * c.sms) {
            pl.kind = LanePlan::kSegWarp;
            pl.ok = true;
            return pl;
        }
    }
    if (cta_fits && n >= kGsCtaMaxRows) try_cta();
    return pl;
}

// Forward sweeps of k columns (n x k column-major x, b) by the lane-per-segment kernel
// (gs_lanes.cuh).  The columns are independent sweeps of the same matrix (the reference
// relaxes each candidate column in turn, interpolation.hpp:91); one launch runs as many
// columns side by side as keep every CTA resident (32 segments per CTA, one CTA per SM).
void gs_lanes_kernel_run(Ctx& c, const DCsr& A, const LanePlan& pl, const double* inv_diag, double* x,
                         const double* b, int nsw, int32_t k) {
    const int32_t n = A.nr;
    const int32_t nf = pl.nf, longest_row = pl.longest_row;
    const int32_t nctas = (nf + kLnLanes - 1) / kLnLanes;
    const int32_t group = std::max<int32_t>(1, std::min<int32_t>(k, c.sms / std::max<int32_t>(1, nctas)));
    const DBuf<int32_t>& segf = pl.segf;
    const size_t stride = static_cast<size_t>(n);
    const size_t cstride = stride * (nsw + 1);
    DBuf<double> X(cstride * group, c.s);
    DBuf<unsigned int> ticket(1, c.s);
    const double bytes = nsw * (12.0 * A.nnz + 4.0 * (n + 1) + 8.0 * n + 16.0 * n);
    // AMGCU_GS_STATS=1: solver iteration / stall counters on stderr
    static const bool want_stats = std::getenv("AMGCU_GS_STATS") != nullptr;
    DBuf<unsigned long long> st;
    for (int32_t c0 = 0; c0 < k; c0 += group) {
        const int32_t g = std::min(group, k - c0);
        for (int32_t j = 0; j < g; ++j) {
            copy_d2d(c, X.get() + cstride * j, x + stride * (c0 + j), static_cast<int64_t>(stride));
            launch(c, k_fill_pending, blocks_for(static_cast<int64_t>(stride) * nsw, 256), 256, 0,
                   static_cast<int64_t>(stride) * nsw, X.get() + cstride * j + stride);
        }
        AMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned int), c.s));
        if (want_stats) {
            st.alloc(32, c.s);
            AMG_CK(cudaMemsetAsync(st.get(), 0, 32 * sizeof(unsigned long long), c.s));
            AMG_CK(cudaMemsetAsync(st.get() + 24, 0xff, sizeof(unsigned long long), c.s));
        }
        const double* bg = b ? b + stride * c0 : nullptr;
        auto runl = [&](auto kern, size_t smem) {
            AMG_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            launch_prof(c, kProfGaussSeidel, bytes * g, kern, static_cast<unsigned>(nctas * g), kLnThreads, smem, n,
                        A.rp.get(), A.ci.get(), A.va.get(), inv_diag, bg, nsw, static_cast<const int32_t*>(segf.get()),
                        nf, X.get(), ticket.get(), st.get(), gs_env_u("AMGCU_GS_POLL_NS", 128u),
                        gs_env_u("AMGCU_GS_PF_NS", 128u), g, cstride);
        };
        if (longest_row <= 9) runl(k_gs_lanes<8, 3, 4, 64>, ln_smem_bytes<8, 3, 4, 64>());
        else runl(k_gs_lanes<20, 2, 2, 32>, ln_smem_bytes<20, 2, 2, 32>());
        for (int32_t j = 0; j < g; ++j)
            copy_d2d(c, x + stride * (c0 + j), X.get() + cstride * j + stride * nsw, static_cast<int64_t>(stride));
        if (want_stats) {
            unsigned long long h[32];
            copy_d2h(c, h, st.get(), 32);
            sync(c);
            std::fprintf(stderr, "[gs lanes] n=%d segs=%d ctas=%d columns=%d iterations(all ctas)=%llu rows=%llu "
                         "lane-iters=%llu record-stalls=%llu value-stalls=%llu\n", n, nf, nctas, g, h[0], h[1], h[2],
                         h[3], h[2] - h[1] - h[3]);
            const double it = static_cast<double>(h[0]);
            std::fprintf(stderr, "[gs lanes] cycles/iteration: rows %.0f sync %.0f publish %.0f total %.0f\n",
                         h[16] / it, h[17] / it, h[18] / it, h[19] / it);
            std::fprintf(stderr, "[gs lanes] solver span %.1f us, max iterations per CTA %llu, max cycles per CTA %llu\n",
                         (h[25] - h[24]) * 1e-3, h[26], h[27]);
        }
    }
}

// The single-CTA shared-memory kernel (k_gs_cta): levels whose iterate fits on one SM
// and whose pattern is structurally symmetric (checked by the caller).
void gs_cta_kernel_run(Ctx& c, const DCsr& A, const double* inv_diag, double* x, const double* b, int k, int nsw,
                       bool symmetric_sweep) {
    const int32_t n = A.nr;
    const size_t smem = gs_cta_smem(n, k);
    std::vector<unsigned char> hb(nsw);
    for (int s = 0; s < nsw; ++s) hb[s] = symmetric_sweep ? static_cast<unsigned char>(s & 1) : 0;
    DBuf<unsigned char> bwd(static_cast<size_t>(nsw), c.s);
    copy_h2d(c, bwd.get(), hb.data(), nsw);
    const double bytes = nsw * (12.0 * A.nnz + 4.0 * (n + 1) + 8.0 * n + 16.0 * n * k);
    auto run = [&](auto kern) {
        AMG_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        launch_prof(c, kProfGaussSeidel, bytes, kern, 1, kCtaWarps * 32, smem, n, A.rp.get(), A.ci.get(), A.va.get(),
                    inv_diag, b, nsw, static_cast<const unsigned char*>(bwd.get()), x, gs_env_u("AMGCU_GS_CTA_NS", 32u));
    };
    switch (k) {
        case 1: run(k_gs_cta<1>); break;
        case 2: run(k_gs_cta<2>); break;
        case 3: run(k_gs_cta<3>); break;
        case 4: run(k_gs_cta<4>); break;
        case 5: run(k_gs_cta<5>); break;
        case 6: run(k_gs_cta<6>); break;
        case 7: run(k_gs_cta<7>); break;
        default: run(k_gs_cta<8>); break;
    }
}

// Warp-per-segment forward sweeps (k_gs_seg_warp) of the k columns.
void gs_segwarp_kernel_run(Ctx& c, const DCsr& A, const LanePlan& pl, const double* inv_diag, double* x,
                           const double* b, int nsw, int32_t k) {
    const int32_t n = A.nr;
    const size_t stride = static_cast<size_t>(n) * k;
    DBuf<double> X(stride * (nsw + 1), c.s);
    copy_d2d(c, X.get(), x, static_cast<int64_t>(stride));
    launch(c, k_fill_pending, blocks_for(static_cast<int64_t>(stride) * nsw, 256), 256, 0,
           static_cast<int64_t>(stride) * nsw, X.get() + stride);
    DBuf<unsigned int> ticket(1, c.s);
    AMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned int), c.s));
    const double bytes = nsw * (12.0 * A.nnz + 4.0 * (n + 1) + 8.0 * n + 16.0 * n * k);
    const unsigned nctas = static_cast<unsigned>((pl.nf + kSwWarps - 1) / kSwWarps);
    auto runs = [&](auto kern) {
        launch_prof(c, kProfGaussSeidel, bytes, kern, nctas, kSwWarps * 32, 0, n, A.rp.get(), A.ci.get(), A.va.get(),
                    inv_diag, b, nsw, static_cast<const int32_t*>(pl.segf.get()), pl.nf, X.get(), ticket.get(),
                    gs_env_u("AMGCU_GS_SW_NS", 64u));
    };
    // rows beyond 32 entries: two entries per lane, so that rows of up to 64 are one pipelined chunk
    const bool wide = seg_warp_wide(pl.longest_row);
    switch (k) {
        case 1: wide ? runs(k_gs_seg_warp<1, 2>) : runs(k_gs_seg_warp<1, 1>); break;
        case 2: wide ? runs(k_gs_seg_warp<2, 2>) : runs(k_gs_seg_warp<2, 1>); break;
        case 3: wide ? runs(k_gs_seg_warp<3, 2>) : runs(k_gs_seg_warp<3, 1>); break;
        default: wide ? runs(k_gs_seg_warp<4, 2>) : runs(k_gs_seg_warp<4, 1>); break;
    }
    copy_d2d(c, x, X.get() + stride * nsw, static_cast<int64_t>(stride));
}

void gs_lanes_run(Ctx& c, const DCsr& A, const LanePlan& pl, const double* inv_diag, double* x, const double* b,
                  int nsw, int32_t k) {
    switch (pl.kind) {
        case LanePlan::kCta: gs_cta_kernel_run(c, A, inv_diag, x, b, k, nsw, false); return;
        case LanePlan::kLanes: gs_lanes_kernel_run(c, A, pl, inv_diag, x, b, nsw, k); return;
        case LanePlan::kSegWarp: gs_segwarp_kernel_run(c, A, pl, inv_diag, x, b, nsw, k); return;
        default: throw std::logic_error("gauss_seidel: no forward-sweep plan");
    }
}

// the symmetric sweeps' use of the single-CTA kernel (the forward plan covers the rest)
bool gs_cta_sym(Ctx& c, const DCsr& A, const double* inv_diag, double* x, const double* b, int k, int nsw) {
    const char* e = std::getenv("AMGCU_GS_CTA");
    if ((e && e[0] == '0') || gs_cta_smem(A.nr, k) > kGsCtaSmem || std::getenv("AMGCU_GS_TRACE")) return false;
    DBuf<int32_t> flag(1, c.s);
    AMG_CK(cudaMemsetAsync(flag.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_pattern_asym, blocks_for(A.nr, 256), 256, 0, A.nr, A.rp.get(), A.ci.get(), flag.get());
    if (read_scalar(c, flag.get())) return false;
    gs_cta_kernel_run(c, A, inv_diag, x, b, k, nsw, true);
    return true;
}

void gauss_seidel(Ctx& c, const DCsr& A, const double* inv_diag, double* x, const double* b, int k, int sweeps,
                  bool symmetric_sweep) {
    if (k > kMaxK) throw InvalidArgument("relax: at most 8 candidate columns on the GPU path");
    const int32_t n = A.nr;
    const int nsw = symmetric_sweep ? 2 * sweeps : sweeps;
    if (nsw == 0 || n == 0) return;
    if (symmetric_sweep) {
        if (gs_cta_sym(c, A, inv_diag, x, b, k, nsw)) return;
    } else {
        const LanePlan pl = lane_plan(c, A, nsw, k);
        if (pl.ok) {
            // the columns are independent sweeps (the reference relaxes each candidate
            // column in turn, interpolation.hpp:91): side by side in one launch
            gs_lanes_run(c, A, pl, inv_diag, x, b, nsw, k);
            return;
        }
    }
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
    // short segments (coarse levels): warp per row
    const int32_t nseg_max = std::max(nf, nb);
    // AMGCU_GS_WARPROWS=1 forces the warp-per-row kernel (comparison runs)
    const char* wr_env = std::getenv("AMGCU_GS_WARPROWS");
    const bool force_wr = wr_env && wr_env[0] == '1';
    // the segment kernel's poll lists hold 32-bit offsets into the sweep buffers
    const bool huge = stride * (nsw + 1) >= (size_t(1) << 32);
    // rows longer than the segment kernel's 32-entry records (dense coarse operators of
    // vector problems) would all take its rolled slow path: warp per row instead
    int32_t longest_row0 = 0;
    {
        DBuf<int32_t> st(2, c.s);
        AMG_CK(cudaMemsetAsync(st.get(), 0, 2 * sizeof(int32_t), c.s));
        launch(c, k_bandwidth, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), st.get());
        longest_row0 = read_scalar(c, st.get() + 1);
    }
    if ((force_wr || huge || longest_row0 > 32 || static_cast<int64_t>(nseg_max) * kShortSegment > n) &&
        !std::getenv("AMGCU_GS_TRACE")) {
        const double bytes = nsw * (12.0 * A.nnz + 4.0 * (n + 1) + 8.0 * n + 16.0 * n * k);
        // forward sweeps whose stale dependencies stay within the resident window: row-major
        bool row_major = false;
        if (!symmetric_sweep && nsw > 1) {
            DBuf<int32_t> bwd_max(2, c.s);
            AMG_CK(cudaMemsetAsync(bwd_max.get(), 0, 2 * sizeof(int32_t), c.s));
            launch(c, k_bandwidth, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), bwd_max.get());
            const int32_t bwidth = read_scalar(c, bwd_max.get());
            int per_sm = 0;
            AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gs_warp_rows<1, true>, kWrWarps * 32, 0));
            const int64_t resident_warps = static_cast<int64_t>(per_sm) * c.sms * kWrWarps;
            row_major = 2 * static_cast<int64_t>(bwidth) + 2 * kWrWarps < resident_warps;
            // AMGCU_GS_ROWMAJOR=0/1 overrides (comparison runs)
            if (const char* e = std::getenv("AMGCU_GS_ROWMAJOR")) row_major = e[0] == '1';
        }
        const int64_t items = row_major ? n : static_cast<int64_t>(nsw) * n;
        const unsigned grid = static_cast<unsigned>((items + kWrWarps - 1) / kWrWarps);
        auto runw = [&](auto kern) {
            launch_prof(c, kProfGaussSeidel, bytes, kern, grid, kWrWarps * 32, 0, n, A.rp.get(), A.ci.get(),
                        A.va.get(), inv_diag, b, nsw, static_cast<const unsigned char*>(bwd.get()), X.get(),
                        ticket.get(), gs_env_u("AMGCU_GS_WR_NS", kWarpRowPollNs));
        };
#define AMGCU_WR(KK) (row_major ? runw(k_gs_warp_rows<KK, true>) : runw(k_gs_warp_rows<KK, false>))
        switch (k) {
            case 1: AMGCU_WR(1); break;
            case 2: AMGCU_WR(2); break;
            case 3: AMGCU_WR(3); break;
            case 4: AMGCU_WR(4); break;
            case 5: AMGCU_WR(5); break;
            case 6: AMGCU_WR(6); break;
            case 7: AMGCU_WR(7); break;
            default: AMGCU_WR(8); break;
        }
#undef AMGCU_WR
        copy_d2d(c, x, X.get() + stride * nsw, static_cast<int64_t>(stride));
        sync(c);
        return;
    }
    // AMGCU_GS_TRACE=<file>: per (sweep, block) globaltimer stamps for the timeline tool
    const char* trace_path = std::getenv("AMGCU_GS_TRACE");
    DBuf<unsigned long long> trace;
    if (trace_path) {
        trace.alloc(static_cast<size_t>(nsw) * n * 4, c.s);
        AMG_CK(cudaMemsetAsync(trace.get(), 0, sizeof(unsigned long long) * nsw * n * 4, c.s));
    }
    const double bytes = nsw * (12.0 * A.nnz + 4.0 * (n + 1) + 8.0 * n + 16.0 * n * k);
    // bandwidth and longest row: the record width E and the segment-major test
    int32_t bwidth = 0, longest_row = 0;
    {
        DBuf<int32_t> st(2, c.s);
        AMG_CK(cudaMemsetAsync(st.get(), 0, 2 * sizeof(int32_t), c.s));
        launch(c, k_bandwidth, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), st.get());
        stage_scalar(c, 0, st.get());
        stage_scalar(c, 1, st.get() + 1);
        sync(c);
        bwidth = staged<int32_t>(c, 0);
        longest_row = staged<int32_t>(c, 1);
    }
    auto run = [&](auto kern, int segs, size_t seg_bytes) {
        // AMGCU_GS_SMEM: request at least this much shared memory per CTA (caps CTAs per SM)
        static const size_t smem_floor = [] {
            const char* e = std::getenv("AMGCU_GS_SMEM");
            return e ? static_cast<size_t>(std::atol(e)) : size_t(0);
        }();
        const size_t smem = std::max(seg_bytes * segs, smem_floor);
        if (smem > 48 * 1024)
            AMG_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        // Forward sweeps run segment-major (each segment relaxes all sweeps in turn) when
        // sweep s + 1 of a segment can only wait on segments that are already resident:
        // the ones reached within the bandwidth must lie inside the resident window.
        int sweep_loop = 0;
        const char* sl_env = std::getenv("AMGCU_GS_SWEEP_LOOP");
        if (!symmetric_sweep && nsw > 1 && !(sl_env && sl_env[0] == '0')) {
            std::vector<int32_t> hs(static_cast<size_t>(nf) + 1);
            copy_d2h(c, hs.data(), segf.get(), nf + 1);
            sync(c);
            int64_t ahead = 0;
            for (int32_t g2 = 0; g2 < nf; ++g2) {
                const int64_t reach = static_cast<int64_t>(hs[g2 + 1]) + bwidth;
                const int64_t last = std::upper_bound(hs.begin(), hs.end(), reach) - hs.begin() - 1;
                ahead = std::max<int64_t>(ahead, last - g2);
            }
            int per_sm = 0;
            AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 3 * segs * 32, smem));
            const int64_t resident = static_cast<int64_t>(per_sm) * c.sms * segs;
            sweep_loop = 2 * (ahead + segs) < resident ? 1 : 0;
        }
        const int32_t items = sweep_loop ? nf : base[nsw];
        launch_prof(c, kProfGaussSeidel, bytes, kern, blocks_for(items, segs), 3 * segs * 32, smem, n,
                    A.rp.get(), A.ci.get(), A.va.get(), inv_diag, b, nsw, static_cast<const unsigned char*>(bwd.get()),
                    static_cast<const int32_t*>(dbase.get()), static_cast<const int32_t*>(segf.get()),
                    static_cast<const int32_t*>(symmetric_sweep ? segb.get() : segf.get()), X.get(), ticket.get(),
                    gs_max_ns(), trace.get(), gs_poll_window(), sweep_loop, gs_spin_ns());
    };
#define AMGCU_GS_RUN(KK) run(k_gs_segments<KK, 32>, gs_segs_per_cta<KK, 32>(), gs_seg_bytes<KK, 32>())
    // short rows: 16-entry records, 8 segments per CTA; poll offsets are 32-bit
    const bool narrow = longest_row <= 16;
    switch (k) {
        case 1:
            if (narrow) run(k_gs_segments<1, 16>, gs_segs_per_cta<1, 16>(), gs_seg_bytes<1, 16>());
            else AMGCU_GS_RUN(1);
            break;
        case 2: AMGCU_GS_RUN(2); break;
        case 3: AMGCU_GS_RUN(3); break;
        case 4: AMGCU_GS_RUN(4); break;
        case 5: AMGCU_GS_RUN(5); break;
        case 6: AMGCU_GS_RUN(6); break;
        case 7: AMGCU_GS_RUN(7); break;
        default: AMGCU_GS_RUN(8); break;
    }
#undef AMGCU_GS_RUN
    copy_d2d(c, x, X.get() + stride * nsw, static_cast<int64_t>(stride));
    sync(c);
    if (trace_path) {
        std::vector<unsigned long long> ht(static_cast<size_t>(nsw) * n * 4);
        std::vector<int32_t> hs(static_cast<size_t>(nf) + 1);
        AMG_CK(cudaMemcpy(ht.data(), trace.get(), ht.size() * 8, cudaMemcpyDeviceToHost));
        AMG_CK(cudaMemcpy(hs.data(), segf.get(), hs.size() * 4, cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen(trace_path, "ab")) {
            const int32_t hdr[3] = {n, nsw, nf};
            std::fwrite(hdr, 4, 3, f);
            std::fwrite(hs.data(), 4, hs.size(), f);
            std::fwrite(ht.data(), 8, ht.size(), f);
            std::fclose(f);
        }
    }
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
