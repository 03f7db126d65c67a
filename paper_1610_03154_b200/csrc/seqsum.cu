// Global sums in the reference's exact order, in one launch (seqsum.cuh has the
// arithmetic and its proof; tests/cpp/seqsum_fuzz.cpp emulates this kernel).
//
// Every BLAS-1 reduction on the setup and solve path -- dot, nrm2, the MGS axpy+dot,
// the PCG update+norm -- is `double s = 0.0; for (i) s += t[i];` in the reference
// (sparse.hpp:309-313, cycle.hpp:190-194, spectral.hpp:47-51).  One launch per sum:
//
//   tile (4096 terms, 256 threads x 16): the terms are produced (and a fused update
//     written) with coalesced loads into shared memory; each thread's approximate
//     starting sum comes from a block scan plus a decoupled look-back over the tiles'
//     (sum, |sum|) aggregates; every thread simulates the exact chain over its 16 terms
//     from there (two parity chains, seqsum.cuh) into a list of pieces and raw
//     elements; a shared-memory tree merges the 256 lists into the tile's list.
//   group (256 tiles): the last tile of a group to finish merges the group's lists.
//   final: the last group merges the group lists, whose first piece is the exact
//     chain from +0.0, and applies the result: *out = the reference's bits.
//
// HBM traffic is the operands once (16 B per term for a dot), plus ~1.2 KB of list per
// tile.  Tickets order the tiles so the look-back only waits on running blocks.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ops.cuh"
#include "seqsum.cuh"

namespace amgcu {

namespace {

using ss::Item;

constexpr int kSsThreads = 256;
// terms per thread: 8 (2048-term tiles) for sums of up to kSsIpt16From terms, 16 above
// (fewer tiles, fewer waves; 2.1M terms: 114 vs 124 us, 234K: 88 vs 113 us)
constexpr int64_t kSsIpt16From = 1500000;
constexpr int kSsThreadCap = 4;   // items per thread list
constexpr int kSsTileCap = 16;    // items per tile list (global)
constexpr int kSsGroupTiles = 64;   // tiles per group merge (groups merge in parallel)
constexpr int kSsGroupCap = 64;   // items per group list (global)
// thread list regions: kSsThreadCap items + one 8-byte word, an odd number of words, so
// the lanes of a warp touch distinct banks when each works on its own list
constexpr int kSsRegion = kSsThreadCap * static_cast<int>(sizeof(Item)) + 8;
constexpr int kSsPool = kSsThreads * kSsRegion / static_cast<int>(sizeof(Item));  // items, group merges
template <int IPT>
struct SsCfg {
    static constexpr int kTile = kSsThreads * IPT;
    static constexpr int kStage = kTile + kTile / 16;  // staged terms, one pad slot per 16
    static constexpr size_t kSmem = static_cast<size_t>(kSsThreads) * kSsRegion + sizeof(double) * kStage;
};

struct TileStatus {
    double agg_s, agg_a, inc_s, inc_a;
    int flag;  // 0 none, 1 aggregate, 2 inclusive prefix
    int pad;
};

struct SsWs {
    unsigned int* counters;  // [0] tile ticket, [1] groups done, [2 + g] tiles done in group g
    TileStatus* status;
    Item* tile_lists;
    int32_t* tile_len;
    Item* group_lists;
    int32_t* group_len;
    long long* trace;  // AMGCU_SS_TRACE=1: %globaltimer stamps per tile and merge phase
};

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// padded so a lane's 16 consecutive terms and the warp's coalesced row both avoid conflicts
__device__ __forceinline__ int stage_idx(int j) { return j + (j >> 4); }

// ---- term producers --------------------------------------------------------------
// load(i): the term, performing the fused update exactly once; recompute(i): the term
// again from the updated operands (raw elements re-simulated after the tile is gone).
struct TDot {
    const double* x;
    const double* y;
    __device__ bool skip() const { return false; }
    __device__ double load(int64_t i) const { return __ldg(x + i) * __ldg(y + i); }
    __device__ double recompute(int64_t i) const { return __ldcg(x + i) * __ldcg(y + i); }
};

// y += sign * (*alpha) * x; term = y_new * z (z null: y_new * y_new)   (axpy then dot)
struct TAxpyDot {
    const double* alpha;
    double sign;
    const double* x;
    double* y;
    const double* z;
    __device__ bool skip() const { return false; }
    __device__ double load(int64_t i) const {
        const double a = sign * (*alpha);
        const double yi = y[i] + a * __ldg(x + i);
        y[i] = yi;
        return yi * (z ? __ldg(z + i) : yi);
    }
    __device__ double recompute(int64_t i) const {
        const double yi = __ldcg(y + i);
        return yi * (z ? __ldcg(z + i) : yi);
    }
};

// PCG (cycle.hpp:190-194): x += a p, r -= a q (a = st[2]), term = r_new^2; skipped when *bad
struct TPcg {
    const double* st;
    const int32_t* bad;
    const double* p;
    const double* q;
    double* x;
    double* r;
    __device__ bool skip() const { return *bad != 0; }
    __device__ double load(int64_t i) const {
        const double a = st[2];
        x[i] = x[i] + a * __ldg(p + i);
        const double ri = r[i] + (-a) * __ldg(q + i);
        r[i] = ri;
        return ri * ri;
    }
    __device__ double recompute(int64_t i) const {
        const double ri = __ldcg(r + i);
        return ri * ri;
    }
};

struct StageTerm {
    const double* tv;
    int64_t base;
    __device__ double operator()(int64_t i) const { return tv[stage_idx(static_cast<int>(i - base))]; }
};
template <class Term>
struct GlobalTerm {
    Term t;
    unsigned long long* ctr;  // AMGCU_SS_TRACE: terms re-read from global memory
    __device__ double operator()(int64_t i) const {
        if (ctr) atomicAdd(ctr, 1ull);
        return t.recompute(i);
    }
};

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ double vloadd(const double* p) { return *reinterpret_cast<const volatile double*>(p); }

// Merge `count` lists (lens[j] items at lists + j * stride) into pool[0 .. return);
// block-cooperative: windows of up to 256 lists are loaded into the pool behind the
// accumulated list, tree-merged, then appended to it.
template <class TermAt>
__device__ int merge_from_global(Item* pool, const Item* lists, const int32_t* lens, int count, int stride,
                                 int acc_cap, const TermAt& term, int* s_off, int* s_len, int* s_misc) {
    const int tid = threadIdx.x;
    int acc = 0;
    int idx = 0;
    while (idx < count) {
        // the window: lengths loaded in parallel, offsets by thread 0 from shared memory
        s_len[tid] = idx + tid < count ? __ldcg(lens + idx + tid) : 0;
        __syncthreads();
        if (tid == 0) {
            int at = acc, m = 0;
            while (idx + m < count && m < kSsThreads) {
                const int l = s_len[m];
                if (at + l > kSsPool) break;
                s_off[m] = at;
                at += l;
                ++m;
            }
            s_misc[0] = m;
        }
        __syncthreads();
        const int m = s_misc[0];
        if (tid < m) {
            const Item* src = lists + static_cast<int64_t>(idx + tid) * stride;
            const double* ps = reinterpret_cast<const double*>(src);
            double* pd = reinterpret_cast<double*>(pool + s_off[tid]);
            constexpr int kWords = static_cast<int>(sizeof(Item) / 8);
            const int nwords = s_len[tid] * kWords;
            if (nwords >= kWords) {  // the first item's words in flight together (most lists hold one)
                double v[kWords];
#pragma unroll
                for (int w = 0; w < kWords; ++w) v[w] = __ldcg(ps + w);
#pragma unroll
                for (int w = 0; w < kWords; ++w) pd[w] = v[w];
            }
            for (int w = kWords; w < nwords; ++w) pd[w] = __ldcg(ps + w);
        }
        __syncthreads();
        for (int step = 1; step < m; step <<= 1) {
            if ((tid % (2 * step)) == 0 && tid + step < m)
                s_len[tid] = ss::merge_pair(pool, s_off[tid], s_len[tid], s_off[tid + step], s_len[tid + step], term);
            __syncthreads();
        }
        if (tid == 0) {
            int a = ss::merge_pair(pool, 0, acc, s_off[0], s_len[0], term);
            s_misc[1] = ss::truncate(pool, a, acc_cap);
        }
        __syncthreads();
        acc = s_misc[1];
        idx += m;
        __syncthreads();
    }
    return acc;
}

template <class Term, int IPT>
__global__ void __launch_bounds__(kSsThreads, 2)
    k_seqsum(Term term, int64_t n, int64_t ntiles, SsWs ws, double* __restrict__ out, bool take_sqrt) {
    extern __shared__ __align__(16) unsigned char ss_smem[];
    Item* pool = reinterpret_cast<Item*>(ss_smem);
    auto region = [&](int t) { return reinterpret_cast<Item*>(ss_smem + static_cast<size_t>(t) * kSsRegion); };
    double* tv = reinterpret_cast<double*>(ss_smem + static_cast<size_t>(kSsThreads) * kSsRegion);
    __shared__ int s_len[kSsThreads];
    __shared__ int s_off[kSsThreads];
    __shared__ int s_misc[4];
    __shared__ double s_ws[kSsThreads / 32], s_wa[kSsThreads / 32];
    __shared__ double s_P, s_A;
    __shared__ long long s_tile;

    if (term.skip()) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = static_cast<long long>(atomicAdd(ws.counters, 1u));
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * SsCfg<IPT>::kTile;
    long long* tr = ws.trace ? ws.trace + tile * 12 : nullptr;
    const long long c_start = clock64();
    if (tr && tid == 0) tr[0] = gtimer();

    // terms, coalesced: warp w stages [w*512, w*512 + 512) of the tile
    for (int k = 0; k < IPT; ++k) {
        const int j = warp * (32 * IPT) + k * 32 + lane;
        const int64_t i = base + j;
        tv[stage_idx(j)] = i < n ? term.load(i) : 0.0;
    }
    __syncthreads();

    // approximate running sums (any order): the thread's sum and |sum|, block scan
    const int64_t i0 = std::min<int64_t>(n, base + static_cast<int64_t>(tid) * IPT);
    const int64_t i1 = std::min<int64_t>(n, i0 + IPT);
    double ts = 0.0, ta = 0.0;
    for (int k = 0; k < IPT; ++k) {
        const double t = tv[stage_idx(tid * IPT + k)];
        ts += t;
        ta += fabs(t);
    }
    double is = ts, ia = ta;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double ys = __shfl_up_sync(0xffffffffu, is, off);
        const double ya = __shfl_up_sync(0xffffffffu, ia, off);
        if (lane >= off) {
            is += ys;
            ia += ya;
        }
    }
    if (lane == 31) {
        s_ws[warp] = is;
        s_wa[warp] = ia;
    }
    __syncthreads();
    if (warp == 0) {
        double vs = lane < kSsThreads / 32 ? s_ws[lane] : 0.0;
        double va = lane < kSsThreads / 32 ? s_wa[lane] : 0.0;
        const double ts_ = vs, ta_ = va;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double ys = __shfl_up_sync(0xffffffffu, vs, off);
            const double ya = __shfl_up_sync(0xffffffffu, va, off);
            if (lane >= off) {
                vs += ys;
                va += ya;
            }
        }
        const double tot_s = __shfl_sync(0xffffffffu, vs, 31);
        const double tot_a = __shfl_sync(0xffffffffu, va, 31);
        if (lane < kSsThreads / 32) {
            s_ws[lane] = vs - ts_;  // exclusive warp offsets
            s_wa[lane] = va - ta_;
        }
        // tile aggregate, then the look-back for the tiles before it
        TileStatus* st = ws.status + tile;
        if (lane == 0) {
            if (tile == 0) {
                st->inc_s = tot_s;
                st->inc_a = tot_a;
                __threadfence();
                *reinterpret_cast<volatile int*>(&st->flag) = 2;
            } else {
                st->agg_s = tot_s;
                st->agg_a = tot_a;
                __threadfence();
                *reinterpret_cast<volatile int*>(&st->flag) = 1;
            }
        }
        double ps = 0.0, pa = 0.0;
        if (tile > 0) {
            int64_t j = tile - 1;
            while (true) {
                const int64_t jj = j - lane;
                int f = 2;
                double vs2 = 0.0, va2 = 0.0;
                if (jj >= 0) {
                    const TileStatus* sj = ws.status + jj;
                    do {
                        f = vload(&sj->flag);
                    } while (f == 0);
                    __threadfence();
                    vs2 = f == 2 ? vloadd(&sj->inc_s) : vloadd(&sj->agg_s);
                    va2 = f == 2 ? vloadd(&sj->inc_a) : vloadd(&sj->agg_a);
                }
                const unsigned m = __ballot_sync(0xffffffffu, f == 2);
                const int first = m ? __ffs(m) - 1 : 32;
                if (lane > first) {
                    vs2 = 0.0;
                    va2 = 0.0;
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    vs2 += __shfl_xor_sync(0xffffffffu, vs2, off);
                    va2 += __shfl_xor_sync(0xffffffffu, va2, off);
                }
                ps += vs2;
                pa += va2;
                if (m) break;
                j -= 32;
            }
            if (lane == 0) {
                st->inc_s = ps + tot_s;
                st->inc_a = pa + tot_a;
                __threadfence();
                *reinterpret_cast<volatile int*>(&st->flag) = 2;
            }
        }
        if (lane == 0) {
            s_P = ps;
            s_A = pa;
        }
    }
    __syncthreads();
    if (tr && tid == 0) tr[1] = gtimer();

    // each thread simulates its terms from its approximate start
    const StageTerm sterm{tv, base};
    {
        const double rep = s_P + (s_ws[warp] + (is - ts));
        const double tau = ldexp(s_A + (s_wa[warp] + (ia - ta)) + ta, -36);
        ss::Out o{region(tid), 0, kSsThreadCap};
        if (i1 > i0) ss::simulate(o, rep, i0 == 0, i0, i1, tau, sterm);
        s_len[tid] = o.n;
    }
    __syncthreads();
    if (tr && tid == 0) {
        tr[2] = gtimer();
        tr[8] = clock64() - c_start;
    }
    for (int step = 1, lv = 0; step < kSsThreads; step <<= 1, ++lv) {
        const long long c0 = clock64();
        if ((tid & (2 * step - 1)) == 0)
            s_len[tid] = ss::merge_ptr(region(tid), s_len[tid], region(tid + step), s_len[tid + step], sterm);
        if (ws.trace && tile == 0 && tid == 0) {
            ws.trace[ntiles * 12 + 2 + lv] = clock64() - c0;
            ws.trace[ntiles * 12 + 10 + lv] = s_len[step] * 100 + s_len[0];
        }
        __syncthreads();
    }
    if (tid == 0) s_misc[0] = ss::truncate(pool, s_len[0], kSsTileCap);
    __syncthreads();
    if (tr && tid == 0) {
        tr[3] = gtimer();
        tr[4] = s_len[0];
    }
    {
        const int L = s_misc[0];
        Item* dst = ws.tile_lists + tile * kSsTileCap;
        for (int k = tid; k < L; k += kSsThreads) dst[k] = pool[k];
        if (tid == 0) ws.tile_len[tile] = L;
    }
    __threadfence();
    __syncthreads();

    // group: the last tile to finish merges the group's lists
    const int64_t group = tile / kSsGroupTiles;
    const int64_t ngroups = (ntiles + kSsGroupTiles - 1) / kSsGroupTiles;
    const int gtiles = static_cast<int>(std::min<int64_t>(kSsGroupTiles, ntiles - group * kSsGroupTiles));
    if (tid == 0) s_misc[2] = atomicAdd(ws.counters + 2 + group, 1u) == static_cast<unsigned>(gtiles - 1);
    __syncthreads();
    if (!s_misc[2]) return;
    __threadfence();
    if (tr && tid == 0) tr[5] = gtimer();
    const GlobalTerm<Term> gterm{term, ws.trace ? reinterpret_cast<unsigned long long*>(ws.trace + ntiles * 12 + 18) : nullptr};
    {
        const int L = merge_from_global(pool, ws.tile_lists + group * kSsGroupTiles * kSsTileCap,
                                        ws.tile_len + group * kSsGroupTiles, gtiles, kSsTileCap, kSsGroupCap, gterm,
                                        s_off, s_len, s_misc);
        Item* dst = ws.group_lists + group * kSsGroupCap;
        for (int k = tid; k < L; k += kSsThreads) dst[k] = pool[k];
        if (tid == 0) ws.group_len[group] = L;
        if (tr && tid == 0) {
            tr[6] = gtimer();
            tr[7] = L;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_misc[2] = atomicAdd(ws.counters + 1, 1u) == static_cast<unsigned>(ngroups - 1);
    __syncthreads();
    if (!s_misc[2]) return;
    __threadfence();
    const int L = merge_from_global(pool, ws.group_lists, ws.group_len, static_cast<int>(ngroups), kSsGroupCap,
                                    kSsPool / 2, gterm, s_off, s_len, s_misc);
    if (tid == 0) {
        const double s = ss::apply(pool, L, 0.0, gterm, static_cast<int64_t*>(nullptr));
        if (ws.trace) {
            ws.trace[ntiles * 12] = gtimer();
            ws.trace[ntiles * 12 + 1] = L;
        }
        *out = take_sqrt ? sqrt(s) : s;
        ws.counters[0] = 0u;
        ws.counters[1] = 0u;
    }
    // reset for the next launch on this stream
    for (int64_t k = tid; k < ngroups; k += kSsThreads) ws.counters[2 + k] = 0u;
    for (int64_t k = tid; k < ntiles; k += kSsThreads) ws.status[k].flag = 0;
}

// Short sums: the whole block stages the terms (performing any fused update once), then
// one thread runs the reference's loop itself, eight staged terms in registers ahead of
// the add chain.  Below the crossover (kSsSmallN) this beats the tile machinery, whose
// latency does not shrink with n.
constexpr int kSsSmallThreads = 1024;
constexpr int kSsSmallN = 8192;  // the single chain costs ~4.3 ns per term; the tiles ~35 us

template <class Term>
__global__ void __launch_bounds__(kSsSmallThreads)
    k_seqsum_small(Term term, int n, double* __restrict__ out, bool take_sqrt) {
    extern __shared__ __align__(16) unsigned char ss_smem[];
    double* tv = reinterpret_cast<double*>(ss_smem);
    if (term.skip()) return;
    for (int i = threadIdx.x; i < n; i += kSsSmallThreads) tv[i] = term.load(i);
    __syncthreads();
    if (threadIdx.x != 0) return;
    double s = 0.0;
    int i = 0;
    for (; i + 8 <= n; i += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = tv[i + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) s += v[k];
    }
    for (; i < n; ++i) s += tv[i];
    *out = take_sqrt ? sqrt(s) : s;
}

template <class Term>
void launch_seqsum(Ctx& c, const Term& term, int64_t n, double* out, bool take_sqrt, double bytes) {
    static const int64_t small_n = [] {
        const char* e = std::getenv("AMGCU_SS_SMALL_N");
        return e ? std::atoll(e) : static_cast<int64_t>(kSsSmallN);
    }();
    if (n > 0 && n <= small_n && n <= kSsSmallN) {
        static bool attr_small = false;
        if (!attr_small) {
            for (const void* k : {reinterpret_cast<const void*>(k_seqsum_small<TDot>),
                                  reinterpret_cast<const void*>(k_seqsum_small<TAxpyDot>),
                                  reinterpret_cast<const void*>(k_seqsum_small<TPcg>)})
                AMG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(sizeof(double) * kSsSmallN)));
            attr_small = true;
        }
        launch_prof(c, c.blas_family, bytes, k_seqsum_small<Term>, 1, kSsSmallThreads, sizeof(double) * n, term,
                    static_cast<int>(n), out, take_sqrt);
        return;
    }
    if (n <= 0) {
        // the reference's empty sum: +0.0 (sqrt(+0) = +0)
        AMG_CK(cudaMemsetAsync(out, 0, sizeof(double), c.s));
        return;
    }
    const bool ipt16 = n > kSsIpt16From;
    const int64_t tile_terms = ipt16 ? SsCfg<16>::kTile : SsCfg<8>::kTile;
    const int64_t ntiles = (n + tile_terms - 1) / tile_terms;
    const int64_t ngroups = (ntiles + kSsGroupTiles - 1) / kSsGroupTiles;
    SeqSumWs& w = c.ssws[c.s == c.main_s ? 0 : 1];
    if (w.tiles < ntiles) {
        const int64_t t = std::max<int64_t>(ntiles, 256);
        const int64_t g = (t + kSsGroupTiles - 1) / kSsGroupTiles;
        w.counters.alloc(static_cast<size_t>(2 + g), c.s);
        w.status.alloc(sizeof(TileStatus) * static_cast<size_t>(t), c.s);
        w.lists.alloc(sizeof(Item) * static_cast<size_t>(t * kSsTileCap + g * kSsGroupCap), c.s);
        w.lens.alloc(static_cast<size_t>(t + g), c.s);
        AMG_CK(cudaMemsetAsync(w.counters.get(), 0, sizeof(unsigned int) * (2 + g), c.s));
        AMG_CK(cudaMemsetAsync(w.status.get(), 0, sizeof(TileStatus) * t, c.s));
        w.tiles = t;
    }
    const int64_t gcap = (w.tiles + kSsGroupTiles - 1) / kSsGroupTiles;
    SsWs ws;
    ws.counters = w.counters.get();
    ws.status = reinterpret_cast<TileStatus*>(w.status.get());
    ws.tile_lists = reinterpret_cast<Item*>(w.lists.get());
    ws.group_lists = ws.tile_lists + w.tiles * kSsTileCap;
    ws.tile_len = w.lens.get();
    ws.group_len = w.lens.get() + w.tiles;
    (void)gcap;
    (void)ngroups;
    static bool attr = false;
    if (!attr) {
        for (const void* k : {reinterpret_cast<const void*>(k_seqsum<TDot, 8>), reinterpret_cast<const void*>(k_seqsum<TAxpyDot, 8>),
                              reinterpret_cast<const void*>(k_seqsum<TPcg, 8>)})
            AMG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SsCfg<8>::kSmem)));
        for (const void* k : {reinterpret_cast<const void*>(k_seqsum<TDot, 16>), reinterpret_cast<const void*>(k_seqsum<TAxpyDot, 16>),
                              reinterpret_cast<const void*>(k_seqsum<TPcg, 16>)})
            AMG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SsCfg<16>::kSmem)));
        attr = true;
    }
    static const bool trace = [] {
        const char* e = std::getenv("AMGCU_SS_TRACE");
        return e && e[0] == '1';
    }();
    ws.trace = nullptr;
    DBuf<long long> tbuf;
    if (trace) {
        tbuf.alloc(static_cast<size_t>(ntiles * 12 + 20), c.s);
        AMG_CK(cudaMemsetAsync(tbuf.get(), 0, sizeof(long long) * (ntiles * 12 + 20), c.s));
        ws.trace = tbuf.get();
    }
    if (ipt16)
        launch_prof(c, c.blas_family, bytes, k_seqsum<Term, 16>, static_cast<unsigned>(ntiles), kSsThreads,
                    SsCfg<16>::kSmem, term, n, ntiles, ws, out, take_sqrt);
    else
        launch_prof(c, c.blas_family, bytes, k_seqsum<Term, 8>, static_cast<unsigned>(ntiles), kSsThreads,
                    SsCfg<8>::kSmem, term, n, ntiles, ws, out, take_sqrt);
    if (trace) {
        std::vector<long long> h(static_cast<size_t>(ntiles * 12 + 20));
        copy_d2h(c, h.data(), tbuf.get(), static_cast<int64_t>(h.size()));
        sync(c);
        long long t0 = h[0], tile_end = 0;
        double lb = 0, sim = 0, tree = 0, items = 0, cyc = 0;
        for (int64_t t = 0; t < ntiles; ++t) {
            const long long* r = h.data() + t * 12;
            cyc += static_cast<double>(r[8]);
            t0 = std::min(t0, r[0]);
            tile_end = std::max(tile_end, r[3]);
            lb += r[1] - r[0];
            sim += r[2] - r[1];
            tree += r[3] - r[2];
            items += static_cast<double>(r[4]);
        }
        long long g0 = LLONG_MAX, g1 = 0;
        for (int64_t t = 0; t < ntiles; ++t)
            if (h[t * 12 + 5]) {
                g0 = std::min(g0, h[t * 12 + 5]);
                g1 = std::max(g1, h[t * 12 + 6]);
            }
        std::fprintf(stderr,
                     "[seqsum] n %lld tiles %lld | per tile (ns): load+scan+lookback %.0f sim %.0f tree %.0f items %.2f | "
                     "span: tiles %lld groups %lld..%lld final %lld (ns from first tile), final items %lld | "
                     "SM MHz during load+sim %.0f\n",
                     static_cast<long long>(n), static_cast<long long>(ntiles), lb / ntiles, sim / ntiles, tree / ntiles,
                     items / ntiles, tile_end - t0, g0 - t0, g1 - t0, h[ntiles * 12] - t0, h[ntiles * 12 + 1],
                     cyc / (lb + sim) * 1e3);
        long long glen = 0, ngr = 0, maxlen = 0;
        for (int64_t t = 0; t < ntiles; ++t) {
            maxlen = std::max(maxlen, h[t * 12 + 4]);
            if (h[t * 12 + 5]) {
                glen += h[t * 12 + 7];
                ++ngr;
            }
        }
        std::fprintf(stderr, "[seqsum] global term re-reads %lld, tile list max %lld, group lists %lld (total items %lld)\n",
                     h[ntiles * 12 + 18], maxlen, ngr, glen);
        std::fprintf(stderr, "[seqsum] tile 0 tree levels (cycles, lenR*100+lenL):");
        for (int lv = 0; lv < 8; ++lv) std::fprintf(stderr, " %lld(%lld)", h[ntiles * 12 + 2 + lv], h[ntiles * 12 + 10 + lv]);
        std::fprintf(stderr, "\n");
    }
}

}  // namespace

void seqsum_dot(Ctx& c, const double* x, const double* y, int64_t n, double* out, bool take_sqrt) {
    launch_seqsum(c, TDot{x, y}, n, out, take_sqrt, (x == y ? 8.0 : 16.0) * n);
}

void seqsum_axpy_dot(Ctx& c, const double* alpha, double sign, const double* x, double* y, const double* z, int64_t n,
                     double* out, bool take_sqrt) {
    launch_seqsum(c, TAxpyDot{alpha, sign, x, y, z}, n, out, take_sqrt, (z ? 32.0 : 24.0) * n);
}

void seqsum_pcg_update_nrm(Ctx& c, const double* st, const int32_t* bad, const double* p, const double* q, double* x,
                           double* r, int64_t n, double* out) {
    launch_seqsum(c, TPcg{st, bad, p, q, x, r}, n, out, true, 56.0 * n);
}

}  // namespace amgcu
