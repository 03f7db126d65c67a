// Sparse core kernels: SpMV, deterministic transpose, SpGEMM, filter,
// symmetry test, diagonal, pattern compaction.  Reference: core/sparse.hpp.
#include <cub/block/block_reduce.cuh>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>

#include "ops.cuh"

namespace amgcu {

namespace {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------------
// SpMV: one thread per row, CSR order (sparse.hpp:145-150).  The solve phase uses
// the sliced-ELL variant in cycle.cu; this one serves setup (Arnoldi, checks).
// ---------------------------------------------------------------------------------
__global__ void k_spmv(int32_t nr, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ va, const double* __restrict__ x, double* __restrict__ y) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    double s = 0.0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) s += va[p] * x[ci[p]];
    y[i] = s;
}

// ---------------------------------------------------------------------------------
// Transpose: count -> scan -> atomic scatter -> per-column rank sort by source
// position (keys unique), which restores the ascending-row order of sparse.hpp:169-177.
// ---------------------------------------------------------------------------------
__global__ void k_col_count(int64_t nnz, const int32_t* __restrict__ ci, int32_t* __restrict__ cnt) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < nnz) atomicAdd(&cnt[ci[p]], 1);
}

__global__ void k_scatter_positions(int32_t nr, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                    const int32_t* __restrict__ colptr, int32_t* __restrict__ cursor,
                                    int32_t* __restrict__ pos_tmp) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = ci[p];
        const int32_t slot = colptr[j] + atomicAdd(&cursor[j], 1);
        pos_tmp[slot] = p;
    }
}

// warp per segment: rank = #keys smaller (keys unique) -> sorted positions
__global__ void k_segment_rank_sort(int32_t nseg, const int32_t* __restrict__ segptr, const int32_t* __restrict__ in,
                                    int32_t* __restrict__ out) {
    const int32_t seg = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    if (seg >= nseg) return;
    const int32_t lo = segptr[seg], hi = segptr[seg + 1], len = hi - lo;
    if (len == 1) {
        if (lane == 0) out[lo] = in[lo];
        return;
    }
    for (int32_t e0 = 0; e0 < len; e0 += kWarp) {
        const int32_t e = e0 + lane;
        const int32_t key = e < len ? in[lo + e] : INT_MAX;
        int32_t rank = 0;
        for (int32_t c0 = 0; c0 < len; c0 += kWarp) {
            const int32_t other = (c0 + lane) < len ? in[lo + c0 + lane] : INT_MAX;
            const int cnt = min(kWarp, len - c0);
            for (int t = 0; t < cnt; ++t) {
                const int32_t o = __shfl_sync(0xffffffffu, other, t);
                rank += (o < key) ? 1 : 0;
            }
        }
        if (e < len) out[lo + rank] = key;
    }
}

__global__ void k_rows_of_entries(int32_t nr, const int32_t* __restrict__ rp, int32_t* __restrict__ rows) {
    const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    if (i >= nr) return;
    for (int32_t p = rp[i] + lane; p < rp[i + 1]; p += kWarp) rows[p] = i;
}

__global__ void k_gather_transpose(int64_t nnz, const int32_t* __restrict__ pos, const int32_t* __restrict__ rows,
                                   const double* __restrict__ va, int32_t* __restrict__ tci, double* __restrict__ tva) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    const int32_t p = pos[q];
    tci[q] = rows[p];
    tva[q] = va[p];
}

// ---------------------------------------------------------------------------------
// SpGEMM (sparse.hpp:183-217).  Products are expanded in the reference order
// (A-row entry t, then B-row entry q); key = (col << 32) | seq; a bitonic sort by
// key groups each output column with its contributions still in sequence order,
// and one lane sums each group from 0.0 in that order.  Exact zeros are dropped.
// Rows with up to kSmallCap products: one warp, shared memory.  Larger rows:
// one block over a global scratch region.
// ---------------------------------------------------------------------------------
constexpr int kSmallCap = 512;
constexpr int kSortCap = 64;  // rows up to this many products: the sort kernel

__global__ void k_product_count(int32_t nr, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                                const int32_t* __restrict__ brp, int64_t* __restrict__ np) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    int64_t s = 0;
    for (int32_t p = arp[i]; p < arp[i + 1]; ++p) {
        const int32_t t = aci[p];
        s += brp[t + 1] - brp[t];
    }
    np[i] = s;
}

__global__ void k_collect_big(int32_t nr, const int64_t* __restrict__ np, int32_t* __restrict__ list,
                              int32_t* __restrict__ count) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    if (np[i] > kSortCap) list[atomicAdd(count, 1)] = i;
}

__device__ __forceinline__ unsigned next_pow2(unsigned v) {
    v--;
    v |= v >> 1;
    v |= v >> 2;
    v |= v >> 4;
    v |= v >> 8;
    v |= v >> 16;
    return v + 1;
}

// expand row i of A*B into keys/vals (shared or global), cooperative over a group of `gsize` threads
__device__ __forceinline__ void expand_row(int32_t i, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                                           const double* __restrict__ ava, const int32_t* __restrict__ brp,
                                           const int32_t* __restrict__ bci, const double* __restrict__ bva,
                                           unsigned long long* keys, double* vals, int tid, int gsize) {
    int64_t base = 0;
    for (int32_t p = arp[i]; p < arp[i + 1]; ++p) {
        const int32_t t = aci[p];
        const double a = ava[p];
        const int32_t lo = brp[t], len = brp[t + 1] - lo;
        for (int32_t q = tid; q < len; q += gsize) {
            const int64_t seq = base + q;
            keys[seq] = (static_cast<unsigned long long>(static_cast<uint32_t>(bci[lo + q])) << 32) |
                        static_cast<unsigned long long>(seq);
            vals[seq] = a * bva[lo + q];
        }
        base += len;
    }
}

constexpr int kGemmWarps = 8;

// Warp-cooperative expansion: lanes take A entries (32 at a time), a warp scan
// of their B-row lengths gives each product's sequence number, and each lane
// writes its B row's products -- the A-entry loop is no longer a chain of
// dependent loads.
__device__ __forceinline__ void expand_row_warp(int32_t i, const int32_t* __restrict__ arp,
                                                const int32_t* __restrict__ aci, const double* __restrict__ ava,
                                                const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                                const double* __restrict__ bva, unsigned long long* keys, double* vals,
                                                int lane) {
    const int32_t alo = arp[i], ahi = arp[i + 1];
    int64_t base = 0;
    for (int32_t p0 = alo; p0 < ahi; p0 += kWarp) {
        const int32_t p = p0 + lane;
        int32_t lo = 0, len = 0;
        double a = 0.0;
        if (p < ahi) {
            const int32_t t = aci[p];
            a = ava[p];
            lo = brp[t];
            len = brp[t + 1] - lo;
        }
        int32_t incl = len;
        for (int off = 1; off < kWarp; off <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        const int64_t my = base + incl - len;
        for (int32_t q = 0; q < len; ++q) {
            const int64_t seq = my + q;
            keys[seq] = (static_cast<unsigned long long>(static_cast<uint32_t>(__ldg(&bci[lo + q]))) << 32) |
                        static_cast<unsigned long long>(seq);
            vals[seq] = a * __ldg(&bva[lo + q]);
        }
        base += __shfl_sync(0xffffffffu, incl, kWarp - 1);
    }
}

// rows with at most kSortCap products: warp bitonic sort of (column, sequence) keys
__global__ void __launch_bounds__(kGemmWarps * kWarp)
    k_spgemm_small(int32_t nr, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                   const double* __restrict__ ava, const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                   const double* __restrict__ bva, const int64_t* __restrict__ poff, int32_t* __restrict__ tcol,
                   double* __restrict__ tval, int32_t* __restrict__ cnt) {
    __shared__ unsigned long long skeys[kGemmWarps][kSortCap];
    __shared__ double svals[kGemmWarps][kSortCap];
    const int w = threadIdx.x / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    const int32_t i = blockIdx.x * kGemmWarps + w;
    if (i >= nr) return;
    const int64_t np = poff[i + 1] - poff[i];
    if (np > kSortCap) return;  // handled by the hash / block kernels
    if (np == 0) {
        if (lane == 0) cnt[i] = 0;
        return;
    }
    unsigned long long* keys = skeys[w];
    double* vals = svals[w];
    expand_row_warp(i, arp, aci, ava, brp, bci, bva, keys, vals, lane);
    const unsigned n2 = max(next_pow2(static_cast<unsigned>(np)), 2u);
    for (unsigned e = static_cast<unsigned>(np) + lane; e < n2; e += kWarp) keys[e] = ~0ull;
    __syncwarp();
    // bitonic sort, ascending
    for (unsigned k = 2; k <= n2; k <<= 1) {
        for (unsigned j = k >> 1; j > 0; j >>= 1) {
            for (unsigned e = lane; e < n2 / 2; e += kWarp) {
                const unsigned lo = 2 * e - (e & (j - 1));
                const unsigned hi = lo + j;
                const bool up = ((lo & k) == 0);
                const unsigned long long a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncwarp();
        }
    }
    // ordered segment sums; compacted write in column order
    int32_t written = 0;
    int32_t* ocol = tcol + poff[i];
    double* oval = tval + poff[i];
    for (int32_t e0 = 0; e0 < np; e0 += kWarp) {
        const int32_t e = e0 + lane;
        bool emit = false;
        uint32_t col = 0;
        double acc = 0.0;
        if (e < np) {
            const unsigned long long key = keys[e];
            col = static_cast<uint32_t>(key >> 32);
            const bool start = (e == 0) || (static_cast<uint32_t>(keys[e - 1] >> 32) != col);
            if (start) {
                for (int32_t r = e; r < np; ++r) {
                    const unsigned long long kr = keys[r];
                    if (static_cast<uint32_t>(kr >> 32) != col) break;
                    acc += vals[static_cast<uint32_t>(kr & 0xffffffffull)];
                }
                emit = (acc != 0.0);
            }
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, emit);
        if (emit) {
            const int32_t at = written + __popc(ballot & ((1u << lane) - 1u));
            ocol[at] = static_cast<int32_t>(col);
            oval[at] = acc;
        }
        written += __popc(ballot);
    }
    if (lane == 0) cnt[i] = written;
}

// Hash accumulation, sort of the distinct columns only.  Products are staged
// in sequence order and consumed 32 at a time: each lane finds its column's
// slot (open addressing, atomicCAS on the key), lanes of one column are grouped
// with __match_any_sync and the lowest one adds the group's products into the
// slot in lane order -- chunks in order, lanes in order: every column's sum is
// the reference's sequential one, starting from 0.0.  The non-zero sums are
// then compacted and only those D <= np entries are bitonic-sorted by column.
constexpr int kHashWarps = 4;
constexpr int kHashSlots = 2 * kSmallCap;  // load factor <= 1/2

template <int CAP>
struct HashSharedT {
    int32_t hkey[2 * CAP];
    double hval[2 * CAP];
    int32_t pcol[CAP];  // staged products: column
    double pval[CAP];   // staged products: value; reused as the sort keys
    double chunk[kWarp];
};
using HashShared = HashSharedT<kSmallCap>;
constexpr int kMidCap = 2048;  // rows of 512..2048 products: one warp per block, 72 KB of shared memory

__device__ __forceinline__ uint32_t col_hash(int32_t col, uint32_t mask) {
    return (static_cast<uint32_t>(col) * 2654435761u) & mask;
}

// CAP products per row at most, W warps (rows) per block, rows of more than MINNP
// products; `list` (optional) names the rows (block b, warp w: list[b * W + w])
template <int CAP, int W, int MINNP>
__global__ void __launch_bounds__(W * kWarp)
    k_spgemm_hash(int32_t nr, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                  const double* __restrict__ ava, const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                  const double* __restrict__ bva, const int64_t* __restrict__ poff, int32_t* __restrict__ tcol,
                  double* __restrict__ tval, int32_t* __restrict__ cnt, const int32_t* __restrict__ list) {
    extern __shared__ unsigned long long hsm[];
    const int w = threadIdx.x / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    const int32_t slot_id = blockIdx.x * W + w;
    if (slot_id >= nr) return;
    const int32_t i = list ? list[slot_id] : slot_id;
    const int64_t np = poff[i + 1] - poff[i];
    if (np > CAP || np <= MINNP) return;  // handled by the block / sort kernels
    HashSharedT<CAP>& sh = reinterpret_cast<HashSharedT<CAP>*>(hsm)[w];
    // table sized to the row: a power of two >= 2 np (load factor <= 1/2)
    const int32_t hs = static_cast<int32_t>(max(64u, next_pow2(2u * static_cast<unsigned>(np))));
    const uint32_t hmask = static_cast<uint32_t>(hs - 1);
    for (int e = lane; e < hs; e += kWarp) {
        sh.hkey[e] = -1;
        sh.hval[e] = 0.0;
    }
    // stage the products in sequence order (warp-cooperative expansion)
    {
        const int32_t alo = arp[i], ahi = arp[i + 1];
        int32_t base = 0;
        for (int32_t p0 = alo; p0 < ahi; p0 += kWarp) {
            const int32_t p = p0 + lane;
            int32_t lo = 0, len = 0;
            double a = 0.0;
            if (p < ahi) {
                const int32_t t = aci[p];
                a = ava[p];
                lo = brp[t];
                len = brp[t + 1] - lo;
            }
            int32_t incl = len;
            for (int off = 1; off < kWarp; off <<= 1) {
                const int32_t v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += v;
            }
            const int32_t my = base + incl - len;
            for (int32_t q = 0; q < len; ++q) {
                sh.pcol[my + q] = __ldg(&bci[lo + q]);
                sh.pval[my + q] = a * __ldg(&bva[lo + q]);
            }
            base += __shfl_sync(0xffffffffu, incl, kWarp - 1);
        }
    }
    __syncwarp();
    // ordered accumulation, 32 products at a time
    const int32_t npi = static_cast<int32_t>(np);
    for (int32_t c0 = 0; c0 < npi; c0 += kWarp) {
        const int32_t e = c0 + lane;
        const bool act = e < npi;
        const unsigned am = __ballot_sync(0xffffffffu, act);
        int32_t slot = -1;
        if (act) {
            const int32_t col = sh.pcol[e];
            uint32_t h = col_hash(col, hmask);
            while (true) {
                const int32_t k = atomicCAS(&sh.hkey[h], -1, col);
                if (k == -1 || k == col) break;
                h = (h + 1) & hmask;
            }
            slot = static_cast<int32_t>(h);
            sh.chunk[lane] = sh.pval[e];
        }
        __syncwarp();
        if (act) {
            const unsigned grp = __match_any_sync(am, slot);
            if (lane == __ffs(grp) - 1) {
                double v = sh.hval[slot];
                for (unsigned g = grp; g; g &= g - 1) v += sh.chunk[__ffs(g) - 1];
                sh.hval[slot] = v;
            }
        }
        __syncwarp();
    }
    // compact the non-zero sums (key = column << 32 | slot) into the staging area
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(sh.pval);
    int32_t d = 0;
    for (int32_t e0 = 0; e0 < hs; e0 += kWarp) {
        const int32_t e = e0 + lane;
        const int32_t col = sh.hkey[e];
        const bool keep = col >= 0 && sh.hval[e] != 0.0;
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (keep)
            keys[d + __popc(b & ((1u << lane) - 1u))] =
                (static_cast<unsigned long long>(static_cast<uint32_t>(col)) << 32) | static_cast<uint32_t>(e);
        d += __popc(b);
    }
    __syncwarp();
    if (d > 1) {
        const unsigned n2 = next_pow2(static_cast<unsigned>(d));
        for (unsigned e = static_cast<unsigned>(d) + lane; e < n2; e += kWarp) keys[e] = ~0ull;
        __syncwarp();
        for (unsigned k = 2; k <= n2; k <<= 1) {
            for (unsigned j = k >> 1; j > 0; j >>= 1) {
                for (unsigned e = lane; e < n2 / 2; e += kWarp) {
                    const unsigned lo = 2 * e - (e & (j - 1));
                    const unsigned hi = lo + j;
                    const bool up = ((lo & k) == 0);
                    const unsigned long long a = keys[lo], b = keys[hi];
                    if ((a > b) == up) {
                        keys[lo] = b;
                        keys[hi] = a;
                    }
                }
                __syncwarp();
            }
        }
    }
    int32_t* ocol = tcol + poff[i];
    double* oval = tval + poff[i];
    for (int32_t e = lane; e < d; e += kWarp) {
        const unsigned long long k = keys[e];
        ocol[e] = static_cast<int32_t>(k >> 32);
        oval[e] = sh.hval[static_cast<uint32_t>(k & 0xffffffffull)];
    }
    if (lane == 0) cnt[i] = d;
}

constexpr int kBigThreads = 512;

__global__ void __launch_bounds__(kBigThreads)
    k_spgemm_big(const int32_t* __restrict__ list, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                 const double* __restrict__ ava, const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                 const double* __restrict__ bva, const int64_t* __restrict__ poff,
                 const int64_t* __restrict__ scratch_off, unsigned long long* __restrict__ gkeys,
                 double* __restrict__ gvals, int32_t* __restrict__ tcol, double* __restrict__ tval,
                 int32_t* __restrict__ cnt, const int32_t* __restrict__ handled) {
    if (handled[blockIdx.x]) return;  // k_spgemm_big_hash wrote the row
    const int32_t i = list[blockIdx.x];
    const int64_t np = poff[i + 1] - poff[i];
    unsigned long long* keys = gkeys + scratch_off[blockIdx.x];
    double* vals = gvals + poff[i];
    expand_row(i, arp, aci, ava, brp, bci, bva, keys, vals, threadIdx.x, blockDim.x);
    int64_t n2 = 1;
    while (n2 < np) n2 <<= 1;
    for (int64_t e = np + threadIdx.x; e < n2; e += blockDim.x) keys[e] = ~0ull;
    __syncthreads();
    for (int64_t k = 2; k <= n2; k <<= 1) {
        for (int64_t j = k >> 1; j > 0; j >>= 1) {
            for (int64_t e = threadIdx.x; e < n2 / 2; e += blockDim.x) {
                const int64_t lo = 2 * e - (e & (j - 1));
                const int64_t hi = lo + j;
                const bool up = ((lo & k) == 0);
                const unsigned long long a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    __shared__ int32_t s_written;
    __shared__ int32_t s_warp[kBigThreads / kWarp];
    if (threadIdx.x == 0) s_written = 0;
    __syncthreads();
    const int lane = threadIdx.x & (kWarp - 1), wid = threadIdx.x / kWarp;
    int32_t* ocol = tcol + poff[i];
    double* oval = tval + poff[i];
    for (int64_t e0 = 0; e0 < np; e0 += blockDim.x) {
        const int64_t e = e0 + threadIdx.x;
        bool emit = false;
        uint32_t col = 0;
        double acc = 0.0;
        if (e < np) {
            const unsigned long long key = keys[e];
            col = static_cast<uint32_t>(key >> 32);
            const bool start = (e == 0) || (static_cast<uint32_t>(keys[e - 1] >> 32) != col);
            if (start) {
                for (int64_t r = e; r < np; ++r) {
                    const unsigned long long kr = keys[r];
                    if (static_cast<uint32_t>(kr >> 32) != col) break;
                    acc += vals[static_cast<uint32_t>(kr & 0xffffffffull)];
                }
                emit = (acc != 0.0);
            }
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, emit);
        if (lane == 0) s_warp[wid] = __popc(ballot);
        __syncthreads();
        int32_t before = s_written;
        for (int t = 0; t < wid; ++t) before += s_warp[t];
        if (emit) {
            const int32_t at = before + __popc(ballot & ((1u << lane) - 1u));
            ocol[at] = static_cast<int32_t>(col);
            oval[at] = acc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int32_t tot = 0;
            for (int t = 0; t < static_cast<int>(blockDim.x / kWarp); ++t) tot += s_warp[t];
            s_written += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) cnt[i] = s_written;
}

// Rows beyond the warp kernels whose DISTINCT columns fit a shared-memory table: the
// columns are hashed first, then the A entries are taken one at a time (a block
// barrier between them) and the B row's products are added to their columns' sums.
// A B row holds each column once, so every column's sum is built in expansion order
// -- the (column, position) order the bitonic kernel sums in -- and the result is
// bitwise the same. The table's columns are then sorted and the nonzero sums written.
// Rows with more distinct columns than kBigHashMax are left to the bitonic kernel.
constexpr int kBigHashSlots = 8192;
constexpr int kBigHashMax = 6144;
constexpr int kBigHashMinB = 128;
constexpr size_t kBigHashSmem = kBigHashSlots * (sizeof(int32_t) + sizeof(double)) +
                                kBigHashSlots * sizeof(unsigned long long);

template <bool G, class T>
__device__ __forceinline__ T bh_ld(const T* p) {
    if constexpr (G) return __ldcg(p);  // global tables: other threads' writes, past L1
    else return *p;
}

// G = false: the table is in shared memory (kBigHashSlots slots, rows of at most
// kBigHashMax distinct columns). G = true: rows the shared table refused, with a
// table in global scratch of the next power of two above the row's product count.
template <bool G>
__global__ void __launch_bounds__(kBigThreads)
    k_spgemm_big_hash(const int32_t* __restrict__ list, const int32_t* __restrict__ arp,
                      const int32_t* __restrict__ aci, const double* __restrict__ ava,
                      const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                      const double* __restrict__ bva, const int64_t* __restrict__ poff, int32_t* __restrict__ tcol,
                      double* __restrict__ tval, int32_t* __restrict__ cnt, int32_t* __restrict__ handled,
                      const int64_t* __restrict__ scratch_off, int32_t* gk, double* gv, unsigned long long* gs) {
    extern __shared__ __align__(16) unsigned char big_smem[];
    __shared__ int32_t s_n, s_over;
    __shared__ int32_t s_warp[kBigThreads / kWarp];
    if (G && handled[blockIdx.x]) return;
    const int32_t i = list[blockIdx.x];
    const int tid = threadIdx.x;
    // one block barrier per A entry: rows whose B rows average under kBigHashMinB
    // products would leave most threads idle, so the bitonic kernel takes them
    if (poff[i + 1] - poff[i] < static_cast<int64_t>(kBigHashMinB) * (arp[i + 1] - arp[i])) {
        if (tid == 0) handled[blockIdx.x] = 0;
        return;
    }
    int32_t* hk;
    double* hv;
    unsigned long long* sk;
    int32_t size, maxd, lg;
    if constexpr (G) {
        const int64_t np = poff[i + 1] - poff[i];
        size = 1;
        lg = 0;
        while (size < np) {
            size <<= 1;
            ++lg;
        }
        maxd = size;
        hk = gk + scratch_off[blockIdx.x];
        hv = gv + scratch_off[blockIdx.x];
        sk = gs + scratch_off[blockIdx.x];
    } else {
        size = kBigHashSlots;
        lg = 13;
        maxd = kBigHashMax;
        hv = reinterpret_cast<double*>(big_smem);
        sk = reinterpret_cast<unsigned long long*>(hv + kBigHashSlots);
        hk = reinterpret_cast<int32_t*>(sk + kBigHashSlots);
    }
    const uint32_t mask = static_cast<uint32_t>(size) - 1u;
    // the shared table refuses a row early (long probe chains or too many columns);
    // the global one is sized to the row and probes to the end
    const int32_t probe_cap = G ? size : 128;
    auto slot = [&](int32_t col) { return (static_cast<uint32_t>(col) * 2654435761u) >> (32 - lg); };
    for (int e = tid; e < size; e += kBigThreads) {
        hk[e] = -1;
        hv[e] = 0.0;
    }
    if (tid == 0) {
        s_n = 0;
        s_over = 0;
    }
    __syncthreads();
    const int32_t alo = arp[i], ahi = arp[i + 1];
    // distinct columns
    for (int32_t p = alo; p < ahi; ++p) {
        const int32_t t = aci[p];
        bool over = false;
        for (int32_t q = brp[t] + tid; q < brp[t + 1] && !over; q += kBigThreads) {
            if (*reinterpret_cast<volatile int32_t*>(&s_over)) break;  // another thread refused the row
            const int32_t col = bci[q];
            uint32_t h = slot(col);
            for (int32_t probe = 0;;) {
                const int32_t k = bh_ld<G>(hk + h);
                if (k == col) break;
                if (k == -1) {
                    const int32_t old = atomicCAS(&hk[h], -1, col);
                    if (old == -1) {
                        over = atomicAdd(&s_n, 1) >= maxd;
                        break;
                    }
                    if (old == col) break;
                }
                h = (h + 1) & mask;
                if (++probe == probe_cap) {
                    over = true;
                    break;
                }
            }
            if (over) s_over = 1;
        }
        if (__syncthreads_or(over)) {
            if (tid == 0) handled[blockIdx.x] = 0;
            return;
        }
    }
    // sums in expansion order, one A entry at a time
    for (int32_t p = alo; p < ahi; ++p) {
        const int32_t t = aci[p];
        const double a = ava[p];
        for (int32_t q = brp[t] + tid; q < brp[t + 1]; q += kBigThreads) {
            const int32_t col = bci[q];
            uint32_t h = slot(col);
            while (bh_ld<G>(hk + h) != col) h = (h + 1) & mask;
            hv[h] = __dadd_rn(bh_ld<G>(hv + h), __dmul_rn(a, bva[q]));
        }
        __syncthreads();
    }
    // compact the occupied slots as (column, slot) keys and sort them
    const int32_t d = s_n;
    int32_t n2 = 1;
    while (n2 < d) n2 <<= 1;
    __syncthreads();
    if (tid == 0) s_n = 0;
    __syncthreads();
    for (int e = tid; e < size; e += kBigThreads) {
        const int32_t k = bh_ld<G>(hk + e);
        if (k != -1) {
            const int32_t at = atomicAdd(&s_n, 1);
            sk[at] = (static_cast<unsigned long long>(static_cast<uint32_t>(k)) << 32) | static_cast<uint32_t>(e);
        }
    }
    for (int e = d + tid; e < n2; e += kBigThreads) sk[e] = ~0ull;
    __syncthreads();
    for (int32_t k = 2; k <= n2; k <<= 1)
        for (int32_t j = k >> 1; j > 0; j >>= 1) {
            for (int32_t e = tid; e < n2 / 2; e += kBigThreads) {
                const int32_t lo = 2 * e - (e & (j - 1));
                const int32_t hi = lo + j;
                const bool up = ((lo & k) == 0);
                const unsigned long long x = bh_ld<G>(sk + lo), y = bh_ld<G>(sk + hi);
                if ((x > y) == up) {
                    sk[lo] = y;
                    sk[hi] = x;
                }
            }
            __syncthreads();
        }
    // nonzero sums in column order
    const int lane = tid & (kWarp - 1), wid = tid / kWarp;
    int32_t* ocol = tcol + poff[i];
    double* oval = tval + poff[i];
    int32_t written = 0;
    for (int32_t e0 = 0; e0 < d; e0 += kBigThreads) {
        const int32_t e = e0 + tid;
        double acc = 0.0;
        bool emit = false;
        if (e < d) {
            acc = bh_ld<G>(hv + static_cast<uint32_t>(bh_ld<G>(sk + e) & 0xffffffffull));
            emit = acc != 0.0;
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, emit);
        if (lane == 0) s_warp[wid] = __popc(ballot);
        __syncthreads();
        int32_t before = written;
        for (int w = 0; w < wid; ++w) before += s_warp[w];
        if (emit) {
            const int32_t at = before + __popc(ballot & ((1u << lane) - 1u));
            ocol[at] = static_cast<int32_t>(bh_ld<G>(sk + e) >> 32);
            oval[at] = acc;
        }
        for (int w = 0; w < kBigThreads / kWarp; ++w) written += s_warp[w];
        __syncthreads();
    }
    if (tid == 0) {
        cnt[i] = written;
        handled[blockIdx.x] = 1;
    }
}

__global__ void k_copy_rows(int32_t nr, const int64_t* __restrict__ poff, const int32_t* __restrict__ tcol,
                            const double* __restrict__ tval, const int32_t* __restrict__ crp, int32_t* __restrict__ cci,
                            double* __restrict__ cva) {
    const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    if (i >= nr) return;
    const int64_t src = poff[i];
    const int32_t dst = crp[i], len = crp[i + 1] - dst;
    for (int32_t e = lane; e < len; e += kWarp) {
        cci[dst + e] = tcol[src + e];
        cva[dst + e] = tval[src + e];
    }
}

// ---------------------------------------------------------------------------------
// filter_matrix (sparse.hpp:236-272), thread per row, two passes.
// ---------------------------------------------------------------------------------
__device__ void filter_thresholds(int32_t i, bool square, const int32_t* rp, const int32_t* ci, const double* va,
                                  bool theta_set, double theta, int32_t k, double* kth_out, double* tmax_out) {
    const int32_t lo = rp[i], hi = rp[i + 1];
    int32_t nm = 0;
    double mx = 0.0;
    bool any = false;
    for (int32_t p = lo; p < hi; ++p) {
        if (square && ci[p] == i) continue;
        const double m = fabs(va[p]);
        mx = any ? (m > mx ? m : mx) : m;
        any = true;
        ++nm;
    }
    double kth = 0.0;
    if (k > 0 && k < nm) {
        // k-th largest magnitude (duplicates counted): the m whose descending
        // rank range [#greater, #greater + #equal) contains k-1
        for (int32_t p = lo; p < hi; ++p) {
            if (square && ci[p] == i) continue;
            const double m = fabs(va[p]);
            int32_t greater = 0, equal = 0;
            for (int32_t q = lo; q < hi; ++q) {
                if (square && ci[q] == i) continue;
                const double o = fabs(va[q]);
                greater += (o > m) ? 1 : 0;
                equal += (o == m) ? 1 : 0;
            }
            if (greater <= k - 1 && k - 1 < greater + equal) {
                kth = m;
                break;
            }
        }
    }
    *kth_out = kth;
    *tmax_out = (theta_set && any) ? theta * mx : 0.0;
}

__device__ __forceinline__ bool filter_keep(int32_t i, int32_t j, double v, bool square, bool theta_set, int32_t k,
                                            double kth, double tmax) {
    const double mag = fabs(v);
    const bool diag = square && j == i;
    const bool keep = diag || ((k <= 0 || mag >= kth) && (!theta_set || mag >= tmax));
    return keep && v != 0.0;
}

__global__ void k_filter_count(int32_t nr, bool square, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const double* __restrict__ va, bool theta_set, double theta, int32_t k,
                               int32_t* __restrict__ cnt) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    double kth, tmax;
    filter_thresholds(i, square, rp, ci, va, theta_set, theta, k, &kth, &tmax);
    int32_t c = 0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) c += filter_keep(i, ci[p], va[p], square, theta_set, k, kth, tmax);
    cnt[i] = c;
}

__global__ void k_filter_write(int32_t nr, bool square, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const double* __restrict__ va, bool theta_set, double theta, int32_t k,
                               const int32_t* __restrict__ frp, int32_t* __restrict__ fci, double* __restrict__ fva) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    double kth, tmax;
    filter_thresholds(i, square, rp, ci, va, theta_set, theta, k, &kth, &tmax);
    int32_t o = frp[i];
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p)
        if (filter_keep(i, ci[p], va[p], square, theta_set, k, kth, tmax)) {
            fci[o] = ci[p];
            fva[o] = va[p];
            ++o;
        }
}

// ---------------------------------------------------------------------------------
// symmetry: for every stored (i, j): |A(i,j) - A(j,i)| <= tol * max|A| (the fast and
// fallback branches of sparse.hpp:288-305 test exactly this set of pairs)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double coeff_at(const int32_t* rp, const int32_t* ci, const double* va, int32_t i, int32_t j) {
    int32_t lo = rp[i], hi = rp[i + 1];
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (ci[mid] < j) lo = mid + 1;
        else hi = mid;
    }
    return (lo < rp[i + 1] && ci[lo] == j) ? va[lo] : 0.0;
}

// bound = tol * max|A| with the maximum read from device memory (k_max_abs's bits): the
// host never needs it, so is_symmetric takes one synchronisation, not two.  A sub-warp of
// LPR lanes per row (1 for short rows; long coarse rows spread their entries -- each a
// binary search in another row -- over 8 or 32 lanes).
template <int LPR>
__global__ void k_asym(int32_t nr, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ va, double tol, const unsigned long long* __restrict__ max_bits,
                       int32_t* __restrict__ bad) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int32_t i = static_cast<int32_t>(t / LPR);
    if (i >= nr) return;
    const double bound = tol * __longlong_as_double(static_cast<long long>(*max_bits));
    for (int32_t p = rp[i] + static_cast<int32_t>(t % LPR); p < rp[i + 1]; p += LPR) {
        const double at = coeff_at(rp, ci, va, ci[p], i);
        if (fabs(va[p] - at) > bound) {
            atomicExch(bad, 1);
            return;
        }
    }
}

__global__ void k_max_abs(int64_t n, const double* __restrict__ v, unsigned long long* __restrict__ out) {
    using BR = cub::BlockReduce<double, 256>;
    __shared__ typename BR::TempStorage tmp;
    double m = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        m = fmax(m, fabs(v[i]));
    const double bm = BR(tmp).Reduce(m, [](double a, double b) { return fmax(a, b); });
    if (threadIdx.x == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(bm)));
}

__global__ void k_diag(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ va, double* __restrict__ d, bool invert, int32_t* __restrict__ bad) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = coeff_at(rp, ci, va, i, i);
    if (invert) {
        if (v == 0.0) atomicMin(bad, i);
        d[i] = 1.0 / v;
    } else {
        d[i] = v;
    }
}

__global__ void k_nonzero_count(int32_t nr, const int32_t* __restrict__ rp, const double* __restrict__ vals,
                                int32_t* __restrict__ cnt) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    int32_t c = 0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) c += vals[p] != 0.0;
    cnt[i] = c;
}

__global__ void k_nonzero_write(int32_t nr, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ vals, const int32_t* __restrict__ orp,
                                int32_t* __restrict__ oci, double* __restrict__ ova) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    int32_t o = orp[i];
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p)
        if (vals[p] != 0.0) {
            oci[o] = ci[p];
            ova[o] = vals[p];
            ++o;
        }
}

}  // namespace

void spmv(Ctx& c, const DCsr& A, const double* x, double* y) {
    launch(c, k_spmv, blocks_for(A.nr, 256), 256, 0, A.nr, A.rp.get(), A.ci.get(), A.va.get(), x, y);
}

void entry_rows(Ctx& c, const DCsr& A, int32_t* rows) {
    launch(c, k_rows_of_entries, blocks_for(static_cast<int64_t>(A.nr) * kWarp, 256), 256, 0, A.nr, A.rp.get(), rows);
}

void transpose_positions(Ctx& c, const DCsr& A, DBuf<int32_t>& colptr, DBuf<int32_t>& pos, DBuf<int32_t>* src_row) {
    DBuf<int32_t> cnt(static_cast<size_t>(A.nc) + 1, c.s);
    AMG_CK(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * (A.nc + 1), c.s));
    launch(c, k_col_count, blocks_for(A.nnz, 256), 256, 0, A.nnz, A.ci.get(), cnt.get());
    colptr.alloc(static_cast<size_t>(A.nc) + 1, c.s);
    exclusive_scan_i32(c, cnt.get(), colptr.get(), A.nc, false);
    AMG_CK(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * (A.nc + 1), c.s));
    DBuf<int32_t> tmp(static_cast<size_t>(A.nnz), c.s);
    launch(c, k_scatter_positions, blocks_for(A.nr, 256), 256, 0, A.nr, A.rp.get(), A.ci.get(),
           static_cast<const int32_t*>(colptr.get()), cnt.get(), tmp.get());
    pos.alloc(static_cast<size_t>(A.nnz), c.s);
    launch(c, k_segment_rank_sort, blocks_for(static_cast<int64_t>(A.nc) * kWarp, 256), 256, 0, A.nc,
           static_cast<const int32_t*>(colptr.get()), static_cast<const int32_t*>(tmp.get()), pos.get());
    if (src_row) {
        src_row->alloc(static_cast<size_t>(A.nnz), c.s);
        entry_rows(c, A, src_row->get());
    }
}

void transpose(Ctx& c, const DCsr& A, DCsr& T) {
    DBuf<int32_t> colptr, pos, rows;
    transpose_positions(c, A, colptr, pos, &rows);
    T.nr = A.nc;
    T.nc = A.nr;
    T.bs = A.bs;
    T.nnz = A.nnz;
    T.rp = std::move(colptr);
    T.ci.alloc(static_cast<size_t>(A.nnz), c.s);
    T.va.alloc(static_cast<size_t>(A.nnz), c.s);
    launch(c, k_gather_transpose, blocks_for(A.nnz, 256), 256, 0, A.nnz, static_cast<const int32_t*>(pos.get()),
           static_cast<const int32_t*>(rows.get()), A.va.get(), T.ci.get(), T.va.get());
}

namespace {
// ---------------------------------------------------------------------------------
// SpGEMM rows of more than kSortCap products whose output columns fall in a window of
// at most kBmWords * 32 (the Galerkin products and patterns of aggregation hierarchies:
// a coarse row's columns are its aggregate's neighbours).  Warp per row, no hashing,
// no sorting:
//   1. window [cmin, cmax] from the first / last column of each B row the row touches;
//   2. symbolic: one bit per output column in a shared bitmap (atomicOr);
//   3. rank of a column = popcount of the bits before it (per-word prefix + popc), so
//      the distinct columns are numbered in ascending order without a sort;
//   4. numeric in the reference's order (sparse.hpp:190-201): A entries in CSR order,
//      each B row's entries by the lanes (distinct columns, so no two lanes share an
//      accumulator), acc[rank] += a * b starting from 0.0, a warp barrier between A
//      entries; bit-identical to the reference's row accumulator;
//   5. the non-zero sums written in column order (exact zeros dropped).
// Rows whose window or distinct count is too large are listed for the hash kernels.
// ---------------------------------------------------------------------------------
constexpr int kBmWords = 256;  // window of 8192 columns
constexpr int kBmAcc = 256;    // distinct output columns held per row (more: the hash kernels)
constexpr int kBmWarps = 8;
struct BmShared {
    uint32_t bits[kBmWords];
    int32_t pre[kBmWords];
    double acc[kBmAcc];
    int32_t at[kWarp], ab0[kWarp], ab1[kWarp];  // a chunk of A entries: column, B row range
    double aa[kWarp];
};

__global__ void __launch_bounds__(kBmWarps * kWarp)
    k_spgemm_bitmap(int32_t nlist, const int32_t* __restrict__ list, const int32_t* __restrict__ arp,
                    const int32_t* __restrict__ aci, const double* __restrict__ ava, const int32_t* __restrict__ brp,
                    const int32_t* __restrict__ bci, const double* __restrict__ bva, const int64_t* __restrict__ poff,
                    int32_t* __restrict__ tcol, double* __restrict__ tval, int32_t* __restrict__ cnt,
                    int32_t* __restrict__ fb, int32_t* __restrict__ fbn) {
    extern __shared__ unsigned long long bm_smem[];
    const int w = threadIdx.x / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    const int32_t slot = blockIdx.x * kBmWarps + w;
    if (slot >= nlist) return;
    BmShared& sh = reinterpret_cast<BmShared*>(bm_smem)[w];
    const int32_t i = list[slot];
    const int32_t alo = arp[i], ahi = arp[i + 1];
    // 1. window
    int32_t cmin = INT_MAX, cmax = -1;
    for (int32_t p = alo + lane; p < ahi; p += kWarp) {
        const int32_t t = __ldg(aci + p);
        const int32_t b0 = __ldg(brp + t), b1 = __ldg(brp + t + 1);
        if (b1 > b0) {
            cmin = min(cmin, __ldg(bci + b0));
            cmax = max(cmax, __ldg(bci + b1 - 1));
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, off));
        cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
    }
    if (cmax < 0) {
        if (lane == 0) cnt[i] = 0;
        return;
    }
    const int32_t width = cmax - cmin + 1;
    if (width > kBmWords * kWarp) {
        if (lane == 0) fb[atomicAdd(fbn, 1)] = i;
        return;
    }
    const int nw = (width + kWarp - 1) / kWarp;
    for (int e = lane; e < kBmWords; e += kWarp) sh.bits[e] = 0u;
    __syncwarp();
    // 2. symbolic
    for (int32_t p0 = alo; p0 < ahi; p0 += kWarp) {
        const int32_t p = p0 + lane;
        if (p < ahi) {
            const int32_t t = __ldg(aci + p);
            sh.ab0[lane] = __ldg(brp + t);
            sh.ab1[lane] = __ldg(brp + t + 1);
        }
        __syncwarp();
        const int m = min(kWarp, ahi - p0);
        for (int u = 0; u < m; ++u) {
            const int32_t q1 = sh.ab1[u];
            for (int32_t q = sh.ab0[u] + lane; q < q1; q += kWarp) {
                const int32_t cc = __ldg(bci + q) - cmin;
                atomicOr(&sh.bits[cc >> 5], 1u << (cc & 31));
            }
        }
        __syncwarp();
    }
    // 3. ranks: lane l owns words [8l, 8l + 8)
    constexpr int kWpl = kBmWords / kWarp;
    int mine = 0;
#pragma unroll
    for (int u = 0; u < kWpl; ++u) mine += __popc(sh.bits[lane * kWpl + u]);
    int incl = mine;
#pragma unroll
    for (int off = 1; off < kWarp; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
    }
    const int D = __shfl_sync(0xffffffffu, incl, kWarp - 1);
    if (D > kBmAcc) {
        if (lane == 0) fb[atomicAdd(fbn, 1)] = i;
        return;
    }
    {
        int r = incl - mine;
#pragma unroll
        for (int u = 0; u < kWpl; ++u) {
            sh.pre[lane * kWpl + u] = r;
            r += __popc(sh.bits[lane * kWpl + u]);
        }
    }
    for (int e = lane; e < D; e += kWarp) sh.acc[e] = 0.0;
    __syncwarp();
    // 4. numeric, A entries in CSR order
    for (int32_t p0 = alo; p0 < ahi; p0 += kWarp) {
        const int32_t p = p0 + lane;
        if (p < ahi) {
            const int32_t t = __ldg(aci + p);
            sh.aa[lane] = __ldg(ava + p);
            sh.ab0[lane] = __ldg(brp + t);
            sh.ab1[lane] = __ldg(brp + t + 1);
        }
        __syncwarp();
        const int m = min(kWarp, ahi - p0);
        for (int u = 0; u < m; ++u) {
            const double a = sh.aa[u];
            const int32_t q1 = sh.ab1[u];
            for (int32_t q = sh.ab0[u] + lane; q < q1; q += kWarp) {
                const int32_t cc = __ldg(bci + q) - cmin;
                const int wd = cc >> 5;
                const int r = sh.pre[wd] + __popc(sh.bits[wd] & ((1u << (cc & 31)) - 1u));
                sh.acc[r] += a * __ldg(bva + q);
            }
            __syncwarp();
        }
    }
    // 5. non-zero sums in column order
    (void)nw;
    int nz = 0;
#pragma unroll
    for (int u = 0; u < kWpl; ++u) {
        const int wd = lane * kWpl + u;
        uint32_t b = sh.bits[wd];
        int r = sh.pre[wd];
        while (b) {
            nz += sh.acc[r] != 0.0 ? 1 : 0;
            ++r;
            b &= b - 1;
        }
    }
    int zin = nz;
#pragma unroll
    for (int off = 1; off < kWarp; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, zin, off);
        if (lane >= off) zin += y;
    }
    const int64_t base = poff[i];
    int o = zin - nz;
#pragma unroll
    for (int u = 0; u < kWpl; ++u) {
        const int wd = lane * kWpl + u;
        uint32_t b = sh.bits[wd];
        int r = sh.pre[wd];
        while (b) {
            const int bit = __ffs(b) - 1;
            const double v = sh.acc[r];
            if (v != 0.0) {
                tcol[base + o] = cmin + wd * kWarp + bit;
                tval[base + o] = v;
                ++o;
            }
            ++r;
            b &= b - 1;
        }
    }
    if (lane == kWarp - 1) cnt[i] = zin;
}

size_t bitmap_smem() {
    static const size_t bytes = [] {
        const size_t b = sizeof(BmShared) * kBmWarps;
        AMG_CK(cudaFuncSetAttribute(k_spgemm_bitmap, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b)));
        return b;
    }();
    return bytes;
}

size_t hash_smem() {
    static const size_t bytes = [] {
        const size_t b = sizeof(HashShared) * kHashWarps;
        AMG_CK(cudaFuncSetAttribute(k_spgemm_hash<kSmallCap, kHashWarps, kSortCap>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b)));
        return b;
    }();
    return bytes;
}
size_t big_hash_smem() {
    static const size_t bytes = [] {
        AMG_CK(cudaFuncSetAttribute(k_spgemm_big_hash<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kBigHashSmem)));
        return kBigHashSmem;
    }();
    return bytes;
}
size_t mid_smem() {
    static const size_t bytes = [] {
        const size_t b = sizeof(HashSharedT<kMidCap>);
        AMG_CK(cudaFuncSetAttribute(k_spgemm_hash<kMidCap, 1, kSmallCap>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(b)));
        return b;
    }();
    return bytes;
}
}  // namespace

// the rows' staged (column, value) lists (at poff, cnt entries each) into canonical CSR
void compact_rows(Ctx& c, int32_t nr, int32_t nc, const DBuf<int64_t>& poff, const DBuf<int32_t>& tcol,
                  const DBuf<double>& tval, DBuf<int32_t>& cnt, DCsr& C) {
    C.nr = nr;
    C.nc = nc;
    C.bs = 1;
    C.rp.alloc(static_cast<size_t>(nr) + 1, c.s);
    const int64_t nnz = exclusive_scan_i32(c, cnt.get(), C.rp.get(), nr);
    C.nnz = nnz;
    C.ci.alloc(static_cast<size_t>(nnz), c.s);
    C.va.alloc(static_cast<size_t>(nnz), c.s);
    launch(c, k_copy_rows, blocks_for(static_cast<int64_t>(nr) * kWarp, 256), 256, 0, nr,
           static_cast<const int64_t*>(poff.get()), static_cast<const int32_t*>(tcol.get()),
           static_cast<const double*>(tval.get()), static_cast<const int32_t*>(C.rp.get()), C.ci.get(), C.va.get());
}

void spgemm(Ctx& c, const DCsr& A, const DCsr& B, DCsr& C, double* ops) {
    if (A.nc != B.nr) throw InvalidArgument("matmul: dimension mismatch");
    const int32_t nr = A.nr;
    DBuf<int64_t> np(static_cast<size_t>(nr) + 1, c.s), poff(static_cast<size_t>(nr) + 1, c.s);
    launch(c, k_product_count, blocks_for(nr, 256), 256, 0, nr, A.rp.get(), A.ci.get(), B.rp.get(), np.get());
    // rows above the sort kernel's capacity are listed now, so the product total and
    // their count come back with one synchronisation
    DBuf<int32_t> big_list(static_cast<size_t>(nr), c.s), big_count(1, c.s);
    AMG_CK(cudaMemsetAsync(big_count.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_collect_big, blocks_for(nr, 256), 256, 0, nr, static_cast<const int64_t*>(np.get()), big_list.get(),
           big_count.get());
    exclusive_scan_i64(c, np.get(), poff.get(), nr, false);
    stage_scalar(c, 0, static_cast<const int64_t*>(poff.get() + nr));
    stage_scalar(c, 1, static_cast<const int32_t*>(big_count.get()));
    sync(c);
    const int64_t total = nr > 0 ? staged<int64_t>(c, 0) : 0;
    const int32_t nlong = staged<int32_t>(c, 1);
    if (ops) *ops = static_cast<double>(total);
    tally(c, static_cast<double>(total));  // matmul's op count (sparse.hpp:195)
    DBuf<int32_t> tcol(static_cast<size_t>(total), c.s), cnt(static_cast<size_t>(nr) + 1, c.s);
    DBuf<double> tval(static_cast<size_t>(total), c.s);
    const double io_bytes = 12.0 * A.nnz + 4.0 * (A.nr + 1) + 12.0 * B.nnz + 4.0 * (B.nr + 1);
    launch_prof(c, kProfSpgemm, io_bytes + 12.0 * static_cast<double>(total) + 4.0 * nr, k_spgemm_small,
                blocks_for(nr, kGemmWarps), kGemmWarps * kWarp, 0, nr, A.rp.get(), A.ci.get(), A.va.get(), B.rp.get(),
                B.ci.get(), B.va.get(), static_cast<const int64_t*>(poff.get()), tcol.get(), tval.get(), cnt.get());
    if (nlong == 0) {
        compact_rows(c, nr, B.nc, poff, tcol, tval, cnt, C);
        return;
    }
    // rows of more than kSortCap products: the bitmap kernel; rows it cannot hold (window
    // or distinct count too large) are listed for the hash kernels
    DBuf<int32_t> fb(static_cast<size_t>(nlong), c.s), fbn(1, c.s);
    AMG_CK(cudaMemsetAsync(fbn.get(), 0, sizeof(int32_t), c.s));
    static const bool bm_on = std::getenv("AMGCU_SPGEMM_NO_BITMAP") == nullptr;
    if (bm_on) {
        launch_prof(c, kProfSpgemm, 0.0, k_spgemm_bitmap, blocks_for(nlong, kBmWarps), kBmWarps * kWarp,
                    bitmap_smem(), nlong, static_cast<const int32_t*>(big_list.get()), A.rp.get(), A.ci.get(),
                    A.va.get(), B.rp.get(), B.ci.get(), B.va.get(), static_cast<const int64_t*>(poff.get()),
                    tcol.get(), tval.get(), cnt.get(), fb.get(), fbn.get());
        stage_scalar(c, 0, static_cast<const int32_t*>(fbn.get()));
        sync(c);
    }
    const int32_t nfb = bm_on ? staged<int32_t>(c, 0) : nlong;
    const int32_t* fl = bm_on ? fb.get() : big_list.get();
    if (nfb > 0) {
        launch_prof(c, kProfSpgemm, 0.0, k_spgemm_hash<kSmallCap, kHashWarps, kSortCap>, blocks_for(nfb, kHashWarps),
                    kHashWarps * kWarp, hash_smem(), nfb, A.rp.get(), A.ci.get(), A.va.get(), B.rp.get(), B.ci.get(),
                    B.va.get(), static_cast<const int64_t*>(poff.get()), tcol.get(), tval.get(), cnt.get(), fl);
        // rows above the warp kernels' capacity: up to kMidCap products one warp per block
        // over the list, the rest block per row
        static const bool mid_on = std::getenv("AMGCU_SPGEMM_NO_MID") == nullptr;
        const int64_t mid_cap = mid_on ? kMidCap : kSmallCap;
        if (mid_on)
            launch_prof(c, kProfSpgemm, 0.0, k_spgemm_hash<kMidCap, 1, kSmallCap>, static_cast<unsigned>(nfb), kWarp,
                        mid_smem(), nfb, A.rp.get(), A.ci.get(), A.va.get(), B.rp.get(), B.ci.get(), B.va.get(),
                        static_cast<const int64_t*>(poff.get()), tcol.get(), tval.get(), cnt.get(), fl);
        std::vector<int32_t> hl(nfb);
        copy_d2h(c, hl.data(), fl, nfb);
        std::vector<int64_t> hpoff(static_cast<size_t>(nr) + 1);
        copy_d2h(c, hpoff.data(), poff.get(), nr + 1);
        sync(c);
        // the rows left for the block kernel, ascending
        hl.erase(std::remove_if(hl.begin(), hl.end(), [&](int32_t r) { return hpoff[r + 1] - hpoff[r] <= mid_cap; }),
                 hl.end());
        const int32_t nb2 = static_cast<int32_t>(hl.size());
        if (nb2 > 0) {
            std::sort(hl.begin(), hl.end());
            std::vector<int64_t> soff(nb2);
            int64_t acc = 0;
            for (int32_t b = 0; b < nb2; ++b) {
                soff[b] = acc;
                int64_t np2 = 1;
                while (np2 < hpoff[hl[b] + 1] - hpoff[hl[b]]) np2 <<= 1;
                acc += np2;
            }
            DBuf<int32_t> dl(static_cast<size_t>(nb2), c.s);
            DBuf<int64_t> doff(static_cast<size_t>(nb2), c.s);
            DBuf<unsigned long long> gkeys(static_cast<size_t>(acc), c.s);
            DBuf<double> gvals(static_cast<size_t>(total), c.s);
            copy_h2d(c, dl.get(), hl.data(), nb2);
            copy_h2d(c, doff.get(), soff.data(), nb2);
            DBuf<int32_t> handled(static_cast<size_t>(nb2), c.s);
            static const bool no_hash = std::getenv("AMGCU_SPGEMM_NO_BIGHASH") != nullptr;
            if (no_hash) AMG_CK(cudaMemsetAsync(handled.get(), 0, sizeof(int32_t) * nb2, c.s));
            else launch(c, k_spgemm_big_hash<false>, static_cast<unsigned>(nb2), kBigThreads, big_hash_smem(),
                        static_cast<const int32_t*>(dl.get()), A.rp.get(), A.ci.get(), A.va.get(), B.rp.get(),
                        B.ci.get(), B.va.get(), static_cast<const int64_t*>(poff.get()), tcol.get(), tval.get(),
                        cnt.get(), handled.get(), static_cast<const int64_t*>(nullptr),
                        static_cast<int32_t*>(nullptr), static_cast<double*>(nullptr),
                        static_cast<unsigned long long*>(nullptr));
            if (!no_hash) {
                // rows the shared table refused: the same with the table in global scratch
                DBuf<int32_t> gk(static_cast<size_t>(acc), c.s);
                DBuf<double> gv(static_cast<size_t>(acc), c.s);
                launch(c, k_spgemm_big_hash<true>, static_cast<unsigned>(nb2), kBigThreads, 0,
                       static_cast<const int32_t*>(dl.get()), A.rp.get(), A.ci.get(), A.va.get(), B.rp.get(),
                       B.ci.get(), B.va.get(), static_cast<const int64_t*>(poff.get()), tcol.get(), tval.get(),
                       cnt.get(), handled.get(), static_cast<const int64_t*>(doff.get()), gk.get(), gv.get(),
                       gkeys.get());
            }
            launch(c, k_spgemm_big, static_cast<unsigned>(nb2), kBigThreads, 0, static_cast<const int32_t*>(dl.get()),
                   A.rp.get(), A.ci.get(), A.va.get(), B.rp.get(), B.ci.get(), B.va.get(),
                   static_cast<const int64_t*>(poff.get()), static_cast<const int64_t*>(doff.get()), gkeys.get(),
                   gvals.get(), tcol.get(), tval.get(), cnt.get(), static_cast<const int32_t*>(handled.get()));
            sync(c);
        }
    }
    compact_rows(c, nr, B.nc, poff, tcol, tval, cnt, C);
}

void galerkin(Ctx& c, const DCsr& R, const DCsr& A, const DCsr& P, DCsr& C, double* ops) {
    if (R.nc != A.nr || A.nc != P.nr) throw InvalidArgument("galerkin_product: dimension mismatch");
    DCsr AP;
    double o1 = 0.0, o2 = 0.0;
    spgemm(c, A, P, AP, &o1);
    spgemm(c, R, AP, C, &o2);
    C.bs = P.bs;
    if (ops) *ops = o1 + o2;
}

void filter_matrix(Ctx& c, const DCsr& G, bool theta_set, double theta, int32_t k, DCsr& F) {
    if (theta_set && (theta < 0.0 || theta > 1.0)) throw InvalidArgument("filter_matrix: theta must lie in [0, 1]");
    if (k < 0) throw InvalidArgument("filter_matrix: k must be >= 1");
    const bool square = G.nr == G.nc;
    DBuf<int32_t> cnt(static_cast<size_t>(G.nr) + 1, c.s);
    launch(c, k_filter_count, blocks_for(G.nr, 128), 128, 0, G.nr, square, G.rp.get(), G.ci.get(), G.va.get(),
           theta_set, theta, k, cnt.get());
    F.nr = G.nr;
    F.nc = G.nc;
    F.bs = G.bs;
    F.rp.alloc(static_cast<size_t>(G.nr) + 1, c.s);
    F.nnz = exclusive_scan_i32(c, cnt.get(), F.rp.get(), G.nr);
    F.ci.alloc(static_cast<size_t>(F.nnz), c.s);
    F.va.alloc(static_cast<size_t>(F.nnz), c.s);
    launch(c, k_filter_write, blocks_for(G.nr, 128), 128, 0, G.nr, square, G.rp.get(), G.ci.get(), G.va.get(),
           theta_set, theta, k, static_cast<const int32_t*>(F.rp.get()), F.ci.get(), F.va.get());
}

double max_abs(Ctx& c, const double* v, int64_t n) {
    DBuf<unsigned long long> out(1, c.s);
    AMG_CK(cudaMemsetAsync(out.get(), 0, sizeof(unsigned long long), c.s));
    const unsigned g = std::min<unsigned>(blocks_for(n, 256), 4u * c.sms);
    launch(c, k_max_abs, std::max(g, 1u), 256, 0, n, v, out.get());
    const unsigned long long bits = read_scalar(c, out.get());
    double r;
    std::memcpy(&r, &bits, sizeof(r));
    return r;
}

bool is_symmetric(Ctx& c, const DCsr& A, double tol) {
    if (A.nr != A.nc) return false;
    DBuf<unsigned long long> mx(1, c.s);
    AMG_CK(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned long long), c.s));
    const unsigned g = std::min<unsigned>(blocks_for(A.nnz, 256), 4u * c.sms);
    launch(c, k_max_abs, std::max(g, 1u), 256, 0, A.nnz, A.va.get(), mx.get());
    DBuf<int32_t> bad(1, c.s);
    AMG_CK(cudaMemsetAsync(bad.get(), 0, sizeof(int32_t), c.s));
    const double avg = A.nr ? static_cast<double>(A.nnz) / A.nr : 0.0;
    const unsigned long long* mb = mx.get();
    if (avg > 48.0)
        launch(c, k_asym<32>, blocks_for(static_cast<int64_t>(A.nr) * 32, 256), 256, 0, A.nr, A.rp.get(), A.ci.get(),
               A.va.get(), tol, mb, bad.get());
    else if (avg > 12.0)
        launch(c, k_asym<8>, blocks_for(static_cast<int64_t>(A.nr) * 8, 256), 256, 0, A.nr, A.rp.get(), A.ci.get(),
               A.va.get(), tol, mb, bad.get());
    else
        launch(c, k_asym<1>, blocks_for(A.nr, 256), 256, 0, A.nr, A.rp.get(), A.ci.get(), A.va.get(), tol, mb,
               bad.get());
    return read_scalar(c, bad.get()) == 0;
}

void inverse_diagonal(Ctx& c, const DCsr& A, double* dinv, const char* prefix) {
    const int32_t b = inverse_diagonal_check(c, A, dinv);
    if (b >= 0) throw RuntimeError(std::string(prefix) + std::to_string(b));
}

int32_t inverse_diagonal_check(Ctx& c, const DCsr& A, double* dinv) {
    const int32_t n = std::min(A.nr, A.nc);
    DBuf<int32_t> bad(1, c.s);
    fill_i32(c, bad.get(), INT_MAX, 1);
    launch(c, k_diag, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), A.va.get(), dinv, true, bad.get());
    const int32_t b = read_scalar(c, bad.get());
    return b == INT_MAX ? -1 : b;
}

void diagonal(Ctx& c, const DCsr& A, double* d) {
    const int32_t n = std::min(A.nr, A.nc);
    launch(c, k_diag, blocks_for(n, 256), 256, 0, n, A.rp.get(), A.ci.get(), A.va.get(), d, false,
           static_cast<int32_t*>(nullptr));
}

void compact_pattern(Ctx& c, const DCsr& N, const double* vals, int32_t bs, DCsr& out) {
    DBuf<int32_t> cnt(static_cast<size_t>(N.nr) + 1, c.s);
    launch(c, k_nonzero_count, blocks_for(N.nr, 256), 256, 0, N.nr, N.rp.get(), vals, cnt.get());
    out.nr = N.nr;
    out.nc = N.nc;
    out.bs = bs;
    out.rp.alloc(static_cast<size_t>(N.nr) + 1, c.s);
    out.nnz = exclusive_scan_i32(c, cnt.get(), out.rp.get(), N.nr);
    out.ci.alloc(static_cast<size_t>(out.nnz), c.s);
    out.va.alloc(static_cast<size_t>(out.nnz), c.s);
    launch(c, k_nonzero_write, blocks_for(N.nr, 256), 256, 0, N.nr, N.rp.get(), N.ci.get(), vals,
           static_cast<const int32_t*>(out.rp.get()), out.ci.get(), out.va.get());
}

}  // namespace amgcu
