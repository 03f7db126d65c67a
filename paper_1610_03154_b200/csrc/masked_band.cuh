// Band-staged masked product Y = (A X)|_N with the constraint projection fused
// (masked_product + project_to_constraints, interpolation.hpp:150-210), for the
// energy-minimisation iterations (interpolation.hpp:298-441).  Included by interp.cu.
//
// The pattern N and the operator are fixed over a level's iterations, so the matching
// of N_i against N_t is done ONCE (the plan) and every iteration streams its result:
//
//   * a CTA owns R consecutive rows.  The rows t its A entries reference form a few
//     runs of consecutive rows (a grid row above, the own one, one below on a 2-D
//     level), and X is stored in N's CSR order, so each run is ONE contiguous piece of
//     X.  The plan lists the runs per CTA; the kernel brings them into shared memory
//     with cp.async.bulk (TMA, completion on an mbarrier) together with the CTA's A
//     records -- no per-entry global gather is left in the iteration.
//   * per A entry the plan stores a 16-byte record {a, word}: word = the shared-memory
//     offset of X_t's slice (16 bits) and the match of N_i against N_t.  Pattern rows of
//     up to 12 slots: for each slot of N_i the position of that column inside N_t as a
//     4-bit index (15 = not in N_t).  Up to 24 slots: both rows are sorted, so the match
//     is monotone and two 24-bit masks hold it (the matched slots of N_i, the matched
//     entries of N_t; the j-th set bit of one pairs with the j-th of the other).
//   * thread per slot (entry of N): it walks its row's records in CSR order and adds
//     a * x for the records that hold its column -- the reference's per-slot order of
//     additions (interpolation.hpp:196-206), so the sums are bit-identical.  Outputs
//     are written coalesced.  The projection takes its row sums in slot order by one
//     thread per row from the shared values (interpolation.hpp:163-176).
//
// Levels whose referenced rows do not fit the run table and the shared-memory budget even
// at 4 rows per CTA (scattered coarse operators such as C4's A^T A on levels 2-3) use the
// DIRECT mode when their pattern rows have at most 16 slots: no staging of X, the record
// word holds the global offset of X_t's slice (32 bits) and two 16-bit masks, and the
// slot threads gather x from global memory (such a level's X is a few MB: L2-resident).
// Anything else keeps the register-merge kernel (k_masked_rows).
#pragma once

// (bitrank.h is included by interp.cu at file scope: this header sits inside its namespaces)
namespace mband {

constexpr int kNibSlots = 12;      // 4-bit indices: slots of N_i a record word holds
constexpr int kNibNt = 15;         //                 entries of N_t an index can address
constexpr int kMaskSlots = 24;     // mask pairs: longest pattern row
constexpr int kDirectSlots = 16;   // direct mode: longest pattern row
enum Mode : int { kNibbles = 0, kMasks = 1, kDirect = 2 };
constexpr int kMaxRuns = 64;       // runs of X a CTA stages
constexpr int kGran = 4;           // rows per bit of the referenced-rows bitmap
constexpr int kBitWords = 2048;    // 32-bit words of that bitmap (window of 262,144 rows)
constexpr int kThreads = 256;
constexpr size_t kSmemBudget = 200 * 1024;

struct Rec {  // one A entry
    double a;
    unsigned long long w;
};
static_assert(sizeof(Rec) == 16, "record is one 16-byte shared-memory load");

struct Run {  // a contiguous piece of X staged by a CTA
    int32_t xs;    // first element (even)
    int32_t len;   // elements (even)
    int32_t soff;  // offset in the stage (even)
    int32_t ta;    // first row (map kernel)
    int32_t tb;    // past-the-end row
    int32_t pad[3];
};

struct Plan {
    bool ok = false;
    int32_t R = 0, nctas = 0;
    int32_t cap_a = 0, cap_x = 0, cap_s = 0;  // records, staged doubles, slots per CTA (maxima)
    int mode = kNibbles;                       // record format (Mode)
    size_t smem = 0;
    DBuf<Rec> recs;
    DBuf<Run> runs;
    DBuf<int32_t> nruns;  // per CTA: {runs, bytes of X they stage}
    DBuf<int32_t> info;  // k_records' failure bits (checked after the iterations)
    DBuf<unsigned long long> matches;  // sum_i sum_{t in A row i} |N_i cap N_t| (interpolation.hpp:200-206)
};

// ---- plan, step 1: the runs of every CTA -------------------------------------------------
// info: [0] failure bits  [1] max records  [2] max staged doubles  [3] max slots  [4] longest row of N
__global__ void __launch_bounds__(kThreads)
    k_runs(int32_t n, int32_t R, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
           const int32_t* __restrict__ nrp, Run* __restrict__ runs, int32_t* __restrict__ nruns,
           int32_t* __restrict__ info, int direct) {
    __shared__ unsigned int bits[kBitWords];
    __shared__ int32_t s_min, s_max;
    const int32_t r0 = blockIdx.x * R, r1 = min(n, r0 + R);
    const int32_t a0 = arp[r0], a1 = arp[r1];
    if (threadIdx.x == 0) {
        s_min = INT_MAX;
        s_max = -1;
    }
    __syncthreads();
    int32_t lo = INT_MAX, hi = -1;
    for (int32_t e = a0 + threadIdx.x; e < a1; e += kThreads) {
        const int32_t t = aci[e];
        lo = min(lo, t);
        hi = max(hi, t);
    }
    for (int off = 16; off > 0; off >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    if ((threadIdx.x & 31) == 0 && hi >= 0) {
        atomicMin(&s_min, lo);
        atomicMax(&s_max, hi);
    }
    __syncthreads();
    // rows with slots but no A entry cannot occur on the path (the diagonal is stored)
    const int32_t nslots = nrp[r1] - nrp[r0];
    {
        int32_t longest = 0;
        for (int32_t i = r0 + threadIdx.x; i < r1; i += kThreads) longest = max(longest, nrp[i + 1] - nrp[i]);
        for (int off = 16; off > 0; off >>= 1) longest = max(longest, __shfl_xor_sync(0xffffffffu, longest, off));
        if ((threadIdx.x & 31) == 0 && longest > 0) atomicMax(&info[4], longest);
    }
    if (s_max < 0 || direct) {  // direct mode stages no X: only the capacities
        if (threadIdx.x == 0) {
            nruns[2 * blockIdx.x] = 0;
            nruns[2 * blockIdx.x + 1] = 0;
            atomicMax(&info[1], a1 - a0);
            atomicMax(&info[3], nslots);
        }
        return;
    }
    const int32_t base = (s_min / kGran) * kGran;
    const int32_t nb = (s_max - base) / kGran + 1;  // bits in use
    if (nb > kBitWords * 32) {
        if (threadIdx.x == 0) {
            atomicOr(&info[0], 1);
            nruns[2 * blockIdx.x] = 0;
            nruns[2 * blockIdx.x + 1] = 0;
        }
        return;
    }
    const int32_t nw = (nb + 31) / 32;
    for (int32_t w = threadIdx.x; w < nw; w += kThreads) bits[w] = 0u;
    __syncthreads();
    for (int32_t e = a0 + threadIdx.x; e < a1; e += kThreads) {
        const int32_t b = (aci[e] - base) / kGran;
        atomicOr(&bits[b >> 5], 1u << (b & 31));
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    // runs of set bits, in order
    int32_t count = 0, soff = 0;
    int32_t b = 0;
    Run* out = runs + static_cast<size_t>(blockIdx.x) * kMaxRuns;
    while (b < nb) {
        // next set bit at or after b
        unsigned int w = bits[b >> 5] >> (b & 31);
        if (w == 0u) {
            b = ((b >> 5) + 1) << 5;
            continue;
        }
        b += __ffs(w) - 1;
        int32_t e = b;
        // first clear bit after b
        for (;;) {
            const unsigned int inv = ~(bits[e >> 5] >> (e & 31));
            // bits beyond the word's end read as clear in inv's high part: mask them
            const int room = 32 - (e & 31);
            const unsigned int m = room == 32 ? inv : (inv & ((1u << room) - 1u));
            if (m != 0u) {
                e += __ffs(m) - 1;
                break;
            }
            e += room;
            if (e >= nb) {
                e = nb;
                break;
            }
        }
        if (e > nb) e = nb;
        const int32_t ta = base + b * kGran, tb = min(n, base + e * kGran);
        const int32_t xs = nrp[ta] & ~1, xe = (nrp[tb] + 1) & ~1;
        if (xe > xs) {
            if (count < kMaxRuns) {
                Run r;
                r.xs = xs;
                r.len = xe - xs;
                r.soff = soff;
                r.ta = ta;
                r.tb = tb;
                r.pad[0] = r.pad[1] = r.pad[2] = 0;
                out[count] = r;
            }
            ++count;
            soff += xe - xs;
        }
        b = e;
    }
    if (count > kMaxRuns) {
        atomicOr(&info[0], 2);
        count = 0;
    }
    if (soff > 65535 - kMaskSlots) atomicOr(&info[0], 4);
    nruns[2 * blockIdx.x] = count;
    nruns[2 * blockIdx.x + 1] = count ? soff * 8 : 0;
    atomicMax(&info[1], a1 - a0);
    atomicMax(&info[2], soff);
    atomicMax(&info[3], nslots);
}

// ---- plan, step 2: the record of every A entry --------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k_records(int32_t n, int32_t R, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
              const double* __restrict__ ava, const int32_t* __restrict__ nrp, const int32_t* __restrict__ nci,
              const Run* __restrict__ runs, const int32_t* __restrict__ nruns, Rec* __restrict__ recs,
              int32_t* __restrict__ info, unsigned long long* __restrict__ matches) {
    __shared__ Run s_runs[kMaxRuns];
    __shared__ int32_t s_arp[129];
    const int32_t r0 = blockIdx.x * R, r1 = min(n, r0 + R);
    const int32_t nr = nruns[2 * blockIdx.x];
    for (int32_t j = threadIdx.x; j < nr; j += kThreads) s_runs[j] = runs[static_cast<size_t>(blockIdx.x) * kMaxRuns + j];
    for (int32_t j = threadIdx.x; j <= r1 - r0; j += kThreads) s_arp[j] = arp[r0 + j];
    __syncthreads();
    const int32_t a0 = s_arp[0], a1 = s_arp[r1 - r0];
    unsigned long long found = 0;  // sum over the entries of |N_i cap N_t| (the masked product's op count)
    for (int32_t e = a0 + threadIdx.x; e < a1; e += kThreads) {
        // row of entry e: last j with s_arp[j] <= e
        int32_t lo = 0, hi = r1 - r0;
        while (hi - lo > 1) {
            const int32_t mid = (lo + hi) >> 1;
            if (s_arp[mid] <= e) lo = mid;
            else hi = mid;
        }
        const int32_t i = r0 + lo;
        const int32_t t = aci[e];
        Rec rec;
        rec.a = ava[e];
        unsigned long long w = MODE == kNibbles ? ~0ull : 0ull;  // no slot of N_i is in N_t
        const int32_t ilo = nrp[i], L = nrp[i + 1] - ilo;
        const int32_t q0 = nrp[t], Lt = nrp[t + 1] - q0;
        if (L > (MODE == kNibbles ? kNibSlots : MODE == kMasks ? kMaskSlots : kDirectSlots) ||
            Lt > (MODE == kNibbles ? kNibNt : MODE == kMasks ? kMaskSlots : kDirectSlots)) {
            atomicOr(&info[0], 8);
        } else if (L > 0 && Lt > 0) {
            // the run holding row t: the last one starting at or before it
            int32_t jl = 0, jh = nr;
            while (jh - jl > 1) {
                const int32_t mid = (jl + jh) >> 1;
                if (s_runs[mid].ta <= t) jl = mid;
                else jh = mid;
            }
            if (MODE != kDirect && (nr == 0 || !(s_runs[jl].ta <= t && t < s_runs[jl].tb))) {
                atomicOr(&info[0], 16);
            } else {
                const unsigned int off = MODE == kDirect ? static_cast<unsigned int>(q0)
                                                         : static_cast<unsigned int>(s_runs[jl].soff + (q0 - s_runs[jl].xs));
                unsigned long long mi = 0ull, mt = 0ull;
                int32_t q = 0;
                for (int32_t s = 0; s < L; ++s) {
                    const int32_t col = nci[ilo + s];
                    while (q < Lt && nci[q0 + q] < col) ++q;
                    if (q < Lt && nci[q0 + q] == col) {
                        ++found;
                        if (MODE != kNibbles) {
                            mi |= 1ull << s;
                            mt |= 1ull << q;
                        } else {
                            const int sh = 16 + 4 * s;
                            w = (w & ~(0xfull << sh)) | (static_cast<unsigned long long>(q) << sh);
                        }
                    }
                }
                if (MODE == kMasks) w = (mi << 16) | (mt << 40);
                if (MODE == kDirect) w = (mi << 32) | (mt << 48) | off;
                else w = (w & ~0xffffull) | off;
            }
        }
        rec.w = w;
        recs[e] = rec;
    }
    for (int off = 16; off > 0; off >>= 1) found += __shfl_xor_sync(0xffffffffu, found, off);
    if ((threadIdx.x & 31) == 0 && found) atomicAdd(matches, found);
}

using ::amgcu::bitrank::nth_set_bit24;  // bitrank.h: position of the j-th set bit of a 24-bit mask

// ---- the iteration kernel -----------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// shared memory: [mbarrier 16 B][records cap_a][stage cap_x][values cap_s][lambda R*k]
//                [arp R+1][nrp R+1][row of slot cap_s (uint8)]
__host__ __device__ inline size_t smem_bytes(int32_t R, int32_t cap_a, int32_t cap_x, int32_t cap_s, int32_t k) {
    size_t b = 16;
    b += static_cast<size_t>(cap_a + 1) * sizeof(Rec);
    b += static_cast<size_t>(cap_x + 2) * 8;
    b += static_cast<size_t>(cap_s) * 8;
    b += static_cast<size_t>(R) * k * 8;
    b += static_cast<size_t>(R + 1) * 4 * 2;
    b += static_cast<size_t>(cap_s);
    return (b + 15) & ~static_cast<size_t>(15);
}

// KT: the candidate count when it is 1..3 (projection sums in registers), 0 = any k <= 8
// MODE: the record format -- 4-bit indices, mask pairs (pattern rows of 13..24 slots), or
// direct (global offset + 16-bit mask pairs, x gathered from global memory)
template <int KT, int MODE>
__global__ void __launch_bounds__(kThreads)
    k_masked_band(int32_t n, int32_t R, int32_t cap_a, int32_t cap_x, int32_t cap_s,
                  const int32_t* __restrict__ arp, const Rec* __restrict__ recs, const int32_t* __restrict__ nrp,
                  const int32_t* __restrict__ nci, const double* __restrict__ x, int32_t k,
                  const double* __restrict__ Bc, int32_t nc, const double* __restrict__ gp,
                  const unsigned char* __restrict__ is_root, double* __restrict__ y, double* __restrict__ yp,
                  const Run* __restrict__ runs, const int32_t* __restrict__ nruns, const int32_t* __restrict__ stop) {
    if (stop && *stop) return;
    if (KT) k = KT;
    constexpr int KM = KT ? KT : 8;
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem);
    Rec* s_rec = reinterpret_cast<Rec*>(smem + 16);
    double* s_x = reinterpret_cast<double*>(s_rec + (cap_a + 1));
    double* s_v = s_x + (cap_x + 2);
    double* s_lam = s_v + cap_s;
    int32_t* s_arp = reinterpret_cast<int32_t*>(s_lam + static_cast<size_t>(R) * k);
    int32_t* s_nrp = s_arp + (R + 1);
    unsigned char* s_row = reinterpret_cast<unsigned char*>(s_nrp + (R + 1));

    const int32_t r0 = blockIdx.x * R, r1 = min(n, r0 + R), nrows = r1 - r0;
    const uint32_t bar_a = smem_addr(bar);
    const int32_t a0 = arp[r0];
    // warp 0 issues the bulk copies with one round of global loads before them: every lane
    // reads the run it will copy (entries beyond the run count are never used) while lane 0
    // reads the CTA's header (run count, staged bytes) and its record range; lane 0 arms the
    // barrier and copies the records (16 bytes each: aligned as they are), then each lane
    // copies its run
    if (threadIdx.x < 32) {
        const Run* rr = runs + static_cast<size_t>(blockIdx.x) * kMaxRuns;
        const int4 h0 = *reinterpret_cast<const int4*>(rr + threadIdx.x);  // xs, len, soff, ta
        const int32_t nr = nruns[2 * blockIdx.x];
        if (threadIdx.x == 0) {
            const uint32_t rec_bytes = static_cast<uint32_t>(arp[r1] - a0) * 16u;
            const uint32_t total = rec_bytes + static_cast<uint32_t>(nruns[2 * blockIdx.x + 1]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(total) : "memory");
            if (rec_bytes) bulk_g2s(s_rec, recs + a0, rec_bytes, bar_a);
        }
        __syncwarp();
        if (static_cast<int32_t>(threadIdx.x) < nr) bulk_g2s(s_x + h0.z, x + h0.x, static_cast<uint32_t>(h0.y) * 8u, bar_a);
        for (int32_t j = threadIdx.x + 32; j < nr; j += 32) {
            const int4 h = *reinterpret_cast<const int4*>(rr + j);
            bulk_g2s(s_x + h.z, x + h.x, static_cast<uint32_t>(h.y) * 8u, bar_a);
        }
    }
    for (int32_t j = threadIdx.x; j <= nrows; j += kThreads) {
        s_arp[j] = arp[r0 + j];
        s_nrp[j] = nrp[r0 + j];
    }
    __syncthreads();
    const int32_t p0 = s_nrp[0], nslots = s_nrp[nrows] - p0;
    for (int32_t r = threadIdx.x; r < nrows; r += kThreads)
        for (int32_t q = s_nrp[r] - p0; q < s_nrp[r + 1] - p0; ++q) s_row[q] = static_cast<unsigned char>(r);
    __syncthreads();
    // wait for the bulk copies (phase 0 of the one-shot barrier)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(bar_a)
                : "memory");
        }
    }
    // phase 1: thread per slot, records in CSR order
    for (int32_t q = threadIdx.x; q < nslots; q += kThreads) {
        const int32_t r = s_row[q];
        const int slot = q - (s_nrp[r] - p0);
        const Rec* e = s_rec + (s_arp[r] - a0);
        const Rec* const ee = s_rec + (s_arp[r + 1] - a0);
        double acc = 0.0;
        if (MODE == kMasks) {
            const unsigned int below = (1u << slot) - 1u;
            for (; e < ee; ++e) {
                const double a = e->a;
                const unsigned long long w = e->w;
                const unsigned int mi = static_cast<unsigned int>(w >> 16) & 0xffffffu;
                if ((mi >> slot) & 1u) {
                    const unsigned int u = nth_set_bit24(static_cast<unsigned int>(w >> 40), __popc(mi & below));
                    acc += a * s_x[(static_cast<unsigned int>(w) & 0xffffu) + u];
                }
            }
        } else if (MODE == kDirect) {
            const unsigned int below = (1u << slot) - 1u;
            for (; e < ee; ++e) {
                const double a = e->a;
                const unsigned long long w = e->w;
                const unsigned int mi = static_cast<unsigned int>(w >> 32) & 0xffffu;
                if ((mi >> slot) & 1u) {
                    const unsigned int u = nth_set_bit24(static_cast<unsigned int>(w >> 48), __popc(mi & below));
                    acc += a * __ldg(x + (static_cast<unsigned int>(w) + u));
                }
            }
        } else {
            const int sh = 16 + 4 * slot;
            for (; e < ee; ++e) {
                const double a = e->a;
                const unsigned long long w = e->w;
                const unsigned int u = static_cast<unsigned int>(w >> sh) & 15u;
                if (u != 15u) acc += a * s_x[(static_cast<unsigned int>(w) & 0xffffu) + u];
            }
        }
        s_v[q] = acc;
        if (y) y[p0 + q] = acc;
    }
    if (!yp) return;
    __syncthreads();
    // phase 2: thread per row, lambda = G^+ (Bc^T y_row) in slot order
    for (int32_t r = threadIdx.x; r < nrows; r += kThreads) {
        const int32_t i = r0 + r;
        if (is_root[i]) continue;
        double ya[KM], lam[KM];
        #pragma unroll
        for (int a = 0; a < KM; ++a) ya[a] = 0.0;
        for (int32_t q = s_nrp[r] - p0; q < s_nrp[r + 1] - p0; ++q) {
            const int32_t cj = nci[p0 + q];
            const double v = s_v[q];
#pragma unroll
            for (int a = 0; a < KM; ++a)
                if (a < k) ya[a] += Bc[static_cast<size_t>(a) * nc + cj] * v;
        }
        const double* G = gp + static_cast<size_t>(i) * k * k;
#pragma unroll
        for (int a = 0; a < KM; ++a) {
            double s2 = 0.0;
#pragma unroll
            for (int b2 = 0; b2 < KM; ++b2)
                if (a < k && b2 < k) s2 += G[a * k + b2] * ya[b2];
            lam[a] = s2;
        }
#pragma unroll
        for (int a = 0; a < KM; ++a)
            if (a < k) s_lam[r * k + a] = lam[a];
    }
    __syncthreads();
    // phase 3: thread per slot
    for (int32_t q = threadIdx.x; q < nslots; q += kThreads) {
        const int32_t r = s_row[q];
        double out = 0.0;
        if (!is_root[r0 + r]) {
            const int32_t cj = nci[p0 + q];
            double t2 = 0.0;
            for (int a = 0; a < k; ++a) t2 += Bc[static_cast<size_t>(a) * nc + cj] * s_lam[r * k + a];
            out = s_v[q] - t2;
        }
        yp[p0 + q] = out;
    }
}

}  // namespace mband
