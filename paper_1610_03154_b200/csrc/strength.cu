// Strength of connection on the GPU (strength.hpp).
//  symmetric / classical: thread per row, count + scan + write.
//  evolution: one warp per row; the distance-`steps` neighbourhood in A + A^T
//  lives in a shared-memory hash (global id -> local slot), the local Jacobi
//  evolution z <- z - W^{-1} (A z) runs lane-parallel over the neighbourhood
//  with each row sum in CSR order (strength.hpp:179-194), and the ring decision
//  (strength.hpp:199-231) is taken over the merged A / A^T row.  Rows whose
//  neighbourhood exceeds the shared capacity fall back to a block-per-row
//  kernel over a direct-mapped global scratch.
#include <climits>

#include "ops.cuh"

namespace amgcu {

namespace {

constexpr int kWarp = 32;

__device__ __forceinline__ double diag_of(const int32_t* rp, const int32_t* ci, const double* va, int32_t i) {
    int32_t lo = rp[i], hi = rp[i + 1];
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (ci[mid] < i) lo = mid + 1;
        else hi = mid;
    }
    return (lo < rp[i + 1] && ci[lo] == i) ? va[lo] : 0.0;
}

// ---- symmetric (strength.hpp:70-107) / classical (29-66) --------------------------------
template <bool kSym>
__device__ __forceinline__ bool strong(const double* d, int32_t i, int32_t j, double v, double theta, double mx,
                                       double* val) {
    if (kSym) {
        const double raw = fabs(v) / sqrt(fabs(d[i]) * fabs(d[j]));
        *val = raw;
        return raw >= theta && raw > 0.0;
    } else {
        const double raw = -v;
        *val = raw;
        return mx > 0.0 && raw > 0.0 && raw >= theta * mx;
    }
}

template <bool kSym>
__global__ void k_soc(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                      const double* __restrict__ va, const double* __restrict__ d, double theta,
                      const int32_t* __restrict__ orp, int32_t* __restrict__ cnt, int32_t* __restrict__ oci,
                      double* __restrict__ ova) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double mx = 0.0;
    if (!kSym)
        for (int32_t p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] != i && mx < -va[p]) mx = -va[p];  // std::max(mx, -a_ip)
    int32_t o = orp ? orp[i] : 0;
    bool dd = false;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = ci[p];
        if (j == i) continue;
        double val;
        if (strong<kSym>(d, i, j, va[p], theta, mx, &val)) {
            if (!dd && j > i) {
                if (orp) {
                    oci[o] = i;
                    ova[o] = 1.0;
                }
                ++o;
                dd = true;
            }
            if (orp) {
                oci[o] = j;
                ova[o] = val;
            }
            ++o;
        }
    }
    if (!dd) {  // diagonal goes last (every emitted column is < i)
        if (orp) {
            oci[o] = i;
            ova[o] = 1.0;
        }
        ++o;
    }
    if (!orp) cnt[i] = o;
}

// ---- normalize_strength (strength.hpp:252-288) --------------------------------------------
__global__ void k_normalize(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ va, const int32_t* __restrict__ orp, int32_t* __restrict__ cnt,
                            int32_t* __restrict__ oci, double* __restrict__ ova) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double mx = 0.0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p)
        if (ci[p] != i && va[p] > mx) mx = va[p];
    int32_t o = orp ? orp[i] : 0;
    bool dd = false;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = ci[p];
        if (j == i || mx <= 0.0) continue;
        const double v = va[p] / mx;
        if (v == 0.0) continue;
        if (!dd && j > i) {
            if (orp) {
                oci[o] = i;
                ova[o] = 1.0;
            }
            ++o;
            dd = true;
        }
        if (orp) {
            oci[o] = j;
            ova[o] = v;
        }
        ++o;
    }
    if (!dd) {
        if (orp) {
            oci[o] = i;
            ova[o] = 1.0;
        }
        ++o;
    }
    if (!orp) cnt[i] = o;
}

__global__ void k_negative_check(int64_t nnz, const double* __restrict__ va, int32_t* __restrict__ bad) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < nnz && va[p] < 0.0) atomicExch(bad, 1);
}

// ---- amalgamate (strength.hpp:292-324): node row = max |s| per block column ----------------
__device__ void amalgamate_row_serial(int32_t bi, int32_t m, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const double* __restrict__ va, const int32_t* __restrict__ orp, int32_t* __restrict__ cnt,
                             int32_t* __restrict__ oci, double* __restrict__ ova) {
    const int32_t lo = rp[bi * m], hi = rp[bi * m + m];
    int32_t o = 0;
    for (int32_t p = lo; p < hi; ++p) {
        const int32_t bc = ci[p] / m;
        bool first = true;  // first occurrence of this block column in the node row
        for (int32_t q = lo; q < p; ++q)
            if (ci[q] / m == bc) {
                first = false;
                break;
            }
        if (!first) continue;
        double mx = 0.0;
        for (int32_t q = p; q < hi; ++q)
            if (ci[q] / m == bc) mx = fmax(mx, fabs(va[q]));
        if (mx == 0.0) continue;
        if (orp) {
            int32_t rank = 0;  // distinct nonzero block columns smaller than bc
            for (int32_t q = lo; q < hi; ++q) {
                const int32_t oc = ci[q] / m;
                if (oc >= bc) continue;
                bool f = true;
                for (int32_t r = lo; r < q; ++r)
                    if (ci[r] / m == oc) {
                        f = false;
                        break;
                    }
                if (!f) continue;
                double om = 0.0;
                for (int32_t r = q; r < hi; ++r)
                    if (ci[r] / m == oc) om = fmax(om, fabs(va[r]));
                rank += (om != 0.0);
            }
            oci[orp[bi] + rank] = bc;
            ova[orp[bi] + rank] = mx;
        }
        ++o;
    }
    if (!orp) cnt[bi] = o;
}

// One warp per node row: the row's block columns are rank-sorted in shared memory
// (ties by position), each distinct block column's max |s| is read off its group and
// the nonzero ones are numbered in ascending order -- the same entries and values as
// the serial restatement above. Longer node rows are listed for k_amalgamate_long.
constexpr int kAmWarps = 4;
constexpr int kAmCap = 640;

__global__ void __launch_bounds__(kAmWarps * 32) k_amalgamate(int32_t nn, int32_t m, const int32_t* __restrict__ rp,
                                                              const int32_t* __restrict__ ci,
                                                              const double* __restrict__ va,
                                                              const int32_t* __restrict__ orp, int32_t* __restrict__ cnt,
                                                              int32_t* __restrict__ oci, double* __restrict__ ova,
                                                              int32_t* __restrict__ long_rows,
                                                              int32_t* __restrict__ n_long) {
    __shared__ int32_t s_in[kAmWarps][kAmCap];
    __shared__ int32_t s_bc[kAmWarps][kAmCap];
    __shared__ double s_v[kAmWarps][kAmCap];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t bi = blockIdx.x * kAmWarps + warp;
    if (bi >= nn) return;
    const int32_t lo = rp[bi * m], hi = rp[bi * m + m], L = hi - lo;
    if (L > kAmCap) {
        if (lane == 0) long_rows[atomicAdd(n_long, 1)] = bi;  // k_amalgamate_long
        return;
    }
    int32_t* in = s_in[warp];
    int32_t* bc = s_bc[warp];
    double* v = s_v[warp];
    for (int32_t j = lane; j < L; j += 32) in[j] = ci[lo + j] / m;
    __syncwarp();
    for (int32_t j = lane; j < L; j += 32) {
        const int32_t k = in[j];
        int32_t r = 0;
        for (int32_t q = 0; q < L; ++q) {
            const int32_t kq = in[q];
            r += (kq < k) || (kq == k && q < j);
        }
        bc[r] = k;
        v[r] = fabs(va[lo + j]);
    }
    __syncwarp();
    int32_t o = 0;
    for (int32_t base = 0; base < L; base += 32) {
        const int32_t j = base + lane;
        bool keep = false;
        int32_t k = 0;
        double mx = 0.0;
        if (j < L && (j == 0 || bc[j - 1] != bc[j])) {
            k = bc[j];
            for (int32_t q = j; q < L && bc[q] == k; ++q) mx = fmax(mx, v[q]);
            keep = mx != 0.0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep && orp) {
            const int32_t pos = orp[bi] + o + __popc(bal & ((1u << lane) - 1u));
            oci[pos] = k;
            ova[pos] = mx;
        }
        o += __popc(bal);
    }
    if (!orp && lane == 0) cnt[bi] = o;
}

// Node rows above kAmCap entries, a block each (grid-stride over the list): the
// (block column, position) keys are bitonic-sorted in shared memory, then each
// distinct block column's max |s| is read in position order. Rows above
// kAmLongCap entries fall back to the serial restatement.
constexpr int kAmLongThreads = 512;
constexpr int kAmLongCap = 16384;

__global__ void __launch_bounds__(kAmLongThreads)
    k_amalgamate_long(const int32_t* __restrict__ long_rows, const int32_t* __restrict__ n_long, int32_t m,
                      const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ va,
                      const int32_t* __restrict__ orp, int32_t* __restrict__ cnt, int32_t* __restrict__ oci,
                      double* __restrict__ ova) {
    extern __shared__ __align__(16) unsigned long long am_keys[];
    __shared__ int32_t s_warp[kAmLongThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int32_t nl = *n_long;
    for (int32_t b = blockIdx.x; b < nl; b += gridDim.x) {
        const int32_t bi = long_rows[b];
        const int32_t lo = rp[bi * m], hi = rp[bi * m + m], L = hi - lo;
        if (L > kAmLongCap) {
            if (tid == 0) amalgamate_row_serial(bi, m, rp, ci, va, orp, cnt, oci, ova);
            continue;
        }
        int32_t n2 = 1;
        while (n2 < L) n2 <<= 1;
        for (int32_t j = tid; j < n2; j += kAmLongThreads)
            am_keys[j] = j < L ? (static_cast<unsigned long long>(static_cast<uint32_t>(ci[lo + j] / m)) << 32) |
                                     static_cast<uint32_t>(j)
                               : ~0ull;
        __syncthreads();
        for (int32_t k = 2; k <= n2; k <<= 1)
            for (int32_t j = k >> 1; j > 0; j >>= 1) {
                for (int32_t e = tid; e < n2 / 2; e += kAmLongThreads) {
                    const int32_t x = 2 * e - (e & (j - 1)), y = x + j;
                    const bool up = (x & k) == 0;
                    const unsigned long long a = am_keys[x], c = am_keys[y];
                    if ((a > c) == up) {
                        am_keys[x] = c;
                        am_keys[y] = a;
                    }
                }
                __syncthreads();
            }
        int32_t o = 0;
        for (int32_t base = 0; base < L; base += kAmLongThreads) {
            const int32_t j = base + tid;
            bool keep = false;
            uint32_t bc = 0;
            double mx = 0.0;
            if (j < L) {
                bc = static_cast<uint32_t>(am_keys[j] >> 32);
                if (j == 0 || static_cast<uint32_t>(am_keys[j - 1] >> 32) != bc) {
                    for (int32_t q = j; q < L && static_cast<uint32_t>(am_keys[q] >> 32) == bc; ++q)
                        mx = fmax(mx, fabs(va[lo + static_cast<uint32_t>(am_keys[q] & 0xffffffffu)]));
                    keep = mx != 0.0;
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_warp[wid] = __popc(bal);
            __syncthreads();
            int32_t before = o;
            for (int w = 0; w < wid; ++w) before += s_warp[w];
            if (keep && orp) {
                const int32_t pos = orp[bi] + before + __popc(bal & ((1u << lane) - 1u));
                oci[pos] = static_cast<int32_t>(bc);
                ova[pos] = mx;
            }
            for (int w = 0; w < kAmLongThreads / 32; ++w) o += s_warp[w];
            __syncthreads();
        }
        if (!orp && tid == 0) cnt[bi] = o;
    }
}

// ---- evolution (strength.hpp:116-238) -------------------------------------------------------
constexpr int kEvWarps = 4;
constexpr int kEvCap = 256;    // neighbourhood capacity per warp
constexpr int kEvHash = 512;   // power of two

struct EvShared {
    int32_t nodes[kEvCap];
    double z[kEvCap];
    double zn[kEvCap];
    int32_t hkey[kEvHash];
    int32_t hval[kEvHash];
    int32_t count;
    int32_t overflow;
};

__device__ __forceinline__ uint32_t hslot(int32_t key) { return (static_cast<uint32_t>(key) * 2654435761u) & (kEvHash - 1); }

__device__ __forceinline__ int32_t h_lookup(const EvShared& sh, int32_t key) {
    uint32_t s = hslot(key);
    for (int probe = 0; probe < kEvHash; ++probe) {
        const int32_t k = sh.hkey[s];
        if (k == key) return sh.hval[s];
        if (k < 0) return -1;
        s = (s + 1) & (kEvHash - 1);
    }
    return -1;
}

// insert; returns the new local id if this call inserted, -1 if present, -2 on overflow
__device__ __forceinline__ int32_t h_insert(EvShared& sh, int32_t key) {
    uint32_t s = hslot(key);
    for (int probe = 0; probe < kEvHash; ++probe) {
        const int32_t prev = atomicCAS(&sh.hkey[s], -1, key);
        if (prev == -1) {
            const int32_t id = atomicAdd(&sh.count, 1);
            if (id >= kEvCap) {
                sh.overflow = 1;
                sh.hval[s] = -1;
                return -2;
            }
            sh.nodes[id] = key;
            sh.hval[s] = id;
            return id;
        }
        if (prev == key) return -1;
        s = (s + 1) & (kEvHash - 1);
    }
    sh.overflow = 1;
    return -2;
}

__device__ __forceinline__ int32_t lower_bound_i32(const int32_t* a, int32_t lo, int32_t hi, int32_t key) {
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kEvWarps * kWarp)
    k_evolution(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ va,
                const int32_t* __restrict__ trp, const int32_t* __restrict__ tci, const double* __restrict__ winv,
                double drop_tol, int steps, const int64_t* __restrict__ ooff, int32_t* __restrict__ cnt,
                int32_t* __restrict__ tcol, double* __restrict__ tval, int32_t* __restrict__ overflow_rows,
                int32_t* __restrict__ n_overflow, const int32_t* __restrict__ rows, int32_t nrows) {
    __shared__ EvShared shm[kEvWarps];
    const int w = threadIdx.x / kWarp, lane = threadIdx.x & (kWarp - 1);
    const int32_t r = blockIdx.x * kEvWarps + w;
    if (r >= nrows) return;
    const int32_t i = rows ? rows[r] : r;
    EvShared& sh = shm[w];
    for (int s = lane; s < kEvHash; s += kWarp) sh.hkey[s] = -1;
    if (lane == 0) {
        sh.count = 0;
        sh.overflow = 0;
    }
    __syncwarp();
    if (lane == 0) h_insert(sh, i);
    __syncwarp();
    int32_t lo = 0;
    for (int st = 0; st < steps; ++st) {
        const int32_t hi = min(sh.count, kEvCap);
        for (int32_t f = lo; f < hi; ++f) {
            const int32_t u = sh.nodes[f];
            for (int32_t p = rp[u] + lane; p < rp[u + 1]; p += kWarp) h_insert(sh, ci[p]);
            for (int32_t p = trp[u] + lane; p < trp[u + 1]; p += kWarp) h_insert(sh, tci[p]);
        }
        __syncwarp();
        lo = hi;
        if (sh.overflow) break;
    }
    __syncwarp();
    if (sh.overflow) {
        if (lane == 0) overflow_rows[atomicAdd(n_overflow, 1)] = i;
        return;
    }
    const int32_t nb = sh.count;
    for (int32_t t = lane; t < nb; t += kWarp) sh.z[t] = (t == 0) ? 1.0 : 0.0;
    __syncwarp();
    double* z = sh.z;
    double* zn = sh.zn;
    for (int st = 0; st < steps; ++st) {
        for (int32_t t = lane; t < nb; t += kWarp) {
            const int32_t u = sh.nodes[t];
            double az = 0.0;
            for (int32_t p = rp[u]; p < rp[u + 1]; ++p) {
                const int32_t lj = h_lookup(sh, ci[p]);
                if (lj >= 0) az += va[p] * z[lj];
            }
            zn[t] = z[t] - winv[u] * az;
        }
        __syncwarp();
        double* tmp = z;
        z = zn;
        zn = tmp;
    }
    // ring: A row i followed by the A^T entries not in A row i, each ranked in the union
    const int32_t alo = rp[i], ahi = rp[i + 1], tlo = trp[i], thi = trp[i + 1];
    const int32_t na = ahi - alo, nt = thi - tlo;
    double mx = 0.0;
    for (int32_t e = lane; e < na + nt; e += kWarp) {
        int32_t j;
        if (e < na) {
            j = ci[alo + e];
        } else {
            j = tci[tlo + e - na];
            const int32_t pos = lower_bound_i32(ci, alo, ahi, j);
            if (pos < ahi && ci[pos] == j) continue;
        }
        if (j == i) continue;
        const int32_t lj = h_lookup(sh, j);
        if (lj >= 0) mx = fmax(mx, fabs(z[lj]));
    }
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const double cutoff = mx / drop_tol;
    const double zi = fabs(z[0]);
    const double dval = zi > 0.0 ? zi : 1.0;
    int32_t* ocol = tcol + ooff[i];
    double* oval = tval + ooff[i];
    // emitted entries: rank among emitted = #emitted ring entries with smaller column,
    // +1 if the diagonal precedes it
    int32_t emitted_total = 0;
    int32_t below_i = 0;  // emitted columns < i
    for (int32_t e0 = 0; e0 < na + nt; e0 += kWarp) {
        const int32_t e = e0 + lane;
        bool emit = false;
        int32_t j = -1;
        double mag = 0.0;
        if (e < na + nt) {
            bool dup = false;
            if (e < na) {
                j = ci[alo + e];
            } else {
                j = tci[tlo + e - na];
                const int32_t pos = lower_bound_i32(ci, alo, ahi, j);
                dup = (pos < ahi && ci[pos] == j);
            }
            if (!dup && j != i) {
                const int32_t lj = h_lookup(sh, j);
                mag = lj >= 0 ? fabs(z[lj]) : 0.0;
                emit = mx > 0.0 && mag >= cutoff && mag > 0.0;
            }
        }
        const unsigned b = __ballot_sync(0xffffffffu, emit);
        emitted_total += __popc(b);
        const unsigned bl = __ballot_sync(0xffffffffu, emit && j < i);
        below_i += __popc(bl);
        if (emit) {
            // rank among emitted: count emitted ring entries with smaller column
            int32_t rank = 0;
            for (int32_t f = 0; f < na + nt; ++f) {
                int32_t jf;
                if (f < na) {
                    jf = ci[alo + f];
                } else {
                    jf = tci[tlo + f - na];
                    const int32_t pos = lower_bound_i32(ci, alo, ahi, jf);
                    if (pos < ahi && ci[pos] == jf) continue;
                }
                if (jf >= j || jf == i) continue;
                const int32_t lf = h_lookup(sh, jf);
                const double mf = lf >= 0 ? fabs(z[lf]) : 0.0;
                rank += (mx > 0.0 && mf >= cutoff && mf > 0.0) ? 1 : 0;
            }
            const int32_t at = rank + (j > i ? 1 : 0);
            ocol[at] = j;
            oval[at] = mag;
        }
    }
    if (lane == 0) {
        ocol[below_i] = i;
        oval[below_i] = dval;
        cnt[i] = emitted_total + 1;
    }
}

// Two evolution steps (the BASELINE configurations), without a neighbourhood.
// z1 = z0 - W^-1 A z0 with z0 = e_i is non-zero only on column i's pattern
// (A^T row i) and at i:  z1[j] = [j == i] - winv[j] * A(j, i)  -- exactly the
// reference's value, its row sum having one non-zero term.  Every row of a
// ring node u (A row i U A^T row i) lies inside the distance-2 ball, so the
// second step needs no truncation:
//   z2[u] = z1[u] - winv[u] * sum_{p in row u, CSR order} a_p z1[c_p],
// where the terms with z1 = +0 are skipped (the sum starts at +0 and adding
// +-0 never changes it; matrices holding inf/NaN are outside this argument).
// One warp per row; A row i and column i's pattern are staged in shared
// memory and looked up by binary search.  Rows with more than kEv2Cap entries
// in either list go to the generic kernel.
constexpr int kEv2Warps = 8;
constexpr int kEv2Cap = 64;

struct Ev2Shared {
    int32_t acol[kEv2Cap];       // A row i
    int32_t tcol[kEv2Cap];       // A^T row i (column i's pattern)
    double z1[kEv2Cap];          // z1 on column i's pattern
    int32_t tonly[kEv2Cap];      // A^T entries absent from A row i: exclusive prefix
    int32_t aemit[kEv2Cap];      // emitted-flag prefix over A row i
    int32_t temit[kEv2Cap];      // emitted-flag prefix over the A^T-only entries (by A^T index)
    double amag[kEv2Cap];
    double tmag[kEv2Cap];
};

__device__ __forceinline__ int32_t find_sorted(const int32_t* a, int32_t n, int32_t key) {
    int32_t lo = lower_bound_i32(a, 0, n, key);
    return (lo < n && a[lo] == key) ? lo : -1;
}

// exclusive warp prefix of flags[0..n) (in place), returns the total
__device__ __forceinline__ int32_t warp_prefix(int32_t* flags, int32_t n, int lane) {
    int32_t base = 0;
    for (int32_t e0 = 0; e0 < n; e0 += kWarp) {
        const int32_t e = e0 + lane;
        const int32_t f = e < n ? flags[e] : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f != 0);
        if (e < n) flags[e] = base + __popc(bal & ((1u << lane) - 1u));
        base += __popc(bal);
    }
    return base;
}

__global__ void __launch_bounds__(kEv2Warps * kWarp)
    k_evolution2(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                 const double* __restrict__ va, const int32_t* __restrict__ trp, const int32_t* __restrict__ tci,
                 const double* __restrict__ tva, const double* __restrict__ winv, double drop_tol,
                 const int64_t* __restrict__ ooff, int32_t* __restrict__ cnt, int32_t* __restrict__ tcol,
                 double* __restrict__ tval, int32_t* __restrict__ overflow_rows, int32_t* __restrict__ n_overflow) {
    __shared__ Ev2Shared shm[kEv2Warps];
    const int w = threadIdx.x / kWarp, lane = threadIdx.x & (kWarp - 1);
    const int32_t i = blockIdx.x * kEv2Warps + w;
    if (i >= n) return;
    Ev2Shared& sh = shm[w];
    const int32_t alo = rp[i], na = rp[i + 1] - alo, tlo = trp[i], nt = trp[i + 1] - tlo;
    if (na > kEv2Cap || nt > kEv2Cap) {
        if (lane == 0) overflow_rows[atomicAdd(n_overflow, 1)] = i;
        return;
    }
    const double wi = winv[i];
    for (int32_t e = lane; e < na; e += kWarp) sh.acol[e] = ci[alo + e];
    for (int32_t e = lane; e < nt; e += kWarp) {
        const int32_t j = tci[tlo + e];
        sh.tcol[e] = j;
        sh.z1[e] = (j == i ? 1.0 : 0.0) - winv[j] * tva[tlo + e];
    }
    __syncwarp();
    // z1 at i when A(i, i) is not stored: 1 - winv_i * (+0)
    const int32_t ti = find_sorted(sh.tcol, nt, i);
    const double z1_i = ti >= 0 ? sh.z1[ti] : 1.0 - wi * 0.0;
    // z2 at a node u (rows in CSR order, z1 looked up on column i's pattern)
    auto z2_at = [&](int32_t u) -> double {
        const int32_t tu = u == i ? -2 : find_sorted(sh.tcol, nt, u);
        const double z1u = u == i ? z1_i : (tu >= 0 ? sh.z1[tu] : 0.0);
        double az = 0.0;
        const int32_t lo = rp[u], hi = rp[u + 1];
        for (int32_t p = lo; p < hi; ++p) {
            const int32_t j = ci[p];
            double zj;
            if (j == i) {
                zj = z1_i;
            } else {
                const int32_t k = find_sorted(sh.tcol, nt, j);
                if (k < 0) continue;
                zj = sh.z1[k];
            }
            az += va[p] * zj;
        }
        return z1u - winv[u] * az;
    };
    // ring = A row i U (A^T row i \ A row i); magnitudes |z2|, i excluded
    double mx = 0.0;
    for (int32_t e = lane; e < na; e += kWarp) {
        const int32_t j = sh.acol[e];
        const double m = j == i ? 0.0 : fabs(z2_at(j));
        sh.amag[e] = m;
        mx = fmax(mx, m);
    }
    for (int32_t e = lane; e < nt; e += kWarp) {
        const int32_t j = sh.tcol[e];
        const bool only = find_sorted(sh.acol, na, j) < 0;
        sh.tonly[e] = only ? 1 : 0;
        const double m = (only && j != i) ? fabs(z2_at(j)) : 0.0;
        sh.tmag[e] = m;
        mx = fmax(mx, m);
    }
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const double cutoff = mx / drop_tol;
    __syncwarp();
    for (int32_t e = lane; e < na; e += kWarp) {
        const double m = sh.amag[e];
        sh.aemit[e] = (sh.acol[e] != i && mx > 0.0 && m >= cutoff && m > 0.0) ? 1 : 0;
    }
    for (int32_t e = lane; e < nt; e += kWarp) {
        const double m = sh.tmag[e];
        sh.temit[e] = (sh.tonly[e] && sh.tcol[e] != i && mx > 0.0 && m >= cutoff && m > 0.0) ? 1 : 0;
    }
    __syncwarp();
    // flags -> positions: keep the flags in registers, prefix in place
    const int32_t a_tot = warp_prefix(sh.aemit, na, lane);
    const int32_t t_tot = warp_prefix(sh.temit, nt, lane);
    __syncwarp();
    // emitted count with column < key, over both lists (prefix arrays are exclusive)
    auto emitted_below = [&](int32_t key) -> int32_t {
        const int32_t pa = lower_bound_i32(sh.acol, 0, na, key);
        const int32_t pt = lower_bound_i32(sh.tcol, 0, nt, key);
        return (pa < na ? sh.aemit[pa] : a_tot) + (pt < nt ? sh.temit[pt] : t_tot);
    };
    int32_t* ocol = tcol + ooff[i];
    double* oval = tval + ooff[i];
    for (int32_t e = lane; e < na; e += kWarp) {
        const int32_t nxt = e + 1 < na ? sh.aemit[e + 1] : a_tot;
        if (nxt != sh.aemit[e]) {  // emitted
            const int32_t j = sh.acol[e];
            const int32_t at = emitted_below(j) + (j > i ? 1 : 0);
            ocol[at] = j;
            oval[at] = sh.amag[e];
        }
    }
    for (int32_t e = lane; e < nt; e += kWarp) {
        const int32_t nxt = e + 1 < nt ? sh.temit[e + 1] : t_tot;
        if (nxt != sh.temit[e]) {
            const int32_t j = sh.tcol[e];
            const int32_t at = emitted_below(j) + (j > i ? 1 : 0);
            ocol[at] = j;
            oval[at] = sh.tmag[e];
        }
    }
    if (lane == 0) {
        const double zi = fabs(z2_at(i));
        const int32_t at = emitted_below(i);
        ocol[at] = i;
        oval[at] = zi > 0.0 ? zi : 1.0;
        cnt[i] = a_tot + t_tot + 1;
    }
}

// WorkLedger count of evolution_strength (strength.hpp:176-194, count at 236):
// per row, `steps` times the sum over the distance-`steps` ball of (entries of
// the node's A row whose column lies in the ball + 1).  Same BFS as the generic
// kernel; rows whose ball overflows the shared capacity are listed for the host.
__global__ void __launch_bounds__(kEvWarps * kWarp)
    k_evolution_count(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                      const int32_t* __restrict__ trp, const int32_t* __restrict__ tci, int steps,
                      unsigned long long* __restrict__ total, int32_t* __restrict__ overflow_rows,
                      int32_t* __restrict__ n_overflow) {
    __shared__ EvShared shm[kEvWarps];
    const int w = threadIdx.x / kWarp, lane = threadIdx.x & (kWarp - 1);
    const int32_t i = blockIdx.x * kEvWarps + w;
    if (i >= n) return;
    EvShared& sh = shm[w];
    for (int s = lane; s < kEvHash; s += kWarp) sh.hkey[s] = -1;
    if (lane == 0) {
        sh.count = 0;
        sh.overflow = 0;
    }
    __syncwarp();
    if (lane == 0) h_insert(sh, i);
    __syncwarp();
    int32_t lo = 0;
    for (int st = 0; st < steps; ++st) {
        const int32_t hi = min(sh.count, kEvCap);
        for (int32_t f = lo; f < hi; ++f) {
            const int32_t u = sh.nodes[f];
            for (int32_t p = rp[u] + lane; p < rp[u + 1]; p += kWarp) h_insert(sh, ci[p]);
            for (int32_t p = trp[u] + lane; p < trp[u + 1]; p += kWarp) h_insert(sh, tci[p]);
        }
        __syncwarp();
        lo = hi;
        if (sh.overflow) break;
    }
    __syncwarp();
    if (sh.overflow) {
        if (lane == 0) overflow_rows[atomicAdd(n_overflow, 1)] = i;
        return;
    }
    unsigned long long cnt = 0;
    for (int32_t t = lane; t < sh.count; t += kWarp) {
        const int32_t u = sh.nodes[t];
        unsigned long long in = 1;
        for (int32_t p = rp[u]; p < rp[u + 1]; ++p)
            if (h_lookup(sh, ci[p]) >= 0) ++in;
        cnt += in;
    }
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if (lane == 0) atomicAdd(total, cnt * static_cast<unsigned long long>(steps));
}

// Fallback: block per row over a direct-mapped global scratch (local id per node).
constexpr int kEvBigThreads = 256;

__global__ void __launch_bounds__(kEvBigThreads)
    k_evolution_big(const int32_t* __restrict__ rows, int32_t n, const int32_t* __restrict__ rp,
                    const int32_t* __restrict__ ci, const double* __restrict__ va, const int32_t* __restrict__ trp,
                    const int32_t* __restrict__ tci, const double* __restrict__ winv, double drop_tol, int steps,
                    const int64_t* __restrict__ ooff, int32_t* __restrict__ cnt, int32_t* __restrict__ tcol,
                    double* __restrict__ tval, int32_t* __restrict__ gslot, int32_t* __restrict__ gnodes,
                    double* __restrict__ gz, double* __restrict__ gzn) {
    const int32_t i = rows[blockIdx.x];
    int32_t* slot = gslot + static_cast<int64_t>(blockIdx.x) * n;
    int32_t* nodes = gnodes + static_cast<int64_t>(blockIdx.x) * n;
    double* z = gz + static_cast<int64_t>(blockIdx.x) * n;
    double* zn = gzn + static_cast<int64_t>(blockIdx.x) * n;
    __shared__ int32_t count;
    __shared__ double red[kEvBigThreads / 32];
    for (int32_t t = threadIdx.x; t < n; t += blockDim.x) slot[t] = -1;
    __syncthreads();
    if (threadIdx.x == 0) {
        slot[i] = 0;
        nodes[0] = i;
        count = 1;
    }
    __syncthreads();
    int32_t lo = 0;
    for (int st = 0; st < steps; ++st) {
        const int32_t hi = count;
        __syncthreads();
        for (int32_t f = lo; f < hi; ++f) {
            const int32_t u = nodes[f];
            for (int32_t p = rp[u] + threadIdx.x; p < rp[u + 1]; p += blockDim.x) {
                const int32_t j = ci[p];
                if (atomicCAS(&slot[j], -1, -2) == -1) {
                    const int32_t id = atomicAdd(&count, 1);
                    nodes[id] = j;
                    atomicExch(&slot[j], id);
                }
            }
            for (int32_t p = trp[u] + threadIdx.x; p < trp[u + 1]; p += blockDim.x) {
                const int32_t j = tci[p];
                if (atomicCAS(&slot[j], -1, -2) == -1) {
                    const int32_t id = atomicAdd(&count, 1);
                    nodes[id] = j;
                    atomicExch(&slot[j], id);
                }
            }
            __syncthreads();
        }
        lo = hi;
    }
    __syncthreads();
    const int32_t nb = count;
    for (int32_t t = threadIdx.x; t < nb; t += blockDim.x) z[t] = (t == 0) ? 1.0 : 0.0;
    __syncthreads();
    for (int st = 0; st < steps; ++st) {
        for (int32_t t = threadIdx.x; t < nb; t += blockDim.x) {
            const int32_t u = nodes[t];
            double az = 0.0;
            for (int32_t p = rp[u]; p < rp[u + 1]; ++p) {
                const int32_t lj = slot[ci[p]];
                if (lj >= 0) az += va[p] * z[lj];
            }
            zn[t] = z[t] - winv[u] * az;
        }
        __syncthreads();
        double* tmp = z;
        z = zn;
        zn = tmp;
    }
    const int32_t alo = rp[i], ahi = rp[i + 1], tlo = trp[i], thi = trp[i + 1];
    const int32_t na = ahi - alo, nt = thi - tlo;
    auto ring_at = [&](int32_t e, bool* dup) -> int32_t {
        if (e < na) {
            *dup = false;
            return ci[alo + e];
        }
        const int32_t j = tci[tlo + e - na];
        const int32_t pos = lower_bound_i32(ci, alo, ahi, j);
        *dup = (pos < ahi && ci[pos] == j);
        return j;
    };
    double mx = 0.0;
    for (int32_t e = threadIdx.x; e < na + nt; e += blockDim.x) {
        bool dup;
        const int32_t j = ring_at(e, &dup);
        if (dup || j == i) continue;
        const int32_t lj = slot[j];
        if (lj >= 0) mx = fmax(mx, fabs(z[lj]));
    }
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
    __syncthreads();
    mx = 0.0;
    for (int t = 0; t < static_cast<int>(blockDim.x / 32); ++t) mx = fmax(mx, red[t]);
    const double cutoff = mx / drop_tol;
    const double zi = fabs(z[0]);
    const double dval = zi > 0.0 ? zi : 1.0;
    int32_t* ocol = tcol + ooff[i];
    double* oval = tval + ooff[i];
    __shared__ int32_t s_tot, s_below;
    if (threadIdx.x == 0) {
        s_tot = 0;
        s_below = 0;
    }
    __syncthreads();
    for (int32_t e = threadIdx.x; e < na + nt; e += blockDim.x) {
        bool dup;
        const int32_t j = ring_at(e, &dup);
        if (dup || j == i) continue;
        const int32_t lj = slot[j];
        const double mag = lj >= 0 ? fabs(z[lj]) : 0.0;
        if (!(mx > 0.0 && mag >= cutoff && mag > 0.0)) continue;
        atomicAdd(&s_tot, 1);
        if (j < i) atomicAdd(&s_below, 1);
        int32_t rank = 0;
        for (int32_t f = 0; f < na + nt; ++f) {
            bool d2;
            const int32_t jf = ring_at(f, &d2);
            if (d2 || jf >= j || jf == i) continue;
            const int32_t lf = slot[jf];
            const double mf = lf >= 0 ? fabs(z[lf]) : 0.0;
            rank += (mx > 0.0 && mf >= cutoff && mf > 0.0) ? 1 : 0;
        }
        const int32_t at = rank + (j > i ? 1 : 0);
        ocol[at] = j;
        oval[at] = mag;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ocol[s_below] = i;
        oval[s_below] = dval;
        cnt[i] = s_tot + 1;
    }
}

__global__ void k_ring_capacity(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ trp,
                                int64_t* __restrict__ cap) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    cap[i] = (rp[i + 1] - rp[i]) + (trp[i + 1] - trp[i]) + 1;
}

__global__ void k_copy_rows64(int32_t nr, const int64_t* __restrict__ off, const int32_t* __restrict__ tcol,
                              const double* __restrict__ tval, const int32_t* __restrict__ orp, int32_t* __restrict__ oci,
                              double* __restrict__ ova) {
    const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    if (i >= nr) return;
    const int64_t src = off[i];
    const int32_t dst = orp[i], len = orp[i + 1] - dst;
    for (int32_t e = lane; e < len; e += kWarp) {
        oci[dst + e] = tcol[src + e];
        ova[dst + e] = tval[src + e];
    }
}

template <typename CountK, typename... Args>
void two_pass(Ctx& c, int32_t n_out_rows, int32_t nc, int32_t bs, DCsr& S, CountK k, unsigned grid, unsigned block,
              Args... args) {
    DBuf<int32_t> cnt(static_cast<size_t>(n_out_rows) + 1, c.s);
    launch(c, k, grid, block, 0, args..., static_cast<const int32_t*>(nullptr), cnt.get(), static_cast<int32_t*>(nullptr),
           static_cast<double*>(nullptr));
    S.nr = n_out_rows;
    S.nc = nc;
    S.bs = bs;
    S.rp.alloc(static_cast<size_t>(n_out_rows) + 1, c.s);
    S.nnz = exclusive_scan_i32(c, cnt.get(), S.rp.get(), n_out_rows);
    S.ci.alloc(static_cast<size_t>(S.nnz), c.s);
    S.va.alloc(static_cast<size_t>(S.nnz), c.s);
    launch(c, k, grid, block, 0, args..., static_cast<const int32_t*>(S.rp.get()), cnt.get(), S.ci.get(), S.va.get());
}

}  // namespace

void symmetric_strength(Ctx& c, const DCsr& A, double theta, DCsr& S) {
    if (A.nr != A.nc) throw InvalidArgument("symmetric_strength: square matrix required");
    if (theta < 0.0 || theta > 1.0) throw InvalidArgument("symmetric_strength: theta must lie in [0, 1]");
    DBuf<double> d(static_cast<size_t>(A.nr), c.s);
    diagonal(c, A, d.get());
    // zero diagonal -> runtime_error with the lowest such row (strength.hpp:75-77)
    DBuf<double> dinv(static_cast<size_t>(A.nr), c.s);
    inverse_diagonal(c, A, dinv.get(), "symmetric_strength: zero diagonal at row ");
    two_pass(c, A.nr, A.nc, A.bs, S, k_soc<true>, blocks_for(A.nr, 128), 128, A.nr, A.rp.get(), A.ci.get(), A.va.get(),
             static_cast<const double*>(d.get()), theta);
    tally(c, static_cast<double>(A.nnz) + A.nr);  // strength.hpp:105
}

void classical_strength(Ctx& c, const DCsr& A, double theta, DCsr& S) {
    if (A.nr != A.nc) throw InvalidArgument("classical_strength: square matrix required");
    if (theta < 0.0 || theta > 1.0) throw InvalidArgument("classical_strength: theta must lie in [0, 1]");
    two_pass(c, A.nr, A.nc, A.bs, S, k_soc<false>, blocks_for(A.nr, 128), 128, A.nr, A.rp.get(), A.ci.get(),
             A.va.get(), static_cast<const double*>(nullptr), theta);
    tally(c, static_cast<double>(A.nr));  // strength.hpp:64
}

void normalize_strength(Ctx& c, const DCsr& S, DCsr& N) {
    if (S.nr != S.nc) throw InvalidArgument("normalize_strength: square matrix required");
    DBuf<int32_t> bad(1, c.s);
    AMG_CK(cudaMemsetAsync(bad.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_negative_check, blocks_for(S.nnz, 256), 256, 0, S.nnz, S.va.get(), bad.get());
    if (read_scalar(c, bad.get())) throw InvalidArgument("normalize_strength: negative strength value");
    two_pass(c, S.nr, S.nc, S.bs, N, k_normalize, blocks_for(S.nr, 128), 128, S.nr, S.rp.get(), S.ci.get(), S.va.get());
    tally(c, static_cast<double>(S.nnz));  // strength.hpp:286
}

void amalgamate(Ctx& c, const DCsr& S, int32_t m, DCsr& N) {
    if (m < 1) throw InvalidArgument("amalgamate: block size must be >= 1");
    if (m == 1) {
        clone_csr(c, S, N);
        return;
    }
    if (S.nr % m != 0 || S.nc % m != 0) throw InvalidArgument("amalgamate: dimensions not divisible by block size");
    const int32_t nn = S.nr / m;
    static const size_t long_smem = [] {
        const size_t b = kAmLongCap * sizeof(unsigned long long);
        AMG_CK(cudaFuncSetAttribute(k_amalgamate_long, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(b)));
        return b;
    }();
    DBuf<int32_t> cnt(static_cast<size_t>(nn) + 1, c.s), long_rows(static_cast<size_t>(nn), c.s), n_long(1, c.s);
    const unsigned long_grid = static_cast<unsigned>(c.sms * 2);
    auto pass = [&](const int32_t* orp, int32_t* oci, double* ova) {
        AMG_CK(cudaMemsetAsync(n_long.get(), 0, sizeof(int32_t), c.s));
        launch(c, k_amalgamate, blocks_for(nn, kAmWarps), kAmWarps * 32, 0, nn, m, S.rp.get(), S.ci.get(), S.va.get(),
               orp, cnt.get(), oci, ova, long_rows.get(), n_long.get());
        launch(c, k_amalgamate_long, long_grid, kAmLongThreads, long_smem, static_cast<const int32_t*>(long_rows.get()),
               static_cast<const int32_t*>(n_long.get()), m, S.rp.get(), S.ci.get(), S.va.get(), orp, cnt.get(), oci,
               ova);
    };
    pass(nullptr, nullptr, nullptr);
    N.nr = nn;
    N.nc = S.nc / m;
    N.bs = 1;
    N.rp.alloc(static_cast<size_t>(nn) + 1, c.s);
    N.nnz = exclusive_scan_i32(c, cnt.get(), N.rp.get(), nn);
    N.ci.alloc(static_cast<size_t>(N.nnz), c.s);
    N.va.alloc(static_cast<size_t>(N.nnz), c.s);
    pass(N.rp.get(), N.ci.get(), N.va.get());
}

EvoCount::~EvoCount() {
    if (done) {
        // the buffers are freed stream-ordered on s: after the count has read them
        cudaStreamWaitEvent(s, done, 0);
        cudaEventDestroy(done);
    }
}

std::unique_ptr<EvoCount> evolution_ops_start(Ctx& c, const DCsr& A, DCsr&& At, int steps) {
    const int32_t n = A.nr;
    auto e = std::make_unique<EvoCount>();
    e->steps = steps;
    e->s = c.s;
    e->At = std::move(At);
    e->total.alloc(1, c.s);
    e->ovf.alloc(static_cast<size_t>(n) + 1, c.s);
    e->novf.alloc(1, c.s);
    AMG_CK(cudaMemsetAsync(e->total.get(), 0, sizeof(unsigned long long), c.s));
    AMG_CK(cudaMemsetAsync(e->novf.get(), 0, sizeof(int32_t), c.s));
    cudaEvent_t ready;
    AMG_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    AMG_CK(cudaEventRecord(ready, c.s));
    AMG_CK(cudaStreamWaitEvent(c.side, ready, 0));
    cudaEventDestroy(ready);
    if (n > 0) {
        k_evolution_count<<<blocks_for(n, kEvWarps), kEvWarps * kWarp, 0, c.side>>>(
            n, A.rp.get(), A.ci.get(), e->At.rp.get(), e->At.ci.get(), steps, e->total.get(), e->ovf.get(),
            e->novf.get());
        ++c.launches;
        AMG_CK(cudaGetLastError());
    }
    AMG_CK(cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming));
    AMG_CK(cudaEventRecord(e->done, c.side));
    return e;
}

double evolution_ops_finish(Ctx& c, const DCsr& A, EvoCount& e) {
    const int32_t n = A.nr;
    const int steps = e.steps;
    AMG_CK(cudaStreamWaitEvent(c.s, e.done, 0));
    stage_scalar(c, 0, e.total.get());
    stage_scalar(c, 1, e.novf.get());
    sync(c);
    double ops = static_cast<double>(staged<unsigned long long>(c, 0));
    const int32_t nbig = staged<int32_t>(c, 1);
    if (nbig > 0) {  // large balls: the reference's BFS on the host
        const HostCsr ha = download_csr(c, A), ht = download_csr(c, e.At);
        std::vector<int32_t> rows(nbig), slot(n, -1), hood;
        copy_d2h(c, rows.data(), e.ovf.get(), nbig);
        sync(c);
        for (int32_t i : rows) {
            hood.assign(1, i);
            slot[i] = 0;
            size_t lo = 0;
            for (int st = 0; st < steps; ++st) {
                const size_t hi = hood.size();
                for (size_t f = lo; f < hi; ++f)
                    for (const HostCsr* M : {&ha, &ht})
                        for (int32_t p = M->row_offsets[hood[f]]; p < M->row_offsets[hood[f] + 1]; ++p)
                            if (slot[M->col_indices[p]] < 0) {
                                slot[M->col_indices[p]] = static_cast<int32_t>(hood.size());
                                hood.push_back(M->col_indices[p]);
                            }
                lo = hi;
            }
            double cnt = 0.0;
            for (int32_t u : hood) {
                cnt += 1.0;
                for (int32_t p = ha.row_offsets[u]; p < ha.row_offsets[u + 1]; ++p)
                    if (slot[ha.col_indices[p]] >= 0) cnt += 1.0;
            }
            ops += steps * cnt;
            for (int32_t u : hood) slot[u] = -1;
        }
    }
    return ops;
}

void evolution_strength(Ctx& c, const DCsr& A, const DCsr& At, const double* winv, double drop_tol, int steps,
                        DCsr& S) {
    const int32_t n = A.nr;
    DBuf<int64_t> cap(static_cast<size_t>(n) + 1, c.s), off(static_cast<size_t>(n) + 1, c.s);
    launch(c, k_ring_capacity, blocks_for(n, 256), 256, 0, n, A.rp.get(), At.rp.get(), cap.get());
    const int64_t total = exclusive_scan_i64(c, cap.get(), off.get(), n);
    DBuf<int32_t> tcol(static_cast<size_t>(total), c.s), cnt(static_cast<size_t>(n) + 1, c.s);
    DBuf<double> tval(static_cast<size_t>(total), c.s);
    DBuf<int32_t> ovf(static_cast<size_t>(n), c.s), novf(1, c.s);
    AMG_CK(cudaMemsetAsync(novf.get(), 0, sizeof(int32_t), c.s));
    const double ev_bytes = 12.0 * A.nnz + 8.0 * (n + 1) + 4.0 * At.nnz + 8.0 * n + 12.0 * total;
    if (steps == 2) {
        // hash-free two-step kernel; rows beyond its capacity go to the generic one
        DBuf<int32_t> ovf2(static_cast<size_t>(n), c.s), novf2(1, c.s);
        AMG_CK(cudaMemsetAsync(novf2.get(), 0, sizeof(int32_t), c.s));
        launch_prof(c, kProfEvolution, ev_bytes, k_evolution2, blocks_for(n, kEv2Warps), kEv2Warps * kWarp, 0, n,
                    A.rp.get(), A.ci.get(), A.va.get(), At.rp.get(), At.ci.get(), At.va.get(), winv, drop_tol,
                    static_cast<const int64_t*>(off.get()), cnt.get(), tcol.get(), tval.get(), ovf2.get(),
                    novf2.get());
        const int32_t n2 = read_scalar(c, novf2.get());
        if (n2 > 0)
            launch(c, k_evolution, blocks_for(n2, kEvWarps), kEvWarps * kWarp, 0, n, A.rp.get(), A.ci.get(),
                   A.va.get(), At.rp.get(), At.ci.get(), winv, drop_tol, steps,
                   static_cast<const int64_t*>(off.get()), cnt.get(), tcol.get(), tval.get(), ovf.get(), novf.get(),
                   static_cast<const int32_t*>(ovf2.get()), n2);
    } else {
        launch_prof(c, kProfEvolution, ev_bytes, k_evolution, blocks_for(n, kEvWarps), kEvWarps * kWarp, 0, n,
                    A.rp.get(), A.ci.get(), A.va.get(), At.rp.get(), At.ci.get(), winv, drop_tol, steps,
                    static_cast<const int64_t*>(off.get()), cnt.get(), tcol.get(), tval.get(), ovf.get(), novf.get(),
                    static_cast<const int32_t*>(nullptr), n);
    }
    const int32_t nbig = read_scalar(c, novf.get());
    if (nbig > 0) {
        const int32_t conc = std::min<int32_t>(nbig, 64);
        DBuf<int32_t> gslot(static_cast<size_t>(conc) * n, c.s), gnodes(static_cast<size_t>(conc) * n, c.s);
        DBuf<double> gz(static_cast<size_t>(conc) * n, c.s), gzn(static_cast<size_t>(conc) * n, c.s);
        for (int32_t b0 = 0; b0 < nbig; b0 += conc) {
            const int32_t nb = std::min(conc, nbig - b0);
            launch(c, k_evolution_big, static_cast<unsigned>(nb), kEvBigThreads, 0,
                   static_cast<const int32_t*>(ovf.get() + b0), n, A.rp.get(), A.ci.get(), A.va.get(), At.rp.get(),
                   At.ci.get(), winv, drop_tol, steps, static_cast<const int64_t*>(off.get()), cnt.get(), tcol.get(),
                   tval.get(), gslot.get(), gnodes.get(), gz.get(), gzn.get());
        }
    }
    S.nr = n;
    S.nc = n;
    S.bs = A.bs;
    S.rp.alloc(static_cast<size_t>(n) + 1, c.s);
    S.nnz = exclusive_scan_i32(c, cnt.get(), S.rp.get(), n);
    S.ci.alloc(static_cast<size_t>(S.nnz), c.s);
    S.va.alloc(static_cast<size_t>(S.nnz), c.s);
    launch(c, k_copy_rows64, blocks_for(static_cast<int64_t>(n) * kWarp, 256), 256, 0, n,
           static_cast<const int64_t*>(off.get()), static_cast<const int32_t*>(tcol.get()),
           static_cast<const double*>(tval.get()), static_cast<const int32_t*>(S.rp.get()), S.ci.get(), S.va.get());
}

}  // namespace amgcu
