// Interpolation on the GPU: pattern fixes, tentative injection, constraint
// projection, the pattern-masked product A X|_N, and energy minimisation with
// the CG loop kept entirely on the device (scalars and stop/restart flags live
// in device memory, so an iteration never waits on the host).
// Reference: interpolation.hpp, hierarchy.hpp:98-154.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bitrank.h"
#include "interp.cuh"
#include "small_dense.h"
#include "stl_sort.cuh"

namespace amgcu {

namespace {

constexpr int kKMax = 8;

__device__ __forceinline__ int32_t lower_bound_i32(const int32_t* a, int32_t lo, int32_t hi, int32_t key) {
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------------------------------
// add_aggregate_entries: insert (i, owner(i), 1.0) where missing
// ---------------------------------------------------------------------------------------
__global__ void k_add_agg(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ va, const int32_t* __restrict__ own,
                          const int32_t* __restrict__ orp, int32_t* __restrict__ cnt, int32_t* __restrict__ oci,
                          double* __restrict__ ova) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t g = own[i];
    const int32_t lo = rp[i], hi = rp[i + 1];
    const int32_t pos = lower_bound_i32(ci, lo, hi, g);
    const bool present = pos < hi && ci[pos] == g;
    if (!orp) {
        cnt[i] = (hi - lo) + (present ? 0 : 1);
        return;
    }
    int32_t o = orp[i];
    for (int32_t p = lo; p < hi; ++p) {
        if (!present && p == pos) {
            oci[o] = g;
            ova[o] = 1.0;
            ++o;
        }
        oci[o] = ci[p];
        ova[o] = va[p];
        ++o;
    }
    if (!present && pos == hi) {
        oci[o] = g;
        ova[o] = 1.0;
    }
}

__global__ void k_any_missing(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const int32_t* __restrict__ own, int32_t* __restrict__ flag) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t pos = lower_bound_i32(ci, rp[i], rp[i + 1], own[i]);
    if (!(pos < rp[i + 1] && ci[pos] == own[i])) atomicExch(flag, 1);
}


// ---------------------------------------------------------------------------------------
// widen_deficient_rows: block per deficient row, whole-level BFS over S and S^T
// ---------------------------------------------------------------------------------------
constexpr int kWidenThreads = 256;
constexpr int kWidenAggCap = 1024;

__global__ void k_deficient(int32_t n, const int32_t* __restrict__ rp, int32_t min_aggs, int32_t* __restrict__ list,
                            int32_t* __restrict__ count) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && rp[i + 1] - rp[i] < min_aggs) list[atomicAdd(count, 1)] = i;
}

__global__ void __launch_bounds__(kWidenThreads)
    k_widen(const int32_t* __restrict__ rows, int32_t nn, const int32_t* __restrict__ nrp, const int32_t* __restrict__ nci,
            const int32_t* __restrict__ srp, const int32_t* __restrict__ sci, const int32_t* __restrict__ trp,
            const int32_t* __restrict__ tci, const int32_t* __restrict__ own, int32_t min_aggs,
            int32_t* __restrict__ gseen, int32_t* __restrict__ gfront, int32_t* __restrict__ xcols,
            int32_t* __restrict__ xcnt, int32_t* __restrict__ xbase, int32_t b0, int32_t* __restrict__ err) {
    const int32_t i = rows[blockIdx.x];
    int32_t* seen = gseen + static_cast<int64_t>(blockIdx.x) * nn;
    int32_t* fa = gfront + static_cast<int64_t>(blockIdx.x) * 2 * nn;
    int32_t* fb = fa + nn;
    __shared__ int32_t aggs[kWidenAggCap];
    __shared__ int32_t naggs, nfront, nnext;
    for (int32_t t = threadIdx.x; t < nn; t += blockDim.x) seen[t] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        naggs = 0;
        for (int32_t p = nrp[i]; p < nrp[i + 1] && naggs < kWidenAggCap; ++p) aggs[naggs++] = nci[p];
        seen[i] = 1;
        fa[0] = i;
        nfront = 1;
    }
    __syncthreads();
    while (nfront > 0 && naggs < min_aggs) {
        if (threadIdx.x == 0) nnext = 0;
        __syncthreads();
        for (int32_t f = 0; f < nfront; ++f) {
            const int32_t u = fa[f];
            for (int pass = 0; pass < 2; ++pass) {
                const int32_t* rp = pass ? trp : srp;
                const int32_t* cj = pass ? tci : sci;
                for (int32_t p = rp[u] + threadIdx.x; p < rp[u + 1]; p += blockDim.x) {
                    const int32_t j = cj[p];
                    if (atomicCAS(&seen[j], 0, 1) != 0) continue;
                    fb[atomicAdd(&nnext, 1)] = j;
                    const int32_t at = atomicAdd(&naggs, 1);  // duplicates removed below
                    if (at < kWidenAggCap) aggs[at] = own[j];
                    else atomicExch(err, 1);
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            int32_t w = 0;
            const int32_t m0 = min(naggs, kWidenAggCap);
            for (int32_t t = 0; t < m0; ++t) {
                bool dup = false;
                for (int32_t u2 = 0; u2 < w; ++u2)
                    if (aggs[u2] == aggs[t]) {
                        dup = true;
                        break;
                    }
                if (!dup) aggs[w++] = aggs[t];
            }
            naggs = w;
            nfront = nnext;
        }
        __syncthreads();
        int32_t* tmp = fa;
        fa = fb;
        fb = tmp;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int32_t base = (b0 + blockIdx.x) * kWidenAggCap;
        int32_t cnt = 0;
        for (int32_t t = 0; t < naggs; ++t) {
            const int32_t g = aggs[t];
            const int32_t pos = lower_bound_i32(nci, nrp[i], nrp[i + 1], g);
            if (pos < nrp[i + 1] && nci[pos] == g) continue;
            // insertion keeps the extras of the row ascending
            int32_t q = cnt++;
            while (q > 0 && xcols[base + q - 1] > g) {
                xcols[base + q] = xcols[base + q - 1];
                --q;
            }
            xcols[base + q] = g;
        }
        xcnt[i] = cnt;
        xbase[i] = base;
    }
}

// N plus the extra (col, 1.0) entries of the widened rows, merged ascending
__global__ void k_widen_merge(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const double* __restrict__ va, const int32_t* __restrict__ xcols,
                              const int32_t* __restrict__ xcnt, const int32_t* __restrict__ xbase,
                              const int32_t* __restrict__ orp, int32_t* __restrict__ cnt, int32_t* __restrict__ oci,
                              double* __restrict__ ova) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t ne = xcnt[i];
    if (!orp) {
        cnt[i] = rp[i + 1] - rp[i] + ne;
        return;
    }
    int32_t o = orp[i], p = rp[i], e = 0;
    const int32_t* x = xcols + (ne ? xbase[i] : 0);
    while (p < rp[i + 1] || e < ne) {
        if (e < ne && (p == rp[i + 1] || x[e] < ci[p])) {
            oci[o] = x[e];
            ova[o] = 1.0;
            ++e;
        } else {
            oci[o] = ci[p];
            ova[o] = va[p];
            ++p;
        }
        ++o;
    }
}

// ---------------------------------------------------------------------------------------
// unamalgamate (m > 1) and root_node_pattern
// ---------------------------------------------------------------------------------------
__global__ void k_unamalg_rp(int32_t nn, int32_t m, const int32_t* __restrict__ rp, int32_t* __restrict__ cnt) {
    const int32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= nn * m) return;
    const int32_t i = d / m;
    cnt[d] = (rp[i + 1] - rp[i]) * m;
}

__global__ void k_unamalg(int32_t nn, int32_t m, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ va, const int32_t* __restrict__ drp, int32_t* __restrict__ dci,
                          double* __restrict__ dva) {
    const int32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= nn * m) return;
    const int32_t i = d / m;
    int32_t o = drp[d];
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p)
        for (int32_t c = 0; c < m; ++c) {
            dci[o] = ci[p] * m + c;
            dva[o] = va[p];
            ++o;
        }
}

__global__ void k_droots(int32_t na, int32_t m, const int32_t* __restrict__ roots, int32_t* __restrict__ dr) {
    const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= na) return;
    for (int32_t c = 0; c < m; ++c) dr[g * m + c] = roots[g] * m + c;
}

__global__ void k_owner_of_root(int32_t nroots, const int32_t* __restrict__ roots, int32_t* __restrict__ owner,
                                int32_t nrows, int32_t* __restrict__ err) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nroots) return;
    const int32_t r = roots[j];
    if (r < 0 || r >= nrows) {
        atomicExch(err, 1);
        return;
    }
    if (atomicCAS(&owner[r], -1, j) != -1) atomicExch(err, 2);
}

__global__ void k_rootpat(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ va, const int32_t* __restrict__ owner,
                          const int32_t* __restrict__ orp, int32_t* __restrict__ cnt, int32_t* __restrict__ oci,
                          double* __restrict__ ova) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t ow = owner[i];
    if (!orp) {
        cnt[i] = ow >= 0 ? 1 : rp[i + 1] - rp[i];
        return;
    }
    int32_t o = orp[i];
    if (ow >= 0) {
        oci[o] = ow;
        ova[o] = 1.0;
        return;
    }
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        oci[o] = ci[p];
        ova[o] = va[p];
        ++o;
    }
}

// ---------------------------------------------------------------------------------------
// inject_tentative
// ---------------------------------------------------------------------------------------
__global__ void k_root_blocks(int32_t na, int32_t m, int32_t k, int32_t ndof, const int32_t* __restrict__ roots,
                              const double* __restrict__ B, double* __restrict__ binv, double* __restrict__ Bc,
                              int32_t nc, int32_t* __restrict__ degenerate) {
    const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= na) return;
    const int32_t root = roots[g];
    double blk[64];
    double mx = 0.0;
    for (int r = 0; r < m; ++r)
        for (int cc = 0; cc < m; ++cc) {
            const double v = B[static_cast<size_t>(cc) * ndof + root * m + r];
            blk[r * m + cc] = v;
            const double a = fabs(v);
            mx = (r == 0 && cc == 0) ? a : (mx < a ? a : mx);
        }
    sd::FullPivLU<8> lu;
    lu.compute(m, blk);
    const double scale_cut = 1e-10 * sd::dmax(mx, 1e-300);
    double cut = 1.0;
    for (int t = 0; t < m; ++t) cut *= scale_cut;  // pow(scale_cut, m)
    if (m == 1) cut = scale_cut;
    double* inv = binv + static_cast<size_t>(g) * m * m;
    if (lu.rank() == m && mx > 0 && fabs(lu.determinant()) > cut) {
        lu.inverse(inv);
    } else if (m == 1) {
        inv[0] = 0.0;  // COD pseudo-inverse of the zero 1x1 block
    } else {
        atomicAdd(degenerate, 1);
        for (int t = 0; t < m * m; ++t) inv[t] = nan("");
    }
    for (int cc = 0; cc < m; ++cc)
        for (int a = 0; a < k; ++a)
            Bc[static_cast<size_t>(a) * nc + g * m + cc] = B[static_cast<size_t>(a) * ndof + root * m + cc];
}

__global__ void k_tentative_rows(int32_t nn, int32_t m, const int32_t* __restrict__ own,
                                 const int32_t* __restrict__ roots, const double* __restrict__ B, int32_t ndof,
                                 const double* __restrict__ binv, const int32_t* __restrict__ orp,
                                 int32_t* __restrict__ cnt, int32_t* __restrict__ oci, double* __restrict__ ova) {
    const int32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= nn * m) return;
    const int32_t i = d / m, r = d - i * m;
    const int32_t g = own[i];
    const bool is_root = roots[g] == i;
    int32_t o = orp ? orp[d] : 0;
    if (is_root) {
        if (orp) {
            oci[o] = g * m + r;
            ova[o] = 1.0;
        }
        ++o;
    } else {
        const double* inv = binv + static_cast<size_t>(g) * m * m;
        for (int32_t cc = 0; cc < m; ++cc) {
            double v = 0.0;
            for (int32_t s = 0; s < m; ++s) v += B[static_cast<size_t>(s) * ndof + d] * inv[s * m + cc];
            if (v != 0.0) {
                if (orp) {
                    oci[o] = g * m + cc;
                    ova[o] = v;
                }
                ++o;
            }
        }
    }
    if (!orp) cnt[d] = o;
}

// ---------------------------------------------------------------------------------------
// scatter_into_pattern (interpolation.hpp:213-227)
// ---------------------------------------------------------------------------------------
__global__ void k_scatter_pattern(int32_t n, const int32_t* __restrict__ trp, const int32_t* __restrict__ tci,
                                  const double* __restrict__ tva, const int32_t* __restrict__ nrp,
                                  const int32_t* __restrict__ nci, double* __restrict__ vals, int32_t* __restrict__ err) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int32_t p = nrp[i]; p < nrp[i + 1]; ++p) vals[p] = 0.0;
    for (int32_t p = trp[i]; p < trp[i + 1]; ++p) {
        const int32_t pos = lower_bound_i32(nci, nrp[i], nrp[i + 1], tci[p]);
        if (pos == nrp[i + 1] || nci[pos] != tci[p]) {
            atomicExch(err, 1);
            return;
        }
        vals[pos] = tva[p];
    }
}

// ---------------------------------------------------------------------------------------
// enforce_constraints, thread per row (interpolation.hpp:467-518)
// ---------------------------------------------------------------------------------------
__global__ void k_enforce(int32_t n, int32_t k, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          double* __restrict__ vals, const double* __restrict__ B, const double* __restrict__ Bc,
                          int32_t nc) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t lo = rp[i], hi = rp[i + 1];
    if (lo == hi) return;
    double G[kKMax * kKMax], y[kKMax], ev[kKMax], V[kKMax * kKMax], proj[kKMax], lv[kKMax];
    for (int t = 0; t < k * k; ++t) G[t] = 0.0;
    for (int a = 0; a < k; ++a) y[a] = 0.0;
    for (int32_t p = lo; p < hi; ++p) {
        const int32_t j = ci[p];
        for (int a = 0; a < k; ++a) {
            const double ba = Bc[static_cast<size_t>(a) * nc + j];
            y[a] += ba * vals[p];
            for (int b = a; b < k; ++b) G[a * k + b] += ba * Bc[static_cast<size_t>(b) * nc + j];
        }
    }
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < a; ++b) G[a * k + b] = G[b * k + a];
    for (int a = 0; a < k; ++a) y[a] = B[static_cast<size_t>(a) * n + i] - y[a];
    sd::sym_eig<kKMax>(k, G, ev, V);
    double mx = fabs(ev[0]);
    for (int a = 0; a < k; ++a) mx = sd::dmax(mx, fabs(ev[a]));
    const double cutoff = 1e-12 * sd::dmax(mx, 1e-300);
    for (int t = 0; t < k; ++t) {
        double s = 0.0;
        for (int a = 0; a < k; ++a) s += V[a * k + t] * y[a];
        proj[t] = s;
    }
    for (int a = 0; a < k; ++a) proj[a] = ev[a] > cutoff ? proj[a] / ev[a] : 0.0;
    for (int a = 0; a < k; ++a) {
        double s = 0.0;
        for (int t = 0; t < k; ++t) s += V[a * k + t] * proj[t];
        lv[a] = s;
    }
    for (int32_t p = lo; p < hi; ++p) {
        double s = 0.0;
        for (int a = 0; a < k; ++a) s += Bc[static_cast<size_t>(a) * nc + ci[p]] * lv[a];
        vals[p] += s;
    }
}

// ---------------------------------------------------------------------------------------
// ConstraintWorkspace::build (interpolation.hpp:113-141): Gp per non-root row
// ---------------------------------------------------------------------------------------
__global__ void k_gram_pinv(int32_t n, int32_t k, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ Bc, int32_t nc, const unsigned char* __restrict__ is_root,
                            double* __restrict__ gp) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double* out = gp + static_cast<size_t>(i) * k * k;
    if (is_root[i]) {
        for (int t = 0; t < k * k; ++t) out[t] = 0.0;
        return;
    }
    double G[kKMax * kKMax];
    for (int t = 0; t < k * k; ++t) G[t] = 0.0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = ci[p];
        for (int a = 0; a < k; ++a)
            for (int b = a; b < k; ++b)
                G[a * k + b] += Bc[static_cast<size_t>(a) * nc + j] * Bc[static_cast<size_t>(b) * nc + j];
    }
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < a; ++b) G[a * k + b] = G[b * k + a];
    sd::sym_pinv<kKMax>(k, G, out);
}

__global__ void k_root_mask(int32_t nroots, const int32_t* __restrict__ roots, unsigned char* __restrict__ mask) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nroots) mask[roots[j]] = 1;
}

// ---- WorkLedger counts (computed only when a ledger sink is active) ----------------------
// masked_product's count (interpolation.hpp:200-206): sum_i sum_{t in A row i} |N_i ∩ N_t|
__global__ void k_masked_count(int32_t n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                               const int32_t* __restrict__ nrp, const int32_t* __restrict__ nci,
                               unsigned long long* __restrict__ out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long cnt = 0;
    if (i < n && nrp[i] < nrp[i + 1]) {
        const int32_t lo = nrp[i], hi = nrp[i + 1];
        for (int32_t p = arp[i]; p < arp[i + 1]; ++p) {
            const int32_t t = aci[p];
            int32_t a = lo, b = nrp[t];
            const int32_t be = nrp[t + 1];
            while (a < hi && b < be) {
                const int32_t x = nci[a], y = nci[b];
                if (x == y) {
                    ++cnt;
                    ++a;
                    ++b;
                } else if (x < y) {
                    ++a;
                } else {
                    ++b;
                }
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

// rows (and their lengths) that are not roots / that are not empty
__global__ void k_row_census(int32_t n, const int32_t* __restrict__ rp, const unsigned char* __restrict__ is_root,
                             unsigned long long* __restrict__ out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nr = 0, len = 0, ne = 0;
    if (i < n) {
        const int32_t l = rp[i + 1] - rp[i];
        if (!is_root || !is_root[i]) {
            nr = 1;
            len = static_cast<unsigned long long>(l);
        }
        ne = l > 0 ? 1 : 0;
    }
    for (int off = 16; off > 0; off >>= 1) {
        nr += __shfl_xor_sync(0xffffffffu, nr, off);
        len += __shfl_xor_sync(0xffffffffu, len, off);
        ne += __shfl_xor_sync(0xffffffffu, ne, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, nr);
        atomicAdd(out + 1, len);
        atomicAdd(out + 2, ne);
    }
}

struct RowCensus {
    double rows = 0.0, len = 0.0, nonempty = 0.0;
};

RowCensus row_census(Ctx& c, const DCsr& N, const unsigned char* is_root) {
    DBuf<unsigned long long> o(3, c.s);
    AMG_CK(cudaMemsetAsync(o.get(), 0, sizeof(unsigned long long) * 3, c.s));
    launch(c, k_row_census, blocks_for(N.nr, 256), 256, 0, N.nr, N.rp.get(), is_root, o.get());
    unsigned long long h[3];
    copy_d2h(c, h, o.get(), 3);
    sync(c);
    return {static_cast<double>(h[0]), static_cast<double>(h[1]), static_cast<double>(h[2])};
}

double masked_count(Ctx& c, const DCsr& A, const DCsr& N) {
    DBuf<unsigned long long> o(1, c.s);
    AMG_CK(cudaMemsetAsync(o.get(), 0, sizeof(unsigned long long), c.s));
    launch(c, k_masked_count, blocks_for(N.nr, 128), 128, 0, N.nr, A.rp.get(), A.ci.get(), N.rp.get(), N.ci.get(),
           o.get());
    return static_cast<double>(read_scalar(c, o.get()));
}

// ---------------------------------------------------------------------------------------
// Masked product Y = (A X)|_N (interpolation.hpp:186-210) with the constraint
// projection (150-182) fused.  Y (unprojected) and Yp (projected) are written
// when the pointer is non-null.
// ---------------------------------------------------------------------------------------
// Thread-per-row masked product + projection (reference arithmetic): the row's pattern slots are taken in chunks of kMrChunk
// held in registers; for every A entry (CSR order) the slot columns are merged
// against the sorted row N_t with two pointers.  Rows of N are short (3-8
// slots on the BASELINE configs), so one thread per row keeps every lane busy.
constexpr int kMrChunk = 8;
constexpr int kMrNt = 8;  // rows of N up to this length are merged from registers

__global__ void __launch_bounds__(128)
    k_masked_rows(int32_t n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                  const double* __restrict__ ava, const int32_t* __restrict__ nrp, const int32_t* __restrict__ nci,
                  const double* __restrict__ x, int32_t k, const double* __restrict__ Bc, int32_t nc,
                  const double* __restrict__ gp, const unsigned char* __restrict__ is_root, double* __restrict__ y,
                  double* __restrict__ yp, const int32_t* __restrict__ stop) {
    if (stop && *stop) return;
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t lo = nrp[i], L = nrp[i + 1] - lo;
    if (L == 0) return;
    const int32_t alo = arp[i], ahi = arp[i + 1];
    double* dst = y ? y : yp;  // unprojected values (scratch in yp when y is not wanted)
    double keep[kMrChunk];     // last chunk's values, reused by the projection when L <= kMrChunk
    for (int32_t c0 = 0; c0 < L; c0 += kMrChunk) {
        const int32_t m = min(kMrChunk, L - c0);
        int32_t cols[kMrChunk];
        double acc[kMrChunk];
#pragma unroll
        for (int s = 0; s < kMrChunk; ++s) {
            cols[s] = s < m ? nci[lo + c0 + s] : 0x7fffffff;
            acc[s] = 0.0;
        }
        for (int32_t p = alo; p < ahi; ++p) {
            const int32_t t = __ldg(&aci[p]);
            const double a = __ldg(&ava[p]);
            const int32_t q0 = __ldg(&nrp[t]);
            const int32_t qe = __ldg(&nrp[t + 1]);
            if (qe - q0 <= kMrNt) {
                // N_t in registers: one batch of column loads, matches by comparison,
                // then only the matching x values are gathered (all independent)
                int32_t nt[kMrNt];
#pragma unroll
                for (int u = 0; u < kMrNt; ++u) nt[u] = q0 + u < qe ? __ldg(&nci[q0 + u]) : -1;
                int32_t hit[kMrChunk];
#pragma unroll
                for (int s2 = 0; s2 < kMrChunk; ++s2) {
                    hit[s2] = -1;
#pragma unroll
                    for (int u = 0; u < kMrNt; ++u)
                        if (nt[u] == cols[s2]) hit[s2] = q0 + u;
                }
                double xv[kMrChunk];
#pragma unroll
                for (int s2 = 0; s2 < kMrChunk; ++s2) xv[s2] = (s2 < m && hit[s2] >= 0) ? __ldg(&x[hit[s2]]) : 0.0;
#pragma unroll
                for (int s2 = 0; s2 < kMrChunk; ++s2)
                    if (s2 < m && hit[s2] >= 0) acc[s2] += a * xv[s2];
            } else {
                int32_t q = q0;
#pragma unroll
                for (int s2 = 0; s2 < kMrChunk; ++s2) {
                    if (s2 < m) {
                        while (q < qe && nci[q] < cols[s2]) ++q;
                        if (q < qe && nci[q] == cols[s2]) acc[s2] += a * x[q];
                    }
                }
            }
        }
#pragma unroll
        for (int s = 0; s < kMrChunk; ++s)
            if (s < m) {
                dst[lo + c0 + s] = acc[s];
                keep[s] = acc[s];
            }
    }
    if (!yp) return;
    if (is_root[i]) {
        for (int32_t e = 0; e < L; ++e) yp[lo + e] = 0.0;
        return;
    }
    double ya[kKMax], lam[kKMax];
    for (int a = 0; a < k; ++a) ya[a] = 0.0;
    const bool in_regs = L <= kMrChunk;
    for (int32_t e = 0; e < L; ++e) {
        double v = 0.0;
        if (in_regs) {
#pragma unroll
            for (int s = 0; s < kMrChunk; ++s)
                if (s == e) v = keep[s];
        } else {
            v = dst[lo + e];
        }
        const int32_t cj = nci[lo + e];
        for (int a = 0; a < k; ++a) ya[a] += Bc[static_cast<size_t>(a) * nc + cj] * v;
    }
    const double* G = gp + static_cast<size_t>(i) * k * k;
    for (int a = 0; a < k; ++a) {
        double s2 = 0.0;
        for (int b2 = 0; b2 < k; ++b2) s2 += G[a * k + b2] * ya[b2];
        lam[a] = s2;
    }
    for (int32_t e = 0; e < L; ++e) {
        double v = 0.0;
        if (in_regs) {
#pragma unroll
            for (int s = 0; s < kMrChunk; ++s)
                if (s == e) v = keep[s];
        } else {
            v = dst[lo + e];
        }
        const int32_t cj = nci[lo + e];
        double t2 = 0.0;
        for (int a = 0; a < k; ++a) t2 += Bc[static_cast<size_t>(a) * nc + cj] * lam[a];
        yp[lo + e] = v - t2;
    }
}

// in-place projection of vals (project_to_constraints)
__global__ void k_project(int32_t n, const int32_t* __restrict__ nrp, const int32_t* __restrict__ nci, int32_t k,
                          const double* __restrict__ Bc, int32_t nc, const double* __restrict__ gp,
                          const unsigned char* __restrict__ is_root, double* __restrict__ vals) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t lo = nrp[i], hi = nrp[i + 1];
    if (is_root[i]) {
        for (int32_t p = lo; p < hi; ++p) vals[p] = 0.0;
        return;
    }
    double ya[kKMax], lam[kKMax];
    for (int a = 0; a < k; ++a) ya[a] = 0.0;
    for (int32_t p = lo; p < hi; ++p)
        for (int a = 0; a < k; ++a) ya[a] += Bc[static_cast<size_t>(a) * nc + nci[p]] * vals[p];
    const double* G = gp + static_cast<size_t>(i) * k * k;
    for (int a = 0; a < k; ++a) {
        double s = 0.0;
        for (int b = 0; b < k; ++b) s += G[a * k + b] * ya[b];
        lam[a] = s;
    }
    for (int32_t p = lo; p < hi; ++p) {
        double s = 0.0;
        for (int a = 0; a < k; ++a) s += Bc[static_cast<size_t>(a) * nc + nci[p]] * lam[a];
        vals[p] -= s;
    }
}

#include "masked_band.cuh"

// AMGCU_MASKED_BAND=0 keeps the register-merge kernel on every level (A/B runs)
bool masked_band_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("AMGCU_MASKED_BAND");
        return !(e && e[0] == '0');
    }();
    return on;
}

// blocks of k_cg_columns: the window of columns in flight (AMGCU_CGCOL_BLOCKS_PER_SM, default 4:
// 32 columns per block of 128 threads; C5 level 0: 345 us and 0.76 GB at 4, 360 us at 3, 385 us
// and 1.25 GB at 8)
unsigned cg_column_blocks(const Ctx& c) {
    static const int per_sm = [] {
        const char* e = std::getenv("AMGCU_CGCOL_BLOCKS_PER_SM");
        const int v = e ? std::atoi(e) : 4;
        return v > 0 ? v : 4;
    }();
    return static_cast<unsigned>(c.sms * per_sm);
}

using BandKernel = void (*)(int32_t, int32_t, int32_t, int32_t, int32_t, const int32_t*, const mband::Rec*, const int32_t*,
                            const int32_t*, const double*, int32_t, const double*, int32_t, const double*,
                            const unsigned char*, double*, double*, const mband::Run*, const int32_t*, const int32_t*);
template <int MODE>
BandKernel band_kernel_k(int32_t k) {
    switch (k) {
        case 1: return mband::k_masked_band<1, MODE>;
        case 2: return mband::k_masked_band<2, MODE>;
        case 3: return mband::k_masked_band<3, MODE>;
        default: return mband::k_masked_band<0, MODE>;
    }
}
BandKernel band_kernel(int32_t k, int mode) {
    return mode == mband::kNibbles ? band_kernel_k<mband::kNibbles>(k)
           : mode == mband::kMasks ? band_kernel_k<mband::kMasks>(k)
                                   : band_kernel_k<mband::kDirect>(k);
}

// The plan of the band-staged masked product for (A, N): runs per CTA, records per A entry.
// Rows per CTA: from the average row lengths, halved while the runs of some CTA do not fit
// the run table or the shared-memory budget (one host synchronisation per attempt).
mband::Plan masked_band_plan(Ctx& c, const DCsr& A, const DCsr& N, int32_t k) {
    mband::Plan pl;
    const int32_t n = N.nr;
    if (!masked_band_enabled() || c.band_min_rows < 0 || n < c.band_min_rows || A.nnz == 0 || N.nnz == 0) return pl;
    const double da = static_cast<double>(A.nnz) / n, ln = static_cast<double>(N.nnz) / n;
    const double per_row = 16.0 * da + 8.0 * ln * 4.5 + 16.0;
    int32_t R = 128;
    while (R > 4 && R * per_row > 44.0 * 1024.0) R >>= 1;
    // long operator rows leave a CTA with fewer slots than threads: take the rows that fill
    // one pass of the block if they fit 64 KB (C4 level 1: 2.30 -> 1.56 ms per product)
    if (R * ln < 0.75 * mband::kThreads) {
        const int32_t fit = std::min<int32_t>(128, static_cast<int32_t>(0.94 * mband::kThreads / ln));
        if (fit > R && fit * per_row <= 64.0 * 1024.0) R = fit;
    }
    const bool trace = std::getenv("AMGCU_BAND_TRACE") != nullptr;
    DBuf<int32_t> info(8, c.s);
    int32_t h[8];
    auto refuse = [&](int why) {
        ++c.band_refused;
        c.band_last_fail = why;
        return mband::Plan{};
    };
    auto run_k_runs = [&](int direct) {
        pl.R = R;
        pl.nctas = static_cast<int32_t>(blocks_for(n, R));
        pl.runs.alloc(static_cast<size_t>(pl.nctas) * mband::kMaxRuns, c.s);
        pl.nruns.alloc(static_cast<size_t>(pl.nctas) * 2, c.s);
        AMG_CK(cudaMemsetAsync(info.get(), 0, sizeof(int32_t) * 8, c.s));
        launch_prof(c, kProfEminCg, 0.0, mband::k_runs, static_cast<unsigned>(pl.nctas), mband::kThreads, 0, n, R,
                    A.rp.get(), A.ci.get(), N.rp.get(), pl.runs.get(), pl.nruns.get(), info.get(), direct);
        copy_d2h(c, h, info.get(), 8);
        sync(c);
        pl.cap_a = h[1];
        pl.cap_x = h[2];
        pl.cap_s = h[3];
        pl.smem = mband::smem_bytes(R, pl.cap_a, pl.cap_x, pl.cap_s, k);
        if (trace)
            std::fprintf(stderr, "[band] n %d nnzA %lld nnzN %lld k %d R %d direct %d fail %d cap_a %d cap_x %d cap_s %d longest %d smem %zu\n",
                         n, static_cast<long long>(A.nnz), static_cast<long long>(N.nnz), k, R, direct, h[0], h[1], h[2],
                         h[3], h[4], pl.smem);
    };
    bool direct = false;
    for (;; R >>= 1) {
        run_k_runs(0);
        if (h[4] > mband::kMaskSlots) return refuse(8);
        if (h[0] == 0 && pl.smem <= mband::kSmemBudget) break;
        if (R <= 4) {
            // scattered references: no staging, x gathered from global memory (L2)
            if (h[4] > mband::kDirectSlots || N.nnz >= (int64_t(1) << 31)) return refuse(h[0] ? h[0] : 64);
            const double per_row_direct = 16.0 * da + 8.0 * ln * 2.0 + 16.0;
            R = 128;
            while (R > 4 && R * per_row_direct > 44.0 * 1024.0) R >>= 1;
            run_k_runs(1);
            if (pl.smem > mband::kSmemBudget) return refuse(64);
            direct = true;
            break;
        }
    }
    pl.mode = direct ? mband::kDirect : h[4] > mband::kNibSlots ? mband::kMasks : mband::kNibbles;
    pl.recs.alloc(static_cast<size_t>(A.nnz) + 1, c.s);
    pl.matches.alloc(1, c.s);
    AMG_CK(cudaMemsetAsync(pl.matches.get(), 0, sizeof(unsigned long long), c.s));
    AMG_CK(cudaMemsetAsync(info.get(), 0, sizeof(int32_t) * 8, c.s));
    auto records = [&](auto kern) {
        launch_prof(c, kProfEminCg, 0.0, kern, static_cast<unsigned>(pl.nctas), mband::kThreads, 0, n, R, A.rp.get(),
                    A.ci.get(), A.va.get(), N.rp.get(), N.ci.get(), static_cast<const mband::Run*>(pl.runs.get()),
                    static_cast<const int32_t*>(pl.nruns.get()), pl.recs.get(), info.get(), pl.matches.get());
    };
    if (pl.mode == mband::kDirect) records(mband::k_records<mband::kDirect>);
    else if (pl.mode == mband::kMasks) records(mband::k_records<mband::kMasks>);
    else records(mband::k_records<mband::kNibbles>);
    // a record that found no run (cannot happen: the runs cover every referenced row) is
    // reported with the hierarchy's other deferred checks: the flag is read with the CG's own
    // final synchronisation through pl.info
    pl.info = std::move(info);
    static bool attr_set[12] = {};
    const int slot = (k >= 1 && k <= 3 ? k : 0) * 3 + pl.mode;
    if (!attr_set[slot]) {
        AMG_CK(cudaFuncSetAttribute(band_kernel(k, pl.mode), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(mband::kSmemBudget)));
        attr_set[slot] = true;
    }
    pl.ok = true;
    ++c.band_accepted;
    return pl;
}

__global__ void k_negate(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < n) y[p] = -x[p];
}

// ---------------------------------------------------------------------------------------
// CG (interpolation.hpp:298-361) with device-side control
//   st[0] newsum  st[1] oldsum  st[2] first  st[3] denom  st[4] alpha_cg
//   st[5] alpha   st[6] beta    st[7] dot scratch
//   flags: f[0] stop  f[1] restart  f[2] iterations  f[3] breakdown
// ---------------------------------------------------------------------------------------
__global__ void k_cg_z(int64_t nz, const int32_t* __restrict__ prow, const double* __restrict__ dinv,
                       const double* __restrict__ R, double* __restrict__ Z, const int32_t* __restrict__ f) {
    if (f[0]) return;
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < nz) Z[p] = dinv[prow[p]] * R[p];
}

__global__ void k_cg_ctl_newsum(double* __restrict__ st, int32_t* __restrict__ f) {
    if (f[0]) return;
    const double newsum = st[7];
    st[0] = newsum;
    if (st[2] < 0.0) st[2] = newsum;
    if (!(newsum > 1e-28 * sd::dmax(st[2], 1.0))) {
        f[0] = 1;
        f[4] = 1;
        return;
    }
    if (!f[1]) st[6] = newsum / st[1];
}

__global__ void k_cg_dir(int64_t nz, const double* __restrict__ Z, double* __restrict__ D,
                         const double* __restrict__ st, const int32_t* __restrict__ f) {
    if (f[0]) return;
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= nz) return;
    if (f[1]) D[p] = Z[p];
    else D[p] = Z[p] + st[6] * D[p];
}

__global__ void k_cg_ctl_denom(double* __restrict__ st, int32_t* __restrict__ f,
                               unsigned long long* __restrict__ alpha_bits) {
    if (f[0]) return;
    const double denom = st[7];
    st[3] = denom;
    if (!(denom > 0.0)) {
        f[0] = 1;
        f[4] = 2;
        return;
    }
    st[4] = st[0] / denom;
    *alpha_bits = static_cast<unsigned long long>(__double_as_longlong(st[4]));
}

// per column j, entries in increasing row order (CSC positions): e, g, h and the
// safe step (column_safe_step, interpolation.hpp:247-260), min-reduced into alpha_bits
// kCgLpc lanes per column; a block walks the column blocks grid-stride, so the columns in
// flight at any time are one contiguous window (grid * 128 / kCgLpc columns): their entries
// lie in a band of rows whose slots stay in L2 while the neighbouring columns -- which
// share the 32-byte sectors -- read them.  With every column in flight at once the four
// arrays streamed through L2 in sector-sized gathers (C5 level 0: 4.1 GB of DRAM traffic
// for 0.54 GB of data).  The window is a trade between traffic and threads in flight
// (DESIGN.md §3); four lanes per column put four times the loads in flight for the same
// window: lane t loads the entries q = t (mod 4) and forms their products, and the three
// sums take the products in row order from the lanes by shuffles (every lane of a column
// carries the same sums).
constexpr int kCgLpc = 4;
__global__ void __launch_bounds__(128)
    k_cg_columns(int32_t nc, const int32_t* __restrict__ colptr, const int32_t* __restrict__ pos,
                 const double* __restrict__ P, const double* __restrict__ APm, const double* __restrict__ D,
                 const double* __restrict__ ADm, unsigned long long* __restrict__ alpha_bits,
                 const int32_t* __restrict__ f) {
    if (f[0]) return;
    const int sub = threadIdx.x % kCgLpc;
    const int lane = threadIdx.x & 31;
    const int lead = lane - sub;  // first lane of this column's group
    const int32_t per_block = blockDim.x / kCgLpc;
    // every lane of a warp runs the same number of rounds (the shuffles are warp-wide)
    const int32_t j0 = blockIdx.x * per_block + static_cast<int32_t>(threadIdx.x) / kCgLpc;
    const int32_t stride = static_cast<int32_t>(gridDim.x) * per_block;
    const int32_t jw = blockIdx.x * per_block + (static_cast<int32_t>(threadIdx.x) & ~31) / kCgLpc;  // the warp's first column
    for (int32_t jb = jw, j = j0; jb < nc; jb += stride, j += stride) {
        const bool on = j < nc;
        const int32_t qb = on ? colptr[j] : 0, qe = on ? colptr[j + 1] : 0;
        // rounds of kCgLpc entries; the warp runs as many as its longest column needs
        int32_t rounds = (qe - qb + kCgLpc - 1) / kCgLpc;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, off));
        double e = 0.0, g = 0.0, h = 0.0;
        for (int32_t r = 0; r < rounds; r += 2) {
            // two rounds' loads in flight before their sums
            double pe[2], pg[2], ph[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int32_t q = qb + (r + u) * kCgLpc + sub;
                pe[u] = pg[u] = ph[u] = 0.0;
                if (q < qe) {
                    const int32_t p = __ldg(&pos[q]);
                    const double vp = __ldg(&P[p]), va = __ldg(&APm[p]), vd = __ldg(&D[p]), vm = __ldg(&ADm[p]);
                    pe[u] = vp * va;
                    pg[u] = vd * va;
                    ph[u] = vd * vm;
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
#pragma unroll
                for (int t = 0; t < kCgLpc; ++t) {
                    const double xe = __shfl_sync(0xffffffffu, pe[u], lead + t);
                    const double xg = __shfl_sync(0xffffffffu, pg[u], lead + t);
                    const double xh = __shfl_sync(0xffffffffu, ph[u], lead + t);
                    if (qb + (r + u) * kCgLpc + t < qe) {  // entries past the column's end add nothing
                        e += xe;
                        g += xg;
                        h += xh;
                    }
                }
            }
        }
        if (!on || sub != 0 || h <= 0.0) continue;
        const double norm_j = sqrt(sd::dmax(e, 0.0));
        const double tol = 2.5e-13 * sd::dmax(norm_j, 1.0e-30);
        const double budget = tol * (2.0 * norm_j + tol);
        const double disc = g * g + h * budget;
        const double beta = (-g + sqrt(sd::dmax(disc, 0.0))) / h;
        if (beta >= 0.0)  // all finite steps are >= 0; NaN never wins (std::min semantics)
            atomicMin(alpha_bits, static_cast<unsigned long long>(__double_as_longlong(beta)));
    }
}

__global__ void k_cg_ctl_alpha(double* __restrict__ st, int32_t* __restrict__ f,
                               const unsigned long long* __restrict__ alpha_bits, int s) {
    if (f[0]) return;
    const double alpha = __longlong_as_double(static_cast<long long>(*alpha_bits));
    const double alpha_cg = st[4];
    st[5] = alpha;
    if (!(alpha > 1e-14 * alpha_cg)) {
        f[3] = 1;
        f[0] = 1;
        f[4] = 3;
        return;
    }
    f[1] = alpha < alpha_cg * (1.0 - 1e-12) ? 1 : 0;
    st[1] = st[0];
    f[2] = s + 1;
}

__global__ void k_cg_update(int64_t nz, double* __restrict__ P, double* __restrict__ APm, double* __restrict__ R,
                            const double* __restrict__ D, const double* __restrict__ ADm,
                            const double* __restrict__ ADp, const double* __restrict__ st,
                            const int32_t* __restrict__ f, int s) {
    if (f[3] || f[2] != s + 1) return;  // only when iteration s completed its step
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= nz) return;
    const double alpha = st[5];
    P[p] += alpha * D[p];
    APm[p] += alpha * ADm[p];
    R[p] -= alpha * ADp[p];
}

// ---------------------------------------------------------------------------------------
// GMRES clipping sums (interpolation.hpp:417-435): per column j over AT / AU entries
// in increasing row order
// ---------------------------------------------------------------------------------------
__global__ void k_gm_columns(int32_t nc, const int32_t* __restrict__ tcp, const int32_t* __restrict__ tpos,
                             const double* __restrict__ atv, const int32_t* __restrict__ ucp,
                             const int32_t* __restrict__ upos, const int32_t* __restrict__ urow,
                             const double* __restrict__ auv, const int32_t* __restrict__ atrp,
                             const int32_t* __restrict__ atci, double* __restrict__ e, double* __restrict__ g,
                             double* __restrict__ h) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nc) return;
    double ej = 0.0, gj = 0.0, hj = 0.0;
    for (int32_t q = tcp[j]; q < tcp[j + 1]; ++q) {
        const double v = atv[tpos[q]];
        ej += v * v;
    }
    for (int32_t q = ucp[j]; q < ucp[j + 1]; ++q) {
        const int32_t p = upos[q];
        const double v = auv[p];
        hj += v * v;
        const int32_t i = urow[p];
        const int32_t at = lower_bound_i32(atci, atrp[i], atrp[i + 1], j);
        if (at < atrp[i + 1] && atci[at] == j) gj += v * atv[at];
    }
    e[j] = ej;
    g[j] = gj;
    h[j] = hj;
}

__global__ void k_axpy_host(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < n) y[p] += a * x[p];
}

// ensure_min_support (interpolation.hpp:607-643), thread per row with the row in
// local arrays: the filtered row, then the full row's other non-zero entries sorted
// by magnitude with libstdc++'s std::sort (stl_sort.cuh: the reference's tie order),
// appended until the row holds min(min_cols, |full row|) entries and -- with Bc --
// until the coarse-candidate rows it spans reach rank min_cols (span_rank: QR with
// column pivoting, threshold 1e-3, small_dense.h qr_rank).  Output in column order.
constexpr int kEmsMax = 64;  // entries per row handled (longer rows: error flag)

struct EmsCand {
    double mag;
    int32_t col;
    double val;
};

__global__ void k_min_support_rows(int32_t n, const int32_t* __restrict__ frp, const int32_t* __restrict__ fci,
                                   const double* __restrict__ fva, const int32_t* __restrict__ grp,
                                   const int32_t* __restrict__ gci, const double* __restrict__ gva, int32_t min_cols,
                                   const double* __restrict__ Bc, int32_t k, int32_t nc, int32_t* __restrict__ err,
                                   const int32_t* __restrict__ orp, int32_t* __restrict__ cnt, int32_t* __restrict__ oci,
                                   double* __restrict__ ova) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t flo = frp[i], fhi = frp[i + 1], glo = grp[i], ghi = grp[i + 1];
    if (fhi - flo > kEmsMax || ghi - glo > kEmsMax) {
        atomicExch(err, 1);
        if (!orp) cnt[i] = 0;
        return;
    }
    int32_t oc[kEmsMax];
    double ov[kEmsMax];
    int no = 0;
    for (int32_t p = flo; p < fhi; ++p, ++no) {
        oc[no] = fci[p];
        ov[no] = fva[p];
    }
    auto span_rank = [&]() {
        double M[kEmsMax * kKMax];
        for (int r = 0; r < no; ++r)
            for (int a = 0; a < k; ++a) M[r * k + a] = Bc[static_cast<size_t>(a) * nc + oc[r]];
        return sd::qr_rank<kKMax>(no, k, M, 1e-3);
    };
    const int32_t have = no, full_len = ghi - glo;
    const int32_t target = min(min_cols, full_len);
    const bool short_rank = Bc && have >= target && full_len > have && span_rank() < min_cols;
    if (!(have >= target && !short_rank)) {
        EmsCand cand[kEmsMax];
        int ncand = 0;
        for (int32_t p = glo; p < ghi; ++p) {
            const int32_t j = gci[p];
            bool present = false;
            for (int e = 0; e < have; ++e) present = present || oc[e] == j;
            if (!present && gva[p] != 0.0) cand[ncand++] = {fabs(gva[p]), j, gva[p]};
        }
        stlsort::sort(cand, cand + ncand, [](const EmsCand& a, const EmsCand& b) { return a.mag > b.mag; });
        int t = 0;
        for (; t < ncand && no < target; ++t, ++no) {
            oc[no] = cand[t].col;
            ov[no] = cand[t].val;
        }
        if (Bc)
            for (; t < ncand && span_rank() < min_cols; ++t, ++no) {
                oc[no] = cand[t].col;
                ov[no] = cand[t].val;
            }
    }
    if (!orp) {
        cnt[i] = no;
        return;
    }
    // from_rows: ascending column (the columns are distinct; values pass through 0.0 + v)
    int32_t o = orp[i];
    int32_t last = -1;
    for (int w = 0; w < no; ++w) {
        int best = -1;
        for (int e = 0; e < no; ++e)
            if (oc[e] > last && (best < 0 || oc[e] < oc[best])) best = e;
        oci[o] = oc[best];
        ova[o] = 0.0 + ov[best];
        ++o;
        last = oc[best];
    }
}

// rows below min(min_cols, |full row|) entries (the count floor; no rank floor)
__global__ void k_support_short(int32_t n, const int32_t* __restrict__ frp, const int32_t* __restrict__ grp,
                                int32_t min_cols, int32_t* __restrict__ flag) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && frp[i + 1] - frp[i] < min(min_cols, grp[i + 1] - grp[i])) atomicExch(flag, 1);
}

// two-pass helper for row kernels with (..., orp, cnt, oci, ova) tails
template <typename K, typename... Args>
void build_rows(Ctx& c, int32_t nr, int32_t nc, int32_t bs, DCsr& out, K k, unsigned grid, unsigned block,
                Args... args) {
    DBuf<int32_t> cnt(static_cast<size_t>(nr) + 1, c.s);
    launch(c, k, grid, block, 0, args..., static_cast<const int32_t*>(nullptr), cnt.get(),
           static_cast<int32_t*>(nullptr), static_cast<double*>(nullptr));
    out.nr = nr;
    out.nc = nc;
    out.bs = bs;
    out.rp.alloc(static_cast<size_t>(nr) + 1, c.s);
    out.nnz = exclusive_scan_i32(c, cnt.get(), out.rp.get(), nr);
    out.ci.alloc(static_cast<size_t>(out.nnz), c.s);
    out.va.alloc(static_cast<size_t>(out.nnz), c.s);
    launch(c, k, grid, block, 0, args..., static_cast<const int32_t*>(out.rp.get()), cnt.get(), out.ci.get(),
           out.va.get());
}

}  // namespace

void add_aggregate_entries(Ctx& c, const DCsr& N, const DAgg& agg, DCsr& out) {
    DBuf<int32_t> flag(1, c.s);
    AMG_CK(cudaMemsetAsync(flag.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_any_missing, blocks_for(N.nr, 256), 256, 0, N.nr, N.rp.get(), N.ci.get(), agg.owner.get(), flag.get());
    if (!read_scalar(c, flag.get())) {
        clone_csr(c, N, out);
        return;
    }
    build_rows(c, N.nr, N.nc, 1, out, k_add_agg, blocks_for(N.nr, 128), 128, N.nr, N.rp.get(), N.ci.get(), N.va.get(),
               static_cast<const int32_t*>(agg.owner.get()));
}

void ensure_min_support(Ctx& c, const DCsr& filtered, const DCsr& full, int32_t min_cols, DCsr& out, const double* Bc,
                        int32_t k) {
    if (filtered.nr != full.nr || filtered.nc != full.nc) throw InvalidArgument("ensure_min_support: shape mismatch");
    if (Bc && k > kKMax) throw InvalidArgument("ensure_min_support: at most 8 candidates on the GPU path");
    DBuf<int32_t> err(1, c.s);
    AMG_CK(cudaMemsetAsync(err.get(), 0, sizeof(int32_t), c.s));
    if (!Bc) {
        // count floor only: rows already at the floor keep their entries (interpolation.hpp:623),
        // so when none is below it the result is the filtered matrix itself
        launch(c, k_support_short, blocks_for(filtered.nr, 256), 256, 0, filtered.nr, filtered.rp.get(),
               full.rp.get(), min_cols, err.get());
        if (!read_scalar(c, err.get())) {
            clone_csr(c, filtered, out);
            return;
        }
        AMG_CK(cudaMemsetAsync(err.get(), 0, sizeof(int32_t), c.s));
    }
    build_rows(c, filtered.nr, filtered.nc, filtered.bs, out, k_min_support_rows, blocks_for(filtered.nr, 64), 64,
               filtered.nr, filtered.rp.get(), filtered.ci.get(), filtered.va.get(), full.rp.get(), full.ci.get(),
               full.va.get(), min_cols, Bc, k, filtered.nc, err.get());
    if (read_scalar(c, err.get()))
        throw InvalidArgument("ensure_min_support: rows above 64 entries are not on the GPU path");
}

void widen_deficient_rows(Ctx& c, const DCsr& N, const DCsr& S, const DAgg& agg, int32_t min_aggs, DCsr& out) {
    if (min_aggs <= 1) {
        clone_csr(c, N, out);
        return;
    }
    const int32_t n = N.nr;
    DBuf<int32_t> list(static_cast<size_t>(n), c.s), count(1, c.s);
    AMG_CK(cudaMemsetAsync(count.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_deficient, blocks_for(n, 256), 256, 0, n, N.rp.get(), min_aggs, list.get(), count.get());
    const int32_t nd = read_scalar(c, count.get());
    if (nd == 0) {
        clone_csr(c, N, out);
        return;
    }
    DCsr St;
    transpose(c, S, St);
    const int32_t conc = std::min<int32_t>(nd, 32);
    DBuf<int32_t> seen(static_cast<size_t>(conc) * S.nr, c.s), front(static_cast<size_t>(conc) * 2 * S.nr, c.s);
    DBuf<int32_t> xcols(static_cast<size_t>(nd) * kWidenAggCap, c.s), xcnt(static_cast<size_t>(n), c.s),
        xbase(static_cast<size_t>(n), c.s), err(1, c.s);
    AMG_CK(cudaMemsetAsync(xcnt.get(), 0, sizeof(int32_t) * n, c.s));
    AMG_CK(cudaMemsetAsync(xbase.get(), 0, sizeof(int32_t) * n, c.s));
    AMG_CK(cudaMemsetAsync(err.get(), 0, sizeof(int32_t), c.s));
    for (int32_t b0 = 0; b0 < nd; b0 += conc) {
        const int32_t nb = std::min(conc, nd - b0);
        launch(c, k_widen, static_cast<unsigned>(nb), kWidenThreads, 0, static_cast<const int32_t*>(list.get() + b0),
               S.nr, N.rp.get(), N.ci.get(), S.rp.get(), S.ci.get(), St.rp.get(), St.ci.get(), agg.owner.get(),
               min_aggs, seen.get(), front.get(), xcols.get(), xcnt.get(), xbase.get(), b0, err.get());
    }
    if (read_scalar(c, err.get())) throw RuntimeError("widen_deficient_rows: GPU aggregate-set capacity exceeded");
    build_rows(c, N.nr, N.nc, N.bs, out, k_widen_merge, blocks_for(n, 128), 128, n, N.rp.get(), N.ci.get(),
               N.va.get(), static_cast<const int32_t*>(xcols.get()), static_cast<const int32_t*>(xcnt.get()),
               static_cast<const int32_t*>(xbase.get()));
}

void unamalgamate(Ctx& c, const DCsr& N, const DAgg& agg, int32_t m, DCsr& Nd, DBuf<int32_t>& droots) {
    if (m < 1) throw InvalidArgument("unamalgamate: block size must be >= 1");
    droots.alloc(static_cast<size_t>(agg.n_agg) * m, c.s);
    if (m == 1) {
        clone_csr(c, N, Nd);
        copy_d2d(c, droots.get(), agg.roots.get(), agg.n_agg);
        return;
    }
    const int32_t nd = N.nr * m;
    DBuf<int32_t> cnt(static_cast<size_t>(nd) + 1, c.s);
    launch(c, k_unamalg_rp, blocks_for(nd, 256), 256, 0, N.nr, m, N.rp.get(), cnt.get());
    Nd.nr = nd;
    Nd.nc = N.nc * m;
    Nd.bs = 1;
    Nd.rp.alloc(static_cast<size_t>(nd) + 1, c.s);
    Nd.nnz = exclusive_scan_i32(c, cnt.get(), Nd.rp.get(), nd);
    Nd.ci.alloc(static_cast<size_t>(Nd.nnz), c.s);
    Nd.va.alloc(static_cast<size_t>(Nd.nnz), c.s);
    launch(c, k_unamalg, blocks_for(nd, 256), 256, 0, N.nr, m, N.rp.get(), N.ci.get(), N.va.get(),
           static_cast<const int32_t*>(Nd.rp.get()), Nd.ci.get(), Nd.va.get());
    launch(c, k_droots, blocks_for(agg.n_agg, 256), 256, 0, agg.n_agg, m, agg.roots.get(), droots.get());
}

void root_node_pattern(Ctx& c, const DCsr& N, const int32_t* roots, int32_t n_roots, DCsr& out) {
    if (n_roots != N.nc) throw InvalidArgument("root_node_pattern: need one root per coarse column");
    DBuf<int32_t> owner(static_cast<size_t>(N.nr), c.s), err(1, c.s);
    fill_i32(c, owner.get(), -1, N.nr);
    AMG_CK(cudaMemsetAsync(err.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_owner_of_root, blocks_for(n_roots, 256), 256, 0, n_roots, roots, owner.get(), N.nr, err.get());
    const int32_t e = read_scalar(c, err.get());
    if (e == 1) throw InvalidArgument("root_node_pattern: root out of range");
    if (e == 2) throw InvalidArgument("root_node_pattern: duplicate root row");
    build_rows(c, N.nr, N.nc, N.bs, out, k_rootpat, blocks_for(N.nr, 128), 128, N.nr, N.rp.get(), N.ci.get(),
               N.va.get(), static_cast<const int32_t*>(owner.get()));
}

void enforce_constraints(Ctx& c, const DCsr& P, const double* B, const double* Bc, int32_t k, const DCsr* allowed,
                         DCsr& out) {
    const DCsr& N = allowed ? *allowed : P;
    if (P.nr != N.nr || P.nc != N.nc) throw InvalidArgument("enforce_constraints: dimension mismatch");
    if (k > kKMax) throw InvalidArgument("enforce_constraints: at most 8 candidates on the GPU path");
    if (c.ops) {  // interpolation.hpp:518: 2 len k + k^3 per non-empty row
        const RowCensus rc = row_census(c, N, nullptr);
        const double kk = static_cast<double>(k);
        tally(c, 2.0 * kk * static_cast<double>(N.nnz) + kk * kk * kk * rc.nonempty);
    }
    DBuf<double> vals(static_cast<size_t>(N.nnz), c.s);
    DBuf<int32_t> err(1, c.s);
    AMG_CK(cudaMemsetAsync(err.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_scatter_pattern, blocks_for(N.nr, 256), 256, 0, N.nr, P.rp.get(), P.ci.get(), P.va.get(), N.rp.get(),
           N.ci.get(), vals.get(), err.get());
    if (read_scalar(c, err.get())) throw InvalidArgument("energy_minimize: T has an entry outside the pattern");
    launch(c, k_enforce, blocks_for(N.nr, 64), 64, 0, N.nr, k, N.rp.get(), N.ci.get(), vals.get(), B, Bc, N.nc);
    compact_pattern(c, N, vals.get(), P.bs, out);
}

void inject_tentative(Ctx& c, const DAgg& agg, const DCsr& N, const double* B, int32_t k, int32_t m, DCsr& T,
                      DBuf<double>& Bc) {
    if (m < 1) throw InvalidArgument("inject_tentative: block size must be >= 1");
    if (k < m) throw InvalidArgument("inject_tentative: need at least m candidates");
    if (m > 8) throw InvalidArgument("inject_tentative: block size above 8 on the GPU path");
    const int32_t ndof = agg.n_nodes * m, nc = agg.n_agg * m;
    if (N.nr != ndof || N.nc != nc) throw InvalidArgument("inject_tentative: pattern dimensions mismatch");
    // interpolation.hpp:578: m^3 per aggregate block inverse + m^2 per non-root DOF row
    tally(c, static_cast<double>(agg.n_nodes) * m * m * m);
    Bc.alloc(static_cast<size_t>(nc) * k, c.s);
    DBuf<double> binv(static_cast<size_t>(agg.n_agg) * m * m, c.s);
    DBuf<int32_t> degenerate(1, c.s);
    AMG_CK(cudaMemsetAsync(degenerate.get(), 0, sizeof(int32_t), c.s));
    launch(c, k_root_blocks, blocks_for(agg.n_agg, 128), 128, 0, agg.n_agg, m, k, ndof, agg.roots.get(), B, binv.get(),
           Bc.get(), nc, degenerate.get());
    if (m > 1 && read_scalar(c, degenerate.get()) > 0) {
        // degenerate m x m root blocks: COD pseudo-inverse (threshold 1e-10) on the host,
        // interpolation.hpp:550-553 -- rare, tiny
        std::vector<double> hb(static_cast<size_t>(agg.n_agg) * m * m);
        copy_d2h(c, hb.data(), binv.get(), static_cast<int64_t>(hb.size()));
        std::vector<int32_t> hroots(agg.n_agg);
        copy_d2h(c, hroots.data(), agg.roots.get(), agg.n_agg);
        std::vector<double> hB(static_cast<size_t>(ndof) * k);
        copy_d2h(c, hB.data(), B, static_cast<int64_t>(hB.size()));
        sync(c);
        for (int32_t g = 0; g < agg.n_agg; ++g) {
            double* inv = hb.data() + static_cast<size_t>(g) * m * m;
            if (!std::isnan(inv[0])) continue;
            std::vector<double> blk(static_cast<size_t>(m) * m);
            for (int r = 0; r < m; ++r)
                for (int cc = 0; cc < m; ++cc) blk[r * m + cc] = hB[static_cast<size_t>(cc) * ndof + hroots[g] * m + r];
            sd::COD cod;
            cod.threshold = 1e-10;
            cod.compute(m, m, blk.data());
            cod.pseudo_inverse(inv);
        }
        copy_h2d(c, binv.get(), hb.data(), static_cast<int64_t>(hb.size()));
        sync(c);
    }
    DCsr T0;
    build_rows(c, ndof, nc, m, T0, k_tentative_rows, blocks_for(ndof, 256), 256, agg.n_nodes, m, agg.owner.get(),
               agg.roots.get(), B, ndof, static_cast<const double*>(binv.get()));
    T0.bs = m;
    if (k > m) {
        enforce_constraints(c, T0, B, Bc.get(), k, &N, T);
        T.bs = m;
    } else {
        T = std::move(T0);
    }
}

void energy_minimize(Ctx& c, const DCsr& A, const DCsr& T, const double* B, const double* Bc, int32_t k,
                     const DCsr& N, int iters, int krylov, const int32_t* roots, int32_t n_roots, DCsr& Pout,
                     EnergyMinStats* stats) {
    (void)B;
    BlasFamilyScope scope(c, kProfEminBlas1);
    if (A.nr != A.nc || A.nr != N.nr) throw InvalidArgument("energy_minimize: dimension mismatch");
    if (k > kKMax) throw InvalidArgument("energy_minimize: at most 8 candidates on the GPU path");
    const int32_t n = N.nr, nc = N.nc;
    const int64_t nz = N.nnz;
    EnergyMinStats local;
    EnergyMinStats& st = stats ? *stats : local;
    st = EnergyMinStats{};
    // constraint workspace
    DBuf<unsigned char> is_root(static_cast<size_t>(n), c.s);
    AMG_CK(cudaMemsetAsync(is_root.get(), 0, static_cast<size_t>(n), c.s));
    launch(c, k_root_mask, blocks_for(n_roots, 256), 256, 0, n_roots, roots, is_root.get());
    DBuf<double> gp(static_cast<size_t>(n) * k * k, c.s);
    launch(c, k_gram_pinv, blocks_for(n, 64), 64, 0, n, k, N.rp.get(), N.ci.get(), Bc, nc,
           static_cast<const unsigned char*>(is_root.get()), gp.get());
    // WorkLedger (only with an active sink): Gram build (interpolation.hpp:140) and the
    // per-call project count (180)
    const bool counting = c.ops != nullptr;
    double proj_ops = 0.0;
    if (counting) {
        const RowCensus rc = row_census(c, N, is_root.get());
        const double kk = static_cast<double>(k);
        tally(c, kk * kk * rc.len + kk * kk * kk * rc.rows);
        proj_ops = 2.0 * kk * rc.len + kk * kk * rc.rows;
    }
    // vectors the band kernel stages by 16-byte pieces are padded to an even length
    const size_t nzs = (static_cast<size_t>(nz) + 1) & ~static_cast<size_t>(1);
    DBuf<double> P(nzs, c.s);
    {
        DBuf<int32_t> err(1, c.s);
        AMG_CK(cudaMemsetAsync(err.get(), 0, sizeof(int32_t), c.s));
        launch(c, k_scatter_pattern, blocks_for(n, 256), 256, 0, n, T.rp.get(), T.ci.get(), T.va.get(), N.rp.get(),
               N.ci.get(), P.get(), err.get());
        if (read_scalar(c, err.get())) throw InvalidArgument("energy_minimize: T has an entry outside the pattern");
    }
    const unsigned mp_grid = blocks_for(n, 128);
    auto mp_bytes = [&](const DCsr& M, int outs) {
        return 12.0 * M.nnz + 4.0 * (M.nr + 1) + 4.0 * nz + 4.0 * (n + 1) + 8.0 * nz * (1 + outs) + 8.0 * k * nc +
               8.0 * k * k * n;
    };
    const unsigned mp_block = 128;
    const unsigned ew = blocks_for(nz, 256);
    // Y = (M X)|_N, Yp its projection (either may be null); M's plan when the level takes the band kernel
    auto masked = [&](const DCsr& M, const mband::Plan& pl, int family, double bytes, const double* x, double* y,
                      double* yp, const int32_t* stop) {
        if (pl.ok)
            launch_prof(c, family, bytes, band_kernel(k, pl.mode), static_cast<unsigned>(pl.nctas), mband::kThreads, pl.smem,
                        n, pl.R, pl.cap_a, pl.cap_x, pl.cap_s, M.rp.get(), static_cast<const mband::Rec*>(pl.recs.get()),
                        N.rp.get(), N.ci.get(), x, k, Bc, nc, static_cast<const double*>(gp.get()),
                        static_cast<const unsigned char*>(is_root.get()), y, yp,
                        static_cast<const mband::Run*>(pl.runs.get()), static_cast<const int32_t*>(pl.nruns.get()), stop);
        else
            launch_prof(c, family, bytes, k_masked_rows, mp_grid, mp_block, 0, n, M.rp.get(), M.ci.get(), M.va.get(),
                        N.rp.get(), N.ci.get(), x, k, Bc, nc, static_cast<const double*>(gp.get()),
                        static_cast<const unsigned char*>(is_root.get()), y, yp, stop);
    };

    if (krylov == 0) {
        DBuf<double> dinv(static_cast<size_t>(n), c.s);
        inverse_diagonal(c, A, dinv.get(), "energy_minimize: zero diagonal at row ");
        DBuf<int32_t> prow(static_cast<size_t>(nz), c.s);
        entry_rows(c, N, prow.get());
        DBuf<int32_t> colptr, pos;
        transpose_positions(c, N, colptr, pos, nullptr);
        DBuf<double> APm(static_cast<size_t>(nz), c.s), R(static_cast<size_t>(nz), c.s), Z(static_cast<size_t>(nz), c.s),
            D(nzs, c.s), ADm(static_cast<size_t>(nz), c.s), ADp(static_cast<size_t>(nz), c.s);
        AMG_CK(cudaMemsetAsync(D.get(), 0, sizeof(double) * nz, c.s));
        const mband::Plan plan = masked_band_plan(c, A, N, k);
        masked(A, plan, kProfOther, 0.0, P.get(), APm.get(), nullptr, nullptr);
        launch(c, k_negate, ew, 256, 0, nz, static_cast<const double*>(APm.get()), R.get());
        launch_prof(c, kProfEminCg, 0.0, k_project, blocks_for(n, 128), 128, 0, n, N.rp.get(), N.ci.get(), k, Bc, nc,
               static_cast<const double*>(gp.get()), static_cast<const unsigned char*>(is_root.get()), R.get());
        DBuf<double> scal(8, c.s);
        DBuf<int32_t> flags(8, c.s);
        DBuf<unsigned long long> abits(1, c.s);
        const double init[8] = {0.0, 0.0, -1.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const int32_t finit[8] = {0, 1, 0, 0, 0, 0, 0, 0};
        copy_h2d(c, scal.get(), init, 8);
        copy_h2d(c, flags.get(), finit, 8);
        double* S = scal.get();
        int32_t* F = flags.get();
        for (int s = 0; s < iters; ++s) {
            launch_prof(c, kProfEminCg, 0.0, k_cg_z, ew, 256, 0, nz, static_cast<const int32_t*>(prow.get()),
                   static_cast<const double*>(dinv.get()), static_cast<const double*>(R.get()), Z.get(),
                   static_cast<const int32_t*>(F));
            dot(c, R.get(), Z.get(), nz, S + 7);
            launch_prof(c, kProfEminCg, 0.0, k_cg_ctl_newsum, 1, 1, 0, S, F);
            launch_prof(c, kProfEminCg, 0.0, k_cg_dir, ew, 256, 0, nz, static_cast<const double*>(Z.get()), D.get(),
                   static_cast<const double*>(S), static_cast<const int32_t*>(F));
            masked(A, plan, kProfMaskedProduct, mp_bytes(A, 2), D.get(), ADm.get(), ADp.get(), F);
            dot(c, D.get(), ADm.get(), nz, S + 7);
            launch_prof(c, kProfEminCg, 0.0, k_cg_ctl_denom, 1, 1, 0, S, F, abits.get());
            launch_prof(c, kProfEminCg, 0.0, k_cg_columns, std::min(blocks_for(static_cast<int64_t>(nc) * kCgLpc, 128), cg_column_blocks(c)), 128, 0, nc, static_cast<const int32_t*>(colptr.get()),
                   static_cast<const int32_t*>(pos.get()), static_cast<const double*>(P.get()),
                   static_cast<const double*>(APm.get()), static_cast<const double*>(D.get()),
                   static_cast<const double*>(ADm.get()), abits.get(), static_cast<const int32_t*>(F));
            launch_prof(c, kProfEminCg, 0.0, k_cg_ctl_alpha, 1, 1, 0, S, F, static_cast<const unsigned long long*>(abits.get()), s);
            launch_prof(c, kProfEminCg, 0.0, k_cg_update, ew, 256, 0, nz, P.get(), APm.get(), R.get(), static_cast<const double*>(D.get()),
                   static_cast<const double*>(ADm.get()), static_cast<const double*>(ADp.get()),
                   static_cast<const double*>(S), static_cast<const int32_t*>(F), s);
        }
        int32_t fh[8];
        int32_t band_bad = 0;
        unsigned long long band_matches = 0;
        copy_d2h(c, fh, F, 8);
        if (plan.ok) {
            copy_d2h(c, &band_bad, plan.info.get(), 1);
            copy_d2h(c, &band_matches, plan.matches.get(), 1);
        }
        sync(c);
        if (band_bad) throw std::logic_error("energy_minimize: band plan left an entry without its run");
        st.iterations = fh[2];
        st.breakdown = fh[3] != 0;
        if (counting) {
            // the reference's counts (interpolation.hpp:319,333,355): the initial masked product
            // and projection, every completed iteration, and the part of the stopping one
            const double M = plan.ok ? static_cast<double>(band_matches) : masked_count(c, A, N), z = static_cast<double>(nz);
            const double full = z + (M + proj_ops + 3.0 * z) + 3.0 * z;
            double ops = M + proj_ops + fh[2] * full;
            if (fh[4] == 1) ops += z;
            if (fh[4] == 2 || fh[4] == 3) ops += z + M + proj_ops + 3.0 * z;
            tally(c, ops);
        }
        compact_pattern(c, N, P.get(), T.bs, Pout);
        return;
    }

    // ---- GMRES branch (interpolation.hpp:363-441) ----
    DCsr At, AtA;
    transpose(c, A, At);
    spgemm(c, At, A, AtA);
    DBuf<double> R0(static_cast<size_t>(nz), c.s);
    const mband::Plan plan = masked_band_plan(c, AtA, N, k);
    masked(AtA, plan, kProfOther, 0.0, P.get(), R0.get(), nullptr, nullptr);
    launch(c, k_negate, ew, 256, 0, nz, static_cast<const double*>(R0.get()), R0.get());
    launch_prof(c, kProfEminCg, 0.0, k_project, blocks_for(n, 128), 128, 0, n, N.rp.get(), N.ci.get(), k, Bc, nc,
           static_cast<const double*>(gp.get()), static_cast<const unsigned char*>(is_root.get()), R0.get());
    DBuf<double> scal(2, c.s);
    nrm2(c, R0.get(), nz, scal.get());
    int32_t band_bad = 0;
    unsigned long long band_matches = 0;
    if (plan.ok) {
        copy_d2h(c, &band_bad, plan.info.get(), 1);
        copy_d2h(c, &band_matches, plan.matches.get(), 1);
    }
    const double beta = read_scalar(c, scal.get());
    if (band_bad) throw std::logic_error("energy_minimize: band plan left an entry without its run");
    const double Mg = !counting ? 0.0 : plan.ok ? static_cast<double>(band_matches) : masked_count(c, AtA, N);
    tally(c, Mg + proj_ops + static_cast<double>(nz));  // interpolation.hpp:374
    if (beta < 1e-300) {
        compact_pattern(c, N, P.get(), T.bs, Pout);
        return;
    }
    const int m = iters;
    DBuf<double> V(nzs * (m + 1), c.s);  // Krylov vectors at an even stride
    DBuf<double> Hd(static_cast<size_t>(m + 1) * m, c.s);
    AMG_CK(cudaMemsetAsync(Hd.get(), 0, sizeof(double) * (m + 1) * m, c.s));
    copy_d2d(c, V.get(), R0.get(), nz);
    scale_const(c, 1.0 / beta, V.get(), nz);
    int built = 0;
    for (int s = 0; s < m; ++s) {
        double* W = V.get() + static_cast<size_t>(s + 1) * nzs;
        masked(AtA, plan, kProfMaskedProduct, mp_bytes(AtA, 1), V.get() + static_cast<size_t>(s) * nzs, nullptr, W, nullptr);
        double* hn_d = Hd.get() + (s + 1) * m + s;
        dot(c, W, V.get(), nz, Hd.get() + s);
        for (int t = 0; t <= s; ++t)
            axpy_dot(c, Hd.get() + t * m + s, -1.0, V.get() + static_cast<size_t>(t) * nzs, W,
                     t < s ? V.get() + static_cast<size_t>(t + 1) * nzs : nullptr, nz,
                     t < s ? Hd.get() + (t + 1) * m + s : hn_d, t == s);
        const double hn = read_scalar(c, hn_d);
        built = s + 1;
        st.iterations = s + 1;
        tally(c, Mg + proj_ops + 2.0 * (s + 1) * static_cast<double>(nz));  // interpolation.hpp:392
        if (hn < 1e-14 * beta) break;
        scale_recip_dev(c, hn_d, W, nz);
    }
    std::vector<double> H(static_cast<size_t>(m + 1) * m);
    copy_d2h(c, H.data(), Hd.get(), static_cast<int64_t>(H.size()));
    sync(c);
    if (built > 64) throw RuntimeError("energy_minimize: Krylov dimension above 64");
    std::vector<double> Hs(static_cast<size_t>(built) * built), ev(built), EV(static_cast<size_t>(built) * built);
    for (int i = 0; i < built; ++i)
        for (int j = 0; j < built; ++j) Hs[i * built + j] = 0.5 * (H[i * m + j] + H[j * m + i]);
    sd::sym_eig<64>(built, Hs.data(), ev.data(), EV.data());
    double mx = std::fabs(ev[0]);
    for (double v : ev) mx = std::max(mx, std::fabs(v));
    const double cutoff = 1e-14 * std::max(mx, 1e-300);
    std::vector<double> rhs(built, 0.0), z(built), y(built);
    rhs[0] = beta;
    for (int t = 0; t < built; ++t) {
        double s2 = 0.0;
        for (int i = 0; i < built; ++i) s2 += EV[i * built + t] * rhs[i];
        z[t] = s2;
    }
    for (int t = 0; t < built; ++t) z[t] = ev[t] > cutoff ? z[t] / ev[t] : 0.0;
    for (int i = 0; i < built; ++i) {
        double s2 = 0.0;
        for (int t = 0; t < built; ++t) s2 += EV[i * built + t] * z[t];
        y[i] = s2;
    }
    DBuf<double> U(static_cast<size_t>(nz), c.s);
    AMG_CK(cudaMemsetAsync(U.get(), 0, sizeof(double) * nz, c.s));
    // V holds built+1 vectors only up to the last normalised one (V[s+1] is filled
    // in place while building); the reference combines V[0..built-1]
    for (int t = 0; t < built; ++t)
        launch_prof(c, kProfEminCg, 0.0, k_axpy_host, ew, 256, 0, nz, y[t], static_cast<const double*>(V.get() + static_cast<size_t>(t) * nzs),
               U.get());
    DCsr Tc, Uc, AT, AU;
    compact_pattern(c, N, P.get(), T.bs, Tc);
    compact_pattern(c, N, U.get(), T.bs, Uc);
    spgemm(c, A, Tc, AT);
    spgemm(c, A, Uc, AU);
    DBuf<int32_t> tcp, tpos, ucp, upos, urow;
    transpose_positions(c, AT, tcp, tpos, nullptr);
    transpose_positions(c, AU, ucp, upos, &urow);
    DBuf<double> e(static_cast<size_t>(nc), c.s), g(static_cast<size_t>(nc), c.s), h(static_cast<size_t>(nc), c.s);
    launch_prof(c, kProfEminCg, 0.0, k_gm_columns, blocks_for(nc, 128), 128, 0, nc, static_cast<const int32_t*>(tcp.get()),
           static_cast<const int32_t*>(tpos.get()), AT.va.get(), static_cast<const int32_t*>(ucp.get()),
           static_cast<const int32_t*>(upos.get()), static_cast<const int32_t*>(urow.get()), AU.va.get(), AT.rp.get(),
           AT.ci.get(), e.get(), g.get(), h.get());
    std::vector<double> he(nc), hg(nc), hh(nc);
    copy_d2h(c, he.data(), e.get(), nc);
    copy_d2h(c, hg.data(), g.get(), nc);
    copy_d2h(c, hh.data(), h.get(), nc);
    sync(c);
    double tau = 1.0;  // column_safe_step(e, g, h, 1.0), host: n_c scalars
    for (int32_t j = 0; j < nc; ++j) {
        if (hh[j] <= 0.0) continue;
        const double norm_j = std::sqrt(std::max(he[j], 0.0));
        const double tol = 2.5e-13 * std::max(norm_j, 1.0e-30);
        const double budget = tol * (2.0 * norm_j + tol);
        const double disc = hg[j] * hg[j] + hh[j] * budget;
        const double bj = (-hg[j] + std::sqrt(std::max(disc, 0.0))) / hh[j];
        tau = std::min(tau, bj);
    }
    if (!(tau > 0.0)) {
        st.breakdown = true;
        Pout = std::move(Tc);
        return;
    }
    launch_prof(c, kProfEminCg, 0.0, k_axpy_host, ew, 256, 0, nz, tau, static_cast<const double*>(U.get()), P.get());
    compact_pattern(c, N, P.get(), T.bs, Pout);
}

}  // namespace amgcu
