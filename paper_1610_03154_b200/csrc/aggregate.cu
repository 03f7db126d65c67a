// Greedy root-node aggregation on the GPU (aggregation.hpp:29-98), bit-exact.
//
// Pass 1 of the reference visits nodes in ascending order and makes node i a
// root when neither i nor any strong neighbour has been claimed.  With
// N[x] = row x of the normalised S (which always holds its diagonal), node i is
// a root iff no lower-index root r has N[r] ∩ N[i] ≠ ∅: pass 1 is the
// lexicographically-first maximal independent set of the conflict graph
// pattern(S S^T).  It is computed by a sync-free wavefront: one thread per
// node, blocks draw tickets in launch order, a node waits only on lower-index
// conflict neighbours (so the nodes it waits on belong to blocks that already
// hold a ticket -- no deadlock) and decides OUT as soon as one of them is a
// root.  Claims, pass 2 (strongest edge, ties to the lowest aggregate id,
// aggregation.hpp:55-76) and the singleton ids (78-82) are then parallel maps
// and scans.
#include <cuda/atomic>

#include <climits>
#include <cstdlib>

#include "ops.cuh"

namespace amgcu {

namespace {

constexpr int kUndecided = 0, kRoot = 1, kOut = 2;
constexpr int kMisThreads = 128;

__global__ void k_unit_diag_check(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ va, int32_t* __restrict__ bad) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t lo = rp[i], hi = rp[i + 1];
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (ci[mid] < i) lo = mid + 1;
        else hi = mid;
    }
    const double d = (lo < rp[i + 1] && ci[lo] == i) ? va[lo] : 0.0;
    if (d != 1.0) atomicExch(bad, 1);
}

__global__ void __launch_bounds__(kMisThreads)
    k_lfmis(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, const int32_t* __restrict__ trp,
            const int32_t* __restrict__ tci, int32_t* __restrict__ state, unsigned int* __restrict__ ticket,
            unsigned max_ns) {
    __shared__ unsigned int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const int32_t i = static_cast<int32_t>(blk) * kMisThreads + threadIdx.x;
    if (i >= n) return;
    // Scan the lower conflict neighbours once, in order; on the first one still
    // undecided, wait on that single state with exponential back-off (one
    // address polled per waiting node), then resume the scan where it stopped.
    // The decision is published inside the loop: a lane leaving a spin loop
    // before storing could wait at the warp's reconvergence point while its
    // neighbours spin on the value it has not written yet.
    cuda::atomic_ref<int32_t, cuda::thread_scope_device> me(state[i]);
    int32_t p = rp[i];
    int32_t q = p < rp[i + 1] ? trp[ci[p]] : 0;
    unsigned ns = 16;
    while (true) {
        bool hit_root = false, pending = false;
        for (; p < rp[i + 1]; ++p) {
            const int32_t x = ci[p];
            if (q < trp[x]) q = trp[x];
            for (; q < trp[x + 1]; ++q) {
                const int32_t r = tci[q];
                if (r >= i) {  // rows of S^T are ascending: nothing lower remains in this column
                    q = trp[x + 1];
                    break;
                }
                cuda::atomic_ref<int32_t, cuda::thread_scope_device> st(state[r]);
                const int32_t v = st.load(cuda::memory_order_relaxed);
                if (v == kRoot) {
                    hit_root = true;
                    break;
                }
                if (v == kUndecided) {
                    pending = true;
                    break;
                }
            }
            if (hit_root || pending) break;
            if (p + 1 < rp[i + 1]) q = trp[ci[p + 1]];
        }
        if (hit_root || !pending) {
            me.store(hit_root ? kOut : kRoot, cuda::memory_order_relaxed);
            break;
        }
        __nanosleep(ns);
        ns = ns < max_ns ? 2 * ns : max_ns;
    }
}

// Lower conflict lists: for node i, every r < i with N[r] ∩ N[i] ≠ ∅, i.e.
// r in S^T row x for x in S row i (duplicates kept; the decision is a set test:
// OUT iff some listed node is a root, ROOT iff all are OUT).
__global__ void k_conf_count(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const int32_t* __restrict__ trp, const int32_t* __restrict__ tci, int32_t* __restrict__ cnt) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t c = 0;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t x = ci[p];
        int32_t lo = trp[x], hi = trp[x + 1];
        const int32_t b = lo;
        while (lo < hi) {  // rows of S^T ascend: count entries < i
            const int32_t mid = (lo + hi) >> 1;
            if (tci[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        c += lo - b;
    }
    cnt[i] = c;
}

__global__ void k_conf_fill(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ trp, const int32_t* __restrict__ tci,
                            const int32_t* __restrict__ off, int32_t* __restrict__ list) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t at = off[i];
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t x = ci[p];
        for (int32_t q = trp[x]; q < trp[x + 1]; ++q) {
            const int32_t r = tci[q];
            if (r >= i) break;
            list[at++] = r;
        }
    }
}

// Sync-free wavefront over the lists: a node loads all listed states at once
// (kMisBatch loads in flight), decides OUT on a root, ROOT when all are OUT,
// otherwise waits on one undecided state and re-checks only the undecided ones.
constexpr int kMisBatch = 8;

__global__ void __launch_bounds__(kMisThreads)
    k_lfmis_lists(int32_t n, const int32_t* __restrict__ off, const int32_t* __restrict__ list,
                  int32_t* __restrict__ state, unsigned int* __restrict__ ticket, unsigned max_ns) {
    __shared__ unsigned int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const int32_t i = static_cast<int32_t>(blk) * kMisThreads + threadIdx.x;
    if (i >= n) return;
    cuda::atomic_ref<int32_t, cuda::thread_scope_device> me(state[i]);
    const int32_t lo = off[i], hi = off[i + 1];
    int32_t first = lo;  // entries before `first` are known OUT
    unsigned ns = 16;
    while (true) {
        bool root_seen = false;
        int32_t undecided_at = -1;
        for (int32_t e0 = first; e0 < hi && !root_seen; e0 += kMisBatch) {
            int32_t r[kMisBatch];
#pragma unroll
            for (int u = 0; u < kMisBatch; ++u) r[u] = e0 + u < hi ? __ldg(&list[e0 + u]) : -1;
            int32_t v[kMisBatch];
#pragma unroll
            for (int u = 0; u < kMisBatch; ++u) {
                v[u] = kOut;
                if (r[u] >= 0) {
                    cuda::atomic_ref<int32_t, cuda::thread_scope_device> st(state[r[u]]);
                    v[u] = st.load(cuda::memory_order_relaxed);
                }
            }
#pragma unroll
            for (int u = 0; u < kMisBatch; ++u) {
                if (v[u] == kRoot) root_seen = true;
                if (v[u] == kUndecided && undecided_at < 0) undecided_at = e0 + u;
            }
        }
        if (root_seen || undecided_at < 0) {
            me.store(root_seen ? kOut : kRoot, cuda::memory_order_relaxed);
            break;
        }
        // everything before the first undecided entry is OUT; wait on it, then re-check from there
        first = undecided_at;
        cuda::atomic_ref<int32_t, cuda::thread_scope_device> w(state[list[undecided_at]]);
        int32_t v = w.load(cuda::memory_order_relaxed);
        while (v == kUndecided) {
            __nanosleep(ns);
            ns = ns < max_ns ? 2 * ns : max_ns;
            v = w.load(cuda::memory_order_relaxed);
        }
        if (v == kRoot) {
            me.store(kOut, cuda::memory_order_relaxed);
            break;
        }
        first = undecided_at + 1;
        ns = 16;
    }
}

__global__ void k_root_flags(int32_t n, const int32_t* __restrict__ state, int32_t* __restrict__ flag) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = state[i] == kRoot ? 1 : 0;
}

// claim N[r] for every root r with id = #roots below r
__global__ void k_claim(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                        const int32_t* __restrict__ state, const int32_t* __restrict__ root_id, int32_t* __restrict__ own,
                        int32_t* __restrict__ roots) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n || state[r] != kRoot) return;
    const int32_t id = root_id[r];
    roots[id] = r;
    own[r] = id;
    for (int32_t p = rp[r]; p < rp[r + 1]; ++p) own[ci[p]] = id;
}

__global__ void k_pass2(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                        const double* __restrict__ va, const int32_t* __restrict__ own, int32_t n_pass1,
                        int32_t* __restrict__ joined) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (own[i] >= 0) {
        joined[i] = own[i];
        return;
    }
    double best = 0.0;
    int32_t best_agg = -1;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = ci[p];
        if (j == i) continue;
        const int32_t a = own[j];
        if (a < 0 || a >= n_pass1) continue;
        const double v = va[p];
        if (v > best || (v == best && best_agg >= 0 && a < best_agg)) {
            best = v;
            best_agg = a;
        }
    }
    joined[i] = best_agg;
}

__global__ void k_leftover_flags(int32_t n, const int32_t* __restrict__ joined, int32_t* __restrict__ flag) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = joined[i] < 0 ? 1 : 0;
}

__global__ void k_singletons(int32_t n, int32_t n_pass1, const int32_t* __restrict__ rank, int32_t* __restrict__ joined,
                             int32_t* __restrict__ roots) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || joined[i] >= 0) return;
    const int32_t id = n_pass1 + rank[i];
    joined[i] = id;
    roots[id] = i;
}

__global__ void k_indicator(int32_t n, const int32_t* __restrict__ own, int32_t* __restrict__ rp,
                            int32_t* __restrict__ ci, double* __restrict__ va) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    rp[i] = i;
    if (i < n) {
        ci[i] = own[i];
        va[i] = 1.0;
    }
}

// poll back-off cap in ns (AMGCU_MIS_NS overrides)
unsigned lfmis_max_ns() {
    static const unsigned v = [] {
        const char* e = std::getenv("AMGCU_MIS_NS");
        return e ? static_cast<unsigned>(std::atoi(e)) : 1024u;
    }();
    return v;
}

}  // namespace

void greedy_aggregate(Ctx& c, const DCsr& S, DAgg& agg) {
    if (S.nr != S.nc) throw InvalidArgument("greedy_aggregate: square matrix required");
    const int32_t n = S.nr;
    {
        DBuf<int32_t> bad(1, c.s);
        AMG_CK(cudaMemsetAsync(bad.get(), 0, sizeof(int32_t), c.s));
        launch(c, k_unit_diag_check, blocks_for(n, 256), 256, 0, n, S.rp.get(), S.ci.get(), S.va.get(), bad.get());
        if (read_scalar(c, bad.get()))
            throw InvalidArgument("greedy_aggregate: strength matrix must be normalized (unit diagonal)");
    }
    DCsr St;  // pattern of S^T (rows ascending) for the conflict sets
    transpose(c, S, St);
    DBuf<int32_t> state(static_cast<size_t>(n), c.s);
    AMG_CK(cudaMemsetAsync(state.get(), 0, sizeof(int32_t) * n, c.s));
    DBuf<unsigned int> ticket(1, c.s);
    AMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned int), c.s));
    {
        DBuf<int32_t> cnt(static_cast<size_t>(n) + 1, c.s), off(static_cast<size_t>(n) + 1, c.s);
        launch(c, k_conf_count, blocks_for(n, 256), 256, 0, n, S.rp.get(), S.ci.get(), St.rp.get(), St.ci.get(),
               cnt.get());
        const int64_t total = exclusive_scan_i32(c, cnt.get(), off.get(), n);
        if (total > INT32_MAX - 1) {
            // lists would overflow 32-bit offsets: scan S and S^T on the fly
            launch_prof(c, kProfAggregate, 8.0 * S.nnz + 8.0 * (n + 1) + 4.0 * n, k_lfmis, blocks_for(n, kMisThreads),
                        kMisThreads, 0, n, S.rp.get(), S.ci.get(), St.rp.get(), St.ci.get(), state.get(),
                        ticket.get(), lfmis_max_ns());
        } else {
            DBuf<int32_t> list(static_cast<size_t>(std::max<int64_t>(total, 1)), c.s);
            launch(c, k_conf_fill, blocks_for(n, 256), 256, 0, n, S.rp.get(), S.ci.get(), St.rp.get(), St.ci.get(),
                   static_cast<const int32_t*>(off.get()), list.get());
            launch_prof(c, kProfAggregate, 8.0 * static_cast<double>(total) + 4.0 * (n + 1) + 4.0 * n,
                        k_lfmis_lists, blocks_for(n, kMisThreads), kMisThreads, 0, n,
                        static_cast<const int32_t*>(off.get()), static_cast<const int32_t*>(list.get()), state.get(),
                        ticket.get(), lfmis_max_ns());
        }
    }
    DBuf<int32_t> flag(static_cast<size_t>(n) + 1, c.s), rid(static_cast<size_t>(n) + 1, c.s);
    launch(c, k_root_flags, blocks_for(n, 256), 256, 0, n, static_cast<const int32_t*>(state.get()), flag.get());
    const int32_t n_pass1 = static_cast<int32_t>(exclusive_scan_i32(c, flag.get(), rid.get(), n));
    DBuf<int32_t> own(static_cast<size_t>(n), c.s), roots(static_cast<size_t>(n), c.s);
    fill_i32(c, own.get(), -1, n);
    launch(c, k_claim, blocks_for(n, 256), 256, 0, n, S.rp.get(), S.ci.get(), static_cast<const int32_t*>(state.get()),
           static_cast<const int32_t*>(rid.get()), own.get(), roots.get());
    DBuf<int32_t> joined(static_cast<size_t>(n), c.s);
    launch(c, k_pass2, blocks_for(n, 256), 256, 0, n, S.rp.get(), S.ci.get(), S.va.get(),
           static_cast<const int32_t*>(own.get()), n_pass1, joined.get());
    launch(c, k_leftover_flags, blocks_for(n, 256), 256, 0, n, static_cast<const int32_t*>(joined.get()), flag.get());
    const int32_t n_left = static_cast<int32_t>(exclusive_scan_i32(c, flag.get(), rid.get(), n));
    launch(c, k_singletons, blocks_for(n, 256), 256, 0, n, n_pass1, static_cast<const int32_t*>(rid.get()),
           joined.get(), roots.get());
    agg.n_nodes = n;
    agg.n_agg = n_pass1 + n_left;
    agg.owner = std::move(joined);
    agg.roots = std::move(roots);
}

void aggregate_indicator(Ctx& c, const DAgg& agg, DCsr& Cm) {
    Cm.alloc(c, agg.n_nodes, agg.n_agg, agg.n_nodes);
    Cm.bs = 1;
    launch(c, k_indicator, blocks_for(agg.n_nodes + 1, 256), 256, 0, agg.n_nodes, agg.owner.get(), Cm.rp.get(),
           Cm.ci.get(), Cm.va.get());
}

}  // namespace amgcu
