// Device plumbing for libamgcu: stream-ordered buffers, the context, device
// CSR, launch accounting and the few generic primitives (scan, fill, copy).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "host_common.h"

namespace amgcu {

#define AMG_CK(call)                                                                              \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            throw ::amgcu::CudaFailure(std::string(#call) + " failed: " + cudaGetErrorString(e_)); \
    } while (0)

// Stream-ordered device buffer (cudaMallocAsync on the context stream; the
// pool keeps freed blocks for reuse, so per-level temporaries are cheap).
template <typename T>
class DBuf {
public:
    DBuf() = default;
    DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }

    void alloc(size_t n, cudaStream_t s) {
        release();
        s_ = s;
        n_ = n;
        if (n) AMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
    }
    void release() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    bool empty() const { return n_ == 0; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

// Per-kernel-family timing with CUDA events on the context stream (bench.py's
// live roofline).  Off by default; when on, every tagged launch is bracketed by
// two events and its algorithmic bytes (the kernel's compulsory I/O) recorded.
enum ProfFamily : int {
    kProfVcycleRelax0Residual = 0,
    kProfVcycleRestrict,
    kProfVcycleProlong,
    kProfVcyclePostRelax,
    kProfKrylovSpmv,
    kProfMaskedProduct,
    kProfSpgemm,
    kProfEvolution,
    kProfGaussSeidel,
    kProfAggregate,
    kProfCoarseSolve,
    kProfBlas1,         // dots, axpys, fused axpy+dot (Krylov, Arnoldi, energy-min CG)
    kProfSpectralSpmv,  // Arnoldi D^-1 A v
    kProfEminCg,        // energy-min CG / GMRES control and column kernels
    kProfOther,         // every launch not tagged with a family
    kProfArnoldiBlas1,  // BLAS-1 inside the spectral-radius Arnoldi
    kProfEminBlas1,     // BLAS-1 inside the energy-minimisation solve
    kProfVcycleCoarseFused,  // levels 1.. of the V-cycle in one cooperative launch
    kProfFamilies
};

struct ProfRecord {
    int64_t launches = 0;
    int64_t syncs = 0;  // host synchronisations of the stream
    double bytes = 0.0;
    double ms = 0.0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    std::vector<const void*> kernels;  // kProfOther with AMGCU_PROF_OTHER: symbol per pending pair
};

// AMGCU_PROF_OTHER=1: untagged launches are also timed per kernel symbol and the
// breakdown is printed to stderr when the profile is read (tools/family_times.py)
// AMGCU_SYNC_TRACE=1 also measures the GPU idle time each synchronisation causes: an
// event before the wait and one right before the next launch on the stream
void gap_before_sync(cudaStream_t s, const char* file, int line);
void gap_before_launch(cudaStream_t s);
void gap_after_sync();
bool sync_trace_on();

bool prof_other_enabled();
void prof_other_add(const void* kernel, double ms);

// workspace of the exact-order reductions (seqsum.cu): tickets, tile look-back status,
// tile and group lists
struct SeqSumWs {
    DBuf<unsigned int> counters;
    DBuf<unsigned char> status;
    DBuf<unsigned char> lists;
    DBuf<int32_t> lens;
    int64_t tiles = 0;
};

// AMGCU_PHASE_TRACE=1: events on the main stream at the setup's phase boundaries
// (per level), printed with their durations when the setup returns (setup.cu)
struct PhaseTrace {
    bool on = false;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
};

struct Ctx {
    bool profile = false;
    uint32_t prof_mask = 0xffffffffu;  // families timed while profile is on
    ProfRecord prof[kProfFamilies];
    std::vector<cudaEvent_t> event_pool;
    int device = 0;
    cudaStream_t s = nullptr;
    cudaStream_t side = nullptr;  // independent side work (the evolution-SOC ledger count)
    cudaStream_t side2 = nullptr;  // candidate Gauss-Seidel, overlapping the aggregation
    int sms = 148;
    cudaStream_t main_s = nullptr;  // the context's own stream (c.s outside StreamScopes)
    bool seq = true;  // global reductions in the reference's order (seqsum.cu); false: trees
    bool cand_overlap = true;  // candidate Gauss-Seidel on side2, beside the aggregation (setup.cu)
    // energy-min masked product: band-staged kernel (masked_band.cuh) on levels of at least
    // this many rows; -1: never
    int32_t band_min_rows = 0;
    int64_t band_accepted = 0, band_refused = 0;  // plans built / refused (failure bits or shared-memory budget)
    int32_t band_last_fail = 0;                   // failure bits of the last refused plan (64: budget)
    int64_t launches = 0;
    int64_t syncs = 0;  // host synchronisations of the stream
    int blas_family = kProfBlas1;  // family the BLAS-1 launchers record under
    double* ops = nullptr;         // WorkLedger sink of the current setup stage (OpCounter, work.hpp:13-22)
    std::string err;
    DBuf<double> scal;         // device scalars for reductions/control
    DBuf<double> partials;     // per-block partial sums
    DBuf<unsigned int> tickets;  // sync-free wavefront tickets
    DBuf<unsigned char> scan_tmp;  // cub::DeviceScan temporary storage
    // pinned host staging: several device scalars are read back with one synchronisation
    int64_t* pin = nullptr;
    static constexpr int kPinSlots = 512;
    // cached Arnoldi start vector 1 + U(-0.5, 0.5) from mt19937(20240911)
    // (spectral.hpp:32-36); prefixes serve every smaller level.
    DBuf<double> arnoldi_v0;
    size_t arnoldi_v0_n = 0;
    // cuSOLVER handle of the dense LU above the Gauss-Jordan kernel's range (setup.cu), created
    // on first use and kept: creating one costs tens of milliseconds
    std::shared_ptr<void> cusolver;
    SeqSumWs ssws[2];  // [0] main stream, [1] any other stream
    PhaseTrace phases;
};

// block-partial scratch and wavefront tickets of the tree reductions (>= count partials)
inline void ensure_reduction_scratch(Ctx& c, size_t count) {
    if (c.partials.size() < count) c.partials.alloc(std::max<size_t>(4096, count), c.s);
    if (c.tickets.size() < 64) {
        c.tickets.alloc(64, c.s);
        AMG_CK(cudaMemsetAsync(c.tickets.get(), 0, sizeof(unsigned int) * 64, c.s));
    }
}

// WorkLedger: add `v` to the current stage's op count (the reference's count(c, v))
inline void tally(Ctx& c, double v) {
    if (c.ops) *c.ops += v;
}

// routes the op counts of a scope to `sink` (nullptr: not counted)
struct OpsScope {
    Ctx& c;
    double* prev;
    OpsScope(Ctx& ctx, double* sink) : c(ctx), prev(ctx.ops) { c.ops = sink; }
    ~OpsScope() { c.ops = prev; }
};

// launches of a scope go to another stream (the context's stream member is swapped)
struct StreamScope {
    Ctx& c;
    cudaStream_t prev;
    StreamScope(Ctx& ctx, cudaStream_t s) : c(ctx), prev(ctx.s) { c.s = s; }
    ~StreamScope() { c.s = prev; }
};

// routes the BLAS-1 launchers' profile records to `family` for a scope
struct BlasFamilyScope {
    Ctx& c;
    int prev;
    BlasFamilyScope(Ctx& ctx, int family) : c(ctx), prev(ctx.blas_family) { c.blas_family = family; }
    ~BlasFamilyScope() { c.blas_family = prev; }
};

struct DCsr {
    int32_t nr = 0, nc = 0, bs = 1;
    int64_t nnz = 0;
    DBuf<int32_t> rp, ci;
    DBuf<double> va;
    void alloc(Ctx& c, int32_t r, int32_t cols, int64_t nz) {
        nr = r;
        nc = cols;
        nnz = nz;
        rp.alloc(static_cast<size_t>(r) + 1, c.s);
        ci.alloc(static_cast<size_t>(nz), c.s);
        va.alloc(static_cast<size_t>(nz), c.s);
    }
};

// Sliced-ELL (slice height 32, no row reordering) mirror of a CSR matrix for
// the solve phase: column-major within each 32-row slice so the per-thread
// row sums (CSR order, reference-exact) load coalesced.
struct DSell {
    int32_t nr = 0, nc = 0;
    int32_t nslices = 0;
    DBuf<int64_t> slice_ptr;   // nslices + 1, element offsets
    DBuf<int32_t> slice_len;   // max row length per slice
    DBuf<int32_t> ci;          // -1 marks padding
    DBuf<double> va;
    int64_t stored = 0;
    // long rows (coarse levels, restriction): the operator's CSR is used by warp-per-row kernels
    bool warp_rows = false;
    const int32_t* crp = nullptr;
    const int32_t* cci = nullptr;
    const double* cva = nullptr;
};

// AMGCU_LAUNCH_CHECK=1 (debugging): synchronise after every launch and name the kernel
// that faulted
bool launch_check_enabled();
void launch_check(Ctx& c, const void* kernel);

template <typename Kern, typename... Args>
inline void launch_raw(Ctx& c, Kern k, unsigned grid, unsigned block, size_t smem, Args... args) {
    if (grid == 0) return;
    if (sync_trace_on()) gap_before_launch(c.s);
    k<<<grid, block, smem, c.s>>>(args...);
    ++c.launches;
    AMG_CK(cudaGetLastError());
    if (launch_check_enabled()) launch_check(c, reinterpret_cast<const void*>(k));
}

template <typename Kern, typename... Args>
inline void launch_prof(Ctx& c, int family, double bytes, Kern k, unsigned grid, unsigned block, size_t smem,
                        Args... args);

// untagged launch: timed under kProfOther when profiling is on
template <typename Kern, typename... Args>
inline void launch(Ctx& c, Kern k, unsigned grid, unsigned block, size_t smem, Args... args) {
    launch_prof(c, kProfOther, 0.0, k, grid, block, smem, args...);
}

inline cudaEvent_t prof_event(Ctx& c) {
    if (!c.event_pool.empty()) {
        cudaEvent_t e = c.event_pool.back();
        c.event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    AMG_CK(cudaEventCreate(&e));
    return e;
}

// launch with timing attribution to a profile family
template <typename Kern, typename... Args>
inline void launch_prof(Ctx& c, int family, double bytes, Kern k, unsigned grid, unsigned block, size_t smem,
                        Args... args) {
    if (grid == 0) return;
    if (!c.profile || !((c.prof_mask >> family) & 1u)) {
        launch_raw(c, k, grid, block, smem, args...);
        return;
    }
    cudaEvent_t e0 = prof_event(c), e1 = prof_event(c);
    AMG_CK(cudaEventRecord(e0, c.s));
    launch_raw(c, k, grid, block, smem, args...);
    AMG_CK(cudaEventRecord(e1, c.s));
    ProfRecord& r = c.prof[family];
    r.launches += 1;
    r.bytes += bytes;
    r.pending.emplace_back(e0, e1);
    if (family == kProfOther && prof_other_enabled()) r.kernels.push_back(reinterpret_cast<const void*>(k));
}

// resolve pending event pairs into milliseconds (synchronises)
inline void prof_collect(Ctx& c) {
    AMG_CK(cudaStreamSynchronize(c.s));
    if (c.side2) AMG_CK(cudaStreamSynchronize(c.side2));
    for (auto& r : c.prof) {
        for (size_t q = 0; q < r.pending.size(); ++q) {
            auto& pr = r.pending[q];
            float ms = 0.f;
            AMG_CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
            r.ms += ms;
            if (q < r.kernels.size()) prof_other_add(r.kernels[q], ms);
            c.event_pool.push_back(pr.first);
            c.event_pool.push_back(pr.second);
        }
        r.pending.clear();
        r.kernels.clear();
    }
}

inline unsigned blocks_for(int64_t n, int per_block) {
    return static_cast<unsigned>((n + per_block - 1) / per_block);
}

// ---- primitives (primitives.cu) ------------------------------------------
// out[0..n] = exclusive prefix sum of in[0..n-1], out[n] = total.  Returns
// the total (synchronising read).  in may alias out only if in == out is false.
int64_t exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int64_t n, bool read_total = true,
                           const char* file = __builtin_FILE(), int line = __builtin_LINE());
int64_t exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n, bool read_total = true,
                           const char* file = __builtin_FILE(), int line = __builtin_LINE());
void fill_f64(Ctx& c, double* p, double v, int64_t n);
void fill_i32(Ctx& c, int32_t* p, int32_t v, int64_t n);
template <typename T>
void copy_d2d(Ctx& c, T* dst, const T* src, int64_t n) {
    if (n > 0) AMG_CK(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
}
template <typename T>
void copy_h2d(Ctx& c, T* dst, const T* src, int64_t n) {
    if (n > 0) AMG_CK(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyHostToDevice, c.s));
}
template <typename T>
void copy_d2h(Ctx& c, T* dst, const T* src, int64_t n) {
    if (n > 0) AMG_CK(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToHost, c.s));
}
// AMGCU_SYNC_TRACE=1: count the host synchronisations per call site (printed at exit)
void note_sync_site(const char* file, int line);

inline void sync(Ctx& c, const char* file = __builtin_FILE(), int line = __builtin_LINE()) {
    ++c.syncs;
    note_sync_site(file, line);
    if (sync_trace_on()) gap_before_sync(c.s, file, line);
    AMG_CK(cudaStreamSynchronize(c.s));
    if (sync_trace_on()) gap_after_sync();
}
template <typename T>
T read_scalar(Ctx& c, const T* dptr, const char* file = __builtin_FILE(), int line = __builtin_LINE()) {
    T v;
    AMG_CK(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, c.s));
    sync(c, file, line);
    return v;
}

// Batched scalar reads: stage(k, dptr) enqueues an async copy into pinned slot k;
// one flush() synchronises for all of them.
inline int64_t* pinned_slots(Ctx& c) {
    if (!c.pin) AMG_CK(cudaMallocHost(&c.pin, sizeof(int64_t) * Ctx::kPinSlots));
    return c.pin;
}
template <typename T>
inline void stage_scalar(Ctx& c, int slot, const T* dptr) {
    static_assert(sizeof(T) <= sizeof(int64_t), "scalar too wide");
    if (slot < 0 || slot >= Ctx::kPinSlots) throw std::logic_error("stage_scalar: slot out of range");
    AMG_CK(cudaMemcpyAsync(pinned_slots(c) + slot, dptr, sizeof(T), cudaMemcpyDeviceToHost, c.s));
}
template <typename T>
inline T staged(Ctx& c, int slot) {
    T v;
    std::memcpy(&v, c.pin + slot, sizeof(T));
    return v;
}

// Device CSR <-> host CSR
void upload_csr(Ctx& c, const amgcu_csr& h, DCsr& d);
void upload_csr(Ctx& c, const HostCsr& h, DCsr& d);
HostCsr download_csr(Ctx& c, const DCsr& d);
void clone_csr(Ctx& c, const DCsr& src, DCsr& dst);

}  // namespace amgcu
