// Generic device primitives: tile-based exclusive scan (3 launches, deterministic),
// fills, CSR upload/download.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "device.cuh"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

namespace amgcu {

namespace {
struct SyncSites {
    std::mutex m;
    std::map<std::string, long> n;
    std::map<std::string, double> idle_ms;  // GPU idle after the synchronisations of a site
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::string open_site;
    cudaEvent_t open_ev = nullptr;
    std::chrono::steady_clock::time_point open_t;  // host time the synchronisation returned
    std::map<std::string, double> host_ms;          // host time from the return to the next launch
    std::map<std::string, double> host_max, idle_max;  // the largest single gap of a site
    bool on = std::getenv("AMGCU_SYNC_TRACE") != nullptr;
    void resolve() {
        for (auto& p : pending) {
            float ms = 0.f;
            if (cudaEventSynchronize(p.second.second) == cudaSuccess &&
                cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) {
                idle_ms[p.first] += ms;
                idle_max[p.first] = std::max<double>(idle_max[p.first], ms);
            }
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        pending.clear();
    }
    ~SyncSites() {
        if (!on) return;
        resolve();
        double tot = 0.0;
        for (auto& kv : n) {
            std::fprintf(stderr, "sync %6ld  idle %8.3f ms (max %7.3f)  host %8.3f ms (max %7.3f)  %s\n", kv.second,
                         idle_ms[kv.first], idle_max[kv.first], host_ms[kv.first], host_max[kv.first],
                         kv.first.c_str());
            tot += idle_ms[kv.first];
        }
        std::fprintf(stderr, "sync total GPU idle after synchronisations: %.3f ms\n", tot);
    }
};
SyncSites& sync_sites() {
    static SyncSites s;
    return s;
}
}  // namespace

bool sync_trace_on() { return sync_sites().on; }

void gap_before_sync(cudaStream_t s, const char* file, int line) {
    SyncSites& ss = sync_sites();
    std::lock_guard<std::mutex> g(ss.m);
    const char* base = std::strrchr(file, '/');
    if (ss.open_ev) cudaEventDestroy(ss.open_ev);  // two syncs without a launch between them
    cudaEventCreate(&ss.open_ev);
    cudaEventRecord(ss.open_ev, s);
    ss.open_site = std::string(base ? base + 1 : file) + ":" + std::to_string(line);
    if (ss.pending.size() > 4096) ss.resolve();
}

void gap_after_sync() {
    SyncSites& ss = sync_sites();
    std::lock_guard<std::mutex> g(ss.m);
    ss.open_t = std::chrono::steady_clock::now();
}

void gap_before_launch(cudaStream_t s) {
    SyncSites& ss = sync_sites();
    std::lock_guard<std::mutex> g(ss.m);
    if (!ss.open_ev) return;
    const double gap = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ss.open_t).count();
    ss.host_ms[ss.open_site] += gap;
    ss.host_max[ss.open_site] = std::max(ss.host_max[ss.open_site], gap);
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ss.pending.push_back({ss.open_site, {ss.open_ev, e}});
    ss.open_ev = nullptr;
}

void note_sync_site(const char* file, int line) {
    SyncSites& s = sync_sites();
    if (!s.on) return;
    const char* base = std::strrchr(file, '/');
    std::lock_guard<std::mutex> g(s.m);
    s.n[std::string(base ? base + 1 : file) + ":" + std::to_string(line)] += 1;
}

namespace {
struct OtherKernels {
    std::mutex m;
    std::map<std::string, std::pair<long, double>> t;  // symbol -> (launches, ms)
    ~OtherKernels() {
        std::vector<std::pair<double, std::string>> v;
        for (auto& kv : t) v.emplace_back(kv.second.second, kv.first);
        std::sort(v.rbegin(), v.rend());
        for (auto& e : v)
            std::fprintf(stderr, "other %9.3f ms %6ld x  %s\n", e.first, t[e.second].first, e.second.c_str());
    }
};
OtherKernels& other_kernels() {
    static OtherKernels o;
    return o;
}
}  // namespace

bool prof_other_enabled() {
    static const bool on = std::getenv("AMGCU_PROF_OTHER") != nullptr;
    return on;
}

void prof_other_add(const void* kernel, double ms) {
    const char* name = nullptr;
    if (cudaFuncGetName(&name, kernel) != cudaSuccess || !name) name = "?";
    OtherKernels& o = other_kernels();
    std::lock_guard<std::mutex> g(o.m);
    auto& e = o.t[name];
    e.first += 1;
    e.second += ms;
}

bool launch_check_enabled() {
    static const bool on = std::getenv("AMGCU_LAUNCH_CHECK") != nullptr;
    return on;
}

void launch_check(Ctx& c, const void* kernel) {
    const cudaError_t e = cudaStreamSynchronize(c.s);
    if (e == cudaSuccess) return;
    const char* name = nullptr;
    if (cudaFuncGetName(&name, kernel) != cudaSuccess || !name) name = "?";
    throw CudaFailure(std::string("kernel ") + name + " failed: " + cudaGetErrorString(e));
}

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kTile = kScanThreads * kScanItems;

template <typename T>
__global__ void k_tile_reduce(const T* __restrict__ in, int64_t n, T* __restrict__ tile_sums) {
    using BR = cub::BlockReduce<T, kScanThreads>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + static_cast<int64_t>(k) * kScanThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    T tot = BR(tmp).Sum(s);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// single block: exclusive scan of the tile sums in place; total -> tile_sums[ntiles]
template <typename T>
__global__ void k_scan_tile_sums(T* __restrict__ sums, int64_t ntiles) {
    using BS = cub::BlockScan<T, kScanThreads>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ T carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < ntiles; base += kTile) {
        T v[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const int64_t i = base + threadIdx.x * kScanItems + k;
            v[k] = i < ntiles ? sums[i] : T(0);
        }
        T agg;
        BS(tmp).ExclusiveSum(v, v, agg);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const int64_t i = base + threadIdx.x * kScanItems + k;
            if (i < ntiles) sums[i] = v[k] + carry;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[ntiles] = carry;
}

template <typename T>
__global__ void k_tile_scan(const T* __restrict__ in, T* __restrict__ out, int64_t n, const T* __restrict__ offs,
                            int64_t ntiles) {
    using BS = cub::BlockScan<T, kScanThreads>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
    T v[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + threadIdx.x * kScanItems + k;
        v[k] = i < n ? in[i] : T(0);
    }
    T agg;
    BS(tmp).ExclusiveSum(v, v, agg);
    const T off = offs ? offs[blockIdx.x] : T(0);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + threadIdx.x * kScanItems + k;
        if (i < n) out[i] = v[k] + off;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = offs ? offs[ntiles] : agg;
}

template <typename T>
struct PadZero {  // in[i] for i < n, 0 at i == n
    const T* in;
    int64_t n;
    __host__ __device__ T operator()(int64_t i) const { return i < n ? in[i] : T(0); }
};

template <typename T>
int64_t scan_impl(Ctx& c, const T* in, T* out, int64_t n, bool read_total, const char* file, int line) {
    if (n == 0) {
        AMG_CK(cudaMemsetAsync(out, 0, sizeof(T), c.s));
        return 0;
    }
    if (n <= kTile) {
        // one tile: one block scans it and writes the total
        const T zero = 0;
        launch(c, k_tile_scan<T>, 1u, kScanThreads, 0, in, out, n, static_cast<const T*>(nullptr), int64_t(0));
        (void)zero;
    } else {
        // single-pass decoupled look-back scan (cub::DeviceScan) over n + 1 items, the last
        // one zero, so out[n] is the total
        auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), PadZero<T>{in, n});
        size_t bytes = 0;
        AMG_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, out, n + 1, c.s));
        if (c.scan_tmp.size() < bytes) c.scan_tmp.alloc(std::max<size_t>(bytes, size_t(1) << 20), c.s);
        AMG_CK(cub::DeviceScan::ExclusiveSum(c.scan_tmp.get(), bytes, it, out, n + 1, c.s));
        c.launches += 2;
    }
    if (!read_total) return -1;
    return static_cast<int64_t>(read_scalar(c, static_cast<const T*>(out + n), file, line));
}

template <typename T>
__global__ void k_fill(T* p, T v, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace

int64_t exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int64_t n, bool read_total, const char* file,
                           int line) {
    return scan_impl<int32_t>(c, in, out, n, read_total, file, line);
}
int64_t exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n, bool read_total, const char* file,
                           int line) {
    return scan_impl<int64_t>(c, in, out, n, read_total, file, line);
}
void fill_f64(Ctx& c, double* p, double v, int64_t n) { launch(c, k_fill<double>, blocks_for(n, 256), 256, 0, p, v, n); }
void fill_i32(Ctx& c, int32_t* p, int32_t v, int64_t n) {
    launch(c, k_fill<int32_t>, blocks_for(n, 256), 256, 0, p, v, n);
}

void upload_csr(Ctx& c, const amgcu_csr& h, DCsr& d) {
    const int64_t nnz = h.row_offsets[h.n_rows];
    d.alloc(c, h.n_rows, h.n_cols, nnz);
    d.bs = h.block_size;
    copy_h2d(c, d.rp.get(), h.row_offsets, h.n_rows + 1);
    copy_h2d(c, d.ci.get(), h.col_indices, nnz);
    copy_h2d(c, d.va.get(), h.values, nnz);
}

void upload_csr(Ctx& c, const HostCsr& h, DCsr& d) {
    d.alloc(c, h.n_rows, h.n_cols, h.nnz());
    d.bs = h.block_size;
    copy_h2d(c, d.rp.get(), h.row_offsets.data(), h.n_rows + 1);
    copy_h2d(c, d.ci.get(), h.col_indices.data(), h.nnz());
    copy_h2d(c, d.va.get(), h.values.data(), h.nnz());
    sync(c);  // host vectors may go out of scope
}

HostCsr download_csr(Ctx& c, const DCsr& d) {
    HostCsr h;
    h.n_rows = d.nr;
    h.n_cols = d.nc;
    h.block_size = d.bs;
    h.row_offsets.resize(static_cast<size_t>(d.nr) + 1);
    h.col_indices.resize(static_cast<size_t>(d.nnz));
    h.values.resize(static_cast<size_t>(d.nnz));
    copy_d2h(c, h.row_offsets.data(), d.rp.get(), d.nr + 1);
    copy_d2h(c, h.col_indices.data(), d.ci.get(), d.nnz);
    copy_d2h(c, h.values.data(), d.va.get(), d.nnz);
    sync(c);
    return h;
}

void clone_csr(Ctx& c, const DCsr& src, DCsr& dst) {
    dst.alloc(c, src.nr, src.nc, src.nnz);
    dst.bs = src.bs;
    copy_d2d(c, dst.rp.get(), src.rp.get(), src.nr + 1);
    copy_d2d(c, dst.ci.get(), src.ci.get(), src.nnz);
    copy_d2d(c, dst.va.get(), src.va.get(), src.nnz);
}

}  // namespace amgcu
