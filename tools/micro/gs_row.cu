// Microbenchmark: cycles per row of the Gauss-Seidel solver warp's phase B
// (lane k resolves term k, the warp chains the shuffled products), with the
// publication steps switched on one at a time.  nvcc -arch=sm_100a -O3 --fmad=false
#include <cstdio>
#include <cuda/atomic>

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void vstore(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

__global__ void k_row(double* out, int reps, int variant, int nterm, long long* cyc) {
    __shared__ double ta[16][32];
    __shared__ int toff[16][32];
    __shared__ double acc0[32], dinv[32];
    __shared__ unsigned long long xb[64];
    __shared__ unsigned long long ring[64];
    __shared__ int tag[64];
    __shared__ volatile int step;
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < 16; ++k) {
        ta[k][lane] = 0.01 * (k + 1);
        toff[k][lane] = (k == 1) ? 1 : -1;  // term 1 = xb of the previous row, others: products
    }
    acc0[lane] = 1.0;
    dinv[lane] = 0.25;
    xb[lane] = __double_as_longlong(0.5);
    xb[lane + 32] = __double_as_longlong(0.5);
    tag[lane] = tag[lane + 32] = -1;
    __syncwarp();
    long long st[4] = {0, 0, 0, 0};
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        for (int t = 0; t < 32; ++t) {
            long long c0 = clock64();
            double p = 0.0;
            const int nt = nterm;
            if (lane < nt) {
                const double ak = ta[lane][t];
                const int off = toff[lane][t];
                if (off < 0) {
                    p = ak;
                } else {
                    unsigned long long v = vload(&xb[(t + 63) & 63]);
                    p = ak * __longlong_as_double(v);
                }
            }
            double a0 = acc0[t];
            long long c1 = clock64();
            if (variant & 8) {
                // lane-0 serial (no shuffles): every lane evaluates all terms from smem
                a0 = acc0[t];
                for (int k = 0; k < nt; ++k) {
                    const double ak = ta[k][t];
                    const int off = toff[k][t];
                    a0 -= off < 0 ? ak : ak * __longlong_as_double(vload(&xb[(t + 63) & 63]));
                }
            } else
            for (int k0 = 0; k0 < nt; k0 += 8) {
                double pk[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) pk[u] = __shfl_sync(0xffffffffu, p, k0 + u);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (k0 + u < nt) a0 -= pk[u];
            }
            const double d = dinv[t];
            long long c2 = clock64();
            if (lane == 0) {
                const double xi = a0 * d;
                const unsigned long long xbits = __double_as_longlong(xi);
                vstore(&xb[t], xbits);
                if (variant & 1) {
                    const int idx = (rep * 32 + t) & 63;
                    *reinterpret_cast<volatile int*>(&tag[idx]) = -1;
                    __threadfence_block();
                    vstore(&ring[idx], xbits);
                    __threadfence_block();
                    *reinterpret_cast<volatile int*>(&tag[idx]) = rep * 32 + t;
                }
                if (variant & 2) {
                    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> o(
                        *reinterpret_cast<unsigned long long*>(&out[(rep * 32 + t) & 4095]));
                    o.store(xbits, cuda::memory_order_relaxed);
                }
                if (variant & 4) step = t + 1;
            }
            __syncwarp();
            long long c3 = clock64();
            st[0] += c1 - c0; st[1] += c2 - c1; st[2] += c3 - c2;
        }
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = st[0]; cyc[2] = st[1]; cyc[3] = st[2]; }
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 16);
    cudaMallocManaged(&cyc, 64);
    const int reps = 200;
    for (int nt : {2, 5, 8, 16})
        for (int v : {0, 3, 8, 11}) {
            k_row<<<1, 32>>>(out, reps, v, nt, cyc);
            cudaDeviceSynchronize();
            const double R = reps * 32.0;
            printf("terms %2d variant %2d (ring %d global %d serial %d): cycles/row %.1f  [resolve %.1f chain %.1f publish %.1f]\n",
                   nt, v, v & 1, (v >> 1) & 1, (v >> 3) & 1, cyc[0] / R, cyc[1] / R, cyc[2] / R, cyc[3] / R);
        }
    return 0;
}
