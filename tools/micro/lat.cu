// Microbenchmark: dependent-latency of the operations on the Gauss-Seidel solver's
// serial path (fp64 add/mul, shared-memory load, shuffle, syncwarp round trip).
#include <cstdio>
__global__ void k_lat(double* out, long long* cyc, int reps) {
    __shared__ double sm[64];
    __shared__ int si[64];
    const int lane = threadIdx.x;
    sm[lane] = 1.0 + lane * 1e-3;
    si[lane] = (lane + 1) & 31;
    __syncwarp();
    double a = out[lane], b = 1e-9;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) a = a - b;  // dependent DADD
    long long t1 = clock64();
    for (int r = 0; r < reps; ++r) a = a * 0.999999;  // dependent DMUL
    long long t2 = clock64();
    int idx = lane;
    for (int r = 0; r < reps; ++r) idx = si[idx];  // dependent LDS
    long long t3 = clock64();
    double v = a;
    for (int r = 0; r < reps; ++r) v = __shfl_sync(0xffffffffu, v, (r + 1) & 31);  // dependent SHFL (double)
    long long t4 = clock64();
    volatile double* vs = sm;
    for (int r = 0; r < reps; ++r) {
        if (lane == 0) vs[r & 63] = v;
        __syncwarp();
        v = vs[r & 63] + 1.0;
    }  // store -> syncwarp -> load round trip
    long long t5 = clock64();
    for (int r = 0; r < reps; ++r) {
        v = vs[(idx + r) & 63];
        v = v * 1.0000001;
        if (lane == 0) vs[(idx + r + 1) & 63] = v;
        __syncwarp();
    }
    long long t6 = clock64();
    if (lane == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    }
    out[lane] = a + v + idx;
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 4096); cudaMemset(out, 0, 4096);
    cudaMallocManaged(&cyc, 64);
    const int reps = 4096;
    k_lat<<<1, 32>>>(out, cyc, reps);
    k_lat<<<1, 32>>>(out, cyc, reps);
    cudaDeviceSynchronize();
    const char* nm[] = {"DADD", "DMUL", "LDS dep", "SHFL f64 dep", "st.shared->syncwarp->ld", "ld->mul->st->syncwarp"};
    for (int i = 0; i < 6; ++i) printf("%-26s %.1f cycles\n", nm[i], double(cyc[i]) / reps);
}
