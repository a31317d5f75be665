// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_exact tools/dmma_exact.cu && /tmp/dmma_exact
// Is DMMA m8n8k4 bit-identical to a sequential fma chain over k (c = fma(a_k, b_k, c), k = 0..3)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ double rnd(uint64_t& s) {   // xorshift -> double with varied exponents and signs
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    double m = (double)(s >> 11) * (1.0 / 9007199254740992.0);
    int e = (int)((s >> 3) & 31) - 16;
    return ((s & 1) ? -1.0 : 1.0) * ldexp(m + 0.5, e);
}
__global__ void k(int trials, unsigned long long* mism, unsigned long long* total, int ksteps) {
    const int lane = threadIdx.x & 31;
    __shared__ double A[8][4 * 64], B[4 * 64][8];
    uint64_t s = 0x9E3779B97F4A7C15ull ^ (blockIdx.x * 1315423911ull + threadIdx.x * 2654435761ull);
    for (int t = 0; t < trials; ++t) {
        for (int e = lane; e < 8 * 4 * ksteps; e += 32) { A[e / (4 * ksteps)][e % (4 * ksteps)] = rnd(s); }
        for (int e = lane; e < 4 * ksteps * 8; e += 32) { B[e / 8][e % 8] = rnd(s); }
        __syncwarp();
        const int r = lane >> 2, kk = lane & 3, c0 = 2 * (lane & 3);
        double d0 = 0.0, d1 = 0.0;
        for (int st = 0; st < ksteps; ++st) dmma(d0, d1, A[r][4 * st + kk], B[4 * st + kk][r]);
        // reference: sequential fma chain over k for outputs (r, c0) and (r, c0 + 1)
        double e0 = 0.0, e1 = 0.0;
        for (int q = 0; q < 4 * ksteps; ++q) { e0 = fma(A[r][q], B[q][c0], e0); e1 = fma(A[r][q], B[q][c0 + 1], e1); }
        unsigned long long m = (__double_as_longlong(d0) != __double_as_longlong(e0)) + (__double_as_longlong(d1) != __double_as_longlong(e1));
        atomicAdd(mism, m); atomicAdd(total, 2ull);
        __syncwarp();
    }
}
int main() {
    unsigned long long *m, *t; cudaMallocManaged(&m, 8); cudaMallocManaged(&t, 8);
    for (int ks = 1; ks <= 32; ks *= 32) {
        *m = 0; *t = 0;
        k<<<148, 32>>>(2000, m, t, ks); cudaDeviceSynchronize();
        printf("k = %d x 4: %llu of %llu outputs differ from the sequential fma chain\n", ks, *m, *t);
    }
    return 0;
}
