// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma8 tools/dfma_operands_bench.cu && /tmp/dfma8
#include <cstdio>
#include <cuda_runtime.h>
// 8 warps per SM, 64 independent fp64 accumulators per thread (the scores / H_j shape):
// acc[a][c] = fma(q[a], k[c], acc[a][c]) with q, k refreshed from shared memory per step
template <bool SMEM>
__global__ void __launch_bounds__(256, 1) k8(double* out, int iters, long long* cyc) {
    __shared__ double sq[16][128], sk[16][128];
    for (int e = threadIdx.x; e < 16 * 128; e += 256) { (&sq[0][0])[e] = e * 1e-7; (&sk[0][0])[e] = e * 2e-7; }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[8][8];
    for (int a = 0; a < 8; ++a) for (int c = 0; c < 8; ++c) acc[a][c] = 0;
    double qv[8], kv[8];
    for (int a = 0; a < 8; ++a) { qv[a] = sq[0][ty + 16 * a]; kv[a] = sk[0][tx + 16 * a]; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int dd = 0; dd < 16; ++dd) {
            if (SMEM) {
#pragma unroll
                for (int a = 0; a < 8; ++a) qv[a] = sq[dd][ty + 16 * a];
#pragma unroll
                for (int c = 0; c < 8; ++c) kv[c] = sk[dd][tx + 16 * c];
            }
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[a][c] = fma(qv[a], kv[c], acc[a][c]);
        }
    }
    long long t1 = clock64();
    double s = 0; for (int a = 0; a < 8; ++a) for (int c = 0; c < 8; ++c) s += acc[a][c];
    out[blockIdx.x * 256 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; long long* cyc; cudaMalloc(&out, 8 * 256 * sms); cudaMalloc(&cyc, 8 * sms);
    for (int smem = 0; smem < 2; ++smem) {
        auto kern = smem ? k8<true> : k8<false>;
        kern<<<sms, 256>>>(out, 10, cyc);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        const int iters = 4000;
        cudaEventRecord(e0); kern<<<sms, 256>>>(out, iters, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double dfma = (double)sms * 256 * iters * 16 * 64;
        printf("smem=%d: %.2f TFLOP/s fp64, %.1f DFMA/clk/SM (8 warps/SM, 64 acc/thread)\n", smem,
               2 * dfma / (ms * 1e-3) / 1e12, dfma / sms / (double)c);
    }
    return 0;
}
