// fp64 FMA throughput probe (B200): every thread runs 8 independent DFMA chains;
// prints DFMA/clk/SM and TFLOP/s at the clock the kernel saw (clock64 over the loop).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma tools/dfma_bench.cu && /tmp/dfma
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, long iters, long long* cyc) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    const double b = 0.999999, c = 1e-7;
    long long t0 = clock64();
    for (long n = 0; n < iters; ++n) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 512, blocks = sms * 4;
    const long iters = 20000;
    double* out; long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    dfma_kernel<<<blocks, threads>>>(out, 100, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long* hc = new long long[blocks];
    cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    long long cmax = 0;
    for (int i = 0; i < blocks; ++i) cmax = hc[i] > cmax ? hc[i] : cmax;
    const double dfma = (double)blocks * threads * iters * 8;
    printf("SMs %d: %.3f ms, %.2f TFLOP/s fp64, %.1f DFMA/clk/SM (4 CTAs x 512 threads per SM; "
           "per-CTA loop %lld cycles => clock %.2f GHz)\n", sms, ms, 2 * dfma / (ms * 1e-3) / 1e12,
           dfma / sms / ((double)cmax), cmax, cmax / (ms * 1e-3) / 1e9);
    return 0;
}
