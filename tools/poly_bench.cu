// Throughput probe for the softmax's exponential paths (elements / clk / SM):
// 0 MUFU ex2.approx.f32, 1 ex2_fma2 (packed FADD2/FFMA2 polynomial + FMNMX + IMAD, no MUFU),
// 2 FFMA2 alone, 3 IMAD (mad.lo.u32) alone, 4 FMNMX alone, 5 the 1:1 MUFU + poly mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_12219_b200/csrc tools/poly_bench.cu -o tools/poly_bench
#include <cstdio>
#include "sm100_ptx.cuh"
using namespace pasa::ptx;
template <int MODE>
__global__ void k(float* out, int iters) {
    float2 a[8];
    for (int i = 0; i < 8; i++) a[i] = make_float2(-0.001f * (threadIdx.x + i), -0.002f * i);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE == 0) { a[i].x = ex2(a[i].x) - 1.0f; a[i].y = ex2(a[i].y) - 1.0f; }
            else if (MODE == 1) { float2 p = ex2_fma2(a[i]); a[i] = make_float2(p.x - 1.0f, p.y - 1.0f); }
            else if (MODE == 2) { a[i] = ffma2(a[i], make_float2(1.0001f, 1.0001f), make_float2(-0.5f, -0.5f)); }
            else if (MODE == 3) { uint32_t r0, r1;
                asm volatile("mad.lo.u32 %0, %1, 8388608, %2;" : "=r"(r0) : "r"(__float_as_uint(a[i].x)), "r"(__float_as_uint(a[i].y)));
                asm volatile("mad.lo.u32 %0, %1, 8388608, %2;" : "=r"(r1) : "r"(__float_as_uint(a[i].y)), "r"(__float_as_uint(a[i].x)));
                a[i] = make_float2(__uint_as_float(r0), __uint_as_float(r1)); }
            else if (MODE == 4) { a[i].x = fmaxf(a[i].x, -125.f + a[i].y); a[i].y = fmaxf(a[i].y, -120.f + a[i].x); }
            else if (MODE == 5) { if (i & 1) { float2 p = ex2_fma2(a[i]); a[i] = make_float2(p.x - 1.0f, p.y - 1.0f); }
                                  else { a[i].x = ex2(a[i].x) - 1.0f; a[i].y = ex2(a[i].y) - 1.0f; } }
        }
    }
    float s = 0;
    for (int i = 0; i < 8; i++) s += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(float* o, const char* name) {
    int iters = 2048, clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        k<MODE><<<148 * 4, 512>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double elems = 148.0 * 4 * 512 * iters * 16;
        if (rep == 2) printf("mode %d %-28s %.3f ms  %.2f elements/clk/SM at max clock %d MHz\n", MODE, name, ms,
                             elems / (ms * 1e-3) / (clk * 1e3) / 148, clk / 1000);
    }
}
int main() {
    float* o; cudaMalloc(&o, 148 * 4 * 512 * 4);
    run<0>(o, "MUFU ex2"); run<1>(o, "ex2_fma2 poly"); run<2>(o, "FFMA2"); run<3>(o, "IMAD");
    run<4>(o, "FMNMX"); run<5>(o, "MUFU:poly 1:1");
    return 0;
}
