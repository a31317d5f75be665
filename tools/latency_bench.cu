// Dependent-chain latency (cycles per instruction, one warp) of the softmax's instructions:
// MUFU.EX2, FADD2, FFMA2, FADD, F2FP pack, LOP3, and MUFU -> FADD2 / MUFU -> F2FP pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lb tools/latency_bench.cu -I paper_2604_12219_b200/csrc
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace pasa::ptx;

template <int MODE>
__global__ void kern(float seed, unsigned long long* cyc, float* sink, int n) {
    float x = seed * threadIdx.x, y = 0.5f;
    float2 v = make_float2(x, y);
    uint32_t u = __float_as_uint(x);
    const unsigned long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (MODE == 0) x = ex2(x) * -1.0f;                       // MUFU (+FMUL)
            if (MODE == 1) v = fadd2(v, make_float2(1e-7f, 2e-7f));   // FADD2
            if (MODE == 2) v = ffma2(v, make_float2(0.999f, 0.999f), make_float2(1e-7f, 1e-7f));
            if (MODE == 3) x = x + 1e-7f;                             // FADD
            if (MODE == 4) u = pack_bf16(__uint_as_float(u), 1.0f);   // F2FP
            if (MODE == 5) u = (u | 0x10u) ^ (u >> 3);                // LOP3 (+shift)
            if (MODE == 6) { const float p = ex2(v.x); v = fadd2(v, make_float2(p, p)); }   // MUFU -> FADD2
            if (MODE == 7) x = fmaf(x, 0.999f, 1e-7f);                // FFMA
        }
    }
    const unsigned long long t1 = clock64();
    sink[threadIdx.x] = x + v.x + v.y + __uint_as_float(u);
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    unsigned long long* c;
    float* s;
    cudaMalloc(&c, 8);
    cudaMalloc(&s, 4096);
    const char* names[] = {"MUFU.EX2 (+FMUL)", "FADD2", "FFMA2", "FADD", "F2FP", "LOP3+SHF",
                           "MUFU->FADD2", "FFMA"};
    for (int m = 0; m < 8; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            const int n = 4096;
            switch (m) {
                case 0: kern<0><<<1, 32>>>(0.001f, c, s, n); break;
                case 1: kern<1><<<1, 32>>>(0.001f, c, s, n); break;
                case 2: kern<2><<<1, 32>>>(0.001f, c, s, n); break;
                case 3: kern<3><<<1, 32>>>(0.001f, c, s, n); break;
                case 4: kern<4><<<1, 32>>>(0.001f, c, s, n); break;
                case 5: kern<5><<<1, 32>>>(0.001f, c, s, n); break;
                case 6: kern<6><<<1, 32>>>(0.001f, c, s, n); break;
                default: kern<7><<<1, 32>>>(0.001f, c, s, n); break;
            }
            unsigned long long h;
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("%-18s %.2f cycles per chain step\n", names[m], (double)h / (n * 16));
        }
    }
    return 0;
}
