// Softmax exponential loop in isolation (one 64-column op per iteration, the next op's
// reference m depending on this op's row sum, so nothing is loop-invariant): cycles per op
// per warp and exponentials per clock per SM with 1, 2, 4 warps per SM sub-partition.
// MODE 0: the attention kernel's loop (FFMA2 -> 2 x MUFU.EX2 -> FADD2 -> F2FP per pair).
// MODE N > 0: every N-th exponential pair on the FMA pipe (ex2_fma2) instead of MUFU.
// (An earlier version of this probe let ptxas hoist half of the exponentials out of the
// loop; check sm__inst_executed_pipe_xu.sum = 64 MUFU per op per warp under ncu.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/eb tools/exps_bench.cu -I paper_2604_12219_b200/csrc
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace pasa::ptx;

template <int MODE>
__global__ void __launch_bounds__(128) kern(const float* in, unsigned long long* cyc, uint32_t* sink,
                                            int ops) {
    uint32_t sa[32], sb[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        sa[c] = __float_as_uint(in[(threadIdx.x + c) & 255]);
        sb[c] = __float_as_uint(in[(threadIdx.x + 7 * c) & 255]);
    }
    float m = 0.f, l = 0.f;
    const float cs = 0.18033688f;
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int op = 0; op < ops; ++op) {
        const float2 cs2 = make_float2(cs, cs), nm2 = make_float2(-m, -m);
        uint32_t pk[32];
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const float2 xa = ffma2(make_float2(__uint_as_float(sa[2 * c]), __uint_as_float(sa[2 * c + 1])), cs2, nm2);
            const float2 xb = ffma2(make_float2(__uint_as_float(sb[2 * c]), __uint_as_float(sb[2 * c + 1])), cs2, nm2);
            float p0, p1, p2, p3;
            if (MODE > 0 && (2 * c) % MODE == 0) {
                const float2 e = ex2_fma2(xa);
                p0 = e.x; p1 = e.y;
            } else {
                p0 = ex2(xa.x); p1 = ex2(xa.y);
            }
            if (MODE > 0 && (2 * c + 1) % MODE == 0) {
                const float2 e = ex2_fma2(xb);
                p2 = e.x; p3 = e.y;
            } else {
                p2 = ex2(xb.x); p3 = ex2(xb.y);
            }
            a0 = fadd2(a0, make_float2(p0, p1));
            a1 = fadd2(a1, make_float2(p2, p3));
            pk[c] = pack_bf16(p0, p1);
            pk[16 + c] = pack_bf16(p2, p3);
        }
        const float h = a0.x + a0.y + a1.x + a1.y;
        l += h;
        m = fmaf(h, 1e-30f, m);   // the next op depends on this one
#pragma unroll
        for (int c = 0; c < 32; c += 2) acc ^= pk[c] + pk[c + 1];
    }
    const unsigned long long t1 = clock64();
    sink[blockIdx.x * 128 + threadIdx.x] = acc + __float_as_uint(l);
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 4 + threadIdx.x / 32] = t1 - t0;
}

template <int MODE>
void run(const float* in, unsigned long long* cyc, uint32_t* sink, int clk) {
    const int ops = 2048;
    for (int bps = 1; bps <= 4; bps *= 2) {
        const int grid = 148 * bps;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            kern<MODE><<<grid, 128>>>(in, cyc, sink, ops);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            static unsigned long long hc[148 * 4 * 4];
            cudaMemcpy(hc, cyc, grid * 4 * 8, cudaMemcpyDeviceToHost);
            double mean = 0;
            for (int i = 0; i < grid * 4; ++i) mean += (double)hc[i];
            mean /= grid * 4;
            const double exps = (double)grid * 128 * 64 * ops;
            if (rep == 1)
                printf("poly 1/%d  warps/SMSP %d: %.0f cycles per op per warp; %.3f ms; %.1f exps/clk/SM (wall, %d MHz)\n",
                       MODE, bps, mean / ops, ms, exps / (ms * 1e-3) / 148.0 / (clk * 1e3), clk / 1000);
        }
    }
}

int main() {
    float* in;
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&in, 256 * 4);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = -3.f + 0.02f * i;
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMalloc(&cyc, 148 * 4 * 4 * 8);
    cudaMalloc(&sink, 148 * 4 * 128 * 4);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    run<0>(in, cyc, sink, clk);
    run<8>(in, cyc, sink, clk);
    run<4>(in, cyc, sink, clk);
    run<3>(in, cyc, sink, clk);
    run<2>(in, cyc, sink, clk);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
