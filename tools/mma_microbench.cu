// mma_microbench.cu -- cycles per tcgen05.mma for the shapes attn_sm100 uses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mmab tools/mma_microbench.cu
// Each CTA (1 per SM) issues N back-to-back MMAs from one thread and times them
// with clock64 around issue + commit + wait.  Operands are whatever is in smem /
// TMEM (values do not matter for timing).
#include <cstdio>
#include <cstdint>
#include "../paper_2604_12219_b200/csrc/sm100_ptx.cuh"

using namespace pasa::ptx;

template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tbase;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        uint32_t idesc;
        if (MODE == 0) idesc = idesc_bf16_f32(128, 64, 0, 0);     // SS  N=64  (QK)
        if (MODE == 1) idesc = idesc_bf16_f32(128, 128, 0, 1);    // TS  N=128 MN-major B (PV)
        if (MODE == 2) idesc = idesc_bf16_f32(128, 128, 0, 0);    // SS  N=128
        if (MODE == 3) idesc = idesc_bf16_f32(128, 128, 0, 0);    // TS  N=128 K-major B (F)
        if (MODE == 4) idesc = idesc_bf16_f32(128, 64, 0, 0);     // TS  N=64 (Q in TMEM)
        if (MODE == 5) idesc = idesc_bf16_f32(128, 256, 0, 0);    // SS  N=256
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint64_t ad = umma_desc_sw128(a + (it & 3) * 32, 16, 1024);
            const uint64_t bd = umma_desc_sw128(b + (it & 3) * 32, MODE == 1 ? 8192 : 16, 1024);
            if (MODE == 0 || MODE == 2 || MODE == 5) mma_ss(t + 256, ad, bd, idesc, it > 0);
            else mma_ts(t, t + 256 + (it & 7) * 8, bd, idesc, it > 0);
        }
        long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        out[blockIdx.x * 2 + 0] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(t, 512); }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 2 * 8);
    unsigned long long h[296];
    const char* names[] = {"SS M128 N64 K16 (QK, Q+K from smem)", "TS M128 N128 K16, B MN-major (PV)",
                           "SS M128 N128 K16", "TS M128 N128 K16, B K-major (F)",
                           "TS M128 N64 K16 (QK with Q in TMEM)", "SS M128 N256 K16"};
    for (int mode = 0; mode < 6; ++mode) {
        for (int grid : {1, 148}) {
            const int iters = 4096;
            void (*k)(unsigned long long*, int) = nullptr;
            switch (mode) {
                case 0: k = bench<0>; break; case 1: k = bench<1>; break; case 2: k = bench<2>; break;
                case 3: k = bench<3>; break; case 4: k = bench<4>; break; default: k = bench<5>; break;
            }
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
            k<<<grid, 128, 70 * 1024>>>(d, iters);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
            double issue = 0, total = 0;
            for (int c = 0; c < grid; ++c) { issue += h[2 * c]; total += h[2 * c + 1]; }
            issue /= grid; total /= grid;
            printf("%-42s grid=%3d  issue %.1f cyc/mma  complete %.1f cyc/mma\n", names[mode], grid,
                   issue / iters, total / iters);
        }
    }
    return 0;
}
