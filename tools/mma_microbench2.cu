// mma_microbench2.cu -- cost of the attention MMA-issuer loop skeleton:
// per "op": [fence] 4x TS N128 (PV) + commit x2, [fence] 8x SS N64 (QK) + commit x2.
// Variants: 0 = MMAs only, 1 = + commits, 2 = + commits + fences, 3 = + waits on
// an mbarrier committed by the previous op (like p_full/pv_done hand-offs).
#include <cstdio>
#include <cstdint>
#include "../paper_2604_12219_b200/csrc/sm100_ptx.cuh"

using namespace pasa::ptx;

template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar[4];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 98304 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
    if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tbase;
    if (threadIdx.x == 0) {
        const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
        const uint32_t idQK = idesc_bf16_f32(128, 64, 0, 0), idPV = idesc_bf16_f32(128, 128, 0, 1);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (MODE >= 3 && it > 0) mbar_wait(&bar[2], (it - 1) & 1);   // previous op's completion
            if (MODE >= 2) tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t bd = umma_desc_sw128(vb + kk * 2048, 8192, 1024);
                mma_ts(t, t + 128 + (it & 1) * 64 + kk * 8, bd, idPV, 1u);
            }
            if (MODE >= 1) { mma_commit(&bar[0]); mma_commit(&bar[2]); }
            if (MODE >= 2) tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk & 3) * 32;
                const uint64_t ad = umma_desc_sw128(q + (kk >> 2) * 16384 + off, 16, 1024);
                const uint64_t bd = umma_desc_sw128(kb + (kk >> 2) * 8192 + off, 16, 1024);
                mma_ss(t + 256 + (it & 1) * 64, ad, bd, idQK, kk > 0);
            }
            if (MODE >= 1) { mma_commit(&bar[1]); mma_commit(&bar[3]); }
        }
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(t, 512); }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    unsigned long long h[148];
    const char* names[] = {"MMAs only", "+ commits", "+ commits + fences", "+ wait prev op done"};
    for (int mode = 0; mode < 4; ++mode) {
        void (*k)(unsigned long long*, int) = mode == 0 ? bench<0> : mode == 1 ? bench<1>
                                            : mode == 2 ? bench<2> : bench<3>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        const int iters = 2000;
        k<<<148, 128, 100 * 1024>>>(d, iters);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double s = 0;
        for (int c = 0; c < 148; ++c) s += h[c];
        printf("%-28s %.1f cycles per op (ideal 4x64 + 8x48 = 640)\n", names[mode], s / 148 / iters);
    }
    return 0;
}
