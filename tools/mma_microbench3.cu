// mma_microbench3.cu -- issuer overheads: cycles per "op" (8x SS N64 K16 + 4x TS N128 K16,
// 4 commits) with extra barrier checks on already-completed mbarriers, and with 1 vs 2
// issuing warps.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mmab3 tools/mma_microbench3.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2604_12219_b200/csrc/sm100_ptx.cuh"

using namespace pasa::ptx;

__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}

template <int MODE, int NWARPS>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar[8];
    __shared__ uint64_t done[3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 98304 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
        for (int i = 0; i < 3; ++i) { mbar_init(&done[i], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) for (int i = 0; i < 3; ++i) mbar_arrive(&done[i]);   // phase 0 complete
    if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tbase;
    if (warp < NWARPS && lane == 0) {
        const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
        const uint32_t idQK = idesc_bf16_f32(128, 64, 0, 0), idPV = idesc_bf16_f32(128, 128, 0, 1);
        const uint64_t dq0 = umma_desc_sw128(q, 16, 1024), dk0 = umma_desc_sw128(kb, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(vb, 8192, 1024);
        const uint32_t tw = t + warp * 256;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (MODE == 1) {   // three sequential suspend-hinted waits on completed barriers
                mbar_wait_sleep(&done[0], 0); mbar_wait_sleep(&done[1], 0); mbar_wait_sleep(&done[2], 0);
            } else if (MODE == 2) {   // three plain try_waits
                mbar_wait(&done[0], 0); mbar_wait(&done[1], 0); mbar_wait(&done[2], 0);
            } else if (MODE == 3) {   // three non-blocking test_waits issued back to back
                bool a = test_wait(&done[0], 0), b = test_wait(&done[1], 0), c = test_wait(&done[2], 0);
                if (!(a && b && c)) { mbar_wait(&done[0], 0); mbar_wait(&done[1], 0); mbar_wait(&done[2], 0); }
            }
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                const uint32_t offk = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                mma_ss(tw + 128 + (it & 1) * 64, dq0 + off, dk0 + offk, idQK, kk > 0);
            }
            mma_commit(&bar[warp * 4 + 0]); mma_commit(&bar[warp * 4 + 1]);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_ts(tw, tw + 128 + (it & 1) * 64 + kk * 8, dv0 + ((kk * 2048) >> 4), idPV, 1u);
            mma_commit(&bar[warp * 4 + 2]); mma_commit(&bar[warp * 4 + 3]);
        }
        long long t1 = clock64();
        out[blockIdx.x * 2 + warp] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(t, 512); }
}

template <int MODE, int NW>
void run(const char* name, unsigned long long* d) {
    unsigned long long h[296];
    auto k = bench<MODE, NW>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 2000;
    k<<<148, 128, 100 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, 148 * 2 * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int c = 0; c < 148; ++c) s += h[2 * c];
    printf("%-44s %.1f cycles per op per warp (%d warp%s)\n", name, s / 148 / iters, NW, NW > 1 ? "s" : "");
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 2 * 8);
    run<0, 1>("MMAs + commits", d);
    run<1, 1>("+ 3 suspend-hinted waits (completed)", d);
    run<2, 1>("+ 3 try_waits (completed)", d);
    run<3, 1>("+ 3 test_waits back to back", d);
    run<0, 2>("MMAs + commits", d);
    run<1, 2>("+ 3 suspend-hinted waits (completed)", d);
    run<3, 2>("+ 3 test_waits back to back", d);
    return 0;
}
