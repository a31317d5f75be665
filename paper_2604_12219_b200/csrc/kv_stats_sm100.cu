// kv_stats_sm100.cu -- the K/V block statistics of pasa_attn on the Blackwell tensor
// cores (bf16, d = 128 or 64): Kbar_j (bf16 copy of the route's fp64 block means),
// Vsum_j, and the grouped first-order statistic
//   Hbar^(g) = (1/|G_g|) sum_{j in G_g} sum_n (K_{j,n} - Kbar_j)^T V_{j,n}
//            = (1/|G_g|) [ sum_{n in G_g} K_n^T V_n  -  sum_{j in G_g} Kbar_j^T Vsum_j ]
// (Eq. 5 + App. B).  The first term is one contraction over all
// of the group's tokens, run on tcgen05 straight from TMA-loaded K / V tiles (both
// operands MN-major: Ht[n][k] = sum_t V[t][n] K[t][k]); the second (the exact centring
// correction, rank 1 per block) is accumulated in fp32 on CUDA cores.  Per-block H_j is
// never materialised.  One CTA per (head, group) -- or per 32-block
// chunk of a group larger than 32 blocks, reduced afterwards in a fixed order --,
// 2-stage (d = 128) / 4-stage (d = 64) TMA ring with two CTAs per SM, HBM bound:
// 2 S d * 2 bytes per head.
// d = 64: the MMA keeps M = 128 with the A operand's second 64-row half pointed at a
// zeroed 8 KB region of the stage (rows 64..127 of the accumulator are 0 and unused).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>

#include "pasa_internal.h"
#include "sm100_ptx.cuh"

namespace pasa {
namespace {

using namespace ptx;

constexpr int kBk = 64;
constexpr int kMaxStages = 4;
constexpr int kBox = kBk * 128;             // 8 KB: 64 tokens x 64 dims (128-byte rows)
constexpr int kMaxG = 32;                   // blocks per group handled by one CTA's smem
constexpr int kThreads = 256;               // warp 0 TMA, warp 1 MMA, warps 4-7 math
constexpr int kChunkBlocks = 32;

template <int D>
struct SGeo {
    static constexpr int NBOX = D / 64;
    static constexpr int TILE = kBk * D * 2;            // one K or V block tile
    // stage: K tile | V tile | (d = 64) zero box for the A operand's padded rows
    static constexpr int STAGE = 2 * TILE + (D == 64 ? kBox : 0);
    // ring depth per CTA: two CTAs per SM (one's epilogue overlaps the other's loads)
    static constexpr int STAGES = D == 64 ? 4 : 2;
};

struct Args {
    int64_t H, NK, NG, S;
    int32_t G;
    const double* kbar;       // [BH][NK][D] fp64 (route)
    __nv_bfloat16* kbar_lp;   // [BH][NK][D]
    __nv_bfloat16* vsum_lp;   // [BH][NK][D]
    __nv_bfloat16* ht;        // [BH][NG][D][D]
    float* part;              // G > kMaxG: fp32 partial sums [BH][NC][D][D] of 32-block chunks
    int64_t NC;               // chunks per head (ceil(N_K / 32)) when part != nullptr
};

struct Ctl {
    uint64_t full[kMaxStages], empty[kMaxStages], acc_full;
    uint32_t tmem_base;
};
template <int D>
struct Scratch {              // dynamic smem after the TMA stages
    float vsum[kMaxG][D];     // fp32 Vsum_j of the group's blocks
    float kb[kMaxG][D];       // fp32 Kbar_j
    float part[4][D];         // per-warp partial column sums
};

template <int D>
__global__ void __launch_bounds__(kThreads, 2)
    kv_stats_sm100_kernel(const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const Args a) {
    using G_ = SGeo<D>;
    constexpr uint32_t kCols = D;             // accumulator columns (N = D)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ Ctl ctl;
    Scratch<D>& sc = *reinterpret_cast<Scratch<D>*>(smem + G_::STAGES * G_::STAGE);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t g = blockIdx.x, bh = blockIdx.y;
    const int64_t b = bh / a.H, h = bh % a.H;
    // one group per CTA (G <= kMaxG), or one 32-block chunk of a large group
    const int64_t j0 = a.part ? g * kChunkBlocks : g * a.G;
    const int nb = (int)min(a.part ? (int64_t)kChunkBlocks : (int64_t)a.G, a.NK - j0);

    if (tid == 0) {
        for (int s = 0; s < G_::STAGES; ++s) {
            mbar_init(&ctl.full[s], 1);
            mbar_init(&ctl.empty[s], 2);     // MMA commit + the math warpgroup
        }
        mbar_init(&ctl.acc_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(&ctl.tmem_base, kCols);
        tmem_relinquish();
    }
    if constexpr (D == 64) {                 // the zero boxes (never written by TMA)
        for (int e = tid; e < G_::STAGES * kBox / 16; e += kThreads) {
            const int s = e / (kBox / 16), w = e % (kBox / 16);
            reinterpret_cast<uint4*>(smem + s * G_::STAGE + 2 * G_::TILE)[w] =
                make_uint4(0u, 0u, 0u, 0u);
        }
        fence_proxy_async();                 // generic-proxy zeros visible to the MMA
    }
    // fp32 Kbar of the group (and its bf16 copy for the attention kernel)
    for (int e = tid; e < nb * D; e += kThreads) {
        const int jj = e / D, d = e % D;
        const double kv = a.kbar[(bh * a.NK + j0 + jj) * D + d];
        sc.kb[jj][d] = (float)kv;
        a.kbar_lp[(bh * a.NK + j0 + jj) * D + d] = __float2bfloat16_rn((float)kv);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = ctl.tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            for (int jj = 0; jj < nb; ++jj) {
                const int s = jj % G_::STAGES;
                mbar_wait_sleep(&ctl.empty[s], ((jj / G_::STAGES) & 1) ^ 1);
                uint8_t* st = smem + s * G_::STAGE;
                mbar_arrive_expect_tx(&ctl.full[s], 2 * G_::TILE);
                const int tok = (int)((j0 + jj) * kBk);
#pragma unroll
                for (int bx = 0; bx < G_::NBOX; ++bx) {
                    tma_load_4d(st + bx * kBox, &tmK, &ctl.full[s], 64 * bx, tok, (int)h, (int)b);
                    tma_load_4d(st + G_::TILE + bx * kBox, &tmV, &ctl.full[s], 64 * bx, tok,
                                (int)h, (int)b);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // Ht[n][k] += sum_t V[t][n] K[t][k]:  A = V^T (M = n, MN-major), B = K (N = k, MN-major)
        // d = 64: A rows 64..127 come from the zero box one LBO (8 KB) after the V tile
        constexpr uint32_t kId = idesc_bf16_f32(128, D, 1, 1);
        const uint64_t d0 = umma_desc_sw128(smem_u32(smem), kBox, 1024);
        for (int jj = 0; jj < nb; ++jj) {
            const int s = jj % G_::STAGES;
            mbar_wait_sleep(&ctl.full[s], (jj / G_::STAGES) & 1);
            tc_fence_after();
            if (lane == 0) {
#pragma unroll
                for (int kk = 0; kk < kBk / 16; ++kk) {
                    const uint32_t offk = ((uint32_t)s * G_::STAGE + kk * 2048) >> 4;
                    const uint32_t offv = ((uint32_t)s * G_::STAGE + G_::TILE + kk * 2048) >> 4;
                    mma_ss(tbase, d0 + offv, d0 + offk, kId, (jj > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(&ctl.empty[s]);
                if (jj == nb - 1) mma_commit(&ctl.acc_full);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // Vsum_j: thread t sums 8 consecutive dims (one 16-byte chunk) over RPT rows
        constexpr int CH = D / 8;                // 16-byte chunks per row
        constexpr int RG = 128 / CH;             // row groups
        constexpr int RPT = kBk / RG;            // rows per thread
        const int mt = tid - 128;                // 0..127
        const int chunk = mt % CH;
        const int rg = mt / CH;
        const int bx = chunk >> 3, c16 = chunk & 7;
        for (int jj = 0; jj < nb; ++jj) {
            const int s = jj % G_::STAGES;
            mbar_wait_sleep(&ctl.full[s], (jj / G_::STAGES) & 1);
            const uint8_t* vt = smem + s * G_::STAGE + G_::TILE + bx * kBox;
            float acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
            for (int rr = 0; rr < RPT; ++rr) {
                const int t = rg * RPT + rr;
                const uint4 u = *reinterpret_cast<const uint4*>(vt + t * 128 + ((c16 ^ (t & 7)) << 4));
                const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(v2[e]);
                    acc[2 * e] += f.x;
                    acc[2 * e + 1] += f.y;
                }
            }
            // reduce the row groups of this warp (lanes with equal chunk), then smem
#pragma unroll
            for (int o = CH; o < 32; o <<= 1)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
            if (lane < CH) {
#pragma unroll
                for (int e = 0; e < 8; ++e) sc.part[warp - 4][chunk * 8 + e] = acc[e];
            }
            bar_sync(1, 128);
            if (mt == 0) mbar_arrive(&ctl.empty[s]);   // this warpgroup is done with the stage
            if (mt < D) {
                const int d = mt;
                const float vs = sc.part[0][d] + sc.part[1][d] + sc.part[2][d] + sc.part[3][d];
                sc.vsum[jj][d] = vs;
                a.vsum_lp[(bh * a.NK + j0 + jj) * D + d] = __float2bfloat16_rn(vs);
            }
            bar_sync(1, 128);
        }
        // epilogue: thread n (n < D) owns row n of Ht (TMEM lane n)
        mbar_wait_sleep(&ctl.acc_full, 0);
        tc_fence_after();
        const int n = mt;
        const uint32_t t_row = tbase + ((uint32_t)((warp & 3) * 32) << 16);
        const float inv = 1.f / (float)nb;
        if (warp - 4 < D / 32) {                      // warps holding lanes 0..D-1
            __nv_bfloat16* out = a.ht + ((bh * a.NG + g) * D + n) * D;
            float* pout = a.part ? a.part + ((bh * a.NC + g) * D + n) * D : nullptr;
#pragma unroll 1
            for (int c0 = 0; c0 < D; c0 += 32) {
                uint32_t raw[32];
                tmem_ld32(t_row + c0, raw);
                tmem_wait_ld();
                float acc[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) acc[c] = __uint_as_float(raw[c]);
                // exact centring: subtract sum_j Vsum_j[n] Kbar_j[k]
                for (int jj = 0; jj < nb; ++jj) {
                    const float vs = sc.vsum[jj][n];
                    const float4* kb4 = reinterpret_cast<const float4*>(&sc.kb[jj][c0]);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 kv = kb4[c];
                        acc[4 * c + 0] = fmaf(-vs, kv.x, acc[4 * c + 0]);
                        acc[4 * c + 1] = fmaf(-vs, kv.y, acc[4 * c + 1]);
                        acc[4 * c + 2] = fmaf(-vs, kv.z, acc[4 * c + 2]);
                        acc[4 * c + 3] = fmaf(-vs, kv.w, acc[4 * c + 3]);
                    }
                }
                if (pout) {                       // partial sum of the chunk (fp32)
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<float4*>(pout + c0)[q] =
                            make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
                    continue;
                }
                uint4 pk[4];
                uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
                for (int c = 0; c < 16; ++c) pw[c] = pack_bf16(acc[2 * c] * inv, acc[2 * c + 1] * inv);
#pragma unroll
                for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(out + c0)[q] = pk[q];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, kCols);
    }
}

// Large groups: H-bar^(g) = (sum of the group's chunk partials, chunks in
// ascending order) / |G_g|, stored bf16.  Chunks never straddle a group (G is a
// multiple of 32, or a single group).
template <int D>
__global__ void __launch_bounds__(256) stats_reduce_kernel(const Args a) {
    const int64_t g = blockIdx.x, bh = blockIdx.z;
    const int64_t e = (int64_t)blockIdx.y * 256 + threadIdx.x;      // element of D x D
    const int64_t c0 = g * a.G / kChunkBlocks;
    const int64_t jend = min((g + 1) * (int64_t)a.G, a.NK);
    const int64_t c1 = (jend + kChunkBlocks - 1) / kChunkBlocks;
    float s = 0.f;
    for (int64_t c = c0; c < c1; ++c) s += a.part[(bh * a.NC + c) * D * D + e];
    const float inv = 1.f / (float)(jend - g * a.G);
    a.ht[(bh * a.NG + g) * D * D + e] = __float2bfloat16_rn(s * inv);
}

template <int D>
cudaError_t launch_d(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r, cudaStream_t st,
                     int* launches) {
    char why[128];
    CUtensorMap mK, mV;
    auto act = [&](CUtensorMap* m, const pasa_tensor& t) {
        uint64_t dims[4] = {(uint64_t)t.D, (uint64_t)t.S, (uint64_t)t.H, (uint64_t)t.B};
        uint64_t str[3] = {(uint64_t)t.sS * 2, (uint64_t)t.sH * 2, (uint64_t)t.sB * 2};
        uint32_t box[4] = {64, (uint32_t)kBk, 1, 1};
        return make_tensor_map(m, t.data, 4, dims, str, box, why, sizeof(why));
    };
    if (!act(&mK, k) || !act(&mV, v)) return cudaErrorInvalidValue;
    Args a;
    a.H = r->H; a.NK = r->NK; a.NG = r->NG; a.S = r->S; a.G = r->cfg.G;
    a.kbar = r->kbar;
    a.kbar_lp = reinterpret_cast<__nv_bfloat16*>(r->kbar_lp);
    a.vsum_lp = reinterpret_cast<__nv_bfloat16*>(r->vsum_lp);
    a.ht = reinterpret_cast<__nv_bfloat16*>(r->ht);
    const bool chunked = r->cfg.G > kMaxG;
    a.part = chunked ? r->part : nullptr;
    a.NC = (r->NK + kChunkBlocks - 1) / kChunkBlocks;
    const size_t smem = (size_t)SGeo<D>::STAGES * SGeo<D>::STAGE + sizeof(Scratch<D>) + 1024;
    auto kern = kv_stats_sm100_kernel<D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)(chunked ? a.NC : r->NG), (unsigned)r->BH);
    kern<<<grid, kThreads, smem, st>>>(mK, mV, a);
    *launches += 1;
    if (chunked) {
        stats_reduce_kernel<D><<<dim3((unsigned)r->NG, D * D / 256, (unsigned)r->BH), 256, 0, st>>>(a);
        *launches += 1;
    }
    return cudaGetLastError();
}

}  // namespace

bool kv_stats_sm100_supported(const pasa_route_s* r) {
    return (r->D == 128 || r->D == 64) &&
           (r->cfg.G <= kMaxG || (r->part != nullptr && (r->cfg.G % kChunkBlocks == 0 ||
                                                         r->cfg.G >= r->NK)));
}

cudaError_t launch_kv_stats_sm100(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r,
                                  cudaStream_t st, int* launches) {
    return r->D == 128 ? launch_d<128>(k, v, r, st, launches) : launch_d<64>(k, v, r, st, launches);
}

}  // namespace pasa
