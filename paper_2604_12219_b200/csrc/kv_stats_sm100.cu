// kv_stats_sm100.cu -- the K/V block statistics of pasa_attn on the Blackwell tensor
// cores (bf16, d = 128 or 64): Kbar_j (bf16 copy of the route's fp64 block means),
// Vsum_j, and the grouped first-order statistic
//   Hbar^(g) = (1/|G_g|) sum_{j in G_g} sum_n (K_{j,n} - Kbar_j)^T V_{j,n}
//            = (1/|G_g|) [ sum_{n in G_g} K_n^T V_n  -  sum_{j in G_g} Kbar_j^T Vsum_j ]
// (Eq. 5 + App. B).  The first term is one contraction over all
// of the group's tokens, run on tcgen05 straight from TMA-loaded K / V tiles (both
// operands MN-major: Ht[n][k] = sum_t V[t][n] K[t][k]); the second (the exact centring
// correction, rank 1 per block) is accumulated in fp32 on CUDA cores.  Per-block H_j is
// never materialised.  Work item = (head, group), or a 32-block chunk of
// a group larger than 32 blocks (reduced afterwards in a fixed order); a persistent CTA
// per SM walks its items with one TMA ring (4 x 32 KB at d = 128) running across them and
// two TMEM accumulators, so item i's epilogue overlaps item i+1's loads.  HBM bound:
// 2 S d * 2 bytes per head.
// d = 64: the MMA keeps M = 128 with the A operand's second 64-row half pointed at a
// zeroed 8 KB region of the stage (rows 64..127 of the accumulator are 0 and unused).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>

#include "pasa_internal.h"
#include "sm100_ptx.cuh"

namespace pasa {
namespace {

using namespace ptx;

constexpr int kBk = 64;
constexpr int kBox = kBk * 128;             // 8 KB: 64 tokens x 64 dims (128-byte rows)
constexpr int kMaxG = 32;                   // blocks per work item (group or 32-block chunk)
constexpr int kThreads = 384;               // warp 0 TMA, warp 1 MMA, 4-7 Vsum, 8-11 epilogue
constexpr int kChunkBlocks = 32;

template <int D>
struct SGeo {
    static constexpr int NBOX = D / 64;
    static constexpr int TILE = kBk * D * 2;            // one K or V block tile
    // stage: K tile | V tile | (d = 64) zero box for the A operand's padded rows
    static constexpr int STAGE = 2 * TILE + (D == 64 ? kBox : 0);
    // ring depth across work items (one CTA per SM): 4 x 32 KB at d = 128, 6 x 24 KB at 64
    static constexpr int STAGES = D == 64 ? 6 : 4;
};

struct Args {
    int64_t H, NK, NG, S;
    int32_t G;
    const double* kbar;       // [BH][NK][D] fp64 (route)
    __nv_bfloat16* kbar_lp;   // [BH][NK][D]
    // FP8 QK^T variant: E4M3 K [BH][S][D] (scale kamax[bh] / 448) converted from the
    // stage's K tile by the Vsum warps, E4M3 Kbar [BH][NK][D] (scale kbamax[bh] / 448)
    uint8_t* k8;
    uint8_t* kb8;
    const uint32_t* kamax;
    const uint32_t* kbamax;
    __nv_bfloat16* vsum_lp;   // [BH][NK][D]
    __nv_bfloat16* ht;        // [BH][NG][D][D]
    float* part;              // G > kMaxG: fp32 partial sums [BH][NC][D][D] of 32-block chunks
    int64_t NC;               // chunks per head (ceil(N_K / 32)) when part != nullptr
    int64_t items_per_head;   // NG, or NC for chunked groups
    int64_t items;            // BH * items_per_head
};

constexpr int kNVS = 4;                     // TMEM slots of the per-block Vsum MMA
constexpr int kVsCols = 16;                 // N of the Vsum MMA (all columns equal)

struct Ctl {
    uint64_t full[8], empty[8];          // TMA ring
    uint64_t vs_full[kNVS], vs_empty[kNVS];   // per-block Vsum in TMEM (MMA <-> Vsum warps)
    uint64_t acc_full[2], acc_empty[2];  // TMEM accumulators (MMA <-> epilogue)
    uint64_t scr_full[2], scr_empty[2];  // Vsum / Kbar scratch (Vsum warps <-> epilogue)
    uint32_t tmem_base;
};
template <int D>
struct Scratch {              // dynamic smem after the TMA stages, double-buffered per item
    float vsum[2][kMaxG][D];  // fp32 Vsum_j of the item's blocks
    float kb[2][kMaxG][D];    // fp32 Kbar_j
    alignas(1024) __nv_bfloat16 ones[kVsCols][kBk];   // B operand of the Vsum MMA (2 KB)
};

// Persistent: one CTA per SM walks work items (head, group) = blockIdx.x, +gridDim.x, ...
// (head-major).  The TMA ring runs across items, the MMA warp accumulates item i in TMEM
// accumulator i & 1, and a separate epilogue warpgroup centres / stores item i while the
// ring and the Vsum warps already work on item i + 1.
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    kv_stats_sm100_kernel(const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const Args a) {
    using G_ = SGeo<D>;
    constexpr uint32_t kCols = D;             // accumulator columns (N = D) per buffer
    constexpr uint32_t kVsBase = 2 * kCols;   // Vsum slots after the two accumulators
    constexpr uint32_t kTmemAlloc = D == 128 ? 512 : 256;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ Ctl ctl;
    Scratch<D>& sc = *reinterpret_cast<Scratch<D>*>(smem + G_::STAGES * G_::STAGE);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    auto item_geo = [&](int64_t it, int64_t& bh, int64_t& g, int64_t& j0, int& nb) {
        bh = it / a.items_per_head;
        g = it % a.items_per_head;
        j0 = a.part ? g * kChunkBlocks : g * a.G;
        nb = (int)min(a.part ? (int64_t)kChunkBlocks : (int64_t)a.G, a.NK - j0);
    };

    if (tid == 0) {
        for (int s = 0; s < G_::STAGES; ++s) {
            mbar_init(&ctl.full[s], 1);
            // MMA commit (both MMAs read the stage) [+ the Vsum warps' E4M3 copy of K]
            mbar_init(&ctl.empty[s], a.k8 ? 2 : 1);
        }
        for (int s = 0; s < kNVS; ++s) {
            mbar_init(&ctl.vs_full[s], 1);
            mbar_init(&ctl.vs_empty[s], 128);
        }
        for (int b2 = 0; b2 < 2; ++b2) {
            mbar_init(&ctl.acc_full[b2], 1);
            mbar_init(&ctl.acc_empty[b2], 1);
            mbar_init(&ctl.scr_full[b2], 2);   // Vsum warpgroup + the Kbar loaders
            mbar_init(&ctl.scr_empty[b2], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(&ctl.tmem_base, kTmemAlloc);
        tmem_relinquish();
    }
    for (int e = tid; e < kVsCols * kBk / 2; e += kThreads)   // bf16 ones (0x3F80 pairs)
        reinterpret_cast<uint32_t*>(&sc.ones[0][0])[e] = 0x3F803F80u;
    fence_proxy_async();                     // generic-proxy ones visible to the MMA
    if constexpr (D == 64) {                 // the zero boxes (never written by TMA)
        for (int e = tid; e < G_::STAGES * kBox / 16; e += kThreads) {
            const int s = e / (kBox / 16), w = e % (kBox / 16);
            reinterpret_cast<uint4*>(smem + s * G_::STAGE + 2 * G_::TILE)[w] =
                make_uint4(0u, 0u, 0u, 0u);
        }
        fence_proxy_async();                 // generic-proxy zeros visible to the MMA
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = ctl.tmem_base;

    if (warp == 0) {
        // ======================= TMA producer (ring across items) =======================
        if (lane == 0) {
            int n = 0;
            for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
                int64_t bh, g, j0;
                int nb;
                item_geo(it, bh, g, j0, nb);
                const int b = (int)(bh / a.H), h = (int)(bh % a.H);
                for (int jj = 0; jj < nb; ++jj, ++n) {
                    const int s = n % G_::STAGES;
                    mbar_wait_sleep(&ctl.empty[s], ((n / G_::STAGES) & 1) ^ 1);
                    uint8_t* st = smem + s * G_::STAGE;
                    mbar_arrive_expect_tx(&ctl.full[s], 2 * G_::TILE);
                    const int tok = (int)((j0 + jj) * kBk);
#pragma unroll
                    for (int bx = 0; bx < G_::NBOX; ++bx) {
                        tma_load_4d(st + bx * kBox, &tmK, &ctl.full[s], 64 * bx, tok, h, b);
                        tma_load_4d(st + G_::TILE + bx * kBox, &tmV, &ctl.full[s], 64 * bx, tok, h,
                                    b);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer =======================
        // Ht[n][k] += sum_t V[t][n] K[t][k]:  A = V^T (M = n, MN-major), B = K (N = k, MN-major)
        // d = 64: A rows 64..127 come from the zero box one LBO (8 KB) after the V tile
        constexpr uint32_t kId = idesc_bf16_f32(128, D, 1, 1);
        // Vsum_j[n] = sum_t V[t][n] * 1: A = V^T as above, B = ones (N = 16, K-major)
        constexpr uint32_t kIdVs = idesc_bf16_f32(128, kVsCols, 1, 0);
        const uint64_t d0 = umma_desc_sw128(smem_u32(smem), kBox, 1024);
        const uint64_t d1 = umma_desc_sw128(smem_u32(&sc.ones[0][0]), 16, 1024);
        int n = 0, li = 0;
        for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x, ++li) {
            int64_t bh, g, j0;
            int nb;
            item_geo(it, bh, g, j0, nb);
            const int ab = li & 1;
            mbar_wait_sleep(&ctl.acc_empty[ab], ((li >> 1) & 1) ^ 1);   // epilogue of li - 2
            tc_fence_after();
            const uint32_t acc = tbase + ab * kCols;
            for (int jj = 0; jj < nb; ++jj, ++n) {
                const int s = n % G_::STAGES, vs = n % kNVS;
                mbar_wait_sleep(&ctl.full[s], (n / G_::STAGES) & 1);
                mbar_wait_sleep(&ctl.vs_empty[vs], ((n / kNVS) & 1) ^ 1);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int kk = 0; kk < kBk / 16; ++kk) {
                        const uint32_t offk = ((uint32_t)s * G_::STAGE + kk * 2048) >> 4;
                        const uint32_t offv = ((uint32_t)s * G_::STAGE + G_::TILE + kk * 2048) >> 4;
                        mma_ss(acc, d0 + offv, d0 + offk, kId, (jj > 0 || kk > 0) ? 1u : 0u);
                        mma_ss(tbase + kVsBase + vs * kVsCols, d0 + offv, d1 + ((kk * 32) >> 4),
                               kIdVs, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&ctl.empty[s]);
                    mma_commit(&ctl.vs_full[vs]);
                    if (jj == nb - 1) mma_commit(&ctl.acc_full[ab]);
                }
                __syncwarp();
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ============ Kbar_j of each item: fp32 copy for the epilogue, bf16 copy out ============
        // (independent loads batched 16 deep: the fp64 means come from L2 / HBM)
        const int lt = tid - 64;                 // 0..63
        int li = 0;
        for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x, ++li) {
            int64_t bh, g, j0;
            int nb;
            item_geo(it, bh, g, j0, nb);
            const int sb = li & 1;
            mbar_wait_sleep(&ctl.scr_empty[sb], ((li >> 1) & 1) ^ 1);   // epilogue of li - 2
            const double* src = a.kbar + (bh * a.NK + j0) * D;
            __nv_bfloat16* dst = a.kbar_lp + (bh * a.NK + j0) * D;
            float* kbs = &sc.kb[sb][0][0];
            const int ne = nb * D;
            float kinv = 1.f;
            if (a.kb8) {
                const float am = __uint_as_float(a.kbamax[bh]);
                kinv = am > 0.f ? 448.f / am : 1.f;
            }
            for (int e0 = lt; e0 < ne; e0 += 64 * 16) {
                double v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int e = e0 + 64 * u;
                    v[u] = e < ne ? __ldg(src + e) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int e = e0 + 64 * u;
                    if (e < ne) {
                        kbs[e] = (float)v[u];
                        dst[e] = __float2bfloat16_rn((float)v[u]);
                    }
                }
                if (a.kb8) {   // E4M3 Kbar, two elements per conversion
#pragma unroll
                    for (int u = 0; u < 16; u += 2) {
                        const int e = e0 + 64 * u;
                        if (e < ne) {
                            const uint16_t pr = cvt_e4m3x2((float)v[u] * kinv, 0.f);
                            a.kb8[(bh * a.NK + j0) * D + e] = (uint8_t)(pr & 0xffu);
                        }
                        const int e1 = e0 + 64 * (u + 1);
                        if (e1 < ne) {
                            const uint16_t pr = cvt_e4m3x2((float)v[u + 1] * kinv, 0.f);
                            a.kb8[(bh * a.NK + j0) * D + e1] = (uint8_t)(pr & 0xffu);
                        }
                    }
                }
            }
            bar_sync(3, 64);
            if (lt == 0) mbar_arrive(&ctl.scr_full[sb]);
        }
    } else if (warp >= 4 && warp < 8) {
        // ============ Vsum_j (and the item's fp32 / bf16 Kbar) per block ============
        // thread mt = TMEM lane mt = head dim n: Vsum_j[n] from the Vsum MMA's slot
        const int mt = tid - 128;                // 0..127
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        int n = 0, li = 0;
        for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x, ++li) {
            int64_t bh, g, j0;
            int nb;
            item_geo(it, bh, g, j0, nb);
            const int sb = li & 1;
            mbar_wait_sleep(&ctl.scr_empty[sb], ((li >> 1) & 1) ^ 1);   // epilogue of li - 2
            float kinv = 1.f;
            if (a.k8) {
                const float am = __uint_as_float(a.kamax[bh]);
                kinv = am > 0.f ? 448.f / am : 1.f;
            }
            for (int jj = 0; jj < nb; ++jj, ++n) {
                const int vs = n % kNVS;
                if (a.k8) {   // E4M3 copy of the stage's K tile: thread = (row, 64-dim box)
                    const int s = n % G_::STAGES;
                    mbar_wait_sleep(&ctl.full[s], (n / G_::STAGES) & 1);
                    const int t = mt >> 1, bx = mt & 1;
                    const int64_t tok = (j0 + jj) * kBk + t;
                    const uint8_t* kt = smem + s * G_::STAGE + bx * kBox + t * 128;
                    uint32_t o[16];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 u = *reinterpret_cast<const uint4*>(kt + ((c ^ (t & 7)) << 4));
                        const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
                        uint16_t pr[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 f = __bfloat1622float2(
                                *reinterpret_cast<const __nv_bfloat162*>(&wd[e]));
                            pr[e] = cvt_e4m3x2(f.x * kinv, f.y * kinv);
                        }
                        o[2 * c] = (uint32_t)pr[0] | ((uint32_t)pr[1] << 16);
                        o[2 * c + 1] = (uint32_t)pr[2] | ((uint32_t)pr[3] << 16);
                    }
                    if (tok < a.S) {
                        uint4* dst = reinterpret_cast<uint4*>(a.k8 + (bh * a.S + tok) * D + bx * 64);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
                    }
                    bar_sync(1, 128);
                    if (mt == 0) mbar_arrive(&ctl.empty[s]);
                }
                mbar_wait_sleep(&ctl.vs_full[vs], (n / kNVS) & 1);
                tc_fence_after();
                const float v = __uint_as_float(tmem_ld1(tbase + lane_off + kVsBase + vs * kVsCols));
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(&ctl.vs_empty[vs]);
                if (mt < D) {
                    sc.vsum[sb][jj][mt] = v;
                    a.vsum_lp[(bh * a.NK + j0 + jj) * D + mt] = __float2bfloat16_rn(v);
                }
            }
            bar_sync(1, 128);                    // every thread's vsum / kb entries written
            if (mt == 0) mbar_arrive(&ctl.scr_full[sb]);   // vsum / kb of the item complete
        }
    } else if (warp >= 8) {
        // ============ epilogue: thread n (n < D) owns row n of Ht (TMEM lane n) ============
        const int n = tid - 256;                     // 0..127
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        int li = 0;
        for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x, ++li) {
            int64_t bh, g, j0;
            int nb;
            item_geo(it, bh, g, j0, nb);
            const int ab = li & 1;
            mbar_wait_sleep(&ctl.acc_full[ab], (li >> 1) & 1);
            mbar_wait_sleep(&ctl.scr_full[ab], (li >> 1) & 1);
            tc_fence_after();
            const uint32_t t_row = tbase + lane_off + ab * kCols;
            const float inv = 1.f / (float)nb;
            if (n < D) {
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
                        const float vs = sc.vsum[ab][jj][n];
                        const float4* kb4 = reinterpret_cast<const float4*>(&sc.kb[ab][jj][c0]);
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
                    for (int c = 0; c < 16; ++c)
                        pw[c] = pack_bf16(acc[2 * c] * inv, acc[2 * c + 1] * inv);
#pragma unroll
                    for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(out + c0)[q] = pk[q];
                }
            }
            tc_fence_before();
            bar_sync(2, 128);
            if (n == 0) {
                mbar_arrive(&ctl.acc_empty[ab]);
                mbar_arrive(&ctl.scr_empty[ab]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, kTmemAlloc);
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
    a.k8 = r->k8;
    a.kb8 = r->kb8;
    a.kamax = r->kamax;
    a.kbamax = r->kbamax;
    a.vsum_lp = reinterpret_cast<__nv_bfloat16*>(r->vsum_lp);
    a.ht = reinterpret_cast<__nv_bfloat16*>(r->ht);
    const bool chunked = r->cfg.G > kMaxG;
    a.part = chunked ? r->part : nullptr;
    a.NC = (r->NK + kChunkBlocks - 1) / kChunkBlocks;
    a.items_per_head = chunked ? a.NC : r->NG;
    a.items = r->BH * a.items_per_head;
    const size_t smem = (size_t)SGeo<D>::STAGES * SGeo<D>::STAGE + sizeof(Scratch<D>) + 1024;
    auto kern = kv_stats_sm100_kernel<D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    static int n_sm = 0;
    if (n_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        if (n_sm <= 0) n_sm = 148;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(a.items, n_sm);
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
