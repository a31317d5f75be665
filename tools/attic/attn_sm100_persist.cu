// attn_sm100_persist.cu -- pasa_attn at d = 64 as a PERSISTENT kernel: the same method, op
// list and per-op pipeline as attn_sm100.cu (Eq. 7; grouped first-order
// term, App. B :503-506; readings R-1..R-5, R-21, R-22), but each CTA
// walks a strided sequence of (head, 128-row q-block) items so that item j+1's ramp-up
// overlaps item j's tail.  At d = 64 a CTA's fixed cost (fill and drain of its pipeline,
// CTA turnover) is ~5 us against ~0.8 us per op -- 13-14 % of the CogVideoX-5B launch
// (profiles/r02_attn_softmax.md §8); here:
//   * the op list of item j+1 is built by warp 3 (idle in attn_sm100.cu) into the second
//     of two list buffers while item j runs;
//   * the K / V rings, the S buffers and every barrier phase continue across items (global
//     op index g): the producers run into item j+1's first tiles as soon as slots free;
//   * the next item's Q tile is loaded into the second Q buffer early; the softmax warps
//     copy it into TMEM right after releasing item j's last P, so QK^T of item j+1 runs
//     during item j's epilogue; the first PV of item j+1 waits only for O's read-out;
//   * TMEM is allocated and the barriers initialised once per CTA.
// Roles (256 threads, 2 CTAs per SM): warp 0 K ring + Q tiles, warp 1 TMEM + MMA issuer,
// warp 2 V ring, warp 3 op lists, warps 4-7 softmax / epilogue (one query row each).
// Domain: bf16, Bq = 128, Bk = 64, d = 64, G in {32, 64, multiples of 128, >= N_K} or no
// grouped term (the small-group bookkeeping of G = 8 / 16 stays in attn_sm100.cu).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "pasa_internal.h"
#include "sm100_ptx.cuh"

namespace pasa {
namespace {

using namespace ptx;

constexpr int kThreads = 256;
constexpr int kBQ = 128, kBK = 64, kD = 64;
constexpr int kMaxNK = 4096;
constexpr int kMaxOps = kMaxNK + kMaxNK / 64 + kMaxNK / 32 + 64;   // G >= 32
constexpr int kTmemCols = 256;
constexpr float kRescaleThresh = 8.f;   // log2 units
constexpr uint32_t kSCol = 64;          // S buffers at 64 + 64 b (O at 0..63)
constexpr uint32_t kQCol = 192;         // Q (bf16 pairs) at 192..223
constexpr int kNB = 2;                  // S buffers = K slots = V slots
constexpr int kQBox = kBQ * 128;        // 16 KB: a Q tile (64 bf16 per row)
constexpr int kSlot = kBK * 128;        // 8 KB: a K / V tile
constexpr int kOffQ = 0;                // two Q buffers
constexpr int kOffK = 2 * kQBox;
constexpr int kOffV = kOffK + kNB * kSlot;
constexpr int kBytes = kOffV + kNB * kSlot;   // 64 KB

enum : int32_t { OP_E = 0, OP_C = 1, OP_F = 2 };
__device__ __forceinline__ uint16_t op_make(int32_t type, int32_t v) {
    return (uint16_t)((type << 14) | v);
}
__device__ __forceinline__ int32_t op_type(int32_t op) { return op >> 14; }
__device__ __forceinline__ int32_t op_val(int32_t op) { return op & 0x3FFF; }

struct Params {
    int64_t S, H, NQ, NK, W;
    int64_t it0, it1;   // the handle's (head, q-block) items
    int32_t G, comp;
    float scale_log2;   // s * log2(e)
    float s;            // 1/sqrt(D)
    const int32_t* idx;
    const int32_t* count;
    const uint32_t* mask;
    __nv_bfloat16* out;
    int64_t osB, osS, osH;
    int32_t* counter;   // dynamic item scheduler (zeroed before the launch)
};

struct List {
    int32_t nops;           // -1: no more items (the scheduler ran past the range)
    int32_t item;
    uint32_t mask[kMaxNK / 32];
    uint16_t ops[kMaxOps];
};

struct Ctl {
    uint64_t q_full[2], q_empty[2];        // per Q buffer (item j & 1)
    uint64_t q_tmem, o_free;               // per item: Q in TMEM / O read out (128 arrivals)
    uint64_t k_full[kNB], k_empty[kNB], s_full[kNB], p_full[kNB], pv_done[kNB];
    uint64_t list_full[2], list_empty[2];  // per list buffer (item j & 1)
    uint32_t tmem_base;
    List list[2];
};
constexpr uint32_t kListReaders = 1 + 1 + 1 + 128;   // K producer, V producer, MMA, softmax

__global__ void __launch_bounds__(kThreads, 2)
    attn_sm100_persist_kernel(const __grid_constant__ CUtensorMap tmQ,
                              const __grid_constant__ CUtensorMap tmK,
                              const __grid_constant__ CUtensorMap tmV,
                              const __grid_constant__ CUtensorMap tmKb,
                              const __grid_constant__ CUtensorMap tmVs,
                              const __grid_constant__ CUtensorMap tmHt, const Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ Ctl ctl;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t NK = p.NK;
    // items come from a global counter in head-major order, so the CTAs in flight always
    // work on neighbouring q-blocks of the same heads and their K / V stay in L2 (a static
    // stride lets the CTAs drift apart: the dual-tile kernel saw 3x the DRAM traffic)

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&ctl.q_full[b], 1);
            mbar_init(&ctl.q_empty[b], 128);
            mbar_init(&ctl.list_full[b], 1);
            mbar_init(&ctl.list_empty[b], kListReaders);
        }
        mbar_init(&ctl.q_tmem, 128);
        mbar_init(&ctl.o_free, 128);
        for (int s = 0; s < kNB; ++s) {
            mbar_init(&ctl.k_full[s], 1);
            mbar_init(&ctl.k_empty[s], 1);
            mbar_init(&ctl.s_full[s], 1);
            mbar_init(&ctl.p_full[s], 129);   // softmax threads + the V producer
            mbar_init(&ctl.pv_done[s], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(&ctl.tmem_base, kTmemCols);
        tmem_relinquish();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
        tma_prefetch(&tmKb); tma_prefetch(&tmVs); tma_prefetch(&tmHt);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = ctl.tmem_base;

    if (warp == 3) {
        // ======================= op lists (one item ahead) =======================
        for (int j = 0;; ++j) {
            const int bb = j & 1;
            mbar_wait_sleep(&ctl.list_empty[bb], (uint32_t)(((j >> 1) & 1) ^ 1));
            List& L = ctl.list[bb];
            int64_t item = 0;
            if (lane == 0) item = p.it0 + atomicAdd(p.counter, 1);
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= p.it1) {
                if (lane == 0) {
                    L.nops = -1;
                    mbar_arrive(&ctl.list_full[bb]);
                }
                break;
            }
            const int64_t row = item;   // item = bh * NQ + i
            const int32_t cnt = p.count[row];
            for (int w = lane; w < p.W; w += 32) L.mask[w] = p.mask[row * p.W + w];
            for (int q = lane; q < cnt; q += 32) L.ops[q] = op_make(OP_E, p.idx[row * NK + q]);
            __syncwarp();
            if (lane == 0) {
                // tail: centroid chunks with a dropped block, then the first-order op of
                // every group that ends inside the chunk (as attn_sm100.cu)
                int n = cnt;
                if (p.comp != PASA_COMP_NONE && cnt < NK) {
                    const int W = (int)p.W;
                    auto dropped_word = [&](int w) {
                        const int64_t rem = NK - 32 * (int64_t)w;
                        const uint32_t inb = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
                        return (~L.mask[w] & inb) != 0u;
                    };
                    const int64_t G = p.G;
                    const int nchunks = (int)((NK + 63) / 64);
                    int64_t g = 0;
                    for (int c = 0; c < nchunks; ++c) {
                        if (dropped_word(2 * c) || (2 * c + 1 < W && dropped_word(2 * c + 1)))
                            L.ops[n++] = op_make(OP_C, c);
                        if (p.comp == PASA_COMP_GROUPED) {
                            const int64_t chunk_end = min(64 * (int64_t)(c + 1), NK);
                            for (; g * G < NK && min((g + 1) * G, NK) <= chunk_end; ++g) {
                                const int w0 = (int)((g * G) >> 5);
                                const int w1 = (int)((min((g + 1) * G, NK) + 31) >> 5);
                                bool any = false;
                                for (int w = w0; w < w1 && !any; ++w) any = dropped_word(w);
                                if (any) L.ops[n++] = op_make(OP_F, (int32_t)g);
                            }
                        }
                    }
                }
                L.nops = n;
                L.item = (int32_t)item;
                mbar_arrive(&ctl.list_full[bb]);   // the warp's writes precede it (__syncwarp)
            }
            __syncwarp();
        }
    } else if (warp == 0) {
        // ======================= Q tiles + K ring =======================
        if (lane == 0) {
            int g0 = 0;
            for (int j = 0;; ++j) {
                const int bb = j & 1;
                mbar_wait_sleep(&ctl.list_full[bb], (uint32_t)((j >> 1) & 1));
                const List& L = ctl.list[bb];
                if (L.nops < 0) break;
                const int64_t item = L.item;
                const int64_t i = item % p.NQ, bh = item / p.NQ;
                const int64_t b = bh / p.H, h = bh % p.H;
                // Q tile of item j into buffer j & 1 once item j-2 no longer reads it
                if (j >= 2) mbar_wait_sleep(&ctl.q_empty[bb], (uint32_t)(((j - 2) >> 1) & 1));
                mbar_arrive_expect_tx(&ctl.q_full[bb], kQBox);
                tma_load_4d(smem + kOffQ + bb * kQBox, &tmQ, &ctl.q_full[bb], 0, (int)(i * kBQ),
                            (int)h, (int)b);
                const int nops = L.nops;
                for (int n = 0; n < nops; ++n) {
                    const int g = g0 + n;
                    const int s = g & 1;
                    mbar_wait_sleep(&ctl.k_empty[s], (uint32_t)(((g >> 1) & 1) ^ 1));
                    uint8_t* dst = smem + kOffK + s * kSlot;
                    const int32_t op = L.ops[n];
                    const int v = op_val(op);
                    if (op_type(op) == OP_F) {
                        mbar_arrive_expect_tx(&ctl.k_full[s], kD * 128);
                        tma_load_3d(dst, &tmHt, &ctl.k_full[s], 0, v * kD, (int)bh);
                    } else {
                        mbar_arrive_expect_tx(&ctl.k_full[s], kSlot);
                        if (op_type(op) == OP_E)
                            tma_load_4d(dst, &tmK, &ctl.k_full[s], 0, v * kBK, (int)h, (int)b);
                        else
                            tma_load_3d(dst, &tmKb, &ctl.k_full[s], 0, v * 64, (int)bh);
                    }
                }
                g0 += nops;
                mbar_arrive(&ctl.list_empty[bb]);
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ======================= V ring =======================
        if (lane == 0) {
            int g0 = 0;
            for (int j = 0;; ++j) {
                const int bb = j & 1;
                mbar_wait_sleep(&ctl.list_full[bb], (uint32_t)((j >> 1) & 1));
                const List& L = ctl.list[bb];
                if (L.nops < 0) break;
                const int64_t item = L.item;
                const int64_t bh = item / p.NQ;
                const int64_t b = bh / p.H, h = bh % p.H;
                const int nops = L.nops;
                for (int n = 0; n < nops; ++n) {
                    const int g = g0 + n;
                    const int s = g & 1;
                    mbar_wait_sleep(&ctl.pv_done[s], (uint32_t)(((g >> 1) & 1) ^ 1));   // PV(g-2)
                    uint8_t* dst = smem + kOffV + s * kSlot;
                    const int32_t op = L.ops[n];
                    const int v = op_val(op);
                    uint64_t* vbar = &ctl.p_full[g & 1];
                    if (op_type(op) == OP_F) {
                        mbar_arrive(vbar);   // d = 64: Hbar^T fits the K slot alone
                    } else {
                        mbar_arrive_expect_tx(vbar, kSlot);
                        if (op_type(op) == OP_E)
                            tma_load_4d(dst, &tmV, vbar, 0, v * kBK, (int)h, (int)b);
                        else
                            tma_load_3d(dst, &tmVs, vbar, 0, v * 64, (int)bh);
                    }
                }
                g0 += nops;
                mbar_arrive(&ctl.list_empty[bb]);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer =======================
        constexpr uint32_t kIdQK = idesc_bf16_f32(128, kBK, 0, 0);   // Q (TMEM) x K^T
        constexpr uint32_t kIdPV = idesc_bf16_f32(128, kD, 0, 1);    // P (TMEM) x V (MN-major)
        constexpr uint32_t kIdF = idesc_bf16_f32(128, kD, 0, 0);     // Aq (TMEM) x Hbar^T
        const uint32_t k_base = smem_u32(smem + kOffK);
        const uint32_t v_base = smem_u32(smem + kOffV);
        const uint64_t dk0 = umma_desc_sw128(k_base, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(v_base, kSlot, 1024);
        auto issue_qk = [&](int g) {
            const int s = g & 1;
            mbar_wait_sleep(&ctl.k_full[s], (uint32_t)((g >> 1) & 1));
            tc_fence_after();
            const uint32_t d = tbase + kSCol + 64 * s;
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
                const uint32_t offk = (s * kSlot + kk * 32) >> 4;
                mma_ts_elect(d, tbase + kQCol + kk * 8, dk0 + offk, kIdQK, kk > 0);
            }
            mma_commit_elect(&ctl.s_full[s]);
            mma_commit_elect(&ctl.k_empty[s]);
            __syncwarp();
        };
        int g0 = 0;
        for (int j = 0;; ++j) {
            const int bb = j & 1;
            mbar_wait_sleep(&ctl.list_full[bb], (uint32_t)((j >> 1) & 1));
            const List& L = ctl.list[bb];
            const int nops = L.nops;
            if (nops < 0) break;
            mbar_wait_sleep(&ctl.q_tmem, (uint32_t)(j & 1));   // item j's Q in TMEM
            tc_fence_after();
            if (nops > 0 && op_type(L.ops[0]) != OP_F) issue_qk(g0);
            for (int n = 0; n < nops; ++n) {
                const int g = g0 + n;
                const int s = g & 1;
                if (n + 1 < nops && op_type(L.ops[n + 1]) != OP_F) issue_qk(g + 1);
                mbar_wait_sleep(&ctl.p_full[s], (uint32_t)((g >> 1) & 1));   // P ready + V
                if (n == 0 && j > 0) mbar_wait_sleep(&ctl.o_free, (uint32_t)((j - 1) & 1));
                tc_fence_after();
                const int32_t op = L.ops[n];
                if (op_type(op) != OP_F) {
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint32_t offv = (s * kSlot + kk * 16 * 128) >> 4;
                        mma_ts_elect(tbase, tbase + kSCol + 64 * s + kk * 8, dv0 + offv, kIdPV,
                                     (n > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit_elect(&ctl.pv_done[s]);
                } else {
                    mbar_wait_sleep(&ctl.k_full[s], (uint32_t)((g >> 1) & 1));   // Hbar^T
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < kD / 16; ++kk) {
                        const uint64_t bd = umma_desc_sw128(k_base + s * kSlot + kk * 32, 16, 1024);
                        mma_ts_elect(tbase, tbase + kSCol + 64 * s + kk * 8, bd, kIdF, 1u);
                    }
                    mma_commit_elect(&ctl.k_empty[s]);
                    mma_commit_elect(&ctl.pv_done[s]);
                }
                __syncwarp();
            }
            g0 += nops;
            if (lane == 0) mbar_arrive(&ctl.list_empty[bb]);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // =================== softmax / correction / epilogue ===================
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t t_o = tbase + lane_off;
        const int n_last = (int)NK - 1;
        const int nlast_len = (int)(p.S - (int64_t)n_last * 64);
        const float cs = p.scale_log2;
        const int G32 = (int)p.G, NK32 = (int)NK;
        int sc0 = 0, sc1 = 0;   // S-type ops seen per S buffer (s_full parity), all items
        auto consume_op = [&](int g) {   // the O-MMA of op g has completed
            if (g < 0) return;
            mbar_wait_sleep(&ctl.pv_done[g & 1], (uint32_t)((g >> 1) & 1));
        };
        // Q row r of item j's tile -> TMEM lane r, columns kQCol.. (bf16 pairs)
        auto q_to_tmem = [&](int j) {
            const int qb = (int)(j & 1);
            mbar_wait_sleep(&ctl.q_full[qb], (uint32_t)((j >> 1) & 1));
            const uint8_t* qrow = smem + kOffQ + qb * kQBox;
            uint32_t qa[32];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const uint4 u = *reinterpret_cast<const uint4*>(qrow + r * 128 + ((cc ^ (r & 7)) << 4));
                qa[cc * 4 + 0] = u.x; qa[cc * 4 + 1] = u.y; qa[cc * 4 + 2] = u.z;
                qa[cc * 4 + 3] = u.w;
            }
            tmem_st32(t_o + kQCol, qa);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&ctl.q_tmem);
        };
        mbar_wait_sleep(&ctl.list_full[0], 0);
        if (ctl.list[0].nops >= 0) q_to_tmem(0);
        int g0 = 0;
        for (int j = 0;; ++j) {
            const int bb = j & 1;
            mbar_wait_sleep(&ctl.list_full[bb], (uint32_t)((j >> 1) & 1));
            const List& L = ctl.list[bb];
            const int nops = L.nops;
            if (nops < 0) break;
            const int item = L.item;
            const int NQ32 = (int)p.NQ, H32 = (int)p.H;
            const int i = item % NQ32, bh = item / NQ32;
            const int b = bh / H32, h = bh % H32;
            const uint8_t* qrow = smem + kOffQ + bb * kQBox;
            float m = -INFINITY, l = 0.f;
            float A_cur = 0.f, A_done = 0.f;
            int g_cur = -1, g_done = -1;
            for (int n = 0; n < nops; ++n) {
                const int g = g0 + n;
                const int bi = g & 1;
                const int32_t op = L.ops[n];
                const int type = op_type(op), v = op_val(op);
                const uint32_t t_buf = tbase + lane_off + kSCol + 64 * bi;
                if (type != OP_F) {
                    const int par = (bi == 0 ? sc0++ : sc1++) & 1;
                    mbar_wait_sleep(&ctl.s_full[bi], (uint32_t)par);
                    tc_fence_after();
                    uint32_t sa[32], sb[32];
                    tmem_ld32(t_buf, sa);
                    tmem_ld32(t_buf + 32, sb);
                    tmem_wait_ld();
                    uint64_t valid;
                    float wlast = 1.f;
                    int clast = -1;
                    if (type == OP_E) {
                        const int nj = v == n_last ? nlast_len : 64;
                        valid = nj >= 64 ? ~0ull : ((1ull << nj) - 1ull);
                    } else {
                        const uint64_t kept = (uint64_t)L.mask[2 * v] |
                                              ((2 * v + 1 < p.W) ? (uint64_t)L.mask[2 * v + 1] << 32 : 0ull);
                        const int rem = NK32 - 64 * v;
                        const uint64_t inb = rem >= 64 ? ~0ull : ((1ull << rem) - 1ull);
                        valid = ~kept & inb;
                        if (rem <= 64) { clast = rem - 1; wlast = (float)nlast_len; }
                    }
                    if (valid != ~0ull) {
#pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            if (!((valid >> c) & 1ull)) sa[c] = 0xff800000u;
                            if (!((valid >> (c + 32)) & 1ull)) sb[c] = 0xff800000u;
                        }
                    }
                    float xlast = -INFINITY;
                    if (clast >= 0) {
#pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            if (c == clast) xlast = __uint_as_float(sa[c]);
                            if (c + 32 == clast) xlast = __uint_as_float(sb[c]);
                        }
                    }
                    // exponentials against the current m first; the exact max only when the
                    // row sum reaches 2^8 (attn_sm100.cu: the same m sequence, the same P)
                    float h0, h1;
                    uint32_t pk[32];
                    const float2 cs2 = make_float2(cs, cs);
                    auto exps = [&](float mref) {
                        const float2 nm2 = make_float2(-mref, -mref);
                        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            const float2 xa = ffma2(make_float2(__uint_as_float(sa[2 * c]),
                                                                __uint_as_float(sa[2 * c + 1])), cs2, nm2);
                            const float2 xb = ffma2(make_float2(__uint_as_float(sb[2 * c]),
                                                                __uint_as_float(sb[2 * c + 1])), cs2, nm2);
                            const float p0 = ex2(xa.x), p1 = ex2(xa.y), p2 = ex2(xb.x), p3 = ex2(xb.y);
                            a0 = fadd2(a0, make_float2(p0, p1));
                            a1 = fadd2(a1, make_float2(p2, p3));
                            pk[c] = pack_bf16(p0, p1);
                            pk[16 + c] = pack_bf16(p2, p3);
                        }
                        h0 = a0.x + a0.y;
                        h1 = a1.x + a1.y;
                    };
                    exps(m);
                    float corr = 1.f;
                    bool resc = false;
                    if (__any_sync(0xffffffffu, !(h0 + h1 < 256.f))) {
                        float mr0 = -INFINITY, mr1 = -INFINITY, mr2 = -INFINITY, mr3 = -INFINITY;
#pragma unroll
                        for (int c = 0; c < 16; c += 2) {
                            mr0 = fmax3(mr0, __uint_as_float(sa[c]), __uint_as_float(sa[c + 1]));
                            mr1 = fmax3(mr1, __uint_as_float(sb[c]), __uint_as_float(sb[c + 1]));
                            mr2 = fmax3(mr2, __uint_as_float(sa[c + 16]), __uint_as_float(sa[c + 17]));
                            mr3 = fmax3(mr3, __uint_as_float(sb[c + 16]), __uint_as_float(sb[c + 17]));
                        }
                        const float mx = fmaxf(fmax3(mr0, mr1, mr2), mr3) * cs;
                        const bool moved = mx > m + kRescaleThresh;
                        if (moved) {
                            corr = ex2(m - mx);
                            resc = n > 0;
                            m = mx;
                            l *= corr;
                            A_cur *= corr;
                        }
                        if (__any_sync(0xffffffffu, moved)) exps(m);
                    }
                    if (__any_sync(0xffffffffu, resc)) {
                        consume_op(g - 2);
                        consume_op(g - 1);
                        tc_fence_after();
                        uint32_t o[32];
                        tmem_ld32(t_o, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                        tmem_st32(t_o, o);
                        tmem_ld32(t_o + 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                        tmem_st32(t_o + 32, o);
                    }
                    const float negm = -m;
                    tmem_st32(t_buf, pk);
                    if (type == OP_E) {
                        l += h0 + h1;
                    } else {
                        const float pl = clast >= 0 ? ex2(fmaf(xlast, cs, negm)) : 0.f;
                        l += 64.f * (h0 + h1) - (64.f - wlast) * pl;
                        const int j0 = 64 * v;
                        const int gg0 = j0 / G32;
                        if (gg0 != g_cur) { A_cur = 0.f; g_cur = gg0; }
                        A_cur += h0;
                        if (j0 + 32 < NK32) {
                            const int gg1 = (j0 + 32) / G32;
                            if (gg1 != gg0) { A_done = A_cur; g_done = gg0; A_cur = h1; g_cur = gg1; }
                            else A_cur += h1;
                        }
                    }
                    tmem_wait_st();
                } else {
                    // F(g): Aq = bf16(s * A_{t,g} * q_t) into the S buffer (R-21); the buffer's
                    // previous reader was PV(g-2) (attn_sm100.cu explains why not g-1)
                    const float A = v == g_done ? A_done : A_cur;
                    const float w = p.s * A;
                    const uint32_t w2 = pack_bf16(w, w);
                    consume_op(g - 2);
                    tc_fence_after();
                    uint32_t aq[32];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 u = *reinterpret_cast<const uint4*>(qrow + r * 128 + ((c ^ (r & 7)) << 4));
                        aq[c * 4 + 0] = hmul2_bf16(u.x, w2);
                        aq[c * 4 + 1] = hmul2_bf16(u.y, w2);
                        aq[c * 4 + 2] = hmul2_bf16(u.z, w2);
                        aq[c * 4 + 3] = hmul2_bf16(u.w, w2);
                    }
                    tmem_st32(t_buf, aq);
                    tmem_wait_st();
                }
                tc_fence_before();
                mbar_arrive(&ctl.p_full[bi]);
            }
            // ---- transition: the next item's Q into TMEM (item j's last QK^T has completed:
            // its S was consumed above), so its first QK^T runs during this epilogue ----
            {
                const int nb = (j + 1) & 1;
                mbar_wait_sleep(&ctl.list_full[nb], (uint32_t)(((j + 1) >> 1) & 1));
                if (ctl.list[nb].nops >= 0) q_to_tmem(j + 1);
            }
            // ---- epilogue of item j: O / l -> bf16 -> global ----
            consume_op(g0 + nops - 2);
            consume_op(g0 + nops - 1);
            tc_fence_after();
            const int t = i * kBQ + r;
            const float inv = 1.f / l;
            __nv_bfloat16* orow = p.out + (int64_t)b * p.osB + (int64_t)h * p.osH + (int64_t)t * p.osS;
#pragma unroll 1
            for (int c0 = 0; c0 < kD; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(t_o + c0, o);
                tmem_wait_ld();
                if (t < p.S) {
                    uint4 pkt[4];
                    uint32_t* pw = reinterpret_cast<uint32_t*>(pkt);
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        pw[c] = pack_bf16(__uint_as_float(o[2 * c]) * inv, __uint_as_float(o[2 * c + 1]) * inv);
#pragma unroll
                    for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(orow + c0)[q] = pkt[q];
                }
            }
            tc_fence_before();
            mbar_arrive(&ctl.o_free);          // O read out: the next item's first PV may start
            mbar_arrive(&ctl.q_empty[bb]);     // this item's Q tile (F ops) no longer read
            mbar_arrive(&ctl.list_empty[bb]);
            g0 += nops;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, kTmemCols);
    }
}

}  // namespace

bool attn_sm100_persist_supported(const pasa_route_s* r) {
    return r->cfg.Bq == kBQ && r->cfg.Bk == kBK && r->D == kD && r->NK <= kMaxNK && !r->cfg.qk_fp8 &&
           (r->cfg.comp != PASA_COMP_GROUPED || r->cfg.G == 32 || r->cfg.G == 64 ||
            r->cfg.G % 128 == 0 || r->cfg.G >= r->NK);
}

cudaError_t launch_attn_sm100_persist(const pasa_tensor& q, const pasa_tensor& k,
                                      const pasa_tensor& v, pasa_route_s* r,
                                      const pasa_tensor& out, cudaStream_t st, int* launches,
                                      char* why, size_t why_len) {
    if (!attn_sm100_persist_supported(r)) {
        snprintf(why, why_len, "persistent kernel: Bq = 128, Bk = 64, d = 64, bf16, "
                 "G in {32, 64, multiples of 128, >= N_K}");
        return cudaErrorNotSupported;
    }
    CUtensorMap mQ, mK, mV, mKb, mVs, mHt;
    auto act = [&](CUtensorMap* m, const pasa_tensor& t, uint32_t rows) {
        uint64_t dims[4] = {(uint64_t)t.D, (uint64_t)t.S, (uint64_t)t.H, (uint64_t)t.B};
        uint64_t str[3] = {(uint64_t)t.sS * 2, (uint64_t)t.sH * 2, (uint64_t)t.sB * 2};
        uint32_t box[4] = {64, rows, 1, 1};
        return make_tensor_map(m, t.data, 4, dims, str, box, why, why_len);
    };
    if (!act(&mQ, q, kBQ) || !act(&mK, k, kBK) || !act(&mV, v, kBK)) return cudaErrorNotSupported;
    {
        uint64_t dims[3] = {(uint64_t)kD, (uint64_t)r->NK, (uint64_t)r->BH};
        uint64_t str[2] = {(uint64_t)kD * 2, (uint64_t)r->NK * kD * 2};
        uint32_t box[3] = {64, 64, 1};
        if (!make_tensor_map(&mKb, r->kbar_lp, 3, dims, str, box, why, why_len) ||
            !make_tensor_map(&mVs, r->vsum_lp, 3, dims, str, box, why, why_len))
            return cudaErrorNotSupported;
    }
    {
        uint64_t dims[3] = {(uint64_t)kD, (uint64_t)r->NG * kD, (uint64_t)r->BH};
        uint64_t str[2] = {(uint64_t)kD * 2, (uint64_t)r->NG * kD * kD * 2};
        uint32_t box[3] = {64, (uint32_t)kD, 1};
        if (!make_tensor_map(&mHt, r->ht, 3, dims, str, box, why, why_len)) return cudaErrorNotSupported;
    }
    Params prm;
    prm.S = r->S; prm.H = r->H; prm.NQ = r->NQ; prm.NK = r->NK; prm.W = r->W;
    prm.it0 = r->it0; prm.it1 = r->it1;
    prm.G = (int32_t)(r->cfg.G < r->NK ? r->cfg.G : r->NK);   // one global group: G = N_K
    prm.comp = r->cfg.comp;
    const double s = 1.0 / sqrt((double)kD);
    prm.s = (float)s;
    prm.scale_log2 = (float)(s * 1.4426950408889634);
    prm.idx = r->idx; prm.count = r->count; prm.mask = r->mask;
    prm.out = reinterpret_cast<__nv_bfloat16*>(out.data);
    prm.osB = out.sB; prm.osS = out.sS; prm.osH = out.sH;
    prm.counter = r->hdr + 1;   // a free word of the route header
    cudaError_t ez = cudaMemsetAsync(prm.counter, 0, sizeof(int32_t), st);
    if (ez != cudaSuccess) return ez;
    // 80 KB of dynamic shared memory (+ ~19 KB static): two CTAs per SM, never three
    const size_t smem = 80 * 1024;
    static_assert(kBytes + 1024 <= 80 * 1024, "shared memory budget");
    cudaError_t e = cudaFuncSetAttribute(attn_sm100_persist_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = r->it1 - r->it0;
    const unsigned grid = (unsigned)(items < 2LL * sms ? items : 2LL * sms);
    if (grid == 0) return cudaSuccess;
    attn_sm100_persist_kernel<<<grid, kThreads, smem, st>>>(mQ, mK, mV, mKb, mVs, mHt, prm);
    e = cudaGetLastError();
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace pasa
