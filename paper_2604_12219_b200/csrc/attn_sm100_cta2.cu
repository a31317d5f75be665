// attn_sm100_cta2.cu -- pasa_attn for 256-row query blocks (Bq = 256, reading R-29) on a
// CTA PAIR: tcgen05 cta_group::2, M = 256 ("cta_group::2 M = 256
// pairs sharing K/V tiles").  Same method and op list as attn_sm100.cu (Eq. 7,
// PAPER.md:216-228; grouped first-order term, App. B :503-506;
// readings R-1..R-5, R-21, R-22); what changes is where the operands live.
//
// A cluster of two CTAs on the two SMs of a TPC owns one (head, 256-row q-block) item:
// CTA c (cluster rank c) holds query rows 128 c .. 128 c + 127 in its shared memory, its
// own O accumulator and S/P buffers in its own TMEM, and runs the softmax of its rows.
// The leader (rank 0) issues every MMA as one M = 256 tcgen05.mma.cta_group::2: A (Q, or
// P / Aq from TMEM) and D come from each CTA's own rows, and the B operand's N rows are
// split between the two shared memories, so each SM brings HALF of every operand tile an
// op needs from L2:
//   QK^T   B = K_j  [64 keys x 128 d]  -> CTA c holds keys 32 c .. 32 c + 31 (8 KB)
//   PV     B = V_j  [64 keys x 128 d]  -> CTA c holds dims 64 c .. 64 c + 63  (8 KB)
//   C op   Kbar / Vsum chunks, split the same way
//   F op   B = Hbar^(g)T [128 x 128]   -> CTA c holds output dims 64 c .. (2 x 8 KB)
// against 32 KB per op per SM in attn_sm100.cu, with the QK^T shared-memory reads per
// MMA down from 6 KB to 5 KB per SM.  Two pair-CTAs per SM (TMEM 2 x 256 columns, ~81 KB
// of shared memory each), like the Bq = 128 kernel.
//
// Synchronisation (barriers at the same offset in both CTAs; "leader" = only the leader's
// copy is used):
//   q_full   leader: its own Q tile (expect_tx) + the peer's relay arrival   (count 2)
//   q_local  peer: its own Q tile (the peer's softmax reads Q rows for F ops)
//   k_full / v_full [slot]  leader: expect_tx of BOTH halves by the leader's producers;
//            each CTA's TMA (cp.async.bulk.tensor.cta_group::2) completes its bytes there
//   k_empty / s_full / pv_done  both: tcgen05.commit multicast to the two CTAs
//   p_full [S buffer]  leader: one arrival per softmax warp of both CTAs    (count 8)
// Domain: bf16, Bq = 256, Bk = 64, d = 128, G in {32, 64, multiples of 128, >= N_K} or no
// grouped term.  Selected with PASA_ATTN_CTA_PAIR (include/pasa.h).
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
constexpr int kBQ = 256, kBK = 64, kTile = 128, kD = 128;
constexpr int kMaxNK = 4096;
constexpr int kMaxOps = kMaxNK + kMaxNK / 64 + kMaxNK / 8 + 64;
constexpr int kTmemCols = 256;
constexpr uint32_t kSCol = 128;            // S buffer b at column 128 + 64 b (O at 0..127)
constexpr float kRescaleThresh = 8.f;      // log2 units
constexpr int kQBox = kTile * 128;         // 16 KB: one 64-column box of this CTA's Q rows
constexpr int kHalf = 8192;                // bytes of one CTA's half of an operand slot
constexpr int kKBox = 32 * 128;            // 4 KB: one 64-column box of a 32-row K half
constexpr int kOffQ = 0;
constexpr int kOffK = 2 * kQBox;           // two K slots
constexpr int kOffV = kOffK + 2 * kHalf;   // two V slots
constexpr int kBytes = kOffV + 2 * kHalf;  // 64 KB

enum : int32_t { OP_E = 0, OP_C = 1, OP_F = 2 };
__device__ __forceinline__ uint16_t op_make(int32_t type, int32_t v) {
    return (uint16_t)((type << 14) | v);
}
__device__ __forceinline__ int32_t op_type(int32_t op) { return op >> 14; }
__device__ __forceinline__ int32_t op_val(int32_t op) { return op & 0x3FFF; }

struct Params {
    int32_t S, H, NQ, NK, W, G, comp;
    int32_t it0;
    float scale_log2;   // s * log2(e)
    float s;            // 1/sqrt(D)
    const int32_t* idx;
    const int32_t* count;
    const uint32_t* mask;
    __nv_bfloat16* out;
    int64_t osB, osS, osH;
};

struct Ctl {
    uint64_t q_full, q_local;
    uint64_t k_full[2], v_full[2];
    uint64_t k_empty[2], s_full[2], pv_done[2];
    uint64_t p_full[2];
    uint32_t tmem_base;
    int32_t nops;
    uint32_t mask[kMaxNK / 32];
    uint16_t ops[kMaxOps];
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 2)
    attn_sm100_cta2_kernel(const __grid_constant__ CUtensorMap tmQ,
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
    const int c = (int)cluster_rank();           // 0 = leader
    const bool leader = c == 0;
    const int item = p.it0 + (int)(blockIdx.x >> 1);
    const int i = item % p.NQ, bh = item / p.NQ;
    const int b = bh / p.H, h = bh % p.H;
    const int64_t row = (int64_t)bh * p.NQ + i;
    const int32_t cnt = p.count[row];
    const int NK = p.NK;
    const int nchunks = (NK + 63) / 64;

    // ---------------- setup: op list, mask row, barriers, TMEM (both CTAs) ----------------
    for (int w = tid; w < p.W; w += blockDim.x) ctl.mask[w] = p.mask[row * p.W + w];
    for (int q = tid; q < cnt; q += blockDim.x) ctl.ops[q] = op_make(OP_E, p.idx[row * (int64_t)NK + q]);
    if (tid == 0) {
        mbar_init(&ctl.q_full, 2);
        mbar_init(&ctl.q_local, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&ctl.k_full[s], 1);
            mbar_init(&ctl.v_full[s], 1);
            mbar_init(&ctl.k_empty[s], 1);
            mbar_init(&ctl.s_full[s], 1);
            mbar_init(&ctl.pv_done[s], 1);
            mbar_init(&ctl.p_full[s], 8);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc_pair(&ctl.tmem_base, kTmemCols);
        tmem_relinquish_pair();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
        tma_prefetch(&tmKb); tma_prefetch(&tmVs); tma_prefetch(&tmHt);
    }
    __syncthreads();
    if (tid == 0) {
        // tail of the op list (as attn_sm100.cu): centroid chunks with a dropped block,
        // then the first-order op of every group that ends inside the chunk
        int n = cnt;
        if (p.comp != PASA_COMP_NONE && cnt < NK) {
            const int W = p.W;
            auto dropped_word = [&](int w) {
                const int rem = NK - 32 * w;
                const uint32_t inb = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
                return (~ctl.mask[w] & inb) != 0u;
            };
            const int G = p.G;
            int g = 0;
            for (int cc = 0; cc < nchunks; ++cc) {
                if (dropped_word(2 * cc) || (2 * cc + 1 < W && dropped_word(2 * cc + 1)))
                    ctl.ops[n++] = op_make(OP_C, cc);
                if (p.comp == PASA_COMP_GROUPED) {
                    const int chunk_end = min(64 * (cc + 1), NK);
                    for (; (int64_t)g * G < NK && (int)min((int64_t)(g + 1) * G, (int64_t)NK) <= chunk_end; ++g) {
                        const int w0 = (int)(((int64_t)g * G) >> 5);
                        const int w1 = (int)((min((int64_t)(g + 1) * G, (int64_t)NK) + 31) >> 5);
                        bool any = false;
                        for (int w = w0; w < w1 && !any; ++w) any = dropped_word(w);
                        if (any) ctl.ops[n++] = op_make(OP_F, g);
                    }
                }
            }
        }
        ctl.nops = n;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();   // both CTAs' barriers initialised and TMEM allocated before any remote use
    tc_fence_after();
    const int nops = ctl.nops;
    const uint32_t tbase = ctl.tmem_base;

    if (warp == 0) {
        // ============ K-ring producer (each CTA loads its half; leader expects both) ============
        if (lane == 0) {
            if (leader) {
                mbar_arrive_expect_tx(&ctl.q_full, kTile * kD * 2);
#pragma unroll
                for (int a = 0; a < 2; ++a)
                    tma_load_4d(smem + kOffQ + a * kQBox, &tmQ, &ctl.q_full, 64 * a, i * kBQ, h, b);
            } else {
                mbar_arrive_expect_tx(&ctl.q_local, kTile * kD * 2);
#pragma unroll
                for (int a = 0; a < 2; ++a)
                    tma_load_4d(smem + kOffQ + a * kQBox, &tmQ, &ctl.q_local, 64 * a, i * kBQ + kTile,
                                h, b);
                // relay "the peer's Q landed" to the leader's q_full (before any K load: the
                // leader's first QK^T waits for it)
                mbar_wait_sleep(&ctl.q_local, 0);
                mbar_arrive_cluster_release(mapa_leader(&ctl.q_full));
            }
            const uint32_t kfull0 = mapa_leader(&ctl.k_full[0]);
            const uint32_t kfull1 = mapa_leader(&ctl.k_full[1]);
            for (int n = 0; n < nops; ++n) {
                const int s = n & 1;
                mbar_wait_sleep(&ctl.k_empty[s], ((n >> 1) & 1) ^ 1);
                uint8_t* dst = smem + kOffK + s * kHalf;
                const uint32_t bar = s ? kfull1 : kfull0;
                const int32_t op = ctl.ops[n];
                const int v = op_val(op);
                if (leader) mbar_arrive_expect_tx(&ctl.k_full[s], 2 * kHalf);
                if (op_type(op) == OP_F) {   // Hbar^T rows (output dims) 64 c .., columns 0-63
                    tma_load_3d_pair(dst, &tmHt, bar, 0, v * kD + 64 * c, bh);
                } else {
#pragma unroll
                    for (int a = 0; a < 2; ++a) {
                        if (op_type(op) == OP_E)
                            tma_load_4d_pair(dst + a * kKBox, &tmK, bar, 64 * a, v * kBK + 32 * c, h, b);
                        else
                            tma_load_3d_pair(dst + a * kKBox, &tmKb, bar, 64 * a, v * 64 + 32 * c, bh);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ======================= V-ring producer =======================
        if (lane == 0) {
            const uint32_t vfull0 = mapa_leader(&ctl.v_full[0]);
            const uint32_t vfull1 = mapa_leader(&ctl.v_full[1]);
            for (int n = 0; n < nops; ++n) {
                const int s = n & 1;
                mbar_wait_sleep(&ctl.pv_done[s], ((n >> 1) & 1) ^ 1);   // op n-2 read the slot
                uint8_t* dst = smem + kOffV + s * kHalf;
                const uint32_t bar = s ? vfull1 : vfull0;
                const int32_t op = ctl.ops[n];
                const int v = op_val(op);
                if (leader) mbar_arrive_expect_tx(&ctl.v_full[s], 2 * kHalf);
                if (op_type(op) == OP_F)        // Hbar^T rows 64 c .., columns 64-127
                    tma_load_3d_pair(dst, &tmHt, bar, 64, v * kD + 64 * c, bh);
                else if (op_type(op) == OP_E)   // V_j dims 64 c ..
                    tma_load_4d_pair(dst, &tmV, bar, 64 * c, v * kBK, h, b);
                else
                    tma_load_3d_pair(dst, &tmVs, bar, 64 * c, v * 64, bh);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer (leader only) =======================
        if (leader) {
            constexpr uint32_t kIdQK = idesc_bf16_f32(256, kBK, 0, 0);   // Q x K^T, both K-major
            constexpr uint32_t kIdPV = idesc_bf16_f32(256, kD, 0, 1);    // P (TMEM) x V (MN-major)
            constexpr uint32_t kIdF = idesc_bf16_f32(256, kD, 0, 0);     // Aq (TMEM) x Hbar^T
            const uint32_t q_base = smem_u32(smem + kOffQ);
            const uint32_t k_base = smem_u32(smem + kOffK);
            const uint32_t v_base = smem_u32(smem + kOffV);
            const uint64_t dq0 = umma_desc_sw128(q_base, 16, 1024);
            const uint64_t dk0 = umma_desc_sw128(k_base, 16, 1024);
            const uint64_t dv0 = umma_desc_sw128(v_base, kHalf, 1024);
            auto issue_qk = [&](int n) {
                const int s = n & 1;
                mbar_wait_cluster(&ctl.k_full[s], (n >> 1) & 1);
                tc_fence_after();
                const uint32_t d = tbase + kSCol + 64 * s;
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint32_t offq = ((kk >> 2) * kQBox + (kk & 3) * 32) >> 4;
                    const uint32_t offk = (s * kHalf + (kk >> 2) * kKBox + (kk & 3) * 32) >> 4;
                    mma_ss_pair_elect(d, dq0 + offq, dk0 + offk, kIdQK, kk > 0);
                }
                mma_commit_pair_elect(&ctl.s_full[s]);
                mma_commit_pair_elect(&ctl.k_empty[s]);
                __syncwarp();
            };
            mbar_wait_cluster(&ctl.q_full, 0);
            tc_fence_after();
            if (nops > 0 && op_type(ctl.ops[0]) != OP_F) issue_qk(0);
            for (int n = 0; n < nops; ++n) {
                const int s = n & 1;
                if (n + 1 < nops && op_type(ctl.ops[n + 1]) != OP_F) issue_qk(n + 1);
                mbar_wait_cluster(&ctl.p_full[s], (n >> 1) & 1);
                mbar_wait_cluster(&ctl.v_full[s], (n >> 1) & 1);
                tc_fence_after();
                const int32_t op = ctl.ops[n];
                if (op_type(op) != OP_F) {
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint32_t offv = (s * kHalf + kk * 16 * 128) >> 4;
                        mma_ts_pair_elect(tbase, tbase + kSCol + 64 * s + kk * 8, dv0 + offv, kIdPV,
                                          (n > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit_pair_elect(&ctl.pv_done[s]);
                } else {
                    mbar_wait_cluster(&ctl.k_full[s], (n >> 1) & 1);   // Hbar^T columns 0-63
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < kD / 16; ++kk) {
                        const uint32_t box = (kk >> 2) == 0 ? k_base + s * kHalf : v_base + s * kHalf;
                        const uint64_t bd = umma_desc_sw128(box + (kk & 3) * 32, 16, 1024);
                        mma_ts_pair_elect(tbase, tbase + kSCol + 64 * s + kk * 8, bd, kIdF, 1u);
                    }
                    mma_commit_pair_elect(&ctl.k_empty[s]);
                    mma_commit_pair_elect(&ctl.pv_done[s]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // =========== softmax / correction / epilogue of this CTA's 128 rows ===========
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t t_o = tbase + lane_off;
        const uint8_t* qrow = smem + kOffQ;
        const uint32_t pfull_l0 = mapa_leader(&ctl.p_full[0]);
        const uint32_t pfull_l1 = mapa_leader(&ctl.p_full[1]);
        float m = -INFINITY, l = 0.f;
        float A_cur = 0.f, A_done = 0.f;
        int g_cur = -1, g_done = -1;
        int sc0 = 0, sc1 = 0;
        const int n_last = NK - 1;
        const int nlast_len = p.S - n_last * 64;
        const float cs = p.scale_log2;
        auto consume_op = [&](int op) {
            if (op < 0) return;
            mbar_wait_sleep(&ctl.pv_done[op & 1], (op >> 1) & 1);
        };
        bool q_seen = false;   // F ops read this CTA's Q rows from shared memory
        for (int n = 0; n < nops; ++n) {
            const int s = n & 1;
            const int32_t op = ctl.ops[n];
            const int type = op_type(op), v = op_val(op);
            const uint32_t t_buf = t_o + kSCol + 64 * s;
            if (type != OP_F) {
                mbar_wait_sleep(&ctl.s_full[s], (s ? sc1++ : sc0++) & 1);
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
                    const uint64_t kept = (uint64_t)ctl.mask[2 * v] |
                                          ((2 * v + 1 < p.W) ? (uint64_t)ctl.mask[2 * v + 1] << 32 : 0ull);
                    const int rem = NK - 64 * v;
                    const uint64_t inb = rem >= 64 ? ~0ull : ((1ull << rem) - 1ull);
                    valid = ~kept & inb;
                    if (rem <= 64) { clast = rem - 1; wlast = (float)nlast_len; }
                }
                if (valid != ~0ull) {
#pragma unroll
                    for (int cc = 0; cc < 32; ++cc) {
                        if (!((valid >> cc) & 1ull)) sa[cc] = 0xff800000u;
                        if (!((valid >> (cc + 32)) & 1ull)) sb[cc] = 0xff800000u;
                    }
                }
                float xlast = -INFINITY;
                if (clast >= 0) {
#pragma unroll
                    for (int cc = 0; cc < 32; ++cc) {
                        if (cc == clast) xlast = __uint_as_float(sa[cc]);
                        if (cc + 32 == clast) xlast = __uint_as_float(sb[cc]);
                    }
                }
                // exponentials against the current m first; the exact row max only when the
                // row sum reaches 2^8 (attn_sm100.cu: the same m sequence, so the same P)
                float h0, h1;
                uint32_t pk[32];
                const float2 cs2 = make_float2(cs, cs);
                auto exps = [&](float mref) {
                    const float2 nm2 = make_float2(-mref, -mref);
                    float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int cc = 0; cc < 16; ++cc) {
                        const float2 xa = ffma2(make_float2(__uint_as_float(sa[2 * cc]),
                                                            __uint_as_float(sa[2 * cc + 1])), cs2, nm2);
                        const float2 xb = ffma2(make_float2(__uint_as_float(sb[2 * cc]),
                                                            __uint_as_float(sb[2 * cc + 1])), cs2, nm2);
                        const float p0 = ex2(xa.x), p1 = ex2(xa.y), p2 = ex2(xb.x), p3 = ex2(xb.y);
                        a0 = fadd2(a0, make_float2(p0, p1));
                        a1 = fadd2(a1, make_float2(p2, p3));
                        pk[cc] = pack_bf16(p0, p1);
                        pk[16 + cc] = pack_bf16(p2, p3);
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
                    for (int cc = 0; cc < 16; cc += 2) {
                        mr0 = fmax3(mr0, __uint_as_float(sa[cc]), __uint_as_float(sa[cc + 1]));
                        mr1 = fmax3(mr1, __uint_as_float(sb[cc]), __uint_as_float(sb[cc + 1]));
                        mr2 = fmax3(mr2, __uint_as_float(sa[cc + 16]), __uint_as_float(sa[cc + 17]));
                        mr3 = fmax3(mr3, __uint_as_float(sb[cc + 16]), __uint_as_float(sb[cc + 17]));
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
                    consume_op(n - 2);
                    consume_op(n - 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c0 = 0; c0 < kD; c0 += 32) {
                        uint32_t o[32];
                        tmem_ld32(t_o + c0, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int cc = 0; cc < 32; ++cc) o[cc] = __float_as_uint(__uint_as_float(o[cc]) * corr);
                        tmem_st32(t_o + c0, o);
                    }
                }
                const float negm = -m;
                tmem_st32(t_buf, pk);
                if (type == OP_E) {
                    l += h0 + h1;
                } else {
                    // denominator: n_j * p_j; every dropped block has 64 tokens except the last
                    const float pl = clast >= 0 ? ex2(fmaf(xlast, cs, negm)) : 0.f;
                    l += 64.f * (h0 + h1) - (64.f - wlast) * pl;
                    const int j0 = 64 * v;
                    const int g0 = j0 / p.G;
                    if (g0 != g_cur) { A_cur = 0.f; g_cur = g0; }
                    A_cur += h0;
                    if (j0 + 32 < NK) {
                        const int g1 = (j0 + 32) / p.G;
                        if (g1 != g0) { A_done = A_cur; g_done = g0; A_cur = h1; g_cur = g1; }
                        else A_cur += h1;
                    }
                }
                tmem_wait_st();
            } else {
                // F(g): Aq = bf16(s * A_{t,g} * q_t) into the S buffer (R-21)
                if (!q_seen) {
                    mbar_wait_sleep(leader ? &ctl.q_full : &ctl.q_local, 0);
                    q_seen = true;
                }
                const float A = v == g_done ? A_done : A_cur;
                const float w = p.s * A;
                const uint32_t w2 = pack_bf16(w, w);
                consume_op(n - 2);   // the buffer's previous reader (attn_sm100.cu)
                tc_fence_after();
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    uint32_t aq[32];
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const uint4 u = *reinterpret_cast<const uint4*>(
                            qrow + a * kQBox + r * 128 + ((cc ^ (r & 7)) << 4));
                        aq[cc * 4 + 0] = hmul2_bf16(u.x, w2);
                        aq[cc * 4 + 1] = hmul2_bf16(u.y, w2);
                        aq[cc * 4 + 2] = hmul2_bf16(u.z, w2);
                        aq[cc * 4 + 3] = hmul2_bf16(u.w, w2);
                    }
                    tmem_st32(t_buf + 32 * a, aq);
                }
                tmem_wait_st();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&ctl.p_full[s]);
                else mbar_arrive_cluster(s ? pfull_l1 : pfull_l0);
            }
        }
        // ---- epilogue: O / l -> bf16 -> global ----
        consume_op(nops - 2);
        consume_op(nops - 1);
        tc_fence_after();
        const int tok = i * kBQ + c * kTile + r;
        const float inv = 1.f / l;
        __nv_bfloat16* orow = p.out + (int64_t)b * p.osB + (int64_t)h * p.osH + (int64_t)tok * p.osS;
#pragma unroll 1
        for (int c0 = 0; c0 < kD; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(t_o + c0, o);
            tmem_wait_ld();
            if (tok < p.S) {
                uint4 pkt[4];
                uint32_t* pw = reinterpret_cast<uint32_t*>(pkt);
#pragma unroll
                for (int cc = 0; cc < 16; ++cc)
                    pw[cc] = pack_bf16(__uint_as_float(o[2 * cc]) * inv, __uint_as_float(o[2 * cc + 1]) * inv);
#pragma unroll
                for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(orow + c0)[q] = pkt[q];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();   // no CTA leaves while its partner may still signal its barriers
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tbase, kTmemCols);
    }
}

}  // namespace

bool attn_sm100_cta2_supported(const pasa_route_s* r) {
    return r->cfg.Bq == kBQ && r->cfg.Bk == kBK && r->D == kD && r->NK <= kMaxNK &&
           (r->cfg.comp != PASA_COMP_GROUPED || r->cfg.G == 32 || r->cfg.G == 64 ||
            r->cfg.G % 128 == 0 || r->cfg.G >= r->NK);
}

cudaError_t launch_attn_sm100_cta2(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                                   pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                                   int* launches, char* why, size_t why_len) {
    if (!attn_sm100_cta2_supported(r)) {
        snprintf(why, why_len, "CTA-pair kernel: needs Bq=256, Bk=64, d=128, N_K <= 4096, "
                 "G in {32, 64, multiples of 128, >= N_K} for grouped compensation");
        return cudaErrorNotSupported;
    }
    CUtensorMap mQ, mK, mV, mKb, mVs, mHt;
    auto act = [&](CUtensorMap* m, const pasa_tensor& t, uint32_t rows) {
        uint64_t dims[4] = {(uint64_t)t.D, (uint64_t)t.S, (uint64_t)t.H, (uint64_t)t.B};
        uint64_t str[3] = {(uint64_t)t.sS * 2, (uint64_t)t.sH * 2, (uint64_t)t.sB * 2};
        uint32_t box[4] = {64, rows, 1, 1};
        return make_tensor_map(m, t.data, 4, dims, str, box, why, why_len);
    };
    // Q: this CTA's 128 rows; K: a 32-key half; V: all 64 keys of a 64-dim half
    if (!act(&mQ, q, kTile) || !act(&mK, k, 32) || !act(&mV, v, kBK)) return cudaErrorNotSupported;
    {
        uint64_t dims[3] = {(uint64_t)kD, (uint64_t)r->NK, (uint64_t)r->BH};
        uint64_t str[2] = {(uint64_t)kD * 2, (uint64_t)r->NK * kD * 2};
        uint32_t boxk[3] = {64, 32, 1}, boxv[3] = {64, 64, 1};
        if (!make_tensor_map(&mKb, r->kbar_lp, 3, dims, str, boxk, why, why_len) ||
            !make_tensor_map(&mVs, r->vsum_lp, 3, dims, str, boxv, why, why_len))
            return cudaErrorNotSupported;
    }
    {
        uint64_t dims[3] = {(uint64_t)kD, (uint64_t)r->NG * kD, (uint64_t)r->BH};
        uint64_t str[2] = {(uint64_t)kD * 2, (uint64_t)r->NG * kD * kD * 2};
        uint32_t box[3] = {64, 64, 1};
        if (!make_tensor_map(&mHt, r->ht, 3, dims, str, box, why, why_len)) return cudaErrorNotSupported;
    }
    Params prm;
    prm.S = (int32_t)r->S; prm.H = (int32_t)r->H; prm.NQ = (int32_t)r->NQ; prm.NK = (int32_t)r->NK;
    prm.W = (int32_t)r->W;
    prm.G = (int32_t)(r->cfg.G < r->NK ? r->cfg.G : r->NK);   // one global group: G = N_K
    prm.comp = r->cfg.comp;
    const double s = 1.0 / sqrt((double)kD);
    prm.s = (float)s;
    prm.scale_log2 = (float)(s * 1.4426950408889634);
    prm.idx = r->idx; prm.count = r->count; prm.mask = r->mask;
    prm.out = reinterpret_cast<__nv_bfloat16*>(out.data);
    prm.osB = out.sB; prm.osS = out.sS; prm.osH = out.sH;
    prm.it0 = (int32_t)r->it0;
    // >= 80 KB so at most two CTAs share an SM (2 x 256 TMEM columns)
    size_t smem = (size_t)kBytes + 1024;
    if (smem < 80 * 1024) smem = 80 * 1024;
    cudaError_t e = cudaFuncSetAttribute(attn_sm100_cta2_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = 2u * (unsigned)(r->it1 - r->it0);   // one CTA pair per item
    if (grid == 0) return cudaSuccess;
    attn_sm100_cta2_kernel<<<grid, kThreads, smem, st>>>(mQ, mK, mV, mKb, mVs, mHt, prm);
    e = cudaGetLastError();
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace pasa
