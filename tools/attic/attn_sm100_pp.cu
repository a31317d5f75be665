// attn_sm100_pp.cu -- pasa_attn on the tcgen05 tensor cores, one CTA per SM with
// two softmax warpgroups that take alternate ops ("ping-pong").  Same method and
// op list as attn_sm100.cu (Eq. 7; grouped first-order term,
// PAPER.md:310-313, App. B :503-506; readings R-1..R-5, R-21, R-22).
//
// Why this shape: the 2-CTA/SM kernel reads Q from shared memory
// for every QK^T (SS MMA: 48 KB of operand reads per 64-key op at d = 128) while
// TMA writes the next K and V tiles (32 KB) into the same shared memory; with PV's
// 16 KB that is 96 KB per op through one 128 B/clk port, more than the tensor
// math needs.  Here Q sits in TMEM and QK^T is a TS MMA (only the 16 KB K tile is
// read from shared memory), which needs 64 TMEM columns more than the 2-CTA layout
// has.  So one CTA owns the SM's 512 columns: O (D) + Q (D/2) + four S/P buffers
// of 64.  Op n uses buffer / K slot / V slot n % 4 and is worked on by softmax
// warpgroup n % 2, so each warpgroup has the S of its next op computed while it
// works on the current one, and QK(n+4) is issued right after PV(n).
// Measured (PASA_ATTN_PINGPONG, parity-tested): slower than the default kernel
// (25.3 vs 22.6 ms at Wan-14B, 1.45 vs 1.18 ms at CogVideoX): the Wan-14B launch
// runs at the board power limit and this layout spends more energy per launch
// (profiles/r01_attn_power.md).
//
// What the two warpgroups share, and how:
//   * the running max m.  It is the same sequential rule as the single-warpgroup
//     kernel (m_n = mx_n if mx_n > m_{n-1} + 8 else m_{n-1}), passed along the op
//     sequence per row: op n reads m_{n-1} from ctl.mchain[row] after a named
//     barrier the other warpgroup arrives on right after its own decision (early
//     in its op), and publishes m_n the same way.  The barrier phases alternate
//     strictly, because op n+1 cannot decide before op n has.
//   * O.  PVs accumulate in op order (one MMA issuer); when op n moves m, its
//     warpgroup waits for PV(n-1) and PV(n-2) and rescales O before it releases
//     P(n), so PV(n) and every later PV see the new reference.
//   * l.  Each warpgroup sums its own ops' denominators against the reference it
//     last saw and rescales its partial when the reference moves; the two partials
//     are added in the epilogue.
//   * the first-order weights A_{t,g}.  For G = 32 or 64 each group lies inside one
//     64-block centroid chunk, so A_{t,g} comes from exactly one C op, published per
//     row in ctl.cpub; an F op on the other warpgroup waits for it on a named
//     barrier (an F op never moves m, so no rescale is needed in between).
// Warp roles (384 threads): warp 0 K-ring TMA producer, warp 1 TMEM allocator +
// MMA issuer, warp 2 V-ring TMA producer, warp 3 idle; warps 4-7 softmax
// warpgroup 0 (even ops), warps 8-11 softmax warpgroup 1 (odd ops); both copy
// their rows of Q from shared memory into TMEM before the first QK^T.
// Domain: bf16, Bq = 128, Bk = 64, d = 64 or 128, compensation NONE / ZEROTH /
// GROUPED with G = 32 or 64 (other G: attn_sm100.cu).
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

constexpr int kThreads = 384;
constexpr int kBQ = 128, kBK = 64;
constexpr int kMaxOps = 2048 + 32 + 64 + 64;
constexpr int kTmemCols = 512;
constexpr float kRescaleThresh = 8.f;   // log2 units
// named barriers (0 = __syncthreads)
constexpr uint32_t kBarEpi = 1;      // epilogue: the two l partials
constexpr uint32_t kBarChain = 2;    // + w: warpgroup w published m for its latest op
constexpr uint32_t kBarCpub = 4;     // a C op's group sums are in ctl.cpub

// ops are 16 bit: type in bits 14-15, block / chunk / group in bits 0-13
enum : uint32_t { OP_E = 0, OP_C = 1, OP_F = 2 };
__device__ __forceinline__ uint16_t op_make(uint32_t type, uint32_t v) {
    return (uint16_t)((type << 14) | v);
}
__device__ __forceinline__ uint32_t op_type(uint32_t op) { return op >> 14; }
__device__ __forceinline__ uint32_t op_val(uint32_t op) { return op & 0x3FFFu; }

constexpr int NS = 4;   // S/P buffers in TMEM = K slots = V slots; op n uses buffer n % NS

template <int D>
struct Geo {
    // TMEM columns: O [0, D), Q [D, D + D/2) (bf16 pairs), S/P buffer b at SCOL + 64 b
    static constexpr uint32_t QCOL = D;
    static constexpr uint32_t SCOL = D + 64;
    static_assert(SCOL + 64 * NS <= 512, "TMEM budget");
    static constexpr int NBOX = D / 64;
    static constexpr int QBOX = kBQ * 128;          // bytes per 64-col box of Q
    static constexpr int KVBOX = kBK * 128;         // bytes per 64-col box of a K/V tile
    static constexpr int SLOT = kBK * D * 2;        // bytes per K or V slot
    static constexpr int HTBOX = D * 128;           // bytes per 64-col box of Hbar^T
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = kBQ * D * 2;
    static constexpr int OFF_V = OFF_K + NS * SLOT;
    static constexpr int BYTES = OFF_V + NS * SLOT;
    static_assert(HTBOX <= SLOT, "an Hbar^T box must fit one ring slot");
};

struct Params {
    int32_t S, H, NQ, NK, W;
    int32_t G, comp;
    float scale_log2;   // s * log2(e)
    float s;            // 1/sqrt(D)
    const int32_t* idx;
    const int32_t* count;
    const uint32_t* mask;
    __nv_bfloat16* out;
    int64_t osB, osS, osH;
};

struct Ctl {
    uint64_t q_full, q_tmem;                       // Q landed in smem / copied into TMEM
    uint64_t k_full[NS], k_empty[NS], s_full[NS];  // per K slot / S buffer (n % NS)
    uint64_t p_full[NS], pv_done[NS];              // per buffer: P ready + V landed; O-MMA done
    uint32_t tmem_base;
    int32_t nops;
    uint32_t mask[64];
    float mchain[kBQ];       // reference max after the latest decided op, per row
    float2 cpub[2][kBQ];     // 32-block half sums (h0, h1) of the latest C op, slot = chunk & 1
    float lpart[2][kBQ];     // epilogue: per-warpgroup denominators
    uint16_t ops[kMaxOps];
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_sm100_pp_kernel(const __grid_constant__ CUtensorMap tmQ,
                         const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV,
                         const __grid_constant__ CUtensorMap tmKb,
                         const __grid_constant__ CUtensorMap tmVs,
                         const __grid_constant__ CUtensorMap tmHt, const Params p) {
    using G_ = Geo<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ Ctl ctl;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int i = blockIdx.x, bh = blockIdx.y;
    const int b = bh / p.H, h = bh % p.H;
    const int64_t row = (int64_t)bh * p.NQ + i;
    const int32_t cnt = p.count[row];
    const int NK = p.NK;
    const int nchunks = (NK + 63) / 64;

    // ---------------- setup: op list, mask row, barriers, TMEM ----------------
    for (int w = tid; w < p.W; w += blockDim.x) ctl.mask[w] = p.mask[row * p.W + w];
    for (int q = tid; q < cnt; q += blockDim.x) ctl.ops[q] = op_make(OP_E, (uint32_t)p.idx[row * (int64_t)NK + q]);
    if (tid == 0) {
        mbar_init(&ctl.q_full, 1);
        mbar_init(&ctl.q_tmem, 256);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&ctl.k_full[s], 1);
            mbar_init(&ctl.k_empty[s], 1);
            mbar_init(&ctl.s_full[s], 1);
            mbar_init(&ctl.p_full[s], 129);   // 128 softmax threads + the V producer (expect_tx)
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
    __syncthreads();
    if (tid == 0) {
        // tail of the op list: every centroid chunk with a dropped block, then the
        // first-order op of each group inside the chunk that has a dropped block
        // (G = 32: groups 2c and 2c+1; G = 64: group c)
        int n = cnt;
        if (p.comp != PASA_COMP_NONE && cnt < NK) {
            const int W = (int)p.W;
            auto dropped_word = [&](int w) {
                const int rem = NK - 32 * w;
                const uint32_t inb = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
                return (~ctl.mask[w] & inb) != 0u;
            };
            for (int c = 0; c < nchunks; ++c) {
                const bool d0 = dropped_word(2 * c);
                const bool d1 = 2 * c + 1 < W && dropped_word(2 * c + 1);
                if (!(d0 || d1)) continue;
                ctl.ops[n++] = op_make(OP_C, (uint32_t)c);
                if (p.comp == PASA_COMP_GROUPED) {
                    if (p.G == 64) {
                        ctl.ops[n++] = op_make(OP_F, (uint32_t)c);
                    } else {
                        if (d0) ctl.ops[n++] = op_make(OP_F, (uint32_t)(2 * c));
                        if (d1) ctl.ops[n++] = op_make(OP_F, (uint32_t)(2 * c + 1));
                    }
                }
            }
        }
        ctl.nops = n;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int nops = ctl.nops;
    const uint32_t tbase = ctl.tmem_base;

    if (warp < 4) {
        if (warp == 0) {
            // ======================= K-ring producer =======================
            if (lane == 0) {
                mbar_arrive_expect_tx(&ctl.q_full, kBQ * D * 2);
#pragma unroll
                for (int a = 0; a < G_::NBOX; ++a)
                    tma_load_4d(smem + G_::OFF_Q + a * G_::QBOX, &tmQ, &ctl.q_full, 64 * a,
                                i * kBQ, h, b);
                for (int n = 0; n < nops; ++n) {
                    const int s = n % NS;
                    mbar_wait_sleep(&ctl.k_empty[s], ((n / NS) & 1) ^ 1);
                    uint8_t* dst = smem + G_::OFF_K + s * G_::SLOT;
                    const uint32_t op = ctl.ops[n];
                    const int v = (int)op_val(op);
                    if (op_type(op) == OP_F) {
                        mbar_arrive_expect_tx(&ctl.k_full[s], G_::HTBOX);
                        tma_load_3d(dst, &tmHt, &ctl.k_full[s], 0, v * D, bh);
                    } else {
                        mbar_arrive_expect_tx(&ctl.k_full[s], G_::SLOT);
#pragma unroll
                        for (int a = 0; a < G_::NBOX; ++a) {
                            if (op_type(op) == OP_E)
                                tma_load_4d(dst + a * G_::KVBOX, &tmK, &ctl.k_full[s], 64 * a,
                                            v * kBK, h, b);
                            else
                                tma_load_3d(dst + a * G_::KVBOX, &tmKb, &ctl.k_full[s], 64 * a,
                                            v * 64, bh);
                        }
                    }
                }
            }
            __syncwarp();
        } else if (warp == 2) {
            // ======================= V-ring producer =======================
            if (lane == 0) {
                for (int n = 0; n < nops; ++n) {
                    const int s = n % NS;
                    mbar_wait_sleep(&ctl.pv_done[s], ((n / NS) & 1) ^ 1);   // PV(n-NS) read the slot
                    uint8_t* dst = smem + G_::OFF_V + s * G_::SLOT;
                    const uint32_t op = ctl.ops[n];
                    const int v = (int)op_val(op);
                    if (op_type(op) == OP_F) {
                        if (G_::NBOX == 2) {
                            mbar_arrive_expect_tx(&ctl.p_full[s], G_::HTBOX);
                            tma_load_3d(dst, &tmHt, &ctl.p_full[s], 64, v * D, bh);
                        } else {
                            mbar_arrive(&ctl.p_full[s]);
                        }
                    } else {
                        mbar_arrive_expect_tx(&ctl.p_full[s], G_::SLOT);
#pragma unroll
                        for (int a = 0; a < G_::NBOX; ++a) {
                            if (op_type(op) == OP_E)
                                tma_load_4d(dst + a * G_::KVBOX, &tmV, &ctl.p_full[s], 64 * a,
                                            v * kBK, h, b);
                            else
                                tma_load_3d(dst + a * G_::KVBOX, &tmVs, &ctl.p_full[s], 64 * a,
                                            v * 64, bh);
                        }
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            // ======================= MMA issuer =======================
            // QK^T reads Q from TMEM (TS MMA: only the K tile comes from shared memory).
            // Per op n (buffer s = n % NS): wait P(n) -> PV(n) (or F(n)) -> QK(n+NS) into the
            // same buffer (tcgen05 ops run in issue order, so PV(n) has read P(n) first).
            constexpr uint32_t kIdQK = idesc_bf16_f32(128, kBK, 0, 0);   // Q (TMEM) x K^T (K-major)
            constexpr uint32_t kIdPV = idesc_bf16_f32(128, D, 0, 1);     // P (TMEM) x V (MN-major)
            constexpr uint32_t kIdF = idesc_bf16_f32(128, D, 0, 0);      // Aq (TMEM) x Hbar^T (K-major)
            const uint32_t k_base = smem_u32(smem + G_::OFF_K);
            const uint32_t v_base = smem_u32(smem + G_::OFF_V);
            const uint64_t dk0 = umma_desc_sw128(k_base, 16, 1024);
            const uint64_t dv0 = umma_desc_sw128(v_base, G_::KVBOX, 1024);
            auto issue_qk = [&](int n) {
                const int s = n % NS;
                mbar_wait_sleep(&ctl.k_full[s], (n / NS) & 1);
                tc_fence_after();
                const uint32_t d = tbase + G_::SCOL + 64 * s;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t offk = (s * G_::SLOT + (kk >> 2) * G_::KVBOX + (kk & 3) * 32) >> 4;
                    mma_ts_elect(d, tbase + G_::QCOL + kk * 8, dk0 + offk, kIdQK, kk > 0);
                }
                mma_commit_elect(&ctl.s_full[s]);
                mma_commit_elect(&ctl.k_empty[s]);
                __syncwarp();
            };
            mbar_wait_sleep(&ctl.q_tmem, 0);   // the softmax warps copied Q into TMEM
            tc_fence_after();
            for (int m = 0; m < NS && m < nops; ++m)
                if (op_type(ctl.ops[m]) != OP_F) issue_qk(m);
            for (int n = 0; n < nops; ++n) {
                const int s = n % NS;
                mbar_wait_sleep(&ctl.p_full[s], (n / NS) & 1);   // P(n) ready and V(n) landed
                tc_fence_after();
                const uint32_t op = ctl.ops[n];
                if (op_type(op) != OP_F) {
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint32_t offv = (s * G_::SLOT + kk * 16 * 128) >> 4;
                        mma_ts_elect(tbase, tbase + G_::SCOL + 64 * s + kk * 8, dv0 + offv, kIdPV,
                                     (n > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit_elect(&ctl.pv_done[s]);
                } else {
                    mbar_wait_sleep(&ctl.k_full[s], (n / NS) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t box = (kk >> 2) == 0 ? k_base + s * G_::SLOT
                                                            : v_base + s * G_::SLOT;
                        const uint64_t bd = umma_desc_sw128(box + (kk & 3) * 32, 16, 1024);
                        mma_ts_elect(tbase, tbase + G_::SCOL + 64 * s + kk * 8, bd, kIdF, 1u);
                    }
                    mma_commit_elect(&ctl.k_empty[s]);
                    mma_commit_elect(&ctl.pv_done[s]);
                }
                __syncwarp();
                if (n + NS < nops && op_type(ctl.ops[n + NS]) != OP_F) issue_qk(n + NS);
            }
        }
    } else {
        // =================== softmax / correction / epilogue ===================
        const int wg = (warp >> 2) - 1;                       // 0: even ops, 1: odd ops
        const int r = (warp & 3) * 32 + lane;                 // query row in the block
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t t_o = tbase + lane_off;
        const uint8_t* qrow = smem + G_::OFF_Q;
        // Q -> TMEM (the A operand of QK^T): warpgroup w copies 64-column box w of its rows
        mbar_wait_sleep(&ctl.q_full, 0);
        if (wg < G_::NBOX) {
            uint32_t qa[32];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const uint4 u = *reinterpret_cast<const uint4*>(qrow + wg * G_::QBOX + r * 128 +
                                                                ((cc ^ (r & 7)) << 4));
                qa[cc * 4 + 0] = u.x; qa[cc * 4 + 1] = u.y; qa[cc * 4 + 2] = u.z; qa[cc * 4 + 3] = u.w;
            }
            tmem_st32(t_o + G_::QCOL + 32 * wg, qa);
            tmem_wait_st();
        }
        tc_fence_before();
        mbar_arrive(&ctl.q_tmem);
        float m_ref = -INFINITY;   // the reference max this warpgroup's l is relative to
        float l = 0.f;
        int sc0 = 0, sc1 = 0;      // S-type ops seen on this warpgroup's two buffers (s_full parity)
        const int n_last = NK - 1;
        const int nlast_len = p.S - n_last * 64;
        const float cs = p.scale_log2;   // logits in log2 units: x = S * s * log2(e)
        // pv_done[b] completes once per op on buffer b (ops b, b+NS, ...): op m's completion is
        // phase m / NS of pv_done[m % NS]; only the latest op issued on a buffer is ever
        // awaited (PV(n) cannot start before P(n) is released), so the parity test is exact.
        auto consume_op = [&](int op) {
            if (op < 0) return;
            mbar_wait_sleep(&ctl.pv_done[op % NS], (op / NS) & 1);
        };
        // m_{n-1}: decided by the other warpgroup (op n-1); n = 0 starts from -inf
        auto chain_get = [&](int n) -> float {
            if (n == 0) return -INFINITY;
            bar_sync(kBarChain + (1 - wg), 256);
            return ctl.mchain[r];
        };
        auto chain_put = [&](float mv) {
            ctl.mchain[r] = mv;
            bar_arrive(kBarChain + wg, 256);
        };
        for (int n = wg; n < nops; n += 2) {
            const uint32_t op = ctl.ops[n];
            const uint32_t type = op_type(op);
            const int v = (int)op_val(op);
            const int bsel = (n >> 1) & 1;                    // which of this warpgroup's buffers
            const uint32_t t_buf = tbase + lane_off + G_::SCOL + 64 * (n % NS);
            if (type != OP_F) {
                mbar_wait_sleep(&ctl.s_full[n % NS], ((bsel ? sc1++ : sc0++)) & 1);
                tc_fence_after();
                uint32_t sa[32], sb[32];
                tmem_ld32(t_buf, sa);
                tmem_ld32(t_buf + 32, sb);
                tmem_wait_ld();
                // valid columns and denominator weights
                uint64_t valid;
                float wlast = 1.f;     // token count of block n_last (C ops)
                int clast = -1;        // column of block n_last in this chunk (C ops)
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
                if (valid != ~0ull) {   // masked columns -> -inf (ragged block, kept blocks)
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        if (!((valid >> c) & 1ull)) sa[c] = 0xff800000u;
                        if (!((valid >> (c + 32)) & 1ull)) sb[c] = 0xff800000u;
                    }
                }
                float mr0 = -INFINITY, mr1 = -INFINITY, mr2 = -INFINITY, mr3 = -INFINITY;
#pragma unroll
                for (int c = 0; c < 16; c += 2) {
                    mr0 = fmax3(mr0, __uint_as_float(sa[c]), __uint_as_float(sa[c + 1]));
                    mr1 = fmax3(mr1, __uint_as_float(sb[c]), __uint_as_float(sb[c + 1]));
                    mr2 = fmax3(mr2, __uint_as_float(sa[c + 16]), __uint_as_float(sa[c + 17]));
                    mr3 = fmax3(mr3, __uint_as_float(sb[c + 16]), __uint_as_float(sb[c + 17]));
                }
                const float mx = fmaxf(fmax3(mr0, mr1, mr2), mr3) * cs;
                float xlast = -INFINITY;
                if (clast >= 0) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        if (c == clast) xlast = __uint_as_float(sa[c]);
                        if (c + 32 == clast) xlast = __uint_as_float(sb[c]);
                    }
                }
                // the max decision, passed along the op sequence
                const float m_prev = chain_get(n);
                const float m = mx > m_prev + kRescaleThresh ? mx : m_prev;
                chain_put(m);
                if (m != m_ref) { l *= ex2(m_ref - m); m_ref = m; }   // ex2(-inf) = 0, l = 0 then
                const bool resc = n > 0 && m != m_prev;
                if (__any_sync(0xffffffffu, resc)) {
                    // O holds PV(..n-1) at m_prev: wait for the last two, rescale in place
                    const float corr = resc ? ex2(m_prev - m) : 1.f;
                    consume_op(n - 2);
                    consume_op(n - 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c0 = 0; c0 < D; c0 += 32) {
                        uint32_t o[32];
                        tmem_ld32(t_o + c0, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                        tmem_st32(t_o + c0, o);
                    }
                }
                float h0 = 0.f, h1 = 0.f;
                uint32_t pk[32];
                const float negm = -m;
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float p0 = ex2(fmaf(__uint_as_float(sa[2 * c]), cs, negm));
                    const float p1 = ex2(fmaf(__uint_as_float(sa[2 * c + 1]), cs, negm));
                    const float p2 = ex2(fmaf(__uint_as_float(sb[2 * c]), cs, negm));
                    const float p3 = ex2(fmaf(__uint_as_float(sb[2 * c + 1]), cs, negm));
                    h0 += p0 + p1;
                    h1 += p2 + p3;
                    pk[c] = pack_bf16(p0, p1);
                    pk[16 + c] = pack_bf16(p2, p3);
                }
                tmem_st32(t_buf, pk);
                if (type == OP_E) {
                    l += h0 + h1;
                } else {
                    // denominator: n_j * p_j; every dropped block has 64 tokens except the last
                    const float pl = clast >= 0 ? ex2(fmaf(xlast, cs, negm)) : 0.f;
                    l += 64.f * (h0 + h1) - (64.f - wlast) * pl;
                    if (p.comp == PASA_COMP_GROUPED) {
                        // the 32-block half sums for the F ops of this chunk's groups; the
                        // next op (other warpgroup) is F exactly when it needs them now
                        ctl.cpub[v & 1][r] = make_float2(h0, h1);
                        if (n + 1 < nops && op_type(ctl.ops[n + 1]) == OP_F) bar_arrive(kBarCpub, 256);
                    }
                }
                tmem_wait_st();
            } else {
                // F(g): Aq = bf16(s * A_{t,g} * q_t) into this warpgroup's buffer (R-21).
                // The group's C op is op n-1 (other warpgroup: wait for its sums) or op n-2
                // (this warpgroup, G = 32, the chunk's second group).
                if (op_type(ctl.ops[n - 1]) == OP_C) bar_sync(kBarCpub, 256);
                const int c = p.G == 64 ? v : (v >> 1);
                const float2 hs = ctl.cpub[c & 1][r];
                const float A = p.G == 64 ? hs.x + hs.y : ((v & 1) ? hs.y : hs.x);
                // m passes through an F op unchanged (read the sums before publishing it)
                const float m_prev = chain_get(n);
                chain_put(m_prev);
                if (m_prev != m_ref) { l *= ex2(m_ref - m_prev); m_ref = m_prev; }
                const float w = p.s * A;
                const uint32_t w2 = pack_bf16(w, w);
                consume_op(n - NS);   // the buffer's previous reader
                tc_fence_after();
#pragma unroll
                for (int a = 0; a < G_::NBOX; ++a) {
                    uint32_t aq[32];
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const uint4 u = *reinterpret_cast<const uint4*>(
                            qrow + a * G_::QBOX + r * 128 + ((cc ^ (r & 7)) << 4));
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
            mbar_arrive(&ctl.p_full[n % NS]);
        }
        // ---- epilogue: final reference max, l = l_0 + l_1, O / l -> bf16 -> global ----
        if (((nops - 1) & 1) != wg) {   // the other warpgroup decided the last op
            const float m_fin = chain_get(nops);
            if (m_fin != m_ref) { l *= ex2(m_ref - m_fin); m_ref = m_fin; }
        }
        ctl.lpart[wg][r] = l;
        bar_sync(kBarEpi, 256);
        const float inv = 1.f / (ctl.lpart[0][r] + ctl.lpart[1][r]);
        // every PV done.  Parity waits are exact only while the barrier is at most one phase
        // behind: this warpgroup's last op guarantees PV(nops-6) complete, so first wait for
        // op nops-4 (its predecessor on the barrier, nops-8, is complete), which completes
        // every PV up to nops-4 and makes the wait for nops-1 exact.
        consume_op(nops - 4);
        consume_op(nops - 1);
        tc_fence_after();
        const int t = i * kBQ + r;
        __nv_bfloat16* orow = p.out + (int64_t)b * p.osB + (int64_t)h * p.osH + (int64_t)t * p.osS;
#pragma unroll 1
        for (int c0 = wg * (D / 2); c0 < (wg + 1) * (D / 2); c0 += 32) {
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
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, kTmemCols);
    }
}

// ---------------------------------------------------------------- host --
template <int D>
cudaError_t launch_d(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                     pasa_route_s* r, const pasa_tensor& out, cudaStream_t st, char* why,
                     size_t why_len) {
    CUtensorMap mQ, mK, mV, mKb, mVs, mHt;
    auto act = [&](CUtensorMap* m, const pasa_tensor& t, uint32_t rows) {
        uint64_t dims[4] = {(uint64_t)t.D, (uint64_t)t.S, (uint64_t)t.H, (uint64_t)t.B};
        uint64_t str[3] = {(uint64_t)t.sS * 2, (uint64_t)t.sH * 2, (uint64_t)t.sB * 2};
        uint32_t box[4] = {64, rows, 1, 1};
        return make_tensor_map(m, t.data, 4, dims, str, box, why, why_len);
    };
    if (!act(&mQ, q, kBQ) || !act(&mK, k, kBK) || !act(&mV, v, kBK))
        return cudaErrorNotSupported;
    {
        uint64_t dims[3] = {(uint64_t)D, (uint64_t)r->NK, (uint64_t)r->BH};
        uint64_t str[2] = {(uint64_t)D * 2, (uint64_t)r->NK * D * 2};
        uint32_t box[3] = {64, 64, 1};
        if (!make_tensor_map(&mKb, r->kbar_lp, 3, dims, str, box, why, why_len) ||
            !make_tensor_map(&mVs, r->vsum_lp, 3, dims, str, box, why, why_len))
            return cudaErrorNotSupported;
    }
    {
        uint64_t dims[3] = {(uint64_t)D, (uint64_t)r->NG * D, (uint64_t)r->BH};
        uint64_t str[2] = {(uint64_t)D * 2, (uint64_t)r->NG * D * D * 2};
        uint32_t box[3] = {64, (uint32_t)D, 1};
        if (!make_tensor_map(&mHt, r->ht, 3, dims, str, box, why, why_len)) return cudaErrorNotSupported;
    }
    Params prm;
    prm.S = (int32_t)r->S; prm.H = (int32_t)r->H; prm.NQ = (int32_t)r->NQ; prm.NK = (int32_t)r->NK;
    prm.W = (int32_t)r->W;
    prm.G = r->cfg.G; prm.comp = r->cfg.comp;
    const double s = 1.0 / sqrt((double)D);
    prm.s = (float)s;
    prm.scale_log2 = (float)(s * 1.4426950408889634);
    prm.idx = r->idx; prm.count = r->count; prm.mask = r->mask;
    prm.out = reinterpret_cast<__nv_bfloat16*>(out.data);
    prm.osB = out.sB; prm.osS = out.sS; prm.osH = out.sH;
    // one CTA per SM (it allocates all 512 TMEM columns): request more than half the
    // shared memory so a second CTA never waits in tcgen05.alloc
    size_t smem = (size_t)Geo<D>::BYTES + 1024;
    if (smem < 120 * 1024) smem = 120 * 1024;
    auto kern = attn_sm100_pp_kernel<D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)r->NQ, (unsigned)r->BH);
    kern<<<grid, kThreads, smem, st>>>(mQ, mK, mV, mKb, mVs, mHt, prm);
    return cudaGetLastError();
}

}  // namespace

bool attn_sm100_pp_supported(const pasa_route_s* r) {
    return r->cfg.Bq == kBQ && r->cfg.Bk == kBK && (r->D == 128 || r->D == 64) && r->W <= 64 &&
           (r->cfg.comp != PASA_COMP_GROUPED || r->cfg.G == 32 || r->cfg.G == 64);
}

cudaError_t launch_attn_sm100_pp(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                                 pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                                 int* launches, char* why, size_t why_len) {
    if (!attn_sm100_pp_supported(r)) {
        snprintf(why, why_len, "two-warpgroup kernel: needs Bq=128, Bk=64, d in {64, 128}, "
                 "N_K <= 2048, G in {32, 64} for grouped compensation");
        return cudaErrorNotSupported;
    }
    cudaError_t e = r->D == 128 ? launch_d<128>(q, k, v, r, out, st, why, why_len)
                                : launch_d<64>(q, k, v, r, out, st, why, why_len);
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace pasa
