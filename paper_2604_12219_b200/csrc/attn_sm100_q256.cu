// attn_sm100_q256.cu -- pasa_attn for 256-row query blocks (Bq = 256; SURVEY.md
// §8f NEXT 4, a reading of R-7: one route per 256 queries) on the tcgen05 tensor
// cores.  Same method and op list as attn_sm100.cu (Eq. 7, PAPER.md:216-228;
// grouped first-order term, App. B :503-506; readings R-1..R-5,
// R-21, R-22); what changes is the data movement: every operand tile an op brings
// from L2 (K_j + V_j, a Kbar / Vsum chunk, or Hbar^(g)T) feeds TWO 128-row M tiles.
//
// Built to test whether the L2 bytes per FLOP bound the Bq = 128 kernel (every op
// costs ~1,000 SM cycles whatever its softmax or MMA work): it halves them, and is
// slower (24.1 vs 22.6 ms at Wan-14B), because that launch runs at the board power
// limit and this layout spends more energy per launch (DESIGN.md §7,
// profiles/r01_attn_power.md).  Here one CTA per SM owns the SM's 512 TMEM
// columns as two independent halves, tile t in {0, 1} at column 256 t:
//   O_t (D columns) + two S/P buffers of 64 columns,
// and two softmax warpgroups (warps 4-7: rows 0-127, warps 8-11: rows 128-255),
// each running the single-warpgroup softmax of attn_sm100.cu on its own rows with
// its own running max, denominator and group sums -- nothing is shared between
// them but the op list and the K/V ring.  The MMA warp issues every tcgen05 op
// twice, once per tile, on the same shared-memory B operand.
// Warp roles (384 threads): warp 0 K-ring TMA producer, warp 1 TMEM allocator +
// MMA issuer, warp 2 V-ring TMA producer, warp 3 idle, warps 4-11 softmax.
// Domain: bf16, Bq = 256, Bk = 64, d = 64 or 128, G in {32, 64, multiples of 128,
// >= N_K} or no grouped term.
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
constexpr int kBQ = 256, kBK = 64, kTile = 128;
// op list: kept blocks (<= N_K <= 4096) + centroid chunks (<= 64) + first-order ops
// (<= N_K / 8 for G >= 8) + slack; 16-bit entries (type in the top 2 bits)
constexpr int kMaxNK = 4096;
constexpr int kMaxOps = kMaxNK + kMaxNK / 64 + kMaxNK / 8 + 64;
constexpr int kTmemCols = 512;
constexpr float kRescaleThresh = 8.f;   // log2 units

enum : int32_t { OP_E = 0, OP_C = 1, OP_F = 2 };
__device__ __forceinline__ uint16_t op_make(int32_t type, int32_t v) {
    return (uint16_t)((type << 14) | v);
}
__device__ __forceinline__ int32_t op_type(int32_t op) { return op >> 14; }
__device__ __forceinline__ int32_t op_val(int32_t op) { return op & 0x3FFF; }

template <int D>
struct Geo {
    static constexpr uint32_t SCOL = D;             // S buffer s of tile t at 256 t + D + 64 s
    static constexpr int NBOX = D / 64;
    static constexpr int QBOX = kTile * 128;        // bytes per 64-col box of one Q tile
    static constexpr int KVBOX = kBK * 128;         // bytes per 64-col box of a K/V tile
    static constexpr int SLOT = kBK * D * 2;        // bytes per K or V slot
    static constexpr int HTBOX = D * 128;           // bytes per 64-col box of Hbar^T
    static constexpr int OFF_Q = 0;                 // tile t, box a at (t NBOX + a) QBOX
    static constexpr int OFF_K = kBQ * D * 2;
    static constexpr int OFF_V = OFF_K + 2 * SLOT;
    static constexpr int BYTES = OFF_V + 2 * SLOT;
    static_assert(HTBOX <= SLOT, "an Hbar^T box must fit one ring slot");
    static_assert(D + 128 <= 256, "per-tile TMEM budget");
};

struct Params {
    int32_t S, H, NQ, NK, W, G, comp;
    int32_t it0;        // first (head, q-block) item of the handle's range (grid.x covers it)
    float scale_log2;   // s * log2(e)
    float s;            // 1/sqrt(D)
    const int32_t* idx;
    const int32_t* count;
    const uint32_t* mask;
    __nv_bfloat16* out;
    int64_t osB, osS, osH;
};

struct Ctl {
    uint64_t q_full;
    uint64_t k_full[2], k_empty[2];     // K ring (n & 1)
    uint64_t v_full[2], v_empty[2];     // V ring (n & 1)
    uint64_t s_full[2][2];              // [tile][S buffer n & 1]: QK^T done
    uint64_t p_full[2][2];              // [tile][n & 1]: the tile's 128 softmax threads released P
    uint64_t pv_done[2][2];             // [tile][n & 1]: the tile's O-MMA of the op done
    uint32_t tmem_base;
    int32_t nops;
    uint32_t mask[kMaxNK / 32];
    uint16_t ops[kMaxOps];
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_sm100_q256_kernel(const __grid_constant__ CUtensorMap tmQ,
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
    const int item = p.it0 + (int)blockIdx.x;
    const int i = item % p.NQ, bh = item / p.NQ;
    const int b = bh / p.H, h = bh % p.H;
    const int64_t row = (int64_t)bh * p.NQ + i;
    const int32_t cnt = p.count[row];
    const int NK = p.NK;
    const int nchunks = (NK + 63) / 64;

    // ---------------- setup: op list, mask row, barriers, TMEM ----------------
    for (int w = tid; w < p.W; w += blockDim.x) ctl.mask[w] = p.mask[row * p.W + w];
    for (int q = tid; q < cnt; q += blockDim.x) ctl.ops[q] = op_make(OP_E, p.idx[row * (int64_t)NK + q]);
    if (tid == 0) {
        mbar_init(&ctl.q_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&ctl.k_full[s], 1);
            mbar_init(&ctl.k_empty[s], 1);
            mbar_init(&ctl.v_full[s], 1);
            mbar_init(&ctl.v_empty[s], 1);
            for (int t = 0; t < 2; ++t) {
                mbar_init(&ctl.s_full[t][s], 1);
                mbar_init(&ctl.p_full[t][s], 128);
                mbar_init(&ctl.pv_done[t][s], 1);
            }
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
            for (int c = 0; c < nchunks; ++c) {
                if (dropped_word(2 * c) || (2 * c + 1 < W && dropped_word(2 * c + 1)))
                    ctl.ops[n++] = op_make(OP_C, c);
                if (p.comp == PASA_COMP_GROUPED) {
                    const int chunk_end = min(64 * (c + 1), NK);
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
    tc_fence_after();
    const int nops = ctl.nops;
    const uint32_t tbase = ctl.tmem_base;

    if (warp == 0) {
        // ======================= K-ring producer =======================
        if (lane == 0) {
            mbar_arrive_expect_tx(&ctl.q_full, kBQ * D * 2);
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int a = 0; a < G_::NBOX; ++a)
                    tma_load_4d(smem + G_::OFF_Q + (t * G_::NBOX + a) * G_::QBOX, &tmQ, &ctl.q_full,
                                64 * a, i * kBQ + t * kTile, h, b);
            for (int n = 0; n < nops; ++n) {
                const int s = n & 1;
                mbar_wait_sleep(&ctl.k_empty[s], ((n >> 1) & 1) ^ 1);
                uint8_t* dst = smem + G_::OFF_K + s * G_::SLOT;
                const int32_t op = ctl.ops[n];
                const int v = op_val(op);
                if (op_type(op) == OP_F) {
                    mbar_arrive_expect_tx(&ctl.k_full[s], G_::HTBOX);
                    tma_load_3d(dst, &tmHt, &ctl.k_full[s], 0, v * D, bh);
                } else {
                    mbar_arrive_expect_tx(&ctl.k_full[s], G_::SLOT);
#pragma unroll
                    for (int a = 0; a < G_::NBOX; ++a) {
                        if (op_type(op) == OP_E)
                            tma_load_4d(dst + a * G_::KVBOX, &tmK, &ctl.k_full[s], 64 * a, v * kBK, h, b);
                        else
                            tma_load_3d(dst + a * G_::KVBOX, &tmKb, &ctl.k_full[s], 64 * a, v * 64, bh);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ======================= V-ring producer =======================
        if (lane == 0) {
            for (int n = 0; n < nops; ++n) {
                const int s = n & 1;
                mbar_wait_sleep(&ctl.v_empty[s], ((n >> 1) & 1) ^ 1);   // both O-MMAs of op n-2 done
                uint8_t* dst = smem + G_::OFF_V + s * G_::SLOT;
                const int32_t op = ctl.ops[n];
                const int v = op_val(op);
                if (op_type(op) == OP_F) {
                    if (G_::NBOX == 2) {
                        mbar_arrive_expect_tx(&ctl.v_full[s], G_::HTBOX);
                        tma_load_3d(dst, &tmHt, &ctl.v_full[s], 64, v * D, bh);
                    } else {
                        mbar_arrive(&ctl.v_full[s]);
                    }
                } else {
                    mbar_arrive_expect_tx(&ctl.v_full[s], G_::SLOT);
#pragma unroll
                    for (int a = 0; a < G_::NBOX; ++a) {
                        if (op_type(op) == OP_E)
                            tma_load_4d(dst + a * G_::KVBOX, &tmV, &ctl.v_full[s], 64 * a, v * kBK, h, b);
                        else
                            tma_load_3d(dst + a * G_::KVBOX, &tmVs, &ctl.v_full[s], 64 * a, v * 64, bh);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer =======================
        // QK(n+1) of both tiles is issued before PV(n); each tcgen05 op runs once per tile
        // (A operand / accumulator of tile t, the same B tile from shared memory).
        constexpr uint32_t kIdQK = idesc_bf16_f32(128, kBK, 0, 0);   // Q x K^T, both K-major
        constexpr uint32_t kIdPV = idesc_bf16_f32(128, D, 0, 1);     // P (TMEM) x V (MN-major)
        constexpr uint32_t kIdF = idesc_bf16_f32(128, D, 0, 0);      // Aq (TMEM) x Hbar^T (K-major)
        const uint32_t q_base = smem_u32(smem + G_::OFF_Q);
        const uint32_t k_base = smem_u32(smem + G_::OFF_K);
        const uint32_t v_base = smem_u32(smem + G_::OFF_V);
        const uint64_t dq0 = umma_desc_sw128(q_base, 16, 1024);
        const uint64_t dk0 = umma_desc_sw128(k_base, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(v_base, G_::KVBOX, 1024);
        auto issue_qk = [&](int n) {
            const int s = n & 1;
            mbar_wait_sleep(&ctl.k_full[s], (n >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const uint32_t d = tbase + 256 * t + G_::SCOL + 64 * s;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t offq = (((t * G_::NBOX) + (kk >> 2)) * G_::QBOX + (kk & 3) * 32) >> 4;
                    const uint32_t offk = (s * G_::SLOT + (kk >> 2) * G_::KVBOX + (kk & 3) * 32) >> 4;
                    mma_ss_elect(d, dq0 + offq, dk0 + offk, kIdQK, kk > 0);
                }
                mma_commit_elect(&ctl.s_full[t][s]);
            }
            mma_commit_elect(&ctl.k_empty[s]);
            __syncwarp();
        };
        mbar_wait_sleep(&ctl.q_full, 0);
        tc_fence_after();
        if (nops > 0 && op_type(ctl.ops[0]) != OP_F) issue_qk(0);
        for (int n = 0; n < nops; ++n) {
            const int s = n & 1;
            if (n + 1 < nops && op_type(ctl.ops[n + 1]) != OP_F) issue_qk(n + 1);
            const int32_t op = ctl.ops[n];
            const bool f_op = op_type(op) == OP_F;
            mbar_wait_sleep(&ctl.v_full[s], (n >> 1) & 1);
            if (f_op) mbar_wait_sleep(&ctl.k_full[s], (n >> 1) & 1);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                mbar_wait_sleep(&ctl.p_full[t][s], (n >> 1) & 1);
                tc_fence_after();
                const uint32_t o = tbase + 256 * t;
                const uint32_t a0 = o + G_::SCOL + 64 * s;
                if (!f_op) {
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint32_t offv = (s * G_::SLOT + kk * 16 * 128) >> 4;
                        mma_ts_elect(o, a0 + kk * 8, dv0 + offv, kIdPV, (n > 0 || kk > 0) ? 1u : 0u);
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t box = (kk >> 2) == 0 ? k_base + s * G_::SLOT : v_base + s * G_::SLOT;
                        const uint64_t bd = umma_desc_sw128(box + (kk & 3) * 32, 16, 1024);
                        mma_ts_elect(o, a0 + kk * 8, bd, kIdF, 1u);
                    }
                }
                // the slot releases precede tile 1's pv_done: the last asynchronous arrival
                // of the CTA is then one the softmax warps wait for before the epilogue (a
                // commit still in flight at exit would land in the next CTA's barriers)
                if (t == 1) {
                    if (f_op) mma_commit_elect(&ctl.k_empty[s]);
                    mma_commit_elect(&ctl.v_empty[s]);
                }
                mma_commit_elect(&ctl.pv_done[t][s]);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ============ softmax / correction / epilogue of tile t (rows 128 t ..) ============
        const int t = (warp >> 2) - 1;
        const int r = (warp & 3) * 32 + lane;                 // row in the tile
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t t_o = tbase + lane_off + 256 * t;
        const uint8_t* qrow = smem + G_::OFF_Q + t * G_::NBOX * G_::QBOX;
        float m = -INFINITY, l = 0.f;
        float A_cur = 0.f, A_done = 0.f;
        int g_cur = -1, g_done = -1;
        int sc0 = 0, sc1 = 0;   // S-type ops seen per S buffer (s_full parity)
        const int n_last = NK - 1;
        const int nlast_len = p.S - n_last * 64;
        const float cs = p.scale_log2;
        // pv_done[t][b] completes once per op on buffer b (ops b, b+2, ...); only the latest
        // op issued on a buffer is ever awaited, so the parity test is exact (attn_sm100.cu)
        auto consume_op = [&](int op) {
            if (op < 0) return;
            mbar_wait_sleep(&ctl.pv_done[t][op & 1], (op >> 1) & 1);
        };
        for (int n = 0; n < nops; ++n) {
            const int s = n & 1;
            const int32_t op = ctl.ops[n];
            const int type = op_type(op), v = op_val(op);
            const uint32_t t_buf = t_o + G_::SCOL + 64 * s;
            if (type != OP_F) {
                mbar_wait_sleep(&ctl.s_full[t][s], (s ? sc1++ : sc0++) & 1);
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
                float corr = 1.f;
                bool resc = false;
                if (mx > m + kRescaleThresh) {
                    corr = ex2(m - mx);
                    resc = n > 0;
                    m = mx;
                    l *= corr;
                    A_cur *= corr;
                }
                if (__any_sync(0xffffffffu, resc)) {
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
                    const float pl = clast >= 0 ? ex2(fmaf(xlast, cs, negm)) : 0.f;
                    l += 64.f * (h0 + h1) - (64.f - wlast) * pl;
                    // group sums A_{t,g} (each 32-block half lies in one group)
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
                const float A = v == g_done ? A_done : A_cur;
                const float w = p.s * A;
                const uint32_t w2 = pack_bf16(w, w);
                consume_op(n - 2);   // the buffer's previous reader
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
            mbar_arrive(&ctl.p_full[t][s]);
        }
        // ---- epilogue: O / l -> bf16 -> global ----
        consume_op(nops - 2);
        consume_op(nops - 1);
        tc_fence_after();
        const int tok = i * kBQ + t * kTile + r;
        const float inv = 1.f / l;
        __nv_bfloat16* orow = p.out + (int64_t)b * p.osB + (int64_t)h * p.osH + (int64_t)tok * p.osS;
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(t_o + c0, o);
            tmem_wait_ld();
            if (tok < p.S) {
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
    if (!act(&mQ, q, kTile) || !act(&mK, k, kBK) || !act(&mV, v, kBK)) return cudaErrorNotSupported;
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
    prm.G = (int32_t)(r->cfg.G < r->NK ? r->cfg.G : r->NK);   // one global group: G = N_K
    prm.comp = r->cfg.comp;
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
    auto kern = attn_sm100_q256_kernel<D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    prm.it0 = (int32_t)r->it0;
    const unsigned grid = (unsigned)(r->it1 - r->it0);   // head-major items
    kern<<<grid, kThreads, smem, st>>>(mQ, mK, mV, mKb, mVs, mHt, prm);
    return cudaGetLastError();
}

}  // namespace

bool attn_sm100_q256_supported(const pasa_route_s* r) {
    return r->cfg.Bq == kBQ && r->cfg.Bk == kBK && (r->D == 128 || r->D == 64) && r->NK <= kMaxNK &&
           (r->cfg.comp != PASA_COMP_GROUPED || r->cfg.G == 32 || r->cfg.G == 64 ||
            r->cfg.G % 128 == 0 || r->cfg.G >= r->NK);   // the attn_sm100.cu group set minus 8, 16
}

cudaError_t launch_attn_sm100_q256(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                                   pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                                   int* launches, char* why, size_t why_len) {
    if (!attn_sm100_q256_supported(r)) {
        snprintf(why, why_len, "Bq = 256 kernel: needs Bk=64, d in {64, 128}, N_K <= 4096, "
                 "G in {32, 64, multiples of 128, >= N_K} for grouped compensation");
        return cudaErrorNotSupported;
    }
    cudaError_t e = r->D == 128 ? launch_d<128>(q, k, v, r, out, st, why, why_len)
                                : launch_d<64>(q, k, v, r, out, st, why, why_len);
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace pasa
