// attn_sm100.cu -- pasa_attn on the Blackwell tensor cores (sm_100a):
// gather-driven block-sparse attention with the PASA compensation fused into
// the same online softmax (Eq. 7; grouped first-order term,
// PAPER.md:310-313 and App. B :503-506; readings R-1..R-5, R-21, R-22 in
// DESIGN.md §3).  Design notes and measurements: DESIGN.md §7.
//
// One CTA per (head, 128-row query block), one CTA per SM (TMEM: O 128 columns +
// two S/P buffers of 128 columns).  Kept key blocks are processed in PAIRS, so
// QK^T is an M128 x N128 tcgen05 MMA (the N64 shape is shared-memory bound) and
// PV an M128 x N(D) x K128 one.  Warp roles (384 threads):
//   warp 0      TMA producer of the K ring (K block pairs / Kbar chunks / Hbar^T)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warp 2      TMA producer of the V ring (V block pairs / Vsum chunks)
//   warp 3      builds the compensation op list at setup
//   warps 4-7   softmax warpgroup 0: columns 0-63 of every op (the pair's 1st block)
//   warps 8-11  softmax warpgroup 1: columns 64-127 (the pair's 2nd block)
// Warps 4+j and 8+j own the same 32 rows (TMEM lane quarter j) and exchange row
// maxima through shared memory behind a 64-thread named barrier.
// Op list of the CTA:
//   E(n)  kept blocks idx[2n], idx[2n+1]:  S = Q K^T -> softmax -> O += P V
//   C(c)  centroids 128c..128c+127:        S = Q Kbar^T masked to dropped blocks,
//                                          weights n_j in the denominator, O += P Vsum
//   F(g)  group g's first order:           O += (s A_g (.) Q) Hbar^(g)  (A from TMEM)
// Op n uses K-ring entry n and V-ring entry n (an F op's V entry is empty).  QK of
// op n+2 is issued right after op n's PV (double-buffered S).  The running max
// only moves when it grows by more than 2^8 (log2 units), so O corrections are
// rare; they wait for every earlier MMA first.
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
constexpr int kMaxNK = 2048;
constexpr int kMaxTail = 16 + 64 + 8;        // C ops (<= 16 chunks) + F ops (<= 64 groups)
constexpr int kTmemCols = 512;
constexpr int kColS = 256;                    // O_0 at column 0, O_1 at 128, S/P buffers at 256, 384
constexpr float kRescaleThresh = 8.f;         // log2 units

enum : int32_t { OP_E = 0, OP_C = 1, OP_F = 2 };
__device__ __forceinline__ int32_t op_make(int32_t type, int32_t v) { return (type << 24) | v; }
__device__ __forceinline__ int32_t op_type(int32_t op) { return op >> 24; }
__device__ __forceinline__ int32_t op_val(int32_t op) { return op & 0xFFFFFF; }

template <int D>
struct Geo {
    static constexpr int NBOX = D / 64;             // 64-element boxes along d
    static constexpr int DBOX_K = 128 * 128;        // K-ring slot: bytes per d-box (128 rows)
    static constexpr int SLOT = 128 * D * 2;        // a K or V ring slot (two 64-row blocks)
    static constexpr int QBYTES = kBQ * D * 2;
    static constexpr int NSK = D == 128 ? 3 : 6;    // K-ring depth
    static constexpr int NSV = D == 128 ? 2 : 5;    // V-ring depth
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = QBYTES;
    static constexpr int OFF_V = OFF_K + NSK * SLOT;
    static constexpr int BYTES = OFF_V + NSV * SLOT;
    static constexpr int HTBYTES = D * D * 2;       // Hbar^T of one group
    static_assert(HTBYTES <= SLOT, "Hbar^T must fit one K-ring slot");
};

struct Params {
    int64_t S, H, NQ, NK, NG, W;
    int32_t G, comp;
    float scale_log2;   // s * log2(e)
    float s;            // 1/sqrt(D)
    const int32_t* idx;
    const int32_t* count;
    const uint32_t* mask;
    __nv_bfloat16* out;
    int64_t osB, osS, osH;
    unsigned long long* trace;   // diagnostics: clock64 timeline of one CTA, or nullptr
    int32_t trace_x, trace_y;
    int32_t dbg;                 // diagnostics ablations: 1 = softmax skips its math, 2 = no TMA
};

// timeline events (pasa_debug_trace); slot = event * kTraceN + index
constexpr int kTraceN = 4096;
enum { TR_KPROD = 0, TR_VPROD, TR_MMA_P, TR_MMA_V, TR_MMA_QK, TR_SA_W, TR_SA_OK, TR_SA_ARR,
       TR_SB_W, TR_SB_OK, TR_SB_ARR, TR_MMA_QKW, TR_KPROD_W, TR_SA_LD, TR_SA_MAX, TR_SA_EXP,
       TR_SA_ST, TR_NEV };
#define PASA_TR(ev, ix)                                                               \
    do {                                                                              \
        if (tracing && (ix) < kTraceN) p.trace[(ev) * kTraceN + (ix)] = clock64();    \
    } while (0)

struct Ctl {
    uint64_t k_full[8], k_empty[8], v_full[8], v_empty[8];
    uint64_t q_full, s_full[2];
    uint64_t p_full[2][2], pv_done[2][2];   // [warpgroup][buffer]; pv_done: that half's O-MMA done
    uint64_t buf_free[2];   // buffer b free for the next QK (op m-2's O-MMA done, m S-type)
    uint32_t tmem_base;
    int32_t nops, nE, cnt;
    uint32_t mask[64];
    float xchg[2][2][2][kBQ];   // [slot][quantity][warpgroup][row]: F-op / epilogue exchange
    int32_t tail[kMaxTail];
    uint16_t eidx[kMaxNK];
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tmQ,
                      const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmKb,
                      const __grid_constant__ CUtensorMap tmVs,
                      const __grid_constant__ CUtensorMap tmHt, const Params p) {
    using G_ = Geo<D>;
    constexpr int NSK = G_::NSK, NSV = G_::NSV;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ Ctl ctl;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool tracing = p.trace != nullptr && (int)blockIdx.x == p.trace_x &&
                         (int)blockIdx.y == p.trace_y;
    const bool spin = (p.dbg & 4) != 0;   // diagnostics: poll instead of suspend
    const int64_t i = blockIdx.x, bh = blockIdx.y;
    const int64_t b = bh / p.H, h = bh % p.H;
    const int64_t row = bh * p.NQ + i;
    const int64_t NK = p.NK;
    const int W = (int)p.W;
    const int cnt = p.count[row];
    const int nE = (cnt + 1) >> 1;                       // E ops (block pairs)
    const int nchunks = (int)((NK + 127) / 128);         // 128-centroid chunks

    // ---------------- setup: index list, mask, barriers, TMEM ----------------
    for (int w = tid; w < W; w += kThreads) ctl.mask[w] = p.mask[row * W + w];
    for (int q = tid; q < cnt; q += kThreads) ctl.eidx[q] = (uint16_t)p.idx[row * NK + q];
    if (tid == 0) {
        for (int s = 0; s < NSK; ++s) {
            mbar_init(&ctl.k_full[s], 1);
            mbar_init(&ctl.k_empty[s], 1);
        }
        for (int s = 0; s < NSV; ++s) {
            mbar_init(&ctl.v_full[s], 1);
            mbar_init(&ctl.v_empty[s], 1);
        }
        mbar_init(&ctl.q_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&ctl.s_full[s], 1);
            mbar_init(&ctl.buf_free[s], 1);
            for (int w = 0; w < 2; ++w) {
                mbar_init(&ctl.p_full[w][s], 128);
                mbar_init(&ctl.pv_done[w][s], 1);
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
    if (warp == 3 && lane == 0) {
        // compensation tail: C ops for 128-block chunks holding a dropped block, then an
        // F op for every group with a dropped block that ends in the chunk.  Word w of
        // the mask covers blocks [32w, 32w+32), inside one group (G in {32, 64},
        // G % 128 == 0, or a single global group).
        int ntail = 0;
        if (p.comp != PASA_COMP_NONE && cnt < NK) {
            auto dropped_word = [&](int w) {
                const int64_t rem = NK - 32 * (int64_t)w;
                const uint32_t inb = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
                return (~ctl.mask[w] & inb) != 0u;
            };
            const int64_t G = p.G;
            int64_t g = 0;
            for (int c = 0; c < nchunks; ++c) {
                bool any = false;
                for (int w = 4 * c; w < min(4 * c + 4, W) && !any; ++w) any = dropped_word(w);
                if (any) ctl.tail[ntail++] = op_make(OP_C, c);
                if (p.comp == PASA_COMP_GROUPED) {
                    const int64_t chunk_end = min(128 * (int64_t)(c + 1), NK);
                    for (; g * G < NK && min((g + 1) * G, NK) <= chunk_end; ++g) {
                        const int w0 = (int)((g * G) >> 5);
                        const int w1 = (int)((min((g + 1) * G, NK) + 31) >> 5);
                        bool anyg = false;
                        for (int w = w0; w < w1 && !anyg; ++w) anyg = dropped_word(w);
                        if (anyg) ctl.tail[ntail++] = op_make(OP_F, (int32_t)g);
                    }
                }
            }
        }
        ctl.nE = nE;
        ctl.cnt = cnt;
        ctl.nops = nE + ntail;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int nops = ctl.nops;
    const uint32_t tbase = ctl.tmem_base;
    auto op_at = [&](int n) -> int32_t {
        return n < nE ? op_make(OP_E, n) : ctl.tail[n - nE];
    };

    if (warp == 0) {
        // ======================= K-ring producer =======================
        if (lane == 0) {
            mbar_arrive_expect_tx(&ctl.q_full, G_::QBYTES);
#pragma unroll
            for (int a = 0; a < G_::NBOX; ++a)
                tma_load_4d(smem + G_::OFF_Q + a * (kBQ * 128), &tmQ, &ctl.q_full, 64 * a,
                            (int)(i * kBQ), (int)h, (int)b);
            for (int n = 0; n < nops; ++n) {
                const int s = n % NSK;
                PASA_TR(TR_KPROD_W, n);
                mbar_wait_sleep(&ctl.k_empty[s], ((n / NSK) & 1) ^ 1);
                PASA_TR(TR_KPROD, n);
                uint8_t* dst = smem + G_::OFF_K + s * G_::SLOT;
                const int32_t op = op_at(n);
                const int v = op_val(op);
                if (p.dbg & 2) {
                    mbar_arrive(&ctl.k_full[s]);
                } else if (op_type(op) == OP_F) {
                    mbar_arrive_expect_tx(&ctl.k_full[s], G_::HTBYTES);
#pragma unroll
                    for (int a = 0; a < G_::NBOX; ++a)
                        tma_load_3d(dst + a * (D * 128), &tmHt, &ctl.k_full[s], 64 * a, v * D,
                                    (int)bh);
                } else {
                    mbar_arrive_expect_tx(&ctl.k_full[s], G_::SLOT);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                        for (int a = 0; a < G_::NBOX; ++a) {
                            uint8_t* d2 = dst + a * G_::DBOX_K + hh * (kBK * 128);
                            if (op_type(op) == OP_E) {
                                // the odd last op repeats its block (masked by the softmax)
                                const int q = min(2 * v + hh, cnt - 1);
                                tma_load_4d(d2, &tmK, &ctl.k_full[s], 64 * a, ctl.eidx[q] * kBK,
                                            (int)h, (int)b);
                            } else {
                                tma_load_3d(d2, &tmKb, &ctl.k_full[s], 64 * a, v * 128 + hh * 64,
                                            (int)bh);
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ======================= V-ring producer =======================
        if (lane == 0) {
            for (int n = 0; n < nops; ++n) {
                const int s = n % NSV;
                mbar_wait_sleep(&ctl.v_empty[s], ((n / NSV) & 1) ^ 1);
                PASA_TR(TR_VPROD, n);
                uint8_t* dst = smem + G_::OFF_V + s * G_::SLOT;
                const int32_t op = op_at(n);
                const int v = op_val(op);
                if ((p.dbg & 2) || op_type(op) == OP_F) {
                    mbar_arrive(&ctl.v_full[s]);
                } else {
                    mbar_arrive_expect_tx(&ctl.v_full[s], G_::SLOT);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                        for (int a = 0; a < G_::NBOX; ++a) {
                            uint8_t* d2 = dst + a * G_::DBOX_K + hh * (kBK * 128);
                            if (op_type(op) == OP_E) {
                                const int q = min(2 * v + hh, cnt - 1);
                                tma_load_4d(d2, &tmV, &ctl.v_full[s], 64 * a, ctl.eidx[q] * kBK,
                                            (int)h, (int)b);
                            } else {
                                tma_load_3d(d2, &tmVs, &ctl.v_full[s], 64 * a, v * 128 + hh * 64,
                                            (int)bh);
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1 || warp == 3) {
        // ============ MMA issuers: warp 3 issues QK^T, warp 1 issues PV / first order ============
        // Two issue streams: tcgen05.mma issue is nearly synchronous with execution, so
        // while one warp checks its barriers the other warp's MMAs keep the pipe busy.
        constexpr uint32_t kIdQK = idesc_bf16_f32(128, 128, 0, 0);   // Q (K-major) x K^T (K-major)
        constexpr uint32_t kIdPV = idesc_bf16_f32(128, D, 0, 1);     // P (TMEM) x V (MN-major)
        constexpr uint32_t kIdF = idesc_bf16_f32(128, D, 0, 0);      // Aq (TMEM) x Hbar^T (K-major)
        const uint32_t q_base = smem_u32(smem + G_::OFF_Q);
        const uint32_t k_base = smem_u32(smem + G_::OFF_K);
        const uint32_t v_base = smem_u32(smem + G_::OFF_V);
        // descriptors: the 14-bit start-address field is advanced arithmetically
        const uint64_t dq0 = umma_desc_sw128(q_base, 16, 1024);
        const uint64_t dk0 = umma_desc_sw128(k_base, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(v_base, G_::DBOX_K, 1024);
        auto is_s = [&](int n) { return n < nops && op_type(op_at(n)) != OP_F; };
        if (warp == 3) {
            // QK of S-type op m into buffer m&1, once op m-2's O-MMA has released the buffer
            // (buf_free[m&1], one phase per such m, consumed in order) and K entry m landed.
            int bf0 = 0, bf1 = 0;
            mbar_wait_c(&ctl.q_full, 0, spin);
            for (int m = 0; m < nops; ++m) {
                if (!is_s(m)) continue;
                if (m >= 2) {
                    const int par = (m & 1) ? (bf1++ & 1) : (bf0++ & 1);
                    mbar_wait_c(&ctl.buf_free[m & 1], par, spin);
                }
                const int s = m % NSK;
                if (lane == 0) PASA_TR(TR_MMA_QKW, m);
                mbar_wait_c(&ctl.k_full[s], (m / NSK) & 1, spin);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t d = tbase + kColS + 128 * (m & 1);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = ((kk >> 2) * (kBQ * 128) + (kk & 3) * 32) >> 4;
                        const uint32_t offk =
                            ((uint32_t)s * G_::SLOT + (kk >> 2) * G_::DBOX_K + (kk & 3) * 32) >> 4;
                        mma_ss(d, dq0 + off, dk0 + offk, kIdQK, kk > 0);
                    }
                    mma_commit(&ctl.s_full[m & 1]);
                    mma_commit(&ctl.k_empty[s]);
                    PASA_TR(TR_MMA_QK, m);
                }
                __syncwarp();
            }
        } else {
            // PV of op n: warpgroup w's half (keys 64w..64w+63, P at buffer column 64w) into
            // its own accumulator O_w; F ops accumulate (s A_g (.) Q) Hbar^(g) into O_0.
            for (int n = 0; n < nops; ++n) {
                const int bsel = n & 1;
                const bool isF = op_type(op_at(n)) == OP_F;
                mbar_wait_c(&ctl.v_full[n % NSV], (n / NSV) & 1, spin);
                if (isF) mbar_wait_c(&ctl.k_full[n % NSK], (n / NSK) & 1, spin);
                if (lane == 0) PASA_TR(TR_MMA_V, n);
                const uint32_t a_t = tbase + kColS + 128 * bsel;
                if (!isF) {
                    const int s = n % NSV;
#pragma unroll
                    for (int w = 0; w < 2; ++w) {
                        mbar_wait_c(&ctl.p_full[w][bsel], (n >> 1) & 1, spin);
                        tc_fence_after();
                        if (lane == 0) {
#pragma unroll
                            for (int kk = 0; kk < kBK / 16; ++kk) {
                                const uint32_t offv =
                                    ((uint32_t)s * G_::SLOT + w * (kBK * 128) + kk * 2048) >> 4;
                                mma_ts(tbase + 128 * w, a_t + 64 * w + kk * 8, dv0 + offv, kIdPV,
                                       (n > 0 || kk > 0) ? 1u : 0u);
                            }
                            mma_commit(&ctl.pv_done[w][bsel]);
                        }
                        __syncwarp();
                    }
                    if (lane == 0) mma_commit(&ctl.v_empty[s]);
                } else {
                    mbar_wait_c(&ctl.p_full[0][bsel], (n >> 1) & 1, spin);
                    mbar_wait_c(&ctl.p_full[1][bsel], (n >> 1) & 1, spin);
                    tc_fence_after();
                    if (lane == 0) {
                        const int sk = n % NSK;
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            // dims 16kk.. of the operand were written by warpgroup w at column 64w
                            const int w = (16 * kk) / (D / 2);
                            const uint32_t acol = 64 * w + (16 * kk - w * (D / 2)) / 2;
                            const uint32_t offk =
                                ((uint32_t)sk * G_::SLOT + (kk >> 2) * (D * 128) + (kk & 3) * 32) >> 4;
                            mma_ts(tbase, a_t + acol, dk0 + offk, kIdF, 1u);
                        }
                        mma_commit(&ctl.k_empty[sk]);
                        mma_commit(&ctl.v_empty[n % NSV]);
                        mma_commit(&ctl.pv_done[0][bsel]);
                        mma_commit(&ctl.pv_done[1][bsel]);
                    }
                    __syncwarp();
                }
                if (lane == 0) {
                    if (is_s(n + 2)) mma_commit(&ctl.buf_free[bsel]);
                    PASA_TR(TR_MMA_P, n);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // =================== softmax / correction / epilogue ===================
        // Warpgroup wg owns columns 64wg..64wg+63 of every op, its own running max m,
        // denominator l and accumulator O_wg (TMEM columns 128wg..): the two halves of a row
        // are independent online softmaxes, merged in the epilogue.  They exchange values
        // only at F ops (group sums) and at the end.
        constexpr int DH = D / 2;                             // output columns written per half
        const int wg = (warp - 4) >> 2;
        const int r = (warp & 3) * 32 + lane;                 // query row in the block
        const uint32_t bar_id = 1 + (warp & 3);               // pairs warps 4+j and 8+j
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t t_own = tbase + lane_off + 128 * wg;   // O_wg
        const uint8_t* qrow = smem + G_::OFF_Q;
        const bool lead = warp == 4 && lane == 0;
        float m = -INFINITY, l = 0.f;
        float A_cur = 0.f, A_done = 0.f;   // this half's group sums A_{t,g} (reference m)
        int64_t g_cur = -1, g_done = -1;
        int sc0 = 0, sc1 = 0;              // S-type ops seen per buffer (s_full parity)
        int nf = 0;                        // F ops seen (exchange slot parity)
        // pv_done[wg][b] completes once per op on buffer b (ops b, b+2, ...); seen* = last op
        // whose completion was consumed.  Before releasing P of op n, op n-2 is consumed.
        int seen0 = -2, seen1 = -1;
        auto consume_op = [&](int op) {
            if (op < 0) return;
            if (op & 1) {
                while (seen1 < op) { seen1 += 2; mbar_wait_c(&ctl.pv_done[wg][1], (seen1 >> 1) & 1, spin); }
            } else {
                while (seen0 < op) { seen0 += 2; mbar_wait_c(&ctl.pv_done[wg][0], (seen0 >> 1) & 1, spin); }
            }
        };
        const int64_t n_last = NK - 1;
        const int nlast_len = (int)(p.S - n_last * 64);
        const float cs = p.scale_log2;   // logits in log2 units: x = S * s * log2(e)
        for (int n = 0; n < nops; ++n) {
            const int s = n & 1;
            const int32_t op = op_at(n);
            const int type = op_type(op), v = op_val(op);
            const uint32_t t_buf = tbase + lane_off + kColS + 128 * s;
            if (type != OP_F) {
                const int par = (s ? sc1 : sc0) & 1;
                if (s) ++sc1; else ++sc0;
                if (lead) PASA_TR(TR_SA_W, n);
                mbar_wait_c(&ctl.s_full[s], par, spin);
                if (lead) PASA_TR(TR_SA_OK, n);
                tc_fence_after();
                if (!(p.dbg & 1)) {
                uint32_t sa[32], sb[32];
                tmem_ld32(t_buf + 64 * wg, sa);
                tmem_ld32(t_buf + 64 * wg + 32, sb);
                tmem_wait_ld();
                if (lead) PASA_TR(TR_SA_LD, n);
                // valid columns of this half and denominator weights
                uint64_t valid;
                float wlast = 1.f;     // token count of block n_last (C ops)
                int clast = -1;        // column of block n_last in this half (C ops)
                int64_t j0 = 0;        // first centroid of this half (C ops)
                if (type == OP_E) {
                    const int q = 2 * v + wg;
                    if (q < cnt) {
                        const int j = ctl.eidx[q];
                        const int nj = j == n_last ? nlast_len : 64;
                        valid = nj >= 64 ? ~0ull : ((1ull << nj) - 1ull);
                    } else {
                        valid = 0ull;          // odd count: the pair's 2nd block is absent
                    }
                } else {
                    j0 = 128 * (int64_t)v + 64 * wg;
                    const int w0 = (int)(j0 >> 5);
                    const uint64_t kept = (w0 < W ? (uint64_t)ctl.mask[w0] : ~0ull) |
                                          (w0 + 1 < W ? (uint64_t)ctl.mask[w0 + 1] << 32
                                                      : 0xffffffff00000000ull);
                    const int64_t rem = NK - j0;
                    const uint64_t inb = rem >= 64 ? ~0ull : (rem <= 0 ? 0ull : ((1ull << rem) - 1ull));
                    valid = ~kept & inb;
                    if (rem >= 1 && rem <= 64) { clast = (int)(rem - 1); wlast = (float)nlast_len; }
                }
                if (valid != 0ull) {
                if (valid != ~0ull) {   // masked columns -> -inf (ragged / kept blocks)
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        if (!((valid >> c) & 1ull)) sa[c] = 0xff800000u;
                        if (!((valid >> (c + 32)) & 1ull)) sb[c] = 0xff800000u;
                    }
                }
                float mr0 = -INFINITY, mr1 = -INFINITY;   // raw row max (scale > 0 commutes)
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    mr0 = fmax3(mr0, __uint_as_float(sa[c]), __uint_as_float(sa[c + 1]));
                    mr1 = fmax3(mr1, __uint_as_float(sb[c]), __uint_as_float(sb[c + 1]));
                }
                const float mx = fmaxf(mr0, mr1) * cs;
                if (lead) PASA_TR(TR_SA_MAX, n);
                float xlast = -INFINITY;   // raw logit of the ragged last block (C ops)
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
                    corr = ex2(m - mx);          // 0 when m = -inf
                    resc = m != -INFINITY;       // O_wg holds earlier contributions
                    m = mx;
                    l *= corr;
                    A_cur *= corr;
                    A_done *= corr;
                }
                if (__any_sync(0xffffffffu, resc)) {
                    consume_op(n - 2);
                    consume_op(n - 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c0 = 0; c0 < D; c0 += 32) {
                        uint32_t o[32];
                        tmem_ld32(t_own + c0, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                        tmem_st32(t_own + c0, o);
                    }
                }
                float h0 = 0.f, h1 = 0.f;
                uint32_t pk[32];
                const float negm = -m;
                // a quarter of the exponentials run as a polynomial on the FMA pipe
                // (ex2_poly, rel. error < 9e-5), the rest on MUFU
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const bool poly = (c & 1) == 1;
                    const float x0 = fmaf(__uint_as_float(sa[2 * c]), cs, negm);
                    const float x1 = fmaf(__uint_as_float(sa[2 * c + 1]), cs, negm);
                    const float x2 = fmaf(__uint_as_float(sb[2 * c]), cs, negm);
                    const float x3 = fmaf(__uint_as_float(sb[2 * c + 1]), cs, negm);
                    const float p0 = ex2(x0);
                    const float p1 = poly ? ex2_poly(x1) : ex2(x1);
                    const float p2 = ex2(x2);
                    const float p3 = poly ? ex2_poly(x3) : ex2(x3);
                    h0 += p0 + p1;
                    h1 += p2 + p3;
                    pk[c] = pack_bf16(p0, p1);
                    pk[16 + c] = pack_bf16(p2, p3);
                }
                tmem_st32(t_buf + 64 * wg, pk);
                if (lead) PASA_TR(TR_SA_EXP, n);
                if (type == OP_E) {
                    l += h0 + h1;
                } else {
                    // denominator: n_j * p_j; every dropped block has 64 tokens except the last
                    const float pl = clast >= 0 ? ex2(fmaf(xlast, cs, negm)) : 0.f;
                    l += 64.f * (h0 + h1) - (64.f - wlast) * pl;
                    // group sums (each 32-block word lies in one group)
#pragma unroll
                    for (int hw = 0; hw < 2; ++hw) {
                        const int64_t jw = j0 + 32 * hw;
                        if (jw >= NK) break;
                        const int64_t g = jw / p.G;
                        const float hv = hw ? h1 : h0;
                        if (g != g_cur) { A_done = A_cur; g_done = g_cur; A_cur = hv; g_cur = g; }
                        else A_cur += hv;
                    }
                }
                } else {
                    // nothing of this half is live (absent block / all kept): P = 0
                    uint32_t z[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) z[c] = 0u;
                    tmem_st32(t_buf + 64 * wg, z);
                }
                tmem_wait_st();
                if (lead) PASA_TR(TR_SA_ST, n);
                }
            } else if (!(p.dbg & 1)) {
                // F(g): the group sum is this half's part plus the partner's, both brought to
                // warpgroup 0's reference max (the F MMA accumulates into O_0); each half then
                // writes D/2 dims of Aq = bf16(s * A_{t,g} * q_t) at its own column 64wg.
                const float part = v == g_cur ? A_cur : (v == g_done ? A_done : 0.f);
                float* xa = &ctl.xchg[nf & 1][0][0][0];
                float* xmx = &ctl.xchg[nf & 1][1][0][0];
                ++nf;
                xa[wg * kBQ + r] = part;
                xmx[wg * kBQ + r] = m;
                bar_sync(bar_id, 64);
                const float a_o = xa[(wg ^ 1) * kBQ + r], m_o = xmx[(wg ^ 1) * kBQ + r];
                const float a0 = wg == 0 ? part : a_o, a1 = wg == 0 ? a_o : part;
                const float m0 = wg == 0 ? m : m_o, m1 = wg == 0 ? m_o : m;
                const float a_tot = a1 != 0.f ? fmaf(a1, ex2(m1 - m0), a0) : a0;
                const float w = p.s * a_tot;
                const uint32_t w2 = pack_bf16(w, w);
                consume_op(n - 2);     // this half's previous reader of the buffer has finished
                tc_fence_after();
                uint32_t aq[DH / 2];
                const uint8_t* qb = qrow + (wg * DH / 64) * (kBQ * 128) + r * 128;
#pragma unroll
                for (int c = 0; c < DH / 8; ++c) {
                    const int chunk = (wg * DH % 64) / 8 + c;   // 16-byte chunk in the 128-B row
                    const uint4 qv = *reinterpret_cast<const uint4*>(qb + ((chunk ^ (r & 7)) << 4));
                    aq[c * 4 + 0] = hmul2_bf16(qv.x, w2);
                    aq[c * 4 + 1] = hmul2_bf16(qv.y, w2);
                    aq[c * 4 + 2] = hmul2_bf16(qv.z, w2);
                    aq[c * 4 + 3] = hmul2_bf16(qv.w, w2);
                }
                if constexpr (DH == 64) tmem_st32(t_buf + 64 * wg, aq);
                else tmem_st16(t_buf + 64 * wg, aq);
                tmem_wait_st();
            }
            consume_op(n - 2);
            tc_fence_before();
            mbar_arrive(&ctl.p_full[wg][s]);
            if (lead) PASA_TR(TR_SA_ARR, n);
        }
        // ---- epilogue: merge the two halves, O = (O_0 e0 + O_1 e1) / (l0 e0 + l1 e1) ----
        if (nops > 0) {
            consume_op(nops - 2);
            consume_op(nops - 1);
            float* xl = &ctl.xchg[nf & 1][0][0][0];
            float* xm = &ctl.xchg[nf & 1][1][0][0];
            xl[wg * kBQ + r] = l;
            xm[wg * kBQ + r] = m;
            bar_sync(bar_id, 64);
            // the partner's last MMAs completed too (it passed its own consume before the barrier)
            tc_fence_after();
            const float l_o = xl[(wg ^ 1) * kBQ + r], m_o = xm[(wg ^ 1) * kBQ + r];
            const float l0 = wg == 0 ? l : l_o, l1 = wg == 0 ? l_o : l;
            const float m0 = wg == 0 ? m : m_o, m1 = wg == 0 ? m_o : m;
            const float mm = fmaxf(m0, m1);
            const float e0 = m0 == -INFINITY ? 0.f : ex2(m0 - mm);
            const float e1 = m1 == -INFINITY ? 0.f : ex2(m1 - mm);
            const float inv = 1.f / fmaf(l0, e0, l1 * e1);
            const float f0 = e0 * inv, f1 = e1 * inv;
            const int64_t tok = i * kBQ + r;
            __nv_bfloat16* orow = p.out + b * p.osB + h * p.osH + tok * p.osS + wg * DH;
            const uint32_t t_rows = tbase + lane_off;
#pragma unroll 1
            for (int c0 = 0; c0 < DH; c0 += 32) {
                uint32_t o0[32], o1[32];
                tmem_ld32(t_rows + wg * DH + c0, o0);          // O_0
                tmem_ld32(t_rows + 128 + wg * DH + c0, o1);    // O_1
                tmem_wait_ld();
                if (tok < p.S) {
                    uint4 pkt[4];
                    uint32_t* pw = reinterpret_cast<uint32_t*>(pkt);
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        pw[c] = pack_bf16(
                            fmaf(__uint_as_float(o0[2 * c]), f0, __uint_as_float(o1[2 * c]) * f1),
                            fmaf(__uint_as_float(o0[2 * c + 1]), f0, __uint_as_float(o1[2 * c + 1]) * f1));
#pragma unroll
                    for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(orow + c0)[q] = pkt[q];
                }
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
    prm.S = r->S; prm.H = r->H; prm.NQ = r->NQ; prm.NK = r->NK; prm.NG = r->NG; prm.W = r->W;
    prm.G = r->cfg.G; prm.comp = r->cfg.comp;
    const double s = 1.0 / sqrt((double)D);
    prm.s = (float)s;
    prm.scale_log2 = (float)(s * 1.4426950408889634);
    prm.idx = r->idx; prm.count = r->count; prm.mask = r->mask;
    prm.out = reinterpret_cast<__nv_bfloat16*>(out.data);
    prm.osB = out.sB; prm.osS = out.sS; prm.osH = out.sH;
    prm.trace = g_trace_buf;
    prm.trace_x = g_trace_x;
    prm.trace_y = g_trace_y;
    prm.dbg = g_dbg;
    // one CTA per SM (it owns all 512 TMEM columns)
    const size_t smem = (size_t)Geo<D>::BYTES + 1024;
    auto kern = attn_pair_kernel<D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)r->NQ, (unsigned)r->BH);
    kern<<<grid, kThreads, smem, st>>>(mQ, mK, mV, mKb, mVs, mHt, prm);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100_pair(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                              pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                              int* launches, char* why, size_t why_len) {
    if (r->cfg.Bq != kBQ || r->cfg.Bk != kBK) {
        snprintf(why, why_len, "needs Bq=128, Bk=64");
        return cudaErrorNotSupported;
    }
    if (r->cfg.comp == PASA_COMP_GROUPED && !sm100_supports_group(r->cfg.G, r->NK)) {
        snprintf(why, why_len, "grouped compensation needs G in {32, 64}, G %% 128 == 0 or "
                 "G >= N_K (G=%d)", r->cfg.G);
        return cudaErrorNotSupported;
    }
    if (r->W > 64) {
        snprintf(why, why_len, "N_K > 2048");
        return cudaErrorNotSupported;
    }
    cudaError_t e = r->D == 128 ? launch_d<128>(q, k, v, r, out, st, why, why_len)
                                : launch_d<64>(q, k, v, r, out, st, why, why_len);
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace pasa

