// ATTIC -- NOT BUILT.  Round 2's persistent dual-tile kernel, parity-green (81 GPU parity
// tests through the C ABI while it was the default) and measured slower than the two-CTA
// kernel it was meant to replace: Wan-14B 23.2-23.9 vs 22.4-22.7 ms, CogVideoX 1.40 vs
// 1.16 ms.  Why, with the clock64 timeline and ncu evidence: profiles/r02_attn_dual.md.
// It includes csrc/pasa_internal.h and csrc/sm100_ptx.cuh; to rebuild it, copy it back to
// paper_2604_12219_b200/csrc/ and restore its dispatch (git history, round 2).
// attn_sm100_dual.cu -- pasa_attn on the Blackwell tensor cores (sm_100a), the default
// tcgen05 kernel since round 2: persistent, one CTA per SM, TWO independent query tiles
// per CTA, kept KV blocks processed in pairs (N = 128 keys per MMA).  Same method as
// attn_sm100.cu -- gather-driven block-sparse attention with the PASA compensation
// folded into the same online softmax (Eq. 7; grouped first-order
// term, PAPER.md:310-313 and App. B :503-506; readings R-1..R-5, R-21, R-22 in DESIGN.md
// §3) -- with a B200-first schedule:
//
//   * N = 128 QK^T tiles: an M128 x N128 x K16 SS MMA reads 8 KB of shared memory per
//     64 tensor cycles (balanced), where the N = 64 tile of the two-CTA kernel reads
//     6 KB per 32 (shared-memory bound, 48 cycles).
//   * two query tiles (two (head, q-block) items, each with its own route) per CTA, each
//     with its own softmax warpgroup, O accumulator and S/P buffer in TMEM
//     (O_0 | O_1 | S_0 | S_1 = 512 columns at d = 128): while warpgroup t turns S_t into
//     P_t, the tensor pipe runs tile 1-t's PV and QK^T.  No state is shared between the
//     two softmax chains (round 1's ping-pong variants handed the running max along).
//   * persistent: 2 x 148 tile slots walk the (head, q-block) items head-major, so one
//     head's K/V stay in L2 while ~296 of its q-blocks gather from them; TMEM, barriers
//     and tensor maps are set up once per CTA.
//
// Per tile the op list of an item is E(pair e) for e < ceil(count/2) (kept blocks
// idx[2e], idx[2e+1]; an odd count repeats the last block, masked), then the
// compensation tail: C(c) for every 128-centroid chunk holding a dropped block, each
// followed by F(g) for the groups ending in it that hold a dropped block.
//   E / C :  S_t = Q_t K^T (SS)  ->  softmax  ->  P_t (bf16, S_t[0:64))  ->  O_t += P_t V (TS)
//   F(g)  :  Aq = bf16(s A_{t,g} q_t) into S_t[64:) or S_t[0:) (alternating)  ->
//            O_t += Aq Hbar^(g)  (TS, Hbar^T tile through the K or V slot, alternating)
// Warp roles (384 threads):
//   warp 0 / 2   producer of tile 0 / 1: builds the item's op list (lane-parallel from the
//                route mask), then TMA loads Q, K / V pairs, Kbar / Vsum chunks, Hbar^T
//   warp 1       TMEM allocator + tcgen05.mma issuer for both tiles (strict alternation)
//   warp 3       idle
//   warps 4-7    softmax / epilogue of tile 0 (one query row per thread)
//   warps 8-11   softmax / epilogue of tile 1
// Domain: bf16 I/O, Bq = 128, Bk = 64, d in {64, 128}, N_K <= 4096, comp NONE / ZEROTH /
// GROUPED with G in {32, 64, multiples of 128, >= N_K}; other G use attn_sm100.cu.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "pasa_internal.h"
#include "sm100_ptx.cuh"

namespace pasa {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
constexpr int kBQ = 128, kBK = 64, kN = 128;   // query rows, key block, keys per op
constexpr int kMaxW = 128;                       // mask words: N_K <= 4096
constexpr int kMaxChunks = 32;                   // 128-centroid chunks: N_K <= 4096
constexpr int kMaxTail = kMaxChunks + 128;       // C ops + F ops (G >= 32)
constexpr float kRescaleThresh = 8.f;            // log2 units (R-22)
constexpr int kPolyDefault = 0;                  // column pairs of every 4 on the FMA pipe

enum : int { OP_E = 0, OP_C = 1, OP_F = 2 };
__device__ __forceinline__ int op_type(int op) { return op >> 14; }
__device__ __forceinline__ int op_val(int op) { return op & 0x3FFF; }

template <int D>
struct Geo {
    static constexpr int NBOX = D / 64;            // 64-column boxes along d
    static constexpr int QBYTES = kBQ * D * 2;     // one query tile
    static constexpr int DBOX = kN * 128;          // one 64-column box of a 128-row tile
    static constexpr int SLOT = kN * D * 2;        // K or V slot: 128 rows x d
    static constexpr int DEPTH = D == 128 ? 1 : 2; // slots per tile and sequence
    static constexpr int OFF_K = 2 * QBYTES;       // Q_0 | Q_1 | K[t][DEPTH] | V[t][DEPTH]
    static constexpr int OFF_V = OFF_K + 2 * DEPTH * SLOT;
    static constexpr int BYTES = OFF_V + 2 * DEPTH * SLOT;
    static constexpr int HTBYTES = D * D * 2;      // Hbar^T of one group
    static constexpr uint32_t COL_S = 2 * D;       // TMEM: O_t at t*D, S_t at COL_S + 128 t
    static_assert(HTBYTES <= SLOT, "an Hbar^T tile must fit one slot");
};

struct Params {
    int64_t S, H, NQ, NK, NG, W, idx_ld;
    int64_t U;                  // items = B*H*N_Q
    int32_t G, comp;
    float scale_log2;           // s * log2(e)
    float s;                    // 1/sqrt(D)
    const int32_t* idx;
    const int32_t* count;
    const uint32_t* mask;
    int32_t* work;              // item counter (zeroed before the launch): dynamic schedule
    __nv_bfloat16* out;
    int64_t osB, osS, osH;
    int32_t dbg;                // ablations (timing only, results meaningless): 256 = the
                                // softmax skips its math, 512 = the producers skip the TMA loads;
                                // 1024 = critical-path waits poll instead of suspending
    unsigned long long* trace;  // diagnostics: clock64 timeline of CTA trace_cta, or nullptr
    int32_t trace_cta;
};

// timeline events (pasa_debug_trace with pasa_debug_flags bit 2048): slot
// ((ev * 2 + tile) * kTraceN + op index of the tile in this CTA)
constexpr int kTraceN = 4096;
enum { TD_MMA_PW = 0, TD_MMA_PO, TD_MMA_ISS, TD_MMA_QK, TD_SM_SW, TD_SM_SO, TD_SM_AR, TD_SM_FW,
       TD_SM_FO, TD_NEV };

// one item's op list, written by the tile's producer, read by the MMA warp and the
// softmax warpgroup (ring of two per tile: item_full / item_empty)
struct ItemSlot {
    int64_t u;                  // bh * N_Q + i, or -1: no more items for this tile
    int32_t cnt, nE, ntail, last_ragged;
    uint32_t mask[kMaxW];
    uint16_t tail[kMaxTail];
};

struct Ctl {
    uint64_t q_full[2], q_empty[2];
    uint64_t k_full[2][2], k_empty[2][2], v_full[2][2], v_empty[2][2];   // [tile][slot]
    uint64_t s_full[2];
    uint64_t p_full[2][2], mma_done[2][2];                               // [tile][op & 1]
    uint64_t item_full[2][2], item_empty[2][2];                          // [tile][item & 1]
    uint32_t tmem_base;
    ItemSlot items[2][2];
};

__device__ __forceinline__ int op_at(const ItemSlot& it, int n) {
    return n < it.nE ? ((OP_E << 14) | n) : (int)it.tail[n - it.nE];
}

template <int D, int POLY>
__global__ void __launch_bounds__(kThreads, 1)
    attn_dual_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmKb,
                     const __grid_constant__ CUtensorMap tmVs, const __grid_constant__ CUtensorMap tmHt,
                     const Params p) {
    using G_ = Geo<D>;
    constexpr int DEPTH = G_::DEPTH;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ Ctl ctl;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool tracing = p.trace != nullptr && (int)blockIdx.x == p.trace_cta;
    const bool spin = (p.dbg & 1024) != 0;
#define PASA_TD(ev, tt, ix)                                                                   \
    do {                                                                                      \
        if (tracing && (ix) < kTraceN) p.trace[((ev) * 2 + (tt)) * kTraceN + (ix)] = clock64(); \
    } while (0)
    const int64_t NK = p.NK, NQ = p.NQ;
    const int W = (int)p.W;

    if (tid == 0) {
        for (int t = 0; t < 2; ++t) {
            mbar_init(&ctl.q_full[t], 1);
            mbar_init(&ctl.q_empty[t], 128);
            mbar_init(&ctl.s_full[t], 1);
            for (int s = 0; s < 2; ++s) {
                mbar_init(&ctl.k_full[t][s], 1);
                mbar_init(&ctl.k_empty[t][s], 1);
                mbar_init(&ctl.v_full[t][s], 1);
                mbar_init(&ctl.v_empty[t][s], 1);
                mbar_init(&ctl.p_full[t][s], 128);
                mbar_init(&ctl.mma_done[t][s], 1);
                mbar_init(&ctl.item_full[t][s], 1);
                mbar_init(&ctl.item_empty[t][s], 1 + 128);   // MMA warp + softmax warpgroup
            }
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(&ctl.tmem_base, 512);
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

    // register budgets (setmaxnreg at the top of each role): the producer / MMA warpgroup
    // gives registers to the two softmax warpgroups (128 x 80 + 256 x 208 = 63,488 of 65,536)
    if (warp == 0 || warp == 2) {
        setmaxnreg_dec<80>();
        // ============================ producer of tile t ============================
        // Items are handed out dynamically in (head, q-block) order from one counter, so
        // the ~296 q-blocks in flight stay inside one or two heads (their K/V in L2) however
        // the tiles drift.
        const int t = warp >> 1;
        const int nchunks = (int)((NK + 127) / 128);
        int kc = 0, vc = 0;   // loads issued into the K / V slot sequence
        for (int r = 0;; ++r) {
            ItemSlot& it = ctl.items[t][r & 1];
            mbar_wait_sleep(&ctl.item_empty[t][r & 1], ((r >> 1) & 1) ^ 1);
            int64_t u = 0;
            if (lane == 0) u = atomicAdd(p.work, 1);
            u = __shfl_sync(0xffffffffu, u, 0);
            if (u >= p.U) u = -1;
            if (u < 0) {
                if (lane == 0) {
                    it.u = -1;
                    mbar_arrive(&ctl.item_full[t][r & 1]);
                }
                break;
            }
            // ---- op list of item u (lane c looks after 128-centroid chunk c) ----
            const int cnt = p.count[u];
            for (int w = lane; w < W; w += 32) it.mask[w] = p.mask[u * W + w];
            __syncwarp();
            auto dropped_word = [&](int w) {
                const int64_t rem = NK - 32 * (int64_t)w;
                const uint32_t inb = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
                return (~it.mask[w] & inb) != 0u;
            };
            const int c = lane;
            bool cf = false;                      // chunk c holds a dropped block
            if (c < nchunks)
                for (int w = 4 * c; w < min(4 * c + 4, W); ++w) cf |= dropped_word(w);
            const uint32_t cmask = __ballot_sync(0xffffffffu, cf);
            int nmine = 0;
            uint16_t mine[5];
            if (p.comp != PASA_COMP_NONE && cnt < NK && c < nchunks) {
                if (cf) mine[nmine++] = (uint16_t)((OP_C << 14) | c);
                if (p.comp == PASA_COMP_GROUPED) {
                    const int64_t G = p.G;
                    if (G == 32 || G == 64) {          // 4 or 2 groups per chunk, one or two words each
                        const int per = (int)(128 / G), wpg = (int)(G / 32);
                        for (int q = 0; q < per; ++q) {
                            const int g = per * c + q;
                            if ((int64_t)g * G >= NK) break;
                            bool any = false;
                            for (int w = g * wpg; w < min((g + 1) * wpg, W); ++w) any |= dropped_word(w);
                            if (any) mine[nmine++] = (uint16_t)((OP_F << 14) | g);
                        }
                    } else {                           // G % 128 == 0 or one global group
                        const int64_t g = (128 * (int64_t)c) / G;
                        const int c0 = (int)(g * G / 128);
                        const int c1 = (int)((min((g + 1) * G, NK) - 1) / 128);
                        if (c == c1) {
                            const uint32_t span = (c1 - c0 == 31) ? 0xffffffffu
                                                                   : (((1u << (c1 - c0 + 1)) - 1u) << c0);
                            if (cmask & span) mine[nmine++] = (uint16_t)((OP_F << 14) | (int)g);
                        }
                    }
                }
            }
            int off = nmine;                       // inclusive prefix sum over the lanes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, off, o);
                if (lane >= o) off += y;
            }
            const int ntail = __shfl_sync(0xffffffffu, off, 31);
            for (int q = 0; q < nmine; ++q) it.tail[off - nmine + q] = mine[q];
            if (lane == 0) {
                it.u = u;
                it.cnt = cnt;
                it.nE = (cnt + 1) >> 1;
                it.ntail = ntail;
                it.last_ragged = (p.S % kBK != 0) && p.idx[u * p.idx_ld + cnt - 1] == NK - 1;
            }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl.item_full[t][r & 1]);

            // ---- loads ----
            if (lane == 0) {
                const int64_t bh = u / NQ, i = u % NQ;
                const int b = (int)(bh / p.H), h = (int)(bh % p.H);
                if (r > 0) mbar_wait_sleep(&ctl.q_empty[t], (r - 1) & 1);
                uint8_t* qdst = smem + t * G_::QBYTES;
                const bool noload = (p.dbg & 512) != 0;
                if (noload) {
                    mbar_arrive(&ctl.q_full[t]);
                } else {
                    mbar_arrive_expect_tx(&ctl.q_full[t], G_::QBYTES);
#pragma unroll
                    for (int a = 0; a < G_::NBOX; ++a)
                        tma_load_4d(qdst + a * (kBQ * 128), &tmQ, &ctl.q_full[t], 64 * a, (int)(i * kBQ), h, b);
                }
                const int32_t* irow = p.idx + u * p.idx_ld;
                const int nE = (cnt + 1) >> 1, nops = nE + ntail;
                int frun = 0;
                for (int n = 0; n < nops; ++n) {
                    const int op = n < nE ? ((OP_E << 14) | n) : (int)it.tail[n - nE];
                    const int type = op_type(op), v = op_val(op);
                    if (type != OP_F) {
                        int j0 = 0, j1 = 0;
                        if (type == OP_E) {
                            j0 = irow[2 * v];
                            j1 = irow[min(2 * v + 1, cnt - 1)];   // odd count: repeat, masked
                        }
                        for (int kv = 0; kv < 2; ++kv) {
                            const int cq = kv == 0 ? kc++ : vc++;
                            const int s = cq % DEPTH;
                            uint64_t* full = kv == 0 ? &ctl.k_full[t][s] : &ctl.v_full[t][s];
                            mbar_wait_sleep(kv == 0 ? &ctl.k_empty[t][s] : &ctl.v_empty[t][s],
                                            ((cq / DEPTH) & 1) ^ 1);
                            uint8_t* dst = smem + (kv == 0 ? G_::OFF_K : G_::OFF_V) + (t * DEPTH + s) * G_::SLOT;
                            if (noload) { mbar_arrive(full); continue; }
                            mbar_arrive_expect_tx(full, G_::SLOT);
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                                for (int a = 0; a < G_::NBOX; ++a) {
                                    uint8_t* d2 = dst + a * G_::DBOX + hh * (kBK * 128);
                                    if (type == OP_E)
                                        tma_load_4d(d2, kv == 0 ? &tmK : &tmV, full, 64 * a,
                                                    (hh ? j1 : j0) * kBK, h, b);
                                    else
                                        tma_load_3d(d2, kv == 0 ? &tmKb : &tmVs, full, 64 * a,
                                                    v * kN + hh * 64, (int)bh);
                                }
                        }
                        frun = 0;
                    } else {
                        // Hbar^T of group v through the K slot (odd F ops of a run: V slot)
                        const int kv = frun & 1;
                        ++frun;
                        const int cq = kv == 0 ? kc++ : vc++;
                        const int s = cq % DEPTH;
                        uint64_t* full = kv == 0 ? &ctl.k_full[t][s] : &ctl.v_full[t][s];
                        mbar_wait_sleep(kv == 0 ? &ctl.k_empty[t][s] : &ctl.v_empty[t][s],
                                        ((cq / DEPTH) & 1) ^ 1);
                        uint8_t* dst = smem + (kv == 0 ? G_::OFF_K : G_::OFF_V) + (t * DEPTH + s) * G_::SLOT;
                        if (noload) { mbar_arrive(full); continue; }
                        mbar_arrive_expect_tx(full, G_::HTBYTES);
#pragma unroll
                        for (int a = 0; a < G_::NBOX; ++a)
                            tma_load_3d(dst + a * (D * 128), &tmHt, full, 64 * a, v * D, (int)bh);
                    }
                }
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        setmaxnreg_dec<80>();
        // ====================== MMA issuer (both tiles, alternating) ======================
        // tcgen05.mma issue blocks while the tensor pipe's queue is full, so the issuer is busy
        // for about as long as its MMAs run; strict alternation between the tiles staggers
        // their softmaxes (measured: one issuer per tile, a ready-driven order, or chaining a
        // tile's ready F ops all let the two softmaxes run together and contend for MUFU).
        constexpr uint32_t kIdQK = idesc_bf16_f32(128, kN, 0, 0);   // Q (K-major) x K^T (K-major)
        constexpr uint32_t kIdPV = idesc_bf16_f32(128, D, 0, 1);    // P (TMEM) x V (MN-major)
        constexpr uint32_t kIdF = idesc_bf16_f32(128, D, 0, 0);     // Aq (TMEM) x Hbar^T (K-major)
        const uint32_t sbase = smem_u32(smem);
        int r[2] = {0, 0}, n[2] = {0, 0}, gn[2] = {0, 0}, kc[2] = {0, 0}, vc[2] = {0, 0};
        int frun[2] = {0, 0};
        bool pend[2] = {true, true}, done[2] = {false, false};
        const ItemSlot* cur[2] = {nullptr, nullptr};
        auto issue_qk = [&](int t) {
            const int s = kc[t] % DEPTH;
            mbar_wait_c(&ctl.k_full[t][s], (kc[t] / DEPTH) & 1, spin);
            tc_fence_after();
            const uint32_t qa = sbase + t * G_::QBYTES;
            const uint32_t ka = sbase + G_::OFF_K + (t * DEPTH + s) * G_::SLOT;
            const uint32_t d = tbase + G_::COL_S + 128 * t;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t oq = (kk >> 2) * (kBQ * 128) + (kk & 3) * 32;
                const uint32_t ok = (kk >> 2) * G_::DBOX + (kk & 3) * 32;
                mma_ss_elect(d, umma_desc_sw128(qa + oq, 16, 1024), umma_desc_sw128(ka + ok, 16, 1024),
                             kIdQK, kk > 0);
            }
            mma_commit_elect(&ctl.s_full[t]);
            mma_commit_elect(&ctl.k_empty[t][s]);
            ++kc[t];
            __syncwarp();
        };
        // issue the MMAs of op n[t] of tile t (its p_full and operand slot are ready)
        auto issue_op = [&](int t, int op) {
            const uint32_t tO = tbase + t * D, tS = tbase + G_::COL_S + 128 * t;
            if (op_type(op) != OP_F) {
                const int s = vc[t] % DEPTH;
                mbar_wait_c(&ctl.v_full[t][s], (vc[t] / DEPTH) & 1, spin);
                tc_fence_after();
                const uint32_t va = sbase + G_::OFF_V + (t * DEPTH + s) * G_::SLOT;
                const uint64_t dv = umma_desc_sw128(va, G_::DBOX, 1024);
#pragma unroll
                for (int kk = 0; kk < kN / 16; ++kk)
                    mma_ts_elect(tO, tS + kk * 8, dv + ((kk * 16 * 128) >> 4), kIdPV,
                                 (n[t] > 0 || kk > 0) ? 1u : 0u);
                mma_commit_elect(&ctl.v_empty[t][s]);
                ++vc[t];
                frun[t] = 0;
            } else {
                const int kv = frun[t] & 1;
                const uint32_t acol = kv == 0 ? 64u : 0u;   // Aq half (see softmax)
                ++frun[t];
                const int cq = kv == 0 ? kc[t]++ : vc[t]++;
                const int s = cq % DEPTH;
                mbar_wait_c(kv == 0 ? &ctl.k_full[t][s] : &ctl.v_full[t][s], (cq / DEPTH) & 1, spin);
                tc_fence_after();
                const uint32_t ha = sbase + (kv == 0 ? G_::OFF_K : G_::OFF_V) + (t * DEPTH + s) * G_::SLOT;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t oh = (kk >> 2) * (D * 128) + (kk & 3) * 32;
                    mma_ts_elect(tO, tS + acol + kk * 8, umma_desc_sw128(ha + oh, 16, 1024), kIdF, 1u);
                }
                mma_commit_elect(kv == 0 ? &ctl.k_empty[t][s] : &ctl.v_empty[t][s]);
            }
            mma_commit_elect(&ctl.mma_done[t][gn[t] & 1]);
            __syncwarp();
            if (lane == 0) PASA_TD(TD_MMA_ISS, t, gn[t]);
            ++gn[t];
            ++n[t];
        };
        // after op n[t]-1: end the item, or issue the next QK^T
        auto advance = [&](int t) -> bool {   // true: the tile can continue with an F op
            const ItemSlot& it = *cur[t];
            if (n[t] == it.nE + it.ntail) {
                if (lane == 0) mbar_arrive(&ctl.item_empty[t][r[t] & 1]);
                __syncwarp();
                ++r[t];
                n[t] = 0;
                pend[t] = true;
                return false;
            }
            if (op_type(op_at(it, n[t])) != OP_F) {
                issue_qk(t);
                if (lane == 0) PASA_TD(TD_MMA_QK, t, gn[t]);
                return false;
            }
            return true;
        };
        while (!(done[0] && done[1])) {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                if (done[t]) continue;
                if (pend[t]) {
                    // next item: op list, its Q tile, then the first QK^T; return to the other
                    // tile before waiting for this one's softmax
                    mbar_wait_sleep(&ctl.item_full[t][r[t] & 1], (r[t] >> 1) & 1);
                    cur[t] = &ctl.items[t][r[t] & 1];
                    if (cur[t]->u < 0) { done[t] = true; continue; }
                    mbar_wait_sleep(&ctl.q_full[t], r[t] & 1);
                    issue_qk(t);
                    pend[t] = false;
                    continue;
                }
                if (lane == 0) PASA_TD(TD_MMA_PW, t, gn[t]);
                mbar_wait_c(&ctl.p_full[t][gn[t] & 1], (gn[t] >> 1) & 1, spin);
                if (lane == 0) PASA_TD(TD_MMA_PO, t, gn[t]);
                tc_fence_after();
                issue_op(t, op_at(*cur[t], n[t]));
                advance(t);
            }
        }
    } else if (warp == 3) {
        setmaxnreg_dec<80>();
    } else {
        setmaxnreg_inc<208>();
        // ================= softmax / first-order operand / epilogue of tile t =================
        const int t = (warp - 4) >> 2;
        const int row = (warp & 3) * 32 + lane;                  // query row in the tile
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tbase + lane_off + G_::COL_S + 128 * t;
        const uint32_t tO = tbase + lane_off + t * D;
        const uint8_t* qrow = smem + t * G_::QBYTES;
        const float cs = p.scale_log2;
        const float2 cs2 = make_float2(cs, cs);
        const int NK32 = (int)NK;
        const int nlast_len = (int)(p.S - (NK - 1) * kBK);
        const int G32 = p.G;
        int gn = 0, ns = 0;
        for (int r = 0;; ++r) {
            mbar_wait_sleep(&ctl.item_full[t][r & 1], (r >> 1) & 1);
            const ItemSlot& it = ctl.items[t][r & 1];
            const int64_t u = it.u;
            if (u < 0) break;
            const int cnt = it.cnt, nE = it.nE, nops = it.nE + it.ntail;
            const bool last_ragged = it.last_ragged != 0;
            float m = -INFINITY, l = 0.f;
            float A4[4] = {0.f, 0.f, 0.f, 0.f};   // G = 32 / 64: group sums of the last C op
            float A_acc = 0.f;                     // G >= 128: running sum of the current group
            int g_cur = -1, c_last = 0, frun = 0;
            for (int n = 0; n < nops; ++n, ++gn) {
                const int op = op_at(it, n);
                const int type = op_type(op), v = op_val(op);
                if (type != OP_F && (p.dbg & 256)) {
                    mbar_wait_sleep(&ctl.s_full[t], ns & 1);
                    ++ns;
                    frun = 0;
                } else if (type != OP_F) {
                    if (row == 0) PASA_TD(TD_SM_SW, t, gn);
                    mbar_wait_c(&ctl.s_full[t], ns & 1, spin);
                    if (row == 0) PASA_TD(TD_SM_SO, t, gn);
                    ++ns;
                    tc_fence_after();
                    // valid columns: E -- the repeated block of an odd count, the ragged last
                    // block; C -- dropped blocks inside N_K (R-7: true lengths)
                    uint64_t vlo = ~0ull, vhi = ~0ull;
                    int clast = -1;
                    if (type == OP_E) {
                        if (v == nE - 1) {
                            if (cnt & 1) vhi = 0ull;
                            if (last_ragged) {
                                const uint64_t rm = (1ull << nlast_len) - 1ull;
                                if (((cnt - 1) & 1) == 0) vlo = rm; else vhi = rm;
                            }
                        }
                    } else {
                        uint64_t kept[2];
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int w0 = 4 * v + 2 * hh;
                            kept[hh] = (w0 < p.W ? (uint64_t)it.mask[w0] : ~0ull) |
                                       (w0 + 1 < p.W ? (uint64_t)it.mask[w0 + 1] << 32 : (~0ull << 32));
                            const int rem = NK32 - (kN * v + 64 * hh);
                            const uint64_t inb = rem >= 64 ? ~0ull : (rem <= 0 ? 0ull : ((1ull << rem) - 1ull));
                            kept[hh] = ~kept[hh] & inb;
                        }
                        vlo = kept[0];
                        vhi = kept[1];
                        if (NK32 - 1 >= kN * v && NK32 - 1 < kN * (v + 1)) clast = NK32 - 1 - kN * v;
                    }
                    const bool allvalid = (vlo & vhi) == ~0ull;
                    uint32_t pk[64];
                    float hq[4];
                    // Exponentials against the reference mref, one 64-column half at a time
                    // (FFMA2 for s x - m, FADD2 quarter sums): P of half h -> pk[32h..32h+31];
                    // on all-valid ops POLY of every 4 column pairs go to the FMA pipe (ex2_fma2)
                    // instead of MUFU.  The S registers are dead afterwards (reloaded from TMEM
                    // in the rare case the reference moves).
                    auto mask_half = [&](uint32_t (&sv)[64], uint64_t vm) {
                        if (vm != ~0ull) {
#pragma unroll
                            for (int c = 0; c < 64; ++c)
                                if (!((vm >> c) & 1ull)) sv[c] = 0xff800000u;
                        }
                    };
                    // poly: std::integral_constant -- the FMA-pipe share is decided once per op,
                    // never per column pair (a runtime test inside the unrolled loop costs a
                    // branch and a reconvergence barrier per pair)
                    auto exps_half_t = [&](const uint32_t (&sv)[64], int h, float mref, auto polyc) {
                        constexpr bool poly = decltype(polyc)::value;
                        const float2 nm2 = make_float2(-mref, -mref);
#pragma unroll
                        for (int qq = 0; qq < 2; ++qq) {
                            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                            for (int c = 16 * qq; c < 16 * qq + 16; ++c) {
                                const float2 x = ffma2(make_float2(__uint_as_float(sv[2 * c]),
                                                                   __uint_as_float(sv[2 * c + 1])), cs2, nm2);
                                float2 pp;
                                if (POLY > 0 && poly && (c & 3) < POLY) {
                                    pp = ex2_fma2(x);
                                } else {
                                    pp.x = ex2(x.x);
                                    pp.y = ex2(x.y);
                                }
                                acc = fadd2(acc, pp);
                                pk[32 * h + c] = pack_bf16(pp.x, pp.y);
                            }
                            hq[2 * h + qq] = acc.x + acc.y;
                        }
                    };
                    auto exps_half = [&](const uint32_t (&sv)[64], int h, float mref, bool poly) {
                        if (POLY > 0 && poly) exps_half_t(sv, h, mref, std::true_type{});
                        else exps_half_t(sv, h, mref, std::false_type{});
                    };
                    auto ld_half = [&](uint32_t (&sv)[64], int h) {
                        tmem_ld32(tS + 64 * h, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
                        tmem_ld32(tS + 64 * h + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
                    };
                    auto st_half = [&](int h) {
                        tmem_st32(tS + 32 * h, *reinterpret_cast<const uint32_t(*)[32]>(&pk[32 * h]));
                    };
                    float xlast = -INFINITY;   // raw logit of the ragged last block (C ops)
                    auto grab_last = [&](const uint32_t (&sv)[64], int h) {
                        if (clast >= 64 * h && clast < 64 * h + 64) {
#pragma unroll
                            for (int c = 0; c < 64; ++c)
                                if (c + 64 * h == clast) xlast = __uint_as_float(sv[c]);
                        }
                    };
                    {
                        // (no tcgen05.ld may stay in flight across other code: the compiler does
                        // not know its destination registers are written asynchronously)
                        uint32_t sa[64], sb[64];
                        ld_half(sa, 0);
                        ld_half(sb, 1);
                        tmem_wait_ld();
                        mask_half(sa, vlo);
                        grab_last(sa, 0);
                        exps_half(sa, 0, m, allvalid);
                        mask_half(sb, vhi);
                        grab_last(sb, 1);
                        exps_half(sb, 1, m, allvalid);
                    }
                    bool resc = false;
                    float corr = 1.f;
                    if (__any_sync(0xffffffffu, !(hq[0] + hq[1] + hq[2] + hq[3] < 256.f))) {
                        // a row may hold a new maximum (or this is the item's first op): take
                        // the exact row max and move the reference when it grew by > 2^8
                        uint32_t sa[64], sb[64];
                        ld_half(sa, 0);
                        ld_half(sb, 1);
                        tmem_wait_ld();
                        mask_half(sa, vlo);
                        mask_half(sb, vhi);
                        float mr0 = -INFINITY, mr1 = -INFINITY, mr2 = -INFINITY, mr3 = -INFINITY;
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            mr0 = fmax3(mr0, __uint_as_float(sa[c]), __uint_as_float(sa[c + 1]));
                            mr1 = fmax3(mr1, __uint_as_float(sa[32 + c]), __uint_as_float(sa[33 + c]));
                            mr2 = fmax3(mr2, __uint_as_float(sb[c]), __uint_as_float(sb[c + 1]));
                            mr3 = fmax3(mr3, __uint_as_float(sb[32 + c]), __uint_as_float(sb[33 + c]));
                        }
                        const float mx = fmaxf(fmax3(mr0, mr1, mr2), mr3) * cs;
                        const bool moved = mx > m + kRescaleThresh;
                        if (moved) {
                            corr = ex2(m - mx);   // 0 when m = -inf
                            resc = n > 0;
                            m = mx;
                            l *= corr;
                            A_acc *= corr;
                        }
                        // recomputed unconditionally on this (rare) path, so the first pass's
                        // P registers are dead here and the reloaded S fits beside them
                        exps_half(sa, 0, m, allvalid);
                        exps_half(sb, 1, m, allvalid);
                    }
                    if (__any_sync(0xffffffffu, resc)) {
                        // S ready => every earlier MMA of this tile has completed (QK^T of this
                        // op was issued after them): O is final up to op n-1
#pragma unroll 1
                        for (int c0 = 0; c0 < D; c0 += 32) {
                            uint32_t o[32];
                            tmem_ld32(tO + c0, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                            tmem_st32(tO + c0, o);
                        }
                    }
                    // P overwrites S only now: the slow path above may still reload S
                    st_half(0);
                    st_half(1);
                    const float hsum = (hq[0] + hq[1]) + (hq[2] + hq[3]);
                    if (type == OP_E) {
                        l += hsum;
                    } else {
                        // denominator: n_j p_j per dropped block, 64 except the ragged last (R-2)
                        const float pl = clast >= 0 ? ex2(fmaf(xlast, cs, -m)) : 0.f;
                        l += 64.f * hsum - (64.f - (float)nlast_len) * pl;
                        // first-order weights A_{t,g} = sum of p over the group's dropped blocks
                        if (G32 == 32) {
#pragma unroll
                            for (int q = 0; q < 4; ++q) A4[q] = hq[q];
                        } else if (G32 == 64) {
                            A4[0] = hq[0] + hq[1];
                            A4[1] = hq[2] + hq[3];
                        } else {
                            const int g0 = (int)((int64_t)kN * v / G32);
                            if (g0 != g_cur) { A_acc = 0.f; g_cur = g0; }
                            A_acc += hsum;
                        }
                        c_last = v;
                    }
                    tmem_wait_st();
                    frun = 0;
                } else {
                    // F(v): Aq = bf16(s A_{t,v} q_t) into S_t[64:) (first, third, .. F op of a
                    // run) or S_t[0:) (second, fourth, ..).  The previous reader of that half is
                    // op n-2's MMA unless op n-1 was an S op (its S ready => all earlier MMAs done)
                    float A = A_acc;
                    if (G32 == 32 || G32 == 64) {   // register select (no local-memory index)
                        const int kq = v - (G32 == 32 ? 4 : 2) * c_last;
                        A = kq == 0 ? A4[0] : kq == 1 ? A4[1] : kq == 2 ? A4[2] : A4[3];
                    }
                    const uint32_t acol = (frun & 1) == 0 ? 64u : 0u;
                    if (row == 0) PASA_TD(TD_SM_FW, t, gn);
                    if (frun > 0) mbar_wait_c(&ctl.mma_done[t][(gn - 2) & 1], ((gn - 2) >> 1) & 1, spin);
                    if (row == 0) PASA_TD(TD_SM_FO, t, gn);
                    ++frun;
                    tc_fence_after();
                    const uint32_t w2 = pack_bf16(p.s * A, p.s * A);
#pragma unroll
                    for (int a = 0; a < G_::NBOX; ++a) {
                        uint32_t aq[32];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const uint4 q4 = *reinterpret_cast<const uint4*>(
                                qrow + a * (kBQ * 128) + row * 128 + ((c ^ (row & 7)) << 4));
                            aq[4 * c + 0] = hmul2_bf16(q4.x, w2);
                            aq[4 * c + 1] = hmul2_bf16(q4.y, w2);
                            aq[4 * c + 2] = hmul2_bf16(q4.z, w2);
                            aq[4 * c + 3] = hmul2_bf16(q4.w, w2);
                        }
                        tmem_st32(tS + acol + 32 * a, aq);
                    }
                    tmem_wait_st();
                }
                tc_fence_before();
                mbar_arrive(&ctl.p_full[t][gn & 1]);
                if (row == 0) PASA_TD(TD_SM_AR, t, gn);
            }
            // item done with Q_t and the op list
            mbar_arrive(&ctl.q_empty[t]);
            mbar_arrive(&ctl.item_empty[t][r & 1]);
            // ---- epilogue: O / l -> bf16 -> out (rows past S are not stored) ----
            mbar_wait_sleep(&ctl.mma_done[t][(gn - 1) & 1], ((gn - 1) >> 1) & 1);
            tc_fence_after();
            const int64_t bh = u / NQ, i = u % NQ;
            const int64_t b = bh / p.H, h = bh % p.H;
            const int64_t trow = i * kBQ + row;
            const float inv = 1.f / l;
            __nv_bfloat16* orow = p.out + b * p.osB + h * p.osH + trow * p.osS;
#pragma unroll 1
            for (int c0 = 0; c0 < D; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(tO + c0, o);
                tmem_wait_ld();
                if (trow < p.S) {
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
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

// ---------------------------------------------------------------- host --
template <int D>
cudaError_t launch_d(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                     pasa_route_s* r, const pasa_tensor& out, cudaStream_t st, int poly,
                     char* why, size_t why_len) {
    CUtensorMap mQ, mK, mV, mKb, mVs, mHt;
    auto act = [&](CUtensorMap* m, const pasa_tensor& t, uint32_t rows) {
        uint64_t dims[4] = {(uint64_t)t.D, (uint64_t)t.S, (uint64_t)t.H, (uint64_t)t.B};
        uint64_t str[3] = {(uint64_t)t.sS * 2, (uint64_t)t.sH * 2, (uint64_t)t.sB * 2};
        uint32_t box[4] = {64, rows, 1, 1};
        return make_tensor_map(m, t.data, 4, dims, str, box, why, why_len);
    };
    if (!act(&mQ, q, kBQ) || !act(&mK, k, kBK) || !act(&mV, v, kBK)) return cudaErrorNotSupported;
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
    prm.idx_ld = r->idx_ld;
    prm.U = r->BH * r->NQ;
    prm.G = r->cfg.G; prm.comp = r->cfg.comp;
    const double s = 1.0 / sqrt((double)D);
    prm.s = (float)s;
    prm.scale_log2 = (float)(s * 1.4426950408889634);
    prm.idx = r->idx; prm.count = r->count; prm.mask = r->mask;
    prm.work = r->hdr + 8;   // route header word 8: this launch's item counter
    prm.out = reinterpret_cast<__nv_bfloat16*>(out.data);
    prm.osB = out.sB; prm.osS = out.sS; prm.osH = out.sH;
    prm.dbg = g_dbg;
    prm.trace = (g_dbg & 2048) ? g_trace_buf : nullptr;
    prm.trace_cta = g_trace_x;
    const size_t smem = (size_t)Geo<D>::BYTES + 1024;
    auto kern = poly == 2 ? attn_dual_kernel<D, 2> : poly == 1 ? attn_dual_kernel<D, 1>
                                                               : attn_dual_kernel<D, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = (prm.U + 1) / 2;
    const unsigned grid = (unsigned)(need < sms ? need : sms);
    e = cudaMemsetAsync(prm.work, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, st>>>(mQ, mK, mV, mKb, mVs, mHt, prm);
    return cudaGetLastError();
}

}  // namespace

bool attn_sm100_dual_supported(const pasa_route_s* r) {
    const int64_t G = r->cfg.G;
    const bool groups_ok = r->cfg.comp != PASA_COMP_GROUPED || G == 32 || G == 64 || G % 128 == 0 ||
                           G >= r->NK;
    return r->cfg.Bq == kBQ && r->cfg.Bk == kBK && (r->D == 64 || r->D == 128) && r->NK <= 4096 &&
           groups_ok;
}

cudaError_t launch_attn_sm100_dual(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                                   pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                                   int* launches, char* why, size_t why_len) {
    if (!attn_sm100_dual_supported(r)) {
        snprintf(why, why_len, "dual-tile kernel: needs Bq=128, Bk=64, d 64/128, N_K <= 4096, "
                 "G in {32, 64, k*128, >= N_K}");
        return cudaErrorNotSupported;
    }
    // share of the exponentials on the FMA pipe (of every 4 column pairs): pasa_debug_flags
    // bit 7 -> 1, bit 12 -> 2, bit 13 -> 0; default kPolyDefault
    const int poly = (g_dbg & 8192) ? 0 : (g_dbg & 4096) ? 2 : (g_dbg & 128) ? 1 : kPolyDefault;
    cudaError_t e = r->D == 128 ? launch_d<128>(q, k, v, r, out, st, poly, why, why_len)
                                : launch_d<64>(q, k, v, r, out, st, poly, why, why_len);
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace pasa
