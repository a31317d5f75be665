// attn_sm100.cu -- pasa_attn on the Blackwell tensor cores (sm_100a):
// gather-driven block-sparse attention with the PASA compensation fused into
// the same online softmax (Eq. 7; grouped first-order term,
// PAPER.md:310-313 and App. B :503-506; readings R-1..R-5, R-21, R-22 in
// DESIGN.md §3).  Design notes: DESIGN.md §7.
//
// One CTA per (head, 128-row query block); 2 CTAs per SM (TMEM 2 x 256 cols,
// ~97 KB smem each at d = 128) so one CTA's softmax overlaps the other's MMAs.
// Warp roles (256 threads):
//   warp 0  TMA producer of the K ring (K tiles / Kbar chunks / Hbar^T box 0)
//   warp 1  TMEM allocator + tcgen05.mma issuer (warp-converged, elect.sync)
//   warp 2  TMA producer of the V ring (V tiles / Vsum chunks / Hbar^T box 1)
//   warps 4-7  softmax / correction / epilogue, one query row per thread
// The CTA walks one "op" list:
//   E(j)  kept block j:        S = Q K_j^T (SS MMA) -> softmax -> O += P V_j (TS MMA)
//   C(c)  centroid chunk c:    S = Q Kbar_c^T -> masked to the dropped blocks,
//                              weights n_j in the denominator -> O += P Vsum_c
//   F(g)  group g's first order: O += (s A_g (.) Q) Hbar^(g)  (TS MMA, A from TMEM)
// The running max only moves up by more than 2^8 (log2 domain) before O is
// rescaled, so O corrections are rare; they wait for the previous MMA first.
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
constexpr int kBQ = 128, kBK = 64;
// op list: kept blocks (<= N_K <= 4096) + centroid chunks (<= 64) + first-order ops
// (<= N_K / 8 for G >= 8) + slack; 16-bit entries (type in the top 2 bits)
constexpr int kMaxNK = 4096;
constexpr int kMaxOps = kMaxNK + kMaxNK / 64 + kMaxNK / 8 + 64;
constexpr int kTmemCols = 256;
constexpr float kRescaleThresh = 8.f; // log2 units
// d = 64: one exponential pair in PASA_D64_POLY on the FMA pipe (degree-3 polynomial,
// ex2_fma2) instead of MUFU (0 = none); A/B knob, see DESIGN.md §12
#ifndef PASA_D64_POLY
#define PASA_D64_POLY 0
#endif
// d = 64: Q copied into TMEM once per CTA so QK^T is a TS MMA (only the K tile is read
// from shared memory: the SS MMA at N = 64 is shared-memory bound), two S buffers instead
// of three to make room (O 64 + S 2 x 64 + Q 32 columns)
#ifndef PASA_D64_QTMEM
#define PASA_D64_QTMEM 1
#endif
constexpr bool kD64QT = PASA_D64_QTMEM != 0;
// d = 128 (A/B knob): Q in TMEM as well, which leaves room for ONE S buffer (O 128 + S 64 +
// Q 64 columns): QK of op n+1 then follows PV of op n (a serial chain per CTA)
#ifndef PASA_D128_QTMEM
#define PASA_D128_QTMEM 0
#endif
constexpr bool kD128QT = PASA_D128_QTMEM != 0;
// critical-path barrier waits (A/B knob): 0 = try_wait with a suspend-time hint (default);
// bit 0: the MMA warp's waits without the hint, bit 1: the softmax's S wait without the
// hint, bit 2: those waits as test_wait polling loops
// P release (A/B knob): 1 = one arrival per softmax warp after __syncwarp (p_full count
// 4 + the V producer) instead of one per thread (128 + 1)
#ifndef PASA_WARP_ARRIVE
#define PASA_WARP_ARRIVE 0
#endif
// prologue (A/B knob): 1 = thread 0 issues the Q tile and the first kept blocks' K / V
// loads right after initialising the barriers, before the op-list tail, TMEM allocation and
// the CTA barrier (the per-CTA fixed cost is ~6 us per wave: tools/ops_scaling.py)
#ifndef PASA_EARLY_LOADS
#define PASA_EARLY_LOADS 0
#endif
#ifndef PASA_CRIT_WAIT
#define PASA_CRIT_WAIT 0
#endif
__device__ __forceinline__ void crit_wait(uint64_t* bar, uint32_t parity, bool spin) {
    if (PASA_CRIT_WAIT & 4) {
        if (spin) { while (!ptx::mbar_test(bar, parity)) {} return; }
    }
    ptx::mbar_wait_c(bar, parity, spin);
}

enum : int32_t { OP_E = 0, OP_C = 1, OP_F = 2 };
__device__ __forceinline__ uint16_t op_make(int32_t type, int32_t v) {
    return (uint16_t)((type << 14) | v);
}
__device__ __forceinline__ int32_t op_type(int32_t op) { return op >> 14; }
__device__ __forceinline__ int32_t op_val(int32_t op) { return op & 0x3FFF; }

// NB = S/P/Aq buffers in TMEM = K ring slots: 2 at d = 128 (TMEM: O 128 + 2 x 64
// columns), 3 at d = 64 (O 64 + 3 x 64) -- QK of op n+NB-1 is issued before PV of op n.
template <int D>
struct Geo {
    static constexpr bool QT = D == 64 ? kD64QT : kD128QT;   // Q in TMEM
    static constexpr int NB = D == 128 ? (QT ? 1 : 2) : (QT ? 2 : 3);   // S buffers
    static constexpr int NKS = NB < 2 ? 2 : NB;     // K ring slots
    static constexpr uint32_t COLS = D == 128 ? 128 : 64;   // first S buffer column
    static constexpr uint32_t QCOL = 192;           // QT: Q's D/2 columns after the S buffers
    static constexpr int NBOX = D / 64;
    static constexpr int QBOX = kBQ * 128;          // bytes per 64-col box of Q
    static constexpr int KVBOX = kBK * 128;         // bytes per 64-col box of a K/V tile
    static constexpr int SLOT = kBK * D * 2;        // bytes per K or V slot
    static constexpr int HTBOX = D * 128;           // bytes per 64-col box of Hbar^T
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = kBQ * D * 2;
    static constexpr int OFF_V = OFF_K + NKS * SLOT;
    static constexpr int BYTES = OFF_V + 2 * SLOT;
    static_assert(HTBOX <= SLOT, "an Hbar^T box must fit one ring slot");
};

struct Params {
    int64_t S, H, NQ, NK, NG, W;
    int64_t it0;        // first (head, q-block) item of the handle's range (grid.x covers it)
    int32_t G, comp;
    float scale_log2;   // s * log2(e)
    float s;            // 1/sqrt(D)
    const int32_t* idx;
    const int32_t* count;
    const uint32_t* mask;
    __nv_bfloat16* out;
    int64_t osB, osS, osH;
    // FP8 QK^T variant (cfg.qk_fp8): per-row Q scales [BH][S]; per-head max |K| and
    // max |Kbar| (float bits) [BH] each
    const float* sq;
    const uint32_t* kamax;
    const uint32_t* kbamax;
    // zero-copy sequence parallelism (pasa_attn_zc): oP > 0 stores row t into its owner's
    // shard s (tokens [ostart[s], ostart[s+1]) at obase[s], already offset to this rank's
    // first head) instead of out
    int32_t oP;
    int64_t ostart[9];
    __nv_bfloat16* obase[8];
    int64_t oSS, oSH;
    unsigned long long* trace;   // diagnostics: clock64 timeline of one CTA, or nullptr
    int32_t trace_x, trace_y;
    int32_t dbg;                 // diagnostics ablations (see pasa_debug_flags)
};

// timeline events (pasa_debug_trace); slot = event * kTraceN + index
constexpr int kTraceN = 4096;
enum { TR_KPROD = 0, TR_VPROD, TR_MMA_P, TR_MMA_V, TR_MMA_QK, TR_SA_W, TR_SA_OK, TR_SA_ARR,
       TR_SB_W, TR_SB_OK, TR_SB_ARR, TR_MMA_QKW, TR_KPROD_W, TR_SA_LD, TR_SA_MAX, TR_SA_EXP,
       TR_SA_ST, TR_NEV };
#define PASA_TR(ev, ix)                                                               \
    do {                                                                              \
        if (DIAG && tracing && (ix) < kTraceN) p.trace[(ev) * kTraceN + (ix)] = clock64(); \
    } while (0)

struct Ctl {
    uint64_t q_full, q_tmem;
    uint64_t k_full[3], k_empty[3], s_full[3];   // per K slot / S buffer (n % NB)
    // p_full per S buffer (n % NB): P ready + V landed.  With NB = 3 the softmax can finish
    // op n+2 before V(n) has even been requested (QK(n+2) is issued before PV(n)), so a
    // barrier shared by ops n and n+2 would count op n+2's arrivals into op n's phase and
    // let PV(n) read an unloaded V tile; one barrier per S buffer cannot be lapped, since
    // QK(n+NB) follows PV(n).  pv_done per V slot (n & 1): O-MMA done.
    uint64_t p_full[3], pv_done[2];
    uint64_t v_full[2];   // NB = 1 only: the V tile of op n (slot n & 1) landed (own barrier:
                          // the V producer runs two ops ahead of the single P barrier)
    uint32_t tmem_base;
    int32_t nops;
    uint32_t mask[kMaxNK / 32];
    uint16_t ops[kMaxOps];
};
// EXP 1 (groups of 8 or 16 blocks): the 8-column P sums of the last C op, per row
struct CtlSG : Ctl {
    float sg[8][kBQ];
};

// DIAG: diagnostics build (trace points, ablation flags, polling waits); the
// production instantiation compiles all of it out
// F8: QK^T of kept blocks and the centroid logits on the FP8 tensor cores (E4M3 Q / K /
// Kbar tiles from the route's and the statistics pass's FP8 copies, scales folded into
// the per-op softmax scale), PV and the first-order op stay bf16 (d = 128 only)
template <int D, bool DIAG, int EXP, bool F8 = false>
__global__ void __launch_bounds__(kThreads, 2)
    attn_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                      const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmKb,
                      const __grid_constant__ CUtensorMap tmVs,
                      const __grid_constant__ CUtensorMap tmHt, const Params p) {
    using G_ = Geo<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ std::conditional_t<EXP == 1, CtlSG, Ctl> ctl;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool spin_dbg = DIAG && (p.dbg & 4) != 0;   // diagnostics: poll critical-path barriers
    const bool spin = spin_dbg || (PASA_CRIT_WAIT & 1) != 0;      // MMA warp
    const bool spin_s = spin_dbg || (PASA_CRIT_WAIT & 2) != 0;    // softmax S wait
    const bool tracing = p.trace != nullptr && (int)((p.it0 + blockIdx.x) % p.NQ) == p.trace_x &&
                         (int)((p.it0 + blockIdx.x) / p.NQ) == p.trace_y;
    const int64_t item = p.it0 + blockIdx.x;
    const int64_t i = item % p.NQ, bh = item / p.NQ;
    const int64_t b = bh / p.H, h = bh % p.H;
    const int64_t row = bh * p.NQ + i;
    const int32_t cnt = p.count[row];
    const int64_t NK = p.NK;
    const int nchunks = (int)((NK + 63) / 64);

    // ---------------- loads (K ring: warp 0, V ring: warp 2; the first ones by thread 0) ----
    auto load_q = [&]() {
        if constexpr (F8) {
            mbar_arrive_expect_tx(&ctl.q_full, kBQ * D);
            tma_load_3d(smem + G_::OFF_Q, &tmQ, &ctl.q_full, 0, (int)(i * kBQ), (int)bh);
        } else {
            mbar_arrive_expect_tx(&ctl.q_full, kBQ * D * 2);
#pragma unroll
            for (int a = 0; a < G_::NBOX; ++a)
                tma_load_4d(smem + G_::OFF_Q + a * G_::QBOX, &tmQ, &ctl.q_full, 64 * a,
                            (int)(i * kBQ), (int)h, (int)b);
        }
    };
    auto load_k = [&](int n, int32_t op) {   // op n into K slot n % NKS (slot known free)
        const int s = n % G_::NKS;
        uint8_t* dst = smem + G_::OFF_K + s * G_::SLOT;
        const int v = op_val(op);
        if (DIAG && (p.dbg & 2)) {
            mbar_arrive(&ctl.k_full[s]);
        } else if (op_type(op) == OP_F) {
            mbar_arrive_expect_tx(&ctl.k_full[s], G_::HTBOX);
            tma_load_3d(dst, &tmHt, &ctl.k_full[s], 0, v * D, (int)bh);
        } else if constexpr (F8) {   // E4M3 K tile or Kbar chunk: 64 rows x 128 B
            mbar_arrive_expect_tx(&ctl.k_full[s], kBK * D);
            tma_load_3d(dst, op_type(op) == OP_E ? &tmK : &tmKb, &ctl.k_full[s], 0,
                        v * kBK, (int)bh);
        } else {
            mbar_arrive_expect_tx(&ctl.k_full[s], G_::SLOT);
#pragma unroll
            for (int a = 0; a < G_::NBOX; ++a) {
                if (op_type(op) == OP_E)
                    tma_load_4d(dst + a * G_::KVBOX, &tmK, &ctl.k_full[s], 64 * a, v * kBK,
                                (int)h, (int)b);
                else
                    tma_load_3d(dst + a * G_::KVBOX, &tmKb, &ctl.k_full[s], 64 * a, v * 64,
                                (int)bh);
            }
        }
    };
    auto load_v = [&](int n, int32_t op) {   // op n into V slot n & 1 (slot known free)
        const int s = n & 1, pb = n % G_::NB;
        uint64_t* vbar = G_::NB == 1 ? &ctl.v_full[s] : &ctl.p_full[pb];
        uint8_t* dst = smem + G_::OFF_V + s * G_::SLOT;
        const int v = op_val(op);
        if (DIAG && (p.dbg & 2)) {
            mbar_arrive(vbar);
        } else if (op_type(op) == OP_F) {
            if (G_::NBOX == 2) {
                mbar_arrive_expect_tx(vbar, G_::HTBOX);
                tma_load_3d(dst, &tmHt, vbar, 64, v * D, (int)bh);
            } else {
                mbar_arrive(vbar);
            }
        } else {
            mbar_arrive_expect_tx(vbar, G_::SLOT);
#pragma unroll
            for (int a = 0; a < G_::NBOX; ++a) {
                if (op_type(op) == OP_E)
                    tma_load_4d(dst + a * G_::KVBOX, &tmV, vbar, 64 * a, v * kBK,
                                (int)h, (int)b);
                else
                    tma_load_3d(dst + a * G_::KVBOX, &tmVs, vbar, 64 * a, v * 64, (int)bh);
            }
        }
    };
    // ops whose loads thread 0 issues in the prologue: kept blocks only (their index comes
    // straight from the route), as many as the rings hold without waiting
    const int n_pre_k = PASA_EARLY_LOADS ? min(cnt, G_::NKS) : 0;
    const int n_pre_v = PASA_EARLY_LOADS ? min(cnt, 2) : 0;

    // ---------------- setup: op list, mask row, barriers, TMEM ----------------
    for (int w = tid; w < p.W; w += blockDim.x) ctl.mask[w] = p.mask[row * p.W + w];
    for (int q = tid; q < cnt; q += blockDim.x) ctl.ops[q] = op_make(OP_E, p.idx[row * NK + q]);
    if (tid == 0) {
        mbar_init(&ctl.q_full, 1);
        mbar_init(&ctl.q_tmem, 128);          // QT: the softmax threads copied Q into TMEM
        for (int s = 0; s < G_::NKS; ++s) {
            mbar_init(&ctl.k_full[s], 1);
            mbar_init(&ctl.k_empty[s], 1);
        }
        for (int s = 0; s < G_::NB; ++s) mbar_init(&ctl.s_full[s], 1);
        for (int s = 0; s < G_::NB; ++s)
            mbar_init(&ctl.p_full[s], (PASA_WARP_ARRIVE ? 4 : 128) + (G_::NB == 1 ? 0 : 1));   // softmax + V producer
        if (G_::NB == 1) {
            mbar_init(&ctl.v_full[0], 1);
            mbar_init(&ctl.v_full[1], 1);
        }
        mbar_init(&ctl.pv_done[0], 1);
        mbar_init(&ctl.pv_done[1], 1);
        fence_barrier_init();
        if (PASA_EARLY_LOADS) {   // thread 0 = the K producer's issuing lane
            tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
            load_q();
            for (int n = 0; n < max(n_pre_k, n_pre_v); ++n) {
                const int32_t op = op_make(OP_E, p.idx[row * NK + n]);
                if (n < n_pre_k) load_k(n, op);
                if (n < n_pre_v) load_v(n, op);
            }
        }
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
        // tail of the op list: centroid chunks with a dropped block, then the
        // first-order op of every group that ends inside the chunk (G % 32 == 0
        // or one global group: every 32-block half-chunk lies in one group)
        // word-level: word w of the mask covers blocks [32w, 32w+32), inside one group
        int n = cnt;
        if (p.comp != PASA_COMP_NONE && cnt < NK) {
            const int W = (int)p.W;
            auto dropped_word = [&](int w) {
                const int64_t rem = NK - 32 * (int64_t)w;
                const uint32_t inb = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
                return (~ctl.mask[w] & inb) != 0u;
            };
            const int64_t G = p.G;
            int64_t g = 0;                              // next group to close
            for (int c = 0; c < nchunks; ++c) {
                if (dropped_word(2 * c) || (2 * c + 1 < W && dropped_word(2 * c + 1)))
                    ctl.ops[n++] = op_make(OP_C, c);
                if (p.comp == PASA_COMP_GROUPED) {
                    const int64_t chunk_end = min(64 * (int64_t)(c + 1), NK);
                    for (; g * G < NK && min((g + 1) * G, NK) <= chunk_end; ++g) {
                        const int w0 = (int)((g * G) >> 5);
                        const int w1 = (int)((min((g + 1) * G, NK) + 31) >> 5);
                        bool any = false;
                        for (int w = w0; w < w1 && !any; ++w) any = dropped_word(w);
                        if (any) ctl.ops[n++] = op_make(OP_F, (int32_t)g);
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
            if (!PASA_EARLY_LOADS) load_q();
            for (int n = n_pre_k; n < nops; ++n) {
                mbar_wait_sleep(&ctl.k_empty[n % G_::NKS], ((n / G_::NKS) & 1) ^ 1);
                load_k(n, ctl.ops[n]);
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ======================= V-ring producer =======================
        if (lane == 0) {
            for (int n = n_pre_v; n < nops; ++n) {
                mbar_wait_sleep(&ctl.pv_done[n & 1], ((n >> 1) & 1) ^ 1);   // PV(n-2) read the slot
                load_v(n, ctl.ops[n]);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ======================= MMA issuer =======================
        constexpr uint32_t kIdQK = idesc_bf16_f32(128, kBK, 0, 0);   // Q (K-major) x K^T (K-major)
        constexpr uint32_t kIdPV = idesc_bf16_f32(128, D, 0, 1);     // P (TMEM) x V (MN-major)
        constexpr uint32_t kIdF = idesc_bf16_f32(128, D, 0, 0);      // Aq (TMEM) x Hbar^T (K-major)
        const uint32_t q_base = smem_u32(smem + G_::OFF_Q);
        const uint32_t k_base = smem_u32(smem + G_::OFF_K);
        const uint32_t v_base = smem_u32(smem + G_::OFF_V);
        // descriptors: the 14-bit start-address field is advanced arithmetically
        const uint64_t dq0 = umma_desc_sw128(q_base, 16, 1024);
        const uint64_t dk0 = umma_desc_sw128(k_base, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(v_base, G_::KVBOX, 1024);
        auto issue_qk = [&](int n) {
            const int s = n % G_::NKS, sbuf = n % G_::NB;   // K ring slot, S buffer
            if (lane == 0) PASA_TR(TR_MMA_QKW, n);
            crit_wait(&ctl.k_full[s], (n / G_::NKS) & 1, spin);
            if (lane == 0) PASA_TR(TR_SB_W, n);           // K(n) landed
            tc_fence_after();
            // the whole warp runs the issue code with warp-uniform operands; elect.sync
            // picks the issuing lane (no per-instruction elect loop)
            const uint32_t d = tbase + G_::COLS + 64 * sbuf;
            if constexpr (F8) {   // E4M3: 32 elements (bytes) of the 128-byte rows per MMA
                constexpr uint32_t kIdQK8 = idesc_e4m3_f32(128, kBK, 0, 0);
#pragma unroll
                for (int kk = 0; kk < D / 32; ++kk)
                    mma_ss_f8_elect(d, dq0 + ((kk * 32) >> 4),
                                    dk0 + ((s * G_::SLOT + kk * 32) >> 4), kIdQK8, kk > 0);
            } else if constexpr (G_::QT) {   // A = Q from TMEM (8 columns per 16 elements)
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t offk = (s * G_::SLOT + (kk >> 2) * G_::KVBOX + (kk & 3) * 32) >> 4;
                    mma_ts_elect(d, tbase + G_::QCOL + kk * 8, dk0 + offk, kIdQK, kk > 0);
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t offq = ((kk >> 2) * G_::QBOX + (kk & 3) * 32) >> 4;
                    const uint32_t offk = (s * G_::SLOT + (kk >> 2) * G_::KVBOX + (kk & 3) * 32) >> 4;
                    mma_ss_elect(d, dq0 + offq, dk0 + offk, kIdQK, kk > 0);
                }
            }
            mma_commit_elect(&ctl.s_full[sbuf]);
            mma_commit_elect(&ctl.k_empty[s]);
            if (lane == 0) PASA_TR(TR_MMA_QK, n);
            __syncwarp();
        };
        mbar_wait_sleep(G_::QT ? &ctl.q_tmem : &ctl.q_full, 0);
        tc_fence_after();
        for (int m = 0; m < G_::NB - 1 && m < nops; ++m)
            if (op_type(ctl.ops[m]) != OP_F) issue_qk(m);
        for (int n = 0; n < nops; ++n) {
            const int s = n & 1, sb = n % G_::NB;
            const int nq = n + G_::NB - 1;   // its buffer was last read by PV(n-1), issued before
            if (nq < nops && op_type(ctl.ops[nq]) != OP_F) issue_qk(nq);
            // V(n) lands on p_full[s] too (one wait for "P ready and V loaded")
            if (lane == 0) PASA_TR(TR_MMA_V, n);
            crit_wait(&ctl.p_full[sb], (n / G_::NB) & 1, spin);
            if (G_::NB == 1) mbar_wait_c(&ctl.v_full[s], (n >> 1) & 1, spin);
            if (lane == 0) PASA_TR(TR_MMA_P, n);
            tc_fence_after();
            const int32_t op = ctl.ops[n];
            if (op_type(op) != OP_F) {
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    const uint32_t offv = (s * G_::SLOT + kk * 16 * 128) >> 4;
                    mma_ts_elect(tbase, tbase + G_::COLS + 64 * sb + kk * 8, dv0 + offv, kIdPV,
                                 (n > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit_elect(&ctl.pv_done[s]);
                if (lane == 0) PASA_TR(TR_KPROD_W, n);
            } else {
                const int sk = n % G_::NKS;   // the K slot holding H-bar^T box 0
                crit_wait(&ctl.k_full[sk], (n / G_::NKS) & 1, spin);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t box = (kk >> 2) == 0 ? k_base + sk * G_::SLOT
                                                        : v_base + s * G_::SLOT;
                    const uint64_t bd = umma_desc_sw128(box + (kk & 3) * 32, 16, 1024);
                    mma_ts_elect(tbase, tbase + G_::COLS + 64 * sb + kk * 8, bd, kIdF, 1u);
                }
                mma_commit_elect(&ctl.k_empty[sk]);
                mma_commit_elect(&ctl.pv_done[s]);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // =================== softmax / correction / epilogue ===================
        const int r = (warp & 3) * 32 + lane;                 // query row in the block
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t t_o = tbase + lane_off;
        const uint8_t* qrow = smem + G_::OFF_Q;
        if constexpr (G_::QT) {   // Q row r -> TMEM lane r, columns QCOL.. (bf16 pairs)
            mbar_wait_sleep(&ctl.q_full, 0);
#pragma unroll
            for (int a = 0; a < G_::NBOX; ++a) {
                uint32_t qa[32];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const uint4 u = *reinterpret_cast<const uint4*>(qrow + a * G_::QBOX + r * 128 +
                                                                    ((cc ^ (r & 7)) << 4));
                    qa[cc * 4 + 0] = u.x; qa[cc * 4 + 1] = u.y; qa[cc * 4 + 2] = u.z;
                    qa[cc * 4 + 3] = u.w;
                }
                tmem_st32(t_o + G_::QCOL + 32 * a, qa);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&ctl.q_tmem);
        }
        float m = -INFINITY, l = 0.f;
        float A_cur = 0.f, A_done = 0.f;
        int g_cur = -1, g_done = -1;          // group of the running / last closed A sum
        const int G32 = (int)p.G, NK32 = (int)NK;
        int c_last = 0;   // G = 8 or 16: chunk of the last C op (ctl.sg holds its group sums)
        int sc0 = 0, sc1 = 0, sc2 = 0;   // S-type ops seen per S buffer (s_full parity)
        const int64_t n_last = NK - 1;
        const int nlast_len = (int)(p.S - n_last * 64);
        float cs = p.scale_log2;         // logits in log2 units: x = S * s * log2(e)
        // F8: this row's Q scale and the head's K / Kbar scales, folded into the softmax scale
        float sq_row = 1.f, cs_e = cs, cs_c = cs;
        if constexpr (F8) {
            const int64_t t = i * kBQ + r;
            sq_row = t < p.S ? p.sq[bh * p.S + t] : 1.f;
            float ska = __uint_as_float(p.kamax[bh]) * (1.f / 448.f);
            float skb = __uint_as_float(p.kbamax[bh]) * (1.f / 448.f);
            if (!(ska > 0.f)) ska = 1.f;
            if (!(skb > 0.f)) skb = 1.f;
            cs_e = cs * sq_row * ska;
            cs_c = cs * sq_row * skb;
        }
        // pv_done[b] completes once per op on buffer b (ops b, b+2, ...): op m's completion
        // is phase m >> 1 of pv_done[m & 1].  The warps only ever wait for the LATEST op
        // issued on a buffer (the PV of op n cannot start before this warpgroup releases
        // P(n)), so the barrier is never two phases ahead of the awaited one and the parity
        // test is exact without observing every phase.  Nothing waits per op: S(n) is
        // written by QK(n), issued after PV(n-2), and tcgen05 ops execute in issue order.
        auto consume_op = [&](int op) {   // wait until the O-MMA of op `op` has completed
            if (op < 0) return;
            mbar_wait_sleep(&ctl.pv_done[op & 1], (op >> 1) & 1);
        };
        // parity of the next s_full phase of S buffer bi (one phase per S-type op on it)
        auto s_parity = [&](int bi) {
            const int c = bi == 0 ? sc0++ : (bi == 1 ? sc1++ : sc2++);
            return c & 1;
        };
        for (int n = 0; n < nops; ++n) {
            const int s = n & 1, bi = n % G_::NB;
            const int32_t op = ctl.ops[n];
            const int type = op_type(op), v = op_val(op);
            const uint32_t t_buf = tbase + lane_off + G_::COLS + 64 * bi;
            if constexpr (F8) cs = type == OP_E ? cs_e : cs_c;   // E4M3 dequantisation
            if (DIAG && type != OP_F && (p.dbg & 1)) {
                // diagnostics: skip the softmax arithmetic
                mbar_wait_sleep(&ctl.s_full[bi], s_parity(bi));
                if (warp == 4 && lane == 0) PASA_TR(TR_SA_OK, n);
            } else if (type != OP_F) {
                const int par = s_parity(bi);
                if (warp == 4 && lane == 0) PASA_TR(TR_SA_W, n);
                crit_wait(&ctl.s_full[bi], par, spin_s);
                if (warp == 4 && lane == 0) PASA_TR(TR_SA_OK, n);
                tc_fence_after();
                uint32_t sa[32], sb[32];
                tmem_ld32(t_buf, sa);
                tmem_ld32(t_buf + 32, sb);
                tmem_wait_ld();
                if (warp == 4 && lane == 0) PASA_TR(TR_SA_LD, n);
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
                    const int rem = NK32 - 64 * v;
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
                // raw logit of the ragged last block (C ops)
                float xlast = -INFINITY;
                if (clast >= 0) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        if (c == clast) xlast = __uint_as_float(sa[c]);
                        if (c + 32 == clast) xlast = __uint_as_float(sb[c]);
                    }
                }
                // Exponentials against the current reference m first (FFMA2 for s*x - m,
                // FADD2 sums).  If the row sum is below 2^8, every x - m < 8, so the rescale
                // rule (mx > m + 8) cannot fire and the row max is not needed; otherwise
                // (the first op: m = -inf gives NaN; or a possible new maximum) the exact max
                // decides as before and the exponentials are redone if m moved.  The m
                // sequence, and so every P, is the same as with the max taken every op.
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
                        float p0, p1, p2, p3;
                        constexpr int kPoly = D == 64 ? PASA_D64_POLY : 0;
                        if (kPoly > 0 && (2 * c) % kPoly == 0) {
                            const float2 pa = ex2_fma2(xa);
                            p0 = pa.x; p1 = pa.y;
                        } else {
                            p0 = ex2(xa.x); p1 = ex2(xa.y);
                        }
                        if (kPoly > 0 && (2 * c + 1) % kPoly == 0) {
                            const float2 pb = ex2_fma2(xb);
                            p2 = pb.x; p3 = pb.y;
                        } else {
                            p2 = ex2(xb.x); p3 = ex2(xb.y);
                        }
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
                    // raw row max (scale > 0 commutes), four independent chains
                    float mr0 = -INFINITY, mr1 = -INFINITY, mr2 = -INFINITY, mr3 = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 16; c += 2) {
                        mr0 = fmax3(mr0, __uint_as_float(sa[c]), __uint_as_float(sa[c + 1]));
                        mr1 = fmax3(mr1, __uint_as_float(sb[c]), __uint_as_float(sb[c + 1]));
                        mr2 = fmax3(mr2, __uint_as_float(sa[c + 16]), __uint_as_float(sa[c + 17]));
                        mr3 = fmax3(mr3, __uint_as_float(sb[c + 16]), __uint_as_float(sb[c + 17]));
                    }
                    const float mx = fmaxf(fmax3(mr0, mr1, mr2), mr3) * cs;
                    if (warp == 4 && lane == 0) PASA_TR(TR_SA_MAX, n);
                    const bool moved = mx > m + kRescaleThresh;
                    if (moved) {
                        corr = ex2(m - mx);       // 0 when m = -inf
                        resc = n > 0;
                        m = mx;
                        l *= corr;
                        A_cur *= corr;
                    }
                    // warp-uniform redo (lanes whose m did not move recompute the same
                    // values): no divergent path around the warp-collective TMEM store
                    if (__any_sync(0xffffffffu, moved)) exps(m);
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
                const float negm = -m;
                if (warp == 4 && lane == 0) PASA_TR(TR_SA_EXP, n);
                tmem_st32(t_buf, pk);
                if (type == OP_E) {
                    l += h0 + h1;
                } else {
                    // denominator: n_j * p_j; every dropped block has 64 tokens except the last
                    const float pl = clast >= 0 ? ex2(fmaf(xlast, cs, negm)) : 0.f;
                    l += 64.f * (h0 + h1) - (64.f - wlast) * pl;
                    if constexpr (EXP == 1) {
                        // small groups: 8-column sums of this chunk's P (bf16 as stored;
                        // the first-order weight is rounded to bf16 anyway, R-21)
#pragma unroll
                        for (int k8 = 0; k8 < 8; ++k8) {
                            float sgk = 0.f;
#pragma unroll
                            for (int q2 = 0; q2 < 4; ++q2) {
                                const float2 f = __bfloat1622float2(
                                    *reinterpret_cast<const __nv_bfloat162*>(&pk[4 * k8 + q2]));
                                sgk += f.x + f.y;
                            }
                            ctl.sg[k8][r] = sgk;
                        }
                        c_last = v;
                    }
                    // group sums A_{t,g} (each 32-block half lies in one group)
                    const int j0 = 64 * v;
                    const int g0 = j0 / G32;
                    if (g0 != g_cur) { A_cur = 0.f; g_cur = g0; }
                    A_cur += h0;
                    if (j0 + 32 < NK32) {
                        const int g1 = (j0 + 32) / G32;
                        if (g1 != g0) { A_done = A_cur; g_done = g0; A_cur = h1; g_cur = g1; }
                        else A_cur += h1;
                    }
                }
                tmem_wait_st();
                if (warp == 4 && lane == 0) PASA_TR(TR_SA_ST, n);
            } else {
                // F(g): write Aq = bf16(s * A_{t,g} * q_t) into the TMEM A buffer
                // (packed bf16x2 multiply: w is rounded to bf16 once, R-21)
                float A = v == g_done ? A_done : A_cur;
                if constexpr (EXP == 1) {            // group v of the last C op's chunk
                    const int kg = v - (64 * c_last) / p.G;
                    A = 0.f;
#pragma unroll
                    for (int k8 = 0; k8 < 8; ++k8) {
                        if (p.G == 8 && kg == k8) A = ctl.sg[k8][r];
                        if (p.G == 16 && 2 * kg == k8) A = ctl.sg[k8][r] + ctl.sg[k8 + 1][r];
                    }
                }
                const float w = p.s * A;
                const uint32_t w2 = pack_bf16(w, w);
                // the buffer's previous reader (op n-NB) has finished: wait for op n-2 (PVs
                // complete in order, so this covers n-3 at NB = 3).  Not n-1: a parity wait is
                // exact only while the barrier is at most one phase behind, and on entry to an
                // F op only PV(n-4) is known complete (an F op has no s_full wait; the previous
                // op's S(n-1) was computed by a QK issued before PV(n-3)), so pv_done[(n-1)&1]
                // may still be at op n-3's phase -- a wait for n-1 would then pass at once
                // (the round-1 d = 64 hang / NaN under changed softmax timing).  Op n-2 is
                // safe: its predecessor on the barrier, n-4, is complete.
                consume_op(G_::NB == 1 ? n - 1 : n - 2);   // NB = 1: the buffer held P(n - 1)
                tc_fence_after();
#pragma unroll
                for (int a = 0; a < G_::NBOX; ++a) {
                    uint32_t aq[32];
                    if constexpr (F8) {
                        // q_t = sq_row * Q8[t]: 16-byte chunk c of the row holds dims 16c..16c+15
                        const float wq = w * sq_row;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int cc = 4 * a + c;
                            const uint4 u = *reinterpret_cast<const uint4*>(
                                qrow + r * 128 + ((cc ^ (r & 7)) << 4));
                            const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 f0 = e4m3x2_to_float2((uint16_t)(wd[e] & 0xffffu));
                                const float2 f1 = e4m3x2_to_float2((uint16_t)(wd[e] >> 16));
                                aq[c * 8 + 2 * e] = pack_bf16(f0.x * wq, f0.y * wq);
                                aq[c * 8 + 2 * e + 1] = pack_bf16(f1.x * wq, f1.y * wq);
                            }
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const uint4 u = *reinterpret_cast<const uint4*>(
                                qrow + a * G_::QBOX + r * 128 + ((c ^ (r & 7)) << 4));
                            aq[c * 4 + 0] = hmul2_bf16(u.x, w2);
                            aq[c * 4 + 1] = hmul2_bf16(u.y, w2);
                            aq[c * 4 + 2] = hmul2_bf16(u.z, w2);
                            aq[c * 4 + 3] = hmul2_bf16(u.w, w2);
                        }
                    }
                    tmem_st32(t_buf + 32 * a, aq);
                }
                tmem_wait_st();
            }
            tc_fence_before();
            if (PASA_WARP_ARRIVE) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&ctl.p_full[bi]);
            } else {
                mbar_arrive(&ctl.p_full[bi]);
            }
            if (warp == 4 && lane == 0) PASA_TR(TR_SA_ARR, n);
        }
        // ---- epilogue: O / l -> bf16 -> global ----
        consume_op(nops - 2);
        consume_op(nops - 1);
        tc_fence_after();
        const int64_t t = i * kBQ + r;
        const float inv = 1.f / l;
        __nv_bfloat16* orow = p.out + b * p.osB + h * p.osH + t * p.osS;
        if (p.oP > 0 && t < p.S) {   // the output half of the fused Ulysses exchange
            int sh = 0;
            while (sh + 1 < p.oP && t >= p.ostart[sh + 1]) ++sh;
            orow = p.obase[sh] + (t - p.ostart[sh]) * p.oSS + h * p.oSH;
        }
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
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
                     size_t why_len, const ZcShards* osh) {
    CUtensorMap mQ, mK, mV, mKb, mVs, mHt;
    auto act = [&](CUtensorMap* m, const pasa_tensor& t, uint32_t rows) {
        uint64_t dims[4] = {(uint64_t)t.D, (uint64_t)t.S, (uint64_t)t.H, (uint64_t)t.B};
        uint64_t str[3] = {(uint64_t)t.sS * 2, (uint64_t)t.sH * 2, (uint64_t)t.sB * 2};
        uint32_t box[4] = {64, rows, 1, 1};
        return make_tensor_map(m, t.data, 4, dims, str, box, why, why_len);
    };
    const bool f8 = r->cfg.qk_fp8 != 0;
    if (!act(&mV, v, kBK)) return cudaErrorNotSupported;
    if (f8) {   // E4M3 copies [BH][S][D] / [BH][N_K][D], 128-byte rows
        auto u8map = [&](CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
            uint64_t dims[3] = {(uint64_t)D, rows, (uint64_t)r->BH};
            uint64_t str[2] = {(uint64_t)D, rows * D};
            uint32_t box[3] = {(uint32_t)D, box_rows, 1};
            return make_tensor_map(m, base, 3, dims, str, box, why, why_len, true);
        };
        if (!u8map(&mQ, r->q8, (uint64_t)r->S, kBQ) || !u8map(&mK, r->k8, (uint64_t)r->S, kBK) ||
            !u8map(&mKb, r->kb8, (uint64_t)r->NK, 64))
            return cudaErrorNotSupported;
    } else if (!act(&mQ, q, kBQ) || !act(&mK, k, kBK)) {
        return cudaErrorNotSupported;
    }
    {
        uint64_t dims[3] = {(uint64_t)D, (uint64_t)r->NK, (uint64_t)r->BH};
        uint64_t str[2] = {(uint64_t)D * 2, (uint64_t)r->NK * D * 2};
        uint32_t box[3] = {64, 64, 1};
        if ((!f8 && !make_tensor_map(&mKb, r->kbar_lp, 3, dims, str, box, why, why_len)) ||
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
    prm.sq = r->sq8; prm.kamax = r->kamax; prm.kbamax = r->kbamax;
    prm.oP = 0;
    if (osh) {
        prm.oP = osh->P;
        for (int s = 0; s <= osh->P; ++s) prm.ostart[s] = osh->start[s];
        for (int s = 0; s < osh->P; ++s)
            prm.obase[s] = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(osh->base[s])) +
                           r->cfg.head_offset * osh->sH;
        prm.oSS = osh->sS;
        prm.oSH = osh->sH;
    }
    prm.trace = g_trace_buf;
    prm.trace_x = g_trace_x;
    prm.trace_y = g_trace_y;
    prm.dbg = g_dbg;
    // request >= 80 KB so at most two CTAs share an SM (2 x 256 TMEM columns; a third
    // would block in tcgen05.alloc) while two still fit next to the static Ctl
    size_t smem = (size_t)Geo<D>::BYTES + 1024;
    if (smem < (r->cfg.G < 32 ? 80 : 100) * 1024) smem = (r->cfg.G < 32 ? 80 : 100) * 1024;
    // g_dbg bits 0-5 select the diagnostics instantiation
    const bool diag = (g_dbg & 63) != 0 || g_trace_buf != nullptr;
    const bool small_groups = r->cfg.comp == PASA_COMP_GROUPED && r->cfg.G < 32;
    // EXP 1: groups of 8 or 16 blocks (per-8-column sums in shared memory); the G >= 32
    // instantiation carries none of that code
    auto kern = small_groups ? (diag ? attn_sm100_kernel<D, true, 1> : attn_sm100_kernel<D, false, 1>)
                             : (diag ? attn_sm100_kernel<D, true, 0> : attn_sm100_kernel<D, false, 0>);
    if (f8) {
        if (D != 128 || small_groups || diag) {
            snprintf(why, why_len, "FP8 QK^T: d = 128, G >= 32, no diagnostics");
            return cudaErrorNotSupported;
        }
        kern = attn_sm100_kernel<D, false, 0, true>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    prm.it0 = r->it0;
    const unsigned grid = (unsigned)(r->it1 - r->it0);   // head-major items
    kern<<<grid, kThreads, smem, st>>>(mQ, mK, mV, mKb, mVs, mHt, prm);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                              pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                              int* launches, char* why, size_t why_len, const ZcShards* osh) {
    if (r->cfg.Bq != kBQ || r->cfg.Bk != kBK) {
        snprintf(why, why_len, "needs Bq=128, Bk=64");
        return cudaErrorNotSupported;
    }
    if (r->cfg.comp == PASA_COMP_GROUPED && !sm100_supports_group(r->cfg.G, r->NK)) {
        snprintf(why, why_len, "grouped compensation with G = %d (supported: 8, 16, 32, 64, "
                 "multiples of 128, >= N_K)", r->cfg.G);
        return cudaErrorNotSupported;
    }
    if (r->NK > kMaxNK) {
        snprintf(why, why_len, "N_K > %d", kMaxNK);
        return cudaErrorNotSupported;
    }
    cudaError_t e = r->D == 128 ? launch_d<128>(q, k, v, r, out, st, why, why_len, osh)
                                : launch_d<64>(q, k, v, r, out, st, why, why_len, osh);
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace pasa
