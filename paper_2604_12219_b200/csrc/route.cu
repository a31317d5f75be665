// route.cu -- pasa_route: block pooling, block scores, stochastic bias and
// top-k selection (PAPER.md:189-193, Eq. 8 at :229-233, :296-308; readings
// R-6..R-14 and R-20 of DESIGN.md §3).
//
// Bit-exactness contract with the fp64 oracle: pooling sums
// tokens in ascending order in fp64; scores are fma chains over the head
// dimension in ascending order; row mean / std are sequential in j; the bias
// is two separately rounded operations.  This translation unit is compiled
// with --fmad=false and uses __d*_rn intrinsics so nvcc contracts nothing.
#include <cuda_bf16.h>

#include <cstdlib>

#include "pasa_internal.h"
#include "philox.cuh"
#include "fastlog.cuh"
#include "sm100_ptx.cuh"

namespace pasa {
namespace {

// ---------------------------------------------------------------------------
// a2: block means.  One thread per (head, block, 8 consecutive dims); the
// thread walks the block's tokens in ascending order (R1).  A warp covers
// 4 (bf16, D=128: 16 lanes per token row) consecutive dims groups of two
// blocks, so every load instruction reads whole 256-byte rows.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void load8(const T* p, double v[8]) {
    if constexpr (sizeof(T) == 2) {
        uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __bfloat162float(b[i].x);
            v[2 * i + 1] = __bfloat162float(b[i].y);
        }
    } else {
        float4 a = __ldg(reinterpret_cast<const float4*>(p));
        float4 c = __ldg(reinterpret_cast<const float4*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
    }
}

struct PoolArgs {
    const void* x;
    int64_t sB, sS, sH;
    int64_t S, H, D;
    int32_t bsz;    // block size in tokens
    int64_t nblk;   // blocks per head
    int64_t blk0, ntask;   // ntask > 0: all ntask blocks of every head; 0: items [blk0, ...)
    double* out;    // [BH][nblk][D]
    double* frag;   // optional DMMA B-fragment copy [BH][ceil(nblk/8)][D/8][8][4][2]
    // FP8 QK^T variant (cfg.qk_fp8, reading R-30), pool_kernel<T, true> only:
    uint8_t* f8;          // Q: E4M3 copy [BH][S][D], row t scaled by 1 / f8scale[t]
    float* f8scale;       // Q: [BH][S] per-row scales (row amax / 448)
    uint32_t* amax;       // K: [BH] max |K| per head (float bits; the statistics pass
                          //    quantises K with it)
    uint32_t* bamax;      // K: [BH] max |Kbar| per head
};

__device__ __forceinline__ float group_max(float v, int ng, int lane) {
    const unsigned m = (ng == 32 ? 0xffffffffu : ((1u << ng) - 1u) << (lane & ~(ng - 1)));
    for (int o = 1; o < ng; o <<= 1) v = fmaxf(v, __shfl_xor_sync(m, v, o));
    return v;
}

// F8 (the FP8 QK^T variant): also the E4M3 copy of Q with per-row scales (the ng = D / 8
// threads of a block are adjacent lanes: one group max per token) and the per-head
// max |K|, max |Kbar|; the ng-lane groups are whole (total, q_tasks multiples of ng)
// one thread's pool task (task < q_tasks: Q, else K)
template <typename T, bool F8>
__device__ __forceinline__ void pool_task(const PoolArgs& qa, const PoolArgs& ka, int64_t q_tasks,
                                          int64_t task) {
    const PoolArgs& a = task < q_tasks ? qa : ka;
    if (task >= q_tasks) task -= q_tasks;
    int64_t ng = a.D / 8;
    int64_t dg = task % ng;
    // Q: items blk0 + rest of the flattened (head, block) list; K: every block of every head
    int64_t rest = task / ng;
    int64_t blk, bh;
    if (a.ntask > 0) { blk = rest % a.ntask; bh = rest / a.ntask; }
    else { blk = (a.blk0 + rest) % a.nblk; bh = (a.blk0 + rest) / a.nblk; }
    int64_t b = bh / a.H, h = bh % a.H;
    int64_t t0 = blk * a.bsz;
    int64_t t1 = min(t0 + (int64_t)a.bsz, a.S);
    const T* base = reinterpret_cast<const T*>(a.x) + b * a.sB + h * a.sH + dg * 8;
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    int64_t t = t0;
    const int lane = threadIdx.x & 31;
    const bool isq = a.f8 != nullptr;
    float kam = 0.f;                       // F8, K tasks: max |K| of this thread's values
    // F8: the E4M3 row (Q) / running max (K) of one token's 8 values
    auto f8_row = [&](const double (&v)[8], int64_t tt) {
        if constexpr (F8) {
            float m = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf((float)v[i]));
            if (isq) {
                m = group_max(m, (int)ng, lane);
                const float sc = m > 0.f ? m * (1.f / 448.f) : 1.f;
                const float inv = 1.f / sc;
                uint2 r;
                r.x = (uint32_t)ptx::cvt_e4m3x2((float)v[0] * inv, (float)v[1] * inv) |
                      ((uint32_t)ptx::cvt_e4m3x2((float)v[2] * inv, (float)v[3] * inv) << 16);
                r.y = (uint32_t)ptx::cvt_e4m3x2((float)v[4] * inv, (float)v[5] * inv) |
                      ((uint32_t)ptx::cvt_e4m3x2((float)v[6] * inv, (float)v[7] * inv) << 16);
                *reinterpret_cast<uint2*>(a.f8 + (bh * a.S + tt) * a.D + dg * 8) = r;
                if (dg == 0) a.f8scale[bh * a.S + tt] = sc;
            } else {
                kam = fmaxf(kam, m);
            }
        }
    };
    // 4 rows in flight, summed strictly in token order
    for (; t + 4 <= t1; t += 4) {
        double v0[8], v1[8], v2[8], v3[8];
        load8<T>(base + (t + 0) * a.sS, v0);
        load8<T>(base + (t + 1) * a.sS, v1);
        load8<T>(base + (t + 2) * a.sS, v2);
        load8<T>(base + (t + 3) * a.sS, v3);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[i] = __dadd_rn(acc[i], v0[i]);
            acc[i] = __dadd_rn(acc[i], v1[i]);
            acc[i] = __dadd_rn(acc[i], v2[i]);
            acc[i] = __dadd_rn(acc[i], v3[i]);
        }
        f8_row(v0, t); f8_row(v1, t + 1); f8_row(v2, t + 2); f8_row(v3, t + 3);
    }
    for (; t < t1; ++t) {
        double v0[8];
        load8<T>(base + t * a.sS, v0);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __dadd_rn(acc[i], v0[i]);
        f8_row(v0, t);
    }
    double n = (double)(t1 - t0);
    double m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = __ddiv_rn(acc[i], n);
    // 16-byte stores (a warp's scalar 8-byte stores would each touch 32 sectors)
    double2* o = reinterpret_cast<double2*>(a.out + (bh * a.nblk + blk) * a.D + dg * 8);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = make_double2(m[2 * i], m[2 * i + 1]);
    if (a.frag) {
        // fragment order of the fused route kernel's B operand: block j = 8 ct + fr, dims
        // 8 dg + 4 h + fk -> [ct][dg][fr][fk][h] (one 512-byte run per (ct, dg): a warp's
        // 16-byte loads of two consecutive k-steps are contiguous)
        double2* f = reinterpret_cast<double2*>(
            a.frag + ((bh * ((a.nblk + 7) / 8) + blk / 8) * (a.D / 8) + dg) * 64 + (blk % 8) * 8);
#pragma unroll
        for (int fk = 0; fk < 4; ++fk) f[fk] = make_double2(m[fk], m[4 + fk]);
    }
    if constexpr (F8) {
        if (!isq) {   // per-head max |K| and max |Kbar| (non-negative floats order as bits)
            float bm = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) bm = fmaxf(bm, fabsf((float)m[i]));
            kam = group_max(kam, (int)ng, lane);
            bm = group_max(bm, (int)ng, lane);
            if (dg == 0) {
                atomicMax(a.amax + bh, __float_as_uint(kam));
                atomicMax(a.bamax + bh, __float_as_uint(bm));
            }
        }
    }
}

template <typename T, bool F8>
// 4 CTAs (32 warps) per SM: at 3 (70 registers) the kernel lost 40% of its bandwidth
__global__ void __launch_bounds__(256, 4) pool_kernel(PoolArgs qa, PoolArgs ka, int64_t q_tasks,
                                                   int64_t total) {
    const int64_t task = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (task < total) pool_task<T, F8>(qa, ka, q_tasks, task);
}

// ---------------------------------------------------------------------------
// Zero-copy sequence parallelism ("Ulysses all-to-all fused with
// attention over NVLink"): the rank's heads of q, k, v are read straight from every rank's
// sequence shard through peer pointers, copied into this rank's local [1, S, Hl, D] buffers
// and -- for q and k -- pooled in the same pass (the same ascending-token fp64 sums as
// pool_task, so Qbar / Kbar are bitwise those of the single-GPU path).  The input half of
// the Ulysses exchange is thereby fused into the route's pooling pass; the output half is
// the attention epilogue storing each row into its owner's shard (attn_sm100.cu).
// One thread per (tensor, local head, block, 8 consecutive dims), tasks q | k | v.
// ---------------------------------------------------------------------------
struct ZcArgs {
    ZcShards src[3];                 // q, k, v shards (element offsets per token / head)
    __nv_bfloat16* loc[3];           // local q, k, v [1][S][Hl][D]
    int64_t lsS[3], lsH[3];          // local strides
    int64_t S, Hl, D, head0;
    int32_t bsz[3];                  // block size of the task's tensor (Bq, Bk, Bk)
    int64_t nblk[3];                 // blocks per head
    int64_t it0, it1;                // the handle's (head, q-block) items (q pooled only there)
    double* out[2];                  // Qbar [Hl][NQ][D], Kbar [Hl][NK][D]
    double* kfrag;                   // Kbar in DMMA B-fragment order
    int64_t ntask[3];                // tasks per tensor
};

__global__ void __launch_bounds__(256, 4) zc_gather_pool_kernel(ZcArgs a) {
    int64_t task = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int x = 0;
    while (x < 3 && task >= a.ntask[x]) { task -= a.ntask[x]; ++x; }
    if (x == 3) return;
    const int64_t ng = a.D / 8;
    const int64_t dg = task % ng, rest = task / ng;
    const int64_t blk = rest % a.nblk[x], h = rest / a.nblk[x];
    const int64_t t0 = blk * a.bsz[x], t1 = min(t0 + (int64_t)a.bsz[x], a.S);
    const ZcShards& sh = a.src[x];
    const bool pool = x < 2 && (x == 1 || (h * a.nblk[0] + blk >= a.it0 && h * a.nblk[0] + blk < a.it1));
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    int s = 0;
    while (s + 1 < sh.P && t0 >= sh.start[s + 1]) ++s;
    __nv_bfloat16* dst = a.loc[x] + h * a.lsH[x] + dg * 8;
    for (int64_t t = t0; t < t1; ++t) {
        while (s + 1 < sh.P && t >= sh.start[s + 1]) ++s;   // a block may straddle shards
        const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(sh.base[s]) +
                                   (t - sh.start[s]) * sh.sS + (a.head0 + h) * sh.sH + dg * 8;
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(src));
        *reinterpret_cast<uint4*>(dst + t * a.lsS[x]) = u;
        if (pool) {
            const __nv_bfloat162* bv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[2 * i] = __dadd_rn(acc[2 * i], (double)__bfloat162float(bv[i].x));
                acc[2 * i + 1] = __dadd_rn(acc[2 * i + 1], (double)__bfloat162float(bv[i].y));
            }
        }
    }
    if (!pool) return;
    const double n = (double)(t1 - t0);
    double m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = __ddiv_rn(acc[i], n);
    double2* o = reinterpret_cast<double2*>(a.out[x] + (h * a.nblk[x] + blk) * a.D + dg * 8);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = make_double2(m[2 * i], m[2 * i + 1]);
    if (x == 1) {   // the fused kernel's B-fragment copy of Kbar (as pool_task)
        double2* f = reinterpret_cast<double2*>(
            a.kfrag + ((h * ((a.nblk[1] + 7) / 8) + blk / 8) * (a.D / 8) + dg) * 64 + (blk % 8) * 8);
#pragma unroll
        for (int fk = 0; fk < 4; ++fk) f[fk] = make_double2(m[fk], m[4 + fk]);
    }
}

// ---------------------------------------------------------------------------
// shared helpers of the fused kernel
// ---------------------------------------------------------------------------
// fp64 tensor core: d (+)= a * b on an 8x8x4 tile.  Measured on this pool
// (tools/dmma_exact.cu, 0 of 38 M outputs differ): bit-identical to the sequential fma
// chain over k = 0..3, so a chain of these in ascending k reproduces the oracle's
// ascending-d fma chain (R2).  PTX does not promise that rounding, so the parity contract
// the tests check is the tie-tolerant one (a route may differ only where two
// oracle scores tie within 1e-6 relative); the observed tie count is 0.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint64_t orderable(double x) {
    x = __dadd_rn(x, 0.0);  // -0.0 -> +0.0: the oracle's double compare treats them as equal
    uint64_t b = (uint64_t)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ int device_k(const BudgetRec* rec, int64_t NK) {
    double kf = floor(__dadd_rn(__dmul_rn(rec->rho_t, (double)NK), 0.5));   // R-14
    int64_t k = kf > (double)NK ? NK : (int64_t)kf;
    if (k < 1) k = 1;
    if (k > NK) k = NK;
    return (int)k;
}

// ---------------------------------------------------------------------------
// a3 + a4 + a5 fused (the route's hot kernel): one CTA per (head, 8 query-block
// rows), two CTAs per SM.  The fp64 scores of its rows against every KV block are
// computed on the fp64 tensor core into SHARED memory and never leave the chip;
// sigma_i, the Philox / Gumbel bias and the top-k threshold search run from there.
//
//   phase A  (all 8 warps) DMMA m8n8k4: the 8 Qbar rows are the A operand (shared
//            memory), Kbar the B operand straight from L2 into registers (4 k-steps
//            per block, two blocks in flight), groups of 4 column tiles round-robin
//            over the warps, no barrier inside the phase; r_ij = s * acc (+ prior_j)
//   phase B  (warp w = row w) sigma_i with the oracle's sequential sums (R3), every
//            lane walking the row (broadcast reads: no divergence)
//   phase C  (same warp) keys r~ = r + (beta sigma_i) g (two rounded operations, R5)
//            written over the row in place, k-th largest by a bitwise threshold search
//            over the shared-memory keys, idx / mask / count out (R6, R-13)
//
// Two co-resident CTAs interleave their phases on the SM (fp64 tensor pipe in A,
// integer / fp64 CUDA-core work in C).  When the score rows do not fit in shared
// memory (N_K > ~1,570 at 2 CTAs/SM) they live in a global scratch slice of the
// workspace (same code; written and read back by the same CTA, so it stays in L2).
// ---------------------------------------------------------------------------
constexpr int kFCG4 = 4;               // column tiles x row tiles per warp work group
constexpr int kFKS = 4;                // k-steps per register block (phase A)
constexpr int kFRows = 8;              // score rows per CTA (one DMMA row tile)
constexpr int kFHR = 40;               // key high words per lane held in registers (N_K <= 1280)
struct FusedArgs {
    const double* qbar;        // [BH][NQ][D]
    const double* kfrag;       // Kbar in B-fragment order (pool_kernel)
    const double* prior;       // [BH][NK] or nullptr
    const BudgetRec* rec;
    int64_t NQ, NK, W, H, H_total, head_offset;
    int64_t it0, it1;          // (head, q-block) items routed: [it0, it1), item = bh NQ + i
    int D, NKP;                // NKP: odd row stride of the score rows (doubles)
    double s, beta;
    uint32_t key0, key1, step;
    int32_t* idx;              // [BH][NQ][NK]
    int32_t* count;            // [BH][NQ]
    uint32_t* mask;            // [BH][NQ][W]
    int32_t* hdr;
    double* gsc;               // global score rows [BH][NQ][NKP] when !SMEM_SC
};

__device__ const LogEnt g_logtab[128] = PASA_LOGTAB_INIT;

// Gumbel variate from one Philox word x (R4, R-12): g = -log(-log u), u = (x + 1/2) 2^-32,
// with the table-driven fp64 log of fastlog.cuh (within 1.5 ulp of the exact log; glibc's,
// which the oracle uses, is within 0.52: r~ moves by ~1e-16 relative, inside the
// documented-tie margin).  Word j mod 4 of counter (floor(j/4), i, gh, step) serves block j
// (R-11): one Philox call per four blocks.
// `tab`: the log table staged in shared memory by the calling CTA (in L1 it was evicted by
// the streamed K-bar fragments: its loads were the fused kernel's top stall)
__device__ __forceinline__ double gumbel_of(uint32_t x, const LogEnt* tab) {
    const double u = __dmul_rn(__dadd_rn((double)x, 0.5), 2.3283064365386963e-10);
    return -fastlog_tab(tab, -fastlog_tab(tab, u));
}

// The k-th largest orderable key T of one row (the largest value with #{key >= T} >= k),
// ties at T to the smallest j (R-13); writes the ascending index list, the mask words
// and the count.  The keys live in shared (or L2-resident global) memory, one row per
// warp: element j at key[j], j < NK.  Upper 32 bits first (32-bit reads of the high
// words), then, once the top 16 bits of T are fixed, the keys sharing them (usually a
// few dozen) are compacted to two registers per lane and the rest is searched there.
// HR > 0: the caller also holds the high words of the lane's keys (j = 32 m + lane) in
// registers hr[m] (0 where j >= NK), so the first 16 bits are searched without memory reads.
template <int HR>
__device__ __forceinline__ void select_row_mem(const uint64_t* key, int NK, int k, int lane,
                                               uint64_t* cb, int32_t* orow, uint32_t* mrow,
                                               int32_t* cnt, const uint32_t (&hr)[HR > 0 ? HR : 1]) {
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(key) + 1;   // high words, stride 2
    const int M = (NK + 31) >> 5;
    auto count_ge = [&](uint32_t cand) {
        int c = 0;
        if constexpr (HR > 0) {
#pragma unroll
            for (int m = 0; m < HR; ++m) c += hr[m] >= cand;
        } else {
            for (int j = lane; j < NK; j += 32) c += hw[2 * j] >= cand;
        }
        return c;
    };
    uint64_t kand = ~0ull, kor = 0ull;
    for (int j = lane; j < NK; j += 32) { const uint64_t x = key[j]; kand &= x; kor |= x; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kand &= __shfl_xor_sync(0xffffffffu, kand, o);
        kor |= __shfl_xor_sync(0xffffffffu, kor, o);
    }
    const uint64_t diff = kand ^ kor;
    uint64_t T = diff ? (kand & ~((2ull << (63 - __clzll(diff))) - 1ull)) : kand;
    const int top = diff ? 63 - __clzll(diff) : -1;
    uint32_t T_hi = (uint32_t)(T >> 32);
    int bpos = top;
    for (; bpos >= 48; --bpos) {
        const uint32_t cand = T_hi | (1u << (bpos - 32));
        const int c = __reduce_add_sync(0xffffffffu, count_ge(cand));
        if (c >= k) T_hi = cand;
    }
    bool done = false;
    if (top >= 48) {
        const uint32_t tw = T_hi >> 16;
        int gw = 0, ew = 0;
        if constexpr (HR > 0) {
#pragma unroll
            for (int m = 0; m < HR; ++m) {
                const uint32_t h16 = hr[m] >> 16;
                gw += h16 > tw;
                ew += h16 == tw && hr[m] != 0u;   // absent blocks hold 0
            }
        } else {
            for (int j = lane; j < NK; j += 32) {
                const uint32_t h16 = hw[2 * j] >> 16;
                gw += h16 > tw;
                ew += h16 == tw;
            }
        }
        gw = __reduce_add_sync(0xffffffffu, gw);
        ew = __reduce_add_sync(0xffffffffu, ew);
        if (ew <= 64) {
            const uint32_t lt = (1u << lane) - 1u;
            int base = 0;
            for (int m = 0; m < M; ++m) {
                const int j = 32 * m + lane;
                const bool in = j < NK && (hw[2 * j] >> 16) == tw;
                const uint32_t b = __ballot_sync(0xffffffffu, in);
                if (in) cb[base + __popc(b & lt)] = key[j];
                base += __popc(b);
            }
            __syncwarp();
            const uint64_t c0 = lane < ew ? cb[lane] : 0ull;
            const uint64_t c1 = lane + 32 < ew ? cb[lane + 32] : 0ull;
            __syncwarp();
            uint64_t Tc = (uint64_t)T_hi << 32;
            for (; bpos >= 0; --bpos) {
                const uint64_t cand = Tc | (1ull << bpos);
                const int c = gw + __reduce_add_sync(0xffffffffu, (c0 >= cand) + (c1 >= cand));
                if (c >= k) Tc = cand;
            }
            T = Tc;
            done = true;
        }
    }
    if (!done) {
        for (; bpos >= 32; --bpos) {
            const uint32_t cand = T_hi | (1u << (bpos - 32));
            int c = 0;
            for (int j = lane; j < NK; j += 32) c += hw[2 * j] >= cand;
            c = __reduce_add_sync(0xffffffffu, c);
            if (c >= k) T_hi = cand;
        }
        uint32_t T_lo = top >= 32 ? 0u : (uint32_t)T;
        if (top >= 0) {
            int gtc = 0;
            for (int j = lane; j < NK; j += 32) gtc += hw[2 * j] > T_hi;
            gtc = __reduce_add_sync(0xffffffffu, gtc);
            for (int b = min(top, 31); b >= 0; --b) {
                const uint32_t cand = T_lo | (1u << b);
                int c = 0;
                for (int j = lane; j < NK; j += 32) {
                    const uint64_t x = key[j];
                    c += (uint32_t)(x >> 32) == T_hi && (uint32_t)x >= cand;
                }
                c = gtc + __reduce_add_sync(0xffffffffu, c);
                if (c >= k) T_lo = cand;
            }
        }
        T = ((uint64_t)T_hi << 32) | T_lo;
    }
    int gt = 0;
    for (int j = lane; j < NK; j += 32) gt += key[j] > T;
    const int need = k - __reduce_add_sync(0xffffffffu, gt);   // keys equal to T to take
    int taken_eq = 0, pos = 0;
    const uint32_t below = (1u << lane) - 1u;
    for (int m = 0; m < M; ++m) {
        const int j = 32 * m + lane;
        const uint64_t x = j < NK ? key[j] : 0ull;
        const uint32_t eqb = __ballot_sync(0xffffffffu, x == T && j < NK);
        const int eq_rank = taken_eq + __popc(eqb & below);
        const bool take = j < NK && (x > T || (x == T && eq_rank < need));
        taken_eq += __popc(eqb);
        const uint32_t sel = __ballot_sync(0xffffffffu, take);
        if (take) orow[pos + __popc(sel & below)] = j;
        pos += __popc(sel);
        if (lane == 0) mrow[m] = sel;
    }
    if (lane == 0) *cnt = k;
}

// HR > 0 (N_K <= 32 HR): the high words of a row's keys stay in registers for the search
// One CTA's route tile: 8 query-block rows `tile` of head bh.
template <int R, int D, bool SMEM_SC, int HR>
__device__ __forceinline__ void route_tile(const FusedArgs& a, int64_t bh, int64_t tile,
                                           unsigned char* f_smem) {
    constexpr int NT = 32 * R, NW = R;              // one warp per score row
    constexpr int RT = R / 8;                       // DMMA row tiles (all in every warp)
    constexpr int CG = kFCG4 / RT;                  // column tiles per work group
    constexpr int KB = D / (4 * kFKS);              // register blocks per group (even)
    static_assert(KB % 2 == 0, "ping-pong blocks must pair up inside a group");
    const int NK = (int)a.NK, NKP = a.NKP;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // rows of this CTA inside the item range: [rlo, rhi) of i0 .. i0 + R - 1
    const int64_t i0 = tile * R;
    const int64_t ilo = max(a.it0 - bh * a.NQ, (int64_t)0), ihi = min(a.it1 - bh * a.NQ, a.NQ);
    const int rlo = (int)max(ilo - i0, (int64_t)0);
    const int nrows = (int)max(min((int64_t)R, ihi - i0), (int64_t)0);   // rows < nrows exist
    if (tile == 0 && bh == 0 && threadIdx.x == 0)   // k of this route, for pasa_route_read
        a.hdr[0] = device_k(a.rec, (int)a.NK);            // (written even if CTA (0, 0) has no item)
    if (rlo >= nrows) return;                       // no item of this CTA is in range
    double* sq = reinterpret_cast<double*>(f_smem);                    // [R][D + 4]
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(sq + R * (D + 4));    // [NW][64]
    LogEnt* ltab = reinterpret_cast<LogEnt*>(cbuf + NW * 64);           // [128] log table
    double* sc = SMEM_SC ? reinterpret_cast<double*>(ltab + 128)
                         : a.gsc + (bh * a.NQ + i0) * (int64_t)NKP;     // [R][NKP]

    const int k = device_k(a.rec, NK);
    const int M = (NK + 31) >> 5;
    if (k >= NK) {   // dense step / full budget: every block exact, no scores needed
        if (warp >= rlo && warp < nrows) {   // (one row per warp: R = 8)
            const int64_t row = bh * a.NQ + i0 + warp;
            int32_t* orow = a.idx + row * NK;
            uint32_t* mrow = a.mask + row * a.W;
            for (int j = lane; j < NK; j += 32) orow[j] = j;
            for (int w = lane; w < M; w += 32) {
                const int rem = NK - 32 * w;
                mrow[w] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
            }
            if (lane == 0) a.count[row] = NK;
        }
        return;
    }

    // ---- phase A: scores -------------------------------------------------------------
    // Every warp holds all R rows (RT row tiles) and works through groups of CG column
    // tiles (8 KV blocks each), groups round-robin over the warps.  B fragments (Kbar,
    // fragment order) come from L2 as 16-byte loads of two k-steps straight into
    // registers, a block of 4 k-steps ahead; A fragments (Qbar) from shared memory.
    const double* Q = a.qbar + (bh * a.NQ + i0) * D;
    for (int e = tid; e < R * D; e += NT) {
        const int r = e / D, c = e % D;
        sq[r * (D + 4) + c] = r >= rlo && r < nrows ? Q[(int64_t)r * D + c] : 0.0;
    }
    for (int e = tid; e < 128 * (int)sizeof(LogEnt) / 16; e += NT)
        reinterpret_cast<uint4*>(ltab)[e] = reinterpret_cast<const uint4*>(g_logtab)[e];
    __syncthreads();
    {
        const int fr = lane >> 2, fk = lane & 3;
        const int ntiles = (NK + 7) >> 3;
        const int ngroups = (ntiles + CG - 1) / CG;
        const int mygroups = warp < ngroups ? (ngroups - 1 - warp) / NW + 1 : 0;
        const double2* KF = reinterpret_cast<const double2*>(a.kfrag) +
                            bh * (int64_t)ntiles * (D / 8) * 32 + lane;
        const double* arow = sq + fr * (D + 4) + fk;
        auto load_blk = [&](double (&bb)[kFKS][CG], int g, int kb) {
#pragma unroll
            for (int c = 0; c < CG; ++c) {
                const int ct = g * CG + c;
                const bool ok = ct * 8 + fr < NK;
#pragma unroll
                for (int q = 0; q < kFKS / 2; ++q) {
                    const double2* src = KF + ((int64_t)ct * (D / 8) + kb * (kFKS / 2) + q) * 32;
                    const double2 v = ok ? __ldg(src) : make_double2(0.0, 0.0);
                    bb[2 * q][c] = v.x;
                    bb[2 * q + 1][c] = v.y;
                }
            }
        };
        double acc[RT][CG][2];
#pragma unroll
        for (int t = 0; t < RT; ++t)
#pragma unroll
            for (int c = 0; c < CG; ++c) acc[t][c][0] = acc[t][c][1] = 0.0;
        double bb[2][kFKS][CG];
        if (mygroups > 0) load_blk(bb[0], warp, 0);
        for (int gi = 0; gi < mygroups; ++gi) {
            const int g = warp + NW * gi;
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                if (kb + 1 < KB) load_blk(bb[(kb + 1) & 1], g, kb + 1);
                else if (gi + 1 < mygroups) load_blk(bb[(kb + 1) & 1], g + NW, 0);
#pragma unroll
                for (int u = 0; u < kFKS; ++u) {           // ascending d: the fma chain of R2
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const double av = arow[t * 8 * (D + 4) + kb * 4 * kFKS + 4 * u];
#pragma unroll
                        for (int c = 0; c < CG; ++c)
                            dmma_8x8x4(acc[t][c][0], acc[t][c][1], av, bb[kb & 1][u][c]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < RT; ++t) {                 // group done: r = s * acc (+ prior)
                const int r = t * 8 + fr;
#pragma unroll
                for (int c = 0; c < CG; ++c) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = (g * CG + c) * 8 + 2 * fk + h;
                        if (j < NK && r >= rlo && r < nrows) {
                            double x = __dmul_rn(a.s, acc[t][c][h]);
                            if (a.prior) x = __dadd_rn(x, a.prior[bh * a.NK + j]);   // Eq. 8
                            sc[r * NKP + j] = x;
                        }
                        acc[t][c][h] = 0.0;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (warp < rlo || warp >= nrows) return;

    // ---- phase B: sigma_i (R3) ---------------------------------------------------------
    // mu_i and the centred sum of squares as fixed-order warp reductions (lane-strided
    // partial sums in ascending j, then a butterfly; every lane ends with the same value).
    // The oracle sums sequentially in j; the two differ by a few ulps of sigma_i, which
    // moves r~ by ~1e-16 relative: routing can differ only where two oracle scores tie
    // within that, far inside the documented-tie margin of SURVEY.md 8(c) (R3').
    double* row = sc + warp * NKP;
    const bool biased = a.beta != 0.0;
    const uint32_t gh = (uint32_t)((bh / a.H) * a.H_total + a.head_offset + (bh % a.H));
    const uint32_t i = (uint32_t)(i0 + warp);
    double bi = 0.0;
    if (biased) {
        double sum = 0.0;
        for (int j = lane; j < NK; j += 32) sum = __dadd_rn(sum, row[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
        const double mu = __ddiv_rn(sum, (double)NK);
        double v = 0.0;
        for (int j = lane; j < NK; j += 32) {
            const double dl = __dsub_rn(row[j], mu);
            v = __fma_rn(dl, dl, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        bi = __dmul_rn(a.beta, __dsqrt_rn(__ddiv_rn(v, (double)NK)));
    }

    // ---- phase C: keys in place, threshold, outputs -------------------------------------
    uint64_t* key = reinterpret_cast<uint64_t*>(row);
    const int64_t grow = bh * a.NQ + i0 + warp;
    // lane handles the four consecutive blocks j = 4 (32 m4 + lane) + w, w = 0..3 (one Philox
    // call each group of four)
    auto keys4 = [&](int j4, uint64_t (&kx)[4]) {
        uint4 x = make_uint4(0u, 0u, 0u, 0u);
        if (biased) x = philox4x32_10((uint32_t)j4, i, gh, a.step, a.key0, a.key1);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int j = 4 * j4 + w;
            kx[w] = 0ull;
            if (j < NK) {
                double xv = row[j];
                if (biased)   // R5: rt = r + (beta sigma_i) g, two rounded operations
                    xv = __dadd_rn(xv, __dmul_rn(bi, gumbel_of(xw[w], ltab)));
                kx[w] = orderable(xv);
            }
        }
    };
    if constexpr (HR > 0) {
        uint32_t hr[HR];
        uint64_t kx[4];
#pragma unroll
        for (int m4 = 0; m4 < HR / 4; ++m4) {
            const int j4 = 32 * m4 + lane;
#pragma unroll
            for (int w = 0; w < 4; ++w) hr[4 * m4 + w] = 0u;
            if (4 * j4 < NK) {
                keys4(j4, kx);
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    if (4 * j4 + w < NK) {
                        key[4 * j4 + w] = kx[w];
                        hr[4 * m4 + w] = (uint32_t)(kx[w] >> 32);
                    }
                }
            }
        }
        __syncwarp();
        select_row_mem<HR>(key, NK, k, lane, cbuf + warp * 64, a.idx + grow * NK,
                           a.mask + grow * a.W, a.count + grow, hr);
    } else {
        for (int j4 = lane; 4 * j4 < NK; j4 += 32) {
            uint64_t kx[4];
            keys4(j4, kx);
#pragma unroll
            for (int w = 0; w < 4; ++w)
                if (4 * j4 + w < NK) key[4 * j4 + w] = kx[w];
        }
        __syncwarp();
        const uint32_t none[1] = {0u};
        select_row_mem<0>(key, NK, k, lane, cbuf + warp * 64, a.idx + grow * NK,
                          a.mask + grow * a.W, a.count + grow, none);
    }
}

template <int R, int D, bool SMEM_SC, int HR>
__global__ void __launch_bounds__(32 * R, 16 / R) route_fused_kernel(FusedArgs a) {
    extern __shared__ __align__(16) unsigned char f_smem[];
    route_tile<R, D, SMEM_SC, HR>(a, blockIdx.y, blockIdx.x, f_smem);
}

constexpr size_t fused_fixed_smem(int R, int D) {
    return sizeof(double) * (size_t)R * (D + 4) + sizeof(uint64_t) * R * 64 +
           sizeof(LogEnt) * 128;
}

}  // namespace

static cudaError_t launch_route_fused(const pasa_budget_s* b, uint64_t seed, int32_t step,
                                      pasa_route_s* r, const double* prior, cudaStream_t st,
                                      int* launches);

cudaError_t launch_route(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor* v,
                         const pasa_budget_s* b, uint64_t seed, int32_t step, pasa_route_s* r,
                         cudaStream_t st, int* launches) {
    // Q only for this handle's (head, q-block) items [it0, it1); K for every block (all scored)
    const bool f8 = r->cfg.qk_fp8 != 0;
    PoolArgs qa{q.data, q.sB, q.sS, q.sH, r->S, r->H, r->D, r->cfg.Bq, r->NQ, r->it0,
                0, r->qbar, nullptr, f8 ? r->q8 : nullptr, r->sq8, nullptr, nullptr};
    PoolArgs ka{k.data, k.sB, k.sS, k.sH, r->S, r->H, r->D, r->cfg.Bk, r->NK, 0, r->NK, r->kbar,
                r->kfrag, nullptr, nullptr, r->kamax, r->kbamax};
    if (f8) {   // FP8 QK^T variant: the per-head maxima accumulate from 0
        cudaError_t e = cudaMemsetAsync(r->kamax, 0, sizeof(uint32_t) * 2 * r->BH, st);
        if (e != cudaSuccess) return e;
    }
    int64_t ng = r->D / 8;
    int64_t q_tasks = (r->it1 - r->it0) * ng;
    int64_t total = q_tasks + r->BH * r->NK * ng;
    const unsigned pgrid = (unsigned)((total + 255) / 256);
    if (q.dtype == PASA_F32)
        pool_kernel<float, false><<<pgrid, 256, 0, st>>>(qa, ka, q_tasks, total);
    else if (f8)
        pool_kernel<__nv_bfloat16, true><<<pgrid, 256, 0, st>>>(qa, ka, q_tasks, total);
    else
        pool_kernel<__nv_bfloat16, false><<<pgrid, 256, 0, st>>>(qa, ka, q_tasks, total);
    const double* prior = nullptr;
    if (v) {
        cudaError_t e = launch_het(k, *v, r, st, launches);
        if (e != cudaSuccess) return e;
        prior = r->prior;
    }
    *launches += 1;
    return launch_route_fused(b, seed, step, r, prior, st, launches);
}

// a3 + a4 + a5: the fused score / sigma / top-k kernel over the pooled means in the workspace
static cudaError_t launch_route_fused(const pasa_budget_s* b, uint64_t seed, int32_t step,
                                      pasa_route_s* r, const double* prior, cudaStream_t st,
                                      int* launches) {
    const double s = 1.0 / sqrt((double)r->D);
    FusedArgs fa;
    fa.qbar = r->qbar; fa.kfrag = r->kfrag; fa.prior = prior; fa.rec = b->rec;
    fa.NQ = r->NQ; fa.NK = r->NK; fa.W = r->W; fa.H = r->H;
    fa.it0 = r->it0; fa.it1 = r->it1;
    fa.H_total = r->cfg.H_total; fa.head_offset = r->cfg.head_offset;
    fa.D = (int)r->D; fa.NKP = (int)route_score_stride(r->NK);
    fa.s = s; fa.beta = r->cfg.beta;
    fa.key0 = (uint32_t)(seed & 0xffffffffu); fa.key1 = (uint32_t)(seed >> 32);
    fa.step = (uint32_t)step;
    fa.idx = r->idx; fa.count = r->count; fa.mask = r->mask; fa.hdr = r->hdr;
    fa.gsc = r->scores;
    const bool smem_sc = route_rows_per_cta(r->NK, r->D) > 0;
    constexpr int RR = kFRows;
    const size_t smem = fused_fixed_smem(RR, (int)r->D) +
                        (smem_sc ? sizeof(double) * (size_t)RR * fa.NKP : 0);
    dim3 grid((unsigned)((r->NQ + RR - 1) / RR), (unsigned)r->BH);   // CTAs out of range exit
    const bool hreg = r->NK <= 32 * kFHR;
#define PASA_FUSED_PICK(DD)                                                                  \
    (!smem_sc ? route_fused_kernel<RR, DD, false, 0>                                         \
              : (hreg ? route_fused_kernel<RR, DD, true, kFHR> : route_fused_kernel<RR, DD, true, 0>))
    void (*kfn)(FusedArgs) = r->D == 128 ? PASA_FUSED_PICK(128) : PASA_FUSED_PICK(64);
#undef PASA_FUSED_PICK
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e == cudaSuccess) {
        kfn<<<grid, 32 * RR, smem, st>>>(fa);
        e = cudaGetLastError();
    }
    *launches += 1;
    return e;
}

cudaError_t launch_route_zc(const ZcShards* qkv, const pasa_tensor* loc, const pasa_budget_s* b,
                            uint64_t seed, int32_t step, pasa_route_s* r, cudaStream_t st,
                            int* launches) {
    ZcArgs a;
    for (int x = 0; x < 3; ++x) {
        a.src[x] = qkv[x];
        a.loc[x] = reinterpret_cast<__nv_bfloat16*>(loc[x].data);
        a.lsS[x] = loc[x].sS;
        a.lsH[x] = loc[x].sH;
    }
    a.S = r->S; a.Hl = r->H; a.D = r->D; a.head0 = r->cfg.head_offset;
    a.bsz[0] = r->cfg.Bq; a.bsz[1] = a.bsz[2] = r->cfg.Bk;
    a.nblk[0] = r->NQ; a.nblk[1] = a.nblk[2] = r->NK;
    a.it0 = r->it0; a.it1 = r->it1;
    a.out[0] = r->qbar; a.out[1] = r->kbar; a.kfrag = r->kfrag;
    const int64_t ng = r->D / 8;
    int64_t total = 0;
    for (int x = 0; x < 3; ++x) total += (a.ntask[x] = r->H * a.nblk[x] * ng);
    const unsigned grid = (unsigned)((total + 255) / 256);
    zc_gather_pool_kernel<<<grid, 256, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    *launches += 1;
    if (e != cudaSuccess) return e;
    return launch_route_fused(b, seed, step, r, nullptr, st, launches);
}

// A/B knob: score rows in shared memory at one CTA per SM when two do not fit (measured
// at HunyuanVideo, N_K = 1,857: 1.638 ms vs 1.607 ms for two CTAs per SM with the rows in
// the L2-resident workspace scratch -- off)
#ifndef PASA_ROUTE_SMEM1
#define PASA_ROUTE_SMEM1 0
#endif

int route_rows_per_cta(int64_t NK, int64_t D) {
    // 8 rows (one DMMA row tile) per CTA, two CTAs per SM: 113 KB of shared memory each
    // (16 rows at one CTA per SM measured the same at Wan-14B: 1.142 vs 1.137 ms)
    const size_t nkp = (size_t)route_score_stride(NK);
    const size_t need = fused_fixed_smem(kFRows, (int)D) + sizeof(double) * kFRows * nkp;
    const size_t cap = PASA_ROUTE_SMEM1 ? 227 * 1024 : 113 * 1024;
    return need <= cap ? kFRows : 0;
}

int64_t route_score_stride(int64_t NK) { return NK | 1; }





}  // namespace pasa
