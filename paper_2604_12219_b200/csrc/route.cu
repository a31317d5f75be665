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

#include "pasa_internal.h"
#include "philox.cuh"

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
    double* out;    // [BH][nblk][D]
};

template <typename T>
__global__ void __launch_bounds__(256) pool_kernel(PoolArgs qa, PoolArgs ka, int64_t q_tasks,
                                                   int64_t total) {
    int64_t task = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (task >= total) return;
    const PoolArgs& a = task < q_tasks ? qa : ka;
    if (task >= q_tasks) task -= q_tasks;
    int64_t ng = a.D / 8;
    int64_t dg = task % ng;
    int64_t rest = task / ng;
    int64_t blk = rest % a.nblk;
    int64_t bh = rest / a.nblk;
    int64_t b = bh / a.H, h = bh % a.H;
    int64_t t0 = blk * a.bsz;
    int64_t t1 = min(t0 + (int64_t)a.bsz, a.S);
    const T* base = reinterpret_cast<const T*>(a.x) + b * a.sB + h * a.sH + dg * 8;
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    int64_t t = t0;
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
    }
    for (; t < t1; ++t) {
        double v0[8];
        load8<T>(base + t * a.sS, v0);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __dadd_rn(acc[i], v0[i]);
    }
    double n = (double)(t1 - t0);
    double* o = a.out + (bh * a.nblk + blk) * a.D + dg * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = __ddiv_rn(acc[i], n);
}

// ---------------------------------------------------------------------------
// a3: block scores r_ij = s * dot(Qbar_i, Kbar_j), a tiled fp64 GEMM on the fp64
// tensor core.  Every output accumulates an fma chain over the head dimension in
// ascending order (R2: the chain of DMMA 8x8x4 steps is that chain, bit for bit), so
// the per-element result is independent of the tiling.
// ---------------------------------------------------------------------------
constexpr int kST = 128;    // tile edge (rows i x columns j)
constexpr int kSK = 16;     // D chunk staged in smem
constexpr int kSP = kSK + 4;   // padded smem row (doubles): conflict-free DMMA fragments

constexpr int kSThreads = 256;   // 8 warps; warp w owns row tiles 2w, 2w+1 x 16 column tiles

// fp64 tensor core: d (+)= a * b on an 8x8x4 tile.  Measured on this pool
// (tools/dmma_exact.cu): bit-identical to the sequential fma chain over k = 0..3, so
// a chain of these in ascending k is the oracle's ascending-d fma chain (R2).
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kSThreads, 1) scores_kernel(const double* __restrict__ qbar,
                                                        const double* __restrict__ kbar, int64_t NQ,
                                                        int64_t NK, int64_t D, double s,
                                                        const double* __restrict__ prior,
                                                        double* __restrict__ r) {
    __shared__ double sq[kST][kSP];    // rows i of Qbar, one 16-dim chunk
    __shared__ double sk[kST][kSP];    // rows j of Kbar
    const int64_t bh = blockIdx.z;
    const int64_t i0 = (int64_t)blockIdx.y * kST, j0 = (int64_t)blockIdx.x * kST;
    const double* Q = qbar + bh * NQ * D;
    const double* K = kbar + bh * NK * D;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fk = lane & 3;     // DMMA fragment row / k index
    double acc[2][16][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    // register double buffer: chunk d0 + kSK is in flight while chunk d0 is consumed
    constexpr int kPer = kSK * kST / kSThreads;
    double pq[kPer], pk[kPer];
    auto fetch = [&](int64_t d0) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = tid + kSThreads * u;
            const int row = e / kSK, col = e % kSK;
            const int64_t gi = i0 + row, gj = j0 + row;
            pq[u] = gi < NQ ? Q[gi * D + d0 + col] : 0.0;
            pk[u] = gj < NK ? K[gj * D + d0 + col] : 0.0;
        }
    };
    fetch(0);
    for (int64_t d0 = 0; d0 < D; d0 += kSK) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = tid + kSThreads * u;
            sq[e / kSK][e % kSK] = pq[u];
            sk[e / kSK][e % kSK] = pk[u];
        }
        __syncthreads();
        if (d0 + kSK < D) fetch(d0 + kSK);
#pragma unroll
        for (int ks = 0; ks < kSK / 4; ++ks) {      // ascending d: r_ij's fma chain order
            const int kk = 4 * ks + fk;
            const double a0 = sq[(2 * warp) * 8 + fr][kk];
            const double a1 = sq[(2 * warp + 1) * 8 + fr][kk];
            double bv[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) bv[c] = sk[c * 8 + fr][kk];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                dmma_8x8x4(acc[0][c][0], acc[0][c][1], a0, bv[c]);
                dmma_8x8x4(acc[1][c][0], acc[1][c][1], a1, bv[c]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const int64_t gi = i0 + (2 * warp + a) * 8 + fr;
        if (gi >= NQ) continue;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gj = j0 + c * 8 + 2 * fk + h;
                if (gj < NK) {
                    double x = __dmul_rn(s, acc[a][c][h]);
                    if (prior) x = __dadd_rn(x, prior[bh * NK + gj]);   // Eq. 8 prior term
                    r[(bh * NQ + gi) * NK + gj] = x;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// a4 (row statistics): sigma_i, the population std of score row i (R3).  The
// sums run sequentially in ascending j exactly as in the oracle (bit-exact), one
// thread per row; 128 rows per CTA are staged through shared memory in column
// chunks so the loads are coalesced and 128 sequential chains run concurrently.
// ---------------------------------------------------------------------------
constexpr int kRsRows = 64, kRsCols = 32;

__global__ void __launch_bounds__(kRsRows * 2) rowstats_kernel(const double* __restrict__ r,
                                                               int64_t rows, int64_t NK,
                                                               double* __restrict__ sigma) {
    // 128 threads stage a [64 rows x 64 cols] chunk (register prefetch of the next
    // chunk overlaps the sequential sums of the current one); threads 0..63 own a row.
    __shared__ double tile[2][kRsRows][kRsCols + 1];
    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * kRsRows;
    const int nrows = (int)min((int64_t)kRsRows, rows - r0);
    const int nchunk = (int)((NK + kRsCols - 1) / kRsCols);
    constexpr int kPer = kRsRows * kRsCols / (kRsRows * 2);   // 32 loads per thread per chunk
    double buf[kPer];
    auto fetch = [&](int c) {
        const int64_t c0 = (int64_t)c * kRsCols;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = tid + u * (kRsRows * 2);
            const int rr = e / kRsCols, cc = e % kRsCols;
            buf[u] = (rr < nrows && c0 + cc < NK) ? __ldg(r + (r0 + rr) * NK + c0 + cc) : 0.0;
        }
    };
    auto stash = [&](int slot) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = tid + u * (kRsRows * 2);
            tile[slot][e / kRsCols][e % kRsCols] = buf[u];
        }
    };
    double sum = 0.0, mu = 0.0, acc = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
        fetch(0);
        for (int c = 0; c < nchunk; ++c) {
            const int slot = c & 1;
            stash(slot);
            __syncthreads();
            if (c + 1 < nchunk) fetch(c + 1);
            const int nc = (int)min((int64_t)kRsCols, NK - (int64_t)c * kRsCols);
            if (tid < nrows) {
                if (pass == 0) {
                    for (int cc = 0; cc < nc; ++cc) sum = __dadd_rn(sum, tile[slot][tid][cc]);
                } else {
                    for (int cc = 0; cc < nc; ++cc) {
                        const double dl = __dsub_rn(tile[slot][tid][cc], mu);
                        acc = __fma_rn(dl, dl, acc);
                    }
                }
            }
        }
        __syncthreads();
        if (pass == 0) mu = __ddiv_rn(sum, (double)NK);
    }
    if (tid < nrows) sigma[r0 + tid] = __dsqrt_rn(__ddiv_rn(acc, (double)NK));
}

// ---------------------------------------------------------------------------
// a4 + a5: one warp per (head, query block) row.  Element j = 32 m + lane lives in
// register m of lane `lane`.  Gumbel bias, then the k-th largest orderable key T is
// found bit by bit (T = the largest value with #{key >= T} >= k), ties at T go to
// the smallest j (R-13), and the ballot of each 32-block chunk is directly the
// route's mask word; the ascending index list follows from ballot prefix counts.
// ---------------------------------------------------------------------------
constexpr int kSelWarps = 4;
// 5 CTAs (20 warps) per SM for M <= 40: a few spilled registers cost less than the
// lost occupancy (route at Wan-14B 1.52 -> 1.34 ms with the window search below)

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

struct SelArgs {
    const double* r;          // [BH][NQ][NK]
    const double* sigma;      // [BH][NQ]
    const BudgetRec* rec;
    int64_t rows, NQ, NK, W, H, H_total, head_offset;
    double beta;
    uint32_t key0, key1;      // Philox key = (lo32 seed, hi32 seed)
    uint32_t step;
    int32_t* idx;             // [BH][NQ][NK]
    int32_t* count;           // [BH][NQ]
    uint32_t* mask;           // [BH][NQ][W]
    int32_t* hdr;
};

template <int MAXM>
// occupancy over registers: a few spilled keys cost less than idle warps (route at
// Wan-14B 1.52 -> 1.34 ms with 5 CTAs/SM for MAXM <= 40; HunyuanVideo's MAXM = 64
// 2.70 -> 2.03 ms with 4 instead of 2 CTAs/SM, 3, 5 and 6 measured slower)
__global__ void __launch_bounds__(32 * kSelWarps, MAXM <= 40 ? 5 : 4) select_kernel(SelArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kSelWarps + (threadIdx.x >> 5);   // bh * NQ + i
    if (row >= a.rows) return;
    const int64_t bh = row / a.NQ, i = row % a.NQ;
    const int NK = (int)a.NK;
    const int M = (NK + 31) >> 5;
    const int k = device_k(a.rec, NK);
    if (row == 0 && lane == 0) a.hdr[0] = k;
    int32_t* orow = a.idx + row * NK;
    uint32_t* mrow = a.mask + row * a.W;
    if (k >= NK) {  // dense step / full budget: every block exact
        for (int j = lane; j < NK; j += 32) orow[j] = j;
        for (int w = lane; w < M; w += 32) {
            const int rem = NK - 32 * w;
            mrow[w] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
        }
        if (lane == 0) a.count[row] = NK;
        return;
    }
    const double* rr = a.r + row * NK;
    uint64_t key[MAXM];
    const bool biased = a.beta != 0.0;
    const double bi = biased ? __dmul_rn(a.beta, a.sigma[row]) : 0.0;
    const uint32_t gh = (uint32_t)((bh / a.H) * a.H_total + a.head_offset + (bh % a.H));
    uint64_t kand = ~0ull, kor = 0ull;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
        const int j = 32 * m + lane;
        key[m] = 0ull;                       // absent elements sort last (below every key)
        if (m < M && j < NK) {
            double x = __ldg(rr + j);
            if (biased) {   // R4/R5: rt = r + (beta * sigma_i) * g, two rounded operations
                const uint32_t x0 = philox4x32_10_x0((uint32_t)j, (uint32_t)i, gh, a.step, a.key0,
                                                     a.key1);
                const double u = __dmul_rn(__dadd_rn((double)x0, 0.5), 2.3283064365386963e-10);
                x = __dadd_rn(x, __dmul_rn(bi, -log(-log(u))));
            }
            key[m] = orderable(x);
            kand &= key[m];
            kor |= key[m];
        }
    }
    // bits above the highest differing bit are common to every present key
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kand &= __shfl_xor_sync(0xffffffffu, kand, o);
        kor |= __shfl_xor_sync(0xffffffffu, kor, o);
    }
    const uint64_t diff = kand ^ kor;
    uint64_t T = diff ? (kand & ~((2ull << (63 - __clzll(diff))) - 1ull)) : kand;
    const int top = diff ? 63 - __clzll(diff) : -1;
    // T = the largest value with #{key >= T} >= k, bit by bit from the top differing
    // bit.  Upper half first with 32-bit compares (key >= T_hi:0 <=> hi >= T_hi), then
    // the lower half among the keys whose upper half equals T_hi (the others are
    // counted once: hi > T_hi always, hi < T_hi never).
    //
    // Shortcut (top >= 48): once the top 16 bits of T are fixed, the keys sharing them are
    // usually few (a 1/16-binade window around the k-th score).  If there are at most
    // 64, they are compacted into shared memory (two per lane) and the remaining bits
    // are searched over those two registers instead of all M; the keys above the
    // window are counted once.  Same T as the full search.
    __shared__ uint64_t cbuf[kSelWarps][64];
    uint32_t T_hi = (uint32_t)(T >> 32);
    int bpos = top;
    for (; bpos >= 48; --bpos) {
        const uint32_t cand = T_hi | (1u << (bpos - 32));
        int c = 0;
#pragma unroll
        for (int m = 0; m < MAXM; ++m) c += (uint32_t)(key[m] >> 32) >= cand;
        c = __reduce_add_sync(0xffffffffu, c);
        if (c >= k) T_hi = cand;
    }
    if (top >= 48) {
        // window = keys whose top 16 bits equal T's (32-bit compares on the upper half)
        const uint32_t tw = T_hi >> 16;
        int gw = 0, ew = 0;
#pragma unroll
        for (int m = 0; m < MAXM; ++m) {
            const uint32_t h16 = (uint32_t)(key[m] >> 48);
            gw += h16 > tw;
            ew += h16 == tw;   // an absent key (0) can only match if tw = 0; it never counts below
        }
        gw = __reduce_add_sync(0xffffffffu, gw);
        ew = __reduce_add_sync(0xffffffffu, ew);
        if (ew <= 64) {
            uint64_t* cb = cbuf[threadIdx.x >> 5];
            const uint32_t lt = (1u << lane) - 1u;
            int base = 0;
#pragma unroll
            for (int m = 0; m < MAXM; ++m) {
                const bool in = (uint32_t)(key[m] >> 48) == tw;
                const uint32_t b = __ballot_sync(0xffffffffu, in);
                if (in) cb[base + __popc(b & lt)] = key[m];
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
            T_hi = (uint32_t)(Tc >> 32);
            T = Tc;
            bpos = -2;   // done
        }
    }
    for (; bpos >= 32; --bpos) {
        const uint32_t cand = T_hi | (1u << (bpos - 32));
        int c = 0;
#pragma unroll
        for (int m = 0; m < MAXM; ++m) c += (uint32_t)(key[m] >> 32) >= cand;
        c = __reduce_add_sync(0xffffffffu, c);
        if (c >= k) T_hi = cand;
    }
    uint32_t T_lo = top >= 32 ? 0u : (uint32_t)T;
    if (bpos == -2) {
        T_lo = (uint32_t)T;
    } else if (top >= 0) {
        int gtc = 0;
        uint32_t lo[MAXM];
#pragma unroll
        for (int m = 0; m < MAXM; ++m) {
            const uint32_t hi = (uint32_t)(key[m] >> 32);
            gtc += hi > T_hi;
            lo[m] = hi == T_hi ? (uint32_t)key[m] : 0u;   // 0 never reaches a candidate
        }
        gtc = __reduce_add_sync(0xffffffffu, gtc);
        for (int bpos = min(top, 31); bpos >= 0; --bpos) {
            const uint32_t cand = T_lo | (1u << bpos);
            int c = 0;
#pragma unroll
            for (int m = 0; m < MAXM; ++m) c += lo[m] >= cand;
            c = gtc + __reduce_add_sync(0xffffffffu, c);
            if (c >= k) T_lo = cand;
        }
    }
    T = ((uint64_t)T_hi << 32) | T_lo;
    int gt = 0;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) gt += key[m] > T;
    const int need = k - __reduce_add_sync(0xffffffffu, gt);   // keys equal to T to take
    // walk the chunks in ascending j: ties go to the smallest j; the ballot of a chunk
    // is its mask word; positions come from prefix counts
    int taken_eq = 0, pos = 0;
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
        if (m < M) {
            const uint32_t eqb = __ballot_sync(0xffffffffu, key[m] == T);
            const int eq_rank = taken_eq + __popc(eqb & below);
            const bool take = key[m] > T || (key[m] == T && eq_rank < need);
            taken_eq += __popc(eqb);
            const uint32_t sel = __ballot_sync(0xffffffffu, take);
            if (take) orow[pos + __popc(sel & below)] = 32 * m + lane;
            pos += __popc(sel);
            if (lane == 0) mrow[m] = sel;
        }
    }
    if (lane == 0) a.count[row] = k;
}

}  // namespace

cudaError_t launch_route(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor* v,
                         const pasa_budget_s* b, uint64_t seed, int32_t step, pasa_route_s* r,
                         cudaStream_t st, int* launches) {
    PoolArgs qa{q.data, q.sB, q.sS, q.sH, r->S, r->H, r->D, r->cfg.Bq, r->NQ, r->qbar};
    PoolArgs ka{k.data, k.sB, k.sS, k.sH, r->S, r->H, r->D, r->cfg.Bk, r->NK, r->kbar};
    int64_t ng = r->D / 8;
    int64_t q_tasks = r->BH * r->NQ * ng;
    int64_t total = q_tasks + r->BH * r->NK * ng;
    int64_t grid = (total + 255) / 256;
    if (q.dtype == PASA_F32)
        pool_kernel<float><<<(unsigned)grid, 256, 0, st>>>(qa, ka, q_tasks, total);
    else
        pool_kernel<__nv_bfloat16><<<(unsigned)grid, 256, 0, st>>>(qa, ka, q_tasks, total);

    const double* prior = nullptr;
    if (v) {
        cudaError_t e = launch_het(k, *v, r, st, launches);
        if (e != cudaSuccess) return e;
        prior = r->prior;
    }
    const double s = 1.0 / sqrt((double)r->D);
    dim3 sg((unsigned)((r->NK + kST - 1) / kST), (unsigned)((r->NQ + kST - 1) / kST),
            (unsigned)r->BH);
    scores_kernel<<<sg, kSThreads, 0, st>>>(r->qbar, r->kbar, r->NQ, r->NK, r->D, s, prior, r->scores);
    *launches += 2;

    const int64_t rows = r->BH * r->NQ;
    if (r->cfg.beta != 0.0) {
        rowstats_kernel<<<(unsigned)((rows + kRsRows - 1) / kRsRows), kRsRows * 2, 0, st>>>(
            r->scores, rows, r->NK, r->sigma);
        *launches += 1;
    }
    SelArgs sa;
    sa.r = r->scores;
    sa.sigma = r->sigma;
    sa.rec = b->rec;
    sa.rows = rows;
    sa.NQ = r->NQ; sa.NK = r->NK; sa.W = r->W; sa.H = r->H;
    sa.H_total = r->cfg.H_total; sa.head_offset = r->cfg.head_offset;
    sa.beta = r->cfg.beta;
    sa.key0 = (uint32_t)(seed & 0xffffffffu);
    sa.key1 = (uint32_t)(seed >> 32);
    sa.step = (uint32_t)step;
    sa.idx = r->idx; sa.count = r->count; sa.mask = r->mask; sa.hdr = r->hdr;
    const unsigned sg2 = (unsigned)((rows + kSelWarps - 1) / kSelWarps);
    const int M = (int)((r->NK + 31) / 32);
    if (M <= 8) select_kernel<8><<<sg2, 32 * kSelWarps, 0, st>>>(sa);
    else if (M <= 20) select_kernel<20><<<sg2, 32 * kSelWarps, 0, st>>>(sa);
    else if (M <= 40) select_kernel<40><<<sg2, 32 * kSelWarps, 0, st>>>(sa);
    else select_kernel<64><<<sg2, 32 * kSelWarps, 0, st>>>(sa);
    *launches += 1;
    return cudaGetLastError();
}

int route_max_nk() { return 2048; }

}  // namespace pasa
