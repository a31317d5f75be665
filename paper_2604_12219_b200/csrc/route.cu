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
// a3: block scores r_ij = s * dot(Qbar_i, Kbar_j), a tiled fp64 GEMM.  Each
// thread owns a 4x4 output patch and accumulates every output with an fma
// chain over the head dimension in ascending order (R2), so the per-element
// result is independent of the tiling.
// ---------------------------------------------------------------------------
constexpr int kST = 64;     // tile edge
constexpr int kSK = 16;     // D chunk staged in smem

__global__ void __launch_bounds__(256) scores_kernel(const double* __restrict__ qbar,
                                                     const double* __restrict__ kbar, int64_t NQ,
                                                     int64_t NK, int64_t D, double s,
                                                     double* __restrict__ r) {
    __shared__ double sq[kSK][kST + 1];
    __shared__ double sk[kSK][kST + 1];
    int64_t bh = blockIdx.z;
    int64_t i0 = (int64_t)blockIdx.y * kST, j0 = (int64_t)blockIdx.x * kST;
    const double* Q = qbar + bh * NQ * D;
    const double* K = kbar + bh * NK * D;
    int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
    for (int64_t d0 = 0; d0 < D; d0 += kSK) {
        for (int e = threadIdx.x; e < kSK * kST; e += 256) {
            int row = e / kSK, col = e % kSK;
            int64_t gi = i0 + row, gj = j0 + row;
            sq[col][row] = gi < NQ ? Q[gi * D + d0 + col] : 0.0;
            sk[col][row] = gj < NK ? K[gj * D + d0 + col] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int dd = 0; dd < kSK; ++dd) {
            double qv[4], kv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) qv[a] = sq[dd][ty + 16 * a];
#pragma unroll
            for (int c = 0; c < 4; ++c) kv[c] = sk[dd][tx + 16 * c];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][c] = __fma_rn(qv[a], kv[c], acc[a][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        int64_t gi = i0 + ty + 16 * a;
        if (gi >= NQ) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int64_t gj = j0 + tx + 16 * c;
            if (gj < NK) r[(bh * NQ + gi) * NK + gj] = __dmul_rn(s, acc[a][c]);
        }
    }
}

// ---------------------------------------------------------------------------
// a4 + a5: per (head, query block) row: sigma_i, Gumbel bias, top-k by
// (score desc, j asc) via an 8-pass MSB radix select on orderable 64-bit keys,
// then an ascending compaction into idx / count / mask.
// ---------------------------------------------------------------------------
constexpr int kSelThreads = 256;
constexpr int kMaxNK = 2048;   // smem capacity of the select kernel (S <= 131,072 at Bk = 64)

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
    const BudgetRec* rec;
    int64_t NQ, NK, W, H, H_total, head_offset;
    double beta;
    uint32_t key0, key1;      // Philox key = (lo32 seed, hi32 seed)
    uint32_t step;
    int32_t* idx;             // [BH][NQ][NK]
    int32_t* count;           // [BH][NQ]
    uint32_t* mask;           // [BH][NQ][W]
    int32_t* hdr;
};

__global__ void __launch_bounds__(kSelThreads) select_kernel(SelArgs a) {
    __shared__ uint64_t keys[kMaxNK];
    __shared__ double sr[kMaxNK];
    __shared__ uint32_t hist[256];
    __shared__ uint8_t flag[kMaxNK];
    __shared__ double s_sigma;
    __shared__ uint64_t s_prefix;
    __shared__ int s_remaining;
    __shared__ int warp_tot[kSelThreads / 32][2];

    const int64_t row = blockIdx.x;            // bh * NQ + i
    const int64_t bh = row / a.NQ, i = row % a.NQ;
    const int64_t NK = a.NK;
    const int tid = threadIdx.x;
    const int k = device_k(a.rec, NK);
    if (row == 0 && tid == 0) a.hdr[0] = k;

    int32_t* orow = a.idx + row * NK;
    uint32_t* mrow = a.mask + row * a.W;
    if (k >= NK) {  // dense step / full budget: every block exact
        for (int64_t j = tid; j < NK; j += kSelThreads) orow[j] = (int32_t)j;
        for (int64_t w = tid; w < a.W; w += kSelThreads) {
            int64_t rem = NK - 32 * w;
            mrow[w] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
        }
        if (tid == 0) a.count[row] = (int32_t)NK;
        return;
    }

    const double* rr = a.r + row * NK;
    for (int64_t j = tid; j < NK; j += kSelThreads) sr[j] = rr[j];
    __syncthreads();

    if (a.beta != 0.0) {
        // R3: sequential mean and fma-chain variance (one thread; exact order)
        if (tid == 0) {
            double sum = 0.0;
            for (int64_t j = 0; j < NK; ++j) sum = __dadd_rn(sum, sr[j]);
            double mu = __ddiv_rn(sum, (double)NK);
            double acc = 0.0;
            for (int64_t j = 0; j < NK; ++j) {
                double dl = __dsub_rn(sr[j], mu);
                acc = __fma_rn(dl, dl, acc);
            }
            s_sigma = __dsqrt_rn(__ddiv_rn(acc, (double)NK));
        }
        // meanwhile: the Gumbel draws (R-11/R-12), kept in keys[] as doubles
        const uint32_t gh = (uint32_t)((bh / a.H) * a.H_total + a.head_offset + (bh % a.H));
        for (int64_t j = tid; j < NK; j += kSelThreads) {
            uint32_t x0 = philox4x32_10_x0((uint32_t)j, (uint32_t)i, gh, a.step, a.key0, a.key1);
            double u = __dmul_rn(__dadd_rn((double)x0, 0.5), 2.3283064365386963e-10);
            double g = -log(-log(u));
            keys[j] = (uint64_t)__double_as_longlong(g);
        }
        __syncthreads();
        const double bi = __dmul_rn(a.beta, s_sigma);
        for (int64_t j = tid; j < NK; j += kSelThreads) {
            double g = __longlong_as_double((long long)keys[j]);
            keys[j] = orderable(__dadd_rn(sr[j], __dmul_rn(bi, g)));   // R5
        }
    } else {
        for (int64_t j = tid; j < NK; j += kSelThreads) keys[j] = orderable(sr[j]);
    }
    if (tid == 0) { s_prefix = 0; s_remaining = k; }
    __syncthreads();

    // radix select of the k-th largest key
    uint64_t pmask = 0;
    for (int pass = 7; pass >= 0; --pass) {
        const int shift = pass * 8;
        for (int b = tid; b < 256; b += kSelThreads) hist[b] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (int64_t j = tid; j < NK; j += kSelThreads) {
            uint64_t key = keys[j];
            if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            // lane l owns digits 255-8l ... 248-8l (descending)
            uint32_t loc[8];
            uint32_t sum = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) { loc[u] = hist[255 - 8 * tid - u]; sum += loc[u]; }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += v;
            }
            const uint32_t rem = (uint32_t)s_remaining;
            const uint32_t excl = incl - sum;
            const bool hit = excl < rem && incl >= rem;
            const unsigned ball = __ballot_sync(0xffffffffu, hit);
            const int lane = __ffs(ball) - 1;
            if (tid == lane) {
                uint32_t cum = excl;
                int digit = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (cum + loc[u] >= rem) { digit = 255 - 8 * tid - u; break; }
                    cum += loc[u];
                }
                s_prefix = prefix | ((uint64_t)digit << shift);
                s_remaining = (int)(rem - cum);
            }
        }
        pmask |= (uint64_t)255 << shift;
        __syncthreads();
    }
    const uint64_t T = s_prefix;
    const int need = s_remaining;   // how many keys equal to T are taken (lowest j first)

    // ascending compaction: thread t owns a contiguous run of j
    const int64_t per = (NK + kSelThreads - 1) / kSelThreads;
    const int64_t ja = tid * per, jb = min(ja + per, NK);
    int n_gt = 0, n_eq = 0;
    for (int64_t j = ja; j < jb; ++j) {
        uint64_t key = keys[j];
        n_gt += key > T;
        n_eq += key == T;
    }
    // exclusive block scans of n_eq (tie rank) -- then decide, then scan selected
    int lane = tid & 31, wid = tid >> 5;
    int v = n_eq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += x;
    }
    if (lane == 31) warp_tot[wid][0] = v;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < wid; ++w) base += warp_tot[w][0];
    int eq_rank = base + v - n_eq;
    int n_sel = 0;
    for (int64_t j = ja; j < jb; ++j) {
        uint64_t key = keys[j];
        bool take = key > T || (key == T && eq_rank < need);
        eq_rank += key == T;
        flag[j] = take;
        n_sel += take;
    }
    __syncthreads();
    v = n_sel;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += x;
    }
    if (lane == 31) warp_tot[wid][1] = v;
    __syncthreads();
    base = 0;
    for (int w = 0; w < wid; ++w) base += warp_tot[w][1];
    int pos = base + v - n_sel;
    for (int64_t j = ja; j < jb; ++j)
        if (flag[j]) orow[pos++] = (int32_t)j;
    for (int64_t w = tid; w < a.W; w += kSelThreads) {
        uint32_t word = 0;
        for (int u = 0; u < 32; ++u) {
            int64_t j = 32 * w + u;
            if (j < NK && flag[j]) word |= 1u << u;
        }
        mrow[w] = word;
    }
    if (tid == 0) a.count[row] = k;
}

}  // namespace

cudaError_t launch_route(const pasa_tensor& q, const pasa_tensor& k, const pasa_budget_s* b,
                         uint64_t seed, int32_t step, pasa_route_s* r, cudaStream_t st,
                         int* launches) {
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

    const double s = 1.0 / sqrt((double)r->D);
    dim3 sg((unsigned)((r->NK + kST - 1) / kST), (unsigned)((r->NQ + kST - 1) / kST),
            (unsigned)r->BH);
    scores_kernel<<<sg, 256, 0, st>>>(r->qbar, r->kbar, r->NQ, r->NK, r->D, s, r->scores);

    SelArgs sa;
    sa.r = r->scores;
    sa.rec = b->rec;
    sa.NQ = r->NQ; sa.NK = r->NK; sa.W = r->W; sa.H = r->H;
    sa.H_total = r->cfg.H_total; sa.head_offset = r->cfg.head_offset;
    sa.beta = r->cfg.beta;
    sa.key0 = (uint32_t)(seed & 0xffffffffu);
    sa.key1 = (uint32_t)(seed >> 32);
    sa.step = (uint32_t)step;
    sa.idx = r->idx; sa.count = r->count; sa.mask = r->mask; sa.hdr = r->hdr;
    select_kernel<<<(unsigned)(r->BH * r->NQ), kSelThreads, 0, st>>>(sa);
    *launches += 3;
    return cudaGetLastError();
}

int route_max_nk() { return kMaxNK; }

}  // namespace pasa
