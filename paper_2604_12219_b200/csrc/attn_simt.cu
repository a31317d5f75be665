// attn_simt.cu -- pasa_attn on CUDA cores (fp32 arithmetic).  Used for fp32
// I/O (tolerance 1e-5 * max|O|) and, with PASA_ATTN_FORCE_SIMT, as an
// independent cross-check of the tensor-core kernel.  Not a performance path.
//
// Same algorithm as attn_sm100.cu: exact online softmax over
// the kept blocks of the query block's route, then the dropped blocks'
// centroid logits folded into the same running max / sum (Eq. 7, PAPER.md:
// 218-228, denominator weight n_j per reading R-2), then per group the
// first-order term s * A_{t,g} * q_t Hbar^(g) (App. B).
// Two threads per query row, each owning half of the head dimension.
#include <cuda_bf16.h>

#include "pasa_internal.h"

namespace pasa {
namespace {

constexpr int kBk = 64;
constexpr int kTT = 32;   // tokens staged per pass
constexpr float kLog2e = 1.4426950408889634f;

template <typename T> __device__ __forceinline__ float ld(const T* p);
template <> __device__ __forceinline__ float ld<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}
template <typename T> __device__ __forceinline__ T cvt(float x);
template <> __device__ __forceinline__ float cvt<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

struct SimtArgs {
    const void *q, *k, *v;
    void* out;
    int64_t qsB, qsS, qsH, ksB, ksS, ksH, vsB, vsS, vsH, osB, osS, osH;
    int64_t S, H, NQ, NK, NG, W;
    int64_t it0;          // first (head, q-block) item of the handle's range (grid.x covers it)
    int32_t Bq, G, comp;
    float scale_log2;     // s * log2(e)
    float s;
    const int32_t* idx;   // [BH][NQ][NK]
    const int32_t* count;
    const uint32_t* mask;
    const void* kbar_lp;  // [BH][NK][D] (T)
    const void* vsum_lp;
    const void* ht;       // [BH][NG][D][D] (T)
};

template <typename T, int D>
__global__ void __launch_bounds__(256) attn_simt_kernel(SimtArgs a) {
    constexpr int DH = D / 2;
    __shared__ float Ks[kTT][D];
    __shared__ float Vs[kTT][D];

    const int64_t bh = (a.it0 + blockIdx.x) / a.NQ, i = (a.it0 + blockIdx.x) % a.NQ;
    const int64_t b = bh / a.H, h = bh % a.H;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int r = tid >> 1, half = tid & 1;
    const int64_t t = i * a.Bq + r;
    const bool live = r < a.Bq && t < a.S;
    const T* Q = reinterpret_cast<const T*>(a.q) + b * a.qsB + h * a.qsH;
    const T* K = reinterpret_cast<const T*>(a.k) + b * a.ksB + h * a.ksH;
    const T* V = reinterpret_cast<const T*>(a.v) + b * a.vsB + h * a.vsH;

    float q[DH], o[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) {
        q[d] = live ? ld<T>(Q + t * a.qsS + half * DH + d) : 0.f;
        o[d] = 0.f;
    }
    float m = -INFINITY, l = 0.f;

    const int64_t row = bh * a.NQ + i;
    const int32_t cnt = a.count[row];
    const int32_t* sel = a.idx + row * a.NK;
    // ---- exact part over the kept blocks (online softmax, log2 domain) ----
    for (int p = 0; p < cnt; ++p) {
        const int64_t j = sel[p];
        const int64_t u0 = j * kBk;
        const int nj = (int)min((int64_t)kBk, a.S - u0);
        for (int tt = 0; tt < nj; tt += kTT) {
            __syncthreads();
            for (int e = tid; e < kTT * D; e += nthr) {
                const int uu = e / D, d = e % D;
                const bool ok = tt + uu < nj;
                Ks[uu][d] = ok ? ld<T>(K + (u0 + tt + uu) * a.ksS + d) : 0.f;
                Vs[uu][d] = ok ? ld<T>(V + (u0 + tt + uu) * a.vsS + d) : 0.f;
            }
            __syncthreads();
            const int nu = min(kTT, nj - tt);
            for (int uu = 0; uu < nu; ++uu) {
                float part = 0.f;
#pragma unroll
                for (int d = 0; d < DH; ++d) part = fmaf(q[d], Ks[uu][half * DH + d], part);
                const float x = (part + __shfl_xor_sync(0xffffffffu, part, 1)) * a.scale_log2;
                if (x > m) {
                    const float corr = exp2f(m - x);
                    m = x;
                    l *= corr;
#pragma unroll
                    for (int d = 0; d < DH; ++d) o[d] *= corr;
                }
                const float pw = exp2f(x - m);
                l += pw;
#pragma unroll
                for (int d = 0; d < DH; ++d) o[d] = fmaf(pw, Vs[uu][half * DH + d], o[d]);
            }
        }
    }
    // ---- compensation: zeroth order (+ grouped first order) over U_i ----
    if (a.comp != PASA_COMP_NONE && cnt < a.NK) {
        const T* Kb = reinterpret_cast<const T*>(a.kbar_lp) + bh * a.NK * D;
        const T* Vb = reinterpret_cast<const T*>(a.vsum_lp) + bh * a.NK * D;
        const T* Hb = reinterpret_cast<const T*>(a.ht) + bh * a.NG * D * D;
        const uint32_t* mrow = a.mask + row * a.W;
        float A = 0.f;          // A_{t,g} of the current group, same max reference as o, l
        int64_t gcur = 0;
        bool any_u = false;     // CTA-uniform: the group has a dropped block for this q-block
        auto flush = [&](int64_t g) {
            // o += s * A * (q_t Hbar^(g)) on this thread's half of the output dims;
            // (q_t Hbar)_n = sum_k q_k Ht[n][k], the k-sum split across the thread pair
            if (a.comp == PASA_COMP_GROUPED && any_u) {
                const T* Hg = Hb + g * D * D;
                const float w = a.s * A;
                for (int nn = 0; nn < DH; ++nn) {
                    const T* mine = Hg + (half * DH + nn) * D + half * DH;
                    const T* other = Hg + ((1 - half) * DH + nn) * D + half * DH;
                    float pa = 0.f, pb = 0.f;
#pragma unroll 8
                    for (int kk = 0; kk < DH; ++kk) {
                        pa = fmaf(q[kk], ld<T>(mine + kk), pa);
                        pb = fmaf(q[kk], ld<T>(other + kk), pb);
                    }
                    const float y = pa + __shfl_xor_sync(0xffffffffu, pb, 1);
                    o[nn] = fmaf(w, y, o[nn]);
                }
            }
            A = 0.f;
            any_u = false;
        };
        for (int64_t j = 0; j < a.NK; ++j) {
            const int64_t g = j / a.G;
            if (g != gcur) { flush(gcur); gcur = g; }
            if ((mrow[j >> 5] >> (j & 31)) & 1u) continue;
            any_u = true;
            float part = 0.f;
#pragma unroll
            for (int d = 0; d < DH; ++d) part = fmaf(q[d], ld<T>(Kb + j * D + half * DH + d), part);
            const float x = (part + __shfl_xor_sync(0xffffffffu, part, 1)) * a.scale_log2;
            if (x > m) {
                const float corr = exp2f(m - x);
                m = x;
                l *= corr;
                A *= corr;
#pragma unroll
                for (int d = 0; d < DH; ++d) o[d] *= corr;
            }
            const float pw = exp2f(x - m);
            const float nj = (float)min((int64_t)kBk, a.S - j * kBk);
            l = fmaf(nj, pw, l);
            A += pw;
#pragma unroll
            for (int d = 0; d < DH; ++d) o[d] = fmaf(pw, ld<T>(Vb + j * D + half * DH + d), o[d]);
        }
        flush(gcur);
    }
    if (live) {
        T* O = reinterpret_cast<T*>(a.out) + b * a.osB + h * a.osH + t * a.osS + half * DH;
        const float inv = 1.f / l;
#pragma unroll
        for (int d = 0; d < DH; ++d) O[d] = cvt<T>(o[d] * inv);
    }
}

}  // namespace

cudaError_t launch_attn_simt(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                             pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                             int* launches) {
    SimtArgs a;
    a.q = q.data; a.k = k.data; a.v = v.data; a.out = out.data;
    a.qsB = q.sB; a.qsS = q.sS; a.qsH = q.sH;
    a.ksB = k.sB; a.ksS = k.sS; a.ksH = k.sH;
    a.vsB = v.sB; a.vsS = v.sS; a.vsH = v.sH;
    a.osB = out.sB; a.osS = out.sS; a.osH = out.sH;
    a.S = r->S; a.H = r->H; a.NQ = r->NQ; a.NK = r->NK; a.NG = r->NG; a.W = r->W;
    a.Bq = r->cfg.Bq; a.G = r->cfg.G; a.comp = r->cfg.comp;
    a.s = (float)(1.0 / sqrt((double)r->D));
    a.scale_log2 = (float)(1.0 / sqrt((double)r->D) * 1.4426950408889634);
    a.idx = r->idx; a.count = r->count; a.mask = r->mask;
    a.kbar_lp = r->kbar_lp; a.vsum_lp = r->vsum_lp; a.ht = r->ht;
    a.it0 = r->it0;
    const unsigned grid = (unsigned)(r->it1 - r->it0);   // head-major items
    const int threads = 2 * r->cfg.Bq;
    if (q.dtype == PASA_F32) {
        if (r->D == 128) attn_simt_kernel<float, 128><<<grid, threads, 0, st>>>(a);
        else attn_simt_kernel<float, 64><<<grid, threads, 0, st>>>(a);
    } else {
        if (r->D == 128) attn_simt_kernel<__nv_bfloat16, 128><<<grid, threads, 0, st>>>(a);
        else attn_simt_kernel<__nv_bfloat16, 64><<<grid, threads, 0, st>>>(a);
    }
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace pasa
