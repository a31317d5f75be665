// kv_stats.cu -- the key/value block statistics pasa_attn compensates with
// (step a6 of SURVEY.md §8a):
//   Kbar_j     (low-precision copy of the route's fp64 block means),
//   Vsum_j   = sum_n V_{j,n}                                  (Eq. 4 inner sum)
//   Hbar^(g) = (1/|G_g|) sum_{j in G_g} sum_n (K_{j,n} - Kbar_j)^T V_{j,n}
//                                          (Eq. 5 + App. B)
// stored transposed (Ht[n][k] = Hbar[k][n]) so pasa_attn can feed it to the
// tensor cores as a K-major B operand.  Per-block H_j is never materialised
// ("Directly computing H_j for every block results in a memory-bound
// operation"): one CTA per (head, group) streams the group's
// K/V blocks once and contracts the centred keys with the values on the
// tensor cores (bf16 in, fp32 accumulate; R-21).
#include <cuda_bf16.h>

#include "pasa_internal.h"

namespace pasa {
namespace {

constexpr int kBk = 64;
constexpr int kPad = 8;   // bf16 elements of row padding (bank spread)

__device__ __forceinline__ void mma_bf16_16816(float c[4], const uint32_t a[4],
                                               const uint32_t b[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, "
        "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

struct StatsArgs {
    const void* k;
    const void* v;
    int64_t ksB, ksS, ksH, vsB, vsS, vsH;
    int64_t S, H, NK, NG;
    int32_t G;
    const double* kbar;   // [BH][NK][D] fp64 (route)
    void* kbar_lp;        // [BH][NK][D]
    void* vsum_lp;        // [BH][NK][D]
    void* ht;             // [BH][NG][D][D]
};

// ---- bf16: mma.sync contraction, 256 threads, one CTA per (head, group) ----
template <int D>
__global__ void __launch_bounds__(256) stats_bf16_kernel(StatsArgs a) {
    constexpr int NWR = D / 16;          // warps along Ht rows (n)
    constexpr int NWC = 8 / NWR;         // warps along Ht cols (k)
    constexpr int COLS = D / NWC;        // k columns per warp
    constexpr int NT = COLS / 8;         // n8 tiles per warp
    constexpr int LD = kBk + kPad;
    __shared__ __align__(16) __nv_bfloat16 Vt[D][LD];
    __shared__ __align__(16) __nv_bfloat16 Kct[D][LD];
    __shared__ float kb[D];

    const int64_t bh = blockIdx.y, g = blockIdx.x;
    const int64_t b = bh / a.H, h = bh % a.H;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row0 = (warp % NWR) * 16, col0 = (warp / NWR) * COLS;
    const int gq = lane >> 2, cq = lane & 3;
    const __nv_bfloat16* K = reinterpret_cast<const __nv_bfloat16*>(a.k) + b * a.ksB + h * a.ksH;
    const __nv_bfloat16* V = reinterpret_cast<const __nv_bfloat16*>(a.v) + b * a.vsB + h * a.vsH;

    float acc[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[t][e] = 0.f;

    const int64_t j0 = g * a.G, j1 = min(j0 + (int64_t)a.G, a.NK);
    for (int64_t j = j0; j < j1; ++j) {
        const int64_t t0 = j * kBk;
        const int nj = (int)min((int64_t)kBk, a.S - t0);
        const double* kbj = a.kbar + (bh * a.NK + j) * D;
        if (tid < D) {
            kb[tid] = (float)kbj[tid];
            reinterpret_cast<__nv_bfloat16*>(a.kbar_lp)[(bh * a.NK + j) * D + tid] =
                __float2bfloat16_rn((float)kbj[tid]);
        }
        __syncthreads();
        // load + centre + transpose: 8 dims per thread-iteration
        for (int e = tid; e < kBk * (D / 8); e += 256) {
            const int t = e / (D / 8), d8 = (e % (D / 8)) * 8;
            uint4 ku = make_uint4(0, 0, 0, 0), vu = make_uint4(0, 0, 0, 0);
            if (t < nj) {
                ku = __ldg(reinterpret_cast<const uint4*>(K + (t0 + t) * a.ksS + d8));
                vu = __ldg(reinterpret_cast<const uint4*>(V + (t0 + t) * a.vsS + d8));
            }
            const __nv_bfloat16* kk = reinterpret_cast<const __nv_bfloat16*>(&ku);
            const __nv_bfloat16* vv = reinterpret_cast<const __nv_bfloat16*>(&vu);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float kc = t < nj ? __bfloat162float(kk[u]) - kb[d8 + u] : 0.f;
                Kct[d8 + u][t] = __float2bfloat16_rn(kc);
                Vt[d8 + u][t] = vv[u];
            }
        }
        __syncthreads();
        if (tid < D) {
            float s = 0.f;
            for (int t = 0; t < kBk; ++t) s += __bfloat162float(Vt[tid][t]);
            reinterpret_cast<__nv_bfloat16*>(a.vsum_lp)[(bh * a.NK + j) * D + tid] =
                __float2bfloat16_rn(s);
        }
#pragma unroll
        for (int ks = 0; ks < kBk / 16; ++ks) {
            const int tc = ks * 16 + 2 * cq;
            uint32_t af[4];
            af[0] = *reinterpret_cast<const uint32_t*>(&Vt[row0 + gq][tc]);
            af[1] = *reinterpret_cast<const uint32_t*>(&Vt[row0 + gq + 8][tc]);
            af[2] = *reinterpret_cast<const uint32_t*>(&Vt[row0 + gq][tc + 8]);
            af[3] = *reinterpret_cast<const uint32_t*>(&Vt[row0 + gq + 8][tc + 8]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int kcol = col0 + nt * 8 + gq;
                uint32_t bfr[2];
                bfr[0] = *reinterpret_cast<const uint32_t*>(&Kct[kcol][tc]);
                bfr[1] = *reinterpret_cast<const uint32_t*>(&Kct[kcol][tc + 8]);
                mma_bf16_16816(acc[nt], af, bfr);
            }
        }
        __syncthreads();
    }
    const float inv = 1.f / (float)(j1 - j0);
    __nv_bfloat16* Ht = reinterpret_cast<__nv_bfloat16*>(a.ht) + (bh * a.NG + g) * D * D;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int kc = col0 + nt * 8 + 2 * cq;
        __nv_bfloat162 lo = __floats2bfloat162_rn(acc[nt][0] * inv, acc[nt][1] * inv);
        __nv_bfloat162 hi = __floats2bfloat162_rn(acc[nt][2] * inv, acc[nt][3] * inv);
        *reinterpret_cast<__nv_bfloat162*>(&Ht[(row0 + gq) * D + kc]) = lo;
        *reinterpret_cast<__nv_bfloat162*>(&Ht[(row0 + gq + 8) * D + kc]) = hi;
    }
}

// ---- fp32: CUDA-core contraction (fp32 I/O mode; not a performance path) ----
template <int D>
__global__ void __launch_bounds__(256) stats_f32_kernel(StatsArgs a) {
    constexpr int TT = 16;                 // tokens staged per pass
    constexpr int CPT = D * D / 256;       // Ht columns per thread
    constexpr int TPR = D / CPT;           // threads per Ht row
    __shared__ float Ks[TT][D];
    __shared__ float Vs[TT][D];
    __shared__ float kb[D];
    const int64_t bh = blockIdx.y, g = blockIdx.x;
    const int64_t b = bh / a.H, h = bh % a.H;
    const int tid = threadIdx.x;
    const int n = tid / TPR, c0 = (tid % TPR) * CPT;
    const float* K = reinterpret_cast<const float*>(a.k) + b * a.ksB + h * a.ksH;
    const float* V = reinterpret_cast<const float*>(a.v) + b * a.vsB + h * a.vsH;
    float acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.f;
    const int64_t j0 = g * a.G, j1 = min(j0 + (int64_t)a.G, a.NK);
    for (int64_t j = j0; j < j1; ++j) {
        const int64_t t0 = j * kBk;
        const int nj = (int)min((int64_t)kBk, a.S - t0);
        const double* kbj = a.kbar + (bh * a.NK + j) * D;
        float vs = 0.f;
        if (tid < D) {
            kb[tid] = (float)kbj[tid];
            reinterpret_cast<float*>(a.kbar_lp)[(bh * a.NK + j) * D + tid] = (float)kbj[tid];
        }
        for (int tt = 0; tt < nj; tt += TT) {
            __syncthreads();
            for (int e = tid; e < TT * D; e += 256) {
                const int t = e / D, d = e % D;
                const bool ok = tt + t < nj;
                Ks[t][d] = ok ? K[(t0 + tt + t) * a.ksS + d] - kb[d] : 0.f;
                Vs[t][d] = ok ? V[(t0 + tt + t) * a.vsS + d] : 0.f;
            }
            __syncthreads();
            if (tid < D)
                for (int t = 0; t < TT; ++t) vs += Vs[t][tid];
#pragma unroll 4
            for (int t = 0; t < TT; ++t) {
                const float vn = Vs[t][n];
#pragma unroll
                for (int c = 0; c < CPT; ++c) acc[c] = fmaf(vn, Ks[t][c0 + c], acc[c]);
            }
        }
        if (tid < D) reinterpret_cast<float*>(a.vsum_lp)[(bh * a.NK + j) * D + tid] = vs;
        __syncthreads();
    }
    const float inv = 1.f / (float)(j1 - j0);
    float* Ht = reinterpret_cast<float*>(a.ht) + (bh * a.NG + g) * D * D;
#pragma unroll
    for (int c = 0; c < CPT; ++c) Ht[n * D + c0 + c] = acc[c] * inv;
}

}  // namespace

cudaError_t launch_kv_stats(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r,
                            cudaStream_t st, int* launches) {
    StatsArgs a;
    a.k = k.data; a.v = v.data;
    a.ksB = k.sB; a.ksS = k.sS; a.ksH = k.sH;
    a.vsB = v.sB; a.vsS = v.sS; a.vsH = v.sH;
    a.S = r->S; a.H = r->H; a.NK = r->NK; a.NG = r->NG; a.G = r->cfg.G;
    a.kbar = r->kbar; a.kbar_lp = r->kbar_lp; a.vsum_lp = r->vsum_lp; a.ht = r->ht;
    if (k.dtype == PASA_BF16 && kv_stats_sm100_supported(r) && !(g_dbg & 16))
        return launch_kv_stats_sm100(k, v, r, st, launches);
    dim3 grid((unsigned)r->NG, (unsigned)r->BH);
    if (k.dtype == PASA_BF16) {
        if (r->D == 128) stats_bf16_kernel<128><<<grid, 256, 0, st>>>(a);
        else stats_bf16_kernel<64><<<grid, 256, 0, st>>>(a);
    } else {
        if (r->D == 128) stats_f32_kernel<128><<<grid, 256, 0, st>>>(a);
        else stats_f32_kernel<64><<<grid, 256, 0, st>>>(a);
    }
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace pasa
