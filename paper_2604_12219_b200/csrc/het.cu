// het.cu -- Eq. 8's heterogeneity prior (
// SURVEY.md §8f NEXT 1): per KV block j of every head
//     H_j   = sum_n (K_n - Kbar_j)^T V_n            (Eq. 5, d x d)
//     het_j = ||H_j - C||_F                          (Frobenius)
//     prior_j = log(het_j + eps)                     (added to r_ij by scores_kernel)
// with C the global mean Hbar = (1/N_K) sum_j H_j (Eq. 6; Eq. 8 literally,
// PASA_PRIOR_GLOBAL) or the group mean Hbar^(g(j)) (App. B, PASA_PRIOR_GROUP).
//
// fp64 on the CUDA cores: the prior feeds the top-k, so it must agree with the
// fp64 oracle far inside the routing tie tolerance (1e-6 relative);
// fp32 tensor-core accumulation of 64-term sums would sit at that tolerance.
// Three launches: group sums of H_j (one CTA per (head, group), all tokens of
// the group in one accumulator: sum_{j in g} H_j = sum_{n in g} (K_n - Kbar_j(n))^T V_n),
// the means C (fixed group order, deterministic), then one CTA per (head, block)
// recomputing H_j and reducing ||H_j - C||_F^2 in a fixed order.
// Thread layout: D^2/64 threads, each owns a 4-row x 16-column patch of H (fp64
// registers); 16-token chunks of the centred keys and the values are staged in
// shared memory as fp64 (column reads are warp broadcasts).
#include <cuda_bf16.h>

#include <cmath>

#include "pasa_internal.h"

namespace pasa {
namespace {

constexpr int kChunk = 16;   // 2 x 16 x 128 fp64 = 32 KB static smem

struct HetArgs {
    const void* k;
    const void* v;
    int64_t ksB, ksS, ksH, vsB, vsS, vsH;   // element strides
    int64_t S, H, NK, NG, G;
    const double* kbar;    // [BH][NK][D] fp64 block means (pool_kernel)
    double* gsum;          // [BH][NG][D][D] group sums, then (group mode) group means
    const double* cglob;   // [BH][D][D] global mean (NORM pass, global mode)
    int32_t mode;          // PASA_PRIOR_GLOBAL / PASA_PRIOR_GROUP
    double eps;
    double* het;           // [BH][NK]
    double* prior;         // [BH][NK]
};

__device__ __forceinline__ double ld(const float* p) { return (double)*p; }
__device__ __forceinline__ double ld(const __nv_bfloat16* p) { return (double)__bfloat162float(*p); }

template <typename T, int D, bool NORM>
__global__ void __launch_bounds__(D * D / 64, 1) het_kernel(HetArgs a) {
    constexpr int NT = D * D / 64;
    constexpr int RT = D / 4;                // row groups of 4
    __shared__ __align__(16) double kt[kChunk][D];
    __shared__ __align__(16) double vt[kChunk][D];
    __shared__ double red[NT / 32];
    const int tid = threadIdx.x;
    const int r0 = 4 * (tid % RT), c0 = 16 * (tid / RT);
    const int64_t bh = blockIdx.y;
    const int64_t b = bh / a.H, h = bh % a.H;
    const T* K = reinterpret_cast<const T*>(a.k) + b * a.ksB + h * a.ksH;
    const T* V = reinterpret_cast<const T*>(a.v) + b * a.vsB + h * a.vsH;
    const int64_t j_lo = NORM ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * a.G;
    const int64_t j_hi = NORM ? j_lo + 1 : min(j_lo + a.G, a.NK);
    double acc[4][16];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[i][c] = 0.0;
    for (int64_t j = j_lo; j < j_hi; ++j) {
        const double* kb = a.kbar + (bh * a.NK + j) * D;
        const int64_t t0 = j * 64, t1 = min(t0 + 64, a.S);
        for (int64_t tc = t0; tc < t1; tc += kChunk) {
            const int n_chunk = (int)min((int64_t)kChunk, t1 - tc);
            __syncthreads();
            for (int e = tid; e < kChunk * D; e += NT) {
                const int n = e / D, col = e % D;
                double kv = 0.0, vv = 0.0;
                if (n < n_chunk) {
                    kv = ld(K + (tc + n) * a.ksS + col) - kb[col];   // K_n - Kbar_j in fp64
                    vv = ld(V + (tc + n) * a.vsS + col);
                }
                kt[n][col] = kv;
                vt[n][col] = vv;
            }
            __syncthreads();
            for (int n = 0; n < n_chunk; ++n) {
                const double2 k01 = *reinterpret_cast<const double2*>(&kt[n][r0]);
                const double2 k23 = *reinterpret_cast<const double2*>(&kt[n][r0 + 2]);
                const double kr[4] = {k01.x, k01.y, k23.x, k23.y};
                double vr[16];
#pragma unroll
                for (int c = 0; c < 16; c += 2) {
                    const double2 t = *reinterpret_cast<const double2*>(&vt[n][c0 + c]);
                    vr[c] = t.x;
                    vr[c + 1] = t.y;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int c = 0; c < 16; ++c) acc[i][c] = fma(kr[i], vr[c], acc[i][c]);
            }
        }
    }
    if constexpr (!NORM) {
        double* out = a.gsum + (bh * a.NG + blockIdx.x) * (int64_t)D * D;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 16; ++c) out[(r0 + i) * D + c0 + c] = acc[i][c];
    } else {
        const double* C = a.mode == PASA_PRIOR_GROUP
                              ? a.gsum + (bh * a.NG + j_lo / a.G) * (int64_t)D * D
                              : a.cglob + bh * (int64_t)D * D;
        double part = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const double d = acc[i][c] - C[(r0 + i) * D + c0 + c];
                part = fma(d, d, part);
            }
        // fixed-order reduction: xor tree inside each warp, then warps in order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if ((tid & 31) == 0) red[tid >> 5] = part;
        __syncthreads();
        if (tid == 0) {
            double tot = 0.0;
            for (int w = 0; w < NT / 32; ++w) tot += red[w];
            const double hv = sqrt(tot);
            a.het[bh * a.NK + j_lo] = hv;
            a.prior[bh * a.NK + j_lo] = log(hv + a.eps);
        }
    }
}

// C: global mean (1/N_K) sum_g gsum_g (groups in ascending order); in group mode
// the group sums are turned into group means in place (unweighted, App. B).
template <int D>
__global__ void __launch_bounds__(256) het_means_kernel(HetArgs a) {
    const int64_t bh = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (e >= (int64_t)D * D) return;
    double* gs = a.gsum + bh * a.NG * (int64_t)D * D + e;
    double s = 0.0;
    for (int64_t g = 0; g < a.NG; ++g) s += gs[g * (int64_t)D * D];
    const_cast<double*>(a.cglob)[bh * (int64_t)D * D + e] = s / (double)a.NK;
    if (a.mode == PASA_PRIOR_GROUP)
        for (int64_t g = 0; g < a.NG; ++g) {
            const int64_t cnt = min(a.G, a.NK - g * a.G);
            gs[g * (int64_t)D * D] = gs[g * (int64_t)D * D] / (double)cnt;
        }
}

template <typename T, int D>
void launch_d(const HetArgs& a, int64_t BH, cudaStream_t st) {
    het_kernel<T, D, false><<<dim3((unsigned)a.NG, (unsigned)BH), D * D / 64, 0, st>>>(a);
    het_means_kernel<D><<<dim3((unsigned)((D * D + 255) / 256), (unsigned)BH), 256, 0, st>>>(a);
    het_kernel<T, D, true><<<dim3((unsigned)a.NK, (unsigned)BH), D * D / 64, 0, st>>>(a);
}

}  // namespace

cudaError_t launch_het(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r,
                       cudaStream_t st, int* launches) {
    HetArgs a;
    a.k = k.data; a.v = v.data;
    a.ksB = k.sB; a.ksS = k.sS; a.ksH = k.sH;
    a.vsB = v.sB; a.vsS = v.sS; a.vsH = v.sH;
    a.S = r->S; a.H = r->H; a.NK = r->NK; a.NG = r->NG; a.G = r->cfg.G;
    a.kbar = r->kbar; a.gsum = r->hgs; a.cglob = r->hglob;
    a.mode = r->cfg.prior; a.eps = r->cfg.eps;
    a.het = r->het; a.prior = r->prior;
    const bool f32 = k.dtype == PASA_F32;
    if (r->D == 128) {
        if (f32) launch_d<float, 128>(a, r->BH, st); else launch_d<__nv_bfloat16, 128>(a, r->BH, st);
    } else {
        if (f32) launch_d<float, 64>(a, r->BH, st); else launch_d<__nv_bfloat16, 64>(a, r->BH, st);
    }
    *launches += 3;
    return cudaGetLastError();
}

}  // namespace pasa
