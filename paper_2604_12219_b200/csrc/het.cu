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
//
// Three launches, each H_j computed once (B200: 180 GB of HBM, so every block's
// H_j is kept, 8 D^2 bytes per block, rather than recomputed for the norm):
//   1. het_hj_kernel:    H_j of every block into hj[bh][j] (one CTA per chunk of CB
//      consecutive blocks);
//   2. het_means_kernel: C = (1/N_K) sum_j H_j in ascending j (the oracle's order),
//      and in group mode the group means (slot g of hgs);
//   3. het_norm_kernel:  ||H_j - C||_F^2 per block, fixed-order reduction.
// Inside a het_hj_kernel CTA the K/V rows stream through shared memory in 32-token
// units: cp.async copies the raw rows of unit u+1 while unit u is converted to fp64
// (centred keys) and consumed by fp64 tensor-core MMAs (DMMA m8n8k4).
#include <cuda_bf16.h>

#include <cmath>

#include "pasa_internal.h"

namespace pasa {
namespace {

constexpr int kUnit = 32;       // tokens per pipeline unit (half a KV block)

template <typename T, int D>
constexpr size_t het_smem_units() {   // fp64 units with padded rows + the raw double buffer
    return (size_t)2 * kUnit * (D + 8) * sizeof(double) + (size_t)4 * kUnit * D * sizeof(T);
}

struct HetArgs {
    const void* k;
    const void* v;
    int64_t ksB, ksS, ksH, vsB, vsS, vsH;   // element strides
    int64_t S, H, NK, NG, G, CB, NC;
    const double* kbar;    // [BH][NK][D] fp64 block means (pool_kernel)
    double* hj;            // [BH][NK][D][D] H_j of every block
    double* part;          // [BH][>= NG][D][D] group means (group mode)
    double* cglob;         // [BH][D][D] global mean
    int32_t mode;          // PASA_PRIOR_GLOBAL / PASA_PRIOR_GROUP
    double eps;
    double* het;           // [BH][NK]
    double* prior;         // [BH][NK]
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;       // src-size 0: zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ double to_d(float x) { return (double)x; }
__device__ __forceinline__ double to_d(__nv_bfloat16 x) { return (double)__bfloat162float(x); }

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// H_j = Kc^T V per block on the fp64 tensor core (DMMA m8n8k4, operands from registers:
// ~14 fma per loaded double instead of ~3 with the register-tiled DFMA loop).  GEMM
// view: M = N = D (rows r of Kc^T, columns c of V), K = the block's tokens.  Warp w owns
// row tiles [w RTW, (w+1) RTW) x every column tile (32 8x8 tiles, 64 fp64 accumulators
// per thread).  Fragments (PTX m8n8k4.f64): A[r][n] lane (r = lane/4, n = lane%4),
// B[n][c] lane (n = lane%4, c = lane/4), C[r][c] lane (r = lane/4, c = 2(lane%4)+{0,1}).
// Each DMMA step rounds like the sequential fma chain over its four k (tools/dmma_exact.cu),
// but the token sum here runs unit-wise over centred rows in a different grouping from the
// oracle's (and the Frobenius norm sums in another order), so H_j and het_j differ from the
// oracle's by ~1e-16 relative: the prior's tolerance against the oracle is 1e-10 (R-26).
template <typename T, int D>
__global__ void __launch_bounds__(D * D / 64, 1) het_hj_kernel(HetArgs a) {
    constexpr int NT = D * D / 64;                   // threads: 256 at d = 128, 64 at d = 64
    constexpr int NW = NT / 32;
    constexpr int CT = D / 8;                        // column tiles
    constexpr int RTW = (D / 8) / NW;                // row tiles per warp (CT * RTW = 32)
    constexpr int DP = D + 8;                        // padded fp64 row: conflict-free fragments
    constexpr int ROWB = D * (int)sizeof(T);         // bytes per raw row
    constexpr int RAWB = kUnit * ROWB;               // bytes per raw unit per tensor
    extern __shared__ __align__(16) uint8_t smem[];
    double* kt = reinterpret_cast<double*>(smem);                      // [kUnit][DP]
    double* vt = kt + kUnit * DP;                                       // [kUnit][DP]
    uint8_t* raw = reinterpret_cast<uint8_t*>(vt + kUnit * DP);        // [2][K|V][RAWB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fk = lane & 3;         // fragment row / k index
    const int64_t bh = blockIdx.y, chunk = blockIdx.x;
    const int64_t b = bh / a.H, h = bh % a.H;
    const T* K = reinterpret_cast<const T*>(a.k) + b * a.ksB + h * a.ksH;
    const T* V = reinterpret_cast<const T*>(a.v) + b * a.vsB + h * a.vsH;
    const int64_t j_lo = chunk * a.CB, j_hi = min(j_lo + a.CB, a.NK);
    const int n_units = (int)(2 * (j_hi - j_lo));

    auto issue = [&](int u) {                        // raw rows of unit u -> buffer u & 1
        const int64_t t0 = j_lo * 64 + (int64_t)u * kUnit;
        uint8_t* dst = raw + (u & 1) * 2 * RAWB;
        for (int e = tid; e < 2 * RAWB / 16; e += NT) {
            const int tens = e / (RAWB / 16), w = e % (RAWB / 16);
            const int n = w / (ROWB / 16), c16 = w % (ROWB / 16);
            const int64_t tok = t0 + n;
            const bool ok = tok < a.S;
            const T* src = tens ? V + (ok ? tok : 0) * a.vsS : K + (ok ? tok : 0) * a.ksS;
            cp_async16(dst + tens * RAWB + n * ROWB + c16 * 16,
                       reinterpret_cast<const uint8_t*>(src) + c16 * 16, ok);
        }
        cp_async_commit();
    };

    double acc[RTW][CT][2];
#pragma unroll
    for (int i = 0; i < RTW; ++i)
#pragma unroll
        for (int c = 0; c < CT; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;
    if (n_units > 0) issue(0);
    for (int u = 0; u < n_units; ++u) {
        const int64_t j = j_lo + u / 2;
        const int64_t t0 = j * 64 + (u & 1) * kUnit;
        const int valid = (int)max((int64_t)0, min((int64_t)kUnit, a.S - t0));
        cp_async_wait0();
        __syncthreads();                              // raw(u) landed; kt/vt free
        {
            const uint8_t* src = raw + (u & 1) * 2 * RAWB;
            const double* kb = a.kbar + (bh * a.NK + j) * D;
            for (int e = tid; e < kUnit * D; e += NT) {
                const int n = e / D, col = e % D;
                double kv = 0.0, vv = 0.0;
                if (n < valid) {                      // ragged tail rows contribute nothing
                    kv = to_d(reinterpret_cast<const T*>(src)[n * D + col]) - kb[col];
                    vv = to_d(reinterpret_cast<const T*>(src + RAWB)[n * D + col]);
                }
                kt[n * DP + col] = kv;
                vt[n * DP + col] = vv;
            }
        }
        __syncthreads();                              // fp64 unit ready; raw(u) consumed
        if (u + 1 < n_units) issue(u + 1);
        const int nsteps = (valid + 3) >> 2;          // zero rows past `valid` add nothing
        for (int s4 = 0; s4 < nsteps; ++s4) {
            const double* krow = kt + (4 * s4 + fk) * DP;
            const double* vrow = vt + (4 * s4 + fk) * DP;
            double av[RTW], bv[CT];
#pragma unroll
            for (int i = 0; i < RTW; ++i) av[i] = krow[(warp * RTW + i) * 8 + fr];
#pragma unroll
            for (int c = 0; c < CT; ++c) bv[c] = vrow[c * 8 + fr];
#pragma unroll
            for (int i = 0; i < RTW; ++i)
#pragma unroll
                for (int c = 0; c < CT; ++c) dmma_8x8x4(acc[i][c][0], acc[i][c][1], av[i], bv[c]);
        }
        if (u & 1) {                                  // block j complete: store H_j
            double* out = a.hj + (bh * a.NK + j) * (int64_t)D * D;
#pragma unroll
            for (int i = 0; i < RTW; ++i)
#pragma unroll
                for (int c = 0; c < CT; ++c) {
                    const int r = (warp * RTW + i) * 8 + fr, col = c * 8 + 2 * fk;
                    *reinterpret_cast<double2*>(&out[r * D + col]) =
                        make_double2(acc[i][c][0], acc[i][c][1]);
                    acc[i][c][0] = acc[i][c][1] = 0.0;
                }
        }
    }
}

// C: global mean (1/N_K) sum_j H_j, blocks in ascending order (Eq. 6, as the oracle);
// in group mode the group means (unweighted, App. B) into slot g of part.
template <int D>
__global__ void __launch_bounds__(256) het_means_kernel(HetArgs a) {
    const int64_t bh = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (e >= (int64_t)D * D) return;
    const double* hj = a.hj + bh * a.NK * (int64_t)D * D + e;
    double total = 0.0;
    for (int64_t g = 0; g < a.NG; ++g) {
        const int64_t jb = g * a.G, je = min(jb + a.G, a.NK);
        double s = 0.0;
        for (int64_t j = jb; j < je; ++j) {
            const double x = hj[j * (int64_t)D * D];
            s += x;
            total += x;
        }
        if (a.mode == PASA_PRIOR_GROUP)
            a.part[(bh * a.NG + g) * (int64_t)D * D + e] = s / (double)(je - jb);
    }
    a.cglob[bh * (int64_t)D * D + e] = total / (double)a.NK;
}

// het_j = ||H_j - C||_F, log(het_j + eps): one CTA per (block, head), fixed-order
// reduction (thread partials in ascending element order, warps in order).
template <int D>
__global__ void __launch_bounds__(256) het_norm_kernel(HetArgs a) {
    const int64_t j = blockIdx.x, bh = blockIdx.y;
    const double* Hj = a.hj + (bh * a.NK + j) * (int64_t)D * D;
    const double* C = a.mode == PASA_PRIOR_GROUP ? a.part + (bh * a.NG + j / a.G) * (int64_t)D * D
                                                 : a.cglob + bh * (int64_t)D * D;
    __shared__ double red[8];
    double p = 0.0;
    for (int e = threadIdx.x; e < D * D; e += 256) {
        const double d = Hj[e] - C[e];
        p = fma(d, d, p);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < 8; ++w) tot += red[w];
        const double hv = sqrt(tot);
        a.het[bh * a.NK + j] = hv;
        a.prior[bh * a.NK + j] = log(hv + a.eps);
    }
}

template <typename T, int D>
cudaError_t launch_d(const HetArgs& a, int64_t BH, cudaStream_t st) {
    const size_t smem = het_smem_units<T, D>();
    cudaError_t e = cudaFuncSetAttribute(het_hj_kernel<T, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    het_hj_kernel<T, D><<<dim3((unsigned)a.NC, (unsigned)BH), D * D / 64, smem, st>>>(a);
    het_means_kernel<D><<<dim3((unsigned)((D * D + 255) / 256), (unsigned)BH), 256, 0, st>>>(a);
    het_norm_kernel<D><<<dim3((unsigned)a.NK, (unsigned)BH), 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

// chunk size: the largest divisor of G that is <= 32 (32 when one group spans all)
int64_t het_chunk_blocks(int64_t G, int64_t NK) {
    if (G >= NK) return 32;
    for (int64_t d = 32; d > 1; --d)
        if (G % d == 0) return d;
    return 1;
}

cudaError_t launch_het(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r,
                       cudaStream_t st, int* launches) {
    HetArgs a;
    a.k = k.data; a.v = v.data;
    a.ksB = k.sB; a.ksS = k.sS; a.ksH = k.sH;
    a.vsB = v.sB; a.vsS = v.sS; a.vsH = v.sH;
    a.S = r->S; a.H = r->H; a.NK = r->NK; a.NG = r->NG; a.G = r->cfg.G;
    a.CB = het_chunk_blocks(a.G, a.NK);
    a.NC = (a.NK + a.CB - 1) / a.CB;
    a.kbar = r->kbar; a.hj = r->hj; a.part = r->hgs; a.cglob = r->hglob;
    a.mode = r->cfg.prior; a.eps = r->cfg.eps;
    a.het = r->het; a.prior = r->prior;
    const bool f32 = k.dtype == PASA_F32;
    cudaError_t e;
    if (r->D == 128)
        e = f32 ? launch_d<float, 128>(a, r->BH, st) : launch_d<__nv_bfloat16, 128>(a, r->BH, st);
    else
        e = f32 ? launch_d<float, 64>(a, r->BH, st) : launch_d<__nv_bfloat16, 64>(a, r->BH, st);
    *launches += 3;
    return e;
}

}  // namespace pasa
