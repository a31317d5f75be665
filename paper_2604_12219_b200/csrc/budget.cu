// budget.cu -- pasa_budget: the curvature (trajectory-acceleration) reduction
// over the last three latents and the per-step density of Eqs. 9-11
// (readings R-15..R-18 in DESIGN.md §3).
//
// HBM-bound: reads 3 * n * sizeof(elem) bytes once.  Fixed grid of
// kBudgetParts CTAs, each reducing one contiguous chunk in fp64 with a fixed
// shuffle tree, then a single-CTA finaliser that sums the partials in a fixed
// tree: l1 is bit-identical run to run (not bit-identical to the sequential
// oracle; tolerance 1e-12 relative).
#include <cuda_bf16.h>

#include "pasa_internal.h"

namespace pasa {
namespace {

constexpr int kThreads = 256;

template <typename T>
__device__ __forceinline__ void load4(const T* p, int64_t e, double out[4]);

template <>
__device__ __forceinline__ void load4<float>(const float* p, int64_t e, double out[4]) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p + e));
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* p, int64_t e,
                                                     double out[4]) {
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p + e));
    __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&v.x);
    __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v.y);
    out[0] = __bfloat162float(a.x); out[1] = __bfloat162float(a.y);
    out[2] = __bfloat162float(b.x); out[3] = __bfloat162float(b.y);
}
template <typename T>
__device__ __forceinline__ double load1(const T* p, int64_t e) {
    if constexpr (sizeof(T) == 4) return (double)__ldg(p + e);
    else return (double)__bfloat162float(p[e]);
}

// |dv| for one element, B1 of DESIGN.md §3: two subtractions in IEEE double and
// the two velocity scalings as multiplications by the host-computed reciprocals
// 1/h (each within 1 ulp of the division; the mean l1 stays within the 1e-12
// relative tolerance of DESIGN.md §6, and fp64 division would make the kernel
// ALU-bound instead of HBM-bound).
__device__ __forceinline__ double accel(double xt, double x1, double x2, int kind, double rht,
                                        double rh1) {
    if (kind == 1) return fabs(__dsub_rn(xt, x1));
    double a = __dsub_rn(xt, x1);
    double b = __dsub_rn(x1, x2);
    return fabs(__dsub_rn(__dmul_rn(a, rht), __dmul_rn(b, rh1)));
}

// Eq. 10 alpha = l / l-bar; Eq. 11 rho_t = rho * alpha (or the table entry),
// clipped at rho_max (R-18); dense prefix (R-15) -> rho_t = 1.
__device__ __forceinline__ void finish_record(double l, const BudgetParams& p, BudgetRec* rec) {
    const double alpha = l / p.l1_mean;
    double rho_t, dense = 0.0, clipped = 0.0;
    if (p.step < p.dense_steps || p.step < 2) {
        rho_t = 1.0;
        dense = 1.0;
    } else {
        const double rp = p.use_table ? p.table_val : __dmul_rn(p.rho, alpha);
        if (rp > p.rho_max) { rho_t = p.rho_max; clipped = 1.0; }
        else rho_t = rp;
    }
    rec->l1 = l; rec->alpha = alpha; rec->rho_t = rho_t; rec->dense = dense;
    rec->clipped = clipped;
}

// One launch: a fixed grid of kBudgetParts CTAs each reduce one contiguous chunk in
// fp64 with a fixed shuffle tree; the last CTA to finish (completion ticket) sums the
// partials in a fixed tree and writes the record (or, for sharded latents, the local
// sum), then resets the ticket.  Bit-identical run to run.
template <typename T>
__global__ void __launch_bounds__(kThreads) budget_kernel(
    const T* __restrict__ xt, const T* __restrict__ x1, const T* __restrict__ x2, int64_t n,
    int kind, BudgetParams p, double* __restrict__ partials, unsigned int* ticket,
    BudgetRec* __restrict__ rec, double* __restrict__ local_sum) {
    // chunk of a multiple of 4 elements per CTA (vector loads stay aligned)
    const int64_t chunk = ((n + kBudgetParts - 1) / kBudgetParts + 3) & ~int64_t(3);
    const int64_t e0 = (int64_t)blockIdx.x * chunk;
    const int64_t e1 = min(e0 + chunk, n);
    double acc = 0.0;
    if (e0 < e1) {
        const int64_t nv = (e1 - e0) & ~int64_t(3);
        for (int64_t e = e0 + 4 * (int64_t)threadIdx.x; e < e0 + nv; e += 4 * kThreads) {
            double a[4], b[4], c[4];
            load4<T>(xt, e, a);
            load4<T>(x1, e, b);
            if (kind == 0) load4<T>(x2, e, c);
            else { c[0] = c[1] = c[2] = c[3] = 0.0; }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += accel(a[u], b[u], c[u], kind, p.rht, p.rh1);
        }
        for (int64_t e = e0 + nv + threadIdx.x; e < e1; e += kThreads)
            acc += accel(load1<T>(xt, e), load1<T>(x1, e), kind == 0 ? load1<T>(x2, e) : 0.0,
                         kind, p.rht, p.rh1);
    }
    // fixed-order reduction: warp shuffle tree, then warp 0 over the warp sums
    __shared__ double warp_sum[kThreads / 32];
    __shared__ bool last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < kThreads / 32 ? warp_sum[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) {
            partials[blockIdx.x] = v;
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (!last) return;
    // the last CTA: every other CTA's partial is visible (fence before its ticket)
    __threadfence();
    __shared__ double s[kBudgetParts];
    for (int i = threadIdx.x; i < kBudgetParts; i += blockDim.x)
        s[i] = __ldcg(partials + i);
    __syncthreads();
    for (int w = kBudgetParts / 2; w > 0; w >>= 1) {
        for (int i = threadIdx.x; i < w; i += blockDim.x) s[i] = s[i] + s[i + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *ticket = 0u;
        if (local_sum) *local_sum = s[0];
        else finish_record(n > 0 ? s[0] / (double)n : 0.0, p, rec);
    }
}

// sharded latents: l = (sum of the ranks' local sums, in rank order) / n_total
__global__ void budget_from_sums_kernel(const double* __restrict__ sums, int32_t nsums,
                                        int64_t n_total, BudgetParams p,
                                        BudgetRec* __restrict__ rec) {
    double acc = 0.0;
    for (int32_t r = 0; r < nsums; ++r) acc += sums[r];
    finish_record(acc / (double)n_total, p, rec);
}

}  // namespace

cudaError_t launch_budget(const void* xt, const void* xtm1, const void* xtm2, int64_t n, int dtype,
                          int kind, const BudgetParams& p, pasa_budget_s* b, double* local_sum,
                          cudaStream_t st, int* launches) {
    // the completion ticket starts at 0: zeroed once, on the handle's first launch (stream
    // ordered, graph capturable); every launch's last CTA resets it afterwards
    if (!b->ticket_ready) {
        const cudaError_t e = cudaMemsetAsync(b->ticket, 0, sizeof(unsigned int), st);
        if (e != cudaSuccess) return e;
        b->ticket_ready = 1;
    }
    if (dtype == PASA_F32)
        budget_kernel<float><<<kBudgetParts, kThreads, 0, st>>>(
            (const float*)xt, (const float*)xtm1, (const float*)xtm2, n, kind, p, b->partials,
            b->ticket, b->rec, local_sum);
    else
        budget_kernel<__nv_bfloat16><<<kBudgetParts, kThreads, 0, st>>>(
            (const __nv_bfloat16*)xt, (const __nv_bfloat16*)xtm1, (const __nv_bfloat16*)xtm2, n,
            kind, p, b->partials, b->ticket, b->rec, local_sum);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_budget_from_sums(const double* sums, int32_t nsums, int64_t n_total,
                                    const BudgetParams& p, pasa_budget_s* b, cudaStream_t st,
                                    int* launches) {
    budget_from_sums_kernel<<<1, 1, 0, st>>>(sums, nsums, n_total, p, b->rec);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace pasa
