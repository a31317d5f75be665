// pasa_internal.h -- host-side handle layout and kernel launchers of libpasa.so.
// Product code: nothing here includes or calls anything under oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pasa.h"

namespace pasa {

constexpr int kBudgetParts = 1024;   // fixed reduction grid: l1 is bit-reproducible
constexpr int kNGMaxTC = 4096;       // no hard limit for the tcgen05 path (groups stream)

struct BudgetRec {                    // device record, 64 bytes
    double l1, alpha, rho_t, dense, clipped, pad0, pad1, pad2;
};

struct BudgetParams {                 // host-derived scalars of one budget call
    double rht, rh1;                  // 1 / h_t, 1 / h_{t-1}
    int32_t step, dense_steps;
    double rho, l1_mean, rho_max;
    int32_t use_table;
    double table_val;
};

}  // namespace pasa

struct pasa_budget_s {
    pasa::BudgetRec* rec;            // device
    double* partials;                // device [kBudgetParts]
    unsigned int* ticket;            // device: CTAs of the running reduction that finished
    int ticket_ready;                // host: the ticket has been zeroed on a stream
};

struct pasa_route_s {
    pasa_route_cfg cfg;
    int64_t B, S, H, D, NQ, NK, NG, W, BH;
    int64_t it0, it1;                // (head, q-block) items routed / attended: [it0, it1),
                                     // item = bh * NQ + i
    int32_t* hdr;                    // device: [0] = k of the last pasa_route
    double* qbar;                    // [BH][NQ][D]
    double* kbar;                    // [BH][NK][D]
    double* kfrag;                   // Kbar in DMMA B-fragment order [BH][ceil(NK/8)][D/8][64]
    double* scores;                  // [BH][NQ][NKP] fp64 score rows, only when they do not
                                     // fit in shared memory (route_rows_per_cta == 0), else null
    void* kbar_lp;                   // [BH][NK][D]   bf16 or fp32 (4 B/elem capacity)
    void* vsum_lp;                   // [BH][NK][D]
    void* ht;                        // [BH][NG][D][D] Hbar^T per group (row n, col k)
    float* part;                     // [BH][ceil(NK/32)][D][D] fp32 chunk sums (G > 64)
    int32_t* idx;                    // [BH][NQ][idx_ld] (first count entries valid, ascending)
    int64_t idx_ld;                  // row stride of idx (entries)
    int32_t* count;                  // [BH][NQ]
    uint32_t* mask;                  // [BH][NQ][W]
    // FP8 QK^T variant (cfg.qk_fp8) only, else null: E4M3 copies and their scales
    uint8_t* q8;                     // [BH][S][D] E4M3 Q (pool_kernel), row t scaled by 1/sq8[t]
    float* sq8;                      // [BH][S] per-row Q scales (row amax / 448)
    uint8_t* k8;                     // [BH][S][D] E4M3 K (statistics pass), scale kamax / 448
    uint8_t* kb8;                    // [BH][NK][D] E4M3 Kbar (statistics pass), scale kbamax / 448
    uint32_t* kamax;                 // [BH] max |K| per head (float bits, pool_kernel), and
    uint32_t* kbamax;                // [BH] max |Kbar| per head right after it
    double* het;                     // [BH][NK] ||H_j - C||_F (prior-enabled handles only)
    double* prior;                   // [BH][NK] log(het + eps)
    double* hj;                      // [BH][NK][D][D] fp64 H_j of every block (prior handles)
    double* hgs;                     // [BH][NG][D][D] fp64 group means of H_j
    double* hglob;                   // [BH][D][D] fp64 global mean Hbar
    int32_t het_valid;               // a pasa_route_v has filled het
    int32_t route_dtype;             // dtype of the q/k the route was last built from (-1 = none)
    int32_t stats_dtype;             // dtype of the last kv_stats pass (-1 = none)
};

namespace pasa {

// Zero-copy sequence parallelism (pasa_route_zc / pasa_attn_zc): a [1, S, H, D] bf16 tensor
// held as P sequence shards, each addressable from this process (peer / IPC mapped);
// shard s holds tokens [start[s], start[s+1]) at base[s] (its first token, head 0) with
// element strides sS (token) and sH (head)
struct ZcShards {
    int32_t P;
    int64_t start[9];
    const void* base[8];
    int64_t sS, sH;
};
cudaError_t launch_route_zc(const ZcShards* qkv, const pasa_tensor* loc, const pasa_budget_s* b,
                            uint64_t seed, int32_t step, pasa_route_s* r, cudaStream_t st,
                            int* launches);

// ---- launchers (each returns cudaGetLastError() after its launches) -------
// local_sum != nullptr: store the fp64 sum of |dv| there instead of finishing the record
cudaError_t launch_budget(const void* xt, const void* xtm1, const void* xtm2, int64_t n, int dtype,
                          int kind, const BudgetParams& p, pasa_budget_s* b, double* local_sum,
                          cudaStream_t st, int* launches);
cudaError_t launch_budget_from_sums(const double* sums, int32_t nsums, int64_t n_total,
                                    const BudgetParams& p, pasa_budget_s* b, cudaStream_t st,
                                    int* launches);

// v != nullptr: Eq. 8 prior (het.cu) between pooling and scoring
cudaError_t launch_route(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor* v,
                         const pasa_budget_s* b, uint64_t seed, int32_t step, pasa_route_s* r,
                         cudaStream_t st, int* launches);
// fused scores / sigma / top-k kernel: rows of scores per CTA held in shared memory
// (0: they do not fit and live in the workspace's global scratch) and the odd row
// stride of a score row
int route_rows_per_cta(int64_t NK, int64_t D);
int64_t route_score_stride(int64_t NK);
cudaError_t launch_het(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r,
                       cudaStream_t st, int* launches);
// KV blocks per work chunk of the prior kernels (a divisor of G, <= 32)
int64_t het_chunk_blocks(int64_t G, int64_t NK);

cudaError_t launch_kv_stats(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r,
                            cudaStream_t st, int* launches);
// tensor-core statistics pass (bf16, d = 128 or 64); launch_kv_stats dispatches to it
bool kv_stats_sm100_supported(const pasa_route_s* r);
cudaError_t launch_kv_stats_sm100(const pasa_tensor& k, const pasa_tensor& v, pasa_route_s* r,
                                  cudaStream_t st, int* launches);

cudaError_t launch_attn_simt(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                             pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                             int* launches);

// group sizes the tensor-core kernel's group-sum bookkeeping covers: 8 and 16 (per-8-column
// sums of each 64-block chunk kept in shared memory), or every 32-block mask word inside
// one group with at most two groups per 64-block chunk
inline bool sm100_supports_group(int64_t G, int64_t NK) {
    return G == 8 || G == 16 || G == 32 || G == 64 || G % 128 == 0 || G >= NK;
}

// returns cudaErrorNotSupported if the configuration is outside the kernel's domain
cudaError_t launch_attn_sm100(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                              pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                              int* launches, char* why, size_t why_len,
                              const ZcShards* out_shards = nullptr);
// Bq = 256: one CTA per SM, two 128-row tiles sharing every
// operand tile the op brings from L2; attn_sm100_q256.cu
bool attn_sm100_q256_supported(const pasa_route_s* r);
cudaError_t launch_attn_sm100_q256(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                                   pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                                   int* launches, char* why, size_t why_len);
// Bq = 256 on a CTA pair (tcgen05 cta_group::2, M = 256; each SM holds half of every
// operand tile); attn_sm100_cta2.cu, selected with PASA_ATTN_CTA_PAIR
bool attn_sm100_cta2_supported(const pasa_route_s* r);
cudaError_t launch_attn_sm100_cta2(const pasa_tensor& q, const pasa_tensor& k, const pasa_tensor& v,
                                   pasa_route_s* r, const pasa_tensor& out, cudaStream_t st,
                                   int* launches, char* why, size_t why_len);
// tmap.cpp: TMA tensor-map encoding (bf16, 128-byte swizzle, zero OOB fill) and the
// diagnostics state set by pasa_debug_trace / pasa_debug_flags
bool make_tensor_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                     const uint64_t* strides_bytes, const uint32_t* box, char* why,
                     size_t why_len, bool u8 = false);
extern unsigned long long* g_trace_buf;
extern int g_trace_x, g_trace_y, g_dbg;

}  // namespace pasa
