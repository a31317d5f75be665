/*
 * pasa.h -- C ABI of libpasa.so, a B200 (sm_100a) implementation of PASA's
 * per-step sparse self-attention: budget -> route -> attn.
 *
 * Paper: "Ride the Wave: Precision-Allocated Sparse Attention for Smooth
 * Video Generation", arXiv 2604.12219 (cited PAPER.md:<line>).  Readings of
 * the paper where it is silent are numbered R-1..R-24 in DESIGN.md §3.
 *
 * Conventions shared by every call
 * --------------------------------
 *  - Every tensor pointer is a DEVICE pointer unless the argument says HOST.
 *    The caller owns all memory, including the device workspaces (allocate
 *    them with torch.empty / cudaMalloc); the library never allocates or
 *    frees device memory, so every launching call can be captured in a CUDA
 *    graph.  Handles are small host structs that point into a workspace.
 *  - Launching calls are asynchronous on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream).  They validate on the host first
 *    and launch nothing when validation fails.  Device faults surface at the
 *    caller's next synchronisation (CUDA semantics).
 *  - Return value: PASA_OK or an error status; pasa_last_error() returns a
 *    thread-local message describing the last failure on this thread.
 *  - Non-finite inputs are not checked on the hot path (the result is
 *    undefined).
 *  - A handle must not be used concurrently on two streams.
 */
#ifndef PASA_H
#define PASA_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PASA_OK = 0,
    PASA_EINVAL = 1,        /* bad scalar argument (beta < 0, h = 0, step outside [0,T), ...) */
    PASA_ESHAPE = 2,        /* shape / stride mismatch between tensors or with the handle      */
    PASA_EDTYPE = 3,        /* dtype mismatch                                                    */
    PASA_EUNSUPPORTED = 4,  /* D not in {64,128}, Bq not in {64,128,256}, Bk != 64, ...          */
    PASA_EDEGENERATE = 5,   /* l-bar <= 0 (Eq. 10 cannot normalise)                 */
    PASA_ECUDA = 6,         /* a CUDA launch or driver call failed                               */
    PASA_ENOSPACE = 7       /* workspace smaller than the *_workspace_bytes() requirement        */
} pasa_status;

typedef enum { PASA_BF16 = 0, PASA_F32 = 1 } pasa_dtype;

/* A [B, S, H, D] activation.  Strides are in ELEMENTS; D is contiguous (stride 1).
 * The default DiT projection output is BSHD contiguous: sB = S*H*D, sS = H*D,
 * sH = D.  data must be 16-byte aligned and sS, sH, sB multiples of 8 elements
 * (TMA requirement).  (X in R^{B x N x S x D}; any stride order.) */
typedef struct {
    void* data;
    int32_t dtype;          /* pasa_dtype */
    int32_t _pad;
    int64_t B, S, H, D;
    int64_t sB, sS, sH;
} pasa_tensor;

/* A contiguous latent (or velocity) tensor of numel elements, fp32 or bf16. */
typedef struct {
    const void* data;
    int32_t dtype;          /* pasa_dtype */
    int32_t _pad;
    int64_t numel;
} pasa_latent;

typedef enum { PASA_IN_LATENT = 0, PASA_IN_VELOCITY = 1 } pasa_budget_input;

/* Budget schedule (Eqs. 9-11). */
typedef struct {
    int32_t T;               /* total denoising steps (50)                                     */
    int32_t step;            /* current step t, 0-based, in [0, T)                             */
    double rho;              /* baseline density rho (0.15 = "85% sparsity")     */
    double dense_frac;       /* dense prefix fraction (0.20)                     */
    double l1_mean;          /* l-bar of Eq. 9 from calibration; must be > 0                   */
    double h_t, h_tm1;       /* sigma_t - sigma_{t-1}, sigma_{t-1} - sigma_{t-2}; != 0 (R-16)   */
    double rho_max;          /* clip for rho_t (1.0, R-18)                                     */
    const double* rho_table; /* HOST, optional per-step rho_t (offline Eqs. 9-11), or NULL; when
                                set it MUST hold at least T entries (only [step] is read)  */
    int32_t kind;            /* pasa_budget_input                                              */
    int32_t _pad;
} pasa_schedule;

typedef enum { PASA_COMP_GROUPED = 0, PASA_COMP_ZEROTH = 1, PASA_COMP_NONE = 2 } pasa_comp;

/* Eq. 8 heterogeneity prior in the routing score (reading R-9,
 * SURVEY.md §8f NEXT 1): r_ij += log(||H_j - C||_F + eps) with C the global mean
 * Hbar of Eq. 6 (GLOBAL, Eq. 8 literally) or the group mean Hbar^(g(j)) of
 * App. B (GROUP).  Needs V at route time: use pasa_route_v. */
typedef enum { PASA_PRIOR_NONE = 0, PASA_PRIOR_GLOBAL = 1, PASA_PRIOR_GROUP = 2 } pasa_prior;

/* Routing / attention configuration (fixed per route handle). */
typedef struct {
    int32_t Bq;              /* query block: 64, 128 or 256 (reading R-7; 256: bf16 tensor-core 
                              * attention only)                          */
    int32_t Bk;              /* key block: 64                                                  */
    int32_t G;               /* blocks per group, >= 1 (32 default); G >= N_K = PISA global */
    int32_t comp;            /* pasa_comp                                                      */
    double beta;             /* bias scale >= 0 (0.1 default; 0 = deterministic top-k, R-10)   */
    int64_t H_total;         /* global head count; Philox is keyed on the global head          */
    int64_t head_offset;     /* this call's buffers hold global heads [off, off + H)           */
    int32_t prior;           /* pasa_prior (PASA_PRIOR_NONE = the north star's route)          */
    int32_t _pad;
    double eps;              /* epsilon of the prior's log (1e-6); > 0 if prior on */
    int32_t qb_begin;        /* this handle routes and attends only the work items               */
    int32_t qb_end;          /* [qb_begin, qb_end) of its B*H*N_Q (head, query block) items,
                              * item = (b*H + h)*N_Q + i (head-major); (0, 0) = all.  The
                              * flattened (head, q-block) partition of SURVEY.md §8e for head
                              * counts that do not divide the GPU count: one handle (one launch
                              * per kernel) per rank; K/V statistics still cover whole heads,
                              * Philox keys on the global head and block, and rows outside the
                              * range of idx / count / mask / out are not written.            */
    int32_t qk_fp8;          /* 1 = opt-in precision variant (reading R-30):
                              * QK^T of kept blocks and the centroid logits run on the FP8 tensor
                              * cores (E4M3 x E4M3 -> f32).  pasa_route also writes E4M3 copies of
                              * Q (one scale per token row) and K (one per 64-token block), the
                              * statistics pass an E4M3 Kbar (one scale per head); PV and the
                              * first-order term stay bf16.  bf16 I/O, D = 128, Bq = 128, G >= 32
                              * only (else EUNSUPPORTED).  Its own tolerance: 1e-1 max|O| (the
                              * E4M3 rounding alone gives ~5e-2); never the
                              * north-star configuration.  0 = bf16 everywhere (default).     */
    int32_t _pad2;
} pasa_route_cfg;

typedef struct pasa_budget_s* pasa_budget_h;
typedef struct pasa_route_s* pasa_route_h;

/* ---- workspaces and handles --------------------------------------------- */
/* Budget workspace: the device record {l1, alpha, rho_t, dense, clipped} plus
 * fixed-size fp64 partials of the reduction (a fixed grid, so l1 is
 * bit-reproducible run to run). */
size_t pasa_budget_workspace_bytes(void);
/* Route workspace for tensors of shape [B, S, H, D]: pooled Qbar/Kbar (fp64),
 * the low-precision Kbar / Vsum / grouped Hbar used by pasa_attn, the index
 * list idx [B*H][N_Q][N_K] int32 (first count entries valid), count
 * [B*H][N_Q] int32 and mask [B*H][N_Q][ceil(N_K/32)] u32; with the Eq. 8 prior
 * enabled also every block's fp64 H_j (8 D^2 bytes per block and head: 6.2 GB
 * for a Wan-14B layer of 40 heads).  Returns 0 if the configuration is invalid
 * (see pasa_last_error()). */
size_t pasa_route_workspace_bytes(const pasa_route_cfg* cfg, int64_t B, int64_t S, int64_t H,
                                  int64_t D);
/* Bind a handle to caller-owned device workspace `dev_ws` of `bytes` bytes.
 * The handle itself is a host allocation released by *_fini (which never
 * touches the workspace). */
pasa_status pasa_budget_init(void* dev_ws, size_t bytes, pasa_budget_h* out);
pasa_status pasa_route_init(void* dev_ws, size_t bytes, const pasa_route_cfg* cfg, int64_t B,
                            int64_t S, int64_t H, int64_t D, pasa_route_h* out);
void pasa_budget_fini(pasa_budget_h h);
void pasa_route_fini(pasa_route_h h);

/* ---- the three calls of the hot path --------------------------------------
 * pasa_budget -- PAPER.md:269-294, readings R-15..R-18:
 *   l = mean_e |(x_t - x_{t-1})/h_t - (x_{t-1} - x_{t-2})/h_{t-1}|   (LATENT)
 *   l = mean_e |x_t - x_{t-1}|                                      (VELOCITY;
 *        x_tm2 may be NULL)
 *   alpha = l / l1_mean (Eq. 10); rho_t = 1 in the dense prefix
 *   (t < round(dense_frac*T) or t < 2), else min(rho*alpha or rho_table[t],
 *   rho_max) (Eq. 11).  The record stays on the device; nothing syncs.
 *   Latents: same numel and dtype, fp32 or bf16, contiguous.
 *   Errors: EINVAL (T<1, step, h==0, NULL data), ESHAPE, EDTYPE,
 *   EDEGENERATE (l1_mean <= 0). */
pasa_status pasa_budget(const pasa_latent* x_t, const pasa_latent* x_tm1, const pasa_latent* x_tm2,
                        const pasa_schedule* schedule, pasa_budget_h budget, void* stream);

/* Sharded latents ("all_gather of one fp64 partial per rank, summed
 * in rank order"), for callers whose latents are split across ranks (sequence-
 * sharded DiT inference).  Two steps around the caller's all_gather:
 *   pasa_budget_local_sum: dev_sum[0] (DEVICE fp64) = sum over THIS rank's elements of
 *     |dv| (the numerator of pasa_budget's l; same element formula, fixed-order tree);
 *   pasa_budget_from_sums: l = (sums[0] + sums[1] + ... + sums[n-1], in that order) /
 *     n_total, then alpha, rho_t exactly as pasa_budget.  dev_sums: DEVICE, nsums fp64
 *     (the gathered per-rank sums, rank order); n_total: the element count of the full
 *     latent.
 * Errors: as pasa_budget; EINVAL for nsums < 1 or n_total < 1. */
pasa_status pasa_budget_local_sum(const pasa_latent* x_t, const pasa_latent* x_tm1,
                                  const pasa_latent* x_tm2, const pasa_schedule* schedule,
                                  pasa_budget_h budget, double* dev_sum, void* stream);
pasa_status pasa_budget_from_sums(const double* dev_sums, int32_t nsums, int64_t n_total,
                                  const pasa_schedule* schedule, pasa_budget_h budget,
                                  void* stream);

/* pasa_route -- PAPER.md:189-193 (block partition, top-k per query block),
 * Eq. 8 pooled-logit term, stochastic bias
 * (PAPER.md:296-308), readings R-6..R-14, R-20:
 *   Qbar_i, Kbar_j = fp64 block means in ascending token order;
 *   r_ij = s * dot(Qbar_i, Kbar_j) (fp64 fma chain), s = 1/sqrt(D);
 *   rt_ij = r_ij + (beta*sigma_i) * Gumbel(Philox4x32-10(ctr=(j,i,gh,step),
 *           key=seed)), sigma_i the population std of row i;
 *   k = clamp(floor(rho_t*N_K + 0.5), 1, N_K) computed ON THE DEVICE from the
 *   budget record; S_i = top-k of rt under (rt desc, j asc), stored ascending.
 *   q, k: [B,S,H,D], same dtype (bf16 or fp32) and shape as the handle.
 *   gh = b*H_total + head_offset + h.  `seed` is the per-layer key
 *   (pasa_layer_seed(seed, layer)); reusing one seed across layers repeats the
 *   bias and violates PAPER.md:308.
 *   Errors: ESHAPE, EDTYPE, EINVAL (NULL handle). */
pasa_status pasa_route(const pasa_tensor* q, const pasa_tensor* k, pasa_budget_h budget,
                       uint64_t seed, int32_t step, pasa_route_h route, void* stream);

/* pasa_route with Eq. 8's heterogeneity prior (cfg.prior !=
 * PASA_PRIOR_NONE): as pasa_route, but before scoring computes per KV block
 *   H_j = sum_n (K_n - Kbar_j)^T V_n (Eq. 5), het_j = ||H_j - C||_F,
 * in fp64, and scores r_ij = s * dot(Qbar_i, Kbar_j) + log(het_j + eps); sigma_i
 * and the bias then follow as in pasa_route.  v: [B,S,H,D] like k.  The workspace
 * of a prior-enabled handle also holds het, the prior and the fp64 group sums
 * (pasa_route_workspace_bytes accounts for them).  Errors: as pasa_route, plus
 * EINVAL if the handle's cfg.prior is NONE.  pasa_route on a prior-enabled
 * handle returns EINVAL (it has no V). */
pasa_status pasa_route_v(const pasa_tensor* q, const pasa_tensor* k, const pasa_tensor* v,
                         pasa_budget_h budget, uint64_t seed, int32_t step, pasa_route_h route,
                         void* stream);

/* pasa_attn -- Eq. 7 with grouped first-order
 * compensation (App. B :494-506), readings R-1..R-5, R-21,
 * R-22:
 *   for each query row t of block i, with S_i from the route and U_i its
 *   complement,
 *   O_t = [ sum_{u in S_i} e^{s q.K_u - m} V_u + sum_{j in U_i} e^{s q.Kbar_j - m} Vsum_j
 *           + sum_g A_{t,g} s q_t Hbar^(g) ]
 *       / [ sum_{u in S_i} e^{s q.K_u - m} + sum_{j in U_i} n_j e^{s q.Kbar_j - m} ],
 *   A_{t,g} = sum_{j in U_i cap G_g} e^{s q.Kbar_j - m}; comp ZEROTH drops the
 *   Hbar term, NONE drops every U term.  q and k must be the buffers the route
 *   was built from; v and out have the same B,S,H,D (out may have its own
 *   strides).  bf16 I/O with Bq = 128 and G in {8, 16, 32, 64, multiples of 128,
 *   >= N_K} runs the tcgen05/TMEM/TMA kernel (fp32 accumulate; Kbar, Vsum, Hbar
 *   stored bf16, R-21); Bq = 256 (R-29) runs the two-tile tcgen05 kernel, or the
 *   cta_group::2 CTA-pair kernel with PASA_ATTN_CTA_PAIR (bf16,
 *   G in {32, 64, multiples of 128, >= N_K}; anything else at Bq = 256 is
 *   EUNSUPPORTED); fp32 I/O, Bq = 64 or other group sizes run the fp32 CUDA-core
 *   kernel.
 *   Errors: ESHAPE, EDTYPE, EINVAL (route never built). */
pasa_status pasa_attn(const pasa_tensor* q, const pasa_tensor* k, const pasa_tensor* v,
                      pasa_route_h route, pasa_tensor* out, void* stream);

/* pasa_attn with flags:
 *   PASA_ATTN_FORCE_SIMT   run the CUDA-core kernel even for bf16 I/O (cross-check);
 *   PASA_ATTN_STATS_ONLY   launch only the K/V statistics pass (Kbar, Vsum, Hbar^(g));
 *   PASA_ATTN_REUSE_STATS  skip the statistics pass: the caller guarantees that the
 *                          previous STATS_ONLY call on this route saw the same k, v.
 *   PASA_ATTN_CTA_PAIR     Bq = 256 routes only: run the CTA-pair kernel (tcgen05
 *                          cta_group::2, M = 256 over the two SMs of a TPC, each SM
 *                          holding half of every K/V / statistics tile; SURVEY.md §8f
 *                          NEXT 4) instead of the one-CTA two-tile kernel.  Same
 *                          results up to fp32 summation order; d = 128 only, G as
 *                          for Bq = 256; anything else returns EUNSUPPORTED.
 * STATS_ONLY followed by REUSE_STATS is exactly pasa_attn, split so that each
 * kernel can be timed on its own stream position. */
#define PASA_ATTN_FORCE_SIMT 1u
#define PASA_ATTN_STATS_ONLY 2u
#define PASA_ATTN_REUSE_STATS 4u
#define PASA_ATTN_CTA_PAIR 8u
pasa_status pasa_attn_ex(const pasa_tensor* q, const pasa_tensor* k, const pasa_tensor* v,
                         pasa_route_h route, pasa_tensor* out, uint32_t flags, void* stream);

/* Zero-copy sequence parallelism: the Ulysses all-to-all fused into PASA's kernels over
 * peer memory (PAPER.md:321 runs PASA on 8 GPUs).  When the
 * model's activations arrive sequence-sharded (rank r holds tokens [start[r],
 * start[r+1]) of every head), the rank that owns heads [h0, h0 + Hl) reads those heads of
 * every shard directly through peer pointers (NVLink P2P / CUDA IPC mappings the caller
 * set up), and writes each output row straight into the shard of the rank that owns its
 * token: no all-to-all is issued.
 *
 * pasa_shards: one bf16 tensor [1, S, H, D] as P (1..8) sequence shards.  data[s] is the
 * address (valid in this process, device-accessible) of shard s's first token, head 0;
 * sS / sH are element strides (the same in every shard, 16-byte aligned, unit stride in D);
 * start[0] = 0 < start[1] < ... < start[P] = S.  Shard boundaries need not align to blocks. */
typedef struct {
    int32_t dtype;          /* PASA_BF16 */
    int32_t nshards;        /* P */
    int64_t S, H, D;
    int64_t sS, sH;
    int64_t start[9];
    void* data[8];
} pasa_shards;

/* pasa_route for the heads [cfg.head_offset, cfg.head_offset + H) of a route handle created
 * for [1, S, H (this rank's heads), D] with cfg.H_total = the shards' H: one kernel gathers
 * q, k and v of those heads from every shard into the caller's LOCAL buffers q_loc, k_loc,
 * v_loc ([1, S, H, D] bf16, DEVICE, written) and pools q and k in the same pass (the same
 * ascending-token fp64 block sums as pasa_route, so the route is bitwise the single-GPU
 * route of those heads); then the fused score / bias / top-k kernel.  Call pasa_attn_zc
 * next (on the same stream).  The caller guarantees every shard is complete before the
 * call (e.g. a stream synchronise + process-group barrier on all ranks).
 * Errors: EINVAL (NULL, nshards, start, head range), ESHAPE (S, D, local buffers), EDTYPE
 * (not bf16), EUNSUPPORTED (prior-enabled or FP8 handles). */
pasa_status pasa_route_zc(const pasa_shards* q, const pasa_shards* k, const pasa_shards* v,
                          pasa_budget_h budget, uint64_t seed, int32_t step, pasa_route_h route,
                          const pasa_tensor* q_loc, const pasa_tensor* k_loc,
                          const pasa_tensor* v_loc, void* stream);

/* pasa_attn over the local buffers pasa_route_zc filled, with the output rows of this
 * rank's heads stored straight into `out`'s shards (row t of head h -> shard s with
 * start[s] <= t < start[s+1], head cfg.head_offset + h).  bf16, the tensor-core kernel's
 * domain (Bq = 128, G in {8, 16, 32, 64, multiples of 128, >= N_K}); the caller
 * synchronises all ranks before reading its output shard.  Errors: as pasa_attn, plus
 * EINVAL / ESHAPE for `out`, EUNSUPPORTED outside the tensor-core domain. */
pasa_status pasa_attn_zc(const pasa_tensor* q_loc, const pasa_tensor* k_loc,
                         const pasa_tensor* v_loc, pasa_route_h route, const pasa_shards* out,
                         void* stream);

/* Offline calibration of the budget table, Eqs. 9-11 verbatim (
 * readings R-15, R-17..R-19).  HOST pointers; no GPU work.
 *   l1_curves [N][T]: l_t of N calibration trajectories (e.g. pasa_budget's l1
 *     of each step, or mean |v_t - v_{t-1}| of dumped noise_pred); entries of
 *     dense steps are ignored and may be NaN.
 *   lavg_t = (sum_n l1_curves[n][t]) / N (pointwise mean, R-19);
 *   T_sparse = { t >= max(floor(dense_frac*T + 0.5), 2) } (R-15);
 *   l1_mean = mean of lavg over T_sparse (Eq. 9); alpha_t = lavg_t / l1_mean
 *   (Eq. 10); rho_table[t] = min(rho*alpha_t, rho_max), clipped[t] = 1 if the
 *   clip applied (Eq. 11, R-18); dense steps: rho_table = 1, alpha = 0.
 * Outputs rho_table[T], alpha[T], clipped[T] (int32 0/1), *l1_mean; any of
 * alpha / clipped may be NULL.  Errors: EINVAL (N < 1, T < 1, no sparse step,
 * rho < 0, rho_max <= 0, non-finite sparse entry), EDEGENERATE (l1_mean <= 0,
 * SPEC.md:403). */
pasa_status pasa_calibrate(const double* l1_curves, int32_t N, int32_t T, double rho,
                           double dense_frac, double rho_max, double* rho_table, double* alpha,
                           int32_t* clipped, double* l1_mean);

/* Host <-> device 2-D copy on `stream` (runtime plumbing for callers that keep
 * q, k, v or the output in HOST memory): `height` rows of `width` bytes, row
 * pitches `spitch` / `dpitch` bytes, e.g. a contiguous run of heads of a
 * [B, S, H, D] tensor (rows = B*S).  kind: 1 = host to device, 2 = device to
 * host.  Pinned host memory makes the copy asynchronous.  Errors: EINVAL (NULL
 * pointer, width > pitch, bad kind), ECUDA. */
pasa_status pasa_copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                        size_t height, int32_t kind, void* stream);

/* SplitMix64 finaliser of seed + (layer+1)*0x9E3779B97F4A7C15 (reading R-11):
 * one independent Philox key per layer. */
uint64_t pasa_layer_seed(uint64_t seed, int32_t layer);

/* ---- synchronous diagnostics (tests) ------------------------------------- */
/* out (HOST) = {l1, alpha, rho_t, dense, clipped}. Synchronises `stream`. */
pasa_status pasa_budget_read(pasa_budget_h budget, double out[5], void* stream);
/* HOST outputs, each may be NULL: k (1 int), idx [B*H][N_Q][N_K], count
 * [B*H][N_Q], mask [B*H][N_Q][ceil(N_K/32)].  Synchronises `stream`. */
pasa_status pasa_route_read(pasa_route_h route, int32_t* k, int32_t* idx, int32_t* count,
                            uint32_t* mask, void* stream);
/* HOST outputs (may be NULL): qbar [B*H][N_Q][D], kbar [B*H][N_K][D] fp64. */
pasa_status pasa_route_pooled_read(pasa_route_h route, double* qbar, double* kbar, void* stream);
/* HOST outputs (may be NULL) of the last pasa_attn statistics pass, in the I/O dtype
 * (bf16 or fp32): kbar [B*H][N_K][D], vsum [B*H][N_K][D], ht [B*H][N_G][D][D]
 * (ht[.][g][n][k] = Hbar^(g)[k][n]).  `dtype` declares the element type the caller
 * sized its buffers for; it must equal the dtype of that pass (the q/k/v dtype of the
 * last pasa_attn), else EDTYPE and nothing is written.  Synchronises `stream`. */
pasa_status pasa_attn_stats_read(pasa_route_h route, void* kbar, void* vsum, void* ht,
                                 int32_t dtype, void* stream);
/* Geometry of a handle: dims[0..6] = {B, S, H, D, N_Q, N_K, N_G}. */
pasa_status pasa_route_dims(pasa_route_h route, int64_t dims[7]);
/* Synchronous: het [B*H][N_K] fp64 = ||H_j - C||_F of the last pasa_route_v
 * (HOST buffer).  EINVAL if the handle has no prior or it was never computed. */
pasa_status pasa_route_het_read(pasa_route_h route, double* het, void* stream);
/* Diagnostics: make the next tensor-core attention launches record a clock64()
 * timeline of CTA (x, y) into dev_buf (DEVICE, 17 x 4096 uint64: producer, MMA
 * and softmax events per op); NULL disables.  Returns the element count. */
int pasa_debug_trace(void* dev_buf, int x, int y);
/* Diagnostics: performance ablations of the tensor-core attention kernel (1 = the
 * softmax warps skip their arithmetic, 2 = the producers skip the TMA loads).
 * Results are meaningless while set; 0 restores normal operation.  Returns the
 * previous flags. */
int pasa_debug_flags(int flags);
/* Number of kernel launches the last pasa_budget / pasa_route / pasa_attn
 * call on this thread issued (bench accounting). */
int32_t pasa_last_launch_count(void);
const char* pasa_last_error(void);
const char* pasa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PASA_H */
