/*
 * pasa_oracle.h -- fp64 CPU ORACLE for PASA per-step sparse self-attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * The product path (libpasa.so, paper_2604_12219_b200/) never includes,
 * links or calls anything in this directory, and this directory never
 * includes anything from the product path.
 *
 * Paper: "Ride the Wave: Precision-Allocated Sparse Attention for Smooth
 * Video Generation" (arXiv 2604.12219), cited as PAPER.md:<line>.  The
 * readings taken where the paper is silent are listed in DESIGN.md §3
 * (R-1 ... R-24) and cited here by id.
 *
 * Tensor convention for every attention-side function: one array per
 * tensor, fp64, layout [BH][S][D] contiguous (the per-head [S, d] slices of
 * the caller's [B, S, H, D] tensor, bh = b*H + h).  Block j of a head holds
 * tokens [j*Bk, min((j+1)*Bk, S)); its true length n_j may be < Bk for the
 * last block (reading R-7: no padding inside the softmax).
 */
#ifndef PASA_ORACLE_H
#define PASA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- counter-based RNG (reading R-11/R-12) ---------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11).  out = Philox(ctr, key). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* SplitMix64 finaliser of (seed + (layer+1) * 0x9E3779B97F4A7C15). */
uint64_t orc_layer_seed(uint64_t seed, int32_t layer);
/* Standard Gumbel draw for route entry (i, j) of global head gh at step. */
double orc_gumbel(uint64_t seed, int32_t step, int64_t gh, int64_t i, int64_t j);

/* ---- budget: Eqs. 9-11, PAPER.md:276-294 (readings R-15..R-18) --------- */
/* kind: 0 = three latents (x_t, x_t-1, x_t-2), 1 = velocities (x_t, x_t-1).
 * out[5] = { l1, alpha, rho_t, dense (0/1), clipped (0/1) }.
 * returns 0 on success, -1 on invalid input (T<1, step outside [0,T),
 * h == 0, l1_mean <= 0). */
int orc_budget(const double* x_t, const double* x_tm1, const double* x_tm2,
               int64_t n, int kind, double h_t, double h_tm1,
               int32_t T, int32_t step, double rho, double dense_frac,
               double l1_mean, double rho_max, const double* rho_table,
               double out[5]);
/* Mean L1 signal l_t alone (step B1 of DESIGN.md §3). */
double orc_l1(const double* x_t, const double* x_tm1, const double* x_tm2,
              int64_t n, int kind, double h_t, double h_tm1);
/* Offline calibration, Eqs. 9-11 verbatim (readings R-15,
 * R-17..R-19).  curves [N][T]: l_t of N trajectories
 * (entries of dense steps are ignored and may be NaN).
 *   lavg_t = (sum_n curves[n][t]) / N                  (pointwise mean, R-19)
 *   T_sparse = { t : t >= floor(dense_frac*T + 0.5) and t >= 2 }     (R-15)
 *   lbar = (sum_{t in T_sparse} lavg_t) / |T_sparse|    (Eq. 9)
 *   alpha_t = lavg_t / lbar                             (Eq. 10)
 *   rho_t = min(rho * alpha_t, rho_max), clipped_t = rho*alpha_t > rho_max (Eq. 11, R-18)
 *   dense steps: rho_t = 1, alpha_t = 0, clipped_t = 0.
 * Outputs rho_table[T], alpha[T], clipped[T] (0/1), *lbar.  Returns 0, or -1
 * on invalid input (N < 1, T < 1, empty T_sparse, lbar <= 0 or not finite). */
int orc_calibrate(const double* curves, int32_t N, int32_t T, double rho, double dense_frac,
                  double rho_max, double* rho_table, double* alpha, int32_t* clipped,
                  double* lbar);
/* k = clamp(floor(rho_t * n_blocks + 0.5), 1, n_blocks)   (reading R-14) */
int64_t orc_density_to_k(double rho_t, int64_t n_blocks);

/* ---- routing: Eq. 8, :296-308 ------ */
/* Per head bh (gh = b*H_total + head_offset + h with b = bh / H, h = bh % H):
 *   Qbar_i, Kbar_j       block means, sequential token order   (R1, R-6)
 *   r_ij = s * fma-chain dot(Qbar_i, Kbar_j), s = 1/sqrt(D)   (Eq. 8, R-8, R-9)
 *   sigma_i population std of row i                           (R-10)
 *   rt_ij = r_ij + (beta*sigma_i) * gumbel(seed, step, gh, i, j)  (R-10..R-12)
 *   S_i = top-kk of rt under (rt desc, j asc), emitted ascending  (R-13, R-14)
 * Outputs: idx [BH][N_Q][kk] int32, mask [BH][N_Q][ceil(N_K/32)] u32
 * (bit j%32 of word j/32 set iff j in S_i); scores (optional, may be NULL)
 * [BH][N_Q][N_K] = rt. */
void orc_route(const double* q, const double* k, int64_t B, int64_t H, int64_t S, int64_t D,
               int32_t Bq, int32_t Bk, double beta, uint64_t seed, int32_t step,
               int64_t H_total, int64_t head_offset, int64_t kk,
               int32_t* idx, uint32_t* mask, double* scores,
               const double* het, double eps);
/* het (optional, may be NULL): [BH][N_K] heterogeneity norms ||H_j - C||_F of
 * Eq. 8's prior (orc_heterogeneity); then r_ij = s * dot + log(het_j + eps)
 * (the softmax of Eq. 8 is rank preserving and dropped, R-8),
 * and sigma_i is taken over these r_ij. */

/* ---- Eq. 8 heterogeneity prior ---------
 * For one head: het[j] = ||H_j - C||_F (Frobenius), H_j of Eq. 5,
 * C = the global mean Hbar of Eq. 6 (mode 1, Eq. 8 literally) or the group
 * mean Hbar^(g(j)) of App. B (mode 2).  The squared entries are summed row by
 * row in ascending (a, b) order, then sqrt.  Memory: N_K*D*D doubles. */
void orc_heterogeneity(const double* k, const double* v, int64_t S, int64_t D, int32_t Bk,
                       int32_t G, int32_t mode, double* het);
/* Block means (used by routing and by the statistics). out [N][D]. */
void orc_block_means(const double* x, int64_t S, int64_t D, int32_t Bsz, double* out);

/* ---- block statistics: Eqs. 5-6, App. B (:494-497) ---- */
/* For one head: Kbar [N_K][D], Vsum [N_K][D] (Eq. 4's inner sum),
 * Hblk [N_K][D][D] (optional, may be NULL; Eq. 5, H_j[a][b] =
 * sum_n (K_n[a] - Kbar_j[a]) V_n[b]), Hbar [N_G][D][D] (unweighted group mean,
 * groups = contiguous runs of G blocks, last one shorter; R-4, R-5). */
void orc_block_stats(const double* k, const double* v, int64_t S, int64_t D,
                     int32_t Bk, int32_t G, double* Kbar, double* Vsum,
                     double* Hblk, double* Hbar);

/* ---- attention with a given route: Eq. 7 with the grouped
 * first-order surrogate of App. B, readings R-1, R-2, R-3,
 * R-22.  comp: 0 = GROUPED, 1 = ZEROTH, 2 = NONE.  idx [BH][N_Q][kk_stride]
 * with count[BH][N_Q] valid entries per row (ascending, unique).  out
 * [BH][S][D].  Rows are independent; OpenMP over (bh, query block). */
void orc_attn_with_route(const double* q, const double* k, const double* v,
                         int64_t BH, int64_t S, int64_t D, int32_t Bq, int32_t Bk,
                         int32_t G, int32_t comp, const int32_t* idx,
                         const int32_t* count, int64_t kk_stride, double* out);
/* Same, restricted to the listed (bh, q-block) pairs (sampled parity at
 * full size).  pairs[2*p] = bh, pairs[2*p+1] = i.  out [npairs][Bq][D]
 * (rows past S left untouched). */
void orc_attn_pairs(const double* q, const double* k, const double* v,
                    int64_t BH, int64_t S, int64_t D, int32_t Bq, int32_t Bk,
                    int32_t G, int32_t comp, const int32_t* idx,
                    const int32_t* count, int64_t kk_stride,
                    const int64_t* pairs, int64_t npairs, double* out);

int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
