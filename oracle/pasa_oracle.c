/*
 * pasa_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for PASA.
 *
 * TEST INFRASTRUCTURE (see pasa_oracle.h).  Compiled with
 *   gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math
 * so that every floating-point operation below is exactly the IEEE-754
 * double operation it reads as (explicit fma() where the route contract
 * says fma).  No blocking, no fusion: each function follows the paper's
 * formula in the paper's order; summations are sequential in index order,
 * and the attention numerator/denominator use Neumaier-compensated sums.
 *
 * Parity status per function (see DESIGN.md §4 for the pins):
 *   orc_philox4x32_10, orc_layer_seed ......... pinned (library vectors)
 *   orc_budget / orc_l1 / orc_density_to_k .... pinned (worked examples,
 *                                                closed forms)
 *   orc_route ................................. pinned (worked example,
 *                                                brute force, Gumbel-max law)
 *   orc_block_stats ........................... pinned (worked example,
 *                                                invariants, Prop. 1)
 *   orc_attn_with_route / orc_attn_pairs ...... pinned by special cases
 *                                                (dense recovery vs library
 *                                                SDPA, constant keys, Taylor
 *                                                order, invariances); the
 *                                                paper prints no output values.
 */
#include "pasa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10: 10 rounds of the Philox S-box with Weyl key schedule.      */
/* Constants from Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as   */
/* easy as 1, 2, 3" (SC'11), Table 2.                                         */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += W0; k1 += W1; }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* SplitMix64 (Steele, Lea, Flood 2014) output function applied to
 * seed + (layer+1)*golden-gamma: one independent key per layer (R-11,
 * PAPER.md:308 "independently sampled across different layers"). */
uint64_t orc_layer_seed(uint64_t seed, int32_t layer) {
    uint64_t z = seed + (uint64_t)((int64_t)layer + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* R-11/R-12: one Philox4x32-10 call yields four 32-bit words; block j of query block
 * i of global head gh at step `step` takes word w = j mod 4 of counter
 * ctr = (floor(j/4), i, gh, step), key = (lo32(seed), hi32(seed));
 * u = (x_w + 0.5) * 2^-32 in (0,1), g = -ln(-ln u). */
double orc_gumbel(uint64_t seed, int32_t step, int64_t gh, int64_t i, int64_t j) {
    uint32_t ctr[4] = {(uint32_t)(j >> 2), (uint32_t)i, (uint32_t)gh, (uint32_t)step};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t x[4];
    orc_philox4x32_10(ctr, key, x);
    double u = ((double)x[j & 3] + 0.5) * 2.3283064365386963e-10; /* 2^-32 */
    return -log(-log(u));
}

/* ------------------------------------------------------------------------ */
/* Budget.                                                                    */
/* ------------------------------------------------------------------------ */
/* B1: l = (1/n) sum_e |(x_t - x_{t-1})/h_t - (x_{t-1} - x_{t-2})/h_{t-1}|
 * (trajectory acceleration = difference of adjacent velocity fields,
 * PAPER.md:269, :277-278; reading R-16), or for velocity input
 * l = (1/n) sum_e |v_t - v_{t-1}| ("mean L1 distance between predicted
 * velocity fields at adjacent timesteps"). */
double orc_l1(const double* x_t, const double* x_tm1, const double* x_tm2,
              int64_t n, int kind, double h_t, double h_tm1) {
    double acc = 0.0;
    for (int64_t e = 0; e < n; ++e) {
        double dv;
        if (kind == 1) {
            dv = x_t[e] - x_tm1[e];
        } else {
            double a = x_t[e] - x_tm1[e];
            double b = x_tm1[e] - x_tm2[e];
            dv = a / h_t - b / h_tm1;
        }
        acc += fabs(dv);
    }
    return n > 0 ? acc / (double)n : 0.0;
}

int orc_calibrate(const double* curves, int32_t N, int32_t T, double rho, double dense_frac,
                  double rho_max, double* rho_table, double* alpha, int32_t* clipped,
                  double* lbar) {
    if (N < 1 || T < 1) return -1;
    int32_t D = (int32_t)floor(dense_frac * (double)T + 0.5);
    int32_t t0 = D > 2 ? D : 2;                     /* first sparse step (R-15) */
    if (t0 >= T) return -1;
    double* lavg = (double*)malloc(sizeof(double) * T);
    for (int32_t t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int32_t n = 0; n < N; ++n) acc += curves[(int64_t)n * T + t];
        lavg[t] = acc / (double)N;                 /* R-19: pointwise mean over trajectories */
    }
    double acc = 0.0;
    for (int32_t t = t0; t < T; ++t) acc += lavg[t];
    double lb = acc / (double)(T - t0);            /* Eq. 9 */
    if (!(lb > 0.0) || !isfinite(lb)) { free(lavg); return -1; }
    for (int32_t t = 0; t < T; ++t) {
        if (t < t0) { rho_table[t] = 1.0; alpha[t] = 0.0; clipped[t] = 0; continue; }
        double a = lavg[t] / lb;                   /* Eq. 10 */
        double r = rho * a;                        /* Eq. 11 */
        clipped[t] = r > rho_max;
        rho_table[t] = r > rho_max ? rho_max : r;  /* R-18 */
        alpha[t] = a;
    }
    *lbar = lb;
    free(lavg);
    return 0;
}

int64_t orc_density_to_k(double rho_t, int64_t n_blocks) {
    double kf = floor(rho_t * (double)n_blocks + 0.5);
    int64_t k = (kf > (double)n_blocks) ? n_blocks : (int64_t)kf;
    if (k < 1) k = 1;
    if (k > n_blocks) k = n_blocks;
    return k;
}

int orc_budget(const double* x_t, const double* x_tm1, const double* x_tm2,
               int64_t n, int kind, double h_t, double h_tm1,
               int32_t T, int32_t step, double rho, double dense_frac,
               double l1_mean, double rho_max, const double* rho_table,
               double out[5]) {
    if (T < 1 || step < 0 || step >= T) return -1;
    if (kind == 0 && (h_t == 0.0 || h_tm1 == 0.0)) return -1;
    if (!(l1_mean > 0.0)) return -1;
    double l = orc_l1(x_t, x_tm1, x_tm2, n, kind, h_t, h_tm1);
    /* Eq. 10: alpha_t = l_t / l-bar */
    double alpha = l / l1_mean;
    /* B2: dense prefix, first round(0.2 T) steps (R-15) */
    int32_t Dn = (int32_t)floor(dense_frac * (double)T + 0.5);
    double rho_t, dense = 0.0, clipped = 0.0;
    if (step < Dn || step < 2) {
        rho_t = 1.0;
        dense = 1.0;
    } else {
        /* Eq. 11: rho_t = rho * alpha_t, or the calibrated table (R-17) */
        double rp = rho_table ? rho_table[step] : rho * alpha;
        if (rp > rho_max) { rho_t = rho_max; clipped = 1.0; } /* R-18 */
        else rho_t = rp;
    }
    out[0] = l; out[1] = alpha; out[2] = rho_t; out[3] = dense; out[4] = clipped;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Routing.                                                                   */
/* ------------------------------------------------------------------------ */
/* R1: mean of block b = (sum over tokens in ascending order) / n_b. */
void orc_block_means(const double* x, int64_t S, int64_t D, int32_t Bsz, double* out) {
    int64_t nb = (S + Bsz - 1) / Bsz;
    for (int64_t b = 0; b < nb; ++b) {
        int64_t t0 = b * Bsz, t1 = t0 + Bsz < S ? t0 + Bsz : S;
        for (int64_t a = 0; a < D; ++a) {
            double acc = 0.0;
            for (int64_t t = t0; t < t1; ++t) acc += x[t * D + a];
            out[b * D + a] = acc / (double)(t1 - t0);
        }
    }
}

typedef struct { double key; int64_t j; } orc_scored;

/* total order of R-13: larger score first, then smaller block index */
static int orc_cmp_desc(const void* pa, const void* pb) {
    const orc_scored* a = (const orc_scored*)pa;
    const orc_scored* b = (const orc_scored*)pb;
    if (a->key > b->key) return -1;
    if (a->key < b->key) return 1;
    return (a->j < b->j) ? -1 : (a->j > b->j);
}
static int orc_cmp_i32(const void* pa, const void* pb) {
    int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    return (a > b) - (a < b);
}

void orc_route(const double* q, const double* k, int64_t B, int64_t H, int64_t S, int64_t D,
               int32_t Bq, int32_t Bk, double beta, uint64_t seed, int32_t step,
               int64_t H_total, int64_t head_offset, int64_t kk,
               int32_t* idx, uint32_t* mask, double* scores,
               const double* het, double eps) {
    int64_t NQ = (S + Bq - 1) / Bq, NK = (S + Bk - 1) / Bk, W = (NK + 31) / 32;
    int64_t BH = B * H;
    if (kk > NK) kk = NK;
    if (kk < 1) kk = 1;
    double s = 1.0 / sqrt((double)D);
    for (int64_t bh = 0; bh < BH; ++bh) {
        const double* qh = q + bh * S * D;
        const double* kh = k + bh * S * D;
        int64_t gh = (bh / H) * H_total + head_offset + (bh % H);
        double* Qbar = (double*)malloc(sizeof(double) * NQ * D);
        double* Kbar = (double*)malloc(sizeof(double) * NK * D);
        orc_block_means(qh, S, D, Bq, Qbar);
        orc_block_means(kh, S, D, Bk, Kbar);
        #pragma omp parallel for schedule(dynamic)
        for (int64_t i = 0; i < NQ; ++i) {
            double* r = (double*)malloc(sizeof(double) * NK);
            orc_scored* sc = (orc_scored*)malloc(sizeof(orc_scored) * NK);
            /* R2: r_ij = s * dot, dot an fma chain in ascending dimension order */
            for (int64_t j = 0; j < NK; ++j) {
                double dot = 0.0;
                for (int64_t a = 0; a < D; ++a) dot = fma(Qbar[i * D + a], Kbar[j * D + a], dot);
                r[j] = s * dot;
                /* Eq. 8 prior: + log(||H_j - C||_F + eps) */
                if (het) r[j] = r[j] + log(het[bh * NK + j] + eps);
            }
            /* R3: row mean and population standard deviation */
            double sum = 0.0;
            for (int64_t j = 0; j < NK; ++j) sum += r[j];
            double mu = sum / (double)NK;
            double acc = 0.0;
            for (int64_t j = 0; j < NK; ++j) { double dl = r[j] - mu; acc = fma(dl, dl, acc); }
            double sigma = sqrt(acc / (double)NK);
            /* R4/R5: rt = r + (beta*sigma)*g; beta == 0 leaves r bit-for-bit */
            double bi = beta * sigma;
            for (int64_t j = 0; j < NK; ++j) {
                double rt = r[j];
                if (beta != 0.0) rt = r[j] + bi * orc_gumbel(seed, step, gh, i, j);
                sc[j].key = rt;
                sc[j].j = j;
                if (scores) scores[(bh * NQ + i) * NK + j] = rt;
            }
            /* R6: first kk of the total order, emitted ascending */
            qsort(sc, (size_t)NK, sizeof(orc_scored), orc_cmp_desc);
            int32_t* row = idx + (bh * NQ + i) * kk;
            for (int64_t p = 0; p < kk; ++p) row[p] = (int32_t)sc[p].j;
            qsort(row, (size_t)kk, sizeof(int32_t), orc_cmp_i32);
            uint32_t* mrow = mask + (bh * NQ + i) * W;
            for (int64_t w = 0; w < W; ++w) mrow[w] = 0u;
            for (int64_t p = 0; p < kk; ++p) mrow[row[p] >> 5] |= 1u << (row[p] & 31);
            free(r);
            free(sc);
        }
        free(Qbar);
        free(Kbar);
    }
}

/* ------------------------------------------------------------------------ */
/* Block statistics.                                                          */
/* ------------------------------------------------------------------------ */
void orc_block_stats(const double* k, const double* v, int64_t S, int64_t D,
                     int32_t Bk, int32_t G, double* Kbar, double* Vsum,
                     double* Hblk, double* Hbar) {
    int64_t NK = (S + Bk - 1) / Bk;
    int64_t NG = (NK + G - 1) / G;
    orc_block_means(k, S, D, Bk, Kbar);
    for (int64_t j = 0; j < NK; ++j) {
        int64_t t0 = j * Bk, t1 = t0 + Bk < S ? t0 + Bk : S;
        for (int64_t b = 0; b < D; ++b) {
            double acc = 0.0;
            for (int64_t t = t0; t < t1; ++t) acc += v[t * D + b];
            Vsum[j * D + b] = acc;
        }
    }
    #pragma omp parallel for schedule(dynamic)
    for (int64_t g = 0; g < NG; ++g) {
        int64_t j0 = g * G, j1 = j0 + G < NK ? j0 + G : NK;
        double* Hg = Hbar + g * D * D;
        double* Hj = (double*)malloc(sizeof(double) * D * D);
        for (int64_t e = 0; e < D * D; ++e) Hg[e] = 0.0;
        for (int64_t j = j0; j < j1; ++j) {
            int64_t t0 = j * Bk, t1 = t0 + Bk < S ? t0 + Bk : S;
            /* Eq. 5: H_j = sum_n (K_{j,n} - Kbar_j)^T V_{j,n} */
            for (int64_t a = 0; a < D; ++a)
                for (int64_t b = 0; b < D; ++b) {
                    double acc = 0.0;
                    for (int64_t t = t0; t < t1; ++t)
                        acc += (k[t * D + a] - Kbar[j * D + a]) * v[t * D + b];
                    Hj[a * D + b] = acc;
                }
            if (Hblk) memcpy(Hblk + j * D * D, Hj, sizeof(double) * D * D);
            for (int64_t e = 0; e < D * D; ++e) Hg[e] += Hj[e];
        }
        /* App. B: unweighted mean over the blocks of the group */
        for (int64_t e = 0; e < D * D; ++e) Hg[e] = Hg[e] / (double)(j1 - j0);
        free(Hj);
    }
}

/* ------------------------------------------------------------------------ */
/* Heterogeneity prior of Eq. 8.                                              */
/* ------------------------------------------------------------------------ */
void orc_heterogeneity(const double* k, const double* v, int64_t S, int64_t D, int32_t Bk,
                       int32_t G, int32_t mode, double* het) {
    int64_t NK = (S + Bk - 1) / Bk;
    int64_t NG = (NK + G - 1) / G;
    double* Kbar = (double*)malloc(sizeof(double) * NK * D);
    double* Vsum = (double*)malloc(sizeof(double) * NK * D);
    double* Hblk = (double*)malloc(sizeof(double) * NK * D * D);
    double* Hgrp = (double*)malloc(sizeof(double) * NG * D * D);
    double* Hglob = (double*)malloc(sizeof(double) * D * D);
    orc_block_stats(k, v, S, D, Bk, G, Kbar, Vsum, Hblk, Hgrp);
    /* Eq. 6: Hbar = (1/N_B) sum_j H_j, blocks in ascending order */
    for (int64_t e = 0; e < D * D; ++e) {
        double acc = 0.0;
        for (int64_t j = 0; j < NK; ++j) acc += Hblk[j * D * D + e];
        Hglob[e] = acc / (double)NK;
    }
    for (int64_t j = 0; j < NK; ++j) {
        const double* C = mode == 2 ? Hgrp + (j / G) * D * D : Hglob;
        const double* Hj = Hblk + j * D * D;
        double acc = 0.0;
        for (int64_t e = 0; e < D * D; ++e) {
            double d = Hj[e] - C[e];
            acc += d * d;
        }
        het[j] = sqrt(acc);
    }
    free(Kbar); free(Vsum); free(Hblk); free(Hgrp); free(Hglob);
}

/* ------------------------------------------------------------------------ */
/* Attention with a given route.                                              */
/* ------------------------------------------------------------------------ */
static inline void neu_add(double* s, double* c, double x) {
    double t = *s + x;
    if (fabs(*s) >= fabs(x)) *c += (*s - t) + x;
    else *c += (x - t) + *s;
    *s = t;
}

/* One query block i of one head.  Per row t (A2-A4 of DESIGN.md §3):
 *   e_u = s q_t.K_u for tokens u of selected blocks            (Eq. 7, term 1)
 *   c_j = s q_t.Kbar_j for unselected blocks j                  (alpha_{t,j}, R-1)
 *   m   = max over all e_u and c_j (exact row max, R-22)
 *   N   = sum_u e^{e_u-m} V_u + sum_{j in U} e^{c_j-m} Vsum_j   (Eq. 7, terms 1-2)
 *       + sum_g (sum_{j in U cap G_g} e^{c_j-m}) s q_t Hbar^(g)  (App. B, :505)
 *   Den = sum_u e^{e_u-m} + sum_{j in U} n_j e^{c_j-m}           (R-2)
 *   O_t = N / Den. */
static void orc_attn_qblock(const double* qh, const double* kh, const double* vh,
                            const double* Kbar, const double* Vsum, const double* Hbar,
                            int64_t S, int64_t D, int32_t Bq, int32_t Bk, int32_t G,
                            int32_t comp, int64_t i, const int32_t* sel_idx, int64_t cnt,
                            double* out_rows /* [Bq][D], row r = token i*Bq + r */) {
    int64_t NK = (S + Bk - 1) / Bk;
    int64_t NG = (NK + G - 1) / G;
    double s = 1.0 / sqrt((double)D);
    char* sel = (char*)calloc((size_t)NK, 1);
    for (int64_t p = 0; p < cnt; ++p) sel[sel_idx[p]] = 1;
    double* e = (double*)malloc(sizeof(double) * S);
    double* c = (double*)malloc(sizeof(double) * NK);
    double* A = (double*)malloc(sizeof(double) * NG);
    double* Ac = (double*)malloc(sizeof(double) * NG);
    double* Nv = (double*)malloc(sizeof(double) * D);
    double* Nc = (double*)malloc(sizeof(double) * D);
    int64_t t0 = i * Bq, t1 = t0 + Bq < S ? t0 + Bq : S;
    for (int64_t t = t0; t < t1; ++t) {
        const double* qt = qh + t * D;
        double m = -INFINITY;
        /* exact logits over the selected blocks (true lengths, R-7) */
        for (int64_t p = 0; p < cnt; ++p) {
            int64_t j = sel_idx[p];
            int64_t u0 = j * Bk, u1 = u0 + Bk < S ? u0 + Bk : S;
            for (int64_t u = u0; u < u1; ++u) {
                double dot = 0.0;
                for (int64_t a = 0; a < D; ++a) dot += qt[a] * kh[u * D + a];
                e[u] = s * dot;
                if (e[u] > m) m = e[u];
            }
        }
        /* centroid logits over the unselected blocks */
        if (comp != 2) {
            for (int64_t j = 0; j < NK; ++j) {
                if (sel[j]) continue;
                double dot = 0.0;
                for (int64_t a = 0; a < D; ++a) dot += qt[a] * Kbar[j * D + a];
                c[j] = s * dot;
                if (c[j] > m) m = c[j];
            }
        }
        for (int64_t a = 0; a < D; ++a) { Nv[a] = 0.0; Nc[a] = 0.0; }
        for (int64_t g = 0; g < NG; ++g) { A[g] = 0.0; Ac[g] = 0.0; }
        double den = 0.0, denc = 0.0;
        for (int64_t p = 0; p < cnt; ++p) {
            int64_t j = sel_idx[p];
            int64_t u0 = j * Bk, u1 = u0 + Bk < S ? u0 + Bk : S;
            for (int64_t u = u0; u < u1; ++u) {
                double w = exp(e[u] - m);
                neu_add(&den, &denc, w);
                for (int64_t a = 0; a < D; ++a) neu_add(&Nv[a], &Nc[a], w * vh[u * D + a]);
            }
        }
        if (comp != 2) {
            for (int64_t j = 0; j < NK; ++j) {
                if (sel[j]) continue;
                int64_t nj = (j + 1) * Bk < S ? Bk : S - j * Bk;
                double w = exp(c[j] - m);
                neu_add(&den, &denc, (double)nj * w);
                for (int64_t a = 0; a < D; ++a) neu_add(&Nv[a], &Nc[a], w * Vsum[j * D + a]);
                neu_add(&A[j / G], &Ac[j / G], w);
            }
        }
        if (comp == 0) {
            for (int64_t g = 0; g < NG; ++g) {
                double Ag = A[g] + Ac[g];
                if (Ag == 0.0) continue;
                const double* Hg = Hbar + g * D * D;
                for (int64_t b = 0; b < D; ++b) {
                    double y = 0.0; /* (q_t Hbar^(g))_b = sum_a q_t[a] Hbar[a][b] */
                    for (int64_t a = 0; a < D; ++a) y += qt[a] * Hg[a * D + b];
                    neu_add(&Nv[b], &Nc[b], Ag * (s * y));
                }
            }
        }
        double Dt = den + denc;
        for (int64_t a = 0; a < D; ++a) out_rows[(t - t0) * D + a] = (Nv[a] + Nc[a]) / Dt;
    }
    free(sel); free(e); free(c); free(A); free(Ac); free(Nv); free(Nc);
}

void orc_attn_with_route(const double* q, const double* k, const double* v,
                         int64_t BH, int64_t S, int64_t D, int32_t Bq, int32_t Bk,
                         int32_t G, int32_t comp, const int32_t* idx,
                         const int32_t* count, int64_t kk_stride, double* out) {
    int64_t NQ = (S + Bq - 1) / Bq, NK = (S + Bk - 1) / Bk, NG = (NK + G - 1) / G;
    double* Kbar = (double*)malloc(sizeof(double) * NK * D);
    double* Vsum = (double*)malloc(sizeof(double) * NK * D);
    double* Hbar = (double*)malloc(sizeof(double) * NG * D * D);
    for (int64_t bh = 0; bh < BH; ++bh) {
        const double* qh = q + bh * S * D;
        const double* kh = k + bh * S * D;
        const double* vh = v + bh * S * D;
        orc_block_stats(kh, vh, S, D, Bk, G, Kbar, Vsum, NULL, Hbar);
        #pragma omp parallel for schedule(dynamic)
        for (int64_t i = 0; i < NQ; ++i) {
            orc_attn_qblock(qh, kh, vh, Kbar, Vsum, Hbar, S, D, Bq, Bk, G, comp, i,
                            idx + (bh * NQ + i) * kk_stride, count[bh * NQ + i],
                            out + (bh * S + i * Bq) * D);
        }
    }
    free(Kbar); free(Vsum); free(Hbar);
}

void orc_attn_pairs(const double* q, const double* k, const double* v,
                    int64_t BH, int64_t S, int64_t D, int32_t Bq, int32_t Bk,
                    int32_t G, int32_t comp, const int32_t* idx,
                    const int32_t* count, int64_t kk_stride,
                    const int64_t* pairs, int64_t npairs, double* out) {
    int64_t NQ = (S + Bq - 1) / Bq, NK = (S + Bk - 1) / Bk, NG = (NK + G - 1) / G;
    /* statistics once per distinct head that the sample touches */
    int64_t* slot = (int64_t*)malloc(sizeof(int64_t) * BH);
    for (int64_t b = 0; b < BH; ++b) slot[b] = -1;
    int64_t nh = 0;
    for (int64_t p = 0; p < npairs; ++p) if (slot[pairs[2 * p]] < 0) slot[pairs[2 * p]] = nh++;
    double* Kbar = (double*)malloc(sizeof(double) * nh * NK * D);
    double* Vsum = (double*)malloc(sizeof(double) * nh * NK * D);
    double* Hbar = (double*)malloc(sizeof(double) * nh * NG * D * D);
    for (int64_t b = 0; b < BH; ++b) {
        if (slot[b] < 0) continue;
        int64_t h = slot[b];
        orc_block_stats(k + b * S * D, v + b * S * D, S, D, Bk, G, Kbar + h * NK * D,
                        Vsum + h * NK * D, NULL, Hbar + h * NG * D * D);
    }
    #pragma omp parallel for schedule(dynamic)
    for (int64_t p = 0; p < npairs; ++p) {
        int64_t bh = pairs[2 * p], i = pairs[2 * p + 1], h = slot[bh];
        orc_attn_qblock(q + bh * S * D, k + bh * S * D, v + bh * S * D, Kbar + h * NK * D,
                        Vsum + h * NK * D, Hbar + h * NG * D * D, S, D, Bq, Bk, G, comp, i,
                        idx + (bh * NQ + i) * kk_stride, count[bh * NQ + i],
                        out + p * (int64_t)Bq * D);
    }
    free(slot); free(Kbar); free(Vsum); free(Hbar);
}
