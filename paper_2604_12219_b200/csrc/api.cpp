// api.cpp -- the C ABI of libpasa.so (include/pasa.h): argument validation,
// workspace layout and kernel launches.  Every entry point validates on the
// host and launches nothing on failure; no call allocates device memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "pasa_internal.h"

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

pasa_status fail(pasa_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

pasa_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return PASA_OK;
    return fail(PASA_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

constexpr size_t kAlign = 1024;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct RouteLayout {
    int64_t NQ, NK, NG, W, BH;
    size_t off_hdr, off_qbar, off_kbar, off_kfrag, off_q8, off_k8, off_sq8, off_kb8, off_kamax, off_scores, off_kbar_lp, off_vsum, off_ht, off_idx,
        off_count, off_mask, off_het, off_prior, off_hj, off_hgs, off_hglob, off_part, total;
};

pasa_status check_cfg(const pasa_route_cfg* c, int64_t B, int64_t S, int64_t H, int64_t D) {
    if (!c) return fail(PASA_EINVAL, "route cfg is NULL");
    if (B < 1 || S < 1 || H < 1) return fail(PASA_ESHAPE, "B, S, H must be >= 1");
    if (D != 64 && D != 128) return fail(PASA_EUNSUPPORTED, "D=%lld not in {64,128}", (long long)D);
    if (c->Bq != 64 && c->Bq != 128 && c->Bq != 256)
        return fail(PASA_EUNSUPPORTED, "Bq=%d not in {64,128,256}", c->Bq);
    if (c->Bk != 64) return fail(PASA_EUNSUPPORTED, "Bk=%d != 64", c->Bk);
    if (c->G < 1) return fail(PASA_EINVAL, "G=%d < 1", c->G);
    if (c->comp < 0 || c->comp > 2) return fail(PASA_EINVAL, "comp=%d", c->comp);
    if (!(c->beta >= 0.0) || !std::isfinite(c->beta))
        return fail(PASA_EINVAL, "beta must be finite and >= 0");
    if (c->head_offset < 0 || c->H_total < c->head_offset + H)
        return fail(PASA_EINVAL, "head_offset=%lld H=%lld exceed H_total=%lld",
                    (long long)c->head_offset, (long long)H, (long long)c->H_total);
    if (c->prior < PASA_PRIOR_NONE || c->prior > PASA_PRIOR_GROUP)
        return fail(PASA_EINVAL, "prior=%d", c->prior);
    if (c->prior != PASA_PRIOR_NONE && !(c->eps > 0.0 && std::isfinite(c->eps)))
        return fail(PASA_EINVAL, "prior eps must be finite and > 0");
    const int64_t NK = (S + c->Bk - 1) / c->Bk;
    // the tensor-core attention kernels' op list holds 4096 kept blocks (S <= 262,144 at
    // Bk = 64); the route has no limit of its own
    if (NK > 4096) return fail(PASA_EUNSUPPORTED, "N_K=%lld > 4096 (S too long)", (long long)NK);
    if (c->qk_fp8 != 0 && c->qk_fp8 != 1) return fail(PASA_EINVAL, "qk_fp8=%d", c->qk_fp8);
    if (c->qk_fp8 && (D != 128 || c->Bq != 128 || (c->comp == PASA_COMP_GROUPED && c->G < 32)))
        return fail(PASA_EUNSUPPORTED, "qk_fp8 needs D = 128, Bq = 128 and G >= 32");
    const int64_t NQ = (S + c->Bq - 1) / c->Bq;
    if ((c->qb_begin != 0 || c->qb_end != 0) &&
        !(c->qb_begin >= 0 && c->qb_begin < c->qb_end && c->qb_end <= B * H * NQ))
        return fail(PASA_EINVAL, "item range [%d, %d) outside [0, B*H*N_Q=%lld)", c->qb_begin,
                    c->qb_end, (long long)(B * H * NQ));
    return PASA_OK;
}

RouteLayout layout(const pasa_route_cfg* c, int64_t B, int64_t S, int64_t H, int64_t D) {
    RouteLayout L;
    L.NQ = (S + c->Bq - 1) / c->Bq;
    L.NK = (S + c->Bk - 1) / c->Bk;
    L.NG = (L.NK + c->G - 1) / c->G;
    L.W = (L.NK + 31) / 32;
    L.BH = B * H;
    size_t o = 0;
    L.off_hdr = o;      o = align_up(o + 64);
    L.off_qbar = o;     o = align_up(o + sizeof(double) * L.BH * L.NQ * D);
    L.off_kbar = o;     o = align_up(o + sizeof(double) * L.BH * L.NK * D);
    L.off_kfrag = o;    o = align_up(o + sizeof(double) * L.BH * ((L.NK + 7) / 8) * 8 * D);
    const bool f8 = c->qk_fp8 != 0;   // FP8 QK^T variant: E4M3 copies and scales
    L.off_q8 = o;       o = align_up(o + (f8 ? (size_t)L.BH * S * D : 0));
    L.off_k8 = o;       o = align_up(o + (f8 ? (size_t)L.BH * S * D : 0));
    L.off_sq8 = o;      o = align_up(o + (f8 ? sizeof(float) * L.BH * S : 0));
    L.off_kb8 = o;      o = align_up(o + (f8 ? (size_t)L.BH * L.NK * D : 0));
    L.off_kamax = o;    o = align_up(o + (f8 ? sizeof(uint32_t) * 2 * L.BH : 0));
    // fp64 score rows: on chip (shared memory) unless a row tile does not fit there
    const bool gsc = pasa::route_rows_per_cta(L.NK, D) == 0;
    L.off_scores = o;   o = align_up(o + (gsc ? sizeof(double) * L.BH * L.NQ * pasa::route_score_stride(L.NK) : 0));
    L.off_kbar_lp = o;  o = align_up(o + 4 * L.BH * L.NK * D);
    L.off_vsum = o;     o = align_up(o + 4 * L.BH * L.NK * D);
    L.off_ht = o;       o = align_up(o + 4 * L.BH * L.NG * D * D);
    L.off_idx = o;      o = align_up(o + sizeof(int32_t) * L.BH * L.NQ * L.NK);
    L.off_count = o;    o = align_up(o + sizeof(int32_t) * L.BH * L.NQ);
    L.off_mask = o;     o = align_up(o + sizeof(uint32_t) * L.BH * L.NQ * L.W);
    const bool pr = c->prior != PASA_PRIOR_NONE;   // Eq. 8 prior buffers (fp64)
    L.off_het = o;      o = align_up(o + (pr ? sizeof(double) * L.BH * L.NK : 0));
    L.off_prior = o;    o = align_up(o + (pr ? sizeof(double) * L.BH * L.NK : 0));
    // every block's H_j in fp64 (8 D^2 bytes per block: 6.2 GB for a Wan-14B layer),
    // computed once and read by the means and norm passes
    L.off_hj = o;       o = align_up(o + (pr ? sizeof(double) * L.BH * L.NK * D * D : 0));
    L.off_hgs = o;      o = align_up(o + (pr ? sizeof(double) * L.BH * L.NG * D * D : 0));
    L.off_hglob = o;    o = align_up(o + (pr ? sizeof(double) * L.BH * D * D : 0));
    // large groups on the tensor-core statistics kernel: fp32 sums of 32-block chunks
    const bool big = c->G > 32;
    L.off_part = o;     o = align_up(o + (big ? sizeof(float) * L.BH * ((L.NK + 31) / 32) * D * D : 0));
    L.total = o;
    return L;
}

size_t elem_size(int32_t dt) { return dt == PASA_F32 ? 4 : 2; }

pasa_status check_tensor(const pasa_tensor* t, const char* name) {
    if (!t || !t->data) return fail(PASA_EINVAL, "%s is NULL", name);
    if (t->dtype != PASA_BF16 && t->dtype != PASA_F32)
        return fail(PASA_EDTYPE, "%s dtype %d", name, t->dtype);
    if (t->B < 1 || t->S < 1 || t->H < 1) return fail(PASA_ESHAPE, "%s has an empty dim", name);
    if ((reinterpret_cast<uintptr_t>(t->data) & 15) != 0)
        return fail(PASA_ESHAPE, "%s data not 16-byte aligned", name);
    const int64_t m = 16 / (int64_t)elem_size(t->dtype);
    if (t->sS % m || t->sH % m || t->sB % m || t->sS <= 0 || t->sH <= 0 || t->sB <= 0)
        return fail(PASA_ESHAPE, "%s strides (%lld,%lld,%lld) must be positive multiples of 16 B",
                    name, (long long)t->sB, (long long)t->sS, (long long)t->sH);
    return PASA_OK;
}

pasa_status match_route(const pasa_tensor* t, const pasa_route_s* r, const char* name) {
    if (t->B != r->B || t->S != r->S || t->H != r->H || t->D != r->D)
        return fail(PASA_ESHAPE, "%s shape [%lld,%lld,%lld,%lld] != route [%lld,%lld,%lld,%lld]",
                    name, (long long)t->B, (long long)t->S, (long long)t->H, (long long)t->D,
                    (long long)r->B, (long long)r->S, (long long)r->H, (long long)r->D);
    return PASA_OK;
}

pasa_status check_schedule(const pasa_schedule* sc) {
    const bool vel = sc->kind == PASA_IN_VELOCITY;
    if (sc->T < 1 || sc->step < 0 || sc->step >= sc->T)
        return fail(PASA_EINVAL, "step=%d outside [0, T=%d)", sc->step, sc->T);
    if (!vel && (sc->h_t == 0.0 || sc->h_tm1 == 0.0)) return fail(PASA_EINVAL, "h == 0");
    if (!(sc->l1_mean > 0.0)) return fail(PASA_EDEGENERATE, "l1_mean must be > 0 (Eq. 10)");
    if (!(sc->rho >= 0.0) || !(sc->rho_max > 0.0) || !(sc->dense_frac >= 0.0))
        return fail(PASA_EINVAL, "rho / rho_max / dense_frac out of range");
    return PASA_OK;
}

pasa::BudgetParams budget_params(const pasa_schedule* sc) {
    pasa::BudgetParams p;
    p.rht = 1.0 / sc->h_t;
    p.rh1 = 1.0 / sc->h_tm1;
    p.step = sc->step;
    p.dense_steps = (int32_t)std::floor(sc->dense_frac * (double)sc->T + 0.5);
    p.rho = sc->rho;
    p.l1_mean = sc->l1_mean;
    p.rho_max = sc->rho_max;
    p.use_table = sc->rho_table != nullptr;
    p.table_val = p.use_table ? sc->rho_table[sc->step] : 0.0;
    return p;
}

}  // namespace

extern "C" {

const char* pasa_last_error(void) { return g_err.c_str(); }
int32_t pasa_last_launch_count(void) { return g_launches; }
const char* pasa_version(void) { return "pasa-b200 0.1 (sm_100a)"; }

uint64_t pasa_layer_seed(uint64_t seed, int32_t layer) {
    uint64_t z = seed + (uint64_t)((int64_t)layer + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

pasa_status pasa_calibrate(const double* l1_curves, int32_t N, int32_t T, double rho,
                           double dense_frac, double rho_max, double* rho_table, double* alpha,
                           int32_t* clipped, double* l1_mean) {
    if (!l1_curves || !rho_table || !l1_mean) return fail(PASA_EINVAL, "NULL argument");
    if (N < 1 || T < 1) return fail(PASA_EINVAL, "N=%d T=%d", N, T);
    if (!(rho >= 0.0) || !(rho_max > 0.0) || !(dense_frac >= 0.0))
        return fail(PASA_EINVAL, "rho / rho_max / dense_frac out of range");
    const int32_t dense = (int32_t)std::floor(dense_frac * (double)T + 0.5);
    const int32_t t0 = std::max(dense, 2);                       // R-15
    if (t0 >= T) return fail(PASA_EINVAL, "no sparse step (T=%d, dense prefix %d)", T, t0);
    std::vector<double> lavg((size_t)T);
    for (int32_t t = t0; t < T; ++t) {                           // R-19 pointwise mean
        double acc = 0.0;
        for (int32_t n = 0; n < N; ++n) {
            const double x = l1_curves[(int64_t)n * T + t];
            if (!std::isfinite(x)) return fail(PASA_EINVAL, "l1_curves[%d][%d] not finite", n, t);
            acc += x;
        }
        lavg[t] = acc / (double)N;
    }
    double acc = 0.0;
    for (int32_t t = t0; t < T; ++t) acc += lavg[t];
    const double lb = acc / (double)(T - t0);                    // Eq. 9
    if (!(lb > 0.0)) return fail(PASA_EDEGENERATE, "l1_mean = %g <= 0 (Eq. 10)", lb);
    for (int32_t t = 0; t < T; ++t) {
        double a = 0.0, r = 1.0;
        int32_t c = 0;
        if (t >= t0) {
            a = lavg[t] / lb;                                    // Eq. 10
            const double rp = rho * a;                           // Eq. 11
            c = rp > rho_max;
            r = c ? rho_max : rp;                                // R-18
        }
        rho_table[t] = r;
        if (alpha) alpha[t] = a;
        if (clipped) clipped[t] = c;
    }
    *l1_mean = lb;
    return PASA_OK;
}

pasa_status pasa_copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                        size_t height, int32_t kind, void* stream) {
    if (!dst || !src) return fail(PASA_EINVAL, "NULL pointer");
    if (width > dpitch || width > spitch) return fail(PASA_EINVAL, "width exceeds a pitch");
    if (kind != 1 && kind != 2) return fail(PASA_EINVAL, "kind=%d (1 = H2D, 2 = D2H)", kind);
    if (width == 0 || height == 0) return PASA_OK;
    const cudaError_t e =
        cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height,
                          kind == 1 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                          (cudaStream_t)stream);
    return cuda_status(e, "pasa_copy2d");
}

size_t pasa_budget_workspace_bytes(void) {
    // record, one fp64 partial per reduction CTA, the CTAs' completion ticket
    return sizeof(pasa::BudgetRec) + sizeof(double) * pasa::kBudgetParts + 64;
}

size_t pasa_route_workspace_bytes(const pasa_route_cfg* cfg, int64_t B, int64_t S, int64_t H,
                                  int64_t D) {
    if (check_cfg(cfg, B, S, H, D) != PASA_OK) return 0;
    return layout(cfg, B, S, H, D).total;
}

pasa_status pasa_budget_init(void* dev_ws, size_t bytes, pasa_budget_h* out) {
    if (!dev_ws || !out) return fail(PASA_EINVAL, "NULL workspace or handle pointer");
    if (bytes < pasa_budget_workspace_bytes())
        return fail(PASA_ENOSPACE, "budget workspace %zu < %zu", bytes,
                    pasa_budget_workspace_bytes());
    if (reinterpret_cast<uintptr_t>(dev_ws) & 15) return fail(PASA_EINVAL, "workspace misaligned");
    auto* h = new (std::nothrow) pasa_budget_s;
    if (!h) return fail(PASA_EINVAL, "out of host memory");
    h->rec = reinterpret_cast<pasa::BudgetRec*>(dev_ws);
    h->partials = reinterpret_cast<double*>(reinterpret_cast<char*>(dev_ws) +
                                            sizeof(pasa::BudgetRec));
    h->ticket = reinterpret_cast<unsigned int*>(h->partials + pasa::kBudgetParts);
    h->ticket_ready = 0;   // zeroed on the handle's first launch (the kernel then resets it)
    *out = h;
    return PASA_OK;
}

pasa_status pasa_route_init(void* dev_ws, size_t bytes, const pasa_route_cfg* cfg, int64_t B,
                            int64_t S, int64_t H, int64_t D, pasa_route_h* out) {
    pasa_status st = check_cfg(cfg, B, S, H, D);
    if (st != PASA_OK) return st;
    if (!dev_ws || !out) return fail(PASA_EINVAL, "NULL workspace or handle pointer");
    if (reinterpret_cast<uintptr_t>(dev_ws) % 256) return fail(PASA_EINVAL, "workspace must be 256-byte aligned");
    RouteLayout L = layout(cfg, B, S, H, D);
    if (bytes < L.total) return fail(PASA_ENOSPACE, "route workspace %zu < %zu", bytes, L.total);
    auto* r = new (std::nothrow) pasa_route_s;
    if (!r) return fail(PASA_EINVAL, "out of host memory");
    char* w = reinterpret_cast<char*>(dev_ws);
    r->cfg = *cfg;
    r->B = B; r->S = S; r->H = H; r->D = D;
    r->NQ = L.NQ; r->NK = L.NK; r->NG = L.NG; r->W = L.W; r->BH = L.BH;
    const bool all = cfg->qb_begin == 0 && cfg->qb_end == 0;
    r->it0 = all ? 0 : cfg->qb_begin;
    r->it1 = all ? L.BH * L.NQ : cfg->qb_end;
    r->hdr = reinterpret_cast<int32_t*>(w + L.off_hdr);
    r->qbar = reinterpret_cast<double*>(w + L.off_qbar);
    r->kbar = reinterpret_cast<double*>(w + L.off_kbar);
    r->kfrag = reinterpret_cast<double*>(w + L.off_kfrag);
    const bool f8 = cfg->qk_fp8 != 0;
    r->q8 = f8 ? reinterpret_cast<uint8_t*>(w + L.off_q8) : nullptr;
    r->k8 = f8 ? reinterpret_cast<uint8_t*>(w + L.off_k8) : nullptr;
    r->sq8 = f8 ? reinterpret_cast<float*>(w + L.off_sq8) : nullptr;
    r->kb8 = f8 ? reinterpret_cast<uint8_t*>(w + L.off_kb8) : nullptr;
    r->kamax = f8 ? reinterpret_cast<uint32_t*>(w + L.off_kamax) : nullptr;
    r->kbamax = f8 ? r->kamax + L.BH : nullptr;
    r->scores = pasa::route_rows_per_cta(L.NK, D) == 0 ? reinterpret_cast<double*>(w + L.off_scores)
                                                        : nullptr;
    r->kbar_lp = w + L.off_kbar_lp;
    r->vsum_lp = w + L.off_vsum;
    r->ht = w + L.off_ht;
    r->idx = reinterpret_cast<int32_t*>(w + L.off_idx);
    r->idx_ld = L.NK;
    r->count = reinterpret_cast<int32_t*>(w + L.off_count);
    r->mask = reinterpret_cast<uint32_t*>(w + L.off_mask);
    const bool pr = cfg->prior != PASA_PRIOR_NONE;
    r->het = pr ? reinterpret_cast<double*>(w + L.off_het) : nullptr;
    r->prior = pr ? reinterpret_cast<double*>(w + L.off_prior) : nullptr;
    r->hj = pr ? reinterpret_cast<double*>(w + L.off_hj) : nullptr;
    r->hgs = pr ? reinterpret_cast<double*>(w + L.off_hgs) : nullptr;
    r->hglob = pr ? reinterpret_cast<double*>(w + L.off_hglob) : nullptr;
    r->het_valid = 0;
    r->part = cfg->G > 32 ? reinterpret_cast<float*>(w + L.off_part) : nullptr;
    r->route_dtype = -1;
    r->stats_dtype = -1;
    *out = r;
    return PASA_OK;
}

void pasa_budget_fini(pasa_budget_h h) { delete h; }
void pasa_route_fini(pasa_route_h h) { delete h; }

namespace {
// validation shared by pasa_budget and pasa_budget_local_sum; fills xs[3]
pasa_status check_budget(const pasa_latent* x_t, const pasa_latent* x_tm1, const pasa_latent* x_tm2,
                         const pasa_schedule* sc, pasa_budget_h budget, const pasa_latent* xs[3]) {
    if (!budget || !sc || !x_t || !x_tm1) return fail(PASA_EINVAL, "NULL argument");
    const bool vel = sc->kind == PASA_IN_VELOCITY;
    if (sc->kind != PASA_IN_LATENT && !vel) return fail(PASA_EINVAL, "kind=%d", sc->kind);
    if (!vel && !x_tm2) return fail(PASA_EINVAL, "x_tm2 is NULL for latent input");
    pasa_status st = check_schedule(sc);
    if (st != PASA_OK) return st;
    xs[0] = x_t; xs[1] = x_tm1; xs[2] = vel ? x_tm1 : x_tm2;
    for (int i = 0; i < 3; ++i) {
        if (!xs[i]->data) return fail(PASA_EINVAL, "latent %d data is NULL", i);
        if (xs[i]->dtype != x_t->dtype) return fail(PASA_EDTYPE, "latent dtypes differ");
        if (xs[i]->dtype != PASA_BF16 && xs[i]->dtype != PASA_F32)
            return fail(PASA_EDTYPE, "latent dtype %d", xs[i]->dtype);
        if (xs[i]->numel != x_t->numel) return fail(PASA_ESHAPE, "latent numel differ");
        if (reinterpret_cast<uintptr_t>(xs[i]->data) & 15)
            return fail(PASA_ESHAPE, "latent %d not 16-byte aligned", i);
    }
    if (x_t->numel < 1) return fail(PASA_ESHAPE, "empty latent");
    return PASA_OK;
}
}  // namespace

pasa_status pasa_budget(const pasa_latent* x_t, const pasa_latent* x_tm1, const pasa_latent* x_tm2,
                        const pasa_schedule* sc, pasa_budget_h budget, void* stream) {
    g_launches = 0;
    const pasa_latent* xs[3];
    pasa_status st = check_budget(x_t, x_tm1, x_tm2, sc, budget, xs);
    if (st != PASA_OK) return st;
    int launches = 0;
    cudaError_t e = pasa::launch_budget(xs[0]->data, xs[1]->data, xs[2]->data, x_t->numel,
                                        x_t->dtype, sc->kind == PASA_IN_VELOCITY, budget_params(sc),
                                        budget, nullptr, (cudaStream_t)stream, &launches);
    g_launches = launches;
    return cuda_status(e, "pasa_budget launch");
}

pasa_status pasa_budget_local_sum(const pasa_latent* x_t, const pasa_latent* x_tm1,
                                  const pasa_latent* x_tm2, const pasa_schedule* sc,
                                  pasa_budget_h budget, double* dev_sum, void* stream) {
    g_launches = 0;
    if (!dev_sum) return fail(PASA_EINVAL, "dev_sum is NULL");
    const pasa_latent* xs[3];
    pasa_status st = check_budget(x_t, x_tm1, x_tm2, sc, budget, xs);
    if (st != PASA_OK) return st;
    int launches = 0;
    cudaError_t e = pasa::launch_budget(xs[0]->data, xs[1]->data, xs[2]->data, x_t->numel,
                                        x_t->dtype, sc->kind == PASA_IN_VELOCITY, budget_params(sc),
                                        budget, dev_sum, (cudaStream_t)stream, &launches);
    g_launches = launches;
    return cuda_status(e, "pasa_budget_local_sum launch");
}

pasa_status pasa_budget_from_sums(const double* dev_sums, int32_t nsums, int64_t n_total,
                                  const pasa_schedule* sc, pasa_budget_h budget, void* stream) {
    g_launches = 0;
    if (!budget || !sc || !dev_sums) return fail(PASA_EINVAL, "NULL argument");
    if (nsums < 1 || n_total < 1) return fail(PASA_EINVAL, "nsums=%d n_total=%lld", nsums,
                                              (long long)n_total);
    pasa_status st = check_schedule(sc);
    if (st != PASA_OK) return st;
    int launches = 0;
    cudaError_t e = pasa::launch_budget_from_sums(dev_sums, nsums, n_total, budget_params(sc),
                                                  budget, (cudaStream_t)stream, &launches);
    g_launches = launches;
    return cuda_status(e, "pasa_budget_from_sums launch");
}

namespace {
pasa_status route_common(const pasa_tensor* q, const pasa_tensor* k, const pasa_tensor* v,
                         pasa_budget_h budget, uint64_t seed, int32_t step, pasa_route_h route,
                         void* stream) {
    g_launches = 0;
    if (!route || !budget) return fail(PASA_EINVAL, "NULL handle");
    pasa_status st;
    if ((st = check_tensor(q, "q")) != PASA_OK) return st;
    if ((st = check_tensor(k, "k")) != PASA_OK) return st;
    if (q->dtype != k->dtype) return fail(PASA_EDTYPE, "q and k dtypes differ");
    if (route->cfg.qk_fp8 && q->dtype != PASA_BF16)
        return fail(PASA_EUNSUPPORTED, "qk_fp8 needs bf16 q and k");
    if ((st = match_route(q, route, "q")) != PASA_OK) return st;
    if ((st = match_route(k, route, "k")) != PASA_OK) return st;
    if (v) {
        if ((st = check_tensor(v, "v")) != PASA_OK) return st;
        if (v->dtype != k->dtype) return fail(PASA_EDTYPE, "v and k dtypes differ");
        if ((st = match_route(v, route, "v")) != PASA_OK) return st;
    }
    int launches = 0;
    cudaError_t e = pasa::launch_route(*q, *k, v, budget, seed, step, route, (cudaStream_t)stream,
                                       &launches);
    g_launches = launches;
    if (e == cudaSuccess) {
        route->route_dtype = q->dtype;
        route->stats_dtype = -1;   // Kbar changed: the next pasa_attn must recompute the stats
        route->het_valid = v != nullptr;
    }
    return cuda_status(e, "pasa_route launch");
}
}  // namespace

pasa_status pasa_route(const pasa_tensor* q, const pasa_tensor* k, pasa_budget_h budget,
                       uint64_t seed, int32_t step, pasa_route_h route, void* stream) {
    if (route && route->cfg.prior != PASA_PRIOR_NONE)
        return fail(PASA_EINVAL, "this route handle has the Eq. 8 prior enabled: use pasa_route_v");
    return route_common(q, k, nullptr, budget, seed, step, route, stream);
}

pasa_status pasa_route_v(const pasa_tensor* q, const pasa_tensor* k, const pasa_tensor* v,
                         pasa_budget_h budget, uint64_t seed, int32_t step, pasa_route_h route,
                         void* stream) {
    if (route && route->cfg.prior == PASA_PRIOR_NONE)
        return fail(PASA_EINVAL, "pasa_route_v needs a handle with cfg.prior != PASA_PRIOR_NONE");
    if (!v) return fail(PASA_EINVAL, "v is NULL");
    return route_common(q, k, v, budget, seed, step, route, stream);
}

pasa_status pasa_attn_ex(const pasa_tensor* q, const pasa_tensor* k, const pasa_tensor* v,
                         pasa_route_h route, pasa_tensor* out, uint32_t flags, void* stream) {
    g_launches = 0;
    if (!route) return fail(PASA_EINVAL, "NULL route");
    pasa_status st;
    if ((st = check_tensor(q, "q")) != PASA_OK) return st;
    if ((st = check_tensor(k, "k")) != PASA_OK) return st;
    if ((st = check_tensor(v, "v")) != PASA_OK) return st;
    if ((st = check_tensor(out, "out")) != PASA_OK) return st;
    if (q->dtype != k->dtype || q->dtype != v->dtype || q->dtype != out->dtype)
        return fail(PASA_EDTYPE, "q, k, v, out dtypes differ");
    if ((st = match_route(q, route, "q")) != PASA_OK) return st;
    if ((st = match_route(k, route, "k")) != PASA_OK) return st;
    if ((st = match_route(v, route, "v")) != PASA_OK) return st;
    if ((st = match_route(out, route, "out")) != PASA_OK) return st;
    if (route->route_dtype < 0) return fail(PASA_EINVAL, "route was never built (call pasa_route)");
    if (flags & ~(PASA_ATTN_FORCE_SIMT | PASA_ATTN_STATS_ONLY | PASA_ATTN_REUSE_STATS |
                  PASA_ATTN_CTA_PAIR))
        return fail(PASA_EINVAL, "unknown pasa_attn_ex flags 0x%x", flags);
    if (route->cfg.qk_fp8 && (q->dtype != PASA_BF16 || (flags & PASA_ATTN_FORCE_SIMT) ||
                              !pasa::kv_stats_sm100_supported(route)))
        return fail(PASA_EUNSUPPORTED, "qk_fp8 runs only the bf16 tensor-core path");
    int launches = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (!(flags & PASA_ATTN_REUSE_STATS)) {
        cudaError_t e0 = pasa::launch_kv_stats(*k, *v, route, s, &launches);
        if (e0 != cudaSuccess) { g_launches = launches; return cuda_status(e0, "kv_stats launch"); }
        route->stats_dtype = q->dtype;
    } else if (route->stats_dtype != q->dtype) {
        return fail(PASA_EINVAL, "PASA_ATTN_REUSE_STATS without a matching STATS_ONLY call");
    }
    if ((flags & PASA_ATTN_CTA_PAIR) &&
        (q->dtype != PASA_BF16 || (flags & PASA_ATTN_FORCE_SIMT) ||
         !pasa::attn_sm100_cta2_supported(route))) {
        g_launches = launches;
        return fail(PASA_EUNSUPPORTED, "PASA_ATTN_CTA_PAIR: bf16, Bq = 256, d = 128, "
                    "G in {32, 64, k*128, >= N_K}, no FORCE_SIMT");
    }
    if (flags & PASA_ATTN_STATS_ONLY) { g_launches = launches; return PASA_OK; }
    cudaError_t e = cudaSuccess;
    // The tensor-core kernel covers bf16 I/O with Bq = 128 and G % 32 == 0 (or one
    // global group); fp32 I/O, Bq = 64 and finer groups run the CUDA-core kernel
    // (documented in include/pasa.h and DESIGN.md §7).
    const pasa_route_cfg& c = route->cfg;
    if (c.Bq == 256) {
        // Bq = 256 (NEXT 4 throughput variant) exists only as the tensor-core kernel
        if (q->dtype != PASA_BF16 || (flags & PASA_ATTN_FORCE_SIMT) ||
            !pasa::attn_sm100_q256_supported(route)) {
            g_launches = launches;
            return fail(PASA_EUNSUPPORTED, "Bq = 256 runs only the bf16 tensor-core kernel "
                        "(d 64 / 128, G in {32, 64, k*128, >= N_K}, no FORCE_SIMT)");
        }
        char why[256] = {0};
        cudaError_t e = (flags & PASA_ATTN_CTA_PAIR)
                            ? pasa::launch_attn_sm100_cta2(*q, *k, *v, route, *out, s, &launches, why,
                                                           sizeof(why))
                            : pasa::launch_attn_sm100_q256(*q, *k, *v, route, *out, s, &launches, why,
                                                           sizeof(why));
        g_launches = launches;
        if (e == cudaErrorNotSupported) return fail(PASA_EUNSUPPORTED, "tcgen05 attention: %s", why);
        return cuda_status(e, "attention launch");
    }
    const bool fine_groups = c.comp == PASA_COMP_GROUPED && !pasa::sm100_supports_group(c.G, route->NK);
    const bool simt = q->dtype == PASA_F32 || (flags & PASA_ATTN_FORCE_SIMT) || c.Bq != 128 ||
                      fine_groups;

    if (simt) {
        e = pasa::launch_attn_simt(*q, *k, *v, route, *out, s, &launches);
    } else {
        char why[256] = {0};
        e = pasa::launch_attn_sm100(*q, *k, *v, route, *out, s, &launches, why, sizeof(why));
        if (e == cudaErrorNotSupported) {
            g_launches = launches;
            return fail(PASA_EUNSUPPORTED, "tcgen05 attention: %s", why);
        }
    }
    g_launches = launches;
    return cuda_status(e, "attention launch");
}

pasa_status pasa_attn(const pasa_tensor* q, const pasa_tensor* k, const pasa_tensor* v,
                      pasa_route_h route, pasa_tensor* out, void* stream) {
    return pasa_attn_ex(q, k, v, route, out, 0u, stream);
}

namespace {
pasa_status check_shards(const pasa_shards* t, const pasa_route_s* r, const char* name,
                         pasa::ZcShards* out) {
    if (!t) return fail(PASA_EINVAL, "%s is NULL", name);
    if (t->dtype != PASA_BF16) return fail(PASA_EDTYPE, "%s: zero-copy path is bf16 only", name);
    if (t->nshards < 1 || t->nshards > 8) return fail(PASA_EINVAL, "%s: nshards %d not in 1..8", name, t->nshards);
    if (t->S != r->S || t->D != r->D) return fail(PASA_ESHAPE, "%s: S, D differ from the route", name);
    if (r->cfg.head_offset < 0 || r->cfg.head_offset + r->H > t->H)
        return fail(PASA_EINVAL, "%s: route heads [%lld, %lld) outside the shards' H = %lld", name,
                    (long long)r->cfg.head_offset, (long long)(r->cfg.head_offset + r->H), (long long)t->H);
    if (t->start[0] != 0 || t->start[t->nshards] != t->S)
        return fail(PASA_EINVAL, "%s: start[0] must be 0 and start[nshards] = S", name);
    for (int s = 0; s < t->nshards; ++s) {
        if (t->start[s + 1] <= t->start[s]) return fail(PASA_EINVAL, "%s: empty or unordered shard %d", name, s);
        if (!t->data[s] || (reinterpret_cast<uintptr_t>(t->data[s]) & 15))
            return fail(PASA_EINVAL, "%s: shard %d base NULL or not 16-byte aligned", name, s);
    }
    if ((t->sS & 7) || (t->sH & 7) || t->sS <= 0 || t->sH <= 0)
        return fail(PASA_EINVAL, "%s: strides must be positive multiples of 8 elements", name);
    out->P = t->nshards;
    for (int s = 0; s <= t->nshards; ++s) out->start[s] = t->start[s];
    for (int s = 0; s < t->nshards; ++s) out->base[s] = t->data[s];
    out->sS = t->sS;
    out->sH = t->sH;
    return PASA_OK;
}
}  // namespace

pasa_status pasa_route_zc(const pasa_shards* q, const pasa_shards* k, const pasa_shards* v,
                          pasa_budget_h budget, uint64_t seed, int32_t step, pasa_route_h route,
                          const pasa_tensor* q_loc, const pasa_tensor* k_loc,
                          const pasa_tensor* v_loc, void* stream) {
    g_launches = 0;
    if (!route || !budget) return fail(PASA_EINVAL, "NULL handle");
    if (route->cfg.prior != PASA_PRIOR_NONE || route->cfg.qk_fp8)
        return fail(PASA_EUNSUPPORTED, "pasa_route_zc: no Eq. 8 prior / FP8 QK^T handles");
    if (route->B != 1) return fail(PASA_ESHAPE, "pasa_route_zc: B must be 1");
    pasa::ZcShards sh[3];
    pasa_status st;
    if ((st = check_shards(q, route, "q", &sh[0])) != PASA_OK) return st;
    if ((st = check_shards(k, route, "k", &sh[1])) != PASA_OK) return st;
    if ((st = check_shards(v, route, "v", &sh[2])) != PASA_OK) return st;
    const pasa_tensor* loc[3] = {q_loc, k_loc, v_loc};
    const char* nm[3] = {"q_loc", "k_loc", "v_loc"};
    pasa_tensor lt[3];
    for (int x = 0; x < 3; ++x) {
        if ((st = check_tensor(loc[x], nm[x])) != PASA_OK) return st;
        if (loc[x]->dtype != PASA_BF16) return fail(PASA_EDTYPE, "%s must be bf16", nm[x]);
        if ((st = match_route(loc[x], route, nm[x])) != PASA_OK) return st;
        lt[x] = *loc[x];
    }
    int launches = 0;
    cudaError_t e = pasa::launch_route_zc(sh, lt, budget, seed, step, route, (cudaStream_t)stream,
                                          &launches);
    g_launches = launches;
    if (e == cudaSuccess) {
        route->route_dtype = PASA_BF16;
        route->stats_dtype = -1;
        route->het_valid = 0;
    }
    return cuda_status(e, "pasa_route_zc launch");
}

pasa_status pasa_attn_zc(const pasa_tensor* q_loc, const pasa_tensor* k_loc,
                         const pasa_tensor* v_loc, pasa_route_h route, const pasa_shards* out,
                         void* stream) {
    g_launches = 0;
    if (!route) return fail(PASA_EINVAL, "NULL route");
    pasa_status st;
    pasa::ZcShards osh;
    if ((st = check_shards(out, route, "out", &osh)) != PASA_OK) return st;
    if ((st = check_tensor(q_loc, "q_loc")) != PASA_OK) return st;
    if ((st = check_tensor(k_loc, "k_loc")) != PASA_OK) return st;
    if ((st = check_tensor(v_loc, "v_loc")) != PASA_OK) return st;
    if (q_loc->dtype != PASA_BF16 || k_loc->dtype != PASA_BF16 || v_loc->dtype != PASA_BF16)
        return fail(PASA_EDTYPE, "pasa_attn_zc is bf16 only");
    if ((st = match_route(q_loc, route, "q_loc")) != PASA_OK) return st;
    if ((st = match_route(k_loc, route, "k_loc")) != PASA_OK) return st;
    if ((st = match_route(v_loc, route, "v_loc")) != PASA_OK) return st;
    if (route->route_dtype < 0) return fail(PASA_EINVAL, "route was never built (call pasa_route_zc)");
    const pasa_route_cfg& c = route->cfg;
    if (c.Bq != 128 || c.qk_fp8 ||
        (c.comp == PASA_COMP_GROUPED && !pasa::sm100_supports_group(c.G, route->NK)))
        return fail(PASA_EUNSUPPORTED, "pasa_attn_zc: the tensor-core kernel's domain only");
    int launches = 0;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = pasa::launch_kv_stats(*k_loc, *v_loc, route, s, &launches);
    if (e != cudaSuccess) { g_launches = launches; return cuda_status(e, "kv_stats launch"); }
    route->stats_dtype = PASA_BF16;
    char why[256] = {0};
    // the `out` argument is only a shape carrier here: with output shards every row the
    // kernel stores goes to its owner's shard (rows past S are never stored)
    e = pasa::launch_attn_sm100(*q_loc, *k_loc, *v_loc, route, *q_loc, s, &launches, why,
                                sizeof(why), &osh);
    g_launches = launches;
    if (e == cudaErrorNotSupported) return fail(PASA_EUNSUPPORTED, "tcgen05 attention: %s", why);
    return cuda_status(e, "pasa_attn_zc launch");
}

pasa_status pasa_budget_read(pasa_budget_h budget, double out[5], void* stream) {
    if (!budget || !out) return fail(PASA_EINVAL, "NULL argument");
    pasa::BudgetRec rec;
    cudaError_t e = cudaMemcpyAsync(&rec, budget->rec, sizeof(rec), cudaMemcpyDeviceToHost,
                                    (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "pasa_budget_read");
    out[0] = rec.l1; out[1] = rec.alpha; out[2] = rec.rho_t; out[3] = rec.dense; out[4] = rec.clipped;
    return PASA_OK;
}

pasa_status pasa_route_read(pasa_route_h r, int32_t* k, int32_t* idx, int32_t* count,
                            uint32_t* mask, void* stream) {
    if (!r) return fail(PASA_EINVAL, "NULL route");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (k && e == cudaSuccess) e = cudaMemcpyAsync(k, r->hdr, 4, cudaMemcpyDeviceToHost, s);
    if (idx && e == cudaSuccess)
        e = cudaMemcpyAsync(idx, r->idx, sizeof(int32_t) * r->BH * r->NQ * r->NK,
                            cudaMemcpyDeviceToHost, s);
    if (count && e == cudaSuccess)
        e = cudaMemcpyAsync(count, r->count, sizeof(int32_t) * r->BH * r->NQ,
                            cudaMemcpyDeviceToHost, s);
    if (mask && e == cudaSuccess)
        e = cudaMemcpyAsync(mask, r->mask, sizeof(uint32_t) * r->BH * r->NQ * r->W,
                            cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return cuda_status(e, "pasa_route_read");
}

pasa_status pasa_route_pooled_read(pasa_route_h r, double* qbar, double* kbar, void* stream) {
    if (!r) return fail(PASA_EINVAL, "NULL route");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (qbar) e = cudaMemcpyAsync(qbar, r->qbar, sizeof(double) * r->BH * r->NQ * r->D,
                                  cudaMemcpyDeviceToHost, s);
    if (kbar && e == cudaSuccess)
        e = cudaMemcpyAsync(kbar, r->kbar, sizeof(double) * r->BH * r->NK * r->D,
                            cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return cuda_status(e, "pasa_route_pooled_read");
}

pasa_status pasa_attn_stats_read(pasa_route_h r, void* kbar, void* vsum, void* ht, int32_t dtype,
                                 void* stream) {
    if (!r) return fail(PASA_EINVAL, "NULL route");
    if (r->stats_dtype < 0) return fail(PASA_EINVAL, "no statistics pass has run on this route");
    // the host buffers were sized for `dtype`: refuse to write wider elements into them
    if (dtype != r->stats_dtype)
        return fail(PASA_EDTYPE, "statistics are stored as dtype %d, buffers declared as %d",
                    r->stats_dtype, dtype);
    const size_t es = r->stats_dtype == PASA_F32 ? 4 : 2;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (kbar) e = cudaMemcpyAsync(kbar, r->kbar_lp, es * r->BH * r->NK * r->D, cudaMemcpyDeviceToHost, s);
    if (vsum && e == cudaSuccess)
        e = cudaMemcpyAsync(vsum, r->vsum_lp, es * r->BH * r->NK * r->D, cudaMemcpyDeviceToHost, s);
    if (ht && e == cudaSuccess)
        e = cudaMemcpyAsync(ht, r->ht, es * r->BH * r->NG * r->D * r->D, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return cuda_status(e, "pasa_attn_stats_read");
}

pasa_status pasa_route_het_read(pasa_route_h r, double* het, void* stream) {
    if (!r || !het) return fail(PASA_EINVAL, "NULL argument");
    if (r->cfg.prior == PASA_PRIOR_NONE || !r->het_valid)
        return fail(PASA_EINVAL, "no heterogeneity prior has been computed on this route");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(het, r->het, sizeof(double) * r->BH * r->NK,
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return cuda_status(e, "pasa_route_het_read");
}

pasa_status pasa_route_dims(pasa_route_h r, int64_t dims[7]) {
    if (!r || !dims) return fail(PASA_EINVAL, "NULL argument");
    dims[0] = r->B; dims[1] = r->S; dims[2] = r->H; dims[3] = r->D;
    dims[4] = r->NQ; dims[5] = r->NK; dims[6] = r->NG;
    return PASA_OK;
}

}  // extern "C"
