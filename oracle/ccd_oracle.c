/*
 * ccd_oracle.c -- TEST INFRASTRUCTURE ONLY (see ccd_oracle.h).
 *
 * Plain-C restatement of the reference CCD path, statement order kept so
 * that the floating-point results are the reference's bit for bit (compiled
 * with -ffp-contract=off, like the reference's x86-64 build which has no FMA
 * contraction).  Citations are relative to /root/reference/proj/include/bsccs/.
 */
#include "ccd_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

const char* or_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* engine.hpp:56-65 check_xbeta_magnitude; bound 700 for double (:20-23) */
static int check_xbeta(double v) {
    if (!(fabs(v) <= 700.0)) {
        snprintf(g_err, sizeof g_err,
                 "linear predictor overflow: |x'beta| reached %f (bound 700); the fit has diverged",
                 fabs(v));
        return OR_NUMERIC;
    }
    return OR_OK;
}

/* engine.hpp:68-90 refresh_from_xbeta */
static int refresh_from_xbeta(const or_dataset* ds, or_state* st) {
    double max_abs = 0.0;
    for (int64_t k = 0; k < ds->K; ++k) {
        const double a = fabs(st->xbeta[k]);
        max_abs = max_abs < a ? a : max_abs; /* std::max(max_abs, |v|) */
    }
    int rc = check_xbeta(max_abs);
    if (rc) return rc;
    for (int64_t k = 0; k < ds->K; ++k)
        st->l_exp_xbeta[k] = (double)ds->era_lengths[k] * exp(st->xbeta[k]);
    for (int64_t i = 0; i < ds->N; ++i) {
        double total = 0.0;
        for (int32_t k = ds->subject_offsets[i]; k < ds->subject_offsets[i + 1]; ++k)
            total += st->l_exp_xbeta[k];
        st->denominators[i] = total;
    }
    return OR_OK;
}

/* engine.hpp:155-163 / 173-181: xbeta = sum over j ascending of beta_j */
static void rebuild_xbeta(const or_dataset* ds, or_state* st) {
    memset(st->xbeta, 0, sizeof(double) * (size_t)ds->K);
    for (int32_t j = 0; j < ds->J; ++j) {
        const double bj = st->beta[j];
        if (bj == 0.0) continue;
        for (int64_t p = ds->col_ptr[j]; p < ds->col_ptr[j + 1]; ++p)
            st->xbeta[ds->rows[p]] += bj;
    }
}

/* engine.hpp:137-166 init_state */
int or_init_state(const or_dataset* ds, const double* beta, or_state* st) {
    for (int32_t j = 0; j < ds->J; ++j) {
        if (beta && !isfinite(beta[j])) return fail(OR_INPUT, "init_state: non-finite coefficient");
        st->beta[j] = beta ? beta[j] : 0.0;
    }
    rebuild_xbeta(ds, st);
    return refresh_from_xbeta(ds, st);
}

/* engine.hpp:170-183 dense_recompute */
int or_dense_recompute(const or_dataset* ds, or_state* st) {
    rebuild_xbeta(ds, st);
    return refresh_from_xbeta(ds, st);
}

/* engine.hpp:97-132 reduce_column_range + :285-298 fused_grad_hess */
int or_grad_hess(const or_dataset* ds, const or_state* st, int32_t j, double* g, double* h) {
    double gs = 0.0, hs = 0.0;
    int64_t p = ds->col_ptr[j];
    const int64_t hi = ds->col_ptr[j + 1];
    while (p < hi) {
        const int32_t i = ds->subjects[p];
        double numerator = 0.0;
        do {
            numerator += st->l_exp_xbeta[ds->rows[p]];
            ++p;
        } while (p < hi && ds->subjects[p] == i);
        const double den = st->denominators[i];
        if (!(den > 0.0)) return fail(OR_INTERNAL, "fused reduction: nonpositive subject denominator");
        double w = numerator / den;
        if (w > 1.0) w = 1.0;
        const double nw = (double)ds->events_per_subject[i] * w;
        gs += nw;
        hs += nw * (1.0 - w);
    }
    *g = (double)ds->y_dot_x[j] - gs;
    *h = hs == 0.0 ? 0.0 : -hs;
    return OR_OK;
}

/* engine.hpp:205-231 sparse_delta_update */
int or_sparse_update(const or_dataset* ds, or_state* st, int32_t j, double delta) {
    if (!isfinite(delta)) return fail(OR_NUMERIC, "sparse_delta_update: non-finite step");
    if (delta == 0.0) return OR_OK;
    for (int64_t p = ds->col_ptr[j]; p < ds->col_ptr[j + 1]; ++p) {
        const int32_t k = ds->rows[p];
        const double updated = st->xbeta[k] + delta;
        int rc = check_xbeta(updated);
        if (rc) return rc;
        st->xbeta[k] = updated;
        const double fresh = (double)ds->era_lengths[k] * exp(updated);
        st->denominators[ds->subjects[p]] += fresh - st->l_exp_xbeta[k];
        st->l_exp_xbeta[k] = fresh;
    }
    st->beta[j] += delta;
    return OR_OK;
}

/* engine.hpp:404-425 log_likelihood */
int or_log_likelihood(const or_dataset* ds, const or_state* st, double* out) {
    double linear = 0.0;
    for (int64_t k = 0; k < ds->K; ++k)
        if (ds->event_counts[k] != 0) linear += (double)ds->event_counts[k] * st->xbeta[k];
    double logden = 0.0;
    for (int64_t i = 0; i < ds->N; ++i) {
        const double den = st->denominators[i];
        if (!(den > 0.0)) return fail(OR_INTERNAL, "log_likelihood: nonpositive subject denominator");
        logden += (double)ds->events_per_subject[i] * log(den);
    }
    *out = linear - logden;
    return OR_OK;
}

/* prior.hpp:22-24 laplace_scale */
static double laplace_scale(const or_prior* p) {
    return p->variance_is_laplace_scale ? p->variance : sqrt(p->variance / 2.0);
}

/* prior.hpp:27-32 validate_prior */
static int validate_prior(const or_prior* p) {
    if (p->kind != 0 && !(p->variance > 0.0 && isfinite(p->variance)))
        return fail(OR_INPUT, "prior variance must be positive and finite");
    return OR_OK;
}

/* prior.hpp:36-61 log_density */
int or_log_density(const or_prior* prior, const double* beta, int32_t n, double* out) {
    int rc = validate_prior(prior);
    if (rc) return rc;
    if (prior->kind == 0) {
        *out = 0.0;
    } else if (prior->kind == 1) {
        const double v = prior->variance;
        double ss = 0.0;
        for (int32_t j = 0; j < n; ++j) ss += beta[j] * beta[j];
        *out = -0.5 * ss / v - 0.5 * (double)n * log(6.283185307179586 * v);
    } else {
        const double b = laplace_scale(prior);
        double abs_sum = 0.0;
        for (int32_t j = 0; j < n; ++j) abs_sum += fabs(beta[j]);
        *out = -abs_sum / b - (double)n * log(2.0 * b);
    }
    return OR_OK;
}

/* prior.hpp:72-122 penalized_step */
int or_penalized_step(const or_prior* prior, double beta_j, double g, double h, double* out) {
    if (h > 0.0) return fail(OR_INTERNAL, "penalized_step: positive likelihood curvature");
    if (prior->kind == 0) {
        if (h == 0.0) {
            if (g == 0.0) { *out = 0.0; return OR_OK; }
            return fail(OR_NUMERIC, "undefined Newton step: flat likelihood direction with no prior");
        }
        *out = -g / h;
        return OR_OK;
    }
    if (prior->kind == 1) {
        const double v = prior->variance;
        *out = -(g - beta_j / v) / (h - 1.0 / v);
        return OR_OK;
    }
    const double b = laplace_scale(prior);
    if (beta_j != 0.0) {
        if (h == 0.0) { *out = -beta_j; return OR_OK; }
        const double sign = beta_j > 0.0 ? 1.0 : -1.0;
        const double step = -(g - sign / b) / h;
        const double landed = beta_j + step;
        if ((beta_j > 0.0 && landed < 0.0) || (beta_j < 0.0 && landed > 0.0)) { *out = -beta_j; return OR_OK; }
        *out = step;
        return OR_OK;
    }
    if (h == 0.0) { *out = 0.0; return OR_OK; }
    double step = -(g - 1.0 / b) / h;
    if (step > 0.0) { *out = step; return OR_OK; }
    step = -(g + 1.0 / b) / h;
    if (step < 0.0) { *out = step; return OR_OK; }
    *out = 0.0;
    return OR_OK;
}

/* rng.hpp:12-54 xoshiro256** (SolverState::order_rng, solver.hpp:81) */
static uint64_t sm64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static void rng_seed(uint64_t st[4], uint64_t seed, uint64_t stream) {
    uint64_t a = seed, b = ~stream;
    for (int i = 0; i < 4; ++i) st[i] = sm64(&a) ^ sm64(&b);
    if ((st[0] | st[1] | st[2] | st[3]) == 0) st[0] = 0x9E3779B97F4A7C15ull;
}
static uint64_t rng_next(uint64_t s[4]) {
    const uint64_t out = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
}
/* rng.hpp:67-77 below */
static uint64_t rng_below(uint64_t s[4], uint64_t n) {
    uint64_t x, r;
    do { x = rng_next(s); r = x % n; } while (x - r > (uint64_t)0 - n);
    return r;
}

/* solver.hpp:101-166 run_cycle (sparse path) */
int or_run_cycle(const or_dataset* ds, or_state* st, const or_prior* prior,
                 const or_config* cfg, double* trust, int32_t* order,
                 uint64_t rng_state[4], double* snapshot, double* criterion,
                 int64_t* visited) {
    memcpy(snapshot, st->xbeta, sizeof(double) * (size_t)ds->K); /* :108 */
    if (cfg->random_cycle && order) {                             /* :109-114 */
        for (int64_t j = ds->J; j > 1; --j) {
            const int64_t r = (int64_t)rng_below(rng_state, (uint64_t)j);
            const int32_t tmp = order[j - 1];
            order[j - 1] = order[r];
            order[r] = tmp;
        }
    }
    for (int32_t idx = 0; idx < ds->J; ++idx) {
        const int32_t j = order ? order[idx] : idx;
        if (ds->col_ptr[j + 1] == ds->col_ptr[j] && st->beta[j] == 0.0) continue; /* :119-121 */
        if (visited) ++*visited;
        double g, h, unbounded;
        int rc = or_grad_hess(ds, st, j, &g, &h);
        if (rc) return rc;
        rc = or_penalized_step(prior, st->beta[j], g, h, &unbounded);
        if (rc) return rc;
        const double radius = trust[j];
        /* std::clamp(v, lo, hi): v < lo ? lo : (hi < v ? hi : v) */
        const double delta = unbounded < -radius ? -radius : (radius < unbounded ? radius : unbounded);
        if (delta != 0.0) {
            rc = or_sparse_update(ds, st, j, delta);
            if (rc) return rc;
        }
        const double twice = 2.0 * fabs(delta), half = radius / 2.0;
        trust[j] = twice < half ? half : twice; /* std::max(2|d|, r/2) :150 */
    }
    double change = 0.0, magnitude = 0.0; /* :154-165 */
    for (int64_t k = 0; k < ds->K; ++k) {
        change += fabs(st->xbeta[k] - snapshot[k]);
        if (cfg->normalized) magnitude += fabs(st->xbeta[k]);
    }
    *criterion = cfg->normalized ? change / (1.0 + magnitude) : change;
    return OR_OK;
}

/* solver.hpp:170-199 fit_impl<double> + :206-220 fit */
int or_fit(const or_dataset* ds, const or_prior* prior, const or_config* cfg,
           const double* init_beta, double* beta_out, or_result* res) {
    /* solver.hpp:48-64 validate_config (subset exposed here) */
    if (!(cfg->epsilon > 0.0) || !isfinite(cfg->epsilon)) return fail(OR_INPUT, "solver: epsilon must be positive and finite");
    if (cfg->max_cycles < 1) return fail(OR_INPUT, "solver: max_cycles must be at least 1");
    if (!(cfg->trust_init > 0.0) || !isfinite(cfg->trust_init)) return fail(OR_INPUT, "solver: trust region width must be positive and finite");
    if (cfg->dense_refresh_interval < 1) return fail(OR_INPUT, "solver: dense refresh interval must be at least 1");
    int rc = validate_prior(prior);
    if (rc) return rc;
    if (ds->N == 0) return fail(OR_INPUT, "fit: dataset has no subjects");

    or_state st;
    st.beta = beta_out;
    st.xbeta = (double*)malloc(sizeof(double) * (size_t)ds->K);
    st.l_exp_xbeta = (double*)malloc(sizeof(double) * (size_t)ds->K);
    st.denominators = (double*)malloc(sizeof(double) * (size_t)ds->N);
    double* snap = (double*)malloc(sizeof(double) * (size_t)ds->K);
    double* trust = (double*)malloc(sizeof(double) * (size_t)ds->J);
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)ds->J);
    uint64_t rng[4];
    rng_seed(rng, cfg->cycle_seed, 0);
    for (int32_t j = 0; j < ds->J; ++j) { trust[j] = cfg->trust_init; order[j] = j; }
    res->cycles_run = 0;
    res->converged = 0;
    res->final_criterion = INFINITY;
    res->log_posterior = -INFINITY;
    res->coordinates_visited = 0;

    rc = or_init_state(ds, init_beta, &st);
    while (rc == OR_OK && res->cycles_run < cfg->max_cycles) {
        rc = or_run_cycle(ds, &st, prior, cfg, trust, order, rng, snap, &res->final_criterion,
                          &res->coordinates_visited);
        if (rc) break;
        ++res->cycles_run;
        if (res->final_criterion <= cfg->epsilon) { res->converged = 1; break; }
        if (res->cycles_run % cfg->dense_refresh_interval == 0) rc = or_dense_recompute(ds, &st);
    }
    if (rc == OR_OK) rc = or_dense_recompute(ds, &st);
    double ll = 0.0, lp = 0.0;
    if (rc == OR_OK) rc = or_log_likelihood(ds, &st, &ll);
    if (rc == OR_OK) rc = or_log_density(prior, st.beta, ds->J, &lp);
    if (rc == OR_OK) res->log_posterior = ll + lp;
    free(st.xbeta); free(st.l_exp_xbeta); free(st.denominators);
    free(snap); free(trust); free(order);
    return rc;
}
