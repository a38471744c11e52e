// drivers.cpp -- the callers of fit() on the many-fit side of the hot path:
// grid_search_cv (cross_validation.hpp:100-215) and run_bootstrap
// (bootstrap.hpp:79-158), over a device-resident dataset.
//
// Two engines (include/bsccs_b200.h):
//   SUBSET   the reference's own route -- each fold / replicate dataset is
//            materialised on the device (subset.cu) and fitted by the
//            single-fit persistent kernel;
//   BATCHED  R fits at once on the parent dataset with per-subject weights
//            (batch.cu); see DESIGN.md §4.4.
// The host logic (fold construction, warm-start chains, cell validity,
// selection, percentile summaries) restates the reference line by line.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <vector>

#include "devutil.h"
#include "engine.h"

namespace bsccs_b200 {

namespace {

// A dataset built here (subset) with its fit workspaces released on scope exit.
struct OwnedDataset {
    bsccs_dataset* ds = nullptr;
    explicit OwnedDataset(bsccs_dataset* d) : ds(d) {}
    OwnedDataset(const OwnedDataset&) = delete;
    OwnedDataset& operator=(const OwnedDataset&) = delete;
    ~OwnedDataset() {
        if (ds) {
            release_dataset_workspaces(ds);
            dataset_destroy(ds);
        }
    }
};

// predictive_log_likelihood (cross_validation.hpp:89-93): init_state on the
// held-out data at beta, then log_likelihood.
double predictive_ll(const bsccs_dataset* held, const double* beta) {
    bsccs_state* st = state_create(held, beta);
    double ll = 0.0;
    try {
        ll = log_likelihood(st);
    } catch (...) {
        state_destroy(st);
        throw;
    }
    state_destroy(st);
    return ll;
}

// The fold's training and held-out subject lists (cross_validation.hpp:127-144).
void fold_lists(const std::vector<int32_t>& all, const std::vector<int32_t>& sizes, int32_t f, int32_t N,
                std::vector<int32_t>& held, std::vector<int32_t>& rest) {
    int64_t start = 0;
    for (int32_t i = 0; i < f; ++i) start += sizes[static_cast<size_t>(i)];
    held.assign(all.begin() + start, all.begin() + start + sizes[static_cast<size_t>(f)]);
    std::sort(held.begin(), held.end());
    rest.clear();
    rest.reserve(static_cast<size_t>(N) - held.size());
    size_t next = 0;
    for (int32_t i = 0; i < N; ++i) {
        if (next < held.size() && held[next] == i) ++next;
        else rest.push_back(i);
    }
}

bool cell_failure(const Error& e) { return e.code != BSCCS_INPUT_ERROR && e.code != BSCCS_CUDA_ERROR; }

void validate_cv(const bsccs_cv_config* cfg, const double* grid, int32_t points) {
    if (!cfg) input_error("null cross-validation config");
    if (points < 1 || !grid) input_error("cross-validation grid is empty");
    for (int32_t g = 0; g < points; ++g)
        if (!(grid[g] > 0.0) || !std::isfinite(grid[g])) input_error("cross-validation grid values must be positive");
    validate_config(&cfg->solver);
    if (cfg->engine != BSCCS_ENGINE_SUBSET && cfg->engine != BSCCS_ENGINE_BATCHED)
        input_error("cross-validation: unknown engine");
}

std::vector<double> sorted_grid(const double* grid, int32_t points) {
    std::vector<double> g(grid, grid + points);
    std::sort(g.begin(), g.end());
    for (size_t i = 1; i < g.size(); ++i)
        if (g[i] == g[i - 1]) input_error("cross-validation grid has a repeated value");
    return g;
}

void cv_folds(const bsccs_dataset* ds, const bsccs_cv_config* cfg, const std::vector<double>& grid, int32_t f0,
              int32_t f1, bsccs_cv_cell* cells, bsccs_cv_result* res) {
    const int32_t folds = cfg->folds;
    const int32_t points = static_cast<int32_t>(grid.size());
    std::vector<int32_t> all(static_cast<size_t>(ds->N)), sizes(static_cast<size_t>(std::max(folds, 0)));
    kfold_split(ds->N, folds, cfg->seed, all.data(), sizes.data());
    if (f0 < 0 || f1 > folds || f0 > f1) input_error("cross-validation: fold range out of bounds");
    // the batched engine runs the sparse update path; dense-route configs
    // (UpdatePath::dense) take the materialised route
    if (cfg->engine == BSCCS_ENGINE_BATCHED && cfg->solver.path == 0) {
        cv_folds_batched(ds, cfg, grid, all, sizes, f0, f1, cells, res);
        return;
    }
    const int32_t J = ds->J;
    std::vector<int32_t> held, rest;
    std::vector<double> beta(static_cast<size_t>(J)), carried;
    for (int32_t f = f0; f < f1; ++f) {
        fold_lists(all, sizes, f, ds->N, held, rest);
        OwnedDataset train(dataset_subset(ds, rest.data(), static_cast<int64_t>(rest.size()), ds->ctas));
        OwnedDataset hold(dataset_subset(ds, held.data(), static_cast<int64_t>(held.size()), ds->ctas));
        carried.clear();
        for (int32_t g = 0; g < points; ++g) {
            bsccs_prior pr{cfg->prior_kind, cfg->variance_is_laplace_scale, grid[static_cast<size_t>(g)]};
            const PriorParams p = to_params(&pr);
            bsccs_cv_cell& cell = cells[static_cast<size_t>(g) * folds + f];
            cell = bsccs_cv_cell{-std::numeric_limits<double>::infinity(), 0, 0, 0, 0};
            try {
                bsccs_fit_result fr;
                fit_resident(train.ds, p, &cfg->solver, (cfg->warm_start && !carried.empty()) ? carried.data() : nullptr,
                             beta.data(), &fr);
                cell.cycles = fr.cycles_run;
                cell.converged = fr.converged;
                res->fits += 1;
                res->coordinates_visited += fr.coordinates_visited;
                res->device_seconds += fr.device_seconds;
                cell.predictive_ll = predictive_ll(hold.ds, beta.data());
                cell.valid = 1;
                if (cfg->warm_start) carried = beta;
            } catch (const Error& e) {
                if (!cell_failure(e)) throw;
                cell.valid = 0;
            }
        }
    }
}

void cv_select(const std::vector<double>& grid, int32_t folds, const bsccs_cv_cell* cells, double* mean_out,
               bsccs_cv_result* res) {
    const int32_t points = static_cast<int32_t>(grid.size());
    res->points = points;
    res->selected_index = -1;
    res->total_cycles = 0;
    double best = -std::numeric_limits<double>::infinity();
    for (int32_t g = 0; g < points; ++g) {
        double total = 0.0;
        bool usable = true;
        if (mean_out) mean_out[g] = std::numeric_limits<double>::quiet_NaN();
        for (int32_t f = 0; f < folds; ++f) {
            const bsccs_cv_cell& cell = cells[static_cast<size_t>(g) * folds + f];
            res->total_cycles += cell.cycles;
            if (!cell.valid) usable = false;
            else total += cell.predictive_ll;
        }
        if (!usable) continue;
        const double mean = total / static_cast<double>(folds);
        if (mean_out) mean_out[g] = mean;
        // first maximum wins: an equal mean later in the grid never replaces it
        if (mean > best) {
            best = mean;
            res->selected_index = g;
        }
    }
    if (res->selected_index < 0) fail(BSCCS_CONVERGENCE_ERROR, "cross-validation: every grid point failed in some fold");
    res->selected_variance = grid[static_cast<size_t>(res->selected_index)];
}

// ---- bootstrap ----------------------------------------------------------

void validate_bootstrap(const bsccs_bootstrap_config* cfg) {
    if (!cfg) input_error("null bootstrap config");
    if (cfg->replicates < 1) input_error("bootstrap: need at least one replicate");
    if (!(cfg->level > 0.0 && cfg->level < 1.0)) input_error("bootstrap: interval level must lie in (0, 1)");
    validate_config(&cfg->solver);
    (void)to_params(&cfg->prior);
    if (cfg->engine != BSCCS_ENGINE_SUBSET && cfg->engine != BSCCS_ENGINE_BATCHED)
        input_error("bootstrap: unknown engine");
}

void boot_replicates(const bsccs_dataset* ds, const bsccs_bootstrap_config* cfg, const double* beta_full, int32_t r0,
                     int32_t r1, double* est, int32_t* conv, bsccs_bootstrap_result* res) {
    if (r0 < 0 || r1 < r0) input_error("bootstrap: replicate range out of bounds");
    if (cfg->engine == BSCCS_ENGINE_BATCHED && cfg->solver.path == 0) {
        boot_replicates_batched(ds, cfg, beta_full, r0, r1, est, conv, res);
        return;
    }
    const PriorParams p = to_params(&cfg->prior);
    const int32_t J = ds->J;
    std::vector<int32_t> idx(static_cast<size_t>(ds->N));
    for (int32_t r = r0; r < r1; ++r) {
        resample(ds->N, cfg->seed, static_cast<uint64_t>(r) + 1, idx.data());
        OwnedDataset rs(dataset_subset(ds, idx.data(), static_cast<int64_t>(idx.size()), ds->ctas));
        bsccs_fit_result fr;
        double* out = est + static_cast<size_t>(r - r0) * J;
        fit_resident(rs.ds, p, &cfg->solver, cfg->warm_start ? beta_full : nullptr, out, &fr);
        conv[r - r0] = fr.converged;
        res->total_cycles += fr.cycles_run;
        res->coordinates_visited += fr.coordinates_visited;
        res->device_seconds += fr.device_seconds;
    }
}

// detail::percentile (bootstrap.hpp:55-68)
double percentile(const std::vector<double>& sorted, double q) {
    const size_t m = sorted.size();
    if (m == 1) return sorted[0];
    const double pos = q * static_cast<double>(m - 1);
    const size_t lo = static_cast<size_t>(pos);
    if (lo + 1 >= m) return sorted[m - 1];
    const double frac = pos - static_cast<double>(lo);
    return sorted[lo] + frac * (sorted[lo + 1] - sorted[lo]);
}

void boot_summarize(int32_t J, int32_t reps, double level, const double* est, const int32_t* conv, double* lower,
                    double* upper, double* p_hat, bsccs_bootstrap_result* res) {
    res->replicates = reps;
    res->used = 0;
    res->non_converged = 0;
    for (int32_t r = 0; r < reps; ++r) {
        if (conv[r]) ++res->used;
        else ++res->non_converged;
    }
    if (res->used == 0) fail(BSCCS_CONVERGENCE_ERROR, "bootstrap: no replicate converged");
    const double tail = (1.0 - level) / 2.0;
    std::vector<double> column;
    column.reserve(static_cast<size_t>(res->used));
    for (int32_t j = 0; j < J; ++j) {
        column.clear();
        int nonzero = 0;
        for (int32_t r = 0; r < reps; ++r) {
            if (!conv[r]) continue;
            const double b = est[static_cast<size_t>(r) * J + j];
            column.push_back(b);
            if (b != 0.0) ++nonzero;
        }
        std::sort(column.begin(), column.end());
        lower[j] = percentile(column, tail);
        upper[j] = percentile(column, 1.0 - tail);
        p_hat[j] = static_cast<double>(nonzero) / static_cast<double>(res->used);
    }
}

} // namespace
} // namespace bsccs_b200

using namespace bsccs_b200;

extern "C" {

void bsccs_cv_config_default(bsccs_cv_config* c) {
    std::memset(c, 0, sizeof *c);
    c->folds = 10;
    c->prior_kind = PRIOR_LAPLACE;
    c->variance_is_laplace_scale = 0;
    c->warm_start = 1;
    c->seed = 0;
    bsccs_solver_config_default(&c->solver);
    c->engine = BSCCS_ENGINE_SUBSET;
    c->batch = 0;
}

void bsccs_default_variance_grid(double out[13]) {
    const double lo = std::log(0.001), hi = std::log(10.0);
    for (int g = 0; g < 13; ++g) out[g] = std::exp(lo + (hi - lo) * static_cast<double>(g) / 12.0);
}

bsccs_status bsccs_cv_run_folds(const bsccs_dataset* ds, const bsccs_cv_config* cfg, const double* variance_grid,
                                int32_t points, int32_t fold_begin, int32_t fold_end, bsccs_cv_cell* cells,
                                bsccs_cv_result* result) {
    return guard([&] {
        if (!ds || !cells || !result) input_error("cross-validation: null argument");
        validate_cv(cfg, variance_grid, points);
        const std::vector<double> grid = sorted_grid(variance_grid, points);
        DeviceGuard g(ds->device);
        std::memset(result, 0, sizeof *result);
        cv_folds(ds, cfg, grid, fold_begin, fold_end, cells, result);
    });
}

bsccs_status bsccs_cv_select(const double* sorted_grid_in, int32_t points, int32_t folds, const bsccs_cv_cell* cells,
                             double* mean_predictive_ll, bsccs_cv_result* result) {
    return guard([&] {
        if (!sorted_grid_in || points < 1 || folds < 1 || !cells || !result) input_error("cv_select: bad argument");
        const std::vector<double> grid(sorted_grid_in, sorted_grid_in + points);
        cv_select(grid, folds, cells, mean_predictive_ll, result);
    });
}

bsccs_status bsccs_grid_search_cv(const bsccs_dataset* ds, const bsccs_cv_config* cfg, const double* variance_grid,
                                  int32_t points, double* grid_out, bsccs_cv_cell* cells, double* mean_predictive_ll,
                                  bsccs_cv_result* result) {
    return guard([&] {
        if (!ds || !cells || !result) input_error("cross-validation: null argument");
        validate_cv(cfg, variance_grid, points);
        const std::vector<double> grid = sorted_grid(variance_grid, points);
        DeviceGuard g(ds->device);
        std::memset(result, 0, sizeof *result);
        cv_folds(ds, cfg, grid, 0, cfg->folds, cells, result);
        if (grid_out) std::copy(grid.begin(), grid.end(), grid_out);
        cv_select(grid, cfg->folds, cells, mean_predictive_ll, result);
    });
}

void bsccs_bootstrap_config_default(bsccs_bootstrap_config* c) {
    std::memset(c, 0, sizeof *c);
    c->replicates = 200;
    c->warm_start = 1;
    c->level = 0.95;
    c->seed = 0;
    c->prior.kind = PRIOR_NONE; // PriorSpec{} (prior.hpp:17-20)
    c->prior.variance = 1.0;
    c->prior.variance_is_laplace_scale = 0;
    bsccs_solver_config_default(&c->solver);
    c->engine = BSCCS_ENGINE_SUBSET;
    c->batch = 0;
}

bsccs_status bsccs_bootstrap_replicates(const bsccs_dataset* ds, const bsccs_bootstrap_config* cfg,
                                        const double* beta_full, int32_t r_begin, int32_t r_end, double* estimates,
                                        int32_t* converged, bsccs_bootstrap_result* result) {
    return guard([&] {
        if (!ds || !estimates || !converged || !result) input_error("bootstrap: null argument");
        validate_bootstrap(cfg);
        DeviceGuard g(ds->device);
        std::memset(result, 0, sizeof *result);
        boot_replicates(ds, cfg, beta_full, r_begin, r_end, estimates, converged, result);
    });
}

bsccs_status bsccs_bootstrap_summarize(int32_t num_drugs, int32_t replicates, double level, const double* estimates,
                                       const int32_t* converged, double* lower, double* upper, double* p_hat,
                                       bsccs_bootstrap_result* result) {
    return guard([&] {
        if (num_drugs < 1 || replicates < 1 || !estimates || !converged || !lower || !upper || !p_hat || !result)
            input_error("bootstrap summary: bad argument");
        if (!(level > 0.0 && level < 1.0)) input_error("bootstrap: interval level must lie in (0, 1)");
        boot_summarize(num_drugs, replicates, level, estimates, converged, lower, upper, p_hat, result);
    });
}

bsccs_status bsccs_fit_batch(const bsccs_dataset* ds, int32_t R, const bsccs_prior* priors, const int32_t* weights,
                             const double* init_beta, const bsccs_solver_config* cfg, double* beta_out,
                             bsccs_fit_result* results, int32_t* status) {
    return guard([&] {
        if (!ds || !priors || !beta_out || !results || !status) input_error("fit_batch: null argument");
        if (R < 1 || R > 16) input_error("fit_batch: 1..16 fits per batch");
        validate_config(cfg);
        if (cfg->path != 0) input_error("fit_batch: the batched engine runs the sparse update path");
        const int32_t N = ds->N, J = ds->J;
        std::vector<PriorParams> p(static_cast<size_t>(R));
        for (int32_t r = 0; r < R; ++r) p[r] = to_params(&priors[r]);
        const int RB = R <= 8 ? 8 : 16;
        (void)N;
        std::vector<const double*> init(static_cast<size_t>(R), nullptr);
        if (init_beta)
            for (int32_t r = 0; r < R; ++r) init[r] = init_beta + static_cast<size_t>(r) * J;
        std::vector<int> err(static_cast<size_t>(R));
        DeviceGuard g(ds->device);
        Batch* b = batch_create(ds, RB);
        try {
            batch_set_weight_rows(b, weights, R);
            batch_fit(b, R, p.data(), init.data(), cfg, beta_out, results, err.data(), nullptr);
        } catch (...) {
            batch_destroy(b);
            throw;
        }
        batch_destroy(b);
        for (int32_t r = 0; r < R; ++r) {
            status[r] = BSCCS_OK;
            if (err[r] == DERR_OVERFLOW || err[r] == DERR_STEP_NONFINITE || err[r] == DERR_FLAT_NO_PRIOR)
                status[r] = BSCCS_NUMERIC_ERROR;
            else if (err[r] != 0)
                status[r] = BSCCS_INTERNAL_ERROR;
        }
    });
}

bsccs_status bsccs_run_bootstrap(const bsccs_dataset* ds, const bsccs_bootstrap_config* cfg, double* beta_full,
                                 double* lower, double* upper, double* p_hat, bsccs_bootstrap_result* result) {
    return guard([&] {
        if (!ds || !beta_full || !lower || !upper || !p_hat || !result) input_error("bootstrap: null argument");
        validate_bootstrap(cfg);
        DeviceGuard g(ds->device);
        std::memset(result, 0, sizeof *result);
        const PriorParams p = to_params(&cfg->prior);
        bsccs_fit_result full;
        fit_resident(ds, p, &cfg->solver, nullptr, beta_full, &full);
        result->full_converged = full.converged;
        result->total_cycles += full.cycles_run;
        result->coordinates_visited += full.coordinates_visited;
        result->device_seconds += full.device_seconds;
        const int32_t J = ds->J, R = cfg->replicates;
        std::vector<double> est(static_cast<size_t>(R) * J);
        std::vector<int32_t> conv(static_cast<size_t>(R));
        boot_replicates(ds, cfg, beta_full, 0, R, est.data(), conv.data(), result);
        const int32_t fc = result->full_converged;
        boot_summarize(J, R, cfg->level, est.data(), conv.data(), lower, upper, p_hat, result);
        result->full_converged = fc;
    });
}

} // extern "C"
