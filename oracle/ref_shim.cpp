// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/bsccs/*.hpp), built by oracle/Makefile into
// oracle/_ref/libbsccs_ref.so.  Nothing of the reference is copied: this file
// only converts the flat CSC form used across our C ABI into bsccs::Dataset
// and calls the reference's own functions.  Used (a) to pin the C
// restatement oracle/ccd_oracle.c bit for bit, (b) to generate the golden
// fixtures in tests/golden/, and (c) as bench.py's CPU baseline
// (cpu_baseline.kind = "reference").
#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <bsccs/bsccs.hpp>

#include "../include/bsccs_b200.h"

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const bsccs::input_error& e) {
        g_err = e.what();
        return BSCCS_INPUT_ERROR;
    } catch (const bsccs::numeric_error& e) {
        g_err = e.what();
        return BSCCS_NUMERIC_ERROR;
    } catch (const bsccs::convergence_error& e) {
        g_err = e.what();
        return BSCCS_CONVERGENCE_ERROR;
    } catch (const bsccs::internal_error& e) {
        g_err = e.what();
        return BSCCS_INTERNAL_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return BSCCS_INTERNAL_ERROR;
    }
}

bsccs::PriorSpec to_prior(const bsccs_prior* p) {
    bsccs::PriorSpec out;
    out.kind = static_cast<bsccs::PriorKind>(p->kind);
    out.variance = p->variance;
    out.variance_is_laplace_scale = p->variance_is_laplace_scale != 0;
    return out;
}

bsccs::SolverConfig to_cfg(const bsccs_solver_config* c) {
    bsccs::SolverConfig out;
    out.epsilon = c->epsilon;
    out.max_cycles = c->max_cycles;
    out.trust_init = c->trust_init;
    out.convergence = c->convergence ? bsccs::ConvergenceMode::normalized
                                     : bsccs::ConvergenceMode::raw_sum;
    out.precision = c->precision == 0 ? bsccs::Precision::Single : bsccs::Precision::Double;
    out.path = c->path == 1 ? bsccs::UpdatePath::dense : bsccs::UpdatePath::sparse;
    out.partitions = c->partitions;
    out.dense_refresh_interval = c->dense_refresh_interval;
    out.random_cycle = c->random_cycle != 0;
    out.cycle_seed = c->cycle_seed;
    out.min_parallel_nnz = c->min_parallel_nnz;
    return out;
}

struct RefState {
    bsccs::EngineState<double> st;
    std::unique_ptr<bsccs::SolverState<double>> solver;
    std::unique_ptr<bsccs::ThreadPool> pool;
};

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Flat CSC -> bsccs::Dataset (public-field struct, dataset.hpp:53-68).
int ref_dataset_create(int32_t N, int32_t K, int32_t J, int64_t nnz,
                       const int32_t* subject_offsets, const int32_t* events_per_subject,
                       const int32_t* era_lengths, const int32_t* event_counts,
                       const int64_t* col_ptr, const int32_t* rows, const int32_t* subjects,
                       const int64_t* y_dot_x, void** out) {
    return guard([&] {
        auto* ds = new bsccs::Dataset();
        ds->num_subjects = N;
        ds->num_eras = K;
        ds->num_drugs = J;
        ds->subject_offsets.assign(subject_offsets, subject_offsets + N + 1);
        ds->events_per_subject.assign(events_per_subject, events_per_subject + N);
        ds->era_lengths.assign(era_lengths, era_lengths + K);
        ds->event_counts.assign(event_counts, event_counts + K);
        ds->y_dot_x.assign(y_dot_x, y_dot_x + J);
        ds->columns.resize(static_cast<size_t>(J));
        for (int32_t j = 0; j < J; ++j) {
            auto& col = ds->columns[static_cast<size_t>(j)];
            col.rows.assign(rows + col_ptr[j], rows + col_ptr[j + 1]);
            col.subjects.assign(subjects + col_ptr[j], subjects + col_ptr[j + 1]);
            ds->max_column_nnz = std::max<int32_t>(ds->max_column_nnz,
                                                   static_cast<int32_t>(col.rows.size()));
        }
        (void)nnz;
        *out = ds;
    });
}

void ref_dataset_destroy(void* ds) { delete static_cast<bsccs::Dataset*>(ds); }

int64_t ref_dataset_nnz(void* dsp) {
    auto* ds = static_cast<bsccs::Dataset*>(dsp);
    int64_t n = 0;
    for (auto& c : ds->columns) n += static_cast<int64_t>(c.rows.size());
    return n;
}

// sizes: N K J nnz
void ref_dataset_sizes(void* dsp, int64_t out[4]) {
    auto* ds = static_cast<bsccs::Dataset*>(dsp);
    out[0] = ds->num_subjects;
    out[1] = ds->num_eras;
    out[2] = ds->num_drugs;
    out[3] = ref_dataset_nnz(dsp);
}

// bsccs::Dataset -> flat CSC (caller-sized buffers)
void ref_dataset_flatten(void* dsp, int32_t* subject_offsets, int32_t* events_per_subject,
                         int32_t* era_lengths, int32_t* event_counts, int64_t* col_ptr,
                         int32_t* rows, int32_t* subjects, int64_t* y_dot_x) {
    auto* ds = static_cast<bsccs::Dataset*>(dsp);
    std::memcpy(subject_offsets, ds->subject_offsets.data(), sizeof(int32_t) * ds->subject_offsets.size());
    std::memcpy(events_per_subject, ds->events_per_subject.data(), sizeof(int32_t) * ds->events_per_subject.size());
    std::memcpy(era_lengths, ds->era_lengths.data(), sizeof(int32_t) * ds->era_lengths.size());
    std::memcpy(event_counts, ds->event_counts.data(), sizeof(int32_t) * ds->event_counts.size());
    std::memcpy(y_dot_x, ds->y_dot_x.data(), sizeof(int64_t) * ds->y_dot_x.size());
    int64_t p = 0;
    col_ptr[0] = 0;
    for (size_t j = 0; j < ds->columns.size(); ++j) {
        const auto& c = ds->columns[j];
        std::memcpy(rows + p, c.rows.data(), sizeof(int32_t) * c.rows.size());
        std::memcpy(subjects + p, c.subjects.data(), sizeof(int32_t) * c.subjects.size());
        p += static_cast<int64_t>(c.rows.size());
        col_ptr[j + 1] = p;
    }
}

// simulate() (simulate.hpp:50-137) -> Dataset handle
int ref_simulate(int32_t subjects, int32_t drugs, int32_t min_eras, int32_t max_eras,
                 int32_t min_len, int32_t max_len, const double* prevalence,
                 const double* true_beta, double mean, double sd, uint64_t seed, void** out) {
    return guard([&] {
        bsccs::SimConfig cfg;
        cfg.subjects = subjects;
        cfg.drugs = drugs;
        cfg.min_eras = min_eras;
        cfg.max_eras = max_eras;
        cfg.min_era_length = min_len;
        cfg.max_era_length = max_len;
        cfg.prevalence.assign(prevalence, prevalence + drugs);
        cfg.true_beta.assign(true_beta, true_beta + drugs);
        cfg.baseline_log_rate_mean = mean;
        cfg.baseline_log_rate_sd = sd;
        cfg.seed = seed;
        auto sim = bsccs::simulate(cfg);
        *out = new bsccs::Dataset(std::move(sim.dataset));
    });
}

// subset_dataset (dataset.hpp:157-217)
int ref_subset(void* dsp, const int32_t* idx, int64_t n, void** out) {
    return guard([&] {
        std::vector<bsccs::index_t> sel(idx, idx + n);
        *out = new bsccs::Dataset(bsccs::subset_dataset(*static_cast<bsccs::Dataset*>(dsp), sel));
    });
}

// fit (solver.hpp:206-220).  threads > 1 supplies ThreadPool(threads - 1)
// (the caller participates, thread_pool.hpp:22-28).  seconds = fit() wall.
int ref_fit(void* dsp, const bsccs_prior* prior, const bsccs_solver_config* cfg,
            const double* init_beta, int32_t threads, double* beta_out,
            bsccs_fit_result* res, double* seconds) {
    return guard([&] {
        auto* ds = static_cast<bsccs::Dataset*>(dsp);
        std::vector<double> init;
        if (init_beta) init.assign(init_beta, init_beta + ds->num_drugs);
        std::unique_ptr<bsccs::ThreadPool> pool;
        if (threads > 1) pool = std::make_unique<bsccs::ThreadPool>(threads - 1);
        const auto t0 = std::chrono::steady_clock::now();
        bsccs::FitResult r = bsccs::fit(*ds, to_prior(prior), to_cfg(cfg), init, pool.get());
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(beta_out, r.beta_map.data(), sizeof(double) * r.beta_map.size());
        std::memset(res, 0, sizeof *res);
        res->log_posterior = r.log_posterior;
        res->final_criterion = r.final_criterion;
        res->cycles_run = r.cycles_run;
        res->converged = r.converged ? 1 : 0;
    });
}

// read_long_format (io.hpp:88-174) + build_dataset (dataset.hpp:74-152);
// labels: newline-joined into a caller buffer
int ref_read_long_format(const char* path, const char* const* dict, int32_t dict_n, void** out, char* labels,
                         int64_t cap) {
    return guard([&] {
        std::vector<std::string> d;
        for (int32_t j = 0; j < dict_n; ++j) d.emplace_back(dict[j]);
        auto data = bsccs::read_long_format(path, d);
        auto* ds = new bsccs::Dataset(bsccs::build_dataset(
            data.records, static_cast<bsccs::index_t>(data.drug_ids.size()), data.drug_ids));
        std::string joined;
        for (size_t j = 0; j < ds->drug_ids.size(); ++j) {
            if (j) joined += '\n';
            joined += ds->drug_ids[j];
        }
        if (labels && cap > 0) {
            const size_t n = std::min<size_t>(joined.size(), static_cast<size_t>(cap - 1));
            std::memcpy(labels, joined.data(), n);
            labels[n] = '\0';
        }
        *out = ds;
    });
}

// kfold_split (cross_validation.hpp:58-80): fold lists back to back
int ref_kfold_split(void* dsp, int32_t folds, uint64_t seed, int32_t* out, int32_t* sizes) {
    return guard([&] {
        auto lists = bsccs::kfold_split(*static_cast<bsccs::Dataset*>(dsp), folds, seed);
        size_t p = 0;
        for (size_t f = 0; f < lists.size(); ++f) {
            sizes[f] = static_cast<int32_t>(lists[f].size());
            for (auto s : lists[f]) out[p++] = s;
        }
    });
}

// resample (bootstrap.hpp:43-52) from Rng(seed, stream)
int ref_resample(void* dsp, uint64_t seed, uint64_t stream, int32_t* out) {
    return guard([&] {
        bsccs::Rng rng(seed, stream);
        auto idx = bsccs::resample(*static_cast<bsccs::Dataset*>(dsp), rng);
        std::memcpy(out, idx.data(), sizeof(int32_t) * idx.size());
    });
}

// predictive_log_likelihood (cross_validation.hpp:89-93)
int ref_predictive_ll(void* dsp, const double* beta, double* out) {
    return guard([&] {
        auto* ds = static_cast<bsccs::Dataset*>(dsp);
        std::vector<double> b(beta, beta + ds->num_drugs);
        *out = bsccs::predictive_log_likelihood(b, *ds);
    });
}

// grid_search_cv (cross_validation.hpp:100-215).  cells: [points][folds] x
// {predictive_ll, cycles, converged, valid}; threads > 1 supplies a pool.
int ref_grid_search_cv(void* dsp, int32_t folds, int32_t prior_kind, int32_t scale, int32_t warm,
                       uint64_t seed, const bsccs_solver_config* cfg, const double* grid, int32_t points,
                       int32_t threads, double* grid_out, double* cell_ll, int32_t* cell_int,
                       double* mean_ll, int32_t* selected_index, double* selected_variance,
                       int64_t* total_cycles) {
    return guard([&] {
        bsccs::CVConfig c;
        c.folds = folds;
        c.variance_grid.assign(grid, grid + points);
        c.prior_kind = static_cast<bsccs::PriorKind>(prior_kind);
        c.variance_is_laplace_scale = scale != 0;
        c.seed = seed;
        c.solver = to_cfg(cfg);
        c.warm_start = warm != 0;
        std::unique_ptr<bsccs::ThreadPool> pool;
        if (threads > 1) pool = std::make_unique<bsccs::ThreadPool>(threads - 1);
        auto r = bsccs::grid_search_cv(*static_cast<bsccs::Dataset*>(dsp), c, pool.get());
        for (int32_t g = 0; g < points; ++g) {
            grid_out[g] = r.variance_grid[static_cast<size_t>(g)];
            mean_ll[g] = r.mean_predictive_ll[static_cast<size_t>(g)];
            for (int32_t f = 0; f < folds; ++f) {
                const auto& cell = r.cells[static_cast<size_t>(g)][static_cast<size_t>(f)];
                const size_t k = static_cast<size_t>(g) * folds + f;
                cell_ll[k] = cell.predictive_ll;
                cell_int[3 * k] = cell.cycles;
                cell_int[3 * k + 1] = cell.converged ? 1 : 0;
                cell_int[3 * k + 2] = cell.valid ? 1 : 0;
            }
        }
        *selected_index = r.selected_index;
        *selected_variance = r.selected_variance;
        *total_cycles = r.total_cycles;
    });
}

// run_bootstrap (bootstrap.hpp:79-158); ints = {used, non_converged, full_converged}
int ref_run_bootstrap(void* dsp, int32_t replicates, double level, uint64_t seed,
                      const bsccs_prior* prior, const bsccs_solver_config* cfg, int32_t warm,
                      int32_t threads, double* beta_full, double* lower, double* upper,
                      double* p_hat, int32_t* ints) {
    return guard([&] {
        bsccs::BootstrapConfig c;
        c.replicates = replicates;
        c.level = level;
        c.seed = seed;
        c.prior = to_prior(prior);
        c.solver = to_cfg(cfg);
        c.warm_start = warm != 0;
        std::unique_ptr<bsccs::ThreadPool> pool;
        if (threads > 1) pool = std::make_unique<bsccs::ThreadPool>(threads - 1);
        auto r = bsccs::run_bootstrap(*static_cast<bsccs::Dataset*>(dsp), c, pool.get());
        const size_t J = r.beta_full.size();
        std::memcpy(beta_full, r.beta_full.data(), sizeof(double) * J);
        std::memcpy(lower, r.lower.data(), sizeof(double) * J);
        std::memcpy(upper, r.upper.data(), sizeof(double) * J);
        std::memcpy(p_hat, r.p_hat.data(), sizeof(double) * J);
        ints[0] = r.used;
        ints[1] = r.non_converged;
        ints[2] = r.full_converged ? 1 : 0;
    });
}

// ---- engine-level handles --------------------------------------------------
int ref_state_create(void* dsp, const double* beta, const bsccs_solver_config* cfg, void** out) {
    return guard([&] {
        auto* ds = static_cast<bsccs::Dataset*>(dsp);
        std::vector<double> b;
        if (beta) b.assign(beta, beta + ds->num_drugs);
        auto* s = new RefState{bsccs::init_state<double>(*ds, b), nullptr, nullptr};
        bsccs::SolverConfig c = cfg ? to_cfg(cfg) : bsccs::SolverConfig{};
        s->solver = std::make_unique<bsccs::SolverState<double>>(*ds, c);
        *out = s;
    });
}
void ref_state_destroy(void* s) { delete static_cast<RefState*>(s); }

int ref_grad_hess(void* dsp, void* sp, int32_t j, int32_t partitions, double* g, double* h) {
    return guard([&] {
        auto gh = bsccs::parallel_fused_grad_hess(*static_cast<bsccs::Dataset*>(dsp),
                                                  static_cast<RefState*>(sp)->st, j, partitions);
        *g = gh.gradient;
        *h = gh.hessian;
    });
}
int ref_sparse_update(void* dsp, void* sp, int32_t j, double delta) {
    return guard([&] {
        bsccs::sparse_delta_update(*static_cast<bsccs::Dataset*>(dsp), static_cast<RefState*>(sp)->st, j, delta);
    });
}
int ref_dense_recompute(void* dsp, void* sp, const double* beta) {
    return guard([&] {
        auto* ds = static_cast<bsccs::Dataset*>(dsp);
        auto& st = static_cast<RefState*>(sp)->st;
        if (beta) bsccs::dense_recompute(*ds, st, std::vector<double>(beta, beta + ds->num_drugs));
        else bsccs::dense_recompute(*ds, st);
    });
}
int ref_log_likelihood(void* dsp, void* sp, double* out) {
    return guard([&] { *out = bsccs::log_likelihood(*static_cast<bsccs::Dataset*>(dsp), static_cast<RefState*>(sp)->st); });
}
void ref_state_get(void* sp, double* beta, double* xbeta, double* lexp, double* den) {
    auto& st = static_cast<RefState*>(sp)->st;
    if (beta) std::memcpy(beta, st.beta.data(), sizeof(double) * st.beta.size());
    if (xbeta) std::memcpy(xbeta, st.xbeta.data(), sizeof(double) * st.xbeta.size());
    if (lexp) std::memcpy(lexp, st.l_exp_xbeta.data(), sizeof(double) * st.l_exp_xbeta.size());
    if (den) std::memcpy(den, st.denominators.data(), sizeof(double) * st.denominators.size());
}
// threads > 1: the reference's parallel route (ThreadPool(threads-1) passed
// to run_cycle; cfg.partitions selects the chunking, solver.hpp:127-128).
void ref_state_set_threads(void* sp, int32_t threads) {
    auto* s = static_cast<RefState*>(sp);
    s->pool.reset();
    if (threads > 1) s->pool = std::make_unique<bsccs::ThreadPool>(threads - 1);
}
// run_cycle (solver.hpp:101-166) with the handle's SolverState
int ref_run_cycle(void* dsp, void* sp, const bsccs_prior* prior, const bsccs_solver_config* cfg,
                  double* criterion, double* trust_out) {
    return guard([&] {
        auto* s = static_cast<RefState*>(sp);
        *criterion = bsccs::run_cycle(*static_cast<bsccs::Dataset*>(dsp), s->st, *s->solver,
                                      to_prior(prior), to_cfg(cfg), s->pool.get());
        if (trust_out) std::memcpy(trust_out, s->solver->trust.data(), sizeof(double) * s->solver->trust.size());
    });
}
int ref_penalized_step(const bsccs_prior* prior, double beta_j, double g, double h, double* out) {
    return guard([&] { *out = bsccs::penalized_step(to_prior(prior), beta_j, g, h); });
}

// One bootstrap replicate exactly as run_bootstrap's run_replicate does it
// (bootstrap.hpp:103-112): indices from Rng(seed, r + 1), subset_dataset,
// fit warm from init_beta (nullable = cold).  Exposes the per-replicate
// estimate that run_bootstrap keeps internal.
int ref_bootstrap_replicate(void* dsp, uint64_t seed, int32_t r, const bsccs_prior* prior,
                            const bsccs_solver_config* cfg, const double* init_beta, double* beta_out,
                            bsccs_fit_result* res) {
    return guard([&] {
        auto* ds = static_cast<bsccs::Dataset*>(dsp);
        bsccs::Rng rng(seed, static_cast<std::uint64_t>(r) + 1);
        const bsccs::Dataset resampled = bsccs::subset_dataset(*ds, bsccs::resample(*ds, rng));
        std::vector<double> init;
        if (init_beta) init.assign(init_beta, init_beta + ds->num_drugs);
        const bsccs::FitResult f = bsccs::fit(resampled, to_prior(prior), to_cfg(cfg), init);
        std::memcpy(beta_out, f.beta_map.data(), sizeof(double) * f.beta_map.size());
        std::memset(res, 0, sizeof *res);
        res->log_posterior = f.log_posterior;
        res->final_criterion = f.final_criterion;
        res->cycles_run = f.cycles_run;
        res->converged = f.converged ? 1 : 0;
    });
}

// The fast SCCS generator of SURVEY §8(d), written here on the reference's
// own Rng so the bench's reference arm can build its dataset without the
// product library in its process.  Attempted subject s draws from
// Rng(seed, s + 1): phi ~ N(-5, 0.5), E ~ U{10..20} eras; per era
// L ~ U{10..60}, m = min(Poisson(lambda_x), J) distinct drugs (below(J) with
// rejection, or the 1/(j+1) inverse CDF for the Zipf variant) sorted
// ascending, y ~ Poisson(L exp(phi + sum beta_true)); subjects with no
// events are dropped and the rest laid out as build_dataset does
// (dataset.hpp:74-152).  tests/test_oracle.py checks it produces the same
// arrays as the product generator.
int ref_fast_sccs(int64_t attempts, int32_t drugs, double lambda_x, int32_t zipf, uint64_t seed, int32_t threads,
                  void** out) {
    return guard([&] {
        if (attempts < 1 || drugs < 1 || !(lambda_x >= 0.0)) throw bsccs::input_error("fast_sccs: bad arguments");
        std::vector<double> truth(static_cast<size_t>(drugs), 0.0);
        const int32_t stride = drugs >= 10 ? drugs / 10 : 1;
        for (int p = 0; p < 10; ++p) {
            const int64_t j = static_cast<int64_t>(p) * stride;
            if (j < drugs) truth[static_cast<size_t>(j)] = (p % 2 == 0) ? 0.7 : -0.5;
        }
        std::vector<double> cum;
        if (zipf) {
            double acc = 0.0;
            for (int32_t j = 0; j < drugs; ++j) cum.push_back(acc += 1.0 / static_cast<double>(j + 1));
        }
        struct Part {
            std::vector<int32_t> nera, nev, len, y, m, drug;
        };
        const int T = std::max(1, threads);
        const int64_t P = std::min<int64_t>(attempts, 64LL * T);
        std::vector<Part> parts(static_cast<size_t>(P));
        auto make = [&](int64_t b) {
            Part& pt = parts[static_cast<size_t>(b)];
            std::vector<int32_t> picked;
            for (int64_t s = attempts * b / P; s < attempts * (b + 1) / P; ++s) {
                bsccs::Rng rng(seed, static_cast<std::uint64_t>(s) + 1);
                const double phi = rng.normal(-5.0, 0.5);
                const int eras = rng.uniform_int(10, 20);
                const size_t e0 = pt.len.size(), d0 = pt.drug.size();
                int32_t events = 0;
                for (int e = 0; e < eras; ++e) {
                    const int32_t L = rng.uniform_int(10, 60);
                    const int32_t m = std::min<int32_t>(rng.poisson(lambda_x), drugs);
                    picked.clear();
                    while (static_cast<int32_t>(picked.size()) < m) {
                        int32_t d;
                        if (zipf) {
                            const double u = rng.uniform() * cum.back();
                            d = static_cast<int32_t>(std::upper_bound(cum.begin(), cum.end(), u) - cum.begin());
                            d = std::min(d, drugs - 1);
                        } else {
                            d = static_cast<int32_t>(rng.below(static_cast<std::uint64_t>(drugs)));
                        }
                        if (std::find(picked.begin(), picked.end(), d) == picked.end()) picked.push_back(d);
                    }
                    std::sort(picked.begin(), picked.end());
                    double xb = 0.0;
                    for (int32_t d : picked) xb += truth[static_cast<size_t>(d)];
                    const int32_t y = rng.poisson(static_cast<double>(L) * std::exp(phi + xb));
                    events += y;
                    pt.len.push_back(L);
                    pt.y.push_back(y);
                    pt.m.push_back(m);
                    pt.drug.insert(pt.drug.end(), picked.begin(), picked.end());
                }
                if (events == 0) {
                    pt.len.resize(e0);
                    pt.y.resize(e0);
                    pt.m.resize(e0);
                    pt.drug.resize(d0);
                    continue;
                }
                pt.nera.push_back(eras);
                pt.nev.push_back(events);
            }
        };
        {
            std::vector<std::thread> pool;
            for (int t = 0; t < T; ++t)
                pool.emplace_back([&, t] {
                    for (int64_t b = t; b < P; b += T) make(b);
                });
            for (auto& th : pool) th.join();
        }
        auto* ds = new bsccs::Dataset();
        std::unique_ptr<bsccs::Dataset> keep(ds);
        ds->num_drugs = drugs;
        std::vector<int64_t> cnt(static_cast<size_t>(drugs), 0);
        for (const Part& pt : parts)
            for (int32_t d : pt.drug) ++cnt[static_cast<size_t>(d)];
        ds->columns.resize(static_cast<size_t>(drugs));
        for (int32_t j = 0; j < drugs; ++j) {
            ds->columns[static_cast<size_t>(j)].rows.reserve(static_cast<size_t>(cnt[static_cast<size_t>(j)]));
            ds->columns[static_cast<size_t>(j)].subjects.reserve(static_cast<size_t>(cnt[static_cast<size_t>(j)]));
        }
        ds->y_dot_x.assign(static_cast<size_t>(drugs), 0);
        ds->subject_offsets.push_back(0);
        bsccs::index_t row = 0, subj = 0;
        for (const Part& pt : parts) {
            size_t e = 0, d = 0;
            for (size_t s = 0; s < pt.nera.size(); ++s, ++subj) {
                for (int32_t q = 0; q < pt.nera[s]; ++q, ++e, ++row) {
                    ds->era_lengths.push_back(pt.len[e]);
                    ds->event_counts.push_back(pt.y[e]);
                    for (int32_t k = 0; k < pt.m[e]; ++k, ++d) {
                        auto& col = ds->columns[static_cast<size_t>(pt.drug[d])];
                        col.rows.push_back(row);
                        col.subjects.push_back(subj);
                        ds->y_dot_x[static_cast<size_t>(pt.drug[d])] += pt.y[e];
                    }
                }
                ds->subject_offsets.push_back(row);
                ds->events_per_subject.push_back(pt.nev[s]);
            }
        }
        if (subj == 0) throw bsccs::input_error("fast_sccs: no subject drew an event");
        ds->num_subjects = subj;
        ds->num_eras = row;
        for (const auto& c : ds->columns)
            ds->max_column_nnz = std::max<bsccs::index_t>(ds->max_column_nnz, static_cast<bsccs::index_t>(c.rows.size()));
        *out = keep.release();
    });
}

// A column sample of a dataset: the same subjects and eras, only the listed
// columns (in the listed order).  The reference's own run_cycle on it does
// exactly the per-coordinate work of those columns against the full-size
// state -- the bounded CPU sample the bench times.
int ref_dataset_columns(void* dsp, const int32_t* cols, int32_t n, void** out) {
    return guard([&] {
        const auto* src = static_cast<bsccs::Dataset*>(dsp);
        auto* ds = new bsccs::Dataset();
        ds->num_drugs = n;
        ds->num_subjects = src->num_subjects;
        ds->num_eras = src->num_eras;
        ds->event_counts = src->event_counts;
        ds->era_lengths = src->era_lengths;
        ds->subject_offsets = src->subject_offsets;
        ds->events_per_subject = src->events_per_subject;
        for (int32_t i = 0; i < n; ++i) {
            if (cols[i] < 0 || cols[i] >= src->num_drugs) {
                delete ds;
                throw bsccs::input_error("dataset_columns: column out of range");
            }
            ds->columns.push_back(src->columns[static_cast<size_t>(cols[i])]);
            ds->y_dot_x.push_back(src->y_dot_x[static_cast<size_t>(cols[i])]);
            ds->max_column_nnz =
                std::max<bsccs::index_t>(ds->max_column_nnz, static_cast<bsccs::index_t>(ds->columns.back().rows.size()));
        }
        *out = ds;
    });
}
int ref_log_density(const bsccs_prior* prior, const double* beta, int32_t n, double* out) {
    return guard([&] { *out = bsccs::log_density(to_prior(prior), std::vector<double>(beta, beta + n)); });
}

} // extern "C"
