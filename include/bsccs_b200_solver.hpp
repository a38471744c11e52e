// bsccs_b200_solver.hpp -- C++ drop-in for the reference solver entry points.
//
// Header-only shim over the C ABI (bsccs_b200.h).  It keeps the signature
// of the reference's `bsccs::fit` (solver.hpp:206-210):
//
//     FitResult fit(const Dataset& ds, const PriorSpec& prior,
//                   const SolverConfig& cfg = {},
//                   const std::vector<double>& init_beta = {},
//                   ThreadPool* pool = nullptr);
//
// for any Dataset / PriorSpec / SolverConfig / FitResult types with the
// reference's public field names (dataset.hpp:53-68, prior.hpp:17-25,
// solver.hpp:21-46,66-72), so a maintainer switches an existing call site by
// changing the namespace of the call:
//
//     #include <bsccs/bsccs.hpp>
//     #include <bsccs_b200_solver.hpp>
//     bsccs::FitResult r = bsccs_b200::fit(ds, prior, cfg);   // was bsccs::fit
//
// Status codes become the reference exception types again (common.hpp:10-35)
// when the reference's `bsccs` namespace is visible; otherwise std exceptions.
// The dataset is uploaded once per Dataset object and cached in a
// DeviceDataset that the caller may also hold explicitly for repeated fits
// (CV chains, bootstrap replicates).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bsccs_b200.h"

#if __has_include(<bsccs/solver.hpp>)
#include <bsccs/solver.hpp> // reference types: Dataset, PriorSpec, SolverConfig, FitResult, exceptions
#define BSCCS_B200_HAVE_REFERENCE 1
#endif
#if __has_include(<bsccs/cross_validation.hpp>) && __has_include(<bsccs/bootstrap.hpp>)
#include <bsccs/bootstrap.hpp>        // BootstrapConfig / BootstrapResult
#include <bsccs/cross_validation.hpp> // CVConfig / CVCell / CVResult
#define BSCCS_B200_HAVE_REFERENCE_DRIVERS 1
#endif

namespace bsccs_b200 {

struct Error : std::runtime_error {
    bsccs_status code;
    Error(bsccs_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

namespace detail {

template <typename Ex>
[[noreturn]] inline void raise_as(const std::string& msg) {
    throw Ex(msg);
}

// Map a status to the reference exception types when they are available
// (include <bsccs/common.hpp> before this header), else to Error.
inline void check(bsccs_status st) {
    if (st == BSCCS_OK) return;
    const std::string msg = bsccs_last_error();
#if defined(BSCCS_B200_HAVE_REFERENCE)
    switch (st) {
    case BSCCS_INPUT_ERROR: raise_as<::bsccs::input_error>(msg);
    case BSCCS_NUMERIC_ERROR: raise_as<::bsccs::numeric_error>(msg);
    case BSCCS_CONVERGENCE_ERROR: raise_as<::bsccs::convergence_error>(msg);
    case BSCCS_INTERNAL_ERROR: raise_as<::bsccs::internal_error>(msg);
    default: break;
    }
#endif
    throw Error(st, msg);
}

// An input error raised on this side of the C ABI, with its own message
// (bsccs_last_error() would still hold an earlier call's text).
[[noreturn]] inline void input_error(const std::string& msg) {
#if defined(BSCCS_B200_HAVE_REFERENCE)
    raise_as<::bsccs::input_error>(msg);
#else
    throw Error(BSCCS_INPUT_ERROR, msg);
#endif
}

} // namespace detail

// Device-resident copy of a reference-layout Dataset (one upload).
class DeviceDataset {
public:
    template <typename Dataset>
    explicit DeviceDataset(const Dataset& ds, int device = 0, int ctas = 0) {
        const std::size_t J = ds.columns.size();
        std::vector<int64_t> col_ptr(J + 1, 0);
        for (std::size_t j = 0; j < J; ++j) col_ptr[j + 1] = col_ptr[j] + static_cast<int64_t>(ds.columns[j].rows.size());
        std::vector<int32_t> rows(static_cast<std::size_t>(col_ptr[J])), subjects(rows.size());
        for (std::size_t j = 0; j < J; ++j) {
            std::copy(ds.columns[j].rows.begin(), ds.columns[j].rows.end(), rows.begin() + col_ptr[j]);
            std::copy(ds.columns[j].subjects.begin(), ds.columns[j].subjects.end(), subjects.begin() + col_ptr[j]);
        }
        std::vector<int64_t> ydx(ds.y_dot_x.begin(), ds.y_dot_x.end());
        bsccs_dataset* h = nullptr;
        detail::check(bsccs_dataset_create(
            ds.num_subjects, ds.num_eras, static_cast<int32_t>(J), col_ptr[J], ds.subject_offsets.data(),
            ds.events_per_subject.data(), ds.era_lengths.data(), ds.event_counts.data(), col_ptr.data(),
            rows.data(), subjects.data(), ydx.empty() ? nullptr : ydx.data(), device, ctas, &h));
        handle_.reset(h);
        num_drugs_ = static_cast<int32_t>(J);
    }
    // adopt a handle built by the library (read_long_format, subset)
    DeviceDataset(bsccs_dataset* h, int32_t num_drugs) : handle_(h), num_drugs_(num_drugs) {}
    bsccs_dataset* get() const { return handle_.get(); }
    int32_t num_drugs() const { return num_drugs_; }

private:
    struct Del {
        void operator()(bsccs_dataset* p) const { bsccs_dataset_destroy(p); }
    };
    std::unique_ptr<bsccs_dataset, Del> handle_;
    int32_t num_drugs_ = 0;
};

template <typename PriorSpec>
inline bsccs_prior to_c_prior(const PriorSpec& p) {
    bsccs_prior out;
    out.kind = static_cast<int32_t>(p.kind);
    out.variance_is_laplace_scale = p.variance_is_laplace_scale ? 1 : 0;
    out.variance = p.variance;
    return out;
}

template <typename SolverConfig>
inline bsccs_solver_config to_c_config(const SolverConfig& c) {
    bsccs_solver_config out;
    bsccs_solver_config_default(&out);
    out.epsilon = c.epsilon;
    out.max_cycles = c.max_cycles;
    out.convergence = static_cast<int32_t>(c.convergence);
    out.trust_init = c.trust_init;
    out.precision = static_cast<int32_t>(c.precision);
    out.path = static_cast<int32_t>(c.path);
    out.partitions = c.partitions;
    out.dense_refresh_interval = c.dense_refresh_interval;
    out.random_cycle = c.random_cycle ? 1 : 0;
    out.cycle_seed = c.cycle_seed;
    out.min_parallel_nnz = static_cast<uint64_t>(c.min_parallel_nnz);
    return out;
}

// fit on an already resident dataset; FitResult is the caller's type
// (reference: solver.hpp:66-72)
template <typename FitResult, typename PriorSpec, typename SolverConfig>
FitResult fit(const DeviceDataset& dds, const PriorSpec& prior, const SolverConfig& cfg,
              const std::vector<double>& init_beta = {}) {
    const bsccs_prior p = to_c_prior(prior);
    const bsccs_solver_config c = to_c_config(cfg);
    if (!init_beta.empty() && static_cast<int32_t>(init_beta.size()) != dds.num_drugs())
        detail::input_error("init_state: coefficient count does not match drug count"); // engine.hpp:142-144
    FitResult out;
    out.beta_map.assign(static_cast<std::size_t>(dds.num_drugs()), 0.0);
    bsccs_fit_result r;
    detail::check(bsccs_fit(dds.get(), &p, &c, init_beta.empty() ? nullptr : init_beta.data(),
                            out.beta_map.data(), &r));
    out.log_posterior = r.log_posterior;
    out.cycles_run = r.cycles_run;
    out.converged = r.converged != 0;
    out.final_criterion = r.final_criterion;
    return out;
}

// read_long_format (io.hpp:88-174) + build_dataset (dataset.hpp:74-152)
// straight into a device-resident dataset; labels via drug_ids().
inline DeviceDataset read_long_format(const std::string& path, const std::vector<std::string>& dictionary = {},
                                      int device = 0, int threads = 0) {
    std::vector<const char*> d;
    for (const auto& x : dictionary) d.push_back(x.c_str());
    bsccs_dataset* h = nullptr;
    detail::check(bsccs_dataset_read_long_format(path.c_str(), d.empty() ? nullptr : d.data(),
                                                 static_cast<int32_t>(d.size()), device, 0, threads, &h));
    int64_t info[6];
    bsccs_dataset_info(h, info);
    return DeviceDataset(h, static_cast<int32_t>(info[2]));
}

inline std::vector<std::string> drug_ids(const DeviceDataset& dds) {
    int64_t need = 0;
    detail::check(bsccs_dataset_drug_ids(dds.get(), nullptr, 0, &need));
    std::string buf(static_cast<std::size_t>(need), '\0');
    detail::check(bsccs_dataset_drug_ids(dds.get(), buf.data(), need, nullptr));
    buf.resize(buf.size() - 1);
    std::vector<std::string> out;
    if (buf.empty()) return out;
    std::size_t a = 0;
    for (std::size_t b = 0; b <= buf.size(); ++b)
        if (b == buf.size() || buf[b] == '\n') {
            out.push_back(buf.substr(a, b - a));
            a = b + 1;
        }
    return out;
}

} // namespace bsccs_b200

#if defined(BSCCS_B200_HAVE_REFERENCE_DRIVERS)
namespace bsccs_b200 {
// Signature of bsccs::grid_search_cv (cross_validation.hpp:100-104) with the
// device engine as an extra trailing argument; returns the reference's
// CVResult (cells [grid point][fold]).
inline ::bsccs::CVResult grid_search_cv(const DeviceDataset& dds, const ::bsccs::CVConfig& cfg,
                                        int engine = BSCCS_ENGINE_SUBSET) {
    bsccs_cv_config c;
    bsccs_cv_config_default(&c);
    c.folds = cfg.folds;
    c.prior_kind = static_cast<int32_t>(cfg.prior_kind);
    c.variance_is_laplace_scale = cfg.variance_is_laplace_scale ? 1 : 0;
    c.warm_start = cfg.warm_start ? 1 : 0;
    c.seed = cfg.seed;
    c.solver = to_c_config(cfg.solver);
    c.engine = engine;
    const int32_t P = static_cast<int32_t>(cfg.variance_grid.size());
    const std::size_t F = static_cast<std::size_t>(cfg.folds > 0 ? cfg.folds : 1);
    std::vector<double> grid(static_cast<std::size_t>(P > 0 ? P : 1)), mean(grid.size());
    std::vector<bsccs_cv_cell> cells(grid.size() * F);
    bsccs_cv_result r;
    detail::check(bsccs_grid_search_cv(dds.get(), &c, cfg.variance_grid.data(), P, grid.data(), cells.data(),
                                       mean.data(), &r));
    ::bsccs::CVResult out;
    out.variance_grid.assign(grid.begin(), grid.begin() + P);
    out.cells.assign(static_cast<std::size_t>(P), std::vector<::bsccs::CVCell>(F));
    for (int32_t g = 0; g < P; ++g)
        for (std::size_t f = 0; f < F; ++f) {
            const bsccs_cv_cell& x = cells[static_cast<std::size_t>(g) * F + f];
            ::bsccs::CVCell& y = out.cells[static_cast<std::size_t>(g)][f];
            y.predictive_ll = x.predictive_ll;
            y.cycles = x.cycles;
            y.converged = x.converged != 0;
            y.valid = x.valid != 0;
        }
    out.mean_predictive_ll.assign(mean.begin(), mean.begin() + P);
    out.selected_index = r.selected_index;
    out.selected_variance = r.selected_variance;
    out.total_cycles = r.total_cycles;
    return out;
}

inline ::bsccs::CVResult grid_search_cv(const ::bsccs::Dataset& ds, const ::bsccs::CVConfig& cfg,
                                        ::bsccs::ThreadPool* pool = nullptr, int device = 0,
                                        int engine = BSCCS_ENGINE_SUBSET) {
    (void)pool;
    DeviceDataset dds(ds, device);
    return grid_search_cv(dds, cfg, engine);
}

// Signature of bsccs::run_bootstrap (bootstrap.hpp:79-81) plus the engine.
inline ::bsccs::BootstrapResult run_bootstrap(const DeviceDataset& dds, const ::bsccs::BootstrapConfig& cfg,
                                              int engine = BSCCS_ENGINE_SUBSET) {
    bsccs_bootstrap_config c;
    bsccs_bootstrap_config_default(&c);
    c.replicates = cfg.replicates;
    c.warm_start = cfg.warm_start ? 1 : 0;
    c.level = cfg.level;
    c.seed = cfg.seed;
    c.prior = to_c_prior(cfg.prior);
    c.solver = to_c_config(cfg.solver);
    c.engine = engine;
    const std::size_t J = static_cast<std::size_t>(dds.num_drugs());
    ::bsccs::BootstrapResult out;
    out.beta_full.assign(J, 0.0);
    out.lower.assign(J, 0.0);
    out.upper.assign(J, 0.0);
    out.p_hat.assign(J, 0.0);
    bsccs_bootstrap_result r;
    detail::check(bsccs_run_bootstrap(dds.get(), &c, out.beta_full.data(), out.lower.data(), out.upper.data(),
                                      out.p_hat.data(), &r));
    out.full_converged = r.full_converged != 0;
    out.replicates = r.replicates;
    out.used = r.used;
    out.non_converged = r.non_converged;
    return out;
}

inline ::bsccs::BootstrapResult run_bootstrap(const ::bsccs::Dataset& ds, const ::bsccs::BootstrapConfig& cfg,
                                              ::bsccs::ThreadPool* pool = nullptr, int device = 0,
                                              int engine = BSCCS_ENGINE_SUBSET) {
    (void)pool;
    DeviceDataset dds(ds, device);
    return run_bootstrap(dds, cfg, engine);
}
} // namespace bsccs_b200
#endif

#if defined(BSCCS_B200_HAVE_REFERENCE)
namespace bsccs_b200 {
// Signature of bsccs::fit (solver.hpp:206-210): uploads `ds` and fits on
// `device`.  The ThreadPool argument is accepted for drop-in compatibility;
// the device decides its own parallelism.
inline ::bsccs::FitResult fit(const ::bsccs::Dataset& ds, const ::bsccs::PriorSpec& prior,
                              const ::bsccs::SolverConfig& cfg = {}, const std::vector<double>& init_beta = {},
                              ::bsccs::ThreadPool* pool = nullptr, int device = 0) {
    (void)pool;
    DeviceDataset dds(ds, device);
    return fit<::bsccs::FitResult>(dds, prior, cfg, init_beta);
}
} // namespace bsccs_b200
#endif
