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
        detail::check((bsccs_status)BSCCS_INPUT_ERROR);
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

} // namespace bsccs_b200

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
