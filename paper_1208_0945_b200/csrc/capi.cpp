// capi.cpp -- extern "C" boundary and the host-side CCD driver.
//
// The driver is the reference fit loop (solver.hpp:170-220) over device
// sweeps: validate_config / validate_prior, init_state, cycles until
// criterion <= epsilon or max_cycles, dense refresh every
// dense_refresh_interval non-converged cycles, a final clean rebuild, and
// log_posterior = log_likelihood + log_density.  Each cycle is ONE
// persistent-kernel launch (run_sweep); the host only reads back the
// 8-byte criterion.  Shuffled visit orders come from the reference RNG
// stream (SolverState::order_rng, solver.hpp:81,109-114).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "engine.h"
#include "rng.h"

namespace bsccs_b200 {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

PriorParams to_params(const bsccs_prior* p) {
    if (!p) input_error("null prior");
    if (p->kind < 0 || p->kind > 2) input_error("unknown prior kind");
    // validate_prior (prior.hpp:27-32)
    if (p->kind != PRIOR_NONE && !(p->variance > 0.0 && std::isfinite(p->variance)))
        input_error("prior variance must be positive and finite");
    return make_prior_params(p->kind, p->variance, p->variance_is_laplace_scale != 0);
}

// validate_config (solver.hpp:48-64) plus the knobs the device path pins.
void validate_config(const bsccs_solver_config* c) {
    if (!c) input_error("null solver config");
    if (!(c->epsilon > 0.0) || !std::isfinite(c->epsilon)) input_error("solver: epsilon must be positive and finite");
    if (c->max_cycles < 1) input_error("solver: max_cycles must be at least 1");
    if (!(c->trust_init > 0.0) || !std::isfinite(c->trust_init))
        input_error("solver: trust region width must be positive and finite");
    if (c->partitions < 1) input_error("solver: partitions must be at least 1");
    if (c->dense_refresh_interval < 1) input_error("solver: dense refresh interval must be at least 1");
    if (c->precision != 1) input_error("solver: the B200 path computes in double precision only");
    if (c->path != 0 && c->path != 1) input_error("solver: unknown update path");
}

// prior.hpp:36-61
double log_density(const PriorParams& p, const double* beta, int32_t n) {
    if (p.kind == PRIOR_NONE) return 0.0;
    if (p.kind == PRIOR_NORMAL) {
        const double v = p.variance;
        double ss = 0.0;
        for (int32_t j = 0; j < n; ++j) ss += beta[j] * beta[j];
        return -0.5 * ss / v - 0.5 * static_cast<double>(n) * std::log(6.283185307179586 * v);
    }
    const double b = p.laplace_b;
    double abs_sum = 0.0;
    for (int32_t j = 0; j < n; ++j) abs_sum += std::abs(beta[j]);
    return -abs_sum / b - static_cast<double>(n) * std::log(2.0 * b);
}

namespace {

void set_device(int dev) { CUDA_TRY(cudaSetDevice(dev)); }

// Exchange of a multi-rank (or virtual-rank) group: hierarchical unless
// BSCCS_XCHG=flat (every CTA adding into every rank's area, as round 1).
bool group_hier_from_env() {
    const char* e = std::getenv("BSCCS_XCHG");
    return !(e && std::strcmp(e, "flat") == 0);
}

// Shards bound for one fit, plus their exchange plan.
struct FitContext {
    std::vector<bsccs_state*> states;
    ExchangePlan plan;
};

void fill_trust(FitContext& fc, double trust_init) {
    const int32_t J = fc.states[0]->ds->J;
    std::vector<double> t(static_cast<size_t>(J), trust_init);
    for (auto* st : fc.states)
        CUDA_TRY(cudaMemcpyAsync(st->trust, t.data(), sizeof(double) * J, cudaMemcpyHostToDevice, st->stream));
    for (auto* st : fc.states) CUDA_TRY(cudaStreamSynchronize(st->stream));
}

void set_order(FitContext& fc, const std::vector<int32_t>& order) {
    for (auto* st : fc.states) st->order_h = order;
}

// Error agreement.  In a multi-rank group every host step that can fail on
// one rank only (a dense rebuild that overflows, a nonpositive denominator in
// the log-likelihood) runs through agreed(): each rank then learns, by an
// exact all-reduce of the status, whether any rank failed, and all of them
// throw -- a rank that threw alone would stop launching and leave its peers
// polling in the next exchange.  Errors inside a sweep already travel in the
// exchange's error word.  One process: the error is rethrown as is.
using Agree = std::function<void(std::exception_ptr)>;

void rethrow_local(std::exception_ptr e) {
    if (e) std::rethrow_exception(e);
}

void agreed(const Agree& agree, const std::function<void()>& body) {
    std::exception_ptr e;
    try {
        body();
    } catch (...) {
        e = std::current_exception();
    }
    agree(e);
}

// fit_impl (solver.hpp:170-199) over bound shards.
void fit_loop(FitContext& fc, const PriorParams& prior, const bsccs_solver_config* cfg, double* beta_out,
              bsccs_fit_result* res, const std::function<double(double)>& allreduce_sum,
              const Agree& agree = rethrow_local) {
    bsccs_state* s0 = fc.states[0];
    const int32_t J = s0->ds->J;
    const long long launches0 = launch_count();
    s0->sweep_ms = 0.0;
    s0->alg_bytes = 0.0;
    fill_trust(fc, cfg->trust_init);
    std::vector<int32_t> order(static_cast<size_t>(J));
    std::iota(order.begin(), order.end(), 0);
    Xoshiro order_rng(cfg->cycle_seed);
    set_order(fc, {});

    res->cycles_run = 0;
    res->converged = 0;
    res->final_criterion = INFINITY;
    res->log_posterior = -INFINITY;
    res->coordinates_visited = 0;
    res->coordinates_moved = 0;
    res->dense_refreshes = 0;
    while (res->cycles_run < cfg->max_cycles) {
        if (cfg->random_cycle) { // solver.hpp:109-114
            for (size_t j = order.size(); j > 1; --j) {
                const size_t r = static_cast<size_t>(order_rng.below(j));
                std::swap(order[j - 1], order[r]);
            }
            set_order(fc, order);
        }
        const SweepOutcome o = run_sweep(fc.plan, prior, cfg->convergence != 0, cfg->path == 1);
        res->final_criterion = o.criterion;
        res->coordinates_visited += o.visited;
        res->coordinates_moved += o.moved;
        ++res->cycles_run;
        if (res->final_criterion <= cfg->epsilon) {
            res->converged = 1;
            break;
        }
        if (res->cycles_run % cfg->dense_refresh_interval == 0) {
            agreed(agree, [&] {
                for (auto* st : fc.states) dense_recompute(st, nullptr);
            });
            ++res->dense_refreshes;
        }
    }
    // report from a clean rebuild (solver.hpp:192-196): the refresh and the
    // log-likelihood in one pass, the state rebuilt on its next use
    CUDA_TRY(cudaMemcpy(beta_out, s0->beta, sizeof(double) * J, cudaMemcpyDeviceToHost));
    double ll = 0.0;
    agreed(agree, [&] {
        for (auto* st : fc.states) ll += final_log_likelihood(st);
    });
    ++res->dense_refreshes;
    ll = allreduce_sum(ll);
    res->log_posterior = ll + log_density(prior, beta_out, J);
    res->sweep_seconds = s0->sweep_ms * 1e-3;
    res->algorithmic_bytes = s0->alg_bytes;
    res->kernel_launches = launch_count() - launches0;
}

// One reusable fit workspace per dataset: repeated fits on a resident
// dataset do not re-allocate the K/N state vectors.
std::mutex g_ws_mutex;
struct Workspace {
    bsccs_state* st = nullptr;
    bool busy = false;
};
std::vector<std::pair<const bsccs_dataset*, Workspace>> g_ws;

bsccs_state* acquire_state(const bsccs_dataset* ds, const double* init_beta) {
    {
        std::lock_guard<std::mutex> lk(g_ws_mutex);
        for (auto& e : g_ws) {
            if (e.first == ds && !e.second.busy && e.second.st) {
                e.second.busy = true;
                bsccs_state* st = e.second.st;
                try {
                    if (init_beta)
                        for (int32_t j = 0; j < ds->J; ++j)
                            if (!std::isfinite(init_beta[j])) input_error("init_state: non-finite coefficient");
                    CUDA_TRY(cudaSetDevice(ds->device));
                    if (init_beta)
                        CUDA_TRY(cudaMemcpyAsync(st->beta, init_beta, sizeof(double) * ds->J, cudaMemcpyHostToDevice,
                                                 st->stream));
                } catch (...) {
                    e.second.busy = false;
                    throw;
                }
                if (init_beta) dense_recompute(st, nullptr);
                else dense_recompute_zero(st); // cold start: no CSR pass
                return st;
            }
        }
    }
    bsccs_state* st = state_create(ds, init_beta);
    std::lock_guard<std::mutex> lk(g_ws_mutex);
    for (auto& e : g_ws)
        if (e.first == ds && e.second.st == nullptr) {
            e.second.st = st;
            e.second.busy = true;
            return st;
        }
    bool have = false;
    for (auto& e : g_ws) have = have || e.first == ds;
    if (!have) {
        g_ws.push_back({ds, Workspace{st, true}});
    }
    return st;
}

void release_state(bsccs_state* st) {
    std::lock_guard<std::mutex> lk(g_ws_mutex);
    for (auto& e : g_ws)
        if (e.second.st == st) {
            e.second.busy = false;
            return;
        }
    state_destroy(st);
}

void drop_workspaces(const bsccs_dataset* ds) {
    std::lock_guard<std::mutex> lk(g_ws_mutex);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
        if (it->first == ds) {
            state_destroy(it->second.st);
            it = g_ws.erase(it);
        } else {
            ++it;
        }
    }
}

} // namespace

// fit (solver.hpp:206-220) on a resident dataset, validated arguments.
void fit_resident(const bsccs_dataset* ds, const PriorParams& p, const bsccs_solver_config* cfg,
                  const double* init_beta, double* beta_out, bsccs_fit_result* result) {
    NvtxRange nvtx_("bsccs_fit");
    if (ds->N == 0) input_error("fit: dataset has no subjects");
    set_device(ds->device);
    std::memset(result, 0, sizeof *result);
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, nullptr));
    bsccs_state* st = acquire_state(ds, init_beta);
    try {
        FitContext fc;
        fc.states = {st};
        fc.plan.shards = {st};
        fc.plan.dst = {st->slots};
        fc.plan.local_slots = st->slots;
        fc.plan.counter = st->counter;
        fc.plan.total_participants = ds->ctas;
        fc.plan.participant_base = 0;
        fit_loop(fc, p, cfg, beta_out, result, [](double x) { return x; });
    } catch (...) {
        release_state(st);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        throw;
    }
    release_state(st);
    CUDA_TRY(cudaEventRecord(e1, nullptr));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    result->device_seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

void release_dataset_workspaces(const bsccs_dataset* ds) { drop_workspaces(ds); }

} // namespace bsccs_b200

// ---------------------------------------------------------------------------
struct bsccs_group {
    std::vector<bsccs_dataset*> shards; // local shards
    int rank = 0, world = 1;
    std::vector<int32_t> ctas_per_rank;
    unsigned long long* slots = nullptr;   // local slot buffer
    unsigned long long* counter = nullptr; // local sequence word
    std::vector<unsigned long long*> peer; // per rank (own = slots)
    // virtual ranks (one launch, one exchange area per shard)
    std::vector<unsigned long long*> vslots, vcounters;
    // hierarchical exchange (ccd_kernels.cu forward_local): each area is two
    // halves, [0, kXchgAreaWords) polled by the rank (one arrival per rank),
    // [kXchgAreaWords, 2 kXchgAreaWords) taking the rank's own CTAs' adds
    bool hier = false;
    int device = 0;
    int total = 0;
    int base = 0;
};

using namespace bsccs_b200;

extern "C" {

int32_t bsccs_abi_version(void) { return BSCCS_B200_ABI_VERSION; }

const char* bsccs_last_error(void) { return g_last_error.c_str(); }

int64_t bsccs_launch_count(void) { return launch_count(); }

// Profiling hook (not part of the reference surface): phases of the sweep
// kernel to skip -- bit0 grad/hess gathers, bit1 update, bit2 exchange.
void bsccs_debug_set_sweep_flags(int32_t flags) { set_debug_flags(flags); }
// Profiling hook: globaltimer stamps (loop top, publish, gather done, update
// done) of the first `ncoords` coordinates of each subsequent sweep, per CTA.
int32_t bsccs_debug_trace(int32_t ncoords, int32_t ctas, uint64_t* host_out, int64_t words) {
    return guard([&] {
        if (host_out) read_debug_trace(reinterpret_cast<unsigned long long*>(host_out), static_cast<size_t>(words));
        else set_debug_trace(ncoords, ctas);
    });
}

void bsccs_debug_set_sweep(int32_t kind, double beta_limit) { set_debug_sweep(kind, beta_limit); }
int32_t bsccs_debug_last_sweep(void) { return debug_last_sweep(); }
int32_t bsccs_debug_last_rcd_shape(void) { return debug_last_rcd_shape(); }

bsccs_status bsccs_debug_exchange_sum(int32_t device, const double* partials, int32_t n, double* sum,
                                      int32_t* status) {
    return guard([&] {
        if (!partials || !sum || !status || n < 1 || n > 2048) input_error("debug_exchange_sum: bad arguments");
        debug_exchange_sum(device, partials, n, sum, status);
    });
}

bsccs_status bsccs_device_info(int32_t device, int32_t* sms, int32_t* ctas) {
    return guard([&] {
        int n = 0;
        CUDA_TRY(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) input_error("device index out of range");
        int s = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, device));
        if (sms) *sms = s;
        if (ctas) {
            set_device(device);
            *ctas = default_ctas(device);
        }
    });
}

void bsccs_solver_config_default(bsccs_solver_config* c) {
    std::memset(c, 0, sizeof *c);
    c->epsilon = 0.0005;
    c->max_cycles = 1000;
    c->convergence = 0;
    c->trust_init = 1.0;
    c->precision = 1;
    c->path = 0;
    c->partitions = 1;
    c->dense_refresh_interval = 50;
    c->random_cycle = 0;
    c->cycle_seed = 0;
    c->min_parallel_nnz = 4096;
}

bsccs_status bsccs_dataset_create(int32_t N, int32_t K, int32_t J, int64_t nnz, const int32_t* subject_offsets,
                                  const int32_t* events_per_subject, const int32_t* era_lengths,
                                  const int32_t* event_counts, const int64_t* col_ptr, const int32_t* rows,
                                  const int32_t* subjects, const int64_t* y_dot_x, int32_t device,
                                  int32_t num_ctas_override, bsccs_dataset** out) {
    return guard([&] {
        if (!out) input_error("null output handle");
        *out = dataset_create(N, K, J, nnz, subject_offsets, events_per_subject, era_lengths, event_counts, col_ptr,
                              rows, subjects, y_dot_x, nullptr, device, num_ctas_override);
    });
}

bsccs_status bsccs_dataset_create_shard(int32_t N, int32_t K, int32_t J, int64_t nnz,
                                        const int32_t* subject_offsets, const int32_t* events_per_subject,
                                        const int32_t* era_lengths, const int32_t* event_counts,
                                        const int64_t* col_ptr, const int32_t* rows, const int32_t* subjects,
                                        const int64_t* y_dot_x_global, const int64_t* col_nnz_global,
                                        int32_t device, int32_t num_ctas_override, bsccs_dataset** out) {
    return guard([&] {
        if (!out) input_error("null output handle");
        if (!y_dot_x_global || !col_nnz_global) input_error("shard: global y_dot_x and column counts are required");
        *out = dataset_create(N, K, J, nnz, subject_offsets, events_per_subject, era_lengths, event_counts, col_ptr,
                              rows, subjects, y_dot_x_global, col_nnz_global, device, num_ctas_override);
    });
}

bsccs_status bsccs_dataset_destroy(bsccs_dataset* ds) {
    return guard([&] {
        drop_workspaces(ds);
        dataset_destroy(ds);
    });
}

bsccs_status bsccs_dataset_info(const bsccs_dataset* ds, int64_t out[6]) {
    return guard([&] {
        if (!ds) input_error("null dataset");
        out[0] = ds->N;
        out[1] = ds->K;
        out[2] = ds->J;
        out[3] = ds->nnz;
        out[4] = ds->ctas;
        out[5] = ds->device_bytes;
    });
}

bsccs_status bsccs_dataset_read_long_format(const char* path, const char* const* dictionary, int32_t dict_size,
                                           int32_t device, int32_t num_ctas_override, int32_t threads,
                                           bsccs_dataset** out) {
    return guard([&] {
        if (!out) input_error("null output handle");
        *out = load_long_format(path, dictionary, dict_size, device, num_ctas_override, threads);
    });
}

bsccs_status bsccs_dataset_set_drug_ids(bsccs_dataset* ds, const char* const* labels, int32_t n) {
    return guard([&] {
        if (!ds) input_error("null dataset");
        if (n != 0 && n != ds->J) input_error("build_dataset: drug label count does not match drug count");
        ds->drug_ids.clear();
        for (int32_t j = 0; j < n; ++j) ds->drug_ids.emplace_back(labels[j] ? labels[j] : "");
    });
}

bsccs_status bsccs_dataset_drug_ids(const bsccs_dataset* ds, char* buf, int64_t capacity, int64_t* needed) {
    return guard([&] {
        if (!ds) input_error("null dataset");
        std::string joined;
        for (size_t j = 0; j < ds->drug_ids.size(); ++j) {
            if (j) joined += '\n';
            joined += ds->drug_ids[j];
        }
        if (needed) *needed = static_cast<int64_t>(joined.size()) + 1;
        if (buf && capacity > 0) {
            const size_t n = std::min<size_t>(joined.size(), static_cast<size_t>(capacity - 1));
            std::memcpy(buf, joined.data(), n);
            buf[n] = '\0';
        }
    });
}

bsccs_status bsccs_dataset_subset(const bsccs_dataset* ds, const int32_t* subject_indices, int64_t n,
                                  int32_t num_ctas_override, bsccs_dataset** out) {
    return guard([&] {
        if (!out) input_error("null output handle");
        *out = dataset_subset(ds, subject_indices, n, num_ctas_override);
    });
}

bsccs_status bsccs_dataset_export(const bsccs_dataset* ds, int32_t* subject_offsets, int32_t* events_per_subject,
                                  int32_t* era_lengths, int32_t* event_counts, int64_t* col_ptr, int32_t* rows,
                                  int32_t* subjects, int64_t* y_dot_x) {
    return guard([&] {
        dataset_export(ds, subject_offsets, events_per_subject, era_lengths, event_counts, col_ptr, rows, subjects,
                       y_dot_x);
    });
}

bsccs_status bsccs_kfold_split(int32_t num_subjects, int32_t folds, uint64_t seed, int32_t* subjects_out,
                               int32_t* fold_sizes) {
    return guard([&] { kfold_split(num_subjects, folds, seed, subjects_out, fold_sizes); });
}

bsccs_status bsccs_resample(int32_t num_subjects, uint64_t seed, uint64_t stream, int32_t* out) {
    return guard([&] {
        if (!out) input_error("null output");
        resample(num_subjects, seed, stream, out);
    });
}

bsccs_status bsccs_state_create(const bsccs_dataset* ds, const double* beta, bsccs_state** out) {
    return guard([&] { *out = state_create(ds, beta); });
}
bsccs_status bsccs_state_clone(const bsccs_state* src, bsccs_state** out) {
    return guard([&] {
        if (!src) input_error("null state");
        *out = state_clone(src);
    });
}
bsccs_status bsccs_state_destroy(bsccs_state* st) {
    return guard([&] { state_destroy(st); });
}
bsccs_status bsccs_dense_recompute(bsccs_state* st, const double* beta) {
    return guard([&] {
        if (!st) input_error("null state");
        dense_recompute(st, beta);
    });
}
bsccs_status bsccs_grad_hess(bsccs_state* st, int32_t j, double* g, double* h) {
    return guard([&] {
        if (!st) input_error("null state");
        grad_hess(st, j, g, h);
    });
}
bsccs_status bsccs_sparse_update(bsccs_state* st, int32_t j, double delta) {
    return guard([&] {
        if (!st) input_error("null state");
        sparse_update(st, j, delta);
    });
}
bsccs_status bsccs_log_likelihood(bsccs_state* st, double* out) {
    return guard([&] {
        if (!st) input_error("null state");
        *out = log_likelihood(st);
    });
}
bsccs_status bsccs_state_get(bsccs_state* st, double* beta, double* xbeta, double* le, double* den) {
    return guard([&] {
        if (!st) input_error("null state");
        state_get(st, beta, xbeta, le, den);
    });
}

bsccs_status bsccs_penalized_step(const bsccs_prior* prior, double beta_j, double g, double h, double* step) {
    return guard([&] {
        const PriorParams p = to_params(prior);
        // the sweep kernel's form (prior.h penalized_step_pre), checked
        // against the reference expression form below
        double a = 0.0, b = 0.0;
        const int e = penalized_step_pre(p, beta_j, beta_over_v(p, beta_j), g, h, &a);
        const int e2 = penalized_step(p, beta_j, g, h, &b);
        if (e != e2 || (e == 0 && !(a == b || (a != a && b != b))))
            internal_error("penalized_step: precomputed form disagrees with the reference form");
        if (e) throw_device_error(e, 0.0);
        *step = a;
    });
}

bsccs_status bsccs_log_density(const bsccs_prior* prior, const double* beta, int32_t n, double* out) {
    return guard([&] {
        const PriorParams p = to_params(prior);
        *out = log_density(p, beta, n);
    });
}

bsccs_status bsccs_run_cycle(bsccs_state* st, const bsccs_prior* prior, const bsccs_solver_config* cfg,
                             const int32_t* order, double* trust, double* criterion) {
    return guard([&] {
        if (!st || !trust || !criterion) input_error("run_cycle: null argument");
        validate_config(cfg);
        const PriorParams p = to_params(prior);
        const int32_t J = st->ds->J;
        set_device(st->ds->device);
        if (order) {
            std::vector<char> seen(static_cast<size_t>(J), 0);
            for (int32_t i = 0; i < J; ++i) {
                if (order[i] < 0 || order[i] >= J || seen[static_cast<size_t>(order[i])])
                    input_error("run_cycle: order must be a permutation of the coordinates");
                seen[static_cast<size_t>(order[i])] = 1;
            }
            st->order_h.assign(order, order + J);
        } else {
            st->order_h.clear();
        }
        CUDA_TRY(cudaMemcpyAsync(st->trust, trust, sizeof(double) * J, cudaMemcpyHostToDevice, st->stream));
        ExchangePlan plan;
        plan.shards = {st};
        plan.dst = {st->slots};
        plan.local_slots = st->slots;
        plan.counter = st->counter;
        plan.total_participants = st->ds->ctas;
        plan.participant_base = 0;
        const SweepOutcome o = run_sweep(plan, p, cfg->convergence != 0, cfg->path == 1);
        CUDA_TRY(cudaMemcpy(trust, st->trust, sizeof(double) * J, cudaMemcpyDeviceToHost));
        *criterion = o.criterion;
    });
}

bsccs_status bsccs_fit(const bsccs_dataset* ds, const bsccs_prior* prior, const bsccs_solver_config* cfg,
                       const double* init_beta, double* beta_out, bsccs_fit_result* result) {
    return guard([&] {
        if (!ds || !beta_out || !result) input_error("fit: null argument");
        validate_config(cfg);
        const PriorParams p = to_params(prior);
        fit_resident(ds, p, cfg, init_beta, beta_out, result);
    });
}

// ---- groups ----------------------------------------------------------------

int64_t bsccs_group_slot_bytes(int32_t total_ctas) {
    (void)total_ctas; // the fixed-point exchange area does not grow with P
    // polled half + local half (hierarchical exchange)
    return 2 * static_cast<int64_t>(kXchgAreaWords) * static_cast<int64_t>(sizeof(unsigned long long));
}

bsccs_status bsccs_group_create_local(bsccs_dataset* const* shards, int32_t n, bsccs_group** out) {
    return guard([&] {
        if (!shards || n < 1 || n > kMaxLocalShards) input_error("group: 1..8 local shards");
        auto g = std::make_unique<bsccs_group>();
        g->device = shards[0]->device;
        for (int32_t i = 0; i < n; ++i) {
            if (!shards[i] || shards[i]->device != g->device) input_error("group: shards must share one device");
            if (shards[i]->J != shards[0]->J) input_error("group: shards must have the same drug count");
            g->shards.push_back(shards[i]);
            g->total += shards[i]->ctas;
        }
        set_device(g->device);
        CUDA_TRY(cudaMalloc(&g->slots, static_cast<size_t>(bsccs_group_slot_bytes(g->total))));
        CUDA_TRY(cudaMemset(g->slots, 0, static_cast<size_t>(bsccs_group_slot_bytes(g->total))));
        CUDA_TRY(cudaMalloc(&g->counter, sizeof(unsigned long long)));
        CUDA_TRY(cudaMemset(g->counter, 0, sizeof(unsigned long long)));
        g->peer = {g->slots};
        *out = g.release();
    });
}

bsccs_status bsccs_group_create_virtual(bsccs_dataset* const* shards, int32_t n, bsccs_group** out) {
    return guard([&] {
        if (!shards || n < 1 || n > kMaxRanks) input_error("group: 1..8 virtual ranks");
        auto g = std::make_unique<bsccs_group>();
        g->device = shards[0]->device;
        set_device(g->device);
        for (int32_t i = 0; i < n; ++i) {
            if (!shards[i] || shards[i]->device != g->device) input_error("group: shards must share one device");
            if (shards[i]->J != shards[0]->J) input_error("group: shards must have the same drug count");
            g->shards.push_back(shards[i]);
            g->total += shards[i]->ctas;
            unsigned long long* area = nullptr;
            unsigned long long* ctr = nullptr;
            CUDA_TRY(cudaMalloc(&area, static_cast<size_t>(bsccs_group_slot_bytes(0))));
            CUDA_TRY(cudaMemset(area, 0, static_cast<size_t>(bsccs_group_slot_bytes(0))));
            CUDA_TRY(cudaMalloc(&ctr, sizeof(unsigned long long)));
            CUDA_TRY(cudaMemset(ctr, 0, sizeof(unsigned long long)));
            g->vslots.push_back(area);
            g->vcounters.push_back(ctr);
        }
        g->peer = g->vslots;
        g->slots = g->vslots[0];
        g->counter = g->vcounters[0];
        g->hier = n > 1 && group_hier_from_env();
        *out = g.release();
    });
}

bsccs_status bsccs_group_create_rank(bsccs_dataset* shard, int32_t rank, int32_t world,
                                     const int32_t* ctas_per_rank, bsccs_group** out) {
    return guard([&] {
        if (!shard || world < 1 || world > kMaxRanks || rank < 0 || rank >= world || !ctas_per_rank)
            input_error("group: bad rank / world");
        if (ctas_per_rank[rank] != shard->ctas) input_error("group: ctas_per_rank disagrees with the shard");
        auto g = std::make_unique<bsccs_group>();
        g->device = shard->device;
        g->shards = {shard};
        g->rank = rank;
        g->world = world;
        g->ctas_per_rank.assign(ctas_per_rank, ctas_per_rank + world);
        for (int32_t r = 0; r < world; ++r) {
            if (r < rank) g->base += ctas_per_rank[r];
            g->total += ctas_per_rank[r];
        }
        set_device(g->device);
        CUDA_TRY(cudaMalloc(&g->slots, static_cast<size_t>(bsccs_group_slot_bytes(g->total))));
        CUDA_TRY(cudaMemset(g->slots, 0, static_cast<size_t>(bsccs_group_slot_bytes(g->total))));
        CUDA_TRY(cudaMalloc(&g->counter, sizeof(unsigned long long)));
        CUDA_TRY(cudaMemset(g->counter, 0, sizeof(unsigned long long)));
        g->peer.assign(static_cast<size_t>(world), nullptr);
        g->peer[static_cast<size_t>(rank)] = g->slots;
        g->hier = world > 1 && group_hier_from_env();
        *out = g.release();
    });
}

bsccs_status bsccs_group_ipc_handle(bsccs_group* g, uint8_t out[64]) {
    return guard([&] {
        if (!g) input_error("null group");
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
        cudaIpcMemHandle_t h;
        set_device(g->device);
        CUDA_TRY(cudaIpcGetMemHandle(&h, g->slots));
        std::memcpy(out, &h, 64);
    });
}

bsccs_status bsccs_group_open_peers(bsccs_group* g, const uint8_t* handles) {
    return guard([&] {
        if (!g || !handles) input_error("null argument");
        set_device(g->device);
        for (int32_t r = 0; r < g->world; ++r) {
            if (r == g->rank) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + 64 * r, 64);
            void* p = nullptr;
            CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            g->peer[static_cast<size_t>(r)] = static_cast<unsigned long long*>(p);
        }
    });
}

bsccs_status bsccs_group_destroy(bsccs_group* g) {
    return guard([&] {
        if (!g) return;
        cudaSetDevice(g->device);
        if (!g->vslots.empty()) {
            for (auto* p : g->vslots) cudaFree(p);
            for (auto* p : g->vcounters) cudaFree(p);
            delete g;
            return;
        }
        for (int32_t r = 0; r < g->world; ++r)
            if (r != g->rank && g->peer.size() > static_cast<size_t>(r) && g->peer[static_cast<size_t>(r)])
                cudaIpcCloseMemHandle(g->peer[static_cast<size_t>(r)]);
        cudaFree(g->slots);
        cudaFree(g->counter);
        delete g;
    });
}

bsccs_status bsccs_group_fit(bsccs_group* g, const bsccs_prior* prior, const bsccs_solver_config* cfg,
                             const double* init_beta, double* beta_out, bsccs_fit_result* result) {
    return guard([&] {
        NvtxRange nvtx_("bsccs_group_fit");
        if (!g || !beta_out || !result) input_error("group fit: null argument");
        validate_config(cfg);
        const PriorParams p = to_params(prior);
        for (auto* pr : g->peer)
            if (!pr) input_error("group fit: peers not opened");
        set_device(g->device);
        std::memset(result, 0, sizeof *result);
        cudaEvent_t e0, e1;
        CUDA_TRY(cudaEventCreate(&e0));
        CUDA_TRY(cudaEventCreate(&e1));
        CUDA_TRY(cudaEventRecord(e0, nullptr));
        FitContext fc;
        try {
            if (init_beta)
                for (int32_t j = 0; j < g->shards[0]->J; ++j)
                    if (!std::isfinite(init_beta[j])) input_error("init_state: non-finite coefficient");
            // states start from beta = 0 (cannot fail on one rank alone); the
            // caller's start is applied under agreement below
            for (auto* ds : g->shards) fc.states.push_back(acquire_state(ds, g->world > 1 ? nullptr : init_beta));
            fc.plan.shards = fc.states;
            fc.plan.dst = g->peer;
            fc.plan.local_slots = g->slots;
            fc.plan.counter = g->counter;
            fc.plan.total_participants = g->total;
            fc.plan.participant_base = g->base;
            fc.plan.shard_slots = g->vslots;
            fc.plan.shard_counters = g->vcounters;
            fc.plan.hier = g->hier;
            if (g->hier) {
                if (g->vslots.empty()) fc.plan.shard_local = {g->slots + kXchgAreaWords};
                else
                    for (auto* a : g->vslots) fc.plan.shard_local.push_back(a + kXchgAreaWords);
            }
            // per-rank log-likelihood partials summed exactly in the exchange
            // area (positive and negative parts: the words carry values >= 0)
            auto allreduce = [&](double x) {
                if (g->world == 1) return x;
                double pos = 0.0, neg = 0.0;
                plan_allreduce(fc.plan, x > 0.0 ? x : 0.0, x < 0.0 ? -x : 0.0, &pos, &neg);
                return pos - neg;
            };
            // every rank's status, one base-16 digit per status code (at
            // most 8 ranks per digit, so digits never carry)
            Agree agree = rethrow_local;
            if (g->world > 1)
                agree = [&](std::exception_ptr e) {
                    int code = 0;
                    if (e) {
                        try {
                            std::rethrow_exception(e);
                        } catch (const Error& x) {
                            code = static_cast<int>(x.code);
                        } catch (...) {
                            code = BSCCS_INTERNAL_ERROR;
                        }
                    }
                    double tot = 0.0, unused = 0.0;
                    plan_allreduce(fc.plan, code > 0 && code < 8 ? std::ldexp(1.0, 4 * code) : 0.0, 0.0, &tot,
                                   &unused);
                    if (e) std::rethrow_exception(e);
                    for (int c = 1; c < 8; ++c)
                        if (std::fmod(std::floor(std::ldexp(tot, -4 * c)), 16.0) != 0.0)
                            fail(static_cast<bsccs_status>(c), "group fit: another rank of the group failed (status " +
                                                                   std::to_string(c) + "); see that rank's error");
                };
            if (g->world > 1 && init_beta)
                agreed(agree, [&] {
                    for (auto* st : fc.states) dense_recompute(st, init_beta);
                });
            fit_loop(fc, p, cfg, beta_out, result, allreduce, agree);
        } catch (...) {
            for (auto* st : fc.states) release_state(st);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            throw;
        }
        for (auto* st : fc.states) release_state(st);
        CUDA_TRY(cudaEventRecord(e1, nullptr));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        result->device_seconds = ms * 1e-3;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

} // extern "C"
