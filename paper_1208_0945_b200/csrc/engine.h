// engine.h -- device-resident dataset / state and the internal engine API.
//
// HBM layout:
//   pairs     int2[nnz]      {row, subject} of every nonzero, CSC order
//                            (SparseColumn::rows/::subjects interleaved,
//                            dataset.hpp:38-43): dataset build, batched
//                            engine, subset builder, export
//   pq        int4[nnz]      the sweep's view of the same pairs:
//                            {era slot, subject block slot, era length,
//                            subject index within its CTA's range}
//   split     int64[J][C+1]  first pair of column j owned by CTA c; CTAs own
//                            contiguous subject ranges, so a column's pairs
//                            split into C contiguous, subject-aligned slices
//   csr_ptr/  row -> drug list (ascending), built once by a stable radix sort;
//   csr_col                  gives dense_recompute the reference's per-row
//                            addition order (engine.hpp:173-181) w/o atomics
//   X         f64 slots      per subject one block [den, n, x'beta of each
//                            era]: a block of <= 16 slots never straddles a
//                            128-B line, so a scattered pair visit reads ONE
//                            line for its era's x'beta and its subject's
//                            denominator (the L2 fills whole 128-B lines:
//                            scripts/gbench4.cu).  l*exp(x'beta) recomputed.
//   row_slot  int32[K]       slot of era k; bstart int32[N]: block of subject i
//   snap      8 B / era      criterion snapshot (streamed once per cycle)
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h> // header-only NVTX v3: ranges cost nothing unless a tool attaches

#include <cstdint>
#include <string>
#include <vector>

#include "prior.h"
#include "status.h"

namespace bsccs_b200 {

// l*exp(x'beta) is not stored: the reference keeps l_exp_xbeta[k] ==
// era_lengths[k] * exp(xbeta[k]) bit for bit at every write (init_state and
// dense_recompute, engine.hpp:77-78; sparse_delta_update, engine.hpp:221-228),
// so the device recomputes it from x'beta and the length in the pair stream.
//
// Subject blocks: slot bstart[i] = denominator (EngineState::denominators),
// bstart[i] + 1 = n_i as a double (events_per_subject, exact), then one slot
// of x'beta (EngineState::xbeta) per era of the subject in row order.
constexpr int kBlockHeader = 2;
constexpr int kLineSlots = 16;    // 128-B line / 8-B slot
constexpr int kBlockChunk = 64;   // subjects packed per build thread (each chunk starts on a line)

// Pair record of the resident-beta sweep (k_rcd, rsweep.cuh), CSC order,
// 32 B: the subject's index within its CTA's range, the era length, meta =
// the number of OTHER drugs of the era (bits 0-7) | how many of them sort
// before the pair's own drug (bits 8-15) | n_i (bits 16-31), the first
// overflow entry (more than 8 other drugs; each list padded with 0xffff to
// a multiple of 8 entries, 16-B aligned), and up to 8 other drugs of the
// era ascending (0xffff padding).  A pair's x'beta is rebuilt from these and beta in the
// order of engine.hpp:173-181.
struct alignas(16) RRec {
    // meta: other drugs (bits 0-7) | run head (bit 8) | run continues (bit 9) | n_i << 16
    int32_t ls, len, meta, ovf;
    uint16_t o[8];
};
static_assert(sizeof(RRec) == 32, "pair record is 32 B");
constexpr int kRInline = 8;          // other drugs carried in the record
constexpr int kRMaxOthers = 254;     // meta bits 0-7 (an era of at most 255 drugs)
constexpr int32_t kRMaxEvents = 65535; // meta bits 16-31

// Per-state device scalars written by kernels, mirrored to pinned host.
struct DevResult {
    double g, h;              // tier-1 grad/hess
    double criterion;         // last sweep
    double change, magnitude; // criterion components
    double ll_linear, ll_logden;
    double err_value;
    long long visited, moved;
    unsigned long long counter; // exchange sequence after the launch
    int err_code;
    int err_remote; // error seen in the exchange (possibly another shard)
    int refine_at;  // sweep stopped before this visit-list entry: its sums need refinement (run_sweep)
};

struct DevErr {
    int code;
    int pad;
    double value;
};

#ifndef BSCCS_SWEEP_THREADS
#define BSCCS_SWEEP_THREADS 384
#endif
constexpr int kSweepThreads = BSCCS_SWEEP_THREADS;
constexpr int kMaxLocalShards = 8;
constexpr int kMaxRanks = 8;
constexpr int kXchgAreaWords = 512; // exchange words (2 x 7, 256 B apart) + running totals

struct bsccs_dataset_impl;
} // namespace bsccs_b200

// Opaque handle types of the C ABI.
struct bsccs_dataset {
    int device = 0;
    cudaStream_t stream = nullptr; // allocation / build stream (pool frees are ordered on it)
    int32_t N = 0, K = 0, J = 0;
    int64_t nnz = 0;
    int ctas = 0;
    // device arrays
    int2* pairs = nullptr;
    int4* pq = nullptr;               // [nnz] {era slot, block slot, era length, subject - cta_subj[c]}
    int32_t* row_slot = nullptr;      // [K]
    int32_t* bstart = nullptr;        // [N]
    int64_t nslots = 0;               // slots of the per-subject blocks
    int64_t* col_ptr = nullptr;
    int64_t* split = nullptr;         // [J*(ctas+1)]
    int32_t* cta_era = nullptr;       // [ctas+1]
    int32_t* cta_subj = nullptr;      // [ctas+1]
    int32_t* subject_offsets = nullptr;
    int32_t* events_per_subject = nullptr;
    int32_t* era_lengths = nullptr;
    int32_t* event_counts = nullptr;
    int64_t* csr_ptr = nullptr;       // [K+1]
    int32_t* csr_col = nullptr;       // [nnz]
    double* y_dot_x = nullptr;        // [J] global y_dot_x as double
    uint8_t* col_nonempty = nullptr;  // [J] global
    int32_t* col_runs = nullptr;      // [J] subject runs per column (this shard)
    int32_t max_cta_subjects = 0;     // largest CTA subject range (sizes the shared-memory subject tile)
    int32_t max_cta_eras = 0;         // largest CTA era range (sizes the criterion's chunk table)
    int32_t max_slice = 0;            // largest per-CTA slice of any column (streamed path needed above kCap)
    // resident-beta sweep (rsweep.cuh): pair records and overflow drug lists;
    // rq == nullptr when the dataset does not qualify (J > 65535, nnz >= 2^32,
    // an era with more than 256 drugs, n_i >= 2^23, or BSCCS_SWEEP=classic)
    bsccs_b200::RRec* rq = nullptr;
    uint16_t* rovf = nullptr;
    int64_t novf = 0;
    uint8_t* edeg = nullptr;   // [K] drugs per era, [nnz] drugs as u16: the sweep's criterion pass
    uint16_t* ecol = nullptr;
    int32_t max_deg = 0;       // drugs of the largest era
    // host copies of small metadata
    std::vector<int64_t> col_ptr_h;
    std::vector<uint8_t> col_nonempty_h;
    std::vector<int32_t> col_runs_h;
    std::vector<std::string> drug_ids; // labels (Dataset::drug_ids), may be empty
    int64_t device_bytes = 0;
};

struct bsccs_group;

struct bsccs_state {
    const bsccs_dataset* ds = nullptr;
    cudaStream_t stream = nullptr;
    double* X = nullptr;                 // [ds->nslots] subject blocks {den, n, x'beta...}
    double* snap = nullptr;              // [K] criterion snapshot
    double* le_tmp = nullptr;            // [K] scratch for state_get
    double* num = nullptr;               // [N] run numerators of the dense path (lazy)
    double* beta = nullptr;
    double* trust = nullptr;
    int32_t* visit = nullptr;            // [J] this cycle's visit list (device)
    longlong2* vsplit = nullptr;         // [ctas][J] slice bounds in visit order
    uint8_t* moved = nullptr;            // [J] moved flag per visited coordinate
    std::vector<int32_t> order_h;        // visit order (empty = ascending)
    std::vector<int32_t> visit_h;        // visit list last uploaded
    bool visit_valid = false;
    // exchange (own slot buffer; a group overrides it)
    unsigned long long* slots = nullptr; // [2][ctas][4]
    unsigned long long* counter = nullptr;
    bsccs_b200::DevErr* err = nullptr;
    bsccs_b200::DevResult* res = nullptr;   // device
    bsccs_b200::DevResult* res_h = nullptr; // pinned host mirror
    double* scratch = nullptr;              // reduction partials
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // resident-beta sweep: compact denominators [N] and beta at cycle start.
    // The sweep keeps denc current and leaves X's x'beta / headers stale
    // (x_stale) until an op that reads X rebuilds them (sync_x); ops that
    // write X leave denc stale (denc_valid false) until the next sweep
    // gathers it from the headers.
    double* denc = nullptr;
    double* beta_prev = nullptr;
    bool denc_valid = false;
    bool x_stale = false;
    double sweep_ms = 0.0;  // accumulated sweep-kernel time
    double alg_bytes = 0.0; // accumulated algorithmic bytes of the sweeps
    bool snap_valid = false;
    // a fit ended with k_final_xb / k_final_den (its closing refresh computed, not
    // written): the next use of the state rebuilds it (settle_dense)
    bool dense_pending = false;
};

namespace bsccs_b200 {

// NVTX range over a host-side phase (visible in nsys / ncu --nvtx timelines)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

void cuda_check(cudaError_t e, const char* what);
void count_launches(int n);
long long launch_count();
#define CUDA_TRY(x) ::bsccs_b200::cuda_check((x), #x)

int default_ctas(int device);

// ---- dataset / state -------------------------------------------------------
bsccs_dataset* dataset_create(int32_t N, int32_t K, int32_t J, int64_t nnz,
                              const int32_t* subject_offsets, const int32_t* events_per_subject,
                              const int32_t* era_lengths, const int32_t* event_counts,
                              const int64_t* col_ptr, const int32_t* rows, const int32_t* subjects,
                              const int64_t* y_dot_x_global, const int64_t* col_nnz_global,
                              int device, int ctas_override);
void dataset_destroy(bsccs_dataset* ds);
// building blocks of dataset_create, shared with the device-side subset
bsccs_dataset* dataset_new(int32_t N, int32_t K, int32_t J, int64_t nnz, int device, int ctas_override);
void finish_dataset(bsccs_dataset* ds, int32_t* d_rows, int32_t* d_subj, const int64_t* y_dot_x_global,
                    const int64_t* col_nnz_global, cudaEvent_t era_ready = nullptr);
// subset_dataset (dataset.hpp:157-217) built on the device (subset.cu)
bsccs_dataset* dataset_subset(const bsccs_dataset* parent, const int32_t* subject_indices, int64_t n,
                              int ctas_override);
void dataset_export(const bsccs_dataset* ds, int32_t* subject_offsets, int32_t* events_per_subject,
                    int32_t* era_lengths, int32_t* event_counts, int64_t* col_ptr, int32_t* rows, int32_t* subjects,
                    int64_t* y_dot_x);
void kfold_split(int32_t N, int32_t folds, uint64_t seed, int32_t* subjects_out, int32_t* fold_sizes);
// Dataset from host arrays whose pairs come in row order (drug ascending
// within a row): (drug, row, subject) triples; the CSC is built on the
// device by a stable sort on the drug (subset.cu).
bsccs_dataset* dataset_from_row_pairs(int32_t N, int32_t K, int32_t J, int64_t nnz, const int32_t* subject_offsets,
                                      const int32_t* events_per_subject, const int32_t* era_lengths,
                                      const int32_t* event_counts, const uint32_t* drug, const int2* row_subj,
                                      int device, int ctas_override);
// read_long_format (io.hpp:88-174) + build_dataset (dataset.hpp:74-152) into a
// resident dataset (loader.cpp)
bsccs_dataset* load_long_format(const char* path, const char* const* dictionary, int32_t dict_size, int device,
                                int ctas_override, int threads);
void resample(int32_t N, uint64_t seed, uint64_t stream, int32_t* out);

bsccs_state* state_create(const bsccs_dataset* ds, const double* beta_host);
bsccs_state* state_clone(const bsccs_state* src);
void state_destroy(bsccs_state* st);

// ---- engine ops (all synchronous on the state's stream) -----------------
void dense_recompute(bsccs_state* st, const double* beta_host); // nullptr: from state beta
void dense_recompute_zero(bsccs_state* st);                      // beta := 0 and the state it implies
// the closing dense refresh and log-likelihood of a fit, without writing the
// state back (rebuilt on its next use)
double final_log_likelihood(bsccs_state* st);
void grad_hess(bsccs_state* st, int32_t j, double* g, double* h);
void sparse_update(bsccs_state* st, int32_t j, double delta);
double log_likelihood(bsccs_state* st);
void state_get(bsccs_state* st, double* beta, double* xbeta, double* le, double* den);

// ---- sweep ---------------------------------------------------------------
struct SweepOutcome {
    double criterion;
    long long visited, moved;
};

// One cycle over `order` (device array already uploaded, or identity) on a
// set of shards that exchange through the given slot buffers.
struct ExchangePlan {
    std::vector<bsccs_state*> shards;      // local shards (same device)
    std::vector<unsigned long long*> dst;  // slot buffers to publish into
    unsigned long long* local_slots;       // slot buffer to poll
    unsigned long long* counter;           // sequence word (local)
    // virtual ranks inside one launch: per-shard poll area / counter (each
    // shard is its own "rank"; every CTA adds into every area of `dst`)
    std::vector<unsigned long long*> shard_slots, shard_counters;
    int total_participants;                // CTAs across all ranks
    int participant_base;                  // first participant of shard 0
    // hierarchical exchange (multi-rank groups, ccd_kernels.cu forward_local):
    // per local shard the local area its CTAs add into; `dst` then receives
    // one arrival per rank
    bool hier = false;
    std::vector<unsigned long long*> shard_local;
};

SweepOutcome run_sweep(const ExchangePlan& plan, const PriorParams& prior, bool normalized, bool dense = false);
void plan_allreduce(const ExchangePlan& plan, double a, double b, double* ta, double* tb);
void prepare_snapshot(bsccs_state* st);
void set_debug_flags(int flags); // profiling only
void set_debug_sweep(int kind, double beta_limit); // tests only (bsccs_debug_set_sweep)
int debug_last_sweep();
int debug_last_rcd_shape();
void set_debug_trace(int ncoords, int ctas);
void read_debug_trace(unsigned long long* host, size_t words);
void debug_exchange_sum(int device, const double* partials, int n, double* sum, int* status);
unsigned long long* debug_trace_buffer(int* ncoords); // profiling only
void throw_device_error(int code, double value);

// ---- host driver (capi.cpp) ---------------------------------------------
PriorParams to_params(const bsccs_prior* p);                // validate_prior + constants
void validate_config(const bsccs_solver_config* c);         // validate_config + device knobs
double log_density(const PriorParams& p, const double* beta, int32_t n);
void fit_resident(const bsccs_dataset* ds, const PriorParams& p, const bsccs_solver_config* cfg,
                  const double* init_beta, double* beta_out, bsccs_fit_result* result);
void release_dataset_workspaces(const bsccs_dataset* ds);

// ---- batched weighted engine (batch.cu) ---------------------------------
void build_vsplit(const bsccs_dataset* ds, const int32_t* d_visit, int V, longlong2* out, cudaStream_t s);
struct Batch;
Batch* batch_create(const bsccs_dataset* ds, int RB);
void batch_destroy(Batch* b);
void batch_set_weights(Batch* b, const int32_t* m_host, const int32_t* mheld_host); // [N][RB]
void batch_set_resamples(Batch* b, const int32_t* idx_host, int R);                 // [R][N]
void batch_set_weight_rows(Batch* b, const int32_t* rows_host, int R);              // [R][N], NULL = ones
void batch_set_folds(Batch* b, const int32_t* fold_of_host, const int32_t* fold_r, int R);
void batch_fit(Batch* b, int R, const PriorParams* priors, const double* const* init, const bsccs_solver_config* cfg,
               double* beta_out, bsccs_fit_result* res, int* err_code, double* pred_ll);
double batch_sweep_ms(const Batch* b);
double batch_alg_bytes(const Batch* b);
void cv_folds_batched(const bsccs_dataset* ds, const bsccs_cv_config* cfg, const std::vector<double>& grid,
                      const std::vector<int32_t>& fold_subjects, const std::vector<int32_t>& fold_sizes, int32_t f0,
                      int32_t f1, bsccs_cv_cell* cells, bsccs_cv_result* res);
void boot_replicates_batched(const bsccs_dataset* ds, const bsccs_bootstrap_config* cfg, const double* beta_full,
                             int32_t r0, int32_t r1, double* est, int32_t* conv, bsccs_bootstrap_result* res);

} // namespace bsccs_b200
