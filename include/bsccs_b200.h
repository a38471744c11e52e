/*
 * bsccs_b200.h -- C ABI of the B200-native CCD hot path.
 *
 * This is the drop-in boundary for the cyclic-coordinate-descent (CCD)
 * MAP fit of the Bayesian self-controlled case series model
 * (arXiv 1208.0945).  The reference (`bsccs`, header-only C++20 under
 * /root/reference/proj/include/bsccs) has no FFI: its engine is templated
 * over EngineState<RealType> and called directly by the solver.  Every entry
 * point below names the reference symbol it replaces (file:line relative to
 * /root/reference/proj/include/bsccs/).  Plain pointers and sizes only; no
 * C++ or torch types cross this boundary.
 *
 * Conventions
 *   - Every function returns a bsccs_status.  BSCCS_OK == 0.  On failure the
 *     thread-local message is available from bsccs_last_error().  The status
 *     codes mirror the reference exception types (common.hpp:10-35):
 *       BSCCS_INPUT_ERROR       <- bsccs::input_error
 *       BSCCS_NUMERIC_ERROR     <- bsccs::numeric_error
 *       BSCCS_CONVERGENCE_ERROR <- bsccs::convergence_error
 *       BSCCS_INTERNAL_ERROR    <- bsccs::internal_error
 *       BSCCS_CUDA_ERROR        a CUDA runtime failure (no reference analogue)
 *   - Host arrays are borrowed for the duration of the call only.
 *   - A dataset handle owns its device-resident copy and may be shared
 *     read-only by any number of state handles on the same device.
 *   - A state handle owns one fit's mutable device vectors and its stream.
 *     Distinct handles may be used from distinct host threads.
 *   - index type is int32 (common.hpp:8); pair offsets are int64.
 */
#ifndef BSCCS_B200_H
#define BSCCS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSCCS_B200_ABI_VERSION 1

typedef enum bsccs_status {
    BSCCS_OK = 0,
    BSCCS_INPUT_ERROR = 1,
    BSCCS_NUMERIC_ERROR = 2,
    BSCCS_INTERNAL_ERROR = 3,
    BSCCS_CONVERGENCE_ERROR = 4,
    BSCCS_CUDA_ERROR = 5
} bsccs_status;

/* PriorSpec (prior.hpp:17-25).  kind: 0 none, 1 normal, 2 laplace
 * (PriorKind, prior.hpp:10). */
typedef struct bsccs_prior {
    int32_t kind;
    int32_t variance_is_laplace_scale;
    double variance;
} bsccs_prior;

/* SolverConfig (solver.hpp:21-46).  convergence: 0 raw_sum, 1 normalized.
 * precision: 1 Double (0 Single is rejected with BSCCS_INPUT_ERROR: the
 * device path is fp64 only).  path: 0 sparse, 1 dense (the reference's
 * UpdatePath::dense benchmark route, run by k_ccd_dense on an unsharded
 * dataset).
 * partitions / min_parallel_nnz are accepted and ignored: the device
 * reduction fixes its own partition (one per CTA), see DESIGN.md. */
typedef struct bsccs_solver_config {
    double epsilon;
    int32_t max_cycles;
    int32_t convergence;
    double trust_init;
    int32_t precision;
    int32_t path;
    int32_t partitions;
    int32_t dense_refresh_interval;
    int32_t random_cycle;
    int32_t reserved0;
    uint64_t cycle_seed;
    uint64_t min_parallel_nnz;
} bsccs_solver_config;

/* FitResult (solver.hpp:66-72); beta_map goes to a caller buffer. */
typedef struct bsccs_fit_result {
    double log_posterior;
    double final_criterion;
    int32_t cycles_run;
    int32_t converged;
    /* instrumentation, not in the reference struct */
    int64_t coordinates_visited; /* non-skipped coordinate steps, all cycles */
    int64_t coordinates_moved;   /* of those, steps with delta != 0        */
    int64_t dense_refreshes;     /* dense_recompute calls incl. the final */
    double device_seconds;       /* fit() entry -> FitResult, CUDA events  */
    double sweep_seconds;        /* sum of sweep-kernel durations (events on
                                    the launching stream)                  */
    double algorithmic_bytes;    /* SURVEY §8(d) byte model summed over the
                                    sweep kernels of this fit              */
    int64_t kernel_launches;     /* library kernels launched by this fit   */
} bsccs_fit_result;

typedef struct bsccs_dataset bsccs_dataset;
typedef struct bsccs_state bsccs_state;

/* ---- library ---------------------------------------------------------- */
int32_t bsccs_abi_version(void);
const char* bsccs_last_error(void);
/* Number of CTAs the persistent sweep kernel uses on `device` (one per SM
 * times the resident count).  Fixed per dataset at creation. */
bsccs_status bsccs_device_info(int32_t device, int32_t* sm_count, int32_t* ctas);
/* Process-wide count of kernels this library has launched (evidence that
 * the device path ran; bench.py reports it as gpu_launches). */
int64_t bsccs_launch_count(void);
/* Profiling hook, not a reference entry point: sweep phases to skip (bit0
 * grad/hess gathers, bit1 update, bit2 exchange).  0 = normal. */
void bsccs_debug_set_sweep_flags(int32_t flags);
/* Profiling hook: host_out == NULL arms per-CTA globaltimer stamps for the
 * first ncoords coordinates of later sweeps; otherwise copies them out. */
int32_t bsccs_debug_trace(int32_t ncoords, int32_t ctas, uint64_t* host_out, int64_t words);
/* Test hooks, not reference entry points.  Sweep kernel for later cycles:
 * 0 automatic (the resident-beta sweep k_rcd when the dataset qualifies,
 * else k_ccd), 1 always k_ccd.  beta_limit > 0 lowers the |beta_j| bound
 * above which k_rcd hands the cycle to k_ccd (0 = the automatic
 * 700 / largest era).  bsccs_debug_last_sweep: kernel of the last cycle's
 * launches, 1 = k_ccd only, 2 = k_rcd only, 3 = both (handed over). */
void bsccs_debug_set_sweep(int32_t kind, double beta_limit);
int32_t bsccs_debug_last_sweep(void);
/* Test hook: shape of the last k_rcd launch, slots per thread | 16 if the
 * subject tile was in shared memory (0: none yet). */
int32_t bsccs_debug_last_rcd_shape(void);
/* Self-test of the exact all-reduce encoding, not a
 * reference entry point: n (<= 2048) partials in [0, 2^43) are split into
 * limbs and added into one set of exchange words on `device` exactly as n
 * participants would; *sum receives the reconstructed total and *status
 * 0 = ok, 1 = a partial out of range, 2 = total out of range, 3 = the
 * arrival count did not read n. */
bsccs_status bsccs_debug_exchange_sum(int32_t device, const double* partials, int32_t n, double* sum,
                                      int32_t* status);

/* ---- dataset (dataset.hpp:53-68 Dataset / SparseColumn) ---------------
 * Flat CSC form of bsccs::Dataset: column j's pairs are
 * [col_ptr[j], col_ptr[j+1]) of rows[] / subjects[] (SparseColumn::rows and
 * ::subjects concatenated, dataset.hpp:38-43).  y_dot_x may be NULL (it is
 * then recomputed on device from event_counts).  Validates the structural
 * invariants of build_dataset (dataset.hpp:74-152): offsets fenceposts,
 * rows ascending within a column, subject[p] owning rows[p].  subjects may
 * be NULL: each pair's subject is then derived on the device as the owner of
 * its row (what build_dataset stores, dataset.hpp:134), which saves the
 * upload of an array as large as rows.
 * num_ctas_override <= 0 selects the device default. */
bsccs_status bsccs_dataset_create(
    int32_t num_subjects, int32_t num_eras, int32_t num_drugs, int64_t nnz,
    const int32_t* subject_offsets,    /* [num_subjects + 1] */
    const int32_t* events_per_subject, /* [num_subjects]     */
    const int32_t* era_lengths,        /* [num_eras]         */
    const int32_t* event_counts,       /* [num_eras]         */
    const int64_t* col_ptr,            /* [num_drugs + 1]    */
    const int32_t* rows,               /* [nnz]              */
    const int32_t* subjects,           /* [nnz] or NULL      */
    const int64_t* y_dot_x,            /* [num_drugs] or NULL */
    int32_t device, int32_t num_ctas_override,
    bsccs_dataset** out);

/* Shard of a patient-partitioned dataset: the arrays are the
 * shard's own (subjects/eras renumbered from 0), while y_dot_x_global and
 * col_nnz_global describe the whole dataset so that the gradient and the
 * skip rule (solver.hpp:119-121) are the global ones. */
bsccs_status bsccs_dataset_create_shard(
    int32_t num_subjects, int32_t num_eras, int32_t num_drugs, int64_t nnz,
    const int32_t* subject_offsets, const int32_t* events_per_subject,
    const int32_t* era_lengths, const int32_t* event_counts,
    const int64_t* col_ptr, const int32_t* rows, const int32_t* subjects,
    const int64_t* y_dot_x_global, const int64_t* col_nnz_global,
    int32_t device, int32_t num_ctas_override,
    bsccs_dataset** out);

bsccs_status bsccs_dataset_destroy(bsccs_dataset* ds);
/* sizes: N, K, J, nnz, ctas, device bytes resident */
bsccs_status bsccs_dataset_info(const bsccs_dataset* ds, int64_t out[6]);

/* read_long_format (io.hpp:88-174) + build_dataset (dataset.hpp:74-152):
 * the era-level long format (subject_id TAB length_days TAB event_count
 * [TAB space-separated drug labels]) parsed by `threads` host threads (<= 0:
 * all) and laid out as CSC on the device.  Labels are numbered in
 * first-appearance order, or by `dictionary` when dict_size > 0.  Errors
 * (BSCCS_INPUT_ERROR) carry the reference's "path:line: ..." messages; with
 * several errors in a file the earliest line's is reported. */
bsccs_status bsccs_dataset_read_long_format(const char* path,
                                           const char* const* dictionary,
                                           int32_t dict_size, int32_t device,
                                           int32_t num_ctas_override,
                                           int32_t threads,
                                           bsccs_dataset** out);
/* Dataset::drug_ids (dataset.hpp:66): set (n == num_drugs, or 0 to clear)
 * and read back newline-separated (needed = bytes including the NUL). */
bsccs_status bsccs_dataset_set_drug_ids(bsccs_dataset* ds,
                                        const char* const* labels, int32_t n);
bsccs_status bsccs_dataset_drug_ids(const bsccs_dataset* ds, char* buf,
                                    int64_t capacity, int64_t* needed);
/* subset_dataset (dataset.hpp:157-217), built on the device from a resident
 * dataset: subjects in the given order, repeats allowed (each occurrence an
 * independent copy).  Bit-identical layout to the reference's subset.
 * Empty selection or an index out of range: BSCCS_INPUT_ERROR. */
bsccs_status bsccs_dataset_subset(const bsccs_dataset* ds,
                                  const int32_t* subject_indices, int64_t n,
                                  int32_t num_ctas_override,
                                  bsccs_dataset** out);
/* Copies the flat CSC arrays of a resident dataset back to host (sizes from
 * bsccs_dataset_info); any pointer may be NULL. */
bsccs_status bsccs_dataset_export(const bsccs_dataset* ds,
                                  int32_t* subject_offsets,
                                  int32_t* events_per_subject,
                                  int32_t* era_lengths, int32_t* event_counts,
                                  int64_t* col_ptr, int32_t* rows,
                                  int32_t* subjects, int64_t* y_dot_x);
/* kfold_split (cross_validation.hpp:58-80): fold lists back to back in
 * subjects_out[num_subjects], their sizes in fold_sizes[folds]. */
bsccs_status bsccs_kfold_split(int32_t num_subjects, int32_t folds,
                               uint64_t seed, int32_t* subjects_out,
                               int32_t* fold_sizes);
/* resample (bootstrap.hpp:43-52) drawn from Rng(seed, stream); replicate r
 * of run_bootstrap uses stream r + 1 (bootstrap.hpp:104). */
bsccs_status bsccs_resample(int32_t num_subjects, uint64_t seed,
                            uint64_t stream, int32_t* out);

/* ---- tier 1: engine (engine.hpp) --------------------------------------- */
/* init_state (engine.hpp:137-166); beta may be NULL (zeros). */
bsccs_status bsccs_state_create(const bsccs_dataset* ds, const double* beta,
                                bsccs_state** out);
/* EngineState copy (engine.hpp:36-45 is a value type). */
bsccs_status bsccs_state_clone(const bsccs_state* src, bsccs_state** out);
bsccs_status bsccs_state_destroy(bsccs_state* st);
/* dense_recompute (engine.hpp:170-200); beta NULL = rebuild from state. */
bsccs_status bsccs_dense_recompute(bsccs_state* st, const double* beta);
/* fused_grad_hess / parallel_fused_grad_hess (engine.hpp:285-361). */
bsccs_status bsccs_grad_hess(bsccs_state* st, int32_t j, double* gradient,
                             double* hessian);
/* sparse_delta_update (engine.hpp:205-231). */
bsccs_status bsccs_sparse_update(bsccs_state* st, int32_t j, double delta);
/* log_likelihood (engine.hpp:404-425). */
bsccs_status bsccs_log_likelihood(bsccs_state* st, double* out);
/* Copies EngineState vectors to host; any pointer may be NULL. */
bsccs_status bsccs_state_get(bsccs_state* st, double* beta, double* xbeta,
                             double* l_exp_xbeta, double* denominators);

/* ---- prior (prior.hpp) -- host evaluation of the device code --------- */
bsccs_status bsccs_penalized_step(const bsccs_prior* prior, double beta_j,
                                  double g, double h, double* step);
bsccs_status bsccs_log_density(const bsccs_prior* prior, const double* beta,
                               int32_t n, double* out);

/* ---- tier 2: solver (solver.hpp) --------------------------------------- */
/* run_cycle (solver.hpp:101-166): one persistent-kernel sweep.  trust is the
 * per-coordinate radius vector (SolverState::trust, solver.hpp:88), in/out on
 * host; order is the visit order (NULL = ascending). */
bsccs_status bsccs_run_cycle(bsccs_state* st, const bsccs_prior* prior,
                             const bsccs_solver_config* cfg,
                             const int32_t* order, double* trust,
                             double* criterion);
/* fit (solver.hpp:206-220) on a resident dataset.  init_beta may be NULL;
 * beta_out has num_drugs entries. */
bsccs_status bsccs_fit(const bsccs_dataset* ds, const bsccs_prior* prior,
                       const bsccs_solver_config* cfg, const double* init_beta,
                       double* beta_out, bsccs_fit_result* result);
/* Defaults of SolverConfig{} (solver.hpp:21-46). */
void bsccs_solver_config_default(bsccs_solver_config* cfg);

/* ---- callers of fit: cross-validation and bootstrap -------------------- */
/* Engines for the many-fit drivers.
 *   BSCCS_ENGINE_SUBSET   the reference's route: every fold / replicate
 *                         dataset is materialised (bsccs_dataset_subset, on
 *                         the device) and fitted by the single-fit kernel.
 *   BSCCS_ENGINE_BATCHED  R fits share the parent dataset and every
 *                         per-coordinate exchange: a subject taken m times
 *                         carries weight m (0 when left out).  Same model and
 *                         visit order; sums differ from the materialised
 *                         dataset's by rounding only. */
#define BSCCS_ENGINE_SUBSET 0
#define BSCCS_ENGINE_BATCHED 1

/* R independent fits (1 <= R <= 16) on one resident dataset in one batched
 * launch per cycle: fit r weights subject i by weights[r * num_subjects + i]
 * (its multiplicity in the selection: 0 leaves it out, m > 1 repeats it;
 * NULL = every subject once), with its own prior and start (init_beta
 * [R x num_drugs] or NULL).  Equivalent to fit() on the materialised
 * selection (subset_dataset) up to summation order.  status[r] receives the
 * fit's own outcome (a failed fit does not stop the others). */
bsccs_status bsccs_fit_batch(const bsccs_dataset* ds, int32_t R,
                             const bsccs_prior* priors,
                             const int32_t* weights, const double* init_beta,
                             const bsccs_solver_config* cfg, double* beta_out,
                             bsccs_fit_result* results, int32_t* status);

/* CVConfig (cross_validation.hpp:29-41); the grid is passed separately. */
typedef struct bsccs_cv_config {
    int32_t folds;
    int32_t prior_kind;
    int32_t variance_is_laplace_scale;
    int32_t warm_start;
    uint64_t seed;
    bsccs_solver_config solver;
    int32_t engine;     /* BSCCS_ENGINE_* */
    int32_t batch;      /* batched engine: max fits per launch (<= 0: auto) */
} bsccs_cv_config;

/* CVCell (cross_validation.hpp:43-48). */
typedef struct bsccs_cv_cell {
    double predictive_ll;
    int32_t cycles;
    int32_t converged;
    int32_t valid;
    int32_t reserved;
} bsccs_cv_cell;

/* CVResult scalars (cross_validation.hpp:50-57); the vectors go to caller
 * buffers. */
typedef struct bsccs_cv_result {
    int32_t selected_index;
    int32_t points;
    double selected_variance;
    int64_t total_cycles;
    double device_seconds;      /* instrumentation */
    int64_t fits;               /* fits run */
    int64_t coordinates_visited;
} bsccs_cv_result;

/* Defaults of CVConfig{} (cross_validation.hpp:29-41): 10 folds, laplace,
 * seed 0, warm start, default SolverConfig; engine SUBSET. */
void bsccs_cv_config_default(bsccs_cv_config* cfg);
/* The 13-point default grid (cross_validation.hpp:19-27). */
void bsccs_default_variance_grid(double out[13]);

/* grid_search_cv (cross_validation.hpp:100-215).  grid_out[points] receives
 * the sorted grid, cells[points * folds] the cells ([grid point][fold]),
 * mean_predictive_ll[points] the fold means (NaN where a fold failed).  A
 * fit failing with a numeric/internal error marks its cell invalid; input
 * errors propagate; no usable grid point -> BSCCS_CONVERGENCE_ERROR. */
bsccs_status bsccs_grid_search_cv(const bsccs_dataset* ds,
                                  const bsccs_cv_config* cfg,
                                  const double* variance_grid, int32_t points,
                                  double* grid_out, bsccs_cv_cell* cells,
                                  double* mean_predictive_ll,
                                  bsccs_cv_result* result);
/* The fold loop of grid_search_cv for folds [fold_begin, fold_end) only
 * (ranks of a multi-GPU job each run a range); cells as above, only the
 * range's columns written. */
bsccs_status bsccs_cv_run_folds(const bsccs_dataset* ds,
                                const bsccs_cv_config* cfg,
                                const double* variance_grid, int32_t points,
                                int32_t fold_begin, int32_t fold_end,
                                bsccs_cv_cell* cells, bsccs_cv_result* result);
/* The selection step of grid_search_cv over complete cells. */
bsccs_status bsccs_cv_select(const double* sorted_grid, int32_t points,
                             int32_t folds, const bsccs_cv_cell* cells,
                             double* mean_predictive_ll,
                             bsccs_cv_result* result);

/* BootstrapConfig (bootstrap.hpp:17-28). */
typedef struct bsccs_bootstrap_config {
    int32_t replicates;
    int32_t warm_start;
    double level;
    uint64_t seed;
    bsccs_prior prior;
    bsccs_solver_config solver;
    int32_t engine;     /* BSCCS_ENGINE_* */
    int32_t batch;      /* batched engine: max fits per launch (<= 0: auto) */
} bsccs_bootstrap_config;

/* BootstrapResult scalars (bootstrap.hpp:30-41). */
typedef struct bsccs_bootstrap_result {
    int32_t replicates;
    int32_t used;
    int32_t non_converged;
    int32_t full_converged;
    double device_seconds;      /* instrumentation */
    int64_t total_cycles;
    int64_t coordinates_visited;
} bsccs_bootstrap_result;

void bsccs_bootstrap_config_default(bsccs_bootstrap_config* cfg);
/* run_bootstrap (bootstrap.hpp:79-158); every output has num_drugs
 * entries. */
bsccs_status bsccs_run_bootstrap(const bsccs_dataset* ds,
                                 const bsccs_bootstrap_config* cfg,
                                 double* beta_full, double* lower,
                                 double* upper, double* p_hat,
                                 bsccs_bootstrap_result* result);
/* Replicates [r_begin, r_end) of run_bootstrap (replicate r is a pure
 * function of (seed, r), bootstrap.hpp:103-106): estimates row-major
 * [(r_end - r_begin) x num_drugs], converged flags per replicate.
 * beta_full is the warm start (NULL: cold). */
bsccs_status bsccs_bootstrap_replicates(const bsccs_dataset* ds,
                                        const bsccs_bootstrap_config* cfg,
                                        const double* beta_full,
                                        int32_t r_begin, int32_t r_end,
                                        double* estimates, int32_t* converged,
                                        bsccs_bootstrap_result* result);
/* The summary step of run_bootstrap (bootstrap.hpp:120-156). */
bsccs_status bsccs_bootstrap_summarize(int32_t num_drugs, int32_t replicates,
                                       double level, const double* estimates,
                                       const int32_t* converged, double* lower,
                                       double* upper, double* p_hat,
                                       bsccs_bootstrap_result* result);

/* ---- multi-GPU patient sharding ------------------------ */
/* A group binds the shards that exchange (gradient, hessian) partials each
 * coordinate.  Local groups (all shards on one device, one process) are the
 * single-GPU test of the cross-shard protocol; multi-process groups bind the
 * per-rank exchange buffer of every peer through CUDA IPC. */
typedef struct bsccs_group bsccs_group;
/* Size in bytes of one exchange-slot buffer for `total_ctas` participants. */
int64_t bsccs_group_slot_bytes(int32_t total_ctas);
/* Local group over n shards of one device (one cooperative launch). */
bsccs_status bsccs_group_create_local(bsccs_dataset* const* shards, int32_t n,
                                      bsccs_group** out);
/* Virtual ranks: n shards of one device in one launch, each with its own
 * exchange area that every CTA adds into (system-scope adds, per-shard
 * polling) -- the multi-process protocol executed on a single GPU. */
bsccs_status bsccs_group_create_virtual(bsccs_dataset* const* shards, int32_t n,
                                        bsccs_group** out);
/* Multi-process: rank r of world w with its one local shard. */
bsccs_status bsccs_group_create_rank(bsccs_dataset* shard, int32_t rank,
                                     int32_t world, const int32_t* ctas_per_rank,
                                     bsccs_group** out);
/* 64-byte cudaIpcMemHandle of this rank's slot buffer. */
bsccs_status bsccs_group_ipc_handle(bsccs_group* g, uint8_t out[64]);
/* Open the peers' handles (world x 64 bytes, own entry ignored). */
bsccs_status bsccs_group_open_peers(bsccs_group* g, const uint8_t* handles);
bsccs_status bsccs_group_destroy(bsccs_group* g);
/* fit over a group; beta_out / result identical on every shard. */
bsccs_status bsccs_group_fit(bsccs_group* g, const bsccs_prior* prior,
                             const bsccs_solver_config* cfg,
                             const double* init_beta, double* beta_out,
                             bsccs_fit_result* result);

/* ---- synthetic data (simulate.hpp, SURVEY §8(d) generators) ----------- */
typedef struct bsccs_host_dataset bsccs_host_dataset;
/* simulate() restated (simulate.hpp:50-137); prevalence / true_beta have
 * `drugs` entries. */
bsccs_status bsccs_synth_simulate(int32_t subjects, int32_t drugs,
                                  int32_t min_eras, int32_t max_eras,
                                  int32_t min_era_length, int32_t max_era_length,
                                  const double* prevalence, const double* true_beta,
                                  double baseline_log_rate_mean,
                                  double baseline_log_rate_sd, uint64_t seed,
                                  bsccs_host_dataset** out);
/* Fast SCCS generator of SURVEY §8(d); zipf != 0 selects the skewed
 * P(drug j) ~ 1/(j+1) variant.  threads <= 0: all hardware threads. */
bsccs_status bsccs_synth_fast(int64_t attempts, int32_t drugs, double lambda_x,
                              int32_t zipf, uint64_t seed, int32_t threads,
                              bsccs_host_dataset** out);
/* N, K, J, nnz */
bsccs_status bsccs_host_dataset_sizes(const bsccs_host_dataset* h, int64_t out[4]);
/* Borrowed pointers into the handle (valid until destroy). */
bsccs_status bsccs_host_dataset_arrays(const bsccs_host_dataset* h,
                                       const int32_t** subject_offsets,
                                       const int32_t** events_per_subject,
                                       const int32_t** era_lengths,
                                       const int32_t** event_counts,
                                       const int64_t** col_ptr,
                                       const int32_t** rows,
                                       const int32_t** subjects,
                                       const int64_t** y_dot_x);
bsccs_status bsccs_host_dataset_destroy(bsccs_host_dataset* h);

#ifdef __cplusplus
}
#endif
#endif /* BSCCS_B200_H */
