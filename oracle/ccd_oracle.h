/*
 * ccd_oracle.h -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the
 * reference CCD hot path, used as the parity checker for the B200 path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  The product path never calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference itself (oracle/_ref/libbsccs_ref.so, compiled from
 * the untouched headers under /root/reference/proj/include by
 * oracle/Makefile) and against the committed golden vectors in
 * tests/golden/ that were generated from that build.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj/include/bsccs/).
 */
#ifndef CCD_ORACLE_H
#define CCD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes match include/bsccs_b200.h. */
enum { OR_OK = 0, OR_INPUT = 1, OR_NUMERIC = 2, OR_INTERNAL = 3 };

/* Flat CSC form of bsccs::Dataset (dataset.hpp:53-68). */
typedef struct or_dataset {
    int32_t N, K, J;
    int64_t nnz;
    const int32_t* subject_offsets;
    const int32_t* events_per_subject;
    const int32_t* era_lengths;
    const int32_t* event_counts;
    const int64_t* col_ptr;
    const int32_t* rows;
    const int32_t* subjects;
    const int64_t* y_dot_x;
} or_dataset;

/* EngineState<double> (engine.hpp:36-45); arrays owned by the caller. */
typedef struct or_state {
    double* beta;         /* [J] */
    double* xbeta;        /* [K] */
    double* l_exp_xbeta;  /* [K] */
    double* denominators; /* [N] */
} or_state;

typedef struct or_prior {
    int32_t kind; /* 0 none 1 normal 2 laplace (prior.hpp:10) */
    int32_t variance_is_laplace_scale;
    double variance;
} or_prior;

typedef struct or_config {
    double epsilon;
    int32_t max_cycles;
    int32_t normalized;
    double trust_init;
    int32_t dense_refresh_interval;
    int32_t random_cycle;
    uint64_t cycle_seed;
} or_config;

typedef struct or_result {
    double log_posterior;
    double final_criterion;
    int32_t cycles_run;
    int32_t converged;
    int64_t coordinates_visited;
} or_result;

const char* or_last_error(void);
int or_init_state(const or_dataset* ds, const double* beta, or_state* st);
int or_dense_recompute(const or_dataset* ds, or_state* st);
int or_grad_hess(const or_dataset* ds, const or_state* st, int32_t j, double* g, double* h);
int or_sparse_update(const or_dataset* ds, or_state* st, int32_t j, double delta);
int or_log_likelihood(const or_dataset* ds, const or_state* st, double* out);
int or_log_density(const or_prior* prior, const double* beta, int32_t n, double* out);
int or_penalized_step(const or_prior* prior, double beta_j, double g, double h, double* out);
/* one cycle; trust[J] in/out; order[J] (NULL = ascending, updated in place
 * by the shuffle when cfg->random_cycle); snapshot scratch [K]; rng_state[4]
 * is the xoshiro state of SolverState::order_rng. */
int or_run_cycle(const or_dataset* ds, or_state* st, const or_prior* prior,
                 const or_config* cfg, double* trust, int32_t* order,
                 uint64_t rng_state[4], double* snapshot, double* criterion,
                 int64_t* visited);
int or_fit(const or_dataset* ds, const or_prior* prior, const or_config* cfg,
           const double* init_beta, double* beta_out, or_result* res);

#ifdef __cplusplus
}
#endif
#endif
