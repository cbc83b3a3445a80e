/*
 * ldpc_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C, fp64 restatement of the reference decoder path
 * (arxiv/paper_1202_1060, proj/include/ldpc/{rng,channel,tanner,schedule,decoder}.hpp).
 * Every function cites the reference file:line it restates.
 *
 * This library is the CHECKER for the B200 decoder. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it. The product (paper_1202_1060_b200) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks this restatement bit-for-bit against
 * the reference headers compiled unmodified into oracle/_ref/ (see
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 */
#ifndef LDPC_ORACLE_H
#define LDPC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char *orc_last_error(void);

/* ---- rng.hpp:10-90 ---------------------------------------------------- */
typedef struct {
  uint64_t s[4];
  double spare;
  int has_spare;
} orc_rng;

uint64_t orc_splitmix64(uint64_t *state);                 /* rng.hpp:10-15 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream);    /* rng.hpp:19-25 */
void orc_rng_seed(orc_rng *r, uint64_t seed);             /* rng.hpp:31-34 */
uint64_t orc_rng_u64(orc_rng *r);                         /* rng.hpp:36-46 */
double orc_rng_unit(orc_rng *r);                          /* rng.hpp:49 */
double orc_rng_gauss(orc_rng *r);                         /* rng.hpp:52-64 */
uint64_t orc_rng_below(orc_rng *r, uint64_t n);           /* rng.hpp:67-73 */
void orc_rng_shuffle(orc_rng *r, int32_t *a, int64_t n);  /* rng.hpp:75-82 */

/* ---- channel.hpp:21-46 ------------------------------------------------ */
double orc_sigma2_from_ebn0(double ebn0_db, double rate); /* NaN on bad rate */
int orc_transmit_all_zero(double sigma2, uint64_t seed, int n, uint64_t frame_id, double *llr);
/* frames [frame0, frame0+frames) rounded to fp32, row-major [frames][n] */
int orc_transmit_batch_f32(double sigma2, uint64_t seed, int n, uint64_t frame0, int64_t frames, float *llr,
                           int threads);

/* ---- tanner.hpp:21-114, 356-393 --------------------------------------- */
typedef struct orc_graph orc_graph;
orc_graph *orc_graph_create(int n_vars, int n_checks, const int32_t *row_off, const int32_t *cols);
void orc_graph_destroy(orc_graph *g);
int orc_graph_n_edges(const orc_graph *g);
/* var_off[n+1], var_cns[E], var_edges[E] (CN ids ascending, CN-major edge ids) */
void orc_graph_var_view(const orc_graph *g, int32_t *var_off, int32_t *var_cns, int32_t *var_edges);
/* returns n_checks (rows of dc entries in cols_out[m*dc+k]) or -1 */
int orc_random_regular(int n_vars, int dv, int dc, uint64_t seed, int32_t *cols_out);

/* ---- schedule.hpp:54-127, 175-210 ------------------------------------- */
/* generate_groups with Rng(rng_seed); grp_off[G+1]; returns total slots or -1.
 * grp_cns must hold max_slots entries. */
int orc_generate_groups(int n_checks, int n_groups, double overlap, uint64_t rng_seed, int32_t *grp_off,
                        int32_t *grp_cns, int max_slots);
int orc_iteration_budget(int n_checks, int i_max, int kind, int n_groups, int group_size, double overlap);

/* ---- decoder.hpp:39-181 ----------------------------------------------- */
enum { ORC_FLOODING = 0, ORC_DISJOINT = 1, ORC_NONDISJOINT = 2 };

typedef struct {
  int kind;        /* schedule.hpp:16 */
  int n_groups;    /* entries in grp_off - 1 */
  double overlap;  /* overlap_ratio, used only when regrouping */
  uint64_t seed;   /* regroup seed */
  int regroup;     /* regroup_each_iteration */
  const int32_t *grp_off;
  const int32_t *grp_cns;
  /* run_sweep's grouping (sim.hpp:113-117): groups drawn per frame from
   * mix_seed(seed, frame_id); grp_off/grp_cns unused. Frame ids: batch
   * index (decode_batch) or the true frame id (simulate); orc_decode uses 0. */
  int per_frame;
} orc_schedule;

/* decoder.hpp:59-87 on one CN of the given degree */
void orc_check_update(int degree, const double *v2c, double *c2v);

/* decode() (decoder.hpp:143-181). early_stop=0 runs all max_iters
 * (init_state + run_subiteration composition, acceptance.cpp:142-146).
 * Outputs may be NULL. syndrome_trace has max_iters slots (unused = -1).
 * posterior = total_llr at return. Returns 0 or -1. */
int orc_decode(const orc_graph *g, const orc_schedule *s, const double *llr, int max_iters, int early_stop,
               uint8_t *bits, int32_t *iterations, uint8_t *converged, double *posterior, int32_t *syndrome_trace,
               int64_t *cn_updates);

/* Batch of fp32 LLRs (promoted to double), frames in parallel on `threads`
 * host threads pulling frame ids from an atomic counter (sim.hpp:136-150). */
int orc_decode_batch_f32(const orc_graph *g, const orc_schedule *s, const float *llr, int64_t frames,
                         int max_iters, int early_stop, int threads, uint8_t *bits, int32_t *iterations,
                         uint8_t *converged, float *posterior, int32_t *syndrome_trace);

/* init_state + n_subiters x run_subiteration cycling through the groups;
 * dumps c2v[E] and v2c[E] (decoder.hpp:39-52, 112-127). */
int orc_run_subiterations(const orc_graph *g, const orc_schedule *s, const double *llr, int n_subiters,
                          double *c2v_out, double *v2c_out);

/* Monte-Carlo aggregation of one frame range (sim.hpp:111-124, 162-181):
 * counters = {frames, bit_errors, frame_errors, converged_frames, iter_sum,
 * iter_sum_converged}. LLRs come from transmit_all_zero, rounded to fp32 when
 * round_f32 != 0 (the B200 path's input convention). */
int orc_simulate(const orc_graph *g, const orc_schedule *s, double sigma2, uint64_t channel_seed,
                 uint64_t frame_begin, int64_t frame_count, int max_iters, int early_stop, int round_f32,
                 int threads, int64_t *counters);

#ifdef __cplusplus
}
#endif
#endif
