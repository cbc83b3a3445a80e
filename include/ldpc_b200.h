/*
 * ldpc_b200.h -- C ABI of the B200 batched group-shuffled LDPC decoder.
 *
 * Drop-in boundary for the hot path of arxiv/paper_1202_1060: the reference
 * exposes a header-only C++ API (proj/include/ldpc/<module>.hpp) and no FFI; every
 * entry point below names the reference interface it replaces (file:line,
 * relative to proj/include/ldpc/). The C++ mirror of the reference types is
 * include/ldpc_b200.hpp; the ctypes binding is paper_1202_1060_b200/_lib.py.
 *
 * Conventions
 *  - Every call returns an int status (LDPCB_OK = 0); ldpcb_last_error()
 *    gives a thread-local message. No exception crosses the ABI. The
 *    reference's std::invalid_argument maps to LDPCB_EINVAL, its
 *    std::runtime_error to LDPCB_ERUNTIME, its AlistError to LDPCB_EALIST.
 *  - Handles are immutable after creation and safe to share across host
 *    threads (tanner.hpp / SPEC.md "Concurrency Model"). Device copies are
 *    made lazily, once per device, on first use.
 *  - *_device calls take device pointers and a cudaStream_t (as void*) and
 *    are stream-ordered (asynchronous). *_host calls take host pointers and
 *    return when the results are in host memory.
 *  - LLRs are fp32, frame-major [frames][n]; the all-zero codeword / BPSK
 *    0 -> +1 convention of channel.hpp holds; bits are 0/1 bytes
 *    ([frames][n]) or packed little-endian ([frames][ceil(n/8)]).
 *  - Monte-Carlo counters are int64[6] = {frames, bit_errors, frame_errors,
 *    converged_frames, iter_sum, iter_sum_converged} (sim.hpp:162-181) and
 *    are ACCUMULATED into (callers zero them).
 */
#ifndef LDPC_B200_H
#define LDPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LDPCB_OK 0
#define LDPCB_EINVAL (-1)
#define LDPCB_ERUNTIME (-2)
#define LDPCB_EALIST (-3)
#define LDPCB_ECUDA (-4)
#define LDPCB_EUNSUPPORTED (-5)

#define LDPCB_FLOODING 0   /* ScheduleKind::flooding    schedule.hpp:16 */
#define LDPCB_DISJOINT 1   /* ScheduleKind::disjoint                   */
#define LDPCB_NONDISJOINT 2 /* ScheduleKind::nondisjoint               */

typedef struct ldpcb_code_s *ldpcb_code;
typedef struct ldpcb_schedule_s *ldpcb_schedule;

const char *ldpcb_last_error(void);
int ldpcb_abi_version(void);

/* ---- code graphs: TannerGraph (tanner.hpp:21-37) ------------------------ */

/* build_from_check_lists (tanner.hpp:79-114): CSR rows, CN-major edge ids */
int ldpcb_code_from_check_lists(int n_vars, int n_checks, const int32_t *row_off, const int32_t *cols,
                                ldpcb_code *out);
/* random_regular_graph (tanner.hpp:356-393), bit-identical to the reference */
int ldpcb_code_random_regular(int n_vars, int dv, int dc, uint64_t seed, ldpcb_code *out);
/* random_regular_graph followed by deterministic 4-cycle breaking
 * (BASELINE config 1: "random socket-permutation ... with 4-cycles removed") */
int ldpcb_code_random_regular_girth6(int n_vars, int dv, int dc, uint64_t seed, ldpcb_code *out);
/* quasi-cyclic base-matrix expansion (BASELINE config 3; no reference analogue) */
int ldpcb_code_qc(int base_rows, int base_cols, int z, double p_empty, int min_col_degree, uint64_t seed,
                  ldpcb_code *out);
/* irregular VN / regular CN socket matching (BASELINE config 4) */
int ldpcb_code_irregular(int n_vars, int n_classes, const int32_t *vn_degrees, const int32_t *vn_counts, int dc,
                         uint64_t seed, ldpcb_code *out);
/* parse_alist (tanner.hpp:172-282); on LDPCB_EALIST, err_kind and err_line receive
 * the AlistErrorKind (tanner.hpp:48-59) and 1-based line */
int ldpcb_code_parse_alist(const char *text, ldpcb_code *out, int *err_kind, int *err_line);
/* serialize_alist (tanner.hpp:286-317); *len = bytes (without NUL); buf
 * is filled when cap > *len */
int ldpcb_code_serialize_alist(ldpcb_code code, char *buf, int64_t cap, int64_t *len);
int ldpcb_code_dims(ldpcb_code code, int32_t *n_vars, int32_t *n_checks, int32_t *n_edges, int32_t *max_check_degree,
                    int32_t *max_var_degree);
/* any output may be NULL: row_off[m+1], cols[E], var_off[n+1], var_cns[E],
 * var_edges[E] (var_adj / var_edge_ids, tanner.hpp:25-26) */
int ldpcb_code_export(ldpcb_code code, int32_t *row_off, int32_t *cols, int32_t *var_off, int32_t *var_cns,
                      int32_t *var_edges);
int ldpcb_code_count_4cycles(ldpcb_code code, int64_t *count);
void ldpcb_code_destroy(ldpcb_code code);

/* ---- schedules: GroupSchedule (schedule.hpp:32-40) ---------------------- */

/* explicit ordered groups (the route decode() accepts, decoder.hpp:150-157) */
int ldpcb_schedule_from_groups(ldpcb_code code, int kind, int n_groups, const int32_t *grp_off,
                               const int32_t *grp_cns, ldpcb_schedule *out);
int ldpcb_schedule_flooding(ldpcb_code code, ldpcb_schedule *out);                  /* :129-139 */
int ldpcb_schedule_disjoint(ldpcb_code code, int n_groups, uint64_t seed, ldpcb_schedule *out); /* :136-149 */
int ldpcb_schedule_nondisjoint(ldpcb_code code, int n_groups, double overlap, uint64_t seed,
                               ldpcb_schedule *out);                                /* :151-171 */
/* The reference harness's grouping (run_sweep, sim.hpp:113-117): every frame
 * draws its own random groups, make_*_schedule with seed
 * mix_seed(schedule_seed, frame_id), and with regroup_each_iteration redraws
 * them every iteration (decoder.hpp:153-156). Frame ids are the batch index
 * for decode calls and the true frame id for simulate calls. */
int ldpcb_schedule_per_frame(ldpcb_code code, int kind, int n_groups, double overlap, uint64_t schedule_seed,
                             int regroup_each_iteration, ldpcb_schedule *out);
/* The groups a per-frame schedule uses for frames [frame0, frame0+frames) at
 * one iteration (schedule_groups_for, schedule.hpp:121-127), generated on
 * the device: d_cns[f * slots + j], slots = the schedule's total slot count,
 * group g at [group_offsets[g], group_offsets[g+1]) of ldpcb_schedule_export. */
int ldpcb_schedule_per_frame_groups_device(ldpcb_code code, ldpcb_schedule s, int64_t frame0, int64_t frames,
                                           int iteration, uint16_t *d_cns, void *stream);
/* fixed wrapping windows: group g = CNs (g*stride + j) mod M, j < window */
int ldpcb_schedule_windows(ldpcb_code code, int kind, int n_groups, int window, int stride, ldpcb_schedule *out);
int ldpcb_schedule_dims(ldpcb_schedule s, int32_t *kind, int32_t *n_groups, int32_t *n_slots, int32_t *group_size,
                        double *overlap, int64_t *edge_updates_per_iter, int64_t *touched_per_iter);
int ldpcb_schedule_export(ldpcb_schedule s, int32_t *grp_off, int32_t *grp_cns);
int ldpcb_schedule_iteration_budget(ldpcb_schedule s, int i_max, int32_t *budget); /* :206-210 */
/* Layout of the posterior-free resident kernel for this schedule:
 * frames per thread (0: the kernel does not apply to this code / schedule),
 * cells per CTA, first L cell, cells between the two edge-cell copies (flooding;
 * 0 otherwise), CN items over all groups, shared-memory wavefronts per access
 * after bank colouring. ldpcb_schedule_direct_export copies the tables:
 * cn_off[G+1], cn_rec[12 * items], vn_rec[2 n], vn_hold[n], vn_pos[n],
 * edge_rec[2 E] (byte offsets; formats in csrc/host.hpp DirectTables). */
int ldpcb_schedule_direct_layout(ldpcb_schedule s, int32_t *frames_per_thread, int32_t *cells, int32_t *l_base,
                                 int32_t *buffer_cells, int32_t *n_items, double *wavefronts_per_access);
int ldpcb_schedule_direct_export(ldpcb_schedule s, int32_t *cn_off, int32_t *cn_rec, int32_t *vn_rec,
                                 int32_t *vn_hold, int32_t *vn_pos, int32_t *edge_rec);
int ldpcb_schedule_cocsg(ldpcb_schedule s, int32_t *counts /* n_groups-1 */);       /* :175-201 */
void ldpcb_schedule_destroy(ldpcb_schedule s);

/* ---- channel (channel.hpp:21-46) ---------------------------------------- */

int ldpcb_sigma2_from_ebn0(double ebn0_db, double rate, double *sigma2);
/* transmit_all_zero for frames [frame0, frame0+frames), generated on the
 * device with the reference's stream (rng.hpp) in fp64, stored as fp32 */
int ldpcb_channel_llr_device(int n, double sigma2, uint64_t seed, int64_t frame0, int64_t frames, float *d_llr,
                             void *stream);
/* xoshiro256 state of frame `frame`'s noise stream, Rng(mix_seed(seed, frame))
 * (rng.hpp:19-46, channel.hpp:40), after `draws` 64-bit draws, by jump-ahead
 * (x^draws mod the generator's characteristic polynomial). The device
 * channel starts segments of long frames this way; exposed for tests. */
int ldpcb_channel_stream_state(uint64_t seed, uint64_t frame, uint64_t draws, uint64_t state[4]);

/* ---- decoding (decode, decoder.hpp:143-181) ------------------------------ */

/* Batched decode(). early_stop=1: syndrome stop (decoder.hpp:173-177);
 * early_stop=0: exactly max_iters iterations, converged = final syndrome 0.
 * Outputs may be NULL: bits, iterations[frames], converged[frames],
 * posterior[frames][n] (= total_llr), syndrome_trace[frames][max_iters]
 * (-1 after stop), counters[6]. */
int ldpcb_decode_device(ldpcb_code code, ldpcb_schedule s, int64_t frames, const float *d_llr, int max_iters,
                        int early_stop, uint8_t *d_bits, int bits_packed, int32_t *d_iterations,
                        uint8_t *d_converged, float *d_posterior, int32_t *d_syndrome_trace, int64_t *d_counters,
                        void *stream);
/* Same from host memory (pinned for best overlap); H2D / decode / D2H are
 * chunked and overlapped on two streams; blocks until done. Runs on the
 * calling thread's current CUDA device. */
int ldpcb_decode_host(ldpcb_code code, ldpcb_schedule s, int64_t frames, const float *llr, int max_iters,
                      int early_stop, uint8_t *bits, int bits_packed, int32_t *iterations, uint8_t *converged,
                      float *posterior, int32_t *syndrome_trace, int64_t *counters);
/* Monte-Carlo frames [frame_begin, frame_begin+frames): device channel +
 * decode + counters (run_frame + aggregation, sim.hpp:111-124, 162-181) */
int ldpcb_simulate_device(ldpcb_code code, ldpcb_schedule s, double sigma2, uint64_t channel_seed,
                          int64_t frame_begin, int64_t frames, int max_iters, int early_stop, int64_t *d_counters,
                          void *stream);
/* ldpcb_simulate_device with per-frame outcomes (any output may be NULL):
 * bit_errors[f] = hard-decision weight, iterations[f], converged[f] */
int ldpcb_simulate_frames_device(ldpcb_code code, ldpcb_schedule s, double sigma2, uint64_t channel_seed,
                                 int64_t frame_begin, int64_t frames, int max_iters, int early_stop,
                                 int32_t *d_bit_errors, int32_t *d_iterations, uint8_t *d_converged,
                                 int64_t *d_counters, void *stream);
/* run_sweep (sim.hpp:96-186) on one GPU: per Eb/N0 point, frames 0,1,...
 * in waves (wave_frames = 0: automatic) until the smallest prefix holding
 * min_frame_errors frame errors, or max_frames. out: 11 doubles per point =
 * frames, bit_errors, frame_errors, converged_frames, ber, fer,
 * mean_iters_converged, mean_iters_all, iter_limit, wall_seconds, ebn0_db
 * (SimResult, sim.hpp:44-56). Use a per-frame schedule for the harness's
 * own grouping. Rate = (n - m) / n as in run_sweep. */
int ldpcb_run_sweep_host(ldpcb_code code, ldpcb_schedule s, const double *ebn0_db, int n_points, int iter_limit,
                         int64_t max_frames, int min_frame_errors, uint64_t channel_seed, int64_t wave_frames,
                         double *out);
/* ---- several GPUs of one process --------------------------------------
 * One host thread per entry of devices[] (the reference's worker pool,
 * sim.hpp:136-150, with a GPU per worker); frame ids are split into
 * contiguous ranges in list order, frame i of n_devices getting
 * [begin + F*i/n, begin + F*(i+1)/n); frames are keyed by id, so results do
 * not depend on the device count. A device may be listed more than once.
 * Counters are summed on the host (the single-process counterpart of the
 * NCCL allreduce used by one-process-per-GPU jobs). Blocks until done. */
/* simulate over several GPUs: counters (host int64[6]) accumulated */
int ldpcb_simulate_multi(ldpcb_code code, ldpcb_schedule s, const int *devices, int n_devices, double sigma2,
                         uint64_t channel_seed, int64_t frame_begin, int64_t frames, int max_iters, int early_stop,
                         int64_t *counters);
/* run_sweep (sim.hpp:96-186) over several GPUs: every wave is split over the
 * devices and the min-frame-errors prefix stop is taken on the gathered
 * per-frame outcomes in frame order; out as ldpcb_run_sweep_host */
int ldpcb_run_sweep_multi(ldpcb_code code, ldpcb_schedule s, const int *devices, int n_devices,
                          const double *ebn0_db, int n_points, int iter_limit, int64_t max_frames,
                          int min_frame_errors, uint64_t channel_seed, int64_t wave_frames, double *out);
/* ldpcb_simulate_device with host counters; blocks until done */
int ldpcb_simulate_host(ldpcb_code code, ldpcb_schedule s, double sigma2, uint64_t channel_seed, int64_t frame_begin,
                        int64_t frames, int max_iters, int early_stop, int64_t *counters);
/* check_update (decoder.hpp:59-87) on rows x degree explicit inputs */
int ldpcb_check_update_device(int degree, int64_t rows, const float *d_v2c, float *d_c2v, void *stream);
/* init_state + n_subiters x run_subiteration (decoder.hpp:39-52, 112-127),
 * dumping c2v[frames][E] and v2c[frames][E] (CN-major edge ids) */
int ldpcb_run_subiterations_device(ldpcb_code code, ldpcb_schedule s, int64_t frames, const float *d_llr,
                                   int n_subiters, float *d_c2v, float *d_v2c, void *stream);

/* ---- introspection / tuning --------------------------------------------- */

/* kernel: 2 = HBM-streamed (fpc = frames per chunk); SMEM-resident plans
 * report 10 + frames_per_thread (11, 12) with fpc = frames per CTA; the
 * posterior-free resident kernel reports 20 + frames per thread (22, 24) */
int ldpcb_decode_plan(ldpcb_code code, ldpcb_schedule s, int64_t frames, int32_t *kernel, int32_t *fpc,
                      int32_t *threads, int32_t *smem_bytes, int32_t *degree_bucket);
/* 0 = automatic */
int ldpcb_set_tuning(int frames_per_cta, int threads);
/* frames per thread of the resident kernel: 0 = automatic, 1 or 2 */
int ldpcb_set_frames_per_thread(int fv);
/* 0 = automatic (resident when a frame fits shared memory; the posterior-free
 * resident kernel where the code and schedule qualify), 1 = resident
 * posterior-based kernel only, 2 = HBM-streamed, 3 = posterior-free resident
 * kernel (decodes fail when the code or the schedule does not qualify) */
int ldpcb_set_kernel(int kernel);
/* 1 (default): in iterations that do not test the syndrome, skip the exact
 * re-summation of the posteriors (in-place updates carry them); the totals
 * are exact whenever hard decisions are taken. 0: every iteration. */
int ldpcb_set_lazy_totals(int on);
/* number of CUDA kernels this library has launched (process lifetime) */
int64_t ldpcb_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif
