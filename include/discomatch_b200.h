/*
 * discomatch_b200.h — C-ABI of the B200-native DiscoMatch dual-solver hot path.
 *
 * The reference (`prodmatch`, /root/reference/pkg/src/prodmatch) is Python:
 * its only native boundary is the set of numba kernels in kernels.py, each
 * called with flat numpy arrays (FlatBdds, kernels.py:35-92) that it mutates
 * in place.  This header is that boundary re-cut for a device: the flat
 * node table is uploaded once into a `dm_flat` handle (plus the level
 * schedules of the exact averaging passes), and every kernel entry point
 * below replaces one reference kernel, taking device pointers for the
 * vectors it reads/writes and a cudaStream_t (as void*).  Nothing here
 * mentions torch; all sizes are int64, all vectors float64 (the reference
 * computes in binary64 throughout).
 *
 * Return codes: DM_OK (0) or a negative DM_ERR_*; dm_last_error() gives a
 * thread-local message.  Kernels are asynchronous on the given stream.
 *
 * Host-side lowering (rows -> reduced equality diagrams -> chunk splitting
 * -> flat table) is exposed too, because the reference's instance builder
 * (ilp.py:89-108 + bdd.py:478-501 + splitting.py:116-155) is upstream of
 * every kernel and its output layout must be reproduced bit-exactly.
 */
#ifndef DISCOMATCH_B200_H
#define DISCOMATCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DM_OK 0
#define DM_ERR_INVALID (-1)     /* bad argument / malformed instance (ValueError) */
#define DM_ERR_INFEASIBLE (-2)  /* a row has no 0-1 solution (EmptyFeasibleSet, bdd.py:493) */
#define DM_ERR_CUDA (-3)        /* CUDA runtime failure */
#define DM_ERR_UNSUPPORTED (-4) /* instance outside the kernels' envelope */
#define DM_ERR_NOMEM (-5)

/* Thread-local description of the last error. */
const char *dm_last_error(void);
/* Library / kernel build identification ("sm_100a ..."). */
const char *dm_version(void);

/* ------------------------------------------------------------------------
 * Host lowering: integer equality rows -> flat diagram table.
 * Replaces IlpInstance.from_rows (ilp.py:89-108) -> split_instance
 * (splitting.py:116-155) -> FlatBdds (kernels.py:43-92).
 * ---------------------------------------------------------------------- */
typedef struct dm_instance dm_instance;

typedef struct {
    int64_t num_variables; /* after splitting (originals + auxiliaries) */
    int64_t num_bdds;
    int64_t num_layers; /* dual coordinates */
    int64_t num_nodes;
    int64_t max_width;  /* widest layer */
    int64_t max_degree; /* most diagrams sharing one variable */
    int64_t max_layers; /* longest diagram */
} dm_instance_info;

/* rows in CSR form: row r has variables row_var[row_ptr[r]:row_ptr[r+1]]
 * with integer coefficients row_coef[...] and right-hand side row_rhs[r].
 * chunk_size <= 0 disables splitting, otherwise every diagram longer than
 * chunk_size original layers is cut every chunk_size layers (>= 2). */
int dm_instance_from_rows(int64_t num_variables, const double *costs, int64_t num_rows,
                          const int64_t *row_ptr, const int64_t *row_var,
                          const int64_t *row_coef, const int64_t *row_rhs, int64_t chunk_size,
                          dm_instance **out);
/* Same pipeline from already-compiled diagrams (Bdd objects flattened per
 * diagram): layer_node_lo/zeros/ones hold LOCAL next-layer indices like
 * Bdd.zeros/Bdd.ones (bdd.py:55-87).  variable_order may be NULL
 * (identity).  Used for split_instance on arbitrary diagram lists. */
int dm_instance_from_bdds(int64_t num_variables, const double *costs, const int64_t *variable_order,
                          int64_t num_bdds, const int64_t *bdd_layer_lo, const int64_t *layer_var,
                          const int64_t *layer_node_lo, const int32_t *zeros, const int32_t *ones,
                          int64_t chunk_size, dm_instance **out);
/* Variable numbering of a product space (product_space.py): a greedy row
 * colouring — variables in index order take the smallest colour no variable
 * of any of their rows already has (colour_out[V]).  Numbering variables by
 * colour bounds the exact passes' DAG depth by the number of colours (every
 * diagram chain advances at least one colour per layer): C4 1,665 -> 370
 * levels.  No reference counterpart (the reference has no product space). */
int dm_row_colouring(int64_t num_variables, int64_t num_rows, const int64_t *row_ptr, const int64_t *row_var,
                     int64_t *colour_out);
int dm_instance_get_info(const dm_instance *inst, dm_instance_info *info);
/* Copy the FlatBdds arrays out (any pointer may be NULL to skip it):
 * costs[V], variable_order[V], bdd_layer_lo[nb+1], layer_node_lo[L+1],
 * layer_var[L], layer_bdd[L], zero_t[N], one_t[N], proc_ptr[V+1],
 * proc_layers[L], constraint_counts[V]. */
int dm_instance_export(const dm_instance *inst, double *costs, int64_t *variable_order,
                       int64_t *bdd_layer_lo, int64_t *layer_node_lo, int64_t *layer_var,
                       int64_t *layer_bdd, int64_t *zero_t, int64_t *one_t, int64_t *proc_ptr,
                       int64_t *proc_layers, int64_t *constraint_counts);
void dm_instance_free(dm_instance *inst);
/* Conditioning for the primal side (reference bdd.py:243-264 Bdd.condition,
 * bdd.py:278-334 reduce_bdd, primal.py:114-175 fix_and_reduce): every diagram
 * of the flat table (FlatBdds arrays, global node ids) that touches a fixed
 * variable (fixed[v] = 0/1, -1 free) is clamped and re-reduced; diagrams left
 * as a single chain accepting every fix-consistent assignment are dropped
 * (count in *dropped_out); the rest become a new instance with the same
 * costs and variable order, unsplit.  DM_ERR_INFEASIBLE when a diagram
 * empties (the reference raises InfeasibleAfterFixing). */
int dm_condition_flat(int64_t num_variables, const double *costs, const int64_t *variable_order,
                      int64_t num_bdds, const int64_t *bdd_layer_lo, const int64_t *layer_var,
                      const int64_t *layer_node_lo, const int64_t *zero_t, const int64_t *one_t,
                      const int8_t *fixed, int64_t *dropped_out, dm_instance **out);

/* ------------------------------------------------------------------------
 * Device-resident flat table (FlatBdds on the GPU) + exact-pass schedules.
 * ---------------------------------------------------------------------- */
typedef struct dm_flat dm_flat;

typedef struct {
    int64_t num_bdds, num_layers, num_nodes, num_positions;
    /* host arrays, FlatBdds semantics (kernels.py:35-92) */
    const int64_t *bdd_layer_lo;  /* [nb+1] */
    const int64_t *layer_node_lo; /* [L+1] */
    const int64_t *layer_var;     /* [L]   */
    const int64_t *zero_t;        /* [N]   global node id, -1 FALSE, -2 TRUE */
    const int64_t *one_t;         /* [N]   */
    const int64_t *proc_ptr;      /* [P+1] copies per visitation position */
    const int64_t *proc_layers;   /* [L]   layers of each position, ascending */
} dm_flat_desc;

typedef struct {
    int64_t fw_depth, bw_depth; /* DAG levels of the exact forward/backward passes */
    int64_t fw_tasks, bw_tasks; /* warp tasks */
    int64_t mma_grid, mma_block;
    int64_t max_width, max_degree;
    int64_t device_bytes;
    int64_t lanes_per_task;     /* trace / task_levels records per task: 32 (one per BDD copy lane),
                                   8 (node-parallel kernels: one per copy slot) */
    int64_t dfr_node_parallel;  /* 1: dm_dfr_np_* available (layers <= 8 nodes, single-source publish) */
} dm_flat_info;

int dm_flat_create(const dm_flat_desc *desc, int device, void *stream, dm_flat **out);
/* flags: DM_FLAT_NO_EXACT_PLANS skips the exact passes' level schedules and
 * copy records (the deferred schedule, sweeps and vector kernels do not use
 * them; dm_k_mma_* then return DM_ERR_INVALID). */
#define DM_FLAT_NO_EXACT_PLANS 1
int dm_flat_create_ex(const dm_flat_desc *desc, int device, void *stream, int flags, dm_flat **out);
int dm_flat_get_info(const dm_flat *flat, dm_flat_info *info);
/* Synchronises the stream and reports whether an exact pass since the last
 * call was aborted by its watchdog (DM_ERR_CUDA) — resets the word. */
int dm_flat_status(dm_flat *flat, void *stream);
/* Launch shape of the exact passes: block size (multiple of 32, <= 256),
 * resident blocks per SM (<= 0: as many as fit), the back-off between
 * unsuccessful polls, the poll mode (probe != 0: poll one probe word
 * before reading the inputs; 0: poll all inputs) and the progress lookahead
 * (a warp polls its inputs only once a task within `lookahead` levels of its
 * own has finished; 0 disables the gating) in bits 0-15 of `lookahead`;
 * bit 16 enables L2 warming of the polled lines, bit 17 forces the generic
 * tree publish in the forward pass instead of the per-layer descriptors,
 * bit 18 forces the per-copy kernels instead of the node-parallel ones
 * (used by default when layers have <= 8 nodes and variables <= 8 copies).
 * Defaults come from DM_MMA_THREADS / DM_MMA_BLOCKS_PER_SM / DM_MMA_SLEEP_NS /
 * DM_MMA_PROBE / DM_MMA_LOOKAHEAD / DM_MMA_WARM / DM_MMA_DESC / DM_MMA_NP. */
int dm_flat_set_mma_config(dm_flat *flat, int threads, int blocks_per_sm, int sleep_ns, int probe,
                           int lookahead);
/* Profiling hooks: a device buffer of tasks*lanes_per_task*6 u64 receives, per lane (copy slot),
 * %globaltimer stamps (task start, own inputs seen, group go, dual updated, outputs published,
 * issue of the successful input poll) of the
 * following exact passes (NULL disables); dm_flat_task_levels copies the
 * DAG level of every task (and optionally the lanes_per_task lane layers per task) of
 * the forward/backward schedule. */
int dm_flat_set_trace(dm_flat *flat, unsigned long long *trace);
/* Stream-ordered copy of the exact passes' watchdog word into a device
 * double (0 = fine): lets the host check it together with other scalars in
 * one read-back; dm_flat_status then reports and clears a fired watchdog. */
int dm_flat_status_to(const dm_flat *flat, double *slot, void *stream);
int dm_flat_task_levels(const dm_flat *flat, int forward, int32_t *levels, int32_t *lane_layers);
void dm_flat_destroy(dm_flat *flat);

/* --- sweep kernels: one per reference kernel ---------------------------- */
/* kernels.py:95-120 */
int dm_k_backward(const dm_flat *f, const double *lam, double *B, double *bounds, void *stream);
/* dual.py:99-106 on lam + gamma*d (qn.py:147,153), without materialising it */
int dm_k_backward_trial(const dm_flat *f, const double *lam, const double *d, double gamma,
                        double *B, double *bounds, void *stream);
/* qn.py:132-159 find_step_size, the whole trial sequence on the device: the
 * trial sweeps on lam + gamma*d, their bound sums (+ free_contribution) and
 * the reference's shrink/grow/stop decisions, enqueued without host round
 * trips.  `state` (8 device doubles) ends as {gamma, e_init, e_best,
 * gamma_best, e_cur, stop, trials, -}; the caller compares e_best with the
 * current objective.  `bounds` is per-diagram scratch. */
int dm_step_search(const dm_flat *f, const double *lam, const double *d, double gamma_prev,
                   double free_contribution, double shrink, double grow, double min_ascent,
                   int max_trials, double *bounds, double *state, void *stream);
/* qn.py:203-206 + dual.py:164-165 without a host round trip: after
 * dm_step_search, if state[2] (e_best) > base (the current objective)
 * lam += state[3] * d (dm_axpy_host's roundings) and B / bounds are rebuilt
 * (dm_k_backward); otherwise nothing changes.  out[3] = {gamma_best, used
 * (1.0 / 0.0), trials} for the caller's next read-back. */
int dm_qn_move(const dm_flat *f, double *lam, const double *d, double base, const double *state, double *out,
               double *B, double *bounds, void *stream);
/* kernels.py:123-159 */
int dm_k_forward(const dm_flat *f, const double *lam, double *F, double *bounds, void *stream);
/* kernels.py:162-270: exact (bitwise) Gauss-Seidel forward averaging pass */
int dm_k_mma_forward(const dm_flat *f, double *lam, double *F, const double *B, double *bounds,
                     void *stream);
/* kernels.py:273-362: exact backward averaging pass */
int dm_k_mma_backward(const dm_flat *f, double *lam, const double *F, double *B, double *bounds,
                      void *stream);
/* kernels.py:365-398 */
int dm_k_min_marginals(const dm_flat *f, const double *lam, const double *F, const double *B,
                       double *m0, double *m1, void *stream);
/* kernels.py:401-431 */
int dm_k_argmin(const dm_flat *f, const double *lam, const double *B, double *bits, void *stream);
/* The argmin walk (dm_k_argmin) from the per-node decisions the last exact
 * backward pass recorded when it ran the node-parallel kernels — valid only
 * while lam and B are exactly what that pass left (the caller tracks this;
 * DualState does via its distance-table generation).  B must be the table that
 * pass wrote; DM_ERR_INVALID otherwise (also after dm_init_duals,
 * dm_k_mma_forward or a sweep rewrote that table; duals moved by the
 * flat-less vector kernels, e.g. dm_axpy_host, are the caller's to track).  Bit-identical to dm_k_argmin there. */
int dm_k_argmin_from_pass(const dm_flat *flat, const double *B, double *bits, void *stream);

/* --- deferred (throughput) averaging schedule ------------------------------
 * FastDOG's parallel deferred min-marginal averaging (the GPU solver the
 * paper builds on: PAPER.md:282,4924), which the reference replaced by the
 * sequential Gauss-Seidel passes above (kernels.py:162-362)
 * — selected by SolveConfig(mma_schedule="deferred").  Every diagram is
 * processed independently within a pass; per copy with finite min-marginals
 *   lam' = (lam - omega*M) + avg_in,  mbar = omega*M     (M = m1 - m0)
 * and lam' = lam + avg_in, mbar = +inf otherwise; dm_dfr_average turns one
 * pass's escrow mbar into the next pass's avg_in (per-variable mean of the
 * finite mbar over the copies, in copy order; 0 for non-finite copies).
 * mbar == NULL: no min-marginal step (a sweep that only adds avg_in: the
 * flush that makes the duals feasible again, or a plain refresh);
 * avg_in == NULL: nothing to add.
 * Distance tables are INTERLEAVED (dm_dfr_table_size elements; node slot i of
 * layer position k of a diagram's lane in the sweep layout), which only these
 * entry points and dm_dfr_to_nodes read.  bounds[j] = optimum of diagram j
 * under the resulting duals. */
int dm_dfr_table_size(const dm_flat *f, int64_t *elements);
/* forward pass: needs B_il exact for lam when mbar != NULL; writes F_il */
int dm_dfr_forward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *B_il,
                   double *F_il, double *mbar, double *bounds, void *stream);
/* backward pass: needs F_il exact for lam when mbar != NULL; writes B_il and,
 * with record_decisions (layers <= 8 nodes), the argmin decisions that
 * dm_k_argmin_from_pass(f, B_il, ...) walks */
int dm_dfr_backward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *F_il,
                    double *B_il, double *mbar, double *bounds, int record_decisions, void *stream);
/* The same two passes node-parallel (8 lanes per diagram) on tables in the
 * reference NODE order (FlatBdds F / B, as dm_k_forward / dm_k_backward
 * write them); bit-identical to the interleaved ones.  DM_ERR_UNSUPPORTED
 * unless dm_flat_info.dfr_node_parallel. */
int dm_dfr_np_forward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *B,
                      double *F, double *mbar, double *bounds, void *stream);
int dm_dfr_np_backward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *F, double *B,
                       double *mbar, double *bounds, int record_decisions, void *stream);
/* segmented reduction over the variable CSR (proc_ptr / proc_layers) */
int dm_dfr_average(const dm_flat *f, const double *mbar, double *avg_in, void *stream);
/* the flush: lam[l] += the average dm_dfr_average would write (one rounding,
 * identical to a later pass adding avg_in); follow it by a plain
 * dm_dfr_backward (mbar = avg_in = NULL) to rebuild B_il for the new duals */
int dm_dfr_flush(const dm_flat *f, const double *mbar, double *lam, void *stream);
/* Partitioned instances (one instance's diagrams split over ranks; the
 * north star's C4 split, paper_2310_08230_b200/partition.py).
 * dm_dfr_average_csr: dm_dfr_average / dm_dfr_flush (apply != 0) over a
 * caller-supplied visitation CSR (device int32: the rank's variables whose
 * copies are all local).  A variable with copies on several ranks is
 * averaged through an exchange buffer with one slot per copy in global copy
 * order: dm_dfr_boundary_gather writes buf[slot[i]] = mbar[layer[i]] for the
 * rank's boundary copies (buf zeroed before, every slot has one writer, so
 * an allreduce-sum over ranks completes it exactly), and
 * dm_dfr_boundary_average writes (apply: adds) the mean of the finite
 * entries of buf[slot_lo[i], slot_hi[i]) to out[layer[i]] — the same
 * arithmetic as dm_dfr_average, so a partitioned run is bit-identical to
 * the one-GPU run. */
int dm_dfr_average_csr(int64_t P, const int32_t *proc_ptr, const int32_t *proc_layers, const double *mbar,
                       double *out, int apply, void *stream);
int dm_dfr_boundary_gather(int64_t n, const int32_t *layer, const int32_t *slot, const double *mbar, double *buf,
                           void *stream);
int dm_dfr_boundary_average(int64_t n, const int32_t *layer, const int32_t *slot, const int32_t *slot_lo,
                            const int32_t *slot_hi, const double *buf, double *out, int apply, void *stream);
/* interleaved table -> FlatBdds node order */
int dm_dfr_to_nodes(const dm_flat *f, const double *x_il, double *x, void *stream);

/* Perturbation rounding (rounding.py; the paper's primal heuristic, after
 * FastDOG: PAPER.md:5031-5043), one round on fresh min-marginals m0 / m1:
 * per variable (by id) the copies' votes give a direction dir (+1: the
 * copies prefer 0, -1: prefer 1) — unanimous and strict vote, else the sign
 * of the summed differences, else bit 10 of h = splitmix64(seed, round, v);
 * its cost moves by dir * mag * (1 + u), mag = delta (delta * boost when the
 * vote is already unanimous), u = (h >> 11) * 2^-53, split
 * evenly over the copies' duals (lam[l] += that / copies).  values[v] =
 * the voted value (dir > 0 -> 0), agrees[v] = 1 for a unanimous strict
 * vote; *disagree (device int) = variables without one. */
int dm_perturb_round(const dm_flat *f, const double *m0, const double *m1, double *lam, double delta, double boost,
                     uint64_t seed, int round, int8_t *values, int8_t *agrees, int *disagree, void *stream);

/* --- batched quasi-Newton control of a merged instance (config C5) ----------
 * A batch of independent instances concatenated block-diagonally into one
 * flat (paper_2310_08230_b200/batch.py) runs every instance's own L-BFGS
 * iteration side by side: instance k owns diagrams [bdd_off[k],
 * bdd_off[k+1]) and dual coordinates [layer_off[k], layer_off[k+1]); its
 * reductions are taken over its ranges in exactly the order a separate solve
 * takes them (dm_sum's numpy tree per instance, dm_dot's 4096-chunks counted
 * from its first coordinate), so every instance's trajectory is bit-identical
 * to solving it alone.  Vectors that differ per instance (history pairs) are
 * DEVICE arrays of n pointers to merged-length vectors; per-instance scalars
 * are device arrays of n doubles; active[k] = 0 skips instance k.
 *   dm_batch_sum       out[k] = numpy pairwise sum of x over instance k's diagrams
 *   dm_batch_dot       out[k] = dm_dot order of a[k] . b[k] over its coordinates
 *   dm_batch_update    mode 0: x = u; 1: x -= (coef*dot)*u, alpha_out = coef*dot
 *                      (dm_axpy_dev); 2: x = (coef/dot)*x (dm_scale_dev);
 *                      3: x += u*(alpha - coef*dot) (dm_lbfgs_up);
 *                      4: x += coef*u (dm_axpy_host)
 *   dm_batch_curvature s[k] = lam - lam_prev, y[k] = g_prev - g, lam_prev = lam
 *   dm_batch_step_search  dm_step_search per instance (state: 8 doubles per
 *                      instance, same layout), trial sweeps on lam + gamma_k*d */
typedef struct dm_batch dm_batch;
int dm_batch_create(const dm_flat *f, int n, const int64_t *bdd_off, const int64_t *layer_off, void *stream,
                    dm_batch **out);
void dm_batch_destroy(dm_batch *b);
int dm_batch_sum(const dm_batch *b, const double *x, double *out, void *stream);
int dm_batch_dot(const dm_batch *b, const double *const *a, const double *const *bb, const int8_t *active,
                 double *out, void *stream);
int dm_batch_update(const dm_batch *b, int mode, double *x, const double *const *u, const double *coef,
                    const double *dot, const double *alpha, double *alpha_out, const int8_t *active, void *stream);
int dm_batch_curvature(const dm_batch *b, const double *lam, double *lam_prev, const double *g, const double *g_prev,
                       double *const *s, double *const *y, const int8_t *active, void *stream);
int dm_batch_step_search(const dm_flat *f, const dm_batch *b, const double *lam, const double *d,
                         const double *gamma_prev, const double *free_c, const double *min_ascent, double shrink,
                         double grow, int max_trials, const int8_t *active, double *bounds, double *sums,
                         double *state, void *stream);

/* --- vectors over dual coordinates / variables ----------------------------- */
/* dual.py:137-144: lam[l] = costs[var(l)] / count(var(l)); costs indexed by variable */
int dm_init_duals(const dm_flat *f, const double *costs_by_var, double *lam, void *stream);
/* qn.py:118-129: d[l] = d_hat[l] - mean over the copies of var(l) */
int dm_project_direction(const dm_flat *f, const double *d_hat, double *d, void *stream);
/* dual.py:114-119: per-variable sum of lam over its copies (by variable id) */
int dm_lambda_sums(const dm_flat *f, const double *lam, double *sums_by_var, void *stream);
/* primal.py:83-111: agreement votes from fresh min-marginals (by variable id).
 * agrees[v] in {0,1}; preferred[v] in {0,1}; score[v] = |sum of differences| */
int dm_agreement_scores(const dm_flat *f, const double *m0, const double *m1, int8_t *agrees,
                        double *score, int8_t *preferred, void *stream);

/* dm_sum: numpy pairwise summation order (np.add.reduce on contiguous
 * float64): out[0] = 0.0 + pairwise(x[0:n]) — bit-identical to the
 * reference's bound sums.  dm_dot: the fixed inner-product order of the
 * L-BFGS path — numpy pairwise over each 4096-element chunk of a*b, then
 * over the chunk totals (any n: up to 4096 totals in one block, beyond that
 * through the dm_sum tree); the reference's OpenBLAS ddot order
 * is host-dependent, so any fixed order is parity-equivalent.  Results land in device
 * memory.  Reduction trees and their scratch are planned once per (device,
 * length, stream) and cached for the process, so solves on different streams
 * may run concurrently; calls on one stream are ordered by that stream. */
int dm_sum(const double *x, int64_t n, double *out, void *stream);
/* Free every cached reduction plan / dot scratch (all devices; synchronises
 * them first).  For long-running processes between batches, with no work in
 * flight on any stream that used them. */
int dm_release_caches(void);
int dm_dot(const double *a, const double *b, int64_t n, double *out, void *stream);

/* L-BFGS two-loop recursion (reference qn.py:95-115, lbfgs_direction):
 * d = H*g from m curvature pairs, newest first — s[i], y[i] device vectors of
 * length n, rho[i] = 1/sy[i] and sy[i] = s[i].y[i] host scalars.  Each launch
 * fuses one update with the next inner product (dm_dot order), so d is
 * bit-identical to the dm_dot / dm_axpy_dev / dm_scale_dev / dm_lbfgs_up
 * sequence; 2m+2 launches, m <= 64.  Shares dm_dot's per-length scratch. */
int dm_lbfgs_direction(const double *g, const double *const *s, const double *const *y, const double *rho,
                       const double *sy, int m, int64_t n, double *d, void *stream);

/* Curvature pair of one quasi-Newton iteration (reference qn.py:245-252 +
 * update_history's s @ y, qn.py:85-92) in one pass: s = lam - lam_prev,
 * y = g_prev - g, lam_prev = lam, *sy = s . y in dm_dot's order — values
 * identical to dm_sub, dm_sub, dm_dot and a copy.  Shares dm_dot's scratch. */
int dm_curvature_pair(const double *lam, double *lam_prev, const double *g, const double *g_prev, double *s,
                      double *y, int64_t n, double *sy, void *stream);

/* Elementwise updates with numpy's rounding (no contraction):
 *   dm_axpy_dev : x[i] = x[i] - (alpha_host * dot_dev[0]) * y[i]            (qn.py:108-109)
 *   dm_scale_dev: x[i] = (num_host / den_dev[0]) * x[i]                     (qn.py:111-112)
 *   dm_lbfgs_up : x[i] = x[i] + s[i] * (alpha_dev[0] - rho_host * dot_dev[0]) (qn.py:113-115)
 *   dm_axpy_host: x[i] = x[i] + gamma * y[i]                                (dual.py:83-87)
 *   dm_sub      : out[i] = a[i] - b[i]                                      (qn.py:250)
 * alpha_out (optional) receives alpha_host * dot_dev[0] for dm_axpy_dev. */
int dm_axpy_dev(double *x, const double *y, double alpha_host, const double *dot_dev,
                double *alpha_out, int64_t n, void *stream);
int dm_scale_dev(double *x, double num_host, const double *den_dev, int64_t n, void *stream);
int dm_lbfgs_up(double *x, const double *s, const double *alpha_dev, double rho_host,
                const double *dot_dev, int64_t n, void *stream);
int dm_axpy_host(double *x, double gamma, const double *y, int64_t n, void *stream);
int dm_sub(double *out, const double *a, const double *b, int64_t n, void *stream);

/* --- host-side checks of the device plans (tests only, not a fallback) ---- */
/* Evaluates the planned pairwise tree on the host: == np.sum(x). */
int dm_host_pairwise_sum(const double *x, int64_t n, double *out);
/* Runs one exact averaging pass on the host in level-schedule task order
 * with the device kernel's lane semantics (forward != 0: forward pass; F
 * resets F[root] = 0 itself).  Used by the CPU
 * test-suite to prove the schedule reproduces the sequential pass. */
/* Test hook: the exact-pass division of a copy-delta sum by its copy count k
 * (1..8) against __ddiv_rn on n hashed doubles; *mismatches = differing bits. */
int dm_debug_div_check(int k, uint64_t n, uint64_t seed, unsigned long long *mismatches);
int dm_debug_emulate_mma(const dm_flat_desc *desc, int forward, double *lam, double *F, double *B,
                         double *bounds, int64_t *depth_out);

#ifdef __cplusplus
}
#endif
#endif /* DISCOMATCH_B200_H */
