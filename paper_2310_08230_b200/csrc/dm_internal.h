// Internal declarations shared by the host lowering, the schedule builder and
// the CUDA translation units.  Not part of the public C-ABI.
#pragma once

#include <cstdint>
#include <string>
#include <memory>
#include <vector>

#include "../../include/discomatch_b200.h"

namespace dm {

constexpr int32_t kFalse = -1;  // FALSE terminal (bdd.py:24)
constexpr int32_t kTrue = -2;   // TRUE terminal  (bdd.py:25)

void set_error(const std::string &msg);

// One reduced, layered diagram in the reference's Bdd layout (bdd.py:55-87):
// layer l branches on vars[l]; zeros/ones hold local next-layer indices or
// the terminal sentinels; layer_lo[l] .. layer_lo[l+1] indexes zeros/ones.
struct HostBdd {
    std::vector<int64_t> vars;
    std::vector<int64_t> layer_lo;  // size vars.size()+1
    std::vector<int32_t> zeros, ones;
    int64_t width(size_t l) const { return layer_lo[l + 1] - layer_lo[l]; }
};

// Flat table (kernels.py:35-92), int64 like the reference.
struct FlatHost {
    std::vector<double> costs;
    std::vector<int64_t> order, positions, counts;
    std::vector<int64_t> bdd_layer_lo, layer_node_lo, layer_var, layer_bdd;
    std::vector<int64_t> zero_t, one_t, proc_ptr, proc_layers;
    int64_t max_width = 0, max_degree = 0, max_layers = 0;
};

// Returns DM_OK or an error code (message via set_error).
int build_equality_bdd(const int64_t *coef, const int64_t *vars, int64_t n, int64_t rhs,
                       HostBdd &out);
int flatten(std::vector<HostBdd> &bdds, std::vector<double> costs, std::vector<int64_t> order,
            FlatHost &out);

// numpy pairwise-summation tree for a fixed length (loops_utils.h.src
// pairwise_sum: blocks of <= 128 summed with 8 accumulators, splits at
// n/2 rounded down to a multiple of 8).
struct PairwisePlan {
    int64_t n = 0;
    std::vector<int64_t> leaf_off;  // leaves left to right
    std::vector<int32_t> leaf_len;
    // internal nodes ordered by height; children index the value array
    // [leaves..., internal...]
    std::vector<int32_t> left, right;
    std::vector<int32_t> height_lo;  // internal nodes of height h: [height_lo[h-1], height_lo[h])
    int32_t root = 0;                // value index of the root
};
PairwisePlan plan_pairwise(int64_t n);

// Exact-pass schedule: warp tasks of same-level variables; lane i of task k
// handles copy task_layer[32k+i] (global layer id or -1), meta packs the
// lane's group base lane (bits 0-7), group size (8-15), first-layer flag
// (bit 16) and last-layer flag (bit 17).
struct MmaSchedule {
    std::vector<int32_t> task_layer, task_meta, task_level;
    int64_t depth = 0, tasks = 0;
    // one task per visitation position (the node-parallel kernels): positions
    // with copies in level order, and their levels
    std::vector<int32_t> pos_order, pos_order_level;
};
int build_mma_schedule(const int64_t *bdd_layer_lo, int64_t nb, const int64_t *layer_bdd_or_null,
                       const int64_t *layer_var, int64_t L, const int64_t *proc_ptr,
                       const int64_t *proc_layers, int64_t npos, bool forward, MmaSchedule &out);
void pack_mma_tasks(const std::vector<int32_t> &pos_order, const std::vector<int32_t> &pos_order_level,
                    const int32_t *proc_ptr, const int32_t *proc_layers, const uint8_t *layer_flags,
                    MmaSchedule &s);

// The same level orders built on the device (dm_plan.cu), stream-ordered:
// positions with copies sorted by (level, visitation index) into the first
// `nvalid` entries of fw/bw_order, their levels into fw/bw_level (P each);
// words (8 device ints) = {fw queue, fw status, bw queue, bw status,
// fw depth - 1, bw depth - 1}.  Device topology is int32.
int device_level_orders(const int32_t *proc_ptr, const int32_t *proc_layers, const int32_t *layer_bdd,
                        const int32_t *bdd_layer_lo, int64_t P, int64_t L, int64_t nvalid, int32_t *fw_order,
                        int32_t *fw_level, int32_t *bw_order, int32_t *bw_level, int *words, void *stream);
// first/last-layer flags (bit 0/1) per layer
int device_layer_flags(const int32_t *layer_bdd, const int32_t *bdd_layer_lo, int64_t L, uint8_t *flags,
                       void *stream);
// node-parallel copy records (int4 per task and copy slot, 8 slots): task t
// is position order[t] (order null: t itself), P tasks
int device_np_records(const int32_t *proc_ptr, const int32_t *proc_layers, const int32_t *lnl, const uint8_t *flags,
                      const int32_t *order, int64_t P, void *rec, void *stream);

// Uninitialised int32 buffer (every element of the sweep targets is written
// by the parallel fill, so a value-initialising std::vector would only add a
// serial pass over hundreds of MB).
struct I32Buffer {
    std::unique_ptr<int32_t[]> p;
    size_t n = 0;
    void resize(size_t m) {
        p.reset(new int32_t[m]);
        n = m;
    }
    int32_t *data() { return p.get(); }
    const int32_t *data() const { return p.get(); }
    size_t size() const { return n; }
    int32_t &operator[](size_t i) { return p[i]; }
};

// Interleaved sweep layout (dm_layout.cpp): 32 diagrams per warp group,
// layers aligned at the last layer (position 0), node slots interleaved by
// lane, arc targets as local indices into the next layer.
struct SweepLayout {
    int64_t groups = 0, slots = 0, max_width = 0;
    std::vector<int32_t> grp_bdd;     // [groups*32] diagram of each lane, -1 = idle
    std::vector<int32_t> grp_npos;    // [groups] positions (max layers in the group)
    std::vector<int64_t> grp_pos_lo;  // [groups+1] into pos_width / pos_slot
    std::vector<int32_t> pos_width;   // widest layer at each position of each group
    std::vector<int64_t> pos_slot;    // first node slot of each position
    I32Buffer zl, ol;                 // [slots*32] local targets, -1 FALSE, -2 TRUE
};
int build_sweep_layout(const int64_t *bdd_layer_lo, int64_t nb, const int64_t *layer_node_lo,
                       const int64_t *zero_t, const int64_t *one_t, SweepLayout &out);

// Per-layer forward publish descriptors: for each non-final layer, nibble
// 8u (8u+4) names the node whose zero (one) arc enters target u of the next
// layer, 15 = none.  False when a layer is wider than 8 or a target has two
// sources of one arc kind (the tree publish handles those instances).
bool build_relax_by_layer(const int64_t *bdd_layer_lo, int64_t nb, const int64_t *layer_node_lo,
                          const int64_t *zero_t, const int64_t *one_t, std::vector<uint64_t> &desc_out);

// Device view of a SweepLayout plus the reference-layout offsets the sweeps
// need to read duals and write distances (dm_sweep.cu).
struct SweepDev {
    int64_t groups = 0, slots = 0;  // slots * 32 = elements of an interleaved table
    int32_t max_width = 0, max_layers = 0;
    const int32_t *grp_bdd = nullptr, *grp_npos = nullptr, *pos_width = nullptr;
    const int32_t *grp_width = nullptr;  // widest layer of each group (null: max_width)
    const int64_t *grp_pos_lo = nullptr, *pos_slot = nullptr;
    const int32_t *zl = nullptr, *ol = nullptr;
    const int32_t *bdd_layer_lo = nullptr, *lnl = nullptr;
};
// The interleaved layout built on the device (dm_plan.cu): sizes, groups,
// widths and slot offsets into `sd` (device pointers registered in
// allocs/bytes; synchronises `stream` twice for the sizes; 0, -1 CUDA error,
// -2 too large), then device_sweep_fill writes the arc targets.
int device_sweep_layout(const int32_t *bl, const int32_t *lnl, int64_t nb, SweepDev &sd, std::vector<void *> &allocs,
                        int64_t &bytes, void *stream);
int device_sweep_fill(const SweepDev &sd, const int32_t *zero_t, const int32_t *one_t, void *stream);
// forward publish descriptors on the device; *fail != 0 afterwards: unusable
int device_relax(const int32_t *layer_bdd, const int32_t *bl, const int32_t *lnl, const int32_t *zero_t,
                 const int32_t *one_t, int64_t L, uint64_t *desc, unsigned long long *fail, void *stream);
// kernels.py:95-120 (B may be null: trial evaluation, bounds only; d null: plain duals)
// ctl (device step search, dm_step_search): gamma read from ctl[0], the
// launch returns at once when ctl[5] (stop) is set.
// bdd_inst (batched step search, dm_batch.cu): gamma of diagram j = ctl[8 * bdd_inst[j]]
int sweep_backward(const SweepDev &s, const double *lam, const double *d, double gamma, double *B,
                   double *bounds, void *stream, const double *ctl = nullptr, const int32_t *bdd_inst = nullptr);
// kernels.py:123-159
int sweep_forward(const SweepDev &s, const double *lam, double *F, double *bounds, void *stream);
// numpy-order pairwise sum of a device vector into out[0] (dm_device.cu's
// planned pw_leaf / pw_combine kernels, the dm_sum path), stream-ordered.
int pairwise_device(const double *x, int64_t n, double *out, void *stream);
// Chunked inner product (dm_sweep.cu): partial[nchunks] scratch; the chunk
// totals are reduced in the finishing block up to 4096 chunks and by
// pairwise_device beyond (same numpy order: vectors of any length).
int chunk_dot(const double *a, const double *b, int64_t n, double *partial, double *out, void *stream);
constexpr int64_t kDotChunk = 4096;
// L-BFGS two-loop direction (qn.py:95-115) in 2m+2 fused launches; s/y are
// host arrays of m device pointers (newest first), slots >= 3m+1 doubles.
// s = lam - lam_prev, y = g_prev - g, lam_prev = lam and sy = s . y (chunked-dot order), one pass
int curvature_pair(const double *lam, double *lam_prev, const double *g, const double *g_prev, double *s,
                   double *y, int64_t n, double *partial, double *sy, void *stream);
// Deferred (throughput) averaging schedule (dm_deferred.cu): one pass over
// every diagram, forward or backward, on interleaved tables; mbar == null:
// no min-marginal step (a sweep that only adds avg); avg == null: nothing to
// add; dec (backward, W <= 8): argmin decision words per layer.
int dfr_pass(const SweepDev &s, bool forward, double omega, double *lam, const double *avg, const double *in,
             double *out, double *mbar, double *bounds, uint64_t *dec, void *stream);
// apply: lam[l] += average (the flush) instead of avg[l] = average
int dfr_average(int64_t P, const int32_t *proc_ptr, const int32_t *proc_layers, const double *mbar, double *out,
                bool apply, void *stream);
int dfr_to_nodes(const SweepDev &s, const double *x_il, double *x, void *stream);
// the same passes node-parallel (8 lanes per diagram; W <= 8 with single-source
// publish descriptors `relax`), tables in the reference node order
int dfr_np_pass(const SweepDev &s, const int32_t *zero_t, const int32_t *one_t, const uint64_t *relax, bool forward,
                double omega, double *lam, const double *avg, const double *in, double *out, double *mbar,
                double *bounds, uint64_t *dec, void *stream);
int dfr_boundary_gather(int64_t n, const int32_t *layer, const int32_t *slot, const double *mbar, double *buf,
                        void *stream);
int dfr_boundary_average(int64_t n, const int32_t *layer, const int32_t *slot, const int32_t *slot_lo,
                         const int32_t *slot_hi, const double *buf, double *out, bool apply, void *stream);
// bar (3 zeroed words) and partial[2 * nchunks]: the whole recursion in one
// cooperative launch; bar == null: 2m+2 fused launches
int lbfgs_two_loop(const double *g, const double *const *s, const double *const *y, const double *rho,
                   const double *sy, int m, int64_t n, double *d, double *slots, double *partial, void *stream,
                   unsigned *bar = nullptr);

// Batched quasi-Newton control of a merged block-diagonal instance
// (dm_batch.cu): per-instance reduction plans and element -> instance maps.
enum { kBatchCopy = 0, kBatchAxpyDev = 1, kBatchScaleDev = 2, kBatchLbfgsUp = 3, kBatchAxpyHost = 4 };
struct BatchPlan {
    int n = 0;
    int64_t nb = 0, L = 0;
    // per-instance numpy pairwise trees over the diagram segments
    int64_t nleaves = 0, nvals = 0;
    const int64_t *leaf_off = nullptr;
    const int32_t *leaf_len = nullptr, *left = nullptr, *right = nullptr, *int_vid = nullptr;
    const int32_t *hlo = nullptr, *inst_hlo = nullptr, *root = nullptr;
    double *vals = nullptr;
    // chunks of the layer segments (4096, aligned at each instance's first layer)
    int64_t nchunks = 0;
    const int64_t *chunk_off = nullptr;
    const int32_t *chunk_len = nullptr, *chunk_inst = nullptr, *inst_chunk_lo = nullptr;
    const void *tail_plans = nullptr, *tot_plans = nullptr, *full_plan = nullptr;  // SumPlan arrays
    double *partial = nullptr;
    const int32_t *bdd_inst = nullptr, *layer_inst = nullptr;
};
int batch_build(const int64_t *bdd_off, const int64_t *layer_off, int n, BatchPlan &b, std::vector<void *> &allocs,
                void *stream);
int batch_sum(const BatchPlan &b, const double *x, double *out, void *stream);
int batch_dot(const BatchPlan &b, const double *const *a, const double *const *bb, const int8_t *active, double *out,
              void *stream);
int batch_update(const BatchPlan &b, int mode, double *x, const double *const *u, const double *coef,
                 const double *dot, const double *alpha, double *alpha_out, const int8_t *active, void *stream);
int batch_curvature(const BatchPlan &b, const double *lam, double *lam_prev, const double *g, const double *g_prev,
                    double *const *s, double *const *y, const int8_t *active, void *stream);
int batch_step_init(const BatchPlan &b, double *state, const double *gamma, const int8_t *active, void *stream);
int batch_decide(const BatchPlan &b, const double *sums, double *state, const double *free_c,
                 const double *min_ascent, double shrink, double grow, int max_trials, int trial, void *stream);

}  // namespace dm
