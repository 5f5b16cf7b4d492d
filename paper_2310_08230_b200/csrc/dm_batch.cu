// Batched quasi-Newton control for a merged block-diagonal instance (config
// C5, paper_2310_08230_b200/batch.py BatchedSolver): the vector reductions
// and updates of every instance's own L-BFGS iteration, side by side.
//
// Each instance k owns a diagram range and a layer (dual-coordinate) range
// of the merged flat table.  Its reductions are taken over ITS range in
// exactly the order a separate solve of it takes them, so every instance's
// trajectory is bit-identical to its separate qn.solve:
//   * batch_sum   — numpy pairwise sums over each instance's per-diagram
//                   values (the bounds, dual.py:67), one tree per instance;
//   * batch_dot   — the chunked inner product (dm_dot: numpy pairwise over
//                   4096-element chunks counted from the instance's first
//                   layer, then over its chunk totals), per instance;
//   * batch_update — the two-loop's updates (dm_axpy_dev, dm_scale_dev,
//                   dm_lbfgs_up) and the quasi-Newton move (dm_axpy_host)
//                   with per-instance scalars; the same roundings;
//   * batch_curvature — s = lam - lam_prev, y = g_prev - g, lam_prev = lam;
//   * batch_decide — find_step_size's per-trial decision (qn.py:132-159,
//                   dm_step_search's step_decide) on each instance's state.
// Per-instance vectors that differ between instances (the history pairs,
// each instance's own ring of pool slots) are passed as device arrays of n
// pointers to merged-length vectors.  `active` masks instances whose
// separate solve would not run the step (stopped, or no history yet).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "dm_internal.h"

#define DM_INF __longlong_as_double(0x7ff0000000000000LL)

namespace {

#include "dm_reduce.cuh"

constexpr int kChunk = 4096;
constexpr int kChunkBlock = 512;

int fail(cudaError_t e, const char *what) {
    dm::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DM_ERR_CUDA;
}

// numpy pairwise leaves (loops_utils.h.src pairwise_sum, <= 128 elements):
// an octet per leaf, lane q owns accumulator r[q]
__global__ void batch_leaf_kernel(int64_t nleaves, const int64_t *__restrict__ leaf_off,
                                  const int32_t *__restrict__ leaf_len, const double *__restrict__ x,
                                  double *__restrict__ vals) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k = t >> 3;
    const int q = threadIdx.x & 7;
    const bool live = k < nleaves;
    const int64_t off = live ? leaf_off[k] : 0;
    const int32_t n = live ? leaf_len[k] : 0;
    const int32_t stop = n - (n % 8);
    double r = 0.0;
    if (live && n >= 8) {
        r = x[off + q];
        for (int32_t i = 8; i < stop; i += 8) r = __dadd_rn(r, x[off + i + q]);
    }
    const double r1 = __shfl_xor_sync(0xffffffffu, r, 1);
    const double s01 = (q & 1) ? __dadd_rn(r1, r) : __dadd_rn(r, r1);
    const double s2 = __shfl_xor_sync(0xffffffffu, s01, 2);
    const double s03 = (q & 2) ? __dadd_rn(s2, s01) : __dadd_rn(s01, s2);
    const double s4 = __shfl_xor_sync(0xffffffffu, s03, 4);
    const double s07 = (q & 4) ? __dadd_rn(s4, s03) : __dadd_rn(s03, s4);
    if (!live || q != 0) return;
    double res = n < 8 ? 0.0 : s07;
    for (int32_t i = n < 8 ? 0 : stop; i < n; ++i) res = __dadd_rn(res, x[off + i]);
    vals[k] = res;
}

// each instance's tree, height by height (a block per instance)
__global__ void batch_combine_kernel(int n, const int32_t *__restrict__ inst_hlo, const int32_t *__restrict__ hlo,
                                     const int32_t *__restrict__ left, const int32_t *__restrict__ right,
                                     const int32_t *__restrict__ int_vid, const int32_t *__restrict__ root,
                                     double *__restrict__ vals, double *__restrict__ out) {
    const int k = blockIdx.x;
    if (k >= n) return;
    const int32_t h0 = inst_hlo[k], h1 = inst_hlo[k + 1];  // hlo[h0 .. h1): this instance's height bounds
    for (int32_t h = h0 + 1; h < h1; ++h) {
        for (int32_t m = hlo[h - 1] + threadIdx.x; m < hlo[h]; m += blockDim.x)
            vals[int_vid[m]] = __dadd_rn(vals[left[m]], vals[right[m]]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = __dadd_rn(0.0, root[k] >= 0 ? vals[root[k]] : 0.0);
}

// chunk totals of a . b, chunks aligned at each instance's first layer
__global__ void __launch_bounds__(kChunkBlock) batch_chunk_kernel(
    const int64_t *__restrict__ chunk_off, const int32_t *__restrict__ chunk_len,
    const int32_t *__restrict__ chunk_inst, const SumPlan *__restrict__ tail_plans, const SumPlan *__restrict__ full,
    const double *const *__restrict__ a, const double *const *__restrict__ b, const int8_t *__restrict__ active,
    double *__restrict__ partial) {
    __shared__ double buf[kChunk];
    const int64_t c = blockIdx.x;
    const int k = chunk_inst[c];
    if (active && !active[k]) return;
    const int64_t off = chunk_off[c];
    const int len = chunk_len[c];
    const double *pa = a[k] + off, *pb = b[k] + off;
    for (int i = threadIdx.x; i < len; i += blockDim.x) buf[i] = __dmul_rn(pa[i], pb[i]);
    __syncthreads();
    const double t = smem_pairwise(buf, len == kChunk ? *full : tail_plans[k]);
    if (threadIdx.x == 0) partial[c] = t;
}

// per instance: pairwise over its chunk totals
__global__ void __launch_bounds__(kChunkBlock) batch_totals_kernel(int n, const int32_t *__restrict__ inst_chunk_lo,
                                                                   const SumPlan *__restrict__ tot_plans,
                                                                   const double *__restrict__ partial,
                                                                   const int8_t *__restrict__ active,
                                                                   double *__restrict__ out) {
    __shared__ double buf[kChunk];
    const int k = blockIdx.x;
    if (k >= n || (active && !active[k])) return;
    const int32_t lo = inst_chunk_lo[k], nch = inst_chunk_lo[k + 1] - lo;
    for (int i = threadIdx.x; i < nch; i += blockDim.x) buf[i] = partial[lo + i];
    __syncthreads();
    const double t = smem_pairwise(buf, tot_plans[k]);
    if (threadIdx.x == 0) out[k] = t;
}

// two-loop updates and the quasi-Newton move, per instance (a block per chunk)
__global__ void batch_update_kernel(int mode, const int64_t *__restrict__ chunk_off,
                                    const int32_t *__restrict__ chunk_len, const int32_t *__restrict__ chunk_inst,
                                    double *__restrict__ x, const double *const *__restrict__ u,
                                    const double *__restrict__ coef, const double *__restrict__ dot,
                                    const double *__restrict__ alpha, double *__restrict__ alpha_out,
                                    const int8_t *__restrict__ active, const int32_t *__restrict__ inst_chunk_lo) {
    const int64_t c = blockIdx.x;
    const int k = chunk_inst[c];
    if (active && !active[k]) return;
    const int64_t off = chunk_off[c];
    const int len = chunk_len[c];
    double *px = x + off;
    const double *pu = (mode == dm::kBatchScaleDev) ? nullptr : u[k] + off;
    double cf = 0.0;
    switch (mode) {
        case dm::kBatchAxpyDev:  // x -= (coef * dot) * u; alpha_out = coef * dot   (dm_axpy_dev)
            cf = __dmul_rn(coef[k], dot[k]);
            if (alpha_out && threadIdx.x == 0 && c == inst_chunk_lo[k]) alpha_out[k] = cf;
            break;
        case dm::kBatchScaleDev:  // x = (coef / dot) * x                          (dm_scale_dev)
            cf = __ddiv_rn(coef[k], dot[k]);
            break;
        case dm::kBatchLbfgsUp:  // x += u * (alpha - coef * dot)                  (dm_lbfgs_up)
            cf = __dsub_rn(alpha[k], __dmul_rn(coef[k], dot[k]));
            break;
        case dm::kBatchAxpyHost:  // x += coef * u                                 (dm_axpy_host)
            cf = coef[k];
            break;
        default:
            break;
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        switch (mode) {
            case dm::kBatchCopy: px[i] = pu[i]; break;
            case dm::kBatchAxpyDev: px[i] = __dsub_rn(px[i], __dmul_rn(cf, pu[i])); break;
            case dm::kBatchScaleDev: px[i] = __dmul_rn(cf, px[i]); break;
            case dm::kBatchLbfgsUp: px[i] = __dadd_rn(px[i], __dmul_rn(pu[i], cf)); break;
            case dm::kBatchAxpyHost: px[i] = __dadd_rn(px[i], __dmul_rn(cf, pu[i])); break;
            default: break;
        }
    }
}

// s = lam - lam_prev, y = g_prev - g, lam_prev = lam (dm_curvature_pair's vectors)
__global__ void batch_curvature_kernel(const int64_t *__restrict__ chunk_off, const int32_t *__restrict__ chunk_len,
                                       const int32_t *__restrict__ chunk_inst, const double *__restrict__ lam,
                                       double *__restrict__ lam_prev, const double *__restrict__ g,
                                       const double *__restrict__ g_prev, double *const *__restrict__ s,
                                       double *const *__restrict__ y, const int8_t *__restrict__ active) {
    const int64_t c = blockIdx.x;
    const int k = chunk_inst[c];
    if (active && !active[k]) return;
    const int64_t off = chunk_off[c];
    const int len = chunk_len[c];
    double *ps = s[k] + off, *py = y[k] + off;
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const int64_t e = off + i;
        ps[i] = __dsub_rn(lam[e], lam_prev[e]);
        py[i] = __dsub_rn(g_prev[e], g[e]);
        lam_prev[e] = lam[e];
    }
}

// find_step_size's per-trial decision (dm_step_search's step_decide), per
// instance: state = {gamma, e_init, e_best, gamma_best, e_cur, stop, trials, -}
__global__ void batch_decide_kernel(int n, const double *__restrict__ sums, double *__restrict__ state,
                                    const double *__restrict__ free_c, const double *__restrict__ min_ascent,
                                    double shrink, double grow, int max_trials, int trial) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double *ctl = state + 8 * k;
    if (ctl[5] != 0.0) return;
    const double e = __dadd_rn(sums[k], free_c[k]);
    ctl[6] = ctl[6] + 1.0;
    if (trial == 0) {
        ctl[1] = ctl[2] = ctl[4] = e;
        ctl[3] = ctl[0];
    } else {
        ctl[4] = e;
        if (e >= ctl[2]) {
            ctl[3] = ctl[0];
            ctl[2] = e;
        }
        if (__dsub_rn(e, ctl[1]) >= min_ascent[k]) {
            ctl[5] = 1.0;
            return;
        }
    }
    if (trial < max_trials)
        ctl[0] = __dmul_rn(ctl[0], ctl[4] <= ctl[1] ? shrink : grow);
    else
        ctl[5] = 1.0;
}

__global__ void batch_step_init_kernel(int n, double *__restrict__ state, const double *__restrict__ gamma,
                                       const int8_t *__restrict__ active) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double *ctl = state + 8 * k;
    ctl[0] = gamma[k];
    for (int i = 1; i < 8; ++i) ctl[i] = 0.0;
    if (!active[k]) ctl[5] = 1.0;  // no search for this instance
}

template <typename T>
cudaError_t up(std::vector<void *> &allocs, const T **dst, const std::vector<T> &src, cudaStream_t s) {
    T *p = nullptr;
    const size_t bytes = std::max<size_t>(src.size(), 1) * sizeof(T);
    cudaError_t e = cudaMallocAsync((void **)&p, bytes, s);
    if (e) return e;
    allocs.push_back(p);
    if (!src.empty()) e = cudaMemcpyAsync(p, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    *dst = p;
    return e;
}

}  // namespace

namespace dm {

int batch_build(const int64_t *bdd_off, const int64_t *layer_off, int n, BatchPlan &b, std::vector<void *> &allocs,
                void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    b.n = n;
    b.nb = bdd_off[n];
    b.L = layer_off[n];
    // per-instance pairwise trees over the diagram segments, one value space:
    // [every leaf ..., every internal node ...]
    std::vector<PairwisePlan> plans(n);
    {  // the instances' trees are independent: built by a few host threads
        const int nt = std::max(1, std::min(n, 8));
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (int k = t; k < n; k += nt) plans[k] = plan_pairwise(bdd_off[k + 1] - bdd_off[k]);
            });
        for (auto &x : th) x.join();
    }
    int64_t NL = 0, NI = 0;
    for (int k = 0; k < n; ++k) {
        NL += (int64_t)plans[k].leaf_off.size();
        NI += (int64_t)plans[k].left.size();
    }
    if (NL + NI >= INT32_MAX) {
        set_error("batch too large for the per-instance reduction plans");
        return DM_ERR_UNSUPPORTED;
    }
    std::vector<int64_t> leaf_off;
    std::vector<int32_t> leaf_len, left, right, int_vid, hlo, inst_hlo(n + 1, 0), root(n, -1);
    leaf_off.reserve(NL);
    int64_t lbase = 0, ibase = 0;
    for (int k = 0; k < n; ++k) {
        const PairwisePlan &p = plans[k];
        const int64_t nl = (int64_t)p.leaf_off.size(), ni = (int64_t)p.left.size();
        auto vid = [&](int32_t local) { return (int32_t)(local < nl ? lbase + local : NL + ibase + (local - nl)); };
        for (int64_t i = 0; i < nl; ++i) {
            leaf_off.push_back(bdd_off[k] + p.leaf_off[i]);
            leaf_len.push_back(p.leaf_len[i]);
        }
        for (int64_t m = 0; m < ni; ++m) {
            left.push_back(vid(p.left[m]));
            right.push_back(vid(p.right[m]));
            int_vid.push_back((int32_t)(NL + ibase + m));
        }
        // height bounds: hlo[inst_hlo[k] + h] = end of the nodes of height <= h (global internal index)
        inst_hlo[k] = (int32_t)hlo.size();
        hlo.push_back((int32_t)ibase);
        for (size_t h = 1; h < p.height_lo.size(); ++h) hlo.push_back((int32_t)(ibase + p.height_lo[h]));
        if (bdd_off[k + 1] > bdd_off[k]) root[k] = vid(p.root);
        lbase += nl;
        ibase += ni;
    }
    inst_hlo[n] = (int32_t)hlo.size();
    // the combine kernel walks hlo[inst_hlo[k] .. inst_hlo[k+1]) as consecutive height bounds
    b.nleaves = NL;
    b.nvals = NL + NI;
    // chunks of the layer segments, aligned at each instance's first layer
    std::vector<int64_t> chunk_off;
    std::vector<int32_t> chunk_len, chunk_inst, inst_chunk_lo(n + 1, 0);
    std::vector<SumPlan> tail(n), tot(n);
    for (int k = 0; k < n; ++k) {
        inst_chunk_lo[k] = (int32_t)chunk_off.size();
        const int64_t len = layer_off[k + 1] - layer_off[k];
        const int64_t nch = (len + kChunk - 1) / kChunk;
        if (nch > kChunk) {
            set_error("batched dots: an instance longer than 4096 * 4096 dual coordinates");
            return DM_ERR_UNSUPPORTED;
        }
        for (int64_t c = 0; c < nch; ++c) {
            chunk_off.push_back(layer_off[k] + c * kChunk);
            chunk_len.push_back((int32_t)std::min<int64_t>(kChunk, len - c * kChunk));
            chunk_inst.push_back(k);
        }
        tail[k] = make_sum_plan((int)(len % kChunk));
        tot[k] = make_sum_plan((int)nch);
    }
    inst_chunk_lo[n] = (int32_t)chunk_off.size();
    b.nchunks = (int64_t)chunk_off.size();
    std::vector<SumPlan> full{make_sum_plan(kChunk)};
    // element -> instance maps
    std::vector<int32_t> bdd_inst(b.nb), layer_inst(b.L);
    for (int k = 0; k < n; ++k) {
        std::fill(bdd_inst.begin() + bdd_off[k], bdd_inst.begin() + bdd_off[k + 1], k);
        std::fill(layer_inst.begin() + layer_off[k], layer_inst.begin() + layer_off[k + 1], k);
    }
    cudaError_t e;
    const SumPlan *tp = nullptr, *op = nullptr, *fp = nullptr;
    if ((e = up(allocs, &b.leaf_off, leaf_off, s)) || (e = up(allocs, &b.leaf_len, leaf_len, s)) ||
        (e = up(allocs, &b.left, left, s)) || (e = up(allocs, &b.right, right, s)) ||
        (e = up(allocs, &b.int_vid, int_vid, s)) || (e = up(allocs, &b.hlo, hlo, s)) ||
        (e = up(allocs, &b.inst_hlo, inst_hlo, s)) || (e = up(allocs, &b.root, root, s)) ||
        (e = up(allocs, &b.chunk_off, chunk_off, s)) || (e = up(allocs, &b.chunk_len, chunk_len, s)) ||
        (e = up(allocs, &b.chunk_inst, chunk_inst, s)) || (e = up(allocs, &b.inst_chunk_lo, inst_chunk_lo, s)) ||
        (e = up(allocs, &tp, tail, s)) || (e = up(allocs, &op, tot, s)) || (e = up(allocs, &fp, full, s)) ||
        (e = up(allocs, &b.bdd_inst, bdd_inst, s)) || (e = up(allocs, &b.layer_inst, layer_inst, s)))
        return fail(e, "batch plan upload");
    b.tail_plans = tp;
    b.tot_plans = op;
    b.full_plan = fp;
    if ((e = cudaMallocAsync((void **)&b.vals, std::max<int64_t>(b.nvals, 1) * sizeof(double), s)) ||
        (e = cudaMallocAsync((void **)&b.partial, std::max<int64_t>(b.nchunks, 1) * sizeof(double), s)))
        return fail(e, "batch scratch");
    allocs.push_back(b.vals);
    allocs.push_back(b.partial);
    e = cudaStreamSynchronize(s);  // the host staging vectors die with this scope
    return e ? fail(e, "batch plan") : DM_OK;
}

int batch_sum(const BatchPlan &b, const double *x, double *out, void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    if (b.nleaves > 0)
        batch_leaf_kernel<<<(int)((b.nleaves * 8 + 255) / 256), 256, 0, s>>>(b.nleaves, b.leaf_off, b.leaf_len, x,
                                                                              b.vals);
    batch_combine_kernel<<<b.n, 256, 0, s>>>(b.n, b.inst_hlo, b.hlo, b.left, b.right, b.int_vid, b.root, b.vals, out);
    const cudaError_t e = cudaGetLastError();
    return e ? fail(e, "batch_sum") : DM_OK;
}

int batch_dot(const BatchPlan &b, const double *const *a, const double *const *bb, const int8_t *active, double *out,
              void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    if (b.nchunks > 0)
        batch_chunk_kernel<<<(unsigned)b.nchunks, kChunkBlock, 0, s>>>(
            b.chunk_off, b.chunk_len, b.chunk_inst, (const SumPlan *)b.tail_plans, (const SumPlan *)b.full_plan, a, bb,
            active, b.partial);
    batch_totals_kernel<<<b.n, kChunkBlock, 0, s>>>(b.n, b.inst_chunk_lo, (const SumPlan *)b.tot_plans, b.partial,
                                                    active, out);
    const cudaError_t e = cudaGetLastError();
    return e ? fail(e, "batch_dot") : DM_OK;
}

int batch_update(const BatchPlan &b, int mode, double *x, const double *const *u, const double *coef,
                 const double *dot, const double *alpha, double *alpha_out, const int8_t *active, void *stream) {
    if (b.nchunks > 0)
        batch_update_kernel<<<(unsigned)b.nchunks, 256, 0, (cudaStream_t)stream>>>(
            mode, b.chunk_off, b.chunk_len, b.chunk_inst, x, u, coef, dot, alpha, alpha_out, active, b.inst_chunk_lo);
    const cudaError_t e = cudaGetLastError();
    return e ? fail(e, "batch_update") : DM_OK;
}

int batch_curvature(const BatchPlan &b, const double *lam, double *lam_prev, const double *g, const double *g_prev,
                    double *const *s, double *const *y, const int8_t *active, void *stream) {
    if (b.nchunks > 0)
        batch_curvature_kernel<<<(unsigned)b.nchunks, 256, 0, (cudaStream_t)stream>>>(
            b.chunk_off, b.chunk_len, b.chunk_inst, lam, lam_prev, g, g_prev, s, y, active);
    const cudaError_t e = cudaGetLastError();
    return e ? fail(e, "batch_curvature") : DM_OK;
}

int batch_step_init(const BatchPlan &b, double *state, const double *gamma, const int8_t *active, void *stream) {
    batch_step_init_kernel<<<(b.n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(b.n, state, gamma, active);
    const cudaError_t e = cudaGetLastError();
    return e ? fail(e, "batch_step_init") : DM_OK;
}

int batch_decide(const BatchPlan &b, const double *sums, double *state, const double *free_c,
                 const double *min_ascent, double shrink, double grow, int max_trials, int trial, void *stream) {
    batch_decide_kernel<<<(b.n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(b.n, sums, state, free_c, min_ascent,
                                                                              shrink, grow, max_trials, trial);
    const cudaError_t e = cudaGetLastError();
    return e ? fail(e, "batch_decide") : DM_OK;
}

}  // namespace dm
