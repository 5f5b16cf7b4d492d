// Full-table sweeps over the interleaved sweep layout (dm_layout.cpp):
//   sweep_backward  == k_backward  (kernels.py:95-120) and, with d != null,
//                      the step-search trial on lam + gamma*d (qn.py:147,153)
//   sweep_forward   == k_forward   (kernels.py:123-159)
//
// One warp sweeps 32 diagrams of similar shape.  Each step reads the arc
// targets of one layer position for all 32 lanes as contiguous 128-byte
// rows; the neighbouring layer's distances live in shared memory (per-thread
// column, conflict-free), so there is no dependent L2 round trip per layer.
// Arithmetic and tie rules are the reference's: c1 = lam + B[t] (one
// rounding), B = c0 <= c1 ? c0 : c1, forward scatter in (node, zero, one)
// order with strict <.
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "dm_internal.h"
#include "dm_rows.cuh"

#define DM_INF __longlong_as_double(0x7ff0000000000000LL)

namespace {

constexpr int kSweepThreads = 128;

// W: node slots the loops cover (>= the group's widest layer), WS: the slot
// stride of the shared distance rows (the launch's width)
template <int W, int WS, bool kTrial, bool kStore>
__device__ __forceinline__ void sweep_backward_body(const dm::SweepDev &s, const double *__restrict__ lam,
                                                    const double *__restrict__ d, double gamma,
                                                    double *__restrict__ B, double *__restrict__ bounds,
                                                    const double *__restrict__ ctl,
                                                    const int32_t *__restrict__ bdd_inst, int64_t g, double *sm) {
    const int lane = threadIdx.x & 31;
    const int32_t j = s.grp_bdd[g * 32 + lane];
    // batched step search (dm_batch.cu): each diagram's own instance's gamma
    // (stopped searches are evaluated too and ignored by their decision)
    if (kTrial && bdd_inst && j >= 0) gamma = ctl[8 * bdd_inst[j]];
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = s.bdd_layer_lo[j];
        nj = s.bdd_layer_lo[j + 1] - l0;
    }
    const int32_t K = s.grp_npos[g];
    const int64_t p0 = s.grp_pos_lo[g];
    constexpr bool kReg = W <= kRegRowsSweep;
    Row<W, kReg, kSweepThreads> nb, cur;  // distances of position k-1 (next layer) and of position k
    if constexpr (kReg) {
#pragma unroll
        for (int u = 0; u < W; ++u) nb.put(u, DM_INF), cur.put(u, DM_INF);
    } else {
        nb.p = sm + threadIdx.x;
        cur.p = sm + WS * kSweepThreads + threadIdx.x;
    }
    // Register double buffer: the arc targets and dual of position k+1 are
    // loaded while position k is computed, so each step waits on shared
    // memory only (the sweep is otherwise one DRAM round trip per layer).
    int32_t za[W], oa[W];
    double lam_n = 0.0, d_n = 0.0;
    auto fetch = [&](int32_t k, int32_t &w, int64_t &slot) {
        w = s.pos_width[p0 + k];
        slot = s.pos_slot[p0 + k];
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < w) {
                za[i] = s.zl[(slot + i) * 32 + lane];
                oa[i] = s.ol[(slot + i) * 32 + lane];
            }
        if (k < nj) {
            const int32_t l = l0 + nj - 1 - k;
            lam_n = lam[l];
            if (kTrial) d_n = d[l];
        }
    };
    int32_t w_n;
    int64_t slot_n;
    if (K > 0) fetch(0, w_n, slot_n);
    for (int32_t k = 0; k < K; ++k) {
        const int32_t w = w_n;
        int32_t z[W], o[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            z[i] = za[i];
            o[i] = oa[i];
        }
        const bool act = k < nj;
        const int32_t l = l0 + nj - 1 - k;
        double lam_l = act ? lam_n : 0.0;
        if (kTrial && act) lam_l = __dadd_rn(lam_l, __dmul_rn(gamma, d_n));
        if (k + 1 < K) fetch(k + 1, w_n, slot_n);
        int32_t vbase = 0, wl = 0;
        if (kStore && act) {
            vbase = s.lnl[l];
            wl = s.lnl[l + 1] - vbase;
        }
        double vv[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            vv[i] = 0.0;
            if (i < w) {
                const int32_t a = z[i], b = o[i];
                const double c0 = a == dm::kTrue ? 0.0 : (a == dm::kFalse ? DM_INF : nb.get(a));
                const double c1 = b == dm::kTrue ? lam_l : (b == dm::kFalse ? DM_INF : __dadd_rn(lam_l, nb.get(b)));
                const double v = (c0 <= c1) ? c0 : c1;
                cur.put(i, v);
                vv[i] = v;
            }
        }
        if (kStore && wl > 0) {
            // the layer's distances are wl consecutive doubles of this lane's
            // diagram: 16-byte stores on the aligned pairs (each lane writes a
            // different diagram, so every store is its own transaction)
            const int odd = vbase & 1;
            if (odd) B[vbase] = vv[0];
#pragma unroll
            for (int i = 0; i + 1 < W; i += 2) {
                const int e = i + odd;  // first element of the aligned pair
                if (e + 1 < wl) {
                    double2 pr;
                    pr.x = odd ? vv[(i + 1) % W] : vv[i];
                    pr.y = odd ? vv[(i + 2) % W] : vv[i + 1];
                    *reinterpret_cast<double2 *>(B + vbase + e) = pr;
                } else if (e < wl) {
                    B[vbase + e] = odd ? vv[(i + 1) % W] : vv[i];
                }
            }
        }
        swap_rows(nb, cur);
        if (act && k == nj - 1) bounds[j] = nb.at(0);  // root layer: single node
    }
}

// Two-node groups (the long chains of split rows, the sweep's critical
// path on a pruned instance): the per-position metadata is staged per warp
// in shared memory, a window of kSweepMetaWin positions at a time, and the
// arc targets and duals are loaded kRingDepth positions ahead into a
// register ring (the loop unrolled by the ring depth, so every slot index is
// a constant) — a position then waits on neither a dependent metadata load
// nor a load issued one short step earlier.  Same arithmetic as the body
// above, bit for bit.
#ifndef DM_SWEEP_RING
#define DM_SWEEP_RING 1
#endif
constexpr bool kSweepRing = DM_SWEEP_RING != 0;
constexpr int kSweepMetaWin = 64;
#ifndef DM_RING_DEPTH
#define DM_RING_DEPTH 4
#endif
constexpr int kRingDepth = DM_RING_DEPTH;
constexpr int kSweepWarps = kSweepThreads / 32;

template <int W>
struct RingSlot {
    int32_t w;
    int64_t slot;
    int32_t z[W], o[W];
    double lam, d;
};

template <int W, bool kTrial, bool kStore>
__device__ __forceinline__ void sweep_backward_ring(const dm::SweepDev &s, const double *__restrict__ lam,
                                                    const double *__restrict__ d, double gamma,
                                                    double *__restrict__ B, double *__restrict__ bounds,
                                                    const double *__restrict__ ctl,
                                                    const int32_t *__restrict__ bdd_inst, int64_t g, int32_t *mw,
                                                    int64_t *ms) {
    const int lane = threadIdx.x & 31;
    const int32_t j = s.grp_bdd[g * 32 + lane];
    if (kTrial && bdd_inst && j >= 0) gamma = ctl[8 * bdd_inst[j]];
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = s.bdd_layer_lo[j];
        nj = s.bdd_layer_lo[j + 1] - l0;
    }
    const int32_t K = s.grp_npos[g];
    const int64_t p0 = s.grp_pos_lo[g];
    int32_t mlo = 0;  // first position in the metadata window
    auto window = [&](int32_t lo) {
        __syncwarp();
        for (int i = lane; i < kSweepMetaWin; i += 32)
            if (lo + i < K) {
                mw[i] = s.pos_width[p0 + lo + i];
                ms[i] = s.pos_slot[p0 + lo + i];
            }
        __syncwarp();
        mlo = lo;
    };
    window(0);
    auto fetch = [&](RingSlot<W> &r, int32_t k) {
        if (k >= mlo + kSweepMetaWin) window(k);  // uniform: k is the warp's
        r.w = mw[k - mlo];
        r.slot = ms[k - mlo];
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < r.w) {
                r.z[i] = s.zl[(r.slot + i) * 32 + lane];
                r.o[i] = s.ol[(r.slot + i) * 32 + lane];
            }
        if (k < nj) {
            const int32_t l = l0 + nj - 1 - k;
            r.lam = lam[l];
            if (kTrial) r.d = d[l];
        }
    };
    double nb[W], cur[W];
#pragma unroll
    for (int u = 0; u < W; ++u) nb[u] = cur[u] = DM_INF;
    RingSlot<W> ring[kRingDepth];
#pragma unroll
    for (int r = 0; r < kRingDepth; ++r)
        if (r < K) fetch(ring[r], r);
    for (int32_t k0 = 0; k0 < K; k0 += kRingDepth) {
#pragma unroll
        for (int r = 0; r < kRingDepth; ++r) {
            const int32_t k = k0 + r;
            if (k < K) {
                const RingSlot<W> c = ring[r];
                if (k + kRingDepth < K) fetch(ring[r], k + kRingDepth);
                const bool act = k < nj;
                const int32_t l = l0 + nj - 1 - k;
                double lam_l = act ? c.lam : 0.0;
                if (kTrial && act) lam_l = __dadd_rn(lam_l, __dmul_rn(gamma, c.d));
                auto nbget = [&](int32_t a) {
                    double x = nb[0];
#pragma unroll
                    for (int u = 1; u < W; ++u) x = (a == u) ? nb[u] : x;
                    return x;
                };
                double vv[W];
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    vv[i] = 0.0;
                    if (i < c.w) {
                        const int32_t a = c.z[i], b = c.o[i];
                        const double c0 = a == dm::kTrue ? 0.0 : (a == dm::kFalse ? DM_INF : nbget(a));
                        const double c1 =
                            b == dm::kTrue ? lam_l : (b == dm::kFalse ? DM_INF : __dadd_rn(lam_l, nbget(b)));
                        const double v = (c0 <= c1) ? c0 : c1;
                        cur[i] = v;
                        vv[i] = v;
                    }
                }
                if (kStore && act) {
                    const int32_t vbase = s.lnl[l];
                    const int32_t wl = s.lnl[l + 1] - vbase;
#pragma unroll
                    for (int i = 0; i < W; ++i)
                        if (i < wl) B[vbase + i] = vv[i];
                }
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    const double t = nb[u];
                    nb[u] = cur[u];
                    cur[u] = t;
                }
                if (act && k == nj - 1) bounds[j] = nb[0];  // root layer: single node
            }
        }
    }
}

// the group's widest layer picks the narrowest unrolled body (bit-identical)
template <int W, bool kTrial, bool kStore>
__global__ void __launch_bounds__(kSweepThreads) sweep_backward_kernel(dm::SweepDev s, const double *__restrict__ lam,
                                                                        const double *__restrict__ d, double gamma,
                                                                        double *__restrict__ B,
                                                                        double *__restrict__ bounds,
                                                                        const double *__restrict__ ctl,
                                                                        const int32_t *__restrict__ bdd_inst) {
    extern __shared__ double sm[];
    if (kTrial && ctl && !bdd_inst) {  // device step search: ctl = dm_step_search state
        if (ctl[5] != 0.0) return;  // the search already stopped
        gamma = ctl[0];
    }
    if (!kTrial && ctl && *ctl == 0.0) return;  // gated refresh (dm_qn_move's verdict): nothing moved
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= s.groups) return;
    const int gw = s.grp_width ? s.grp_width[g] : W;
    __shared__ int32_t meta_w[kSweepWarps][kSweepMetaWin];
    __shared__ int64_t meta_s[kSweepWarps][kSweepMetaWin];
    const int wid = threadIdx.x >> 5;
    if (W > 2 && gw <= 2 && kSweepRing)
        sweep_backward_ring<2, kTrial, kStore>(s, lam, d, gamma, B, bounds, ctl, bdd_inst, g, meta_w[wid],
                                               meta_s[wid]);
    else if (W > 2 && gw <= 2)
        sweep_backward_body<2, W, kTrial, kStore>(s, lam, d, gamma, B, bounds, ctl, bdd_inst, g, sm);
    else if (W > 4 && gw <= 4)
        sweep_backward_body<4, W, kTrial, kStore>(s, lam, d, gamma, B, bounds, ctl, bdd_inst, g, sm);
    else
        sweep_backward_body<W, W, kTrial, kStore>(s, lam, d, gamma, B, bounds, ctl, bdd_inst, g, sm);
}

template <int W>
__global__ void __launch_bounds__(kSweepThreads) sweep_forward_kernel(dm::SweepDev s, const double *__restrict__ lam,
                                                                       double *__restrict__ F,
                                                                       double *__restrict__ bounds) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31;
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= s.groups) return;
    const int32_t j = s.grp_bdd[g * 32 + lane];
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = s.bdd_layer_lo[j];
        nj = s.bdd_layer_lo[j + 1] - l0;
    }
    const int32_t K = s.grp_npos[g];
    const int64_t p0 = s.grp_pos_lo[g];
    double *cur = sm + threadIdx.x;                      // distances from the root, position k
    double *nxt = sm + W * kSweepThreads + threadIdx.x;  // position k-1
    double tb = DM_INF;
    for (int32_t k = K - 1; k >= 0; --k) {
        if (k >= nj) continue;  // lane's diagram starts lower (lane-divergent, no barriers)
        const int32_t w = s.pos_width[p0 + k];
        const int64_t slot = s.pos_slot[p0 + k];
        const int32_t l = l0 + nj - 1 - k;
        const int32_t vbase = s.lnl[l];
        const int32_t wl = s.lnl[l + 1] - vbase;
        if (k == nj - 1) {  // root layer
            cur[0] = 0.0;
            for (int32_t i = 1; i < W; ++i) cur[i * kSweepThreads] = DM_INF;
        }
        for (int32_t i = 0; i < wl; ++i) F[vbase + i] = cur[i * kSweepThreads];
        const int32_t wn = k > 0 ? s.pos_width[p0 + k - 1] : 0;
        for (int32_t u = 0; u < wn; ++u) nxt[u * kSweepThreads] = DM_INF;
        const double lam_l = lam[l];
        for (int32_t i = 0; i < w; ++i) {
            const double fv = cur[i * kSweepThreads];
            if (fv == DM_INF) continue;
            const int32_t a = s.zl[(slot + i) * 32 + lane];
            const int32_t b = s.ol[(slot + i) * 32 + lane];
            if (a >= 0) {
                if (fv < nxt[a * kSweepThreads]) nxt[a * kSweepThreads] = fv;
            } else if (a == dm::kTrue) {
                if (fv < tb) tb = fv;
            }
            const double c = __dadd_rn(fv, lam_l);
            if (b >= 0) {
                if (c < nxt[b * kSweepThreads]) nxt[b * kSweepThreads] = c;
            } else if (b == dm::kTrue) {
                if (c < tb) tb = c;
            }
        }
        double *t = cur;
        cur = nxt;
        nxt = t;
    }
    if (j >= 0) bounds[j] = tb;
}

int fail(cudaError_t e, const char *what) {
    dm::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DM_ERR_CUDA;
}

template <int W>
int launch_backward(const dm::SweepDev &s, const double *lam, const double *d, double gamma, double *B,
                    double *bounds, cudaStream_t st, const double *ctl, const int32_t *bdd_inst = nullptr) {
    const int blocks = (int)((s.groups * 32 + kSweepThreads - 1) / kSweepThreads);
    const size_t smem = 2 * W * kSweepThreads * sizeof(double);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(sweep_backward_kernel<W, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep_backward_kernel<W, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep_backward_kernel<W, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep_backward_kernel<W, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (d && B)
        sweep_backward_kernel<W, true, true><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds, ctl, bdd_inst);
    else if (d)
        sweep_backward_kernel<W, true, false><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds, ctl, bdd_inst);
    else if (B)
        sweep_backward_kernel<W, false, true><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds, ctl, bdd_inst);
    else
        sweep_backward_kernel<W, false, false><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds, ctl, bdd_inst);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, "sweep_backward");
}

template <int W>
int launch_forward(const dm::SweepDev &s, const double *lam, double *F, double *bounds, cudaStream_t st) {
    const int blocks = (int)((s.groups * 32 + kSweepThreads - 1) / kSweepThreads);
    const size_t smem = 2 * W * kSweepThreads * sizeof(double);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(sweep_forward_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sweep_forward_kernel<W><<<blocks, kSweepThreads, smem, st>>>(s, lam, F, bounds);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, "sweep_forward");
}

}  // namespace

namespace dm {

int sweep_backward(const SweepDev &s, const double *lam, const double *d, double gamma, double *B, double *bounds,
                   void *stream, const double *ctl, const int32_t *bdd_inst) {
    if (s.groups == 0) return DM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (s.max_width <= 8) return launch_backward<8>(s, lam, d, gamma, B, bounds, st, ctl, bdd_inst);
    if (s.max_width <= 16) return launch_backward<16>(s, lam, d, gamma, B, bounds, st, ctl, bdd_inst);
    return launch_backward<32>(s, lam, d, gamma, B, bounds, st, ctl, bdd_inst);
}

int sweep_forward(const SweepDev &s, const double *lam, double *F, double *bounds, void *stream) {
    if (s.groups == 0) return DM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (s.max_width <= 8) return launch_forward<8>(s, lam, F, bounds, st);
    if (s.max_width <= 16) return launch_forward<16>(s, lam, F, bounds, st);
    return launch_forward<32>(s, lam, F, bounds, st);
}

}  // namespace dm

// ===========================================================================
// Chunked inner product (the dot order of the L-BFGS path):
//   dot(a, b) = pairwise(c_0, ..., c_{m-1}),  c_k = pairwise(a*b over chunk k)
// with chunks of 4096 elements (the last one shorter) and numpy's pairwise
// order inside each sum — restated by oracle/solver.py:_dot_chunked.
// Two launches: chunk_step_kernel takes one 128-thread block per FULL chunk —
// a perfect tree over 32 leaves of 128 elements (numpy's 8-accumulator leaf);
// thread (leaf o, pair p) owns accumulators 2p and 2p+1 of leaf o, read as
// 16-byte pairs, and the leaf and tree combines are shuffles — and writes the
// chunk total; chunk_finish_kernel (one block) handles the short tail chunk by
// replaying numpy's recursion from shared memory, then reduces the chunk
// totals the same way.  The stream orders the two, so no atomics or fences.
//
// The fused L-BFGS two-loop (qn.py:95-115) rides on the same pair of kernels:
// each step applies one update of the recursion to x and takes the next inner
// product on the updated values in the same pass.  Rounding and reduction
// order equal dm_axpy_dev / dm_scale_dev / dm_lbfgs_up / dm_dot, so the
// direction is bit-identical to the unfused sequence.
//   kDot   : no update, dot_out = dot(v, x)
//   kCopy  : x = u                                  (q = g.copy())
//   kFirst : a = rho*dot_in; x = x - a*u; alpha_out = a
//   kScale : like kFirst, then x = (sy0 / yy) * x   (last first-loop step)
//   kSecond: x = x + u * (alpha - rho*dot_in)
// then dot_out = chunked_dot(v, x) when v != nullptr.
// ===========================================================================
namespace {

constexpr int kChunk = 4096;
constexpr int kChunkThreads = 128;
constexpr int kFinishThreads = 1024;

enum { kDot = 0, kCopy = 1, kFirst = 2, kScale = 3, kSecond = 4 };

struct ChunkStep {
    double *x;
    const double *u, *v;
    double rho, sy0;
    const double *dot_in, *yy, *alpha_in;
    double *alpha_out, *dot_out;
};

struct StepCoef {
    double coef, r;
};

template <int kMode>
__device__ __forceinline__ StepCoef step_coef(const ChunkStep &a) {
    StepCoef c{0.0, 0.0};
    if (kMode == kFirst || kMode == kScale) c.coef = __dmul_rn(a.rho, a.dot_in[0]);
    if (kMode == kScale) c.r = __ddiv_rn(a.sy0, a.yy[0]);
    if (kMode == kSecond) c.coef = __dsub_rn(a.alpha_in[0], __dmul_rn(a.rho, a.dot_in[0]));
    return c;
}

template <int kMode>
__device__ __forceinline__ double step_update(const StepCoef &c, double xo, double uo) {
    if (kMode == kDot) return xo;
    if (kMode == kCopy) return uo;
    if (kMode == kSecond) return __dadd_rn(xo, __dmul_rn(uo, c.coef));
    const double xi = __dsub_rn(xo, __dmul_rn(c.coef, uo));
    return kMode == kScale ? __dmul_rn(c.r, xi) : xi;
}

#include "dm_reduce.cuh"

struct FinishPlans {
    SumPlan chunk, tail, totals;
};

// element pair (2p, 2p+1) of row i of leaf o, as a double2 index
__device__ __forceinline__ int pair_index(int i) { return (threadIdx.x >> 2) * 64 + (threadIdx.x & 3) + 4 * i; }

// Programmatic dependent launch inside the two-loop: a step's blocks start
// while the previous step's finishing block runs, pull their (constant)
// history vectors into L2, and only then wait for the previous grid.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// One FULL chunk (aligned, 4096 elements) by a 128-thread block: the
// update of x and the chunk total of v . x (a perfect tree over 32 leaves of
// 128, numpy's order); the total is valid on thread 0.
template <int kMode>
__device__ __forceinline__ double full_chunk(const StepCoef &c, double *x, const double *u, const double *v,
                                             int64_t off) {
    __shared__ double leaf_sm[32];
    double2 *x2 = reinterpret_cast<double2 *>(x + off);
    const double2 *u2 = reinterpret_cast<const double2 *>((kMode == kDot ? x : u) + off);
    const double2 *v2 = reinterpret_cast<const double2 *>((v ? v : x) + off);
    const bool dot = v != nullptr;
    double r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int i0 = 0; i0 < 16; i0 += 4) {
        double2 xv[4], uv[4], vv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int j = pair_index(i0 + k);
            if (kMode != kDot) uv[k] = u2[j];
            if (kMode != kCopy) xv[k] = x2[j];
            if (dot) vv[k] = v2[j];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            double2 xn;
            xn.x = step_update<kMode>(c, kMode == kCopy ? 0.0 : xv[k].x, kMode == kDot ? 0.0 : uv[k].x);
            xn.y = step_update<kMode>(c, kMode == kCopy ? 0.0 : xv[k].y, kMode == kDot ? 0.0 : uv[k].y);
            if (kMode != kDot) x2[pair_index(i0 + k)] = xn;
            if (dot) {
                const double p0 = __dmul_rn(vv[k].x, xn.x), p1 = __dmul_rn(vv[k].y, xn.y);
                r0 = (i0 + k == 0) ? p0 : __dadd_rn(r0, p0);
                r1 = (i0 + k == 0) ? p1 : __dadd_rn(r1, p1);
            }
        }
    }
    if (!dot) return 0.0;
    const unsigned m = 0xffffffffu;
    double r = __dadd_rn(r0, r1);
    r = __dadd_rn(r, __shfl_xor_sync(m, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(m, r, 2));
    __syncthreads();  // the previous chunk's leaf totals are consumed
    if ((threadIdx.x & 3) == 0) leaf_sm[threadIdx.x >> 2] = r;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = leaf_sm[threadIdx.x];
#pragma unroll
        for (int w = 1; w < 32; w <<= 1) t = __dadd_rn(t, __shfl_xor_sync(m, t, w));
        t = __dadd_rn(0.0, t);
    }
    return t;
}

template <int kMode>
__global__ void __launch_bounds__(kChunkThreads) chunk_step_kernel(ChunkStep a, double *__restrict__ partial) {
    pdl_launch_dependents();
    const int64_t off = (int64_t)blockIdx.x * kChunk;
    {
        // 32 KB per vector and block: two 128-byte lines per thread
        const char *pu = reinterpret_cast<const char *>((kMode == kDot ? a.x : a.u) + off);
        const char *pv = reinterpret_cast<const char *>((a.v ? a.v : a.x) + off);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int line = (threadIdx.x + k * kChunkThreads) * 128;
            if (kMode != kDot) asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + line));
            if (a.v) asm volatile("prefetch.global.L2 [%0];" ::"l"(pv + line));
        }
    }
    pdl_wait();  // the previous step's x and scalars are complete from here
    const StepCoef c = step_coef<kMode>(a);
    const double t = full_chunk<kMode>(c, a.x, a.u, a.v, off);
    if (a.v && threadIdx.x == 0) partial[blockIdx.x] = t;
}

// Tail chunk (update + its total) and the reduction of all chunk totals.
// `full` = 0 also covers unaligned vectors: every chunk is then done here,
// one at a time.
// totals == false (more than 4096 chunks): only the tail chunk; the chunk
// totals are then reduced by dm::pairwise_device (numpy's order for any length).
template <int kMode>
__global__ void __launch_bounds__(kFinishThreads) chunk_finish_kernel(ChunkStep a, int64_t n, int64_t full,
                                                                      double *__restrict__ partial,
                                                                      const __grid_constant__ FinishPlans plans,
                                                                      bool totals) {
    __shared__ double buf[kChunk];
    pdl_launch_dependents();
    pdl_wait();
    const StepCoef c = step_coef<kMode>(a);
    if ((kMode == kFirst || kMode == kScale) && threadIdx.x == 0 && a.alpha_out) a.alpha_out[0] = c.coef;
    const bool dot = a.v != nullptr;
    const int64_t nch = (n + kChunk - 1) / kChunk;
    constexpr int kPer = kChunk / kFinishThreads;  // elements per thread, loads issued together
    for (int64_t ch = full; ch < nch; ++ch) {
        const int64_t off = ch * kChunk;
        const int len = (int)((n - off) < kChunk ? (n - off) : kChunk);
        double xv[kPer], uv[kPer], vv[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int i = threadIdx.x + k * kFinishThreads;
            xv[k] = (kMode != kCopy && i < len) ? a.x[off + i] : 0.0;
            uv[k] = (kMode != kDot && i < len) ? a.u[off + i] : 0.0;
            vv[k] = (dot && i < len) ? a.v[off + i] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int i = threadIdx.x + k * kFinishThreads;
            if (i >= len) continue;
            const double xi = step_update<kMode>(c, xv[k], uv[k]);
            if (kMode != kDot) a.x[off + i] = xi;
            if (dot) buf[i] = __dmul_rn(vv[k], xi);
        }
        if (!dot) continue;
        __syncthreads();
        const double t = smem_pairwise(buf, len == kChunk ? plans.chunk : plans.tail);
        if (threadIdx.x == 0) partial[ch] = t;
        __syncthreads();
    }
    if (!dot || !totals) return;
    double pv[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = threadIdx.x + k * kFinishThreads;
        pv[k] = i < nch ? __ldcg(partial + i) : 0.0;  // includes this block's own tail total
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = threadIdx.x + k * kFinishThreads;
        if (i < nch) buf[i] = pv[k];
    }
    __syncthreads();
    const double t = smem_pairwise(buf, plans.totals);
    if (threadIdx.x == 0) a.dot_out[0] = t;
}

inline bool aligned16(const void *p) { return p == nullptr || ((uintptr_t)p & 15) == 0; }

template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, bool pdl,
                             Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// `pdl`: the previous launch on the stream is one of these kernels, which
// never write the step's u / v vectors, so they may be read before the wait.
template <int kMode>
cudaError_t chunk_step(const ChunkStep &a, int64_t n, double *partial, cudaStream_t st, bool pdl = false) {
    const bool vec = aligned16(a.x) && aligned16(a.u) && aligned16(a.v);
    const int64_t full = vec ? n / kChunk : 0;
    cudaError_t e;
    if (full > 0 &&
        (e = launch_maybe_pdl(chunk_step_kernel<kMode>, (unsigned)full, kChunkThreads, st, pdl, a, partial)))
        return e;
    const int64_t nch = (n + kChunk - 1) / kChunk;
    const bool two_level = nch > kChunk;
    FinishPlans plans;
    plans.chunk = make_sum_plan(kChunk);
    plans.tail = make_sum_plan((int)(n % kChunk));
    plans.totals = make_sum_plan(two_level ? 0 : (int)nch);
    if ((e = launch_maybe_pdl(chunk_finish_kernel<kMode>, 1, kFinishThreads, st, true, a, n, full, partial, plans,
                              !two_level)))
        return e;
    if (two_level && a.v && dm::pairwise_device(partial, nch, a.dot_out, st)) return cudaErrorUnknown;
    return cudaSuccess;
}

// Curvature pair of one iteration (qn.py:85-92, 245-252) in one pass:
// s = lam - lam_prev, y = g_prev - g, lam_prev = lam, and the chunk totals of
// s . y in the chunked-dot order (every chunk, tail included, here; the
// finishing block only reduces the totals).  Values equal dm_sub x2 + dm_dot.
__global__ void __launch_bounds__(kChunkThreads) curvature_pair_kernel(const double *__restrict__ lam,
                                                                       double *__restrict__ lam_prev,
                                                                       const double *__restrict__ g,
                                                                       const double *__restrict__ g_prev,
                                                                       double *__restrict__ s_out,
                                                                       double *__restrict__ y_out, int64_t n,
                                                                       bool vec, double *__restrict__ partial,
                                                                       const __grid_constant__ FinishPlans plans) {
    __shared__ double buf[kChunk];
    const int64_t off = (int64_t)blockIdx.x * kChunk;
    const int len = (int)((n - off) < kChunk ? (n - off) : kChunk);
    double t = 0.0;
    if (vec && len == kChunk) {
        const double2 *l2 = reinterpret_cast<const double2 *>(lam + off);
        double2 *p2 = reinterpret_cast<double2 *>(lam_prev + off);
        const double2 *g2 = reinterpret_cast<const double2 *>(g + off);
        const double2 *q2 = reinterpret_cast<const double2 *>(g_prev + off);
        double2 *s2 = reinterpret_cast<double2 *>(s_out + off);
        double2 *y2 = reinterpret_cast<double2 *>(y_out + off);
        double r0 = 0.0, r1 = 0.0;
#pragma unroll
        for (int i0 = 0; i0 < 16; i0 += 4) {
            double2 lv[4], pv[4], gv[4], qv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = pair_index(i0 + k);
                lv[k] = l2[j];
                pv[k] = p2[j];
                gv[k] = g2[j];
                qv[k] = q2[j];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = pair_index(i0 + k);
                const double2 sv = make_double2(__dsub_rn(lv[k].x, pv[k].x), __dsub_rn(lv[k].y, pv[k].y));
                const double2 yv = make_double2(__dsub_rn(qv[k].x, gv[k].x), __dsub_rn(qv[k].y, gv[k].y));
                s2[j] = sv;
                y2[j] = yv;
                p2[j] = lv[k];
                const double p0 = __dmul_rn(sv.x, yv.x), p1 = __dmul_rn(sv.y, yv.y);
                r0 = (i0 + k == 0) ? p0 : __dadd_rn(r0, p0);
                r1 = (i0 + k == 0) ? p1 : __dadd_rn(r1, p1);
            }
        }
        const unsigned m = 0xffffffffu;
        double r = __dadd_rn(r0, r1);
        r = __dadd_rn(r, __shfl_xor_sync(m, r, 1));
        r = __dadd_rn(r, __shfl_xor_sync(m, r, 2));
        if ((threadIdx.x & 3) == 0) buf[threadIdx.x >> 2] = r;
        __syncthreads();
        if (threadIdx.x < 32) {
            double x = buf[threadIdx.x];
#pragma unroll
            for (int w = 1; w < 32; w <<= 1) x = __dadd_rn(x, __shfl_xor_sync(m, x, w));
            t = __dadd_rn(0.0, x);
        }
    } else {
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            const double sv = __dsub_rn(lam[off + i], lam_prev[off + i]);
            const double yv = __dsub_rn(g_prev[off + i], g[off + i]);
            s_out[off + i] = sv;
            y_out[off + i] = yv;
            lam_prev[off + i] = lam[off + i];
            buf[i] = __dmul_rn(sv, yv);
        }
        __syncthreads();
        t = smem_pairwise(buf, len == kChunk ? plans.chunk : plans.tail);
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// ---------------------------------------------------------------------------
// The whole two-loop in ONE cooperative launch (dm_lbfgs_direction): each
// block owns chunks b, b+G, ... for every step, so x needs no exchange; per
// step the chunk totals meet in a double-buffered array, one grid barrier,
// and every block reduces them itself (the same totals plan), so the next
// step's coefficient is known grid-wide without a second barrier.  Every
// chunk is computed by full_chunk / the generic path exactly as the
// per-step kernels compute it: the direction is bit-identical (2m+2 barriers
// instead of 4m+4 dependent launches).
constexpr int kMaxTwoLoopPairs = 64;
struct TwoLoopArgs {
    const double *g;
    double *d;
    const double *s[kMaxTwoLoopPairs];
    const double *y[kMaxTwoLoopPairs];
    double rho[kMaxTwoLoopPairs];
    double sy0;
    int m;
    bool vec;
    int64_t n, nch;
    double *partial;  // [2][nch]
    double *slots;    // dot1[m], alpha[m], yy, dot2[m] (as the per-step path)
    unsigned *bar;    // {arrivals, generation, watchdog}
    SumPlan chunk, tail, totals;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// grid barrier (all blocks co-resident: cooperative launch); false when the
// watchdog fired (a block stopped arriving for 2 s) — the kernel then exits
__device__ bool two_loop_barrier(unsigned *bar, unsigned nblocks, unsigned &gen) {
    __shared__ int ok;
    __syncthreads();
    if (threadIdx.x == 0) {
        ok = 1;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            uint64_t t0 = 0;
            unsigned spins = 0;
            while (ld_acquire_u32(bar + 1) == gen) {
                if ((++spins & 255u) == 0) {
                    uint64_t now;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                    if (t0 == 0) t0 = now;
                    if (now - t0 > 2000000000ull || ld_acquire_u32(bar + 2)) {
                        atomicExch(bar + 2, 1u);
                        ok = 0;
                        break;
                    }
                }
            }
        }
        gen += 1;
        __threadfence();
    }
    __syncthreads();
    return ok != 0;
}

// chunk k of one step (update + total on thread 0); `buf`: 4096 doubles
template <int kMode>
__device__ __forceinline__ double two_loop_chunk(const TwoLoopArgs &a, const StepCoef &c, double *x, const double *u,
                                                 const double *v, int64_t k, double *buf) {
    const int64_t off = k * kChunk;
    const int len = (int)((a.n - off) < kChunk ? (a.n - off) : kChunk);
    if (a.vec && len == kChunk) return full_chunk<kMode>(c, x, u, v, off);
    __syncthreads();  // buf is free
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const double xo = kMode != kCopy ? x[off + i] : 0.0;
        const double uo = kMode != kDot ? u[off + i] : 0.0;
        const double xi = step_update<kMode>(c, xo, uo);
        if (kMode != kDot) x[off + i] = xi;
        if (v) buf[i] = __dmul_rn(v[off + i], xi);
    }
    if (!v) return 0.0;
    __syncthreads();
    return smem_pairwise(buf, len == kChunk ? a.chunk : a.tail);
}

template <int kMode>
__device__ __forceinline__ void two_loop_chunks(const TwoLoopArgs &a, const StepCoef &c, double *x, const double *u,
                                                const double *v, double *partial, double *buf) {
    for (int64_t k = blockIdx.x; k < a.nch; k += gridDim.x) {
        const double t = two_loop_chunk<kMode>(a, c, x, u, v, k, buf);
        if (v && threadIdx.x == 0) partial[k] = t;
    }
}

__global__ void __launch_bounds__(kChunkThreads) two_loop_kernel(const __grid_constant__ TwoLoopArgs a) {
    __shared__ double buf[kChunk];
    __shared__ double tot;                    // the last step's dot total
    __shared__ double al[kMaxTwoLoopPairs];  // the first loop's alphas
    const int m = a.m;
    double *dot1 = a.slots, *alpha = a.slots + m, *yy = a.slots + 2 * m, *dot2 = a.slots + 2 * m + 1;
    double yy_v = 0.0, dot_prev = 0.0;
    unsigned gen = 0;
    if (threadIdx.x == 0) gen = ld_acquire_u32(a.bar + 1);
    const int steps = 2 * m + 2;
    for (int t = 0; t < steps; ++t) {
        double *partial = a.partial + (t & 1) * a.nch;
        StepCoef c{0.0, 0.0};
        const double *v = nullptr;
        double *out = nullptr;
        if (t == 0) {  // yy = y0 . y0
            two_loop_chunks<kDot>(a, c, const_cast<double *>(a.y[0]), nullptr, a.y[0], partial, buf);
            out = yy;
            v = a.y[0];
        } else if (t == 1) {  // q = g, dot1[0] = s0 . q
            two_loop_chunks<kCopy>(a, c, a.d, a.g, a.s[0], partial, buf);
            out = dot1;
            v = a.s[0];
        } else if (t <= m) {  // first loop, i = t - 2
            const int i = t - 2;
            c.coef = __dmul_rn(a.rho[i], dot_prev);
            if (threadIdx.x == 0) al[i] = c.coef;
            if (blockIdx.x == 0 && threadIdx.x == 0) alpha[i] = c.coef;
            two_loop_chunks<kFirst>(a, c, a.d, a.y[i], a.s[i + 1], partial, buf);
            out = dot1 + i + 1;
            v = a.s[i + 1];
        } else if (t == m + 1) {  // last first-loop step with the scaling
            const int i = m - 1;
            c.coef = __dmul_rn(a.rho[i], dot_prev);
            c.r = __ddiv_rn(a.sy0, yy_v);
            if (threadIdx.x == 0) al[i] = c.coef;
            if (blockIdx.x == 0 && threadIdx.x == 0) alpha[i] = c.coef;
            two_loop_chunks<kScale>(a, c, a.d, a.y[i], a.y[m - 1], partial, buf);
            out = dot2;
            v = a.y[m - 1];
        } else {  // second loop, k = t - m - 2, i = m - 1 - k
            const int k = t - m - 2, i = m - 1 - k;
            c.coef = __dsub_rn(al[i], __dmul_rn(a.rho[i], dot_prev));
            v = i > 0 ? a.y[i - 1] : nullptr;
            two_loop_chunks<kSecond>(a, c, a.d, a.s[i], v, partial, buf);
            out = v ? dot2 + k + 1 : nullptr;
        }
        if (!v) break;  // the last step has no inner product
        if (!two_loop_barrier(a.bar, gridDim.x, gen)) return;
        // every block reduces the chunk totals itself (numpy's order)
        for (int64_t i = threadIdx.x; i < a.nch; i += blockDim.x) buf[i] = __ldcg(partial + i);
        __syncthreads();
        const double total = smem_pairwise(buf, a.totals);
        if (threadIdx.x == 0) {
            tot = total;
            if (blockIdx.x == 0) *out = total;
        }
        __syncthreads();
        dot_prev = tot;
        if (t == 0) yy_v = tot;
    }
}

}  // namespace

namespace dm {

int curvature_pair(const double *lam, double *lam_prev, const double *g, const double *g_prev, double *s,
                   double *y, int64_t n, double *partial, double *sy, void *stream) {
    const int64_t nch = (n + kChunk - 1) / kChunk;
    if (n <= 0 || nch >= INT32_MAX) return DM_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    const bool vec = aligned16(lam) && aligned16(lam_prev) && aligned16(g) && aligned16(g_prev) && aligned16(s) &&
                     aligned16(y);
    FinishPlans plans;
    plans.chunk = make_sum_plan(kChunk);
    plans.tail = make_sum_plan((int)(n % kChunk));
    plans.totals = make_sum_plan(nch > kChunk ? 0 : (int)nch);
    curvature_pair_kernel<<<(unsigned)nch, kChunkThreads, 0, st>>>(lam, lam_prev, g, g_prev, s, y, n, vec, partial,
                                                                   plans);
    cudaError_t e = cudaGetLastError();
    if (e) return fail(e, "curvature_pair");
    // totals only: every chunk is done (`full` = nch), so the finishing block just reduces them
    if (nch > kChunk) return dm::pairwise_device(partial, nch, sy, st);
    ChunkStep a{};
    a.x = s;
    a.v = y;
    a.dot_out = sy;
    e = launch_maybe_pdl(chunk_finish_kernel<kDot>, 1, kFinishThreads, st, true, a, n, nch, partial, plans, true);
    return e == cudaSuccess ? DM_OK : fail(e, "curvature_pair finish");
}

// the cooperative two-loop: grid size for this device (0: unavailable)
static int two_loop_grid(int64_t nch) {
    static int per_sm = -1, sms = 0;
    if (per_sm < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int b = 0;
        if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, two_loop_kernel, kChunkThreads, 0)) b = 0;
        per_sm = b;
    }
    // one chunk per block: with more chunks than co-resident blocks every
    // block would loop over several and reduce all totals per step (C2,
    // 2,296 chunks on 592 blocks: 1.34 -> 1.48 ms), so the per-step
    // launches stay (C4, 320 chunks: 0.33 -> 0.25 ms)
    const int64_t cap = (int64_t)per_sm * sms;
    return nch <= cap ? (int)nch : 0;
}

static bool two_loop_persistent() {
    static const int v = [] {
        const char *e = std::getenv("DM_TWO_LOOP_PERSIST");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0;
}

int lbfgs_two_loop(const double *g, const double *const *s, const double *const *y, const double *rho,
                   const double *sy, int m, int64_t n, double *d, double *slots, double *partial, void *stream,
                   unsigned *bar) {
    const int64_t nch = (n + kChunk - 1) / kChunk;
    if (n <= 0 || nch >= INT32_MAX || m < 1) return DM_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    int grid = 0;
    if (bar && m <= kMaxTwoLoopPairs && nch <= kChunk && two_loop_persistent() && (grid = two_loop_grid(nch)) > 0) {
        TwoLoopArgs a{};
        a.g = g;
        a.d = d;
        for (int i = 0; i < m; ++i) {
            a.s[i] = s[i];
            a.y[i] = y[i];
            a.rho[i] = rho[i];
        }
        a.sy0 = sy[0];
        a.m = m;
        a.vec = aligned16(g) && aligned16(d);
        for (int i = 0; i < m; ++i) a.vec = a.vec && aligned16(s[i]) && aligned16(y[i]);
        a.n = n;
        a.nch = nch;
        a.partial = partial;
        a.slots = slots;
        a.bar = bar;
        a.chunk = make_sum_plan(kChunk);
        a.tail = make_sum_plan((int)(n % kChunk));
        a.totals = make_sum_plan((int)nch);
        void *args[] = {(void *)&a};
        const cudaError_t e = cudaLaunchCooperativeKernel((const void *)two_loop_kernel, dim3(grid),
                                                          dim3(kChunkThreads), args, 0, st);
        if (e == cudaSuccess) return DM_OK;
        // the grid no longer fits (another context holds part of the device):
        // the per-step launches below compute the same bits
        if (e != cudaErrorCooperativeLaunchTooLarge) return fail(e, "two_loop (cooperative)");
        (void)cudaGetLastError();
    }
    // slots: [0, m) first-loop dots, [m, 2m) alphas, 2m = y0.y0, [2m+1, 3m+1) second-loop dots
    double *dot1 = slots, *alpha = slots + m, *yy = slots + 2 * m, *dot2 = slots + 2 * m + 1;
    if (int rc = dm::chunk_dot(y[0], y[0], n, partial, yy, stream)) return rc;
    cudaError_t e;
    ChunkStep a{};
    a.x = d;
    a.u = g;
    a.v = s[0];
    a.dot_out = dot1;
    if ((e = chunk_step<kCopy>(a, n, partial, st, true))) return fail(e, "two_loop copy");
    for (int i = 0; i < m; ++i) {
        a = ChunkStep{};
        a.x = d;
        a.u = y[i];
        a.rho = rho[i];
        a.dot_in = dot1 + i;
        a.alpha_out = alpha + i;
        if (i + 1 < m) {
            a.v = s[i + 1];
            a.dot_out = dot1 + i + 1;
            e = chunk_step<kFirst>(a, n, partial, st, true);
        } else {  // last step of the first loop carries the scaling and starts the second loop
            a.sy0 = sy[0];
            a.yy = yy;
            a.v = y[m - 1];
            a.dot_out = dot2;
            e = chunk_step<kScale>(a, n, partial, st, true);
        }
        if (e) return fail(e, "two_loop first");
    }
    for (int k = 0; k < m; ++k) {
        const int i = m - 1 - k;
        a = ChunkStep{};
        a.x = d;
        a.u = s[i];
        a.rho = rho[i];
        a.dot_in = dot2 + k;
        a.alpha_in = alpha + i;
        if (i > 0) {
            a.v = y[i - 1];
            a.dot_out = dot2 + k + 1;
        }
        if ((e = chunk_step<kSecond>(a, n, partial, st, true))) return fail(e, "two_loop second");
    }
    return DM_OK;
}

int chunk_dot(const double *a, const double *b, int64_t n, double *partial, double *out, void *stream) {
    const int64_t nch = (n + kChunk - 1) / kChunk;
    if (n <= 0 || nch >= INT32_MAX || !b) return DM_ERR_UNSUPPORTED;
    ChunkStep st{};
    st.x = const_cast<double *>(a);  // read only in kDot mode
    st.v = b;
    st.dot_out = out;
    cudaError_t e = chunk_step<kDot>(st, n, partial, (cudaStream_t)stream);
    return e == cudaSuccess ? DM_OK : fail(e, "chunk_dot");
}

}  // namespace dm
