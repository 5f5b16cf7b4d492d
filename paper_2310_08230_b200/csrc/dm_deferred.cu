// Deferred (throughput) min-marginal averaging schedule — the parallel MMA of
// FastDOG (Abbas & Swoboda 2022) that the paper runs on its GPU
// ("for parallel min-marginal averaging we use the dual
// optimisation algorithm of [FastDOG]"); the reference package replaced it by
// a sequential Gauss-Seidel sweep (kernels.py:162-362).
//
// Within one pass every diagram is independent: at layer l of diagram j the
// pass computes the copy's min-marginal difference M with the distances of
// its own diagram only (the opposite-direction table is still exact there,
// since no later layer of j has changed in this pass), moves the dual by
// -omega*M and keeps omega*M in escrow (mbar[l]); the copy also receives the
// average escrow its variable's copies left in the PREVIOUS pass (avg[l]).
// So the sum over a variable's copies of (lam + mbar) stays equal to its
// cost.  dfr_average_kernel turns one pass's escrow into the next pass's
// per-copy average (a segmented reduction over the variable CSR), and a pass
// without the min-marginal step (mbar == null) redistributes the last escrow
// and rebuilds the table: after it the duals are feasible again.
//
//   lam' = (lam - omega*M) + avg      copies with finite m0, m1 (mbar = omega*M)
//   lam' =  lam + avg                 otherwise                (mbar = +inf)
//   avg  = (sum of finite mbar over the variable's copies, in copy order)
//          / (their count), 0.0 for non-finite copies
//
// M is taken on the duals BEFORE the deferred average is added (FastDOG's
// order).  Arithmetic is binary64 with explicit roundings (-fmad=false), the
// per-diagram order is the reference's (m0/m1 as kernels.py:207-228,
// distances as kernels.py:104-120 / 142-159), so oracle/ckernels.c
// (oracle_dfr_*) reproduces every output bit for bit.
//
// Layout: the interleaved sweep layout (dm_layout.cpp) — 32 diagrams of
// similar shape per warp, one lane per diagram, node slot (k, i) of lane t at
// element (pos_slot[k] + i) * 32 + t.  The passes keep BOTH distance tables
// in that layout (F_il / B_il), so every table access of a warp is one
// 128-byte row per node slot; only lam / avg / mbar are per-lane gathers
// (consecutive layers of one diagram, so a lane walks its own cache lines).
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "dm_internal.h"
#include "dm_rows.cuh"

#define DM_INF __longlong_as_double(0x7ff0000000000000LL)

namespace {

constexpr int kThreads = 128;

struct DfrArgs {
    dm::SweepDev s;
    double omega;
    double *lam;
    const double *avg;   // null: no deferred average to add
    const double *in;    // opposite-direction table (interleaved), null without the MM step
    double *out;         // this direction's table (interleaved)
    double *mbar;        // escrow out (null: no min-marginal step)
    double *bounds;      // per-diagram optimum of the resulting duals
    uint64_t *dec;       // backward only: argmin decisions, one word per layer (W <= 8)
};

__device__ __forceinline__ double c_zero(int32_t a, double fv, const double *nb) {
    return a == dm::kTrue ? fv : (a == dm::kFalse ? DM_INF : __dadd_rn(fv, nb[a * kThreads]));
}
__device__ __forceinline__ double c_one(int32_t b, double fl, const double *nb) {  // fl = fv + lam
    return b == dm::kTrue ? fl : (b == dm::kFalse ? DM_INF : __dadd_rn(fl, nb[b * kThreads]));
}

template <int W, bool kReg, int S>
__device__ __forceinline__ double c_zero(int32_t a, double fv, const Row<W, kReg, S> &nb) {
    return a == dm::kTrue ? fv : (a == dm::kFalse ? DM_INF : __dadd_rn(fv, nb.get(a)));
}
template <int W, bool kReg, int S>
__device__ __forceinline__ double c_one(int32_t b, double fl, const Row<W, kReg, S> &nb) {  // fl = fv + lam
    return b == dm::kTrue ? fl : (b == dm::kFalse ? DM_INF : __dadd_rn(fl, nb.get(b)));
}

// the dual update of one copy (see the header); returns lam'
template <bool kAvg>
__device__ __forceinline__ double dfr_update(double lam_l, double a_l, double m0, double m1, double omega,
                                             double *mbar_slot) {
    if (m0 < DM_INF && m1 < DM_INF) {
        const double wm = __dmul_rn(omega, __dsub_rn(m1, m0));
        lam_l = __dsub_rn(lam_l, wm);
        if (kAvg) lam_l = __dadd_rn(lam_l, a_l);
        *mbar_slot = wm;
    } else {
        if (kAvg) lam_l = __dadd_rn(lam_l, a_l);
        *mbar_slot = DM_INF;
    }
    return lam_l;
}

// Group metadata (width and first slot of every position) staged per warp
// in shared memory, a window of kMetaWin positions at a time: the slot
// addresses of the next positions then need no dependent global load, and
// the passes can warm L2 with the rows kAhead positions ahead of the
// register double buffer (a lane per 128-byte row: arcs, opposite table,
// plus each lane's own dual entries).
constexpr int kMetaWin = 128;
constexpr int kAhead = 3;
#ifndef DM_DFR_WARM
#define DM_DFR_WARM 0
#endif
constexpr bool kWarm = DM_DFR_WARM != 0;  // L2 warm-up of later positions (A/B: slower in the MM passes)
#ifndef DM_DFR_WARM_NARROW
#define DM_DFR_WARM_NARROW 0
#endif
// (A/B at C4: warming L2 in the narrow bodies only is slower too, 141 vs 118 us)
constexpr int kWarmNarrow = DM_DFR_WARM_NARROW;
constexpr int kWarps = kThreads / 32;

struct Meta {
    int32_t *w;
    int64_t *slot;
    int32_t lo;  // first position held
};

__device__ __forceinline__ void meta_window(Meta &m, const dm::SweepDev &s, int64_t p0, int32_t K, int32_t lo,
                                            int lane) {
    __syncwarp();
    for (int i = lane; i < kMetaWin; i += 32) {
        const int32_t k = lo + i;
        if (k < K) {
            m.w[i] = s.pos_width[p0 + k];
            m.slot[i] = s.pos_slot[p0 + k];
        }
    }
    __syncwarp();
    m.lo = lo;
}

__device__ __forceinline__ void l2_prefetch(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// warm L2 with position k's arc rows (lanes 0-7: zero arcs, 8-15: one arcs)
// and, when tab != null, the table rows of position kt (lanes 16-31, two
// lines per row)
template <int W>
__device__ __forceinline__ void warm_rows(const dm::SweepDev &s, int lane, int32_t w, int64_t slot, const double *tab,
                                          int32_t wt, int64_t slot_t) {
    if (lane < 8) {
        if (lane < w) l2_prefetch(s.zl + (slot + lane) * 32);
    } else if (lane < 16) {
        if (lane - 8 < w) l2_prefetch(s.ol + (slot + lane - 8) * 32);
    } else if (tab) {
        const int q = lane - 16;  // row q / 2, half q % 2
        if ((q >> 1) < wt) l2_prefetch(tab + (slot_t + (q >> 1)) * 32 + (q & 1) * 16);
    }
}

// dfr_update with the escrow returned instead of stored
template <bool kAvg>
__device__ __forceinline__ double dfr_update_v(double lam_l, double a_l, double m0, double m1, double omega,
                                               double &mbar_out) {
    return dfr_update<kAvg>(lam_l, a_l, m0, m1, omega, &mbar_out);
}

// Backward direction: positions k = 0 (every lane's last layer) .. K-1.
// W: node slots the loops cover (>= the group's widest layer), WS: the slot
// stride of the shared distance rows (the launch's width).
template <int W, int WS, bool kMM, bool kAvg, bool kDec>
__device__ __forceinline__ void dfr_backward_body(const DfrArgs &a, int64_t g, double *sm, int32_t *meta_w,
                                                  int64_t *meta_s) {
    const dm::SweepDev &s = a.s;
    double *__restrict__ lamp = a.lam;
    const double *__restrict__ avgp = a.avg;
    const double *__restrict__ inp = a.in;
    double *__restrict__ outp = a.out;
    double *__restrict__ mbarp = a.mbar;
    double *__restrict__ boundsp = a.bounds;
    uint64_t *__restrict__ decp = a.dec;
    const int lane = threadIdx.x & 31;
    const int32_t j = s.grp_bdd[g * 32 + lane];
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = s.bdd_layer_lo[j];
        nj = s.bdd_layer_lo[j + 1] - l0;
    }
    const int32_t K = s.grp_npos[g];
    const int64_t p0 = s.grp_pos_lo[g];
    constexpr bool kReg = W <= kRegRowsDfr;
    Row<W, kReg, kThreads> nb, cur;  // distances of position k-1 (next layer) and of position k
    if constexpr (kReg) {
#pragma unroll
        for (int u = 0; u < W; ++u) nb.put(u, DM_INF), cur.put(u, DM_INF);
    } else {
        nb.p = sm + threadIdx.x;
        cur.p = sm + WS * kThreads + threadIdx.x;
    }
    // register double buffer: position k+1's arcs, F row and duals load while k computes
    int32_t za[W], oa[W];
    double fa[W];
    double lam_n = 0.0, avg_n = 0.0;
    int32_t w_n = 0;
    int64_t slot_n = 0;
    Meta meta{meta_w, meta_s, 0};
    meta_window(meta, s, p0, K, 0, lane);
    auto fetch = [&](int32_t k) {
        w_n = meta.w[k - meta.lo];
        slot_n = meta.slot[k - meta.lo];
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < w_n) {
                const int64_t e = (slot_n + i) * 32 + lane;
                za[i] = s.zl[e];
                oa[i] = s.ol[e];
                if (kMM) fa[i] = inp[e];
            }
        if (k < nj) {
            const int32_t l = l0 + nj - 1 - k;
            lam_n = lamp[l];
            if (kAvg) avg_n = avgp[l];
        }
    };
    if (K > 0) fetch(0);
    for (int32_t k = 0; k < K; ++k) {
        // positions k .. k + 1 + kAhead must be in the metadata window (uniform in the warp)
        if (k + 1 + kAhead >= meta.lo + kMetaWin && meta.lo + kMetaWin < K) meta_window(meta, s, p0, K, k, lane);
        {
            const int32_t kp = k + 1 + kAhead;
            if ((kWarm || W <= kWarmNarrow) && kp < K) {
                const int32_t wp = meta.w[kp - meta.lo];
                const int64_t sp = meta.slot[kp - meta.lo];
                warm_rows<W>(s, lane, wp, sp, kMM ? inp : nullptr, wp, sp);
                if (kp < nj) {
                    l2_prefetch(lamp + (l0 + nj - 1 - kp));
                    if (kAvg) l2_prefetch(avgp + (l0 + nj - 1 - kp));
                }
            }
        }
        const int32_t w = w_n;
        const int64_t slot = slot_n;
        int32_t z[W], o[W];
        double f[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            z[i] = za[i];
            o[i] = oa[i];
            if (kMM) f[i] = fa[i];
        }
        const bool act = k < nj;
        const int32_t l = l0 + nj - 1 - k;
        double lam_l = act ? lam_n : 0.0;
        const double a_l = avg_n;
        if (k + 1 < K) fetch(k + 1);
        if (act && (kMM || kAvg)) {
            if (kMM) {
                double m0 = DM_INF, m1 = DM_INF;
#pragma unroll
                for (int i = 0; i < W; ++i)
                    if (i < w) {
                        const double c0 = c_zero(z[i], f[i], nb);
                        const double c1 = c_one(o[i], __dadd_rn(f[i], lam_l), nb);
                        if (c0 < m0) m0 = c0;
                        if (c1 < m1) m1 = c1;
                    }
                lam_l = dfr_update<kAvg>(lam_l, a_l, m0, m1, a.omega, mbarp + l);
            } else {
                lam_l = __dadd_rn(lam_l, a_l);
            }
            lamp[l] = lam_l;
        }
        uint64_t word = 0;
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < w) {
                const int32_t za_ = z[i], ob = o[i];
                const double c0 = za_ == dm::kTrue ? 0.0 : (za_ == dm::kFalse ? DM_INF : nb.get(za_));
                const double c1 =
                    ob == dm::kTrue ? lam_l : (ob == dm::kFalse ? DM_INF : __dadd_rn(lam_l, nb.get(ob)));
                const bool zero_wins = c0 <= c1;
                const double v = zero_wins ? c0 : c1;
                cur.put(i, v);
                outp[(slot + i) * 32 + lane] = v;
                if (kDec && W <= 8) {
                    const int32_t t = zero_wins ? za_ : ob;
                    word |= (uint64_t)((((t >= 0) ? t : 0) << 1) | (zero_wins ? 0 : 1)) << (8 * i);
                }
            }
        if (kDec && W <= 8 && act) decp[l] = word;
        swap_rows(nb, cur);
        if (act && k == nj - 1) boundsp[j] = nb.at(0);  // root layer: single node
    }
}

// The group's widest layer picks the narrowest unrolled body (bit-identical:
// slots past a position's width are never touched): the long chains of a
// split instance are two nodes wide, and a warp walking them runs a quarter
// of the W = 8 instructions per position.
template <int W, bool kMM, bool kAvg, bool kDec>
__global__ void __launch_bounds__(kThreads) dfr_backward_kernel(DfrArgs a) {
    extern __shared__ double sm[];
    __shared__ int32_t meta_w[kWarps][kMetaWin];
    __shared__ int64_t meta_s[kWarps][kMetaWin];
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= a.s.groups) return;
    const int wid = threadIdx.x >> 5;
    const int gw = a.s.grp_width ? a.s.grp_width[g] : W;
    if (W > 2 && gw <= 2)
        dfr_backward_body<2, W, kMM, kAvg, kDec>(a, g, sm, meta_w[wid], meta_s[wid]);
    else if (W > 4 && gw <= 4)
        dfr_backward_body<4, W, kMM, kAvg, kDec>(a, g, sm, meta_w[wid], meta_s[wid]);
    else
        dfr_backward_body<W, W, kMM, kAvg, kDec>(a, g, sm, meta_w[wid], meta_s[wid]);
}

// Forward direction: positions k = K-1 .. 0; lanes whose diagram is shorter
// than the group's longest idle until their root position.
template <int W, int WS, bool kMM, bool kAvg>
__device__ __forceinline__ void dfr_forward_body(const DfrArgs &a, int64_t g, double *sm, int32_t *meta_w,
                                                 int64_t *meta_s) {
    const dm::SweepDev &s = a.s;
    double *__restrict__ lamp = a.lam;
    const double *__restrict__ avgp = a.avg;
    const double *__restrict__ inp = a.in;
    double *__restrict__ outp = a.out;
    double *__restrict__ mbarp = a.mbar;
    double *__restrict__ boundsp = a.bounds;
    uint64_t *__restrict__ decp = a.dec;
    const int lane = threadIdx.x & 31;
    const int32_t j = s.grp_bdd[g * 32 + lane];
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = s.bdd_layer_lo[j];
        nj = s.bdd_layer_lo[j + 1] - l0;
    }
    const int32_t K = s.grp_npos[g];
    const int64_t p0 = s.grp_pos_lo[g];
    constexpr bool kReg = W <= kRegRowsDfr;
    // distances from the root at position k and k-1, B of position k-1 (kMM)
    Row<W, kReg, kThreads> cur, nxt, bn;
    if constexpr (kReg) {
#pragma unroll
        for (int u = 0; u < W; ++u) cur.put(u, DM_INF), nxt.put(u, DM_INF), bn.put(u, DM_INF);
    } else {
        cur.p = sm + threadIdx.x;
        nxt.p = sm + WS * kThreads + threadIdx.x;
        bn.p = sm + 2 * WS * kThreads + threadIdx.x;
    }
    double tb = DM_INF;
    // register double buffer for position k-1
    int32_t za[W], oa[W];
    double ba[W];
    double lam_n = 0.0, avg_n = 0.0;
    int32_t w_n = 0, wb_n = 0;
    int64_t slot_n = 0;
    Meta meta{meta_w, meta_s, 0};
    meta_window(meta, s, p0, K, K > kMetaWin ? K - kMetaWin : 0, lane);
    auto fetch = [&](int32_t k) {  // k < nj
        w_n = meta.w[k - meta.lo];
        slot_n = meta.slot[k - meta.lo];
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < w_n) {
                const int64_t e = (slot_n + i) * 32 + lane;
                za[i] = s.zl[e];
                oa[i] = s.ol[e];
            }
        const int32_t l = l0 + nj - 1 - k;
        lam_n = lamp[l];
        if (kAvg) avg_n = avgp[l];
        if (kMM) {
            wb_n = k > 0 ? meta.w[k - 1 - meta.lo] : 0;
            const int64_t sb = k > 0 ? meta.slot[k - 1 - meta.lo] : 0;
#pragma unroll
            for (int u = 0; u < W; ++u)
                if (u < wb_n) ba[u] = inp[(sb + u) * 32 + lane];
        }
    };
    // positions k - 2 - kAhead .. k must be in the window (uniform in the warp)
    auto window_for = [&](int32_t k) {
        if (k - 2 - kAhead < meta.lo && meta.lo > 0) {
            const int32_t lo = k + 1 > kMetaWin ? k + 1 - kMetaWin : 0;
            meta_window(meta, s, p0, K, lo, lane);
        }
    };
    if (K > 0) window_for(K - 1);
    if (nj > 0) fetch(nj - 1);
    for (int32_t k = K - 1; k >= 0; --k) {
        window_for(k);
        {
            const int32_t kp = k - 1 - kAhead;  // warm L2 for position kp (and the table rows of kp - 1)
            if ((kWarm || W <= kWarmNarrow) && kp >= 0 && kp < nj) {
                const int32_t wp = meta.w[kp - meta.lo];
                const int64_t sp = meta.slot[kp - meta.lo];
                const int32_t wt = kp > 0 ? meta.w[kp - 1 - meta.lo] : 0;
                const int64_t st = kp > 0 ? meta.slot[kp - 1 - meta.lo] : 0;
                warm_rows<W>(s, lane, wp, sp, kMM ? inp : nullptr, wt, st);
                l2_prefetch(lamp + (l0 + nj - 1 - kp));
                if (kAvg) l2_prefetch(avgp + (l0 + nj - 1 - kp));
            }
        }
        if (k >= nj) continue;
        const int32_t w = w_n;
        const int64_t slot = slot_n;
        const int32_t wn = k > 0 ? meta.w[k - 1 - meta.lo] : 0;
        int32_t z[W], o[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            z[i] = za[i];
            o[i] = oa[i];
        }
        if (kMM) {
#pragma unroll
            for (int u = 0; u < W; ++u)
                if (u < wb_n) bn.put(u, ba[u]);
        }
        double lam_l = lam_n;
        const double a_l = avg_n;
        if (k > 0) fetch(k - 1);
        const int32_t l = l0 + nj - 1 - k;
        if (k == nj - 1) {  // root layer: F[root] = 0 (kernels.py:187-193)
            cur.put(0, 0.0);
#pragma unroll
            for (int i = 1; i < W; ++i) cur.put(i, DM_INF);
        }
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < w) outp[(slot + i) * 32 + lane] = cur.at(i);
        if (kMM) {
            double m0 = DM_INF, m1 = DM_INF;
#pragma unroll
            for (int i = 0; i < W; ++i)
                if (i < w) {
                    const double fv = cur.at(i);
                    const double c0 = c_zero(z[i], fv, bn);
                    const double c1 = c_one(o[i], __dadd_rn(fv, lam_l), bn);
                    if (c0 < m0) m0 = c0;
                    if (c1 < m1) m1 = c1;
                }
            lam_l = dfr_update<kAvg>(lam_l, a_l, m0, m1, a.omega, mbarp + l);
            lamp[l] = lam_l;
        } else if (kAvg) {
            lam_l = __dadd_rn(lam_l, a_l);
            lamp[l] = lam_l;
        }
        // push this layer's distances into the next one (kernels.py:241-269)
#pragma unroll
        for (int u = 0; u < W; ++u)
            if (u < wn) nxt.put(u, DM_INF);
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < w) {
                const double fv = cur.at(i);
                if (fv == DM_INF) continue;
                const int32_t za_ = z[i], ob = o[i];
                if (za_ >= 0) {
                    if (fv < nxt.get(za_)) nxt.put_dyn(za_, fv);
                } else if (za_ == dm::kTrue) {
                    if (fv < tb) tb = fv;
                }
                const double c = __dadd_rn(fv, lam_l);
                if (ob >= 0) {
                    if (c < nxt.get(ob)) nxt.put_dyn(ob, c);
                } else if (ob == dm::kTrue) {
                    if (c < tb) tb = c;
                }
            }
        swap_rows(cur, nxt);
    }
    if (j >= 0) boundsp[j] = tb;
}

template <int W, bool kMM, bool kAvg>
__global__ void __launch_bounds__(kThreads) dfr_forward_kernel(DfrArgs a) {
    extern __shared__ double sm[];
    __shared__ int32_t meta_w[kWarps][kMetaWin];
    __shared__ int64_t meta_s[kWarps][kMetaWin];
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= a.s.groups) return;
    const int wid = threadIdx.x >> 5;
    const int gw = a.s.grp_width ? a.s.grp_width[g] : W;
    if (W > 2 && gw <= 2)
        dfr_forward_body<2, W, kMM, kAvg>(a, g, sm, meta_w[wid], meta_s[wid]);
    else if (W > 4 && gw <= 4)
        dfr_forward_body<4, W, kMM, kAvg>(a, g, sm, meta_w[wid], meta_s[wid]);
    else
        dfr_forward_body<W, W, kMM, kAvg>(a, g, sm, meta_w[wid], meta_s[wid]);
}

// ---------------------------------------------------------------------------
// Node-parallel passes (layers of <= 8 nodes with single-source publish
// descriptors — every product-space instance): 8 lanes per diagram, lane q
// holds node q of the diagram's current layer, 4 diagrams per warp (taken in
// the sweep layout's longest-first order).  A position's work is spread over
// the layer's nodes: next-layer distances reach the arcs by shuffles, m0/m1
// are leftmost-minimum trees over the 8 lanes (the same value a sequential
// strict-< scan keeps, ties included), the forward publish reads the
// per-layer source descriptors (dm_plan.cu relax_kernel) and takes, per
// target, the leftmost minimum of its candidates in the reference's scan
// order.  Tables in the reference node order (FlatBdds F / B).  Bit-identical
// to the lane-per-diagram kernels and the oracle.
struct NpArgs {
    const int32_t *order;  // diagrams, longest first (sweep layout lanes; -1 = padding)
    int64_t entries;
    const int32_t *bdd_layer_lo, *lnl, *zero_t, *one_t;
    const uint64_t *relax;
    double omega;
    double *lam;
    const double *avg;
    const double *in;  // opposite-direction table (node order)
    double *out;       // this direction's table (node order)
    double *mbar, *bounds;
    uint64_t *dec;
};

constexpr int kNpThreads = 256;
constexpr unsigned kFullMask = 0xffffffffu;

// leftmost minimum over the 8 lanes of a group (combine(left, right) keeps
// left unless right < left): equals a sequential strict-< scan from +inf
__device__ __forceinline__ double lmin8(double v, int q) {
#pragma unroll
    for (int s = 1; s < 8; s <<= 1) {
        const double o = __shfl_xor_sync(kFullMask, v, s);
        v = (q & s) ? ((v < o) ? v : o) : ((o < v) ? o : v);
    }
    return v;
}

template <bool kMM, bool kAvg, bool kDec>
__global__ void __launch_bounds__(kNpThreads) dfr_np_backward_kernel(NpArgs a) {
    const int lane = threadIdx.x & 31, q = lane & 7, gb = lane & ~7;
    const int64_t e = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4 + (lane >> 3);
    const int32_t j = e < a.entries ? a.order[e] : -1;
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = a.bdd_layer_lo[j];
        nj = a.bdd_layer_lo[j + 1] - l0;
    }
    int32_t K = nj;
    K = max(K, __shfl_xor_sync(kFullMask, K, 8));
    K = max(K, __shfl_xor_sync(kFullMask, K, 16));
    if (K == 0) return;
    // prefetch: node range of position k+1, and the rows of position k
    int32_t base_n = 0, end_n = 0;  // [lnl[l], lnl[l+1]) of the next position
    auto range = [&](int32_t k, int32_t &b, int32_t &en) {
        if (k < nj) {
            const int32_t l = l0 + nj - 1 - k;
            b = a.lnl[l];
            en = a.lnl[l + 1];
        } else {
            b = en = 0;
        }
    };
    int32_t z_n = dm::kFalse, o_n = dm::kFalse;
    double f_n = 0.0, lam_n = 0.0, avg_n = 0.0;
    int32_t base_c = 0, end_c = 0;
    auto rows = [&](int32_t k, int32_t b, int32_t en) {
        if (k < nj) {
            const int32_t l = l0 + nj - 1 - k;
            if (q < en - b) {
                z_n = a.zero_t[b + q];
                o_n = a.one_t[b + q];
                if (kMM) f_n = a.in[b + q];
            }
            lam_n = a.lam[l];
            if (kAvg) avg_n = a.avg[l];
        }
    };
    range(0, base_c, end_c);
    range(1, base_n, end_n);
    rows(0, base_c, end_c);
    double bnext = DM_INF;  // B of node q of the next layer (position k-1)
    int32_t nbase = 0;
    for (int32_t k = 0; k < K; ++k) {
        const bool act = k < nj;
        const int32_t l = l0 + nj - 1 - k;
        const int32_t base = base_c, w = end_c - base_c;
        const int32_t z = z_n, o = o_n;
        const double fv = f_n;
        double lam_l = lam_n;
        const double a_l = avg_n;
        const bool valid = act && q < w;
        // issue the next position's loads
        base_c = base_n;
        end_c = end_n;
        z_n = o_n = dm::kFalse;
        if (k + 1 < K) rows(k + 1, base_c, end_c);
        if (k + 2 < K) range(k + 2, base_n, end_n);
        // next-layer distances of this node's arcs (terminals: lane unused)
        const double bz = __shfl_sync(kFullMask, bnext, gb + (z >= 0 ? z - nbase : 0));
        const double bo = __shfl_sync(kFullMask, bnext, gb + (o >= 0 ? o - nbase : 0));
        if (kMM) {
            double c0 = DM_INF, c1 = DM_INF;
            if (valid) {
                c0 = z == dm::kTrue ? fv : (z == dm::kFalse ? DM_INF : __dadd_rn(fv, bz));
                const double fl = __dadd_rn(fv, lam_l);
                c1 = o == dm::kTrue ? fl : (o == dm::kFalse ? DM_INF : __dadd_rn(fl, bo));
            }
            const double m0 = lmin8(c0, q), m1 = lmin8(c1, q);
            if (act) {
                double mb;
                lam_l = dfr_update_v<kAvg>(lam_l, a_l, m0, m1, a.omega, mb);
                if (q == 0) a.mbar[l] = mb;
            }
        } else if (kAvg && act) {
            lam_l = __dadd_rn(lam_l, a_l);
        }
        if ((kMM || kAvg) && act && q == 0) a.lam[l] = lam_l;
        const double c0 = z == dm::kTrue ? 0.0 : (z == dm::kFalse ? DM_INF : bz);
        const double c1 = o == dm::kTrue ? lam_l : (o == dm::kFalse ? DM_INF : __dadd_rn(lam_l, bo));
        const bool zero_wins = c0 <= c1;
        const double bq = zero_wins ? c0 : c1;
        if (valid) a.out[base + q] = bq;
        if (kDec) {
            const int32_t t = zero_wins ? z : o;
            uint64_t word = valid ? (uint64_t)((((t >= 0) ? t - nbase : 0) << 1) | (zero_wins ? 0 : 1)) << (8 * q) : 0ull;
            word |= __shfl_xor_sync(kFullMask, word, 1);
            word |= __shfl_xor_sync(kFullMask, word, 2);
            word |= __shfl_xor_sync(kFullMask, word, 4);
            if (act && q == 0) a.dec[l] = word;
        }
        bnext = valid ? bq : DM_INF;
        nbase = base;
        if (act && k == nj - 1 && q == 0) a.bounds[j] = bq;  // root layer: single node
    }
}

template <bool kMM, bool kAvg>
__global__ void __launch_bounds__(kNpThreads) dfr_np_forward_kernel(NpArgs a) {
    const int lane = threadIdx.x & 31, q = lane & 7, gb = lane & ~7;
    const int64_t e = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4 + (lane >> 3);
    const int32_t j = e < a.entries ? a.order[e] : -1;
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = a.bdd_layer_lo[j];
        nj = a.bdd_layer_lo[j + 1] - l0;
    }
    int32_t K = nj;
    K = max(K, __shfl_xor_sync(kFullMask, K, 8));
    K = max(K, __shfl_xor_sync(kFullMask, K, 16));
    if (K == 0) return;
    // position p = layer l0 + p; prefetch node ranges two ahead, rows one ahead
    int32_t b_n = 0, e_n = 0, e2_n = 0;  // lnl[l], lnl[l+1], lnl[l+2] of position p+1
    auto range = [&](int32_t p, int32_t &b, int32_t &en, int32_t &en2) {
        if (p < nj) {
            const int32_t l = l0 + p;
            b = a.lnl[l];
            en = a.lnl[l + 1];
            en2 = p + 1 < nj ? a.lnl[l + 2] : en;
        } else {
            b = en = en2 = 0;
        }
    };
    int32_t z_n = dm::kFalse, o_n = dm::kFalse;
    double bn_n = DM_INF, lam_n = 0.0, avg_n = 0.0;
    uint64_t desc_n = ~0ull;
    int32_t b_c = 0, e_c = 0, e2_c = 0;
    auto rows = [&](int32_t p, int32_t b, int32_t en, int32_t en2) {
        if (p < nj) {
            const int32_t l = l0 + p;
            if (q < en - b) {
                z_n = a.zero_t[b + q];
                o_n = a.one_t[b + q];
            }
            if (kMM && q < en2 - en) bn_n = a.in[en + q];
            lam_n = a.lam[l];
            if (kAvg) avg_n = a.avg[l];
            desc_n = a.relax[l];
        }
    };
    range(0, b_c, e_c, e2_c);
    range(1, b_n, e_n, e2_n);
    rows(0, b_c, e_c, e2_c);
    double fq = q == 0 ? 0.0 : DM_INF;  // F of node q of the current layer (root: F[root] = 0)
    double tb = DM_INF;
    for (int32_t p = 0; p < K; ++p) {
        const bool act = p < nj;
        const int32_t l = l0 + p;
        const int32_t base = b_c, w = e_c - b_c, nbase = e_c, wn = e2_c - e_c;
        const int32_t z = z_n, o = o_n;
        const double bnq = bn_n;
        double lam_l = lam_n;
        const double a_l = avg_n;
        const uint64_t desc = desc_n;
        const bool valid = act && q < w;
        b_c = b_n;
        e_c = e_n;
        e2_c = e2_n;
        z_n = o_n = dm::kFalse;
        bn_n = DM_INF;
        if (p + 1 < K) rows(p + 1, b_c, e_c, e2_c);
        if (p + 2 < K) range(p + 2, b_n, e_n, e2_n);
        if (valid) a.out[base + q] = fq;
        if (kMM) {
            const double bz = __shfl_sync(kFullMask, bnq, gb + (z >= 0 ? z - nbase : 0));
            const double bo = __shfl_sync(kFullMask, bnq, gb + (o >= 0 ? o - nbase : 0));
            double c0 = DM_INF, c1 = DM_INF;
            if (valid) {
                c0 = z == dm::kTrue ? fq : (z == dm::kFalse ? DM_INF : __dadd_rn(fq, bz));
                const double fl = __dadd_rn(fq, lam_l);
                c1 = o == dm::kTrue ? fl : (o == dm::kFalse ? DM_INF : __dadd_rn(fl, bo));
            }
            const double m0 = lmin8(c0, q), m1 = lmin8(c1, q);
            if (act) {
                double mb;
                lam_l = dfr_update_v<kAvg>(lam_l, a_l, m0, m1, a.omega, mb);
                if (q == 0) {
                    a.mbar[l] = mb;
                    a.lam[l] = lam_l;
                }
            }
        } else if (kAvg && act) {
            lam_l = __dadd_rn(lam_l, a_l);
            if (q == 0) a.lam[l] = lam_l;
        }
        // TRUE arcs of this layer: leftmost minimum in (node, zero-before-one) order
        double t_loc = DM_INF;
        if (valid && fq != DM_INF) {
            if (z == dm::kTrue) t_loc = fq;
            const double c = __dadd_rn(fq, lam_l);
            if (o == dm::kTrue && c < t_loc) t_loc = c;
        }
        t_loc = lmin8(t_loc, q);
        if (act && t_loc < tb) tb = t_loc;
        // publish into the next layer: target u = q, its (at most one) zero and one source
        const int zs = (int)((desc >> (8 * q)) & 15), os = (int)((desc >> (8 * q + 4)) & 15);
        const double fz = __shfl_sync(kFullMask, fq, gb + (zs < 8 ? zs : 0));
        const double fo = __shfl_sync(kFullMask, fq, gb + (os < 8 ? os : 0));
        double fnew = DM_INF;
        if (act && q < wn) {
            const double cz = zs < 8 ? fz : DM_INF;  // INF sources never win a strict <
            const double co = os < 8 ? __dadd_rn(fo, lam_l) : DM_INF;
            const double first = (os < zs) ? co : cz, second = (os < zs) ? cz : co;  // same node: zero first
            if (first < fnew) fnew = first;
            if (second < fnew) fnew = second;
        }
        fq = fnew;
    }
    if (j >= 0 && q == 0) a.bounds[j] = tb;
}

// ---------------------------------------------------------------------------
// Node-parallel passes with a 2-deep register ring (diagrams of at most
// kNpRingLayers layers): each 8-lane group stages its diagram's layer-node
// offsets in shared memory once, so a position's row addresses need no
// dependent global load, and the rows (arc targets, opposite-table values,
// dual, average, publish descriptor) are loaded two positions ahead — the
// loop unrolled by two so both ring slots are registers.  The per-position
// arithmetic is the one-ahead kernels' above, operand for operand.
constexpr int kNpRingLayers = 256;
constexpr int kNpGroups = kNpThreads / 8;

struct NpFwRow {
    int32_t z, o, b, e, e2;
    double bn, lam, avg;
    uint64_t desc;
};

template <bool kMM, bool kAvg>
__global__ void __launch_bounds__(kNpThreads) dfr_np_forward_ring_kernel(NpArgs a) {
    __shared__ int32_t lnl_s[kNpGroups][kNpRingLayers + 1];
    const int lane = threadIdx.x & 31, q = lane & 7, gb = lane & ~7;
    const int64_t e = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4 + (lane >> 3);
    const int32_t j = e < a.entries ? a.order[e] : -1;
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = a.bdd_layer_lo[j];
        nj = a.bdd_layer_lo[j + 1] - l0;
    }
    int32_t K = nj;
    K = max(K, __shfl_xor_sync(kFullMask, K, 8));
    K = max(K, __shfl_xor_sync(kFullMask, K, 16));
    if (K == 0) return;
    int32_t *ln = lnl_s[threadIdx.x >> 3];
    for (int i = q; i <= nj; i += 8) ln[i] = a.lnl[l0 + i];
    __syncwarp();
    auto load = [&](NpFwRow &r, int32_t p) {
        r.z = r.o = dm::kFalse;
        r.bn = DM_INF;
        r.b = r.e = r.e2 = 0;
        r.lam = r.avg = 0.0;
        r.desc = ~0ull;
        if (p < nj) {
            const int32_t l = l0 + p;
            r.b = ln[p];
            r.e = ln[p + 1];
            r.e2 = p + 1 < nj ? ln[p + 2] : r.e;
            if (q < r.e - r.b) {
                r.z = a.zero_t[r.b + q];
                r.o = a.one_t[r.b + q];
            }
            if (kMM && q < r.e2 - r.e) r.bn = a.in[r.e + q];
            r.lam = a.lam[l];
            if (kAvg) r.avg = a.avg[l];
            r.desc = a.relax[l];
        }
    };
    double fq = q == 0 ? 0.0 : DM_INF;  // F of node q of the current layer (root: F[root] = 0)
    double tb = DM_INF;
    auto body = [&](int32_t p, const NpFwRow &c) {
        const bool act = p < nj;
        const int32_t l = l0 + p;
        const int32_t base = c.b, w = c.e - c.b, nbase = c.e, wn = c.e2 - c.e;
        const int32_t z = c.z, o = c.o;
        const double bnq = c.bn;
        double lam_l = c.lam;
        const double a_l = c.avg;
        const uint64_t desc = c.desc;
        const bool valid = act && q < w;
        if (valid) a.out[base + q] = fq;
        if (kMM) {
            const double bz = __shfl_sync(kFullMask, bnq, gb + (z >= 0 ? z - nbase : 0));
            const double bo = __shfl_sync(kFullMask, bnq, gb + (o >= 0 ? o - nbase : 0));
            double c0 = DM_INF, c1 = DM_INF;
            if (valid) {
                c0 = z == dm::kTrue ? fq : (z == dm::kFalse ? DM_INF : __dadd_rn(fq, bz));
                const double fl = __dadd_rn(fq, lam_l);
                c1 = o == dm::kTrue ? fl : (o == dm::kFalse ? DM_INF : __dadd_rn(fl, bo));
            }
            const double m0 = lmin8(c0, q), m1 = lmin8(c1, q);
            if (act) {
                double mb;
                lam_l = dfr_update_v<kAvg>(lam_l, a_l, m0, m1, a.omega, mb);
                if (q == 0) {
                    a.mbar[l] = mb;
                    a.lam[l] = lam_l;
                }
            }
        } else if (kAvg && act) {
            lam_l = __dadd_rn(lam_l, a_l);
            if (q == 0) a.lam[l] = lam_l;
        }
        double t_loc = DM_INF;
        if (valid && fq != DM_INF) {
            if (z == dm::kTrue) t_loc = fq;
            const double cc = __dadd_rn(fq, lam_l);
            if (o == dm::kTrue && cc < t_loc) t_loc = cc;
        }
        t_loc = lmin8(t_loc, q);
        if (act && t_loc < tb) tb = t_loc;
        const int zs = (int)((desc >> (8 * q)) & 15), os = (int)((desc >> (8 * q + 4)) & 15);
        const double fz = __shfl_sync(kFullMask, fq, gb + (zs < 8 ? zs : 0));
        const double fo = __shfl_sync(kFullMask, fq, gb + (os < 8 ? os : 0));
        double fnew = DM_INF;
        if (act && q < wn) {
            const double cz = zs < 8 ? fz : DM_INF;
            const double co = os < 8 ? __dadd_rn(fo, lam_l) : DM_INF;
            const double first = (os < zs) ? co : cz, second = (os < zs) ? cz : co;
            if (first < fnew) fnew = first;
            if (second < fnew) fnew = second;
        }
        fq = fnew;
    };
    NpFwRow r0, r1;
    load(r0, 0);
    load(r1, 1);
    for (int32_t p0 = 0; p0 < K; p0 += 2) {
        {
            const NpFwRow c = r0;
            if (p0 + 2 < K) load(r0, p0 + 2);
            body(p0, c);
        }
        if (p0 + 1 < K) {
            const NpFwRow c = r1;
            if (p0 + 3 < K) load(r1, p0 + 3);
            body(p0 + 1, c);
        }
    }
    if (j >= 0 && q == 0) a.bounds[j] = tb;
}

struct NpBwRow {
    int32_t z, o, b, e;
    double f, lam, avg;
};

template <bool kMM, bool kAvg, bool kDec>
__global__ void __launch_bounds__(kNpThreads) dfr_np_backward_ring_kernel(NpArgs a) {
    __shared__ int32_t lnl_s[kNpGroups][kNpRingLayers + 1];
    const int lane = threadIdx.x & 31, q = lane & 7, gb = lane & ~7;
    const int64_t e = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4 + (lane >> 3);
    const int32_t j = e < a.entries ? a.order[e] : -1;
    int32_t l0 = 0, nj = 0;
    if (j >= 0) {
        l0 = a.bdd_layer_lo[j];
        nj = a.bdd_layer_lo[j + 1] - l0;
    }
    int32_t K = nj;
    K = max(K, __shfl_xor_sync(kFullMask, K, 8));
    K = max(K, __shfl_xor_sync(kFullMask, K, 16));
    if (K == 0) return;
    int32_t *ln = lnl_s[threadIdx.x >> 3];
    for (int i = q; i <= nj; i += 8) ln[i] = a.lnl[l0 + i];
    __syncwarp();
    auto load = [&](NpBwRow &r, int32_t k) {  // position k = layer l0 + nj - 1 - k
        r.z = r.o = dm::kFalse;
        r.f = 0.0;
        r.b = r.e = 0;
        r.lam = r.avg = 0.0;
        if (k < nj) {
            const int32_t l = l0 + nj - 1 - k;
            r.b = ln[nj - 1 - k];
            r.e = ln[nj - k];
            if (q < r.e - r.b) {
                r.z = a.zero_t[r.b + q];
                r.o = a.one_t[r.b + q];
                if (kMM) r.f = a.in[r.b + q];
            }
            r.lam = a.lam[l];
            if (kAvg) r.avg = a.avg[l];
        }
    };
    double bnext = DM_INF;  // B of node q of the next layer (position k-1)
    int32_t nbase = 0;
    auto body = [&](int32_t k, const NpBwRow &c) {
        const bool act = k < nj;
        const int32_t l = l0 + nj - 1 - k;
        const int32_t base = c.b, w = c.e - c.b;
        const int32_t z = c.z, o = c.o;
        const double fv = c.f;
        double lam_l = c.lam;
        const double a_l = c.avg;
        const bool valid = act && q < w;
        const double bz = __shfl_sync(kFullMask, bnext, gb + (z >= 0 ? z - nbase : 0));
        const double bo = __shfl_sync(kFullMask, bnext, gb + (o >= 0 ? o - nbase : 0));
        if (kMM) {
            double c0 = DM_INF, c1 = DM_INF;
            if (valid) {
                c0 = z == dm::kTrue ? fv : (z == dm::kFalse ? DM_INF : __dadd_rn(fv, bz));
                const double fl = __dadd_rn(fv, lam_l);
                c1 = o == dm::kTrue ? fl : (o == dm::kFalse ? DM_INF : __dadd_rn(fl, bo));
            }
            const double m0 = lmin8(c0, q), m1 = lmin8(c1, q);
            if (act) {
                double mb;
                lam_l = dfr_update_v<kAvg>(lam_l, a_l, m0, m1, a.omega, mb);
                if (q == 0) a.mbar[l] = mb;
            }
        } else if (kAvg && act) {
            lam_l = __dadd_rn(lam_l, a_l);
        }
        if ((kMM || kAvg) && act && q == 0) a.lam[l] = lam_l;
        const double c0 = z == dm::kTrue ? 0.0 : (z == dm::kFalse ? DM_INF : bz);
        const double c1 = o == dm::kTrue ? lam_l : (o == dm::kFalse ? DM_INF : __dadd_rn(lam_l, bo));
        const bool zero_wins = c0 <= c1;
        const double bq = zero_wins ? c0 : c1;
        if (valid) a.out[base + q] = bq;
        if (kDec) {
            const int32_t t = zero_wins ? z : o;
            uint64_t word = valid ? (uint64_t)((((t >= 0) ? t - nbase : 0) << 1) | (zero_wins ? 0 : 1)) << (8 * q) : 0ull;
            word |= __shfl_xor_sync(kFullMask, word, 1);
            word |= __shfl_xor_sync(kFullMask, word, 2);
            word |= __shfl_xor_sync(kFullMask, word, 4);
            if (act && q == 0) a.dec[l] = word;
        }
        bnext = valid ? bq : DM_INF;
        nbase = base;
        if (act && k == nj - 1 && q == 0) a.bounds[j] = bq;  // root layer: single node
    };
    NpBwRow r0, r1;
    load(r0, 0);
    load(r1, 1);
    for (int32_t k0 = 0; k0 < K; k0 += 2) {
        {
            const NpBwRow c = r0;
            if (k0 + 2 < K) load(r0, k0 + 2);
            body(k0, c);
        }
        if (k0 + 1 < K) {
            const NpBwRow c = r1;
            if (k0 + 3 < K) load(r1, k0 + 3);
            body(k0 + 1, c);
        }
    }
}

// ---------------------------------------------------------------------------
// Pipelined passes (W = 8, the product-space instances): every position's
// inputs go through a per-warp ring of kStages shared-memory stages filled
// by cp.async — the arc rows, the opposite table's rows (coalesced 16-byte
// copies spread over the warp's lanes) and each lane's own dual / average
// entry — so a lane walking a long diagram waits on memory once per
// kStages - 1 positions instead of once per position.  Arithmetic and
// operand order are those of the register kernels above (bit-identical).
constexpr int kStages = 4;
constexpr int kPW = 8;  // node slots per position

struct PipeStage {
    int32_t z[kPW][32], o[kPW][32];
    double t[kPW][32];  // opposite-direction table rows (MM passes)
    double lam[32], avg[32];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Stage fill: arc rows of position `ka` (w rows), table rows `kt` (wt rows),
// this lane's dual and average at layer `l` (l < 0: none).  A row of int32 is
// 128 bytes = 8 chunks, a row of doubles 256 bytes = 16 chunks; chunk c of
// the stage goes to lane c % 32.
template <bool kTab, bool kAvg>
__device__ __forceinline__ void fill_stage(PipeStage &st, const dm::SweepDev &s, int lane, int32_t w, int64_t slot,
                                           const double *tab, int32_t wt, int64_t slot_t, const double *lam,
                                           const double *avg, int32_t l) {
#pragma unroll
    for (int c = lane; c < 2 * kPW * 8; c += 32) {  // zero / one arc rows
        const int arr = c / (kPW * 8), row = (c / 8) % kPW, q = c % 8;
        if (row < w) {
            const int32_t *src = (arr ? s.ol : s.zl) + (slot + row) * 32 + q * 4;
            cp16((arr ? &st.o[row][0] : &st.z[row][0]) + q * 4, src);
        }
    }
    if (kTab) {
#pragma unroll
        for (int c = lane; c < kPW * 16; c += 32) {
            const int row = c / 16, q = c % 16;
            if (row < wt) cp16(&st.t[row][q * 2], tab + (slot_t + row) * 32 + q * 2);
        }
    }
    if (l >= 0) {
        cp8(&st.lam[lane], lam + l);
        if (kAvg) cp8(&st.avg[lane], avg + l);
    }
}

template <bool kMM, bool kAvg, bool kDec>
__global__ void __launch_bounds__(kThreads) dfr_backward_pipe_kernel(DfrArgs a) {
    constexpr int W = kPW;
    extern __shared__ double sm[];
    const dm::SweepDev &s = a.s;
    double *__restrict__ lamp = a.lam;
    const double *__restrict__ avgp = a.avg;
    const double *__restrict__ inp = a.in;
    double *__restrict__ outp = a.out;
    double *__restrict__ mbarp = a.mbar;
    double *__restrict__ boundsp = a.bounds;
    uint64_t *__restrict__ decp = a.dec;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
    double *nb = sm + threadIdx.x;                  // distances of position k-1 (next layer)
    double *cur = sm + W * kThreads + threadIdx.x;  // position k
    PipeStage *ring = reinterpret_cast<PipeStage *>(sm + 2 * W * kThreads) + wid * kStages;
    __shared__ int32_t meta_w[kWarps][kMetaWin];
    __shared__ int64_t meta_s[kWarps][kMetaWin];
    Meta meta{meta_w[wid], meta_s[wid], 0};
    meta_window(meta, s, p0, K, 0, lane);
    auto issue = [&](int32_t kk) {  // fill the stage of position kk (a commit group per position, maybe empty)
        if (kk < K) {
            const int32_t w = meta.w[kk - meta.lo];
            const int64_t slot = meta.slot[kk - meta.lo];
            fill_stage<kMM, kAvg>(ring[kk % kStages], s, lane, w, slot, inp, w, slot, lamp, avgp,
                                  kk < nj ? l0 + nj - 1 - kk : -1);
        }
        cp_commit();
    };
#pragma unroll
    for (int kk = 0; kk < kStages - 1; ++kk) issue(kk);
    for (int32_t k = 0; k < K; ++k) {
        // positions k .. k + kStages - 1 must be in the metadata window (uniform in the warp)
        if (k + kStages - 1 >= meta.lo + kMetaWin && meta.lo + kMetaWin < K) meta_window(meta, s, p0, K, k, lane);
        cp_wait<kStages - 2>();  // position k's stage has landed (this lane's copies) ...
        __syncwarp();            // ... and every lane's
        const PipeStage &st = ring[k % kStages];
        const int32_t w = meta.w[k - meta.lo];
        const int64_t slot = meta.slot[k - meta.lo];
        const bool act = k < nj;
        const int32_t l = l0 + nj - 1 - k;
        double lam_l = act ? st.lam[lane] : 0.0;
        if (act && (kMM || kAvg)) {
            const double a_l = kAvg ? st.avg[lane] : 0.0;
            if (kMM) {
                double m0 = DM_INF, m1 = DM_INF;
#pragma unroll
                for (int i = 0; i < W; ++i)
                    if (i < w) {
                        const double fv = st.t[i][lane];
                        const double c0 = c_zero(st.z[i][lane], fv, nb);
                        const double c1 = c_one(st.o[i][lane], __dadd_rn(fv, lam_l), nb);
                        if (c0 < m0) m0 = c0;
                        if (c1 < m1) m1 = c1;
                    }
                lam_l = dfr_update<kAvg>(lam_l, a_l, m0, m1, a.omega, mbarp + l);
            } else {
                lam_l = __dadd_rn(lam_l, a_l);
            }
            lamp[l] = lam_l;
        }
        uint64_t word = 0;
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i < w) {
                const int32_t za_ = st.z[i][lane], ob = st.o[i][lane];
                const double c0 = za_ == dm::kTrue ? 0.0 : (za_ == dm::kFalse ? DM_INF : nb[za_ * kThreads]);
                const double c1 =
                    ob == dm::kTrue ? lam_l : (ob == dm::kFalse ? DM_INF : __dadd_rn(lam_l, nb[ob * kThreads]));
                const bool zero_wins = c0 <= c1;
                const double v = zero_wins ? c0 : c1;
                cur[i * kThreads] = v;
                outp[(slot + i) * 32 + lane] = v;
                if (kDec) {
                    const int32_t t = zero_wins ? za_ : ob;
                    word |= (uint64_t)((((t >= 0) ? t : 0) << 1) | (zero_wins ? 0 : 1)) << (8 * i);
                }
            }
        if (kDec && act) decp[l] = word;
        __syncwarp();  // every lane is done with this stage before it is refilled
        issue(k + kStages - 1);
        double *t = nb;
        nb = cur;
        cur = t;
        if (act && k == nj - 1) boundsp[j] = nb[0];  // root layer: single node
    }
    cp_wait<0>();
}

template <bool kMM, bool kAvg>
__global__ void __launch_bounds__(kThreads) dfr_forward_pipe_kernel(DfrArgs a) {
    constexpr int W = kPW;
    extern __shared__ double sm[];
    const dm::SweepDev &s = a.s;
    double *__restrict__ lamp = a.lam;
    const double *__restrict__ avgp = a.avg;
    const double *__restrict__ inp = a.in;
    double *__restrict__ outp = a.out;
    double *__restrict__ mbarp = a.mbar;
    double *__restrict__ boundsp = a.bounds;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
    double *cur = sm + threadIdx.x;                 // distances from the root, position k
    double *nxt = sm + W * kThreads + threadIdx.x;  // position k-1
    PipeStage *ring = reinterpret_cast<PipeStage *>(sm + 2 * W * kThreads) + wid * kStages;
    __shared__ int32_t meta_w[kWarps][kMetaWin];
    __shared__ int64_t meta_s[kWarps][kMetaWin];
    Meta meta{meta_w[wid], meta_s[wid], 0};
    meta_window(meta, s, p0, K, K > kMetaWin ? K - kMetaWin : 0, lane);
    double tb = DM_INF;
    // step n handles position k = K - 1 - n (the walk runs from the roots down)
    auto issue = [&](int32_t n) {
        const int32_t kk = K - 1 - n;
        if (kk >= 0) {
            const int32_t w = meta.w[kk - meta.lo];
            const int64_t slot = meta.slot[kk - meta.lo];
            const int32_t wt = kk > 0 ? meta.w[kk - 1 - meta.lo] : 0;
            const int64_t st = kk > 0 ? meta.slot[kk - 1 - meta.lo] : 0;
            fill_stage<kMM, kAvg>(ring[n % kStages], s, lane, w, slot, inp, wt, st, lamp, avgp,
                                  kk < nj ? l0 + nj - 1 - kk : -1);
        }
        cp_commit();
    };
    // positions k - kStages .. k must be in the window (uniform in the warp)
    auto window_for = [&](int32_t k) {
        if (k - kStages < meta.lo && meta.lo > 0) {
            const int32_t lo = k + 1 > kMetaWin ? k + 1 - kMetaWin : 0;
            meta_window(meta, s, p0, K, lo, lane);
        }
    };
    window_for(K - 1);
#pragma unroll
    for (int n = 0; n < kStages - 1; ++n) issue(n);
    for (int32_t n = 0; n < K; ++n) {
        const int32_t k = K - 1 - n;
        window_for(k);
        cp_wait<kStages - 2>();
        __syncwarp();
        const PipeStage &st = ring[n % kStages];
        if (k < nj) {
            const int32_t w = meta.w[k - meta.lo];
            const int64_t slot = meta.slot[k - meta.lo];
            const int32_t wn = k > 0 ? meta.w[k - 1 - meta.lo] : 0;
            double lam_l = st.lam[lane];
            const int32_t l = l0 + nj - 1 - k;
            if (k == nj - 1) {  // root layer: F[root] = 0 (kernels.py:187-193)
                cur[0] = 0.0;
#pragma unroll
                for (int i = 1; i < W; ++i) cur[i * kThreads] = DM_INF;
            }
#pragma unroll
            for (int i = 0; i < W; ++i)
                if (i < w) outp[(slot + i) * 32 + lane] = cur[i * kThreads];
            if (kMM) {
                const double a_l = kAvg ? st.avg[lane] : 0.0;
                double m0 = DM_INF, m1 = DM_INF;
#pragma unroll
                for (int i = 0; i < W; ++i)
                    if (i < w) {
                        const double fv = cur[i * kThreads];
                        const int32_t za_ = st.z[i][lane], ob = st.o[i][lane];
                        const double c0 = za_ == dm::kTrue ? fv : (za_ == dm::kFalse ? DM_INF : __dadd_rn(fv, st.t[za_][lane]));
                        const double fl = __dadd_rn(fv, lam_l);
                        const double c1 = ob == dm::kTrue ? fl : (ob == dm::kFalse ? DM_INF : __dadd_rn(fl, st.t[ob][lane]));
                        if (c0 < m0) m0 = c0;
                        if (c1 < m1) m1 = c1;
                    }
                lam_l = dfr_update<kAvg>(lam_l, a_l, m0, m1, a.omega, mbarp + l);
                lamp[l] = lam_l;
            } else if (kAvg) {
                lam_l = __dadd_rn(lam_l, st.avg[lane]);
                lamp[l] = lam_l;
            }
            // push this layer's distances into the next one (kernels.py:241-269)
#pragma unroll
            for (int u = 0; u < W; ++u)
                if (u < wn) nxt[u * kThreads] = DM_INF;
#pragma unroll
            for (int i = 0; i < W; ++i)
                if (i < w) {
                    const double fv = cur[i * kThreads];
                    if (fv == DM_INF) continue;
                    const int32_t za_ = st.z[i][lane], ob = st.o[i][lane];
                    if (za_ >= 0) {
                        if (fv < nxt[za_ * kThreads]) nxt[za_ * kThreads] = fv;
                    } else if (za_ == dm::kTrue) {
                        if (fv < tb) tb = fv;
                    }
                    const double c = __dadd_rn(fv, lam_l);
                    if (ob >= 0) {
                        if (c < nxt[ob * kThreads]) nxt[ob * kThreads] = c;
                    } else if (ob == dm::kTrue) {
                        if (c < tb) tb = c;
                    }
                }
            double *t = cur;
            cur = nxt;
            nxt = t;
        }
        __syncwarp();
        issue(n + kStages - 1);
    }
    cp_wait<0>();
    if (j >= 0) boundsp[j] = tb;
}

// One pass's escrow -> the next pass's per-copy average: thread per
// visitation position (variable), copies summed in copy order.  kApply (the
// flush): the average goes straight into the duals, lam[l] += avg (the same
// single rounding a pass applies), instead of into avg[].
template <bool kApply>
__global__ void dfr_average_kernel(int32_t P, const int32_t *__restrict__ proc_ptr,
                                   const int32_t *__restrict__ proc_layers, const double *__restrict__ mbar,
                                   double *__restrict__ out) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int32_t lo = proc_ptr[p], hi = proc_ptr[p + 1];
    if (hi == lo) return;
    constexpr int kReg = 8;  // copies held in registers; the rest re-read
    double v[kReg], lv[kReg];
    int32_t ls[kReg];
    double sum = 0.0;
    int32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < kReg; ++i)
        if (lo + i < hi) {
            ls[i] = proc_layers[lo + i];
            v[i] = mbar[ls[i]];
            if (kApply) lv[i] = out[ls[i]];
        }
    for (int32_t t = lo; t < hi; ++t) {
        const double x = t - lo < kReg ? v[t - lo] : mbar[proc_layers[t]];
        if (x != DM_INF) {
            sum = __dadd_rn(sum, x);
            ++cnt;
        }
    }
    const double mean = cnt ? __ddiv_rn(sum, (double)cnt) : 0.0;
#pragma unroll
    for (int i = 0; i < kReg; ++i)
        if (lo + i < hi) {
            const double a = v[i] != DM_INF ? mean : 0.0;
            out[ls[i]] = kApply ? __dadd_rn(lv[i], a) : a;
        }
    for (int32_t t = lo + kReg; t < hi; ++t) {
        const int32_t l = proc_layers[t];
        const double a = mbar[l] != DM_INF ? mean : 0.0;
        out[l] = kApply ? __dadd_rn(out[l], a) : a;
    }
}

// interleaved table -> reference node order (tests, and consumers of F / B)
__global__ void dfr_to_nodes_kernel(dm::SweepDev s, const double *__restrict__ x_il, double *__restrict__ x) {
    const int lane = threadIdx.x & 31;
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= s.groups) return;
    const int32_t j = s.grp_bdd[g * 32 + lane];
    if (j < 0) return;
    const int32_t l0 = s.bdd_layer_lo[j], nj = s.bdd_layer_lo[j + 1] - l0;
    const int64_t p0 = s.grp_pos_lo[g];
    for (int32_t k = 0; k < nj; ++k) {
        const int32_t l = l0 + nj - 1 - k;
        const int32_t v0 = s.lnl[l], w = s.lnl[l + 1] - v0;
        const int64_t slot = s.pos_slot[p0 + k];
        for (int32_t i = 0; i < w; ++i) x[v0 + i] = x_il[(slot + i) * 32 + lane];
    }
}

// --------------------------------------------------------------------------
// Partitioned instances (partition.py): the diagrams are split over ranks,
// and a variable whose copies span ranks ("boundary" variable) is averaged
// from an exchange buffer that holds one slot per copy in global copy order
// (each rank writes its copies' escrow, zeros elsewhere; one allreduce-sum
// per pass makes it whole — exact, every slot has one contributor).
__global__ void dfr_boundary_gather_kernel(int64_t n, const int32_t *__restrict__ layer,
                                           const int32_t *__restrict__ slot, const double *__restrict__ mbar,
                                           double *__restrict__ buf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) buf[slot[i]] = mbar[layer[i]];
}

// per local boundary copy i: the mean of the finite escrow in
// buf[slot_lo[i], slot_hi[i]) (copy order, from 0.0 — dfr_average_kernel's
// arithmetic), written to out[layer[i]] (apply: added to it)
template <bool kApply>
__global__ void dfr_boundary_average_kernel(int64_t n, const int32_t *__restrict__ layer,
                                            const int32_t *__restrict__ slot, const int32_t *__restrict__ slot_lo,
                                            const int32_t *__restrict__ slot_hi, const double *__restrict__ buf,
                                            double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double sum = 0.0;
    int32_t cnt = 0;
    for (int32_t t = slot_lo[i]; t < slot_hi[i]; ++t) {
        const double x = buf[t];
        if (x != DM_INF) {
            sum = __dadd_rn(sum, x);
            ++cnt;
        }
    }
    const double mean = cnt ? __ddiv_rn(sum, (double)cnt) : 0.0;
    const double a = buf[slot[i]] != DM_INF ? mean : 0.0;
    const int32_t l = layer[i];
    out[l] = kApply ? __dadd_rn(out[l], a) : a;
}

int fail(cudaError_t e, const char *what) {
    dm::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DM_ERR_CUDA;
}

template <typename Kern>
int launch(Kern kern, const DfrArgs &a, size_t smem, cudaStream_t st, const char *what) {
    const int blocks = (int)((a.s.groups * 32 + kThreads - 1) / kThreads);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<blocks, kThreads, smem, st>>>(a);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, what);
}

bool np_ring() {
    static const int v = [] {
        const char *e = std::getenv("DM_DFR_NP_RING");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0;
}

bool use_pipe() {
    static const int v = [] {
        const char *e = std::getenv("DM_DFR_PIPE");
        return e ? std::atoi(e) : 0;  // A/B: the ring costs occupancy; slower than the register kernels
    }();
    return v != 0;
}

int backward_pipe(const DfrArgs &a, cudaStream_t st) {
    const size_t smem = 2 * kPW * kThreads * sizeof(double) + kWarps * kStages * sizeof(PipeStage);
    const bool mm = a.mbar != nullptr, avg = a.avg != nullptr, dec = a.dec != nullptr;
    if (mm && avg) return launch(dfr_backward_pipe_kernel<true, true, false>, a, smem, st, "dfr_backward");
    if (mm) return launch(dfr_backward_pipe_kernel<true, false, false>, a, smem, st, "dfr_backward");
    if (avg && dec) return launch(dfr_backward_pipe_kernel<false, true, true>, a, smem, st, "dfr_backward");
    if (avg) return launch(dfr_backward_pipe_kernel<false, true, false>, a, smem, st, "dfr_backward");
    if (dec) return launch(dfr_backward_pipe_kernel<false, false, true>, a, smem, st, "dfr_backward");
    return launch(dfr_backward_pipe_kernel<false, false, false>, a, smem, st, "dfr_backward");
}

int forward_pipe(const DfrArgs &a, cudaStream_t st) {
    const size_t smem = 2 * kPW * kThreads * sizeof(double) + kWarps * kStages * sizeof(PipeStage);
    const bool mm = a.mbar != nullptr, avg = a.avg != nullptr;
    if (mm && avg) return launch(dfr_forward_pipe_kernel<true, true>, a, smem, st, "dfr_forward");
    if (mm) return launch(dfr_forward_pipe_kernel<true, false>, a, smem, st, "dfr_forward");
    if (avg) return launch(dfr_forward_pipe_kernel<false, true>, a, smem, st, "dfr_forward");
    return launch(dfr_forward_pipe_kernel<false, false>, a, smem, st, "dfr_forward");
}

template <int W>
int backward_w(const DfrArgs &a, cudaStream_t st) {
    const size_t smem = 2 * W * kThreads * sizeof(double);
    const bool mm = a.mbar != nullptr, avg = a.avg != nullptr, dec = a.dec != nullptr && W <= 8;
    if (mm && avg) return launch(dfr_backward_kernel<W, true, true, false>, a, smem, st, "dfr_backward");
    if (mm) return launch(dfr_backward_kernel<W, true, false, false>, a, smem, st, "dfr_backward");
    if (avg && dec) return launch(dfr_backward_kernel<W, false, true, true>, a, smem, st, "dfr_backward");
    if (avg) return launch(dfr_backward_kernel<W, false, true, false>, a, smem, st, "dfr_backward");
    if (dec) return launch(dfr_backward_kernel<W, false, false, true>, a, smem, st, "dfr_backward");
    return launch(dfr_backward_kernel<W, false, false, false>, a, smem, st, "dfr_backward");
}

template <int W>
int forward_w(const DfrArgs &a, cudaStream_t st) {
    const size_t smem = 3 * W * kThreads * sizeof(double);
    const bool mm = a.mbar != nullptr, avg = a.avg != nullptr;
    if (mm && avg) return launch(dfr_forward_kernel<W, true, true>, a, smem, st, "dfr_forward");
    if (mm) return launch(dfr_forward_kernel<W, true, false>, a, smem, st, "dfr_forward");
    if (avg) return launch(dfr_forward_kernel<W, false, true>, a, smem, st, "dfr_forward");
    return launch(dfr_forward_kernel<W, false, false>, a, smem, st, "dfr_forward");
}

}  // namespace

namespace dm {

int dfr_pass(const SweepDev &s, bool forward, double omega, double *lam, const double *avg, const double *in,
             double *out, double *mbar, double *bounds, uint64_t *dec, void *stream) {
    if (s.groups == 0) return DM_OK;
    DfrArgs a{s, omega, lam, avg, in, out, mbar, bounds, forward ? nullptr : dec};
    cudaStream_t st = (cudaStream_t)stream;
    if (forward) {
        if (s.max_width <= 8 && use_pipe()) return forward_pipe(a, st);
        if (s.max_width <= 8) return forward_w<8>(a, st);
        if (s.max_width <= 16) return forward_w<16>(a, st);
        return forward_w<32>(a, st);
    }
    if (s.max_width <= 8 && use_pipe()) return backward_pipe(a, st);
    if (s.max_width <= 8) return backward_w<8>(a, st);
    if (s.max_width <= 16) return backward_w<16>(a, st);
    return backward_w<32>(a, st);
}

int dfr_average(int64_t P, const int32_t *proc_ptr, const int32_t *proc_layers, const double *mbar, double *out,
                bool apply, void *stream) {
    if (P == 0) return DM_OK;
    constexpr int kT = 256;
    const int blocks = (int)((P + kT - 1) / kT);
    if (apply)
        dfr_average_kernel<true><<<blocks, kT, 0, (cudaStream_t)stream>>>((int32_t)P, proc_ptr, proc_layers, mbar, out);
    else
        dfr_average_kernel<false><<<blocks, kT, 0, (cudaStream_t)stream>>>((int32_t)P, proc_ptr, proc_layers, mbar, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, "dfr_average");
}

int dfr_to_nodes(const SweepDev &s, const double *x_il, double *x, void *stream) {
    if (s.groups == 0) return DM_OK;
    const int blocks = (int)((s.groups * 32 + kThreads - 1) / kThreads);
    dfr_to_nodes_kernel<<<blocks, kThreads, 0, (cudaStream_t)stream>>>(s, x_il, x);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, "dfr_to_nodes");
}

int dfr_boundary_gather(int64_t n, const int32_t *layer, const int32_t *slot, const double *mbar, double *buf,
                        void *stream) {
    if (n <= 0) return DM_OK;
    dfr_boundary_gather_kernel<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, layer, slot, mbar, buf);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, "dfr_boundary_gather");
}

int dfr_boundary_average(int64_t n, const int32_t *layer, const int32_t *slot, const int32_t *slot_lo,
                         const int32_t *slot_hi, const double *buf, double *out, bool apply, void *stream) {
    if (n <= 0) return DM_OK;
    const int blocks = (int)((n + 255) / 256);
    if (apply)
        dfr_boundary_average_kernel<true><<<blocks, 256, 0, (cudaStream_t)stream>>>(n, layer, slot, slot_lo, slot_hi,
                                                                                     buf, out);
    else
        dfr_boundary_average_kernel<false><<<blocks, 256, 0, (cudaStream_t)stream>>>(n, layer, slot, slot_lo,
                                                                                      slot_hi, buf, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, "dfr_boundary_average");
}

int dfr_np_pass(const SweepDev &s, const int32_t *zero_t, const int32_t *one_t, const uint64_t *relax, bool forward,
                double omega, double *lam, const double *avg, const double *in, double *out, double *mbar,
                double *bounds, uint64_t *dec, void *stream) {
    if (s.groups == 0) return DM_OK;
    NpArgs a{s.grp_bdd, s.groups * 32, s.bdd_layer_lo, s.lnl, zero_t, one_t, relax, omega, lam, avg, in, out, mbar,
             bounds, forward ? nullptr : dec};
    const int64_t warps = (a.entries + 3) / 4;
    const int blocks = (int)((warps * 32 + kNpThreads - 1) / kNpThreads);
    const cudaStream_t st = (cudaStream_t)stream;
    const bool mm = mbar != nullptr, av = avg != nullptr, dc = a.dec != nullptr;
    if (s.max_layers > 0 && s.max_layers <= kNpRingLayers && np_ring()) {
        if (forward) {
            if (mm && av) dfr_np_forward_ring_kernel<true, true><<<blocks, kNpThreads, 0, st>>>(a);
            else if (mm) dfr_np_forward_ring_kernel<true, false><<<blocks, kNpThreads, 0, st>>>(a);
            else if (av) dfr_np_forward_ring_kernel<false, true><<<blocks, kNpThreads, 0, st>>>(a);
            else dfr_np_forward_ring_kernel<false, false><<<blocks, kNpThreads, 0, st>>>(a);
        } else {
            if (mm && av) dfr_np_backward_ring_kernel<true, true, false><<<blocks, kNpThreads, 0, st>>>(a);
            else if (mm) dfr_np_backward_ring_kernel<true, false, false><<<blocks, kNpThreads, 0, st>>>(a);
            else if (av && dc) dfr_np_backward_ring_kernel<false, true, true><<<blocks, kNpThreads, 0, st>>>(a);
            else if (av) dfr_np_backward_ring_kernel<false, true, false><<<blocks, kNpThreads, 0, st>>>(a);
            else if (dc) dfr_np_backward_ring_kernel<false, false, true><<<blocks, kNpThreads, 0, st>>>(a);
            else dfr_np_backward_ring_kernel<false, false, false><<<blocks, kNpThreads, 0, st>>>(a);
        }
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? DM_OK : fail(e, forward ? "dfr_np_forward" : "dfr_np_backward");
    }
    if (forward) {
        if (mm && av) dfr_np_forward_kernel<true, true><<<blocks, kNpThreads, 0, st>>>(a);
        else if (mm) dfr_np_forward_kernel<true, false><<<blocks, kNpThreads, 0, st>>>(a);
        else if (av) dfr_np_forward_kernel<false, true><<<blocks, kNpThreads, 0, st>>>(a);
        else dfr_np_forward_kernel<false, false><<<blocks, kNpThreads, 0, st>>>(a);
    } else {
        if (mm && av) dfr_np_backward_kernel<true, true, false><<<blocks, kNpThreads, 0, st>>>(a);
        else if (mm) dfr_np_backward_kernel<true, false, false><<<blocks, kNpThreads, 0, st>>>(a);
        else if (av && dc) dfr_np_backward_kernel<false, true, true><<<blocks, kNpThreads, 0, st>>>(a);
        else if (av) dfr_np_backward_kernel<false, true, false><<<blocks, kNpThreads, 0, st>>>(a);
        else if (dc) dfr_np_backward_kernel<false, false, true><<<blocks, kNpThreads, 0, st>>>(a);
        else dfr_np_backward_kernel<false, false, false><<<blocks, kNpThreads, 0, st>>>(a);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DM_OK : fail(e, forward ? "dfr_np_forward" : "dfr_np_backward");
}

}  // namespace dm


