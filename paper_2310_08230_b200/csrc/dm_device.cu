// B200 (sm_100a) kernels of the DiscoMatch dual solver and the device half
// of the C-ABI (include/discomatch_b200.h).
//
// Every kernel reproduces its reference counterpart bit-for-bit: binary64
// only, no FMA contraction (-fmad=false plus explicit __d*_rn intrinsics on
// the exact paths), identical association order and tie rules.
//
// Layout: the flat node table of FlatBdds (kernels.py:35-92) as int32 SoA
// arrays in HBM; dual vectors (lam, F, B, bounds) float64.
//
// Exact averaging passes (kernels.py:162-362).  The reference visits
// variables one at a time; a variable's update only depends on the copies
// of the previous (forward) / next (backward) layer of each of its
// diagrams.  The host turns that DAG into levels and packs same-level
// variables into 32-lane warp tasks (one lane per diagram copy).  A
// persistent cooperative kernel walks the tasks in level order; instead of
// grid barriers it uses *self-validating* distances: before a pass every
// distance the pass will produce is set to a NaN sentinel, a lane polls its
// inputs with relaxed gpu-scope loads until none is the sentinel, and
// producers publish with relaxed stores.  Each 8-byte value is written once
// per pass, so no fences or flags are needed and the critical path is one
// L2 round trip per DAG level.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <map>
#include <mutex>
#include <memory>
#include <chrono>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "dm_internal.h"

#define DM_INF __longlong_as_double(0x7ff0000000000000LL)

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kSentinel = 0x7ff4dead0badf00dULL;  // signalling-NaN payload

__device__ __forceinline__ double ld_relaxed(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double((long long)v);
}
// p[0], p[1] as one 16-byte relaxed load when p is 16-byte aligned and the
// pair is adjacent (two 8-byte loads otherwise)
__device__ __forceinline__ void ld_relaxed_pair(const double *p0, const double *p1, double &v0, double &v1) {
    if (p1 == p0 + 1 && ((uintptr_t)p0 & 15) == 0) {
        unsigned long long a, b;
        asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p0) : "memory");
        v0 = __longlong_as_double((long long)a);
        v1 = __longlong_as_double((long long)b);
    } else {
        v0 = ld_relaxed(p0);
        v1 = ld_relaxed(p1);
    }
}
// Loads p[min(i, n-1)] for i < 8 (n >= 1) in ONE asm block of unpredicated
// loads, so that all of them are in flight before the first sentinel check
// (separately predicated loads get interleaved with the checks by the
// scheduler, which serialises the round trips).  Slots i >= n re-read element
// n-1, a real input, so checking all 8 is exact.
__device__ __forceinline__ void ld8_relaxed(const double *p, int n, double *v) {
    unsigned long long r[8];
    const double *q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = p + (i < n ? i : n - 1);
    asm volatile(
        "ld.relaxed.gpu.global.b64 %0, [%8];\n\t"
        "ld.relaxed.gpu.global.b64 %1, [%9];\n\t"
        "ld.relaxed.gpu.global.b64 %2, [%10];\n\t"
        "ld.relaxed.gpu.global.b64 %3, [%11];\n\t"
        "ld.relaxed.gpu.global.b64 %4, [%12];\n\t"
        "ld.relaxed.gpu.global.b64 %5, [%13];\n\t"
        "ld.relaxed.gpu.global.b64 %6, [%14];\n\t"
        "ld.relaxed.gpu.global.b64 %7, [%15];"
        : "=l"(r[0]), "=l"(r[1]), "=l"(r[2]), "=l"(r[3]), "=l"(r[4]), "=l"(r[5]), "=l"(r[6]), "=l"(r[7])
        : "l"(q[0]), "l"(q[1]), "l"(q[2]), "l"(q[3]), "l"(q[4]), "l"(q[5]), "l"(q[6]), "l"(q[7])
        : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __longlong_as_double((long long)r[i]);
}

// Polls the n <= W inputs at p into v: true when none is the sentinel.
// Slots i >= n come back as +INF (padding nodes).  kFence: see below.
template <int W, bool kFence>
__device__ __forceinline__ bool poll_inputs(const double *p, int n, double (&v)[W]) {
    static_assert(W % 8 == 0, "layer width bound must be a multiple of 8");
    double t[W];
#pragma unroll
    for (int g = 0; g < W; g += 8) {
        if (g == 0 || g < n) ld8_relaxed(p + g, n - g, t + g);
    }
    // scheduling fence: keeps ptxas from interleaving the checks with the
    // loads in the forward kernel (it pairs them there, paying one round trip
    // per pair; the backward kernel's schedule is fine without it, and the
    // fence costs it ~5%)
    if (kFence) __syncwarp(__activemask());
    unsigned long long bad = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        if (i >= 8 && i >= ((n + 7) & ~7)) t[i] = DM_INF;  // group not loaded
        bad |= (unsigned long long)(__double_as_longlong(t[i]) == (long long)kSentinel);
    }
#pragma unroll
    for (int i = 0; i < W; ++i) v[i] = i < n ? t[i] : DM_INF;
    return bad == 0;
}

__device__ __forceinline__ void st_relaxed(double *p, double x) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(x))
                 : "memory");
}
// p[0] = x0 (if n > 0), p[1] = x1 (if n > 1): one 16-byte relaxed store when
// both are written and p is 16-byte aligned
__device__ __forceinline__ void st_relaxed_pair(double *p, double x0, double x1, int n) {
    if (n > 1 && ((uintptr_t)p & 15) == 0) {
        asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(__double_as_longlong(x0)),
                     "l"(__double_as_longlong(x1))
                     : "memory");
    } else {
        if (n > 0) st_relaxed(p, x0);
        if (n > 1) st_relaxed(p + 1, x1);
    }
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// A lane waits at most this long for its inputs; past it the pass aborts
// (status word set, every warp drains) instead of hanging the device.
constexpr uint64_t kWaitLimitNs = 4000000000ull;

__device__ __forceinline__ bool is_sentinel(double x) {
    return (unsigned long long)__double_as_longlong(x) == kSentinel;
}

// --------------------------------------------------------------------------
// per-layer / per-diagram kernels on the reference layout (the full-table
// sweeps live in dm_sweep.cu on the interleaved layout)
// --------------------------------------------------------------------------
__global__ void k_min_marginals_kernel(int32_t L, const int32_t *__restrict__ lnl,
                                       const int32_t *__restrict__ zero_t, const int32_t *__restrict__ one_t,
                                       const double *__restrict__ lam, const double *__restrict__ F,
                                       const double *__restrict__ B, double *__restrict__ m0_out,
                                       double *__restrict__ m1_out) {
    const int32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    const double lam_l = lam[l];
    double m0 = DM_INF, m1 = DM_INF;
    for (int32_t v = lnl[l]; v < lnl[l + 1]; ++v) {
        const double fv = F[v];
        if (fv == DM_INF) continue;
        const int32_t a = zero_t[v], b = one_t[v];
        const double c0 = a == dm::kTrue ? fv : (a == dm::kFalse ? DM_INF : __dadd_rn(fv, B[a]));
        if (c0 < m0) m0 = c0;
        const double c1 = b == dm::kTrue ? __dadd_rn(fv, lam_l)
                                         : (b == dm::kFalse ? DM_INF : __dadd_rn(__dadd_rn(fv, lam_l), B[b]));
        if (c1 < m1) m1 = c1;
    }
    m0_out[l] = m0;
    m1_out[l] = m1;
}

__global__ void k_argmin_kernel(int32_t nb, const int32_t *__restrict__ bdd_layer_lo,
                                const int32_t *__restrict__ lnl, const int32_t *__restrict__ zero_t,
                                const int32_t *__restrict__ one_t, const double *__restrict__ lam,
                                const double *__restrict__ B, double *__restrict__ bits) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nb) return;
    int32_t v = lnl[bdd_layer_lo[j]];
    for (int32_t l = bdd_layer_lo[j]; l < bdd_layer_lo[j + 1]; ++l) {
        const int32_t a = zero_t[v], b = one_t[v];
        const double c0 = a == dm::kTrue ? 0.0 : (a == dm::kFalse ? DM_INF : B[a]);
        const double c1 = b == dm::kTrue ? lam[l] : (b == dm::kFalse ? DM_INF : __dadd_rn(lam[l], B[b]));
        int32_t nxt;
        if (c0 <= c1) {
            bits[l] = 0.0;
            nxt = a;
        } else {
            bits[l] = 1.0;
            nxt = b;
        }
        if (nxt >= 0) v = nxt;
    }
}

// The same walk from the decisions the node-parallel backward pass recorded
// (one byte per node: (next-layer slot << 1) | bit, an L2-resident table):
// one dependent byte load per layer instead of two table lookups.
__global__ void k_argmin_walk_kernel(int32_t nb, const int32_t *__restrict__ bdd_layer_lo,
                                     const int32_t *__restrict__ lnl, const uint64_t *__restrict__ dec,
                                     double *__restrict__ bits) {
    (void)lnl;
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nb) return;
    int32_t slot = 0;  // the root
    for (int32_t l = bdd_layer_lo[j]; l < bdd_layer_lo[j + 1]; ++l) {
        const int32_t code = (int32_t)(dec[l] >> (8 * slot)) & 0xff;
        bits[l] = (double)(code & 1);
        slot = code >> 1;
    }
}

// --------------------------------------------------------------------------
// per-variable kernels (thread per visitation position)
// --------------------------------------------------------------------------
__global__ void init_duals_kernel(int32_t L, const int32_t *__restrict__ layer_var,
                                  const int32_t *__restrict__ var_count, const double *__restrict__ costs,
                                  double *__restrict__ lam) {
    const int32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    const int32_t v = layer_var[l];
    lam[l] = __ddiv_rn(costs[v], (double)var_count[v]);
}

__global__ void project_kernel(int32_t P, const int32_t *__restrict__ proc_ptr,
                               const int32_t *__restrict__ proc_layers, const double *__restrict__ dh,
                               double *__restrict__ d) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int32_t lo = proc_ptr[p], hi = proc_ptr[p + 1];
    if (hi == lo) return;
    double s = 0.0;
    for (int32_t t = lo; t < hi; ++t) s = __dadd_rn(s, dh[proc_layers[t]]);
    const double mean = __ddiv_rn(s, (double)(hi - lo));
    for (int32_t t = lo; t < hi; ++t) {
        const int32_t l = proc_layers[t];
        d[l] = __dsub_rn(dh[l], mean);
    }
}

__global__ void lambda_sums_kernel(int32_t P, const int32_t *__restrict__ proc_ptr,
                                   const int32_t *__restrict__ proc_layers,
                                   const int32_t *__restrict__ pos_var, const double *__restrict__ lam,
                                   double *__restrict__ out) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    if (pos_var[p] < 0) return;  // unconstrained: the host fills its cost
    double s = 0.0;
    for (int32_t t = proc_ptr[p]; t < proc_ptr[p + 1]; ++t) s = __dadd_rn(s, lam[proc_layers[t]]);
    out[pos_var[p]] = s;
}

__global__ void agreement_kernel(int32_t P, const int32_t *__restrict__ proc_ptr,
                                 const int32_t *__restrict__ proc_layers, const int32_t *__restrict__ pos_var,
                                 const double *__restrict__ m0, const double *__restrict__ m1,
                                 int8_t *__restrict__ agrees, double *__restrict__ score,
                                 int8_t *__restrict__ preferred) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || pos_var[p] < 0) return;  // unconstrained: host defaults (no vote)
    double vmax = -2.0, vmin = 2.0, total = 0.0;
    const int32_t lo = proc_ptr[p], hi = proc_ptr[p + 1];
    for (int32_t t = lo; t < hi; ++t) {
        const int32_t l = proc_layers[t];
        const double a = m0[l], b = m1[l];
        const bool fa = a != DM_INF, fb = b != DM_INF;
        double diff;
        if (fa && fb) diff = __dsub_rn(b, a);
        else if (fa) diff = DM_INF;      // one-branch forced to 0
        else if (fb) diff = -DM_INF;     // forced to 1
        else diff = __longlong_as_double(0x7ff8000000000000LL);  // impossible in co-reachable diagrams
        const double vote = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : (diff == 0.0 ? 0.0 : diff));
        vmax = fmax(vmax, vote);  // np.maximum propagates NaN; unreachable here
        vmin = fmin(vmin, vote);
        total = __dadd_rn(total, diff);
    }
    const int32_t v = pos_var[p];
    agrees[v] = (vmax == vmin) && (vmax != 0.0) && (hi > lo);
    const double t = total != total ? 0.0 : total;
    score[v] = fabs(t);
    preferred[v] = vmax > 0.0 ? 0 : 1;
}

// --------------------------------------------------------------------------
// Perturbation rounding (rounding.py; the paper's primal heuristic after
// FastDOG): per variable, the copies' min-marginal
// votes decide a push direction (unanimous vote, else the sign of their
// sum, else a hashed coin), the cost moves by dir * delta * (1 + u) (delta *
// boost for variables whose vote is already unanimous) with u a
// hashed uniform in [0, 1), spread evenly over the copies' duals so they
// stay feasible for the perturbed costs.  values[v] = the voted value,
// agrees[v] = unanimous and strict; *disagree counts the others.
__device__ __forceinline__ uint64_t dm_mix64(uint64_t seed, int32_t round, int32_t v) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((((uint64_t)(uint32_t)round) << 32) + (uint64_t)(uint32_t)v + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void perturb_kernel(int32_t P, const int32_t *__restrict__ proc_ptr, const int32_t *__restrict__ proc_layers,
                               const int32_t *__restrict__ pos_var, const double *__restrict__ m0,
                               const double *__restrict__ m1, double *__restrict__ lam, double delta, double boost,
                               uint64_t seed, int32_t round, int8_t *__restrict__ values, int8_t *__restrict__ agrees,
                               int *__restrict__ disagree) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || pos_var[p] < 0) return;
    const int32_t lo = proc_ptr[p], hi = proc_ptr[p + 1];
    double vmax = -2.0, vmin = 2.0, total = 0.0;
    for (int32_t t = lo; t < hi; ++t) {
        const int32_t l = proc_layers[t];
        const double a = m0[l], b = m1[l];
        const bool fa = a != DM_INF, fb = b != DM_INF;
        const double diff = (fa && fb) ? __dsub_rn(b, a) : (fa ? DM_INF : -DM_INF);
        const double vote = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
        vmax = fmax(vmax, vote);
        vmin = fmin(vmin, vote);
        total = __dadd_rn(total, diff);
    }
    const int32_t v = pos_var[p];
    const bool agree = vmax == vmin && vmax != 0.0;
    const uint64_t h = dm_mix64(seed, round, v);
    double dir;
    if (agree) dir = vmax;
    else if (total > 0.0) dir = 1.0;
    else if (total < 0.0) dir = -1.0;
    else dir = ((h >> 10) & 1ull) ? 1.0 : -1.0;  // tie or inf - inf
    const double u = (double)(h >> 11) * 0x1.0p-53;
    const double mag = agree ? __dmul_rn(delta, boost) : delta;  // settled variables pushed harder
    const double d = __dmul_rn(__dmul_rn(dir, mag), __dadd_rn(1.0, u));
    const double share = __ddiv_rn(d, (double)(hi - lo));
    for (int32_t t = lo; t < hi; ++t) {
        const int32_t l = proc_layers[t];
        lam[l] = __dadd_rn(lam[l], share);
    }
    values[v] = dir > 0.0 ? 0 : 1;
    agrees[v] = agree;
    if (!agree) atomicAdd(disagree, 1);
}

// --------------------------------------------------------------------------
// elementwise vectors (numpy rounding: one rounding per operation)
// --------------------------------------------------------------------------
__global__ void axpy_dev_kernel(double *__restrict__ x, const double *__restrict__ y, double alpha,
                                const double *__restrict__ dot, double *__restrict__ alpha_out, int64_t n) {
    const double a = __dmul_rn(alpha, dot[0]);
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 == 0 && alpha_out) alpha_out[0] = a;
    for (int64_t i = i0; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dsub_rn(x[i], __dmul_rn(a, y[i]));
}

__global__ void scale_dev_kernel(double *__restrict__ x, double num, const double *__restrict__ den, int64_t n) {
    const double r = __ddiv_rn(num, den[0]);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dmul_rn(r, x[i]);
}

__global__ void lbfgs_up_kernel(double *__restrict__ x, const double *__restrict__ s,
                                const double *__restrict__ alpha, double rho, const double *__restrict__ dot,
                                int64_t n) {
    const double c = __dsub_rn(alpha[0], __dmul_rn(rho, dot[0]));
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], __dmul_rn(s[i], c));
}

// qn.py:203-206 on the device: the step search's verdict (e_best > base)
// decides, and lam += gamma_best * d with axpy_host's two roundings; out =
// {gamma_best, used, trials} for the host's end-of-iteration read-back
__global__ void qn_move_kernel(double *__restrict__ x, const double *__restrict__ y, double base,
                               const double *__restrict__ state, double *__restrict__ out, int64_t n) {
    const bool used = state[2] > base;
    const double g = state[3];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[0] = g;
        out[1] = used ? 1.0 : 0.0;
        out[2] = state[6];
    }
    if (!used) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], __dmul_rn(g, y[i]));
}

__global__ void axpy_host_kernel(double *__restrict__ x, double g, const double *__restrict__ y, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], __dmul_rn(g, y[i]));
}

__global__ void sub_kernel(double *__restrict__ out, const double *__restrict__ a, const double *__restrict__ b,
                           int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __dsub_rn(a[i], b[i]);
}

// --------------------------------------------------------------------------
// numpy pairwise summation (loops_utils.h.src pairwise_sum)
// --------------------------------------------------------------------------
template <bool kDot>
__device__ __forceinline__ double pw_elem(const double *__restrict__ a, const double *__restrict__ b, int64_t i) {
    if (kDot) return __dmul_rn(a[i], b[i]);
    return a[i];
}

// One leaf per 8 lanes: lane q of the octet owns numpy's accumulator r[q]
// (elements q, q+8, q+16, ... of the leaf, summed in that order), so a warp
// reads four contiguous 64-byte segments per step; the octet then combines
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) with shuffles and lane 0 adds the
// n % 8 tail sequentially — exactly loops_utils.h.src pairwise_sum's leaf.
template <bool kDot>
__global__ void pw_leaf_kernel(int32_t nleaves, const int64_t *__restrict__ leaf_off,
                               const int32_t *__restrict__ leaf_len, const double *__restrict__ a,
                               const double *__restrict__ b, double *__restrict__ vals,
                               const double *__restrict__ skip = nullptr) {
    if (skip && *skip != 0.0) return;  // device step search already stopped
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t k = t >> 3;
    const int q = threadIdx.x & 7;
    const bool live = k < nleaves;
    int64_t off = 0;
    int32_t n = 0;
    if (live) {
        off = leaf_off[k];
        n = leaf_len[k];
    }
    const double *pa = a + off;
    const double *pb = kDot ? b + off : nullptr;
    const int32_t stop = n - (n % 8);
    double r = 0.0;
    if (live && n >= 8) {
        r = pw_elem<kDot>(pa, pb, q);
        for (int32_t i = 8; i < stop; i += 8) r = __dadd_rn(r, pw_elem<kDot>(pa, pb, i + q));
    }
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) within the octet
    const double r1 = __shfl_xor_sync(0xffffffffu, r, 1);
    const double s01 = (q & 1) ? __dadd_rn(r1, r) : __dadd_rn(r, r1);
    const double s2 = __shfl_xor_sync(0xffffffffu, s01, 2);
    const double s03 = (q & 2) ? __dadd_rn(s2, s01) : __dadd_rn(s01, s2);
    const double s4 = __shfl_xor_sync(0xffffffffu, s03, 4);
    const double s07 = (q & 4) ? __dadd_rn(s4, s03) : __dadd_rn(s03, s4);
    if (!live || q != 0) return;
    double res;
    int32_t i;
    if (n < 8) {
        res = 0.0;
        i = 0;
    } else {
        res = s07;
        i = stop;
    }
    for (; i < n; ++i) res = __dadd_rn(res, pw_elem<kDot>(pa, pb, i));
    vals[k] = res;
}

// Device step search (qn.py:132-159 find_step_size): state ctl =
// {gamma, e_init, e_best, gamma_best, e_cur, stop, trials, -}; after trial
// `trial`'s bound sum, the same comparisons and gamma updates as the host
// loop, in double.
struct StepParams {
    double free_c, shrink, grow, min_ascent;
    int32_t max_trials;
};

__device__ void step_decide(double *ctl, double sum, const StepParams &p, int trial) {
    const double e = __dadd_rn(sum, p.free_c);  // dual_objective: bounds sum + free variables
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
        if (__dsub_rn(e, ctl[1]) >= p.min_ascent) {
            ctl[5] = 1.0;
            return;
        }
    }
    if (trial < p.max_trials)
        ctl[0] = __dmul_rn(ctl[0], ctl[4] <= ctl[1] ? p.shrink : p.grow);
    else
        ctl[5] = 1.0;
}

__global__ void pw_combine_kernel(int32_t nleaves, int32_t maxh, const int32_t *__restrict__ height_lo,
                                  const int32_t *__restrict__ left, const int32_t *__restrict__ right,
                                  int32_t root, double *__restrict__ vals, double *__restrict__ out,
                                  double *__restrict__ ctl = nullptr, StepParams prm = {}, int trial = 0) {
    if (ctl && ctl[5] != 0.0) return;
    for (int32_t h = 1; h <= maxh; ++h) {
        const int32_t lo = height_lo[h - 1], hi = height_lo[h];
        for (int32_t k = lo + threadIdx.x; k < hi; k += blockDim.x)
            vals[nleaves + k] = __dadd_rn(vals[left[k]], vals[right[k]]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double res = __dadd_rn(0.0, vals[root]);
        if (ctl)
            step_decide(ctl, res, prm, trial);
        else
            out[0] = res;
    }
}

// the exact passes' watchdog word as a double, next to the bound sums the
// host reads in one copy (dm_flat_status_to)
__global__ void status_to_slot_kernel(const int *status, double *slot) { *slot = (double)*status; }

__global__ void step_init_kernel(double *ctl, double gamma) {
    ctl[0] = gamma;
    for (int i = 1; i < 8; ++i) ctl[i] = 0.0;
}

// --------------------------------------------------------------------------
// exact averaging passes
// --------------------------------------------------------------------------
__global__ void fill_kernel(double *__restrict__ x, int64_t n, double v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void roots_kernel(int32_t nb, const int32_t *__restrict__ bdd_layer_lo,
                             const int32_t *__restrict__ lnl, double *__restrict__ F) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nb) F[lnl[bdd_layer_lo[j]]] = 0.0;
}

struct MmaArgs {
    int64_t ntasks;
    const int32_t *task_layer, *task_meta;
    const int32_t *lnl, *zero_t, *one_t, *layer_bdd;
    double *lam, *F, *B, *bounds;
    int *status;                // 0 ok, 1 watchdog fired
    unsigned sleep_ns;          // back-off between unsuccessful polls
    int probe;                  // 1: poll one probe word before reading the layer; 0: poll all inputs
    unsigned long long *trace;  // optional [task*32+lane][6]: start, own inputs seen, group go, dual updated,
                                // published, issue of the successful poll
    const int32_t *task_level;  // DAG level of each task
    int *progress;              // highest level of a finished task (monotone hint)
    int lookahead;              // start polling inputs once progress >= level - lookahead (0: always)
    int warm;                   // prefetch the polled lines into L2 at task start
    int hints;                  // streaming (evict-first) loads: 1 copy records, 2 arcs, 4 the static table
    const uint64_t *relax_layer;  // per-layer source nibbles (forward, W == 8 only)
    // node-parallel kernels: task -> visitation position, its copies (CSR) and
    // per-layer first/last flags (bit 0 first layer of its BDD, bit 1 last)
    const int32_t *task_pos, *proc_ptr, *proc_layers;
    const uint8_t *layer_flags;
    // per position p, 8 copy records {layer, first node, w | wn<<8 | flags<<16 | k<<24, 0}
    const int4 *np_rec;
    int *task_counter;  // dynamic task queue of the node-parallel kernels
    uint64_t *dec;      // node-parallel backward: per layer, byte i = node i's (chosen next-layer slot << 1) | bit
};

// Progress gating: a warp whose task is far ahead of the wavefront watches a
// single word (one L2 line for all warps) instead of polling its inputs, so
// the SM's load queue stays free for the warps on the critical path.  Safe
// for lookahead >= 1: the lowest unfinished level m always sees
// progress >= m - 1.
__device__ __forceinline__ bool wait_progress(const MmaArgs &a, int64_t task, uint64_t t_start, unsigned &spins);
__device__ __forceinline__ void publish_progress(const MmaArgs &a, int64_t task, int lane) {
    if (a.lookahead > 0 && lane == 0)
        asm volatile("red.relaxed.gpu.global.max.s32 [%0], %1;" ::"l"(a.progress), "r"(a.task_level[task]) : "memory");
}

__device__ __forceinline__ void trace_mark(const MmaArgs &a, int64_t task, int lane, int slot, uint64_t t) {
    if (a.trace) a.trace[(task * 32 + lane) * 6 + slot] = t;
}

// true when this warp must abandon the pass (own timeout or another's)
__device__ __forceinline__ bool watchdog(const MmaArgs &a, uint64_t t_start, unsigned &spins) {
    if ((++spins & 63u) != 0) return false;
    if (*(volatile int *)a.status) return true;
    if (global_ns() - t_start > kWaitLimitNs) {
        atomicExch(a.status, 1);
        return true;
    }
    return false;
}

__device__ __forceinline__ bool wait_progress(const MmaArgs &a, int64_t task, uint64_t t_start, unsigned &spins) {
    if (a.lookahead <= 0) return true;
    const int need = a.task_level[task] - a.lookahead;
    if (need < 0) return true;
    while (true) {
        int p;
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(p) : "l"(a.progress) : "memory");
        if (p >= need) return true;
        if (watchdog(a, t_start, spins)) return false;
        __nanosleep(a.sleep_ns ? a.sleep_ns : 64);
    }
}

// Lanes [gbase, gbase+gcnt) hold the copies of one variable in copy order.
__device__ __forceinline__ unsigned group_mask(int32_t meta) {
    const int gbase = meta & 0xff, gcnt = (meta >> 8) & 0xff;
    return (gcnt >= 32 ? 0xffffffffu : ((1u << gcnt) - 1u)) << gbase;
}

// Leftmost minimum: keeps `a` unless `b` is strictly smaller.  Folding a
// sequence with it in any left-to-right tree returns exactly what the
// reference's sequential `if c < m: m = c` loop returns (the first element
// of minimal value), so tree reductions stay bit-identical.
__device__ __forceinline__ double lmin(double a, double b) { return (b < a) ? b : a; }

template <int N>
__device__ __forceinline__ double tree_lmin(double (&v)[N]) {
#pragma unroll
    for (int s = 1; s < N; s *= 2)
#pragma unroll
        for (int i = 0; i + s < N; i += 2 * s) v[i] = lmin(v[i], v[i + s]);
    return v[0];
}

// Sum of the finite min-marginal differences of the lane's variable in copy
// order (kernels.py:200-233) and the lane's new dual (kernels.py:234-240).
// Whole warp executes it; only lanes with `go` use the result.  The group's
// deltas are gathered with independent shuffles, then summed sequentially.
//
// Non-finite lanes contribute +0.0 instead of being skipped: the running sum
// starts at +0.0 and binary64 addition never produces -0.0 from it (exact
// cancellation gives +0.0, sums of nonzero values never round to zero), so
// adding +0.0 leaves it bit-unchanged.  Division by a power-of-two count is a
// multiplication by its exact reciprocal (both correctly rounded from the same
// real quotient); other counts take __ddiv_rn.
// 1/n for n a power of two, built from the exponent bits (no table lookup)
__device__ __forceinline__ double exact_inverse_pow2(int n) {
    return __longlong_as_double((long long)(1023 - (__ffs(n) - 1)) << 52);
}

template <int K>
__device__ __forceinline__ double average_in_group(bool go, int32_t meta, unsigned gmask, double m0, double m1,
                                                   double lam_l) {
    const bool fin = go && m0 != DM_INF && m1 != DM_INF;
    const double dlt = fin ? __dsub_rn(m1, m0) : 0.0;
    const unsigned finmask = __ballot_sync(kFull, fin);
    const int gbase = meta & 0xff, gcnt = (meta >> 8) & 0xff;
    double dk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) dk[k] = __shfl_sync(kFull, dlt, (gbase + k) & 31);
    double fsum = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (k < gcnt) fsum = __dadd_rn(fsum, dk[k]);
    const int fcnt = __popc(finmask & gmask);
    if (fin && fcnt > 0) {
        double avg;
        if ((fcnt & (fcnt - 1)) == 0)
            avg = __dmul_rn(fsum, exact_inverse_pow2(fcnt));
        else
            avg = __ddiv_rn(fsum, (double)fcnt);
        lam_l = __dadd_rn(lam_l, __dsub_rn(avg, dlt));
    }
    return lam_l;
}

// Min-marginals of one layer (kernels.py:205-230), as two leftmost-min trees
// over c0[i] = F[i] + t0[i] and c1[i] = (F[i] + lam) + t1[i].  The arc terms
// are prepared before the wait: the target's distance for an inner arc,
// -0.0 for an arc to TRUE (x + -0.0 == x bit for bit, the reference's plain
// F[i]) and +INF for an arc to FALSE or a padding node (F is never -INF or
// NaN, so the sum is +INF, a candidate that never wins — the reference's
// `continue`).
template <int W>
__device__ __forceinline__ void layer_marginals(const double (&f)[W], const double (&t0)[W],
                                                const double (&t1)[W], double lam_l, double &m0, double &m1) {
    double c0[W], c1[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
        c0[i] = __dadd_rn(f[i], t0[i]);
        c1[i] = __dadd_rn(__dadd_rn(f[i], lam_l), t1[i]);
    }
    m0 = tree_lmin<W>(c0);
    m1 = tree_lmin<W>(c1);
}

// additive arc term of layer_marginals for an arc to `t` whose distance is `d`
__device__ __forceinline__ double arc_term(int32_t t, double d) {
    return t == dm::kFalse ? DM_INF : (t == dm::kTrue ? -0.0 : d);
}

// Forward pass.  Warp w takes tasks w, w+W, ... (level order).  Inside a task
// each variable (lane group) proceeds as soon as its own inputs are
// published, independently of the other groups in the warp.
template <int W, int K, bool D = false>
__global__ void __launch_bounds__(256) mma_forward_kernel(MmaArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t task = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; task < a.ntasks; task += nwarps) {
        const int32_t l = a.task_layer[task * 32 + lane];
        const int32_t meta = a.task_meta[task * 32 + lane];
        const bool act = l >= 0;
        const bool last = meta & (1 << 17);
        const uint64_t desc = (D && act) ? a.relax_layer[l] : 0ull;
        int32_t nlo = 0, w = 0, n0 = 0, wn = 0;
        double lam_l = 0.0;
        int32_t z[W], o[W];
        double bz[W], bo[W], f[W];
        if (act) {
            nlo = a.lnl[l];
            w = a.lnl[l + 1] - nlo;
            if (!last) {
                n0 = a.lnl[l + 1];
                wn = a.lnl[l + 2] - n0;
            }
            lam_l = a.lam[l];
        }
        // static inputs: topology and the backward distances (valid all pass),
        // folded into the marginal arc terms
#pragma unroll
        for (int i = 0; i < W; ++i) {
            z[i] = o[i] = dm::kFalse;
            bz[i] = bo[i] = f[i] = DM_INF;
            if (i < w) {
                z[i] = a.zero_t[nlo + i];
                o[i] = a.one_t[nlo + i];
                bz[i] = arc_term(z[i], z[i] >= 0 ? a.B[z[i]] : 0.0);
                bo[i] = arc_term(o[i], o[i] >= 0 ? a.B[o[i]] : 0.0);
            }
        }
        // pull the lines this lane will poll into L2 while it waits
        if (a.warm && act) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.F + nlo));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.F + nlo + w - 1));
        }
        const unsigned gmask = act ? group_mask(meta) : 0u;
        bool have = !act;
        unsigned pending = __ballot_sync(kFull, act);
        unsigned spins = 0;
        const uint64_t t_wait = global_ns();
        if (act) trace_mark(a, task, lane, 0, t_wait);
        if (!wait_progress(a, task, t_wait, spins)) return;
        while (pending) {
            if (!have && ((pending >> lane) & 1u)) {
                if (!a.probe || !is_sentinel(ld_relaxed(a.F + nlo + w - 1))) {
                    const uint64_t t_issue = a.trace ? global_ns() : 0;
                    const bool ok = poll_inputs<W, true>(a.F + nlo, w, f);
                    have = ok;
                    if (ok && a.trace) {
                        trace_mark(a, task, lane, 1, global_ns());
                        trace_mark(a, task, lane, 5, t_issue);
                    }
                }
            }
            const unsigned hm = __ballot_sync(kFull, have);
            const bool go = act && ((pending >> lane) & 1u) && ((hm & gmask) == gmask);
            const unsigned gom = __ballot_sync(kFull, go);
            if (gom == 0u) {
                if (watchdog(a, t_wait, spins)) {
                    __syncwarp();
                    return;
                }
                if (a.sleep_ns) __nanosleep(a.sleep_ns);
                continue;
            }
            pending &= ~gom;
            if (go && a.trace) trace_mark(a, task, lane, 2, global_ns());
            double m0, m1;
            layer_marginals<W>(f, bz, bo, lam_l, m0, m1);
            const double lam_new = average_in_group<K>(go, meta, gmask, m0, m1, lam_l);
            if (!go) continue;
            lam_l = lam_new;
            a.lam[l] = lam_l;
            if (a.trace) trace_mark(a, task, lane, 3, global_ns());
            // propagate to the next layer (kernels.py:241-269): every target's
            // value is the leftmost minimum over (v ascending, zero-arc,
            // one-arc) of the reference's scatter, computed for all targets
            // at once.
            if (!last && D) {
                // host-built per-layer source nibbles (dm_layout.cpp
                // build_relax_by_layer): at most one zero- and one one-arc
                // source per target, so the leftmost minimum is one compare.
                double fl[W + 1];
#pragma unroll
                for (int i = 0; i < W; ++i) fl[i] = f[i];
                fl[W] = DM_INF;
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    if (u < wn) {
                        const int zi = (int)(desc >> (8 * u)) & 15, oi = (int)(desc >> (8 * u + 4)) & 15;
                        const double A = fl[zi < W ? zi : W];
                        const double C = __dadd_rn(fl[oi < W ? oi : W], lam_l);
                        st_relaxed(a.F + n0 + u, (C < A || (C == A && oi < zi)) ? C : A);
                    }
                }
                if (a.trace) trace_mark(a, task, lane, 4, global_ns());
                continue;
            }
            double c[W];
#pragma unroll
            for (int i = 0; i < W; ++i) c[i] = __dadd_rn(f[i], lam_l);
            if (!last) {
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    if (u < wn) {
                        const int32_t tgt = n0 + u;
                        double cand[2 * W];
#pragma unroll
                        for (int i = 0; i < W; ++i) {
                            cand[2 * i] = z[i] == tgt ? f[i] : DM_INF;
                            cand[2 * i + 1] = o[i] == tgt ? c[i] : DM_INF;
                        }
                        st_relaxed(a.F + tgt, tree_lmin<2 * W>(cand));
                    }
                }
            } else {
                double cand[2 * W];
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    cand[2 * i] = z[i] == dm::kTrue ? f[i] : DM_INF;
                    cand[2 * i + 1] = o[i] == dm::kTrue ? c[i] : DM_INF;
                }
                a.bounds[a.layer_bdd[l]] = tree_lmin<2 * W>(cand);
            }
            if (a.trace) trace_mark(a, task, lane, 4, global_ns());
        }
        publish_progress(a, task, lane);
    }
}

// Backward pass: mirror image; a lane waits for the distances to TRUE of the
// next layer and rebuilds its own layer's distances with the updated dual.
template <int W, int K>
__global__ void __launch_bounds__(256) mma_backward_kernel(MmaArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t task = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; task < a.ntasks; task += nwarps) {
        const int32_t l = a.task_layer[task * 32 + lane];
        const int32_t meta = a.task_meta[task * 32 + lane];
        const bool act = l >= 0;
        const bool last = meta & (1 << 17);
        int32_t nlo = 0, w = 0, probe = -1, wnext = 0, n0n = 0;
        double lam_l = 0.0;
        // per node: slot of the zero/one arc target in the next layer (W for
        // TRUE/FALSE/padding, whose slot holds -0.0), the marginal bases
        // F (zero arc) and F + lam (one arc) — +INF for FALSE arcs and padding
        // — and the rebuild offsets (see the rebuild below)
        int32_t iz[W], io[W];
        double f0[W], f1[W], rz[W], ro[W];
        double nbv[W];
        if (act) {
            nlo = a.lnl[l];
            w = a.lnl[l + 1] - nlo;
            if (!last) {
                n0n = a.lnl[l + 1];
                probe = a.lnl[l + 2] - 1;
                wnext = probe + 1 - n0n;
            }
            lam_l = a.lam[l];
        }
#pragma unroll
        for (int i = 0; i < W; ++i) {
            iz[i] = io[i] = W;
            f0[i] = f1[i] = DM_INF;
            rz[i] = ro[i] = DM_INF;
            nbv[i] = -0.0;
            if (i < w) {
                const int32_t z = a.zero_t[nlo + i], o = a.one_t[nlo + i];
                const double fv = a.F[nlo + i];
                iz[i] = z >= 0 ? ((z - n0n) & (W - 1)) : W;
                io[i] = o >= 0 ? ((o - n0n) & (W - 1)) : W;
                f0[i] = z == dm::kFalse ? DM_INF : fv;
                f1[i] = o == dm::kFalse ? DM_INF : __dadd_rn(fv, lam_l);
                rz[i] = z == dm::kFalse ? DM_INF : (z == dm::kTrue ? 0.0 : -0.0);
                ro[i] = o == dm::kFalse ? DM_INF : -0.0;
            }
        }
        if (a.warm && act && !last) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.B + a.lnl[l + 1]));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.B + probe));
        }
        const unsigned gmask = act ? group_mask(meta) : 0u;
        bool have = !act || last;
        unsigned pending = __ballot_sync(kFull, act);
        unsigned spins = 0;
        const uint64_t t_wait = global_ns();
        if (act) trace_mark(a, task, lane, 0, t_wait);
        if (!wait_progress(a, task, t_wait, spins)) return;
        while (pending) {
            if (!have && ((pending >> lane) & 1u)) {
                if (!a.probe || !is_sentinel(ld_relaxed(a.B + probe))) {
                    // read the next layer contiguously (like the forward pass reads
                    // its own layer); routing to the arc targets happens once, at go
                    const uint64_t t_issue = a.trace ? global_ns() : 0;
                    const bool ok = poll_inputs<W, false>(a.B + n0n, wnext, nbv);
                    have = ok;
                    if (ok && a.trace) {
                        trace_mark(a, task, lane, 1, global_ns());
                        trace_mark(a, task, lane, 5, t_issue);
                    }
                }
            }
            const unsigned hm = __ballot_sync(kFull, have);
            const bool go = act && ((pending >> lane) & 1u) && ((hm & gmask) == gmask);
            const unsigned gom = __ballot_sync(kFull, go);
            if (gom == 0u) {
                if (watchdog(a, t_wait, spins)) {
                    __syncwarp();
                    return;
                }
                if (a.sleep_ns) __nanosleep(a.sleep_ns);
                continue;
            }
            pending &= ~gom;
            if (go && a.trace) trace_mark(a, task, lane, 2, global_ns());
            // route the next layer's distances to the arc targets through a
            // dynamically indexed (local-memory, L1-resident) copy: measured
            // 20% faster per pass than W x W register selects.  Slot W holds
            // -0.0, the term of arcs to a terminal.
            double tz[W], to[W];
            {
                double nbl[W + 1];
#pragma unroll
                for (int u = 0; u < W; ++u) nbl[u] = nbv[u];
                nbl[W] = -0.0;
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    tz[i] = nbl[iz[i]];
                    to[i] = nbl[io[i]];
                }
            }
            double m0, m1;
            {
                double c0[W], c1[W];
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    c0[i] = __dadd_rn(f0[i], tz[i]);
                    c1[i] = __dadd_rn(f1[i], to[i]);
                }
                m0 = tree_lmin<W>(c0);
                m1 = tree_lmin<W>(c1);
            }
            const double lam_new = average_in_group<K>(go, meta, gmask, m0, m1, lam_l);
            if (!go) continue;
            lam_l = lam_new;
            a.lam[l] = lam_l;
            if (a.trace) trace_mark(a, task, lane, 3, global_ns());
            // rebuild this layer's distances to TRUE (kernels.py:340-358):
            //   zero arc: B[z] (inner), +0.0 (TRUE), +INF (FALSE)  = rz + tz
            //   one arc : lam + B[o], lam, +INF                    = (lam + to) + ro
            // (x + -0.0 == x; +0.0 + -0.0 == +0.0; INF + finite == INF)
            double first = 0.0;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                if (i < w) {
                    const double c0 = __dadd_rn(rz[i], tz[i]);
                    const double c1 = __dadd_rn(__dadd_rn(lam_l, to[i]), ro[i]);
                    const double bv = (c0 <= c1) ? c0 : c1;
                    st_relaxed(a.B + nlo + i, bv);
                    if (i == 0) first = bv;
                }
            }
            if (meta & (1 << 16)) a.bounds[a.layer_bdd[l]] = first;  // kernels.py:359-361
            if (a.trace) trace_mark(a, task, lane, 4, global_ns());
        }
        publish_progress(a, task, lane);
    }
}

// ===========================================================================
// Node-parallel exact passes: one warp task per visitation position (one
// variable), 4 lanes per BDD copy, 2 nodes per lane (layers up to 8 nodes,
// up to 8 copies).  Lane 4c+q handles nodes 2q, 2q+1 of copy c's layer.
// Same DAG schedule, same arithmetic and reduction trees as the per-copy
// kernels above — the min trees are split across the copy's 4 lanes with
// xor shuffles that keep tree_lmin<8>'s shape — so the duals are
// bit-identical; a task's post-wait work is ~4x fewer instructions and runs
// once (one group per warp).
// ===========================================================================
constexpr int kNpCopies = 8;

__device__ __forceinline__ void np_trace(const MmaArgs &a, int64_t task, int c, int q, int slot, uint64_t t) {
    if (a.trace && q == 0) a.trace[(task * kNpCopies + c) * 6 + slot] = t;
}

// leftmost min across the 4 lanes of a copy (lower lane = lower node index)
__device__ __forceinline__ double np_lmin4(double v, int q) {
#pragma unroll
    for (int s = 1; s < 4; s <<= 1) {
        const double o = __shfl_xor_sync(kFull, v, s);
        v = (q & s) ? lmin(o, v) : lmin(v, o);
    }
    return v;
}

// value of node i (0..7) of copy c from the lane pair that holds it
__device__ __forceinline__ double np_node(double v0, double v1, int c, int i) {
    const int src = 4 * c + ((i >> 1) & 3);
    const double a = __shfl_sync(kFull, v0, src), b = __shfl_sync(kFull, v1, src);
    return (i & 1) ? b : a;
}

// Division of the copy-delta sum by the copy count, prepared before the
// wait: the count of a task's copies is known from its record, so the
// reciprocal is ready when the sum arrives.  Powers of two multiply by their
// exact reciprocal; other counts (3, 5, 6, 7) take Markstein's correction:
// with y = RN(1/k) and q = RN(a*y) (within one ulp of a/k), the residual
// r = a - q*k is exact in one fma and RN(q + r*y) = RN(a/k) — the quotient
// of a normal a by k = 2^s * odd is either exact or has an infinite binary
// expansion, so it is never a rounding tie.  Sums below 2^-960 (where the
// intermediate could leave the normal range) take __ddiv_rn.
// tests/test_gpu_parity.py checks it against __ddiv_rn (dm_debug_div_check).
struct NpDiv {
    double r, kd;
    bool pow2;
};

__device__ __forceinline__ NpDiv np_div(int k) {
    NpDiv d;
    k = max(k, 1);
    d.kd = (double)k;
    d.pow2 = (k & (k - 1)) == 0;
    d.r = d.pow2 ? exact_inverse_pow2(k) : __ddiv_rn(1.0, d.kd);
    return d;
}

__device__ __forceinline__ double div_by_count(double a, const NpDiv &d) {
    if (d.pow2) return __dmul_rn(a, d.r);
    if (fabs(a) < 0x1p-960) return __ddiv_rn(a, d.kd);
    const double q = __dmul_rn(a, d.r);
    const double res = __fma_rn(-q, d.kd, a);
    return res == 0.0 ? q : __fma_rn(res, d.r, q);
}

// Sequential sum of the copies' deltas in copy order + the new dual, as
// average_in_group (same +0.0 / exact-reciprocal identities).  The deltas
// are gathered with shuffles; copy slots j >= k belong to inactive lanes and
// hold +0.0, so all eight are added unconditionally (bit-neutral, and no
// select on the dependent chain: tools/workbench.cu measured 461 -> 369
// cycles per task).  `dv` is np_div(k): when every copy is finite (the common
// case, decided by a warp-uniform count) the divisor is the one prepared
// before the wait.
__device__ __forceinline__ double np_average(bool act, int k, int q, double m0, double m1, double lam_l,
                                             const NpDiv &dv) {
    const bool fin = act && m0 != DM_INF && m1 != DM_INF;
    const double dlt = fin ? __dsub_rn(m1, m0) : 0.0;
    const unsigned finmask = __ballot_sync(kFull, fin && q == 0);
    double dk[kNpCopies];
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j) dk[j] = __shfl_sync(kFull, dlt, 4 * j);
    double fsum = 0.0;
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j) fsum = __dadd_rn(fsum, dk[j]);
    const int fcnt = __popc(finmask);  // warp-uniform
    double avg = 0.0;
    if (fcnt == k)
        avg = div_by_count(fsum, dv);
    else if (fcnt > 0)
        avg = (fcnt & (fcnt - 1)) == 0 ? __dmul_rn(fsum, exact_inverse_pow2(fcnt)) : __ddiv_rn(fsum, (double)fcnt);
    return fin ? __dadd_rn(lam_l, __dsub_rn(avg, dlt)) : lam_l;
}

// dm_debug_div_check: div_by_count against __ddiv_rn on hashed doubles
// spanning the exponent range, plus scaled small integers
__global__ void div_check_kernel(int k, uint64_t n, uint64_t seed, unsigned long long *mismatches) {
    const NpDiv dv = np_div(k);
    unsigned long long bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = (i + seed) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        double a;
        if (i & 1) {
            const uint64_t e = 1 + (h >> 53) % 2045;  // normal exponents
            a = __longlong_as_double((long long)(((h & 1) << 63) | (e << 52) | ((h >> 1) & 0xfffffffffffffull)));
        } else {
            a = (double)(int64_t)((h >> 40) - (1ull << 23)) * __longlong_as_double((long long)((1023 + (int)((h >> 8) & 63) - 32) << 52 & 0x7ff0000000000000ll));
        }
        const double got = div_by_count(a, dv), want = __ddiv_rn(a, (double)k);
        if (__double_as_longlong(got) != __double_as_longlong(want)) ++bad;
    }
    if (bad) atomicAdd(mismatches, bad);
}

struct NpLane {
    int c, q, k;
    bool act, first, last;
    int32_t l, nlo, w;
};

struct NpLaneX : NpLane {
    int32_t wn;  // width of the next layer (0 for a last layer)
};

// One load per task and copy: the packed record, stored in task order.
// watchdog with a lazily taken start time (no %globaltimer read per task)
__device__ __forceinline__ bool np_watchdog(const MmaArgs &a, uint64_t &t_start, unsigned &spins) {
    if ((++spins & 63u) != 0) return false;
    if (*(volatile int *)a.status) return true;
    const uint64_t now = global_ns();
    if (t_start == 0) t_start = now;
    if (now - t_start > kWaitLimitNs) {
        atomicExch(a.status, 1);
        return true;
    }
    return false;
}

__device__ __forceinline__ NpLaneX np_lane(const MmaArgs &a, int64_t task, int lane) {
    NpLaneX r;
    r.c = lane >> 2;
    r.q = lane & 3;
    const int4 *rp = a.np_rec + task * kNpCopies + r.c;  // records stored in this pass's task order
    const int4 rec = (a.hints & 1) ? __ldcs(rp) : *rp;
    const unsigned m = (unsigned)rec.z;
    r.k = (int)(m >> 24);
    r.act = r.c < r.k;
    r.l = rec.x;
    r.nlo = rec.y;
    r.w = (int)(m & 0xff);
    r.wn = (int)((m >> 8) & 0xff);
    r.first = (m >> 16) & 1;
    r.last = (m >> 17) & 1;
    return r;
}

// Next task of this warp from the pass's queue (tasks are level-ordered, so a
// warp only ever waits on tasks already taken by running warps).
__device__ __forceinline__ int64_t np_next_task(const MmaArgs &a, int lane) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.task_counter, 1);
    return __shfl_sync(kFull, t, 0);
}

// Per warp: node values of each copy (9 slots, slot 8 the arc-to-nothing
// value) in shared memory.
constexpr int kNpWarps = 8;  // 256-thread blocks
struct NpShared {
    double node[kNpWarps][kNpCopies][9];
};

// Poll loop of the node-parallel kernels (needs `have`, `take`, `a`, `t_wait`,
// `spins`).  A value read as non-sentinel is final (each is written once per
// pass).  (Two interleaved poll streams offset by half a round trip measured
// 15% slower: the doubled poll traffic costs more than the earlier detection.)
#define NP_POLL_LOOP(SRC0, SRC1, PAIR)                                                        \
    while (true) {                                                                      \
        if (!have) {                                                                    \
            const uint64_t t_issue = a.trace ? global_ns() : 0;                         \
            double v0, v1;                                                              \
            if (PAIR) ld_relaxed_pair(SRC0, SRC1, v0, v1);                              \
            else v0 = ld_relaxed(SRC0), v1 = ld_relaxed(SRC1);                          \
            take(v0, v1, t_issue);                                                      \
        }                                                                               \
        if (__all_sync(kFull, have)) break;                                             \
        if (__any_sync(kFull, np_watchdog(a, t_wait, spins))) return;                   \
        if (a.sleep_ns) __nanosleep(a.sleep_ns);                                        \
    }

template <bool D>
__global__ void __launch_bounds__(256) mma_np_forward_kernel(MmaArgs a) {
    __shared__ NpShared sh;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int64_t task = np_next_task(a, lane); task < a.ntasks; task = np_next_task(a, lane)) {
        __syncwarp();  // the previous task's shared-memory reads are done
        const NpLaneX r = np_lane(a, task, lane);
        const NpDiv dv = np_div(r.k);
        double *nodes = sh.node[wib][r.c];
        const int i0 = 2 * r.q, i1 = i0 + 1;
        int32_t n0 = 0, wn = 0;
        double lam_l = 0.0;
        int32_t z0 = dm::kFalse, z1 = dm::kFalse, o0 = dm::kFalse, o1 = dm::kFalse;
        uint64_t desc = 0;
        if (r.act) {
            if (!r.last) {
                n0 = r.nlo + r.w;
                wn = r.wn;
                if (D) desc = a.relax_layer[r.l];
            }
            lam_l = a.lam[r.l];
            if (a.hints & 2) {
                if (i0 < r.w) z0 = __ldcs(a.zero_t + r.nlo + i0), o0 = __ldcs(a.one_t + r.nlo + i0);
                if (i1 < r.w) z1 = __ldcs(a.zero_t + r.nlo + i1), o1 = __ldcs(a.one_t + r.nlo + i1);
            } else {
                if (i0 < r.w) z0 = a.zero_t[r.nlo + i0], o0 = a.one_t[r.nlo + i0];
                if (i1 < r.w) z1 = a.zero_t[r.nlo + i1], o1 = a.one_t[r.nlo + i1];
            }
        }
        // marginal arc terms (see layer_marginals): +INF FALSE/padding, -0.0 TRUE
        auto bt = [&](int32_t t) { return t >= 0 ? ((a.hints & 4) ? __ldcs(a.B + t) : a.B[t]) : 0.0; };
        const double t00 = arc_term(z0, bt(z0)), t01 = arc_term(z1, bt(z1));
        const double t10 = arc_term(o0, bt(o0)), t11 = arc_term(o1, bt(o1));
        double f0 = DM_INF, f1 = DM_INF;
        bool have = !r.act || i0 >= r.w;
        nodes[i0] = DM_INF;
        nodes[i1] = DM_INF;
        if (r.q == 0) nodes[8] = DM_INF;
        unsigned spins = 0;
        uint64_t t_wait = 0;
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 0, global_ns());
        const double *src0 = a.F + r.nlo + (i0 < r.w ? i0 : 0), *src1 = a.F + r.nlo + (i1 < r.w ? i1 : i0 < r.w ? i0 : 0);
        auto take = [&](double v0, double v1, uint64_t t_issue) {
            if (have || is_sentinel(v0) || is_sentinel(v1)) return;
            have = true;
            f0 = v0;
            f1 = i1 < r.w ? v1 : DM_INF;
            nodes[i0] = f0;
            nodes[i1] = f1;
            if (a.trace) {
                np_trace(a, task, r.c, r.q, 1, global_ns());
                np_trace(a, task, r.c, r.q, 5, t_issue);
            }
        };
        NP_POLL_LOOP(src0, src1, true)  // 16-byte polls where aligned: forward 4.41 -> 4.33 ms
        __syncwarp();  // the node rows written by `take` are visible to the publish below
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 2, global_ns());
        // min-marginals over the layer (tree_lmin<8> split over the 4 lanes)
        const double m0 = np_lmin4(lmin(__dadd_rn(f0, t00), __dadd_rn(f1, t01)), r.q);
        const double m1 = np_lmin4(lmin(__dadd_rn(__dadd_rn(f0, lam_l), t10), __dadd_rn(__dadd_rn(f1, lam_l), t11)), r.q);
        lam_l = np_average(r.act, r.k, r.q, m0, m1, lam_l, dv);
        if (r.act && r.q == 0) a.lam[r.l] = lam_l;
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 3, global_ns());
        const double c0 = __dadd_rn(f0, lam_l), c1 = __dadd_rn(f1, lam_l);
        if (D) {
            // targets 2q, 2q+1 of the next layer from the per-layer source nibbles
            double out[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int u = i0 + j;
                const int zi = (int)(desc >> (8 * u)) & 15, oi = (int)(desc >> (8 * u + 4)) & 15;
                const double A = nodes[zi < 8 ? zi : 8];                  // slot 8: +INF
                const double C = __dadd_rn(nodes[oi < 8 ? oi : 8], lam_l);  // +INF + lam = +INF
                out[j] = (C < A || (C == A && oi < zi)) ? C : A;
            }
            // one 16-byte store where the pair is aligned: 4.33 -> 4.17 ms
            if (r.act && !r.last) st_relaxed_pair(a.F + n0 + i0, out[0], out[1], min(wn - i0, 2));
        } else {
            // generic scatter: every target is the leftmost minimum over (node
            // ascending, zero arc, one arc), gathered from all 8 nodes
            double fv[8], cv[8];
            int32_t zv[8], ov[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                fv[i] = np_node(f0, f1, r.c, i);
                cv[i] = np_node(c0, c1, r.c, i);
                const int src = 4 * r.c + (i >> 1);
                const int32_t za = __shfl_sync(kFull, z0, src), zb = __shfl_sync(kFull, z1, src);
                const int32_t oa = __shfl_sync(kFull, o0, src), ob = __shfl_sync(kFull, o1, src);
                zv[i] = (i & 1) ? zb : za;
                ov[i] = (i & 1) ? ob : oa;
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int u = i0 + j;
                const int32_t tgt = n0 + u;
                double cand[16];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cand[2 * i] = zv[i] == tgt ? fv[i] : DM_INF;
                    cand[2 * i + 1] = ov[i] == tgt ? cv[i] : DM_INF;
                }
                const double v = tree_lmin<16>(cand);
                if (r.act && !r.last && u < wn) st_relaxed(a.F + tgt, v);
            }
        }
        if (__any_sync(kFull, r.act && r.last)) {
            // bound of a diagram whose last layer this is: leftmost min over
            // (node, zero arc, one arc) of the arcs into TRUE (tree_lmin<16>
            // split over the 4 lanes; every lane shuffles, the warp stays converged)
            const double a0 = z0 == dm::kTrue ? f0 : DM_INF, b0 = o0 == dm::kTrue ? c0 : DM_INF;
            const double a1 = z1 == dm::kTrue ? f1 : DM_INF, b1 = o1 == dm::kTrue ? c1 : DM_INF;
            const double bound = np_lmin4(lmin(lmin(a0, b0), lmin(a1, b1)), r.q);
            if (r.act && r.last && r.q == 0) a.bounds[a.layer_bdd[r.l]] = bound;
        }
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 4, global_ns());
    }
}

__global__ void __launch_bounds__(256) mma_np_backward_kernel(MmaArgs a) {
    __shared__ NpShared sh;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int64_t task = np_next_task(a, lane); task < a.ntasks; task = np_next_task(a, lane)) {
        __syncwarp();  // the previous task's shared-memory reads are done
        const NpLaneX r = np_lane(a, task, lane);
        const NpDiv dv = np_div(r.k);
        double *nodes = sh.node[wib][r.c];  // next layer's distances, slot 8 = -0.0
        const int i0 = 2 * r.q, i1 = i0 + 1;
        int32_t n0n = 0, wnext = 0;
        double lam_l = 0.0;
        if (r.act) {
            if (!r.last) {
                n0n = r.nlo + r.w;
                wnext = r.wn;
            }
            lam_l = a.lam[r.l];
        }
        // per node: next-layer slot of each arc (8 = terminal/padding: -0.0),
        // marginal bases and rebuild offsets as in mma_backward_kernel
        int iz[2] = {8, 8}, io[2] = {8, 8};
        int32_t zt[2] = {dm::kFalse, dm::kFalse}, ot[2] = {dm::kFalse, dm::kFalse};
        double f0b[2] = {DM_INF, DM_INF}, f1b[2] = {DM_INF, DM_INF}, rz[2] = {DM_INF, DM_INF},
               ro[2] = {DM_INF, DM_INF};
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int i = i0 + j;
            if (r.act && i < r.w) {
                const int32_t z = (a.hints & 2) ? __ldcs(a.zero_t + r.nlo + i) : a.zero_t[r.nlo + i];
                const int32_t o = (a.hints & 2) ? __ldcs(a.one_t + r.nlo + i) : a.one_t[r.nlo + i];
                const double fv = (a.hints & 4) ? __ldcs(a.F + r.nlo + i) : a.F[r.nlo + i];
                zt[j] = z;
                ot[j] = o;
                iz[j] = z >= 0 ? ((z - n0n) & 7) : 8;
                io[j] = o >= 0 ? ((o - n0n) & 7) : 8;
                f0b[j] = z == dm::kFalse ? DM_INF : fv;
                f1b[j] = o == dm::kFalse ? DM_INF : __dadd_rn(fv, lam_l);
                rz[j] = z == dm::kFalse ? DM_INF : (z == dm::kTrue ? 0.0 : -0.0);
                ro[j] = o == dm::kFalse ? DM_INF : -0.0;
            }
        }
        // this lane polls next-layer nodes 2q, 2q+1
        double nb0 = -0.0, nb1 = -0.0;
        bool have = !r.act || r.last || i0 >= wnext;
        nodes[i0] = -0.0;
        nodes[i1] = -0.0;
        if (r.q == 0) nodes[8] = -0.0;
        unsigned spins = 0;
        uint64_t t_wait = 0;
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 0, global_ns());
        const double *src0 = a.B + n0n + (i0 < wnext ? i0 : 0);
        const double *src1 = a.B + n0n + (i1 < wnext ? i1 : i0 < wnext ? i0 : 0);
        auto take = [&](double v0, double v1, uint64_t t_issue) {
            if (have || is_sentinel(v0) || is_sentinel(v1)) return;
            have = true;
            nb0 = v0;
            nb1 = i1 < wnext ? v1 : -0.0;
            nodes[i0] = nb0;
            nodes[i1] = nb1;
            if (a.trace) {
                np_trace(a, task, r.c, r.q, 1, global_ns());
                np_trace(a, task, r.c, r.q, 5, t_issue);
            }
        };
        NP_POLL_LOOP(src0, src1, false)  // (16-byte polls measured 4.91 -> 4.97 ms here)
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 2, global_ns());
        // route the next layer's distances to this lane's arcs (slot 8: -0.0)
        __syncwarp();
        double tz[2], to[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            tz[j] = nodes[iz[j]];
            to[j] = nodes[io[j]];
        }
        const double m0 = np_lmin4(lmin(__dadd_rn(f0b[0], tz[0]), __dadd_rn(f0b[1], tz[1])), r.q);
        const double m1 = np_lmin4(lmin(__dadd_rn(f1b[0], to[0]), __dadd_rn(f1b[1], to[1])), r.q);
        lam_l = np_average(r.act, r.k, r.q, m0, m1, lam_l, dv);
        if (r.act && r.q == 0) a.lam[r.l] = lam_l;
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 3, global_ns());
        // rebuild this layer's distances to TRUE (kernels.py:340-358)
        uint32_t db = 0;  // this lane's two decision bytes
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int i = i0 + j;
            if (r.act && i < r.w) {
                const double cz = __dadd_rn(rz[j], tz[j]);
                const double co = __dadd_rn(__dadd_rn(lam_l, to[j]), ro[j]);
                const bool zero_wins = cz <= co;
                const double bv = zero_wins ? cz : co;
                st_relaxed(a.B + r.nlo + i, bv);  // (16-byte pair stores measured 4.87 -> 5.09 ms here)
                // the argmin walk's decision at this node (kernels.py:402-431 on
                // the final duals and distances: same operands, same compare)
                const int32_t t = zero_wins ? zt[j] : ot[j];
                db |= (uint32_t)(((t >= 0 ? t - n0n : 0) << 1) | (zero_wins ? 0 : 1)) << (8 * j);
                if (i == 0 && r.first) a.bounds[a.layer_bdd[r.l]] = bv;  // kernels.py:359-361
            }
        }
        if (a.dec) {
            // the copy's eight decision bytes meet in lane q == 0: one aligned
            // 8-byte store per layer instead of a byte store per node
            uint64_t w = (uint64_t)db << (16 * r.q);
            w |= __shfl_xor_sync(kFull, w, 1);
            w |= __shfl_xor_sync(kFull, w, 2);
            if (r.act && r.q == 0) a.dec[r.l] = w;
        }
        if (a.trace && r.act) np_trace(a, task, r.c, r.q, 4, global_ns());
    }
}

}  // namespace

// ===========================================================================
// device handle
// ===========================================================================
struct DevPlan {
    int64_t n = 0;
    int32_t nleaves = 0, maxh = 0, root = 0;
    int64_t *leaf_off = nullptr;
    int32_t *leaf_len = nullptr, *left = nullptr, *right = nullptr, *height_lo = nullptr;
    double *vals = nullptr;
};

struct dm_flat {
    int device = 0;
    int64_t nb = 0, L = 0, N = 0, P = 0;
    int32_t *bdd_layer_lo = nullptr, *lnl = nullptr, *layer_bdd = nullptr, *layer_var = nullptr;
    int32_t *zero_t = nullptr, *one_t = nullptr, *proc_ptr = nullptr, *proc_layers = nullptr;
    int32_t *pos_var = nullptr, *var_count = nullptr;
    int32_t *fw_layer = nullptr, *fw_meta = nullptr, *bw_layer = nullptr, *bw_meta = nullptr;
    int64_t fw_tasks = 0, bw_tasks = 0, fw_depth = 0, bw_depth = 0;
    int64_t max_width = 0, max_degree = 0;
    int *status = nullptr;  // device watchdog word of the exact passes
    int *progress = nullptr;  // progress hint word of the exact passes
    int32_t *fw_task_level = nullptr, *bw_task_level = nullptr;
    int mma_lookahead = 0;
    int mma_warm = 1;
    uint64_t *relax_layer = nullptr;  // forward publish descriptors (W == 8 instances)
    bool relax_ok = false;
    bool mma_desc = true;
    // node-parallel exact passes (layers <= 8 nodes, <= 8 copies per variable)
    bool np_ok = false, mma_np = false;
    int32_t *fw_pos = nullptr, *bw_pos = nullptr;
    uint8_t *layer_flags = nullptr;
    int4 *np_rec_fw = nullptr, *np_rec_bw = nullptr;  // copy records in each pass's task order
    uint64_t *dec = nullptr;         // decisions of the last node-parallel backward pass (one word per layer)
    const double *dec_B = nullptr;   // ... and the distance table it wrote (nullptr: none)
    int64_t np_fw_tasks = 0, np_bw_tasks = 0;
    int32_t *fw_lev = nullptr, *bw_lev = nullptr;  // levels of fw_pos / bw_pos (device)
    int mma_w = 8, mma_k = 8;
    int mma_threads = 256, mma_blocks_per_sm = 0;
    unsigned mma_sleep_ns = 0;
    int mma_probe = 0;
    unsigned long long *trace = nullptr;
    std::vector<int32_t> fw_level, bw_level;  // host copy: DAG level of each task
    std::vector<int32_t> fw_layer_h, bw_layer_h;  // host copy of the lane layers (profiling, lazy upload)
    std::vector<int32_t> fw_meta_h, bw_meta_h;    // per-copy kernel lane metadata (lazy upload)
    bool classic_uploaded = false;
    int mma_grid_fw = 0, mma_grid_bw = 0;
    int64_t bytes = 0;
    bool exact_plans = true;  // false: created with DM_FLAT_NO_EXACT_PLANS (no exact averaging passes)
    dm::SweepDev sweep;  // interleaved layout for the full-table sweeps
    std::vector<void *> allocs;
};

namespace {

thread_local std::string g_cuda_err;

int cuda_fail(cudaError_t e, const char *what) {
    dm::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DM_ERR_CUDA;
}
#define DM_CUDA(call)                                  \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// Instance arrays come from the device's stream-ordered pool, which keeps
// freed blocks (release threshold raised once): re-creating a flat for the
// next solve reuses them instead of paying cudaMalloc again.
void keep_pool_memory(int device) {
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[device] = true;
}

template <typename T>
int upload(dm_flat *f, T **dst, const T *src, int64_t n, cudaStream_t s) {
    size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
    DM_CUDA(cudaMallocAsync((void **)dst, bytes, s));
    f->allocs.push_back(*dst);
    f->bytes += bytes;
    if (n > 0 && src) DM_CUDA(cudaMemcpyAsync(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return DM_OK;
}

// Host -> device staging through a small ring of pinned slots.  Copies from
// pageable memory go through the driver's own bounce buffer one chunk at a
// time (measured ~0.2 s for the C2 topology); here host threads fill a pinned
// slot (converting int64 -> int32 on the way where the device layout is
// narrower) while the copy engine drains the previous ones.  Rings are pooled
// for the process lifetime; concurrent creates each take their own.
constexpr size_t kStageSlotBytes = size_t(16) << 20;
constexpr int kStageSlots = 4;
constexpr int kStageFillThreads = 8;
struct StageRing {
    int device = -1;
    char *buf = nullptr;
    cudaEvent_t ev[kStageSlots] = {};
};
std::mutex g_ring_mu;
std::vector<StageRing *> g_rings;

class Stager {
  public:
    Stager(int device, cudaStream_t s) : s_(s) {
        {
            std::lock_guard<std::mutex> lk(g_ring_mu);
            for (size_t i = 0; i < g_rings.size(); ++i)
                if (g_rings[i]->device == device) {
                    ring_ = g_rings[i];
                    g_rings.erase(g_rings.begin() + i);
                    break;
                }
        }
        if (!ring_) {
            auto *r = new StageRing;
            r->device = device;
            if (cudaHostAlloc((void **)&r->buf, kStageSlotBytes * kStageSlots, cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                delete r;
                return;
            }
            for (auto &e : r->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            ring_ = r;
        }
    }
    ~Stager() {
        if (!ring_) return;
        for (auto &e : ring_->ev) cudaEventSynchronize(e);  // the slots are free again
        std::lock_guard<std::mutex> lk(g_ring_mu);
        g_rings.push_back(ring_);
    }
    // device array of n elements of T; element i is produced by
    // fill(T *dst, int64_t first, int64_t count) writing elements
    // [first, first + count) to dst (run on up to kStageFillThreads threads per slot)
    template <typename T, typename Fill>
    int put(dm_flat *f, T **dst, int64_t n, Fill &&fill) {
        int rc = upload(f, dst, (const T *)nullptr, n, s_);
        if (rc) return rc;
        if (!ring_) {  // no pinned memory: fill a pageable buffer and copy from it
            std::vector<T> tmp(std::max<int64_t>(n, 0));
            if (n > 0) {
                fill(tmp.data(), 0, n);
                DM_CUDA(cudaMemcpyAsync(*dst, tmp.data(), n * sizeof(T), cudaMemcpyHostToDevice, s_));
                DM_CUDA(cudaStreamSynchronize(s_));
            }
            return DM_OK;
        }
        const int64_t per = (int64_t)(kStageSlotBytes / sizeof(T));
        for (int64_t lo = 0; lo < n; lo += per) {
            const int64_t cnt = std::min(per, n - lo);
            const int slot = next_++ % kStageSlots;
            DM_CUDA(cudaEventSynchronize(ring_->ev[slot]));
            T *buf = (T *)(ring_->buf + slot * kStageSlotBytes);
            const int nt = cnt * (int64_t)sizeof(T) >= (int64_t(1) << 20) ? kStageFillThreads : 1;
            if (nt == 1) {
                fill(buf, lo, cnt);
            } else {
                std::thread th[kStageFillThreads];
                for (int t = 0; t < nt; ++t) {
                    const int64_t a = cnt * t / nt, b = cnt * (t + 1) / nt;
                    th[t] = std::thread([&, a, b] { fill(buf + a, lo + a, b - a); });
                }
                for (int t = 0; t < nt; ++t) th[t].join();
            }
            DM_CUDA(cudaMemcpyAsync(*dst + lo, buf, cnt * sizeof(T), cudaMemcpyHostToDevice, s_));
            DM_CUDA(cudaEventRecord(ring_->ev[slot], s_));
        }
        return DM_OK;
    }
    template <typename T>
    int copy(dm_flat *f, T **dst, const T *src, int64_t n) {
        return put(f, dst, n, [src](T *d, int64_t lo, int64_t c) { std::memcpy(d, src + lo, c * sizeof(T)); });
    }
    int narrow(dm_flat *f, int32_t **dst, const int64_t *src, int64_t n) {
        return put(f, dst, n, [src](int32_t *d, int64_t lo, int64_t c) {
            for (int64_t i = 0; i < c; ++i) d[i] = (int32_t)src[lo + i];
        });
    }

  private:
    cudaStream_t s_;
    StageRing *ring_ = nullptr;
    int next_ = 0;
};

// Pairwise plans are cached per (device, length, stream) for the process
// lifetime: a plan's value scratch belongs to one stream, so instances solved
// concurrently on different streams never share it.
std::mutex g_plan_mu;
using ScratchKey = std::tuple<int, int64_t, uintptr_t>;
std::map<ScratchKey, DevPlan> g_plans;

template <typename T>
int plan_upload(T **dst, const std::vector<T> &src, size_t extra = 0) {
    size_t n = src.size() + extra;
    DM_CUDA(cudaMalloc((void **)dst, std::max<size_t>(n, 1) * sizeof(T)));
    if (!src.empty()) DM_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    return DM_OK;
}

int get_plan(int64_t n, cudaStream_t stream, DevPlan **out) {
    int dev;
    DM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_plan_mu);
    auto key = ScratchKey(dev, n, (uintptr_t)stream);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
        *out = &it->second;
        return DM_OK;
    }
    dm::PairwisePlan p = dm::plan_pairwise(n);
    DevPlan d;
    d.n = n;
    d.nleaves = (int32_t)p.leaf_off.size();
    d.maxh = (int32_t)p.height_lo.size() - 1;
    d.root = p.root;
    int rc;
    if ((rc = plan_upload(&d.leaf_off, p.leaf_off))) return rc;
    if ((rc = plan_upload(&d.leaf_len, p.leaf_len))) return rc;
    if ((rc = plan_upload(&d.left, p.left))) return rc;
    if ((rc = plan_upload(&d.right, p.right))) return rc;
    if ((rc = plan_upload(&d.height_lo, p.height_lo))) return rc;
    if ((rc = plan_upload(&d.vals, std::vector<double>(), p.leaf_off.size() + p.left.size()))) return rc;
    auto res = g_plans.emplace(key, d);
    *out = &res.first->second;
    return DM_OK;
}

inline int blocks_for(int64_t n, int threads) { return (int)std::max<int64_t>(1, (n + threads - 1) / threads); }
inline int grid_stride_blocks(int64_t n) { return (int)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (n + 255) / 256)); }

// The descriptor-driven forward publish is a separate instantiation, used only
// when every non-final layer of the instance has one source per arc kind.
template <int W, int K>
const void *mma_fn(const dm_flat *f, bool forward) {
    if constexpr (W == 8 && K == 8) {
        if (f->mma_np) {
            if (!forward) return (const void *)mma_np_backward_kernel;
            return f->relax_ok && f->mma_desc ? (const void *)mma_np_forward_kernel<true>
                                              : (const void *)mma_np_forward_kernel<false>;
        }
    }
    if (!forward) return (const void *)mma_backward_kernel<W, K>;
    if constexpr (W == 8) {
        if (f->relax_ok && f->mma_desc) return (const void *)mma_forward_kernel<8, K, true>;
    }
    return (const void *)mma_forward_kernel<W, K, false>;
}

template <int W, int K>
int launch_mma(const dm_flat *f, bool forward, MmaArgs &args, cudaStream_t s) {
    void *params[] = {&args};
    const void *fn = mma_fn<W, K>(f, forward);
    const int grid = forward ? f->mma_grid_fw : f->mma_grid_bw;
    DM_CUDA(cudaLaunchCooperativeKernel(fn, grid, f->mma_threads, params, 0, s));
    return DM_OK;
}

// Persistent grid: min(requested, resident) blocks per SM x SM count.
template <int W, int K>
int mma_grid_for(const dm_flat *f, bool forward, int threads, int want_per_sm, int *grid) {
    int dev, sms, per;
    DM_CUDA(cudaGetDevice(&dev));
    DM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const void *fn = mma_fn<W, K>(f, forward);
    DM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, 0));
    if (per < 1) {
        dm::set_error("exact averaging kernel cannot be resident");
        return DM_ERR_CUDA;
    }
    if (want_per_sm > 0) per = std::min(per, want_per_sm);
    *grid = sms * per;
    if (const char *cap = std::getenv("DM_MMA_MAX_BLOCKS"))  // profiling: shrink the persistent grid
        if (std::atoi(cap) > 0) *grid = std::min(*grid, std::atoi(cap));
    return DM_OK;
}

}  // namespace

// Instantiations: W = widest layer (8/16/32), K = most copies per variable (8/32).
#define DM_MMA_DISPATCH(f, CALL)                                  \
    (f->mma_k <= 8 ? (f->mma_w == 8 ? CALL(8, 8) : f->mma_w == 16 ? CALL(16, 8) : CALL(32, 8)) \
                   : (f->mma_w == 8 ? CALL(8, 32) : f->mma_w == 16 ? CALL(16, 32) : CALL(32, 32)))

// The per-copy kernels' warp tasks are packed and uploaded the first time
// those kernels are selected (the node-parallel ones need only positions).
static int ensure_per_copy_schedules(dm_flat *f, cudaStream_t s) {
    if (f->classic_uploaded) return DM_OK;
    const int64_t n = f->np_fw_tasks;
    std::vector<int32_t> fpos(n), flev(n), bpos(n), blev(n);
    std::vector<uint8_t> flags(f->L);
    std::vector<int32_t> pp(f->P + 1), pl(f->L);
    DM_CUDA(cudaStreamSynchronize(s));
    DM_CUDA(cudaMemcpy(pp.data(), f->proc_ptr, pp.size() * 4, cudaMemcpyDeviceToHost));
    DM_CUDA(cudaMemcpy(pl.data(), f->proc_layers, pl.size() * 4, cudaMemcpyDeviceToHost));
    DM_CUDA(cudaMemcpy(fpos.data(), f->fw_pos, n * 4, cudaMemcpyDeviceToHost));
    DM_CUDA(cudaMemcpy(flev.data(), f->fw_lev, n * 4, cudaMemcpyDeviceToHost));
    DM_CUDA(cudaMemcpy(bpos.data(), f->bw_pos, n * 4, cudaMemcpyDeviceToHost));
    DM_CUDA(cudaMemcpy(blev.data(), f->bw_lev, n * 4, cudaMemcpyDeviceToHost));
    DM_CUDA(cudaMemcpy(flags.data(), f->layer_flags, f->L, cudaMemcpyDeviceToHost));
    dm::MmaSchedule fw, bw;
    dm::pack_mma_tasks(fpos, flev, pp.data(), pl.data(), flags.data(), fw);
    dm::pack_mma_tasks(bpos, blev, pp.data(), pl.data(), flags.data(), bw);
    f->fw_tasks = fw.tasks;
    f->bw_tasks = bw.tasks;
    int rc;
    if ((rc = upload(f, &f->fw_layer, fw.task_layer.data(), (int64_t)fw.task_layer.size(), s))) return rc;
    if ((rc = upload(f, &f->fw_meta, fw.task_meta.data(), (int64_t)fw.task_meta.size(), s))) return rc;
    if ((rc = upload(f, &f->bw_layer, bw.task_layer.data(), (int64_t)bw.task_layer.size(), s))) return rc;
    if ((rc = upload(f, &f->bw_meta, bw.task_meta.data(), (int64_t)bw.task_meta.size(), s))) return rc;
    if ((rc = upload(f, &f->fw_task_level, fw.task_level.data(), (int64_t)fw.task_level.size(), s))) return rc;
    if ((rc = upload(f, &f->bw_task_level, bw.task_level.data(), (int64_t)bw.task_level.size(), s))) return rc;
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_fail(cudaGetLastError(), "per-copy schedule upload");
    f->fw_level = std::move(fw.task_level);
    f->bw_level = std::move(bw.task_level);
    f->fw_layer_h = std::move(fw.task_layer);
    f->bw_layer_h = std::move(bw.task_layer);
    f->classic_uploaded = true;
    return DM_OK;
}

static int configure_mma(dm_flat *f, int threads, int blocks_per_sm, unsigned sleep_ns, int probe, int lookahead) {
    f->mma_lookahead = lookahead < 0 ? 0 : (lookahead & 0xffff);
    f->mma_warm = (lookahead >> 16) & 1;   // bit 16 of the lookahead word: L2 warming
    f->mma_desc = !((lookahead >> 17) & 1);  // bit 17: force the tree publish
    f->mma_np = f->np_ok && !((lookahead >> 18) & 1);  // bit 18: force the per-copy kernels
    if (threads < 32 || threads > 256 || threads % 32) {
        dm::set_error("exact-pass block size must be a multiple of 32 in [32, 256]");
        return DM_ERR_INVALID;
    }
#define DM_GRID(W, K)                                                          \
    (mma_grid_for<W, K>(f, true, threads, blocks_per_sm, &f->mma_grid_fw) ||      \
     mma_grid_for<W, K>(f, false, threads, blocks_per_sm, &f->mma_grid_bw))
    if (DM_MMA_DISPATCH(f, DM_GRID)) return DM_ERR_CUDA;
#undef DM_GRID
    f->mma_threads = threads;
    f->mma_blocks_per_sm = blocks_per_sm;
    f->mma_sleep_ns = sleep_ns;
    f->mma_probe = probe ? 1 : 0;
    return DM_OK;
}

namespace {

double host_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}

int check_stream_error(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    return DM_OK;
}

}  // namespace

extern "C" {

const char *dm_version(void) {
    return "discomatch_b200 0.1 (sm_100a, fp64 exact)";
}

int dm_flat_create(const dm_flat_desc *desc, int device, void *stream, dm_flat **out) {
    return dm_flat_create_ex(desc, device, stream, 0, out);
}

int dm_flat_create_ex(const dm_flat_desc *desc, int device, void *stream, int flags, dm_flat **out) {
    const bool exact_plans = !(flags & DM_FLAT_NO_EXACT_PLANS);
    if (!desc || !out) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    *out = nullptr;
    const double t_begin = host_seconds();
    const int64_t nb = desc->num_bdds, L = desc->num_layers, N = desc->num_nodes, P = desc->num_positions;
    if (nb < 0 || L < 0 || N < 0 || P < 0 || L >= INT32_MAX || N >= INT32_MAX - 2 || P >= INT32_MAX) {
        dm::set_error("instance sizes outside the int32 device layout");
        return DM_ERR_UNSUPPORTED;
    }
    // validate the structure the kernels rely on (bdd.py:336-359 invariants)
    const int64_t *bl = desc->bdd_layer_lo, *lnl = desc->layer_node_lo;
    if (bl[0] != 0 || bl[nb] != L || lnl[0] != 0 || lnl[L] != N || desc->proc_ptr[0] != 0 || desc->proc_ptr[P] != L) {
        dm::set_error("inconsistent flat table offsets");
        return DM_ERR_INVALID;
    }
    dm::I32Buffer layer_bdd, pos_var;  // every element written below
    layer_bdd.resize(L);
    pos_var.resize(P);
    if (env_int("DM_VERBOSE", 0) >= 2)
        std::fprintf(stderr, "  [dm_flat_create] buffers %.4f\n", host_seconds() - t_begin);
    std::vector<int32_t> var_count;
    int64_t max_width = 0, max_degree = 0;
    {
        // diagram ranges validated in parallel; the first failing range reports
        constexpr int kThreads = 8;
        int64_t widths[kThreads] = {0};
        int codes[kThreads] = {DM_OK};
        const char *msgs[kThreads] = {nullptr};
        std::vector<std::thread> th;
        for (int t = 0; t < kThreads; ++t)
            th.emplace_back([&, t] {
                const int64_t jlo = nb * t / kThreads, jhi = nb * (t + 1) / kThreads;
                int64_t wmax = 0;  // thread-local (widths[] would false-share)
                for (int64_t j = jlo; j < jhi; ++j) {
                    if (bl[j + 1] <= bl[j] || lnl[bl[j] + 1] - lnl[bl[j]] != 1) {
                        codes[t] = DM_ERR_INVALID;
                        msgs[t] = "every diagram needs >= 1 layer and a single root node";
                        return;
                    }
                    for (int64_t l = bl[j]; l < bl[j + 1]; ++l) {
                        layer_bdd[l] = (int32_t)j;
                        const int64_t w = lnl[l + 1] - lnl[l];
                        if (w <= 0) {
                            codes[t] = DM_ERR_INVALID;
                            msgs[t] = "empty layer";
                            return;
                        }
                        wmax = std::max(wmax, w);
                    }
                }
                widths[t] = wmax;
            });
        for (auto &x : th) x.join();
        for (int t = 0; t < kThreads; ++t) {
            if (codes[t] != DM_OK) {
                dm::set_error(msgs[t]);
                return codes[t];
            }
            max_width = std::max(max_width, widths[t]);
        }
    }
    if (max_width > 32) {
        dm::set_error("instance outside the kernels' envelope: a layer has " + std::to_string(max_width) +
                      " nodes (the sweep and averaging kernels support at most 32)");
        return DM_ERR_UNSUPPORTED;
    }
    const bool vb2v = env_int("DM_VERBOSE", 0) >= 2;
    if (vb2v) std::fprintf(stderr, "  [dm_flat_create] diagrams checked %.4f\n", host_seconds() - t_begin);
    // variable range, then the visitation CSR (degrees, position -> variable)
    // in parallel; the first failing range reports
    constexpr int kVThreads = 8;
    auto par = [&](int64_t n, auto &&fn) {
        std::vector<std::thread> th;
        for (int t = 0; t < kVThreads; ++t) th.emplace_back([&, t] { fn(t, n * t / kVThreads, n * (t + 1) / kVThreads); });
        for (auto &x : th) x.join();
    };
    int64_t vmax[kVThreads], dmax[kVThreads] = {0}, nval[kVThreads] = {0};
    const char *vmsg[kVThreads] = {nullptr};
    par(L, [&](int t, int64_t lo, int64_t hi) {
        int64_t m = -1;
        for (int64_t l = lo; l < hi; ++l) m = std::max(m, desc->layer_var[l]);
        vmax[t] = m;
    });
    int64_t max_var = -1;
    for (int t = 0; t < kVThreads; ++t) max_var = std::max(max_var, vmax[t]);
    const int64_t V = std::max<int64_t>(max_var + 1, P);
    var_count.assign(V, 0);
    if (vb2v) std::fprintf(stderr, "  [dm_flat_create] variables ranged %.4f\n", host_seconds() - t_begin);
    par(P, [&](int t, int64_t plo, int64_t phi) {
        int64_t dm_ = 0, nv_ = 0;  // thread-local (the shared arrays would false-share)
        struct Flush {
            int64_t &a, &b, &da, &nb;
            ~Flush() { da = a, nb = b; }
        } flush{dm_, nv_, dmax[t], nval[t]};
        for (int64_t p = plo; p < phi; ++p) {
            const int64_t lo = desc->proc_ptr[p], hi = desc->proc_ptr[p + 1];
            if (hi < lo || hi > L) {
                vmsg[t] = "visitation offsets must be non-decreasing and within the layers";
                return;
            }
            if (hi - lo > 32) {
                vmsg[t] = "instance outside the kernels' envelope: a variable is shared by more than 32 diagrams "
                          "(the exact averaging kernels support at most 32)";
                return;
            }
            dm_ = std::max(dm_, hi - lo);
            for (int64_t q = lo; q < hi; ++q)
                if (desc->proc_layers[q] < 0 || desc->proc_layers[q] >= L) {
                    vmsg[t] = "visited layer out of range";
                    return;
                }
            if (hi > lo) {
                ++nv_;
                const int64_t v = desc->layer_var[desc->proc_layers[lo]];
                if (v < 0) {
                    vmsg[t] = "negative variable id";
                    return;
                }
                pos_var[p] = (int32_t)v;
                var_count[v] = (int32_t)(hi - lo);
            } else {
                pos_var[p] = -1;
            }
        }
    });
    int64_t nvalid = 0;  // positions with copies (= exact-pass tasks of the node-parallel kernels)
    for (int t = 0; t < kVThreads; ++t) {
        if (vmsg[t]) {
            dm::set_error(vmsg[t]);
            return std::strstr(vmsg[t], "at most 32") ? DM_ERR_UNSUPPORTED : DM_ERR_INVALID;
        }
        max_degree = std::max(max_degree, dmax[t]);
        nvalid += nval[t];
    }
    const double t_valid = host_seconds();
    // Every plan is built on the device (dm_plan.cu) while the host stages
    // the topology: the exact-pass schedules and copy records on one stream
    // once the visitation CSR is there, the sweep layout on another (its
    // sizes are read back on a host thread), its fill and the forward
    // publish descriptors once the arc targets are there.
    const bool want_np = max_width <= 8 && max_degree <= 8;
    const bool vb2 = env_int("DM_VERBOSE", 0) >= 2;
    auto mark = [&](const char *what) {
        if (vb2) std::fprintf(stderr, "  [dm_flat_create] %s %.4f\n", what, host_seconds() - t_begin);
    };
    int rc = DM_OK;
    DM_CUDA(cudaSetDevice(device));
    keep_pool_memory(device);
    cudaStream_t s = (cudaStream_t)stream;
    auto f = std::make_unique<dm_flat>();
    // on any error return: the device blocks allocated so far go back to the
    // pool (destroyed after the staging ring and plan streams below, which
    // synchronise their work first)
    struct FreeOnError {
        std::unique_ptr<dm_flat> &f;
        ~FreeOnError() {
            if (!f) return;
            cudaDeviceSynchronize();
            for (void *p : f->allocs) cudaFreeAsync(p, 0);
            cudaGetLastError();
        }
    } free_on_error{f};
    f->device = device;
    f->nb = nb;
    f->L = L;
    f->N = N;
    f->P = P;
    f->max_width = max_width;
    f->max_degree = max_degree;
    auto up = [&](int32_t **dst, const std::vector<int32_t> &v) {
        return upload(f.get(), dst, v.data(), (int64_t)v.size(), s);
    };
    auto alloc = [&](auto **dst, int64_t n) {
        using T = std::remove_reference_t<decltype(**dst)>;
        return upload(f.get(), dst, (const T *)nullptr, n, s);
    };
    mark("validated");
    Stager stage(device, s);
    mark("stager");
    if ((rc = stage.narrow(f.get(), &f->bdd_layer_lo, bl, nb + 1))) return rc;
    if ((rc = stage.narrow(f.get(), &f->lnl, lnl, L + 1))) return rc;
    if ((rc = stage.narrow(f.get(), &f->proc_ptr, desc->proc_ptr, P + 1))) return rc;
    if ((rc = stage.narrow(f.get(), &f->proc_layers, desc->proc_layers, L))) return rc;
    if ((rc = stage.copy(f.get(), &f->layer_bdd, layer_bdd.data(), L))) return rc;
    mark("csr staged");
    int *plan_words = nullptr;
    if ((rc = alloc(&f->layer_flags, L))) return rc;
    if ((rc = alloc(&f->fw_pos, P))) return rc;
    if ((rc = alloc(&f->bw_pos, P))) return rc;
    if ((rc = alloc(&f->fw_lev, P))) return rc;
    if ((rc = alloc(&f->bw_lev, P))) return rc;
    if ((rc = alloc(&plan_words, 8))) return rc;
    if (want_np && ((rc = alloc(&f->np_rec_fw, nvalid * 8)) || (rc = alloc(&f->np_rec_bw, nvalid * 8)))) return rc;
    // device plans on their own stream, after the CSR upload
    unsigned long long *relax_fail = nullptr;
    if ((rc = alloc(&relax_fail, 1))) return rc;
    // written by the sweep-layout thread: declared before `ps`, whose
    // destructor joins that thread on every return path
    std::vector<void *> sweep_allocs;
    int64_t sweep_bytes = 0;
    int rc_sl = DM_OK;
    std::string err_sl;
    double t_sweep = 0;
    struct PlanStreams {
        cudaStream_t s = nullptr, ss = nullptr;
        cudaEvent_t ready = nullptr, done = nullptr, zo_ready = nullptr, ss_done = nullptr;
        std::thread th;
        ~PlanStreams() {
            if (th.joinable()) th.join();
            for (cudaStream_t x : {s, ss})
                if (x) cudaStreamSynchronize(x), cudaStreamDestroy(x);
            for (cudaEvent_t e : {ready, done, zo_ready, ss_done})
                if (e) cudaEventDestroy(e);
        }
    } ps;
    DM_CUDA(cudaStreamCreateWithFlags(&ps.s, cudaStreamNonBlocking));
    DM_CUDA(cudaStreamCreateWithFlags(&ps.ss, cudaStreamNonBlocking));
    for (cudaEvent_t *e : {&ps.ready, &ps.done, &ps.zo_ready, &ps.ss_done})
        DM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    DM_CUDA(cudaMemsetAsync(relax_fail, 0, sizeof(unsigned long long), s));
    DM_CUDA(cudaEventRecord(ps.ready, s));
    DM_CUDA(cudaStreamWaitEvent(ps.s, ps.ready, 0));
    DM_CUDA(cudaStreamWaitEvent(ps.ss, ps.ready, 0));
    // sweep layout sizes on a host thread (two small read-backs)
    ps.th = std::thread([&] {
        const double t0 = host_seconds();
        cudaSetDevice(device);
        rc_sl = dm::device_sweep_layout(f->bdd_layer_lo, f->lnl, nb, f->sweep, sweep_allocs, sweep_bytes, ps.ss);
        if (rc_sl) err_sl = dm_last_error();
        t_sweep = host_seconds() - t0;
    });
    if (dm::device_layer_flags(f->layer_bdd, f->bdd_layer_lo, L, f->layer_flags, ps.s)) return DM_ERR_CUDA;
    cudaEvent_t walk_ev[2] = {nullptr, nullptr};
    if (vb2) {
        for (auto &e : walk_ev) cudaEventCreate(&e);
        cudaEventRecord(walk_ev[0], ps.s);
    }
    if (exact_plans && dm::device_level_orders(f->proc_ptr, f->proc_layers, f->layer_bdd, f->bdd_layer_lo, P, L,
                                               nvalid, f->fw_pos, f->fw_lev, f->bw_pos, f->bw_lev, plan_words, ps.s))
        return DM_ERR_CUDA;
    if (!exact_plans) DM_CUDA(cudaMemsetAsync(plan_words, 0, 8 * sizeof(int), ps.s));
    if (vb2) cudaEventRecord(walk_ev[1], ps.s);
    if (exact_plans && want_np && (dm::device_np_records(f->proc_ptr, f->proc_layers, f->lnl, f->layer_flags, f->fw_pos, nvalid,
                                          f->np_rec_fw, ps.s) ||
                    dm::device_np_records(f->proc_ptr, f->proc_layers, f->lnl, f->layer_flags, f->bw_pos, nvalid,
                                          f->np_rec_bw, ps.s)))
        return DM_ERR_CUDA;
    DM_CUDA(cudaEventRecord(ps.done, ps.s));
    mark("plans queued");
    if ((rc = stage.narrow(f.get(), &f->layer_var, desc->layer_var, L))) return rc;
    // arc targets: narrowed and range-checked in the same pass (they must
    // reach the next layer, or a terminal from a last layer)
    std::atomic<bool> bad_arc{false};
    auto narrow_arcs = [&](int32_t **dst, const int64_t *src) {
        return stage.put(f.get(), dst, N, [&, src](int32_t *d, int64_t lo, int64_t c) {
            int64_t l = std::upper_bound(lnl, lnl + L + 1, lo) - lnl - 1;
            bool bad = false;
            for (int64_t i = 0; i < c; ++i) {
                const int64_t v = lo + i;
                while (v >= lnl[l + 1]) ++l;
                const int64_t tt = src[v];
                const bool last = l + 1 == bl[layer_bdd[l] + 1];
                bad |= last ? (tt >= 0 || tt < -2) : (tt < -2 || tt == -2 || (tt >= 0 && (tt < lnl[l + 1] || tt >= lnl[l + 2])));
                d[i] = (int32_t)tt;
            }
            if (bad) bad_arc = true;
        });
    };
    if ((rc = narrow_arcs(&f->zero_t, desc->zero_t))) return rc;
    if ((rc = narrow_arcs(&f->one_t, desc->one_t))) return rc;
    if (bad_arc) {
        dm::set_error("arc targets must reach the next layer (or a terminal from the last layer)");
        return DM_ERR_UNSUPPORTED;
    }
    if ((rc = stage.copy(f.get(), &f->pos_var, pos_var.data(), P))) return rc;
    if ((rc = stage.copy(f.get(), &f->var_count, var_count.data(), (int64_t)var_count.size()))) return rc;
    const std::vector<int32_t> progress_init{-1, 0}, status_init{0};
    if ((rc = up(&f->progress, progress_init))) return rc;  // progress hint, task queue
    if ((rc = up(&f->status, status_init))) return rc;
    mark("topology staged");
    ps.th.join();
    mark("sweep sizes joined");
    f->allocs.insert(f->allocs.end(), sweep_allocs.begin(), sweep_allocs.end());
    f->bytes += sweep_bytes;
    if (rc_sl) {
        dm::set_error(err_sl);
        return rc_sl == -2 ? DM_ERR_UNSUPPORTED : DM_ERR_CUDA;
    }
    const double t_plans = host_seconds();
    // arc targets staged: sweep fill and publish descriptors
    DM_CUDA(cudaEventRecord(ps.zo_ready, s));
    DM_CUDA(cudaStreamWaitEvent(ps.ss, ps.zo_ready, 0));
    if (dm::device_sweep_fill(f->sweep, f->zero_t, f->one_t, ps.ss)) return DM_ERR_CUDA;
    const bool want_relax = max_width <= 8;
    if (want_relax) {
        if ((rc = alloc(&f->relax_layer, L))) return rc;
        DM_CUDA(cudaEventRecord(ps.zo_ready, s));  // the allocation is ordered on s
        DM_CUDA(cudaStreamWaitEvent(ps.ss, ps.zo_ready, 0));
        if (dm::device_relax(f->layer_bdd, f->bdd_layer_lo, f->lnl, f->zero_t, f->one_t, L, f->relax_layer,
                             relax_fail, ps.ss))
            return DM_ERR_CUDA;
    }
    DM_CUDA(cudaEventRecord(ps.ss_done, ps.ss));
    f->mma_w = max_width <= 8 ? 8 : (max_width <= 16 ? 16 : 32);
    f->mma_k = max_degree <= 8 ? 8 : 32;
    f->np_fw_tasks = f->np_bw_tasks = nvalid;
    f->np_ok = want_np;
    DevPlan *dummy;
    if ((rc = get_plan(nb, s, &dummy))) return rc;
    if ((rc = get_plan(L, s, &dummy))) return rc;
    DM_CUDA(cudaStreamWaitEvent(s, ps.done, 0));
    DM_CUDA(cudaStreamWaitEvent(s, ps.ss_done, 0));
    mark("tail queued");
    DM_CUDA(cudaStreamSynchronize(s));  // the host staging vectors die with this scope
    mark("synchronised");
    if (vb2) {
        float ms = 0;
        cudaEventElapsedTime(&ms, walk_ev[0], walk_ev[1]);
        std::fprintf(stderr, "  [dm_flat_create] level orders on the device: %.2f ms\n", ms);
        for (auto &e : walk_ev) cudaEventDestroy(e);
    }
    int words[8];
    unsigned long long rfail = 1;
    DM_CUDA(cudaMemcpy(words, plan_words, sizeof(words), cudaMemcpyDeviceToHost));
    DM_CUDA(cudaMemcpy(&rfail, relax_fail, sizeof(rfail), cudaMemcpyDeviceToHost));
    f->relax_ok = want_relax && rfail == 0;
    rc = configure_mma(f.get(), env_int("DM_MMA_THREADS", 256), env_int("DM_MMA_BLOCKS_PER_SM", 3),
                       (unsigned)env_int("DM_MMA_SLEEP_NS", 32), env_int("DM_MMA_PROBE", 0),
                       env_int("DM_MMA_LOOKAHEAD", 0) | (env_int("DM_MMA_WARM", 1) << 16) |
                           ((env_int("DM_MMA_DESC", 1) ? 0 : 1) << 17) | ((env_int("DM_MMA_NP", 1) ? 0 : 1) << 18));
    if (rc) return rc;
    if (words[1] || words[3]) {
        dm::set_error("device schedule: level walk stalled (watchdog)");
        return DM_ERR_CUDA;
    }
    f->fw_depth = nvalid && exact_plans ? words[4] + 1 : 0;
    f->bw_depth = nvalid && exact_plans ? words[5] + 1 : 0;
    f->exact_plans = exact_plans;
    if (exact_plans && !f->mma_np && (rc = ensure_per_copy_schedules(f.get(), s))) return rc;
    if (env_int("DM_VERBOSE", 0))
        std::fprintf(stderr,
                     "[dm_flat_create] validate %.3fs, topology staging + device plans %.3fs, plan tail %.3fs "
                     "(sweep layout sizes %.3f)\n",
                     t_valid - t_begin, t_plans - t_valid, host_seconds() - t_plans, t_sweep);
    *out = f.release();
    return DM_OK;
}

int dm_flat_get_info(const dm_flat *f, dm_flat_info *info) {
    if (!f || !info) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    info->fw_depth = f->fw_depth;
    info->bw_depth = f->bw_depth;
    info->fw_tasks = f->mma_np ? f->np_fw_tasks : f->fw_tasks;
    info->bw_tasks = f->mma_np ? f->np_bw_tasks : f->bw_tasks;
    info->dfr_node_parallel = f->relax_ok ? 1 : 0;
    info->lanes_per_task = f->mma_np ? 8 : 32;
    info->mma_grid = f->mma_grid_fw;
    info->mma_block = f->mma_threads;
    info->max_width = f->max_width;
    info->max_degree = f->max_degree;
    info->device_bytes = f->bytes;
    return DM_OK;
}

// Every entry point runs on the device its data lives on and restores the
// caller's current device on return (a flat's device, or the stream's).
struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        int cur;
        if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess)
            prev = cur;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
inline int stream_device(void *stream) {
    int dev = -1;
    if (stream && cudaStreamGetDevice((cudaStream_t)stream, &dev) != cudaSuccess) {
        cudaGetLastError();
        dev = -1;
    }
    return dev;
}
#define DM_CHECK_FLAT(f)                        \
    if (!(f)) {                                 \
        dm::set_error("null flat handle");      \
        return DM_ERR_INVALID;                  \
    }                                           \
    DevGuard dm_guard_((f)->device)
#define DM_STREAM_GUARD(stream) DevGuard dm_guard_(stream_device(stream))

int dm_flat_set_mma_config(dm_flat *f, int threads, int blocks_per_sm, int sleep_ns, int probe, int lookahead) {
    if (!f) {
        dm::set_error("null flat handle");
        return DM_ERR_INVALID;
    }
    int rc = configure_mma(f, threads, blocks_per_sm, (unsigned)std::max(0, sleep_ns), probe, lookahead);
    if (rc == DM_OK && !f->mma_np) rc = ensure_per_copy_schedules(f, 0);
    return rc;
}

int dm_flat_set_trace(dm_flat *f, unsigned long long *trace) {
    if (!f) {
        dm::set_error("null flat handle");
        return DM_ERR_INVALID;
    }
    f->trace = trace;
    return DM_OK;
}

int dm_flat_task_levels(const dm_flat *f, int forward, int32_t *levels, int32_t *lane_layers) {
    if (!f) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    if (f->mma_np) {  // one task per position, 8 copy slots per task
        const int64_t n = f->np_fw_tasks;
        DM_CUDA(cudaDeviceSynchronize());
        if (levels) DM_CUDA(cudaMemcpy(levels, forward ? f->fw_lev : f->bw_lev, n * 4, cudaMemcpyDeviceToHost));
        if (lane_layers) {
            std::vector<int32_t> pos(n);
            DM_CUDA(cudaMemcpy(pos.data(), forward ? f->fw_pos : f->bw_pos, n * 4, cudaMemcpyDeviceToHost));
            std::vector<int32_t> pp(f->P + 1), pl(f->L);
            DM_CUDA(cudaMemcpy(pp.data(), f->proc_ptr, pp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
            DM_CUDA(cudaMemcpy(pl.data(), f->proc_layers, pl.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
            for (size_t t = 0; t < pos.size(); ++t)
                for (int c = 0; c < 8; ++c) {
                    const int32_t lo = pp[pos[t]], k = pp[pos[t] + 1] - lo;
                    lane_layers[t * 8 + c] = c < k ? pl[lo + c] : -1;
                }
        }
        return DM_OK;
    }
    const auto &v = forward ? f->fw_level : f->bw_level;
    const auto &w = forward ? f->fw_layer_h : f->bw_layer_h;
    if (levels) std::memcpy(levels, v.data(), v.size() * sizeof(int32_t));
    if (lane_layers) std::memcpy(lane_layers, w.data(), w.size() * sizeof(int32_t));
    return DM_OK;
}

int dm_flat_status_to(const dm_flat *f, double *slot, void *stream) {
    DM_CHECK_FLAT(f);
    if (!slot) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    status_to_slot_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(f->status, slot);
    return check_stream_error("status copy");
}

int dm_flat_status(dm_flat *f, void *stream) {
    DM_CHECK_FLAT(f);
    int v = 0;
    DM_CUDA(cudaMemcpyAsync(&v, f->status, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    DM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (v != 0) {
        const int zero = 0;
        cudaMemcpy(f->status, &zero, sizeof(int), cudaMemcpyHostToDevice);
        dm::set_error("exact averaging pass aborted by its watchdog (a lane waited > 4 s for its inputs)");
        return DM_ERR_CUDA;
    }
    return DM_OK;
}

void dm_flat_destroy(dm_flat *f) {
    if (!f) return;
    // the flat may still be in use by work on any (possibly non-blocking)
    // stream: wait for its device, then hand the blocks back to the pool;
    // the caller's current device is restored (this runs from GC)
    DevGuard guard(f->device);
    cudaDeviceSynchronize();
    for (void *p : f->allocs) cudaFreeAsync(p, 0);
    cudaGetLastError();
    delete f;
}

int dm_k_backward(const dm_flat *f, const double *lam, double *B, double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->nb == 0) return DM_OK;
    if (!B) {
        dm::set_error("k_backward needs B");
        return DM_ERR_INVALID;
    }
    if (f->dec_B == B) const_cast<dm_flat *>(f)->dec_B = nullptr;  // recorded decisions no longer match B
    return dm::sweep_backward(f->sweep, lam, nullptr, 0.0, B, bounds, stream);
}

int dm_qn_move(const dm_flat *f, double *lam, const double *d, double base, const double *state, double *out,
               double *B, double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    if (!lam || !d || !state || !out || !B || !bounds) {
        dm::set_error("dm_qn_move: invalid arguments");
        return DM_ERR_INVALID;
    }
    const cudaStream_t s = (cudaStream_t)stream;
    qn_move_kernel<<<grid_stride_blocks(f->L), 256, 0, s>>>(lam, d, base, state, out, f->L);
    if (int rc = check_stream_error("qn_move")) return rc;
    if (f->nb == 0) return DM_OK;
    if (f->dec_B == B) const_cast<dm_flat *>(f)->dec_B = nullptr;
    // the averaging pass's refresh of B (dual.py:164-165), skipped on the device when nothing moved
    return dm::sweep_backward(f->sweep, lam, nullptr, 0.0, B, bounds, stream, out + 1);
}

int dm_k_backward_trial(const dm_flat *f, const double *lam, const double *d, double gamma, double *B,
                        double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->nb == 0) return DM_OK;
    return dm::sweep_backward(f->sweep, lam, d, gamma, B, bounds, stream);
}

int dm_debug_div_check(int k, uint64_t n, uint64_t seed, unsigned long long *mismatches) {
    if (k < 1 || k > 8 || !mismatches) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    unsigned long long *d;
    DM_CUDA(cudaMalloc(&d, sizeof(*d)));
    DM_CUDA(cudaMemset(d, 0, sizeof(*d)));
    div_check_kernel<<<148 * 8, 256>>>(k, n, seed, d);
    const cudaError_t e = cudaMemcpy(mismatches, d, sizeof(*d), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e) return cuda_fail(e, "div check");
    return DM_OK;
}

int dm_step_search(const dm_flat *f, const double *lam, const double *d, double gamma_prev, double free_contribution,
                   double shrink, double grow, double min_ascent, int max_trials, double *bounds, double *state,
                   void *stream) {
    DM_CHECK_FLAT(f);
    if (!lam || !d || !bounds || !state || max_trials < 0) {
        dm::set_error("invalid step search arguments");
        return DM_ERR_INVALID;
    }
    if (f->nb == 0) {
        dm::set_error("step search needs at least one diagram");
        return DM_ERR_INVALID;
    }
    const cudaStream_t s = (cudaStream_t)stream;
    DevPlan *p;
    int rc = get_plan(f->nb, s, &p);
    if (rc) return rc;
    const StepParams prm{free_contribution, shrink, grow, min_ascent, max_trials};
    step_init_kernel<<<1, 1, 0, s>>>(state, gamma_prev);
    // every trial is enqueued up front; the ones after the stop return at once
    for (int t = 0; t <= max_trials; ++t) {
        if ((rc = dm::sweep_backward(f->sweep, lam, d, 0.0, nullptr, bounds, stream, state))) return rc;
        pw_leaf_kernel<false><<<blocks_for((int64_t)p->nleaves * 8, 256), 256, 0, s>>>(
            p->nleaves, p->leaf_off, p->leaf_len, bounds, nullptr, p->vals, state + 5);
        pw_combine_kernel<<<1, 1024, 0, s>>>(p->nleaves, p->maxh, p->height_lo, p->left, p->right, p->root, p->vals,
                                             nullptr, state, prm, t);
    }
    return check_stream_error("step search");
}

int dm_k_forward(const dm_flat *f, const double *lam, double *F, double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->dec_B == F) const_cast<dm_flat *>(f)->dec_B = nullptr;
    if (f->nb == 0) return DM_OK;
    return dm::sweep_forward(f->sweep, lam, F, bounds, stream);
}

static int mma_pass(const dm_flat *f, bool forward, double *lam, double *F, double *B, double *bounds,
                    cudaStream_t s) {
    if (f->nb == 0) return DM_OK;
    if (!f->exact_plans) {
        dm::set_error("exact averaging pass on a flat created without its plans (DM_FLAT_NO_EXACT_PLANS)");
        return DM_ERR_INVALID;
    }
    double sent;
    std::memcpy(&sent, &kSentinel, sizeof(sent));
    if (forward) {
        fill_kernel<<<grid_stride_blocks(f->N), 256, 0, s>>>(F, f->N, sent);
        roots_kernel<<<blocks_for(f->nb, 256), 256, 0, s>>>((int32_t)f->nb, f->bdd_layer_lo, f->lnl, F);
    } else {
        fill_kernel<<<grid_stride_blocks(f->N), 256, 0, s>>>(B, f->N, sent);
    }
    int rc = check_stream_error("mma fill");
    if (rc) return rc;
    if (!f->mma_np && (rc = ensure_per_copy_schedules(const_cast<dm_flat *>(f), s))) return rc;
    MmaArgs args;
    args.ntasks = forward ? f->fw_tasks : f->bw_tasks;
    args.task_layer = forward ? f->fw_layer : f->bw_layer;
    args.task_meta = forward ? f->fw_meta : f->bw_meta;
    args.lnl = f->lnl;
    args.zero_t = f->zero_t;
    args.one_t = f->one_t;
    args.layer_bdd = f->layer_bdd;
    args.lam = lam;
    args.F = F;
    args.B = B;
    args.bounds = bounds;
    args.status = f->status;
    args.sleep_ns = f->mma_sleep_ns;
    args.probe = f->mma_probe;
    args.trace = f->trace;
    args.task_level = forward ? f->fw_task_level : f->bw_task_level;
    args.progress = f->progress;
    args.lookahead = f->mma_lookahead;
    args.warm = f->mma_warm;
    // A/B (tools/ab_hints.py, profiles/r02_mma_c2_full.md): hints 7 = bw -1 % at C2 / -3 % at C4, fw
    // flat, but +10 % DRAM bytes per launch (4.43 / 4.30 GB vs 4.00 / 3.86): off by default
    args.hints = env_int("DM_MMA_HINTS", 0);
    args.relax_layer = f->relax_layer;
    args.task_pos = forward ? f->fw_pos : f->bw_pos;
    args.proc_ptr = f->proc_ptr;
    args.proc_layers = f->proc_layers;
    args.layer_flags = f->layer_flags;
    args.np_rec = forward ? f->np_rec_fw : f->np_rec_bw;
    args.dec = nullptr;
    if (f->mma_np && !forward) {
        dm_flat *m = const_cast<dm_flat *>(f);
        if (!m->dec) {
            DM_CUDA(cudaMallocAsync((void **)&m->dec, (size_t)std::max<int64_t>(f->L, 1) * 8, s));
            m->allocs.push_back(m->dec);
            m->bytes += (size_t)std::max<int64_t>(f->L, 1) * 8;
        }
        args.dec = m->dec;
        m->dec_B = B;
    } else if (!forward) {
        const_cast<dm_flat *>(f)->dec_B = nullptr;
    }
    args.task_counter = f->progress + 1;
    if (f->mma_np) {
        args.ntasks = forward ? f->np_fw_tasks : f->np_bw_tasks;
        args.lookahead = 0;  // the progress gate indexes per-copy task levels
    }
    DM_CUDA(cudaMemsetAsync(f->progress, 0xff, sizeof(int), s));  // -1: nothing finished
    DM_CUDA(cudaMemsetAsync(f->progress + 1, 0, sizeof(int), s));  // empty task queue
#define DM_LAUNCH(W, K) launch_mma<W, K>(f, forward, args, s)
    return DM_MMA_DISPATCH(f, DM_LAUNCH);
#undef DM_LAUNCH
}

int dm_k_mma_forward(const dm_flat *f, double *lam, double *F, const double *B, double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    const_cast<dm_flat *>(f)->dec_B = nullptr;  // the duals move: recorded decisions are stale
    return mma_pass(f, true, lam, F, const_cast<double *>(B), bounds, (cudaStream_t)stream);
}

int dm_k_mma_backward(const dm_flat *f, double *lam, const double *F, double *B, double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    return mma_pass(f, false, lam, const_cast<double *>(F), B, bounds, (cudaStream_t)stream);
}

int dm_k_min_marginals(const dm_flat *f, const double *lam, const double *F, const double *B, double *m0,
                       double *m1, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->L == 0) return DM_OK;
    k_min_marginals_kernel<<<blocks_for(f->L, 256), 256, 0, (cudaStream_t)stream>>>(
        (int32_t)f->L, f->lnl, f->zero_t, f->one_t, lam, F, B, m0, m1);
    return check_stream_error("k_min_marginals");
}

int dm_k_argmin(const dm_flat *f, const double *lam, const double *B, double *bits, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->nb == 0) return DM_OK;
    k_argmin_kernel<<<blocks_for(f->nb, 128), 128, 0, (cudaStream_t)stream>>>(
        (int32_t)f->nb, f->bdd_layer_lo, f->lnl, f->zero_t, f->one_t, lam, B, bits);
    return check_stream_error("k_argmin");
}

int dm_k_argmin_from_pass(const dm_flat *f, const double *B, double *bits, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->nb == 0) return DM_OK;
    if (!f->dec || f->dec_B != B || !B) {
        dm::set_error("dm_k_argmin_from_pass: no node-parallel backward pass wrote this distance table");
        return DM_ERR_INVALID;
    }
    k_argmin_walk_kernel<<<blocks_for(f->nb, 128), 128, 0, (cudaStream_t)stream>>>(
        (int32_t)f->nb, f->bdd_layer_lo, f->lnl, f->dec, bits);
    return check_stream_error("k_argmin_walk");
}

// --- deferred (throughput) averaging schedule: dm_deferred.cu -------------
int dm_dfr_table_size(const dm_flat *f, int64_t *elements) {
    DM_CHECK_FLAT(f);
    if (!elements) {
        dm::set_error("dm_dfr_table_size: null output");
        return DM_ERR_INVALID;
    }
    *elements = f->sweep.slots * 32;
    return DM_OK;
}

int dm_dfr_forward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *B_il,
                   double *F_il, double *mbar, double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    if (!lam || !F_il || !bounds || (mbar && !B_il)) {
        dm::set_error("dm_dfr_forward: lam, F_il, bounds (and B_il with mbar) are required");
        return DM_ERR_INVALID;
    }
    if (f->dec_B == F_il) const_cast<dm_flat *>(f)->dec_B = nullptr;
    return dm::dfr_pass(f->sweep, true, omega, lam, avg_in, B_il, F_il, mbar, bounds, nullptr, stream);
}

int dm_dfr_backward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *F_il,
                    double *B_il, double *mbar, double *bounds, int record_decisions, void *stream) {
    DM_CHECK_FLAT(f);
    if (!lam || !B_il || !bounds || (mbar && !F_il)) {
        dm::set_error("dm_dfr_backward: lam, B_il, bounds (and F_il with mbar) are required");
        return DM_ERR_INVALID;
    }
    dm_flat *m = const_cast<dm_flat *>(f);
    uint64_t *dec = nullptr;
    if (record_decisions && f->sweep.max_width <= 8 && f->L > 0) {
        if (!m->dec) {
            DM_CUDA(cudaMallocAsync((void **)&m->dec, (size_t)f->L * 8, (cudaStream_t)stream));
            m->allocs.push_back(m->dec);
            m->bytes += (size_t)f->L * 8;
        }
        dec = m->dec;
    }
    const int rc = dm::dfr_pass(f->sweep, false, omega, lam, avg_in, F_il, B_il, mbar, bounds, dec, stream);
    m->dec_B = (rc == DM_OK && dec) ? B_il : (m->dec_B == B_il ? nullptr : m->dec_B);
    return rc;
}

int dm_dfr_np_forward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *B,
                      double *F, double *mbar, double *bounds, void *stream) {
    DM_CHECK_FLAT(f);
    if (!f->relax_ok) {
        dm::set_error("dm_dfr_np_forward: needs layers of <= 8 nodes with single-source publish descriptors");
        return DM_ERR_UNSUPPORTED;
    }
    if (!lam || !F || !bounds || (mbar && !B)) {
        dm::set_error("dm_dfr_np_forward: lam, F, bounds (and B with mbar) are required");
        return DM_ERR_INVALID;
    }
    if (f->dec_B == F) const_cast<dm_flat *>(f)->dec_B = nullptr;
    return dm::dfr_np_pass(f->sweep, f->zero_t, f->one_t, f->relax_layer, true, omega, lam, avg_in, B, F, mbar, bounds,
                           nullptr, stream);
}

int dm_dfr_np_backward(const dm_flat *f, double omega, double *lam, const double *avg_in, const double *F, double *B,
                       double *mbar, double *bounds, int record_decisions, void *stream) {
    DM_CHECK_FLAT(f);
    if (!f->relax_ok) {
        dm::set_error("dm_dfr_np_backward: needs layers of <= 8 nodes with single-source publish descriptors");
        return DM_ERR_UNSUPPORTED;
    }
    if (!lam || !B || !bounds || (mbar && !F)) {
        dm::set_error("dm_dfr_np_backward: lam, B, bounds (and F with mbar) are required");
        return DM_ERR_INVALID;
    }
    dm_flat *m = const_cast<dm_flat *>(f);
    uint64_t *dec = nullptr;
    if (record_decisions && f->L > 0) {
        if (!m->dec) {
            DM_CUDA(cudaMallocAsync((void **)&m->dec, (size_t)f->L * 8, (cudaStream_t)stream));
            m->allocs.push_back(m->dec);
            m->bytes += (size_t)f->L * 8;
        }
        dec = m->dec;
    }
    const int rc = dm::dfr_np_pass(f->sweep, f->zero_t, f->one_t, f->relax_layer, false, omega, lam, avg_in, F, B,
                                   mbar, bounds, dec, stream);
    m->dec_B = (rc == DM_OK && dec) ? B : (m->dec_B == B ? nullptr : m->dec_B);
    return rc;
}

int dm_dfr_average(const dm_flat *f, const double *mbar, double *avg_in, void *stream) {
    DM_CHECK_FLAT(f);
    if (!mbar || !avg_in) {
        dm::set_error("dm_dfr_average: null vector");
        return DM_ERR_INVALID;
    }
    return dm::dfr_average(f->P, f->proc_ptr, f->proc_layers, mbar, avg_in, false, stream);
}

int dm_dfr_flush(const dm_flat *f, const double *mbar, double *lam, void *stream) {
    DM_CHECK_FLAT(f);
    if (!mbar || !lam) {
        dm::set_error("dm_dfr_flush: null vector");
        return DM_ERR_INVALID;
    }
    const_cast<dm_flat *>(f)->dec_B = nullptr;  // the duals move
    return dm::dfr_average(f->P, f->proc_ptr, f->proc_layers, mbar, lam, true, stream);
}

int dm_dfr_average_csr(int64_t P, const int32_t *proc_ptr, const int32_t *proc_layers, const double *mbar,
                       double *out, int apply, void *stream) {
    DM_STREAM_GUARD(stream);
    if (P < 0 || P >= INT32_MAX || (P > 0 && (!proc_ptr || !proc_layers || !mbar || !out))) {
        dm::set_error("dm_dfr_average_csr: invalid arguments");
        return DM_ERR_INVALID;
    }
    return dm::dfr_average(P, proc_ptr, proc_layers, mbar, out, apply != 0, stream);
}

int dm_dfr_boundary_gather(int64_t n, const int32_t *layer, const int32_t *slot, const double *mbar, double *buf,
                           void *stream) {
    DM_STREAM_GUARD(stream);
    if (n < 0 || (n > 0 && (!layer || !slot || !mbar || !buf))) {
        dm::set_error("dm_dfr_boundary_gather: invalid arguments");
        return DM_ERR_INVALID;
    }
    return dm::dfr_boundary_gather(n, layer, slot, mbar, buf, stream);
}

int dm_dfr_boundary_average(int64_t n, const int32_t *layer, const int32_t *slot, const int32_t *slot_lo,
                            const int32_t *slot_hi, const double *buf, double *out, int apply, void *stream) {
    DM_STREAM_GUARD(stream);
    if (n < 0 || (n > 0 && (!layer || !slot || !slot_lo || !slot_hi || !buf || !out))) {
        dm::set_error("dm_dfr_boundary_average: invalid arguments");
        return DM_ERR_INVALID;
    }
    return dm::dfr_boundary_average(n, layer, slot, slot_lo, slot_hi, buf, out, apply != 0, stream);
}

int dm_dfr_to_nodes(const dm_flat *f, const double *x_il, double *x, void *stream) {
    DM_CHECK_FLAT(f);
    if (!x_il || !x) {
        dm::set_error("dm_dfr_to_nodes: null table");
        return DM_ERR_INVALID;
    }
    return dm::dfr_to_nodes(f->sweep, x_il, x, stream);
}

int dm_perturb_round(const dm_flat *f, const double *m0, const double *m1, double *lam, double delta, double boost,
                     uint64_t seed, int round, int8_t *values, int8_t *agrees, int *disagree, void *stream) {
    DM_CHECK_FLAT(f);
    if (!m0 || !m1 || !lam || !values || !agrees || !disagree) {
        dm::set_error("dm_perturb_round: null argument");
        return DM_ERR_INVALID;
    }
    DM_CUDA(cudaMemsetAsync(disagree, 0, sizeof(int), (cudaStream_t)stream));
    const_cast<dm_flat *>(f)->dec_B = nullptr;  // the duals move
    if (f->P == 0) return DM_OK;
    perturb_kernel<<<blocks_for(f->P, 256), 256, 0, (cudaStream_t)stream>>>(
        (int32_t)f->P, f->proc_ptr, f->proc_layers, f->pos_var, m0, m1, lam, delta, boost, seed, round, values,
        agrees, disagree);
    return check_stream_error("perturb_round");
}

// --- batched quasi-Newton control of a merged instance: dm_batch.cu -------
struct dm_batch {
    int device = 0;
    dm::BatchPlan plan;
    std::vector<void *> allocs;
};

int dm_batch_create(const dm_flat *f, int n, const int64_t *bdd_off, const int64_t *layer_off, void *stream,
                    dm_batch **out) {
    DM_CHECK_FLAT(f);
    if (n < 1 || !bdd_off || !layer_off || !out || bdd_off[0] != 0 || layer_off[0] != 0 || bdd_off[n] != f->nb ||
        layer_off[n] != f->L) {
        dm::set_error("dm_batch_create: offsets must partition the flat's diagrams and layers");
        return DM_ERR_INVALID;
    }
    for (int k = 0; k < n; ++k)
        if (bdd_off[k + 1] < bdd_off[k] || layer_off[k + 1] < layer_off[k]) {
            dm::set_error("dm_batch_create: offsets must be non-decreasing");
            return DM_ERR_INVALID;
        }
    auto b = std::make_unique<dm_batch>();
    b->device = f->device;
    const int rc = dm::batch_build(bdd_off, layer_off, n, b->plan, b->allocs, stream);
    if (rc) {
        for (void *p : b->allocs) cudaFree(p);
        return rc;
    }
    *out = b.release();
    return DM_OK;
}

void dm_batch_destroy(dm_batch *b) {
    if (!b) return;
    DevGuard guard(b->device);
    cudaDeviceSynchronize();
    for (void *p : b->allocs) cudaFreeAsync(p, 0);
    cudaGetLastError();
    delete b;
}

#define DM_CHECK_BATCH(b)                         \
    if (!(b)) {                                   \
        dm::set_error("null batch handle");       \
        return DM_ERR_INVALID;                    \
    }                                             \
    DevGuard dm_bguard_((b)->device)

int dm_batch_sum(const dm_batch *b, const double *x, double *out, void *stream) {
    DM_CHECK_BATCH(b);
    return dm::batch_sum(b->plan, x, out, stream);
}

int dm_batch_dot(const dm_batch *b, const double *const *a, const double *const *bb, const int8_t *active,
                 double *out, void *stream) {
    DM_CHECK_BATCH(b);
    return dm::batch_dot(b->plan, a, bb, active, out, stream);
}

int dm_batch_update(const dm_batch *b, int mode, double *x, const double *const *u, const double *coef,
                    const double *dot, const double *alpha, double *alpha_out, const int8_t *active, void *stream) {
    DM_CHECK_BATCH(b);
    if (mode < dm::kBatchCopy || mode > dm::kBatchAxpyHost) {
        dm::set_error("dm_batch_update: unknown mode");
        return DM_ERR_INVALID;
    }
    return dm::batch_update(b->plan, mode, x, u, coef, dot, alpha, alpha_out, active, stream);
}

int dm_batch_curvature(const dm_batch *b, const double *lam, double *lam_prev, const double *g, const double *g_prev,
                       double *const *s, double *const *y, const int8_t *active, void *stream) {
    DM_CHECK_BATCH(b);
    return dm::batch_curvature(b->plan, lam, lam_prev, g, g_prev, s, y, active, stream);
}

int dm_batch_step_search(const dm_flat *f, const dm_batch *b, const double *lam, const double *d,
                         const double *gamma_prev, const double *free_c, const double *min_ascent, double shrink,
                         double grow, int max_trials, const int8_t *active, double *bounds, double *sums,
                         double *state, void *stream) {
    DM_CHECK_FLAT(f);
    if (!b || !lam || !d || !gamma_prev || !free_c || !min_ascent || !active || !bounds || !sums || !state ||
        max_trials < 0) {
        dm::set_error("dm_batch_step_search: invalid arguments");
        return DM_ERR_INVALID;
    }
    int rc;
    if ((rc = dm::batch_step_init(b->plan, state, gamma_prev, active, stream))) return rc;
    // every trial is enqueued; stopped searches are evaluated too and ignored by their decision
    for (int t = 0; t <= max_trials; ++t) {
        if ((rc = dm::sweep_backward(f->sweep, lam, d, 0.0, nullptr, bounds, stream, state, b->plan.bdd_inst)))
            return rc;
        if ((rc = dm::batch_sum(b->plan, bounds, sums, stream))) return rc;
        if ((rc = dm::batch_decide(b->plan, sums, state, free_c, min_ascent, shrink, grow, max_trials, t, stream)))
            return rc;
    }
    return DM_OK;
}

int dm_init_duals(const dm_flat *f, const double *costs_by_var, double *lam, void *stream) {
    DM_CHECK_FLAT(f);
    const_cast<dm_flat *>(f)->dec_B = nullptr;  // new duals: recorded decisions are stale
    if (f->L == 0) return DM_OK;
    init_duals_kernel<<<blocks_for(f->L, 256), 256, 0, (cudaStream_t)stream>>>(
        (int32_t)f->L, f->layer_var, f->var_count, costs_by_var, lam);
    return check_stream_error("init_duals");
}

int dm_project_direction(const dm_flat *f, const double *d_hat, double *d, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->P == 0) return DM_OK;
    project_kernel<<<blocks_for(f->P, 256), 256, 0, (cudaStream_t)stream>>>(
        (int32_t)f->P, f->proc_ptr, f->proc_layers, d_hat, d);
    return check_stream_error("project_direction");
}

int dm_lambda_sums(const dm_flat *f, const double *lam, double *sums_by_var, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->P == 0) return DM_OK;
    lambda_sums_kernel<<<blocks_for(f->P, 256), 256, 0, (cudaStream_t)stream>>>(
        (int32_t)f->P, f->proc_ptr, f->proc_layers, f->pos_var, lam, sums_by_var);
    return check_stream_error("lambda_sums");
}

int dm_agreement_scores(const dm_flat *f, const double *m0, const double *m1, int8_t *agrees, double *score,
                        int8_t *preferred, void *stream) {
    DM_CHECK_FLAT(f);
    if (f->P == 0) return DM_OK;
    agreement_kernel<<<blocks_for(f->P, 256), 256, 0, (cudaStream_t)stream>>>(
        (int32_t)f->P, f->proc_ptr, f->proc_layers, f->pos_var, m0, m1, agrees, score, preferred);
    return check_stream_error("agreement_scores");
}

static int pairwise(const double *a, const double *b, int64_t n, double *out, cudaStream_t s) {
    if (n < 0 || n >= INT32_MAX || (n > 0 && !a) || !out) {
        dm::set_error("invalid reduction arguments");
        return DM_ERR_INVALID;
    }
    DevPlan *p;
    int rc = get_plan(n, s, &p);
    if (rc) return rc;
    if (b)
        pw_leaf_kernel<true><<<blocks_for((int64_t)p->nleaves * 8, 256), 256, 0, s>>>(p->nleaves, p->leaf_off, p->leaf_len, a, b, p->vals);
    else
        pw_leaf_kernel<false><<<blocks_for((int64_t)p->nleaves * 8, 256), 256, 0, s>>>(p->nleaves, p->leaf_off, p->leaf_len, a, nullptr, p->vals);
    pw_combine_kernel<<<1, 1024, 0, s>>>(p->nleaves, p->maxh, p->height_lo, p->left, p->right, p->root, p->vals, out);
    return check_stream_error("pairwise sum");
}

int dm_sum(const double *x, int64_t n, double *out, void *stream) {
    DM_STREAM_GUARD(stream);
    return pairwise(x, nullptr, n, out, (cudaStream_t)stream);
}

// Per-(device, length, stream) scratch of the chunked dot: chunk totals and
// the two-loop scalars (same per-stream ownership as the pairwise plans).
struct DotScratch {
    double *partial = nullptr;  // chunk totals (two buffers: the cooperative two-loop alternates them)
    double *slots = nullptr;    // two-loop scalars (dm_lbfgs_direction)
    unsigned *bar = nullptr;    // the cooperative two-loop's grid barrier {arrivals, generation, watchdog}
};
static std::map<ScratchKey, DotScratch> g_dot;
constexpr int kMaxPairs = 64;

static int dot_scratch(int64_t n, void *stream, bool slots, DotScratch **out) {
    const int64_t nch = (n + dm::kDotChunk - 1) / dm::kDotChunk;
    int dev;
    DM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_plan_mu);
    auto key = ScratchKey(dev, n, (uintptr_t)stream);
    auto it = g_dot.find(key);
    if (it == g_dot.end()) {
        DotScratch d;
        DM_CUDA(cudaMalloc((void **)&d.partial, 2 * nch * sizeof(double)));
        it = g_dot.emplace(key, d).first;
    }
    if (slots && !it->second.slots) {
        DM_CUDA(cudaMalloc((void **)&it->second.slots, (3 * kMaxPairs + 1) * sizeof(double)));
        DM_CUDA(cudaMalloc((void **)&it->second.bar, 4 * sizeof(unsigned)));
        DM_CUDA(cudaMemset(it->second.bar, 0, 4 * sizeof(unsigned)));
    }
    *out = &it->second;
    return DM_OK;
}

// Frees every cached reduction plan and dot scratch (all devices): the
// caches are keyed by (device, length, stream) and otherwise live for the
// process — a long-running service calls this between batches, with no
// work in flight.
int dm_release_caches(void) {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    auto release = [&](int dev, std::initializer_list<void *> ptrs) {
        cudaSetDevice(dev);
        cudaDeviceSynchronize();
        for (void *p : ptrs)
            if (p) cudaFree(p);
    };
    for (auto &kv : g_plans) {
        const DevPlan &p = kv.second;
        release(std::get<0>(kv.first), {p.leaf_off, p.leaf_len, p.left, p.right, p.height_lo, p.vals});
    }
    g_plans.clear();
    for (auto &kv : g_dot) release(std::get<0>(kv.first), {kv.second.partial, kv.second.slots, kv.second.bar});
    g_dot.clear();
    cudaSetDevice(cur);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "release caches");
    return DM_OK;
}

int dm_dot(const double *a, const double *b, int64_t n, double *out, void *stream) {
    DM_STREAM_GUARD(stream);
    if (!a || !b || !out || n < 0) {
        if (n == 0 && out) {
            cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)stream);  // empty dot = 0.0
            return check_stream_error("dm_dot");
        }
        dm::set_error("dm_dot needs two vectors and an output");
        return DM_ERR_INVALID;
    }
    if (n == 0) {
        DM_CUDA(cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)stream));
        return DM_OK;
    }
    DotScratch *sc;
    if (int rc = dot_scratch(n, stream, false, &sc)) return rc;
    return dm::chunk_dot(a, b, n, sc->partial, out, stream);
}

int dm_lbfgs_direction(const double *g, const double *const *s, const double *const *y, const double *rho,
                       const double *sy, int m, int64_t n, double *d, void *stream) {
    DM_STREAM_GUARD(stream);
    if (!g || !s || !y || !rho || !sy || !d || m < 1 || m > kMaxPairs || n < 1) {
        dm::set_error("dm_lbfgs_direction: needs g, d, 1 <= m <= 64 pairs and n >= 1");
        return DM_ERR_INVALID;
    }
    for (int i = 0; i < m; ++i)
        if (!s[i] || !y[i]) {
            dm::set_error("dm_lbfgs_direction: null pair vector");
            return DM_ERR_INVALID;
        }
    DotScratch *sc;
    if (int rc = dot_scratch(n, stream, true, &sc)) return rc;
    return dm::lbfgs_two_loop(g, s, y, rho, sy, m, n, d, sc->slots, sc->partial, stream, sc->bar);
}

int dm_curvature_pair(const double *lam, double *lam_prev, const double *g, const double *g_prev, double *s,
                      double *y, int64_t n, double *sy, void *stream) {
    DM_STREAM_GUARD(stream);
    if (!lam || !lam_prev || !g || !g_prev || !s || !y || !sy || n < 1) {
        dm::set_error("dm_curvature_pair: needs six vectors of length n >= 1 and an output");
        return DM_ERR_INVALID;
    }
    DotScratch *sc;
    if (int rc = dot_scratch(n, stream, false, &sc)) return rc;
    return dm::curvature_pair(lam, lam_prev, g, g_prev, s, y, n, sc->partial, sy, stream);
}

int dm_axpy_dev(double *x, const double *y, double alpha_host, const double *dot_dev, double *alpha_out, int64_t n,
                void *stream) {
    DM_STREAM_GUARD(stream);
    axpy_dev_kernel<<<grid_stride_blocks(n), 256, 0, (cudaStream_t)stream>>>(x, y, alpha_host, dot_dev, alpha_out, n);
    return check_stream_error("axpy_dev");
}

int dm_scale_dev(double *x, double num_host, const double *den_dev, int64_t n, void *stream) {
    DM_STREAM_GUARD(stream);
    scale_dev_kernel<<<grid_stride_blocks(n), 256, 0, (cudaStream_t)stream>>>(x, num_host, den_dev, n);
    return check_stream_error("scale_dev");
}

int dm_lbfgs_up(double *x, const double *s, const double *alpha_dev, double rho_host, const double *dot_dev, int64_t n,
                void *stream) {
    DM_STREAM_GUARD(stream);
    lbfgs_up_kernel<<<grid_stride_blocks(n), 256, 0, (cudaStream_t)stream>>>(x, s, alpha_dev, rho_host, dot_dev, n);
    return check_stream_error("lbfgs_up");
}

int dm_axpy_host(double *x, double gamma, const double *y, int64_t n, void *stream) {
    DM_STREAM_GUARD(stream);
    axpy_host_kernel<<<grid_stride_blocks(n), 256, 0, (cudaStream_t)stream>>>(x, gamma, y, n);
    return check_stream_error("axpy_host");
}

int dm_sub(double *out, const double *a, const double *b, int64_t n, void *stream) {
    DM_STREAM_GUARD(stream);
    sub_kernel<<<grid_stride_blocks(n), 256, 0, (cudaStream_t)stream>>>(out, a, b, n);
    return check_stream_error("sub");
}

}  // extern "C"

namespace dm {
int pairwise_device(const double *x, int64_t n, double *out, void *stream) {
    return pairwise(x, nullptr, n, out, (cudaStream_t)stream);
}
}  // namespace dm

