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

#include <string>

#include "dm_internal.h"

#define DM_INF __longlong_as_double(0x7ff0000000000000LL)

namespace {

constexpr int kSweepThreads = 128;

template <int W, bool kTrial, bool kStore>
__global__ void __launch_bounds__(kSweepThreads) sweep_backward_kernel(dm::SweepDev s, const double *__restrict__ lam,
                                                                        const double *__restrict__ d, double gamma,
                                                                        double *__restrict__ B,
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
    double *nb = sm + threadIdx.x;                       // distances of position k-1 (next layer)
    double *cur = sm + W * kSweepThreads + threadIdx.x;  // distances of position k
    for (int32_t k = 0; k < K; ++k) {
        const int32_t w = s.pos_width[p0 + k];
        const int64_t slot = s.pos_slot[p0 + k];
        const bool act = k < nj;
        const int32_t l = l0 + nj - 1 - k;
        double lam_l = 0.0;
        int32_t vbase = 0, wl = 0;
        if (act) {
            lam_l = lam[l];
            if (kTrial) lam_l = __dadd_rn(lam_l, __dmul_rn(gamma, d[l]));
            if (kStore) {
                vbase = s.lnl[l];
                wl = s.lnl[l + 1] - vbase;
            }
        }
#pragma unroll 4
        for (int32_t i = 0; i < w; ++i) {
            const int32_t a = s.zl[(slot + i) * 32 + lane];
            const int32_t b = s.ol[(slot + i) * 32 + lane];
            const double c0 = a == dm::kTrue ? 0.0 : (a == dm::kFalse ? DM_INF : nb[a * kSweepThreads]);
            const double c1 = b == dm::kTrue ? lam_l : (b == dm::kFalse ? DM_INF : __dadd_rn(lam_l, nb[b * kSweepThreads]));
            const double v = (c0 <= c1) ? c0 : c1;
            cur[i * kSweepThreads] = v;
            if (kStore && i < wl) B[vbase + i] = v;
        }
        double *t = nb;
        nb = cur;
        cur = t;
        if (act && k == nj - 1) bounds[j] = nb[0];  // root layer: single node
    }
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
                    double *bounds, cudaStream_t st) {
    const int blocks = (int)((s.groups * 32 + kSweepThreads - 1) / kSweepThreads);
    const size_t smem = 2 * W * kSweepThreads * sizeof(double);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(sweep_backward_kernel<W, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep_backward_kernel<W, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep_backward_kernel<W, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep_backward_kernel<W, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (d && B)
        sweep_backward_kernel<W, true, true><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds);
    else if (d)
        sweep_backward_kernel<W, true, false><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds);
    else if (B)
        sweep_backward_kernel<W, false, true><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds);
    else
        sweep_backward_kernel<W, false, false><<<blocks, kSweepThreads, smem, st>>>(s, lam, d, gamma, B, bounds);
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
                   void *stream) {
    if (s.groups == 0) return DM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (s.max_width <= 8) return launch_backward<8>(s, lam, d, gamma, B, bounds, st);
    if (s.max_width <= 16) return launch_backward<16>(s, lam, d, gamma, B, bounds, st);
    return launch_backward<32>(s, lam, d, gamma, B, bounds, st);
}

int sweep_forward(const SweepDev &s, const double *lam, double *F, double *bounds, void *stream) {
    if (s.groups == 0) return DM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (s.max_width <= 8) return launch_forward<8>(s, lam, F, bounds, st);
    if (s.max_width <= 16) return launch_forward<16>(s, lam, F, bounds, st);
    return launch_forward<32>(s, lam, F, bounds, st);
}

}  // namespace dm
