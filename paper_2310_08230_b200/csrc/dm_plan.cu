// Exact-pass schedules and node-parallel copy records built on the device.
//
// The host builder (build_mma_schedule, dm_host.cpp) walks the visitation
// order once per direction: a position's level is one more than the deepest
// level among the previous layers (forward) / next layers (backward) of its
// copies' diagrams, then positions are bucketed by level keeping visitation
// order inside a level.  Here the same DAG is walked by a persistent kernel
// that resolves each position's level as soon as its predecessors' levels are
// published (self-validating data: -1 until written), and a stable radix sort
// by level replaces the bucketing, so pos_order is identical to the host's.
// tests/test_gpu_parity.py compares both.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#include "dm_internal.h"

namespace dm {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kPlanWaitNs = 4000000000ull;  // watchdog of the level walk

__device__ __forceinline__ int ld_relaxed_i32(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_i32(int32_t *p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t now_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// layer -> position that visits it
__global__ void layer_pos_kernel(const int32_t *proc_ptr, const int32_t *proc_layers, int64_t P, int32_t *layer_pos) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x)
        for (int32_t t = proc_ptr[p]; t < proc_ptr[p + 1]; ++t) layer_pos[proc_layers[t]] = (int32_t)p;
}

// visitation index k -> position (forward: k, backward: P-1-k), and the
// level keys primed with the sentinel; positions without copies get INT_MAX
// (they sort last and are cut off)
__global__ void level_init_kernel(const int32_t *proc_ptr, int64_t P, bool forward, int32_t *order_in,
                                  int32_t *level) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = forward ? k : P - 1 - k;
        order_in[k] = (int32_t)p;
        level[p] = proc_ptr[p + 1] == proc_ptr[p] ? INT_MAX : -1;
    }
}

// Persistent walk: warps take 32 consecutive visitation indices from a
// counter; a position depends only on positions visited before it, which
// warps that took earlier chunks hold (or the same warp), so the walk cannot
// deadlock.  Consecutive positions mostly share diagrams, so a chunk is
// often one dependency chain: levels resolved inside the chunk are handed
// on through the warp's shared-memory row (one __syncwarp per step) instead
// of a global store -> poll round trip.
constexpr int kWalkWarps = 8;
__global__ void __launch_bounds__(256) level_walk_kernel(const int32_t *proc_ptr, const int32_t *proc_layers,
                                                         const int32_t *layer_bdd, const int32_t *bdd_layer_lo,
                                                         const int32_t *layer_pos, int64_t P, bool forward,
                                                         int32_t *level, int *counter, int *status) {
    __shared__ int32_t row_s[kWalkWarps][32];
    const int lane = threadIdx.x & 31;
    volatile int32_t *row = row_s[threadIdx.x >> 5];
    while (true) {
        int base = 0;
        if (lane == 0) base = atomicAdd(counter, 32);
        base = __shfl_sync(kFull, base, 0);
        if (base >= P) return;
        const int64_t k = base + lane;
        const int64_t p = forward ? k : P - 1 - k;
        bool done = k >= P;
        int32_t t = 0, hi = 0, lev = 0;
        if (!done) {
            t = proc_ptr[p];
            hi = proc_ptr[p + 1];
            done = t == hi;
        }
        row[lane] = -1;
        __syncwarp();
        unsigned spins = 0;
        uint64_t t0 = 0;
        while (!__all_sync(kFull, done)) {
            if (!done) {
                for (; t < hi; ++t) {
                    const int32_t l = proc_layers[t], j = layer_bdd[l];
                    const bool first = forward ? l == bdd_layer_lo[j] : l + 1 == bdd_layer_lo[j + 1];
                    if (first) continue;
                    const int32_t q = layer_pos[forward ? l - 1 : l + 1];
                    const int64_t kq = forward ? q : P - 1 - q;
                    const int v = kq >= base ? row[kq - base] : ld_relaxed_i32(level + q);
                    if (v < 0) break;
                    lev = max(lev, v + 1);
                }
                if (t == hi) {
                    st_relaxed_i32(level + p, lev);
                    row[lane] = lev;
                    done = true;
                }
            }
            __syncwarp();
            if ((++spins & 255u) == 0) {
                const uint64_t now = now_ns();
                if (t0 == 0) t0 = now;
                if (*(volatile int *)status || now - t0 > kPlanWaitNs) {
                    if (lane == 0) atomicExch(status, 1);
                    return;
                }
            }
        }
    }
}

__global__ void layer_flags_kernel(const int32_t *layer_bdd, const int32_t *bdd_layer_lo, int64_t L, uint8_t *flags) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = layer_bdd[l];
        flags[l] = (uint8_t)((l == bdd_layer_lo[j] ? 1 : 0) | (l + 1 == bdd_layer_lo[j + 1] ? 2 : 0));
    }
}

// one packed record per (position, copy slot): {layer, first node,
// width | next width << 8 | flags << 16 | copies << 24, 0}; unused slots
// {-1, 0, copies << 24, 0} (the node-parallel kernels' np_lane)
__global__ void np_records_kernel(const int32_t *proc_ptr, const int32_t *proc_layers, const int32_t *lnl,
                                  const uint8_t *flags, const int32_t *order, int64_t n, int4 *rec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * 8; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = order ? order[i >> 3] : i >> 3;
        const int c = (int)(i & 7);
        const int32_t lo = proc_ptr[p], k = proc_ptr[p + 1] - lo;
        int4 r{-1, 0, (int)((unsigned)k << 24), 0};
        if (c < k) {
            const int32_t l = proc_layers[lo + c];
            const unsigned fl = flags[l];
            const int32_t w = lnl[l + 1] - lnl[l];
            const int32_t wn = (fl & 2) ? 0 : lnl[l + 2] - lnl[l + 1];
            r.x = l;
            r.y = lnl[l];
            r.z = (int)((unsigned)w | ((unsigned)wn << 8) | (fl << 16) | ((unsigned)k << 24));
        }
        rec[i] = r;
    }
}

__global__ void gather_levels_kernel(const int32_t *order_in, const int32_t *level, int64_t P, int32_t *keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x)
        keys[k] = level[order_in[k]];
}


// ---- interleaved sweep layout (build_sweep_layout, dm_layout.cpp) ----------

// shape key: more layers first, then more nodes (ties: diagram id, the
// radix sort being stable over ascending ids)
__global__ void sweep_keys_kernel(const int32_t *bl, const int32_t *lnl, int64_t nb, uint64_t *key, int32_t *idx) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t L = (uint64_t)(bl[j + 1] - bl[j]), Nn = (uint64_t)(lnl[bl[j + 1]] - lnl[bl[j]]);
        key[j] = (~L << 32) | (~Nn & 0xffffffffull);
        idx[j] = (int32_t)j;
    }
}

// lanes of each group and its position count (the first lane has the most layers)
__global__ void sweep_groups_kernel(const int32_t *bl, const int32_t *sorted, int64_t nb, int64_t groups,
                                    int32_t *grp_bdd, int32_t *grp_npos) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < groups * 32;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = i < nb ? sorted[i] : -1;
        grp_bdd[i] = j;
        if ((i & 31) == 0) grp_npos[i >> 5] = bl[j + 1] - bl[j];
    }
}

__global__ void sweep_total_kernel(const int32_t *cnt, const int64_t *excl, int64_t n, int64_t *total) {
    *total = n ? excl[n - 1] + cnt[n - 1] : 0;
}

// widest layer at each position of each group (warp per group)
__global__ void sweep_widths_kernel(const int32_t *bl, const int32_t *lnl, const int32_t *grp_bdd,
                                    const int32_t *grp_npos, const int64_t *grp_pos_lo, int64_t groups,
                                    int32_t *pos_width, int32_t *grp_width, unsigned long long *max_width) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned wmax = 0;
    for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < groups; g += warps) {
        const int32_t j = grp_bdd[g * 32 + lane], K = grp_npos[g];
        const int32_t nl = j >= 0 ? bl[j + 1] - bl[j] : 0, top = j >= 0 ? bl[j + 1] - 1 : 0;
        unsigned gmax = 0;
        for (int32_t k = 0; k < K; ++k) {
            const unsigned w = k < nl ? (unsigned)(lnl[top - k + 1] - lnl[top - k]) : 0u;
            const unsigned m = __reduce_max_sync(kFull, w);
            if (lane == 0) pos_width[grp_pos_lo[g] + k] = (int32_t)m;
            gmax = max(gmax, m);
        }
        if (lane == 0) grp_width[g] = (int32_t)gmax;
        wmax = max(wmax, gmax);
    }
    if (lane == 0 && wmax) atomicMax(max_width, (unsigned long long)wmax);
}

// node slots interleaved by lane, arc targets local to the next layer
// (-1 FALSE and padding, -2 TRUE); warp per group, coalesced stores
__global__ void sweep_fill_kernel(const int32_t *bl, const int32_t *lnl, const int32_t *zero_t, const int32_t *one_t,
                                  const int32_t *grp_bdd, const int32_t *grp_npos, const int64_t *grp_pos_lo,
                                  const int32_t *pos_width, const int64_t *pos_slot, int64_t groups, int32_t *zl,
                                  int32_t *ol) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < groups; g += warps) {
        const int32_t j = grp_bdd[g * 32 + lane], K = grp_npos[g];
        const int32_t nl = j >= 0 ? bl[j + 1] - bl[j] : 0, top = j >= 0 ? bl[j + 1] - 1 : 0;
        const int64_t p0 = grp_pos_lo[g];
        for (int32_t k = 0; k < K; ++k) {
            const int32_t wk = pos_width[p0 + k];
            const int64_t base = pos_slot[p0 + k] * 32 + lane;
            int32_t v0 = 0, w = 0, next0 = 0;
            if (k < nl) {
                const int32_t l = top - k;
                v0 = lnl[l];
                w = lnl[l + 1] - v0;
                next0 = lnl[l + 1];
            }
            for (int32_t v = 0; v < wk; ++v) {
                int32_t a = kFalse, b = kFalse;
                if (v < w) {
                    a = zero_t[v0 + v];
                    b = one_t[v0 + v];
                    a = a >= 0 ? a - next0 : a;
                    b = b >= 0 ? b - next0 : b;
                }
                zl[base + (int64_t)v * 32] = a;
                ol[base + (int64_t)v * 32] = b;
            }
        }
    }
}

// forward publish descriptors (build_relax_by_layer, dm_layout.cpp): a
// target with two sources of one arc kind, or a layer wider than 8,
// raises *fail and the tree publish is used instead
__global__ void relax_kernel(const int32_t *layer_bdd, const int32_t *bl, const int32_t *lnl, const int32_t *zero_t,
                             const int32_t *one_t, int64_t L, uint64_t *desc_out, unsigned long long *fail) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x) {
        uint64_t desc = ~0ull;
        const int32_t j = layer_bdd[l];
        if (l + 1 != bl[j + 1]) {
            const int32_t v0 = lnl[l], w = lnl[l + 1] - v0, n0 = lnl[l + 1], wn = lnl[l + 2] - n0;
            bool ok = w <= 8 && wn <= 8;
            for (int32_t i = 0; i < w && ok; ++i) {
                const int32_t tg[2] = {zero_t[v0 + i], one_t[v0 + i]};
                for (int k = 0; k < 2 && ok; ++k) {
                    if (tg[k] < 0) continue;
                    const int32_t u = tg[k] - n0;
                    const int sh = 8 * u + 4 * k;
                    if (u < 0 || u >= wn || ((desc >> sh) & 15) != 15) {
                        ok = false;
                        break;
                    }
                    desc = (desc & ~(15ull << sh)) | ((uint64_t)i << sh);
                }
            }
            if (!ok) atomicOr(fail, 1ull);
        }
        desc_out[l] = desc;
    }
}

int grid_for(int64_t n, int threads);

int grid_for(int64_t n, int threads) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16));
}

}  // namespace

int device_layer_flags(const int32_t *layer_bdd, const int32_t *bdd_layer_lo, int64_t L, uint8_t *flags,
                       void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    if (L > 0) layer_flags_kernel<<<grid_for(L, 256), 256, 0, s>>>(layer_bdd, bdd_layer_lo, L, flags);
    const cudaError_t e = cudaGetLastError();
    if (e) set_error(std::string("layer flags: ") + cudaGetErrorString(e));
    return e ? -1 : 0;
}

int device_np_records(const int32_t *proc_ptr, const int32_t *proc_layers, const int32_t *lnl, const uint8_t *flags,
                      const int32_t *order, int64_t P, void *rec, void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    if (P > 0)
        np_records_kernel<<<grid_for(P * 8, 256), 256, 0, s>>>(proc_ptr, proc_layers, lnl, flags, order, P,
                                                               (int4 *)rec);
    const cudaError_t e = cudaGetLastError();
    if (e) set_error(std::string("copy records: ") + cudaGetErrorString(e));
    return e ? -1 : 0;
}

// Both directions' level orders, stream-ordered (no host synchronisation).
// `fw_order`/`bw_order` get the positions with copies sorted by (level,
// visitation index) in their first `nvalid` entries and `fw_level`/`bw_level`
// (P entries each) the matching levels; `words` (8 device ints) receives
// {fw queue, fw status, bw queue, bw status, fw depth - 1, bw depth - 1}.
// A non-zero status after the stream synchronises means a walk stalled.
int device_level_orders(const int32_t *proc_ptr, const int32_t *proc_layers, const int32_t *layer_bdd,
                        const int32_t *bdd_layer_lo, int64_t P, int64_t L, int64_t nvalid, int32_t *fw_order,
                        int32_t *fw_level, int32_t *bw_order, int32_t *bw_level, int *words, void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    auto fail = [&](cudaError_t e, const char *what) {
        set_error(std::string("device schedule: ") + what + ": " + cudaGetErrorString(e));
        return -1;
    };
    cudaError_t e;
    if ((e = cudaMemsetAsync(words, 0, 8 * sizeof(int), s))) return fail(e, "memset");
    if (P == 0 || nvalid == 0) return 0;
    // the two directions walk concurrently on two streams; each walk is
    // latency-bound and its polls contend in L2, so it runs on a small grid
    // (DM_WALK_DIV: 1/32 of the resident blocks)
    int32_t *layer_pos = nullptr, *order_in[2] = {nullptr, nullptr}, *lev[2] = {nullptr, nullptr};
    void *tmp[2] = {nullptr, nullptr};
    size_t tmp_bytes = 0;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const int32_t *)nullptr, (int32_t *)nullptr,
                                             (const int32_t *)nullptr, (int32_t *)nullptr, (int)P, 0, 31, s)))
        return fail(e, "sort size");
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    if ((e = cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking)) ||
        (e = cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming)) ||
        (e = cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming)))
        return fail(e, "stream");
    struct Cleanup {
        cudaStream_t s2;
        cudaEvent_t *ev;
        ~Cleanup() {
            if (s2) cudaStreamDestroy(s2);  // released once its queued work completes
            for (int i = 0; i < 2; ++i)
                if (ev[i]) cudaEventDestroy(ev[i]);
        }
    } cleanup{s2, ev};
    if ((e = cudaMallocAsync((void **)&layer_pos, std::max<int64_t>(L, 1) * 4, s)))
        return fail(e, "allocation");
    for (int d = 0; d < 2; ++d)
        if ((e = cudaMallocAsync((void **)&order_in[d], P * 4, s)) || (e = cudaMallocAsync((void **)&lev[d], P * 4, s)) ||
            (e = cudaMallocAsync(&tmp[d], tmp_bytes, s)))
            return fail(e, "allocation");
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_walk_kernel, 256, 0);
    const char *wd = std::getenv("DM_WALK_DIV");
    const int walk_div = std::max(wd ? std::atoi(wd) : 32, 1);  // measured: 65 ms at 1 -> 12 ms at 16..128 (C2)
    layer_pos_kernel<<<grid_for(P, 256), 256, 0, s>>>(proc_ptr, proc_layers, P, layer_pos);
    if ((e = cudaEventRecord(ev[0], s)) || (e = cudaStreamWaitEvent(s2, ev[0], 0))) return fail(e, "event");
    int rc = 0;
    for (int dir = 0; dir < 2 && rc == 0; ++dir) {
        const bool forward = dir == 0;
        const cudaStream_t sd = forward ? s : s2;
        int32_t *order = forward ? fw_order : bw_order, *lv = forward ? fw_level : bw_level;
        level_init_kernel<<<grid_for(P, 256), 256, 0, sd>>>(proc_ptr, P, forward, order_in[dir], lev[dir]);
        level_walk_kernel<<<std::max(sms * per_sm / walk_div, 1), 256, 0, sd>>>(
            proc_ptr, proc_layers, layer_bdd, bdd_layer_lo, layer_pos, P, forward, lev[dir], words + 2 * dir,
            words + 2 * dir + 1);
        // keys in visitation order (lv is scratch until the sorted keys land in it)
        gather_levels_kernel<<<grid_for(P, 256), 256, 0, sd>>>(order_in[dir], lev[dir], P, lv);
        if ((e = cudaGetLastError())) {
            rc = fail(e, "launch");
            break;
        }
        if ((e = cub::DeviceRadixSort::SortPairs(tmp[dir], tmp_bytes, lv, lev[dir], order_in[dir], order, (int)P, 0,
                                                 31, sd)) ||
            (e = cudaMemcpyAsync(lv, lev[dir], P * 4, cudaMemcpyDeviceToDevice, sd)) ||
            (e = cudaMemcpyAsync(words + 4 + dir, lv + nvalid - 1, 4, cudaMemcpyDeviceToDevice, sd)))
            rc = fail(e, "sort");
    }
    if (!rc && ((e = cudaEventRecord(ev[1], s2)) || (e = cudaStreamWaitEvent(s, ev[1], 0)))) rc = fail(e, "event");
    if (rc) cudaStreamSynchronize(s2);
    cudaFreeAsync(layer_pos, s);
    for (int d = 0; d < 2; ++d) {
        cudaFreeAsync(order_in[d], s);
        cudaFreeAsync(lev[d], s);
        cudaFreeAsync(tmp[d], s);
    }
    return rc;
}

// ---- sweep layout + relax on the device -------------------------------------

namespace {
template <typename T>
cudaError_t dalloc(T **p, int64_t n, cudaStream_t s, std::vector<void *> &allocs, int64_t &bytes) {
    const size_t b = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
    const cudaError_t e = cudaMallocAsync((void **)p, b, s);
    if (e == cudaSuccess) {
        allocs.push_back(*p);
        bytes += (int64_t)b;
    }
    return e;
}
}  // namespace

int device_sweep_layout(const int32_t *bl, const int32_t *lnl, int64_t nb, SweepDev &sd, std::vector<void *> &allocs,
                        int64_t &bytes, void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    auto fail = [&](cudaError_t e, const char *what) {
        set_error(std::string("device sweep layout: ") + what + ": " + cudaGetErrorString(e));
        return -1;
    };
    cudaError_t e;
    const int64_t groups = (nb + 31) / 32;
    sd.groups = groups;
    sd.bdd_layer_lo = bl;
    sd.lnl = lnl;
    if (nb == 0) return 0;
    uint64_t *key = nullptr, *key2 = nullptr;
    int32_t *idx = nullptr, *idx2 = nullptr, *grp_bdd = nullptr, *grp_npos = nullptr, *pos_width = nullptr;
    int32_t *grp_width = nullptr;
    int64_t *grp_pos_lo = nullptr, *pos_slot = nullptr, *stats = nullptr;
    int32_t *zl = nullptr, *ol = nullptr;
    void *tmp = nullptr;
    size_t tmp_sort = 0, tmp_scan1 = 0, tmp_scan2 = 0;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                             (const int32_t *)nullptr, (int32_t *)nullptr, (int)nb, 0, 64, s)) ||
        (e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan1, (const int32_t *)nullptr, (int64_t *)nullptr,
                                           (int)groups, s)))
        return fail(e, "temp size");
    std::vector<void *> scratch;
    int64_t scratch_bytes = 0;
    if ((e = dalloc(&key, nb, s, scratch, scratch_bytes)) || (e = dalloc(&key2, nb, s, scratch, scratch_bytes)) ||
        (e = dalloc(&idx, nb, s, scratch, scratch_bytes)) || (e = dalloc(&idx2, nb, s, scratch, scratch_bytes)) ||
        (e = dalloc(&stats, 4, s, scratch, scratch_bytes)) || (e = dalloc(&grp_bdd, groups * 32, s, allocs, bytes)) ||
        (e = dalloc(&grp_npos, groups, s, allocs, bytes)) || (e = dalloc(&grp_width, groups, s, allocs, bytes)) ||
        (e = dalloc(&grp_pos_lo, groups + 1, s, allocs, bytes)))
        return fail(e, "allocation");
    auto release = [&] {
        for (void *p : scratch) cudaFreeAsync(p, s);
        if (tmp) cudaFreeAsync(tmp, s);
    };
    size_t tmp_bytes = std::max(tmp_sort, tmp_scan1);
    if ((e = cudaMallocAsync(&tmp, tmp_bytes, s))) return release(), fail(e, "allocation");
    int rc = 0;
    int64_t host[4] = {0, 0, 0, 0};
    const char *verbose = std::getenv("DM_VERBOSE");
    const bool vb = verbose && std::atoi(verbose) >= 2;
    auto T0 = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (vb)
            std::fprintf(stderr, "  [sweep layout] %s %.4f\n", what,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - T0).count());
    };
    do {
        if ((e = cudaMemsetAsync(stats, 0, 4 * sizeof(int64_t), s))) break;
        sweep_keys_kernel<<<grid_for(nb, 256), 256, 0, s>>>(bl, lnl, nb, key, idx);
        if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_sort, key, key2, idx, idx2, (int)nb, 0, 64, s))) break;
        sweep_groups_kernel<<<grid_for(groups * 32, 256), 256, 0, s>>>(bl, idx2, nb, groups, grp_bdd, grp_npos);
        if ((e = cub::DeviceScan::ExclusiveSum(tmp, tmp_scan1, grp_npos, grp_pos_lo, (int)groups, s))) break;
        sweep_total_kernel<<<1, 1, 0, s>>>(grp_npos, grp_pos_lo, groups, grp_pos_lo + groups);
        mark("queued");
        if ((e = cudaMemcpyAsync(host, grp_pos_lo + groups, 8, cudaMemcpyDeviceToHost, s)) ||
            (e = cudaStreamSynchronize(s)))
            break;
        mark("positions");
        const int64_t npos_total = host[0];
        if ((e = dalloc(&pos_width, npos_total, s, allocs, bytes)) ||
            (e = dalloc(&pos_slot, npos_total, s, allocs, bytes)))
            break;
        sweep_widths_kernel<<<grid_for(groups * 32, 256), 256, 0, s>>>(bl, lnl, grp_bdd, grp_npos, grp_pos_lo, groups,
                                                                       pos_width, grp_width,
                                                                       (unsigned long long *)stats + 1);
        if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan2, pos_width, pos_slot, (int)npos_total, s))) break;
        if (tmp_scan2 > tmp_bytes) {
            cudaFreeAsync(tmp, s);
            tmp = nullptr;
            if ((e = cudaMallocAsync(&tmp, tmp_scan2, s))) break;
            tmp_bytes = tmp_scan2;
        }
        if ((e = cub::DeviceScan::ExclusiveSum(tmp, tmp_scan2, pos_width, pos_slot, (int)npos_total, s))) break;
        sweep_total_kernel<<<1, 1, 0, s>>>(pos_width, pos_slot, npos_total, stats);
        // the longest diagram's layers: the first group's (groups are longest first)
        if ((e = cudaMemcpyAsync(stats + 2, grp_npos, sizeof(int32_t), cudaMemcpyDeviceToDevice, s))) break;
        if ((e = cudaMemcpyAsync(host, stats, 24, cudaMemcpyDeviceToHost, s)) || (e = cudaStreamSynchronize(s)))
            break;
        mark("slots");
        const int64_t slots = host[0];
        if (slots * 32 >= INT32_MAX) {
            set_error("sweep layout exceeds the int32 element range");
            rc = -2;
            break;
        }
        sd.max_width = (int32_t)host[1];
        sd.max_layers = (int32_t)(host[2] & 0xffffffff);
        sd.slots = slots;
        if ((e = dalloc(&zl, slots * 32, s, allocs, bytes)) || (e = dalloc(&ol, slots * 32, s, allocs, bytes))) break;
        e = cudaGetLastError();
        mark("allocated");
    } while (false);
    release();
    if (rc) return rc;
    if (e) return fail(e, "build");
    sd.grp_bdd = grp_bdd;
    sd.grp_npos = grp_npos;
    sd.grp_width = grp_width;
    sd.grp_pos_lo = grp_pos_lo;
    sd.pos_width = pos_width;
    sd.pos_slot = pos_slot;
    sd.zl = zl;
    sd.ol = ol;
    return 0;
}

int device_sweep_fill(const SweepDev &sd, const int32_t *zero_t, const int32_t *one_t, void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    if (sd.groups > 0)
        sweep_fill_kernel<<<grid_for(sd.groups * 32, 256), 256, 0, s>>>(
            sd.bdd_layer_lo, sd.lnl, zero_t, one_t, sd.grp_bdd, sd.grp_npos, sd.grp_pos_lo, sd.pos_width, sd.pos_slot,
            sd.groups, const_cast<int32_t *>(sd.zl), const_cast<int32_t *>(sd.ol));
    const cudaError_t e = cudaGetLastError();
    if (e) set_error(std::string("sweep layout fill: ") + cudaGetErrorString(e));
    return e ? -1 : 0;
}

int device_relax(const int32_t *layer_bdd, const int32_t *bl, const int32_t *lnl, const int32_t *zero_t,
                 const int32_t *one_t, int64_t L, uint64_t *desc, unsigned long long *fail, void *stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    if (L > 0) relax_kernel<<<grid_for(L, 256), 256, 0, s>>>(layer_bdd, bl, lnl, zero_t, one_t, L, desc, fail);
    const cudaError_t e = cudaGetLastError();
    if (e) set_error(std::string("relax descriptors: ") + cudaGetErrorString(e));
    return e ? -1 : 0;
}

}  // namespace dm
