// Poll round-trip under load (GPU tool, standalone): every warp of a
// persistent grid repeatedly issues 8 relaxed gpu-scope loads per lane and
// waits for them, either scattered (each lane its own 64-byte run, like the
// exact passes' layer polls) or coalesced (a warp reads 8 x 256 contiguous
// bytes).  Reports the mean time of one poll.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pollbench tools/pollbench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int kKind>
__device__ __forceinline__ unsigned long long ldr(const double *p) {
    unsigned long long v;
    if (kKind == 0)
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (kKind == 1)
        asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (kKind == 2)
        asm volatile("ld.volatile.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <bool kCoalesced, int kKind>
__global__ void poll(const double *buf, size_t nwords, int iters, unsigned long long *out, unsigned long long *sink) {
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // pseudo-random base per warp/lane
    size_t h = (warp * 0x9E3779B97F4A7C15ull + lane * 0xBF58476D1CE4E5B9ull) % (nwords / 2048);
    unsigned long long acc = 0;
    const unsigned long long t0 = now();
    for (int it = 0; it < iters; ++it) {
        const size_t base = ((h + it * 7919) % (nwords / 2048)) * 2048;
        unsigned long long v[8];
        if (kCoalesced) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = ldr<kKind>(buf + base + i * 32 + lane);
        } else {
            const size_t b = base + lane * 64;
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = ldr<kKind>(buf + b + i);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += v[i];
        acc = __shfl_sync(0xffffffffu, acc, 0);  // the whole warp waits for all lanes
    }
    const unsigned long long t1 = now();
    if (lane == 0) out[warp] = (t1 - t0) / iters;
    if (acc == 42) sink[0] = acc;
}

int main() {
    const size_t nwords = 1ull << 20;  // 8 MB: L2-resident
    double *buf;
    unsigned long long *out, *sink;
    cudaMalloc(&buf, nwords * 8);
    cudaMemset(buf, 0, nwords * 8);
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&sink, 8);
    unsigned long long h[4096];
    const char *kinds[4] = {"relaxed.gpu", "cg", "volatile", "weak"};
    for (int kind = 0; kind < 4; ++kind)
        for (int coal = 0; coal < 2; ++coal)
            for (int warps : {1, 8}) {
                const int blocks = 148, threads = warps * 32;
                for (int rep = 0; rep < 2; ++rep) {
#define L(C, K) poll<C, K><<<blocks, threads>>>(buf, nwords, 2000, out, sink)
                    if (coal) {
                        if (kind == 0) L(true, 0); else if (kind == 1) L(true, 1); else if (kind == 2) L(true, 2); else L(true, 3);
                    } else {
                        if (kind == 0) L(false, 0); else if (kind == 1) L(false, 1); else if (kind == 2) L(false, 2); else L(false, 3);
                    }
                }
                cudaDeviceSynchronize();
                const int nw = blocks * warps;
                cudaMemcpy(h, out, nw * 8, cudaMemcpyDeviceToHost);
                double s = 0;
                for (int i = 0; i < nw; ++i) s += h[i];
                printf("{\"kind\": \"%s\", \"coalesced\": %d, \"warps_per_sm\": %d, \"poll_ns\": %.1f}\n", kinds[kind], coal,
                       warps, s / nw);
            }
    // small working set: the polled lines stay L2-resident
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
