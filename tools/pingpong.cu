// Producer->consumer visibility latency between two SMs with relaxed
// gpu-scope stores/loads (the exact passes' synchronisation primitive).
// mode 0: hot  - every round trip reuses one 8-byte slot pair
// mode 1: cold - round trip i uses slots spread over a 1 GiB region that a
//          preceding fill kernel wrote (mostly evicted from L2)
// mode 2: cold + prefetch.global.L2 of the slot before polling it
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void str(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void fill(unsigned long long *x, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) x[i] = ~0ull;
}

__global__ void pingpong(unsigned long long *buf, int iters, int mode, size_t stride, unsigned long long *out) {
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x;  // 0 = ping, 1 = pong
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        size_t base = mode == 0 ? 0 : (size_t)i * stride;
        unsigned long long *ping = buf + base, *pong = buf + base + 1 + stride / 2;
        if (me == 0) {
            str(ping, (unsigned long long)i);
            if (mode == 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(pong));
            while (ldr(pong) != (unsigned long long)i) {}
        } else {
            if (mode == 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(ping));
            while (ldr(ping) != (unsigned long long)i) {}
            str(pong, (unsigned long long)i);
        }
    }
    if (me == 0) out[0] = clock64() - t0;
}

int main() {
    const size_t n = (1ull << 30) / 8;
    unsigned long long *buf, *out;
    cudaMalloc(&buf, n * 8);
    cudaMalloc(&out, 8);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 20000;
    for (int mode = 0; mode < 3; ++mode) {
        fill<<<1184, 256>>>(buf, n);
        cudaMemset(buf, 0xff, 64);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        // blocks 0 and 1 land on different SMs (one block per SM at this size)
        pingpong<<<2, 32>>>(buf, iters, mode, (n - 8) / iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc;
        cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
        printf("{\"mode\": %d, \"round_trip_ns\": %.1f, \"round_trip_cycles\": %.1f}\n", mode, ms * 1e6 / iters,
               (double)cyc / iters);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
