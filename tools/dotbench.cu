// Access-pattern experiments for the chunked dot (GPU tool, standalone).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dotbench tools/dotbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChunk = 4096;

__device__ __forceinline__ int pair_index(int i) { return (threadIdx.x >> 2) * 64 + (threadIdx.x & 3) + 4 * i; }

// V1: paired leaf layout, 128 threads per chunk, write chunk partial only
template <int kThreads>
__global__ void __launch_bounds__(kThreads) v_pair(const double *a, const double *b, double *partial) {
    const double2 *a2 = reinterpret_cast<const double2 *>(a + (size_t)blockIdx.x * kChunk);
    const double2 *b2 = reinterpret_cast<const double2 *>(b + (size_t)blockIdx.x * kChunk);
    double r0 = 0, r1 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const double2 x = a2[pair_index(i)], y = b2[pair_index(i)];
        r0 = __dadd_rn(r0, __dmul_rn(x.x, y.x));
        r1 = __dadd_rn(r1, __dmul_rn(x.y, y.y));
    }
    double r = __dadd_rn(r0, r1);
    r = __dadd_rn(r, __shfl_xor_sync(~0u, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(~0u, r, 2));
    __shared__ double leaf[32];
    if ((threadIdx.x & 3) == 0) leaf[threadIdx.x >> 2] = r;
    __syncthreads();
    if (threadIdx.x < 32) {
        double x = leaf[threadIdx.x];
        for (int w = 1; w < 32; w <<= 1) x = __dadd_rn(x, __shfl_xor_sync(~0u, x, w));
        if (threadIdx.x == 0) partial[blockIdx.x] = x;
    }
}

// V2: coalesced contiguous double2 per thread (no numpy order), 128 threads per chunk
__global__ void __launch_bounds__(128) v_coal(const double *a, const double *b, double *partial) {
    const double2 *a2 = reinterpret_cast<const double2 *>(a + (size_t)blockIdx.x * kChunk);
    const double2 *b2 = reinterpret_cast<const double2 *>(b + (size_t)blockIdx.x * kChunk);
    double r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const double2 x = a2[threadIdx.x + 128 * i], y = b2[threadIdx.x + 128 * i];
        r += x.x * y.x + x.y * y.y;
    }
    for (int w = 1; w < 32; w <<= 1) r += __shfl_xor_sync(~0u, r, w);
    __shared__ double s[4];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = r;
    __syncthreads();
    if (threadIdx.x == 0) partial[blockIdx.x] = s[0] + s[1] + s[2] + s[3];
}

// V3: grid-stride, persistent, coalesced double2 (bandwidth reference)
__global__ void __launch_bounds__(256) v_stride(const double *a, const double *b, size_t n2, double *partial) {
    const double2 *a2 = reinterpret_cast<const double2 *>(a);
    const double2 *b2 = reinterpret_cast<const double2 *>(b);
    double r = 0;
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n2; i += (size_t)gridDim.x * 256) {
        const double2 x = a2[i], y = b2[i];
        r += x.x * y.x + x.y * y.y;
    }
    for (int w = 1; w < 32; w <<= 1) r += __shfl_xor_sync(~0u, r, w);
    if ((threadIdx.x & 31) == 0) partial[blockIdx.x * 8 + (threadIdx.x >> 5)] = r;
}

// V4: TMA-less smem staging: coalesced loads into smem, then leaf sums from smem
__global__ void __launch_bounds__(256) v_smem(const double *a, const double *b, double *partial) {
    __shared__ double2 sp[kChunk / 2];
    const double2 *a2 = reinterpret_cast<const double2 *>(a + (size_t)blockIdx.x * kChunk);
    const double2 *b2 = reinterpret_cast<const double2 *>(b + (size_t)blockIdx.x * kChunk);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const double2 x = a2[threadIdx.x + 256 * i], y = b2[threadIdx.x + 256 * i];
        sp[threadIdx.x + 256 * i] = make_double2(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y));
    }
    __syncthreads();
    const double *p = reinterpret_cast<const double *>(sp);
    const int o = threadIdx.x >> 3, q = threadIdx.x & 7;
    double r = p[o * 128 + q];
    for (int i = 1; i < 16; ++i) r = __dadd_rn(r, p[o * 128 + q + 8 * i]);
    for (int w = 1; w < 8; w <<= 1) r = __dadd_rn(r, __shfl_xor_sync(~0u, r, w));
    __shared__ double leaf[32];
    if (q == 0) leaf[o] = r;
    __syncthreads();
    if (threadIdx.x < 32) {
        double x = leaf[threadIdx.x];
        for (int w = 1; w < 32; w <<= 1) x = __dadd_rn(x, __shfl_xor_sync(~0u, x, w));
        if (threadIdx.x == 0) partial[blockIdx.x] = x;
    }
}

// numpy's recursion over leaf sums (left to right), depth <= 6 for 4096 elements
__device__ double combine_leaves(const double *leaf_val, int len, int &k) {
    if (len <= 128) return leaf_val[k++];
    int n2 = len / 2;
    n2 -= n2 % 8;
    const double l = combine_leaves(leaf_val, n2, k);
    const double r = combine_leaves(leaf_val, len - n2, k);
    return __dadd_rn(l, r);
}

// numpy pairwise_sum of x[0:n] (n <= kChunk) by one block (any multiple of
// 32 threads); leaves (<= 32) are found by replaying the recursion on one
// thread, octets sum them.  kDot: terms a[i]*b[i]; b may have been written by
// this block before a __syncthreads, so it is read through L2 (ld.global.cg).
template <bool kDot>
__device__ double block_pairwise(const double *__restrict__ a, const double *b, int n) {
    __shared__ int leaf_off[32], leaf_len[32], nleaves;
    __shared__ double leaf_val[32];
    if (threadIdx.x == 0) {
        int stack_off[16], stack_len[16], sp = 0, k = 0;
        stack_off[sp] = 0;
        stack_len[sp++] = n;
        while (sp) {  // pre-order, left first: leaves come out left to right
            const int off = stack_off[--sp], len = stack_len[sp];
            if (len <= 128) {
                leaf_off[k] = off;
                leaf_len[k++] = len;
                continue;
            }
            int n2 = len / 2;
            n2 -= n2 % 8;
            stack_off[sp] = off + n2;
            stack_len[sp++] = len - n2;  // right pushed first, popped second
            stack_off[sp] = off;
            stack_len[sp++] = n2;
        }
        nleaves = k;
    }
    __syncthreads();
    const int q = threadIdx.x & 7;
    auto term = [&](int i) { return kDot ? __dmul_rn(a[i], __ldcg(b + i)) : __ldcg(a + i); };
    for (int base = 0; base < nleaves; base += blockDim.x >> 3) {
        const int oct = base + (threadIdx.x >> 3);
        const bool live = oct < nleaves;
        const int off = live ? leaf_off[oct] : 0, len = live ? leaf_len[oct] : 0;
        const int stop = len - (len % 8);
        double r = 0.0;
        if (len >= 8) {
            r = term(off + q);
            for (int i = 8; i < stop; i += 8) r = __dadd_rn(r, term(off + i + q));
        }
        const unsigned m = 0xffffffffu;
#pragma unroll
        for (int w = 1; w < 8; w <<= 1) r = __dadd_rn(r, __shfl_xor_sync(m, r, w));  // a+b == b+a exactly
        if (live && q == 0) {
            double res = len < 8 ? 0.0 : r;
            for (int i = len < 8 ? 0 : stop; i < len; ++i) res = __dadd_rn(res, term(off + i));
            leaf_val[oct] = res;
        }
    }
    __syncthreads();
    double total = 0.0;
    if (threadIdx.x == 0) {
        int k = 0;
        total = __dadd_rn(0.0, combine_leaves(leaf_val, n, k));
    }
    return total;  // valid on thread 0
}

// chunk total -> partial[c]; the last block reduces the partials into *out.
// The counter increment is a release atomic (orders this block's partial
// before it) and only the last block pays an acquire fence — a
// __threadfence per block compiles to an SC fence plus an L1 invalidation,
// which costs more than the chunk's loads.  The barrier carries the acquire
// to the reading threads, which read through L2.
__device__ __forceinline__ unsigned atomic_add_release(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void finish_chunk(double v, int64_t nch, double *partial, unsigned *counter, double *out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = v;
        last = atomic_add_release(counter, 1u) == (unsigned)(nch - 1);
        if (last) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    if (!last) return;
    const double t = block_pairwise<false>(partial, nullptr, (int)nch);
    if (threadIdx.x == 0) {
        out[0] = t;
        *counter = 0;  // ready for the next call
    }
}


// V5: pair128 + finish (partial, release atomic, last block reduces)
__global__ void __launch_bounds__(128) v_pair_finish(const double *a, const double *b, double *partial, unsigned *counter, double *out, int nch, int mode) {
    const double2 *a2 = reinterpret_cast<const double2 *>(a + (size_t)blockIdx.x * kChunk);
    const double2 *b2 = reinterpret_cast<const double2 *>(b + (size_t)blockIdx.x * kChunk);
    double r0 = 0, r1 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const double2 x = a2[pair_index(i)], y = b2[pair_index(i)];
        r0 = __dadd_rn(r0, __dmul_rn(x.x, y.x));
        r1 = __dadd_rn(r1, __dmul_rn(x.y, y.y));
    }
    double r = __dadd_rn(r0, r1);
    r = __dadd_rn(r, __shfl_xor_sync(~0u, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(~0u, r, 2));
    __shared__ double leaf[32];
    if ((threadIdx.x & 3) == 0) leaf[threadIdx.x >> 2] = r;
    __syncthreads();
    double v = 0;
    if (threadIdx.x < 32) {
        double x = leaf[threadIdx.x];
        for (int w = 1; w < 32; w <<= 1) x = __dadd_rn(x, __shfl_xor_sync(~0u, x, w));
        v = x;
    }
    if (mode == 0) { if (threadIdx.x == 0) partial[blockIdx.x] = v; return; }
    if (mode == 1) {  // atomic only
        if (threadIdx.x == 0) { partial[blockIdx.x] = v; atomic_add_release(counter, 1u); }
        return;
    }
    finish_chunk(v, nch, partial, counter, out);
}

int main() {
    const size_t n = 9402880, nch = n / kChunk;
    double *a, *b, *partial;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMalloc(&partial, 1 << 20);
    cudaMemset(a, 0, n * 8);
    cudaMemset(b, 0, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / 20;
        printf("%-10s %8.1f us  %7.0f GB/s  (%s)\n", name, us, 16.0 * n / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    unsigned *counter;
    double *out;
    cudaMalloc(&counter, 4);
    cudaMemset(counter, 0, 4);
    cudaMalloc(&out, 8);
    run("pair128", [&] { v_pair<128><<<nch, 128>>>(a, b, partial); });
    run("pf_mode0", [&] { v_pair_finish<<<nch, 128>>>(a, b, partial, counter, out, nch, 0); });
    run("pf_atomic", [&] { v_pair_finish<<<nch, 128>>>(a, b, partial, counter, out, nch, 1); });
    cudaMemset(counter, 0, 4);
    run("pf_finish", [&] { v_pair_finish<<<nch, 128>>>(a, b, partial, counter, out, nch, 2); });
    run("coal128", [&] { v_coal<<<nch, 128>>>(a, b, partial); });
    run("stride", [&] { v_stride<<<148 * 8, 256>>>(a, b, n / 2, partial); });
    run("stride4", [&] { v_stride<<<148 * 4, 256>>>(a, b, n / 2, partial); });
    run("smem256", [&] { v_smem<<<nch, 256>>>(a, b, partial); });
    return 0;
}
