// A lane's distance row of one position in the interleaved sweep layout:
// W doubles kept in registers (narrow bodies: every access of a dynamic node
// index is an unrolled select, no shared-memory round trip on the per-layer
// dependency chain) or in shared memory with a stride of STRIDE threads.
#pragma once

template <int W, bool kReg, int STRIDE>
struct Row;

template <int W, int STRIDE>
struct Row<W, true, STRIDE> {
    double v[W];
    __device__ __forceinline__ double get(int32_t i) const {  // i in [0, W)
        double x = v[0];
#pragma unroll
        for (int u = 1; u < W; ++u) x = (i == u) ? v[u] : x;
        return x;
    }
    __device__ __forceinline__ double at(int u) const { return v[u]; }  // u: unrolled-loop constant
    __device__ __forceinline__ void put(int u, double x) { v[u] = x; }
    __device__ __forceinline__ void put_dyn(int32_t i, double x) {
#pragma unroll
        for (int u = 0; u < W; ++u)
            if (i == u) v[u] = x;
    }
};

template <int W, int STRIDE>
struct Row<W, false, STRIDE> {
    double *p;
    __device__ __forceinline__ double get(int32_t i) const { return p[i * STRIDE]; }
    __device__ __forceinline__ double at(int u) const { return p[u * STRIDE]; }
    __device__ __forceinline__ void put(int u, double x) { p[u * STRIDE] = x; }
    __device__ __forceinline__ void put_dyn(int32_t i, double x) { p[i * STRIDE] = x; }
};

template <int W, bool kReg, int STRIDE>
__device__ __forceinline__ void swap_rows(Row<W, kReg, STRIDE> &a, Row<W, kReg, STRIDE> &b) {
    const Row<W, kReg, STRIDE> t = a;
    a = b;
    b = t;
}

// rows in registers up to this width: the full-table sweeps (C4 node-order
// refresh 130 -> 112 us); the deferred MM passes keep shared-memory rows
// (register rows there: C4 flat, C2 forward 295 -> 400 us)
constexpr int kRegRowsSweep = 4;
constexpr int kRegRowsDfr = 0;
