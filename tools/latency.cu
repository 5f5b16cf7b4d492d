// Dependent-chain latencies of the instructions on the exact passes' critical path.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b, int n) {
    double x = a, y = b;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
    t1 = clock64(); cyc[0] = t1 - t0;
    // DSETP + select chain (min)
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double c = __dadd_rn(y, (double)i); x = (c < x) ? c : x; }
    t1 = clock64(); cyc[1] = t1 - t0;
    // DDIV chain
    double z = x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) z = __ddiv_rn(z, 3.0 + (i & 1));
    t1 = clock64(); cyc[2] = t1 - t0;
    // shfl chain
    double s = z;
    t0 = clock64();
    for (int i = 0; i < n; ++i) s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 1) & 31) + 1.0;
    t1 = clock64(); cyc[3] = t1 - t0;
    // integer add chain (baseline)
    long long q = (long long)a;
    t0 = clock64();
    for (int i = 0; i < n; ++i) q = q * 3 + 1;
    t1 = clock64(); cyc[4] = t1 - t0;
    out[threadIdx.x] = x + z + s + (double)q;
}
int main() {
    double *o; long long *c, h[5];
    cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 5 * 8);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 32>>>(o, c, 1.0, 1e-9, n);
        cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    }
    const char *names[] = {"dadd", "dadd+dsetp+sel", "ddiv", "shfl+dadd", "imad64"};
    for (int i = 0; i < 5; ++i) printf("{\"op\": \"%s\", \"cycles_per_iter\": %.2f}\n", names[i], (double)h[i] / n);
    return 0;
}
