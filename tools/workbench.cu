// Post-wait work latency of one node-parallel forward task, in isolation
// (GPU tool): one warp runs the min-marginal trees, the copy averaging and
// the publish of mma_np_forward_kernel back to back, each iteration's inputs
// being the previous iteration's outputs, and reports cycles per iteration
// for the full chain and for pieces of it.
// nvcc -O3 -std=c++17 -fmad=false -gencode arch=compute_100a,code=sm_100a \
//      -I include -o tools/workbench tools/workbench.cu
#include "../paper_2310_08230_b200/csrc/dm_device.cu"

namespace {

// candidate: deltas gathered with shuffles, the warp-uniform copy count
// bounding the sequential sum (same sum order and identities as np_average)
__device__ __forceinline__ double np_average_shfl(bool act, int k, int c, int q, double m0, double m1, double lam_l) {
    const bool fin = act && m0 != DM_INF && m1 != DM_INF;
    const double dlt = fin ? __dsub_rn(m1, m0) : 0.0;
    const unsigned finmask = __ballot_sync(kFull, fin && q == 0);
    double dk[kNpCopies];
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j) dk[j] = __shfl_sync(kFull, dlt, 4 * j);
    double fsum = 0.0;
    if (k <= 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < k) fsum = __dadd_rn(fsum, dk[j]);
    } else {
#pragma unroll
        for (int j = 0; j < kNpCopies; ++j)
            if (j < k) fsum = __dadd_rn(fsum, dk[j]);
    }
    const int fcnt = __popc(finmask);
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

// 1/n correctly rounded for n = 1..8 (selects, no table)
__device__ __forceinline__ double inv_small(int n) {
    const double r3 = 0.3333333333333333, r5 = 0.2, r6 = 0.16666666666666666, r7 = 0.14285714285714285;
    return n == 3 ? r3 : n == 5 ? r5 : n == 6 ? r6 : n == 7 ? r7 : exact_inverse_pow2(n);
}

// a / n correctly rounded without a division: q = RN(a * RN(1/n)), exact
// residual, one correction (Markstein); power-of-two n are exact products
template <int kMode>
__device__ __forceinline__ double np_average_v(bool act, int k, int c, int q, double m0, double m1, double lam_l) {
    const bool fin = act && m0 != DM_INF && m1 != DM_INF;
    const double dlt = fin ? __dsub_rn(m1, m0) : 0.0;
    const unsigned finmask = __ballot_sync(kFull, fin && q == 0);
    double dk[kNpCopies];
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j) dk[j] = __shfl_sync(kFull, dlt, 4 * j);
    double fsum = 0.0;
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j)
        if (j < k) fsum = __dadd_rn(fsum, dk[j]);
    const int fcnt = max(__popc(finmask), 1);
    double avg;
    if (kMode == 0) {
        avg = fsum;
    } else if (kMode == 2) {
        avg = __dmul_rn(fsum, exact_inverse_pow2(fcnt));
    } else if (kMode == 3) {
        avg = __dmul_rn(fsum, inv_small(fcnt));
    } else {
        const double r = inv_small(fcnt);
        const double q0 = __dmul_rn(fsum, r);
        const double res = __fma_rn(-q0, (double)fcnt, fsum);
        avg = (fcnt & (fcnt - 1)) == 0 || res == 0.0 ? q0 : __fma_rn(res, r, q0);
    }
    return fin ? __dadd_rn(lam_l, __dsub_rn(avg, dlt)) : lam_l;
}

// sequential sum of the first k of dk (k warp-uniform: one uniform branch,
// exactly k dependent adds)
__device__ __forceinline__ double seq_sum(const double *dk, int k) {
    double s = 0.0;
    switch (k) {
        case 8: s = __dadd_rn(s, dk[0]); s = __dadd_rn(s, dk[1]); s = __dadd_rn(s, dk[2]); s = __dadd_rn(s, dk[3]);
                s = __dadd_rn(s, dk[4]); s = __dadd_rn(s, dk[5]); s = __dadd_rn(s, dk[6]); s = __dadd_rn(s, dk[7]); break;
        case 7: s = __dadd_rn(s, dk[0]); s = __dadd_rn(s, dk[1]); s = __dadd_rn(s, dk[2]); s = __dadd_rn(s, dk[3]);
                s = __dadd_rn(s, dk[4]); s = __dadd_rn(s, dk[5]); s = __dadd_rn(s, dk[6]); break;
        case 6: s = __dadd_rn(s, dk[0]); s = __dadd_rn(s, dk[1]); s = __dadd_rn(s, dk[2]); s = __dadd_rn(s, dk[3]);
                s = __dadd_rn(s, dk[4]); s = __dadd_rn(s, dk[5]); break;
        case 5: s = __dadd_rn(s, dk[0]); s = __dadd_rn(s, dk[1]); s = __dadd_rn(s, dk[2]); s = __dadd_rn(s, dk[3]);
                s = __dadd_rn(s, dk[4]); break;
        case 4: s = __dadd_rn(s, dk[0]); s = __dadd_rn(s, dk[1]); s = __dadd_rn(s, dk[2]); s = __dadd_rn(s, dk[3]); break;
        case 3: s = __dadd_rn(s, dk[0]); s = __dadd_rn(s, dk[1]); s = __dadd_rn(s, dk[2]); break;
        case 2: s = __dadd_rn(s, dk[0]); s = __dadd_rn(s, dk[1]); break;
        case 1: s = __dadd_rn(s, dk[0]); break;
        default: break;
    }
    return s;
}

__device__ __forceinline__ double np_average_u(bool act, int k, int c, int q, double m0, double m1, double lam_l) {
    const bool fin = act && m0 != DM_INF && m1 != DM_INF;
    const double dlt = fin ? __dsub_rn(m1, m0) : 0.0;
    const unsigned finmask = __ballot_sync(kFull, fin && q == 0);
    double dk[kNpCopies];
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j) dk[j] = __shfl_sync(kFull, dlt, 4 * j);
    const double fsum = seq_sum(dk, k);
    const int fcnt = __popc(finmask);  // warp-uniform
    double avg;
    if ((fcnt & (fcnt - 1)) == 0)
        avg = __dmul_rn(fsum, exact_inverse_pow2(max(fcnt, 1)));
    else
        avg = __ddiv_rn(fsum, (double)fcnt);
    return fin ? __dadd_rn(lam_l, __dsub_rn(avg, dlt)) : lam_l;
}

template <int kSum>
__device__ __forceinline__ double np_average_z(bool act, int k, int c, int q, double m0, double m1, double lam_l,
                                               const NpDiv &dv) {
    const bool fin = act && m0 != DM_INF && m1 != DM_INF;
    const double dlt = fin ? __dsub_rn(m1, m0) : 0.0;
    const unsigned finmask = __ballot_sync(kFull, fin && q == 0);
    double dk[kNpCopies];
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j) dk[j] = __shfl_sync(kFull, dlt, 4 * j);
    // copies j >= k hold +0.0 (inactive lanes): adding them is bit-neutral
    double fsum = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) fsum = __dadd_rn(fsum, dk[j]);
    if (kSum == 0 || k > 4) {
#pragma unroll
        for (int j = 4; j < kNpCopies; ++j) fsum = __dadd_rn(fsum, dk[j]);
    }
    const int fcnt = __popc(finmask);
    double avg = 0.0;
    if (fcnt == k)
        avg = div_by_count(fsum, dv);
    else if (fcnt > 0)
        avg = (fcnt & (fcnt - 1)) == 0 ? __dmul_rn(fsum, exact_inverse_pow2(fcnt)) : __ddiv_rn(fsum, (double)fcnt);
    return fin ? __dadd_rn(lam_l, __dsub_rn(avg, dlt)) : lam_l;
}

template <bool kSeq>
__device__ __forceinline__ double np_average_s(bool act, int k, int c, int q, double m0, double m1, double lam_l,
                                               const NpDiv &dv) {
    const bool fin = act && m0 != DM_INF && m1 != DM_INF;
    const double dlt = fin ? __dsub_rn(m1, m0) : 0.0;
    const unsigned finmask = __ballot_sync(kFull, fin && q == 0);
    double dk[kNpCopies];
#pragma unroll
    for (int j = 0; j < kNpCopies; ++j) dk[j] = __shfl_sync(kFull, dlt, 4 * j);
    double fsum = 0.0;
    if (kSeq) {
        fsum = seq_sum(dk, k);
    } else {
#pragma unroll
        for (int j = 0; j < kNpCopies; ++j)
            if (j < k) fsum = __dadd_rn(fsum, dk[j]);
    }
    const int fcnt = __popc(finmask);
    double avg = 0.0;
    if (fcnt == k)
        avg = div_by_count(fsum, dv);
    else if (fcnt > 0)
        avg = (fcnt & (fcnt - 1)) == 0 ? __dmul_rn(fsum, exact_inverse_pow2(fcnt)) : __ddiv_rn(fsum, (double)fcnt);
    return fin ? __dadd_rn(lam_l, __dsub_rn(avg, dlt)) : lam_l;
}

template <int kVariant>
__global__ void work_kernel(int iters, int k, uint64_t desc, double seed, double *out, long long *cycles) {
    __shared__ NpShared sh;
    const int lane = threadIdx.x & 31, c = lane >> 2, q = lane & 3;
    const int i0 = 2 * q, i1 = i0 + 1;
    const bool act = c < k;
    double *nodes = sh.node[0][c];
    const NpDiv dv = np_div(k);
    double f0 = seed + lane, f1 = seed - lane, lam = 0.25 * lane;
    const double t00 = 0.5, t01 = -0.0, t10 = 1.5, t11 = 2.0;
    nodes[8] = DM_INF;
    __syncwarp();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        nodes[i0] = f0;
        nodes[i1] = f1;
        const double m0 = np_lmin4(lmin(__dadd_rn(f0, t00), __dadd_rn(f1, t01)), q);
        const double m1 = np_lmin4(lmin(__dadd_rn(__dadd_rn(f0, lam), t10), __dadd_rn(__dadd_rn(f1, lam), t11)), q);
        double lam_l = lam;
        if (kVariant == 1) {  // trees only
            lam_l = __dadd_rn(lam, __dsub_rn(m1, m0));
            __syncwarp();
        } else if (kVariant == 4) {
            lam_l = np_average_v<1>(act, k, c, q, m0, m1, lam);
        } else if (kVariant == 5) {
            lam_l = np_average_v<0>(act, k, c, q, m0, m1, lam);
        } else if (kVariant == 7) {
            lam_l = np_average_v<2>(act, k, c, q, m0, m1, lam);
        } else if (kVariant == 8) {
            lam_l = np_average_v<3>(act, k, c, q, m0, m1, lam);
        } else if (kVariant == 9) {
            __syncwarp();
            lam_l = np_average_s<false>(act, k, c, q, m0, m1, lam, dv);
        } else if (kVariant == 10) {
            __syncwarp();
            lam_l = np_average_s<true>(act, k, c, q, m0, m1, lam, dv);
        } else if (kVariant == 11) {
            __syncwarp();
            lam_l = np_average_z<0>(act, k, c, q, m0, m1, lam, dv);
        } else if (kVariant == 12) {
            __syncwarp();
            lam_l = np_average_z<1>(act, k, c, q, m0, m1, lam, dv);
        } else if (kVariant == 6) {
            lam_l = np_average_u(act, k, c, q, m0, m1, lam);
        } else if (kVariant == 3) {
            lam_l = np_average_shfl(act, k, c, q, m0, m1, lam);
        } else {
            __syncwarp();
            lam_l = np_average(act, k, q, m0, m1, lam, dv);
        }
        double o[2];
        if (kVariant == 2) {  // no publish: feed the dual back directly
            o[0] = __dadd_rn(f0, lam_l);
            o[1] = __dadd_rn(f1, lam_l);
        } else {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int u = i0 + j;
                const int zi = (int)(desc >> (8 * u)) & 15, oi = (int)(desc >> (8 * u + 4)) & 15;
                const double A = nodes[zi < 8 ? zi : 8];
                const double C = __dadd_rn(nodes[oi < 8 ? oi : 8], lam_l);
                o[j] = (C < A || (C == A && oi < zi)) ? C : A;
            }
        }
        f0 = o[0] * 0.5;  // keep values bounded; the next iteration depends on this one
        f1 = o[1] * 0.5;
        lam = lam_l * 0.5;
        __syncwarp();
    }
    long long t1 = clock64();
    out[lane] = f0 + f1 + lam;
    if (lane == 0) *cycles = t1 - t0;
}

// backward task chain: next-layer distances routed to the lane's arcs
// through shared memory (kShfl = 0, as mma_np_backward_kernel) or shuffles
template <int kShfl>
__global__ void work_bw_kernel(int iters, int k, double seed, double *out, long long *cycles) {
    __shared__ NpShared sh;
    const int lane = threadIdx.x & 31, c = lane >> 2, q = lane & 3;
    const int i0 = 2 * q, i1 = i0 + 1;
    const bool act = c < k;
    double *nodes = sh.node[0][c];
    const NpDiv dv = np_div(k);
    int iz[2] = {(i0 + 1) & 7, (i0 + 3) & 7}, io[2] = {(i0 + 2) & 7, (i0 + 5) & 7};
    double f0b[2] = {0.5 * lane, 0.25 * lane}, f1b[2] = {1.5, 2.5}, rz[2] = {-0.0, -0.0}, ro[2] = {-0.0, -0.0};
    double nb0 = seed + lane, nb1 = seed - lane, lam = 0.25 * lane;
    nodes[8] = -0.0;
    __syncwarp();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double tz[2], to[2];
        if (kShfl) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int sz = 4 * c + (iz[j] >> 1), so = 4 * c + (io[j] >> 1);
                const double za = __shfl_sync(kFull, nb0, sz), zb = __shfl_sync(kFull, nb1, sz);
                const double oa = __shfl_sync(kFull, nb0, so), ob = __shfl_sync(kFull, nb1, so);
                tz[j] = (iz[j] & 1) ? zb : za;
                to[j] = (io[j] & 1) ? ob : oa;
            }
        } else {
            nodes[i0] = nb0;
            nodes[i1] = nb1;
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                tz[j] = nodes[iz[j]];
                to[j] = nodes[io[j]];
            }
        }
        const double m0 = np_lmin4(lmin(__dadd_rn(f0b[0], tz[0]), __dadd_rn(f0b[1], tz[1])), q);
        const double m1 = np_lmin4(lmin(__dadd_rn(f1b[0], to[0]), __dadd_rn(f1b[1], to[1])), q);
        const double lam_l = np_average(act, k, q, m0, m1, lam, dv);
        double bv[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const double cz = __dadd_rn(rz[j], tz[j]);
            const double co = __dadd_rn(__dadd_rn(lam_l, to[j]), ro[j]);
            bv[j] = cz <= co ? cz : co;
        }
        nb0 = bv[0] * 0.5;
        nb1 = bv[1] * 0.5;
        lam = lam_l * 0.5;
        __syncwarp();
    }
    long long t1 = clock64();
    out[lane] = nb0 + nb1 + lam;
    if (lane == 0) *cycles = t1 - t0;
}

}  // namespace

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    // each target u <- zero source u, one source (u+1)%8 (a valid one-source-per-kind publish)
    uint64_t desc = 0;
    for (int u = 0; u < 8; ++u) desc |= (uint64_t)(u | (((u + 1) % 8) << 4)) << (8 * u);
    const int iters = 20000;
    for (int k : {2, 4, 5}) {
        long long h[13];
        work_kernel<0><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[0], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<1><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[1], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<2><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[2], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<3><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[3], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<4><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[4], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<5><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[5], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<6><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[6], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<7><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[7], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<8><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[8], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<9><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[9], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<10><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[10], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<11><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[11], cyc, 8, cudaMemcpyDeviceToHost);
        work_kernel<12><<<1, 32>>>(iters, k, desc, 1.0, out, cyc);
        cudaMemcpy(&h[12], cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("{\"copies\": %d, \"full_cycles\": %.1f, \"trees_publish_cycles\": %.1f, "
                    "\"trees_average_cycles\": %.1f, \"full_shfl_average_cycles\": %.1f, "
                    "\"full_markstein_cycles\": %.1f, \"full_no_division_cycles\": %.1f, \"full_uniform_cycles\": %.1f, \"pow2_mul_only\": %.1f, \"table_mul_only\": %.1f, \"new_shfl\": %.1f, \"new_shfl_seq\": %.1f, \"zero_pad8\": %.1f, \"zero_pad_4_4\": %.1f}\n",
                    k, (double)h[0] / iters, (double)h[1] / iters, (double)h[2] / iters, (double)h[3] / iters,
                    (double)h[4] / iters, (double)h[5] / iters, (double)h[6] / iters, (double)h[7] / iters, (double)h[8] / iters, (double)h[9] / iters, (double)h[10] / iters, (double)h[11] / iters, (double)h[12] / iters);
    }
    for (int k : {4, 5}) {
        long long h[2];
        work_bw_kernel<0><<<1, 32>>>(iters, k, 1.0, out, cyc);
        cudaMemcpy(&h[0], cyc, 8, cudaMemcpyDeviceToHost);
        work_bw_kernel<1><<<1, 32>>>(iters, k, 1.0, out, cyc);
        cudaMemcpy(&h[1], cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("{\"backward\": true, \"copies\": %d, \"smem_route_cycles\": %.1f, \"shfl_route_cycles\": %.1f}\n",
                    k, (double)h[0] / iters, (double)h[1] / iters);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e) std::printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
