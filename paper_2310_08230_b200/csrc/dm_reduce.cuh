// numpy-order pairwise sums of up to 4096 shared-memory values (the chunked
// inner products of the L-BFGS path, dm_sweep.cu, and the per-instance sums
// of batched solves, dm_batch.cu).  Textually included inside each user's
// anonymous namespace (TU-local definitions); needs <vector>, <cstdint> and
// the CUDA runtime headers before it.
// numpy's pairwise recursion for one length n <= kChunk, planned on the host:
// the leaves (<= 32 runs of <= 128 elements, left to right) are nodes
// 0..nleaves-1; the additions are nodes nleaves.. in post-order (the root
// last), each with its two children and its height above the leaves.
// Up to 33 leaves for n <= 4096 (e.g. 217 lengths in [3849, 4095]).
constexpr int kMaxLeaves = 33;
struct SumPlan {
    int32_t nleaves, nint, height;
    uint16_t off[kMaxLeaves];
    uint8_t len[kMaxLeaves];
    uint8_t left[kMaxLeaves - 1], right[kMaxLeaves - 1], h[kMaxLeaves - 1];
};

int plan_rec(SumPlan &p, int off, int len, int &height, std::vector<int> &post) {
    if (len <= 128) {
        p.off[p.nleaves] = (uint16_t)off;
        p.len[p.nleaves] = (uint8_t)len;
        height = 0;
        return p.nleaves++;
    }
    int n2 = len / 2;
    n2 -= n2 % 8;
    int hl, hr;
    const int l = plan_rec(p, off, n2, hl, post);
    const int r = plan_rec(p, off + n2, len - n2, hr, post);
    height = 1 + (hl > hr ? hl : hr);
    post.push_back(l);
    post.push_back(r);
    post.push_back(height);
    return -(int)(post.size() / 3);  // internal node k (1-based) as -k
}

SumPlan make_sum_plan(int n) {
    SumPlan p{};
    if (n <= 0) return p;
    std::vector<int> post;
    int height;
    plan_rec(p, 0, n, height, post);
    p.nint = (int)post.size() / 3;
    p.height = height;
    auto id = [&](int v) { return v >= 0 ? v : p.nleaves + (-v - 1); };
    for (int k = 0; k < p.nint; ++k) {
        p.left[k] = (uint8_t)id(post[3 * k]);
        p.right[k] = (uint8_t)id(post[3 * k + 1]);
        p.h[k] = (uint8_t)post[3 * k + 2];
    }
    return p;
}

// 0.0 + numpy pairwise_sum(sm[0:n]) of shared-memory values, by a block of
// any multiple of 32 threads: one octet per leaf (numpy's 8 accumulators),
// then warp 0 adds the tree level by level.  Result on thread 0.
__device__ double smem_pairwise(const double *sm, const SumPlan &p) {
    __shared__ double node[2 * kMaxLeaves];
    const int q = threadIdx.x & 7;
    // octets in passes of blockDim/8 (uniform trip count: whole warps shuffle)
    for (int base = 0; base < p.nleaves; base += (int)(blockDim.x >> 3)) {
        const int oct = base + (int)(threadIdx.x >> 3);
        const bool live = oct < p.nleaves;
        const int off = live ? p.off[oct] : 0, len = live ? p.len[oct] : 0;
        const int stop = len - (len % 8);
        double r = 0.0;
        if (len >= 8) {
            r = sm[off + q];
            for (int i = 8; i < stop; i += 8) r = __dadd_rn(r, sm[off + i + q]);
        }
#pragma unroll
        for (int w = 1; w < 8; w <<= 1) r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, w));  // a+b == b+a exactly
        if (live && q == 0) {
            double res = len < 8 ? 0.0 : r;
            for (int i = len < 8 ? 0 : stop; i < len; ++i) res = __dadd_rn(res, sm[off + i]);
            node[oct] = res;
        }
    }
    __syncthreads();
    double total = 0.0;
    if (threadIdx.x < 32 && p.nleaves > 0) {
        const int k = threadIdx.x;  // internal nodes: at most 32, one per lane
        for (int h = 1; h <= p.height; ++h) {
            if (k < p.nint && p.h[k] == h) node[p.nleaves + k] = __dadd_rn(node[p.left[k]], node[p.right[k]]);
            __syncwarp();
        }
        total = __dadd_rn(0.0, node[p.nleaves + p.nint - 1]);
    }
    return total;
}

