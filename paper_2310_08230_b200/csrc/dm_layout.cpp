// Interleaved "sweep layout" of the diagram table for the full-table sweeps
// (k_backward, the step-search trials, k_forward).
//
// The reference layout (FlatBdds) stores each diagram contiguously, which
// makes a thread-per-diagram sweep read 32 unrelated cache lines per warp
// instruction.  Here diagrams of similar shape are grouped 32 to a warp
// (sorted by layer count, then node count), their layers are aligned at the
// LAST layer (position k = 0 is every lane's last layer), and the node slots
// of one position are interleaved by lane: slot (k, i) of lane t lives at
// element (pos_slot[k] + i) * 32 + t.  A warp instruction then reads 128
// contiguous bytes.  Arc targets are stored as LOCAL indices into the next
// layer (position k - 1), so a sweep keeps the neighbouring layer's
// distances in shared memory instead of re-reading them from L2.
// Padded slots (lanes whose diagram is shorter / narrower) have both arcs
// to FALSE and never feed a real node.
#include <algorithm>
#include <numeric>
#include <thread>
#include <vector>

#include "dm_internal.h"

namespace dm {

int build_sweep_layout(const int64_t *bdd_layer_lo, int64_t nb, const int64_t *lnl, const int64_t *zero_t,
                       const int64_t *one_t, SweepLayout &s) {
    auto nlay = [&](int64_t j) { return bdd_layer_lo[j + 1] - bdd_layer_lo[j]; };
    constexpr int kThreads = 8;
    auto par = [&](int64_t n, auto &&fn) {  // fn(lo, hi) over kThreads contiguous ranges
        std::vector<std::thread> th;
        for (int t = 0; t < kThreads; ++t)
            th.emplace_back([&, t] { fn(n * t / kThreads, n * (t + 1) / kThreads); });
        for (auto &x : th) x.join();
    };
    // shape order: more layers first, then more nodes, then diagram id
    std::vector<std::pair<uint64_t, int64_t>> key(nb);
    par(nb, [&](int64_t lo, int64_t hi) {
        for (int64_t j = lo; j < hi; ++j) {
            const uint64_t L = (uint64_t)nlay(j), Nn = (uint64_t)(lnl[bdd_layer_lo[j + 1]] - lnl[bdd_layer_lo[j]]);
            key[j] = {(~L << 32) | (~Nn & 0xffffffffull), j};
        }
    });
    std::sort(key.begin(), key.end());
    s.groups = (nb + 31) / 32;
    s.grp_bdd.assign(s.groups * 32, -1);
    s.grp_npos.assign(s.groups, 0);
    s.grp_pos_lo.assign(s.groups + 1, 0);
    for (int64_t g = 0; g < s.groups; ++g) {
        int64_t K = 0;
        for (int t = 0; t < 32 && g * 32 + t < nb; ++t) {
            const int64_t j = key[g * 32 + t].second;
            s.grp_bdd[g * 32 + t] = (int32_t)j;
            K = std::max(K, nlay(j));
        }
        s.grp_npos[g] = (int32_t)K;
        s.grp_pos_lo[g + 1] = s.grp_pos_lo[g] + K;
    }
    const int64_t npos_total = s.grp_pos_lo[s.groups];
    s.pos_width.assign(npos_total, 0);
    par(s.groups, [&](int64_t glo, int64_t ghi) {
        for (int64_t g = glo; g < ghi; ++g)
            for (int t = 0; t < 32; ++t) {
                const int32_t j = s.grp_bdd[g * 32 + t];
                if (j < 0) continue;
                for (int64_t k = 0; k < nlay(j); ++k) {
                    const int64_t l = bdd_layer_lo[j + 1] - 1 - k;
                    int32_t &w = s.pos_width[s.grp_pos_lo[g] + k];
                    w = std::max<int32_t>(w, (int32_t)(lnl[l + 1] - lnl[l]));
                }
            }
    });
    s.pos_slot.assign(npos_total, 0);
    s.max_width = 0;
    int64_t slots = 0;
    for (int64_t q = 0; q < npos_total; ++q) {
        s.pos_slot[q] = slots;
        slots += s.pos_width[q];
        s.max_width = std::max<int64_t>(s.max_width, s.pos_width[q]);
    }
    if (slots * 32 >= INT32_MAX) {
        set_error("sweep layout exceeds the int32 element range");
        return DM_ERR_UNSUPPORTED;
    }
    s.slots = slots;
    s.zl.resize(slots * 32);
    s.ol.resize(slots * 32);
    // groups own disjoint slot ranges: fill them in parallel
    std::vector<std::thread> th;
    for (int th_i = 0; th_i < kThreads; ++th_i)
        th.emplace_back([&, th_i] {
    const int64_t glo = s.groups * th_i / kThreads, ghi = s.groups * (th_i + 1) / kThreads;
    if (glo < ghi) {
        const int64_t slo = s.pos_slot[s.grp_pos_lo[glo]] * 32;
        const int64_t shi = (ghi == s.groups ? slots : s.pos_slot[s.grp_pos_lo[ghi]]) * 32;
        std::fill(s.zl.data() + slo, s.zl.data() + shi, kFalse);
        std::fill(s.ol.data() + slo, s.ol.data() + shi, kFalse);
    }
    for (int64_t g = glo; g < ghi; ++g) {
        const int64_t p0 = s.grp_pos_lo[g];
        for (int t = 0; t < 32; ++t) {
            const int32_t j = s.grp_bdd[g * 32 + t];
            if (j < 0) continue;
            for (int64_t k = 0; k < nlay(j); ++k) {
                const int64_t l = bdd_layer_lo[j + 1] - 1 - k;
                const int64_t next0 = lnl[l + 1];
                for (int64_t v = lnl[l]; v < lnl[l + 1]; ++v) {
                    const int64_t at = (s.pos_slot[p0 + k] + (v - lnl[l])) * 32 + t;
                    const int64_t a = zero_t[v], b = one_t[v];
                    s.zl[at] = (int32_t)(a >= 0 ? a - next0 : a);
                    s.ol[at] = (int32_t)(b >= 0 ? b - next0 : b);
                }
            }
        }
    }
        });
    for (auto &t : th) t.join();
    return DM_OK;
}

}  // namespace dm

// Host-only timing of the plans dm_flat_create builds (test/profiling hook).
#include <chrono>
extern "C" int dm_debug_time_plans(const dm_flat_desc *d, double *seconds3) {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    dm::MmaSchedule fw, bw;
    int rc = dm::build_mma_schedule(d->bdd_layer_lo, d->num_bdds, nullptr, d->layer_var, d->num_layers, d->proc_ptr,
                                    d->proc_layers, d->num_positions, true, fw);
    if (rc) return rc;
    auto t1 = clk::now();
    rc = dm::build_mma_schedule(d->bdd_layer_lo, d->num_bdds, nullptr, d->layer_var, d->num_layers, d->proc_ptr,
                                d->proc_layers, d->num_positions, false, bw);
    if (rc) return rc;
    auto t2 = clk::now();
    dm::SweepLayout sl;
    rc = dm::build_sweep_layout(d->bdd_layer_lo, d->num_bdds, d->layer_node_lo, d->zero_t, d->one_t, sl);
    if (rc) return rc;
    auto t3 = clk::now();
    seconds3[0] = std::chrono::duration<double>(t1 - t0).count();
    seconds3[1] = std::chrono::duration<double>(t2 - t1).count();
    seconds3[2] = std::chrono::duration<double>(t3 - t2).count();
    return DM_OK;
}

namespace dm {

// Forward relax descriptors, one per layer l (targets in layer l+1, or the
// TRUE terminal for a last layer at u = 0): bits 8u..8u+3 = local index of
// the zero-arc source of target u, bits 8u+4..8u+7 = its one-arc source,
// 15 = none.  Returns false when some layer is wider than 8 or has a target
// with two sources of one kind (then the tree-min kernel is used).
bool build_relax_by_layer(const int64_t *bdd_layer_lo, int64_t nb, const int64_t *lnl, const int64_t *zero_t,
                          const int64_t *one_t, std::vector<uint64_t> &desc_out) {
    const int64_t L = nb ? bdd_layer_lo[nb] : 0;
    desc_out.assign(L, ~0ull);
    constexpr int kThreads = 6;
    bool ok[kThreads];
    std::vector<std::thread> th;
    for (int t = 0; t < kThreads; ++t)
        th.emplace_back([&, t] {
            ok[t] = true;
            for (int64_t j = nb * t / kThreads; j < nb * (t + 1) / kThreads && ok[t]; ++j)
                for (int64_t l = bdd_layer_lo[j]; l < bdd_layer_lo[j + 1] && ok[t]; ++l) {
                    if (l + 1 == bdd_layer_lo[j + 1]) continue;  // last layers keep the tree path
                    const int64_t v0 = lnl[l], w = lnl[l + 1] - v0;
                    const int64_t n0 = lnl[l + 1];
                    const int64_t wn = lnl[l + 2] - n0;
                    if (w > 8 || wn > 8) {
                        ok[t] = false;
                        break;
                    }
                    uint64_t desc = ~0ull;
                    for (int64_t i = 0; i < w && ok[t]; ++i) {
                        const int64_t tg[2] = {zero_t[v0 + i], one_t[v0 + i]};
                        for (int k = 0; k < 2; ++k) {
                            if (tg[k] < 0) continue;  // terminal
                            const int64_t u = tg[k] - n0;
                            const int sh = 8 * (int)u + 4 * k;
                            if (u < 0 || u >= wn || ((desc >> sh) & 15) != 15) {
                                ok[t] = false;
                                break;
                            }
                            desc &= ~(15ull << sh);
                            desc |= (uint64_t)i << sh;
                        }
                    }
                    desc_out[l] = desc;
                }
        });
    for (auto &x : th) x.join();
    for (int t = 0; t < kThreads; ++t)
        if (!ok[t]) return false;
    return true;
}

}  // namespace dm
