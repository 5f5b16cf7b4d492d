// Host-side lowering for the B200 dual solver:
//   integer equality rows -> reduced layered diagrams   (bdd.py:362-501)
//   -> chunk splitting with one-hot coupling variables  (splitting.py:35-155)
//   -> flat node table + visitation CSR                 (kernels.py:35-92)
// plus the two plans the device needs: the numpy pairwise-summation tree and
// the level schedule of the exact averaging passes.
//
// Output layout is bit-identical to the reference pipeline
// IlpInstance.from_rows -> split_instance -> FlatBdds (checked against
// golden fixtures of the real reference in tests/test_lowering.py).
#include <algorithm>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <map>
#include <thread>
#include <vector>

#include "dm_internal.h"

namespace dm {

static thread_local std::string g_error;
void set_error(const std::string &msg) { g_error = msg; }

// ---------------------------------------------------------------------------
// Equality rows: states are partial sums of the prefix, windowed by what the
// suffix can still add ([rhs - maxrem, rhs - minrem] intersected with the
// prefix range), trimmed to states both reachable from 0 and co-reachable to
// rhs.  Surviving states of a layer are numbered in ascending sum order,
// which makes the diagram reduced (distinct sums have distinct futures after
// trimming) and reproduces the reference's node numbering.
int build_equality_bdd(const int64_t *coef, const int64_t *vars, int64_t n, int64_t rhs,
                       HostBdd &out) {
    if (n <= 0) {
        set_error("empty constraint row");
        return DM_ERR_INVALID;
    }
    std::vector<int64_t> suf_neg(n + 1, 0), suf_pos(n + 1, 0), pre_neg(n + 1, 0), pre_pos(n + 1, 0);
    for (int64_t l = n - 1; l >= 0; --l) {
        suf_neg[l] = suf_neg[l + 1] + std::min<int64_t>(coef[l], 0);
        suf_pos[l] = suf_pos[l + 1] + std::max<int64_t>(coef[l], 0);
    }
    for (int64_t l = 0; l < n; ++l) {
        pre_neg[l + 1] = pre_neg[l] + std::min<int64_t>(coef[l], 0);
        pre_pos[l + 1] = pre_pos[l] + std::max<int64_t>(coef[l], 0);
    }
    std::vector<int64_t> lo(n + 1), hi(n + 1), base(n + 2, 0);
    for (int64_t l = 0; l <= n; ++l) {
        lo[l] = std::max(pre_neg[l], rhs - suf_pos[l]);
        hi[l] = std::min(pre_pos[l], rhs - suf_neg[l]);
        base[l + 1] = base[l] + std::max<int64_t>(hi[l] - lo[l] + 1, 0);
    }
    const int64_t total = base[n + 1];
    auto infeasible = [&]() {
        set_error("no 0-1 solution of row == " + std::to_string(rhs));
        return DM_ERR_INFEASIBLE;
    };
    if (total == 0 || !(lo[0] <= 0 && 0 <= hi[0]) || !(lo[n] <= rhs && rhs <= hi[n]))
        return infeasible();
    auto slot = [&](int64_t l, int64_t s) -> int64_t {
        return (s < lo[l] || s > hi[l]) ? -1 : base[l] + (s - lo[l]);
    };
    std::vector<uint8_t> alive(total, 0);
    alive[slot(0, 0)] = 1;
    for (int64_t l = 0; l < n; ++l)
        for (int64_t s = lo[l]; s <= hi[l]; ++s) {
            if (!alive[slot(l, s)]) continue;
            int64_t a = slot(l + 1, s), b = slot(l + 1, s + coef[l]);
            if (a >= 0) alive[a] = 1;
            if (b >= 0) alive[b] = 1;
        }
    std::vector<uint8_t> good(total, 0);
    good[slot(n, rhs)] = 1;
    for (int64_t l = n - 1; l >= 0; --l)
        for (int64_t s = lo[l]; s <= hi[l]; ++s) {
            int64_t a = slot(l + 1, s), b = slot(l + 1, s + coef[l]);
            good[slot(l, s)] = (a >= 0 && good[a]) || (b >= 0 && good[b]);
        }
    std::vector<int64_t> id(total, -1);
    out.vars.assign(vars, vars + n);
    out.layer_lo.assign(n + 1, 0);
    for (int64_t l = 0; l < n; ++l) {
        int64_t cnt = 0;
        for (int64_t k = base[l]; k < base[l + 1]; ++k)
            if (alive[k] && good[k]) id[k] = cnt++;
        out.layer_lo[l + 1] = out.layer_lo[l] + cnt;
    }
    if (out.layer_lo[1] == 0) return infeasible();
    out.zeros.assign(out.layer_lo[n], kFalse);
    out.ones.assign(out.layer_lo[n], kFalse);
    for (int64_t l = 0; l < n; ++l)
        for (int64_t s = lo[l]; s <= hi[l]; ++s) {
            int64_t me = id[slot(l, s)];
            if (me < 0) continue;
            int64_t at = out.layer_lo[l] + me;
            if (l == n - 1) {
                out.zeros[at] = (s == rhs) ? kTrue : kFalse;
                out.ones[at] = (s + coef[l] == rhs) ? kTrue : kFalse;
            } else {
                int64_t a = slot(l + 1, s), b = slot(l + 1, s + coef[l]);
                int64_t ta = a >= 0 ? id[a] : -1, tb = b >= 0 ? id[b] : -1;
                out.zeros[at] = ta >= 0 ? (int32_t)ta : kFalse;
                out.ones[at] = tb >= 0 ? (int32_t)tb : kFalse;
            }
        }
    return DM_OK;
}

// ---------------------------------------------------------------------------
// Splitting (splitting.py:35-96).  Cut after `cut` layers; the k nodes of the
// crossing layer become k auxiliary variables y_t.  Left = prefix followed by
// a lattice accepting exactly y = e_t when the prefix reached node t; right =
// a lattice reading the one-hot y followed by the suffix from node t.
static void push_layer(HostBdd &b, int64_t var, const std::vector<int32_t> &z,
                       const std::vector<int32_t> &o) {
    b.vars.push_back(var);
    b.zeros.insert(b.zeros.end(), z.begin(), z.end());
    b.ones.insert(b.ones.end(), o.begin(), o.end());
    b.layer_lo.push_back(b.layer_lo.back() + (int64_t)z.size());
}

static void split_bdd(const HostBdd &src, int64_t cut, int64_t &fresh, HostBdd &left,
                      HostBdd &right, std::vector<int64_t> &aux) {
    const int64_t n = (int64_t)src.vars.size();
    const int64_t k = src.width(cut);
    aux.clear();
    for (int64_t t = 0; t < k; ++t) aux.push_back(fresh++);
    left = HostBdd();
    left.layer_lo.push_back(0);
    for (int64_t l = 0; l < cut; ++l) {
        std::vector<int32_t> z(src.zeros.begin() + src.layer_lo[l], src.zeros.begin() + src.layer_lo[l + 1]);
        std::vector<int32_t> o(src.ones.begin() + src.layer_lo[l], src.ones.begin() + src.layer_lo[l + 1]);
        push_layer(left, src.vars[l], z, o);
    }
    for (int64_t q = 0; q < k; ++q) {
        const int64_t pend = k - q;
        const bool final_ = q == k - 1;
        std::vector<int32_t> z(pend + (q > 0 ? 1 : 0), kFalse), o(z.size(), kFalse);
        o[0] = final_ ? kTrue : (int32_t)(pend - 1);  // choose y_q: into the "done" slot
        if (!final_)
            for (int64_t p = 1; p < pend; ++p) z[p] = (int32_t)(p - 1);  // still pending
        if (q > 0) z[pend] = final_ ? kTrue : (int32_t)(pend - 1);     // done: y stays 0
        push_layer(left, aux[q], z, o);
    }
    right = HostBdd();
    right.layer_lo.push_back(0);
    for (int64_t q = 0; q < k; ++q) {
        const bool final_ = q == k - 1;
        std::vector<int32_t> z(q + 1, kFalse), o(q + 1, kFalse);
        o[0] = (int32_t)(final_ ? q : q + 1);  // place the one-bit at t = q
        if (!final_) z[0] = 0;
        for (int64_t t = 0; t < q; ++t) z[t + 1] = (int32_t)(final_ ? t : t + 1);
        push_layer(right, aux[q], z, o);
    }
    for (int64_t l = cut; l < n; ++l) {
        std::vector<int32_t> z(src.zeros.begin() + src.layer_lo[l], src.zeros.begin() + src.layer_lo[l + 1]);
        std::vector<int32_t> o(src.ones.begin() + src.layer_lo[l], src.ones.begin() + src.layer_lo[l + 1]);
        push_layer(right, src.vars[l], z, o);
    }
}

// ---------------------------------------------------------------------------
int flatten(std::vector<HostBdd> &bdds, std::vector<double> costs, std::vector<int64_t> order,
            FlatHost &f) {
    const int64_t nv = (int64_t)costs.size();
    const int64_t nb = (int64_t)bdds.size();
    f.costs = std::move(costs);
    f.order = std::move(order);
    f.positions.assign(nv, -1);
    for (int64_t p = 0; p < nv; ++p) {
        int64_t v = f.order[p];
        if (v < 0 || v >= nv || f.positions[v] >= 0) {
            set_error("variable_order must be a permutation of all variables");
            return DM_ERR_INVALID;
        }
        f.positions[v] = p;
    }
    f.counts.assign(nv, 0);
    f.bdd_layer_lo.assign(nb + 1, 0);
    int64_t L = 0, N = 0;
    for (int64_t j = 0; j < nb; ++j) {
        const HostBdd &b = bdds[j];
        const int64_t n = (int64_t)b.vars.size();
        for (int64_t l = 0; l < n; ++l) {
            int64_t v = b.vars[l];
            if (v < 0 || v >= nv) {
                set_error("constraint references unknown variable");
                return DM_ERR_INVALID;
            }
            if (l > 0 && f.positions[v] <= f.positions[b.vars[l - 1]]) {
                set_error("constraint variables must follow the global order");
                return DM_ERR_INVALID;
            }
            f.counts[v] += 1;
        }
        L += n;
        N += b.layer_lo[n];
        f.bdd_layer_lo[j + 1] = L;
        f.max_layers = std::max(f.max_layers, n);
    }
    f.layer_node_lo.assign(L + 1, 0);
    f.layer_var.resize(L);
    f.layer_bdd.resize(L);
    f.zero_t.resize(N);
    f.one_t.resize(N);
    int64_t l_at = 0;
    for (int64_t j = 0; j < nb; ++j) {
        HostBdd &b = bdds[j];
        const int64_t n = (int64_t)b.vars.size();
        for (int64_t l = 0; l < n; ++l, ++l_at) {
            const int64_t w = b.width(l);
            f.max_width = std::max(f.max_width, w);
            f.layer_var[l_at] = b.vars[l];
            f.layer_bdd[l_at] = j;
            const int64_t node0 = f.layer_node_lo[l_at];
            const int64_t next0 = node0 + w;  // first node of the next layer
            f.layer_node_lo[l_at + 1] = next0;
            for (int64_t i = 0; i < w; ++i) {
                int32_t z = b.zeros[b.layer_lo[l] + i], o = b.ones[b.layer_lo[l] + i];
                f.zero_t[node0 + i] = z >= 0 ? next0 + z : z;
                f.one_t[node0 + i] = o >= 0 ? next0 + o : o;
            }
        }
        HostBdd().vars.swap(b.vars);  // release as we go
        std::vector<int32_t>().swap(b.zeros);
        std::vector<int32_t>().swap(b.ones);
    }
    // stable counting sort of layers by visitation position
    f.proc_ptr.assign(nv + 1, 0);
    for (int64_t l = 0; l < L; ++l) f.proc_ptr[f.positions[f.layer_var[l]] + 1] += 1;
    for (int64_t p = 0; p < nv; ++p) {
        f.max_degree = std::max(f.max_degree, f.proc_ptr[p + 1]);
        f.proc_ptr[p + 1] += f.proc_ptr[p];
    }
    std::vector<int64_t> fill(f.proc_ptr.begin(), f.proc_ptr.end() - 1);
    f.proc_layers.resize(L);
    for (int64_t l = 0; l < L; ++l) f.proc_layers[fill[f.positions[f.layer_var[l]]]++] = l;
    return DM_OK;
}

// ---------------------------------------------------------------------------
PairwisePlan plan_pairwise(int64_t n) {
    PairwisePlan p;
    p.n = n;
    struct Tmp { int32_t l, r, h; };
    std::vector<Tmp> inner;
    std::vector<int32_t> leaf_h;  // unused, leaves have height 0
    // returns encoded id: >= 0 leaf index, < 0 -(inner index + 1); height via out
    std::vector<int64_t> dummy;
    struct Rec {
        PairwisePlan &p;
        std::vector<Tmp> &inner;
        int64_t go(int64_t off, int64_t len, int32_t &h) {
            if (len <= 128) {
                p.leaf_off.push_back(off);
                p.leaf_len.push_back((int32_t)len);
                h = 0;
                return (int64_t)p.leaf_off.size() - 1;
            }
            int64_t n2 = len / 2;
            n2 -= n2 % 8;
            int32_t hl, hr;
            int64_t a = go(off, n2, hl);
            int64_t b = go(off + n2, len - n2, hr);
            inner.push_back({(int32_t)a, (int32_t)b, std::max(hl, hr) + 1});
            h = inner.back().h;
            return -(int64_t)inner.size();
        }
    } rec{p, inner};
    int32_t h;
    int64_t root = rec.go(0, n, h);
    const int64_t nl = (int64_t)p.leaf_off.size();
    const int64_t ni = (int64_t)inner.size();
    // order internal nodes by height (stable), remap child ids to value slots
    std::vector<int64_t> idx(ni);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return inner[a].h < inner[b].h; });
    std::vector<int64_t> rank(ni);
    for (int64_t r = 0; r < ni; ++r) rank[idx[r]] = r;
    auto slot = [&](int64_t enc) -> int32_t {
        return enc >= 0 ? (int32_t)enc : (int32_t)(nl + rank[-enc - 1]);
    };
    int32_t maxh = ni ? inner[idx[ni - 1]].h : 0;
    p.height_lo.assign(maxh + 1, 0);
    p.left.resize(ni);
    p.right.resize(ni);
    for (int64_t r = 0; r < ni; ++r) {
        const Tmp &t = inner[idx[r]];
        p.left[r] = slot(t.l);
        p.right[r] = slot(t.r);
        p.height_lo[t.h] = (int32_t)(r + 1);  // running end of height t.h
    }
    // height_lo[h] = end of nodes with height <= h ; fill gaps monotonically
    for (int32_t k = 1; k <= maxh; ++k) p.height_lo[k] = std::max(p.height_lo[k], p.height_lo[k - 1]);
    p.root = slot(root);
    return p;
}

// ---------------------------------------------------------------------------
int build_mma_schedule(const int64_t *bdd_layer_lo, int64_t nb, const int64_t *layer_bdd,
                       const int64_t *layer_var, int64_t L, const int64_t *proc_ptr,
                       const int64_t *proc_layers, int64_t npos, bool forward, MmaSchedule &s) {
    (void)layer_var;
    (void)layer_bdd;
    // Level of each position along the dependency DAG: a copy at layer l
    // depends on the copy at layer l-1 (forward) / l+1 (backward) of its
    // diagram, which the visitation order processes just before — so it is
    // the diagram's most recently processed layer, and a per-diagram "level
    // of the last processed layer" (small, cache-resident) replaces random
    // reads of a per-layer table.  The per-copy diagram ids and end flags are
    // gathered in parallel first.
    std::vector<int32_t> lbdd(L), cb(L);
    std::vector<uint8_t> ce(L);
    {
        constexpr int kThreads = 8;
        auto par = [&](int64_t n, auto &&fn) {
            std::vector<std::thread> th;
            for (int t = 0; t < kThreads; ++t) th.emplace_back([&, t] { fn(n * t / kThreads, n * (t + 1) / kThreads); });
            for (auto &x : th) x.join();
        };
        par(nb, [&](int64_t lo, int64_t hi) {
            for (int64_t j = lo; j < hi; ++j)
                for (int64_t l = bdd_layer_lo[j]; l < bdd_layer_lo[j + 1]; ++l) lbdd[l] = (int32_t)j;
        });
        par(L, [&](int64_t lo, int64_t hi) {
            for (int64_t t = lo; t < hi; ++t) {
                const int64_t l = proc_layers[t];
                const int32_t j = lbdd[l];
                cb[t] = j;
                ce[t] = forward ? (l == bdd_layer_lo[j]) : (l + 1 == bdd_layer_lo[j + 1]);
            }
        });
    }
    std::vector<int32_t> last_level(nb, 0);
    std::vector<int32_t> pos_level(npos, -1);
    int32_t depth = 0;
    for (int64_t k = 0; k < npos; ++k) {
        const int64_t p = forward ? k : npos - 1 - k;
        const int64_t lo = proc_ptr[p], hi = proc_ptr[p + 1];
        if (hi == lo) continue;
        if (hi - lo > 32) {
            set_error("exact averaging pass supports at most 32 diagrams per variable (got " +
                      std::to_string(hi - lo) + ")");
            return DM_ERR_UNSUPPORTED;
        }
        int32_t lev = 0;
        for (int64_t t = lo; t < hi; ++t)
            if (!ce[t]) lev = std::max(lev, last_level[cb[t]] + 1);
        for (int64_t t = lo; t < hi; ++t) last_level[cb[t]] = lev;
        pos_level[p] = lev;
        depth = std::max(depth, lev + 1);
    }
    // bucket positions by level, keeping visitation order inside a level
    std::vector<int64_t> cnt(depth + 1, 0);
    for (int64_t p = 0; p < npos; ++p)
        if (pos_level[p] >= 0) cnt[pos_level[p] + 1]++;
    for (int32_t d = 0; d < depth; ++d) cnt[d + 1] += cnt[d];
    std::vector<int64_t> bylevel(cnt[depth]);
    {
        std::vector<int64_t> at(cnt.begin(), cnt.end() - 1);
        for (int64_t k = 0; k < npos; ++k) {
            const int64_t p = forward ? k : npos - 1 - k;
            if (pos_level[p] >= 0) bylevel[at[pos_level[p]]++] = p;
        }
    }
    s.pos_order.resize(bylevel.size());
    s.pos_order_level.resize(bylevel.size());
    for (size_t i = 0; i < bylevel.size(); ++i) {
        s.pos_order[i] = (int32_t)bylevel[i];
        s.pos_order_level[i] = pos_level[bylevel[i]];
    }
    s.depth = depth;
    s.task_layer.clear();
    s.task_meta.clear();
    s.task_level.clear();
    s.tasks = 0;
    return DM_OK;
}

// Per-copy warp tasks (the fallback kernels): same-level positions packed
// into 32-lane tasks, copies of a position adjacent in copy order.
void pack_mma_tasks(const std::vector<int32_t> &pos_order, const std::vector<int32_t> &pos_order_level,
                    const int32_t *proc_ptr, const int32_t *proc_layers, const uint8_t *layer_flags,
                    MmaSchedule &s) {
    s.task_layer.clear();
    s.task_meta.clear();
    s.task_level.clear();
    int used = 32;  // lanes used in the open task (32 = none open)
    int32_t open_level = -1;
    auto open_task = [&]() {
        s.task_layer.insert(s.task_layer.end(), 32, -1);
        s.task_meta.insert(s.task_meta.end(), 32, 0);
        used = 0;
    };
    for (size_t i = 0; i < pos_order.size(); ++i) {
        const int64_t p = pos_order[i];
        const int64_t lo = proc_ptr[p], hi = proc_ptr[p + 1];
        const int c = (int)(hi - lo);
        if (pos_order_level[i] != open_level || used + c > 32) {
            open_task();
            open_level = pos_order_level[i];
            s.task_level.push_back(open_level);
        }
        const size_t base = s.task_layer.size() - 32;
        for (int k = 0; k < c; ++k) {
            const int64_t l = proc_layers[lo + k];
            int32_t meta = used | (c << 8);
            if (layer_flags[l] & 1) meta |= 1 << 16;
            if (layer_flags[l] & 2) meta |= 1 << 17;
            s.task_layer[base + used + k] = (int32_t)l;
            s.task_meta[base + used + k] = meta;
        }
        used += c;
    }
    s.tasks = (int64_t)s.task_layer.size() / 32;
}

}  // namespace dm

// ===========================================================================
// C-ABI: host instances
// ===========================================================================
struct dm_instance {
    dm::FlatHost flat;
};

// splitting.py:116-155 then kernels.py:43-92
static int split_and_flatten(std::vector<dm::HostBdd> &bdds, std::vector<double> cst,
                             std::vector<int64_t> order, int64_t chunk_size, dm_instance **out) {
    const int64_t num_variables = (int64_t)cst.size();
    bool any = false;
    if (chunk_size > 0)
        for (auto &b : bdds) any |= (int64_t)b.vars.size() > chunk_size;
    if (any) {
        int64_t fresh = num_variables;
        std::vector<std::vector<int64_t>> after(num_variables);
        std::vector<dm::HostBdd> outb;
        outb.reserve(bdds.size());
        std::vector<int64_t> aux;
        for (auto &b : bdds) {
            const int64_t n = (int64_t)b.vars.size();
            if (n <= chunk_size) {
                outb.push_back(std::move(b));
                continue;
            }
            dm::HostBdd rest = b, left, right;
            int64_t prev = 0, carried = 0;
            for (int64_t cut = chunk_size; cut < n; cut += chunk_size) {
                dm::split_bdd(rest, carried + cut - prev, fresh, left, right, aux);
                auto &slot = after[b.vars[cut - 1]];
                slot.insert(slot.end(), aux.begin(), aux.end());
                outb.push_back(std::move(left));
                rest = std::move(right);
                carried = (int64_t)aux.size();
                prev = cut;
            }
            outb.push_back(std::move(rest));
        }
        bdds.swap(outb);
        cst.resize(fresh, 0.0);
        std::vector<int64_t> norder;
        norder.reserve(fresh);
        for (int64_t x : order) {
            norder.push_back(x);
            norder.insert(norder.end(), after[x].begin(), after[x].end());
        }
        order.swap(norder);
    }
    auto inst = std::make_unique<dm_instance>();
    int rc = dm::flatten(bdds, std::move(cst), std::move(order), inst->flat);
    if (rc != DM_OK) return rc;
    *out = inst.release();
    return DM_OK;
}

extern "C" {

const char *dm_last_error(void) { return dm::g_error.c_str(); }

int dm_instance_from_rows(int64_t num_variables, const double *costs, int64_t num_rows,
                          const int64_t *row_ptr, const int64_t *row_var,
                          const int64_t *row_coef, const int64_t *row_rhs, int64_t chunk_size,
                          dm_instance **out) {
    if (!out || num_variables < 0 || num_rows < 0 || (num_variables && !costs) ||
        (num_rows && (!row_ptr || !row_var || !row_coef || !row_rhs))) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    if (chunk_size > 0 && chunk_size < 2) {
        dm::set_error("chunk_size must be at least 2");
        return DM_ERR_INVALID;
    }
    *out = nullptr;
    std::vector<dm::HostBdd> bdds;
    bdds.reserve(num_rows);
    std::vector<int64_t> perm, v, c;
    // ilp.py:94-107: each row is canonicalised by a stable sort of its ids
    for (int64_t r = 0; r < num_rows; ++r) {
        const int64_t lo = row_ptr[r], hi = row_ptr[r + 1];
        const int64_t n = hi - lo;
        perm.resize(n);
        std::iota(perm.begin(), perm.end(), 0);
        std::stable_sort(perm.begin(), perm.end(),
                         [&](int64_t a, int64_t b) { return row_var[lo + a] < row_var[lo + b]; });
        v.resize(n);
        c.resize(n);
        for (int64_t k = 0; k < n; ++k) {
            v[k] = row_var[lo + perm[k]];
            c[k] = row_coef[lo + perm[k]];
            if (k && v[k] == v[k - 1]) {
                dm::set_error("duplicate variable in constraint (row " + std::to_string(r) + ")");
                return DM_ERR_INVALID;
            }
        }
        bdds.emplace_back();
        int rc = dm::build_equality_bdd(c.data(), v.data(), n, row_rhs[r], bdds.back());
        if (rc != DM_OK) {
            dm::set_error(std::string(dm_last_error()) + " (row " + std::to_string(r) + ")");
            return rc;
        }
    }
    std::vector<double> cst(costs, costs + num_variables);
    std::vector<int64_t> order(num_variables);
    std::iota(order.begin(), order.end(), 0);
    return split_and_flatten(bdds, std::move(cst), std::move(order), chunk_size, out);
}

int dm_instance_from_bdds(int64_t num_variables, const double *costs, const int64_t *variable_order,
                          int64_t num_bdds, const int64_t *bdd_layer_lo, const int64_t *layer_var,
                          const int64_t *layer_node_lo, const int32_t *zeros, const int32_t *ones,
                          int64_t chunk_size, dm_instance **out) {
    if (!out || num_variables < 0 || num_bdds < 0 || (num_variables && !costs) ||
        (num_bdds && (!bdd_layer_lo || !layer_var || !layer_node_lo || !zeros || !ones))) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    if (chunk_size > 0 && chunk_size < 2) {
        dm::set_error("chunk_size must be at least 2");
        return DM_ERR_INVALID;
    }
    *out = nullptr;
    std::vector<dm::HostBdd> bdds(num_bdds);
    for (int64_t j = 0; j < num_bdds; ++j) {
        dm::HostBdd &b = bdds[j];
        const int64_t l0 = bdd_layer_lo[j], l1 = bdd_layer_lo[j + 1];
        if (l1 <= l0) {
            dm::set_error("a diagram needs at least one variable");
            return DM_ERR_INVALID;
        }
        b.vars.assign(layer_var + l0, layer_var + l1);
        b.layer_lo.assign(1, 0);
        const int64_t n0 = layer_node_lo[l0];
        for (int64_t l = l0; l < l1; ++l) b.layer_lo.push_back(layer_node_lo[l + 1] - n0);
        b.zeros.assign(zeros + n0, zeros + layer_node_lo[l1]);
        b.ones.assign(ones + n0, ones + layer_node_lo[l1]);
    }
    std::vector<double> cst(costs, costs + num_variables);
    std::vector<int64_t> order(num_variables);
    if (variable_order)
        order.assign(variable_order, variable_order + num_variables);
    else
        std::iota(order.begin(), order.end(), 0);
    return split_and_flatten(bdds, std::move(cst), std::move(order), chunk_size, out);
}

// Conditioning for the primal side (bdd.py:243-264 Bdd.condition +
// reduce_bdd bdd.py:278-334, primal.py:114-175 fix_and_reduce): clamp the
// fixed variables of every touched diagram, re-reduce it (prune dead arcs
// bottom-up, drop unreachable nodes, merge isomorphic nodes keeping
// first-occurrence order), drop diagrams that became a single chain
// accepting every fix-consistent assignment, and lower what remains as a new
// instance (same costs and variable order, no splitting).
namespace {

// local arcs: >= 0 next-layer node, FALSE (-1), TRUE (-2); returns false when emptied
bool reduce_local(std::vector<std::vector<int32_t>> &zs, std::vector<std::vector<int32_t>> &os) {
    const size_t n = zs.size();
    std::vector<std::vector<char>> alive(n);
    for (size_t l = n; l-- > 0;) {
        for (auto *arcs : {&zs[l], &os[l]})
            if (l + 1 < n)
                for (auto &t : *arcs)
                    if (t >= 0 && !alive[l + 1][t]) t = dm::kFalse;
        alive[l].resize(zs[l].size());
        for (size_t i = 0; i < zs[l].size(); ++i) alive[l][i] = zs[l][i] != dm::kFalse || os[l][i] != dm::kFalse;
    }
    if (!alive[0][0]) return false;
    std::vector<std::vector<char>> reach(n);
    reach[0].assign(1, 1);
    for (size_t l = 0; l + 1 < n; ++l) {
        reach[l + 1].assign(zs[l + 1].size(), 0);
        for (auto *arcs : {&zs[l], &os[l]})
            for (size_t i = 0; i < arcs->size(); ++i)
                if (reach[l][i] && (*arcs)[i] >= 0) reach[l + 1][(*arcs)[i]] = 1;
    }
    std::vector<int64_t> remap;  // old id in layer l+1 -> new id (or FALSE)
    for (size_t l = n; l-- > 0;) {
        const size_t w = zs[l].size();
        std::vector<int32_t> nz, no;
        std::vector<int64_t> rm(w, dm::kFalse);
        // merge key exactly as reduce_bdd forms it: (z + 2) * (width of THIS
        // layer + 3) + (o + 2), first occurrence wins
        std::map<int64_t, int32_t> first;
        for (size_t i = 0; i < w; ++i) {
            if (!(alive[l][i] && reach[l][i])) continue;
            int32_t z = zs[l][i], o = os[l][i];
            if (z >= 0) z = (int32_t)remap[z];
            if (o >= 0) o = (int32_t)remap[o];
            const int64_t key = ((int64_t)z + 2) * ((int64_t)w + 3) + ((int64_t)o + 2);
            auto it = first.find(key);
            if (it == first.end()) {
                const int32_t id = (int32_t)nz.size();
                first.emplace(key, id);
                nz.push_back(z);
                no.push_back(o);
                rm[i] = id;
            } else {
                rm[i] = it->second;
            }
        }
        zs[l] = std::move(nz);
        os[l] = std::move(no);
        remap = std::move(rm);
    }
    return true;
}

}  // namespace

int dm_condition_flat(int64_t num_variables, const double *costs, const int64_t *variable_order, int64_t num_bdds,
                      const int64_t *bdd_layer_lo, const int64_t *layer_var, const int64_t *layer_node_lo,
                      const int64_t *zero_t, const int64_t *one_t, const int8_t *fixed, int64_t *dropped_out,
                      dm_instance **out) {
    if (!out || !fixed || num_variables < 0 || num_bdds < 0 || (num_variables && !costs) ||
        (num_bdds && (!bdd_layer_lo || !layer_var || !layer_node_lo || !zero_t || !one_t))) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    *out = nullptr;
    std::vector<dm::HostBdd> kept;
    int64_t dropped = 0;
    for (int64_t j = 0; j < num_bdds; ++j) {
        const int64_t l0 = bdd_layer_lo[j], l1 = bdd_layer_lo[j + 1], n = l1 - l0;
        bool touched = false;
        for (int64_t l = l0; l < l1; ++l) touched |= fixed[layer_var[l]] >= 0;
        std::vector<std::vector<int32_t>> zs(n), os(n);
        for (int64_t l = l0; l < l1; ++l) {
            const int64_t a = layer_node_lo[l], b = layer_node_lo[l + 1], nxt = layer_node_lo[l + 1];
            for (int64_t v = a; v < b; ++v) {
                const int64_t z = zero_t[v], o = one_t[v];
                zs[l - l0].push_back((int32_t)(z >= 0 ? z - nxt : z));
                os[l - l0].push_back((int32_t)(o >= 0 ? o - nxt : o));
            }
            const int8_t fx = fixed[layer_var[l]];
            if (fx == 1) std::fill(zs[l - l0].begin(), zs[l - l0].end(), dm::kFalse);
            if (fx == 0) std::fill(os[l - l0].begin(), os[l - l0].end(), dm::kFalse);
        }
        if (touched) {
            if (!reduce_local(zs, os)) {
                dm::set_error("conditioning emptied constraint " + std::to_string(j));
                return DM_ERR_INFEASIBLE;
            }
            // primal.py:114-130: a single chain accepting every fix-consistent assignment
            bool constant = true;
            for (int64_t k = 0; k < n && constant; ++k) {
                if (zs[k].size() != 1) constant = false;
                else if (fixed[layer_var[l0 + k]] >= 0) continue;
                else if (zs[k][0] == dm::kFalse || zs[k][0] != os[k][0]) constant = false;
            }
            if (constant) {
                ++dropped;
                continue;
            }
        }
        dm::HostBdd hb;
        hb.vars.assign(layer_var + l0, layer_var + l1);
        hb.layer_lo.assign(1, 0);
        for (int64_t k = 0; k < n; ++k) {
            hb.layer_lo.push_back(hb.layer_lo.back() + (int64_t)zs[k].size());
            hb.zeros.insert(hb.zeros.end(), zs[k].begin(), zs[k].end());
            hb.ones.insert(hb.ones.end(), os[k].begin(), os[k].end());
        }
        kept.push_back(std::move(hb));
    }
    if (dropped_out) *dropped_out = dropped;
    std::vector<double> cst(costs, costs + num_variables);
    std::vector<int64_t> order(num_variables);
    if (variable_order)
        order.assign(variable_order, variable_order + num_variables);
    else
        std::iota(order.begin(), order.end(), 0);
    return split_and_flatten(kept, std::move(cst), std::move(order), 0, out);
}

int dm_row_colouring(int64_t num_variables, int64_t num_rows, const int64_t *row_ptr, const int64_t *row_var,
                     int64_t *colour_out) {
    if (num_variables < 0 || num_rows < 0 || (num_rows && (!row_ptr || !row_var)) || (num_variables && !colour_out)) {
        dm::set_error("dm_row_colouring: invalid arguments");
        return DM_ERR_INVALID;
    }
    // variable -> rows (CSR)
    std::vector<int64_t> vptr(num_variables + 1, 0);
    for (int64_t r = 0; r < num_rows; ++r)
        for (int64_t i = row_ptr[r]; i < row_ptr[r + 1]; ++i) {
            const int64_t v = row_var[i];
            if (v < 0 || v >= num_variables) {
                dm::set_error("dm_row_colouring: variable id out of range");
                return DM_ERR_INVALID;
            }
            ++vptr[v + 1];
        }
    for (int64_t v = 0; v < num_variables; ++v) vptr[v + 1] += vptr[v];
    std::vector<int64_t> vrows(vptr[num_variables]), fill(vptr.begin(), vptr.end() - 1);
    for (int64_t r = 0; r < num_rows; ++r)
        for (int64_t i = row_ptr[r]; i < row_ptr[r + 1]; ++i) vrows[fill[row_var[i]]++] = r;
    // colours each row already holds, as growing bitsets
    std::vector<std::vector<uint64_t>> used(num_rows);
    std::vector<uint64_t> taken;
    for (int64_t v = 0; v < num_variables; ++v) {
        taken.assign(taken.size(), 0);
        for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k) {
            const auto &u = used[vrows[k]];
            if (u.size() > taken.size()) taken.resize(u.size(), 0);
            for (size_t w = 0; w < u.size(); ++w) taken[w] |= u[w];
        }
        size_t w = 0;
        while (w < taken.size() && taken[w] == ~0ull) ++w;
        const int64_t c = (int64_t)(w * 64 + (w < taken.size() ? __builtin_ctzll(~taken[w]) : 0));
        colour_out[v] = c;
        const size_t cw = (size_t)(c >> 6);
        for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k) {
            auto &u = used[vrows[k]];
            if (u.size() <= cw) u.resize(cw + 1, 0);
            u[cw] |= 1ull << (c & 63);
        }
    }
    return DM_OK;
}

int dm_instance_get_info(const dm_instance *inst, dm_instance_info *info) {
    if (!inst || !info) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    const dm::FlatHost &f = inst->flat;
    info->num_variables = (int64_t)f.costs.size();
    info->num_bdds = (int64_t)f.bdd_layer_lo.size() - 1;
    info->num_layers = (int64_t)f.layer_var.size();
    info->num_nodes = (int64_t)f.zero_t.size();
    info->max_width = f.max_width;
    info->max_degree = f.max_degree;
    info->max_layers = f.max_layers;
    return DM_OK;
}

int dm_instance_export(const dm_instance *inst, double *costs, int64_t *variable_order,
                       int64_t *bdd_layer_lo, int64_t *layer_node_lo, int64_t *layer_var,
                       int64_t *layer_bdd, int64_t *zero_t, int64_t *one_t, int64_t *proc_ptr,
                       int64_t *proc_layers, int64_t *constraint_counts) {
    if (!inst) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    const dm::FlatHost &f = inst->flat;
    auto cp = [](auto *dst, const auto &src) {
        if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
    };
    cp(costs, f.costs);
    cp(variable_order, f.order);
    cp(bdd_layer_lo, f.bdd_layer_lo);
    cp(layer_node_lo, f.layer_node_lo);
    cp(layer_var, f.layer_var);
    cp(layer_bdd, f.layer_bdd);
    cp(zero_t, f.zero_t);
    cp(one_t, f.one_t);
    cp(proc_ptr, f.proc_ptr);
    cp(proc_layers, f.proc_layers);
    cp(constraint_counts, f.counts);
    return DM_OK;
}

void dm_instance_free(dm_instance *inst) { delete inst; }

}  // extern "C"

// ===========================================================================
// Host emulation of the device plans (test hooks, never on the product path)
// ===========================================================================
namespace {

double host_leaf(const double *a, int64_t off, int32_t n) {
    const double *p = a + off;
    if (n < 8) {
        double res = 0.0;
        for (int32_t i = 0; i < n; ++i) res += p[i];
        return res;
    }
    double r[8];
    for (int q = 0; q < 8; ++q) r[q] = p[q];
    int32_t i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int q = 0; q < 8; ++q) r[q] += p[i + q];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += p[i];
    return res;
}

}  // namespace

extern "C" {

int dm_host_pairwise_sum(const double *x, int64_t n, double *out) {
    if (n < 0 || (n && !x) || !out) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    dm::PairwisePlan p = dm::plan_pairwise(n);
    const size_t nl = p.leaf_off.size();
    std::vector<double> vals(nl + p.left.size());
    for (size_t k = 0; k < nl; ++k) vals[k] = host_leaf(x, p.leaf_off[k], p.leaf_len[k]);
    for (size_t k = 0; k < p.left.size(); ++k) vals[nl + k] = vals[p.left[k]] + vals[p.right[k]];
    *out = 0.0 + vals[p.root];
    return DM_OK;
}

// Executes the level schedule of one exact averaging pass task by task, with
// the device kernel's lane semantics.  Proves on the host that the schedule
// (levels + lane packing) reproduces the sequential reference pass.
int dm_debug_emulate_mma(const dm_flat_desc *d, int forward, double *lam, double *F, double *B,
                         double *bounds, int64_t *depth_out) {
    if (!d) {
        dm::set_error("invalid arguments");
        return DM_ERR_INVALID;
    }
    const int64_t nb = d->num_bdds, L = d->num_layers, P = d->num_positions;
    dm::MmaSchedule s;
    int rc = dm::build_mma_schedule(d->bdd_layer_lo, nb, nullptr, d->layer_var, L, d->proc_ptr,
                                    d->proc_layers, P, forward != 0, s);
    if (rc != DM_OK) return rc;
    {
        std::vector<uint8_t> flags(L, 0);
        for (int64_t j = 0; j < nb; ++j) {
            flags[d->bdd_layer_lo[j]] |= 1;
            flags[d->bdd_layer_lo[j + 1] - 1] |= 2;
        }
        std::vector<int32_t> pp(P + 1), pl(L);
        for (int64_t p = 0; p <= P; ++p) pp[p] = (int32_t)d->proc_ptr[p];
        for (int64_t l = 0; l < L; ++l) pl[l] = (int32_t)d->proc_layers[l];
        dm::pack_mma_tasks(s.pos_order, s.pos_order_level, pp.data(), pl.data(), flags.data(), s);
    }
    if (depth_out) *depth_out = s.depth;
    std::vector<int64_t> layer_bdd(L);
    for (int64_t j = 0; j < nb; ++j)
        for (int64_t l = d->bdd_layer_lo[j]; l < d->bdd_layer_lo[j + 1]; ++l) layer_bdd[l] = j;
    const int64_t *lnl = d->layer_node_lo, *zt = d->zero_t, *ot = d->one_t;
    const double INF = __builtin_inf();
    if (forward)
        for (int64_t j = 0; j < nb; ++j) F[lnl[d->bdd_layer_lo[j]]] = 0.0;
    for (int64_t t = 0; t < s.tasks; ++t) {
        double m0[32], m1[32];
        for (int ln = 0; ln < 32; ++ln) {
            const int64_t l = s.task_layer[t * 32 + ln];
            m0[ln] = m1[ln] = INF;
            if (l < 0) continue;
            for (int64_t v = lnl[l]; v < lnl[l + 1]; ++v) {
                const double fv = F[v];
                if (fv == INF) continue;
                const int64_t a = zt[v], b = ot[v];
                const double c0 = a == dm::kTrue ? fv : (a == dm::kFalse ? INF : fv + B[a]);
                if (c0 < m0[ln]) m0[ln] = c0;
                const double c1 = b == dm::kTrue ? fv + lam[l] : (b == dm::kFalse ? INF : (fv + lam[l]) + B[b]);
                if (c1 < m1[ln]) m1[ln] = c1;
            }
        }
        for (int ln = 0; ln < 32; ++ln) {
            const int64_t l = s.task_layer[t * 32 + ln];
            if (l < 0) continue;
            const int32_t meta = s.task_meta[t * 32 + ln];
            const int gb = meta & 0xff, gc = (meta >> 8) & 0xff;
            double fsum = 0.0;
            int fcnt = 0;
            for (int k = 0; k < gc; ++k)
                if (m0[gb + k] != INF && m1[gb + k] != INF) {
                    fsum += m1[gb + k] - m0[gb + k];
                    ++fcnt;
                }
            if (fcnt > 0 && m0[ln] != INF && m1[ln] != INF) lam[l] += fsum / fcnt - (m1[ln] - m0[ln]);
        }
        for (int ln = 0; ln < 32; ++ln) {
            const int64_t l = s.task_layer[t * 32 + ln];
            if (l < 0) continue;
            const int32_t meta = s.task_meta[t * 32 + ln];
            const int64_t j = layer_bdd[l];
            if (forward) {
                if (!(meta & (1 << 17))) {
                    for (int64_t w = lnl[l + 1]; w < lnl[l + 2]; ++w) F[w] = INF;
                    for (int64_t v = lnl[l]; v < lnl[l + 1]; ++v) {
                        const double fv = F[v];
                        if (fv == INF) continue;
                        if (zt[v] >= 0 && fv < F[zt[v]]) F[zt[v]] = fv;
                        const double c = fv + lam[l];
                        if (ot[v] >= 0 && c < F[ot[v]]) F[ot[v]] = c;
                    }
                } else {
                    double tb = INF;
                    for (int64_t v = lnl[l]; v < lnl[l + 1]; ++v) {
                        const double fv = F[v];
                        if (fv == INF) continue;
                        if (zt[v] == dm::kTrue && fv < tb) tb = fv;
                        const double c = fv + lam[l];
                        if (ot[v] == dm::kTrue && c < tb) tb = c;
                    }
                    bounds[j] = tb;
                }
            } else {
                for (int64_t v = lnl[l]; v < lnl[l + 1]; ++v) {
                    const int64_t a = zt[v], b = ot[v];
                    const double c0 = a == dm::kTrue ? 0.0 : (a == dm::kFalse ? INF : B[a]);
                    const double c1 = b == dm::kTrue ? lam[l] : (b == dm::kFalse ? INF : lam[l] + B[b]);
                    B[v] = c0 <= c1 ? c0 : c1;
                }
                if (meta & (1 << 16)) bounds[j] = B[lnl[l]];
            }
        }
    }
    return DM_OK;
}

}  // extern "C"
