/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's numba sweep kernels
 * (/root/reference/pkg/src/prodmatch/kernels.py) and of the equality-row
 * diagram compiler (/root/reference/pkg/src/prodmatch/bdd.py:362-475).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the CPU baseline; the product path never touches it.
 *
 * Arithmetic follows the reference exactly: IEEE binary64, no contraction
 * (compiled with -ffp-contract=off), the same association order
 * ((F[v] + lam_l) + B[t]), the same strict/non-strict comparisons and the
 * same per-variable summation order, so results are bitwise equal to the
 * numba kernels.  Kernels the reference runs with prange are OpenMP-parallel
 * over the same independent units (diagrams / layers); each unit writes only
 * its own slots, so results do not depend on the thread count.
 *
 * Array conventions follow FlatBdds (kernels.py:35-92): node targets are
 * global node ids, -1 = FALSE terminal, -2 = TRUE terminal.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TGT_FALSE (-1)
#define TGT_TRUE (-2)

typedef int64_t i64;

int oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n < 1) n = 1;
    omp_set_num_threads(n);
    return n;
#else
    (void)n;
    return 1;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* kernels.py:95-120 — distance to TRUE, bottom-up per diagram. */
void oracle_k_backward(i64 nb, const i64 *bdd_layer_lo, const i64 *layer_node_lo,
                       const i64 *zero_t, const i64 *one_t, const double *lam,
                       double *B, double *bounds) {
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 j = 0; j < nb; ++j) {
        i64 l_lo = bdd_layer_lo[j], l_hi = bdd_layer_lo[j + 1];
        for (i64 l = l_hi - 1; l >= l_lo; --l) {
            double lam_l = lam[l];
            for (i64 v = layer_node_lo[l]; v < layer_node_lo[l + 1]; ++v) {
                i64 a = zero_t[v], b = one_t[v];
                double c0 = a == TGT_TRUE ? 0.0 : (a == TGT_FALSE ? INFINITY : B[a]);
                double c1 = b == TGT_TRUE ? lam_l : (b == TGT_FALSE ? INFINITY : lam_l + B[b]);
                B[v] = (c0 <= c1) ? c0 : c1;
            }
        }
        bounds[j] = B[layer_node_lo[l_lo]];
    }
}

/* Same sweep on lam + gamma*d materialised per layer with numpy's two
 * roundings (qn.py:147,153: `lam + gamma * d`), used by the step search. */
void oracle_k_backward_trial(i64 nb, const i64 *bdd_layer_lo, const i64 *layer_node_lo,
                             const i64 *zero_t, const i64 *one_t, const double *lam,
                             const double *d, double gamma, double *B, double *bounds) {
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 j = 0; j < nb; ++j) {
        i64 l_lo = bdd_layer_lo[j], l_hi = bdd_layer_lo[j + 1];
        for (i64 l = l_hi - 1; l >= l_lo; --l) {
            double step = gamma * d[l];
            double lam_l = lam[l] + step;
            for (i64 v = layer_node_lo[l]; v < layer_node_lo[l + 1]; ++v) {
                i64 a = zero_t[v], b = one_t[v];
                double c0 = a == TGT_TRUE ? 0.0 : (a == TGT_FALSE ? INFINITY : B[a]);
                double c1 = b == TGT_TRUE ? lam_l : (b == TGT_FALSE ? INFINITY : lam_l + B[b]);
                B[v] = (c0 <= c1) ? c0 : c1;
            }
        }
        bounds[j] = B[layer_node_lo[l_lo]];
    }
}

/* kernels.py:123-159 — distance from the root, push to the next layer. */
void oracle_k_forward(i64 nb, const i64 *bdd_layer_lo, const i64 *layer_node_lo,
                      const i64 *zero_t, const i64 *one_t, const double *lam,
                      double *F, double *bounds) {
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 j = 0; j < nb; ++j) {
        i64 l_lo = bdd_layer_lo[j], l_hi = bdd_layer_lo[j + 1];
        i64 root = layer_node_lo[l_lo];
        for (i64 v = root; v < layer_node_lo[l_lo + 1]; ++v) F[v] = INFINITY;
        F[root] = 0.0;
        double tb = INFINITY;
        for (i64 l = l_lo; l < l_hi; ++l) {
            if (l + 1 < l_hi)
                for (i64 w = layer_node_lo[l + 1]; w < layer_node_lo[l + 2]; ++w) F[w] = INFINITY;
            double lam_l = lam[l];
            for (i64 v = layer_node_lo[l]; v < layer_node_lo[l + 1]; ++v) {
                double fv = F[v];
                if (fv == INFINITY) continue;
                i64 a = zero_t[v];
                if (a >= 0) {
                    if (fv < F[a]) F[a] = fv;
                } else if (a == TGT_TRUE) {
                    if (fv < tb) tb = fv;
                }
                i64 b = one_t[v];
                double c = fv + lam_l;
                if (b >= 0) {
                    if (c < F[b]) F[b] = c;
                } else if (b == TGT_TRUE) {
                    if (c < tb) tb = c;
                }
            }
        }
        bounds[j] = tb;
    }
}

/* (m0, m1) of one layer from F (layer l) and B (targets). kernels.py:205-228 */
static inline void layer_min_marginals(i64 l, const i64 *layer_node_lo, const i64 *zero_t,
                                       const i64 *one_t, double lam_l, const double *F,
                                       const double *B, double *m0p, double *m1p) {
    double m0 = INFINITY, m1 = INFINITY;
    for (i64 v = layer_node_lo[l]; v < layer_node_lo[l + 1]; ++v) {
        double fv = F[v];
        if (fv == INFINITY) continue;
        i64 a = zero_t[v];
        double c0 = a == TGT_TRUE ? fv : (a == TGT_FALSE ? INFINITY : fv + B[a]);
        if (c0 < m0) m0 = c0;
        i64 b = one_t[v];
        double c1;
        if (b == TGT_TRUE) c1 = fv + lam_l;
        else if (b == TGT_FALSE) c1 = INFINITY;
        else { double t = fv + lam_l; c1 = t + B[b]; }
        if (c1 < m1) m1 = c1;
    }
    *m0p = m0;
    *m1p = m1;
}

/* Averaging step shared by both passes: kernels.py:199-240 / :297-339. */
static inline void average_variable(i64 lo, i64 hi, const i64 *proc_layers, double *lam,
                                    const double *m0s, const double *m1s) {
    double fsum = 0.0;
    i64 fcnt = 0;
    for (i64 t = lo; t < hi; ++t) {
        double m0 = m0s[t - lo], m1 = m1s[t - lo];
        if (m0 < INFINITY && m1 < INFINITY) {
            fsum += m1 - m0;
            fcnt += 1;
        }
    }
    if (fcnt > 0) {
        double avg = fsum / (double)fcnt;
        for (i64 t = lo; t < hi; ++t) {
            double m0 = m0s[t - lo], m1 = m1s[t - lo];
            if (m0 < INFINITY && m1 < INFINITY) lam[proc_layers[t]] += avg - (m1 - m0);
        }
    }
}

/* kernels.py:162-270 — sequential forward averaging pass. */
void oracle_k_mma_forward(i64 nb, i64 num_pos, const i64 *bdd_layer_lo, const i64 *layer_node_lo,
                          const i64 *layer_bdd, const i64 *zero_t, const i64 *one_t,
                          const i64 *proc_ptr, const i64 *proc_layers, double *lam, double *F,
                          const double *B, double *bounds, double *m0s, double *m1s) {
    for (i64 j = 0; j < nb; ++j) {
        i64 l_lo = bdd_layer_lo[j];
        i64 root = layer_node_lo[l_lo];
        for (i64 v = root; v < layer_node_lo[l_lo + 1]; ++v) F[v] = INFINITY;
        F[root] = 0.0;
        bounds[j] = INFINITY;
    }
    for (i64 p = 0; p < num_pos; ++p) {
        i64 lo = proc_ptr[p], hi = proc_ptr[p + 1];
        if (hi == lo) continue;
        for (i64 t = lo; t < hi; ++t) {
            i64 l = proc_layers[t];
            layer_min_marginals(l, layer_node_lo, zero_t, one_t, lam[l], F, B, &m0s[t - lo], &m1s[t - lo]);
        }
        average_variable(lo, hi, proc_layers, lam, m0s, m1s);
        for (i64 t = lo; t < hi; ++t) {
            i64 l = proc_layers[t];
            i64 j = layer_bdd[l];
            double lam_l = lam[l];
            int last = (l + 1 == bdd_layer_lo[j + 1]);
            if (!last)
                for (i64 w = layer_node_lo[l + 1]; w < layer_node_lo[l + 2]; ++w) F[w] = INFINITY;
            double tb = bounds[j];
            for (i64 v = layer_node_lo[l]; v < layer_node_lo[l + 1]; ++v) {
                double fv = F[v];
                if (fv == INFINITY) continue;
                i64 a = zero_t[v];
                if (a >= 0) {
                    if (fv < F[a]) F[a] = fv;
                } else if (a == TGT_TRUE) {
                    if (fv < tb) tb = fv;
                }
                i64 b = one_t[v];
                double c = fv + lam_l;
                if (b >= 0) {
                    if (c < F[b]) F[b] = c;
                } else if (b == TGT_TRUE) {
                    if (c < tb) tb = c;
                }
            }
            bounds[j] = tb;
        }
    }
}

/* kernels.py:273-362 — sequential backward averaging pass. */
void oracle_k_mma_backward(i64 nb, i64 num_pos, const i64 *bdd_layer_lo, const i64 *layer_node_lo,
                           const i64 *layer_bdd, const i64 *zero_t, const i64 *one_t,
                           const i64 *proc_ptr, const i64 *proc_layers, double *lam,
                           const double *F, double *B, double *bounds, double *m0s, double *m1s) {
    (void)layer_bdd;
    for (i64 p = num_pos - 1; p >= 0; --p) {
        i64 lo = proc_ptr[p], hi = proc_ptr[p + 1];
        if (hi == lo) continue;
        for (i64 t = lo; t < hi; ++t) {
            i64 l = proc_layers[t];
            layer_min_marginals(l, layer_node_lo, zero_t, one_t, lam[l], F, B, &m0s[t - lo], &m1s[t - lo]);
        }
        average_variable(lo, hi, proc_layers, lam, m0s, m1s);
        for (i64 t = lo; t < hi; ++t) {
            i64 l = proc_layers[t];
            double lam_l = lam[l];
            for (i64 v = layer_node_lo[l]; v < layer_node_lo[l + 1]; ++v) {
                i64 a = zero_t[v], b = one_t[v];
                double c0 = a == TGT_TRUE ? 0.0 : (a == TGT_FALSE ? INFINITY : B[a]);
                double c1 = b == TGT_TRUE ? lam_l : (b == TGT_FALSE ? INFINITY : lam_l + B[b]);
                B[v] = (c0 <= c1) ? c0 : c1;
            }
        }
    }
    for (i64 j = 0; j < nb; ++j) bounds[j] = B[layer_node_lo[bdd_layer_lo[j]]];
}

/* kernels.py:365-398 */
void oracle_k_min_marginals(i64 num_layers, const i64 *layer_node_lo, const i64 *zero_t,
                            const i64 *one_t, const double *lam, const double *F, const double *B,
                            double *m0_out, double *m1_out) {
#pragma omp parallel for schedule(static)
    for (i64 l = 0; l < num_layers; ++l)
        layer_min_marginals(l, layer_node_lo, zero_t, one_t, lam[l], F, B, &m0_out[l], &m1_out[l]);
}

/* kernels.py:401-431 */
void oracle_k_argmin(i64 nb, const i64 *bdd_layer_lo, const i64 *layer_node_lo,
                     const i64 *zero_t, const i64 *one_t, const double *lam, const double *B,
                     double *bits) {
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 j = 0; j < nb; ++j) {
        i64 v = layer_node_lo[bdd_layer_lo[j]];
        for (i64 l = bdd_layer_lo[j]; l < bdd_layer_lo[j + 1]; ++l) {
            i64 a = zero_t[v], b = one_t[v];
            double c0 = a == TGT_TRUE ? 0.0 : (a == TGT_FALSE ? INFINITY : B[a]);
            double c1 = b == TGT_TRUE ? lam[l] : (b == TGT_FALSE ? INFINITY : lam[l] + B[b]);
            i64 nxt;
            if (c0 <= c1) {
                bits[l] = 0.0;
                nxt = a;
            } else {
                bits[l] = 1.0;
                nxt = b;
            }
            if (nxt >= 0) v = nxt;
        }
    }
}

/*
 * bdd.py:362-475 — node tables of the reduced diagram of sum(c*x) == rhs.
 * Windowed partial-sum states, trimmed by exact forward reachability and
 * backward co-reachability, renumbered per layer in ascending sum order.
 * Outputs: widths[n] and flattened zero/one tables (local next-layer index,
 * -1 FALSE, -2 TRUE).  zero_out/one_out must hold the total node count,
 * which is bounded by sum over layers of the window width; the caller
 * queries it with zero_out == NULL first.  Returns the node count, or 0 when
 * the row has no 0-1 solution.
 */
i64 oracle_equality_tables(i64 n, const i64 *c, i64 rhs, i64 *widths, int32_t *zero_out,
                           int32_t *one_out) {
    i64 *minrem = calloc(n + 1, sizeof(i64)), *maxrem = calloc(n + 1, sizeof(i64));
    i64 *plo = calloc(n + 1, sizeof(i64)), *phi = calloc(n + 1, sizeof(i64));
    i64 *wlo = calloc(n + 1, sizeof(i64)), *whi = calloc(n + 1, sizeof(i64));
    i64 *off = calloc(n + 2, sizeof(i64));
    i64 result = 0;
    for (i64 l = n - 1; l >= 0; --l) {
        minrem[l] = minrem[l + 1] + (c[l] < 0 ? c[l] : 0);
        maxrem[l] = maxrem[l + 1] + (c[l] > 0 ? c[l] : 0);
    }
    for (i64 l = 0; l < n; ++l) {
        plo[l + 1] = plo[l] + (c[l] < 0 ? c[l] : 0);
        phi[l + 1] = phi[l] + (c[l] > 0 ? c[l] : 0);
    }
    for (i64 l = 0; l <= n; ++l) {
        i64 a = rhs - maxrem[l], b = rhs - minrem[l];
        wlo[l] = plo[l] > a ? plo[l] : a;
        whi[l] = phi[l] < b ? phi[l] : b;
        i64 w = whi[l] - wlo[l] + 1;
        off[l + 1] = off[l] + (w > 0 ? w : 0);
    }
    i64 total = off[n + 1];
    unsigned char *reach = NULL, *co = NULL;
    i64 *idx = NULL;
    if (total == 0) goto done;
    reach = calloc(total, 1);
    co = calloc(total, 1);
    idx = malloc(total * sizeof(i64));
    if (!(wlo[0] <= 0 && 0 <= whi[0])) goto done;
    reach[off[0] - wlo[0]] = 1;
    for (i64 l = 0; l < n; ++l)
        for (i64 s = wlo[l]; s <= whi[l]; ++s) {
            if (!reach[off[l] + s - wlo[l]]) continue;
            if (wlo[l + 1] <= s && s <= whi[l + 1]) reach[off[l + 1] + s - wlo[l + 1]] = 1;
            i64 s2 = s + c[l];
            if (wlo[l + 1] <= s2 && s2 <= whi[l + 1]) reach[off[l + 1] + s2 - wlo[l + 1]] = 1;
        }
    if (!(wlo[n] <= rhs && rhs <= whi[n])) goto done;
    co[off[n] + rhs - wlo[n]] = 1;
    for (i64 l = n - 1; l >= 0; --l)
        for (i64 s = wlo[l]; s <= whi[l]; ++s) {
            unsigned char ok = 0;
            if (wlo[l + 1] <= s && s <= whi[l + 1]) ok = co[off[l + 1] + s - wlo[l + 1]];
            if (!ok) {
                i64 s2 = s + c[l];
                if (wlo[l + 1] <= s2 && s2 <= whi[l + 1]) ok = co[off[l + 1] + s2 - wlo[l + 1]];
            }
            co[off[l] + s - wlo[l]] = ok;
        }
    i64 nodes = 0;
    for (i64 k = 0; k < total; ++k) idx[k] = -1;
    for (i64 l = 0; l < n; ++l) {
        i64 cnt = 0;
        for (i64 k = off[l]; k < off[l + 1]; ++k)
            if (reach[k] && co[k]) idx[k] = cnt++;
        widths[l] = cnt;
        nodes += cnt;
    }
    if (widths[0] == 0) goto done;
    result = nodes;
    if (!zero_out) goto done;
    {
        i64 pos = 0;
        for (i64 l = 0; l < n; ++l) {
            for (i64 s = wlo[l]; s <= whi[l]; ++s) {
                i64 i = idx[off[l] + s - wlo[l]];
                if (i < 0) continue;
                i64 at = pos + i;
                if (l == n - 1) {
                    zero_out[at] = s == rhs ? TGT_TRUE : TGT_FALSE;
                    one_out[at] = s + c[l] == rhs ? TGT_TRUE : TGT_FALSE;
                } else {
                    i64 t0 = TGT_FALSE, t1 = TGT_FALSE;
                    if (wlo[l + 1] <= s && s <= whi[l + 1]) {
                        t0 = idx[off[l + 1] + s - wlo[l + 1]];
                        if (t0 < 0) t0 = TGT_FALSE;
                    }
                    i64 s2 = s + c[l];
                    if (wlo[l + 1] <= s2 && s2 <= whi[l + 1]) {
                        t1 = idx[off[l + 1] + s2 - wlo[l + 1]];
                        if (t1 < 0) t1 = TGT_FALSE;
                    }
                    zero_out[at] = (int32_t)t0;
                    one_out[at] = (int32_t)t1;
                }
            }
            pos += widths[l];
        }
    }
done:
    free(minrem); free(maxrem); free(plo); free(phi); free(wlo); free(whi); free(off);
    free(reach); free(co); free(idx);
    return result;
}

/* ------------------------------------------------------------------------
 * Deferred (throughput) averaging schedule — restates the B200 path's
 * FastDOG-style parallel deferred min-marginal averaging
 * (paper_2310_08230_b200/csrc/dm_deferred.cu; the reference package has no
 * parallel MMA: kernels.py:162-362 is the sequential pass
 * and PAPER.md:4924 defer to FastDOG).  Per diagram, layer by layer, with
 * the reference's min-marginal and distance formulas (kernels.py:207-228,
 * 104-120, 142-159); per copy with finite m0, m1:
 *     lam' = (lam - omega*(m1-m0)) + avg[l],  mbar[l] = omega*(m1-m0)
 * else lam' = lam + avg[l], mbar[l] = +inf; avg == NULL: nothing added;
 * mbar == NULL: no min-marginal step.  F and B are in node order here.
 * ---------------------------------------------------------------------- */
static double dfr_update(double lam_l, const double *avg, i64 l, double m0, double m1, double omega,
                         double *mbar) {
    if (m0 < INFINITY && m1 < INFINITY) {
        double wm = omega * (m1 - m0);
        lam_l = lam_l - wm;
        if (avg) lam_l = lam_l + avg[l];
        mbar[l] = wm;
    } else {
        if (avg) lam_l = lam_l + avg[l];
        mbar[l] = INFINITY;
    }
    return lam_l;
}

static void dfr_marginals(i64 l, const i64 *lnl, const i64 *zero_t, const i64 *one_t, double lam_l,
                          const double *F, const double *B, double *m0o, double *m1o) {
    double m0 = INFINITY, m1 = INFINITY;
    for (i64 v = lnl[l]; v < lnl[l + 1]; ++v) {
        double fv = F[v];
        if (fv == INFINITY) continue;
        i64 a = zero_t[v], b = one_t[v];
        double c0 = a == TGT_TRUE ? fv : (a == TGT_FALSE ? INFINITY : fv + B[a]);
        if (c0 < m0) m0 = c0;
        double c1 = b == TGT_TRUE ? fv + lam_l : (b == TGT_FALSE ? INFINITY : (fv + lam_l) + B[b]);
        if (c1 < m1) m1 = c1;
    }
    *m0o = m0;
    *m1o = m1;
}

void oracle_dfr_forward(i64 nb, const i64 *bdd_layer_lo, const i64 *lnl, const i64 *zero_t, const i64 *one_t,
                        double omega, double *lam, const double *avg, const double *B, double *F, double *mbar,
                        double *bounds) {
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 j = 0; j < nb; ++j) {
        i64 l_lo = bdd_layer_lo[j], l_hi = bdd_layer_lo[j + 1];
        i64 root = lnl[l_lo];
        for (i64 v = root; v < lnl[l_lo + 1]; ++v) F[v] = INFINITY;
        F[root] = 0.0;
        double tb = INFINITY;
        for (i64 l = l_lo; l < l_hi; ++l) {
            double lam_l = lam[l];
            if (mbar) {
                double m0, m1;
                dfr_marginals(l, lnl, zero_t, one_t, lam_l, F, B, &m0, &m1);
                lam_l = dfr_update(lam_l, avg, l, m0, m1, omega, mbar);
            } else if (avg) {
                lam_l = lam_l + avg[l];
            }
            lam[l] = lam_l;
            if (l + 1 < l_hi)
                for (i64 w = lnl[l + 1]; w < lnl[l + 2]; ++w) F[w] = INFINITY;
            for (i64 v = lnl[l]; v < lnl[l + 1]; ++v) {
                double fv = F[v];
                if (fv == INFINITY) continue;
                i64 a = zero_t[v], b = one_t[v];
                if (a >= 0) {
                    if (fv < F[a]) F[a] = fv;
                } else if (a == TGT_TRUE) {
                    if (fv < tb) tb = fv;
                }
                double c = fv + lam_l;
                if (b >= 0) {
                    if (c < F[b]) F[b] = c;
                } else if (b == TGT_TRUE) {
                    if (c < tb) tb = c;
                }
            }
        }
        bounds[j] = tb;
    }
}

void oracle_dfr_backward(i64 nb, const i64 *bdd_layer_lo, const i64 *lnl, const i64 *zero_t, const i64 *one_t,
                         double omega, double *lam, const double *avg, const double *F, double *B, double *mbar,
                         double *bounds) {
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 j = 0; j < nb; ++j) {
        i64 l_lo = bdd_layer_lo[j], l_hi = bdd_layer_lo[j + 1];
        for (i64 l = l_hi - 1; l >= l_lo; --l) {
            double lam_l = lam[l];
            if (mbar) {
                double m0, m1;
                dfr_marginals(l, lnl, zero_t, one_t, lam_l, F, B, &m0, &m1);
                lam_l = dfr_update(lam_l, avg, l, m0, m1, omega, mbar);
            } else if (avg) {
                lam_l = lam_l + avg[l];
            }
            lam[l] = lam_l;
            for (i64 v = lnl[l]; v < lnl[l + 1]; ++v) {
                i64 a = zero_t[v], b = one_t[v];
                double c0 = a == TGT_TRUE ? 0.0 : (a == TGT_FALSE ? INFINITY : B[a]);
                double c1 = b == TGT_TRUE ? lam_l : (b == TGT_FALSE ? INFINITY : lam_l + B[b]);
                B[v] = (c0 <= c1) ? c0 : c1;
            }
        }
        bounds[j] = B[lnl[l_lo]];
    }
}

/* one pass's escrow -> next pass's per-copy average (copy order sums) */
void oracle_dfr_average(i64 P, const i64 *proc_ptr, const i64 *proc_layers, const double *mbar, double *avg) {
#pragma omp parallel for schedule(static)
    for (i64 p = 0; p < P; ++p) {
        double s = 0.0;
        i64 c = 0;
        for (i64 t = proc_ptr[p]; t < proc_ptr[p + 1]; ++t) {
            double x = mbar[proc_layers[t]];
            if (x != INFINITY) {
                s = s + x;
                ++c;
            }
        }
        double mean = c ? s / (double)c : 0.0;
        for (i64 t = proc_ptr[p]; t < proc_ptr[p + 1]; ++t) {
            i64 l = proc_layers[t];
            avg[l] = mbar[l] != INFINITY ? mean : 0.0;
        }
    }
}

/* Greedy row colouring of a product space's variables (product_space.py's
 * numbering of pruned spaces; the product computes it in dm_row_colouring):
 * variables in index order take the smallest colour that no variable of any
 * of their rows holds.  Lets the CPU arm build the same instance without the
 * product library.  Returns the number of colours, -1 on bad input. */
i64 oracle_row_colouring(i64 nv, i64 nrows, const i64 *row_ptr, const i64 *row_var, i64 *colour) {
    i64 *vptr = calloc((size_t)nv + 1, sizeof(i64));
    if (!vptr) return -1;
    for (i64 r = 0; r < nrows; ++r)
        for (i64 i = row_ptr[r]; i < row_ptr[r + 1]; ++i) {
            if (row_var[i] < 0 || row_var[i] >= nv) {
                free(vptr);
                return -1;
            }
            ++vptr[row_var[i] + 1];
        }
    for (i64 v = 0; v < nv; ++v) vptr[v + 1] += vptr[v];
    i64 *vrows = malloc((size_t)(vptr[nv] ? vptr[nv] : 1) * sizeof(i64));
    i64 *fill = malloc((size_t)(nv ? nv : 1) * sizeof(i64));
    for (i64 v = 0; v < nv; ++v) fill[v] = vptr[v];
    for (i64 r = 0; r < nrows; ++r)
        for (i64 i = row_ptr[r]; i < row_ptr[r + 1]; ++i) vrows[fill[row_var[i]]++] = r;
    /* a colour bound: one more than the largest number of row neighbours */
    i64 bound = 1;
    for (i64 v = 0; v < nv; ++v) {
        i64 d = 1;
        for (i64 k = vptr[v]; k < vptr[v + 1]; ++k) d += row_ptr[vrows[k] + 1] - row_ptr[vrows[k]] - 1;
        if (d > bound) bound = d;
    }
    const i64 words = bound / 64 + 1;
    uint64_t *used = calloc((size_t)(nrows ? nrows : 1) * (size_t)words, sizeof(uint64_t));
    uint64_t *taken = malloc((size_t)words * sizeof(uint64_t));
    i64 ncol = 0;
    for (i64 v = 0; v < nv; ++v) {
        for (i64 w = 0; w < words; ++w) taken[w] = 0;
        for (i64 k = vptr[v]; k < vptr[v + 1]; ++k) {
            const uint64_t *u = used + vrows[k] * words;
            for (i64 w = 0; w < words; ++w) taken[w] |= u[w];
        }
        i64 c = 0;
        while (taken[c >> 6] >> (c & 63) & 1) ++c;
        colour[v] = c;
        if (c + 1 > ncol) ncol = c + 1;
        for (i64 k = vptr[v]; k < vptr[v + 1]; ++k) used[vrows[k] * words + (c >> 6)] |= 1ull << (c & 63);
    }
    free(vptr);
    free(vrows);
    free(fill);
    free(used);
    free(taken);
    return ncol;
}
