/*
 * CPU ORACLE — test infrastructure only.
 *
 * A plain-C restatement of the reference's differentiable STA path
 * (/root/reference/pkg/src/stasim), used ONLY by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the checker.  The product package
 * (paper_2603_28381_b200/) never links, imports or executes anything here.
 *
 * Every function restates one reference routine statement for statement, in
 * the same floating-point operation order (compile with -ffp-contract=off, as
 * the reference does: pkg/setup.py:21-23), so the hard pass is bit-identical
 * with the reference's compiled backend.  numpy reduction orders are restated
 * too: np.add.reduceat(x, s) is x[s] + pairwise(x[s+1:e]) and ndarray.sum()
 * is pairwise(x) from 0.0 (numpy's pairwise_sum, unroll 8, block 128).
 * exp/log/log1p come from libm and may differ from numpy's SIMD versions by
 * an ulp; the gradient tolerance (1e-4 rel) covers that.
 *
 * Pinned against the reference: tests/test_oracle_golden.py checks these
 * functions against tests/golden/*.npz, produced by running the reference
 * itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* ------------------------------------------------------------------ */
/* flatten.py:176-298 — index maps                                     */

void orc_maps(i64 n_pins, i64 n_nets, const i64 *net_ptr, const i64 *net_root,
              const i64 *mem_pin, const i64 *mem_parent_pin,
              i64 *member_of_pin, i64 *root_net_of_pin, i64 *mem_parent_loc,
              i64 *mem_net, i64 *mem_local)
{
    for (i64 p = 0; p < n_pins; p++) { member_of_pin[p] = -1; root_net_of_pin[p] = -1; }
    for (i64 i = 0; i < n_nets; i++) {
        i64 s = net_ptr[i], e = net_ptr[i + 1];
        root_net_of_pin[net_root[i]] = i;
        for (i64 k = 0; k < e - s; k++) {
            i64 f = s + k, par = mem_parent_pin[f];
            /* local_of = {root: 0, member_k: k+1} (flatten.py:198-203) */
            i64 loc = -1;
            if (par == net_root[i]) loc = 0;
            for (i64 q = k - 1; q >= 0 && loc < 0; q--)
                if (mem_pin[s + q] == par) loc = q + 1;
            mem_parent_loc[f] = loc;
            mem_net[f] = i;
            mem_local[f] = k;
            member_of_pin[mem_pin[f]] = f;
        }
    }
}

/* stable grouping of ids 0..n-1 by key (key < 0 dropped), ascending id per
 * key: net_in (flatten.py:247-256) and mem_out (flatten.py:259-268) */
void orc_group(i64 n, const i64 *key, i64 n_keys, i64 *ptr, i64 *idx)
{
    memset(ptr, 0, sizeof(i64) * (size_t)(n_keys + 1));
    for (i64 a = 0; a < n; a++) if (key[a] >= 0) ptr[key[a] + 1]++;
    for (i64 k = 0; k < n_keys; k++) ptr[k + 1] += ptr[k];
    i64 *cur = (i64 *)malloc(sizeof(i64) * (size_t)(n_keys + 1));
    memcpy(cur, ptr, sizeof(i64) * (size_t)(n_keys + 1));
    for (i64 a = 0; a < n; a++) if (key[a] >= 0) idx[cur[key[a]]++] = a;
    free(cur);
}

/* levelize (flatten.py:44-80) over _net_deps (netlist.py:316-331).
 * Returns the number of levels, or -(1 + net) for the lowest-index net left
 * with unresolved dependencies (the CycleError pin is that net's root). */
i64 orc_levelize(i64 n_pins, i64 n_nets, const i64 *net_ptr, const i64 *net_root,
                 const i64 *mem_pin, i64 n_arcs, const i64 *arc_from, const i64 *arc_to,
                 i64 *level)
{
    i64 *member_of = (i64 *)malloc(sizeof(i64) * (size_t)(n_pins > 0 ? n_pins : 1));
    for (i64 p = 0; p < n_pins; p++) member_of[p] = -1;
    for (i64 i = 0; i < n_nets; i++)
        for (i64 f = net_ptr[i]; f < net_ptr[i + 1]; f++) member_of[mem_pin[f]] = i;
    /* arcs grouped by target pin, in arc order (src_of_target) */
    i64 *tptr = (i64 *)calloc((size_t)(n_pins + 1), sizeof(i64));
    i64 *tarc = (i64 *)malloc(sizeof(i64) * (size_t)(n_arcs > 0 ? n_arcs : 1));
    orc_group(n_arcs, arc_to, n_pins, tptr, tarc);
    /* deps as deduplicated lists */
    i64 *dptr = (i64 *)calloc((size_t)(n_nets + 1), sizeof(i64));
    i64 cap = n_arcs + n_nets + 1;
    i64 *dep = (i64 *)malloc(sizeof(i64) * (size_t)cap);
    i64 nd = 0;
    for (i64 j = 0; j < n_nets; j++) {
        i64 r = net_root[j];
        i64 s0 = nd;
        for (i64 t = tptr[r]; t < tptr[r + 1]; t++) {
            i64 src = arc_from[tarc[t]];
            i64 d = member_of[src];
            if (d < 0) continue;
            int seen = 0;
            for (i64 q = s0; q < nd; q++) if (dep[q] == d) { seen = 1; break; }
            if (!seen) dep[nd++] = d;
        }
        if (member_of[r] >= 0) {
            i64 d = member_of[r];
            int seen = 0;
            for (i64 q = s0; q < nd; q++) if (dep[q] == d) { seen = 1; break; }
            if (!seen) dep[nd++] = d;
        }
        dptr[j + 1] = nd;
    }
    /* consumers: reverse edges */
    i64 *indeg = (i64 *)malloc(sizeof(i64) * (size_t)(n_nets > 0 ? n_nets : 1));
    i64 *cptr = (i64 *)calloc((size_t)(n_nets + 1), sizeof(i64));
    i64 *cons = (i64 *)malloc(sizeof(i64) * (size_t)(nd > 0 ? nd : 1));
    for (i64 j = 0; j < n_nets; j++) {
        indeg[j] = dptr[j + 1] - dptr[j];
        for (i64 q = dptr[j]; q < dptr[j + 1]; q++) cptr[dep[q] + 1]++;
    }
    for (i64 i = 0; i < n_nets; i++) cptr[i + 1] += cptr[i];
    i64 *cc = (i64 *)malloc(sizeof(i64) * (size_t)(n_nets + 1));
    memcpy(cc, cptr, sizeof(i64) * (size_t)(n_nets + 1));
    for (i64 j = 0; j < n_nets; j++)
        for (i64 q = dptr[j]; q < dptr[j + 1]; q++) cons[cc[dep[q]]++] = j;
    /* Kahn, FIFO (flatten.py:62-73) */
    i64 *queue = (i64 *)malloc(sizeof(i64) * (size_t)(n_nets > 0 ? n_nets : 1));
    i64 qh = 0, qt = 0, done = 0;
    for (i64 i = 0; i < n_nets; i++) { level[i] = 0; if (indeg[i] == 0) queue[qt++] = i; }
    while (qh < qt) {
        i64 i = queue[qh++];
        done++;
        for (i64 q = cptr[i]; q < cptr[i + 1]; q++) {
            i64 j = cons[q];
            if (level[i] + 1 > level[j]) level[j] = level[i] + 1;
            if (--indeg[j] == 0) queue[qt++] = j;
        }
    }
    i64 ret;
    if (done != n_nets) {
        i64 stuck = 0;
        while (indeg[stuck] == 0) stuck++;
        ret = -(1 + stuck);
    } else {
        i64 mx = -1;
        for (i64 i = 0; i < n_nets; i++) if (level[i] > mx) mx = level[i];
        ret = mx + 1;
    }
    free(member_of); free(tptr); free(tarc); free(dptr); free(dep); free(indeg);
    free(cptr); free(cons); free(cc); free(queue);
    return ret;
}

/* ------------------------------------------------------------------ */
/* _kernels.pyx:15-81 — bilinear LUT interpolation                     */

static double interp(i64 lut, const i64 *s_ptr, const i64 *l_ptr, const i64 *t_ptr,
                     const double *s_flat, const double *l_flat, const double *t_flat,
                     double qs, double ql)
{
    i64 s0 = s_ptr[lut], nS = s_ptr[lut + 1] - s0;
    i64 l0 = l_ptr[lut], nL = l_ptr[lut + 1] - l0;
    i64 t0 = t_ptr[lut];
    i64 lo, hi, mid, si, li, si2, li2;
    double st, lt, v0, v1;
    if (nS > 1) {
        lo = 0; hi = nS;
        while (lo < hi) { mid = (lo + hi) / 2; if (s_flat[s0 + mid] <= qs) lo = mid + 1; else hi = mid; }
        si = lo - 1;
        if (si < 0) si = 0; else if (si > nS - 2) si = nS - 2;
        st = (qs - s_flat[s0 + si]) / (s_flat[s0 + si + 1] - s_flat[s0 + si]);
        if (st < 0.0) st = 0.0; else if (st > 1.0) st = 1.0;
        si2 = si + 1;
    } else { si = 0; st = 0.0; si2 = 0; }
    if (nL > 1) {
        lo = 0; hi = nL;
        while (lo < hi) { mid = (lo + hi) / 2; if (l_flat[l0 + mid] <= ql) lo = mid + 1; else hi = mid; }
        li = lo - 1;
        if (li < 0) li = 0; else if (li > nL - 2) li = nL - 2;
        lt = (ql - l_flat[l0 + li]) / (l_flat[l0 + li + 1] - l_flat[l0 + li]);
        if (lt < 0.0) lt = 0.0; else if (lt > 1.0) lt = 1.0;
        li2 = li + 1;
    } else { li = 0; lt = 0.0; li2 = 0; }
    v0 = (1.0 - lt) * t_flat[t0 + si * nL + li] + lt * t_flat[t0 + si * nL + li2];
    v1 = (1.0 - lt) * t_flat[t0 + si2 * nL + li] + lt * t_flat[t0 + si2 * nL + li2];
    return (1.0 - st) * v0 + st * v1;
}

double orc_interp(i64 lut, const i64 *s_ptr, const i64 *l_ptr, const i64 *t_ptr,
                  const double *s_flat, const double *l_flat, const double *t_flat,
                  double qs, double ql)
{
    return interp(lut, s_ptr, l_ptr, t_ptr, s_flat, l_flat, t_flat, qs, ql);
}

/* _kernels.pyx:84-156 — RC: loads, cumulative Elmore delays, impulses */
int orc_rc_level(i64 n_lv, const i64 *nets, const i64 *net_ptr, const i64 *net_root,
                 const double *root_cap, const i64 *mem_pin, const i64 *mem_parent_loc,
                 const double *mem_res, const double *mem_cap, const i64 *root_net_of_pin,
                 double *load, double *net_delay, double *impulse, int w)
{
    i64 max_m = 0;
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni];
        if (net_ptr[net + 1] - net_ptr[net] > max_m) max_m = net_ptr[net + 1] - net_ptr[net];
    }
    double *buf = (double *)malloc(sizeof(double) * (size_t)(max_m > 0 ? max_m : 1));
    double *dbuf = (double *)malloc(sizeof(double) * (size_t)(max_m > 0 ? max_m : 1));
    double *partials = (double *)malloc(sizeof(double) * (size_t)w);
    if (!buf || !dbuf || !partials) { free(buf); free(dbuf); free(partials); return -1; }
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni], s = net_ptr[net], e = net_ptr[net + 1], m = e - s, root = net_root[net];
        for (int c = 0; c < 4; c++) {
            for (i64 k = 0; k < m; k++) buf[k] = mem_cap[(s + k) * 4 + c];
            for (i64 k = m - 1; k > 0; k--) {
                i64 pl = mem_parent_loc[s + k];
                if (pl > 0) buf[pl - 1] += buf[k];
            }
            for (int lane = 0; lane < w; lane++) {
                double p = 0.0;
                for (i64 i = lane; i < m; i += w) p = p + buf[i];
                partials[lane] = p;
            }
            for (int stride = 1; stride < w; stride *= 2)
                for (int lane = 0; lane < w; lane += 2 * stride)
                    partials[lane] = partials[lane] + partials[lane + stride];
            load[root * 4 + c] = root_cap[net * 4 + c] + partials[0];
            for (i64 k = 0; k < m; k++) {
                i64 pl = mem_parent_loc[s + k];
                double dp = pl == 0 ? 0.0 : dbuf[pl - 1];
                double t = mem_res[(s + k) * 4 + c] * buf[k];
                dbuf[k] = dp + t;
            }
            for (i64 k = 0; k < m; k++) {
                double r = mem_res[(s + k) * 4 + c];
                double cp = mem_cap[(s + k) * 4 + c];
                double d = dbuf[k];
                double rad = 2.0 * r * cp * d - d * d;
                double imp = rad > 0.0 ? sqrt(rad) : 0.0;
                i64 pin = mem_pin[s + k];
                if (root_net_of_pin[pin] < 0) load[pin * 4 + c] = buf[k];
                net_delay[pin * 4 + c] = dbuf[k];
                impulse[pin * 4 + c] = imp;
            }
        }
    }
    free(buf); free(dbuf); free(partials);
    return 0;
}

/* _kernels.pyx:159-210 — arc merge (late max / early min, first arc wins),
 * winning-arc slew, then member arrival/slew */
void orc_forward_level(i64 n_lv, const i64 *nets, const i64 *net_ptr, const i64 *net_root,
                       const i64 *root_kind, const i64 *mem_pin, const i64 *net_in_ptr,
                       const i64 *net_in_arc, const i64 *arc_from, const i64 *arc_dlut,
                       const i64 *arc_slut, const i64 *s_ptr, const i64 *l_ptr, const i64 *t_ptr,
                       const double *s_flat, const double *l_flat, const double *t_flat,
                       const double *load, const double *net_delay, const double *impulse,
                       double *slew, double *arrival, double *arc_delay)
{
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni], root = net_root[net];
        if (root_kind[net] == 0) {
            for (int c = 0; c < 4; c++) {
                int late = c >= 2;
                double best = late ? -INFINITY : INFINITY;
                i64 wa = -1;
                double root_ld = load[root * 4 + c];
                for (i64 t = net_in_ptr[net]; t < net_in_ptr[net + 1]; t++) {
                    i64 a = net_in_arc[t], fp = arc_from[a];
                    double d = interp(arc_dlut[a * 4 + c], s_ptr, l_ptr, t_ptr, s_flat, l_flat,
                                      t_flat, slew[fp * 4 + c], root_ld);
                    arc_delay[a * 4 + c] = d;
                    double v = arrival[fp * 4 + c] + d;
                    if (late ? (v > best) : (v < best)) { best = v; wa = a; }
                }
                arrival[root * 4 + c] = best;
                slew[root * 4 + c] = interp(arc_slut[wa * 4 + c], s_ptr, l_ptr, t_ptr, s_flat,
                                            l_flat, t_flat, slew[arc_from[wa] * 4 + c], root_ld);
            }
        }
        for (i64 k = net_ptr[net]; k < net_ptr[net + 1]; k++) {
            i64 pin = mem_pin[k];
            for (int c = 0; c < 4; c++) {
                arrival[pin * 4 + c] = arrival[root * 4 + c] + net_delay[pin * 4 + c];
                double sr = slew[root * 4 + c], ii = impulse[pin * 4 + c];
                slew[pin * 4 + c] = sqrt(sr * sr + ii * ii);
            }
        }
    }
}

/* _kernels.pyx:213-249 — required times (late min / early max) */
void orc_backward_level(i64 n_lv, const i64 *nets, const i64 *net_ptr, const i64 *net_root,
                        const i64 *mem_pin, const i64 *mem_out_ptr, const i64 *mem_out_arc,
                        const i64 *arc_to, const double *net_delay, double *required,
                        const double *arc_delay)
{
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni], s = net_ptr[net], e = net_ptr[net + 1], root = net_root[net];
        for (i64 k = s; k < e; k++) {
            i64 pin = mem_pin[k];
            for (int c = 0; c < 4; c++) {
                int late = c >= 2;
                double r = required[pin * 4 + c];
                for (i64 t = mem_out_ptr[k]; t < mem_out_ptr[k + 1]; t++) {
                    i64 a = mem_out_arc[t];
                    double v = required[arc_to[a] * 4 + c] - arc_delay[a * 4 + c];
                    if (late ? (v < r) : (v > r)) r = v;
                }
                required[pin * 4 + c] = r;
            }
        }
        for (int c = 0; c < 4; c++) {
            int late = c >= 2;
            double r = required[root * 4 + c];
            for (i64 k = s; k < e; k++) {
                i64 pin = mem_pin[k];
                double v = required[pin * 4 + c] - net_delay[pin * 4 + c];
                if (late ? (v < r) : (v > r)) r = v;
            }
            required[root * 4 + c] = r;
        }
    }
}

/* ------------------------------------------------------------------ */
/* diff.py — LSE forward, endpoint loss, reverse gradients (late cols) */

/* numpy pairwise_sum (unroll 8, blocksize 128) over x[0..n) stride st */
static double pairwise(const double *x, i64 n, i64 st)
{
    if (n < 8) {
        double r = 0.0;
        for (i64 i = 0; i < n; i++) r += x[i * st];
        return r;
    } else if (n <= 128) {
        double r[8], res;
        i64 i;
        for (int j = 0; j < 8; j++) r[j] = x[j * st];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += x[(i + j) * st];
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += x[i * st];
        return res;
    } else {
        i64 n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise(x, n2, st) + pairwise(x + n2 * st, n - n2, st);
    }
}

double orc_pairwise(const double *x, i64 n) { return pairwise(x, n, 1); }

/* _lse_forward_level (diff.py:123-146).  lse_at (P,2), arc_d (A,2) late arc
 * delays, path (M,2) cumulative late net delays, weights (A,2) or NULL.
 * scratch must hold 2*max_in_arcs doubles. */
void orc_lse_level(i64 n_lv, const i64 *nets, const i64 *net_ptr, const i64 *net_root,
                   const i64 *root_kind, const i64 *mem_pin, const i64 *net_in_ptr,
                   const i64 *net_in_arc, const i64 *arc_from, double g, double *lse_at,
                   const double *arc_d, const double *path, double *weights, double *scratch)
{
    /* arcs of arc-driven nets, then members (all nets of the level), per j */
    for (int j = 0; j < 2; j++) {
        for (i64 ni = 0; ni < n_lv; ni++) {
            i64 net = nets[ni];
            if (root_kind[net] != 0) continue;
            i64 a0 = net_in_ptr[net], a1 = net_in_ptr[net + 1], cnt = a1 - a0;
            double *x = scratch, *z = scratch + cnt;
            double c = -INFINITY;
            for (i64 t = 0; t < cnt; t++) {
                i64 a = net_in_arc[a0 + t];
                x[t] = lse_at[arc_from[a] * 2 + j] + arc_d[a * 2 + j];
                if (t == 0 || x[t] > c) c = x[t];          /* np.maximum.reduceat */
            }
            for (i64 t = 0; t < cnt; t++) z[t] = exp((x[t] - c) / g);
            double s = z[0] + pairwise(z + 1, cnt - 1, 1);   /* np.add.reduceat */
            lse_at[net_root[net] * 2 + j] = c + g * log(s);
            if (weights)
                for (i64 t = 0; t < cnt; t++) weights[net_in_arc[a0 + t] * 2 + j] = z[t] / s;
        }
    }
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni], root = net_root[net];
        for (i64 k = net_ptr[net]; k < net_ptr[net + 1]; k++)
            for (int j = 0; j < 2; j++)
                lse_at[mem_pin[k] * 2 + j] = lse_at[root * 2 + j] + path[k * 2 + j];
    }
}

/* _endpoint_loss (diff.py:192-212): returns loss, fills adj (P,2) seeds
 * (adj must be zeroed by the caller).  kind 0 hinge, 1 softplus.
 * scratch holds 2*E doubles. */
double orc_endpoint_loss(i64 n_ep, const i64 *ep_pin, const double *ep_required,
                         const double *lse_at, double gamma, int kind, double *adj,
                         double *scratch)
{
    if (n_ep == 0) return 0.0;
    double *term = scratch;
    for (i64 e = 0; e < n_ep; e++)
        for (int j = 0; j < 2; j++) {
            double v = lse_at[ep_pin[e] * 2 + j] - ep_required[e * 4 + 2 + j];
            double mx = v > 0.0 ? v : 0.0;   /* np.maximum(v, 0.0) */
            if (v != v) mx = v;
            if (kind == 0) term[e * 2 + j] = mx;
            else term[e * 2 + j] = mx + gamma * log1p(exp(-fabs(v) / gamma));
        }
    double loss = pairwise(term, 2 * n_ep, 1);
    for (int j = 0; j < 2; j++)
        for (i64 e = 0; e < n_ep; e++) {
            double v = lse_at[ep_pin[e] * 2 + j] - ep_required[e * 4 + 2 + j];
            double gg = kind == 0 ? (v > 0.0 ? 1.0 : 0.0) : 1.0 / (1.0 + exp(-v / gamma));
            adj[ep_pin[e] * 2 + j] += gg;
        }
    return loss;
}

/* _grad_backward_level (diff.py:215-241) */
void orc_grad_level(i64 n_lv, const i64 *nets, const i64 *net_ptr, const i64 *net_root,
                    const i64 *root_kind, const i64 *mem_pin, const i64 *mem_parent_loc,
                    const i64 *net_in_ptr, const i64 *net_in_arc, const i64 *arc_from,
                    double *adj, double *d_arc, double *d_edge, const double *arc_weights)
{
    /* d_edge[mem] = adj[mem_pin] for the whole level first */
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni];
        for (i64 k = net_ptr[net]; k < net_ptr[net + 1]; k++)
            for (int j = 0; j < 2; j++) d_edge[k * 2 + j] = adj[mem_pin[k] * 2 + j];
    }
    /* fold deepest position first; nets never share a target within one
     * position group, so the per-net descending loop is the same order */
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni], s = net_ptr[net], e = net_ptr[net + 1], root = net_root[net];
        for (i64 k = e - 1; k >= s; k--) {
            i64 pl = mem_parent_loc[k];
            for (int j = 0; j < 2; j++) {
                if (pl > 0) d_edge[(s + pl - 1) * 2 + j] += d_edge[k * 2 + j];
                else adj[root * 2 + j] += d_edge[k * 2 + j];
            }
        }
    }
    for (int j = 0; j < 2; j++)
        for (i64 ni = 0; ni < n_lv; ni++) {
            i64 net = nets[ni];
            if (root_kind[net] != 0) continue;
            double ar = adj[net_root[net] * 2 + j];
            for (i64 t = net_in_ptr[net]; t < net_in_ptr[net + 1]; t++) {
                i64 a = net_in_arc[t];
                double contrib = ar * arc_weights[a * 2 + j];
                d_arc[a * 2 + j] = contrib;
                adj[arc_from[a] * 2 + j] += contrib;
            }
        }
}

/* ------------------------------------------------------------------ */
/* Position model and position gradients (north_star: "gradients w.r.t.
 * pin/cell positions").  The reference stops at
 * delay-space gradients (diff.py:5-7; SPEC.md "Non-goals: pin-location
 * gradients"), so this part has no reference routine to restate: it is the
 * exact reverse-mode derivative of the reference's own forward functions
 * (rc_level _kernels.pyx:84-156, _interp :15-81, forward_level :159-210,
 * _lse_forward_level diff.py:123-146) composed with a Manhattan wire model,
 * and it is pinned by central finite differences of the reference-restated
 * loss (tests/test_place_oracle.py) — "parity pinned by FD", not by golden
 * vectors.
 *
 * Wire model: member k of a net, parent pin q (the root for depth 0, else
 * its parent member), length l_k = |x_k - x_q| + |y_k - y_q|;
 *   mem_res[k,c] = res0[k,c] + r_unit[c] * l_k
 *   mem_cap[k,c] = cap0[k,c] + c_unit[c] * l_k                               */

void orc_wire(i64 M, const i64 *mem_pin, const i64 *parent_pin, const double *xy,
              const double *res0, const double *cap0, const double *ru, const double *cu,
              double *res, double *cap)
{
    for (i64 k = 0; k < M; k++) {
        i64 p = mem_pin[k], q = parent_pin[k];
        double l = fabs(xy[p * 2] - xy[q * 2]) + fabs(xy[p * 2 + 1] - xy[q * 2 + 1]);
        for (int c = 0; c < 4; c++) {
            res[k * 4 + c] = res0[k * 4 + c] + ru[c] * l;
            cap[k * 4 + c] = cap0[k * 4 + c] + cu[c] * l;
        }
    }
}

/* d out / d qs and d out / d ql of _interp (_kernels.pyx:15-81): the partial
 * derivatives of the bilinear form inside the located cell; 0 along an axis
 * whose fraction was clamped (query outside the table) or with one point. */
static void interp_grad(i64 lut, const i64 *s_ptr, const i64 *l_ptr, const i64 *t_ptr,
                        const double *s_flat, const double *l_flat, const double *t_flat,
                        double qs, double ql, double *ds, double *dl)
{
    i64 s0 = s_ptr[lut], nS = s_ptr[lut + 1] - s0;
    i64 l0 = l_ptr[lut], nL = l_ptr[lut + 1] - l0;
    i64 t0 = t_ptr[lut];
    i64 lo, hi, mid, si, li, si2, li2;
    double st, lt, hs = 0.0, hl = 0.0;
    int fs = 0, fl = 0;
    if (nS > 1) {
        lo = 0; hi = nS;
        while (lo < hi) { mid = (lo + hi) / 2; if (s_flat[s0 + mid] <= qs) lo = mid + 1; else hi = mid; }
        si = lo - 1;
        if (si < 0) si = 0; else if (si > nS - 2) si = nS - 2;
        hs = s_flat[s0 + si + 1] - s_flat[s0 + si];
        st = (qs - s_flat[s0 + si]) / hs;
        if (st < 0.0) st = 0.0; else if (st > 1.0) st = 1.0; else fs = 1;
        si2 = si + 1;
    } else { si = 0; st = 0.0; si2 = 0; }
    if (nL > 1) {
        lo = 0; hi = nL;
        while (lo < hi) { mid = (lo + hi) / 2; if (l_flat[l0 + mid] <= ql) lo = mid + 1; else hi = mid; }
        li = lo - 1;
        if (li < 0) li = 0; else if (li > nL - 2) li = nL - 2;
        hl = l_flat[l0 + li + 1] - l_flat[l0 + li];
        lt = (ql - l_flat[l0 + li]) / hl;
        if (lt < 0.0) lt = 0.0; else if (lt > 1.0) lt = 1.0; else fl = 1;
        li2 = li + 1;
    } else { li = 0; lt = 0.0; li2 = 0; }
    double t00 = t_flat[t0 + si * nL + li], t01 = t_flat[t0 + si * nL + li2];
    double t10 = t_flat[t0 + si2 * nL + li], t11 = t_flat[t0 + si2 * nL + li2];
    double v0 = (1.0 - lt) * t00 + lt * t01;
    double v1 = (1.0 - lt) * t10 + lt * t11;
    *ds = fs ? (v1 - v0) / hs : 0.0;
    *dl = fl ? ((1.0 - st) * (t01 - t00) + st * (t11 - t10)) / hl : 0.0;
}

void orc_interp_grad(i64 lut, const i64 *s_ptr, const i64 *l_ptr, const i64 *t_ptr,
                     const double *s_flat, const double *l_flat, const double *t_flat,
                     double qs, double ql, double *out2)
{
    interp_grad(lut, s_ptr, l_ptr, t_ptr, s_flat, l_flat, t_flat, qs, ql, out2, out2 + 1);
}

/* One level of the reverse sweep (levels descending), late conditions only
 * (the loss sees only lse_arrival, diff.py:21).  With adj = dL/dlse_at (the
 * GradientState adjoint) and d_arc = dL/darc_delay:
 *   gs[p]   = dL/dslew[p]  = sum over out-arcs a of gsa[a]
 *                            (+ gsr[p] when p roots a feedthrough net)
 *   gsa[a]  = d_arc[a] dD_a/dslew + [a wins its root] gs[root] dS_a/dslew
 *   gsr[r]  = sum over members m of gs[m] slew[r] / slew[m]   (slew = sqrt(sr^2 + imp^2))
 *   gl[n]   = dL/dload[root] = sum_a d_arc[a] dD_a/dload + gs[root] dS_w/dload
 * then the Elmore adjoint of the net (rc_level order: buf = downstream caps,
 * d = cumulative delay, imp = sqrt(2 r cap d - d^2)):
 *   A_k = adj[m_k] + gimp_k (r_k cap_k - d_k) / imp_k,  gimp_k = gs[m_k] imp_k / slew[m_k]
 *   D_k = A_k + sum over children D_child
 *   d_res[k] = D_k buf_k + gimp_k cap_k d_k / imp_k
 *   B_k = D_k r_k + gl[n] + B_parent(k)      (load[root] = root_cap + sum_k buf_k)
 *   d_cap[k] = B_k + gimp_k r_k d_k / imp_k,  d_root_cap[n] = gl[n]
 * scratch: 3 * max members doubles. */
void orc_posgrad_level(i64 n_lv, const i64 *nets, const i64 *net_ptr, const i64 *net_root,
                       const i64 *root_kind, const i64 *mem_pin, const i64 *mem_parent_loc,
                       const i64 *net_in_ptr, const i64 *net_in_arc, const i64 *arc_from,
                       const i64 *arc_dlut, const i64 *arc_slut, const i64 *pin_out_ptr,
                       const i64 *pin_out_arc, const i64 *root_net_of_pin,
                       const i64 *s_ptr, const i64 *l_ptr, const i64 *t_ptr,
                       const double *s_flat, const double *l_flat, const double *t_flat,
                       const double *mem_res, const double *mem_cap, const double *load,
                       const double *net_delay, const double *impulse, const double *slew,
                       const double *arrival, const double *arc_delay, const double *adj,
                       const double *d_arc, double *gs, double *gsr, double *gsa, double *gl_out,
                       double *d_res, double *d_cap, double *d_root_cap, double *scratch)
{
    for (i64 ni = 0; ni < n_lv; ni++) {
        i64 net = nets[ni], s = net_ptr[net], e = net_ptr[net + 1], m = e - s, root = net_root[net];
        double *gimp = scratch, *buf = scratch + m, *acc = scratch + 2 * m;
        for (int j = 0; j < 2; j++) {
            int c = 2 + j;
            double sr = slew[root * 4 + c], gsum = 0.0, gl = 0.0;
            for (i64 k = s; k < e; k++) {
                i64 pin = mem_pin[k];
                double g = 0.0;
                for (i64 t = pin_out_ptr[pin]; t < pin_out_ptr[pin + 1]; t++)
                    g += gsa[pin_out_arc[t] * 2 + j];
                if (root_net_of_pin[pin] >= 0) g += gsr[pin * 2 + j];
                gs[pin * 2 + j] = g;
                double sm = slew[pin * 4 + c];
                if (sm > 0.0) {
                    gsum += g * (sr / sm);
                    gimp[k - s] = g * (impulse[pin * 4 + c] / sm);
                } else {
                    gimp[k - s] = 0.0;
                }
            }
            if (root_kind[net] == 2) {
                gsr[root * 2 + j] = gsum;          /* the parent net's member loop adds it */
            } else {
                double groot = gsum;
                for (i64 t = pin_out_ptr[root]; t < pin_out_ptr[root + 1]; t++)
                    groot += gsa[pin_out_arc[t] * 2 + j];
                gs[root * 2 + j] = groot;
                if (root_kind[net] == 0) {
                    double ld = load[root * 4 + c], best = -INFINITY;
                    i64 w = -1;
                    for (i64 t = net_in_ptr[net]; t < net_in_ptr[net + 1]; t++) {
                        i64 a = net_in_arc[t];
                        double v = arrival[arc_from[a] * 4 + c] + arc_delay[a * 4 + c];
                        if (v > best) { best = v; w = a; }
                    }
                    for (i64 t = net_in_ptr[net]; t < net_in_ptr[net + 1]; t++) {
                        i64 a = net_in_arc[t];
                        double ds, dl;
                        interp_grad(arc_dlut[a * 4 + c], s_ptr, l_ptr, t_ptr, s_flat, l_flat, t_flat,
                                    slew[arc_from[a] * 4 + c], ld, &ds, &dl);
                        gsa[a * 2 + j] = d_arc[a * 2 + j] * ds;
                        gl += d_arc[a * 2 + j] * dl;
                    }
                    if (w >= 0) {
                        double ds, dl;
                        interp_grad(arc_slut[w * 4 + c], s_ptr, l_ptr, t_ptr, s_flat, l_flat, t_flat,
                                    slew[arc_from[w] * 4 + c], ld, &ds, &dl);
                        gsa[w * 2 + j] += groot * ds;
                        gl += groot * dl;
                    }
                }
            }
            gl_out[net * 2 + j] = gl;
            d_root_cap[net * 2 + j] = gl;
            /* Elmore adjoint */
            for (i64 k = 0; k < m; k++) buf[k] = mem_cap[(s + k) * 4 + c];
            for (i64 k = m - 1; k > 0; k--) {
                i64 pl = mem_parent_loc[s + k];
                if (pl > 0) buf[pl - 1] += buf[k];
            }
            for (i64 k = 0; k < m; k++) {
                i64 pin = mem_pin[s + k];
                double r = mem_res[(s + k) * 4 + c], cp = mem_cap[(s + k) * 4 + c];
                double d = net_delay[pin * 4 + c], im = impulse[pin * 4 + c];
                acc[k] = adj[pin * 2 + j];
                if (im > 0.0) acc[k] += gimp[k] * ((r * cp - d) / im);
            }
            for (i64 k = m - 1; k > 0; k--) {
                i64 pl = mem_parent_loc[s + k];
                if (pl > 0) acc[pl - 1] += acc[k];
            }
            for (i64 k = 0; k < m; k++) {
                i64 pin = mem_pin[s + k];
                double r = mem_res[(s + k) * 4 + c], cp = mem_cap[(s + k) * 4 + c];
                double d = net_delay[pin * 4 + c], im = impulse[pin * 4 + c];
                double dr = acc[k] * buf[k];
                if (im > 0.0) dr += gimp[k] * ((cp * d) / im);
                d_res[(s + k) * 2 + j] = dr;
                acc[k] = acc[k] * r + gl;          /* acc now holds B_k (direct part) */
            }
            for (i64 k = 1; k < m; k++) {
                i64 pl = mem_parent_loc[s + k];
                if (pl > 0) acc[k] += acc[pl - 1];
            }
            for (i64 k = 0; k < m; k++) {
                i64 pin = mem_pin[s + k];
                double r = mem_res[(s + k) * 4 + c];
                double d = net_delay[pin * 4 + c], im = impulse[pin * 4 + c];
                double dc = acc[k];
                if (im > 0.0) dc += gimp[k] * ((r * d) / im);
                d_cap[(s + k) * 2 + j] = dc;
            }
        }
    }
}

/* dL/dl_k = sum_j d_res[k,j] r_unit[2+j] + d_cap[k,j] c_unit[2+j], then
 * dL/dx: +dL/dl_k sign(x_k - x_q) on the member pin, minus it on the parent
 * pin q (sign(0) = 0); y likewise.  dxy (P,2) must be zeroed. */
void orc_pos_reduce(i64 M, const i64 *mem_pin, const i64 *parent_pin, const double *xy,
                    const double *ru, const double *cu, const double *d_res, const double *d_cap,
                    double *g_len, double *dxy)
{
    for (i64 k = 0; k < M; k++) {
        double g = 0.0;
        for (int j = 0; j < 2; j++) g += d_res[k * 2 + j] * ru[2 + j] + d_cap[k * 2 + j] * cu[2 + j];
        g_len[k] = g;
        i64 p = mem_pin[k], q = parent_pin[k];
        for (int a = 0; a < 2; a++) {
            double dd = xy[p * 2 + a] - xy[q * 2 + a];
            double sg = dd > 0.0 ? 1.0 : (dd < 0.0 ? -1.0 : 0.0);
            dxy[p * 2 + a] += g * sg;
            dxy[q * 2 + a] -= g * sg;
        }
    }
}
