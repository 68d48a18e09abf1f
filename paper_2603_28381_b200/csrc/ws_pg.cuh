// Position-gradient sweep bodies shared by the stand-alone sweep kernels
// (ws_place.cu: k_pg_mem / k_pg_level, used by the sequential and two-stream
// modes) and the fused backward level kernel (ws_pass.cu: k_bwd<..., PG>,
// the fused mode), so both paths run the same arithmetic in the same order.
//
// The math is oracle/sta_oracle.c's orc_posgrad_level (see ws_place.cu's
// header): per reverse level, the slew adjoint of every member from its
// out-arcs and the feedthrough net it roots, the impulse adjoint, the
// root-slew terms, the LUT partials of the in-arcs of every net (bilinear
// cell derivatives of _interp, _kernels.pyx:15-81), dL/dload and the Elmore
// adjoint -> d_res / d_cap / d_root_cap.  Only late columns (j = 0, 1 ->
// cond 2 + j) reach the loss.  Pass state written by other thread blocks is
// read through L2 (ld.global.cg).
#pragma once
#include "ws_internal.h"

namespace ws {
namespace {
namespace pg {

constexpr double PG_INF = __builtin_huge_val();

// the located cell of a query on an n > 1 point axis: upper_bound - 1
// clamped to [0, n - 2] (_kernels.pyx:15-81), by lut_locate's three
// branch-free halving steps for n <= 8
__device__ __forceinline__ int axis_cell(const double* ax, int n, double q)
{
    int lo;
    if (n <= 8) {
        lo = 0;
#pragma unroll
        for (int s = 4; s >= 1; s >>= 1)
            if (lo + s <= n && ax[lo + s - 1] <= q) lo += s;
    } else {
        lo = upper_bound_long(ax, n, q);
    }
    int i = lo - 1;
    if (i < 0) i = 0; else if (i > n - 2) i = n - 2;
    return i;
}

// d out / d qs and d out / d ql of _interp (_kernels.pyx:15-81) inside the
// located cell; 0 along an axis whose fraction was clamped (orc interp_grad)
__device__ __forceinline__ void interp_grad(const LutView& L, int lut, double qs, double ql, double& ds,
                                            double& dl)
{
    const int s0 = L.s_ptr[lut], nS = L.s_ptr[lut + 1] - s0;
    const int l0 = L.l_ptr[lut], nL = L.l_ptr[lut + 1] - l0;
    const int t0 = L.t_ptr[lut];
    int si, li, si2, li2;
    double st, lt, hs = 0.0, hl = 0.0;
    bool fs = false, fl = false;
    if (nS > 1) {
        si = axis_cell(L.s + s0, nS, qs);
        hs = __dsub_rn(L.s[s0 + si + 1], L.s[s0 + si]);
        st = __ddiv_rn(__dsub_rn(qs, L.s[s0 + si]), hs);
        if (st < 0.0) st = 0.0; else if (st > 1.0) st = 1.0; else fs = true;
        si2 = si + 1;
    } else { si = 0; st = 0.0; si2 = 0; }
    if (nL > 1) {
        li = axis_cell(L.l + l0, nL, ql);
        hl = __dsub_rn(L.l[l0 + li + 1], L.l[l0 + li]);
        lt = __ddiv_rn(__dsub_rn(ql, L.l[l0 + li]), hl);
        if (lt < 0.0) lt = 0.0; else if (lt > 1.0) lt = 1.0; else fl = true;
        li2 = li + 1;
    } else { li = 0; lt = 0.0; li2 = 0; }
    const double t00 = L.t[t0 + si * nL + li], t01 = L.t[t0 + si * nL + li2];
    const double t10 = L.t[t0 + si2 * nL + li], t11 = L.t[t0 + si2 * nL + li2];
    const double v0 = __dadd_rn(__dmul_rn(__dsub_rn(1.0, lt), t00), __dmul_rn(lt, t01));
    const double v1 = __dadd_rn(__dmul_rn(__dsub_rn(1.0, lt), t10), __dmul_rn(lt, t11));
    ds = fs ? __ddiv_rn(__dsub_rn(v1, v0), hs) : 0.0;
    dl = fl ? __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(1.0, st), __dsub_rn(t01, t00)),
                                  __dmul_rn(st, __dsub_rn(t11, t10))), hl)
            : 0.0;
}

// RC-tree net: the oracle's sequential Elmore adjoint recursion (one lane)
__device__ void pg_tree_net(const Topo& t, const Corner& C, const PlaceCorner& G, int s, int m, int j,
                            double gl)
{
    const int c = 2 + j;
    double* gimp = G.sc_gimp + (size_t)s * 2 + j;
    double* buf = G.sc_buf + (size_t)s * 2 + j;
    double* acc = G.sc_acc + (size_t)s * 2 + j;
    for (int k = 0; k < m; k++) buf[2 * k] = __ldcg(C.mem_cap + (size_t)(s + k) * 4 + c);
    for (int k = m - 1; k > 0; k--) {
        const int pl = t.mem_parent_loc[s + k];
        if (pl > 0) buf[2 * (pl - 1)] = __dadd_rn(buf[2 * (pl - 1)], buf[2 * k]);
    }
    for (int k = 0; k < m; k++) {
        const int pin = t.mem_pin[s + k];
        const double r = __ldcg(C.mem_res + (size_t)(s + k) * 4 + c);
        const double cp = __ldcg(C.mem_cap + (size_t)(s + k) * 4 + c);
        const double d = __ldcg(C.net_delay + (size_t)pin * 4 + c), im = __ldcg(C.impulse + (size_t)pin * 4 + c);
        double a = __ldcg(C.adjoint + (size_t)pin * 2 + j);
        if (im > 0.0) a = __dadd_rn(a, __dmul_rn(__ldcg(gimp + 2 * k), __ddiv_rn(__dsub_rn(__dmul_rn(r, cp), d), im)));
        acc[2 * k] = a;
    }
    for (int k = m - 1; k > 0; k--) {
        const int pl = t.mem_parent_loc[s + k];
        if (pl > 0) acc[2 * (pl - 1)] = __dadd_rn(acc[2 * (pl - 1)], acc[2 * k]);
    }
    for (int k = 0; k < m; k++) {
        const int pin = t.mem_pin[s + k];
        const double r = __ldcg(C.mem_res + (size_t)(s + k) * 4 + c);
        const double cp = __ldcg(C.mem_cap + (size_t)(s + k) * 4 + c);
        const double d = __ldcg(C.net_delay + (size_t)pin * 4 + c), im = __ldcg(C.impulse + (size_t)pin * 4 + c);
        double dr = __dmul_rn(acc[2 * k], buf[2 * k]);
        if (im > 0.0) dr = __dadd_rn(dr, __dmul_rn(__ldcg(gimp + 2 * k), __ddiv_rn(__dmul_rn(cp, d), im)));
        G.d_res[(size_t)(s + k) * 2 + j] = dr;
        acc[2 * k] = __dadd_rn(__dmul_rn(acc[2 * k], r), gl);
    }
    for (int k = 1; k < m; k++) {
        const int pl = t.mem_parent_loc[s + k];
        if (pl > 0) acc[2 * k] = __dadd_rn(acc[2 * k], acc[2 * (pl - 1)]);
    }
    for (int k = 0; k < m; k++) {
        const int pin = t.mem_pin[s + k];
        const double r = __ldcg(C.mem_res + (size_t)(s + k) * 4 + c);
        const double d = __ldcg(C.net_delay + (size_t)pin * 4 + c), im = __ldcg(C.impulse + (size_t)pin * 4 + c);
        double dc = acc[2 * k];
        if (im > 0.0) dc = __dadd_rn(dc, __dmul_rn(__ldcg(gimp + 2 * k), __ddiv_rn(__dmul_rn(r, d), im)));
        G.d_cap[(size_t)(s + k) * 2 + j] = dc;
    }
}

// one member term, (task-order member slot u, late column j): the pass-state
// loads (static once the member's backward level ran) ...
struct MemberIn {
    int pin, o1, fl, f;
    bool tree;
    double sm, im, sr, rr, cp, d, adj;
    double gsa1, gsr;   // gsa of the first out-arc, gsr of the pin (read after the wait)
};

__device__ __forceinline__ MemberIn member_load(const Topo& t, const PgDev& pd, const Corner& C, int u, int j)
{
    const int c = 2 + j;
    MemberIn r;
    r.pin = t.tm_pin[u];
    r.o1 = t.tm_o1_arc[u];
    r.fl = t.tm_flags[u];
    r.f = pd.tm_f[u];
    const int root = pd.tm_root[u];
    r.tree = t.net_tree[t.mem_net[r.f]] != 0;
    r.sm = __ldcg(C.slew + (size_t)r.pin * 4 + c);
    r.im = __ldcg(C.impulse + (size_t)r.pin * 4 + c);
    r.sr = __ldcg(C.slew + (size_t)root * 4 + c);
    r.rr = __ldcg(C.mem_res + (size_t)r.f * 4 + c);
    r.cp = __ldcg(C.mem_cap + (size_t)r.f * 4 + c);
    r.d = __ldcg(C.net_delay + (size_t)r.pin * 4 + c);
    r.adj = __ldcg(C.adjoint + (size_t)r.pin * 2 + j);
    return r;
}

// the sweep-dynamic reads of a member (higher levels' gsa / gsr)
__device__ __forceinline__ void member_load_dyn(const PlaceCorner& G, int j, MemberIn& r)
{
    r.gsa1 = r.o1 >= 0 ? __ldcg(G.gsa + (size_t)r.o1 * 2 + j) : 0.0;
    r.gsr = (r.fl & TM_ROOT) ? __ldcg(G.gsr + (size_t)r.pin * 2 + j) : 0.0;
}

// ... and its terms once the higher levels' gsa / gsr are final: slew
// adjoint g (out-arcs' gsa + the fed net's gsr), the root-slew term
// g * (sr / sm), the impulse adjoint, and on star nets the Elmore adjoint up
// to the dL/dload term: A = adj + gimp (r cap - d) / imp,
// d_res = A cap + gimp cap d / imp, x = A r, y = gimp r d / imp
// (d_cap = (x + gl) + y, pg_net_group)
// Where a level's member terms live between the member step and the net
// step: the root-slew term t and (star nets) the Elmore pieces x, y.  The
// stand-alone sweep and chunked / looped tasks keep them in the global
// scratch (original member index f); the fused kernel keeps a task's terms
// in shared memory (task member slot mi).
struct TermsGlobal {
    const PlaceCorner* G;
    __device__ __forceinline__ void put_t(int f, int, int j, double v) const { G->sc_t[(size_t)f * 2 + j] = v; }
    __device__ __forceinline__ void put_xy(int f, int, int j, double x, double y) const
    {
        G->sc_buf[(size_t)f * 2 + j] = x;
        G->sc_acc[(size_t)f * 2 + j] = y;
    }
    __device__ __forceinline__ double t(int f, int, int j) const { return __ldcg(G->sc_t + (size_t)f * 2 + j); }
    __device__ __forceinline__ double x(int f, int, int j) const { return __ldcg(G->sc_buf + (size_t)f * 2 + j); }
    __device__ __forceinline__ double y(int f, int, int j) const { return __ldcg(G->sc_acc + (size_t)f * 2 + j); }
};

struct TermsSmem {
    double *st, *sx, *sy;   // [TASK_M * 2] each
    __device__ __forceinline__ void put_t(int, int mi, int j, double v) const { st[mi * 2 + j] = v; }
    __device__ __forceinline__ void put_xy(int, int mi, int j, double x, double y) const
    {
        sx[mi * 2 + j] = x;
        sy[mi * 2 + j] = y;
    }
    __device__ __forceinline__ double t(int, int mi, int j) const { return st[mi * 2 + j]; }
    __device__ __forceinline__ double x(int, int mi, int j) const { return sx[mi * 2 + j]; }
    __device__ __forceinline__ double y(int, int mi, int j) const { return sy[mi * 2 + j]; }
};

template <class Terms>
__device__ __forceinline__ void member_finish(const Topo& t, const PlaceCorner& G, int u, int j,
                                              const MemberIn& m, int mi, const Terms& out)
{
    double g = 0.0;
    if (m.o1 >= 0) {
        g = __dadd_rn(g, m.gsa1);
        for (int v = t.tm_optr[u] + 1; v < t.tm_optr[u + 1]; v++)
            g = __dadd_rn(g, __ldcg(G.gsa + (size_t)t.to_arc[v] * 2 + j));
    }
    if (m.fl & TM_ROOT) g = __dadd_rn(g, m.gsr);
    G.gs[(size_t)m.pin * 2 + j] = g;
    double gi = 0.0, tk = 0.0;
    if (m.sm > 0.0) {
        tk = __dmul_rn(g, __ddiv_rn(m.sr, m.sm));
        gi = __dmul_rn(g, __ddiv_rn(m.im, m.sm));
    }
    const size_t fj = (size_t)m.f * 2 + j;
    out.put_t(m.f, mi, j, tk);
    if (m.tree) {
        G.sc_gimp[fj] = gi;
        return;
    }
    double a = m.adj;
    if (m.im > 0.0) a = __dadd_rn(a, __dmul_rn(gi, __ddiv_rn(__dsub_rn(__dmul_rn(m.rr, m.cp), m.d), m.im)));
    double dr = __dmul_rn(a, m.cp);
    if (m.im > 0.0) dr = __dadd_rn(dr, __dmul_rn(gi, __ddiv_rn(__dmul_rn(m.cp, m.d), m.im)));
    G.d_res[fj] = dr;
    out.put_xy(m.f, mi, j, __dmul_rn(a, m.rr),
               m.im > 0.0 ? __dmul_rn(gi, __ddiv_rn(__dmul_rn(m.rr, m.d), m.im)) : 0.0);
}

// 16-byte global -> shared asynchronous copy through L2 (cp.async.cg)
__device__ __forceinline__ void cp16(void* dst, const void* src)
{
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct NoWait {
    __device__ void operator()() const {}
};

// What the net step reads: the net's task records, its root load, its
// in-arcs' pass state (arrival + arc_delay and slew of the source pin,
// d_arc, LUT ids) and the member terms.  SrcGlobal reads global memory (the
// stand-alone sweep, and fused tasks whose net spans tasks); SrcSmem reads
// the fused kernel's prologue prefetch in shared memory.
struct NetRec { int net, root, fl, f0, m, a0, na, mb; };
struct PgArc { double v, sf, da; int a; int dl, sl; };

struct SrcGlobal : TermsGlobal {
    const Topo* tp;
    const Corner* C;
    __device__ __forceinline__ NetRec rec(int q) const
    {
        const Topo& t = *tp;
        NetRec r;
        r.net = t.lv_nets[q]; r.root = t.tq_root[q]; r.fl = t.tq_flags[q]; r.f0 = t.tq_f0[q];
        r.mb = 0;
        r.m = t.tq_mptr[q + 1] - t.tq_mptr[q];
        r.a0 = t.tq_aptr[q]; r.na = t.tq_aptr[q + 1] - r.a0;
        return r;
    }
    __device__ __forceinline__ double ld(const NetRec& r, int, int c) const
    {
        return __ldcg(C->load + (size_t)r.root * 4 + c);
    }
    __device__ __forceinline__ PgArc arc(const NetRec& n, int qa, int c, int j) const
    {
        const Topo& t = *tp;
        PgArc r;
        const int fp = t.ta_from[n.a0 + qa];
        r.a = t.ta_arc[n.a0 + qa];
        r.dl = lut_id(t.ta_lut + (2 * (size_t)(n.a0 + qa)), c);
        r.sl = lut_id(t.ta_lut + (2 * (size_t)(n.a0 + qa) + 1), c);
        r.v = __dadd_rn(__ldcg(C->arrival + (size_t)fp * 4 + c), __ldcg(C->arc_delay + (size_t)r.a * 4 + c));
        r.sf = __ldcg(C->slew + (size_t)fp * 4 + c);
        r.da = __ldcg(C->d_arc + (size_t)r.a * 2 + j);
        return r;
    }
};

// the fused kernel's per-task prefetch (ws_pass.cu BwdPgSmem): nets by task
// position ii = q - q0, in-arcs by task arc slot a0 - a0t + qa, members by
// task member slot; late columns only (double2 = conds 2, 3)
struct SrcSmem : TermsSmem {
    const int *root, *flags, *f0, *net, *aptr, *mptr;   // NetSmem
    int q0, a0t, m0;
    const double2* pa;      // [TASK_A * 3]: arrival[from], arc_delay[arc], slew[from]
    const int4* plut;       // [TASK_A]: delay LUT ids (cond 2, 3), slew LUT ids (cond 2, 3)
    const int* arcs;        // [TASK_A] arc ids
    const double* da;       // [TASK_A * 2] d_arc
    const double2* pl;      // [TASK_Q] root load
    __device__ __forceinline__ NetRec rec(int q) const
    {
        const int ii = q - q0;
        NetRec r;
        r.net = net[ii]; r.root = root[ii]; r.fl = flags[ii]; r.f0 = f0[ii];
        r.mb = mptr[ii] - m0;
        r.m = mptr[ii + 1] - mptr[ii];
        r.a0 = aptr[ii]; r.na = aptr[ii + 1] - r.a0;
        return r;
    }
    __device__ __forceinline__ double ld(const NetRec&, int q, int c) const
    {
        const double2 v = pl[q - q0];
        return c == 2 ? v.x : v.y;
    }
    __device__ __forceinline__ PgArc arc(const NetRec& n, int qa, int c, int j) const
    {
        const int s = n.a0 - a0t + qa;
        PgArc r;
        r.a = arcs[s];
        const int4 l = plut[s];
        r.dl = j ? l.y : l.x;
        r.sl = j ? l.w : l.z;
        const double2 at = pa[3 * s], ad = pa[3 * s + 1], sf = pa[3 * s + 2];
        r.v = __dadd_rn(j ? at.y : at.x, j ? ad.y : ad.x);
        r.sf = j ? sf.y : sf.x;
        r.da = da[s * 2 + j];
        return r;
    }
};

// One net per GW-lane group (lane = GW * group + 2 * slot + j, GW / 2 slots
// per late column), called by every lane of the warp (warp-uniform loop
// bounds; q < 0 marks an idle group).  Member-slot-strided root-slew sum,
// then a fixed xor tree over the slots -> root: the first strict late max
// winner over the in-arcs, LUT partials of every in-arc, gsa, dL/dload in arc
// order -> d_cap finish (star) or the oracle's recursion (tree).  `wait` runs
// after the group's first loads, before anything the previous sweep step
// writes is read (the stand-alone kernel's PDL wait).
template <int GW, class Src, class Wait = NoWait>
__device__ void pg_net_group(const Topo& t, const LutView& L, const Corner& C, const PlaceCorner& G, int q,
                             const Src& src, Wait wait = Wait())
{
    constexpr int PS = GW / 2;
    const int lane = threadIdx.x & 31, j = lane & 1, c = 2 + j;
    const int slot = (lane % GW) >> 1;
    const bool act = q >= 0;
    // ---- hop 1: level-major task records of the group's net
    const NetRec nr = act ? src.rec(q) : NetRec{0, 0, ROOT_PI, 0, 0, 0, 0, 0};
    const int net = nr.net, root = nr.root, fl = nr.fl, f0 = nr.f0, m = nr.m, na = nr.na, mb = nr.mb;
    const int kind = fl & TQ_KIND;
    const bool tree = fl & TQ_TREE;
    int rm = (m + PS - 1) / PS, ra = (na + PS - 1) / PS;
    for (int o = 16; o > 0; o >>= 1) {
        rm = max(rm, __shfl_xor_sync(WS_FULL, rm, o));
        ra = max(ra, __shfl_xor_sync(WS_FULL, ra, o));
    }
    // ---- hop 2 / 3 of round 0: root load, first in-arc slot
    const double ld = (act && kind == ROOT_ARC) ? src.ld(nr, q, c) : 0.0;
    using Arc = PgArc;
    auto load_arc = [&](int qa) {
        Arc r{-PG_INF, 0.0, 0.0, -1, 0, 0};
        if (kind == ROOT_ARC && qa < na) r = src.arc(nr, qa, c, j);
        return r;
    };
    const Arc arc0 = load_arc(slot);
    wait();
    // ---- root-slew terms of the members: the fixed order of
    // member_term_sum (8 interleaved partials, pairwise combine); slot s of
    // the group holds the partials of the residues s, s + 2, s + 4, s + 6
    static_assert(GW == 4, "the root-slew sum order is laid out for 2 slots per column");
    double x[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = 0; r < rm; r += 4)
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int k = (r + i) * PS + slot;        // residue k mod 8 = 2 i + slot
            if (r + i < rm && k < m) x[i] = __dadd_rn(x[i], src.t(f0 + k, mb + k, j));
        }
    double y[4];
#pragma unroll
    for (int i = 0; i < 4; i++) y[i] = __dadd_rn(x[i], __shfl_xor_sync(WS_FULL, x[i], 2, GW));   // P(2i) + P(2i+1)
    const double gsum = __dadd_rn(__dadd_rn(y[0], y[1]), __dadd_rn(y[2], y[3]));
    // ---- root
    double gl = 0.0, groot = gsum;
    if (act && kind == ROOT_FEED && slot == 0) G.gsr[(size_t)root * 2 + j] = gsum;
    if (act && kind != ROOT_FEED && slot == 0) {
        for (int v = t.pin_out_ptr[root]; v < t.pin_out_ptr[root + 1]; v++)
            groot = __dadd_rn(groot, __ldcg(G.gsa + (size_t)t.pin_out_arc[v] * 2 + j));
        G.gs[(size_t)root * 2 + j] = groot;
    }
    groot = __shfl_sync(WS_FULL, groot, j, GW);
    // winner: late = first strict max over the in-arcs in order
    double best = -PG_INF;
    int w = -1;
    for (int r = 0; r < ra; r++) {
        const Arc A = r == 0 ? arc0 : load_arc(r * PS + slot);
        for (int k = 0; k < PS; k++) {
            const double vk = __shfl_sync(WS_FULL, A.v, 2 * k + j, GW);
            if (r * PS + k < na && vk > best) { best = vk; w = r * PS + k; }
        }
    }
    double slw = 0.0;
    for (int r = 0; r < ra; r++) {
        const int qa = r * PS + slot;
        const Arc A = r == 0 ? arc0 : load_arc(qa);
        double term = 0.0, sl = 0.0;
        if (qa < na && kind == ROOT_ARC) {
            double ds, dl;
            interp_grad(L, A.dl, A.sf, ld, ds, dl);
            double ga = __dmul_rn(A.da, ds);
            term = __dmul_rn(A.da, dl);
            if (qa == w) {
                double ss;
                interp_grad(L, A.sl, A.sf, ld, ss, sl);
                ga = __dadd_rn(ga, __dmul_rn(groot, ss));
            }
            G.gsa[(size_t)A.a * 2 + j] = ga;
        }
        for (int k = 0; k < PS; k++) {          // arc order (oracle order)
            const double tk = __shfl_sync(WS_FULL, term, 2 * k + j, GW);
            if (r * PS + k < na) gl = __dadd_rn(gl, tk);
        }
        const bool here = w >= r * PS && w < (r + 1) * PS;
        const double slr = __shfl_sync(WS_FULL, sl, here ? 2 * (w - r * PS) + j : j, GW);
        if (here) slw = slr;
    }
    if (w >= 0) gl = __dadd_rn(gl, __dmul_rn(groot, slw));
    if (!act) return;
    if (slot == 0) {
        G.gl[(size_t)net * 2 + j] = gl;
        G.d_root_cap[(size_t)net * 2 + j] = gl;
    }
    // ---- Elmore adjoint: finish d_cap (star) / the oracle's recursion (tree)
    if (tree) {
        if (slot == 0) pg_tree_net(t, C, G, f0, m, j, gl);
        return;
    }
#pragma unroll 4
    for (int k = slot; k < m; k += PS)
        G.d_cap[(size_t)(f0 + k) * 2 + j] = __dadd_rn(__dadd_rn(src.x(f0 + k, mb + k, j), gl),
                                                      src.y(f0 + k, mb + k, j));
}

}  // namespace pg
}  // namespace
}  // namespace ws
