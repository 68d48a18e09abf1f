// Position model and position gradients on sm_100a (north_star: "run
// backward for gradients w.r.t. pin/cell positions").
//
// The reference stops at delay-space gradients (diff.py:5-7, SPEC.md
// "Non-goals: pin-location gradients"), so this file extends its pass with
//   k_wire       positions -> mem_res / mem_cap (Manhattan wire model);
//   k_pg_level   one reverse level of the slew / load adjoint sweep and the
//                Elmore adjoint of each net -> d_res, d_cap, d_root_cap;
//   k_pg_len     dL/dlength of every net edge;
//   k_pg_xy      dL/dx, dL/dy per pin, gathered (deterministic order).
// The arithmetic and its order are those of oracle/sta_oracle.c
// (orc_wire, orc_posgrad_level, orc_pos_reduce), whose header states the
// model and the derivative; the oracle is pinned by central finite
// differences of the reference-restated loss.
//
// Only late conditions (cols 2, 3) reach the loss (diff.py:21), so every
// gradient array is (., 2).  The sweep reads the finished pass state (hard
// arrival / slew / load / impulse / net_delay / arc_delay, the GradientState
// adjoint and d_arc): it runs after the fused pass on the same stream.
#include <math.h>

#include <algorithm>
#include <vector>

#include "ws_internal.h"

namespace ws {
namespace {

constexpr double INF = __builtin_huge_val();

// Programmatic dependent launch between the sweep's kernels: each kernel
// loads its records and every pass output it needs (final before the sweep
// began), then waits for its predecessor and only then lets its successor
// start.  A kernel's prologue therefore overlaps the previous kernel's body
// and may read anything written two or more launches earlier.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    WS_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

__device__ __forceinline__ int lut_c(int4 v, int c)
{
    return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// d out / d qs and d out / d ql of _interp (_kernels.pyx:15-81) inside the
// located cell; 0 along an axis whose fraction was clamped (orc interp_grad)
__device__ __forceinline__ void interp_grad(const LutView& L, int lut, double qs, double ql, double& ds, double& dl)
{
    const int s0 = L.s_ptr[lut], nS = L.s_ptr[lut + 1] - s0;
    const int l0 = L.l_ptr[lut], nL = L.l_ptr[lut + 1] - l0;
    const int t0 = L.t_ptr[lut];
    int si, li, si2, li2;
    double st, lt, hs = 0.0, hl = 0.0;
    bool fs = false, fl = false;
    if (nS > 1) {
        int lo = 0, hi = nS;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (L.s[s0 + mid] <= qs) lo = mid + 1; else hi = mid;
        }
        si = lo - 1;
        if (si < 0) si = 0; else if (si > nS - 2) si = nS - 2;
        hs = __dsub_rn(L.s[s0 + si + 1], L.s[s0 + si]);
        st = __ddiv_rn(__dsub_rn(qs, L.s[s0 + si]), hs);
        if (st < 0.0) st = 0.0; else if (st > 1.0) st = 1.0; else fs = true;
        si2 = si + 1;
    } else { si = 0; st = 0.0; si2 = 0; }
    if (nL > 1) {
        int lo = 0, hi = nL;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (L.l[l0 + mid] <= ql) lo = mid + 1; else hi = mid;
        }
        li = lo - 1;
        if (li < 0) li = 0; else if (li > nL - 2) li = nL - 2;
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

// positions -> RC of every member edge (orc_wire); one thread per member
__global__ void k_wire(int M, const int* __restrict__ mem_pin, const int* __restrict__ parent_pin,
                       const PgArgs* __restrict__ pa)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const PgArgs& A = pa[blockIdx.y];
    const double2* __restrict__ xy = reinterpret_cast<const double2*>(A.g.xy);
    const double4* __restrict__ res0 = reinterpret_cast<const double4*>(A.g.res0);
    const double4* __restrict__ cap0 = reinterpret_cast<const double4*>(A.g.cap0);
    const double* __restrict__ wire = A.g.wire;
    double4* __restrict__ res = reinterpret_cast<double4*>(A.d.mem_res);
    double4* __restrict__ cap = reinterpret_cast<double4*>(A.d.mem_cap);
    const double2 p = xy[mem_pin[k]], q = xy[parent_pin[k]];
    const double l = __dadd_rn(fabs(__dsub_rn(p.x, q.x)), fabs(__dsub_rn(p.y, q.y)));
    const double4 r0 = res0[k], c0 = cap0[k];
    res[k] = make_double4(__dadd_rn(r0.x, __dmul_rn(wire[0], l)), __dadd_rn(r0.y, __dmul_rn(wire[1], l)),
                          __dadd_rn(r0.z, __dmul_rn(wire[2], l)), __dadd_rn(r0.w, __dmul_rn(wire[3], l)));
    cap[k] = make_double4(__dadd_rn(c0.x, __dmul_rn(wire[4], l)), __dadd_rn(c0.y, __dmul_rn(wire[5], l)),
                          __dadd_rn(c0.z, __dmul_rn(wire[6], l)), __dadd_rn(c0.w, __dmul_rn(wire[7], l)));
}

// one reverse level.  An 8-lane group per net (4 nets per warp): lane =
// 8 * group + 2 * slot + j (j = late column), 4 members / in-arcs per round.
// Member phase (slew adjoint of each member from its out-arcs and the
// feedthrough net it roots; on star nets the Elmore adjoint up to the
// dL/dload term) -> ordered group sum of the root-slew terms -> root (winner,
// LUT partials of the in-arcs, dL/dload, in arc order) -> d_cap.  RC-tree
// nets run the oracle's sequential recursion (pg_tree_net).  Every load of
// round 0 is issued before the first store so a net costs ~3 dependent
// memory hops.
constexpr int PG_WARPS = 8, PG_G = 8, PG_S = PG_G / 2;

__device__ void pg_tree_net(const Topo& t, const Corner& C, const PlaceCorner& G, int s, int m,
                            int j, double gl)
{
    const int c = 2 + j;
    double* gimp = G.sc_gimp + (size_t)s * 2 + j;
    double* buf = G.sc_buf + (size_t)s * 2 + j;
    double* acc = G.sc_acc + (size_t)s * 2 + j;
    for (int k = 0; k < m; k++) buf[2 * k] = C.mem_cap[(size_t)(s + k) * 4 + c];
    for (int k = m - 1; k > 0; k--) {
        const int pl = t.mem_parent_loc[s + k];
        if (pl > 0) buf[2 * (pl - 1)] = __dadd_rn(buf[2 * (pl - 1)], buf[2 * k]);
    }
    for (int k = 0; k < m; k++) {
        const int pin = t.mem_pin[s + k];
        const double r = C.mem_res[(size_t)(s + k) * 4 + c], cp = C.mem_cap[(size_t)(s + k) * 4 + c];
        const double d = C.net_delay[(size_t)pin * 4 + c], im = C.impulse[(size_t)pin * 4 + c];
        double a = C.adjoint[(size_t)pin * 2 + j];
        if (im > 0.0) a = __dadd_rn(a, __dmul_rn(gimp[2 * k], __ddiv_rn(__dsub_rn(__dmul_rn(r, cp), d), im)));
        acc[2 * k] = a;
    }
    for (int k = m - 1; k > 0; k--) {
        const int pl = t.mem_parent_loc[s + k];
        if (pl > 0) acc[2 * (pl - 1)] = __dadd_rn(acc[2 * (pl - 1)], acc[2 * k]);
    }
    for (int k = 0; k < m; k++) {
        const int pin = t.mem_pin[s + k];
        const double r = C.mem_res[(size_t)(s + k) * 4 + c], cp = C.mem_cap[(size_t)(s + k) * 4 + c];
        const double d = C.net_delay[(size_t)pin * 4 + c], im = C.impulse[(size_t)pin * 4 + c];
        double dr = __dmul_rn(acc[2 * k], buf[2 * k]);
        if (im > 0.0) dr = __dadd_rn(dr, __dmul_rn(gimp[2 * k], __ddiv_rn(__dmul_rn(cp, d), im)));
        G.d_res[(size_t)(s + k) * 2 + j] = dr;
        acc[2 * k] = __dadd_rn(__dmul_rn(acc[2 * k], r), gl);
    }
    for (int k = 1; k < m; k++) {
        const int pl = t.mem_parent_loc[s + k];
        if (pl > 0) acc[2 * k] = __dadd_rn(acc[2 * k], acc[2 * (pl - 1)]);
    }
    for (int k = 0; k < m; k++) {
        const int pin = t.mem_pin[s + k];
        const double r = C.mem_res[(size_t)(s + k) * 4 + c];
        const double d = C.net_delay[(size_t)pin * 4 + c], im = C.impulse[(size_t)pin * 4 + c];
        double dc = acc[2 * k];
        if (im > 0.0) dc = __dadd_rn(dc, __dmul_rn(gimp[2 * k], __ddiv_rn(__dmul_rn(r, d), im)));
        G.d_cap[(size_t)(s + k) * 2 + j] = dc;
    }
}

// member phase of one reverse level, thread = (member slot u of the level in
// task order, late column j): slew adjoint g from the member's out-arcs and
// the feedthrough net it roots; impulse adjoint; the root-slew term
// g * (sr / sm); on star nets the Elmore adjoint up to the dL/dload term
//   A = adj + gimp (r cap - d) / imp,  d_res = A cap + gimp cap d / imp,
//   x = A r,  y = gimp r d / imp   (d_cap = (x + gl) + y, k_pg_level)
// (orc_posgrad_level with buf = cap).  RC-tree nets keep gimp only.
__global__ void __launch_bounds__(256) k_pg_mem(Topo t, PlaceTopo pt, const PgArgs* __restrict__ pa,
                                                int u_begin, int n2)
{
    const Corner& C = pa[blockIdx.y].d;
    const PlaceCorner& G = pa[blockIdx.y].g;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n2) {
        pdl_wait();
        pdl_trigger();
        return;
    }
    const int u = u_begin + (i >> 1), j = i & 1, c = 2 + j;
    const int pin = t.tm_pin[u], o1 = t.tm_o1_arc[u], fl = t.tm_flags[u];
    const int f = pt.tm_f[u], root = pt.tm_root[u];
    const bool tree = t.net_tree[t.mem_net[f]] != 0;
    const double sm = C.slew[(size_t)pin * 4 + c], im = C.impulse[(size_t)pin * 4 + c];
    const double sr = C.slew[(size_t)root * 4 + c];
    const double rr = C.mem_res[(size_t)f * 4 + c], cp = C.mem_cap[(size_t)f * 4 + c];
    const double d = C.net_delay[(size_t)pin * 4 + c], adj = C.adjoint[(size_t)pin * 2 + j];
    pdl_wait();          // gsa / gsr of the higher levels
    pdl_trigger();
    double g = 0.0;
    if (o1 >= 0) {
        g = __dadd_rn(g, G.gsa[(size_t)o1 * 2 + j]);
        for (int v = t.tm_optr[u] + 1; v < t.tm_optr[u + 1]; v++)
            g = __dadd_rn(g, G.gsa[(size_t)t.to_arc[v] * 2 + j]);
    }
    if (fl & TM_ROOT) g = __dadd_rn(g, G.gsr[(size_t)pin * 2 + j]);
    G.gs[(size_t)pin * 2 + j] = g;
    double gi = 0.0, tk = 0.0;
    if (sm > 0.0) {
        tk = __dmul_rn(g, __ddiv_rn(sr, sm));
        gi = __dmul_rn(g, __ddiv_rn(im, sm));
    }
    const size_t fj = (size_t)f * 2 + j;
    G.sc_t[fj] = tk;
    if (tree) {
        G.sc_gimp[fj] = gi;
        return;
    }
    double a = adj;
    if (im > 0.0) a = __dadd_rn(a, __dmul_rn(gi, __ddiv_rn(__dsub_rn(__dmul_rn(rr, cp), d), im)));
    double dr = __dmul_rn(a, cp);
    if (im > 0.0) dr = __dadd_rn(dr, __dmul_rn(gi, __ddiv_rn(__dmul_rn(cp, d), im)));
    G.d_res[fj] = dr;
    G.sc_buf[fj] = __dmul_rn(a, rr);
    G.sc_acc[fj] = im > 0.0 ? __dmul_rn(gi, __ddiv_rn(__dmul_rn(rr, d), im)) : 0.0;
}

__global__ void __launch_bounds__(PG_WARPS * 32, 3) k_pg_level(Topo t, LutSrc ls, bool use_smem,
                                                               const PgArgs* __restrict__ pa, int q0, int nq)
{
    const Corner& C = pa[blockIdx.y].d;
    const PlaceCorner& G = pa[blockIdx.y].g;
    extern __shared__ __align__(16) unsigned char smem[];
    const LutView L = stage_luts(ls, C.lut_t_flat, use_smem, smem);
    const int lane = threadIdx.x & 31, grp = lane / PG_G, j = lane & 1, c = 2 + j;
    const int slot = (lane % PG_G) >> 1;
    const int wq = (blockIdx.x * PG_WARPS + (threadIdx.x >> 5)) * (32 / PG_G);
    if (wq >= nq) {                              // whole warp idle
        pdl_wait();
        pdl_trigger();
        return;
    }
    const int qi = wq + grp;
    const bool act = qi < nq;
    // ---- hop 1: level-major task records of the group's net
    int net = 0, root = 0, fl = ROOT_PI, f0 = 0, u0 = 0, m = 0, a0 = 0, na = 0;
    if (act) {
        const int q = q0 + qi;
        net = t.lv_nets[q]; root = t.tq_root[q]; fl = t.tq_flags[q]; f0 = t.tq_f0[q];
        u0 = t.tq_mptr[q]; m = t.tq_mptr[q + 1] - u0;
        a0 = t.tq_aptr[q]; na = t.tq_aptr[q + 1] - a0;
    }
    const int kind = fl & TQ_KIND;
    const bool tree = fl & TQ_TREE;
    int rm = (m + PG_S - 1) / PG_S, ra = (na + PG_S - 1) / PG_S;
    for (int o = 16; o > 0; o >>= 1) {
        rm = max(rm, __shfl_xor_sync(WS_FULL, rm, o));
        ra = max(ra, __shfl_xor_sync(WS_FULL, ra, o));
    }
    // ---- hop 2 / 3 of round 0: root, first in-arc slot, first member slot
    const double sr = act ? C.slew[(size_t)root * 4 + c] : 0.0;
    const double ld = (act && kind == ROOT_ARC) ? C.load[(size_t)root * 4 + c] : 0.0;
    struct Arc { double v, sf, da; int a; int dl, sl; };
    auto load_arc = [&](int qa) {
        Arc r{-INF, 0.0, 0.0, -1, 0, 0};
        if (kind == ROOT_ARC && qa < na) {
            const int fp = t.ta_from[a0 + qa];
            r.a = t.ta_arc[a0 + qa];
            r.dl = lut_c(t.ta_lut[2 * (size_t)(a0 + qa)], c);
            r.sl = lut_c(t.ta_lut[2 * (size_t)(a0 + qa) + 1], c);
            r.v = __dadd_rn(C.arrival[(size_t)fp * 4 + c], C.arc_delay[(size_t)r.a * 4 + c]);
            r.sf = C.slew[(size_t)fp * 4 + c];
            r.da = C.d_arc[(size_t)r.a * 2 + j];
        }
        return r;
    };
    const Arc arc0 = load_arc(slot);
    pdl_wait();          // this level's k_pg_mem (member terms), higher levels' gsa
    pdl_trigger();
    // ---- root-slew terms of the members (k_pg_mem), summed in slot order
    const double* __restrict__ sct = G.sc_t;
    double part = 0.0;
#pragma unroll 4
    for (int r = 0; r < rm; r++) {
        const int k = r * PG_S + slot;
        if (k < m) part = __dadd_rn(part, sct[(size_t)(f0 + k) * 2 + j]);
    }
    // fixed-order sum over the slots of column j within the group
    for (int o = 2; o < PG_G; o <<= 1) part = __dadd_rn(part, __shfl_xor_sync(WS_FULL, part, o, PG_G));
    const double gsum = part;
    // ---- root
    double gl = 0.0, groot = gsum;
    if (act && kind == ROOT_FEED && slot == 0) G.gsr[(size_t)root * 2 + j] = gsum;
    if (act && kind != ROOT_FEED && slot == 0) {
        for (int v = t.pin_out_ptr[root]; v < t.pin_out_ptr[root + 1]; v++)
            groot = __dadd_rn(groot, G.gsa[(size_t)t.pin_out_arc[v] * 2 + j]);
        G.gs[(size_t)root * 2 + j] = groot;
    }
    groot = __shfl_sync(WS_FULL, groot, j, PG_G);
    // winner: late = first strict max over the in-arcs in order
    double best = -INF;
    int w = -1;
    for (int r = 0; r < ra; r++) {
        const Arc A = r == 0 ? arc0 : load_arc(r * PG_S + slot);
        for (int k = 0; k < PG_S; k++) {
            const double vk = __shfl_sync(WS_FULL, A.v, 2 * k + j, PG_G);
            if (r * PG_S + k < na && vk > best) { best = vk; w = r * PG_S + k; }
        }
    }
    double slw = 0.0;
    for (int r = 0; r < ra; r++) {
        const int qa = r * PG_S + slot;
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
        for (int k = 0; k < PG_S; k++) {          // arc order (oracle order)
            const double tk = __shfl_sync(WS_FULL, term, 2 * k + j, PG_G);
            if (r * PG_S + k < na) gl = __dadd_rn(gl, tk);
        }
        const bool here = w >= r * PG_S && w < (r + 1) * PG_S;
        const double slr = __shfl_sync(WS_FULL, sl, here ? 2 * (w - r * PG_S) + j : j, PG_G);
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
    const double* __restrict__ xs = G.sc_buf;
    const double* __restrict__ ys = G.sc_acc;
    double* __restrict__ dcap = G.d_cap;
#pragma unroll 4
    for (int k = slot; k < m; k += PG_S) {
        const size_t f = (size_t)(f0 + k) * 2 + j;
        dcap[f] = __dadd_rn(__dadd_rn(xs[f], gl), ys[f]);
    }
}

__device__ __forceinline__ double sgn(double d) { return d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0); }

// dL/dlength of member edge k and its signed x / y contributions
// e_k = dL/dlength * sign(member - parent) (orc_pos_reduce's g * sg)
__global__ void k_pg_len(int M, const int* __restrict__ mem_pin, const int* __restrict__ parent_pin,
                         const PgArgs* __restrict__ pa)
{
    const PlaceCorner& G = pa[blockIdx.y].g;
    pdl_wait();
    pdl_trigger();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const double* w = G.wire;
    const double2 dr = reinterpret_cast<const double2*>(G.d_res)[k];
    const double2 dc = reinterpret_cast<const double2*>(G.d_cap)[k];
    double g = 0.0;
    g = __dadd_rn(g, __dadd_rn(__dmul_rn(dr.x, w[2]), __dmul_rn(dc.x, w[6])));
    g = __dadd_rn(g, __dadd_rn(__dmul_rn(dr.y, w[3]), __dmul_rn(dc.y, w[7])));
    G.g_len[k] = g;
    const double2 xp = reinterpret_cast<const double2*>(G.xy)[mem_pin[k]];
    const double2 xq = reinterpret_cast<const double2*>(G.xy)[parent_pin[k]];
    reinterpret_cast<double2*>(G.sc_buf)[k] =
        make_double2(__dmul_rn(g, sgn(__dsub_rn(xp.x, xq.x))), __dmul_rn(g, sgn(__dsub_rn(xp.y, xq.y))));
}

// dL/dxy of pin p: + its own edge (as a member), - the edges of its children
// (as a parent), merged in ascending member order = orc_pos_reduce's order
__global__ void k_pg_xy(int P, const int* __restrict__ member_of_pin, const int* __restrict__ pc_ptr,
                        const int* __restrict__ pc_mem, const PgArgs* __restrict__ pa)
{
    const double2* __restrict__ e = reinterpret_cast<const double2*>(pa[blockIdx.y].g.sc_buf);
    double2* __restrict__ d_xy = reinterpret_cast<double2*>(pa[blockIdx.y].g.d_xy);
    pdl_wait();
    pdl_trigger();
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int own = member_of_pin[p];
    const int q0 = pc_ptr[p], q1 = pc_ptr[p + 1];
    double gx = 0.0, gy = 0.0;
    bool own_done = own < 0;
    if (!own_done && (q0 == q1 || own < pc_mem[q0])) {
        const double2 v = e[own];
        gx = __dadd_rn(gx, v.x);
        gy = __dadd_rn(gy, v.y);
        own_done = true;
    }
#pragma unroll 4
    for (int q = q0; q < q1; q++) {
        const int k = pc_mem[q];
        if (!own_done && own < k) {
            const double2 v = e[own];
            gx = __dadd_rn(gx, v.x);
            gy = __dadd_rn(gy, v.y);
            own_done = true;
        }
        const double2 v = e[k];
        gx = __dsub_rn(gx, v.x);
        gy = __dsub_rn(gy, v.y);
    }
    if (!own_done) {
        const double2 v = e[own];
        gx = __dadd_rn(gx, v.x);
        gy = __dadd_rn(gy, v.y);
    }
    d_xy[p] = make_double2(gx, gy);
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

void place_enable(Context& ctx)
{
    if (ctx.pt.ready) return;
    const Topo& t = ctx.t;
    const int P = t.P, M = t.M, N = t.N;
    // parent pin per member and the child edges of each pin (host, once)
    std::vector<int> net_ptr(N + 1), net_root(N), mem_pin(M), mpl(M);
    WS_CUDA(cudaMemcpy(net_ptr.data(), t.net_ptr, sizeof(int) * (N + 1), cudaMemcpyDeviceToHost));
    if (N) WS_CUDA(cudaMemcpy(net_root.data(), t.net_root, sizeof(int) * N, cudaMemcpyDeviceToHost));
    if (M) {
        WS_CUDA(cudaMemcpy(mem_pin.data(), t.mem_pin, sizeof(int) * M, cudaMemcpyDeviceToHost));
        WS_CUDA(cudaMemcpy(mpl.data(), t.mem_parent_loc, sizeof(int) * M, cudaMemcpyDeviceToHost));
    }
    std::vector<int> par(M), cptr(P + 1, 0), cmem(M);
    for (int n = 0; n < N; n++)
        for (int k = net_ptr[n]; k < net_ptr[n + 1]; k++)
            par[k] = mpl[k] > 0 ? mem_pin[net_ptr[n] + mpl[k] - 1] : net_root[n];
    for (int k = 0; k < M; k++) cptr[par[k] + 1]++;
    for (int p = 0; p < P; p++) cptr[p + 1] += cptr[p];
    {
        std::vector<int> fill(cptr.begin(), cptr.end() - 1);
        for (int k = 0; k < M; k++) cmem[fill[par[k]]++] = k;   // ascending k per pin
    }
    // task-order member slot -> original member index / root pin
    std::vector<int> tq_mptr(N + 1), tq_f0(N), tq_root(N), tm_f(M), tm_root(M);
    WS_CUDA(cudaMemcpy(tq_mptr.data(), t.tq_mptr, sizeof(int) * (N + 1), cudaMemcpyDeviceToHost));
    if (N) {
        WS_CUDA(cudaMemcpy(tq_f0.data(), t.tq_f0, sizeof(int) * N, cudaMemcpyDeviceToHost));
        WS_CUDA(cudaMemcpy(tq_root.data(), t.tq_root, sizeof(int) * N, cudaMemcpyDeviceToHost));
    }
    for (int q = 0; q < N; q++)
        for (int u = tq_mptr[q]; u < tq_mptr[q + 1]; u++) {
            tm_f[u] = tq_f0[q] + (u - tq_mptr[q]);
            tm_root[u] = tq_root[q];
        }
    ctx.pt.tq_mptr_host = tq_mptr;
    Arena& ar = ctx.topo_mem;
    ctx.pt.tm_f = ar.alloc<int>(std::max(M, 1));
    ctx.pt.tm_root = ar.alloc<int>(std::max(M, 1));
    if (M) {
        WS_CUDA(cudaMemcpy(ctx.pt.tm_f, tm_f.data(), sizeof(int) * M, cudaMemcpyHostToDevice));
        WS_CUDA(cudaMemcpy(ctx.pt.tm_root, tm_root.data(), sizeof(int) * M, cudaMemcpyHostToDevice));
    }
    ctx.pt.parent_pin = ar.alloc<int>(std::max(M, 1));
    ctx.pt.pc_ptr = ar.alloc<int>(P + 1);
    ctx.pt.pc_mem = ar.alloc<int>(std::max(M, 1));
    if (M) {
        WS_CUDA(cudaMemcpy(ctx.pt.parent_pin, par.data(), sizeof(int) * M, cudaMemcpyHostToDevice));
        WS_CUDA(cudaMemcpy(ctx.pt.pc_mem, cmem.data(), sizeof(int) * M, cudaMemcpyHostToDevice));
    }
    WS_CUDA(cudaMemcpy(ctx.pt.pc_ptr, cptr.data(), sizeof(int) * (P + 1), cudaMemcpyHostToDevice));
    // per corner: positions = 0, base RC = the corner's current RC, wire = 0
    // (the model then reproduces the current values exactly)
    Arena& vr = ctx.val_mem;
    ctx.place.resize(ctx.corners.size());
    for (size_t ci = 0; ci < ctx.corners.size(); ci++) {
        PlaceCorner& g = ctx.place[ci];
        const Corner& d = ctx.corners[ci].d;
        g.xy = vr.alloc<double>(2 * (size_t)P);
        g.res0 = vr.alloc<double>(4 * (size_t)M);
        g.cap0 = vr.alloc<double>(4 * (size_t)M);
        g.wire = vr.alloc<double>(8);
        g.gs = vr.alloc<double>(2 * (size_t)P);
        g.gsr = vr.alloc<double>(2 * (size_t)P);
        g.gsa = vr.alloc<double>(2 * (size_t)t.A);
        g.gl = vr.alloc<double>(2 * (size_t)N);
        g.d_res = vr.alloc<double>(2 * (size_t)M);
        g.d_cap = vr.alloc<double>(2 * (size_t)M);
        g.d_root_cap = vr.alloc<double>(2 * (size_t)N);
        g.g_len = vr.alloc<double>((size_t)M);
        g.d_xy = vr.alloc<double>(2 * (size_t)P);
        g.sc_gimp = vr.alloc<double>(2 * (size_t)M);
        g.sc_buf = vr.alloc<double>(2 * (size_t)M);
        g.sc_acc = vr.alloc<double>(2 * (size_t)M);
        g.sc_t = vr.alloc<double>(2 * (size_t)M);
        WS_CUDA(cudaMemset(g.xy, 0, sizeof(double) * 2 * std::max(P, 1)));
        WS_CUDA(cudaMemset(g.wire, 0, sizeof(double) * 8));
        if (M) {
            WS_CUDA(cudaMemcpy(g.res0, d.mem_res, sizeof(double) * 4 * M, cudaMemcpyDeviceToDevice));
            WS_CUDA(cudaMemcpy(g.cap0, d.mem_cap, sizeof(double) * 4 * M, cudaMemcpyDeviceToDevice));
        }
        for (double* z : {g.gs, g.gsr, g.d_xy})
            WS_CUDA(cudaMemset(z, 0, sizeof(double) * 2 * std::max(P, 1)));
        for (double* z : {g.d_res, g.d_cap, g.sc_gimp, g.sc_buf, g.sc_acc, g.sc_t})
            WS_CUDA(cudaMemset(z, 0, sizeof(double) * 2 * std::max(M, 1)));
        WS_CUDA(cudaMemset(g.g_len, 0, sizeof(double) * std::max(M, 1)));
        WS_CUDA(cudaMemset(g.gsa, 0, sizeof(double) * 2 * std::max(t.A, 1)));
        WS_CUDA(cudaMemset(g.gl, 0, sizeof(double) * 2 * std::max(N, 1)));
        WS_CUDA(cudaMemset(g.d_root_cap, 0, sizeof(double) * 2 * std::max(N, 1)));
    }
    std::vector<PgArgs> pa(ctx.corners.size());
    for (size_t ci = 0; ci < ctx.corners.size(); ci++) pa[ci] = PgArgs{ctx.corners[ci].d, ctx.place[ci]};
    ctx.pg_args = ctx.topo_mem.alloc<PgArgs>(pa.size());
    WS_CUDA(cudaMemcpy(ctx.pg_args, pa.data(), sizeof(PgArgs) * pa.size(), cudaMemcpyHostToDevice));
    ctx.pt.ready = true;
}

int launch_wire(Context& ctx, int c0, int nc, cudaStream_t s)
{
    const Topo& t = ctx.t;
    if (!t.M) return 0;
    k_wire<<<dim3((t.M + 255) / 256, nc), 256, 0, s>>>(t.M, t.mem_pin, ctx.pt.parent_pin,
                                                        ctx.pg_args + c0);
    WS_CHECK_LAUNCH();
    return 1;
}

int launch_posgrad(Context& ctx, int c0, int nc, cudaStream_t s_pass, cudaStream_t gs,
                   const std::vector<cudaEvent_t>* bwd_done)
{
    // with bwd_done the sweep runs on gs; every PG_GROUP levels it waits for
    // the pass's backward level at the group's bottom (which implies the
    // group's upper levels), and the kernel after each wait is launched
    // without PDL so its prologue cannot run ahead of that dependency
    constexpr int PG_GROUP = 4;
    const cudaStream_t s = bwd_done ? gs : s_pass;
    const Topo& t = ctx.t;
    int count = 0;
    const LutSrc ls{t.lut_s_ptr, t.lut_l_ptr, t.lut_t_ptr, t.lut_s_flat, t.lut_l_flat, t.NL,
                    ctx.lut_s_len, ctx.lut_l_len, ctx.lut_t_len, t.lut_info};
    // the 9 KB pool stays L1-resident; per-block smem staging would cost more
    // than the few located queries of a net's in-arcs
    const size_t lut_bytes = 0;
    const bool use_smem = false;
    // arcs of lower-level targets are read before written: start from 0
    for (int k = c0; k < c0 + nc; k++) {
        const PlaceCorner& g = ctx.place[k];
        if (t.A) WS_CUDA(cudaMemsetAsync(g.gsa, 0, sizeof(double) * 2 * (size_t)t.A, s));
        if (t.P) WS_CUDA(cudaMemsetAsync(g.gsr, 0, sizeof(double) * 2 * (size_t)t.P, s));
    }
    const PgArgs* pa = ctx.pg_args + c0;   // blockIdx.y = corner
    bool pdl = false;        // the first sweep kernel waits for the whole pass
    int waited = t.L;        // lowest backward level known complete
    for (int li = t.L - 1; li >= 0; li--) {
        const int q0 = ctx.lv_ptr_host[li], nq = ctx.lv_ptr_host[li + 1] - q0;
        if (bwd_done && li < waited) {
            waited = std::max(0, li - PG_GROUP + 1);
            WS_CUDA(cudaStreamWaitEvent(s, (*bwd_done)[waited], 0));
            pdl = false;
        }
        if (nq <= 0) continue;
        const int ub = ctx.pt.tq_mptr_host[q0], un = ctx.pt.tq_mptr_host[q0 + nq] - ub;
        if (un > 0) {
            launch_pdl(pdl, k_pg_mem, dim3((2 * un + 255) / 256, nc), dim3(256), 0, s, t, ctx.pt, pa, ub,
                       2 * un);
            pdl = true;
            count++;
        }
        launch_pdl(pdl, k_pg_level,
                   dim3((nq + PG_WARPS * (32 / PG_G) - 1) / (PG_WARPS * (32 / PG_G)), nc),
                   dim3(PG_WARPS * 32), lut_bytes, s, t, ls, use_smem, pa, q0, nq);
        pdl = true;
        count++;
    }
    if (t.M) {
        launch_pdl(pdl, k_pg_len, dim3((t.M + 255) / 256, nc), dim3(256), 0, s, t.M,
                   (const int*)t.mem_pin, (const int*)ctx.pt.parent_pin, pa);
        pdl = true;
        count++;
    }
    if (t.P) {
        launch_pdl(pdl, k_pg_xy, dim3((t.P + 255) / 256, nc), dim3(256), 0, s, t.P,
                   (const int*)t.member_of_pin, (const int*)ctx.pt.pc_ptr, (const int*)ctx.pt.pc_mem, pa);
        count++;
    }
    WS_CHECK_LAUNCH();
    return count;
}

}  // namespace ws
