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

struct Lut {
    const int *s_ptr, *l_ptr, *t_ptr;
    const double *s, *l, *t;
};

// d out / d qs and d out / d ql of _interp (_kernels.pyx:15-81) inside the
// located cell; 0 along an axis whose fraction was clamped (orc interp_grad)
__device__ void interp_grad(const Lut& L, int lut, double qs, double ql, double& ds, double& dl)
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
                       const double2* __restrict__ xy, const double4* __restrict__ res0,
                       const double4* __restrict__ cap0, const double* __restrict__ wire,
                       double4* __restrict__ res, double4* __restrict__ cap)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const double2 p = xy[mem_pin[k]], q = xy[parent_pin[k]];
    const double l = __dadd_rn(fabs(__dsub_rn(p.x, q.x)), fabs(__dsub_rn(p.y, q.y)));
    const double4 r0 = res0[k], c0 = cap0[k];
    res[k] = make_double4(__dadd_rn(r0.x, __dmul_rn(wire[0], l)), __dadd_rn(r0.y, __dmul_rn(wire[1], l)),
                          __dadd_rn(r0.z, __dmul_rn(wire[2], l)), __dadd_rn(r0.w, __dmul_rn(wire[3], l)));
    cap[k] = make_double4(__dadd_rn(c0.x, __dmul_rn(wire[4], l)), __dadd_rn(c0.y, __dmul_rn(wire[5], l)),
                          __dadd_rn(c0.z, __dmul_rn(wire[6], l)), __dadd_rn(c0.w, __dmul_rn(wire[7], l)));
}

// one reverse level: thread = (net of the level, late column j)
__global__ void __launch_bounds__(128) k_pg_level(Topo t, Lut L, Corner C, PlaceCorner G, int q0, int nq)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * nq) return;
    const int net = t.lv_nets[q0 + (i >> 1)], j = i & 1, c = 2 + j;
    const int s = t.net_ptr[net], e = t.net_ptr[net + 1], m = e - s, root = t.net_root[net];
    double* gimp = G.sc_gimp + (size_t)s * 2 + j;     // member scratch, stride 2
    double* buf = G.sc_buf + (size_t)s * 2 + j;
    double* acc = G.sc_acc + (size_t)s * 2 + j;
    const double sr = C.slew[(size_t)root * 4 + c];
    double gsum = 0.0, gl = 0.0;
    // members: slew adjoint (out-arcs + the feedthrough net they root)
    for (int k = 0; k < m; k++) {
        const int pin = t.mem_pin[s + k];
        double g = 0.0;
        for (int q = t.pin_out_ptr[pin]; q < t.pin_out_ptr[pin + 1]; q++)
            g = __dadd_rn(g, G.gsa[(size_t)t.pin_out_arc[q] * 2 + j]);
        if (t.root_net_of_pin[pin] >= 0) g = __dadd_rn(g, G.gsr[(size_t)pin * 2 + j]);
        G.gs[(size_t)pin * 2 + j] = g;
        const double sm = C.slew[(size_t)pin * 4 + c];
        if (sm > 0.0) {
            gsum = __dadd_rn(gsum, __dmul_rn(g, __ddiv_rn(sr, sm)));
            gimp[2 * k] = __dmul_rn(g, __ddiv_rn(C.impulse[(size_t)pin * 4 + c], sm));
        } else {
            gimp[2 * k] = 0.0;
        }
    }
    const int kind = t.root_kind[net];
    if (kind == ROOT_FEED) {
        G.gsr[(size_t)root * 2 + j] = gsum;
    } else {
        double groot = gsum;
        for (int q = t.pin_out_ptr[root]; q < t.pin_out_ptr[root + 1]; q++)
            groot = __dadd_rn(groot, G.gsa[(size_t)t.pin_out_arc[q] * 2 + j]);
        G.gs[(size_t)root * 2 + j] = groot;
        if (kind == ROOT_ARC) {
            const double ld = C.load[(size_t)root * 4 + c];
            const int a0 = t.net_in_ptr[net], a1 = t.net_in_ptr[net + 1];
            double best = -INF;
            int w = -1;
            for (int q = a0; q < a1; q++) {
                const int a = t.net_in_arc[q];
                const double v = __dadd_rn(C.arrival[(size_t)t.arc_from[a] * 4 + c], C.arc_delay[(size_t)a * 4 + c]);
                if (v > best) { best = v; w = a; }
            }
            for (int q = a0; q < a1; q++) {
                const int a = t.net_in_arc[q];
                double ds, dl;
                interp_grad(L, t.arc_dlut[(size_t)a * 4 + c], C.slew[(size_t)t.arc_from[a] * 4 + c], ld, ds, dl);
                const double da = C.d_arc[(size_t)a * 2 + j];
                G.gsa[(size_t)a * 2 + j] = __dmul_rn(da, ds);
                gl = __dadd_rn(gl, __dmul_rn(da, dl));
            }
            if (w >= 0) {
                double ds, dl;
                interp_grad(L, t.arc_slut[(size_t)w * 4 + c], C.slew[(size_t)t.arc_from[w] * 4 + c], ld, ds, dl);
                G.gsa[(size_t)w * 2 + j] = __dadd_rn(G.gsa[(size_t)w * 2 + j], __dmul_rn(groot, ds));
                gl = __dadd_rn(gl, __dmul_rn(groot, dl));
            }
        }
    }
    G.gl[(size_t)net * 2 + j] = gl;
    G.d_root_cap[(size_t)net * 2 + j] = gl;
    // Elmore adjoint of the net (rc_level order, _kernels.pyx:118-151)
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

// dL/dlength of member edge k (orc_pos_reduce, first line)
__global__ void k_pg_len(int M, PlaceCorner G)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const double* w = G.wire;
    double g = 0.0;
    for (int j = 0; j < 2; j++)
        g = __dadd_rn(g, __dadd_rn(__dmul_rn(G.d_res[(size_t)k * 2 + j], w[2 + j]),
                                   __dmul_rn(G.d_cap[(size_t)k * 2 + j], w[6 + j])));
    G.g_len[k] = g;
}

__device__ __forceinline__ double sgn(double d) { return d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0); }

// dL/dxy of pin p: its own edge (as a member) and the edges of its children
// (as a parent), merged in ascending member order = orc_pos_reduce's order
__global__ void k_pg_xy(int P, Topo t, PlaceTopo pt, PlaceCorner G)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const double2 xp = reinterpret_cast<const double2*>(G.xy)[p];
    const int own = t.member_of_pin[p];
    double gx = 0.0, gy = 0.0;
    bool own_done = own < 0;
    auto add_own = [&]() {
        const double2 xq = reinterpret_cast<const double2*>(G.xy)[pt.parent_pin[own]];
        const double g = G.g_len[own];
        gx = __dadd_rn(gx, __dmul_rn(g, sgn(__dsub_rn(xp.x, xq.x))));
        gy = __dadd_rn(gy, __dmul_rn(g, sgn(__dsub_rn(xp.y, xq.y))));
        own_done = true;
    };
    for (int q = pt.pc_ptr[p]; q < pt.pc_ptr[p + 1]; q++) {
        const int k = pt.pc_mem[q];
        if (!own_done && own < k) add_own();
        const double2 xk = reinterpret_cast<const double2*>(G.xy)[t.mem_pin[k]];
        const double g = G.g_len[k];
        gx = __dsub_rn(gx, __dmul_rn(g, sgn(__dsub_rn(xk.x, xp.x))));
        gy = __dsub_rn(gy, __dmul_rn(g, sgn(__dsub_rn(xk.y, xp.y))));
    }
    if (!own_done) add_own();
    reinterpret_cast<double2*>(G.d_xy)[p] = make_double2(gx, gy);
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
    Arena& ar = ctx.topo_mem;
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
        WS_CUDA(cudaMemset(g.xy, 0, sizeof(double) * 2 * std::max(P, 1)));
        WS_CUDA(cudaMemset(g.wire, 0, sizeof(double) * 8));
        if (M) {
            WS_CUDA(cudaMemcpy(g.res0, d.mem_res, sizeof(double) * 4 * M, cudaMemcpyDeviceToDevice));
            WS_CUDA(cudaMemcpy(g.cap0, d.mem_cap, sizeof(double) * 4 * M, cudaMemcpyDeviceToDevice));
        }
        for (double* z : {g.gs, g.gsr, g.d_xy})
            WS_CUDA(cudaMemset(z, 0, sizeof(double) * 2 * std::max(P, 1)));
        for (double* z : {g.d_res, g.d_cap, g.sc_gimp, g.sc_buf, g.sc_acc})
            WS_CUDA(cudaMemset(z, 0, sizeof(double) * 2 * std::max(M, 1)));
        WS_CUDA(cudaMemset(g.g_len, 0, sizeof(double) * std::max(M, 1)));
        WS_CUDA(cudaMemset(g.gsa, 0, sizeof(double) * 2 * std::max(t.A, 1)));
        WS_CUDA(cudaMemset(g.gl, 0, sizeof(double) * 2 * std::max(N, 1)));
        WS_CUDA(cudaMemset(g.d_root_cap, 0, sizeof(double) * 2 * std::max(N, 1)));
    }
    ctx.pt.ready = true;
}

int launch_wire(Context& ctx, int c0, int nc, cudaStream_t s)
{
    const Topo& t = ctx.t;
    if (!t.M) return 0;
    for (int k = c0; k < c0 + nc; k++) {
        const PlaceCorner& g = ctx.place[k];
        const Corner& d = ctx.corners[k].d;
        k_wire<<<(t.M + 255) / 256, 256, 0, s>>>(
            t.M, t.mem_pin, ctx.pt.parent_pin, reinterpret_cast<const double2*>(g.xy),
            reinterpret_cast<const double4*>(g.res0), reinterpret_cast<const double4*>(g.cap0), g.wire,
            reinterpret_cast<double4*>(d.mem_res), reinterpret_cast<double4*>(d.mem_cap));
        WS_CHECK_LAUNCH();
    }
    return nc;
}

int launch_posgrad(Context& ctx, int c0, int nc, cudaStream_t s)
{
    const Topo& t = ctx.t;
    int count = 0;
    for (int k = c0; k < c0 + nc; k++) {
        const PlaceCorner& g = ctx.place[k];
        const Corner& d = ctx.corners[k].d;
        const Lut L{t.lut_s_ptr, t.lut_l_ptr, t.lut_t_ptr, t.lut_s_flat, t.lut_l_flat, d.lut_t_flat};
        // arcs of lower-level targets are read before written: start from 0
        if (t.A) WS_CUDA(cudaMemsetAsync(g.gsa, 0, sizeof(double) * 2 * (size_t)t.A, s));
        if (t.P) WS_CUDA(cudaMemsetAsync(g.gsr, 0, sizeof(double) * 2 * (size_t)t.P, s));
        for (int li = t.L - 1; li >= 0; li--) {
            const int q0 = ctx.lv_ptr_host[li], nq = ctx.lv_ptr_host[li + 1] - q0;
            if (nq <= 0) continue;
            k_pg_level<<<(2 * nq + 127) / 128, 128, 0, s>>>(t, L, d, g, q0, nq);
            count++;
        }
        if (t.M) {
            k_pg_len<<<(t.M + 255) / 256, 256, 0, s>>>(t.M, g);
            count++;
        }
        if (t.P) {
            k_pg_xy<<<(t.P + 255) / 256, 256, 0, s>>>(t.P, t, ctx.pt, g);
            count++;
        }
        WS_CHECK_LAUNCH();
    }
    return count;
}

}  // namespace ws
