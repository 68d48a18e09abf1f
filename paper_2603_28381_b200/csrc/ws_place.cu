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
#include "ws_pg.cuh"

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

// one reverse level, in two launches: k_pg_mem (member terms, thread =
// (member slot u of the level in task order, late column j)) then
// k_pg_level (a PG_G-lane group per net: ordered group sum of the root-slew
// terms -> root winner, LUT partials, gsa, dL/dload -> d_cap).  The bodies
// are ws_pg.cuh's, shared with the fused backward kernel (k_bwd<..., PG>).
constexpr int PG_WARPS = 8, PG_G = 4;

__global__ void __launch_bounds__(256) k_pg_mem(Topo t, PgDev pd, int u_begin, int n2)
{
    const Corner& C = pd.pa[blockIdx.y].d;
    const PlaceCorner& G = pd.pa[blockIdx.y].g;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n2) {
        pdl_wait();
        pdl_trigger();
        return;
    }
    const int u = u_begin + (i >> 1), j = i & 1;
    pg::MemberIn m = pg::member_load(t, pd, C, u, j);
    pdl_wait();          // gsa / gsr of the higher levels
    pdl_trigger();
    pg::member_load_dyn(G, j, m);
    pg::member_finish(t, G, u, j, m, 0, pg::TermsGlobal{&G});
}

struct PdlWait {
    __device__ void operator()() const
    {
        pdl_wait();      // this level's k_pg_mem (member terms), higher levels' gsa
        pdl_trigger();
    }
};

__global__ void __launch_bounds__(PG_WARPS * 32, 3) k_pg_level(Topo t, LutSrc ls, bool use_smem,
                                                               PgDev pd, int q0, int nq)
{
    const Corner& C = pd.pa[blockIdx.y].d;
    const PlaceCorner& G = pd.pa[blockIdx.y].g;
    extern __shared__ __align__(16) unsigned char smem[];
    const LutView L = stage_luts(ls, C.lut_t_flat, use_smem, smem);
    const int lane = threadIdx.x & 31;
    const int wq = (blockIdx.x * PG_WARPS + (threadIdx.x >> 5)) * (32 / PG_G);
    if (wq >= nq) {                              // whole warp idle
        pdl_wait();
        pdl_trigger();
        return;
    }
    const int qi = wq + lane / PG_G;
    pg::pg_net_group<PG_G>(t, L, C, G, qi < nq ? q0 + qi : -1, pg::SrcGlobal{{&G}, &t, &C}, PdlWait());
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

PgDev pg_dev(const Context& ctx, int c0)
{
    return PgDev{ctx.pt.tm_f, ctx.pt.tm_root, ctx.pg_args + c0};
}

// arcs of lower-level targets are read before written: the sweep starts
// from gsa = gsr = 0
void posgrad_reset(Context& ctx, int c0, int nc, cudaStream_t s)
{
    const Topo& t = ctx.t;
    for (int k = c0; k < c0 + nc; k++) {
        const PlaceCorner& g = ctx.place[k];
        if (t.A) WS_CUDA(cudaMemsetAsync(g.gsa, 0, sizeof(double) * 2 * (size_t)t.A, s));
        if (t.P) WS_CUDA(cudaMemsetAsync(g.gsr, 0, sizeof(double) * 2 * (size_t)t.P, s));
    }
}

int launch_posgrad_tail(Context& ctx, int c0, int nc, cudaStream_t s, bool pdl)
{
    const Topo& t = ctx.t;
    const PgArgs* pa = ctx.pg_args + c0;
    int count = 0;
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
    posgrad_reset(ctx, c0, nc, s);
    const PgDev pd = pg_dev(ctx, c0);   // blockIdx.y = corner
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
            launch_pdl(pdl, k_pg_mem, dim3((2 * un + 255) / 256, nc), dim3(256), 0, s, t, pd, ub, 2 * un);
            pdl = true;
            count++;
        }
        launch_pdl(pdl, k_pg_level,
                   dim3((nq + PG_WARPS * (32 / PG_G) - 1) / (PG_WARPS * (32 / PG_G)), nc),
                   dim3(PG_WARPS * 32), lut_bytes, s, t, ls, use_smem, pd, q0, nq);
        pdl = true;
        count++;
    }
    count += launch_posgrad_tail(ctx, c0, nc, s, pdl);
    return count;
}

}  // namespace ws
