// C ABI (include/warpstar.h): context lifetime, value upload, pass launch,
// result download, and the legacy per-level shims.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "ws_internal.h"

struct ws_ctx {
    ws::Context c;
};

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_pin = -1;

template <class F>
int guarded(F&& f)
{
    try {
        f();
        return WS_OK;
    } catch (const ws::Error& e) {
        g_err = e.what();
        g_err_pin = e.pin;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return WS_ERR_NOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return WS_ERR_CUDA;
    }
}

void check_corner(const ws::Context& c, int corner, int n = 1)
{
    if (corner < 0 || n < 1 || corner + n > (int)c.corners.size())
        throw ws::Error(WS_ERR_VALUE, "corner index out of range");
}

int64_t value_len(const ws::Context& c, int field)
{
    const ws::Topo& t = c.t;
    switch (field) {
    case WS_V_MEM_RES: case WS_V_MEM_CAP: return 4ll * t.M;
    case WS_V_ROOT_CAP: return 4ll * t.N;
    case WS_V_LUT_T: return c.lut_t_len;
    case WS_V_PI_ARRIVAL: case WS_V_PI_SLEW: return 4ll * t.I;
    case WS_V_EP_REQUIRED: return 4ll * t.E;
    case WS_V_XY: return 2ll * t.P;
    case WS_V_RES0: case WS_V_CAP0: return 4ll * t.M;
    case WS_V_WIRE: return 8;
    default: throw ws::Error(WS_ERR_VALUE, "unknown value field");
    }
}

bool place_field(int field) { return field >= WS_V_XY && field <= WS_V_WIRE; }

double* value_ptr(ws::Context& c, int corner, int field)
{
    if (place_field(field)) {
        ws::place_enable(c);
        ws::PlaceCorner& g = c.place[corner];
        switch (field) {
        case WS_V_XY: return g.xy;
        case WS_V_RES0: return g.res0;
        case WS_V_CAP0: return g.cap0;
        default: return g.wire;
        }
    }
    ws::Corner& d = c.corners[corner].d;
    switch (field) {
    case WS_V_MEM_RES: return d.mem_res;
    case WS_V_MEM_CAP: return d.mem_cap;
    case WS_V_ROOT_CAP: return d.root_cap;
    case WS_V_LUT_T: return d.lut_t_flat;
    case WS_V_PI_ARRIVAL: return d.pi_arrival;
    case WS_V_PI_SLEW: return d.pi_slew;
    case WS_V_EP_REQUIRED: return d.ep_required;
    default: throw ws::Error(WS_ERR_VALUE, "unknown value field");
    }
}

int64_t state_len(const ws::Context& c, int field)
{
    const ws::Topo& t = c.t;
    switch (field) {
    case WS_F_LOAD: case WS_F_NET_DELAY: case WS_F_IMPULSE: case WS_F_SLEW: case WS_F_ARRIVAL:
    case WS_F_REQUIRED: case WS_F_SLACK: return 4ll * t.P;
    case WS_F_ARC_DELAY: return 4ll * t.A;
    case WS_F_LSE_ARRIVAL: case WS_F_ADJOINT: return 2ll * t.P;
    case WS_F_ARC_WEIGHTS: case WS_F_D_ARC: return 2ll * t.A;
    case WS_F_D_EDGE: return 2ll * t.M;
    case WS_F_SUMMARY: return 3;
    case WS_F_D_RES: case WS_F_D_CAP: return 2ll * t.M;
    case WS_F_D_ROOT_CAP: return 2ll * t.N;
    case WS_F_D_SLEW: case WS_F_D_XY: return 2ll * t.P;
    case WS_F_D_LEN: return t.M;
    case WS_F_D_ARC_SUM: return 2ll * t.A;
    case WS_F_D_EDGE_SUM: return 2ll * t.M;
    default: throw ws::Error(WS_ERR_VALUE, "unknown state field");
    }
}

// the batch-gradient buffers (zeroed once: entries of arcs that feed no net
// root are never written by a pass)
void ensure_dsum(ws::Context& c)
{
    if (c.dsum_arc) return;
    c.dsum_arc = c.val_mem.alloc<double>(2 * (size_t)c.t.A);
    c.dsum_edge = c.val_mem.alloc<double>(2 * (size_t)c.t.M);
    WS_CUDA(cudaMemset(c.dsum_arc, 0, sizeof(double) * 2 * (size_t)std::max(c.t.A, 1)));
    WS_CUDA(cudaMemset(c.dsum_edge, 0, sizeof(double) * 2 * (size_t)std::max(c.t.M, 1)));
}

double* state_ptr(ws::Context& c, int corner, int field)
{
    if (field == WS_F_D_ARC_SUM || field == WS_F_D_EDGE_SUM) {
        ensure_dsum(c);
        return field == WS_F_D_ARC_SUM ? c.dsum_arc : c.dsum_edge;
    }
    if (field >= WS_F_D_RES && field <= WS_F_D_XY) {
        ws::place_enable(c);
        ws::PlaceCorner& g = c.place[corner];
        switch (field) {
        case WS_F_D_RES: return g.d_res;
        case WS_F_D_CAP: return g.d_cap;
        case WS_F_D_ROOT_CAP: return g.d_root_cap;
        case WS_F_D_SLEW: return g.gs;
        case WS_F_D_LEN: return g.g_len;
        default: return g.d_xy;
        }
    }
    ws::Corner& d = c.corners[corner].d;
    switch (field) {
    case WS_F_LOAD: return d.load;
    case WS_F_NET_DELAY: return d.net_delay;
    case WS_F_IMPULSE: return d.impulse;
    case WS_F_SLEW: return d.slew;
    case WS_F_ARRIVAL: return d.arrival;
    case WS_F_REQUIRED: return d.required;
    case WS_F_SLACK: return d.slack;
    case WS_F_ARC_DELAY: return d.arc_delay;
    case WS_F_LSE_ARRIVAL: return d.lse_at;
    case WS_F_ARC_WEIGHTS: return d.weights;
    case WS_F_D_ARC: return d.d_arc;
    case WS_F_D_EDGE: return d.d_edge;
    case WS_F_ADJOINT: return d.adjoint;
    case WS_F_SUMMARY: return d.summary;
    default: throw ws::Error(WS_ERR_VALUE, "unknown state field");
    }
}

cudaStream_t as_stream(void* s, cudaStream_t dflt) { return s ? static_cast<cudaStream_t>(s) : dflt; }

}  // namespace

namespace ws {

// Every corner's copy of a field lives in ONE allocation at a uniform stride
// (corner k = corner 0 + k * stride), so a kernel that maps corners onto
// lanes (the corner-batched level kernels) derives a lane's pointers from
// corner 0's with one multiply-add instead of loading a pointer table.
void alloc_corners(Context& ctx, int n)
{
    const Topo& t = ctx.t;
    Arena& ar = ctx.val_mem;
    CornerStrides& st = ctx.cstride;
    st.P4 = 4 * (long long)t.P; st.P2 = 2 * (long long)t.P;
    st.A4 = 4 * (long long)t.A; st.A2 = 2 * (long long)t.A;
    st.M4 = 4 * (long long)t.M; st.M2 = 2 * (long long)t.M;
    st.N4 = 4 * (long long)t.N; st.LT = ctx.lut_t_len;
    st.I4 = 4 * (long long)t.I; st.E4 = 4 * (long long)t.E;
    const int nl = ctx.tns_plan ? std::max(1, ctx.tns_plan->n_leaves) : 1;
    st.RT = 3 * (long long)(2 * nl);
    st.BP = 8 * (long long)std::max(t.n_parts, 1);
    st.BC = 4 * (long long)std::max(t.n_big, 1);
    ctx.corners.resize(n);
    auto block = [&](long long len, double* Corner::*f, bool zero) {
        double* b = ar.alloc<double>((size_t)n * (size_t)std::max(len, 1ll));
        if (zero) WS_CUDA(cudaMemset(b, 0, sizeof(double) * (size_t)n * (size_t)std::max(len, 1ll)));
        for (int k = 0; k < n; k++) ctx.corners[k].d.*f = b + (size_t)k * (size_t)len;
    };
    block(st.M4, &Corner::mem_res, false);
    block(st.M4, &Corner::mem_cap, false);
    block(st.N4, &Corner::root_cap, false);
    block(st.LT, &Corner::lut_t_flat, false);
    block(st.I4, &Corner::pi_arrival, false);
    block(st.I4, &Corner::pi_slew, false);
    block(st.E4, &Corner::ep_required, false);
    block(st.P4, &Corner::load, false);
    block(st.P4, &Corner::net_delay, false);
    block(st.P4, &Corner::impulse, false);
    block(st.P4, &Corner::slew, false);
    block(st.P4, &Corner::arrival, false);
    block(st.P4, &Corner::required, false);
    // arrays that are not fully rewritten by every pass start defined
    block(st.P4, &Corner::slack, true);
    block(st.A4, &Corner::arc_delay, true);
    block(st.P2, &Corner::lse_at, true);
    block(st.A2, &Corner::weights, true);
    block(st.A2, &Corner::d_arc, true);
    block(st.M2, &Corner::d_edge, true);
    block(st.P2, &Corner::adjoint, true);
    block(st.RT, &Corner::red_tmp, false);
    block(4, &Corner::summary, true);
    block(st.BP, &Corner::big_part, false);
    {
        unsigned* sc = ar.alloc<unsigned>((size_t)n * 4);
        WS_CUDA(cudaMemset(sc, 0, sizeof(unsigned) * (size_t)n * 4));
        unsigned* bc = ar.alloc<unsigned>((size_t)n * (size_t)st.BC);
        WS_CUDA(cudaMemset(bc, 0, sizeof(unsigned) * (size_t)n * (size_t)st.BC));
        for (int k = 0; k < n; k++) {
            Corner& d = ctx.corners[k].d;
            d.sync_ctr = sc + 4 * (size_t)k;
            d.big_ctr = bc + (size_t)k * (size_t)st.BC;
            // tree-net RC scratch only when the design has RC trees (or w != 8
            // is requested later: allocated lazily then)
            d.mem_buf = nullptr;
            d.mem_dbuf = nullptr;
        }
    }
}

void ensure_tree_scratch(Context& ctx)
{
    if (!ctx.corners.empty() && !ctx.corners[0].d.mem_buf) {
        const size_t n = ctx.corners.size(), len = 4 * (size_t)ctx.t.M;
        double* b = ctx.val_mem.alloc<double>(n * len);
        double* db = ctx.val_mem.alloc<double>(n * len);
        for (size_t k = 0; k < n; k++) {
            ctx.corners[k].d.mem_buf = b + k * len;
            ctx.corners[k].d.mem_dbuf = db + k * len;
        }
    }
    std::vector<Corner> v;
    for (auto& cs : ctx.corners) v.push_back(cs.d);
    WS_CUDA(cudaMemcpy(ctx.d_corners, v.data(), sizeof(Corner) * v.size(), cudaMemcpyHostToDevice));
}

void upload_values(Context& ctx, int corner, const ws_design_desc* d)
{
    Corner& c = ctx.corners[corner].d;
    const Topo& t = ctx.t;
    auto up = [&](double* dst, const double* src, size_t n) {
        if (n) WS_CUDA(cudaMemcpy(dst, src, n * sizeof(double), cudaMemcpyHostToDevice));
    };
    up(c.mem_res, d->mem_res, 4 * (size_t)t.M);
    up(c.mem_cap, d->mem_cap, 4 * (size_t)t.M);
    up(c.root_cap, d->root_cap, 4 * (size_t)t.N);
    up(c.lut_t_flat, d->lut_t_flat, (size_t)ctx.lut_t_len);
    up(c.pi_arrival, d->pi_arrival, 4 * (size_t)t.I);
    up(c.pi_slew, d->pi_slew, 4 * (size_t)t.I);
    up(c.ep_required, d->ep_required, 4 * (size_t)t.E);
}

}  // namespace ws

extern "C" {

int ws_abi_version(void) { return WS_ABI_VERSION; }
const char* ws_last_error(void) { return g_err.c_str(); }
int64_t ws_last_error_pin(void) { return g_err_pin; }

int ws_create(const ws_design_desc* d, int n_corners, ws_ctx** out)
{
    ws_ctx* h = nullptr;
    int rc = guarded([&] {
        if (!d || !out) throw ws::Error(WS_ERR_VALUE, "null argument");
        if (n_corners < 1) throw ws::Error(WS_ERR_VALUE, "n_corners must be >= 1");
        if (!(d->clock_period > 0.0)) throw ws::Error(WS_ERR_VALUE, "clock_period must be positive");
        h = new ws_ctx();
        ws::Context& c = h->c;
        c.clock_period = d->clock_period;
        {
            const char* e = getenv("WS_LUT_GLOBAL");
            c.lut_global = e && e[0] == '1';
            const char* r = getenv("WS_RC_SCHEME");
            c.rc_cte = r && std::string(r) == "cte";
            c.rc_pin_order = r && std::string(r) == "pin";
            const char* sp = getenv("WS_SPLIT");
            c.split_min = sp ? atoi(sp) : 8;   // measured: 16 corners 11.21 -> 10.56 ms, 8 corners 5.83 -> 5.28 ms
            const char* spp = getenv("WS_SPLIT_PARTS");
            c.split_parts = spp ? atoi(spp) : 2;
            const char* rr = getenv("WS_RC_ROOTS");
            c.rc_roots = !rr ? 0 : std::string(rr) == "net" ? -1 : std::string(rr) == "fold" ? 1 : 0;
        }
        // blocking streams: with a NULL stream argument the context's work is
        // ordered after (and before) work on the legacy default stream, the
        // stream a caller that never chose one (torch's default) writes on
        WS_CUDA(cudaStreamCreateWithFlags(&c.s_main, cudaStreamDefault));
        WS_CUDA(cudaStreamCreateWithFlags(&c.s_grad, cudaStreamDefault));
        ws::build_topology(c, d);
        ws::summary_plan_init(c);
        ws::alloc_corners(c, n_corners);
        for (int k = 0; k < n_corners; k++) ws::upload_values(c, k, d);
        c.d_corners = c.topo_mem.alloc<ws::Corner>(n_corners);
        ws::ensure_tree_scratch(c);   // tree-net RC and big-net fold scratch
        std::vector<ws::Corner> v;
        for (auto& cs : c.corners) v.push_back(cs.d);
        WS_CUDA(cudaMemcpy(c.d_corners, v.data(), sizeof(ws::Corner) * v.size(), cudaMemcpyHostToDevice));
        WS_CUDA(cudaDeviceSynchronize());
    });
    if (rc != WS_OK) {
        if (h) ws_destroy(h);
        return rc;
    }
    *out = h;
    return WS_OK;
}

void ws_destroy(ws_ctx* h)
{
    if (!h) return;
    ws::Context& c = h->c;
    cudaDeviceSynchronize();
    for (auto& g : c.graphs) cudaGraphExecDestroy(g.exec);
    for (auto e : c.events) cudaEventDestroy(e);
    for (auto e : c.pg_events) cudaEventDestroy(e);
    for (auto e : c.timed_events) cudaEventDestroy(e);
    ws::summary_plan_free(c);
    c.val_mem.release();
    c.topo_mem.release();
    c.scratch.release();
    if (c.s_main) cudaStreamDestroy(c.s_main);
    if (c.s_grad) cudaStreamDestroy(c.s_grad);
    for (cudaStream_t x : c.split_streams) cudaStreamDestroy(x);
    delete h;
}

int ws_dims(ws_ctx* h, int64_t* dims)
{
    return guarded([&] {
        if (!h || !dims) throw ws::Error(WS_ERR_VALUE, "null argument");
        const ws::Topo& t = h->c.t;
        const int64_t v[WS_DIMS_LEN] = {t.P, t.N, t.M, t.A, t.I, t.E, t.L, t.NL,
                                        (int64_t)h->c.corners.size(), t.max_in, t.max_m};
        memcpy(dims, v, sizeof(v));
    });
}

int64_t ws_topology_len(ws_ctx* h, int field)
{
    int64_t n = -1;
    int rc = guarded([&] {
        if (!h) throw ws::Error(WS_ERR_VALUE, "null context");
        n = ws::topo_field_len(h->c, field);
    });
    return rc == WS_OK ? n : -1;
}

int ws_get_topology(ws_ctx* h, int field, int64_t* dst)
{
    return guarded([&] {
        if (!h || !dst) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::topo_field_to_host(h->c, field, dst);
    });
}

int ws_set_values(ws_ctx* h, int corner, int field, const double* src, int src_on_device, void* stream)
{
    return guarded([&] {
        if (!h || !src) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::Context& c = h->c;
        check_corner(c, corner);
        const int64_t n = value_len(c, field);
        cudaStream_t s = as_stream(stream, c.s_main);
        if (n)
            WS_CUDA(cudaMemcpyAsync(value_ptr(c, corner, field), src, (size_t)n * sizeof(double),
                                    src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        if (!stream) WS_CUDA(cudaStreamSynchronize(s));
    });
}

int ws_perturb_values(ws_ctx* h, int corner, int base_corner, uint64_t seed, double sigma,
                      void* stream)
{
    return guarded([&] {
        if (!h) throw ws::Error(WS_ERR_VALUE, "null context");
        ws::Context& c = h->c;
        check_corner(c, corner);
        check_corner(c, base_corner);
        if (!(sigma >= 0.0 && sigma < 1.0 / 3.0))
            throw ws::Error(WS_ERR_VALUE, "sigma must be in [0, 1/3) so every factor stays positive");
        cudaStream_t s = as_stream(stream, c.s_main);
        if (corner != base_corner) {
            const ws::Corner& a = c.corners[base_corner].d;
            const ws::Corner& b = c.corners[corner].d;
            auto cp = [&](double* dst, const double* src, size_t n) {
                if (n) WS_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
            };
            cp(b.lut_t_flat, a.lut_t_flat, (size_t)c.lut_t_len);
            cp(b.pi_arrival, a.pi_arrival, 4 * (size_t)c.t.I);
            cp(b.pi_slew, a.pi_slew, 4 * (size_t)c.t.I);
            cp(b.ep_required, a.ep_required, 4 * (size_t)c.t.E);
        }
        ws::launch_perturb(c, corner, base_corner, (unsigned long long)seed, sigma, s);
        if (!stream) WS_CUDA(cudaStreamSynchronize(s));
    });
}

int ws_run(ws_ctx* h, int corner0, int n_corners, uint32_t flags, double gamma, int loss_kind,
           int reduce_width, int granularity, void* stream, void* stream_grad)
{
    return guarded([&] {
        if (!h) throw ws::Error(WS_ERR_VALUE, "null context");
        ws::Context& c = h->c;
        check_corner(c, corner0, n_corners);
        if ((flags & (WS_RUN_LSE | WS_RUN_GRAD)) && !(gamma > 0.0 && gamma < __builtin_huge_val()))
            throw ws::Error(WS_ERR_VALUE, "gamma must be positive and finite");
        if (loss_kind != WS_LOSS_HINGE && loss_kind != WS_LOSS_SOFTPLUS)
            throw ws::Error(WS_ERR_VALUE, "unknown loss kind");
        if (reduce_width < 0 || reduce_width > 32 || (reduce_width & (reduce_width - 1)))
            throw ws::Error(WS_ERR_VALUE, "reduce_width must be 0 (np.add.reduceat order) or a power "
                                          "of two in [1, 32]");
        if (granularity < 1) throw ws::Error(WS_ERR_VALUE, "granularity must be >= 1");
        cudaStream_t s = as_stream(stream, c.s_main);
        cudaStream_t g = as_stream(stream_grad, c.s_grad);
        const unsigned need = WS_RUN_HARD | WS_RUN_LSE | WS_RUN_GRAD;
        if ((flags & WS_RUN_POSGRAD) && (flags & need) != need)
            throw ws::Error(WS_ERR_STATE, "WS_RUN_POSGRAD needs HARD|LSE|GRAD in the same run");
        if ((flags & WS_RUN_TIMED) && (flags & (WS_RUN_TWO_STREAM | WS_RUN_PERSISTENT | WS_RUN_GRAPH)))
            throw ws::Error(WS_ERR_VALUE,
                            "WS_RUN_TIMED needs the sequential or fused mode without graph capture");
        if ((flags & WS_RUN_POSGRAD) && (flags & WS_RUN_PERSISTENT))
            throw ws::Error(WS_ERR_VALUE, "WS_RUN_POSGRAD is not available with WS_RUN_PERSISTENT");
        if (flags & (WS_RUN_WIRE | WS_RUN_POSGRAD)) ws::place_enable(c);
        if (flags & WS_RUN_CORNER_SUM) {
            if (!(flags & WS_RUN_GRAD))
                throw ws::Error(WS_ERR_STATE, "WS_RUN_CORNER_SUM needs WS_RUN_GRAD in the same run");
            if (n_corners > 16)
                throw ws::Error(WS_ERR_VALUE, "WS_RUN_CORNER_SUM sums at most 16 corners per run");
            ensure_dsum(c);
        }
        if (flags & WS_RUN_GRAPH) {
            // graph cache: one executable per (flags, corners, loss, granularity,
            // reduce width), least recently used first out beyond
            // kGraphCache entries.  A new gamma keeps the executable: the
            // pass is re-captured and its kernel parameters swapped in by
            // cudaGraphExecUpdate (same topology), no re-instantiation.
            const unsigned key = flags & ~WS_RUN_GRAPH;
            const int gran = granularity * 64 + reduce_width;
            auto capture = [&]() {
                cudaStream_t cap, capg;
                WS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
                WS_CUDA(cudaStreamCreateWithFlags(&capg, cudaStreamNonBlocking));
                WS_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
                ws::run_pass(c, corner0, n_corners, key, gamma, loss_kind, granularity, cap, capg,
                             reduce_width);
                cudaGraph_t graph;
                WS_CUDA(cudaStreamEndCapture(cap, &graph));
                cudaStreamDestroy(cap);
                cudaStreamDestroy(capg);
                return graph;
            };
            size_t hit = c.graphs.size();
            for (size_t i = 0; i < c.graphs.size(); i++) {
                const auto& e = c.graphs[i];
                if (e.key == key && e.c0 == corner0 && e.nc == n_corners && e.loss == loss_kind &&
                    e.gran == gran) hit = i;
            }
            if (hit < c.graphs.size() && c.graphs[hit].gamma != gamma) {
                cudaGraph_t graph = capture();
                cudaGraphExecUpdateResultInfo info;
                const cudaError_t ue = cudaGraphExecUpdate(c.graphs[hit].exec, graph, &info);
                if (ue != cudaSuccess) {       // topology changed: a fresh executable
                    cudaGetLastError();
                    cudaGraphExec_t exec;
                    WS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
                    cudaGraphExecDestroy(c.graphs[hit].exec);
                    c.graphs[hit].exec = exec;
                }
                WS_CUDA(cudaGraphDestroy(graph));
                c.graphs[hit].gamma = gamma;
                c.graph_launches[hit] = c.launches_last_run;
            } else if (hit == c.graphs.size()) {
                cudaGraph_t graph = capture();
                cudaGraphExec_t exec;
                WS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
                WS_CUDA(cudaGraphDestroy(graph));
                if (c.graphs.size() >= ws::kGraphCache) {   // evict the least recently used
                    cudaGraphExecDestroy(c.graphs.front().exec);
                    c.graphs.erase(c.graphs.begin());
                    c.graph_launches.erase(c.graph_launches.begin());
                }
                c.graphs.push_back({key, corner0, n_corners, gamma, loss_kind, gran, exec});
                c.graph_launches.push_back(c.launches_last_run);
                hit = c.graphs.size() - 1;
            }
            // most recently used last
            std::rotate(c.graphs.begin() + hit, c.graphs.begin() + hit + 1, c.graphs.end());
            std::rotate(c.graph_launches.begin() + hit, c.graph_launches.begin() + hit + 1,
                        c.graph_launches.end());
            WS_CUDA(cudaGraphLaunch(c.graphs.back().exec, s));
            c.launches_last_run = c.graph_launches.back();
        } else {
            ws::run_pass(c, corner0, n_corners, flags, gamma, loss_kind, granularity, s, g,
                         reduce_width);
        }
        if (flags & WS_RUN_HARD)
            for (int k = 0; k < n_corners; k++) c.corners[corner0 + k].has_lse = false;
        if (flags & WS_RUN_LSE)
            for (int k = 0; k < n_corners; k++) c.corners[corner0 + k].has_lse = true;
        if (!stream) WS_CUDA(cudaStreamSynchronize(s));
    });
}

int ws_run_kernel(ws_ctx* h, int corner, int kind, int level, double gamma, int loss_kind,
                  int reduce_width, void* stream)
{
    return guarded([&] {
        if (!h) throw ws::Error(WS_ERR_VALUE, "null context");
        ws::Context& c = h->c;
        check_corner(c, corner);
        if ((kind == 3 || kind == 4 || kind == 5) && !(gamma > 0.0 && gamma < __builtin_huge_val()))
            throw ws::Error(WS_ERR_VALUE, "gamma must be positive and finite");
        if (loss_kind != WS_LOSS_HINGE && loss_kind != WS_LOSS_SOFTPLUS)
            throw ws::Error(WS_ERR_VALUE, "unknown loss kind");
        if (reduce_width < 0 || reduce_width > 32 || (reduce_width & (reduce_width - 1)))
            throw ws::Error(WS_ERR_VALUE, "reduce_width must be 0 (np.add.reduceat order) or a power "
                                          "of two in [1, 32]");
        cudaStream_t s = as_stream(stream, c.s_main);
        ws::run_kernel(c, corner, kind, level, gamma, loss_kind, reduce_width, s);
        if (!stream) WS_CUDA(cudaStreamSynchronize(s));
    });
}

int ws_set_state(ws_ctx* h, int corner, int field, const double* src, int src_on_device, void* stream)
{
    return guarded([&] {
        if (!h || !src) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::Context& c = h->c;
        check_corner(c, corner);
        const int64_t n = state_len(c, field);
        cudaStream_t s = as_stream(stream, c.s_main);
        if (n)
            WS_CUDA(cudaMemcpyAsync(state_ptr(c, corner, field), src, (size_t)n * sizeof(double),
                                    src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        if (!stream) WS_CUDA(cudaStreamSynchronize(s));
    });
}

int ws_get(ws_ctx* h, int corner, int field, double* dst, int dst_on_device, void* stream)
{
    return guarded([&] {
        if (!h || !dst) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::Context& c = h->c;
        check_corner(c, corner);
        const int64_t n = state_len(c, field);
        cudaStream_t s = as_stream(stream, c.s_main);
        if (n)
            WS_CUDA(cudaMemcpyAsync(dst, state_ptr(c, corner, field), (size_t)n * sizeof(double),
                                    dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        WS_CUDA(cudaStreamSynchronize(s));
    });
}

int ws_device_ptr(ws_ctx* h, int corner, int field, void** dptr, int64_t* n_elems)
{
    return guarded([&] {
        if (!h || !dptr) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::Context& c = h->c;
        check_corner(c, corner);
        *dptr = state_ptr(c, corner, field);
        if (n_elems) *n_elems = state_len(c, field);
    });
}

int ws_value_ptr(ws_ctx* h, int corner, int field, void** dptr, int64_t* n_elems)
{
    return guarded([&] {
        if (!h || !dptr) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::Context& c = h->c;
        check_corner(c, corner);
        *dptr = value_ptr(c, corner, field);
        if (n_elems) *n_elems = value_len(c, field);
    });
}

int ws_summary(ws_ctx* h, int corner, double* out, void* stream)
{
    return guarded([&] {
        if (!h || !out) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::Context& c = h->c;
        check_corner(c, corner);
        cudaStream_t s = as_stream(stream, c.s_main);
        WS_CUDA(cudaMemcpyAsync(out, c.corners[corner].d.summary, 3 * sizeof(double),
                                cudaMemcpyDeviceToHost, s));
        WS_CUDA(cudaStreamSynchronize(s));
    });
}

int ws_last_launch_count(ws_ctx* h) { return h ? h->c.launches_last_run : -1; }

int ws_kernel_times(ws_ctx* h, int* kind, int* level, float* ms, int cap)
{
    int n = -1;
    const int rc = guarded([&] {
        if (!h || (cap > 0 && (!kind || !level || !ms))) throw ws::Error(WS_ERR_VALUE, "null argument");
        ws::Context& c = h->c;
        n = std::max(0, std::min(cap, c.timed_n - 1));
        if (c.timed_n > 0) WS_CUDA(cudaEventSynchronize(c.timed_events[c.timed_n - 1]));
        for (int i = 0; i < n; i++) {
            float t = 0.f;
            WS_CUDA(cudaEventElapsedTime(&t, c.timed_events[i], c.timed_events[i + 1]));
            kind[i] = c.timed_kind[i + 1];
            level[i] = c.timed_level[i + 1];
            ms[i] = t;
        }
    });
    return rc == WS_OK ? n : -1;
}

int ws_set_probe(ws_ctx* h, void* device_buf)
{
    return guarded([&] {
        if (!h) throw ws::Error(WS_ERR_VALUE, "null context");
        h->c.t.probe = static_cast<unsigned long long*>(device_buf);
    });
}

// ---------------------------------------------------------------------------
// legacy per-level shims

namespace {

struct ShimArena {
    ws::Arena ar;
    ~ShimArena() { ar.release(); }
    int* i32(const int64_t* src, int64_t n)
    {
        std::vector<int> v((size_t)std::max<int64_t>(n, 1));
        for (int64_t i = 0; i < n; i++) {
            if (src[i] < INT32_MIN || src[i] > INT32_MAX)
                throw ws::Error(WS_ERR_VALUE, "index exceeds the int32 range");
            v[(size_t)i] = (int)src[i];
        }
        int* d = ar.alloc<int>(v.size());
        WS_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
        return d;
    }
    double* f64(const double* src, int64_t n)
    {
        double* d = ar.alloc<double>((size_t)std::max<int64_t>(n, 1));
        if (n) WS_CUDA(cudaMemcpy(d, src, (size_t)n * sizeof(double), cudaMemcpyHostToDevice));
        return d;
    }
    ws::Corner* corner(const ws::Corner& c)
    {
        ws::Corner* d = ar.alloc<ws::Corner>(1);
        WS_CUDA(cudaMemcpy(d, &c, sizeof(c), cudaMemcpyHostToDevice));
        return d;
    }
};

void back(double* dst, const double* src, int64_t n)
{
    if (n) WS_CUDA(cudaMemcpy(dst, src, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost));
}

}  // namespace

int ws_rc_level(int64_t n_lv, const int64_t* nets, int64_t n_nets, const int64_t* net_ptr,
                const int64_t* net_root, const double* root_cap, int64_t n_mem,
                const int64_t* mem_pin, const int64_t* mem_parent_loc, const double* mem_res,
                const double* mem_cap, int64_t n_pins, const int64_t* root_net_of_pin,
                double* load, double* net_delay, double* impulse, int reduce_width)
{
    return guarded([&] {
        if (reduce_width < 0 || reduce_width > 32 || (reduce_width & (reduce_width - 1)))
            throw ws::Error(WS_ERR_VALUE, "reduce_width must be 0 (np.add.reduceat order) or a power "
                                          "of two in [1, 32]");
        ShimArena sa;
        ws::Topo t{};
        t.N = (int)n_nets; t.M = (int)n_mem; t.P = (int)n_pins;
        t.net_ptr = sa.i32(net_ptr, n_nets + 1);
        t.net_root = sa.i32(net_root, n_nets);
        t.mem_pin = sa.i32(mem_pin, n_mem);
        t.mem_parent_loc = sa.i32(mem_parent_loc, n_mem);
        t.root_net_of_pin = sa.i32(root_net_of_pin, n_pins);
        std::vector<int64_t> tree((size_t)std::max<int64_t>(n_nets, 1), 0);
        for (int64_t n = 0; n < n_nets; n++)
            for (int64_t f = net_ptr[n]; f < net_ptr[n + 1]; f++)
                if (mem_parent_loc[f] > 0) tree[(size_t)n] = 1;
        t.net_tree = sa.i32(tree.data(), n_nets);
        int* list = sa.i32(nets, n_lv);
        ws::Corner c{};
        c.root_cap = sa.f64(root_cap, 4 * n_nets);
        c.mem_res = sa.f64(mem_res, 4 * n_mem);
        c.mem_cap = sa.f64(mem_cap, 4 * n_mem);
        c.load = sa.f64(load, 4 * n_pins);
        c.net_delay = sa.f64(net_delay, 4 * n_pins);
        c.impulse = sa.f64(impulse, 4 * n_pins);
        c.mem_buf = sa.ar.alloc<double>(4 * (size_t)std::max<int64_t>(n_mem, 1));
        c.mem_dbuf = sa.ar.alloc<double>(4 * (size_t)std::max<int64_t>(n_mem, 1));
        ws::launch_rc_list(t, sa.corner(c), list, (int)n_lv, reduce_width, 0);
        WS_CUDA(cudaDeviceSynchronize());
        back(load, c.load, 4 * n_pins);
        back(net_delay, c.net_delay, 4 * n_pins);
        back(impulse, c.impulse, 4 * n_pins);
    });
}

int ws_forward_level(int64_t n_lv, const int64_t* nets, int64_t n_nets, const int64_t* net_ptr,
                     const int64_t* net_root, const int64_t* root_kind, int64_t n_mem,
                     const int64_t* mem_pin, const int64_t* net_in_ptr, const int64_t* net_in_arc,
                     int64_t n_arcs, const int64_t* arc_from, const int64_t* arc_dlut,
                     const int64_t* arc_slut, int64_t n_luts, const int64_t* lut_s_ptr,
                     const int64_t* lut_l_ptr, const int64_t* lut_t_ptr, const double* lut_s_flat,
                     const double* lut_l_flat, const double* lut_t_flat, int64_t n_pins,
                     const double* load, const double* net_delay, const double* impulse,
                     double* slew, double* arrival, double* arc_delay)
{
    return guarded([&] {
        ShimArena sa;
        ws::Topo t{};
        t.N = (int)n_nets; t.M = (int)n_mem; t.P = (int)n_pins; t.A = (int)n_arcs; t.NL = (int)n_luts;
        t.lv_nets = sa.i32(nets, n_lv);
        t.net_ptr = sa.i32(net_ptr, n_nets + 1);
        t.net_root = sa.i32(net_root, n_nets);
        t.root_kind = sa.i32(root_kind, n_nets);
        t.mem_pin = sa.i32(mem_pin, n_mem);
        t.net_in_ptr = sa.i32(net_in_ptr, n_nets + 1);
        const int64_t n_in = n_nets > 0 ? net_in_ptr[n_nets] : 0;
        t.net_in_arc = sa.i32(net_in_arc, n_in);
        t.arc_from = sa.i32(arc_from, n_arcs);
        t.arc_dlut = sa.i32(arc_dlut, 4 * n_arcs);
        t.arc_slut = sa.i32(arc_slut, 4 * n_arcs);
        t.lut_s_ptr = sa.i32(lut_s_ptr, n_luts + 1);
        t.lut_l_ptr = sa.i32(lut_l_ptr, n_luts + 1);
        t.lut_t_ptr = sa.i32(lut_t_ptr, n_luts + 1);
        const int64_t sl = n_luts ? lut_s_ptr[n_luts] : 0, ll = n_luts ? lut_l_ptr[n_luts] : 0,
                      tl = n_luts ? lut_t_ptr[n_luts] : 0;
        t.lut_s_flat = sa.f64(lut_s_flat, sl);
        t.lut_l_flat = sa.f64(lut_l_flat, ll);
        ws::Corner c{};
        c.lut_t_flat = sa.f64(lut_t_flat, tl);
        c.load = sa.f64(load, 4 * n_pins);
        c.net_delay = sa.f64(net_delay, 4 * n_pins);
        c.impulse = sa.f64(impulse, 4 * n_pins);
        c.slew = sa.f64(slew, 4 * n_pins);
        c.arrival = sa.f64(arrival, 4 * n_pins);
        c.arc_delay = sa.f64(arc_delay, 4 * n_arcs);
        ws::launch_fwd_list(t, sa.corner(c), (int)n_lv, (int)sl, (int)ll, (int)tl, 0);
        WS_CUDA(cudaDeviceSynchronize());
        back(slew, c.slew, 4 * n_pins);
        back(arrival, c.arrival, 4 * n_pins);
        back(arc_delay, c.arc_delay, 4 * n_arcs);
    });
}

int ws_backward_level(int64_t n_lv, const int64_t* nets, int64_t n_nets, const int64_t* net_ptr,
                      const int64_t* net_root, int64_t n_mem, const int64_t* mem_pin,
                      const int64_t* mem_out_ptr, const int64_t* mem_out_arc, int64_t n_arcs,
                      const int64_t* arc_to, int64_t n_pins, const double* net_delay,
                      double* required, const double* arc_delay)
{
    return guarded([&] {
        ShimArena sa;
        ws::Topo t{};
        t.N = (int)n_nets; t.M = (int)n_mem; t.P = (int)n_pins; t.A = (int)n_arcs;
        t.lv_nets = sa.i32(nets, n_lv);
        t.net_ptr = sa.i32(net_ptr, n_nets + 1);
        t.net_root = sa.i32(net_root, n_nets);
        t.mem_pin = sa.i32(mem_pin, n_mem);
        t.mem_out_ptr = sa.i32(mem_out_ptr, n_mem + 1);
        const int64_t n_out = n_mem > 0 ? mem_out_ptr[n_mem] : 0;
        t.mem_out_arc = sa.i32(mem_out_arc, n_out);
        t.arc_to = sa.i32(arc_to, n_arcs);
        ws::Corner c{};
        c.net_delay = sa.f64(net_delay, 4 * n_pins);
        c.required = sa.f64(required, 4 * n_pins);
        c.arc_delay = sa.f64(arc_delay, 4 * n_arcs);
        ws::launch_bwd_list(t, sa.corner(c), (int)n_lv, 0);
        WS_CUDA(cudaDeviceSynchronize());
        back(required, c.required, 4 * n_pins);
    });
}

}  // extern "C"
