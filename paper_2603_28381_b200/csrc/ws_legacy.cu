// Legacy per-level kernels behind the reference's raw level-kernel ABI
// (ws_rc_level / ws_forward_level / ws_backward_level; _kernels.pyx:84-249).
//
// One warp per net over an arbitrary caller-supplied net list, lane =
// 4*slot + cond; reductions ordered so results are the reference's bit for
// bit (earlier slot wins ties; RC root load = 8 strided partials + pairwise
// tree by shfl_down 4/8/16).  The production pass (ws_pass.cu) uses the
// level-major task layout instead; both are parity-tested against the golden
// fixtures.
#include <algorithm>

#include "ws_internal.h"

namespace ws {
namespace legacy {

constexpr int WPB = 4;
constexpr int NET_TPB = 32 * WPB;
constexpr double INF = __builtin_huge_val();

__device__ void rc_net_seq(const Topo& t, const Corner& C, int net, int c, int w)
{
    const int s = t.net_ptr[net], e = t.net_ptr[net + 1], m = e - s, root = t.net_root[net];
    double* buf = C.mem_buf + (size_t)s * 4 + c;     // stride 4
    double* dbuf = C.mem_dbuf + (size_t)s * 4 + c;
    for (int k = 0; k < m; k++) buf[4 * k] = C.mem_cap[(size_t)(s + k) * 4 + c];
    for (int k = m - 1; k > 0; k--) {
        const int pl = t.mem_parent_loc[s + k];
        if (pl > 0) buf[4 * (pl - 1)] = __dadd_rn(buf[4 * (pl - 1)], buf[4 * k]);
    }
    double partials[32];
    for (int lane = 0; lane < w; lane++) {
        double p = 0.0;
        for (int i = lane; i < m; i += w) p = __dadd_rn(p, buf[4 * i]);
        partials[lane] = p;
    }
    for (int stride = 1; stride < w; stride *= 2)
        for (int lane = 0; lane < w; lane += 2 * stride)
            partials[lane] = __dadd_rn(partials[lane], partials[lane + stride]);
    C.load[(size_t)root * 4 + c] = __dadd_rn(C.root_cap[(size_t)net * 4 + c], partials[0]);
    for (int k = 0; k < m; k++) {
        const int pl = t.mem_parent_loc[s + k];
        const double dp = pl == 0 ? 0.0 : dbuf[4 * (pl - 1)];
        const double tt = __dmul_rn(C.mem_res[(size_t)(s + k) * 4 + c], buf[4 * k]);
        dbuf[4 * k] = __dadd_rn(dp, tt);
    }
    for (int k = 0; k < m; k++) {
        const double r = C.mem_res[(size_t)(s + k) * 4 + c];
        const double cp = C.mem_cap[(size_t)(s + k) * 4 + c];
        const double d = dbuf[4 * k];
        const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r), cp), d), __dmul_rn(d, d));
        const double imp = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
        const int pin = t.mem_pin[s + k];
        if (t.root_net_of_pin[pin] < 0) C.load[(size_t)pin * 4 + c] = buf[4 * k];
        C.net_delay[(size_t)pin * 4 + c] = d;
        C.impulse[(size_t)pin * 4 + c] = imp;
    }
}

// star net, reduce_width 8: lane (y, c) owns members i == y (mod 8)
__device__ __forceinline__ void rc_net_star8(const Topo& t, const Corner& C, int net, int lane)
{
    const int y = lane >> 2, c = lane & 3;
    const int s = t.net_ptr[net], e = t.net_ptr[net + 1], m = e - s;
    double p = 0.0;
    for (int i = y; i < m; i += 8) {
        const size_t f = (size_t)(s + i);
        const double b = C.mem_cap[f * 4 + c];
        const double r = C.mem_res[f * 4 + c];
        p = __dadd_rn(p, b);
        const double d = __dadd_rn(0.0, __dmul_rn(r, b));
        const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r), b), d), __dmul_rn(d, d));
        const double imp = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
        const int pin = t.mem_pin[f];
        if (t.root_net_of_pin[pin] < 0) C.load[(size_t)pin * 4 + c] = b;
        C.net_delay[(size_t)pin * 4 + c] = d;
        C.impulse[(size_t)pin * 4 + c] = imp;
    }
#pragma unroll
    for (int st = 1; st < 8; st <<= 1) {
        const double po = __shfl_down_sync(WS_FULL, p, 4 * st);
        if ((y & (2 * st - 1)) == 0) p = __dadd_rn(p, po);
    }
    if (y == 0) C.load[(size_t)t.net_root[net] * 4 + c] = __dadd_rn(C.root_cap[(size_t)net * 4 + c], p);
}

__global__ void __launch_bounds__(NET_TPB) k_rc(Topo t, const Corner* __restrict__ cs, int c0, int w,
                                               const int* __restrict__ list, int n)
{
    const Corner C = cs[c0 + blockIdx.y];
    const int q = blockIdx.x * WPB + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= n) return;
    const int net = list ? list[q] : q;
    if (w == 8 && !t.net_tree[net]) {
        rc_net_star8(t, C, net, lane);
    } else if (lane < 4) {
        rc_net_seq(t, C, net, lane, w);
    }
}

__device__ __forceinline__ void fwd_hard_net(const Topo& t, const Corner& C, const LutView& L,
                                             int net, int lane)
{
    const int slot = lane >> 2, c = lane & 3;
    const bool late = c >= 2;
    const int root = t.net_root[net];
    double at_r, sl_r;
    if (t.root_kind[net] == ROOT_ARC) {
        const int a0 = t.net_in_ptr[net], a1 = t.net_in_ptr[net + 1];
        const double ld = C.load[(size_t)root * 4 + c];
        double best = late ? -INF : INF;
        int wa = -1;
        for (int base = a0; base < a1; base += 8) {
            const int q = base + slot;
            double v = late ? -INF : INF;
            int a = -1;
            if (q < a1) {
                a = t.net_in_arc[q];
                const int fp = t.arc_from[a];
                const double d = lut_interp(L, t.arc_dlut[a * 4 + c], C.slew[(size_t)fp * 4 + c], ld);
                C.arc_delay[(size_t)a * 4 + c] = d;
                v = __dadd_rn(C.arrival[(size_t)fp * 4 + c], d);
            }
#pragma unroll
            for (int st = 1; st < 8; st <<= 1) {
                const double vo = __shfl_down_sync(WS_FULL, v, 4 * st);
                const int ao = __shfl_down_sync(WS_FULL, a, 4 * st);
                if ((slot & (2 * st - 1)) == 0 && later_wins(late, v, vo)) { v = vo; a = ao; }
            }
            if (later_wins(late, best, v)) { best = v; wa = a; }
        }
        best = __shfl_sync(WS_FULL, best, c);
        wa = __shfl_sync(WS_FULL, wa, c);
        double sl = 0.0;
        if (slot == 0) {
            sl = lut_interp(L, t.arc_slut[wa * 4 + c], C.slew[(size_t)t.arc_from[wa] * 4 + c], ld);
            C.arrival[(size_t)root * 4 + c] = best;
            C.slew[(size_t)root * 4 + c] = sl;
        }
        at_r = best;
        sl_r = __shfl_sync(WS_FULL, sl, c);
    } else {
        at_r = C.arrival[(size_t)root * 4 + c];
        sl_r = C.slew[(size_t)root * 4 + c];
    }
    const int s = t.net_ptr[net], e = t.net_ptr[net + 1];
    for (int k = s + slot; k < e; k += 8) {
        const size_t pin = (size_t)t.mem_pin[k];
        C.arrival[pin * 4 + c] = __dadd_rn(at_r, C.net_delay[pin * 4 + c]);
        const double ii = C.impulse[pin * 4 + c];
        C.slew[pin * 4 + c] = __dsqrt_rn(__dadd_rn(__dmul_rn(sl_r, sl_r), __dmul_rn(ii, ii)));
    }
}

__global__ void __launch_bounds__(NET_TPB) k_fwd(Topo t, LutSrc ls, const Corner* __restrict__ cs,
                                                 int c0, int lv0, int lv1, bool use_smem)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const Corner C = cs[c0 + blockIdx.y];
    LutView L;
    L = stage_luts(ls, C.lut_t_flat, use_smem, smem);
    const int q = lv0 + blockIdx.x * WPB + (threadIdx.x >> 5);
    if (q >= lv1) return;
    const int net = t.lv_nets[q];
    const int lane = threadIdx.x & 31;
    fwd_hard_net(t, C, L, net, lane);
}

__device__ __forceinline__ void bwd_hard_net(const Topo& t, const Corner& C, int net, int lane)
{
    const int slot = lane >> 2, c = lane & 3;
    const bool mx = c < 2;   // early: max, late: min
    const int s = t.net_ptr[net], e = t.net_ptr[net + 1], root = t.net_root[net];
    double rr = C.required[(size_t)root * 4 + c];
    for (int base = s; base < e; base += 8) {
        const int k = base + slot;
        double v = mx ? -INF : INF;
        if (k < e) {
            const size_t pin = (size_t)t.mem_pin[k];
            double r = C.required[pin * 4 + c];
            for (int q = t.mem_out_ptr[k]; q < t.mem_out_ptr[k + 1]; q++) {
                const int a = t.mem_out_arc[q];
                const double vv = __dsub_rn(C.required[(size_t)t.arc_to[a] * 4 + c],
                                            C.arc_delay[(size_t)a * 4 + c]);
                if (later_wins(mx, r, vv)) r = vv;
            }
            C.required[pin * 4 + c] = r;
            v = __dsub_rn(r, C.net_delay[pin * 4 + c]);
        }
#pragma unroll
        for (int st = 1; st < 8; st <<= 1) {
            const double vo = __shfl_down_sync(WS_FULL, v, 4 * st);
            if ((slot & (2 * st - 1)) == 0 && later_wins(mx, v, vo)) v = vo;
        }
        if (later_wins(mx, rr, v)) rr = v;
    }
    if (slot == 0) C.required[(size_t)root * 4 + c] = rr;
}

__global__ void __launch_bounds__(NET_TPB) k_bwd(Topo t, const Corner* __restrict__ cs, int c0,
                                                 int lv0, int lv1)
{
    const Corner C = cs[c0 + blockIdx.y];
    const int q = lv0 + blockIdx.x * WPB + (threadIdx.x >> 5);
    if (q >= lv1) return;
    const int net = t.lv_nets[q];
    const int lane = threadIdx.x & 31;
    bwd_hard_net(t, C, net, lane);
}

}  // namespace legacy

void launch_rc_list(const Topo& t, const Corner* dcs, const int* list, int n, int w, cudaStream_t s)
{
    if (n <= 0) return;
    legacy::k_rc<<<dim3((n + legacy::WPB - 1) / legacy::WPB, 1), legacy::NET_TPB, 0, s>>>(t, dcs, 0, w, list, n);
    WS_CHECK_LAUNCH();
}

void launch_fwd_list(const Topo& t, const Corner* dcs, int n, int lut_s_len, int lut_l_len,
                     int lut_t_len, cudaStream_t s)
{
    if (n <= 0) return;
    LutSrc ls{t.lut_s_ptr, t.lut_l_ptr, t.lut_t_ptr, t.lut_s_flat, t.lut_l_flat, t.NL,
              lut_s_len, lut_l_len, lut_t_len, nullptr};
    size_t bytes = lut_smem_bytes(t.NL, lut_s_len, lut_l_len, lut_t_len);
    const bool use_smem = bytes <= 48 * 1024;
    legacy::k_fwd<<<dim3((n + legacy::WPB - 1) / legacy::WPB, 1), legacy::NET_TPB, use_smem ? bytes : 0, s>>>(
        t, ls, dcs, 0, 0, n, use_smem);
    WS_CHECK_LAUNCH();
}

void launch_bwd_list(const Topo& t, const Corner* dcs, int n, cudaStream_t s)
{
    if (n <= 0) return;
    legacy::k_bwd<<<dim3((n + legacy::WPB - 1) / legacy::WPB, 1), legacy::NET_TPB, 0, s>>>(t, dcs, 0, 0, n);
    WS_CHECK_LAUNCH();
}

}  // namespace ws
