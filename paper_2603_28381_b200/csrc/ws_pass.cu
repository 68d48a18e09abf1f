// The differentiable STA pass on sm_100a (north_star items 2-5).
//
// Work layout: the level-major task arrays of ws_build.cu.  A level is a
// contiguous range of thread blocks; a block owns <= BLK_Q nets (<= BLK_M
// members), or one "big" net (> BIG_M members).  Every level kernel runs two
// phases separated by one __syncthreads:
//   forward : (net, cond) threads merge the in-arcs of their net (NLDM LUT
//             interpolation against the shared-memory LUT pool; late max /
//             early min with the first arc winning ties, then the winning
//             arc's output slew; LSE smooth max for the late conditions),
//             then (member, cond) threads write member arrival / slew / lse;
//   backward: (member, cond) threads fold required times over out-arcs,
//             write slack, gather adjoints (seed + d_arc of out-arcs), then
//             (net, cond) threads fold the members into the root's required
//             time and adjoint and emit d_arc = adjoint(root) * weight.
// Each phase reads its task records with one coalesced load and gathers the
// pin data it needs, so a level costs ~3 dependent memory round trips.
//
// Numerics: every fold keeps the reference's order (sequential per thread,
// or an ordered tree where the earlier element wins ties), so the hard pass,
// TNS and WNS equal the reference bit for bit; gradients equal it except for
// the device exp/log ulps (and a blocked summation order for nets with more
// than BIG_M members).
//
// Nothing is written twice: there is no init pass.  Each TimingState /
// GradientState entry is produced by the kernel that finalizes it (members
// and roots in the level kernels, pins in no net by k_free / k_fin).
#include <curand_kernel.h>
#include <math.h>

#include <algorithm>
#include <vector>

#include "ws_internal.h"

namespace ws {

constexpr int MAXC = 16;   // corners per launch (blockIdx.y)
struct Corners {
    Corner c[MAXC];
};

namespace {

constexpr double INF = __builtin_huge_val();

// np.maximum.at / np.minimum.at merges of endpoint RATs into +-inf
// (sta.py:55-67); early columns max, late columns min, NaN sticky.
__device__ __forceinline__ double init_required(const Topo& t, const Corner& C, int pin, int c,
                                                bool has_ep)
{
    double r = c < 2 ? -INF : INF;
    if (has_ep)
        for (int q = t.pin_ep_ptr[pin]; q < t.pin_ep_ptr[pin + 1]; q++) {
            const double x = C.ep_required[(size_t)t.pin_ep_idx[q] * 4 + c];
            if (c < 2) r = (r >= x || r != r) ? r : x;
            else r = (r <= x || r != r) ? r : x;
        }
    return r;
}

// endpoint-loss seed of a pin (diff.py:192-212): sum over its endpoint
// entries, in entry order, of 1[v>0] (hinge) or sigmoid(v/gamma) (softplus)
__device__ __forceinline__ double seed_adj(const Topo& t, const Corner& C, int pin, int j,
                                           double lse_pin, double g, int kind)
{
    double a = 0.0;
    for (int q = t.pin_ep_ptr[pin]; q < t.pin_ep_ptr[pin + 1]; q++) {
        const double v = __dsub_rn(lse_pin, C.ep_required[(size_t)t.pin_ep_idx[q] * 4 + 2 + j]);
        if (kind == 0) a = __dadd_rn(a, v > 0.0 ? 1.0 : 0.0);
        else a = __dadd_rn(a, __ddiv_rn(1.0, __dadd_rn(1.0, exp(__ddiv_rn(-v, g)))));
    }
    return a;
}

// per-block copy of the task records of the block's nets
struct BlockNets {
    int q0, nq, m0, m1;
    bool big;
};

__device__ __forceinline__ BlockNets block_nets(const Topo& t, int b, int* s_root, int* s_flags,
                                                int* s_mptr, int* s_aptr, int* s_f0, int* s_net)
{
    BlockNets B;
    B.q0 = t.blk_q0[b];
    B.nq = t.blk_q0[b + 1] - B.q0;
    for (int i = threadIdx.x; i <= B.nq; i += blockDim.x) {
        const int q = B.q0 + i;
        s_mptr[i] = t.tq_mptr[q];
        s_aptr[i] = t.tq_aptr[q];
        if (i < B.nq) {
            s_root[i] = t.tq_root[q];
            s_flags[i] = t.tq_flags[q];
            s_f0[i] = t.tq_f0[q];
            s_net[i] = t.lv_nets[q];
        }
    }
    __syncthreads();
    B.m0 = s_mptr[0];
    B.m1 = s_mptr[B.nq];
    B.big = B.nq == 1 && (s_flags[0] & TQ_BIG);
    return B;
}

#define WS_BLOCK_SMEM                                                              \
    __shared__ int s_root[BLK_Q], s_flags[BLK_Q], s_f0[BLK_Q], s_net[BLK_Q];       \
    __shared__ int s_mptr[BLK_Q + 1], s_aptr[BLK_Q + 1];

// ---------------------------------------------------------------------------
// pins in no net: their whole TimingState is the initial one (sta.py:51-68)

__global__ void k_free(Topo t, Corners cs, bool lse)
{
    const Corner& C = cs.c[blockIdx.y];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.n_free) return;
    const int p = t.free_pins[i];
    double at[4] = {0, 0, 0, 0}, sl[4] = {0, 0, 0, 0}, rq[4];
    const int pi = t.pin_pi[p];
    if (pi >= 0)
        for (int c = 0; c < 4; c++) { at[c] = C.pi_arrival[pi * 4 + c]; sl[c] = C.pi_slew[pi * 4 + c]; }
    const bool ep = t.pin_ep_ptr[p + 1] > t.pin_ep_ptr[p];
    for (int c = 0; c < 4; c++) rq[c] = init_required(t, C, p, c, ep);
    const double4 zero = make_double4(0, 0, 0, 0);
    reinterpret_cast<double4*>(C.load)[p] = zero;
    reinterpret_cast<double4*>(C.net_delay)[p] = zero;
    reinterpret_cast<double4*>(C.impulse)[p] = zero;
    reinterpret_cast<double4*>(C.slew)[p] = make_double4(sl[0], sl[1], sl[2], sl[3]);
    reinterpret_cast<double4*>(C.arrival)[p] = make_double4(at[0], at[1], at[2], at[3]);
    reinterpret_cast<double4*>(C.required)[p] = make_double4(rq[0], rq[1], rq[2], rq[3]);
    reinterpret_cast<double4*>(C.slack)[p] =
        make_double4(__dsub_rn(at[0], rq[0]), __dsub_rn(at[1], rq[1]), __dsub_rn(rq[2], at[2]),
                     __dsub_rn(rq[3], at[3]));
    if (lse) reinterpret_cast<double2*>(C.lse_at)[p] = make_double2(at[2], at[3]);
}

// ---------------------------------------------------------------------------
// RC (rc_level, _kernels.pyx:84-156) for every net in one launch: RC depends
// only on values, so level order is irrelevant (sta.compute_rc).

// the reference's exact sequential algorithm for one (net, cond): tree nets
// and reduce widths other than 8
__device__ void rc_seq(const Topo& t, const Corner& C, int net, int root, int s, int m, int c,
                       int w, bool root_member)
{
    double* buf = C.mem_buf + (size_t)s * 4 + c;
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
    if (!root_member) {
        C.net_delay[(size_t)root * 4 + c] = 0.0;
        C.impulse[(size_t)root * 4 + c] = 0.0;
    }
    for (int k = 0; k < m; k++) {
        const int pl = t.mem_parent_loc[s + k];
        const double dp = pl == 0 ? 0.0 : dbuf[4 * (pl - 1)];
        dbuf[4 * k] = __dadd_rn(dp, __dmul_rn(C.mem_res[(size_t)(s + k) * 4 + c], buf[4 * k]));
    }
    for (int k = 0; k < m; k++) {
        const double r = C.mem_res[(size_t)(s + k) * 4 + c];
        const double cp = C.mem_cap[(size_t)(s + k) * 4 + c];
        const double d = dbuf[4 * k];
        const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r), cp), d), __dmul_rn(d, d));
        const int pin = t.mem_pin[s + k];
        if (t.root_net_of_pin[pin] < 0) C.load[(size_t)pin * 4 + c] = buf[4 * k];
        C.net_delay[(size_t)pin * 4 + c] = d;
        C.impulse[(size_t)pin * 4 + c] = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
    }
}

__global__ void __launch_bounds__(PASS_TPB) k_rc(Topo t, Corners cs, int w)
{
    const Corner& C = cs.c[blockIdx.y];
    WS_BLOCK_SMEM
    __shared__ double s_cap[BLK_M * 4];
    __shared__ double s_part[8 * 4];
    const BlockNets B = block_nets(t, blockIdx.x, s_root, s_flags, s_mptr, s_aptr, s_f0, s_net);
    const bool fast = w == 8;
    // phase A: members of star nets, one (member, cond) per thread
    for (int i = threadIdx.x; i < (B.m1 - B.m0) * 4; i += blockDim.x) {
        const int u = B.m0 + (i >> 2), c = i & 3;
        const int fl = t.tm_flags[u], qi = fl >> 8;
        if (!fast || (s_flags[qi] & TQ_TREE)) continue;
        const size_t f = (size_t)(s_f0[qi] + (u - s_mptr[qi]));
        const double b = C.mem_cap[f * 4 + c];
        const double r = C.mem_res[f * 4 + c];
        const double d = __dadd_rn(0.0, __dmul_rn(r, b));
        const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r), b), d), __dmul_rn(d, d));
        const size_t pin = (size_t)t.tm_pin[u];
        if (!(fl & TM_ROOT)) C.load[pin * 4 + c] = b;
        C.net_delay[pin * 4 + c] = d;
        C.impulse[pin * 4 + c] = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
        if (!B.big) s_cap[(u - B.m0) * 4 + c] = b;
    }
    __syncthreads();
    // phase B: root loads
    if (!B.big) {
        const int qi = threadIdx.x >> 2, c = threadIdx.x & 3;
        if (qi >= B.nq) return;
        const int fl = s_flags[qi], root = s_root[qi], net = s_net[qi];
        const int k0 = s_mptr[qi] - B.m0, m = s_mptr[qi + 1] - s_mptr[qi];
        if (!fast || (fl & TQ_TREE)) {
            rc_seq(t, C, net, root, s_f0[qi], m, c, w, fl & TQ_ROOT_MEMBER);
            return;
        }
        // 8 strided partials summed from 0.0, then p[l] += p[l+s], s = 1, 2, 4
        double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int base = 0; base < m; base += 8)
#pragma unroll
            for (int y = 0; y < 8; y++)
                if (base + y < m) p[y] = __dadd_rn(p[y], s_cap[(k0 + base + y) * 4 + c]);
        p[0] = __dadd_rn(p[0], p[1]); p[2] = __dadd_rn(p[2], p[3]);
        p[4] = __dadd_rn(p[4], p[5]); p[6] = __dadd_rn(p[6], p[7]);
        p[0] = __dadd_rn(p[0], p[2]); p[4] = __dadd_rn(p[4], p[6]);
        p[0] = __dadd_rn(p[0], p[4]);
        C.load[(size_t)root * 4 + c] = __dadd_rn(C.root_cap[(size_t)net * 4 + c], p[0]);
        if (!(fl & TQ_ROOT_MEMBER)) {
            C.net_delay[(size_t)root * 4 + c] = 0.0;
            C.impulse[(size_t)root * 4 + c] = 0.0;
        }
        return;
    }
    // big net: 32 threads (y, c) build the strided partials
    const int fl = s_flags[0], root = s_root[0], net = s_net[0], s = s_f0[0];
    const int m = B.m1 - B.m0;
    if (!fast || (fl & TQ_TREE)) {
        if (threadIdx.x < 4) rc_seq(t, C, net, root, s, m, threadIdx.x, w, fl & TQ_ROOT_MEMBER);
        return;
    }
    if (threadIdx.x < 32) {
        const int y = threadIdx.x >> 2, c = threadIdx.x & 3;
        double p = 0.0;
        for (int i = y; i < m; i += 8) p = __dadd_rn(p, C.mem_cap[(size_t)(s + i) * 4 + c]);
        s_part[y * 4 + c] = p;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        const int c = threadIdx.x;
        double* p = s_part;
        const double p0 = __dadd_rn(p[0 * 4 + c], p[1 * 4 + c]), p2 = __dadd_rn(p[2 * 4 + c], p[3 * 4 + c]);
        const double p4 = __dadd_rn(p[4 * 4 + c], p[5 * 4 + c]), p6 = __dadd_rn(p[6 * 4 + c], p[7 * 4 + c]);
        const double tot = __dadd_rn(__dadd_rn(p0, p2), __dadd_rn(p4, p6));
        C.load[(size_t)root * 4 + c] = __dadd_rn(C.root_cap[(size_t)net * 4 + c], tot);
        if (!(fl & TQ_ROOT_MEMBER)) {
            C.net_delay[(size_t)root * 4 + c] = 0.0;
            C.impulse[(size_t)root * 4 + c] = 0.0;
        }
    }
}

// ---------------------------------------------------------------------------
// forward level (forward_level, _kernels.pyx:159-210) + LSE (diff.py:123-146)

__device__ __forceinline__ unsigned short lut_c(ushort4 v, int c)
{
    return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// LSE of one arc-driven root, late column j (cond c = j + 2):
// x_t = lse_at[from] + arc_delay; c = max x (first of equals);
// s = z_0 + pairwise(z_1..) exactly like np.add.reduceat; weights z/s.
__device__ __forceinline__ double lse_root(const Topo& t, const Corner& C, int a0, int a1, int c,
                                           double g)
{
    const int j = c - 2;
    double cmax = -INF;
    for (int q = a0; q < a1; q++) {
        const double x = __dadd_rn(C.lse_at[(size_t)t.ta_from[q] * 2 + j],
                                   C.arc_delay[(size_t)t.ta_arc[q] * 4 + c]);
        if (q == a0 || x > cmax) cmax = x;
    }
    auto z_of = [&](int q) {
        const double x = __dadd_rn(C.lse_at[(size_t)t.ta_from[q] * 2 + j],
                                   C.arc_delay[(size_t)t.ta_arc[q] * 4 + c]);
        return exp(__ddiv_rn(__dsub_rn(x, cmax), g));
    };
    const int n = a1 - a0;
    double rest;
    if (n - 1 < 8) {                       // numpy pairwise_sum, n < 8: sequential from 0.0
        rest = 0.0;
        for (int q = a0 + 1; q < a1; q++) rest = __dadd_rn(rest, z_of(q));
    } else if (n - 1 <= 128) {             // 8 accumulators, combined pairwise, tail
        double r[8];
        for (int k = 0; k < 8; k++) r[k] = z_of(a0 + 1 + k);
        int i = 8;
        const int nn = n - 1;
        for (; i < nn - (nn % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], z_of(a0 + 1 + i + k));
        rest = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < nn; i++) rest = __dadd_rn(rest, z_of(a0 + 1 + i));
    } else {                               // > 129 in-arcs: sequential (documented)
        rest = 0.0;
        for (int q = a0 + 1; q < a1; q++) rest = __dadd_rn(rest, z_of(q));
    }
    const double s = __dadd_rn(z_of(a0), rest);
    for (int q = a0; q < a1; q++) C.weights[(size_t)t.ta_arc[q] * 2 + j] = __ddiv_rn(z_of(q), s);
    return __dadd_rn(cmax, __dmul_rn(g, log(s)));
}

template <bool HARD, bool LSE>
__global__ void __launch_bounds__(PASS_TPB) k_fwd(Topo t, LutSrc ls, Corners cs, int b0,
                                                  bool use_smem, double g)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const Corner& C = cs.c[blockIdx.y];
    WS_BLOCK_SMEM
    __shared__ double s_at[BLK_Q * 4], s_sl[BLK_Q * 4], s_lr[BLK_Q * 2];
    LutView L;
    if (HARD) L = stage_luts(ls, C.lut_t_flat, use_smem, smem);
    const BlockNets B = block_nets(t, b0 + blockIdx.x, s_root, s_flags, s_mptr, s_aptr, s_f0, s_net);
    // phase 1: one (net, cond) per thread
    {
        const int qi = threadIdx.x >> 2, c = threadIdx.x & 3;
        if (qi < B.nq) {
            const bool late = c >= 2;
            const int root = s_root[qi], fl = s_flags[qi], kind = fl & TQ_KIND;
            const int a0 = s_aptr[qi], a1 = s_aptr[qi + 1];
            double at, sl, lr = 0.0;
            if (kind == ROOT_ARC) {
                if (HARD) {
                    const double ld = C.load[(size_t)root * 4 + c];
                    double best = late ? -INF : INF;
                    int wq = a0;
                    for (int q = a0; q < a1; q++) {
                        const int fp = t.ta_from[q];
                        const double d = lut_interp(L, lut_c(t.ta_lut[2 * (size_t)q], c),
                                                    C.slew[(size_t)fp * 4 + c], ld);
                        C.arc_delay[(size_t)t.ta_arc[q] * 4 + c] = d;
                        const double v = __dadd_rn(C.arrival[(size_t)fp * 4 + c], d);
                        if (later_wins(late, best, v)) { best = v; wq = q; }
                    }
                    at = best;
                    sl = lut_interp(L, lut_c(t.ta_lut[2 * (size_t)wq + 1], c),
                                    C.slew[(size_t)t.ta_from[wq] * 4 + c], ld);
                    C.arrival[(size_t)root * 4 + c] = at;
                    C.slew[(size_t)root * 4 + c] = sl;
                }
                if (LSE && late) {
                    lr = lse_root(t, C, a0, a1, c, g);
                    C.lse_at[(size_t)root * 2 + (c - 2)] = lr;
                }
            } else if (kind == ROOT_FEED) {
                // driven by its parent net's member update (a lower level)
                at = C.arrival[(size_t)root * 4 + c];
                sl = C.slew[(size_t)root * 4 + c];
                if (LSE && late) lr = C.lse_at[(size_t)root * 2 + (c - 2)];
            } else {
                // primary-input root (or undriven): the seeded values
                at = 0.0;
                sl = 0.0;
                if (fl & TQ_ROOT_PI) {
                    const int pi = t.pin_pi[root];
                    at = C.pi_arrival[(size_t)pi * 4 + c];
                    sl = C.pi_slew[(size_t)pi * 4 + c];
                }
                if (HARD) {
                    C.arrival[(size_t)root * 4 + c] = at;
                    C.slew[(size_t)root * 4 + c] = sl;
                }
                if (LSE && late) {
                    lr = at;
                    C.lse_at[(size_t)root * 2 + (c - 2)] = lr;
                }
            }
            if (HARD) { s_at[qi * 4 + c] = at; s_sl[qi * 4 + c] = sl; }
            if (LSE && late) s_lr[qi * 2 + (c - 2)] = lr;
        }
    }
    __syncthreads();
    // phase 2: one (member, cond) per thread
    for (int i = threadIdx.x; i < (B.m1 - B.m0) * 4; i += blockDim.x) {
        const int u = B.m0 + (i >> 2), c = i & 3;
        const int qi = t.tm_flags[u] >> 8;
        const size_t pin = (size_t)t.tm_pin[u];
        const double nd = C.net_delay[pin * 4 + c];
        if (HARD) {
            const double sr = s_sl[qi * 4 + c], ii = C.impulse[pin * 4 + c];
            C.arrival[pin * 4 + c] = __dadd_rn(s_at[qi * 4 + c], nd);
            C.slew[pin * 4 + c] = __dsqrt_rn(__dadd_rn(__dmul_rn(sr, sr), __dmul_rn(ii, ii)));
        }
        if (LSE && c >= 2) C.lse_at[pin * 2 + (c - 2)] = __dadd_rn(s_lr[qi * 2 + (c - 2)], nd);
    }
}

// ---------------------------------------------------------------------------
// backward level (backward_level, _kernels.pyx:213-249) + reverse adjoint
// (diff.py:215-241, gather form)

template <bool HARD, bool GRAD>
__global__ void __launch_bounds__(PASS_TPB) k_bwd(Topo t, Corners cs, int b0, double g, int kind)
{
    const Corner& C = cs.c[blockIdx.y];
    WS_BLOCK_SMEM
    __shared__ double s_v[BLK_M * 4], s_de[BLK_M * 2];
    __shared__ double s_red[64 * 4];
    const BlockNets B = block_nets(t, b0 + blockIdx.x, s_root, s_flags, s_mptr, s_aptr, s_f0, s_net);
    // phase A: one (member, cond) per thread
    for (int i = threadIdx.x; i < (B.m1 - B.m0) * 4; i += blockDim.x) {
        const int u = B.m0 + (i >> 2), c = i & 3;
        const int fl = t.tm_flags[u], qi = fl >> 8;
        const size_t pin = (size_t)t.tm_pin[u];
        const int o0 = t.tm_optr[u], o1 = t.tm_optr[u + 1];
        const size_t f = (size_t)(s_f0[qi] + (u - s_mptr[qi]));
        if (HARD) {
            const bool mx = c < 2;
            double r = (fl & TM_ROOT) ? C.required[pin * 4 + c]
                                      : init_required(t, C, (int)pin, c, fl & TM_EP);
            for (int o = o0; o < o1; o++) {
                const double vv = __dsub_rn(C.required[(size_t)t.to_to[o] * 4 + c],
                                            C.arc_delay[(size_t)t.to_arc[o] * 4 + c]);
                if (later_wins(mx, r, vv)) r = vv;
            }
            C.required[pin * 4 + c] = r;
            const double at = C.arrival[pin * 4 + c];
            C.slack[pin * 4 + c] = mx ? __dsub_rn(at, r) : __dsub_rn(r, at);
            const double v = __dsub_rn(r, C.net_delay[pin * 4 + c]);
            if (B.big) C.mem_buf[f * 4 + c] = v;
            else s_v[(u - B.m0) * 4 + c] = v;
        }
        if (GRAD && c >= 2) {
            const int j = c - 2;
            double ad;
            if (fl & TM_ROOT) ad = C.adjoint[pin * 2 + j];
            else ad = (fl & TM_EP) ? seed_adj(t, C, (int)pin, j, C.lse_at[pin * 2 + j], g, kind) : 0.0;
            for (int o = o0; o < o1; o++) ad = __dadd_rn(ad, C.d_arc[(size_t)t.to_arc[o] * 2 + j]);
            C.adjoint[pin * 2 + j] = ad;
            C.d_edge[f * 2 + j] = ad;
            if (!B.big) s_de[(u - B.m0) * 2 + j] = ad;
        }
    }
    __syncthreads();
    if (!B.big) {
        // phase B: one (net, cond) per thread, members in order
        const int qi = threadIdx.x >> 2, c = threadIdx.x & 3;
        if (qi >= B.nq) return;
        const int root = s_root[qi], fl = s_flags[qi];
        const int k0 = s_mptr[qi] - B.m0, k1 = s_mptr[qi + 1] - B.m0;
        if (HARD) {
            const bool mx = c < 2;
            double rr = init_required(t, C, root, c, fl & TQ_ROOT_EP);
            for (int k = k0; k < k1; k++) {
                const double v = s_v[k * 4 + c];
                if (later_wins(mx, rr, v)) rr = v;
            }
            C.required[(size_t)root * 4 + c] = rr;
            if (!(fl & TQ_ROOT_MEMBER)) {
                const double at = C.arrival[(size_t)root * 4 + c];
                C.slack[(size_t)root * 4 + c] = mx ? __dsub_rn(at, rr) : __dsub_rn(rr, at);
            }
        }
        if (GRAD && c >= 2) {
            const int j = c - 2;
            double ar = (fl & TQ_ROOT_EP)
                            ? seed_adj(t, C, root, j, C.lse_at[(size_t)root * 2 + j], g, kind) : 0.0;
            if (fl & TQ_TREE) {
                // parents gather children, deepest member first (diff.py:222-233)
                const int s = s_f0[qi];
                for (int k = k1 - k0 - 1; k >= 0; k--) {
                    const double dk = C.d_edge[(size_t)(s + k) * 2 + j];
                    const int pl = t.mem_parent_loc[s + k];
                    if (pl > 0) {
                        double* dp = C.d_edge + (size_t)(s + pl - 1) * 2 + j;
                        *dp = __dadd_rn(*dp, dk);
                    } else {
                        ar = __dadd_rn(ar, dk);
                    }
                }
            } else {
                for (int k = k1 - 1; k >= k0; k--) ar = __dadd_rn(ar, s_de[k * 2 + j]);
            }
            C.adjoint[(size_t)root * 2 + j] = ar;
            if ((fl & TQ_KIND) == ROOT_ARC)
                for (int q = s_aptr[qi]; q < s_aptr[qi + 1]; q++) {
                    const size_t a = (size_t)t.ta_arc[q];
                    C.d_arc[a * 2 + j] = __dmul_rn(ar, C.weights[a * 2 + j]);
                }
        }
        return;
    }
    // ---- one big net: ordered parallel folds over contiguous member ranges
    const int root = s_root[0], fl = s_flags[0], s = s_f0[0], m = B.m1 - B.m0;
    const int slot = threadIdx.x >> 2, c = threadIdx.x & 3;
    const int per = (m + 63) / 64, k0 = min(m, slot * per), k1 = min(m, k0 + per);
    if (HARD) {
        const bool mx = c < 2;
        double part = mx ? -INF : INF;
        for (int k = k0; k < k1; k++) {
            const double v = C.mem_buf[(size_t)(s + k) * 4 + c];
            if (later_wins(mx, part, v)) part = v;
        }
        s_red[slot * 4 + c] = part;
        __syncthreads();
        if (slot == 0) {
            double rr = init_required(t, C, root, c, fl & TQ_ROOT_EP);
            for (int sl = 0; sl < 64; sl++)
                if (later_wins(mx, rr, s_red[sl * 4 + c])) rr = s_red[sl * 4 + c];
            C.required[(size_t)root * 4 + c] = rr;
            if (!(fl & TQ_ROOT_MEMBER)) {
                const double at = C.arrival[(size_t)root * 4 + c];
                C.slack[(size_t)root * 4 + c] = mx ? __dsub_rn(at, rr) : __dsub_rn(rr, at);
            }
        }
        __syncthreads();
    }
    if (GRAD) {
        const int j = c - 2;
        if (!(fl & TQ_TREE)) {
            double part = 0.0;
            if (c >= 2)
                for (int k = k1 - 1; k >= k0; k--) part = __dadd_rn(part, C.d_edge[(size_t)(s + k) * 2 + j]);
            s_red[slot * 4 + c] = part;
        }
        __syncthreads();
        if (slot == 0 && c >= 2) {
            double ar = (fl & TQ_ROOT_EP)
                            ? seed_adj(t, C, root, j, C.lse_at[(size_t)root * 2 + j], g, kind) : 0.0;
            if (fl & TQ_TREE) {
                for (int k = m - 1; k >= 0; k--) {
                    const double dk = C.d_edge[(size_t)(s + k) * 2 + j];
                    const int pl = t.mem_parent_loc[s + k];
                    if (pl > 0) {
                        double* dp = C.d_edge + (size_t)(s + pl - 1) * 2 + j;
                        *dp = __dadd_rn(*dp, dk);
                    } else {
                        ar = __dadd_rn(ar, dk);
                    }
                }
            } else {
                for (int sl = 63; sl >= 0; sl--) ar = __dadd_rn(ar, s_red[sl * 4 + c]);
            }
            C.adjoint[(size_t)root * 2 + j] = ar;
            if ((fl & TQ_KIND) == ROOT_ARC)
                for (int q = s_aptr[0]; q < s_aptr[1]; q++) {
                    const size_t a = (size_t)t.ta_arc[q];
                    C.d_arc[a * 2 + j] = __dmul_rn(ar, C.weights[a * 2 + j]);
                }
        }
    }
}

// pins finished after the level loop: pins in no net (seed + out-arcs) and
// PI roots that also source arcs (their level-loop adjoint + out-arcs)
__global__ void k_fin(Topo t, Corners cs, double g, int kind)
{
    const Corner& C = cs.c[blockIdx.y];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * t.n_fin) return;
    const int p = t.fin_pins[i >> 1], j = i & 1;
    double ad = t.fin_flags[i >> 1] ? C.adjoint[(size_t)p * 2 + j]
                                    : seed_adj(t, C, p, j, C.lse_at[(size_t)p * 2 + j], g, kind);
    for (int q = t.pin_out_ptr[p]; q < t.pin_out_ptr[p + 1]; q++)
        ad = __dadd_rn(ad, C.d_arc[(size_t)t.pin_out_arc[q] * 2 + j]);
    C.adjoint[(size_t)p * 2 + j] = ad;
}

// slack over every pin from the current arrival / required (WS_RUN_SLACK)
__global__ void k_slack_all(Topo t, Corners cs)
{
    const Corner& C = cs.c[blockIdx.y];
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= t.P) return;
    const double4 at = reinterpret_cast<const double4*>(C.arrival)[p];
    const double4 rq = reinterpret_cast<const double4*>(C.required)[p];
    reinterpret_cast<double4*>(C.slack)[p] =
        make_double4(__dsub_rn(at.x, rq.x), __dsub_rn(at.y, rq.y), __dsub_rn(rq.z, at.z),
                     __dsub_rn(rq.w, at.w));
}

// lse seed from the hard arrival when LSE runs on a supplied state (diff.py:176)
__global__ void k_lse_seed(Topo t, Corners cs)
{
    const Corner& C = cs.c[blockIdx.y];
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= t.P) return;
    reinterpret_cast<double2*>(C.lse_at)[p] =
        make_double2(C.arrival[(size_t)p * 4 + 2], C.arrival[(size_t)p * 4 + 3]);
}

// ---------------------------------------------------------------------------
// TNS / WNS / loss.  ndarray.sum() is numpy's pairwise tree (8 accumulators,
// leaves <= 128 elements); SumPlan holds that exact tree for the 2E endpoint
// terms, so TNS and the loss equal the reference's bit for bit.  One warp per
// leaf; the last block to finish combines the tree.

__device__ __forceinline__ void summary_terms(const Topo& t, const Corner& C, int i, double g,
                                              int kind, bool want_loss, double& tns_term,
                                              double& slack, double& loss_term)
{
    const int e = i >> 1, j = i & 1;
    const int pin = t.ep_pin[e];
    slack = C.slack[(size_t)pin * 4 + 2 + j];
    tns_term = (slack <= 0.0 || slack != slack) ? slack : 0.0;      // np.minimum(s, 0.0)
    loss_term = 0.0;
    if (want_loss) {
        const double v = __dsub_rn(C.lse_at[(size_t)pin * 2 + j], C.ep_required[(size_t)e * 4 + 2 + j]);
        const double mxv = (v >= 0.0 || v != v) ? v : 0.0;           // np.maximum(v, 0.0)
        if (kind == 0) loss_term = mxv;
        else loss_term = __dadd_rn(mxv, __dmul_rn(g, log1p(exp(__ddiv_rn(-fabs(v), g)))));
    }
}

__global__ void __launch_bounds__(256) k_summary(Topo t, Corners cs, const int* leaf_off,
                                                 const int* leaf_len, int n_leaves,
                                                 const int* in_left, const int* in_right,
                                                 const int* height_ptr, int n_heights, double g,
                                                 int kind, bool want_loss, bool want_sta)
{
    const Corner& C = cs.c[blockIdx.y];
    __shared__ double s_t[8][128], s_l[8][128];
    __shared__ bool s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lf = blockIdx.x * 8 + warp;
    double* nv = C.red_tmp;   // [3 * nodes]: tns, loss, wns per node
    const int nn = 2 * n_leaves - 1;
    if (lf < n_leaves) {
        const int off = leaf_off[lf], n = leaf_len[lf];
        double wmin = INF;
        for (int k = lane; k < n; k += 32) {
            double tt, sl, lt;
            summary_terms(t, C, off + k, g, kind, want_loss, tt, sl, lt);
            s_t[warp][k] = tt;
            s_l[warp][k] = lt;
            wmin = (sl < wmin || sl != sl) ? sl : wmin;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double w2 = __shfl_down_sync(WS_FULL, wmin, o);
            wmin = (w2 < wmin || w2 != w2) ? w2 : wmin;
        }
        __syncwarp();
        // lanes 0..7 own accumulator j of numpy's unrolled pairwise leaf
        double rt = 0.0, rl = 0.0;
        if (n >= 8 && lane < 8) {
            rt = s_t[warp][lane];
            rl = s_l[warp][lane];
            for (int i = 8; i < n - (n % 8); i += 8) {
                rt = __dadd_rn(rt, s_t[warp][i + lane]);
                rl = __dadd_rn(rl, s_l[warp][i + lane]);
            }
        }
        double r8t[8], r8l[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            r8t[k] = __shfl_sync(WS_FULL, rt, k);
            r8l[k] = __shfl_sync(WS_FULL, rl, k);
        }
        if (lane == 0) {
            double ts, ls;
            int i;
            if (n < 8) {
                ts = 0.0; ls = 0.0; i = 0;
            } else {
                ts = __dadd_rn(__dadd_rn(__dadd_rn(r8t[0], r8t[1]), __dadd_rn(r8t[2], r8t[3])),
                               __dadd_rn(__dadd_rn(r8t[4], r8t[5]), __dadd_rn(r8t[6], r8t[7])));
                ls = __dadd_rn(__dadd_rn(__dadd_rn(r8l[0], r8l[1]), __dadd_rn(r8l[2], r8l[3])),
                               __dadd_rn(__dadd_rn(r8l[4], r8l[5]), __dadd_rn(r8l[6], r8l[7])));
                i = n - (n % 8);
            }
            for (; i < n; i++) {
                ts = __dadd_rn(ts, s_t[warp][i]);
                ls = __dadd_rn(ls, s_l[warp][i]);
            }
            nv[lf] = ts;
            nv[nn + lf] = ls;
            nv[2 * nn + lf] = wmin;
        }
    }
    // the last block to finish combines the tree
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(C.sync_ctr, 1u);
        s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int h = 0; h < n_heights; h++) {
        for (int k = height_ptr[h] + threadIdx.x; k < height_ptr[h + 1]; k += blockDim.x) {
            const int l = in_left[k], r = in_right[k], me = n_leaves + k;
            nv[me] = __dadd_rn(nv[l], nv[r]);
            nv[nn + me] = __dadd_rn(nv[nn + l], nv[nn + r]);
            const double a = nv[2 * nn + l], b = nv[2 * nn + r];
            nv[2 * nn + me] = (b < a || b != b) ? b : a;
        }
        __threadfence_block();
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int top = nn - 1;
        if (want_sta) { C.summary[0] = nv[top]; C.summary[1] = nv[2 * nn + top]; }
        if (want_loss) C.summary[2] = nv[nn + top];
        *C.sync_ctr = 0u;
    }
}

__global__ void k_summary_empty(Corners cs, bool want_loss, bool want_sta)
{
    const Corner& C = cs.c[blockIdx.y];
    if (threadIdx.x == 0) {
        if (want_sta) { C.summary[0] = 0.0; C.summary[1] = INF; }
        if (want_loss) C.summary[2] = 0.0;
    }
}

struct PlanNode { int left, right, off, len, height; };
int plan_rec(std::vector<PlanNode>& nodes, int off, int n)
{
    if (n <= 128) {
        nodes.push_back({-1, -1, off, n, 0});
        return (int)nodes.size() - 1;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    const int l = plan_rec(nodes, off, n2);
    const int r = plan_rec(nodes, off + n2, n - n2);
    nodes.push_back({l, r, off, n, std::max(nodes[l].height, nodes[r].height) + 1});
    return (int)nodes.size() - 1;
}

// C4 placement-loop stand-in: per member (res, cap) and per
// net (root cap) one factor 1 + sigma*clip(z, -3, 3), z ~ N(0,1) from a
// counter-based Philox stream keyed by (seed, element), applied to all four
// conditions so early == late stays intact where the design has it.
__device__ __forceinline__ double perturb_factor(unsigned long long seed, unsigned long long id,
                                                 double sigma)
{
    curandStatePhilox4_32_10_t st;
    curand_init(seed, id, 0, &st);
    double z = curand_normal_double(&st);
    z = z < -3.0 ? -3.0 : (z > 3.0 ? 3.0 : z);
    return 1.0 + sigma * z;
}

__global__ void k_perturb(int M, int N, Corner D, Corner S, unsigned long long seed, double sigma)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < M) {
        const double fr = perturb_factor(seed, 2ull * i, sigma);
        const double fc = perturb_factor(seed, 2ull * i + 1, sigma);
        for (int c = 0; c < 4; c++) {
            D.mem_res[(size_t)i * 4 + c] = S.mem_res[(size_t)i * 4 + c] * fr;
            D.mem_cap[(size_t)i * 4 + c] = S.mem_cap[(size_t)i * 4 + c] * fc;
        }
    } else if (i < M + N) {
        const int n = i - M;
        const double f = perturb_factor(seed, 2ull * M + n, sigma);
        for (int c = 0; c < 4; c++) D.root_cap[(size_t)n * 4 + c] = S.root_cap[(size_t)n * 4 + c] * f;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

void summary_plan_init(Context& ctx)
{
    SumPlan* pl = new SumPlan();
    pl->n = 2 * ctx.t.E;
    std::vector<PlanNode> nodes;
    if (pl->n > 0) plan_rec(nodes, 0, pl->n);
    std::vector<int> id(nodes.size());
    std::vector<int> loff, llen;
    for (size_t i = 0; i < nodes.size(); i++)
        if (nodes[i].left < 0) { id[i] = (int)loff.size(); loff.push_back(nodes[i].off); llen.push_back(nodes[i].len); }
    pl->n_leaves = (int)loff.size();
    std::vector<int> inner;
    for (size_t i = 0; i < nodes.size(); i++) if (nodes[i].left >= 0) inner.push_back((int)i);
    std::stable_sort(inner.begin(), inner.end(),
                     [&](int a, int b) { return nodes[a].height < nodes[b].height; });
    pl->n_inner = (int)inner.size();
    for (size_t k = 0; k < inner.size(); k++) id[inner[k]] = pl->n_leaves + (int)k;
    std::vector<int> il, ir;
    pl->height_ptr.assign(1, 0);
    int cur_h = 1;
    for (size_t k = 0; k < inner.size(); k++) {
        const PlanNode& nd = nodes[inner[k]];
        while (nd.height > cur_h) { pl->height_ptr.push_back((int)k); cur_h++; }
        il.push_back(id[nd.left]);
        ir.push_back(id[nd.right]);
        pl->max_height = nd.height;
    }
    pl->height_ptr.push_back((int)inner.size());
    Arena& ar = ctx.topo_mem;
    pl->leaf_off = ar.alloc<int>(std::max<size_t>(1, loff.size()));
    pl->leaf_len = ar.alloc<int>(std::max<size_t>(1, llen.size()));
    pl->in_left = ar.alloc<int>(std::max<size_t>(1, il.size()));
    pl->in_right = ar.alloc<int>(std::max<size_t>(1, ir.size()));
    pl->d_height_ptr = ar.alloc<int>(pl->height_ptr.size());
    if (!loff.empty()) {
        WS_CUDA(cudaMemcpy(pl->leaf_off, loff.data(), loff.size() * 4, cudaMemcpyHostToDevice));
        WS_CUDA(cudaMemcpy(pl->leaf_len, llen.data(), llen.size() * 4, cudaMemcpyHostToDevice));
    }
    if (!il.empty()) {
        WS_CUDA(cudaMemcpy(pl->in_left, il.data(), il.size() * 4, cudaMemcpyHostToDevice));
        WS_CUDA(cudaMemcpy(pl->in_right, ir.data(), ir.size() * 4, cudaMemcpyHostToDevice));
    }
    WS_CUDA(cudaMemcpy(pl->d_height_ptr, pl->height_ptr.data(), pl->height_ptr.size() * 4,
                       cudaMemcpyHostToDevice));
    ctx.tns_plan = pl;
}

void summary_plan_free(Context& ctx)
{
    delete ctx.tns_plan;
    ctx.tns_plan = nullptr;
}

void launch_perturb(const Context& ctx, int dst, int src, unsigned long long seed, double sigma,
                    cudaStream_t s)
{
    const int n = ctx.t.M + ctx.t.N;
    if (n <= 0) return;
    k_perturb<<<(n + 255) / 256, 256, 0, s>>>(ctx.t.M, ctx.t.N, ctx.corners[dst].d,
                                              ctx.corners[src].d, seed, sigma);
    WS_CHECK_LAUNCH();
}

namespace {

struct Launcher {
    Context& ctx;
    Corners cs;
    int nc;
    int count = 0;
    LutSrc ls;
    size_t lut_bytes;
    bool use_smem;
    Launcher(Context& c, int c0, int nc_) : ctx(c), nc(nc_)
    {
        for (int k = 0; k < nc; k++) cs.c[k] = ctx.corners[c0 + k].d;
        const Topo& t = ctx.t;
        ls = {t.lut_s_ptr, t.lut_l_ptr, t.lut_t_ptr, t.lut_s_flat, t.lut_l_flat, t.NL,
              ctx.lut_s_len, ctx.lut_l_len, ctx.lut_t_len};
        lut_bytes = lut_smem_bytes(t.NL, ctx.lut_s_len, ctx.lut_l_len, ctx.lut_t_len);
        use_smem = lut_bytes <= 96 * 1024;
        if (!use_smem) lut_bytes = 0;
    }
    dim3 grid1(int n, int tpb) const { return dim3((unsigned)std::max(1, (n + tpb - 1) / tpb), nc); }
    int blocks(int li) const { return ctx.lvb_ptr_host[li + 1] - ctx.lvb_ptr_host[li]; }

    void free_pins(cudaStream_t s, bool lse)
    {
        if (!ctx.t.n_free) return;
        k_free<<<grid1(ctx.t.n_free, 256), 256, 0, s>>>(ctx.t, cs, lse);
        count++;
    }
    void rc(cudaStream_t s, int w)
    {
        if (!ctx.t.n_blocks) return;
        k_rc<<<dim3(ctx.t.n_blocks, nc), PASS_TPB, 0, s>>>(ctx.t, cs, w);
        count++;
    }
    template <bool H, bool Lse>
    void fwd(cudaStream_t s, int li, double g)
    {
        const int nb = blocks(li);
        if (nb <= 0) return;
        k_fwd<H, Lse><<<dim3(nb, nc), PASS_TPB, H ? lut_bytes : 0, s>>>(
            ctx.t, ls, cs, ctx.lvb_ptr_host[li], use_smem, g);
        count++;
    }
    template <bool H, bool G>
    void bwd(cudaStream_t s, int li, double g, int kind)
    {
        const int nb = blocks(li);
        if (nb <= 0) return;
        k_bwd<H, G><<<dim3(nb, nc), PASS_TPB, 0, s>>>(ctx.t, cs, ctx.lvb_ptr_host[li], g, kind);
        count++;
    }
    void fin(cudaStream_t s, double g, int kind)
    {
        if (!ctx.t.n_fin) return;
        k_fin<<<grid1(2 * ctx.t.n_fin, 256), 256, 0, s>>>(ctx.t, cs, g, kind);
        count++;
    }
    void slack_all(cudaStream_t s)
    {
        if (!ctx.t.P) return;
        k_slack_all<<<grid1(ctx.t.P, 256), 256, 0, s>>>(ctx.t, cs);
        count++;
    }
    void lse_seed(cudaStream_t s)
    {
        if (!ctx.t.P) return;
        k_lse_seed<<<grid1(ctx.t.P, 256), 256, 0, s>>>(ctx.t, cs);
        count++;
    }
    void summary(cudaStream_t s, double g, int kind, bool want_loss, bool want_sta)
    {
        const SumPlan* pl = ctx.tns_plan;
        if (pl->n == 0) {
            k_summary_empty<<<dim3(1, nc), 32, 0, s>>>(cs, want_loss, want_sta);
            count++;
            return;
        }
        k_summary<<<dim3((pl->n_leaves + 7) / 8, nc), 256, 0, s>>>(
            ctx.t, cs, pl->leaf_off, pl->leaf_len, pl->n_leaves, pl->in_left, pl->in_right,
            pl->d_height_ptr, (int)pl->height_ptr.size() - 1, g, kind, want_loss, want_sta);
        count++;
    }
};

void run_chunk(Context& ctx, int c0, int nc, unsigned flags, double g, int kind, int gran,
               cudaStream_t s, cudaStream_t gs, int w, int& count)
{
    const int L = ctx.t.L;
    Launcher la(ctx, c0, nc);
    if (la.lut_bytes > 48 * 1024) {
        WS_CUDA(cudaFuncSetAttribute(k_fwd<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la.lut_bytes));
        WS_CUDA(cudaFuncSetAttribute(k_fwd<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la.lut_bytes));
    }
    const bool hard = flags & WS_RUN_HARD, lse = flags & WS_RUN_LSE, grad = flags & WS_RUN_GRAD;
    const bool fused = (flags & WS_RUN_FUSED) && hard && lse && grad;
    const bool two = (flags & WS_RUN_TWO_STREAM) && hard && (lse || grad) && !fused;

    if (fused) {
        la.free_pins(s, true);
        la.rc(s, w);
        for (int li = 0; li < L; li++) la.fwd<true, true>(s, li, g);
        for (int li = L - 1; li >= 0; li--) la.bwd<true, true>(s, li, g, kind);
        la.fin(s, g, kind);
        la.summary(s, g, kind, true, true);
    } else if (two) {
        // stream S: the hard pass; stream G: LSE + gradients, gated per
        // granularity-g level group on S's forward (fusion.py:151-157)
        std::vector<cudaEvent_t>& ev = ctx.events;
        const int n_groups = (L + gran - 1) / gran;
        while ((int)ev.size() < n_groups + 3) {
            cudaEvent_t e;
            WS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev.push_back(e);
        }
        WS_CUDA(cudaEventRecord(ev[n_groups + 2], s));   // fork
        WS_CUDA(cudaStreamWaitEvent(gs, ev[n_groups + 2], 0));
        la.free_pins(s, true);
        la.rc(s, w);
        for (int gi = 0; gi < n_groups; gi++) {
            const int l0 = gi * gran, l1 = std::min(L, l0 + gran);
            for (int li = l0; li < l1; li++) la.fwd<true, false>(s, li, g);
            WS_CUDA(cudaEventRecord(ev[gi], s));
            if (lse) {
                WS_CUDA(cudaStreamWaitEvent(gs, ev[gi], 0));
                for (int li = l0; li < l1; li++) la.fwd<false, true>(gs, li, g);
            }
        }
        for (int li = L - 1; li >= 0; li--) {
            la.bwd<true, false>(s, li, g, kind);
            if (li == L - 1) WS_CUDA(cudaEventRecord(ev[n_groups], s));
        }
        if (grad) {
            if (L) WS_CUDA(cudaStreamWaitEvent(gs, ev[n_groups], 0));  // slack_bwd:L-1 -> grad_bwd:L-1
            for (int li = L - 1; li >= 0; li--) la.bwd<false, true>(gs, li, g, kind);
            la.fin(gs, g, kind);
        }
        WS_CUDA(cudaEventRecord(ev[n_groups + 1], gs));   // join
        WS_CUDA(cudaStreamWaitEvent(s, ev[n_groups + 1], 0));
        la.summary(s, g, kind, grad, true);
    } else {
        if (hard) {
            la.free_pins(s, lse);
            la.rc(s, w);
            for (int li = 0; li < L; li++) la.fwd<true, false>(s, li, g);
        }
        if (lse) {
            if (!hard) la.lse_seed(s);
            for (int li = 0; li < L; li++) la.fwd<false, true>(s, li, g);
        }
        if (hard)
            for (int li = L - 1; li >= 0; li--) la.bwd<true, false>(s, li, g, kind);
        if (grad) {
            for (int li = L - 1; li >= 0; li--) la.bwd<false, true>(s, li, g, kind);
            la.fin(s, g, kind);
        }
        if (!hard && (flags & WS_RUN_SLACK)) la.slack_all(s);
        if (hard || grad || (flags & WS_RUN_SUMMARY))
            la.summary(s, g, kind, grad, hard || (flags & WS_RUN_SUMMARY));
    }
    WS_CHECK_LAUNCH();
    count += la.count;
}

}  // namespace

void run_pass(Context& ctx, int c0, int nc, unsigned flags, double gamma, int loss_kind,
              int granularity, cudaStream_t s, cudaStream_t gs, int w)
{
    int count = 0;
    for (int k = 0; k < nc; k += MAXC)
        run_chunk(ctx, c0 + k, std::min(MAXC, nc - k), flags, gamma, loss_kind, granularity, s, gs,
                  w, count);
    ctx.launches_last_run = count;
}

}  // namespace ws
