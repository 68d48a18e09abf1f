// The differentiable STA pass on sm_100a (north_star items 2-5).
//
// Work unit: a *task* (ws_build.cu build_tasks) = one thread block's share of
// one level: <= 64 nets with <= 64 in-arcs and <= 64 members in total, so a
// 256-thread block holds one (item, condition) per thread for each of the
// three item kinds.  Every level kernel is three memory rounds deep:
//   R1  the task record;
//   R2  the nets' / arcs' / members' records (level-major task arrays, one
//       coalesced load each);
//   R3  every pin gather the task needs, all issued together (from-pin
//       slew/arrival/lse, root load, member net_delay/impulse, out-arc
//       required/arc_delay/d_arc, ...);
// then compute in three block phases separated by __syncthreads:
//   forward : (arc, cond) interpolate the delay LUT in shared memory and form
//             arrival candidates -> (net, cond) merge them in arc order (late
//             max / early min, first arc wins ties), interpolate the winner's
//             slew LUT, LSE smooth max of the late conditions -> (member,
//             cond) member arrival / slew / lse;
//   backward: (member, cond) fold required times over out-arcs, slack,
//             adjoint = seed + d_arc of out-arcs -> (net, cond) fold members
//             into the root's required time and adjoint, emit d_arc.
// Big star nets are split into chunks of 64 members (one task each; the last
// chunk to finish combines the ordered partial folds); nets with > 64
// in-arcs or big RC trees take a single-net task with sequential folds.
//
// Numerics: every fold keeps the reference's order (sequential, or an
// ordered combine where the earlier element wins ties), so the hard pass,
// TNS and WNS equal the reference bit for bit; gradients equal it up to the
// device exp/log ulps (and a chunk-blocked sum order for nets with > 64
// members).  Nothing is written twice: there is no init pass — each output
// entry is produced by the kernel that finalizes it.
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

struct Task {
    int q0, nq, a0, na, m0, nm, flags, slot;
};

__device__ __forceinline__ Task load_task(const Topo& t, int k)
{
    const int4 a = t.tk_a[k], b = t.tk_b[k];
    return Task{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}

// required-time init of a pin: np.maximum.at / np.minimum.at merges of its
// endpoint RATs into -inf / +inf (sta.py:55-67); NaN sticky like numpy
__device__ __forceinline__ double merge_req(double r, double x, int c)
{
    if (c < 2) return (r >= x || r != r) ? r : x;
    return (r <= x || r != r) ? r : x;
}

__device__ double init_required_multi(const Topo& t, const Corner& C, int pin, int c)
{
    double r = c < 2 ? -INF : INF;
    for (int q = t.pin_ep_ptr[pin]; q < t.pin_ep_ptr[pin + 1]; q++)
        r = merge_req(r, C.ep_required[(size_t)t.pin_ep_idx[q] * 4 + c], c);
    return r;
}

// endpoint-loss seed (diff.py:192-212): 1[v>0] (hinge) or sigmoid(v/gamma)
__device__ __forceinline__ double seed_term(double v, double g, int kind)
{
    if (kind == 0) return v > 0.0 ? 1.0 : 0.0;
    return __ddiv_rn(1.0, __dadd_rn(1.0, exp(__ddiv_rn(-v, g))));
}

__device__ double seed_multi(const Topo& t, const Corner& C, int pin, int j, double lse_pin,
                             double g, int kind)
{
    double a = 0.0;
    for (int q = t.pin_ep_ptr[pin]; q < t.pin_ep_ptr[pin + 1]; q++)
        a = __dadd_rn(a, seed_term(__dsub_rn(lse_pin, C.ep_required[(size_t)t.pin_ep_idx[q] * 4 + 2 + j]),
                                   g, kind));
    return a;
}

__device__ __forceinline__ unsigned short lut_c(ushort4 v, int c)
{
    return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// per-task copy of the nets' records
struct NetSmem {
    int root[TASK_Q], flags[TASK_Q], f0[TASK_Q], net[TASK_Q], e1[TASK_Q];
    int aptr[TASK_Q + 1];   // absolute ta_* offsets
    int mptr[TASK_Q + 1];   // absolute tm_* offsets
};

__device__ __forceinline__ void load_nets(const Topo& t, const Task& T, NetSmem& S)
{
    const int i = threadIdx.x;
    if (i <= T.nq) {
        const int q = T.q0 + i;
        S.aptr[i] = t.tq_aptr[q];
        S.mptr[i] = t.tq_mptr[q];
        if (i < T.nq) {
            S.root[i] = t.tq_root[q];
            S.flags[i] = t.tq_flags[q];
            S.f0[i] = t.tq_f0[q];
            S.net[i] = t.lv_nets[q];
            S.e1[i] = t.tq_e1[q];
        }
    }
}

// LSE of one arc-driven root, late column j = c - 2, read from global memory:
// x_t = lse_at[from] + arc_delay; c = max x (first of equals);
// s = z_0 + pairwise(z_1..) exactly like np.add.reduceat; weights z/s.
__device__ double lse_root_global(const Topo& t, const Corner& C, int a0, int a1, int c, double g,
                                  bool write_w)
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
    double rest = 0.0;
    if (n - 1 >= 8 && n - 1 <= 128) {     // numpy pairwise: 8 accumulators, then tail
        double r[8];
        for (int k = 0; k < 8; k++) r[k] = z_of(a0 + 1 + k);
        int i = 8;
        const int nn = n - 1;
        for (; i < nn - (nn % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], z_of(a0 + 1 + i + k));
        rest = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < nn; i++) rest = __dadd_rn(rest, z_of(a0 + 1 + i));
    } else {                              // < 8 (numpy: sequential); > 129 in-arcs: sequential
        for (int q = a0 + 1; q < a1; q++) rest = __dadd_rn(rest, z_of(q));
    }
    const double s = __dadd_rn(z_of(a0), rest);
    if (write_w)
        for (int q = a0; q < a1; q++) C.weights[(size_t)t.ta_arc[q] * 2 + j] = __ddiv_rn(z_of(q), s);
    return __dadd_rn(cmax, __dmul_rn(g, log(s)));
}

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
    for (int c = 0; c < 4; c++) rq[c] = init_required_multi(t, C, p, c);
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
// RC (rc_level, _kernels.pyx:84-156).  RC depends only on values, so one
// launch covers every task of every level (sta.compute_rc).

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

// root load of a star net with reduce width 8: 8 strided partials summed
// sequentially from 0.0, then p[l] += p[l+s] for s = 1, 2, 4
__device__ __forceinline__ double root_load8(const double* caps, int stride, int m)
{
    double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int base = 0; base < m; base += 8)
#pragma unroll
        for (int y = 0; y < 8; y++)
            if (base + y < m) p[y] = __dadd_rn(p[y], caps[(size_t)(base + y) * stride]);
    p[0] = __dadd_rn(p[0], p[1]); p[2] = __dadd_rn(p[2], p[3]);
    p[4] = __dadd_rn(p[4], p[5]); p[6] = __dadd_rn(p[6], p[7]);
    p[0] = __dadd_rn(p[0], p[2]); p[4] = __dadd_rn(p[4], p[6]);
    return __dadd_rn(p[0], p[4]);
}

__device__ __forceinline__ bool last_chunk(unsigned* ctr, int nch, int* s_flag)
{
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(ctr, 1u);
        *s_flag = prev == (unsigned)(nch - 1);
        if (*s_flag) *ctr = 0u;
    }
    __syncthreads();
    if (*s_flag) __threadfence();
    return *s_flag;
}

__global__ void __launch_bounds__(PASS_TPB) k_rc(Topo t, Corners cs, int w)
{
    const Corner& C = cs.c[blockIdx.y];
    __shared__ NetSmem S;
    __shared__ double s_cap[TASK_M * 4];
    __shared__ int s_flag;
    const Task T = load_task(t, blockIdx.x);
    const int tid = threadIdx.x;
    const bool fast = w == 8;
    // R2: records
    load_nets(t, T, S);
    int pin = 0, fl = 0;
    const int mi = tid >> 2, c = tid & 3;
    const bool mem_item = mi < T.nm && !(T.flags & TK_LOOP);
    if (mem_item) {
        pin = t.tm_pin[T.m0 + mi];
        fl = t.tm_flags[T.m0 + mi];
    }
    __syncthreads();
    // R3 + member phase (star nets, w == 8)
    if (mem_item && fast && !(S.flags[fl >> 8] & TQ_TREE)) {
        const int qi = fl >> 8;
        const size_t f = (size_t)(S.f0[qi] + (T.m0 + mi - S.mptr[qi]));
        const double b = C.mem_cap[f * 4 + c];
        const double r = C.mem_res[f * 4 + c];
        const double d = __dadd_rn(0.0, __dmul_rn(r, b));
        const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r), b), d), __dmul_rn(d, d));
        if (!(fl & TM_ROOT)) C.load[(size_t)pin * 4 + c] = b;
        C.net_delay[(size_t)pin * 4 + c] = d;
        C.impulse[(size_t)pin * 4 + c] = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
        s_cap[mi * 4 + c] = b;
    }
    if (T.flags & TK_CHUNK) {
        // big star net: the last chunk sums every member's cap in order
        const int root = S.root[0], net = S.net[0], s = S.f0[0];
        const int m = S.mptr[1] - S.mptr[0];
        if (!fast) {
            if (last_chunk(C.big_ctr + 4 * T.slot + 0, t.bn_nch[T.slot], &s_flag) && tid < 4)
                rc_seq(t, C, net, root, s, m, tid, w, S.flags[0] & TQ_ROOT_MEMBER);
            return;
        }
        if (!last_chunk(C.big_ctr + 4 * T.slot + 0, t.bn_nch[T.slot], &s_flag)) return;
        if (tid < 4) {
            const double l = root_load8(C.mem_cap + (size_t)s * 4 + tid, 4, m);
            C.load[(size_t)root * 4 + tid] = __dadd_rn(C.root_cap[(size_t)net * 4 + tid], l);
            if (!(S.flags[0] & TQ_ROOT_MEMBER)) {
                C.net_delay[(size_t)root * 4 + tid] = 0.0;
                C.impulse[(size_t)root * 4 + tid] = 0.0;
            }
        }
        return;
    }
    __syncthreads();
    // net phase: root loads
    const int qi = tid >> 2;
    if (qi >= T.nq) return;
    const int fq = S.flags[qi], root = S.root[qi], net = S.net[qi];
    const int m = S.mptr[qi + 1] - S.mptr[qi];
    if (!fast || (fq & TQ_TREE) || (T.flags & TK_LOOP)) {
        rc_seq(t, C, net, root, S.f0[qi], m, c, w, fq & TQ_ROOT_MEMBER);
        return;
    }
    const double l = root_load8(s_cap + (S.mptr[qi] - T.m0) * 4 + c, 4, m);
    C.load[(size_t)root * 4 + c] = __dadd_rn(C.root_cap[(size_t)net * 4 + c], l);
    if (!(fq & TQ_ROOT_MEMBER)) {
        C.net_delay[(size_t)root * 4 + c] = 0.0;
        C.impulse[(size_t)root * 4 + c] = 0.0;
    }
}

// ---------------------------------------------------------------------------
// forward level (forward_level, _kernels.pyx:159-210) + LSE (diff.py:123-146)

struct FwdSmem {
    NetSmem n;
    double cand[TASK_A * 4];    // arrival candidate of (arc, cond)
    double slf[TASK_A * 4];     // slew at the arc's source
    double x[TASK_A * 2];       // LSE operand of (arc, late col)
    unsigned short slut[TASK_A * 4];
    double ld[TASK_Q * 4];      // root load
    double at[TASK_Q * 4], sl[TASK_Q * 4], lr[TASK_Q * 2];   // root results
};

template <bool HARD, bool LSE>
__global__ void __launch_bounds__(PASS_TPB) k_fwd(Topo t, LutSrc ls, Corners cs, int k0,
                                                  bool use_smem, double g)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ FwdSmem S;
    const Corner& C = cs.c[blockIdx.y];
    const int tid = threadIdx.x, c = tid & 3, ii = tid >> 2;
    const bool late = c >= 2;
    const Task T = load_task(t, k0 + blockIdx.x);                       // R1
    LutView L;
    if (HARD) L = stage_luts(ls, C.lut_t_flat, use_smem, smem);
    const bool wide = T.flags & TK_WIDE;
    // R2: records
    load_nets(t, T, S.n);
    const bool arc_item = ii < T.na && !wide;
    int from = 0, root = 0, arc = 0, aq = 0;
    ushort4 ld_ids{}, ls_ids{};
    if (arc_item) {
        const int q = T.a0 + ii;
        from = t.ta_from[q];
        root = t.ta_root[q];
        arc = t.ta_arc[q];
        aq = t.ta_q[q];
        if (HARD) { ld_ids = t.ta_lut[2 * (size_t)q]; ls_ids = t.ta_lut[2 * (size_t)q + 1]; }
    }
    const bool mem_item = ii < T.nm;
    int mpin = 0, mfl = 0;
    if (mem_item) { mpin = t.tm_pin[T.m0 + ii]; mfl = t.tm_flags[T.m0 + ii]; }
    // R3: gathers
    double slf = 0, atf = 0, ld = 0, xl = 0, dd = 0;
    if (arc_item) {
        if (HARD) {
            slf = C.slew[(size_t)from * 4 + c];
            atf = C.arrival[(size_t)from * 4 + c];
            ld = C.load[(size_t)root * 4 + c];
        } else {
            dd = C.arc_delay[(size_t)arc * 4 + c];
        }
        if (LSE && late) xl = C.lse_at[(size_t)from * 2 + (c - 2)];
    }
    double mnd = 0, mim = 0;
    if (mem_item) {
        mnd = C.net_delay[(size_t)mpin * 4 + c];
        if (HARD) mim = C.impulse[(size_t)mpin * 4 + c];
    }
    __syncthreads();                  // LUT pool + net records visible
    // arc phase
    if (arc_item) {
        if (HARD) {
            dd = lut_interp(L, lut_c(ld_ids, c), slf, ld);
            C.arc_delay[(size_t)arc * 4 + c] = dd;
            S.cand[ii * 4 + c] = __dadd_rn(atf, dd);
            S.slf[ii * 4 + c] = slf;
            S.slut[ii * 4 + c] = lut_c(ls_ids, c);
            S.ld[aq * 4 + c] = ld;
        }
        if (LSE && late) S.x[ii * 2 + (c - 2)] = __dadd_rn(xl, dd);
    } else if (HARD && wide) {
        // one net with > TASK_A in-arcs: arc delays in a loop, merge from global
        const int rt = S.n.root[0];
        for (int i = tid; i < T.na * 4; i += blockDim.x) {
            const int q = T.a0 + (i >> 2), cc = i & 3;
            const int fp = t.ta_from[q];
            const double d = lut_interp(L, lut_c(t.ta_lut[2 * (size_t)q], cc),
                                        C.slew[(size_t)fp * 4 + cc], C.load[(size_t)rt * 4 + cc]);
            C.arc_delay[(size_t)t.ta_arc[q] * 4 + cc] = d;
        }
    }
    __syncthreads();
    // net phase: one (net, cond) per thread
    const bool first = !(T.flags & TK_CHUNK) || T.m0 == S.n.mptr[0];
    if (ii < T.nq) {
        const int rt = S.n.root[ii], fl = S.n.flags[ii], kind = fl & TQ_KIND;
        double at = 0, sl = 0, lr = 0;
        if (kind == ROOT_ARC) {
            const int a0 = S.n.aptr[ii] - T.a0, a1 = S.n.aptr[ii + 1] - T.a0;
            if (!wide) {
                if (HARD) {
                    double best = late ? -INF : INF;
                    int wq = a0;
                    for (int q = a0; q < a1; q++) {
                        const double v = S.cand[q * 4 + c];
                        if (later_wins(late, best, v)) { best = v; wq = q; }
                    }
                    at = best;
                    sl = lut_interp(L, S.slut[wq * 4 + c], S.slf[wq * 4 + c], S.ld[ii * 4 + c]);
                }
                if (LSE && late) {
                    const int j = c - 2;
                    double cm = -INF;
                    for (int q = a0; q < a1; q++) {
                        const double x = S.x[q * 2 + j];
                        if (q == a0 || x > cm) cm = x;
                    }
                    double z0 = 0.0, rest = 0.0;
                    const int n = a1 - a0;
                    if (n - 1 >= 8 && n - 1 <= 128) {
                        // numpy pairwise leaf over z_1..z_{n-1}
                        double r[8];
                        for (int k = 0; k < 8; k++)
                            r[k] = exp(__ddiv_rn(__dsub_rn(S.x[(a0 + 1 + k) * 2 + j], cm), g));
                        int i = 8;
                        const int nn = n - 1;
                        for (; i < nn - (nn % 8); i += 8)
                            for (int k = 0; k < 8; k++)
                                r[k] = __dadd_rn(r[k], exp(__ddiv_rn(__dsub_rn(S.x[(a0 + 1 + i + k) * 2 + j], cm), g)));
                        rest = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                        for (; i < nn; i++)
                            rest = __dadd_rn(rest, exp(__ddiv_rn(__dsub_rn(S.x[(a0 + 1 + i) * 2 + j], cm), g)));
                    } else {
                        for (int q = a0 + 1; q < a1; q++)
                            rest = __dadd_rn(rest, exp(__ddiv_rn(__dsub_rn(S.x[q * 2 + j], cm), g)));
                    }
                    z0 = exp(__ddiv_rn(__dsub_rn(S.x[a0 * 2 + j], cm), g));
                    const double ssum = __dadd_rn(z0, rest);
                    lr = __dadd_rn(cm, __dmul_rn(g, log(ssum)));
                    if (first)
                        for (int q = a0; q < a1; q++) {
                            const double z = exp(__ddiv_rn(__dsub_rn(S.x[q * 2 + j], cm), g));
                            C.weights[(size_t)t.ta_arc[T.a0 + q] * 2 + j] = __ddiv_rn(z, ssum);
                        }
                }
            } else {
                const int qa0 = S.n.aptr[0], qa1 = S.n.aptr[1];
                if (HARD) {
                    double best = late ? -INF : INF;
                    int wq = qa0;
                    for (int q = qa0; q < qa1; q++) {
                        const double v = __dadd_rn(C.arrival[(size_t)t.ta_from[q] * 4 + c],
                                                   C.arc_delay[(size_t)t.ta_arc[q] * 4 + c]);
                        if (later_wins(late, best, v)) { best = v; wq = q; }
                    }
                    at = best;
                    sl = lut_interp(L, lut_c(t.ta_lut[2 * (size_t)wq + 1], c),
                                    C.slew[(size_t)t.ta_from[wq] * 4 + c], C.load[(size_t)rt * 4 + c]);
                }
                if (LSE && late) lr = lse_root_global(t, C, qa0, qa1, c, g, first);
            }
            if (first) {
                if (HARD) {
                    C.arrival[(size_t)rt * 4 + c] = at;
                    C.slew[(size_t)rt * 4 + c] = sl;
                }
                if (LSE && late) C.lse_at[(size_t)rt * 2 + (c - 2)] = lr;
            }
        } else if (kind == ROOT_FEED) {
            // driven by its parent net's member update (a lower level)
            if (HARD) {
                at = C.arrival[(size_t)rt * 4 + c];
                sl = C.slew[(size_t)rt * 4 + c];
            }
            if (LSE && late) lr = C.lse_at[(size_t)rt * 2 + (c - 2)];
        } else {
            // primary-input root (or undriven): the seeded values
            if (fl & TQ_ROOT_PI) {
                const int pi = t.pin_pi[rt];
                at = C.pi_arrival[(size_t)pi * 4 + c];
                sl = C.pi_slew[(size_t)pi * 4 + c];
            }
            if (first) {
                if (HARD) {
                    C.arrival[(size_t)rt * 4 + c] = at;
                    C.slew[(size_t)rt * 4 + c] = sl;
                }
                if (LSE && late) C.lse_at[(size_t)rt * 2 + (c - 2)] = at;
            }
            lr = at;
        }
        S.at[ii * 4 + c] = at;
        S.sl[ii * 4 + c] = sl;
        if (late) S.lr[ii * 2 + (c - 2)] = lr;
    }
    __syncthreads();
    // member phase: one (member, cond) per thread
    for (int i = tid; i < T.nm * 4; i += blockDim.x) {
        int pin = mpin, fl = mfl;
        double nd = mnd, im = mim;
        if (i != tid) {       // TK_LOOP tasks only
            pin = t.tm_pin[T.m0 + (i >> 2)];
            fl = t.tm_flags[T.m0 + (i >> 2)];
            nd = C.net_delay[(size_t)pin * 4 + c];
            if (HARD) im = C.impulse[(size_t)pin * 4 + c];
        }
        const int qi = fl >> 8;
        if (HARD) {
            const double sr = S.sl[qi * 4 + c];
            C.arrival[(size_t)pin * 4 + c] = __dadd_rn(S.at[qi * 4 + c], nd);
            C.slew[(size_t)pin * 4 + c] = __dsqrt_rn(__dadd_rn(__dmul_rn(sr, sr), __dmul_rn(im, im)));
        }
        if (LSE && late) C.lse_at[(size_t)pin * 2 + (c - 2)] = __dadd_rn(S.lr[qi * 2 + (c - 2)], nd);
    }
}

// ---------------------------------------------------------------------------
// backward level (backward_level, _kernels.pyx:213-249) + reverse adjoint
// (diff.py:215-241 in gather form: a pin's adjoint is its seed plus the
// d_arc of its out-arcs, read when the pin's own level runs)

struct BwdSmem {
    NetSmem n;
    double v[TASK_M * 4];      // member required - net delay
    double de[TASK_M * 2];     // member d_edge
    double w[TASK_A * 2];      // in-arc softmax weights
    int arc[TASK_A];
    int flag;
};

// one member (u, c): fold required over out-arcs, slack, adjoint.
template <bool HARD, bool GRAD>
__device__ __forceinline__ void bwd_member(const Topo& t, const Corner& C, int u, int pin, int fl,
                                           int c, double g, int kind, double r0, double rto,
                                           double ado, double nd, double at, double adj0,
                                           double lse, double epl, double dout, double& v,
                                           double& de)
{
    const int o0 = t.tm_optr[u], o1 = t.tm_optr[u + 1];
    if (HARD) {
        const bool mx = c < 2;
        double r = r0;
        if (o1 > o0) {
            const double vv = __dsub_rn(rto, ado);
            if (later_wins(mx, r, vv)) r = vv;
            for (int o = o0 + 1; o < o1; o++) {
                const double v2 = __dsub_rn(C.required[(size_t)t.to_to[o] * 4 + c],
                                            C.arc_delay[(size_t)t.to_arc[o] * 4 + c]);
                if (later_wins(mx, r, v2)) r = v2;
            }
        }
        C.required[(size_t)pin * 4 + c] = r;
        C.slack[(size_t)pin * 4 + c] = mx ? __dsub_rn(at, r) : __dsub_rn(r, at);
        v = __dsub_rn(r, nd);
    }
    if (GRAD && c >= 2) {
        const int j = c - 2;
        double ad;
        if (fl & TM_ROOT) ad = adj0;            // includes the seed (root fold, higher level)
        else if (fl & TM_MULTI_EP) ad = seed_multi(t, C, pin, j, lse, g, kind);
        else if (fl & TM_EP) ad = __dadd_rn(0.0, seed_term(__dsub_rn(lse, epl), g, kind));
        else ad = 0.0;
        if (o1 > o0) {
            ad = __dadd_rn(ad, dout);
            for (int o = o0 + 1; o < o1; o++) ad = __dadd_rn(ad, C.d_arc[(size_t)t.to_arc[o] * 2 + j]);
        }
        C.adjoint[(size_t)pin * 2 + j] = ad;
        de = ad;
    }
}

template <bool HARD, bool GRAD>
__global__ void __launch_bounds__(PASS_TPB) k_bwd(Topo t, Corners cs, int k0, double g, int kind,
                                                  int variant)
{
    __shared__ BwdSmem S;
    const Corner& C = cs.c[blockIdx.y];
    const int tid = threadIdx.x, c = tid & 3, ii = tid >> 2;
    const bool late = c >= 2;
    const int j = c - 2;
    const Task T = load_task(t, k0 + blockIdx.x);                       // R1
    const bool loop = T.flags & TK_LOOP, chunk = T.flags & TK_CHUNK, wide = T.flags & TK_WIDE;
    // R2: records
    load_nets(t, T, S.n);
    const bool mem_item = ii < T.nm;
    const int u = T.m0 + ii;
    int pin = 0, fl = 0, o1t = -1, o1a = -1, e1 = -1;
    if (mem_item) {
        pin = t.tm_pin[u];
        fl = t.tm_flags[u];
        o1t = t.tm_o1_to[u];
        o1a = t.tm_o1_arc[u];
        e1 = t.tm_e1[u];
    }
    const bool arc_item = GRAD && late && ii < T.na && !wide;
    int arc = 0;
    if (arc_item) arc = t.ta_arc[T.a0 + ii];
    // R3: gathers
    double r0 = 0, rto = 0, ado = 0, nd = 0, at = 0, adj0 = 0, lse = 0, epl = 0, dout = 0;
    if (mem_item) {
        if (HARD) {
            if (fl & TM_ROOT) r0 = C.required[(size_t)pin * 4 + c];
            else if (fl & TM_MULTI_EP) r0 = init_required_multi(t, C, pin, c);
            else r0 = merge_req(c < 2 ? -INF : INF, (fl & TM_EP) ? C.ep_required[(size_t)e1 * 4 + c]
                                                                : (c < 2 ? -INF : INF), c);
            if (o1a >= 0) {
                rto = C.required[(size_t)o1t * 4 + c];
                ado = C.arc_delay[(size_t)o1a * 4 + c];
            }
            nd = C.net_delay[(size_t)pin * 4 + c];
            at = C.arrival[(size_t)pin * 4 + c];
        }
        if (GRAD && late) {
            if (fl & TM_ROOT) adj0 = C.adjoint[(size_t)pin * 2 + j];
            if (fl & TM_EP) {
                lse = C.lse_at[(size_t)pin * 2 + j];
                epl = C.ep_required[(size_t)e1 * 4 + 2 + j];
            }
            if (o1a >= 0) dout = C.d_arc[(size_t)o1a * 2 + j];
        }
    }
    double wgt = 0;
    if (arc_item) wgt = C.weights[(size_t)arc * 2 + j];
    __syncthreads();                                   // net records visible
    // member phase
    for (int i = tid; i < T.nm * 4; i += blockDim.x) {
        int uu = u, pp = pin, ff = fl;
        double a_r0 = r0, a_rto = rto, a_ado = ado, a_nd = nd, a_at = at, a_adj0 = adj0,
               a_lse = lse, a_epl = epl, a_dout = dout;
        if (i != tid) {           // TK_LOOP tasks: later members load here
            uu = T.m0 + (i >> 2);
            pp = t.tm_pin[uu];
            ff = t.tm_flags[uu];
            const int ot = t.tm_o1_to[uu], oa = t.tm_o1_arc[uu], ee = t.tm_e1[uu];
            if (HARD) {
                a_r0 = (ff & TM_ROOT) ? C.required[(size_t)pp * 4 + c] : init_required_multi(t, C, pp, c);
                if (oa >= 0) { a_rto = C.required[(size_t)ot * 4 + c]; a_ado = C.arc_delay[(size_t)oa * 4 + c]; }
                a_nd = C.net_delay[(size_t)pp * 4 + c];
                a_at = C.arrival[(size_t)pp * 4 + c];
            }
            if (GRAD && late) {
                if (ff & TM_ROOT) a_adj0 = C.adjoint[(size_t)pp * 2 + j];
                if (ff & TM_EP) { a_lse = C.lse_at[(size_t)pp * 2 + j]; a_epl = C.ep_required[(size_t)ee * 4 + 2 + j]; }
                if (oa >= 0) a_dout = C.d_arc[(size_t)oa * 2 + j];
            }
        }
        double v = 0, de = 0;
        bwd_member<HARD, GRAD>(t, C, uu, pp, ff, c, g, kind, a_r0, a_rto, a_ado, a_nd, a_at, a_adj0,
                               a_lse, a_epl, a_dout, v, de);
        const int qi = ff >> 8;
        const size_t f = (size_t)(S.n.f0[qi] + (uu - S.n.mptr[qi]));
        if (HARD) {
            if (loop) C.mem_buf[f * 4 + c] = v;
            else S.v[(i >> 2) * 4 + c] = v;
        }
        if (GRAD && late) {
            C.d_edge[f * 2 + j] = de;
            if (!loop) S.de[(i >> 2) * 2 + j] = de;
        }
    }
    if (arc_item) { S.w[ii * 2 + j] = wgt; S.arc[ii] = arc; }
    __syncthreads();
    if (chunk) {
        // one chunk of a big star net: ordered partial folds, last chunk combines
        const int nch = t.bn_nch[T.slot];
        const int ch = (T.m0 - S.n.mptr[0]) / TASK_M;
        double* part = C.big_part + (size_t)(t.bn_part0[T.slot] + ch) * 8;
        if (tid < 4) {
            if (HARD) {
                const bool mx = c < 2;
                double pr = mx ? -INF : INF;
                for (int k = 0; k < T.nm; k++)
                    if (later_wins(mx, pr, S.v[k * 4 + c])) pr = S.v[k * 4 + c];
                part[c] = pr;
            }
            if (GRAD && late) {
                double ps = 0.0;
                for (int k = T.nm - 1; k >= 0; k--) ps = __dadd_rn(ps, S.de[k * 2 + j]);
                part[4 + j] = ps;
            }
        }
        if (!last_chunk(C.big_ctr + 4 * T.slot + variant, nch, &S.flag)) return;
        if (tid >= 4) return;
        const int rt = S.n.root[0], fq = S.n.flags[0];
        const double* p0 = C.big_part + (size_t)t.bn_part0[T.slot] * 8;
        if (HARD) {
            const bool mx = c < 2;
            double rr = (fq & TQ_MULTI_EP) ? init_required_multi(t, C, rt, c)
                                           : merge_req(c < 2 ? -INF : INF,
                                                       (fq & TQ_ROOT_EP) ? C.ep_required[(size_t)S.n.e1[0] * 4 + c]
                                                                         : (c < 2 ? -INF : INF), c);
            for (int k = 0; k < nch; k++)
                if (later_wins(mx, rr, p0[k * 8 + c])) rr = p0[k * 8 + c];
            C.required[(size_t)rt * 4 + c] = rr;
            if (!(fq & TQ_ROOT_MEMBER)) {
                const double a = C.arrival[(size_t)rt * 4 + c];
                C.slack[(size_t)rt * 4 + c] = mx ? __dsub_rn(a, rr) : __dsub_rn(rr, a);
            }
        }
        if (GRAD && late) {
            double ar = 0.0;
            if (fq & TQ_ROOT_EP) {
                const double l = C.lse_at[(size_t)rt * 2 + j];
                ar = (fq & TQ_MULTI_EP) ? seed_multi(t, C, rt, j, l, g, kind)
                                        : __dadd_rn(0.0, seed_term(__dsub_rn(l, C.ep_required[(size_t)S.n.e1[0] * 4 + 2 + j]), g, kind));
            }
            for (int k = nch - 1; k >= 0; k--) ar = __dadd_rn(ar, p0[k * 8 + 4 + j]);
            C.adjoint[(size_t)rt * 2 + j] = ar;
            if ((fq & TQ_KIND) == ROOT_ARC)
                for (int q = 0; q < T.na; q++)
                    C.d_arc[(size_t)S.arc[q] * 2 + j] = __dmul_rn(ar, S.w[q * 2 + j]);
        }
        return;
    }
    // net phase: one (net, cond) per thread
    if (ii >= T.nq) return;
    const int rt = S.n.root[ii], fq = S.n.flags[ii];
    const int k0m = S.n.mptr[ii] - T.m0, k1m = S.n.mptr[ii + 1] - T.m0;
    if (HARD) {
        const bool mx = c < 2;
        double rr = (fq & TQ_MULTI_EP) ? init_required_multi(t, C, rt, c)
                                       : merge_req(c < 2 ? -INF : INF,
                                                   (fq & TQ_ROOT_EP) ? C.ep_required[(size_t)S.n.e1[ii] * 4 + c]
                                                                     : (c < 2 ? -INF : INF), c);
        if (loop) {
            const int s = S.n.f0[ii];
            for (int k = 0; k < k1m - k0m; k++) {
                const double v = C.mem_buf[(size_t)(s + k) * 4 + c];
                if (later_wins(mx, rr, v)) rr = v;
            }
        } else {
            for (int k = k0m; k < k1m; k++)
                if (later_wins(mx, rr, S.v[k * 4 + c])) rr = S.v[k * 4 + c];
        }
        C.required[(size_t)rt * 4 + c] = rr;
        if (!(fq & TQ_ROOT_MEMBER)) {
            const double a = C.arrival[(size_t)rt * 4 + c];
            C.slack[(size_t)rt * 4 + c] = mx ? __dsub_rn(a, rr) : __dsub_rn(rr, a);
        }
    }
    if (GRAD && late) {
        double ar = 0.0;
        if (fq & TQ_ROOT_EP) {
            const double l = C.lse_at[(size_t)rt * 2 + j];
            ar = (fq & TQ_MULTI_EP) ? seed_multi(t, C, rt, j, l, g, kind)
                                    : __dadd_rn(0.0, seed_term(__dsub_rn(l, C.ep_required[(size_t)S.n.e1[ii] * 4 + 2 + j]), g, kind));
        }
        if ((fq & TQ_TREE) || loop) {
            // parents gather children, deepest member first (diff.py:222-233)
            const int s = S.n.f0[ii];
            for (int k = k1m - k0m - 1; k >= 0; k--) {
                const double dk = C.d_edge[(size_t)(s + k) * 2 + j];
                const int pl = (fq & TQ_TREE) ? t.mem_parent_loc[s + k] : 0;
                if (pl > 0) {
                    double* dp = C.d_edge + (size_t)(s + pl - 1) * 2 + j;
                    *dp = __dadd_rn(*dp, dk);
                } else {
                    ar = __dadd_rn(ar, dk);
                }
            }
        } else {
            for (int k = k1m - 1; k >= k0m; k--) ar = __dadd_rn(ar, S.de[k * 2 + j]);
        }
        C.adjoint[(size_t)rt * 2 + j] = ar;
        if ((fq & TQ_KIND) == ROOT_ARC) {
            if (!wide) {
                for (int q = S.n.aptr[ii] - T.a0; q < S.n.aptr[ii + 1] - T.a0; q++)
                    C.d_arc[(size_t)S.arc[q] * 2 + j] = __dmul_rn(ar, S.w[q * 2 + j]);
            } else {
                for (int q = S.n.aptr[0]; q < S.n.aptr[1]; q++) {
                    const size_t a = (size_t)t.ta_arc[q];
                    C.d_arc[a * 2 + j] = __dmul_rn(ar, C.weights[a * 2 + j]);
                }
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
                                    : seed_multi(t, C, p, j, C.lse_at[(size_t)p * 2 + j], g, kind);
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
    int tasks(int li) const { return ctx.lvt_ptr_host[li + 1] - ctx.lvt_ptr_host[li]; }

    void free_pins(cudaStream_t s, bool lse)
    {
        if (!ctx.t.n_free) return;
        k_free<<<grid1(ctx.t.n_free, 256), 256, 0, s>>>(ctx.t, cs, lse);
        count++;
    }
    void rc(cudaStream_t s, int w)
    {
        if (!ctx.t.n_tasks) return;
        k_rc<<<dim3(ctx.t.n_tasks, nc), PASS_TPB, 0, s>>>(ctx.t, cs, w);
        count++;
    }
    template <bool H, bool Lse>
    void fwd(cudaStream_t s, int li, double g)
    {
        const int nt = tasks(li);
        if (nt <= 0) return;
        k_fwd<H, Lse><<<dim3(nt, nc), PASS_TPB, H ? lut_bytes : 0, s>>>(
            ctx.t, ls, cs, ctx.lvt_ptr_host[li], use_smem, g);
        count++;
    }
    template <bool H, bool G>
    void bwd(cudaStream_t s, int li, double g, int kind)
    {
        const int nt = tasks(li);
        if (nt <= 0) return;
        const int variant = H && G ? 3 : (H ? 1 : 2);
        k_bwd<H, G><<<dim3(nt, nc), PASS_TPB, 0, s>>>(ctx.t, cs, ctx.lvt_ptr_host[li], g, kind,
                                                      variant);
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
