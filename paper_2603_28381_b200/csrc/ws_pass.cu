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

#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "ws_internal.h"
#include "ws_pg.cuh"

namespace ws {

#ifndef WS_MINB
#define WS_MINB 2   // min resident blocks per SM of the level kernels
#endif
#ifndef WS_MINB_PG_BATCH
#define WS_MINB_PG_BATCH 3   // ... of the fused position-gradient backward level kernel in batches (>= 4 slots)
#endif
#ifndef WS_MINB_BATCH
#define WS_MINB_BATCH 4   // ... of the fused level kernels in corner batches (>= 4 corners)
#endif

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


// Programmatic dependent launch (sm_90+): every pass kernel lets the next
// kernel in the stream start launching immediately, runs its static prologue
// (task record, topology records, LUT staging), and only then waits for the
// previous kernel's results.  A no-op when launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
    // np.add.reduceat: the first term plus numpy's pairwise sum of the rest
    const double rest = np_pairwise(z_of, a0 + 1, a1 - a0 - 1);
    const double s = __dadd_rn(z_of(a0), rest);
    if (write_w)
        for (int q = a0; q < a1; q++) C.weights[(size_t)t.ta_arc[q] * 2 + j] = __ddiv_rn(z_of(q), s);
    return __dadd_rn(cmax, __dmul_rn(g, log(s)));
}

// ---------------------------------------------------------------------------
// pins in no net: their whole TimingState is the initial one (sta.py:51-68)

__device__ void free_pin(const Topo& t, const Corner& C, int i, bool lse)
{
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

__global__ void k_free(Topo t, Corners cs, bool lse)
{
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < t.n_free) free_pin(t, cs.c[blockIdx.y], i, lse);
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
    if (w == 0) {
        // reduce mode "sequential" of run_reference (sta.py:236-240): the
        // member loads summed by np.add.reduceat — first + pairwise rest;
        // a net without members keeps root_cap
        const double* bb = buf;
        auto get = [bb](int i) { return bb[4 * i]; };
        const double rc = C.root_cap[(size_t)net * 4 + c];
        C.load[(size_t)root * 4 + c] = m ? __dadd_rn(rc, __dadd_rn(buf[0], np_pairwise(get, 1, m - 1))) : rc;
    } else {
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
    }
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

// ---------------------------------------------------------------------------
// Task bodies shared by the per-level kernels and the persistent kernel.
// Each task kind is split into *records* (static topology: safe to load
// before the previous level finished -> PDL prologue / prefetch before the
// grid barrier) and *body* (gathers of the previous level's results and the
// compute phases).  State written by other thread blocks during the pass is
// read with ld.global.cg (L2), never through a possibly stale L1 line.

#define LDG(p) __ldcg(p)

#ifdef WS_PROBE
// per-launch block timeline: 0 start | 1 records loaded | 2 PDL wait released | 3 end | 4 SM id
// | 5-7 phases of the fused position-gradient backward level
#define LSTAMP(slot)                                                                          \
    do {                                                                                      \
        if (threadIdx.x == 0 && t.probe) {                                                    \
            unsigned long long _v;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_v));                            \
            t.probe[(size_t)blockIdx.x * 8 + (slot)] = _v;                                     \
            if ((slot) == 0) {                                                                \
                unsigned _sm;                                                                 \
                asm volatile("mov.u32 %0, %%smid;" : "=r"(_sm));                              \
                t.probe[(size_t)blockIdx.x * 8 + 4] = _sm;                                    \
            }                                                                                 \
        }                                                                                     \
    } while (0)
#else
#define LSTAMP(slot) do { } while (0)
#endif

// WS_PROBE builds: phase stamps inside task bodies of the persistent kernel
// (plev >= 0), laid out after the per-level stamps
#ifdef WS_PROBE
#define BSTAMP(slot)                                                                          \
    do {                                                                                      \
        if (plev >= 0 && threadIdx.x == 0 && t.probe) {                                       \
            unsigned long long _v;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_v));                            \
            t.probe[(size_t)2 * t.L * 2048 * 4 + ((size_t)plev * 2048 + blockIdx.x) * 4 + (slot)] = _v; \
        }                                                                                     \
    } while (0)
#else
#define BSTAMP(slot) do { (void)plev; } while (0)
#endif

// ---- RC --------------------------------------------------------------------

struct RcSmem {
    NetSmem n;
    double cap[TASK_M * 4];
    int flag;
};

struct RcRec {
    int pin[ITEMS], fl[ITEMS];
};

__device__ __forceinline__ void rc_records(const Topo& t, const Task& T, RcSmem& S, RcRec& R)
{
    load_nets(t, T, S.n);
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int mi = (threadIdx.x >> 2) + k * TASK_Q;
        R.pin[k] = -1;
        if (mi < T.nm && !(T.flags & TK_LOOP)) {
            R.pin[k] = t.tm_pin[T.m0 + mi];
            R.fl[k] = t.tm_flags[T.m0 + mi];
        }
    }
}

__device__ void rc_body(const Topo& t, const Corner& C, const Task& T, RcSmem& S, const RcRec& R,
                        int w)
{
    const int tid = threadIdx.x, c = tid & 3;
    const bool fast = w == 8;
    __syncthreads();                         // net records visible
    // member phase (star nets, w == 8): one (member, cond) per item
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int mi = (tid >> 2) + k * TASK_Q;
        if (R.pin[k] < 0) continue;
        const int qi = R.fl[k] >> 8;
        if (!fast || (S.n.flags[qi] & TQ_TREE)) continue;
        const size_t f = (size_t)(S.n.f0[qi] + (T.m0 + mi - S.n.mptr[qi]));
        const double b = C.mem_cap[f * 4 + c];
        const double r = C.mem_res[f * 4 + c];
        const double d = __dadd_rn(0.0, __dmul_rn(r, b));
        const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r), b), d), __dmul_rn(d, d));
        const size_t pin = (size_t)R.pin[k];
        if (!(R.fl[k] & TM_ROOT)) C.load[pin * 4 + c] = b;
        C.net_delay[pin * 4 + c] = d;
        C.impulse[pin * 4 + c] = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
        S.cap[mi * 4 + c] = b;
    }
    if (T.flags & TK_CHUNK) {
        // big star net: the last chunk sums every member's cap in order
        const int root = S.n.root[0], net = S.n.net[0], s = S.n.f0[0];
        const int m = S.n.mptr[1] - S.n.mptr[0];
        const bool last = last_chunk(C.big_ctr + 4 * T.slot + 0, t.bn_nch[T.slot], &S.flag);
        if (last && tid < 4) {
            if (!fast) {
                rc_seq(t, C, net, root, s, m, tid, w, S.n.flags[0] & TQ_ROOT_MEMBER);
            } else {
                const double l = root_load8(C.mem_cap + (size_t)s * 4 + tid, 4, m);
                C.load[(size_t)root * 4 + tid] = __dadd_rn(C.root_cap[(size_t)net * 4 + tid], l);
                if (!(S.n.flags[0] & TQ_ROOT_MEMBER)) {
                    C.net_delay[(size_t)root * 4 + tid] = 0.0;
                    C.impulse[(size_t)root * 4 + tid] = 0.0;
                }
            }
        }
        __syncthreads();
        return;
    }
    __syncthreads();
    // net phase: root loads
    const int qi = tid >> 2;
    if (qi < T.nq) {
        const int fq = S.n.flags[qi], root = S.n.root[qi], net = S.n.net[qi];
        const int m = S.n.mptr[qi + 1] - S.n.mptr[qi];
        if (!fast || (fq & TQ_TREE) || (T.flags & TK_LOOP)) {
            rc_seq(t, C, net, root, S.n.f0[qi], m, c, w, fq & TQ_ROOT_MEMBER);
        } else {
            const double l = root_load8(S.cap + (S.n.mptr[qi] - T.m0) * 4 + c, 4, m);
            C.load[(size_t)root * 4 + c] = __dadd_rn(C.root_cap[(size_t)net * 4 + c], l);
            if (!(fq & TQ_ROOT_MEMBER)) {
                C.net_delay[(size_t)root * 4 + c] = 0.0;
                C.impulse[(size_t)root * 4 + c] = 0.0;
            }
        }
    }
    __syncthreads();                         // smem reusable by the next task
}

// ---- forward level (forward_level, _kernels.pyx:159-210) + LSE (diff.py:123-146)
//
// Net-centric: the thread of (net, cond) item (qi, c) evaluates all in-arcs
// of its net itself (generated netlists have <= 3 in-arcs per net; up to
// FWD_NA are held in registers, more take a loop over global records), so
// the arc delays, the ordered max/min merge, the winner's output slew and
// the whole LSE (max, exp, reduceat sum, log, softmax weights) need no
// shared-memory exchange and no barrier.  One barrier then publishes the
// root results to the member phase.

constexpr int FWD_NA = 3;

struct FwdSmem {
    NetSmem n;
    double at[TASK_Q * 4], sl[TASK_Q * 4], lr[TASK_Q * 2];   // root results
};

struct FwdRec {
    int na, a0;                       // the net item's in-arcs: ta_*[a0 .. a0 + na)
    int from[FWD_NA], arc[FWD_NA];
    int dl[FWD_NA], sl[FWD_NA];
    int mpin[ITEMS], mfl[ITEMS];
    int nroot, nflags;                // this lane's (net, cond) item
    // pass-static gathers (RC outputs), prefetched by the persistent kernel
    double ld, mnd[ITEMS], mim[ITEMS];
};


template <bool HARD>
__device__ __forceinline__ void fwd_records(const Topo& t, const Task& T, FwdSmem& S, FwdRec& R)
{
    load_nets(t, T, S.n);
    const int c = threadIdx.x & 3, qi = threadIdx.x >> 2;
    const bool wide = T.flags & TK_WIDE;
    R.nroot = -1;
    R.na = 0;
    if (qi < T.nq) {
        const int q = T.q0 + qi;
        R.nroot = t.tq_root[q];
        R.nflags = t.tq_flags[q];
        if ((R.nflags & TQ_KIND) == ROOT_ARC && !wide) {
            R.a0 = t.tq_aptr[q];
            R.na = t.tq_aptr[q + 1] - R.a0;
            if (R.na > 0 && R.na <= FWD_NA) {
                // slots past the last arc repeat arc 0: the net phase then
                // runs FWD_NA independent chains without branches
#pragma unroll
                for (int k = 0; k < FWD_NA; k++) {
                    const int qa = R.a0 + (k < R.na ? k : 0);
                    R.from[k] = t.ta_from[qa];
                    R.arc[k] = t.ta_arc[qa];
                    if (HARD) {
                        R.dl[k] = lut_id(t.ta_lut + (2 * (size_t)qa), c);
                        R.sl[k] = lut_id(t.ta_lut + (2 * (size_t)qa + 1), c);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int ii = qi + k * TASK_Q;
        R.mpin[k] = -1;
        if (ii < T.nm) {
            R.mpin[k] = t.tm_pin[T.m0 + ii];
            R.mfl[k] = t.tm_flags[T.m0 + ii];
        }
    }
}



// arc-driven root with more than FWD_NA (but <= TASK_A) in-arcs: the same
// arithmetic in the same order, records read in a loop
template <bool HARD, bool LSE>
__device__ void fwd_net_loop(const Topo& t, const LutView& L, const Corner& C, int a0, int a1, int rt,
                             double ld, int c, double g, bool first, double& at, double& sl, double& lr)
{
    const bool late = c >= 2;
    if (HARD) {
        double best = late ? -INF : INF;
        int wq = a0;
        for (int q = a0; q < a1; q++) {
            const double d = lut_interp(L, lut_id(t.ta_lut + (2 * (size_t)q), c),
                                        LDG(C.slew + (size_t)t.ta_from[q] * 4 + c), ld);
            C.arc_delay[(size_t)t.ta_arc[q] * 4 + c] = d;
            const double v = __dadd_rn(LDG(C.arrival + (size_t)t.ta_from[q] * 4 + c), d);
            if (later_wins(late, best, v)) { best = v; wq = q; }
        }
        at = best;
        sl = lut_interp(L, lut_id(t.ta_lut + (2 * (size_t)wq + 1), c), LDG(C.slew + (size_t)t.ta_from[wq] * 4 + c), ld);
    }
    if (LSE && late) lr = lse_root_global(t, C, a0, a1, c, g, first);
}

// the root of a TK_WIDE task (> TASK_A in-arcs): arc delays are in global
template <bool HARD, bool LSE>
__device__ void fwd_net_wide(const Topo& t, const LutView& L, const Corner& C, int qa0, int qa1,
                                          int rt, int c, double g, bool first, double& at, double& sl,
                                          double& lr)
{
    const bool late = c >= 2;
    if (HARD) {
        double best = late ? -INF : INF;
        int wq = qa0;
        for (int q = qa0; q < qa1; q++) {
            const double v = __dadd_rn(LDG(C.arrival + (size_t)t.ta_from[q] * 4 + c),
                                       LDG(C.arc_delay + (size_t)t.ta_arc[q] * 4 + c));
            if (later_wins(late, best, v)) { best = v; wq = q; }
        }
        at = best;
        sl = lut_interp(L, lut_id(t.ta_lut + (2 * (size_t)wq + 1), c),
                        LDG(C.slew + (size_t)t.ta_from[wq] * 4 + c), LDG(C.load + (size_t)rt * 4 + c));
    }
    if (LSE && late) lr = lse_root_global(t, C, qa0, qa1, c, g, first);
}

// arc delays of a TK_WIDE task, all block threads
__device__ void fwd_wide_delays(const Topo& t, const LutView& L, const Corner& C, const Task& T,
                                             int rt)
{
    for (int i = threadIdx.x; i < T.na * 4; i += blockDim.x) {
        const int q = T.a0 + (i >> 2), cc = i & 3;
        const int fp = t.ta_from[q];
        const double d = lut_interp(L, lut_id(t.ta_lut + (2 * (size_t)q), cc),
                                    LDG(C.slew + (size_t)fp * 4 + cc), LDG(C.load + (size_t)rt * 4 + cc));
        C.arc_delay[(size_t)t.ta_arc[q] * 4 + cc] = d;
    }
}

// The (net, cond) item of a forward level: in-arcs of the net in arc order
// (first arc wins ties), the winner's output slew, the LSE of the late
// columns; writes the arc delays, weights and the root's arrival / slew /
// lse (when `first`).  The LSE shuffles need the net's four cond lanes
// together in one quad.
template <bool HARD, bool LSE>
__device__ __forceinline__ void fwd_net_item(const Topo& t, const LutView& L, const Corner& C, const FwdRec& R,
                                             int kind, int rt, bool wide, int wa0, int wa1, bool first,
                                             const double* slf, const double* atf, const double* xl, double* dd,
                                             double ld, double n_at, double n_sl, double n_lr, int c, double g,
                                             double ginv, double& at, double& sl, double& lr)
{
    const bool late = c >= 2;
    const int j = c - 2;
    if (kind == ROOT_ARC) {
        if (wide) {
            fwd_net_wide<HARD, LSE>(t, L, C, wa0, wa1, rt, c, g, first, at, sl, lr);
        } else if (R.na > FWD_NA) {
            fwd_net_loop<HARD, LSE>(t, L, C, R.a0, R.a0 + R.na, rt, ld, c, g, first, at, sl, lr);
        } else {
            if (HARD) {
                // every slot's delay and output slew (independent chains),
                // then the ordered merge; the root load is located once
                // on the first arc's load axis
                // every slot's delay (independent chains) and the ordered
                // merge (first arc wins ties); only the winner's output slew
                // is interpolated, reusing its located cells when the slew
                // table shares the delay table's axes.  The root load is
                // located once on the first arc's load axis.
                const int4 d0 = L.info[R.dl[0]];
                const Loc ll0 = lut_locate(L.l + d0.z, d0.w, ld);
                double best = late ? -INF : INF;
                Loc wls{}, wll{};
                int4 wdi = d0;
                int wsl = R.sl[0];
                double wslf = slf[0];
#pragma unroll
                for (int k = 0; k < FWD_NA; k++) {
                    const int4 di = L.info[R.dl[k]];
                    const Loc lsd = lut_locate(L.s + di.x, di.y, slf[k]);
                    const Loc lld = (di.z == d0.z && di.w == d0.w) ? ll0 : lut_locate(L.l + di.z, di.w, ld);
                    dd[k] = lut_blend(L.t + L.t_ptr[R.dl[k]], di.w, lsd, lld);
                    if (k == 0) { wls = lsd; wll = lld; }   // the slot-0 default (no strict winner)
                    if (k < R.na) {
                        C.arc_delay[(size_t)R.arc[k] * 4 + c] = dd[k];
                        const double v = __dadd_rn(atf[k], dd[k]);
                        if (later_wins(late, best, v)) {
                            best = v;
                            wls = lsd; wll = lld; wdi = di; wsl = R.sl[k]; wslf = slf[k];
                        }
                    }
                }
                {
                    const int4 si = L.info[wsl];
                    const Loc lss = (si.x == wdi.x && si.y == wdi.y) ? wls : lut_locate(L.s + si.x, si.y, wslf);
                    const Loc lls = (si.z == wdi.z && si.w == wdi.w) ? wll : lut_locate(L.l + si.z, si.w, ld);
                    sl = lut_blend(L.t + L.t_ptr[wsl], si.w, lss, lls);
                }
                at = best;
            }
            if (LSE) {
                // The LSE of the two late columns, spread over the
                // net's 4 lanes: column j's owner (lane 2 + j) forms
                // x = lse_at[from] + delay and its first max am; of the
                // (column, in-arc) exponentials only the <= 4 non-max
                // ones are not exactly 1, so lane c takes column c >> 1's
                // (c & 1)-th non-max in-arc: one exp per lane instead
                // of three on the late lanes.  Same arithmetic as the
                // reference order (np.maximum.reduceat, z0 + sequential
                // rest, z / s).
                const int qb = threadIdx.x & 28;                 // the quad's cond-0 lane
                const unsigned qmask = 0xFu << qb;
                double x0 = 0.0, x1 = 0.0, x2 = 0.0, cm = -INF;
                int am = 0;
                if (late) {
                    x0 = __dadd_rn(xl[0], dd[0]);
                    x1 = __dadd_rn(xl[1], dd[1]);
                    x2 = __dadd_rn(xl[2], dd[2]);
                    cm = x0;                                       // np.maximum.reduceat
                    if (1 < R.na && x1 > cm) { cm = x1; am = 1; }
                    if (2 < R.na && x2 > cm) { cm = x2; am = 2; }
                }
                const double d0 = __dsub_rn(x0, cm), d1 = __dsub_rn(x1, cm), d2 = __dsub_rn(x2, cm);
                const int own = qb + 2 + (c >> 1);                // owner of column c >> 1
                const int amj = __shfl_sync(qmask, am, own);
                const double dA = __shfl_sync(qmask, am == 0 ? d1 : d0, own);   // first non-max
                const double dB = __shfl_sync(qmask, am == 2 ? d1 : d2, own);   // second non-max
                const int i1 = c & 1, kk = i1 + (i1 >= amj ? 1 : 0);
                const double dm = i1 ? dB : dA;
                // the max element's +0 / g = +0 and exp(+0) = 1 need no
                // division (whose zero dividend takes the IEEE slow path)
                // exp((x - max) / gamma) with 1 / gamma from the host (the
                // argument within an ulp and a half of the quotient's)
                const double e = (kk >= R.na || dm == 0.0) ? 1.0 : exp(__dmul_rn(dm, ginv));
                const double zA = __shfl_sync(qmask, e, qb + 2 * i1);
                const double zB = __shfl_sync(qmask, e, qb + 2 * i1 + 1);
                double sc = 1.0;
                if (late) {
                    const double z0 = am == 0 ? 1.0 : zA;
                    const double z1 = am == 1 ? 1.0 : (am == 0 ? zA : zB);
                    const double z2 = am == 2 ? 1.0 : zB;
                    double rest = 0.0;
                    if (1 < R.na) rest = __dadd_rn(rest, z1);   // reduceat: z0 + sequential (n < 9)
                    if (2 < R.na) rest = __dadd_rn(rest, z2);
                    sc = __dadd_rn(z0, rest);
                    lr = __dadd_rn(cm, __dmul_rn(g, log(sc)));
                }
                if (first) {
                    // weights z / s: the owner's 1 / s (its column's max,
                    // z = 1, exactly) and every lane's non-max in-arc of
                    // column c >> 1 as z * (1 / s) (within an ulp of z / s:
                    // one division per column instead of one per weight)
                    const double rinv = late ? __ddiv_rn(1.0, sc) : 0.0;
                    const double rj = __shfl_sync(qmask, rinv, own);
                    auto arc_of = [&](int k) { return k == 0 ? R.arc[0] : (k == 1 ? R.arc[1] : R.arc[2]); };
                    if (kk < R.na) C.weights[(size_t)arc_of(kk) * 2 + (c >> 1)] = __dmul_rn(e, rj);
                    if (late) C.weights[(size_t)arc_of(am) * 2 + j] = rinv;
                }
            }
        }
        if (first) {
            if (HARD) {
                C.arrival[(size_t)rt * 4 + c] = at;
                C.slew[(size_t)rt * 4 + c] = sl;
            }
            if (LSE && late) C.lse_at[(size_t)rt * 2 + j] = lr;
        }
    } else if (kind == ROOT_FEED) {
        // driven by its parent net's member update (a lower level)
        at = n_at;
        sl = n_sl;
        lr = n_lr;
    } else {
        // primary-input root (or undriven): the seeded values
        at = n_at;
        sl = n_sl;
        lr = at;
        if (first) {
            if (HARD) {
                C.arrival[(size_t)rt * 4 + c] = at;
                C.slew[(size_t)rt * 4 + c] = sl;
            }
            if (LSE && late) C.lse_at[(size_t)rt * 2 + j] = at;
        }
    }
}

template <bool HARD, bool LSE, bool STATIC = false>
__device__ void fwd_body(const Topo& t, const LutView& L, const Corner& C, const Task& T,
                         FwdSmem& S, const FwdRec& R, double g, double ginv, int plev = -1)
{
    const int tid = threadIdx.x, c = tid & 3, qi = tid >> 2;
    const bool late = c >= 2;
    const int j = c - 2;
    const bool wide = T.flags & TK_WIDE;
    // ---- R3: every gather of the task at once
    double slf[FWD_NA], atf[FWD_NA], xl[FWD_NA], dd[FWD_NA], mnd[ITEMS], mim[ITEMS];
    double ld = 0;
#pragma unroll
    for (int k = 0; k < FWD_NA; k++) {
        slf[k] = atf[k] = xl[k] = dd[k] = 0.0;
        if (R.na > 0 && R.na <= FWD_NA) {
            if (HARD) {
                slf[k] = LDG(C.slew + (size_t)R.from[k] * 4 + c);
                atf[k] = LDG(C.arrival + (size_t)R.from[k] * 4 + c);
            } else {
                dd[k] = LDG(C.arc_delay + (size_t)R.arc[k] * 4 + c);
            }
            if (LSE && late) xl[k] = LDG(C.lse_at + (size_t)R.from[k] * 2 + j);
        }
    }
    if (HARD && R.na > 0) ld = STATIC ? R.ld : LDG(C.load + (size_t)R.nroot * 4 + c);
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        mnd[k] = mim[k] = 0.0;
        if (R.mpin[k] >= 0) {
            if (STATIC) {
                mnd[k] = R.mnd[k];
                if (HARD) mim[k] = R.mim[k];
            } else {
                mnd[k] = LDG(C.net_delay + (size_t)R.mpin[k] * 4 + c);
                if (HARD) mim[k] = LDG(C.impulse + (size_t)R.mpin[k] * 4 + c);
            }
        }
    }
    // seeds of roots not driven by an in-arc
    double n_at = 0, n_sl = 0, n_lr = 0;
    if (R.nroot >= 0) {
        const int kind = R.nflags & TQ_KIND;
        if (kind == ROOT_FEED) {
            if (HARD) {
                n_at = LDG(C.arrival + (size_t)R.nroot * 4 + c);
                n_sl = LDG(C.slew + (size_t)R.nroot * 4 + c);
            }
            if (LSE && late) n_lr = LDG(C.lse_at + (size_t)R.nroot * 2 + j);
        } else if (kind != ROOT_ARC && (R.nflags & TQ_ROOT_PI)) {
            const int pi = t.pin_pi[R.nroot];
            n_at = C.pi_arrival[(size_t)pi * 4 + c];
            n_sl = C.pi_slew[(size_t)pi * 4 + c];
        }
    }
    if (!STATIC) asm volatile("cp.async.wait_all;" ::: "memory");   // the LUT pool (stage_luts_async)
    __syncthreads();                  // net records (and the LUT pool) visible
    BSTAMP(0);
    if (HARD && wide) {
        // one net with > TASK_A in-arcs: arc delays in a loop, merge from global
        fwd_wide_delays(t, L, C, T, S.n.root[0]);
        __syncthreads();
    }
    BSTAMP(1);
    // ---- net phase: in-arcs of the own net, merge in arc order (first arc
    // wins ties), winner's output slew, LSE
    const bool first = !(T.flags & TK_CHUNK) || T.m0 == S.n.mptr[0];
    if (qi < T.nq) {
        const int fl = S.n.flags[qi];
        const int kind = fl & TQ_KIND;
        const int rt = S.n.root[qi];
        double at = 0, sl = 0, lr = 0;
        fwd_net_item<HARD, LSE>(t, L, C, R, kind, rt, wide, S.n.aptr[0], S.n.aptr[1], first, slf, atf, xl, dd,
                                ld, n_at, n_sl, n_lr, c, g, ginv, at, sl, lr);
        if (HARD) { S.at[qi * 4 + c] = at; S.sl[qi * 4 + c] = sl; }
        if (LSE && late) S.lr[qi * 2 + j] = lr;
    }
    __syncthreads();
    BSTAMP(2);
    // ---- member phase: one (member, cond) per item
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        if (R.mpin[k] < 0) continue;
        const size_t pin = (size_t)R.mpin[k];
        const int mq = R.mfl[k] >> 8;
        if (HARD) {
            const double sr = S.sl[mq * 4 + c];
            C.arrival[pin * 4 + c] = __dadd_rn(S.at[mq * 4 + c], mnd[k]);
            C.slew[pin * 4 + c] = __dsqrt_rn(__dadd_rn(__dmul_rn(sr, sr), __dmul_rn(mim[k], mim[k])));
        }
        if (LSE && late) C.lse_at[pin * 2 + j] = __dadd_rn(S.lr[mq * 2 + j], mnd[k]);
    }
    for (int i = tid + ITEMS * PASS_TPB; i < T.nm * 4; i += blockDim.x) {   // TK_LOOP tasks
        const int u = T.m0 + (i >> 2);
        const size_t pin = (size_t)t.tm_pin[u];
        const int mq = t.tm_flags[u] >> 8;
        const double nd = LDG(C.net_delay + pin * 4 + c);
        if (HARD) {
            const double sr = S.sl[mq * 4 + c], im = LDG(C.impulse + pin * 4 + c);
            C.arrival[pin * 4 + c] = __dadd_rn(S.at[mq * 4 + c], nd);
            C.slew[pin * 4 + c] = __dsqrt_rn(__dadd_rn(__dmul_rn(sr, sr), __dmul_rn(im, im)));
        }
        if (LSE && late) C.lse_at[pin * 2 + j] = __dadd_rn(S.lr[mq * 2 + j], nd);
    }
    if (STATIC) __syncthreads();             // (persistent kernel) smem reusable by the next task
}

// ---- backward level (backward_level, _kernels.pyx:213-249) + reverse adjoint
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

// k_bwd<..., PG>: the position-gradient sweep's per-task shared state, in
// dynamic shared memory after the staged LUT pool.  Late columns only
// (double2 = conds 2, 3).  The pass-static inputs are prefetched by
// cp.async in the prologue (before the PDL wait), the sweep-dynamic ones
// (higher levels' gsa / gsr) right after it, so the sweep step adds no
// dependent global round trip to the level.
struct PgSmem {
    double pt[TASK_M * 2], px[TASK_M * 2], py[TASK_M * 2];   // member terms t, x, y
    double2 pm[TASK_M * 6];    // slew, impulse, net_delay of the pin; mem_res, mem_cap; root slew
    double2 pgsa[TASK_M], pgsr[TASK_M];   // gsa of the first out-arc, gsr of the pin
    int4 pmr[TASK_M];          // pin, first out-arc, tm_flags, original member index
    double2 pa[TASK_A * 3];    // in-arcs: arrival[from], arc_delay[arc], slew[from]
    int4 plut[TASK_A];         // delay LUT ids (cond 2, 3), slew LUT ids (cond 2, 3)
    int aq[TASK_A];            // net of the in-arc within the task
    double da[TASK_A * 2];     // d_arc of the in-arcs (net phase)
    double term[TASK_A * 2];   // dL/dload terms of the in-arcs
    double2 pl[TASK_Q];        // root load
    double groot[TASK_Q * 2], slw[TASK_Q * 2], wss[TASK_Q * 2];   // root slew adjoint; winner's dS/dload, dS/dslew
    int win[TASK_Q * 2];       // first strict late max in-arc (-1: none)
    int2 pop[TASK_Q];          // the root's out-arcs: pin_out_arc[x .. y)
};

// the prologue prefetch of a task whose nets lie within it (not chunked,
// looped or wide): records by plain loads, pass state by cp.async.  The
// first half of the block takes the members, the second the in-arcs and
// nets, so no thread's copies wait behind another item's record loads.
__device__ void pg_prefetch_static(const Topo& t, const PgDev& pd, const Corner& C, const Task& T,
                                   PgSmem& P)
{
    constexpr int H = PASS_TPB / 2;
    if (threadIdx.x < H) {
        for (int i = threadIdx.x; i < T.nm; i += H) {
            const int u = T.m0 + i;
            const int pin = t.tm_pin[u], f = pd.tm_f[u], root = pd.tm_root[u];
            P.pmr[i] = make_int4(pin, t.tm_o1_arc[u], t.tm_flags[u], f);
            pg::cp16(&P.pm[i * 6 + 0], C.slew + (size_t)pin * 4 + 2);
            pg::cp16(&P.pm[i * 6 + 1], C.impulse + (size_t)pin * 4 + 2);
            pg::cp16(&P.pm[i * 6 + 2], C.net_delay + (size_t)pin * 4 + 2);
            pg::cp16(&P.pm[i * 6 + 3], C.mem_res + (size_t)f * 4 + 2);
            pg::cp16(&P.pm[i * 6 + 4], C.mem_cap + (size_t)f * 4 + 2);
            pg::cp16(&P.pm[i * 6 + 5], C.slew + (size_t)root * 4 + 2);
        }
    } else {
        for (int s = threadIdx.x - H; s < max(T.na, T.nq); s += H) {
            int root = -1;
            if (s < T.nq) root = t.tq_root[T.q0 + s];
            if (s < T.na) {
                const int qa = T.a0 + s;
                const int from = t.ta_from[qa], arc = t.ta_arc[qa];
                const int4 dl = t.ta_lut[2 * (size_t)qa], sl = t.ta_lut[2 * (size_t)qa + 1];
                P.plut[s] = make_int4(dl.z, dl.w, sl.z, sl.w);
                P.aq[s] = t.ta_q[qa];
                pg::cp16(&P.pa[3 * s + 0], C.arrival + (size_t)from * 4 + 2);
                pg::cp16(&P.pa[3 * s + 1], C.arc_delay + (size_t)arc * 4 + 2);
                pg::cp16(&P.pa[3 * s + 2], C.slew + (size_t)from * 4 + 2);
            }
            if (root >= 0) {
                pg::cp16(&P.pl[s], C.load + (size_t)root * 4 + 2);
                P.pop[s] = make_int2(t.pin_out_ptr[root], t.pin_out_ptr[root + 1]);
            }
        }
    }
    pg::cp_commit();
}

// after the PDL wait: the higher levels' gsa / gsr (same thread mapping as
// the static prefetch, so P.pmr[i] is the thread's own write)
__device__ void pg_prefetch_dyn(const PlaceCorner& G, const Task& T, PgSmem& P)
{
    constexpr int H = PASS_TPB / 2;
    if (threadIdx.x < H)
    for (int i = threadIdx.x; i < T.nm; i += H) {
        const int4 r = P.pmr[i];
        if (r.y >= 0) pg::cp16(&P.pgsa[i], G.gsa + (size_t)r.y * 2);
        if (r.z & TM_ROOT) pg::cp16(&P.pgsr[i], G.gsr + (size_t)r.x * 2);
    }
    pg::cp_commit();
}

struct BwdRec {
    int pin[ITEMS], fl[ITEMS], o1t[ITEMS], o1a[ITEMS], e1[ITEMS], arc[ITEMS], no[ITEMS], o0[ITEMS];
    int nroot, nflags, ne1;     // this lane's (net, cond) item
    // pass-static gathers (forward outputs), prefetched by the persistent kernel
    double ado[ITEMS], nd[ITEMS], at[ITEMS], lse[ITEMS], epl[ITEMS], wgt[ITEMS], r0[ITEMS];
    double n_at, n_rr, n_seed;
};

template <bool GRAD>
__device__ __forceinline__ void bwd_records(const Topo& t, const Task& T, BwdSmem& S, BwdRec& R)
{
    load_nets(t, T, S.n);
    const bool late = (threadIdx.x & 3) >= 2;
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int ii = (threadIdx.x >> 2) + k * TASK_Q;
        R.pin[k] = -1;
        if (ii < T.nm) {
            const int u = T.m0 + ii;
            R.pin[k] = t.tm_pin[u];
            R.fl[k] = t.tm_flags[u];
            R.o1t[k] = t.tm_o1_to[u];
            R.o1a[k] = t.tm_o1_arc[u];
            R.e1[k] = t.tm_e1[u];
            R.o0[k] = t.tm_optr[u];
            R.no[k] = t.tm_optr[u + 1] - R.o0[k];
        }
        R.arc[k] = -1;
        if (GRAD && late && ii < T.na && !(T.flags & TK_WIDE)) R.arc[k] = t.ta_arc[T.a0 + ii];
    }
    R.nroot = -1;
    const int qi = threadIdx.x >> 2;
    if (qi < T.nq) {
        const int q = T.q0 + qi;
        R.nroot = t.tq_root[q];
        R.nflags = t.tq_flags[q];
        R.ne1 = t.tq_e1[q];
    }
}


// one member (u, c): fold required over out-arcs, slack, adjoint.
template <bool HARD, bool GRAD>
__device__ __forceinline__ void bwd_member(const Topo& t, const Corner& C, int o0, int o1, int pin,
                                           int fl, int c, double g, int kind, double r0, double rto,
                                           double ado, double nd, double at, double adj0,
                                           double lse, double epl, double dout, double& v,
                                           double& de)
{
    if (HARD) {
        const bool mx = c < 2;
        // pins with several endpoint entries merge their RATs here, not in
        // the gather round (keeps its loads straight-line)
        double r = ((fl & TM_MULTI_EP) && !(fl & TM_ROOT)) ? init_required_multi(t, C, pin, c) : r0;
        if (o1 > o0) {
            const double vv = __dsub_rn(rto, ado);
            if (later_wins(mx, r, vv)) r = vv;
            for (int o = o0 + 1; o < o1; o++) {
                const double v2 = __dsub_rn(LDG(C.required + (size_t)t.to_to[o] * 4 + c),
                                            LDG(C.arc_delay + (size_t)t.to_arc[o] * 4 + c));
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
            for (int o = o0 + 1; o < o1; o++) ad = __dadd_rn(ad, LDG(C.d_arc + (size_t)t.to_arc[o] * 2 + j));
        }
        C.adjoint[(size_t)pin * 2 + j] = ad;
        de = ad;
    }
}

template <bool HARD, bool GRAD>
__device__ __forceinline__ void bwd_gather(const Corner& C, int pin, int fl, int o1t, int o1a,
                                           int e1, int c, const Topo& t, double& r0, double& rto,
                                           double& ado, double& nd, double& at, double& adj0,
                                           double& lse, double& epl, double& dout)
{
    const int j = c - 2;
    if (HARD) {
        if (fl & TM_ROOT) r0 = LDG(C.required + (size_t)pin * 4 + c);
        else if (fl & TM_MULTI_EP) r0 = 0.0;      // merged in bwd_member
        // merge_req(+-INF, x) is x bit for bit (x = +-INF returns the same
        // infinity, NaN stays NaN): the single endpoint RAT or the identity
        else r0 = (fl & TM_EP) ? C.ep_required[(size_t)e1 * 4 + c] : (c < 2 ? -INF : INF);
        if (o1a >= 0) {
            rto = LDG(C.required + (size_t)o1t * 4 + c);
            ado = LDG(C.arc_delay + (size_t)o1a * 4 + c);
        }
        nd = LDG(C.net_delay + (size_t)pin * 4 + c);
        at = LDG(C.arrival + (size_t)pin * 4 + c);
    }
    if (GRAD && c >= 2) {
        if (fl & TM_ROOT) adj0 = LDG(C.adjoint + (size_t)pin * 2 + j);
        if (fl & TM_EP) {
            lse = LDG(C.lse_at + (size_t)pin * 2 + j);
            epl = C.ep_required[(size_t)e1 * 4 + 2 + j];
        }
        if (o1a >= 0) dout = LDG(C.d_arc + (size_t)o1a * 2 + j);
    }
}

__device__ __forceinline__ double root_init_required(const Topo& t, const Corner& C, int rt, int fq,
                                                      int e1, int c)
{
    if (fq & TQ_MULTI_EP) return init_required_multi(t, C, rt, c);
    // merge_req(+-INF, x) == x bit for bit
    return (fq & TQ_ROOT_EP) ? C.ep_required[(size_t)e1 * 4 + c] : (c < 2 ? -INF : INF);
}

__device__ __forceinline__ double root_seed(const Topo& t, const Corner& C, int rt, int fq, int e1,
                                            int j, double g, int kind)
{
    if (!(fq & TQ_ROOT_EP)) return 0.0;
    const double l = LDG(C.lse_at + (size_t)rt * 2 + j);
    if (fq & TQ_MULTI_EP) return seed_multi(t, C, rt, j, l, g, kind);
    return __dadd_rn(0.0, seed_term(__dsub_rn(l, C.ep_required[(size_t)e1 * 4 + 2 + j]), g, kind));
}



// PG (fused mode with position gradients): the level's position-gradient
// sweep step (ws_pg.cuh) runs inside the backward level kernel once the
// members' adjoints and the in-arcs' d_arc are final: member terms after
// the member phase, the per-net step after the net phase.
// The net step of the sweep for a task whose nets lie within it, phase-
// parallel over the task (the arithmetic and order of pg::pg_net_group, so
// both sweeps agree bit for bit): (net, j) member-term sum, root, winner ->
// (in-arc, j) LUT partials, gsa, dL/dload terms -> (net, j) dL/dload and
// (member, j) d_cap.  RC-tree nets run the oracle's recursion.
__device__ void pg_task_nets(const Topo& t, const LutView& L, const Corner& C, const PlaceCorner& G,
                             const Task& T, const BwdSmem& S, PgSmem& P)
{
    const int tid = threadIdx.x;
    auto late = [](double2 v, int j) { return j ? v.y : v.x; };
    for (int i = tid; i < T.nq * 2; i += blockDim.x) {
        const int ii = i >> 1, j = i & 1;
        const int fl = S.n.flags[ii], kind = fl & TQ_KIND, root = S.n.root[ii];
        const int mb = S.n.mptr[ii] - T.m0, m = S.n.mptr[ii + 1] - S.n.mptr[ii];
        // root-slew terms: 8 interleaved partials P(k mod 8), combined
        // ((P0 + P1) + (P2 + P3)) + ((P4 + P5) + (P6 + P7)) (pg_net_group's order)
        double pp[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int k = 0; k < m; k += 8)
#pragma unroll
            for (int a = 0; a < 8; a++)
                if (k + a < m) pp[a] = __dadd_rn(pp[a], P.pt[(mb + k + a) * 2 + j]);
        const double gsum = __dadd_rn(__dadd_rn(__dadd_rn(pp[0], pp[1]), __dadd_rn(pp[2], pp[3])),
                                      __dadd_rn(__dadd_rn(pp[4], pp[5]), __dadd_rn(pp[6], pp[7])));
        double groot = gsum;
        if (kind == ROOT_FEED) {
            G.gsr[(size_t)root * 2 + j] = gsum;
        } else {
            for (int v = P.pop[ii].x; v < P.pop[ii].y; v++)
                groot = __dadd_rn(groot, __ldcg(G.gsa + (size_t)t.pin_out_arc[v] * 2 + j));
            G.gs[(size_t)root * 2 + j] = groot;
        }
        int w = -1;
        if (kind == ROOT_ARC) {
            double best = -INF;
            const int s0 = S.n.aptr[ii] - T.a0, na = S.n.aptr[ii + 1] - S.n.aptr[ii];
            for (int k = 0; k < na; k++) {
                const double v = __dadd_rn(late(P.pa[3 * (s0 + k)], j), late(P.pa[3 * (s0 + k) + 1], j));
                if (v > best) { best = v; w = k; }
            }
            if (w >= 0) {   // the winner's slew-LUT partials (its gsa term and dS/dload)
                const int sw = s0 + w;
                double ss, sl;
                pg::interp_grad(L, j ? P.plut[sw].w : P.plut[sw].z, late(P.pa[3 * sw + 2], j),
                                late(P.pl[ii], j), ss, sl);
                P.wss[i] = ss;
                P.slw[i] = sl;
            }
        }
        P.groot[i] = groot;
        P.win[i] = w;
    }
    __syncthreads();
    LSTAMP(7);
    for (int i = tid; i < T.na * 2; i += blockDim.x) {
        const int s = i >> 1, j = i & 1, ii = P.aq[s];
        const int4 lu = P.plut[s];
        const double sf = late(P.pa[3 * s + 2], j), ld = late(P.pl[ii], j), da = P.da[s * 2 + j];
        double ds, dl;
        pg::interp_grad(L, j ? lu.y : lu.x, sf, ld, ds, dl);
        double ga = __dmul_rn(da, ds);
        P.term[s * 2 + j] = __dmul_rn(da, dl);
        if (s - (S.n.aptr[ii] - T.a0) == P.win[ii * 2 + j])
            ga = __dadd_rn(ga, __dmul_rn(P.groot[ii * 2 + j], P.wss[ii * 2 + j]));
        G.gsa[(size_t)S.arc[s] * 2 + j] = ga;
    }
    __syncthreads();
    // dL/dload of net ii, column j: the in-arc terms in arc order, then the
    // winner's slew term
    auto net_gl = [&](int ii, int j) {
        double gl = 0.0;
        if ((S.n.flags[ii] & TQ_KIND) == ROOT_ARC) {
            const int s0 = S.n.aptr[ii] - T.a0, na = S.n.aptr[ii + 1] - S.n.aptr[ii];
            for (int k = 0; k < na; k++) gl = __dadd_rn(gl, P.term[(s0 + k) * 2 + j]);
            if (P.win[ii * 2 + j] >= 0) gl = __dadd_rn(gl, __dmul_rn(P.groot[ii * 2 + j], P.slw[ii * 2 + j]));
        }
        return gl;
    };
    for (int i = tid; i < (T.nq + T.nm) * 2; i += blockDim.x) {
        const int j = i & 1;
        if (i < T.nq * 2) {
            const int ii = i >> 1;
            const double gl = net_gl(ii, j);
            const int net = S.n.net[ii];
            G.gl[(size_t)net * 2 + j] = gl;
            G.d_root_cap[(size_t)net * 2 + j] = gl;
            if (S.n.flags[ii] & TQ_TREE)
                pg::pg_tree_net(t, C, G, S.n.f0[ii], S.n.mptr[ii + 1] - S.n.mptr[ii], j, gl);
        } else {
            const int mi = (i >> 1) - T.nq;
            const int4 r = P.pmr[mi];
            const int ii = r.z >> 8;
            if (S.n.flags[ii] & TQ_TREE) continue;
            G.d_cap[(size_t)r.w * 2 + j] = __dadd_rn(__dadd_rn(P.px[mi * 2 + j], net_gl(ii, j)), P.py[mi * 2 + j]);
        }
    }
}

template <bool HARD, bool GRAD, bool STATIC = false, bool PG = false>
__device__ void bwd_body(const Topo& t, const Corner& C, const Task& T, BwdSmem& S,
                         const BwdRec& R, double g, int kind, int variant, int plev = -1,
                         const LutView* pL = nullptr, const PgDev* ppd = nullptr, PgSmem* pP = nullptr)
{
    const int tid = threadIdx.x, c = tid & 3, ii = tid >> 2;
    const bool late = c >= 2;
    const int j = c - 2;
    const bool loop = T.flags & TK_LOOP, chunk = T.flags & TK_CHUNK, wide = T.flags & TK_WIDE;
    // ---- R3: gathers
    double r0[ITEMS], rto[ITEMS], ado[ITEMS], nd[ITEMS], at[ITEMS], adj0[ITEMS], lse[ITEMS],
        epl[ITEMS], dout[ITEMS], wgt[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        r0[k] = rto[k] = ado[k] = nd[k] = at[k] = adj0[k] = lse[k] = epl[k] = dout[k] = wgt[k] = 0.0;
        if (STATIC) {
            if (R.pin[k] >= 0) {
                const int pin = R.pin[k], fl = R.fl[k];
                ado[k] = R.ado[k]; nd[k] = R.nd[k]; at[k] = R.at[k];
                lse[k] = R.lse[k]; epl[k] = R.epl[k]; r0[k] = R.r0[k];
                if (HARD) {
                    if (fl & TM_ROOT) r0[k] = LDG(C.required + (size_t)pin * 4 + c);
                    if (R.o1a[k] >= 0) rto[k] = LDG(C.required + (size_t)R.o1t[k] * 4 + c);
                }
                if (GRAD && late) {
                    if (fl & TM_ROOT) adj0[k] = LDG(C.adjoint + (size_t)pin * 2 + j);
                    if (R.o1a[k] >= 0) dout[k] = LDG(C.d_arc + (size_t)R.o1a[k] * 2 + j);
                }
            }
            wgt[k] = R.wgt[k];
        } else {
            if (R.pin[k] >= 0)
                bwd_gather<HARD, GRAD>(C, R.pin[k], R.fl[k], R.o1t[k], R.o1a[k], R.e1[k], c, t, r0[k],
                                       rto[k], ado[k], nd[k], at[k], adj0[k], lse[k], epl[k], dout[k]);
            if (R.arc[k] >= 0) wgt[k] = LDG(C.weights + (size_t)R.arc[k] * 2 + j);
        }
    }
    // (net, cond) item: the root's arrival (slack), init required and seed
    double n_at = 0, n_rr = 0, n_seed = 0;
    if (STATIC) {
        n_at = R.n_at; n_rr = R.n_rr; n_seed = R.n_seed;
    } else if (R.nroot >= 0) {
        if (HARD) {
            if (!(R.nflags & TQ_ROOT_MEMBER)) n_at = LDG(C.arrival + (size_t)R.nroot * 4 + c);
            n_rr = root_init_required(t, C, R.nroot, R.nflags, R.ne1, c);
        }
        if (GRAD && late) n_seed = root_seed(t, C, R.nroot, R.nflags, R.ne1, j, g, kind);
    }
    __syncthreads();                                   // net records visible
    BSTAMP(0);
    // ---- member phase
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        if (R.pin[k] < 0) continue;
        const int mi = ii + k * TASK_Q, u = T.m0 + mi;
        double v = 0, de = 0;
        bwd_member<HARD, GRAD>(t, C, R.o0[k], R.o0[k] + R.no[k], R.pin[k], R.fl[k], c, g, kind, r0[k],
                               rto[k], ado[k], nd[k], at[k], adj0[k], lse[k], epl[k], dout[k], v, de);
        const int qi = R.fl[k] >> 8;
        const size_t f = (size_t)(S.n.f0[qi] + (u - S.n.mptr[qi]));
        if (HARD) {
            if (loop) C.mem_buf[f * 4 + c] = v;
            else S.v[mi * 4 + c] = v;
        }
        if (GRAD && late) {
            C.d_edge[f * 2 + j] = de;
            if (!loop) S.de[mi * 2 + j] = de;
        }
    }
    for (int i = tid + ITEMS * PASS_TPB; i < T.nm * 4; i += blockDim.x) {   // TK_LOOP tasks
        const int u = T.m0 + (i >> 2);
        const int pp = t.tm_pin[u], ff = t.tm_flags[u];
        double a_r0 = 0, a_rto = 0, a_ado = 0, a_nd = 0, a_at = 0, a_adj0 = 0, a_lse = 0, a_epl = 0,
               a_dout = 0;
        bwd_gather<HARD, GRAD>(C, pp, ff, t.tm_o1_to[u], t.tm_o1_arc[u], t.tm_e1[u], c, t, a_r0,
                               a_rto, a_ado, a_nd, a_at, a_adj0, a_lse, a_epl, a_dout);
        double v = 0, de = 0;
        bwd_member<HARD, GRAD>(t, C, t.tm_optr[u], t.tm_optr[u + 1], pp, ff, c, g, kind, a_r0, a_rto,
                               a_ado, a_nd, a_at, a_adj0, a_lse, a_epl, a_dout, v, de);
        const size_t f = (size_t)(S.n.f0[0] + (u - S.n.mptr[0]));
        if (HARD) C.mem_buf[f * 4 + c] = v;
        if (GRAD && late) C.d_edge[f * 2 + j] = de;
    }
#pragma unroll
    for (int k = 0; k < ITEMS; k++)
        if (R.arc[k] >= 0) {
            const int ai = ii + k * TASK_Q;
            S.w[ai * 2 + j] = wgt[k];
            S.arc[ai] = R.arc[k];
        }
    if (PG) pg::cp_wait_all();               // the sweep's prefetch, published by the barrier
    __syncthreads();
    BSTAMP(1);
    if (PG) LSTAMP(5);
    // position-gradient sweep: a task's member terms stay in shared memory
    // unless the net spans several tasks (chunks) or exceeds them (loop)
    const bool pg_glob = chunk || loop || wide;
    if (PG) {   // member terms of the sweep: the members' adjoints are final
        const PlaceCorner& G = ppd->pa[blockIdx.y].g;
        PgSmem& P = *pP;
        for (int i = tid; i < T.nm * 2; i += blockDim.x) {
            const int u = T.m0 + (i >> 1), jj = i & 1;
            if (pg_glob) {
                pg::MemberIn mv = pg::member_load(t, *ppd, C, u, jj);
                pg::member_load_dyn(G, jj, mv);
                pg::member_finish(t, G, u, jj, mv, 0, pg::TermsGlobal{&G});
            } else {
                const int mi = i >> 1;
                const int4 r = P.pmr[mi];
                auto late = [&](double2 v) { return jj ? v.y : v.x; };
                pg::MemberIn mv;
                mv.pin = r.x; mv.o1 = r.y; mv.fl = r.z; mv.f = r.w;
                mv.tree = S.n.flags[r.z >> 8] & TQ_TREE;
                mv.sm = late(P.pm[mi * 6 + 0]); mv.im = late(P.pm[mi * 6 + 1]);
                mv.d = late(P.pm[mi * 6 + 2]); mv.rr = late(P.pm[mi * 6 + 3]);
                mv.cp = late(P.pm[mi * 6 + 4]); mv.sr = late(P.pm[mi * 6 + 5]);
                mv.adj = S.de[mi * 2 + jj];   // the member phase's adjoint
                mv.gsa1 = late(P.pgsa[mi]); mv.gsr = late(P.pgsr[mi]);
                pg::member_finish(t, G, u, jj, mv, mi, pg::TermsSmem{P.pt, P.px, P.py});
            }
        }
    }
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
        const bool last = last_chunk(C.big_ctr + 4 * T.slot + variant, nch, &S.flag);
        if (last && tid < 4) {
            const int rt = S.n.root[0], fq = S.n.flags[0];
            const double* p0 = C.big_part + (size_t)t.bn_part0[T.slot] * 8;
            if (HARD) {
                const bool mx = c < 2;
                double rr = root_init_required(t, C, rt, fq, S.n.e1[0], c);
                for (int k = 0; k < nch; k++)
                    if (later_wins(mx, rr, LDG(p0 + k * 8 + c))) rr = LDG(p0 + k * 8 + c);
                C.required[(size_t)rt * 4 + c] = rr;
                if (!(fq & TQ_ROOT_MEMBER)) {
                    const double a = LDG(C.arrival + (size_t)rt * 4 + c);
                    C.slack[(size_t)rt * 4 + c] = mx ? __dsub_rn(a, rr) : __dsub_rn(rr, a);
                }
            }
            if (GRAD && late) {
                double ar = root_seed(t, C, rt, fq, S.n.e1[0], j, g, kind);
                for (int k = nch - 1; k >= 0; k--) ar = __dadd_rn(ar, LDG(p0 + k * 8 + 4 + j));
                C.adjoint[(size_t)rt * 2 + j] = ar;
                if ((fq & TQ_KIND) == ROOT_ARC)
                    for (int q = 0; q < T.na; q++)
                        C.d_arc[(size_t)S.arc[q] * 2 + j] = __dmul_rn(ar, S.w[q * 2 + j]);
            }
        }
        __syncthreads();
        // the big net's sweep step, once every chunk's member terms are in
        // (last_chunk fenced them) and its in-arcs' d_arc are written
        if (PG && last && tid < 32)
            pg::pg_net_group<4>(t, *pL, C, ppd->pa[blockIdx.y].g, tid < 4 ? T.q0 : -1,
                                pg::SrcGlobal{{&ppd->pa[blockIdx.y].g}, &t, &C});
        return;
    }
    // ---- net phase: one (net, cond) per thread
    if (ii < T.nq) {
        const int rt = S.n.root[ii], fq = S.n.flags[ii];
        const int k0m = S.n.mptr[ii] - T.m0, k1m = S.n.mptr[ii + 1] - T.m0;
        // star / small-tree nets of ordinary tasks: one reverse pass over the
        // members does the required fold and (late columns) the adjoint sum
        const bool fold_sum = HARD && GRAD && late && !loop && !(fq & TQ_TREE);
        double ar = n_seed;
        if (HARD) {
            const bool mx = c < 2;
            double rr = n_rr;
            if (loop) {
                const int s = S.n.f0[ii];
                for (int k = 0; k < k1m - k0m; k++) {
                    const double v = LDG(C.mem_buf + (size_t)(s + k) * 4 + c);
                    if (later_wins(mx, rr, v)) rr = v;
                }
            } else {
                // the ordered max / min fold as one max over sign-flipped
                // values (the flips are exact), members visited deepest
                // first with ties to the earlier member (>=), the root's
                // initial value ahead of them all (>): ties, signed zeros
                // and NaN stickiness are those of the forward later_wins fold
                const double sg = mx ? 1.0 : -1.0;
                double ms = -INF;
                for (int k = k1m - 1; k >= k0m; k--) {
                    const double v = __dmul_rn(sg, S.v[k * 4 + c]);
                    if (v >= ms) ms = v;
                    if (fold_sum) ar = __dadd_rn(ar, S.de[k * 2 + j]);
                }
                const double rs0 = __dmul_rn(sg, rr);
                rr = __dmul_rn(sg, ms > rs0 ? ms : rs0);
            }
            C.required[(size_t)rt * 4 + c] = rr;
            if (!(fq & TQ_ROOT_MEMBER))
                C.slack[(size_t)rt * 4 + c] = mx ? __dsub_rn(n_at, rr) : __dsub_rn(rr, n_at);
        }
        if (GRAD && late) {
            if (fold_sum) {
                // summed with the fold above
            } else if ((fq & TQ_TREE) || loop) {
                // parents gather children, deepest member first (diff.py:222-233)
                const int s = S.n.f0[ii];
                for (int k = k1m - k0m - 1; k >= 0; k--) {
                    const double dk = LDG(C.d_edge + (size_t)(s + k) * 2 + j);
                    const int pl = (fq & TQ_TREE) ? t.mem_parent_loc[s + k] : 0;
                    if (pl > 0) {
                        double* dp = C.d_edge + (size_t)(s + pl - 1) * 2 + j;
                        *dp = __dadd_rn(LDG(dp), dk);
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
                    for (int q = S.n.aptr[ii] - T.a0; q < S.n.aptr[ii + 1] - T.a0; q++) {
                        const double da = __dmul_rn(ar, S.w[q * 2 + j]);
                        C.d_arc[(size_t)S.arc[q] * 2 + j] = da;
                        if (PG) pP->da[q * 2 + j] = da;
                    }
                } else {
                    for (int q = S.n.aptr[0]; q < S.n.aptr[1]; q++) {
                        const size_t a = (size_t)t.ta_arc[q];
                        C.d_arc[a * 2 + j] = __dmul_rn(ar, LDG(C.weights + a * 2 + j));
                    }
                }
            }
        }
    }
    if (PG) {
        __syncthreads();                     // the in-arcs' d_arc, the member terms
        LSTAMP(6);
        const LutView& LG = *pL;
        const PlaceCorner& G = ppd->pa[blockIdx.y].g;
        if (pg_glob) pg::pg_net_group<4>(t, LG, C, G, ii < T.nq ? T.q0 + ii : -1, pg::SrcGlobal{{&G}, &t, &C});
        else pg_task_nets(t, LG, C, G, T, S, *pP);
    }
    if (STATIC) __syncthreads();             // (persistent kernel) smem reusable by the next task
}

// sum over the corners of a batch, in corner order (WS_RUN_CORNER_SUM): the
// gradient of the batch objective sum_k loss_k.  Every corner's copy of a
// field sits at a uniform stride from corner c0's (alloc_corners).
__global__ void k_corner_sum(Corner c0, CornerStrides cst, int A, int M, int nc, double* dsum_arc,
                             double* dsum_edge)
{
    pdl_trigger();
    pdl_wait();
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const double* src;
    long long stride;
    double* dst;
    if (i < 2 * (size_t)A) {
        src = c0.d_arc + i; stride = cst.A2; dst = dsum_arc + i;
    } else if (i < 2 * (size_t)A + 2 * (size_t)M) {
        const size_t e = i - 2 * (size_t)A;
        src = c0.d_edge + e; stride = cst.M2; dst = dsum_edge + e;
    } else {
        return;
    }
    double tot = src[0];
    for (int k = 1; k < nc; k++) tot = __dadd_rn(tot, src[(size_t)k * stride]);
    *dst = tot;
}

// ---- streaming RC (reduce width 8) --------------------------------------
// The RC stage has no level dependencies, so it runs as one HBM-streaming
// launch instead of per-task blocks: member blocks take RC_ITEMS
// (member, cond) items per thread in flat member order (mem_res / mem_cap
// read once, fully coalesced); net blocks take one (net, cond) item: the
// root load of a star net (root_cap + root_load8 over its contiguous member
// caps).  Net blocks come first in the grid so the sequential folds of big
// nets overlap the streaming member blocks (RC 116 -> 108 us at C3).
constexpr int RC_TPB = 256, RC_ITEMS = 4;

// pin_order: the streaming blocks walk (pin, cond) items instead of
// (member, cond): the member's res / cap are gathered (32 B per pin) and the
// pin's load / net_delay / impulse rows are written contiguously (full
// lines), the non-member roots' zero delay / impulse included.
// FOLD (corner batches): no net blocks (nbn == 0); the member blocks fold
// the star-net root loads.  The single-corner instance has no shared memory.
template <bool FOLD>
__global__ void __launch_bounds__(RC_TPB) k_rc_flat(Topo t, Corners cs, int nbm, int nbn, int nbf,
                                                    bool lse, bool pin_order, const int* __restrict__ bnet)
{
    pdl_trigger();
    const Corner& C = cs.c[blockIdx.y];
    if ((int)blockIdx.x >= nbn + nbm) {         // pins in no net: their initial state (k_free)
        pdl_wait();
        const int i = ((int)blockIdx.x - nbn - nbm) * RC_TPB + threadIdx.x;
        if (i < t.n_free) free_pin(t, C, i, lse);
        return;
    }
    // net blocks first: the sequential root-load folds of big nets start
    // early and overlap the streaming member blocks
    const int bx = (int)blockIdx.x < nbn ? (int)blockIdx.x + nbm : (int)blockIdx.x - nbn;
    if (bx < nbm && pin_order) {
        const size_t base = (size_t)bx * RC_TPB * RC_ITEMS + threadIdx.x;
        const size_t n4 = (size_t)t.P * 4;
        int code[RC_ITEMS];
#pragma unroll
        for (int k = 0; k < RC_ITEMS; k++) {
            const size_t i = base + (size_t)k * RC_TPB;
            code[k] = i < n4 ? LDG(t.rc_pcode + (i >> 2)) : 0;
        }
        pdl_wait();
        double b[RC_ITEMS], r[RC_ITEMS];
#pragma unroll
        for (int k = 0; k < RC_ITEMS; k++) {
            const size_t i = base + (size_t)k * RC_TPB;
            b[k] = r[k] = 0.0;
            if (code[k] & 1) {
                const size_t f = (size_t)(code[k] >> 2) * 4 + (i & 3);
                b[k] = __ldcs(C.mem_cap + f);
                r[k] = __ldcs(C.mem_res + f);
            }
        }
#pragma unroll
        for (int k = 0; k < RC_ITEMS; k++) {
            const size_t i = base + (size_t)k * RC_TPB;
            if (code[k] & 1) {
                const double d = __dadd_rn(0.0, __dmul_rn(r[k], b[k]));
                const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r[k]), b[k]), d), __dmul_rn(d, d));
                if (!(code[k] & 2)) C.load[i] = b[k];
                C.net_delay[i] = d;
                C.impulse[i] = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
            } else if (code[k] == 2) {
                C.net_delay[i] = 0.0;
                C.impulse[i] = 0.0;
            }
        }
        return;
    }
    if (bx < nbm) {
        const size_t base = (size_t)bx * RC_TPB * RC_ITEMS + threadIdx.x;
        const size_t n4 = (size_t)t.M * 4;
        int code[RC_ITEMS];
#pragma unroll
        for (int k = 0; k < RC_ITEMS; k++) {
            const size_t i = base + (size_t)k * RC_TPB;
            code[k] = i < n4 ? LDG(t.rc_code + (i >> 2)) : -1;
        }
        pdl_wait();
        // values loaded independently of the codes: one round trip
        double b[RC_ITEMS], r[RC_ITEMS];
#pragma unroll
        for (int k = 0; k < RC_ITEMS; k++) {
            const size_t i = base + (size_t)k * RC_TPB;
            b[k] = r[k] = 0.0;
            if (i < n4) { b[k] = __ldcs(C.mem_cap + i); r[k] = __ldcs(C.mem_res + i); }
        }
#pragma unroll
        for (int k = 0; k < RC_ITEMS; k++) {
            if (code[k] < 0) continue;
            const int c = (int)((base + (size_t)k * RC_TPB) & 3);
            const double d = __dadd_rn(0.0, __dmul_rn(r[k], b[k]));
            const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r[k]), b[k]), d), __dmul_rn(d, d));
            const size_t pin = (size_t)(code[k] >> 1);
            if (!(code[k] & 1)) C.load[pin * 4 + c] = b[k];
            C.net_delay[pin * 4 + c] = d;
            C.impulse[pin * 4 + c] = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
        }
        if (FOLD) {
            // root loads of the star nets whose members start in this block
            // (no separate net blocks): the block's caps from shared memory,
            // a net running past the block's end from global; the same
            // 8-partial fold as root_load8
            __shared__ double sc[RC_MPB * 4];
            const size_t mb0 = (size_t)bx * RC_MPB, mb1 = mb0 + RC_MPB;
#pragma unroll
            for (int k = 0; k < RC_ITEMS; k++) sc[threadIdx.x + k * RC_TPB] = b[k];
            __syncthreads();
            const int n0 = LDG(bnet + bx), n1 = LDG(bnet + bx + 1);
            for (int x = threadIdx.x; x < (n1 - n0) * 4; x += RC_TPB) {
                const int n = n0 + (x >> 2), c = x & 3;
                if (LDG(t.net_tree + n)) continue;       // k_rc_tree
                const int s = LDG(t.net_ptr + n), m = LDG(t.net_ptr + n + 1) - s, root = LDG(t.net_root + n);
                double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int b0 = 0; b0 < m; b0 += 8)
#pragma unroll
                    for (int y = 0; y < 8; y++)
                        if (b0 + y < m) {
                            const size_t j = (size_t)(s + b0 + y);
                            const double cp = j < mb1 ? sc[(j - mb0) * 4 + c] : LDG(C.mem_cap + j * 4 + c);
                            p[y] = __dadd_rn(p[y], cp);
                        }
                p[0] = __dadd_rn(p[0], p[1]); p[2] = __dadd_rn(p[2], p[3]);
                p[4] = __dadd_rn(p[4], p[5]); p[6] = __dadd_rn(p[6], p[7]);
                p[0] = __dadd_rn(p[0], p[2]); p[4] = __dadd_rn(p[4], p[6]);
                const double l = __dadd_rn(p[0], p[4]);
                C.load[(size_t)root * 4 + c] = __dadd_rn(LDG(C.root_cap + (size_t)n * 4 + c), l);
                if (LDG(t.member_of_pin + root) < 0) {
                    C.net_delay[(size_t)root * 4 + c] = 0.0;
                    C.impulse[(size_t)root * 4 + c] = 0.0;
                }
            }
        }
        return;
    }
    const int i = (bx - nbm) * RC_TPB + threadIdx.x;
    const int n = i >> 2, c = i & 3;
    if (n >= t.N) return;
    if (LDG(t.net_tree + n)) return;             // k_rc_tree
    const int s = LDG(t.net_ptr + n), m = LDG(t.net_ptr + n + 1) - s, root = LDG(t.net_root + n);
    const bool rm = LDG(t.member_of_pin + root) >= 0;
    pdl_wait();
    const double l = root_load8(C.mem_cap + (size_t)s * 4 + c, 4, m);
    C.load[(size_t)root * 4 + c] = __dadd_rn(LDG(C.root_cap + (size_t)n * 4 + c), l);
    if (!rm && !pin_order) {
        C.net_delay[(size_t)root * 4 + c] = 0.0;
        C.impulse[(size_t)root * 4 + c] = 0.0;
    }
}


// ---- CTE-scheme RC (the paper's Algorithm 2 ablation) ---
// A block owns CTE_NETS consecutive nets (thread = net): an exclusive scan of
// their (members x 4) workloads in shared memory, then the block's threads
// stride over the flattened (member, cond) tasks, each locating its net by
// binary search in the scan.  Star-net members get their Elmore delay /
// impulse / load there; the (net, cond) root loads use the same ordered
// 8-partial fold as k_rc_flat.  Results are bitwise those of k_rc_flat
// (WS_RC_SCHEME=cte selects it; RC-tree nets stay with k_rc_tree).
constexpr int CTE_NETS = 256;

__global__ void __launch_bounds__(CTE_NETS) k_rc_cte(Topo t, Corners cs)
{
    __shared__ int pre[CTE_NETS + 1], s0[CTE_NETS];
    __shared__ unsigned char tree[CTE_NETS];
    pdl_trigger();
    const Corner& C = cs.c[blockIdx.y];
    const int n0 = blockIdx.x * CTE_NETS, tid = threadIdx.x;
    const int n = n0 + tid;
    int w = 0;
    if (n < t.N) {
        const int a = t.net_ptr[n], b = t.net_ptr[n + 1];
        s0[tid] = a;
        tree[tid] = t.net_tree[n] ? 1 : 0;
        w = tree[tid] ? 0 : (b - a) * 4;
    }
    pre[tid + 1] = w;
    if (tid == 0) pre[0] = 0;
    __syncthreads();
    // inclusive Hillis-Steele scan over pre[1..CTE_NETS]
    for (int off = 1; off < CTE_NETS; off <<= 1) {
        const int v = tid >= off ? pre[tid + 1 - off] : 0;
        __syncthreads();
        pre[tid + 1] += v;
        __syncthreads();
    }
    pdl_wait();
    const int total = pre[CTE_NETS];
    for (int task = tid; task < total; task += CTE_NETS) {
        int lo = 0, hi = CTE_NETS;        // last net with pre[net] <= task
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= task) lo = mid; else hi = mid;
        }
        const int rel = task - pre[lo], k = rel >> 2, c = rel & 3;
        const size_t i = (size_t)(s0[lo] + k) * 4 + c;
        const int code = t.rc_code[s0[lo] + k];
        const double b = C.mem_cap[i], r = C.mem_res[i];
        const double d = __dadd_rn(0.0, __dmul_rn(r, b));
        const double rad = __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, r), b), d), __dmul_rn(d, d));
        const size_t pin = (size_t)(code >> 1);
        if (!(code & 1)) C.load[pin * 4 + c] = b;
        C.net_delay[pin * 4 + c] = d;
        C.impulse[pin * 4 + c] = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
    }
    for (int it = tid; it < CTE_NETS * 4; it += CTE_NETS) {
        const int nl = it >> 2, c = it & 3, nn = n0 + nl;
        if (nn >= t.N || tree[nl]) continue;
        const int s = s0[nl], m = t.net_ptr[nn + 1] - s, root = t.net_root[nn];
        const double l = root_load8(C.mem_cap + (size_t)s * 4 + c, 4, m);
        C.load[(size_t)root * 4 + c] = __dadd_rn(C.root_cap[(size_t)nn * 4 + c], l);
        if (t.member_of_pin[root] < 0) {
            C.net_delay[(size_t)root * 4 + c] = 0.0;
            C.impulse[(size_t)root * 4 + c] = 0.0;
        }
    }
}

// tree nets (any member with a non-root parent): the whole Elmore recursion
// per (net, cond), sequential like the reference
__global__ void __launch_bounds__(RC_TPB) k_rc_tree(Topo t, Corners cs)
{
    pdl_trigger();
    const Corner& C = cs.c[blockIdx.y];
    const int i = blockIdx.x * RC_TPB + threadIdx.x;
    const int n = i >> 2, c = i & 3;
    bool tree = false;
    int s = 0, m = 0, root = 0;
    if (n < t.N && LDG(t.net_tree + n)) {
        tree = true;
        s = LDG(t.net_ptr + n);
        m = LDG(t.net_ptr + n + 1) - s;
        root = LDG(t.net_root + n);
    }
    pdl_wait();
    if (tree) rc_seq(t, C, n, root, s, m, c, 8, LDG(t.member_of_pin + root) >= 0);
}

// ---- per-level kernels (one task per block; PDL prologue = records) --------

__global__ void __launch_bounds__(PASS_TPB, 2) k_rc(Topo t, Corners cs, int w, int k0)
{
    __shared__ RcSmem S;
    pdl_trigger();
    const Task T = load_task(t, k0 + blockIdx.x);
    RcRec R;
    rc_records(t, T, S, R);
    pdl_wait();
    rc_body(t, cs.c[blockIdx.y], T, S, R, w);
}

// MB: min resident blocks per SM.  Single corners are latency-bound on the
// level chain (2: the full register budget); corner batches are
// throughput-bound and run a 4-block variant (WS_MINB_BATCH).
template <bool HARD, bool LSE, int MB = WS_MINB>
__global__ void __launch_bounds__(PASS_TPB, MB) k_fwd(Topo t, LutSrc ls, Corners cs, int k0,
                                                     bool use_smem, double g, double ginv)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ FwdSmem S;
    pdl_trigger();
    LSTAMP(0);
    const Corner& C = cs.c[blockIdx.y];
    LutView L;
    if (HARD) L = stage_luts_async(ls, C.lut_t_flat, use_smem, smem);
    const int k = k0 + blockIdx.x;
    const Task T = load_task(t, k);
    FwdRec R;
    fwd_records<HARD>(t, T, S, R);
    LSTAMP(1);
    pdl_wait();          // the previous level's results are now visible
    LSTAMP(2);
    fwd_body<HARD, LSE>(t, L, C, T, S, R, g, ginv);
    LSTAMP(3);
}

template <bool HARD, bool GRAD, int MB = WS_MINB, bool PG = false>
__global__ void __launch_bounds__(PASS_TPB, MB) k_bwd(Topo t, Corners cs, int k0, double g, int kind,
                                                     int variant, LutSrc ls, bool use_smem, PgDev pd,
                                                     int pg_off)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ BwdSmem S;
    // the sweep: the LUT pool staged in the prologue (the member phase's
    // barrier precedes the first use), its per-task state after it
    LutView L;
    PgSmem* P = nullptr;
    if (PG) {
        L = stage_luts_async(ls, cs.c[blockIdx.y].lut_t_flat, use_smem, smem);
        P = reinterpret_cast<PgSmem*>(smem + pg_off);
    }
    pdl_trigger();
    LSTAMP(0);
    const int k = k0 + blockIdx.x;
    const Task T = load_task(t, k);
    BwdRec R;
    bwd_records<GRAD>(t, T, S, R);
    const bool pg_pref = PG && !(T.flags & (TK_CHUNK | TK_LOOP | TK_WIDE));
    if (pg_pref) pg_prefetch_static(t, pd, cs.c[blockIdx.y], T, *P);
    LSTAMP(1);
    pdl_wait();          // the next-higher level's results are now visible
    LSTAMP(2);
    if (pg_pref) pg_prefetch_dyn(pd.pa[blockIdx.y].g, T, *P);
    bwd_body<HARD, GRAD, false, PG>(t, cs.c[blockIdx.y], T, S, R, g, kind, variant, -1, &L, &pd, P);
    LSTAMP(3);
}

// pins finished after the level loop: pins in no net (seed + out-arcs) and
// PI roots that also source arcs (their level-loop adjoint + out-arcs)
__device__ void fin_item(const Topo& t, const Corner& C, int i, double g, int kind)
{
    const int p = t.fin_pins[i >> 1], j = i & 1;
    double ad = t.fin_flags[i >> 1] ? LDG(C.adjoint + (size_t)p * 2 + j)
                                    : seed_multi(t, C, p, j, LDG(C.lse_at + (size_t)p * 2 + j), g, kind);
    for (int q = t.pin_out_ptr[p]; q < t.pin_out_ptr[p + 1]; q++)
        ad = __dadd_rn(ad, LDG(C.d_arc + (size_t)t.pin_out_arc[q] * 2 + j));
    C.adjoint[(size_t)p * 2 + j] = ad;
}

__global__ void k_fin(Topo t, Corners cs, double g, int kind)
{
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 2 * t.n_fin) fin_item(t, cs.c[blockIdx.y], i, g, kind);
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
    slack = LDG(C.slack + (size_t)pin * 4 + 2 + j);
    tns_term = (slack <= 0.0 || slack != slack) ? slack : 0.0;      // np.minimum(s, 0.0)
    loss_term = 0.0;
    if (want_loss) {
        const double v = __dsub_rn(LDG(C.lse_at + (size_t)pin * 2 + j), C.ep_required[(size_t)e * 4 + 2 + j]);
        const double mxv = (v >= 0.0 || v != v) ? v : 0.0;           // np.maximum(v, 0.0)
        if (kind == 0) loss_term = mxv;
        else loss_term = __dadd_rn(mxv, __dmul_rn(g, log1p(exp(__ddiv_rn(-fabs(v), g)))));
    }
}

struct SumArgs {
    const int *leaf_off, *leaf_len;
    int n_leaves;
    const int *in_left, *in_right, *height_ptr;
    int n_heights;
};

struct SumSmem {
    double t[8][128], l[8][128];    // leaf phase: one warp's terms
    int last;
};

// dynamic shared memory of k_summary: the whole tree (node values and the
// plan), when it fits (sum_tree_bytes)
__host__ __device__ inline size_t sum_tree_bytes(int n_nodes, int n_inner, int n_heights)
{
    return (size_t)n_nodes * 3 * 8 + (size_t)n_inner * 2 * 4 + (size_t)(n_heights + 1) * 4;
}

// leaves strided over the warps of `ncta` blocks; the last block to finish
// combines the tree (sync_ctr[0] counts finished blocks)
__device__ void summary_phase(const Topo& t, const Corner& C, const SumArgs& P, double g, int kind,
                              bool want_loss, bool want_sta, int cta, int ncta, SumSmem& S,
                              unsigned char* tree = nullptr)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* nv = C.red_tmp;   // [3 * nodes]: tns, loss, wns per node
#ifdef WS_PROBE
#define SSTAMP(slot)                                                                          \
    do {                                                                                      \
        if (threadIdx.x == 0 && t.probe) {                                                    \
            unsigned long long _v;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_v));                            \
            t.probe[(size_t)cta * 8 + (slot)] = _v;                                           \
        }                                                                                     \
    } while (0)
#else
#define SSTAMP(slot) do { } while (0)
#endif
    SSTAMP(0);
    const int nn = 2 * P.n_leaves - 1;
    for (int lf = cta * 8 + warp; lf < P.n_leaves; lf += ncta * 8) {
        const int off = P.leaf_off[lf], n = P.leaf_len[lf];
        double wmin = INF;
        // leaves hold <= 128 terms: a lane's <= 4 terms are gathered together
        // (one round trip), then folded in the original k order
        double tt[4], sl[4], lt[4];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            tt[r] = sl[r] = lt[r] = 0.0;
            if (lane + 32 * r < n) summary_terms(t, C, off + lane + 32 * r, g, kind, want_loss, tt[r], sl[r], lt[r]);
        }
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int k = lane + 32 * r;
            if (k < n) {
                S.t[warp][k] = tt[r];
                S.l[warp][k] = lt[r];
                wmin = (sl[r] < wmin || sl[r] != sl[r]) ? sl[r] : wmin;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double w2 = __shfl_down_sync(WS_FULL, wmin, o);
            wmin = (w2 < wmin || w2 != w2) ? w2 : wmin;
        }
        __syncwarp();
        // lanes 0..7 own accumulator j of numpy's unrolled pairwise leaf
        double rt = 0.0, rl = 0.0;
        if (n >= 8 && lane < 8) {
            rt = S.t[warp][lane];
            rl = S.l[warp][lane];
            for (int i = 8; i < n - (n % 8); i += 8) {
                rt = __dadd_rn(rt, S.t[warp][i + lane]);
                rl = __dadd_rn(rl, S.l[warp][i + lane]);
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
                ts = __dadd_rn(ts, S.t[warp][i]);
                ls = __dadd_rn(ls, S.l[warp][i]);
            }
            nv[lf] = ts;
            nv[nn + lf] = ls;
            nv[2 * nn + lf] = wmin;
        }
        __syncwarp();
    }
    // the last block to finish combines the tree
    SSTAMP(1);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(C.sync_ctr, 1u);
        S.last = prev == (unsigned)(ncta - 1);
    }
    __syncthreads();
    SSTAMP(2);
    if (!S.last) return;
    __threadfence();
    if (tree) {
        // the whole tree in shared memory: leaves and plan in one round trip,
        // then one barrier per height instead of a global-memory round trip
        const int ni = nn - P.n_leaves;
        double* nd = reinterpret_cast<double*>(tree);            // [3][nn]
        int* il = reinterpret_cast<int*>(nd + 3 * (size_t)nn);   // [ni]
        int* ir = il + ni;                                       // [ni]
        int* hp = ir + ni;                                       // [n_heights + 1]
        for (int i = threadIdx.x; i < P.n_leaves; i += blockDim.x) {
            nd[i] = LDG(nv + i);
            nd[nn + i] = LDG(nv + nn + i);
            nd[2 * nn + i] = LDG(nv + 2 * nn + i);
        }
        for (int k = threadIdx.x; k < ni; k += blockDim.x) {
            il[k] = P.in_left[k];
            ir[k] = P.in_right[k];
        }
        for (int h = threadIdx.x; h <= P.n_heights; h += blockDim.x) hp[h] = P.height_ptr[h];
        __syncthreads();
        for (int h = 0; h < P.n_heights; h++) {
            for (int k = hp[h] + threadIdx.x; k < hp[h + 1]; k += blockDim.x) {
                const int l = il[k], r = ir[k], me = P.n_leaves + k;
                nd[me] = __dadd_rn(nd[l], nd[r]);
                nd[nn + me] = __dadd_rn(nd[nn + l], nd[nn + r]);
                const double a = nd[2 * nn + l], b = nd[2 * nn + r];
                nd[2 * nn + me] = (b < a || b != b) ? b : a;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const int top = nn - 1;
            if (want_sta) { C.summary[0] = nd[top]; C.summary[1] = nd[2 * nn + top]; }
            if (want_loss) C.summary[2] = nd[nn + top];
            *C.sync_ctr = 0u;
        }
        SSTAMP(3);
        return;
    }
    for (int h = 0; h < P.n_heights; h++) {
        for (int k = P.height_ptr[h] + threadIdx.x; k < P.height_ptr[h + 1]; k += blockDim.x) {
            const int l = P.in_left[k], r = P.in_right[k], me = P.n_leaves + k;
            nv[me] = __dadd_rn(LDG(nv + l), LDG(nv + r));
            nv[nn + me] = __dadd_rn(LDG(nv + nn + l), LDG(nv + nn + r));
            const double a = LDG(nv + 2 * nn + l), b = LDG(nv + 2 * nn + r);
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

__global__ void __launch_bounds__(256) k_summary(Topo t, Corners cs, SumArgs P, double g, int kind,
                                                 bool want_loss, bool want_sta, bool smem_tree)
{
    __shared__ SumSmem S;
    extern __shared__ __align__(16) unsigned char tree[];
    pdl_trigger();
    pdl_wait();
    summary_phase(t, cs.c[blockIdx.y], P, g, kind, want_loss, want_sta, blockIdx.x, gridDim.x, S,
                  smem_tree ? tree : nullptr);
}

// the adjoints finished after the level loop (k_fin) and the summary
// (k_summary) are independent: one launch, fin blocks first
__global__ void __launch_bounds__(256) k_fin_summary(Topo t, Corners cs, SumArgs P, double g, int kind,
                                                     bool want_loss, bool want_sta, bool smem_tree,
                                                     int nb_fin)
{
    __shared__ SumSmem S;
    extern __shared__ __align__(16) unsigned char tree[];
    pdl_trigger();
    pdl_wait();
    const Corner& C = cs.c[blockIdx.y];
    if ((int)blockIdx.x < nb_fin) {
        const int i = blockIdx.x * blockDim.x + threadIdx.x;
        if (i < 2 * t.n_fin) fin_item(t, C, i, g, kind);
        return;
    }
    summary_phase(t, C, P, g, kind, want_loss, want_sta, (int)blockIdx.x - nb_fin, (int)gridDim.x - nb_fin,
                  S, smem_tree ? tree : nullptr);
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


// ---------------------------------------------------------------------------
// Persistent pass: ONE cooperative launch runs the whole differentiable pass.
// Every block stages the LUT pool once, then walks RC, the forward levels and
// the backward levels; blocks of a corner meet at a grid barrier between
// levels.  Before each barrier a block already loads the records of its
// first task of the next level (static topology), so after the barrier only
// the gathers of the just-finished level remain on the critical path.

__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Split grid barrier over the `n` blocks of one corner (all co-resident:
// cooperative launch).  grid_arrive() publishes this block's writes and
// returns the counter value that completes the barrier; the caller may do
// independent work (prefetch the next level's records) before grid_wait().
// The counter only grows, so no reset / generation word is needed.
__device__ __forceinline__ unsigned long long grid_arrive(unsigned long long* ctr, unsigned n,
                                                          unsigned long long* s_target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long old = atomicAdd(ctr, 1ull);
        *s_target = (old / n + 1) * n;
    }
    return 0;
}

__device__ __forceinline__ void grid_wait(unsigned long long* ctr, unsigned long long* s_target)
{
    if (threadIdx.x == 0) {
        const unsigned long long target = *s_target;
        while (ld_acquire64(ctr) < target) { }
        __threadfence();
    }
    __syncthreads();
}



// ---- per-task record blobs in shared memory (persistent kernel) ---------
// A block's next task's records (static topology) are fetched by TMA bulk
// copies (cp.async.bulk, completion on an mbarrier) while the current task
// computes and the grid barrier drains, so a level starts with its records
// already in shared memory.
struct FwdBlob {
    int4 tk[2];                 // tk_a, tk_b (the Task record)
    int4 n[2 * (TASK_Q + 1)];
    int4 q[TASK_Q];
    int2 a[TASK_Q * 3];
    int4 l[TASK_Q * 3 * 2];     // delay ids, slew ids (per cond) of each slot
    int2 m[TASK_M];
};
struct BwdBlob {
    int4 tk[2];
    int4 n[2 * (TASK_Q + 1)];
    int4 m[2 * TASK_M];
    int4 q[TASK_Q];
};
union __align__(16) BlobBuf {
    FwdBlob f;
    BwdBlob b;
};

__device__ __forceinline__ unsigned smem_u32(const void* p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(mb)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned phase)
{
    asm volatile("{\n\t.reg .pred p;\n\tWS_MBW:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WS_MBW;\n\t}" :: "r"(smem_u32(mb)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mb)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)) : "memory");
}

// thread 0: fetch task k's forward (bwd = false) or backward records
__device__ __forceinline__ void issue_blob(const Topo& t, int k, bool bwd, BlobBuf& B, unsigned long long* mb)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of B
    const size_t kn = (size_t)k * (TASK_Q + 1) * 2;
    if (!bwd) {
        mbar_expect_tx(mb, (unsigned)sizeof(FwdBlob));
        bulk_g2s(&B.f.tk[0], t.tk_a + k, 16, mb);
        bulk_g2s(&B.f.tk[1], t.tk_b + k, 16, mb);
        bulk_g2s(B.f.n, t.fb_n + kn, sizeof(B.f.n), mb);
        bulk_g2s(B.f.q, t.fb_q + (size_t)k * TASK_Q, sizeof(B.f.q), mb);
        bulk_g2s(B.f.a, t.fb_a + (size_t)k * TASK_Q * 3, sizeof(B.f.a), mb);
        bulk_g2s(B.f.l, t.fb_l + (size_t)k * TASK_Q * 3 * 2, sizeof(B.f.l), mb);
        bulk_g2s(B.f.m, t.fb_m + (size_t)k * TASK_M, sizeof(B.f.m), mb);
    } else {
        mbar_expect_tx(mb, (unsigned)sizeof(BwdBlob));
        bulk_g2s(&B.b.tk[0], t.tk_a + k, 16, mb);
        bulk_g2s(&B.b.tk[1], t.tk_b + k, 16, mb);
        bulk_g2s(B.b.n, t.fb_n + kn, sizeof(B.b.n), mb);
        bulk_g2s(B.b.m, t.bb_m + (size_t)k * TASK_M * 2, sizeof(B.b.m), mb);
        bulk_g2s(B.b.q, t.bb_q + (size_t)k * TASK_Q, sizeof(B.b.q), mb);
    }
}

__device__ __forceinline__ void nets_from_blob(const int4* n, const Task& T, NetSmem& S)
{
    const int i = threadIdx.x;
    if (i <= T.nq) {
        const int4 a = n[2 * i], b = n[2 * i + 1];
        S.aptr[i] = b.y;
        S.mptr[i] = b.z;
        if (i < T.nq) {
            S.root[i] = a.x;
            S.flags[i] = a.y;
            S.f0[i] = a.z;
            S.net[i] = a.w;
            S.e1[i] = b.x;
        }
    }
}

template <bool HARD>
__device__ __forceinline__ void fwd_records_smem(const FwdBlob& B, const Task& T, FwdSmem& S, FwdRec& R)
{
    nets_from_blob(B.n, T, S.n);
    const int c = threadIdx.x & 3, qi = threadIdx.x >> 2;
    const int4 fq = B.q[qi];
    R.nroot = fq.x;
    R.nflags = fq.y;
    R.a0 = fq.z;
    R.na = fq.w;
#pragma unroll
    for (int s = 0; s < FWD_NA; s++) {
        const int2 fa = B.a[qi * 3 + s];
        R.from[s] = fa.x;
        R.arc[s] = fa.y;
        if (HARD) {
            R.dl[s] = lut_id(B.l + (2 * (qi * 3 + s)), c);
            R.sl[s] = lut_id(B.l + (2 * (qi * 3 + s) + 1), c);
        }
    }
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        const int2 fm = B.m[qi + s * TASK_Q];
        R.mpin[s] = fm.x;
        R.mfl[s] = fm.y;
    }
}

template <bool GRAD>
__device__ __forceinline__ void bwd_records_smem(const BwdBlob& B, const Task& T, BwdSmem& S, BwdRec& R)
{
    nets_from_blob(B.n, T, S.n);
    const bool late = (threadIdx.x & 3) >= 2;
    const int qi = threadIdx.x >> 2;
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        const int4 m1 = B.m[2 * (qi + s * TASK_Q)], m2 = B.m[2 * (qi + s * TASK_Q) + 1];
        R.pin[s] = m1.x;
        R.fl[s] = m1.y;
        R.o1t[s] = m1.z;
        R.o1a[s] = m1.w;
        R.e1[s] = m2.x;
        R.o0[s] = m2.y;
        R.no[s] = m2.z;
        R.arc[s] = (GRAD && late) ? m2.w : -1;
    }
    const int4 bq = B.q[qi];
    R.nroot = bq.x;
    R.nflags = bq.y;
    R.ne1 = bq.z;
}

// a block's task sequence: forward levels 0..L-1, then backward levels
// L-1..0; within a level tasks lvt_ptr[li] + cta, + ncta, ...
struct Seq {
    int step;   // 0 .. 2L-1 (forward levels, then backward levels), 2L = done
    int k;      // task index or -1 at the end of a level
};
__device__ __forceinline__ int seq_level(const Topo& t, int step) { return step < t.L ? step : 2 * t.L - 1 - step; }
// the first task at or after level position `step` (skipping empty levels)
__device__ __forceinline__ Seq seq_first(const Topo& t, int step, int cta)
{
    for (; step < 2 * t.L; step++) {
        const int li = seq_level(t, step);
        const int k = t.lvt_ptr[li] + cta;
        if (k < t.lvt_ptr[li + 1]) return Seq{step, k};
    }
    return Seq{2 * t.L, -1};
}
__device__ __forceinline__ Seq seq_next(const Topo& t, Seq s, int cta, int ncta)
{
    const int li = seq_level(t, s.step);
    if (s.k + ncta < t.lvt_ptr[li + 1]) return Seq{s.step, s.k + ncta};
    return seq_first(t, s.step + 1, cta);
}

// ---- next task's sweep-static gathers, staged by cp.async -----------------
// Issued right after the current task's body (addresses from the next
// task's records, already in smem), they land while the block waits at the
// grid barrier; afterwards the block only reads them back from smem.  The
// staged arrays are final for the sweep (RC outputs for the forward sweep,
// forward outputs for the backward sweep) and are never read through L1
// before they are final, so the L1-allocating cp.async.ca sees current data.
struct FwdStage {
    double mnd[ITEMS][PASS_TPB], mim[ITEMS][PASS_TPB], ld[PASS_TPB];
};
struct BwdStage {
    double ado[ITEMS][PASS_TPB], nd[ITEMS][PASS_TPB], at[ITEMS][PASS_TPB], lse[ITEMS][PASS_TPB],
        epl[ITEMS][PASS_TPB], wgt[ITEMS][PASS_TPB], epr[ITEMS][PASS_TPB];
    double n_at[PASS_TPB], n_epr[PASS_TPB], n_lse[PASS_TPB], n_epl[PASS_TPB];
};
union __align__(16) StageBuf {
    FwdStage f;
    BwdStage b;
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <bool HARD>
__device__ __forceinline__ void fwd_stage_issue(const Corner& C, const FwdRec& R, FwdStage& st)
{
    const int c = threadIdx.x & 3, i = threadIdx.x;
#pragma unroll
    for (int k = 0; k < ITEMS; k++)
        if (R.mpin[k] >= 0) {
            cp_async8(&st.mnd[k][i], C.net_delay + (size_t)R.mpin[k] * 4 + c);
            if (HARD) cp_async8(&st.mim[k][i], C.impulse + (size_t)R.mpin[k] * 4 + c);
        }
    if (HARD && R.na > 0) cp_async8(&st.ld[i], C.load + (size_t)R.nroot * 4 + c);
    cp_async_commit();
}

template <bool HARD>
__device__ __forceinline__ void fwd_stage_take(const FwdStage& st, FwdRec& R)
{
    const int i = threadIdx.x;
    cp_async_wait_all();
#pragma unroll
    for (int k = 0; k < ITEMS; k++)
        if (R.mpin[k] >= 0) {
            R.mnd[k] = st.mnd[k][i];
            if (HARD) R.mim[k] = st.mim[k][i];
        }
    R.ld = (HARD && R.na > 0) ? st.ld[i] : 0.0;
}

template <bool HARD, bool GRAD>
__device__ __forceinline__ void bwd_stage_issue(const Corner& C, const BwdRec& R, BwdStage& st)
{
    const int c = threadIdx.x & 3, j = c - 2, i = threadIdx.x;
    const bool late = c >= 2;
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        if (R.pin[k] >= 0) {
            const int pin = R.pin[k], fl = R.fl[k];
            if (HARD) {
                if (R.o1a[k] >= 0) cp_async8(&st.ado[k][i], C.arc_delay + (size_t)R.o1a[k] * 4 + c);
                cp_async8(&st.nd[k][i], C.net_delay + (size_t)pin * 4 + c);
                cp_async8(&st.at[k][i], C.arrival + (size_t)pin * 4 + c);
                if (!(fl & TM_ROOT) && !(fl & TM_MULTI_EP) && (fl & TM_EP))
                    cp_async8(&st.epr[k][i], C.ep_required + (size_t)R.e1[k] * 4 + c);
            }
            if (GRAD && late && (fl & TM_EP)) {
                cp_async8(&st.lse[k][i], C.lse_at + (size_t)pin * 2 + j);
                cp_async8(&st.epl[k][i], C.ep_required + (size_t)R.e1[k] * 4 + 2 + j);
            }
        }
        if (R.arc[k] >= 0) cp_async8(&st.wgt[k][i], C.weights + (size_t)R.arc[k] * 2 + j);
    }
    if (R.nroot >= 0) {
        if (HARD && !(R.nflags & TQ_ROOT_MEMBER)) cp_async8(&st.n_at[i], C.arrival + (size_t)R.nroot * 4 + c);
        if ((R.nflags & TQ_ROOT_EP) && !(R.nflags & TQ_MULTI_EP)) {
            if (HARD) cp_async8(&st.n_epr[i], C.ep_required + (size_t)R.ne1 * 4 + c);
            if (GRAD && late) {
                cp_async8(&st.n_lse[i], C.lse_at + (size_t)R.nroot * 2 + j);
                cp_async8(&st.n_epl[i], C.ep_required + (size_t)R.ne1 * 4 + 2 + j);
            }
        }
    }
    cp_async_commit();
}

// the backward sweep-static values from the staged copies (multi-endpoint pins, rare,
// still fold their endpoint entries from global memory here)
template <bool HARD, bool GRAD>
__device__ __forceinline__ void bwd_stage_take(const Topo& t, const Corner& C, const BwdStage& st,
                                               BwdRec& R, double g, int kind)
{
    const int c = threadIdx.x & 3, j = c - 2, i = threadIdx.x;
    const bool late = c >= 2;
    cp_async_wait_all();
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        R.ado[k] = R.nd[k] = R.at[k] = R.lse[k] = R.epl[k] = R.wgt[k] = R.r0[k] = 0.0;
        if (R.pin[k] >= 0) {
            const int pin = R.pin[k], fl = R.fl[k];
            if (HARD) {
                if (R.o1a[k] >= 0) R.ado[k] = st.ado[k][i];
                R.nd[k] = st.nd[k][i];
                R.at[k] = st.at[k][i];
                if (!(fl & TM_ROOT))
                    R.r0[k] = (fl & TM_MULTI_EP) ? init_required_multi(t, C, pin, c)
                                                 : merge_req(c < 2 ? -INF : INF,
                                                             (fl & TM_EP) ? st.epr[k][i] : (c < 2 ? -INF : INF), c);
            }
            if (GRAD && late && (fl & TM_EP)) {
                R.lse[k] = st.lse[k][i];
                R.epl[k] = st.epl[k][i];
            }
        }
        if (R.arc[k] >= 0) R.wgt[k] = st.wgt[k][i];
    }
    R.n_at = R.n_rr = R.n_seed = 0.0;
    if (R.nroot >= 0) {
        const int fq = R.nflags;
        if (HARD) {
            if (!(fq & TQ_ROOT_MEMBER)) R.n_at = st.n_at[i];
            R.n_rr = (fq & TQ_MULTI_EP) ? init_required_multi(t, C, R.nroot, c)
                                        : merge_req(c < 2 ? -INF : INF,
                                                    (fq & TQ_ROOT_EP) ? st.n_epr[i] : (c < 2 ? -INF : INF), c);
        }
        if (GRAD && late && (fq & TQ_ROOT_EP)) {
            if (fq & TQ_MULTI_EP) R.n_seed = root_seed(t, C, R.nroot, fq, R.ne1, j, g, kind);
            else R.n_seed = __dadd_rn(0.0, seed_term(__dsub_rn(st.n_lse[i], st.n_epl[i]), g, kind));
        }
    }
}

union PassSmem {
    FwdSmem f;
    BwdSmem b;
    SumSmem s;
};

#ifdef WS_PROBE
#define PSTAMP(level, slot)                                                                   \
    do {                                                                                      \
        if (threadIdx.x == 0 && t.probe) {                                                    \
            unsigned long long _v;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_v));                            \
            t.probe[((size_t)(level) * 2048 + blockIdx.x) * 4 + (slot)] = _v;                 \
        }                                                                                     \
    } while (0)
// whole-kernel phases: 0 start | 1 RC done | 2 forward done | 3 backward done
#define KSTAMP(slot)                                                                          \
    do {                                                                                      \
        if (threadIdx.x == 0 && t.probe) {                                                    \
            unsigned long long _v;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_v));                            \
            t.probe[(size_t)4 * t.L * 2048 * 4 + (size_t)blockIdx.x * 4 + (slot)] = _v;       \
        }                                                                                     \
    } while (0)
#else
#define PSTAMP(level, slot) do { } while (0)
#define KSTAMP(slot) do { } while (0)
#endif

template <bool LSE, bool GRAD>
__global__ void __launch_bounds__(PASS_TPB, 2) k_pass(Topo t, LutSrc ls, Corners cs, SumArgs P,
                                                      int w, double g, int kind, bool use_smem)
{
    const double ginv = __ddiv_rn(1.0, g);      // = the host's 1.0 / g (correctly rounded)
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ PassSmem S;
    __shared__ BlobBuf blob[2];
    __shared__ __align__(8) unsigned long long mbar[2];
    // dynamic smem: the staging buffer, then the LUT pool
    StageBuf& stg = *reinterpret_cast<StageBuf*>(smem);
    const Corner& C = cs.c[blockIdx.y];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(C.sync_ctr + 2);
    __shared__ unsigned long long s_target;
    const int cta = blockIdx.x, ncta = gridDim.x;
    KSTAMP(0);
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // pins in no net and the RC of every net ran as ordinary (fully
    // parallel) kernels before this launch: RC is static for the pass
    Seq cur = seq_first(t, 0, cta);
    int buf = 0;
    unsigned phase[2] = {0u, 0u};
    if (threadIdx.x == 0 && cur.k >= 0) issue_blob(t, cur.k, cur.step >= t.L, blob[0], &mbar[0]);
    const LutView L = stage_luts(ls, C.lut_t_flat, use_smem, smem + sizeof(StageBuf), false);
    KSTAMP(1);
    Task T{};
    Seq nxt{2 * t.L, -1};
    bool fetch_due = false;      // nxt's blob not yet requested
    // `cur`'s records from its blob and the cp.async of its sweep-static
    // gathers (right after the previous body, before the grid barrier) ...
    auto take = [&](bool bwd_rec, FwdRec& RF, BwdRec& RB) {
        nxt = seq_next(t, cur, cta, ncta);
        fetch_due = true;
        mbar_wait(&mbar[buf], phase[buf]);
        phase[buf] ^= 1u;
        {
            const int4 a = blob[buf].f.tk[0], b = blob[buf].f.tk[1];   // same offset in both layouts
            T = Task{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        }
        if (!bwd_rec) {
            fwd_records_smem<true>(blob[buf].f, T, S.f, RF);
            fwd_stage_issue<true>(C, RF, stg.f);
        } else {
            bwd_records_smem<GRAD>(blob[buf].b, T, S.b, RB);
            bwd_stage_issue<true, GRAD>(C, RB, stg.b);
        }
    };
    // ... then (inside the barrier window) the blob fetch of the task after
    // it into the other buffer
    auto fetch_next = [&]() {
        if (fetch_due && threadIdx.x == 0 && nxt.k >= 0)
            issue_blob(t, nxt.k, nxt.step >= t.L, blob[buf ^ 1], &mbar[buf ^ 1]);
        fetch_due = false;
    };
    // ---- forward levels
    {
        FwdRec R;
        BwdRec RB_unused;
        bool have = false;
        for (int li = 0; li < t.L; li++) {
            PSTAMP(li, 0);
            while (cur.k >= 0 && cur.step == li) {
                if (!have) { take(false, R, RB_unused); fetch_next(); }
                fwd_stage_take<true>(stg.f, R);
                fwd_body<true, LSE, true>(t, L, C, T, S.f, R, g, ginv, li);
                buf ^= 1;
                cur = nxt;
                have = false;
                if (cur.k >= 0 && cur.step == li) { take(false, R, RB_unused); fetch_next(); have = true; }
            }
            // the next forward task's records and static-gather issue precede
            // the arrival; the copies land while the barrier drains
            if (!have && cur.k >= 0 && cur.step < t.L) { take(false, R, RB_unused); have = true; }
            PSTAMP(li, 1);
            grid_arrive(bar, ncta, &s_target);
            if (have) fetch_next();
            PSTAMP(li, 2);
            grid_wait(bar, &s_target);
        }
    }
    KSTAMP(2);
    // ---- backward levels
    {
        BwdRec R;
        FwdRec RF_unused;
        bool have = false;
        for (int li = t.L - 1; li >= 0; li--) {
            const int step = 2 * t.L - 1 - li;
            PSTAMP(t.L + li, 0);
            while (cur.k >= 0 && cur.step == step) {
                if (!have) { take(true, RF_unused, R); fetch_next(); }
                bwd_stage_take<true, GRAD>(t, C, stg.b, R, g, kind);
                bwd_body<true, GRAD, true>(t, C, T, S.b, R, g, kind, GRAD ? 3 : 1, t.L + li);
                buf ^= 1;
                cur = nxt;
                have = false;
                if (cur.k >= 0 && cur.step == step) { take(true, RF_unused, R); fetch_next(); have = true; }
            }
            if (!have && cur.k >= 0) { take(true, RF_unused, R); have = true; }
            PSTAMP(t.L + li, 1);
            grid_arrive(bar, ncta, &s_target);
            if (have) fetch_next();
            PSTAMP(t.L + li, 2);
            grid_wait(bar, &s_target);
        }
    }
    KSTAMP(3);
    // ---- pins finished after the level loop, then TNS / WNS / loss
    if (GRAD)
        for (int i = cta * PASS_TPB + threadIdx.x; i < 2 * t.n_fin; i += ncta * PASS_TPB)
            fin_item(t, C, i, g, kind);
    if (P.n_leaves > 0) {
        summary_phase(t, C, P, g, kind, GRAD, true, cta, ncta, S.s);
    } else if (cta == 0 && threadIdx.x == 0) {
        C.summary[0] = 0.0;
        C.summary[1] = INF;
        if (GRAD) C.summary[2] = 0.0;
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

// every pass kernel is launched with programmatic stream serialization so
// its static prologue overlaps the previous kernel (see pdl_wait)
template <typename... KArgs, typename... Args>
void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
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
    cfg.numAttrs = 1;
    WS_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

struct Launcher {
    Context& ctx;
    Corners cs;
    int c0;
    int nc;
    bool pg = false;     // fused position-gradient sweep inside the backward levels
    int count = 0;
    LutSrc ls;
    size_t lut_bytes;
    bool use_smem;
    Launcher(Context& c, int c0_, int nc_) : ctx(c), c0(c0_), nc(nc_)
    {
        for (int k = 0; k < nc; k++) cs.c[k] = ctx.corners[c0 + k].d;
        const Topo& t = ctx.t;
        ls = {t.lut_s_ptr, t.lut_l_ptr, t.lut_t_ptr, t.lut_s_flat, t.lut_l_flat, t.NL,
              ctx.lut_s_len, ctx.lut_l_len, ctx.lut_t_len, t.lut_info};
        lut_bytes = lut_smem_bytes(t.NL, ctx.lut_s_len, ctx.lut_l_len, ctx.lut_t_len);
        use_smem = lut_bytes <= 96 * 1024 && !ctx.lut_global;
        if (!use_smem) lut_bytes = 0;
    }
    dim3 grid1(int n, int tpb) const { return dim3((unsigned)std::max(1, (n + tpb - 1) / tpb), nc); }
    // WS_RUN_TIMED: an event after the launch just issued, tagged (kind, level)
    bool timed = false;
    void mark(cudaStream_t s, int kind, int level)
    {
        if (!timed) return;
        auto& ev = ctx.timed_events;
        if ((int)ev.size() <= ctx.timed_n) {
            cudaEvent_t e;
            WS_CUDA(cudaEventCreate(&e));
            ev.push_back(e);
            ctx.timed_kind.push_back(0);
            ctx.timed_level.push_back(0);
        }
        WS_CUDA(cudaEventRecord(ev[ctx.timed_n], s));
        ctx.timed_kind[ctx.timed_n] = kind;
        ctx.timed_level[ctx.timed_n] = level;
        ctx.timed_n++;
    }
    int tasks(int li) const { return ctx.lvt_ptr_host[li + 1] - ctx.lvt_ptr_host[li]; }

    void free_pins(cudaStream_t s, bool lse)
    {
        if (!ctx.t.n_free) return;
        launch(k_free, grid1(ctx.t.n_free, 256), dim3(256), 0, s, ctx.t, cs, lse);
        count++;
    }
    // with_free (streaming RC only): the free pins' initial state rides in
    // the same launch (returns true when it did)
    bool rc(cudaStream_t s, int w, bool with_free = false, bool lse = false)
    {
        if (!ctx.t.n_tasks) return false;
        bool took_free = false;
        if (w == 8) {
            const bool po = ctx.rc_pin_order;
            const int nbm = (int)(((size_t)(po ? ctx.t.P : ctx.t.M) * 4 + RC_TPB * RC_ITEMS - 1) /
                                  (RC_TPB * RC_ITEMS));
            const int nbn = (int)(((size_t)ctx.t.N * 4 + RC_TPB - 1) / RC_TPB);
            // star-net root loads: corner batches fold them in the member
            // blocks (no net blocks: the caps are read once, 16-corner batch
            // -1.9%); a single corner keeps the net blocks first, whose folds
            // overlap the member stream (the in-block fold costs it +0.3%).
            // WS_RC_ROOTS=net / fold forces either.
            static_assert(RC_TPB * RC_ITEMS == 4 * RC_MPB, "RC member block shape");
            const bool fold_in_members = !po && !ctx.rc_cte && ctx.t.M > 0 &&
                                         (ctx.rc_roots > 0 || (ctx.rc_roots == 0 && nc >= 4));
            const int nbn_flat = fold_in_members ? 0 : nbn;
            const int nbf = (with_free && !ctx.rc_cte) ? (ctx.t.n_free + RC_TPB - 1) / RC_TPB : 0;
            took_free = with_free && !ctx.rc_cte;
            if (ctx.rc_cte)
                launch(k_rc_cte, dim3((ctx.t.N + CTE_NETS - 1) / CTE_NETS, nc), dim3(CTE_NETS), 0, s, ctx.t, cs);
            else
                launch(fold_in_members ? k_rc_flat<true> : k_rc_flat<false>, dim3(nbm + nbn_flat + nbf, nc),
                       dim3(RC_TPB), 0, s, ctx.t, cs, nbm, nbn_flat, nbf, lse, po,
                       (const int*)ctx.rc_bnet);
            if (ctx.any_tree) {
                count++;
                launch(k_rc_tree, dim3(nbn, nc), dim3(RC_TPB), 0, s, ctx.t, cs);
            }
        } else {
            launch(k_rc, dim3(ctx.t.n_tasks, nc), dim3(PASS_TPB), 0, s, ctx.t, cs, w, 0);
        }
        count++;
        return took_free;
    }
    // the RC of one level's tasks (the per-kernel pipeline's net_rc:level)
    void rc_level(cudaStream_t s, int li, int w)
    {
        const int nt = tasks(li);
        if (nt <= 0) return;
        launch(k_rc, dim3(nt, nc), dim3(PASS_TPB), 0, s, ctx.t, cs, w, ctx.lvt_ptr_host[li]);
        count++;
    }
    // WS_PROBE builds: launch i stamps into probe + i * PROBE_STRIDE
    static constexpr size_t PROBE_STRIDE = 8 * 2048;
    Topo probed(int nt) const
    {
        Topo tt = ctx.t;
        tt.probe = (ctx.t.probe && nt <= 2048) ? ctx.t.probe + (size_t)count * PROBE_STRIDE : nullptr;
        return tt;
    }
    template <bool H, bool Lse>
    void fwd(cudaStream_t s, int li, double g)
    {
        const int nt = tasks(li);
        if (nt <= 0) return;
        if (H && Lse && nc >= 4)
            launch(k_fwd<H, Lse, WS_MINB_BATCH>, dim3(nt, nc), dim3(PASS_TPB), lut_bytes, s, probed(nt), ls,
                   cs, ctx.lvt_ptr_host[li], use_smem, g, 1.0 / g);
        else
            launch(k_fwd<H, Lse>, dim3(nt, nc), dim3(PASS_TPB), H ? lut_bytes : 0, s, probed(nt), ls, cs,
                   ctx.lvt_ptr_host[li], use_smem, g, 1.0 / g);
        count++;
    }
    template <bool H, bool G>
    void bwd(cudaStream_t s, int li, double g, int kind)
    {
        const int nt = tasks(li);
        if (nt <= 0) return;
        const int variant = H && G ? 3 : (H ? 1 : 2);
        const PgDev pd = pg ? pg_dev(ctx, c0) : PgDev{nullptr, nullptr, nullptr};
        if (H && G && pg) {
            // candidate batches: 3 blocks/SM (80 registers; 16 candidates
            // 18.62 -> 18.14 ms); one candidate keeps 2 (1.48 vs 1.65 ms)
            if (nc >= 4)
                launch(k_bwd<H, G, WS_MINB_PG_BATCH, true>, dim3(nt, nc), dim3(PASS_TPB), pg_smem_bytes(), s,
                       probed(nt), cs, ctx.lvt_ptr_host[li], g, kind, variant, ls, use_smem, pd, pg_off());
            else
                launch(k_bwd<H, G, WS_MINB, true>, dim3(nt, nc), dim3(PASS_TPB), pg_smem_bytes(), s, probed(nt),
                       cs, ctx.lvt_ptr_host[li], g, kind, variant, ls, use_smem, pd, pg_off());
        } else if (H && G && nc >= 4)
            launch(k_bwd<H, G, WS_MINB_BATCH>, dim3(nt, nc), dim3(PASS_TPB), 0, s, probed(nt), cs,
                   ctx.lvt_ptr_host[li], g, kind, variant, ls, false, pd, 0);
        else
            launch(k_bwd<H, G>, dim3(nt, nc), dim3(PASS_TPB), 0, s, probed(nt), cs, ctx.lvt_ptr_host[li],
                   g, kind, variant, ls, false, pd, 0);
        count++;
    }
    // k_bwd<..., PG>: the staged pool, then the sweep's per-task state
    int pg_off() const { return (int)((lut_bytes + 15) & ~(size_t)15); }
    size_t pg_smem_bytes() const { return (size_t)pg_off() + sizeof(PgSmem); }
    // sum_k d_arc / d_edge over the batch
    void corner_sum(cudaStream_t s)
    {
        const size_t n = 2 * ((size_t)ctx.t.A + (size_t)ctx.t.M);
        if (!n) return;
        launch(k_corner_sum, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, cs.c[0], ctx.cstride,
               ctx.t.A, ctx.t.M, nc, ctx.dsum_arc, ctx.dsum_edge);
        count++;
    }
    void fin(cudaStream_t s, double g, int kind)
    {
        if (!ctx.t.n_fin) return;
        launch(k_fin, grid1(2 * ctx.t.n_fin, 256), dim3(256), 0, s, ctx.t, cs, g, kind);
        count++;
    }
    // fin + summary as one launch (fused pass)
    void fin_summary(cudaStream_t s, double g, int kind)
    {
        const SumPlan* pl = ctx.tns_plan;
        if (pl->n == 0) {
            fin(s, g, kind);
            summary(s, g, kind, true, true);
            return;
        }
        const int nb_fin = ctx.t.n_fin ? (2 * ctx.t.n_fin + 255) / 256 : 0;
        const int nn = 2 * pl->n_leaves - 1;
        const size_t tb = sum_tree_bytes(nn, pl->n_inner, (int)pl->height_ptr.size() - 1);
        const bool smem_tree = tb <= 160 * 1024;
        if (smem_tree && tb > 48 * 1024)
            WS_CUDA(cudaFuncSetAttribute(k_fin_summary, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb));
        launch(k_fin_summary, dim3(nb_fin + (pl->n_leaves + 7) / 8, nc), dim3(256), smem_tree ? tb : 0, s,
               ctx.t, cs, sum_args(), g, kind, true, true, smem_tree, nb_fin);
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
    SumArgs sum_args() const
    {
        const SumPlan* pl = ctx.tns_plan;
        return SumArgs{pl->leaf_off, pl->leaf_len, pl->n_leaves, pl->in_left, pl->in_right,
                       pl->d_height_ptr, (int)pl->height_ptr.size() - 1};
    }
    // the whole pass as one cooperative kernel
    template <bool Lse, bool G>
    void persistent(cudaStream_t s, int w, double g, int kind)
    {
        auto kern = k_pass<Lse, G>;
        const size_t dyn = sizeof(StageBuf) + lut_bytes;
        WS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        int per_sm = 0, dev = 0, n_sm = 0;
        WS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PASS_TPB, dyn));
        WS_CUDA(cudaGetDevice(&dev));
        WS_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
        int max_tasks = 1;
        for (int li = 0; li < ctx.t.L; li++) max_tasks = std::max(max_tasks, tasks(li));
        const int cap = per_sm * n_sm / nc;
        if (cap < 1) throw Error(WS_ERR_VALUE, "persistent pass: too many corners for one launch");
        const int ncta = std::min(cap, std::max(max_tasks, std::min(ctx.t.n_tasks, cap)));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ncta, nc);
        cfg.blockDim = dim3(PASS_TPB);
        cfg.dynamicSmemBytes = dyn;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        WS_CUDA(cudaLaunchKernelEx(&cfg, kern, ctx.t, ls, cs, sum_args(), w, g, kind, use_smem));
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
        const int nn = 2 * pl->n_leaves - 1;
        const size_t tb = sum_tree_bytes(nn, pl->n_inner, (int)pl->height_ptr.size() - 1);
        const bool smem_tree = tb <= 160 * 1024;
        if (smem_tree && tb > 48 * 1024)
            WS_CUDA(cudaFuncSetAttribute(k_summary, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb));
        launch(k_summary, dim3((pl->n_leaves + 7) / 8, nc), dim3(256), smem_tree ? tb : 0, s,
               probed((pl->n_leaves + 7) / 8), cs, sum_args(), g, kind, want_loss, want_sta, smem_tree);
        count++;
    }
};

void run_chunk(Context& ctx, int c0, int nc, unsigned flags, double g, int kind, int gran,
               cudaStream_t s, cudaStream_t gs, int w, int& count,
               const std::vector<cudaEvent_t>* bwd_done = nullptr, bool pg_fused = false)
{
    const int L = ctx.t.L;
    Launcher la(ctx, c0, nc);
    if (la.lut_bytes > 48 * 1024) {
        WS_CUDA(cudaFuncSetAttribute(k_fwd<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la.lut_bytes));
        WS_CUDA(cudaFuncSetAttribute(k_fwd<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la.lut_bytes));
        WS_CUDA(cudaFuncSetAttribute(k_fwd<true, true, WS_MINB_BATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)la.lut_bytes));
    }
    if (pg_fused) {   // the staged pool + the sweep's per-task state exceed the default 48 KB
        WS_CUDA(cudaFuncSetAttribute(k_bwd<true, true, WS_MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)la.pg_smem_bytes()));
        WS_CUDA(cudaFuncSetAttribute(k_bwd<true, true, WS_MINB_PG_BATCH, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la.pg_smem_bytes()));
    }
    const bool hard = flags & WS_RUN_HARD, lse = flags & WS_RUN_LSE, grad = flags & WS_RUN_GRAD;
    const bool fused = (flags & WS_RUN_FUSED) && hard && lse && grad;
    const bool two = (flags & WS_RUN_TWO_STREAM) && hard && (lse || grad) && !fused;

    if ((flags & WS_RUN_PERSISTENT) && hard && ((lse && grad) || (!lse && !grad))) {
        la.free_pins(s, lse);
        la.rc(s, w);
        if (lse) la.persistent<true, true>(s, w, g, kind);
        else la.persistent<false, false>(s, w, g, kind);
        if (lse && (flags & WS_RUN_CORNER_SUM)) la.corner_sum(s);
    } else if (fused && !bwd_done && !(flags & WS_RUN_TIMED) && gs && ctx.split_min > 0 &&
               nc >= ctx.split_min) {
        // large corner batches: two half batches as independent fused passes
        // on the two streams, so one half's level-boundary gaps (PDL release,
        // the last wave) fill with the other's blocks; the batch gradient sum
        // runs after the join over all corners in corner order (bitwise the
        // lockstep batch)
        // parts: WS_SPLIT_PARTS (default 2), each part >= 4 corners
        const int parts = std::max(2, std::min(std::min(ctx.split_parts, nc / 4), 8));
        std::vector<cudaEvent_t>& ev = ctx.events;
        while ((int)ev.size() < 1 + parts) {
            cudaEvent_t e;
            WS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev.push_back(e);
        }
        while ((int)ctx.split_streams.size() < parts - 2) {
            cudaStream_t x;
            WS_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            ctx.split_streams.push_back(x);
        }
        std::vector<cudaStream_t> st(parts);
        st[0] = s;
        st[1] = gs;
        for (int x = 2; x < parts; x++) st[x] = ctx.split_streams[x - 2];
        WS_CUDA(cudaEventRecord(ev[0], s));   // fork
        for (int x = 1; x < parts; x++) WS_CUDA(cudaStreamWaitEvent(st[x], ev[0], 0));
        std::vector<Launcher> lh;
        lh.reserve(parts);
        for (int x = 0; x < parts; x++) {
            const int a = nc * x / parts, b = nc * (x + 1) / parts;
            lh.emplace_back(ctx, c0 + a, b - a);
        }
        for (int x = 0; x < parts; x++)
            if (!lh[x].rc(st[x], w, true, true)) lh[x].free_pins(st[x], true);
        for (int li = 0; li < L; li++)
            for (int x = 0; x < parts; x++) lh[x].fwd<true, true>(st[x], li, g);
        for (int x = 0; x < parts; x++) {
            lh[x].pg = pg_fused;
            if (pg_fused) posgrad_reset(ctx, lh[x].c0, lh[x].nc, st[x]);
        }
        for (int li = L - 1; li >= 0; li--)
            for (int x = 0; x < parts; x++) lh[x].bwd<true, true>(st[x], li, g, kind);
        for (int x = 0; x < parts; x++) {
            lh[x].fin_summary(st[x], g, kind);
            if (pg_fused) lh[x].count += launch_posgrad_tail(ctx, lh[x].c0, lh[x].nc, st[x], true);
        }
        for (int x = 1; x < parts; x++) {     // join
            WS_CUDA(cudaEventRecord(ev[x], st[x]));
            WS_CUDA(cudaStreamWaitEvent(s, ev[x], 0));
        }
        for (int x = 0; x < parts; x++) la.count += lh[x].count;
        if (flags & WS_RUN_CORNER_SUM) la.corner_sum(s);
    } else if (fused) {
        // WS_RUN_TIMED: kinds 0 RC, 1 fused forward+LSE level, 2 fused
        // backward+gradient level, 5 tail (the events serialise the PDL overlap)
        la.timed = flags & WS_RUN_TIMED;
        la.mark(s, 5, -1);
        if (!la.rc(s, w, true, true)) la.free_pins(s, true);
        la.mark(s, 0, 0);
        for (int li = 0; li < L; li++) {
            la.fwd<true, true>(s, li, g);
            la.mark(s, 1, li);
        }
        la.pg = pg_fused;
        if (pg_fused) posgrad_reset(ctx, c0, nc, s);
        for (int li = L - 1; li >= 0; li--) {
            la.bwd<true, true>(s, li, g, kind);
            if (bwd_done) WS_CUDA(cudaEventRecord((*bwd_done)[li], s));
            la.mark(s, 2, li);
        }
        la.fin_summary(s, g, kind);
        if (pg_fused) la.count += launch_posgrad_tail(ctx, c0, nc, s, true);
        if (flags & WS_RUN_CORNER_SUM) la.corner_sum(s);
        la.mark(s, 5, -1);
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
        if (grad && (flags & WS_RUN_CORNER_SUM)) la.corner_sum(s);
    } else {
        // kinds of fusion.py's KernelGraph: 0 net_rc, 1 cell_delay_at,
        // 2 slack_bwd, 3 lse_fwd, 4 grad_bwd, 5 other
        la.timed = flags & WS_RUN_TIMED;
        la.mark(s, 5, -1);                       // start
        if (hard) {
            la.free_pins(s, lse);
            la.mark(s, 5, -1);
            la.rc(s, w);                         // one launch: the RC of every level
            la.mark(s, 0, 0);
            for (int li = 0; li < L; li++) {
                la.fwd<true, false>(s, li, g);
                la.mark(s, 1, li);
            }
        }
        if (lse) {
            if (!hard) la.lse_seed(s);
            for (int li = 0; li < L; li++) {
                la.fwd<false, true>(s, li, g);
                la.mark(s, 3, li);
            }
        }
        if (hard)
            for (int li = L - 1; li >= 0; li--) {
                la.bwd<true, false>(s, li, g, kind);
                la.mark(s, 2, li);
            }
        if (grad) {
            for (int li = L - 1; li >= 0; li--) {
                la.bwd<false, true>(s, li, g, kind);
                la.mark(s, 4, li);
            }
            la.fin(s, g, kind);
            la.mark(s, 5, -1);
        }
        if (!hard && (flags & WS_RUN_SLACK)) la.slack_all(s);
        if (hard || grad || (flags & WS_RUN_SUMMARY))
            la.summary(s, g, kind, grad, hard || (flags & WS_RUN_SUMMARY));
        if (grad && (flags & WS_RUN_CORNER_SUM)) la.corner_sum(s);
        la.mark(s, 5, -1);
    }
    WS_CHECK_LAUNCH();
    count += la.count;
}

}  // namespace

// One kernel of the fusion pipeline's graph (fusion.py:113-160 kinds), for
// the host-side dependency discipline of PipelineRun (fusion.py:307-312):
// 0 net_rc (level 0 also seeds the pins in no net), 1 cell_delay_at,
// 2 slack_bwd, 3 lse_fwd, 4 grad_bwd, 5 finish (free-pin / PI-root
// adjoints, TNS / WNS / loss).  The same device functions as ws_run.
void run_kernel(Context& ctx, int c0, int kind, int level, double g, int loss_kind, int w,
                cudaStream_t s)
{
    Launcher la(ctx, c0, 1);
    if (la.lut_bytes > 48 * 1024) {
        WS_CUDA(cudaFuncSetAttribute(k_fwd<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la.lut_bytes));
        WS_CUDA(cudaFuncSetAttribute(k_fwd<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la.lut_bytes));
    }
    if (kind != 5 && (level < 0 || level >= ctx.t.L))
        throw Error(WS_ERR_VALUE, "kernel level out of range");
    switch (kind) {
    case 0:
        if (level == 0) la.free_pins(s, true);
        la.rc_level(s, level, w);
        break;
    case 1: la.fwd<true, false>(s, level, g); break;
    case 2: la.bwd<true, false>(s, level, g, loss_kind); break;
    case 3: la.fwd<false, true>(s, level, g); break;
    case 4: la.bwd<false, true>(s, level, g, loss_kind); break;
    case 5:
        la.fin(s, g, loss_kind);
        la.summary(s, g, loss_kind, true, true);
        break;
    default: throw Error(WS_ERR_VALUE, "unknown kernel kind");
    }
    WS_CHECK_LAUNCH();
    ctx.launches_last_run = la.count;
}

void run_pass(Context& ctx, int c0, int nc, unsigned flags, double gamma, int loss_kind,
              int granularity, cudaStream_t s, cudaStream_t gs, int w)
{
    int count = 0;
    ctx.timed_n = 0;
    if (flags & WS_RUN_WIRE) count += launch_wire(ctx, c0, nc, s);
    // fused mode: the position-gradient sweep runs inside the backward level
    // kernels (k_bwd<..., PG>).  WS_PG_SWEEP=stream keeps the stand-alone
    // sweep kernels on the second stream instead, level l waiting only for
    // backward level l (ablation).
    const bool fused_pass = (flags & WS_RUN_POSGRAD) && (flags & WS_RUN_FUSED) &&
                            !(flags & WS_RUN_PERSISTENT) && ctx.t.L > 0;
    const char* sweep_env = getenv("WS_PG_SWEEP");
    const bool stream_sweep = sweep_env && !strcmp(sweep_env, "stream");
    const bool pg_fused = fused_pass && !stream_sweep;
    const bool overlap = fused_pass && stream_sweep && nc <= MAXC;
    std::vector<cudaEvent_t>& ev = ctx.pg_events;
    if (overlap) {
        while ((int)ev.size() < ctx.t.L + 2) {
            cudaEvent_t e;
            WS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev.push_back(e);
        }
        WS_CUDA(cudaEventRecord(ev[ctx.t.L], s));          // fork: after everything queued on s
        WS_CUDA(cudaStreamWaitEvent(gs, ev[ctx.t.L], 0));
    }
    for (int k = 0; k < nc; k += MAXC)
        run_chunk(ctx, c0 + k, std::min(MAXC, nc - k), flags, gamma, loss_kind, granularity, s, gs,
                  w, count, overlap ? &ev : nullptr, pg_fused);
    if ((flags & WS_RUN_POSGRAD) && !pg_fused) {
        if (overlap) {
            count += launch_posgrad(ctx, c0, nc, s, gs, &ev);
            WS_CUDA(cudaEventRecord(ev[ctx.t.L + 1], gs));  // join
            WS_CUDA(cudaStreamWaitEvent(s, ev[ctx.t.L + 1], 0));
        } else {
            count += launch_posgrad(ctx, c0, nc, s);
        }
    }
    ctx.launches_last_run = count;
}

}  // namespace ws
