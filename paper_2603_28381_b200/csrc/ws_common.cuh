// Shared device-side definitions for the B200 STA engine (sm_100a).
//
// Numerics contract: compiled with -fmad=false so no a*b+c is contracted to
// an FMA (the reference builds with -ffp-contract=off, pkg/setup.py:21-23);
// double '/' and sqrt are IEEE correctly rounded on the device, so the hard
// pass reproduces the reference bit for bit.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define WS_FULL 0xffffffffu

// WS_PROBE builds record globaltimer stamps at phase boundaries of block
// (blockIdx.x) into t.probe[blockIdx.x * 8 + slot] (profiling only).
#ifdef WS_PROBE
#define WS_STAMP(t, slot)                                                                   \
    do {                                                                                    \
        if (threadIdx.x == 0 && (t).probe) {                                                \
            unsigned long long _v;                                                          \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_v));                          \
            (t).probe[(size_t)blockIdx.x * 8 + (slot)] = _v;                                \
        }                                                                                   \
    } while (0)
#else
#define WS_STAMP(t, slot) do { } while (0)
#endif

namespace ws {

constexpr int ROOT_ARC = 0, ROOT_PI = 1, ROOT_FEED = 2;

// Topology: int32 indices, shared by every corner.
struct Topo {
    int P, N, M, A, I, E, L, NL;     // pins nets members arcs PIs endpoints levels luts
    int n_free;                      // pins in no net
    int max_in, max_m;
    // FlatDesign arrays (flatten.py:83-136)
    int *net_ptr, *net_root, *root_kind, *mem_pin, *mem_parent_loc, *mem_net, *mem_local;
    int *arc_from, *arc_to, *arc_dlut, *arc_slut;
    int *net_in_ptr, *net_in_arc, *mem_out_ptr, *mem_out_arc;
    int *member_of_pin, *root_net_of_pin, *pi_pin, *ep_pin;
    int *net_m, *net_a, *net_o;
    uint8_t *is_endpoint;
    int *lut_s_ptr, *lut_l_ptr, *lut_t_ptr;
    double *lut_s_flat, *lut_l_flat;
    int4 *lut_info;    // canonical (deduplicated) axis offsets: s_off, nS, l_off, nL
    // level schedule (flatten.py:31-80): lv_nets = nets sorted by (level, id)
    int *level_of, *lv_ptr, *lv_nets;
    // derived work lists
    int *net_tree;                   // 1 if any member has a non-root parent
    int *rc_code;                    // per member: -1 (tree net) or pin << 1 | (pin is a root)
    int *rc_pcode;                   // per pin: the pin-order RC code (ws_build.cu k_rc_pcode)
    int *pin_ep_ptr, *pin_ep_idx;    // endpoint entries grouped by pin (stable)
    int *pin_pi;                     // pin -> PI index or -1
    int *pin_out_ptr, *pin_out_arc;  // arcs grouped by source pin (all pins)
    int *free_pins;                  // pins that belong to no net (n_free)
    int *nonmem_src;                 // non-member pins that source arcs
    int n_nonmem_src;

    // ---- level-major task layout (ws_build.cu: build_tasks) --------------
    // q = position in lv_nets (nets level by level, ascending id per level).
    // Everything a level kernel needs about net q, its in-arcs and its
    // members is stored contiguously in q order so one coalesced load per
    // array replaces the reference's pointer chasing.
    int *tq_root;      // [N] root pin
    int *tq_flags;     // [N] TQ_* bits
    int *tq_f0;        // [N] first member index (original member order)
    int *tq_aptr;      // [N+1] in-arcs of q: ta_*[tq_aptr[q] .. tq_aptr[q+1])
    int *tq_mptr;      // [N+1] members of q: tm_*[tq_mptr[q] .. tq_mptr[q+1])
    int *tq_e1;        // [N] first endpoint entry of the root (or -1)
    int *ta_arc;       // [A'] original arc id
    int *ta_from;      // [A'] arc source pin
    int *ta_root;      // [A'] root pin of the arc's net
    int *ta_q;         // [A'] index of the arc's net within its task
    int4 *ta_lut;      // [2*A'] delay LUT ids (ER EF LR LF), then slew LUT ids (32-bit: any pool size)
    int4 *tq_lut1;     // [N] delay LUT ids of q's first in-arc (-1: no in-arc)
    int *tm_pin;       // [M] member pin
    int *tm_flags;     // [M] TM_* bits | (net index within its task) << 8
    int *tm_optr;      // [M+1] out-arcs of member slot u: to_*[tm_optr[u] .. )
    int *tm_o1_to;     // [M] first out-arc's target pin (or -1)
    int *tm_o1_arc;    // [M] first out-arc id (or -1)
    int *tm_e1;        // [M] first endpoint entry of the pin (or -1)
    int *to_arc;       // [A''] original arc id
    int *to_to;        // [A''] arc target pin
    // tasks: a level is a contiguous task range; a task is one thread block's
    // unit of work: <= TASK_Q nets, <= TASK_A in-arcs, <= TASK_M members
    int4 *tk_a;        // [T] q0, nq, a0, na
    int4 *tk_b;        // [T] m0, nm, flags (TK_*), big-net slot (TK_CHUNK) or -1
    int n_tasks;
    int *lvt_ptr;      // [L+1] first task of each level
    int *bn_nch;       // [n_big] chunks of big (chunked) net slot
    int *bn_part0;     // [n_big] first partial of the slot
    int n_big, n_parts;
    unsigned long long *probe;   // WS_PROBE builds: per-block phase timestamps
    // per-task record blobs (ws_build.cu: k_blob): every record a level
    // kernel's prologue needs, at addresses computable from the task index
    // alone, so the prologue is one dependent memory round trip
    int4 *fb_n;        // [T * (TASK_Q+1) * 2] NetSmem: {root, flags, f0, net}, {e1, aptr, mptr, 0}
    int4 *fb_q;        // [T * TASK_Q] forward net item: {root | -1, flags, a0, na (0: not net-centric)}
    int2 *fb_a;        // [T * TASK_Q * 3] forward in-arc slots: {from, arc}
    int4 *fb_l;        // [T * TASK_Q * 3 * 2] their delay LUT ids, then slew LUT ids (per cond)
    int2 *fb_m;        // [T * TASK_M] member slots: {pin | -1, tm_flags}
    int4 *bb_m;        // [T * TASK_M * 2] backward member: {pin | -1, fl, o1_to, o1_arc}, {e1, o0, no, arc}
    int4 *bb_q;        // [T * TASK_Q] backward net item: {root | -1, flags, e1, 0}
    int *fin_pins;     // pins finished after the level loop (free pins, PI roots with out-arcs)
    int *fin_flags;    // 1 = accumulate onto the level-loop adjoint (root), 0 = fresh
    int n_fin;
};

// tq_flags
constexpr int TQ_KIND = 3, TQ_ROOT_MEMBER = 4, TQ_TREE = 8, TQ_ROOT_EP = 16, TQ_ROOT_PI = 32,
              TQ_MULTI_EP = 64;
// tm_flags
constexpr int TM_ROOT = 1, TM_EP = 2, TM_MULTI_EP = 4;
// task limits: a 256-thread block holds one (net, cond) item and ITEMS
// (arc, cond) / (member, cond) items per thread
#ifndef WS_TPB
#define WS_TPB 256
#endif
#ifndef WS_ITEMS
#define WS_ITEMS 2
#endif
constexpr int PASS_TPB = WS_TPB, ITEMS = WS_ITEMS;
constexpr int RC_MPB = 256;   // members per streaming-RC block (k_rc_flat: RC_TPB x RC_ITEMS (member, cond) items)
constexpr int TASK_Q = PASS_TPB / 4, TASK_A = ITEMS * PASS_TPB / 4, TASK_M = ITEMS * PASS_TPB / 4;
// task flags: CHUNK = one chunk of a big star net's members; WIDE = one net
// with more than TASK_A in-arcs; LOOP = one tree net with more than TASK_M
// members (member phase loops, folds are sequential)
constexpr int TK_CHUNK = 1, TK_WIDE = 2, TK_LOOP = 4;

// Values and state of one corner.  (P,4) arrays are row-major 32-byte
// records, exactly the reference's TimingState layout (sta.py:41-48).
struct Corner {
    // values (what a corner / a placement step changes)
    double *mem_res, *mem_cap, *root_cap, *lut_t_flat, *pi_arrival, *pi_slew, *ep_required;
    // TimingState
    double *load, *net_delay, *impulse, *slew, *arrival, *required, *slack, *arc_delay;
    // GradientState (late cols only; diff.py:61-72)
    double *lse_at, *weights, *d_arc, *d_edge, *adjoint;
    // scratch for tree nets (RC fold) and the summary reductions
    double *mem_buf, *mem_dbuf;      // [M*4] each: RC tree fold / big-net fold scratch
    double *red_tmp;   // pairwise-sum node values
    double *summary;   // [tns, wns, loss]
    unsigned *sync_ctr;  // last-block-done counter of the summary kernel
    double *big_part;    // [n_parts * 8] per-chunk partial folds of big nets
    unsigned *big_ctr;   // [n_big * 4] last-chunk-done counters (rc, hard, grad, fused)
};

// Per-field distance (in elements) between consecutive corners' copies: every
// corner's copy of a field is one allocation (ws_capi.cu alloc_corners).
struct CornerStrides {
    long long P4, P2, A4, A2, M4, M2, N4, LT, I4, E4, RT, BP, BC;
};

// corner c0 + k of a batch whose corner c0 is `c`
__host__ __device__ __forceinline__ Corner corner_at(const Corner& c, const CornerStrides& s, int k)
{
    Corner r = c;
    const long long kk = k;
    r.mem_res += kk * s.M4; r.mem_cap += kk * s.M4; r.root_cap += kk * s.N4;
    r.lut_t_flat += kk * s.LT; r.pi_arrival += kk * s.I4; r.pi_slew += kk * s.I4;
    r.ep_required += kk * s.E4;
    r.load += kk * s.P4; r.net_delay += kk * s.P4; r.impulse += kk * s.P4; r.slew += kk * s.P4;
    r.arrival += kk * s.P4; r.required += kk * s.P4; r.slack += kk * s.P4;
    r.arc_delay += kk * s.A4;
    r.lse_at += kk * s.P2; r.weights += kk * s.A2; r.d_arc += kk * s.A2; r.d_edge += kk * s.M2;
    r.adjoint += kk * s.P2;
    r.red_tmp += kk * s.RT; r.summary += kk * 4; r.sync_ctr += kk * 4;
    r.big_part += kk * s.BP; r.big_ctr += kk * s.BC;
    if (r.mem_buf) { r.mem_buf += kk * s.M4; r.mem_dbuf += kk * s.M4; }   // tree-net scratch
    return r;
}

// component c of an int4 LUT-id record read as one 32-bit word: a register
// select of a loaded int4 compiles to four predicated scalar loads per id
__device__ __forceinline__ int lut_id(const int4* rec, int c) { return reinterpret_cast<const int*>(rec)[c]; }

struct LutView {
    const int *s_ptr, *l_ptr, *t_ptr;
    const double *s, *l, *t;
    const int4 *info;   // per LUT: canonical slew-axis offset, nS, canonical load-axis offset, nL
};

// _kernels.pyx:15-81 / sta.py:79-113: upper_bound-1 clamped to [0,n-2],
// fraction clamped to [0,1], 1-point axes are constants.  Same operation
// order as the reference; no FMA (-fmad=false).
__device__ __forceinline__ double lut_interp(const LutView& L, int lut, double qs, double ql)
{
    const int s0 = L.s_ptr[lut], nS = L.s_ptr[lut + 1] - s0;
    const int l0 = L.l_ptr[lut], nL = L.l_ptr[lut + 1] - l0;
    const int t0 = L.t_ptr[lut];
    int si, li, si2, li2;
    double st, lt;
    if (nS > 1) {
        int lo = 0, hi = nS;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (L.s[s0 + mid] <= qs) lo = mid + 1; else hi = mid;
        }
        si = lo - 1;
        if (si < 0) si = 0; else if (si > nS - 2) si = nS - 2;
        st = (qs - L.s[s0 + si]) / (L.s[s0 + si + 1] - L.s[s0 + si]);
        if (st < 0.0) st = 0.0; else if (st > 1.0) st = 1.0;
        si2 = si + 1;
    } else { si = 0; st = 0.0; si2 = 0; }
    if (nL > 1) {
        int lo = 0, hi = nL;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (L.l[l0 + mid] <= ql) lo = mid + 1; else hi = mid;
        }
        li = lo - 1;
        if (li < 0) li = 0; else if (li > nL - 2) li = nL - 2;
        lt = (ql - L.l[l0 + li]) / (L.l[l0 + li + 1] - L.l[l0 + li]);
        if (lt < 0.0) lt = 0.0; else if (lt > 1.0) lt = 1.0;
        li2 = li + 1;
    } else { li = 0; lt = 0.0; li2 = 0; }
    const double v0 = __dadd_rn(__dmul_rn(1.0 - lt, L.t[t0 + si * nL + li]),
                                __dmul_rn(lt, L.t[t0 + si * nL + li2]));
    const double v1 = __dadd_rn(__dmul_rn(1.0 - lt, L.t[t0 + si2 * nL + li]),
                                __dmul_rn(lt, L.t[t0 + si2 * nL + li2]));
    return __dadd_rn(__dmul_rn(1.0 - st, v0), __dmul_rn(st, v1));
}

// The same arithmetic split in two: locate a query on an axis (index and
// clamped fraction), then blend a table at located positions.  An arc's
// delay and slew tables share their axes in practice (the build dedupes
// identical axis arrays), so one locate serves both.
struct Loc {
    int i0, i1;
    double f;
};

static __device__ __noinline__ int upper_bound_long(const double* ax, int n, double q)
{
    int hi = n, lo = 0;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ax[mid] <= q) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ Loc lut_locate(const double* ax, int n, double q)
{
    Loc r;
    if (n > 1) {
        int lo;
        if (n <= 8) {
            // upper_bound on a sorted axis = number of entries <= q (a
            // monotone prefix): three fixed branch-free halving steps reach
            // lo <= 7; for n = 8, lo = 7 and lo = 8 clamp to the same cell
            // (n - 2), so the fourth step of a full search is not needed
            lo = 0;
#pragma unroll
            for (int s = 4; s >= 1; s >>= 1)
                if (lo + s <= n && ax[lo + s - 1] <= q) lo += s;
        } else {
            lo = upper_bound_long(ax, n, q);
        }
        int i = lo - 1;
        if (i < 0) i = 0; else if (i > n - 2) i = n - 2;
        double t = (q - ax[i]) / (ax[i + 1] - ax[i]);
        if (t < 0.0) t = 0.0; else if (t > 1.0) t = 1.0;
        r.i0 = i; r.i1 = i + 1; r.f = t;
    } else {
        r.i0 = 0; r.i1 = 0; r.f = 0.0;
    }
    return r;
}

__device__ __forceinline__ double lut_blend(const double* tab, int nL, const Loc& s, const Loc& l)
{
    const double v0 = __dadd_rn(__dmul_rn(1.0 - l.f, tab[s.i0 * nL + l.i0]), __dmul_rn(l.f, tab[s.i0 * nL + l.i1]));
    const double v1 = __dadd_rn(__dmul_rn(1.0 - l.f, tab[s.i1 * nL + l.i0]), __dmul_rn(l.f, tab[s.i1 * nL + l.i1]));
    return __dadd_rn(__dmul_rn(1.0 - s.f, v0), __dmul_rn(s.f, v1));
}

// numpy's pairwise summation of n terms get(i0 .. i0+n-1) (the inner loop of
// ndarray.sum / np.add.reduce / reduceat): < 8 terms sequentially from 0.0;
// <= 128 terms in 8 strided accumulators combined as ((r0+r1)+(r2+r3))+
// ((r4+r5)+(r6+r7)) plus the tail; longer runs split at n/2 rounded down to a
// multiple of 8, left half + right half.  The split recursion runs on an
// explicit stack (device recursion would need an unbounded call stack).
// No FMA.
template <class Get>
__device__ __forceinline__ double np_pairwise_leaf(const Get& get, int i0, int n)
{
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; i++) r = __dadd_rn(r, get(i0 + i));
        return r;
    }
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; k++) r[k] = get(i0 + k);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], get(i0 + i + k));
    double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) s = __dadd_rn(s, get(i0 + i));
    return s;
}

template <class Get>
__device__ double np_pairwise(const Get& get, int i0, int n)
{
    if (n <= 128) return np_pairwise_leaf(get, i0, n);
    // frames: (first term, count, state 0 = left pending / 1 = right pending
    // / 2 = both done, left sum)
    int fi[32], fn[32], fs[32];
    double fl[32];
    int sp = 1;
    fi[0] = i0; fn[0] = n; fs[0] = 0;
    double ret = 0.0;
    while (sp > 0) {
        const int k = sp - 1;
        if (fn[k] <= 128) {
            ret = np_pairwise_leaf(get, fi[k], fn[k]);
            sp--;
            continue;
        }
        int n2 = fn[k] / 2;
        n2 -= n2 % 8;
        if (fs[k] == 0) {
            fs[k] = 1;
            fi[sp] = fi[k]; fn[sp] = n2; fs[sp] = 0; sp++;
        } else if (fs[k] == 1) {
            fl[k] = ret;
            fs[k] = 2;
            fi[sp] = fi[k] + n2; fn[sp] = fn[k] - n2; fs[sp] = 0; sp++;
        } else {
            ret = __dadd_rn(fl[k], ret);
            sp--;
        }
    }
    return ret;
}

// Ordered selection with the reference's strict comparisons: `cand` comes
// later in the sequence than `cur`, so it wins only when strictly better
// (first element wins ties, _kernels.pyx:195-197, 238-239, 247-248).
__device__ __forceinline__ bool later_wins(bool late_max, double cur, double cand)
{
    return late_max ? (cand > cur) : (cand < cur);
}

// ---------------------------------------------------------------------------
// LUT pool staging into shared memory (north_star item 3)

struct LutSrc {
    const int *s_ptr, *l_ptr, *t_ptr;
    const double *s, *l;
    int nl, s_len, l_len, t_len;
    const int4 *info;
};

__host__ __device__ inline size_t lut_smem_bytes(int nl, int s_len, int l_len, int t_len)
{
    size_t ints = 3 * (size_t)(nl + 1);
    ints = (ints + 3) & ~(size_t)3;
    return ints * 4 + (size_t)nl * 16 + (size_t)(s_len + l_len + t_len) * 8;
}

// the pool read in place through L1 (read-only for the whole pass)
__device__ __forceinline__ LutView lut_view_global(const LutSrc& src, const double* t_flat)
{
    LutView v;
    v.s_ptr = src.s_ptr; v.l_ptr = src.l_ptr; v.t_ptr = src.t_ptr;
    v.s = src.s; v.l = src.l; v.t = t_flat; v.info = src.info;
    return v;
}

// Copies the pool (axes + this corner's tables) into smem when it fits
// (use_smem), else views global memory.  Ends with __syncthreads unless
// `sync` is false (the caller then owns the barrier before first use).
__device__ __forceinline__ LutView stage_luts(const LutSrc& src, const double* t_flat,
                                              bool use_smem, unsigned char* smem, bool sync = true)
{
    LutView v;
    if (!use_smem) {
        v.s_ptr = src.s_ptr; v.l_ptr = src.l_ptr; v.t_ptr = src.t_ptr;
        v.s = src.s; v.l = src.l; v.t = t_flat; v.info = src.info;
        return v;
    }
    const int n1 = src.nl + 1;
    int* ip = reinterpret_cast<int*>(smem);
    size_t ints = 3 * (size_t)n1;
    ints = (ints + 3) & ~(size_t)3;
    int4* inf = reinterpret_cast<int4*>(smem + ints * 4);
    double* dp = reinterpret_cast<double*>(smem + ints * 4 + (size_t)src.nl * 16);
    for (int i = threadIdx.x; i < n1; i += blockDim.x) {
        ip[i] = src.s_ptr[i];
        ip[n1 + i] = src.l_ptr[i];
        ip[2 * n1 + i] = src.t_ptr[i];
    }
    if (src.info)
        for (int i = threadIdx.x; i < src.nl; i += blockDim.x) inf[i] = src.info[i];
    for (int i = threadIdx.x; i < src.s_len; i += blockDim.x) dp[i] = src.s[i];
    for (int i = threadIdx.x; i < src.l_len; i += blockDim.x) dp[src.s_len + i] = src.l[i];
    for (int i = threadIdx.x; i < src.t_len; i += blockDim.x) dp[src.s_len + src.l_len + i] = t_flat[i];
    if (sync) __syncthreads();
    v.s_ptr = ip; v.l_ptr = ip + n1; v.t_ptr = ip + 2 * n1;
    v.s = dp; v.l = dp + src.s_len; v.t = dp + src.s_len + src.l_len;
    v.info = inf;
    return v;
}

// The same staging by cp.async (no thread waits on the pool's loads, so a
// kernel prologue's record loads are not serialized behind it).  The caller
// must cp.async.wait_all + __syncthreads before the first use.
__device__ __forceinline__ void cpa_(void* dst, const void* src, int bytes)
{
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    if (bytes == 16) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ LutView stage_luts_async(const LutSrc& src, const double* t_flat, bool use_smem,
                                                    unsigned char* smem)
{
    LutView v;
    if (!use_smem) {
        v.s_ptr = src.s_ptr; v.l_ptr = src.l_ptr; v.t_ptr = src.t_ptr;
        v.s = src.s; v.l = src.l; v.t = t_flat; v.info = src.info;
        return v;
    }
    const int n1 = src.nl + 1;
    int* ip = reinterpret_cast<int*>(smem);
    size_t ints = 3 * (size_t)n1;
    ints = (ints + 3) & ~(size_t)3;
    int4* inf = reinterpret_cast<int4*>(smem + ints * 4);
    double* dp = reinterpret_cast<double*>(smem + ints * 4 + (size_t)src.nl * 16);
    for (int i = threadIdx.x; i < n1; i += blockDim.x) {
        cpa_(ip + i, src.s_ptr + i, 4);
        cpa_(ip + n1 + i, src.l_ptr + i, 4);
        cpa_(ip + 2 * n1 + i, src.t_ptr + i, 4);
    }
    if (src.info)
        for (int i = threadIdx.x; i < src.nl; i += blockDim.x) cpa_(inf + i, src.info + i, 16);
    for (int i = threadIdx.x; i < src.s_len; i += blockDim.x) cpa_(dp + i, src.s + i, 8);
    for (int i = threadIdx.x; i < src.l_len; i += blockDim.x) cpa_(dp + src.s_len + i, src.l + i, 8);
    for (int i = threadIdx.x; i < src.t_len; i += blockDim.x) cpa_(dp + src.s_len + src.l_len + i, t_flat + i, 8);
    asm volatile("cp.async.commit_group;" ::: "memory");
    v.s_ptr = ip; v.l_ptr = ip + n1; v.t_ptr = ip + 2 * n1;
    v.s = dp; v.l = dp + src.s_len; v.t = dp + src.s_len + src.l_len;
    v.info = inf;
    return v;
}

}  // namespace ws
