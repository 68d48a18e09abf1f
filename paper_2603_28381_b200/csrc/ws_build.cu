// Device-side flatten + levelize (north_star item 1).
//
// Reproduces, bit for bit, the index arrays of the reference's
// flatten (flatten.py:170-316) and the longest-path Kahn levelization over
// _net_deps (flatten.py:44-80, netlist.py:316-331):
//   * maps member_of_pin / root_net_of_pin ("last wins" like the Python dict
//     assignments) via atomicMax,
//   * mem_parent_loc / mem_net / mem_local,
//   * arcs grouped by driven net and by source member with ascending arc id
//     per group: stable LSD radix sort (CUB) keyed by the group id,
//   * levels: level-synchronous frontier Kahn — a net's level is the round in
//     which its last dependency retires, i.e. max(level(dep)) + 1, exactly the
//     reference's longest-chain level; nets then stable-sorted by level so
//     each level lists ascending net ids (flatten.py:79),
//   * CycleError: the root pin of the lowest-index net left unresolved
//     (flatten.py:74-77), which is independent of processing order.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <unordered_map>

#include "ws_internal.h"

namespace ws {
namespace {

constexpr int TPB = 256;
inline int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + TPB - 1) / TPB); }

__global__ void k_fill(int* a, int n, int v)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

__global__ void k_iota(int* a, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

__global__ void k_scatter_last(const int* keys, int n, int* map)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicMax(&map[keys[i]], i);
}

__global__ void k_mem_fields(const int* net_ptr, int N, int M, const int* net_root,
                             const int* mem_parent_pin, const int* member_of_pin,
                             int* mem_net, int* mem_local, int* mem_parent_loc, int* net_tree)
{
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= M) return;
    // upper_bound(net_ptr, f) - 1 over nets with members
    int lo = 0, hi = N;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (net_ptr[mid + 1] <= f) lo = mid + 1; else hi = mid;
    }
    const int n = lo, s = net_ptr[n];
    mem_net[f] = n;
    mem_local[f] = f - s;
    const int par = mem_parent_pin[f];
    int loc;
    if (par == net_root[n]) {
        loc = 0;
    } else {
        const int g = member_of_pin[par];
        loc = (g >= s && g < f) ? g - s + 1 : -1;  // -1: not a tree (validate() rejects)
    }
    mem_parent_loc[f] = loc;
    if (loc > 0) net_tree[n] = 1;
}

// group keys: arc -> driven net / source member / source pin (-1 -> sentinel)
__global__ void k_arc_keys(const int* arc_from, const int* arc_to, int A,
                           const int* root_net_of_pin, const int* member_of_pin, int N, int M,
                           int P, int* key_in, int* key_out, int* key_pin)
{
    int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= A) return;
    const int j = root_net_of_pin[arc_to[a]];
    key_in[a] = j >= 0 ? j : N;
    const int f = member_of_pin[arc_from[a]];
    key_out[a] = f >= 0 ? f : M;
    key_pin[a] = arc_from[a];
    (void)P;
}

__global__ void k_count(const int* keys, int n, int n_keys, int* cnt)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && keys[i] < n_keys) atomicAdd(&cnt[keys[i]], 1);
}

__global__ void k_net_stats(int N, const int* net_ptr, const int* net_in_ptr, const int* mem_out_ptr,
                            const int* net_root, const int* member_of_pin, int* root_kind,
                            int* net_m, int* net_a, int* net_o)
{
    int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int a = net_in_ptr[n + 1] - net_in_ptr[n];
    net_m[n] = net_ptr[n + 1] - net_ptr[n];
    net_a[n] = a;
    net_o[n] = mem_out_ptr[net_ptr[n + 1]] - mem_out_ptr[net_ptr[n]];
    // flatten.py:281-292 (undriven roots are ROOT_PI, like the reference)
    root_kind[n] = a > 0 ? ROOT_ARC : (member_of_pin[net_root[n]] >= 0 ? ROOT_FEED : ROOT_PI);
}

__global__ void k_flags_u8(const int* idx, int n, uint8_t* flag)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[idx[i]] = 1;
}

// dependency edges (src net -> dst net), slot a for arc a, slot A+j for the
// feedthrough edge of net j; invalid slots get src = N (sorted to the end)
__global__ void k_dep_edges(int A, int N, const int* arc_from, const int* arc_to,
                            const int* root_net_of_pin, const int* member_of_pin,
                            const int* mem_net, const int* net_root, int* src, int* dst,
                            int* indeg)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A + N) return;
    int s = N, d = 0;
    if (i < A) {
        const int j = root_net_of_pin[arc_to[i]];
        const int f = member_of_pin[arc_from[i]];
        if (j >= 0 && f >= 0) { s = mem_net[f]; d = j; }
    } else {
        const int j = i - A;
        const int f = member_of_pin[net_root[j]];
        if (f >= 0) { s = mem_net[f]; d = j; }
    }
    src[i] = s;
    dst[i] = d;
    if (s < N) atomicAdd(&indeg[d], 1);
}

__global__ void k_frontier0(const int* indeg, int N, int* front, int* cnt)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N && indeg[i] == 0) front[atomicAdd(cnt, 1)] = i;
}

__global__ void k_kahn_round(const int* front, int nf, const int* cptr, const int* cons,
                             int* indeg, int* level, int next_level, int* next, int* cnt)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nf) return;
    const int i = front[t];
    for (int q = cptr[i]; q < cptr[i + 1]; q++) {
        const int j = cons[q];
        if (atomicSub(&indeg[j], 1) == 1) {
            level[j] = next_level;
            next[atomicAdd(cnt, 1)] = j;
        }
    }
}

__global__ void k_first_stuck(const int* indeg, int N, int* out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N && indeg[i] > 0) atomicMin(out, i);
}

__global__ void k_free_flags(int P, const int* member_of_pin, const int* root_net_of_pin,
                             const int* pin_out_ptr, uint8_t* free_flag, uint8_t* src_flag)
{
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const bool nonmem = member_of_pin[p] < 0;
    free_flag[p] = nonmem && root_net_of_pin[p] < 0;
    src_flag[p] = nonmem && (pin_out_ptr[p + 1] > pin_out_ptr[p]);
}

__global__ void k_csr(int N, const int* net_ptr, const int* net_root, const int* mem_pin,
                      int* pin_list, int* net_index)
{
    int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n > N) return;
    const int base = net_ptr[n] + n;
    net_index[n] = base;
    if (n == N) return;
    pin_list[base] = net_root[n];
    for (int f = net_ptr[n]; f < net_ptr[n + 1]; f++) pin_list[base + 1 + f - net_ptr[n]] = mem_pin[f];
}


// ---- level-major task layout ------------------------------------------------

__global__ void k_tq(int N, const int* lv_nets, const int* net_root, const int* root_kind,
                     const int* member_of_pin, const int* net_tree, const int* pin_ep_ptr,
                     const int* pin_ep_idx, const int* pin_pi, const int* net_ptr,
                     const int* net_a, const int* net_m, int* tq_root, int* tq_flags, int* tq_f0,
                     int* tq_e1, int* acnt, int* mcnt)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= N) return;
    const int n = lv_nets[q], r = net_root[n];
    int fl = root_kind[n] & TQ_KIND;
    if (member_of_pin[r] >= 0) fl |= TQ_ROOT_MEMBER;
    if (net_tree[n]) fl |= TQ_TREE;
    const int ne = pin_ep_ptr[r + 1] - pin_ep_ptr[r];
    if (ne > 0) fl |= TQ_ROOT_EP;
    if (ne > 1) fl |= TQ_MULTI_EP;
    if (pin_pi[r] >= 0) fl |= TQ_ROOT_PI;
    tq_root[q] = r;
    tq_flags[q] = fl;
    tq_f0[q] = net_ptr[n];
    tq_e1[q] = ne > 0 ? pin_ep_idx[pin_ep_ptr[r]] : -1;
    acnt[q] = (root_kind[n] == ROOT_ARC) ? net_a[n] : 0;
    mcnt[q] = net_m[n];
}

__global__ void k_ta(int N, const int* lv_nets, const int* tq_aptr, const int* tq_root,
                     const int* net_in_ptr, const int* net_in_arc, const int* arc_from,
                     const int* arc_dlut, const int* arc_slut, int* ta_arc, int* ta_from,
                     int* ta_root, int4* ta_lut)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= N) return;
    const int n = lv_nets[q];
    const int cnt = tq_aptr[q + 1] - tq_aptr[q];
    for (int k = 0; k < cnt; k++) {
        const int t = tq_aptr[q] + k, a = net_in_arc[net_in_ptr[n] + k];
        ta_arc[t] = a;
        ta_from[t] = arc_from[a];
        ta_root[t] = tq_root[q];
        const int* d = arc_dlut + 4 * (size_t)a;
        const int* sl = arc_slut + 4 * (size_t)a;
        ta_lut[2 * (size_t)t] = make_int4(d[0], d[1], d[2], d[3]);
        ta_lut[2 * (size_t)t + 1] = make_int4(sl[0], sl[1], sl[2], sl[3]);
    }
}

__global__ void k_tm(int N, const int* lv_nets, const int* tq_mptr, const int* net_ptr,
                     const int* mem_pin, const int* root_net_of_pin, const int* pin_ep_ptr,
                     const int* pin_ep_idx, const int* mem_out_ptr, const int* mem_out_arc,
                     const int* arc_to, int* tm_pin, int* tm_flags, int* tm_o1_to,
                     int* tm_o1_arc, int* tm_e1, int* ocnt)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= N) return;
    const int n = lv_nets[q];
    const int cnt = tq_mptr[q + 1] - tq_mptr[q];
    for (int k = 0; k < cnt; k++) {
        const int u = tq_mptr[q] + k, f = net_ptr[n] + k, pin = mem_pin[f];
        tm_pin[u] = pin;
        int fl = 0;
        if (root_net_of_pin[pin] >= 0) fl |= TM_ROOT;
        const int ne = pin_ep_ptr[pin + 1] - pin_ep_ptr[pin];
        if (ne > 0) fl |= TM_EP;
        if (ne > 1) fl |= TM_MULTI_EP;
        tm_flags[u] = fl;
        tm_e1[u] = ne > 0 ? pin_ep_idx[pin_ep_ptr[pin]] : -1;
        const int o0 = mem_out_ptr[f], o1 = mem_out_ptr[f + 1];
        ocnt[u] = o1 - o0;
        tm_o1_arc[u] = o1 > o0 ? mem_out_arc[o0] : -1;
        tm_o1_to[u] = o1 > o0 ? arc_to[mem_out_arc[o0]] : -1;
    }
}

__global__ void k_to(int N, const int* lv_nets, const int* tq_mptr, const int* net_ptr,
                     const int* tm_optr, const int* mem_out_ptr, const int* mem_out_arc,
                     const int* arc_to, int* to_arc, int* to_to)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= N) return;
    const int n = lv_nets[q];
    const int cnt = tq_mptr[q + 1] - tq_mptr[q];
    for (int k = 0; k < cnt; k++) {
        const int u = tq_mptr[q] + k, f = net_ptr[n] + k;
        for (int o = mem_out_ptr[f]; o < mem_out_ptr[f + 1]; o++) {
            const int v = tm_optr[u] + (o - mem_out_ptr[f]);
            const int a = mem_out_arc[o];
            to_arc[v] = a;
            to_to[v] = arc_to[a];
        }
    }
}

// task-local net index of every arc and member
__global__ void k_task_local(int T, const int4* tk_a, const int4* tk_b, const int* tq_aptr,
                             const int* tq_mptr, int* ta_q, int* tm_flags)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= T) return;
    const int4 a = tk_a[k], b = tk_b[k];
    for (int qi = 0; qi < a.y; qi++) {
        const int q = a.x + qi;
        for (int t = tq_aptr[q]; t < tq_aptr[q + 1]; t++) ta_q[t] = qi;
        const int u0 = max(tq_mptr[q], b.x), u1 = min(tq_mptr[q + 1], b.x + b.y);
        for (int u = u0; u < u1; u++) tm_flags[u] = (tm_flags[u] & 0xff) | (qi << 8);
    }
}

__global__ void k_fin_flags(int P, const int* member_of_pin, const int* root_net_of_pin,
                            const int* pin_out_ptr, uint8_t* flag)
{
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const bool nonmem = member_of_pin[p] < 0;
    const bool root = root_net_of_pin[p] >= 0;
    flag[p] = nonmem && (!root || pin_out_ptr[p + 1] > pin_out_ptr[p]);
}

__global__ void k_fin_kind(int n, const int* fin_pins, const int* root_net_of_pin, int* fin_flags)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) fin_flags[i] = root_net_of_pin[fin_pins[i]] >= 0 ? 1 : 0;
}

int bits_for(int maxkey)
{
    int b = 1;
    while ((1ll << b) <= (long long)maxkey) b++;
    return b;
}

// stable sort of (key, value) pairs; keys in [0, maxkey]
void sort_pairs(Scratch& sc, const int* kin, int* kout, const int* vin, int* vout, int n,
                int maxkey, cudaStream_t s)
{
    if (n == 0) return;
    size_t bytes = 0;
    int eb = bits_for(maxkey);
    WS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, eb, s));
    void* tmp = sc.get(bytes);
    WS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, n, 0, eb, s));
}

// ptr[0..n_keys] = exclusive scan of per-key counts
void counts_to_ptr(Scratch& sc, const int* keys, int n, int n_keys, int* ptr, cudaStream_t s)
{
    WS_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int) * (size_t)(n_keys + 1), s));
    if (n > 0) {
        k_count<<<blocks_for(n), TPB, 0, s>>>(keys, n, n_keys, ptr);
        WS_CHECK_LAUNCH();
    }
    size_t bytes = 0;
    WS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, ptr, ptr, n_keys + 1, s));
    void* tmp = sc.get(bytes);
    WS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, ptr, ptr, n_keys + 1, s));
}

int select_flagged(Scratch& sc, Arena& ar, const uint8_t* flags, int n, int** out, cudaStream_t s)
{
    int* iota = ar.alloc<int>(n);
    k_iota<<<blocks_for(n), TPB, 0, s>>>(iota, n);
    WS_CHECK_LAUNCH();
    int* res = ar.alloc<int>(n);
    int* cnt = ar.alloc<int>(1);
    size_t bytes = 0;
    WS_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, iota, flags, res, cnt, n, s));
    void* tmp = sc.get(bytes);
    WS_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, iota, flags, res, cnt, n, s));
    int h = 0;
    WS_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    WS_CUDA(cudaStreamSynchronize(s));
    *out = res;
    return h;
}

template <class T>
T* upload(Arena& ar, const T* src, size_t n, cudaStream_t s)
{
    T* d = ar.alloc<T>(n);
    if (n) WS_CUDA(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}

int reduce_max(Scratch& sc, Arena& ar, const int* a, int n, cudaStream_t s)
{
    if (n == 0) return 0;
    int* o = ar.alloc<int>(1);
    size_t bytes = 0;
    WS_CUDA(cub::DeviceReduce::Max(nullptr, bytes, a, o, n, s));
    void* tmp = sc.get(bytes);
    WS_CUDA(cub::DeviceReduce::Max(tmp, bytes, a, o, n, s));
    int h = 0;
    WS_CUDA(cudaMemcpyAsync(&h, o, sizeof(int), cudaMemcpyDeviceToHost, s));
    WS_CUDA(cudaStreamSynchronize(s));
    return h;
}

// delay LUT ids of each task net's first in-arc (the root-load locate axis)
__global__ void k_tq_lut1(int N, const int* tq_aptr, const int4* ta_lut, int4* out)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= N) return;
    out[q] = tq_aptr[q + 1] > tq_aptr[q] ? ta_lut[2 * (size_t)tq_aptr[q]]
                                         : make_int4(-1, -1, -1, -1);
}

// streaming-RC member code: -1 for members of tree nets (handled per net),
// else pin << 1 | (pin roots a net: its load comes from that net)
__global__ void k_rc_code(int M, const int* mem_pin, const int* mem_net, const int* net_tree,
                          const int* root_net_of_pin, int* code)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= M) return;
    const int pin = mem_pin[f];
    code[f] = net_tree[mem_net[f]] ? -1 : (pin << 1) | (root_net_of_pin[pin] >= 0 ? 1 : 0);
}

// per-pin code of the pin-order streaming RC: (member << 2) | (pin roots a
// net) << 1 | 1 for a star-net member, 2 for a root that is no member (its
// delay and impulse are 0), 0 for pins the kernel skips (tree-net members:
// k_rc_tree; pins in no net: the free-pin blocks)
__global__ void k_rc_pcode(int P, const int* member_of_pin, const int* root_net_of_pin,
                           const int* mem_net, const int* net_tree, int* pcode)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int f = member_of_pin[p], rn = root_net_of_pin[p];
    int code = 0;
    if (f >= 0) code = net_tree[mem_net[f]] ? 0 : ((f << 2) | (rn >= 0 ? 2 : 0) | 1);
    else if (rn >= 0) code = 2;
    pcode[p] = code;
}

// the nets whose root load a streaming-RC member block folds: block b owns
// nets [bnet[b], bnet[b + 1]) (lower bound of b * RC_MPB in net_ptr); the
// last block also owns the trailing member-less nets
__global__ void k_rc_bnet(int nb, int N, const int* net_ptr, int* bnet)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    if (b == nb) { bnet[b] = N; return; }
    const int key = b * RC_MPB;
    int lo = 0, hi = N;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (net_ptr[mid] < key) lo = mid + 1; else hi = mid;
    }
    bnet[b] = lo;
}

}  // namespace


// Level-major task arrays and the task partition of every level.

// per-task record blobs (see Topo::fb_*): the records of task k's level
// kernels, laid out by (task, slot) so a block loads them from its task index
__global__ void k_blob(Topo t)
{
    const int k = blockIdx.x, tid = threadIdx.x;
    const int4 A = t.tk_a[k], B = t.tk_b[k];
    const int q0 = A.x, nq = A.y, a0 = A.z, na_t = A.w, m0 = B.x, nm = B.y, tflags = B.z;
    const bool wide = tflags & TK_WIDE;
    if (tid <= TASK_Q) {
        int4 a = make_int4(0, 0, 0, 0), b = make_int4(0, 0, 0, 0);
        if (tid <= nq) {
            const int q = q0 + tid;
            b.y = t.tq_aptr[q];
            b.z = t.tq_mptr[q];
            if (tid < nq) {
                a = make_int4(t.tq_root[q], t.tq_flags[q], t.tq_f0[q], t.lv_nets[q]);
                b.x = t.tq_e1[q];
            }
        }
        t.fb_n[2 * ((size_t)k * (TASK_Q + 1) + tid)] = a;
        t.fb_n[2 * ((size_t)k * (TASK_Q + 1) + tid) + 1] = b;
    }
    if (tid < TASK_Q) {
        const int qi = tid;
        int4 fq = make_int4(-1, 0, 0, 0), bq = make_int4(-1, 0, -1, 0);
        if (qi < nq) {
            const int q = q0 + qi;
            fq.x = t.tq_root[q];
            fq.y = t.tq_flags[q];
            if ((fq.y & TQ_KIND) == ROOT_ARC && !wide) {
                fq.z = t.tq_aptr[q];
                fq.w = t.tq_aptr[q + 1] - fq.z;
            }
            bq = make_int4(fq.x, fq.y, t.tq_e1[q], 0);
        }
        t.fb_q[(size_t)k * TASK_Q + qi] = fq;
        t.bb_q[(size_t)k * TASK_Q + qi] = bq;
        for (int s = 0; s < 3; s++) {
            int2 fa = make_int2(0, 0);
            int4 fd = make_int4(0, 0, 0, 0), fs = make_int4(0, 0, 0, 0);
            if (fq.w > 0 && fq.w <= 3) {
                // slots past the last arc repeat arc 0 (branch-free net phase)
                const int qa = fq.z + (s < fq.w ? s : 0);
                fa = make_int2(t.ta_from[qa], t.ta_arc[qa]);
                fd = t.ta_lut[2 * (size_t)qa];
                fs = t.ta_lut[2 * (size_t)qa + 1];
            }
            t.fb_a[((size_t)k * TASK_Q + qi) * 3 + s] = fa;
            t.fb_l[2 * (((size_t)k * TASK_Q + qi) * 3 + s)] = fd;
            t.fb_l[2 * (((size_t)k * TASK_Q + qi) * 3 + s) + 1] = fs;
        }
    }
    if (tid < TASK_M) {
        const int ii = tid;
        int2 fm = make_int2(-1, 0);
        int4 m1 = make_int4(-1, 0, -1, -1), m2 = make_int4(-1, 0, 0, -1);
        if (ii < nm) {
            const int u = m0 + ii;
            fm = make_int2(t.tm_pin[u], t.tm_flags[u]);
            m1 = make_int4(fm.x, fm.y, t.tm_o1_to[u], t.tm_o1_arc[u]);
            m2.x = t.tm_e1[u];
            m2.y = t.tm_optr[u];
            m2.z = t.tm_optr[u + 1] - m2.y;
        }
        if (ii < na_t && !wide) m2.w = t.ta_arc[a0 + ii];
        t.fb_m[(size_t)k * TASK_M + ii] = fm;
        t.bb_m[2 * ((size_t)k * TASK_M + ii)] = m1;
        t.bb_m[2 * ((size_t)k * TASK_M + ii) + 1] = m2;
    }
}

void build_tasks(Context& ctx)
{
    Topo& t = ctx.t;
    Arena& ar = ctx.topo_mem;
    Scratch& sc = ctx.scratch;
    cudaStream_t s = ctx.s_main;
    const int N = t.N, M = t.M, P = t.P;
    t.tq_root = ar.alloc<int>(N);
    t.tq_flags = ar.alloc<int>(N);
    t.tq_f0 = ar.alloc<int>(N);
    t.tq_e1 = ar.alloc<int>(N);
    t.tq_aptr = ar.alloc<int>(N + 1);
    t.tq_mptr = ar.alloc<int>(N + 1);
    int* acnt = ar.alloc<int>(N + 1);
    int* mcnt = ar.alloc<int>(N + 1);
    WS_CUDA(cudaMemsetAsync(acnt, 0, sizeof(int) * (size_t)(N + 1), s));
    WS_CUDA(cudaMemsetAsync(mcnt, 0, sizeof(int) * (size_t)(N + 1), s));
    if (N) {
        k_tq<<<blocks_for(N), TPB, 0, s>>>(N, t.lv_nets, t.net_root, t.root_kind, t.member_of_pin,
                                           t.net_tree, t.pin_ep_ptr, t.pin_ep_idx, t.pin_pi,
                                           t.net_ptr, t.net_a, t.net_m, t.tq_root, t.tq_flags,
                                           t.tq_f0, t.tq_e1, acnt, mcnt);
        WS_CHECK_LAUNCH();
    }
    auto scan = [&](int* in, int* out, int n) {
        size_t bytes = 0;
        WS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n + 1, s));
        void* tmp = sc.get(bytes);
        WS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n + 1, s));
    };
    scan(acnt, t.tq_aptr, N);
    scan(mcnt, t.tq_mptr, N);
    int na = 0;
    WS_CUDA(cudaMemcpyAsync(&na, t.tq_aptr + N, sizeof(int), cudaMemcpyDeviceToHost, s));
    WS_CUDA(cudaStreamSynchronize(s));
    t.ta_arc = ar.alloc<int>(na);
    t.ta_from = ar.alloc<int>(na);
    t.ta_root = ar.alloc<int>(na);
    t.ta_q = ar.alloc<int>(na);
    t.ta_lut = ar.alloc<int4>(2 * (size_t)na);
    t.tm_pin = ar.alloc<int>(M);
    t.tm_flags = ar.alloc<int>(M);
    t.tm_optr = ar.alloc<int>(M + 1);
    t.tm_o1_to = ar.alloc<int>(M);
    t.tm_o1_arc = ar.alloc<int>(M);
    t.tm_e1 = ar.alloc<int>(M);
    int* ocnt = ar.alloc<int>(M + 1);
    WS_CUDA(cudaMemsetAsync(ocnt, 0, sizeof(int) * (size_t)(M + 1), s));
    if (N) {
        k_ta<<<blocks_for(N), TPB, 0, s>>>(N, t.lv_nets, t.tq_aptr, t.tq_root, t.net_in_ptr,
                                           t.net_in_arc, t.arc_from, t.arc_dlut, t.arc_slut,
                                           t.ta_arc, t.ta_from, t.ta_root, t.ta_lut);
        k_tm<<<blocks_for(N), TPB, 0, s>>>(N, t.lv_nets, t.tq_mptr, t.net_ptr, t.mem_pin,
                                           t.root_net_of_pin, t.pin_ep_ptr, t.pin_ep_idx,
                                           t.mem_out_ptr, t.mem_out_arc, t.arc_to, t.tm_pin,
                                           t.tm_flags, t.tm_o1_to, t.tm_o1_arc, t.tm_e1, ocnt);
        WS_CHECK_LAUNCH();
    }
    t.tq_lut1 = ar.alloc<int4>(N);
    if (N) {
        k_tq_lut1<<<blocks_for(N), TPB, 0, s>>>(N, t.tq_aptr, t.ta_lut, t.tq_lut1);
        WS_CHECK_LAUNCH();
    }
    scan(ocnt, t.tm_optr, M);
    int no = 0;
    WS_CUDA(cudaMemcpyAsync(&no, t.tm_optr + M, sizeof(int), cudaMemcpyDeviceToHost, s));
    WS_CUDA(cudaStreamSynchronize(s));
    t.to_arc = ar.alloc<int>(no);
    t.to_to = ar.alloc<int>(no);
    if (N) {
        k_to<<<blocks_for(N), TPB, 0, s>>>(N, t.lv_nets, t.tq_mptr, t.net_ptr, t.tm_optr,
                                           t.mem_out_ptr, t.mem_out_arc, t.arc_to, t.to_arc, t.to_to);
        WS_CHECK_LAUNCH();
    }
    // ---- task partition, level by level (host; one-time) -------------------
    std::vector<int> mptr(N + 1), aptr(N + 1), fl(N);
    WS_CUDA(cudaMemcpy(mptr.data(), t.tq_mptr, sizeof(int) * (size_t)(N + 1), cudaMemcpyDeviceToHost));
    WS_CUDA(cudaMemcpy(aptr.data(), t.tq_aptr, sizeof(int) * (size_t)(N + 1), cudaMemcpyDeviceToHost));
    if (N) WS_CUDA(cudaMemcpy(fl.data(), t.tq_flags, sizeof(int) * (size_t)N, cudaMemcpyDeviceToHost));
    std::vector<int4> ta_, tb_;
    std::vector<int> nch, part0;
    int n_parts = 0;
    ctx.lvt_ptr_host.assign(t.L + 1, 0);
    for (int li = 0; li < t.L; li++) {
        ctx.lvt_ptr_host[li] = (int)ta_.size();
        int cq = -1, cn = 0, ca = 0, cm = 0;
        auto flush = [&]() {
            if (cq >= 0) {
                ta_.push_back(make_int4(cq, cn, aptr[cq], ca));
                tb_.push_back(make_int4(mptr[cq], cm, 0, -1));
            }
            cq = -1; cn = ca = cm = 0;
        };
        for (int q = ctx.lv_ptr_host[li]; q < ctx.lv_ptr_host[li + 1]; q++) {
            const int m = mptr[q + 1] - mptr[q], a = aptr[q + 1] - aptr[q];
            const bool tree = fl[q] & TQ_TREE;
            if (a > TASK_A || (m > TASK_M && tree)) {
                flush();
                int f = 0;
                if (a > TASK_A) f |= TK_WIDE;
                if (m > TASK_M) f |= TK_LOOP;
                ta_.push_back(make_int4(q, 1, aptr[q], a));
                tb_.push_back(make_int4(mptr[q], m, f, -1));
                continue;
            }
            if (m > TASK_M) {           // big star net: chunks of TASK_M members
                flush();
                const int k = (m + TASK_M - 1) / TASK_M, slot = (int)nch.size();
                nch.push_back(k);
                part0.push_back(n_parts);
                n_parts += k;
                for (int c = 0; c < k; c++) {
                    ta_.push_back(make_int4(q, 1, aptr[q], a));
                    tb_.push_back(make_int4(mptr[q] + c * TASK_M, std::min(TASK_M, m - c * TASK_M),
                                            TK_CHUNK, slot));
                }
                continue;
            }
            if (cq < 0 || cn >= TASK_Q || ca + a > TASK_A || cm + m > TASK_M) {
                flush();
                cq = q;
            }
            cn++;
            ca += a;
            cm += m;
        }
        flush();
    }
    ctx.lvt_ptr_host[t.L] = (int)ta_.size();
    t.n_tasks = (int)ta_.size();
    t.lvt_ptr = ar.alloc<int>(t.L + 1);
    WS_CUDA(cudaMemcpy(t.lvt_ptr, ctx.lvt_ptr_host.data(), sizeof(int) * (size_t)(t.L + 1),
                       cudaMemcpyHostToDevice));
    t.tk_a = ar.alloc<int4>(ta_.size());
    t.tk_b = ar.alloc<int4>(tb_.size());
    if (!ta_.empty()) {
        WS_CUDA(cudaMemcpy(t.tk_a, ta_.data(), sizeof(int4) * ta_.size(), cudaMemcpyHostToDevice));
        WS_CUDA(cudaMemcpy(t.tk_b, tb_.data(), sizeof(int4) * tb_.size(), cudaMemcpyHostToDevice));
    }
    t.n_big = (int)nch.size();
    t.n_parts = n_parts;
    t.bn_nch = ar.alloc<int>(nch.size());
    t.bn_part0 = ar.alloc<int>(part0.size());
    if (!nch.empty()) {
        WS_CUDA(cudaMemcpy(t.bn_nch, nch.data(), sizeof(int) * nch.size(), cudaMemcpyHostToDevice));
        WS_CUDA(cudaMemcpy(t.bn_part0, part0.data(), sizeof(int) * part0.size(), cudaMemcpyHostToDevice));
    }
    if (t.n_tasks) {
        k_task_local<<<blocks_for(t.n_tasks), TPB, 0, s>>>(t.n_tasks, t.tk_a, t.tk_b, t.tq_aptr,
                                                           t.tq_mptr, t.ta_q, t.tm_flags);
        WS_CHECK_LAUNCH();
    }
    {
        const size_t T = (size_t)std::max(t.n_tasks, 1);
        t.fb_n = ar.alloc<int4>(T * (TASK_Q + 1) * 2);
        t.fb_q = ar.alloc<int4>(T * TASK_Q);
        t.fb_a = ar.alloc<int2>(T * TASK_Q * 3);
        t.fb_l = ar.alloc<int4>(T * TASK_Q * 3 * 2);
        t.fb_m = ar.alloc<int2>(T * TASK_M);
        t.bb_m = ar.alloc<int4>(T * TASK_M * 2);
        t.bb_q = ar.alloc<int4>(T * TASK_Q);
        if (t.n_tasks) {
            k_blob<<<t.n_tasks, PASS_TPB, 0, s>>>(t);   // after k_task_local: tm_flags final
            WS_CHECK_LAUNCH();
        }
    }
    // pins finished after the level loop
    uint8_t* ff = ar.alloc<uint8_t>(P);
    if (P) {
        k_fin_flags<<<blocks_for(P), TPB, 0, s>>>(P, t.member_of_pin, t.root_net_of_pin,
                                                  t.pin_out_ptr, ff);
        WS_CHECK_LAUNCH();
    }
    t.n_fin = P ? select_flagged(sc, ar, ff, P, &t.fin_pins, s) : 0;
    t.fin_flags = ar.alloc<int>(t.n_fin);
    if (t.n_fin) {
        k_fin_kind<<<blocks_for(t.n_fin), TPB, 0, s>>>(t.n_fin, t.fin_pins, t.root_net_of_pin,
                                                       t.fin_flags);
        WS_CHECK_LAUNCH();
    }
}

void build_topology(Context& ctx, const ws_design_desc* d)
{
    Topo& t = ctx.t;
    Arena& ar = ctx.topo_mem;
    Scratch& sc = ctx.scratch;
    cudaStream_t s = ctx.s_main;
    const int64_t lim = (int64_t)INT32_MAX - 2;
    if (d->n_pins < 0 || d->n_nets < 0 || d->n_members < 0 || d->n_arcs < 0 || d->n_pi < 0 ||
        d->n_ep < 0 || d->n_luts < 0)
        throw Error(WS_ERR_VALUE, "negative size in design descriptor");
    if (d->n_pins > lim || d->n_members > lim || d->n_arcs > lim || d->n_nets > lim)
        throw Error(WS_ERR_VALUE, "design exceeds the int32 index range");
    t.P = (int)d->n_pins; t.N = (int)d->n_nets; t.M = (int)d->n_members; t.A = (int)d->n_arcs;
    t.I = (int)d->n_pi; t.E = (int)d->n_ep; t.NL = (int)d->n_luts;
    const int P = t.P, N = t.N, M = t.M, A = t.A;

    // host-side range checks on the indices (the device build assumes them)
    auto chk = [&](const int32_t* a, int64_t n, int64_t hi, const char* what) {
        for (int64_t i = 0; i < n; i++)
            if (a[i] < 0 || a[i] >= hi)
                throw Error(WS_ERR_VALUE, std::string(what) + " index out of range");
    };
    chk(d->net_root, N, P, "net_root");
    chk(d->mem_pin, M, P, "mem_pin");
    chk(d->mem_parent_pin, M, P, "mem_parent_pin");
    chk(d->arc_from, A, P, "arc_from");
    chk(d->arc_to, A, P, "arc_to");
    chk(d->arc_dlut, 4 * (int64_t)A, t.NL, "arc_dlut");
    chk(d->arc_slut, 4 * (int64_t)A, t.NL, "arc_slut");
    chk(d->pi_pin, t.I, P, "pi_pin");
    chk(d->ep_pin, t.E, P, "ep_pin");
    if (d->net_mptr[0] != 0 || d->net_mptr[N] != M)
        throw Error(WS_ERR_VALUE, "net_mptr does not span the members");
    for (int64_t i = 0; i < N; i++)
        if (d->net_mptr[i + 1] < d->net_mptr[i]) throw Error(WS_ERR_VALUE, "net_mptr not monotone");
    for (int64_t i = 0; i < t.NL; i++) {
        const int ns = d->lut_s_ptr[i + 1] - d->lut_s_ptr[i];
        const int nl = d->lut_l_ptr[i + 1] - d->lut_l_ptr[i];
        if (ns < 1 || nl < 1 || d->lut_t_ptr[i + 1] - d->lut_t_ptr[i] != ns * nl)
            throw Error(WS_ERR_VALUE, "malformed LUT pool");
    }

    // ---- upload topology ------------------------------------------------
    std::vector<int> nptr(N + 1);
    for (int i = 0; i <= N; i++) nptr[i] = (int)d->net_mptr[i];
    t.net_ptr = upload(ar, nptr.data(), N + 1, s);
    t.net_root = upload(ar, d->net_root, N, s);
    t.mem_pin = upload(ar, d->mem_pin, M, s);
    int* mem_parent_pin = upload(ar, d->mem_parent_pin, M, s);
    t.arc_from = upload(ar, d->arc_from, A, s);
    t.arc_to = upload(ar, d->arc_to, A, s);
    t.arc_dlut = upload(ar, d->arc_dlut, 4 * (size_t)A, s);
    t.arc_slut = upload(ar, d->arc_slut, 4 * (size_t)A, s);
    t.pi_pin = upload(ar, d->pi_pin, t.I, s);
    t.ep_pin = upload(ar, d->ep_pin, t.E, s);
    t.lut_s_ptr = upload(ar, d->lut_s_ptr, t.NL + 1, s);
    t.lut_l_ptr = upload(ar, d->lut_l_ptr, t.NL + 1, s);
    t.lut_t_ptr = upload(ar, d->lut_t_ptr, t.NL + 1, s);
    ctx.lut_s_len = (int)d->lut_s_len;
    ctx.lut_l_len = (int)d->lut_l_len;
    ctx.lut_t_len = (int)d->lut_t_len;
    t.lut_s_flat = upload(ar, d->lut_s_flat, d->lut_s_len, s);
    t.lut_l_flat = upload(ar, d->lut_l_flat, d->lut_l_len, s);
    {
        // canonical axis offsets: LUTs whose axis arrays hold identical values
        // share one offset, so the level kernels locate a query once for both
        // an arc's delay and slew tables (same result, bit for bit)
        std::vector<int4> info((size_t)std::max<int64_t>(d->n_luts, 1));
        // (hashed on the axis bytes: O(n) for pools of any size; identical
        // bits are a stricter test than ==, so merging stays exact)
        auto canon = [](const double* flat, const int32_t* ptr, int64_t nl, std::vector<int>& out) {
            out.assign((size_t)nl, 0);
            std::unordered_map<std::string, int> first;
            first.reserve((size_t)nl);
            for (int64_t i = 0; i < nl; i++) {
                const char* b = reinterpret_cast<const char*>(flat + ptr[i]);
                std::string key(b, sizeof(double) * (size_t)(ptr[i + 1] - ptr[i]));
                out[(size_t)i] = first.emplace(std::move(key), ptr[i]).first->second;
            }
        };
        std::vector<int> cs_, cl_;
        canon(d->lut_s_flat, d->lut_s_ptr, d->n_luts, cs_);
        canon(d->lut_l_flat, d->lut_l_ptr, d->n_luts, cl_);
        for (int64_t i = 0; i < d->n_luts; i++)
            info[(size_t)i] = make_int4(cs_[(size_t)i], d->lut_s_ptr[i + 1] - d->lut_s_ptr[i],
                                        cl_[(size_t)i], d->lut_l_ptr[i + 1] - d->lut_l_ptr[i]);
        t.lut_info = upload(ar, info.data(), info.size(), s);
        WS_CUDA(cudaStreamSynchronize(s));
    }

    // ---- maps (flatten.py:190-206) --------------------------------------
    t.member_of_pin = ar.alloc<int>(P);
    t.root_net_of_pin = ar.alloc<int>(P);
    k_fill<<<blocks_for(P), TPB, 0, s>>>(t.member_of_pin, P, -1);
    k_fill<<<blocks_for(P), TPB, 0, s>>>(t.root_net_of_pin, P, -1);
    if (M) k_scatter_last<<<blocks_for(M), TPB, 0, s>>>(t.mem_pin, M, t.member_of_pin);
    if (N) k_scatter_last<<<blocks_for(N), TPB, 0, s>>>(t.net_root, N, t.root_net_of_pin);
    WS_CHECK_LAUNCH();
    t.mem_net = ar.alloc<int>(M);
    t.mem_local = ar.alloc<int>(M);
    t.mem_parent_loc = ar.alloc<int>(M);
    t.net_tree = ar.alloc<int>(N);
    WS_CUDA(cudaMemsetAsync(t.net_tree, 0, sizeof(int) * (size_t)std::max(N, 1), s));
    if (M) {
        k_mem_fields<<<blocks_for(M), TPB, 0, s>>>(t.net_ptr, N, M, t.net_root, mem_parent_pin,
                                                   t.member_of_pin, t.mem_net, t.mem_local,
                                                   t.mem_parent_loc, t.net_tree);
        WS_CHECK_LAUNCH();
    }

    // ---- arc groupings (flatten.py:246-268) ------------------------------
    int* key_in = ar.alloc<int>(A);
    int* key_out = ar.alloc<int>(A);
    int* key_pin = ar.alloc<int>(A);
    int* iota = ar.alloc<int>(A);
    int* ksorted = ar.alloc<int>(A);
    if (A) {
        k_arc_keys<<<blocks_for(A), TPB, 0, s>>>(t.arc_from, t.arc_to, A, t.root_net_of_pin,
                                                 t.member_of_pin, N, M, P, key_in, key_out, key_pin);
        k_iota<<<blocks_for(A), TPB, 0, s>>>(iota, A);
        WS_CHECK_LAUNCH();
    }
    int* in_arc_all = ar.alloc<int>(A);
    int* out_arc_all = ar.alloc<int>(A);
    t.pin_out_arc = ar.alloc<int>(A);
    sort_pairs(sc, key_in, ksorted, iota, in_arc_all, A, N, s);
    sort_pairs(sc, key_out, ksorted, iota, out_arc_all, A, M, s);
    sort_pairs(sc, key_pin, ksorted, iota, t.pin_out_arc, A, P, s);
    t.net_in_ptr = ar.alloc<int>(N + 1);
    t.mem_out_ptr = ar.alloc<int>(M + 1);
    t.pin_out_ptr = ar.alloc<int>(P + 1);
    counts_to_ptr(sc, key_in, A, N, t.net_in_ptr, s);
    counts_to_ptr(sc, key_out, A, M, t.mem_out_ptr, s);
    counts_to_ptr(sc, key_pin, A, P, t.pin_out_ptr, s);
    t.net_in_arc = in_arc_all;    // entries beyond net_in_ptr[N] are the sentinel group
    t.mem_out_arc = out_arc_all;

    // ---- per-net stats, root kinds (flatten.py:281-298) -----------------
    t.root_kind = ar.alloc<int>(N);
    t.net_m = ar.alloc<int>(N);
    t.net_a = ar.alloc<int>(N);
    t.net_o = ar.alloc<int>(N);
    if (N) {
        k_net_stats<<<blocks_for(N), TPB, 0, s>>>(N, t.net_ptr, t.net_in_ptr, t.mem_out_ptr,
                                                  t.net_root, t.member_of_pin, t.root_kind,
                                                  t.net_m, t.net_a, t.net_o);
        WS_CHECK_LAUNCH();
    }
    t.is_endpoint = ar.alloc<uint8_t>(P);
    WS_CUDA(cudaMemsetAsync(t.is_endpoint, 0, (size_t)std::max(P, 1), s));
    if (t.E) k_flags_u8<<<blocks_for(t.E), TPB, 0, s>>>(t.ep_pin, t.E, t.is_endpoint);
    t.pin_pi = ar.alloc<int>(P);
    k_fill<<<blocks_for(P), TPB, 0, s>>>(t.pin_pi, P, -1);
    if (t.I) k_scatter_last<<<blocks_for(t.I), TPB, 0, s>>>(t.pi_pin, t.I, t.pin_pi);
    WS_CHECK_LAUNCH();
    // endpoint entries grouped by pin, entry order kept (np.minimum.at order)
    {
        int* eiota = ar.alloc<int>(t.E);
        int* ek = ar.alloc<int>(t.E);
        t.pin_ep_idx = ar.alloc<int>(t.E);
        if (t.E) {
            k_iota<<<blocks_for(t.E), TPB, 0, s>>>(eiota, t.E);
            WS_CHECK_LAUNCH();
        }
        sort_pairs(sc, t.ep_pin, ek, eiota, t.pin_ep_idx, t.E, P, s);
        t.pin_ep_ptr = ar.alloc<int>(P + 1);
        counts_to_ptr(sc, t.ep_pin, t.E, P, t.pin_ep_ptr, s);
    }

    // ---- levelize: dependency edges + frontier Kahn ----------------------
    t.level_of = ar.alloc<int>(N);
    WS_CUDA(cudaMemsetAsync(t.level_of, 0, sizeof(int) * (size_t)std::max(N, 1), s));
    int n_levels = 0;
    if (N) {
        const int ne = A + N;
        int* esrc = ar.alloc<int>(ne);
        int* edst = ar.alloc<int>(ne);
        int* esrc_s = ar.alloc<int>(ne);
        int* cons = ar.alloc<int>(ne);
        int* indeg = ar.alloc<int>(N);
        WS_CUDA(cudaMemsetAsync(indeg, 0, sizeof(int) * (size_t)N, s));
        k_dep_edges<<<blocks_for(ne), TPB, 0, s>>>(A, N, t.arc_from, t.arc_to, t.root_net_of_pin,
                                                   t.member_of_pin, t.mem_net, t.net_root, esrc,
                                                   edst, indeg);
        WS_CHECK_LAUNCH();
        sort_pairs(sc, esrc, esrc_s, edst, cons, ne, N, s);
        int* cptr = ar.alloc<int>(N + 1);
        counts_to_ptr(sc, esrc, ne, N, cptr, s);
        int* fa = ar.alloc<int>(N);
        int* fb = ar.alloc<int>(N);
        int* cnt = ar.alloc<int>(1);
        WS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), s));
        k_frontier0<<<blocks_for(N), TPB, 0, s>>>(indeg, N, fa, cnt);
        WS_CHECK_LAUNCH();
        int nf = 0;
        WS_CUDA(cudaMemcpyAsync(&nf, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
        WS_CUDA(cudaStreamSynchronize(s));
        int done = 0;
        while (nf > 0) {
            done += nf;
            n_levels++;
            WS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), s));
            k_kahn_round<<<blocks_for(nf), TPB, 0, s>>>(fa, nf, cptr, cons, indeg, t.level_of,
                                                        n_levels, fb, cnt);
            WS_CHECK_LAUNCH();
            WS_CUDA(cudaMemcpyAsync(&nf, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
            WS_CUDA(cudaStreamSynchronize(s));
            std::swap(fa, fb);
        }
        if (done != N) {
            int* st = ar.alloc<int>(1);
            k_fill<<<1, 1, 0, s>>>(st, 1, N);
            k_first_stuck<<<blocks_for(N), TPB, 0, s>>>(indeg, N, st);
            WS_CHECK_LAUNCH();
            int stuck = 0, root = 0;
            WS_CUDA(cudaMemcpyAsync(&stuck, st, sizeof(int), cudaMemcpyDeviceToHost, s));
            WS_CUDA(cudaStreamSynchronize(s));
            WS_CUDA(cudaMemcpy(&root, t.net_root + stuck, sizeof(int), cudaMemcpyDeviceToHost));
            throw Error(WS_ERR_CYCLE, "combinational cycle through pin " + std::to_string(root), root);
        }
    }
    t.L = n_levels;
    // nets sorted by (level, id): stable radix sort of ids keyed by level
    t.lv_nets = ar.alloc<int>(N);
    t.lv_ptr = ar.alloc<int>(t.L + 1);
    if (N) {
        int* niota = ar.alloc<int>(N);
        int* lk = ar.alloc<int>(N);
        k_iota<<<blocks_for(N), TPB, 0, s>>>(niota, N);
        WS_CHECK_LAUNCH();
        sort_pairs(sc, t.level_of, lk, niota, t.lv_nets, N, std::max(t.L - 1, 0), s);
    }
    counts_to_ptr(sc, t.level_of, N, t.L, t.lv_ptr, s);

    // ---- derived work lists ----------------------------------------------
    {
        uint8_t* ff = ar.alloc<uint8_t>(P);
        uint8_t* sf = ar.alloc<uint8_t>(P);
        if (P) {
            k_free_flags<<<blocks_for(P), TPB, 0, s>>>(P, t.member_of_pin, t.root_net_of_pin,
                                                       t.pin_out_ptr, ff, sf);
            WS_CHECK_LAUNCH();
        }
        t.n_free = P ? select_flagged(sc, ar, ff, P, &t.free_pins, s) : 0;
        t.n_nonmem_src = P ? select_flagged(sc, ar, sf, P, &t.nonmem_src, s) : 0;
    }
    t.max_in = reduce_max(sc, ar, t.net_a, N, s);
    t.max_m = reduce_max(sc, ar, t.net_m, N, s);
    t.rc_code = ar.alloc<int>(M);
    if (M) {
        k_rc_code<<<blocks_for(M), TPB, 0, s>>>(M, t.mem_pin, t.mem_net, t.net_tree,
                                                  t.root_net_of_pin, t.rc_code);
        WS_CHECK_LAUNCH();
    }
    t.rc_pcode = ar.alloc<int>(P);
    if (P) {
        k_rc_pcode<<<blocks_for(P), TPB, 0, s>>>(P, t.member_of_pin, t.root_net_of_pin, t.mem_net,
                                                 t.net_tree, t.rc_pcode);
        WS_CHECK_LAUNCH();
    }

    // host copies of the level schedule and per-level shape stats
    ctx.lv_ptr_host.assign(t.L + 1, 0);
    if (t.L) WS_CUDA(cudaMemcpy(ctx.lv_ptr_host.data(), t.lv_ptr, sizeof(int) * (t.L + 1),
                                cudaMemcpyDeviceToHost));
    {
        std::vector<int> lvn(N), nm(N), tr(N);
        if (N) {
            WS_CUDA(cudaMemcpy(lvn.data(), t.lv_nets, sizeof(int) * N, cudaMemcpyDeviceToHost));
            WS_CUDA(cudaMemcpy(nm.data(), t.net_m, sizeof(int) * N, cudaMemcpyDeviceToHost));
            WS_CUDA(cudaMemcpy(tr.data(), t.net_tree, sizeof(int) * N, cudaMemcpyDeviceToHost));
        }
        ctx.lv_maxm_host.assign(t.L, 0);
        ctx.lv_tree_host.assign(t.L, 0);
        ctx.any_tree = false;
        for (int n = 0; n < N; n++) ctx.any_tree |= tr[n] != 0;
        for (int li = 0; li < t.L; li++)
            for (int q = ctx.lv_ptr_host[li]; q < ctx.lv_ptr_host[li + 1]; q++) {
                ctx.lv_maxm_host[li] = std::max(ctx.lv_maxm_host[li], nm[lvn[q]]);
                ctx.lv_tree_host[li] |= tr[lvn[q]];
            }
    }

    build_tasks(ctx);
    {
        // last in the arena: the batch-only RC owner table leaves the
        // addresses of everything the single-corner pass reads unchanged
        const int nb = (M + RC_MPB - 1) / RC_MPB;
        ctx.rc_bnet = ar.alloc<int>(nb + 1);
        k_rc_bnet<<<blocks_for(nb + 1), TPB, 0, s>>>(nb, N, t.net_ptr, ctx.rc_bnet);
        WS_CHECK_LAUNCH();
    }
    WS_CUDA(cudaStreamSynchronize(s));
}

int64_t topo_field_len(Context& ctx, int field)
{
    const Topo& t = ctx.t;
    switch (field) {
    case WS_T_NET_PTR: return t.N + 1;
    case WS_T_NET_ROOT: case WS_T_ROOT_KIND: case WS_T_NET_M: case WS_T_NET_A: case WS_T_NET_O:
    case WS_T_LEVEL_OF: case WS_T_LEVEL_NETS: return t.N;
    case WS_T_MEM_PIN: case WS_T_MEM_PARENT_LOC: case WS_T_MEM_NET: case WS_T_MEM_LOCAL: return t.M;
    case WS_T_ARC_FROM: case WS_T_ARC_TO: return t.A;
    case WS_T_ARC_DLUT: case WS_T_ARC_SLUT: return 4ll * t.A;
    case WS_T_NET_IN_PTR: return t.N + 1;
    case WS_T_MEM_OUT_PTR: return t.M + 1;
    case WS_T_NET_IN_ARC: {
        int v = 0;
        WS_CUDA(cudaMemcpy(&v, t.net_in_ptr + t.N, sizeof(int), cudaMemcpyDeviceToHost));
        return v;
    }
    case WS_T_MEM_OUT_ARC: {
        int v = 0;
        WS_CUDA(cudaMemcpy(&v, t.mem_out_ptr + t.M, sizeof(int), cudaMemcpyDeviceToHost));
        return v;
    }
    case WS_T_MEMBER_OF_PIN: case WS_T_ROOT_NET_OF_PIN: case WS_T_IS_ENDPOINT: return t.P;
    case WS_T_LEVEL_PTR: return t.L + 1;
    case WS_T_CSR_PIN_LIST: return (int64_t)t.N + t.M;
    case WS_T_CSR_NET_INDEX: return t.N + 1;
    default: throw Error(WS_ERR_VALUE, "unknown topology field");
    }
}

void topo_field_to_host(Context& ctx, int field, int64_t* dst)
{
    const Topo& t = ctx.t;
    const int64_t n = topo_field_len(ctx, field);
    if (n == 0) return;
    std::vector<int> tmp((size_t)n);
    const int* src = nullptr;
    Arena scratch_arena;
    switch (field) {
    case WS_T_NET_PTR: src = t.net_ptr; break;
    case WS_T_NET_ROOT: src = t.net_root; break;
    case WS_T_ROOT_KIND: src = t.root_kind; break;
    case WS_T_MEM_PIN: src = t.mem_pin; break;
    case WS_T_MEM_PARENT_LOC: src = t.mem_parent_loc; break;
    case WS_T_MEM_NET: src = t.mem_net; break;
    case WS_T_MEM_LOCAL: src = t.mem_local; break;
    case WS_T_ARC_FROM: src = t.arc_from; break;
    case WS_T_ARC_TO: src = t.arc_to; break;
    case WS_T_ARC_DLUT: src = t.arc_dlut; break;
    case WS_T_ARC_SLUT: src = t.arc_slut; break;
    case WS_T_NET_IN_PTR: src = t.net_in_ptr; break;
    case WS_T_NET_IN_ARC: src = t.net_in_arc; break;
    case WS_T_MEM_OUT_PTR: src = t.mem_out_ptr; break;
    case WS_T_MEM_OUT_ARC: src = t.mem_out_arc; break;
    case WS_T_NET_M: src = t.net_m; break;
    case WS_T_NET_A: src = t.net_a; break;
    case WS_T_NET_O: src = t.net_o; break;
    case WS_T_MEMBER_OF_PIN: src = t.member_of_pin; break;
    case WS_T_ROOT_NET_OF_PIN: src = t.root_net_of_pin; break;
    case WS_T_LEVEL_OF: src = t.level_of; break;
    case WS_T_LEVEL_PTR: src = t.lv_ptr; break;
    case WS_T_LEVEL_NETS: src = t.lv_nets; break;
    case WS_T_IS_ENDPOINT: {
        std::vector<uint8_t> b((size_t)n);
        WS_CUDA(cudaMemcpy(b.data(), t.is_endpoint, (size_t)n, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; i++) dst[i] = b[(size_t)i];
        return;
    }
    case WS_T_CSR_PIN_LIST:
    case WS_T_CSR_NET_INDEX: {
        int* pl = scratch_arena.alloc<int>((size_t)t.N + t.M);
        int* ni = scratch_arena.alloc<int>((size_t)t.N + 1);
        k_csr<<<blocks_for(t.N + 1), TPB, 0, ctx.s_main>>>(t.N, t.net_ptr, t.net_root, t.mem_pin,
                                                           pl, ni);
        WS_CHECK_LAUNCH();
        WS_CUDA(cudaStreamSynchronize(ctx.s_main));
        src = field == WS_T_CSR_PIN_LIST ? pl : ni;
        break;
    }
    default: throw Error(WS_ERR_VALUE, "unknown topology field");
    }
    WS_CUDA(cudaMemcpy(tmp.data(), src, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
    scratch_arena.release();
    for (int64_t i = 0; i < n; i++) dst[i] = tmp[(size_t)i];
}

}  // namespace ws
