// Host-side internals shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "ws_common.cuh"
#include "../../include/warpstar.h"

namespace ws {

struct Error : std::runtime_error {
    int code;
    int64_t pin;
    Error(int c, const std::string& m, int64_t p = -1) : std::runtime_error(m), code(c), pin(p) {}
};

#define WS_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) {                                                          \
            if (_e == cudaErrorMemoryAllocation)                                          \
                throw ::ws::Error(WS_ERR_NOMEM, std::string("cuda: out of device memory at ") + #call); \
            throw ::ws::Error(WS_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(_e) + \
                                                " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
        }                                                                                 \
    } while (0)

#define WS_CHECK_LAUNCH() WS_CUDA(cudaGetLastError())

// Tracked device allocations (freed with the context).
struct Arena {
    std::vector<void*> ptrs;
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        if (n < 16) n = 16;   // empty designs still get valid (tiny) buffers
        WS_CUDA(cudaMalloc(&p, n * sizeof(T)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    void release() {
        for (void* p : ptrs) cudaFree(p);
        ptrs.clear();
    }
};

// Reusable scratch (CUB temp storage etc.).
struct Scratch {
    void* p = nullptr;
    size_t n = 0;
    void* get(size_t want) {
        if (want > n) {
            if (p) cudaFree(p);
            p = nullptr;
            WS_CUDA(cudaMalloc(&p, want));
            n = want;
        }
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// numpy pairwise-sum tree over the 2E endpoint terms (ws_sta.cu)
struct SumPlan {
    int n = 0, n_leaves = 0, n_inner = 0;
    int *leaf_off = nullptr, *leaf_len = nullptr;     // device
    int *in_left = nullptr, *in_right = nullptr;      // device, children node ids
    std::vector<int> height_ptr;                      // inner nodes grouped by height
    int* d_height_ptr = nullptr;
    int max_height = 0;
};

// position model (ws_place.cu): topology extras, built on first use
struct PlaceTopo {
    int* parent_pin = nullptr;   // [M] parent pin of each member edge
    int* pc_ptr = nullptr;       // [P+1] member edges whose parent is the pin
    int* pc_mem = nullptr;       // [M]   (ascending member index)
    int* tm_f = nullptr;         // [M] task-order member slot -> original member index
    int* tm_root = nullptr;      // [M] task-order member slot -> root pin of its net
    std::vector<int> tq_mptr_host;   // [N+1] first task-order member slot of level position q
    bool ready = false;
};

// per corner: positions, wire model, gradients (late cols) and scratch
struct PlaceCorner {
    double* xy = nullptr;        // (P,2) pin coordinates
    double *res0 = nullptr, *cap0 = nullptr;   // (M,4) base RC of each member edge
    double* wire = nullptr;      // [8] r_unit[4], c_unit[4]
    double *gs = nullptr, *gsr = nullptr;      // (P,2) dL/dslew, feedthrough-root partials
    double* gsa = nullptr;       // (A,2) slew adjoint an arc sends to its source pin
    double* gl = nullptr;        // (N,2) dL/dload[root]
    double *d_res = nullptr, *d_cap = nullptr; // (M,2)
    double* d_root_cap = nullptr;  // (N,2)
    double* g_len = nullptr;     // (M)   dL/dlength
    double* d_xy = nullptr;      // (P,2)
    double *sc_gimp = nullptr, *sc_buf = nullptr, *sc_acc = nullptr;   // (M,2) scratch
    double* sc_t = nullptr;      // (M,2) root-slew terms of the members
};

// one corner's engine + placement pointers, read by the batched sweep kernels
// (blockIdx.y = corner)
struct PgArgs {
    Corner d;
    PlaceCorner g;
};

// read-only device view of the sweep's topology extras (PlaceTopo minus the
// host vector) and the per-corner {engine, placement} pointer table
struct PgDev {
    const int* tm_f;      // [M] task-order member slot -> original member index
    const int* tm_root;   // [M] task-order member slot -> root pin of its net
    const PgArgs* pa;     // per corner of the launch (blockIdx.y)
};

struct CornerSlot {
    Corner d;                  // device pointers
    bool has_lse = false;      // LSE forward done since the last hard pass
};

constexpr size_t kGraphCache = 16;   // CUDA-graph executables kept per context

struct Context {
    Topo t{};
    CornerStrides cstride{};          // corner k's field = corner 0's + k * stride
    double *dsum_arc = nullptr, *dsum_edge = nullptr;   // WS_RUN_CORNER_SUM outputs (A,2) (M,2)
    Arena topo_mem;
    Arena val_mem;
    Scratch scratch;
    std::vector<CornerSlot> corners;
    Corner* d_corners = nullptr;      // device copy of every corner's pointers
    double clock_period = 0.0;
    int lut_t_len = 0, lut_s_len = 0, lut_l_len = 0;
    std::vector<int> lv_ptr_host;     // L+1
    std::vector<int> lv_maxm_host;    // per level: max member count
    std::vector<int> lv_tree_host;     // per level: any tree net
    bool any_tree = false;             // any net with a non-root parent (k_rc_tree needed)
    std::vector<int> lvt_ptr_host;    // per level: first task (L+1)
    cudaStream_t s_main = nullptr, s_grad = nullptr;
    std::vector<cudaEvent_t> events;
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr, ev_g1 = nullptr;
    float last_ms_sta = 0.f, last_ms_total = 0.f;
    SumPlan* tns_plan = nullptr;      // over 2E slack terms
    int launches_last_run = 0;
    bool lut_global = false;
    int* rc_bnet = nullptr;      // per streaming-RC member block b (+1): first net whose members start at or after b * RC_MPB (k_rc_flat<true>; kept out of Topo so the level kernels' parameters stay put)
    int split_parts = 2;         // WS_SPLIT_PARTS: streams a split batch runs on (parts of >= 4 corners)
    std::vector<cudaStream_t> split_streams;   // the parts beyond s_main / s_grad
    int split_min = 8;           // WS_SPLIT=n: fused corner batches of >= n corners run as two half batches on two streams (0: never)
    int rc_roots = 0;            // WS_RC_ROOTS: star-net root loads in net blocks (net, -1) / member blocks (fold, 1) / by batch size (0)
    bool rc_pin_order = false;   // WS_RC_SCHEME=pin: the pin-order streaming RC
    bool rc_cte = false;       // WS_RC_SCHEME=cte: the paper's CTE-scheme RC kernel (ablation)   // WS_LUT_GLOBAL=1: read the LUT pool through L1 instead of staging it
    // CUDA graph cache: key -> exec
    struct GraphEntry { unsigned key; int c0, nc; double gamma; int loss; int gran; cudaGraphExec_t exec; };
    std::vector<GraphEntry> graphs;
    std::vector<int> graph_launches;  // kernels per captured graph
    PlaceTopo pt;
    std::vector<PlaceCorner> place;   // per corner once place_enable ran
    PgArgs* pg_args = nullptr;        // device copy of {corner, place} per corner
    std::vector<cudaEvent_t> pg_events;   // [L + 2]: per backward level, fork, join
    // WS_RUN_TIMED: an event after every launch of a sequential pass, tagged
    // with the reference's kernel kind and level (fusion.py:113-160)
    std::vector<cudaEvent_t> timed_events;
    std::vector<int> timed_kind, timed_level;
    int timed_n = 0;
};

void build_topology(Context& ctx, const ws_design_desc* d);
void alloc_corners(Context& ctx, int n);
void upload_values(Context& ctx, int corner, const ws_design_desc* d);
void run_pass(Context& ctx, int c0, int nc, unsigned flags, double gamma, int loss_kind,
              int granularity, cudaStream_t s, cudaStream_t g, int w);
void run_kernel(Context& ctx, int c0, int kind, int level, double g, int loss_kind, int w,
                cudaStream_t s);
// level-list launches for the legacy per-level shims
void launch_rc_list(const Topo& t, const Corner* dcs, const int* list, int n, int w, cudaStream_t s);
void launch_fwd_list(const Topo& t, const Corner* dcs, int n, int lut_s_len, int lut_l_len,
                     int lut_t_len, cudaStream_t s);
void launch_bwd_list(const Topo& t, const Corner* dcs, int n, cudaStream_t s);
void launch_perturb(const Context& ctx, int dst, int src, unsigned long long seed, double sigma,
                    cudaStream_t s);
void place_enable(Context& ctx);
int launch_wire(Context& ctx, int c0, int nc, cudaStream_t s);
// position-gradient sweep; with `bwd_done` (one event per level, recorded
// after that level's backward kernel on the pass stream) it runs on stream
// `gs` and level l starts as soon as the pass's backward level l is done
int launch_posgrad(Context& ctx, int c0, int nc, cudaStream_t s, cudaStream_t gs = nullptr,
                   const std::vector<cudaEvent_t>* bwd_done = nullptr);
// the fused mode's pieces of the sweep: gsa / gsr reset before the backward
// levels (which run the per-level sweep inside k_bwd), then dL/dlength and
// dL/dxy after them
PgDev pg_dev(const Context& ctx, int c0);
void posgrad_reset(Context& ctx, int c0, int nc, cudaStream_t s);
int launch_posgrad_tail(Context& ctx, int c0, int nc, cudaStream_t s, bool pdl);
void summary_plan_init(Context& ctx);
void summary_plan_free(Context& ctx);
void topo_field_to_host(Context& ctx, int field, int64_t* dst);
int64_t topo_field_len(Context& ctx, int field);

}  // namespace ws
