/*
 * warpstar.h — C ABI of the B200-native differentiable STA engine
 * (libwarpstar_b200.so, built from paper_2603_28381_b200/csrc/).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as opaque `void*` cudaStream_t handles, NULL = the
 * context's own stream).  Every entry point returns a status code; the text
 * of the last error is available from ws_last_error().  Status -> exception
 * mapping used by the Python layer mirrors the reference:
 *   WS_ERR_VALUE -> ValueError, WS_ERR_CYCLE -> CycleError(pin),
 *   WS_ERR_NOMEM -> MemoryError, WS_ERR_CUDA/WS_ERR_STATE -> RuntimeError.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/stasim):
 *   ws_rc_level        <- _kernels.pyx:84-156   rc_level        (backend.py:43-48)
 *   ws_forward_level   <- _kernels.pyx:159-210  forward_level   (backend.py:51-59)
 *   ws_backward_level  <- _kernels.pyx:213-249  backward_level  (backend.py:62-66)
 *   ws_create          <- flatten.py:170-316 flatten + flatten.py:44-80 levelize
 *                         (+ netlist.py:370-380 build_csr via ws_get_topology)
 *   ws_run(WS_RUN_HARD)<- warp.py:462-476 run_engine
 *   ws_run(WS_RUN_LSE) <- diff.py:164-189 forward_lse_arrival
 *   ws_run(WS_RUN_GRAD)<- diff.py:244-263 backward_tns_grad (+ _endpoint_loss 192-212)
 *   ws_run(HARD|LSE|GRAD|TWO_STREAM) <- fusion.py:435-450 execute_fused
 *   ws_summary         <- sta.py:408-421 tns / wns, GradientState.loss
 *   ws_get / ws_device_ptr <- TimingState / GradientState fields (sta.py:37-48, diff.py:61-72)
 */
#ifndef WARPSTAR_H
#define WARPSTAR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WS_ABI_VERSION 1

enum ws_status {
    WS_OK = 0,
    WS_ERR_VALUE = 1,   /* bad argument / malformed design */
    WS_ERR_CYCLE = 2,   /* combinational cycle; ws_last_error_pin() names a pin on it */
    WS_ERR_NOMEM = 3,   /* device or host allocation failed */
    WS_ERR_CUDA = 4,    /* CUDA runtime fault (incl. no device) */
    WS_ERR_STATE = 5    /* call out of order (e.g. GRAD before LSE) */
};

/* Flat ingest format (host pointers).  Orders are the reference's:
 * nets in design order, members concatenated net by net in topological
 * order; arcs cells-in-order then arcs-in-order (flatten.py:222); LUT ids
 * index a pool deduplicated in first-appearance order (flatten.py:211-244);
 * condition order ER, EF, LR, LF (netlist.py:41-45). */
typedef struct ws_design_desc {
    int64_t n_pins, n_nets, n_members, n_arcs, n_luts, n_pi, n_ep;
    int64_t lut_s_len, lut_l_len, lut_t_len;
    double clock_period;
    const int32_t *net_root;        /* [N]   root pin of each net */
    const int64_t *net_mptr;        /* [N+1] member offsets */
    const int32_t *mem_pin;         /* [M]   member pin */
    const int32_t *mem_parent_pin;  /* [M]   parent PIN (the root or an earlier member) */
    const double *mem_res;          /* [M*4] edge resistance parent->member */
    const double *mem_cap;          /* [M*4] member pin capacitance */
    const double *root_cap;         /* [N*4] */
    const int32_t *arc_from, *arc_to;    /* [A] */
    const int32_t *arc_dlut, *arc_slut;  /* [A*4] LUT ids (delay, output slew) */
    const int32_t *lut_s_ptr, *lut_l_ptr, *lut_t_ptr;  /* [n_luts+1] */
    const double *lut_s_flat, *lut_l_flat, *lut_t_flat; /* packed axes / row-major tables */
    const int32_t *pi_pin;          /* [I] */
    const double *pi_arrival, *pi_slew;  /* [I*4] */
    const int32_t *ep_pin;          /* [E] endpoint entries (duplicates allowed) */
    const double *ep_required;      /* [E*4] */
} ws_design_desc;

typedef struct ws_ctx ws_ctx;

/* per-corner value arrays (ws_set_values) */
enum ws_value_field {
    WS_V_MEM_RES = 0, WS_V_MEM_CAP = 1, WS_V_ROOT_CAP = 2, WS_V_LUT_T = 3,
    WS_V_PI_ARRIVAL = 4, WS_V_PI_SLEW = 5, WS_V_EP_REQUIRED = 6,
    /* position model (no reference counterpart: SURVEY.md §8(f) rank 1; the
     * reference's gradients stop at d_arc / d_edge, diff.py:5-7).  Setting any
     * of these enables it for every corner; until set, positions are 0, the
     * base RC is the corner's RC and the wire coefficients are 0. */
    WS_V_XY = 7,          /* [P*2] pin x, y */
    WS_V_RES0 = 8,        /* [M*4] base resistance of each member edge */
    WS_V_CAP0 = 9,        /* [M*4] base capacitance of each member edge */
    WS_V_WIRE = 10        /* [8] r_unit[4], c_unit[4]: res = res0 + r_unit*len, cap = cap0 + c_unit*len,
                             len = |dx| + |dy| between a member pin and its parent pin */
};

/* per-corner result arrays (ws_get / ws_device_ptr); float64 */
enum ws_state_field {
    WS_F_LOAD = 0, WS_F_NET_DELAY = 1, WS_F_IMPULSE = 2, WS_F_SLEW = 3, WS_F_ARRIVAL = 4,
    WS_F_REQUIRED = 5, WS_F_SLACK = 6, WS_F_ARC_DELAY = 7,             /* (P,4) / (A,4) */
    WS_F_LSE_ARRIVAL = 8, WS_F_ARC_WEIGHTS = 9, WS_F_D_ARC = 10,       /* (P,2) (A,2) (A,2) */
    WS_F_D_EDGE = 11, WS_F_ADJOINT = 12,                               /* (M,2) (P,2) */
    WS_F_SUMMARY = 13,                                                 /* (3,) TNS WNS loss */
    /* position gradients (late cols; WS_RUN_POSGRAD) */
    WS_F_D_RES = 14, WS_F_D_CAP = 15,   /* (M,2) dL/dmem_res, dL/dmem_cap */
    WS_F_D_ROOT_CAP = 16,               /* (N,2) dL/droot_cap (= dL/dload of the root) */
    WS_F_D_SLEW = 17,                   /* (P,2) dL/dslew */
    WS_F_D_LEN = 18,                    /* (M,)  dL/dlength of each member edge */
    WS_F_D_XY = 19,                     /* (P,2) dL/dx, dL/dy */
    /* batch gradients of the last WS_RUN_CORNER_SUM run (the corner argument
     * is ignored: one per context) */
    WS_F_D_ARC_SUM = 20,                /* (A,2) sum over the run's corners of d_arc */
    WS_F_D_EDGE_SUM = 21                /* (M,2) sum over the run's corners of d_edge */
};

/* topology arrays (ws_get_topology); int64 on the host like FlatDesign */
enum ws_topo_field {
    WS_T_NET_PTR = 0, WS_T_NET_ROOT, WS_T_ROOT_KIND, WS_T_MEM_PIN, WS_T_MEM_PARENT_LOC,
    WS_T_MEM_NET, WS_T_MEM_LOCAL, WS_T_ARC_FROM, WS_T_ARC_TO, WS_T_ARC_DLUT, WS_T_ARC_SLUT,
    WS_T_NET_IN_PTR, WS_T_NET_IN_ARC, WS_T_MEM_OUT_PTR, WS_T_MEM_OUT_ARC, WS_T_NET_M,
    WS_T_NET_A, WS_T_NET_O, WS_T_MEMBER_OF_PIN, WS_T_ROOT_NET_OF_PIN, WS_T_IS_ENDPOINT,
    WS_T_LEVEL_OF, WS_T_LEVEL_PTR, WS_T_LEVEL_NETS, WS_T_CSR_PIN_LIST, WS_T_CSR_NET_INDEX,
    WS_T_COUNT
};

/* dims returned by ws_dims: P N M A I E L n_luts n_corners max_in max_m */
enum { WS_DIMS_LEN = 11 };

/* ws_run flags */
enum ws_run_flags {
    WS_RUN_HARD = 1u,        /* init + RC + forward + backward + slack + TNS/WNS  (run_engine) */
    WS_RUN_LSE = 2u,         /* LSE smooth forward (needs the hard forward)        */
    WS_RUN_GRAD = 4u,        /* endpoint loss + reverse adjoint (needs LSE)        */
    WS_RUN_TWO_STREAM = 8u,  /* LSE/GRAD on the grad stream, event-gated every granularity levels */
    WS_RUN_FUSED = 16u,      /* single stream, forward+LSE and backward+grad fused per level */
    WS_RUN_GRAPH = 32u,      /* capture the pass into a CUDA graph once, replay afterwards */
    WS_RUN_SUMMARY = 64u,    /* TNS/WNS (sta.py:408-421) from the corner's current slack */
    WS_RUN_SLACK = 128u,     /* slack (warp.py:474-475) from the current arrival/required */
    WS_RUN_PERSISTENT = 256u,/* with HARD (and LSE|GRAD): the whole pass as one cooperative
                                kernel, grid barrier between levels */
    WS_RUN_WIRE = 512u,      /* first: mem_res / mem_cap from the positions (WS_V_XY ...) */
    WS_RUN_POSGRAD = 1024u,  /* last (needs HARD|LSE|GRAD in the same call): slew / load
                                adjoint sweep, Elmore adjoint, dL/dxy */
    WS_RUN_TIMED = 2048u,    /* sequential or fused mode, no graph: a CUDA event after every
                                launch, read back with ws_kernel_times (measured costs) */
    WS_RUN_CORNER_SUM = 4096u /* with GRAD, n_corners <= 16: also sum_k d_arc and sum_k d_edge
                                over the run's corners (WS_F_D_ARC_SUM / WS_F_D_EDGE_SUM), the
                                gradient of the batch objective sum_k loss_k */
};

enum ws_loss_kind { WS_LOSS_HINGE = 0, WS_LOSS_SOFTPLUS = 1 };

int ws_abi_version(void);
const char *ws_last_error(void);
int64_t ws_last_error_pin(void);

/* Upload a design, build the FlatDesign arrays and the level schedule on the
 * device; values of every corner start as the design's own. */
int ws_create(const ws_design_desc *d, int n_corners, ws_ctx **out);
void ws_destroy(ws_ctx *ctx);
int ws_dims(ws_ctx *ctx, int64_t *dims /* WS_DIMS_LEN */);
int64_t ws_topology_len(ws_ctx *ctx, int field);
int ws_get_topology(ws_ctx *ctx, int field, int64_t *dst /* host */);

/* Replace one value array of one corner (src host or device pointer). */
int ws_set_values(ws_ctx *ctx, int corner, int field, const double *src, int src_on_device,
                  void *stream);
/* Scale-perturb values on the device: x *= 1 + sigma * clip(N(0,1), +-3) per
 * element of mem_res, mem_cap and root_cap of `corner`, counter-based RNG
 * keyed by seed (BASELINE.md §2 C4 placement-loop stand-in). base_corner
 * supplies the unperturbed values. */
int ws_perturb_values(ws_ctx *ctx, int corner, int base_corner, uint64_t seed, double sigma,
                      void *stream);

int ws_run(ws_ctx *ctx, int corner0, int n_corners, uint32_t flags, double gamma,
           int loss_kind, int reduce_width, int granularity, void *stream, void *stream_grad);

/* One kernel of the fusion pipeline's graph (fusion.py:113-160), launched
 * alone on `stream`: kind 0 net_rc, 1 cell_delay_at, 2 slack_bwd, 3 lse_fwd,
 * 4 grad_bwd at `level`; 5 finish (free-pin / PI-root adjoints, TNS / WNS /
 * loss; level ignored).  The caller owns the ordering — the Python
 * PipelineRun checks each kernel's dependencies before launching it and
 * raises FusionError on a violation (replaces fusion.py:307-312). */
int ws_run_kernel(ws_ctx *ctx, int corner, int kind, int level, double gamma, int loss_kind,
                  int reduce_width, void *stream);

/* Overwrite a result array of one corner (e.g. a caller-supplied TimingState
 * handed to forward_lse_arrival). */
int ws_set_state(ws_ctx *ctx, int corner, int field, const double *src, int src_on_device,
                 void *stream);
int ws_get(ws_ctx *ctx, int corner, int field, double *dst, int dst_on_device, void *stream);
int ws_device_ptr(ws_ctx *ctx, int corner, int field, void **dptr, int64_t *n_elems);
int ws_value_ptr(ws_ctx *ctx, int corner, int field, void **dptr, int64_t *n_elems);
/* out[0]=TNS out[1]=WNS out[2]=loss (synchronizes the stream) */
int ws_summary(ws_ctx *ctx, int corner, double *out, void *stream);
/* Profiling hook: device buffer receiving per-block phase timestamps in
 * builds compiled with -DWS_PROBE (a no-op otherwise); NULL disables. */
int ws_set_probe(ws_ctx *ctx, void *device_buf);
/* number of kernels launched by the last ws_run */
int ws_last_launch_count(ws_ctx *ctx);
/* Per-launch device times of the last WS_RUN_TIMED run (synchronizes):
 * kind[i] in {0 net_rc, 1 cell_delay_at, 2 slack_bwd, 3 lse_fwd, 4 grad_bwd,
 * 5 other} and level[i] as in fusion.py:113-160 build_kernel_graph, ms[i] the
 * time since the previous mark.  Returns the number of entries (<= cap), or
 * -1 on error.  Feeds fusion.measured_kernel_costs -> schedule_fused
 * (fusion.py:216-249), the makespan model the reference simulates. */
int ws_kernel_times(ws_ctx *ctx, int *kind, int *level, float *ms, int cap);

/* Legacy per-level shims with the reference's raw kernel semantics
 * (int64 indices, float64 values, host buffers, outputs updated in place). */
int ws_rc_level(int64_t n_lv, const int64_t *nets, int64_t n_nets, const int64_t *net_ptr,
                const int64_t *net_root, const double *root_cap, int64_t n_mem,
                const int64_t *mem_pin, const int64_t *mem_parent_loc, const double *mem_res,
                const double *mem_cap, int64_t n_pins, const int64_t *root_net_of_pin,
                double *load, double *net_delay, double *impulse, int reduce_width);
int ws_forward_level(int64_t n_lv, const int64_t *nets, int64_t n_nets, const int64_t *net_ptr,
                     const int64_t *net_root, const int64_t *root_kind, int64_t n_mem,
                     const int64_t *mem_pin, const int64_t *net_in_ptr, const int64_t *net_in_arc,
                     int64_t n_arcs, const int64_t *arc_from, const int64_t *arc_dlut,
                     const int64_t *arc_slut, int64_t n_luts, const int64_t *lut_s_ptr,
                     const int64_t *lut_l_ptr, const int64_t *lut_t_ptr, const double *lut_s_flat,
                     const double *lut_l_flat, const double *lut_t_flat, int64_t n_pins,
                     const double *load, const double *net_delay, const double *impulse,
                     double *slew, double *arrival, double *arc_delay);
int ws_backward_level(int64_t n_lv, const int64_t *nets, int64_t n_nets, const int64_t *net_ptr,
                      const int64_t *net_root, int64_t n_mem, const int64_t *mem_pin,
                      const int64_t *mem_out_ptr, const int64_t *mem_out_arc, int64_t n_arcs,
                      const int64_t *arc_to, int64_t n_pins, const double *net_delay,
                      double *required, const double *arc_delay);

#ifdef __cplusplus
}
#endif
#endif /* WARPSTAR_H */
