// Cost of the NLDM arc interpolation (locate + blend) on B200 (profiling aid).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I../../paper_2603_28381_b200/csrc interp_micro.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ws_common.cuh"
using namespace ws;

// variant 1: the production locate
__device__ __forceinline__ Loc loc_v1(const double* ax, int n, double q) { return lut_locate(ax, n, q); }

// variant 2: branchless fixed-trip binary search (n <= 8)
__device__ __forceinline__ Loc loc_v2(const double* ax, int n, double q)
{
    Loc r;
    if (n > 1) {
        int lo = 0;
        // upper_bound over n entries: count of ax[k] <= q, via a fixed 3-step search for n <= 8
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) cnt += (k < n && ax[k] <= q) ? 1 : 0;
        lo = cnt;
        int i = lo - 1;
        i = i < 0 ? 0 : (i > n - 2 ? n - 2 : i);
        double t = (q - ax[i]) / (ax[i + 1] - ax[i]);
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
        r.i0 = i; r.i1 = i + 1; r.f = t;
    } else { r.i0 = 0; r.i1 = 0; r.f = 0.0; }
    return r;
}

template <int V>
__global__ void k(const double* gs, const double* gl, const double* gt, const double* q, double* out,
                  int reps, long long* cyc)
{
    __shared__ double s[5], l[5], tab[32 * 25];
    if (threadIdx.x < 5) { s[threadIdx.x] = gs[threadIdx.x]; l[threadIdx.x] = gl[threadIdx.x]; }
    for (int i = threadIdx.x; i < 800; i += blockDim.x) tab[i] = gt[i];
    __syncthreads();
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    double qs0 = q[(gid * 4) & 4095], ql0 = q[(gid * 4 + 1) & 4095];
    double qs1 = q[(gid * 4 + 2) & 4095], ql1 = q[(gid * 4 + 3) & 4095];
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        const int lut0 = (gid + r) & 31, lut1 = (gid + 7 * r) & 31;
        Loc a, b, c, d;
        if (V == 1) { a = loc_v1(s, 5, qs0); b = loc_v1(l, 5, ql0); c = loc_v1(s, 5, qs1); d = loc_v1(l, 5, ql1); }
        else { a = loc_v2(s, 5, qs0); b = loc_v2(l, 5, ql0); c = loc_v2(s, 5, qs1); d = loc_v2(l, 5, ql1); }
        const double d0 = lut_blend(tab + lut0 * 25, 5, a, b), s0 = lut_blend(tab + (lut0 ^ 1) * 25, 5, a, b);
        const double d1 = lut_blend(tab + lut1 * 25, 5, c, d), s1 = lut_blend(tab + (lut1 ^ 1) * 25, 5, c, d);
        acc += d0 + s0 + d1 + s1;
        qs0 += 1e-13; ql0 += 1e-16; qs1 += 1e-13; ql1 += 1e-16;
    }
    long long t1 = clock64();
    out[gid] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main()
{
    double hs[5], hl[5], ht[800], hq[4096];
    for (int i = 0; i < 5; i++) { hs[i] = 1e-12 * pow(200.0, i / 4.0); hl[i] = 5e-16 * pow(600.0, i / 4.0); }
    for (int i = 0; i < 800; i++) ht[i] = 1e-11 * (1 + (i % 37) * 0.01);
    for (int i = 0; i < 4096; i++) hq[i] = (i & 1) ? 1e-15 * (1 + (i % 97)) : 1e-12 * (1 + (i % 89));
    double *ds, *dl, *dt, *dq, *out;
    long long* cyc;
    cudaMalloc(&ds, 40); cudaMalloc(&dl, 40); cudaMalloc(&dt, 6400); cudaMalloc(&dq, 32768);
    cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
    cudaMemcpy(ds, hs, 40, cudaMemcpyHostToDevice); cudaMemcpy(dl, hl, 40, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, ht, 6400, cudaMemcpyHostToDevice); cudaMemcpy(dq, hq, 32768, cudaMemcpyHostToDevice);
    const int reps = 100;
    for (int v = 1; v <= 2; v++)
        for (int cfg = 0; cfg < 3; cfg++) {
            const int blocks = cfg == 0 ? 1 : 148 * (cfg == 1 ? 2 : 4), threads = cfg == 0 ? 32 : 256;
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            auto go = [&] { if (v == 1) k<1><<<blocks, threads>>>(ds, dl, dt, dq, out, reps, cyc); else k<2><<<blocks, threads>>>(ds, dl, dt, dq, out, reps, cyc); };
            go(); cudaEventRecord(e0); go(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("v%d %-14s: %7.1f cycles per 2-item arc step (4 locates + 4 blends), kernel %7.2f us -> %6.2f us per step\n",
                   v, cfg == 0 ? "1 warp" : (cfg == 1 ? "2 blk/SM x256" : "4 blk/SM x256"), (double)c / reps, ms * 1e3, ms * 1e3 / reps);
        }
    return 0;
}
