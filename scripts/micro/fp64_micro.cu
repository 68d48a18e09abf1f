// FP64 latency / throughput micro-benchmarks on the B200 (profiling aid).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false fp64_micro.cu -o fp64_micro
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double a, double b, int iters, long long* cyc)
{
    double x = a + threadIdx.x * 1e-9, y = b;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (OP == 0) x = __dadd_rn(x, y);
        else if (OP == 1) x = __dmul_rn(x, 1.0000001);
        else if (OP == 2) x = __ddiv_rn(x, y) + 1.0;
        else if (OP == 3) x = exp(x * 1e-3) + 0.5;
        else if (OP == 4) x = log(x) + 2.0;
        else if (OP == 5) x = __dsqrt_rn(x) + 1.0;
        else if (OP == 6) x = __fma_rn(x, y, 0.5);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main()
{
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 26);
    cudaMalloc(&cyc, 1 << 20);
    const char* names[] = {"dadd", "dmul", "ddiv", "exp", "log", "dsqrt", "dfma"};
    const int iters = 1000;
    for (int op = 0; op < 7; op++) {
        for (int cfg = 0; cfg < 2; cfg++) {
            const int blocks = cfg == 0 ? 1 : 148 * 4, threads = cfg == 0 ? 32 : 256;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto launch = [&] {
                switch (op) {
                case 0: chain<0><<<blocks, threads>>>(out, 1.5, 1e-9, iters, cyc); break;
                case 1: chain<1><<<blocks, threads>>>(out, 1.5, 1e-9, iters, cyc); break;
                case 2: chain<2><<<blocks, threads>>>(out, 1.5, 1.7, iters, cyc); break;
                case 3: chain<3><<<blocks, threads>>>(out, 1.5, 1.7, iters, cyc); break;
                case 4: chain<4><<<blocks, threads>>>(out, 1.5, 1.7, iters, cyc); break;
                case 5: chain<5><<<blocks, threads>>>(out, 1.5, 1.7, iters, cyc); break;
                case 6: chain<6><<<blocks, threads>>>(out, 1.5, 0.5, iters, cyc); break;
                }
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double per_op_ns = ms * 1e6 / iters;
            const double ops = (double)blocks * threads * iters;
            printf("%-6s %s: %7.1f cycles/op/thread (latency chain), %8.2f Gop/s, %7.3f us total\n",
                   names[op], cfg == 0 ? "1 warp      " : "148x4x256thr", (double)c / iters,
                   ops / (ms * 1e-3) / 1e9, ms * 1e3);
            (void)per_op_ns;
        }
    }
    return 0;
}
