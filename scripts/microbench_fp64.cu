// Measurement tool (not product code): FP64 pipe latency and throughput on
// the local GPU.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   scripts/microbench_fp64.cu -o /tmp/mb_fp64 ; run: /tmp/mb_fp64
// Prints, for DFMA / DMUL chains with ILP independent chains per thread and
// W warps per SM: achieved FP64 instructions per second (lane-ops) and the
// single-warp dependent latency in cycles.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_chain(double *out, int iters, double a, double b, long long *cyc) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-9 + k;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void run(int warps_per_sm, int nsm, double *out, long long *cyc) {
    const int iters = 2000;
    const int threads = 32 * warps_per_sm;
    dfma_chain<ILP><<<nsm, threads>>>(out, 10, 0.999999, 1e-7, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_chain<ILP><<<nsm, threads>>>(out, iters, 0.999999, 1e-7, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double lane_ops = (double)nsm * threads * iters * 16.0 * ILP;
    const double per_dep = (double)c / (iters * 16.0);
    printf("ILP=%d warps/SM=%2d: %.3e DFMA lane-ops/s  (%.1f%% of 148x64xf), cycles per dependent step %.2f\n", ILP,
           warps_per_sm, lane_ops / (ms * 1e-3), 0.0, per_dep);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("%s, %d SMs, clock attr %d MHz\n", p.name, p.multiProcessorCount, clk_khz / 1000);
    double *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(double) * 148 * 2048);
    cudaMalloc(&cyc, 8);
    const int nsm = p.multiProcessorCount;
    for (int w : {1, 4, 8, 16, 32}) {
        run<1>(w, nsm, out, cyc);
        run<2>(w, nsm, out, cyc);
        run<4>(w, nsm, out, cyc);
        run<8>(w, nsm, out, cyc);
    }
    return 0;
}
