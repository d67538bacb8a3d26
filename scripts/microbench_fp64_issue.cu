// Measurement tool (not product code): how fast does one SM sub-partition
// issue FP64 warp instructions depending on operand freshness, instruction
// type, independent chains per warp (ILP) and resident warps?  Answers the
// round-2 question behind the stage kernel's ~57 % FP64-pipe activity
// (DESIGN.md §4.2): is the ~3-cycle cross-warp FP64 issue of
// microbench_fp64.cu a register-operand (reuse cache) effect or a warp-switch
// effect, and do integer / shared-memory instructions hide in FP64 gaps?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   scripts/microbench_fp64_issue.cu -o /tmp/mb_issue ; run: /tmp/mb_issue
// Prints warp instructions per cycle per SMSP (FP64 peak 0.5) for each case.
#include <cstdio>
#include <cuda_runtime.h>

enum { OP_FMA_REUSE = 0, OP_FMA_FRESH, OP_MUL_FRESH, OP_ADD_FRESH, OP_FMA_CONST, OP_FMA_INT, OP_FMA_LDS, OP_MIX };

template <int OP, int ILP>
__global__ void kern(double *out, int iters, double a, double b, long long *cyc) {
    __shared__ double sh[1024];
    double x[ILP], y[ILP], z[ILP];
    unsigned iv[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        x[k] = threadIdx.x * 1e-9 + k;
        y[k] = 0.5 + k * 1e-3;
        z[k] = -0.25 - k * 1e-3;
        iv[k] = threadIdx.x + k;
    }
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = i;
    __syncthreads();
    unsigned sidx = threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int k = 0; k < ILP; ++k) {
                if constexpr (OP == OP_FMA_REUSE) {
                    x[k] = fma(x[k], a, b);
                } else if constexpr (OP == OP_FMA_FRESH) {
                    // three live operands, rotated: no operand repeats in a slot
                    x[k] = fma(y[k], z[k], x[k]);
                    y[k] = fma(z[k], x[k], y[k]);
                    z[k] = fma(x[k], y[k], z[k]);
                } else if constexpr (OP == OP_MUL_FRESH) {
                    x[k] = y[k] * z[k];
                    y[k] = z[k] * x[k];
                    z[k] = x[k] * y[k];
                } else if constexpr (OP == OP_ADD_FRESH) {
                    x[k] = y[k] + z[k];
                    y[k] = z[k] - x[k];
                    z[k] = x[k] + y[k];
                } else if constexpr (OP == OP_FMA_CONST) {
                    x[k] = fma(y[k], a, x[k]);
                    y[k] = fma(x[k], b, y[k]);
                    z[k] = fma(z[k], a, y[k]);
                } else if constexpr (OP == OP_FMA_INT) {
                    // one independent integer instruction per DFMA
                    x[k] = fma(y[k], z[k], x[k]);
                    iv[k] = iv[k] * 3u + 7u;
                    y[k] = fma(z[k], x[k], y[k]);
                    iv[k] = iv[k] * 5u + 1u;
                    z[k] = fma(x[k], y[k], z[k]);
                    iv[k] = iv[k] * 9u + 3u;
                } else if constexpr (OP == OP_FMA_LDS) {
                    // one shared-memory load per DFMA (its value feeds the chain later)
                    const double s0 = sh[(sidx + 32 * k) & 1023];
                    x[k] = fma(y[k], z[k], x[k]);
                    y[k] = fma(z[k], x[k], y[k]);
                    z[k] = fma(x[k], y[k], s0 + z[k]);
                    sidx += 1;
                } else {  // OP_MIX: stage-kernel-like 45 % non-FP64 (int + moves)
                    x[k] = fma(y[k], z[k], x[k]);
                    iv[k] = iv[k] * 3u + 7u;
                    y[k] = y[k] * x[k];
                    z[k] = z[k] + y[k];
                    iv[k] ^= iv[k] >> 3;
                }
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k] + y[k] + z[k] + iv[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

constexpr int fp_per_k(int op) { return op == OP_FMA_REUSE ? 1 : (op == OP_MIX ? 3 : 3); }
constexpr int all_per_k(int op) {
    return op == OP_FMA_INT ? 6 : (op == OP_MIX ? 5 : (op == OP_FMA_LDS ? 5 : fp_per_k(op)));
}
static const char *names[] = {"DFMA x=fma(x,a,b)", "DFMA 3 fresh regs", "DMUL fresh", "DADD fresh",
                              "DFMA const-bank", "DFMA + IMAD 1:1", "DFMA + LDS 3:1", "mix 3 FP64 : 2 int"};

template <int OP, int ILP>
void run(int wps, int nsm, double *out, long long *cyc, int clk_mhz) {
    const int iters = 1000;
    const int threads = 32 * 4 * wps;  // wps warps per SMSP, 1 CTA per SM
    kern<OP, ILP><<<nsm, threads>>>(out, 10, 0.999999, 1e-7, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<OP, ILP><<<nsm, threads>>>(out, iters, 0.999999, 1e-7, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double fp_warp_inst_per_smsp = (double)wps * iters * 8.0 * ILP * fp_per_k(OP);
    const double all_warp_inst_per_smsp = (double)wps * iters * 8.0 * ILP * all_per_k(OP);
    printf("%-22s ILP=%d warps/SMSP=%d: FP64 %.3f  all %.3f warp-inst/cycle/SMSP (clock64), %.3e FP64 lane-ops/s\n",
           names[OP], ILP, wps, fp_warp_inst_per_smsp / c, all_warp_inst_per_smsp / c,
           fp_warp_inst_per_smsp * 32.0 * 4.0 * nsm / (ms * 1e-3));
    (void)clk_mhz;
}

template <int OP>
void sweep(int nsm, double *out, long long *cyc, int clk) {
    for (int w : {1, 2, 3, 4}) {
        run<OP, 1>(w, nsm, out, cyc, clk);
        run<OP, 2>(w, nsm, out, cyc, clk);
        run<OP, 4>(w, nsm, out, cyc, clk);
    }
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("%s, %d SMs, clock attr %d MHz\n", p.name, p.multiProcessorCount, clk_khz / 1000);
    double *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(double) * 148 * 4096);
    cudaMalloc(&cyc, 8);
    const int nsm = p.multiProcessorCount, clk = clk_khz / 1000;
    sweep<OP_FMA_REUSE>(nsm, out, cyc, clk);
    sweep<OP_FMA_FRESH>(nsm, out, cyc, clk);
    sweep<OP_MUL_FRESH>(nsm, out, cyc, clk);
    sweep<OP_ADD_FRESH>(nsm, out, cyc, clk);
    sweep<OP_FMA_CONST>(nsm, out, cyc, clk);
    sweep<OP_FMA_INT>(nsm, out, cyc, clk);
    sweep<OP_FMA_LDS>(nsm, out, cyc, clk);
    sweep<OP_MIX>(nsm, out, cyc, clk);
    return 0;
}
