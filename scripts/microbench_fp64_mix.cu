// Measurement tool (not product code): do non-FP64 instructions (uniform
// datapath, vector integer, moves, shared-memory loads) issue "for free" in
// the gaps of an FP64 stream whose cost is set by 64-bit register-operand
// reads (microbench_fp64_issue.cu: DFMA with 3 fresh register operands = 3
// cycles, DMUL = 2, DFMA with a constant-bank operand = 2)?  And does a
// register named twice in one instruction count twice?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/microbench_fp64_mix.cu -o /tmp/mb_mix
#include <cstdio>
#include <cuda_runtime.h>

enum { BASE = 0, UNIF, VINT, VINT1, LDS1, DUPREG, ABSADD, MOVIMM, SHFL1, SEL2 , NCASE};
static const char *names[] = {"DFMA 3 fresh (base)", "+1 uniform op / DFMA", "+1 IADD3 (2 reg) / DFMA",
                              "+1 IADD3 (1 reg) / DFMA", "+1 LDS.64 / DFMA", "DFMA Ra,Ra,Rb (dup)",
                              "DADD Ra,|Ra| (dup)", "+1 MOV imm / DFMA", "+1 SHFL / DFMA", "+2 FSEL / DFMA"};

template <int C>
__global__ void kern(double *out, int iters, long long *cyc, int ub) {
    __shared__ double sh[1024 * 5];
    constexpr int ILP = 4;
    double x[ILP], y[ILP], z[ILP];
    unsigned iv[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        x[k] = threadIdx.x * 1e-9 + k;
        y[k] = 0.5 + k * 1e-3;
        z[k] = -0.25 - k * 1e-3;
        iv[k] = threadIdx.x * 7 + k;
    }
    for (int i = threadIdx.x; i < 5120; i += blockDim.x) sh[i] = i;
    __syncthreads();
    unsigned u = ub;
    unsigned sa = (unsigned)__cvta_generic_to_shared(sh) + (threadIdx.x & 31) * 8;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int k = 0; k < ILP; ++k) {
                if constexpr (C == DUPREG) {
                    x[k] = fma(y[k], y[k], x[k]);
                    y[k] = fma(z[k], z[k], y[k]);
                    z[k] = fma(x[k], x[k], z[k]);
                } else if constexpr (C == ABSADD) {
                    x[k] = fma(y[k], z[k], x[k]);
                    asm("add.f64 %0, %0, %1;" : "+d"(y[k]) : "d"(fabs(x[k])));  // DADD y, y, |x|
                    asm("{.reg .f64 t; abs.f64 t, %1; add.f64 %0, %1, t;}" : "=d"(z[k]) : "d"(y[k]));  // DADD z, y, |y|
                } else {
                    x[k] = fma(y[k], z[k], x[k]);
                    y[k] = fma(z[k], x[k], y[k]);
                    z[k] = fma(x[k], y[k], z[k]);
                }
                if constexpr (C == UNIF) {
                    asm volatile("{.reg .u32 t; mul.lo.u32 t, %0, 3; add.u32 %0, t, %1;}" : "+r"(u) : "r"(it));
                    asm volatile("xor.b32 %0, %0, %1;" : "+r"(u) : "r"(r * 5 + k));
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(u) : "r"(it));
                } else if constexpr (C == VINT) {
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(iv[k]) : "r"(iv[(k + 1) % ILP]));
                    asm volatile("xor.b32 %0, %0, %1;" : "+r"(iv[k]) : "r"(iv[(k + 2) % ILP]));
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(iv[k]) : "r"(iv[(k + 3) % ILP]));
                } else if constexpr (C == VINT1) {
                    asm volatile("add.u32 %0, %0, 7;" : "+r"(iv[k]));
                    asm volatile("xor.b32 %0, %0, 5;" : "+r"(iv[k]));
                    asm volatile("add.u32 %0, %0, 3;" : "+r"(iv[k]));
                } else if constexpr (C == LDS1) {
                    unsigned a0, a1, a2, h0, h1, h2;
                    const unsigned ad = sa + ((it * 8 + r) & 7) * 64 + k * 256;
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a0), "=r"(h0) : "r"(ad));
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a1), "=r"(h1) : "r"(ad + 2048));
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a2), "=r"(h2) : "r"(ad + 4096));
                    iv[k] ^= a0 ^ a1 ^ a2;
                } else if constexpr (C == MOVIMM) {
                    unsigned t0, t1, t2;
                    asm volatile("mov.u32 %0, 12345;" : "=r"(t0));
                    asm volatile("mov.u32 %0, 54321;" : "=r"(t1));
                    asm volatile("mov.u32 %0, 999;" : "=r"(t2));
                    iv[k] += (r == 7) ? (t0 ^ t1 ^ t2) : 0u;
                } else if constexpr (C == SHFL1) {
                    iv[k] = __shfl_xor_sync(0xffffffffu, iv[k], 1);
                    iv[k] = __shfl_xor_sync(0xffffffffu, iv[k], 2);
                    iv[k] = __shfl_xor_sync(0xffffffffu, iv[k], 4);
                } else if constexpr (C == SEL2) {
                    double s;
                    asm volatile("{.reg .pred p; setp.lt.u32 p, %1, 1000; selp.f64 %0, %2, %3, p;}" : "=d"(s) : "r"(iv[k]), "d"(x[k]), "d"(y[k]));
                    asm volatile("{.reg .pred p; setp.lt.u32 p, %1, 1000; selp.f64 %0, %2, %3, p;}" : "=d"(s) : "r"(iv[k]), "d"(s), "d"(z[k]));
                    asm volatile("{.reg .pred p; setp.lt.u32 p, %1, 1000; selp.f64 %0, %2, %3, p;}" : "=d"(s) : "r"(iv[k]), "d"(s), "d"(x[k]));
                    iv[k] += __double2loint(s) & (r == 7 ? 1 : 0);
                }
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k] + y[k] + z[k] + iv[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + u;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int wps, int nsm, double *out, long long *cyc) {
    const int iters = 1000, threads = 128 * wps;
    kern<C><<<nsm, threads>>>(out, 10, cyc, 1);
    kern<C><<<nsm, threads>>>(out, iters, cyc, 1);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double groups = (double)wps * iters * 8.0 * 4;  // (k, r) groups per SMSP: 3 FP64 + 3 extra each
    printf("%-26s warps/SMSP=%d: %.2f cycles per group of 3 FP64 (+3 others)\n", names[C], wps, c / groups);
}
template <int C>
void sweep(int nsm, double *out, long long *cyc) {
    for (int w : {1, 2, 3}) run<C>(w, nsm, out, cyc);
}
int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(double) * 148 * 4096);
    cudaMalloc(&cyc, 8);
    const int nsm = p.multiProcessorCount;
    sweep<BASE>(nsm, out, cyc);
    sweep<UNIF>(nsm, out, cyc);
    sweep<VINT>(nsm, out, cyc);
    sweep<VINT1>(nsm, out, cyc);
    sweep<LDS1>(nsm, out, cyc);
    sweep<DUPREG>(nsm, out, cyc);
    sweep<ABSADD>(nsm, out, cyc);
    sweep<MOVIMM>(nsm, out, cyc);
    sweep<SHFL1>(nsm, out, cyc);
    sweep<SEL2>(nsm, out, cyc);
    return 0;
}
