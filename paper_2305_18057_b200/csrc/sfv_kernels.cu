// sfv_kernels.cu -- sm_100a kernels of the SENSEI finite-volume hot path.
//
// The stage kernel fuses, for one explicit RK stage (Eq. 6)
// over one block: limiter + MUSCL extrapolation (Eq. 7),
// the Roe/Harten face flux (Eq. 2 normal flux; readings
// A-R1, A-R2), the flux-difference residual (Eq. 5), the
// stage update, the physical-boundary ghost writes of the new state
// (PAPER.md:138-139), the residual-norm partials ("residual print",
// PAPER.md:120) and the CFL reduction for the next step (reading A-R6).
//
// Design: every CTA is one independent warp that owns a
// strip of 32*CPL-2 contiguous j columns (+1 halo column each side) and
// marches along i over a segment of rows.  Each row (state, metrics,
// pointwise RK inputs) is staged into small per-warp shared-memory rings by
// 2D TMA tensor copies (cp.async.bulk.tensor.2d, mbarrier complete_tx),
// issued by the whole warp via elect.sync, at least one row ahead of use.
// Along i every lane keeps its column's stencil window in registers, so each
// i-face flux is evaluated once and carried to the next row; along j the
// face states and fluxes move between neighbouring lanes through shared
// memory, so each j-face is evaluated once too.  Each limiter value Psi is
// computed once per cell, direction and component (the paper's §5
// de-duplication), on chip.  No CTA-wide barrier in the main
// loop; kernels chain with programmatic dependent launch.
//
// Template variants: PEER -- the edge tasks also store their edge layers
// into the neighbour block's ghost frame and signal / wait on per-edge flags
// (device-initiated halo exchange); VISC -- the Navier-Stokes
// mode subtracts the viscous residual formed by gradvisc_kernel /
// grad_kernel + visc_kernel (further below).
#include "sfv_internal.h"

#include <cstdio>
#include <cstdlib>
#include <algorithm>

namespace sfv {

// --------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// 32-bit shared-window address variants (addresses precomputed once per warp)
__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "SFV_WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SFV_WAITS_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void elect_issue_s(unsigned dst, const CUtensorMap *map, int x, int y, unsigned bar,
                                              unsigned bytes) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %5;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        "\n\t}" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void elect_tma_s(unsigned dst, const CUtensorMap *map, int x, int y, unsigned bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        "\n\t}" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// Programmatic dependent launch (PDL): let the next grid be scheduled, and
// wait for the previous grid's completion + memory visibility.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------ device-initiated halo exchange
// System-scope acquire / release on flags that a peer GPU writes over
// NVLink (or another block of this process in loopback peer mode).
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#ifndef SFV_TIMELINE
#define SFV_TIMELINE 0  // diagnostic build: per-task globaltimer stamps of the stage kernel (scripts/timeline.py)
#endif
#if SFV_TIMELINE
// [stage slot 0..7][task][10]: entry, after griddepcontrol.wait, first flux data ready, loop end,
// smid | warpid << 16, rows, stamps at rows i_start+4, +8, +12, +16 (first segment)
__device__ unsigned long long g_timeline[8][8192][10];
#endif
constexpr unsigned long long HALO_TIMEOUT_NS = 20ull * 1000 * 1000 * 1000;
// Wait (all lanes) until the neighbour has published stage sequence >= need
// for this edge, then make its data visible to the async (TMA) proxy.  A
// neighbour that never signals sets the sticky halo error after
// HALO_TIMEOUT_NS instead of hanging the device; later waits then return at
// once (the step's results are invalid and sfv_sync reports SFV_ERR_HALO).
__device__ __forceinline__ void wait_flag(const unsigned long long *f, unsigned long long need, unsigned *herr) {
    if (ld_acquire_sys(f) < need) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys(f) < need) {
            if (*(volatile unsigned *)herr) break;
            if (globaltimer_ns() - t0 > HALO_TIMEOUT_NS) {
                atomicExch(herr, 1u);
                break;
            }
            __nanosleep(100);
        }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Fast reciprocal / reciprocal square root: MUFU seed + one cubic-convergent
// correction (relative error ~ seed^3 << 2^-53, i.e. within ~1 ulp).
__device__ __forceinline__ double frcp(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    return fma(y, fma(e, e, e), y);
}
#ifndef SFV_DIET
#define SFV_DIET 0  // FP64 diet v2: limiter max-form, rho tests folded into a~^2 > 0, |x| by a sign-bit mask
#endif
#ifndef SFV_WALL_FIRST
#define SFV_WALL_FIRST 1  // edge strips' tasks at the lowest blockIdx (high issue priority)
#endif
#ifndef SFV_WALL_OFF
#define SFV_WALL_OFF 148  // first blockIdx of the edge strips' tasks (one CTA per SM of B200 before them)
#endif
#ifndef SFV_GHOST_LEAN
#define SFV_GHOST_LEAN 1  // S/N wall ghosts: per-lane mode and column decided once per task
#endif
#ifndef SFV_LIM_RCP2
#define SFV_LIM_RCP2 1
#endif
#ifndef SFV_RV_AHEAD
#define SFV_RV_AHEAD 1  // NS: register double buffer for the viscous sums (+1.4%, profiles/r1_ns_rv_ahead.txt)
#endif
// Limiter reciprocal: one quadratic Newton step (relative error ~ seed^2,
// ~1e-14) instead of the cubic one: the limiter value only scales a
// difference.  C2 +1.5% (profiles/r1_ab_lim_rcp2.txt); parity margins in
// DESIGN.md §4.2 (C1 gates 4 orders inside; the perturbed-inlet 1000-step
// difference stays at the oracle's own 1-ulp sensitivity)
__device__ __forceinline__ double frcp_lim(double d) {
#if SFV_LIM_RCP2
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    return fma(y, fma(-d, y, 1.0), y);
#else
    return frcp(d);
#endif
}
__device__ __forceinline__ double frsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-(x * y), y, 1.0);          // 1 - x y^2
    return fma(y * e, fma(0.375, e, 0.5), y);  // y (1 + e/2 + 3e^2/8)
}

__device__ __forceinline__ unsigned long long err_key(long long n, int nstages, int stage, int phase,
                                                      long long cell) {
    return ((unsigned long long)((n * nstages + (stage - 1)) * 2 + phase) << 32) | (unsigned long long)cell;
}

// ------------------------------------------------------- MUSCL (Eq. 7)
// For one cell and one direction, component by component: centre value w,
// backward difference b = w - w_prev, forward difference f = w_next - w.
// Returns qU (state at the cell's upper face, +1/2) and qD (lower face, -1/2):
//   qU = w + c1 psi(f,b) b + c2 psi(b,f) f
//   qD = w - c2 psi(f,b) b - c1 psi(b,f) f
// with psi(a,b) the limiter value for difference b given neighbour a
// (reading A-R4).  For VA1 both psi(f,b) b and psi(b,f) f share one
// denominator b^2 + f^2 + delta: one reciprocal per cell, direction and
// component.
template <bool FAST>
__device__ __forceinline__ void muscl_cell(double w, double b, double f, const Params &P, double &qU,
                                           double &qD) {
    if constexpr (FAST && SFV_DIET) {
        // eps = 1 (c1 = 1/2): s1 = max(0, (bf + d/2) / (b^2+f^2+d)); qU = w + s1 b, qD = w - s1 f
        const double r = frcp_lim(fma(b, b, fma(f, f, P.delta)));
        const double s1 = fmax(fma(b, f, P.c1dh + P.c1dh) * r, 0.0);  // c1dh = delta/4 when eps = 1
        qU = fma(s1, b, w);
        qD = fma(-s1, f, w);
        return;
    }
    if constexpr (FAST) {
        // bounded van Albada, kappa = -1 (c2 = 0): s1 = c1 max(0, (2bf+d)/(b^2+f^2+d))
        //   qU = w + s1 b,  qD = w - s1 f
        // with h = s1/2 = c1 (bf + d/2) / (b^2+f^2+d): max(0, 2h) = h + |h| exactly
        const double r = frcp_lim(fma(b, b, fma(f, f, P.delta)));
        const double h = fma(P.c1h, b * f, P.c1dh) * r;
        const double s1 = h + fabs(h);
        qU = fma(s1, b, w);
        qD = fma(-s1, f, w);
        return;
    }
    double pb, pf;  // psi(f,b)*b, psi(b,f)*f
    if (P.limiter == 0) {
        double bf = b * f;
        double r = frcp(fma(b, b, fma(f, f, P.delta)));
        double bfd = bf + P.delta;
        pb = fma(f, f, bfd) * b * r;
        pf = fma(b, b, bfd) * f * r;
        if (bf < 0.0) { pb = 0.0; pf = 0.0; }
    } else if (P.limiter == 1) {
        double bf = b * f;
        double s = fma(2.0, bf, P.delta) * frcp(fma(b, b, fma(f, f, P.delta)));
        s = s > 0.0 ? s : 0.0;
        pb = s * b;
        pf = s * f;
    } else {
        pb = b;
        pf = f;
    }
    qU = fma(P.c1, pb, fma(P.c2, pf, w));
    qD = fma(-P.c2, pb, fma(-P.c1, pf, w));
}

// ------------------------------------------------- Roe + Harten face flux
// |x| by clearing the sign bit (integer pipe; fabs as a value costs a DADD)
__device__ __forceinline__ double dabs(double x) {
    return __longlong_as_double(__double_as_longlong(x) & 0x7fffffffffffffffLL);
}
// Flux through a face of area A with unit normal (nx, ny), times A
// (eigenvector form re-associated into the compact
// dissipation form; Roe averages with sqrt(rho) weights from one rsqrt per
// side).  Returns false if rho <= 0, p <= 0 or a~^2 <= 0 on either side.
__device__ __forceinline__ bool roe_flux(const double qL[4], const double qR[4], double nx, double ny,
                                         double hA, const Params &P, double G[4]) {
    const double gm1 = P.gm1;
    const double rsL = frsqrt(qL[0]), rsR = frsqrt(qR[0]);
    const double irL = rsL * rsL, irR = rsR * rsR;
    const double uL = qL[1] * irL, vL = qL[2] * irL;
    const double uR = qR[1] * irR, vR = qR[2] * irR;
    const double pL = gm1 * fma(-0.5, fma(qL[1], uL, qL[2] * vL), qL[3]);
    const double pR = gm1 * fma(-0.5, fma(qR[1], uR, qR[2] * vR), qR[3]);
    const double VnL = fma(uL, nx, vL * ny), VnR = fma(uR, nx, vR * ny);
    const double EpL = qL[3] + pL, EpR = qR[3] + pR;

    const double sL = qL[0] * rsL, sR = qR[0] * rsR;
    const double w = frcp(sL + sR);
    const double ut = fma(qL[1], rsL, qR[1] * rsR) * w;
    const double vt = fma(qL[2], rsL, qR[2] * rsR) * w;
    const double Ht = fma(EpL, rsL, EpR * rsR) * w;
    const double rhot = sL * sR;
    const double q2h = 0.5 * fma(ut, ut, vt * vt);
    const double a2 = gm1 * (Ht - q2h);
    // (rho <= 0 makes the rsqrt NaN or inf, hence a2 NaN: the a2 test covers it)
    const bool ok = SFV_DIET ? ((pL > 0.0) & (pR > 0.0) & (a2 > 0.0))
                             : ((qL[0] > 0.0) & (qR[0] > 0.0) & (pL > 0.0) & (pR > 0.0) & (a2 > 0.0));
    const double ra = frsqrt(a2);
    const double at = a2 * ra;
    const double ia2 = ra * ra;
    const double Vnt = fma(ut, nx, vt * ny);

    const double drho = qR[0] - qL[0], dp = pR - pL, du = uR - uL, dv = vR - vL, dVn = VnR - VnL;
    const double tt = rhot * at * dVn;
    const double hia2 = 0.5 * ia2;
    const double a1 = (dp - tt) * hia2;
    const double a4 = (dp + tt) * hia2;
    const double a2w = fma(-dp, ia2, drho);

    double l1 = SFV_DIET ? dabs(Vnt - at) : fabs(Vnt - at);
    const double l2 = fabs(Vnt);
    double l4 = SFV_DIET ? dabs(Vnt + at) : fabs(Vnt + at);
    double dH = P.heps * at;
    const bool floor_h = dH < 1e-12;
    const double inv2dH = floor_h ? 0.5e12 : P.hinv * ra;  // 1/(2 eps a) = (0.5/eps) (1/a)
    dH = floor_h ? 1e-12 : dH;
    const double dH2 = dH * dH;
    const double l1f = fma(l1, l1, dH2) * inv2dH, l4f = fma(l4, l4, dH2) * inv2dH;
    l1 = l1 < dH ? l1f : l1;
    l4 = l4 < dH ? l4f : l4;

    const double a1l = l1 * a1, a4l = l4 * a4, a2l = l2 * a2w, r = l2 * rhot;
    const double S = a1l + a4l, Dd = a4l - a1l;
    const double D0 = S + a2l;
    const double T = fma(Dd, at, -r * dVn);
    const double D1 = fma(D0, ut, fma(T, nx, r * du));
    const double D2 = fma(D0, vt, fma(T, ny, r * dv));
    const double D3 = fma(S, Ht, fma(a2l, q2h, fma(T, Vnt, r * fma(ut, du, vt * dv))));

    const double ps = pL + pR;
    const double F0 = fma(qL[0], VnL, qR[0] * VnR);
    const double F1 = fma(qL[1], VnL, fma(qR[1], VnR, ps * nx));
    const double F2 = fma(qL[2], VnL, fma(qR[2], VnR, ps * ny));
    const double F3 = fma(EpL, VnL, EpR * VnR);
    G[0] = (F0 - D0) * hA;  // hA = A/2 from the metrics
    G[1] = (F1 - D1) * hA;
    G[2] = (F2 - D2) * hA;
    G[3] = (F3 - D3) * hA;
    return ok;
}

__device__ __forceinline__ void mirror(const double u[4], double nx, double ny, double g[4]) {
    double mn2 = 2.0 * fma(u[1], nx, u[2] * ny);
    g[0] = u[0];
    g[1] = fma(-mn2, nx, u[1]);
    g[2] = fma(-mn2, ny, u[2]);
    g[3] = u[3];
}

// no-slip adiabatic wall ghost (reading N-R4): momentum negated, rho and E copied
__device__ __forceinline__ void noslip(const double u[4], double g[4]) {
    g[0] = u[0];
    g[1] = -u[1];
    g[2] = -u[2];
    g[3] = u[3];
}

__device__ __forceinline__ void store4(double *buf, int PJ, int i, int j, const double u[4]) {
    double *p = buf + (size_t)((i + 2) * 4) * PJ + (j + JOFF);
#pragma unroll
    for (int c = 0; c < 4; ++c) p[(size_t)c * PJ] = u[c];
}

// ------------------------------------------------------------ stage kernel
// Warp-independent layout: every warp owns a strip of WOUT = 30 output
// columns [j0, j0+30) plus one halo lane on each side (lane l <-> column
// j0-1+l) and marches along i over a segment of rows with its own TMA rings
// and mbarriers.  j-face states / fluxes move between lanes by __shfl, so the
// main loop has no CTA-wide barrier; warps drift independently.

#ifndef SFV_MIN_WARPS
#define SFV_MIN_WARPS (CPL == 1 ? 12 : 8)  // resident warps per SM the register allocation targets (no spills)
#endif
#ifndef SFV_DEEP_MASK
// rings with 2 rows in flight instead of 1 (bit 0: stencil, 1: metrics, 2:
// pointwise).  Measured on C2 / C3 (profiles/r1_ab_ring_depth.txt): pointwise
// +0.3% / +1.3%, stencil -0.2% / +0.3%, all three -8% / -1%; on v20 stencil+pointwise
// -1.3%, metrics+pointwise -8.6% (C2)
#define SFV_DEEP_MASK 4
#endif
#ifndef SFV_PARK
#define SFV_PARK 0  // park the row-carried values in shared memory (fewer registers, more resident warps)
#endif
#ifndef SFV_XSHFL
// lane exchange of j-face states / fluxes by shuffles instead of shared memory
// (round 2b A/B: C2 +1.0 %, C3 +0.6 %, profiles/r2b_ab_xshfl_l2hint.txt; bitwise the same)
#define SFV_XSHFL 1
#endif
#ifndef SFV_PARK_WARPS
#define SFV_PARK_WARPS 14  // resident warps per SM targeted by the parked variants
#endif
template <int MODE>
struct StageTraits {
    static constexpr int NPW = (MODE == M_OWN || MODE == M_RES) ? 0 : (MODE == M_RK4F ? 3 : 1);
    // parked variants: the i-direction values carried from row to row (the
    // cell's last upper-face state, its forward difference, its west-face
    // flux) and the stage-1 norm accumulators live in a per-lane shared-memory
    // slot instead of registers across the two Roe evaluations
    static constexpr bool PARK = SFV_PARK && MODE != M_RK4F;
    static constexpr int PK_PER_COL = 12 + (MODE == M_OWN ? 8 : 0);  // QL[4] fp[4] GW[4] (+ nrm[8])
    static constexpr int K_SLOT = PARK ? CPL * PK_PER_COL * 32 : 0;
    static constexpr int MINW = PARK ? SFV_PARK_WARPS : SFV_MIN_WARPS;
    // the RK4 final stage (3 pointwise inputs) keeps 1 row in flight per ring
    // (12 CTAs/SM fit in 228 KB only so)
    static constexpr bool DEEP = MODE != M_RK4F;
    static constexpr int WS = DEEP && (SFV_DEEP_MASK & 1) ? 5 : 4;  // stencil ring: rows v..v+2 resident + (WS-3) in flight
    static constexpr int MS = DEEP && (SFV_DEEP_MASK & 2) ? 3 : 2;  // metrics ring: row v + (MS-1) in flight
    static constexpr int PS = DEEP && (SFV_DEEP_MASK & 4) && !(PARK && SFV_PARK_WARPS > 12) ? 3 : 2;  // pointwise ring: row v + (PS-1) in flight
    static constexpr int W_SLOT = 4 * WROW;           // 1152 B
    static constexpr int M_SLOT = (NMET * WROW + 15) / 16 * 16;  // 128 B aligned
    static constexpr int P_SLOT = 4 * NPW * WROW;
    static constexpr int X_SLOT = SFV_XSHFL ? 0 : 8 * 32;  // lane exchange: north states [4][32], south fluxes [4][32]
    static constexpr int NBAR = WS + MS + PS;
    static constexpr int WARP_DBL = WS * W_SLOT + MS * M_SLOT + PS * P_SLOT + X_SLOT + 16 + K_SLOT;  // + <= 16 mbarriers
};

template <int MODE>
__host__ __device__ constexpr size_t stage_smem() {
    return sizeof(double) * ((size_t)WPC * StageTraits<MODE>::WARP_DBL + 8 * (NT / 32));
}

#ifndef SFV_UNROLL
#define SFV_UNROLL 1  // row-loop unroll: lets ptxas rename the carried window instead of moving it
#endif
constexpr int kRowUnroll = SFV_UNROLL;


template <int MODE, bool NORMS, bool DTMAX, bool FAST, bool PEER, bool VISC>
__global__ void __launch_bounds__(NT, StageTraits<MODE>::MINW / WPC) stage_kernel(const __grid_constant__ StageArgs a) {
    using TR = StageTraits<MODE>;
    extern __shared__ __align__(128) double smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    double *wbase = smem + warp * TR::WARP_DBL;
    double *wring = wbase;                      // [WS][4][WROW]
    double *mring = wring + TR::WS * TR::W_SLOT;  // [MS][7][WROW]
    double *pring = mring + TR::MS * TR::M_SLOT;  // [PS][4*NPW][WROW]
    double *xch = pring + TR::PS * TR::P_SLOT;  // [8][32] lane exchange
    uint64_t *wbar = reinterpret_cast<uint64_t *>(xch + TR::X_SLOT);   // [WS]
    uint64_t *mbar = wbar + TR::WS;                                      // [MS]
    uint64_t *pbar = mbar + TR::MS;                                      // [PS]
    double *park = xch + TR::X_SLOT + 16;       // [CPL][PK_PER_COL][32] parked row-carried values
    double *red = smem + WPC * TR::WARP_DBL;    // [8][WPC]

    const Params &P = a.P;
    // step index and dt are read after griddepcontrol.wait (programmatic
    // dependent launch: the previous kernel may still be running until then)
    long long n = 0;
    double dt = 0.0, coef = 0.0;
    auto read_step = [&]() {
        // the last CTA of the step's last launch advances the counter
        n = *a.step_ctr;
        double sg = 0.0;
        bool tab = false;
        if constexpr (PEER) tab = a.sig_ranks > 0;  // (peer variants only: keeps the default kernel's code as is)
        if (tab) {
            // device-side max over ranks: lane r waits for rank r's sigma of
            // step n, then a warp max (warp-uniform call)
            const int ln = threadIdx.x & 31;
            double v = 0.0;
            if (ln < a.sig_ranks) {
                wait_flag(a.sig_flag + ln, (unsigned long long)n, a.halo_err);
                v = *(volatile double *)(a.sig_tab + (n & 1) * SIG_RANKS_MAX + ln);
            }
            for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
            sg = v;
        } else {
            sg = a.sig[n & 1];
        }
        dt = P.dt_fixed > 0.0 ? P.dt_fixed : P.cfl / sg;
        coef = a.coef * dt;
    };
    const int PJ = a.PJ;
    double nrm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    double smax = 0.0;

    // warp tasks: nstrips x nseg segments of rows [row_lo, row_split), then
    // (single-wave launches) nstrips x nseg2 short trailing segments of
    // [row_split, row_hi) that the CTA scheduler hands to the slots the
    // first-finishing warps free (the per-sub-partition issue
    // priority makes equal segments end over a wide spread)
    const int task = blockIdx.x * WPC + warp;
    const int ntask1 = a.nstrips * a.nseg;
    if (task < ntask1 + a.nstrips * a.nseg2) {
        const bool trailing = task >= ntask1;
        const int tt = trailing ? task - ntask1 : task;
        int strip = tt % a.nstrips, seg = tt / a.nstrips;
        if (SFV_WALL_FIRST && !trailing && a.nstrips >= 3) {
            // the two edge strips' tasks first: the lowest blockIdx take the
            // sub-partitions' high-priority warp slots, and these strips carry the
            // per-row wall-ghost work (profiles/r2e_timeline_strips.txt)
            // (after the first SFV_WALL_OFF tasks: the first CTA dispatched to
            // each SM ends late in stages that follow a stage of the same step)
            const int nb = 2 * a.nseg;
            const int off = ntask1 >= SFV_WALL_OFF + nb ? SFV_WALL_OFF : 0;
            if (tt >= off && tt < off + nb) {
                strip = ((tt - off) & 1) ? a.nstrips - 1 : 0;
                seg = (tt - off) >> 1;
            } else {
                const int ti = tt < off ? tt : tt - nb;
                strip = 1 + ti % (a.nstrips - 2);
                seg = ti / (a.nstrips - 2);
            }
        }
        const int j0 = strip * WOUT;
        const int j1 = min(j0 + WOUT, a.nj);
        const int jc = j0 - 1 + CPL * lane;          // this lane's first column (CPL columns per lane)
        const int own = CPL * lane + 1;              // its index in a staged row
        bool is_out[CPL], jflux[CPL];                // owns output cell / its j-face is needed
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int col = jc + k;
            is_out[k] = col >= j0 && col < j1;
            jflux[k] = col >= j0 && col <= j1;
        }
        auto writes_ghost = [&](int e) {
            return a.bc[e] == E_SLIP || a.bc[e] == E_OUTFLOW || (VISC && a.bc[e] == E_NOSLIP);
        };
        // edges whose ghost frame this task reads (and, for peer edges, whose
        // neighbour ghost frame it writes): segments at i = 0 / ni, strips
        // whose staged columns reach j = -1 / nj
        const bool ghost_sn = (writes_ghost(2) && j0 == 0) || (writes_ghost(3) && j1 >= a.nj - 1);
        const bool ghost_w = writes_ghost(0), ghost_e = writes_ghost(1);
#if SFV_GHOST_LEAN
        // S / N physical-wall ghosts this lane writes every row (reading A-R11):
        // mode per wall (1 slip mirror, 2 outflow copy into 2 columns, 3 no-slip;
        // bits 0-1 S, 2-3 N), decided once per task instead of per row
        int gmode[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int jk = jc + k;
            int mS = 0, mN = 0;
            if (a.bc[2] == E_SLIP && jk <= 1) mS = 1;
            else if (a.bc[2] == E_OUTFLOW && jk == 0) mS = 2;
            else if (VISC && a.bc[2] == E_NOSLIP && jk <= 1) mS = 3;
            if (a.bc[3] == E_SLIP && jk >= a.nj - 2) mN = 1;
            else if (a.bc[3] == E_OUTFLOW && jk == a.nj - 1) mN = 2;
            else if (VISC && a.bc[3] == E_NOSLIP && jk >= a.nj - 2) mN = 3;
            gmode[k] = is_out[k] ? (mS | mN << 2) : 0;
        }
#endif
        const int lo = trailing ? a.row_split : a.row_lo, ns = trailing ? a.nseg2 : a.nseg;
        const int nrows = (trailing ? a.row_hi : a.row_split) - lo;
        const int i_start = lo + (int)(((long long)nrows * seg) / ns);
        const int i_end = lo + (int)(((long long)nrows * (seg + 1)) / ns);
        const int r0 = i_start - 2, r_last = i_end + 1;  // stencil rows
        unsigned touch = 0;  // bit e: peer edge e (W, E, S, N) touched by this task
        if constexpr (PEER) {
            touch = (a.peer_out[0] != nullptr && i_start == 0 ? 1u : 0u) |
                    (a.peer_out[1] != nullptr && i_end == a.ni ? 2u : 0u) |
                    (a.peer_out[2] != nullptr && j0 == 0 ? 4u : 0u) |
                    (a.peer_out[3] != nullptr && j1 >= a.nj - 1 ? 8u : 0u);
        }
        // j-cut peer columns of this lane, bits 2k (S: columns 0, 1) and 2k+1
        // (N: columns nj-2, nj-1), precomputed once (a combined in-loop test
        // `(touch & 12) && is_out` was mis-evaluated for tasks touching both S
        // and N by ptxas 12.9 in the peer variants: stores skipped, caught by
        // tests/test_gpu_peer.py with py = 3)
        unsigned pcol = 0;
        if constexpr (PEER) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int col = jc + k;
                if ((touch & 4u) && is_out[k] && col <= 1) pcol |= 1u << (2 * k);
                if ((touch & 8u) && is_out[k] && col >= a.nj - 2) pcol |= 2u << (2 * k);
            }
        }
        const int m0 = i_start - 1, m_last = i_end - 1;  // metric rows
        constexpr unsigned ROWB = WROW * 8u;

        auto wslot = [&](int r) -> const double * { return wring + ((unsigned)(r - r0) % TR::WS) * TR::W_SLOT; };
        auto pk = [&](int k, int q) { return (k * TR::PK_PER_COL + q) * 32 + lane; };  // parked value q of column k
        auto mslot = [&](int r) -> const double * { return mring + ((unsigned)(r - m0) % TR::MS) * TR::M_SLOT; };
        // one 2D TMA box per ring row (36 columns x 4 / 7 rows), issued by the
        // whole warp through elect.sync (operands are warp-uniform: 1 warp/CTA);
        // shared-window addresses are computed once
        const int tx = j0 - 2 + JOFF;
        const unsigned wring_s = smem_u32(wring), mring_s = smem_u32(mring), pring_s = smem_u32(pring);
        const unsigned wbar_s = smem_u32(wbar), mbar_s = smem_u32(mbar), pbar_s = smem_u32(pbar);
        auto issue_w = [&](int r) {
            const unsigned s = (unsigned)(r - r0) % TR::WS;
            elect_issue_s(wring_s + s * (TR::W_SLOT * 8u), &a.tm_in, tx, (r + 2) * 4, wbar_s + 8u * s, 4u * ROWB);
        };
        auto issue_m = [&](int r) {
            const unsigned s = (unsigned)(r - m0) % TR::MS;
            elect_issue_s(mring_s + s * (TR::M_SLOT * 8u), &a.tm_met, tx, (r + 1) * NMET, mbar_s + 8u * s,
                          (unsigned)NMET * ROWB);
        };
        auto issue_p = [&](int r) {  // pointwise rows: ring of PS, slot (r - i_start) % PS
            if constexpr (TR::NPW > 0) {
                const unsigned s = (unsigned)(r - i_start) % TR::PS;
                const unsigned dst = pring_s + s * (TR::P_SLOT * 8u), bar = pbar_s + 8u * s;
                elect_issue_s(dst, &a.tm_pw[0], tx, (r + 2) * 4, bar, 4u * TR::NPW * ROWB);
#pragma unroll
                for (int p = 1; p < TR::NPW; ++p)
                    elect_tma_s(dst + p * (4u * WROW * 8u), &a.tm_pw[p], tx, (r + 2) * 4, bar);
            }
        };
        auto wait_w = [&](int r) {
            mbar_wait_s(wbar_s + 8u * ((unsigned)(r - r0) % TR::WS), ((unsigned)(r - r0) / TR::WS) & 1u);
        };
        auto wait_m = [&](int r) {
            mbar_wait_s(mbar_s + 8u * ((unsigned)(r - m0) % TR::MS), ((unsigned)(r - m0) / TR::MS) & 1u);
        };

#if SFV_TIMELINE
        const unsigned long long tl_entry = globaltimer_ns();
        unsigned long long tl_ready = 0, tl_first = 0, tl_row[4] = {0, 0, 0, 0};
#endif
        if (lane == 0) {
            for (int s = 0; s < TR::NBAR; ++s) mbar_init(&wbar[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncwarp();
        // metrics are read-only: prefetch them before waiting for the previous grid
        for (int r = m0; r <= m0 + TR::MS - 1 && r <= m_last; ++r) issue_m(r);
        pdl_wait();
        // trigger only after the wait: at most one dependent grid is pending, so
        // its waiting CTAs cannot hold slots this grid still needs
        pdl_launch_dependents();
        read_step();
#if SFV_TIMELINE
        tl_ready = globaltimer_ns();
#endif
        if constexpr (PEER) {
            // the stage input's ghost layers on a peer edge are the neighbour's
            // previous-stage edge layers: wait for its signal (sequence n*s + k - 1)
            const unsigned long long need = (unsigned long long)(n * a.nstages + a.stage - 1);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (touch & (1u << e)) wait_flag(a.in_flag + e * FLAG_STRIDE, need, a.halo_err);
        }
        for (int r = r0; r <= r0 + TR::WS - 1 && r <= r_last; ++r) issue_w(r);
        for (int r = i_start; r <= i_start + TR::PS - 2 && r < i_end; ++r) issue_p(r);

        // ---- peeled prologue: rows i_start-2, i_start-1 (i direction only) ---
        double Wc[CPL][4], fp[CPL][4], QLp[CPL][4], GW[CPL][4];
        double nWx[CPL], nWy[CPL];            // i-face(0) normal (W-edge slip ghosts)
        double wfx[CPL], wfy[CPL], wfA[CPL];  // west face of the current row (dt)
        wait_w(r0);
        wait_w(r0 + 1);
        wait_w(r0 + 2);
        {
            const double *s0 = wslot(r0), *s1 = wslot(r0 + 1), *s2 = wslot(r0 + 2);
#pragma unroll
            for (int k = 0; k < CPL; ++k)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int o = own + k;
                    const double w0 = s0[c * WROW + o], w1 = s1[c * WROW + o], w2 = s2[c * WROW + o];
                    double qU, qD;
                    muscl_cell<FAST>(w1, w1 - w0, w2 - w1, P, qU, qD);  // cell i_start-1
                    QLp[k][c] = qU;
                    fp[k][c] = w2 - w1;
                    Wc[k][c] = w2;
                }
        }
        __syncwarp();  // rows r0, r0+1 consumed
        for (int r = r0 + TR::WS; r <= r0 + TR::WS + 1 && r <= r_last; ++r) issue_w(r);
        wait_w(r0 + 3);
        wait_m(m0);
#if SFV_TIMELINE
        tl_first = globaltimer_ns();
#endif
        {
            const double *s3 = wslot(r0 + 3);
            const double *m = mslot(m0);
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int o = own + k;
                double qU[4], qD[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const double wn = s3[c * WROW + o];
                    const double f = wn - Wc[k][c];
                    muscl_cell<FAST>(Wc[k][c], fp[k][c], f, P, qU[c], qD[c]);  // cell i_start
                    fp[k][c] = f;
                    Wc[k][c] = wn;
                }
                const double nx = m[0 * WROW + o], ny = m[1 * WROW + o], A = m[2 * WROW + o];
                const bool ok = roe_flux(QLp[k], qD, nx, ny, A, P, GW[k]);
                if (!ok && is_out[k])
                    atomicMin(a.err,
                              err_key(n, a.nstages, a.stage, 0, (long long)(a.gj0 + jc + k) * a.NI + a.gi0 + i_start));
                nWx[k] = nx; nWy[k] = ny;
                wfx[k] = nx; wfy[k] = ny; wfA[k] = A;
#pragma unroll
                for (int c = 0; c < 4; ++c) QLp[k][c] = qU[c];
                if constexpr (TR::PARK) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        park[pk(k, c)] = QLp[k][c];
                        park[pk(k, 4 + c)] = fp[k][c];
                        park[pk(k, 8 + c)] = GW[k][c];
                    }
                    if constexpr (NORMS) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) park[pk(k, 12 + q)] = 0.0;
                    }
                }
            }
        }

        // ---- main loop: one output row per iteration ---------------------------
        double *outp = a.out + (size_t)((i_start + 2) * 4) * PJ + (jc + JOFF);
#if SFV_RV_AHEAD
        double rvn[CPL][4];  // NS: next row's viscous sums (register double buffer)
        if constexpr (VISC) {
#pragma unroll
            for (int k = 0; k < CPL; ++k)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    rvn[k][c] = __ldg(a.rv + (size_t)((i_start + 2) * 4 + c) * PJ + (jc + k + JOFF));
        }
#endif
#pragma unroll kRowUnroll
        for (int v = i_start; v < i_end; ++v) {
#if SFV_TIMELINE
            if (((v - i_start) & 3) == 0 && v > i_start && v - i_start <= 16) tl_row[(v - i_start) / 4 - 1] = globaltimer_ns();
#endif
            // NS: this row's viscous sum, loaded before the fluxes so the load
            // latency hides behind them
            double rvv[CPL][4];
            if constexpr (VISC) {
#if SFV_RV_AHEAD
                // rows v+1's sums load now, row v's were loaded one iteration ago
#pragma unroll
                for (int k = 0; k < CPL; ++k)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        rvv[k][c] = rvn[k][c];
                        rvn[k][c] = v + 1 < i_end ? __ldg(a.rv + (size_t)((v + 3) * 4 + c) * PJ + (jc + k + JOFF)) : 0.0;
                    }
#else
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const double *rvp = a.rv + (size_t)((v + 2) * 4) * PJ + (jc + k + JOFF);
#pragma unroll
                    for (int c = 0; c < 4; ++c) rvv[k][c] = __ldg(rvp + (size_t)c * PJ);
                }
#endif
            }
            if constexpr (TR::PARK) {
                // the row-carried values come back from the lane's parked slot;
                // W(v+1) from the stencil ring (row v+1 is resident)
                const double *s1 = wslot(v + 1);
#pragma unroll
                for (int k = 0; k < CPL; ++k)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        fp[k][c] = park[pk(k, 4 + c)];
                        QLp[k][c] = park[pk(k, c)];
                        Wc[k][c] = s1[c * WROW + own + k];
                    }
            }
            wait_w(v + 2);
            double qD[CPL][4], qU[CPL][4], qS[CPL][4], qN[CPL][4], Wv[CPL][4];
            {
                const double *sn = wslot(v + 2);
                const double *sv = wslot(v);
#pragma unroll
                for (int k = 0; k < CPL; ++k)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {  // i: reconstruct cell (v+1, column k)
                        const double wn = sn[c * WROW + own + k];
                        const double f = wn - Wc[k][c];
                        muscl_cell<FAST>(Wc[k][c], fp[k][c], f, P, qU[k][c], qD[k][c]);
                        fp[k][c] = f;
                        Wc[k][c] = wn;
                        if constexpr (TR::PARK) {
                            park[pk(k, c)] = qU[k][c];  // (this row's QLp was loaded above)
                            park[pk(k, 4 + c)] = f;
                        }
                    }
                double qNup[CPL][4];
#pragma unroll
                for (int k = 0; k < CPL; ++k)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {  // j: reconstruct cell (v, column k)
                        const int o = own + k;
                        const double wm = sv[c * WROW + o - 1];
                        const double w = sv[c * WROW + o];
                        const double wp = sv[c * WROW + o + 1];
                        muscl_cell<FAST>(w, w - wm, wp - w, P, qNup[k][c], qS[k][c]);
                        Wv[k][c] = w;
                    }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if constexpr (SFV_XSHFL)  // lane 0 keeps its own value (as the shared-memory form)
                        qN[0][c] = __shfl_up_sync(0xffffffffu, qNup[CPL - 1][c], 1);
                    else
                        xch[c * 32 + lane] = qNup[CPL - 1][c];  // north state of the last column, read by the lane above
#pragma unroll
                    for (int k = 1; k < CPL; ++k) qN[k][c] = qNup[k - 1][c];
                }
            }
            __syncwarp();  // stencil row v-1, metric row v-1, pointwise slot consumed
            // steady state: row v-1's slots are free -> rows v+WS-1, v+MS-1, v+PS-1
            if (v + TR::WS - 1 >= r0 + TR::WS + 2 && v + TR::WS - 1 <= r_last) issue_w(v + TR::WS - 1);
            if (v + TR::MS - 1 <= m_last && v + TR::MS - 1 >= m0 + TR::MS) issue_m(v + TR::MS - 1);
            if (v + TR::PS - 1 < i_end) issue_p(v + TR::PS - 1);
            wait_m(v);
            const double *mv = mslot(v);
            if constexpr (!SFV_XSHFL) {
#pragma unroll
                for (int c = 0; c < 4; ++c) qN[0][c] = xch[c * 32 + (lane > 0 ? lane - 1 : 0)];
            }
            double GE[CPL][4], GS[CPL][4];
            bool okE[CPL], okS[CPL];
            // all face fluxes of this row: 2 x CPL independent Roe evaluations
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int o = own + k;
                okE[k] = roe_flux(QLp[k], qD[k], mv[0 * WROW + o], mv[1 * WROW + o], mv[2 * WROW + o], P, GE[k]);
                okS[k] = roe_flux(qN[k], qS[k], mv[3 * WROW + o], mv[4 * WROW + o], mv[5 * WROW + o], P, GS[k]);
            }
            double GN[CPL][4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
#pragma unroll
                for (int k = 0; k < CPL; ++k) QLp[k][c] = qU[k][c];
                if constexpr (SFV_XSHFL)
                    GN[CPL - 1][c] = __shfl_down_sync(0xffffffffu, GS[0][c], 1);  // lane 31 keeps its own
                else
                    xch[(4 + c) * 32 + lane] = GS[0][c];  // south flux of column 0 = north flux of the lane below
#pragma unroll
                for (int k = 0; k + 1 < CPL; ++k) GN[k][c] = GS[k + 1][c];
            }
            __syncwarp();
            if constexpr (!SFV_XSHFL) {
#pragma unroll
                for (int c = 0; c < 4; ++c) GN[CPL - 1][c] = xch[(4 + c) * 32 + (lane < 31 ? lane + 1 : 31)];
            }
            const double *prow = pring + ((unsigned)(v - i_start) % TR::PS) * TR::P_SLOT;
            if constexpr (TR::NPW > 0)
                mbar_wait_s(pbar_s + 8u * ((unsigned)(v - i_start) % TR::PS), ((unsigned)(v - i_start) / TR::PS) & 1u);
            bool bad = false;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int o = own + k;
                // ---- residual (Eq. 5) and stage update (Eq. 6): every lane computes,
                // output lanes store (no divergence in the common path)
                const double iV = mv[6 * WROW + o];
                if constexpr (TR::PARK) {
                    const double *svr = wslot(v);  // row v is still resident
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        GW[k][c] = park[pk(k, 8 + c)];
                        Wv[k][c] = svr[c * WROW + o];
                    }
                }
                double R[4], U[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) R[c] = ((GE[k][c] - GW[k][c]) + GN[k][c]) - GS[k][c];
                if constexpr (VISC) {  // R = sum (F - F_v) ds (Eq. 5): the viscous sum of this cell
#pragma unroll
                    for (int c = 0; c < 4; ++c) R[c] -= rvv[k][c];
                }
                const double mcv = -coef * iV;  // -(stage coefficient x dt) / V, once per cell
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if constexpr (MODE == M_OWN) {
                        U[c] = fma(mcv, R[c], Wv[k][c]);
                    } else if constexpr (MODE == M_UN) {
                        U[c] = fma(mcv, R[c], prow[c * WROW + o]);
                    } else if constexpr (MODE == M_RK4F) {
                        const double un = prow[c * WROW + o];
                        const double d2 = prow[(4 + c) * WROW + o] - un;
                        const double d3 = prow[(8 + c) * WROW + o] - un;
                        const double d4 = Wv[k][c] - un;
                        const double comb = (fma(2.0, d3, d2) + d4) * (1.0 / 3.0);
                        U[c] = un + fma(mcv, R[c], comb);
                    } else if constexpr (MODE == M_HEUNF) {
                        const double un = prow[c * WROW + o];
                        U[c] = un + fma(mcv, R[c], 0.5 * (Wv[k][c] - un));
                    } else {  // M_RES: the residual itself (sfv_residual)
                        U[c] = R[c];
                    }
                }
                if (is_out[k]) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) outp[(size_t)c * PJ + k] = U[c];
                }
                // new-state validity: rho > 0 and 2 rho E > |m|^2 (<=> p > 0)
                const bool st_ok = MODE == M_RES || ((U[0] > 0.0) & (2.0 * U[0] * U[3] > fma(U[1], U[1], U[2] * U[2])));
                const int jk = jc + k;
                bad |= (is_out[k] & (!okE[k] | !st_ok)) | (jflux[k] & !okS[k]);
                // physical-boundary ghosts of the new state (reading A-R11), behind one
                // warp-uniform test: only strips at the S / N walls and rows 0, 1, ni-2, ni-1
#if SFV_GHOST_LEAN
                if (MODE != M_RES && ghost_sn) {  // warp-uniform: the S / N wall strips
                    // column 0's (S) / column nj's (N) j-face normal sits at staged index 2 - j0 (+ nj)
                    auto wall = [&](int m, int col, int kk, int col2) {
                        double g[4];
                        if (m == 1) mirror(U, mv[3 * WROW + kk], mv[4 * WROW + kk], g);
                        else if (m == 3) { g[0] = U[0]; g[1] = -U[1]; g[2] = -U[2]; g[3] = U[3]; }
                        else { g[0] = U[0]; g[1] = U[1]; g[2] = U[2]; g[3] = U[3]; }
                        store4(a.out, PJ, v, col, g);
                        if (m == 2) store4(a.out, PJ, v, col2, U);
                    };
                    if (gmode[k] & 3) wall(gmode[k] & 3, -1 - jk, 2 - j0, -2);  // (outflow: jk = 0 -> column -1)
                    if (gmode[k] >> 2) wall(gmode[k] >> 2, a.nj + (a.nj - 1 - jk), 2 - j0 + a.nj, a.nj + 1);
                }
                if (MODE != M_RES && ((ghost_w && v <= 1) || (ghost_e && v >= a.ni - 2)) && is_out[k]) {
#else
                if (MODE != M_RES && (ghost_sn || (ghost_w && v <= 1) || (ghost_e && v >= a.ni - 2)) && is_out[k]) {
#endif
#if !SFV_GHOST_LEAN
                    if (a.bc[2] == E_SLIP && jk <= 1) {
                        double g[4];
                        const int k0 = o - jk;  // column 0
                        mirror(U, mv[3 * WROW + k0], mv[4 * WROW + k0], g);
                        store4(a.out, PJ, v, -1 - jk, g);
                    } else if (a.bc[2] == E_OUTFLOW && jk == 0) {
                        store4(a.out, PJ, v, -1, U);
                        store4(a.out, PJ, v, -2, U);
                    } else if (VISC && a.bc[2] == E_NOSLIP && jk <= 1) {
                        const double g[4] = {U[0], -U[1], -U[2], U[3]};
                        store4(a.out, PJ, v, -1 - jk, g);
                    }
                    if (a.bc[3] == E_SLIP && jk >= a.nj - 2) {
                        double g[4];
                        const int kN = o + (a.nj - jk);  // column nj
                        mirror(U, mv[3 * WROW + kN], mv[4 * WROW + kN], g);
                        store4(a.out, PJ, v, a.nj + (a.nj - 1 - jk), g);
                    } else if (a.bc[3] == E_OUTFLOW && jk == a.nj - 1) {
                        store4(a.out, PJ, v, a.nj, U);
                        store4(a.out, PJ, v, a.nj + 1, U);
                    } else if (VISC && a.bc[3] == E_NOSLIP && jk >= a.nj - 2) {
                        const double g[4] = {U[0], -U[1], -U[2], U[3]};
                        store4(a.out, PJ, v, a.nj + (a.nj - 1 - jk), g);
                    }
#endif
                    if (a.bc[0] == E_SLIP && v <= 1) {  // segments start at 0 or >= 4 (choose_launch)
                        double g[4];
                        if constexpr (TR::PARK)  // i-face(0) normal: metrics row 0 (rare path)
                            mirror(U, a.met[(size_t)0 * PJ + jk + JOFF], a.met[(size_t)1 * PJ + jk + JOFF], g);
                        else
                            mirror(U, nWx[k], nWy[k], g);
                        store4(a.out, PJ, -1 - v, jk, g);
                    } else if (a.bc[0] == E_OUTFLOW && v == 0) {
                        store4(a.out, PJ, -1, jk, U);
                        store4(a.out, PJ, -2, jk, U);
                    } else if (VISC && a.bc[0] == E_NOSLIP && v <= 1) {
                        const double g[4] = {U[0], -U[1], -U[2], U[3]};
                        store4(a.out, PJ, -1 - v, jk, g);
                    }
                    if (a.bc[1] == E_SLIP && v >= a.ni - 2) {
                        double g[4];
                        wait_m(a.ni - 1);  // i-face(ni) lives in metric row ni-1 (issued: <= v+1)
                        const double *mE = mslot(a.ni - 1);
                        mirror(U, mE[0 * WROW + o], mE[1 * WROW + o], g);
                        store4(a.out, PJ, a.ni + (a.ni - 1 - v), jk, g);
                    } else if (a.bc[1] == E_OUTFLOW && v == a.ni - 1) {
                        store4(a.out, PJ, a.ni, jk, U);
                        store4(a.out, PJ, a.ni + 1, jk, U);
                    } else if (VISC && a.bc[1] == E_NOSLIP && v >= a.ni - 2) {
                        const double g[4] = {U[0], -U[1], -U[2], U[3]};
                        store4(a.out, PJ, a.ni + (a.ni - 1 - v), jk, g);
                    }
                }
                if constexpr (PEER) {
                    // peer edges: the new state's 2 edge layers go straight into the
                    // neighbour's ghost frame ("boundary data exchange")
                    // (j-cut columns here; i-cut rows after the loop)
                    if (pcol & (1u << (2 * k))) store4(a.peer_out[2], a.peer_PJ[2], v, a.peer_n[2] + jk, U);
                    if (pcol & (2u << (2 * k))) store4(a.peer_out[3], a.peer_PJ[3], v, jk - a.nj, U);
                }
                if constexpr (NORMS) {
                    if constexpr (TR::PARK) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const double s2 = park[pk(k, 12 + c)], mx = park[pk(k, 16 + c)];
                            park[pk(k, 12 + c)] = is_out[k] ? fma(R[c], R[c], s2) : s2;
                            park[pk(k, 16 + c)] = is_out[k] ? fmax(mx, fabs(R[c])) : mx;
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            nrm[c] = is_out[k] ? fma(R[c], R[c], nrm[c]) : nrm[c];
                            nrm[4 + c] = is_out[k] ? fmax(nrm[4 + c], fabs(R[c])) : nrm[4 + c];
                        }
                    }
                }
                if constexpr (DTMAX) {
                    // sigma/V of the new state for dt_{n+1} (reading A-R6)
                    const double ir = frcp(U[0]);
                    const double u = U[1] * ir, vv = U[2] * ir;
                    const double p = P.gm1 * fma(-0.5, fma(U[1], u, U[2] * vv), U[3]);
                    const double x = P.gamma * p * ir;
                    const double snd = x * frsqrt(x);
                    const double tW = (fabs(fma(u, wfx[k], vv * wfy[k])) + snd) * wfA[k];
                    const double tE =
                        (fabs(fma(u, mv[0 * WROW + o], vv * mv[1 * WROW + o])) + snd) * mv[2 * WROW + o];
                    const double tS =
                        (fabs(fma(u, mv[3 * WROW + o], vv * mv[4 * WROW + o])) + snd) * mv[5 * WROW + o];
                    const double tN = (fabs(fma(u, mv[3 * WROW + o + 1], vv * mv[4 * WROW + o + 1])) + snd) *
                                      mv[5 * WROW + o + 1];
                    // metrics hold A/2: twice the half-area sum (exact scaling)
                    double sv = ((((tW + tE) + tS) + tN) * iV) * 2.0;
                    if constexpr (VISC) {  // viscous spectral radius (reading N-R6)
                        const double sI = wfA[k] + mv[2 * WROW + o];  // (A/2 + A/2: the mean area)
                        const double sJ = mv[5 * WROW + o] + mv[5 * WROW + o + 1];
                        sv = fma(P.visc_dt * ir * fma(sI, sI, sJ * sJ), iV * iV, sv);
                    }
                    smax = (is_out[k] && sv > smax) ? sv : smax;
                    wfx[k] = mv[0 * WROW + o];
                    wfy[k] = mv[1 * WROW + o];
                    wfA[k] = mv[2 * WROW + o];
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    GW[k][c] = GE[k][c];
                    if constexpr (TR::PARK) park[pk(k, 8 + c)] = GE[k][c];
                }
            }
            outp += (size_t)4 * PJ;
            // rare path behind one warp vote: invalid face or new states (reading A-R28)
            if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const int jk = jc + k;
                    if (is_out[k] && !okE[k]) {
                        int I = a.gi0 + v + 1;
                        if (I > a.NI - 1) I = a.NI - 1;
                        atomicMin(a.err, err_key(n, a.nstages, a.stage, 0, (long long)(a.gj0 + jk) * a.NI + I));
                    }
                    if (jflux[k] && !okS[k]) {
                        int J = a.gj0 + jk;
                        if (J > a.NJ - 1) J = a.NJ - 1;
                        atomicMin(a.err, err_key(n, a.nstages, a.stage, 0, (long long)J * a.NI + a.gi0 + v));
                    }
                    if (MODE != M_RES && is_out[k]) {
                        const double *pr = outp - (size_t)4 * PJ;  // the row just stored
                        const double u0 = pr[k], u3 = pr[(size_t)3 * PJ + k];
                        const double u1 = pr[(size_t)PJ + k], u2 = pr[(size_t)2 * PJ + k];
                        if (!((u0 > 0.0) & (2.0 * u0 * u3 > fma(u1, u1, u2 * u2))))
                            atomicMin(a.err,
                                      err_key(n, a.nstages, a.stage, 1, (long long)(a.gj0 + jk) * a.NI + a.gi0 + v));
                    }
                }
            }
        }
#if SFV_TIMELINE
        if (lane == 0 && task < 8192) {
            unsigned smid, wid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
            unsigned long long *tl = g_timeline[(a.stage - 1) & 7][task];
            tl[0] = tl_entry; tl[1] = tl_ready; tl[2] = tl_first; tl[3] = globaltimer_ns();
            tl[4] = smid | (wid << 16); tl[5] = (unsigned long long)(i_end - i_start);
            for (int q = 0; q < 4; ++q) tl[6 + q] = tl_row[q];
        }
#endif
        if constexpr (TR::PARK && NORMS) {
#pragma unroll
            for (int k = 0; k < CPL; ++k)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    nrm[c] += park[pk(k, 12 + c)];
                    nrm[4 + c] = fmax(nrm[4 + c], park[pk(k, 16 + c)]);
                }
        }
        if constexpr (PEER) {
            // arrival of this task on every peer edge it touches; the last of
            // the launch's writers on an edge publishes the stage sequence
            // n*s + k to the neighbour's inbound flag (release, system scope)
            if (touch & 3u) {
                // i-cut edge rows: each lane forwards the 2 rows it just stored
                // (its own writes, L2-resident) to the neighbour's ghost rows
                const int r_lo = (touch & 1u) ? 0 : a.ni - 2, r_hi = (touch & 2u) ? a.ni : 2;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    if (!is_out[k]) continue;
                    const int jk = jc + k;
                    for (int v = r_lo; v < r_hi; ++v) {
                        if (v >= 2 && v < a.ni - 2) continue;
                        const double *src = a.out + (size_t)((v + 2) * 4) * PJ + (jk + JOFF);
                        double u[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) u[c] = src[(size_t)c * PJ];
                        if ((touch & 1u) && v <= 1) store4(a.peer_out[0], a.peer_PJ[0], a.peer_n[0] + v, jk, u);
                        if ((touch & 2u) && v >= a.ni - 2) store4(a.peer_out[1], a.peer_PJ[1], v - a.ni, jk, u);
                    }
                }
            }
            if (touch) {  // warp-uniform
                __threadfence_system();  // every lane: its peer stores before the arrival
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (!(touch & (1u << e))) continue;
                        unsigned *cnt = a.edge_cnt + e * CNT_STRIDE;
                        if (atom_add_acq_rel_gpu(cnt, 1u) == (unsigned)a.edge_writers[e] - 1u) {
                            *cnt = 0u;
                            __threadfence_system();
                            st_release_sys(a.peer_flag[e], (unsigned long long)(n * a.nstages + a.stage));
                        }
                    }
                }
            }
        }
    }
    else {
        pdl_wait();
        pdl_launch_dependents();
        read_step();
    }

    // ---- CTA reductions --------------------------------------------------
    if (DTMAX) {
        for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
        if (lane == 0) red[warp] = smax;
        __syncthreads();
        if (t == 0) {
            double m = red[0];
            for (int w = 1; w < WPC; ++w) m = fmax(m, red[w]);
            atomicMax(reinterpret_cast<unsigned long long *>(&a.sig[(n + 1) & 1]),
                      (unsigned long long)__double_as_longlong(m));
        }
    }
    if (NORMS) {
        // per-CTA partials, ring slot n % pring of [8][ncta]; reduced in fixed
        // order by norms_kernel (batched, off the per-step critical path)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            double x = nrm[q];
            for (int o = 16; o > 0; o >>= 1) {
                double y = __shfl_xor_sync(0xffffffffu, x, o);
                x = q < 4 ? x + y : fmax(x, y);
            }
            if (lane == 0) red[q * WPC + warp] = x;
        }
        __syncthreads();
        if (t < 8) {
            double x = red[t * WPC];
            for (int w = 1; w < WPC; ++w) x = t < 4 ? x + red[t * WPC + w] : fmax(x, red[t * WPC + w]);
            a.partials[((size_t)(n % a.pring) * 8 + t) * a.part_stride + a.part_base + blockIdx.x] = x;
        }
    }
    if (a.bump) {
        // end of step n: the last CTA to arrive records dt_n, clears sigma slot
        // n&1 (the slot step n+1's last stage fills) and advances the counter.
        // Every CTA of every launch of the step has read the counter and the
        // slot by then (earlier launches completed before this grid's
        // griddepcontrol.wait; this grid's CTAs before their arrival).
        __syncthreads();
        if (t == 0) {
            __threadfence();
            if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
                __threadfence();
                a.dt_hist[n % a.cap] = dt;  // dt_n as every CTA of the step used it
                if (!(P.dt_fixed > 0.0)) {
                    if (PEER && a.sig_ranks > 0) {
                        // publish this rank's sigma of U^{n+1} (complete: every CTA
                        // of the launch has arrived) to every rank's table, then flag it
                        const double mine = *(volatile double *)(a.sig + ((n + 1) & 1));
                        for (int r = 0; r < a.sig_ranks; ++r)
                            a.rtab[r][((n + 1) & 1) * SIG_RANKS_MAX + a.rank] = mine;
                        __threadfence_system();
                        for (int r = 0; r < a.sig_ranks; ++r)
                            st_release_sys(a.rflag[r] + a.rank, (unsigned long long)(n + 1));
                    }
                    a.sig[n & 1] = 0.0;
                }
                *a.done = 0u;
                *a.step_ctr = n + 1;
            }
        }
    }
}

// Deterministic fixed-order reduction of a block's per-CTA norm partials
// into the history ("residual print"; reading A-R20): one CTA
// per step, batched every `pring` steps and on demand at query time, so it is
// not on the per-step critical path.
constexpr int FIN_T = 256;
__global__ void __launch_bounds__(FIN_T) norms_kernel(NormsArgs f) {
    __shared__ double part[8][FIN_T / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long n = (f.first >= 0 ? f.first : *f.step_ctr - f.count) + blockIdx.x;
    const double *src = f.partials + (size_t)(n % f.pring) * 8 * f.ncta;
    // fixed assignment (thread t: partials t, t+256, ...) and fixed-order
    // shuffle / warp trees: deterministic for a given launch geometry
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = t; b < f.ncta; b += FIN_T) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double x = src[(size_t)q * f.ncta + b];
            acc[q] = q < 4 ? acc[q] + x : fmax(acc[q], x);
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        double x = acc[q];
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, x, o);
            x = q < 4 ? x + y : fmax(x, y);
        }
        if (lane == 0) part[q][warp] = x;
    }
    __syncthreads();
    if (t < 8) {
        double x = part[t][0];
        for (int w = 1; w < FIN_T / 32; ++w) x = t < 4 ? x + part[t][w] : fmax(x, part[t][w]);
        f.norm_hist[((size_t)(n % f.cap) * f.nblocks + f.block_id) * 8 + t] = x;
    }
}

cudaError_t launch_norms(const NormsArgs &f, cudaStream_t st) {
    if (f.count <= 0) return cudaSuccess;
    norms_kernel<<<f.count, FIN_T, 0, st>>>(f);
    return cudaGetLastError();
}

template <int MODE, bool NORMS, bool DTMAX, bool FAST, bool PEER, bool VISC>
static cudaError_t launch_t(const StageArgs &a, cudaStream_t st) {
    auto k = stage_kernel<MODE, NORMS, DTMAX, FAST, PEER, VISC>;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((a.nstrips * (a.nseg + a.nseg2) + WPC - 1) / WPC);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = stage_smem<MODE>();  // attribute set by prepare_stage_kernels()
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, a);
}

template <int MODE, bool NORMS, bool DTMAX, bool FAST, bool PEER, bool VISC>
static cudaError_t occ_t(int *n) {
    auto k = stage_kernel<MODE, NORMS, DTMAX, FAST, PEER, VISC>;
    const size_t sm = stage_smem<MODE>();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, k, NT, sm);
}

#define SFV_DISPATCH_F(FN, F, Q, V, ...)                                               \
    switch (mode * 4 + (norms ? 2 : 0) + (dtmax ? 1 : 0)) {                              \
        case M_OWN * 4 + 2: return FN<M_OWN, true, false, F, Q, V>(__VA_ARGS__);         \
        case M_OWN * 4 + 0: return FN<M_OWN, false, false, F, Q, V>(__VA_ARGS__);        \
        case M_UN * 4 + 0: return FN<M_UN, false, false, F, Q, V>(__VA_ARGS__);          \
        case M_UN * 4 + 1: return FN<M_UN, false, true, F, Q, V>(__VA_ARGS__);           \
        case M_RK4F * 4 + 1: return FN<M_RK4F, false, true, F, Q, V>(__VA_ARGS__);       \
        case M_RK4F * 4 + 0: return FN<M_RK4F, false, false, F, Q, V>(__VA_ARGS__);      \
        case M_HEUNF * 4 + 1: return FN<M_HEUNF, false, true, F, Q, V>(__VA_ARGS__);     \
        case M_HEUNF * 4 + 0: return FN<M_HEUNF, false, false, F, Q, V>(__VA_ARGS__);    \
        case M_RES * 4 + 0: return FN<M_RES, false, false, F, Q, V>(__VA_ARGS__);        \
        default: return cudaErrorInvalidValue;                                           \
    }
#define SFV_DISPATCH(FN, ...)                                                             \
    if (fast) {                                                                           \
        if (peer && visc) { SFV_DISPATCH_F(FN, true, true, true, __VA_ARGS__) }           \
        else if (peer) { SFV_DISPATCH_F(FN, true, true, false, __VA_ARGS__) }             \
        else if (visc) { SFV_DISPATCH_F(FN, true, false, true, __VA_ARGS__) }             \
        else { SFV_DISPATCH_F(FN, true, false, false, __VA_ARGS__) }                      \
    } else {                                                                              \
        if (peer && visc) { SFV_DISPATCH_F(FN, false, true, true, __VA_ARGS__) }          \
        else if (peer) { SFV_DISPATCH_F(FN, false, true, false, __VA_ARGS__) }            \
        else if (visc) { SFV_DISPATCH_F(FN, false, false, true, __VA_ARGS__) }            \
        else { SFV_DISPATCH_F(FN, false, false, false, __VA_ARGS__) }                     \
    }

// fast = bounded van Albada with kappa = -1 (the default scheme, reading A-R3/A-R7)
bool fast_path(const Params &P) { return P.limiter == 1 && P.c2 == 0.0 && (!SFV_DIET || P.c1 == 0.5); }
cudaError_t launch_stage(const StageArgs &a, int mode, bool norms, bool dtmax, bool peer, bool visc,
                         cudaStream_t st) {
    const bool fast = fast_path(a.P);
    SFV_DISPATCH(launch_t, a, st)
}
cudaError_t stage_occupancy(int mode, bool norms, bool dtmax, bool fast, bool peer, int *n) {
    const bool visc = false;
    SFV_DISPATCH(occ_t, n)
}
cudaError_t stage_occupancy_visc(int mode, bool norms, bool dtmax, bool fast, bool peer, int *n) {
    const bool visc = true;
    SFV_DISPATCH(occ_t, n)
}
cudaError_t prepare_stage_kernels() {
    const int variants[9][3] = {{M_OWN, 1, 0}, {M_OWN, 0, 0}, {M_UN, 0, 0}, {M_UN, 0, 1},  {M_RK4F, 0, 1},
                                {M_RK4F, 0, 0}, {M_HEUNF, 0, 1}, {M_HEUNF, 0, 0}, {M_RES, 0, 0}};
    for (auto &v : variants)
        for (int f = 0; f < 8; ++f) {
            int n = 0;
            cudaError_t e = f < 4 ? stage_occupancy(v[0], v[1] != 0, v[2] != 0, (f & 1) != 0, (f & 2) != 0, &n)
                                  : stage_occupancy_visc(v[0], v[1] != 0, v[2] != 0, (f & 1) != 0, (f & 2) != 0, &n);
            if (e != cudaSuccess) return e;
        }
    return cudaSuccess;
}
size_t stage_smem_bytes(int mode) {
    switch (mode) {
        case M_RES: return stage_smem<M_RES>();
        case M_OWN: return stage_smem<M_OWN>();
        case M_UN: return stage_smem<M_UN>();
        case M_RK4F: return stage_smem<M_RK4F>();
        default: return stage_smem<M_HEUNF>();
    }
}

// ------------------------------------------------------------------ metrics
// IEEE round-to-nearest intrinsics, no contraction: the same arithmetic as
// the paper's metric definitions.
__global__ void metrics_kernel(const MetricsArgs a) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;  // node column
    const int i = blockIdx.y;                             // node row
    if (j > a.nj) return;
    const int W = a.ni + 1;
    auto X = [&](int ii, int jj) { return a.x[(size_t)jj * W + ii]; };
    auto Y = [&](int ii, int jj) { return a.y[(size_t)jj * W + ii]; };
    // memory row m holds i-face(m) (fields 0-2) and j-face(m-1), 1/V(m-1) (fields 3-6)
    double *rowI = a.met + (size_t)(i * NMET) * a.PJ + (j + JOFF);
    double *rowJ = a.met + (size_t)((i + 1) * NMET) * a.PJ + (j + JOFF);
    if (j < a.nj) {  // i-face (i, j)
        const double tx = __dsub_rn(X(i, j + 1), X(i, j)), ty = __dsub_rn(Y(i, j + 1), Y(i, j));
        const double A = __dsqrt_rn(__dadd_rn(__dmul_rn(tx, tx), __dmul_rn(ty, ty)));
        rowI[0 * (size_t)a.PJ] = __ddiv_rn(ty, A);
        rowI[1 * (size_t)a.PJ] = __ddiv_rn(-tx, A);
        rowI[2 * (size_t)a.PJ] = 0.5 * A;  // A/2: the flux's 1/2 (F - D) factor (exact)
    }
    if (i < a.ni) {  // j-face (i, j)
        const double tx = __dsub_rn(X(i + 1, j), X(i, j)), ty = __dsub_rn(Y(i + 1, j), Y(i, j));
        const double A = __dsqrt_rn(__dadd_rn(__dmul_rn(tx, tx), __dmul_rn(ty, ty)));
        rowJ[3 * (size_t)a.PJ] = __ddiv_rn(-ty, A);
        rowJ[4 * (size_t)a.PJ] = __ddiv_rn(tx, A);
        rowJ[5 * (size_t)a.PJ] = 0.5 * A;
        if (j < a.nj) {
            const double V = __dmul_rn(
                0.5, __dsub_rn(__dmul_rn(__dsub_rn(X(i + 1, j + 1), X(i, j)), __dsub_rn(Y(i, j + 1), Y(i + 1, j))),
                               __dmul_rn(__dsub_rn(Y(i + 1, j + 1), Y(i, j)), __dsub_rn(X(i, j + 1), X(i + 1, j)))));
            rowJ[6 * (size_t)a.PJ] = __ddiv_rn(1.0, V);
            if (!(V > 0.0)) atomicMin(a.bad, (unsigned long long)((long long)j * a.ni + i));
        }
    }
}

cudaError_t launch_metrics(const MetricsArgs &a, cudaStream_t st) {
    dim3 g((a.nj + 1 + 127) / 128, a.ni + 1);
    metrics_kernel<<<g, 128, 0, st>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------ Navier-Stokes
// Per stage: Green-Gauss gradients of (u, v, T) (reading N-R2) with the
// ghost gradients of physical edges (N-R1; connected edges are exchanged by
// the host), then the viscous residual sum_f F_v . n A per cell (Eq. 2 viscous
// flux, N-R3/N-R5), which the stage kernel subtracts from the inviscid one.
// Straightforward one-thread-per-cell kernels: correctness first.
// The arithmetic of one cell's (u, v, T), one cell's gradient and one face's
// viscous flux is shared by the two-kernel path and the fused tile kernel and
// written with round-to-nearest intrinsics (no FMA contraction left to the
// compiler), so both paths give bitwise the same numbers wherever they are
// inlined (the loopback decomposition tests compare a fused single block with
// exchanged-gradient blocks bitwise).
#define DM __dmul_rn
#define DA __dadd_rn
#define DS __dsub_rn
__device__ __forceinline__ void uvT_core(double r, double mx, double my, double E, const Params &P, double o[3]) {
    const double ir = frcp(r);
    const double u = DM(mx, ir), v = DM(my, ir);
    const double p = DM(P.gm1, DS(E, DM(0.5, DA(DM(mx, u), DM(my, v)))));
    o[0] = u;
    o[1] = v;
    o[2] = DM(DM(p, ir), P.rgas_inv);
}
__device__ __forceinline__ void uvT(const double *buf, int PJ, int i, int j, const Params &P, double o[3]) {
    const double *q = buf + (size_t)((i + 2) * 4) * PJ + (j + JOFF);
    uvT_core(q[0], q[PJ], q[2 * (size_t)PJ], q[3 * (size_t)PJ], P, o);
}
__device__ __forceinline__ double metf(const double *met, int PJ, int row, int f, int j) {
    return met[(size_t)(row * NMET + f) * PJ + j + JOFF];
}
__device__ __forceinline__ double *gradp(double *grad, int PG, int i, int j, int q) {
    return grad + (size_t)((i + 1) * 6 + q) * PG + (j + 1);
}

// Green-Gauss gradient (reading N-R2) of cell (i, j) from the (u, v, T) of
// the cell and its 4 face neighbours; faces: the mean of the two cells times A
// the cell's metric values: W i-face (nx, ny, A/2) = m0[0..2] (metrics row i),
// E i-face = m1[0..2], S j-face = m1[3..5], 1/V = m1[6] (row i+1, column j),
// N j-face = mn[0..2] (row i+1 fields 3..5, column j+1)
__device__ __forceinline__ void gg_core(const double m0[3], const double m1[7], const double mn[3], const double c[3],
                                        const double w[3], const double e[3], const double s[3], const double n[3],
                                        double g[6]) {
    // per face: n A / (2 V), so grad = sum_f (phi_L + phi_R) n A / (2 V) with outward signs
    const double h = m1[6];  // (the metrics hold A/2)
    const double hW = DM(m0[2], h), hE = DM(m1[2], h);
    const double hS = DM(m1[5], h), hN = DM(mn[2], h);
    const double kWx = DM(m0[0], hW), kWy = DM(m0[1], hW);
    const double kEx = DM(m1[0], hE), kEy = DM(m1[1], hE);
    const double kSx = DM(m1[3], hS), kSy = DM(m1[4], hS);
    const double kNx = DM(mn[0], hN), kNy = DM(mn[1], hN);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double sE = DA(c[q], e[q]), sW = DA(w[q], c[q]), sN = DA(c[q], n[q]), sS = DA(s[q], c[q]);
        // explicit fma: the same rounding wherever this is inlined
        g[2 * q] = fma(-sS, kSx, fma(sN, kNx, fma(-sW, kWx, DM(sE, kEx))));
        g[2 * q + 1] = fma(-sS, kSy, fma(sN, kNy, fma(-sW, kWy, DM(sE, kEy))));
    }
}
__device__ __forceinline__ void gg_cell(const double *met, int PJ, int i, int j, const double c[3], const double w[3],
                                        const double e[3], const double s[3], const double n[3], double g[6]) {
    const double m0[3] = {metf(met, PJ, i, 0, j), metf(met, PJ, i, 1, j), metf(met, PJ, i, 2, j)};
    double m1[7];
#pragma unroll
    for (int f = 0; f < 7; ++f) m1[f] = metf(met, PJ, i + 1, f, j);
    const double mn[3] = {metf(met, PJ, i + 1, 3, j + 1), metf(met, PJ, i + 1, 4, j + 1), metf(met, PJ, i + 1, 5, j + 1)};
    gg_core(m0, m1, mn, c, w, e, s, n, g);
}

// Peer mode (a.peer): edges whose ghosts a CTA of grad_kernel / visc_kernel
// (grid (ceil(nj/128), ni), one cell per thread) reads: W row 0, E row ni-1,
// S the CTA holding column 0, N the one holding column nj-1
__device__ __forceinline__ unsigned visc_touch(const ViscArgs &a) {
    const int i = blockIdx.y;
    return (a.peer_grad[0] && i == 0 ? 1u : 0u) | (a.peer_grad[1] && i == a.ni - 1 ? 2u : 0u) |
           (a.peer_grad[2] && blockIdx.x == 0 ? 4u : 0u) | (a.peer_grad[3] && blockIdx.x == gridDim.x - 1 ? 8u : 0u);
}

__global__ void grad_kernel(const ViscArgs a) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    const unsigned touch = a.peer ? visc_touch(a) : 0u;
    unsigned long long seq = 0;
    if (touch) {  // CTA-uniform: the stage input's ghost layers are the neighbour's stage k-1 edge rows
        seq = (unsigned long long)(*a.step_ctr * a.nstages + a.stage);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (touch & (1u << e)) wait_flag(a.in_flag + e * FLAG_STRIDE, seq - 1, a.halo_err);
    }
    if (j < a.nj) {
        double c[3], w[3], e[3], s[3], n[3], g[6];
        uvT(a.in, a.PJ, i, j, a.P, c);
        uvT(a.in, a.PJ, i - 1, j, a.P, w);
        uvT(a.in, a.PJ, i + 1, j, a.P, e);
        uvT(a.in, a.PJ, i, j - 1, a.P, s);
        uvT(a.in, a.PJ, i, j + 1, a.P, n);
        gg_cell(a.met, a.PJ, i, j, c, w, e, s, n, g);
        // physical-edge ghost cells take this cell's gradient (reading N-R1)
        const bool gw = i == 0 && a.bc[0] != E_CONNECTED, ge = i == a.ni - 1 && a.bc[1] != E_CONNECTED;
        const bool gs = j == 0 && a.bc[2] != E_CONNECTED, gn = j == a.nj - 1 && a.bc[3] != E_CONNECTED;
        // peer edges: the neighbour's ghost gradient is this edge cell's (bit copy)
        const bool pw = (touch & 1u) != 0, pe = (touch & 2u) != 0;
        const bool ps = (touch & 4u) && j == 0, pn = (touch & 8u) && j == a.nj - 1;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            *gradp(a.grad, a.PG, i, j, q) = g[q];
            if (gw) *gradp(a.grad, a.PG, -1, j, q) = g[q];
            if (ge) *gradp(a.grad, a.PG, a.ni, j, q) = g[q];
            if (gs) *gradp(a.grad, a.PG, i, -1, q) = g[q];
            if (gn) *gradp(a.grad, a.PG, i, a.nj, q) = g[q];
            if (pw) *gradp(a.peer_grad[0], a.peer_PG[0], a.peer_n[0], j, q) = g[q];
            if (pe) *gradp(a.peer_grad[1], a.peer_PG[1], -1, j, q) = g[q];
            if (ps) *gradp(a.peer_grad[2], a.peer_PG[2], i, a.peer_n[2], q) = g[q];
            if (pn) *gradp(a.peer_grad[3], a.peer_PG[3], i, -1, q) = g[q];
        }
    }
    if (touch) {
        // arrival of this CTA on every peer edge it touches; the launch's last
        // writer on an edge publishes the sequence to the neighbour's gradient flag
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (!(touch & (1u << e))) continue;
                unsigned *cnt = a.gcnt + e * CNT_STRIDE;
                if (atom_add_acq_rel_gpu(cnt, 1u) == (unsigned)a.gwriters[e] - 1u) {
                    *cnt = 0u;
                    __threadfence_system();
                    st_release_sys(a.peer_gflag[e], seq);
                }
            }
        }
    }
}

// F_v . n A of the face between cells L and R (the lower-index cell is L):
// mean gradients and (u, v) of the two cells (reading N-R3)
__device__ __forceinline__ void face_visc_core(const double gl[6], const double gr[6], const double pl[3],
                                               const double pr[3], double nx, double ny, double A, const Params &P,
                                               double F[4]) {
    // mean gradients / velocities with the 1/2 folded into the coefficients
    double g[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) g[q] = DA(gl[q], gr[q]);          // 2 x mean
    const double u = DM(0.5, DA(pl[0], pr[0])), v = DM(0.5, DA(pl[1], pr[1]));
    const double mu = DM(0.5, P.mu), lam = DM(-2.0 / 3.0, mu), div = DA(g[0], g[3]);
    const double txx = fma(DM(2.0, mu), g[0], DM(lam, div)), tyy = fma(DM(2.0, mu), g[3], DM(lam, div));
    const double txy = DM(mu, DA(g[1], g[2]));
    const double hk = DM(0.5, P.kcond);
    const double thx = fma(hk, g[4], fma(v, txy, DM(u, txx)));
    const double thy = fma(hk, g[5], fma(v, tyy, DM(u, txy)));
    const double A2 = DA(A, A);  // the metrics hold A/2 (exact doubling)
    const double ax = DM(nx, A2), ay = DM(ny, A2);
    F[0] = 0.0;
    F[1] = fma(txy, ay, DM(txx, ax));
    F[2] = fma(tyy, ay, DM(txy, ax));
    F[3] = fma(thy, ay, DM(thx, ax));
}
__device__ __forceinline__ void face_visc(const ViscArgs &a, int iL, int jL, int iR, int jR, const double pl[3],
                                          const double pr[3], double nx, double ny, double A, double F[4]) {
    double gl[6], gr[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        gl[q] = *gradp(a.grad, a.PG, iL, jL, q);
        gr[q] = *gradp(a.grad, a.PG, iR, jR, q);
    }
    face_visc_core(gl, gr, pl, pr, nx, ny, A, a.P, F);
}

// sum over the 4 faces, written to rv (state layout)
__device__ __forceinline__ void store_rv(const ViscArgs &a, int i, int j, const double FW[4], const double FE[4],
                                         const double FS[4], const double FN[4]) {
    double *o = a.rv + (size_t)((i + 2) * 4) * a.PJ + (j + JOFF);
#pragma unroll
    for (int c = 0; c < 4; ++c) o[(size_t)c * a.PJ] = DS(DA(DS(FE[c], FW[c]), FN[c]), FS[c]);
}

__global__ void visc_kernel(const ViscArgs a) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (a.peer) {
        const unsigned touch = visc_touch(a);
        if (touch) {  // the neighbours' edge gradients of this stage (and, already met, its ghost state)
            const unsigned long long seq = (unsigned long long)(*a.step_ctr * a.nstages + a.stage);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (touch & (1u << e)) {
                    wait_flag(a.in_flag + e * FLAG_STRIDE, seq - 1, a.halo_err);
                    wait_flag(a.in_gflag + e * FLAG_STRIDE, seq, a.halo_err);
                }
        }
    }
    if (j >= a.nj) return;
    double c[3], w[3], e[3], s[3], n[3];
    uvT(a.in, a.PJ, i, j, a.P, c);
    uvT(a.in, a.PJ, i - 1, j, a.P, w);
    uvT(a.in, a.PJ, i + 1, j, a.P, e);
    uvT(a.in, a.PJ, i, j - 1, a.P, s);
    uvT(a.in, a.PJ, i, j + 1, a.P, n);
    double FW[4], FE[4], FS[4], FN[4];
    face_visc(a, i - 1, j, i, j, w, c, metf(a.met, a.PJ, i, 0, j), metf(a.met, a.PJ, i, 1, j),
              metf(a.met, a.PJ, i, 2, j), FW);
    face_visc(a, i, j, i + 1, j, c, e, metf(a.met, a.PJ, i + 1, 0, j), metf(a.met, a.PJ, i + 1, 1, j),
              metf(a.met, a.PJ, i + 1, 2, j), FE);
    face_visc(a, i, j - 1, i, j, s, c, metf(a.met, a.PJ, i + 1, 3, j), metf(a.met, a.PJ, i + 1, 4, j),
              metf(a.met, a.PJ, i + 1, 5, j), FS);
    face_visc(a, i, j, i, j + 1, c, n, metf(a.met, a.PJ, i + 1, 3, j + 1), metf(a.met, a.PJ, i + 1, 4, j + 1),
              metf(a.met, a.PJ, i + 1, 5, j + 1), FN);
    store_rv(a, i, j, FW, FE, FS, FN);
}

// Fused gradient + viscous residual for a block without connected edges
// (every ghost gradient is a copy of the adjacent interior cell's, N-R1): a
// CTA takes a VT_I x VT_J tile, stages the (u, v, T) of the tile + 2 rings
// and the gradients of the tile + 1 ring in shared memory, so gradients are
// computed once and never go through global memory.
constexpr int VT_J = 32, VT_I = 12;  // (tile height sweep: profiles/r1_ns_tile_height.txt)
constexpr int VP_J = VT_J + 4, VP_I = VT_I + 4;  // (u, v, T) region
constexpr int VG_J = VT_J + 2, VG_I = VT_I + 2;  // gradient region

__global__ void __launch_bounds__(VT_J * VT_I) gradvisc_kernel(const ViscArgs a) {
    __shared__ double pr[VP_I][VP_J][3];
    __shared__ double gs[VG_I][VG_J][7];  // (6 gradients, padded: conflict-free banks)
    const int i0 = blockIdx.y * VT_I, j0 = blockIdx.x * VT_J;
    const int tid = threadIdx.y * VT_J + threadIdx.x;
    // (u, v, T) of cells i0-2 .. i0+VT_I+1, j0-2 .. j0+VT_J+1 inside the ghost frame
    for (int k = tid; k < VP_I * VP_J; k += VT_J * VT_I) {
        const int ti = k / VP_J, tj = k % VP_J, i = i0 - 2 + ti, j = j0 - 2 + tj;
        const bool iin = i >= 0 && i < a.ni, jin = j >= 0 && j < a.nj;
        if (i >= -2 && i < a.ni + 2 && j >= -2 && j < a.nj + 2 && (iin || jin))  // (no corners)
            uvT(a.in, a.PJ, i, j, a.P, pr[ti][tj]);
    }
    __syncthreads();
    // gradients of interior cells i0-1 .. i0+VT_I, j0-1 .. j0+VT_J
    for (int k = tid; k < VG_I * VG_J; k += VT_J * VT_I) {
        const int ti = k / VG_J, tj = k % VG_J, i = i0 - 1 + ti, j = j0 - 1 + tj;
        if (i >= 0 && i < a.ni && j >= 0 && j < a.nj)
            gg_cell(a.met, a.PJ, i, j, pr[ti + 1][tj + 1], pr[ti][tj + 1], pr[ti + 2][tj + 1], pr[ti + 1][tj],
                    pr[ti + 1][tj + 2], gs[ti][tj]);
    }
    __syncthreads();
    // physical ghost ring inside the gradient region: the adjacent interior cell's
    for (int k = tid; k < VG_I * VG_J; k += VT_J * VT_I) {
        const int ti = k / VG_J, tj = k % VG_J, i = i0 - 1 + ti, j = j0 - 1 + tj;
        const bool iin = i >= 0 && i < a.ni, jin = j >= 0 && j < a.nj;
        if (iin == jin) continue;  // interior (done) or corner (never used)
        if (!iin && (i == -1 || i == a.ni) && jin) {
            const int si = i < 0 ? ti + 1 : ti - 1;
            for (int q = 0; q < 6; ++q) gs[ti][tj][q] = gs[si][tj][q];
        } else if (!jin && (j == -1 || j == a.nj) && iin) {
            const int sj = j < 0 ? tj + 1 : tj - 1;
            for (int q = 0; q < 6; ++q) gs[ti][tj][q] = gs[ti][sj][q];
        }
    }
    __syncthreads();
    const int i = i0 + threadIdx.y, j = j0 + threadIdx.x;
    if (i >= a.ni || j >= a.nj) return;
    const int ti = threadIdx.y + 1, tj = threadIdx.x + 1;  // gradient-region index
    const double *c = pr[ti + 1][tj + 1];
    double FW[4], FE[4], FS[4], FN[4];
    face_visc_core(gs[ti - 1][tj], gs[ti][tj], pr[ti][tj + 1], c, metf(a.met, a.PJ, i, 0, j),
                   metf(a.met, a.PJ, i, 1, j), metf(a.met, a.PJ, i, 2, j), a.P, FW);
    face_visc_core(gs[ti][tj], gs[ti + 1][tj], c, pr[ti + 2][tj + 1], metf(a.met, a.PJ, i + 1, 0, j),
                   metf(a.met, a.PJ, i + 1, 1, j), metf(a.met, a.PJ, i + 1, 2, j), a.P, FE);
    face_visc_core(gs[ti][tj - 1], gs[ti][tj], pr[ti + 1][tj], c, metf(a.met, a.PJ, i + 1, 3, j),
                   metf(a.met, a.PJ, i + 1, 4, j), metf(a.met, a.PJ, i + 1, 5, j), a.P, FS);
    face_visc_core(gs[ti][tj], gs[ti][tj + 1], c, pr[ti + 1][tj + 2], metf(a.met, a.PJ, i + 1, 3, j + 1),
                   metf(a.met, a.PJ, i + 1, 4, j + 1), metf(a.met, a.PJ, i + 1, 5, j + 1), a.P, FN);
    store_rv(a, i, j, FW, FE, FS, FN);
}

// Row-marching fused gradient + viscous residual (blocks without connected
// edges; round 2c): a warp owns 28 output columns (lane l <-> column
// j0 - 2 + l; lanes 2..29 write) and marches along i, carrying the (u, v, T)
// of rows v, v+1 and the gradients of rows v, v+1 in registers; j neighbours
// come by shuffles, the W face flux is the previous row's E face and the S
// face flux is the N face of the lane below.  Every gradient and every face
// flux is evaluated once, with the same helpers and argument values as the
// tile and two-kernel paths (bitwise the same viscous residual).
constexpr int VM_OUT = 28;
#ifndef SFV_NS_MBLK
#define SFV_NS_MBLK 2
#endif
#ifndef SFV_NS_RING
#define SFV_NS_RING 0  // rows of a per-warp cp.async prefetch ring (0: one row ahead in registers; 3 and 4 measured -1 % / -2.5 %, profiles/r2e_ab_ns_ring.txt)
#endif
#ifndef SFV_NS_JEDGE
#define SFV_NS_JEDGE 1  // physical ghost-column gradient shuffles only in the edge strips
#endif
constexpr int VM_RF = 14;  // doubles per lane and row in the ring: raw state (4) + metrics (10)
constexpr size_t VM_SMEM = SFV_NS_RING > 0 ? (size_t)4 * SFV_NS_RING * VM_RF * 32 * sizeof(double) : 0;
__device__ __forceinline__ void cp_async8(unsigned dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(128, SFV_NS_MBLK) gradvisc_march_kernel(const ViscArgs a, int nstrips, int nseg) {
    const int lane = threadIdx.x & 31, task = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (task >= nstrips * nseg) return;
#if SFV_NS_RING > 0
    // per-warp ring [SFV_NS_RING][VM_RF][32]: slot r % SFV_NS_RING holds state
    // row r and metrics row r of this lane's columns (each lane copies and
    // reads only its own elements: no warp synchronisation)
    extern __shared__ double vm_ring[];
    double *ring = vm_ring + (size_t)(threadIdx.x >> 5) * SFV_NS_RING * VM_RF * 32 + lane;
#endif
    const int strip = task % nstrips, seg = task / nstrips;
    const int jc = strip * VM_OUT - 2 + lane;  // this lane's column (may lie in the ghost frame or beyond)
    const int i_s = (int)(((long long)a.ni * seg) / nseg), i_e = (int)(((long long)a.ni * (seg + 1)) / nseg);
    const int jl = min(max(jc, -2), a.nj + 1);   // loadable column (state)
    const int jg = min(max(jc, 0), a.nj - 1);    // interior column (metrics of a cell)
    const int jn = min(max(jc + 1, 0), a.nj);    // the N j-face's column
    const bool jedge = strip * VM_OUT - 2 <= -1 || strip * VM_OUT + 29 >= a.nj;  // physical ghost column in the warp
    const int PJ = a.PJ;
    // raw state of row r at this lane's column; metric values a row's gradient
    // and faces need (see gg_core): i-face row fields 0..2 at jg, fields 3..6
    // at jg, fields 3..5 at jn
    auto load_state = [&](int r, double q[4]) {
        const double *p = a.in + (size_t)((r + 2) * 4) * PJ + (jl + JOFF);
#pragma unroll
        for (int c = 0; c < 4; ++c) q[c] = __ldg(p + (size_t)c * PJ);
    };
    auto load_met = [&](int m, double mr[10]) {  // metrics row m
#pragma unroll
        for (int f = 0; f < 7; ++f) mr[f] = __ldg(a.met + (size_t)(m * NMET + f) * PJ + jg + JOFF);
#pragma unroll
        for (int f = 0; f < 3; ++f) mr[7 + f] = __ldg(a.met + (size_t)(m * NMET + 3 + f) * PJ + jn + JOFF);
    };
    auto to_uvt = [&](const double q[4], double o[3]) { uvT_core(q[0], q[1], q[2], q[3], a.P, o); };
    // gradient of cell row r from its (u, v, T) c (W w, E e; S/N by shuffles) and
    // metrics rows r (mA) and r+1 (mB); physical ghost columns (-1, nj) take the
    // adjacent interior column's (reading N-R1)
    auto grad_row = [&](const double mA[10], const double mB[10], const double c[3], const double w[3],
                        const double e[3], double g[6]) {
        double sS[3], sN[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            sS[q] = __shfl_up_sync(0xffffffffu, c[q], 1);
            sN[q] = __shfl_down_sync(0xffffffffu, c[q], 1);
        }
        const double m0[3] = {mA[0], mA[1], mA[2]};
        const double mn[3] = {mB[7], mB[8], mB[9]};
        gg_core(m0, mB, mn, c, w, e, sS, sN, g);
        if (!SFV_NS_JEDGE || jedge) {  // warp-uniform: only strips holding column -1 or nj
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const double fromE = __shfl_down_sync(0xffffffffu, g[q], 1),
                             fromW = __shfl_up_sync(0xffffffffu, g[q], 1);
                g[q] = jc == -1 ? fromE : (jc == a.nj ? fromW : g[q]);
            }
        }
    };
#if SFV_NS_RING > 0
    // ring entry r (state row r, metrics row r; rows <= ni exist) -> slot r % SFV_NS_RING;
    // one commit group per entry (empty past the last row) so wait_group counts rows
    auto issue_ring = [&](int r) {
        if (r <= a.ni) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(ring + (size_t)(r % SFV_NS_RING) * VM_RF * 32);
            const double *ps = a.in + (size_t)((r + 2) * 4) * PJ + (jl + JOFF);
#pragma unroll
            for (int c = 0; c < 4; ++c) cp_async8(d + c * 256, ps + (size_t)c * PJ);
#pragma unroll
            for (int f = 0; f < 7; ++f) cp_async8(d + (4 + f) * 256, a.met + (size_t)(r * NMET + f) * PJ + jg + JOFF);
#pragma unroll
            for (int f = 0; f < 3; ++f)
                cp_async8(d + (11 + f) * 256, a.met + (size_t)(r * NMET + 3 + f) * PJ + jn + JOFF);
        }
        cp_async_commit();
    };
    for (int r = i_s + 2; r < i_s + 2 + SFV_NS_RING; ++r) issue_ring(r);  // in flight during the prologue
#endif
    // ---- prologue: rows i_s-1 .. i_s+1, gradients of rows i_s-1 and i_s, W face of row i_s
    double uA[3], uB[3], uC[3], g1[6], FW[4];
    double mr1[10], mr2[10];  // metrics rows v+1, v+2
    double sN2[4];            // prefetched: state row v+2 (as raw)
    {
        double q[4], mr0[10], g0[6];
        load_state(i_s - 1, q); to_uvt(q, uA);
        load_state(i_s, q); to_uvt(q, uB);
        load_state(i_s + 1, q); to_uvt(q, uC);
        load_met(i_s, mr0);
        load_met(i_s + 1, mr1);
        grad_row(mr0, mr1, uB, uA, uC, g1);  // row i_s
        if (i_s == 0) {
#pragma unroll
            for (int k = 0; k < 6; ++k) g0[k] = g1[k];
        } else {
            double um[3], mrm[10];
            load_state(i_s - 2, q); to_uvt(q, um);
            load_met(i_s - 1, mrm);
            grad_row(mrm, mr0, uA, um, uB, g0);  // row i_s - 1
        }
        // i-face i_s between cells i_s-1 and i_s: metrics row i_s fields 0-2
        face_visc_core(g0, g1, uA, uB, mr0[0], mr0[1], mr0[2], a.P, FW);
        // rotate to the loop state: uA = row v, uB = row v+1 (uC), mr1 = row v+1
#pragma unroll
        for (int k = 0; k < 3; ++k) { uA[k] = uB[k]; uB[k] = uC[k]; }
#if SFV_NS_RING == 0
        if (i_s + 1 < a.ni) {
            load_met(i_s + 2, mr2);
            load_state(i_s + 2, sN2);
        }
#endif
    }
    // loop state at the top of iteration v: uA = (u, v, T) of row v, uB = row
    // v+1, g1 = gradient of row v, FW = W face flux of row v, mr1 = metrics
    // row v+1, mr2 = row v+2 and sN2 = raw state of row v+2 (if v+1 < ni),
    // (each iteration prefetches the state and metrics rows the next one needs)
    for (int v = i_s; v < i_e; ++v) {
        double gn[6];
        if (v + 1 < a.ni) {
            double uN[3];
#if SFV_NS_RING > 0
            {  // ring entry v+2: state and metrics rows v+2
                cp_async_wait<SFV_NS_RING - 1>();
                const double *sl = ring + (size_t)((v + 2) % SFV_NS_RING) * VM_RF * 32;
#pragma unroll
                for (int c = 0; c < 4; ++c) sN2[c] = sl[c * 32];
#pragma unroll
                for (int f = 0; f < 10; ++f) mr2[f] = sl[(4 + f) * 32];
            }
#endif
            to_uvt(sN2, uN);  // row v+2
#if SFV_NS_RING == 0
            // prefetch one row ahead: state row v+3, metrics row v+4
            double sN3[4], mN[10];
            if (v + 2 < a.ni) {
                load_state(v + 3, sN3);
                load_met(v + 3, mN);
            }
#endif
            grad_row(mr1, mr2, uB, uA, uN, gn);  // row v+1
            // E face of row v (i-face v+1: metrics row v+1 fields 0-2), N face (row v+1 fields 3-5 at jn)
            double FE[4], FN[4], FS[4];
            face_visc_core(g1, gn, uA, uB, mr1[0], mr1[1], mr1[2], a.P, FE);
            {
                double gE[6], uE[3];
#pragma unroll
                for (int q = 0; q < 6; ++q) gE[q] = __shfl_down_sync(0xffffffffu, g1[q], 1);
#pragma unroll
                for (int q = 0; q < 3; ++q) uE[q] = __shfl_down_sync(0xffffffffu, uA[q], 1);
                face_visc_core(g1, gE, uA, uE, mr1[7], mr1[8], mr1[9], a.P, FN);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) FS[c] = __shfl_up_sync(0xffffffffu, FN[c], 1);
            if (lane >= 2 && lane < 2 + VM_OUT && jc < a.nj) store_rv(a, v, jc, FW, FE, FS, FN);
#pragma unroll
            for (int c = 0; c < 4; ++c) FW[c] = FE[c];
#pragma unroll
            for (int q = 0; q < 6; ++q) g1[q] = gn[q];
#pragma unroll
            for (int k = 0; k < 3; ++k) { uA[k] = uB[k]; uB[k] = uN[k]; }
#if SFV_NS_RING > 0
#pragma unroll
            for (int f = 0; f < 10; ++f) mr1[f] = mr2[f];
            issue_ring(v + 2 + SFV_NS_RING);  // into the slot just read
#else
#pragma unroll
            for (int f = 0; f < 10; ++f) { mr1[f] = mr2[f]; mr2[f] = mN[f]; }
#pragma unroll
            for (int c = 0; c < 4; ++c) sN2[c] = sN3[c];
#endif
        } else {
            // last row (v = ni-1): the E neighbour is the ghost row ni, whose
            // gradient is row ni-1's (physical E edge)
            double FE[4], FN[4], FS[4];
            face_visc_core(g1, g1, uA, uB, mr1[0], mr1[1], mr1[2], a.P, FE);
            {
                double gE[6], uE[3];
#pragma unroll
                for (int q = 0; q < 6; ++q) gE[q] = __shfl_down_sync(0xffffffffu, g1[q], 1);
#pragma unroll
                for (int q = 0; q < 3; ++q) uE[q] = __shfl_down_sync(0xffffffffu, uA[q], 1);
                face_visc_core(g1, gE, uA, uE, mr1[7], mr1[8], mr1[9], a.P, FN);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) FS[c] = __shfl_up_sync(0xffffffffu, FN[c], 1);
            if (lane >= 2 && lane < 2 + VM_OUT && jc < a.nj) store_rv(a, v, jc, FW, FE, FS, FN);
        }
    }
#if SFV_NS_RING > 0
    cp_async_wait<0>();
#endif
}

cudaError_t launch_gradvisc_march(const ViscArgs &v, cudaStream_t st) {
    // one wave of warp tasks: segments per strip = resident warps / strips
    // (SFV_NS_MROWS overrides with a segment height)
    static int resident = 0;
    if (!resident) {
        int dev = 0, nsm = 0, blk = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (VM_SMEM > 48 * 1024)
            cudaFuncSetAttribute(gradvisc_march_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)VM_SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blk, gradvisc_march_kernel, 128, VM_SMEM);
        resident = std::max(1, nsm * std::max(1, blk) * 4);
    }
    const int nstrips = (v.nj + VM_OUT - 1) / VM_OUT;
    const char *er = getenv("SFV_NS_MROWS");
    int nseg = std::max(1, resident / nstrips);
    if (er && *er) nseg = std::max(1, (v.ni + std::max(4, atoi(er)) - 1) / std::max(4, atoi(er)));
    nseg = std::min(nseg, std::max(1, v.ni / 4));
    const int tasks = nstrips * nseg;
    gradvisc_march_kernel<<<(tasks + 3) / 4, 128, VM_SMEM, st>>>(v, nstrips, nseg);
    return cudaGetLastError();
}

cudaError_t launch_gradvisc(const ViscArgs &v, cudaStream_t st) {
    gradvisc_kernel<<<dim3((v.nj + VT_J - 1) / VT_J, (v.ni + VT_I - 1) / VT_I), dim3(VT_J, VT_I), 0, st>>>(v);
    return cudaGetLastError();
}

cudaError_t launch_grad(const ViscArgs &v, cudaStream_t st) {
    grad_kernel<<<dim3((v.nj + 127) / 128, v.ni), 128, 0, st>>>(v);
    return cudaGetLastError();
}
cudaError_t launch_visc(const ViscArgs &v, cudaStream_t st) {
    visc_kernel<<<dim3((v.nj + 127) / 128, v.ni), 128, 0, st>>>(v);
    return cudaGetLastError();
}

// --------------------------------------------------------- init / transpose
__global__ void fill_kernel(double *p, long long n, double v) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        p[k] = v;
}
cudaError_t launch_fill(double *buf, long long n, double v, cudaStream_t st) {
    fill_kernel<<<592, 256, 0, st>>>(buf, n, v);
    return cudaGetLastError();
}

// Corner ghosts (both indices outside the interior) are never read by the
// dimension-split stencil (reading A-R18); NaN makes any read visible.
__global__ void corners_kernel(double *buf, int ni, int nj, int PJ) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x - 2;  // -2 .. nj+1
    const int i = blockIdx.y - 2;
    if (j > nj + 1) return;
    const bool iout = i < 0 || i >= ni, jout = j < 0 || j >= nj;
    if (!(iout && jout)) return;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    for (int c = 0; c < 4; ++c) buf[(size_t)((i + 2) * 4 + c) * PJ + j + JOFF] = nan;
}
cudaError_t launch_poison_corners(double *buf, int ni, int nj, int PJ, cudaStream_t st) {
    dim3 g((nj + 4 + 127) / 128, ni + 4);
    corners_kernel<<<g, 128, 0, st>>>(buf, ni, nj, PJ);
    return cudaGetLastError();
}

// Physical-edge ghost fill of a whole buffer (used at set_state; during
// stepping the stage kernel writes these ghosts itself).  Same rules as
// SURVEY §8(c).2 step 2.
__global__ void bc_fill_kernel(double *buf, const double *met, int ni, int nj, int PJ, int4 bc, double4 in0,
                               double4 in1, double4 in2, double4 in3) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = blockIdx.y;  // layer 0/1
    auto ld = [&](int i, int j, double u[4]) {
        for (int c = 0; c < 4; ++c) u[c] = buf[(size_t)((i + 2) * 4 + c) * PJ + j + JOFF];
    };
    auto st = [&](int i, int j, const double u[4]) {
        for (int c = 0; c < 4; ++c) buf[(size_t)((i + 2) * 4 + c) * PJ + j + JOFF] = u[c];
    };
    auto metv = [&](int r, int f, int j) { return met[(size_t)(r * NMET + f) * PJ + j + JOFF]; };
    double u[4], g[4];
    if (k < nj) {  // W and E edges, column k
        const int j = k;
        if (bc.x == E_INFLOW) { double q[4] = {in0.x, in0.y, in0.z, in0.w}; st(-1 - m, j, q); }
        else if (bc.x == E_OUTFLOW) { ld(0, j, u); st(-1 - m, j, u); }
        else if (bc.x == E_SLIP) { ld(m, j, u); mirror(u, metv(0, 0, j), metv(0, 1, j), g); st(-1 - m, j, g); }
        else if (bc.x == E_NOSLIP) { ld(m, j, u); noslip(u, g); st(-1 - m, j, g); }
        if (bc.y == E_INFLOW) { double q[4] = {in1.x, in1.y, in1.z, in1.w}; st(ni + m, j, q); }
        else if (bc.y == E_OUTFLOW) { ld(ni - 1, j, u); st(ni + m, j, u); }
        else if (bc.y == E_SLIP) { ld(ni - 1 - m, j, u); mirror(u, metv(ni, 0, j), metv(ni, 1, j), g); st(ni + m, j, g); }
        else if (bc.y == E_NOSLIP) { ld(ni - 1 - m, j, u); noslip(u, g); st(ni + m, j, g); }
    }
    if (k < ni) {  // S and N edges, row k
        const int i = k;
        if (bc.z == E_INFLOW) { double q[4] = {in2.x, in2.y, in2.z, in2.w}; st(i, -1 - m, q); }
        else if (bc.z == E_OUTFLOW) { ld(i, 0, u); st(i, -1 - m, u); }
        else if (bc.z == E_SLIP) { ld(i, m, u); mirror(u, metv(i + 1, 3, 0), metv(i + 1, 4, 0), g); st(i, -1 - m, g); }
        else if (bc.z == E_NOSLIP) { ld(i, m, u); noslip(u, g); st(i, -1 - m, g); }
        if (bc.w == E_INFLOW) { double q[4] = {in3.x, in3.y, in3.z, in3.w}; st(i, nj + m, q); }
        else if (bc.w == E_OUTFLOW) { ld(i, nj - 1, u); st(i, nj + m, u); }
        else if (bc.w == E_SLIP) { ld(i, nj - 1 - m, u); mirror(u, metv(i + 1, 3, nj), metv(i + 1, 4, nj), g); st(i, nj + m, g); }
        else if (bc.w == E_NOSLIP) { ld(i, nj - 1 - m, u); noslip(u, g); st(i, nj + m, g); }
    }
}
cudaError_t launch_bc_fill(double *buf, const double *met, int ni, int nj, int PJ, const int bc[4],
                           const double in[4][4], cudaStream_t st) {
    const int n = ni > nj ? ni : nj;
    dim3 g((n + 127) / 128, 2);
    bc_fill_kernel<<<g, 128, 0, st>>>(buf, met, ni, nj, PJ, make_int4(bc[0], bc[1], bc[2], bc[3]),
                                      make_double4(in[0][0], in[0][1], in[0][2], in[0][3]),
                                      make_double4(in[1][0], in[1][1], in[1][2], in[1][3]),
                                      make_double4(in[2][0], in[2][1], in[2][2], in[2][3]),
                                      make_double4(in[3][0], in[3][1], in[3][2], in[3][3]));
    return cudaGetLastError();
}

// staging [j][i][4] <-> layout [i][c][j]
__global__ void scatter_kernel(const double *s, double *buf, int ni, int nj, int PJ) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (j >= nj) return;
    for (int c = 0; c < 4; ++c) buf[(size_t)((i + 2) * 4 + c) * PJ + j + JOFF] = s[((size_t)j * ni + i) * 4 + c];
}
__global__ void gather_kernel(const double *buf, double *s, int ni, int nj, int PJ) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (j >= nj) return;
    for (int c = 0; c < 4; ++c) s[((size_t)j * ni + i) * 4 + c] = buf[(size_t)((i + 2) * 4 + c) * PJ + j + JOFF];
}
cudaError_t launch_scatter(const double *s, double *buf, int ni, int nj, int PJ, cudaStream_t st) {
    dim3 g((nj + 127) / 128, ni);
    scatter_kernel<<<g, 128, 0, st>>>(s, buf, ni, nj, PJ);
    return cudaGetLastError();
}
cudaError_t launch_gather(const double *buf, double *s, int ni, int nj, int PJ, cudaStream_t st) {
    dim3 g((nj + 127) / 128, ni);
    gather_kernel<<<g, 128, 0, st>>>(buf, s, ni, nj, PJ);
    return cudaGetLastError();
}

// rho > 0 and p > 0 for an initial state (exact test as the oracle: p from
// u = m/rho); smallest global cell index into *err (key phase 0, stage 0).
__global__ void check_state_kernel(const double *buf, int ni, int nj, int PJ, int gi0, int gj0, int NI,
                                   unsigned long long *err) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (j >= nj) return;
    double u[4];
    for (int c = 0; c < 4; ++c) u[c] = buf[(size_t)((i + 2) * 4 + c) * PJ + j + JOFF];
    bool ok = u[0] > 0.0;
    if (ok) {
        const double uu = u[1] / u[0], vv = u[2] / u[0];
        ok = (u[3] - 0.5 * u[0] * (uu * uu + vv * vv)) > 0.0;
    }
    if (!ok) atomicMin(err, (unsigned long long)((long long)(gj0 + j) * NI + gi0 + i));
}
cudaError_t launch_check_state(const double *buf, int ni, int nj, int PJ, int gi0, int gj0, int NI,
                               unsigned long long *err, cudaStream_t st) {
    dim3 g((nj + 127) / 128, ni);
    check_state_kernel<<<g, 128, 0, st>>>(buf, ni, nj, PJ, gi0, gj0, NI, err);
    return cudaGetLastError();
}

// max over cells of sigma/V for dt_0 (set_state); atomicMax into *sig.
__global__ void sigma_kernel(const double *buf, const double *met, int ni, int nj, int PJ, Params P, double *sig) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    double s = 0.0;
    if (j < nj) {
        double U[4];
        for (int c = 0; c < 4; ++c) U[c] = buf[(size_t)((i + 2) * 4 + c) * PJ + j + JOFF];
        auto m = [&](int r, int f, int jj) { return met[(size_t)(r * NMET + f) * PJ + jj + JOFF]; };
        const double ir = frcp(U[0]);
        const double u = U[1] * ir, vv = U[2] * ir;
        const double p = P.gm1 * fma(-0.5, fma(U[1], u, U[2] * vv), U[3]);
        const double x = P.gamma * p * ir;
        const double snd = x * frsqrt(x);
        const double tW = (fabs(fma(u, m(i, 0, j), vv * m(i, 1, j))) + snd) * m(i, 2, j);
        const double tE = (fabs(fma(u, m(i + 1, 0, j), vv * m(i + 1, 1, j))) + snd) * m(i + 1, 2, j);
        const double tS = (fabs(fma(u, m(i + 1, 3, j), vv * m(i + 1, 4, j))) + snd) * m(i + 1, 5, j);
        const double tN = (fabs(fma(u, m(i + 1, 3, j + 1), vv * m(i + 1, 4, j + 1))) + snd) * m(i + 1, 5, j + 1);
        s = ((((tW + tE) + tS) + tN) * m(i + 1, 6, j)) * 2.0;  // metrics hold A/2
        if (P.visc_dt > 0.0) {  // viscous spectral radius (reading N-R6)
            const double sI = m(i, 2, j) + m(i + 1, 2, j), sJ = m(i + 1, 5, j) + m(i + 1, 5, j + 1);
            const double iV = m(i + 1, 6, j);
            s = fma(P.visc_dt * ir * fma(sI, sI, sJ * sJ), iV * iV, s);
        }
    }
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if ((threadIdx.x & 31) == 0 && s > 0.0)
        atomicMax(reinterpret_cast<unsigned long long *>(sig), (unsigned long long)__double_as_longlong(s));
}
cudaError_t launch_sigma(const double *buf, const double *met, int ni, int nj, int PJ, Params P, double *sig,
                         cudaStream_t st) {
    dim3 g((nj + 127) / 128, ni);
    sigma_kernel<<<g, 128, 0, st>>>(buf, met, ni, nj, PJ, P, sig);
    return cudaGetLastError();
}

// j-cut halo pack / unpack (NCCL path): 2 columns starting at j_first,
// rows i in [0, ni), 4 components -> contiguous [i][c][2].
__global__ void pack_cols_kernel(const double *buf, double *dst, int ni, int PJ, int j_first) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;  // (i, c)
    if (k >= ni * 4) return;
    const int i = k >> 2, c = k & 3;
    const double *p = buf + (size_t)((i + 2) * 4 + c) * PJ + j_first + JOFF;
    dst[2 * k] = p[0];
    dst[2 * k + 1] = p[1];
}
__global__ void unpack_cols_kernel(const double *src, double *buf, int ni, int PJ, int j_first) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ni * 4) return;
    const int i = k >> 2, c = k & 3;
    double *p = buf + (size_t)((i + 2) * 4 + c) * PJ + j_first + JOFF;
    p[0] = src[2 * k];
    p[1] = src[2 * k + 1];
}
cudaError_t launch_pack_cols(const double *buf, double *dst, int ni, int PJ, int j_first, cudaStream_t st) {
    pack_cols_kernel<<<(ni * 4 + 255) / 256, 256, 0, st>>>(buf, dst, ni, PJ, j_first);
    return cudaGetLastError();
}
cudaError_t launch_unpack_cols(const double *src, double *buf, int ni, int PJ, int j_first, cudaStream_t st) {
    unpack_cols_kernel<<<(ni * 4 + 255) / 256, 256, 0, st>>>(src, buf, ni, PJ, j_first);
    return cudaGetLastError();
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t make_row_tensor_map(CUtensorMap *m, const double *base, unsigned long long rows, int PJ, int box_rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)PJ, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)PJ * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)WROW, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

__global__ void debug_math_kernel(int which, const double *in, double *out, long long n) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double x = in[k];
    out[k] = which == 0 ? frcp(x) : which == 1 ? frsqrt(x) : x * frsqrt(x);
}
cudaError_t launch_debug_math(int which, const double *in, double *out, long long n, cudaStream_t st) {
    debug_math_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(which, in, out, n);
    return cudaGetLastError();
}

}  // namespace sfv

#if SFV_TIMELINE
// diagnostic export (timeline builds only; not part of include/sfv.h)
extern "C" int sfv_debug_timeline(void *host, unsigned long long bytes) {
    if (bytes > sizeof(sfv::g_timeline)) bytes = sizeof(sfv::g_timeline);
    return (int)cudaMemcpyFromSymbol(host, sfv::g_timeline, bytes);
}
#endif
