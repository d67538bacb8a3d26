// sfv_internal.h -- shared host/device declarations of libsfv (product path).
// Not part of the C ABI (include/sfv.h is).  No code here is shared with the
// oracle (oracle/), which is test infrastructure.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sfv {

// Device layout of one block's state buffer ("[i][c][j]", j fastest):
//   element (i, j, c) at ((i + 2) * 4 + c) * PJ + (j + JOFF),
//   i in [-2, ni+2), j in [-2, nj+2), c = rho, rho u, rho v, rho E.
// The partitioned index i is the slow one, so the 2 edge rows of an i-cut
// are one contiguous run (zero-copy halo send/recv).
// Metrics: memory row m in [0, ni] holds 7 fields, each PJ doubles at column
// j + JOFF: i-face (m, j) nx, ny, A/2; j-face (m-1, j) nx, ny, A/2; 1/V(m-1, j),
// so the stage kernel's iteration over cell row v stages one metrics row
// (m = v+1) holding its east face, its south face and its volume.
constexpr int JOFF = 4;
constexpr int NMET = 7;
constexpr int SMEM_ROW = 132;     // doubles per staged row in shared memory
constexpr int ROW_COLS = 130;     // columns staged per row: j0-2 .. j0+127
#ifndef SFV_NT
#define SFV_NT 32
#endif
constexpr int NT = SFV_NT;        // threads per CTA of the stage kernel (independent warps)
constexpr int WPC = NT / 32;      // independent warps per CTA
#ifndef SFV_CPL
#define SFV_CPL 1                 // columns per lane of the stage kernel
#endif
constexpr int CPL = SFV_CPL;
constexpr int WOUT = 32 * CPL - 2;  // output columns per warp strip (+1 halo column each side)
constexpr int WROW = 32 * CPL + 4;  // staged doubles per row: columns j0-2 .. j0+32*CPL+1


enum Mode { M_OWN = 0, M_UN = 1, M_RK4F = 2, M_HEUNF = 3, M_RES = 4 };  // M_RES: write R, no update
enum Edge { E_INFLOW = 0, E_OUTFLOW = 1, E_SLIP = 2, E_NOSLIP = 3, E_CONNECTED = 4 };

struct Params {
    double gamma, gm1;
    double c1, c2;          // eps(1-kappa)/4, eps(1+kappa)/4 (Eq. 7)
    double c1h, c1dh;       // c1, c1 delta / 2 (fast path: bounded van Albada, kappa = -1)
    double delta;           // limiter guard
    double heps, hinv;      // Harten eps and 0.5/eps
    double cfl, dt_fixed;
    int limiter;
    // Navier-Stokes (readings N-R1..N-R6)
    double mu, kcond, rgas, rgas_inv;  // viscosity, conductivity mu c_p / Pr, gas constant
    double visc_dt;                    // 4 max(4/3, gamma) mu / Pr: viscous spectral radius factor (N-R6)
};

struct StageArgs {
    // 2D TMA descriptors: state buffers as [(ni+4)*4 rows][PJ] doubles,
    // metrics as [(ni+1)*7 rows][PJ]; boxes of 36 columns x 4 (7) rows
    CUtensorMap tm_in, tm_met, tm_pw[3];
    const double *in;       // stage input (stencil)
    double *out;            // stage output
    const double *pw0, *pw1, *pw2;   // pointwise inputs (U^n, W2, W3)
    const double *met;
    int ni, nj, PJ;
    int gi0, gj0, NI, NJ;
    int nstrips, nseg;
    int row_lo, row_hi;     // rows of this launch (edge strips / interior split)
    int row_split, nseg2;   // trailing short segments: nseg over [row_lo, row_split), nseg2 over [row_split, row_hi)
    int part_base, part_stride;  // column range of this launch in the norm partials
    int bc[4];              // Edge per W, E, S, N
    double coef;            // this stage's dt multiplier
    double *sig;            // [2] max over cells of sigma/V (bits, atomicMax)
    long long *step_ctr;
    double *dt_hist;        // [cap]
    double *norm_hist;      // [cap][nblocks][8]
    int cap, block_id, nblocks;
    double *partials;       // [pring][8][part_stride] norm partials ring (stage 1 of step n: slot n % pring)
    int pring;
    unsigned *done;         // CTA arrival counter of the step's last launch (bump)
    int bump;               // last launch of the step: record dt_n, clear its sigma slot, advance the counter
    unsigned long long *err;
    int stage, nstages;
    // device-initiated halo exchange (halo mode SFV_HALO_PEER):
    // per edge W, E, S, N the neighbour's copy of this stage's output buffer
    // (NULL = not a peer edge), its pitch and its ni (W) / nj (S), the
    // neighbour's inbound flag for the shared edge (signalled with the stage
    // sequence number), this block's own inbound flags and writer arrival
    // counters, and the number of CTAs of this launch that touch each edge
    double *peer_out[4];
    unsigned long long *peer_flag[4];
    int peer_PJ[4], peer_n[4];
    unsigned long long *in_flag;  // [4 * FLAG_STRIDE]
    unsigned *edge_cnt;           // [4 * CNT_STRIDE]
    int edge_writers[4];
    unsigned *halo_err;           // sticky: a peer never signalled (timeout)
    // device-side CFL max across ranks (peer mode, nranks > 1):
    // every rank's sigma of step n lands in slot n&1 of each rank's table and
    // is flagged with n; stage kernels take dt_n = cfl / max_r table[n&1][r]
    int sig_ranks, rank;          // 0 = off (local sigma: one rank, or NCCL all-reduce)
    double *sig_tab;              // local [2][SIG_RANKS_MAX]
    unsigned long long *sig_flag; // local [SIG_RANKS_MAX]: rank r published slot for step >= value
    double *const *rtab;          // [sig_ranks] every rank's sig_tab (mapped; own included)
    unsigned long long *const *rflag;  // [sig_ranks] every rank's sig_flag
    const double *rv;             // NS: viscous residual sum_f F_v . n A, state layout (NULL = Euler)
    Params P;
};
constexpr int FLAG_STRIDE = 16;   // u64 per inbound flag (own 128-B line)
constexpr int CNT_STRIDE = 32;    // u32 per arrival counter
// per block: state flags [0, 512), state-writer counters [512, 1024), and in
// Navier-Stokes peer mode gradient flags [1024, 1536), gradient-writer
// counters [1536, 2048); the block's gradient frame follows at the next
// 256-byte boundary on every rank (sfv_peer_connect derives it)
constexpr size_t PEER_SYNC_BYTES = 2048;
constexpr size_t PEER_ECNT_OFF = 512, PEER_GFLAG_OFF = 1024, PEER_GCNT_OFF = 1536;
constexpr int SIG_RANKS_MAX = 32;
// workspace misc region (same offsets on every rank)
constexpr size_t MISC_BYTES = 2048;
constexpr size_t MISC_SIGTAB = 256;    // double [2][SIG_RANKS_MAX]
constexpr size_t MISC_SIGFLAG = 768;   // u64 [SIG_RANKS_MAX]
constexpr size_t MISC_RTAB = 1024;     // double * [SIG_RANKS_MAX]
constexpr size_t MISC_RFLAG = 1536;    // u64 * [SIG_RANKS_MAX]  // per block: flags [0, 512), counters [512, 1024)

// Reduction of `count` steps of one block's norm partials into the history:
// steps first .. first+count-1 (first < 0: the `count` steps before *step_ctr).
struct NormsArgs {
    const double *partials;  // ring [pring][8][ncta]
    int ncta, pring;
    double *norm_hist;
    const long long *step_ctr;
    long long first;
    int count, cap, block_id, nblocks;
};

struct MetricsArgs {
    const double *x, *y;    // block-local nodes (nj+1) x (ni+1), [j][i]
    double *met;
    int ni, nj, PJ;
    unsigned long long *bad;  // smallest j*ni+i with V <= 0 (block-local)
};

// launchers (sfv_kernels.cu); all asynchronous on `st`
cudaError_t launch_stage(const StageArgs &a, int mode, bool norms, bool dtmax, bool peer, bool visc,
                         cudaStream_t st);
// Navier-Stokes per stage: Green-Gauss gradients of (u, v, T)
// of a block's stage input into grad ([(i+1)*6+q]*PG + j+1, i in [-1, ni],
// j in [-1, nj]), physical-edge ghost gradients, then the viscous residual
struct ViscArgs {
    const double *in;        // stage input (state layout, ghosts filled)
    const double *met;
    double *grad;
    double *rv;              // out: sum over the 4 faces of F_v . n A (state layout)
    int ni, nj, PJ, PG;
    int bc[4];               // Edge per W, E, S, N (E_CONNECTED: exchanged ghosts)
    Params P;
    // device-initiated halos (SFV_HALO_PEER): grad_kernel waits
    // for the stage input's ghost layers (inbound state flags, sequence
    // n*s + k - 1), stores its edge gradients into the neighbour's gradient
    // frame and publishes n*s + k to the neighbour's inbound gradient flag;
    // visc_kernel's edge CTAs wait for that flag.  peer = 0: copy mode.
    int peer;
    double *peer_grad[4];                  // neighbour's gradient frame per edge W, E, S, N (NULL: none)
    int peer_PG[4], peer_n[4];             // its pitch, its ni (W) / nj (S)
    unsigned long long *peer_gflag[4];     // neighbour's inbound gradient flag for the shared edge
    const unsigned long long *in_flag;     // this block's inbound state flags [4 * FLAG_STRIDE]
    unsigned long long *in_gflag;          // this block's inbound gradient flags [4 * FLAG_STRIDE]
    unsigned *gcnt;                        // gradient-writer arrival counters [4 * CNT_STRIDE]
    int gwriters[4];                       // CTAs of the grad launch touching each edge
    unsigned *halo_err;
    const long long *step_ctr;
    int stage, nstages;
};
cudaError_t launch_grad(const ViscArgs &v, cudaStream_t st);
cudaError_t launch_visc(const ViscArgs &v, cudaStream_t st);
cudaError_t launch_gradvisc(const ViscArgs &v, cudaStream_t st);  // blocks without connected edges
cudaError_t launch_gradvisc_march(const ViscArgs &v, cudaStream_t st);  // (same, row-marching warps)
cudaError_t launch_norms(const NormsArgs &f, cudaStream_t st);
cudaError_t stage_occupancy(int mode, bool norms, bool dtmax, bool fast, bool peer, int *ctas_per_sm);
cudaError_t stage_occupancy_visc(int mode, bool norms, bool dtmax, bool fast, bool peer, int *ctas_per_sm);
bool fast_path(const Params &P);
cudaError_t prepare_stage_kernels();
size_t stage_smem_bytes(int mode);
cudaError_t launch_metrics(const MetricsArgs &a, cudaStream_t st);
cudaError_t launch_fill(double *buf, long long n, double v, cudaStream_t st);
cudaError_t launch_poison_corners(double *buf, int ni, int nj, int PJ, cudaStream_t st);
cudaError_t launch_bc_fill(double *buf, const double *met, int ni, int nj, int PJ, const int bc[4],
                           const double inflow[4][4], cudaStream_t st);
cudaError_t launch_scatter(const double *stage_jik, double *buf, int ni, int nj, int PJ, cudaStream_t st);
cudaError_t launch_gather(const double *buf, double *stage_jik, int ni, int nj, int PJ, cudaStream_t st);
cudaError_t launch_check_state(const double *buf, int ni, int nj, int PJ, int gi0, int gj0, int NI,
                               unsigned long long *err, cudaStream_t st);
cudaError_t launch_sigma(const double *buf, const double *met, int ni, int nj, int PJ, Params P,
                         double *sig, cudaStream_t st);
cudaError_t launch_pack_cols(const double *buf, double *dst, int ni, int PJ, int j_first, cudaStream_t st);
cudaError_t launch_unpack_cols(const double *src, double *buf, int ni, int PJ, int j_first, cudaStream_t st);
// cuTensorMapEncodeTiled through the runtime's driver entry point
cudaError_t make_row_tensor_map(CUtensorMap *m, const double *base, unsigned long long rows, int PJ, int box_rows);
cudaError_t launch_debug_math(int which, const double *in, double *out, long long n, cudaStream_t st);

}  // namespace sfv
