/* sfv.h -- C ABI of the B200-native structured-grid finite-volume hot path
 * of SENSEI (Xue, Wang, Roy, arXiv 2305.18057).
 *
 * What one step computes (PAPER.md citations; DESIGN.md lists the readings
 * A-R* of every point the paper leaves open):
 *   - ghost refresh of the stage input: physical boundary conditions
 *     ("ghost cell extrapolation") and halo exchange with
 *     neighbouring partitions ("boundary data exchange"),
 *     2 layers deep because Eq. 7 reads i-1..i+2;
 *   - MUSCL extrapolation with limiters Psi, Eq. 7, each
 *     Psi computed once per cell and direction;
 *   - the inviscid normal face flux of Eq. 2 by Roe's
 *     scheme with Harten's entropy fix (reading A-R1/A-R2);
 *   - flux-difference accumulation R_h = sum_f F_n ds, Eq. 5;
 *   - the explicit s-stage Runge-Kutta update of Eq. 6
 *     applied to |Omega| dU/dt + R_h = 0, Eq. 4;
 *   - per step: the CFL time step (reading A-R6) and the residual norms of
 *     R(U^n) ("residual print"; reading A-R20);
 *   - optionally (sfv_config.viscous) the viscous normal flux of Eq. 2
 *     (PAPER.md:73-79): R_h = sum_f (F - F_v) ds with Green-Gauss gradients,
 *     no-slip adiabatic walls and a viscous term in the time step
 *     (readings N-R1..N-R6).
 * Everything is IEEE binary64 on the device.
 *
 * Conventions
 *   Ownership: the caller owns every host array and the device workspace.
 *     Host inputs are copied before the call returns; no caller pointer is
 *     retained, except the workspace given to sfv_bind, which must outlive
 *     the ctx.  The library never frees the workspace.
 *   Layouts (host):
 *     nodes  x, y : (ni+1)*(nj+1) doubles, index j*(ni+1)+i
 *     state  U    : ni*nj*4 doubles, index (j*ni+i)*4+k,
 *                   k = rho, rho*u, rho*v, rho*E (conserved)
 *     norms       : per step 8 doubles: L2[4] (RMS) then Linf[4] of R(U^n)
 *   Errors: every call returns an sfv_status; sfv_last_error() gives text.
 *     Physical-validity failures (rho <= 0 or p <= 0 in a face state or a
 *     new stage state) are detected on the device into a sticky word and
 *     reported by the next synchronising call (sfv_sync, sfv_get_*) as
 *     SFV_ERR_STATE with the first failing (step, stage) and, within it,
 *     the smallest global cell index j*ni+i (sfv_error_info).  After
 *     SFV_ERR_STATE the state is undefined until the next sfv_set_state.
 *   Concurrency: one ctx per process and GPU; calls on a ctx from one host
 *     thread.  Device work is enqueued on the stream given to sfv_bind and
 *     is asynchronous unless stated.
 */
#ifndef SFV_H
#define SFV_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct sfv_ctx sfv_ctx;

typedef enum {
    SFV_OK = 0,
    SFV_ERR_ARG = 1,         /* invalid argument or configuration */
    SFV_ERR_GEOMETRY = 2,    /* a cell volume <= 0 */
    SFV_ERR_STATE = 3,       /* rho <= 0 or p <= 0 */
    SFV_ERR_SEQUENCE = 4,    /* call out of order, or history not available */
    SFV_ERR_CUDA = 5,        /* CUDA runtime failure (incl. no device) */
    SFV_ERR_NCCL = 6,        /* NCCL failure or NCCL library not loadable */
    SFV_ERR_OOM = 7,         /* workspace too small */
    SFV_ERR_UNSUPPORTED = 8,
    SFV_ERR_HALO = 9         /* device-initiated halo exchange: a neighbour never signalled */
} sfv_status;

typedef enum { SFV_BC_INFLOW = 0, SFV_BC_OUTFLOW = 1, SFV_BC_SLIP_WALL = 2,
               SFV_BC_NOSLIP_WALL = 3 /* adiabatic; viscous only (reading N-R4) */ } sfv_bc;
typedef enum { SFV_LIM_VAN_ALBADA = 0, SFV_LIM_VAN_ALBADA2 = 1, SFV_LIM_NONE = 2 } sfv_limiter;
typedef enum { SFV_RK4_CLASSIC = 0, SFV_RK2_HEUN = 1, SFV_RK4_JAMESON = 2 } sfv_rk;
/* How the ghost layers of connected edges are refreshed after each stage
 * ("boundary data exchange"):
 *   COPY : device copies between local blocks / NCCL send/recv between ranks
 *          on a high-priority stream, overlapped with the interior launch;
 *   PEER : device-initiated -- the stage kernel's edge tasks store the new
 *          state's 2 edge layers straight into the neighbour's ghost frame
 *          (loopback: same device; ranks: CUDA-IPC mapping over NVLink) and
 *          publish the stage sequence number to the neighbour's inbound flag;
 *          the neighbour's edge tasks wait on it before staging ghosts.  With
 *          nranks <= 32 the CFL max across ranks also goes through peer
 *          memory (no per-step NCCL call). */
typedef enum { SFV_HALO_COPY = 0, SFV_HALO_PEER = 1 } sfv_halo;

typedef struct {
    int32_t ni, nj;              /* interior cells (paper N_l, N_w; N_d = 1), each >= 2 */
    double gamma;                /* ratio of specific heats, > 1 (1.4) */
    double muscl_eps;            /* epsilon of Eq. 7, 0 or 1 */
    double muscl_kappa;          /* kappa of Eq. 7, in [-1, 1] (-1) */
    int32_t limiter;             /* sfv_limiter (VAN_ALBADA)                             reading A-R3 */
    double lim_delta;            /* limiter guard delta (1e-12) */
    double harten_eps;           /* Harten constant; delta_H = max(eps*a, 1e-12) (0.1)   reading A-R2 */
    int32_t rk;                  /* sfv_rk                                               reading A-R5 */
    double cfl;                  /* CFL number of the 4-face dt (0.8 RK4)                reading A-R6 */
    double dt_fixed;             /* > 0: fixed time step, cfl ignored */
    int32_t bc[4];               /* physical boundary per edge W, E, S, N (sfv_bc)      reading A-R11/12 */
    double inflow_U[4][4];       /* conserved inflow state per edge, used if INFLOW      reading A-R27 */
    int64_t max_history;         /* capacity (steps) of the dt / norm history, >= 1 */
    /* Navier-Stokes (Eq. 2 viscous flux; readings N-R1..N-R6):
     * R_h = sum_f (F - F_v) ds with Green-Gauss gradients of (u, v, T).
     * Halo mode SFV_HALO_COPY (loopback blocks or NCCL ranks). */
    int32_t viscous;             /* 0 = Euler, 1 = Navier-Stokes */
    double mu;                   /* constant dynamic viscosity, >= 0            reading N-R5 */
    double prandtl;              /* Prandtl number, > 0 (0.72)                   reading N-R5 */
    double gas_R;                /* gas constant, > 0 (287): T = p / (rho R)     reading N-R5 */
} sfv_config;

/* Validate cfg and copy the node arrays.  Host only (no device work).
 * ARG: ni<2 || nj<2, gamma<=1, |kappa|>1, eps not in {0,1}, cfl<=0 without
 *      dt_fixed, unknown enum, max_history<1, a no-slip wall without viscous,
 *      viscous with mu<0, prandtl<=0 or gas_R<=0.
 * GEOMETRY: some cell volume <= 0 (sfv_error_info gives its i, j). */
sfv_status sfv_create(const sfv_config *cfg, const double *x_nodes, const double *y_nodes,
                      sfv_ctx **out);

/* Decompose the grid into px*py blocks (reading A-R16/24/25):
 * integer largest-remainder widths per direction from the optional integer
 * weights wx[px], wy[py] (NULL = equal); block (bx, by) has rank index
 * bx + px*by and owns [i0,i1) x [j0,j1).
 *   nranks == 1 : all blocks live on this process's device and exchange
 *                 halos by device copies ("loopback"; any px, py).
 *   nranks  > 1 : px*py must equal nranks; this process owns block `rank`
 *                 and exchanges halos with NCCL send/recv; nccl_unique_id
 *                 (128 bytes from sfv_nccl_unique_id on rank 0, broadcast by
 *                 the caller) is required.
 * cuda_device is the device this ctx runs on.  Host only when nranks == 1,
 * and when nranks > 1 with nccl_unique_id == NULL ("planning" mode: maps and
 * halo plans are queryable, sfv_bind then fails with SFV_ERR_NCCL).
 * ARG: px*py inconsistent with nranks, any block width < 2, weight <= 0.
 * NCCL: communicator initialisation failed.  SEQUENCE: after sfv_bind. */
sfv_status sfv_partition(sfv_ctx *ctx, int32_t px, int32_t py, const int32_t *wx, const int32_t *wy,
                         int32_t rank, int32_t nranks, const void *nccl_unique_id, int32_t cuda_device);

/* Rank 0 calls this; the caller broadcasts the 128 bytes (torch.distributed). */
sfv_status sfv_nccl_unique_id(void *out128);

/* Partition map of block `block` (global block index): out8 =
 * i0, i1, j0, j1, neighbour block W, E, S, N (-1 = physical boundary).
 * Host only.  Bit-exact with the oracle's maps. */
sfv_status sfv_partition_map(const sfv_ctx *ctx, int32_t block, int32_t *out8);

/* Halo-exchange plan of block `block` (readings A-R16, A-R18):
 * for each edge W, E, S, N nine int32 (out36[9*e + ...]):
 *   neighbour block (-1 = physical edge, rest 0),
 *   send cells [si0, si1) x [sj0, sj1)   (this block's 2 edge layers),
 *   recv cells [ri0, ri1) x [rj0, rj1)   (its ghost layers, = the neighbour's
 *                                          2 edge layers), global indices.
 * The exchange (device copies or NCCL send/recv) executes exactly this plan;
 * no corner or diagonal messages.  Host only. */
sfv_status sfv_halo_plan(const sfv_ctx *ctx, int32_t block, int32_t *out36);

/* Host-only integer largest-remainder split: starts[parts+1]. */
sfv_status sfv_split(int32_t n, int32_t parts, const int32_t *weights, int32_t *starts);

/* Bytes of device workspace this process needs for its blocks. */
sfv_status sfv_workspace_size(const sfv_ctx *ctx, size_t *bytes);

/* Bind caller-owned device memory (e.g. torch.empty(bytes, uint8, cuda)),
 * >= sfv_workspace_size bytes, 256-byte aligned, and a CUDA stream
 * (cudaStream_t; 0 = legacy default stream).  Computes the metrics (face
 * normals, areas, inverse volumes) on the device.
 * OOM: workspace too small.  CUDA: no device / launch failure. */
sfv_status sfv_bind(sfv_ctx *ctx, void *device_workspace, size_t bytes, void *cuda_stream);

/* Load the initial state U^0 of the explicit scheme (Eq. 6, PAPER.md:105-113:
 * the RK stages start from U^n; the paper's host side "sets up" the data,
 * PAPER.md:120) from a host array, full grid, layout (j*ni + i)*4 + k,
 * k = rho, rho u, rho v, rho E (states must have rho > 0, p > 0);
 * every rank passes the full array and keeps its blocks.  Fills the ghost
 * frames (boundary conditions, + halo exchange),
 * computes dt_0, resets the step counter, histories and
 * error word.  The caller's array is only read during the call.  Synchronous;
 * collective when nranks > 1 (all ranks agree on the error before returning).
 * STATE: some rho <= 0 or p <= 0 (the globally first cell in sfv_error_info).
 * NCCL: exchange / all-reduce failed or timed out (see sfv_set_comm_timeout). */
sfv_status sfv_set_state(sfv_ctx *ctx, const double *U_global);

/* Enqueue nsteps full explicit RK steps U^n -> U^{n+1} (Eq. 6, PAPER.md:105-113;
 * each stage: ghost refresh, limiter + MUSCL Eq. 7,
 * PAPER.md:141-151, Roe flux, residual Eq. 5, PAPER.md:97-101,
 * update) on the bound stream (a CUDA graph per step); returns immediately.
 * Invalid states found on the device are reported by the next synchronising
 * call ("aborts the step with stage index").  Collective in the
 * sense that every rank must step the same number of times.
 * SEQUENCE: before sfv_set_state.  NCCL: communicator aborted earlier. */
sfv_status sfv_step(sfv_ctx *ctx, int32_t nsteps);

/* Wait for enqueued work; *device_ms (may be NULL) = CUDA-event time of the
 * steps enqueued since the previous sfv_sync (the per-iteration time the
 * paper's model is written in, Eq. 8/14).  Surfaces this
 * rank's device errors (SFV_ERR_STATE with step, stage, i, j: SPEC.md:241,
 * :289; SFV_ERR_HALO when a device-side peer wait timed out).  With NCCL
 * ranks the wait is bounded: no step completing within the comm timeout (a
 * neighbour that never sends), or an NCCL async error, aborts the
 * communicator and returns SFV_ERR_NCCL naming this rank's edges and the
 * pending step ("missing neighbor message beyond a configurable
 * timeout -> deadlock error naming the edge"). */
sfv_status sfv_sync(sfv_ctx *ctx, double *device_ms);

/* Steps completed, n of U^n (Eq. 6).  Synchronising (bounded
 * wait as sfv_sync). */
sfv_status sfv_steps_done(sfv_ctx *ctx, int64_t *out);

/* The spatial residual R_h(U) of Eq. 5 (Navier-Stokes
 * mode: sum_f (F - F_v) ds) of a given host state (full grid, sfv_set_state
 * layout) into R (same layout): ghost fill of U by the boundary conditions
 * and the partition exchange, then the fused residual kernel.  Does not
 * touch the solver's state or histories (uses a stage scratch buffer).
 * Synchronising; single rank (loopback blocks).  STATE: an invalid face
 * state of U (cell in sfv_error_info).  UNSUPPORTED: nranks > 1. */
sfv_status sfv_residual(sfv_ctx *ctx, const double *U_global, double *R_global_out);

/* The "residual print" of the solver loop (reading A-R20):
 * per step n in first..first+count-1, out[n*8 + k] = L2_k = sqrt(sum_c
 * R_k(U^n)_c^2 / (ni nj)) and out[n*8 + 4 + k] = Linf_k = max_c |R_k(U^n)_c|,
 * R the Eq. 5 residual of the step's first stage, raw
 * units, count x 8 host doubles owned by the caller.  Reduced over all
 * blocks and ranks in a fixed order (deterministic).  Synchronising;
 * collective when nranks > 1 (device errors are agreed over ranks first).
 * SEQUENCE: range not completed or older than max_history steps. */
sfv_status sfv_get_residual_norms(sfv_ctx *ctx, int64_t first, int64_t count, double *out);

/* Time steps dt_n used by steps first..first+count-1 (count host doubles):
 * dt_n = CFL min_c V_c / sum_f (|u.n_f| + a) A_f of U^n (SPEC.md:294-302,
 * reading A-R6; "if stability conditions are satisfied"), or
 * dt_fixed.  Identical on every rank.  Synchronising (bounded wait).
 * SEQUENCE: range not available. */
sfv_status sfv_get_dt(sfv_ctx *ctx, int64_t first, int64_t count, double *out);

/* "Solution output": copy the current interior state U^n to a
 * host array owned by the caller (full grid, same layout as sfv_set_state).
 * Collective when nranks > 1: every rank receives the full state (each
 * rank's block is broadcast in turn through a device buffer the size of the
 * largest block).  Synchronising; device errors are agreed over ranks first.
 * STATE: the run hit an invalid state.  NCCL: gather failed / timed out. */
sfv_status sfv_get_state(sfv_ctx *ctx, double *U_global_out);

/* "Solution output" of one local block (each rank writes its
 * own part, as the paper's MPI ranks do): U^n of block `block` (a block of
 * this rank: sfv_partition_map gives its extent [i0,i1) x [j0,j1)) into a
 * caller-owned host array of (i1-i0)*(j1-j0)*4 doubles, index
 * ((j-j0)*(i1-i0) + (i-i0))*4 + k.  Not collective; synchronising.
 * ARG: block not local.  SEQUENCE: no state.  STATE: the run hit an invalid
 * state (this rank's view). */
sfv_status sfv_get_block_state(sfv_ctx *ctx, int32_t block, double *U_block_out);

/* Details of the last SFV_ERR_STATE / GEOMETRY: out4 = step, stage, i, j
 * (-1 where not applicable). */
sfv_status sfv_error_info(const sfv_ctx *ctx, int64_t *out4);

/* Diagnostic: launch geometry of the stage kernel of local block 0:
 * out4 = strips, segments, threads per CTA, resident CTAs per SM. */
sfv_status sfv_launch_info(const sfv_ctx *ctx, int32_t *out4);

/* Diagnostic: evaluate the device math helpers used by the stage kernel on
 * n device doubles (which: 0 = reciprocal, 1 = reciprocal square root,
 * 2 = square root) into out (device), on the bound stream; synchronising. */
sfv_status sfv_debug_math(sfv_ctx *ctx, int32_t which, const double *in_dev, double *out_dev, int64_t n);

/* Select the halo-exchange mode (sfv_halo; default COPY).  After sfv_bind;
 * synchronises the stream and requires a new sfv_set_state (the step counter
 * and the peer flags restart there).  PEER with nranks > 1 needs
 * sfv_peer_connect first.  ARG: unknown mode.  SEQUENCE: order violated.
 * A peer that never signals is reported by the next synchronising call as
 * SFV_ERR_HALO (after a 20 s device-side timeout; no hang).  Navier-Stokes
 * mode (viscous = 1) in PEER: the gradient kernel also stores its edge
 * gradients into the neighbour's gradient frame and signals (PAPER.md:120
 * "exchange ghost cells", here the 1-layer gradient ghosts the viscous
 * flux of Eq. 2, needs). */
sfv_status sfv_set_halo_mode(sfv_ctx *ctx, int32_t mode);

/* nranks > 1, after sfv_bind: 128 opaque bytes describing this rank's block
 * for its neighbours (CUDA-IPC handle of the allocation holding the
 * workspace, the workspace offset, buffer and flag offsets, ni, nj, pitch,
 * block id).  The workspace must come from cudaMalloc (e.g. PyTorch's default
 * caching allocator), not from a VMM / expandable segment.  CUDA: no IPC. */
sfv_status sfv_peer_handle(sfv_ctx *ctx, void *out128);

/* nranks > 1: map the face neighbours' workspaces.  handles = nranks x 128
 * bytes, entry r = sfv_peer_handle of rank r (all-gathered by the caller).
 * ARG: an entry inconsistent with the partition.  CUDA: IPC open failed
 * (no peer access between the devices). */
sfv_status sfv_peer_connect(sfv_ctx *ctx, const void *handles);

/* Diagnostic: copy state buffer k (0 = U^n, 1.. = stage buffers of the
 * tableau) of local block `block`, ghost frame included, to the host:
 * out[((i+2)*4 + c)*(nj_b+4) + (j+2)] for i in [-2, ni_b+2), c in 0..3,
 * j in [-2, nj_b+2) (block-local indices; corner ghosts are NaN).
 * Navier-Stokes mode also: k = -1 the last stage's viscous residual
 * sum_f F_v . n A (same layout, interior meaningful), k = -2 the gradient
 * frame (u_x, u_y, v_x, v_y, T_x, T_y): out[((i+1)*6 + q)*(nj_b+2) + j+1],
 * i in [-1, ni_b], j in [-1, nj_b].
 * Synchronising.  ARG: block not local or k out of range. */
sfv_status sfv_debug_block_buffer(sfv_ctx *ctx, int32_t block, int32_t k, double *out);

/* Per-class stage timing (the paper's iteration breakdown: interior
 * residual, boundary work and data exchange, PAPER.md:157, :172, :195;
 * SPEC.md:338-341 StageTimings).  on != 0: subsequent sfv_step calls enqueue
 * each stage without the CUDA graph, with CUDA events around every class of
 * work (slower per step: a diagnostic mode); accumulators are reset.
 * Synchronising.  SEQUENCE: before sfv_bind. */
sfv_status sfv_set_profiling(sfv_ctx *ctx, int32_t on);

/* Accumulated device milliseconds since sfv_set_profiling(ctx, 1), out[9]:
 * [0] edge-row stage kernels (launched first when a connected i-cut is
 * overlapped), [1] interior stage kernels (all stage kernels when not split),
 * [2] row-halo exchange (on the comm stream when overlapped; every exchange
 * when not), [3] column-halo pack/exchange/unpack, [4] exposed wait of the
 * compute stream for the comm stream, [5] dt all-reduce, [6] Navier-Stokes
 * viscous kernels, [7] norms batches, [8] number of profiled steps.
 * Classes on different streams overlap in time.  Synchronising. */
sfv_status sfv_get_stage_timings(sfv_ctx *ctx, double *out9);

/* Failure detection of the NCCL path: a synchronising call
 * that sees no step complete for `seconds` (default 60) aborts the
 * communicator and returns SFV_ERR_NCCL naming the edges.  ARG: seconds <= 0. */
sfv_status sfv_set_comm_timeout(sfv_ctx *ctx, double seconds);

/* Text of the last error on ctx (ctx-owned, valid until the next call). */
const char *sfv_last_error(const sfv_ctx *ctx);

/* Free library-owned host, CUDA-graph and NCCL resources (not the workspace).
 * Drains the bound stream first (and, in peer mode across ranks, an
 * all-reduce barrier so no neighbour still stores into this workspace), so
 * the caller may release the workspace once this returns. */
void sfv_destroy(sfv_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
