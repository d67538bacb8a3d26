// sfv_host.cu -- host runtime behind include/sfv.h: validation, partition
// and ghost maps, workspace carve-up, per-step CUDA graph, halo exchange
// (device copies between local blocks, NCCL send/recv between ranks, or the
// device-initiated peer mode with CUDA-IPC mappings), the Navier-Stokes
// per-stage kernels, and history / error bookkeeping.  See DESIGN.md §3-§6.
#include <dlfcn.h>
#include <nccl.h>

#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <memory>
#include <thread>
#include <cmath>
#include <deque>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sfv.h"
#include "sfv_internal.h"

using namespace sfv;

namespace {

constexpr int NSEG_MAX = 256;
constexpr long long kMaxInflight = 8;  // NCCL-rank steps enqueued ahead of completion
constexpr size_t PADD = 512;  // padding doubles after each array (bulk-copy over-read)

// ------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl &nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return n;
#define SFV_SYM(f) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, "nccl" #f))
    SFV_SYM(GetUniqueId);
    SFV_SYM(CommInitRank);
    SFV_SYM(CommDestroy);
    SFV_SYM(Send);
    SFV_SYM(Recv);
    SFV_SYM(GroupStart);
    SFV_SYM(GroupEnd);
    SFV_SYM(AllReduce);
    SFV_SYM(Broadcast);
    SFV_SYM(CommGetAsyncError);
    SFV_SYM(CommAbort);
    SFV_SYM(GetErrorString);
#undef SFV_SYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Send && n.Recv && n.GroupStart && n.GroupEnd &&
           n.AllReduce && n.Broadcast && n.CommGetAsyncError && n.CommAbort && n.GetErrorString;
    return n;
}

// A neighbour's state buffers and inbound flags as this process sees them
// (its own pointers in loopback mode, CUDA-IPC mappings across ranks).
struct PeerView {
    double *buf[4] = {nullptr, nullptr, nullptr, nullptr};
    unsigned long long *flags = nullptr;
    double *grad = nullptr;  // Navier-Stokes: the neighbour's gradient frame (pitch nj + 2)
    int PJ = 0, ni = 0, nj = 0;
};

// 128-byte descriptor one rank publishes for device-initiated halo exchange
// (sfv_peer_handle / sfv_peer_connect).
struct PeerHandle {
    cudaIpcMemHandle_t ipc;      // the allocation containing the workspace
    int64_t ws_off;              // workspace offset in that allocation
    int64_t flags_off;           // block's inbound flags, offset in the workspace
    int64_t buf_off[4];          // state buffers, offsets in the workspace
    int32_t ni, nj, PJ, block;
};
static_assert(sizeof(PeerHandle) == 128, "PeerHandle must be 128 bytes");

struct Block {
    int id = 0, bx = 0, by = 0;
    int i0 = 0, i1 = 0, j0 = 0, j1 = 0, ni = 0, nj = 0, PJ = 0;
    int nbr[4] = {-1, -1, -1, -1};
    int edge[4] = {0, 0, 0, 0};  // Edge kind per W, E, S, N
    int nstrips = 1, nseg = 1, nsegF = 1;
    // launch plan of a stage: edge rows first (2 rows per connected i-cut,
    // exchanged while the interior runs), then the interior rows
    int nlaunch = 1, row_lo[3] = {0, 0, 0}, row_hi[3] = {0, 0, 0}, lseg[3] = {1, 1, 1}, lbase[3] = {0, 0, 0};
    int lsegF[3] = {1, 1, 1};  // segments per launch part for the RK4 final stage (its own occupancy)
    // trailing short segments of a single-wave launch, per
    // occupancy class (0: main, 1: RK4 final stage): nstrips x tseg2 tasks over rows [tsplit, ni)
    int tseg2[2] = {0, 0}, tsplit[2] = {0, 0};
    int ncta_total = 1;
    bool split = false;
    double *buf[4] = {nullptr, nullptr, nullptr, nullptr};
    double *met = nullptr, *nodes = nullptr, *stage = nullptr, *partials = nullptr;
    double *xs[2] = {nullptr, nullptr}, *xr[2] = {nullptr, nullptr};  // j-cut pack buffers (S, N)
    unsigned long long *flags = nullptr;  // inbound halo flags [4 * FLAG_STRIDE] (peer mode)
    unsigned *ecnt = nullptr;             // writer arrival counters [4 * CNT_STRIDE]
    PeerView pv[4];                       // neighbour per edge (peer mode)
    double *grad = nullptr, *rv = nullptr;  // Navier-Stokes: gradients (1-layer ghost frame), viscous residual
    double *resb = nullptr;                 // sfv_residual output (state layout)
    int PG = 0;
    CUtensorMap tm_buf[4], tm_met;  // 2D TMA descriptors (made at sfv_bind)
    size_t buf_elems() const { return (size_t)(ni + 4) * 4 * PJ + PADD; }
    size_t met_elems() const { return (size_t)(ni + 1) * NMET * PJ + PADD; }
};

int nbuf_of(int rk) { return rk == SFV_RK4_CLASSIC ? 4 : (rk == SFV_RK2_HEUN ? 2 : 3); }
int nstages_of(int rk) { return rk == SFV_RK2_HEUN ? 2 : 4; }

struct StageSpec {
    int in, out, mode;
    double coef;
    int pw[3];
};
// Data flow of each tableau (reading A-R5).  Algebraically
// equal to Eq. 6: RK4's last stage recovers sum b_j R_j from the stored
// stage states, U^{n+1} = U^n + ((W2-U^n) + 2(W3-U^n) + (W4-U^n))/3 - dt R4/(6V).
StageSpec stage_spec(int rk, int k) {
    if (rk == SFV_RK4_CLASSIC) {
        switch (k) {
            case 1: return {0, 1, M_OWN, 0.5, {-1, -1, -1}};
            case 2: return {1, 2, M_UN, 0.5, {0, -1, -1}};
            case 3: return {2, 3, M_UN, 1.0, {0, -1, -1}};
            default: return {3, 0, M_RK4F, 1.0 / 6.0, {0, 1, 2}};
        }
    }
    if (rk == SFV_RK2_HEUN) {
        if (k == 1) return {0, 1, M_OWN, 1.0, {-1, -1, -1}};
        return {1, 0, M_HEUNF, 0.5, {0, -1, -1}};
    }
    switch (k) {  // Jameson 4-stage, alpha = 1/4, 1/3, 1/2, 1
        case 1: return {0, 1, M_OWN, 0.25, {-1, -1, -1}};
        case 2: return {1, 2, M_UN, 1.0 / 3.0, {0, -1, -1}};
        case 3: return {2, 1, M_UN, 0.5, {0, -1, -1}};
        default: return {1, 0, M_UN, 1.0, {0, -1, -1}};
    }
}

}  // namespace

enum ProfClass { P_EDGE = 0, P_INTERIOR, P_XROW, P_XCOL, P_WAIT, P_DT, P_VISC, P_NORMS, NPROF };

struct sfv_ctx {
    sfv_config cfg{};
    std::vector<double> X, Y;
    int px = 1, py = 1;
    std::vector<int> xs, ys;
    int rank = 0, nranks = 1, device = 0;
    bool partitioned = false, bound = false, have_state = false;
    std::vector<Block> blocks;  // local blocks
    int nblocks_total = 1;
    uint8_t *ws = nullptr;
    size_t ws_bytes = 0;
    cudaStream_t st = nullptr;
    double *sig = nullptr;
    long long *step_ctr = nullptr;
    unsigned *done = nullptr;
    int pring = 1;  // steps of norm partials kept before a batched reduction
    unsigned long long *err = nullptr, *geo_bad = nullptr;
    double *dt_hist = nullptr, *norm_hist = nullptr, *gbuf = nullptr;
    size_t gbuf_elems = 0;
    int nsm = 148, occ = 1, occ_f = 1;  // resident stage-kernel CTAs per SM (RK4 final stage: occ_f)
    Params P{};
    long long steps_enq = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaStream_t comm_st = nullptr;                  // halo exchange stream (overlap)
    cudaEvent_t ev_edge = nullptr, ev_comm = nullptr;
    bool timing_open = false;
    cudaGraphExec_t gexec = nullptr, gexec_norms = nullptr;  // step; step + norms batch
    bool graph_failed = false;
    ncclComm_t comm = nullptr;
    int halo = SFV_HALO_COPY;                // halo-exchange mode
    bool peer_ready = false;                 // sfv_peer_connect done (nranks > 1)
    unsigned *halo_err = nullptr;            // sticky peer-wait timeout
    std::vector<void *> ipc_open;            // CUDA-IPC mappings to close
    bool sig_dev = false;                    // dt max across ranks through peer memory (peer mode)
    double *sig_tab = nullptr;               // [2][SIG_RANKS_MAX]
    unsigned long long *sig_flag = nullptr;  // [SIG_RANKS_MAX]
    double **rtab = nullptr;                 // device array [nranks]
    unsigned long long **rflag = nullptr;    // device array [nranks]
    // failure detection of the NCCL path (a missing neighbour
    // message beyond a configurable timeout is a deadlock error naming the
    // edge): one event per enqueued step marks progress; a synchronising call
    // that sees no step complete for comm_timeout seconds (or an NCCL async
    // error) aborts the communicator and returns SFV_ERR_NCCL
    double comm_timeout = 60.0;
    bool comm_dead = false;
    std::deque<std::pair<cudaEvent_t, long long>> prog;  // (event, step index) in stream order
    std::vector<cudaEvent_t> ev_pool;
    // profiling mode (sfv_set_profiling): steps enqueued stage by stage with
    // CUDA events around each class of work (edge / interior stage kernels,
    // row exchange on the comm stream, column exchange, exposed wait for the
    // comm stream, dt all-reduce, viscous kernels, norms batch)
    bool prof = false;
    struct Span { int cls; cudaEvent_t a, b; };
    std::vector<Span> spans;
    std::vector<cudaEvent_t> tev_pool;
    double prof_ms[NPROF] = {0};
    long long prof_steps = 0;
    std::string msg;
    long long einfo[4] = {-1, -1, -1, -1};
};

namespace {

sfv_status fail(sfv_ctx *c, sfv_status s, const char *fmt, ...) {
    if (c) {
        char b[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(b, sizeof b, fmt, ap);
        va_end(ap);
        c->msg = b;
    }
    return s;
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return fail(c, SFV_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)
#define NK(call)                                                                                   \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess) return fail(c, SFV_ERR_NCCL, "%s: %s", #call, nccl().GetErrorString(r_)); \
    } while (0)

// Largest-remainder split (reading A-R24).
sfv_status split_impl(int32_t n, int32_t parts, const int32_t *w, int32_t *starts) {
    if (parts < 1 || n < 1) return SFV_ERR_ARG;
    long long sw = 0;
    for (int r = 0; r < parts; ++r) {
        long long x = w ? w[r] : 1;
        if (x <= 0) return SFV_ERR_ARG;
        sw += x;
    }
    std::vector<long long> base(parts), rem(parts);
    long long used = 0;
    for (int r = 0; r < parts; ++r) {
        long long x = w ? w[r] : 1;
        base[r] = (long long)n * x / sw;
        rem[r] = (long long)n * x % sw;
        used += base[r];
    }
    std::vector<int> order(parts);
    for (int r = 0; r < parts; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rem[a] > rem[b]; });
    for (long long k = 0; k < n - used; ++k) base[order[k]] += 1;
    sfv_status s = SFV_OK;
    starts[0] = 0;
    for (int r = 0; r < parts; ++r) {
        if (base[r] < 2) s = SFV_ERR_ARG;
        starts[r + 1] = starts[r] + (int32_t)base[r];
    }
    return s;
}

size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

int pitch_of(int nj) { return ((nj + JOFF + 2 + 15) / 16) * 16; }

void build_params(sfv_ctx *c) {
    const sfv_config &f = c->cfg;
    Params &P = c->P;
    P.gamma = f.gamma;
    P.gm1 = f.gamma - 1.0;
    P.c1 = f.muscl_eps * (1.0 - f.muscl_kappa) / 4.0;
    P.c2 = f.muscl_eps * (1.0 + f.muscl_kappa) / 4.0;
    P.delta = f.lim_delta;
    P.c1h = P.c1;
    P.c1dh = 0.5 * P.c1 * f.lim_delta;
    P.heps = f.harten_eps;
    P.hinv = f.harten_eps > 0.0 ? 0.5 / f.harten_eps : 0.0;
    P.cfl = f.cfl;
    P.dt_fixed = f.dt_fixed;
    P.limiter = f.limiter;
    P.mu = f.viscous ? f.mu : 0.0;
    P.rgas = f.gas_R > 0.0 ? f.gas_R : 287.0;
    P.rgas_inv = 1.0 / P.rgas;
    P.visc_dt = f.viscous ? 4.0 * std::max(4.0 / 3.0, f.gamma) * f.mu / f.prandtl : 0.0;
    P.kcond = f.viscous ? f.mu * (f.gamma * P.rgas / (f.gamma - 1.0)) / f.prandtl : 0.0;
}

// Launch geometry: strips of <= NT-4 columns (even starts), segments along i
// so that strips*segments fills the device in whole waves.
int choose_nseg(const sfv_ctx *c, const Block &b, int occ) {
    const int slots = c->nsm * std::max(1, occ) * WPC;  // resident warps
    // minimise (longest segment + prologue) x waves: a segment's time is its
    // row count plus ~1.5 rows of prologue / pipeline fill, and a launch lasts
    // as long as its longest segment in each wave
    int best = 1;
    double best_cost = 1e300;
    const int cap = std::min(NSEG_MAX, std::max(1, b.ni / 4));
    for (int s = 1; s <= cap; ++s) {
        const double rows = std::ceil((double)b.ni / s);
        const double waves = std::ceil((double)b.nstrips * s / slots);
        const double cost = (rows + 1.5) * waves;
        if (cost <= best_cost + 1e-9) {  // ties: more segments (less contention per SM)
            best_cost = cost;
            best = s;
        }
    }
    int nseg = std::min(best, b.ni);
    // experiment override: SFV_WAVES = w forces about w waves of warp tasks
    if (const char *ev = getenv("SFV_WAVES")) {
        const double w = atof(ev);
        if (w > 0) nseg = std::max(1, std::min(cap, (int)std::lround(w * slots / b.nstrips)));
    }
    return nseg;
}
// Launch geometry of a block: warp tasks = strips x segments, one segment
// count per occupancy class (the RK4 final stage keeps fewer resident warps
// than the other stage kernels)
void choose_launch(sfv_ctx *c, Block &b) {
    b.nstrips = (b.nj + WOUT - 1) / WOUT;
    b.nseg = choose_nseg(c, b, c->occ);
    b.nsegF = choose_nseg(c, b, c->occ_f);
}

// Stage launch plan of a block: with a connected i-cut and
// overlap enabled, the 2 edge rows at each cut are computed first so their
// exchange overlaps the interior launch.
void plan_launches(sfv_ctx *c, Block &b) {
    const bool cw = b.nbr[0] >= 0, ce = b.nbr[1] >= 0;
    const char *ov = getenv("SFV_OVERLAP");
    const bool overlap = !(ov && ov[0] == '0');
    // peer mode: one launch per stage; the edge tasks store into the
    // neighbours' ghost frames themselves
    b.split = overlap && (cw || ce) && b.ni >= 8 && c->halo != SFV_HALO_PEER && !c->cfg.viscous;
    int n = 0;
    int lo = 0, hi = b.ni;
    if (b.split) {
        if (cw) { b.row_lo[n] = 0; b.row_hi[n] = 2; b.lseg[n] = b.lsegF[n] = 1; ++n; lo = 2; }
        if (ce) { b.row_lo[n] = b.ni - 2; b.row_hi[n] = b.ni; b.lseg[n] = b.lsegF[n] = 1; ++n; hi = b.ni - 2; }
        // interior: re-run the segment choice on the interior rows
        Block t = b;
        t.ni = hi - lo;
        choose_launch(c, t);
        b.row_lo[n] = lo; b.row_hi[n] = hi; b.lseg[n] = t.nseg; b.lsegF[n] = t.nsegF; ++n;
    } else {
        b.row_lo[0] = 0; b.row_hi[0] = b.ni; b.lseg[0] = b.nseg; b.lsegF[0] = b.nsegF; n = 1;
    }
    b.nlaunch = n;
    int base = 0;
    for (int q = 0; q < n; ++q) {
        b.lbase[q] = base;
        base += (b.nstrips * b.lseg[q] + WPC - 1) / WPC;
    }
    b.ncta_total = base;
    b.nseg = b.lseg[n - 1];
    // trailing short segments (single launch, single wave): the first wave's
    // segments cover rows [0, tsplit); the last SFV_TAIL_FRAC of the rows go
    // into segments of ~SFV_TAIL_ROWS rows that the CTA scheduler places in
    // the slots of the first warps to finish
    const char *ef = getenv("SFV_TAIL_FRAC"), *er = getenv("SFV_TAIL_ROWS");
    const char *emf = getenv("SFV_TAIL_MFRAC"), *emr = getenv("SFV_TAIL_MROWS");
    for (int q = 0; q < 2; ++q) {
        b.tseg2[q] = 0;
        b.tsplit[q] = b.ni;
        const int nseg = q ? b.lsegF[0] : b.lseg[0];
        const long long slots = (long long)c->nsm * std::max(1, q ? c->occ_f : c->occ) * WPC;
        const bool single = (long long)b.nstrips * nseg <= slots;
        // single wave: the measured optimum on C2 (profiles/r2b_ab_tail_segments.txt);
        // multi-wave launches (the scheduler refills slots already): the last wave only
        const double frac = single ? (ef ? atof(ef) : 0.10) : (emf ? atof(emf) : 0.04);
        const int trows = std::max(2, single ? (er ? atoi(er) : 4) : (emr ? atoi(emr) : 16));
        const int tail = (int)std::lround(frac * b.ni);
        if (n != 1 || frac <= 0.0 || tail < 2 * trows || b.ni - tail < 4 * nseg)
            continue;
        b.tseg2[q] = std::min(tail / trows, NSEG_MAX - nseg);
        b.tsplit[q] = b.tseg2[q] > 0 ? b.ni - tail : b.ni;
    }
    b.ncta_total = std::max(b.ncta_total, b.nstrips * (b.lseg[0] + b.tseg2[0]));
}

sfv_status build_blocks(sfv_ctx *c) {
    c->blocks.clear();
    const int nb = c->px * c->py;
    c->nblocks_total = nb;
    for (int id = 0; id < nb; ++id) {
        if (c->nranks > 1 && id != c->rank) continue;
        Block b;
        b.id = id;
        b.bx = id % c->px;
        b.by = id / c->px;
        b.i0 = c->xs[b.bx];
        b.i1 = c->xs[b.bx + 1];
        b.j0 = c->ys[b.by];
        b.j1 = c->ys[b.by + 1];
        b.ni = b.i1 - b.i0;
        b.nj = b.j1 - b.j0;
        b.PJ = pitch_of(b.nj);
        b.nbr[0] = b.bx > 0 ? id - 1 : -1;
        b.nbr[1] = b.bx < c->px - 1 ? id + 1 : -1;
        b.nbr[2] = b.by > 0 ? id - c->px : -1;
        b.nbr[3] = b.by < c->py - 1 ? id + c->px : -1;
        for (int e = 0; e < 4; ++e) b.edge[e] = b.nbr[e] >= 0 ? E_CONNECTED : c->cfg.bc[e];
        b.nstrips = (b.nj + WOUT - 1) / WOUT;
        b.nseg = 1;
        c->blocks.push_back(b);
    }
    return SFV_OK;
}

size_t layout(sfv_ctx *c, bool assign) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += al(bytes);
        return o;
    };
    const int cap = (int)c->cfg.max_history;
    const int nbuf = nbuf_of(c->cfg.rk);
    c->pring = std::min(32, cap);
    size_t o_misc = take(MISC_BYTES);
    size_t o_dt = take(sizeof(double) * cap);
    size_t o_norm = take(sizeof(double) * (size_t)cap * c->nblocks_total * 8);
    size_t gb = 0;
    if (c->nranks > 1) {  // get_state's per-block broadcast, get_residual_norms' chunked all-reduce
        size_t big = 0;
        for (int bx = 0; bx < c->px; ++bx)
            for (int by = 0; by < c->py; ++by)
                big = std::max(big, (size_t)(c->xs[bx + 1] - c->xs[bx]) * (c->ys[by + 1] - c->ys[by]) * 4);
        gb = std::max(big, (size_t)c->nblocks_total * 8 * 4096);
    }
    size_t o_g = take(sizeof(double) * gb);
    if (assign) {
        c->sig = reinterpret_cast<double *>(c->ws + o_misc);
        c->step_ctr = reinterpret_cast<long long *>(c->ws + o_misc + 16);
        c->err = reinterpret_cast<unsigned long long *>(c->ws + o_misc + 24);
        c->geo_bad = reinterpret_cast<unsigned long long *>(c->ws + o_misc + 32);
        c->done = reinterpret_cast<unsigned *>(c->ws + o_misc + 40);
        c->halo_err = reinterpret_cast<unsigned *>(c->ws + o_misc + 48);
        c->sig_tab = reinterpret_cast<double *>(c->ws + o_misc + MISC_SIGTAB);
        c->sig_flag = reinterpret_cast<unsigned long long *>(c->ws + o_misc + MISC_SIGFLAG);
        c->rtab = reinterpret_cast<double **>(c->ws + o_misc + MISC_RTAB);
        c->rflag = reinterpret_cast<unsigned long long **>(c->ws + o_misc + MISC_RFLAG);
        c->dt_hist = reinterpret_cast<double *>(c->ws + o_dt);
        c->norm_hist = reinterpret_cast<double *>(c->ws + o_norm);
        c->gbuf = gb ? reinterpret_cast<double *>(c->ws + o_g) : nullptr;
        c->gbuf_elems = gb;
    }
    for (Block &b : c->blocks) {
        size_t ob[4];
        for (int k = 0; k < nbuf; ++k) ob[k] = take(sizeof(double) * b.buf_elems());
        size_t om = take(sizeof(double) * b.met_elems());
        size_t on = take(sizeof(double) * 2 * (size_t)(b.ni + 1) * (b.nj + 1));
        size_t os = take(sizeof(double) * 4 * (size_t)b.ni * b.nj);
        const int max_cta = (((b.nj + WOUT - 1) / WOUT) * (NSEG_MAX + 2) + WPC - 1) / WPC + 2;
        size_t op = take(sizeof(double) * 8 * (size_t)max_cta * c->pring);
        size_t of = take(PEER_SYNC_BYTES);
        const int PG = b.nj + 2;
        size_t og = take(c->cfg.viscous ? sizeof(double) * (size_t)(b.ni + 2) * 6 * PG : 0);
        size_t orv = take(c->cfg.viscous ? sizeof(double) * b.buf_elems() : 0);
        size_t ors = take(sizeof(double) * b.buf_elems());
        size_t ox[4];
        for (int k = 0; k < 4; ++k) ox[k] = take(c->nranks > 1 ? sizeof(double) * 8 * (size_t)b.ni : 0);
        if (assign) {
            for (int k = 0; k < nbuf; ++k) b.buf[k] = reinterpret_cast<double *>(c->ws + ob[k]);
            b.met = reinterpret_cast<double *>(c->ws + om);
            b.nodes = reinterpret_cast<double *>(c->ws + on);
            b.stage = reinterpret_cast<double *>(c->ws + os);
            b.partials = reinterpret_cast<double *>(c->ws + op);
            b.xs[0] = reinterpret_cast<double *>(c->ws + ox[0]);
            b.xs[1] = reinterpret_cast<double *>(c->ws + ox[1]);
            b.xr[0] = reinterpret_cast<double *>(c->ws + ox[2]);
            b.xr[1] = reinterpret_cast<double *>(c->ws + ox[3]);
            b.flags = reinterpret_cast<unsigned long long *>(c->ws + of);
            b.ecnt = reinterpret_cast<unsigned *>(c->ws + of + PEER_ECNT_OFF);
            b.PG = PG;
            b.grad = c->cfg.viscous ? reinterpret_cast<double *>(c->ws + og) : nullptr;
            b.rv = c->cfg.viscous ? reinterpret_cast<double *>(c->ws + orv) : nullptr;
            b.resb = reinterpret_cast<double *>(c->ws + ors);
        }
    }
    return off;
}

// Halo plan of a block in global cell indices (see sfv_halo_plan).
struct EdgePlan {
    int nbr, si0, si1, sj0, sj1, ri0, ri1, rj0, rj1;
};
void halo_plan(const sfv_ctx *c, int id, EdgePlan p[4]) {
    const int bx = id % c->px, by = id / c->px;
    const int i0 = c->xs[bx], i1 = c->xs[bx + 1], j0 = c->ys[by], j1 = c->ys[by + 1];
    const int nb[4] = {bx > 0 ? id - 1 : -1, bx < c->px - 1 ? id + 1 : -1, by > 0 ? id - c->px : -1,
                       by < c->py - 1 ? id + c->px : -1};
    p[0] = {nb[0], i0, i0 + 2, j0, j1, i0 - 2, i0, j0, j1};
    p[1] = {nb[1], i1 - 2, i1, j0, j1, i1, i1 + 2, j0, j1};
    p[2] = {nb[2], i0, i1, j0, j0 + 2, i0, i1, j0 - 2, j0};
    p[3] = {nb[3], i0, i1, j1 - 2, j1, i0, i1, j1, j1 + 2};
    for (int e = 0; e < 4; ++e)
        if (nb[e] < 0) p[e] = {-1, 0, 0, 0, 0, 0, 0, 0, 0};
}

Block *local_block(sfv_ctx *c, int id) {
    for (Block &b : c->blocks)
        if (b.id == id) return &b;
    return nullptr;
}

// Halo exchange of state buffer k after a stage ("boundary
// data exchange"; reading A-R16/A-R18: 2 layers, face neighbours only).
// i-cuts: the 2 edge rows are one contiguous run in the [i][c][j] layout;
// j-cuts: 2 columns, strided.
// Halo exchange of state buffer k after a stage ("boundary
// data exchange"; reading A-R16/A-R18: 2 layers, face neighbours only).
// i-cuts (rows): the 2 edge rows are one contiguous run in the [i][c][j]
// layout (zero-copy); j-cuts (columns): strided, packed for NCCL.
sfv_status exchange_rows(sfv_ctx *c, int k, cudaStream_t st) {
    if (c->px == 1) return SFV_OK;
    if (c->nranks == 1) {
        for (Block &b : c->blocks) {
            if (b.nbr[1] >= 0) {  // E neighbour e: b rows ni-2,ni-1 -> e rows -2,-1; e rows 0,1 -> b rows ni,ni+1
                Block &e = *local_block(c, b.nbr[1]);
                const size_t run = (size_t)2 * 4 * b.PJ;
                CK(cudaMemcpyAsync(e.buf[k], b.buf[k] + (size_t)(b.ni) * 4 * b.PJ, run * 8, cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpyAsync(b.buf[k] + (size_t)(b.ni + 2) * 4 * b.PJ, e.buf[k] + (size_t)2 * 4 * e.PJ, run * 8,
                                   cudaMemcpyDeviceToDevice, st));
            }
        }
        return SFV_OK;
    }
    // NCCL: one block per rank (block id == rank); executes halo_plan()'s i-cuts.
    Block &b = c->blocks[0];
    Nccl &N = nccl();
    EdgePlan p[4];
    halo_plan(c, b.id, p);
    NK(N.GroupStart());
    const size_t run = (size_t)2 * 4 * b.PJ;  // 2 rows x 4 comps x pitch: contiguous in [i][c][j]
    for (int e = 0; e < 2; ++e) {
        const EdgePlan &q = p[e];
        if (q.nbr < 0) continue;
        NK(N.Send(b.buf[k] + (size_t)(q.si0 - b.i0 + 2) * 4 * b.PJ, run, ncclDouble, q.nbr, c->comm, st));
        NK(N.Recv(b.buf[k] + (size_t)(q.ri0 - b.i0 + 2) * 4 * b.PJ, run, ncclDouble, q.nbr, c->comm, st));
    }
    NK(N.GroupEnd());
    return SFV_OK;
}

sfv_status exchange_cols(sfv_ctx *c, int k, cudaStream_t st) {
    if (c->py == 1) return SFV_OK;
    if (c->nranks == 1) {
        for (Block &b : c->blocks) {
            if (b.nbr[3] >= 0) {  // N neighbour: b cols nj-2,nj-1 -> n cols -2,-1; n cols 0,1 -> b cols nj,nj+1
                Block &n = *local_block(c, b.nbr[3]);
                CK(cudaMemcpy2DAsync(n.buf[k] + (size_t)8 * n.PJ + (-2 + JOFF), (size_t)n.PJ * 8,
                                     b.buf[k] + (size_t)8 * b.PJ + (b.nj - 2 + JOFF), (size_t)b.PJ * 8, 16,
                                     (size_t)b.ni * 4, cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpy2DAsync(b.buf[k] + (size_t)8 * b.PJ + (b.nj + JOFF), (size_t)b.PJ * 8,
                                     n.buf[k] + (size_t)8 * n.PJ + (0 + JOFF), (size_t)n.PJ * 8, 16,
                                     (size_t)n.ni * 4, cudaMemcpyDeviceToDevice, st));
            }
        }
        return SFV_OK;
    }
    Block &b = c->blocks[0];
    Nccl &N = nccl();
    EdgePlan p[4];
    halo_plan(c, b.id, p);
    for (int s = 0; s < 2; ++s) {  // pack the 2 send columns
        const EdgePlan &q = p[2 + s];
        if (q.nbr < 0) continue;
        CK(launch_pack_cols(b.buf[k], b.xs[s], b.ni, b.PJ, q.sj0 - b.j0, st));
    }
    NK(N.GroupStart());
    for (int s = 0; s < 2; ++s) {
        const EdgePlan &q = p[2 + s];
        if (q.nbr < 0) continue;
        NK(N.Send(b.xs[s], (size_t)8 * b.ni, ncclDouble, q.nbr, c->comm, st));
        NK(N.Recv(b.xr[s], (size_t)8 * b.ni, ncclDouble, q.nbr, c->comm, st));
    }
    NK(N.GroupEnd());
    for (int s = 0; s < 2; ++s) {
        const EdgePlan &q = p[2 + s];
        if (q.nbr < 0) continue;
        CK(launch_unpack_cols(b.xr[s], b.buf[k], b.ni, b.PJ, q.rj0 - b.j0, st));
    }
    return SFV_OK;
}

sfv_status exchange(sfv_ctx *c, int k, cudaStream_t st) {
    sfv_status r = exchange_rows(c, k, st);
    if (r != SFV_OK) return r;
    return exchange_cols(c, k, st);
}

StageArgs make_args(sfv_ctx *c, Block &b, int k) {
    const StageSpec sp = stage_spec(c->cfg.rk, k);
    StageArgs a{};
    a.tm_in = b.tm_buf[sp.in];
    a.tm_met = b.tm_met;
    for (int q = 0; q < 3; ++q) a.tm_pw[q] = b.tm_buf[sp.pw[q] >= 0 ? sp.pw[q] : sp.in];
    a.in = b.buf[sp.in];
    a.out = b.buf[sp.out];
    a.pw0 = sp.pw[0] >= 0 ? b.buf[sp.pw[0]] : nullptr;
    a.pw1 = sp.pw[1] >= 0 ? b.buf[sp.pw[1]] : nullptr;
    a.pw2 = sp.pw[2] >= 0 ? b.buf[sp.pw[2]] : nullptr;
    a.met = b.met;
    a.ni = b.ni;
    a.nj = b.nj;
    a.PJ = b.PJ;
    a.gi0 = b.i0;
    a.gj0 = b.j0;
    a.NI = c->cfg.ni;
    a.NJ = c->cfg.nj;
    a.nstrips = b.nstrips;
    a.nseg = b.nseg;
    a.row_lo = 0;
    a.row_hi = b.ni;
    a.row_split = b.ni;
    a.nseg2 = 0;
    a.part_base = 0;
    a.part_stride = b.ncta_total;
    for (int e = 0; e < 4; ++e) a.bc[e] = b.edge[e];
    a.coef = sp.coef;
    a.sig = c->sig;
    a.step_ctr = c->step_ctr;
    a.dt_hist = c->dt_hist;
    a.norm_hist = c->norm_hist;
    a.cap = (int)c->cfg.max_history;
    a.block_id = b.id;
    a.nblocks = c->nblocks_total;
    a.partials = b.partials;
    a.pring = c->pring;
    a.done = c->done;
    a.bump = 0;
    a.err = c->err;
    a.stage = k;
    a.nstages = nstages_of(c->cfg.rk);
    a.P = c->P;
    if (c->halo == SFV_HALO_PEER) {
        static const int opp[4] = {1, 0, 3, 2};
        for (int e = 0; e < 4; ++e) {
            const PeerView &v = b.pv[e];
            if (b.nbr[e] < 0 || !v.flags) continue;
            a.peer_out[e] = v.buf[sp.out];
            a.peer_flag[e] = v.flags + opp[e] * FLAG_STRIDE;
            a.peer_PJ[e] = v.PJ;
            a.peer_n[e] = e == 0 ? v.ni : (e == 2 ? v.nj : 0);
        }
        a.in_flag = b.flags;
        a.edge_cnt = b.ecnt;
        a.halo_err = c->halo_err;
        if (c->sig_dev) {
            a.sig_ranks = c->nranks;
            a.rank = c->rank;
            a.sig_tab = c->sig_tab;
            a.sig_flag = c->sig_flag;
            a.rtab = c->rtab;
            a.rflag = c->rflag;
        }
    }
    a.rv = c->cfg.viscous ? b.rv : nullptr;
    return a;
}

// Navier-Stokes: gradients of every block's stage input, physical-edge ghost
// gradients, loopback exchange of the connected ones (1 layer: rows for
// i-cuts, columns for j-cuts), then every block's viscous residual
// (readings N-R1..N-R3)
// stage > 0 in peer mode: device-initiated gradient halos (grad_kernel stores
// its edge gradients into the neighbours' frames and signals; visc_kernel's
// edge CTAs wait), no copies; stage 0 (sfv_residual): copy exchange.
sfv_status enqueue_viscous(sfv_ctx *c, int in, cudaStream_t st, int stage = 0) {
    const bool peer = stage > 0 && c->halo == SFV_HALO_PEER;
    auto args = [&](Block &b) {
        ViscArgs v{};
        if (peer) {
            static const int opp[4] = {1, 0, 3, 2};
            v.peer = 1;
            for (int e = 0; e < 4; ++e) {
                const PeerView &pv = b.pv[e];
                if (b.nbr[e] < 0 || !pv.grad) continue;
                v.peer_grad[e] = pv.grad;
                v.peer_PG[e] = pv.nj + 2;
                v.peer_n[e] = e == 0 ? pv.ni : (e == 2 ? pv.nj : 0);
                v.peer_gflag[e] = pv.flags + PEER_GFLAG_OFF / 8 + opp[e] * FLAG_STRIDE;
                v.gwriters[e] = e < 2 ? (b.nj + 127) / 128 : b.ni;  // grad_kernel's grid: (ceil(nj/128), ni)
            }
            v.in_flag = b.flags;
            v.in_gflag = b.flags + PEER_GFLAG_OFF / 8;
            v.gcnt = reinterpret_cast<unsigned *>(reinterpret_cast<uint8_t *>(b.flags) + PEER_GCNT_OFF);
            v.halo_err = c->halo_err;
            v.step_ctr = c->step_ctr;
            v.stage = stage;
            v.nstages = nstages_of(c->cfg.rk);
        }
        v.in = b.buf[in];
        v.met = b.met;
        v.grad = b.grad;
        v.rv = b.rv;
        v.ni = b.ni;
        v.nj = b.nj;
        v.PJ = b.PJ;
        v.PG = b.PG;
        for (int e = 0; e < 4; ++e) v.bc[e] = b.edge[e];
        v.P = c->P;
        return v;
    };
    const char *fv = getenv("SFV_NS_FUSED");
    const bool fuse_ok = !(fv && fv[0] == '0');
    bool all_fused = true;
    for (Block &b : c->blocks) {
        const bool iso = b.nbr[0] < 0 && b.nbr[1] < 0 && b.nbr[2] < 0 && b.nbr[3] < 0;
        if (iso && fuse_ok) {  // gradients never leave the SM (registers / shared memory)
            const char *em = getenv("SFV_NS_MARCH");
            if (em && em[0] == '0') CK(launch_gradvisc(args(b), st));
            else CK(launch_gradvisc_march(args(b), st));
        }
        else { CK(launch_grad(args(b), st)); all_fused = false; }  // (writes the physical ghost gradients too)
    }
    if (all_fused) return SFV_OK;
    if (peer) {  // every block's grads (and their peer stores) precede every visc in stream order
        for (Block &b : c->blocks) {
            const bool iso = b.nbr[0] < 0 && b.nbr[1] < 0 && b.nbr[2] < 0 && b.nbr[3] < 0;
            if (!(iso && fuse_ok)) CK(launch_visc(args(b), st));
        }
        return SFV_OK;
    }
    if (c->nranks > 1) {
        // NCCL: this rank's block; rows (i-cuts) straight from / into the frame,
        // columns (j-cuts) through the pack buffers
        Block &b = c->blocks[0];
        Nccl &N = nccl();
        const size_t rowd = (size_t)6 * b.PG;
        for (int sd = 0; sd < 2; ++sd)
            if (b.nbr[2 + sd] >= 0)
                CK(cudaMemcpy2DAsync(b.xs[sd], 8, b.grad + (size_t)6 * b.PG + (sd == 0 ? 1 : b.nj), (size_t)b.PG * 8,
                                     8, (size_t)b.ni * 6, cudaMemcpyDeviceToDevice, st));
        NK(N.GroupStart());
        if (b.nbr[0] >= 0) {
            NK(N.Send(b.grad + rowd, rowd, ncclDouble, b.nbr[0], c->comm, st));
            NK(N.Recv(b.grad, rowd, ncclDouble, b.nbr[0], c->comm, st));
        }
        if (b.nbr[1] >= 0) {
            NK(N.Send(b.grad + (size_t)b.ni * rowd, rowd, ncclDouble, b.nbr[1], c->comm, st));
            NK(N.Recv(b.grad + (size_t)(b.ni + 1) * rowd, rowd, ncclDouble, b.nbr[1], c->comm, st));
        }
        for (int sd = 0; sd < 2; ++sd)
            if (b.nbr[2 + sd] >= 0) {
                NK(N.Send(b.xs[sd], (size_t)6 * b.ni, ncclDouble, b.nbr[2 + sd], c->comm, st));
                NK(N.Recv(b.xr[sd], (size_t)6 * b.ni, ncclDouble, b.nbr[2 + sd], c->comm, st));
            }
        NK(N.GroupEnd());
        for (int sd = 0; sd < 2; ++sd)
            if (b.nbr[2 + sd] >= 0)
                CK(cudaMemcpy2DAsync(b.grad + (size_t)6 * b.PG + (sd == 0 ? 0 : b.nj + 1), (size_t)b.PG * 8, b.xr[sd],
                                     8, 8, (size_t)b.ni * 6, cudaMemcpyDeviceToDevice, st));
        CK(launch_visc(args(b), st));
        return SFV_OK;
    }
    for (Block &b : c->blocks) {
        const size_t rowd = (size_t)6 * b.PG;  // one i-row of the gradient frame
        if (b.nbr[1] >= 0) {  // E neighbour e: b row ni-1 -> e row -1; e row 0 -> b row ni
            Block &e = *local_block(c, b.nbr[1]);
            CK(cudaMemcpyAsync(e.grad, b.grad + (size_t)b.ni * rowd, rowd * 8, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(b.grad + (size_t)(b.ni + 1) * rowd, e.grad + rowd, rowd * 8, cudaMemcpyDeviceToDevice,
                               st));
        }
        if (b.nbr[3] >= 0) {  // N neighbour n: b column nj-1 -> n column -1; n column 0 -> b column nj
            Block &n = *local_block(c, b.nbr[3]);
            CK(cudaMemcpy2DAsync(n.grad + (size_t)6 * n.PG + 0, (size_t)n.PG * 8, b.grad + (size_t)6 * b.PG + b.nj,
                                 (size_t)b.PG * 8, 8, (size_t)b.ni * 6, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpy2DAsync(b.grad + (size_t)6 * b.PG + b.nj + 1, (size_t)b.PG * 8, n.grad + (size_t)6 * n.PG + 1,
                                 (size_t)n.PG * 8, 8, (size_t)n.ni * 6, cudaMemcpyDeviceToDevice, st));
        }
    }
    for (Block &b : c->blocks) {
        const bool iso = b.nbr[0] < 0 && b.nbr[1] < 0 && b.nbr[2] < 0 && b.nbr[3] < 0;
        if (!(iso && fuse_ok)) CK(launch_visc(args(b), st));
    }
    return SFV_OK;
}

// Tasks of a launch (nseg segments over all rows) that touch edge e: the same
// predicate as the stage kernel's `touch` (segments at i = 0 / ni; strip 0;
// strips whose columns reach nj - 1).
int edge_writers(const Block &b, int nseg, int e) {
    if (e < 2) return b.nstrips;
    int strips = 0;
    for (int s = 0; s < b.nstrips; ++s) {
        const int j0 = s * WOUT, j1 = std::min(j0 + WOUT, b.nj);
        strips += e == 2 ? (j0 == 0) : (j1 >= b.nj - 1);
    }
    return strips * nseg;
}

// Norm partials of `count` steps -> history, every local block (first < 0:
// the `count` steps before the device step counter).
sfv_status enqueue_norms(sfv_ctx *c, long long first, int count, cudaStream_t st) {
    for (Block &b : c->blocks) {
        NormsArgs f{};
        f.partials = b.partials;
        f.ncta = b.ncta_total;
        f.pring = c->pring;
        f.norm_hist = c->norm_hist;
        f.step_ctr = c->step_ctr;
        f.first = first;
        f.count = count;
        f.cap = (int)c->cfg.max_history;
        f.block_id = b.id;
        f.nblocks = c->nblocks_total;
        CK(launch_norms(f, st));
    }
    return SFV_OK;
}

// Profiling spans (active only in profiling mode, never inside graph capture).
int span_begin(sfv_ctx *c, int cls, cudaStream_t st) {
    if (!c->prof) return -1;
    auto get = [&]() {
        cudaEvent_t e = nullptr;
        if (!c->tev_pool.empty()) {
            e = c->tev_pool.back();
            c->tev_pool.pop_back();
        } else if (cudaEventCreate(&e) != cudaSuccess) {
            e = nullptr;
        }
        return e;
    };
    sfv_ctx::Span sp{cls, get(), get()};
    if (!sp.a || !sp.b || cudaEventRecord(sp.a, st) != cudaSuccess) return -1;
    c->spans.push_back(sp);
    return (int)c->spans.size() - 1;
}
void span_end(sfv_ctx *c, int id, cudaStream_t st) {
    if (id >= 0) cudaEventRecord(c->spans[id].b, st);
}
// after the stream has drained: accumulate and recycle
void spans_collect(sfv_ctx *c) {
    for (auto &sp : c->spans) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess) c->prof_ms[sp.cls] += ms;
        c->tev_pool.push_back(sp.a);
        c->tev_pool.push_back(sp.b);
    }
    c->spans.clear();
    cudaGetLastError();
}

sfv_status enqueue_step(sfv_ctx *c, cudaStream_t st, bool norms_batch) {
    const int s = nstages_of(c->cfg.rk);
    const bool cflmode = !(c->cfg.dt_fixed > 0.0);
    bool any_split = false;
    for (Block &b : c->blocks) any_split |= b.split;
    for (int k = 1; k <= s; ++k) {
        const StageSpec sp = stage_spec(c->cfg.rk, k);
        if (c->cfg.viscous) {
            const int sv = span_begin(c, P_VISC, st);
            sfv_status r = enqueue_viscous(c, sp.in, st, k);
            if (r != SFV_OK) return r;
            span_end(c, sv, st);
        }
        auto launch_part = [&](Block &b, int q) -> sfv_status {
            StageArgs a = make_args(c, b, k);
            // the step's last launch in stream order advances the step counter
            a.bump = (k == s && &b == &c->blocks.back() && q == b.nlaunch - 1) ? 1 : 0;
            a.row_lo = b.row_lo[q];
            a.row_hi = b.row_hi[q];
            a.nseg = sp.mode == M_RK4F ? b.lsegF[q] : b.lseg[q];
            {
                const int cls = sp.mode == M_RK4F ? 1 : 0;
                const bool tail = b.nlaunch == 1 && c->halo != SFV_HALO_PEER;
                a.nseg2 = tail ? b.tseg2[cls] : 0;
                a.row_split = a.nseg2 > 0 ? b.tsplit[cls] : a.row_hi;
            }
            a.part_base = b.lbase[q];
            for (int e = 0; e < 4; ++e) a.edge_writers[e] = a.peer_out[e] ? edge_writers(b, a.nseg, e) : 0;
            CK(launch_stage(a, sp.mode, k == 1, k == s && cflmode, c->halo == SFV_HALO_PEER, c->cfg.viscous != 0, st));
            return SFV_OK;
        };
        if (any_split) {
            // edge rows -> [comm stream: row exchange] || interior rows -> join
            const int se = span_begin(c, P_EDGE, st);
            for (Block &b : c->blocks)
                for (int q = 0; q + 1 < b.nlaunch; ++q) {
                    sfv_status r = launch_part(b, q);
                    if (r != SFV_OK) return r;
                }
            span_end(c, se, st);
            CK(cudaEventRecord(c->ev_edge, st));
            CK(cudaStreamWaitEvent(c->comm_st, c->ev_edge, 0));
            const int sx = span_begin(c, P_XROW, c->comm_st);
            sfv_status r = exchange_rows(c, sp.out, c->comm_st);
            if (r != SFV_OK) return r;
            span_end(c, sx, c->comm_st);
            CK(cudaEventRecord(c->ev_comm, c->comm_st));
            const int si = span_begin(c, P_INTERIOR, st);
            for (Block &b : c->blocks) {
                r = launch_part(b, b.nlaunch - 1);
                if (r != SFV_OK) return r;
            }
            span_end(c, si, st);
        } else {
            const int si = span_begin(c, P_INTERIOR, st);
            for (Block &b : c->blocks) {
                sfv_status r = launch_part(b, 0);
                if (r != SFV_OK) return r;
            }
            span_end(c, si, st);
        }
        if (c->halo == SFV_HALO_PEER) continue;  // the stage kernels exchanged the halos
        if (any_split) {
            const int sc = span_begin(c, P_XCOL, st);
            sfv_status r = exchange_cols(c, sp.out, st);
            if (r != SFV_OK) return r;
            span_end(c, sc, st);
            const int sw = span_begin(c, P_WAIT, st);  // compute stream idles until the rows arrived
            CK(cudaStreamWaitEvent(st, c->ev_comm, 0));
            span_end(c, sw, st);
        } else {
            bool connected = false;
            for (Block &b : c->blocks)
                for (int e = 0; e < 4; ++e) connected |= b.nbr[e] >= 0;
            const int sx = connected ? span_begin(c, P_XROW, st) : -1;
            sfv_status r = exchange(c, sp.out, st);
            if (r != SFV_OK) return r;
            span_end(c, sx, st);
        }
    }
    // dt max across ranks: in the bump CTA through peer memory (peer mode), else NCCL
    const bool dev_dt = c->halo == SFV_HALO_PEER && c->sig_dev;
    if (c->nranks > 1 && cflmode && !dev_dt) {
        const int sd = span_begin(c, P_DT, st);
        NK(nccl().AllReduce(c->sig, c->sig, 2, ncclDouble, ncclMax, c->comm, st));
        span_end(c, sd, st);
    }
    if (norms_batch) {
        const int sn = span_begin(c, P_NORMS, st);
        sfv_status r = enqueue_norms(c, -1, c->pring, st);
        span_end(c, sn, st);
        return r;
    }
    return SFV_OK;
}

// Neighbours of this rank's block, for error messages ("W: rank 1, E: rank 3").
std::string edge_names(const sfv_ctx *c) {
    static const char *nm[4] = {"W", "E", "S", "N"};
    std::string r;
    if (c->blocks.empty()) return r;
    for (int e = 0; e < 4; ++e)
        if (c->blocks[0].nbr[e] >= 0) {
            if (!r.empty()) r += ", ";
            r += std::string(nm[e]) + " edge <-> rank " + std::to_string(c->blocks[0].nbr[e]);
        }
    return r.empty() ? std::string("no connected edge") : r;
}

// Wait for the bound stream.  With NCCL ranks (copy-mode halos, all-reduces)
// the wait polls the stream, the per-step progress events and
// ncclCommGetAsyncError: an async error, or no step completing within
// comm_timeout seconds, aborts the communicator (unblocking the stream) and
// returns SFV_ERR_NCCL naming this rank's edges and the pending step
// instead of hanging.
// Abort the communicator after a failure: ncclCommAbort runs on a detached
// thread -- it unblocks the stream's NCCL kernels, but with a dead
// peer it may itself wait on the transport, and the caller must get its
// error within the timeout.  Bounded wait of 2 s for it here.
void abort_comm(sfv_ctx *c) {
    // (the step graphs stay: destroying an executable graph that still has
    // launches in flight behind the stalled exchange would block here)
    auto done = std::make_shared<std::atomic<bool>>(false);
    ncclComm_t comm = c->comm;
    std::thread([comm, done]() {
        nccl().CommAbort(comm);
        done->store(true);
    }).detach();
    for (int k = 0; k < 2000 && !done->load(); ++k) usleep(1000);
}

// Poll until the stream has drained (inflight < 0) or at most `inflight`
// tracked steps are still pending, watching NCCL's async error and progress.
sfv_status poll_wait(sfv_ctx *c, const char *what, long long inflight) {
    Nccl &N = nccl();
    using clk = std::chrono::steady_clock;
    auto last = clk::now();
    for (;;) {
        bool moved = false;
        while (!c->prog.empty() && cudaEventQuery(c->prog.front().first) == cudaSuccess) {
            c->ev_pool.push_back(c->prog.front().first);
            c->prog.pop_front();
            moved = true;
        }
        if (inflight >= 0) {
            if ((long long)c->prog.size() <= inflight) return SFV_OK;
        } else {
            const cudaError_t q = cudaStreamQuery(c->st);
            if (q == cudaSuccess) return SFV_OK;
            if (q != cudaErrorNotReady) return fail(c, SFV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(q));
        }
        if (moved) last = clk::now();
        ncclResult_t ar = ncclSuccess;
        N.CommGetAsyncError(c->comm, &ar);
        const double idle = std::chrono::duration<double>(clk::now() - last).count();
        if ((ar != ncclSuccess && ar != ncclInProgress) || idle > c->comm_timeout) {
            const long long pend = c->prog.empty() ? -1 : c->prog.front().second;
            const bool dbg = getenv("SFV_DEBUG_WAIT") != nullptr;
            if (dbg) fprintf(stderr, "[sfv] %s: async=%d idle=%.1fs pending step %lld: aborting\n", what, (int)ar, idle, pend);
            abort_comm(c);
            if (dbg) fprintf(stderr, "[sfv] %s: communicator abort issued\n", what);
            c->comm = nullptr;
            c->comm_dead = true;
            c->have_state = false;
            if (ar != ncclSuccess && ar != ncclInProgress)
                return fail(c, SFV_ERR_NCCL, "%s: NCCL async error '%s' on rank %d (%s), step %lld; communicator aborted",
                            what, N.GetErrorString(ar), c->rank, edge_names(c).c_str(), pend);
            return fail(c, SFV_ERR_NCCL,
                        "%s: deadlock: no progress for %.1f s on rank %d -- halo exchange / all-reduce with (%s) "
                        "pending at step %lld; communicator aborted",
                        what, c->comm_timeout, c->rank, edge_names(c).c_str(), pend);
        }
        usleep(inflight >= 0 ? 20 : 200);
    }
}

sfv_status wait_stream(sfv_ctx *c, const char *what) {
    if (c->comm_dead) return fail(c, SFV_ERR_NCCL, "%s: the NCCL communicator was aborted by an earlier failure", what);
    if (c->nranks <= 1 || !c->comm) {
        CK(cudaStreamSynchronize(c->st));
    } else {
        sfv_status r = poll_wait(c, what, -1);
        if (r != SFV_OK) return r;
    }
    for (auto &pe : c->prog) c->ev_pool.push_back(pe.first);
    c->prog.clear();
    if (!c->spans.empty()) {
        CK(cudaStreamSynchronize(c->comm_st));  // (joined into st: complete)
        spans_collect(c);
    }
    return SFV_OK;
}
#define SYNC(what)                                \
    do {                                          \
        sfv_status s_ = wait_stream(c, (what));   \
        if (s_ != SFV_OK) return s_;              \
    } while (0)

// With NCCL ranks every rank must take the same branch before a collective
// (an error one rank sees must not leave the others blocked in the next
// all-reduce): the sticky words are agreed over ranks -- the smallest error
// key (the global first failure: keys carry global cell indices) and the
// max of the halo-timeout flag.
sfv_status agree_errors(sfv_ctx *c) {
    if (c->nranks <= 1 || !c->comm) return SFV_OK;
    Nccl &N = nccl();
    NK(N.AllReduce(c->err, c->err, 1, ncclUint64, ncclMin, c->comm, c->st));
    NK(N.AllReduce(c->halo_err, c->halo_err, 1, ncclUint32, ncclMax, c->comm, c->st));
    SYNC("error agreement");
    return SFV_OK;
}

// Block <-> full-grid host array ([j][i][4]): one contiguous copy when the
// block spans the full width (single block, slabs along j), else a 2D copy.
cudaError_t copy_block_h2d(const Block &b, const double *U, int NI, cudaStream_t st) {
    const double *src = U + ((size_t)b.j0 * NI + b.i0) * 4;
    if (b.ni == NI) return cudaMemcpyAsync(b.stage, src, (size_t)b.ni * b.nj * 32, cudaMemcpyHostToDevice, st);
    return cudaMemcpy2DAsync(b.stage, (size_t)b.ni * 32, src, (size_t)NI * 32, (size_t)b.ni * 32, b.nj,
                             cudaMemcpyHostToDevice, st);
}
cudaError_t copy_block_d2h(const Block &b, double *U, int NI, cudaStream_t st) {
    double *dst = U + ((size_t)b.j0 * NI + b.i0) * 4;
    if (b.ni == NI) return cudaMemcpyAsync(dst, b.stage, (size_t)b.ni * b.nj * 32, cudaMemcpyDeviceToHost, st);
    return cudaMemcpy2DAsync(dst, (size_t)NI * 32, b.stage, (size_t)b.ni * 32, (size_t)b.ni * 32, b.nj,
                             cudaMemcpyDeviceToHost, st);
}

sfv_status check_device_error(sfv_ctx *c, bool collective = false) {
    if (collective) {
        sfv_status a = agree_errors(c);
        if (a != SFV_OK) return a;
    }
    if (c->halo == SFV_HALO_PEER || collective) {
        unsigned h = 0;
        CK(cudaMemcpy(&h, c->halo_err, sizeof h, cudaMemcpyDeviceToHost));
        if (h) {
            c->have_state = false;
            return fail(c, SFV_ERR_HALO, "device-initiated halo exchange: a neighbour did not signal within %llu s",
                        (unsigned long long)20);
        }
    }
    unsigned long long e = ~0ull;
    CK(cudaMemcpy(&e, c->err, sizeof e, cudaMemcpyDeviceToHost));
    if (e == ~0ull) return SFV_OK;
    const long long hi = (long long)(e >> 32), cell = (long long)(e & 0xffffffffull);
    const int s = nstages_of(c->cfg.rk);
    const long long q = hi / 2, phase = hi % 2;
    c->einfo[0] = q / s;
    c->einfo[1] = q % s + 1;
    c->einfo[2] = cell % c->cfg.ni;
    c->einfo[3] = cell / c->cfg.ni;
    c->have_state = false;
    return fail(c, SFV_ERR_STATE, "invalid %s at step %lld stage %lld cell (%lld,%lld)",
                phase ? "state (rho<=0 or p<=0)" : "face state", c->einfo[0], c->einfo[1], c->einfo[2],
                c->einfo[3]);
}

}  // namespace

// ======================================================================= ABI
extern "C" {

sfv_status sfv_split(int32_t n, int32_t parts, const int32_t *weights, int32_t *starts) {
    return split_impl(n, parts, weights, starts);
}

sfv_status sfv_create(const sfv_config *cfg, const double *x, const double *y, sfv_ctx **out) {
    if (!out || !cfg || !x || !y) return SFV_ERR_ARG;
    *out = nullptr;
    const sfv_config &f = *cfg;
    if (f.ni < 2 || f.nj < 2 || !(f.gamma > 1.0) || !(std::fabs(f.muscl_kappa) <= 1.0) ||
        !(f.muscl_eps == 0.0 || f.muscl_eps == 1.0) || (!(f.dt_fixed > 0.0) && !(f.cfl > 0.0)) ||
        f.max_history < 1 || f.rk < 0 || f.rk > 2 || f.limiter < 0 || f.limiter > 2 || !(f.lim_delta >= 0.0) ||
        !(f.harten_eps >= 0.0))
        return SFV_ERR_ARG;
    for (int e = 0; e < 4; ++e)
        if (f.bc[e] < 0 || f.bc[e] > 3 || (f.bc[e] == SFV_BC_NOSLIP_WALL && !f.viscous)) return SFV_ERR_ARG;
    if (f.viscous != 0 && f.viscous != 1) return SFV_ERR_ARG;
    if (f.viscous && !(f.mu >= 0.0 && f.prandtl > 0.0 && f.gas_R > 0.0)) return SFV_ERR_ARG;
    if ((long long)f.ni * f.nj >= (1ll << 31)) return SFV_ERR_UNSUPPORTED;
    sfv_ctx *c = new sfv_ctx();
    c->cfg = f;
    const size_t nn = (size_t)(f.ni + 1) * (f.nj + 1);
    c->X.assign(x, x + nn);
    c->Y.assign(y, y + nn);
    build_params(c);
    // volume check on the host (GEOMETRY error names the cell)
    const int W = f.ni + 1;
    for (int j = 0; j < f.nj; ++j)
        for (int i = 0; i < f.ni; ++i) {
            auto X = [&](int ii, int jj) { return c->X[(size_t)jj * W + ii]; };
            auto Y = [&](int ii, int jj) { return c->Y[(size_t)jj * W + ii]; };
            const double V = 0.5 * ((X(i + 1, j + 1) - X(i, j)) * (Y(i, j + 1) - Y(i + 1, j)) -
                                    (Y(i + 1, j + 1) - Y(i, j)) * (X(i, j + 1) - X(i + 1, j)));
            if (!(V > 0.0)) {
                c->einfo[0] = -1; c->einfo[1] = -1; c->einfo[2] = i; c->einfo[3] = j;
                *out = c;
                fail(c, SFV_ERR_GEOMETRY, "non-positive cell volume at (%d,%d)", i, j);
                return SFV_ERR_GEOMETRY;
            }
        }
    c->xs = {0, f.ni};
    c->ys = {0, f.nj};
    build_blocks(c);
    c->partitioned = true;
    *out = c;
    return SFV_OK;
}

sfv_status sfv_nccl_unique_id(void *out128) {
    if (!out128) return SFV_ERR_ARG;
    Nccl &N = nccl();
    if (!N.ok) return SFV_ERR_NCCL;
    ncclUniqueId id;
    if (N.GetUniqueId(&id) != ncclSuccess) return SFV_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out128, &id, 128);
    return SFV_OK;
}

sfv_status sfv_partition(sfv_ctx *c, int32_t px, int32_t py, const int32_t *wx, const int32_t *wy, int32_t rank,
                         int32_t nranks, const void *uid, int32_t device) {
    if (!c) return SFV_ERR_ARG;
    if (c->bound) return fail(c, SFV_ERR_SEQUENCE, "sfv_partition after sfv_bind");
    if (px < 1 || py < 1 || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(c, SFV_ERR_ARG, "bad px/py/rank/nranks");
    if (nranks > 1 && px * py != nranks) return fail(c, SFV_ERR_ARG, "px*py (%d) != nranks (%d)", px * py, nranks);
    std::vector<int> xs(px + 1), ys(py + 1);
    if (split_impl(c->cfg.ni, px, wx, xs.data()) != SFV_OK || split_impl(c->cfg.nj, py, wy, ys.data()) != SFV_OK)
        return fail(c, SFV_ERR_ARG, "partition: block width < 2 or weight <= 0");
    c->px = px;
    c->py = py;
    c->xs = xs;
    c->ys = ys;
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    build_blocks(c);
    if (nranks > 1 && uid) {  // NULL id: host-only planning mode
        Nccl &N = nccl();
        if (!N.ok) return fail(c, SFV_ERR_NCCL, "libnccl.so.2 not loadable");
        CK(cudaSetDevice(device));
        ncclUniqueId id;
        memcpy(&id, uid, 128);
        NK(N.CommInitRank(&c->comm, nranks, id, rank));
    }
    c->partitioned = true;
    return SFV_OK;
}

sfv_status sfv_partition_map(const sfv_ctx *c, int32_t block, int32_t *out8) {
    if (!c || !out8 || block < 0 || block >= c->px * c->py) return SFV_ERR_ARG;
    const int bx = block % c->px, by = block / c->px;
    out8[0] = c->xs[bx];
    out8[1] = c->xs[bx + 1];
    out8[2] = c->ys[by];
    out8[3] = c->ys[by + 1];
    out8[4] = bx > 0 ? block - 1 : -1;
    out8[5] = bx < c->px - 1 ? block + 1 : -1;
    out8[6] = by > 0 ? block - c->px : -1;
    out8[7] = by < c->py - 1 ? block + c->px : -1;
    return SFV_OK;
}

sfv_status sfv_halo_plan(const sfv_ctx *c, int32_t block, int32_t *out36) {
    if (!c || !out36 || block < 0 || block >= c->px * c->py) return SFV_ERR_ARG;
    EdgePlan p[4];
    halo_plan(c, block, p);
    for (int e = 0; e < 4; ++e) {
        const int v[9] = {p[e].nbr, p[e].si0, p[e].si1, p[e].sj0, p[e].sj1, p[e].ri0, p[e].ri1, p[e].rj0, p[e].rj1};
        for (int q = 0; q < 9; ++q) out36[9 * e + q] = v[q];
    }
    return SFV_OK;
}

sfv_status sfv_workspace_size(const sfv_ctx *c, size_t *bytes) {
    if (!c || !bytes) return SFV_ERR_ARG;
    *bytes = layout(const_cast<sfv_ctx *>(c), false) + 256;
    return SFV_OK;
}

sfv_status sfv_bind(sfv_ctx *c, void *ws, size_t bytes, void *stream) {
    if (!c || !ws) return SFV_ERR_ARG;
    if (c->bound) return fail(c, SFV_ERR_SEQUENCE, "already bound");
    if (c->nranks > 1 && !c->comm) return fail(c, SFV_ERR_NCCL, "nranks > 1 without an NCCL communicator");
    size_t need = layout(c, false);
    if (bytes < need) return fail(c, SFV_ERR_OOM, "workspace %zu < %zu bytes", bytes, need);
    if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(c, SFV_ERR_ARG, "workspace not 256-byte aligned");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(c, SFV_ERR_CUDA, "no CUDA device");
    CK(cudaSetDevice(c->device));
    c->ws = static_cast<uint8_t *>(ws);
    c->ws_bytes = bytes;
    c->st = static_cast<cudaStream_t>(stream);
    layout(c, true);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, c->device));
    c->nsm = prop.multiProcessorCount;
    int o = 1;
    CK(prepare_stage_kernels());
    CK(stage_occupancy(M_UN, false, false, fast_path(c->P), false, &o));
    c->occ = std::max(1, o);
    CK(stage_occupancy(M_RK4F, false, true, fast_path(c->P), false, &o));
    c->occ_f = std::max(1, o);
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreateWithFlags(&c->ev_edge, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
    {
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c->comm_st, cudaStreamNonBlocking, hi));
    }
    cudaStream_t st = c->st;
    CK(cudaMemsetAsync(c->ws, 0, need, st));
    CK(cudaMemsetAsync(c->geo_bad, 0xff, 8, st));
    const int W = c->cfg.ni + 1;
    const int nbuf = nbuf_of(c->cfg.rk);
    for (Block &b : c->blocks) {
        choose_launch(c, b);
        plan_launches(c, b);
        for (int k = 0; k < nbuf; ++k)
            CK(make_row_tensor_map(&b.tm_buf[k], b.buf[k], (unsigned long long)(b.ni + 4) * 4, b.PJ, 4));
        CK(make_row_tensor_map(&b.tm_met, b.met, (unsigned long long)(b.ni + 1) * NMET, b.PJ, NMET));
        // block-local nodes, [j][i]
        std::vector<double> h(2 * (size_t)(b.ni + 1) * (b.nj + 1));
        const size_t nn = (size_t)(b.ni + 1) * (b.nj + 1);
        for (int j = 0; j <= b.nj; ++j)
            for (int i = 0; i <= b.ni; ++i) {
                h[(size_t)j * (b.ni + 1) + i] = c->X[(size_t)(b.j0 + j) * W + b.i0 + i];
                h[nn + (size_t)j * (b.ni + 1) + i] = c->Y[(size_t)(b.j0 + j) * W + b.i0 + i];
            }
        CK(cudaMemcpyAsync(b.nodes, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
        MetricsArgs m{b.nodes, b.nodes + nn, b.met, b.ni, b.nj, b.PJ, c->geo_bad};
        CK(launch_metrics(m, st));
        CK(cudaStreamSynchronize(st));  // h is freed at scope end
    }
    unsigned long long bad = ~0ull;
    CK(cudaMemcpy(&bad, c->geo_bad, 8, cudaMemcpyDeviceToHost));
    if (bad != ~0ull) return fail(c, SFV_ERR_GEOMETRY, "non-positive volume (device metrics)");
    c->bound = true;
    return SFV_OK;
}

sfv_status sfv_set_state(sfv_ctx *c, const double *U) {
    if (!c || !U) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "sfv_set_state before sfv_bind");
    cudaStream_t st = c->st;
    const int nbuf = nbuf_of(c->cfg.rk);
    const int NI = c->cfg.ni;
    int bcfill[4];
    if (c->halo == SFV_HALO_PEER) {
        // every rank's earlier steps (which signal into this rank's flags)
        // complete before any rank resets its flags: an all-reduce barrier here,
        // and the sigma all-reduce below before anyone steps again
        if (c->nranks > 1) NK(nccl().AllReduce(c->sig, c->sig, 1, ncclDouble, ncclMax, c->comm, st));
        for (Block &b : c->blocks) CK(cudaMemsetAsync(b.flags, 0, PEER_SYNC_BYTES, st));
        CK(cudaMemsetAsync(c->sig_flag, 0, sizeof(unsigned long long) * SIG_RANKS_MAX, st));
        CK(cudaMemsetAsync(c->halo_err, 0, sizeof(unsigned), st));
    }
    CK(cudaMemsetAsync(c->err, 0xff, 8, st));
    // SFV_DEBUG_TIMING: host-side phase times of this call (diagnostic)
    const bool tdbg = getenv("SFV_DEBUG_TIMING") != nullptr;
    auto t_0 = std::chrono::steady_clock::now();
    auto tmark = [&](const char *what) {
        if (!tdbg) return;
        cudaStreamSynchronize(st);
        fprintf(stderr, "[sfv] set_state %s: %.3f ms\n", what,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_0).count());
    };
    for (Block &b : c->blocks) {
        CK(copy_block_h2d(b, U, NI, st));
        tmark("h2d");
        CK(launch_scatter(b.stage, b.buf[0], b.ni, b.nj, b.PJ, st));
        for (int e = 0; e < 4; ++e) bcfill[e] = b.edge[e] == E_CONNECTED ? -1 : b.edge[e];
        for (int k = 0; k < nbuf; ++k) {
            CK(launch_poison_corners(b.buf[k], b.ni, b.nj, b.PJ, st));
            CK(launch_bc_fill(b.buf[k], b.met, b.ni, b.nj, b.PJ, bcfill, c->cfg.inflow_U, st));
        }
        CK(launch_check_state(b.buf[0], b.ni, b.nj, b.PJ, b.i0, b.j0, NI, c->err, st));
    }
    tmark("ghosts + check");
    sfv_status r = exchange(c, 0, st);
    if (r != SFV_OK) return r;
    CK(cudaMemsetAsync(c->sig, 0, 24, st));  // sig[2], step counter
    CK(cudaMemsetAsync(c->done, 0, sizeof(unsigned), st));
    // norm partials: columns a launch configuration does not write (trailing
    // segments off in peer mode) must read as zero
    for (Block &b : c->blocks)
        CK(cudaMemsetAsync(b.partials, 0, sizeof(double) * 8 * (size_t)b.ncta_total * c->pring, st));
    CK(cudaMemsetAsync(c->dt_hist, 0, sizeof(double) * c->cfg.max_history, st));
    CK(cudaMemsetAsync(c->norm_hist, 0, sizeof(double) * c->cfg.max_history * c->nblocks_total * 8, st));
    SYNC("sfv_set_state");
    {  // every rank branches on the same (global) first invalid cell
        sfv_status ag = agree_errors(c);
        if (ag != SFV_OK) return ag;
    }
    unsigned long long e = ~0ull;
    CK(cudaMemcpy(&e, c->err, 8, cudaMemcpyDeviceToHost));
    if (e != ~0ull) {
        c->einfo[0] = -1; c->einfo[1] = 0; c->einfo[2] = (long long)(e % NI); c->einfo[3] = (long long)(e / NI);
        c->have_state = false;
        return fail(c, SFV_ERR_STATE, "invalid state (rho<=0 or p<=0) at cell (%lld,%lld)", c->einfo[2], c->einfo[3]);
    }
    if (!(c->cfg.dt_fixed > 0.0)) {
        for (Block &b : c->blocks) CK(launch_sigma(b.buf[0], b.met, b.ni, b.nj, b.PJ, c->P, c->sig, st));
    }
    if (c->nranks > 1) NK(nccl().AllReduce(c->sig, c->sig, 2, ncclDouble, ncclMax, c->comm, st));
    if (c->halo == SFV_HALO_PEER && c->sig_dev)  // every rank's slot 0 = the global sigma_0 (flags = 0)
        for (int r = 0; r < c->nranks; ++r)
            CK(cudaMemcpyAsync(c->sig_tab + r, c->sig, sizeof(double), cudaMemcpyDeviceToDevice, st));
    SYNC("sfv_set_state");
    tmark("dt_0 (done)");
    c->steps_enq = 0;
    c->have_state = true;
    c->timing_open = false;
    return SFV_OK;
}

sfv_status sfv_step(sfv_ctx *c, int32_t nsteps) {
    if (!c) return SFV_ERR_ARG;
    if (!c->have_state) return fail(c, SFV_ERR_SEQUENCE, "sfv_step before sfv_set_state");
    if (nsteps < 0) return fail(c, SFV_ERR_ARG, "nsteps < 0");
    if (nsteps == 0) return SFV_OK;
    if (!c->gexec && !c->graph_failed) {
        // two graphs: one step, and one step followed by the batched norms
        // reduction (every pring-th step)
        for (int v = 0; v < 2; ++v) {
            cudaStream_t cap;
            CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            cudaGraph_t g = nullptr;
            cudaGraphExec_t ge = nullptr;
            bool ok = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            sfv_status r = SFV_OK;
            if (ok) {
                r = enqueue_step(c, cap, v == 1);
                ok = (cudaStreamEndCapture(cap, &g) == cudaSuccess) && r == SFV_OK;
            }
            if (ok) ok = cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
            if (g) cudaGraphDestroy(g);
            cudaStreamDestroy(cap);
            if (!ok) {
                c->graph_failed = true;
                cudaGetLastError();
                if (ge) cudaGraphExecDestroy(ge);
                if (c->gexec) cudaGraphExecDestroy(c->gexec);
                c->gexec = nullptr;
                break;
            }
            (v == 0 ? c->gexec : c->gexec_norms) = ge;
        }
    }
    if (!c->timing_open) {
        CK(cudaEventRecord(c->ev0, c->st));
        c->timing_open = true;
    }
    if (c->comm_dead) return fail(c, SFV_ERR_NCCL, "the NCCL communicator was aborted by an earlier failure");
    const bool track = c->nranks > 1 && c->comm;  // progress events for the deadlock timeout
    const bool dbg = getenv("SFV_DEBUG_WAIT") != nullptr;
    for (int s = 0; s < nsteps; ++s) {
        const bool batch = (c->steps_enq + s + 1) % c->pring == 0;
        if (dbg) fprintf(stderr, "[sfv] step %lld: launch (in flight %zu)\n", c->steps_enq + s, c->prog.size());
        if (c->gexec && !c->prof) {
            CK(cudaGraphLaunch(batch ? c->gexec_norms : c->gexec, c->st));
        } else {
            sfv_status r = enqueue_step(c, c->st, batch);
            if (r != SFV_OK) return r;
        }
        if (track) {
            // at most kMaxInflight NCCL steps queued: a launch behind a stalled
            // exchange can block inside the runtime, so the wait stays ours
            // (bounded)
            if ((long long)c->prog.size() >= kMaxInflight) {
                sfv_status r = poll_wait(c, "sfv_step", kMaxInflight - 1);
                if (r != SFV_OK) return r;
            }
            cudaEvent_t ev = nullptr;
            if (!c->ev_pool.empty()) {
                ev = c->ev_pool.back();
                c->ev_pool.pop_back();
            } else {
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            }
            CK(cudaEventRecord(ev, c->st));
            c->prog.emplace_back(ev, c->steps_enq + s);
            if (dbg) fprintf(stderr, "[sfv] step %lld: recorded\n", c->steps_enq + s);
        }
    }
    CK(cudaEventRecord(c->ev1, c->st));
    c->steps_enq += nsteps;
    if (c->prof) c->prof_steps += nsteps;
    return SFV_OK;
}

sfv_status sfv_sync(sfv_ctx *c, double *ms) {
    if (!c) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "not bound");
    SYNC("sfv_sync");
    if (ms) *ms = 0.0;
    if (c->timing_open) {
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, c->ev0, c->ev1));
        if (ms) *ms = f;
        c->timing_open = false;
    }
    return check_device_error(c);
}

sfv_status sfv_steps_done(sfv_ctx *c, int64_t *out) {
    if (!c || !out) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "not bound");
    SYNC("sfv_steps_done");
    long long n = 0;
    CK(cudaMemcpy(&n, c->step_ctr, 8, cudaMemcpyDeviceToHost));
    *out = n;
    return SFV_OK;
}

static sfv_status hist_range(sfv_ctx *c, int64_t first, int64_t count, long long *done) {
    sfv_status s = sfv_steps_done(c, (int64_t *)done);
    if (s != SFV_OK) return s;
    if (first < 0 || count < 0 || first + count > *done || first < *done - c->cfg.max_history)
        return fail(c, SFV_ERR_SEQUENCE, "history range [%lld,%lld) not available (done %lld, cap %lld)",
                    (long long)first, (long long)(first + count), *done, (long long)c->cfg.max_history);
    return SFV_OK;
}

sfv_status sfv_get_residual_norms(sfv_ctx *c, int64_t first, int64_t count, double *out) {
    if (!c || (!out && count)) return SFV_ERR_ARG;
    long long done = 0;
    sfv_status s = hist_range(c, first, count, &done);
    if (s != SFV_OK) return s;
    s = check_device_error(c, true);  // collective: every rank takes the same path
    if (s != SFV_OK) return s;
    // steps after the last batched reduction: reduce them now (idempotent)
    if (done % c->pring) {
        s = enqueue_norms(c, done - done % c->pring, (int)(done % c->pring), c->st);
        if (s != SFV_OK) return s;
        SYNC("sfv_get_residual_norms");
    }
    const int nb = c->nblocks_total;
    const long long cap = c->cfg.max_history;
    std::vector<double> h((size_t)count * nb * 8);
    // per step: nb x 8 partials (sum of squares, max |R|); the ring is copied in
    // at most two contiguous pieces
    for (long long q = 0; q < count;) {
        const long long slot = (first + q) % cap;
        const long long m = std::min(count - q, cap - slot);
        CK(cudaMemcpy(h.data() + (size_t)q * nb * 8, c->norm_hist + (size_t)slot * nb * 8,
                      sizeof(double) * nb * 8 * m, cudaMemcpyDeviceToHost));
        q += m;
    }
    if (c->nranks > 1) {  // non-local blocks are zero: a sum all-reduce gathers them
        for (long long q0 = 0; q0 < count; q0 += 4096) {
            const long long m = std::min<long long>(4096, count - q0);
            CK(cudaMemcpy(c->gbuf, h.data() + (size_t)q0 * nb * 8, sizeof(double) * m * nb * 8,
                          cudaMemcpyHostToDevice));
            NK(nccl().AllReduce(c->gbuf, c->gbuf, (size_t)m * nb * 8, ncclDouble, ncclSum, c->comm, c->st));
            SYNC("sfv_get_residual_norms");
            CK(cudaMemcpy(h.data() + (size_t)q0 * nb * 8, c->gbuf, sizeof(double) * m * nb * 8,
                          cudaMemcpyDeviceToHost));
        }
    }
    const double N = (double)c->cfg.ni * (double)c->cfg.nj;
    for (long long q = 0; q < count; ++q) {
        const double *p = h.data() + (size_t)q * nb * 8;
        for (int k = 0; k < 4; ++k) {
            double sum = 0.0, mx = 0.0;
            for (int b = 0; b < nb; ++b) {
                sum += p[b * 8 + k];
                mx = std::max(mx, p[b * 8 + 4 + k]);
            }
            out[q * 8 + k] = std::sqrt(sum / N);
            out[q * 8 + 4 + k] = mx;
        }
    }
    return SFV_OK;
}

sfv_status sfv_get_dt(sfv_ctx *c, int64_t first, int64_t count, double *out) {
    if (!c || (!out && count)) return SFV_ERR_ARG;
    long long done = 0;
    sfv_status s = hist_range(c, first, count, &done);
    if (s != SFV_OK) return s;
    const long long cap = c->cfg.max_history;
    for (long long q = 0; q < count;) {
        const long long slot = (first + q) % cap;
        const long long m = std::min(count - q, cap - slot);
        CK(cudaMemcpy(out + q, c->dt_hist + slot, 8 * m, cudaMemcpyDeviceToHost));
        q += m;
    }
    return check_device_error(c);
}

sfv_status sfv_get_state(sfv_ctx *c, double *U) {
    if (!c || !U) return SFV_ERR_ARG;
    if (!c->have_state) return fail(c, SFV_ERR_SEQUENCE, "no state");
    SYNC("sfv_get_state");
    sfv_status s = check_device_error(c, true);  // collective: every rank takes the same path
    if (s != SFV_OK) return s;
    const int NI = c->cfg.ni;
    if (c->nranks == 1) {
        for (Block &b : c->blocks) {
            CK(launch_gather(b.buf[0], b.stage, b.ni, b.nj, b.PJ, c->st));
            CK(copy_block_d2h(b, U, NI, c->st));
        }
        CK(cudaStreamSynchronize(c->st));
        return SFV_OK;
    }
    // all-gather, one block at a time: rank r broadcasts its block (packed
    // [j][i][4]) into gbuf, which is sized for the largest block, and every
    // rank copies it into place in U (no full-grid device buffer)
    Block &b = c->blocks[0];
    CK(launch_gather(b.buf[0], b.stage, b.ni, b.nj, b.PJ, c->st));
    for (int r = 0; r < c->nranks; ++r) {
        const int bx = r % c->px, by = r / c->px;
        const int i0 = c->xs[bx], ni = c->xs[bx + 1] - i0, j0 = c->ys[by], nj = c->ys[by + 1] - j0;
        const size_t n = (size_t)ni * nj * 4;
        NK(nccl().Broadcast(r == c->rank ? b.stage : c->gbuf, c->gbuf, n, ncclDouble, r, c->comm, c->st));
        CK(cudaMemcpy2DAsync(U + ((size_t)j0 * NI + i0) * 4, (size_t)NI * 32, c->gbuf, (size_t)ni * 32,
                             (size_t)ni * 32, nj, cudaMemcpyDeviceToHost, c->st));
        SYNC("sfv_get_state");  // gbuf is reused by the next block
    }
    return SFV_OK;
}

sfv_status sfv_get_block_state(sfv_ctx *c, int32_t block, double *U) {
    if (!c || !U) return SFV_ERR_ARG;
    if (!c->have_state) return fail(c, SFV_ERR_SEQUENCE, "no state");
    Block *b = local_block(c, block);
    if (!b) return fail(c, SFV_ERR_ARG, "block %d is not local to rank %d", block, c->rank);
    SYNC("sfv_get_block_state");
    sfv_status s = check_device_error(c);
    if (s != SFV_OK) return s;
    CK(launch_gather(b->buf[0], b->stage, b->ni, b->nj, b->PJ, c->st));
    CK(cudaMemcpyAsync(U, b->stage, sizeof(double) * 4 * (size_t)b->ni * b->nj, cudaMemcpyDeviceToHost, c->st));
    SYNC("sfv_get_block_state");
    return SFV_OK;
}

sfv_status sfv_error_info(const sfv_ctx *c, int64_t *out4) {
    if (!c || !out4) return SFV_ERR_ARG;
    for (int k = 0; k < 4; ++k) out4[k] = c->einfo[k];
    return SFV_OK;
}

sfv_status sfv_launch_info(const sfv_ctx *c, int32_t *out4) {
    if (!c || !out4 || c->blocks.empty()) return SFV_ERR_ARG;
    out4[0] = c->blocks[0].nstrips;
    out4[1] = c->blocks[0].lseg[c->blocks[0].nlaunch - 1];
    out4[2] = NT;
    out4[3] = c->occ;
    return SFV_OK;
}

sfv_status sfv_debug_math(sfv_ctx *c, int32_t which, const double *in, double *out, int64_t n) {
    if (!c || !c->bound) return SFV_ERR_SEQUENCE;
    CK(launch_debug_math(which, in, out, n, c->st));
    CK(cudaStreamSynchronize(c->st));
    return SFV_OK;
}

sfv_status sfv_peer_handle(sfv_ctx *c, void *out128) {
    if (!c || !out128) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "sfv_peer_handle before sfv_bind");
    if (c->nranks < 2 || c->blocks.size() != 1) return fail(c, SFV_ERR_ARG, "sfv_peer_handle needs nranks > 1");
    static CUresult (*range)(CUdeviceptr *, size_t *, CUdeviceptr) = nullptr;
    if (!range) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            return fail(c, SFV_ERR_CUDA, "cuMemGetAddressRange unavailable");
        range = reinterpret_cast<decltype(range)>(p);
    }
    CUdeviceptr base = 0;
    size_t sz = 0;
    if (range(&base, &sz, reinterpret_cast<CUdeviceptr>(c->ws)) != CUDA_SUCCESS)
        return fail(c, SFV_ERR_CUDA, "cuMemGetAddressRange failed on the workspace");
    PeerHandle h{};
    CK(cudaIpcGetMemHandle(&h.ipc, reinterpret_cast<void *>(base)));
    const Block &b = c->blocks[0];
    h.ws_off = (int64_t)(reinterpret_cast<CUdeviceptr>(c->ws) - base);
    h.flags_off = reinterpret_cast<uint8_t *>(b.flags) - c->ws;
    for (int k = 0; k < 4; ++k) h.buf_off[k] = b.buf[k] ? reinterpret_cast<uint8_t *>(b.buf[k]) - c->ws : -1;
    h.ni = b.ni;
    h.nj = b.nj;
    h.PJ = b.PJ;
    h.block = b.id;
    memcpy(out128, &h, 128);
    return SFV_OK;
}

sfv_status sfv_peer_connect(sfv_ctx *c, const void *handles) {
    if (!c || !handles) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "sfv_peer_connect before sfv_bind");
    if (c->nranks < 2 || c->blocks.size() != 1) return fail(c, SFV_ERR_ARG, "sfv_peer_connect needs nranks > 1");
    if (c->peer_ready) return fail(c, SFV_ERR_SEQUENCE, "already connected");
    Block &b = c->blocks[0];
    const PeerHandle *H = static_cast<const PeerHandle *>(handles);
    for (int r = 0; r < c->nranks; ++r)
        if (H[r].block != r) return fail(c, SFV_ERR_ARG, "peer handle %d names block %d", r, H[r].block);
    // every other rank's workspace, mapped once (face neighbours: halo
    // stores; all ranks: the dt table)
    const bool all = c->nranks <= SIG_RANKS_MAX;
    std::vector<uint8_t *> ws(c->nranks, nullptr);
    ws[c->rank] = c->ws;
    for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) continue;
        bool face = false;
        for (int e = 0; e < 4; ++e) face |= b.nbr[e] == r;
        if (!face && !all) continue;
        void *p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, H[r].ipc, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_open.push_back(p);
        ws[r] = static_cast<uint8_t *>(p) + H[r].ws_off;
    }
    for (int e = 0; e < 4; ++e) {
        if (b.nbr[e] < 0) continue;
        const PeerHandle &h = H[b.nbr[e]];
        const bool along_i = e < 2;
        if ((along_i ? h.nj != b.nj : h.ni != b.ni) || h.PJ < h.nj + JOFF + 2)
            return fail(c, SFV_ERR_ARG, "peer handle of block %d inconsistent with the partition", b.nbr[e]);
        uint8_t *w = ws[b.nbr[e]];
        PeerView &v = b.pv[e];
        for (int k = 0; k < 4; ++k) v.buf[k] = h.buf_off[k] >= 0 ? reinterpret_cast<double *>(w + h.buf_off[k]) : nullptr;
        v.flags = reinterpret_cast<unsigned long long *>(w + h.flags_off);
        v.grad = c->cfg.viscous ? reinterpret_cast<double *>(w + h.flags_off + al(PEER_SYNC_BYTES)) : nullptr;
        v.PJ = h.PJ;
        v.ni = h.ni;
        v.nj = h.nj;
    }
    if (all) {
        std::vector<double *> t(c->nranks);
        std::vector<unsigned long long *> f(c->nranks);
        for (int r = 0; r < c->nranks; ++r) {
            t[r] = reinterpret_cast<double *>(ws[r] + MISC_SIGTAB);
            f[r] = reinterpret_cast<unsigned long long *>(ws[r] + MISC_SIGFLAG);
        }
        CK(cudaMemcpy(c->rtab, t.data(), sizeof(double *) * c->nranks, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->rflag, f.data(), sizeof(unsigned long long *) * c->nranks, cudaMemcpyHostToDevice));
        const char *ev = getenv("SFV_DEVICE_DT");
        c->sig_dev = !(ev && ev[0] == '0');
    }
    c->peer_ready = true;
    return SFV_OK;
}

sfv_status sfv_set_halo_mode(sfv_ctx *c, int32_t mode) {
    if (!c) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "sfv_set_halo_mode before sfv_bind");
    if (mode != SFV_HALO_COPY && mode != SFV_HALO_PEER) return fail(c, SFV_ERR_ARG, "unknown halo mode %d", mode);
    if (mode == SFV_HALO_PEER && c->nranks > 1 && !c->peer_ready)
        return fail(c, SFV_ERR_SEQUENCE, "SFV_HALO_PEER across ranks needs sfv_peer_connect first");
    CK(cudaStreamSynchronize(c->st));
    c->halo = mode;
    if (mode == SFV_HALO_PEER && c->nranks == 1)
        for (Block &b : c->blocks)
            for (int e = 0; e < 4; ++e) {
                b.pv[e] = PeerView{};
                if (b.nbr[e] < 0) continue;
                const Block &n = *local_block(c, b.nbr[e]);
                for (int k = 0; k < 4; ++k) b.pv[e].buf[k] = n.buf[k];
                b.pv[e].flags = n.flags;
                b.pv[e].grad = n.grad;
                b.pv[e].PJ = n.PJ;
                b.pv[e].ni = n.ni;
                b.pv[e].nj = n.nj;
            }
    for (Block &b : c->blocks) {
        choose_launch(c, b);
        plan_launches(c, b);
    }
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->gexec_norms) cudaGraphExecDestroy(c->gexec_norms);
    c->gexec = c->gexec_norms = nullptr;
    c->graph_failed = false;
    c->have_state = false;  // flags and step counter restart at sfv_set_state
    return SFV_OK;
}

sfv_status sfv_residual(sfv_ctx *c, const double *U, double *R) {
    if (!c || !U || !R) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "sfv_residual before sfv_bind");
    if (c->nranks > 1) return fail(c, SFV_ERR_UNSUPPORTED, "sfv_residual is single-rank (loopback blocks)");
    cudaStream_t st = c->st;
    CK(cudaStreamSynchronize(st));
    if (c->have_state) {  // a failed run reports first
        sfv_status s0 = check_device_error(c);
        if (s0 != SFV_OK) return s0;
    }
    CK(cudaMemsetAsync(c->err, 0xff, 8, st));
    const int NI = c->cfg.ni, k = 1;  // stage buffer 1 is scratch between steps
    int bcfill[4];
    for (Block &b : c->blocks) {
        CK(cudaMemcpy2DAsync(b.stage, (size_t)b.ni * 32, U + ((size_t)b.j0 * NI + b.i0) * 4, (size_t)NI * 32,
                             (size_t)b.ni * 32, b.nj, cudaMemcpyHostToDevice, st));
        CK(launch_scatter(b.stage, b.buf[k], b.ni, b.nj, b.PJ, st));
        for (int e = 0; e < 4; ++e) bcfill[e] = b.edge[e] == E_CONNECTED ? -1 : b.edge[e];
        CK(launch_poison_corners(b.buf[k], b.ni, b.nj, b.PJ, st));
        CK(launch_bc_fill(b.buf[k], b.met, b.ni, b.nj, b.PJ, bcfill, c->cfg.inflow_U, st));
    }
    sfv_status r = exchange(c, k, st);
    if (r != SFV_OK) return r;
    if (c->cfg.viscous) {
        r = enqueue_viscous(c, k, st);
        if (r != SFV_OK) return r;
    }
    for (Block &b : c->blocks) {
        StageArgs a = make_args(c, b, 1);
        a.tm_in = b.tm_buf[k];
        for (int q = 0; q < 3; ++q) a.tm_pw[q] = b.tm_buf[k];
        a.in = b.buf[k];
        a.out = b.resb;
        a.pw0 = a.pw1 = a.pw2 = nullptr;
        a.bump = 0;
        a.row_lo = 0;
        a.row_hi = b.ni;
        CK(launch_stage(a, M_RES, false, false, false, c->cfg.viscous != 0, st));
    }
    CK(cudaStreamSynchronize(st));
    unsigned long long e = ~0ull;
    CK(cudaMemcpy(&e, c->err, sizeof e, cudaMemcpyDeviceToHost));
    if (e != ~0ull) {  // an invalid face state of U: report it, leave the solver's error word clean
        CK(cudaMemset(c->err, 0xff, 8));
        const long long cell = (long long)(e & 0xffffffffull);
        c->einfo[0] = -1; c->einfo[1] = -1; c->einfo[2] = cell % NI; c->einfo[3] = cell / NI;
        return fail(c, SFV_ERR_STATE, "invalid face state of the given state at cell (%lld,%lld)", c->einfo[2],
                    c->einfo[3]);
    }
    for (Block &b : c->blocks) {
        CK(launch_gather(b.resb, b.stage, b.ni, b.nj, b.PJ, st));
        CK(cudaMemcpy2DAsync(R + ((size_t)b.j0 * NI + b.i0) * 4, (size_t)NI * 32, b.stage, (size_t)b.ni * 32,
                             (size_t)b.ni * 32, b.nj, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    return SFV_OK;
}

sfv_status sfv_debug_block_buffer(sfv_ctx *c, int32_t block, int32_t k, double *out) {
    if (!c || !out) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "not bound");
    Block *b = local_block(c, block);
    if (!b || k < -2 || k >= nbuf_of(c->cfg.rk) || (k < 0 && !c->cfg.viscous))
        return fail(c, SFV_ERR_ARG, "no local block %d / buffer %d", block, k);
    CK(cudaStreamSynchronize(c->st));
    if (k == -2) {  // Navier-Stokes gradient frame [(ni+2)*6][nj+2]
        CK(cudaMemcpy(out, b->grad, sizeof(double) * (size_t)(b->ni + 2) * 6 * b->PG, cudaMemcpyDeviceToHost));
        return SFV_OK;
    }
    const double *src = k == -1 ? b->rv : b->buf[k];
    // rows i = -2 .. ni+1, components, columns j = -2 .. nj+1
    CK(cudaMemcpy2D(out, sizeof(double) * (b->nj + 4), src + (JOFF - 2), sizeof(double) * b->PJ,
                    sizeof(double) * (b->nj + 4), (size_t)(b->ni + 4) * 4, cudaMemcpyDeviceToHost));
    return SFV_OK;
}

sfv_status sfv_set_profiling(sfv_ctx *c, int32_t on) {
    if (!c) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "sfv_set_profiling before sfv_bind");
    SYNC("sfv_set_profiling");
    c->prof = on != 0;
    for (double &v : c->prof_ms) v = 0.0;
    c->prof_steps = 0;
    return SFV_OK;
}

sfv_status sfv_get_stage_timings(sfv_ctx *c, double *out) {
    if (!c || !out) return SFV_ERR_ARG;
    if (!c->bound) return fail(c, SFV_ERR_SEQUENCE, "not bound");
    SYNC("sfv_get_stage_timings");
    for (int k = 0; k < NPROF; ++k) out[k] = c->prof_ms[k];
    out[NPROF] = (double)c->prof_steps;
    return SFV_OK;
}

sfv_status sfv_set_comm_timeout(sfv_ctx *c, double seconds) {
    if (!c || !(seconds > 0.0)) return SFV_ERR_ARG;
    c->comm_timeout = seconds;
    return SFV_OK;
}

const char *sfv_last_error(const sfv_ctx *c) { return c ? c->msg.c_str() : "null ctx"; }

void sfv_destroy(sfv_ctx *c) {
    if (!c) return;
    if (c->bound) {
        // peer mode across ranks: neighbours store into this workspace; a
        // barrier (all-reduce) before anyone releases it, then drain the stream
        if (c->halo == SFV_HALO_PEER && c->nranks > 1 && c->comm && !c->comm_dead)
            nccl().AllReduce(c->sig, c->sig, 1, ncclDouble, ncclMax, c->comm, c->st);
        if (wait_stream(c, "sfv_destroy") != SFV_OK) cudaGetLastError();
    }
    for (auto &pe : c->prog) cudaEventDestroy(pe.first);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (auto &sp : c->spans) { cudaEventDestroy(sp.a); cudaEventDestroy(sp.b); }
    for (cudaEvent_t e : c->tev_pool) cudaEventDestroy(e);
    // after an aborted communicator the stream may never drain: the step graphs
    // are left to the process teardown (destroying them would wait on it)
    if (c->gexec && !c->comm_dead) cudaGraphExecDestroy(c->gexec);
    if (c->gexec_norms && !c->comm_dead) cudaGraphExecDestroy(c->gexec_norms);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->ev_edge) cudaEventDestroy(c->ev_edge);
    if (c->ev_comm) cudaEventDestroy(c->ev_comm);
    if (c->comm_st) cudaStreamDestroy(c->comm_st);
    if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
    for (void *p : c->ipc_open) cudaIpcCloseMemHandle(p);
    delete c;
}

}  // extern "C"
