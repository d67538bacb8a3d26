/* oracle.c -- plain, slow, single-threaded CPU oracle (TEST INFRASTRUCTURE).
 *
 * What it computes is SENSEI's explicit finite-volume Euler step as the
 * paper states it, with every point the paper leaves open fixed by the
 * DESIGN.md readings (A-R*):
 *   - Eq. 2: conserved vector and inviscid normal flux;
 *   - Eq. 5: R_h = sum over the 4 faces of F_n * ds (S = 0);
 *   - Eq. 4: |Omega| dU/dt + R_h = 0;
 *   - Eq. 6: explicit s-stage Runge-Kutta;
 *   - Eq. 7: MUSCL extrapolation with limiters Psi;
 *   - PAPER.md:120, 138: ghost-cell boundary enforcement every RK substep,
 *     connected boundaries filled by exchange between partitions;
 *   - PAPER.md:174: 1D (and, for config C5, 2D) decomposition;
 *   - Navier-Stokes mode (cfg.viscous): the viscous flux of Eq. 2
 *      with Stokes' hypothesis, R_h = sum (F - F_v) ds
 *     (Eq. 5), Green-Gauss gradients and a no-slip adiabatic wall (SPEC.md:
 *     201-227; readings N-R1..N-R5 in DESIGN.md).
 * Numerical choices the paper does not make come from SPEC.md: Roe flux with
 * Harten's entropy fix, van Albada limiter (SPEC.md:177,
 * :255), eps=1, kappa=-1, Heun RK2 / classical RK4
 * (SPEC.md:309), the 4-face CFL time step, the largest
 * remainder partition.
 *
 * Parity unpinned (conventions, checked only by GPU-vs-oracle consistency;
 * DESIGN.md §2): the Harten constant and wave set, the bounded van Albada
 * form among admissible limiters, the CFL number, the ramp node
 * distribution, the Jameson-4 coefficients, the NS ghost-gradient /
 * face-average rules beyond their exactness pins, the viscous dt constant.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's oracle legs use this
 * file.  It is built with -O2 -ffp-contract=off; '/' and sqrt() are IEEE.
 * The same source built with -fopenmp (liboracle_omp.so, bench.py's
 * all-cores CPU baseline only) shares the row loops among threads: every
 * cell, face and stage value is computed by the same expression, the norm
 * sums stay serial and the dt minimum / first-error key are exact min
 * reductions, so it is bitwise equal to the single-threaded build
 * (tests/test_oracle_pins.py::test_openmp_build_is_bitwise_single_thread).
 * No blocking, fusion or reordering: each step of the algorithm is a
 * separate loop in the order SURVEY.md §8(c).2 lists them.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------
 * Metrics (reading A-R10).
 * i-face (i,j) joins nodes (i,j)-(i,j+1); j-face (i,j) joins (i,j)-(i+1,j).
 * A = |tangent|, n = tangent rotated -90 deg (i-face) / +90 deg (j-face), so
 * normals point to +i / +j on a right-handed grid.  Cell volume (area x unit
 * depth) by the diagonal form of the shoelace formula.
 * ---------------------------------------------------------------------- */
int orc_metrics(int32_t ni, int32_t nj, const double *X, const double *Y,
                double *iface, double *jface, double *vol, int64_t *bad_cell)
{
    const int64_t W = (int64_t)ni + 1;
#define NX(i, j) X[(int64_t)(j) * W + (i)]
#define NY(i, j) Y[(int64_t)(j) * W + (i)]
    for (int32_t j = 0; j < nj; ++j)
        for (int32_t i = 0; i <= ni; ++i) {
            double tx = NX(i, j + 1) - NX(i, j);
            double ty = NY(i, j + 1) - NY(i, j);
            double A = sqrt(tx * tx + ty * ty);
            double *f = iface + ((int64_t)j * (ni + 1) + i) * 3;
            f[0] = ty / A;
            f[1] = -tx / A;
            f[2] = A;
        }
    for (int32_t j = 0; j <= nj; ++j)
        for (int32_t i = 0; i < ni; ++i) {
            double tx = NX(i + 1, j) - NX(i, j);
            double ty = NY(i + 1, j) - NY(i, j);
            double A = sqrt(tx * tx + ty * ty);
            double *f = jface + ((int64_t)j * ni + i) * 3;
            f[0] = -ty / A;
            f[1] = tx / A;
            f[2] = A;
        }
    for (int32_t j = 0; j < nj; ++j)
        for (int32_t i = 0; i < ni; ++i) {
            double V = 0.5 * ((NX(i + 1, j + 1) - NX(i, j)) * (NY(i, j + 1) - NY(i + 1, j))
                              - (NY(i + 1, j + 1) - NY(i, j)) * (NX(i, j + 1) - NX(i + 1, j)));
            vol[(int64_t)j * ni + i] = V;
            if (!(V > 0.0)) {
                if (bad_cell) *bad_cell = (int64_t)j * ni + i;
                return ORC_ERR_GEOMETRY;
            }
        }
#undef NX
#undef NY
    return ORC_OK;
}

/* Primitive variables:
 * u = mx/rho, v = my/rho, p = (gamma-1)(E - rho (u^2+v^2)/2). */
int orc_primitive(const double U[4], double gamma, double prim[4])
{
    double rho = U[0];
    if (!(rho > 0.0)) return ORC_ERR_STATE;
    double u = U[1] / rho, v = U[2] / rho;
    double p = (gamma - 1.0) * (U[3] - 0.5 * rho * (u * u + v * v));
    prim[0] = rho; prim[1] = u; prim[2] = v; prim[3] = p;
    if (!(p > 0.0)) return ORC_ERR_STATE;
    return ORC_OK;
}

/* Limiter value psi(a, b) for difference b with neighbouring difference a,
 * i.e. psi(r) at r = a/b (reading A-R3).  VA1 = van Albada in difference
 * form with delta added to numerator and denominator. */
double orc_limiter(int32_t kind, double a, double b, double delta)
{
    if (kind == ORC_LIM_NONE) return 1.0;
    if (kind == ORC_LIM_VAN_ALBADA2) {
        double s = (2.0 * a * b + delta) / (a * a + b * b + delta);
        return s > 0.0 ? s : 0.0;
    }
    if (a * b < 0.0) return 0.0;
    return (a * a + a * b + delta) / (a * a + b * b + delta);
}

/* MUSCL extrapolation, Eq. 7, for one component at the
 * face between w[1] and w[2]; w = values at cells (i-2, i-1, i, i+1).
 * Psi^+_f = psi(D_{f+1}, D_f), Psi^-_f = psi(D_{f-1}, D_f) (reading A-R4). */
void orc_muscl(const double w[4], double eps, double kappa, int32_t kind,
               double delta, double *qL, double *qR)
{
    double Dm = w[1] - w[0];
    double D0 = w[2] - w[1];
    double Dp = w[3] - w[2];
    *qL = w[1] + (eps / 4.0) * ((1.0 - kappa) * orc_limiter(kind, D0, Dm, delta) * Dm
                                + (1.0 + kappa) * orc_limiter(kind, Dm, D0, delta) * D0);
    *qR = w[2] - (eps / 4.0) * ((1.0 + kappa) * orc_limiter(kind, Dp, D0, delta) * D0
                                + (1.0 - kappa) * orc_limiter(kind, D0, Dp, delta) * Dp);
}

/* Roe flux with Harten's entropy fix, eigenvector form (readings A-R1, A-R2;
 * SPEC.md:192-200).  Returns the flux per unit face area, F_n of Eq. 2 for
 * Q_L = Q_R. */
int orc_roe_flux(const double QL[4], const double QR[4], double nx, double ny,
                 double gamma, double harten_eps, double F[4])
{
    double rhoL = QL[0], rhoR = QR[0];
    if (!(rhoL > 0.0) || !(rhoR > 0.0)) return ORC_ERR_STATE;
    double uL = QL[1] / rhoL, vL = QL[2] / rhoL;
    double uR = QR[1] / rhoR, vR = QR[2] / rhoR;
    double pL = (gamma - 1.0) * (QL[3] - 0.5 * rhoL * (uL * uL + vL * vL));
    double pR = (gamma - 1.0) * (QR[3] - 0.5 * rhoR * (uR * uR + vR * vR));
    if (!(pL > 0.0) || !(pR > 0.0)) return ORC_ERR_STATE;
    double HL = (QL[3] + pL) / rhoL, HR = (QR[3] + pR) / rhoR;
    double VnL = uL * nx + vL * ny, VnR = uR * nx + vR * ny;

    /* Roe averages */
    double Rt = sqrt(rhoR / rhoL);
    double rhot = Rt * rhoL;
    double ut = (uL + Rt * uR) / (1.0 + Rt);
    double vt = (vL + Rt * vR) / (1.0 + Rt);
    double Ht = (HL + Rt * HR) / (1.0 + Rt);
    double q2t = ut * ut + vt * vt;
    double a2t = (gamma - 1.0) * (Ht - 0.5 * q2t);
    if (!(a2t > 0.0)) return ORC_ERR_STATE;
    double at = sqrt(a2t);
    double Vnt = ut * nx + vt * ny;

    /* jumps and wave strengths */
    double drho = rhoR - rhoL, dp = pR - pL, du = uR - uL, dv = vR - vL;
    double dVn = VnR - VnL;
    double a1 = (dp - rhot * at * dVn) / (2.0 * a2t);
    double a4 = (dp + rhot * at * dVn) / (2.0 * a2t);
    double a2 = drho - dp / a2t;

    /* eigenvalues with Harten's fix on the acoustic waves */
    double l1 = fabs(Vnt - at), l2 = fabs(Vnt), l4 = fabs(Vnt + at);
    double dH = harten_eps * at;
    if (dH < 1e-12) dH = 1e-12;
    if (l1 < dH) l1 = (l1 * l1 + dH * dH) / (2.0 * dH);
    if (l4 < dH) l4 = (l4 * l4 + dH * dH) / (2.0 * dH);

    /* right eigenvectors */
    double r1[4] = {1.0, ut - at * nx, vt - at * ny, Ht - at * Vnt};
    double r2[4] = {1.0, ut, vt, 0.5 * q2t};
    double r3[4] = {0.0, du - dVn * nx, dv - dVn * ny, ut * du + vt * dv - Vnt * dVn};
    double r4[4] = {1.0, ut + at * nx, vt + at * ny, Ht + at * Vnt};

    double FL[4] = {rhoL * VnL, QL[1] * VnL + pL * nx, QL[2] * VnL + pL * ny, (QL[3] + pL) * VnL};
    double FR[4] = {rhoR * VnR, QR[1] * VnR + pR * nx, QR[2] * VnR + pR * ny, (QR[3] + pR) * VnR};
    for (int k = 0; k < 4; ++k) {
        double D = l1 * a1 * r1[k] + l2 * (a2 * r2[k] + rhot * r3[k]) + l4 * a4 * r4[k];
        F[k] = 0.5 * (FL[k] + FR[k]) - 0.5 * D;
    }
    return ORC_OK;
}

/* Integer largest-remainder split of n cells over parts with integer weights
 * (reading A-R24): base_r = floor(n w_r / sum w),
 * rem_r = n w_r mod sum w; leftovers one each by descending rem_r, ties to the
 * lower r.  starts has parts+1 entries.  Every width must be >= 2 (A-R16). */
int orc_split(int32_t n, int32_t parts, const int32_t *weights, int32_t *starts)
{
    if (parts < 1 || n < 1) return ORC_ERR_ARG;
    int64_t sw = 0;
    for (int32_t r = 0; r < parts; ++r) {
        int64_t w = weights ? weights[r] : 1;
        if (w <= 0) return ORC_ERR_ARG;
        sw += w;
    }
    int64_t *base = (int64_t *)calloc((size_t)parts, sizeof(int64_t));
    int64_t *rem = (int64_t *)calloc((size_t)parts, sizeof(int64_t));
    char *taken = (char *)calloc((size_t)parts, 1);
    int64_t used = 0;
    for (int32_t r = 0; r < parts; ++r) {
        int64_t w = weights ? weights[r] : 1;
        base[r] = ((int64_t)n * w) / sw;
        rem[r] = ((int64_t)n * w) % sw;
        used += base[r];
    }
    for (int64_t left = n - used; left > 0; --left) {
        int32_t best = -1;
        for (int32_t r = 0; r < parts; ++r)
            if (!taken[r] && (best < 0 || rem[r] > rem[best])) best = r;
        taken[best] = 1;
        base[best] += 1;
    }
    int status = ORC_OK;
    starts[0] = 0;
    for (int32_t r = 0; r < parts; ++r) {
        if (base[r] < 2) status = ORC_ERR_ARG;
        starts[r + 1] = starts[r] + (int32_t)base[r];
    }
    free(base); free(rem); free(taken);
    return status;
}

/* ------------------------------------------------------------------------
 * Whole solver.
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t i0, i1, j0, j1, ni, nj;
    int32_t nbr[4];           /* W, E, S, N block index or -1 (physical) */
    double *iface, *jface, *vol;
    double *Un;               /* interior, (j*ni+i)*4+k */
    double *W;                /* stage input with a 2-cell ghost frame */
    double *R[4];             /* residual of each stage, interior */
    double *GI, *GJ;          /* face fluxes x area */
    double *grad;             /* NS: interior cell gradients, (j*ni+i)*6 */
} orc_block;

struct orc_ctx {
    orc_config cfg;
    double *X, *Y;
    int32_t px, py, nblocks;
    int32_t *xs, *ys;
    orc_block *b;
    int have_state;
    int64_t steps_done;
    double dt_next;
    double *hist;             /* max_history x 9: dt, L2[4], Linf[4] */
    int64_t err[4];
    char msg[256];
};

static int stages_of(int32_t rk) { return rk == ORC_RK2_HEUN ? 2 : 4; }

/* Butcher coefficients a_{k+1,j} (row k+1, 1-based) and b_j (reading A-R5). */
static double tab_a(int32_t rk, int row, int col)
{
    if (rk == ORC_RK4_CLASSIC) {
        if (row == 2 && col == 1) return 1.0 / 2.0;
        if (row == 3 && col == 2) return 1.0 / 2.0;
        if (row == 4 && col == 3) return 1.0;
        return 0.0;
    }
    if (rk == ORC_RK2_HEUN) return (row == 2 && col == 1) ? 1.0 : 0.0;
    /* Jameson 4-stage: a_{k+1,k} = 1/4, 1/3, 1/2 */
    if (row == 2 && col == 1) return 1.0 / 4.0;
    if (row == 3 && col == 2) return 1.0 / 3.0;
    if (row == 4 && col == 3) return 1.0 / 2.0;
    return 0.0;
}
static double tab_b(int32_t rk, int col)
{
    if (rk == ORC_RK4_CLASSIC) {
        static const double b[4] = {1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0};
        return b[col - 1];
    }
    if (rk == ORC_RK2_HEUN) return 1.0 / 2.0;
    return col == 4 ? 1.0 : 0.0;
}

#define FR(bk, i, j) ((((int64_t)(j) + 2) * ((bk)->ni + 4) + ((i) + 2)) * 4)
#define IN(bk, i, j) ((((int64_t)(j)) * (bk)->ni + (i)) * 4)

static void set_err(orc_ctx *c, int64_t step, int64_t stage, int64_t i, int64_t j, const char *what)
{
    c->err[0] = step; c->err[1] = stage; c->err[2] = i; c->err[3] = j;
    snprintf(c->msg, sizeof c->msg, "%s at step %lld stage %lld cell (%lld,%lld)", what,
             (long long)step, (long long)stage, (long long)i, (long long)j);
}

static void free_blocks(orc_ctx *c)
{
    if (!c->b) return;
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
        free(bk->iface); free(bk->jface); free(bk->vol); free(bk->Un); free(bk->W);
        for (int s = 0; s < 4; ++s) free(bk->R[s]);
        free(bk->GI); free(bk->GJ); free(bk->grad);
    }
    free(c->b); c->b = NULL;
    free(c->xs); free(c->ys); c->xs = c->ys = NULL;
}

int orc_create(const orc_config *cfg, const double *X, const double *Y, orc_ctx **out)
{
    *out = NULL;
    if (cfg->ni < 2 || cfg->nj < 2 || !(cfg->gamma > 1.0) || fabs(cfg->muscl_kappa) > 1.0
        || !(cfg->muscl_eps == 0.0 || cfg->muscl_eps == 1.0)
        || (cfg->dt_fixed <= 0.0 && !(cfg->cfl > 0.0)) || cfg->max_history < 1
        || cfg->rk < 0 || cfg->rk > 2 || cfg->limiter < 0 || cfg->limiter > 2)
        return ORC_ERR_ARG;
    for (int e = 0; e < 4; ++e)
        if (cfg->bc[e] < 0 || cfg->bc[e] > 3 || (cfg->bc[e] == 3 && !cfg->viscous)) return ORC_ERR_ARG;
    if (cfg->viscous && !(cfg->mu >= 0.0 && cfg->prandtl > 0.0 && cfg->gas_R > 0.0)) return ORC_ERR_ARG;
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->cfg = *cfg;
    size_t nn = (size_t)(cfg->ni + 1) * (size_t)(cfg->nj + 1);
    c->X = (double *)malloc(nn * sizeof(double));
    c->Y = (double *)malloc(nn * sizeof(double));
    memcpy(c->X, X, nn * sizeof(double));
    memcpy(c->Y, Y, nn * sizeof(double));
    c->hist = (double *)calloc((size_t)cfg->max_history * 9, sizeof(double));
    int st = orc_partition(c, 1, 1, NULL, NULL);
    if (st != ORC_OK) { orc_destroy(c); return st; }
    *out = c;
    return ORC_OK;
}

int orc_partition(orc_ctx *c, int32_t px, int32_t py, const int32_t *wx, const int32_t *wy)
{
    if (px < 1 || py < 1) return ORC_ERR_ARG;
    int32_t *xs = (int32_t *)calloc((size_t)px + 1, sizeof(int32_t));
    int32_t *ys = (int32_t *)calloc((size_t)py + 1, sizeof(int32_t));
    if (orc_split(c->cfg.ni, px, wx, xs) != ORC_OK || orc_split(c->cfg.nj, py, wy, ys) != ORC_OK) {
        free(xs); free(ys);
        snprintf(c->msg, sizeof c->msg, "partition: block width < 2 or bad weights");
        return ORC_ERR_ARG;
    }
    free_blocks(c);
    c->px = px; c->py = py; c->nblocks = px * py; c->xs = xs; c->ys = ys;
    c->b = (orc_block *)calloc((size_t)c->nblocks, sizeof(orc_block));
    for (int32_t by = 0; by < py; ++by)
        for (int32_t bx = 0; bx < px; ++bx) {
            orc_block *bk = &c->b[bx + px * by];   /* rank = bx + px*by (A-R25) */
            bk->i0 = xs[bx]; bk->i1 = xs[bx + 1]; bk->j0 = ys[by]; bk->j1 = ys[by + 1];
            bk->ni = bk->i1 - bk->i0; bk->nj = bk->j1 - bk->j0;
            bk->nbr[0] = bx > 0 ? (bx - 1) + px * by : -1;
            bk->nbr[1] = bx < px - 1 ? (bx + 1) + px * by : -1;
            bk->nbr[2] = by > 0 ? bx + px * (by - 1) : -1;
            bk->nbr[3] = by < py - 1 ? bx + px * (by + 1) : -1;
            int64_t ncell = (int64_t)bk->ni * bk->nj;
            int64_t nfr = (int64_t)(bk->ni + 4) * (bk->nj + 4) * 4;
            bk->iface = (double *)malloc(sizeof(double) * 3 * (size_t)((bk->ni + 1) * (int64_t)bk->nj));
            bk->jface = (double *)malloc(sizeof(double) * 3 * (size_t)(bk->ni * (int64_t)(bk->nj + 1)));
            bk->vol = (double *)malloc(sizeof(double) * (size_t)ncell);
            bk->Un = (double *)malloc(sizeof(double) * 4 * (size_t)ncell);
            bk->W = (double *)malloc(sizeof(double) * (size_t)nfr);
            for (int64_t q = 0; q < nfr; ++q) bk->W[q] = NAN;   /* corner ghosts stay NaN (A-R18) */
            for (int s = 0; s < 4; ++s) bk->R[s] = (double *)malloc(sizeof(double) * 4 * (size_t)ncell);
            bk->GI = (double *)malloc(sizeof(double) * 4 * (size_t)((bk->ni + 1) * (int64_t)bk->nj));
            bk->GJ = (double *)malloc(sizeof(double) * 4 * (size_t)(bk->ni * (int64_t)(bk->nj + 1)));
            bk->grad = (double *)calloc(6 * (size_t)(bk->ni * (int64_t)bk->nj), sizeof(double));
            /* block-local nodes -> metrics; same arithmetic on the same values
             * as the single-block computation, hence bitwise equal */
            int64_t bw = bk->ni + 1, bh = bk->nj + 1;
            double *lx = (double *)malloc(sizeof(double) * (size_t)(bw * bh));
            double *ly = (double *)malloc(sizeof(double) * (size_t)(bw * bh));
            for (int64_t j = 0; j < bh; ++j)
                for (int64_t i = 0; i < bw; ++i) {
                    int64_t g = (bk->j0 + j) * (int64_t)(c->cfg.ni + 1) + (bk->i0 + i);
                    lx[j * bw + i] = c->X[g];
                    ly[j * bw + i] = c->Y[g];
                }
            int64_t bad = -1;
            int st = orc_metrics(bk->ni, bk->nj, lx, ly, bk->iface, bk->jface, bk->vol, &bad);
            free(lx); free(ly);
            if (st != ORC_OK) {
                int64_t bi = bad % bk->ni, bj = bad / bk->ni;
                set_err(c, -1, -1, bk->i0 + bi, bk->j0 + bj, "non-positive cell volume");
                return st;
            }
        }
    c->have_state = 0;
    return ORC_OK;
}

int orc_partition_map(const orc_ctx *c, int32_t block, int32_t out8[8])
{
    if (block < 0 || block >= c->nblocks) return ORC_ERR_ARG;
    const orc_block *bk = &c->b[block];
    out8[0] = bk->i0; out8[1] = bk->i1; out8[2] = bk->j0; out8[3] = bk->j1;
    for (int e = 0; e < 4; ++e) out8[4 + e] = bk->nbr[e];
    return ORC_OK;
}

/* slip-wall mirror in conserved form: m' = m - 2 (m.n) n, rho and E copied */
static void mirror(const double *w, double nx, double ny, double *g)
{
    double mn = w[1] * nx + w[2] * ny;
    g[0] = w[0];
    g[1] = w[1] - 2.0 * mn * nx;
    g[2] = w[2] - 2.0 * mn * ny;
    g[3] = w[3];
}

/* no-slip adiabatic wall (reading N-R4): ghost layer m = interior
 * layer m with the velocity negated (rho, p and T copied) */
static void noslip(const double *w, double *g)
{
    g[0] = w[0];
    g[1] = -w[1];
    g[2] = -w[2];
    g[3] = w[3];
}

/* Ghost fill of the stage input W (reading A-R11):
 * physical edges by boundary condition, connected edges by bit-copies of the
 * neighbour's interior layers (step 10; "boundary data
 * exchange"). Corner ghosts are never written. */
static void fill_ghosts(orc_ctx *c)
{
    const orc_config *cf = &c->cfg;
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
        double *W = bk->W;
        for (int m = 0; m < 2; ++m) {
            /* W edge */
            for (int32_t j = 0; j < bk->nj; ++j) {
                double *g = W + FR(bk, -1 - m, j);
                if (bk->nbr[0] >= 0) {
                    orc_block *nb = &c->b[bk->nbr[0]];
                    memcpy(g, nb->W + FR(nb, nb->ni - 1 - m, j), 4 * sizeof(double));
                } else if (cf->bc[0] == ORC_BC_INFLOW) {
                    memcpy(g, cf->inflow_U[0], 4 * sizeof(double));
                } else if (cf->bc[0] == ORC_BC_OUTFLOW) {
                    memcpy(g, W + FR(bk, 0, j), 4 * sizeof(double));
                } else if (cf->bc[0] == ORC_BC_NOSLIP_WALL) {
                    noslip(W + FR(bk, m, j), g);
                } else {
                    const double *f = bk->iface + ((int64_t)j * (bk->ni + 1) + 0) * 3;
                    mirror(W + FR(bk, m, j), f[0], f[1], g);
                }
            }
            /* E edge */
            for (int32_t j = 0; j < bk->nj; ++j) {
                double *g = W + FR(bk, bk->ni + m, j);
                if (bk->nbr[1] >= 0) {
                    orc_block *nb = &c->b[bk->nbr[1]];
                    memcpy(g, nb->W + FR(nb, m, j), 4 * sizeof(double));
                } else if (cf->bc[1] == ORC_BC_INFLOW) {
                    memcpy(g, cf->inflow_U[1], 4 * sizeof(double));
                } else if (cf->bc[1] == ORC_BC_OUTFLOW) {
                    memcpy(g, W + FR(bk, bk->ni - 1, j), 4 * sizeof(double));
                } else if (cf->bc[1] == ORC_BC_NOSLIP_WALL) {
                    noslip(W + FR(bk, bk->ni - 1 - m, j), g);
                } else {
                    const double *f = bk->iface + ((int64_t)j * (bk->ni + 1) + bk->ni) * 3;
                    mirror(W + FR(bk, bk->ni - 1 - m, j), f[0], f[1], g);
                }
            }
            /* S edge */
            for (int32_t i = 0; i < bk->ni; ++i) {
                double *g = W + FR(bk, i, -1 - m);
                if (bk->nbr[2] >= 0) {
                    orc_block *nb = &c->b[bk->nbr[2]];
                    memcpy(g, nb->W + FR(nb, i, nb->nj - 1 - m), 4 * sizeof(double));
                } else if (cf->bc[2] == ORC_BC_INFLOW) {
                    memcpy(g, cf->inflow_U[2], 4 * sizeof(double));
                } else if (cf->bc[2] == ORC_BC_OUTFLOW) {
                    memcpy(g, W + FR(bk, i, 0), 4 * sizeof(double));
                } else if (cf->bc[2] == ORC_BC_NOSLIP_WALL) {
                    noslip(W + FR(bk, i, m), g);
                } else {
                    const double *f = bk->jface + ((int64_t)0 * bk->ni + i) * 3;
                    mirror(W + FR(bk, i, m), f[0], f[1], g);
                }
            }
            /* N edge */
            for (int32_t i = 0; i < bk->ni; ++i) {
                double *g = W + FR(bk, i, bk->nj + m);
                if (bk->nbr[3] >= 0) {
                    orc_block *nb = &c->b[bk->nbr[3]];
                    memcpy(g, nb->W + FR(nb, i, m), 4 * sizeof(double));
                } else if (cf->bc[3] == ORC_BC_INFLOW) {
                    memcpy(g, cf->inflow_U[3], 4 * sizeof(double));
                } else if (cf->bc[3] == ORC_BC_OUTFLOW) {
                    memcpy(g, W + FR(bk, i, bk->nj - 1), 4 * sizeof(double));
                } else if (cf->bc[3] == ORC_BC_NOSLIP_WALL) {
                    noslip(W + FR(bk, i, bk->nj - 1 - m), g);
                } else {
                    const double *f = bk->jface + ((int64_t)bk->nj * bk->ni + i) * 3;
                    mirror(W + FR(bk, i, bk->nj - 1 - m), f[0], f[1], g);
                }
            }
        }
    }
}

/* ------------------------------------------------------------------------
 * Navier-Stokes pieces (Eq. 2).
 * ---------------------------------------------------------------------- */
/* viscous normal flux: Stokes' hypothesis lambda = -2 mu / 3,
 * tau_xx = 2 mu u_x + lambda (u_x + v_y), tau_yy = 2 mu v_y + lambda (u_x + v_y),
 * tau_xy = mu (u_y + v_x), Theta_i = u tau_xi + v tau_yi + k T_i;
 * F_v . n = (0, tau_xx nx + tau_xy ny, tau_xy nx + tau_yy ny, Theta_x nx + Theta_y ny) */
void orc_viscous_flux(const double g[6], double u, double v, double nx, double ny, double mu, double k,
                      double Fv[4])
{
    double lambda = -2.0 * mu / 3.0;
    double div = g[0] + g[3];
    double txx = 2.0 * mu * g[0] + lambda * div;
    double tyy = 2.0 * mu * g[3] + lambda * div;
    double txy = mu * (g[1] + g[2]);
    double thx = u * txx + v * txy + k * g[4];
    double thy = u * txy + v * tyy + k * g[5];
    Fv[0] = 0.0;
    Fv[1] = txx * nx + txy * ny;
    Fv[2] = txy * nx + tyy * ny;
    Fv[3] = thx * nx + thy * ny;
}

/* (u, v, T) of a conserved state, T = p / (rho R) */
static void uvT(const double *w, double gamma, double R, double out[3])
{
    double prim[4];
    orc_primitive(w, gamma, prim);
    out[0] = prim[1];
    out[1] = prim[2];
    out[2] = prim[3] / (prim[0] * R);
}

/* Green-Gauss gradient of (u, v, T) in every interior cell of a block from
 * the ghost-filled W (reading N-R2): grad phi = (1/V) sum_f phi_f n_f A_f
 * over the 4 faces with outward normals, phi_f the arithmetic mean of the
 * two cells sharing the face.  Needs only face-neighbour ghosts. */
static void gradients_block(orc_ctx *c, orc_block *bk)
{
    const orc_config *cf = &c->cfg;
    for (int32_t j = 0; j < bk->nj; ++j)
        for (int32_t i = 0; i < bk->ni; ++i) {
            double pc[3], pw[3], pe[3], ps[3], pn[3];
            uvT(bk->W + FR(bk, i, j), cf->gamma, cf->gas_R, pc);
            uvT(bk->W + FR(bk, i - 1, j), cf->gamma, cf->gas_R, pw);
            uvT(bk->W + FR(bk, i + 1, j), cf->gamma, cf->gas_R, pe);
            uvT(bk->W + FR(bk, i, j - 1), cf->gamma, cf->gas_R, ps);
            uvT(bk->W + FR(bk, i, j + 1), cf->gamma, cf->gas_R, pn);
            const double *fW = bk->iface + ((int64_t)j * (bk->ni + 1) + i) * 3;
            const double *fE = bk->iface + ((int64_t)j * (bk->ni + 1) + i + 1) * 3;
            const double *fS = bk->jface + ((int64_t)j * bk->ni + i) * 3;
            const double *fN = bk->jface + ((int64_t)(j + 1) * bk->ni + i) * 3;
            double V = bk->vol[(int64_t)j * bk->ni + i];
            for (int q = 0; q < 3; ++q) {
                double phE = 0.5 * (pc[q] + pe[q]), phW = 0.5 * (pw[q] + pc[q]);
                double phN = 0.5 * (pc[q] + pn[q]), phS = 0.5 * (ps[q] + pc[q]);
                double gx = phE * fE[0] * fE[2] - phW * fW[0] * fW[2] + phN * fN[0] * fN[2] - phS * fS[0] * fS[2];
                double gy = phE * fE[1] * fE[2] - phW * fW[1] * fW[2] + phN * fN[1] * fN[2] - phS * fS[1] * fS[2];
                bk->grad[IN(bk, i, j) / 4 * 6 + 2 * q] = gx / V;
                bk->grad[IN(bk, i, j) / 4 * 6 + 2 * q + 1] = gy / V;
            }
        }
}

/* gradient of cell (i, j) of a block, i in [-1, ni], j in [-1, nj] (not a
 * corner): interior cells their own; a connected edge's ghost the
 * neighbour's cell; a physical edge's ghost the adjacent interior cell's
 * (reading N-R1) */
static const double *cell_grad(orc_ctx *c, orc_block *bk, int32_t i, int32_t j)
{
    if (i < 0 || i >= bk->ni) {
        int e = i < 0 ? 0 : 1;
        if (bk->nbr[e] >= 0) {
            orc_block *nb = &c->b[bk->nbr[e]];
            return nb->grad + IN(nb, i < 0 ? nb->ni - 1 : 0, j) / 4 * 6;
        }
        return bk->grad + IN(bk, i < 0 ? 0 : bk->ni - 1, j) / 4 * 6;
    }
    if (j < 0 || j >= bk->nj) {
        int e = j < 0 ? 2 : 3;
        if (bk->nbr[e] >= 0) {
            orc_block *nb = &c->b[bk->nbr[e]];
            return nb->grad + IN(nb, i, j < 0 ? nb->nj - 1 : 0) / 4 * 6;
        }
        return bk->grad + IN(bk, i, j < 0 ? 0 : bk->nj - 1) / 4 * 6;
    }
    return bk->grad + IN(bk, i, j) / 4 * 6;
}

/* F_v . n of the face between cells L and R (reading N-R3): gradients and
 * (u, v) are arithmetic means of the two cells */
static void face_viscous(orc_ctx *c, orc_block *bk, int32_t iL, int32_t jL, int32_t iR, int32_t jR,
                         double nx, double ny, double Fv[4])
{
    const orc_config *cf = &c->cfg;
    const double *gL = cell_grad(c, bk, iL, jL), *gR = cell_grad(c, bk, iR, jR);
    double g[6], pL[3], pR[3];
    for (int q = 0; q < 6; ++q) g[q] = 0.5 * (gL[q] + gR[q]);
    uvT(bk->W + FR(bk, iL, jL), cf->gamma, cf->gas_R, pL);
    uvT(bk->W + FR(bk, iR, jR), cf->gamma, cf->gas_R, pR);
    double k = cf->mu * (cf->gamma * cf->gas_R / (cf->gamma - 1.0)) / cf->prandtl;
    orc_viscous_flux(g, 0.5 * (pL[0] + pR[0]), 0.5 * (pL[1] + pR[1]), nx, ny, cf->mu, k, Fv);
}

/* Residual R = sum_f G_f (Eq. 5 with S = 0):
 * every face evaluated once with L = the lower-index cell, then
 * R(i,j) = ((G^I(i+1,j) - G^I(i,j)) + G^J(i,j+1)) - G^J(i,j) (A-R10).
 * A failing face state is attributed to global cell (min(I,NI-1), J) for
 * i-faces and (I, min(J,NJ-1)) for j-faces; the smallest J*NI+I is kept. */
static int residual_block(orc_ctx *c, orc_block *bk, double *R, int64_t *bad)
{
    const orc_config *cf = &c->cfg;
    const int64_t NI = cf->ni, NJ = cf->nj;
    int status = ORC_OK;
    if (cf->residual_kind == ORC_RES_LINEAR) {
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i)
                for (int k = 0; k < 4; ++k)
                    R[IN(bk, i, j) + k] = cf->linear_rate * bk->vol[(int64_t)j * bk->ni + i]
                                          * bk->W[FR(bk, i, j) + k];
        return ORC_OK;
    }
#pragma omp parallel for schedule(static)
    for (int32_t j = 0; j < bk->nj; ++j)
        for (int32_t i = 0; i <= bk->ni; ++i) {
            double QL[4], QR[4], F[4];
            for (int k = 0; k < 4; ++k) {
                double w[4] = {bk->W[FR(bk, i - 2, j) + k], bk->W[FR(bk, i - 1, j) + k],
                               bk->W[FR(bk, i, j) + k], bk->W[FR(bk, i + 1, j) + k]};
                orc_muscl(w, cf->muscl_eps, cf->muscl_kappa, cf->limiter, cf->lim_delta, &QL[k], &QR[k]);
            }
            const double *f = bk->iface + ((int64_t)j * (bk->ni + 1) + i) * 3;
            if (orc_roe_flux(QL, QR, f[0], f[1], cf->gamma, cf->harten_eps, F) != ORC_OK) {
                int64_t gi = bk->i0 + i; if (gi > NI - 1) gi = NI - 1;
                int64_t key = (bk->j0 + j) * NI + gi;
#pragma omp critical(orc_bad)
                {
                    if (*bad < 0 || key < *bad) *bad = key;
                    status = ORC_ERR_STATE;
                }
                for (int k = 0; k < 4; ++k) F[k] = NAN;
            }
            if (cf->viscous) {
                double Fv[4];
                face_viscous(c, bk, i - 1, j, i, j, f[0], f[1], Fv);
                for (int k = 0; k < 4; ++k) F[k] = F[k] - Fv[k];
            }
            for (int k = 0; k < 4; ++k) bk->GI[((int64_t)j * (bk->ni + 1) + i) * 4 + k] = F[k] * f[2];
        }
#pragma omp parallel for schedule(static)
    for (int32_t j = 0; j <= bk->nj; ++j)
        for (int32_t i = 0; i < bk->ni; ++i) {
            double QL[4], QR[4], F[4];
            for (int k = 0; k < 4; ++k) {
                double w[4] = {bk->W[FR(bk, i, j - 2) + k], bk->W[FR(bk, i, j - 1) + k],
                               bk->W[FR(bk, i, j) + k], bk->W[FR(bk, i, j + 1) + k]};
                orc_muscl(w, cf->muscl_eps, cf->muscl_kappa, cf->limiter, cf->lim_delta, &QL[k], &QR[k]);
            }
            const double *f = bk->jface + ((int64_t)j * bk->ni + i) * 3;
            if (orc_roe_flux(QL, QR, f[0], f[1], cf->gamma, cf->harten_eps, F) != ORC_OK) {
                int64_t gj = bk->j0 + j; if (gj > NJ - 1) gj = NJ - 1;
                int64_t key = gj * NI + (bk->i0 + i);
#pragma omp critical(orc_bad)
                {
                    if (*bad < 0 || key < *bad) *bad = key;
                    status = ORC_ERR_STATE;
                }
                for (int k = 0; k < 4; ++k) F[k] = NAN;
            }
            if (cf->viscous) {
                double Fv[4];
                face_viscous(c, bk, i, j - 1, i, j, f[0], f[1], Fv);
                for (int k = 0; k < 4; ++k) F[k] = F[k] - Fv[k];
            }
            for (int k = 0; k < 4; ++k) bk->GJ[((int64_t)j * bk->ni + i) * 4 + k] = F[k] * f[2];
        }
#pragma omp parallel for schedule(static)
    for (int32_t j = 0; j < bk->nj; ++j)
        for (int32_t i = 0; i < bk->ni; ++i)
            for (int k = 0; k < 4; ++k) {
                double GW = bk->GI[((int64_t)j * (bk->ni + 1) + i) * 4 + k];
                double GE = bk->GI[((int64_t)j * (bk->ni + 1) + i + 1) * 4 + k];
                double GS = bk->GJ[((int64_t)j * bk->ni + i) * 4 + k];
                double GN = bk->GJ[((int64_t)(j + 1) * bk->ni + i) * 4 + k];
                R[IN(bk, i, j) + k] = ((GE - GW) + GN) - GS;
            }
    return status;
}

/* rho <= 0 or p <= 0 in a (new) state: smallest global cell index */
static int check_states(orc_ctx *c, int use_W, int64_t *bad)
{
    int status = ORC_OK;
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
#pragma omp parallel for schedule(static)
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i) {
                const double *u = use_W ? bk->W + FR(bk, i, j) : bk->Un + IN(bk, i, j);
                double prim[4];
                if (orc_primitive(u, c->cfg.gamma, prim) != ORC_OK) {
                    int64_t key = (int64_t)(bk->j0 + j) * c->cfg.ni + (bk->i0 + i);
#pragma omp critical(orc_bad)
                    {
                        if (*bad < 0 || key < *bad) *bad = key;
                        status = ORC_ERR_STATE;
                    }
                }
            }
    }
    return status;
}

/* CFL time step from U^n interior cells (reading A-R6):
 * dt = CFL * min_c V_c / sigma_c, sigma = ((t_W + t_E) + t_S) + t_N,
 * t_f = (|u nx + v ny| + a) A_f.  cell_v_over_sigma returns V/sigma of one
 * cell (faces W, E, S, N as {nx, ny, A}). */
static int cell_v_over_sigma(const double *U, const double *fW, const double *fE, const double *fS,
                             const double *fN, double V, double gamma, double visc, double *r)
{
    double prim[4];
    if (orc_primitive(U, gamma, prim) != ORC_OK) return ORC_ERR_STATE;
    double u = prim[1], v = prim[2];
    double a = sqrt(gamma * prim[3] / prim[0]);
    double tW = (fabs(u * fW[0] + v * fW[1]) + a) * fW[2];
    double tE = (fabs(u * fE[0] + v * fE[1]) + a) * fE[2];
    double tS = (fabs(u * fS[0] + v * fS[1]) + a) * fS[2];
    double tN = (fabs(u * fN[0] + v * fN[1]) + a) * fN[2];
    double sigma = ((tW + tE) + tS) + tN;
    if (visc > 0.0) {
        /* viscous spectral radius (reading N-R6, revised): visc = 4 max(4/3, gamma) mu / Pr,
         * sigma_v = visc / rho * (S_I^2 + S_J^2) / V with S_I, S_J the mean face areas */
        double sI = 0.5 * (fW[2] + fE[2]), sJ = 0.5 * (fS[2] + fN[2]);
        sigma = sigma + visc / prim[0] * (sI * sI + sJ * sJ) / V;
    }
    *r = V / sigma;
    return ORC_OK;
}

static double visc_factor(const orc_config *cf)
{
    if (!cf->viscous) return 0.0;
    double m = cf->gamma > 4.0 / 3.0 ? cf->gamma : 4.0 / 3.0;
    return 4.0 * m * cf->mu / cf->prandtl;
}

static int compute_dt(orc_ctx *c, double *dt)
{
    if (c->cfg.dt_fixed > 0.0) { *dt = c->cfg.dt_fixed; return ORC_OK; }
    double mn = INFINITY;
    int bad = 0;
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
#pragma omp parallel for schedule(static) reduction(min : mn) reduction(| : bad)
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i) {
                double r;
                if (cell_v_over_sigma(bk->Un + IN(bk, i, j),
                                      bk->iface + ((int64_t)j * (bk->ni + 1) + i) * 3,
                                      bk->iface + ((int64_t)j * (bk->ni + 1) + i + 1) * 3,
                                      bk->jface + ((int64_t)j * bk->ni + i) * 3,
                                      bk->jface + ((int64_t)(j + 1) * bk->ni + i) * 3,
                                      bk->vol[(int64_t)j * bk->ni + i], c->cfg.gamma, visc_factor(&c->cfg),
                                      &r) != ORC_OK)
                    bad = 1;
                else if (r < mn)
                    mn = r;
            }
    }
    if (bad) return ORC_ERR_STATE;
    *dt = c->cfg.cfl * mn;
    return ORC_OK;
}

/* The same dt for a whole grid without a solver context, processed in bands
 * of rows so that very large grids (config C3) fit in memory. */
int orc_stable_dt(int32_t ni, int32_t nj, const double *X, const double *Y, const double *U, double gamma,
                  double cfl, double *dt)
{
    const int32_t band = 64;
    double mn = INFINITY;
    double *fi = (double *)malloc(sizeof(double) * 3 * (size_t)(ni + 1) * band);
    double *fj = (double *)malloc(sizeof(double) * 3 * (size_t)ni * (band + 1));
    double *vol = (double *)malloc(sizeof(double) * (size_t)ni * band);
    int st = ORC_OK;
    for (int32_t j0 = 0; j0 < nj && st == ORC_OK; j0 += band) {
        int32_t nb = nj - j0 < band ? nj - j0 : band;
        const double *Xb = X + (int64_t)j0 * (ni + 1), *Yb = Y + (int64_t)j0 * (ni + 1);
        st = orc_metrics(ni, nb, Xb, Yb, fi, fj, vol, NULL);
        for (int32_t j = 0; j < nb && st == ORC_OK; ++j)
            for (int32_t i = 0; i < ni; ++i) {
                double r;
                st = cell_v_over_sigma(U + ((int64_t)(j0 + j) * ni + i) * 4, fi + ((int64_t)j * (ni + 1) + i) * 3,
                                       fi + ((int64_t)j * (ni + 1) + i + 1) * 3, fj + ((int64_t)j * ni + i) * 3,
                                       fj + ((int64_t)(j + 1) * ni + i) * 3, vol[(int64_t)j * ni + i], gamma, 0.0, &r);
                if (st != ORC_OK) break;
                if (r < mn) mn = r;
            }
    }
    free(fi); free(fj); free(vol);
    *dt = cfl * mn;
    return st;
}

int orc_set_state(orc_ctx *c, const double *U)
{
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i)
                memcpy(bk->Un + IN(bk, i, j),
                       U + ((int64_t)(bk->j0 + j) * c->cfg.ni + (bk->i0 + i)) * 4, 4 * sizeof(double));
    }
    int64_t bad = -1;
    c->have_state = 0;
    if (check_states(c, 0, &bad) != ORC_OK) {
        set_err(c, -1, 0, bad % c->cfg.ni, bad / c->cfg.ni, "invalid state (rho<=0 or p<=0)");
        return ORC_ERR_STATE;
    }
    if (compute_dt(c, &c->dt_next) != ORC_OK) return ORC_ERR_STATE;
    c->steps_done = 0;
    c->have_state = 1;
    memset(c->hist, 0, sizeof(double) * 9 * (size_t)c->cfg.max_history);
    return ORC_OK;
}

/* One explicit RK step (Eq. 6):
 * W_1 = U^n; for k = 1..s: ghost-fill W_k, R_k = R(W_k);
 * W_{k+1} = U^n - dt*S/V, S = sum_{j<=k, a_{k+1,j}!=0} a_{k+1,j} R_j;
 * U^{n+1} = U^n - dt*(sum_j b_j R_j)/V.  dU/dt = -R/|Omega| (Eq. 4). */
int orc_step(orc_ctx *c, int32_t nsteps)
{
    if (!c->have_state) { snprintf(c->msg, sizeof c->msg, "step before set_state"); return ORC_ERR_SEQUENCE; }
    const orc_config *cf = &c->cfg;
    const int s = stages_of(cf->rk);
    for (int32_t it = 0; it < nsteps; ++it) {
        const int64_t step = c->steps_done;
        const double dt = c->dt_next;
        double *h = c->hist + (step % cf->max_history) * 9;
        h[0] = dt;
        for (int32_t n = 0; n < c->nblocks; ++n) {
            orc_block *bk = &c->b[n];
#pragma omp parallel for schedule(static)
            for (int32_t j = 0; j < bk->nj; ++j)
                for (int32_t i = 0; i < bk->ni; ++i)
                    memcpy(bk->W + FR(bk, i, j), bk->Un + IN(bk, i, j), 4 * sizeof(double));
        }
        for (int k = 1; k <= s; ++k) {
            fill_ghosts(c);
            int64_t bad = -1;
            int st = ORC_OK;
            if (cf->viscous)  /* every block's gradients first: ghost gradients are the neighbours' */
                for (int32_t n = 0; n < c->nblocks; ++n) gradients_block(c, &c->b[n]);
            for (int32_t n = 0; n < c->nblocks; ++n)
                if (residual_block(c, &c->b[n], c->b[n].R[k - 1], &bad) != ORC_OK) st = ORC_ERR_STATE;
            if (st != ORC_OK) {
                set_err(c, step, k, bad % cf->ni, bad / cf->ni, "invalid face state");
                c->have_state = 0;
                return ORC_ERR_STATE;
            }
            if (k == 1) {
                /* residual norms of R(U^n) (reading A-R20), j outer / i inner
                 * over the global grid */
                double sum[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
                for (int32_t by = 0; by < c->py; ++by)
                    for (int32_t jj = c->ys[by]; jj < c->ys[by + 1]; ++jj)
                        for (int32_t bx = 0; bx < c->px; ++bx) {
                            orc_block *bk = &c->b[bx + c->px * by];
                            for (int32_t i = 0; i < bk->ni; ++i)
                                for (int q = 0; q < 4; ++q) {
                                    double r = bk->R[0][IN(bk, i, jj - bk->j0) + q];
                                    sum[q] += r * r;
                                    if (fabs(r) > mx[q]) mx[q] = fabs(r);
                                }
                        }
                for (int q = 0; q < 4; ++q) {
                    h[1 + q] = sqrt(sum[q] / ((double)cf->ni * (double)cf->nj));
                    h[5 + q] = mx[q];
                }
            }
            for (int32_t n = 0; n < c->nblocks; ++n) {
                orc_block *bk = &c->b[n];
#pragma omp parallel for schedule(static)
                for (int32_t j = 0; j < bk->nj; ++j)
                    for (int32_t i = 0; i < bk->ni; ++i) {
                        double V = bk->vol[(int64_t)j * bk->ni + i];
                        for (int q = 0; q < 4; ++q) {
                            double S = 0.0;
                            int first = 1;
                            for (int jc = 1; jc <= k; ++jc) {
                                double coef = (k < s) ? tab_a(cf->rk, k + 1, jc) : tab_b(cf->rk, jc);
                                if (coef == 0.0) continue;
                                double term = coef * bk->R[jc - 1][IN(bk, i, j) + q];
                                S = first ? term : S + term;
                                first = 0;
                            }
                            double un = bk->Un[IN(bk, i, j) + q];
                            double nv = un - dt * S / V;
                            if (k < s) bk->W[FR(bk, i, j) + q] = nv;
                            else bk->Un[IN(bk, i, j) + q] = nv;
                        }
                    }
            }
            if (check_states(c, k < s, &bad) != ORC_OK) {
                set_err(c, step, k, bad % cf->ni, bad / cf->ni, "invalid state (rho<=0 or p<=0)");
                c->have_state = 0;
                return ORC_ERR_STATE;
            }
        }
        c->steps_done = step + 1;
        if (compute_dt(c, &c->dt_next) != ORC_OK) return ORC_ERR_STATE;
    }
    return ORC_OK;
}

int orc_get_state(const orc_ctx *c, double *U)
{
    if (!c->have_state) return ORC_ERR_SEQUENCE;
    for (int32_t n = 0; n < c->nblocks; ++n) {
        const orc_block *bk = &c->b[n];
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i)
                memcpy(U + ((int64_t)(bk->j0 + j) * c->cfg.ni + (bk->i0 + i)) * 4,
                       bk->Un + IN(bk, i, j), 4 * sizeof(double));
    }
    return ORC_OK;
}

static int hist_range_ok(const orc_ctx *c, int64_t first, int64_t count)
{
    return first >= 0 && count >= 0 && first + count <= c->steps_done
           && first >= c->steps_done - c->cfg.max_history;
}

int orc_get_residual_norms(const orc_ctx *c, int64_t first, int64_t count, double *out)
{
    if (!hist_range_ok(c, first, count)) return ORC_ERR_SEQUENCE;
    for (int64_t n = 0; n < count; ++n)
        memcpy(out + n * 8, c->hist + ((first + n) % c->cfg.max_history) * 9 + 1, 8 * sizeof(double));
    return ORC_OK;
}

int orc_get_dt(const orc_ctx *c, int64_t first, int64_t count, double *out)
{
    if (!hist_range_ok(c, first, count)) return ORC_ERR_SEQUENCE;
    for (int64_t n = 0; n < count; ++n) out[n] = c->hist[((first + n) % c->cfg.max_history) * 9];
    return ORC_OK;
}

/* R(U) for a global state U: ghost fill (BC + exchange) then Eq. 5. */
int orc_residual(orc_ctx *c, const double *U, double *R)
{
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i)
                memcpy(bk->W + FR(bk, i, j), U + ((int64_t)(bk->j0 + j) * c->cfg.ni + (bk->i0 + i)) * 4,
                       4 * sizeof(double));
    }
    fill_ghosts(c);
    int64_t bad = -1;
    int st = ORC_OK;
    if (c->cfg.viscous)
        for (int32_t n = 0; n < c->nblocks; ++n) gradients_block(c, &c->b[n]);
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
        if (residual_block(c, bk, bk->R[0], &bad) != ORC_OK) st = ORC_ERR_STATE;
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i)
                memcpy(R + ((int64_t)(bk->j0 + j) * c->cfg.ni + (bk->i0 + i)) * 4, bk->R[0] + IN(bk, i, j),
                       4 * sizeof(double));
    }
    if (st != ORC_OK) set_err(c, -1, -1, bad % c->cfg.ni, bad / c->cfg.ni, "invalid face state");
    return st;
}

/* Ghost frame of a single-block ctx after ghost fill: (ni+4)*(nj+4)*4,
 * index ((j+2)*(ni+4)+(i+2))*4+k; corner ghosts are NaN. */
int orc_ghost_frame(orc_ctx *c, const double *U, double *frame)
{
    if (c->nblocks != 1) return ORC_ERR_ARG;
    orc_block *bk = &c->b[0];
    for (int32_t j = 0; j < bk->nj; ++j)
        for (int32_t i = 0; i < bk->ni; ++i)
            memcpy(bk->W + FR(bk, i, j), U + ((int64_t)j * c->cfg.ni + i) * 4, 4 * sizeof(double));
    fill_ghosts(c);
    memcpy(frame, bk->W, sizeof(double) * 4 * (size_t)((bk->ni + 4) * (int64_t)(bk->nj + 4)));
    return ORC_OK;
}

int orc_gradients(orc_ctx *c, const double *U, double *grad)
{
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i)
                memcpy(bk->W + FR(bk, i, j), U + ((int64_t)(bk->j0 + j) * c->cfg.ni + (bk->i0 + i)) * 4,
                       4 * sizeof(double));
    }
    fill_ghosts(c);
    for (int32_t n = 0; n < c->nblocks; ++n) {
        orc_block *bk = &c->b[n];
        gradients_block(c, bk);
        for (int32_t j = 0; j < bk->nj; ++j)
            for (int32_t i = 0; i < bk->ni; ++i)
                memcpy(grad + ((int64_t)(bk->j0 + j) * c->cfg.ni + (bk->i0 + i)) * 6, bk->grad + IN(bk, i, j) / 4 * 6,
                       6 * sizeof(double));
    }
    return ORC_OK;
}

int64_t orc_steps_done(const orc_ctx *c) { return c->steps_done; }
void orc_error_info(const orc_ctx *c, int64_t out4[4]) { memcpy(out4, c->err, sizeof c->err); }
const char *orc_last_error(const orc_ctx *c) { return c->msg; }

void orc_destroy(orc_ctx *c)
{
    if (!c) return;
    free_blocks(c);
    free(c->X); free(c->Y); free(c->hist);
    free(c);
}
