/* oracle.h -- plain, slow, single-threaded CPU oracle for the SENSEI
 * finite-volume hot path (arXiv 2305.18057).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path (paper_2305_18057_b200/csrc, include/sfv.h); the two agree only on
 * the array layouts documented below and on the numeric codes of the enums,
 * which each side defines for itself.
 *
 * Precision: IEEE binary64, compiled with -O2 -ffp-contract=off, IEEE '/'
 * and sqrt(), expressions evaluated left to right as written (DESIGN.md
 * reading A-R23).
 *
 * Array conventions (host memory, caller-owned, copied during the call):
 *   nodes  X, Y : (ni+1)*(nj+1) doubles, index j*(ni+1)+i
 *   state  U    : ni*nj*4 doubles, index (j*ni+i)*4+k, k = rho, rho u, rho v, rho E
 *   i-face metrics: (ni+1)*nj*3 doubles, index (j*(ni+1)+i)*3 + {nx, ny, A}
 *   j-face metrics: ni*(nj+1)*3 doubles, index (j*ni+i)*3 + {nx, ny, A}
 *   volumes: ni*nj doubles, index j*ni+i
 * Every function returns 0 on success or an ORC_ERR_* code.
 */
#ifndef SFV_ORACLE_H
#define SFV_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_GEOMETRY = 2, ORC_ERR_STATE = 3,
       ORC_ERR_SEQUENCE = 4 };
enum { ORC_BC_INFLOW = 0, ORC_BC_OUTFLOW = 1, ORC_BC_SLIP_WALL = 2, ORC_BC_NOSLIP_WALL = 3 };
enum { ORC_LIM_VAN_ALBADA = 0, ORC_LIM_VAN_ALBADA2 = 1, ORC_LIM_NONE = 2 };
enum { ORC_RK4_CLASSIC = 0, ORC_RK2_HEUN = 1, ORC_RK4_JAMESON = 2 };
enum { ORC_RES_EULER = 0, ORC_RES_LINEAR = 1 };

typedef struct {
    int32_t ni, nj;
    double gamma;
    double muscl_eps, muscl_kappa;
    int32_t limiter;
    double lim_delta;
    double harten_eps;
    int32_t rk;
    double cfl, dt_fixed;
    int32_t bc[4];              /* W, E, S, N */
    double inflow_U[4][4];      /* conserved inflow state per edge */
    int64_t max_history;
    int32_t residual_kind;      /* test hook: ORC_RES_LINEAR => R = rate*V*U */
    double linear_rate;
    /* Navier-Stokes (Eq. 2 viscous flux; readings N-R*): */
    int32_t viscous;            /* 0 = Euler, 1 = Navier-Stokes */
    double mu, prandtl, gas_R;  /* constant viscosity, Prandtl number, gas constant */
} orc_config;

typedef struct orc_ctx orc_ctx;

/* ---- pointwise pieces (exposed so tests can pin each one) ---- */
int orc_metrics(int32_t ni, int32_t nj, const double *X, const double *Y,
                double *iface, double *jface, double *vol, int64_t *bad_cell);
int orc_primitive(const double U[4], double gamma, double prim[4]);
double orc_limiter(int32_t kind, double a, double b, double delta);
void orc_muscl(const double w[4], double eps, double kappa, int32_t kind,
               double delta, double *qL, double *qR);
int orc_roe_flux(const double QL[4], const double QR[4], double nx, double ny,
                 double gamma, double harten_eps, double F[4]);
int orc_split(int32_t n, int32_t parts, const int32_t *weights, int32_t *starts);
/* viscous normal flux F_v . n (Eq. 2) from the face gradients
 * g = (u_x, u_y, v_x, v_y, T_x, T_y) and face values u, v (reading N-R3) */
void orc_viscous_flux(const double g[6], double u, double v, double nx, double ny, double mu, double k,
                      double Fv[4]);
int orc_stable_dt(int32_t ni, int32_t nj, const double *X, const double *Y, const double *U, double gamma,
                  double cfl, double *dt);

/* ---- whole-solver mirror of the sfv C ABI ---- */
int orc_create(const orc_config *cfg, const double *X, const double *Y, orc_ctx **out);
int orc_partition(orc_ctx *c, int32_t px, int32_t py, const int32_t *wx, const int32_t *wy);
int orc_partition_map(const orc_ctx *c, int32_t block, int32_t out8[8]);
int orc_set_state(orc_ctx *c, const double *U);
int orc_step(orc_ctx *c, int32_t nsteps);
int orc_get_state(const orc_ctx *c, double *U);
int orc_get_residual_norms(const orc_ctx *c, int64_t first, int64_t count, double *out);
int orc_get_dt(const orc_ctx *c, int64_t first, int64_t count, double *out);
int orc_residual(orc_ctx *c, const double *U, double *R);
int orc_ghost_frame(orc_ctx *c, const double *U, double *frame);
/* Green-Gauss cell gradients (u_x, u_y, v_x, v_y, T_x, T_y) of U after the
 * ghost fill, ni*nj*6 doubles, index (j*ni+i)*6+q (reading N-R2) */
int orc_gradients(orc_ctx *c, const double *U, double *grad);
int64_t orc_steps_done(const orc_ctx *c);
void orc_error_info(const orc_ctx *c, int64_t out4[4]);
const char *orc_last_error(const orc_ctx *c);
void orc_destroy(orc_ctx *c);

#ifdef __cplusplus
}
#endif
#endif
