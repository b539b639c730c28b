/*
 * sg.h -- C ABI of the B200-native sparse-grid time-discontinuous Galerkin
 * streamline-diffusion strip solver (arXiv:2204.05988, "the paper").
 *
 * Line numbers "l.N" refer to PAPER.md (the paper's LaTeX).  The boundary is
 * plain C: opaque handle, plain pointers and sizes, int status codes.  Every
 * compute step runs in CUDA kernels of libsg.so (sm_100a); there is no CPU
 * fallback: on a machine without a CUDA device sg_create returns SG_ERR_CUDA.
 *
 * Conventions
 *  - Factor domains: x in Omega^(1) subset R^d, v in Omega^(2) subset R^d,
 *    d in {1,2,3} (l.47).  Level l of a factor mesh has nc*2^(l-1) cells per
 *    axis; meshes are the Kuhn triangulation of the box lattice (2D: squares
 *    split along the (1,1) diagonal; 3D: 6 tetrahedra per cube), nested under
 *    halving (l.64-67).  Node numbering: lexicographic lattice order, axis 0
 *    fastest, absent lattice points skipped (L-shape).
 *  - Component grids (l.392-413): active set |l|_1 = L, l1 = 1..L-1 (grid
 *    index g = l1-1); coarse (preconditioner) set |l|_1 = L-1, l1 = 1..L-2.
 *    The paper's L is this L minus one (reading R2).
 *  - Block vector of a grid: S x n1 x n2 fp64, row-major [s][k1][k2]
 *    (time basis index s slowest, v index fastest) = kron(time, x, v) order
 *    (l.406-411).  S = q+1, Legendre time basis on each strip (reading R6).
 *    A set vector is the concatenation of its grids' blocks in grid order
 *    (offsets from sg_grid_offset).  A "spatial" set vector has S = 1.
 *  - Ownership: the handle owns all meshes, factor matrices and workspaces
 *    (device memory).  Vector arguments are caller-owned DEVICE pointers
 *    unless a function says "host or device"; they must not alias unless
 *    stated.  All work is enqueued on the handle's stream (sg_create); calls
 *    returning values computed on the device synchronise that stream.
 *    Handles that share a device must share that stream (or be serialised by
 *    the caller): the pass-2 kernels stage their per-level coefficient tables
 *    in the module's constant bank right before each launch.
 *  - Errors: functions return SG_OK (0) or an SG_ERR_* code; sg_last_error()
 *    returns a thread-local message.  After SG_ERR_CUDA the handle must be
 *    destroyed.
 */
#ifndef SG_H
#define SG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_ERR_ARG 1
#define SG_ERR_CUDA 2
#define SG_ERR_STATE 3
#define SG_ERR_UNSUPPORTED 4
#define SG_ERR_NOCONV 5   /* iteration limit reached before the tolerance (result still written) */

#define SG_MESH_BOX 0
#define SG_MESH_LSHAPE 1 /* [-1,1]^2 minus the open quadrant {x>0, y<0} */

#define SG_SET_ACTIVE 0
#define SG_SET_COARSE 1
#define SG_FACTOR_X 0
#define SG_FACTOR_V 1

typedef struct sg_problem sg_problem;

/* beta = sum_r a_r(x) b_r(v) e_{axis_r}  (l.486-488); a, b affine:
 * a(x) = a[0] + sum_i a[1+i] x_i, b(v) = b[0] + sum_i b[1+i] v_i;
 * axis in 0..2d-1 (0..d-1 x axes, d..2d-1 v axes). */
typedef struct {
    int axis;
    double a[4];
    double b[4];
} sg_beta_term;

/* rank-1 initial value term coef * gx(x) * gv(v), g(y) = s exp(-|y-c|^2 / w) */
typedef struct {
    double coef;
    double xc[3], xw, xs;
    double vc[3], vw, vs;
} sg_gauss_term;

typedef struct {
    int d;           /* 1..3 */
    int nc;          /* cells per axis on level 1 */
    int L;           /* combination level, >= 2 */
    int q;           /* dG order in time: 0 or 1 */
    int xkind, vkind;/* SG_MESH_* (L-shape only for d = 2) */
    double xlo[3], xhi[3], vlo[3], vhi[3];
    double tau;      /* strip length */
    double delta;    /* streamline-diffusion parameter; <= 0 selects h_min (reading R5) */
    double sigma;    /* constant reaction coefficient (l.487, p q constant) */
    int nbeta;       /* <= 6 */
    sg_beta_term beta[6];
    int nu0;         /* <= 4 */
    sg_gauss_term u0[4];
    int inflow;      /* 0: g = 0; 1: g = u0(r - beta t), constant beta, d = 1 (configs[0]) */
} sg_config;

/* ---- lifecycle ---------------------------------------------------------- */
/* Validate cfg, select the CUDA device's stream (cudaStream_t, NULL = legacy
 * default), expand the Kronecker terms of A^(delta) (l.462-477) on the host.
 * Errors: SG_ERR_ARG (invalid cfg), SG_ERR_CUDA (no device), SG_ERR_UNSUPPORTED. */
int sg_create(const sg_config* cfg, void* stream, sg_problem** out);
/* Build the nested meshes of both factors for levels 1..L-1 on the device:
 * lattice coordinates, ELL sparsity pattern, prolongation E_{l<-l-1} and its
 * transpose (l.64-67, l.506).  Bit-exact, deterministic. */
int sg_build_meshes(sg_problem* P);
/* Assemble every factor matrix the term list needs on every level, exactly
 * (eq. (14) l.450-461, l.486-504), precombine time blocks, allocate solver
 * workspaces.  Requires sg_build_meshes. */
int sg_assemble_factors(sg_problem* P);
void sg_destroy(sg_problem* P);
const char* sg_last_error(void);

/* ---- queries ------------------------------------------------------------ */
int sg_S(const sg_problem* P);
int sg_num_grids(const sg_problem* P, int set);
int sg_grid_info(const sg_problem* P, int set, int g, int* l1, int* l2, int64_t* n1, int64_t* n2);
/* offset (in doubles) of grid g in a set vector with S_vec time coefficients */
int64_t sg_grid_offset(const sg_problem* P, int set, int g, int S_vec);
int64_t sg_set_size(const sg_problem* P, int set, int S_vec);
double sg_delta(const sg_problem* P);
/* mesh of factor (SG_FACTOR_X/V) at level: n nodes, ELL width W, lattice m */
int sg_mesh_info(const sg_problem* P, int factor, int level, int64_t* n, int* width, int* m);
/* copy to HOST: lattice (n*d int32, node-major), pattern cols (n*W int32,
 * row-major, ascending, -1 padded); any pointer may be NULL */
int sg_mesh_export(const sg_problem* P, int factor, int level, int32_t* lattice, int32_t* cols);
/* copy to HOST the prolongation E_{level<-level-1} (level >= 2) as ELL width 2
 * (n_fine*2 cols, vals; -1/0 padded) and the restriction E^T (n_coarse*W) */
int sg_transfer_export(const sg_problem* P, int factor, int level, int32_t* pcols, double* pvals,
                       int32_t* rcols, double* rvals);
/* Kronecker terms: count, then term t's (S x S) time block (host, row-major)
 * and its x/v factor-matrix spec ids */
int sg_num_terms(const sg_problem* P);
int sg_term_info(const sg_problem* P, int t, double* Tblock, int* xspec, int* vspec);
int sg_num_specs(const sg_problem* P, int factor);
/* spec: kind (0 vol, 1 face); weight[10] coefficients of
 * [1, y0, y1, y2, y0y0, y0y1, y0y2, y1y1, y1y2, y2y2]; trial_d/test_d (-1 none);
 * chi_axis/chi_sign (chi_{sign*y_axis>0}, axis -1 none); face_axis/face_sign */
int sg_spec_info(const sg_problem* P, int factor, int spec, int* kind, double* weight, int* trial_d,
                 int* test_d, int* chi_axis, int* chi_sign, int* face_axis, int* face_sign);
/* copy to HOST the factor matrix values (n*W, row-major on the ELL pattern) */
int sg_factor_export(const sg_problem* P, int factor, int spec, int level, double* vals);

/* ---- the hot path -------------------------------------------------------- */
/* Y = A^(delta)_{l,l} X on ONE component grid (set, g): the matrix-free strip
 * operator sum_t T_t (x) A_t (x) B_t (l.462-477, application order l.516-532).
 * X, Y: device, S x n1 x n2, must not alias. */
int sg_apply_strip_operator(sg_problem* P, int set, int g, const double* X, double* Y);
/* Y = A^(delta) X on the active set including all cross-grid blocks
 * A_{l,l'} = E^T A_F E (l.506-516).  X, Y: device active set vectors (S). */
int sg_apply_full(sg_problem* P, const double* X, double* Y);
/* Y = (Tb (x) M^x (x) M^v) X over the active set with cross-grid blocks;
 * Tb: HOST row-major S_out x S_in.  Used for the jump load (l.94) and L2 norms. */
int sg_apply_mass_full(sg_problem* P, const double* Tb, int S_out, int S_in, const double* X, double* Y);
/* Kronecker-factored transfer along one factor of a block [S][n1][n2]:
 * prolongate: out = E_{lf<-lc} in (+ beta*out), restrict: out = E^T in (+ beta*out);
 * factor selects the axis, level_other the level of the other factor. */
int sg_prolongate(sg_problem* P, int factor, int lf, int lc, int level_other, int S, const double* in,
                  double* out, double beta);
int sg_restrict(sg_problem* P, int factor, int lc, int lf, int level_other, int S, const double* in,
                double* out, double beta);
/* combination (l.557-565): du_l = dhat_l - (E^(1) x Id) dhat_{l1-1,l2};
 * dhat_active/du_active: active set vectors, dhat_coarse: coarse set vector (S). */
int sg_combine(sg_problem* P, const double* dhat_active, const double* dhat_coarse, double* du_active);
/* U_0^- = I_L u0: nodal interpolants on active and coarse grids, combined (reading R8).
 * u: active spatial vector (S = 1). */
int sg_interp_u0(sg_problem* P, double* u);
/* right-hand side of strip j >= 1 (eq. (4)): jump load from trace_prev (active
 * spatial vector U_{j-1}^-) plus the inflow load (cfg.inflow).  b: active (S). */
int sg_rhs(sg_problem* P, int j, const double* trace_prev, double* b);
/* Richardson with the combination preconditioner (l.540-566), entirely on the device
 * (one CUDA graph with conditional nodes; the only host synchronisation is at the end).
 * b, u: active (S) vectors; u is used as initial guess (zero it for the paper's
 * u^(0) = 0).  du = P^{-1} r is the preconditioned residual; the step is u -= omega du
 * with omega = 1 (the paper) or, after the safeguard of reading R13 engaged, the
 * residual-minimising omega.  Stops when ||du||_{L2(I_j x Omega)} <= rtol*||u||.
 * Inner block solves (15): BiCGStab to relative residual inner_rtol (cap 500).
 * Returns SG_ERR_NOCONV when max_iter iterations did not reach rtol (u, iters and
 * last_norm are still written), SG_ERR_STATE on a non-finite update. */
int sg_solve_strip(sg_problem* P, const double* b, double* u, double rtol, double inner_rtol, int max_iter,
                   int* iters, double* last_norm);
/* nsteps strips starting at strip j0 >= 1: trace (active spatial vector,
 * HOST or DEVICE) holds U_{j0-1}^- on entry and U_{j0+nsteps-1}^- on exit.
 * The strips are enqueued back to back (max_iter 200 each) and the handle's stream is
 * synchronised once at the end; SG_ERR_NOCONV if any strip solve hit max_iter. */
int sg_step(sg_problem* P, int j0, int nsteps, double* trace, double rtol, double inner_rtol);

/* ---- instrumentation ----------------------------------------------------- */
/* Counters since the last reset (synchronises the handle's stream): strip-operator
 * applies and DOFs applied (the block solves of the strip solver count on the device,
 * applies issued through sg_apply_strip_operator on the host), our kernel launches
 * (graph executions are expanded to the kernels they ran), Richardson and inner
 * (BiCGStab) iterations. */
int sg_stats(sg_problem* P, int64_t* n_applies, int64_t* dof_applied, int64_t* launches,
             int64_t* outer_iters, int64_t* inner_iters);
/* Solver health since the last reset: strip solves that stopped at max_iter, solves
 * stopped by a non-finite update, inner block solves that stopped at their iteration
 * cap, inner BiCGStab breakdowns (a grid's rho or omega became 0 / non-finite; the grid
 * keeps its last iterate).  A bench line with non-zero counts is flagged. */
int sg_solver_health(sg_problem* P, int64_t* outer_unconverged, int64_t* outer_nonfinite, int64_t* inner_maxit,
                     int64_t* inner_breakdowns);
int sg_reset_stats(sg_problem* P);
/* number of strip solves (since the last reset) in which the outer Richardson
 * iteration switched to residual-minimising step lengths because the update
 * norm grew (safeguard, reading R13); SG_OUTER=1 disables it */
int sg_outer_switches(sg_problem* P, int64_t* switches);
/* Update norms ||du||_{L2(I_j x Omega)} and step lengths omega of every outer iteration of
 * the last strip solve (at most 256); *n = its iteration count (host arrays, may be NULL). */
int sg_solve_history(sg_problem* P, int max_n, double* nd, double* omega, int* n);
/* Timing mode: device timestamps (globaltimer, in the captured graphs too) bracket every
 * strip-operator apply; sg_kernel_time returns the summed device time (ms) of the applies
 * that did work (converged grids excluded), their count, their algorithmic bytes (read X +
 * write Y + the factor data the launched kernels read) and algorithmic FLOPs (2 per
 * multiply-add on the structural nonzeros of the factor matrices). */
int sg_set_timing(sg_problem* P, int on);
int sg_kernel_time(sg_problem* P, double* ms, int64_t* launches, double* alg_bytes, double* alg_flops);

#ifdef __cplusplus
}
#endif
#endif
