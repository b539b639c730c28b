// Internal data structures of libsg (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/sg.h"

namespace sg {

constexpr int MAXD = 3;
constexpr int NPOLY = 10;   // [1, y0, y1, y2, y0y0, y0y1, y0y2, y1y1, y1y2, y2y2]
constexpr int MAXS = 2;     // q <= 1
constexpr int MAX_ENTRIES = 128;   // gather entries per launch (kernel parameter space allows > 4 KB on sm_100)
constexpr int MAX_FANOUT = 12;
constexpr int MAX_SEG = 64;

void set_error(const std::string& msg);
#define SG_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            ::sg::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));      \
            return SG_ERR_CUDA;                                                        \
        }                                                                              \
    } while (0)
#define SG_TRY(call)                 \
    do {                             \
        int r_ = (call);             \
        if (r_ != SG_OK) return r_;  \
    } while (0)

// Factor matrix spec (eq. (14); see oracle/fem.py for the same definition)
struct Spec {
    int kind = 0;          // 0 vol, 1 face
    double w[NPOLY] = {0}; // polynomial weight
    int trial_d = -1, test_d = -1;
    int chi_axis = -1, chi_sign = 0;
    int face_axis = -1, face_sign = 0;
    bool same(const Spec& o) const;
};


struct Term {
    double T[MAXS * MAXS];  // row-major S x S (row = test s, col = trial s')
    int xs, vs;             // spec ids in the x / v factor
};

// stencil offsets of a box-lattice level (sorted ascending; slot k <-> offset)
struct StencilOff {
    int64_t off[15];
};

// one level of one factor mesh
struct Level {
    int64_t n = 0;
    int m = 0;                  // lattice points per axis
    int32_t* lat = nullptr;     // [d][n]
    int32_t* cols = nullptr;    // [W][n] ELL pattern (column-major ELL), -1 padded
    int32_t* pcols = nullptr;   // prolongation from level-1: [2][n]
    double* pvals = nullptr;
    int32_t* rcols = nullptr;   // restriction to level-1: [W][n_{l-1}]
    double* rvals = nullptr;
    std::vector<double*> fm;    // per spec id: [W][n], nullptr if unused
    std::vector<double*> fst;   // per spec id: stencil format [W][n] (box lattices), nullptr if unused
    std::vector<double*> fcls;  // per spec id: class table [27][W] if translation invariant
    uint8_t* bflag = nullptr;   // 1 for lattice-boundary nodes
    uint8_t* bmask = nullptr;   // x-levels: bit j set when boundary-only v-group j has this row in its face (null: use bflag)
    int64_t nbnd = 0;           // number of boundary nodes
    StencilOff so;              // stencil offsets (box lattices)
};

struct Factor {
    int kind = SG_MESH_BOX;
    int d = 1;
    int nc = 2;
    double lo[MAXD] = {0}, hi[MAXD] = {0};
    int W = 3;                   // ELL width 2^(d+1)-1
    std::vector<Level> lev;      // index = level (0 unused)
    std::vector<Spec> specs;
    int add_spec(const Spec& s);  // dedup
};

// gather entry: out[s_out] += scale * (M along dir) in[s_in]
struct Entry {
    const double* in;
    const double* vals;
    double scale;
    int s_out, s_in;
};
struct EntryList {
    int ne;
    int sbeg[3];   // entries sorted by s_out: [sbeg[s], sbeg[s+1]) (set by launch_gather)
    Entry e[MAX_ENTRIES];
};
struct FanoutList {
    int no;
    const double* vals[MAX_FANOUT];
    double* out[MAX_FANOUT];
};

// combined (time-mixed) matrix of one group at one level
struct CombEntry {
    int s_out, s_in;
    double* vals;   // [W][n] device (owned)
    double* st = nullptr;   // stencil format (box lattice of the other factor), owned
    double* ctab = nullptr; // class table [27][W] if translation invariant, owned
    int64_t nnz = 0;        // structural nonzeros (FLOP count)
};
struct Group {                 // terms sharing one spec on the "inner" factor
    int spec;                  // shared spec id (v-spec for lower/x-groups, x-spec for upper)
    std::vector<int> terms;
    bool bonly = false;        // other-factor matrices live on boundary rows only (face terms)
    // combined matrices of the OTHER factor per level: comb[level] = entries
    std::vector<std::vector<CombEntry>> comb;
};

constexpr int MAXG = 40;   // v-groups handled by the stencil pass-1 kernels (configs[3] has > 24)
struct VfanParams {
    int ng, ng_int;
    const double* vst[MAXG];
    double* out[MAXG];
};
struct XgatEntry {
    const double* in;
    const double* cst;
    int s_out, s_in, bonly;
    double scale;
    const double* ctab = nullptr;   // class-compressed rows [27][W] (translation-invariant matrices) or null
};
struct XfanParams {
    int ng, ng_int;
    const double* cst[MAXG];
    const double* ctab[MAXG];
    double* out[MAXG];
};
struct XgatParams {
    int ne;
    XgatEntry e[MAX_ENTRIES];
};

constexpr int MAX_JOBS = 36;
struct Job {
    const double* in;
    const double* add;
    double* out;
    const int32_t* cols;
    const double* vals;
    int64_t n1_in, n2_in, nrows_out;
    double scale;
    int S, dir, W, blk0;
    int64_t opitch = 0;   // output row pitch (0: natural n2_out)
    int box_mf = 0;       // transfer on a box lattice: fine lattice points per axis (0: use the ELL arrays)
    int box_d = 0;        // ... and its dimension (prolongation jobs, W = 2)
    const uint8_t* rmask = nullptr;   // box transfers: only the x-rows r with bit rbit of rmask[r] set are computed
    int rbit = 0;                     // (face groups of the cross-grid apply live on the rows of their own face)
};
struct JobList {
    int nj, total_blocks;
    Job j[MAX_JOBS];
};

struct GraphKey {
    const double* X;
    double* Y;
    int S_out, S_in;
    bool mass;
    double T[4];
    bool same(const GraphKey& o) const {
        if (X != o.X || Y != o.Y || S_out != o.S_out || S_in != o.S_in || mass != o.mass) return false;
        for (int i = 0; i < 4; ++i)
            if (T[i] != o.T[i]) return false;
        return true;
    }
};
struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    int64_t nlaunch;
};

// Device-resident state of the strip solver (strip_solver.cu), one per handle.  The
// cond_* words mirror the conditional-node values for the uncaptured (host-loop) path.
struct SolveCtl {
    int it, mr, have_r, done;        // outer iteration; MR steps on; r current; 0 run / 1 conv / 2 max_iter / 3 non-finite
    int inner_it, cond_inner, cond_outer, cond_need_r, cond_mr, pad0;
    double nd, nd_prev, nu2, omega;
    double dots[4];
    // cumulative counters (reset by sg_reset_stats)
    long long outer_iters, inner_iters, need_r_runs, mr_runs, mr_switches;
    long long inner_breakdowns, inner_maxit, outer_unconverged, outer_nonfinite;
    long long n_applies, timed_applies;
    double dof_applied, alg_bytes, alg_flops, apply_ns;
    unsigned long long t0[64];       // per-slot start stamps (concurrent applies)
    int act[64];                     // grid active in the current inner iteration
    double hist_nd[256];             // ||du|| of every outer iteration of the last strip solve
    double hist_om[256];             // its step length omega
};

struct Grid {
    int l1, l2;
    int64_t n1, n2;
    int64_t off1;   // offset in doubles for S=1 vectors (multiply by S for S-vectors)
};

struct Segs {  // block -> segment map for batched vector kernels over a set vector
    int nseg;
    int64_t off[MAX_SEG + 1];   // element offsets (for the given S)
    int blk[MAX_SEG + 1];       // first block of each segment
};

}  // namespace sg

struct sg_problem {
    sg_config cfg;
    cudaStream_t stream = nullptr;
    int S = 1;
    int F = 1;                      // finest level L-1
    double delta = 0;
    sg::Factor fx, fv;
    std::vector<sg::Term> terms;
    std::vector<sg::Group> vgroups; // grouped by v-spec; comb = x-matrices (lower part / diag v-first)
    std::vector<sg::Group> xgroups; // grouped by x-spec; comb = v-matrices (upper part)
    int mass_x = -1, mass_v = -1;   // spec ids of the unweighted mass
    std::vector<int> vorder;        // v-groups, interior first then boundary-only
    std::vector<int> xorder;        // x-groups, interior first then boundary-only
    int nxg_int = 0;
    int ng_int = 0;
    std::vector<sg::Grid> active, coarse;
    bool meshes_built = false, assembled = false;
    // workspaces
    double* wsZ = nullptr; size_t wsZ_n = 0;      // fanout outputs / chain buffers
    double* wsA = nullptr; size_t wsA_n = 0;      // Horner ping
    double* wsB = nullptr; size_t wsB_n = 0;      // Horner pong
    double* wsH = nullptr;                        // per-target Horner buffers [2][active S-set]
    double* red = nullptr;                        // reduction partials
    double* scal = nullptr;                       // per-grid scalars (BiCGStab)
    std::vector<double*> vec;                     // solver vectors
    double* trace_dev = nullptr;
    double* dinv = nullptr;                       // block-Jacobi inverse (solve set)
    bool use_tma = true;           // SG_NO_TMA: pass 2 by the register line sweep k_xfanin
    bool use_graphs = true;        // SG_NO_GRAPHS: cross-grid applies and strip solves uncaptured
    sg::SolveCtl* ctl = nullptr;   // device-resident solver state
    sg::SolveCtl* hctl = nullptr;  // pinned host copy
    const double* skip = nullptr;  // convergence flag of the grid being applied (kernels exit if != 0)
    bool capturing = false;        // enqueueing into a strip-solve graph
    bool in_solve = false;         // applies are counted on the device (inner control kernel)
    std::vector<cudaStream_t> cap_streams;   // capture streams of nested conditional bodies
    // concurrent per-grid applies in the block solver (small configurations, launch-latency bound):
    // one stream and one private intermediate workspace per solve grid
    bool par_applies = false;
    // concurrent cross-grid transfer chains (one branch per group, small configurations)
    bool par_cross = false;
    std::vector<cudaStream_t> cx_streams;
    std::vector<double*> cx_ws, cx_h, cx_y;
    size_t cx_ws_n = 0;
    int64_t cx_h_n = 0, cx_y_n = 0;
    cudaEvent_t ev_cx_fork = nullptr;
    std::vector<cudaEvent_t> ev_cx_join;
    int stamp_slot = 63;           // timestamp slot of the apply being enqueued
    std::vector<cudaStream_t> par_streams;
    std::vector<double*> par_ws;
    std::vector<size_t> par_ws_n;
    cudaEvent_t ev_fork = nullptr;
    std::vector<cudaEvent_t> ev_join;
    struct SolveGraph {
        const double *b, *u;
        double rtol, inner_rtol;
        int max_iter, mode, timing;
        cudaGraphExec_t exec;
        int64_t l_pre, l_outer, l_need_r, l_mr, l_inner;   // launches per region execution
    };
    std::vector<SolveGraph> solve_graphs;
    std::vector<double> gdof, gbytes, gflops;   // per solve grid (active then coarse): DOF, alg. bytes / flops per apply
    cudaStream_t gstream = nullptr;   // library stream for captured graphs
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    std::vector<sg::GraphEntry> graphs;
    // pass 2 line sweeps, per x-level: class tables [3^d][groups][W] of the combined x matrices,
    // interior-group class tables [3^d][ng_int][W] and the interior-class coefficients
    std::vector<double*> xfi_tab;
    std::vector<double*> xfi_itab;
    std::vector<std::vector<double>> xfi_cint;
    // ... and per boundary class the boundary-only (face) groups with a nonzero row or column there
    std::vector<std::vector<uint8_t>> xfi_cmask;
    // whole-x pass 2 (tiny x-lattices), per x-level: compact [group][pair] coefficient table
    std::vector<double*> xw_tab;   // non-null when the whole-x tables exist
    std::vector<double*> xw_dev;
    std::vector<int> xw_np;
    // fused whole-x apply (tiny x-lattices): [g][pair] tables per x-level, SG_NO_FUSED disables
    std::vector<double*> fw_dev;
    int fw_np = 0;
    bool use_fused = true;
    // fused batched apply for d = 1 (d1fused.cu): per-level device tables
    bool d1_ok = false;
    std::vector<double**> d1_bst;   // [l2] -> [nb] stencil-format v matrices
    std::vector<void*> d1_ent;      // [l1] -> entries grouped by v-group
    std::vector<int*> d1_ebeg;      // [l1] -> [nb + 1] entry ranges
    std::vector<int> d1_nent;
    // L2-resident column chunks of the two-pass apply: intermediates per chunk (bytes; 0 = off)
    int64_t l2_chunk_bytes = 0;
    int64_t l2_chunk_mincols = 64;
    // batched cross-grid lower part: stage-0 fan-outs of all v-groups and the Horner
    // results per target and group (even pitch); also used by the batched upper part
    double* cross_q = nullptr;
    double* cross_h = nullptr;
    bool cross_batched_tried = false;
    int64_t cross_q_n = 0, cross_h_n = 0;
    bool use_cross_batched = true; // SG_NO_CROSS_BATCH disables
    int outer_mode = 0;            // 0 Richardson + minimal-residual safeguard, 1 plain Richardson, 2 MR always
    int64_t mr_switches = 0;
    // moment pass 1 (vmoment.cu), per v-level
    std::vector<int> vm_ok;        // moment tables verified
    std::vector<double*> vm_tab;   // [3^d][10][W] shifted-moment class tables
    std::vector<std::vector<double>> vm_int;   // interior class [10][15]
    std::vector<int*> vm_blist;    // boundary v-nodes
    std::vector<int> vm_nb;
    std::vector<int> vm_slot;      // interior group position -> monomial slot
    int64_t vm_tab_n = 0;          // doubles of one level's moment class table (byte count)
    int vm_nchi = 0;               // boundary-only groups handled as chi-weighted moments (0: stencil kernel)
    int vm_chax[6] = {0}, vm_chkeep[6] = {0};
    // instrumentation
    // (host-side counters of applies issued outside the strip solver; the solver counts on the device)
    int64_t n_applies = 0, dof_applied = 0, launches = 0;
    bool timing = false;           // globaltimer stamps around every strip-operator apply (k_tstamp)
    bool verbose = false;
    // per factor/level/spec structural nonzeros (|a_ij| > 1e-12 max|a|) for the FLOP count
    std::vector<std::vector<int64_t>> nnz_x, nnz_v;
};

namespace sg {
// mesh.cu
int build_factor_meshes(sg_problem* P, Factor& f, int F);
// assemble.cu
int assemble_spec(sg_problem* P, Factor& f, int spec, int level);
// kernels.cu launch helpers
int launch_fanout(sg_problem* P, int dir, int W, int S, int64_t n1_in, int64_t n2_in, int64_t nrows_out,
                  const int32_t* cols, const double* in, const FanoutList& fl);
int launch_gather(sg_problem* P, int dir, int W, int S_out, int64_t n1_in, int64_t n2_in, int64_t nrows_out,
                  const int32_t* cols, const EntryList& el, double* out, double beta);
int launch_axpby(sg_problem* P, int64_t n, double a, const double* x, double b, double* y);
int launch_copy(sg_problem* P, int64_t n, const double* x, double* y);
int launch_zero(sg_problem* P, int64_t n, double* y);
constexpr int MAX_SUM = 32;
int launch_sum_into(sg_problem* P, int64_t n, int k, double* const* xs, double* y);
int launch_ell_to_stencil(sg_problem* P, int64_t n, int W, const int32_t* cols, const double* vals,
                          const StencilOff& so, double* out);
int launch_vfan_st(sg_problem* P, int d, int S, int64_t n1, int64_t n2, const StencilOff& so, const uint8_t* xflag,
                   const VfanParams& vp, const double* X, int64_t opitch = 0, int64_t c0 = 0, int64_t c1 = 0,
                   int maskmode = 0);
int launch_xgat_st(sg_problem* P, int d, int S_out, int64_t n1, int64_t n2, const StencilOff& so,
                   const uint8_t* xflag, const XgatParams& ep, double* Y, double beta, int m = 0);
int class_compress(sg_problem* P, const Factor& f, int l, const double* st, double** ctab);
int launch_jobs(sg_problem* P, std::vector<Job>& jobs);
int launch_vgat_st(sg_problem* P, int d, int S_out, int64_t n1, int64_t n2, const StencilOff& so,
                   const XgatParams& ep, double* Y, double beta, const uint8_t* xflag = nullptr);
int launch_xfan_st(sg_problem* P, int d, int S, int64_t n1, int64_t n2, const StencilOff& so, int m,
                   const uint8_t* xflag, const XfanParams& fp, const double* X);
// xfanin.cu
int prepare_xfanin(sg_problem* P);
int launch_xfanin(sg_problem* P, int l1, int64_t n1, int64_t n2, const double* Z, int64_t gstride, double* Y,
                  double beta);
int launch_xwhole(sg_problem* P, int l1, int64_t n1, int64_t n2, int64_t pitch, const double* Z, int64_t gstride,
                  double* Y);
int prepare_fwhole(sg_problem* P);

int launch_fwhole(sg_problem* P, int l1, int l2, int64_t n2, const double* X, double* Y);
// d1fused.cu
int prepare_d1fused(sg_problem* P);
void free_d1fused(sg_problem* P);
int launch_d1fused(sg_problem* P, int n, const Grid* const* grids, const double* const* X, double* const* Y,
                   const double* const* skips, double* fbytes);
int launch_tstamp_batch(sg_problem* P, int n, const double* const* skips, const double* bytes, const double* flops);
double apply_flops(const sg_problem* P, const Grid& g);
// vmoment.cu
int prepare_vmom(sg_problem* P);
int launch_vmom(sg_problem* P, int l2, int64_t nrows, int64_t n2, int64_t pitch, const double* X, double* const* outs,
                const uint8_t* xflag, int64_t n1x, int64_t c0 = 0, int64_t c1 = 0);
// xfanin_tma.cu
int launch_xfanin_tma(sg_problem* P, int l1, int64_t n1, int64_t n2, int64_t pitch, const double* Z,
                      int64_t gstride, double* Y, int64_t ypitch = 0, bool stage_tab = true);
// solver.cu
int apply_diag(sg_problem* P, const Grid& g, const double* X, double* Y, const double* skip = nullptr);
int apply_cost(sg_problem* P, const Grid& g, double* bytes, double* flops);
int count_nnz(sg_problem* P);
int pass1_vgroups(sg_problem* P, int l1, int l2, const double* X, double* const* outs, int64_t pitch,
                  double* fbytes = nullptr, int64_t c0 = 0, int64_t c1 = 0, bool fine_mask = false);
int apply_cross_prepare(sg_problem* P);
int apply_cross(sg_problem* P, const std::vector<Term>* terms_override, const double* Tb, int S_out, int S_in,
                const double* X, double* Y);
int64_t set_size(const sg_problem* P, int set, int S);
int build_block_jacobi(sg_problem* P);
// strip_solver.cu
int solver_init(sg_problem* P);
int solver_destroy(sg_problem* P);
int sync_stats(sg_problem* P);
int reset_device_stats(sg_problem* P);
int combine(sg_problem* P, int S, const double* dhat_a, const double* dhat_c, double* du);
int solve_strip(sg_problem* P, const double* b, double* u, double rtol, double inner_rtol, int max_iter, int* iters,
                double* last);
int step(sg_problem* P, int j0, int nsteps, double* trace_dev, double rtol, double inner_rtol);
// solver.cu (data)
int rhs(sg_problem* P, int j, const double* trace, double* b);
int trace_of(sg_problem* P, const double* u, double* tr);
int interp_u0(sg_problem* P, double* u);
__global__ void k_tstamp(SolveCtl* c, const double* skip, int slot, int phase, double bytes, double flops);
int prepare_stencils(sg_problem* P);
}  // namespace sg
