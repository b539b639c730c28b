// C ABI of libsg (include/sg.h).  Argument checking, allocation, dispatch.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "sg_internal.cuh"

namespace sg {
const char* last_error();
int expand_terms(sg_problem* P);
int combine_group(sg_problem* P, Group& g, bool other_is_x);
}  // namespace sg

using namespace sg;

#define CHECK_ARG(cond, msg)      \
    do {                          \
        if (!(cond)) {            \
            set_error(msg);       \
            return SG_ERR_ARG;    \
        }                         \
    } while (0)

extern "C" const char* sg_last_error(void) { return last_error(); }

extern "C" int sg_create(const sg_config* cfg, void* stream, sg_problem** out) {
    CHECK_ARG(cfg && out, "null argument");
    *out = nullptr;
    CHECK_ARG(cfg->d >= 1 && cfg->d <= 3, "d must be 1..3");
    CHECK_ARG(cfg->L >= 2 && cfg->L <= 40, "L must be >= 2");
    CHECK_ARG(cfg->q == 0 || cfg->q == 1, "q must be 0 or 1");
    CHECK_ARG(cfg->nc >= 1, "nc >= 1");
    CHECK_ARG(cfg->tau > 0, "tau > 0");
    CHECK_ARG(cfg->nbeta >= 0 && cfg->nbeta <= 6 && cfg->nu0 >= 0 && cfg->nu0 <= 4, "nbeta <= 6, nu0 <= 4");
    CHECK_ARG(cfg->xkind == SG_MESH_BOX || (cfg->xkind == SG_MESH_LSHAPE && cfg->d == 2), "xkind");
    CHECK_ARG(cfg->vkind == SG_MESH_BOX || (cfg->vkind == SG_MESH_LSHAPE && cfg->d == 2), "vkind");
    CHECK_ARG(cfg->inflow == 0 || cfg->d == 1, "inflow data only for d = 1");
    for (int i = 0; i < cfg->nbeta; ++i) CHECK_ARG(cfg->beta[i].axis >= 0 && cfg->beta[i].axis < 2 * cfg->d, "beta axis");
    for (int i = 0; i < cfg->d; ++i) CHECK_ARG(cfg->xhi[i] > cfg->xlo[i] && cfg->vhi[i] > cfg->vlo[i], "domain bounds");
    if ((cfg->xkind == SG_MESH_LSHAPE || cfg->vkind == SG_MESH_LSHAPE) && (cfg->nc % 2) != 0) {
        set_error("L-shape needs an even number of level-1 cells");
        return SG_ERR_ARG;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_error("no CUDA device: libsg has no CPU fallback");
        return SG_ERR_CUDA;
    }
    sg_problem* P = new (std::nothrow) sg_problem();
    if (!P) return SG_ERR_STATE;
    P->cfg = *cfg;
    P->stream = (cudaStream_t)stream;
    P->verbose = getenv("SG_VERBOSE") != nullptr;
    P->use_graphs = getenv("SG_NO_GRAPHS") == nullptr;
    // fallback of the TMA line sweep (register line sweep k_xfanin)
    P->use_tma = getenv("SG_NO_TMA") == nullptr;
    // fused whole-x apply on the tiny x-lattices (fallback: moment pass 1 + whole-x pass 2)
    P->use_fused = getenv("SG_NO_FUSED") == nullptr;
    // experiment knobs of the L2-resident chunked apply (MB of intermediates per chunk; 0 = off)
    if (getenv("SG_L2_MB")) P->l2_chunk_bytes = (int64_t)(atof(getenv("SG_L2_MB")) * 1048576.0);
    if (getenv("SG_L2_MINCOLS")) P->l2_chunk_mincols = atoi(getenv("SG_L2_MINCOLS"));
    // fallback of the batched cross-grid lower part (also taken when its buffers do not fit)
    P->use_cross_batched = getenv("SG_NO_CROSS_BATCH") == nullptr;
    // outer step length (reading R13): 0 Richardson + MR safeguard, 1 plain, 2 MR always
    P->outer_mode = getenv("SG_OUTER") ? atoi(getenv("SG_OUTER")) : 0;
    if (cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_b, cudaEventDisableTiming) != cudaSuccess) {
        set_error("stream/event creation failed");
        delete P;
        return SG_ERR_CUDA;
    }
    P->S = cfg->q + 1;
    P->F = cfg->L - 1;
    auto setf = [&](Factor& f, int kind, const double* lo, const double* hi) {
        f.kind = kind;
        f.d = cfg->d;
        f.nc = cfg->nc;
        for (int i = 0; i < 3; ++i) {
            f.lo[i] = i < cfg->d ? lo[i] : 0.0;
            f.hi[i] = i < cfg->d ? hi[i] : 0.0;
        }
        f.W = (1 << (cfg->d + 1)) - 1;
    };
    setf(P->fx, cfg->xkind, cfg->xlo, cfg->xhi);
    setf(P->fv, cfg->vkind, cfg->vlo, cfg->vhi);
    // delta = finest edge length (reading R5)
    if (cfg->delta > 0) {
        P->delta = cfg->delta;
    } else {
        const double cells = (double)(cfg->nc) * std::ldexp(1.0, P->F - 1);
        double h = 1e300;
        for (int i = 0; i < cfg->d; ++i) {
            h = std::min(h, (cfg->xhi[i] - cfg->xlo[i]) / cells);
            h = std::min(h, (cfg->vhi[i] - cfg->vlo[i]) / cells);
        }
        P->delta = h;
    }
    int rc = expand_terms(P);
    if (rc != SG_OK) {
        delete P;
        return rc;
    }
    *out = P;
    return SG_OK;
}

extern "C" int sg_build_meshes(sg_problem* P) {
    CHECK_ARG(P, "null handle");
    if (P->meshes_built) return SG_OK;
    SG_TRY(build_factor_meshes(P, P->fx, P->F));
    SG_TRY(build_factor_meshes(P, P->fv, P->F));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    // component grids
    const int L = P->cfg.L;
    int64_t off = 0;
    P->active.clear();
    P->coarse.clear();
    for (int l1 = 1; l1 <= L - 1; ++l1) {
        Grid g{l1, L - l1, P->fx.lev[l1].n, P->fv.lev[L - l1].n, off};
        off += g.n1 * g.n2;
        P->active.push_back(g);
    }
    off = 0;
    for (int l1 = 1; l1 <= L - 2; ++l1) {
        Grid g{l1, L - 1 - l1, P->fx.lev[l1].n, P->fv.lev[L - 1 - l1].n, off};
        off += g.n1 * g.n2;
        P->coarse.push_back(g);
    }
    if (P->active.size() + P->coarse.size() > (size_t)MAX_SEG) {
        set_error("too many component grids");
        return SG_ERR_UNSUPPORTED;
    }
    P->meshes_built = true;
    return SG_OK;
}

extern "C" int sg_assemble_factors(sg_problem* P) {
    CHECK_ARG(P, "null handle");
    if (!P->meshes_built) {
        set_error("sg_build_meshes first");
        return SG_ERR_STATE;
    }
    if (P->assembled) return SG_OK;
    const int F = P->F, S = P->S, L = P->cfg.L;
    for (int l = 1; l <= F; ++l) {
        SG_TRY(assemble_spec(P, P->fx, P->mass_x, l));
        SG_TRY(assemble_spec(P, P->fv, P->mass_v, l));
        for (auto& g : P->vgroups) SG_TRY(assemble_spec(P, P->fv, g.spec, l));
        for (auto& g : P->xgroups) SG_TRY(assemble_spec(P, P->fx, g.spec, l));
    }
    for (auto& g : P->vgroups) SG_TRY(combine_group(P, g, true));
    for (auto& g : P->xgroups) SG_TRY(combine_group(P, g, false));
    SG_TRY(prepare_stencils(P));
    // workspaces
    int64_t maxg = 0;
    // (even row pitch of the pass-2 intermediates, TMA strides are multiples of 16 bytes)
    for (auto& g : P->active) maxg = std::max(maxg, g.n1 * (g.n2 + (g.n2 & 1)));
    for (auto& g : P->coarse) maxg = std::max(maxg, g.n1 * (g.n2 + (g.n2 & 1)));
    const int ng = (int)P->active.size();
    int64_t chain = 0, chain_up = 0;
    for (int pp = 1; pp <= ng; ++pp)
        for (int k = 0; k <= ng - pp; ++k) chain += P->fx.lev[pp].n * P->fv.lev[L - pp - k].n;
    for (int pp = 2; pp <= ng; ++pp)
        for (int k = 0; k <= pp - 1; ++k) chain_up += P->fx.lev[pp - k].n * P->fv.lev[L - pp].n;
    const size_t nbz = std::max(std::max(P->vgroups.size(), P->xgroups.size()), (size_t)1);
    P->wsZ_n = (size_t)std::max<int64_t>(std::max<int64_t>(nbz * S * maxg, S * chain), S * chain_up);
    P->wsA_n = P->wsB_n = (size_t)(S * maxg);
    SG_CUDA(cudaMalloc(&P->wsZ, sizeof(double) * P->wsZ_n));
    SG_CUDA(cudaMemsetAsync(P->wsZ, 0, sizeof(double) * P->wsZ_n, P->stream));   // finite garbage only
    SG_CUDA(cudaMalloc(&P->wsA, sizeof(double) * P->wsA_n));
    SG_CUDA(cudaMalloc(&P->wsB, sizeof(double) * P->wsB_n));
    SG_CUDA(cudaMalloc(&P->wsH, sizeof(double) * 2 * set_size(P, SG_SET_ACTIVE, S)));
    const int64_t Na = set_size(P, SG_SET_ACTIVE, S), Nc = set_size(P, SG_SET_COARSE, S);
    const int64_t nblk = (Na + Nc) / 2048 + 2 * MAX_SEG + 8;
    SG_CUDA(cudaMalloc(&P->red, sizeof(double) * 3 * nblk));
    SG_CUDA(cudaMalloc(&P->scal, sizeof(double) * 10 * (MAX_SEG + 1)));
    SG_CUDA(cudaMemset(P->scal, 0, sizeof(double) * 10 * (MAX_SEG + 1)));
    const int64_t nF = std::max(P->fx.lev[F].n, P->fv.lev[F].n) + 16;
    const int64_t sizes[17] = {Na + Nc, Na + Nc, Na + Nc, Na + Nc, Na + Nc, Na + Nc, Na, Na + Nc, Na + Nc, Na,
                               std::max(Na, 4 * nF), Na, Na, Na + Nc, Na + Nc, Na, Na + Nc};
    P->vec.assign(17, nullptr);
    for (int i = 0; i < 17; ++i) SG_CUDA(cudaMalloc(&P->vec[i], sizeof(double) * sizes[i]));
    SG_TRY(build_block_jacobi(P));
    SG_TRY(count_nnz(P));
    SG_TRY(solver_init(P));
    SG_CUDA(cudaMalloc(&P->trace_dev, sizeof(double) * set_size(P, SG_SET_ACTIVE, 1)));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    P->assembled = true;
    // buffers of the batched cross-grid apply (allocated here, never inside a graph capture)
    SG_TRY(apply_cross_prepare(P));
    return SG_OK;
}

static void free_level(Level& L) {
    cudaFree(L.lat); cudaFree(L.cols); cudaFree(L.pcols); cudaFree(L.pvals); cudaFree(L.rcols); cudaFree(L.rvals);
    cudaFree(L.bflag);
    cudaFree(L.bmask);
    for (double* p : L.fm) cudaFree(p);
    for (double* p : L.fst) cudaFree(p);
    for (double* p : L.fcls) cudaFree(p);
}

extern "C" void sg_destroy(sg_problem* P) {
    if (!P) return;
    cudaStreamSynchronize(P->stream);
    for (auto& L : P->fx.lev) free_level(L);
    for (auto& L : P->fv.lev) free_level(L);
    for (auto* gs : {&P->vgroups, &P->xgroups})
        for (auto& g : *gs)
            for (auto& lv : g.comb)
                for (auto& ce : lv) {
                    cudaFree(ce.vals);
                    cudaFree(ce.st);
                    cudaFree(ce.ctab);
                }
    free_d1fused(P);
    cudaFree(P->wsZ); cudaFree(P->wsA); cudaFree(P->wsB); cudaFree(P->wsH); cudaFree(P->red); cudaFree(P->scal);
    cudaFree(P->cross_q); cudaFree(P->cross_h);
    for (double* t : P->xfi_tab) cudaFree(t);
    for (double* t : P->xfi_itab) cudaFree(t);
    for (double* t : P->vm_tab) cudaFree(t);
    for (double* t : P->xw_dev) cudaFree(t);
    for (double* t : P->fw_dev) cudaFree(t);
    for (int* t : P->vm_blist) cudaFree(t);
    solver_destroy(P);
    for (auto s : P->cx_streams) cudaStreamDestroy(s);
    for (auto e : P->ev_cx_join) cudaEventDestroy(e);
    for (auto w : P->cx_ws) cudaFree(w);
    for (auto w : P->cx_h) cudaFree(w);
    for (auto w : P->cx_y) cudaFree(w);
    if (P->ev_cx_fork) cudaEventDestroy(P->ev_cx_fork);
    for (double* v : P->vec) cudaFree(v);
    cudaFree(P->trace_dev);
    cudaFree(P->dinv);
    for (auto& g : P->graphs) cudaGraphExecDestroy(g.exec);
    if (P->gstream) cudaStreamDestroy(P->gstream);
    if (P->ev_a) cudaEventDestroy(P->ev_a);
    if (P->ev_b) cudaEventDestroy(P->ev_b);
    delete P;
}

// ---------------------------------------------------------------- queries
extern "C" int sg_S(const sg_problem* P) { return P ? P->S : -1; }
extern "C" double sg_delta(const sg_problem* P) { return P ? P->delta : -1.0; }
extern "C" int sg_num_grids(const sg_problem* P, int set) {
    if (!P) return -1;
    if (set == SG_SET_ACTIVE) return P->cfg.L - 1;
    return P->cfg.L - 2;
}
extern "C" int sg_grid_info(const sg_problem* P, int set, int g, int* l1, int* l2, int64_t* n1, int64_t* n2) {
    CHECK_ARG(P && P->meshes_built, "handle / meshes");
    const auto& gs = set == SG_SET_ACTIVE ? P->active : P->coarse;
    CHECK_ARG(g >= 0 && g < (int)gs.size(), "grid index");
    if (l1) *l1 = gs[g].l1;
    if (l2) *l2 = gs[g].l2;
    if (n1) *n1 = gs[g].n1;
    if (n2) *n2 = gs[g].n2;
    return SG_OK;
}
extern "C" int64_t sg_grid_offset(const sg_problem* P, int set, int g, int S_vec) {
    if (!P || !P->meshes_built) return -1;
    const auto& gs = set == SG_SET_ACTIVE ? P->active : P->coarse;
    if (g < 0 || g >= (int)gs.size()) return -1;
    return gs[g].off1 * S_vec;
}
extern "C" int64_t sg_set_size(const sg_problem* P, int set, int S_vec) {
    if (!P || !P->meshes_built) return -1;
    return set_size(P, set, S_vec);
}
static const Factor* factor_of(const sg_problem* P, int f) { return f == SG_FACTOR_X ? &P->fx : &P->fv; }

extern "C" int sg_mesh_info(const sg_problem* P, int factor, int level, int64_t* n, int* width, int* m) {
    CHECK_ARG(P && P->meshes_built, "handle / meshes");
    const Factor* f = factor_of(P, factor);
    CHECK_ARG(level >= 1 && level <= P->F, "level");
    if (n) *n = f->lev[level].n;
    if (width) *width = f->W;
    if (m) *m = f->lev[level].m;
    return SG_OK;
}

template <typename T>
static int ell_to_host_rowmajor(const T* dev, int64_t n, int W, T* host) {
    std::vector<T> tmp((size_t)n * W);
    SG_CUDA(cudaMemcpy(tmp.data(), dev, sizeof(T) * n * W, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < W; ++k) host[i * W + k] = tmp[(size_t)k * n + i];
    return SG_OK;
}

extern "C" int sg_mesh_export(const sg_problem* P, int factor, int level, int32_t* lattice, int32_t* cols) {
    CHECK_ARG(P && P->meshes_built, "handle / meshes");
    CHECK_ARG(level >= 1 && level <= P->F, "level");
    const Factor* f = factor_of(P, factor);
    const Level& L = f->lev[level];
    SG_CUDA(cudaStreamSynchronize(P->stream));
    if (lattice) SG_TRY(ell_to_host_rowmajor<int32_t>(L.lat, L.n, f->d, lattice));
    if (cols) SG_TRY(ell_to_host_rowmajor<int32_t>(L.cols, L.n, f->W, cols));
    return SG_OK;
}

extern "C" int sg_transfer_export(const sg_problem* P, int factor, int level, int32_t* pcols, double* pvals,
                                  int32_t* rcols, double* rvals) {
    CHECK_ARG(P && P->meshes_built, "handle / meshes");
    CHECK_ARG(level >= 2 && level <= P->F, "level");
    const Factor* f = factor_of(P, factor);
    const Level& L = f->lev[level];
    const Level& C = f->lev[level - 1];
    SG_CUDA(cudaStreamSynchronize(P->stream));
    if (pcols) SG_TRY(ell_to_host_rowmajor<int32_t>(L.pcols, L.n, 2, pcols));
    if (pvals) SG_TRY(ell_to_host_rowmajor<double>(L.pvals, L.n, 2, pvals));
    if (rcols) SG_TRY(ell_to_host_rowmajor<int32_t>(L.rcols, C.n, f->W, rcols));
    if (rvals) SG_TRY(ell_to_host_rowmajor<double>(L.rvals, C.n, f->W, rvals));
    return SG_OK;
}

extern "C" int sg_num_terms(const sg_problem* P) { return P ? (int)P->terms.size() : -1; }
extern "C" int sg_term_info(const sg_problem* P, int t, double* Tblock, int* xspec, int* vspec) {
    CHECK_ARG(P && t >= 0 && t < (int)P->terms.size(), "term index");
    if (Tblock)
        for (int i = 0; i < P->S * P->S; ++i) Tblock[i] = P->terms[t].T[i];
    if (xspec) *xspec = P->terms[t].xs;
    if (vspec) *vspec = P->terms[t].vs;
    return SG_OK;
}
extern "C" int sg_num_specs(const sg_problem* P, int factor) {
    return P ? (int)factor_of(P, factor)->specs.size() : -1;
}
extern "C" int sg_spec_info(const sg_problem* P, int factor, int spec, int* kind, double* weight, int* trial_d,
                            int* test_d, int* chi_axis, int* chi_sign, int* face_axis, int* face_sign) {
    CHECK_ARG(P, "null handle");
    const Factor* f = factor_of(P, factor);
    CHECK_ARG(spec >= 0 && spec < (int)f->specs.size(), "spec index");
    const Spec& s = f->specs[spec];
    if (kind) *kind = s.kind;
    if (weight)
        for (int i = 0; i < NPOLY; ++i) weight[i] = s.w[i];
    if (trial_d) *trial_d = s.trial_d;
    if (test_d) *test_d = s.test_d;
    if (chi_axis) *chi_axis = s.chi_axis;
    if (chi_sign) *chi_sign = s.chi_sign;
    if (face_axis) *face_axis = s.face_axis;
    if (face_sign) *face_sign = s.face_sign;
    return SG_OK;
}
extern "C" int sg_factor_export(const sg_problem* P, int factor, int spec, int level, double* vals) {
    CHECK_ARG(P && P->assembled, "handle / assembly");
    const Factor* f = factor_of(P, factor);
    CHECK_ARG(level >= 1 && level <= P->F && spec >= 0 && spec < (int)f->specs.size(), "spec / level");
    const Level& L = f->lev[level];
    if (spec >= (int)L.fm.size() || !L.fm[spec]) {
        set_error("factor matrix not assembled (unused spec)");
        return SG_ERR_STATE;
    }
    SG_CUDA(cudaStreamSynchronize(P->stream));
    return ell_to_host_rowmajor<double>(L.fm[spec], L.n, f->W, vals);
}

// ---------------------------------------------------------------- hot path
#define NEED_ASSEMBLED(P)                                       \
    do {                                                        \
        CHECK_ARG(P, "null handle");                            \
        if (!(P)->assembled) {                                  \
            set_error("sg_assemble_factors first");             \
            return SG_ERR_STATE;                                \
        }                                                       \
    } while (0)

extern "C" int sg_apply_strip_operator(sg_problem* P, int set, int g, const double* X, double* Y) {
    NEED_ASSEMBLED(P);
    const auto& gs = set == SG_SET_ACTIVE ? P->active : P->coarse;
    CHECK_ARG(g >= 0 && g < (int)gs.size(), "grid index");
    CHECK_ARG(X && Y && X != Y, "X, Y must be distinct device pointers");
    return apply_diag(P, gs[g], X, Y);
}

extern "C" int sg_apply_full(sg_problem* P, const double* X, double* Y) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(X && Y && X != Y, "X, Y");
    return apply_cross(P, nullptr, nullptr, P->S, P->S, X, Y);
}

extern "C" int sg_apply_mass_full(sg_problem* P, const double* Tb, int S_out, int S_in, const double* X, double* Y) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(Tb && X && Y && X != Y, "args");
    CHECK_ARG(S_out >= 1 && S_out <= MAXS && S_in >= 1 && S_in <= MAXS, "S_out/S_in");
    return apply_cross(P, nullptr, Tb, S_out, S_in, X, Y);
}

static int transfer(sg_problem* P, int factor, int lf, int lc, int level_other, int S, const double* in, double* out,
                    double beta, bool prolong) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(lf == lc + 1, "transfers are one level at a time (lf = lc + 1)");
    CHECK_ARG(lc >= 1 && lf <= P->F && level_other >= 1 && level_other <= P->F, "levels");
    CHECK_ARG(S >= 1 && S <= MAXS && in && out && in != out, "args");
    Factor& f = factor == SG_FACTOR_X ? P->fx : P->fv;
    Factor& o = factor == SG_FACTOR_X ? P->fv : P->fx;
    const int64_t no = o.lev[level_other].n;
    const int dir = factor == SG_FACTOR_X ? 0 : 1;
    const Level& F_ = f.lev[lf];
    const int64_t nin = prolong ? f.lev[lc].n : F_.n, nout = prolong ? F_.n : f.lev[lc].n;
    EntryList el;
    el.ne = 0;
    for (int s = 0; s < S; ++s) el.e[el.ne++] = {in, prolong ? F_.pvals : F_.rvals, 1.0, s, s};
    const int W = prolong ? 2 : f.W;
    const int32_t* cols = prolong ? F_.pcols : F_.rcols;
    if (dir == 0) return launch_gather(P, 0, W, S, nin, no, nout, cols, el, out, beta);
    return launch_gather(P, 1, W, S, no, nin, nout, cols, el, out, beta);
}

extern "C" int sg_prolongate(sg_problem* P, int factor, int lf, int lc, int level_other, int S, const double* in,
                             double* out, double beta) {
    return transfer(P, factor, lf, lc, level_other, S, in, out, beta, true);
}
extern "C" int sg_restrict(sg_problem* P, int factor, int lc, int lf, int level_other, int S, const double* in,
                           double* out, double beta) {
    return transfer(P, factor, lf, lc, level_other, S, in, out, beta, false);
}

extern "C" int sg_combine(sg_problem* P, const double* dhat_active, const double* dhat_coarse, double* du) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(dhat_active && du && (dhat_coarse || P->coarse.empty()), "args");
    return combine(P, P->S, dhat_active, dhat_coarse, du);
}

extern "C" int sg_interp_u0(sg_problem* P, double* u) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(u, "u");
    return interp_u0(P, u);
}

extern "C" int sg_rhs(sg_problem* P, int j, const double* trace_prev, double* b) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(j >= 1 && trace_prev && b, "args");
    return rhs(P, j, trace_prev, b);
}

extern "C" int sg_solve_strip(sg_problem* P, const double* b, double* u, double rtol, double inner_rtol, int max_iter,
                              int* iters, double* last_norm) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(b && u && b != u && rtol > 0 && inner_rtol > 0 && max_iter > 0, "args");
    return solve_strip(P, b, u, rtol, inner_rtol, max_iter, iters, last_norm);
}

extern "C" int sg_step(sg_problem* P, int j0, int nsteps, double* trace, double rtol, double inner_rtol) {
    NEED_ASSEMBLED(P);
    CHECK_ARG(trace && j0 >= 1 && nsteps >= 0 && rtol > 0 && inner_rtol > 0, "args");
    cudaPointerAttributes at;
    bool host = true;
    if (cudaPointerGetAttributes(&at, trace) == cudaSuccess && at.type == cudaMemoryTypeDevice) host = false;
    cudaGetLastError();
    const int64_t n = set_size(P, SG_SET_ACTIVE, 1);
    double* tr = host ? P->trace_dev : trace;
    if (host) SG_CUDA(cudaMemcpyAsync(tr, trace, sizeof(double) * n, cudaMemcpyHostToDevice, P->stream));
    SG_TRY(step(P, j0, nsteps, tr, rtol, inner_rtol));
    if (host) SG_CUDA(cudaMemcpyAsync(trace, tr, sizeof(double) * n, cudaMemcpyDeviceToHost, P->stream));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    return SG_OK;
}

// ---------------------------------------------------------- instrumentation
// host counters (applies issued directly through the ABI) + device counters (strip solver)
extern "C" int sg_stats(sg_problem* P, int64_t* n_applies, int64_t* dof_applied, int64_t* launches,
                        int64_t* outer_iters, int64_t* inner_iters) {
    CHECK_ARG(P, "null handle");
    SG_TRY(sync_stats(P));
    const SolveCtl* c = P->hctl;
    if (n_applies) *n_applies = P->n_applies + (c ? c->n_applies : 0);
    if (dof_applied) *dof_applied = P->dof_applied + (c ? (int64_t)c->dof_applied : 0);
    if (launches) *launches = P->launches;
    if (outer_iters) *outer_iters = c ? c->outer_iters : 0;
    if (inner_iters) *inner_iters = c ? c->inner_iters : 0;
    return SG_OK;
}
extern "C" int sg_solver_health(sg_problem* P, int64_t* outer_unconverged, int64_t* outer_nonfinite,
                                int64_t* inner_maxit, int64_t* inner_breakdowns) {
    CHECK_ARG(P, "null handle");
    SG_TRY(sync_stats(P));
    const SolveCtl* c = P->hctl;
    if (outer_unconverged) *outer_unconverged = c ? c->outer_unconverged : 0;
    if (outer_nonfinite) *outer_nonfinite = c ? c->outer_nonfinite : 0;
    if (inner_maxit) *inner_maxit = c ? c->inner_maxit : 0;
    if (inner_breakdowns) *inner_breakdowns = c ? c->inner_breakdowns : 0;
    return SG_OK;
}
extern "C" int sg_reset_stats(sg_problem* P) {
    CHECK_ARG(P, "null handle");
    P->n_applies = P->dof_applied = P->launches = 0;
    return reset_device_stats(P);
}
extern "C" int sg_set_timing(sg_problem* P, int on) {
    CHECK_ARG(P, "null handle");
    P->timing = on != 0;
    return SG_OK;
}
extern "C" int sg_kernel_time(sg_problem* P, double* ms, int64_t* launches, double* alg_bytes, double* alg_flops) {
    CHECK_ARG(P, "null handle");
    SG_TRY(sync_stats(P));
    const SolveCtl* c = P->hctl;
    if (ms) *ms = c ? c->apply_ns * 1e-6 : 0.0;
    if (launches) *launches = c ? c->timed_applies : 0;
    if (alg_bytes) *alg_bytes = c ? c->alg_bytes : 0.0;
    if (alg_flops) *alg_flops = c ? c->alg_flops : 0.0;
    return SG_OK;
}

extern "C" int sg_solve_history(sg_problem* P, int max_n, double* nd, double* omega, int* n) {
    CHECK_ARG(P && n && max_n >= 0, "null argument");
    SG_TRY(sync_stats(P));
    const SolveCtl* c = P->hctl;
    const int it = c ? std::min(c->it, 256) : 0;
    *n = it;
    for (int i = 0; i < std::min(it, max_n); ++i) {
        if (nd) nd[i] = c->hist_nd[i];
        if (omega) omega[i] = c->hist_om[i];
    }
    return SG_OK;
}

extern "C" int sg_outer_switches(sg_problem* P, int64_t* switches) {
    CHECK_ARG(P && switches, "null argument");
    SG_TRY(sync_stats(P));
    *switches = P->hctl ? P->hctl->mr_switches : 0;
    return SG_OK;
}
