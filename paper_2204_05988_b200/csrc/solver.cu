// Strip operator applies, cross-grid blocks, combination preconditioner,
// Richardson strip solver and time stepping.  PAPER.md sec. 4.2-4.3, eq. (4).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mesh_dev.cuh"
#include "sg_internal.cuh"

namespace sg {

int64_t set_size(const sg_problem* P, int set, int S) {
    const auto& gs = set == SG_SET_ACTIVE ? P->active : P->coarse;
    int64_t n = 0;
    for (const auto& g : gs) n += g.n1 * g.n2;
    return n * S;
}

static inline int64_t gsize(const Grid& g) { return g.n1 * g.n2; }
constexpr int VMT_NR = 16;   // rows of a moment class table (10 monomials + 6 chi groups)

// generic pass 2 on box x-lattices (band kernel over the stencil-format matrices)
static int xgather(sg_problem* P, const Grid& g, const XgatParams& ep, double* Y, double beta) {
    const Level& Lx = P->fx.lev[g.l1];
    return launch_xgat_st(P, P->fx.d, P->S, g.n1, g.n2, Lx.so, Lx.bflag, ep, Y, beta, Lx.m);
}

// Algorithmic FLOPs of one strip-operator apply on grid g (2 per multiply-add), counted on the
// structural nonzeros of the factor matrices (count_nnz): pass 1 applies B_b to every used x-row
// (interior groups: all S*n1 rows, boundary-only face groups: the S*nbnd x-boundary rows),
// pass 2 applies every combined x matrix C_b^{ss'} to all n2 columns.
static double diag_flops(const sg_problem* P, const Grid& g) {
    const int S = P->S;
    const int64_t nb1 = P->fx.lev[g.l1].nbnd;
    double f = 0.0;
    for (int o = 0; o < (int)P->vorder.size(); ++o) {
        const Group& gr = P->vgroups[P->vorder[o]];
        const double rows = gr.bonly ? (double)nb1 : (double)g.n1;
        f += 2.0 * S * rows * (double)P->nnz_v[g.l2][gr.spec];
        for (const auto& ce : gr.comb[g.l1]) f += 2.0 * (double)ce.nnz * (double)g.n2;
    }
    return f;
}

double apply_flops(const sg_problem* P, const Grid& g) { return diag_flops(P, g); }

static bool l_has_xfi(const sg_problem* P, int l1) {
    return P->use_tma && l1 < (int)P->xfi_tab.size() && P->xfi_tab[l1] != nullptr &&
           ((P->fx.d == 3 && P->ng_int == 10) || (P->fx.d == 2 && P->ng_int == 6)) && P->fx.lev[l1].m >= 3;
}

// pass 1 of the per-grid operator on grid (l1, l2): Z_o = (Id x Id x B_o) X for every v-group o
// (vorder; boundary-only groups on x-boundary rows only), written with row pitch `pitch`
int pass1_vgroups(sg_problem* P, int l1, int l2, const double* X, double* const* outs, int64_t pitch, double* fbytes,
                  int64_t c0, int64_t c1, bool fine_mask) {
    // columns [c0, c1) of the grid (default: all), written at output columns 0 .. c1 - c0;
    // fine_mask (diagonal apply): boundary-only groups only on the x-rows of their own faces
    const int S = P->S;
    double fb_dummy = 0.0;
    if (!fbytes) fbytes = &fb_dummy;
    const Level& Lx = P->fx.lev[l1];
    const Level& Lv = P->fv.lev[l2];
    const int64_t n1 = Lx.n, n2 = Lv.n;
    const int nb = (int)P->vorder.size();
    const bool vbox = P->fv.kind == SG_MESH_BOX && nb <= MAXG;
    if (c1 <= 0) c1 = n2;
    const bool whole = c0 == 0 && c1 == n2;
    const int mm = fine_mask && Lx.bmask && nb - P->ng_int <= 8 ? 1 : 0;
    const uint8_t* xfl = mm ? Lx.bmask : Lx.bflag;
    const double cfrac = (double)(c1 - c0) / (double)n2;
    if (vbox) {
        VfanParams vp;
        vp.ng = nb;
        vp.ng_int = P->ng_int;
        for (int o = 0; o < nb; ++o) {
            vp.vst[o] = Lv.fst[P->vgroups[P->vorder[o]].spec];
            vp.out[o] = outs[o];
        }
        int rc = SG_ERR_UNSUPPORTED;
        const bool vmom_here = P->fv.d == 2 || n1 < 64;
        if (vmom_here) {
            // interior groups by shifted moments, boundary-only (face) groups by the stencil kernel
            rc = launch_vmom(P, l2, (int64_t)S * n1, n2, pitch, X, vp.out, Lx.bflag, n1, c0, c1);
            if (rc == SG_OK && c0 == 0) *fbytes += 8.0 * (double)P->vm_tab_n;   // class tables
            if (rc == SG_OK && nb > P->ng_int && P->vm_nchi == 0) {
                VfanParams vb;
                vb.ng = nb - P->ng_int;
                vb.ng_int = 0;
                for (int o = 0; o < vb.ng; ++o) {
                    vb.vst[o] = vp.vst[P->ng_int + o];
                    vb.out[o] = vp.out[P->ng_int + o];
                }
                rc = launch_vfan_st(P, P->fv.d, S, n1, n2, Lv.so, xfl, vb, X, pitch, c0, c1, mm);
                *fbytes += 8.0 * vb.ng * P->fv.W * (double)n2 * cfrac;   // per-column stencil coefficients
            }
        }
        if (rc == SG_ERR_UNSUPPORTED) {
            rc = launch_vfan_st(P, P->fv.d, S, n1, n2, Lv.so, xfl, vp, X, pitch, c0, c1, mm);
            *fbytes += 8.0 * nb * P->fv.W * (double)n2 * cfrac;
        }
        return rc;
    }
    if (pitch != n2 || !whole) return SG_ERR_UNSUPPORTED;
    for (int b0 = 0; b0 < nb; b0 += MAX_FANOUT) {
        FanoutList fl;
        fl.no = std::min(MAX_FANOUT, nb - b0);
        for (int o = 0; o < fl.no; ++o) {
            fl.vals[o] = Lv.fm[P->vgroups[P->vorder[b0 + o]].spec];
            fl.out[o] = outs[b0 + o];
        }
        SG_TRY(launch_fanout(P, 1, P->fv.W, S, n1, n2, n2, Lv.cols, X, fl));
        *fbytes += (8.0 * fl.no + 4.0) * P->fv.W * (double)n2;   // ELL values + pattern
    }
    return SG_OK;
}

// pass 2 on grid (l1, l2) over all v-groups (vorder) from intermediates with group stride gstr:
// Y = sum_o C_o Z_o with the line-swept kernels; SG_ERR_UNSUPPORTED if they do not cover it
static int pass2_fast(sg_problem* P, int l1, int l2, const double* Z, int64_t pitch, int64_t gstr, double* Y) {
    const int64_t n1 = P->fx.lev[l1].n, n2 = P->fv.lev[l2].n;
    if (P->fx.kind != SG_MESH_BOX || P->fv.kind != SG_MESH_BOX || P->S != 1) return SG_ERR_UNSUPPORTED;
    int rc = launch_xwhole(P, l1, n1, n2, pitch, Z, gstr, Y);
    if (rc == SG_ERR_UNSUPPORTED && (pitch & 1) == 0 && l_has_xfi(P, l1))
        rc = launch_xfanin_tma(P, l1, n1, n2, pitch, Z, gstr, Y);
    if (rc == SG_ERR_UNSUPPORTED && pitch == n2) rc = launch_xfanin(P, l1, n1, n2, Z, gstr, Y, 0.0);
    return rc;
}

// ------------------------------------------------ diagonal block (one grid)
// Y = sum_t T_t (x) A_t (x) B_t X, grouped by the v-spec b:
//   Z_b = (Id x Id x B_b) X           (pass 1, along v)
//   Y   = sum_b sum_{s,s'} (e_s e_s'^T (x) C_b^{ss'} (x) Id) Z_b,  C_b^{ss'} = sum_{t in b} T_t[s,s'] A_t
// (application order of l.516-532 with S^(2) first, the intermediates stay on
// the grid's own level because l = l').  *fbytes: factor data the launched kernels read.
static int apply_diag_impl(sg_problem* P, const Grid& g, const double* X, double* Y, double* fbytes) {
    const int S = P->S;
    const int64_t n = gsize(g);
    const Level& Lx = P->fx.lev[g.l1];
    const int nb = (int)P->vorder.size();
    const bool vbox = P->fv.kind == SG_MESH_BOX && nb <= MAXG;
    const bool xbox = P->fx.kind == SG_MESH_BOX;
    // ---- d = 1: fused two-sided kernel (one node per thread, 3 x 3 neighbourhood), no intermediates
    if (P->d1_ok) {
        const Grid* gp = &g;
        const double* sk = P->skip;
        return launch_d1fused(P, 1, &gp, &X, &Y, &sk, fbytes);
    }
    // ---- fused single pass (tiny x-lattices): no intermediates
    {
        const int rc = launch_fwhole(P, g.l1, g.l2, g.n2, X, Y);
        if (rc == SG_OK) {
            int ncls = 1;
            for (int q = 0; q < P->fv.d; ++q) ncls *= 3;
            *fbytes += 8.0 * (ncls * (VMT_NR * P->fv.W) + 16.0 * 223);   // moment class table + x table
            return SG_OK;
        }
        if (rc != SG_ERR_UNSUPPORTED) return rc;
    }
    // ---- pass 1: Z_b = (Id x Id x B_b) X for every v-group b (interior groups first)
    // (TMA pass 2 reads the intermediates with an even row pitch)
    const bool tma2 = vbox && xbox && S == 1 && l_has_xfi(P, g.l1);
    // ---- L2-resident column chunks (north_star subsystem (1): the intermediates
    // of the two-sided apply are not stored): pass 1 and pass 2 alternate on chunks of v-columns
    // whose intermediates Z_b (all x-rows x chunk columns x groups) fit in the L2 cache; the same
    // workspace lines are overwritten chunk after chunk and never leave the L2.
    if (tma2 && P->l2_chunk_bytes > 0 && P->fx.lev[g.l1].m >= 5) {
        const int64_t nb1 = Lx.nbnd;
        const double colbytes = 8.0 * ((double)P->ng_int * g.n1 + (double)(nb - P->ng_int) * nb1);
        int64_t wc = (int64_t)((double)P->l2_chunk_bytes / colbytes);
        if (wc < g.n2 && wc >= P->l2_chunk_mincols) {
            int64_t nch = (g.n2 + wc - 1) / wc;
            wc = (g.n2 + nch - 1) / nch;
            wc = (wc + 31) / 32 * 32;   // chunk starts on 256-byte column boundaries of X
            nch = (g.n2 + wc - 1) / wc;
            const int64_t pc = wc;      // even row pitch (TMA strides)
            const int64_t gstr_c = g.n1 * pc;
            if ((size_t)nb * gstr_c > P->wsZ_n) {
                set_error("apply_diag: workspace too small");
                return SG_ERR_STATE;
            }
            std::vector<double*> outs(nb);
            for (int o = 0; o < nb; ++o) outs[o] = P->wsZ + (int64_t)o * gstr_c;
            for (int64_t ch = 0; ch < nch; ++ch) {
                const int64_t c0 = ch * wc, c1 = std::min(g.n2, c0 + wc);
                SG_TRY(pass1_vgroups(P, g.l1, g.l2, X, outs.data(), pc, fbytes, c0, c1, true));
                int rc2 = launch_xfanin_tma(P, g.l1, g.n1, c1 - c0, pc, P->wsZ, gstr_c, Y + c0, g.n2, ch == 0);
                if (rc2 != SG_OK) {
                    if (rc2 == SG_ERR_UNSUPPORTED) set_error("apply_diag: TMA pass 2 rejected a column chunk");
                    return rc2 == SG_ERR_UNSUPPORTED ? SG_ERR_STATE : rc2;
                }
            }
            int ncls = 1;
            for (int q = 0; q < P->fx.d; ++q) ncls *= 3;
            *fbytes += 8.0 * ncls * nb * P->fx.W;
            return SG_OK;
        }
    }
    const int64_t pitch = tma2 ? g.n2 + (g.n2 & 1) : g.n2;
    const int64_t gstr = (int64_t)S * g.n1 * pitch;
    if ((size_t)nb * gstr > P->wsZ_n) {
        set_error("apply_diag: workspace too small");
        return SG_ERR_STATE;
    }
    {
        std::vector<double*> outs(nb);
        for (int o = 0; o < nb; ++o) outs[o] = P->wsZ + (int64_t)o * gstr;
        SG_TRY(pass1_vgroups(P, g.l1, g.l2, X, outs.data(), pitch, fbytes, 0, 0, true));
    }
    // ---- pass 2: Y = sum_b sum_{s,s'} (e_s e_s'^T (x) C_b^{ss'} (x) Id) Z_b
    double beta = 0.0;
    int rcx = SG_ERR_UNSUPPORTED;
    if (vbox && xbox && S == 1) {
        rcx = launch_xwhole(P, g.l1, g.n1, g.n2, pitch, P->wsZ, gstr, Y);
        if (rcx != SG_OK && rcx != SG_ERR_UNSUPPORTED) return rcx;
    }
    if (tma2 && rcx != SG_OK) {
        rcx = launch_xfanin_tma(P, g.l1, g.n1, g.n2, pitch, P->wsZ, gstr, Y);
        if (rcx != SG_OK && rcx != SG_ERR_UNSUPPORTED) return rcx;
        if (rcx == SG_ERR_UNSUPPORTED && pitch != g.n2) {
            set_error("apply_diag: TMA pass 2 rejected a padded layout");
            return SG_ERR_STATE;
        }
    }
    if (rcx != SG_OK && xbox) {
        rcx = launch_xfanin(P, g.l1, g.n1, g.n2, P->wsZ, (int64_t)S * n, Y, 0.0);
        if (rcx != SG_OK && rcx != SG_ERR_UNSUPPORTED) return rcx;
    }
    if (rcx == SG_OK) {
        int ncls = 1;
        for (int q = 0; q < P->fx.d; ++q) ncls *= 3;
        *fbytes += 8.0 * ncls * nb * P->fx.W;   // class tables of the line-swept kernels
    } else if (xbox) {
        XgatParams ep;
        ep.ne = 0;
        for (int o = 0; o < nb; ++o) {
            const Group& gr = P->vgroups[P->vorder[o]];
            for (const auto& ce : gr.comb[g.l1]) {
                if (ep.ne == MAX_ENTRIES) {
                    SG_TRY(xgather(P, g, ep, Y, beta));
                    beta = 1.0;
                    ep.ne = 0;
                }
                ep.e[ep.ne++] = {P->wsZ + (int64_t)o * S * n, ce.st, ce.s_out, ce.s_in, gr.bonly ? 1 : 0, 1.0, ce.ctab};
                *fbytes += ce.ctab ? 8.0 * 27 * P->fx.W : 8.0 * P->fx.W * (double)g.n1;
            }
        }
        SG_TRY(xgather(P, g, ep, Y, beta));
    } else {
        EntryList el;
        el.ne = 0;
        *fbytes += 4.0 * P->fx.W * (double)g.n1;   // ELL pattern
        for (int o = 0; o < nb; ++o) {
            for (const auto& ce : P->vgroups[P->vorder[o]].comb[g.l1]) {
                if (el.ne == MAX_ENTRIES) {
                    SG_TRY(launch_gather(P, 0, P->fx.W, S, g.n1, g.n2, g.n1, Lx.cols, el, Y, beta));
                    beta = 1.0;
                    el.ne = 0;
                }
                el.e[el.ne++] = {P->wsZ + (int64_t)o * S * n, ce.vals, 1.0, ce.s_out, ce.s_in};
                *fbytes += 8.0 * P->fx.W * (double)g.n1;
            }
        }
        SG_TRY(launch_gather(P, 0, P->fx.W, S, g.n1, g.n2, g.n1, Lx.cols, el, Y, beta));
    }
    return SG_OK;
}

// One strip-operator apply.  skip: the grid's convergence flag inside the batched block solver
// (every kernel of the apply exits when it is non-zero).  Timing mode brackets the apply with
// device timestamps (k_tstamp) that also accumulate its algorithmic bytes (read X + write Y +
// the factor data its kernels read) and FLOPs (structural nonzeros).
int apply_diag(sg_problem* P, const Grid& g, const double* X, double* Y, const double* skip) {
    const int S = P->S;
    const int64_t n = gsize(g);
    if (P->timing) {
        k_tstamp<<<1, 1, 0, P->stream>>>(P->ctl, skip, P->stamp_slot, 0, 0.0, 0.0);
        P->launches++;
    }
    P->skip = skip;
    double fbytes = 0.0;
    const int rc = apply_diag_impl(P, g, X, Y, &fbytes);
    P->skip = nullptr;
    if (rc != SG_OK) return rc;
    if (P->timing) {
        k_tstamp<<<1, 1, 0, P->stream>>>(P->ctl, skip, P->stamp_slot, 1, 16.0 * S * (double)n + fbytes,
                                           diag_flops(P, g));
        P->launches++;
        SG_CUDA(cudaGetLastError());
    }
    if (!P->in_solve) {   // inside the strip solver the device counts the applies
        P->n_applies++;
        P->dof_applied += S * n;
    }
    return SG_OK;
}

// Structural nonzeros (|a_ij| > 1e-12 max |a|) of every factor matrix and combined x matrix,
// for the FLOP count of diag_flops (setup time).
__global__ void k_absmax(int64_t n, const double* __restrict__ v, unsigned long long* out) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v[i]));
        m = b > m ? b : m;
    }
    atomicMax(out, m);
}
__global__ void k_count_nz(int64_t n, const double* __restrict__ v, const unsigned long long* mx,
                           unsigned long long* out) {
    const double th = 1e-12 * __longlong_as_double((long long)*mx);
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += fabs(v[i]) > th;
    atomicAdd(out, c);
}
static int nnz_of(sg_problem* P, const double* vals, int64_t n, unsigned long long* dbuf, int64_t* out) {
    if (!vals) {
        *out = 0;
        return SG_OK;
    }
    SG_CUDA(cudaMemsetAsync(dbuf, 0, 2 * sizeof(unsigned long long), P->stream));
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_absmax<<<std::max(blocks, 1), 256, 0, P->stream>>>(n, vals, dbuf);
    k_count_nz<<<std::max(blocks, 1), 256, 0, P->stream>>>(n, vals, dbuf, dbuf + 1);
    P->launches += 2;
    unsigned long long h[2];
    SG_CUDA(cudaMemcpyAsync(h, dbuf, sizeof(h), cudaMemcpyDeviceToHost, P->stream));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    *out = (int64_t)h[1];
    return SG_OK;
}
int count_nnz(sg_problem* P) {
    unsigned long long* dbuf;
    SG_CUDA(cudaMalloc(&dbuf, 2 * sizeof(unsigned long long)));
    int rc = SG_OK;
    for (int which = 0; which < 2 && rc == SG_OK; ++which) {
        Factor& f = which == 0 ? P->fx : P->fv;
        auto& tab = which == 0 ? P->nnz_x : P->nnz_v;
        tab.assign(P->F + 1, std::vector<int64_t>(f.specs.size(), 0));
        for (int l = 1; l <= P->F && rc == SG_OK; ++l)
            for (size_t sp = 0; sp < f.specs.size() && rc == SG_OK; ++sp)
                if (sp < f.lev[l].fm.size())
                    rc = nnz_of(P, f.lev[l].fm[sp], f.lev[l].n * f.W, dbuf, &tab[l][sp]);
    }
    for (auto& gr : P->vgroups)
        for (int l = 1; l <= P->F && rc == SG_OK; ++l)
            for (auto& ce : gr.comb[l]) {
                rc = nnz_of(P, ce.vals, P->fx.lev[l].n * P->fx.W, dbuf, &ce.nnz);
                if (rc != SG_OK) break;
            }
    cudaFree(dbuf);
    return rc;
}

// stencil offsets / boundary flags / stencil-format matrices for box lattices
__global__ void k_bflag(int64_t n, int d, int m, const int32_t* lat, uint8_t* f) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t b = 0;
    for (int k = 0; k < d; ++k) {
        int z = lat[k * n + i];
        b |= (z == 0 || z == m - 1);
    }
    f[i] = b;
}

int prepare_stencils(sg_problem* P) {
    for (Factor* f : {&P->fx, &P->fv}) {
        for (int l = 1; l <= P->F; ++l) {
            Level& L = f->lev[l];
            SG_CUDA(cudaMalloc(&L.bflag, L.n));
            if (f->kind == SG_MESH_BOX) {
                k_bflag<<<(int)((L.n + 255) / 256), 256, 0, P->stream>>>(L.n, f->d, L.m, L.lat, L.bflag);
                P->launches++;
                {
                    int64_t inner = 1;
                    for (int q = 0; q < f->d; ++q) inner *= (L.m - 2);
                    L.nbnd = L.n - inner;
                }
                std::vector<int64_t> offs;
                for (int S_ = 0; S_ < (1 << f->d); ++S_) {
                    int64_t o = 0, st = 1;
                    for (int i = 0; i < f->d; ++i) {
                        if ((S_ >> i) & 1) o += st;
                        st *= L.m;
                    }
                    offs.push_back(o);
                    if (o) offs.push_back(-o);
                }
                std::sort(offs.begin(), offs.end());
                for (int k = 0; k < 15; ++k) L.so.off[k] = k < (int)offs.size() ? offs[k] : 0;
            } else {
                SG_CUDA(cudaMemsetAsync(L.bflag, 1, L.n, P->stream));   // no skipping off box lattices
                L.nbnd = L.n;
            }
        }
    }
    // group ordering: interior groups first, boundary-only (face) groups last
    P->vorder.clear();
    for (int pass = 0; pass < 2; ++pass)
        for (size_t gi = 0; gi < P->vgroups.size(); ++gi) {
            Group& g = P->vgroups[gi];
            bool bonly = true;
            for (int t : g.terms) bonly &= P->fx.specs[P->terms[t].xs].kind == 1;
            g.bonly = bonly;
            if ((pass == 0) != bonly) P->vorder.push_back((int)gi);
        }
    P->ng_int = 0;
    for (int gi : P->vorder) P->ng_int += P->vgroups[gi].bonly ? 0 : 1;
    // x-groups: "boundary-only" means the x matrix is a face mass (nonzero on boundary x-rows only)
    P->xorder.clear();
    for (int pass = 0; pass < 2; ++pass)
        for (size_t gi = 0; gi < P->xgroups.size(); ++gi) {
            Group& g = P->xgroups[gi];
            const bool bonly = P->fx.specs[g.spec].kind == 1;
            g.bonly = bonly;
            if ((pass == 0) != bonly) P->xorder.push_back((int)gi);
        }
    P->nxg_int = 0;
    for (int gi : P->xorder) P->nxg_int += P->xgroups[gi].bonly ? 0 : 1;
    // stencil-format copies
    auto ensure_fst = [&](Factor& f, int spec, int l) -> int {
        Level& L = f.lev[l];
        if ((int)L.fst.size() < (int)f.specs.size()) L.fst.resize(f.specs.size(), nullptr);
        if (!L.fst[spec]) {
            SG_CUDA(cudaMalloc(&L.fst[spec], sizeof(double) * f.W * L.n));
            SG_TRY(launch_ell_to_stencil(P, L.n, f.W, L.cols, L.fm[spec], L.so, L.fst[spec]));
        }
        return SG_OK;
    };
    for (int l = 1; l <= P->F; ++l) {
        if (P->fx.kind == SG_MESH_BOX) {
            SG_TRY(ensure_fst(P->fx, P->mass_x, l));
            for (auto& g : P->xgroups) SG_TRY(ensure_fst(P->fx, g.spec, l));
            Level& L = P->fx.lev[l];
            L.fcls.assign(P->fx.specs.size(), nullptr);
            for (size_t sp = 0; sp < P->fx.specs.size(); ++sp)
                    if (L.fst.size() > sp && L.fst[sp]) SG_TRY(class_compress(P, P->fx, l, L.fst[sp], &L.fcls[sp]));
        }
        if (P->fv.kind == SG_MESH_BOX) {
            SG_TRY(ensure_fst(P->fv, P->mass_v, l));
            for (auto& g : P->xgroups)
                for (auto& ce : g.comb[l]) {
                    SG_CUDA(cudaMalloc(&ce.st, sizeof(double) * P->fv.W * P->fv.lev[l].n));
                    SG_TRY(launch_ell_to_stencil(P, P->fv.lev[l].n, P->fv.W, P->fv.lev[l].cols, ce.vals, P->fv.lev[l].so,
                                                 ce.st));
                }
        }
    }
    for (auto& g : P->vgroups) {
        for (int l = 1; l <= P->F; ++l) {
            if (P->fv.kind == SG_MESH_BOX) {
                Level& L = P->fv.lev[l];
                if ((int)L.fst.size() < (int)P->fv.specs.size()) L.fst.resize(P->fv.specs.size(), nullptr);
                if (!L.fst[g.spec]) {
                    SG_CUDA(cudaMalloc(&L.fst[g.spec], sizeof(double) * P->fv.W * L.n));
                    SG_TRY(launch_ell_to_stencil(P, L.n, P->fv.W, L.cols, L.fm[g.spec], L.so, L.fst[g.spec]));
                }
            }
            if (P->fx.kind == SG_MESH_BOX) {
                Level& L = P->fx.lev[l];
                for (auto& ce : g.comb[l]) {
                    SG_CUDA(cudaMalloc(&ce.st, sizeof(double) * P->fx.W * L.n));
                    SG_TRY(launch_ell_to_stencil(P, L.n, P->fx.W, L.cols, ce.vals, L.so, ce.st));
                    SG_TRY(class_compress(P, P->fx, l, ce.st, &ce.ctab));
                }
            }
        }
    }
    SG_TRY(prepare_xfanin(P));
    SG_TRY(prepare_vmom(P));
    SG_TRY(prepare_fwhole(P));
    SG_TRY(prepare_d1fused(P));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    return SG_OK;
}

// --------------------------------------------------- cross-grid full apply
// Y_p = sum_{p'} A_{p,p'} X_{p'} over the active set (l.512-516) with the
// cross-level factors A_{l,l'} = A_l E_{l<-l'} (l >= l') and E^T A_{l'} (l < l'),
// which equal E_F^T A_F E_F (l.506-509) because the factor forms are
// integrated exactly on every level.
//  lower part (l1 >= l1'): per v-group b: Z = B_b X_{p'}, restrict in v down to
//    the target's v-level, Horner-prolong in x up to the target's x-level, then
//    gather with the group's combined x matrices;
//  upper part (l1 < l1'): per x-group a symmetric with the roles of x, v swapped.
// "mass" mode (Tb != nullptr): single term Tb (x) M^x (x) M^v, S_out x S_in.
static int apply_cross_impl(sg_problem* P, const double* Tb, int S_out, int S_in, const double* X, double* Y);
static int cross_lower_batched(sg_problem* P, const double* X, double* Y);

// The cross-grid apply is a fixed sequence of ~10^3 small launches (transfer
// chains per group); it is captured once per (X, Y, Tb) into a CUDA graph on the
// library's own stream and replayed, which removes the per-launch CPU cost
// (dominant on the 2D configurations).
int apply_cross_prepare(sg_problem* P) {
    if (P->cross_batched_tried) return SG_OK;
    int rc = cross_lower_batched(P, nullptr, nullptr);   // allocation only (never inside a capture)
    if (rc != SG_OK && rc != SG_ERR_UNSUPPORTED) return rc;
    P->cross_batched_tried = true;
    // concurrent per-group branches of the per-group (unbatched) path: the configurations whose
    // cross-grid apply is a long chain of tiny launches (d = 1), when the private workspaces fit
    const int nbr = (int)(P->vgroups.size() + P->xgroups.size());
    const int64_t Na = set_size(P, SG_SET_ACTIVE, P->S);
    const size_t per = P->wsZ_n + 3 * (size_t)Na;
    if (P->fx.d == 1 && P->fv.d == 1 && getenv("SG_SERIAL_CROSS") == nullptr && nbr <= MAX_SUM &&
        per * nbr * sizeof(double) <= ((size_t)1 << 30)) {
        SG_CUDA(cudaEventCreateWithFlags(&P->ev_cx_fork, cudaEventDisableTiming));
        for (int i = 0; i < nbr; ++i) {
            cudaStream_t s;
            cudaEvent_t e;
            double *w, *h, *y;
            SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            SG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            SG_CUDA(cudaMalloc(&w, sizeof(double) * P->wsZ_n));
            SG_CUDA(cudaMalloc(&h, sizeof(double) * 2 * Na));
            SG_CUDA(cudaMalloc(&y, sizeof(double) * Na));
            SG_CUDA(cudaMemset(w, 0, sizeof(double) * P->wsZ_n));
            P->cx_streams.push_back(s);
            P->ev_cx_join.push_back(e);
            P->cx_ws.push_back(w);
            P->cx_h.push_back(h);
            P->cx_y.push_back(y);
        }
        P->cx_ws_n = P->wsZ_n;
        P->cx_h_n = 2 * Na;
        P->cx_y_n = Na;
        P->par_cross = true;
        SG_CUDA(cudaDeviceSynchronize());
    }
    return SG_OK;
}

int apply_cross(sg_problem* P, const std::vector<Term>* /*unused*/, const double* Tb, int S_out, int S_in,
                const double* X, double* Y) {
    SG_TRY(apply_cross_prepare(P));
    if (!P->use_graphs || P->capturing) return apply_cross_impl(P, Tb, S_out, S_in, X, Y);
    GraphKey key;
    key.X = X;
    key.Y = Y;
    key.S_out = S_out;
    key.S_in = S_in;
    key.mass = Tb != nullptr;
    for (int i = 0; i < 4; ++i) key.T[i] = (Tb && i < S_out * S_in) ? Tb[i] : 0.0;
    GraphEntry* ge = nullptr;
    for (auto& e : P->graphs)
        if (e.key.same(key)) ge = &e;
    cudaStream_t gs = P->gstream;
    if (!ge) {
        if (P->graphs.size() >= 24) {
            cudaGraphExecDestroy(P->graphs.front().exec);
            P->graphs.erase(P->graphs.begin());
        }
        const int64_t l0 = P->launches;
        cudaStream_t saved = P->stream;
        P->stream = gs;
        SG_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        int rc = apply_cross_impl(P, Tb, S_out, S_in, X, Y);
        cudaGraph_t graph;
        cudaError_t ce = cudaStreamEndCapture(gs, &graph);
        P->stream = saved;
        if (rc != SG_OK) return rc;
        SG_CUDA(ce);
        GraphEntry e;
        e.key = key;
        e.nlaunch = P->launches - l0;
        P->launches = l0;
        SG_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
        cudaGraphDestroy(graph);
        P->graphs.push_back(e);
        ge = &P->graphs.back();
    }
    // order: user stream -> graph stream -> user stream
    SG_CUDA(cudaEventRecord(P->ev_a, P->stream));
    SG_CUDA(cudaStreamWaitEvent(gs, P->ev_a, 0));
    SG_CUDA(cudaGraphLaunch(ge->exec, gs));
    SG_CUDA(cudaEventRecord(P->ev_b, gs));
    SG_CUDA(cudaStreamWaitEvent(P->stream, P->ev_b, 0));
    P->launches += ge->nlaunch;
    return SG_OK;
}


// Batched lower part of the cross-grid apply (see apply_cross_impl), S = 1 box lattices only.
// Memory: Q0 = stage-0 fan-outs of every group at every source (natural pitch), H = Horner
// results of every group at every target (even pitch, TMA-readable), both allocated once.
static int cross_lower_batched(sg_problem* P, const double* X, double* Y) {
    if (!P->use_cross_batched || P->S != 1 || P->fx.kind != SG_MESH_BOX || P->fv.kind != SG_MESH_BOX || P->fx.d < 2)
        return SG_ERR_UNSUPPORTED;
    const auto& A = P->active;
    const int ng = (int)A.size();
    const int L = P->cfg.L;
    const int nga = (int)P->vorder.size();
    const int Wv = P->fv.W;
    auto n1 = [&](int l) { return P->fx.lev[l].n; };
    auto n2 = [&](int l) { return P->fv.lev[l].n; };
    auto pit = [&](int l) { return n2(l) + (n2(l) & 1); };
    // every target must be covered by the fast gathers
    for (int p = 1; p <= ng; ++p) {
        const int m = P->fx.lev[p].m;
        const bool whole = ((P->fx.d == 3 && m == 3) || (P->fx.d == 2 && (m == 3 || m == 5))) &&
                           nga <= 16 && p < (int)P->xfi_tab.size() && P->xfi_tab[p];
        if (!whole && (p == 1 || !l_has_xfi(P, p))) return SG_ERR_UNSUPPORTED;
    }
    std::vector<int64_t> qo(ng + 2, 0), ho(ng + 2, 0);
    for (int p = 1; p <= ng; ++p) {
        qo[p + 1] = qo[p] + (int64_t)nga * n1(p) * n2(L - p);
        ho[p + 1] = ho[p] + (int64_t)nga * n1(p) * pit(L - p);
    }
    if (!P->cross_batched_tried) {
        // first use: allocate outside any stream capture (apply_cross calls us uncaptured first);
        // sized for the lower part (v-groups) and the batched upper part (x-groups)
        P->cross_batched_tried = true;
        const int nxg = (int)P->xgroups.size();
        int64_t qu = 0, hu = 0;
        for (int pp = 2; pp <= ng; ++pp) qu += (int64_t)nxg * n1(pp) * n2(L - pp);
        for (int p = 1; p <= ng - 1; ++p) hu += (int64_t)nxg * n1(p) * n2(L - p);
        P->cross_q_n = std::max<int64_t>(qo[ng + 1], qu);
        P->cross_h_n = std::max<int64_t>(ho[ng + 1], hu);
        qo[ng + 1] = P->cross_q_n;
        ho[ng + 1] = P->cross_h_n;
        if (cudaMalloc(&P->cross_q, sizeof(double) * qo[ng + 1]) != cudaSuccess ||
            cudaMalloc(&P->cross_h, sizeof(double) * ho[ng + 1]) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(P->cross_q);
            cudaFree(P->cross_h);
            P->cross_q = P->cross_h = nullptr;
            if (P->verbose) fprintf(stderr, "[sg] batched cross-grid apply: not enough memory, per-group path\n");
            return SG_ERR_UNSUPPORTED;
        }
        // finite contents for rows a boundary-only group never writes (they meet zero coefficients)
        SG_CUDA(cudaMemset(P->cross_q, 0, sizeof(double) * qo[ng + 1]));
        SG_CUDA(cudaMemset(P->cross_h, 0, sizeof(double) * ho[ng + 1]));
        SG_CUDA(cudaDeviceSynchronize());
        return SG_OK;   // allocation-only call
    }
    if (!P->cross_q || !P->cross_h) return SG_ERR_UNSUPPORTED;
    auto Q0 = [&](int pp, int o) { return P->cross_q + qo[pp] + (int64_t)o * n1(pp) * n2(L - pp); };
    auto H = [&](int p, int o) { return P->cross_h + ho[p] + (int64_t)o * n1(p) * pit(L - p); };
    // 1. stage-0 fan-out of all groups at every source: Q0[pp][o] = (Id x B_o) X_pp
    for (int pp = 1; pp <= ng; ++pp) {
        std::vector<double*> outs(nga);
        for (int o = 0; o < nga; ++o) outs[o] = Q0(pp, o);
        SG_TRY(pass1_vgroups(P, pp, L - pp, X + A[pp - 1].off1, outs.data(), n2(L - pp), nullptr, 0, 0, true));
    }
    // 2./3. per group: restriction chains in v and Horner prolongation in x; the last
    // Horner stage of target p (m = p) writes H[p][o] with the even pitch
    std::vector<std::vector<int64_t>> qoff(ng);
    for (int o = 0; o < nga; ++o) {
        // boundary-only (face) groups: their intermediates are needed on the x-rows of their own face
        // only (prolongation in x keeps a face inside itself), all other rows meet zero coefficients
        const bool face_rows = o >= P->ng_int && nga - P->ng_int <= 8 && P->fv.kind == SG_MESH_BOX;
        int64_t pos = 0;
        for (int pp = 1; pp <= ng; ++pp) {
            qoff[pp - 1].assign(ng - pp + 1, 0);
            for (int k = 1; k <= ng - pp; ++k) {
                qoff[pp - 1][k] = pos;
                pos += n1(pp) * n2(L - pp - k);
            }
        }
        if ((size_t)pos > P->wsZ_n) {
            set_error("apply_cross: chain workspace too small");
            return SG_ERR_STATE;
        }
        auto Q = [&](int pp, int k) -> double* { return k == 0 ? Q0(pp, o) : P->wsZ + qoff[pp - 1][k]; };
        for (int k = 1; k <= ng - 1; ++k) {
            std::vector<Job> jobs;
            for (int pp = 1; pp <= ng - k; ++pp) {
                const int lv0 = L - pp, lf = lv0 - k + 1, lc = lv0 - k;
                jobs.push_back({Q(pp, k - 1), nullptr, Q(pp, k), P->fv.lev[lf].rcols, P->fv.lev[lf].rvals, n1(pp), n2(lf),
                                n2(lc), 1.0, 1, 1, Wv, 0});
                if (P->fv.kind == SG_MESH_BOX) jobs.back().box_mf = P->fv.lev[lf].m;
                if (face_rows && P->fx.lev[pp].bmask) {   // face group: rows of its own face only
                    jobs.back().rmask = P->fx.lev[pp].bmask;
                    jobs.back().rbit = o - P->ng_int;
                }
            }
            SG_TRY(launch_jobs(P, jobs));
        }
        double* hb[2] = {P->wsH, P->wsH + set_size(P, SG_SET_ACTIVE, 1)};
        for (int m = 2; m <= ng; ++m) {
            std::vector<Job> jobs;
            for (int p = m; p <= ng; ++p) {
                const int lv = L - p;
                const double* in = m == 2 ? Q(1, p - 1) : hb[(m - 1) & 1] + A[p - 1].off1;
                Job J{in, Q(m, p - m), hb[m & 1] + A[p - 1].off1, P->fx.lev[m].pcols, P->fx.lev[m].pvals, n1(m - 1), n2(lv),
                      n1(m), 1.0, 1, 0, 2, 0};
                if (p == m) {
                    J.out = H(p, o);
                    J.opitch = pit(lv);
                }
                J.box_mf = P->fx.lev[m].m;   // (box factor: checked by cross_lower_batched)
                J.box_d = P->fx.d;
                if (face_rows && P->fx.lev[m].bmask) {
                    J.rmask = P->fx.lev[m].bmask;
                    J.rbit = o - P->ng_int;
                }
                jobs.push_back(J);
            }
            SG_TRY(launch_jobs(P, jobs));
        }
    }
    // 4. one gather over all groups per target: Y_p = sum_o C_o^{(p)} H[p][o]
    for (int p = 1; p <= ng; ++p) {
        const int lv = L - p;
        const double* base = p == 1 ? Q0(1, 0) : H(p, 0);
        const int64_t pitch = p == 1 ? n2(lv) : pit(lv);
        const int64_t gstr = p == 1 ? n1(1) * n2(lv) : n1(p) * pit(lv);
        int rc = pass2_fast(P, p, lv, base, pitch, gstr, Y + A[p - 1].off1);
        if (rc != SG_OK) {
            if (rc == SG_ERR_UNSUPPORTED) set_error("apply_cross: batched gather unsupported after setup");
            return rc == SG_ERR_UNSUPPORTED ? SG_ERR_STATE : rc;
        }
    }
    return SG_OK;
}


// Batched upper part of the cross-grid apply (targets p < sources p'), S = 1 box lattices:
// all x-groups fanned out once per source (k_xfan_st, every row), per group the restriction
// chains in x and the Horner prolongation in v (last stage -> Hu[p][a]), then ONE v-gather
// over all x-groups per target (k_vgat_st, one read-modify-write of Y instead of one per group).
static int cross_upper_batched(sg_problem* P, const double* X, double* Y) {
    if (!P->use_cross_batched || P->S != 1 || P->fx.kind != SG_MESH_BOX || P->fv.kind != SG_MESH_BOX || P->fx.d < 2 ||
        !P->cross_q || !P->cross_h)
        return SG_ERR_UNSUPPORTED;
    const auto& A = P->active;
    const int ng = (int)A.size();
    const int L = P->cfg.L;
    const int nxg = (int)P->xgroups.size();
    const int Wx = P->fx.W;
    if (ng < 2) return SG_OK;
    if (nxg > MAXG || nxg > MAX_ENTRIES) return SG_ERR_UNSUPPORTED;
    for (int a = 0; a < nxg; ++a)
        for (int l = 1; l <= P->F; ++l)
            if (P->xgroups[a].comb[l].size() != 1) return SG_ERR_UNSUPPORTED;
    auto n1 = [&](int l) { return P->fx.lev[l].n; };
    auto n2 = [&](int l) { return P->fv.lev[l].n; };
    std::vector<int64_t> qo(ng + 2, 0), ho(ng + 2, 0);
    for (int pp = 2; pp <= ng; ++pp) qo[pp + 1] = qo[pp] + (int64_t)nxg * n1(pp) * n2(L - pp);
    qo[ng + 1] = std::max(qo[ng + 1], qo[ng]);
    for (int p = 1; p <= ng - 1; ++p) ho[p + 1] = ho[p] + (int64_t)nxg * n1(p) * n2(L - p);
    if (qo[ng + 1] > P->cross_q_n || ho[ng] > P->cross_h_n) return SG_ERR_UNSUPPORTED;
    auto Q0 = [&](int pp, int a) { return P->cross_q + qo[pp] + (int64_t)a * n1(pp) * n2(L - pp); };
    auto H = [&](int p, int a) { return P->cross_h + ho[p] + (int64_t)a * n1(p) * n2(L - p); };
    // 1. x fan-out of every x-group at every source pp >= 2 (all rows: the chains mix rows)
    for (int pp = 2; pp <= ng; ++pp) {
        const Level& Lx = P->fx.lev[pp];
        XfanParams fp;
        fp.ng = fp.ng_int = nxg;
        for (int a = 0; a < nxg; ++a) {
            const int sp = P->xgroups[a].spec;
            fp.cst[a] = Lx.fst[sp];
            fp.ctab[a] = Lx.fcls.size() > (size_t)sp ? Lx.fcls[sp] : nullptr;
            fp.out[a] = Q0(pp, a);
        }
        SG_TRY(launch_xfan_st(P, P->fx.d, 1, n1(pp), n2(L - pp), Lx.so, Lx.m, Lx.bflag, fp, X + A[pp - 1].off1));
    }
    // 2./3. per group: restriction chains in x, Horner prolongation in v
    std::vector<std::vector<int64_t>> qoff(ng);
    for (int a = 0; a < nxg; ++a) {
        int64_t pos = 0;
        for (int pp = 2; pp <= ng; ++pp) {
            const int lv = L - pp;
            qoff[pp - 1].assign(pp, 0);
            for (int k = 1; k <= pp - 1; ++k) {   // k: x-level pp-k
                qoff[pp - 1][k] = pos;
                pos += n1(pp - k) * n2(lv);
            }
        }
        if ((size_t)pos > P->wsZ_n) {
            set_error("apply_cross: chain workspace too small (upper)");
            return SG_ERR_STATE;
        }
        auto Q = [&](int pp, int k) -> double* { return k == 0 ? Q0(pp, a) : P->wsZ + qoff[pp - 1][k]; };
        for (int k = 1; k <= ng - 1; ++k) {
            std::vector<Job> jobs;
            for (int pp = k + 1; pp <= ng; ++pp) {
                const int lv = L - pp, lf = pp - k + 1, lc = pp - k;
                jobs.push_back({Q(pp, k - 1), nullptr, Q(pp, k), P->fx.lev[lf].rcols, P->fx.lev[lf].rvals, n1(lf), n2(lv),
                                n1(lc), 1.0, 1, 0, Wx, 0});
                if (P->fx.kind == SG_MESH_BOX) jobs.back().box_mf = P->fx.lev[lf].m;
            }
            SG_TRY(launch_jobs(P, jobs));
        }
        double* hb[2] = {P->wsH, P->wsH + set_size(P, SG_SET_ACTIVE, 1)};
        for (int q = 1; q <= ng - 1; ++q) {
            std::vector<Job> jobs;
            const int lvn = L - ng + q;
            for (int p = 1; p <= ng - q; ++p) {
                const double* in = q == 1 ? Q(ng, ng - p) : hb[(q - 1) & 1] + A[p - 1].off1;
                const int pp = ng - q;
                const double* add = pp > p ? Q(pp, pp - p) : nullptr;
                double* out = (q == ng - p) ? H(p, a) : hb[q & 1] + A[p - 1].off1;
                jobs.push_back({in, add, out, P->fv.lev[lvn].pcols, P->fv.lev[lvn].pvals, n1(p), n2(lvn - 1), n2(lvn), 1.0,
                                1, 1, 2, 0});
                jobs.back().box_mf = P->fv.lev[lvn].m;   // (box factor: checked by cross_upper_batched)
                jobs.back().box_d = P->fv.d;
            }
            SG_TRY(launch_jobs(P, jobs));
        }
    }
    // 4. one v-gather over all x-groups per target
    for (int p = 1; p <= ng - 1; ++p) {
        const int lvt = L - p;
        XgatParams ep;
        ep.ne = 0;
        for (int a = 0; a < nxg; ++a) {
            const auto& ce = P->xgroups[a].comb[lvt][0];
            // face x-groups: their chain results are exact zeros on interior x-rows (skipped there)
            ep.e[ep.ne++] = {H(p, a), ce.st, ce.s_out, ce.s_in, P->xgroups[a].bonly ? 1 : 0, 1.0};
        }
        SG_TRY(launch_vgat_st(P, P->fv.d, 1, n1(p), n2(lvt), P->fv.lev[lvt].so, ep, Y + A[p - 1].off1, 1.0,
                              P->fx.lev[p].bflag));
    }
    return SG_OK;
}

static int apply_cross_impl(sg_problem* P, const double* Tb, int S_out, int S_in, const double* X, double* Y) {
    const bool mass = Tb != nullptr;
    const auto& A = P->active;
    const int ng = (int)A.size();
    const int L = P->cfg.L;
    const int Wx = P->fx.W, Wv = P->fv.W;
    const bool vbox = P->fv.kind == SG_MESH_BOX, xbox = P->fx.kind == SG_MESH_BOX;
    std::vector<int64_t> offIn(ng), offOut(ng);
    for (int p = 0; p < ng; ++p) {
        offIn[p] = A[p].off1 * S_in;
        offOut[p] = A[p].off1 * S_out;
    }
    SG_TRY(launch_zero(P, set_size(P, SG_SET_ACTIVE, S_out), Y));
    auto n1 = [&](int l) { return P->fx.lev[l].n; };
    auto n2 = [&](int l) { return P->fv.lev[l].n; };
    // chain buffer layout: Q[p'][k], p' = 1..ng (index p'-1), k = 0..(#targets-1)
    std::vector<std::vector<int64_t>> qoff(ng);
    // ---------------- lower part
    // batched variant: all v-groups fanned out at once per source, per-group restriction
    // chains and Horner prolongation, and ONE line-swept x gather over all groups per target
    // (PAPER.md l.506-516 with A_{l,l'} = A_l E; same arithmetic, fewer passes over Y and X)
    bool lower_done = false;
    if (!mass) {
        int rc = cross_lower_batched(P, X, Y);
        if (rc == SG_OK) lower_done = true;
        else if (rc != SG_ERR_UNSUPPORTED) return rc;
    }
    const int nvg = lower_done ? 0 : (mass ? 1 : (int)P->vgroups.size());
    // Concurrent groups (small configurations): every group's transfer chain and gathers run as
    // an independent branch (own stream, chain and Horner workspaces, partial output), summed at
    // the end; otherwise all groups run serially on the handle's stream into Y.
    const int nxg_all = ng >= 2 ? (mass ? 1 : (int)P->xgroups.size()) : 0;
    // (not inside the strip-solve graph: forking these streams there crashed the driver in
    //  cuStreamEndCapture on the box's driver 580.159, profiles/r2d/dbg_gdb.log)
    const bool par = P->par_cross && !P->capturing && !lower_done && nvg + nxg_all <= (int)P->cx_streams.size() &&
                     (int64_t)set_size(P, SG_SET_ACTIVE, S_out) <= P->cx_y_n &&
                     (int64_t)set_size(P, SG_SET_ACTIVE, S_in) * 2 <= P->cx_h_n;
    cudaStream_t main_stream = P->stream;
    double* const wsZ0 = P->wsZ;
    double* const wsH0 = P->wsH;
    int nbranch = 0;
    if (par) SG_CUDA(cudaEventRecord(P->ev_cx_fork, main_stream));
    auto branch_begin = [&](double** Yd) -> int {
        if (!par) {
            *Yd = Y;
            return SG_OK;
        }
        const int br = nbranch++;
        P->stream = P->cx_streams[br];
        SG_CUDA(cudaStreamWaitEvent(P->stream, P->ev_cx_fork, 0));
        P->wsZ = P->cx_ws[br];
        P->wsH = P->cx_h[br];
        *Yd = P->cx_y[br];
        return launch_zero(P, set_size(P, SG_SET_ACTIVE, S_out), *Yd);
    };
    auto branch_end = [&]() -> int {
        if (!par) return SG_OK;
        SG_CUDA(cudaEventRecord(P->ev_cx_join[nbranch - 1], P->stream));
        P->stream = main_stream;
        P->wsZ = wsZ0;
        P->wsH = wsH0;
        return SG_OK;
    };
    for (int b = 0; b < nvg; ++b) {
        double* Yd = Y;
        SG_TRY(branch_begin(&Yd));
        const int vspec = mass ? P->mass_v : P->vgroups[b].spec;
        int64_t pos = 0;
        for (int pp = 1; pp <= ng; ++pp) {
            const int lx = pp, lv0 = L - pp;
            qoff[pp - 1].clear();
            for (int k = 0; k <= ng - pp; ++k) {
                qoff[pp - 1].push_back(pos);
                pos += (int64_t)S_in * n1(lx) * n2(lv0 - k);
            }
        }
        if ((size_t)pos > (par ? P->cx_ws_n : P->wsZ_n)) {
            set_error("apply_cross: chain workspace too small");
            return SG_ERR_STATE;
        }
        for (int pp = 1; pp <= ng; ++pp) {
            const int lx = pp, lv0 = L - pp;
            if (vbox) {
                VfanParams vp;
                vp.ng = vp.ng_int = 1;
                vp.vst[0] = P->fv.lev[lv0].fst[vspec];
                vp.out[0] = P->wsZ + qoff[pp - 1][0];
                SG_TRY(launch_vfan_st(P, P->fv.d, S_in, n1(lx), n2(lv0), P->fv.lev[lv0].so, P->fx.lev[lx].bflag, vp,
                                      X + offIn[pp - 1]));
            } else {
                FanoutList fl;
                fl.no = 1;
                fl.vals[0] = P->fv.lev[lv0].fm[vspec];
                fl.out[0] = P->wsZ + qoff[pp - 1][0];
                SG_TRY(launch_fanout(P, 1, Wv, S_in, n1(lx), n2(lv0), n2(lv0), P->fv.lev[lv0].cols, X + offIn[pp - 1], fl));
            }
        }
        // restriction chains in v, batched over sources: stage k maps Q[p'][k-1] -> Q[p'][k]
        for (int k = 1; k <= ng - 1; ++k) {
            std::vector<Job> jobs;
            for (int pp = 1; pp <= ng - k; ++pp) {
                const int lv0 = L - pp, lf = lv0 - k + 1, lc = lv0 - k;
                jobs.push_back({P->wsZ + qoff[pp - 1][k - 1], nullptr, P->wsZ + qoff[pp - 1][k], P->fv.lev[lf].rcols,
                                P->fv.lev[lf].rvals, n1(pp), n2(lf), n2(lc), 1.0, S_in, 1, Wv, 0});
                if (P->fv.kind == SG_MESH_BOX) jobs.back().box_mf = P->fv.lev[lf].m;
            }
            SG_TRY(launch_jobs(P, jobs));
        }
        // Horner prolongation in x, batched over targets: stage m lifts every target p >= m
        // from x-level m-1 to m and adds Q[m][p-m]
        double* hb[2] = {P->wsH, P->wsH + set_size(P, SG_SET_ACTIVE, S_in)};
        for (int m = 2; m <= ng; ++m) {
            std::vector<Job> jobs;
            for (int p = m; p <= ng; ++p) {
                const int lv = L - p;
                const double* in = m == 2 ? P->wsZ + qoff[0][p - 1] : hb[(m - 1) & 1] + offIn[p - 1];
                jobs.push_back({in, P->wsZ + qoff[m - 1][p - m], hb[m & 1] + offIn[p - 1], P->fx.lev[m].pcols,
                                P->fx.lev[m].pvals, n1(m - 1), n2(lv), n1(m), 1.0, S_in, 0, 2, 0});
                if (P->fx.kind == SG_MESH_BOX) {
                    jobs.back().box_mf = P->fx.lev[m].m;
                    jobs.back().box_d = P->fx.d;
                }
            }
            SG_TRY(launch_jobs(P, jobs));
        }
        for (int p = 1; p <= ng; ++p) {
            const int lv = L - p;
            const double* acc = p == 1 ? P->wsZ + qoff[0][0] : hb[p & 1] + offIn[p - 1];
            if (xbox) {
                XgatParams ep;
                ep.ne = 0;
                const int bo = mass ? 0 : (P->vgroups[b].bonly ? 1 : 0);
                if (mass) {
                    for (int s = 0; s < S_out; ++s)
                        for (int sp = 0; sp < S_in; ++sp)
                            if (Tb[s * S_in + sp] != 0.0)
                                ep.e[ep.ne++] = {acc, P->fx.lev[p].fst[P->mass_x], s, sp, 0, Tb[s * S_in + sp], P->fx.lev[p].fcls[P->mass_x]};
                } else {
                    for (const auto& ce : P->vgroups[b].comb[p]) ep.e[ep.ne++] = {acc, ce.st, ce.s_out, ce.s_in, bo, 1.0, ce.ctab};
                }
                if (ep.ne) SG_TRY(launch_xgat_st(P, P->fx.d, S_out, n1(p), n2(lv), P->fx.lev[p].so, P->fx.lev[p].bflag, ep,
                                                 Yd + offOut[p - 1], 1.0, P->fx.lev[p].m));
            } else {
                EntryList el;
                el.ne = 0;
                if (mass) {
                    for (int s = 0; s < S_out; ++s)
                        for (int sp = 0; sp < S_in; ++sp)
                            if (Tb[s * S_in + sp] != 0.0)
                                el.e[el.ne++] = {acc, P->fx.lev[p].fm[P->mass_x], Tb[s * S_in + sp], s, sp};
                } else {
                    for (const auto& ce : P->vgroups[b].comb[p]) el.e[el.ne++] = {acc, ce.vals, 1.0, ce.s_out, ce.s_in};
                }
                if (el.ne) SG_TRY(launch_gather(P, 0, Wx, S_out, n1(p), n2(lv), n1(p), P->fx.lev[p].cols, el,
                                                Yd + offOut[p - 1], 1.0));
            }
        }
        SG_TRY(branch_end());
    }
    // ---------------- upper part (targets p < sources p')
    bool upper_done = false;
    if (!mass && lower_done) {
        int rc = cross_upper_batched(P, X, Y);
        if (rc == SG_OK) upper_done = true;
        else if (rc != SG_ERR_UNSUPPORTED) return rc;
    }
    if (ng >= 2 && !upper_done) {
        const int nxg = mass ? 1 : (int)P->xgroups.size();
        for (int a = 0; a < nxg; ++a) {
            double* Yd = Y;
            SG_TRY(branch_begin(&Yd));
            const int xspec = mass ? P->mass_x : P->xgroups[a].spec;
            int64_t pos = 0;
            for (int pp = 2; pp <= ng; ++pp) {
                const int lv = L - pp;
                qoff[pp - 1].clear();
                for (int k = 0; k <= pp - 1; ++k) {       // k: x-level pp-k
                    qoff[pp - 1].push_back(pos);
                    pos += (int64_t)S_in * n1(pp - k) * n2(lv);
                }
            }
            if ((size_t)pos > (par ? P->cx_ws_n : P->wsZ_n)) {
                set_error("apply_cross: chain workspace too small (upper)");
                return SG_ERR_STATE;
            }
            for (int pp = 2; pp <= ng; ++pp) {
                const int lv = L - pp;
                if (xbox) {
                    XgatParams ep;
                    ep.ne = 0;
                    for (int s = 0; s < S_in; ++s)
                        ep.e[ep.ne++] = {X + offIn[pp - 1], P->fx.lev[pp].fst[xspec], s, s, 0, 1.0, P->fx.lev[pp].fcls[xspec]};
                    SG_TRY(launch_xgat_st(P, P->fx.d, S_in, n1(pp), n2(lv), P->fx.lev[pp].so, P->fx.lev[pp].bflag, ep,
                                          P->wsZ + qoff[pp - 1][0], 0.0, P->fx.lev[pp].m));
                } else {
                    FanoutList fl;
                    fl.no = 1;
                    fl.vals[0] = P->fx.lev[pp].fm[xspec];
                    fl.out[0] = P->wsZ + qoff[pp - 1][0];
                    SG_TRY(launch_fanout(P, 0, Wx, S_in, n1(pp), n2(lv), n1(pp), P->fx.lev[pp].cols, X + offIn[pp - 1], fl));
                }
            }
            // restriction chains in x, batched over sources: stage k maps x-level pp-k+1 -> pp-k
            for (int k = 1; k <= ng - 1; ++k) {
                std::vector<Job> jobs;
                for (int pp = k + 1; pp <= ng; ++pp) {
                    const int lv = L - pp, lf = pp - k + 1, lc = pp - k;
                    jobs.push_back({P->wsZ + qoff[pp - 1][k - 1], nullptr, P->wsZ + qoff[pp - 1][k],
                                    P->fx.lev[lf].rcols, P->fx.lev[lf].rvals, n1(lf), n2(lv), n1(lc), 1.0, S_in, 0, Wx,
                                    0});
                    if (P->fx.kind == SG_MESH_BOX) jobs.back().box_mf = P->fx.lev[lf].m;
                }
                SG_TRY(launch_jobs(P, jobs));
            }
            // Horner prolongation in v, batched over targets: at stage q every target p <= ng-q is
            // lifted from v-level L-ng+q-1 to L-ng+q and gets the source p' = ng-q added (if p' > p)
            double* hb[2] = {P->wsH, P->wsH + set_size(P, SG_SET_ACTIVE, S_in)};
            for (int q = 1; q <= ng - 1; ++q) {
                std::vector<Job> jobs;
                const int lvn = L - ng + q;
                for (int p = 1; p <= ng - q; ++p) {
                    const double* in = q == 1 ? P->wsZ + qoff[ng - 1][ng - p] : hb[(q - 1) & 1] + offIn[p - 1];
                    const int pp = ng - q;
                    const double* add = pp > p ? P->wsZ + qoff[pp - 1][pp - p] : nullptr;
                    jobs.push_back({in, add, hb[q & 1] + offIn[p - 1], P->fv.lev[lvn].pcols, P->fv.lev[lvn].pvals, n1(p),
                                    n2(lvn - 1), n2(lvn), 1.0, S_in, 1, 2, 0});
                    if (P->fv.kind == SG_MESH_BOX) {
                        jobs.back().box_mf = P->fv.lev[lvn].m;
                        jobs.back().box_d = P->fv.d;
                    }
                }
                SG_TRY(launch_jobs(P, jobs));
            }
            for (int p = 1; p <= ng - 1; ++p) {
                const int lvt = L - p;
                const double* acc = hb[(ng - p) & 1] + offIn[p - 1];   // written at stage q = ng - p
                if (vbox) {
                    XgatParams ep;
                    ep.ne = 0;
                    if (mass) {
                        for (int s = 0; s < S_out; ++s)
                            for (int sp = 0; sp < S_in; ++sp)
                                if (Tb[s * S_in + sp] != 0.0)
                                    ep.e[ep.ne++] = {acc, P->fv.lev[lvt].fst[P->mass_v], s, sp, 0, Tb[s * S_in + sp]};
                    } else {
                        for (const auto& ce : P->xgroups[a].comb[lvt]) ep.e[ep.ne++] = {acc, ce.st, ce.s_out, ce.s_in, 0, 1.0};
                    }
                    if (ep.ne) SG_TRY(launch_vgat_st(P, P->fv.d, S_out, n1(p), n2(lvt), P->fv.lev[lvt].so, ep,
                                                     Yd + offOut[p - 1], 1.0));
                } else {
                    EntryList el;
                    el.ne = 0;
                    if (mass) {
                        for (int s = 0; s < S_out; ++s)
                            for (int sp = 0; sp < S_in; ++sp)
                                if (Tb[s * S_in + sp] != 0.0)
                                    el.e[el.ne++] = {acc, P->fv.lev[lvt].fm[P->mass_v], Tb[s * S_in + sp], s, sp};
                    } else {
                        for (const auto& ce : P->xgroups[a].comb[lvt]) el.e[el.ne++] = {acc, ce.vals, 1.0, ce.s_out, ce.s_in};
                    }
                    if (el.ne) SG_TRY(launch_gather(P, 1, Wv, S_out, n1(p), n2(lvt), n2(lvt), P->fv.lev[lvt].cols, el,
                                                    Yd + offOut[p - 1], 1.0));
                }
            }
            SG_TRY(branch_end());
        }
    }
    if (par && nbranch > 0) {   // join the branches and sum their partial outputs
        for (int i = 0; i < nbranch; ++i) SG_CUDA(cudaStreamWaitEvent(main_stream, P->ev_cx_join[i], 0));
        SG_TRY(launch_sum_into(P, set_size(P, SG_SET_ACTIVE, S_out), nbranch, P->cx_y.data(), Y));
    }
    return SG_OK;
}

// ------------------------------------------------------- data (u0, inflow)
__global__ void k_gauss_nodes(int64_t n, int d, const int32_t* lat, double lo0, double lo1, double lo2, double h0,
                              double h1, double h2, double c0, double c1, double c2, double w, double scale,
                              double shift0, double shift1, double shift2, double* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double lo[3] = {lo0, lo1, lo2}, h[3] = {h0, h1, h2}, c[3] = {c0, c1, c2}, sh[3] = {shift0, shift1, shift2};
    double r2 = 0.0;
    for (int k = 0; k < d; ++k) {
        double y = lo[k] + h[k] * lat[k * n + i] - sh[k] - c[k];
        r2 += y * y;
    }
    out[i] = scale * exp(-r2 / w);
}

// out[k][m] (+)= coef * gx[k] * gv[m]
__global__ void k_outer(int64_t n1, int64_t n2, double coef, const double* gx, const double* gv, double* out,
                        int accumulate) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n1 * n2) return;
    int64_t k = t / n2, m = t - k * n2;
    double v = coef * gx[k] * gv[m];
    out[t] = accumulate ? out[t] + v : v;
}

// y[i*sy] += a * x[i*sx]
__global__ void k_axpy_strided(int64_t n, double a, const double* x, int64_t sx, double* y, int64_t sy) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i * sy] += a * x[i * sx];
}

static int gauss_on_level(sg_problem* P, Factor& f, int l, const double* c, double w, double s, const double* shift,
                          double* out) {
    Level& L = f.lev[l];
    const int cells = f.nc << (l - 1);
    double h[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, sh[3] = {0, 0, 0}, cc[3] = {0, 0, 0};
    for (int i = 0; i < f.d; ++i) {
        h[i] = (f.hi[i] - f.lo[i]) / cells;
        lo[i] = f.lo[i];
        cc[i] = c[i];
        if (shift) sh[i] = shift[i];
    }
    k_gauss_nodes<<<(int)((L.n + 255) / 256), 256, 0, P->stream>>>(L.n, f.d, L.lat, lo[0], lo[1], lo[2], h[0], h[1],
                                                                  h[2], cc[0], cc[1], cc[2], w, s, sh[0], sh[1],
                                                                  sh[2], out);
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

// U_0^- = combination of nodal interpolants of u0 (reading R8)
int interp_u0(sg_problem* P, double* u) {
    double* va = P->vec[7];
    const int64_t Na = set_size(P, SG_SET_ACTIVE, 1);
    double* gx = P->vec[10];
    double* gv = gx + (P->fx.lev[P->F].n + 16);
    for (int set = 0; set < 2; ++set) {
        const auto& gs = set == 0 ? P->active : P->coarse;
        for (const auto& g : gs) {
            double* dst = va + (set == 0 ? 0 : Na) + g.off1;
            for (int r = 0; r < P->cfg.nu0; ++r) {
                const sg_gauss_term& tm = P->cfg.u0[r];
                SG_TRY(gauss_on_level(P, P->fx, g.l1, tm.xc, tm.xw, tm.xs, nullptr, gx));
                SG_TRY(gauss_on_level(P, P->fv, g.l2, tm.vc, tm.vw, tm.vs, nullptr, gv));
                int64_t n = g.n1 * g.n2;
                k_outer<<<(int)((n + 255) / 256), 256, 0, P->stream>>>(g.n1, g.n2, tm.coef, gx, gv, dst, r > 0);
                P->launches++;
            }
        }
    }
    SG_CUDA(cudaGetLastError());
    return combine(P, 1, va, va + Na, u);
}

// inflow load for g = u0(r - beta t), constant beta, d = 1 (reading R9)
static int inflow_load(sg_problem* P, double t0, double* b) {
    const int S = P->S, F = P->F;
    const sg_config& c = P->cfg;
    double beta[2] = {0, 0};
    for (int r = 0; r < c.nbeta; ++r) beta[c.beta[r].axis] += c.beta[r].a[0] * c.beta[r].b[0];
    const double r6 = std::sqrt(6.0 / 5.0);
    const double xa = std::sqrt(3.0 / 7.0 - 2.0 / 7.0 * r6), xb = std::sqrt(3.0 / 7.0 + 2.0 / 7.0 * r6);
    const double wa = (18.0 + std::sqrt(30.0)) / 36.0, wb = (18.0 - std::sqrt(30.0)) / 36.0;
    const double gx_[4] = {-xb, -xa, xa, xb}, gw_[4] = {wb, wa, wa, wb};
    double* tmp = P->vec[10];
    const int64_t nF = std::max(P->fx.lev[F].n, P->fv.lev[F].n) + 16;
    double* gF = tmp;
    double* lF = tmp + nF;
    double* chainA = tmp + 2 * nF;
    double* chainB = tmp + 3 * nF;
    for (int mu = 0; mu < 4; ++mu) {
        const double t = t0 + c.tau * (gx_[mu] + 1.0) / 2.0;
        const double wt = gw_[mu] * c.tau / 2.0;
        double eta[2] = {1.0, gx_[mu]};
        for (int face = 0; face < 2; ++face) {          // 0: x faces, 1: v faces
            Factor& fb = face == 0 ? P->fv : P->fx;     // factor along the face
            Factor& fn = face == 0 ? P->fx : P->fv;     // factor normal to the face
            const double bn_axis = beta[face];
            for (int sface = -1; sface <= 1; sface += 2) {
                const double bn = sface * bn_axis;
                if (!(bn < 0.0)) continue;
                const double ypt = sface < 0 ? fn.lo[0] : fn.hi[0];
                for (int r = 0; r < c.nu0; ++r) {
                    const sg_gauss_term& tm = c.u0[r];
                    // normal factor value at the face point, shifted
                    const double* cn = face == 0 ? tm.xc : tm.vc;
                    const double wn = face == 0 ? tm.xw : tm.vw, sn = face == 0 ? tm.xs : tm.vs;
                    const double yy = ypt - bn_axis * t - cn[0];
                    const double gnorm = sn * std::exp(-yy * yy / wn);
                    const double* cb = face == 0 ? tm.vc : tm.xc;
                    const double wb2 = face == 0 ? tm.vw : tm.xw, sb = face == 0 ? tm.vs : tm.xs;
                    double shift[3] = {beta[1 - face] * t, 0, 0};
                    SG_TRY(gauss_on_level(P, fb, F, cb, wb2, sb, shift, gF));
                    // lF = M_F gF
                    EntryList el;
                    el.ne = 1;
                    const int mspec = face == 0 ? P->mass_v : P->mass_x;
                    el.e[0] = {gF, fb.lev[F].fm[mspec], 1.0, 0, 0};
                    SG_TRY(launch_gather(P, 1, fb.W, 1, 1, fb.lev[F].n, fb.lev[F].n, fb.lev[F].cols, el, lF, 0.0));
                    // per active grid: restrict to the grid's level along the face factor
                    for (const auto& g : P->active) {
                        const int lb = face == 0 ? g.l2 : g.l1;
                        const double* cur = lF;
                        double* bufs[2] = {chainA, chainB};
                        int k = 0;
                        for (int l = F; l > lb; --l) {
                            EntryList e2;
                            e2.ne = 1;
                            e2.e[0] = {cur, fb.lev[l].rvals, 1.0, 0, 0};
                            SG_TRY(launch_gather(P, 1, fb.W, 1, 1, fb.lev[l].n, fb.lev[l - 1].n, fb.lev[l].rcols, e2,
                                                 bufs[k], 0.0));
                            cur = bufs[k];
                            k ^= 1;
                        }
                        const int64_t nb_ = fb.lev[lb].n;
                        const int64_t node = sface < 0 ? 0 : (face == 0 ? g.n1 - 1 : g.n2 - 1);
                        for (int s = 0; s < S; ++s) {
                            double a = -bn * wt * eta[s] * c.u0[r].coef * gnorm;
                            double* dst = b + g.off1 * S + (int64_t)s * g.n1 * g.n2;
                            if (face == 0)
                                k_axpy_strided<<<(int)((nb_ + 255) / 256), 256, 0, P->stream>>>(
                                    nb_, a, cur, 1, dst + node * g.n2, 1);
                            else
                                k_axpy_strided<<<(int)((nb_ + 255) / 256), 256, 0, P->stream>>>(
                                    nb_, a, cur, 1, dst + node, g.n2);
                            P->launches++;
                        }
                    }
                }
            }
        }
    }
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

// b = eta(t_{j-1}^+) (x) M_cross trace + inflow
int rhs(sg_problem* P, int j, const double* trace, double* b) {
    const int S = P->S;
    double em[2] = {1.0, -1.0};
    SG_TRY(apply_cross(P, nullptr, em, S, 1, trace, b));
    if (P->cfg.inflow) SG_TRY(inflow_load(P, (j - 1) * P->cfg.tau, b));
    return SG_OK;
}

// trace = sum_s eta_s(t_j^-) u_s  (eta(1) = 1 for Legendre)
int trace_of(sg_problem* P, const double* u, double* tr) {
    const int S = P->S;
    for (const auto& g : P->active) {
        const int64_t n = gsize(g);
        SG_TRY(launch_copy(P, n, u + g.off1 * S, tr + g.off1));
        for (int s = 1; s < S; ++s) SG_TRY(launch_axpby(P, n, 1.0, u + g.off1 * S + s * n, 1.0, tr + g.off1));
    }
    return SG_OK;
}

}  // namespace sg
