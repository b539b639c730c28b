// Device-resident strip solver (sec. 4.3, l.540-566): the paper's Richardson
// iteration with the combination-technique preconditioner, whose block solves (15) run as
// batched block-Jacobi-preconditioned BiCGStab over all component grids at once.
//
// Every scalar of both iterations (Krylov coefficients, per-grid convergence flags, the
// outer step length, the update and solution norms, the stopping decision) lives on the
// device.  With graphs enabled (default) the whole strip solve is ONE CUDA graph: a
// conditional WHILE node for the Richardson iteration, nested IF nodes for the residual
// recomputation and the minimal-residual step (reading R13), and a nested WHILE node for
// the inner BiCGStab iteration whose body ends in a control kernel that sets the loop
// condition (cudaGraphSetConditional).  Apply kernels of converged grids exit on their
// grid's flag.  sg_solve_strip synchronises once, at the end, to read the counters.
// Without graphs (SG_NO_GRAPHS) the same bodies are enqueued by a host loop that reads the
// condition words from the device (one sync per loop test; debugging path).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sg_internal.cuh"

namespace sg {

static inline int64_t gsize(const Grid& g) { return g.n1 * g.n2; }

// ------------------------------------------------------- segmented vectors
struct SegTab {
    int nseg;
    int64_t off[MAX_SEG + 1];
    int blk[MAX_SEG + 1];
};
constexpr int SEG_CHUNK = 2048;

static SegTab make_segs(const std::vector<int64_t>& offs) {   // offs: nseg+1 element offsets
    SegTab t;
    t.nseg = (int)offs.size() - 1;
    int b = 0;
    for (int i = 0; i <= t.nseg; ++i) {
        t.off[i] = offs[i];
        t.blk[i] = b;
        if (i < t.nseg) b += (int)((offs[i + 1] - offs[i] + SEG_CHUNK - 1) / SEG_CHUNK);
    }
    return t;
}

__device__ inline int seg_of(const SegTab& t, int blk) {
    int g = 0;
    while (g + 1 < t.nseg && t.blk[g + 1] <= blk) ++g;
    return g;
}

// per-grid scalars: [0] rho [1] alpha [2] omega [3] bnorm2 [4] rnorm2 [5] conv [6] r0v [7] ts [8] tt [9] rr
constexpr int NSC = 10;

// partial[blk*K + j] = sum over the block's chunk of a_j * b_j
template <int K>
__global__ void k_seg_dot(SegTab t, const double* a0, const double* b0, const double* a1, const double* b1,
                          double* partial, const double* a2 = nullptr, const double* b2 = nullptr,
                          const double* scal = nullptr) {
    __shared__ double sh[K][8];
    const int g = seg_of(t, blockIdx.x);
    if (scal && scal[g * NSC + 5] != 0.0) {   // converged grid: its scalars are frozen
        if (threadIdx.x < K) partial[(int64_t)blockIdx.x * K + threadIdx.x] = 0.0;
        return;
    }
    const int64_t lo = t.off[g] + (int64_t)(blockIdx.x - t.blk[g]) * SEG_CHUNK;
    const int64_t hi = min(lo + SEG_CHUNK, t.off[g + 1]);
    double s[K];
    for (int j = 0; j < K; ++j) s[j] = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        s[0] += a0[i] * b0[i];
        if (K > 1) s[1] += a1[i] * b1[i];
        if (K > 2) s[2] += a2[i] * b2[i];
    }
    for (int j = 0; j < K; ++j) {
        double v = s[j];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) sh[j][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sh[threadIdx.x][w];
        partial[(int64_t)blockIdx.x * K + threadIdx.x] = v;
    }
}

// reduce partials of each segment into scal[g*NSC + slot_j], then apply `op`
// op 0: init (rho = bnorm2 = rr; conv if 0)
// op 1: alpha = rho / r0v
// op 2: omega = ts / tt
// op 3: rho_new, rnorm2 -> beta, convergence
__global__ void k_seg_finalize(SegTab t, int K, const double* partial, double* scal, int s0, int s1, int op,
                               double tol2) {
    const int g = blockIdx.x;
    if (g >= t.nseg) return;
    __shared__ double sh[3][32];
    double v[3] = {0.0, 0.0, 0.0};
    for (int b = t.blk[g] + threadIdx.x; b < t.blk[g + 1]; b += blockDim.x)
        for (int j = 0; j < K; ++j) v[j] += partial[(int64_t)b * K + j];
    for (int j = 0; j < K; ++j) {
        double x = v[j];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) sh[j][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double r[3] = {0.0, 0.0, 0.0};
    for (int j = 0; j < K; ++j)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r[j] += sh[j][w];
    double* sc = scal + g * NSC;
    if (op < 0) {
        sc[s0] = r[0];
        return;
    }
    if (op == 0) {
        sc[0] = r[0];
        sc[3] = r[0];
        sc[4] = r[0];
        sc[5] = (r[0] == 0.0) ? 1.0 : 0.0;
        sc[1] = 0.0;
        sc[2] = 0.0;
        sc[6] = 0.0;
        return;
    }
    if (sc[5] != 0.0) return;   // converged grid: scalars frozen
    if (op == 1) {              // alpha = rho / (r0.v)
        const double a = sc[0] / r[0];
        if (r[0] == 0.0 || !isfinite(a)) {
            sc[1] = 0.0;
            sc[2] = 0.0;
            sc[5] = 2.0;        // breakdown
        } else {
            sc[1] = a;
        }
    } else if (op == 2) {       // r = (t.s, t.t, s.s): omega, or converge at the half step
        if (r[2] <= tol2 * sc[3]) {
            sc[2] = 0.0;        // x += alpha p, r = s
            sc[7] = 1.0;        // converge after the update
        } else {
            const double om = r[0] / r[1];
            sc[2] = (r[1] > 0.0 && isfinite(om)) ? om : 0.0;
            sc[7] = 0.0;
        }
    } else if (op == 3) {       // r = (r0.r, r.r)
        const double rho_new = r[0];
        sc[4] = r[1];
        double beta = 0.0;
        if (sc[0] != 0.0 && sc[2] != 0.0) beta = (rho_new / sc[0]) * (sc[1] / sc[2]);
        sc[0] = rho_new;
        sc[6] = isfinite(beta) ? beta : 0.0;
        if (sc[7] != 0.0 || r[1] <= tol2 * sc[3]) sc[5] = 1.0;
        else if (rho_new == 0.0 || !isfinite(rho_new) || !isfinite(r[1]) || sc[2] == 0.0) sc[5] = 2.0;
    }
}

// s = r - alpha v
__global__ void k_bicg_s(SegTab t, const double* scal, const double* r, const double* v, double* s) {
    const int g = seg_of(t, blockIdx.x);
    const double* sc = scal + g * NSC;
    if (sc[5] != 0.0) return;
    const double al = sc[1];
    const int64_t lo = t.off[g] + (int64_t)(blockIdx.x - t.blk[g]) * SEG_CHUNK;
    const int64_t hi = min(lo + SEG_CHUNK, t.off[g + 1]);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s[i] = r[i] - al * v[i];
}

// x += alpha p + omega s ; r = s - omega t ; partial dots (r0.r, r.r)
__global__ void k_bicg_xr(SegTab tb, const double* scal, double* x, double* r, const double* p, const double* sx,
                          const double* s, const double* t, const double* r0, double* partial) {
    __shared__ double sh[2][8];
    const int g = seg_of(tb, blockIdx.x);
    const double* sc = scal + g * NSC;
    const bool active = sc[5] == 0.0;
    if (!active) {   // converged grid: frozen, no traffic
        if (threadIdx.x < 2) partial[(int64_t)blockIdx.x * 2 + threadIdx.x] = 0.0;
        return;
    }
    const double al = sc[1], om = sc[2];
    const int64_t lo = tb.off[g] + (int64_t)(blockIdx.x - tb.blk[g]) * SEG_CHUNK;
    const int64_t hi = min(lo + SEG_CHUNK, tb.off[g + 1]);
    double a0 = 0.0, a1 = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        double ri = r[i];
        if (active) {
            x[i] += al * p[i] + om * sx[i];
            ri = s[i] - om * t[i];
            r[i] = ri;
        }
        a0 += r0[i] * ri;
        a1 += ri * ri;
    }
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = a0;
        sh[1][threadIdx.x >> 5] = a1;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sh[threadIdx.x][w];
        partial[(int64_t)blockIdx.x * 2 + threadIdx.x] = v;
    }
}

// fused S = 1 variants with the point-Jacobi preconditioner: s = r - alpha v, sh = D^{-1} s
__global__ void k_bicg_s_pc(SegTab t, const double* scal, const double* r, const double* v, double* s,
                            const double* Dinv, double* sh) {
    const int g = seg_of(t, blockIdx.x);
    const double* sc = scal + g * NSC;
    if (sc[5] != 0.0) return;
    const double al = sc[1];
    const int64_t lo = t.off[g] + (int64_t)(blockIdx.x - t.blk[g]) * SEG_CHUNK;
    const int64_t hi = min(lo + SEG_CHUNK, t.off[g + 1]);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double si = r[i] - al * v[i];
        s[i] = si;
        sh[i] = Dinv[i] * si;
    }
}
// p = r + beta (p - omega v), ph = D^{-1} p (the next iteration's preconditioned direction)
__global__ void k_bicg_p_pc(SegTab t, const double* scal, double* p, const double* r, const double* v,
                            const double* Dinv, double* ph) {
    const int g = seg_of(t, blockIdx.x);
    const double* sc = scal + g * NSC;
    if (sc[5] != 0.0) return;
    const double be = sc[6], om = sc[2];
    const int64_t lo = t.off[g] + (int64_t)(blockIdx.x - t.blk[g]) * SEG_CHUNK;
    const int64_t hi = min(lo + SEG_CHUNK, t.off[g + 1]);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double pi = r[i] + be * (p[i] - om * v[i]);
        p[i] = pi;
        ph[i] = Dinv[i] * pi;
    }
}

// p = r + beta (p - omega v)
__global__ void k_bicg_p(SegTab t, const double* scal, double* p, const double* r, const double* v) {
    const int g = seg_of(t, blockIdx.x);
    const double* sc = scal + g * NSC;
    if (sc[5] != 0.0) return;
    const double be = sc[6], om = sc[2];
    const int64_t lo = t.off[g] + (int64_t)(blockIdx.x - t.blk[g]) * SEG_CHUNK;
    const int64_t hi = min(lo + SEG_CHUNK, t.off[g + 1]);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) p[i] = r[i] + be * (p[i] - om * v[i]);
}

// ---------------------------------------------- point-block Jacobi (time)
// D_k = sum_t T_t diag(A_t)_i diag(B_t)_a, an S x S block per node k = (i, a);
// the inner solver is right-preconditioned with D^{-1} (the paper
// uses GMRES+ILU for eq. (15); this is the GPU-friendly point-block variant).
struct DiagTerm {
    double T[4];
    const double* dA;
    const double* dB;
};
__global__ void k_extract_diag(int64_t n, int W, const int32_t* cols, const double* vals, double* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = 0.0;
    for (int k = 0; k < W; ++k)
        if (cols[k * n + i] == (int32_t)i) d += vals[k * n + i];
    out[i] = d;
}
__global__ void k_diag_block_inv(int64_t n1, int64_t n2, int S, int nt, const DiagTerm* terms, double* Dinv) {
    const int64_t n = n1 * n2;
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t i = k / n2, a = k - i * n2;
    double D[4] = {0, 0, 0, 0};
    for (int t = 0; t < nt; ++t) {
        const double f = terms[t].dA[i] * terms[t].dB[a];
        for (int q = 0; q < S * S; ++q) D[q] += terms[t].T[q] * f;
    }
    if (S == 1) {
        Dinv[k] = 1.0 / D[0];
    } else {
        const double det = D[0] * D[3] - D[1] * D[2];
        Dinv[0 * n + k] = D[3] / det;
        Dinv[1 * n + k] = -D[1] / det;
        Dinv[2 * n + k] = -D[2] / det;
        Dinv[3 * n + k] = D[0] / det;
    }
}

int build_block_jacobi(sg_problem* P) {
    const int S = P->S;
    std::vector<const Grid*> gr;
    for (auto& g : P->active) gr.push_back(&g);
    for (auto& g : P->coarse) gr.push_back(&g);
    int64_t tot = 0;
    for (auto* g : gr) tot += (int64_t)S * S * gsize(*g);
    SG_CUDA(cudaMalloc(&P->dinv, sizeof(double) * tot));
    // diagonal vectors of every used spec on every level
    auto diagvec = [&](Factor& f, int spec, int l, double** out) -> int {
        Level& L = f.lev[l];
        SG_CUDA(cudaMalloc(out, sizeof(double) * L.n));
        k_extract_diag<<<(int)((L.n + 255) / 256), 256, 0, P->stream>>>(L.n, f.W, L.cols, L.fm[spec], *out);
        P->launches++;
        return SG_OK;
    };
    std::vector<double*> tmp;
    DiagTerm* dterms;
    SG_CUDA(cudaMalloc(&dterms, sizeof(DiagTerm) * P->terms.size()));
    int64_t off = 0;
    for (auto* g : gr) {
        std::vector<DiagTerm> ht;
        for (auto& t : P->terms) {
            DiagTerm d;
            for (int q = 0; q < 4; ++q) d.T[q] = t.T[q];
            double *a, *b;
            SG_TRY(diagvec(P->fx, t.xs, g->l1, &a));
            SG_TRY(diagvec(P->fv, t.vs, g->l2, &b));
            tmp.push_back(a);
            tmp.push_back(b);
            d.dA = a;
            d.dB = b;
            ht.push_back(d);
        }
        SG_CUDA(cudaMemcpyAsync(dterms, ht.data(), sizeof(DiagTerm) * ht.size(), cudaMemcpyHostToDevice, P->stream));
        const int64_t n = gsize(*g);
        k_diag_block_inv<<<(int)((n + 255) / 256), 256, 0, P->stream>>>(g->n1, g->n2, S, (int)ht.size(), dterms,
                                                                       P->dinv + off);
        P->launches++;
        SG_CUDA(cudaGetLastError());
        SG_CUDA(cudaStreamSynchronize(P->stream));
        for (double* q : tmp) cudaFree(q);
        tmp.clear();
        off += (int64_t)S * S * n;
    }
    cudaFree(dterms);
    return SG_OK;
}

// out = D^{-1} in on every segment (segment = one grid, S x n block)
__global__ void k_seg_precond(SegTab t, int S, const double* scal, const double* Dinv, const double* in, double* out) {
    const int g = seg_of(t, blockIdx.x);
    if (scal[g * NSC + 5] != 0.0) return;
    const int64_t base = t.off[g];
    const int64_t n = (t.off[g + 1] - base) / S;
    const double* Dg = Dinv + base * S;
    const int64_t lo = base + (int64_t)(blockIdx.x - t.blk[g]) * SEG_CHUNK;
    const int64_t hi = min(lo + SEG_CHUNK, t.off[g + 1]);
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        if (S == 1) {
            out[e] = Dg[e - base] * in[e];
        } else {
            const int64_t le = e - base;
            const int s = (int)(le / n);
            const int64_t k = le - s * n;
            out[e] = Dg[(s * 2 + 0) * n + k] * in[base + k] + Dg[(s * 2 + 1) * n + k] * in[base + n + k];
        }
    }
}


// ------------------------------------------------------------ combination
// du_p = dhat_p - (E^(1)_{l1<-l1-1} x Id) dhat_{(l1-1,l2)}  (l.557-565)
int combine(sg_problem* P, int S, const double* dhat_a, const double* dhat_c, double* du) {
    const auto& A = P->active;
    for (size_t p = 0; p < A.size(); ++p) {
        const Grid& g = A[p];
        SG_TRY(launch_copy(P, S * gsize(g), dhat_a + g.off1 * S, du + g.off1 * S));
        if (g.l1 > 1) {
            const Grid& c = P->coarse[g.l1 - 2];   // (l1-1, l2)
            EntryList el;
            el.ne = 0;
            for (int s = 0; s < S; ++s)
                el.e[el.ne++] = {dhat_c + c.off1 * S, P->fx.lev[g.l1].pvals, -1.0, s, s};
            SG_TRY(launch_gather(P, 0, 2, S, c.n1, c.n2, g.n1, P->fx.lev[g.l1].pcols, el, du + g.off1 * S, 1.0));
        }
    }
    return SG_OK;
}


// ============================================================ solver control
// one-segment reduction of K partial sums into out[0..K-1]
__global__ void k_dot_final(const double* partial, int nblk, int K, double* out) {
    __shared__ double sh[3][32];
    double v[3] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nblk; b += blockDim.x)
        for (int j = 0; j < K; ++j) v[j] += partial[(int64_t)b * K + j];
    for (int j = 0; j < K; ++j) {
        double x = v[j];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) sh[j][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double r = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sh[threadIdx.x][w];
        out[threadIdx.x] = r;
    }
}

struct Conds {                          // conditional handles of the captured solve (use = 0: host loop)
    cudaGraphConditionalHandle outer, need_r, inner, mr;
    int use;
};
__device__ __forceinline__ void set_cond(cudaGraphConditionalHandle h, int use, int v, int* word) {
    *word = v;
    if (use) cudaGraphSetConditional(h, v ? 1u : 0u);
}

struct GridTab {                        // per solve grid: DOF of one apply
    int ng;
    double dof[MAX_SEG];
};

__global__ void k_outer_init(SolveCtl* c, int mode, Conds cd) {
    c->it = 0;
    c->mr = mode == 2;
    c->have_r = 0;
    c->done = 0;
    c->nd = c->nd_prev = 0.0;
    c->omega = 1.0;
    c->nu2 = c->dots[0];                // (u0, M u0) of the initial guess
    set_cond(cd.outer, cd.use, 1, &c->cond_outer);
}

// top of a Richardson iteration: recompute r = A u - b unless the MR recursion kept it current
__global__ void k_outer_begin(SolveCtl* c, Conds cd) {
    c->it++;
    c->outer_iters++;
    const int need_r = !c->have_r;
    c->need_r_runs += need_r;
    c->mr_runs += c->mr;
    set_cond(cd.need_r, cd.use, need_r, &c->cond_need_r);
    set_cond(cd.mr, cd.use, c->mr, &c->cond_mr);
    c->omega = 1.0;                     // plain Richardson step unless the MR branch sets it
    c->have_r = 0;
}

// residual-minimising step length omega = (r, A du) / (A du, A du) (reading R13)
__global__ void k_mr_omega(SolveCtl* c) {
    const double rw = c->dots[2], ww = c->dots[3];
    const double om = rw / ww;
    c->omega = (ww > 0.0 && isfinite(om)) ? om : 1.0;
    c->have_r = 1;                      // r <- r - omega A du follows
}

// y += sign * omega * x (omega from the device)
__global__ void k_axpy_omega(int64_t n, const SolveCtl* c, double sign, const double* __restrict__ x,
                             double* __restrict__ y) {
    const double a = sign * c->omega;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] += a * x[i];
}

// end of a Richardson iteration: dots[0] = (u_old, M du), dots[1] = (du, M du).
// ||u_new||^2 = ||u_old||^2 - 2 omega (u_old, M du) + omega^2 ||du||^2 (exact identity);
// stop when ||du||_M <= rtol ||u||_M (the unscaled preconditioned residual P^{-1} r, also in MR mode).
__global__ void k_outer_end(SolveCtl* c, double rtol, int max_iter, int mode, Conds cd) {
    const double om = c->omega, nd2 = c->dots[1];
    const double nu2 = c->nu2 - 2.0 * om * c->dots[0] + om * om * nd2;
    c->nu2 = nu2;
    const double nd = sqrt(fmax(nd2, 0.0)), nu = sqrt(fmax(nu2, 0.0));
    c->nd = nd;
    int done = 0;
    if (!isfinite(nd2) || !isfinite(nu2)) {
        done = 3;
        c->outer_nonfinite++;
    } else if (nd <= rtol * nu || nd == 0.0) {
        done = 1;
    } else {
        // safeguard (reading R13): the update norm grew -> residual-minimising steps from now on
        if (!c->mr && mode == 0 && c->it >= 2 && nd > c->nd_prev) {
            c->mr = 1;
            c->mr_switches++;
        }
        if (c->it >= max_iter) {
            done = 2;
            c->outer_unconverged++;
        }
    }
    if (c->it >= 1 && c->it <= 256) {
        c->hist_nd[c->it - 1] = nd;
        c->hist_om[c->it - 1] = om;
    }
    c->nd_prev = nd;
    c->done = done;
    set_cond(cd.outer, cd.use, done == 0, &c->cond_outer);
}

// after the BiCGStab initialisation: grids with b = 0 are converged; start the loop if any is not
__global__ void k_inner_init(SolveCtl* c, const double* scal, int ng, Conds cd) {
    int any = 0;
    for (int g = 0; g < ng; ++g) {
        c->act[g] = scal[g * NSC + 5] == 0.0;
        any |= c->act[g];
    }
    c->inner_it = 0;
    set_cond(cd.inner, cd.use, any, &c->cond_inner);
}

// end of a BiCGStab iteration: count the applies of the grids that were active, continue while
// any grid is unconverged and inner_it < maxit; record breakdowns and max-iteration exits
__global__ void k_inner_ctl(SolveCtl* c, const double* scal, GridTab gt, int maxit, Conds cd) {
    c->inner_it++;
    c->inner_iters++;
    int any = 0;
    for (int g = 0; g < gt.ng; ++g) {
        if (c->act[g]) {
            c->n_applies += 2;
            c->dof_applied += 2.0 * gt.dof[g];
        }
        c->act[g] = scal[g * NSC + 5] == 0.0;
        any |= c->act[g];
    }
    if (!any || c->inner_it >= maxit) {
        for (int g = 0; g < gt.ng; ++g) {
            const double f = scal[g * NSC + 5];
            if (f == 2.0) c->inner_breakdowns++;
            else if (f == 0.0) c->inner_maxit++;
        }
        any = 0;
    }
    set_cond(cd.inner, cd.use, any, &c->cond_inner);
}

// device timestamps around a strip-operator apply (timing mode): phase 0 start, phase 1 end
// (accumulates the elapsed globaltimer ns and the apply's algorithmic bytes / FLOPs unless the
// grid is converged, i.e. its kernels exited without work)
__global__ void k_tstamp(SolveCtl* c, const double* skip, int slot, int phase, double bytes, double flops) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (phase == 0) {
        c->t0[slot] = t;
        return;
    }
    if (skip && *skip != 0.0) return;
    atomicAdd(&c->apply_ns, (double)(t - c->t0[slot]));   // (concurrent applies: atomics)
    atomicAdd((unsigned long long*)&c->timed_applies, 1ull);
    atomicAdd(&c->alg_bytes, bytes);
    atomicAdd(&c->alg_flops, flops);
}

// ------------------------------------------------------------------ helpers
static int dot_into(sg_problem* P, int64_t n, const double* a0, const double* b0, const double* a1,
                    const double* b1, double* out) {
    std::vector<int64_t> offs = {0, n};
    SegTab t = make_segs(offs);
    const int nblk = t.blk[1];
    if (a1) {
        k_seg_dot<2><<<nblk, 256, 0, P->stream>>>(t, a0, b0, a1, b1, P->red);
        k_dot_final<<<1, 256, 0, P->stream>>>(P->red, nblk, 2, out);
    } else {
        k_seg_dot<1><<<nblk, 256, 0, P->stream>>>(t, a0, b0, nullptr, nullptr, P->red);
        k_dot_final<<<1, 256, 0, P->stream>>>(P->red, nblk, 1, out);
    }
    P->launches += 2;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

static int axpy_omega(sg_problem* P, int64_t n, double sign, const double* x, double* y) {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_axpy_omega<<<std::max(blocks, 1), 256, 0, P->stream>>>(n, P->ctl, sign, x, y);
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

// A structured control node.  Graph mode: a conditional node (WHILE or IF) added to the graph
// being captured on P->stream, its body captured on the next nesting stream.  Host mode: the
// host evaluates the condition word (written by the kernel that sets the condition).
template <class F>
static int cond_region(sg_problem* P, bool graph, cudaGraphConditionalHandle h, bool is_while, int depth,
                       const int* dev_word, int64_t* body_launches, F body) {
    if (graph) {
        cudaStreamCaptureStatus st;
        cudaGraph_t cg;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        SG_CUDA(cudaStreamGetCaptureInfo(P->stream, &st, nullptr, &cg, &deps, &nd));
        if (st != cudaStreamCaptureStatusActive) {
            set_error("cond_region: stream not capturing");
            return SG_ERR_STATE;
        }
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = is_while ? cudaGraphCondTypeWhile : cudaGraphCondTypeIf;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        SG_CUDA(cudaGraphAddNode(&node, cg, deps, nd, &np));
        SG_CUDA(cudaStreamUpdateCaptureDependencies(P->stream, &node, 1, cudaStreamSetCaptureDependencies));
        cudaGraph_t bodyg = np.conditional.phGraph_out[0];
        while ((int)P->cap_streams.size() <= depth) {
            cudaStream_t s;
            SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            P->cap_streams.push_back(s);
        }
        cudaStream_t outer = P->stream, bs = P->cap_streams[depth];
        SG_CUDA(cudaStreamBeginCaptureToGraph(bs, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        P->stream = bs;
        const int64_t l0 = P->launches;
        int rc = body();
        *body_launches = P->launches - l0;
        P->launches = l0;
        P->stream = outer;
        cudaGraph_t dummy;
        cudaError_t ce = cudaStreamEndCapture(bs, &dummy);
        if (rc != SG_OK) return rc;
        SG_CUDA(ce);
        return SG_OK;
    }
    for (;;) {
        int w = 0;
        SG_CUDA(cudaMemcpyAsync(&P->hctl->pad0, dev_word, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
        SG_CUDA(cudaStreamSynchronize(P->stream));
        w = P->hctl->pad0;
        if (!w) break;
        SG_TRY(body());
        if (!is_while) break;
    }
    return SG_OK;
}

// ------------------------------------------------------------------ the solve
struct SolveArgs {
    const double* b;
    double* u;
    double rtol, inner_rtol;
    int max_iter;
};
struct RegionLaunches {                 // our launches per execution of each region
    int64_t pre = 0, outer = 0, need_r = 0, mr = 0, inner = 0;
};

static void solve_grids(sg_problem* P, std::vector<const Grid*>& gr, std::vector<int64_t>& offs) {
    gr.clear();
    for (auto& g : P->active) gr.push_back(&g);
    for (auto& g : P->coarse) gr.push_back(&g);
    offs.assign(1, 0);
    for (auto* g : gr) offs.push_back(offs.back() + (int64_t)P->S * gsize(*g));
}

// BiCGStab on all solve grids (active then coarse) for the block systems (15), right-preconditioned
// with the point-block Jacobi D^{-1}; x = 0 initial guess; per-grid stopping ||r_g|| <= rtol ||b_g||.
static int enqueue_bicgstab(sg_problem* P, bool graph, const Conds& cd, const double* b, double* x, double rtol,
                            int maxit, RegionLaunches* rl) {
    const int S = P->S;
    std::vector<const Grid*> gr;
    std::vector<int64_t> offs;
    solve_grids(P, gr, offs);
    const int64_t N = offs.back();
    SegTab t = make_segs(offs);
    const int nblk = t.blk[t.nseg];
    double *r = P->vec[0], *r0 = P->vec[1], *p = P->vec[2], *v = P->vec[3], *s = P->vec[4], *tt = P->vec[5];
    double *ph = P->vec[13], *sh = P->vec[14];
    const bool fuse = S == 1;   // preconditioner fused into the s / p updates
    const double tol2 = rtol * rtol;
    SG_TRY(launch_zero(P, N, x));
    SG_TRY(launch_copy(P, N, b, r));
    SG_TRY(launch_copy(P, N, b, r0));
    SG_TRY(launch_copy(P, N, b, p));
    k_seg_dot<1><<<nblk, 256, 0, P->stream>>>(t, b, b, nullptr, nullptr, P->red);
    k_seg_finalize<<<t.nseg, 256, 0, P->stream>>>(t, 1, P->red, P->scal, 9, 9, 0, 0.0);
    P->launches += 2;
    if (fuse) {   // ph = D^{-1} p for the first iteration (later produced by k_bicg_p_pc)
        k_seg_precond<<<nblk, 256, 0, P->stream>>>(t, S, P->scal, P->dinv, p, ph);
        P->launches++;
    }
    k_inner_init<<<1, 1, 0, P->stream>>>(P->ctl, P->scal, t.nseg, cd);
    P->launches++;
    SG_CUDA(cudaGetLastError());
    GridTab gt;
    gt.ng = t.nseg;
    for (int i = 0; i < t.nseg; ++i) gt.dof[i] = (double)(offs[i + 1] - offs[i]);
    // all grids' applies of one half-iteration: serial on P->stream, or (small configurations)
    // forked onto one stream per grid with private workspaces and joined again
    auto applies = [&](const double* in, double* out) -> int {
        if (P->d1_ok) {
            // d = 1: every grid's fused apply in ONE launch (per-grid convergence flags inside)
            const int n = (int)gr.size();
            std::vector<const double*> xs(n), sk(n);
            std::vector<double*> ys(n);
            std::vector<double> by(n, 0.0), fl(n, 0.0);
            if (P->timing) {
                k_tstamp<<<1, 1, 0, P->stream>>>(P->ctl, nullptr, P->stamp_slot, 0, 0.0, 0.0);
                P->launches++;
            }
            for (int i = 0; i < n; ++i) {
                xs[i] = in + offs[i];
                ys[i] = out + offs[i];
                sk[i] = P->scal + i * NSC + 5;
            }
            for (int i = 0; i < n; ++i) {   // (factor bytes per grid for the roofline accounting)
                double fb = 0.0;
                if (P->timing) {
                    const double* x1 = xs[i];
                    (void)x1;
                    fb = 8.0 * 3 * ((double)P->vorder.size() * gr[i]->n2 + P->d1_nent[gr[i]->l1] * (double)gr[i]->n1);
                    by[i] = 16.0 * S * (double)gsize(*gr[i]) + fb;
                    fl[i] = apply_flops(P, *gr[i]);
                }
            }
            SG_TRY(launch_d1fused(P, n, gr.data(), xs.data(), ys.data(), sk.data(), nullptr));
            if (P->timing) SG_TRY(launch_tstamp_batch(P, n, sk.data(), by.data(), fl.data()));
            return SG_OK;
        }
        if (!P->par_applies) {
            for (size_t i = 0; i < gr.size(); ++i)
                SG_TRY(apply_diag(P, *gr[i], in + offs[i], out + offs[i], P->scal + i * NSC + 5));
            return SG_OK;
        }
        cudaStream_t main = P->stream;
        double* ws0 = P->wsZ;
        const size_t wsn0 = P->wsZ_n;
        SG_CUDA(cudaEventRecord(P->ev_fork, main));
        int rc = SG_OK;
        for (size_t i = 0; i < gr.size() && rc == SG_OK; ++i) {
            SG_CUDA(cudaStreamWaitEvent(P->par_streams[i], P->ev_fork, 0));
            P->stream = P->par_streams[i];
            P->wsZ = P->par_ws[i];
            P->wsZ_n = P->par_ws_n[i];
            P->stamp_slot = (int)i;
            rc = apply_diag(P, *gr[i], in + offs[i], out + offs[i], P->scal + i * NSC + 5);
            if (rc == SG_OK && cudaEventRecord(P->ev_join[i], P->par_streams[i]) != cudaSuccess) rc = SG_ERR_CUDA;
        }
        P->stream = main;
        P->stamp_slot = 63;
        P->wsZ = ws0;
        P->wsZ_n = wsn0;
        SG_TRY(rc);
        for (size_t i = 0; i < gr.size(); ++i) SG_CUDA(cudaStreamWaitEvent(main, P->ev_join[i], 0));
        return SG_OK;
    };
    auto body = [&]() -> int {
        // v = A D^{-1} p
        if (!fuse) {
            k_seg_precond<<<nblk, 256, 0, P->stream>>>(t, S, P->scal, P->dinv, p, ph);
            P->launches++;
        }
        SG_TRY(applies(ph, v));
        k_seg_dot<1><<<nblk, 256, 0, P->stream>>>(t, r0, v, nullptr, nullptr, P->red, nullptr, nullptr, P->scal);
        k_seg_finalize<<<t.nseg, 256, 0, P->stream>>>(t, 1, P->red, P->scal, 6, 6, 1, tol2);
        P->launches += 2;
        if (fuse) {
            k_bicg_s_pc<<<nblk, 256, 0, P->stream>>>(t, P->scal, r, v, s, P->dinv, sh);
            P->launches++;
        } else {
            k_bicg_s<<<nblk, 256, 0, P->stream>>>(t, P->scal, r, v, s);
            k_seg_precond<<<nblk, 256, 0, P->stream>>>(t, S, P->scal, P->dinv, s, sh);
            P->launches += 2;
        }
        // t = A D^{-1} s
        SG_TRY(applies(sh, tt));
        k_seg_dot<3><<<nblk, 256, 0, P->stream>>>(t, tt, s, tt, tt, P->red, s, s, P->scal);
        k_seg_finalize<<<t.nseg, 256, 0, P->stream>>>(t, 3, P->red, P->scal, 7, 8, 2, tol2);
        k_bicg_xr<<<nblk, 256, 0, P->stream>>>(t, P->scal, x, r, ph, sh, s, tt, r0, P->red);
        k_seg_finalize<<<t.nseg, 256, 0, P->stream>>>(t, 2, P->red, P->scal, 0, 4, 3, tol2);
        if (fuse)
            k_bicg_p_pc<<<nblk, 256, 0, P->stream>>>(t, P->scal, p, r, v, P->dinv, ph);
        else
            k_bicg_p<<<nblk, 256, 0, P->stream>>>(t, P->scal, p, r, v);
        k_inner_ctl<<<1, 1, 0, P->stream>>>(P->ctl, P->scal, gt, maxit, cd);
        P->launches += 6;
        SG_CUDA(cudaGetLastError());
        return SG_OK;
    };
    return cond_region(P, graph, cd.inner, true, 1, &P->ctl->cond_inner, &rl->inner, body);
}

// The strip solve (l.540-566) enqueued on P->stream (captured or not).
static int enqueue_solve(sg_problem* P, bool graph, const Conds& cd, const SolveArgs& a, RegionLaunches* rl) {
    const int S = P->S;
    const int64_t Na = set_size(P, SG_SET_ACTIVE, S), Nc = set_size(P, SG_SET_COARSE, S);
    double* r = P->vec[6];
    double* rhs = P->vec[7];      // [active | coarse]
    double* dhat = P->vec[8];     // [active | coarse]
    double* du = P->vec[9];
    double* Mw = P->vec[10];
    double* w = P->vec[15];       // A du (minimal-residual steps)
    double Mt[4] = {0, 0, 0, 0};  // time mass of the L2(I_j x Omega) norm
    Mt[0] = P->cfg.tau;
    if (S == 2) Mt[3] = P->cfg.tau / 3.0;
    (void)Nc;
    const int64_t l0 = P->launches;
    // ||u0||^2 of the initial guess, then the loop state
    SG_TRY(apply_cross(P, nullptr, Mt, S, S, a.u, Mw));
    SG_TRY(dot_into(P, Na, a.u, Mw, nullptr, nullptr, P->ctl->dots));
    k_outer_init<<<1, 1, 0, P->stream>>>(P->ctl, P->outer_mode, cd);
    P->launches++;
    SG_CUDA(cudaGetLastError());
    rl->pre = P->launches - l0;
    auto outer_body = [&]() -> int {
        k_outer_begin<<<1, 1, 0, P->stream>>>(P->ctl, cd);
        P->launches++;
        // r = A u - b (skipped while the MR recursion keeps r current)
        SG_TRY(cond_region(P, graph, cd.need_r, false, 1, &P->ctl->cond_need_r, &rl->need_r, [&]() -> int {
            SG_TRY(apply_cross(P, nullptr, nullptr, S, S, a.u, r));
            return launch_axpby(P, Na, -1.0, a.b, 1.0, r);
        }));
        // block right-hand sides: r on |l| = L, (Id x E^T x Id) r on |l| = L-1 (l.550-553)
        SG_TRY(launch_copy(P, Na, r, rhs));
        for (size_t c = 0; c < P->coarse.size(); ++c) {
            const Grid& cg = P->coarse[c];
            const Grid& src = P->active[cg.l1];   // (c1+1, c2)
            EntryList el;
            el.ne = 0;
            for (int s = 0; s < S; ++s) el.e[el.ne++] = {r + src.off1 * S, P->fx.lev[src.l1].rvals, 1.0, s, s};
            SG_TRY(launch_gather(P, 0, P->fx.W, S, src.n1, src.n2, cg.n1, P->fx.lev[src.l1].rcols, el,
                                 rhs + Na + cg.off1 * S, 0.0));
        }
        // block solves (15)
        SG_TRY(enqueue_bicgstab(P, graph, cd, rhs, dhat, a.inner_rtol, 500, rl));
        // combination (l.557-565): du = P^{-1} r
        SG_TRY(combine(P, S, dhat, dhat + Na, du));
        // minimal-residual step length (reading R13): w = A du, omega = (r,w)/(w,w), r -= omega w
        SG_TRY(cond_region(P, graph, cd.mr, false, 1, &P->ctl->cond_mr, &rl->mr, [&]() -> int {
            SG_TRY(apply_cross(P, nullptr, nullptr, S, S, du, w));
            SG_TRY(dot_into(P, Na, r, w, w, w, P->ctl->dots + 2));
            k_mr_omega<<<1, 1, 0, P->stream>>>(P->ctl);
            P->launches++;
            return axpy_omega(P, Na, -1.0, w, r);
        }));
        // norms: (u, M du), (du, M du); u -= omega du; stopping test and safeguard
        SG_TRY(apply_cross(P, nullptr, Mt, S, S, du, Mw));
        SG_TRY(dot_into(P, Na, a.u, Mw, du, Mw, P->ctl->dots));
        SG_TRY(axpy_omega(P, Na, -1.0, du, a.u));
        k_outer_end<<<1, 1, 0, P->stream>>>(P->ctl, a.rtol, a.max_iter, P->outer_mode, cd);
        P->launches++;
        SG_CUDA(cudaGetLastError());
        return SG_OK;
    };
    int64_t outer_total = 0;
    SG_TRY(cond_region(P, graph, cd.outer, true, 0, &P->ctl->cond_outer, &outer_total, outer_body));
    rl->outer = outer_total;   // the body's own launches (nested regions counted separately)
    // (host mode counts every launch as it happens; graph mode multiplies the per-region counts
    // by the device's execution counters after the solve)
    return SG_OK;
}

// cached graph of the whole strip solve for (b, u, tolerances, mode, timing)
static int solve_graph(sg_problem* P, const SolveArgs& a, sg_problem::SolveGraph** out) {
    for (auto& sgp : P->solve_graphs)
        if (sgp.b == a.b && sgp.u == a.u && sgp.rtol == a.rtol && sgp.inner_rtol == a.inner_rtol &&
            sgp.max_iter == a.max_iter && sgp.mode == P->outer_mode && sgp.timing == (int)P->timing) {
            *out = &sgp;
            return SG_OK;
        }
    if (P->solve_graphs.size() >= 8) {
        cudaGraphExecDestroy(P->solve_graphs.front().exec);
        P->solve_graphs.erase(P->solve_graphs.begin());
    }
    cudaGraph_t g;
    SG_CUDA(cudaGraphCreate(&g, 0));
    Conds cd;
    cd.use = 1;
    SG_CUDA(cudaGraphConditionalHandleCreate(&cd.outer, g, 0, 0));
    SG_CUDA(cudaGraphConditionalHandleCreate(&cd.need_r, g, 0, 0));
    SG_CUDA(cudaGraphConditionalHandleCreate(&cd.inner, g, 0, 0));
    SG_CUDA(cudaGraphConditionalHandleCreate(&cd.mr, g, 0, 0));
    cudaStream_t saved = P->stream;
    SG_CUDA(cudaStreamBeginCaptureToGraph(P->gstream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    P->stream = P->gstream;
    P->capturing = true;
    RegionLaunches rl;
    const int64_t l0 = P->launches;
    int rc = enqueue_solve(P, true, cd, a, &rl);
    P->launches = l0;
    P->capturing = false;
    P->stream = saved;
    cudaGraph_t captured;
    cudaError_t ce = cudaStreamEndCapture(P->gstream, &captured);
    if (rc != SG_OK) {
        cudaGraphDestroy(g);
        return rc;
    }
    SG_CUDA(ce);
    sg_problem::SolveGraph sgp;
    sgp.b = a.b;
    sgp.u = a.u;
    sgp.rtol = a.rtol;
    sgp.inner_rtol = a.inner_rtol;
    sgp.max_iter = a.max_iter;
    sgp.mode = P->outer_mode;
    sgp.timing = (int)P->timing;
    sgp.l_pre = rl.pre;
    sgp.l_outer = rl.outer;
    sgp.l_need_r = rl.need_r;
    sgp.l_mr = rl.mr;
    sgp.l_inner = rl.inner;
    cudaError_t ie = cudaGraphInstantiate(&sgp.exec, g, 0);
    cudaGraphDestroy(g);
    SG_CUDA(ie);
    P->solve_graphs.push_back(sgp);
    *out = &P->solve_graphs.back();
    if (P->verbose)
        fprintf(stderr, "[sg] strip-solve graph: launches pre %lld outer %lld need_r %lld mr %lld inner %lld\n",
                (long long)rl.pre, (long long)rl.outer, (long long)rl.need_r, (long long)rl.mr, (long long)rl.inner);
    return SG_OK;
}

// launches executed by the graph since the counters were last folded into P->launches
static void fold_graph_launches(sg_problem* P, const sg_problem::SolveGraph& sgp, const SolveCtl& before,
                                const SolveCtl& after, int64_t nsolves) {
    P->launches += nsolves * sgp.l_pre + (after.outer_iters - before.outer_iters) * sgp.l_outer +
                   (after.need_r_runs - before.need_r_runs) * sgp.l_need_r + (after.mr_runs - before.mr_runs) * sgp.l_mr +
                   (after.inner_iters - before.inner_iters) * sgp.l_inner;
}

static int enqueue_strip_solve(sg_problem* P, const SolveArgs& a, sg_problem::SolveGraph** used) {
    *used = nullptr;
    P->in_solve = true;
    int rc;
    if (P->use_graphs) {
        sg_problem::SolveGraph* sgp = nullptr;
        rc = solve_graph(P, a, &sgp);
        if (rc == SG_OK) {
            cudaError_t e = cudaGraphLaunch(sgp->exec, P->stream);
            if (e != cudaSuccess) {
                set_error(std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
                rc = SG_ERR_CUDA;
            }
            *used = sgp;
        }
    } else {
        Conds cd;
        std::memset(&cd, 0, sizeof(cd));
        RegionLaunches rl;
        rc = enqueue_solve(P, false, cd, a, &rl);
    }
    P->in_solve = false;
    return rc;
}

// ------------------------------------------------------------------ public
int solver_init(sg_problem* P) {
    SG_CUDA(cudaMalloc(&P->ctl, sizeof(SolveCtl)));
    SG_CUDA(cudaMemset(P->ctl, 0, sizeof(SolveCtl)));
    SG_CUDA(cudaMallocHost(&P->hctl, sizeof(SolveCtl)));
    std::memset(P->hctl, 0, sizeof(SolveCtl));
    // Concurrent per-grid applies when the configuration is launch-latency bound (every grid
    // small) and the private intermediates fit: d = 1 only, whose pass kernels read no
    // per-level constant-bank tables (the TMA / whole-x kernels of d >= 2 stage theirs in the
    // module's constant bank and must stay serialised on one stream).
    std::vector<const Grid*> gr;
    for (auto& g : P->active) gr.push_back(&g);
    for (auto& g : P->coarse) gr.push_back(&g);
    size_t tot = 0, gmax = 0;
    const size_t nb = std::max<size_t>(P->vorder.size(), 1);
    for (auto* g : gr) {
        const size_t w = nb * P->S * (size_t)g->n1 * (size_t)(g->n2 + (g->n2 & 1));
        tot += w;
        gmax = std::max<size_t>(gmax, (size_t)g->n1 * g->n2);
    }
    P->par_applies = P->fx.d == 1 && P->fv.d == 1 && getenv("SG_SERIAL_APPLIES") == nullptr &&
                     gmax <= ((size_t)1 << 20) && tot * sizeof(double) <= ((size_t)1 << 30);
    if (P->par_applies) {
        SG_CUDA(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
        for (auto* g : gr) {
            cudaStream_t s;
            cudaEvent_t e;
            double* w;
            const size_t n = nb * P->S * (size_t)g->n1 * (size_t)(g->n2 + (g->n2 & 1));
            SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            SG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            SG_CUDA(cudaMalloc(&w, sizeof(double) * n));
            SG_CUDA(cudaMemset(w, 0, sizeof(double) * n));
            P->par_streams.push_back(s);
            P->ev_join.push_back(e);
            P->par_ws.push_back(w);
            P->par_ws_n.push_back(n);
        }
    }
    return SG_OK;
}

int solver_destroy(sg_problem* P) {
    for (auto& s : P->solve_graphs) cudaGraphExecDestroy(s.exec);
    P->solve_graphs.clear();
    for (auto s : P->cap_streams) cudaStreamDestroy(s);
    P->cap_streams.clear();
    for (auto s : P->par_streams) cudaStreamDestroy(s);
    for (auto e : P->ev_join) cudaEventDestroy(e);
    for (auto w : P->par_ws) cudaFree(w);
    if (P->ev_fork) cudaEventDestroy(P->ev_fork);
    P->par_streams.clear();
    P->ev_join.clear();
    P->par_ws.clear();
    cudaFree(P->ctl);
    if (P->hctl) cudaFreeHost(P->hctl);
    P->ctl = nullptr;
    P->hctl = nullptr;
    return SG_OK;
}

// copy the device counters to P->hctl (synchronises the stream)
int sync_stats(sg_problem* P) {
    if (!P->ctl) return SG_OK;
    SG_CUDA(cudaMemcpyAsync(P->hctl, P->ctl, sizeof(SolveCtl), cudaMemcpyDeviceToHost, P->stream));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    return SG_OK;
}

int reset_device_stats(sg_problem* P) {
    if (!P->ctl) return SG_OK;
    SG_TRY(sync_stats(P));
    SolveCtl z = *P->hctl;
    z.outer_iters = z.inner_iters = z.need_r_runs = z.mr_runs = z.mr_switches = 0;
    z.inner_breakdowns = z.inner_maxit = z.outer_unconverged = z.outer_nonfinite = 0;
    z.n_applies = z.timed_applies = 0;
    z.dof_applied = z.alg_bytes = z.alg_flops = z.apply_ns = 0.0;
    SG_CUDA(cudaMemcpyAsync(P->ctl, &z, sizeof(SolveCtl), cudaMemcpyHostToDevice, P->stream));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    *P->hctl = z;
    return SG_OK;
}

// Richardson strip solve; one synchronisation at the end (iteration count, last norm, status)
int solve_strip(sg_problem* P, const double* b, double* u, double rtol, double inner_rtol, int max_iter, int* iters,
                double* last) {
    SG_TRY(sync_stats(P));
    const SolveCtl before = *P->hctl;
    SolveArgs a{b, u, rtol, inner_rtol, max_iter};
    sg_problem::SolveGraph* used = nullptr;
    SG_TRY(enqueue_strip_solve(P, a, &used));
    SG_TRY(sync_stats(P));
    const SolveCtl& after = *P->hctl;
    if (used) fold_graph_launches(P, *used, before, after, 1);
    if (iters) *iters = after.it;
    if (last) *last = after.nd;
    if (P->verbose)
        fprintf(stderr, "[sg] strip solve: %d outer its, |du| %.3e, |u|^2 %.3e, done %d, inner its %lld\n", after.it,
                after.nd, after.nu2, after.done, (long long)(after.inner_iters - before.inner_iters));
    if (after.done == 3) {
        set_error("solve_strip: non-finite update (inner solver breakdown)");
        return SG_ERR_STATE;
    }
    if (after.done == 2) {
        set_error("solve_strip: no convergence within max_iter (solution returned)");
        return SG_ERR_NOCONV;
    }
    return SG_OK;
}

// nsteps strips; the strips are enqueued back to back (no host synchronisation between them)
// and the counters are read once at the end
int step(sg_problem* P, int j0, int nsteps, double* trace_dev, double rtol, double inner_rtol) {
    const int S = P->S;
    const int64_t Na = set_size(P, SG_SET_ACTIVE, S);
    double* b = P->vec[11];
    double* u = P->vec[12];
    SG_TRY(sync_stats(P));
    const SolveCtl before = *P->hctl;
    sg_problem::SolveGraph* used = nullptr;
    for (int j = j0; j < j0 + nsteps; ++j) {
        SG_TRY(rhs(P, j, trace_dev, b));
        SG_TRY(launch_zero(P, Na, u));
        SolveArgs a{b, u, rtol, inner_rtol, 200};
        SG_TRY(enqueue_strip_solve(P, a, &used));
        SG_TRY(trace_of(P, u, trace_dev));
    }
    SG_TRY(sync_stats(P));
    const SolveCtl& after = *P->hctl;
    if (used) fold_graph_launches(P, *used, before, after, nsteps);
    if (after.outer_nonfinite > before.outer_nonfinite) {
        set_error("step: non-finite update in a strip solve");
        return SG_ERR_STATE;
    }
    if (after.outer_unconverged > before.outer_unconverged) {
        set_error("step: a strip solve did not converge within max_iter (solution returned)");
        return SG_ERR_NOCONV;
    }
    return SG_OK;
}

}  // namespace sg
