// Pass 2 of the strip-operator apply on box x-lattices ("x fan-in", line-swept):
//
//   Y[i][a] = beta*Y[i][a] + sum_g sum_k C_g^{cls(i)}[k] Z_g[i + off_k][a]
//
// (PAPER.md l.462-477 / l.516-532: the x-factor of every Kronecker term, applied
// after the v-factor; C_g = sum_{t in g} T_t A_t is the time-combined x matrix of
// v-group g, translation invariant on the lattice up to the boundary class of
// the row, cls = per axis {low face, interior, high face}).
//
// Work decomposition.  An x-lattice "line" is the set of rows with fixed
// (i1, i2) (axis 0 fastest).  One warp owns a block of target lines (2x2 lines
// for d = 3, 4 lines for d = 2) and 32*CPT v-columns (lane = column, coalesced),
// and sweeps the line position i0 = t from 0 to m-1.  At every t it loads, for
// every group g, the source points (line s, t) of the 14 (d = 3) / 6 (d = 2)
// lines that neighbour the block exactly once and scatters them into a rolling
// window of accumulators for the target positions t-1, t, t+1 (registers).
// Each Z value is therefore read once per line block (3.5 / 1.5 loads per
// output and group instead of W), and the Kuhn stencil becomes 60 / 28
// register FMAs per source step.
//
// Coefficients.  Away from the lattice boundary (all targets interior) the
// class is the interior one and the coefficients are compile-time indexed
// kernel parameters (constant-bank operands of DFMA, no loads); near the
// boundary they are read from the class table tab[cls][g][k] with warp-uniform
// addresses (broadcast), and the boundary-only (face) groups are included.
#include <array>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sg_internal.cuh"
#include "vmom.cuh"

namespace sg {
namespace xfi {

// Kuhn offsets (d0, d1, d2) in the sorted order of StencilOff (lexicographic
// value d0 + m d1 + m^2 d2, m >= 3)
__host__ __device__ constexpr int d0_3(int k) {
    return k == 0 ? -1 : k == 1 ? 0 : k == 2 ? -1 : k == 3 ? 0 : k == 4 ? -1 : k == 5 ? 0 : k == 6 ? -1 : k == 7 ? 0
         : k == 8 ? 1 : k == 9 ? 0 : k == 10 ? 1 : k == 11 ? 0 : k == 12 ? 1 : k == 13 ? 0 : 1;
}
__host__ __device__ constexpr int d1_3(int k) {
    return k == 0 ? -1 : k == 1 ? -1 : k == 2 ? 0 : k == 3 ? 0 : k == 4 ? -1 : k == 5 ? -1 : k == 6 ? 0 : k == 7 ? 0
         : k == 8 ? 0 : k == 9 ? 1 : k == 10 ? 1 : k == 11 ? 0 : k == 12 ? 0 : k == 13 ? 1 : 1;
}
__host__ __device__ constexpr int d2_3(int k) { return k < 4 ? -1 : (k < 11 ? 0 : 1); }
__host__ __device__ constexpr int d0_2(int k) {
    return k == 0 ? -1 : k == 1 ? 0 : k == 2 ? -1 : k == 3 ? 0 : k == 4 ? 1 : k == 5 ? 0 : 1;
}
__host__ __device__ constexpr int d1_2(int k) { return k < 2 ? -1 : (k < 5 ? 0 : 1); }

template <int D> struct Geo;
template <> struct Geo<3> {
    static constexpr int W = 15, NT = 4, NE1 = 4, NE2 = 4;   // 2x2 target lines, sources e in [-1,2]^2
    static constexpr int B1 = 2, B2 = 2;
    __host__ __device__ static constexpr int u1(int u) { return u & 1; }
    __host__ __device__ static constexpr int u2(int u) { return u >> 1; }
    __host__ __device__ static constexpr int d0(int k) { return d0_3(k); }
    __host__ __device__ static constexpr int d1(int k) { return d1_3(k); }
    __host__ __device__ static constexpr int d2(int k) { return d2_3(k); }
};
template <> struct Geo<2> {
    static constexpr int W = 7, NT = 4, NE1 = 6, NE2 = 1;    // 4 target lines, sources e1 in [-1,4]
    static constexpr int B1 = 4, B2 = 1;
    __host__ __device__ static constexpr int u1(int u) { return u; }
    __host__ __device__ static constexpr int u2(int) { return 0; }
    __host__ __device__ static constexpr int d0(int k) { return d0_2(k); }
    __host__ __device__ static constexpr int d1(int k) { return d1_2(k); }
    __host__ __device__ static constexpr int d2(int) { return 0; }
};

template <int D>
__host__ __device__ constexpr bool pair_ok(int s, int u, int k) {
    using G = Geo<D>;
    return (s % G::NE1) - 1 == G::u1(u) + G::d1(k) && (s / G::NE1) - (D == 3 ? 1 : 0) == G::u2(u) + G::d2(k);
}
template <int D>
__host__ __device__ constexpr bool src_used(int s) {
    for (int u = 0; u < Geo<D>::NT; ++u)
        for (int k = 0; k < Geo<D>::W; ++k)
            if (pair_ok<D>(s, u, k)) return true;
    return false;
}

}  // namespace xfi

constexpr int XFI_MAXG = 12;
struct XfiCoef {
    double c[XFI_MAXG][15];   // interior-class coefficients of the interior groups
};

template <int D, int NGI, int CPT>
__global__ void __launch_bounds__(256, CPT == 1 ? 2 : 1)
    k_xfanin(const double* __restrict__ Z, long long gstride, int nga, int n2, int m, int nlb1, int nlb, int nseg,
             int seglen, int nsub, int ntask, const double* __restrict__ tab, const __grid_constant__ XfiCoef cint,
             double* __restrict__ Y, double beta, const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    using G = xfi::Geo<D>;
    constexpr int W = G::W, NT = G::NT, NS = G::NE1 * G::NE2;
    const int lane = threadIdx.x & 31;
    // tasks = (line block, segment of the line sweep, column tile); a warp runs nsub
    // tasks side by side when the v factor has fewer than 32 columns
    int sub = 0, cl = lane;
    if (nsub > 1) {
        sub = lane / n2;
        cl = lane - sub * n2;
        if (sub >= nsub) return;
    }
    const int task = (blockIdx.x * 8 + (threadIdx.x >> 5)) * nsub + sub;
    if (task >= ntask) return;
    const int lb = task % nlb, rest = task / nlb;
    const int seg = rest % nseg, ct = rest / nseg;
    const int t0 = seg * seglen, t1 = min(m, t0 + seglen);
    // target line block origin
    const int b1 = (lb % nlb1) * G::B1, b2 = (lb / nlb1) * G::B2;
    int col[CPT];
    bool cval[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        col[c] = ct * 32 * CPT + c * 32 + cl;
        cval[c] = col[c] < n2;
        if (!cval[c]) col[c] = n2 - 1;
    }
    // source line bases (element index of (t = 0, line s, column col[0])); clamped lines
    // only ever meet zero coefficients (absent neighbours of boundary rows)
    int sbase[NS];
    bool lines_interior = true;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        int e1 = b1 + (s % G::NE1) - 1;
        int e2 = D == 3 ? b2 + (s / G::NE1) - 1 : 0;
        e1 = e1 < 0 ? 0 : (e1 >= m ? m - 1 : e1);
        e2 = e2 < 0 ? 0 : (e2 >= m ? m - 1 : e2);
        const int line = D == 3 ? e1 + m * e2 : e1;
        sbase[s] = line * m * n2 + col[0];
    }
    // target lines
    int tline[NT];
    bool tval[NT];
    int tcls12[NT];   // class contribution of axes 1, 2
#pragma unroll
    for (int u = 0; u < NT; ++u) {
        const int z1 = b1 + G::u1(u), z2 = D == 3 ? b2 + G::u2(u) : 0;
        tval[u] = z1 < m && z2 < m;
        tline[u] = D == 3 ? z1 + m * z2 : z1;
        const int c1 = z1 == 0 ? 0 : (z1 >= m - 1 ? 2 : 1);
        const int c2 = z2 == 0 ? 0 : (z2 >= m - 1 ? 2 : 1);
        tcls12[u] = 3 * c1 + (D == 3 ? 9 * c2 : 0);
        lines_interior &= tval[u] && c1 == 1 && (D == 2 || c2 == 1);
    }
    double acc[NT][3][CPT];
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int w = 0; w < 3; ++w)
#pragma unroll
            for (int c = 0; c < CPT; ++c) acc[u][w][c] = 0.0;

    auto flush = [&](int p) {   // target position p complete in window slot 0
#pragma unroll
        for (int u = 0; u < NT; ++u) {
            if (!tval[u]) continue;
            double* yr = Y + ((long long)p + (long long)m * tline[u]) * n2;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                if (!cval[c]) continue;
                double* y = yr + col[c];
                *y = beta == 0.0 ? acc[u][0][c] : fma(beta, *y, acc[u][0][c]);
            }
        }
    };

    const int ts = max(t0 - 1, 0), te = min(t1, m - 1);   // sources of the targets [t0, t1)
    for (int t = ts; t <= te; ++t) {
        const long long toff = (long long)t * n2;
        if (lines_interior && t >= 2 && t <= m - 3) {
            // ---- interior: constant coefficients from the kernel parameters
#pragma unroll
            for (int g = 0; g < NGI; ++g) {
                const double* Zg = Z + g * gstride + toff;
                double src[NS][CPT];
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    if (xfi::src_used<D>(s))
#pragma unroll
                        for (int c = 0; c < CPT; ++c) src[s][c] = __ldg(Zg + sbase[s] + 32 * c);
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int u = 0; u < NT; ++u)
#pragma unroll
                        for (int k = 0; k < W; ++k)
                            if (xfi::pair_ok<D>(s, u, k)) {
                                const double cf = cint.c[g][k];
                                const int slot = 1 - G::d0(k);
#pragma unroll
                                for (int c = 0; c < CPT; ++c) acc[u][slot][c] = fma(cf, src[s][c], acc[u][slot][c]);
                            }
            }
        } else {
            // ---- boundary: class-table coefficients, all groups (incl. face groups)
            int cb[NT][3];
#pragma unroll
            for (int u = 0; u < NT; ++u)
#pragma unroll
                for (int w = 0; w < 3; ++w) {
                    const int p = t + w - 1;
                    const int c0 = p <= 0 ? 0 : (p >= m - 1 ? 2 : 1);
                    cb[u][w] = (c0 + tcls12[u]) * nga * W;
                }
            for (int g = 0; g < nga; ++g) {
                const double* Zg = Z + g * gstride + toff;
                const double* tg = tab + g * W;
                double src[NS][CPT];
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    if (xfi::src_used<D>(s))
#pragma unroll
                        for (int c = 0; c < CPT; ++c) src[s][c] = __ldg(Zg + sbase[s] + 32 * c);
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int u = 0; u < NT; ++u)
#pragma unroll
                        for (int k = 0; k < W; ++k)
                            if (xfi::pair_ok<D>(s, u, k)) {
                                const int slot = 1 - G::d0(k);
                                const double cf = __ldg(tg + cb[u][slot] + k);
#pragma unroll
                                for (int c = 0; c < CPT; ++c) acc[u][slot][c] = fma(cf, src[s][c], acc[u][slot][c]);
                            }
            }
        }
        if (t - 1 >= t0) flush(t - 1);
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                acc[u][0][c] = acc[u][1][c];
                acc[u][1][c] = acc[u][2][c];
                acc[u][2][c] = 0.0;
            }
    }
    if (t1 == m) flush(m - 1);
}

int prepare_xwhole(sg_problem* P);

// per-row mask of the boundary-only (face) groups from the row's boundary class
struct ClsMask {
    unsigned char m[27];
};
__global__ void k_bmask(int n, int d, int m, ClsMask cm, uint8_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int z = i, c = 0, mul = 1;
    for (int q = 0; q < d; ++q) {
        const int zq = z % m;
        z /= m;
        c += mul * (zq == 0 ? 0 : (zq == m - 1 ? 2 : 1));
        mul *= 3;
    }
    out[i] = cm.m[c];
}

// host: class tables of the combined x matrices of every v-group (vorder) per x-level
int prepare_xfanin(sg_problem* P) {
    P->xfi_tab.assign(P->F + 1, nullptr);
    P->xfi_itab.assign(P->F + 1, nullptr);
    P->xfi_cint.assign(P->F + 1, {});
    P->xfi_cmask.assign(P->F + 1, {});
    if (P->fx.kind != SG_MESH_BOX || P->S != 1 || P->fx.d < 2 ) return SG_OK;
    const int nga = (int)P->vorder.size();
    if (P->ng_int > XFI_MAXG) return SG_OK;
    const int d = P->fx.d, W = P->fx.W;
    int ncls = 1, icls = 0, mul = 1;
    for (int q = 0; q < d; ++q) {
        icls += mul;
        mul *= 3;
        ncls *= 3;
    }
    for (int l = 1; l <= P->F; ++l) {
        std::vector<double> h((size_t)ncls * nga * W, 0.0);
        bool ok = true;
        for (int o = 0; o < nga && ok; ++o) {
            const Group& gr = P->vgroups[P->vorder[o]];
            if (gr.comb[l].size() != 1 || !gr.comb[l][0].ctab) {
                ok = false;
                break;
            }
            std::vector<double> t27(27 * W);
            SG_CUDA(cudaMemcpy(t27.data(), gr.comb[l][0].ctab, sizeof(double) * 27 * W, cudaMemcpyDeviceToHost));
            for (int c = 0; c < ncls; ++c)
                for (int k = 0; k < W; ++k) h[((size_t)c * nga + o) * W + k] = t27[c * W + k];
        }
        if (!ok) continue;
        double* dt;
        SG_CUDA(cudaMalloc(&dt, sizeof(double) * h.size()));
        SG_CUDA(cudaMemcpy(dt, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
        P->xfi_tab[l] = dt;
        {
            std::vector<double> hi((size_t)ncls * P->ng_int * W);
            for (int c = 0; c < ncls; ++c)
                for (int o = 0; o < P->ng_int; ++o)
                    for (int k = 0; k < W; ++k)
                        hi[((size_t)c * P->ng_int + o) * W + k] = h[((size_t)c * nga + o) * W + k];
            SG_CUDA(cudaMalloc(&P->xfi_itab[l], sizeof(double) * std::max<size_t>(hi.size(), 1)));
            SG_CUDA(cudaMemcpy(P->xfi_itab[l], hi.data(), sizeof(double) * hi.size(), cudaMemcpyHostToDevice));
        }
        std::vector<double> ci((size_t)XFI_MAXG * 15, 0.0);
        for (int o = 0; o < P->ng_int; ++o)
            for (int k = 0; k < W; ++k) ci[o * 15 + k] = h[((size_t)icls * nga + o) * W + k];
        P->xfi_cint[l] = ci;
        // boundary-only groups per boundary class: group j is "present" in class c when a node of that
        // class has a nonzero coefficient in its row or is the source of one (enumerated on a small
        // lattice with the same class structure)
        const int nbo = nga - P->ng_int;
        const int m = P->fx.lev[l].m;
        if (nbo >= 0 && nbo <= 8 && m >= 3 && P->fx.lev[l].n < (1LL << 31)) {
            std::vector<uint8_t> cm(27, 0);
            const int mq = std::min(m, 5);
            auto cls_of = [&](const int* z) {
                int c = 0, mu = 1;
                for (int q = 0; q < d; ++q) {
                    c += mu * (z[q] == 0 ? 0 : (z[q] == mq - 1 ? 2 : 1));
                    mu *= 3;
                }
                return c;
            };
            int tot = 1;
            for (int q = 0; q < d; ++q) tot *= mq;
            for (int i = 0; i < tot; ++i) {
                int z[3] = {i % mq, (i / mq) % mq, d == 3 ? i / (mq * mq) : 0};
                const int c = cls_of(z);
                for (int o = P->ng_int; o < nga; ++o)
                    for (int k = 0; k < W; ++k) {
                        if (h[((size_t)c * nga + o) * W + k] == 0.0) continue;
                        const int dk[3] = {d == 3 ? xfi::d0_3(k) : xfi::d0_2(k), d == 3 ? xfi::d1_3(k) : xfi::d1_2(k),
                                           d == 3 ? xfi::d2_3(k) : 0};
                        int zn[3] = {z[0] + dk[0], z[1] + dk[1], z[2] + dk[2]};
                        bool in = true;
                        for (int q = 0; q < d; ++q) in &= zn[q] >= 0 && zn[q] < mq;
                        cm[c] |= (uint8_t)(1u << (o - P->ng_int));
                        if (in) cm[cls_of(zn)] |= (uint8_t)(1u << (o - P->ng_int));
                    }
            }
            P->xfi_cmask[l] = cm;
            Level& Lx = P->fx.lev[l];
            ClsMask cmk;
            std::memcpy(cmk.m, cm.data(), 27);
            SG_CUDA(cudaMalloc(&Lx.bmask, Lx.n));
            k_bmask<<<(unsigned)((Lx.n + 255) / 256), 256, 0, P->stream>>>((int)Lx.n, d, m, cmk, Lx.bmask);
            P->launches++;
            SG_CUDA(cudaGetLastError());
        }
    }
    SG_TRY(prepare_xwhole(P));
    return SG_OK;
}

// Y = beta*Y + sum_g C_g Z_g over the v-groups of the diagonal apply of grid g;
// SG_ERR_UNSUPPORTED when the line-swept kernel does not cover this shape.
int launch_xfanin(sg_problem* P, int l1, int64_t n1, int64_t n2, const double* Z, int64_t gstride, double* Y,
                  double beta) {
    if (l1 >= (int)P->xfi_tab.size() || !P->xfi_tab[l1]) return SG_ERR_UNSUPPORTED;
    const int d = P->fx.d, m = P->fx.lev[l1].m;
    const int nga = (int)P->vorder.size(), ngi = P->ng_int;
    if (m < 3 || n1 * n2 >= (1LL << 31)) return SG_ERR_UNSUPPORTED;
    constexpr int cpt = 1;   // (2 columns per lane measured slower in round 1)
    const int nct = (int)((n2 + 32 * cpt - 1) / (32 * cpt));
    const int nsub = n2 <= 16 ? (int)(32 / n2) : 1;
    int nlb1, nlb;
    if (d == 3) {
        nlb1 = (m + 1) / 2;
        nlb = nlb1 * nlb1;
    } else {
        nlb1 = (m + 3) / 4;
        nlb = nlb1;
    }
    // split the line sweep into segments until the machine has >= 16 warps per SM of work
    int seglen = m;
    while (seglen > 16 && (long long)nlb * nct * ((m + seglen - 1) / seglen) < 148LL * 16 * nsub)
        seglen = (seglen + 1) / 2;
    const int nseg = (m + seglen - 1) / seglen;
    const long long ntask = (long long)nlb * nseg * nct;
    const long long warps = (ntask + nsub - 1) / nsub;
    const long long blocks = (warps + 7) / 8;
    if (ntask >= (1LL << 31)) return SG_ERR_UNSUPPORTED;
    XfiCoef ci;
    std::memcpy(ci.c, P->xfi_cint[l1].data(), sizeof(ci.c));
    const double* tab = P->xfi_tab[l1];
#define XFI(DD, NG, CC)                                                                                           \
    k_xfanin<DD, NG, CC><<<(unsigned)blocks, 256, 0, P->stream>>>(Z, (long long)gstride, nga, (int)n2, m, nlb1, nlb, \
                                                                  nseg, seglen, nsub, (int)ntask, tab, ci, Y, beta, P->skip)
#define XFI_C(DD, NG) XFI(DD, NG, 1)
    if (d == 3 && ngi == 10) XFI_C(3, 10);
    else if (d == 2 && ngi == 6) XFI_C(2, 6);
    else if (d == 3 && ngi == 6) XFI_C(3, 6);
    else if (d == 2 && ngi == 10) XFI_C(2, 10);
    else if (d == 2 && ngi == 3) XFI_C(2, 3);
    else if (d == 3 && ngi == 4) XFI_C(3, 4);
    else return SG_ERR_UNSUPPORTED;
#undef XFI_C
#undef XFI
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

}  // namespace sg

namespace sg {
// =====================================================================
// Whole-x pass 2 for tiny x lattices (m^d <= 27 rows: the level-1 grids):
// every thread owns one v-column and ALL x-rows in registers; every row has
// its own boundary class, so the coefficient of (group g, row r, offset k) is
// c_xw[g][r][k] with (r, k) compile-time and g warp-uniform (uniform constant
// loads, no L1 traffic), and absent neighbours are dropped at compile time.
// =====================================================================
constexpr int XW_MAXG = 16, XW_MAXN = 27;
constexpr int XW_MAXP = 223;   // valid (row, offset) pairs of the 3^3 lattice (3^2: 41, 5^2: 137)

namespace xw {
template <int D> __host__ __device__ constexpr int kd(int k, int ax) {
    return D == 3 ? (ax == 0 ? xfi::d0_3(k) : ax == 1 ? xfi::d1_3(k) : xfi::d2_3(k))
                  : (ax == 0 ? xfi::d0_2(k) : ax == 1 ? xfi::d1_2(k) : 0);
}
template <int D, int M> __host__ __device__ constexpr int nbr(int r, int k) {   // neighbour row or -1
    int z0 = r % M, z1 = (r / M) % M, z2 = D == 3 ? r / (M * M) : 0;
    z0 += kd<D>(k, 0);
    z1 += kd<D>(k, 1);
    z2 += kd<D>(k, 2);
    if (z0 < 0 || z0 >= M || z1 < 0 || z1 >= M || (D == 3 && (z2 < 0 || z2 >= M))) return -1;
    return z0 + M * (z1 + M * z2);
}
template <int D, int M> __host__ __device__ constexpr int pidx(int r, int k) {   // compact pair index
    constexpr int W = D == 3 ? 15 : 7;
    int c = 0;
    for (int rr = 0; rr < r; ++rr)
        for (int kk = 0; kk < W; ++kk) c += nbr<D, M>(rr, kk) >= 0;
    for (int kk = 0; kk < k; ++kk) c += nbr<D, M>(r, kk) >= 0;
    return c;
}
template <int D, int M> __host__ __device__ constexpr int npairs() {
    return pidx<D, M>(D == 3 ? M * M * M : M * M, 0);
}
}  // namespace xw

__constant__ double c_xw[XW_MAXG * XW_MAXP];   // [g][pair] of the launched level (compact)

template <int D, int M>
__global__ void __launch_bounds__(256, 2) k_xwhole(const double* __restrict__ Z, long long gstride, int nga, int n2,
                                                   long long pitch, double* __restrict__ Y, const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    constexpr int N = D == 3 ? M * M * M : M * M;
    constexpr int W = D == 3 ? 15 : 7;
    constexpr int NP = D == 3 ? (M == 3 ? 223 : 0) : (M == 3 ? 41 : 137);   // xw::npairs<D, M>()
    const int col = blockIdx.x * 256 + threadIdx.x;
    if (col >= n2) return;
    double acc[N];
#pragma unroll
    for (int r = 0; r < N; ++r) acc[r] = 0.0;
    for (int g = 0; g < nga; ++g) {
        const double* Zg = Z + g * gstride + col;
        double z[N];
#pragma unroll
        for (int r = 0; r < N; ++r) z[r] = __ldg(Zg + r * pitch);
        const double* cg = c_xw + g * NP;
        int pi = 0;   // compact pair index (a compile-time constant after unrolling)
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (xw::nbr<D, M>(r, k) >= 0) {
                    acc[r] = fma(cg[pi], z[xw::nbr<D, M>(r, k)], acc[r]);
                    ++pi;
                }
    }
#pragma unroll
    for (int r = 0; r < N; ++r) Y[(long long)r * n2 + col] = acc[r];
}

// [g][r][k] coefficient tables of the tiny x-levels (setup time: never allocate inside a capture)
int prepare_xwhole(sg_problem* P) {
    P->xw_tab.assign(P->F + 1, nullptr);
    P->xw_dev.assign(P->F + 1, nullptr);
    P->xw_np.assign(P->F + 1, 0);
    const int d = P->fx.d, W = P->fx.W;
    const int nga = (int)P->vorder.size();
    if (nga > XW_MAXG) return SG_OK;
    for (int l1 = 1; l1 <= P->F && l1 < (int)P->xfi_tab.size(); ++l1) {
        if (!P->xfi_tab[l1]) continue;
        const int m = P->fx.lev[l1].m;
        const int64_t n1 = P->fx.lev[l1].n;
        const bool ok = (d == 3 && m == 3) || (d == 2 && (m == 3 || m == 5));
        if (!ok || n1 > XW_MAXN) continue;
        int ncls = 1;
        for (int q = 0; q < d; ++q) ncls *= 3;
        std::vector<double> cls((size_t)ncls * nga * W), h((size_t)nga * n1 * W, 0.0);
        SG_CUDA(cudaMemcpy(cls.data(), P->xfi_tab[l1], sizeof(double) * cls.size(), cudaMemcpyDeviceToHost));
        for (int r = 0; r < n1; ++r) {
            int z = r, c = 0, mul = 1;
            for (int q = 0; q < d; ++q) {
                const int zq = z % m;
                z /= m;
                c += mul * (zq == 0 ? 0 : (zq == m - 1 ? 2 : 1));
                mul *= 3;
            }
            for (int g = 0; g < nga; ++g)
                for (int k = 0; k < W; ++k) h[((size_t)g * n1 + r) * W + k] = cls[((size_t)c * nga + g) * W + k];
        }
        // compact [g][pair] for the kernel parameters
        std::vector<double> cmp((size_t)XW_MAXG * XW_MAXP, 0.0);
        int np = 0;
        for (int r = 0; r < n1; ++r)
            for (int k = 0; k < W; ++k) {
                int z = r, zz[3] = {0, 0, 0};
                for (int q = 0; q < d; ++q) {
                    zz[q] = z % m;
                    z /= m;
                }
                bool ok2 = true;
                for (int q = 0; q < d; ++q) {
                    const int dq = d == 3 ? (q == 0 ? xfi::d0_3(k) : q == 1 ? xfi::d1_3(k) : xfi::d2_3(k))
                                          : (q == 0 ? xfi::d0_2(k) : xfi::d1_2(k));
                    ok2 &= zz[q] + dq >= 0 && zz[q] + dq < m;
                }
                if (!ok2) continue;
                ++np;
            }
        int pi = 0;
        for (int r = 0; r < n1; ++r)
            for (int k = 0; k < W; ++k) {
                int z = r, zz[3] = {0, 0, 0};
                for (int q = 0; q < d; ++q) {
                    zz[q] = z % m;
                    z /= m;
                }
                bool ok2 = true;
                for (int q = 0; q < d; ++q) {
                    const int dq = d == 3 ? (q == 0 ? xfi::d0_3(k) : q == 1 ? xfi::d1_3(k) : xfi::d2_3(k))
                                          : (q == 0 ? xfi::d0_2(k) : xfi::d1_2(k));
                    ok2 &= zz[q] + dq >= 0 && zz[q] + dq < m;
                }
                if (!ok2) continue;
                for (int g = 0; g < nga; ++g) cmp[(size_t)g * np + pi] = h[((size_t)g * n1 + r) * W + k];
                ++pi;
            }
        if (np > XW_MAXP) continue;
        P->xw_np[l1] = np;
        SG_CUDA(cudaMalloc(&P->xw_dev[l1], sizeof(double) * (size_t)nga * np));
        for (int g = 0; g < nga; ++g)
            SG_CUDA(cudaMemcpy(P->xw_dev[l1] + (size_t)g * np, cmp.data() + (size_t)g * np, sizeof(double) * np,
                               cudaMemcpyHostToDevice));
        P->xw_tab[l1] = P->xw_dev[l1];
    }
    return SG_OK;
}

int launch_xwhole(sg_problem* P, int l1, int64_t n1, int64_t n2, int64_t pitch, const double* Z, int64_t gstride,
                  double* Y) {
    if (l1 >= (int)P->xfi_tab.size() || !P->xfi_tab[l1]) return SG_ERR_UNSUPPORTED;
    const int d = P->fx.d, m = P->fx.lev[l1].m;
    const int nga = (int)P->vorder.size();
    const bool ok = (d == 3 && m == 3) || (d == 2 && (m == 3 || m == 5));
    if (!ok || nga > XW_MAXG || n1 * n2 >= (1LL << 31) || n1 > XW_MAXN) return SG_ERR_UNSUPPORTED;
    if (l1 >= (int)P->xw_tab.size() || !P->xw_tab[l1]) return SG_ERR_UNSUPPORTED;   // built in prepare_xfanin
    const int np = P->xw_np[l1];
    SG_CUDA(cudaMemcpyToSymbolAsync(c_xw, P->xw_dev[l1], sizeof(double) * nga * np, 0, cudaMemcpyDeviceToDevice,
                                    P->stream));
    const unsigned blocks = (unsigned)((n2 + 255) / 256);
    if (d == 3) {
        if (np != 223) return SG_ERR_UNSUPPORTED;
        k_xwhole<3, 3><<<blocks, 256, 0, P->stream>>>(Z, gstride, nga, (int)n2, pitch, Y, P->skip);
    } else if (m == 3) {
        if (np != 41) return SG_ERR_UNSUPPORTED;
        k_xwhole<2, 3><<<blocks, 256, 0, P->stream>>>(Z, gstride, nga, (int)n2, pitch, Y, P->skip);
    } else {
        if (np != 137) return SG_ERR_UNSUPPORTED;
        k_xwhole<2, 5><<<blocks, 256, 0, P->stream>>>(Z, gstride, nga, (int)n2, pitch, Y, P->skip);
    }
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}
}  // namespace sg

namespace sg {
// =====================================================================
// Fused single-pass strip operator on grids with a tiny x factor (level-1 x-lattice of
// m^d <= 27 rows; d = 2 also m = 5): the two-sided apply
//     Y[r][a] = sum_g sum_k C_g[r, r + off_k] Z_g[r + off_k][a],   Z_g = (Id x B_g) X
// (application order l.516-532) without intermediates in memory.
// One thread owns one v-column a and ALL x-rows: for every source x-row r it loads the W
// v-neighbours X[r][a + off_k] (L1/L2), forms the shifted-moment sums ZR_m (vmoment.cu:
// compile-time kernel-parameter coefficients when the whole warp is interior, the shared-
// memory class table otherwise), combines them into Z_g for every interior monomial group
// and the chi-weighted inflow groups (x-boundary rows only), and scatters Z_g into the
// register accumulators of the x-rows whose stencil contains r.  The x coefficients are
// the per-row class values of the combined matrices C_g in the constant bank, laid out in
// the kernel's visiting order (source row, group, target, offset) so every address is a
// compile-time constant.  X is read once (its v-halo from cache), Y written once.
// =====================================================================
constexpr int FW_NG = VM_NP + VM_NC;
static_assert(FW_NG <= XW_MAXG, "fused whole-x table shares the whole-x constant bank");
#define c_fw c_xw   // [g][pair in (source, target, offset) order]; staged before every launch

namespace fw {
// compile-time pair lists: for source row R the (target, offset) pairs with nbr(target, offset) = R
struct PairList {
    int n;
    int t[15];
};
template <int D, int M>
__host__ __device__ constexpr PairList make_pairs(int R) {
    PairList p{0, {0}};
    constexpr int N = D == 3 ? M * M * M : M * M;
    constexpr int W = D == 3 ? 15 : 7;
    for (int t = 0; t < N; ++t)
        for (int k = 0; k < W; ++k)
            if (xw::nbr<D, M>(t, k) == R) p.t[p.n++] = t;
    return p;
}
template <int D, int M>
__host__ __device__ constexpr int pair_base(int R) {   // pairs of the source rows before R
    int c = 0;
    for (int r = 0; r < R; ++r) c += make_pairs<D, M>(r).n;
    return c;
}
template <int D, int M, int R>
struct Row {
    static constexpr PairList p = make_pairs<D, M>(R);
    static constexpr int base = pair_base<D, M>(R);
    static constexpr bool xbnd = [] {
        int zz = R;
        bool b = false;
        for (int q = 0; q < D; ++q) {
            const int zq = zz % M;
            zz /= M;
            b = b || zq == 0 || zq == M - 1;
        }
        return b;
    }();
};
// acc[t_j] += c[j] * z for the compile-time pairs j of source row R
template <int D, int M, int R, int J>
struct Scatter {
    template <int N>
    __device__ __forceinline__ static void run(double (&acc)[N], const double* c, double z) {
        if constexpr (J < Row<D, M, R>::p.n) {
            constexpr int t = Row<D, M, R>::p.t[J];
            acc[t] = fma(c[J], z, acc[t]);
            Scatter<D, M, R, J + 1>::run(acc, c, z);
        }
    }
};
}  // namespace fw

struct FwCtx {                 // per-thread state of the fused whole-x kernel
    const double* x;           // X + column
    int n2;
    unsigned nbmask;           // bit k: neighbour a + off_k inside the v-lattice
    bool warp_int;             // every column of the warp is interior (d = 2 path)
    const double* ct;          // class row of the moment table (shared memory)
    double y[3];
};

template <int D, int M, int NP, int R>
__device__ __forceinline__ void fw_row(double (&acc)[D == 3 ? M * M * M : M * M], const FwCtx& cx, const VmCoef& cf) {
    constexpr int N = D == 3 ? M * M * M : M * M;
    constexpr int W = D == 3 ? 15 : 7;
    if constexpr (R < N) {
        const double* xr = cx.x + (long long)R * cx.n2;
        // moment sums.  d = 3: class-table row of the column (shared memory, one broadcast address
        // for the interior columns) in a rolled offset loop, which keeps the 27 unrolled source rows
        // small enough for the instruction cache (measured 5.89 -> 5.12 ms on configs[4] grid (1,7));
        // d = 2: fully unrolled, compile-time kernel-parameter coefficients for interior warps
        // (measured faster there: grid (1,11) of configs[2] 1.00 -> 0.81 ms)
        double zr[VM_NP];
#pragma unroll
        for (int n = 0; n < VM_NP; ++n) zr[n] = 0.0;
        if constexpr (D == 3) {
#pragma unroll 5
            for (int k = 0; k < W; ++k) {
                const double xk = (cx.nbmask >> k) & 1u ? __ldg(xr + cf.off[k]) : 0.0;
#pragma unroll
                for (int n = 0; n < VM_NP; ++n)
                    if (vm::mono_in(D, n)) zr[n] = fma(cx.ct[n * W + k], xk, zr[n]);
            }
        } else {
            double xv[W];
#pragma unroll
            for (int k = 0; k < W; ++k) xv[k] = (cx.nbmask >> k) & 1u ? __ldg(xr + cf.off[k]) : 0.0;
            if (cx.warp_int) {
#pragma unroll
                for (int n = 0; n < VM_NP; ++n)
                    if (vm::mono_in(D, n))
#pragma unroll
                        for (int k = 0; k < W; ++k) zr[n] = fma(cf.R[n][k], xv[k], zr[n]);
            } else {
#pragma unroll
                for (int n = 0; n < VM_NP; ++n)
                    if (vm::mono_in(D, n))
#pragma unroll
                        for (int k = 0; k < W; ++k) zr[n] = fma(cx.ct[n * W + k], xv[k], zr[n]);
            }
        }
        constexpr int base = fw::Row<D, M, R>::base;
        const double* y = cx.y;
#pragma unroll
        for (int g = 0; g < VM_NP; ++g) {
            if (!vm::mono_in(D, g)) continue;
            double zg;
            if (g == 0) {
                zg = zr[0];
            } else if (g <= 3) {
                zg = fma(y[g - 1], zr[0], zr[g]);
            } else {
                const int i = vm::mono_ax(g, 0), j = vm::mono_ax(g, 1);
                if (i == j)
                    zg = fma(y[i] * y[i], zr[0], fma(2.0 * y[i], zr[vm::lin(i)], zr[g]));
                else
                    zg = fma(y[i] * y[j], zr[0], fma(y[i], zr[vm::lin(j)], fma(y[j], zr[vm::lin(i)], zr[g])));
            }
            fw::Scatter<D, M, R, 0>::run(acc, c_xw + g * NP + base, zg);
        }
        if constexpr (fw::Row<D, M, R>::xbnd) {   // chi-weighted inflow groups (x-boundary rows)
#pragma unroll 1
            for (int c = 0; c < cf.nchi; ++c) {
                const int i = cf.chax[c];
                const double yi = i == 0 ? y[0] : (i == 1 ? y[1] : y[2]);
                const double zi = i == 0 ? zr[1] : (i == 1 ? zr[2] : zr[3]);
                double zg = cf.chkeep[c] * yi > 0.0 ? fma(yi, zr[0], zi) : 0.0;
                if (yi == 0.0) {   // column on the plane y_i = 0: half stencil (X reloaded, rare)
                    zg = 0.0;
                    const double* hc = cx.ct + (VM_NP + c) * W;
                    for (int k = 0; k < W; ++k)
                        if ((cx.nbmask >> k) & 1u) zg = fma(hc[k], __ldg(xr + cf.off[k]), zg);
                }
                fw::Scatter<D, M, R, 0>::run(acc, c_xw + (VM_NP + c) * NP + base, zg);
            }
        }
        fw_row<D, M, NP, R + 1>(acc, cx, cf);
    }
}

template <int D, int M>
__global__ void __launch_bounds__(128) k_fwhole(const double* __restrict__ X, double* __restrict__ Y, int n2, int mv,
                                                const double* __restrict__ tab, const __grid_constant__ VmCoef cf,
                                                double lo0, double lo1, double lo2, double h0, double h1, double h2,
                                                const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    constexpr int N = D == 3 ? M * M * M : M * M;
    constexpr int W = D == 3 ? 15 : 7;
    constexpr int NP = fw::pair_base<D, M>(N);
    constexpr int NC = D == 3 ? 27 : 9;
    constexpr int NR = VM_NP + VM_NC;
    constexpr int CS = NR * W + 1;
    constexpr int ICLS = D == 3 ? 13 : 4;
    extern __shared__ double st[];   // [NC][CS] moment class table
    for (int i = threadIdx.x; i < NC * NR * W; i += blockDim.x) {
        const int c = i / (NR * W);
        st[c * CS + (i - c * NR * W)] = tab[i];
    }
    __syncthreads();
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = a < n2;
    const int ac = valid ? a : n2 - 1;
    const int z[3] = {ac % mv, (ac / mv) % mv, D == 3 ? ac / (mv * mv) : 0};
    int cls = 0, mul = 1;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        cls += mul * (z[q] == 0 ? 0 : (z[q] == mv - 1 ? 2 : 1));
        mul *= 3;
    }
    FwCtx cx;
    cx.x = X + ac;
    cx.n2 = n2;
    cx.warp_int = __all_sync(0xffffffffu, cls == ICLS);
    cx.ct = st + cls * CS;
    cx.y[0] = lo0 + h0 * z[0];
    cx.y[1] = lo1 + h1 * z[1];
    cx.y[2] = lo2 + h2 * z[2];
    cx.nbmask = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int c = ac + cf.off[k];
        cx.nbmask |= (c >= 0 && c < n2) ? (1u << k) : 0u;   // (absent neighbours have zero coefficients)
    }
    double acc[N];
#pragma unroll
    for (int r = 0; r < N; ++r) acc[r] = 0.0;
    fw_row<D, M, NP, 0>(acc, cx, cf);
    if (!valid) return;
#pragma unroll
    for (int r = 0; r < N; ++r) Y[(long long)r * n2 + a] = acc[r];
}

// [g][pair] tables of the fused whole-x kernel (setup time, after prepare_vmom): group slot
// g < VM_NP is the interior group of monomial g, g >= VM_NP the chi group g - VM_NP (vorder);
// pairs in the kernel's visiting order (source row r, target t, offset k with nbr(t,k) = r).
int prepare_fwhole(sg_problem* P) {
    P->fw_dev.assign(P->F + 1, nullptr);
    const int d = P->fx.d, W = P->fx.W;
    const int nga = (int)P->vorder.size();
    if (P->fx.kind != SG_MESH_BOX || P->fv.kind != SG_MESH_BOX || P->S != 1 || d < 2) return SG_OK;
    if (P->vm_nchi != nga - P->ng_int || P->ng_int > VM_NP) return SG_OK;
    int slot_group[FW_NG];
    for (int g = 0; g < FW_NG; ++g) slot_group[g] = -1;
    for (int o = 0; o < P->ng_int; ++o) {
        if (P->vm_slot[o] < 0) return SG_OK;
        slot_group[P->vm_slot[o]] = o;
    }
    for (int c = 0; c < P->vm_nchi; ++c) slot_group[VM_NP + c] = P->ng_int + c;
    for (int l1 = 1; l1 <= P->F && l1 < (int)P->xfi_tab.size(); ++l1) {
        if (!P->xfi_tab[l1]) continue;
        const int m = P->fx.lev[l1].m;
        const bool ok = (d == 3 && m == 3) || (d == 2 && (m == 3 || m == 5));
        if (!ok) continue;
        const int64_t n1 = P->fx.lev[l1].n;
        int ncls = 1;
        for (int q = 0; q < d; ++q) ncls *= 3;
        std::vector<double> cls((size_t)ncls * nga * W);
        SG_CUDA(cudaMemcpy(cls.data(), P->xfi_tab[l1], sizeof(double) * cls.size(), cudaMemcpyDeviceToHost));
        auto lat = [&](int r, int* zz) {
            for (int q = 0; q < d; ++q) {
                zz[q] = r % m;
                r /= m;
            }
        };
        auto nbr = [&](int t, int k) {
            int zz[3] = {0, 0, 0};
            lat(t, zz);
            int out = 0, mul = 1;
            for (int q = 0; q < d; ++q) {
                const int dq = d == 3 ? (q == 0 ? xfi::d0_3(k) : q == 1 ? xfi::d1_3(k) : xfi::d2_3(k))
                                      : (q == 0 ? xfi::d0_2(k) : xfi::d1_2(k));
                const int v = zz[q] + dq;
                if (v < 0 || v >= m) return -1;
                out += mul * v;
                mul *= m;
            }
            return out;
        };
        std::vector<std::array<int, 2>> pairs;   // (target, offset) in visiting order
        for (int r = 0; r < n1; ++r)
            for (int t = 0; t < n1; ++t)
                for (int k = 0; k < W; ++k)
                    if (nbr(t, k) == r) pairs.push_back({t, k});
        const int np = (int)pairs.size();
        if (np > XW_MAXP) continue;
        std::vector<double> tab((size_t)FW_NG * np, 0.0);
        for (int g = 0; g < FW_NG; ++g) {
            const int o = slot_group[g];
            if (o < 0) continue;
            for (int j = 0; j < np; ++j) {
                const int t = pairs[j][0], k = pairs[j][1];
                int zz[3] = {0, 0, 0};
                lat(t, zz);
                int c = 0, mul = 1;
                for (int q = 0; q < d; ++q) {
                    c += mul * (zz[q] == 0 ? 0 : (zz[q] == m - 1 ? 2 : 1));
                    mul *= 3;
                }
                tab[(size_t)g * np + j] = cls[((size_t)c * nga + o) * W + k];
            }
        }
        SG_CUDA(cudaMalloc(&P->fw_dev[l1], sizeof(double) * tab.size()));
        SG_CUDA(cudaMemcpy(P->fw_dev[l1], tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
        P->fw_np = np;
    }
    return SG_OK;
}

// the whole strip-operator apply of grid (l1, l2) in one fused launch; SG_ERR_UNSUPPORTED if the
// grid is not covered (x-lattice not tiny, moment tables unavailable, S = 2, ...)
int launch_fwhole(sg_problem* P, int l1, int l2, int64_t n2, const double* X, double* Y) {
    if (!P->use_fused || l1 >= (int)P->fw_dev.size() || !P->fw_dev[l1]) return SG_ERR_UNSUPPORTED;
    if (l2 >= (int)P->vm_ok.size() || !P->vm_ok[l2] || !P->vm_tab[l2]) return SG_ERR_UNSUPPORTED;
    const int d = P->fx.d, m = P->fx.lev[l1].m;
    const int n1 = (int)P->fx.lev[l1].n;
    if ((int64_t)n1 * n2 >= (1LL << 31)) return SG_ERR_UNSUPPORTED;
    VmCoef cf;
    double lo[3], h[3];
    vmom_coef(P, l2, &cf, lo, h);
    const int np = d == 3 ? 223 : (m == 3 ? 41 : 137);
    SG_CUDA(cudaMemcpyToSymbolAsync(c_fw, P->fw_dev[l1], sizeof(double) * FW_NG * np, 0, cudaMemcpyDeviceToDevice,
                                    P->stream));
    const int W = P->fv.W;
    const int smb = (d == 3 ? 27 : 9) * ((VM_NP + VM_NC) * W + 1) * (int)sizeof(double);
    const unsigned blocks = (unsigned)((n2 + 127) / 128);
    const int mv = P->fv.lev[l2].m;
#define FWL(DD, MM)                                                                                              \
    do {                                                                                                         \
        cudaFuncSetAttribute(k_fwhole<DD, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);                \
        k_fwhole<DD, MM><<<blocks, 128, smb, P->stream>>>(X, Y, (int)n2, mv, P->vm_tab[l2], cf, lo[0], lo[1],   \
                                                           lo[2], h[0], h[1], h[2], P->skip);                    \
    } while (0)
    if (d == 3 && m == 3) FWL(3, 3);
    else if (d == 2 && m == 3) FWL(2, 3);
    else if (d == 2 && m == 5) FWL(2, 5);
    else return SG_ERR_UNSUPPORTED;
#undef FWL
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

}  // namespace sg
