// Pass 2 of the strip-operator apply on box x-lattices, TMA-pipelined version
// of the line-swept x fan-in (xfanin.cu has the register-only variant and the
// derivation):
//
//   Y[i][a] = sum_g sum_k C_g^{cls(i)}[k] Z_g[i + off_k][a]
//
// A CTA owns a tile of target x-lines (WL1 x WL2 warp blocks of 2x2 lines for
// d = 3, WL1 blocks of 4 lines for d = 2) and 32*WC v-columns, and sweeps the
// line position t.  For every (t, g) one elected producer thread issues ONE
// cp.async.bulk.tensor load of the box
//     Z_g[t][halo lines of the tile][32*WC columns]
// into a ring of shared-memory stages (mbarrier complete_tx); lattice lines
// outside the domain and columns >= n2 arrive as zeros (TMA out-of-bounds fill),
// which only ever meet zero coefficients.  The consumer warps scatter the stage
// into a rolling register window of targets t-1, t, t+1 exactly as the register
// kernel does (interior coefficients as compile-time kernel parameters, class
// tables near the boundary), then release the stage.  Z uses an even row pitch
// (TMA strides must be multiples of 16 bytes).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "sg_internal.cuh"

namespace sg {
namespace xft {
// Kuhn offsets in StencilOff order (same tables as xfanin.cu)
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
    static constexpr int W = 15, NT = 4, NE1 = 4, NE2 = 4, B1 = 2, B2 = 2;
    __host__ __device__ static constexpr int u1(int u) { return u & 1; }
    __host__ __device__ static constexpr int u2(int u) { return u >> 1; }
    __host__ __device__ static constexpr int d0(int k) { return d0_3(k); }
    __host__ __device__ static constexpr int d1(int k) { return d1_3(k); }
    __host__ __device__ static constexpr int d2(int k) { return d2_3(k); }
};
template <> struct Geo<2> {
    static constexpr int W = 7, NT = 4, NE1 = 6, NE2 = 1, B1 = 4, B2 = 1;
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

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}
template <int D>
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2, int c3,
                                         int c4) {
    if (D == 3)
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
            "%6}], [%7];" ::"r"(saddr(dst)),
            "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(saddr(bar))
            : "memory");
    else
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5}], [%6];" ::"r"(saddr(dst)),
            "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(saddr(bar))
            : "memory");
}
}  // namespace xft

constexpr int XFT_MAXG = 12;
// class table [3^d][groups][W] of the launched level in constant memory: the boundary path's
// coefficient loads are warp-uniform and go through the constant cache, not L1
constexpr int XFT_CTAB = 27 * 10 * 15;   // interior groups only (bonly groups read the global table)
__constant__ double c_xft[XFT_CTAB];
struct XftCoef {
    double c[XFT_MAXG][15];
};
struct XftMask {
    int nbo;                   // boundary-only groups (<= 8)
    unsigned char m[27];       // per boundary class: bit j set when boundary-only group j has a nonzero there
};
struct XftTile {
    int wl1, wl2, wc, nw;      // warp blocks per tile (axis 1, axis 2), column groups, consumer warps
    int e1, e2, bc;            // stage box: halo lines (axis 1, axis 2), columns
    int ntl1, ntl2, nct, nseg, seglen;
    int nst;                   // pipeline depth
    int np;                    // producer lanes (each loads 1/np of the stage box along the slowest line axis)
};

// TABM: where the boundary path finds the class coefficients of the interior groups:
//   0 whole class table in shared memory (small lattices), 1 constant bank, 2 per-tile compact
//   table in shared memory ([3 x tile lines][NGI][W]: the classes of the tile's own target lines)
// CPT: v-columns per lane (2: adjacent columns, 128-bit stage loads; every coefficient load feeds 2 multiply-adds)
template <int D, int NGI, int TABM, int CPT = 1>
__global__ void __launch_bounds__(CPT == 2 ? 32 * 9 : 32 * 17, 1)
    k_xfanin_tma(const __grid_constant__ CUtensorMap tmap, int nga, int n2, int m, XftTile tl,
                 const double* __restrict__ tab, const __grid_constant__ XftCoef cint, double* __restrict__ Y, const double* __restrict__ skip,
                 long long ypitch, const __grid_constant__ XftMask cmask) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    using G = xft::Geo<D>;
    constexpr int W = G::W, NT = G::NT, NS = G::NE1 * G::NE2;
    extern __shared__ __align__(128) unsigned char smraw[];
    const int stage_elems = tl.e1 * tl.e2 * tl.bc;
    double* stages = reinterpret_cast<double*>(smraw);
    const int nst = tl.nst;
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw + (size_t)nst * stage_elems * 8);
    uint64_t* empty = full + nst;
    // tiny all-boundary lattices (!CTAB): the class table [3^D][groups][W] lives in shared memory
    // (every coefficient is a warp-uniform broadcast load; the global table cost a 64-bit address
    // computation and an L1 lookup per multiply-add)
    double* stab = reinterpret_cast<double*>(smraw + (size_t)nst * stage_elems * 8 + 2 * (size_t)nst * sizeof(uint64_t));
    constexpr bool CTAB = TABM != 0;
    if (TABM == 0) {
        const int ntab = (D == 3 ? 27 : 9) * nga * G::W;
        for (int i = threadIdx.x; i < ntab; i += blockDim.x) stab[i] = __ldg(tab + i);
    }

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // CTA -> (line tile, segment, column tile)
    int bid = blockIdx.x;
    const int tl1 = bid % tl.ntl1;
    bid /= tl.ntl1;
    const int tl2 = bid % tl.ntl2;
    bid /= tl.ntl2;
    const int seg = bid % tl.nseg;
    const int ct = bid / tl.nseg;
    const int L1 = tl1 * tl.wl1 * G::B1, L2 = tl2 * tl.wl2 * G::B2;   // first target line of the tile
    const int t0 = seg * tl.seglen, t1 = min(m, t0 + tl.seglen);
    const int ts = max(t0 - 1, 0), te = min(t1, m - 1);
    const int TL1 = tl.wl1 * G::B1, TL2 = D == 3 ? tl.wl2 * G::B2 : 1;   // target lines of the tile
    if (TABM == 2) {
        const int ntab = 3 * TL1 * TL2 * NGI * W;
        for (int i = threadIdx.x; i < ntab; i += blockDim.x) {
            const int lc = i / (NGI * W), rem = i - lc * NGI * W, g = rem / W, k = rem - g * W;
            const int c0 = lc % 3, j1 = (lc / 3) % TL1, j2 = lc / (3 * TL1);
            const int z1 = L1 + j1, z2 = L2 + j2;
            const int c1 = z1 == 0 ? 0 : (z1 >= m - 1 ? 2 : 1);
            const int c2 = D == 3 ? (z2 == 0 ? 0 : (z2 >= m - 1 ? 2 : 1)) : 0;
            stab[i] = __ldg(tab + ((c0 + 3 * c1 + 9 * c2) * nga + g) * W + k);
        }
    }
    // CTA-level: are all target lines of the tile interior lines?
    const bool cta_lines_int = L1 >= 1 && L1 + tl.wl1 * G::B1 - 1 <= m - 2 &&
                               (D == 2 || (L2 >= 1 && L2 + tl.wl2 * G::B2 - 1 <= m - 2));

    // boundary-only (face) groups: a stage (t, g) exists only when some target row of the tile in the
    // window t-1..t+1 lies in a boundary class where group g is nonzero (producer and consumers agree)
    unsigned lm[3] = {0u, 0u, 0u};
    {
        unsigned s1 = 0, s2 = D == 3 ? 0u : 1u;   // class sets of the tile's target lines per axis
        for (int i = 0; i < tl.wl1 * G::B1; ++i) {
            const int z = L1 + i;
            if (z < m) s1 |= 1u << (z == 0 ? 0 : (z >= m - 1 ? 2 : 1));
        }
        if (D == 3)
            for (int i = 0; i < tl.wl2 * G::B2; ++i) {
                const int z = L2 + i;
                if (z < m) s2 |= 1u << (z == 0 ? 0 : (z >= m - 1 ? 2 : 1));
            }
        for (int c1 = 0; c1 < 3; ++c1)
            for (int c2 = 0; c2 < (D == 3 ? 3 : 1); ++c2)
                if (((s1 >> c1) & 1u) && ((s2 >> c2) & 1u))
                    for (int c0 = 0; c0 < 3; ++c0) lm[c0] |= cmask.m[c0 + 3 * c1 + 9 * c2];
    }
    auto win_mask = [&](const unsigned (&mm)[3], int t) -> unsigned {
        unsigned r = 0;
#pragma unroll
        for (int w = -1; w <= 1; ++w) {
            const int p = t + w;
            if (p >= 0 && p < m) r |= mm[p == 0 ? 0 : (p >= m - 1 ? 2 : 1)];
        }
        return r;
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            xft::mbar_init(&full[i], tl.np);
            xft::mbar_init(&empty[i], tl.nw);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == tl.nw) {
        // ---------------- producer: np elected lanes, each issues the TMA load of its slice of
        // the stage box (loads issued by one thread were measured to overlap poorly)
        if (lane < tl.np) {
            const int esplit = (D == 3 ? tl.e2 : tl.e1) / tl.np;          // lines of the split axis per slice
            const int slice_elems = stage_elems / tl.np;
            const uint32_t bytes = (uint32_t)slice_elems * 8u;
            int q = 0, pb = 0;
            uint32_t pph = 0;
            for (int t = ts; t <= te; ++t) {
                const unsigned cm_t = win_mask(lm, t);
                for (int g = 0; g < nga; ++g) {
                    if (g >= NGI && !((cm_t >> (g - NGI)) & 1u)) continue;
                    const int b = pb;
                    if (q >= nst) xft::mbar_wait(&empty[b], pph ^ 1u);
                    if (++pb == nst) {
                        pb = 0;
                        pph ^= 1u;
                    }
                    xft::mbar_expect_tx(&full[b], bytes);
                    double* dst = stages + (size_t)b * stage_elems + (size_t)lane * slice_elems;
                    if (D == 3)
                        xft::tma_load<3>(dst, &tmap, &full[b], ct * tl.bc, t, L1 - 1, L2 - 1 + lane * esplit, g);
                    else
                        xft::tma_load<2>(dst, &tmap, &full[b], ct * tl.bc, t, L1 - 1 + lane * esplit, g, 0);
                    ++q;
                }
            }
        }
        return;
    }

    // ---------------- consumers: warp -> (column group, warp block of lines)
    const int wc = warp % tl.wc, wl = warp / tl.wc;
    const int wl1 = wl % tl.wl1, wl2 = wl / tl.wl1;
    const int col = ct * tl.bc + (wc * 32 + lane) * CPT;
    bool cval[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) cval[c] = col + c < n2;
    const int lb1 = wl1 * G::B1, lb2 = wl2 * G::B2;   // warp's first target line inside the tile
    // stage offsets of the warp's source lines (local halo coordinates)
    int soff[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int le1 = lb1 + (s % G::NE1);                 // (lb1 + e1r + 1), e1r = s%NE1 - 1
        const int le2 = D == 3 ? lb2 + (s / G::NE1) : 0;
        soff[s] = (le2 * tl.e1 + le1) * tl.bc + (wc * 32 + lane) * CPT;
    }
    int tline[NT], tcls12[NT];
    bool tval[NT];
    bool lines_int = true;
#pragma unroll
    for (int u = 0; u < NT; ++u) {
        const int z1 = L1 + lb1 + G::u1(u), z2 = D == 3 ? L2 + lb2 + G::u2(u) : 0;
        tval[u] = z1 < m && z2 < m;
        tline[u] = D == 3 ? z1 + m * z2 : z1;
        const int c1 = z1 == 0 ? 0 : (z1 >= m - 1 ? 2 : 1);
        const int c2 = z2 == 0 ? 0 : (z2 >= m - 1 ? 2 : 1);
        tcls12[u] = 3 * c1 + (D == 3 ? 9 * c2 : 0);
        lines_int &= tval[u] && c1 == 1 && (D == 2 || c2 == 1);
    }
    unsigned wm[3] = {0u, 0u, 0u};   // the warp's own target lines
#pragma unroll
    for (int u = 0; u < NT; ++u)
        if (tval[u])
#pragma unroll
            for (int c0 = 0; c0 < 3; ++c0) wm[c0] |= cmask.m[c0 + tcls12[u]];
    double acc[NT][3][CPT];
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[u][0][c] = acc[u][1][c] = acc[u][2][c] = 0.0;
    auto load_src = [&](const double* st, double (&src)[NS][CPT]) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (xft::src_used<D>(s)) {
                if (CPT == 2) {
                    const double2 v = *reinterpret_cast<const double2*>(st + soff[s]);
                    src[s][0] = v.x;
                    src[s][CPT - 1] = v.y;
                } else {
                    src[s][0] = st[soff[s]];
                }
            }
    };

    int q = 0, cbuf = 0;
    uint32_t cph = 0;
    for (int t = ts; t <= te; ++t) {
        const unsigned cm_t = win_mask(lm, t), wm_t = win_mask(wm, t);
        const bool wint = lines_int && t >= 2 && t <= m - 3;
        int cb[NT][3], cbi[NT][3];
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int w = 0; w < 3; ++w) {
                const int p = t + w - 1;
                const int c0 = p <= 0 ? 0 : (p >= m - 1 ? 2 : 1);
                cb[u][w] = (c0 + tcls12[u]) * nga * W;
                cbi[u][w] = TABM == 2 ? (c0 + 3 * ((lb1 + G::u1(u)) + TL1 * (lb2 + G::u2(u)))) * NGI * W
                                      : (c0 + tcls12[u]) * NGI * W;
            }
#pragma unroll
        for (int g = 0; g < NGI; ++g, ++q) {
            const int b = cbuf;
            xft::mbar_wait(&full[b], cph);
            if (++cbuf == nst) {
                cbuf = 0;
                cph ^= 1u;
            }
            const double* st = stages + (size_t)b * stage_elems;
            double src[NS][CPT];
            load_src(st, src);
            if (wint) {
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int u = 0; u < NT; ++u)
#pragma unroll
                        for (int k = 0; k < W; ++k)
                            if (xft::pair_ok<D>(s, u, k)) {
                                const int slot = 1 - G::d0(k);
#pragma unroll
                                for (int c = 0; c < CPT; ++c) acc[u][slot][c] = fma(cint.c[g][k], src[s][c], acc[u][slot][c]);
                            }
            } else {
                // near the boundary: constant-cache table when boundary steps are a minority
                // (m >= 9), global class table (L1 broadcast) on the tiny all-boundary lattices
                const double* tg = TABM == 1 ? c_xft + g * W : stab + g * W;
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int u = 0; u < NT; ++u)
#pragma unroll
                        for (int k = 0; k < W; ++k)
                            if (xft::pair_ok<D>(s, u, k)) {
                                const int slot = 1 - G::d0(k);
                                const double cf = TABM != 0 ? tg[cbi[u][slot] + k] : tg[cb[u][slot] + k];
#pragma unroll
                                for (int c = 0; c < CPT; ++c) acc[u][slot][c] = fma(cf, src[s][c], acc[u][slot][c]);
                            }
            }
            __syncwarp();
            if (lane == 0) xft::mbar_arrive(&empty[b]);
        }
        if (cm_t) {
            for (int g = NGI; g < nga; ++g) {
                if (!((cm_t >> (g - NGI)) & 1u)) continue;
                ++q;
                const int b = cbuf;
                xft::mbar_wait(&full[b], cph);
                if (++cbuf == nst) {
                    cbuf = 0;
                    cph ^= 1u;
                }
                if ((wm_t >> (g - NGI)) & 1u) {
                    const double* st = stages + (size_t)b * stage_elems;
                    const double* tg = CTAB ? tab + g * W : stab + g * W;
                    double src[NS][CPT];
                    load_src(st, src);
#pragma unroll
                    for (int s = 0; s < NS; ++s)
#pragma unroll
                        for (int u = 0; u < NT; ++u)
#pragma unroll
                            for (int k = 0; k < W; ++k)
                                if (xft::pair_ok<D>(s, u, k)) {
                                    const int slot = 1 - G::d0(k);
                                    const double cf = CTAB ? __ldg(tg + cb[u][slot] + k) : tg[cb[u][slot] + k];
#pragma unroll
                                    for (int c = 0; c < CPT; ++c) acc[u][slot][c] = fma(cf, src[s][c], acc[u][slot][c]);
                                }
                }
                __syncwarp();
                if (lane == 0) xft::mbar_arrive(&empty[b]);
            }
        }
        // target t-1 complete
        if (t - 1 >= t0) {
#pragma unroll
            for (int u = 0; u < NT; ++u)
#pragma unroll
                for (int c = 0; c < CPT; ++c)
                    if (tval[u] && cval[c])
                        Y[((long long)(t - 1) + (long long)m * tline[u]) * ypitch + col + c] = acc[u][0][c];
        }
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                acc[u][0][c] = acc[u][1][c];
                acc[u][1][c] = acc[u][2][c];
                acc[u][2][c] = 0.0;
            }
    }
    if (t1 == m) {
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int c = 0; c < CPT; ++c)
                if (tval[u] && cval[c]) Y[((long long)(m - 1) + (long long)m * tline[u]) * ypitch + col + c] = acc[u][0][c];
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// tile choice: minimise TMA source-line loads per valid target line
constexpr int XFT_MINW = 4;   // at least 4 consumer warps per CTA
static XftTile choose_tile(int d, int m, int64_t n2, int force_wc, int box_kb, int cpt = 1, int max_nw = 16) {
    XftTile best{};
    double best_cost = 1e30;
    const int B1 = d == 3 ? 2 : 4;
    const int lines1 = m, lines2 = d == 3 ? m : 1;
    for (int wc = 1; wc <= 8; wc *= 2) {
        if (wc == 8 && force_wc != 8) continue;
        if (wc > 1 && n2 < 32LL * wc * cpt) continue;
        if (force_wc > 0 && wc != force_wc) continue;
        for (int w1 = 1; w1 <= 16; ++w1)
            for (int w2 = 1; w2 <= (d == 3 ? 16 : 1); ++w2) {
                const int nw = w1 * w2 * wc;
                if (nw < XFT_MINW || nw > max_nw) continue;
                const int e1 = w1 * B1 + 2, e2 = d == 3 ? w2 * 2 + 2 : 1;
                const int bc = 32 * wc * cpt;
                if ((double)e1 * e2 * bc * 8 > box_kb * 1024.0) continue;
                const int nt1 = (lines1 + w1 * B1 - 1) / (w1 * B1);
                const int nt2 = d == 3 ? (lines2 + w2 * 2 - 1) / (w2 * 2) : 1;
                const int64_t nct = (n2 + bc - 1) / bc;
                const double loads = (double)nt1 * nt2 * e1 * e2 * nct * bc;
                const double useful = (double)lines1 * lines2 * (double)n2;
                double cost = loads / useful + 0.02 * (16 - nw) / 16.0;
                if (cost < best_cost) {
                    best_cost = cost;
                    best = XftTile{w1, w2, wc, nw, e1, e2, bc, nt1, nt2, (int)nct, 1, m};
                }
            }
    }
    return best;
}

int launch_xfanin_tma(sg_problem* P, int l1, int64_t n1, int64_t n2, int64_t pitch, const double* Z,
                      int64_t gstride, double* Y, int64_t ypitch, bool stage_tab) {
    if (l1 >= (int)P->xfi_cmask.size() || P->xfi_cmask[l1].size() != 27) return SG_ERR_UNSUPPORTED;
    XftMask cmk;
    cmk.nbo = (int)P->vorder.size() - P->ng_int;
    if (cmk.nbo > 8) return SG_ERR_UNSUPPORTED;
    std::memcpy(cmk.m, P->xfi_cmask[l1].data(), 27);
    // n2 columns of Z (row pitch `pitch`) -> n2 columns of Y (row pitch ypitch: a column chunk of a wider grid)
    if (ypitch <= 0) ypitch = n2;
    if (l1 >= (int)P->xfi_tab.size() || !P->xfi_tab[l1]) return SG_ERR_UNSUPPORTED;
    const int d = P->fx.d, m = P->fx.lev[l1].m;
    const int nga = (int)P->vorder.size(), ngi = P->ng_int;
    if (m < 3 || (pitch & 1) || n1 * n2 >= (1LL << 31) || (d == 3 && ngi != 10) || (d == 2 && ngi != 6))
        return SG_ERR_UNSUPPORTED;
    auto enc = get_encode();
    if (!enc) return SG_ERR_UNSUPPORTED;
    // wide boxes (4 column groups = 1 KB rows) measured fastest on the m >= 9 lattices
    // (grid (5,3): 1.67 -> 1.25 ms) and slowest on m = 5 (3.3 -> 4.7 ms)
    // (3D: 8 column groups = 2 KB rows, the TMA box limit of 256 elements, are 4-15 % faster still:
    // (3,5) 1.59 -> 1.34 ms, (4,4) 1.10 -> 1.00 ms, profiles/r2o, r2p; no gain on the 2D lattices)
    const int wc_auto = (m >= 9 && n2 >= 128) ? ((d == 3 && n2 >= 256) ? 8 : 4) : 0;
    // ... and small CTAs (one 2x2 line block x 4 column groups, 16 KB stages) beat larger tiles
    // on those lattices: more independent TMA producers per SM (grid (3,5): 2.02 -> 1.82 ms)
    // (round-2 sweeps profiles/r2g, r2m: 4x6 / 4x8 / 6x6-line boxes with 2-6 stages are equal or slower)
    const int box_kb = wc_auto ? (d == 3 ? (wc_auto == 8 ? 32 : 16) : 8) : 24;
    // two columns per lane on the wide 3D tiles: (4,4) 0.98 -> 0.85 ms, (3,5) 1.23 -> 1.06 ms (profiles/r2D)
    // (and on the other families with at least 64 columns: configs[2] (6,6) 0.25 -> 0.21 ms, (7,5) 0.32 ->
    // 0.26 ms; configs[4] (6,2) 1.30 -> 1.24 ms)
    int cpt = (d == 3 && wc_auto == 8) ? 2 : 1;
    XftTile tl{};
    if (cpt == 2) {
        tl = choose_tile(d, m, n2, 4, box_kb, 2, 8);
    } else if (m >= 9 && n2 >= 64 && (d == 2 || wc_auto == 0)) {
        cpt = 2;
        tl = d == 2 ? choose_tile(d, m, n2, n2 >= 256 ? 4 : (n2 >= 128 ? 2 : 1), 16, 2, 8) : choose_tile(d, m, n2, 0, 40, 2, 8);
        if (tl.nw == 0) {
            cpt = 1;
            tl = choose_tile(d, m, n2, wc_auto, box_kb);
        }
    } else {
        tl = choose_tile(d, m, n2, wc_auto, box_kb);
    }
    if (tl.nw == 0) tl = choose_tile(d, m, n2, 0, 24);
    // split the sweep until there are >= 2 CTAs per SM
    const int64_t base = (int64_t)tl.ntl1 * tl.ntl2 * tl.nct;
    int seglen = m;
    while (seglen > 8 && base * ((m + seglen - 1) / seglen) < 148 * 3) seglen = (seglen + 1) / 2;
    tl.seglen = seglen;
    tl.np = 1;   // (2-6 producer lanes per stage measured no different, profiles/r2o)
    tl.nseg = (m + seglen - 1) / seglen;
    const int64_t nblk = base * tl.nseg;
    if (nblk >= (1LL << 31)) return SG_ERR_UNSUPPORTED;

    CUtensorMap tm;
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    int rank;
    if (d == 3) {
        rank = 5;
        dims[0] = (cuuint64_t)n2; dims[1] = m; dims[2] = m; dims[3] = m; dims[4] = nga;
        strides[0] = (cuuint64_t)pitch * 8;
        strides[1] = (cuuint64_t)pitch * 8 * m;
        strides[2] = (cuuint64_t)pitch * 8 * m * m;
        strides[3] = (cuuint64_t)gstride * 8;
        box[0] = tl.bc; box[1] = 1; box[2] = tl.e1; box[3] = tl.e2 / tl.np; box[4] = 1;
    } else {
        rank = 4;
        dims[0] = (cuuint64_t)n2; dims[1] = m; dims[2] = m; dims[3] = nga;
        strides[0] = (cuuint64_t)pitch * 8;
        strides[1] = (cuuint64_t)pitch * 8 * m;
        strides[2] = (cuuint64_t)gstride * 8;
        box[0] = tl.bc; box[1] = 1; box[2] = tl.e1 / tl.np; box[3] = 1;
    }
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(Z), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed");
        return SG_ERR_CUDA;
    }
    XftCoef ci;
    std::memcpy(ci.c, P->xfi_cint[l1].data(), sizeof(ci.c));
    const size_t stage_b = (size_t)tl.e1 * tl.e2 * tl.bc * 8;
    // 4 stages measured best (deeper rings shrink L1 and were slower: (2,6) 3.3 -> 5.1 ms at 8 stages)
    // (3 stages on the wide-box 3D tiles: 1.2 % faster than 4)
    tl.nst = (wc_auto || cpt == 2) && d == 3 ? 3 : 4;
    if (P->verbose)
        fprintf(stderr, "xft l1=%d m=%d n2=%lld tile w1=%d w2=%d wc=%d nw=%d box=%dx%dx%d nst=%d seglen=%d np=%d nblk=%lld\n", l1, m,
                (long long)n2, tl.wl1, tl.wl2, tl.wc, tl.nw, tl.e1, tl.e2, tl.bc, tl.nst, tl.seglen, tl.np, (long long)nblk);
    // class table of the boundary path: constant bank where boundary steps are a minority, shared
    // memory on the small lattices (3D m = 5: pass 2 of grid (2,6) 2.80 -> 1.93 ms; 2D m <= 17:
    // 0.38 -> 0.33 ms on (3,9); the 52 KB 3D table costs too much occupancy from m = 9 on; profiles/r2r)
    const bool ctab = d == 3 ? m >= 9 : m >= 33;
    if (!ctab && d == 3) tl.nst = 3;   // room for two CTAs per SM next to the 52 KB shared-memory class table
    // 3D tiles of 2 x 2 target lines: the 12 class rows of the tile in shared memory (14 KB)
    // ((3,5) 1.35 -> 1.22 ms, (4,4) 1.00 -> 0.97 ms; no gain from m = 33 on; profiles/r2x)
    const bool tile_tab = ctab && d == 3 && tl.wl1 == 1 && tl.wl2 == 1 && m <= 17;
    size_t smem = (size_t)tl.nst * stage_b + 2 * tl.nst * sizeof(uint64_t);
    if (!ctab) smem += sizeof(double) * (d == 3 ? 27 : 9) * nga * P->fx.W;
    if (tile_tab) smem += sizeof(double) * 3 * 4 * ngi * P->fx.W;
    {
        int ncls = 1;
        for (int q = 0; q < d; ++q) ncls *= 3;
        const size_t nt = (size_t)ncls * ngi * P->fx.W;
        if (nt > (size_t)XFT_CTAB || !P->xfi_itab[l1]) return SG_ERR_UNSUPPORTED;
        if (stage_tab)   // (later column chunks of the same apply reuse the staged table)
        SG_CUDA(cudaMemcpyToSymbolAsync(c_xft, P->xfi_itab[l1], sizeof(double) * nt, 0, cudaMemcpyDeviceToDevice,
                                        P->stream));
    }
    const int threads = 32 * (tl.nw + 1);
    const double* tab = P->xfi_tab[l1];
#define XFT(DD, NG, ...)                                                                                          \
    do {                                                                                                         \
        cudaFuncSetAttribute(k_xfanin_tma<DD, NG, __VA_ARGS__>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        k_xfanin_tma<DD, NG, __VA_ARGS__><<<(unsigned)nblk, threads, smem, P->stream>>>(tm, nga, (int)n2, m, tl, tab, ci, Y, P->skip, (long long)ypitch, cmk); \
    } while (0)
    if (d == 3) {
        if (cpt == 2 && tile_tab) XFT(3, 10, 2, 2); else if (cpt == 2 && ctab) XFT(3, 10, 1, 2);
        else if (tile_tab) XFT(3, 10, 2); else if (ctab) XFT(3, 10, 1); else XFT(3, 10, 0);
    } else {
        if (cpt == 2 && ctab) XFT(2, 6, 1, 2); else if (cpt == 2) XFT(2, 6, 0, 2);
        else if (ctab) XFT(2, 6, 1); else XFT(2, 6, 0);
    }
#undef XFT
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

}  // namespace sg
