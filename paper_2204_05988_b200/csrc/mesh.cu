// sg_build_meshes: nested structured Kuhn P1 meshes on the device.
// PAPER.md l.64-67 (nested FE spaces by uniform refinement), l.506 (embedding E).
#include <algorithm>

#include "mesh_dev.cuh"
#include "sg_internal.cuh"

namespace sg {

__global__ void k_mesh_nodes(int kind, int d, int m, int64_t n, int32_t* lat) {
    int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (id >= n) return;
    int z[MAXD] = {0, 0, 0};
    node_lattice(kind, d, m, id, z);
    for (int i = 0; i < d; ++i) lat[i * n + id] = z[i];
}

// Row of the P1 pattern: node z and every z' = z + sgn e_S (S nonempty) that
// shares a lattice cell of the domain with z (Kuhn edges connect exactly the
// cell vertices whose difference is a 0/1 vector of one sign).
__global__ void k_mesh_pattern(int kind, int d, int m, int64_t n, const int32_t* lat, int W, int32_t* cols) {
    int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (id >= n) return;
    const int cells = m - 1;
    int z[MAXD] = {0, 0, 0};
    for (int i = 0; i < d; ++i) z[i] = lat[i * n + id];
    int64_t nb[16];
    int cnt = 0;
    nb[cnt++] = id;
    for (int S = 1; S < (1 << d); ++S) {
        for (int sg = -1; sg <= 1; sg += 2) {
            int zp[MAXD] = {0, 0, 0};
            for (int i = 0; i < d; ++i) zp[i] = z[i] + (((S >> i) & 1) ? sg : 0);
            int64_t j = node_index(kind, d, m, zp);
            if (j < 0) continue;
            // cells containing both: corner c_i = min(z_i, zp_i) for i in S, z_i-1 or z_i otherwise
            bool ok = false;
            int nfree = 0, freeax[MAXD];
            for (int i = 0; i < d; ++i)
                if (!((S >> i) & 1)) freeax[nfree++] = i;
            for (int comb = 0; comb < (1 << nfree) && !ok; ++comb) {
                int c[MAXD] = {0, 0, 0};
                for (int i = 0; i < d; ++i) c[i] = ((S >> i) & 1) ? min(z[i], zp[i]) : z[i];
                for (int f = 0; f < nfree; ++f)
                    if ((comb >> f) & 1) c[freeax[f]] -= 1;
                ok = cell_in_domain(kind, d, cells, c);
            }
            if (ok) nb[cnt++] = j;
        }
    }
    // insertion sort (<= 15 entries)
    for (int a = 1; a < cnt; ++a) {
        int64_t v = nb[a];
        int b = a - 1;
        while (b >= 0 && nb[b] > v) {
            nb[b + 1] = nb[b];
            --b;
        }
        nb[b + 1] = v;
    }
    for (int k = 0; k < W; ++k) cols[k * n + id] = k < cnt ? (int32_t)nb[k] : -1;
}

// E_{l <- l-1}[f, c] = phi_c(x_f): 1 at coincident nodes, 1/2 at the midpoint
// of the coarse Kuhn edge (z - e_S)/2 -- (z + e_S)/2, S = odd coordinates of z.
__global__ void k_prolong(int kind, int d, int mf, int64_t nf, const int32_t* latf, int mc, int32_t* pc,
                          double* pv) {
    int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (f >= nf) return;
    int z[MAXD] = {0, 0, 0}, S = 0;
    for (int i = 0; i < d; ++i) {
        z[i] = latf[i * nf + f];
        if (z[i] & 1) S |= (1 << i);
    }
    if (S == 0) {
        int zc[MAXD] = {0, 0, 0};
        for (int i = 0; i < d; ++i) zc[i] = z[i] / 2;
        pc[f] = (int32_t)node_index(kind, d, mc, zc);
        pc[nf + f] = -1;
        pv[f] = 1.0;
        pv[nf + f] = 0.0;
        return;
    }
    int za[MAXD] = {0, 0, 0}, zb[MAXD] = {0, 0, 0};
    for (int i = 0; i < d; ++i) {
        int o = (S >> i) & 1;
        za[i] = (z[i] - o) / 2;
        zb[i] = (z[i] + o) / 2;
    }
    int64_t a = node_index(kind, d, mc, za), b = node_index(kind, d, mc, zb);
    if (a > b) {
        int64_t t = a; a = b; b = t;
    }
    pc[f] = (int32_t)a;
    pc[nf + f] = (int32_t)b;
    pv[f] = 0.5;
    pv[nf + f] = 0.5;
}

// E^T row of coarse node c: the fine node at 2 z_c (weight 1) and all its fine
// Kuhn neighbours (the midpoints of coarse edges at c, weight 1/2).
__global__ void k_restrict_rows(int kind, int d, int mc, int64_t nc_, const int32_t* latc, int mf, int64_t nf,
                                const int32_t* colsf, int W, int32_t* rc, double* rv) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc_) return;
    int z[MAXD] = {0, 0, 0};
    for (int i = 0; i < d; ++i) z[i] = 2 * latc[i * nc_ + c];
    int64_t fc = node_index(kind, d, mf, z);
    for (int k = 0; k < W; ++k) {
        int32_t col = colsf[k * nf + fc];
        rc[k * nc_ + c] = col;
        rv[k * nc_ + c] = col < 0 ? 0.0 : (col == fc ? 1.0 : 0.5);
    }
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

int build_factor_meshes(sg_problem* P, Factor& f, int F) {
    f.W = (1 << (f.d + 1)) - 1;
    f.lev.assign(F + 1, Level());
    for (int l = 1; l <= F; ++l) {
        Level& L = f.lev[l];
        const int cells = f.nc << (l - 1);
        L.m = cells + 1;
        L.n = mesh_nodes(f.kind, f.d, L.m);
        SG_CUDA(cudaMalloc(&L.lat, sizeof(int32_t) * f.d * L.n));
        SG_CUDA(cudaMalloc(&L.cols, sizeof(int32_t) * f.W * L.n));
        k_mesh_nodes<<<nblk(L.n, 256), 256, 0, P->stream>>>(f.kind, f.d, L.m, L.n, L.lat);
        k_mesh_pattern<<<nblk(L.n, 128), 128, 0, P->stream>>>(f.kind, f.d, L.m, L.n, L.lat, f.W, L.cols);
        P->launches += 2;
        if (l >= 2) {
            Level& C = f.lev[l - 1];
            SG_CUDA(cudaMalloc(&L.pcols, sizeof(int32_t) * 2 * L.n));
            SG_CUDA(cudaMalloc(&L.pvals, sizeof(double) * 2 * L.n));
            SG_CUDA(cudaMalloc(&L.rcols, sizeof(int32_t) * f.W * C.n));
            SG_CUDA(cudaMalloc(&L.rvals, sizeof(double) * f.W * C.n));
            k_prolong<<<nblk(L.n, 256), 256, 0, P->stream>>>(f.kind, f.d, L.m, L.n, L.lat, C.m, L.pcols, L.pvals);
            k_restrict_rows<<<nblk(C.n, 256), 256, 0, P->stream>>>(f.kind, f.d, C.m, C.n, C.lat, L.m, L.n, L.cols,
                                                                   f.W, L.rcols, L.rvals);
            P->launches += 2;
        }
        SG_CUDA(cudaGetLastError());
    }
    return SG_OK;
}

}  // namespace sg
