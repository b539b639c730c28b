// Fused two-sided strip-operator apply for d = 1 (2D phase space), batched over component grids:
//
//   Y[s][i][a] = sum_b sum_{e in b, s_out(e) = s} sum_k C_e[i, i+k-1] ( sum_j B_b[a, a+j-1] X[s_in(e)][i+k-1][a+j-1] )
//
// (application order l.516-532 with S^(2) first).  On 1D factor meshes both
// stencils have three points, so one thread owns one node (i, a), reads the 3 x 3 neighbourhood
// of X once per time component, forms the three v-sums of a group in registers, folds them with
// the time-mixed x-stencils of the group's entries and writes Y: no intermediates (north_star
// subsystem (1)).  ONE launch serves any number of component grids (block -> grid map in the
// parameter block): the 2D configurations have hundreds of 10^2..10^4-node grids per inner
// iteration and are bound by launch count, not by arithmetic.
#include <algorithm>
#include <cstring>
#include <vector>

#include "sg_internal.cuh"

namespace sg {

struct D1Ent {
    const double* cst;   // [3][n1] stencil-format combined x matrix of the entry
    int s_out, s_in;
};
constexpr int D1_MAXGRIDS = 48;
struct D1Grid {
    const double* X;
    double* Y;
    const double* skip;          // convergence flag of the grid (kernel exits when != 0) or null
    const double* const* bst;    // [nb] stencil-format v matrices [3][n2] of the grid's v level
    const D1Ent* ent;            // entries of the grid's x level, grouped by v-group
    const int* ebeg;             // [nb + 1] entry ranges per v-group
    int n1, n2, blk0;
};
struct D1Batch {
    int ng, nb, total_blocks;
    D1Grid g[D1_MAXGRIDS];
};

template <int S>
__global__ void __launch_bounds__(256) k_d1fused(const __grid_constant__ D1Batch B) {
    int gi = 0;
    while (gi + 1 < B.ng && B.g[gi + 1].blk0 <= (int)blockIdx.x) ++gi;
    const D1Grid& G = B.g[gi];
    if (G.skip && *G.skip != 0.0) return;   // grid converged (batched block solver)
    const int n1 = G.n1, n2 = G.n2;
    const int t = (blockIdx.x - G.blk0) * 256 + threadIdx.x;
    if (t >= n1 * n2) return;
    const int i = t / n2, a = t - i * n2;
    // 3 x 3 neighbourhood (absent neighbours: clamped index, zero coefficient)
    const int ik[3] = {max(i - 1, 0), i, min(i + 1, n1 - 1)};
    const int aj[3] = {max(a - 1, 0), a, min(a + 1, n2 - 1)};
    double x[S][3][3];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int j = 0; j < 3; ++j) x[s][k][j] = __ldg(G.X + ((size_t)s * n1 + ik[k]) * n2 + aj[j]);
    double acc[S];
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = 0.0;
    for (int b = 0; b < B.nb; ++b) {
        const int e0 = G.ebeg[b], e1 = G.ebeg[b + 1];
        if (e0 == e1) continue;
        const double* bs = G.bst[b];
        const double b0 = __ldg(bs + a), b1 = __ldg(bs + n2 + a), b2 = __ldg(bs + 2 * (size_t)n2 + a);
        double z[S][3];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int k = 0; k < 3; ++k) z[s][k] = fma(b2, x[s][k][2], fma(b1, x[s][k][1], b0 * x[s][k][0]));
        for (int e = e0; e < e1; ++e) {
            const D1Ent E = G.ent[e];
            const double c0 = __ldg(E.cst + i), c1 = __ldg(E.cst + n1 + i), c2 = __ldg(E.cst + 2 * (size_t)n1 + i);
            double v = 0.0;
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (s == E.s_in) v = fma(c2, z[s][2], fma(c1, z[s][1], c0 * z[s][0]));
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (s == E.s_out) acc[s] += v;
        }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) G.Y[((size_t)s * n1 + i) * n2 + a] = acc[s];
}

// device tables per level: v-matrix pointers [l2][nb], entries [l1] grouped by v-group
int prepare_d1fused(sg_problem* P) {
    P->d1_ok = false;
    if (P->fx.d != 1 || P->fv.d != 1 || P->fx.kind != SG_MESH_BOX || P->fv.kind != SG_MESH_BOX || P->S > 2 ||
        getenv("SG_NO_FUSED") != nullptr)
        return SG_OK;
    const int nb = (int)P->vorder.size();
    P->d1_bst.assign(P->F + 1, nullptr);
    P->d1_ent.assign(P->F + 1, nullptr);
    P->d1_ebeg.assign(P->F + 1, nullptr);
    P->d1_nent.assign(P->F + 1, 0);
    for (int l = 1; l <= P->F; ++l) {
        std::vector<const double*> hb(nb);
        for (int o = 0; o < nb; ++o) {
            const int sp = P->vgroups[P->vorder[o]].spec;
            if ((int)P->fv.lev[l].fst.size() <= sp || !P->fv.lev[l].fst[sp]) return SG_OK;   // (no stencil copy: keep two-pass)
            hb[o] = P->fv.lev[l].fst[sp];
        }
        std::vector<D1Ent> he;
        std::vector<int> beg(nb + 1, 0);
        for (int o = 0; o < nb; ++o) {
            beg[o] = (int)he.size();
            for (const auto& ce : P->vgroups[P->vorder[o]].comb[l]) {
                if (!ce.st) return SG_OK;
                he.push_back({ce.st, ce.s_out, ce.s_in});
            }
        }
        beg[nb] = (int)he.size();
        SG_CUDA(cudaMalloc(&P->d1_bst[l], sizeof(double*) * nb));
        SG_CUDA(cudaMemcpy(P->d1_bst[l], hb.data(), sizeof(double*) * nb, cudaMemcpyHostToDevice));
        SG_CUDA(cudaMalloc(&P->d1_ent[l], sizeof(D1Ent) * std::max<size_t>(he.size(), 1)));
        if (!he.empty())
        SG_CUDA(cudaMemcpy(P->d1_ent[l], he.data(), sizeof(D1Ent) * he.size(), cudaMemcpyHostToDevice));
        SG_CUDA(cudaMalloc(&P->d1_ebeg[l], sizeof(int) * (nb + 1)));
        SG_CUDA(cudaMemcpy(P->d1_ebeg[l], beg.data(), sizeof(int) * (nb + 1), cudaMemcpyHostToDevice));
        P->d1_nent[l] = (int)he.size();
    }
    P->d1_ok = true;
    return SG_OK;
}

void free_d1fused(sg_problem* P) {
    for (auto p : P->d1_bst) cudaFree(p);
    for (auto p : P->d1_ent) cudaFree(p);
    for (auto p : P->d1_ebeg) cudaFree(p);
}

// Y_g = A_{g,g} X_g for a batch of component grids in one launch (skips[g]: convergence flags or null).
// *fbytes: factor data read (v stencils per column, entry stencils per row), *flops are the caller's.
int launch_d1fused(sg_problem* P, int n, const Grid* const* grids, const double* const* X, double* const* Y,
                   const double* const* skips, double* fbytes) {
    if (!P->d1_ok) return SG_ERR_UNSUPPORTED;
    const int nb = (int)P->vorder.size();
    for (int g0 = 0; g0 < n; g0 += D1_MAXGRIDS) {
        D1Batch B;
        B.ng = std::min(D1_MAXGRIDS, n - g0);
        B.nb = nb;
        int blk = 0;
        for (int q = 0; q < B.ng; ++q) {
            const Grid& g = *grids[g0 + q];
            if (g.n1 * g.n2 >= (1LL << 31)) return SG_ERR_UNSUPPORTED;
            D1Grid& D = B.g[q];
            D.X = X[g0 + q];
            D.Y = Y[g0 + q];
            D.skip = skips ? skips[g0 + q] : nullptr;
            D.bst = reinterpret_cast<const double* const*>(P->d1_bst[g.l2]);
            D.ent = reinterpret_cast<const D1Ent*>(P->d1_ent[g.l1]);
            D.ebeg = P->d1_ebeg[g.l1];
            D.n1 = (int)g.n1;
            D.n2 = (int)g.n2;
            D.blk0 = blk;
            blk += (int)((g.n1 * g.n2 + 255) / 256);
            if (fbytes) *fbytes += 8.0 * 3 * (nb * (double)g.n2 + P->d1_nent[g.l1] * (double)g.n1);
        }
        B.total_blocks = blk;
        if (P->S == 1)
            k_d1fused<1><<<blk, 256, 0, P->stream>>>(B);
        else
            k_d1fused<2><<<blk, 256, 0, P->stream>>>(B);
        P->launches++;
        SG_CUDA(cudaGetLastError());
    }
    return SG_OK;
}

// end-of-batch timestamp: one launch accounts every grid of a batched apply (time once, bytes and
// FLOPs of the grids that were not skipped)
struct StampBatch {
    int n;
    const double* skip[D1_MAXGRIDS];
    double bytes[D1_MAXGRIDS], flops[D1_MAXGRIDS];
};
__global__ void k_tstamp_batch(SolveCtl* c, int slot, const __grid_constant__ StampBatch sb) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    double by = 0.0, fl = 0.0;
    unsigned long long na = 0;
    for (int i = 0; i < sb.n; ++i) {
        if (sb.skip[i] && *sb.skip[i] != 0.0) continue;
        by += sb.bytes[i];
        fl += sb.flops[i];
        ++na;
    }
    if (na == 0) return;
    atomicAdd(&c->apply_ns, (double)(t - c->t0[slot]));
    atomicAdd((unsigned long long*)&c->timed_applies, na);
    atomicAdd(&c->alg_bytes, by);
    atomicAdd(&c->alg_flops, fl);
}
int launch_tstamp_batch(sg_problem* P, int n, const double* const* skips, const double* bytes, const double* flops) {
    for (int g0 = 0; g0 < n; g0 += D1_MAXGRIDS) {
        StampBatch sb;
        sb.n = std::min(D1_MAXGRIDS, n - g0);
        for (int i = 0; i < sb.n; ++i) {
            sb.skip[i] = skips ? skips[g0 + i] : nullptr;
            sb.bytes[i] = bytes[g0 + i];
            sb.flops[i] = flops[g0 + i];
        }
        k_tstamp_batch<<<1, 1, 0, P->stream>>>(P->ctl, P->stamp_slot, sb);
        P->launches++;
    }
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

}  // namespace sg
