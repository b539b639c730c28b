// Pass 1 of the strip-operator apply on box v-lattices by shifted moments:
//
//   Z_g[r][a] = sum_k B_g[a, a + off_k] X[r][a + off_k]     for the interior v-groups g
//
// (the v-factor B_t of every Kronecker term; l.516-532
// applies it first).  The interior v-groups of the streaming configurations
// are weighted masses B_n = int y^n phi_a phi_b with monomial weights y^n,
// |n| <= 2 (the 1, v_i and v_i v_j of beta = (v, 0) in eq. (14)).  Expanding
// the weight around the row node y_a,
//     y^n = sum_{m <= n} binom(n, m) y_a^{n-m} (y - y_a)^m ,
// every row is a polynomial in y_a times the SHIFTED-moment stencils
//     R_m^{cls}[k] = int (y - y_a)^m phi_a phi_{a+off_k} dy ,
// which depend only on the boundary class of a (per axis low/interior/high)
// and scale as h^{d+|m|} with the level.  So instead of reading 10 x 15
// stored coefficients per v-node, the kernels form the 10 (d = 3) / 6 (d = 2)
// moment sums ZR_m = sum_k R_m[k] X[r][a + off_k] with CONSTANT coefficients
// (compile-time kernel parameters for interior columns; a shared-memory class
// table for boundary columns) and combine them with powers of y_a:
//     Z_{y_i}     = y_i ZR_0 + ZR_i
//     Z_{y_i y_j} = y_i y_j ZR_0 + y_i ZR_j + y_j ZR_i + ZR_ij
//     Z_{y_i^2}   = y_i^2 ZR_0 + 2 y_i ZR_i + ZR_ii .
// The R tables are derived once from the level-1 assembled matrices (every
// class has exactly one level-1 node, |y_a| <= h_1 keeps the shift exact to
// rounding) and scaled by exact powers of two; every level is verified row by
// row against its assembled stencils before the path is enabled.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "sg_internal.cuh"
#include "vmom.cuh"

namespace sg {

template <int D>
__device__ __forceinline__ void vm_combine(const double (&zr)[VM_NP], const double* y, const VmOut& o, long long idx) {
#pragma unroll
    for (int n = 0; n < VM_NP; ++n) {
        if (!vm::mono_in(D, n)) continue;
        double* p = o.p[n];
        if (!p) continue;
        double v;
        if (n == 0) {
            v = zr[0];
        } else if (n <= 3) {
            const int i = n - 1;
            v = fma(y[i], zr[0], zr[n]);
        } else {
            const int i = vm::mono_ax(n, 0), j = vm::mono_ax(n, 1);
            if (i == j)
                v = fma(y[i] * y[i], zr[0], fma(2.0 * y[i], zr[vm::lin(i)], zr[n]));
            else
                v = fma(y[i] * y[j], zr[0], fma(y[i], zr[vm::lin(j)], fma(y[j], zr[vm::lin(i)], zr[n])));
        }
        p[idx] = v;
    }
}

// all v-columns in natural order (full-sector stores): thread = (column a, block of VR consecutive
// rows); the class of a selects its row of the shared-memory table [3^D][VM_NP + VM_NC][W]
// (class stride padded against bank conflicts); each coefficient load feeds VR rows.
constexpr int VR = 4;
template <int D>
__global__ void __launch_bounds__(256, 2)
    k_vmom(int nthr, int n2, int nrows, int rstride, int m, long long pitch, const double* __restrict__ X,
           const __grid_constant__ VmOut o, const uint8_t* __restrict__ xflag, int n1x,
           const double* __restrict__ tab, const __grid_constant__ VmCoef cf, double lo0, double lo1, double lo2,
           double h0, double h1, double h2, const double* __restrict__ skip, int c0, int ncol) {
    // columns [c0, c0 + ncol) only (L2-resident column chunks); output column a - c0
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    constexpr int W = D == 3 ? 15 : 7;
    constexpr int NC = D == 3 ? 27 : 9;
    constexpr int NR = VM_NP + VM_NC;
    constexpr int CS = NR * W + 1;   // padded class stride (doubles)
    extern __shared__ double st[];   // [NC][CS]
    for (int i = threadIdx.x; i < NC * NR * W; i += 256) {
        const int c = i / (NR * W);
        st[c * CS + (i - c * NR * W)] = tab[i];
    }
    __syncthreads();
    const int t = blockIdx.x * 256 + threadIdx.x;
    if (t >= nthr) return;
    const int a = c0 + t % ncol, q0 = t / ncol;
    int z[3] = {a % m, (a / m) % m, D == 3 ? a / (m * m) : 0};
    int cls = 0, mul = 1;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        cls += mul * (z[q] == 0 ? 0 : (z[q] == m - 1 ? 2 : 1));
        mul *= 3;
    }
    const double y[3] = {lo0 + h0 * z[0], lo1 + h1 * z[1], lo2 + h2 * z[2]};
    const double* ct = st + cls * CS;
    bool nb_ok[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int c = a + cf.off[k];
        nb_ok[k] = c >= 0 && c < n2;   // (absent neighbours have zero coefficients)
    }
    const bool padcol = (a == c0 + ncol - 1) && pitch > ncol;   // keep the stored rows full 32-byte sectors
    for (int rb = q0 * VR; rb < nrows; rb += rstride * VR) {
        double acc[VM_NP][VR];
#pragma unroll
        for (int n = 0; n < VM_NP; ++n)
#pragma unroll
            for (int r = 0; r < VR; ++r) acc[n][r] = 0.0;
        const double* xb = X + (long long)rb * n2 + a;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            double xv[VR];
#pragma unroll
            for (int r = 0; r < VR; ++r)
                xv[r] = (nb_ok[k] && rb + r < nrows) ? __ldg(xb + (r * n2 + cf.off[k])) : 0.0;
#pragma unroll
            for (int n = 0; n < VM_NP; ++n) {
                if (!vm::mono_in(D, n)) continue;
                const double c = ct[n * W + k];
#pragma unroll
                for (int r = 0; r < VR; ++r) acc[n][r] = fma(c, xv[r], acc[n][r]);
            }
        }
#pragma unroll
        for (int r = 0; r < VR; ++r) {
            const int row = rb + r;
            if (row >= nrows) break;
            double zr[VM_NP];
#pragma unroll
            for (int n = 0; n < VM_NP; ++n) zr[n] = acc[n][r];
            const long long idx = (long long)row * pitch + (a - c0);
            vm_combine<D>(zr, y, o, idx);
            const bool xb_row = cf.nchi && xflag[row % n1x];
            if (xb_row) {
                // chi groups (unrolled for d = 2: compile-time parameter offsets; rolled for d = 3,
                // where unrolling spills); half stencils need the row's X values again (plane rows only)
#pragma unroll(D == 2 ? VM_NC : 1)
                for (int c = 0; c < VM_NC; ++c) {
                    if (c >= cf.nchi) break;
                    const int i = cf.chax[c];
                    const double yi = i == 0 ? y[0] : (i == 1 ? y[1] : y[2]);
                    const double zi = i == 0 ? zr[1] : (i == 1 ? zr[2] : zr[3]);
                    double v = cf.chkeep[c] * yi > 0.0 ? fma(yi, zr[0], zi) : 0.0;
                    if (yi == 0.0) {
                        v = 0.0;
                        const double* hc = ct + (VM_NP + c) * W;
                        const double* xr = X + (long long)row * n2 + a;
#pragma unroll
                        for (int k = 0; k < W; ++k)
                            if (nb_ok[k]) v = fma(hc[k], __ldg(xr + cf.off[k]), v);
                    }
                    o.pc[c][idx] = v;
                }
            }
            if (padcol) {
#pragma unroll
                for (int n = 0; n < VM_NP; ++n)
                    if (vm::mono_in(D, n) && o.p[n]) o.p[n][idx + 1] = 0.0;
                if (xb_row)
                    for (int c = 0; c < cf.nchi; ++c) o.pc[c][idx + 1] = 0.0;
            }
        }
    }
}

// verification: max |B_n[a][k] - reconstruction| and max |B_n| over all rows (per monomial group)
__global__ void k_vmom_check(int D, int n, int m, int W, int mono, const double* __restrict__ st,
                             const double* __restrict__ tab, double lo0, double lo1, double lo2, double h0, double h1,
                             double h2, double* out2, int chi_c, int chi_ax, int chi_keep) {
    __shared__ double sm[2][8];
    double dev = 0.0, mag = 0.0;
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
        int z[3] = {a % m, (a / m) % m, D == 3 ? a / (m * m) : 0};
        int cls = 0, mul = 1;
        for (int q = 0; q < D; ++q) {
            cls += mul * (z[q] == 0 ? 0 : (z[q] == m - 1 ? 2 : 1));
            mul *= 3;
        }
        const double y[3] = {lo0 + h0 * z[0], lo1 + h1 * z[1], lo2 + h2 * z[2]};
        const double* ct = tab + cls * (VM_NP + VM_NC) * W;
        for (int k = 0; k < W; ++k) {
            double zr[VM_NP];
            for (int q = 0; q < VM_NP; ++q) zr[q] = ct[q * W + k];
            double v;
            if (chi_c >= 0) {
                const double yi = y[chi_ax];
                v = chi_keep * yi > 0.0 ? yi * zr[0] + zr[1 + chi_ax] : 0.0;
                if (yi == 0.0) v = ct[(VM_NP + chi_c) * W + k];
            } else if (mono == 0) v = zr[0];
            else if (mono <= 3) v = y[mono - 1] * zr[0] + zr[mono];
            else {
                const int i = vm::mono_ax(mono, 0), j = vm::mono_ax(mono, 1);
                v = (i == j) ? y[i] * y[i] * zr[0] + 2.0 * y[i] * zr[vm::lin(i)] + zr[mono]
                             : y[i] * y[j] * zr[0] + y[i] * zr[vm::lin(j)] + y[j] * zr[vm::lin(i)] + zr[mono];
            }
            const double s = st[(long long)k * n + a];
            dev = fmax(dev, fabs(v - s));
            mag = fmax(mag, fabs(s));
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        mag = fmax(mag, __shfl_xor_sync(0xffffffffu, mag, o));
    }
    if ((threadIdx.x & 31) == 0) {
        sm[0][threadIdx.x >> 5] = dev;
        sm[1][threadIdx.x >> 5] = mag;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a = fmax(a, sm[0][w]);
            b = fmax(b, sm[1][w]);
        }
        out2[2 * blockIdx.x] = a;
        out2[2 * blockIdx.x + 1] = b;
    }
}

static int pure_monomial(const Spec& s, int d) {   // monomial slot of a plain weighted mass, -1 otherwise
    if (s.kind != 0 || s.trial_d >= 0 || s.test_d >= 0 || s.chi_axis >= 0) return -1;
    int slot = -1;
    for (int i = 0; i < NPOLY; ++i) {
        if (s.w[i] == 0.0) continue;
        if (s.w[i] != 1.0 || slot >= 0) return -1;
        slot = i;
    }
    if (slot < 0 || !vm::mono_in(d, slot)) return -1;
    return slot;
}

static bool chi_linear(const Spec& s, int d, int* axis, int* keep) {   // y_i chi(keep y_i > 0) mass
    if (s.kind != 0 || s.trial_d >= 0 || s.test_d >= 0 || s.chi_axis < 0 || s.chi_axis >= d) return false;
    for (int i = 0; i < NPOLY; ++i)
        if (s.w[i] != (i == 1 + s.chi_axis ? 1.0 : 0.0)) return false;
    *axis = s.chi_axis;
    *keep = s.chi_sign;
    return true;
}

int prepare_vmom(sg_problem* P) {
    P->vm_ok.assign(P->F + 1, 0);
    P->vm_tab.assign(P->F + 1, nullptr);
    P->vm_int.assign(P->F + 1, {});
    P->vm_blist.assign(P->F + 1, nullptr);
    P->vm_nb.assign(P->F + 1, 0);
    P->vm_slot.assign(MAXG, -1);
    P->vm_nchi = 0;
    const Factor& f = P->fv;
    const int d = f.d, W = f.W;
    constexpr int NR = VM_NP + VM_NC;
    if (f.kind != SG_MESH_BOX || d < 2 ) return SG_OK;
    // interior groups must be plain monomial-weighted masses, and the set must be closed
    int spec_of[VM_NP];
    for (int n = 0; n < VM_NP; ++n) spec_of[n] = -1;
    for (int o = 0; o < P->ng_int; ++o) {
        const int sp = P->vgroups[P->vorder[o]].spec;
        const int slot = pure_monomial(f.specs[sp], d);
        if (slot < 0 || spec_of[slot] >= 0) return SG_OK;
        spec_of[slot] = sp;
        P->vm_slot[o] = slot;
    }
    for (int n = 0; n < VM_NP; ++n) {
        if (spec_of[n] < 0) continue;
        if (spec_of[0] < 0) return SG_OK;
        for (int w = 0; w < 2; ++w) {
            const int ax = vm::mono_ax(n, w);
            if (ax >= 0 && spec_of[vm::lin(ax)] < 0) return SG_OK;
        }
    }
    // boundary-only groups: inflow masses y_i chi(keep y_i > 0) (all of them, or none by moments)
    const int nbo = (int)P->vorder.size() - P->ng_int;
    int chi_spec[VM_NC], chi_ax[VM_NC], chi_keep[VM_NC];
    int nchi = 0;
    if (nbo > 0 && nbo <= VM_NC) {
        bool all = true;
        for (int o = 0; o < nbo && all; ++o) {
            const int sp = P->vgroups[P->vorder[P->ng_int + o]].spec;
            int ax, kp;
            all = chi_linear(f.specs[sp], d, &ax, &kp) && spec_of[vm::lin(ax)] >= 0;
            if (all) {
                chi_spec[o] = sp;
                chi_ax[o] = ax;
                chi_keep[o] = kp;
            }
        }
        if (all) nchi = nbo;
    }
    // level-1 rows: one node per class
    const Level& L1 = f.lev[1];
    if (L1.m != 3 || L1.fst.empty()) return SG_OK;
    const int n1 = (int)L1.n;
    double h1[3] = {0, 0, 0}, lo[3] = {0, 0, 0};
    for (int q = 0; q < d; ++q) {
        h1[q] = (f.hi[q] - f.lo[q]) / (L1.m - 1);
        lo[q] = f.lo[q];
    }
    auto fetch = [&](const Level& L, int sp, std::vector<double>& out) -> int {
        if ((int)L.fst.size() <= sp || !L.fst[sp]) return SG_ERR_UNSUPPORTED;
        out.resize((size_t)W * L.n);
        SG_CUDA(cudaMemcpy(out.data(), L.fst[sp], sizeof(double) * W * L.n, cudaMemcpyDeviceToHost));
        return SG_OK;
    };
    std::vector<std::vector<double>> M(VM_NP), Hc(VM_NC);
    for (int n = 0; n < VM_NP; ++n)
        if (spec_of[n] >= 0 && fetch(L1, spec_of[n], M[n]) != SG_OK) return SG_OK;
    for (int c = 0; c < nchi; ++c)
        if (fetch(L1, chi_spec[c], Hc[c]) != SG_OK) return SG_OK;
    int ncls = 1;
    for (int q = 0; q < d; ++q) ncls *= 3;
    std::vector<double> R1((size_t)ncls * NR * W, 0.0);   // [cls][slot | chi][k], level-1 units
    for (int a = 0; a < n1; ++a) {
        int z[3] = {a % 3, (a / 3) % 3, d == 3 ? a / 9 : 0};
        const int cls = z[0] + 3 * z[1] + 9 * z[2];
        double y[3];
        for (int q = 0; q < 3; ++q) y[q] = q < d ? lo[q] + h1[q] * z[q] : 0.0;
        for (int k = 0; k < W; ++k) {
            auto mv = [&](int n) { return M[n][(size_t)k * n1 + a]; };
            double* r = &R1[((size_t)cls * NR) * W + k];
            r[0 * W] = mv(0);
            for (int n = 1; n < VM_NP; ++n) {
                if (spec_of[n] < 0) continue;
                if (n <= 3) {
                    const int i = n - 1;
                    r[n * W] = mv(n) - y[i] * mv(0);
                } else {
                    const int i = vm::mono_ax(n, 0), j = vm::mono_ax(n, 1);
                    if (i == j)
                        r[n * W] = mv(n) - 2.0 * y[i] * mv(vm::lin(i)) + y[i] * y[i] * mv(0);
                    else
                        r[n * W] = mv(n) - y[j] * mv(vm::lin(i)) - y[i] * mv(vm::lin(j)) + y[i] * y[j] * mv(0);
                }
            }
            // half stencils on the plane y_i = 0 (level-1 nodes with z_i = 1; y_i = 0 there, so
            // int chi y_i phi phi = int chi (y_i - y_a,i) phi phi: a first shifted moment)
            for (int c = 0; c < nchi; ++c)
                if (z[chi_ax[c]] == 1) r[(VM_NP + c) * W] = Hc[c][(size_t)k * n1 + a];
        }
    }
    const int icls = d == 3 ? 13 : 4;
    for (int l = 1; l <= P->F; ++l) {
        const Level& L = f.lev[l];
        if (L.m < 3) continue;
        double hl[3] = {0, 0, 0};
        for (int q = 0; q < d; ++q) hl[q] = (f.hi[q] - f.lo[q]) / (L.m - 1);
        // exact power-of-two rescaling: R_l = R_1 * prod_q (h_l/h_1)^(1 + m_q)
        std::vector<double> Rl(R1.size());
        for (int c = 0; c < ncls; ++c)
            for (int n = 0; n < NR; ++n) {
                double s = 1.0;
                for (int q = 0; q < d; ++q) s *= hl[q] / h1[q];
                if (n < VM_NP) {
                    for (int w = 0; w < vm::mono_deg(n); ++w) s *= hl[vm::mono_ax(n, w)] / h1[vm::mono_ax(n, w)];
                } else if (n - VM_NP < nchi) {
                    s *= hl[chi_ax[n - VM_NP]] / h1[chi_ax[n - VM_NP]];
                }
                for (int k = 0; k < W; ++k)
                    Rl[((size_t)c * NR + n) * W + k] = R1[((size_t)c * NR + n) * W + k] * s;
            }
        double* dt;
        SG_CUDA(cudaMalloc(&dt, sizeof(double) * Rl.size()));
        SG_CUDA(cudaMemcpy(dt, Rl.data(), sizeof(double) * Rl.size(), cudaMemcpyHostToDevice));
        // verify every row of every group against its assembled stencil
        bool ok = true;
        const int nbk = 128;
        double* out2;
        SG_CUDA(cudaMalloc(&out2, sizeof(double) * 2 * nbk));
        std::vector<double> hbuf(2 * nbk);
        for (int n = 0; n < VM_NP + nchi && ok; ++n) {
            const bool chi = n >= VM_NP;
            const int c = n - VM_NP;
            const int sp = chi ? chi_spec[c] : spec_of[n];
            if (sp < 0) continue;
            if ((int)L.fst.size() <= sp || !L.fst[sp]) {
                ok = false;
                break;
            }
            k_vmom_check<<<nbk, 256, 0, P->stream>>>(d, (int)L.n, L.m, W, chi ? 0 : n, L.fst[sp], dt, lo[0], lo[1],
                                                      lo[2], hl[0], hl[1], hl[2], out2, chi ? c : -1,
                                                      chi ? chi_ax[c] : 0, chi ? chi_keep[c] : 0);
            P->launches++;
            SG_CUDA(cudaMemcpyAsync(hbuf.data(), out2, sizeof(double) * 2 * nbk, cudaMemcpyDeviceToHost, P->stream));
            SG_CUDA(cudaStreamSynchronize(P->stream));
            double dev = 0, mag = 0;
            for (int b = 0; b < nbk; ++b) {
                dev = std::max(dev, hbuf[2 * b]);
                mag = std::max(mag, hbuf[2 * b + 1]);
            }
            if (!(dev <= 1e-13 * mag)) ok = false;
            if (P->verbose) fprintf(stderr, "[sg] vmom level %d %s %d: dev %.3e mag %.3e\n", l, chi ? "chi" : "mono",
                                    chi ? c : n, dev, mag);
        }
        cudaFree(out2);
        if (!ok) {
            cudaFree(dt);
            continue;
        }
        P->vm_tab[l] = dt;
        P->vm_tab_n = (int64_t)Rl.size();
        std::vector<double> ci((size_t)NR * 15, 0.0);
        for (int n = 0; n < NR; ++n)
            for (int k = 0; k < W; ++k) ci[n * 15 + k] = Rl[((size_t)icls * NR + n) * W + k];
        P->vm_int[l] = ci;
        // boundary columns (natural order)
        std::vector<int> bl;
        for (int64_t a = 0; a < L.n; ++a) {
            int64_t zz = a;
            bool b = false;
            for (int q = 0; q < d; ++q) {
                const int zq = (int)(zz % L.m);
                zz /= L.m;
                b |= (zq == 0 || zq == L.m - 1);
            }
            if (b) bl.push_back((int)a);
        }
        SG_CUDA(cudaMalloc(&P->vm_blist[l], sizeof(int) * std::max<size_t>(bl.size(), 1)));
        SG_CUDA(cudaMemcpy(P->vm_blist[l], bl.data(), sizeof(int) * bl.size(), cudaMemcpyHostToDevice));
        P->vm_nb[l] = (int)bl.size();
        P->vm_ok[l] = 1;
    }
    P->vm_nchi = nchi;
    for (int c = 0; c < nchi; ++c) {
        P->vm_chax[c] = chi_ax[c];
        P->vm_chkeep[c] = chi_keep[c];
    }
    return SG_OK;
}

// interior-class moment stencils, chi-group descriptors, lattice offsets and coordinates of v-level l2
void vmom_coef(const sg_problem* P, int l2, VmCoef* cf, double* lo, double* h) {
    const Factor& f = P->fv;
    const Level& L = f.lev[l2];
    std::memcpy(cf->R, P->vm_int[l2].data(), sizeof(cf->R));
    std::memcpy(cf->H, P->vm_int[l2].data() + VM_NP * 15, sizeof(cf->H));
    cf->nchi = P->vm_nchi;
    for (int c = 0; c < VM_NC; ++c) {
        cf->chax[c] = c < cf->nchi ? P->vm_chax[c] : 0;
        cf->chkeep[c] = c < cf->nchi ? P->vm_chkeep[c] : 0;
    }
    for (int k = 0; k < 15; ++k) cf->off[k] = (int)L.so.off[k];
    for (int q = 0; q < 3; ++q) {
        lo[q] = q < f.d ? f.lo[q] : 0.0;
        h[q] = q < f.d ? (f.hi[q] - f.lo[q]) / (L.m - 1) : 0.0;
    }
}

// Z_g for the interior v-groups of grid (l1, l2) by moments; SG_ERR_UNSUPPORTED if unavailable
int launch_vmom(sg_problem* P, int l2, int64_t nrows, int64_t n2, int64_t pitch, const double* X,
                double* const* outs, const uint8_t* xflag, int64_t n1x, int64_t c0, int64_t c1) {
    if (l2 >= (int)P->vm_ok.size() || !P->vm_ok[l2]) return SG_ERR_UNSUPPORTED;
    if (c1 <= 0) c1 = n2;
    const int64_t ncol = c1 - c0;
    const Factor& f = P->fv;
    const Level& L = f.lev[l2];
    const int d = f.d, m = L.m;
    if (nrows * n2 >= (1LL << 40)) return SG_ERR_UNSUPPORTED;
    VmOut o;
    for (int n = 0; n < VM_NP; ++n) o.p[n] = nullptr;
    for (int g = 0; g < P->ng_int; ++g) o.p[P->vm_slot[g]] = outs[g];
    VmCoef cf;
    double lo[3], h[3];
    vmom_coef(P, l2, &cf, lo, h);
    for (int c = 0; c < VM_NC; ++c) o.pc[c] = c < cf.nchi ? outs[P->ng_int + c] : nullptr;
    const int W = f.W;
    // threads = columns x row blocks (VR rows each), about 16 resident warps per SM
    const long long target = 148LL * 2048;
    const long long rblocks = (nrows + VR - 1) / VR;
    const int ph = (int)std::max<long long>(1, std::min<long long>(target / ncol, rblocks));
    const long long nthr = ncol * (long long)ph;
    if (nthr >= (1LL << 31)) return SG_ERR_UNSUPPORTED;
    const unsigned nb = (unsigned)((nthr + 255) / 256);
    const int smb = (d == 3 ? 27 : 9) * ((VM_NP + VM_NC) * W + 1) * (int)sizeof(double);
#define VMA(DD)                                                                                                     \
    do {                                                                                                            \
        cudaFuncSetAttribute(k_vmom<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);                         \
        k_vmom<DD><<<nb, 256, smb, P->stream>>>((int)nthr, (int)n2, (int)nrows, ph, m, pitch, X, o, xflag, (int)n1x, \
                                                P->vm_tab[l2], cf, lo[0], lo[1], lo[2], h[0], h[1], h[2], P->skip, (int)c0, (int)ncol); \
    } while (0)
    if (d == 3) VMA(3); else VMA(2);
#undef VMA
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

}  // namespace sg
