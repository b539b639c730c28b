// sg_assemble_factors: exact P1 factor matrices on the device, row by row.
// PAPER.md eq. (14) l.450-461 and the tensor reduction l.484-504:
//   vol : F[a,b] = int w(y) chi(y) (D^p phi_b)(D^q phi_a) dy   (b trial/column, a test/row)
//   face: F[a,b] = int_{Gamma_{s e_i}} phi_b phi_a ds
// Element integrals use the collapsed (Duffy) Gauss-Legendre rule with 4 points
// per direction, exact for the polynomial integrands here (degree <= 4, the
// Duffy Jacobian adds <= 2).  One thread owns one matrix row (deterministic,
// no atomics).  Kuhn simplex of cell c and permutation pi: v_0 = c,
// v_k = v_{k-1} + e_{pi(k-1)}; grad lam_0 = -e_{pi0}/h, grad lam_k =
// e_{pi(k-1)}/h - e_{pi(k)}/h, grad lam_d = e_{pi(d-1)}/h.
#include "mesh_dev.cuh"
#include "sg_internal.cuh"

namespace sg {

struct SpecDev {
    int kind;
    double w[NPOLY];
    int trial_d, test_d, chi_axis, chi_sign, face_axis, face_sign;
};

__device__ inline double poly_eval(const double* w, int d, const double* y) {
    double y0 = y[0], y1 = d > 1 ? y[1] : 0.0, y2 = d > 2 ? y[2] : 0.0;
    return w[0] + w[1] * y0 + w[2] * y1 + w[3] * y2 + w[4] * y0 * y0 + w[5] * y0 * y1 + w[6] * y0 * y2 +
           w[7] * y1 * y1 + w[8] * y1 * y2 + w[9] * y2 * y2;
}

__constant__ double c_gl4_x[4];
__constant__ double c_gl4_w[4];

__device__ inline void perm_of(int d, int idx, int* pi) {
    // permutations of {0..d-1} in lexicographic order (idx < d!)
    int avail[MAXD] = {0, 1, 2};
    int fact = 1;
    for (int i = 2; i < d; ++i) fact *= i;
    for (int k = 0; k < d; ++k) {
        int f = 1;
        for (int i = 2; i <= d - 1 - k; ++i) f *= i;
        int j = idx / f;
        idx %= f;
        pi[k] = avail[j];
        for (int t = j; t < d - 1 - k; ++t) avail[t] = avail[t + 1];
    }
    (void)fact;
}

template <int D>
__global__ void k_assemble_row(int kind, int64_t n, int m, const int32_t* lat, const int32_t* cols, int W,
                               double lo0, double lo1, double lo2, double h0, double h1, double h2, SpecDev sp,
                               double* vals) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    const double lo[3] = {lo0, lo1, lo2};
    const double h[3] = {h0, h1, h2};
    const int cells = m - 1;
    int za[3] = {0, 0, 0};
    for (int i = 0; i < D; ++i) za[i] = lat[i * n + a];
    double acc[15];
    int32_t rowc[15];
    for (int k = 0; k < W; ++k) {
        acc[k] = 0.0;
        rowc[k] = cols[k * n + a];
    }
    int nperm = (D == 1) ? 1 : (D == 2 ? 2 : 6);
    double hprod = 1.0;
    for (int i = 0; i < D; ++i) hprod *= h[i];
    double dfact = (D == 1) ? 1.0 : (D == 2 ? 2.0 : 6.0);
    double volK = hprod / dfact;
    for (int dc = 0; dc < (1 << D); ++dc) {
        int c[3] = {0, 0, 0};
        for (int i = 0; i < D; ++i) c[i] = za[i] - ((dc >> i) & 1);
        if (!cell_in_domain(kind, D, cells, c)) continue;
        for (int pidx = 0; pidx < nperm; ++pidx) {
            int pi[3] = {0, 1, 2};
            perm_of(D, pidx, pi);
            // vertices of the simplex
            int vz[D + 1][3];
            for (int i = 0; i < 3; ++i) vz[0][i] = c[i];
            for (int k = 1; k <= D; ++k) {
                for (int i = 0; i < 3; ++i) vz[k][i] = vz[k - 1][i];
                vz[k][pi[k - 1]] += 1;
            }
            int ka = -1;
            for (int k = 0; k <= D; ++k) {
                bool eq = true;
                for (int i = 0; i < D; ++i) eq &= (vz[k][i] == za[i]);
                if (eq) ka = k;
            }
            if (ka < 0) continue;
            int64_t vid[D + 1];
            int slot[D + 1];
            for (int k = 0; k <= D; ++k) {
                vid[k] = node_index(kind, D, m, vz[k]);
                slot[k] = -1;
                for (int s = 0; s < W; ++s)
                    if (rowc[s] == (int32_t)vid[k]) slot[k] = s;
            }
            double yv[D + 1][3];
            for (int k = 0; k <= D; ++k)
                for (int i = 0; i < 3; ++i) yv[k][i] = (i < D) ? lo[i] + h[i] * vz[k][i] : 0.0;
            if (sp.kind == 1) {
                // axis facets: opposite v_0 (normal +e_{pi0}), opposite v_D (normal -e_{pi(D-1)})
                for (int side = 0; side < 2; ++side) {
                    int opp = side == 0 ? 0 : D;
                    int ax = side == 0 ? pi[0] : pi[D - 1];
                    int sgn = side == 0 ? 1 : -1;
                    if (ax != sp.face_axis || sgn != sp.face_sign) continue;
                    if (ka == opp) continue;
                    int cn[3] = {c[0], c[1], c[2]};
                    cn[ax] += sgn;
                    if (cell_in_domain(kind, D, cells, cn)) continue;  // interior face
                    double fa = 1.0;
                    for (int i = 0; i < D; ++i)
                        if (i != ax) fa *= h[i];
                    double dp1f = (D == 1) ? 2.0 : (D == 2 ? 6.0 : 24.0);
                    for (int kb = 0; kb <= D; ++kb) {
                        if (kb == opp) continue;
                        double v = fa * (kb == ka ? 2.0 : 1.0) / dp1f;
                        if (slot[kb] >= 0) acc[slot[kb]] += v;
                    }
                }
                continue;
            }
            // chi at the centroid
            if (sp.chi_axis >= 0) {
                double cen = 0.0;
                for (int k = 0; k <= D; ++k) cen += yv[k][sp.chi_axis];
                cen /= (D + 1);
                if (!(sp.chi_sign * cen > 0.0)) continue;
            }
            // gradients of the barycentric coordinates
            double g[D + 1][3];
            for (int k = 0; k <= D; ++k)
                for (int i = 0; i < 3; ++i) g[k][i] = 0.0;
            g[0][pi[0]] = -1.0 / h[pi[0]];
            for (int k = 1; k < D; ++k) {
                g[k][pi[k - 1]] += 1.0 / h[pi[k - 1]];
                g[k][pi[k]] -= 1.0 / h[pi[k]];
            }
            g[D][pi[D - 1]] = 1.0 / h[pi[D - 1]];
            // quadrature
            double row[D + 1];
            for (int k = 0; k <= D; ++k) row[k] = 0.0;
            const int NQ = 4;
            int nq = 1;
            for (int i = 0; i < D; ++i) nq *= NQ;
            for (int q = 0; q < nq; ++q) {
                int qi[3] = {q % NQ, (q / NQ) % NQ, (q / (NQ * NQ)) % NQ};
                double u[3], wq = 1.0;
                for (int i = 0; i < D; ++i) {
                    u[i] = c_gl4_x[qi[i]];
                    wq *= c_gl4_w[qi[i]];
                }
                double xi[3] = {0, 0, 0}, J = 1.0;
                if (D == 1) {
                    xi[0] = u[0];
                } else if (D == 2) {
                    xi[0] = u[0];
                    xi[1] = u[1] * (1.0 - u[0]);
                    J = 1.0 - u[0];
                } else {
                    xi[0] = u[0];
                    xi[1] = u[1] * (1.0 - u[0]);
                    xi[2] = u[2] * (1.0 - u[0]) * (1.0 - u[1]);
                    J = (1.0 - u[0]) * (1.0 - u[0]) * (1.0 - u[1]);
                }
                double lam[D + 1];
                double s = 0.0;
                for (int k = 1; k <= D; ++k) {
                    lam[k] = xi[k - 1];
                    s += xi[k - 1];
                }
                lam[0] = 1.0 - s;
                double y[3] = {0, 0, 0};
                for (int i = 0; i < D; ++i)
                    for (int k = 0; k <= D; ++k) y[i] += lam[k] * yv[k][i];
                double wgt = wq * J * dfact * volK * poly_eval(sp.w, D, y);
                double fa = sp.test_d >= 0 ? g[ka][sp.test_d] : lam[ka];
                for (int kb = 0; kb <= D; ++kb) {
                    double fb = sp.trial_d >= 0 ? g[kb][sp.trial_d] : lam[kb];
                    row[kb] += wgt * fa * fb;
                }
            }
            for (int kb = 0; kb <= D; ++kb)
                if (slot[kb] >= 0) acc[slot[kb]] += row[kb];
        }
    }
    for (int k = 0; k < W; ++k) vals[k * n + a] = acc[k];
}

static bool g_consts_set = false;

int assemble_spec(sg_problem* P, Factor& f, int spec, int level) {
    if (!g_consts_set) {
        // 4-point Gauss-Legendre on [0,1] (closed forms)
        const double r = sqrt(6.0 / 5.0);
        const double xa = sqrt(3.0 / 7.0 - 2.0 / 7.0 * r), xb = sqrt(3.0 / 7.0 + 2.0 / 7.0 * r);
        const double wa = (18.0 + sqrt(30.0)) / 36.0, wb = (18.0 - sqrt(30.0)) / 36.0;
        double x[4] = {0.5 * (1 - xb), 0.5 * (1 - xa), 0.5 * (1 + xa), 0.5 * (1 + xb)};
        double w[4] = {0.5 * wb, 0.5 * wa, 0.5 * wa, 0.5 * wb};
        SG_CUDA(cudaMemcpyToSymbol(c_gl4_x, x, sizeof(x)));
        SG_CUDA(cudaMemcpyToSymbol(c_gl4_w, w, sizeof(w)));
        g_consts_set = true;
    }
    Level& L = f.lev[level];
    if ((int)L.fm.size() < (int)f.specs.size()) L.fm.resize(f.specs.size(), nullptr);
    if (L.fm[spec]) return SG_OK;
    SG_CUDA(cudaMalloc(&L.fm[spec], sizeof(double) * f.W * L.n));
    const Spec& s = f.specs[spec];
    SpecDev sd;
    sd.kind = s.kind;
    for (int i = 0; i < NPOLY; ++i) sd.w[i] = s.w[i];
    sd.trial_d = s.trial_d; sd.test_d = s.test_d;
    sd.chi_axis = s.chi_axis; sd.chi_sign = s.chi_sign;
    sd.face_axis = s.face_axis; sd.face_sign = s.face_sign;
    const int cells = f.nc << (level - 1);
    double h[3] = {0, 0, 0}, lo[3] = {0, 0, 0};
    for (int i = 0; i < f.d; ++i) {
        h[i] = (f.hi[i] - f.lo[i]) / cells;
        lo[i] = f.lo[i];
    }
    int nb = (int)((L.n + 127) / 128);
    if (f.d == 1)
        k_assemble_row<1><<<nb, 128, 0, P->stream>>>(f.kind, L.n, L.m, L.lat, L.cols, f.W, lo[0], lo[1], lo[2], h[0],
                                                    h[1], h[2], sd, L.fm[spec]);
    else if (f.d == 2)
        k_assemble_row<2><<<nb, 128, 0, P->stream>>>(f.kind, L.n, L.m, L.lat, L.cols, f.W, lo[0], lo[1], lo[2], h[0],
                                                    h[1], h[2], sd, L.fm[spec]);
    else
        k_assemble_row<3><<<nb, 128, 0, P->stream>>>(f.kind, L.n, L.m, L.lat, L.cols, f.W, lo[0], lo[1], lo[2], h[0],
                                                    h[1], h[2], sd, L.fm[spec]);
    P->launches += 1;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

}  // namespace sg
