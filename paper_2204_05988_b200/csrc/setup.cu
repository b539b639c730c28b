// Host-side setup: Kronecker term expansion of A^(delta) and precombined group
// matrices.  PAPER.md sec. 4.2 l.440-504 (this is an independent C++
// implementation of the expansion; reading R1 for the delta on K~).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

#include "sg_internal.cuh"

namespace sg {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

bool Spec::same(const Spec& o) const {
    if (kind != o.kind || trial_d != o.trial_d || test_d != o.test_d || chi_axis != o.chi_axis ||
        chi_sign != o.chi_sign || face_axis != o.face_axis || face_sign != o.face_sign)
        return false;
    for (int i = 0; i < NPOLY; ++i)
        if (w[i] != o.w[i]) return false;
    return true;
}

int Factor::add_spec(const Spec& s) {
    for (size_t i = 0; i < specs.size(); ++i)
        if (specs[i].same(s)) return (int)i;
    specs.push_back(s);
    return (int)specs.size() - 1;
}

// ---- polynomials: [1, y0, y1, y2, y0y0, y0y1, y0y2, y1y1, y1y2, y2y2]
static int qidx(int i, int j) {
    if (i > j) std::swap(i, j);
    static const int tab[3][3] = {{4, 5, 6}, {5, 7, 8}, {6, 8, 9}};
    return tab[i][j];
}
struct Poly {
    double c[NPOLY] = {0};
};
static Poly affine(const double* a, int d) {
    Poly p;
    p.c[0] = a[0];
    for (int i = 0; i < d; ++i) p.c[1 + i] = a[1 + i];
    return p;
}
static Poly pmul(const Poly& p, const Poly& q) {   // deg(p), deg(q) <= 1
    Poly r;
    r.c[0] = p.c[0] * q.c[0];
    for (int i = 0; i < 3; ++i) r.c[1 + i] = p.c[0] * q.c[1 + i] + q.c[0] * p.c[1 + i];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.c[qidx(i, j)] += p.c[1 + i] * q.c[1 + j];
    return r;
}

struct SpaceTerm {
    Spec x, v;
    double coef;
};

static Spec volspec(const Poly& w, int trial, int test) {
    Spec s;
    s.kind = 0;
    for (int i = 0; i < NPOLY; ++i) s.w[i] = w.c[i];
    s.trial_d = trial;
    s.test_d = test;
    return s;
}
static Spec transpose(const Spec& s) {
    Spec t = s;
    if (s.kind == 0) std::swap(t.trial_d, t.test_d);
    return t;
}
// pull the first nonzero weight coefficient out of a vol spec
static double canonical(Spec& s) {
    if (s.kind != 0) return 1.0;
    for (int i = 0; i < NPOLY; ++i)
        if (s.w[i] != 0.0) {
            double c = s.w[i];
            for (int j = 0; j < NPOLY; ++j) s.w[j] /= c;
            return c;
        }
    return 1.0;
}

// inflow weight spec int chi_{w<0} w phi' phi for w = c0 or c*y_i (nullptr if empty)
static int chi_weighted(const Poly& w, int d, Spec* out) {
    int nlin = 0, li = -1;
    for (int i = 0; i < d; ++i)
        if (w.c[1 + i] != 0.0) {
            nlin++;
            li = i;
        }
    for (int k = 4; k < NPOLY; ++k)
        if (w.c[k] != 0.0) return SG_ERR_UNSUPPORTED;
    if (nlin == 0) {
        if (w.c[0] < 0.0) {
            *out = volspec(w, -1, -1);
            return 1;
        }
        return 0;
    }
    if (nlin > 1 || w.c[0] != 0.0) return SG_ERR_UNSUPPORTED;
    Spec s = volspec(w, -1, -1);
    s.chi_axis = li;
    s.chi_sign = w.c[1 + li] > 0 ? -1 : 1;   // c*y<0 <=> (-sign c) y > 0
    *out = s;
    return 1;
}

int expand_terms(sg_problem* P) {
    const sg_config& c = P->cfg;
    const int d = c.d, S = P->S;
    const double tau = c.tau, dl = P->delta, sig = c.sigma;
    Poly one;
    one.c[0] = 1.0;
    std::vector<SpaceTerm> M, T, TT, C, G;
    M.push_back({volspec(one, -1, -1), volspec(one, -1, -1), 1.0});
    for (int r = 0; r < c.nbeta; ++r) {
        const sg_beta_term& b = c.beta[r];
        Poly a = affine(b.a, d), bb = affine(b.b, d);
        if (b.axis < d)
            T.push_back({volspec(a, b.axis, -1), volspec(bb, -1, -1), 1.0});
        else
            T.push_back({volspec(a, -1, -1), volspec(bb, b.axis - d, -1), 1.0});
    }
    for (auto& t : T) TT.push_back({transpose(t.x), transpose(t.v), t.coef});
    for (int r = 0; r < c.nbeta; ++r)
        for (int r2 = 0; r2 < c.nbeta; ++r2) {
            const sg_beta_term &b1 = c.beta[r], &b2 = c.beta[r2];
            Poly ax = pmul(affine(b1.a, d), affine(b2.a, d));
            Poly bv = pmul(affine(b1.b, d), affine(b2.b, d));
            int xd1 = b1.axis < d ? b1.axis : -1, xd2 = b2.axis < d ? b2.axis : -1;
            int vd1 = b1.axis >= d ? b1.axis - d : -1, vd2 = b2.axis >= d ? b2.axis - d : -1;
            C.push_back({volspec(ax, xd1, xd2), volspec(bv, vd1, vd2), 1.0});
        }
    // inflow boundary G^r (eq. (14) l.459, factorised per face as in l.706-716)
    for (int ax = 0; ax < 2 * d; ++ax) {
        int cnt = 0, r = -1;
        for (int k = 0; k < c.nbeta; ++k)
            if (c.beta[k].axis == ax) {
                cnt++;
                r = k;
            }
        if (cnt == 0) continue;
        if (cnt > 1) {
            set_error("inflow factorisation supports one beta term per axis");
            return SG_ERR_UNSUPPORTED;
        }
        Poly a = affine(c.beta[r].a, d), b = affine(c.beta[r].b, d);
        for (int s = -1; s <= 1; s += 2) {
            Spec face;
            face.kind = 1;
            face.face_axis = ax < d ? ax : ax - d;
            face.face_sign = s;
            if (ax < d) {
                for (int i = 0; i < d; ++i)
                    if (a.c[1 + i] != 0.0) {
                        set_error("inflow: a(x) must be constant on x faces");
                        return SG_ERR_UNSUPPORTED;
                    }
                Poly w;
                for (int i = 0; i < NPOLY; ++i) w.c[i] = s * a.c[0] * b.c[i];
                Spec vs;
                int rc = chi_weighted(w, d, &vs);
                if (rc < 0 || rc > 1) return SG_ERR_UNSUPPORTED;
                if (rc == 1) G.push_back({face, vs, 1.0});
            } else {
                for (int i = 0; i < d; ++i)
                    if (b.c[1 + i] != 0.0) {
                        set_error("inflow: b(v) must be constant on v faces");
                        return SG_ERR_UNSUPPORTED;
                    }
                Poly w;
                for (int i = 0; i < NPOLY; ++i) w.c[i] = s * b.c[0] * a.c[i];
                Spec xs;
                int rc = chi_weighted(w, d, &xs);
                if (rc < 0 || rc > 1) return SG_ERR_UNSUPPORTED;
                if (rc == 1) G.push_back({xs, face, 1.0});
            }
        }
    }
    // time blocks, Legendre basis on the strip (closed forms)
    double Mt[4] = {0}, Tt[4] = {0}, Ct[4] = {0}, Gt[4] = {0};
    if (S == 1) {
        Mt[0] = tau;
        Gt[0] = 1.0;
    } else {
        Mt[0] = tau;
        Mt[3] = tau / 3.0;
        Tt[1] = 2.0;                 // int P1' P0 dxi (row s=0 test, col s'=1 trial)
        Ct[3] = 2.0 / tau * 2.0;     // (2/tau) int P1' P1' dxi
        Gt[0] = 1.0; Gt[1] = -1.0; Gt[2] = -1.0; Gt[3] = 1.0;
    }
    auto tr = [&](const double* A, double* B) {
        for (int i = 0; i < S; ++i)
            for (int j = 0; j < S; ++j) B[i * S + j] = A[j * S + i];
    };
    double TtT[4];
    tr(Tt, TtT);
    struct Acc {
        Spec x, v;
        double T[4];
    };
    std::vector<Acc> acc;
    auto add = [&](const double* Tb, double scale, const std::vector<SpaceTerm>& lst) {
        for (const auto& st : lst) {
            Spec xs = st.x, vs = st.v;
            double cx = canonical(xs), cv = canonical(vs);
            double f = scale * st.coef * cx * cv;
            int found = -1;
            for (size_t i = 0; i < acc.size(); ++i)
                if (acc[i].x.same(xs) && acc[i].v.same(vs)) found = (int)i;
            if (found < 0) {
                Acc a;
                a.x = xs;
                a.v = vs;
                for (int i = 0; i < 4; ++i) a.T[i] = 0.0;
                acc.push_back(a);
                found = (int)acc.size() - 1;
            }
            for (int i = 0; i < S * S; ++i) acc[found].T[i] += f * Tb[i];
        }
    };
    double A0[4];
    for (int i = 0; i < S * S; ++i) A0[i] = Tt[i] + dl * Ct[i] + Gt[i];
    add(A0, 1.0, M);             // (T^t + delta C^t) (x) M  +  G^t (x) M
    add(Tt, dl, TT);             // delta T^t (x) (T^r)^T
    add(TtT, dl, T);             // delta (T^t)^T (x) T^r
    add(TtT, dl * sig, M);       // delta (T^t)^T (x) K^r
    add(Mt, 1.0, T);             // M^t (x) T^r
    add(Mt, dl, C);              // M^t (x) delta C^r
    add(Mt, sig, M);             // M^t (x) K^r
    add(Mt, dl * sig, TT);       // M^t (x) delta K~^r  (reading R1)
    add(Mt, -1.0, G);            // M^t (x) (-G^r)
    P->terms.clear();
    for (auto& a : acc) {
        bool nz = false;
        for (int i = 0; i < S * S; ++i) nz |= (a.T[i] != 0.0);
        if (!nz) continue;
        Term t;
        for (int i = 0; i < 4; ++i) t.T[i] = a.T[i];
        t.xs = P->fx.add_spec(a.x);
        t.vs = P->fv.add_spec(a.v);
        P->terms.push_back(t);
    }
    Spec mx = volspec(one, -1, -1);
    P->mass_x = P->fx.add_spec(mx);
    P->mass_v = P->fv.add_spec(mx);
    // groups
    P->vgroups.clear();
    P->xgroups.clear();
    for (size_t t = 0; t < P->terms.size(); ++t) {
        const Term& tm = P->terms[t];
        int gv = -1, gx = -1;
        for (size_t g = 0; g < P->vgroups.size(); ++g)
            if (P->vgroups[g].spec == tm.vs) gv = (int)g;
        if (gv < 0) {
            Group g;
            g.spec = tm.vs;
            P->vgroups.push_back(g);
            gv = (int)P->vgroups.size() - 1;
        }
        P->vgroups[gv].terms.push_back((int)t);
        for (size_t g = 0; g < P->xgroups.size(); ++g)
            if (P->xgroups[g].spec == tm.xs) gx = (int)g;
        if (gx < 0) {
            Group g;
            g.spec = tm.xs;
            P->xgroups.push_back(g);
            gx = (int)P->xgroups.size() - 1;
        }
        P->xgroups[gx].terms.push_back((int)t);
    }
    return SG_OK;
}

// out = sum_i coef_i * in_i over ELL value arrays of equal size
__global__ void k_lincomb(int64_t n, int k, const double* const* in, const double* coef, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double a = 0.0;
        for (int j = 0; j < k; ++j) a += coef[j] * in[j][i];
        out[i] = a;
    }
}

// Combined matrices of a group on every level of the OTHER factor:
// comb[l] = { (s, s', sum_{t in group} T_t[s,s'] * A_{other spec of t}^l) }
int combine_group(sg_problem* P, Group& g, bool other_is_x) {
    Factor& f = other_is_x ? P->fx : P->fv;
    const int S = P->S;
    g.comb.assign(P->F + 1, {});
    for (int l = 1; l <= P->F; ++l) {
        Level& L = f.lev[l];
        const int64_t nn = (int64_t)f.W * L.n;
        for (int s = 0; s < S; ++s)
            for (int sp = 0; sp < S; ++sp) {
                std::vector<const double*> ptrs;
                std::vector<double> cf;
                for (int t : g.terms) {
                    const Term& tm = P->terms[t];
                    double v = tm.T[s * S + sp];
                    if (v == 0.0) continue;
                    int spec = other_is_x ? tm.xs : tm.vs;
                    SG_TRY(assemble_spec(P, f, spec, l));
                    ptrs.push_back(L.fm[spec]);
                    cf.push_back(v);
                }
                if (ptrs.empty()) continue;
                CombEntry ce;
                ce.s_out = s;
                ce.s_in = sp;
                SG_CUDA(cudaMalloc(&ce.vals, sizeof(double) * nn));
                const double** dptr;
                double* dcf;
                SG_CUDA(cudaMalloc(&dptr, sizeof(double*) * ptrs.size()));
                SG_CUDA(cudaMalloc(&dcf, sizeof(double) * cf.size()));
                SG_CUDA(cudaMemcpyAsync(dptr, ptrs.data(), sizeof(double*) * ptrs.size(), cudaMemcpyHostToDevice,
                                        P->stream));
                SG_CUDA(cudaMemcpyAsync(dcf, cf.data(), sizeof(double) * cf.size(), cudaMemcpyHostToDevice,
                                        P->stream));
                int nb = (int)std::min<int64_t>((nn + 255) / 256, 148 * 32);
                k_lincomb<<<nb, 256, 0, P->stream>>>(nn, (int)ptrs.size(), dptr, dcf, ce.vals);
                P->launches++;
                SG_CUDA(cudaGetLastError());
                SG_CUDA(cudaStreamSynchronize(P->stream));
                cudaFree(dptr);
                cudaFree(dcf);
                g.comb[l].push_back(ce);
            }
    }
    return SG_OK;
}

}  // namespace sg
