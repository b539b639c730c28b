// Shared definitions of the shifted-moment v-side (vmoment.cu, fused whole-x kernel in xfanin.cu).
#pragma once
#include "sg_internal.cuh"

namespace sg {

namespace vm {
// NPOLY monomial slots [1, y0, y1, y2, y0y0, y0y1, y0y2, y1y1, y1y2, y2y2]
__host__ __device__ constexpr int mono_ax(int n, int which) {   // axes of monomial n (-1 none)
    return n == 0 ? -1
         : n <= 3 ? (which == 0 ? n - 1 : -1)
         : n == 4 ? 0 : n == 5 ? (which == 0 ? 0 : 1) : n == 6 ? (which == 0 ? 0 : 2)
         : n == 7 ? 1 : n == 8 ? (which == 0 ? 1 : 2) : 2;
}
__host__ __device__ constexpr int mono_deg(int n) { return n == 0 ? 0 : (n <= 3 ? 1 : 2); }
__host__ __device__ constexpr int lin(int i) { return 1 + i; }
__host__ __device__ constexpr int quad(int i, int j) {
    return i > j ? quad(j, i) : (i == 0 ? 4 + j : (i == 1 ? 6 + j : 9));
}
__host__ __device__ constexpr bool mono_in(int D, int n) {   // monomial uses only axes < D
    return mono_deg(n) == 0 || (mono_ax(n, 0) < D && (mono_deg(n) == 1 || mono_ax(n, 1) < D));
}
}  // namespace vm

constexpr int VM_NP = 10;
constexpr int VM_NC = 6;   // inflow (chi-weighted) groups
struct VmOut {
    double* p[VM_NP];   // output (group buffer) per monomial slot, nullptr if absent
    double* pc[VM_NC];  // outputs of the chi-weighted groups (x-boundary rows only)
};
struct VmCoef {
    double R[VM_NP][15];   // interior-class shifted-moment stencils
    double H[VM_NC][15];   // interior-class half stencils of the chi groups (rows on the plane y_i = 0)
    int off[15];           // lattice offsets of the Kuhn stencil
    int nchi;
    int chax[VM_NC], chkeep[VM_NC];   // chi group: weight y_i chi(keep * y_i > 0)
};

void vmom_coef(const sg_problem* P, int l2, VmCoef* cf, double* lo, double* h);

}  // namespace sg
