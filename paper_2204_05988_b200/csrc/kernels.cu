// Kronecker-factored sparse applies along one factor of a block [S][n1][n2]
// ((S^t x Id x Id)(Id x S^1 x Id)(Id x Id x S^2) u).
//
//  fanout<DIR>: one input, NO outputs, no time mixing
//      out_o[s][r][c] = sum_k M_o[k][row] * in[s][...col_k...]
//  gather<DIR>: NE (input, matrix, scale, s_out, s_in) entries, one output
//      out[s] = beta*out[s] + sum_{e: s_out=s} scale_e * (M_e along DIR) in_e[s_in]
//
// DIR = 1 acts on the fastest (v) index: M is n2_out x n2_in, row = c;
// DIR = 0 acts on the middle (x) index:  M is n1_out x n1_in, row = r.
// Matrices are column-major ELL: vals[k * nrows + row], cols[k * nrows + row]
// (-1 padded, value 0).  Threads are flattened over (r, c) with c fastest so
// every warp reads consecutive c (coalesced rows of the block).
#include "sg_internal.cuh"

namespace sg {

template <int DIR, int W, int NO>
__global__ void __launch_bounds__(256) k_fanout(int S, int64_t n1, int64_t n2_in, int64_t n1_out, int64_t n2_out,
                                                const int32_t* __restrict__ cols, const double* __restrict__ in,
                                                FanoutList fl, int o0) {
    const int64_t per_s = n1_out * n2_out;
    const int64_t total = per_s * S;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t / per_s);
        const int64_t rc = t - s * per_s;
        const int64_t r = rc / n2_out;
        const int64_t c = rc - r * n2_out;
        double x[W];
        int64_t row;
        int64_t nrows;
        if (DIR == 1) {
            row = c; nrows = n2_out;
            const double* base = in + ((int64_t)s * n1 + r) * n2_in;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                int32_t col = __ldg(cols + k * nrows + row);
                x[k] = col >= 0 ? __ldg(base + col) : 0.0;
            }
        } else {
            row = r; nrows = n1_out;
            const double* base = in + (int64_t)s * n1 * n2_in + c;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                int32_t col = __ldg(cols + k * nrows + row);
                x[k] = col >= 0 ? __ldg(base + (int64_t)col * n2_in) : 0.0;
            }
        }
#pragma unroll
        for (int o = 0; o < NO; ++o) {
            const double* v = fl.vals[o0 + o];
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) acc = fma(__ldg(v + k * nrows + row), x[k], acc);
            fl.out[o0 + o][t] = acc;
        }
    }
}

template <int DIR, int W>
__global__ void __launch_bounds__(256) k_gather(int S_out, int64_t n1_in, int64_t n2_in, int64_t n1_out,
                                                int64_t n2_out, const int32_t* __restrict__ cols, EntryList el,
                                                double* __restrict__ out, double beta) {
    const int64_t per_s = n1_out * n2_out;
    const int64_t total = per_s * S_out;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t / per_s);
        const int64_t rc = t - s * per_s;
        const int64_t r = rc / n2_out;
        const int64_t c = rc - r * n2_out;
        const int64_t nrows = DIR == 1 ? n2_out : n1_out;
        const int64_t row = DIR == 1 ? c : r;
        int32_t cl[W];
#pragma unroll
        for (int k = 0; k < W; ++k) cl[k] = __ldg(cols + k * nrows + row);
        double acc = 0.0;
        for (int e = 0; e < el.ne; ++e) {
            if (el.e[e].s_out != s) continue;
            const double* v = el.e[e].vals;
            const double* base;
            if (DIR == 1)
                base = el.e[e].in + ((int64_t)el.e[e].s_in * n1_in + r) * n2_in;
            else
                base = el.e[e].in + (int64_t)el.e[e].s_in * n1_in * n2_in + c;
            double a2 = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                if (cl[k] < 0) continue;
                const double xv = DIR == 1 ? __ldg(base + cl[k]) : __ldg(base + (int64_t)cl[k] * n2_in);
                a2 = fma(__ldg(v + k * nrows + row), xv, a2);
            }
            acc = fma(el.e[e].scale, a2, acc);
        }
        out[t] = beta == 0.0 ? acc : fma(beta, out[t], acc);
    }
}

static int grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    if (b > 148 * 64) b = 148 * 64;
    if (b < 1) b = 1;
    return (int)b;
}

template <int DIR, int W>
static void fanout_dispatch(sg_problem* P, int S, int64_t n1_in, int64_t n2_in, int64_t n1_out, int64_t n2_out,
                            const int32_t* cols, const double* in, const FanoutList& fl) {
    const int64_t total = (int64_t)S * n1_out * n2_out;
    const int g = grid_for(total);
    int o = 0;
    while (o < fl.no) {
        int left = fl.no - o;
        if (left >= 4) {
            k_fanout<DIR, W, 4><<<g, 256, 0, P->stream>>>(S, n1_in, n2_in, n1_out, n2_out, cols, in, fl, o);
            o += 4;
        } else if (left >= 2) {
            k_fanout<DIR, W, 2><<<g, 256, 0, P->stream>>>(S, n1_in, n2_in, n1_out, n2_out, cols, in, fl, o);
            o += 2;
        } else {
            k_fanout<DIR, W, 1><<<g, 256, 0, P->stream>>>(S, n1_in, n2_in, n1_out, n2_out, cols, in, fl, o);
            o += 1;
        }
        P->launches++;
    }
}

int launch_fanout(sg_problem* P, int dir, int W, int S, int64_t n1_in, int64_t n2_in, int64_t nrows_out,
                  const int32_t* cols, const double* in, const FanoutList& fl) {
    const int64_t n1_out = dir == 0 ? nrows_out : n1_in;
    const int64_t n2_out = dir == 1 ? nrows_out : n2_in;
    if (n1_out * n2_out == 0 || fl.no == 0) return SG_OK;
#define FO(D, WW) fanout_dispatch<D, WW>(P, S, n1_in, n2_in, n1_out, n2_out, cols, in, fl)
    if (dir == 1) {
        if (W == 3) FO(1, 3); else if (W == 7) FO(1, 7); else if (W == 15) FO(1, 15); else if (W == 2) FO(1, 2);
        else return SG_ERR_ARG;
    } else {
        if (W == 3) FO(0, 3); else if (W == 7) FO(0, 7); else if (W == 15) FO(0, 15); else if (W == 2) FO(0, 2);
        else return SG_ERR_ARG;
    }
#undef FO
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

int launch_gather(sg_problem* P, int dir, int W, int S_out, int64_t n1_in, int64_t n2_in, int64_t nrows_out,
                  const int32_t* cols, const EntryList& el, double* out, double beta) {
    const int64_t n1_out = dir == 0 ? nrows_out : n1_in;
    const int64_t n2_out = dir == 1 ? nrows_out : n2_in;
    const int64_t total = (int64_t)S_out * n1_out * n2_out;
    if (total == 0) return SG_OK;
    const int g = grid_for(total);
#define GA(D, WW) k_gather<D, WW><<<g, 256, 0, P->stream>>>(S_out, n1_in, n2_in, n1_out, n2_out, cols, el, out, beta)
    if (dir == 1) {
        if (W == 3) GA(1, 3); else if (W == 7) GA(1, 7); else if (W == 15) GA(1, 15); else if (W == 2) GA(1, 2);
        else return SG_ERR_ARG;
    } else {
        if (W == 3) GA(0, 3); else if (W == 7) GA(0, 7); else if (W == 15) GA(0, 15); else if (W == 2) GA(0, 2);
        else return SG_ERR_ARG;
    }
#undef GA
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

// ---------------------------------------------------------------- vectors
__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = (b == 0.0 ? 0.0 : b * y[i]) + a * x[i];
}
__global__ void k_fill(int64_t n, double v, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = v;
}

int launch_axpby(sg_problem* P, int64_t n, double a, const double* x, double b, double* y) {
    if (n == 0) return SG_OK;
    k_axpby<<<grid_for(n), 256, 0, P->stream>>>(n, a, x, b, y);
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}
int launch_copy(sg_problem* P, int64_t n, const double* x, double* y) {
    if (n == 0) return SG_OK;
    SG_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, P->stream));
    return SG_OK;
}
int launch_zero(sg_problem* P, int64_t n, double* y) {
    if (n == 0) return SG_OK;
    SG_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * n, P->stream));
    return SG_OK;
}

}  // namespace sg
