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
#include <algorithm>
#include <cstdlib>

#include "sg_internal.cuh"

namespace sg {

// (index arithmetic in 32 bits: every caller has S * n1 * n2 < 2^31 and S <= 2, checked on the host)
template <int DIR, int W, int NO>
__global__ void __launch_bounds__(256) k_fanout(int S, int64_t n1, int64_t n2_in, int64_t n1_out, int64_t n2_out,
                                                const int32_t* __restrict__ cols, const double* __restrict__ in,
                                                FanoutList fl, int o0, const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    const unsigned per_s = (unsigned)(n1_out * n2_out);
    const unsigned total = per_s * (unsigned)S;
    const unsigned n2o = (unsigned)n2_out;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int s = t >= per_s ? 1 : 0;
        const unsigned rc = t - s * per_s;
        const int64_t r = rc / n2o;
        const int64_t c = rc - (unsigned)r * n2o;
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
                                                int64_t n2_out, const int32_t* __restrict__ cols,
                                                const __grid_constant__ EntryList el, double* __restrict__ out,
                                                double beta, const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    const unsigned per_s = (unsigned)(n1_out * n2_out);
    const unsigned total = per_s * (unsigned)S_out;
    const unsigned n2o = (unsigned)n2_out;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int s = t >= per_s ? 1 : 0;
        const unsigned rc = t - s * per_s;
        const int64_t r = rc / n2o;
        const int64_t c = rc - (unsigned)r * n2o;
        const int64_t nrows = DIR == 1 ? n2_out : n1_out;
        const int64_t row = DIR == 1 ? c : r;
        int32_t cl[W];
#pragma unroll
        for (int k = 0; k < W; ++k) cl[k] = __ldg(cols + k * nrows + row);
        double acc = 0.0;
        for (int e = el.sbeg[s]; e < el.sbeg[s + 1]; ++e) {
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

// x-side gather for S_out = 2 (dG(1)): one thread produces both time components of (r, c), and
// entries sharing an input (same group and s_in, consecutive after the host sort) reuse the W
// loaded values, so every intermediate value is read once per output node instead of S_out times.
template <int W>
__global__ void __launch_bounds__(256) k_gather_s2(int64_t n1_in, int64_t n2_in, int64_t n1_out,
                                                   const int32_t* __restrict__ cols,
                                                   const __grid_constant__ EntryList el, double* __restrict__ out,
                                                   double beta, const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    const unsigned n2o = (unsigned)n2_in;
    const unsigned per_s = (unsigned)(n1_out * n2_in);
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < per_s; t += gridDim.x * blockDim.x) {
        const unsigned r = t / n2o, c = t - r * n2o;
        int32_t cl[W];
#pragma unroll
        for (int k = 0; k < W; ++k) cl[k] = __ldg(cols + (size_t)k * n1_out + r);
        double acc0 = 0.0, acc1 = 0.0;
        double xv[W];
        const double* prev = nullptr;
        int prev_s = -1;
        for (int e = 0; e < el.ne; ++e) {
            const Entry& E = el.e[e];
            if (E.in != prev || E.s_in != prev_s) {
                prev = E.in;
                prev_s = E.s_in;
                const double* base = E.in + (size_t)E.s_in * n1_in * n2_in + c;
#pragma unroll
                for (int k = 0; k < W; ++k) xv[k] = cl[k] >= 0 ? __ldg(base + (size_t)cl[k] * n2_in) : 0.0;
            }
            const double* v = E.vals;
            double a2 = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (cl[k] >= 0) a2 = fma(__ldg(v + (size_t)k * n1_out + r), xv[k], a2);
            if (E.s_out == 0) acc0 = fma(E.scale, a2, acc0);
            else acc1 = fma(E.scale, a2, acc1);
        }
        double* y0 = out + t;
        double* y1 = out + per_s + t;
        *y0 = beta == 0.0 ? acc0 : fma(beta, *y0, acc0);
        *y1 = beta == 0.0 ? acc1 : fma(beta, *y1, acc1);
    }
}

// ... the same with CPT columns per thread (columns lane, lane + 32, ... of a 32*CPT-wide tile): a warp
// works on ONE row r, so every coefficient load (warp-uniform broadcast) feeds CPT multiply-adds
// and the pattern row is read once per warp tile.
template <int W, int CPT, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_gather_s2c(int64_t n1_in, int64_t n2_in, int64_t n1_out,
                                                    const int32_t* __restrict__ cols,
                                                    const __grid_constant__ EntryList el, double* __restrict__ out,
                                                    double beta, int ncoltiles, const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    const int lane = threadIdx.x & 31;
    // block = 8 consecutive rows x one column tile: neighbouring rows share their sources through L1
    const long long nrb = (n1_out + 7) / 8, nblk = nrb * ncoltiles;
    const size_t per_in = (size_t)n1_in * n2_in, per_out = (size_t)n1_out * n2_in;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int ct = (int)(blk % ncoltiles);
        const long long rr = (blk / ncoltiles) * 8 + (threadIdx.x >> 5);
        if (rr >= n1_out) continue;
        const int r = (int)rr;
        int32_t cl[W];
#pragma unroll
        for (int k = 0; k < W; ++k) cl[k] = __ldg(cols + (size_t)k * n1_out + r);
        int c[CPT];
        bool cv[CPT];
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            c[j] = ct * 32 * CPT + j * 32 + lane;
            cv[j] = c[j] < n2_in;
            if (!cv[j]) c[j] = 0;
        }
        double acc0[CPT], acc1[CPT], xv[W][CPT];
#pragma unroll
        for (int j = 0; j < CPT; ++j) acc0[j] = acc1[j] = 0.0;
        const double* prev = nullptr;
        int prev_s = -1;
        for (int e = 0; e < el.ne; ++e) {
            const Entry& E = el.e[e];
            if (E.in != prev || E.s_in != prev_s) {
                prev = E.in;
                prev_s = E.s_in;
                const double* base = E.in + (size_t)E.s_in * per_in;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const double* row = base + (size_t)(cl[k] >= 0 ? cl[k] : 0) * n2_in;
#pragma unroll
                    for (int j = 0; j < CPT; ++j) xv[k][j] = cl[k] >= 0 ? __ldg(row + c[j]) : 0.0;
                }
            }
            const double* v = E.vals + r;
            double a2[CPT];
#pragma unroll
            for (int j = 0; j < CPT; ++j) a2[j] = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const double cf = __ldg(v + (size_t)k * n1_out);   // (zero where the neighbour is absent)
#pragma unroll
                for (int j = 0; j < CPT; ++j) a2[j] = fma(cf, xv[k][j], a2[j]);
            }
            if (E.s_out == 0) {
#pragma unroll
                for (int j = 0; j < CPT; ++j) acc0[j] = fma(E.scale, a2[j], acc0[j]);
            } else {
#pragma unroll
                for (int j = 0; j < CPT; ++j) acc1[j] = fma(E.scale, a2[j], acc1[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            if (!cv[j]) continue;
            double* y0 = out + (size_t)r * n2_in + c[j];
            double* y1 = y0 + per_out;
            *y0 = beta == 0.0 ? acc0[j] : fma(beta, *y0, acc0[j]);
            *y1 = beta == 0.0 ? acc1[j] : fma(beta, *y1, acc1[j]);
        }
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
            k_fanout<DIR, W, 4><<<g, 256, 0, P->stream>>>(S, n1_in, n2_in, n1_out, n2_out, cols, in, fl, o, P->skip);
            o += 4;
        } else if (left >= 2) {
            k_fanout<DIR, W, 2><<<g, 256, 0, P->stream>>>(S, n1_in, n2_in, n1_out, n2_out, cols, in, fl, o, P->skip);
            o += 2;
        } else {
            k_fanout<DIR, W, 1><<<g, 256, 0, P->stream>>>(S, n1_in, n2_in, n1_out, n2_out, cols, in, fl, o, P->skip);
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
    if ((int64_t)S * n1_out * n2_out >= (1LL << 31) || S > 2) {
        set_error("fanout too large for 32-bit indexing");
        return SG_ERR_UNSUPPORTED;
    }
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
                  const int32_t* cols, const EntryList& el_in, double* out, double beta) {
    // entries grouped by output time component (each thread only walks its own s_out)
    EntryList el;
    el.ne = 0;
    for (int s = 0; s < S_out && s < 2; ++s) {
        el.sbeg[s] = el.ne;
        for (int e = 0; e < el_in.ne; ++e)
            if (el_in.e[e].s_out == s) el.e[el.ne++] = el_in.e[e];
    }
    for (int s = std::min(S_out, 2); s <= 2; ++s) el.sbeg[s] = el.ne;
    if (dir == 0 && S_out == 2 && n1_in * n2_in < (1LL << 31) && nrows_out * n2_in < (1LL << 31)) {
        // sort by (input, s_in) so that entries sharing an input are adjacent
        EntryList es;
        es.ne = el_in.ne;
        for (int e = 0; e < el_in.ne; ++e) es.e[e] = el_in.e[e];
        std::stable_sort(es.e, es.e + es.ne, [](const Entry& a, const Entry& b) {
            return a.in != b.in ? a.in < b.in : a.s_in < b.s_in;
        });
        es.sbeg[0] = es.sbeg[1] = es.sbeg[2] = 0;
        if (W == 7 && n2_in >= 128) {   // (narrower grids: the flattened kernel below measured faster)
            // several columns per thread: one coefficient load per CPT multiply-adds
            // 4 columns per thread unless the 128-column tiles would pad the rows by more than 6 %
            // (two CTAs per SM at 128 registers: (6,5) 1.56 -> 1.29 ms, profiles/r2z)
            const int64_t pad4 = (n2_in + 127) / 128 * 128;
            const int cpt = pad4 * 100 <= n2_in * 106 ? 4 : 2;
            const int64_t nct = (n2_in + 32 * cpt - 1) / (32 * cpt);
            const int64_t nblk = std::min<int64_t>((nrows_out + 7) / 8 * nct, 148 * 64);
            if (cpt == 4)
                k_gather_s2c<7, 4, 2><<<(unsigned)nblk, 256, 0, P->stream>>>(n1_in, n2_in, nrows_out, cols, es, out, beta,
                                                                             (int)nct, P->skip);
            else
                k_gather_s2c<7, 2, 2><<<(unsigned)nblk, 256, 0, P->stream>>>(n1_in, n2_in, nrows_out, cols, es, out, beta,
                                                                             (int)nct, P->skip);
            P->launches++;
            SG_CUDA(cudaGetLastError());
            return SG_OK;
        }
        const int g = grid_for(nrows_out * n2_in);
#define GS2(WW) k_gather_s2<WW><<<g, 256, 0, P->stream>>>(n1_in, n2_in, nrows_out, cols, es, out, beta, P->skip)
        if (W == 3) GS2(3); else if (W == 7) GS2(7); else if (W == 15) GS2(15); else if (W == 2) GS2(2);
        else return SG_ERR_ARG;
#undef GS2
        P->launches++;
        SG_CUDA(cudaGetLastError());
        return SG_OK;
    }
    const int64_t n1_out = dir == 0 ? nrows_out : n1_in;
    const int64_t n2_out = dir == 1 ? nrows_out : n2_in;
    const int64_t total = (int64_t)S_out * n1_out * n2_out;
    if (total == 0) return SG_OK;
    if (total >= (1LL << 31) || S_out > 2) {
        set_error("gather too large for 32-bit indexing");
        return SG_ERR_UNSUPPORTED;
    }
    const int g = grid_for(total);
#define GA(D, WW) k_gather<D, WW><<<g, 256, 0, P->stream>>>(S_out, n1_in, n2_in, n1_out, n2_out, cols, el, out, beta, P->skip)
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
struct SumList {
    int k;
    const double* x[MAX_SUM];
};
__global__ void k_sum_into(int64_t n, SumList sl, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = y[i];
        for (int j = 0; j < sl.k; ++j) v += sl.x[j][i];
        y[i] = v;
    }
}
// y += sum_j xs[j]
int launch_sum_into(sg_problem* P, int64_t n, int k, double* const* xs, double* y) {
    if (k > MAX_SUM) return SG_ERR_UNSUPPORTED;
    SumList sl;
    sl.k = k;
    for (int j = 0; j < k; ++j) sl.x[j] = xs[j];
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_sum_into<<<blocks, 256, 0, P->stream>>>(n, sl, y);
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

int launch_zero(sg_problem* P, int64_t n, double* y) {
    if (n == 0) return SG_OK;
    SG_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * n, P->stream));
    return SG_OK;
}



// =====================================================================
// Stencil-format kernels for box-lattice factors (v2 hot path).
//
// On a box lattice numbered lexicographically, the Kuhn P1 neighbours of
// node i are i + off_k with 2^(d+1)-1 constant offsets (d = 1: 3, d = 2: 7,
// d = 3: 15); sorted ascending they form runs of consecutive integers
// ("bands": d = 1: {3}; d = 2: {2,3,2}; d = 3: {2,2,2,3,2,2,2}).  A factor
// matrix is stored as st[k][i] = A[i, i + off_k] (0 where the neighbour is
// absent).  Sharing the band loads between T consecutive target rows cuts the
// loads per output from W to about (W + 2 * bands * ...) / T.
// =====================================================================
namespace stc {
template <int D> struct Bands;
template <> struct Bands<1> {
    static constexpr int NB = 1, W = 3;
    __host__ __device__ static constexpr int lo(int) { return 0; }
    __host__ __device__ static constexpr int len(int) { return 3; }
};
template <> struct Bands<2> {
    static constexpr int NB = 3, W = 7;
    __host__ __device__ static constexpr int lo(int b) { return b == 0 ? 0 : (b == 1 ? 2 : 5); }
    __host__ __device__ static constexpr int len(int b) { return b == 1 ? 3 : 2; }
};
template <> struct Bands<3> {
    static constexpr int NB = 7, W = 15;
    __host__ __device__ static constexpr int lo(int b) { return b < 3 ? 2 * b : (b == 3 ? 6 : 9 + 2 * (b - 4)); }
    __host__ __device__ static constexpr int len(int b) { return b == 3 ? 3 : 2; }
};
}  // namespace stc

__global__ void k_ell_to_stencil(int64_t n, int W, const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                 StencilOff so, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v[15];
    for (int k = 0; k < W; ++k) v[k] = 0.0;
    for (int e = 0; e < W; ++e) {
        int32_t c = cols[e * n + i];
        if (c < 0) continue;
        int64_t off = (int64_t)c - i;
        for (int k = 0; k < W; ++k)
            if (so.off[k] == off) v[k] += vals[e * n + i];
    }
    for (int k = 0; k < W; ++k) out[k * n + i] = v[k];
}

int launch_ell_to_stencil(sg_problem* P, int64_t n, int W, const int32_t* cols, const double* vals,
                          const StencilOff& so, double* out) {
    k_ell_to_stencil<<<(int)((n + 255) / 256), 256, 0, P->stream>>>(n, W, cols, vals, so, out);
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

// Pass 1 (v side): Z_g[row][a] = sum_k Bst_g[k][a] X[row][a + off_k] for all groups g,
// row = (s, j) over S*n1 rows.  Block = 64 columns x 4 row lanes; the block's
// coefficients live in shared memory [g][k][64] and are reused for all rows
// of the block; each thread handles R rows at a time (registers).  Groups with
// index >= ng_int are only needed on x-boundary rows (face terms).
constexpr int VF_TC = 32;   // columns per block
constexpr int VF_RL = 8;    // row lanes per block
template <int D, int R, int MINB = 2, int NGI = 0>
__global__ void __launch_bounds__(VF_TC * VF_RL, MINB) k_vfan_st(int64_t nrows, int64_t n1, int64_t n2, StencilOff so,
                                                              const uint8_t* __restrict__ xflag, VfanParams vp,
                                                              const double* __restrict__ X, int64_t rows_per_block,
                                                              int64_t opitch, const double* __restrict__ skip,
                                                              int64_t c0, int64_t c1, int maskmode) {
    // columns [c0, c1) only (L2-resident column chunks); output column a - c0.
    // xflag[row]: maskmode 0: non-zero on x-boundary rows (all boundary-only groups computed there);
    // maskmode 1: bit j set when boundary-only group ng_int + j is needed on this row
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    constexpr int W = stc::Bands<D>::W;
    extern __shared__ double sm[];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t a = c0 + blockIdx.x * VF_TC + tx;
    const bool aval = a < c1;
    const int tot = vp.ng * W * VF_TC;
    for (int idx = ty * VF_TC + tx; idx < tot; idx += VF_TC * VF_RL) {
        const int g = idx / (W * VF_TC), rem = idx - g * W * VF_TC, k = rem / VF_TC, c = rem - k * VF_TC;
        const int64_t ac = c0 + blockIdx.x * VF_TC + c;
        sm[idx] = ac < c1 ? __ldg(vp.vst[g] + k * n2 + ac) : 0.0;
    }
    __syncthreads();
    // X is addressed as uniform base + 32-bit byte offset (nrows * n2 * 8 < 2^32 checked on the host):
    // one integer add per load instead of a 64-bit address computation
    uint32_t addr8[W];   // byte offsets of the stencil columns within a row
#pragma unroll
    for (int k = 0; k < W; ++k) {
        int64_t c = a + so.off[k];
        addr8[k] = (uint32_t)(c < 0 ? 0 : (c >= n2 ? n2 - 1 : c)) * 8u;
    }
    const int rb = (int)(blockIdx.y * rows_per_block);
    const int re = (int)min(nrows, (int64_t)rb + rows_per_block);
    const int n1i = (int)n1;
    const bool one_s = nrows == n1;
    const uint32_t row8 = (uint32_t)n2 * 8u;
    uint32_t xoff8 = (uint32_t)(rb + ty * R) * row8;
    const uint32_t xstep8 = (uint32_t)(VF_RL * R) * row8;
    int64_t ooff = (int64_t)(rb + ty * R) * opitch + (a - c0);
    const int64_t ostep = (int64_t)VF_RL * R * opitch;
    const char* Xb = reinterpret_cast<const char*>(X);
    for (int r0 = rb + ty * R; r0 < re; r0 += VF_RL * R, xoff8 += xstep8, ooff += ostep) {
        double x[R][W];
        unsigned rm = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int row = r0 + r;
            const bool ok = row < re && aval;
            const uint32_t rbase = xoff8 + (uint32_t)r * row8;
#pragma unroll
            for (int k = 0; k < W; ++k)
                x[r][k] = ok ? __ldg(reinterpret_cast<const double*>(Xb + (uint32_t)(rbase + addr8[k]))) : 0.0;
            if (row < re) rm |= xflag[one_s ? row : row % n1i];
        }
        const unsigned long long bneed = maskmode ? (unsigned long long)rm : (rm ? ~0ULL : 0ULL);
        auto group = [&](int g) {
            double acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const double c = sm[(g * W + k) * VF_TC + tx];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = fma(c, x[r][k], acc[r]);
            }
            double* o = vp.out[g] + ooff;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r0 + r < re && aval) o[r * opitch] = acc[r];
        };
        if (NGI > 0) {
            // interior groups: compile-time count (unrolled: immediate shared-memory offsets and
            // output pointers from the parameter bank)
#pragma unroll
            for (int g = 0; g < NGI; ++g) group(g);
        } else {
            for (int g = 0; g < vp.ng_int; ++g) group(g);
        }
        if (bneed)
            for (int g = vp.ng_int; g < vp.ng; ++g)
                if ((bneed >> (g - vp.ng_int)) & 1ULL) group(g);
    }
}

// Pass 2 (x side): Y[s][i][a] = beta*Y + sum_e [s_out(e)=s] sum_k Cst_e[k][i] Z_e[s_in][i + off_k][a].
// Block = 8 warps x T consecutive target rows (32 rows); warp lanes = columns,
// CPT columns per lane.  The block's coefficients (chunk of entries) are staged
// in shared memory and read as broadcasts; Z rows are shared between the T
// targets of a warp band by band (Kuhn offsets form runs of consecutive rows).
constexpr int XG_ECH = 12;   // entries per shared-memory chunk
template <int D, int T, int SO, int CPT>
__global__ void __launch_bounds__(256, 2) k_xgat_st(int n1, int n2, StencilOff so, const uint8_t* __restrict__ xflag,
                                                    XgatParams ep, double* __restrict__ Y, double beta,
                                                    int ncoltiles, int m, const double* __restrict__ skip) {
    if (skip && *skip != 0.0) return;   // grid converged (batched block solver)
    using B = stc::Bands<D>;
    constexpr int W = B::W;
    constexpr int ROWS = 8 * T;
    __shared__ double cs[XG_ECH][W][ROWS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // column-tile-major traversal: concurrently resident blocks cover consecutive
    // row groups of the same columns, so the x-halo rows of Z stay in L2
    const int rgroups = (n1 + ROWS - 1) / ROWS;
    const int ct = blockIdx.x / rgroups, rg = blockIdx.x % rgroups;
    const int iblk = rg * ROWS;
    const int i0 = iblk + warp * T;
    int acol[CPT];
    bool aval[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        acol[c] = ct * 32 * CPT + c * 32 + lane;
        aval[c] = acol[c] < n2;
        if (!aval[c]) acol[c] = 0;
    }
    bool anyb = false;
#pragma unroll
    for (int t = 0; t < T; ++t)
        if (i0 + t < n1) anyb |= xflag[i0 + t] != 0;
    double acc[SO][T][CPT];
#pragma unroll
    for (int s = 0; s < SO; ++s)
#pragma unroll
        for (int t = 0; t < T; ++t)
#pragma unroll
            for (int c = 0; c < CPT; ++c) acc[s][t][c] = 0.0;
    const long long plane = (long long)n1 * n2;
    for (int e0 = 0; e0 < ep.ne; e0 += XG_ECH) {
        const int ech = min(XG_ECH, ep.ne - e0);
        __syncthreads();
        for (int idx = threadIdx.x; idx < ech * W * ROWS; idx += 256) {
            const int e = idx / (W * ROWS), rem = idx - e * W * ROWS, k = rem / ROWS, r = rem - k * ROWS;
            const int i = iblk + r;
            const double* ct_ = ep.e[e0 + e].ctab;
            double v = 0.0;
            if (i < n1) {
                if (ct_) {
                    int z = i, cls = 0, mul = 1;
#pragma unroll
                    for (int q = 0; q < D; ++q) {
                        const int zq = z % m;
                        z /= m;
                        cls += mul * (zq == 0 ? 0 : (zq == m - 1 ? 2 : 1));
                        mul *= 3;
                    }
                    v = __ldg(ct_ + cls * W + k);
                } else {
                    v = __ldg(ep.e[e0 + e].cst + (long long)k * n1 + i);
                }
            }
            cs[e][k][r] = v;
        }
        __syncthreads();
        if (i0 >= n1) continue;
        for (int e = 0; e < ech; ++e) {
            const XgatEntry& E = ep.e[e0 + e];
            if (E.bonly && !anyb) continue;
            const double* Z = E.in + (long long)E.s_in * plane;
            double tmp[T][CPT];
#pragma unroll
            for (int t = 0; t < T; ++t)
#pragma unroll
                for (int c = 0; c < CPT; ++c) tmp[t][c] = 0.0;
#pragma unroll
            for (int b = 0; b < B::NB; ++b) {
                constexpr int MAXL = 3;
                const int klo = B::lo(b), len = B::len(b);
                const int base = i0 + (int)so.off[klo];
                double z[T + MAXL - 1][CPT];
#pragma unroll
                for (int q = 0; q < T + MAXL - 1; ++q) {
                    if (q < T + len - 1) {
                        int r = base + q;
                        r = r < 0 ? 0 : (r >= n1 ? n1 - 1 : r);
                        const double* zr = Z + (long long)r * n2;
#pragma unroll
                        for (int c = 0; c < CPT; ++c) z[q][c] = __ldg(zr + acol[c]);
                    }
                }
#pragma unroll
                for (int kk = 0; kk < MAXL; ++kk) {
                    if (kk < len) {
#pragma unroll
                        for (int t = 0; t < T; ++t) {
                            const double cf = cs[e][klo + kk][warp * T + t];
#pragma unroll
                            for (int c = 0; c < CPT; ++c) tmp[t][c] = fma(cf, z[t + kk][c], tmp[t][c]);
                        }
                    }
                }
            }
#pragma unroll
            for (int s = 0; s < SO; ++s)
                if (s == E.s_out)
#pragma unroll
                    for (int t = 0; t < T; ++t)
#pragma unroll
                        for (int c = 0; c < CPT; ++c) acc[s][t][c] = fma(E.scale, tmp[t][c], acc[s][t][c]);
        }
    }
    if (i0 >= n1) return;
#pragma unroll
    for (int s = 0; s < SO; ++s)
#pragma unroll
        for (int t = 0; t < T; ++t) {
            if (i0 + t >= n1) continue;
            double* yr = Y + (long long)s * plane + (long long)(i0 + t) * n2;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                if (!aval[c]) continue;
                double* y = yr + acol[c];
                *y = beta == 0.0 ? acc[s][t][c] : fma(beta, *y, acc[s][t][c]);
            }
        }
}

// x-side fanout (x-first two-pass order for grids with n1 > n2):
// U_g[s][i][a] = sum_k A_g[i, i + off_k] X[s][i + off_k][a] for all x-groups g.
// Warp = 32*CPT columns x T consecutive target rows; the X band rows are loaded
// once and reused for every group; coefficients come from the class tables
// (translation-invariant x matrices) or the stencil arrays.
template <int D, int T, int CPT>
__global__ void __launch_bounds__(256, 2) k_xfan_st(int n1, int n2, StencilOff so, int m, const uint8_t* __restrict__ xflag,
                                                    XfanParams fp, const double* __restrict__ X, int ncoltiles) {
    using B = stc::Bands<D>;
    constexpr int W = B::W;
    constexpr int ROWS = 8 * T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rgroups = (n1 + ROWS - 1) / ROWS;
    const int s = blockIdx.y;
    const int ct = blockIdx.x / rgroups, rg = blockIdx.x % rgroups;
    const int i0 = rg * ROWS + warp * T;
    if (i0 >= n1) return;
    const long long plane = (long long)n1 * n2;
    const double* Xs = X + s * plane;
    int acol[CPT];
    bool aval[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        acol[c] = ct * 32 * CPT + c * 32 + lane;
        aval[c] = acol[c] < n2;
        if (!aval[c]) acol[c] = 0;
    }
    bool anyb = false;
    int cls[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int it = min(i0 + t, n1 - 1);
        anyb |= (i0 + t < n1) && xflag[it] != 0;
        int z = it, cl = 0, mul = 1;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const int zq = z % m;
            z /= m;
            cl += mul * (zq == 0 ? 0 : (zq == m - 1 ? 2 : 1));
            mul *= 3;
        }
        cls[t] = cl;
    }
    constexpr int MAXL = 3;
    double z[B::NB][T + MAXL - 1][CPT];
#pragma unroll
    for (int b = 0; b < B::NB; ++b) {
        const int klo = B::lo(b), len = B::len(b);
        const int base = i0 + (int)so.off[klo];
#pragma unroll
        for (int q = 0; q < T + MAXL - 1; ++q) {
            if (q < T + len - 1) {
                int r = base + q;
                r = r < 0 ? 0 : (r >= n1 ? n1 - 1 : r);
                const double* zr = Xs + (long long)r * n2;
#pragma unroll
                for (int c = 0; c < CPT; ++c) z[b][q][c] = __ldg(zr + acol[c]);
            }
        }
    }
    const int ngu = anyb ? fp.ng : fp.ng_int;
    for (int g = 0; g < ngu; ++g) {
        const double* tab = fp.ctab[g];
        const double* st = fp.cst[g];
        double acc[T][CPT];
#pragma unroll
        for (int t = 0; t < T; ++t)
#pragma unroll
            for (int c = 0; c < CPT; ++c) acc[t][c] = 0.0;
#pragma unroll
        for (int b = 0; b < B::NB; ++b) {
            const int klo = B::lo(b), len = B::len(b);
#pragma unroll
            for (int kk = 0; kk < MAXL; ++kk) {
                if (kk < len) {
#pragma unroll
                    for (int t = 0; t < T; ++t) {
                        const int it = min(i0 + t, n1 - 1);
                        const double cf = tab ? __ldg(tab + cls[t] * W + klo + kk) : __ldg(st + (long long)(klo + kk) * n1 + it);
#pragma unroll
                        for (int c = 0; c < CPT; ++c) acc[t][c] = fma(cf, z[b][t + kk][c], acc[t][c]);
                    }
                }
            }
        }
        double* o = fp.out[g] + s * plane;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            if (i0 + t >= n1) continue;
#pragma unroll
            for (int c = 0; c < CPT; ++c)
                if (aval[c]) o[(long long)(i0 + t) * n2 + acol[c]] = acc[t][c];
        }
    }
}

int launch_xfan_st(sg_problem* P, int d, int S, int64_t n1, int64_t n2, const StencilOff& so, int m,
                   const uint8_t* xflag, const XfanParams& fp, const double* X) {
    constexpr int T = 4;
    const int cpt = n2 >= 64 ? 2 : 1;
    const int64_t ctiles = (n2 + 32 * cpt - 1) / (32 * cpt);
    const int64_t rgroups = (n1 + 8 * T - 1) / (8 * T);
    const int64_t nb = ctiles * rgroups;
    if (n1 * n2 >= (1LL << 31) || nb >= (1LL << 31)) return SG_ERR_UNSUPPORTED;
    dim3 grid((unsigned)nb, (unsigned)S);
#define XF(DD, CC) k_xfan_st<DD, T, CC><<<grid, 256, 0, P->stream>>>((int)n1, (int)n2, so, m, xflag, fp, X, (int)ctiles)
    if (cpt == 2) {
        if (d == 1) XF(1, 2); else if (d == 2) XF(2, 2); else XF(3, 2);
    } else {
        if (d == 1) XF(1, 1); else if (d == 2) XF(2, 1); else XF(3, 1);
    }
#undef XF
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

// v-side gather with time mixing on box v-lattices (cross-grid upper part):
// Y[s][j][a] = beta*Y + sum_e [s_out=s] scale_e sum_k st_e[k][a] in_e[s_in][j][a + off_k]
// Block = 32 columns x 8 row lanes; the block's coefficients (all entries) are
// staged once in shared memory and reused for every row the block sweeps.
template <int D>
__global__ void __launch_bounds__(256) k_vgat_st(int S_out, int n1, int n2, StencilOff so, XgatParams ep,
                                                 double* __restrict__ Y, double beta, int rows_per_block,
                                                 const uint8_t* __restrict__ xflag) {
    constexpr int W = stc::Bands<D>::W;
    extern __shared__ double cs[];   // [ne][W][32]
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int a = blockIdx.x * 32 + tx;
    const bool aval = a < n2;
    for (int idx = ty * 32 + tx; idx < ep.ne * W * 32; idx += 256) {
        const int e = idx / (W * 32), rem = idx - e * W * 32, k = rem >> 5, c = rem & 31;
        const int ac = blockIdx.x * 32 + c;
        cs[idx] = ac < n2 ? __ldg(ep.e[e].cst + (long long)k * n2 + ac) : 0.0;
    }
    __syncthreads();
    if (!aval) return;
    int addr[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        int c = a + (int)so.off[k];
        addr[k] = c < 0 ? 0 : (c >= n2 ? n2 - 1 : c);
    }
    const int R = S_out * n1;
    const int rb = blockIdx.y * rows_per_block, re = min(R, rb + rows_per_block);
    for (int r = rb + ty; r < re; r += 8) {
        const int s = r / n1, j = r - s * n1;
        const bool bnd = xflag == nullptr || xflag[j] != 0;
        double acc = 0.0;
        for (int e = 0; e < ep.ne; ++e) {
            const XgatEntry& E = ep.e[e];
            if (E.s_out != s || (E.bonly && !bnd)) continue;
            const double* row = E.in + ((long long)E.s_in * n1 + j) * n2;
            const double* c = cs + e * W * 32 + tx;
            double a2 = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) a2 = fma(c[k * 32], __ldg(row + addr[k]), a2);
            acc = fma(E.scale, a2, acc);
        }
        double* y = Y + (long long)r * n2 + a;
        *y = beta == 0.0 ? acc : fma(beta, *y, acc);
    }
}

int launch_vgat_st(sg_problem* P, int d, int S_out, int64_t n1, int64_t n2, const StencilOff& so,
                   const XgatParams& ep, double* Y, double beta, const uint8_t* xflag) {
    const int64_t R = (int64_t)S_out * n1;
    if (R * n2 == 0 || ep.ne == 0) return SG_OK;
    const int W = (1 << (d + 1)) - 1;
    const int64_t ctiles = (n2 + 31) / 32;
    int64_t rchunks = std::max<int64_t>(1, (148 * 8 + ctiles - 1) / ctiles);
    rchunks = std::min<int64_t>(rchunks, (R + 7) / 8);
    rchunks = std::min<int64_t>(std::max<int64_t>(rchunks, 1), 65535);
    const int rpb = (int)((R + rchunks - 1) / rchunks);
    const size_t smem = sizeof(double) * ep.ne * W * 32;
    dim3 grid((unsigned)ctiles, (unsigned)rchunks), block(32, 8);
#define VG(DD)                                                                                       \
    do {                                                                                             \
        cudaFuncSetAttribute(k_vgat_st<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        k_vgat_st<DD><<<grid, block, smem, P->stream>>>(S_out, (int)n1, (int)n2, so, ep, Y, beta, rpb, xflag); \
    } while (0)
    if (d == 1) VG(1); else if (d == 2) VG(2); else VG(3);
#undef VG
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

// ---- class compression of translation-invariant stencil matrices on box lattices:
// row i depends only on its boundary class (per axis: low face / interior / high face).
__global__ void k_class_check(int64_t n, int d, int m, int W, const double* st, const double* tab, double* out2) {
    __shared__ double sm[2][8];
    double dev = 0.0, mag = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t z = i;
        int cls = 0, mul = 1;
        for (int q = 0; q < d; ++q) {
            const int zq = (int)(z % m);
            z /= m;
            cls += mul * (zq == 0 ? 0 : (zq == m - 1 ? 2 : 1));
            mul *= 3;
        }
        for (int k = 0; k < W; ++k) {
            const double a = st[k * n + i];
            dev = fmax(dev, fabs(a - tab[cls * W + k]));
            mag = fmax(mag, fabs(a));
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

int class_compress(sg_problem* P, const Factor& f, int l, const double* st, double** ctab) {
    *ctab = nullptr;
    if (f.kind != SG_MESH_BOX) return SG_OK;
    const Level& L = f.lev[l];
    const int d = f.d, W = f.W, m = L.m;
    int ncls = 1;
    for (int q = 0; q < d; ++q) ncls *= 3;
    std::vector<double> tab(27 * W, 0.0);
    for (int c = 0; c < ncls; ++c) {
        int cc = c;
        int64_t idx = 0, mul = 1;
        for (int q = 0; q < d; ++q) {
            const int s = cc % 3;
            cc /= 3;
            const int z = s == 0 ? 0 : (s == 2 ? m - 1 : (m - 1) / 2);
            idx += z * mul;
            mul *= m;
        }
        for (int k = 0; k < W; ++k)
            SG_CUDA(cudaMemcpy(&tab[c * W + k], st + (int64_t)k * L.n + idx, sizeof(double), cudaMemcpyDeviceToHost));
    }
    double* dtab;
    SG_CUDA(cudaMalloc(&dtab, sizeof(double) * 27 * W));
    SG_CUDA(cudaMemcpy(dtab, tab.data(), sizeof(double) * 27 * W, cudaMemcpyHostToDevice));
    const int nb = 256;
    double* out2;
    SG_CUDA(cudaMalloc(&out2, sizeof(double) * 2 * nb));
    k_class_check<<<nb, 256, 0, P->stream>>>(L.n, d, m, W, st, dtab, out2);
    P->launches++;
    std::vector<double> h(2 * nb);
    SG_CUDA(cudaMemcpyAsync(h.data(), out2, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, P->stream));
    SG_CUDA(cudaStreamSynchronize(P->stream));
    cudaFree(out2);
    double dev = 0, mag = 0;
    for (int b = 0; b < nb; ++b) {
        dev = std::max(dev, h[2 * b]);
        mag = std::max(mag, h[2 * b + 1]);
    }
    if (dev <= 1e-14 * mag) {
        *ctab = dtab;
    } else {
        cudaFree(dtab);
    }
    return SG_OK;
}

int launch_vfan_st(sg_problem* P, int d, int S, int64_t n1, int64_t n2, const StencilOff& so, const uint8_t* xflag,
                   const VfanParams& vp, const double* X, int64_t opitch, int64_t c0, int64_t c1, int maskmode) {
    if (c1 <= 0) c1 = n2;
    if (opitch <= 0) opitch = c1 - c0;
    const int W = (1 << (d + 1)) - 1;
    const int64_t nrows = (int64_t)S * n1;
    const int64_t ctiles = (c1 - c0 + VF_TC - 1) / VF_TC;
    if (nrows * n2 >= (1LL << 29)) {
        set_error("k_vfan_st: grid too large for 32-bit byte offsets");
        return SG_ERR_UNSUPPORTED;
    }
    // enough blocks to fill the machine, as many rows per block as possible (coefficient reuse)
    constexpr int vf_mult = 12;   // blocks per SM, measured best in round 1
    int64_t rchunks = std::max<int64_t>(1, (148 * vf_mult + ctiles - 1) / ctiles);
    rchunks = std::min<int64_t>(rchunks, (nrows + 15) / 16);
    rchunks = std::max<int64_t>(rchunks, 1);
    const int64_t rpb = (nrows + rchunks - 1) / rchunks;
    const size_t smem = sizeof(double) * vp.ng * W * VF_TC;
    dim3 grid((unsigned)ctiles, (unsigned)rchunks), block(VF_TC, VF_RL);
    if (d == 1) {
        cudaFuncSetAttribute(k_vfan_st<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_vfan_st<1, 2><<<grid, block, smem, P->stream>>>(nrows, n1, n2, so, xflag, vp, X, rpb, opitch, P->skip, c0, c1, maskmode);
    } else if (d == 2) {
        cudaFuncSetAttribute(k_vfan_st<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_vfan_st<2, 2><<<grid, block, smem, P->stream>>>(nrows, n1, n2, so, xflag, vp, X, rpb, opitch, P->skip, c0, c1, maskmode);
    } else {
        // R = 2 rows per thread (R = 3/4 measured 4-11 % slower in round 1: register-starved)
        if (vp.ng_int == 10) {
            cudaFuncSetAttribute(k_vfan_st<3, 2, 2, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_vfan_st<3, 2, 2, 10><<<grid, block, smem, P->stream>>>(nrows, n1, n2, so, xflag, vp, X, rpb, opitch, P->skip, c0,
                                                                     c1, maskmode);
        } else {
            cudaFuncSetAttribute(k_vfan_st<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_vfan_st<3, 2><<<grid, block, smem, P->stream>>>(nrows, n1, n2, so, xflag, vp, X, rpb, opitch, P->skip, c0, c1,
                                                              maskmode);
        }
    }
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

int launch_xgat_st(sg_problem* P, int d, int S_out, int64_t n1, int64_t n2, const StencilOff& so,
                   const uint8_t* xflag, const XgatParams& ep, double* Y, double beta, int m) {
    constexpr int T = 4;
    const int cpt = n2 >= 64 ? 2 : 1;
    const int64_t ctiles = (n2 + 32 * cpt - 1) / (32 * cpt);
    const int64_t rgroups = (n1 + 8 * T - 1) / (8 * T);
    const int64_t nb = ctiles * rgroups;
    if (n1 * n2 >= (1LL << 31) || nb >= (1LL << 31)) {
        set_error("grid too large for 32-bit stencil indexing");
        return SG_ERR_UNSUPPORTED;
    }
#define XG(DD, SS, CC) k_xgat_st<DD, T, SS, CC><<<(unsigned)nb, 256, 0, P->stream>>>((int)n1, (int)n2, so, xflag, ep, Y, beta, (int)ctiles, m, P->skip)
#define XGD(SS, CC) do { if (d == 1) XG(1, SS, CC); else if (d == 2) XG(2, SS, CC); else XG(3, SS, CC); } while (0)
    if (S_out == 1) {
        if (cpt == 2) XGD(1, 2); else XGD(1, 1);
    } else {
        if (cpt == 2) XGD(2, 2); else XGD(2, 1);
    }
#undef XGD
#undef XG
    P->launches++;
    SG_CUDA(cudaGetLastError());
    return SG_OK;
}

}  // namespace sg

namespace sg {
// =====================================================================
// Batched transfer jobs: independent Kronecker-factored ELL applies (the
// restriction / prolongation chains of the cross-grid apply) in ONE launch.
//   out[t] = (add ? add[t] : 0) + scale * sum_k M[k][row] * in[... col_k ...]
// Block b serves job j with blk0[j] <= b < blk0[j+1].
// =====================================================================
__global__ void __launch_bounds__(256) k_jobs(JobList jl) {
    int j = 0;
    while (j + 1 < jl.nj && jl.j[j + 1].blk0 <= (int)blockIdx.x) ++j;
    const Job& J = jl.j[j];
    // 32-bit index arithmetic (every job has < 2^31 outputs, checked on the host)
    const unsigned n1_out = (unsigned)(J.dir == 0 ? J.nrows_out : J.n1_in);
    const unsigned n2_out = (unsigned)(J.dir == 1 ? J.nrows_out : J.n2_in);
    const unsigned per_s = n1_out * n2_out;
    const unsigned total = per_s * (unsigned)J.S;
    const unsigned nrows = (unsigned)J.nrows_out;
    const unsigned n1i = (unsigned)J.n1_in, n2i = (unsigned)J.n2_in;
    const int nblk = (j + 1 < jl.nj ? jl.j[j + 1].blk0 : jl.total_blocks) - J.blk0;
    const int W = J.W;
    for (unsigned t = (unsigned)(blockIdx.x - J.blk0) * blockDim.x + threadIdx.x; t < total;
         t += (unsigned)nblk * blockDim.x) {
        const unsigned s = t >= per_s ? 1u : 0u;   // S <= 2
        const unsigned rc = t - s * per_s;
        const unsigned r = rc / n2_out, c = rc - r * n2_out;
        double acc = 0.0;
        if (J.dir == 1) {
            const double* in = J.in + ((size_t)s * n1i + r) * n2i;
            for (int k = 0; k < W; ++k) {
                const int32_t col = __ldg(J.cols + k * nrows + c);
                if (col >= 0) acc = fma(__ldg(J.vals + k * nrows + c), __ldg(in + col), acc);
            }
        } else {
            const double* in = J.in + (size_t)s * n1i * n2i + c;
            for (int k = 0; k < W; ++k) {
                const int32_t col = __ldg(J.cols + k * nrows + r);
                if (col >= 0) acc = fma(__ldg(J.vals + k * nrows + r), __ldg(in + (size_t)col * n2i), acc);
            }
        }
        const double v = (J.add ? J.add[t] : 0.0) + J.scale * acc;
        if (J.opitch > 0)
            J.out[((size_t)s * n1_out + r) * (size_t)J.opitch + c] = v;
        else
            J.out[t] = v;
    }
}

// Restriction (E^T) on a box lattice as a stencil: the coarse node c with
// lattice coordinates z collects the fine node 2z (weight 1) and the midpoints 2z + delta of its
// Kuhn edges (weight 1/2), delta in {0,1}^D u {0,-1}^D \ {0}; no pattern/value arrays are read.
template <int D>
__global__ void __launch_bounds__(256) k_jobs_rbox(JobList jl) {
    int j = 0;
    while (j + 1 < jl.nj && jl.j[j + 1].blk0 <= (int)blockIdx.x) ++j;
    const Job& J = jl.j[j];
    const unsigned n1_out = (unsigned)(J.dir == 0 ? J.nrows_out : J.n1_in);
    const unsigned n2_out = (unsigned)(J.dir == 1 ? J.nrows_out : J.n2_in);
    const unsigned per_s = n1_out * n2_out;
    const unsigned total = per_s * (unsigned)J.S;
    const unsigned n1i = (unsigned)J.n1_in, n2i = (unsigned)J.n2_in;
    const int mf = J.box_mf, mc = (mf + 1) / 2;
    const int nblk = (j + 1 < jl.nj ? jl.j[j + 1].blk0 : jl.total_blocks) - J.blk0;
    for (unsigned t = (unsigned)(blockIdx.x - J.blk0) * blockDim.x + threadIdx.x; t < total;
         t += (unsigned)nblk * blockDim.x) {
        const unsigned s = t >= per_s ? 1u : 0u;
        const unsigned rc = t - s * per_s;
        const unsigned r = rc / n2_out, c = rc - r * n2_out;
        if (J.rmask && !((J.rmask[r] >> J.rbit) & 1)) continue;   // row outside the group's face
        unsigned node = J.dir == 1 ? c : r;   // coarse node
        int z[D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
            z[q] = (int)(node % (unsigned)mc);
            node /= (unsigned)mc;
        }
        int stride[D], fb = 0;
        {
            int st = 1;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                stride[q] = st;
                fb += 2 * z[q] * st;
                st *= mf;
            }
        }
        const double* base = J.dir == 1 ? J.in + ((size_t)s * n1i + r) * n2i : J.in + (size_t)s * n1i * n2i + c;
        const size_t fs = J.dir == 1 ? 1 : n2i;   // element stride of one fine node
        double acc = base[(size_t)fb * fs];
#pragma unroll
        for (int sg = -1; sg <= 1; sg += 2)
#pragma unroll
            for (int mask = 1; mask < (1 << D); ++mask) {
                bool ok = true;
                int off = 0;
#pragma unroll
                for (int q = 0; q < D; ++q)
                    if ((mask >> q) & 1) {
                        const int fz = 2 * z[q] + sg;
                        ok &= fz >= 0 && fz < mf;
                        off += sg * stride[q];
                    }
                if (ok) acc = fma(0.5, __ldg(base + (size_t)(fb + off) * fs), acc);
            }
        const double v = (J.add ? J.add[t] : 0.0) + J.scale * acc;
        if (J.opitch > 0)
            J.out[((size_t)s * n1_out + r) * (size_t)J.opitch + c] = v;
        else
            J.out[t] = v;
    }
}

// Prolongation (E) on a box lattice as a stencil: fine node f with lattice
// parity pi = f mod 2 takes its coarse node f/2 (pi = 0) or the mean of the two ends (f -+ pi)/2
// of the coarse Kuhn edge it bisects; no pattern/value arrays are read.
template <int D>
__global__ void __launch_bounds__(256) k_jobs_pbox(JobList jl) {
    int j = 0;
    while (j + 1 < jl.nj && jl.j[j + 1].blk0 <= (int)blockIdx.x) ++j;
    const Job& J = jl.j[j];
    const unsigned n1_out = (unsigned)(J.dir == 0 ? J.nrows_out : J.n1_in);
    const unsigned n2_out = (unsigned)(J.dir == 1 ? J.nrows_out : J.n2_in);
    const unsigned per_s = n1_out * n2_out;
    const unsigned total = per_s * (unsigned)J.S;
    const unsigned n1i = (unsigned)J.n1_in, n2i = (unsigned)J.n2_in;
    const int mf = J.box_mf, mc = (mf + 1) / 2;
    const int nblk = (j + 1 < jl.nj ? jl.j[j + 1].blk0 : jl.total_blocks) - J.blk0;
    for (unsigned t = (unsigned)(blockIdx.x - J.blk0) * blockDim.x + threadIdx.x; t < total;
         t += (unsigned)nblk * blockDim.x) {
        const unsigned s = t >= per_s ? 1u : 0u;
        const unsigned rc = t - s * per_s;
        const unsigned r = rc / n2_out, c = rc - r * n2_out;
        if (J.rmask && !((J.rmask[r] >> J.rbit) & 1)) continue;   // row outside the group's face
        unsigned node = J.dir == 1 ? c : r;   // fine node
        int lo = 0, hi = 0, st = 1;
        bool mid = false;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const int f = (int)(node % (unsigned)mf);
            node /= (unsigned)mf;
            const int pq = f & 1;
            mid |= pq != 0;
            lo += ((f - pq) >> 1) * st;
            hi += ((f + pq) >> 1) * st;
            st *= mc;
        }
        const double* base = J.dir == 1 ? J.in + ((size_t)s * n1i + r) * n2i : J.in + (size_t)s * n1i * n2i + c;
        const size_t fs = J.dir == 1 ? 1 : n2i;
        const double acc = mid ? 0.5 * __ldg(base + (size_t)lo * fs) + 0.5 * __ldg(base + (size_t)hi * fs)
                               : __ldg(base + (size_t)lo * fs);
        const double v = (J.add ? J.add[t] : 0.0) + J.scale * acc;
        if (J.opitch > 0)
            J.out[((size_t)s * n1_out + r) * (size_t)J.opitch + c] = v;
        else
            J.out[t] = v;
    }
}

int launch_jobs(sg_problem* P, std::vector<Job>& jobs) {
    size_t i = 0;
    while (i < jobs.size()) {
        JobList jl;
        jl.nj = 0;
        int blk = 0;
        while (i < jobs.size() && jl.nj < MAX_JOBS) {
            Job J = jobs[i++];
            const int64_t n1_out = J.dir == 0 ? J.nrows_out : J.n1_in;
            const int64_t n2_out = J.dir == 1 ? J.nrows_out : J.n2_in;
            const int64_t total = n1_out * n2_out * J.S;
            if (total == 0) continue;
            if (total >= (1LL << 31) || J.S > 2) {
                set_error("transfer job too large for 32-bit indexing");
                return SG_ERR_UNSUPPORTED;
            }
            J.blk0 = blk;
            blk += (int)std::min<int64_t>((total + 2047) / 2048, 148 * 8);
            jl.j[jl.nj++] = J;
        }
        if (jl.nj == 0) continue;
        jl.total_blocks = blk;
        bool rbox = true;
        for (int q = 0; q < jl.nj; ++q) rbox &= jl.j[q].box_mf > 0 && jl.j[q].W == jl.j[0].W;
        const int dd = jl.j[0].W == 3 ? 1 : (jl.j[0].W == 7 ? 2 : (jl.j[0].W == 15 ? 3 : 0));
        bool pbox = true;
        for (int q = 0; q < jl.nj; ++q) pbox &= jl.j[q].box_mf > 0 && jl.j[q].W == 2 && jl.j[q].box_d == jl.j[0].box_d;
        if (pbox && jl.j[0].box_d == 3) k_jobs_pbox<3><<<blk, 256, 0, P->stream>>>(jl);
        else if (pbox && jl.j[0].box_d == 2) k_jobs_pbox<2><<<blk, 256, 0, P->stream>>>(jl);
        else if (pbox && jl.j[0].box_d == 1) k_jobs_pbox<1><<<blk, 256, 0, P->stream>>>(jl);
        else if (rbox && dd == 3) k_jobs_rbox<3><<<blk, 256, 0, P->stream>>>(jl);
        else if (rbox && dd == 2) k_jobs_rbox<2><<<blk, 256, 0, P->stream>>>(jl);
        else if (rbox && dd == 1) k_jobs_rbox<1><<<blk, 256, 0, P->stream>>>(jl);
        else k_jobs<<<blk, 256, 0, P->stream>>>(jl);
        P->launches++;
        SG_CUDA(cudaGetLastError());
    }
    return SG_OK;
}
}  // namespace sg
