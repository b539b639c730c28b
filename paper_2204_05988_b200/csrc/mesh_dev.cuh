// Structured Kuhn-lattice mesh helpers shared by the device kernels of libsg.
// (Product code; the oracle has its own, independent mesh construction.)
#pragma once
#include <stdint.h>

#include "../../include/sg.h"

namespace sg {

// lattice point -> node id (-1 if absent).  Lexicographic, axis 0 fastest.
// L-shape: [-1,1]^2 minus the open quadrant x>0, y<0; c = (m-1)/2 is the centre.
__host__ __device__ inline int64_t node_index(int kind, int d, int m, const int* z) {
    for (int i = 0; i < d; ++i)
        if (z[i] < 0 || z[i] >= m) return -1;
    if (kind == SG_MESH_LSHAPE) {
        const int c = (m - 1) / 2;
        if (z[0] > c && z[1] < c) return -1;
        if (z[1] < c) return (int64_t)z[1] * (c + 1) + z[0];
        return (int64_t)c * (c + 1) + (int64_t)(z[1] - c) * m + z[0];
    }
    int64_t id = 0;
    for (int i = d - 1; i >= 0; --i) id = id * m + z[i];
    return id;
}

__host__ __device__ inline void node_lattice(int kind, int d, int m, int64_t id, int* z) {
    if (kind == SG_MESH_LSHAPE) {
        const int c = (m - 1) / 2;
        const int64_t low = (int64_t)c * (c + 1);
        if (id < low) {
            z[1] = (int)(id / (c + 1));
            z[0] = (int)(id % (c + 1));
        } else {
            z[1] = c + (int)((id - low) / m);
            z[0] = (int)((id - low) % m);
        }
        return;
    }
    for (int i = 0; i < d; ++i) {
        z[i] = (int)(id % m);
        id /= m;
    }
}

__host__ __device__ inline int64_t mesh_nodes(int kind, int d, int m) {
    if (kind == SG_MESH_LSHAPE) {
        const int64_t c = (m - 1) / 2;
        return (int64_t)m * m - c * c;
    }
    int64_t n = 1;
    for (int i = 0; i < d; ++i) n *= m;
    return n;
}

// is the lattice cell with lower corner c part of the domain?
__host__ __device__ inline bool cell_in_domain(int kind, int d, int cells, const int* c) {
    for (int i = 0; i < d; ++i)
        if (c[i] < 0 || c[i] >= cells) return false;
    if (kind == SG_MESH_LSHAPE) {
        const int h = cells / 2;
        if (c[0] >= h && c[1] < h) return false;
    }
    return true;
}

}  // namespace sg
