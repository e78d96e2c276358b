// U-matrix: per-node mean fp64 distance to its grid neighbours, stored f32
// (umatrix.py:26-45).  Neighbours follow grid.py:52-73 exactly: Moore-8 in
// row-major scan order, planar maps drop out-of-range cells, toroids wrap and
// drop duplicates and the node itself.  Hex (extension): the 6 unit-distance
// offset-row neighbours under the same rules.
#include "common.cuh"

namespace somb {

__global__ void umatrix_kernel(const float *__restrict__ W, int d, MapDev m, float *__restrict__ U) {
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    const int K = m.nx * m.ny;
    if (j >= K) return;
    const int col = j % m.nx, row = j / m.nx;
    int nb[8];
    int cntn = 0;
    for (int o = 0; o < 8; ++o) {
        int dc, dr;
        if (!m.hex) {
            int q = o < 4 ? o : o + 1;        // skip the centre of the 3x3 scan
            dc = q % 3 - 1;
            dr = q / 3 - 1;
        } else {
            if (o >= 6) break;
            const int odd[6][2] = {{0, -1}, {1, -1}, {-1, 0}, {1, 0}, {0, 1}, {1, 1}};
            const int even[6][2] = {{-1, -1}, {0, -1}, {-1, 0}, {1, 0}, {-1, 1}, {0, 1}};
            dc = (row & 1) ? odd[o][0] : even[o][0];
            dr = (row & 1) ? odd[o][1] : even[o][1];
        }
        int c = col + dc, r = row + dr;
        if (m.toroid) {
            c = ((c % m.nx) + m.nx) % m.nx;
            r = ((r % m.ny) + m.ny) % m.ny;
        } else if (c < 0 || c >= m.nx || r < 0 || r >= m.ny) {
            continue;
        }
        int idx = r * m.nx + c;
        if (idx == j) continue;
        bool dup = false;
        for (int q = 0; q < cntn; ++q) dup |= nb[q] == idx;
        if (dup) continue;
        nb[cntn++] = idx;
    }
    double total = 0.0;
    const float *wj = W + (int64_t)j * d;
    for (int q = 0; q < cntn; ++q) {
        const float *wn = W + (int64_t)nb[q] * d;
        double s = 0.0;
        for (int k = lane; k < d; k += 32) {
            double df = (double)wn[k] - (double)wj[k];
            s = __fma_rn(df, df, s);
        }
        s = warp_sum(s);
        total += sqrt(s);
    }
    if (lane == 0) U[j] = cntn ? (float)(total / (double)cntn) : 0.0f;
}

}  // namespace somb

using namespace somb;

extern "C" int somb_umatrix(const float *W, int32_t d, const somb_map *map, float *U, void *stream) {
    SOMB_REQUIRE(map && map->n_columns >= 1 && map->n_rows >= 1 && d > 0, SOMB_E_INPUT, "umatrix: bad shape");
    MapDev m{map->n_columns, map->n_rows, map->grid == SOMB_GRID_HEX, map->topology == SOMB_TOROID};
    int K = m.nx * m.ny;
    umatrix_kernel<<<(K + 7) / 8, 256, 0, as_stream(stream)>>>(W, d, m, U);
    note_launch();
    SOMB_LAUNCH_CHECK("umatrix");
    return SOMB_OK;
}
