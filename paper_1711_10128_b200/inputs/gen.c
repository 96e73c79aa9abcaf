/*
 * Seeded synthetic inputs for the TRPL+K hot path (BASELINE.json configs C1-C5).
 *
 * This module holds NONE of the method's arithmetic: it only builds the
 * matrices A, B (CSR, both triangles, columns strictly increasing) and the
 * random diagonal perturbation d.  It is shared by the oracle tests and the
 * CUDA path as the common source of inputs.
 *
 * Grid numbering (reading R14): natural lexicographic order,
 * x fastest, row = x + N*(y + N*z); Dirichlet boundary = out-of-grid
 * neighbours omitted.
 *
 * Counter-based U[0,1) generator (reading R13): splitmix64-style finaliser
 *   key = seed*0xD1B54A32D192ED03 ^ stream*0xABC98388FB8FAC03
 *   z   = key + (index+1)*0x9E3779B97F4A7C15
 *   z   = (z ^ (z>>30)) * 0xBF58476D1CE4E5B9
 *   z   = (z ^ (z>>27)) * 0x94D049BB133111EB
 *   z  ^= z>>31;   u = (z>>11) * 2^-53
 * (all arithmetic mod 2^64).  Stream 1 = diag(d), index = global row.
 */
#include <stdint.h>
#include <stddef.h>

double gen_u01(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t key = (seed * 0xD1B54A32D192ED03ULL) ^ (stream * 0xABC98388FB8FAC03ULL);
    uint64_t z = key + (index + 1ULL) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

void gen_u01_fill(uint64_t seed, uint64_t stream, uint64_t index0, int64_t count, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) out[i] = gen_u01(seed, stream, index0 + (uint64_t)i);
}

/* Offsets of a stencil: dim=1 -> 3-point line; dim=3, npts=7 -> faces; dim=3, npts=27 -> full cube. */
static int stencil_offsets(int dim, int npts, int off[27][3]) {
    int c = 0;
    if (dim == 1) {
        for (int dx = -1; dx <= 1; ++dx) { off[c][0] = dx; off[c][1] = 0; off[c][2] = 0; ++c; }
        return c;
    }
    /* lexicographic (z slowest, x fastest) so that column ids come out increasing */
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int nz = (dx != 0) + (dy != 0) + (dz != 0);
                if (npts == 7 && nz > 1) continue;
                off[c][0] = dx; off[c][1] = dy; off[c][2] = dz; ++c;
            }
    return c;
}

/* Number of stored entries of each row r in [r0,r1): rowptr[0..r1-r0] (rowptr[0]=0). Returns nnz. */
int64_t gen_stencil_rowptr(int dim, int npts, int64_t N, int64_t r0, int64_t r1, int64_t* rowptr) {
    int off[27][3];
    int ns = stencil_offsets(dim, npts, off);
    int64_t NY = (dim == 1) ? 1 : N, NZ = (dim == 1) ? 1 : N;
    rowptr[0] = 0;
    int64_t acc = 0;
    for (int64_t r = r0; r < r1; ++r) {
        int64_t x = r % N, y = (r / N) % NY, z = r / (N * NY);
        int cnt = 0;
        for (int s = 0; s < ns; ++s) {
            int64_t xx = x + off[s][0], yy = y + off[s][1], zz = z + off[s][2];
            if (xx < 0 || xx >= N || yy < 0 || yy >= NY || zz < 0 || zz >= NZ) continue;
            ++cnt;
        }
        acc += cnt;
        rowptr[r - r0 + 1] = acc;
    }
    return acc;
}

/* Fill columns and values: diagonal = center + dscale*U(seed,1,row), off-diagonals = offval. */
void gen_stencil_fill(int dim, int npts, int64_t N, int64_t r0, int64_t r1, const int64_t* rowptr,
                      int64_t* col, double* val, double center, double offval, double dscale,
                      uint64_t seed) {
    int off[27][3];
    int ns = stencil_offsets(dim, npts, off);
    int64_t NY = (dim == 1) ? 1 : N, NZ = (dim == 1) ? 1 : N;
#pragma omp parallel for schedule(static)
    for (int64_t r = r0; r < r1; ++r) {
        int64_t x = r % N, y = (r / N) % NY, z = r / (N * NY);
        int64_t p = rowptr[r - r0];
        for (int s = 0; s < ns; ++s) {
            int64_t xx = x + off[s][0], yy = y + off[s][1], zz = z + off[s][2];
            if (xx < 0 || xx >= N || yy < 0 || yy >= NY || zz < 0 || zz >= NZ) continue;
            int64_t c = xx + N * (yy + NY * zz);
            col[p] = c;
            if (c == r) {
                double d = (dscale != 0.0) ? dscale * gen_u01(seed, 1, (uint64_t)r) : 0.0;
                val[p] = center + d;
            } else {
                val[p] = offval;
            }
            ++p;
        }
    }
}
