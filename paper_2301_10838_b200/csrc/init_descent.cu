// init_descent.cu -- K1 + K2: total-order keys, steepest-descent
// initialisation of the triplet store, tile-local descent.
//
// Paper: Alg. 1 lines 2-3 start from T[u] = (u, u), the triplet store of the
// edgeless graph, and the merge phase turns any normalized
// store of a subgraph into the store of the whole graph, edge by edge
// (PAPER.md:219-221).  We start instead from the store of the steepest-descent
// forest F (every non-minimum u linked to its lowest lower neighbour): its
// triplets (u, u, w) with key(w) < key(u) are valid and normalized, so the
// merge phase over the remaining edges yields the same final store (DESIGN.md
// derivation B).  Within a tile held in shared memory each vertex follows its
// descent path until it reaches a minimum of the tile or leaves the tile, and
// stores that vertex: T[u] = (u, p(u)) -- still a valid triplet (u and p(u)
// are joined below key(u) along the path), so every later climb through the
// forest takes one hop per tile instead of one per vertex.
//
// Layout: f float32[n] x-fastest (reading R10); C = 16-byte working cells
// (common.cuh: key(s), owner key, v), written once.
// One CTA of 256 threads = 8 warps owns a 32 x TY x TZ tile (TY*TZ = 64
// rows, 2048 vertices); its f halo (+-1 in x, y, z) is staged in shared
// memory as uint32 order keys (4 B/vertex read once from HBM, coalesced
// 128-B rows), and the cells are written once with coalesced 512-B row stores.
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

constexpr int TX = 32;
constexpr uint32_t ABSENT = 0xffffffffu;  // larger than every finite order key
constexpr uint8_t DIR_MIN = 6;

template <int TY, int TZ>
__global__ void __launch_bounds__(256)
init_descent_kernel(const float* __restrict__ f, Cell* __restrict__ C, uint32_t nx, uint32_t ny,
                    uint32_t nz, uint32_t tiles_x, uint32_t tiles_y, uint32_t flip,
                    unsigned long long* __restrict__ counters) {
    constexpr int HX = TX + 2, HY = TY + 2, HZ = TZ + 2;
    constexpr int HALO = HX * HY * HZ;
    __shared__ uint32_t s_ord[HALO];
    __shared__ uint8_t s_dir[TZ * TY * TX];

    const uint32_t b = blockIdx.x;
    const uint32_t bx = b % tiles_x, by = (b / tiles_x) % tiles_y, bz = b / (tiles_x * tiles_y);
    const int64_t x0 = int64_t(bx) * TX, y0 = int64_t(by) * TY, z0 = int64_t(bz) * TZ;
    const uint64_t sxy = uint64_t(nx) * ny;

    // --- stage the haloed tile of order keys (K1 fused into the load) ----
    bool bad = false;
    for (int i = threadIdx.x; i < HALO; i += blockDim.x) {
        const int hx = i % HX, hy = (i / HX) % HY, hz = i / (HX * HY);
        const int64_t gx = x0 + hx - 1, gy = y0 + hy - 1, gz = z0 + hz - 1;
        uint32_t o = ABSENT;
        if (gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz) {
            const float v = __ldg(f + (uint64_t(gz) * sxy + uint64_t(gy) * nx + uint64_t(gx)));
            // only the tile's own cells report non-finite values (halo cells belong to neighbours)
            bad |= nonfinite(v) && hx >= 1 && hx <= TX && hy >= 1 && hy <= TY && hz >= 1 && hz <= TZ;
            o = ord32(v) ^ flip;
        }
        s_ord[i] = o;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(counters + CTR_ERR, ERR_NONFINITE);

    // --- steepest descent direction of every tile vertex -----------------
    const int lx = threadIdx.x & 31;
    const int ly0 = threadIdx.x >> 5;  // 0..7
    // neighbour offsets in the halo array and in global ids: -x +x -y +y -z +z
    const int hoff[6] = {-1, 1, -HX, HX, -HX * HY, HX * HY};
    for (int r = ly0; r < TY * TZ; r += 8) {
        const int ly = r % TY, lz = r / TY;
        const int h = (lz + 1) * HX * HY + (ly + 1) * HX + (lx + 1);
        const int64_t gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        uint8_t dir = DIR_MIN;
        if (gx < nx && gy < ny && gz < nz) {
            const uint32_t id = uint32_t(gz * sxy + gy * nx + gx);
            uint64_t best = key_of(s_ord[h], id);
            const int64_t gid_off[6] = {-1, 1, -int64_t(nx), int64_t(nx), -int64_t(sxy), int64_t(sxy)};
#pragma unroll
            for (int d = 0; d < 6; ++d) {
                const uint32_t o = s_ord[h + hoff[d]];
                if (o == ABSENT) continue;
                const uint64_t k = key_of(o, uint32_t(int64_t(id) + gid_off[d]));
                if (k < best) {
                    best = k;
                    dir = uint8_t(d);
                }
            }
        }
        s_dir[r * TX + lx] = dir;
    }
    __syncthreads();

    // --- tile-local descent: follow directions while inside the tile -----
    for (int r = ly0; r < TY * TZ; r += 8) {
        const int ly = r % TY, lz = r / TY;
        const int64_t gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        if (gx >= nx || gy >= ny || gz >= nz) continue;
        const uint64_t u = uint64_t(gz) * sxy + uint64_t(gy) * nx + uint64_t(gx);
        int cx = lx, cy = ly, cz = lz;
        uint8_t d = s_dir[r * TX + lx];
        while (d != DIR_MIN) {
            const int step = (d & 1) ? 1 : -1;  // d: 0 -x, 1 +x, 2 -y, 3 +y, 4 -z, 5 +z
            const int axis = d >> 1;
            cx += axis == 0 ? step : 0;
            cy += axis == 1 ? step : 0;
            cz += axis == 2 ? step : 0;
            if (cx < 0 || cx >= TX || cy < 0 || cy >= TY || cz < 0 || cz >= TZ) break;  // left the tile
            d = s_dir[(cz * TY + cy) * TX + cx];
        }
        const uint64_t p = uint64_t(z0 + cz) * sxy + uint64_t(y0 + cy) * nx + uint64_t(x0 + cx);
        // (u, u, p(u)); p(u) = u at a minimum: root (u, u, u).  16-B cell:
        // key(s) = key(u), owner order key, v.
        const uint32_t o = s_ord[(lz + 1) * HX * HY + (ly + 1) * HX + (lx + 1)];
        C[u] = make_cell(key_of(o, uint32_t(u)), o, uint32_t(p));
    }
}

// Compress the steepest-descent forest: every regular cell (u, u, p) is
// re-pointed at the root of its descent tree, the basin minimum m(u).
// (u, u, m(u)) is a valid triplet (the descent path from u to m(u) lies below
// key(u)) and is the representative Alg. 4 returns at level key(u) in the
// forest, so this is Alg. 5 applied to the start state (DESIGN.md
// derivation F).  Walks run in place; concurrent shortcuts only ever point
// further down the same tree, and each thread writes only its own v field.
__global__ void __launch_bounds__(256) compress_kernel(Cell* C, uint64_t n) {
    for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n;
         u += uint64_t(gridDim.x) * blockDim.x) {
        const Cell c = ld_cell(C + u);
        const uint32_t v = cv_of(c);
        if (v == uint32_t(u)) continue;           // basin minimum (root)
        uint32_t x = v;
        while (true) {
            const Cell cx = ld_cell(C + x);
            const uint32_t nx = cv_of(cx);
            if (nx == x) break;
            x = nx;
        }
        if (x != v) st_cell_v(C + u, x);
    }
}

}  // namespace

void launch_compress(Cell* C, uint64_t n, int num_sms, cudaStream_t stream) {
    uint64_t blocks = (n + 255) / 256;
    const uint64_t cap = uint64_t(num_sms) * 8 * 32;
    if (blocks > cap) blocks = cap;
    compress_kernel<<<uint32_t(blocks), 256, 0, stream>>>(C, n);
}

void launch_init_descent(const float* f, Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, uint32_t flip,
                         unsigned long long* counters, cudaStream_t stream) {
    if (nz == 1) {
        constexpr int TY = 64, TZ = 1;
        const uint32_t tx = (nx + TX - 1) / TX, ty = (ny + TY - 1) / TY, tz = 1;
        init_descent_kernel<TY, TZ><<<tx * ty * tz, 256, 0, stream>>>(f, C, nx, ny, nz, tx, ty, flip, counters);
    } else {
        constexpr int TY = 8, TZ = 8;
        const uint32_t tx = (nx + TX - 1) / TX, ty = (ny + TY - 1) / TY, tz = (nz + TZ - 1) / TZ;
        init_descent_kernel<TY, TZ><<<tx * ty * tz, 256, 0, stream>>>(f, C, nx, ny, nz, tx, ty, flip, counters);
    }
}

}  // namespace mt
