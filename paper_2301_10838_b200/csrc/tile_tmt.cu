// tile_tmt.cu -- K1 + K2 + tile-local K3/K4: the triplet merge tree of every
// 32 x TY x TZ tile (4096 vertices) of the grid, computed in shared memory.
//
// Paper: Alg. 1 applied to the subgraph G_t made of the
// tile's vertices and the grid edges between them.  The merge phase of the
// paper turns a normalized store of a subgraph into the store of a larger
// graph edge by edge, so the union of the tiles' stores is
// a valid starting store for the remaining (tile-crossing) edges, which the
// global kernel merge_cross.cu adds (DESIGN.md derivation G).
//
// Per tile, in shared memory: uint32 order keys ord[] (K1: ord(f) with -0 ->
// +0 and the split complement) and 64-bit cells
//     ord(f[s]) << 32 | s_local << 16 | v_local
// so that the saddle's key (ord_s, s) -- the tie break by local id equals the
// tie break by global id inside a tile, both being lexicographic in (z, y, x)
// -- is compared straight from the cell, without a lookup:
//   a. steepest descent over in-tile neighbours -> forest of (u, u, w) cells
//      (derivation B);
//   b. compress with path compression: every regular cell points at its
//      basin minimum (derivation F);
//   c. compact the in-tile edges between two basins into a list;
//   d. merge them: Alg. 4-style walks at the edge level with path splitting,
//      then Alg. 3 with 64-bit shared-memory CAS and the root guards R4/R5
//      (DESIGN.md), as a warp-converged state machine (one shared-memory
//      round-trip per lane per step; idle lanes take the next listed edge);
//   e. repair (Alg. 5 with Alg. 4's walk, reading R20): the tile store is
//      minimal for G_t;
//   f. write the 16-byte global cells (common.cuh) with global ids.
// No halo is needed: only in-tile edges are used here.
//
// Layout: f float32[n] x fastest (reading R10) read once (coalesced 128-B
// rows); 16-B cells written once (coalesced 512-B rows).  One CTA of 512
// threads per tile; 72 KB of dynamic shared memory.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

constexpr int TX = 32;
constexpr int THREADS = 512;
constexpr int NV = 4096;                       // vertices per tile
constexpr uint32_t ABSENT = 0xffffffffu;       // order key of a tile slot outside the grid
constexpr size_t SMEM_BYTES = NV * 8 + NV * 4 + NV * 3 * 2 + 16;

__device__ __forceinline__ uint32_t c_v(uint64_t c) { return uint32_t(c) & 0xffffu; }
__device__ __forceinline__ uint32_t c_s(uint64_t c) { return (uint32_t(c) >> 16) & 0xffffu; }
__device__ __forceinline__ uint64_t c_key(uint64_t c) { return c >> 16; }     // (ord_s, s)
__device__ __forceinline__ uint64_t c_make(uint32_t ord_s, uint32_t s, uint32_t v) {
    return (uint64_t(ord_s) << 32) | (s << 16) | v;
}
__device__ __forceinline__ uint64_t key48(const uint32_t* ord, uint32_t x) {
    return (uint64_t(ord[x]) << 16) | x;
}
__device__ __forceinline__ uint64_t sld64(const uint64_t* p) {
    return *reinterpret_cast<const volatile uint64_t*>(p);
}
__device__ __forceinline__ void sst64(uint64_t* p, uint64_t v) {
    *reinterpret_cast<volatile uint64_t*>(p) = v;
}
__device__ __forceinline__ uint64_t scas64(uint64_t* p, uint64_t cmp, uint64_t val) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(p), cmp, val);
}

template <int TY, int TZ, int MODE>
__global__ void __launch_bounds__(THREADS)
tile_tmt_kernel(const float* __restrict__ f, Cell* __restrict__ C, uint32_t nx, uint32_t ny, uint32_t z_begin,
                uint32_t z_end, uint32_t tiles_x, uint32_t tiles_y, uint32_t flip, unsigned long long* __restrict__ counters,
                unsigned long long* __restrict__ stats) {
    constexpr int ROWS = TY * TZ;               // 128 rows of 32
    static_assert(TX * ROWS == NV, "tile size");
    constexpr int RSTEP = THREADS / TX;         // 16 rows per pass
    constexpr int PER = ROWS / RSTEP;           // 8 vertices per thread
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* cell = reinterpret_cast<uint64_t*>(smem);
    uint32_t* ord = reinterpret_cast<uint32_t*>(smem + NV * 8);
    uint16_t* elist = reinterpret_cast<uint16_t*>(smem + NV * 12);
    uint32_t* s_ctl = reinterpret_cast<uint32_t*>(smem + NV * 12 + NV * 6);   // [0] list length, [1] fetch

    unsigned long long n_edges = 0, n_hops = 0, n_iters = 0, n_rep = 0, n_cmp = 0, n_steps = 0, n_active = 0;
    long long t_mark = clock64();
    // per-phase SM cycles (stats mode): thread 0 accumulates the time between barriers
    auto phase_time = [&](int slot) {
        if (stats && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(stats + slot, (unsigned long long)(t - t_mark));
            t_mark = t;
        }
    };

    const uint32_t b = blockIdx.x;
    const uint32_t bx = b % tiles_x, by = (b / tiles_x) % tiles_y, bz = b / (tiles_x * tiles_y);
    // f and C are indexed by GLOBAL vertex id (the caller passes pointers shifted by the
    // slab's first id); this CTA's tile starts at global plane z0
    const uint32_t x0 = bx * TX, y0 = by * TY, z0 = z_begin + bz * TZ;
    const uint64_t sxy = uint64_t(nx) * ny;
    const int lx = threadIdx.x & (TX - 1);
    const int r0 = threadIdx.x / TX;
    const int lane = threadIdx.x & 31;

    // ---- K1: load f once, order keys into shared memory ------------------------------
    bool bad = false;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int r = r0 + k * RSTEP;
        const int ly = r % TY, lz = r / TY;
        const uint32_t gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        uint32_t o = ABSENT;
        if (gx < nx && gy < ny && gz < z_end) {
            const float val = __ldg(f + (uint64_t(gz) * sxy + uint64_t(gy) * nx + gx));
            bad |= nonfinite(val);
            o = ord32(val) ^ flip;
        }
        ord[r * TX + lx] = o;
    }
    if (threadIdx.x < 2) s_ctl[threadIdx.x] = 0;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(counters + CTR_ERR, ERR_NONFINITE);
    phase_time(ST_CYC_LOAD);

    // ---- a. steepest descent over in-tile neighbours -----------------------------------
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int r = r0 + k * RSTEP;
        const int ly = r % TY, lz = r / TY;
        const uint32_t u = r * TX + lx;
        uint32_t best = u;
        const uint32_t ou = ord[u];
        if (ou != ABSENT) {
            uint64_t kb = (uint64_t(ou) << 16) | u;
            const uint32_t nb[6] = {lx > 0 ? u - 1 : u, lx + 1 < TX ? u + 1 : u,
                                    ly > 0 ? u - TX : u, ly + 1 < TY ? u + TX : u,
                                    lz > 0 ? u - TX * TY : u, lz + 1 < TZ ? u + TX * TY : u};
#pragma unroll
            for (int d = 0; d < 6; ++d) {
                const uint32_t w = nb[d];
                const uint32_t ow = ord[w];
                const uint64_t kw = (uint64_t(ow) << 16) | w;
                if (w != u && ow != ABSENT && kw < kb) {
                    kb = kw;
                    best = w;
                }
            }
        }
        cell[u] = c_make(ou, u, best);
    }
    __syncthreads();
    phase_time(ST_CYC_DESCENT);

    // ---- b. compress with path compression ---------------------------------------------
#pragma unroll 1
    for (int k = 0; k < PER; ++k) {
        const uint32_t u = (r0 + k * RSTEP) * TX + lx;
        const uint32_t v = c_v(cell[u]);
        if (v == u) continue;
        uint32_t x = v;
        while (true) {
            const uint32_t y = c_v(sld64(cell + x));
            if (y == x) break;
            x = y;
            ++n_cmp;
        }
        // every regular cell on the path gets the root too (same tree, same basin)
        uint32_t y = v;
        while (y != x) {
            const uint64_t cy = sld64(cell + y);
            const uint32_t nxt = c_v(cy);
            if (nxt != x) sst64(cell + y, (cy & ~0xffffull) | x);
            y = nxt;
        }
        sst64(cell + u, (cell[u] & ~0xffffull) | x);
    }
    __syncthreads();
    phase_time(ST_CYC_COMPRESS);

    // ---- c. list the in-tile edges between two basins ----------------------------------
#pragma unroll 1
    for (int k = 0; k < PER; ++k) {
        const int r = r0 + k * RSTEP;
        const int ly = r % TY, lz = r / TY;
        const uint32_t u = r * TX + lx;
        uint32_t mine = 0;                     // up to 3 entries, bit-packed
        int cnt = 0;
        if (ord[u] != ABSENT) {
            const uint64_t cu = cell[u];
            const uint32_t bu = c_v(cu);       // basin (a minimum points at itself)
            const bool ok[3] = {lx + 1 < TX, ly + 1 < TY, lz + 1 < TZ};
            const uint32_t off[3] = {1u, uint32_t(TX), uint32_t(TX * TY)};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                if (!ok[d]) continue;
                const uint32_t w = u + off[d];
                if (ord[w] == ABSENT) continue;
                if (c_v(cell[w]) != bu) {
                    mine |= uint32_t(d) << (2 * cnt);
                    ++cnt;
                }
            }
        }
        // warp-aggregated append
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t tot = __shfl_sync(FULL_MASK, incl, 31);
        uint32_t base = 0;
        if (lane == 31 && tot) base = atomicAdd(s_ctl, tot);
        base = __shfl_sync(FULL_MASK, base, 31) + incl - cnt;
        for (int i = 0; i < cnt; ++i) elist[base + i] = uint16_t((u << 2) | ((mine >> (2 * i)) & 3u));
    }
    __syncthreads();
    phase_time(ST_CYC_LIST);
    const uint32_t nlist = s_ctl[0];

    // ---- d. merge the listed edges -------------------------------------------------------
    if (MODE == 1) {
        // per-thread loops: thread t takes entries t, t + 512, ...
#pragma unroll 1
        for (uint32_t i = threadIdx.x; i < nlist; i += THREADS) {
            const uint32_t e = elist[i];
            const uint32_t u = e >> 2, d = e & 3u;
            const uint32_t w = u + (d == 0 ? 1u : (d == 1 ? uint32_t(TX) : uint32_t(TX * TY)));
            const uint64_t ku = key48(ord, u), kw = key48(ord, w);
            const uint64_t cu0 = sld64(cell + u), cw0 = sld64(cell + w);
            const uint32_t bu = c_s(cu0) == u ? c_v(cu0) : u;
            const uint32_t bw = c_s(cw0) == w ? c_v(cw0) : w;
            const uint64_t L = ku > kw ? ku : kw;
            ++n_edges;
            uint32_t rr[2];
#pragma unroll
            for (int side = 0; side < 2; ++side) {       // walks at level L with path splitting
                uint32_t x = (side == 0) == (ku > kw) ? bu : bw;
                uint64_t c = sld64(cell + x);
                uint32_t xp = x;
                uint64_t cp = 0;
                bool has_prev = false;
                while (c_v(c) != x && c_key(c) <= L) {
                    if (has_prev && c_key(c) <= c_key(cp)) scas64(cell + xp, cp, (cp & ~0xffffull) | c_v(c));
                    xp = x;
                    cp = c;
                    has_prev = true;
                    x = c_v(c);
                    c = sld64(cell + x);
                    ++n_hops;
                }
                rr[side] = x;
            }
            if (rr[0] == rr[1]) continue;
            uint32_t mu = rr[0], mv = rr[1];
            uint64_t S = L;
            uint32_t my_iters = 0;
            while (true) {                                // Alg. 3
                ++n_iters;
                ++my_iters;
                const uint64_t cu = sld64(cell + mu), cv = sld64(cell + mv);
                if (c_v(cu) != mu && c_key(cu) < S) { mu = c_v(cu); continue; }   // l.2-4 + R4
                if (c_v(cv) != mv && c_key(cv) < S) { mv = c_v(cv); continue; }   // l.5-8 + R4
                if (mu == mv) break;                                                // l.9-10
                uint32_t uu = mu, vv = mv;
                uint64_t cvv = cv;
                if (key48(ord, mv) < key48(ord, mu)) { uu = mv; vv = mu; cvv = cu; }  // l.11-12
                if (scas64(cell + vv, cvv, (S << 16) | uu) == cvv) {               // l.14
                    if (c_v(cvv) == vv) break;                                      // R5
                    mu = uu;                                                        // l.15
                    S = c_key(cvv);
                    mv = c_v(cvv);
                } else {
                    mu = uu;                                                        // l.17
                    mv = vv;
                }
            }
            if (stats) {
                atomicMax(stats + ST_TILE_MAXITER, (unsigned long long)my_iters);
                if (my_iters > 32) atomicAdd(stats + ST_TILE_LONG, 1ull);
            }
        }
    } else {
    {
        uint32_t pool_next = 0, pool_end = 0;  // warp-uniform
        bool exhausted = false;
        int phase = 0;                          // 0 idle, 1 climb hi, 2 climb lo, 3 merge load, 4 cas, 5 done
        uint32_t x = 0, xp = 0, mlo = 0, rh = 0, mu = 0, mv = 0;
        uint64_t c = 0, cp = 0, cu = 0, cv = 0, L = 0, S = 0, desired = 0, got = 0;
        bool has_prev = false;
        while (true) {
            const uint32_t need = __ballot_sync(FULL_MASK, phase == 0);
            if (need) {
                if (pool_next == pool_end && !exhausted) {
                    uint32_t b0 = 0;
                    if (lane == 0) b0 = atomicAdd(s_ctl + 1, 64u);
                    b0 = __shfl_sync(FULL_MASK, b0, 0);
                    pool_next = b0 < nlist ? b0 : nlist;
                    pool_end = b0 + 64 < nlist ? b0 + 64 : nlist;
                    exhausted = pool_next == pool_end;
                }
                const uint32_t rank = __popc(need & ((1u << lane) - 1u));
                const uint32_t avail = pool_end - pool_next;
                if (phase == 0) {
                    if (rank < avail) {
                        const uint32_t e = elist[pool_next + rank];
                        const uint32_t u = e >> 2, d = e & 3u;
                        const uint32_t w = u + (d == 0 ? 1u : (d == 1 ? uint32_t(TX) : uint32_t(TX * TY)));
                        const uint64_t ku = key48(ord, u), kw = key48(ord, w);
                        // basins: a regular cell (s = self) is static and points at its
                        // minimum; a minimum (possibly merged already) is its own basin
                        const uint64_t cu0 = sld64(cell + u), cw0 = sld64(cell + w);
                        const uint32_t bu = c_s(cu0) == u ? c_v(cu0) : u;
                        const uint32_t bw = c_s(cw0) == w ? c_v(cw0) : w;
                        L = ku > kw ? ku : kw;
                        x = ku > kw ? bu : bw;
                        mlo = ku > kw ? bw : bu;
                        has_prev = false;
                        phase = 1;
                        ++n_edges;
                    } else if (exhausted) {
                        phase = 5;
                    }
                }
                pool_next += avail < uint32_t(__popc(need)) ? avail : uint32_t(__popc(need));
            }
            const uint32_t live = __ballot_sync(FULL_MASK, phase != 5);
            if (live == 0) break;
            if (stats) {
                const uint32_t busy = __ballot_sync(FULL_MASK, phase != 0);   // lanes with an edge this step
                if (lane == 0) {
                    ++n_steps;
                    n_active += __popc(busy & live);
                }
            }
            // one shared-memory round-trip
            if (phase == 1 || phase == 2) {
                c = sld64(cell + x);
            } else if (phase == 3) {
                cu = sld64(cell + mu);
                cv = sld64(cell + mv);
            } else if (phase == 4) {
                got = scas64(cell + mv, cv, desired);
            }
            // advance
            if (phase == 1 || phase == 2) {
                if (c_v(c) != x && c_key(c) <= L) {                         // followable at level L
                    if (has_prev && c_key(c) <= c_key(cp))                   // path splitting
                        scas64(cell + xp, cp, (cp & ~0xffffull) | c_v(c));
                    xp = x;
                    cp = c;
                    has_prev = true;
                    x = c_v(c);
                    ++n_hops;
                } else if (phase == 1) {
                    rh = x;
                    x = mlo;
                    has_prev = false;
                    phase = 2;
                } else if (x == rh) {
                    phase = 0;                                               // already joined
                } else {
                    mu = rh;                                                 // Merge(T, rh, hi, x)
                    mv = x;
                    S = L;
                    phase = 3;
                }
            } else if (phase == 3) {
                ++n_iters;
                if (c_v(cu) != mu && c_key(cu) < S) {                        // l.2-4 + R4
                    mu = c_v(cu);
                } else if (c_v(cv) != mv && c_key(cv) < S) {                 // l.5-8 + R4
                    mv = c_v(cv);
                } else if (mu == mv) {                                       // l.9-10
                    phase = 0;
                } else {
                    if (key48(ord, mv) < key48(ord, mu)) {                   // l.11-12
                        const uint32_t t = mu; mu = mv; mv = t;
                        const uint64_t tc = cu; cu = cv; cv = tc;
                    }
                    desired = (S << 16) | mu;                                // l.14: (s, u) into T[v]
                    phase = 4;
                }
            } else if (phase == 4) {
                if (got == cv) {
                    if (c_v(cv) == mv) {
                        phase = 0;                                           // displaced a root (R5)
                    } else {
                        S = c_key(cv);                                       // l.15
                        mv = c_v(cv);
                        phase = 3;
                    }
                } else {
                    phase = 3;                                               // l.17
                }
            }
        }
    }
    }
    __syncthreads();
    phase_time(ST_CYC_MERGE);

    // ---- e. repair: every cell points at its representative (minimal tile store) -------
#pragma unroll 1
    for (int k = 0; k < PER; ++k) {
        const uint32_t u = (r0 + k * RSTEP) * TX + lx;
        const uint64_t cu = cell[u];
        const uint32_t v = c_v(cu);
        if (v == u) continue;
        const uint64_t a = c_key(cu);
        uint32_t x = v;
        while (true) {
            const uint64_t cx = sld64(cell + x);
            if (c_v(cx) == x || c_key(cx) > a) break;
            x = c_v(cx);
            ++n_rep;
        }
        if (x != v) sst64(cell + u, (cu & ~0xffffull) | x);
    }
    __syncthreads();
    phase_time(ST_CYC_REPAIR);

    // ---- f. write the global 16-byte cells ---------------------------------------------
    const uint64_t gbase = uint64_t(z0) * sxy + uint64_t(y0) * nx + x0;
    auto gid = [&](uint32_t l) -> uint32_t {
        const uint32_t l_x = l % TX, l_r = l / TX;
        return uint32_t(gbase + uint64_t(l_r / TY) * sxy + uint64_t(l_r % TY) * nx + l_x);
    };
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int r = r0 + k * RSTEP;
        const int ly = r % TY, lz = r / TY;
        const uint32_t u = r * TX + lx;
        const uint32_t ou = ord[u];
        if (ou == ABSENT) continue;
        const uint64_t cu = cell[u];
        const uint32_t s = c_s(cu), v = c_v(cu);
        C[gbase + uint64_t(lz) * sxy + uint64_t(ly) * nx + lx] =
            make_cell(key_of(uint32_t(cu >> 32), gid(s)), ou, gid(v));
    }
    phase_time(ST_CYC_WRITE);
    if (stats) {
        atomicAdd(stats + ST_TILE_EDGES, n_edges);
        atomicAdd(stats + ST_TILE_HOPS, n_hops);
        atomicAdd(stats + ST_TILE_ITERS, n_iters);
        atomicAdd(stats + ST_TILE_REPAIR, n_rep);
        atomicAdd(stats + ST_TILE_COMPRESS, n_cmp);
        atomicAdd(stats + ST_TILE_STEPS, n_steps);
        atomicAdd(stats + ST_TILE_ACTIVE, n_active);
    }
}

}  // namespace

void tile_shape(uint32_t nz_global, uint32_t* ty, uint32_t* tz) {
    if (nz_global == 1) {
        *ty = 128;
        *tz = 1;
    } else {
        *ty = 16;
        *tz = 8;
    }
}

void launch_tile_tmt(const float* f, Cell* C, const Slab& sl, uint32_t flip, unsigned long long* counters,
                     unsigned long long* stats, cudaStream_t stream) {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("MT_TILE_MODE");  // diagnostics: 0 state machine, 1 per-thread loops
        mode = e ? atoi(e) : 1;
        cudaFuncSetAttribute(tile_tmt_kernel<128, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
        cudaFuncSetAttribute(tile_tmt_kernel<16, 8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
        cudaFuncSetAttribute(tile_tmt_kernel<128, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
        cudaFuncSetAttribute(tile_tmt_kernel<16, 8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    }
    uint32_t ty, tz;
    tile_shape(sl.nz, &ty, &tz);
    const uint32_t nzl = sl.z_end - sl.z_begin;
    const uint32_t tx = (sl.nx + TX - 1) / TX, tyn = (sl.ny + ty - 1) / ty, tzn = (nzl + tz - 1) / tz;
    const uint32_t grid = tx * tyn * tzn;
    if (grid == 0) return;
#define MT_TILE_LAUNCH(TY_, TZ_, M_)                                                                     \
    tile_tmt_kernel<TY_, TZ_, M_><<<grid, THREADS, SMEM_BYTES, stream>>>(f, C, sl.nx, sl.ny, sl.z_begin, \
                                                                         sl.z_end, tx, tyn, flip, counters, stats)
    if (sl.nz == 1 && mode == 0)
        MT_TILE_LAUNCH(128, 1, 0);
    else if (sl.nz == 1)
        MT_TILE_LAUNCH(128, 1, 1);
    else if (mode == 0)
        MT_TILE_LAUNCH(16, 8, 0);
    else
        MT_TILE_LAUNCH(16, 8, 1);
#undef MT_TILE_LAUNCH
}

}  // namespace mt
