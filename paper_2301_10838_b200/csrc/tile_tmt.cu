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
//   b. compress by synchronous pointer jumping: every regular cell points at
//      its basin minimum (derivations F, F');
//   c. list the in-tile edges between two basins, keeping the lowest per
//      basin pair (staged per warp, inserted 32 at a time into a hash table);
//   d. merge them: Alg. 3 from the two basins at the edge's level with 64-bit
//      shared-memory CAS and the root guards R4/R5, one lane per
//      pair, one shared-memory round trip per loop iteration; a lane whose
//      pair is done takes the next pair of the warp's compacted run;
//   e. repair (Alg. 5 with Alg. 4's walk, reading R20): the tile store is
//      minimal for G_t (each thread's walks in lock-step rounds);
//   f. write the 16-byte global cells (common.cuh) with global ids, and each
//      vertex's tile representative at its own level for the crossing edges
//      (derivation C''').
// No halo is needed: only in-tile edges are used here.
//
// Layout: f float32[n] x fastest (reading R10) read once (coalesced 128-B
// rows); 16-B cells written once (coalesced 512-B rows).  One CTA of 512
// threads per tile; 112 KB of dynamic shared memory (2 CTAs per SM).
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

#ifndef TILE_SPLIT
#define TILE_SPLIT 1   // path splitting in the merge-phase walks (A/B knob)
#endif
#ifndef TILE_STOP
#define TILE_STOP 0    // timing only (WRONG results): run phases < k: 1 load+descent, 2 +compress, 3 +list, 4 +merge
#endif
#ifndef TILE_LEAN
#define TILE_LEAN 1    // merge phase: Alg. 3 only, no phase variable (requires TILE_OWNRUN)
#endif
#ifndef TILE_WALK
#define TILE_WALK 0    // merge phase: filter walks (with path splitting) before Alg. 3
#endif
#ifndef LIST_STAGE
#define LIST_STAGE 1   // list phase: per-warp staging of the candidate edges, inserts 32 at a time
#endif
#ifndef TILE_MINB
#define TILE_MINB 2    // __launch_bounds__ min blocks per SM (register budget knob)
#endif
#ifndef TILE_REP_ILP
#define TILE_REP_ILP 1 // in-tile repair: own vertices in lock-step rounds, results in registers
#endif
#ifndef TILE_PJ
#define TILE_PJ 1      // compress by synchronous pointer jumping (else walks + path compression)
#endif
#ifndef TILE_OWNRUN
#define TILE_OWNRUN 1  // each warp merges the pairs of its own compacted run (no CTA counter)
#endif
#if TILE_LEAN && (TILE_WALK || !TILE_OWNRUN)
#error "TILE_LEAN needs TILE_OWNRUN and no TILE_WALK"
#endif

constexpr int TX = 32;
constexpr uint32_t ABSENT = 0xffffffffu;       // order key of a tile slot outside the grid
constexpr uint64_t EMPTY = ~0ull;
// tile of NV vertices, NV / 8 threads (8 vertices each), basin-pair table of 1.5 NV slots
// (2 NV without the staging buffers), staging buffer of 128 entries per warp
constexpr int table_slots(int nv) { return LIST_STAGE ? 3 * nv / 2 : 2 * nv; }
template <int NV>
constexpr size_t smem_bytes() {
    return size_t(NV) * 8 + size_t(NV) * 4 + size_t(table_slots(NV)) * 8 + (LIST_STAGE ? size_t(NV) * 4 : 0);
}

template <int TABLE>
__device__ __forceinline__ uint32_t pair_hash(uint32_t p) {
    p ^= p >> 13;
    p *= 0x5bd1e995u;
    p ^= p >> 15;
    return uint32_t((uint64_t(p) * TABLE) >> 32);
}

__device__ __forceinline__ uint32_t c_v(uint64_t c) { return uint32_t(c) & 0xffffu; }
__device__ __forceinline__ uint32_t c_s(uint64_t c) { return (uint32_t(c) >> 16) & 0xffffu; }
__device__ __forceinline__ uint64_t c_key(uint64_t c) { return c >> 16; }     // (ord_s, s)
__device__ __forceinline__ uint64_t c_make(uint32_t ord_s, uint32_t s, uint32_t v) {
    return (uint64_t(ord_s) << 32) | (s << 16) | v;
}
__device__ __forceinline__ uint64_t key48(const uint32_t* ord, uint32_t x) {
    return (uint64_t(ord[x]) << 16) | x;
}
__device__ __forceinline__ bool lkey_lt(const uint32_t* ord, uint32_t a, uint32_t b) {
    return key48(ord, a) < key48(ord, b);
}
__device__ __forceinline__ uint64_t sld64(const uint64_t* p) {
    return *reinterpret_cast<const volatile uint64_t*>(p);
}
[[maybe_unused]] __device__ __forceinline__ void sst64(uint64_t* p, uint64_t v) {
    *reinterpret_cast<volatile uint64_t*>(p) = v;
}
__device__ __forceinline__ uint64_t scas64(uint64_t* p, uint64_t cmp, uint64_t val) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(p), cmp, val);
}

template <int TY, int TZ, bool STATS, int NV = TX * TY * TZ, int THREADS = NV / 8, int TABLE = table_slots(NV)>
__global__ void __launch_bounds__(THREADS, TILE_MINB)
tile_tmt_kernel(const float* __restrict__ f, Cell* __restrict__ C, uint64_t* __restrict__ T0,
                uint64_t* __restrict__ xface, uint32_t nx,
                uint32_t ny, uint32_t z_begin,
                uint32_t z_end, uint32_t tiles_x, uint32_t tiles_y, uint32_t flip, unsigned long long* __restrict__ counters,
                unsigned long long* __restrict__ stats) {
    constexpr int ROWS = TY * TZ;               // 128 rows of 32
    static_assert(TX * ROWS == NV, "tile size");
    constexpr int RSTEP = THREADS / TX;         // 16 rows per pass
    constexpr int PER = ROWS / RSTEP;           // 8 vertices per thread
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* cell = reinterpret_cast<uint64_t*>(smem);
    uint32_t* ord = reinterpret_cast<uint32_t*>(smem + NV * 8);
    uint64_t* table = reinterpret_cast<uint64_t*>(smem + NV * 12);
    __shared__ int s_overflow;
    __shared__ uint32_t s_fetch, s_row, s_row_b, s_row_e;
#if !TILE_OWNRUN
    __shared__ uint32_t s_wcnt[THREADS / 32], s_wpre[THREADS / 32 + 1];
#endif

    unsigned long long n_edges = 0, n_pairs = 0, n_hops = 0, n_iters = 0, n_rep = 0, n_cmp = 0;
    long long t_mark = clock64();
    // per-phase SM cycles (stats mode): thread 0 accumulates the time between barriers
    auto phase_time = [&](int slot) {
        if (STATS && threadIdx.x == 0) {
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
    for (int i = threadIdx.x; i < TABLE; i += THREADS) table[i] = EMPTY;
    if (threadIdx.x == 0) {
        s_overflow = 0;
        s_fetch = 0;
        s_row = 0;
        s_row_b = 0;
        s_row_e = 0;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(counters + CTR_ERR, ERR_NONFINITE);
    phase_time(ST_CYC_LOAD);

    // ---- a. steepest descent over in-tile neighbours -----------------------------------
    uint32_t par[PER];  // descent pointer of each owned vertex (then its basin, phase b)
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
        par[k] = best;
    }
    __syncthreads();
    phase_time(ST_CYC_DESCENT);

    // ---- b. compress: every regular cell points at its basin minimum ----------------------
#if TILE_PJ
    // synchronous pointer jumping, par <- par(par), on the thread's own 8 vertices (8
    // independent load chains per round), until every pointer is a root: ceil(log2 depth) + 1
    // rounds.  Rounds run in place: a pointer read while its owner rewrites it is the old or
    // the new ancestor, both in the same descent tree (derivation F), so the v fields (16-bit
    // stores) only ever move up the tree.
#pragma unroll 1
    while (TILE_STOP == 0 || TILE_STOP > 1) {
        bool changed = false;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t q = *reinterpret_cast<const volatile uint16_t*>(cell + par[k]);
            if (q != par[k]) {
                par[k] = q;
                changed = true;
                *reinterpret_cast<volatile uint16_t*>(cell + (r0 + k * RSTEP) * TX + lx) = uint16_t(q);
                if (STATS) ++n_cmp;
            }
        }
        if (!__syncthreads_or(changed)) break;
    }
#else
    // rows handed out dynamically, one warp per row (no warp waits on a long walk of another)
#pragma unroll 1
    while (TILE_STOP == 0 || TILE_STOP > 1) {
        int rr = 0;
        if ((threadIdx.x & 31) == 0) rr = int(atomicAdd(&s_row_b, 1u));
        rr = __shfl_sync(FULL_MASK, rr, 0);
        if (rr >= ROWS) break;
        const uint32_t u = rr * TX + lx;
        const uint32_t v = c_v(cell[u]);
        if (v == u) continue;
        uint32_t x = v;
        while (true) {
            const uint32_t y = c_v(sld64(cell + x));
            if (y == x) break;
            x = y;
            if (STATS) ++n_cmp;
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
#endif
    __syncthreads();
    phase_time(ST_CYC_COMPRESS);

    // ---- c. one edge per pair of adjacent basins: the lowest --------------------------------
    // Between two basins A and B only the lowest edge matters: any other A-B edge at level
    // L' joins vertices that are already connected at L' through their descent paths and
    // that lowest edge (DESIGN.md derivation C'').  A shared-memory hash table keyed by the
    // basin pair keeps, per pair, the edge's upper endpoint of lowest key.
    const int lane_c = threadIdx.x & 31;
    // keep, per basin pair, the edge of lowest level (entry = pair << 12 | upper endpoint)
    auto insert_entry = [&](uint64_t entry) {
        const uint32_t pair = uint32_t(entry >> 12);
        const uint64_t kh = key48(ord, uint32_t(entry) & 0xfffu);
        uint32_t h = pair_hash<TABLE>(pair);
        for (uint32_t probe = 0;;) {
            const uint64_t cur = sld64(table + h);
            if (cur == EMPTY) {
                if (scas64(table + h, EMPTY, entry) == EMPTY) break;
                continue;                                        // lost the slot: re-read it
            }
            if (uint32_t(cur >> 12) != pair) {
                h = h + 1 == uint32_t(TABLE) ? 0u : h + 1;
                if (++probe < uint32_t(TABLE)) continue;
                // table full (e.g. a checkerboard: every vertex pair of basins is adjacent):
                // record the edge in the overflow flag; phase d' merges all edges then
                s_overflow = 1;
                break;
            }
            if (kh >= key48(ord, uint32_t(cur) & 0xfffu)) break;  // the stored edge is lower
            if (scas64(table + h, cur, entry) == cur) break;
        }
    };
    // the in-tile edge (u, w) in direction d (+x, +y, +z) if its ends lie in two basins
    auto candidate = [&](uint32_t u, uint32_t ou, uint32_t bu, bool ok, uint32_t off, uint64_t* entry) {
        if (ou == ABSENT || !ok) return false;
        const uint32_t w = u + off;
        const uint32_t ow = ord[w];
        if (ow == ABSENT) return false;
        const uint32_t bw = c_v(cell[w]);
        if (bw == bu) return false;
        const bool u_hi = ((uint64_t(ow) << 16) | w) < ((uint64_t(ou) << 16) | u);
        const uint32_t hi = u_hi ? u : w;
        const uint32_t pair = bu < bw ? (bu << 12) | bw : (bw << 12) | bu;
        // bit 63: the upper endpoint lies in the pair's first (smaller) basin
        *entry = (uint64_t(pair) << 12) | hi | (uint64_t((u_hi ? bu : bw) == (bu < bw ? bu : bw)) << 63);
        return true;
    };
#if LIST_STAGE
    // each warp lists the edges of its own rows into a 128-entry staging buffer (ballot +
    // popc) and inserts them 32 at a time, so the insert code runs with every lane busy
    // (about 40 % of the in-tile edges join two basins)
    if (TILE_STOP == 0 || TILE_STOP > 2) {
        uint64_t* stage = reinterpret_cast<uint64_t*>(smem + NV * 12 + TABLE * 8) + (threadIdx.x >> 5) * 128;
        const uint32_t lt = (1u << lane_c) - 1u;
        uint32_t nst = 0;
#pragma unroll 1
        for (int k = 0; k < PER; ++k) {
            const int r = r0 + k * RSTEP;
            const int ly = r % TY, lz = r / TY;
            const uint32_t u = r * TX + lx;
            const uint32_t ou = ord[u];
            const uint32_t bu = c_v(cell[u]);      // basin (a minimum points at itself)
            const bool ok[3] = {lx + 1 < TX, ly + 1 < TY, lz + 1 < TZ};
            const uint32_t off[3] = {1u, uint32_t(TX), uint32_t(TX * TY)};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                uint64_t entry = 0;
                const bool valid = candidate(u, ou, bu, ok[d], off[d], &entry);
                const uint32_t m = __ballot_sync(FULL_MASK, valid);
                if (valid) stage[nst + __popc(m & lt)] = entry;
                nst += __popc(m);
                if (STATS && valid) ++n_edges;
            }
            __syncwarp();
            while (nst >= 32) {
                const uint64_t e = stage[nst - 32 + lane_c];
                __syncwarp();
                nst -= 32;
                insert_entry(e);
            }
        }
        if (uint32_t(lane_c) < nst) insert_entry(stage[lane_c]);
    }
#else
    // rows of 32 vertices are handed out dynamically (a warp per row) so that warps with
    // contended inserts do not hold the barrier for the others
#pragma unroll 1
    while (TILE_STOP == 0 || TILE_STOP > 2) {
        int r = 0;
        if (lane_c == 0) r = int(atomicAdd(&s_row, 1u));
        r = __shfl_sync(FULL_MASK, r, 0);
        if (r >= ROWS) break;
        const int ly = r % TY, lz = r / TY;
        const uint32_t u = r * TX + lx;
        const uint32_t ou = ord[u];
        const uint32_t bu = c_v(cell[u]);      // basin (a minimum points at itself)
        const bool ok[3] = {lx + 1 < TX, ly + 1 < TY, lz + 1 < TZ};
        const uint32_t off[3] = {1u, uint32_t(TX), uint32_t(TX * TY)};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            uint64_t entry = 0;
            if (!candidate(u, ou, bu, ok[d], off[d], &entry)) continue;
            if (STATS) ++n_edges;
            insert_entry(entry);
        }
    }
#endif
    __syncthreads();
    phase_time(ST_CYC_LIST);

    // ---- d. merge one edge per basin pair ------------------------------------------------
    // join basins bh (the one holding the edge's upper endpoint) and bl at level L
    auto merge_at = [&](uint32_t bh, uint32_t bl, uint64_t L) {
        uint32_t rr[2];
#pragma unroll
        for (int side = 0; side < 2; ++side) {           // walks at level L with path splitting
            uint32_t x = side == 0 ? bh : bl;
            uint64_t c = sld64(cell + x);
            uint32_t xp = x;
            uint64_t cp = 0;
            bool has_prev = false;
            while (c_v(c) != x && c_key(c) <= L) {
                if (TILE_SPLIT && has_prev && c_key(c) <= c_key(cp))
                    scas64(cell + xp, cp, (cp & ~0xffffull) | c_v(c));
                xp = x;
                cp = c;
                has_prev = true;
                x = c_v(c);
                c = sld64(cell + x);
                if (STATS) ++n_hops;
            }
            rr[side] = x;
        }
        if (rr[0] == rr[1]) return;
        uint32_t mu = rr[0], mv = rr[1];
        uint64_t S = L;
        while (true) {                                    // Alg. 3
            if (STATS) ++n_iters;
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
    };
    // basin of x: a regular cell (s = x) is static and points at the minimum
    auto basin = [&](uint32_t x) {
        const uint64_t c = sld64(cell + x);
        return c_s(c) == x ? c_v(c) : x;
    };
    // d0. most table slots are empty (c5: ~1200 pairs in 8192 slots): every warp compacts
    // its 1/NW of the table in place (a chunk of 32 slots is read before any of its lanes
    // writes, and a write never lands past the chunk being read), then the pairs are handed
    // out one per fetch from a CTA counter over the concatenated runs, so that every
    // fetch yields a pair and every lane of a warp works on one
    constexpr int NW = THREADS / 32, REG = TABLE / NW;
    const int warp_d = threadIdx.x >> 5;
    uint64_t* const run = table + warp_d * REG;          // this warp's run of pairs
    uint32_t run_len = 0;
#pragma unroll 4
    for (int c = 0; c < REG; c += 32) {
        const uint64_t e = run[c + lane_c];
        const uint32_t m = __ballot_sync(FULL_MASK, e != EMPTY);
        __syncwarp();
        if (e != EMPTY) run[run_len + __popc(m & ((1u << lane_c) - 1u))] = e;
        run_len += __popc(m);
    }
    if (TILE_STOP != 0 && TILE_STOP <= 3) run_len = 0;
#if !TILE_OWNRUN
    if (lane_c == 0) s_wcnt[warp_d] = run_len;
    __syncthreads();
    if (threadIdx.x < 32) {     // exclusive prefix of the NW run lengths
        const uint32_t c = threadIdx.x < NW ? s_wcnt[threadIdx.x] : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane_c >= o) incl += t;
        }
        if (threadIdx.x <= NW) s_wpre[threadIdx.x] = incl - c;
    }
    __syncthreads();
#endif
#if !TILE_OWNRUN
    const uint32_t n_listed = s_wpre[NW];
    auto listed = [&](uint32_t j) {                       // pair j of the concatenated runs
        int w = 0;                                        // (binary search over the run starts)
#pragma unroll
        for (int step = NW / 2; step > 0; step >>= 1)
            if (s_wpre[w + step] <= j) w += step;
        return table[w * REG + (j - s_wpre[w])];
    };
#endif
#if TILE_LEAN
    // d1. Alg. 3 per lane, one iteration (the two cell loads, + the CAS) per loop iteration; a
    // lane whose pair is done takes the next pair of the warp's run at the top of the next
    // iteration (ballot + popc), so the lanes of a warp stay busy and converged instead of
    // waiting for the longest merge of the warp.  Merge(T, bh, hi, bl) starts straight from
    // the two basins (bh holds the edge's upper endpoint hi, level L = key(hi)).
    bool busy = false;
    uint64_t S = 0;
    uint32_t mu = 0, mv = 0, run_pos = 0;
#pragma unroll 1
    while (true) {
        const uint32_t need = __ballot_sync(FULL_MASK, !busy);
        if (need) {
            if (!busy) {
                const uint32_t j = run_pos + __popc(need & ((1u << lane_c) - 1u));
                if (j < run_len) {
                    const uint64_t e = run[j];
                    if (STATS) ++n_pairs;
                    const uint32_t pair = uint32_t(e >> 12) & 0xffffffu, hi = uint32_t(e) & 0xfffu;
                    const uint32_t ba = pair >> 12, bb = pair & 0xfffu;
                    const bool first = e >> 63;
                    mu = first ? ba : bb;
                    mv = first ? bb : ba;
                    S = key48(ord, hi);
                    busy = true;
                }
            }
            run_pos += __popc(need);
        }
        if (!__any_sync(FULL_MASK, busy)) break;
        if (busy) {
            if (STATS) ++n_iters;
            const uint64_t cu = sld64(cell + mu), cv = sld64(cell + mv);
            if (c_v(cu) != mu && c_key(cu) < S) {         // l.2-4 + R4
                mu = c_v(cu);
            } else if (c_v(cv) != mv && c_key(cv) < S) {  // l.5-8 + R4
                mv = c_v(cv);
            } else if (mu == mv) {                        // l.9-10
                busy = false;
            } else {
                uint32_t uu = mu, vv = mv;
                uint64_t cvv = cv;
                if (key48(ord, mv) < key48(ord, mu)) { uu = mv; vv = mu; cvv = cu; }   // l.11-12
                const uint64_t got = scas64(cell + vv, cvv, (S << 16) | uu);          // l.14
                mu = uu;
                if (got == cvv) {
                    if (c_v(cvv) == vv) busy = false;      // R5: displaced a root
                    S = c_key(cvv);                       // l.15: Merge(T, u, s_v, v')
                    mv = c_v(cvv);
                } else {
                    mv = vv;                              // l.17: restart
                }
            }
        }
    }
#else
    // d1. one state machine per lane, advanced by one shared-memory round trip per loop
    // iteration (a walk step, the pair of Alg. 3 loads (+ CAS)); a lane whose pair is done
    // takes the next listed pair at the top of the next iteration, so the lanes of a warp
    // stay busy and converged instead of waiting for the longest merge of the warp
    enum { P_IDLE = 0, P_W0 = 1, P_W1 = 2, P_A3 = 3, P_DONE = 4 };
    int ph = P_IDLE;
    uint64_t L = 0, S = 0, cp = 0;
    uint32_t x = 0, xp = 0, lo = 0, r0v = 0, mu = 0, mv = 0;
    bool has_prev = false;
    uint32_t run_pos = 0;
#pragma unroll 1
    while (true) {
#if TILE_OWNRUN
        // the warp's own run is its pool: idle lanes take the next pairs in lane order
        const uint32_t need = __ballot_sync(FULL_MASK, ph == P_IDLE);
        if (need) {
            if (ph == P_IDLE) {
                const uint32_t j = run_pos + __popc(need & ((1u << lane_c) - 1u));
                if (j < run_len) {
                    const uint64_t e = run[j];
#else
        if (ph == P_IDLE) {
            {
                const uint32_t j = atomicAdd(&s_fetch, 1u);
                if (j < n_listed) {
                    const uint64_t e = listed(j);
#endif
                    if (STATS) ++n_pairs;
                    const uint32_t pair = uint32_t(e >> 12), hi = uint32_t(e) & 0xfffu;
                    const uint32_t ba = pair >> 12, bb = pair & 0xfffu;
                    const uint32_t bh = basin(hi);
                    L = key48(ord, hi);                   // join bh and the other basin at level L
                    x = bh;
                    lo = bh == ba ? bb : ba;
                    has_prev = false;
                    ph = P_W0;
                    if (!TILE_WALK) {                     // Merge(T, bh, hi, bl) straight away
                        mu = bh;
                        mv = lo;
                        S = L;
                        ph = P_A3;
                    }
                } else {
                    ph = P_DONE;
                }
            }
#if TILE_OWNRUN
            run_pos += __popc(need);
#endif
        }
        if (__all_sync(FULL_MASK, ph == P_DONE)) break;
        if (ph == P_W0 || ph == P_W1) {                   // walks at level L with path splitting
            const uint64_t c = sld64(cell + x);
            if (c_v(c) != x && c_key(c) <= L) {
                if (TILE_SPLIT && has_prev && c_key(c) <= c_key(cp))
                    scas64(cell + xp, cp, (cp & ~0xffffull) | c_v(c));
                xp = x;
                cp = c;
                has_prev = true;
                x = c_v(c);
                if (STATS) ++n_hops;
            } else if (ph == P_W0) {
                r0v = x;
                x = lo;
                has_prev = false;
                ph = P_W1;
            } else if (x == r0v) {
                ph = P_IDLE;                              // joined below L already
            } else {
                mu = r0v;
                mv = x;
                S = L;
                ph = P_A3;
            }
        } else if (ph == P_A3) {                          // Alg. 3, one iteration
            if (STATS) ++n_iters;
            const uint64_t cu = sld64(cell + mu), cv = sld64(cell + mv);
            if (c_v(cu) != mu && c_key(cu) < S) {         // l.2-4 + R4
                mu = c_v(cu);
            } else if (c_v(cv) != mv && c_key(cv) < S) {  // l.5-8 + R4
                mv = c_v(cv);
            } else if (mu == mv) {                        // l.9-10
                ph = P_IDLE;
            } else {
                uint32_t uu = mu, vv = mv;
                uint64_t cvv = cv;
                if (key48(ord, mv) < key48(ord, mu)) { uu = mv; vv = mu; cvv = cu; }   // l.11-12
                if (scas64(cell + vv, cvv, (S << 16) | uu) == cvv) {                  // l.14
                    if (c_v(cvv) == vv) {
                        ph = P_IDLE;                      // R5
                    } else {
                        mu = uu;                          // l.15
                        S = c_key(cvv);
                        mv = c_v(cvv);
                    }
                } else {
                    mu = uu;                              // l.17
                    mv = vv;
                }
            }
        }
    }
#endif
    if (s_overflow) {  // (uniform: written before the last barrier) the table dropped edges
#pragma unroll 1
        for (int k = 0; k < PER; ++k) {
            const int r = r0 + k * RSTEP;
            const int ly = r % TY, lz = r / TY;
            const uint32_t u = r * TX + lx;
            if (ord[u] == ABSENT) continue;
            const bool ok[3] = {lx + 1 < TX, ly + 1 < TY, lz + 1 < TZ};
            const uint32_t off[3] = {1u, uint32_t(TX), uint32_t(TX * TY)};
#pragma unroll 1
            for (int d = 0; d < 3; ++d) {
                if (!ok[d]) continue;
                const uint32_t w = u + off[d];
                if (ord[w] == ABSENT) continue;
                const uint32_t bu = basin(u), bw = basin(w);
                if (bu == bw) continue;
                const bool u_hi = lkey_lt(ord, w, u);
                merge_at(u_hi ? bu : bw, u_hi ? bw : bu, key48(ord, u_hi ? u : w));
            }
        }
    }
    __syncthreads();
    phase_time(ST_CYC_MERGE);

    // ---- e. repair: every cell points at its representative (minimal tile store) -------
#if TILE_REP_ILP
    // each thread walks its own 8 vertices in lock-step rounds (8 independent shared-memory
    // load chains in flight); the cells are final after the merge barrier and this phase only
    // reads them, so the representatives stay in registers and go straight to phase f
    uint32_t rep[PER];
    uint32_t act = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint32_t u = (r0 + k * RSTEP) * TX + lx;
        rep[k] = c_v(cell[u]);
        if (rep[k] != u && (TILE_STOP == 0 || TILE_STOP > 4)) act |= 1u << k;
    }
#pragma unroll 1
    while (act) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            if (!((act >> k) & 1u)) continue;
            const uint64_t cx = cell[rep[k]];
            const uint64_t a = c_key(cell[(r0 + k * RSTEP) * TX + lx]);
            if (c_v(cx) == rep[k] || c_key(cx) > a) {
                act &= ~(1u << k);
            } else {
                rep[k] = c_v(cx);
                if (STATS) ++n_rep;
            }
        }
    }
#else
#pragma unroll 1
    while (TILE_STOP == 0 || TILE_STOP > 4) {
        int rr = 0;
        if ((threadIdx.x & 31) == 0) rr = int(atomicAdd(&s_row_e, 1u));
        rr = __shfl_sync(FULL_MASK, rr, 0);
        if (rr >= ROWS) break;
        const uint32_t u = rr * TX + lx;
        const uint64_t cu = cell[u];
        const uint32_t v = c_v(cu);
        if (v == u) continue;
        const uint64_t a = c_key(cu);
        uint32_t x = v;
        while (true) {
            const uint64_t cx = sld64(cell + x);
            if (c_v(cx) == x || c_key(cx) > a) break;
            x = c_v(cx);
            if (STATS) ++n_rep;
        }
        if (x != v) sst64(cell + u, (cu & ~0xffffull) | x);
    }
    __syncthreads();
#endif
    phase_time(ST_CYC_REPAIR);

    // ---- f. write the tile store T0 (8 B per vertex) and the tile minima's 16-byte cells ------
    // T0[u] = s << 32 | v with global ids, into the caller's triplet buffer: for a regular vertex
    // (u, Rep_tile(u, key(u))) -- its s is final and the repair only re-points v; for a tile
    // minimum its tile triplet.  Only tile minima (s != u, or the tile root) get a 16-byte
    // working cell: the global merge only ever reads or writes cells of tile minima (the
    // crossing edges start at tile representatives, which are minima, and every cell on a v
    // chain from a minimum is a minimum's; DESIGN.md derivation C'''), so regular vertices need
    // none (the x-face records carry (order key, R) for the tile's x faces, coalesced).
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
#if TILE_REP_ILP
        const uint32_t s = c_s(cu), v = rep[k];
#else
        const uint32_t s = c_s(cu), v = c_v(cu);
#endif
        const uint64_t g = gbase + uint64_t(lz) * sxy + uint64_t(ly) * nx + lx;
        const uint32_t gu = uint32_t(g), gv = gid(v);
        const bool minimum = s != u || v == u;
        const uint32_t gs = s == u ? gu : gid(s);
        T0[g] = pack(gs, gv);
        if (minimum) C[g] = make_cell(key_of(uint32_t(cu >> 32), gs), ou, gv);
        // the tile's x faces (lanes 0 and 31) again, compactly: (order key, R) per row, R =
        // Rep_tile(u, key(u)) for a regular vertex, u for a minimum, so that the crossing edges of
        // the x faces read them coalesced (in the grid they are 128 B apart)
        if (lx == 0 || lx == TX - 1)
            xface[(uint64_t(b) * 2 + (lx == TX - 1)) * ROWS + r] = (uint64_t(ou) << 32) | (s == u ? gv : gu);
    }
    phase_time(ST_CYC_WRITE);
    if (STATS) {
        atomicAdd(stats + ST_TILE_EDGES, n_edges);
        atomicAdd(stats + ST_TILE_HOPS, n_hops);
        atomicAdd(stats + ST_TILE_ITERS, n_iters);
        atomicAdd(stats + ST_TILE_REPAIR, n_rep);
        atomicAdd(stats + ST_TILE_COMPRESS, n_cmp);
        atomicAdd(stats + ST_TILE_PAIRS, n_pairs);
    }
}

}  // namespace

uint64_t xface_entries(const Slab& sl) {
    uint32_t ty, tz;
    tile_shape(sl.nz, &ty, &tz);
    const uint64_t nzl = sl.z_end - sl.z_begin;
    const uint64_t tiles = uint64_t((sl.nx + TX - 1) / TX) * ((sl.ny + ty - 1) / ty) * ((nzl + tz - 1) / tz);
    return tiles * 2 * ty * tz;
}

#ifndef MT_TILE_NV
#define MT_TILE_NV 4096   // vertices per tile (build knob: 4096 or 2048); tile_shape follows it
#endif
constexpr int tile_vertices() { return MT_TILE_NV; }

void tile_shape(uint32_t nz_global, uint32_t* ty, uint32_t* tz) {
    const int nv = tile_vertices();
    if (nz_global == 1) {
        *ty = uint32_t(nv / TX);
        *tz = 1;
    } else {
        *ty = nv == 4096 ? 16 : 8;
        *tz = 8;
    }
}

template <int TY, int TZ>
void launch_tile(const float* f, Cell* C, uint64_t* T0, uint64_t* xface, const Slab& sl, uint32_t tx, uint32_t tyn, uint32_t grid,
                 uint32_t flip, unsigned long long* counters, unsigned long long* stats, cudaStream_t stream) {
    constexpr int NV = TX * TY * TZ;
    ensure_smem_attr(reinterpret_cast<const void*>(tile_tmt_kernel<TY, TZ, false>), int(smem_bytes<NV>()));
    ensure_smem_attr(reinterpret_cast<const void*>(tile_tmt_kernel<TY, TZ, true>), int(smem_bytes<NV>()));
    if (stats)
        tile_tmt_kernel<TY, TZ, true><<<grid, NV / 8, smem_bytes<NV>(), stream>>>(f, C, T0, xface, sl.nx, sl.ny,
                                                                                 sl.z_begin, sl.z_end, tx, tyn,
                                                                                 flip, counters, stats);
    else
        tile_tmt_kernel<TY, TZ, false><<<grid, NV / 8, smem_bytes<NV>(), stream>>>(f, C, T0, xface, sl.nx, sl.ny, sl.z_begin, sl.z_end, tx,
                                                                       tyn, flip, counters, stats);
}

void launch_tile_tmt(const float* f, Cell* C, uint64_t* T0, uint64_t* xface, const Slab& sl, uint32_t flip,
                     unsigned long long* counters, unsigned long long* stats, cudaStream_t stream) {
    uint32_t ty, tz;
    tile_shape(sl.nz, &ty, &tz);
    const uint32_t nzl = sl.z_end - sl.z_begin;
    const uint32_t tx = (sl.nx + TX - 1) / TX, tyn = (sl.ny + ty - 1) / ty, tzn = (nzl + tz - 1) / tz;
    const uint32_t grid = tx * tyn * tzn;
    if (grid == 0) return;
    const bool big = tile_vertices() == 4096;
    if (sl.nz == 1 && big)
        launch_tile<128, 1>(f, C, T0, xface, sl, tx, tyn, grid, flip, counters, stats, stream);
    else if (sl.nz == 1)
        launch_tile<64, 1>(f, C, T0, xface, sl, tx, tyn, grid, flip, counters, stats, stream);
    else if (big)
        launch_tile<16, 8>(f, C, T0, xface, sl, tx, tyn, grid, flip, counters, stats, stream);
    else
        launch_tile<8, 8>(f, C, T0, xface, sl, tx, tyn, grid, flip, counters, stats, stream);
}

}  // namespace mt
