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
//   c. one edge per pair of adjacent basins, the lowest (derivation C''): every in-tile edge
//      (u, w) between two basins is a candidate; a shared-memory hash table keyed by the basin
//      pair keeps the one of lowest level (64-bit CAS).  Candidates go through a per-warp ring
//      of staged entries and every lane runs its insert as a state machine, one probe per loop
//      iteration, taking the next staged entry as soon as its insert is done (TILE_RINS), so a
//      warp pays the lanes' average probe count rather than their maximum.  (TILE_KRUSKAL=1: a
//      bucketed Kruskal filter instead, derivation K -- measured slower.)
//   d. merge the kept edges (one per basin pair): Alg. 3 from the two basins at the edge's level
//      with 64-bit shared-memory CAS and the root guards R4/R5,
//      one lane per edge, one shared-memory round trip per loop iteration; a
//      lane whose edge is done takes the next one of the warp's slice;
//   e. repair (Alg. 5 with Alg. 4's walk, reading R20): the tile store is
//      minimal for G_t (each thread walks its vertices one after the other);
//   f. write the tile store T0 (8 B per vertex) and the tile minima's 16-byte
//      working cells (common.cuh) with global ids, and the x-face records.
// No halo is needed: only in-tile edges are used here.
//
// Layout: f float32[n] x fastest (reading R10) read once (coalesced 128-B
// rows).  One CTA of 512 threads per tile.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

#ifndef TILE_KRUSKAL
#define TILE_KRUSKAL 0 // phase c: bucketed Kruskal filter (1) or the basin-pair hash table (0)
#endif
#ifndef TILE_NB
#define TILE_NB 16     // level buckets of the Kruskal filter (4, 8, 16 or 32)
#endif
#ifndef TILE_KCAP
#define TILE_KCAP 2048 // kept edges a tile can hold (more: the overflow path merges every edge)
#endif
#ifndef TILE_MINB
#define TILE_MINB 2    // __launch_bounds__ min blocks per SM (register budget knob)
#endif
#ifndef TILE_REP_SEQ
#define TILE_REP_SEQ 1 // in-tile repair: walks one after the other (else lock-step rounds)
#endif
#ifndef TILE_ORDBITS
#define TILE_ORDBITS 0 // hash insert: compare levels by the order-key bits the entries carry first
#endif
#ifndef TILE_MPASS
#define TILE_MPASS 1   // hash variant: merge the pairs in this many level passes (1: one pass)
#endif
#ifndef TILE_BOTHCLIMB
#define TILE_BOTHCLIMB 1  // Alg. 3 loop: climb u and v in the same iteration when both can climb
#endif
#ifndef TILE_TQ
#define TILE_TQ 6      // basin-pair table: TILE_TQ / 4 slots per tile vertex
#endif
#ifndef TILE_FULLSECTOR
#define TILE_FULLSECTOR 0  // tile minima cells written as whole 32-B sectors (a copy in the partner slot)
#endif
#ifndef TILE_CLIMB2
#define TILE_CLIMB2 0  // merge loop: two climb steps per iteration
#endif
#ifndef TILE_RCHAIN
#define TILE_RCHAIN 1  // in-tile repair: a walk continues the thread's previous one (same start, higher threshold)
#endif
#ifndef TILE_ZREG
#define TILE_ZREG 1    // volumes: the +-z neighbours' order keys / basins from the thread's own registers
#endif
#ifndef TILE_RINS
#define TILE_RINS 1    // hash list: refilling insert loop over a per-warp ring (lanes' average probes)
#endif
#ifndef TILE_ZRUN
#define TILE_ZRUN 0    // hash list: a thread's z column keeps one edge per run of equal basin pairs
#endif
#ifndef TILE_VPT
#define TILE_VPT 8     // vertices per thread (8: 512 threads per tile, 4: 1024)
#endif
#ifndef TILE_STOP
#define TILE_STOP 0    // timing only (WRONG results): run phases < k: 1 load+descent, 2 +compress, 3 +list, 4 +merge
#endif

constexpr int TX = 32;
constexpr uint32_t ABSENT = 0xffffffffu;       // order key of a tile slot outside the grid
constexpr uint64_t EMPTY = ~0ull;
constexpr int LOG2NB = TILE_NB == 32 ? 5 : TILE_NB == 16 ? 4 : TILE_NB == 8 ? 3 : 2;
static_assert((1 << LOG2NB) == TILE_NB, "TILE_NB: 4, 8, 16 or 32");
// hash variant: basin-pair table of TILE_TQ / 4 NV slots + a staging buffer of 128 entries per warp
constexpr int table_slots(int nv) { return TILE_TQ * nv / 4; }
template <int NV>
constexpr size_t smem_bytes() {
    return TILE_KRUSKAL ? size_t(NV) * 8 + size_t(NV) * 4 + size_t(NV) * 2 /* uf */ + size_t(NV) * 2 /* vlist */ +
                              size_t(TILE_KCAP) * 4
                        : size_t(NV) * 8 + size_t(NV) * 4 + size_t(table_slots(NV)) * 8 + size_t(NV) * 4;
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
__device__ __forceinline__ uint64_t scas64(uint64_t* p, uint64_t cmp, uint64_t val) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(p), cmp, val);
}

#if TILE_KRUSKAL
__device__ __forceinline__ uint32_t sld16(const uint16_t* p) { return *reinterpret_cast<const volatile uint16_t*>(p); }

// union-find over basin minima (local ids, 16-bit parents): find with path halving -- the
// halving stores only ever shortcut to an ancestor in the same tree, so they are safe next to
// concurrent finds and unions
__device__ __forceinline__ uint32_t uf_find(uint16_t* uf, uint32_t x) {
    while (true) {
        const uint32_t p = sld16(uf + x);
        if (p == x) return x;
        const uint32_t g = sld16(uf + p);
        if (g == p) return p;
        *reinterpret_cast<volatile uint16_t*>(uf + x) = uint16_t(g);
        x = g;
    }
}
// link the younger root under the older (a fixed order: no cycles); retried on a lost race
__device__ __forceinline__ void uf_union(uint16_t* uf, const uint32_t* ord, uint32_t a, uint32_t b) {
    while (true) {
        a = uf_find(uf, a);
        b = uf_find(uf, b);
        if (a == b) return;
        if (lkey_lt(ord, a, b)) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(reinterpret_cast<unsigned short*>(uf + a), (unsigned short)a, (unsigned short)b) ==
            (unsigned short)a)
            return;
    }
}
#endif

// ---- TMA (cp.async.bulk.tensor) staging of a tile's f into shared memory -----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MT_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MT_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// one tile box {32, TY, TZ} of f at (x, y, z) (slab-local coordinates) into dst; out-of-grid
// elements arrive as zeros (the kernel masks them by coordinates)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of a tile box (no shared memory, no barrier): the tile a later CTA will load
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(x), "r"(y),
                 "r"(z)
                 : "memory");
}

// Output pointers of one tree.  DUAL launches compute two trees from one read of f: the merge
// (join) tree into the first set and the split tree (complemented order keys, reading R16) into
// the second.
struct TileOut {
    Cell* C;
    uint64_t* T0;
    uint64_t* xface;
    unsigned long long* counters;
};

template <int TY, int TZ, bool STATS, bool DUAL, bool TMA, bool PERSIST, int NV = TX * TY * TZ,
          int THREADS = NV / TILE_VPT, int TABLE = table_slots(NV)>
__global__ void __launch_bounds__(THREADS, TILE_MINB)
tile_tmt_kernel(const __grid_constant__ CUtensorMap fmap, const float* __restrict__ f, TileOut out0, TileOut out1,
                uint32_t ntiles, uint32_t nx,
                uint32_t ny, uint32_t z_begin,
                uint32_t z_end, uint32_t tiles_x, uint32_t tiles_y, uint32_t flip,
                unsigned long long* __restrict__ stats, uint32_t pf_dist) {
    constexpr int ROWS = TY * TZ;               // 128 rows of 32
    static_assert(TX * ROWS == NV, "tile size");
    constexpr int RSTEP = THREADS / TX;         // 16 rows per pass
    constexpr int PER = ROWS / RSTEP;           // 8 vertices per thread
    constexpr int NW = THREADS / 32;
    constexpr int LB = NV > 4096 ? 13 : 12;          // bits of a local vertex id
    constexpr uint32_t LMASK = (1u << LB) - 1u, PMASK = (1u << (2 * LB)) - 1u;
    static_assert(NV <= 8192, "local ids: 13 bits (and 16-bit cell fields)");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* cell = reinterpret_cast<uint64_t*>(smem);
    uint32_t* ord = reinterpret_cast<uint32_t*>(smem + NV * 8);
    __shared__ int s_overflow;
    __shared__ uint32_t s_omin, s_omax, s_nkept;
#if TILE_KRUSKAL
    uint16_t* uf = reinterpret_cast<uint16_t*>(smem + NV * 12);
    uint16_t* vlist = reinterpret_cast<uint16_t*>(smem + NV * 14);
    uint32_t* kept = reinterpret_cast<uint32_t*>(smem + NV * 16);
    __shared__ uint32_t s_hist[TILE_NB][NW];    // per bucket and warp: count, then offset
    __shared__ uint32_t s_boff[TILE_NB + 1];
#else
    uint64_t* table = reinterpret_cast<uint64_t*>(smem + NV * 12);
#endif

    unsigned long long n_edges = 0, n_pairs = 0, n_iters = 0, n_rep = 0, n_cmp = 0;
    long long t_mark = clock64();
    // per-phase SM cycles (stats mode): thread 0 accumulates the time between barriers
    auto phase_time = [&](int slot) {
        if (STATS && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(stats + slot, (unsigned long long)(t - t_mark));
            t_mark = t;
        }
    };

    const uint64_t sxy = uint64_t(nx) * ny;
    const int lx = threadIdx.x & (TX - 1);
    const int r0 = threadIdx.x / TX;
    const int lane_c = threadIdx.x & 31;
    const int warp_d = threadIdx.x >> 5;
    __shared__ alignas(8) uint64_t s_fbar;
    // PERSIST (TMA, hash variant): one CTA per resident slot walks the tiles b = blockIdx.x +
    // i * gridDim.x; tile i+1's f is bulk-copied into the list phase's staging buffer (idle
    // from the end of tile i's list phase on) while tile i merges, repairs and writes
    [[maybe_unused]] float* const fpre =
        reinterpret_cast<float*>(smem + NV * 12 + TABLE * 8);   // NV floats = the staging buffer
    auto tile_origin = [&](uint32_t t, uint32_t* ox, uint32_t* oy, uint32_t* oz) {
        *ox = (t % tiles_x) * TX;
        *oy = ((t / tiles_x) % tiles_y) * TY;
        *oz = z_begin + (t / (tiles_x * tiles_y)) * TZ;
    };
    if (PERSIST) {
        if (threadIdx.x == 0 && blockIdx.x < ntiles) {
            uint32_t px, py, pz;
            tile_origin(blockIdx.x, &px, &py, &pz);
            mbar_init(&s_fbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(&s_fbar, uint32_t(NV) * 4u);
            tma_load_3d(fpre, &fmap, int(px), int(py), int(pz - z_begin), &s_fbar);
        }
        __syncthreads();
    }
    uint32_t it = 0;
    __shared__ uint32_t s_next;       // PERSIST: the CTA's next tile (dynamic tickets)
    if (PERSIST && threadIdx.x == 0) s_next = ntiles;
#pragma unroll 1
    for (uint32_t b = blockIdx.x; b < (PERSIST ? ntiles : blockIdx.x + 1); ++it) {
    uint32_t x0 = 0, y0 = 0, z0 = 0;
    // (TMA tiles: thread 0 alone divides -- it issues the copy -- and the others read the origin
    // after the barrier that publishes the mbarrier's init)
    __shared__ uint32_t s_org[3];
    if (!(TMA && !PERSIST) || threadIdx.x == 0) tile_origin(b, &x0, &y0, &z0);
    if (TMA && !PERSIST && threadIdx.x == 0) {
        s_org[0] = x0;
        s_org[1] = y0;
        s_org[2] = z0;
    }
    // f and C are indexed by GLOBAL vertex id (the caller passes pointers shifted by the
    // slab's first id); this tile starts at global plane z0

    // ---- K1: load f once, order keys into shared memory ------------------------------
    bool bad = false;
    if (TMA && !PERSIST) {
        // the whole tile box in one bulk tensor copy issued by one thread (the f staging is the
        // ord array itself: 4 B per vertex, converted in place below); the table init overlaps it
        if (threadIdx.x == 0) {
            mbar_init(&s_fbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(&s_fbar, uint32_t(NV) * 4u);
            tma_load_3d(ord, &fmap, int(x0), int(y0), int(z0 - z_begin), &s_fbar);
            // the tile the CTA pf_dist launches later will load (about one wave of resident CTAs
            // later): into L2 now, so its load meets L2 latency instead of HBM's
            if (pf_dist && b + pf_dist < ntiles) {
                uint32_t px, py, pz;
                tile_origin(b + pf_dist, &px, &py, &pz);
                tma_prefetch_3d(&fmap, int(px), int(py), int(pz - z_begin));
            }
        }
    } else {
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
    }
#if TILE_KRUSKAL
    for (int i = threadIdx.x; i < NV; i += THREADS) uf[i] = uint16_t(i);
    if (threadIdx.x < TILE_NB * NW) (&s_hist[0][0])[threadIdx.x] = 0;
#else
    for (int i = threadIdx.x; i < TABLE; i += THREADS) table[i] = EMPTY;
#endif
    if (threadIdx.x == 0) {
        s_overflow = 0;
        s_omin = ~0u;
        s_omax = 0;
        s_nkept = 0;
    }
    if (TMA) {
        if (!PERSIST) {
            __syncthreads();             // (the barrier's init is visible to every waiting thread)
            x0 = s_org[0];
            y0 = s_org[1];
            z0 = s_org[2];
        }
        mbar_wait(&s_fbar, PERSIST ? (it & 1u) : 0u);
        const float* fv = PERSIST ? fpre : reinterpret_cast<const float*>(ord);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int r = r0 + k * RSTEP;
            const int ly = r % TY, lz = r / TY;
            const uint32_t i = r * TX + lx;
            uint32_t o = ABSENT;
            if (x0 + lx < nx && y0 + ly < ny && z0 + lz < z_end) {
                const float val = fv[i];
                bad |= nonfinite(val);
                o = ord32(val) ^ flip;
            }
            ord[i] = o;                  // in place: every element is owned by one thread
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) {
        atomicOr(out0.counters + CTR_ERR, ERR_NONFINITE);
        if (DUAL) atomicOr(out1.counters + CTR_ERR, ERR_NONFINITE);
    }
    phase_time(ST_CYC_LOAD);

#pragma unroll 1
    for (int pass = 0; pass < (DUAL ? 2 : 1); ++pass) {
    Cell* const C = pass ? out1.C : out0.C;
    uint64_t* const T0 = pass ? out1.T0 : out0.T0;
    uint64_t* const xface = pass ? out1.xface : out0.xface;
    if (DUAL && pass) {
        // the split tree of the same values: complemented order keys (reading R16), state reset
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t i = (r0 + k * RSTEP) * TX + lx;
            if (ord[i] != ABSENT) ord[i] = ~ord[i];
        }
#if TILE_KRUSKAL
        for (int i = threadIdx.x; i < NV; i += THREADS) uf[i] = uint16_t(i);
        if (threadIdx.x < TILE_NB * NW) (&s_hist[0][0])[threadIdx.x] = 0;
#else
        for (int i = threadIdx.x; i < TABLE; i += THREADS) table[i] = EMPTY;
#endif
        if (threadIdx.x == 0) {
            s_overflow = 0;
            s_omin = ~0u;
            s_omax = 0;
            s_nkept = 0;
        }
        __syncthreads();
    }

    // ---- a. steepest descent over in-tile neighbours -----------------------------------
    // the key-least of u and its neighbours: visiting them in ascending id order (-z, -y, -x,
    // u, +x, +y, +z: local ids are lexicographic in (z, y, x) like global ids) and taking a
    // strictly smaller order key breaks ties by id (reading R1) with 32-bit compares only
    {
        // (ZREG, volumes: the +-z neighbours of vertex k are the thread's own vertices k -+ 1)
        constexpr bool ZREG = TILE_ZREG && TY == RSTEP;
        uint32_t oreg[PER];
        if (ZREG) {
#pragma unroll
            for (int k = 0; k < PER; ++k) oreg[k] = ord[(r0 + k * RSTEP) * TX + lx];
        }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int r = r0 + k * RSTEP;
        const int ly = r % TY, lz = r / TY;
        const uint32_t u = r * TX + lx;
        const uint32_t ou = ZREG ? oreg[k] : ord[u];
        uint32_t best = u;
        if (ou != ABSENT) {
            uint32_t bo = ABSENT;
            auto visit = [&](bool ok, uint32_t w) {
                if (!ok) return;
                const uint32_t ow = ord[w];
                if (ow < bo) {
                    bo = ow;
                    best = w;
                }
            };
            auto visit_kn = [&](bool ok, uint32_t w, uint32_t ow) {
                if (ok && ow < bo) {
                    bo = ow;
                    best = w;
                }
            };
            if (ZREG) visit_kn(k > 0, u - TX * TY, oreg[k > 0 ? k - 1 : 0]);
            else visit(lz > 0, u - TX * TY);
            visit(ly > 0, u - TX);
            visit(lx > 0, u - 1);
            if (ZREG) visit_kn(true, u, ou);
            else visit(true, u);
            visit(lx + 1 < TX, u + 1);
            visit(ly + 1 < TY, u + TX);
            if (ZREG) visit_kn(k + 1 < PER, u + TX * TY, oreg[k + 1 < PER ? k + 1 : k]);
            else visit(lz + 1 < TZ, u + TX * TY);
        }
        cell[u] = c_make(ou, u, best);
    }
    }
    __syncthreads();
    phase_time(ST_CYC_DESCENT);

    // ---- b. compress: every regular cell points at its basin minimum ----------------------
    // synchronous pointer jumping, par <- par(par), on the thread's own 8 vertices (8
    // independent load chains per round), until every pointer is a root: ceil(log2 depth) + 1
    // rounds.  Rounds run in place: a pointer read while its owner rewrites it is the old or
    // the new ancestor, both in the same descent tree (derivation F), so the v fields (16-bit
    // stores) only ever move up the tree.
    {
        uint32_t par[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) par[k] = c_v(cell[(r0 + k * RSTEP) * TX + lx]);
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
    }
    __syncthreads();
    phase_time(ST_CYC_COMPRESS);

    // basin of x after the compress: a regular cell (s = x) is static and points at the minimum
    auto basin = [&](uint32_t x) {
        const uint64_t c = sld64(cell + x);
        return c_s(c) == x ? c_v(c) : x;
    };

#if TILE_KRUSKAL
    // ---- c. bucketed Kruskal filter over the basin graph --------------------------------
    // Level buckets at sample quantiles: warp 0 sorts 32 order keys spread over the tile
    // (bitonic, in registers) and keeps NB - 1 of them as splitters; a vertex's bucket is the
    // number of splitters <= its key, so the buckets hold roughly equal numbers of vertices
    // whatever the value distribution (a skewed field would put most of a tile into one bucket
    // of a range split).
    __shared__ uint32_t s_split[TILE_NB];
    if (warp_d == 0) {
        uint32_t o = ord[(uint32_t(lane_c) * (NV / 32) + NV / 64) % NV];   // ABSENT sorts last
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const uint32_t p = __shfl_xor_sync(FULL_MASK, o, j);
                const bool up = ((lane_c & k) == 0), lower = (lane_c & j) == 0;
                o = (lower == up) ? min(o, p) : max(o, p);
            }
        }
        // lane i holds the i-th smallest sample; splitter j = sample (j + 1) * 32 / NB
        if (lane_c % (32 / TILE_NB) == (32 / TILE_NB) - 1 && lane_c / (32 / TILE_NB) < TILE_NB - 1)
            s_split[lane_c / (32 / TILE_NB)] = o;
    }
    __syncthreads();
    auto bucket_of = [&](uint32_t o) {
        int lo = 0, hi = TILE_NB - 1;           // number of splitters <= o, by binary search
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_split[mid] <= o) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    // counting sort of the vertices by bucket: per-warp counts, bucket-major prefix, scatter
    {
        uint32_t rank[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t o = ord[(r0 + k * RSTEP) * TX + lx];
            rank[k] = o != ABSENT ? atomicAdd(&s_hist[bucket_of(o)][warp_d], 1u) : 0u;
        }
        __syncthreads();
        if (warp_d == 0) {                     // exclusive prefix over (bucket, warp), bucket-major
            constexpr int E = TILE_NB * NW / 32;   // entries per lane
            static_assert(E * 32 == TILE_NB * NW, "prefix layout");
            uint32_t* h = &s_hist[0][0];
            uint32_t c[E], tot = 0;
#pragma unroll
            for (int j = 0; j < E; ++j) {
                c[j] = h[lane_c * E + j];
                tot += c[j];
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
                if (lane_c >= o) incl += t;
            }
            uint32_t off = incl - tot;
#pragma unroll
            for (int j = 0; j < E; ++j) {
                h[lane_c * E + j] = off;
                if ((lane_c * E + j) % NW == 0) s_boff[(lane_c * E + j) / NW] = off;
                off += c[j];
            }
            if (lane_c == 31) s_boff[TILE_NB] = off;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t u = (r0 + k * RSTEP) * TX + lx;
            const uint32_t o = ord[u];
            if (o != ABSENT) vlist[s_hist[bucket_of(o)][warp_d] + rank[k]] = uint16_t(u);
        }
    }
    __syncthreads();
    // bucket by bucket: A. keep the down-edges of the bucket's vertices whose basins the
    // union-find (kept edges of the lower buckets) does not join yet; B. unite them
#pragma unroll 1
    for (int bk = 0; bk < TILE_NB && (TILE_STOP == 0 || TILE_STOP > 2); ++bk) {
        const uint32_t vb = s_boff[bk], ve = s_boff[bk + 1];
        if (vb == ve) continue;                               // (uniform)
        const uint32_t kb = s_nkept;
        for (uint32_t i = vb + threadIdx.x; i < ve; i += THREADS) {
            const uint32_t u = vlist[i];
            const uint32_t ou = ord[u];
            const uint32_t bu = basin(u);
            const uint32_t ux = u % TX, uy = (u / TX) % TY, uz = u / (TX * TY);
            uint32_t ru = 0xffffu;
            auto down = [&](bool ok, uint32_t w, bool lower_id) {
                if (!ok) return;
                const uint32_t ow = ord[w];
                if (ow == ABSENT || !(ow < ou || (ow == ou && lower_id))) return;   // not below u
                const uint32_t bw = basin(w);
                if (bw == bu) return;
                if (STATS) ++n_edges;
                if (ru == 0xffffu) ru = uf_find(uf, bu);
                if (uf_find(uf, bw) == ru) return;            // joined below this bucket: redundant
                const uint32_t j = atomicAdd(&s_nkept, 1u);
                if (j < TILE_KCAP) kept[j] = (u << 16) | w;
                else s_overflow = 1;
            };
            down(uz > 0, u - TX * TY, true);
            down(uy > 0, u - TX, true);
            down(ux > 0, u - 1, true);
            down(ux + 1 < TX, u + 1, false);
            down(uy + 1 < TY, u + TX, false);
            down(uz + 1 < TZ, u + TX * TY, false);
        }
        __syncthreads();
        const uint32_t ke = min(s_nkept, uint32_t(TILE_KCAP));
        for (uint32_t j = kb + threadIdx.x; j < ke; j += THREADS) {
            const uint32_t e = kept[j];
            uf_union(uf, ord, basin(e >> 16), basin(e & 0xffffu));
        }
        __syncthreads();
    }
    phase_time(ST_CYC_LIST);
    const uint32_t n_kept = min(s_nkept, uint32_t(TILE_KCAP));
    // this warp's slice of the kept edges
    const uint32_t run_b = uint32_t(uint64_t(n_kept) * warp_d / NW);
    const uint32_t run_len = uint32_t(uint64_t(n_kept) * (warp_d + 1) / NW) - run_b;
    auto run_edge = [&](uint32_t j, uint32_t* mu, uint32_t* mv, uint64_t* S) {
        const uint32_t e = kept[run_b + j];
        const uint32_t hi = e >> 16;
        *mu = basin(hi);
        *mv = basin(e & 0xffffu);
        *S = key48(ord, hi);
    };
#else
    // ---- c. one edge per pair of adjacent basins: the lowest --------------------------------
    // Between two basins A and B only the lowest edge matters: any other A-B edge at level
    // L' joins vertices that are already connected at L' through their descent paths and
    // that lowest edge (DESIGN.md derivation C'').  A shared-memory hash table keyed by the
    // basin pair keeps, per pair, the edge's upper endpoint of lowest key.
    // entry = orientation << 63 | top OB bits of ord(hi) << 3 LB | pair << LB | hi: the level is
    // compared from the entries themselves, with a lookup of ord only on a tie of those bits
    constexpr int OB = 63 - 3 * LB;
    constexpr uint64_t OBMASK = (1ull << OB) - 1;
    auto insert_entry = [&](uint64_t entry) {
        const uint32_t pair = uint32_t(entry >> LB) & PMASK;
        const uint64_t mo = TILE_ORDBITS ? (entry >> (3 * LB)) & OBMASK : 0;
        const uint32_t hme = uint32_t(entry) & LMASK, ome = ord[hme];
        uint32_t h = pair_hash<TABLE>(pair);
        for (uint32_t probe = 0;;) {
            const uint64_t cur = sld64(table + h);
            if (cur == EMPTY) {
                if (scas64(table + h, EMPTY, entry) == EMPTY) break;
                continue;                                        // lost the slot: re-read it
            }
            if ((uint32_t(cur >> LB) & PMASK) != pair) {
                h = h + 1 == uint32_t(TABLE) ? 0u : h + 1;
                if (++probe < uint32_t(TABLE)) continue;
                s_overflow = 1;                                  // table full: merge every edge
                break;
            }
            const uint64_t co = TILE_ORDBITS ? (cur >> (3 * LB)) & OBMASK : 0;
            if (mo > co) break;                                  // the stored edge is lower
            if (mo == co) {                                      // the stored edge is lower or equal
                const uint32_t hcu = uint32_t(cur) & LMASK, ocu = ord[hcu];
                if (ome > ocu || (ome == ocu && hme >= hcu)) break;
            }
            if (scas64(table + h, cur, entry) == cur) break;
        }
    };
    // (candidate_kn: the neighbour's order key and basin already in registers)
    auto candidate_kn = [&](uint32_t u, uint32_t ou, uint32_t bu, bool ok, uint32_t w, uint32_t ow, uint32_t bw,
                            uint64_t* entry) {
        if (ou == ABSENT || !ok || ow == ABSENT || bw == bu) return false;
        const bool u_hi = ow < ou;   // w has the larger id: on a tie w is the upper end
        const uint32_t hi = u_hi ? u : w, oh = u_hi ? ou : ow;
        const bool lo_first = bu < bw;
        const uint32_t pair = lo_first ? (bu << LB) | bw : (bw << LB) | bu;
        *entry = (uint64_t(u_hi == lo_first) << 63) | (TILE_ORDBITS ? uint64_t(oh >> (32 - OB)) << (3 * LB) : 0ull) |
                 (uint64_t(pair) << LB) | hi;
        return true;
    };
    auto candidate = [&](uint32_t u, uint32_t ou, uint32_t bu, bool ok, uint32_t off, uint64_t* entry) {
        if (ou == ABSENT || !ok) return false;
        const uint32_t w = u + off;
        const uint32_t ow = ord[w];
        if (ow == ABSENT) return false;
        const uint32_t bw = c_v(cell[w]);
        if (bw == bu) return false;
        const bool u_hi = ow < ou;   // w = u + off has the larger id: on a tie w is the upper end
        const uint32_t hi = u_hi ? u : w, oh = u_hi ? ou : ow;
        const bool lo_first = bu < bw;
        const uint32_t pair = lo_first ? (bu << LB) | bw : (bw << LB) | bu;
        // bit 63: the upper endpoint lies in the pair's first (smaller) basin
        *entry = (uint64_t(u_hi == lo_first) << 63) | (TILE_ORDBITS ? uint64_t(oh >> (32 - OB)) << (3 * LB) : 0ull) |
                 (uint64_t(pair) << LB) | hi;
        return true;
    };
#if TILE_RINS
    if (TILE_STOP == 0 || TILE_STOP > 2) {
        // The warp's candidates go through a ring of 128 staged entries; every lane runs one
        // insert as a state machine, one table probe per loop iteration, and a lane whose insert
        // is done takes the next staged entry at the top of the next iteration (as in the merge
        // loop below), so the warp's iterations are the lanes' average probe count instead of
        // their maximum.  After each vertex row at most 32 entries stay pending (+ <= 96 new).
        constexpr uint32_t RING = 128;
        static_assert(NV / (2 * NW) == int(RING), "staging ring: 128 entries per warp");
        uint64_t* stage = reinterpret_cast<uint64_t*>(smem + NV * 12 + TABLE * 8) + warp_d * RING;
        const uint32_t lt = (1u << lane_c) - 1u;
        uint32_t head = 0, tail = 0;          // warp-uniform ring positions
        bool ibusy = false;
        uint64_t ient = 0;
        uint32_t ih = 0, ipair = 0, iprobe = 0;
        // run the warp's inserts until at most `keep` entries are pending (keep == 0: all done)
        auto pump = [&](uint32_t keep) {
#pragma unroll 1
            while (true) {
                const uint32_t pend = tail - head;
                const uint32_t need = __ballot_sync(FULL_MASK, !ibusy);
                if (pend <= keep && (keep || need == FULL_MASK)) break;
                if (need && pend) {
                    if (!ibusy) {
                        const uint32_t r = __popc(need & lt);
                        if (r < pend) {
                            ient = stage[(head + r) & (RING - 1)];
                            ipair = uint32_t(ient >> LB) & PMASK;
                            ih = pair_hash<TABLE>(ipair);
                            iprobe = 0;
                            ibusy = true;
                        }
                    }
                    head += min(__popc(need), pend);
                }
                if (ibusy) {                 // one probe of the insert (insert_entry's loop body)
                    const uint64_t cur = sld64(table + ih);
                    if (cur == EMPTY) {
                        if (scas64(table + ih, EMPTY, ient) == EMPTY) ibusy = false;
                    } else if ((uint32_t(cur >> LB) & PMASK) != ipair) {
                        ih = ih + 1 == uint32_t(TABLE) ? 0u : ih + 1;
                        if (++iprobe >= uint32_t(TABLE)) {
                            s_overflow = 1;          // table full: merge every edge
                            ibusy = false;
                        }
                    } else {
                        const uint32_t hme = uint32_t(ient) & LMASK, hcu = uint32_t(cur) & LMASK;
                        const uint32_t ome = ord[hme], ocu = ord[hcu];
                        if (ome > ocu || (ome == ocu && hme >= hcu)) ibusy = false;   // stored edge is lower
                        else if (scas64(table + ih, cur, ient) == cur) ibusy = false;
                    }
                }
            }
        };
        // (ZREG, volumes: the +z neighbour of vertex k is the thread's own vertex k + 1, so its order
        // key and basin are loaded once and carried to the next iteration)
        constexpr bool ZREG = TILE_ZREG && TY == RSTEP;
        uint32_t ou_n = 0, bu_n = 0;
        if (ZREG) {
            ou_n = ord[r0 * TX + lx];
            bu_n = c_v(cell[r0 * TX + lx]);
        }
#pragma unroll 1
        for (int k = 0; k < PER; ++k) {
            const int r = r0 + k * RSTEP;
            const int ly = r % TY, lz = r / TY;
            const uint32_t u = r * TX + lx;
            uint32_t ou, bu;
            if (ZREG) {
                ou = ou_n;
                bu = bu_n;
                if (k + 1 < PER) {
                    ou_n = ord[u + TX * TY];
                    bu_n = c_v(cell[u + TX * TY]);
                }
            } else {
                ou = ord[u];
                bu = c_v(cell[u]);                 // basin (a minimum points at itself)
            }
            const bool ok[3] = {lx + 1 < TX, ly + 1 < TY, lz + 1 < TZ};
            const uint32_t off[3] = {1u, uint32_t(TX), uint32_t(TX * TY)};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                uint64_t entry = 0;
                const bool valid = (ZREG && d == 2) ? candidate_kn(u, ou, bu, ok[d], u + TX * TY, ou_n, bu_n, &entry)
                                                    : candidate(u, ou, bu, ok[d], off[d], &entry);
                if (STATS && valid) ++n_edges;
                const uint32_t m = __ballot_sync(FULL_MASK, valid);
                if (valid) stage[(tail + __popc(m & lt)) & (RING - 1)] = entry;
                tail += __popc(m);
            }
            __syncwarp();
            pump(32);
        }
        __syncwarp();
        pump(0);
    }
#else
    if (TILE_STOP == 0 || TILE_STOP > 2) {
        constexpr int STAGE = NV / (2 * NW);   // per-warp staging entries (>= 64: flushed per direction)
        static_assert(STAGE >= 64, "staging buffer");
        uint64_t* stage = reinterpret_cast<uint64_t*>(smem + NV * 12 + TABLE * 8) + warp_d * STAGE;
        const uint32_t lt = (1u << lane_c) - 1u;
        uint32_t nst = 0;
        // append the lanes' valid entries to the warp's staging buffer; insert 32 at a time
        auto stage_entry = [&](bool valid, uint64_t entry, bool flush_now) {
            const uint32_t m = __ballot_sync(FULL_MASK, valid);
            if (valid) stage[nst + __popc(m & lt)] = entry;
            nst += __popc(m);
            if (flush_now) {
                __syncwarp();
                while (nst >= 32) {
                    const uint64_t e = stage[nst - 32 + lane_c];
                    __syncwarp();
                    nst -= 32;
                    insert_entry(e);
                }
            }
        };
#if TILE_ZRUN
        // a thread's 8 vertices are one z column: its consecutive +x (+y, +z) edges often cross
        // the same basin boundary, so a run of edges of one basin pair keeps only its lowest edge
        // in registers (derivation C'') and stages that one when the pair changes
        uint64_t run_e[3] = {0, 0, 0};
        uint32_t run_p[3] = {~0u, ~0u, ~0u}, run_o[3] = {0, 0, 0};
#endif
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
                bool valid = candidate(u, ou, bu, ok[d], off[d], &entry);
                if (STATS && valid) ++n_edges;
#if TILE_ZRUN
                bool out = false;
                uint64_t oe = 0;
                if (valid) {
                    const uint32_t pr = uint32_t(entry >> LB) & PMASK, hi = uint32_t(entry) & LMASK;
                    const uint32_t oh = hi == u ? ou : ord[hi];
                    if (pr == run_p[d]) {
                        const uint32_t rhi = uint32_t(run_e[d]) & LMASK;
                        if (oh < run_o[d] || (oh == run_o[d] && hi < rhi)) {
                            run_e[d] = entry;
                            run_o[d] = oh;
                        }
                    } else {
                        out = run_p[d] != ~0u;
                        oe = run_e[d];
                        run_p[d] = pr;
                        run_e[d] = entry;
                        run_o[d] = oh;
                    }
                }
                stage_entry(out, oe, STAGE < 128);
#else
                stage_entry(valid, entry, STAGE < 128);
#endif
            }
            if (STAGE >= 128) stage_entry(false, 0, true);   // flush after the vertex's directions
        }
#if TILE_ZRUN
#pragma unroll
        for (int d = 0; d < 3; ++d) stage_entry(run_p[d] != ~0u, run_e[d], true);
#endif
        if (uint32_t(lane_c) < nst) insert_entry(stage[lane_c]);
    }
#endif
    __syncthreads();
    phase_time(ST_CYC_LIST);
    if (PERSIST && threadIdx.x == 0 && pass == (DUAL ? 1 : 0)) {
        // the staging buffer is idle until the next tile's list phase: the next tile (a dynamic
        // ticket, so that CTAs with cheap tiles take more) has its f copied there now
        const uint32_t nb = gridDim.x + uint32_t(atomicAdd(out0.counters + CTR_TILE, 1ull));
        s_next = nb;
        if (nb < ntiles) {
            uint32_t px, py, pz;
            tile_origin(nb, &px, &py, &pz);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // after the generic-proxy staging
            mbar_expect_tx(&s_fbar, uint32_t(NV) * 4u);
            tma_load_3d(fpre, &fmap, int(px), int(py), int(pz - z_begin), &s_fbar);
        }
    }
    // most table slots are empty: every warp compacts its 1/NW of the table in place (a chunk of
    // 32 slots is read before any of its lanes writes, and a write never lands past the chunk
    // being read); the warp then merges the pairs of its own run
    constexpr int REG = TABLE / NW;
    uint64_t* const run = table + warp_d * REG;
    uint32_t run_len = 0;
#pragma unroll 4
    for (int c = 0; c < REG; c += 32) {
        const uint64_t e = run[c + lane_c];
        const uint32_t m = __ballot_sync(FULL_MASK, e != EMPTY);
        __syncwarp();
        if (e != EMPTY) run[run_len + __popc(m & ((1u << lane_c) - 1u))] = e;
        run_len += __popc(m);
    }
    auto run_edge = [&](uint32_t j, uint32_t* mu, uint32_t* mv, uint64_t* S) {
        const uint64_t e = run[j];
        const uint32_t pair = uint32_t(e >> LB) & PMASK, hi = uint32_t(e) & LMASK;
        const uint32_t ba = pair >> LB, bb = pair & LMASK;
        const bool first = e >> 63;
        *mu = first ? ba : bb;
        *mv = first ? bb : ba;
        *S = key48(ord, hi);
    };
#endif

    // ---- d. merge: Alg. 3 per lane --------------------------------------------------------
    // One iteration (the two cell loads, + the CAS) per loop iteration; a lane whose edge is done
    // takes the next edge of the warp's slice at the top of the next iteration (ballot + popc),
    // so the lanes of a warp stay busy and converged instead of waiting for the longest merge of
    // the warp.  Merge(T, bh, hi, bl) starts straight from the two basins (bh holds the edge's
    // upper endpoint hi, level L = key(hi)).
#if !TILE_KRUSKAL && TILE_MPASS > 1
    // TILE_MPASS level passes: pass p merges the pairs whose upper endpoint's order key (its top
    // OB bits, carried by the entry) falls in the p-th slice of the tile's range, so most merges
    // arrive after the lower ones they would otherwise displace (Alg. 3 accepts any order)
    uint32_t lev_lo = 0, lev_step = 0;
    {
        uint32_t omin = ~0u, omax = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t o = ord[(r0 + k * RSTEP) * TX + lx];
            if (o != ABSENT) {
                omin = min(omin, o);
                omax = max(omax, o);
            }
        }
        omin = __reduce_min_sync(FULL_MASK, omin);
        omax = __reduce_max_sync(FULL_MASK, omax);
        if (lane_c == 0) {
            atomicMin(&s_omin, omin);
            atomicMax(&s_omax, omax);
        }
        __syncthreads();
        lev_lo = s_omin >> (32 - OB);
        const uint32_t hi_b = s_omax >> (32 - OB);
        lev_step = hi_b >= lev_lo ? (hi_b - lev_lo) / TILE_MPASS + 1 : 1;
    }
    constexpr int NPASS = TILE_MPASS;
#else
    constexpr int NPASS = 1;
#endif
#pragma unroll 1
    for (int mp = 0; mp < NPASS; ++mp) {
        bool busy = false;
        uint64_t S = 0, S16 = 0;
        uint32_t mu = 0, mv = 0, run_pos = 0;
        const uint32_t run_n = (TILE_STOP == 0 || TILE_STOP > 3) ? run_len : 0u;
#pragma unroll 1
        while (true) {
            const uint32_t need = __ballot_sync(FULL_MASK, !busy);
            if (need) {
                if (!busy) {
                    const uint32_t j = run_pos + __popc(need & ((1u << lane_c) - 1u));
                    if (j < run_n) {
#if !TILE_KRUSKAL && TILE_MPASS > 1
                        const uint32_t lv = uint32_t((run[j] >> (3 * LB)) & OBMASK);
                        const int p = min(int((lv - lev_lo) / lev_step), NPASS - 1);
                        if (p == mp) {
#else
                        {
#endif
                            if (STATS) ++n_pairs;
                            run_edge(j, &mu, &mv, &S);
                            S16 = S << 16;                    // the level as a cell bound
                            busy = true;
                        }
                    }
                }
                run_pos += __popc(need);
            }
            if (!__any_sync(FULL_MASK, busy) && run_pos >= run_n) break;
            if (busy) {
                if (STATS) ++n_iters;
                const uint64_t cu = sld64(cell + mu), cv = sld64(cell + mv);   // c_key(c) < S <=> c < S16
                const bool up_u = c_v(cu) != mu && cu < S16;        // l.2-4 + R4
                const bool up_v = c_v(cv) != mv && cv < S16;        // l.5-8 + R4
                if (TILE_BOTHCLIMB && (up_u || up_v)) {
                    // the two climbs are independent under one S: both advance in this iteration
                    if (up_u) mu = c_v(cu);
                    if (up_v) mv = c_v(cv);
                    if (TILE_CLIMB2) {
                        // (one more step of each climb still under way: the loop's refill and vote
                        // overhead is paid once for two climb steps)
                        const uint64_t cu2 = up_u ? sld64(cell + mu) : 0ull, cv2 = up_v ? sld64(cell + mv) : 0ull;
                        if (up_u && c_v(cu2) != mu && cu2 < S16) mu = c_v(cu2);
                        if (up_v && c_v(cv2) != mv && cv2 < S16) mv = c_v(cv2);
                    }
                } else if (up_u) {
                    mu = c_v(cu);
                } else if (up_v) {
                    mv = c_v(cv);
                } else if (mu == mv) {                        // l.9-10
                    busy = false;
                } else {
                    uint32_t uu = mu, vv = mv;
                    uint64_t cvv = cv;
                    const uint32_t omv = ord[mv], omu = ord[mu];
                    if (omv < omu || (omv == omu && mv < mu)) { uu = mv; vv = mu; cvv = cu; }   // l.11-12
                    const uint64_t got = scas64(cell + vv, cvv, S16 | uu);                // l.14
                    mu = uu;
                    if (got == cvv) {
                        if (c_v(cvv) == vv) busy = false;      // R5: displaced a root
                        S16 = cvv & ~0xffffull;               // l.15: Merge(T, u, s_v, v')
                        mv = c_v(cvv);
                    } else {
                        mv = vv;                              // l.17: restart
                    }
                }
            }
        }
        if (NPASS > 1) __syncthreads();
    }
    __syncthreads();
    if (s_overflow) {  // (uniform) kept edges / table entries were dropped: merge every edge
        // Merge(T, bh, hi, bl) at level L for every in-tile edge between two basins, one edge at a
        // time per thread (Alg. 3 accepts the edges in any order, redundant ones included)
        auto merge_at = [&](uint32_t bh, uint32_t bl, uint64_t L) {
            uint32_t mu = bh, mv = bl;
            uint64_t S = L;
            while (true) {                                    // Alg. 3
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
        __syncthreads();
    }
    phase_time(ST_CYC_MERGE);

    // ---- e. repair: every cell points at its representative (minimal tile store) -------
    // each thread walks its own 8 vertices in lock-step rounds (8 independent shared-memory
    // load chains in flight); the cells are final after the merge barrier and this phase only
    // reads them, so the representatives stay in registers and go straight to phase f
    uint32_t rep[PER];
#if TILE_REP_SEQ
    // one walk after the other (the loops run the sum of the chain lengths).  TILE_RCHAIN: a walk
    // that starts where the previous one of the thread started, at a threshold not below it,
    // continues from the previous result (the cells are read-only here, so the chain from a start
    // is fixed and Rep(x, a') for a' >= a lies on it past Rep(x, a)); the thread's vertices form a
    // z column and mostly share their basin
    [[maybe_unused]] uint32_t pc_x0 = 0xffffffffu, pc_res = 0;
    [[maybe_unused]] uint64_t pc_a16 = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint64_t cu = cell[(r0 + k * RSTEP) * TX + lx];
        uint32_t x = c_v(cu);
        if (TILE_STOP == 0 || TILE_STOP > 4) {
            const uint64_t a16 = cu | 0xffffull;   // c_key(cx) > c_key(cu)  <=>  cx > a16
            const uint32_t x0 = x;
            if (TILE_RCHAIN && x0 == pc_x0 && a16 >= pc_a16) x = pc_res;
#pragma unroll 1
            while (true) {
                const uint64_t cx = cell[x];
                if (c_v(cx) == x || cx > a16) break;
                x = c_v(cx);
                if (STATS) ++n_rep;
            }
            if (TILE_RCHAIN) {
                pc_x0 = x0;
                pc_a16 = a16;
                pc_res = x;
            }
        }
        rep[k] = x;
    }
#else
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
#endif
    phase_time(ST_CYC_REPAIR);

    // ---- f. write the tile store T0 (8 B per vertex) and the tile minima's 16-byte cells ------
    // T0[u] (into the caller's triplet buffer) = ord(u) << 32 | R(u): for a tile-regular vertex
    // R = Rep_tile(u, key(u)) -- its s = u is final and the repair only re-points v, starting at
    // R with threshold key(u); for a tile minimum R = u.  Only tile minima (s != u, or the tile root) get a 16-byte
    // working cell: the global merge only ever reads or writes cells of tile minima (the
    // crossing edges start at tile representatives, which are minima, and every cell on a v
    // chain from a minimum is a minimum's; DESIGN.md derivation C'''), so regular vertices need
    // none (the x-face records carry (order key, R) for the tile's x faces, coalesced).
    // global ids in 32-bit arithmetic: every id and every partial sum is below n < 2^32
    const uint32_t sxy32 = nx * ny;
    const uint32_t gbase = z0 * sxy32 + y0 * nx + x0;
    auto gid = [&](uint32_t l) -> uint32_t {
        const uint32_t l_x = l % TX, l_r = l / TX;
        return gbase + (l_r / TY) * sxy32 + (l_r % TY) * nx + l_x;
    };
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int r = r0 + k * RSTEP;
        const int ly = r % TY, lz = r / TY;
        const uint32_t u = r * TX + lx;
        const uint32_t ou = ord[u];
        if (ou == ABSENT) continue;
        const uint32_t v = rep[k];
        const uint32_t gu = gbase + uint32_t(lz) * sxy32 + uint32_t(ly) * nx + lx, gv = gid(v);
        const uint64_t cu = cell[u];
        const uint32_t s = c_s(cu);
        const bool minimum = s != u || v == u;
        // T0 = ord(u) << 32 | R(u), R = Rep_tile(u, key(u)) for a tile-regular vertex, u itself for
        // a tile minimum (so R(u) == u tells a minimum apart); the crossing edges read their key and
        // tile representative from it, the repair its threshold and walk start
        const uint64_t t0 = (uint64_t(ou) << 32) | (minimum ? gu : gv);
        T0[gu] = t0;
        // the tile's x faces (lanes 0 and 31) again, compactly (in the grid they are 128 B apart)
        if (lx == 0 || lx == TX - 1) xface[(uint64_t(b) * 2 + (lx == TX - 1)) * ROWS + r] = t0;
        if (minimum) {
            const Cell cc = make_cell(key_of(uint32_t(cu >> 32), s == u ? gu : gid(s)), ou, gv);
            // TILE_FULLSECTOR, even nx: the cell's 32-B sector partner is its x neighbour gu ^ 1 in
            // the same row and tile, never a tile minimum, so one 256-bit store writes the cell into
            // both slots: the whole sector is written and L2 needs no DRAM fill for a partial write
            if (TILE_FULLSECTOR && !(nx & 1u))
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %1, %2};" ::"l"(C + (gu & ~1u)), "l"(cc.lo),
                             "l"(cc.hi)
                             : "memory");
            else
                C[gu] = cc;
        }
    }
    phase_time(ST_CYC_WRITE);
    }   // pass
    if (PERSIST) {
        __syncthreads();            // the next tile overwrites ord and the cells
        b = s_next;
    } else {
        b = ntiles;
    }
    }   // tile
    if (STATS) {
        atomicAdd(stats + ST_TILE_EDGES, n_edges);
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
#define MT_TILE_NV 4096   // vertices per tile (build knob: 8192, 4096 or 2048); tile_shape follows it
#endif
constexpr int tile_vertices() { return MT_TILE_NV; }

void tile_shape(uint32_t nz_global, uint32_t* ty, uint32_t* tz) {
    const int nv = tile_vertices();
    if (nz_global == 1) {
        *ty = uint32_t(nv / TX);
        *tz = 1;
    } else {
        *ty = nv == 2048 ? 8 : 16;
        *tz = nv == 8192 ? 16 : 8;
    }
}

#ifndef TILE_TMA
#define TILE_TMA 1     // stage each tile's f with one TMA bulk tensor copy (grids with nx % 4 == 0)
#endif

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// the slab's f as a 3-D tensor {nx, ny, nz_local} of float32 with tile boxes {32, TY, TZ}; false
// when TMA does not apply (row stride not a multiple of 16 B, unaligned base, no encoder)
template <int TY, int TZ>
bool make_fmap(CUtensorMap* m, const float* f_local, const Slab& sl) {
    const uint64_t nzl = sl.z_end - sl.z_begin;
    if (!TILE_TMA || sl.nx % 4 || (reinterpret_cast<uintptr_t>(f_local) % 16) || nzl == 0) return false;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {sl.nx, sl.ny, nzl};
    const cuuint64_t strides[2] = {uint64_t(sl.nx) * 4, uint64_t(sl.nx) * sl.ny * 4};
    const cuuint32_t box[3] = {uint32_t(TX), uint32_t(TY), uint32_t(TZ)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(f_local), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef TILE_L2PF
#define TILE_L2PF 1    // TMA tiles: L2-prefetch the tile TILE_L2PF waves of resident CTAs ahead (0: off)
#endif

#ifndef TILE_PERSIST
#define TILE_PERSIST 0 // TMA tiles: persistent CTAs, the next tile's f prefetched during the merge
#endif

template <int TY, int TZ, bool STATS, bool DUAL, bool TMA>
void launch_tile_v(const CUtensorMap& m, const float* f, const TileOut& o0, const TileOut& o1, const Slab& sl,
                   uint32_t tx, uint32_t tyn, uint32_t grid, uint32_t flip, unsigned long long* stats,
                   cudaStream_t stream) {
    constexpr int NV = TX * TY * TZ;
    constexpr bool PERSIST = TMA && TILE_PERSIST && !TILE_KRUSKAL;
    auto kern = tile_tmt_kernel<TY, TZ, STATS, DUAL, TMA, PERSIST>;
    ensure_smem_attr(reinterpret_cast<const void*>(kern), int(smem_bytes<NV>()));
    uint32_t blocks = grid, pf = 0;
    if (PERSIST || (TMA && TILE_L2PF)) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint64_t slots = uint64_t(sms) *
                               occupancy_per_sm(reinterpret_cast<const void*>(kern), NV / TILE_VPT, smem_bytes<NV>());
        if (PERSIST && slots < blocks) blocks = uint32_t(slots);   // one CTA per resident slot
        if (!PERSIST) pf = uint32_t(slots * TILE_L2PF);
    }
    kern<<<blocks, NV / TILE_VPT, smem_bytes<NV>(), stream>>>(m, f, o0, o1, grid, sl.nx, sl.ny, sl.z_begin, sl.z_end,
                                                              tx, tyn, flip, stats, pf);
}

template <int TY, int TZ, bool TMA>
void launch_tile_t(const CUtensorMap& m, const float* f, const TileOut& o0, const TileOut* o1, const Slab& sl,
                   uint32_t tx, uint32_t tyn, uint32_t grid, uint32_t flip, unsigned long long* stats,
                   cudaStream_t stream) {
    if (o1) {
        if (stats) launch_tile_v<TY, TZ, true, true, TMA>(m, f, o0, *o1, sl, tx, tyn, grid, 0u, stats, stream);
        else launch_tile_v<TY, TZ, false, true, TMA>(m, f, o0, *o1, sl, tx, tyn, grid, 0u, stats, stream);
    } else {
        if (stats) launch_tile_v<TY, TZ, true, false, TMA>(m, f, o0, o0, sl, tx, tyn, grid, flip, stats, stream);
        else launch_tile_v<TY, TZ, false, false, TMA>(m, f, o0, o0, sl, tx, tyn, grid, flip, stats, stream);
    }
}

template <int TY, int TZ>
void launch_tile(const float* f, const TileOut& o0, const TileOut* o1, const Slab& sl, uint32_t tx, uint32_t tyn,
                 uint32_t grid, uint32_t flip, unsigned long long* stats, cudaStream_t stream) {
    CUtensorMap m;
    memset(&m, 0, sizeof(m));
    if (make_fmap<TY, TZ>(&m, f + sl.base + uint64_t(0), sl))   // f is shifted by -base: the slab's own array
        launch_tile_t<TY, TZ, true>(m, f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
    else
        launch_tile_t<TY, TZ, false>(m, f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
}

void launch_tile_any(const float* f, const TileOut& o0, const TileOut* o1, const Slab& sl, uint32_t flip,
                     unsigned long long* stats, cudaStream_t stream) {
    uint32_t ty, tz;
    tile_shape(sl.nz, &ty, &tz);
    const uint32_t nzl = sl.z_end - sl.z_begin;
    const uint32_t tx = (sl.nx + TX - 1) / TX, tyn = (sl.ny + ty - 1) / ty, tzn = (nzl + tz - 1) / tz;
    const uint32_t grid = tx * tyn * tzn;
    if (grid == 0) return;
#if MT_TILE_NV == 8192
    if (sl.nz == 1) launch_tile<256, 1>(f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
    else launch_tile<16, 16>(f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
#elif MT_TILE_NV == 4096
    if (sl.nz == 1) launch_tile<128, 1>(f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
    else launch_tile<16, 8>(f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
#else
    if (sl.nz == 1) launch_tile<64, 1>(f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
    else launch_tile<8, 8>(f, o0, o1, sl, tx, tyn, grid, flip, stats, stream);
#endif
}

void launch_tile_tmt(const float* f, Cell* C, uint64_t* T0, uint64_t* xface, const Slab& sl, uint32_t flip,
                     unsigned long long* counters, unsigned long long* stats, cudaStream_t stream) {
    launch_tile_any(f, TileOut{C, T0, xface, counters}, nullptr, sl, flip, stats, stream);
}

void launch_tile_tmt_dual(const float* f, Cell* C_join, uint64_t* T0_join, uint64_t* xface_join,
                          unsigned long long* counters_join, Cell* C_split, uint64_t* T0_split,
                          uint64_t* xface_split, unsigned long long* counters_split, const Slab& sl,
                          unsigned long long* stats, cudaStream_t stream) {
    const TileOut o1{C_split, T0_split, xface_split, counters_split};
    launch_tile_any(f, TileOut{C_join, T0_join, xface_join, counters_join}, &o1, sl, 0u, stats, stream);
}

}  // namespace mt
