// repair_diagram.cu -- K4: the repair phase of Alg. 1 (lines 9-11,
// PAPER.md:255-257; Alg. 5 "Repair", with Alg. 4
// "Representative") and K5: the ordered extraction of the
// 0-dimensional persistence diagram (one point (f(a), f(b))
// per branch).
//
// Repair (repair_brick_kernel): T[u] = (s, v) becomes (s, Rep(u, key(s))), Rep
// following cells while key(s') <= key(s) and the cell is not a root.
// Reading R20: the walk returns the vertex it stopped at (Alg. 4 as printed
// returns the next, too-deep v).  The walks only read the working cells (the
// repaired pointer goes to T), so they see the fixed post-merge store.
//   The cells are read-only during the repair, so the walks use non-coherent
// L1-cached loads: the vertices of a brick mostly walk the same few chains of
// cells (their tile representatives and the minima these merged into), which
// stay in L1.  (A shared-memory memo of the brick's distinct chains, one walk
// per distinct start vertex, was measured slower: c5 19.0 vs 14.0 ms.)
//
// Diagram: after the merge phase the s fields are final (repair only rewrites
// v).  A cell with s != u is the branch born at u dying at saddle s (finite
// pair) and a root (u, u, u) is an essential class.  The
// repair bricks, which read every cell anyway, stage these records per
// segment (a brick row: <= 32 consecutive ids) with the segment's counts;
// diagram_kernel then walks the segments in id order and places the records
// with a single-pass ordered compaction (CTA scan + decoupled look-back over
// 16-B tile records), so the pairs come out in ascending u.  Tiles take
// dynamic ticket numbers so every predecessor is already resident.
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

// cell / value access for the repair walk: everything local (one GPU), or local
// cells plus the merged boundary forest of all slabs (multi-GPU, slab.cu)
#ifndef MT_REPAIR_NC
#define MT_REPAIR_NC 1      // the repair reads cells no thread writes: L1-cached non-coherent loads
#endif
#ifndef MT_REPAIR_SEQ
#define MT_REPAIR_SEQ 1     // walks one after the other (else lock-step rounds over the thread's vertices)
#endif
#ifndef MT_REPAIR_ZPAIR
#define MT_REPAIR_ZPAIR 1   // volumes: launch the bricks of one tile depth back to back (c5 repair 10.15 -> 9.99 ms)
#endif
#ifndef MT_REPAIR_BLOCK
#define MT_REPAIR_BLOCK 1   // volumes (with ZPAIR): bricks in 4 x 4 x 4 blocks of tile columns (c5 repair 9.89 -> 9.67 ms)
#endif
#ifndef MT_REPAIR_STOP
#define MT_REPAIR_STOP 0    // timing only (WRONG results): 1 the T0 -> T stream alone, 2 + cells and records
#endif
#ifndef MT_REPAIR_FIXSTAGE
#define MT_REPAIR_FIXSTAGE 1  // grid bricks stage their records at a fixed offset (no global atomic; c5 repair 9.67 -> 8.91 ms)
#endif
#ifndef MT_REPAIR_PRE
#define MT_REPAIR_PRE 0     // walks: the first cells of this many walks loaded together (0: off; 1, 2 or 4)
#endif
#ifndef MT_REPAIR_SEGSTAGE
#define MT_REPAIR_SEGSTAGE 0  // grid bricks: 16 staging slots per segment (no prefix, no barrier)
#endif
#ifndef MT_REPAIR_CHAIN
#define MT_REPAIR_CHAIN 0   // a thread's walks in threshold order, chained from a shared start
#endif
#ifndef MT_REPAIR_SKIPW
#define MT_REPAIR_SKIPW 0   // tiled: no store for a tile-regular vertex whose T0 is already final
#endif
#ifndef MT_REPAIR_MINB
#define MT_REPAIR_MINB 3    // __launch_bounds__ min blocks per SM (register budget knob)
#endif
__device__ __forceinline__ Cell ld_cell_ro(const Cell* p) { return MT_REPAIR_NC ? ld_cell_nc(p) : ld_cell(p); }

struct LocalView {
    __device__ __forceinline__ Cell cell(const Cell* C, uint32_t x) const { return ld_cell_ro(C + x); }
    __device__ __forceinline__ float value(const float* f, uint32_t x) const { return __ldg(f + x); }
};

struct ForestView {
    ForestRef F;
    uint64_t base, n;  // owned global ids [base, base + n)
    __device__ __forceinline__ bool mine(uint32_t x) const { return uint64_t(x) - base < n; }
    __device__ __forceinline__ Cell cell(const Cell* C, uint32_t x) const {
        if (mine(x)) return ld_cell_ro(C + x);
        const uint32_t i = forest_lookup(F, x);
        if (i == FOREST_MISS) {            // incomplete records: report, stop the walk here
            atomicOr(F.err, ERR_FOREST);
            return Cell{~0ull, x};
        }
        return Cell{F.cells[i].lo, F.cells[i].hi};
    }
    // f of a remote saddle with a zero value (the only ones the repair gathers): a record's own
    // f bits, else the saddle table of forest_build
    __device__ __forceinline__ float value(const float* f, uint32_t x) const {
        if (mine(x)) return __ldg(f + x);
        const uint32_t i = forest_lookup(F, x);
        if (i != FOREST_MISS) return __uint_as_float(F.recs[i].f_bits);
        uint32_t bits = 0;
        if (!forest_value(F, x, &bits)) atomicOr(F.err, ERR_FOREST);
        return __uint_as_float(bits);
    }
};

// bit pattern of the float whose order key is o (inverse of ord32 for every value but -0)
__device__ __forceinline__ uint32_t inv_ord(uint32_t o) { return (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o; }

// ============================ K4: repair ====================================
// Brick of 32 x BY x BZ vertices (BY * BZ = RB_ROWS rows of 32), one CTA of
// RB_THREADS; each warp owns RB_ROWS / 16 rows (lane = x).  LINEAR bricks are
// 4096 consecutive ids instead (graphs, thin grids).  A row of a brick is a
// "segment" of at most 32 consecutive ids; segments are numbered in id order.
constexpr int RB_THREADS = 512;
#ifndef MT_REPAIR_ROWS
#define MT_REPAIR_ROWS 64   // rows of 32 per brick (a 32 x 16 x 4 brick; 2-D: 32 x 64): 4 vertices per thread
#endif
constexpr int RB_ROWS = MT_REPAIR_ROWS;
constexpr int RB_PER = RB_ROWS / (RB_THREADS / 32);   // rows (vertices) per thread
constexpr int RB_NV = RB_ROWS * 32;

struct RepairSmem {
    uint32_t rowcnt[RB_ROWS];          // finite | essential << 16 records of each row
    uint32_t rowoff[RB_ROWS];          // their offset in the brick's staging run
    uint64_t rowbase[RB_ROWS];         // first id of each row
    uint64_t rowseg[RB_ROWS];          // its segment number
    uint32_t rowlim[RB_ROWS];          // lanes of the row inside the grid
    uint32_t rowfm[RB_ROWS], rowem[RB_ROWS];   // lanes holding a finite pair / a root
    uint32_t base;
};

struct BrickGeom {
    uint32_t by, bx_n, by_n;   // brick rows along y; bricks along x and y (brick mode)
    uint32_t blocked;          // MT_REPAIR_BLOCK: tile-pair columns visited in 4 x 4 x 4 blocks
};

template <class View, int BY, bool TILED, bool COUNT>
__global__ void __launch_bounds__(RB_THREADS, MT_REPAIR_MINB)
repair_brick_kernel(View view, const Cell* C, uint64_t* __restrict__ T, const float* __restrict__ f, Slab sl,
                    BrickGeom g, uint32_t flip, mt_pair* __restrict__ stage, uint64_t stage_cap,
                    uint16_t* __restrict__ seg_cnt, uint32_t* __restrict__ seg_pos,
                    unsigned long long* __restrict__ counters, unsigned long long* __restrict__ stats) {
    // TILED (grids): T holds the tile store T0 written by tile_tmt and only tile minima have
    // working cells; a regular vertex's walk starts at its tile representative T0.v with
    // threshold key(u) (its s = u is final).  Otherwise (explicit graphs) every vertex has a
    // working cell and T is output only.
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RepairSmem& S = *reinterpret_cast<RepairSmem*>(smem_raw);
    constexpr bool LINEAR = BY == 0;       // id-range bricks (graphs, thin grids)
    constexpr uint32_t BYD = LINEAR ? 1u : uint32_t(BY);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;

    // brick origin and the id-order number of its first segment
    uint64_t u0 = 0, seg0 = 0;
    uint32_t x0 = 0, y0 = 0, z0 = 0, bxi = 0;
    if (LINEAR) {
        u0 = uint64_t(blockIdx.x) * RB_NV;
        seg0 = uint64_t(blockIdx.x) * RB_ROWS;
    } else {
        // (MT_REPAIR_ZPAIR, volumes: the two bricks of one tile depth run back to back, so that
        // the second finds the tile's minima cells still in L2)
        constexpr bool ZP = MT_REPAIR_ZPAIR && BY == 16;
        // origin of brick number bi in launch order
        auto origin = [&](uint32_t bi, uint32_t* ox, uint32_t* oy, uint32_t* oz) {
            const uint32_t b = ZP ? bi >> 1 : bi;
            uint32_t bx, byi, bzi;
            if (ZP && MT_REPAIR_BLOCK && g.blocked) {
                // 4 x 4 x 4 blocks of tile-pair columns, one block after the other: the neighbours
                // a tile's walks reach (its z neighbours too) run close in time
                const uint32_t blk = b >> 6, w = b & 63u, nbx = g.bx_n >> 2, nby = g.by_n >> 2;
                bx = (blk % nbx) * 4 + (w & 3u);
                byi = ((blk / nbx) % nby) * 4 + ((w >> 2) & 3u);
                bzi = (blk / nbx / nby) * 4 + (w >> 4);
            } else {
                bx = b % g.bx_n;
                byi = (b / g.bx_n) % g.by_n;
                bzi = b / g.bx_n / g.by_n;
            }
            *ox = bx;
            *oy = byi * BYD;
            *oz = sl.z_begin + (bzi * (ZP ? 2 : 1) + (ZP ? (bi & 1) : 0)) * (RB_ROWS / BYD);
        };
        origin(blockIdx.x, &bxi, &y0, &z0);
        x0 = bxi * 32;
    }
    // the warp's rows (item k = row warp + 16 k): first id, valid lanes and segment number, computed
    // once by lanes 0..RB_PER-1 (integer divisions) and read back from shared memory
    if (lane < RB_PER) {
        const uint32_t r = uint32_t(warp + 16 * lane);
        uint64_t rb, seg;
        uint32_t lim;
        if (LINEAR) {
            rb = sl.base + u0 + uint64_t(r) * 32;
            const uint64_t left = u0 + uint64_t(r) * 32 < sl.n ? sl.n - (u0 + uint64_t(r) * 32) : 0;
            lim = left > 32 ? 32u : uint32_t(left);
            seg = seg0 + r;
        } else {
            const uint32_t y = y0 + r % BYD, z = z0 + r / BYD;
            rb = (uint64_t(z) * sl.ny + y) * sl.nx + x0;
            lim = (y < sl.ny && z < sl.z_end) ? min(32u, sl.nx - x0) : 0u;
            seg = (uint64_t(z - sl.z_begin) * sl.ny + y) * g.bx_n + bxi;
        }
        S.rowbase[r] = rb;
        S.rowseg[r] = seg;
        S.rowlim[r] = lim;
    }
    __syncwarp();
    uint32_t inb = 0;
#pragma unroll
    for (int k = 0; k < RB_PER; ++k) inb |= uint32_t(uint32_t(lane) < S.rowlim[warp + 16 * k]) << k;
#define UID(k) (S.rowbase[warp + 16 * (k)] + lane)
#define INB(k) ((inb >> (k)) & 1u)
    uint64_t key[RB_PER];     // threshold key(s)
    uint32_t sv[RB_PER];      // s of the vertex
    uint32_t xs[RB_PER];      // walk start (then position)
    uint32_t mins = 0;        // rows k whose vertex has a working cell (bit k)
    if (TILED) {
        // every load of the thread in flight at once: the tile store of all its vertices (its
        // order key and tile representative), then the working cells of the tile minima among them
        uint64_t t0[RB_PER];
#pragma unroll
        for (int k = 0; k < RB_PER; ++k) t0[k] = INB(k) ? T[UID(k)] : 0;
#pragma unroll
        for (int k = 0; k < RB_PER; ++k) {
            const uint32_t u = uint32_t(UID(k));
            if (cell_v(t0[k]) != u) {            // regular in its tile: s = u is final
                key[k] = key_of(cell_s(t0[k]), u);
                sv[k] = u;
                xs[k] = cell_v(t0[k]);
            } else {
                mins |= uint32_t(INB(k)) << k;
                key[k] = 0;
                sv[k] = u;
                xs[k] = u;
            }
        }
    } else {
        mins = inb;
    }
    if (MT_REPAIR_STOP == 1 && TILED) {   // timing only (WRONG results): the T0 -> T stream alone
#pragma unroll
        for (int k = 0; k < RB_PER; ++k)
            if (INB(k)) T[UID(k)] = pack(sv[k], xs[k]);
        return;
    }
#pragma unroll
    for (int k = 0; k < RB_PER; ++k) {
        if (!((mins >> k) & 1u)) continue;
        const Cell c = ld_cell_ro(C + UID(k));               // a minimum's working cell
        key[k] = c.lo;
        sv[k] = cs_of(c);
        xs[k] = cv_of(c);
    }
    // diagram records of each row: finite pairs (s != u) and roots (v == u)
#define FMASK(k) __ballot_sync(FULL_MASK, INB(k) && sv[k] != uint32_t(UID(k)))
#define EMASK(k) __ballot_sync(FULL_MASK, INB(k) && xs[k] == uint32_t(UID(k)))
    uint32_t recbits = 0;     // rows k where this lane holds a finite pair (bit k) / a root (bit 8 + k)
#pragma unroll
    for (int k = 0; k < RB_PER; ++k) {
        const uint32_t fm = FMASK(k), em = EMASK(k);
        recbits |= (((fm >> lane) & 1u) << k) | (((em >> lane) & 1u) << (8 + k));
        if (lane == 0) {
            S.rowcnt[warp + 16 * k] = __popc(fm) | (__popc(em) << 16);
            S.rowfm[warp + 16 * k] = fm;
            S.rowem[warp + 16 * k] = em;
        }
    }
    // MT_REPAIR_SEGSTAGE (grid bricks): every segment (row) stages its records at a fixed run of
    // 16 (strict minima of <= 32 x-consecutive vertices: an independent set of a path, so at most
    // half of them), so a warp needs nothing from the other warps: no barrier, no brick prefix
    constexpr bool SEGST = MT_REPAIR_SEGSTAGE && !LINEAR;
    if (SEGST) __syncwarp();
    else __syncthreads();   // row counts in

    // warp 0: the brick's staging run (one global atomic) and each row's offset in it
    if (!SEGST && warp == 0) {
        uint32_t c[RB_ROWS / 32], tot = 0;
#pragma unroll
        for (int j = 0; j < RB_ROWS / 32; ++j) {
            const uint32_t rc = S.rowcnt[lane * (RB_ROWS / 32) + j];
            c[j] = (rc & 0xffffu) + (rc >> 16);
            tot += c[j];
        }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        uint32_t off = incl - tot;
#pragma unroll
        for (int j = 0; j < RB_ROWS / 32; ++j) {
            S.rowoff[lane * (RB_ROWS / 32) + j] = off;
            off += c[j];
        }
        const uint32_t all = __shfl_sync(FULL_MASK, incl, 31);
        uint32_t base = 0;
        if (MT_REPAIR_FIXSTAGE && !LINEAR) {
            // grid bricks: a fixed run of RB_NV / 2 records per brick (its records are strict
            // minima, an independent set of the bipartite brick, so at most half its vertices):
            // no global atomic, no wait for one
            base = uint32_t(blockIdx.x) * uint32_t(RB_NV / 2);
        } else if (lane == 0 && all) {
            base = uint32_t(atomicAdd(counters + CTR_STAGE, (unsigned long long)all));
        }
        if (lane == 0) S.base = base;
    }

    if (!SEGST) __syncthreads();   // staging base and row offsets in

    // staging records of every row, in id order within the row: finite pairs, then roots.
    // Lanes 0..7 publish the counts and staging offsets of the warp's 8 rows; then every lane
    // stages only its own records (few: ~5 % of the vertices at c5), so the record code runs
    // max-over-lanes times instead of once per row
    const uint32_t sbase = SEGST ? 0u : S.base;
    if (lane < RB_PER) {
        const int r = warp + 16 * lane;
        if (S.rowlim[r] > 0) {   // every row holding a vertex of the grid is a segment
            const uint64_t seg = S.rowseg[r];
            seg_cnt[seg] = uint16_t(S.rowcnt[r] & 0xffffu) | uint16_t((S.rowcnt[r] >> 16) << 8);
            if (!SEGST) seg_pos[seg] = sbase + S.rowoff[r];
        }
    }
    uint32_t rm = (recbits | (recbits >> 8)) & 0xffu;
#pragma unroll 1
    while (rm) {
        const int k = __ffs(rm) - 1;
        rm &= rm - 1;
        const int r = warp + 16 * k;
        const uint32_t fm = S.rowfm[r], em = S.rowem[r];
        const bool isf = (recbits >> k) & 1u;
        const uint64_t u = S.rowbase[r] + lane;
        // this row's cell again (an L1 hit: loaded above through the non-coherent path) rather
        // than a dynamically indexed register array
        const Cell cu = ld_cell_ro(C + u);
        const uint32_t s = cs_of(cu), ou = uint32_t(cu.hi >> 32), os = uint32_t(cu.lo >> 32);
        const uint64_t pos = (SEGST ? S.rowseg[r] * 16u : uint64_t(sbase) + S.rowoff[r]) +
                             (isf ? __popc(fm & lt) : __popc(fm) + __popc(em & lt));
        mt_pair rec;
        if (isf) {
            // values f[u] and f[s]: the cell carries ord(f[u]) (hi) and ord(f[s]) (lo); invert
            // them (exact for every value but zero, whose sign the canonicalisation -0 -> +0
            // dropped: gather those, reading R14)
            const uint32_t bb = inv_ord(ou ^ flip);
            const uint32_t db = inv_ord(os ^ flip);
            rec = mt_pair{uint32_t(u), s, bb == 0u ? __ldg(f + u) : __uint_as_float(bb),
                          db == 0u ? view.value(f, s) : __uint_as_float(db)};
        } else {
            rec = mt_pair{uint32_t(u), uint32_t(u), __ldg(f + u), __int_as_float(0x7f800000)};
        }
        if (pos < stage_cap) stage[pos] = rec;
        else atomicOr(counters + CTR_ERR, ERR_CAPACITY);
    }

    if (MT_REPAIR_STOP == 2 && TILED) {   // timing only (WRONG results): no walks
#pragma unroll
        for (int k = 0; k < RB_PER; ++k)
            if (INB(k)) T[UID(k)] = pack(sv[k], xs[k]);
        return;
    }
    // Rep(u, key(s)): walk from v through cells with key(s') <= key(s) that are not roots
    unsigned long long hops = 0;   // (COUNT builds only: mt_set_stats)
    [[maybe_unused]] uint32_t moved = 0;   // rows whose walk left its start (bit k)
#if MT_REPAIR_CHAIN
    // The thread's walks in ascending threshold order, each continuing from the result of the
    // previous walk when both start at the same vertex: the cells are read-only here, so the
    // chain from a start vertex is fixed and Rep(x, a') for a' >= a lies on it past Rep(x, a)
    // (Alg. 4 stops at the first cell that is a root or has key(s) > a).  A thread's vertices
    // form a z column and mostly share their tile representative, so the chain is walked about
    // once instead of once per vertex.  Sorted in registers (5 compare-exchanges); T is written
    // in that order.
    static_assert(RB_PER == 4 && !MT_REPAIR_SKIPW, "repair chaining: 4 vertices per thread");
    {
        uint64_t tk[RB_PER];
        uint32_t tx[RB_PER], ts[RB_PER], ti[RB_PER];
#pragma unroll
        for (int k = 0; k < RB_PER; ++k) {
            const bool walk = INB(k) && xs[k] != uint32_t(UID(k));
            tk[k] = INB(k) ? key[k] : ~0ull;
            tx[k] = xs[k];
            ts[k] = sv[k];
            ti[k] = uint32_t(k) | (uint32_t(walk) << 8) | (uint32_t(INB(k)) << 9);
        }
        auto cx = [&](int a, int b) {
            if (tk[b] < tk[a]) {
                uint64_t t = tk[a]; tk[a] = tk[b]; tk[b] = t;
                uint32_t u = tx[a]; tx[a] = tx[b]; tx[b] = u;
                u = ts[a]; ts[a] = ts[b]; ts[b] = u;
                u = ti[a]; ti[a] = ti[b]; ti[b] = u;
            }
        };
        cx(0, 1);
        cx(2, 3);
        cx(0, 2);
        cx(1, 3);
        cx(1, 2);
        // memo: the previous walk's start, result and the result's cell (which stopped that walk:
        // a root or a saddle above its threshold) -- a chained walk first tests that cell in
        // registers, so it loads nothing when the same cell stops it too
        uint32_t memo_x0 = ~0u, memo_res = 0;
        Cell memo_c{0, 0};
#pragma unroll
        for (int r = 0; r < RB_PER; ++r) {
            if (!((ti[r] >> 9) & 1u)) continue;
            uint32_t x = tx[r];
            if ((ti[r] >> 8) & 1u) {
                const uint32_t x0 = x;
                Cell c{0, 0};
                bool have = false;
                if (x0 == memo_x0) {
                    x = memo_res;
                    c = memo_c;
                    have = true;
                }
#pragma unroll 1
                while (true) {
                    if (!have) c = view.cell(C, x);
                    have = false;
                    if (cv_of(c) == x || c.lo > tk[r]) break;   // Alg. 4, reading R20
                    x = cv_of(c);
                    if (COUNT) ++hops;
                }
                memo_x0 = x0;
                memo_res = x;
                memo_c = c;
            }
            T[S.rowbase[warp + 16 * (ti[r] & 0xffu)] + lane] = pack(ts[r], x);
        }
    }
#elif MT_REPAIR_SEQ
    // one walk after the other (the loop runs the sum of the chain lengths, not RB_PER times
    // the longest); MT_REPAIR_PRE: the first cells of MT_REPAIR_PRE walks are loaded together
    // (independent loads in flight), the walks then continue one after the other
#if MT_REPAIR_PRE
    static_assert(RB_PER % MT_REPAIR_PRE == 0, "MT_REPAIR_PRE divides the vertices per thread");
#pragma unroll
    for (int k0 = 0; k0 < RB_PER; k0 += MT_REPAIR_PRE) {
        uint64_t plo[MT_REPAIR_PRE];
        uint32_t pv[MT_REPAIR_PRE];
#pragma unroll
        for (int j = 0; j < MT_REPAIR_PRE; ++j) {
            const int k = k0 + j;
            plo[j] = 0;
            pv[j] = 0;
            if (INB(k) && xs[k] != uint32_t(UID(k))) {
                const Cell c = view.cell(C, xs[k]);
                plo[j] = c.lo;
                pv[j] = cv_of(c);
            }
        }
#pragma unroll
        for (int j = 0; j < MT_REPAIR_PRE; ++j) {
            const int k = k0 + j;
            if (!INB(k) || xs[k] == uint32_t(UID(k))) continue;
            uint32_t x = xs[k];
            uint64_t clo = plo[j];
            uint32_t cv = pv[j];
#pragma unroll 1
            while (true) {
                if (cv == x || clo > key[k]) break;   // Alg. 4, reading R20
                x = cv;
                if (COUNT) ++hops;
                const Cell c = view.cell(C, x);
                clo = c.lo;
                cv = cv_of(c);
            }
            moved |= uint32_t(x != xs[k]) << k;
            xs[k] = x;
        }
    }
#else
#pragma unroll
    for (int k = 0; k < RB_PER; ++k) {
        if (!INB(k) || xs[k] == uint32_t(UID(k))) continue;
        uint32_t x = xs[k];
#pragma unroll 1
        while (true) {
            const Cell c = view.cell(C, x);
            if (cv_of(c) == x || c.lo > key[k]) break;   // Alg. 4, reading R20
            x = cv_of(c);
            if (COUNT) ++hops;
        }
        moved |= uint32_t(x != xs[k]) << k;
        xs[k] = x;
    }
#endif
#else
    // the thread's walks advance in lock-step rounds: independent load chains in flight
    uint32_t act = 0;
#pragma unroll
    for (int k = 0; k < RB_PER; ++k)
        if (INB(k) && xs[k] != uint32_t(UID(k))) act |= 1u << k;
#pragma unroll 1
    while (act) {
#pragma unroll
        for (int k = 0; k < RB_PER; ++k) {
            if (!((act >> k) & 1u)) continue;
            const Cell c = view.cell(C, xs[k]);
            if (cv_of(c) == xs[k] || c.lo > key[k]) {     // Alg. 4, reading R20
                act &= ~(1u << k);
            } else {
                xs[k] = cv_of(c);
                moved |= 1u << k;
                if (COUNT) ++hops;
            }
        }
    }
#endif
#if !MT_REPAIR_CHAIN
    // a tile-regular vertex whose walk stayed at its tile representative keeps T0 = (u, R)
    const uint32_t keep = (TILED && MT_REPAIR_SKIPW) ? ~(moved | mins) : 0u;
#pragma unroll
    for (int k = 0; k < RB_PER; ++k)
        if (INB(k) && !((keep >> k) & 1u)) T[UID(k)] = pack(sv[k], xs[k]);
#endif
    if (COUNT && hops) atomicAdd(stats + ST_REPAIR_HOPS, hops);
#undef UID
#undef INB
#undef FMASK
#undef EMASK
}

// ============================ K5: diagram ===================================
// One thread per segment, segments in id order: the counts give each record's
// place in the diagram (ordered compaction: CTA scan + decoupled look-back);
// the records are copied from the staging runs the repair wrote.
constexpr int THREADS = 256;
#ifndef DG_SPT_BIG
#define DG_SPT_BIG 2        // diagram: segments per thread on grids of >= DG_BIG segments (c5: 2 0.98 ms, 4 1.04, 8 1.14)
#endif
#ifndef DG_BIG
#define DG_BIG (1ull << 24) // diagram: from this many segments on, 4 segments per thread (fewer tiles in the
#endif                      // look-back chain: c5 1.31 -> 1.07 ms in round 1; 1 below: c4 0.39 vs 0.56 ms)
constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_VAL = (1ull << 62) - 1;

template <int DG_SPT>
__global__ void __launch_bounds__(THREADS)
diagram_kernel(const uint16_t* __restrict__ seg_cnt, const uint32_t* __restrict__ seg_pos, uint64_t nseg,
               const mt_pair* __restrict__ stage, unsigned long long* __restrict__ counters, Cell* __restrict__ status,
               mt_pair* __restrict__ out, uint64_t out_cap, mt_pair* __restrict__ ess, uint64_t ess_cap,
               uint64_t ntiles, bool seg16) {
    __shared__ uint64_t s_tile;
    __shared__ uint32_t s_w[THREADS / 32], s_we[THREADS / 32];
    __shared__ uint64_t s_prefix, s_eprefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(counters + CTR_TICKET, 1ull);
    __syncthreads();
    const uint64_t tile = s_tile;
    // DG_SPT consecutive segments per thread (fewer tiles in the look-back chain)
    const uint64_t seg = (tile * THREADS + threadIdx.x) * DG_SPT;
    uint32_t cnts[DG_SPT];
    uint32_t cf = 0, ce = 0;
#pragma unroll
    for (int j = 0; j < DG_SPT; ++j) {
        cnts[j] = seg + j < nseg ? seg_cnt[seg + j] : 0u;
        cf += cnts[j] & 0xffu;
        ce += cnts[j] >> 8;
    }
    // the staging offsets and every segment's first record are loaded before the scans and the
    // look-back, so those loads overlap the chain instead of following it
    uint32_t spos[DG_SPT];
    mt_pair first[DG_SPT];
#pragma unroll
    for (int j = 0; j < DG_SPT; ++j) {
        spos[j] = cnts[j] ? (seg16 ? uint32_t((seg + j) * 16u) : seg_pos[seg + j]) : 0u;
        if (cnts[j]) first[j] = stage[spos[j]];
    }
    // block-wide exclusive scans (finite, essential)
    uint32_t incl = cf, eincl = ce;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
        const uint32_t te = __shfl_up_sync(FULL_MASK, eincl, o);
        if (lane >= o) {
            incl += t;
            eincl += te;
        }
    }
    if (lane == 31) {
        s_w[warp] = incl;
        s_we[warp] = eincl;
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < THREADS / 32 ? s_w[lane] : 0u, we = lane < THREADS / 32 ? s_we[lane] : 0u;
        uint32_t wi = w, wei = we;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, wi, o);
            const uint32_t te = __shfl_up_sync(FULL_MASK, wei, o);
            if (lane >= o) {
                wi += t;
                wei += te;
            }
        }
        if (lane < THREADS / 32) {
            s_w[lane] = wi - w;
            s_we[lane] = wei - we;
        }
        const uint32_t agg = __shfl_sync(FULL_MASK, wi, 31), eagg = __shfl_sync(FULL_MASK, wei, 31);
        const uint64_t fl = tile == 0 ? ST_PRE : ST_AGG;
        if (lane == 0) st_cell(status + tile, Cell{fl | agg, fl | eagg});
        uint64_t prefix = 0, eprefix = 0;
        int64_t j = int64_t(tile) - 1;
        while (j >= 0) {
            const int64_t idx = j - lane;
            const Cell sv = idx >= 0 ? ld_cell(status + idx) : Cell{ST_PRE, ST_PRE};
            const uint64_t flag = sv.lo >> 62;
            const uint32_t pmask = __ballot_sync(FULL_MASK, flag == 2);
            const uint32_t xmask = __ballot_sync(FULL_MASK, flag == 0);
            const int first_p = pmask ? __ffs(pmask) - 1 : 31;
            const uint32_t upto = first_p == 31 ? FULL_MASK : ((2u << first_p) - 1u);
            if (xmask & upto) continue;               // a needed predecessor has not published
            uint64_t val = lane <= first_p ? (sv.lo & ST_VAL) : 0;
            uint64_t eval = lane <= first_p ? (sv.hi & ST_VAL) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                val += __shfl_xor_sync(FULL_MASK, val, o);
                eval += __shfl_xor_sync(FULL_MASK, eval, o);
            }
            prefix += val;
            eprefix += eval;
            if (pmask) break;
            j -= 32;
        }
        if (lane == 0) {
            s_prefix = prefix;
            s_eprefix = eprefix;
            if (tile != 0) st_cell(status + tile, Cell{ST_PRE | (prefix + agg), ST_PRE | (eprefix + eagg)});
            if (tile == ntiles - 1) {
                counters[CTR_FIN] = prefix + agg;
                counters[CTR_ESS] = eprefix + eagg;
            }
        }
    }
    __syncthreads();
    if (!(cf | ce)) return;
    const uint64_t pos = s_prefix + s_w[warp] + incl - cf;
    const uint64_t epos = s_eprefix + s_we[warp] + eincl - ce;
    uint64_t p = pos, ep = epos;
#pragma unroll
    for (int j = 0; j < DG_SPT; ++j) {
        const uint32_t fj = cnts[j] & 0xffu, ej = cnts[j] >> 8;
        if (!(fj | ej)) continue;
        const mt_pair* src = stage + spos[j];
        for (uint32_t i = 0; i < fj; ++i) {
            if (p + i < out_cap) out[p + i] = i ? src[i] : first[j];
            else atomicOr(counters + CTR_ERR, ERR_CAPACITY);
        }
        for (uint32_t i = 0; i < ej; ++i) {
            if (ep + i < ess_cap) ess[ep + i] = (fj + i) ? src[fj + i] : first[j];
            else atomicOr(counters + CTR_ERR, ERR_ESS_CAPACITY);
        }
        p += fj;
        ep += ej;
    }
}

// Appends the essential classes (already in ascending vertex order) after the
// finite pairs and checks the capacity.
__global__ void finish_diagram_kernel(unsigned long long* __restrict__ counters, mt_pair* __restrict__ out,
                                      uint64_t out_cap, mt_pair* __restrict__ ess, uint64_t ess_cap) {
    const uint64_t nfin = counters[CTR_FIN];
    uint64_t ness = counters[CTR_ESS];
    if (ness > ess_cap) ness = ess_cap;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < ness; i += uint64_t(gridDim.x) * blockDim.x) {
        if (nfin + i < out_cap) out[nfin + i] = ess[i];
        else atomicOr(counters + CTR_ERR, ERR_CAPACITY);
    }
}

template <class View, int BY, bool TILED, bool COUNT>
void launch_brick_v(const View& view, const Cell* C, uint64_t* T, const float* f, const Slab& sl, BrickGeom g,
                    uint64_t nb, uint32_t flip, const RepairOut& o, unsigned long long* stats, cudaStream_t stream) {
    auto kern = repair_brick_kernel<View, BY, TILED, COUNT>;
    ensure_smem_attr(reinterpret_cast<const void*>(kern), int(sizeof(RepairSmem)));
    kern<<<uint32_t(nb), RB_THREADS, sizeof(RepairSmem), stream>>>(view, C, T, f, sl, g, flip, o.stage, o.stage_cap,
                                                                  o.seg_cnt, o.seg_pos, o.counters, stats);
}

template <class View, int BY>
void launch_brick(const View& view, const Cell* C, uint64_t* T, const float* f, const Slab& sl, BrickGeom g,
                  uint64_t nb, uint32_t flip, const RepairOut& o, bool tiled, unsigned long long* stats,
                  cudaStream_t stream) {
    // the hop counter of the statistics costs an add per walk step: a separate instantiation
    if (tiled && stats) launch_brick_v<View, BY, true, true>(view, C, T, f, sl, g, nb, flip, o, stats, stream);
    else if (tiled) launch_brick_v<View, BY, true, false>(view, C, T, f, sl, g, nb, flip, o, stats, stream);
    else if (stats) launch_brick_v<View, BY, false, true>(view, C, T, f, sl, g, nb, flip, o, stats, stream);
    else launch_brick_v<View, BY, false, false>(view, C, T, f, sl, g, nb, flip, o, stats, stream);
}

// brick geometry: 3-D bricks 32 x 16 x (RB_ROWS / 16) on volumes, 32 x RB_ROWS on images, id ranges otherwise
bool brick_mode(const Slab& sl, BrickGeom* g, uint64_t* nb, uint64_t* nseg) {
    const uint32_t nzl = sl.z_end - sl.z_begin;
    uint32_t by = 0;
    if (nzl >= uint32_t(RB_ROWS / 16) && sl.ny >= 16) by = 16;
    else if (sl.nz == 1 && sl.ny >= uint32_t(RB_ROWS)) by = RB_ROWS;
    if (by && sl.nx >= 32) {
        const uint32_t bz = RB_ROWS / by;
        const uint32_t bx_n = (sl.nx + 31) / 32, by_n = (sl.ny + by - 1) / by, bz_n = (nzl + bz - 1) / bz;
        const uint32_t bz2 = (bz_n + 1) / 2;   // tile-pair layers (ZPAIR)
        const bool blocked = MT_REPAIR_ZPAIR && by == 16 && bx_n % 4 == 0 && by_n % 4 == 0 && bz2 % 4 == 0;
        *g = BrickGeom{by, bx_n, by_n, blocked ? 1u : 0u};
        *nb = uint64_t(bx_n) * by_n * ((MT_REPAIR_ZPAIR && by == 16) ? bz2 * 2 : bz_n);
        *nseg = uint64_t(bx_n) * sl.ny * nzl;
        return true;
    }
    *g = BrickGeom{1, 1, 1, 0};
    *nb = (sl.n + RB_NV - 1) / RB_NV;
    *nseg = (sl.n + 31) / 32;
    return false;
}

template <class View>
void launch_repair_view(const View& view, const Cell* C, uint64_t* T, const float* f, const Slab& sl, uint32_t flip,
                        const RepairOut& o, bool tiled, unsigned long long* stats, cudaStream_t stream) {
    BrickGeom g;
    uint64_t nb, nseg;
    if (!brick_mode(sl, &g, &nb, &nseg)) launch_brick<View, 0>(view, C, T, f, sl, g, nb, flip, o, tiled, stats, stream);
    else if (g.by == 16) launch_brick<View, 16>(view, C, T, f, sl, g, nb, flip, o, tiled, stats, stream);
    else launch_brick<View, RB_ROWS>(view, C, T, f, sl, g, nb, flip, o, tiled, stats, stream);
}

}  // namespace

uint64_t repair_segments(const Slab& sl) {
    BrickGeom g;
    uint64_t nb, nseg;
    brick_mode(sl, &g, &nb, &nseg);
    return nseg;
}
uint64_t repair_segments_bound(uint64_t n) { return n / 16 + 2; }
uint64_t repair_stage_records(const Slab& sl) {
    BrickGeom g;
    uint64_t nb, nseg;
    if (sl.n == 0 || !brick_mode(sl, &g, &nb, &nseg)) return 0;
    if (MT_REPAIR_SEGSTAGE) return nseg * 16;
    return MT_REPAIR_FIXSTAGE ? nb * uint64_t(RB_NV / 2) : 0;
}
static int diagram_spt(uint64_t nseg) { return nseg >= DG_BIG ? DG_SPT_BIG : 1; }
uint64_t diagram_tiles(uint64_t nseg) {
    const uint64_t per = uint64_t(THREADS) * diagram_spt(nseg);
    return (nseg + per - 1) / per;
}
uint64_t diagram_tiles_bound(uint64_t nseg) { return (nseg + THREADS - 1) / THREADS; }

void launch_repair(const Cell* C, uint64_t* T, const float* f, const Slab& sl, uint32_t flip, const RepairOut& o,
                   bool tiled, unsigned long long* stats, const ForestRef* forest, cudaStream_t stream) {
    if (sl.n == 0) return;
    if (forest) launch_repair_view(ForestView{*forest, sl.base, sl.n}, C, T, f, sl, flip, o, tiled, stats, stream);
    else launch_repair_view(LocalView{}, C, T, f, sl, flip, o, tiled, stats, stream);
}

void launch_diagram(const Slab& sl, const RepairOut& o, void* status, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                    uint64_t ess_cap, cudaStream_t stream) {
    const uint64_t nseg = sl.n ? repair_segments(sl) : 0;
    BrickGeom bg;
    uint64_t bnb, bns;
    const bool seg16 = MT_REPAIR_SEGSTAGE && sl.n && brick_mode(sl, &bg, &bnb, &bns);   // as the repair staged
    const uint64_t ntiles = diagram_tiles(nseg);
    if (ntiles == 0) return;
    if (diagram_spt(nseg) == DG_SPT_BIG)
        diagram_kernel<DG_SPT_BIG><<<uint32_t(ntiles), THREADS, 0, stream>>>(o.seg_cnt, o.seg_pos, nseg, o.stage, o.counters,
                                                                    static_cast<Cell*>(status), out, out_cap, ess,
                                                                    ess_cap, ntiles, seg16);
    else
        diagram_kernel<1><<<uint32_t(ntiles), THREADS, 0, stream>>>(o.seg_cnt, o.seg_pos, nseg, o.stage, o.counters,
                                                                    static_cast<Cell*>(status), out, out_cap, ess,
                                                                    ess_cap, ntiles, seg16);
}

void launch_finish_diagram(unsigned long long* counters, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                           uint64_t ess_cap, cudaStream_t stream) {
    uint64_t blocks = (ess_cap + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    finish_diagram_kernel<<<uint32_t(blocks ? blocks : 1), 256, 0, stream>>>(counters, out, out_cap, ess, ess_cap);
}

}  // namespace mt
