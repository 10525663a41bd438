// merge_cross.cu -- K3 on the global store: merge the grid edges that cross a
// tile face (the in-tile edges were merged by tile_tmt.cu) with Alg. 3
// "Parallel Merge" over 128-bit CAS cells.  Two kernels:
//
// dedupe_cross: the crossing edges are enumerated directly (e in
// [0, Ex + Ey + Ez) decodes to an x-, y- or z-face edge; 32 consecutive e are
// neighbours on one face, one per lane).  Each edge is reduced to the pair of
// tile representatives of its ends at their own levels (tile_tmt's R array,
// DESIGN.md derivation C''') and its level L = max(key(a), key(b)); lanes
// holding the same pair (__match_any_sync) keep only the lowest edge
// (derivation C''), and the survivors are queued as (L, R_hi, R_lo).  On
// grids whose faces tile into 32 x 16 patches (nx % 32 = ny % 16 = nz % 16 =
// 0) the faces are enumerated patch by patch instead (z, then y, then x
// faces), one patch per CTA step of 512 threads, and the dedupe is CTA-wide:
// a shared-memory table pair -> lowest level (CAS + 64-bit atomicMin) over the
// 16 rows of the patch (a whole tile z face).
//
// merge_queue: persistent warps take batches of 256 queue entries per global
// atomic; each lane runs its entry as a state machine advanced by ONE memory
// round-trip per step (a cell load, a pair of independent cell loads, or a
// CAS), and idle lanes are refilled at every step, so a warp stays converged
// and keeps up to 32 independent loads in flight (a per-thread nested-loop
// version left 2.5 active lanes per instruction, ncu profiles/r1_c4_ncu_v1.md).
//
// Each lane runs its edge as a state machine advanced by ONE memory
// round-trip per step (a cell load, a pair of independent cell loads, or a
// CAS), and idle lanes are refilled at every step, so a warp stays converged
// and keeps up to 32 independent loads in flight (a per-thread nested-loop
// version left 2.5 active lanes per instruction, ncu profiles/r1_c4_ncu_v1.md).
//
// Per entry: both basins (joined to the edge's ends below their own keys) are
// walked through cells with key(s) <= L (Alg. 4's walk at level L, with path
// splitting by 128-bit CAS, derivation E'); if the walks meet, the edge joins
// nothing new (derivation C'); otherwise Merge(T, r_hi, hi, r_lo) runs: climbs
// with the root guard R4, the swap of l.11-12, the CAS of l.14, the
// re-merge of a displaced non-root pair (l.15, guard R5), restarts (l.17)
// that re-read both cells.
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

#ifndef DC_XFACE
#define DC_XFACE 1        // x-face edges read tile_tmt's compact face records
#endif
#ifndef DC_ROWS
#define DC_ROWS 16        // patch rows (a CTA step = 32 x DC_ROWS face edges = DC_THREADS threads)
#endif
#define DC_THREADS (32 * DC_ROWS)
#define DC_LOG2T (DC_ROWS == 16 ? 10 : 9)   // log2 of the 2 x DC_THREADS table slots
#ifndef DC_PATCH
#define DC_PATCH 1        // z faces in 32 x 8 patches with a CTA-wide dedupe
#endif
#ifndef DC_YPATCH
#define DC_YPATCH 1       // the y faces in 32 x 8 patches too
#endif
#ifndef DC_PATCH_ONLY
#define DC_PATCH_ONLY 1   // patch steps: skip the warp dedupe (the CTA-wide one does it all)
#endif
#ifndef DC_XPATCH
#define DC_XPATCH 1       // the x faces in 32 (y) x 8 (z) patches too
#endif
#ifndef DC_NDEDUP
#define DC_NDEDUP 1       // patch steps: drop edges whose neighbour lane has the same pair lower
#endif
#ifndef DC_STEPQ
#define DC_STEPQ 0        // stepped crossing-edge queue: survivors at their step's own positions + a count per step (measured slower)
#endif
#ifndef DC_MIN32
#define DC_MIN32 1        // patch table: the lowest level by two native 32-bit minima (order key, id)
#endif
#ifndef DC_REDUCE
#define DC_REDUCE 0       // group minimum by two __reduce_min_sync (else a 32-lane shuffle scan)
#endif
#ifndef DC_MATCH
#define DC_MATCH 1        // dedupe_cross: whole-warp groups by __match_any_sync (else neighbour lanes)
#endif

struct CrossGeom {
    uint32_t nx, ny, nz, tx, ty, tz;   // slab (nz = local planes) and tile shape
    uint32_t tiles_x, tiles_y;         // tiles along x and y
    uint32_t patch;                    // DC_PATCH: z faces first, in 32 x 8 patches (one per CTA step)
    uint32_t ypatch;                   // ... then the y faces in 32 (x) x 8 (z) patches
    uint32_t xpatch;                   // ... then the x faces in 32 (y) x 8 (z) patches
    uint64_t base;                     // global id of the slab's first vertex
    uint64_t ex, ey, ez;               // number of crossing edges on x-, y-, z-faces
};

__device__ __forceinline__ void decode_edge(const CrossGeom& g, uint64_t e, uint32_t* a, uint32_t* b) {
    // every face count and every per-boundary count is below n < 2^32, so the index
    // arithmetic inside a face runs in 32 bits (64-bit division is ~4x the instructions)
    const uint64_t sxy = uint64_t(g.nx) * g.ny;
    uint64_t u, step;
    if (e < g.ex) {                               // x-face k: x = (k+1) tx - 1 -> +1
        const uint32_t ee = uint32_t(e), per = g.ny * g.nz;
        const uint32_t k = ee / per, r = ee - k * per;
        const uint32_t z = r / g.ny, y = r - z * g.ny;
        u = z * sxy + uint64_t(y) * g.nx + uint64_t(k + 1) * g.tx - 1;
        step = 1;
    } else if ((e -= g.ex) < g.ey) {              // y-face k: y = (k+1) ty - 1 -> +nx
        const uint32_t ee = uint32_t(e), per = g.nx * g.nz;
        const uint32_t k = ee / per, r = ee - k * per;
        const uint32_t z = r / g.nx, x = r - z * g.nx;
        u = z * sxy + (uint64_t(k + 1) * g.ty - 1) * g.nx + x;
        step = g.nx;
    } else {                                      // z-face k: z = (k+1) tz - 1 -> +nx ny
        e -= g.ey;
        const uint32_t ee = uint32_t(e), per = uint32_t(sxy);
        const uint32_t k = ee / per, r = ee - k * per;
        u = (uint64_t(k + 1) * g.tz - 1) * sxy + r;
        step = sxy;
    }
    *a = uint32_t(g.base + u);        // global ids
    *b = uint32_t(g.base + u + step);
}

struct QEntry {
    uint64_t L;      // key of the edge's upper endpoint (the merge level)
    uint32_t m_hi;   // descent basin of the upper endpoint
    uint32_t m_lo;   // descent basin of the lower endpoint
};

__global__ void __launch_bounds__(DC_THREADS)
dedupe_cross_kernel(const float* __restrict__ f, const uint64_t* __restrict__ T0,
                    const uint64_t* __restrict__ xface, CrossGeom g, uint32_t flip,
                    QEntry* __restrict__ q, uint64_t cap, unsigned long long* __restrict__ qlen,
                    uint32_t* __restrict__ qcnt, unsigned long long* __restrict__ stats) {
    __shared__ uint32_t s_warp[DC_THREADS / 32];
    __shared__ unsigned long long s_base;
    __shared__ unsigned long long s_key[2 * DC_THREADS];   // DC_PATCH: pair -> lowest level
#if DC_MIN32
    __shared__ uint32_t s_mo[2 * DC_THREADS], s_mi[2 * DC_THREADS];   // its order key, then its id
#else
    __shared__ unsigned long long s_min[2 * DC_THREADS];
#endif
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t total = g.ex + g.ey + g.ez;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    unsigned long long n_edges = 0;
    for (uint64_t e0 = uint64_t(blockIdx.x) * blockDim.x; e0 < total; e0 += stride) {
        const uint64_t e_raw = e0 + threadIdx.x;
        const bool valid = e_raw < total;
        QEntry en{0, 0, 0};
        uint64_t pair = ~0ull;
        // DC_PATCH order: the z faces first, each CTA step one 32 x 8 patch of a z face (so the
        // CTA dedupe below sees 8 rows of one tile face), then the x and the y faces
        const uint64_t yend = g.ez + (g.ypatch ? g.ey : 0);
        const uint64_t xend = yend + (g.xpatch ? g.ex : 0);
        const bool zpatch = g.patch && e0 < xend;   // uniform over the CTA (ez, ey, ex % DC_THREADS == 0)
        uint64_t e = e_raw;
        // patch steps know their edge's face, plane and position directly: the ends a, b (and,
        // for an x face, its record's tile and row) without decode_edge's divisions.  A step's
        // 512 edges lie in one patch (every face size is a multiple of 512), so k and the patch
        // index derive from the CTA-uniform e0.
        bool direct = false;
        uint32_t a = 0, b = 0, xk = 0, xy = 0, xz = 0;
        bool xrec = false;
        if (g.patch) {
            const uint32_t pxn = g.nx / 32, w = threadIdx.x;
            const uint64_t sxy = uint64_t(g.nx) * g.ny;
            if (e0 < g.ez) {
                const uint64_t k = e0 / sxy;
                const uint32_t pidx = uint32_t((e0 - k * sxy) / DC_THREADS);
                const uint32_t x = (pidx % pxn) * 32 + (w & 31), y = (pidx / pxn) * DC_ROWS + (w >> 5);
                const uint64_t u = (uint64_t(k + 1) * g.tz - 1) * sxy + uint64_t(y) * g.nx + x;
                a = uint32_t(g.base + u);
                b = uint32_t(g.base + u + sxy);
                direct = true;
            } else if (e0 < yend) {
                const uint64_t sxz = uint64_t(g.nx) * g.nz, ey0 = e0 - g.ez;
                const uint64_t k = ey0 / sxz;
                const uint32_t pidx = uint32_t((ey0 - k * sxz) / DC_THREADS);
                const uint32_t x = (pidx % pxn) * 32 + (w & 31), z = (pidx / pxn) * DC_ROWS + (w >> 5);
                const uint64_t u = uint64_t(z) * sxy + (uint64_t(k + 1) * g.ty - 1) * g.nx + x;
                a = uint32_t(g.base + u);
                b = uint32_t(g.base + u + g.nx);
                direct = true;
            } else if (e0 < xend) {
                const uint64_t syz = uint64_t(g.ny) * g.nz, ex0 = e0 - yend;
                const uint64_t k = ex0 / syz;
                const uint32_t pidx = uint32_t((ex0 - k * syz) / DC_THREADS), pyn = g.ny / 32;
                const uint32_t y = (pidx % pyn) * 32 + (w & 31), z = (pidx / pyn) * DC_ROWS + (w >> 5);
                const uint64_t u = uint64_t(z) * sxy + uint64_t(y) * g.nx + (uint64_t(k + 1) * g.tx - 1);
                a = uint32_t(g.base + u);
                b = uint32_t(g.base + u + 1);
                xk = uint32_t(k);
                xy = y;
                xz = z;
                xrec = DC_XFACE;
                direct = true;
            } else if (g.ypatch) {
                e = e_raw - yend;                    // the x faces, in their own order
            } else {
                e = e_raw - g.ez;                    // x faces, then y faces
            }
        }
        if (valid) {
            if (!direct) {
                decode_edge(g, e, &a, &b);
                if (DC_XFACE && e < g.ex) {
                    const uint32_t ee = uint32_t(e), per = g.ny * g.nz;
                    xk = ee / per;
                    const uint32_t rr = ee - xk * per;
                    xz = rr / g.ny;
                    xy = rr - xz * g.ny;
                    xrec = true;
                }
            }
            uint64_t ka, kb;
            uint32_t ba, bb;
            if (xrec) {
                // x-face edge: both ends from tile_tmt's compact face records (order key, R)
                // -- in the grid they sit 128 B apart, one line per lane
                const uint32_t rows = g.ty * g.tz, row = (xz % g.tz) * g.ty + xy % g.ty;
                const uint64_t t = xk + uint64_t(g.tiles_x) * (xy / g.ty + uint64_t(g.tiles_y) * (xz / g.tz));
                const uint64_t ea = __ldg(xface + (t * 2 + 1) * rows + row);        // right face of tile k
                const uint64_t eb = __ldg(xface + ((t + 1) * 2) * rows + row);      // left face of tile k + 1
                ka = key_of(uint32_t(ea >> 32), a);
                kb = key_of(uint32_t(eb >> 32), b);
                ba = uint32_t(ea);
                bb = uint32_t(eb);
            } else {
                // the tile store holds each vertex's order key and its tile representative at its
                // own level (DESIGN.md derivation C-3): ord(u) << 32 | R(u)
                const uint64_t ta = __ldg(reinterpret_cast<const unsigned long long*>(T0 + a));
                const uint64_t tb = __ldg(reinterpret_cast<const unsigned long long*>(T0 + b));
                ka = key_of(uint32_t(ta >> 32), a);
                kb = key_of(uint32_t(tb >> 32), b);
                ba = uint32_t(ta);
                bb = uint32_t(tb);
            }
            en = ka > kb ? QEntry{ka, ba, bb} : QEntry{kb, bb, ba};
            pair = ba < bb ? (uint64_t(ba) << 32 | bb) : (uint64_t(bb) << 32 | ba);
            ++n_edges;
        }
        // lanes with the same pair keep the lowest edge only
        bool keep = valid;
#if DC_MATCH
        if (!(DC_PATCH_ONLY && zpatch)) {   // (patch steps: the CTA-wide dedupe alone)
        const uint32_t group = __match_any_sync(FULL_MASK, pair);
#if DC_REDUCE
        {   // lowest L = (ord << 32 | id) of the group: min of the order keys, then of the ids
            const uint32_t o = uint32_t(en.L >> 32), id = uint32_t(en.L);
            const uint32_t m1 = __reduce_min_sync(group, o);
            const uint32_t tie = group & __ballot_sync(FULL_MASK, o == m1);
            if (o != m1) keep = false;
            else if (id != __reduce_min_sync(tie, id)) keep = false;
        }
#else
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
            const uint64_t Lj = __shfl_sync(FULL_MASK, en.L, j);
            if (((group >> j) & 1u) && Lj < en.L) keep = false;
        }
#endif
        }
#else
        {   // (cheaper) neighbouring lanes only: an edge with a lower one of the same pair in the
            // previous or next lane is dropped; the lowest of every run of lanes survives
            const uint64_t pu = __shfl_up_sync(FULL_MASK, pair, 1), pd = __shfl_down_sync(FULL_MASK, pair, 1);
            const uint64_t lu = __shfl_up_sync(FULL_MASK, en.L, 1), ld = __shfl_down_sync(FULL_MASK, en.L, 1);
            if ((lane > 0 && pu == pair && lu < en.L) || (lane < 31 && pd == pair && ld < en.L)) keep = false;
        }
#endif
#if DC_NDEDUP
        if (zpatch) {
            // neighbouring lanes of a patch hold neighbouring edges of one face, mostly between the
            // same two tile representatives: an edge with a lower one of its pair in the next or
            // previous lane is dropped before the CTA table (derivation C''; upper ends differ, so
            // levels never tie)
            const uint64_t pu = __shfl_up_sync(FULL_MASK, pair, 1), pd = __shfl_down_sync(FULL_MASK, pair, 1);
            const uint64_t lu = __shfl_up_sync(FULL_MASK, en.L, 1), ld = __shfl_down_sync(FULL_MASK, en.L, 1);
            if (keep && ((lane > 0 && pu == pair && lu < en.L) || (lane < 31 && pd == pair && ld < en.L)))
                keep = false;
        }
#endif
        if (DC_PATCH && zpatch) {
            // CTA-wide: the warps' survivors keep the lowest edge of each pair over the patch
            s_key[threadIdx.x] = ~0ull;
            s_key[threadIdx.x + DC_THREADS] = ~0ull;
#if DC_MIN32
            s_mo[threadIdx.x] = ~0u;
            s_mo[threadIdx.x + DC_THREADS] = ~0u;
            s_mi[threadIdx.x] = ~0u;
            s_mi[threadIdx.x + DC_THREADS] = ~0u;
#else
            s_min[threadIdx.x] = ~0ull;
            s_min[threadIdx.x + DC_THREADS] = ~0ull;
#endif
            __syncthreads();
            uint32_t h = 0;
            if (keep) {
                h = uint32_t((pair * 0x9E3779B97F4A7C15ull) >> (64 - DC_LOG2T));
                while (true) {
                    const unsigned long long k = atomicCAS(&s_key[h], ~0ull, pair);
                    if (k == ~0ull || k == pair) break;
                    h = (h + 1) & (2u * DC_THREADS - 1u);
                }
#if DC_MIN32
                atomicMin(&s_mo[h], uint32_t(en.L >> 32));   // (native 32-bit minima: no CAS loop)
#else
                atomicMin(&s_min[h], (unsigned long long)en.L);
#endif
            }
            __syncthreads();
#if DC_MIN32
            // the lowest order key first, then the lowest id among the edges that have it
            if (keep && s_mo[h] != uint32_t(en.L >> 32)) keep = false;
            if (keep) atomicMin(&s_mi[h], uint32_t(en.L));
            __syncthreads();
            if (keep && s_mi[h] != uint32_t(en.L)) keep = false;
#else
            if (keep && s_min[h] != en.L) keep = false;
#endif
        }
        const uint32_t km = __ballot_sync(FULL_MASK, keep);
        if (lane == 0) s_warp[warp] = __popc(km);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < DC_THREADS / 32; ++w) {
                const uint32_t t = s_warp[w];
                s_warp[w] = tot;
                tot += t;
            }
            if (qcnt) {
                // stepped queue: this step's survivors at its own edge positions [e0, e0 + tot)
                // and their count -- no global atomic (merge_queue reads step by step)
                qcnt[e0 / DC_THREADS] = tot;
                s_base = e0;
            } else {
                s_base = tot ? atomicAdd(qlen, (unsigned long long)tot) : 0;
            }
        }
        __syncthreads();
        const uint64_t pos = s_base + s_warp[warp] + __popc(km & ((1u << lane) - 1u));
        if (keep && pos < cap) q[pos] = en;
        __syncthreads();  // s_warp / s_base are rewritten next iteration
    }
    if (stats) atomicAdd(stats + ST_EDGES, n_edges);
}

#ifndef MQ_SPLIT
#define MQ_SPLIT 1        // merge_queue walks: 1 path splitting, 2 path halving (128-bit CAS), 0 none
#endif
#ifndef MQ_BOTHCLIMB
#define MQ_BOTHCLIMB 1    // Alg. 3 step: climb u and v in the same round trip when both can climb
#endif
#ifndef MQ_WALK
#define MQ_WALK 0         // filter walks (with path splitting) before Alg. 3 (measured slower than MQ_CSPLIT)
#endif
#ifndef MQ_CSPLIT
#define MQ_CSPLIT 1       // path splitting inside the Alg. 3 climbs (with MQ_WALK 0)
#endif
#ifndef MQ_BATCH
#define MQ_BATCH 256      // queue entries a warp takes per fetch (one global atomic each)
#endif
#ifndef MQ_MIN_BLOCKS
#define MQ_MIN_BLOCKS 4   // 4 x 256 threads per SM: <= 64 registers (the climbs keep their previous cells), 32 warps of loads in flight
#endif

enum Phase : int { IDLE = 0, CLIMB_HI = 2, CLIMB_LO = 3, MERGE_LD = 4, MERGE_CAS = 5, DONE = 6 };

template <bool STATS>
__global__ void __launch_bounds__(256, MQ_MIN_BLOCKS)
merge_queue_kernel(Cell* C, const QEntry* __restrict__ q, uint64_t cap, const unsigned long long* __restrict__ qlen,
                   const uint32_t* __restrict__ qcnt, uint64_t nsteps, unsigned long long* __restrict__ fetch,
                   unsigned long long* __restrict__ stats) {
    constexpr uint64_t BATCH = MQ_BATCH;
    constexpr uint64_t STEP = DC_THREADS;   // stepped queue: entries per dedupe_cross step
    const int lane = threadIdx.x & 31;
    const uint64_t qn = *reinterpret_cast<const volatile unsigned long long*>(qlen);
    const uint64_t total = qn < cap ? qn : cap;
    uint64_t pool_next = 0, pool_end = 0;  // warp-uniform
    bool exhausted = false;                // warp-uniform

    // The state that lives from one round trip to the next, shared between the phases (the
    // phases are exclusive, so one set of registers serves all of them):
    //   climbs (CLIMB_HI / CLIMB_LO): lev = L, p0 = x (walk position), p1 = xp (previous cell),
    //     p2 = lo (the other end's representative), p3 = rh (where the first walk stopped),
    //     held = the previous cell's value (path splitting);
    //   Alg. 3 (MERGE_LD / MERGE_CAS): lev = S, p0 = u, p1 = v, held = T[v] as loaded (the
    //     expected value of the CAS; the desired value is rebuilt from it).
    int phase = IDLE;
    uint64_t lev = 0;
    uint32_t p0 = 0, p1 = 0, p2 = 0, p3 = 0;
    bool has_prev = false;
    Cell held{0, 0};
    // MQ_CSPLIT: the previous cell of each Alg. 3 climb (path splitting)
    [[maybe_unused]] Cell hu{0, 0}, hv{0, 0};
    [[maybe_unused]] uint32_t xu = 0, xv = 0;
    [[maybe_unused]] bool has_u = false, has_v = false;
    unsigned long long n_edges = 0, n_hops = 0, n_iters = 0, n_fail = 0, n_skip = 0;

    while (true) {
        const uint32_t need = __ballot_sync(FULL_MASK, phase == IDLE);
        if (need) {
            if (qcnt) {
                // stepped queue (dedupe_cross): one step's survivors at a time, empty steps skipped
                while (pool_next == pool_end && !exhausted) {
                    unsigned long long st = 0;
                    if (lane == 0) st = atomicAdd(fetch, 1ull);
                    st = __shfl_sync(FULL_MASK, st, 0);
                    if (st >= nsteps) {
                        exhausted = true;
                    } else {
                        const uint32_t c = qcnt[st];
                        pool_next = st * STEP;
                        pool_end = pool_next + (c < STEP ? c : STEP);
                    }
                }
            } else if (pool_next == pool_end && !exhausted) {
                unsigned long long b0 = 0;
                if (lane == 0) b0 = atomicAdd(fetch, (unsigned long long)BATCH);
                b0 = __shfl_sync(FULL_MASK, b0, 0);
                pool_next = b0 < total ? b0 : total;
                pool_end = b0 + BATCH < total ? b0 + BATCH : total;
                exhausted = pool_next == pool_end;
            }
            const uint32_t rank = __popc(need & ((1u << lane) - 1u));
            const uint64_t avail = pool_end - pool_next;
            if (phase == IDLE) {
                if (rank < avail) {
                    const QEntry en = q[pool_next + rank];
                    lev = en.L;
                    p0 = en.m_hi;                     // walk the upper end's basin first
                    p2 = en.m_lo;
                    has_prev = false;
                    phase = CLIMB_HI;
                    if (!MQ_WALK) {                   // Merge(T, R_hi, hi, R_lo) straight away
                        p1 = en.m_lo;
                        phase = MERGE_LD;
                        has_u = has_v = false;
                    }
                    if (STATS) n_edges++;
                } else if (exhausted) {
                    phase = DONE;
                }
            }
            pool_next += avail < __popc(need) ? avail : __popc(need);
        }
        if (__ballot_sync(FULL_MASK, phase != DONE) == 0) break;

        // ---- one memory round-trip, then advance ----
        if (phase == CLIMB_HI || phase == CLIMB_LO) {
            const Cell c = ld_cell(C + p0);
            if (cv_of(c) != p0 && c.lo <= lev) {       // followable at level L
                if (STATS) n_hops++;
                const bool split = MQ_SPLIT && has_prev && c.lo <= held.lo;
                if (split)                                 // path splitting: prev skips x
                    cas_cell(C + p1, held, Cell{held.lo, (held.hi & 0xffffffff00000000ull) | cv_of(c)});
                if (MQ_SPLIT == 2 && split) {
                    has_prev = false;                      // path halving: every other cell
                } else {
                    p1 = p0;
                    held = c;
                    has_prev = true;
                }
                p0 = cv_of(c);
            } else if (phase == CLIMB_HI) {
                p3 = p0;
                p0 = p2;
                has_prev = false;
                phase = CLIMB_LO;
            } else if (p0 == p3) {                     // walks met: nothing to join
                if (STATS) n_skip++;
                phase = IDLE;
            } else {
                p1 = p0;                               // Merge(T, r_hi, hi, r_lo) at level L
                p0 = p3;
                phase = MERGE_LD;
            }
        } else if (phase == MERGE_LD) {
            Cell cu = ld_cell(C + p0), cv = ld_cell(C + p1);
            if (STATS) n_iters++;
            const bool up_u = cv_of(cu) != p0 && cu.lo < lev;   // l.2-4 (+ R4)
            const bool up_v = cv_of(cv) != p1 && cv.lo < lev;   // l.5-8 (+ R4)
            if (MQ_CSPLIT && (up_u || up_v)) {
                // both climbs advance, each splitting its path: the cell climbed from before
                // (x -> y) is re-pointed past y when y's saddle is not above x's (x then joins
                // v(y) at its own level; any value a cell holds stays a valid triplet), so the
                // repair later walks shorter chains
                if (up_u) {
                    if (has_u && cu.lo <= hu.lo)
                        cas_cell(C + xu, hu, Cell{hu.lo, (hu.hi & 0xffffffff00000000ull) | cv_of(cu)});
                    xu = p0;
                    hu = cu;
                    has_u = true;
                    p0 = cv_of(cu);
                }
                if (up_v) {
                    if (has_v && cv.lo <= hv.lo)
                        cas_cell(C + xv, hv, Cell{hv.lo, (hv.hi & 0xffffffff00000000ull) | cv_of(cv)});
                    xv = p1;
                    hv = cv;
                    has_v = true;
                    p1 = cv_of(cv);
                }
            } else if (MQ_BOTHCLIMB && (up_u || up_v)) {        // independent climbs: both advance
                if (up_u) p0 = cv_of(cu);
                if (up_v) p1 = cv_of(cv);
            } else if (up_u) {                         // climb u, restart
                p0 = cv_of(cu);
            } else if (up_v) {                         // climb v, restart
                p1 = cv_of(cv);
            } else if (p0 == p1) {                     // l.9-10
                phase = IDLE;
            } else {
                if (self_key(cv, p1) < self_key(cu, p0)) {   // l.11-12: swap
                    const uint32_t t = p0; p0 = p1; p1 = t;
                    cv = cu;
                }
                held = cv;                             // l.14: (s, u) into T[v], next round trip
                phase = MERGE_CAS;
                has_u = has_v = false;                 // (the climbs start afresh after the CAS)
            }
        } else if (phase == MERGE_CAS) {
            const Cell got = cas_cell(C + p1, held, Cell{lev, (held.hi & 0xffffffff00000000ull) | p0});
            if (got.lo == held.lo && got.hi == held.hi) {
                const uint32_t vp = cv_of(held);
                if (vp == p1) {
                    phase = IDLE;                      // displaced a root (R5)
                } else {
                    lev = held.lo;                     // l.15: Merge(T, u, s_v, v')
                    p1 = vp;
                    phase = MERGE_LD;
                }
            } else {
                if (STATS) n_fail++;
                phase = MERGE_LD;                      // l.17: restart
            }
        }
    }
    if (STATS) {
        atomicAdd(stats + ST_QUEUED, n_edges);
        atomicAdd(stats + ST_PRE_HOPS, n_hops);
        atomicAdd(stats + ST_MERGE_ITERS, n_iters);
        atomicAdd(stats + ST_CAS_FAIL, n_fail);
        atomicAdd(stats + ST_SKIPPED, n_skip);
    }
}

}  // namespace

int launch_dedupe_cross(const float* f, const uint64_t* T0, const uint64_t* xface, const Slab& sl, uint32_t flip,
                        void* queue,
                        uint64_t cap, unsigned long long* qlen, uint32_t* qcnt, unsigned long long* stats,
                        int num_sms, cudaStream_t stream) {
    CrossGeom g{};
    g.nx = sl.nx;
    g.ny = sl.ny;
    g.nz = sl.z_end - sl.z_begin;
    g.base = sl.base;
    g.tx = 32;
    tile_shape(sl.nz, &g.ty, &g.tz);
    g.tiles_x = (g.nx + g.tx - 1) / g.tx;
    g.tiles_y = (g.ny + g.ty - 1) / g.ty;
    g.patch = DC_PATCH && g.nx % 32 == 0 && g.ny % DC_ROWS == 0 ? 1u : 0u;
    g.ypatch = g.patch && DC_YPATCH && g.nz % DC_ROWS == 0 ? 1u : 0u;
    g.xpatch = g.ypatch && DC_XPATCH && g.ny % 32 == 0 ? 1u : 0u;
    const uint64_t kx = (g.nx + g.tx - 1) / g.tx - 1, ky = (g.ny + g.ty - 1) / g.ty - 1,
                   kz = g.nz ? (g.nz + g.tz - 1) / g.tz - 1 : 0;
    g.ex = g.nz ? kx * g.ny * g.nz : 0;
    g.ey = g.nz ? ky * g.nx * g.nz : 0;
    g.ez = kz * uint64_t(g.nx) * g.ny;
    const uint64_t total = cross_edges(sl);
    if (total == 0) return 0;
    QEntry* q = static_cast<QEntry*>(queue);
    uint64_t blocks = (total + DC_THREADS - 1) / DC_THREADS;
    if (blocks > uint64_t(num_sms) * 32) blocks = uint64_t(num_sms) * 32;
    dedupe_cross_kernel<<<uint32_t(blocks), DC_THREADS, 0, stream>>>(f, T0, xface, g, flip, q, cap, qlen,
                                                                      DC_STEPQ ? qcnt : nullptr, stats);
    return 1;
}

static_assert(DC_THREADS >= 128, "the workspace sizes the stepped queue's counts for steps of >= 128 edges");
uint64_t cross_steps(const Slab& sl) { return (cross_edges(sl) + DC_THREADS - 1) / DC_THREADS; }
bool cross_stepped() { return DC_STEPQ != 0; }

void launch_merge_queue(Cell* C, const void* queue, uint64_t cap, const unsigned long long* qlen,
                        const uint32_t* qcnt, uint64_t nsteps,
                        unsigned long long* fetch, unsigned long long* stats, int num_sms, cudaStream_t stream) {
    const QEntry* q = static_cast<const QEntry*>(queue);
    // persistent grid: as many CTAs as fit on every SM of this device
    const int per_sm = stats ? occupancy_per_sm(reinterpret_cast<const void*>(merge_queue_kernel<true>), 256, 0)
                             : occupancy_per_sm(reinterpret_cast<const void*>(merge_queue_kernel<false>), 256, 0);
    const uint32_t pblocks = uint32_t(num_sms) * per_sm;
    if (stats)
        merge_queue_kernel<true><<<pblocks, 256, 0, stream>>>(C, q, cap, qlen, qcnt, nsteps, fetch, stats);
    else
        merge_queue_kernel<false><<<pblocks, 256, 0, stream>>>(C, q, cap, qlen, qcnt, nsteps, fetch, stats);
}

uint64_t cross_edges(const Slab& sl) {
    uint32_t ty, tz;
    tile_shape(sl.nz, &ty, &tz);
    const uint64_t nzl = sl.z_end - sl.z_begin;
    if (!nzl || !sl.nx || !sl.ny) return 0;
    const uint64_t kx = (sl.nx + 31) / 32 - 1, ky = (sl.ny + ty - 1) / ty - 1, kz = (nzl + tz - 1) / tz - 1;
    return kx * sl.ny * nzl + ky * uint64_t(sl.nx) * nzl + kz * uint64_t(sl.nx) * sl.ny;
}

size_t cross_queue_entry_bytes() { return sizeof(QEntry); }

}  // namespace mt
