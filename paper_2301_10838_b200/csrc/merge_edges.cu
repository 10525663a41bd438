// merge_edges.cu -- K3: the concurrent edge-merge phase of Alg. 1 (lines 4-8,
// PAPER.md:248-254) with Alg. 3 "Parallel Merge" as an
// iterative loop over 64-bit compare-and-swap (Alg. 2; the
// pair (s, v) packed in one word as in PAPER.md:389-394).
//
// Readings: R4 -- the climbs of Alg. 3 lines 2-8 only follow a
// cell that is not a root (T[x] = (x, x) has nowhere to go; as printed the
// call would recurse on identical arguments forever); R5 -- after a successful
// CAS the displaced pair is merged again (line 15) only if it was not a root;
// R6 -- strict "<" in the climbs as printed, over the (value, id) keys.
//
// Start state: the compressed steepest-descent forest (compress kernel), so
// an edge inside one descent basin is dropped by comparing two basin ids.
//
// Redundant-edge pre-filter (DESIGN.md derivation C'): for the edge (hi, lo)
// at level L = key(hi), follow cells whose saddle key is <= L from both ends
// (Alg. 4's walk at level L on the current store).  If both walks end at the
// same vertex the endpoints are already joined below L, the edge changes no
// sublevel component and is skipped; otherwise Merge(T, r_hi, hi, r_lo) joins
// the two components at level L (the same union Merge(T, hi, hi, lo) performs,
// started after the climbs it would make).  Any cell value ever written is a
// valid triplet, so stale reads only make the filter conservative.
//
// Memory: the 16-byte cells (common.cuh) carry key(s) and the owner's key, so
// no comparison gathers f; they are read with ld.relaxed.gpu.b128 (never a
// stale L1 line) and updated only by atom.cas.b128.
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

struct Stats {
    unsigned long long edges = 0, skipped = 0, pre_hops = 0, iters = 0, cas_fail = 0;
};

// Alg. 4 walk on the current store: last vertex reached from x through cells
// with key(s) <= L (roots stop).  Returns the vertex and leaves its cell in *cx.
// Path halving: when the next cell (s_y, z) is itself followable at the
// level of the current one (key(s_y) <= key(s_x)), x is re-pointed to z with a
// 128-bit CAS.  (s_x, z) is a valid triplet -- x reaches z below key(s_x)
// through y -- and it is exactly the replacement Alg. 5 makes, so the store
// stays a valid normalized store (DESIGN.md derivation E'); a concurrent merge
// that changed x's cell makes the CAS fail and nothing is written.
template <bool STATS>
__device__ __forceinline__ uint32_t climb_le(Cell* C, uint32_t x, uint64_t L, Cell* cx, Stats& st) {
    Cell c = ld_cell(C + x);
    while (cv_of(c) != x && c.lo <= L) {            // not a root and key(s) <= L
        const uint32_t y = cv_of(c);
        const Cell cy = ld_cell(C + y);
        if (STATS) st.pre_hops++;
        if (cv_of(cy) != y && cy.lo <= c.lo) {      // y is passed at x's own level: halve
            const uint32_t z = cv_of(cy);
            cas_cell(C + x, c, Cell{c.lo, (c.hi & 0xffffffff00000000ull) | z});
            x = z;
            c = ld_cell(C + z);
            if (STATS) st.pre_hops++;
        } else {
            x = y;
            c = cy;
        }
    }
    *cx = c;
    return x;
}

// Basin of x in the compressed descent forest: a regular cell (x, x, m)
// points at its basin minimum m (DESIGN.md derivation F); a minimum is its
// own basin.  Regular cells are never CAS targets of the merge phase (every
// CAS hits a vertex reached by a climb from a basin minimum), so this value
// is stable while the kernel runs.
__device__ __forceinline__ uint32_t basin_of(const Cell& c, uint32_t x) {
    return (cs_of(c) == x && cv_of(c) != x) ? cv_of(c) : x;
}

// Alg. 3, iterative.  Joins the components of u and v at level s (key ks).
// cu is the current cell of u (from the pre-filter walk).
template <bool STATS>
__device__ __forceinline__ void merge(Cell* C, uint32_t u, Cell cu, uint64_t ks, uint32_t v, Stats& st) {
    bool have_cu = true;                             // cu is fresh on the first pass only
    while (true) {                                   // every restart re-reads T[u] and T[v]
        if (STATS) st.iters++;
        if (!have_cu) cu = ld_cell(C + u);
        have_cu = false;
        if (cv_of(cu) != u && cu.lo < ks) {          // l.2-4 (+ guard R4): climb u
            u = cv_of(cu);
            continue;
        }
        Cell cv = ld_cell(C + v);
        if (cv_of(cv) != v && cv.lo < ks) {          // l.5-8 (+ guard R4): climb v
            v = cv_of(cv);
            continue;
        }
        if (u == v) return;                          // l.9-10
        if (self_key(cv, v) < self_key(cu, u)) {     // l.11-12: swap the triplets
            const uint32_t t = u; u = v; v = t;
            const Cell tc = cu; cu = cv; cv = tc;
        }
        // l.14: CAS(T[v], (s_v, v'), (s, u)); the owner key of v is unchanged
        const Cell desired = Cell{ks, (cv.hi & 0xffffffff00000000ull) | u};
        const Cell old = cas_cell(C + v, cv, desired);
        if (old.lo == cv.lo && old.hi == cv.hi) {
            const uint32_t vp = cv_of(cv);
            if (vp == v) return;                     // displaced a root (guard R5)
            ks = cv.lo;                              // l.15: Merge(T, u, s_v, v')
            v = vp;
        } else if (STATS) {
            st.cas_fail++;                           // l.17: start again with (u, s, v)
        }
    }
}

template <bool STATS>
__device__ __forceinline__ void merge_edge(Cell* C, uint32_t a, const Cell& ca, uint32_t b, Stats& st) {
    if (STATS) st.edges++;
    const Cell cb = ld_cell(C + b);
    const uint32_t ma = basin_of(ca, a), mb = basin_of(cb, b);
    if (ma == mb) {                                  // same descent basin: joined below both keys
        if (STATS) st.skipped++;
        return;
    }
    const uint64_t ka = self_key(ca, a), kb = self_key(cb, b);
    const uint64_t L = ka > kb ? ka : kb;            // Alg. 1 l.5-8: the edge enters at max(key)
    Cell ch, cl;
    // walks start at the basin minima (the regular cells' single hop is free)
    const uint32_t rh = climb_le<STATS>(C, ka > kb ? ma : mb, L, &ch, st);
    const uint32_t rl = climb_le<STATS>(C, ka > kb ? mb : ma, L, &cl, st);
    if (rh == rl) {                                  // already joined below L
        if (STATS) st.skipped++;
        return;
    }
    merge<STATS>(C, rh, ch, L, rl, st);
}

template <bool STATS>
__global__ void __launch_bounds__(256)
merge_edges_kernel(Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t n, unsigned long long* stats,
                   const unsigned long long* guard, uint64_t guard_cap) {
    // fallback mode: run only if the edge queue overflowed (guard = queue length)
    if (guard && *reinterpret_cast<const volatile unsigned long long*>(guard) <= guard_cap) return;
    const uint64_t sxy = uint64_t(nx) * ny;
    Stats st;
    for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n;
         u += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t x = uint32_t(u % nx);
        const uint64_t yz = u / nx;
        const uint32_t y = uint32_t(yz % ny), z = uint32_t(yz / ny);
        // (re-read per edge: u's own cell changes during the kernel if u is a minimum)
        if (x + 1 < nx) merge_edge<STATS>(C, uint32_t(u), ld_cell(C + u), uint32_t(u + 1), st);
        if (y + 1 < ny) merge_edge<STATS>(C, uint32_t(u), ld_cell(C + u), uint32_t(u + nx), st);
        if (z + 1 < nz) merge_edge<STATS>(C, uint32_t(u), ld_cell(C + u), uint32_t(u + sxy), st);
    }
    if (STATS) {
        atomicAdd(stats + ST_EDGES, st.edges);
        atomicAdd(stats + ST_SKIPPED, st.skipped);
        atomicAdd(stats + ST_PRE_HOPS, st.pre_hops);
        atomicAdd(stats + ST_MERGE_ITERS, st.iters);
        atomicAdd(stats + ST_CAS_FAIL, st.cas_fail);
    }
}

}  // namespace

void launch_merge_edges(Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, int num_sms,
                        unsigned long long* stats, const unsigned long long* guard, uint64_t guard_cap,
                        cudaStream_t stream) {
    const uint64_t n = uint64_t(nx) * ny * nz;
    uint64_t blocks = (n + 255) / 256;
    // grid-stride beyond this; as the overflow fallback (guard) keep the grid small so the
    // common early exit costs one short launch
    const uint64_t cap = uint64_t(num_sms) * 8 * (guard ? 1 : 64);
    if (blocks > cap) blocks = cap;
    if (stats)
        merge_edges_kernel<true><<<uint32_t(blocks), 256, 0, stream>>>(C, nx, ny, nz, n, stats, guard, guard_cap);
    else
        merge_edges_kernel<false><<<uint32_t(blocks), 256, 0, stream>>>(C, nx, ny, nz, n, stats, guard, guard_cap);
}

}  // namespace mt
