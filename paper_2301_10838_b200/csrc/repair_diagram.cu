// repair_diagram.cu -- K4 + K5: the repair phase of Alg. 1 (lines 9-11,
// PAPER.md:255-257; Alg. 5 "Repair", with Alg. 4
// "Representative") fused with the ordered extraction of the
// 0-dimensional persistence diagram (one point (f(a), f(b))
// per branch).
//
// Repair: T[u] = (s, v) becomes (s, Rep(u, key(s))), Rep following cells while
// key(s') <= key(s) and the cell is not a root.  Reading R20: the walk returns
// the vertex it stopped at (Alg. 4 as printed returns the next, too-deep v).
// The walks only read the working cells (the repaired pointer goes to T), so
// they see the fixed post-merge store.
//
// Diagram: after the merge phase the s fields are final (repair only rewrites
// v), so a cell with s != u is the branch born at u dying at saddle s (finite
// pair), and a root (u, u, u) is an essential class.  The
// finite pairs are written in ascending u with a single-pass ordered
// compaction: warp ballots + a CTA scan give each tile's count, published
// BEFORE the tile does its repair walks, and a decoupled look-back over the
// predecessors' published counts gives the tile's output offset.  Tiles take
// dynamic ticket numbers so every predecessor is already resident.
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

// cell / value access for the repair walk: everything local (one GPU), or local
// cells plus the merged boundary forest of all slabs (multi-GPU, slab.cu)
struct LocalView {
    __device__ __forceinline__ Cell cell(const Cell* C, uint32_t x) const { return ld_cell(C + x); }
    __device__ __forceinline__ float value(const float* f, uint32_t x) const { return __ldg(f + x); }
};

struct ForestView {
    ForestRef F;
    uint64_t base, n;  // owned global ids [base, base + n)
    __device__ __forceinline__ bool mine(uint32_t x) const { return uint64_t(x) - base < n; }
    __device__ __forceinline__ Cell cell(const Cell* C, uint32_t x) const {
        if (mine(x)) return ld_cell(C + x);
        const uint32_t i = forest_lookup(F, x);
        if (i == FOREST_MISS) {            // incomplete records: report, stop the walk here
            atomicOr(F.err, ERR_FOREST);
            return Cell{~0ull, x};
        }
        return Cell{F.cells[i].lo, F.cells[i].hi};
    }
    __device__ __forceinline__ float value(const float* f, uint32_t x) const {
        if (mine(x)) return __ldg(f + x);
        uint32_t bits = 0;
        if (!forest_value(F, x, &bits)) atomicOr(F.err, ERR_FOREST);
        return __uint_as_float(bits);
    }
};

constexpr int THREADS = 256;
constexpr int ITEMS = 4;
constexpr int TILE = THREADS * ITEMS;  // 1024 vertices per ticket
constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_VAL = (1ull << 62) - 1;

template <class View>
__global__ void __launch_bounds__(THREADS)
repair_diagram_kernel(View view, Cell* C, uint64_t* __restrict__ T, const float* __restrict__ f, uint64_t base, uint64_t n,
                      uint32_t flip,
                      unsigned long long* __restrict__ counters, uint64_t* __restrict__ status,
                      uint64_t* __restrict__ status_ess,
                      mt_pair* __restrict__ out, uint64_t out_cap, mt_pair* __restrict__ ess, uint64_t ess_cap,
                      uint64_t ntiles, unsigned long long* __restrict__ stats) {
    __shared__ uint64_t s_tile;
    __shared__ uint32_t s_cnt[ITEMS * 8], s_ecnt[ITEMS * 8];
    __shared__ uint64_t s_prefix, s_eprefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(counters + CTR_TICKET, 1ull);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t first = tile * TILE;  // local index of the tile's first vertex

    Cell cell[ITEMS];
    bool fin[ITEMS], root[ITEMS];
    uint32_t mask[ITEMS], emask[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const uint64_t l = first + uint64_t(k) * THREADS + threadIdx.x;
        const uint64_t u = base + l;     // global id (C, T, f are indexed by global id)
        cell[k] = l < n ? ld_cell(C + u) : Cell{0, 0};
        fin[k] = l < n && cs_of(cell[k]) != uint32_t(u);
        root[k] = l < n && cv_of(cell[k]) == uint32_t(u);   // (u, u, u): an essential class
        mask[k] = __ballot_sync(FULL_MASK, fin[k]);
        emask[k] = __ballot_sync(FULL_MASK, root[k]);
        if (lane == 0) {
            s_cnt[k * 8 + warp] = __popc(mask[k]);
            s_ecnt[k * 8 + warp] = __popc(emask[k]);
        }
    }
    __syncthreads();
    // exclusive scans of the 32 (k, warp) counts in u order: finite pairs by
    // warp 0, essential classes by warp 1; each publishes the tile's count
    // before the walks
    if (warp < 2) {
        uint32_t* cnt = warp == 0 ? s_cnt : s_ecnt;
        uint64_t* st = warp == 0 ? status : status_ess;
        const uint32_t c = cnt[lane];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        cnt[lane] = incl - c;
        const uint32_t agg = __shfl_sync(FULL_MASK, incl, 31);
        if (lane == 0) st_relaxed(st + tile, (tile == 0 ? ST_PRE : ST_AGG) | agg);
    }

    // --- repair (Alg. 5 with Alg. 4's walk) ------------------------------
    // The ITEMS walks of a thread advance together, one hop each per round,
    // so up to ITEMS independent cell loads are in flight per thread.
    unsigned long long hops = 0;
    uint32_t x[ITEMS];
    uint32_t active = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const uint64_t l = first + uint64_t(k) * THREADS + threadIdx.x;
        const uint64_t u = base + l;
        x[k] = cv_of(cell[k]);
        if (l >= n) continue;
        if (root[k]) {                                // root (u, u, u): written with the diagram below
            T[u] = pack(uint32_t(u), uint32_t(u));
            continue;
        }
        active |= 1u << k;
    }
    const uint32_t todo = active;
    while (active) {
        Cell c[ITEMS];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
            if (active & (1u << k)) c[k] = view.cell(C, x[k]);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (!(active & (1u << k))) continue;
            if (cv_of(c[k]) == x[k] || c[k].lo > cell[k].lo) {   // root, or key(s_x) > key(s): Rep(u, key(s))
                active &= ~(1u << k);
            } else {
                x[k] = cv_of(c[k]);
                ++hops;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (!(todo & (1u << k))) continue;
        const uint64_t u = base + first + uint64_t(k) * THREADS + threadIdx.x;
        // (no in-place shortcut of the working cell: the 4-B partial write would dirty a
        // 32-B sector per vertex -- ~17 GB of write-back at 1024^3 for walks of ~2.5 hops)
        T[u] = pack(cs_of(cell[k]), x[k]);
    }
    if (stats) atomicAdd(stats + ST_REPAIR_HOPS, hops);

    // --- decoupled look-backs for the tile's output offsets --------------
    __syncthreads();
    if (warp < 2) {
        uint64_t* stat = warp == 0 ? status : status_ess;
        uint64_t prefix = 0;
        int64_t j = int64_t(tile) - 1;
        while (j >= 0) {
            const int64_t idx = j - lane;
            const uint64_t st = idx >= 0 ? ld_relaxed(stat + idx) : ST_PRE;
            const uint64_t flag = st >> 62;
            const uint32_t pmask = __ballot_sync(FULL_MASK, flag == 2);
            const uint32_t xmask = __ballot_sync(FULL_MASK, flag == 0);
            const int first_p = pmask ? __ffs(pmask) - 1 : 31;
            const uint32_t upto = first_p == 31 ? FULL_MASK : ((2u << first_p) - 1u);
            if (xmask & upto) continue;               // a needed predecessor has not published
            uint64_t val = lane <= first_p ? (st & ST_VAL) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL_MASK, val, o);
            prefix += val;
            if (pmask) break;
            j -= 32;
        }
        if (lane == 0) (warp == 0 ? s_prefix : s_eprefix) = prefix;
    }
    __syncthreads();
    const uint64_t prefix = s_prefix, eprefix = s_eprefix;
    // inclusive prefix = prefix + this tile's aggregate; s_cnt holds exclusive
    // offsets, so the aggregate is the last offset + the last (k, warp) count,
    // which the last thread's own ballot holds.
    if (threadIdx.x == THREADS - 1) {
        const uint64_t total = prefix + s_cnt[(ITEMS - 1) * 8 + 7] + __popc(mask[ITEMS - 1]);
        const uint64_t etotal = eprefix + s_ecnt[(ITEMS - 1) * 8 + 7] + __popc(emask[ITEMS - 1]);
        if (tile != 0) {
            st_relaxed(status + tile, ST_PRE | total);
            st_relaxed(status_ess + tile, ST_PRE | etotal);
        }
        if (tile == ntiles - 1) {
            counters[CTR_FIN] = total;
            counters[CTR_ESS] = etotal;
        }
    }

    // --- essential classes in ascending u (into the essential buffer) ------
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (!root[k]) continue;
        const uint64_t u = base + first + uint64_t(k) * THREADS + threadIdx.x;
        const uint64_t pos = eprefix + s_ecnt[k * 8 + warp] + __popc(emask[k] & ((1u << lane) - 1u));
        if (pos < ess_cap) ess[pos] = mt_pair{uint32_t(u), uint32_t(u), __ldg(f + u), __int_as_float(0x7f800000)};
        else atomicOr(counters + CTR_ERR, ERR_ESS_CAPACITY);
    }

    // --- write this tile's finite pairs in ascending u --------------------
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (!fin[k]) continue;
        const uint64_t u = base + first + uint64_t(k) * THREADS + threadIdx.x;
        const uint64_t pos = prefix + s_cnt[k * 8 + warp] + __popc(mask[k] & ((1u << lane) - 1u));
        const uint32_t s = cs_of(cell[k]);
        // death value f[s]: the cell carries ord(f[s]); invert it (exact for every value but
        // zero, whose sign the canonicalisation -0 -> +0 dropped: gather those, reading R14)
        const uint32_t o = uint32_t(cell[k].lo >> 32) ^ flip;
        const uint32_t bits = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
        const float death = bits == 0u ? view.value(f, s) : __uint_as_float(bits);
        if (pos < out_cap) out[pos] = mt_pair{uint32_t(u), s, __ldg(f + u), death};
        else atomicOr(counters + CTR_ERR, ERR_CAPACITY);
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

}  // namespace

uint64_t repair_tiles(uint64_t n) { return (n + TILE - 1) / TILE; }

void launch_repair_diagram(Cell* C, uint64_t* T, const float* f, uint64_t base, uint64_t n, uint32_t flip,
                           unsigned long long* counters,
                           uint64_t* status, uint64_t* status_ess, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                           uint64_t ess_cap,
                           unsigned long long* stats, const ForestRef* forest, cudaStream_t stream) {
    const uint64_t ntiles = repair_tiles(n);
    if (ntiles == 0) return;
    if (forest)
        repair_diagram_kernel<<<uint32_t(ntiles), THREADS, 0, stream>>>(ForestView{*forest, base, n}, C, T, f, base, n, flip,
                                                                         counters, status, status_ess, out, out_cap,
                                                                         ess, ess_cap,
                                                                         ntiles, stats);
    else
        repair_diagram_kernel<<<uint32_t(ntiles), THREADS, 0, stream>>>(LocalView{}, C, T, f, base, n, flip, counters,
                                                                         status, status_ess, out, out_cap, ess,
                                                                         ess_cap, ntiles,
                                                                         stats);
}

void launch_finish_diagram(unsigned long long* counters, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                           uint64_t ess_cap, cudaStream_t stream) {
    uint64_t blocks = (ess_cap + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    finish_diagram_kernel<<<uint32_t(blocks ? blocks : 1), 256, 0, stream>>>(counters, out, out_cap, ess, ess_cap);
}

}  // namespace mt
