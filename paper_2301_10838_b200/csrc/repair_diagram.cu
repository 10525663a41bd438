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
                      unsigned long long* __restrict__ counters, uint64_t* __restrict__ status,
                      mt_pair* __restrict__ out, uint64_t out_cap, mt_pair* __restrict__ ess, uint32_t ess_cap,
                      uint64_t ntiles, unsigned long long* __restrict__ stats) {
    __shared__ uint64_t s_tile;
    __shared__ uint32_t s_cnt[ITEMS * 8];
    __shared__ uint64_t s_prefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(counters + CTR_TICKET, 1ull);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t first = tile * TILE;  // local index of the tile's first vertex

    Cell cell[ITEMS];
    bool fin[ITEMS];
    uint32_t mask[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const uint64_t l = first + uint64_t(k) * THREADS + threadIdx.x;
        const uint64_t u = base + l;     // global id (C, T, f are indexed by global id)
        cell[k] = l < n ? ld_cell(C + u) : Cell{0, 0};
        fin[k] = l < n && cs_of(cell[k]) != uint32_t(u);
        mask[k] = __ballot_sync(FULL_MASK, fin[k]);
        if (lane == 0) s_cnt[k * 8 + warp] = __popc(mask[k]);
    }
    __syncthreads();
    // exclusive scan of the 32 (k, warp) counts in u order, by warp 0
    if (warp == 0) {
        const uint32_t c = s_cnt[lane];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        s_cnt[lane] = incl - c;
        const uint32_t agg = __shfl_sync(FULL_MASK, incl, 31);
        if (lane == 0) {
            st_relaxed(status + tile, (tile == 0 ? ST_PRE : ST_AGG) | agg);  // publish before walking
        }
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
        if (x[k] == uint32_t(u)) {                    // root (u, u, u): essential class
            const uint32_t i = atomicAdd(reinterpret_cast<unsigned int*>(counters + CTR_ESS), 1u);
            if (i < ess_cap) ess[i] = mt_pair{uint32_t(u), uint32_t(u), __ldg(f + u), __int_as_float(0x7f800000)};
            else atomicOr(counters + CTR_ERR, ERR_ESS_CAPACITY);
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

    // --- decoupled look-back for the tile's output offset ----------------
    __syncthreads();
    if (warp == 0) {
        uint64_t prefix = 0;
        int64_t j = int64_t(tile) - 1;
        while (j >= 0) {
            const int64_t idx = j - lane;
            const uint64_t st = idx >= 0 ? ld_relaxed(status + idx) : ST_PRE;
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
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    const uint64_t prefix = s_prefix;
    // inclusive prefix = prefix + this tile's aggregate; s_cnt holds exclusive
    // offsets, so the aggregate is the last offset + the last (k, warp) count,
    // which the last thread's own ballot holds.
    if (threadIdx.x == THREADS - 1) {
        const uint64_t total = prefix + s_cnt[(ITEMS - 1) * 8 + 7] + __popc(mask[ITEMS - 1]);
        if (tile != 0) st_relaxed(status + tile, ST_PRE | total);
        if (tile == ntiles - 1) counters[CTR_FIN] = total;
    }

    // --- write this tile's finite pairs in ascending u --------------------
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (!fin[k]) continue;
        const uint64_t u = base + first + uint64_t(k) * THREADS + threadIdx.x;
        const uint64_t pos = prefix + s_cnt[k * 8 + warp] + __popc(mask[k] & ((1u << lane) - 1u));
        const uint32_t s = cs_of(cell[k]);
        if (pos < out_cap) out[pos] = mt_pair{uint32_t(u), s, __ldg(f + u), view.value(f, s)};
        else atomicOr(counters + CTR_ERR, ERR_CAPACITY);
    }
}

// Appends the essential classes (ascending vertex) after the finite pairs and
// checks the capacity.  One CTA; the number of essential classes is the number
// of connected components (one for a non-empty grid).
__global__ void finish_diagram_kernel(unsigned long long* __restrict__ counters, mt_pair* __restrict__ out,
                                      uint64_t out_cap, mt_pair* __restrict__ ess, uint32_t ess_cap) {
    const uint64_t nfin = counters[CTR_FIN];
    uint32_t ness = uint32_t(counters[CTR_ESS]);
    if (ness > ess_cap) ness = ess_cap;
    if (threadIdx.x == 0) {
        // insertion sort by vertex (ness is tiny)
        for (uint32_t i = 1; i < ness; ++i) {
            mt_pair p = ess[i];
            uint32_t j = i;
            while (j > 0 && ess[j - 1].birth_v > p.birth_v) { ess[j] = ess[j - 1]; --j; }
            ess[j] = p;
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < ness; i += blockDim.x) {
        if (nfin + i < out_cap) out[nfin + i] = ess[i];
        else atomicOr(counters + CTR_ERR, ERR_CAPACITY);
    }
}

}  // namespace

uint64_t repair_tiles(uint64_t n) { return (n + TILE - 1) / TILE; }

void launch_repair_diagram(Cell* C, uint64_t* T, const float* f, uint64_t base, uint64_t n, unsigned long long* counters,
                           uint64_t* status, mt_pair* out, uint64_t out_cap, mt_pair* ess, uint32_t ess_cap,
                           unsigned long long* stats, const ForestRef* forest, cudaStream_t stream) {
    const uint64_t ntiles = repair_tiles(n);
    if (ntiles == 0) return;
    if (forest)
        repair_diagram_kernel<<<uint32_t(ntiles), THREADS, 0, stream>>>(ForestView{*forest, base, n}, C, T, f, base, n,
                                                                         counters, status, out, out_cap, ess, ess_cap,
                                                                         ntiles, stats);
    else
        repair_diagram_kernel<<<uint32_t(ntiles), THREADS, 0, stream>>>(LocalView{}, C, T, f, base, n, counters,
                                                                         status, out, out_cap, ess, ess_cap, ntiles,
                                                                         stats);
}

void launch_finish_diagram(unsigned long long* counters, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                           uint32_t ess_cap, cudaStream_t stream) {
    finish_diagram_kernel<<<1, 128, 0, stream>>>(counters, out, out_cap, ess, ess_cap);
}

}  // namespace mt
