// common.cuh -- device helpers shared by the sm_100a kernels of libmt_b200.
//
// Total order (step a1, SURVEY.md 8a / DESIGN.md "K1"): the paper compares raw
// values f(u) < f(v) and never resolves ties;
// reading R1 breaks ties by vertex id, i.e. vertices are ordered by the 64-bit
// key  key(u) = ord(f[u]) << 32 | u  compared as an unsigned integer, where
// ord() maps IEEE float32 bits to uint32 monotonically (-0.0 canonicalised to
// +0.0 first, reading R2).  For the split tree (reading R16)
// ord is complemented: ~ord(x) orders like ord(-x) and ids stay ascending.
#pragma once
#include <cstdint>

namespace mt {

constexpr uint32_t FULL_MASK = 0xffffffffu;

// uint32 whose unsigned order equals the IEEE order of finite floats.
__device__ __forceinline__ uint32_t ord32(float x) {
    uint32_t b = __float_as_uint(x);
    b = (b == 0x80000000u) ? 0u : b;                     // -0.0 -> +0.0
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ bool nonfinite(float x) {
    return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}

// ord of f[x] with the split-tree complement mask (0 or ~0) applied.
__device__ __forceinline__ uint32_t ordf(const float* __restrict__ f, uint32_t x, uint32_t flip) {
    return ord32(__ldg(f + x)) ^ flip;
}

__device__ __forceinline__ uint64_t key_of(uint32_t ord, uint32_t id) {
    return (static_cast<uint64_t>(ord) << 32) | id;
}

__device__ __forceinline__ uint64_t keyf(const float* __restrict__ f, uint32_t x, uint32_t flip) {
    return key_of(ordf(f, x, flip), x);
}

// Packed triplet cell (reading R11): s high, v low.
__device__ __forceinline__ uint64_t pack(uint32_t s, uint32_t v) {
    return (static_cast<uint64_t>(s) << 32) | v;
}
__device__ __forceinline__ uint32_t cell_s(uint64_t c) { return static_cast<uint32_t>(c >> 32); }
__device__ __forceinline__ uint32_t cell_v(uint64_t c) { return static_cast<uint32_t>(c); }

// Coherent (L1-bypassing) loads/stores of cells that other threads CAS
// concurrently: a plain ld.global may hit a stale L1 line and livelock a CAS
// retry loop (reading R8).
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t cas64(uint64_t* p, uint64_t expected, uint64_t desired) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(p), expected, desired);
}

// ---- 16-byte working cells of the merge phase --------------------------
// During the merge the store lives in the workspace as 16-byte cells
//   lo = key(s) = ord(f[s]) << 32 | s        (the packed (s, v) of the paper,
//   hi = ord(f[u]) << 32 | v                  widened by the two order keys)
// so that a climb step (Alg. 3 l.2-8, Alg. 4 l.3) needs ONE dependent load:
// the saddle's key and the owner's key travel with the cell instead of being
// gathered from f.  Updates are single 128-bit CAS (atom.cas.b128, sm_90+);
// loads are single-copy-atomic ld.relaxed.gpu.b128.  The output store T[u] =
// s << 32 | v (reading R11) is written from these cells by the repair kernel.
struct Cell {
    uint64_t lo, hi;
};
__device__ __forceinline__ Cell make_cell(uint64_t key_s, uint32_t ord_u, uint32_t v) {
    return Cell{key_s, (static_cast<uint64_t>(ord_u) << 32) | v};
}
__device__ __forceinline__ uint32_t cv_of(const Cell& c) { return static_cast<uint32_t>(c.hi); }
__device__ __forceinline__ uint32_t cs_of(const Cell& c) { return static_cast<uint32_t>(c.lo); }
__device__ __forceinline__ uint64_t self_key(const Cell& c, uint32_t u) {
    return (c.hi & 0xffffffff00000000ull) | u;
}
__device__ __forceinline__ Cell ld_cell(const Cell* p) {
    Cell c;
    asm volatile("{\n\t.reg .b128 d;\n\tld.relaxed.gpu.global.b128 d, [%2];\n\tmov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(c.lo), "=l"(c.hi) : "l"(p) : "memory");
    return c;
}
// non-coherent (L1-cached) 16-byte load: only for cells no thread writes during the kernel
__device__ __forceinline__ Cell ld_cell_nc(const Cell* p) {
    Cell c;
    asm("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(c.lo), "=l"(c.hi) : "l"(p));
    return c;
}
__device__ __forceinline__ void st_cell(Cell* p, const Cell& c) {
    asm volatile("{\n\t.reg .b128 d;\n\tmov.b128 d, {%1, %2};\n\tst.relaxed.gpu.global.b128 [%0], d;\n\t}"
                 ::"l"(p), "l"(c.lo), "l"(c.hi) : "memory");
}
// v field alone (single-copy atomic 32-bit store; a concurrent 128-bit load
// sees either the old or the new v with the unchanged key fields)
__device__ __forceinline__ void st_cell_v(Cell* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(reinterpret_cast<char*>(p) + 8), "r"(v) : "memory");
}
// 128-bit compare-and-swap; returns the previous value.
__device__ __forceinline__ Cell cas_cell(Cell* p, const Cell& expected, const Cell& desired) {
    Cell old;
    asm volatile(
        "{\n\t.reg .b128 d, c, v;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\t"
        "atom.relaxed.gpu.global.cas.b128 d, [%6], c, v;\n\tmov.b128 {%0, %1}, d;\n\t}"
        : "=l"(old.lo), "=l"(old.hi)
        : "l"(expected.lo), "l"(expected.hi), "l"(desired.lo), "l"(desired.hi), "l"(p)
        : "memory");
    return old;
}

// Error bits (sticky, in the workspace counters).
constexpr uint32_t ERR_NONFINITE = 1u;
constexpr uint32_t ERR_CAPACITY = 2u;
constexpr uint32_t ERR_ESS_CAPACITY = 4u;
constexpr uint32_t ERR_FOREST = 8u;   // a vertex missing from the gathered boundary forest

// Workspace counter slots (uint64 each).
enum CounterSlot : int {
    CTR_TICKET = 0,     // dynamic tile ticket of the repair/diagram kernel
    CTR_ERR = 1,        // error bits
    CTR_ESS = 2,        // number of essential classes found
    CTR_FIN = 3,        // number of finite pairs (written by the last tile)
    CTR_FFETCH = 4,     // next inter-slab edge to hand out (forest_merge)
    CTR_QLEN = 5,       // crossing-edge queue length (dedupe_cross)
    CTR_QFETCH = 6,     // next queue entry to hand out (merge_queue)
    CTR_FCOUNT = 7,     // boundary-forest records of this slab
    CTR_FILT_TICKET = 8,  // mt_filter_diagram: tile tickets
    CTR_FILT_KEPT = 9,    // mt_filter_diagram: records kept
    CTR_STAGE = 10,       // diagram records staged by the repair bricks
    CTR_FQLEN = 11,       // deduplicated inter-slab edges queued (forest_dedupe)
    CTR_TILE = 12,        // persistent tile_tmt: next tile ticket
    CTR_COUNT = 16
};

// Optional diagnostics (mt_set_stats): event counters in the workspace.
enum StatSlot : int {
    ST_EDGES = 0,        // tile-crossing edges examined by the global merge kernel
    ST_SKIPPED = 1,      // of those, edges whose walks met (nothing to join)
    ST_PRE_HOPS = 2,     // cells followed by the walks at the edge level
    ST_MERGE_ITERS = 3,  // iterations of the Alg. 3 loop
    ST_CAS_FAIL = 4,     // failed CAS (Alg. 3 l.17 restarts)
    ST_REPAIR_HOPS = 5,  // cells followed by the repair walks
    ST_TILE_EDGES = 6,   // in-tile edges between two basins (tile kernel)
    ST_TILE_HOPS = 7,    // cells followed by the in-tile walks
    ST_TILE_ITERS = 8,   // in-tile Alg. 3 loop iterations
    ST_TILE_REPAIR = 9,  // cells followed by the in-tile repair
    ST_TILE_COMPRESS = 10,  // cells followed by the in-tile compress
    ST_CYC_LOAD = 11,    // SM cycles (summed over tiles) of each tile phase
    ST_CYC_DESCENT = 12,
    ST_CYC_COMPRESS = 13,
    ST_CYC_MERGE = 14,
    ST_CYC_REPAIR = 15,
    ST_CYC_WRITE = 16,
    ST_CYC_LIST = 17,
    ST_TILE_PAIRS = 18,  // adjacent basin pairs (one merged edge each)
    ST_QUEUED = 19,      // tile-crossing edges left after the warp-level basin-pair dedupe
    ST_UNUSED_20 = 20,        // (retired: repair memo statistics)
    ST_UNUSED_21 = 21,
    ST_COUNT = 24
};

}  // namespace mt
