// kernels.cuh -- host launchers of the sm_100a kernels (internal to libmt_b200).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "mt.h"

namespace mt {

// Per-device launch attributes (mt_api.cu).  A CUfunction's attributes belong to the device's
// context, so each device a context runs on needs its own opt-in; both helpers are thread safe
// and cache per (kernel, current device).
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) once per kernel and device
cudaError_t ensure_smem_attr(const void* func, int bytes);
// resident CTAs per SM of a kernel on the current device (cached)
int occupancy_per_sm(const void* func, int threads, size_t smem);

// The part of the global grid one context computes: planes [z_begin, z_end) of an
// nx x ny x nz grid (the whole grid on one GPU; a z-slab per rank on several).
// Vertex ids are global; device pointers handed to the launchers are shifted by
// -base so that they are indexed by global id.
struct Slab {
    uint32_t nx, ny, nz;        // global grid
    uint32_t z_begin, z_end;    // owned planes
    uint64_t base;              // global id of the first owned vertex = nx ny z_begin
    uint64_t n;                 // owned vertices
};

// Boundary forest of all slabs (multi-GPU, slab.cu): records of every rank in one
// array, an open-addressing table view id -> record index, 16-B cells with view
// ids after the forest merge, and the f bits of each record's vertex.
struct ForestRef {
    const uint64_t* table;      // (id << 32 | index) or ~0 (empty); size mask + 1
    const uint64_t* vtable;     // (id << 32 | f bits) of the zero-valued saddles; same size
    uint32_t mask;
    Cell* cells;                // merged cells, view ids
    const mt_forest_record* recs;
    const uint32_t* vid;        // view id of each record's vertex
    unsigned long long* err;    // error bits (ERR_FOREST on a missing id)
};

constexpr int MAX_SLABS = 64;

// The gathered records in this rank's view (slab.cu header): slab k's ids at voff[k] + local id
// (own slab, k == self) or voff[k] + compressed id (other slabs; in 32-bit mode the compressed id
// is the local id and voff[k] = nx ny z_begin(k), so view ids are global ids).
struct ForestXlate {
    uint32_t nslabs, self, flip;
    bool wide;
    uint64_t rec_off[MAX_SLABS + 1];   // first record of slab k
    uint32_t voff[MAX_SLABS];
    uint64_t real_base[MAX_SLABS];     // global id of slab k's first vertex
    uint32_t dec_lo, own_lo;           // wide: lowest remote view id, first own view id
    uint64_t own_n;
    // index of remote view id y in the decode array (the own range is skipped)
    __device__ __forceinline__ uint64_t dec_index(uint32_t y) const {
        return y < own_lo ? uint64_t(y - dec_lo) : uint64_t(own_lo - dec_lo) + (uint64_t(y) - own_lo - own_n);
    }
};

// view id -> 64-bit global id (identity in 32-bit mode)
struct IdDecode {
    bool wide;
    uint32_t dec_lo, own_lo;
    uint64_t own_n, own_gid0;
    const uint64_t* dec;
    __device__ __forceinline__ uint64_t gid(uint32_t y) const {
        if (!wide) return y;
        const uint64_t k = uint64_t(y) - own_lo;
        if (k < own_n) return own_gid0 + k;
        return y < own_lo ? dec[y - dec_lo] : dec[uint64_t(own_lo - dec_lo) + (uint64_t(y) - own_lo - own_n)];
    }
};

__device__ __forceinline__ uint32_t forest_hash(uint32_t id, uint32_t mask) {
    uint32_t h = id ^ (id >> 16);   // integer mixer: consecutive face ids spread over the table
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h & mask;
}
constexpr uint32_t FOREST_MISS = 0xffffffffu;
// index of id's record, or FOREST_MISS (an empty slot ends the probe)
__device__ __forceinline__ uint32_t forest_lookup(const ForestRef& F, uint32_t id) {
    uint32_t h = forest_hash(id, F.mask);
    for (uint32_t probe = 0; probe <= F.mask; ++probe) {
        const uint64_t e = F.table[h];
        if (e == ~0ull) return FOREST_MISS;
        if (uint32_t(e >> 32) == id) return uint32_t(e);
        h = (h + 1) & F.mask;
    }
    return FOREST_MISS;
}

__device__ __forceinline__ bool forest_value(const ForestRef& F, uint32_t id, uint32_t* bits) {
    uint32_t h = forest_hash(id, F.mask);
    for (uint32_t probe = 0; probe <= F.mask; ++probe) {
        const uint64_t e = F.vtable[h];
        if (e == ~0ull) return false;
        if (uint32_t(e >> 32) == id) {
            *bits = uint32_t(e);
            return true;
        }
        h = (h + 1) & F.mask;
    }
    return false;
}

// tile shape (32 x ty x tz, 4096 vertices) for a grid with nz planes
void tile_shape(uint32_t nz_global, uint32_t* ty, uint32_t* tz);

// K1 + K2 + in-tile K3/K4: keys, steepest descent, tile-local merge tree (tile_tmt.cu)
// x-face records of the tiles (2 faces x rows per tile, 8 B each: order key << 32 | R)
uint64_t xface_entries(const Slab& sl);
// writes the tile store T0 (8 B per vertex, s << 32 | v, global ids) into the triplet buffer,
// 16-B cells for the tile minima only, and the x-face records
void launch_tile_tmt(const float* f, Cell* C, uint64_t* T0, uint64_t* xface, const Slab& sl, uint32_t flip,
                     unsigned long long* counters, unsigned long long* stats, cudaStream_t stream);

// both trees from one read of f: the merge tree into the first set of
// buffers, the split tree into the second
void launch_tile_tmt_dual(const float* f, Cell* C_join, uint64_t* T0_join, uint64_t* xface_join,
                          unsigned long long* counters_join, Cell* C_split, uint64_t* T0_split,
                          uint64_t* xface_split, unsigned long long* counters_split, const Slab& sl,
                          unsigned long long* stats, cudaStream_t stream);

// K3: merge of the tile-crossing grid edges on the global store (merge_cross.cu)
uint64_t cross_edges(const Slab& sl);
size_t cross_queue_entry_bytes();
// returns 0 when the slab has a single tile (no crossing edges, no kernel launched)
// Stepped queue (cross_stepped()): every 512-edge step of the enumeration writes its survivors at
// its own edge positions and their count to qcnt[step] (cross_steps() steps), no global counter.
int launch_dedupe_cross(const float* f, const uint64_t* T0, const uint64_t* xface, const Slab& sl, uint32_t flip,
                        void* queue,
                        uint64_t cap, unsigned long long* qlen, uint32_t* qcnt, unsigned long long* stats,
                        int num_sms, cudaStream_t stream);
uint64_t cross_steps(const Slab& sl);
bool cross_stepped();

// the queue consumer alone (queue entries: {uint64 L, uint32 basin_hi, uint32 basin_lo}); qcnt null:
// a compact queue of *qlen entries, else nsteps steps of 512 entries with qcnt[step] of them used
void launch_merge_queue(Cell* C, const void* queue, uint64_t cap, const unsigned long long* qlen,
                        const uint32_t* qcnt, uint64_t nsteps,
                        unsigned long long* fetch, unsigned long long* stats, int num_sms, cudaStream_t stream);

// explicit graphs in CSR form (graph.cu)
void launch_graph_init(const float* f, const uint64_t* row, const uint32_t* col, uint32_t n, uint32_t flip, Cell* C,
                       unsigned long long* counters, int num_sms, cudaStream_t stream);
void launch_graph_edges(const uint64_t* row, const uint32_t* col, uint32_t n, Cell* C, uint32_t* basin, void* queue,
                        uint64_t cap, unsigned long long* qlen, unsigned long long* counters, int num_sms,
                        cudaStream_t stream);

// K4: repair (memoised walks per brick, diagram records staged per segment)
// and K5: the ordered diagram (repair_diagram.cu)
struct RepairOut {
    mt_pair* stage;                 // staging runs of the bricks' diagram records
    uint64_t stage_cap;
    uint16_t* seg_cnt;              // per segment (<= 32 consecutive ids): finite | essential << 8
    uint32_t* seg_pos;              // per segment: first staged record
    unsigned long long* counters;
};
uint64_t repair_segments(const Slab& sl);     // segments of the slab
uint64_t repair_segments_bound(uint64_t n);   // >= repair_segments of any slab of n vertices
// staging records the repair of this slab addresses when its bricks stage at fixed offsets (0: it
// uses a global counter and needs at most one record per minimum)
uint64_t repair_stage_records(const Slab& sl);
uint64_t diagram_tiles(uint64_t nseg);        // diagram tiles; one 16-B status record each
uint64_t diagram_tiles_bound(uint64_t nseg);  // >= diagram_tiles of any nseg' <= nseg (status sizing)
// tiled: T holds tile_tmt's T0 and only tile minima have cells (grids); else every vertex has a
// cell and T is output only (explicit graphs)
void launch_repair(const Cell* C, uint64_t* T, const float* f, const Slab& sl, uint32_t flip, const RepairOut& o,
                   bool tiled, unsigned long long* stats, const ForestRef* forest, cudaStream_t stream);
void launch_diagram(const Slab& sl, const RepairOut& o, void* status, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                    uint64_t ess_cap, cudaStream_t stream);
void launch_finish_diagram(unsigned long long* counters, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                           uint64_t ess_cap, cudaStream_t stream);

// persistence simplification of the diagram (diagram_filter.cu)
uint64_t filter_tiles(uint64_t n);
void launch_filter_diagram(const mt_pair* in, uint64_t n_fin, uint64_t n_all, float eps, mt_pair* out, uint64_t cap,
                           unsigned long long* ctl, uint64_t* status, cudaStream_t stream);

// multi-GPU boundary forest (slab.cu)
// T0: the slab's tile store (regular vertices have no working cell, see launch_tile_tmt); the
// faces marked are the slab's inter-slab faces (below / above)
void launch_forest_mark(const Cell* C, const uint64_t* T0, const Slab& sl, bool has_bottom, bool has_top,
                        uint8_t* flag, cudaStream_t stream);
// records with slab-local ids (compressed ids = local ids)
// (the face vertices' records at fixed slots: the bottom face first, then the top face, then the
// rest; returns the kernels launched)
int launch_forest_compact(const Cell* C, const uint64_t* T0, const float* f, const Slab& sl, const uint8_t* flag,
                          mt_forest_record* recs, uint64_t cap, unsigned long long* count, bool has_bottom,
                          bool has_top, int num_sms, cudaStream_t stream);
// wide mode: the records' compressed ids (top face from local id top_begin on; UINT64_MAX: none);
// scratch >= forest_compress_scratch_bytes(n); returns the kernels launched
size_t forest_compress_scratch_bytes(uint64_t n);
int launch_forest_compress(mt_forest_record* recs, const unsigned long long* count, uint64_t n, uint64_t top_begin,
                           void* scratch, int num_sms, cudaStream_t stream);
// open-addressing table slots for n_all gathered records (>= 4 n_all, a power of two), or 0
// when that exceeds 2^31 (32-bit table indices)
uint64_t forest_table_size(uint64_t n_all);
// cells, view ids and (wide) the decode array of the gathered records
void launch_forest_build(const mt_forest_record* all, uint64_t n_all, const ForestXlate& X, uint64_t* table,
                         uint64_t* vtable, uint32_t mask, Cell* cells, uint32_t* vid, uint64_t* dec, int num_sms,
                         cudaStream_t stream);
// inter-slab edges: deduplicated by tile-representative pairs into `queue`, then merged;
// boundary k joins view ids a0[k] + r and b0[k] + r, r < nx ny
size_t forest_queue_entry_bytes();
// ia0 / ib0 (or null): record index of vertex (0, 0) of each boundary's lower / upper face
void launch_forest_merge(const ForestRef& F, const Slab& sl, uint32_t nslabs, const uint32_t* a0, const uint32_t* b0,
                         const uint32_t* ia0, const uint32_t* ib0, void* queue, unsigned long long* qlen,
                         unsigned long long* fetch, int num_sms, cudaStream_t stream);
void launch_forest_writeback(const ForestRef& F, uint64_t n_all, Cell* C, const uint64_t* T0, const Slab& sl,
                             int num_sms, cudaStream_t stream);
// view ids -> 64-bit global ids
void launch_triplets64(const uint64_t* T, uint64_t count, const IdDecode& d, mt_triplet64* out, int num_sms,
                       cudaStream_t stream);
void launch_pairs64(const mt_pair* in, uint64_t count, const IdDecode& d, mt_pair64* out, int num_sms,
                    cudaStream_t stream);

}  // namespace mt
