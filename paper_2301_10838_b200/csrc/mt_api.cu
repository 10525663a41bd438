// mt_api.cu -- the C ABI of libmt_b200 (declared and documented in
// include/mt.h): context, caller-owned workspace layout, sticky errors, stream
// plumbing and the launch sequence of the hot path:
//   zero counters -> tile_tmt (K1, K2, in-tile K3/K4) -> merge_cross (K3 on
//   the tile-crossing edges) -> repair_diagram (K4 + K5) -> finish_diagram
//   -> K4+K5 repair_diagram -> finish_diagram
// All launches are asynchronous on the caller's stream; only mt_diagram /
// mt_diagram_view / mt_last_error synchronise.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <set>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"
#include "mt.h"

namespace mt {

namespace {
std::mutex g_attr_mutex;
std::set<std::pair<const void*, int>> g_smem_done;
std::map<std::pair<const void*, int>, int> g_occupancy;
}  // namespace

cudaError_t ensure_smem_attr(const void* func, int bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_attr_mutex);
    if (g_smem_done.count({func, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) g_smem_done.insert({func, dev});
    return e;
}

int occupancy_per_sm(const void* func, int threads, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    std::lock_guard<std::mutex> lock(g_attr_mutex);
    auto it = g_occupancy.find({func, dev});
    if (it != g_occupancy.end()) return it->second;
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, func, threads, smem) != cudaSuccess || per < 1) per = 1;
    g_occupancy[{func, dev}] = per;
    return per;
}

struct DistState;
void dist_destroy(DistState* d);
mt_status dist_compute(mt_ctx* c, DistState* d, const float* f, uint64_t* T, uint32_t flags, cudaStream_t s);

}  // namespace mt

namespace {

constexpr size_t ALIGN = 256;
constexpr uint32_t ESS_CAP = 64;  // essential classes = connected components (1 per grid)
constexpr int MAX_EVENTS = 16;

size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

struct Layout {
    size_t counters, status, status_bytes, stats, ess, cells, xface, queue, qcnt, pairs, stage, seg_cnt, seg_pos, flags,
        recs, total;
    uint64_t pairs_cap, recs_cap, queue_cap, ess_cap, seg_cap, stage_cap;
};

bool valid_dims(const uint32_t dims[3], int conn) {
    if (!dims) return false;
    if (conn != 4 && conn != 6) return false;
    if (conn == 4 && dims[2] > 1) return false;
    return true;
}

// n vertices; ncross queue entries; ess_cap essential records (components);
// slab: add the boundary-forest buffers
Layout layout_for(uint64_t n, uint64_t ncross, bool slab = false, uint64_t ess_cap = ESS_CAP, uint64_t nxface = 0,
                  uint64_t stage_recs = 0) {
    Layout L{};
    // records = #minima.  On a grid the strict minima form an independent set,
    // so at most ceil(n/2) (+1 slack); a general graph (ess_cap = n) may have n.
    L.pairs_cap = n ? (ess_cap >= n ? n : (n + 1) / 2 + 1) : 0;
    L.seg_cap = n ? mt::repair_segments_bound(n) : 0;
    // tile records of the diagram compaction (16 B) / of mt_filter_diagram (8 B)
    L.status_bytes = std::max(mt::diagram_tiles_bound(L.seg_cap) * sizeof(mt::Cell),
                              mt::filter_tiles(L.pairs_cap + ess_cap) * sizeof(uint64_t));
    size_t off = 0;
    L.counters = off;
    off += align_up(mt::CTR_COUNT * sizeof(uint64_t));
    L.status = off;  // contiguous with counters: one memset zeroes the chunk status records too
    off = align_up(off + L.status_bytes);
    L.stats = off;
    off += align_up(mt::ST_COUNT * sizeof(uint64_t));
    L.ess = off;
    L.ess_cap = ess_cap;
    off += align_up(ess_cap * sizeof(mt_pair));
    L.cells = off;  // 16-byte working cells of the merge phase (grids: written for tile minima only)
    off += align_up(n * sizeof(mt::Cell));
    L.xface = off;  // x-face records of the tiles (tile_tmt -> dedupe_cross)
    off += align_up(nxface * sizeof(uint64_t));
    L.queue = off;  // deduplicated tile-crossing edges
    L.queue_cap = ncross;
    off += align_up(ncross * mt::cross_queue_entry_bytes());
    L.qcnt = off;   // stepped queue: survivors per step of the enumeration (steps of >= 128 edges)
    off += align_up((ncross + 127) / 128 * sizeof(uint32_t));
    L.pairs = off;
    off += align_up(L.pairs_cap * sizeof(mt_pair));
    L.stage = off;    // diagram records staged by the repair (at most one per minimum, or fixed brick runs)
    L.stage_cap = std::max(L.pairs_cap, stage_recs);
    off += align_up(L.stage_cap * sizeof(mt_pair));
    L.seg_cnt = off;
    off += align_up(L.seg_cap * sizeof(uint16_t));
    L.seg_pos = off;
    off += align_up(L.seg_cap * sizeof(uint32_t));
    if (slab) {  // boundary forest of the slab: a flag per vertex (then the wide-mode compression
                 // scratch), at most n records
        L.flags = off;
        off += align_up(std::max<size_t>(n, mt::forest_compress_scratch_bytes(n)));
        L.recs = off;
        L.recs_cap = n;
        off += align_up(n * sizeof(mt_forest_record));
    }
    L.total = off;
    return L;
}

// workspace of a grid context owning planes [z_begin, z_end)
Layout grid_layout(const uint32_t dims[3], uint32_t z_begin, uint32_t z_end, bool slab) {
    const uint64_t n = uint64_t(dims[0]) * dims[1] * (z_end - z_begin);
    const mt::Slab sl{dims[0], dims[1], dims[2], z_begin, z_end, uint64_t(dims[0]) * dims[1] * z_begin, n};
    return layout_for(n, mt::cross_edges(sl), slab, ESS_CAP, mt::xface_entries(sl), mt::repair_stage_records(sl));
}

}  // namespace

struct mt_ctx {
    uint32_t nx, ny, nz;
    uint64_t n;              // vertices this context owns
    mt::Slab slab;           // owned planes of the global grid (all of them for mt_create), in the
                             // context's id view (slab.cu header; wide mode: a virtual grid)
    uint32_t z_begin, z_end; // owned planes of the real grid
    uint64_t gid0;           // global id of the first owned vertex
    bool wide = false;       // wide ids (f3): view ids != global ids
    mt::IdDecode decode{};   // view -> global ids of the last result
    bool decode_ok = false;
    bool multi = false;      // created by mt_create_slab
    bool graph = false;      // created by mt_create_graph (CSR adjacency instead of a grid)
    bool local_done = false; // mt_compute_local ran, mt_compute_global pending
    uint64_t* local_T = nullptr;  // the triplet buffer mt_compute_local wrote the tile store into
    const float* f = nullptr;
    uint32_t flip = 0;
    uint64_t n_adj = 0;      // graph contexts: adjacency entries (the queue capacity)
    int conn;
    int device;
    int num_sms;
    char* ws;
    size_t ws_bytes;
    Layout L;
    mt_pair* reg_out = nullptr;
    uint64_t reg_cap = 0;
    bool computed = false;
    mt_status sticky = MT_OK;
    uint64_t* host_ctr = nullptr;  // pinned
    uint32_t launches = 0;
    bool profiling = false;
    bool stats = false;
    cudaEvent_t ev[MAX_EVENTS + 1] = {};
    const char* ev_name[MAX_EVENTS] = {};
    int nev = 0;
    mt::DistState* dist = nullptr;  // mt_create_dist: communicator + exchange buffers (dist.cu)
    // mt_compute_host: streams and events of the host pipeline (created at first use)
    cudaStream_t hs[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t hev[6] = {};
};

namespace mt {
void slab_forest(mt_ctx* c, mt_forest_record** recs, unsigned long long** count_dev, uint64_t* cap) {
    *recs = reinterpret_cast<mt_forest_record*>(c->ws + c->L.recs);
    *count_dev = reinterpret_cast<unsigned long long*>(c->ws + c->L.counters) + CTR_FCOUNT;
    *cap = c->L.recs_cap;
}
void attach_dist(mt_ctx* c, DistState* d) { c->dist = d; }
}  // namespace mt

namespace {

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

unsigned long long* counters_of(mt_ctx* c) { return reinterpret_cast<unsigned long long*>(c->ws + c->L.counters); }
mt::Cell* cells_of(mt_ctx* c) { return reinterpret_cast<mt::Cell*>(c->ws + c->L.cells) - c->slab.base; }
unsigned long long* stats_of(mt_ctx* c) {
    return c->stats ? reinterpret_cast<unsigned long long*>(c->ws + c->L.stats) : nullptr;
}
mt_pair* target_of(mt_ctx* c, uint64_t* cap) {
    if (c->reg_out) {
        *cap = c->reg_cap;
        return c->reg_out;
    }
    *cap = c->L.pairs_cap;
    return reinterpret_cast<mt_pair*>(c->ws + c->L.pairs);
}

void mark(mt_ctx* c, const char* name, cudaStream_t s) {
    if (!c->profiling || c->nev >= MAX_EVENTS) return;
    c->ev_name[c->nev] = name;
    cudaEventRecord(c->ev[c->nev], s);
    c->nev++;
}

// Sync the stream, read the device counters, fold device error bits into the
// sticky status.
mt_status sync_counters(mt_ctx* c, cudaStream_t s) {
    if (!c->computed) return MT_ERR_STATE;
    if (c->n == 0) {
        c->host_ctr[mt::CTR_FCOUNT] = 0;
        c->host_ctr[mt::CTR_FIN] = 0;
        c->host_ctr[mt::CTR_ESS] = 0;
        c->host_ctr[mt::CTR_ERR] = 0;
        return c->sticky;
    }
    if (cudaMemcpyAsync(c->host_ctr, counters_of(c), mt::CTR_COUNT * sizeof(uint64_t), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return c->sticky = MT_ERR_CUDA;
    const uint64_t err = c->host_ctr[mt::CTR_ERR];
    if (err & mt::ERR_NONFINITE) c->sticky = MT_ERR_NONFINITE;
    else if (err & mt::ERR_FOREST) c->sticky = MT_ERR_INVALID_ARG;
    else if (err & (mt::ERR_CAPACITY | mt::ERR_ESS_CAPACITY)) c->sticky = MT_ERR_CAPACITY;
    return c->sticky;
}


}  // namespace
extern "C" void mt_destroy(mt_ctx* c);
namespace {

// wide mode: the slab's planes in a virtual grid of 32-bit ids, centred so that the other slabs'
// referenced vertices fit below and above (slab.cu header); false if the slab itself cannot fit
bool wide_view(const uint32_t dims[3], uint32_t z_begin, uint32_t z_end, mt::Slab* v) {
    const uint64_t sxy = uint64_t(dims[0]) * dims[1], nzl = z_end - z_begin;
    if (sxy == 0 || sxy > 0xffffffffull) return false;
    const uint64_t planes = 0xffffffffull / sxy;   // view ids stay below 2^32 - 1
    if (planes < nzl + 2) return false;
    const uint64_t zb = (planes - nzl) / 2;
    *v = mt::Slab{dims[0], dims[1], uint32_t(planes), uint32_t(zb), uint32_t(zb + nzl), zb * sxy, nzl * sxy};
    return true;
}

bool n_global_fits(const uint32_t dims[3]) {   // nx ny nz < 2^63 (64-bit global ids)
    const uint64_t sxy = uint64_t(dims[0]) * dims[1];
    return sxy == 0 || dims[2] <= (1ull << 63) / sxy;
}

mt_status create_ctx(mt_ctx** out, const uint32_t dims[3], int conn, uint32_t z_begin, uint32_t z_end, bool multi,
                     int cuda_device, void* workspace, size_t workspace_bytes, const Layout* graph_layout = nullptr,
                     uint32_t options = 0) {
    if (!out) return MT_ERR_INVALID_ARG;
    *out = nullptr;
    if (!graph_layout && !valid_dims(dims, conn)) return MT_ERR_INVALID_ARG;
    if (!n_global_fits(dims)) return MT_ERR_TOO_LARGE;
    const bool wide = multi && ((options & MT_SLAB_WIDE_IDS) ||
                                uint64_t(dims[0]) * dims[1] * dims[2] > 0xffffffffull);
    mt::Slab view{};
    if (wide && !wide_view(dims, z_begin, z_end, &view)) return MT_ERR_TOO_LARGE;
    if (!wide && uint64_t(dims[0]) * dims[1] * dims[2] > 0xffffffffull) return MT_ERR_TOO_LARGE;
    const uint64_t n = uint64_t(dims[0]) * dims[1] * (z_end - z_begin);
    const Layout L = graph_layout ? *graph_layout
                                  : grid_layout(dims, z_begin, z_end, multi);
    if (!workspace || workspace_bytes < L.total || (reinterpret_cast<uintptr_t>(workspace) % ALIGN))
        return MT_ERR_WORKSPACE;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) return MT_ERR_CUDA;
    if (cuda_device < 0 || cuda_device >= ndev) return MT_ERR_INVALID_ARG;
    DeviceGuard g(cuda_device);
    if (!g.ok) return MT_ERR_CUDA;
    mt_ctx* c = new (std::nothrow) mt_ctx();
    if (!c) return MT_ERR_CUDA;
    c->nx = dims[0];
    c->ny = dims[1];
    c->nz = dims[2];
    c->n = n;
    c->slab = wide ? view : mt::Slab{dims[0], dims[1], dims[2], z_begin, z_end, uint64_t(dims[0]) * dims[1] * z_begin, n};
    c->z_begin = z_begin;
    c->z_end = z_end;
    c->gid0 = uint64_t(dims[0]) * dims[1] * z_begin;
    c->wide = wide;
    c->decode_ok = !wide;
    c->multi = multi;
    c->graph = graph_layout != nullptr;
    c->conn = conn;
    c->device = cuda_device;
    c->ws = static_cast<char*>(workspace);
    c->ws_bytes = workspace_bytes;
    c->L = L;
    if (cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cuda_device) != cudaSuccess ||
        cudaMallocHost(&c->host_ctr, mt::CTR_COUNT * sizeof(uint64_t)) != cudaSuccess) {
        delete c;
        return MT_ERR_CUDA;
    }
    for (int i = 0; i <= MAX_EVENTS; ++i)
        if (cudaEventCreate(&c->ev[i]) != cudaSuccess) {
            mt_destroy(c);
            return MT_ERR_CUDA;
        }
    *out = c;
    return MT_OK;
}

// shared by mt_compute and mt_compute_local: reset, then the slab's own merge tree; T (the
// caller's triplet buffer, indexed from the slab's first vertex) receives the tile store T0
// reset the context for a new compute: state, statistics, counters and chunk status records
mt_status prepare_compute(mt_ctx* c, const float* f, uint32_t flags, cudaStream_t s) {
    c->decode = mt::IdDecode{};   // 32-bit mode: view ids are global ids
    c->decode_ok = !c->wide;
    c->launches = 0;
    c->nev = 0;
    c->sticky = MT_OK;
    c->computed = true;
    c->f = f;
    c->flip = (flags & MT_FLAG_SPLIT_TREE) ? 0xffffffffu : 0u;
    unsigned long long* stats = stats_of(c);
    if (stats && cudaMemsetAsync(stats, 0, mt::ST_COUNT * sizeof(uint64_t), s) != cudaSuccess)
        return c->sticky = MT_ERR_CUDA;
    mark(c, "zero", s);
    if (cudaMemsetAsync(c->ws + c->L.counters, 0, c->L.status - c->L.counters + c->L.status_bytes,
                        s) != cudaSuccess)
        return c->sticky = MT_ERR_CUDA;
    return MT_OK;
}

uint64_t* xface_of(mt_ctx* c) { return reinterpret_cast<uint64_t*>(c->ws + c->L.xface); }

// the tile-crossing edges: dedupe + the queue merge (none on a single-tile grid)
void launch_cross(mt_ctx* c, uint64_t* T0, cudaStream_t s) {
    unsigned long long* ctr = counters_of(c);
    unsigned long long* stats = stats_of(c);
    mark(c, "dedupe_cross", s);
    uint32_t* qcnt = mt::cross_stepped() ? reinterpret_cast<uint32_t*>(c->ws + c->L.qcnt) : nullptr;
    int nl = mt::launch_dedupe_cross(c->f - c->slab.base, T0, xface_of(c), c->slab, c->flip, c->ws + c->L.queue,
                                     c->L.queue_cap, ctr + mt::CTR_QLEN, qcnt, stats, c->num_sms, s);
    if (nl) {
        mark(c, "merge_queue", s);
        mt::launch_merge_queue(cells_of(c), c->ws + c->L.queue, c->L.queue_cap, ctr + mt::CTR_QLEN, qcnt,
                               mt::cross_steps(c->slab), ctr + mt::CTR_QFETCH, stats, c->num_sms, s);
        ++nl;
    }
    c->launches += nl;
}

// shared by mt_compute and mt_compute_local: reset, then the slab's own merge tree; T (the
// caller's triplet buffer, indexed from the slab's first vertex) receives the tile store T0
mt_status start_compute(mt_ctx* c, const float* f, uint64_t* T, uint32_t flags, cudaStream_t s) {
    const mt_status st = prepare_compute(c, f, flags, s);
    if (st != MT_OK) return st;
    uint64_t* T0 = T - c->slab.base;
    mark(c, "tile_tmt", s);
    mt::launch_tile_tmt(f - c->slab.base, cells_of(c), T0, xface_of(c), c->slab, c->flip, counters_of(c),
                        stats_of(c), s);
    c->launches = 1;
    launch_cross(c, T0, s);
    return MT_OK;
}

// repair (with the merged forest on multi-GPU) + diagram into the target buffer
mt_status finish_compute(mt_ctx* c, uint64_t* T, const mt::ForestRef* forest, cudaStream_t s) {
    unsigned long long* ctr = counters_of(c);
    uint64_t cap = 0;
    mt_pair* out = target_of(c, &cap);
    mt_pair* ess = reinterpret_cast<mt_pair*>(c->ws + c->L.ess);
    const uint64_t base = c->slab.base;
    const mt::RepairOut ro{reinterpret_cast<mt_pair*>(c->ws + c->L.stage), c->L.stage_cap,
                           reinterpret_cast<uint16_t*>(c->ws + c->L.seg_cnt),
                           reinterpret_cast<uint32_t*>(c->ws + c->L.seg_pos), ctr};
    mark(c, "repair", s);
    mt::launch_repair(cells_of(c), T - base, c->f - base, c->slab, c->flip, ro, !c->graph, stats_of(c), forest, s);
    mark(c, "diagram", s);
    mt::launch_diagram(c->slab, ro, c->ws + c->L.status, out, cap, ess, c->L.ess_cap, s);
    mark(c, "finish_diagram", s);
    mt::launch_finish_diagram(ctr, out, cap, ess, c->L.ess_cap, s);
    if (c->profiling) cudaEventRecord(c->ev[c->nev], s);
    c->launches += 3;
    if (cudaGetLastError() != cudaSuccess) return c->sticky = MT_ERR_CUDA;
    return MT_OK;
}

}  // namespace

extern "C" {

int mt_abi_version(void) { return 3; }

const char* mt_status_string(mt_status s) {
    switch (s) {
        case MT_OK: return "ok";
        case MT_ERR_INVALID_ARG: return "invalid argument";
        case MT_ERR_TOO_LARGE: return "vertex ids do not fit (32-bit ids on one GPU / in a slab's view)";
        case MT_ERR_NONFINITE: return "non-finite value in f";
        case MT_ERR_CUDA: return "CUDA error";
        case MT_ERR_NCCL: return "NCCL error";
        case MT_ERR_STATE: return "call out of order";
        case MT_ERR_CAPACITY: return "output capacity too small";
        case MT_ERR_WORKSPACE: return "workspace missing, too small or misaligned";
    }
    return "unknown status";
}

size_t mt_workspace_bytes(const uint32_t dims[3], int conn) {
    if (!valid_dims(dims, conn)) return 0;
    const uint64_t n = uint64_t(dims[0]) * dims[1] * dims[2];
    if (n > 0xffffffffull) return 0;
    return grid_layout(dims, 0, dims[2], false).total;
}

mt_status mt_create(mt_ctx** out, const uint32_t dims[3], int conn, int cuda_device, void* workspace,
                    size_t workspace_bytes) {
    if (!dims) return MT_ERR_INVALID_ARG;
    return create_ctx(out, dims, conn, 0, dims[2], false, cuda_device, workspace, workspace_bytes);
}

size_t mt_slab_workspace_bytes(const uint32_t dims[3], int conn, uint32_t z_begin, uint32_t z_end) {
    if (!valid_dims(dims, conn) || dims[2] < 2 || z_begin >= z_end || z_end > dims[2]) return 0;
    mt::Slab v{};
    if (!n_global_fits(dims) || !wide_view(dims, z_begin, z_end, &v)) return 0;   // the slab fits 32-bit ids
    return grid_layout(dims, z_begin, z_end, true).total;
}

mt_status mt_create_slab(mt_ctx** out, const uint32_t dims[3], int conn, uint32_t z_begin, uint32_t z_end,
                         uint32_t options, int cuda_device, void* workspace, size_t workspace_bytes) {
    if (!out) return MT_ERR_INVALID_ARG;
    *out = nullptr;
    if (!dims || dims[2] < 2 || conn != 6 || z_begin >= z_end || z_end > dims[2]) return MT_ERR_INVALID_ARG;
    if (options & ~uint32_t(MT_SLAB_WIDE_IDS)) return MT_ERR_INVALID_ARG;
    return create_ctx(out, dims, conn, z_begin, z_end, true, cuda_device, workspace, workspace_bytes, nullptr,
                      options);
}

mt_status mt_set_diagram_output(mt_ctx* c, mt_pair* buf, uint64_t capacity) {
    if (!c) return MT_ERR_INVALID_ARG;
    c->reg_out = buf;
    c->reg_cap = buf ? capacity : 0;
    return MT_OK;
}

// ---- explicit graphs -----------------------------------
size_t mt_graph_workspace_bytes(uint32_t n, uint64_t n_adj) {
    return layout_for(n, n_adj, false, n ? n : 1).total;
}

mt_status mt_create_graph(mt_ctx** out, uint32_t n, uint64_t n_adj, int cuda_device, void* workspace,
                          size_t workspace_bytes) {
    if (!out) return MT_ERR_INVALID_ARG;
    const uint32_t dims[3] = {n, 1, 1};
    const Layout L = layout_for(n, n_adj, false, n ? n : 1);
    mt_status st = create_ctx(out, dims, 0, 0, 1, false, cuda_device, workspace, workspace_bytes, &L);
    if (st == MT_OK) (*out)->n_adj = n_adj;
    return st;
}

mt_status mt_compute_graph(mt_ctx* c, const float* f, const uint64_t* row, const uint32_t* col, uint64_t* T,
                           uint32_t flags, mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    if (flags & ~uint32_t(MT_FLAG_SPLIT_TREE)) return MT_ERR_INVALID_ARG;
    if (!c->graph) return MT_ERR_STATE;
    c->launches = 0;
    c->nev = 0;
    c->sticky = MT_OK;
    c->computed = true;
    if (c->n == 0) return MT_OK;
    if (!f || !row || !T) return MT_ERR_INVALID_ARG;  // col may be NULL for an edgeless graph
    DeviceGuard g(c->device);
    if (!g.ok) return MT_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    c->f = f;
    c->flip = (flags & MT_FLAG_SPLIT_TREE) ? 0xffffffffu : 0u;
    unsigned long long* ctr = counters_of(c);
    mt::Cell* cells = cells_of(c);
    unsigned long long* stats = stats_of(c);
    if (stats && cudaMemsetAsync(stats, 0, mt::ST_COUNT * sizeof(uint64_t), s) != cudaSuccess)
        return c->sticky = MT_ERR_CUDA;
    mark(c, "zero", s);
    if (cudaMemsetAsync(c->ws + c->L.counters, 0, c->L.status - c->L.counters + c->L.status_bytes,
                        s) != cudaSuccess)
        return c->sticky = MT_ERR_CUDA;
    mark(c, "graph_init", s);
    mt::launch_graph_init(f, row, col, uint32_t(c->n), c->flip, cells, ctr, c->num_sms, s);
    mark(c, "graph_edges", s);
    mt::launch_graph_edges(row, col, uint32_t(c->n), cells, nullptr, c->ws + c->L.queue, c->L.queue_cap,
                           ctr + mt::CTR_QLEN, ctr, c->num_sms, s);
    mark(c, "merge_queue", s);
    mt::launch_merge_queue(cells, c->ws + c->L.queue, c->L.queue_cap, ctr + mt::CTR_QLEN, nullptr, 0,
                           ctr + mt::CTR_QFETCH, stats, c->num_sms, s);
    c->launches = 4;
    return finish_compute(c, T, nullptr, s);
}

mt_status mt_compute(mt_ctx* c, const float* f, uint64_t* T, uint32_t flags, mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    if (flags & ~uint32_t(MT_FLAG_SPLIT_TREE)) return MT_ERR_INVALID_ARG;
    if (c->dist) {   // mt_create_dist: local phase, NCCL exchange, global phase (dist.cu)
        if (!f || !T) return MT_ERR_INVALID_ARG;
        DeviceGuard g(c->device);
        if (!g.ok) return MT_ERR_CUDA;
        const mt_status st = mt::dist_compute(c, c->dist, f, T, flags, static_cast<cudaStream_t>(stream));
        if (st != MT_OK && c->sticky == MT_OK) c->sticky = st;
        return st;
    }
    if (c->multi || c->graph) return MT_ERR_STATE;  // slab contexts use mt_compute_local / mt_compute_global
    if (c->n == 0) {
        c->computed = true;
        c->sticky = MT_OK;
        c->launches = 0;
        return MT_OK;
    }
    if (!f || !T) return MT_ERR_INVALID_ARG;
    DeviceGuard g(c->device);
    if (!g.ok) return MT_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const mt_status st = start_compute(c, f, T, flags, s);
    if (st != MT_OK) return st;
    return finish_compute(c, T, nullptr, s);
}

mt_status mt_compute_join_split(mt_ctx* cj, mt_ctx* cs, const float* f, uint64_t* T_join, uint64_t* T_split,
                                mt_stream_t stream) {
    if (!cj || !cs || cj == cs) return MT_ERR_INVALID_ARG;
    if (cj->multi || cj->graph || cj->dist || cs->multi || cs->graph || cs->dist) return MT_ERR_STATE;
    if (cj->nx != cs->nx || cj->ny != cs->ny || cj->nz != cs->nz || cj->conn != cs->conn || cj->device != cs->device)
        return MT_ERR_INVALID_ARG;
    if (cj->n == 0) {
        for (mt_ctx* c : {cj, cs}) {
            c->computed = true;
            c->sticky = MT_OK;
            c->launches = 0;
        }
        return MT_OK;
    }
    if (!f || !T_join || !T_split || T_join == T_split) return MT_ERR_INVALID_ARG;
    DeviceGuard g(cj->device);
    if (!g.ok) return MT_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    mt_status st = prepare_compute(cj, f, 0, s);
    if (st == MT_OK) st = prepare_compute(cs, f, MT_FLAG_SPLIT_TREE, s);
    if (st != MT_OK) return st;
    mark(cj, "tile_tmt", s);
    mt::launch_tile_tmt_dual(f, cells_of(cj), T_join, xface_of(cj), counters_of(cj), cells_of(cs), T_split,
                             xface_of(cs), counters_of(cs), cj->slab, stats_of(cj), s);
    cj->launches = 1;
    launch_cross(cj, T_join, s);
    launch_cross(cs, T_split, s);
    st = finish_compute(cj, T_join, nullptr, s);
    if (st != MT_OK) return st;
    return finish_compute(cs, T_split, nullptr, s);
}

size_t mt_host_staging_bytes(const mt_ctx* c) {
    if (!c || c->multi || c->graph) return 0;
    return 2 * (align_up(c->n * sizeof(float)) + align_up(c->n * sizeof(uint64_t)) +
                align_up(c->L.pairs_cap * sizeof(mt_pair)));
}

mt_status mt_compute_host(mt_ctx* c, uint32_t k, const float* const* f_hosts, uint64_t* const* T_hosts,
                          mt_pair* const* rec_hosts, uint64_t rec_cap, uint64_t* counts, uint32_t flags,
                          void* staging, size_t staging_bytes, mt_stream_t stream) {
    if (!c || (k && (!f_hosts || !T_hosts || !rec_hosts || !counts))) return MT_ERR_INVALID_ARG;
    if (c->multi || c->graph) return MT_ERR_STATE;
    if (flags & ~uint32_t(MT_FLAG_SPLIT_TREE)) return MT_ERR_INVALID_ARG;
    if (k == 0) return MT_OK;
    if (!staging || staging_bytes < mt_host_staging_bytes(c) || reinterpret_cast<uintptr_t>(staging) % ALIGN)
        return MT_ERR_WORKSPACE;
    DeviceGuard g(c->device);
    if (!g.ok) return MT_ERR_CUDA;
    if (!c->hs[0]) {
        for (cudaStream_t& st : c->hs)
            if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return MT_ERR_CUDA;
        for (cudaEvent_t& e : c->hev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return MT_ERR_CUDA;
    }
    cudaStream_t s_h2d = c->hs[0], s_comp = c->hs[1], s_d2h = c->hs[2];
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    // the pipeline starts after the work already on the caller's stream and the caller's stream
    // continues after the pipeline (events recorded on it bracket the whole host->host run)
    if (cudaEventRecord(c->hev[0], caller) != cudaSuccess) return MT_ERR_CUDA;
    for (cudaStream_t sx : c->hs)
        if (cudaStreamWaitEvent(sx, c->hev[0], 0) != cudaSuccess) return MT_ERR_CUDA;
    cudaEvent_t* h2d_done = c->hev;          // [2]
    cudaEvent_t* comp_done = c->hev + 2;     // [2]
    cudaEvent_t* d2h_done = c->hev + 4;      // [2]
    // double-buffered device staging: f, T, diagram records (the registered diagram output)
    char* p = static_cast<char*>(staging);
    float* f_dev[2];
    uint64_t* T_dev[2];
    mt_pair* r_dev[2];
    for (int b = 0; b < 2; ++b) {
        f_dev[b] = reinterpret_cast<float*>(p);
        p += align_up(c->n * sizeof(float));
        T_dev[b] = reinterpret_cast<uint64_t*>(p);
        p += align_up(c->n * sizeof(uint64_t));
        r_dev[b] = reinterpret_cast<mt_pair*>(p);
        p += align_up(c->L.pairs_cap * sizeof(mt_pair));
    }
    mt_pair* const saved_out = c->reg_out;
    const uint64_t saved_cap = c->reg_cap;
    for (int b = 0; b < 2; ++b)
        if (cudaEventRecord(comp_done[b], s_comp) != cudaSuccess || cudaEventRecord(d2h_done[b], s_comp) != cudaSuccess)
            return MT_ERR_CUDA;
    auto h2d = [&](uint32_t i) {   // field i into f_dev[i % 2] once compute i-2 stopped reading it
        const int b = int(i % 2);
        return cudaStreamWaitEvent(s_h2d, comp_done[b], 0) == cudaSuccess &&
               cudaMemcpyAsync(f_dev[b], f_hosts[i], c->n * sizeof(float), cudaMemcpyHostToDevice, s_h2d) ==
                   cudaSuccess &&
               cudaEventRecord(h2d_done[b], s_h2d) == cudaSuccess;
    };
    mt_status st = MT_OK;
    if (!h2d(0)) st = MT_ERR_CUDA;
    for (uint32_t i = 0; i < k && st == MT_OK; ++i) {
        const int b = int(i % 2);
        if (cudaStreamWaitEvent(s_comp, h2d_done[b], 0) != cudaSuccess ||
            cudaStreamWaitEvent(s_comp, d2h_done[b], 0) != cudaSuccess) {
            st = MT_ERR_CUDA;
            break;
        }
        c->reg_out = r_dev[b];
        c->reg_cap = c->L.pairs_cap;
        st = mt_compute(c, f_dev[b], T_dev[b], flags, s_comp);
        if (st != MT_OK) break;
        if (cudaEventRecord(comp_done[b], s_comp) != cudaSuccess) { st = MT_ERR_CUDA; break; }
        if (i + 1 < k && !h2d(i + 1)) { st = MT_ERR_CUDA; break; }   // overlaps compute i
        uint64_t np = 0, ne = 0;
        st = mt_diagram(c, nullptr, 0, &np, &ne, s_comp);              // waits for compute i
        if (st != MT_OK) break;
        counts[2 * i] = np;
        counts[2 * i + 1] = ne;
        if (np + ne > rec_cap) { st = MT_ERR_CAPACITY; break; }
        if (cudaStreamWaitEvent(s_d2h, comp_done[b], 0) != cudaSuccess ||
            cudaMemcpyAsync(T_hosts[i], T_dev[b], c->n * sizeof(uint64_t), cudaMemcpyDeviceToHost, s_d2h) !=
                cudaSuccess ||
            (np + ne && cudaMemcpyAsync(rec_hosts[i], r_dev[b], (np + ne) * sizeof(mt_pair), cudaMemcpyDeviceToHost,
                                        s_d2h) != cudaSuccess) ||
            cudaEventRecord(d2h_done[b], s_d2h) != cudaSuccess)   // overlaps compute i + 1
            st = MT_ERR_CUDA;
    }
    for (int j = 0; j < 3; ++j)
        if ((cudaEventRecord(c->hev[j], c->hs[j]) != cudaSuccess ||
             cudaStreamWaitEvent(caller, c->hev[j], 0) != cudaSuccess) && st == MT_OK)
            st = MT_ERR_CUDA;
    if (cudaStreamSynchronize(caller) != cudaSuccess && st == MT_OK) st = MT_ERR_CUDA;
    c->reg_out = saved_out;
    c->reg_cap = saved_cap;
    return st;
}

mt_status mt_compute_local(mt_ctx* c, const float* f, uint64_t* T, uint32_t flags, mt_stream_t stream) {
    if (!c || !f || !T) return MT_ERR_INVALID_ARG;
    if (flags & ~uint32_t(MT_FLAG_SPLIT_TREE)) return MT_ERR_INVALID_ARG;
    if (!c->multi) return MT_ERR_STATE;
    DeviceGuard g(c->device);
    if (!g.ok) return MT_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint8_t* flag = reinterpret_cast<uint8_t*>(c->ws + c->L.flags);
    if (cudaMemsetAsync(flag, 0, c->n, s) != cudaSuccess) return c->sticky = MT_ERR_CUDA;
    mt_status st = start_compute(c, f, T, flags, s);
    if (st != MT_OK) return st;
    c->local_T = T;
    const bool has_bottom = c->z_begin > 0, has_top = c->z_end < c->nz;
    mark(c, "forest_mark", s);
    mt::launch_forest_mark(cells_of(c), T - c->slab.base, c->slab, has_bottom, has_top, flag, s);
    mark(c, "forest_compact", s);
    mt_forest_record* recs = reinterpret_cast<mt_forest_record*>(c->ws + c->L.recs);
    unsigned long long* fcount = counters_of(c) + mt::CTR_FCOUNT;
    c->launches += 1 + mt::launch_forest_compact(cells_of(c), T - c->slab.base, f - c->slab.base, c->slab, flag, recs,
                                                 c->L.recs_cap, fcount, has_bottom, has_top, c->num_sms, s);
    if (c->wide) {   // the flags are dead after the compaction: their space holds the bitmap
        mark(c, "forest_compress", s);
        const uint64_t sxy = uint64_t(c->nx) * c->ny;
        // the top face moves to the end of the compressed range (a one-plane slab's only plane is
        // its bottom face too and keeps compressed ids 0 .. nx ny - 1)
        c->launches += mt::launch_forest_compress(recs, fcount, c->n, has_top && c->n > sxy ? c->n - sxy : ~0ull,
                                                  flag, c->num_sms, s);
    }
    mark(c, "exchange", s);  // closes at mt_compute_global's first mark: host sync + all-gather
    c->local_done = true;
    if (cudaGetLastError() != cudaSuccess) return c->sticky = MT_ERR_CUDA;
    return MT_OK;
}

mt_status mt_forest_view(mt_ctx* c, const mt_forest_record** records, uint64_t* n_records, mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    if (!c->multi || !c->local_done) return MT_ERR_STATE;
    DeviceGuard g(c->device);
    const mt_status st = sync_counters(c, static_cast<cudaStream_t>(stream));
    if (st == MT_ERR_CUDA || st == MT_ERR_STATE) return st;
    const uint64_t n = c->host_ctr[mt::CTR_FCOUNT];
    if (n_records) *n_records = n;
    if (records) *records = reinterpret_cast<const mt_forest_record*>(c->ws + c->L.recs);
    if (n > c->L.recs_cap) return MT_ERR_CAPACITY;
    return st;
}

// id tables (2) | merged cells | queue of deduplicated inter-slab edges (every face vertex of a
// boundary has a record, so a boundary's nx ny edges are at most half of the records)
// + the view id of each record and (wide mode) the global id of every remote view id (at most
// 2 per record)
size_t mt_forest_scratch_bytes(uint64_t n_all) {
    const uint64_t t = mt::forest_table_size(n_all);
    if (t == 0) return 0;
    return 2 * align_up(size_t(t) * sizeof(uint64_t)) + align_up(n_all * sizeof(mt::Cell)) +
           align_up((n_all / 2 + 1) * mt::forest_queue_entry_bytes()) + align_up(n_all * sizeof(uint32_t)) +
           align_up(2 * n_all * sizeof(uint64_t));
}

mt_status mt_compute_global(mt_ctx* c, const mt_forest_record* all, const uint64_t* counts, const uint32_t* z_bounds,
                            uint32_t nslabs, void* scratch, size_t scratch_bytes, uint64_t* T, mt_stream_t stream) {
    if (!c || !z_bounds || !counts || !T) return MT_ERR_INVALID_ARG;
    if (!c->multi || !c->local_done) return MT_ERR_STATE;
    if (T != c->local_T) return MT_ERR_INVALID_ARG;   // the buffer holding mt_compute_local's tile store
    if (nslabs < 1 || nslabs > uint32_t(mt::MAX_SLABS) || z_bounds[0] != 0 || z_bounds[nslabs] != c->nz)
        return MT_ERR_INVALID_ARG;
    uint32_t self = nslabs;
    uint64_t n_all = 0;
    for (uint32_t k = 0; k < nslabs; ++k) {
        if (z_bounds[k] >= z_bounds[k + 1]) return MT_ERR_INVALID_ARG;
        if (z_bounds[k] == c->z_begin && z_bounds[k + 1] == c->z_end) self = k;
        n_all += counts[k];
    }
    if (self == nslabs) return MT_ERR_INVALID_ARG;
    if (n_all && !all) return MT_ERR_INVALID_ARG;
    if (n_all > 0xffffffffull || mt::forest_table_size(n_all) == 0) return MT_ERR_TOO_LARGE;
    if (!scratch || scratch_bytes < mt_forest_scratch_bytes(n_all) || reinterpret_cast<uintptr_t>(scratch) % ALIGN)
        return MT_ERR_WORKSPACE;
    // this rank's view of every slab's ids (slab.cu header)
    const uint64_t sxy = uint64_t(c->nx) * c->ny;
    mt::ForestXlate X{};
    X.nslabs = nslabs;
    X.self = self;
    X.flip = c->flip;
    X.wide = c->wide;
    uint64_t span[mt::MAX_SLABS];
    for (uint32_t k = 0; k < nslabs; ++k) {
        X.rec_off[k + 1] = X.rec_off[k] + counts[k];
        X.real_base[k] = uint64_t(z_bounds[k]) * sxy;
        span[k] = k == self ? c->n : c->wide ? 2 * counts[k] : uint64_t(z_bounds[k + 1] - z_bounds[k]) * sxy;
    }
    if (c->wide) {
        const uint64_t own = c->slab.base;
        uint64_t below = 0, above = 0;
        for (uint32_t k = 0; k < self; ++k) below += span[k];
        for (uint32_t k = self + 1; k < nslabs; ++k) above += span[k];
        if (below > own || own + c->n + above > 0xffffffffull) return MT_ERR_TOO_LARGE;
        uint64_t at = own - below;
        for (uint32_t k = 0; k < nslabs; ++k) {
            X.voff[k] = uint32_t(at);
            at += span[k];
        }
        X.dec_lo = X.voff[0];
        X.own_lo = uint32_t(own);
        X.own_n = c->n;
    } else {
        for (uint32_t k = 0; k < nslabs; ++k) X.voff[k] = uint32_t(X.real_base[k]);
    }
    uint32_t a0[mt::MAX_SLABS], b0[mt::MAX_SLABS], ia0[mt::MAX_SLABS], ib0[mt::MAX_SLABS];
    for (uint32_t k = 0; k + 1 < nslabs; ++k) {   // the faces of boundary k in the view
        const bool one_plane = z_bounds[k + 1] - z_bounds[k] == 1;   // its top face is its bottom face
        a0[k] = uint32_t(one_plane ? X.voff[k] : X.voff[k] + span[k] - sxy);
        b0[k] = X.voff[k + 1];
        // their records' fixed slots (forest_compact): slab k's top face after its bottom face
        // (none for slab 0; a one-plane slab has one face region), slab k + 1's bottom face first
        ia0[k] = uint32_t(X.rec_off[k] + ((k > 0 && !one_plane) ? sxy : 0));
        ib0[k] = uint32_t(X.rec_off[k + 1]);
    }
    DeviceGuard g(c->device);
    if (!g.ok) return MT_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t tsize = uint32_t(mt::forest_table_size(n_all));
    char* p = static_cast<char*>(scratch);
    uint64_t* table = reinterpret_cast<uint64_t*>(p);
    uint64_t* vtable = reinterpret_cast<uint64_t*>(p + align_up(size_t(tsize) * 8));
    p += 2 * align_up(size_t(tsize) * 8);
    mt::Cell* fcells = reinterpret_cast<mt::Cell*>(p);
    p += align_up(n_all * sizeof(mt::Cell));
    void* fqueue = p;
    p += align_up((n_all / 2 + 1) * mt::forest_queue_entry_bytes());
    uint32_t* vid = reinterpret_cast<uint32_t*>(p);
    p += align_up(n_all * sizeof(uint32_t));
    uint64_t* dec = reinterpret_cast<uint64_t*>(p);
    mt::ForestRef F{table, vtable, tsize - 1, fcells, all, vid, counters_of(c) + mt::CTR_ERR};
    mark(c, "forest_build", s);
    if (cudaMemsetAsync(table, 0xff, 2 * align_up(size_t(tsize) * 8), s) != cudaSuccess)
        return c->sticky = MT_ERR_CUDA;
    mt::launch_forest_build(all, n_all, X, table, vtable, tsize - 1, fcells, vid, dec, c->num_sms, s);
    mark(c, "forest_merge", s);
    mt::launch_forest_merge(F, c->slab, nslabs, a0, b0, ia0, ib0, fqueue, counters_of(c) + mt::CTR_FQLEN,
                            counters_of(c) + mt::CTR_FFETCH, c->num_sms, s);
    mark(c, "forest_writeback", s);
    mt::launch_forest_writeback(F, n_all, cells_of(c), T - c->slab.base, c->slab, c->num_sms, s);
    c->launches += 3;
    c->local_done = false;
    c->decode = mt::IdDecode{c->wide, X.dec_lo, X.own_lo, X.own_n, c->gid0, dec};
    c->decode_ok = true;
    return finish_compute(c, T, &F, s);
}

mt_status mt_diagram(mt_ctx* c, mt_pair* out, uint64_t capacity, uint64_t* n_pairs, uint64_t* n_essential,
                     mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    if (c->wide) return MT_ERR_TOO_LARGE;   // view ids: mt_diagram64
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const mt_status st = sync_counters(c, s);
    if (st == MT_ERR_STATE || st == MT_ERR_CUDA) return st;
    const uint64_t nfin = c->host_ctr[mt::CTR_FIN], ness = c->host_ctr[mt::CTR_ESS];
    if (n_pairs) *n_pairs = nfin;
    if (n_essential) *n_essential = ness;
    if (st != MT_OK) return st;
    uint64_t cap = 0;
    mt_pair* src = target_of(c, &cap);
    if (out && out != src && nfin + ness) {
        if (capacity < nfin + ness) return MT_ERR_CAPACITY;
        if (cudaMemcpyAsync(out, src, (nfin + ness) * sizeof(mt_pair), cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return c->sticky = MT_ERR_CUDA;
    } else if (out == src && out && capacity < nfin + ness) {
        return MT_ERR_CAPACITY;
    }
    return MT_OK;
}

mt_status mt_diagram_view(mt_ctx* c, const mt_pair** records, uint64_t* n_pairs, uint64_t* n_essential,
                          mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    if (c->wide) return MT_ERR_TOO_LARGE;
    DeviceGuard g(c->device);
    const mt_status st = sync_counters(c, static_cast<cudaStream_t>(stream));
    if (st == MT_ERR_STATE || st == MT_ERR_CUDA) return st;
    if (n_pairs) *n_pairs = c->host_ctr[mt::CTR_FIN];
    if (n_essential) *n_essential = c->host_ctr[mt::CTR_ESS];
    uint64_t cap = 0;
    if (records) *records = target_of(c, &cap);
    return st;
}

mt_status mt_triplets64(mt_ctx* c, const uint64_t* T, uint64_t first, uint64_t count, mt_triplet64* out,
                        mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    if (!c->computed || !c->decode_ok || c->local_done) return MT_ERR_STATE;
    if (first > c->n || count > c->n - first) return MT_ERR_INVALID_ARG;
    if (count == 0) return MT_OK;
    if (!T || !out) return MT_ERR_INVALID_ARG;
    DeviceGuard g(c->device);
    if (!g.ok) return MT_ERR_CUDA;
    mt::launch_triplets64(T + first, count, c->decode, out, c->num_sms, static_cast<cudaStream_t>(stream));
    return cudaGetLastError() == cudaSuccess ? MT_OK : MT_ERR_CUDA;
}

mt_status mt_diagram64(mt_ctx* c, mt_pair64* out, uint64_t capacity, uint64_t* n_pairs, uint64_t* n_essential,
                       mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const mt_status st = sync_counters(c, s);
    if (st == MT_ERR_STATE || st == MT_ERR_CUDA) return st;
    if (!c->decode_ok || c->local_done) return MT_ERR_STATE;
    const uint64_t nfin = c->host_ctr[mt::CTR_FIN], ness = c->host_ctr[mt::CTR_ESS];
    if (n_pairs) *n_pairs = nfin;
    if (n_essential) *n_essential = ness;
    if (st != MT_OK || !out || nfin + ness == 0) return st;
    if (capacity < nfin + ness) return MT_ERR_CAPACITY;
    uint64_t cap = 0;
    const mt_pair* src = target_of(c, &cap);
    mt::launch_pairs64(src, nfin + ness, c->decode, out, c->num_sms, s);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) return c->sticky = MT_ERR_CUDA;
    return MT_OK;
}

mt_status mt_last_error(mt_ctx* c, mt_stream_t stream) {
    if (!c) return MT_ERR_INVALID_ARG;
    if (!c->computed) return MT_OK;
    DeviceGuard g(c->device);
    return sync_counters(c, static_cast<cudaStream_t>(stream));
}

mt_status mt_filter_diagram(mt_ctx* c, float eps, mt_pair* out, uint64_t capacity, uint64_t* n_pairs_kept,
                            uint64_t* n_essential, mt_stream_t stream) {
    if (!c || !(eps >= 0.f)) return MT_ERR_INVALID_ARG;
    if (c->wide) return MT_ERR_TOO_LARGE;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const mt_status st = sync_counters(c, s);
    if (st != MT_OK) return st;
    const uint64_t nfin = c->host_ctr[mt::CTR_FIN], ness = c->host_ctr[mt::CTR_ESS];
    const uint64_t n_all = nfin + ness;
    uint64_t kept = 0;
    if (n_all) {
        if (!out) return MT_ERR_INVALID_ARG;
        uint64_t cap = 0;
        const mt_pair* src = target_of(c, &cap);
        if (out == src) return MT_ERR_INVALID_ARG;  // not in place
        unsigned long long* ctl = counters_of(c) + mt::CTR_FILT_TICKET;
        uint64_t* status = reinterpret_cast<uint64_t*>(c->ws + c->L.status);  // free after the repair
        if (mt::filter_tiles(n_all) * sizeof(uint64_t) > c->L.status_bytes) return MT_ERR_STATE;
        if (cudaMemsetAsync(ctl, 0, 2 * sizeof(uint64_t), s) != cudaSuccess ||
            cudaMemsetAsync(status, 0, mt::filter_tiles(n_all) * sizeof(uint64_t), s) != cudaSuccess)
            return MT_ERR_CUDA;
        mt::launch_filter_diagram(src, nfin, n_all, eps, out, capacity, ctl, status, s);
        uint64_t host = 0;
        if (cudaMemcpyAsync(&host, ctl + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return MT_ERR_CUDA;
        kept = host;
    }
    if (n_pairs_kept) *n_pairs_kept = kept - ness;
    if (n_essential) *n_essential = ness;
    return kept > capacity ? MT_ERR_CAPACITY : MT_OK;
}

uint32_t mt_last_launch_count(const mt_ctx* c) { return c ? c->launches : 0; }

mt_status mt_set_profiling(mt_ctx* c, int enable) {
    if (!c) return MT_ERR_INVALID_ARG;
    c->profiling = enable != 0;
    return MT_OK;
}

int mt_kernel_times(mt_ctx* c, const char** names, float* ms, int max) {
    if (!c || !c->profiling || c->nev == 0) return 0;
    DeviceGuard g(c->device);
    if (cudaEventSynchronize(c->ev[c->nev]) != cudaSuccess) return 0;
    int k = 0;
    for (int i = 0; i < c->nev && k < max; ++i, ++k) {
        float t = 0.f;
        cudaEventElapsedTime(&t, c->ev[i], c->ev[i + 1]);
        if (names) names[k] = c->ev_name[i];
        if (ms) ms[k] = t;
    }
    return k;
}

mt_status mt_set_stats(mt_ctx* c, int enable) {
    if (!c) return MT_ERR_INVALID_ARG;
    c->stats = enable != 0;
    return MT_OK;
}

int mt_stats(mt_ctx* c, uint64_t* out, int max, mt_stream_t stream) {
    if (!c || !out || !c->stats || !c->computed || c->n == 0) return 0;
    DeviceGuard g(c->device);
    const int k = max < int(mt::ST_COUNT) ? max : int(mt::ST_COUNT);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(out, c->ws + c->L.stats, k * sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return 0;
    return k;
}

void mt_destroy(mt_ctx* c) {
    if (!c) return;
    DeviceGuard g(c->device);
    mt::dist_destroy(c->dist);
    for (cudaStream_t& st : c->hs)
        if (st) cudaStreamDestroy(st);
    for (cudaEvent_t& e : c->hev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i <= MAX_EVENTS; ++i)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    if (c->host_ctr) cudaFreeHost(c->host_ctr);
    delete c;
}

}  // extern "C"
