// dist.cu -- the multi-GPU z-slab path with its exchange inside the library
// (distribution is the paper's stated future work,
// "distributed ... 64-bit ... across multiple nodes").
//
// One process per GPU.  mt_create_dist builds a slab context (mt_create_slab)
// for the rank's planes and an NCCL communicator from a unique id that rank 0
// made with mt_get_unique_id and the caller broadcast.  mt_compute on such a
// context runs, on the caller's stream:
//   mt_compute_local  (the slab's merge tree + its boundary forest, kernels)
//   ncclAllGather     (every rank's forest record count, 8 B each)
//   one host sync     (the counts size the exact-length exchange below)
//   ncclBroadcast x P (grouped: each rank's records, exact length, into one
//                      contiguous array in rank order -- no padding; in wide
//                      mode the records carry compressed ids, slab.cu)
//   mt_compute_global (forest merge, write-back, repair, diagram: kernels)
// so a rank calls mt_compute / mt_diagram exactly as on one GPU.  NCCL is
// loaded at run time (dlopen of libnccl.so.2; the copy torch already loaded
// is reused when present), so libmt_b200.so has no link-time NCCL dependency
// and loads on hosts without it; only mt_get_unique_id / mt_create_dist need
// it.  The gathered records and the forest tables live in device buffers the
// context owns and grows on demand (a steady-state step allocates nothing).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "kernels.cuh"
#include "mt.h"

namespace mt {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the process's copy (torch's)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.Broadcast && api.GroupStart &&
                 api.GroupEnd && api.CommDestroy;
    });
    return api;
}

constexpr size_t RECORD = sizeof(mt_forest_record);

}  // namespace

struct DistState {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    std::vector<uint32_t> bounds;       // nranks + 1 plane boundaries
    uint64_t* counts_dev = nullptr;     // nranks record counts (device)
    uint64_t* counts_host = nullptr;    // pinned
    char* gather = nullptr;             // every rank's records, rank order
    size_t gather_cap = 0;
    char* scratch = nullptr;            // forest tables of mt_compute_global
    size_t scratch_cap = 0;
};

// z boundaries of the slabs: as equal as possible, on multiples of the tile depth when the
// grid allows it (the cut faces are then tile faces), every slab at least one plane
bool slab_bounds(uint32_t nz, int nranks, uint32_t* b) {
    if (nranks < 1 || nranks > MAX_SLABS || uint32_t(nranks) > nz) return false;
    uint32_t ty = 0, tz = 0;
    tile_shape(nz, &ty, &tz);
    const uint64_t P = uint64_t(nranks), align = nz >= P * tz ? tz : 1;
    b[0] = 0;
    for (uint64_t k = 1; k < P; ++k) {
        uint64_t z = (2 * k * nz + P * align) / (2 * P * align) * align;   // round half up
        if (z < uint64_t(b[k - 1]) + 1) z = b[k - 1] + 1;
        if (z > nz - (P - k)) z = nz - (P - k);
        b[k] = uint32_t(z);
    }
    b[P] = nz;
    return true;
}

static mt_status grow(char** buf, size_t* cap, size_t need) {
    if (need <= *cap) return MT_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    if (cudaMalloc(reinterpret_cast<void**>(buf), need + need / 8) != cudaSuccess) return MT_ERR_CUDA;
    *cap = need + need / 8;
    return MT_OK;
}

void dist_destroy(DistState* d) {
    if (!d) return;
    if (d->comm && nccl().ok) nccl().CommDestroy(d->comm);
    if (d->counts_dev) cudaFree(d->counts_dev);
    if (d->counts_host) cudaFreeHost(d->counts_host);
    if (d->gather) cudaFree(d->gather);
    if (d->scratch) cudaFree(d->scratch);
    delete d;
}

// ctx accessors implemented in mt_api.cu
void slab_forest(mt_ctx* c, mt_forest_record** recs, unsigned long long** count_dev, uint64_t* cap);
void attach_dist(mt_ctx* c, DistState* d);

mt_status dist_compute(mt_ctx* c, DistState* d, const float* f, uint64_t* T, uint32_t flags, cudaStream_t s) {
    const NcclApi& N = nccl();
    if (!N.ok) return MT_ERR_NCCL;
    mt_status st = mt_compute_local(c, f, T, flags, s);
    if (st != MT_OK) return st;
    mt_forest_record* recs = nullptr;
    unsigned long long* count_dev = nullptr;
    uint64_t cap = 0;
    slab_forest(c, &recs, &count_dev, &cap);
    if (N.AllGather(count_dev, d->counts_dev, 1, ncclUint64, d->comm, s) != ncclSuccess) return MT_ERR_NCCL;
    if (cudaMemcpyAsync(d->counts_host, d->counts_dev, size_t(d->nranks) * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                        s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return MT_ERR_CUDA;
    std::vector<uint64_t> off(size_t(d->nranks) + 1, 0);
    (void)cap;   // forest_compact never counts past its capacity (the slab's n vertices)
    for (int r = 0; r < d->nranks; ++r) off[r + 1] = off[r] + d->counts_host[r];
    const uint64_t n_all = off[d->nranks];
    if ((st = grow(&d->gather, &d->gather_cap, size_t(n_all) * RECORD + 256)) != MT_OK) return st;
    const size_t need = mt_forest_scratch_bytes(n_all);
    if (need == 0) return MT_ERR_TOO_LARGE;
    if ((st = grow(&d->scratch, &d->scratch_cap, need + 256)) != MT_OK) return st;
    if (N.GroupStart() != ncclSuccess) return MT_ERR_NCCL;
    ncclResult_t nr = ncclSuccess;
    for (int r = 0; r < d->nranks && nr == ncclSuccess; ++r) {
        if (!d->counts_host[r]) continue;
        char* dst = d->gather + off[r] * RECORD;
        const void* src = r == d->rank ? static_cast<const void*>(recs) : dst;
        nr = N.Broadcast(src, dst, size_t(d->counts_host[r]) * (RECORD / 8), ncclUint64, r, d->comm, s);
    }
    if (N.GroupEnd() != ncclSuccess || nr != ncclSuccess) return MT_ERR_NCCL;
    char* sp = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(d->scratch) + 255) / 256 * 256);
    return mt_compute_global(c, reinterpret_cast<const mt_forest_record*>(d->gather), d->counts_host,
                             d->bounds.data(), uint32_t(d->nranks), sp, need, T, s);
}

}  // namespace mt

extern "C" {

mt_status mt_get_unique_id(uint8_t id[128]) {
    if (!id) return MT_ERR_INVALID_ARG;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    const mt::NcclApi& N = mt::nccl();
    if (!N.ok) return MT_ERR_NCCL;
    ncclUniqueId u;
    if (N.GetUniqueId(&u) != ncclSuccess) return MT_ERR_NCCL;
    memcpy(id, &u, sizeof(u));
    return MT_OK;
}

mt_status mt_dist_slab_bounds(uint32_t nz, int nranks, uint32_t* bounds) {
    if (!bounds) return MT_ERR_INVALID_ARG;
    return mt::slab_bounds(nz, nranks, bounds) ? MT_OK : MT_ERR_INVALID_ARG;
}

size_t mt_dist_workspace_bytes(const uint32_t global_dims[3], int conn, int rank, int nranks) {
    if (!global_dims || rank < 0 || rank >= nranks) return 0;
    uint32_t b[mt::MAX_SLABS + 1];
    if (!mt::slab_bounds(global_dims[2], nranks, b)) return 0;
    return mt_slab_workspace_bytes(global_dims, conn, b[rank], b[rank + 1]);
}

mt_status mt_create_dist(mt_ctx** out, const uint32_t global_dims[3], int conn, int rank, int nranks,
                         const uint8_t nccl_id[128], uint32_t options, int cuda_device, void* workspace,
                         size_t workspace_bytes) {
    if (!out) return MT_ERR_INVALID_ARG;
    *out = nullptr;
    if (!global_dims || !nccl_id || rank < 0 || rank >= nranks) return MT_ERR_INVALID_ARG;
    uint32_t b[mt::MAX_SLABS + 1];
    if (!mt::slab_bounds(global_dims[2], nranks, b)) return MT_ERR_INVALID_ARG;
    const mt::NcclApi& N = mt::nccl();
    if (!N.ok) return MT_ERR_NCCL;
    mt_ctx* c = nullptr;
    mt_status st = mt_create_slab(&c, global_dims, conn, b[rank], b[rank + 1], options, cuda_device, workspace,
                                  workspace_bytes);
    if (st != MT_OK) return st;
    mt::DistState* d = new (std::nothrow) mt::DistState();
    if (!d) {
        mt_destroy(c);
        return MT_ERR_CUDA;
    }
    d->rank = rank;
    d->nranks = nranks;
    d->bounds.assign(b, b + nranks + 1);
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(cuda_device);
    ncclUniqueId u;
    memcpy(&u, nccl_id, sizeof(u));
    if (cudaMalloc(reinterpret_cast<void**>(&d->counts_dev), size_t(nranks) * sizeof(uint64_t)) != cudaSuccess ||
        cudaMallocHost(reinterpret_cast<void**>(&d->counts_host), size_t(nranks) * sizeof(uint64_t)) !=
            cudaSuccess)
        st = MT_ERR_CUDA;
    else if (N.CommInitRank(&d->comm, nranks, u, rank) != ncclSuccess)
        st = MT_ERR_NCCL;
    if (prev >= 0) cudaSetDevice(prev);
    if (st != MT_OK) {
        d->comm = nullptr;
        mt::dist_destroy(d);
        mt_destroy(c);
        return st;
    }
    mt::attach_dist(c, d);
    *out = c;
    return MT_OK;
}

}  // extern "C"
