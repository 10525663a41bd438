/*
 * mt.h -- C ABI of the B200-native triplet merge tree + 0-dimensional
 * persistence diagram library (libmt_b200.so).  arXiv 2301.10838.
 *
 * Problem (PAPER.md = the paper's text):
 *   f : V -> R on the vertices of a grid graph G = (V, E) ("we connect
 *   neighboring grid points, obtaining a graph with the function defined on
 *   its vertices"; "f : V -> R").
 *   Output 1 -- the merge tree as the normalized, minimal triplet map
 *   T[u] = (s, v): one triplet (u, s, v) per vertex u with
 *   f(v) < f(u) <= f(s), u and v in one component of G_{f(s)}, v the deepest
 *   vertex of that component; (u, u, u) for the minimum of a component.
 *   Output 2 -- the 0-dimensional persistence diagram, "one point per branch
 *   (a, b) of the merge tree": a pair (f(u), f(s)) for every
 *   triplet with s != u, and one essential class (f(m), +inf) per component.
 *
 * Readings fixed for both this library and the oracle:
 *   R1 ties in f are broken by vertex id (lexicographic (value, id) order);
 *   R2 -0.0 and +0.0 are equal values;  R3 NaN/+-Inf are rejected;
 *   R9/R10 grid: 4-connectivity in 2D (nz = 1), 6-connectivity in 3D, no
 *   periodic faces, ids x fastest: id = x + nx * (y + ny * z);
 *   R11 packed cell = (uint64)s << 32 | v ("a pair can be packed into a 64-bit
 *   integer"; s in the high half);
 *   R14 diagram values are copied from the input f (also for the split tree);
 *   R16 split tree = merge tree of -f with the id tie break unchanged.
 *
 * Conventions: every data pointer is a DEVICE pointer unless marked (host).
 * The caller owns all memory (static, pre-sized device
 * buffers; the library never allocates on the hot path).  No call throws;
 * every call returns mt_status.  Data errors found on the device (non-finite
 * input, output capacity) are sticky and reported by the next syncing call
 * (mt_diagram, mt_last_error).  A context is bound to one device and is not
 * thread-safe; calls on one context must be issued from one host thread.
 */
#ifndef MT_B200_H
#define MT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mt_ctx mt_ctx; /* opaque */
typedef void *mt_stream_t;    /* a cudaStream_t (0 = legacy default stream) */

typedef enum {
    MT_OK = 0,
    MT_ERR_INVALID_ARG = 1, /* NULL pointer, conn not in {4,6}, conn 4 with nz != 1, bad rank */
    MT_ERR_TOO_LARGE = 2,   /* ids past 32 bits where they must fit (one GPU: nx*ny*nz <= 2^32 - 1) */
    MT_ERR_NONFINITE = 3,   /* NaN or +-Inf in f (reading R3); sticky */
    MT_ERR_CUDA = 4,        /* a CUDA runtime call failed */
    MT_ERR_NCCL = 5,        /* NCCL missing or an NCCL call failed (mt_create_dist contexts) */
    MT_ERR_STATE = 6,       /* call out of order, e.g. mt_diagram before mt_compute */
    MT_ERR_CAPACITY = 7,    /* output buffer too small; required count returned */
    MT_ERR_WORKSPACE = 8    /* workspace NULL, too small or misaligned (needs 256 B) */
} mt_status;

enum { MT_FLAG_SPLIT_TREE = 1u }; /* merge tree of -f (split tree) */

/* One diagram point, 16 bytes.  Finite pair: birth_v = the minimum u,
 * death_v = the saddle s, birth = f[u], death = f[s].  Essential class:
 * death_v = birth_v = the component minimum, death = +INFINITY. */
typedef struct {
    uint32_t birth_v, death_v;
    float birth, death;
} mt_pair;

/* Bytes of device workspace mt_create needs for grid dims[3] = {nx,ny,nz}
 * (host array) and connectivity conn.  0 on invalid arguments. */
size_t mt_workspace_bytes(const uint32_t dims[3], int conn);

/* Create a context for an nx*ny*nz grid (host dims; 2D: nz = 1) on CUDA
 * device `cuda_device`.  `workspace` (device, >= mt_workspace_bytes, 256-B
 * aligned) stays owned by the caller and must outlive the context.
 * n = 0 is allowed (every compute is empty).  On error *out is set to NULL. */
mt_status mt_create(mt_ctx **out, const uint32_t dims[3], int conn, int cuda_device,
                    void *workspace, size_t workspace_bytes);

/* Compute the merge tree of f (device, n float32, x fastest; borrowed until
 * the stream reaches the end of this call's work) into `triplets` (device,
 * n uint64, written: the normalized minimal store T[u] = s << 32 | v; it also
 * holds the tile store between the tile and repair kernels), and the
 * persistence diagram into the context (see mt_diagram).  Asynchronous on
 * `stream`: kernels only, no host synchronisation, no allocation.
 * flags: 0 or MT_FLAG_SPLIT_TREE.
 * Steps: keys (value, id) -> steepest-descent init with
 * tile-local descent -> concurrent CAS edge merge (Alg. 3) -> repair by
 * representatives (Alg. 4/5) fused with the ordered diagram compaction. */
mt_status mt_compute(mt_ctx *ctx, const float *f, uint64_t *triplets, uint32_t flags,
                     mt_stream_t stream);

/* End to end from host memory (the e2e path): k fields f_hosts[i] (host, n
 * float32; pinned for overlap) in, their triplet stores T_hosts[i] (host, n
 * uint64) and diagrams rec_hosts[i] (host, rec_cap records each) out, counts
 * (host, 2k: n_pairs, n_essential per field).  Three streams the context
 * creates at first use overlap, step by step, the host->device copy of field
 * i+1, the computation of field i and the device->host copies of field i-1;
 * `staging` (device, >= mt_host_staging_bytes, 256-B aligned, caller-owned)
 * holds the double-buffered device copies.  The pipeline starts after the work
 * already queued on `stream` and `stream` waits for the pipeline, so events the
 * caller records on it around the call bracket the whole host->host run.
 * Synchronous: returns when every output is in host memory.  MT_ERR_CAPACITY
 * when a diagram exceeds rec_cap. */
size_t mt_host_staging_bytes(const mt_ctx *ctx);
mt_status mt_compute_host(mt_ctx *ctx, uint32_t k, const float *const *f_hosts, uint64_t *const *T_hosts,
                          mt_pair *const *rec_hosts, uint64_t rec_cap, uint64_t *counts, uint32_t flags,
                          void *staging, size_t staging_bytes, mt_stream_t stream);

/* Both trees of one field from ONE read of f (the join and
 * split trees are the two inputs of a contour tree; the paper
 * computes the split tree of its densities): ctx_join and
 * ctx_split are two contexts of the same grid and device (mt_create).  The tile
 * kernel loads f once and builds both tile stores; each tree then runs its own
 * crossing-edge merge, repair and diagram on its context, so mt_diagram(ctx_join)
 * reports the merge tree's diagram and mt_diagram(ctx_split) the split tree's
 * (exactly mt_compute with flags 0 and MT_FLAG_SPLIT_TREE).  T_join / T_split:
 * device, n uint64 each, distinct.  Asynchronous like mt_compute. */
mt_status mt_compute_join_split(mt_ctx *ctx_join, mt_ctx *ctx_split, const float *f, uint64_t *T_join,
                                uint64_t *T_split, mt_stream_t stream);

/* Register a caller-owned device buffer that later mt_compute calls write
 * the diagram into directly (zero-copy); capacity in records.  NULL detaches.
 * Without a registered buffer the diagram is kept in the workspace. */
mt_status mt_set_diagram_output(mt_ctx *ctx, mt_pair *buf, uint64_t capacity);

/* Wait for the last mt_compute on `stream`, then report the diagram:
 * *n_pairs (host) finite pairs ordered by ascending birth_v, followed by
 * *n_essential (host) essential classes ordered by ascending vertex.
 * If `out` (device) is non-NULL and is not the registered buffer, the
 * n_pairs + n_essential records are copied there (capacity in records;
 * MT_ERR_CAPACITY if too small, counts still returned).  `out` may be NULL
 * to query counts only.  Returns the sticky data error if any (e.g.
 * MT_ERR_NONFINITE; the triplets are then unspecified). */
mt_status mt_diagram(mt_ctx *ctx, mt_pair *out, uint64_t capacity, uint64_t *n_pairs,
                     uint64_t *n_essential, mt_stream_t stream);

/* Device pointer to the diagram records of the last compute (registered
 * buffer or workspace); valid until the next mt_compute.  Syncs like
 * mt_diagram. */
mt_status mt_diagram_view(mt_ctx *ctx, const mt_pair **records, uint64_t *n_pairs,
                          uint64_t *n_essential, mt_stream_t stream);

/* Persistence simplification ("short branches ... can
 * be intuitively interpreted as topological noise"): copy to
 * `out` (device, capacity records, must not be the diagram buffer itself) the
 * finite pairs of the last compute with |death - birth| > eps (evaluated in
 * float32, the precision of the values) followed by every essential class,
 * in the order of mt_diagram.  eps >= 0.  Syncs; *n_pairs_kept and
 * *n_essential (host) receive the counts; MT_ERR_CAPACITY if they exceed
 * capacity (counts still returned). */
mt_status mt_filter_diagram(mt_ctx *ctx, float eps, mt_pair *out, uint64_t capacity, uint64_t *n_pairs_kept,
                            uint64_t *n_essential, mt_stream_t stream);

/* Synchronise `stream` and return the sticky error state of the context. */
mt_status mt_last_error(mt_ctx *ctx, mt_stream_t stream);

/* Kernel launches issued by the most recent mt_compute (host counter). */
uint32_t mt_last_launch_count(const mt_ctx *ctx);

/* Per-kernel device time (ms) of the most recent mt_compute, measured with
 * CUDA events recorded on `stream` when profiling is enabled with
 * mt_set_profiling(ctx, 1).  names[i] are static strings.  Returns the
 * number of entries written (<= max). */
mt_status mt_set_profiling(mt_ctx *ctx, int enable);
int mt_kernel_times(mt_ctx *ctx, const char **names, float *ms, int max);

/* ---- Multi-GPU: z-slab decomposition (distribution is the
 * paper's future work) --------------------------------
 * Rank r of P owns planes [z_begin, z_end) of the global grid; 3D grids only
 * (conn 6), at most 64 slabs.  Per step:
 *   1. mt_compute_local  -- merge tree of the slab subgraph + its boundary
 *      forest (the cells reachable from the slab's inter-slab faces);
 *   2. mt_forest_view    -- the forest records (the caller all-gathers them,
 *      e.g. with NCCL, concatenating the slabs' records in SLAB ORDER);
 *   3. mt_compute_global -- merges every inter-slab edge on the union of the
 *      forests, then repairs the slab and extracts its diagram: the slab's
 *      finite pairs (births in the slab, ascending) and, on the rank owning
 *      the global minimum, the essential class.
 * The result equals the single-GPU result (the store is unique, PAPER.md:
 * 196-200).
 *
 * Vertex ids.  The paper packs two 32-bit ids into one
 * 64-bit CAS word and names that limit as the obstacle to distribution
 * (PAPER.md:389-396, 1063-1066).  Here every kernel keeps 32-bit ids and the
 * packed 8-B store; the global ids may pass 2^32:
 *   - 32-bit mode (nx*ny*nz <= 2^32 - 1): the triplets and the diagram hold
 *     GLOBAL ids (mt_diagram as on one GPU);
 *   - wide mode (nx*ny*nz > 2^32 - 1, or MT_SLAB_WIDE_IDS): each context works
 *     in its own 32-bit VIEW of the id space -- its slab's vertices at a fixed
 *     offset, the vertices of other slabs that the gathered forest references
 *     compressed below and above it in global order (each slab numbers its
 *     referenced vertices by rank, an order-preserving compression, so every
 *     comparison of the method -- the (value, id) key, reading R1 -- gives the
 *     global answer).  mt_triplets64 / mt_diagram64 translate the results to
 *     64-bit global ids; mt_diagram returns MT_ERR_TOO_LARGE.
 *   A wide slab needs (z_end - z_begin + 2) * nx * ny < 2^32 and the
 *   gathered forest must fit the view beside it (MT_ERR_TOO_LARGE otherwise).
 *
 * Forest record (32 B): the vertex, its cell (s, v) and the f bits of the
 * vertex and of s (a saddle travels with displaced pairs across slabs;
 * diagram values are copied from the input f, reading R14; the order keys
 * are recomputed from the bits).  Ids are slab-local (global id minus
 * nx*ny*z_begin); the *_c fields are the compressed ids of wide mode (equal
 * to the local ids in 32-bit mode). */
typedef struct {
    uint32_t id;       /* slab-local vertex id */
    uint32_t s;        /* slab-local id of its saddle s */
    uint32_t v;        /* slab-local id of v */
    uint32_t f_bits;   /* bits of f[id] */
    uint32_t s_f_bits; /* bits of f[s] */
    uint32_t id_c, s_c, v_c;  /* compressed ids (wide mode) */
} mt_forest_record;    /* 32 bytes */

enum { MT_SLAB_WIDE_IDS = 1u }; /* mt_create_slab / mt_create_dist option: wide mode at any size */

/* 64-bit results (wide mode; also valid, widened, in 32-bit mode and on one GPU). */
typedef struct {
    uint64_t s, v;
} mt_triplet64;
typedef struct {
    uint64_t birth_v, death_v;
    float birth, death;
} mt_pair64;           /* 24 bytes */

size_t mt_slab_workspace_bytes(const uint32_t global_dims[3], int conn, uint32_t z_begin, uint32_t z_end);
/* options: 0 or MT_SLAB_WIDE_IDS (wide mode is automatic past 2^32 - 1 vertices). */
mt_status mt_create_slab(mt_ctx **out, const uint32_t global_dims[3], int conn, uint32_t z_begin,
                         uint32_t z_end, uint32_t options, int cuda_device, void *workspace,
                         size_t workspace_bytes);
/* f_slab (device): the slab's nx*ny*(z_end-z_begin) values, borrowed until
 * mt_compute_global's work completes; triplets_slab (device, n_local uint64):
 * receives the slab's tile store now and the final triplets from
 * mt_compute_global, which must be given the same buffer.  Asynchronous. */
mt_status mt_compute_local(mt_ctx *ctx, const float *f_slab, uint64_t *triplets_slab, uint32_t flags,
                           mt_stream_t stream);
/* Syncs; device pointer to the slab's forest records (valid until the next
 * mt_compute_local) and their number. */
mt_status mt_forest_view(mt_ctx *ctx, const mt_forest_record **records, uint64_t *n_records,
                         mt_stream_t stream);
/* Device scratch bytes mt_compute_global needs for n_all gathered records; 0 when the id
 * tables would pass 2^31 slots (n_all > 2^29: mt_compute_global returns MT_ERR_TOO_LARGE). */
size_t mt_forest_scratch_bytes(uint64_t n_all);
/* all (device): the records of every slab concatenated in slab order, counts[k]
 * (host) of slab k, nslabs of them (n_all = their sum); z_bounds (host): the
 * P+1 plane boundaries of all slabs (z_bounds[0] = 0, z_bounds[P] = nz);
 * scratch (device, >= mt_forest_scratch_bytes(n_all), 256-B aligned; it also
 * holds the id translation of wide mode and must stay intact until the last
 * mt_triplets64 / mt_diagram64 of this step); triplets_slab (device): the
 * buffer given to mt_compute_local (MT_ERR_INVALID_ARG otherwise), overwritten
 * with the slab's n_local triplets.  Asynchronous. */
mt_status mt_compute_global(mt_ctx *ctx, const mt_forest_record *all, const uint64_t *counts,
                            const uint32_t *z_bounds, uint32_t nslabs, void *scratch,
                            size_t scratch_bytes, uint64_t *triplets_slab, mt_stream_t stream);

/* Triplets first .. first+count-1 of the context's last result (triplets: the
 * buffer mt_compute / mt_compute_global wrote, device) with 64-bit global ids
 * into out (device, count records).  Asynchronous. */
mt_status mt_triplets64(mt_ctx *ctx, const uint64_t *triplets, uint64_t first, uint64_t count,
                        mt_triplet64 *out, mt_stream_t stream);
/* mt_diagram with 64-bit global ids (out: device, capacity records). */
mt_status mt_diagram64(mt_ctx *ctx, mt_pair64 *out, uint64_t capacity, uint64_t *n_pairs,
                       uint64_t *n_essential, mt_stream_t stream);

/* ---- Multi-GPU with the exchange inside the library ----------
 * One process per GPU.  Rank 0 calls mt_get_unique_id and the caller
 * broadcasts the 128 bytes to every rank (e.g. over torch.distributed); each
 * rank then creates its context with mt_create_dist and calls mt_compute /
 * mt_diagram (mt_triplets64 / mt_diagram64 in wide mode) exactly as on one
 * GPU, with its slab of f and of the triplets (planes [z_begin, z_end) of
 * mt_dist_slab_bounds).
 * mt_compute on such a context runs the local phase, then on `stream` an
 * ncclAllGather of the boundary-forest sizes (8 B per rank), ONE host sync to
 * read them, a grouped ncclBroadcast of every rank's records (exact length,
 * rank order) and the global phase (mt_compute_local / mt_compute_global
 * above), so it is not fully asynchronous.  NCCL (libnccl.so.2) is loaded at
 * run time: MT_ERR_NCCL if it is missing or a collective fails.  The
 * gathered records and the forest tables are device buffers the context owns
 * and grows on demand (cudaMalloc only when a step needs more than any
 * earlier one); mt_destroy frees them and the communicator.  3-D grids, conn
 * 6, 1 <= nranks <= min(64, nz). */
mt_status mt_get_unique_id(uint8_t id[128]);
/* bounds (host, nranks + 1): the planes of each rank's slab -- as equal as
 * possible, on multiples of the tile depth (8) when nz >= 8 nranks. */
mt_status mt_dist_slab_bounds(uint32_t nz, int nranks, uint32_t *bounds);
size_t mt_dist_workspace_bytes(const uint32_t global_dims[3], int conn, int rank, int nranks);
mt_status mt_create_dist(mt_ctx **out, const uint32_t global_dims[3], int conn, int rank, int nranks,
                         const uint8_t nccl_id[128], uint32_t options, int cuda_device, void *workspace,
                         size_t workspace_bytes);

/* ---- Explicit graphs ----------------------------------
 * The same computation on an undirected graph G = (V, E) (PAPER.md:128-131:
 * "the space is a graph G = (V, E), and the function is defined only on the
 * vertices") given in CSR form: the neighbours of u are col[row[u] ..
 * row[u+1]) (row: n+1 uint64, col: row[n] uint32 vertex ids, both device).
 * Every undirected edge must be listed in both directions; self-loops and
 * duplicate entries are allowed (they change nothing).  A graph may have
 * several components: one essential class each, ascending.  n_adj bounds
 * row[n] for the workspace size. */
size_t mt_graph_workspace_bytes(uint32_t n, uint64_t n_adj);
mt_status mt_create_graph(mt_ctx **out, uint32_t n, uint64_t n_adj, int cuda_device, void *workspace,
                          size_t workspace_bytes);
/* Asynchronous like mt_compute; f, row, col borrowed until the stream passes
 * this call's work; triplets (device, n uint64) out.  mt_diagram as usual; an
 * adjacency longer than the context's n_adj (row[n] > n_adj) is never dropped
 * silently: the sticky status becomes MT_ERR_CAPACITY (mt_diagram /
 * mt_last_error). */
mt_status mt_compute_graph(mt_ctx *ctx, const float *f, const uint64_t *row, const uint32_t *col,
                           uint64_t *triplets, uint32_t flags, mt_stream_t stream);

/* Diagnostics: while enabled, mt_compute counts events of the merge and
 * repair kernels: [0] edges examined, [1] edges skipped as redundant,
 * [2] cells followed by the pre-filter walks, [3] Alg. 3 loop iterations,
 * [4] failed CAS, [5] cells followed by the repair walks, [6..10] the
 * same for the in-tile phase (edges, walk hops, merge iterations, repair
 * hops, compress hops), [11..17] SM cycles of the tile phases (load,
 * descent, compress, merge, repair, write, edge list; summed over tiles),
 * [18] adjacent basin pairs in the tiles, [19] crossing edges queued,
 * [20..21] unused (0).  mt_stats syncs
 * `stream` and copies up to `max` counters to out (host); returns the
 * number written (0 if disabled). */
mt_status mt_set_stats(mt_ctx *ctx, int enable);
int mt_stats(mt_ctx *ctx, uint64_t *out, int max, mt_stream_t stream);

const char *mt_status_string(mt_status s);
void mt_destroy(mt_ctx *ctx);

/* Version of this ABI (bumped on any signature change; 2: mt_compute_local takes the
 * triplet buffer; 3: wide ids -- forest record v3, slab counts in mt_compute_global,
 * options in mt_create_slab / mt_create_dist, mt_triplets64, mt_diagram64). */
int mt_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MT_B200_H */
