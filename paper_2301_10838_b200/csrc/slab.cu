// slab.cu -- multi-GPU z-slab decomposition: the boundary forest of a slab,
// its merge across all slabs, and the write-back (DESIGN.md
// section 9; distribution is the paper's future work).
//
// After each rank computed the store of its slab subgraph (tile_tmt +
// merge_cross), the global store is the union of the slab stores: a valid
// normalized store of G minus the inter-slab edges.  Merging an inter-slab
// edge (Alg. 3) only ever reads or writes cells reachable from the edge's two
// endpoints by following v pointers (climbs, the CAS target, the displaced
// pair, path splitting), and a displaced pair points into the same chain, so
// the set of cells touched by ALL inter-slab merges is contained in the
// closure of the face vertices under v (DESIGN.md derivation H).  Each rank
//   1. marks that closure in its slab (forest_mark) and compacts it into
//      records (forest_compact) -- the records of all ranks are all-gathered;
//   2. builds an id -> record table over the union (forest_build) and merges
//      every inter-slab edge on it (forest_merge; the same walks + Alg. 3 as
//      merge_cross.cu, with cell access through the table);
//   3. writes the merged cells of its own vertices back (forest_writeback);
// then the repair walks local cells and, past a remote id, the merged forest
// (repair_diagram.cu, ForestView).  Every rank merges the whole forest
// redundantly; the post-repair store is unique, so the ranks agree.
//
// Ids (PAPER.md:389-396 and 1063-1066 name the 32-bit
// packing as the obstacle to distribution).  Every kernel of a context works in
// the context's 32-bit VIEW of the id space: its own vertices at view ids
// [base, base + n), the vertices of other slabs the gathered forest references
// at view ids below and above, in global order.  32-bit mode: the view is the
// global id (base = nx ny z_begin).  Wide mode (global ids past 2^32): each
// slab numbers the vertices its records reference (ids and saddles) by rank --
// an order-preserving compression (forest_refmark / popc_* / forest_compress)
// -- and each receiver places slab k's compressed ids at its own offset voff[k]
// (forest_build).  Every decision of the method compares (value, id) keys or
// tests ids for equality (Alg. 3-5, reading R1), and an order-preserving
// relabelling keeps all of them, so each rank computes its slab's result with
// view ids, which mt_triplets64 / mt_diagram64 translate (id_decode).
#include "common.cuh"
#include "kernels.cuh"

#ifndef FOREST_FACEIDX
#define FOREST_FACEIDX 1   // face records at fixed slots; forest_dedupe indexes them directly
#endif

namespace mt {

namespace {

// a vertex that is regular in its tile has no working cell: T0 = ord(x) << 32 | R(x) with its
// tile representative R(x) != x (a tile minimum has R(x) == x and a cell)
__device__ __forceinline__ bool tile_regular(const uint64_t* T0, uint32_t x, uint32_t* rep, uint32_t* ord_x) {
    const uint64_t t = T0[x];
    *rep = cell_v(t);
    *ord_x = cell_s(t);
    return cell_v(t) != x;
}

__global__ void __launch_bounds__(256)
forest_mark_kernel(const Cell* C, const uint64_t* T0, uint32_t nx, uint32_t ny, uint64_t bottom, uint64_t top,
                   bool has_bottom, bool has_top, uint64_t base, uint8_t* flag) {
    const uint64_t sxy = uint64_t(nx) * ny;
    const uint64_t nface = uint64_t(has_bottom) + uint64_t(has_top);
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < nface * sxy;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const bool first = t < sxy;
        const uint64_t plane = (first && has_bottom) ? bottom : top;
        uint32_t x = uint32_t(plane + (t % sxy));
        // the face vertex itself, then (from its tile representative on) the chain of minima cells,
        // flagging each; stop at a flagged cell (its chain is taken)
        uint8_t* fl = flag + (uint64_t(x) - base);
        if (*reinterpret_cast<volatile uint8_t*>(fl)) continue;
        *reinterpret_cast<volatile uint8_t*>(fl) = 1;
        uint32_t rep, ox;
        if (tile_regular(T0, x, &rep, &ox)) {
            x = rep;
        } else {
            const Cell c = ld_cell(C + x);
            if (cv_of(c) == x) continue;
            x = cv_of(c);
        }
        while (true) {
            fl = flag + (uint64_t(x) - base);
            if (*reinterpret_cast<volatile uint8_t*>(fl)) break;
            *reinterpret_cast<volatile uint8_t*>(fl) = 1;
            const Cell c = ld_cell(C + x);
            if (cv_of(c) == x) break;
            x = cv_of(c);
        }
    }
}

__global__ void __launch_bounds__(256)
forest_compact_kernel(const Cell* C, const uint64_t* T0, const float* f, uint64_t base, uint64_t n,
                      const uint8_t* __restrict__ flag, mt_forest_record* __restrict__ recs, uint64_t cap,
                      unsigned long long* count, uint64_t bot_hi, uint64_t top_lo, uint64_t top_at, uint64_t nf) {
    // FOREST_FACEIDX: the face vertices (every one is a record) take fixed slots -- the bottom face
    // (local ids [0, bot_hi)) at its local id, the top face (from top_lo on) at top_at + offset --
    // and the rest are appended after the nf face slots, so a face vertex's record index follows
    // from its position (forest_dedupe reads the boundary records without id lookups)
    const int lane = threadIdx.x & 31;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint32_t b = uint32_t(base);
    for (uint64_t l0 = uint64_t(blockIdx.x) * blockDim.x; l0 < n; l0 += stride) {
        const uint64_t l = l0 + threadIdx.x;
        const bool take = l < n && flag[l];
        const bool face = l < bot_hi || l >= top_lo;
        const uint32_t m = __ballot_sync(FULL_MASK, take && !face);
        unsigned long long b0 = 0;
        if (lane == 0 && m) b0 = atomicAdd(count, (unsigned long long)__popc(m));
        b0 = __shfl_sync(FULL_MASK, b0, 0);
        if (take) {
            const uint64_t pos = l < bot_hi ? l : l >= top_lo ? top_at + (l - top_lo)
                                                              : nf + b0 + __popc(m & ((1u << lane) - 1u));
            const uint32_t u = uint32_t(base + l);
            uint32_t rep, o;
            const uint32_t fb = __float_as_uint(f[u]);
            const uint32_t lu = uint32_t(l);
            mt_forest_record rec;
            if (tile_regular(T0, u, &rep, &o)) {
                // the cell the vertex would have: (u, u, R) at its own key
                rec = mt_forest_record{lu, lu, rep - b, fb, fb, lu, lu, rep - b};
            } else {
                const Cell c = ld_cell(C + u);
                const uint32_t ls = cs_of(c) - b, lv = cv_of(c) - b;
                rec = mt_forest_record{lu, ls, lv, fb, __float_as_uint(f[cs_of(c)]), lu, ls, lv};
            }
            if (pos < cap) recs[pos] = rec;
        }
    }
}

// ---- wide mode, sender side: order-preserving compression of the referenced local ids ----
// referenced = the records' vertices and their saddles (every v is a record's vertex: the forest
// is closed under v).  c(l) = #referenced ids below l, plus a gap before the top face so that the
// top face of a slab with count records sits at [2 count - nx ny, 2 count) -- the receivers know
// where a face is without the slab's exact number of referenced ids (2 count bounds it); the
// bottom face, the lowest referenced ids, is [0, nx ny) (a one-plane slab: both faces).
__global__ void __launch_bounds__(256)
forest_refmark_kernel(const mt_forest_record* __restrict__ recs, const unsigned long long* __restrict__ count,
                      uint32_t* __restrict__ bits) {
    const uint64_t nrec = *count;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nrec;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t id = recs[i].id, sd = recs[i].s;
        atomicOr(bits + (id >> 5), 1u << (id & 31));
        if (sd != id) atomicOr(bits + (sd >> 5), 1u << (sd & 31));
    }
}

constexpr int PC_THREADS = 1024, PC_WORDS = 8;   // one CTA: 8192 bitmap words
__device__ __forceinline__ uint32_t cta_exclusive_scan(uint32_t x, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL_MASK, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < int(blockDim.x >> 5) ? s_warp[lane] : 0u, wi = w;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL_MASK, wi, d);
            if (lane >= d) wi += y;
        }
        s_warp[lane] = wi - w;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    const uint32_t r = s_warp[warp] + incl - x;
    *total = s_warp[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(PC_THREADS)
popc_block_kernel(const uint32_t* __restrict__ bits, uint64_t nwords, uint32_t* __restrict__ bsum) {
    __shared__ uint32_t s_warp[33];
    const uint64_t w0 = uint64_t(blockIdx.x) * PC_THREADS * PC_WORDS + uint64_t(threadIdx.x) * PC_WORDS;
    uint32_t c = 0;
    for (int k = 0; k < PC_WORDS; ++k)
        if (w0 + k < nwords) c += __popc(bits[w0 + k]);
    uint32_t tot = 0;
    cta_exclusive_scan(c, s_warp, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// one CTA: exclusive scan of the block sums in place, the total into bsum[nblocks]
__global__ void __launch_bounds__(PC_THREADS) popc_scan_kernel(uint32_t* __restrict__ bsum, uint32_t nblocks) {
    __shared__ uint32_t s_warp[33];
    const uint32_t per = (nblocks + PC_THREADS - 1) / PC_THREADS;
    const uint32_t b0 = threadIdx.x * per;
    uint32_t c = 0;
    for (uint32_t k = 0; k < per; ++k)
        if (b0 + k < nblocks) c += bsum[b0 + k];
    uint32_t tot = 0;
    uint32_t run = cta_exclusive_scan(c, s_warp, &tot);
    for (uint32_t k = 0; k < per; ++k)
        if (b0 + k < nblocks) {
            const uint32_t x = bsum[b0 + k];
            bsum[b0 + k] = run;
            run += x;
        }
    if (threadIdx.x == 0) bsum[nblocks] = tot;
}

__global__ void __launch_bounds__(PC_THREADS)
popc_prefix_kernel(const uint32_t* __restrict__ bits, uint64_t nwords, const uint32_t* __restrict__ bsum,
                   uint32_t* __restrict__ pre) {
    __shared__ uint32_t s_warp[33];
    const uint64_t w0 = uint64_t(blockIdx.x) * PC_THREADS * PC_WORDS + uint64_t(threadIdx.x) * PC_WORDS;
    uint32_t w[PC_WORDS], c = 0;
    for (int k = 0; k < PC_WORDS; ++k) {
        w[k] = w0 + k < nwords ? bits[w0 + k] : 0u;
        c += __popc(w[k]);
    }
    uint32_t tot = 0;
    uint32_t run = bsum[blockIdx.x] + cta_exclusive_scan(c, s_warp, &tot);
    for (int k = 0; k < PC_WORDS; ++k)
        if (w0 + k < nwords) {
            pre[w0 + k] = run;
            run += __popc(w[k]);
        }
}

__global__ void __launch_bounds__(256)
forest_compress_kernel(mt_forest_record* __restrict__ recs, const unsigned long long* __restrict__ count,
                       const uint32_t* __restrict__ bits, const uint32_t* __restrict__ pre,
                       const uint32_t* __restrict__ total, uint64_t top_begin) {
    const uint64_t nrec = *count;
    const uint64_t gap = 2 * nrec - *total;   // >= 0: at most 2 referenced ids per record
    auto rank = [&](uint32_t l) -> uint32_t {
        const uint32_t c = pre[l >> 5] + __popc(bits[l >> 5] & ((1u << (l & 31)) - 1u));
        return uint32_t(c + (l >= top_begin ? gap : 0));
    };
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nrec;
         i += uint64_t(gridDim.x) * blockDim.x) {
        mt_forest_record r = recs[i];
        r.id_c = rank(r.id);
        r.s_c = rank(r.s);
        r.v_c = rank(r.v);
        recs[i] = r;
    }
}

// insert (id -> payload) unless id is present already
__device__ __forceinline__ void table_put(unsigned long long* t, uint32_t mask, uint32_t id, uint32_t payload) {
    const unsigned long long e = (static_cast<unsigned long long>(id) << 32) | payload;
    uint32_t h = forest_hash(id, mask);
    while (true) {
        const unsigned long long old = atomicCAS(t + h, ~0ull, e);
        if (old == ~0ull || uint32_t(old >> 32) == id) return;
        h = (h + 1) & mask;
    }
}

// slab of gathered record i (records concatenated in slab order)
__device__ __forceinline__ uint32_t slab_of(const ForestXlate& X, uint64_t i) {
    uint32_t lo = 0, hi = X.nslabs - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (X.rec_off[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(256)
forest_build_kernel(const mt_forest_record* __restrict__ all, uint64_t n_all, ForestXlate X,
                    unsigned long long* table, unsigned long long* vtable, uint32_t mask, Cell* cells,
                    uint32_t* __restrict__ vid, uint64_t* __restrict__ dec) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_all;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const mt_forest_record r = all[i];
        const uint32_t k = slab_of(X, i);
        const bool own = k == X.self;
        // the record in this rank's view: own slab at base + local id, slab k's compressed ids at voff[k]
        const uint32_t id = X.voff[k] + (own ? r.id : r.id_c);
        const uint32_t sv = X.voff[k] + (own ? r.s : r.s_c);
        const uint32_t vv = X.voff[k] + (own ? r.v : r.v_c);
        const uint32_t ou = ord32(__uint_as_float(r.f_bits)) ^ X.flip;
        const uint32_t os = ord32(__uint_as_float(r.s_f_bits)) ^ X.flip;
        cells[i] = Cell{key_of(os, sv), key_of(ou, vv)};
        vid[i] = id;
        table_put(table, mask, id, uint32_t(i));
        // the f bits of a record's saddle are needed only where the order key cannot give them
        // back: a zero value (-0 and +0 share one key, reading R2; diagram values are copied from
        // the input, R14) -- every other value is the inverse of the key's order bits
        if ((r.s_f_bits & 0x7fffffffu) == 0u) table_put(vtable, mask, sv, r.s_f_bits);
        if (X.wide && !own) {                      // 64-bit global ids of the remote view ids
            dec[X.dec_index(id)] = X.real_base[k] + r.id;
            dec[X.dec_index(sv)] = X.real_base[k] + r.s;
        }
    }
}

struct BoundaryGeom {
    uint32_t nx, ny;
    uint32_t nb;                   // inter-slab boundaries
    uint32_t direct;               // ia0 / ib0 valid (FOREST_FACEIDX)
    uint32_t a0[MAX_SLABS];        // view id of vertex (0, 0) of the lower face of boundary k
    uint32_t b0[MAX_SLABS];        // ... and of its upper face (faces are consecutive view ids)
    uint32_t ia0[MAX_SLABS];       // record index of vertex (0, 0) of the lower face of boundary k
    uint32_t ib0[MAX_SLABS];       // ... and of its upper face
};

// Inter-slab edges reduced to pairs of tile representatives (DESIGN.md derivation C-3, the
// reduction dedupe_cross applies to the tile faces): edge (a, b) at level L = max(key a, key b)
// joins R(a) and R(b) at L, R = the tile representative at the vertex's own level (its forest
// record's v for a tile-regular vertex, the vertex itself for a minimum), so of the edges with
// one pair only the lowest is queued.  One CTA step = 512 consecutive edges of one boundary; a
// shared-memory table keeps, per pair, the lowest level.  Every rank runs it on the gathered
// records (the result is the same on all).
struct FQEntry {
    uint64_t L;
    uint32_t r_hi, r_lo;
};
constexpr int FD_THREADS = 512;

__global__ void __launch_bounds__(FD_THREADS)
forest_dedupe_kernel(ForestRef F, BoundaryGeom g, FQEntry* __restrict__ q, unsigned long long* __restrict__ qlen) {
    __shared__ unsigned long long s_key[2 * FD_THREADS], s_min[2 * FD_THREADS];
    __shared__ uint32_t s_warp[FD_THREADS / 32];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t sxy = uint64_t(g.nx) * g.ny;
    const uint64_t total = sxy * g.nb;
    for (uint64_t e0 = uint64_t(blockIdx.x) * FD_THREADS; e0 < total; e0 += uint64_t(gridDim.x) * FD_THREADS) {
        const uint64_t e = e0 + threadIdx.x;
        bool keep = false;
        FQEntry en{0, 0, 0};
        uint64_t pair = ~0ull;
        if (e < total) {
            const uint64_t k = e / sxy, r = e % sxy;
            const uint32_t a = g.a0[k] + uint32_t(r), b = g.b0[k] + uint32_t(r);
            uint32_t ia = FOREST_MISS, ib = FOREST_MISS;
            if (g.direct) {   // the face records' fixed slots (forest_compact), checked against their ids
                ia = g.ia0[k] + uint32_t(r);
                ib = g.ib0[k] + uint32_t(r);
                if (F.vid[ia] != a) ia = FOREST_MISS;
                if (F.vid[ib] != b) ib = FOREST_MISS;
            }
            if (ia == FOREST_MISS) ia = forest_lookup(F, a);
            if (ib == FOREST_MISS) ib = forest_lookup(F, b);
            if (ia == FOREST_MISS || ib == FOREST_MISS) {
                atomicOr(F.err, ERR_FOREST);
            } else {
                const Cell ca = F.cells[ia], cb = F.cells[ib];
                const uint64_t ka = self_key(ca, a), kb = self_key(cb, b);
                const uint32_t ra = cs_of(ca) == a ? cv_of(ca) : a, rb = cs_of(cb) == b ? cv_of(cb) : b;
                en = ka > kb ? FQEntry{ka, ra, rb} : FQEntry{kb, rb, ra};
                pair = ra < rb ? (uint64_t(ra) << 32 | rb) : (uint64_t(rb) << 32 | ra);
                keep = true;
            }
        }
        s_key[threadIdx.x] = ~0ull;
        s_key[threadIdx.x + FD_THREADS] = ~0ull;
        s_min[threadIdx.x] = ~0ull;
        s_min[threadIdx.x + FD_THREADS] = ~0ull;
        __syncthreads();
        uint32_t h = 0;
        if (keep) {
            h = uint32_t((pair * 0x9E3779B97F4A7C15ull) >> 54);   // 10 bits: 2 x FD_THREADS slots
            while (true) {
                const unsigned long long old = atomicCAS(&s_key[h], ~0ull, pair);
                if (old == ~0ull || old == pair) break;
                h = (h + 1) & (2u * FD_THREADS - 1u);
            }
            atomicMin(&s_min[h], (unsigned long long)en.L);
        }
        __syncthreads();
        if (keep && s_min[h] != en.L) keep = false;
        const uint32_t km = __ballot_sync(FULL_MASK, keep);
        if (lane == 0) s_warp[warp] = __popc(km);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < FD_THREADS / 32; ++w) {
                const uint32_t t = s_warp[w];
                s_warp[w] = tot;
                tot += t;
            }
            s_base = tot ? atomicAdd(qlen, (unsigned long long)tot) : 0;
        }
        __syncthreads();
        if (keep) q[s_base + s_warp[warp] + __popc(km & ((1u << lane) - 1u))] = en;
        __syncthreads();
    }
}

enum Phase : int { IDLE = 0, CLIMB_HI = 2, CLIMB_LO = 3, MERGE_LD = 4, MERGE_CAS = 5, DONE = 6 };

#ifndef FM_CSPLIT
#define FM_CSPLIT 1   // forest_merge: Alg. 3 straight from the representatives, path splitting in the climbs
#endif
// merge_cross.cu's state machine on the forest: every cell access goes through the table
__global__ void __launch_bounds__(256)
forest_merge_kernel(ForestRef F, const FQEntry* __restrict__ q, const unsigned long long* __restrict__ qlen,
                    unsigned long long* __restrict__ fetch) {
    constexpr uint64_t BATCH = 256;
    const int lane = threadIdx.x & 31;
    const uint64_t total = *reinterpret_cast<const volatile unsigned long long*>(qlen);
    uint64_t pool_next = 0, pool_end = 0;
    bool exhausted = false;
    int phase = IDLE;
    // merge_queue_kernel's state machine with every cell reached through the id table; one set
    // of registers serves the exclusive phases (ids p*, table indices i*):
    //   climbs: lev = L, p0/i0 = x, i1 = previous cell, p2/i2 = lo, p3/i3 = rh, held = previous cell;
    //   Alg. 3: lev = S, p0/i0 = u, p1/i1 = v, held = T[v] as loaded (the CAS's expected value).
    uint64_t lev = 0;
    uint32_t p0 = 0, p1 = 0, p2 = 0, p3 = 0, i0 = 0, i1 = 0, i2 = 0, i3 = 0;
    bool has_prev = false;
    Cell held{0, 0};
    // FM_CSPLIT: the previous cell (table index, value) of each Alg. 3 climb
    [[maybe_unused]] Cell hu{0, 0}, hv{0, 0};
    [[maybe_unused]] uint32_t ju = 0, jv = 0;
    [[maybe_unused]] bool has_u = false, has_v = false;
    auto at = [&](uint32_t i) { return F.cells + i; };
    auto lookup = [&](uint32_t id, uint32_t* i) {
        *i = forest_lookup(F, id);
        if (*i == FOREST_MISS) {
            atomicOr(F.err, ERR_FOREST);
            return false;
        }
        return true;
    };
    while (true) {
        const uint32_t need = __ballot_sync(FULL_MASK, phase == IDLE);
        if (need) {
            if (pool_next == pool_end && !exhausted) {
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
                    // a deduplicated edge: walk from R_hi, then R_lo, at level L (forest_dedupe_kernel)
                    const FQEntry en = q[pool_next + rank];
                    lev = en.L;
                    p0 = en.r_hi;
                    p2 = en.r_lo;
                    has_prev = false;
                    phase = (lookup(p0, &i0) && lookup(p2, &i2)) ? CLIMB_HI : IDLE;
                    if (FM_CSPLIT && phase == CLIMB_HI) {   // Merge(T, R_hi, hi, R_lo) straight away
                        p1 = p2;
                        i1 = i2;
                        has_u = has_v = false;
                        phase = MERGE_LD;
                    }
                } else if (exhausted) {
                    phase = DONE;
                }
            }
            pool_next += avail < __popc(need) ? avail : __popc(need);
        }
        if (__ballot_sync(FULL_MASK, phase != DONE) == 0) break;

        if (phase == CLIMB_HI || phase == CLIMB_LO) {
            const Cell c = ld_cell(at(i0));
            if (cv_of(c) != p0 && c.lo <= lev) {                    // followable at level L
                if (has_prev && c.lo <= held.lo)                    // path splitting
                    cas_cell(at(i1), held, Cell{held.lo, (held.hi & 0xffffffff00000000ull) | cv_of(c)});
                i1 = i0;
                held = c;
                has_prev = true;
                p0 = cv_of(c);
                if (!lookup(p0, &i0)) phase = IDLE;
            } else if (phase == CLIMB_HI) {
                p3 = p0;
                i3 = i0;
                p0 = p2;
                i0 = i2;
                has_prev = false;
                phase = CLIMB_LO;
            } else if (p0 == p3) {
                phase = IDLE;                                       // already joined below L
            } else {
                p1 = p0;                                            // Merge(T, r_hi, hi, r_lo) at level L
                i1 = i0;
                p0 = p3;
                i0 = i3;
                phase = MERGE_LD;
            }
        } else if (phase == MERGE_LD) {
            Cell cu = ld_cell(at(i0)), cv = ld_cell(at(i1));
            const bool up_u = cv_of(cu) != p0 && cu.lo < lev;       // l.2-4 (+ R4)
            const bool up_v = cv_of(cv) != p1 && cv.lo < lev;       // l.5-8 (+ R4)
            if (FM_CSPLIT && (up_u || up_v)) {
                // independent climbs, each splitting its path (merge_cross.cu, MQ_CSPLIT)
                if (up_u) {
                    if (has_u && cu.lo <= hu.lo)
                        cas_cell(at(ju), hu, Cell{hu.lo, (hu.hi & 0xffffffff00000000ull) | cv_of(cu)});
                    ju = i0;
                    hu = cu;
                    has_u = true;
                    p0 = cv_of(cu);
                    if (!lookup(p0, &i0)) phase = IDLE;
                }
                if (up_v) {
                    if (has_v && cv.lo <= hv.lo)
                        cas_cell(at(jv), hv, Cell{hv.lo, (hv.hi & 0xffffffff00000000ull) | cv_of(cv)});
                    jv = i1;
                    hv = cv;
                    has_v = true;
                    p1 = cv_of(cv);
                    if (!lookup(p1, &i1)) phase = IDLE;
                }
            } else if (up_u || up_v) {                              // independent climbs (derivation J)
                if (up_u) {
                    p0 = cv_of(cu);
                    if (!lookup(p0, &i0)) phase = IDLE;
                }
                if (up_v) {
                    p1 = cv_of(cv);
                    if (!lookup(p1, &i1)) phase = IDLE;
                }
            } else if (p0 == p1) {                                  // l.9-10
                phase = IDLE;
            } else {
                if (self_key(cv, p1) < self_key(cu, p0)) {          // l.11-12
                    uint32_t t = p0; p0 = p1; p1 = t;
                    t = i0; i0 = i1; i1 = t;
                    cv = cu;
                }
                held = cv;                                          // l.14, next round trip
                phase = MERGE_CAS;
                has_u = has_v = false;
            }
        } else if (phase == MERGE_CAS) {
            const Cell got = cas_cell(at(i1), held, Cell{lev, (held.hi & 0xffffffff00000000ull) | p0});
            if (got.lo == held.lo && got.hi == held.hi) {
                const uint32_t vp = cv_of(held);
                if (vp == p1) {
                    phase = IDLE;                                   // displaced a root (R5)
                } else {
                    lev = held.lo;                                  // l.15
                    p1 = vp;
                    phase = lookup(p1, &i1) ? MERGE_LD : IDLE;
                }
            } else {
                phase = MERGE_LD;                                   // l.17
            }
        }
    }
}

__global__ void __launch_bounds__(256)
forest_writeback_kernel(ForestRef F, uint64_t n_all, Cell* C, const uint64_t* T0, uint64_t base, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_all;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t id = F.vid[i];
        uint32_t rep, o;
        // (a tile-regular face vertex keeps its T0: the repair walks from its R through the forest)
        if (uint64_t(id) - base < n && !tile_regular(T0, id, &rep, &o)) {
            const Cell c = F.cells[i];
            st_cell(C + id, c);
        }
    }
}

// ---- view ids -> 64-bit global ids (mt_triplets64 / mt_diagram64) ----
__global__ void __launch_bounds__(256)
triplets64_kernel(const uint64_t* __restrict__ T, uint64_t count, IdDecode d, mt_triplet64* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t t = T[i];
        out[i] = mt_triplet64{d.gid(cell_s(t)), d.gid(cell_v(t))};
    }
}

__global__ void __launch_bounds__(256)
pairs64_kernel(const mt_pair* __restrict__ in, uint64_t count, IdDecode d, mt_pair64* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const mt_pair p = in[i];
        out[i] = mt_pair64{d.gid(p.birth_v), d.gid(p.death_v), p.birth, p.death};
    }
}

uint32_t grid_for(uint64_t work, int num_sms) {
    uint64_t b = (work + 255) / 256;
    const uint64_t cap = uint64_t(num_sms) * 8 * 16;
    if (b > cap) b = cap;
    return uint32_t(b ? b : 1);
}

}  // namespace

void launch_forest_mark(const Cell* C, const uint64_t* T0, const Slab& sl, bool has_bottom, bool has_top,
                        uint8_t* flag, cudaStream_t stream) {
    if (!has_bottom && !has_top) return;
    const uint64_t sxy = uint64_t(sl.nx) * sl.ny;
    const uint64_t work = sxy * (uint64_t(has_bottom) + uint64_t(has_top));
    forest_mark_kernel<<<grid_for(work, 148), 256, 0, stream>>>(C, T0, sl.nx, sl.ny, uint64_t(sl.z_begin) * sxy,
                                                                uint64_t(sl.z_end - 1) * sxy, has_bottom, has_top,
                                                                sl.base, flag);
}

__global__ void add_count_kernel(unsigned long long* count, uint64_t add) { *count += add; }

int launch_forest_compact(const Cell* C, const uint64_t* T0, const float* f, const Slab& sl, const uint8_t* flag,
                          mt_forest_record* recs, uint64_t cap, unsigned long long* count, bool has_bottom,
                          bool has_top, int num_sms, cudaStream_t stream) {
    if (sl.n == 0) return 0;
    const uint64_t sxy = uint64_t(sl.nx) * sl.ny;
    uint64_t bot_hi = 0, top_lo = ~0ull, top_at = 0, nf = 0;
    if (FOREST_FACEIDX && sxy && sl.n % sxy == 0) {
        if (has_bottom) bot_hi = sxy;
        if (has_top && !(has_bottom && sl.n == sxy)) {   // (a one-plane slab's only plane: the bottom region)
            top_lo = sl.n - sxy;
            top_at = bot_hi;
        }
        nf = bot_hi + (top_lo == ~0ull ? 0 : sxy);
    }
    forest_compact_kernel<<<grid_for(sl.n, num_sms), 256, 0, stream>>>(C, T0, f, sl.base, sl.n, flag, recs, cap,
                                                                       count, bot_hi, top_lo, top_at, nf);
    if (nf) {
        add_count_kernel<<<1, 1, 0, stream>>>(count, nf);   // the count covers the face slots too
        return 2;
    }
    return 1;
}

size_t forest_compress_scratch_bytes(uint64_t n) {
    const uint64_t words = (n + 31) / 32, blocks = (words + PC_THREADS * PC_WORDS - 1) / (PC_THREADS * PC_WORDS);
    return size_t(2 * words + blocks + 1) * sizeof(uint32_t) + 512;
}

int launch_forest_compress(mt_forest_record* recs, const unsigned long long* count, uint64_t n, uint64_t top_begin,
                           void* scratch, int num_sms, cudaStream_t stream) {
    if (n == 0) return 0;
    const uint64_t words = (n + 31) / 32, blocks = (words + PC_THREADS * PC_WORDS - 1) / (PC_THREADS * PC_WORDS);
    uint32_t* bits = static_cast<uint32_t*>(scratch);
    uint32_t* pre = bits + words;
    uint32_t* bsum = pre + words;
    cudaMemsetAsync(bits, 0, words * sizeof(uint32_t), stream);
    const uint32_t g = uint32_t(num_sms) * 8;
    forest_refmark_kernel<<<g, 256, 0, stream>>>(recs, count, bits);
    popc_block_kernel<<<uint32_t(blocks), PC_THREADS, 0, stream>>>(bits, words, bsum);
    popc_scan_kernel<<<1, PC_THREADS, 0, stream>>>(bsum, uint32_t(blocks));
    popc_prefix_kernel<<<uint32_t(blocks), PC_THREADS, 0, stream>>>(bits, words, bsum, pre);
    forest_compress_kernel<<<g, 256, 0, stream>>>(recs, count, bits, pre, bsum + blocks, top_begin);
    return 5;
}

uint64_t forest_table_size(uint64_t n_all) {
    uint64_t s = 1024;
    while (s < 4 * n_all) s <<= 1;   // the value table holds up to 2 entries per record
    return s > (1ull << 31) ? 0 : s; // table indices and the mask are 32-bit
}

void launch_forest_build(const mt_forest_record* all, uint64_t n_all, const ForestXlate& X, uint64_t* table,
                         uint64_t* vtable, uint32_t mask, Cell* cells, uint32_t* vid, uint64_t* dec, int num_sms,
                         cudaStream_t stream) {
    if (n_all == 0) return;
    forest_build_kernel<<<grid_for(n_all, num_sms), 256, 0, stream>>>(
        all, n_all, X, reinterpret_cast<unsigned long long*>(table), reinterpret_cast<unsigned long long*>(vtable),
        mask, cells, vid, dec);
}

size_t forest_queue_entry_bytes() { return sizeof(FQEntry); }

void launch_forest_merge(const ForestRef& F, const Slab& sl, uint32_t nslabs, const uint32_t* a0, const uint32_t* b0,
                         const uint32_t* ia0, const uint32_t* ib0, void* queue, unsigned long long* qlen,
                         unsigned long long* fetch, int num_sms, cudaStream_t stream) {
    if (nslabs < 2) return;
    BoundaryGeom g{};
    g.nx = sl.nx;
    g.ny = sl.ny;
    g.nb = nslabs - 1;
    g.direct = (FOREST_FACEIDX && ia0 && ib0) ? 1u : 0u;
    for (uint32_t k = 0; k + 1 < nslabs; ++k) {
        g.a0[k] = a0[k];
        g.b0[k] = b0[k];
        g.ia0[k] = g.direct ? ia0[k] : 0u;
        g.ib0[k] = g.direct ? ib0[k] : 0u;
    }
    FQEntry* q = static_cast<FQEntry*>(queue);
    const uint64_t total = uint64_t(g.nx) * g.ny * g.nb;
    uint64_t blocks = (total + FD_THREADS - 1) / FD_THREADS;
    if (blocks > uint64_t(num_sms) * 8) blocks = uint64_t(num_sms) * 8;
    forest_dedupe_kernel<<<uint32_t(blocks), FD_THREADS, 0, stream>>>(F, g, q, qlen);
    forest_merge_kernel<<<uint32_t(num_sms) * 4, 256, 0, stream>>>(F, q, qlen, fetch);
}

void launch_forest_writeback(const ForestRef& F, uint64_t n_all, Cell* C, const uint64_t* T0, const Slab& sl,
                             int num_sms, cudaStream_t stream) {
    if (n_all == 0) return;
    forest_writeback_kernel<<<grid_for(n_all, num_sms), 256, 0, stream>>>(F, n_all, C, T0, sl.base, sl.n);
}

void launch_triplets64(const uint64_t* T, uint64_t count, const IdDecode& d, mt_triplet64* out, int num_sms,
                       cudaStream_t stream) {
    if (count == 0) return;
    triplets64_kernel<<<grid_for(count, num_sms), 256, 0, stream>>>(T, count, d, out);
}

void launch_pairs64(const mt_pair* in, uint64_t count, const IdDecode& d, mt_pair64* out, int num_sms,
                    cudaStream_t stream) {
    if (count == 0) return;
    pairs64_kernel<<<grid_for(count, num_sms), 256, 0, stream>>>(in, count, d, out);
}

}  // namespace mt
