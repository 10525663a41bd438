// merge_queue.cu -- K3 as two kernels: (a) filter the grid edges down to the
// ones that join two different descent basins, into a queue; (b) merge the
// queued edges with persistent warps whose lanes each run Alg. 3 (PAPER.md:
// 281-308) as a state machine advanced one memory round-trip per step.
//
// Why: the edge merge is a chain of dependent loads (climbs) of very uneven
// length.  Written as nested loops per thread, a warp waits for its slowest
// lane at every loop exit (ncu: 2.5 active threads per issued instruction);
// advancing every lane by exactly one cell load (or one CAS) per step and
// refilling idle lanes from the queue keeps the warp converged, so each step
// puts up to 32 independent loads in flight per warp.
//
// The algorithm per edge is unchanged from merge_edges.cu: the edge (hi, lo)
// enters at L = key(hi); both ends are walked from their basin minima through
// cells with key(s) <= L (Alg. 4's walk, with path splitting); if the walks
// meet the edge is redundant (derivation C'); otherwise Merge(T, r_hi, hi, r_lo)
// runs with the root guards R4/R5 and restarts that re-read both cells.
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

struct QEntry {
    uint64_t L;      // key of the edge's upper endpoint (the merge level)
    uint32_t m_hi;   // basin minimum of the upper endpoint
    uint32_t m_lo;   // basin minimum of the lower endpoint
};

__device__ __forceinline__ uint32_t basin(const Cell& c, uint32_t x) {
    return (cs_of(c) == x && cv_of(c) != x) ? cv_of(c) : x;
}

__device__ __forceinline__ Cell ld_cell_plain(const Cell* p) {
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
    return Cell{v.x, v.y};
}

// (a) filter: one thread per vertex, its +x/+y/+z edges; edges inside one
// basin are dropped (derivation C), the rest appended with warp-aggregated
// reservations.  Cells are static while this kernel runs.
__global__ void __launch_bounds__(256)
filter_edges_kernel(const Cell* __restrict__ C, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t n,
                    QEntry* __restrict__ q, uint64_t cap, unsigned long long* __restrict__ qctl) {
    constexpr int ITEMS = 4;  // vertices per thread per iteration (one queue reservation per 1024 vertices)
    __shared__ uint32_t s_warp[8];
    __shared__ unsigned long long s_base;
    const uint64_t sxy = uint64_t(nx) * ny;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * ITEMS;
    for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x * ITEMS; base < n; base += stride) {
        QEntry e[3 * ITEMS];
#pragma unroll
        for (int i = 0; i < 3 * ITEMS; ++i) e[i] = QEntry{0, 0xffffffffu, 0xffffffffu};  // holes
        int k = 0;
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const uint64_t u = base + uint64_t(it) * blockDim.x + threadIdx.x;
            if (u >= n) continue;
            const uint32_t x = uint32_t(u % nx);
            const uint64_t yz = u / nx;
            const uint32_t y = uint32_t(yz % ny), z = uint32_t(yz / ny);
            const Cell cu = ld_cell_plain(C + u);
            const uint32_t mu = basin(cu, uint32_t(u));
            const uint64_t ku = self_key(cu, uint32_t(u));
            const uint64_t off[3] = {1, nx, sxy};
            const bool ok[3] = {x + 1 < nx, y + 1 < ny, z + 1 < nz};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                bool keep = false;
                QEntry en{0, 0, 0};
                if (ok[d]) {
                    const uint32_t w = uint32_t(u + off[d]);
                    const Cell cw = ld_cell_plain(C + w);
                    const uint32_t mw = basin(cw, w);
                    if (mw != mu) {
                        const uint64_t kw = self_key(cw, w);
                        en = ku > kw ? QEntry{ku, mu, mw} : QEntry{kw, mw, mu};
                        keep = true;
                    }
                }
                // static register slots: entry (it, d) goes to slot it*3+d, compacted below
                e[it * 3 + d] = en;
                k += keep;
                if (!keep) e[it * 3 + d].m_hi = e[it * 3 + d].m_lo = 0xffffffffu;  // hole marker
            }
        }
        // CTA-aggregated reservation
        uint32_t incl = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < 8; ++w) {
                const uint32_t t = s_warp[w];
                s_warp[w] = tot;
                tot += t;
            }
            s_base = tot ? atomicAdd(qctl, (unsigned long long)tot) : 0;
        }
        __syncthreads();
        uint64_t pos = s_base + s_warp[warp] + incl - k;
        __syncthreads();  // s_warp / s_base are rewritten next iteration
#pragma unroll
        for (int i = 0; i < 3 * ITEMS; ++i) {
            if (e[i].m_hi == 0xffffffffu && e[i].m_lo == 0xffffffffu) continue;
            if (pos < cap) q[pos] = e[i];
            ++pos;
        }
    }
}

enum Phase : int { IDLE = 0, CLIMB_HI = 1, CLIMB_LO = 2, MERGE_LD = 3, MERGE_CAS = 4, DONE = 5 };

struct LaneStats {
    unsigned long long hops = 0, iters = 0, cas_fail = 0, skipped = 0;
};

// (b) merge: persistent warps; each lane holds one edge's state machine.
template <bool STATS>
__global__ void __launch_bounds__(256)
merge_queue_kernel(Cell* C, const QEntry* __restrict__ q, uint64_t cap, unsigned long long* __restrict__ qctl,
                   unsigned long long* __restrict__ stats) {
    const int lane = threadIdx.x & 31;
    const uint64_t qn_raw = *reinterpret_cast<volatile unsigned long long*>(qctl);
    const uint64_t qn = qn_raw < cap ? qn_raw : cap;
    unsigned long long* fetch = qctl + 1;
    if (STATS && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats + ST_QUEUED, qn_raw);

    constexpr uint64_t BATCH = 256;  // queue entries a warp takes per global atomic
    uint64_t pool_next = 0, pool_end = 0;  // warp-uniform
    bool exhausted = false;                // warp-uniform
    int phase = IDLE;
    uint64_t L = 0, ks = 0;
    uint32_t x = 0, xp = 0, m_lo = 0, rh = 0, u = 0, v = 0;
    bool has_prev = false;
    Cell c{0, 0}, cp{0, 0}, ch{0, 0}, cu{0, 0}, cv{0, 0}, desired{0, 0}, got{0, 0};
    LaneStats st;

    while (true) {
        // refill idle lanes from the queue (one atomic per warp)
        const uint32_t need = __ballot_sync(FULL_MASK, phase == IDLE);
        if (need) {
            if (pool_next == pool_end && !exhausted) {
                unsigned long long b = 0;
                if (lane == 0) b = atomicAdd(fetch, (unsigned long long)BATCH);
                b = __shfl_sync(FULL_MASK, b, 0);
                pool_next = b < qn ? b : qn;
                pool_end = b + BATCH < qn ? b + BATCH : qn;
                exhausted = pool_next == pool_end;
            }
            const uint32_t rank = __popc(need & ((1u << lane) - 1u));
            const uint64_t avail = pool_end - pool_next;
            if (phase == IDLE) {
                if (rank < avail) {
                    const QEntry e = q[pool_next + rank];
                    L = e.L;
                    x = e.m_hi;
                    m_lo = e.m_lo;
                    has_prev = false;
                    phase = CLIMB_HI;
                } else if (exhausted) {
                    phase = DONE;
                }
            }
            const uint64_t taken = avail < __popc(need) ? avail : __popc(need);
            pool_next += taken;
        }
        if (__ballot_sync(FULL_MASK, phase != DONE) == 0) break;

        // one memory round-trip per lane
        if (phase == CLIMB_HI || phase == CLIMB_LO) {
            c = ld_cell(C + x);
        } else if (phase == MERGE_LD) {
            cu = ld_cell(C + u);
            cv = ld_cell(C + v);
        } else if (phase == MERGE_CAS) {
            got = cas_cell(C + v, cv, desired);
        }

        // advance the state machine
        if (phase == CLIMB_HI || phase == CLIMB_LO) {
            if (cv_of(c) != x && c.lo <= L) {          // followable at level L
                if (STATS) st.hops++;
                if (has_prev && c.lo <= cp.lo)         // path splitting: prev skips x
                    cas_cell(C + xp, cp, Cell{cp.lo, (cp.hi & 0xffffffff00000000ull) | cv_of(c)});
                xp = x;
                cp = c;
                has_prev = true;
                x = cv_of(c);
            } else if (phase == CLIMB_HI) {
                rh = x;
                ch = c;
                x = m_lo;
                has_prev = false;
                phase = CLIMB_LO;
            } else if (x == rh) {                      // walks met: redundant edge
                if (STATS) st.skipped++;
                phase = IDLE;
            } else {
                u = rh;                                // Merge(T, r_hi, hi, r_lo) at level L
                v = x;
                ks = L;
                phase = MERGE_LD;
            }
        } else if (phase == MERGE_LD) {
            if (STATS) st.iters++;
            if (cv_of(cu) != u && cu.lo < ks) {        // l.2-4 (+ R4): climb u, restart
                u = cv_of(cu);
            } else if (cv_of(cv) != v && cv.lo < ks) { // l.5-8 (+ R4): climb v, restart
                v = cv_of(cv);
            } else if (u == v) {                       // l.9-10
                phase = IDLE;
            } else {
                if (self_key(cv, v) < self_key(cu, u)) {   // l.11-12: swap
                    const uint32_t t = u; u = v; v = t;
                    const Cell tc = cu; cu = cv; cv = tc;
                }
                desired = Cell{ks, (cv.hi & 0xffffffff00000000ull) | u};  // l.14: (s, u) into T[v]
                phase = MERGE_CAS;
            }
        } else if (phase == MERGE_CAS) {
            if (got.lo == cv.lo && got.hi == cv.hi) {
                const uint32_t vp = cv_of(cv);
                if (vp == v) {
                    phase = IDLE;                      // displaced a root (R5)
                } else {
                    ks = cv.lo;                        // l.15: Merge(T, u, s_v, v')
                    v = vp;
                    phase = MERGE_LD;
                }
            } else {
                if (STATS) st.cas_fail++;
                phase = MERGE_LD;                      // l.17: restart
            }
        }
    }
    if (STATS) {
        atomicAdd(stats + ST_PRE_HOPS, st.hops);
        atomicAdd(stats + ST_MERGE_ITERS, st.iters);
        atomicAdd(stats + ST_CAS_FAIL, st.cas_fail);
        atomicAdd(stats + ST_SKIPPED, st.skipped);
    }
}

}  // namespace

size_t queue_entry_bytes() { return sizeof(QEntry); }

void launch_filter_edges(const Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, void* q, uint64_t cap,
                         unsigned long long* qctl, int num_sms, cudaStream_t stream) {
    const uint64_t n = uint64_t(nx) * ny * nz;
    uint64_t blocks = (n + 255) / 256;
    const uint64_t lim = uint64_t(num_sms) * 8 * 32;
    if (blocks > lim) blocks = lim;
    filter_edges_kernel<<<uint32_t(blocks), 256, 0, stream>>>(C, nx, ny, nz, n, static_cast<QEntry*>(q), cap, qctl);
}

void launch_merge_queue(Cell* C, const void* q, uint64_t cap, unsigned long long* qctl, unsigned long long* stats,
                        int num_sms, cudaStream_t stream) {
    static int per_sm[2] = {0, 0};  // persistent grid: as many CTAs as fit on every SM
    const int t = stats ? 1 : 0;
    if (!per_sm[t]) {
        if (stats)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[t], merge_queue_kernel<true>, 256, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[t], merge_queue_kernel<false>, 256, 0);
        if (per_sm[t] < 1) per_sm[t] = 1;
    }
    const uint32_t blocks = uint32_t(num_sms) * per_sm[t];
    if (stats)
        merge_queue_kernel<true><<<blocks, 256, 0, stream>>>(C, static_cast<const QEntry*>(q), cap, qctl, stats);
    else
        merge_queue_kernel<false><<<blocks, 256, 0, stream>>>(C, static_cast<const QEntry*>(q), cap, qctl, stats);
}

}  // namespace mt
