// diagram_filter.cu -- persistence simplification of the diagram (SURVEY.md
// 8f row f2a): keep the finite pairs whose persistence |f(b) - f(a)| exceeds
// eps and every essential class.  "Short branches, i.e., branches such that
// |f(a) - f(b)| is small, can be intuitively interpreted as topological noise"
// (PAPER.md:14-15).  The persistence is evaluated in float32 -- the precision
// of the values, which are copied from the input (reading R14) -- and the
// oracle takes the same decision in the same precision.
//
// Single-pass ordered compaction: each CTA owns 1024 records (dynamic
// tickets), publishes its kept count, and finds its output offset by a
// decoupled look-back over its predecessors, so the records keep their order
// (finite pairs by birth vertex, then the essential classes).
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

constexpr int THREADS = 256;
constexpr int ITEMS = 4;
constexpr int TILE = THREADS * ITEMS;
constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(THREADS)
filter_kernel(const mt_pair* __restrict__ in, uint64_t n_fin, uint64_t n_all, float eps, mt_pair* __restrict__ out,
              uint64_t cap, unsigned long long* __restrict__ ctl, uint64_t* __restrict__ status, uint64_t ntiles) {
    __shared__ uint64_t s_tile, s_prefix;
    __shared__ uint32_t s_cnt[ITEMS * 8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(ctl, 1ull);
    __syncthreads();
    const uint64_t tile = s_tile;
    mt_pair rec[ITEMS];
    bool keep[ITEMS];
    uint32_t mask[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const uint64_t i = tile * TILE + uint64_t(k) * THREADS + threadIdx.x;
        keep[k] = false;
        if (i < n_all) {
            rec[k] = in[i];
            keep[k] = i >= n_fin || fabsf(rec[k].death - rec[k].birth) > eps;
        }
        mask[k] = __ballot_sync(FULL_MASK, keep[k]);
        if (lane == 0) s_cnt[k * 8 + warp] = __popc(mask[k]);
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t c = s_cnt[lane];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        s_cnt[lane] = incl - c;
        const uint64_t agg = __shfl_sync(FULL_MASK, incl, 31);
        uint64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_relaxed(status, ST_PRE | agg);
        } else {
            if (lane == 0) st_relaxed(status + tile, ST_AGG | agg);
            int64_t j = int64_t(tile) - 1;
            while (j >= 0) {
                const int64_t idx = j - lane;
                const uint64_t st = idx >= 0 ? ld_relaxed(status + idx) : ST_PRE;
                const uint64_t flag = st >> 62;
                const uint32_t pmask = __ballot_sync(FULL_MASK, flag == 2);
                const uint32_t xmask = __ballot_sync(FULL_MASK, flag == 0);
                const int first_p = pmask ? __ffs(pmask) - 1 : 31;
                const uint32_t upto = first_p == 31 ? FULL_MASK : ((2u << first_p) - 1u);
                if (xmask & upto) continue;
                uint64_t val = lane <= first_p ? (st & ST_VAL) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL_MASK, val, o);
                prefix += val;
                if (pmask) break;
                j -= 32;
            }
            if (lane == 0) st_relaxed(status + tile, ST_PRE | (prefix + agg));
        }
        if (lane == 0) {
            s_prefix = prefix;
            if (tile == ntiles - 1) ctl[1] = prefix + agg;   // records kept
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (!keep[k]) continue;
        const uint64_t pos = s_prefix + s_cnt[k * 8 + warp] + __popc(mask[k] & ((1u << lane) - 1u));
        if (pos < cap) out[pos] = rec[k];
    }
}

}  // namespace

uint64_t filter_tiles(uint64_t n) { return (n + TILE - 1) / TILE; }

void launch_filter_diagram(const mt_pair* in, uint64_t n_fin, uint64_t n_all, float eps, mt_pair* out, uint64_t cap,
                           unsigned long long* ctl, uint64_t* status, cudaStream_t stream) {
    const uint64_t ntiles = filter_tiles(n_all);
    if (ntiles == 0) return;
    filter_kernel<<<uint32_t(ntiles), THREADS, 0, stream>>>(in, n_fin, n_all, eps, out, cap, ctl, status, ntiles);
}

}  // namespace mt
