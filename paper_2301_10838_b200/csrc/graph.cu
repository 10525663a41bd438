// graph.cu -- explicit graphs: the same hot path on an
// undirected graph given in CSR form (row[n+1], col[row[n]]), "f : V -> R on
// the vertices of a graph G = (V, E)".
//
//   graph_init  : K1 keys + steepest descent over the adjacency list
//                 (derivation B), then every regular cell is pointed at its
//                 descent root (derivation F) by in-place walks;
//   graph_edges : every edge {u, w} whose ends lie in different basins
//                 (derivation C) is queued once as (L, basin_hi, basin_lo);
//   merge_queue : the persistent Alg. 3 state machine of merge_cross.cu;
//   repair      : repair_diagram.cu with ordered essential classes (a graph
//                 may have many components).
// Self-loops never pass the strict key test and duplicate edges are
// harmless (Alg. 3 l.9-10 / the walk filter).
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

struct QEntryG {
    uint64_t L;
    uint32_t m_hi, m_lo;
};

__global__ void __launch_bounds__(256)
graph_descent_kernel(const float* __restrict__ f, const uint64_t* __restrict__ row, const uint32_t* __restrict__ col,
                     uint32_t n, uint32_t flip, Cell* __restrict__ C,
                     unsigned long long* __restrict__ counters) {
    bool bad = false;
    for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n; u += uint64_t(gridDim.x) * blockDim.x) {
        const float fu = __ldg(f + u);
        bad |= nonfinite(fu);
        const uint32_t ou = ord32(fu) ^ flip;
        const uint64_t ku = key_of(ou, uint32_t(u));
        uint64_t kb = ku;
        uint32_t best = uint32_t(u);
        for (uint64_t j = __ldg(row + u), e = __ldg(row + u + 1); j < e; ++j) {
            const uint32_t w = __ldg(col + j);
            const uint64_t kw = key_of(ord32(__ldg(f + w)) ^ flip, w);
            if (kw < kb) {
                kb = kw;
                best = w;
            }
        }
        C[u] = make_cell(ku, ou, best);   // (u, u, lowest lower neighbour) or the root (u, u, u)
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(counters + CTR_ERR, ERR_NONFINITE);
}

__global__ void __launch_bounds__(256) graph_compress_kernel(Cell* C, uint32_t n) {
    for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n; u += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = cv_of(ld_cell(C + u));
        if (v == uint32_t(u)) continue;
        uint32_t x = v;
        while (true) {
            const uint32_t y = cv_of(ld_cell(C + x));
            if (y == x) break;
            x = y;
        }
        if (x != v) st_cell_v(C + u, x);   // walkers only ever see pointers into the same tree
    }
}

__global__ void __launch_bounds__(256)
graph_edges_kernel(const uint64_t* __restrict__ row, const uint32_t* __restrict__ col, uint32_t n, const Cell* C,
                   QEntryG* __restrict__ q, uint64_t cap, unsigned long long* __restrict__ qlen,
                   unsigned long long* __restrict__ counters) {
    for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n; u += uint64_t(gridDim.x) * blockDim.x) {
        const Cell cu = ld_cell(C + u);
        const uint32_t bu = cv_of(cu);               // after compress: the basin (a root is its own)
        const uint64_t ku = self_key(cu, uint32_t(u));
        for (uint64_t j = __ldg(row + u), e = __ldg(row + u + 1); j < e; ++j) {
            const uint32_t w = __ldg(col + j);
            if (w <= u) continue;                    // each undirected edge once (and no self-loop)
            const Cell cw = ld_cell(C + w);
            const uint32_t bw = cv_of(cw);
            if (bw == bu) continue;
            const uint64_t kw = self_key(cw, w);
            const unsigned long long pos = atomicAdd(qlen, 1ull);
            if (pos < cap) q[pos] = ku > kw ? QEntryG{ku, bu, bw} : QEntryG{kw, bw, bu};
            else atomicOr(counters + CTR_ERR, ERR_CAPACITY);   // row[n] > n_adj: reported, never dropped
        }
    }
}

uint32_t grid_of(uint64_t n, int num_sms) {
    uint64_t b = (n + 255) / 256;
    const uint64_t lim = uint64_t(num_sms) * 32;
    return uint32_t(b > lim ? lim : (b ? b : 1));
}

}  // namespace

void launch_graph_init(const float* f, const uint64_t* row, const uint32_t* col, uint32_t n, uint32_t flip, Cell* C,
                       unsigned long long* counters, int num_sms, cudaStream_t stream) {
    if (!n) return;
    graph_descent_kernel<<<grid_of(n, num_sms), 256, 0, stream>>>(f, row, col, n, flip, C, counters);
    graph_compress_kernel<<<grid_of(n, num_sms), 256, 0, stream>>>(C, n);
}

void launch_graph_edges(const uint64_t* row, const uint32_t* col, uint32_t n, Cell* C, uint32_t* /*basin*/,
                        void* queue, uint64_t cap, unsigned long long* qlen, unsigned long long* counters,
                        int num_sms, cudaStream_t stream) {
    if (!n) return;
    graph_edges_kernel<<<grid_of(n, num_sms), 256, 0, stream>>>(row, col, n, C, static_cast<QEntryG*>(queue), cap,
                                                                qlen, counters);
}

}  // namespace mt
