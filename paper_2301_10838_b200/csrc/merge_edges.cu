// merge_edges.cu -- K3: the concurrent edge-merge phase of Alg. 1 (lines 4-8,
// PAPER.md:248-254) with Alg. 3 "Parallel Merge" as an
// iterative loop over 64-bit compare-and-swap (Alg. 2; the
// pair (s, v) packed in one word as in PAPER.md:389-394).
//
// Readings: R4 -- the climbs of Alg. 3 lines 2-8 only follow a
// cell that is not a root (T[x] = (x, x) has nowhere to go; as printed the
// call would recurse on identical arguments forever); R5 -- after a successful
// CAS the displaced pair is merged again (line 15) only if it was not a root;
// R6 -- strict "<" in the climbs as printed, over the (value, id) keys.
//
// Redundant-edge pre-filter (DESIGN.md derivation C'): for the edge (hi, lo)
// at level L = key(hi), follow cells whose saddle key is <= L from both ends
// (Alg. 4's walk at level L on the current store).  If both walks end at the
// same vertex the endpoints are already joined below L, the edge changes no
// sublevel component and is skipped; otherwise Merge(T, r_hi, hi, r_lo) joins
// the two components at level L (the same union Merge(T, hi, hi, lo) performs,
// started after the climbs it would make).  Any cell value ever written is a
// valid triplet, so stale reads only make the filter conservative.
//
// Memory: T cells are read with ld.relaxed.gpu (never a stale L1 line) and
// updated only by atom.cas.b64; f is immutable (read-only path).
#include "common.cuh"
#include "kernels.cuh"

namespace mt {

namespace {

// Alg. 4 walk on the current store: last vertex reached from x through cells
// (s, v) with key(s) <= L (roots stop).
__device__ __forceinline__ uint32_t climb_le(const uint64_t* T, const float* __restrict__ f, uint32_t flip,
                                             uint32_t x, uint64_t L) {
    while (true) {
        const uint64_t c = ld_relaxed(T + x);
        const uint32_t s = cell_s(c), v = cell_v(c);
        if (v == x) return x;                       // root
        if (keyf(f, s, flip) > L) return x;
        x = v;
    }
}

// Alg. 3, iterative.  Joins the components of u and v at level s (key ks).
__device__ __forceinline__ void merge(uint64_t* T, const float* __restrict__ f, uint32_t flip, uint32_t u,
                                      uint32_t s, uint64_t ks, uint32_t v) {
    while (true) {
        uint64_t cu = ld_relaxed(T + u);
        uint32_t su = cell_s(cu), up = cell_v(cu);
        if (up != u && keyf(f, su, flip) < ks) {    // l.2-4 (+ guard R4)
            u = up;
            continue;
        }
        uint64_t cv = ld_relaxed(T + v);
        uint32_t sv = cell_s(cv), vp = cell_v(cv);
        if (vp != v && keyf(f, sv, flip) < ks) {    // l.5-8 (+ guard R4)
            v = vp;
            continue;
        }
        if (u == v) return;                          // l.9-10
        if (keyf(f, v, flip) < keyf(f, u, flip)) {   // l.11-12: swap the triplets
            uint32_t t = u; u = v; v = t;
            uint64_t tc = cu; cu = cv; cv = tc;
            t = su; su = sv; sv = t;
            t = up; up = vp; vp = t;
        }
        const uint64_t old = cas64(T + v, cv, pack(s, u));  // l.14
        if (old == cv) {
            if (vp == v) return;                     // displaced a root (guard R5)
            s = sv;                                  // l.15: Merge(T, u, s_v, v')
            ks = keyf(f, sv, flip);
            v = vp;
        }
        // else l.17: start again with the same (u, s, v)
    }
}

__device__ __forceinline__ void merge_edge(uint64_t* T, const float* __restrict__ f, uint32_t flip, uint32_t a,
                                           uint64_t ka, uint32_t b) {
    const uint64_t kb = keyf(f, b, flip);
    const uint32_t hi = ka > kb ? a : b, lo = ka > kb ? b : a;   // Alg. 1 l.5-8 orientation
    const uint64_t L = ka > kb ? ka : kb;
    const uint32_t rh = climb_le(T, f, flip, hi, L);
    const uint32_t rl = climb_le(T, f, flip, lo, L);
    if (rh == rl) return;                            // already joined below L
    merge(T, f, flip, rh, hi, L, rl);
}

__global__ void __launch_bounds__(256)
merge_edges_kernel(uint64_t* T, const float* __restrict__ f, uint32_t nx, uint32_t ny, uint32_t nz,
                   uint64_t n, uint32_t flip) {
    const uint64_t sxy = uint64_t(nx) * ny;
    for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n;
         u += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t x = uint32_t(u % nx);
        const uint64_t yz = u / nx;
        const uint32_t y = uint32_t(yz % ny), z = uint32_t(yz / ny);
        const uint64_t ku = keyf(f, uint32_t(u), flip);
        if (x + 1 < nx) merge_edge(T, f, flip, uint32_t(u), ku, uint32_t(u + 1));
        if (y + 1 < ny) merge_edge(T, f, flip, uint32_t(u), ku, uint32_t(u + nx));
        if (z + 1 < nz) merge_edge(T, f, flip, uint32_t(u), ku, uint32_t(u + sxy));
    }
}

}  // namespace

void launch_merge_edges(uint64_t* T, const float* f, uint32_t nx, uint32_t ny, uint32_t nz, uint32_t flip,
                        int num_sms, cudaStream_t stream) {
    const uint64_t n = uint64_t(nx) * ny * nz;
    uint64_t blocks = (n + 255) / 256;
    const uint64_t cap = uint64_t(num_sms) * 8 * 64;  // grid-stride beyond this
    if (blocks > cap) blocks = cap;
    merge_edges_kernel<<<uint32_t(blocks), 256, 0, stream>>>(T, f, nx, ny, nz, n, flip);
}

}  // namespace mt
