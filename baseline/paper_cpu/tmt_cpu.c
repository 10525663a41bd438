/* tmt_cpu.c -- the paper's own method on the host CPU: Alg. 1 with Alg. 2-5
 * run concurrently on all host cores with 64-bit compare-and-swap on the packed store
 * T[u] = s << 32 | v, the analogue of the paper's OpenMP backend column
 * (SURVEY.md 8(d) "optional second CPU baseline").
 *
 * A REPORTED BASELINE, not the oracle and not the product: bench.py times it beside the GPU path;
 * tests check it against the oracle O1.  It shares no code with either.
 *
 * Readings: vertices are ordered by key(u) = ord(f[u]) << 32 | u with -0
 * canonicalised to +0 (R1, R2; the split tree complements ord, R16); Alg. 3 climbs only through
 * non-root cells (R4) and re-merges a displaced pair only if it was not a root (R5); Alg. 4
 * returns the vertex its walk stopped at (R20).  The three phases are the paper's three
 * parallel_for's: init over vertices, merge over edges, repair over vertices.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>

enum { TC_OK = 0, TC_INVALID = 1, TC_TOO_LARGE = 2, TC_NONFINITE = 3, TC_NOMEM = 8 };

static inline uint32_t ord_of(float x, uint32_t flip) {
    union { float f; uint32_t u; } c = {x};
    uint32_t b = c.u == 0x80000000u ? 0u : c.u;
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return b ^ flip;
}
static inline uint64_t pack(uint32_t s, uint32_t v) { return ((uint64_t)s << 32) | v; }
static inline uint32_t s_of(uint64_t c) { return (uint32_t)(c >> 32); }
static inline uint32_t v_of(uint64_t c) { return (uint32_t)c; }
static inline uint64_t ld(const uint64_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }

/* Alg. 3 Merge(T, u, s, v) with Alg. 2's CAS (concurrent form): K holds the order keys. */
static void merge(uint64_t* T, const uint64_t* K, uint32_t u, uint32_t s, uint32_t v) {
    for (;;) {
        uint64_t cu = ld(T + u);
        if (v_of(cu) != u && K[s_of(cu)] < K[s]) {        /* l.2-4 (+ R4) */
            u = v_of(cu);
            continue;
        }
        uint64_t cv = ld(T + v);
        if (v_of(cv) != v && K[s_of(cv)] < K[s]) {        /* l.5-8 (+ R4) */
            v = v_of(cv);
            continue;
        }
        if (u == v) return;                               /* l.9-10 */
        if (K[v] < K[u]) {                                /* l.11-12 */
            uint32_t t = u;
            u = v;
            v = t;
            cv = cu;
        }
        uint64_t expect = cv;                             /* l.14: T[v] <- (s, u) */
        if (__atomic_compare_exchange_n(T + v, &expect, pack(s, u), 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
            if (v_of(cv) == v) return;                    /* R5: displaced a root */
            s = s_of(cv);                                 /* l.15: Merge(T, u, s_v, v') */
            v = v_of(cv);
        }                                                 /* else l.17: restart */
    }
}

/* f: float32[nx*ny*nz], x fastest; conn 4 (nz == 1) or 6; flip: 0 merge tree, 1 split tree.
 * T: uint64[n] output (s << 32 | v).  threads <= 0: all cores. */
int tmt_cpu_merge_tree(const float* f, uint32_t nx, uint32_t ny, uint32_t nz, int conn, int split, uint64_t* T,
                       int threads) {
    if (!f || !T || (conn != 4 && conn != 6) || (conn == 4 && nz != 1)) return TC_INVALID;
    const uint64_t n = (uint64_t)nx * ny * nz;
    if (n > 0xffffffffull) return TC_TOO_LARGE;
    if (threads > 0) omp_set_num_threads(threads);
    const uint32_t flip = split ? 0xffffffffu : 0u;
    uint64_t* K = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!K) return TC_NOMEM;
    int bad = 0;
    const uint64_t sxy = (uint64_t)nx * ny;
    /* order keys and Alg. 1 l.2-3: T[u] = (u, u) */
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const float x = f[i];
        if (!isfinite(x)) bad = 1;
        K[i] = ((uint64_t)ord_of(x, flip) << 32) | (uint64_t)i;
        T[i] = pack((uint32_t)i, (uint32_t)i);
    }
    if (bad) {
        free(K);
        return TC_NONFINITE;
    }
    /* Alg. 1 l.4-8: every edge, Merge(T, hi, hi, lo) (each vertex enumerates its +x, +y, +z edges) */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const uint32_t u = (uint32_t)i;
        const uint64_t x = (uint64_t)i % nx, y = ((uint64_t)i / nx) % ny, z = (uint64_t)i / sxy;
        const uint32_t nb[3] = {x + 1 < nx ? u + 1 : u, y + 1 < ny ? u + nx : u,
                                (conn == 6 && z + 1 < nz) ? (uint32_t)(u + sxy) : u};
        for (int d = 0; d < 3; ++d) {
            const uint32_t w = nb[d];
            if (w == u) continue;
            if (K[w] < K[u]) merge(T, K, u, u, w);
            else merge(T, K, w, w, u);
        }
    }
    /* Alg. 1 l.9-11, Alg. 5 with Alg. 4 (R20): T[u] = (s, Rep(u, key(s))), in place */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const uint32_t u0 = (uint32_t)i;
        const uint64_t c0 = ld(T + u0);
        const uint64_t a = K[s_of(c0)];
        uint32_t u = u0;
        uint64_t c = c0;
        while (K[s_of(c)] <= a && s_of(c) != v_of(c)) {
            u = v_of(c);
            c = ld(T + u);
        }
        if (u != u0) __atomic_store_n(T + u0, pack(s_of(c0), u), __ATOMIC_RELAXED);
    }
    free(K);
    return TC_OK;
}

int tmt_cpu_max_threads(void) { return omp_get_max_threads(); }
