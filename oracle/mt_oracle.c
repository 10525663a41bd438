/*
 * oracle/mt_oracle.c -- O1: serial union-find (Kruskal-style) merge tree +
 * elder-rule 0-dimensional persistence pairs, written from the paper's plain
 * definitions.  TEST INFRASTRUCTURE ONLY: nothing under paper_2301_10838_b200/
 * may include, link or call this file; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may.  It shares no code,
 * header, table or constant with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   - merge tree of f on a graph G=(V,E), sublevel sets G_c = {v : f(v) <= c}
 *     (Sec. 2.1 "Merge Trees");
 *   - computed "in O(m log n) time ... using the union-find data structure.
 *     First, one sorts the vertices by values of the function.  Then the
 *     algorithm goes over the sorted vertices ... (1) local minimum creates a
 *     new component; (2) belongs to exactly one component; (3) multiple
 *     components are merged";
 *   - emitted as the normalized, minimal triplet representation
 *     (Sec. 2.1 "Triplet merge trees"): one triplet (u,s,v)
 *     per vertex u, v = deepest vertex of u's component of G_{f(s)};
 *     (u,u,u) for the minimum of each connected component;
 *   - persistence pairs (f(a), f(b)), one per branch (a = minimum,
 *     b = saddle); which branch ends at a saddle follows the
 *     branch semantics "a branch ... is created and ... merged with an older
 *     component": the younger (higher) minimum dies.
 *
 * Readings: ties in f are broken by vertex
 * id ascending (R1, simulation of simplicity); -0.0 == +0.0 as IEEE values
 * (R2); NaN/Inf rejected (R3); split tree = merge tree of -f with the same
 * ascending-id tie break (R16); grid ids x-fastest (R10); 4-/6-neighbour grid
 * graph without periodic faces (R9).  Comparisons are plain IEEE float
 * compares (no bit tricks); build WITHOUT -ffast-math.
 *
 * Packing of the output cell ("a pair can be packed into a
 * 64-bit integer"): T[u] = (uint64)s << 32 | v  (reading R11: s high).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_TOO_LARGE 2
#define OR_NONFINITE 3
#define OR_NOMEM 8
#define OR_CAPACITY 9

typedef struct {
    uint32_t birth_v, death_v;
    float birth, death;
} oracle_pair;

typedef struct {
    float g;     /* g = f (merge tree) or -f (split tree) */
    uint32_t id; /* vertex id, the tie break */
} vkey;

/* less(a,b) := g(a) < g(b) || (g(a) == g(b) && a < b)    (reading R1) */
static int key_less(float ga, uint32_t a, float gb, uint32_t b) {
    if (ga < gb) return 1;
    if (ga == gb && a < b) return 1;
    return 0;
}

static int cmp_vkey(const void *pa, const void *pb) {
    const vkey *a = (const vkey *)pa, *b = (const vkey *)pb;
    if (key_less(a->g, a->id, b->g, b->id)) return -1;
    if (key_less(b->g, b->id, a->g, a->id)) return 1;
    return 0;
}

/* Disjoint sets: parent pointers, find with path halving,
 * union by size. */
static uint32_t ds_find(uint32_t *parent, uint32_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

/* The graph: a grid (implicit 4/6-neighbour adjacency) or an explicit CSR
 * adjacency list (row[n+1], col[]), SURVEY.md 8f f4 / PAPER.md:128-131. */
typedef struct {
    uint32_t nx, ny, nz;
    const uint64_t *row;  /* NULL for a grid */
    const uint32_t *col;
} graph_t;

/* Grid neighbours of u: +-x, +-y, +-z inside the box (reading R9, R10). */
static int grid_neighbours(uint64_t u, uint32_t nx, uint32_t ny, uint32_t nz, uint32_t out[6]) {
    uint64_t x = u % nx, y = (u / nx) % ny, z = u / ((uint64_t)nx * ny);
    uint64_t sxy = (uint64_t)nx * ny;
    int k = 0;
    if (x > 0) out[k++] = (uint32_t)(u - 1);
    if (x + 1 < nx) out[k++] = (uint32_t)(u + 1);
    if (y > 0) out[k++] = (uint32_t)(u - nx);
    if (y + 1 < ny) out[k++] = (uint32_t)(u + nx);
    if (z > 0) out[k++] = (uint32_t)(u - sxy);
    if (z + 1 < nz) out[k++] = (uint32_t)(u + sxy);
    return k;
}

/*
 * oracle_merge_tree: returns OR_* status.
 *   f        : n = nx*ny*nz float32 values, x fastest
 *   conn     : 4 (2D, nz must be 1) or 6
 *   split    : 0 = merge (join) tree of f; 1 = split tree (merge tree of -f)
 *   T        : out, n words (s << 32 | v), may be NULL
 *   pairs    : out, room for pairs_cap records, may be NULL; finite pairs by
 *              ascending birth vertex, then essential classes by ascending
 *              vertex (death_v = birth_v, death = +inf)
 *   pairs_cap: records `pairs` holds (OR_CAPACITY when the diagram needs more; a grid
 *              has at most ceil(n/2) records: strict minima are an independent set)
 *   n_pairs, n_ess : out counts
 */
static int sweep(const float *f, uint64_t n, const graph_t *G, int split, uint64_t *T, oracle_pair *pairs,
                 uint64_t pairs_cap, uint64_t *n_pairs, uint64_t *n_ess);

int oracle_merge_tree(const float *f, uint32_t nx, uint32_t ny, uint32_t nz, int conn, int split,
                      uint64_t *T, oracle_pair *pairs, uint64_t pairs_cap, uint64_t *n_pairs, uint64_t *n_ess) {
    if (!f && (uint64_t)nx * ny * nz != 0) return OR_INVALID;
    if (conn != 4 && conn != 6) return OR_INVALID;
    if (conn == 4 && nz != 1) return OR_INVALID;
    graph_t G = {nx, ny, nz, NULL, NULL};
    return sweep(f, (uint64_t)nx * ny * nz, &G, split, T, pairs, pairs_cap, n_pairs, n_ess);
}

/* Explicit graph: the neighbours of u are col[row[u] .. row[u+1]). */
int oracle_merge_tree_graph(const float *f, uint32_t n, const uint64_t *row, const uint32_t *col, int split,
                            uint64_t *T, oracle_pair *pairs, uint64_t pairs_cap, uint64_t *n_pairs,
                            uint64_t *n_ess) {
    if (n && (!f || !row)) return OR_INVALID;
    for (uint32_t u = 0; u < n; u++)
        for (uint64_t j = row[u]; j < row[u + 1]; j++)
            if (col[j] >= n) return OR_INVALID;
    graph_t G = {n, 1, 1, row, col};
    return sweep(f, n, &G, split, T, pairs, pairs_cap, n_pairs, n_ess);
}

static int sweep(const float *f, uint64_t n, const graph_t *G, int split, uint64_t *T, oracle_pair *pairs,
                 uint64_t pairs_cap, uint64_t *n_pairs, uint64_t *n_ess) {
    if (n > 4294967295ull) return OR_TOO_LARGE; /* 32-bit ids */
    if (n_pairs) *n_pairs = 0;
    if (n_ess) *n_ess = 0;
    if (n == 0) return OR_OK;
    for (uint64_t i = 0; i < n; i++)
        if (!isfinite(f[i])) return OR_NONFINITE;

    vkey *order = (vkey *)malloc(n * sizeof(vkey));
    uint32_t *parent = (uint32_t *)malloc(n * sizeof(uint32_t));
    uint32_t *size = (uint32_t *)malloc(n * sizeof(uint32_t));
    uint32_t *cmin = (uint32_t *)malloc(n * sizeof(uint32_t));  /* deepest vertex of a set (valid at roots) */
    uint32_t *death = (uint32_t *)malloc(n * sizeof(uint32_t)); /* saddle where a minimum's branch ends */
    uint8_t *done = (uint8_t *)calloc(n, 1);                      /* swept already <=> less(w, u) */
    uint64_t *Tl = T ? T : (uint64_t *)malloc(n * sizeof(uint64_t));
    if (!order || !parent || !size || !cmin || !death || !done || !Tl) {
        free(order); free(parent); free(size); free(cmin); free(death); free(done);
        if (!T) free(Tl);
        return OR_NOMEM;
    }
    float *g = (float *)malloc(n * sizeof(float)); /* g by vertex id */
    if (!g) { free(order); free(parent); free(size); free(cmin); free(death); free(done); if (!T) free(Tl); return OR_NOMEM; }

    for (uint64_t i = 0; i < n; i++) {
        g[i] = split ? -f[i] : f[i];
        order[i].g = g[i];
        order[i].id = (uint32_t)i;
        death[i] = UINT32_MAX;
    }
    /* "First, one sorts the vertices by values of the function". */
    qsort(order, n, sizeof(vkey), cmp_vkey);

    uint32_t nb[6];
    uint64_t rcap = 64;
    uint32_t *R = (uint32_t *)malloc(rcap * sizeof(uint32_t));
    if (!R) { free(order); free(parent); free(size); free(cmin); free(death); free(done); free(g); if (!T) free(Tl); return OR_NOMEM; }
    for (uint64_t k = 0; k < n; k++) {
        uint32_t u = order[k].id;
        const uint32_t *adj;
        uint64_t deg;
        if (G->row) {
            adj = G->col + G->row[u];
            deg = G->row[u + 1] - G->row[u];
        } else {
            deg = (uint64_t)grid_neighbours(u, G->nx, G->ny, G->nz, nb);
            adj = nb;
        }
        if (deg > rcap) {
            while (rcap < deg) rcap *= 2;
            uint32_t *R2 = (uint32_t *)realloc(R, rcap * sizeof(uint32_t));
            if (!R2) { free(R); free(order); free(parent); free(size); free(cmin); free(death); free(done); free(g); if (!T) free(Tl); return OR_NOMEM; }
            R = R2;
        }
        /* R = distinct components of the lower neighbours of u */
        uint64_t nr = 0;
        for (uint64_t j = 0; j < deg; j++) {
            uint32_t w = adj[j];
            if (!done[w]) continue; /* not yet in the sublevel set <=> !less(w,u) (self-loops: not done) */
            uint32_t r = ds_find(parent, w);
            int dup = 0;
            for (uint64_t t = 0; t < nr; t++) dup |= (R[t] == r);
            if (!dup) R[nr++] = r;
        }
        done[u] = 1;
        if (nr == 0) {
            /* (1) local minimum: "creates a new connected component" */
            parent[u] = u;
            size[u] = 1;
            cmin[u] = u;
            continue;
        }
        /* m* = deepest vertex over the merged components (the oldest branch). */
        uint32_t mstar = cmin[R[0]];
        for (uint64_t t = 1; t < nr; t++) {
            uint32_t m = cmin[R[t]];
            if (key_less(g[m], m, g[mstar], mstar)) mstar = m;
        }
        /* (3) merge: every younger minimum's branch ends at saddle u, merged
         * into the branch of m* (elder rule; triplet (m, u, m*)). */
        for (uint64_t t = 0; t < nr; t++) {
            uint32_t m = cmin[R[t]];
            if (m != mstar) {
                Tl[m] = ((uint64_t)u << 32) | mstar;
                death[m] = u;
            }
        }
        /* u itself: (u, u, m*) -- m* is the deepest vertex of u's component
         * of G_{f(u)} (minimality). */
        Tl[u] = ((uint64_t)u << 32) | mstar;
        /* union u and all of R, the union's deepest vertex is m* */
        uint32_t root = R[0];
        for (uint64_t t = 1; t < nr; t++) {
            uint32_t a = root, b = R[t];
            if (size[a] < size[b]) { uint32_t tmp = a; a = b; b = tmp; }
            parent[b] = a;
            size[a] += size[b];
            root = a;
        }
        parent[u] = root;
        size[root] += 1;
        cmin[root] = mstar;
    }
    /* Survivors: the minimum of each connected component, triplet (m,m,m)
     * (PAPER.md:190-191), essential class (f(m), +inf). */
    uint64_t np = 0, ne = 0;
    /* The deepest vertex of each final set is a minimum that never died:
     * exactly one per connected component. */
    for (uint64_t u = 0; u < n; u++) {
        uint32_t r = ds_find(parent, (uint32_t)u);
        if (cmin[r] == u) Tl[u] = ((uint64_t)u << 32) | u;
    }
    for (uint64_t u = 0; u < n; u++) {
        if (death[u] != UINT32_MAX) np++;
        else if (cmin[ds_find(parent, (uint32_t)u)] == u) ne++;
    }
    int status = OR_OK;
    if (pairs && np + ne > pairs_cap) status = OR_CAPACITY;
    if (pairs && status == OR_OK) {
        uint64_t k = 0;
        for (uint64_t u = 0; u < n; u++) {
            if (death[u] != UINT32_MAX) {
                pairs[k].birth_v = (uint32_t)u;
                pairs[k].death_v = death[u];
                pairs[k].birth = f[u];          /* values copied from the input f (reading R14) */
                pairs[k].death = f[death[u]];
                k++;
            }
        }
        for (uint64_t u = 0; u < n; u++) {
            uint32_t r = ds_find(parent, (uint32_t)u);
            if (cmin[r] == u) {
                pairs[k].birth_v = (uint32_t)u;
                pairs[k].death_v = (uint32_t)u;
                pairs[k].birth = f[u];
                pairs[k].death = INFINITY;
                k++;
            }
        }
    }
    if (n_pairs) *n_pairs = np;
    if (n_ess) *n_ess = ne;

    free(R);
    free(order); free(parent); free(size); free(cmin); free(death); free(done); free(g);
    if (!T) free(Tl);
    return status;
}

/* Version tag so the Python loader can detect a stale build. */
int oracle_abi_version(void) { return 1; }

/* ------------------------------------------------------------------------------------------
 * O4: the triplet of ONE vertex from the definition, by bounded floods (for sampled checks of
 * full-size outputs that O1 cannot process in a test).  PAPER.md:185-200 (Sec. 2.1, "Triplet
 * merge trees"): T[u] = (s, v) with f(v) < f(u) <= f(s), u and v in one component of the
 * sublevel set G_{f(s)}, v the deepest vertex of that component (reading R12: of u's
 * component), s = u unless u is a local minimum; a minimum's s is the lowest level at which
 * its component reaches a deeper vertex; the component minimum is
 * (u, u, u).  All comparisons are key_less (readings R1, R2, R16).
 *   - s: a Prim-style flood from u that always enters the lowest vertex adjacent to the
 *     region; the first deeper vertex it enters is reached at the smallest possible level,
 *     and that level is the largest key entered so far (its vertex is s).  If u has a lower
 *     neighbour the flood's first step enters it and s = u.
 *   - v: breadth-first search of u's component of {x : key(x) <= key(s)}, keeping the least.
 * Returns 1 and (s, v) on success, 0 when a flood would visit more than `cap` vertices
 * (the caller skips that sample), negative on bad arguments or memory.
 * ------------------------------------------------------------------------------------------ */
/* O4 works with 64-bit vertex ids so that it also checks grids past 2^32 vertices (SURVEY.md 8f
 * row f3; PAPER.md:389-396 limits the paper's ids to 32 bits).  key_less / the grid adjacency
 * are the ones above, widened. */
typedef struct {
    float g;
    uint64_t id;
} vkey64;

static int key_less64(float ga, uint64_t a, float gb, uint64_t b) {   /* reading R1, as key_less */
    if (ga < gb) return 1;
    if (ga == gb && a < b) return 1;
    return 0;
}

static int grid_neighbours64(uint64_t u, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t out[6]) {
    uint64_t x = u % nx, y = (u / nx) % ny, z = u / ((uint64_t)nx * ny);
    uint64_t sxy = (uint64_t)nx * ny;
    int k = 0;
    if (x > 0) out[k++] = u - 1;
    if (x + 1 < nx) out[k++] = u + 1;
    if (y > 0) out[k++] = u - nx;
    if (y + 1 < ny) out[k++] = u + nx;
    if (z > 0) out[k++] = u - sxy;
    if (z + 1 < nz) out[k++] = u + sxy;
    return k;
}

typedef struct { uint64_t *keys; uint64_t mask, count; } idset;

static int set_init(idset *S, uint64_t cap) {
    uint64_t m = 1;
    while (m < 2 * cap + 2) m <<= 1;
    S->keys = (uint64_t *)malloc(m * sizeof(uint64_t));
    if (!S->keys) return 0;
    memset(S->keys, 0xff, m * sizeof(uint64_t));
    S->mask = m - 1;
    S->count = 0;
    return 1;
}
/* 1 if inserted, 0 if already present (ids are < 2^63: all-ones marks a free slot) */
static int set_add(idset *S, uint64_t x) {
    uint64_t h = (x * 0x9E3779B97F4A7C15ull) >> 20;
    for (;; ++h) {
        uint64_t *k = &S->keys[h & S->mask];
        if (*k == ~0ull) { *k = x; ++S->count; return 1; }
        if (*k == x) return 0;
    }
}

typedef struct { vkey64 *a; uint64_t n, cap; } vheap;
static int heap_less(const vkey64 *x, const vkey64 *y) { return key_less64(x->g, x->id, y->g, y->id); }
static int heap_push(vheap *H, vkey64 k) {
    if (H->n == H->cap) {
        uint64_t nc = H->cap ? 2 * H->cap : 1024;
        vkey64 *na = (vkey64 *)realloc(H->a, nc * sizeof(vkey64));
        if (!na) return 0;
        H->a = na;
        H->cap = nc;
    }
    uint64_t i = H->n++;
    H->a[i] = k;
    while (i && heap_less(&H->a[i], &H->a[(i - 1) / 2])) {
        vkey64 t = H->a[i]; H->a[i] = H->a[(i - 1) / 2]; H->a[(i - 1) / 2] = t;
        i = (i - 1) / 2;
    }
    return 1;
}
static vkey64 heap_pop(vheap *H) {
    vkey64 top = H->a[0];
    H->a[0] = H->a[--H->n];
    uint64_t i = 0;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < H->n && heap_less(&H->a[l], &H->a[m])) m = l;
        if (r < H->n && heap_less(&H->a[r], &H->a[m])) m = r;
        if (m == i) break;
        vkey64 t = H->a[i]; H->a[i] = H->a[m]; H->a[m] = t;
        i = m;
    }
    return top;
}

int oracle_triplet_at64(const float *f, uint32_t nx, uint32_t ny, uint32_t nz, int conn, int split, uint64_t u,
                        uint64_t cap, uint64_t *s_out, uint64_t *v_out) {
    const uint64_t sxy = (uint64_t)nx * ny;
    if (!f || (conn != 4 && conn != 6) || (conn == 4 && nz != 1) || sxy == 0 || nz > (1ull << 63) / sxy) return -1;
    const uint64_t n = sxy * nz;
    if (u >= n) return -1;
    const float sg = split ? -1.0f : 1.0f;
#define G_OF(x) (sg * f[(x)] + 0.0f)
    uint64_t nb[6];
    int rc = -2;
    idset S = {0}, B = {0};
    vheap H = {0};
    uint64_t *queue = NULL;
    if (!set_init(&S, cap) || !set_init(&B, cap)) goto out;
    /* s: Prim flood from u */
    const float gu = G_OF(u);
    uint64_t s = u;
    int found = 0;
    float gs = gu;
    set_add(&S, u);
    if (!heap_push(&H, (vkey64){gu, u})) goto out;
    while (H.n) {
        vkey64 x = heap_pop(&H);
        if (key_less64(x.g, x.id, gu, u)) { found = 1; break; }   /* entered a deeper vertex */
        if (key_less64(gs, s, x.g, x.id)) { gs = x.g; s = x.id; } /* the level rises to key(x) */
        int d = grid_neighbours64(x.id, nx, ny, nz, nb);
        for (int i = 0; i < d; ++i)
            if (set_add(&S, nb[i])) {
                if (S.count > cap) { rc = 0; goto out; }
                if (!heap_push(&H, (vkey64){G_OF(nb[i]), nb[i]})) goto out;
            }
    }
    if (!found) {                 /* the whole component lies above u: u is its minimum */
        *s_out = u;
        *v_out = u;
        rc = 1;
        goto out;
    }
    /* v: deepest vertex of u's component of {x : key(x) <= key(s)} */
    queue = (uint64_t *)malloc((cap + 1) * sizeof(uint64_t));
    if (!queue) goto out;
    uint64_t qh = 0, qt = 0;
    uint64_t v = u;
    float gv = gu;
    set_add(&B, u);
    queue[qt++] = u;
    while (qh < qt) {
        const uint64_t x = queue[qh++];
        const float gx = G_OF(x);
        if (key_less64(gx, x, gv, v)) { gv = gx; v = x; }
        int d = grid_neighbours64(x, nx, ny, nz, nb);
        for (int i = 0; i < d; ++i) {
            const float gy = G_OF(nb[i]);
            if (!key_less64(gy, nb[i], gs, s) && nb[i] != s) continue;   /* above level key(s) */
            if (set_add(&B, nb[i])) {
                if (B.count > cap) { rc = 0; goto out; }
                queue[qt++] = nb[i];
            }
        }
    }
    *s_out = s;
    *v_out = v;
    rc = 1;
out:
#undef G_OF
    free(S.keys);
    free(B.keys);
    free(H.a);
    free(queue);
    return rc;
}

/* the 32-bit form (grids below 2^32 - 1 vertices) */
int oracle_triplet_at(const float *f, uint32_t nx, uint32_t ny, uint32_t nz, int conn, int split, uint32_t u,
                      uint64_t cap, uint32_t *s_out, uint32_t *v_out) {
    if ((uint64_t)nx * ny * nz >= 0xffffffffull) return -1;
    uint64_t s = 0, v = 0;
    const int rc = oracle_triplet_at64(f, nx, ny, nz, conn, split, u, cap, &s, &v);
    if (rc == 1) {
        *s_out = (uint32_t)s;
        *v_out = (uint32_t)v;
    }
    return rc;
}
