/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this file's shared object.  It shares no code
 * with the CUDA path (paper_2207_07847_b200/csrc) and must never be linked
 * into it.
 *
 * Plain, sequential C transcription of the aggregation step of PAPER.md §2.2
 * ("Aggregation"):
 *
 *   "we use the maximal weighted matching (MWM) ... MWM visits the vertices in
 *    the graph in random order and matches each unaggregated vertex to its
 *    neighbor with the maximal edge weight."
 *   "If there are leftover nodes after performing the matching scheme, we add
 *    each leftover node to the aggregation that has its heaviest neighbor."
 *
 *
 * and of the coarse graph implied by P^T L P (Eq. def:P and the coarse blocks
 * of Eq. def:L_ell): coarse weight(A,B) = sum of fine weights between A and B.
 *
 * Readings:
 *  R1  "random order" = vertices sorted by the counter-based key
 *      (visit_priority(seed, level, v), v); the same generator is implemented
 *      independently on the GPU side.
 *  R2  ties in "maximal edge weight" (and in "heaviest neighbor") are broken
 *      toward the lowest vertex index.
 *  R3  aggregates are numbered in increasing order of the smaller vertex of
 *      their matched pair; a leftover joins the aggregate of its heaviest
 *      neighbour (no size cap: the paper states none).
 *  R4  coarse weights are summed left-to-right in increasing (u, v) order of
 *      the contributing fine (row, column) pairs (fixes the fp64 rounding so
 *      the hierarchy is reproducible bit for bit).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t mix64(uint64_t z) {
    /* splitmix64 finaliser (Steele, Lea, Flood 2014) */
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_visit_priority(uint64_t seed, int32_t level, int64_t v) {
    return mix64(mix64(seed + 0x9E3779B97F4A7C15ULL * (uint64_t)(level + 1)) ^ (uint64_t)v);
}

typedef struct { uint64_t key; int64_t v; } keyed_t;

static int cmp_keyed(const void* a, const void* b) {
    const keyed_t* x = (const keyed_t*)a;
    const keyed_t* y = (const keyed_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->v != y->v) return x->v < y->v ? -1 : 1;
    return 0;
}

/* Visit order of level `level` (R1). order_out[k] = k-th visited vertex. */
void oracle_visit_order(int64_t n, uint64_t seed, int32_t level, int64_t* order_out) {
    keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t v = 0; v < n; ++v) { kv[v].key = oracle_visit_priority(seed, level, v); kv[v].v = v; }
    qsort(kv, (size_t)n, sizeof(keyed_t), cmp_keyed);
    for (int64_t k = 0; k < n; ++k) order_out[k] = kv[k].v;
    free(kv);
}

/*
 * MWM aggregation of one level.
 *   rowptr/col/w : symmetric CSR, columns strictly increasing per row.
 *   order        : visit order (n entries) -- e.g. from oracle_visit_order,
 *                  or forced by a test (§3.1 example).
 *   mate_out     : matched partner or -1 (leftover).
 *   agg_out      : aggregate id of each vertex.
 * Returns the number of aggregates, or -1 if some vertex has no neighbour.
 */
int64_t oracle_mwm(int64_t n, const int64_t* rowptr, const int32_t* col, const double* w,
                   const int64_t* order, int32_t* mate_out, int32_t* agg_out) {
    for (int64_t v = 0; v < n; ++v) { mate_out[v] = -1; agg_out[v] = -1; }
    /* sequential visit */
    for (int64_t k = 0; k < n; ++k) {
        int64_t v = order[k];
        if (mate_out[v] != -1) continue;
        int64_t best = -1; double bw = 0.0;
        for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e) {
            int64_t u = col[e];
            if (u == v || mate_out[u] != -1) continue;
            if (best == -1 || w[e] > bw) { best = u; bw = w[e]; }  /* R2: ascending cols => lowest index on ties */
        }
        if (best != -1) { mate_out[v] = (int32_t)best; mate_out[best] = (int32_t)v; }
    }
    /* number the matched pairs by their smaller vertex (R3) */
    int64_t na = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (mate_out[v] > v) { agg_out[v] = (int32_t)na; agg_out[mate_out[v]] = (int32_t)na; ++na; }
    }
    /* leftovers join the aggregate of their heaviest neighbour */
    for (int64_t v = 0; v < n; ++v) {
        if (mate_out[v] != -1) continue;
        int64_t best = -1; double bw = 0.0;
        for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e) {
            int64_t u = col[e];
            if (u == v) continue;
            if (best == -1 || w[e] > bw) { best = u; bw = w[e]; }
        }
        if (best == -1) return -1;               /* isolated vertex: not a connected graph */
        agg_out[v] = agg_out[best];               /* best is matched (maximality) */
    }
    return na;
}

/*
 * Coarse (Galerkin) graph of an aggregation: weight(A,B) = sum over fine
 * edges (u,v), u in A, v in B, A != B (R4 summation order).  Output CSR with
 * sorted columns; ccol/cw must hold at least nnz(fine) entries.
 * Returns the coarse nnz.
 */
int64_t oracle_coarsen(int64_t n, const int64_t* rowptr, const int32_t* col, const double* w,
                       const int32_t* agg, int64_t nc,
                       int64_t* crowptr, int32_t* ccol, double* cw) {
    /* members of each aggregate in increasing vertex order (counting sort) */
    int64_t* start = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    int64_t* members = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t v = 0; v < n; ++v) start[agg[v] + 1]++;
    for (int64_t a = 0; a < nc; ++a) start[a + 1] += start[a];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
    for (int64_t a = 0; a < nc; ++a) fill[a] = start[a];
    for (int64_t v = 0; v < n; ++v) members[fill[agg[v]]++] = v;

    double* acc = (double*)calloc((size_t)(nc > 0 ? nc : 1), sizeof(double));
    int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
    int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
    for (int64_t a = 0; a < nc; ++a) mark[a] = -1;
    int64_t nnz = 0;
    crowptr[0] = 0;
    for (int64_t a = 0; a < nc; ++a) {
        int64_t nt = 0;
        for (int64_t k = start[a]; k < start[a + 1]; ++k) {
            int64_t u = members[k];
            for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
                int64_t b = agg[col[e]];
                if (b == a) continue;
                if (mark[b] != a) { mark[b] = a; acc[b] = 0.0; touched[nt++] = b; }
                acc[b] += w[e];
            }
        }
        /* sort touched coarse columns (insertion sort: rows are short) */
        for (int64_t i = 1; i < nt; ++i) {
            int64_t t = touched[i], j = i - 1;
            while (j >= 0 && touched[j] > t) { touched[j + 1] = touched[j]; --j; }
            touched[j + 1] = t;
        }
        for (int64_t i = 0; i < nt; ++i) { ccol[nnz] = (int32_t)touched[i]; cw[nnz] = acc[touched[i]]; ++nnz; }
        crowptr[a + 1] = nnz;
    }
    free(start); free(members); free(fill); free(acc); free(mark); free(touched);
    return nnz;
}
