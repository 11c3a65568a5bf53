/*
 * pmflow_oracle.c -- CPU restatement of the reference solver path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load the library built from it.
 *
 * It restates, step for step and in exact int64 arithmetic, the numpy
 * reference in /root/reference/pkg/src/pmflow:
 *
 *   orc_push_relabel      solvers.py:88-141   push_relabel_residual
 *     exact_heights       solvers.py:54-85    _exact_heights (BFS from t,
 *                                              then source-return band)
 *   orc_source_side       solvers.py:144-158  source_side
 *   orc_sink_side         solvers.py:161-174  sink_side
 *   orc_maxflow           solvers.py:177-191  extract_canonical_cut +
 *                                              maxflow_pushrelabel
 *   orc_solve_composite   supergraph.py:190-207 solve_composite
 *
 * Grids are row-major (p = y*W + x, grid.py:3); nbr is (4, n) with rows
 * LEFT, RIGHT, UP, DOWN (grid.py:23-25).  The pulse order is the
 * reference's: sink push, then LEFT, RIGHT, UP, DOWN pushes (each
 * direction vectorised over all pixels with the excess as it stood before
 * that direction), then source return, then a Jacobi relabel; the exact
 * relabel is re-applied as max(h, exact) every 64 pulses.  Because it is
 * the same schedule, pulse counts match the reference exactly (pinned in
 * tests/test_oracle.py).
 *
 * Parity: pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) -- see DESIGN.md section "Oracle".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_NOCONV (-1)      /* SolverError: pulse limit (solvers.py:137-139) */
#define ORC_ERR_PREFLOW (-2)     /* NonMaximalFlowError: excess left (solvers.py:183-184) */
#define ORC_ERR_SRCSIDE (-3)     /* NonMaximalFlowError: source side hits sink arc (:156-157) */
#define ORC_ERR_SNKSIDE (-4)     /* NonMaximalFlowError: sink side hits source arc (:172-173) */
#define ORC_ERR_NOMEM (-5)

#define GR_INTERVAL 64           /* GLOBAL_RELABEL_INTERVAL, solvers.py:28 */
static const int64_t BIG = (int64_t)1 << 40;   /* _BIG, solvers.py:30 */

enum { L = 0, R = 1, U = 2, D = 3 };
static const int OPP[4] = {R, L, D, U};

/* flat index of p's d-neighbour, or -1 off-grid (grid.py:133-156 semantics) */
static inline int64_t nb(int64_t p, int d, int W, int H) {
    int64_t x = p % W, y = p / W;
    switch (d) {
    case L: return x > 0 ? p - 1 : -1;
    case R: return x + 1 < W ? p + 1 : -1;
    case U: return y > 0 ? p - W : -1;
    default: return y + 1 < H ? p + W : -1;
    }
}

/* BFS over residual arcs toward a seed set: v joins when nbr[d][v] > 0 and
 * its d-neighbour is already reached.  Levels of the queue BFS equal the
 * frontier levels of solvers.py:61-71 (BFS distances are unique). */
static void bfs_to_set(int W, int H, const int64_t *nbr, unsigned char *seen,
                       int64_t *h, int64_t *queue, int64_t qn, int64_t base) {
    int64_t n = (int64_t)W * H, head = 0;
    /* level of queued items is stored in h as base + level */
    while (head < qn) {
        int64_t u = queue[head++];
        int64_t lu = h[u];
        for (int d = 0; d < 4; d++) {
            /* v is u's OPP[d]-neighbour; arc v -> u is direction d from v */
            int64_t v = nb(u, OPP[d], W, H);
            if (v < 0 || seen[v]) continue;
            if (nbr[(int64_t)d * n + v] > 0) {
                seen[v] = 1;
                h[v] = lu + 1;
                queue[qn++] = v;
            }
        }
    }
    (void)base;
}

/* _exact_heights, solvers.py:54-85 */
static void exact_heights(int W, int H, const int64_t *to_sink, const int64_t *to_source,
                          const int64_t *nbr, int64_t nv, int64_t *h,
                          unsigned char *seen, int64_t *queue) {
    int64_t n = (int64_t)W * H, qn = 0;
    for (int64_t p = 0; p < n; p++) {
        h[p] = nv + n + 1;
        seen[p] = 0;
        if (to_sink[p] > 0) { seen[p] = 1; h[p] = 1; queue[qn++] = p; }
    }
    bfs_to_set(W, H, nbr, seen, h, queue, qn, 0);
    qn = 0;
    for (int64_t p = 0; p < n; p++)
        if (!seen[p] && to_source[p] > 0) { seen[p] = 1; h[p] = nv + 1; queue[qn++] = p; }
    bfs_to_set(W, H, nbr, seen, h, queue, qn, 0);
}

/*
 * push_relabel_residual, solvers.py:88-141.  Inputs src, snk (n) and nbr
 * (4n) are the admitted capacities.  Outputs (caller-allocated, n or 4n
 * int64): e, from_source, to_source, to_sink, nbr_res; *flow, *pulses,
 * *global_relabels.
 */
int orc_push_relabel(int W, int H, const int64_t *src, const int64_t *snk,
                     const int64_t *nbr, int64_t *e, int64_t *from_source,
                     int64_t *to_source, int64_t *to_sink, int64_t *nbr_res,
                     int64_t *flow, int64_t *pulses_out, int64_t *relabels_out) {
    int64_t n = (int64_t)W * H;
    int64_t nv = n + 2;                                   /* N = H*W + 2, :92 */
    int64_t limit = 40 * nv > 10000 ? 40 * nv : 10000;    /* :101 */
    int64_t *h = malloc(sizeof(int64_t) * n);
    int64_t *tmp = malloc(sizeof(int64_t) * n);
    int64_t *delta = malloc(sizeof(int64_t) * n);
    int64_t *queue = malloc(sizeof(int64_t) * n);
    unsigned char *seen = malloc(n ? n : 1);
    if (!h || !tmp || !delta || !queue || !seen) {
        free(h); free(tmp); free(delta); free(queue); free(seen);
        return ORC_ERR_NOMEM;
    }
    for (int64_t p = 0; p < n; p++) {                     /* :93-98 */
        e[p] = src[p];
        from_source[p] = 0;
        to_source[p] = src[p];
        to_sink[p] = snk[p];
    }
    memcpy(nbr_res, nbr, sizeof(int64_t) * 4 * n);
    exact_heights(W, H, to_sink, to_source, nbr_res, nv, h, seen, queue);  /* :99 */
    int64_t pulses = 0, relabels = 1;
    int rc = ORC_OK;
    for (;;) {
        int any = 0;                                      /* :103 */
        for (int64_t p = 0; p < n && !any; p++) any = e[p] > 0;
        if (!any) break;
        if (pulses && pulses % GR_INTERVAL == 0) {        /* :105-106 */
            exact_heights(W, H, to_sink, to_source, nbr_res, nv, tmp, seen, queue);
            for (int64_t p = 0; p < n; p++) if (tmp[p] > h[p]) h[p] = tmp[p];
            relabels++;
        }
        for (int64_t p = 0; p < n; p++) {                 /* sink push :107-111 */
            if (e[p] > 0 && h[p] == 1 && to_sink[p] > 0) {
                int64_t dl = e[p] < to_sink[p] ? e[p] : to_sink[p];
                e[p] -= dl;
                to_sink[p] -= dl;
            }
        }
        for (int d = 0; d < 4; d++) {                     /* neighbour pushes :112-120 */
            int64_t *cap = nbr_res + (int64_t)d * n;
            int64_t *rev = nbr_res + (int64_t)OPP[d] * n;
            for (int64_t p = 0; p < n; p++) {
                delta[p] = 0;
                if (e[p] <= 0 || cap[p] <= 0) continue;
                int64_t q = nb(p, d, W, H);
                if (q < 0 || h[p] != h[q] + 1) continue;
                delta[p] = e[p] < cap[p] ? e[p] : cap[p];
            }
            for (int64_t p = 0; p < n; p++) {
                int64_t dl = delta[p];
                if (!dl) continue;
                int64_t q = nb(p, d, W, H);
                cap[p] -= dl;
                rev[q] += dl;
                e[p] -= dl;
                e[q] += dl;
            }
        }
        for (int64_t p = 0; p < n; p++) {                 /* source return :121-126 */
            if (e[p] > 0 && h[p] == nv + 1 && to_source[p] > 0) {
                int64_t dl = e[p] < to_source[p] ? e[p] : to_source[p];
                e[p] -= dl;
                to_source[p] -= dl;
                from_source[p] += dl;
            }
        }
        for (int64_t p = 0; p < n; p++) {                 /* Jacobi relabel :127-136 */
            tmp[p] = h[p];
            if (e[p] <= 0) continue;
            int64_t best = to_sink[p] > 0 ? 1 : BIG;
            for (int d = 0; d < 4; d++) {
                if (nbr_res[(int64_t)d * n + p] <= 0) continue;
                int64_t q = nb(p, d, W, H);
                int64_t cand = (q < 0 ? BIG : h[q]) + 1;
                if (cand < best) best = cand;
            }
            if (to_source[p] > 0 && nv + 1 < best) best = nv + 1;
            if (best > h[p]) tmp[p] = best;
        }
        memcpy(h, tmp, sizeof(int64_t) * n);
        pulses++;
        if (pulses > limit) { rc = ORC_ERR_NOCONV; break; }  /* :137-139 */
    }
    int64_t f = 0;                                        /* :140 */
    for (int64_t p = 0; p < n; p++) f += snk[p] - to_sink[p];
    *flow = f;
    if (pulses_out) *pulses_out = pulses;
    if (relabels_out) *relabels_out = relabels;
    free(h); free(tmp); free(delta); free(queue); free(seen);
    return rc;
}

/* source_side, solvers.py:144-158: forward BFS from {from_source > 0}. */
int orc_source_side(int W, int H, const int64_t *from_source, const int64_t *to_sink,
                    const int64_t *nbr_res, unsigned char *reach) {
    int64_t n = (int64_t)W * H, qn = 0, head = 0;
    int64_t *queue = malloc(sizeof(int64_t) * (n ? n : 1));
    if (!queue) return ORC_ERR_NOMEM;
    for (int64_t p = 0; p < n; p++) {
        reach[p] = from_source[p] > 0;
        if (reach[p]) queue[qn++] = p;
    }
    while (head < qn) {
        int64_t u = queue[head++];
        for (int d = 0; d < 4; d++) {
            if (nbr_res[(int64_t)d * n + u] <= 0) continue;
            int64_t v = nb(u, d, W, H);
            if (v >= 0 && !reach[v]) { reach[v] = 1; queue[qn++] = v; }
        }
    }
    free(queue);
    for (int64_t p = 0; p < n; p++)
        if (reach[p] && to_sink[p] > 0) return ORC_ERR_SRCSIDE;
    return ORC_OK;
}

/* sink_side, solvers.py:161-174: backward BFS from {to_sink > 0}. */
int orc_sink_side(int W, int H, const int64_t *from_source, const int64_t *to_sink,
                  const int64_t *nbr_res, unsigned char *reach) {
    int64_t n = (int64_t)W * H, qn = 0, head = 0;
    int64_t *queue = malloc(sizeof(int64_t) * (n ? n : 1));
    if (!queue) return ORC_ERR_NOMEM;
    for (int64_t p = 0; p < n; p++) {
        reach[p] = to_sink[p] > 0;
        if (reach[p]) queue[qn++] = p;
    }
    while (head < qn) {
        int64_t u = queue[head++];
        for (int d = 0; d < 4; d++) {
            int64_t v = nb(u, OPP[d], W, H);      /* arc v -> u has direction d */
            if (v < 0 || reach[v]) continue;
            if (nbr_res[(int64_t)d * n + v] > 0) { reach[v] = 1; queue[qn++] = v; }
        }
    }
    free(queue);
    for (int64_t p = 0; p < n; p++)
        if (reach[p] && from_source[p] > 0) return ORC_ERR_SNKSIDE;
    return ORC_OK;
}

/*
 * solve_composite, supergraph.py:190-207 (nseg == 0 <=> layout None, which
 * is also maxflow_pushrelabel, solvers.py:188-191).  Swapped spans carry
 * ~sink_side over every row of their columns (:201-206).
 */
int orc_solve_composite(int W, int H, const int64_t *src, const int64_t *snk,
                        const int64_t *nbr, int nseg, const int32_t *seg_off,
                        const int32_t *seg_w, const unsigned char *seg_swapped,
                        int64_t *flow, unsigned char *labels, int64_t *pulses) {
    int64_t n = (int64_t)W * H;
    int64_t *buf = malloc(sizeof(int64_t) * 8 * (n ? n : 1));
    unsigned char *keep = NULL;
    if (!buf) return ORC_ERR_NOMEM;
    int64_t *e = buf, *fs = buf + n, *ts = buf + 2 * n, *tk = buf + 3 * n, *nr = buf + 4 * n;
    int rc = orc_push_relabel(W, H, src, snk, nbr, e, fs, ts, tk, nr, flow, pulses, NULL);
    if (rc) goto out;
    for (int64_t p = 0; p < n; p++)                          /* solvers.py:183-184 */
        if (e[p]) { rc = ORC_ERR_PREFLOW; goto out; }
    rc = orc_source_side(W, H, fs, tk, nr, labels);
    if (rc) goto out;
    int any_swapped = 0;
    for (int s = 0; s < nseg; s++) any_swapped |= seg_swapped[s] != 0;
    if (any_swapped) {
        keep = malloc(n ? n : 1);
        if (!keep) { rc = ORC_ERR_NOMEM; goto out; }
        rc = orc_sink_side(W, H, fs, tk, nr, keep);
        if (rc) goto out;
        for (int s = 0; s < nseg; s++) {
            if (!seg_swapped[s]) continue;
            for (int y = 0; y < H; y++)
                for (int x = seg_off[s]; x < seg_off[s] + seg_w[s]; x++)
                    labels[(int64_t)y * W + x] = !keep[(int64_t)y * W + x];
        }
    }
out:
    free(buf);
    free(keep);
    return rc;
}

int orc_maxflow(int W, int H, const int64_t *src, const int64_t *snk, const int64_t *nbr,
                int64_t *flow, unsigned char *labels, int64_t *pulses) {
    return orc_solve_composite(W, H, src, snk, nbr, 0, NULL, NULL, NULL, flow, labels, pulses);
}
