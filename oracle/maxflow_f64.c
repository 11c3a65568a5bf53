/*
 * maxflow_f64.c -- double-precision max-flow / minimal min-cut on a grid
 * graph (Dinic).  TEST INFRASTRUCTURE ONLY: the fp64 checker of the float-
 * capacity mode (paper_1509_06004_b200/floatcap.py).  The reference has no
 * float solver (SURVEY.md section 8c "Float path": floats only enter through
 * quantize_weights, harness/synth.py:139-151), so the float mode is checked
 * against an independent fp64 max-flow on the unquantised capacities: flow
 * within 1e-5 relative error, label differences reported as tie pixels.
 *
 * Graph: pixels 0..n-1 row-major (grid.py:3), S = n, T = n + 1; arcs S->p
 * (src), p->T (snk), p->q (nbr[d][p], rows LEFT, RIGHT, UP, DOWN) paired
 * with their reverse arc q->p (nbr[opp(d)][q]).  Residuals below eps =
 * 1e-12 x the largest capacity count as saturated.  Labels: 1 = reachable
 * from S in the final residual graph (the minimal source side, the same
 * convention as solvers.py:144-158).  Pinned on integer-valued graphs
 * against the reference's own vectors (tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t nn, ne;
    int64_t *start, *to, *frm, *rev;
    double *cap;
} Net;

static int64_t add_arc(Net *g, int64_t *fill, int64_t u, int64_t v, double c, double rc) {
    const int64_t a = fill[u]++, b = fill[v]++;
    g->to[a] = v;
    g->frm[a] = u;
    g->cap[a] = c;
    g->rev[a] = b;
    g->to[b] = u;
    g->frm[b] = v;
    g->cap[b] = rc;
    g->rev[b] = a;
    return a;
}

int orc_maxflow_f64(int W, int H, const double *src, const double *snk, const double *nbr, double *flow_out,
                    uint8_t *labels) {
    const int64_t n = (int64_t)W * H, S = n, T = n + 1, nn = n + 2;
    Net g;
    g.nn = nn;
    int64_t *deg = calloc((size_t)nn + 1, sizeof(int64_t));
    if (!deg) return -5;
    /* arc pairs: S-p, p-T, p-right, p-down */
    for (int64_t p = 0; p < n; p++) {
        const int64_t x = p % W, y = p / W;
        deg[S]++, deg[p]++;
        deg[p]++, deg[T]++;
        if (x + 1 < W) deg[p]++, deg[p + 1]++;
        if (y + 1 < H) deg[p]++, deg[p + W]++;
    }
    g.start = malloc(sizeof(int64_t) * ((size_t)nn + 1));
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)nn);
    g.start[0] = 0;
    for (int64_t u = 0; u < nn; u++) g.start[u + 1] = g.start[u] + deg[u];
    g.ne = g.start[nn];
    g.to = malloc(sizeof(int64_t) * (size_t)g.ne);
    g.frm = malloc(sizeof(int64_t) * (size_t)g.ne);
    g.rev = malloc(sizeof(int64_t) * (size_t)g.ne);
    g.cap = malloc(sizeof(double) * (size_t)g.ne);
    int64_t *level = malloc(sizeof(int64_t) * (size_t)nn), *it = malloc(sizeof(int64_t) * (size_t)nn);
    int64_t *queue = malloc(sizeof(int64_t) * (size_t)nn), *stack = malloc(sizeof(int64_t) * (size_t)nn);
    if (!g.start || !fill || !g.to || !g.frm || !g.rev || !g.cap || !level || !it || !queue || !stack) return -5;
    memcpy(fill, g.start, sizeof(int64_t) * (size_t)nn);
    double cmax = 0;
    for (int64_t p = 0; p < n; p++) {
        const int64_t x = p % W, y = p / W;
        add_arc(&g, fill, S, p, src[p], 0.0);
        add_arc(&g, fill, p, T, snk[p], 0.0);
        if (x + 1 < W) add_arc(&g, fill, p, p + 1, nbr[1 * n + p], nbr[0 * n + p + 1]);
        if (y + 1 < H) add_arc(&g, fill, p, p + W, nbr[3 * n + p], nbr[2 * n + p + W]);
        /* eps scale: the largest FINITE capacity (+inf marks hard constraints) */
        if (isfinite(src[p])) cmax = fmax(cmax, src[p]);
        if (isfinite(snk[p])) cmax = fmax(cmax, snk[p]);
        for (int d = 0; d < 4; d++)
            if (isfinite(nbr[d * n + p])) cmax = fmax(cmax, nbr[d * n + p]);
    }
    const double eps = 1e-12 * (cmax > 0 ? cmax : 1.0);
    double flow = 0;
    for (;;) {
        /* BFS levels over residual arcs */
        for (int64_t u = 0; u < nn; u++) level[u] = -1;
        int64_t qh = 0, qt = 0;
        level[S] = 0;
        queue[qt++] = S;
        while (qh < qt) {
            const int64_t u = queue[qh++];
            for (int64_t a = g.start[u]; a < g.start[u + 1]; a++)
                if (g.cap[a] > eps && level[g.to[a]] < 0) {
                    level[g.to[a]] = level[u] + 1;
                    queue[qt++] = g.to[a];
                }
        }
        if (level[T] < 0) break;
        memcpy(it, g.start, sizeof(int64_t) * (size_t)nn);
        /* blocking flow: iterative augmenting-path search in the level graph */
        for (;;) {
            int64_t top = 0, u = S;
            while (u != T) {
                while (it[u] < g.start[u + 1]) {
                    const int64_t a = it[u];
                    if (g.cap[a] > eps && level[g.to[a]] == level[u] + 1) break;
                    it[u]++;
                }
                if (it[u] == g.start[u + 1]) {   /* dead end: retreat */
                    level[u] = -1;
                    if (top == 0) break;
                    u = g.frm[stack[--top]];
                    it[u]++;
                    continue;
                }
                stack[top++] = it[u];
                u = g.to[it[u]];
            }
            if (u != T) break;
            double f = INFINITY;
            for (int64_t k = 0; k < top; k++) f = fmin(f, g.cap[stack[k]]);
            for (int64_t k = 0; k < top; k++) {
                g.cap[stack[k]] -= f;
                g.cap[g.rev[stack[k]]] += f;
            }
            flow += f;
        }
    }
    /* minimal source side: reachable from S over residual arcs */
    memset(labels, 0, (size_t)n);
    for (int64_t u = 0; u < nn; u++) level[u] = -1;
    int64_t qh = 0, qt = 0;
    level[S] = 0;
    queue[qt++] = S;
    while (qh < qt) {
        const int64_t u = queue[qh++];
        if (u < n) labels[u] = 1;
        for (int64_t a = g.start[u]; a < g.start[u + 1]; a++)
            if (g.cap[a] > eps && level[g.to[a]] < 0) {
                level[g.to[a]] = 0;
                queue[qt++] = g.to[a];
            }
    }
    *flow_out = flow;
    free(deg), free(fill), free(g.start), free(g.to), free(g.frm), free(g.rev), free(g.cap);
    free(level), free(it), free(queue), free(stack);
    return 0;
}
