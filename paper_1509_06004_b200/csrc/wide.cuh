// wide.cuh -- the int64 state variant of the solver, for admitted graphs
// whose excess can leave int32 (grid.py:102-130 admits every capacity in
// [0, CAP_MAX = 2^30] and a total below 2^62, solvers.py:88-141 runs on
// int64 numpy arrays).  The tile engine keeps excess and residuals in int32
// (or u8) words, which bounds a pixel's excess by its positive terminal plus
// its incoming arc pairs < 2^31; graphs past that bound (CAP_MAX interior
// arc pairs, CAP_MAX seeds next to CAP_MAX arcs) run here instead of being
// refused (engine.cu selects it at the boundary).
//
// State, row-major per grid and concatenated over the grids of a batch:
//   e  int64  reduced terminal state (> 0 excess, < 0 residual sink arc)
//   r  int64  four residual planes (L, R, U, D), plane d at r + d * P
//   h  int32  distance label (HINF: cannot reach the sink)
//   lab u8    source-side closure
// Same algorithm and certificates as the tile engine:
// phase-1 push-relabel to a maximum preflow with exact global relabels
// (_exact_heights, solvers.py:54-85) every `pulses` lock-step pulses
// (push then relabel, solvers.py:107-136, with the admissibility h(p) > h(q)),
// then the residual closure of the excess pixels = minimal source side
// (solvers.py:144-158) and {h < HINF} of the final exact relabel = sink side
// (solvers.py:161-174).  Results (flow, minimal source side) are unique, so
// they are bit-identical to the reference's.
#pragma once
#include "engine.cuh"

namespace pmf {

constexpr int WT = 32;                 // tile edge (one pixel per thread, 1024 threads)
constexpr int WRW = WT + 2;            // ring-padded row stride of the BFS frame

struct WGrid {
    int64_t base;       // first pixel of the grid in the state planes
    int32_t W, H;
    int64_t out_off;    // label bytes: out[out_off + y * pitch + xoff + x]
    int32_t pitch, xoff;
    int32_t cs_off;     // per-column swapped flags at colswap + cs_off, -1: none
    int32_t flow_idx;   // slot of the grid's flow in flows[]
    int32_t prob, lam;  // seed batches: problem / lambda index (builder)
};

struct WTile {
    int32_t g, x0, y0, pad;
};

struct WCtx {
    int64_t *e;
    int64_t *r;
    int32_t *h;
    uint8_t *lab;
    int64_t P;                 // pixels in the state planes
    const WGrid *grids;
    const WTile *tiles;
    int32_t ntiles;
    int64_t *snk_sum;          // per grid: sum of the sink capacities
    int64_t *drain;            // per grid: unused sink residual
    int32_t *err;
    const uint8_t *colswap;
    uint8_t *out;
    int64_t *flows;
    unsigned long long *count; // active-pixel counter
};

__device__ __forceinline__ void atomic_add64(int64_t *p, int64_t v) {
    atomicAdd(reinterpret_cast<unsigned long long *>(p), static_cast<unsigned long long>(v));
}

// pixel of this thread in tile t: grid, coordinates, state index (-1: outside the grid)
struct WPix {
    int32_t g, x, y, W, H;
    int64_t p;
};
__device__ __forceinline__ WPix wpix(const WCtx &c, int32_t t) {
    const WTile tl = c.tiles[t];
    const WGrid &gd = c.grids[tl.g];
    WPix o;
    o.g = tl.g;
    o.x = tl.x0 + int32_t(threadIdx.x & (WT - 1));
    o.y = tl.y0 + int32_t(threadIdx.x / WT);
    o.W = gd.W;
    o.H = gd.H;
    o.p = (o.x < gd.W && o.y < gd.H) ? gd.base + int64_t(o.y) * gd.W + o.x : -1;
    return o;
}

__device__ __forceinline__ int64_t wblock_sum(int64_t v) {
    __shared__ int64_t red[32];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t s = 0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    __syncthreads();
    return s;   // valid in thread 0
}

// ---- loaders ---------------------------------------------------------------

// Composite planes (int32, already range-checked to [0, CAP_MAX]) of grid g
// at plane_off[g]: src | snk | nbr(4n), concatenated as staged by
// solve_composites_t.
__global__ void __launch_bounds__(1024) k_wide_load_comp(WCtx c, const int32_t *src, const int32_t *snk,
                                                         const int32_t *nbr, const int64_t *plane_off) {
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        int64_t k = 0;
        if (px.p >= 0) {
            const int64_t off = plane_off[px.g], n = int64_t(px.W) * px.H, q = int64_t(px.y) * px.W + px.x;
            const int64_t s = src[off + q];
            k = snk[off + q];
            c.e[px.p] = s - k;
#pragma unroll
            for (int d = 0; d < 4; d++) c.r[d * c.P + px.p] = nbr[4 * off + d * n + q];
        }
        k = wblock_sum(k);
        if (threadIdx.x == 0 && k) atomic_add64(&c.snk_sum[px.g], k);
    }
}

// lambda-graph (prob, lam) of a staged seed batch, instantiated on the
// device (parametric.py:147-165) in its original orientation: the batch
// reports the minimal source side of the original graph, which is what
// split() returns for a swapped segment too (supergraph.py:177-187).
__global__ void __launch_bounds__(1024) k_wide_build_seed(WCtx c, const int32_t *base, const int32_t *slope,
                                                          const int32_t *sink, const int32_t *pw,
                                                          const uint8_t *mask, const int64_t *plane_off,
                                                          const int64_t *pw_off, const int64_t *lambdas) {
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        int64_t k = 0;
        if (px.p >= 0) {
            const WGrid &gd = c.grids[px.g];
            const int64_t n = int64_t(px.W) * px.H, q = int64_t(px.y) * px.W + px.x;
            const int64_t po = plane_off[gd.prob];
            const uint8_t m = mask[int64_t(gd.prob) * n + q];
            const int64_t s = m == 1 ? CAP_MAX : int64_t(base[po + q]) + lambdas[gd.lam] * int64_t(slope[po + q]);
            k = m == 2 ? CAP_MAX : int64_t(sink[po + q]);
            c.e[px.p] = s - k;
            const int32_t *pp = pw + pw_off[gd.prob];
#pragma unroll
            for (int d = 0; d < 4; d++) c.r[d * c.P + px.p] = pp[d * n + q];
        }
        k = wblock_sum(k);
        if (threadIdx.x == 0 && k) atomic_add64(&c.snk_sum[px.g], k);
    }
}

// ---- global relabel / label closure -----------------------------------------

// h = 1 on sink-residual pixels, HINF elsewhere (sink == 0); lab = excess
// pixels (sink == 1)
__global__ void __launch_bounds__(1024) k_wide_init(WCtx c, int sink) {
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        if (px.p < 0) continue;
        const int64_t e = c.e[px.p];
        if (sink) c.h[px.p] = e < 0 ? 1 : HINF;
        else c.lab[px.p] = e > 0;
    }
}

// One relaxation launch over every tile: tile-local Bellman-Ford to the
// fixpoint in shared memory on a ring-padded frame (ring = neighbour tiles'
// current values), then write-back.  sink: d(p) = min(d(p), d(q) + 1) over
// arcs p -> q with residual (distance to the sink, solvers.py:54-71).
// !sink: reachability from the excess pixels, lab(q) |= lab(p) over arcs
// p -> q with residual (solvers.py:144-158); reaching a sink-residual pixel
// means the preflow was not maximum (err 4, NonMaximalFlowError).  Values
// only decrease (grow, for labels), so tiles of one launch may read each
// other's values at any point.  chg is set when any value changed.
__global__ void __launch_bounds__(1024) k_wide_relax(WCtx c, int sink, int32_t *chg) {
    __shared__ int32_t s_v[WRW * (WT + 2)];
    __shared__ int s_any;
    constexpr int OFF[4] = {-1, 1, -WRW, WRW};
    const int lx = threadIdx.x & (WT - 1), ly = threadIdx.x / WT;
    const int q = (ly + 1) * WRW + lx + 1;
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        // ring: facing pixels of the neighbour tiles (HINF off the grid)
        if (threadIdx.x < 4 * WT) {
            const int s = threadIdx.x / WT, j = threadIdx.x % WT;
            const WTile tl = c.tiles[t];
            const WGrid &gd = c.grids[tl.g];
            int xx = tl.x0 + j, yy = tl.y0 + j, ri;
            switch (s) {
            case DL: xx = tl.x0 - 1; ri = (j + 1) * WRW; break;
            case DR: xx = tl.x0 + WT; ri = (j + 1) * WRW + WT + 1; break;
            case DU: yy = tl.y0 - 1; ri = j + 1; break;
            default: yy = tl.y0 + WT; ri = (WT + 1) * WRW + j + 1; break;
            }
            int32_t v = HINF;
            if (xx >= 0 && yy >= 0 && xx < gd.W && yy < gd.H) {
                const int64_t pn = gd.base + int64_t(yy) * gd.W + xx;
                v = sink ? c.h[pn] : (c.lab[pn] ? 0 : HINF);
            }
            s_v[ri] = v;
        }
        int32_t v0 = HINF;
        int mk = 0;
        if (px.p >= 0) {
            if (sink) {
                v0 = c.h[px.p];
#pragma unroll
                for (int d = 0; d < 4; d++) mk |= (c.r[d * c.P + px.p] > 0) << d;
            } else {
                v0 = c.lab[px.p] ? 0 : HINF;
                // neighbour q_d has a residual arc into this pixel: r(q_d -> p) = plane opp(d) at q_d
                const int64_t nb[4] = {px.p - 1, px.p + 1, px.p - px.W, px.p + px.W};
                const bool in[4] = {px.x > 0, px.x + 1 < px.W, px.y > 0, px.y + 1 < px.H};
#pragma unroll
                for (int d = 0; d < 4; d++)
                    if (in[d]) mk |= (c.r[opp(d) * c.P + nb[d]] > 0) << d;
            }
        }
        s_v[q] = v0;
        if (threadIdx.x == 0) s_any = 0;
        __syncthreads();
        const int cost = sink ? 1 : 0;
        int32_t v = v0;
        for (;;) {
            int32_t m = v;
#pragma unroll
            for (int d = 0; d < 4; d++)
                if ((mk >> d) & 1) m = min(m, s_v[q + OFF[d]] + cost);
            m = min(m, HINF);
            const bool ch = m < v;
            __syncthreads();
            if (ch) {
                v = m;
                s_v[q] = m;
            }
            if (!__syncthreads_or(ch)) break;
        }
        if (px.p >= 0 && v != v0) {
            if (sink) {
                c.h[px.p] = v;
            } else {
                c.lab[px.p] = 1;
                if (c.e[px.p] < 0) atomicExch(c.err, 4);
            }
            s_any = 1;
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_any) atomicExch(chg, 1);
        __syncthreads();
    }
}

// ---- push-relabel pulse -------------------------------------------------------

__global__ void __launch_bounds__(1024) k_wide_count(WCtx c) {
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        const int64_t a = px.p >= 0 && c.e[px.p] > 0 && c.h[px.p] < HINF;
        const int64_t s = wblock_sum(a);
        if (threadIdx.x == 0 && s) atomicAdd(c.count, (unsigned long long)s);
    }
}

// Push phase of a pulse: every active pixel pushes min(e, r) down every arc
// with h(p) > h(q) (heights are fixed during the launch, so an arc pair is
// never pushed both ways and every residual word has one writer; inflow
// lands with int64 atomics).
__global__ void __launch_bounds__(1024) k_wide_push(WCtx c) {
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        if (px.p < 0) continue;
        const int64_t e0 = c.e[px.p];
        const int32_t h = c.h[px.p];
        if (e0 <= 0 || h >= HINF) continue;
        const int64_t nb[4] = {px.p - 1, px.p + 1, px.p - px.W, px.p + px.W};
        int64_t rem = e0;
#pragma unroll
        for (int d = 0; d < 4; d++) {
            if (rem <= 0) break;
            const int64_t rd = c.r[d * c.P + px.p];
            if (rd <= 0 || c.h[nb[d]] >= h) continue;   // rd > 0 only for arcs inside the grid
            const int64_t dl = min(rem, rd);
            rem -= dl;
            c.r[d * c.P + px.p] = rd - dl;
            c.r[opp(d) * c.P + nb[d]] += dl;
            atomic_add64(&c.e[nb[d]], dl);
        }
        if (rem != e0) atomic_add64(&c.e[px.p], rem - e0);
    }
}

// Relabel phase: an active pixel without an admissible arc rises to one
// above its lowest residual neighbour (HINF when it has none that can reach
// the sink: frozen).
__global__ void __launch_bounds__(1024) k_wide_relabel(WCtx c) {
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        if (px.p < 0) continue;
        const int32_t h = c.h[px.p];
        if (c.e[px.p] <= 0 || h >= HINF) continue;
        const int64_t nb[4] = {px.p - 1, px.p + 1, px.p - px.W, px.p + px.W};
        int32_t m = HINF;
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (c.r[d * c.P + px.p] > 0) m = min(m, c.h[nb[d]]);
        if (m >= h) c.h[px.p] = m >= HINF - 1 ? HINF : m + 1;
    }
}

// ---- outputs ----------------------------------------------------------------

// Label bytes (swapped composite columns: ~sink side, supergraph.py:201-206)
// and the per-grid unused sink residual.
__global__ void __launch_bounds__(1024) k_wide_emit(WCtx c) {
    for (int32_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const WPix px = wpix(c, t);
        int64_t dr = 0;
        if (px.p >= 0) {
            const WGrid &gd = c.grids[px.g];
            const bool cs = gd.cs_off >= 0 && c.colswap[gd.cs_off + gd.xoff + px.x];
            c.out[gd.out_off + int64_t(px.y) * gd.pitch + gd.xoff + px.x] =
                cs ? uint8_t(c.h[px.p] >= HINF) : c.lab[px.p];
            const int64_t e = c.e[px.p];
            dr = e < 0 ? -e : 0;
        }
        dr = wblock_sum(dr);
        if (threadIdx.x == 0 && dr) atomic_add64(&c.drain[px.g], dr);
    }
}

__global__ void k_wide_finalize(WCtx c, int32_t ngrids) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngrids; g += gridDim.x * blockDim.x)
        c.flows[c.grids[g].flow_idx] = c.snk_sum[g] - c.drain[g];
}

}  // namespace pmf
