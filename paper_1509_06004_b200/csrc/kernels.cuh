// kernels.cuh -- sm_100a kernels of the supergraph min-cut path.
//
// Algorithm: phase-1 push-relabel on the reduced
// network (terminal pair src/snk folded into one signed value w, the NPPI
// convention of SPEC.md:121 / PAPER.md:536; every cut is lowered by the same
// constant so optima are unchanged), discharged tile by tile in shared
// memory, with an exact global relabel (BFS from the sink) between rounds.
// Pixels that cannot reach the sink are frozen at HINF, so no "return
// excess to the source" phase is needed: the minimal source side is the
// residual closure of the excess pixels of the maximum preflow, which is
// what the reference's source_side() computes after its phase 2
// (solvers.py:144-158; proof in DESIGN.md), and the sink side
// (solvers.py:161-174) is {h < HINF} of the final exact relabel.
#pragma once
#include "engine.cuh"

namespace pmf {

// ---------------------------------------------------------------------------
// Builders (supergraph.py:95-154, parametric.py:133-166 fused on device)
// ---------------------------------------------------------------------------

struct SeedArgs {
    const int32_t *base, *slope, *sink, *pw;   // row-major int32 planes
    const uint8_t *mask;                        // 1 = fg seed, 2 = bg seed; problem p at p*n
    const int64_t *plane_off;                   // per problem offset into base/slope/sink
    const int64_t *pw_off;                      // per problem offset into pw ((4, n))
    const int64_t *lambdas;
    int32_t nprob, nlam, W, H, mid, swap_mode;
    int32_t *swap_cnt;                          // [2*nprob] negative / positive counts
    int32_t *swapped;                           // [nprob]
};

// Terminal balance at the mid-schedule lambda (supergraph.py:77-92, 210-212).
__global__ void k_swap_count(SeedArgs a) {
    int64_t n = int64_t(a.W) * a.H;
    int64_t lam = a.lambdas[a.mid];
    int neg = 0, pos = 0;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n * a.nprob;
         idx += int64_t(gridDim.x) * blockDim.x) {
        int32_t p = int32_t(idx / n);
        int64_t r = idx - int64_t(p) * n;
        int64_t q = a.plane_off[p] + r;
        uint8_t m = a.mask[idx];
        int64_t src = m == 1 ? CAP_MAX : int64_t(a.base[q]) + lam * int64_t(a.slope[q]);
        int64_t snk = m == 2 ? CAP_MAX : int64_t(a.sink[q]);
        int64_t d = src - snk;
        neg = d < 0;
        pos = d > 0;
        // warp-aggregated atomics: at most one per warp and problem
        unsigned mm = __match_any_sync(__activemask(), p);
        int nn = __popc(__ballot_sync(mm, neg)), pp = __popc(__ballot_sync(mm, pos));
        if ((threadIdx.x & 31) == __ffs(mm) - 1) {
            if (nn) atomicAdd(&a.swap_cnt[2 * p], nn);
            if (pp) atomicAdd(&a.swap_cnt[2 * p + 1], pp);
        }
    }
}

__global__ void k_swap_decide(SeedArgs a) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.nprob) return;
    if (a.swap_mode == 1) a.swapped[p] = 1;
    else if (a.swap_mode == 2) a.swapped[p] = 0;
    else a.swapped[p] = a.swap_cnt[2 * p] > a.swap_cnt[2 * p + 1];
}

__device__ __forceinline__ int64_t block_sum64(int64_t v, int64_t *red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; i++) s += red[i];
    __syncthreads();
    return s;
}

// One CTA per tile: instantiate (problem, lambda), swap if flagged, write
// the reduced state w = src - snk and the residual arcs.
template <class E>
__global__ void __launch_bounds__(NT) k_build_seed(Ctx c, SeedArgs a) {
    __shared__ int64_t red[NT / 32];
    for (int64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        TileGeo g = tile_geo(c, int32_t(t));
        const GridDesc &gd = c.grids[g.g];
        const int64_t lam = a.lambdas[gd.lam];
        const int sw = c.swapflag[gd.prob];
        const int64_t po = a.plane_off[gd.prob];
        const int32_t *pw = a.pw + a.pw_off[gd.prob];
        const int64_t n = int64_t(a.W) * a.H;
        int64_t snk_acc = 0;
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            int x = g.x0 + (i & (TW - 1)), y = g.y0 + i / TW;
            int64_t p = t * TPIX + i;
            int32_t wv = 0;
            int rl = 0, rr = 0, ru = 0, rd = 0;
            if (x < g.W && y < g.H) {
                int64_t q = int64_t(y) * a.W + x;
                uint8_t m = a.mask[int64_t(gd.prob) * n + q];
                int64_t src = m == 1 ? CAP_MAX : int64_t(a.base[po + q]) + lam * int64_t(a.slope[po + q]);
                int64_t snk = m == 2 ? CAP_MAX : int64_t(a.sink[po + q]);
                if (sw) {  // apply_swap, supergraph.py:95-109
                    int64_t tmp = src; src = snk; snk = tmp;
                    rl = x > 0 ? pw[1 * n + q - 1] : 0;
                    rr = x + 1 < a.W ? pw[0 * n + q + 1] : 0;
                    ru = y > 0 ? pw[3 * n + q - a.W] : 0;
                    rd = y + 1 < a.H ? pw[2 * n + q + a.W] : 0;
                } else {
                    rl = pw[0 * n + q]; rr = pw[1 * n + q];
                    ru = pw[2 * n + q]; rd = pw[3 * n + q];
                }
                wv = int32_t(src - snk);
                snk_acc += snk;
            }
            c.w[p] = wv;
            E::store(c.r, p, E::pack(rl, rr, ru, rd));
        }
        int64_t s = block_sum64(snk_acc, red);
        if (threadIdx.x == 0) atomicAdd((unsigned long long *)&c.snk_sum[g.g], (unsigned long long)s);
    }
}

struct CompArgs {
    const int32_t *src, *snk, *nbr;   // row-major int32 planes, concatenated
    const int64_t *plane_off;         // per grid offsets (src/snk: n, nbr: 4n at 4*off)
};

// Composite loader: the (already admitted) GridGraph planes of
// pmf_solve_composites into the reduced tile-major state.
template <class E>
__global__ void __launch_bounds__(NT) k_load_comp(Ctx c, CompArgs a) {
    __shared__ int64_t red[NT / 32];
    for (int64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        TileGeo g = tile_geo(c, int32_t(t));
        const int64_t off = a.plane_off[g.g];
        const int64_t n = int64_t(g.W) * g.H;
        int64_t snk_acc = 0;
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            int x = g.x0 + (i & (TW - 1)), y = g.y0 + i / TW;
            int64_t p = t * TPIX + i;
            int32_t wv = 0;
            int e[4] = {0, 0, 0, 0};
            if (x < g.W && y < g.H) {
                int64_t q = int64_t(y) * g.W + x;
                int32_t s = a.src[off + q], k = a.snk[off + q];
                wv = s - k;
                snk_acc += k;
                for (int d = 0; d < 4; d++) e[d] = a.nbr[4 * off + d * n + q];
            }
            c.w[p] = wv;
            E::store(c.r, p, E::pack(e[0], e[1], e[2], e[3]));
        }
        int64_t s = block_sum64(snk_acc, red);
        if (threadIdx.x == 0) atomicAdd((unsigned long long *)&c.snk_sum[g.g], (unsigned long long)s);
    }
}

// ---------------------------------------------------------------------------
// Global relabel: exact distance to the sink over residual arcs
// (_exact_heights' first BFS, solvers.py:54-71), tile-local relaxation to a
// fixpoint, tiles re-listed while their halo keeps changing.
// ---------------------------------------------------------------------------

// h = 1 on pixels with sink residual (w < 0), HINF elsewhere; lists every
// tile holding such a pixel.  Tiles of finished grids are left untouched.
__global__ void __launch_bounds__(NT) k_gr_init(Ctx c) {
    for (int64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        if (!c.live[c.tile_grid[t]]) continue;
        int any = 0;
        for (int j = 0; j < PPT; j++) {
            int64_t p = t * TPIX + threadIdx.x + j * NT;
            int32_t wv = c.w[p];
            c.h[p] = wv < 0 ? 1 : HINF;
            any |= wv < 0;
        }
        if (__syncthreads_or(any) && threadIdx.x == 0) enqueue(c, 0, int32_t(t));
    }
}

template <class E>
__global__ void __launch_bounds__(NT) k_bfs_sink(Ctx c, int k) {
    __shared__ int32_t sd[TPIX];
    __shared__ uint8_t sm[TPIX];
    __shared__ int32_t hd[4][TW];
    __shared__ int s_side[4];
    const int32_t n = c.cnt[k % 3];
    const int32_t *lst = list_of(c, k);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c.cnt[(k + 2) % 3] = 0;
        atomicAdd(&c.stat[ST_BFS], (unsigned long long)n);
    }
    for (int li = blockIdx.x; li < n; li += gridDim.x) {
        const int32_t t = lst[li];
        TileGeo g = tile_geo(c, t);
        const int64_t base = int64_t(t) * TPIX;
        int32_t h0[PPT];
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            h0[j] = c.h[base + i];
            sd[i] = h0[j];
            typename E::Word wd = E::load(c.r, base + i);
            sm[i] = uint8_t((E::lane(wd, 0) > 0) | ((E::lane(wd, 1) > 0) << 1) |
                            ((E::lane(wd, 2) > 0) << 2) | ((E::lane(wd, 3) > 0) << 3));
        }
        if (threadIdx.x < 4 * TW) {
            int s = threadIdx.x / TW, j = threadIdx.x % TW;
            hd[s][j] = g.nb[s] >= 0 ? c.h[int64_t(g.nb[s]) * TPIX + halo_index(s, j)] : HINF;
            if (j == 0) s_side[s] = 0;
        }
        if (threadIdx.x == 0) inq_of(c, k)[t] = 0;
        __syncthreads();
        for (;;) {
            int changed = 0;
            for (int j = 0; j < PPT; j++) {
                int i = threadIdx.x + j * NT;
                int32_t v = sd[i];
                int mk = sm[i];
                if (v <= 1 || !mk) continue;
                int lx = i & (TW - 1), ly = i / TW;
                int32_t m = HINF;
                if (mk & 1) m = min(m, lx ? sd[i - 1] : hd[DL][ly]);
                if (mk & 2) m = min(m, lx < TW - 1 ? sd[i + 1] : hd[DR][ly]);
                if (mk & 4) m = min(m, ly ? sd[i - TW] : hd[DU][lx]);
                if (mk & 8) m = min(m, ly < TH - 1 ? sd[i + TW] : hd[DD][lx]);
                if (m + 1 < v) { sd[i] = m + 1; changed = 1; }
            }
            if (!__syncthreads_or(changed)) break;
        }
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            if (sd[i] != h0[j]) {
                c.h[base + i] = sd[i];
                int lx = i & (TW - 1), ly = i / TW;
                if (lx == 0) s_side[DL] = 1;
                if (lx == TW - 1) s_side[DR] = 1;
                if (ly == 0) s_side[DU] = 1;
                if (ly == TH - 1) s_side[DD] = 1;
            }
        }
        __syncthreads();
        if (threadIdx.x < 4 && s_side[threadIdx.x] && g.nb[threadIdx.x] >= 0)
            enqueue(c, k + 1, g.nb[threadIdx.x]);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Push-relabel discharge of one tile in shared memory (solvers.py:107-136
// semantics: push min(e, r) along admissible arcs h(p) == h(q) + 1, in
// direction order L, R, U, D; relabel to 1 + min residual-neighbour height).
// ---------------------------------------------------------------------------

// Lists every tile of a live grid that holds an active pixel (w > 0,
// h < HINF); counts active pixels per grid.
__global__ void __launch_bounds__(NT) k_seed_push(Ctx c) {
    for (int64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        int32_t gid = c.tile_grid[t];
        if (!c.live[gid]) continue;
        int a = 0;
        for (int j = 0; j < PPT; j++) {
            int64_t p = t * TPIX + threadIdx.x + j * NT;
            a += c.w[p] > 0 && c.h[p] < HINF;
        }
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if ((threadIdx.x & 31) == 0 && a) atomicAdd(&c.act[gid], a);
        if (__syncthreads_or(a) && threadIdx.x == 0) enqueue(c, 0, int32_t(t));
    }
}

__global__ void k_update_live(Ctx c, int32_t ngrids) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngrids) return;
    if (c.live[g] && c.act[g] == 0) c.live[g] = 0;
    c.act[g] = 0;
}

template <class E>
__global__ void __launch_bounds__(NT) k_push(Ctx c, int k, int iters) {
    __shared__ int32_t sw[TPIX], sh[TPIX], sin_[TPIX];
    __shared__ int32_t sr[4][TPIX];
    __shared__ int32_t hh[4][TW], hacc[4][TW];
    __shared__ int s_out[4];
    const int32_t n = c.cnt[k % 3];
    const int32_t *lst = list_of(c, k);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c.cnt[(k + 2) % 3] = 0;
        atomicAdd(&c.stat[ST_PUSH], (unsigned long long)n);
    }
    const int tid = threadIdx.x;
    for (int li = blockIdx.x; li < n; li += gridDim.x) {
        const int32_t t = lst[li];
        TileGeo g = tile_geo(c, t);
        const int64_t base = int64_t(t) * TPIX;
        int32_t wv[PPT];
        typename E::Word rv[PPT];
        for (int j = 0; j < PPT; j++) {
            int i = tid + j * NT;
            wv[j] = c.w[base + i];
            sw[i] = wv[j];
            sh[i] = c.h[base + i];
            sin_[i] = 0;
            rv[j] = E::load(c.r, base + i);
            for (int d = 0; d < 4; d++) sr[d][i] = E::lane(rv[j], d);
        }
        if (tid < 4 * TW) {
            int s = tid / TW, j = tid % TW;
            hh[s][j] = g.nb[s] >= 0 ? c.h[int64_t(g.nb[s]) * TPIX + halo_index(s, j)] : HINF;
            hacc[s][j] = 0;
            if (j == 0) s_out[s] = 0;
        }
        if (tid == 0) inq_of(c, k)[t] = 0;
        __syncthreads();
        for (int it = 0; it < iters; it++) {
            // ---- push along admissible arcs (heights fixed in this phase, so
            // no arc is pushed in both directions: plain adds are race-free;
            // incoming excess gathers in sin_ with shared atomics)
            for (int j = 0; j < PPT; j++) {
                int i = tid + j * NT;
                int32_t e = sw[i], hp = sh[i];
                if (e <= 0 || hp >= HINF) continue;
                int lx = i & (TW - 1), ly = i / TW;
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    int32_t rr = sr[d][i];
                    if (rr <= 0) continue;
                    int q;
                    bool in;
                    int32_t hq;
                    int pos;
                    if (d == DL) { in = lx > 0; q = i - 1; pos = ly; }
                    else if (d == DR) { in = lx < TW - 1; q = i + 1; pos = ly; }
                    else if (d == DU) { in = ly > 0; q = i - TW; pos = lx; }
                    else { in = ly < TH - 1; q = i + TW; pos = lx; }
                    hq = in ? sh[q] : hh[d][pos];
                    if (hp != hq + 1) continue;
                    int32_t dl = min(e, rr);
                    e -= dl;
                    sr[d][i] = rr - dl;
                    if (in) {
                        sr[opp(d)][q] += dl;
                        atomicAdd(&sin_[q], dl);
                    } else {
                        hacc[d][pos] += dl;
                    }
                    if (!e) break;
                }
                sw[i] = e;
            }
            __syncthreads();
            // ---- absorb inflow, relabel what is still active
            int act = 0;
            for (int j = 0; j < PPT; j++) {
                int i = tid + j * NT;
                int32_t e = sw[i] + sin_[i];
                sin_[i] = 0;
                sw[i] = e;
                if (e <= 0 || sh[i] >= HINF) continue;
                int lx = i & (TW - 1), ly = i / TW;
                int32_t m = HINF;
                if (sr[DL][i] > 0) m = min(m, lx ? sh[i - 1] : hh[DL][ly]);
                if (sr[DR][i] > 0) m = min(m, lx < TW - 1 ? sh[i + 1] : hh[DR][ly]);
                if (sr[DU][i] > 0) m = min(m, ly ? sh[i - TW] : hh[DU][lx]);
                if (sr[DD][i] > 0) m = min(m, ly < TH - 1 ? sh[i + TW] : hh[DD][lx]);
                int32_t nh = m >= HINF ? HINF : m + 1;
                if (nh > sh[i]) sh[i] = nh;
                act |= sh[i] < HINF;
            }
            if (!__syncthreads_or(act)) break;
        }
        __syncthreads();
        // ---- write back: interior pixels plainly, border pixels as deltas
        // (neighbour tiles may have pushed into them meanwhile)
        int still = 0;
        for (int j = 0; j < PPT; j++) {
            int i = tid + j * NT;
            int64_t p = base + i;
            int32_t e = sw[i];
            typename E::Word nw = E::pack(sr[0][i], sr[1][i], sr[2][i], sr[3][i]);
            if (!on_border(i)) {
                c.w[p] = e;
                E::store(c.r, p, nw);
            } else {
                if (e != wv[j]) atomicAdd(&c.w[p], e - wv[j]);
                E::store_delta(c.r, p, nw, rv[j]);
            }
            c.h[p] = sh[i];
            still |= e > 0 && sh[i] < HINF;
        }
        if (tid < 4 * TW) {
            int s = tid / TW, j = tid % TW;
            int32_t a = hacc[s][j];
            if (a > 0) {
                int64_t q = int64_t(g.nb[s]) * TPIX + halo_index(s, j);
                atomicAdd(&c.w[q], a);
                E::add(c.r, q, opp(s), a);
                s_out[s] = 1;
            }
        }
        still = __syncthreads_or(still);
        if (tid == 0 && still) enqueue(c, k + 1, t);
        if (tid < 4 && s_out[tid]) enqueue(c, k + 1, g.nb[tid]);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Labels: source-side closure of the excess pixels (solvers.py:144-158),
// then per-grid label bytes and flows.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(NT) k_lab_seed(Ctx c) {
    for (int64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        const GridDesc &gd = c.grids[c.tile_grid[t]];
        if (grid_swapped(c, gd)) continue;
        int any = 0;
        for (int j = 0; j < PPT; j++) {
            int64_t p = t * TPIX + threadIdx.x + j * NT;
            int v = c.w[p] > 0;
            c.lab[p] = uint8_t(v);
            any |= v;
        }
        if (__syncthreads_or(any) && threadIdx.x == 0) enqueue(c, 0, int32_t(t));
    }
}

template <class E>
__global__ void __launch_bounds__(NT) k_bfs_src(Ctx c, int k) {
    __shared__ uint8_t sl[TPIX];
    __shared__ uint8_t sm[TPIX];      // bit d: the d-neighbour has a residual arc INTO this pixel
    __shared__ uint8_t hl[4][TW];     // halo pixel reached and its arc into us residual
    __shared__ int s_side[4];
    const int32_t n = c.cnt[k % 3];
    const int32_t *lst = list_of(c, k);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c.cnt[(k + 2) % 3] = 0;
        atomicAdd(&c.stat[ST_LAB], (unsigned long long)n);
    }
    __shared__ uint32_t sword[TPIX];  // packed "arc > 0" bits per pixel
    for (int li = blockIdx.x; li < n; li += gridDim.x) {
        const int32_t t = lst[li];
        TileGeo g = tile_geo(c, t);
        const int64_t base = int64_t(t) * TPIX;
        uint8_t l0[PPT];
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            l0[j] = c.lab[base + i];
            sl[i] = l0[j];
            typename E::Word wd = E::load(c.r, base + i);
            sword[i] = uint32_t((E::lane(wd, 0) > 0) | ((E::lane(wd, 1) > 0) << 1) |
                                ((E::lane(wd, 2) > 0) << 2) | ((E::lane(wd, 3) > 0) << 3));
        }
        if (threadIdx.x < 4 * TW) {
            int s = threadIdx.x / TW, j = threadIdx.x % TW;
            uint8_t v = 0;
            if (g.nb[s] >= 0) {
                int64_t q = int64_t(g.nb[s]) * TPIX + halo_index(s, j);
                v = c.lab[q] && E::lane(E::load(c.r, q), opp(s)) > 0;
            }
            hl[s][j] = v;
            if (j == 0) s_side[s] = 0;
        }
        if (threadIdx.x == 0) inq_of(c, k)[t] = 0;
        __syncthreads();
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            int lx = i & (TW - 1), ly = i / TW;
            int mk = 0;
            if (lx && (sword[i - 1] & (1u << DR))) mk |= 1;
            if (lx < TW - 1 && (sword[i + 1] & (1u << DL))) mk |= 2;
            if (ly && (sword[i - TW] & (1u << DD))) mk |= 4;
            if (ly < TH - 1 && (sword[i + TW] & (1u << DU))) mk |= 8;
            sm[i] = uint8_t(mk);
        }
        __syncthreads();
        for (;;) {
            int changed = 0;
            for (int j = 0; j < PPT; j++) {
                int i = threadIdx.x + j * NT;
                if (sl[i]) continue;
                int lx = i & (TW - 1), ly = i / TW;
                int mk = sm[i];
                int r = 0;
                if (lx == 0) r |= hl[DL][ly];
                else if (mk & 1) r |= sl[i - 1];
                if (lx == TW - 1) r |= hl[DR][ly];
                else if (mk & 2) r |= sl[i + 1];
                if (ly == 0) r |= hl[DU][lx];
                else if (mk & 4) r |= sl[i - TW];
                if (ly == TH - 1) r |= hl[DD][lx];
                else if (mk & 8) r |= sl[i + TW];
                if (r) { sl[i] = 1; changed = 1; }
            }
            if (!__syncthreads_or(changed)) break;
        }
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            if (sl[i] != l0[j]) {
                c.lab[base + i] = 1;
                if (c.w[base + i] < 0) atomicExch(c.err, 4);   // NonMaximalFlowError
                int lx = i & (TW - 1), ly = i / TW;
                if (lx == 0) s_side[DL] = 1;
                if (lx == TW - 1) s_side[DR] = 1;
                if (ly == 0) s_side[DU] = 1;
                if (ly == TH - 1) s_side[DD] = 1;
            }
        }
        __syncthreads();
        if (threadIdx.x < 4 && s_side[threadIdx.x] && g.nb[threadIdx.x] >= 0)
            enqueue(c, k + 1, g.nb[threadIdx.x]);
        __syncthreads();
    }
}

// Label bytes in row-major order and the per-grid unused sink residual.
//   batch grid:  swapped ? sink side (h < HINF) : source side
//                (= split()'s decoded mask of the original graph)
//   composite:   swapped column ? ~sink side : source side
//                (supergraph.py:201-206)
__global__ void __launch_bounds__(NT) k_emit(Ctx c) {
    __shared__ int64_t red[NT / 32];
    for (int64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
        TileGeo g = tile_geo(c, int32_t(t));
        const GridDesc &gd = c.grids[g.g];
        int64_t drain = 0;
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            int x = g.x0 + (i & (TW - 1)), y = g.y0 + i / TW;
            if (x >= g.W || y >= g.H) continue;
            int64_t p = t * TPIX + i;
            int32_t wv = c.w[p];
            if (wv < 0) drain -= wv;
            uint8_t v;
            if (gd.kind == 1) {
                v = c.colswap[gd.colswap_off + x] ? uint8_t(c.h[p] >= HINF) : c.lab[p];
            } else {
                v = grid_swapped(c, gd) ? uint8_t(c.h[p] < HINF) : c.lab[p];
            }
            c.out[gd.out_off + int64_t(y) * g.W + x] = v;
        }
        int64_t s = block_sum64(drain, red);
        if (threadIdx.x == 0 && s) atomicAdd((unsigned long long *)&c.drain[g.g], (unsigned long long)s);
    }
}

}  // namespace pmf
