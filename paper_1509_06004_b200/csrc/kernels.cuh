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
#include <type_traits>

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

// Seed masks of a batch from its index lists (1 = fg seed, 2 = bg seed;
// mask zeroed by the caller): seeds[sofs[2p] .. sofs[2p+1]) are problem p's
// fg pixels, seeds[sofs[2p+1] .. sofs[2p+2]) its bg pixels (disjoint,
// checked on the host).
__global__ void k_seed_masks(uint8_t *mask, const int32_t *seeds, const int64_t *sofs, int32_t nprob, int64_t n) {
    for (int p = blockIdx.x; p < nprob; p += gridDim.x) {
        uint8_t *m = mask + int64_t(p) * n;
        for (int64_t j = sofs[2 * p] + threadIdx.x; j < sofs[2 * p + 2]; j += blockDim.x)
            m[seeds[j]] = j < sofs[2 * p + 1] ? 1 : 2;
    }
}

// ---------------------------------------------------------------------------
// On-device synthesis of CPMC seed batches (harness/synth.py:52-100): the
// planes of every (image, seed) problem are derived from the 8-bit images
// instead of crossing the host link (pmf_synth_stage).  Same integer
// arithmetic as the reference (INTENSITY_MAX = 255):
//   dsim = |I - I(seed)|          (problem_for_seed, synth.py:82)
//   unary_base  = 1 + (255 - dsim) * 15 / 255
//   unary_slope = 1 + (255 - dsim) *  7 / 255
//   sink_base   = 1 +        dsim  * 63 / 255
//   pairwise    = 1 + (255 - |dI|) * 63 / 255 on both arcs of an edge,
//                 0 on arcs leaving the image        (_pairwise_weights :52-64)
// Planes row-major, laid out as pmf_seed_stage stages them: three int32
// planes per (image, seed) (the seed types of a seed share them) and four
// pairwise planes per image.
// ---------------------------------------------------------------------------
constexpr int kIntensityMax = 255;

// one thread per 4 pixels of one (image, seed) problem; grid-stride.  With
// n % 4 == 0 every plane row of 4 pixels is one aligned 16 B store (and the
// 4 intensities one 4 B load); otherwise scalar stores.
__device__ __forceinline__ void synth_terms(int v, int s, int32_t &b, int32_t &sl, int32_t &sk) {
    const int d = abs(v - s);
    b = 1 + ((kIntensityMax - d) * 15) / kIntensityMax;
    sl = 1 + ((kIntensityMax - d) * 7) / kIntensityMax;
    sk = 1 + (d * 63) / kIntensityMax;
}

__global__ void __launch_bounds__(256) k_synth_planes(const uint8_t *img, int64_t n, int32_t nseed,
                                                      const int32_t *seed_pix, int64_t nu, int32_t *planes) {
    const int64_t n4 = (n + 3) / 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const bool vec = (n & 3) == 0;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nu * n4; t += stride) {
        const int64_t u = t / n4, q0 = (t % n4) * 4;
        const uint8_t *im = img + (u / nseed) * n;
        const int s = im[seed_pix[u]];
        int32_t *pb = planes + 3 * u * n;
        if (vec) {
            const uchar4 v = *reinterpret_cast<const uchar4 *>(im + q0);
            int4 b, sl, sk;
            synth_terms(v.x, s, b.x, sl.x, sk.x);
            synth_terms(v.y, s, b.y, sl.y, sk.y);
            synth_terms(v.z, s, b.z, sl.z, sk.z);
            synth_terms(v.w, s, b.w, sl.w, sk.w);
            *reinterpret_cast<int4 *>(pb + q0) = b;
            *reinterpret_cast<int4 *>(pb + n + q0) = sl;
            *reinterpret_cast<int4 *>(pb + 2 * n + q0) = sk;
            continue;
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int64_t q = q0 + k;
            if (q >= n) break;
            synth_terms(im[q], s, pb[q], pb[n + q], pb[2 * n + q]);
        }
    }
}

// one thread per pixel of one image: its four arcs (L, R, U, D)
__global__ void __launch_bounds__(256) k_synth_pw(const uint8_t *img, int32_t W, int32_t H, int32_t nimg,
                                                  int32_t *pw) {
    const int64_t n = int64_t(W) * H;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    auto w = [](int a, int b) { return 1 + ((kIntensityMax - abs(a - b)) * 63) / kIntensityMax; };
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < int64_t(nimg) * n; t += stride) {
        const int64_t i = t / n, q = t % n;
        const int x = int(q % W), y = int(q / W);
        const uint8_t *im = img + i * n;
        const int v = im[q];
        int32_t *o = pw + 4 * i * n;
        o[q] = x > 0 ? w(v, im[q - 1]) : 0;
        o[n + q] = x < W - 1 ? w(v, im[q + 1]) : 0;
        o[2 * n + q] = y > 0 ? w(v, im[q - W]) : 0;
        o[3 * n + q] = y < H - 1 ? w(v, im[q + W]) : 0;
    }
}

// Terminal balance at the mid-schedule lambda (supergraph.py:77-92, 210-212).
__device__ __forceinline__ int64_t block_sum64(int64_t v, int64_t *red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < int(blockDim.x >> 5); i++) s += red[i];
    __syncthreads();
    return s;
}

// One CTA per (problem, pixel chunk): block-reduced counts, two atomics.
__global__ void __launch_bounds__(256) k_swap_count(SeedArgs a, int chunks) {
    __shared__ int64_t red[256 / 32];
    const int32_t n = a.W * a.H;   // < 2^31 (checked by the stage)
    const int32_t per = int32_t((int64_t(n) + chunks - 1) / chunks);
    const int64_t lam = a.lambdas[a.mid];
    for (int64_t blk = blockIdx.x; blk < int64_t(a.nprob) * chunks; blk += gridDim.x) {
        const int p = int(blk / chunks);
        const int32_t lo = int32_t(blk % chunks) * per, hi = min(n, lo + per);
        const int32_t *bp = a.base + a.plane_off[p], *sp = a.slope + a.plane_off[p], *kp = a.sink + a.plane_off[p];
        const uint8_t *mask = a.mask + int64_t(p) * n;
        int64_t neg = 0, pos = 0;
        for (int32_t q = lo + threadIdx.x; q < hi; q += blockDim.x) {
            const uint8_t m = mask[q];
            const int64_t src = m == 1 ? CAP_MAX : int64_t(bp[q]) + lam * int64_t(sp[q]);
            const int64_t snk = m == 2 ? CAP_MAX : int64_t(kp[q]);
            neg += src < snk;
            pos += src > snk;
        }
        neg = block_sum64(neg, red);
        pos = block_sum64(pos, red);
        if (threadIdx.x == 0) {
            if (neg) atomicAdd(&a.swap_cnt[2 * p], int32_t(neg));
            if (pos) atomicAdd(&a.swap_cnt[2 * p + 1], int32_t(pos));
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
        const GridDesc &gd = c.grids[g.g];
        const int64_t off = a.plane_off[g.g];
        const int64_t n = int64_t(gd.pitch) * g.H;   // the composite's plane size
        int64_t snk_acc = 0;
        for (int j = 0; j < PPT; j++) {
            int i = threadIdx.x + j * NT;
            int x = g.x0 + (i & (TW - 1)), y = g.y0 + i / TW;
            int64_t p = t * TPIX + i;
            int32_t wv = 0;
            int e[4] = {0, 0, 0, 0};
            if (x < g.W && y < g.H) {
                int64_t q = int64_t(y) * gd.pitch + gd.xoff + x;
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

// Full-batch scans (relabel / seed / label / emit / advance in the
// step-synchronous mode) run one WARP per tile: lane l owns column l, and
// row r of the tile is pixel l + 32 r (TW == 32), so every row is one
// coalesced 128-byte access and a tile needs no block barrier.  Warps take
// their grid-stride tiles 32 at a time, testing the per-grid predicate
// (live, due) lane-parallel, so a skipped tile costs no load round trip of
// its own (one CTA per tile spent ~100 us a scan on C5, ~70% of whose tiles
// a rolling step skips).
static_assert(TW == 32 && TH == 32, "warp-per-tile scans assume 32x32 tiles");
// rows loaded before any store of the batch (stores may alias the loads, so
// the compiler cannot hoist the next row's loads above them)
constexpr int SCAN_ROWS = 8;
template <class Pred, class F>
__device__ __forceinline__ void for_tiles(const Ctx &c, Pred pred, F f) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t G = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = 0; w0 + r * G < c.ntiles; r += 32) {
        const int64_t t = w0 + (r + lane) * G;
        unsigned m = __ballot_sync(0xffffffffu, t < c.ntiles && pred(c.tile_grid[t]));
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            f(w0 + (r + k) * G, lane);
        }
    }
}

// Worklist / queue insertions of a seeding scan, as a mask per tile: bit 0
// the tile itself, bit 1 + s its neighbour on side s.
__device__ __forceinline__ void seed_mask(const Ctx &c, int32_t t, unsigned mask) {
    if (mask & 1u) seed_tile(c, t);
    for (int s = 0; s < 4; s++)
        if ((mask >> (s + 1)) & 1u) {
            const int32_t nb = tile_nb(c, t, s);
            if (nb >= 0) seed_tile(c, nb);
        }
}

// for_tiles for seeding scans: f returns the tile's seed mask (warp-
// uniform); the insertions -- dependent atomics on the worklist or queue
// state -- run after the warp's round of up to 32 tiles, each lane doing
// those of its own tile, so they overlap instead of stalling the warp tile
// after tile.  (A worklist's order does not matter.)
template <class Pred, class F>
__device__ __forceinline__ void for_tiles_seed(const Ctx &c, Pred pred, F f) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t G = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = 0; w0 + r * G < c.ntiles; r += 32) {
        const int64_t t = w0 + (r + lane) * G;
        unsigned m = __ballot_sync(0xffffffffu, t < c.ntiles && pred(c.tile_grid[t]));
        unsigned mine = 0;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const unsigned sm = f(w0 + (r + k) * G, lane);
            if (lane == k) mine = sm;
        }
        if (mine) seed_mask(c, int32_t(t), mine);
    }
}

// Seed mask of a BFS phase (warp per tile): the tile if it holds a seed
// pixel, and every neighbour facing a seed on its border -- a seed never
// "changes", so the relaxation of the tile alone would never hand it
// across the tile boundary.  `seeds` bit r = pixel (lane, row r) is a seed.
// need_open: a tile whose every pixel is a seed is not listed itself (its
// relaxation could add nothing), only the neighbours facing its border.
__device__ __forceinline__ unsigned halo_seed_mask(unsigned seeds, bool need_open = false) {
    const unsigned cols = __ballot_sync(0xffffffffu, seeds != 0);
    const unsigned top = __ballot_sync(0xffffffffu, seeds & 1u), bottom = __ballot_sync(0xffffffffu, seeds >> (TH - 1));
    const bool open = !need_open || __any_sync(0xffffffffu, seeds != 0xffffffffu);
    if (!cols) return 0u;
    return (open ? 1u : 0u) | (cols & 1u ? 2u << DL : 0u) | (cols >> 31 ? 2u << DR : 0u) | (top ? 2u << DU : 0u) |
           (bottom ? 2u << DD : 0u);
}

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// h = 1 on pixels with sink residual (w < 0), HINF elsewhere; lists every
// tile holding such a pixel (and its neighbours facing one).  Tiles of
// finished grids are left untouched.
__global__ void __launch_bounds__(NT) k_gr_init(Ctx c) {
    for_tiles_seed(c, [&](int32_t g) { return c.live[g] && !(c.keeph && c.keeph[g]); }, [&](int64_t t, int lane) {
        unsigned seeds = 0;
        const int64_t p0 = t * TPIX + lane;
#pragma unroll
        for (int r0 = 0; r0 < TH; r0 += SCAN_ROWS) {
            int32_t wv[SCAN_ROWS];   // loads of the batch before its stores (they may alias)
#pragma unroll
            for (int k = 0; k < SCAN_ROWS; k++) wv[k] = c.w[p0 + TW * (r0 + k)];
#pragma unroll
            for (int k = 0; k < SCAN_ROWS; k++) {
                c.h[p0 + TW * (r0 + k)] = wv[k] < 0 ? 1 : HINF;
                seeds |= unsigned(wv[k] < 0) << (r0 + k);
            }
        }
        return halo_seed_mask(seeds);
    });
}

// ---------------------------------------------------------------------------
// Push-relabel discharge of one tile in shared memory (solvers.py:107-136
// semantics: push min(e, r) along admissible arcs h(p) == h(q) + 1, in
// direction order L, R, U, D; relabel to 1 + min residual-neighbour height).
// ---------------------------------------------------------------------------

// Lists every tile of a live grid that holds an active pixel (w > 0,
// h < HINF); counts active pixels per grid.
__global__ void __launch_bounds__(NT) k_seed_push(Ctx c) {
    for_tiles_seed(c, [&](int32_t g) { return c.live[g] != 0; }, [&](int64_t t, int lane) {
        int a = 0;
#pragma unroll 8
        for (int r = 0; r < TH; r++) {
            const int64_t p = t * TPIX + lane + TW * r;
            a += c.w[p] > 0 && c.h[p] < HINF;
        }   // no stores: the loads pipeline
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0 && a) {
            atomicAdd(&c.act[c.tile_grid[t]], a);
            if (c.tfresh) c.tfresh[t] = 1;   // its heights are this relabel's exact distances
        }
        return a ? 1u : 0u;
    });
}

// Reset the worklist (sweep mode) or queue (persistent mode) state for a
// new phase and, in graph mode, arm the conditional of the loop that
// follows.  Replaces host memsets so the whole solve can run as one graph.
__global__ void k_phase_begin(Ctx c, int persistent, cudaGraphConditionalHandle cond, int has_cond) {
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t t = tid; t < c.ntiles; t += stride) {
        if (persistent) {
            c.qstate[t] = Q_IDLE;
            c.ring[t] = -1;
        } else {
            c.inq0[t] = 0;
            c.inq1[t] = 0;
        }
    }
    if (persistent)
        for (int64_t g = tid; g < c.ngrids; g += stride) c.gpend[g] = 0;
    if (tid == 0) {
        c.cnt[0] = c.cnt[1] = c.cnt[2] = 0;
        for (int q = 0; q < 4; q++) c.qctr[q] = 0;
        c.ctl->k = 0;
        c.ctl->done = 0;
        c.ctl->t0 = ~0ull;
        c.ctl->t1 = 0;
        if (has_cond) cudaGraphSetConditional(cond, 1u);
    }
}

// End of a seeding pass (one CTA): retire grids without active pixels,
// record how many tiles were seeded, size the next discharge's pop budget,
// count the cycle and decide (graph mode: via the cycle loop's conditional)
// whether another discharge + global relabel round is needed.
__global__ void __launch_bounds__(1024) k_cycle_ctl(Ctx c, int32_t ngrids, int persistent,
                                                    unsigned budget_factor, int64_t max_cycles,
                                                    cudaGraphConditionalHandle cond, int has_cond,
                                                    cudaGraphConditionalHandle cond_lab, int has_lab) {
    __shared__ int s_fin;
    if (threadIdx.x == 0) s_fin = 0;
    __syncthreads();
    int nfin = 0;
    for (int g = threadIdx.x; g < ngrids; g += blockDim.x) {
        // seeded with kept heights (relabel from the next cycle on); their
        // HINF marks may come from a speculative finish and certify nothing,
        // so a grid with no active pixel finishes speculatively
        const bool kept = c.keeph && c.keeph[g];
        if (kept) c.keeph[g] = 0;
        if (c.live[g] && c.act[g] == 0) {
            c.live[g] = 0;
            if (c.rolling) {
                c.fin[g] = 1;
                if (kept) c.specg[g] = 1;
                nfin++;
            }
        }
        c.act[g] = 0;
    }
    if (nfin) atomicAdd(&s_fin, nfin);
    __syncthreads();
    if (threadIdx.x == 0) {
        Ctl *ctl = c.ctl;
        int32_t nact = persistent ? int32_t(c.qctr[QC_PENDING]) : c.cnt[0];
        int32_t cyc = ++ctl->cycle;
        ctl->cycles_total++;
        int stop = nact == 0;
        if (!stop && cyc > max_cycles) {
            ctl->noconv = 1;
            stop = 1;
        }
        ctl->nact = nact;
        ctl->nfin = s_fin;
        // pop budget of the discharge that follows (0 = run none)
        uint64_t cap = uint64_t(64) * uint64_t(c.ntiles) + 1024;
        uint64_t want = budget_factor ? uint64_t(budget_factor) * uint64_t(nact) + 64 : cap;
        ctl->budget = stop ? 0u : unsigned(want < cap ? want : cap);
        // rolling mode: finished grids run the label block (which decides
        // whether the cycle loop goes on once they have advanced)
        if (has_cond) cudaGraphSetConditional(cond, (!stop || (s_fin && !ctl->noconv)) ? 1u : 0u);
        if (has_lab) cudaGraphSetConditional(cond_lab, s_fin ? 1u : 0u);
    }
}

// Rolling mode, after a discharge: a live unswapped grid none of whose tiles
// is still queued or running drained its discharge.  That alone certifies
// nothing (see async.cuh), but the label closure of its excess pixels does:
// the grid joins this cycle's label round speculatively (specg = 1); a
// closure that reaches a sink-residual pixel marks it spoiled (2) and
// k_unspoil sends it back to relabel and discharge.
__global__ void __launch_bounds__(1024) k_push_spec(Ctx c, int32_t ngrids, cudaGraphConditionalHandle cond,
                                                    int has_cond, cudaGraphConditionalHandle cond_lab,
                                                    int has_lab) {
    __shared__ int s_fin;
    if (threadIdx.x == 0) s_fin = 0;
    __syncthreads();
    int nfin = 0;
    for (int g = threadIdx.x; g < ngrids; g += blockDim.x) {
        if (c.live[g] && c.gpend[g] == 0 && !grid_swapped(c, c.grids[g])) {
            c.live[g] = 0;
            c.fin[g] = 1;
            c.specg[g] = 1;
            nfin++;
        }
    }
    if (nfin) atomicAdd(&s_fin, nfin);
    __syncthreads();
    if (threadIdx.x == 0 && s_fin && !c.ctl->noconv) {
        c.ctl->nfin += s_fin;
        atomicAdd(&c.stat[ST_SPEC_ROLL], (unsigned long long)s_fin);
        if (has_cond) cudaGraphSetConditional(cond, 1u);
        if (has_lab) cudaGraphSetConditional(cond_lab, 1u);
    }
}

// After the label closure of a rolling round: spoiled speculative grids go
// back to the live set (no labels, no advance); the others finish.
__global__ void __launch_bounds__(1024) k_unspoil(Ctx c, int32_t ngrids) {
    int n = 0;
    for (int g = threadIdx.x; g < ngrids; g += blockDim.x) {
        const int sp = c.specg[g];
        if (sp == 2) {
            c.fin[g] = 0;
            c.live[g] = 1;
            if (c.labok) c.labok[g] = 0;   // lab holds a spoiled closure
            n++;
        }
        if (sp) c.specg[g] = 0;
    }
    if (n) atomicAdd(&c.stat[ST_SPOIL_ROLL], (unsigned long long)n);
}

// ---------------------------------------------------------------------------
// Labels: source-side closure of the excess pixels (solvers.py:144-158),
// then per-grid label bytes and flows.
// ---------------------------------------------------------------------------

// Seeds of the label closure: the excess pixels, plus -- chain grids whose
// previous lambda's labels are final (c.labok) -- that lambda's minimal
// source side, still in lab: minimal source sides are nested along a
// monotone schedule (parametric.py:191-201), and its pixels never regain a
// sink residual (w >= 0 stays >= 0), so the closure is unchanged and only
// travels the new ring.  Tiles already inside it are not relaxed.
__global__ void __launch_bounds__(NT) k_lab_seed(Ctx c) {
    for_tiles_seed(c, [&](int32_t g) { return grid_due(c, g) && !grid_swapped(c, c.grids[g]); }, [&](int64_t t, int lane) {
        const bool nested = c.labok && c.labok[c.tile_grid[t]];
        unsigned seeds = 0;
        const int64_t p0 = t * TPIX + lane;
#pragma unroll
        for (int r0 = 0; r0 < TH; r0 += SCAN_ROWS) {
            int32_t wv[SCAN_ROWS];
            uint8_t lv[SCAN_ROWS];
#pragma unroll
            for (int k = 0; k < SCAN_ROWS; k++) {
                wv[k] = c.w[p0 + TW * (r0 + k)];
                lv[k] = nested ? c.lab[p0 + TW * (r0 + k)] : 0;
            }
#pragma unroll
            for (int k = 0; k < SCAN_ROWS; k++) {
                const bool v = wv[k] > 0 || lv[k];
                c.lab[p0 + TW * (r0 + k)] = uint8_t(v);
                seeds |= unsigned(v) << (r0 + k);
            }
        }
        return halo_seed_mask(seeds, nested);
    });
}

// Label bytes in row-major order and the per-grid unused sink residual.
//   batch grid:  swapped ? sink side (h < HINF) : source side
//                (= split()'s decoded mask of the original graph)
//   composite:   swapped column ? ~sink side : source side
//                (supergraph.py:201-206)
__global__ void __launch_bounds__(NT) k_emit(Ctx c) {
    for_tiles(c, [&](int32_t g) { return grid_due(c, g); }, [&](int64_t t, int lane) {
        const TileGeo g = tile_geo(c, int32_t(t));
        const GridDesc &gd = c.grids[g.g];
        const bool comp = gd.kind == 1, swapped = !comp && grid_swapped(c, gd);
        const int x = g.x0 + lane;
        const bool cswap = comp && x < g.W && c.colswap[gd.colswap_off + x];
        const int64_t off = comp ? gd.out_off + gd.xoff : (int64_t(gd.prob) * c.nlam + c.cur_lam[g.g]) * (int64_t(g.W) * g.H);
        int64_t drain = 0;
        const int rows = min(TH, g.H - g.y0);
        // h decides the side when the grid (column) is swapped, lab otherwise
        const bool use_h = comp ? cswap : swapped;
        const bool h_inf_side = comp;   // composite swapped column: side = h >= HINF
        if (x < g.W)
#pragma unroll
            for (int r0 = 0; r0 < TH; r0 += SCAN_ROWS) {
                int32_t wv[SCAN_ROWS];
                uint8_t v[SCAN_ROWS];
#pragma unroll
                for (int k = 0; k < SCAN_ROWS; k++) {
                    const int64_t p = t * TPIX + lane + TW * (r0 + k);
                    const bool in = r0 + k < rows;
                    wv[k] = in ? c.w[p] : 0;
                    v[k] = !in ? 0 : use_h ? uint8_t((c.h[p] >= HINF) == h_inf_side) : c.lab[p];
                }
#pragma unroll
                for (int k = 0; k < SCAN_ROWS; k++) {
                    if (wv[k] < 0) drain -= wv[k];
                    if (r0 + k < rows) c.out[off + int64_t(g.y0 + r0 + k) * gd.pitch + x] = v[k];
                }
            }
        drain = warp_sum64(drain);
        if (lane == 0 && drain) atomicAdd((unsigned long long *)&c.drain[g.g], (unsigned long long)drain);
    });
}

}  // namespace pmf

namespace pmf {

// Label bytes (0/1) -> bit array for the D2H (8x fewer bytes over the host
// link): bit j of word w is byte 32*w + j.  One thread per word: two 16-byte
// loads, and each 4-byte group's low bits gathered by one multiply
// ((v & 0x01010101) * 0x10204080 puts bytes 0..3 at bits 28..31).
__device__ __forceinline__ uint32_t gather4(uint32_t v) { return ((v & 0x01010101u) * 0x10204080u) >> 28; }
__global__ void k_pack_bits(const uint8_t *__restrict__ bytes, uint32_t *__restrict__ bits, int64_t n) {
    const int64_t nw = n / 32;
    for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < (n + 31) / 32;
         w += int64_t(gridDim.x) * blockDim.x) {
        uint32_t out = 0;
        if (w < nw) {
            const uint4 u = __ldcs(reinterpret_cast<const uint4 *>(bytes) + 2 * w);
            const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(bytes) + 2 * w + 1);
            out = gather4(u.x) | gather4(u.y) << 4 | gather4(u.z) << 8 | gather4(u.w) << 12 |
                  gather4(v.x) << 16 | gather4(v.y) << 20 | gather4(v.z) << 24 | gather4(v.w) << 28;
        } else {
            for (int64_t i = 32 * w; i < n; i++) out |= uint32_t(bytes[i] != 0) << (i - 32 * w);
        }
        bits[w] = out;
    }
}

// Arm a conditional node (graph mode): 1 before the loop it controls.
__global__ void k_arm(cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, 1u); }

// Per-grid results of a solved step: flow = sum of (embedded) sink
// capacities minus the sink residual left unused (solvers.py:140, reduced
// network), stored at the grid's (problem, lambda) slot.
__global__ void k_finalize(Ctx c, int32_t ngrids) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngrids; g += gridDim.x * blockDim.x) {
        if (!grid_due(c, g)) continue;
        const GridDesc &gd = c.grids[g];
        const int64_t idx = gd.kind == 1 ? g : int64_t(gd.prob) * c.nlam + c.cur_lam[g];
        c.flows[idx] = c.snk_sum[g] - c.drain[g];
        c.drain[g] = 0;
    }
}

// Warm start along the nested schedule: the maximum
// preflow of lambda_i stays a valid preflow of lambda_{i+1} -- only the
// terminal capacities grow (source arcs of unswapped grids, sink arcs of
// swapped ones, parametric.py:147) -- so the next solve starts from it.
// Non-fg pixels gain (lambda_{i+1} - lambda_i) * slope of source (w +=) or,
// embedded swapped, of sink capacity (w -=).
// Rolling warm start, fused k_emit + k_advance_tiles for seed-batch grids
// (one pass over w instead of two): label bytes and unused sink residual of
// the finished lambda, then -- when the chain has a next lambda -- its
// terminal advance w += sign * (lambda_{i+1} - lambda_i) * slope.
#ifndef EMIT_ROWS
#define EMIT_ROWS 1
#endif
#ifndef EMIT_MINB
#define EMIT_MINB 8
#endif
// One row per step, per-tile base pointers advanced per row: 32 registers,
// full occupancy (the unrolled 8-row form needed 76 registers -- a third of
// the SM's warps in flight, 2.6 TB/s; this form: C5 step -1.2 %).
__global__ void __launch_bounds__(NT, EMIT_MINB) k_emit_advance(Ctx c, SeedArgs a) {
    constexpr int ER = EMIT_ROWS;
    const int64_t n = int64_t(a.W) * a.H;
    for_tiles(c, [&](int32_t g) { return grid_due(c, g); }, [&](int64_t t, int lane) {
        const TileGeo g = tile_geo(c, int32_t(t));
        const GridDesc &gd = c.grids[g.g];
        const bool swapped = grid_swapped(c, gd);
        const int cur = c.cur_lam[g.g];
        const bool next = cur + 1 < gd.lam_end;
        const int64_t mul = next ? int64_t(c.swapflag[gd.prob] ? -1 : 1) * (a.lambdas[cur + 1] - a.lambdas[cur]) : 0;
        int64_t drain = 0;
        const int x = g.x0 + lane, rows = min(TH, g.H - g.y0);
        if (x < g.W) {
            // row pointers advanced per chunk; rows inside a chunk at
            // constant (tile) or one-multiply (image) offsets, so no
            // per-row 64-bit induction variables stay live
            int32_t *wp = c.w + t * TPIX + lane;
            const int32_t *hp = c.h + t * TPIX + lane;
            const uint8_t *lp = c.lab + t * TPIX + lane;
            const int64_t q0 = int64_t(g.y0) * a.W + x;
            const uint8_t *mp = a.mask + int64_t(gd.prob) * n + q0;
            const int32_t *sp = a.slope + a.plane_off[gd.prob] + q0;
            uint8_t *op = c.out + (int64_t(gd.prob) * c.nlam + cur) * n + int64_t(g.y0) * g.W + x;
            const int aw = a.W, gw = g.W;
#pragma unroll 1
            for (int r0 = 0; r0 < rows; r0 += ER) {
                int32_t wv[ER], d[ER];
                uint8_t v[ER];
#pragma unroll
                for (int k = 0; k < ER; k++) {
                    const bool in = r0 + k < rows;
                    wv[k] = in ? wp[TW * k] : 0;
                    // swapped grid: its sink side {h < HINF}; else the source-side closure
                    v[k] = !in ? 0 : swapped ? uint8_t(hp[TW * k] < HINF) : lp[TW * k];
                    const uint8_t m = in && next ? mp[k * aw] : 1;   // fg seed: CAP_MAX either way
                    const int32_t sv = in && next ? sp[k * aw] : 0;
                    d[k] = m != 1 ? int32_t(mul * int64_t(sv)) : 0;
                }
#pragma unroll
                for (int k = 0; k < ER; k++) {
                    if (wv[k] < 0) drain -= wv[k];
                    if (r0 + k < rows) {
                        op[k * gw] = v[k];
                        if (d[k]) wp[TW * k] = wv[k] + d[k];
                    }
                }
                wp += ER * TW;
                hp += ER * TW;
                lp += ER * TW;
                mp += ER * aw;
                sp += ER * aw;
                op += ER * gw;
            }
        }
        drain = warp_sum64(drain);
        if (lane == 0 && drain) atomicAdd((unsigned long long *)&c.drain[g.g], (unsigned long long)drain);
    });
}

__global__ void __launch_bounds__(NT) k_advance_tiles(Ctx c, SeedArgs a) {
    const int64_t n = int64_t(a.W) * a.H;
    for_tiles(c, [&](int32_t g) { return grid_due(c, g) && c.cur_lam[g] + 1 < c.grids[g].lam_end; },
              [&](int64_t t, int lane) {
        const TileGeo g = tile_geo(c, int32_t(t));
        const GridDesc &gd = c.grids[g.g];
        const int cur = c.cur_lam[g.g];
        const int64_t dl = a.lambdas[cur + 1] - a.lambdas[cur];
        const int sign = c.swapflag[gd.prob] ? -1 : 1;
        const int32_t *slope = a.slope + a.plane_off[gd.prob];
        const uint8_t *mask = a.mask + int64_t(gd.prob) * n;
        const int x = g.x0 + lane, rows = min(TH, g.H - g.y0);
        if (x < g.W)
#pragma unroll
            for (int r0 = 0; r0 < TH; r0 += SCAN_ROWS) {
                int32_t d[SCAN_ROWS], wv[SCAN_ROWS];
#pragma unroll
                for (int k = 0; k < SCAN_ROWS; k++) {
                    const bool in = r0 + k < rows;
                    const int64_t q = int64_t(g.y0 + r0 + k) * a.W + x;
                    // fg seed: CAP_MAX either way (both loads issued, no load behind a load)
                    const uint8_t m = in ? mask[q] : 1;
                    const int32_t sv = in ? slope[q] : 0;
                    d[k] = m != 1 ? int32_t(sign * dl * int64_t(sv)) : 0;
                    wv[k] = in ? c.w[t * TPIX + lane + TW * (r0 + k)] : 0;
                }
#pragma unroll
                for (int k = 0; k < SCAN_ROWS; k++)
                    if (d[k]) c.w[t * TPIX + lane + TW * (r0 + k)] = wv[k] + d[k];
            }
    });
}

// Integrity certificate per (problem, lambda) (grid.py:159-178 cut_cost;
// the reference checks it in split(), supergraph.py:181-186, and in the RPC
// client, rpc.py:328-331): the cut cost of the emitted mask of the ORIGINAL
// graph must equal the flow.
// One CTA per (problem, chunk of pixels): a thread loads its VPX pixels'
// terms once per VLAM lambdas and then issues every label load of the pass
// unconditionally (no load behind a branch on another load: the pass is
// latency-bound, so the loads must be in flight together); partial cut
// costs are summed per (problem, lambda) into acc (zeroed by the caller) and
// compared with the flows by k_verify_check.  Pixel indices within a plane
// are 32-bit (launch_verify rejects planes of 2^31 pixels or more).
constexpr int VPX = 2;     // pixels per thread per round
constexpr int VLAM = 10;   // lambdas per pass over the problem's planes (register accumulators)
// NARROW: pairwise capacities <= 255 (EdgeU8 batches), so a source-side
// pixel's cost (sink <= CAP_MAX = 2^30 plus four arcs) fits 32 bits
template <bool NARROW>
__global__ void __launch_bounds__(NT, 3) k_verify(Ctx c, SeedArgs a, unsigned long long *acc, int chunks) {
    using SS = typename std::conditional<NARROW, int32_t, int64_t>::type;
    __shared__ unsigned long long s_acc[VLAM];
    const int32_t n = a.W * a.H;
    const int32_t per = int32_t((int64_t(n) + chunks - 1) / chunks);
    for (int64_t blk = blockIdx.x; blk < int64_t(a.nprob) * chunks; blk += gridDim.x) {
        const int p = int(blk / chunks);
        const int32_t lo = int32_t(blk % chunks) * per, hi = min(n, lo + per);
        const int32_t *bp = a.base + a.plane_off[p], *sp = a.slope + a.plane_off[p], *kp = a.sink + a.plane_off[p];
        const int32_t *pw = a.pw + a.pw_off[p];
        const uint8_t *mask = a.mask + int64_t(p) * n;
        for (int j0 = 0; j0 < a.nlam; j0 += VLAM) {
            const int nj = min(VLAM, a.nlam - j0);
            int64_t cost[VLAM];
#pragma unroll
            for (int jj = 0; jj < VLAM; jj++) cost[jj] = 0;
            if (threadIdx.x < VLAM) s_acc[threadIdx.x] = 0;
            for (int32_t q0 = lo; q0 < hi; q0 += NT * VPX) {
                int32_t qq[VPX], a0[VPX], a1[VPX], a2[VPX], a3[VPX], sk[VPX];
                int64_t bs[VPX], sl[VPX];
#pragma unroll
                for (int k = 0; k < VPX; k++) {
                    const int32_t q = q0 + threadIdx.x + k * NT;
                    const bool ok = q < hi;
                    qq[k] = ok ? q : lo;   // a pixel past the chunk reads a valid label and adds 0
                    const int32_t x = ok ? q % a.W : 0, y = ok ? q / a.W : 0;
                    const uint8_t m = ok ? mask[q] : 0;
                    // m == 1 (fg seed): CAP_MAX when on the sink side; m == 2 (bg
                    // seed): CAP_MAX when on the source side
                    bs[k] = !ok ? 0 : m == 1 ? CAP_MAX : bp[q];
                    sl[k] = !ok || m == 1 ? 0 : sp[q];
                    sk[k] = !ok ? 0 : m == 2 ? int32_t(CAP_MAX) : kp[q];
                    a0[k] = ok && x > 0 ? pw[q] : 0;
                    a1[k] = ok && x + 1 < a.W ? pw[int64_t(n) + q] : 0;
                    a2[k] = ok && y > 0 ? pw[2 * int64_t(n) + q] : 0;
                    a3[k] = ok && y + 1 < a.H ? pw[3 * int64_t(n) + q] : 0;
                }
                const uint8_t *lab = c.out + (int64_t(p) * a.nlam + j0) * n;
                // no branches in here: every load of the pass can be in flight at
                // once (lambdas past nj re-read the last plane and add 0)
#pragma unroll
                for (int jj = 0; jj < VLAM; jj++) {
                    const int j = min(jj, nj - 1);
                    const uint8_t *l = lab + int64_t(j) * n;
                    const int64_t lam = a.lambdas[j0 + j];
#pragma unroll
                    for (int k = 0; k < VPX; k++) {
                        const int32_t q = qq[k];
                        const uint8_t l0 = l[q];
                        const uint8_t ll = a0[k] ? l[q - 1] : 1, lr = a1[k] ? l[q + 1] : 1;
                        const uint8_t lu = a2[k] ? l[q - a.W] : 1, ld = a3[k] ? l[q + a.W] : 1;
                        // arcs leaving the source side (off-grid counts as source side)
                        const SS src_side = SS(sk[k]) + SS(ll ? 0 : a0[k]) + SS(lr ? 0 : a1[k]) +
                                            SS(lu ? 0 : a2[k]) + SS(ld ? 0 : a3[k]);
                        const int64_t v = l0 ? int64_t(src_side) : bs[k] + lam * sl[k];
                        cost[jj] += jj < nj ? v : 0;
                    }
                }
            }
            __syncthreads();
#pragma unroll
            for (int jj = 0; jj < VLAM; jj++) {
                int64_t v = cost[jj];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_acc[jj], (unsigned long long)v);
            }
            __syncthreads();
            if (threadIdx.x < nj && s_acc[threadIdx.x])
                atomicAdd(acc + int64_t(p) * a.nlam + j0 + threadIdx.x, s_acc[threadIdx.x]);
            __syncthreads();
        }
    }
}

// Scores of every emitted mask against its problem's ground-truth mask
// (harness/bench.py:36-45 overlap, :104-111 foreground): per (problem,
// lambda) plane the foreground count |S|, |S & G| and |S | G|, summed into
// acc[3 * plane + {0, 1, 2}] (zeroed by the caller).  One CTA per (plane,
// pixel chunk), 16 bytes per thread per step.
__global__ void __launch_bounds__(NT) k_score(const uint8_t *__restrict__ out, const uint8_t *__restrict__ truth,
                                              int32_t nprob, int32_t nlam, int64_t n, int chunks,
                                              unsigned long long *acc) {
    __shared__ int64_t red[NT / 32];
    const int64_t per = ((n + chunks - 1) / chunks + 15) / 16 * 16;
    for (int64_t blk = blockIdx.x; blk < int64_t(nprob) * nlam * chunks; blk += gridDim.x) {
        const int64_t plane = blk / chunks;
        const int64_t lo = (blk % chunks) * per, hi = min(n, lo + per);
        const uint8_t *m = out + plane * n;
        const uint8_t *g = truth + (plane / nlam) * n;
        int64_t fg = 0, in = 0, un = 0;
        for (int64_t q = lo + threadIdx.x; q < hi; q += NT) {
            const int a = m[q] != 0, b = g[q] != 0;
            fg += a;
            in += a & b;
            un += a | b;
        }
        const int64_t sf = block_sum64(fg, red), si = block_sum64(in, red), su = block_sum64(un, red);
        if (threadIdx.x == 0) {
            if (sf) atomicAdd(acc + 3 * plane + 0, (unsigned long long)sf);
            if (si) atomicAdd(acc + 3 * plane + 1, (unsigned long long)si);
            if (su) atomicAdd(acc + 3 * plane + 2, (unsigned long long)su);
        }
    }
}

// k_verify for images with W % 4 == 0: a thread owns 4 consecutive pixels of
// one row, so per lambda its labels, the row above and the row below are
// three 4-byte loads plus two predicated edge bytes (5 loads per 4 pixels
// instead of 20), and its terms are 16-byte loads.  Every offset (plane_off,
// pw_off, label planes) is a multiple of n, hence of 4.
// lambdas per pass over the problem planes: 10 (C5's 20-lambda ladder in
// two passes instead of three, 80 registers without spills; 8 -> 10 measured
// -0.5 % of the C5 step, 20 spills)
#ifndef PMF_VLAM4
#define PMF_VLAM4 10
#endif
constexpr int VLAM4 = PMF_VLAM4;
template <bool NARROW>
#ifndef PMF_VMINB
#define PMF_VMINB 4
#endif
__global__ void __launch_bounds__(NT, PMF_VMINB) k_verify4(Ctx c, SeedArgs a, unsigned long long *acc, int chunks) {
    using SS = typename std::conditional<NARROW, int32_t, int64_t>::type;
    __shared__ unsigned long long s_acc[VLAM4];
    const int32_t n = a.W * a.H, n4 = n / 4, W = a.W;
    const int32_t per = int32_t((int64_t(n4) + chunks - 1) / chunks);
    for (int64_t blk = blockIdx.x; blk < int64_t(a.nprob) * chunks; blk += gridDim.x) {
        const int p = int(blk / chunks);
        const int32_t lo = int32_t(blk % chunks) * per, hi = min(n4, lo + per);
        const int4 *bp = reinterpret_cast<const int4 *>(a.base + a.plane_off[p]);
        const int4 *sp = reinterpret_cast<const int4 *>(a.slope + a.plane_off[p]);
        const int4 *kp = reinterpret_cast<const int4 *>(a.sink + a.plane_off[p]);
        const int4 *pw = reinterpret_cast<const int4 *>(a.pw + a.pw_off[p]);
        const uint32_t *mask = reinterpret_cast<const uint32_t *>(a.mask + int64_t(p) * n);
        for (int j0 = 0; j0 < a.nlam; j0 += VLAM4) {
            const int nj = min(VLAM4, a.nlam - j0);
            int64_t cost[VLAM4];
#pragma unroll
            for (int jj = 0; jj < VLAM4; jj++) cost[jj] = 0;
            if (threadIdx.x < VLAM4) s_acc[threadIdx.x] = 0;
            for (int32_t g0 = lo; g0 < hi; g0 += NT) {
                const int32_t g = g0 + threadIdx.x;
                const bool ok = g < hi;
                const int32_t gq = ok ? g : lo, q = 4 * gq;   // a group past the chunk adds 0
                const int32_t x = q % W, y = q / W;
                const uint32_t m4 = mask[gq];
                const int4 B = bp[gq], S = sp[gq], K = kp[gq];
                int4 A0 = pw[gq], A1 = pw[n4 + gq], A2 = pw[2 * n4 + gq], A3 = pw[3 * n4 + gq];
                if (x == 0) A0.x = 0;
                if (x + 4 == W) A1.w = 0;
                if (y == 0) A2 = make_int4(0, 0, 0, 0);
                if (y + 1 == a.H) A3 = make_int4(0, 0, 0, 0);
                if (!ok) A0 = A1 = A2 = A3 = make_int4(0, 0, 0, 0);
                const int32_t bb[4] = {B.x, B.y, B.z, B.w}, ss[4] = {S.x, S.y, S.z, S.w}, kk[4] = {K.x, K.y, K.z, K.w};
                const int32_t a0[4] = {A0.x, A0.y, A0.z, A0.w}, a1[4] = {A1.x, A1.y, A1.z, A1.w};
                const int32_t a2[4] = {A2.x, A2.y, A2.z, A2.w}, a3[4] = {A3.x, A3.y, A3.z, A3.w};
                int64_t bs[4], sl[4];
                int32_t sk[4];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const uint32_t m = (m4 >> (8 * i)) & 0xffu;
                    bs[i] = !ok ? 0 : m == 1 ? CAP_MAX : bb[i];
                    sl[i] = !ok || m == 1 ? 0 : ss[i];
                    sk[i] = !ok ? 0 : m == 2 ? int32_t(CAP_MAX) : kk[i];
                }
                const uint8_t *lab = c.out + (int64_t(p) * a.nlam + j0) * n;
#pragma unroll
                for (int jj = 0; jj < VLAM4; jj++) {
                    const int j = min(jj, nj - 1);
                    const uint8_t *l = lab + int64_t(j) * n + q;
                    const int64_t lam = a.lambdas[j0 + j];
                    const uint32_t L = *reinterpret_cast<const uint32_t *>(l);
                    // off-grid neighbours count as source side (their arcs are 0 anyway)
                    const uint32_t U = y > 0 ? *reinterpret_cast<const uint32_t *>(l - W) : 0x01010101u;
                    const uint32_t D = y + 1 < a.H ? *reinterpret_cast<const uint32_t *>(l + W) : 0x01010101u;
                    const uint32_t lb = x > 0 ? l[-1] : 1u, rb = x + 4 < W ? l[4] : 1u;
                    const uint32_t left = (L << 8) | lb, right = (L >> 8) | (rb << 24);
                    int64_t v = 0;
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int sh = 8 * i;
                        const SS src_side = SS(sk[i]) + SS((left >> sh) & 1u ? 0 : a0[i]) +
                                            SS((right >> sh) & 1u ? 0 : a1[i]) + SS((U >> sh) & 1u ? 0 : a2[i]) +
                                            SS((D >> sh) & 1u ? 0 : a3[i]);
                        v += (L >> sh) & 1u ? int64_t(src_side) : bs[i] + lam * sl[i];
                    }
                    cost[jj] += jj < nj ? v : 0;
                }
            }
            __syncthreads();
#pragma unroll
            for (int jj = 0; jj < VLAM4; jj++) {
                int64_t v = cost[jj];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_acc[jj], (unsigned long long)v);
            }
            __syncthreads();
            if (threadIdx.x < nj && s_acc[threadIdx.x])
                atomicAdd(acc + int64_t(p) * a.nlam + j0 + threadIdx.x, s_acc[threadIdx.x]);
            __syncthreads();
        }
    }
}

__global__ void k_flip_label(uint8_t *out, int64_t q) { out[q] ^= 1; }

// Integrity certificate of a composite solve (supergraph.py:181-186 split's
// sum check, rpc.py:328-331 the client's check): the cut cost of every
// composite's emitted labels on its own (admitted) planes, summed into
// acc[c] and compared with its flow on the host.  Swapped spans carry the
// maximal source side of their segment (supergraph.py:201-206), also a
// minimum cut, so the cost equals the flow there as well.  One CTA per
// (composite, pixel chunk); planes row-major int32 as staged
// (src | snk | nbr(4n) per composite at off).
struct CompV {
    int64_t off, out_off;
    int32_t W, H;
};
__global__ void __launch_bounds__(NT) k_comp_verify(const int32_t *__restrict__ in, int64_t total_px,
                                                    const CompV *__restrict__ cv, const uint8_t *__restrict__ out,
                                                    int32_t ncomp, int chunks, unsigned long long *acc) {
    __shared__ int64_t red[NT / 32];
    for (int64_t blk = blockIdx.x; blk < int64_t(ncomp) * chunks; blk += gridDim.x) {
        const int c = int(blk / chunks);
        const CompV v = cv[c];
        const int64_t n = int64_t(v.W) * v.H, per = (n + chunks - 1) / chunks;
        const int64_t lo = (blk % chunks) * per, hi = min(n, lo + per);
        const int32_t *src = in + v.off, *snk = in + total_px + v.off, *nb = in + 2 * total_px + 4 * v.off;
        const uint8_t *l = out + v.out_off;
        int64_t cost = 0;
        for (int64_t q = lo + threadIdx.x; q < hi; q += NT) {
            if (!l[q]) {
                cost += src[q];
                continue;
            }
            const int32_t x = int32_t(q % v.W), y = int32_t(q / v.W);
            cost += snk[q];
            if (x > 0 && !l[q - 1]) cost += nb[q];
            if (x + 1 < v.W && !l[q + 1]) cost += nb[n + q];
            if (y > 0 && !l[q - v.W]) cost += nb[2 * n + q];
            if (y + 1 < v.H && !l[q + v.W]) cost += nb[3 * n + q];
        }
        cost = block_sum64(cost, red);
        if (threadIdx.x == 0 && cost) atomicAdd(acc + c, (unsigned long long)cost);
    }
}


__global__ void k_verify_check(Ctx c, int64_t nplanes, const unsigned long long *acc) {
    for (int64_t plane = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; plane < nplanes;
         plane += int64_t(gridDim.x) * blockDim.x)
        if (int64_t(acc[plane]) != c.flows[plane]) atomicExch(c.err, 5);
}

// One CTA: advance every grid with a next lambda (cur_lam, live, embedded
// sink-capacity sum) and tell the step loop whether another step runs.
__global__ void __launch_bounds__(1024) k_advance_grids(Ctx c, SeedArgs a, const int64_t *slope_sum,
                                                        int32_t ngrids, cudaGraphConditionalHandle cond,
                                                        int has_cond) {
    int any = 0;
    for (int g = threadIdx.x; g < ngrids && a.nprob > 0; g += blockDim.x) {
        if (c.rolling) {   // only the grids that just finished; the loop runs on while any grid is live
            const int due = c.fin[g];
            c.fin[g] = 0;
            if (!due) {
                any |= c.live[g];
                continue;
            }
        }
        const GridDesc &gd = c.grids[g];
        const int cur = c.cur_lam[g];
        if (cur + 1 >= gd.lam_end) continue;
        if (c.swapflag[gd.prob]) c.snk_sum[g] += (a.lambdas[cur + 1] - a.lambdas[cur]) * slope_sum[gd.prob];
        c.cur_lam[g] = cur + 1;
        c.live[g] = 1;
        if (c.labok) c.labok[g] = !c.swapflag[gd.prob];   // lab holds this lambda's source side
        // unswapped: lambda_{i+1} only lowers sink residuals, the exact
        // heights of lambda_i stay a valid labelling -- skip one relabel
        if (c.keeph && !c.swapflag[gd.prob]) c.keeph[g] = 1;
        any = 1;
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) {
        c.ctl->cycle = 0;   // the non-convergence guard counts cycles per step
        c.ctl->steps++;
        c.ctl->more = any;
        if (has_cond) cudaGraphSetConditional(cond, any ? 1u : 0u);
    }
}

}  // namespace pmf
