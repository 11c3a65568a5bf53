// async.cuh -- one persistent kernel solves a whole seed batch.
//
// Every grid (a warm-start chain of lambda-graphs, or one cold lambda-graph)
// walks its own phase machine
//
//   BINIT -> BFS -> SEED -+-> PUSH -+-> BINIT ...           (budget spent: relabel cycle)
//                         |         +-> LINIT               (drained: speculative closure)
//                         +-> LINIT -> LAB -+-> EMIT -+-> SEED (next lambda, unswapped) / BFS (swapped)
//                                           |         +-> done
//                                           +-> BINIT       (speculative closure spoiled)
//
// and the tiles of all grids share one work queue (engine.cuh q_*): a CTA
// pops a tile, runs the body of its grid's current phase, requests the
// neighbours it touched, and the CTA that retires the last tile of a grid's
// phase performs that grid's transition (decides the next phase, enqueues
// its tiles).  No grid ever waits for another one at a phase boundary, so
// the latency-bound tails of one grid overlap the dense work of the others.
//
// Phase bodies (one CTA of 1024 threads, one 32x32 tile):
//   BINIT  h = 1 on sink-residual pixels, HINF elsewhere; flag BFS seeds   (k_gr_init)
//   BFS    exact distance to the sink, tile-local fixpoint                 (bfs_sink_tile)
//   SEED   count active pixels (w > 0, h < HINF); flag active tiles       (k_seed_push)
//   PUSH   discharge under a per-grid pop budget                           (push_tile)
//   LINIT  lab = (w > 0); flag label seeds                                 (k_lab_seed)
//   LAB    residual closure of the excess pixels                           (bfs_src_tile)
//   EMIT   label bytes, unused sink residual, warm-start advance of w      (k_emit, k_advance_tiles)
// The reference semantics of each body are documented at the kernels named.
#pragma once
#include "kernels.cuh"
#include "tile.cuh"

namespace pmf {

enum { PH_BINIT = 0, PH_BFS, PH_SEED, PH_PUSH, PH_LINIT, PH_LAB, PH_EMIT, PH_DONE };
// scan phases (BINIT, SEED, LINIT, EMIT) run as tasks of SCAN_GROUP
// consecutive tiles, queued by their first tile
constexpr int SCAN_GROUP = 16;
__host__ __device__ constexpr bool scan_phase(int ph) {
    return ph == PH_BINIT || ph == PH_SEED || ph == PH_LINIT || ph == PH_EMIT;
}
// extra pass counters (Ctx::stat) of the scan phases
enum { ST_BINIT = 9, ST_SEED = 10, ST_LINIT = 11, ST_EMIT = 12, ST_LAMS = 13, ST_ASYNC_NS = 14,
       ST_SPEC = 32, ST_SPOILED = 33,    // speculative label closures tried / spoiled
       ST_YIELDED = 37 };                // CTAs that left an idle tail early
// CTA-busy nanoseconds per phase kind (ST_BUSY + PH_*), then queue wait,
// hand-off (requests + retire) and grid transitions
constexpr int ST_BUSY = 16;
enum { BUSY_WAIT = 8, BUSY_FOLLOW = 9, BUSY_TRANS = 10, BUSY_N = 11 };

struct GridRun {
    int32_t phase;
    int32_t pops;      // discharge tile passes in the current PUSH phase
    int32_t budget;    // ... and their cap
    int32_t act;       // active pixels found by the current SEED phase
    int32_t cut;       // the current PUSH phase hit its budget
    int32_t cycles;    // relabel cycles of the current lambda
    int32_t spec;      // the current label closure is speculative (after a drained discharge)
    int32_t spoiled;   // ... and reached a sink-residual pixel: not done yet
    int32_t labok;     // lab holds the previous lambda's source side (nested seeding)
    int32_t pad;
    int64_t drain;     // unused sink residual (EMIT)
};

struct AsyncArgs {
    SeedArgs sa;
    const int64_t *slope_sum;
    GridRun *gr;
    uint8_t *tflag;    // per tile: listed for the next flagged phase
    int iters, relabel_every;
    unsigned budget_factor;
    int32_t budget_add;    // discharge pop budget: factor x seeded tiles + this
    int32_t max_cycles;
    int32_t cont;      // continuation hand-off between neighbouring tiles
    int32_t prefetch;  // take the next ticket while the queue is deep
    int32_t spec;      // a drained discharge goes straight to a speculative label closure
    int32_t keep_h;    // unswapped grids enter the next lambda with their current heights
    // CTAs with blockIdx >= yield_keep leave the kernel after yield_ns of an
    // empty queue (no ticket held), so a concurrent run gets their SM slots
    // in this run's latency-bound tail (0: never)
    unsigned long long yield_ns;
    int32_t yield_keep;
    unsigned long long *plog;   // diagnostics (nullable): per grid PLOG entries (phase << 56 | globaltimer)
};
constexpr int PLOG = 512;

// A grid reports its sink side: a swapped seed-batch grid, or a composite
// grid whose columns are all swapped (the asynchronous solver runs only
// composites whose every grid is uniform: one grid per segment span, or no
// swapped column at all).
__device__ __forceinline__ bool async_swapped(const Ctx &c, const GridDesc &gd) {
    return gd.kind == 1 ? c.colswap[gd.colswap_off] != 0 : grid_swapped(c, gd);
}

// ---- scan phases: one task = up to SCAN_GROUP consecutive tiles of a grid,
// all processed at once (SCAN_GROUP pixels per thread, loads issued
// together), with per-tile flags / counts gathered in shared memory.
struct ScanShared {
    int any[SCAN_GROUP];     // tile has a flagged pixel / active-pixel count
    int sides[SCAN_GROUP];   // border sides of flagged pixels
};
__shared__ ScanShared s_scan;

__device__ __forceinline__ void scan_reset() {
    if (threadIdx.x < SCAN_GROUP) s_scan.any[threadIdx.x] = 0, s_scan.sides[threadIdx.x] = 0;
    __syncthreads();
}

// thread k < ntl: flag tile t0 + k for the next flagged phase when it holds a
// flagged pixel, plus each neighbour facing a flagged border pixel (a seed
// never changes, so the tile alone would never hand it across the border;
// halo_seed_mask() of the worklist kernels)
// (bit 4 of sides, when `need_open` is set: the tile also has an unflagged
// pixel -- a tile whose every pixel is flagged is not listed itself, only
// the neighbours facing its border)
__device__ __forceinline__ void scan_flag(const Ctx &c, const AsyncArgs &A, int32_t t0, int ntl,
                                          bool need_open = false) {
    __syncthreads();
    const int k = threadIdx.x;
    if (k < ntl && s_scan.any[k]) {
        const int32_t t = t0 + k;
        if (!need_open || (s_scan.sides[k] & 16)) A.tflag[t] = 1;
        for (int s = 0; s < 4; s++)
            if ((s_scan.sides[k] >> s) & 1) {
                const int32_t nb = tile_nb(c, t, s);
                if (nb >= 0) A.tflag[nb] = 1;
            }
    }
}

// per-pixel flag contribution of pixel i of tile k (warp-aggregated)
__device__ __forceinline__ void scan_mark(int k, int flagged) {
    const int i = threadIdx.x;
    const unsigned b = __ballot_sync(0xffffffffu, flagged);
    if (!b) return;
    const int sides = flagged ? border_sides(i & 31, i >> 5) : 0;
    const int orr = __reduce_or_sync(0xffffffffu, sides);
    if ((i & 31) == 0) {
        atomicOr(&s_scan.any[k], 1);
        if (orr) atomicOr(&s_scan.sides[k], orr);
    }
}

// BINIT (k_gr_init): h = 1 on sink-residual pixels, HINF elsewhere
__device__ __forceinline__ void binit_group(const Ctx &c, const AsyncArgs &A, int32_t t0, int ntl) {
    const int i = threadIdx.x;
    scan_reset();
    int32_t wv[SCAN_GROUP];
#pragma unroll
    for (int k = 0; k < SCAN_GROUP; k++) wv[k] = k < ntl ? __ldcg(c.w + int64_t(t0 + k) * TPIX + i) : 0;
#pragma unroll
    for (int k = 0; k < SCAN_GROUP; k++)
        if (k < ntl) {
            c.h[int64_t(t0 + k) * TPIX + i] = wv[k] < 0 ? 1 : HINF;
            scan_mark(k, wv[k] < 0);
        }
    scan_flag(c, A, t0, ntl);
}

// SEED (k_seed_push): count active pixels (w > 0, h < HINF) per tile
__device__ __forceinline__ void seed_group(const Ctx &c, const AsyncArgs &A, int32_t t0, int ntl, int32_t g) {
    const int i = threadIdx.x;
    scan_reset();
    int a[SCAN_GROUP];
#pragma unroll
    for (int k = 0; k < SCAN_GROUP; k++) {
        const int64_t p = int64_t(t0 + k) * TPIX + i;
        a[k] = k < ntl && __ldcg(c.w + p) > 0 && __ldcg(c.h + p) < HINF;
    }
#pragma unroll
    for (int k = 0; k < SCAN_GROUP; k++) {
        const int v = __reduce_add_sync(0xffffffffu, a[k]);
        if ((i & 31) == 0 && v) atomicAdd(&s_scan.any[k], v);
    }
    __syncthreads();
    if (i < ntl && s_scan.any[i]) {
        atomicAdd(&A.gr[g].act, s_scan.any[i]);
        A.tflag[t0 + i] = 1;
        if (c.tfresh) c.tfresh[t0 + i] = 1;   // its heights are this relabel's exact distances
    }
}

// LINIT (k_lab_seed): lab = (w > 0), label BFS seeds (swapped grids report
// the sink side and run no label BFS: nothing to flag)
// Past the first lambda of a chain the previous lambda's source side also
// seeds the closure: minimal source sides are nested along a monotone
// schedule (parametric.py:191-201), so S(lambda_i) is inside
// S(lambda_{i+1}) and adding it changes nothing but the distance the
// closure has to travel; tiles already fully inside are not relaxed.
__device__ __forceinline__ void linit_group(const Ctx &c, const AsyncArgs &A, int32_t t0, int ntl, int32_t g,
                                            bool swapped) {
    const int i = threadIdx.x;
    const bool nested = __ldcg(c.cur_lam + g) > c.grids[g].lam && __ldcg(&A.gr[g].labok);
    scan_reset();
    int v[SCAN_GROUP];
#pragma unroll
    for (int k = 0; k < SCAN_GROUP; k++) {
        const int64_t p = int64_t(t0 + k) * TPIX + i;
        v[k] = k < ntl && (__ldcg(c.w + p) > 0 || (nested && __ldcg(c.lab + p)));
    }
#pragma unroll
    for (int k = 0; k < SCAN_GROUP; k++)
        if (k < ntl) {
            c.lab[int64_t(t0 + k) * TPIX + i] = uint8_t(v[k]);
            if (!swapped) {
                scan_mark(k, v[k]);
                if (__any_sync(0xffffffffu, !v[k]) && (i & 31) == 0) atomicOr(&s_scan.sides[k], 16);
            }
        }
    if (!swapped) scan_flag(c, A, t0, ntl, true);
}

// EMIT (k_emit + k_advance_tiles): label bytes (swapped grids: sink side
// {h < HINF} of the final exact relabel; else the source-side closure),
// unused sink residual, and -- when the chain has a next lambda -- the
// warm-start advance of w followed by that lambda's BINIT
__device__ __forceinline__ void emit_group(const Ctx &c, const AsyncArgs &A, int32_t t0, int ntl, int32_t g) {
    __shared__ int64_t red[NTT / 32];
    const SeedArgs &a = A.sa;
    const GridDesc &gd = c.grids[g];
    const int i = threadIdx.x;
    const int cur = __ldcg(c.cur_lam + g);   // advanced by other CTAs' transitions
    const bool next = cur + 1 < gd.lam_end;
    const bool swapped = async_swapped(c, gd);
    const bool comp = gd.kind == 1;
    const int64_t n = int64_t(gd.W) * gd.H;
    const int64_t dl = next ? a.lambdas[cur + 1] - a.lambdas[cur] : 0;
    const int sign = !comp && c.swapflag[gd.prob] ? -1 : 1;
    // composites (no next lambda): the span's columns of the composite's
    // output, swapped columns as ~sink side (supergraph.py:201-206, k_emit)
    uint8_t *out = comp ? c.out + gd.out_off + gd.xoff : c.out + (int64_t(gd.prob) * c.nlam + cur) * n;
    const int64_t pitch = comp ? gd.pitch : gd.W;
    const uint8_t *mask = next ? a.mask + int64_t(gd.prob) * n : nullptr;
    const int32_t *slope = next ? a.slope + a.plane_off[gd.prob] : nullptr;
    // unswapped grids may keep their heights into the next lambda (knob
    // adv_keep_h, see the EMIT transition); swapped ones get that lambda's
    // BINIT fused in here
    const bool reinit = next && (swapped || !A.keep_h);
    // kept heights: the next lambda's SEED, fused (active = w > 0, h < HINF)
    const bool seed = next && !reinit;
    if (reinit || seed) scan_reset();
    int64_t drain = 0;
    const int32_t l0 = int32_t(t0 - gd.tile_base);
#pragma unroll 2
    for (int k = 0; k < SCAN_GROUP; k++) {
        if (k >= ntl) break;
        const int32_t l = l0 + k;
        const int x = (l % gd.ntx) * TW + (i & 31), y = (l / gd.ntx) * TH + (i >> 5);
        const int64_t p = int64_t(t0 + k) * TPIX + i;
        int32_t wv = __ldcg(c.w + p);
        if (x < gd.W && y < gd.H) {
            if (wv < 0) drain -= wv;
            const int64_t q = int64_t(y) * gd.W + x;
            out[int64_t(y) * pitch + x] =
                swapped ? uint8_t((__ldcg(c.h + p) < HINF) != comp) : __ldcg(c.lab + p);
            if (next && mask[q] != 1) {   // fg seed: CAP_MAX either way
                wv += int32_t(sign * dl * int64_t(slope[q]));
                c.w[p] = wv;
            }
        }
        if (reinit) {   // the next lambda's BINIT, fused
            c.h[p] = wv < 0 ? 1 : HINF;
            scan_mark(k, wv < 0);
        }
        if (seed) {
            const int act = __reduce_add_sync(0xffffffffu, int(wv > 0 && __ldcg(c.h + p) < HINF));
            if ((i & 31) == 0 && act) atomicAdd(&s_scan.any[k], act);
        }
    }
    const int64_t s = block_sum64(drain, red);
    if (i == 0 && s) atomicAdd((unsigned long long *)&A.gr[g].drain, (unsigned long long)s);
    if (reinit) scan_flag(c, A, t0, ntl);
    if (seed) {
        __syncthreads();
        if (i < ntl && s_scan.any[i]) {
            atomicAdd(&A.gr[g].act, s_scan.any[i]);
            A.tflag[t0 + i] = 1;
        }
    }
}

// Whole CTA, after the last tile of grid g's phase `ph` retired (nothing of
// g is queued or running): pick the next phase and enqueue its tiles.  A
// flagged phase with no flagged tile is empty and falls through at once.
// The phase (and a discharge's budget) is published before any of its tiles
// is queued; poppers read it after their pop (fences on both sides).
__device__ void grid_transition(const Ctx &c, const AsyncArgs &A, int32_t g, int ph) {
    __shared__ int s_next, s_cnt;
    const GridDesc &gd = c.grids[g];
    GridRun &R = A.gr[g];
    const int64_t t0 = gd.tile_base;
    const int32_t nt = gd.ntx * gd.nty;
    for (;;) {
        if (threadIdx.x == 0) {
            int next = PH_DONE;
            const bool swapped = async_swapped(c, gd);
            switch (ph) {
            case PH_BINIT: next = PH_BFS; break;
            case PH_BFS:
                R.act = 0;
                next = PH_SEED;
                break;
            case PH_SEED:
                if (__ldcg(&R.act) == 0) {
                    next = PH_LINIT;
                } else if ((R.cycles = __ldcg(&R.cycles) + 1) > A.max_cycles) {
                    c.ctl->noconv = 1;
                } else {
                    next = PH_PUSH;
                    R.pops = 0;
                    R.cut = 0;
                    atomicAdd(&c.ctl->cycles_total, 1);
                }
                break;
            case PH_PUSH:
                // A drained discharge is not a certificate by itself (the
                // lock-free rule h(p) > h(q) against a halo height read at
                // pass start can push into a pixel frozen meanwhile, giving
                // it a residual path out).  The label closure of the excess
                // pixels IS one (it is source_side, solvers.py:144-158): run
                // it speculatively -- if it never reaches a sink-residual
                // pixel the preflow is maximum and the labels are final;
                // otherwise relabel and discharge on.  Swapped grids need
                // the sink side of an exact relabel.
                if (A.spec && !__ldcg(&R.cut) && !swapped) {
                    R.spec = 1;
                    R.spoiled = 0;
                    atomicAdd(&c.stat[ST_SPEC], 1ull);
                    next = PH_LINIT;
                } else {
                    next = PH_BINIT;
                }
                break;
            case PH_LINIT:
                next = swapped ? PH_EMIT : PH_LAB;
                R.act = 0;   // EMIT may seed the next lambda
                break;
            case PH_LAB:
                if (R.spec && __ldcg(&R.spoiled)) {
                    atomicAdd(&c.stat[ST_SPOILED], 1ull);
                    R.labok = 0;   // lab now holds a spoiled closure
                    next = PH_BINIT;
                } else {
                    next = PH_EMIT;
                    R.act = 0;   // EMIT may seed the next lambda
                }
                R.spec = 0;
                R.spoiled = 0;
                break;
            case PH_EMIT: {
                const int cur = __ldcg(c.cur_lam + g);
                const int64_t snk = int64_t(__ldcg((const unsigned long long *)(c.snk_sum + g)));
                c.flows[gd.kind == 1 ? int64_t(g) : int64_t(gd.prob) * c.nlam + cur] =
                    snk - int64_t(__ldcg((const unsigned long long *)&R.drain));
                R.drain = 0;
                atomicAdd(&c.stat[ST_LAMS], 1ull);
                if (cur + 1 < gd.lam_end) {
                    if (swapped)
                        c.snk_sum[g] = snk + (A.sa.lambdas[cur + 1] - A.sa.lambdas[cur]) * A.slope_sum[gd.prob];
                    c.cur_lam[g] = cur + 1;
                    R.cycles = 0;
                    R.labok = 1;     // lab holds this lambda's source side
                    if (swapped || !A.keep_h) {
                        next = PH_BFS;   // EMIT ran the next lambda's BINIT
                    } else {
                        // lambda_{i+1} only lowers sink residuals of an
                        // unswapped grid (w += dl * slope): no residual path
                        // appears, so lambda_i's exact distances stay a valid
                        // labelling (lower bounds, HINF exact): seed the
                        // discharge straight away (EMIT ran that
                        // lambda's seeding)
                        if (__ldcg(&R.act) == 0) {
                            // kept heights may carry HINF marks of a
                            // speculative finish, which certify nothing: the
                            // closure decides (speculative, falls back)
                            next = PH_LINIT;
                            R.spec = 1;
                            R.spoiled = 0;
                            atomicAdd(&c.stat[ST_SPEC], 1ull);
                        } else {
                            next = PH_PUSH;
                            R.cycles = 1;
                            R.pops = 0;
                            R.cut = 0;
                            atomicAdd(&c.ctl->cycles_total, 1);
                        }
                    }
                }
                break;
            }
            default: break;
            }
            s_next = next;
            s_cnt = 0;
        }
        __syncthreads();
        const int next = s_next;
        if (next == PH_DONE) {
            if (threadIdx.x == 0) {
                R.phase = PH_DONE;
                if (A.plog) {
                    unsigned long long *lg = A.plog + int64_t(g) * PLOG;
                    const unsigned long long k = lg[0];
                    if (k + 1 < PLOG) {
                        lg[k + 1] = (unsigned long long)PH_DONE << 56 | (gtimer() & ((1ull << 56) - 1));
                        lg[0] = k + 1;
                    }
                }
                qfence();
            }
            __syncthreads();
            return;
        }
        const bool all = scan_phase(next);
        // count the tasks the phase will run
        int mine = 0;
        for (int32_t j = threadIdx.x; j < nt; j += blockDim.x)
            mine += all ? j % SCAN_GROUP == 0 : __ldcg(&A.tflag[t0 + j]) != 0;
        if (mine) atomicAdd(&s_cnt, mine);
        __syncthreads();
        const int cnt = s_cnt;
        if (cnt == 0) {   // empty flagged phase: go on to the one after it
            ph = next;
            __syncthreads();
            continue;
        }
        if (threadIdx.x == 0) {
            if (next == PH_PUSH)   // pop budget: factor x seeded tiles (k_cycle_ctl)
                R.budget = A.budget_factor ? int32_t(A.budget_factor) * cnt + A.budget_add : 0x7fffffff;
            R.phase = next;
            if (A.plog) {   // diagnostics: phase timeline of the grid
                unsigned long long *lg = A.plog + int64_t(g) * PLOG;
                const unsigned long long k = lg[0];
                if (k + 1 < PLOG) {
                    lg[k + 1] = (unsigned long long)next << 56 | (gtimer() & ((1ull << 56) - 1));
                    lg[0] = k + 1;
                }
            }
            // hold the phase open while its tiles are being queued: a tile
            // popped and retired meanwhile must not see the count reach zero
            atomicAdd(&c.gpend[g], 1);
            qfence();
        }
        __syncthreads();
        qfence();
        for (int32_t j = threadIdx.x; j < nt; j += blockDim.x) {
            const int32_t t = int32_t(t0 + j);
            bool go = all && j % SCAN_GROUP == 0;
            if (!all && __ldcg(&A.tflag[t])) {
                A.tflag[t] = 0;
                go = true;
            }
            if (go) q_request(c, t);
        }
        qfence();
        __syncthreads();
        if (threadIdx.x == 0) s_next = atomicSub(&c.gpend[g], 1) == 1;
        __syncthreads();
        if (!s_next) return;
        ph = next;   // every tile of the new phase already finished: next transition
        __syncthreads();
    }
}

// Retire (or requeue) the running tile t.  Returns 0: requeued, 1: retired,
// 2: retired as the last queued/running tile of its grid's phase.  The
// global pending count is left to the caller (it drops after a transition
// has queued the next phase, so it never touches zero in between).
__device__ __forceinline__ int aq_finish(const Ctx &c, int32_t t, bool again) {
    for (;;) {
        if (again) {
            atomicExch(&c.qstate[t], Q_QUEUED);
            q_push(c, t);
            return 0;
        }
        if (atomicCAS(&c.qstate[t], Q_RUNNING, Q_IDLE) == Q_RUNNING)
            return atomicSub(&c.gpend[c.tile_grid[t]], 1) == 1 ? 2 : 1;
        again = true;   // dirtied while running
    }
}

template <class E>
__global__ void __launch_bounds__(NTT, 2) k_async(Ctx c, AsyncArgs A) {
    __shared__ int32_t s_t, s_cont;
    __shared__ int s_fin, s_ok;
    const int i = threadIdx.x;
    push_prepare();
    if (i == 0) {
        s_cont = -1;
        atomicMin(&c.ctl->t0, gtimer());
    }
    // ticket taken ahead while the queue is deep (its tile is then already
    // queued, so holding it while this CTA works delays nobody)
    unsigned pre = ~0u;
    for (;;) {
        if (i == 0) {
            const unsigned long long tw = gtimer();
            int32_t t = s_cont;
            s_cont = -1;
            if (t < 0 && pre == ~0u && A.yield_ns && int(blockIdx.x) >= A.yield_keep) {
                // idle without a ticket: wait for queued work without taking
                // one; after yield_ns leave the SM to a concurrent run
                const unsigned long long t_idle = gtimer();
                for (;;) {
                    if (ld_volatile(&c.qctr[QC_TAIL]) > ld_volatile(&c.qctr[QC_HEAD])) break;
                    if (ld_volatile(&c.qctr[QC_PENDING]) == 0) break;
                    if (gtimer() - t_idle > A.yield_ns) {
                        t = -2;
                        break;
                    }
                    __nanosleep(256);
                }
            }
            if (t == -2) {
                atomicAdd(&c.stat[ST_YIELDED], 1ull);
            } else if (t < 0) {
                t = pre != ~0u ? q_wait(c, pre) : q_next(c);
                pre = ~0u;
            }
            if (t >= 0 && A.prefetch && pre == ~0u) {   // at most one ticket held
                const unsigned hd = ld_volatile(&c.qctr[QC_HEAD]), tl = ld_volatile(&c.qctr[QC_TAIL]);
                if (tl > hd && tl - hd > 2u * gridDim.x) pre = atomicAdd(&c.qctr[QC_HEAD], 1u);
            }
            qfence();
            s_t = t;
            atomicAdd(&c.stat[ST_BUSY + BUSY_WAIT], gtimer() - tw);
        }
        __syncthreads();
        const int32_t t = s_t;
        if (t < 0) break;
        qfence();   // popper side: state write < data reads
        const unsigned long long tb = i == 0 ? gtimer() : 0ull;
        const int32_t g = __ldg(c.tile_grid + t);
        const int ph = __ldcg(&A.gr[g].phase);
        TileResult r{0, 0};
        int stat = -1, npass = 1;
        if (scan_phase(ph)) {
            const GridDesc &gd = c.grids[g];
            const int ntl = int(min(int64_t(SCAN_GROUP), gd.tile_base + int64_t(gd.ntx) * gd.nty - t));
            switch (ph) {
            case PH_BINIT: binit_group(c, A, t, ntl); break;
            case PH_SEED: seed_group(c, A, t, ntl, g); break;
            case PH_LINIT: linit_group(c, A, t, ntl, g, async_swapped(c, gd)); break;
            default: emit_group(c, A, t, ntl, g); break;
            }
            stat = ph == PH_BINIT ? ST_BINIT : ph == PH_SEED ? ST_SEED : ph == PH_LINIT ? ST_LINIT : ST_EMIT;
            npass = ntl;
        } else if (ph == PH_BFS) {
            r = bfs_sink_tile<E>(c, t);
            stat = ST_BFS;
        } else if (ph == PH_PUSH) {
            if (i == 0) {
                // budget spent: the tile waits for the relabel that follows
                s_ok = atomicAdd(&A.gr[g].pops, 1) < __ldcg(&A.gr[g].budget);
                if (!s_ok) A.gr[g].cut = 1;
            }
            __syncthreads();
            if (s_ok) {
                r = push_tile<E>(c, t, A.iters, A.relabel_every);
                stat = ST_PUSH;
            }
        } else if (ph == PH_LAB) {
            // one CTA-uniform decision (the flag changes under our feet)
            if (i == 0) s_ok = !__ldcg(&A.gr[g].spoiled);
            __syncthreads();
            if (s_ok)   // else: a spoiled speculative closure has nothing left to learn
                r = bfs_src_tile<E>(c, t, __ldcg(&A.gr[g].spec) ? &A.gr[g].spoiled : nullptr);
            stat = ST_LAB;
        }
        const unsigned long long tf = i == 0 ? gtimer() : 0ull;
        if (i == 0) atomicAdd(&c.stat[ST_BUSY + ph], tf - tb);
        qfence();   // requester side: data writes < queue-state reads
        __syncthreads();
        if (i < 32) {
            // neighbours this pass touched (same phase); the lowest one is
            // taken over directly when the tile itself is done
            const unsigned flags = unsigned(r.out) & 15u;
            const int want = (A.cont && !r.again && flags) ? __ffs(flags) : 0;
            // the neighbours are counted pending before this tile retires
            // (so its grid's count cannot touch zero meanwhile); their ring
            // insertion overlaps the retirement
            int32_t nb = -1;
            bool push = false;
            if (i >= 1 && i <= 4 && ((flags >> (i - 1)) & 1)) {
                nb = tile_nb(c, t, i - 1);
                if (nb >= 0) {
                    if (i == want && q_claim(c, nb)) s_cont = nb;
                    else push = q_mark(c, nb);
                }
                qfence();
            }
            __syncwarp();
            if (push) q_push(c, nb);
            if (i == 0) {
                s_fin = aq_finish(c, t, r.again != 0);
                if (stat >= 0) atomicAdd(&c.stat[stat], (unsigned long long)npass);
            }
        }
        __syncthreads();
        const int fin = s_fin;
        const unsigned long long tt = i == 0 ? gtimer() : 0ull;
        if (i == 0) atomicAdd(&c.stat[ST_BUSY + BUSY_FOLLOW], tt - tf);
        if (fin == 2) {
            qfence();
            grid_transition(c, A, g, ph);
            if (i == 0) atomicAdd(&c.stat[ST_BUSY + BUSY_TRANS], gtimer() - tt);
        }
        if (i == 0 && fin) {
            qfence();
            atomicSub(&c.qctr[QC_PENDING], 1u);
        }
    }
    if (i == 0) {
        atomicMax(&c.ctl->t1, gtimer());
        qfence();
        if (atomicAdd(&c.ctl->done, 1u) == gridDim.x - 1) {
            qfence();
            const unsigned long long t0 = *(volatile unsigned long long *)&c.ctl->t0;
            const unsigned long long t1 = *(volatile unsigned long long *)&c.ctl->t1;
            c.stat[ST_ASYNC_NS] = t1 > t0 ? t1 - t0 : 0ull;
        }
    }
}

// Start of an asynchronous batch (after k_phase_begin reset the queue):
// every grid in BINIT with all its tiles queued.
__global__ void k_async_begin(Ctx c, AsyncArgs A, int32_t ngrids) {
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t g = tid; g < ngrids; g += stride) {
        GridRun &R = A.gr[g];
        R.phase = PH_BINIT;
        R.pops = R.budget = R.act = R.cut = R.cycles = 0;
        R.spec = R.spoiled = R.labok = R.pad = 0;
        R.drain = 0;
    }
    for (int64_t t = tid; t < c.ntiles; t += stride) A.tflag[t] = 0;
}

__global__ void k_async_queue_all(Ctx c) {
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t t = tid; t < c.ntiles; t += stride) {
        const GridDesc &gd = c.grids[c.tile_grid[t]];
        if ((t - gd.tile_base) % SCAN_GROUP == 0) q_request(c, int32_t(t));   // BINIT task leaders
    }
}

}  // namespace pmf
