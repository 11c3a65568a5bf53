// tile.cuh -- the per-tile kernels: push-relabel discharge and the two BFS
// sweeps, all built on one shared-memory primitive, tile_relax().
//
// One CTA of 1024 threads owns one 32x32 tile at a time, one pixel per
// thread (warp = row for row work, warp = column for column work).  The
// CTA walks the tiles of the current worklist (grid-stride) and appends to
// the next worklist the tiles that still / newly need work.
#pragma once
#include "engine.cuh"

namespace pmf {

constexpr int NTT = 1024;        // threads per tile CTA
constexpr int SP = TW + 1;       // padded shared-memory row stride (conflict-free columns)

// Bit d of a pull mask: this pixel may take the value of its d-neighbour
// (plus the step cost).  Halo values hv[side][j] stand for the neighbour
// tile's facing pixels (HINF where there is none).
//
// tile_relax: Bellman-Ford to the fixpoint of
//     d(p) = min(d(p), d(q) + cost)   for every pull arc p <- q
// computed as alternating row / column passes.  A pass is two segmented
// min-plus scans along warp shuffles -- rightward (value - cost*x carried
// through runs of consecutive pull-from-left arcs) and leftward -- so a
// straight run of any length settles in one pass and a path with k turns in
// about k passes.  The two scans are independent (a shortest path never
// reverses inside one line), so they run interleaved from the same input,
// and their segment bounds depend only on the masks: computed once per call
// with ballots, each scan step is a single shuffle.
// segment bounds of a line scan, packed: bits 0-4 first lane of my
// rightward segment, bits 5-9 last lane of my leftward segment
__device__ __forceinline__ unsigned line_seg(int m, int lane, int blo, int bhi) {
    const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || !(m & blo));
    const unsigned tails = __ballot_sync(0xffffffffu, lane == 31 || !(m & bhi));
    const unsigned lo = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
    const unsigned hi = __ffs(tails & (0xffffffffu << lane)) - 1;
    return lo | (hi << 5);
}

// one line, both directions: lo = pull from the lower index neighbour (bit
// blo; lane 0 from *halo_lo), hi = pull from the higher one (bit bhi; lane
// 31 from *halo_hi)
__device__ __forceinline__ int32_t line_relax(int32_t v, int m, int lane, unsigned seg, int blo, int bhi,
                                              const int32_t *halo_lo, const int32_t *halo_hi, int cost) {
    int32_t a = v, b = v;
    if (lane == 0 && (m & blo)) a = min(a, *halo_lo + cost);
    if (lane == 31 && (m & bhi)) b = min(b, *halo_hi + cost);
    const int lo = seg & 31, hi = (seg >> 5) & 31;
    int32_t ua = a - cost * lane, ub = b + cost * lane;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int32_t oa = __shfl_up_sync(0xffffffffu, ua, off);
        const int32_t ob = __shfl_down_sync(0xffffffffu, ub, off);
        if (lane - off >= lo) ua = min(ua, oa);
        if (lane + off <= hi) ub = min(ub, ob);
    }
    return min(min(ua + cost * lane, ub - cost * lane), HINF);
}

// d: [32][SP] values, mk: [32][32] pull masks, hv: halo values.  All 1024
// threads call it.  Runs to the fixpoint (bit 0 of the result set) or stops
// after max_sweeps sweeps (> 0; bit 0 clear if it had not converged) -- a
// capped relax only gives upper bounds.  Bits 1.. hold the sweeps run.
//
// A line pass leaves its line at the line's own fixpoint (the halo values
// are constant), so after the first sweep a row needs its pass again only
// if the column pass before it changed one of its pixels, and a column only
// if the row pass changed one of its pixels: the passes publish their
// change ballots (s_rchg[row] / s_cchg[column]) and clean lines skip their
// scans.  The relax ends when a column pass changes nothing.
__shared__ unsigned s_rchg[TH], s_cchg[TW];
template <bool kSkip = true>
__device__ int tile_relax(int32_t *d, const uint8_t *mk, const int32_t (*hv)[TW], int cost,
                          int max_sweeps = 0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // rows: warp = y, lane = x; bits L (1) / R (2).  columns: warp = x,
    // lane = y; bits U (4) / D (8).  Masks and segment bounds of both
    // passes packed in one register (bits 0-3 row mask, 4-7 column mask,
    // 8-17 row segments, 18-27 column segments).
    unsigned pk;
    {
        const int mr = mk[warp * TW + lane], mc = mk[lane * TW + warp];
        pk = unsigned(mr) | (unsigned(mc) << 4) | (line_seg(mr, lane, 1, 2) << 8) | (line_seg(mc, lane, 4, 8) << 18);
    }
    int sweeps = 0;
    if constexpr (!kSkip) {
        for (;;) {
            int changed = 0;
            {
                const int32_t v0 = d[warp * SP + lane];
                const int32_t v = line_relax(v0, pk & 15, lane, pk >> 8, 1, 2, &hv[DL][warp], &hv[DR][warp], cost);
                if (v != v0) { d[warp * SP + lane] = v; changed = 1; }
            }
            __syncthreads();
            {
                const int32_t v0 = d[lane * SP + warp];
                const int32_t v = line_relax(v0, (pk >> 4) & 15, lane, pk >> 18, 4, 8, &hv[DU][warp],
                                             &hv[DD][warp], cost);
                if (v != v0) { d[lane * SP + warp] = v; changed = 1; }
            }
            sweeps++;
            if (!__syncthreads_or(changed)) return 1 | (sweeps << 1);
            if (max_sweeps && sweeps >= max_sweeps) return sweeps << 1;
        }
    } else {
        for (;;) {
            {
                unsigned chg = 0;
                if (sweeps == 0 || __any_sync(0xffffffffu, (s_cchg[lane] >> warp) & 1u)) {
                    const int32_t v0 = d[warp * SP + lane];
                    const int32_t v = line_relax(v0, pk & 15, lane, pk >> 8, 1, 2, &hv[DL][warp], &hv[DR][warp], cost);
                    if (v != v0) d[warp * SP + lane] = v;
                    chg = __ballot_sync(0xffffffffu, v != v0);
                }
                if (lane == 0) s_rchg[warp] = chg;
            }
            __syncthreads();
            unsigned chg = 0;
            if (sweeps == 0 || __any_sync(0xffffffffu, (s_rchg[lane] >> warp) & 1u)) {
                const int32_t v0 = d[lane * SP + warp];
                const int32_t v = line_relax(v0, (pk >> 4) & 15, lane, pk >> 18, 4, 8, &hv[DU][warp], &hv[DD][warp],
                                             cost);
                if (v != v0) d[lane * SP + warp] = v;
                chg = __ballot_sync(0xffffffffu, v != v0);
            }
            if (lane == 0) s_cchg[warp] = chg;
            sweeps++;
            // done when a column pass changes nothing: the rows are then at
            // their fixpoint too
            if (!__syncthreads_or(chg != 0)) return 1 | (sweeps << 1);
            if (max_sweeps && sweeps >= max_sweeps) return sweeps << 1;
        }
    }
}

// diagnostics: K_MULTI sweeps as trace entries of kind 4 + stat (start
// stamp, listed tiles; the span is filled in by the next entry)
__device__ __forceinline__ void trace_sweep(Ctl *ctl, int stat, int32_t n) {
    const int ix = ctl->ntrace;
    if (ix >= kTrace) return;
    const unsigned long long now = gtimer();
    ctl->trace_kind[ix] = 4 + stat;
    ctl->trace_t0[ix] = now;
    ctl->trace_ns[ix] = 0;
    ctl->trace_tiles[ix] = (unsigned long long)(uint32_t)n;
    if (ix > 0 && ctl->trace_kind[ix - 1] == 4 + stat) ctl->trace_ns[ix - 1] = now - ctl->trace_t0[ix - 1];
    ctl->ntrace = ix + 1;
}

struct TileResult {
    int again;   // the tile itself still has work
    int out;     // bit s: the neighbour on side s needs (re)processing
};

// Follow-up tiles of a processed tile into worklist k, one candidate per
// thread j = 0..4 (0: the tile itself, 1..4: the neighbour on side j - 1)
// so that the enqueue atomics overlap instead of running back to back.
__device__ __forceinline__ void enqueue_follow(const Ctx &c, int k, int32_t t, const TileResult &r, int j) {
    if (j == 0) {
        if (r.again) enqueue(c, k, t);
    } else if ((r.out >> (j - 1)) & 1) {
        const int32_t nb = tile_nb(c, t, j - 1);
        if (nb >= 0) enqueue(c, k, nb);
    }
}

// Per-launch bookkeeping shared by all CTAs of a tile kernel: device-clock
// span of the launch (earliest CTA start .. latest CTA end, %globaltimer) and,
// in graph-driven mode, the advance of the sweep index plus the decision
// whether the enclosing conditional while node runs another sweep.
struct LaunchCtl {
    int stat;                         // ST_PUSH / ST_BFS / ST_LAB
    cudaGraphConditionalHandle cond;  // loop condition to set (graph mode)
    int has_cond;
    int max_k;                        // stop the loop after this many sweeps (0 = no cap)
};

__device__ __forceinline__ void launch_enter(const Ctx &c) {
    if (threadIdx.x == 0) atomicMin(&c.ctl->t0, gtimer());
}

// Called by thread 0 of each of the `parts` participating CTAs when it
// leaves the kernel (sweep mode: only CTAs that received a tile take part,
// the rest exit without touching the control block).  k_next is the sweep
// index that follows (K_DEVICE mode) or -1.
__device__ __forceinline__ void launch_exit(const Ctx &c, const LaunchCtl &lc, int k_next,
                                            unsigned parts) {
    atomicMax(&c.ctl->t1, gtimer());
    __threadfence();
    if (atomicAdd(&c.ctl->done, 1u) != parts - 1) return;
    // last CTA of the launch
    __threadfence();
    Ctl *ctl = c.ctl;
    unsigned long long t0 = *(volatile unsigned long long *)&ctl->t0;
    unsigned long long t1 = *(volatile unsigned long long *)&ctl->t1;
    atomicAdd(&c.stat[ST_PUSH_NS + lc.stat], t1 > t0 ? t1 - t0 : 0ull);
    atomicAdd(&c.stat[ST_PUSH_L + lc.stat], 1ull);
    {   // launch trace (diagnostics): tiles = passes counted so far minus the previous entry
        int ix = ctl->ntrace;
        if (ix < kTrace) {
            unsigned long long tot = *(volatile unsigned long long *)&c.stat[lc.stat];
            unsigned long long prev = 0;
            for (int j = ix - 1; j >= 0; j--)
                if (ctl->trace_kind[j] == lc.stat) { prev = ctl->trace_tiles[j] >> 32; break; }
            ctl->trace_kind[ix] = lc.stat;
            ctl->trace_ns[ix] = t1 > t0 ? t1 - t0 : 0ull;
            ctl->trace_t0[ix] = t0;
            ctl->trace_tiles[ix] = (tot << 32) | ((tot - prev) & 0xffffffffull);
            ctl->ntrace = ix + 1;
        }
    }
    ctl->t0 = ~0ull;
    ctl->t1 = 0;
    ctl->done = 0;
    ctl->bar_count = 0;   // every CTA has passed its last grid barrier
    if (k_next >= 0) {
        int next = *(volatile int32_t *)&c.cnt[k_next % 3];
        ctl->k = k_next;
        if (lc.has_cond)
            cudaGraphSetConditional(lc.cond, (next > 0 && (lc.max_k == 0 || k_next < lc.max_k)) ? 1u : 0u);
    }
}

// Outer loop shared by the tile kernels.
//  * sweep mode (k >= 0, or K_DEVICE with k read from the control block):
//    walk worklist k once, list follow-up tiles in worklist k + 1;
//  * persistent mode (K_PERSISTENT): pop tiles from the device queue until
//    the phase drains (or its pop budget is spent); follow-up tiles are
//    queued and picked up by whichever CTA is free, with no kernel boundary.
// Persistent-queue hand-off of a processed tile, by the lanes of one warp:
// lanes 1..4 request the flagged neighbours concurrently, then lane 0
// retires or requeues the tile (after the requests, so the pending count
// never touches zero while follow-up work is being registered).
__device__ __forceinline__ void q_follow(const Ctx &c, int32_t t, const TileResult &r, int lane, int stat,
                                         int32_t *cont = nullptr) {
    // continuation candidate (cont != nullptr): the lowest flagged side,
    // when the tile itself is done
    const unsigned flags = unsigned(r.out) & 15u;
    const int want = (cont && !r.again && flags) ? __ffs(flags) : 0;
    // neighbours are counted pending before this tile retires; their ring
    // insertion overlaps the retirement
    int32_t nb = -1;
    bool push = false;
    if (lane >= 1 && lane <= 4 && ((flags >> (lane - 1)) & 1)) {
        nb = tile_nb(c, t, lane - 1);
        if (nb >= 0) {
            if (lane == want && q_claim(c, nb)) *cont = nb;
            else push = q_mark(c, nb);
        }
        qfence();
    }
    __syncwarp();
    if (push) q_push(c, nb);
    if (lane == 0) {
        q_finish(c, t, r.again != 0);
        atomicAdd(&c.stat[stat], 1ull);
    }
}

template <class Body>
__device__ __forceinline__ void tile_loop(const Ctx &c, int k, const LaunchCtl &lc, Body &&body) {
    __shared__ int32_t s_t, s_n;
    const int i = threadIdx.x;
    if (k == K_MULTI) {
        // every sweep of the phase in one cooperative launch: the same
        // worklist discipline as sweep mode, a grid barrier in place of the
        // kernel boundary
        launch_enter(c);
        if (i == 0) s_t = *(volatile int32_t *)&c.ctl->k;
        __syncthreads();
        int kk = s_t, sweeps = 0;
        for (;;) {
            if (i == 0) s_n = *(volatile int32_t *)&c.cnt[kk % 3];
            __syncthreads();
            const int32_t n = s_n;
            if (n == 0) break;
            const int32_t *lst = list_of(c, kk);
            if (blockIdx.x == 0 && i == 0) {
                c.cnt[(kk + 2) % 3] = 0;
                atomicAdd(&c.stat[lc.stat], (unsigned long long)n);
                trace_sweep(c.ctl, lc.stat, n);
            }
            for (int li = blockIdx.x; li < n; li += gridDim.x) {
                const int32_t t = __ldcg(lst + li);
                if (i == 0) inq_of(c, kk)[t] = 0;
                TileResult r = body(t);
                if (i < 5) enqueue_follow(c, kk + 1, t, r, i);
                __syncthreads();
            }
            grid_sync(c.ctl, sweeps);
            kk++;
            sweeps++;
        }
        if (i == 0) {
            if (blockIdx.x == 0) {
                c.ctl->k = kk;
                if (sweeps > 1) atomicAdd(&c.stat[ST_PUSH_L + lc.stat], (unsigned long long)(sweeps - 1));
            }
            launch_exit(c, lc, -1, gridDim.x);
        }
        return;
    }
    if (k != K_PERSISTENT) {
        if (i == 0) {
            if (k == K_DEVICE) k = *(volatile int32_t *)&c.ctl->k;
            s_t = k;
            s_n = *(volatile int32_t *)&c.cnt[k % 3];
        }
        __syncthreads();
        k = s_t;
        const int32_t n = s_n;
        // CTAs without a tile leave at once; the others (or block 0 when
        // the list is empty) do the launch bookkeeping
        const unsigned parts = unsigned(max(1, min(n, int32_t(gridDim.x))));
        if (blockIdx.x >= parts) return;
        launch_enter(c);
        const int32_t *lst = list_of(c, k);
        if (blockIdx.x == 0 && i == 0) {
            c.cnt[(k + 2) % 3] = 0;
            atomicAdd(&c.stat[lc.stat], (unsigned long long)n);
        }
        for (int li = blockIdx.x; li < n; li += gridDim.x) {
            const int32_t t = lst[li];
            if (i == 0) inq_of(c, k)[t] = 0;
            TileResult r = body(t);
            if (i < 5) enqueue_follow(c, k + 1, t, r, i);
            __syncthreads();
        }
        if (i == 0) launch_exit(c, lc, k + 1, parts);
        return;
    }
    launch_enter(c);
    // Hand-off ordering (store-buffering pattern): a requester writes tile
    // data, then reads the neighbour's queue state; a popper writes the
    // state, then reads the data.  Each side needs a gpu-scope SC fence
    // between its write and its read in every participating thread, i.e.
    // on both sides of the CTA barrier that separates the data threads from
    // thread 0.
    __shared__ int32_t s_cont;
    if (i == 0) s_cont = -1;
    for (;;) {
        if (i == 0) {
            int32_t t = s_cont;
            s_cont = -1;
            if (t < 0) t = q_next(c);
            qfence();
            s_t = t;
        }
        __syncthreads();
        const int32_t t = s_t;
        if (t < 0) break;
        qfence();                     // popper side: state write < data reads
        TileResult r = body(t);
        qfence();                     // requester side: data writes < ...
        __syncthreads();
        if (i < 32) q_follow(c, t, r, i, lc.stat, &s_cont);
    }
    if (i == 0) launch_exit(c, lc, -1, gridDim.x);
}

// ---------------------------------------------------------------------------
// Global relabel: exact distance to the sink over residual arcs
// (solvers.py:54-71).  h holds 1 on sink-residual pixels and HINF elsewhere
// after k_gr_init; each tile relaxes to its fixpoint given its halo and
// flags the neighbours facing any border pixel that went down.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int border_sides(int lx, int ly) {
    return (lx == 0 ? 1 << DL : 0) | (lx == TW - 1 ? 1 << DR : 0) | (ly == 0 ? 1 << DU : 0) |
           (ly == TH - 1 ? 1 << DD : 0);
}

// Tile-pass scratch in shared memory, shared by the tile bodies below (one
// body runs at a time in a CTA; kernels allocate only what they reference).
__shared__ int32_t s_sd[TH * SP];     // tile_relax values
__shared__ uint8_t s_sm[TPIX];        // tile_relax pull masks
__shared__ uint8_t s_bits[TPIX];      // label BFS: own outgoing-arc bits
__shared__ int32_t s_hv[4][TW];       // halo values per side
__shared__ int s_side;                // sides whose neighbour needs work

// A thread's inputs of a sink-BFS tile pass: its pixel's height and
// residual word, and (threads < 4 * TW) one halo height -- each halo
// thread reads only its own side's neighbour id (C5 sink BFS -3 % against
// every thread reading all four; issuing the next tile's loads ahead of
// the current relaxation measured no better and was dropped).
template <class E>
struct BfsIn {
    int32_t h0;
    typename E::Word wd;
    int32_t hv;
};
template <class E>
__device__ __forceinline__ BfsIn<E> bfs_sink_load(const Ctx &c, int32_t t) {
    const int i = threadIdx.x;
    const int64_t p = int64_t(t) * TPIX + i;
    BfsIn<E> in;
    in.h0 = __ldcg(c.h + p);
    in.wd = E::load(c.r, p);
    in.hv = HINF;
    if (i < 4 * TW) {
        const int s = i / TW, j = i % TW;
        const int32_t nb = tile_nb(c, t, s);
        if (nb >= 0) in.hv = __ldcg(c.h + int64_t(nb) * TPIX + halo_index(s, j));
    }
    return in;
}

template <class E>
__device__ __forceinline__ TileResult bfs_sink_tile(const Ctx &c, int32_t t, const BfsIn<E> &in) {
    const int i = threadIdx.x, lx = i & 31, ly = i >> 5;
    const int32_t h0 = in.h0;
    const typename E::Word wd = in.wd;
    s_sd[ly * SP + lx] = h0;
    const int mk = (E::lane(wd, 0) > 0) | ((E::lane(wd, 1) > 0) << 1) | ((E::lane(wd, 2) > 0) << 2) |
                   ((E::lane(wd, 3) > 0) << 3);
    s_sm[i] = uint8_t(mk);
    if (i < 4 * TW) s_hv[i / TW][i % TW] = in.hv;
    if (i == 0) s_side = 0;
    __syncthreads();
    // Most passes of a relabel revisit a tile whose heights are already a
    // fixpoint for its new halo (59 % at C5: the neighbour's improvement
    // does not reach it).  One test of every pull arc p <- q -- h(p) <=
    // h(q) + 1 -- proves it and skips the relaxation (exactly the pass the
    // relaxation would have found unchanged).
    {
        int open = 0;
        if (h0 > 1) {
            const int32_t hl = lx > 0 ? s_sd[ly * SP + lx - 1] : s_hv[DL][ly];
            const int32_t hr = lx < TW - 1 ? s_sd[ly * SP + lx + 1] : s_hv[DR][ly];
            const int32_t hu = ly > 0 ? s_sd[(ly - 1) * SP + lx] : s_hv[DU][lx];
            const int32_t hd = ly < TH - 1 ? s_sd[(ly + 1) * SP + lx] : s_hv[DD][lx];
            open = ((mk & 1) && hl + 1 < h0) | ((mk & 2) && hr + 1 < h0) | ((mk & 4) && hu + 1 < h0) |
                   ((mk & 8) && hd + 1 < h0);
        }
        if (!__syncthreads_or(open)) return TileResult{0, 0};
    }
    // (plain sweeps: line skipping measured 1-3 % slower here, where most
    // relaxations settle in one or two sweeps)
    tile_relax<false>(s_sd, s_sm, s_hv, 1);
    // (positions recomputed after the relax: fewer registers live across it)
    const int j = threadIdx.x, h1 = s_sd[(j >> 5) * SP + (j & 31)];
    if (h1 != h0) {
        c.h[int64_t(t) * TPIX + j] = h1;
        if (int b = border_sides(j & 31, j >> 5)) atomicOr(&s_side, b);
    }
    __syncthreads();
    return TileResult{0, s_side};
}

template <class E>
__device__ __forceinline__ TileResult bfs_sink_tile(const Ctx &c, int32_t t) {
    return bfs_sink_tile<E>(c, t, bfs_sink_load<E>(c, t));
}

template <class E>
__global__ void __launch_bounds__(NTT, 2) k_bfs_sink(Ctx c, int k, LaunchCtl lc) {
    tile_loop(c, k, lc, [&](int32_t t) { return bfs_sink_tile<E>(c, t); });
}

// ---------------------------------------------------------------------------
// Source-side closure (solvers.py:144-158): lab = 1 where reachable from an
// excess pixel along residual arcs (relaxation with cost 0 over the arcs
// INTO each pixel); touching a sink-residual pixel means the preflow was
// not maximal (NonMaximalFlowError).
// ---------------------------------------------------------------------------
// spoil != nullptr: a speculative closure (asynchronous solver) -- reaching
// a sink-residual pixel only marks the attempt spoiled instead of raising
template <class E>
__device__ __forceinline__ TileResult bfs_src_tile(const Ctx &c, int32_t t, int32_t *spoil = nullptr) {
    const int i = threadIdx.x, lx = i & 31, ly = i >> 5;
    const int64_t p = int64_t(t) * TPIX + i;
    const uint8_t l0 = __ldcg(c.lab + p);
    // a tile whose every pixel is already in the closure cannot change
    if (__syncthreads_and(l0)) return TileResult{0, 0};
    typename E::Word wd = E::load(c.r, p);
    s_sd[ly * SP + lx] = l0 ? 0 : HINF;
    s_bits[i] = uint8_t((E::lane(wd, 0) > 0) | ((E::lane(wd, 1) > 0) << 1) | ((E::lane(wd, 2) > 0) << 2) |
                        ((E::lane(wd, 3) > 0) << 3));
    if (i < 4 * TW) {
        int s = i / TW, j = i % TW;
        int32_t v = HINF;
        const int32_t nb = tile_nb(c, t, s);   // (own side's id only, as in bfs_sink_load)
        if (nb >= 0 && __ldcg(c.lab + int64_t(nb) * TPIX + halo_index(s, j))) v = 0;
        s_hv[s][j] = v;
    }
    if (i == 0) s_side = 0;
    __syncthreads();
    // pull mask: bit d set when the d-neighbour has a residual arc into us
    int mk = 0;
    if (lx > 0) mk |= (s_bits[i - 1] >> DR) & 1;
    if (lx < TW - 1) mk |= ((s_bits[i + 1] >> DL) & 1) << 1;
    if (ly > 0) mk |= ((s_bits[i - TW] >> DD) & 1) << 2;
    if (ly < TH - 1) mk |= ((s_bits[i + TW] >> DU) & 1) << 3;
    // border pixels: the facing neighbour's arc into us (its id read by the
    // border threads of that side only)
    if (lx == 0) {
        const int32_t nb = tile_nb(c, t, DL);
        if (nb >= 0) mk |= (E::lane(E::load(c.r, int64_t(nb) * TPIX + halo_index(DL, ly)), DR) > 0) << 0;
    }
    if (lx == TW - 1) {
        const int32_t nb = tile_nb(c, t, DR);
        if (nb >= 0) mk |= (E::lane(E::load(c.r, int64_t(nb) * TPIX + halo_index(DR, ly)), DL) > 0) << 1;
    }
    if (ly == 0) {
        const int32_t nb = tile_nb(c, t, DU);
        if (nb >= 0) mk |= (E::lane(E::load(c.r, int64_t(nb) * TPIX + halo_index(DU, lx)), DD) > 0) << 2;
    }
    if (ly == TH - 1) {
        const int32_t nb = tile_nb(c, t, DD);
        if (nb >= 0) mk |= (E::lane(E::load(c.r, int64_t(nb) * TPIX + halo_index(DD, lx)), DU) > 0) << 3;
    }
    s_sm[i] = uint8_t(mk);
    __syncthreads();
    tile_relax(s_sd, s_sm, s_hv, 0);
    if (s_sd[ly * SP + lx] == 0 && !l0) {
        c.lab[p] = 1;
        if (__ldcg(c.w + p) < 0) {
            if (spoil) *spoil = 2;            // the preflow was not maximum yet
            else atomicExch(c.err, 4);        // NonMaximalFlowError
        }
        if (int b = border_sides(lx, ly)) atomicOr(&s_side, b);
    }
    __syncthreads();
    return TileResult{0, s_side};
}

template <class E>
__global__ void __launch_bounds__(NTT, 2) k_bfs_src(Ctx c, int k, LaunchCtl lc) {
    tile_loop(c, k, lc, [&](int32_t t) {
        int32_t *sp = nullptr;   // rolling mode: a speculative closure only marks its grid spoiled
        if (c.specg) {
            const int32_t g = __ldg(c.tile_grid + t);
            if (__ldcg(c.specg + g)) sp = c.specg + g;
        }
        return bfs_src_tile<E>(c, t, sp);
    });
}

// ---------------------------------------------------------------------------
// Push-relabel discharge of one tile (solvers.py:107-136 semantics with the
// lock-free admissibility rule h(p) > h(q), which tolerates the stale halo
// heights of concurrently discharged neighbour tiles).
//
// Registers hold the pixel's excess/sink state e and its four residuals.
// Heights and inflow live in shared memory on a ring-padded 34x34 frame:
// the ring holds the neighbour tiles' facing pixels, so every neighbour
// access is one unconditional load at a fixed offset.  A push into the
// d-neighbour adds to that neighbour's inflow slot for direction opp(d)
// (one writer per slot per iteration -- no atomics); in-tile slots are
// absorbed (and zeroed) by their owner after the barrier, ring slots
// accumulate over the pass and leave as one global atomic per halo pixel.
// At load (and every `relabel_every` iterations) the tile runs an exact
// local relabel: the distance, inside the tile, to a sink-residual pixel
// (1) or to a halo pixel (its height + 1) -- HINF means every path out ends
// in frozen pixels, a certificate that the pixel cannot reach the sink.
// ---------------------------------------------------------------------------
constexpr int RW = TW + 2;             // ring-padded row stride
constexpr int RPIX = RW * (TH + 2);    // ring-padded frame size

__device__ __forceinline__ int ring_index(int s, int j) {
    switch (s) {
    case DL: return (j + 1) * RW;
    case DR: return (j + 1) * RW + TW + 1;
    case DU: return j + 1;
    default: return (TH + 1) * RW + j + 1;
    }
}

__shared__ int32_t s_ph[RPIX];        // discharge heights (ring: neighbour tiles)
__shared__ int32_t s_in[1][4][RPIX];  // s_in[0][d][q]: flow pushed into q by its d-neighbour
__shared__ int s_rowin[1][TH + 2];    // ring-frame row received inflow

// Discharge scratch invariant: inflow slots and row flags are zero at every
// pass boundary; established once per CTA by push_prepare().
__device__ __forceinline__ void push_prepare() {
    for (int j = threadIdx.x; j < 4 * RPIX; j += blockDim.x) (&s_in[0][0][0])[j] = 0;
    if (threadIdx.x < TH + 2) (&s_rowin[0][0])[threadIdx.x] = 0;
}

// Residuals of one pixel held in registers: EdgeU8 keeps the packed u8x4
// word (lane arithmetic on the word is exact: every lane stays in [0, 255])
// -- one register instead of four, which the 32-register discharge needs.
template <class E>
struct RegRes;
template <>
struct RegRes<EdgeU8> {
    uint32_t w;
    __device__ __forceinline__ explicit RegRes(uint32_t word) : w(word) {}
    __device__ __forceinline__ int get(int d) const { return int((w >> (8 * d)) & 0xffu); }
    __device__ __forceinline__ bool pos(int d) const { return ((w >> (8 * d)) & 0xffu) != 0u; }
    __device__ __forceinline__ void add(int d, int v) { w += uint32_t(v) << (8 * d); }
    __device__ __forceinline__ void sub(int d, int v) { w -= uint32_t(v) << (8 * d); }
    __device__ __forceinline__ uint8_t mask() const {
        const uint32_t x = __vcmpne4(w, 0u);   // 0xff per nonzero byte
        return uint8_t(((x >> 7) & 1u) | ((x >> 14) & 2u) | ((x >> 21) & 4u) | ((x >> 28) & 8u));
    }
    __device__ __forceinline__ uint32_t word() const { return w; }
};
template <>
struct RegRes<EdgeI32> {
    int32_t r[4];
    __device__ __forceinline__ explicit RegRes(int4 v) : r{v.x, v.y, v.z, v.w} {}
    __device__ __forceinline__ int get(int d) const { return r[d]; }
    __device__ __forceinline__ bool pos(int d) const { return r[d] > 0; }
    __device__ __forceinline__ void add(int d, int v) { r[d] += v; }
    __device__ __forceinline__ void sub(int d, int v) { r[d] -= v; }
    __device__ __forceinline__ uint8_t mask() const {
        return uint8_t((r[0] > 0) | ((r[1] > 0) << 1) | ((r[2] > 0) << 2) | ((r[3] > 0) << 3));
    }
    __device__ __forceinline__ int4 word() const { return make_int4(r[0], r[1], r[2], r[3]); }
};

// Mid-pass hand-off (knob push_flush, queue modes): flow pushed across the
// tile border so far is applied to the neighbour tiles now and they are
// requested, so they start while this pass goes on, instead of one pass
// (up to `iters` iterations) later.  The border pixels' own deltas are
// written first, so a u8 residual lane never holds the neighbour's
// increment on top of a decrement not yet applied (each side only ever
// adds what it may); w0 / rv0 advance so the final write-back adds only
// what follows.
__shared__ int s_flush;
template <class E>
__device__ __forceinline__ void push_flush(const Ctx &c, int32_t t, int64_t p, int i, int32_t e, int32_t h,
                                           const RegRes<E> &R, int32_t &w0, typename E::Word &rv0) {
    int pending = 0;
    if (i < 4 * TW) {
        const int s = i / TW, j = i % TW;
        pending = s_in[0][opp(s)][ring_index(s, j)] > 0;
    }
    if (i == 0) s_flush = 0;
    if (!__syncthreads_or(pending)) return;
    if (on_border(i)) {
        const typename E::Word rv = R.word();
        if (e != w0) atomicAdd(&c.w[p], e - w0);
        E::store_delta(c.r, p, rv, rv0);
        c.h[p] = h;
        w0 = e;
        rv0 = rv;
    }
    __syncthreads();
    if (i < 4 * TW) {
        const int s = i / TW, j = i % TW;
        int32_t *slot = &s_in[0][opp(s)][ring_index(s, j)];
        const int32_t a = *slot;
        if (a > 0) {
            *slot = 0;
            const int64_t qn = int64_t(tile_nb(c, t, s)) * TPIX + halo_index(s, j);
            atomicAdd(&c.w[qn], a);
            E::add(c.r, qn, opp(s), a);
            atomicOr(&s_flush, 1 << s);
        }
    }
    qfence();   // requester side: data writes < queue-state RMWs
    __syncthreads();
    if (i >= 1 && i <= 4 && ((s_flush >> (i - 1)) & 1)) {
        const int32_t nb = tile_nb(c, t, i - 1);
        if (nb >= 0) q_request(c, nb);
    }
    __syncthreads();
}

template <class E>
__device__ __forceinline__ TileResult push_tile(const Ctx &c, int32_t t, int iters, int relabel_every) {
    constexpr int OFF[4] = {-1, 1, -RW, RW};
    const int i = threadIdx.x, lx = i & 31, ly = i >> 5, pi = ly * SP + lx;
    const int q = (ly + 1) * RW + lx + 1;
    const int64_t p = int64_t(t) * TPIX + i;
    int32_t w0 = __ldcg(c.w + p);
    typename E::Word rv0 = E::load(c.r, p);
    int32_t e = w0, h = __ldcg(c.h + p);
    RegRes<E> R(rv0);
    if (i < 4 * TW) {
        const int s = i / TW, j = i % TW;
        const int32_t nb = tile_nb(c, t, s);
        const int32_t v = nb >= 0 ? __ldcg(c.h + int64_t(nb) * TPIX + halo_index(s, j)) : HINF;
        s_hv[s][j] = v;
        s_ph[ring_index(s, j)] = v;
    }
    if (i == 0) s_side = 0;
    // a tile requested only for inflow that its deficits absorbed has nothing
    // to discharge (21 % of the passes at C2): no local relabel, no write-back
    if (!__syncthreads_or(e > 0 && h < HINF)) return TileResult{0, 0};
    // first pass after an exact relabel: the local relabel would reproduce
    // the heights (exact global distances restricted to the tile), skip it
    bool fresh = false;
    if (c.tfresh) {
        fresh = __ldcg(c.tfresh + t) != 0;
        __syncthreads();   // everyone has read the flag before it is cleared
        if (fresh && i == 0) c.tfresh[t] = 0;
    }
    int act = 1;
    int until_relabel = fresh ? relabel_every : 0, its = 0;
    for (int it = 0; it < iters; it++) {
        its++;
        if (c.push_flush && it > 0 && it % c.push_flush == 0 && c.persistent)
            push_flush<E>(c, t, p, i, e, h, R, w0, rv0);
        if (relabel_every && until_relabel == 0) {
            until_relabel = relabel_every;
            // exact local relabel (frozen pixels stay frozen)
            s_sd[pi] = e < 0 ? 1 : HINF;
            s_sm[i] = R.mask();
            __syncthreads();
            const unsigned long long tr0 = i == 0 ? gtimer() : 0ull;
            const int rr = tile_relax(s_sd, s_sm, s_hv, 1), conv = rr & 1;
            if (i == 0) {   // diagnostics
                atomicAdd(&c.stat[ST_RELAX_NS], gtimer() - tr0);
                atomicAdd(&c.stat[ST_RELAX_N], 1ull);
                atomicAdd(&c.stat[ST_RELAX_SW], (unsigned long long)(rr >> 1));
            }
            // an unconverged relax may not freeze anyone (keep the old
            // height where it found nothing)
            if (h < HINF && (conv || s_sd[pi] < HINF)) h = s_sd[pi];
            s_ph[q] = h;
            act = __syncthreads_or(e > 0 && h < HINF);
            if (!act) break;
        } else if (it == 0) {
            s_ph[q] = h;
            act = __syncthreads_or(e > 0 && h < HINF);
            if (!act) break;
        }
        until_relabel--;
        // warp == tile row: rows without an active pixel skip the push
        // work, rows nobody pushed into skip the merge (barriers stay).
        // Every pixel reads its neighbours' heights here, before the
        // relabels of this iteration write any: a pixel that becomes active
        // by inflow relabels from these values too (no read of s_ph races
        // with a relabel write; racecheck-clean)
        const bool mine = e > 0 && h < HINF;
        int32_t hn[4];
#pragma unroll
        for (int d = 0; d < 4; d++) hn[d] = s_ph[q + OFF[d]];
        if (__any_sync(0xffffffffu, mine)) {
            // ---- push downhill (heights are fixed during this phase, so
            // an arc is never pushed both ways and every inflow slot has
            // one writer)
            if (mine) {
                int pushed = 0;
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    const int rd = R.get(d);
                    if (e > 0 && rd > 0 && h > hn[d]) {
                        const int32_t dl = min(e, rd);
                        e -= dl;
                        R.sub(d, dl);
                        s_in[0][opp(d)][q + OFF[d]] += dl;
                        pushed |= 1 << d;
                    }
                }
                if (pushed & ((1 << DL) | (1 << DR))) s_rowin[0][ly + 1] = 1;
                if (pushed & (1 << DU)) s_rowin[0][ly] = 1;
                if (pushed & (1 << DD)) s_rowin[0][ly + 2] = 1;
            }
        }
        __syncthreads();
        // ---- absorb inflow, relabel what is still active
        if (s_rowin[0][ly + 1]) {
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const int32_t v = s_in[0][d][q];
                if (v) {
                    e += v;
                    R.add(d, v);
                    s_in[0][d][q] = 0;
                }
            }
            __syncwarp();
            if (lx == 0) s_rowin[0][ly + 1] = 0;
        }
        if (e > 0 && h < HINF) {
            int32_t m = HINF;
#pragma unroll
            for (int d = 0; d < 4; d++)
                if (R.pos(d)) m = min(m, hn[d]);
            if (m >= h) {
                h = m >= HINF ? HINF : m + 1;
                s_ph[q] = h;
            }
        }
        act = __syncthreads_or(e > 0 && h < HINF);
        if (!act) break;
    }
    if (i == 0) atomicAdd(&c.stat[ST_PUSH_ITERS], (unsigned long long)its);   // diagnostics
    // ---- write back: interior pixels plainly, border pixels as deltas
    // (neighbour tiles may have pushed into them meanwhile)
    const typename E::Word rv = R.word();
    if (!on_border(i)) {
        c.w[p] = e;
        E::store(c.r, p, rv);
    } else {
        if (e != w0) atomicAdd(&c.w[p], e - w0);
        E::store_delta(c.r, p, rv, rv0);
    }
    c.h[p] = h;
    if (i < 2) s_rowin[0][i * (TH + 1)] = 0;   // ring rows are never absorbed
    __syncthreads();
    if (i < 4 * TW) {
        const int s = i / TW, j = i % TW;
        int32_t *slot = &s_in[0][opp(s)][ring_index(s, j)];
        const int32_t a = *slot;
        if (a > 0) {
            *slot = 0;
            const int64_t qn = int64_t(tile_nb(c, t, s)) * TPIX + halo_index(s, j);
            atomicAdd(&c.w[qn], a);
            E::add(c.r, qn, opp(s), a);
            atomicOr(&s_side, 1 << s);
        }
    }
    __syncthreads();
    return TileResult{act, s_side};
}

template <class E>
__global__ void __launch_bounds__(NTT, 2) k_push(Ctx c, int k, int iters, int relabel_every, LaunchCtl lc) {
    push_prepare();
    tile_loop(c, k, lc, [&](int32_t t) { return push_tile<E>(c, t, iters, relabel_every); });
}

}  // namespace pmf
