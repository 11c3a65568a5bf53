// engine.cuh -- device data layout and small helpers shared by the kernels.
//
// Layout: every independent grid graph of a
// batch (one lambda-graph, or one whole composite) is cut into 32x32 tiles;
// tiles of all grids are numbered 0..T-1 and each per-pixel plane is stored
// tile-major, pixel p = tile*1024 + ly*32 + lx.  Planes:
//   w  int32  combined terminal state of the reduced network: w > 0 is excess,
//             w < 0 is the residual capacity of the pixel->sink arc
//   h  int32  distance label (HINF = cannot reach the sink: frozen)
//   r  u8x4   residuals of the 4 neighbour arcs packed in one word (EdgeU8)
//      int4   or four int32 (EdgeI32) when a capacity pair exceeds 255
//   lab u8    source-side reachability (label BFS)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pmf {

constexpr int TW = 32;              // tile width  (one warp across)
constexpr int TH = 32;              // tile height
constexpr int TPIX = TW * TH;       // pixels per tile
constexpr int NT = 256;             // threads per CTA
constexpr int PPT = TPIX / NT;      // pixels per thread (4)
constexpr int32_t HINF = 0x3fffffff;
constexpr int64_t CAP_MAX = int64_t(1) << 30;   // grid.py:19

enum { DL = 0, DR = 1, DU = 2, DD = 3 };         // grid.py:23 order
__host__ __device__ constexpr int opp(int d) { return d ^ 1; }

// statistics counters (device, unsigned long long): tile passes per kernel
// kind, launches and their device-clock spans (ns, %globaltimer)
enum {
    ST_PUSH = 0, ST_BFS = 1, ST_LAB = 2,
    ST_PUSH_NS = 3, ST_BFS_NS = 4, ST_LAB_NS = 5,
    ST_PUSH_L = 6, ST_BFS_L = 7, ST_LAB_L = 8,
    ST_PUSH_ITERS = 28,   // discharge iterations executed (diagnostics)
    ST_RELAX_NS = 29, ST_RELAX_N = 30, ST_RELAX_SW = 31,   // discharge local relabels: time, count, sweeps
    ST_SPEC_ROLL = 34, ST_SPOIL_ROLL = 35,   // rolling mode: speculative label rounds tried / spoiled
    ST_NSTAT = 40
};

// sweep index convention of the list-driven tile kernels
constexpr int K_PERSISTENT = -1;   // one launch drains the device queue
constexpr int K_DEVICE = -2;       // sweep index lives in Ctl (graph-driven loop)
constexpr int K_MULTI = -3;        // one cooperative launch runs every sweep (grid barriers)

// Device-side control block of a solve (graph-driven mode keeps all loop
// state here; the host never reads it mid-solve).
// diagnostics builds may lengthen the launch trace (-DPMF_KTRACE=...)
#ifndef PMF_KTRACE
#define PMF_KTRACE 256
#endif
struct Ctl {
    int32_t k;              // sweep index of the current list phase
    uint32_t done;          // CTAs finished in the current launch
    int32_t cycle;          // global relabel cycles so far
    uint32_t budget;        // pop budget of the next persistent discharge
    int32_t nact;           // tiles seeded for discharge this cycle
    int32_t noconv;         // non-convergence guard tripped
    int32_t cycles_total;   // cycles over all warm-start steps
    int32_t steps;          // warm-start steps run
    int32_t more;           // another warm-start step follows
    int32_t nfin;           // rolling mode: grids that finished in this cycle
    unsigned long long t0;  // earliest CTA start of the current launch (ns)
    unsigned long long t1;  // latest CTA end of the current launch (ns)
    uint32_t bar_count;     // grid barrier (K_MULTI): arrivals so far in the launch
    uint32_t bar_pad;
    // trace of the first kTrace tile-kernel launches: kind, span (ns), tile passes
    int32_t ntrace;
    int32_t trace_kind[PMF_KTRACE];
    unsigned long long trace_ns[PMF_KTRACE];
    unsigned long long trace_tiles[PMF_KTRACE];
    unsigned long long trace_t0[PMF_KTRACE];  // absolute start of the launch (ns)
};
constexpr int kTrace = PMF_KTRACE;

// Grid-wide barrier for cooperative launches (every CTA co-resident): a
// monotonic arrival counter; barrier `round` (0, 1, ...) of the launch
// completes when it reaches (round + 1) * gridDim.x.  The last CTA to leave
// the launch resets it (launch_exit).  Release/acquire at gpu scope orders
// each CTA's tile writes before the other CTAs' reads in the next sweep.
__device__ __forceinline__ void grid_sync(Ctl *ctl, int round) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t target = uint32_t(round + 1) * gridDim.x;
        uint32_t *ctr = &ctl->bar_count;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        uint32_t v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct GridDesc {
    int32_t W, H, ntx, nty;
    int64_t tile_base;
    int64_t out_off;        // offset of this grid's label bytes in the output
    int32_t kind;           // 0: batch lambda-graph, 1: composite (column spans)
    int32_t colswap_off;    // composite: offset of its per-column swap flags
    int32_t prob, lam;      // builder: problem / first lambda index of the grid's chain
    int32_t lam_end;        // one past the last lambda index of the chain (warm start)
    int32_t pitch, xoff;    // composite span grids: row pitch of the composite's planes and
                            // output, and the span's first column (W and 0 otherwise)
};

struct Ctx {
    int32_t *w;
    int32_t *h;
    void *r;
    uint8_t *lab;
    const int32_t *tile_grid;
    const int4 *tnb;        // per tile: neighbour tile per side (L, R, U, D), -1 if none
    const GridDesc *grids;
    int32_t *live;          // per grid: still has work
    int32_t *fin;           // per grid (rolling mode): finished its lambda this cycle, labels due
    int32_t *gpend;         // per grid: its tiles queued or running in the current persistent phase
    int32_t *specg;         // rolling mode (nullable): 1 label closure speculative, 2 spoiled
    int32_t *keeph;         // warm chains (nullable): grid entered its lambda with valid heights, skip its relabel
    int32_t *labok;         // warm chains (nullable): lab holds the grid's previous lambda's minimal
                            // source side (nested seeding of the next label closure)
    int32_t ngrids;
    int32_t rolling;        // rolling warm start: grids emit and advance as they finish
    uint8_t *tfresh;        // per tile: heights are exact from the last relabel (first discharge
                            // pass skips its local relabel, a no-op then); nullptr: off
    int32_t push_flush;     // discharge: hand border inflow to the neighbours every this many iterations (0 off)
    int32_t *act;           // per grid active-pixel count of the last seed pass
    int32_t *list0, *list1; // double-buffered tile worklists
    int32_t *inq0, *inq1;   // "already listed" flags per tile, per buffer
    int32_t *cnt;           // 3 rolling list lengths
    int64_t *snk_sum;       // per grid sum of (embedded) sink capacities
    int64_t *drain;         // per grid sum of unused sink residual
    int32_t *err;           // device error code (0 ok)
    unsigned long long *stat;
    const uint8_t *colswap; // composite per-column swapped flags
    const int32_t *swapflag;// batch: per-problem swap decision (device-made)
    uint8_t *out;           // label output bytes
    int64_t ntiles;
    // persistent work queue: ring of tile ids (-1 =
    // empty slot), per-tile state, counters {head, tail, pending, pops}
    int32_t *ring;
    int32_t *qstate;
    unsigned int *qctr;
    int32_t qcap;
    int32_t persistent;     // seed kernels feed the queue (1) or list 0 (0)
    unsigned int budget;    // max tile pops of a persistent phase (0 = none)
    Ctl *ctl;               // device control block
    int32_t budget_dev;     // persistent discharge reads its budget from ctl
    int32_t *cur_lam;       // per grid: lambda index being solved (warm-start chains)
    int64_t *flows;         // per (problem, lambda) [seed batch] or per grid [composites]
    int32_t nlam;           // lambdas per problem (seed batch)
};

enum { Q_IDLE = 0, Q_QUEUED = 1, Q_RUNNING = 2, Q_DIRTY = 3 };
enum { QC_HEAD = 0, QC_TAIL = 1, QC_PENDING = 2, QC_CONT = 3 };   // HEAD: tickets taken; CONT: continuations

// Queue hand-off fence.  Every cross-CTA hand-off of a tile goes through a
// read-modify-write of that tile's queue state (requests CAS it, pops and
// retirements exchange / CAS it), so the data written before a request is
// published by release / acquire through the same location; gpu-scope
// acq_rel fences suffice where sequential consistency would cost more.
__device__ __forceinline__ void qfence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_volatile(const unsigned *p) {
    return *(const volatile unsigned *)p;
}

// Append t (whose state the caller just moved to QUEUED) to the ring.
__device__ __forceinline__ void q_push(const Ctx &c, int32_t t) {
    unsigned idx = atomicAdd(&c.qctr[QC_TAIL], 1u);
    int32_t *slot = &c.ring[idx % unsigned(c.qcap)];
    while (atomicCAS(slot, -1, t) != -1) __nanosleep(64);
}

// Ask for tile t to be (re)processed: idle -> queued, running -> dirty.
// Always an RMW on the state (see qfence).  Split in two so a hand-off can
// overlap the ring insertion with the retirement of its own tile:
// q_mark() changes the state and counts the tile as pending (returns true
// when the caller must q_push it), q_push() inserts it.
__device__ __forceinline__ bool q_mark(const Ctx &c, int32_t t) {
    int s = atomicCAS(&c.qstate[t], Q_IDLE, Q_QUEUED);
    for (;;) {
        if (s == Q_IDLE) {
            atomicAdd(&c.qctr[QC_PENDING], 1u);
            atomicAdd(&c.gpend[c.tile_grid[t]], 1);
            return true;
        }
        if (s == Q_QUEUED || s == Q_DIRTY) return false;
        // running: mark dirty (it requeues itself when done)
        const int o = atomicCAS(&c.qstate[t], Q_RUNNING, Q_DIRTY);
        if (o == Q_RUNNING) return false;
        s = o == Q_IDLE ? atomicCAS(&c.qstate[t], Q_IDLE, Q_QUEUED) : o;
    }
}

__device__ __forceinline__ void q_request(const Ctx &c, int32_t t) {
    if (q_mark(c, t)) q_push(c, t);
}

// The running tile t is done; requeue it if it still has work or was
// dirtied meanwhile, else retire it (pending only drops on retirement, so
// pending == 0 means nothing is queued or running anywhere).
__device__ __forceinline__ void q_finish(const Ctx &c, int32_t t, bool again) {
    for (;;) {
        if (again) {
            atomicExch(&c.qstate[t], Q_QUEUED);
            q_push(c, t);
            return;
        }
        if (atomicCAS(&c.qstate[t], Q_RUNNING, Q_IDLE) == Q_RUNNING) {
            atomicSub(&c.gpend[c.tile_grid[t]], 1);
            atomicSub(&c.qctr[QC_PENDING], 1u);
            return;
        }
        again = true;   // dirtied while running
    }
}

// Thread 0 of a persistent CTA: next tile to process, or -1 when the phase
// is over (nothing queued or running) or its pop budget is spent.  Poppers
// take a ticket (ring position) with one fetch-add -- no CAS retry loop on
// a contended head -- and wait for a tile to land in that slot.  Any waiter
// on a slot may take any tile that lands there, so tickets that alias a
// slot (more waiters than ring slots) only reorder work.  Tickets taken
// after the phase drained are discarded by the next k_phase_begin.
// Wait for the tile of ticket hd (a ring position), or -1 when the phase is
// over (nothing queued or running).
__device__ __forceinline__ int32_t q_wait(const Ctx &c, unsigned hd) {
    int32_t *slot = &c.ring[hd % unsigned(c.qcap)];
    for (;;) {
        if (*(volatile int32_t *)slot != -1) {
            const int32_t t = atomicExch(slot, -1);
            if (t >= 0) {
                atomicExch(&c.qstate[t], Q_RUNNING);
                return t;
            }
        }
        if (ld_volatile(&c.qctr[QC_PENDING]) == 0) return -1;
        __nanosleep(64);
    }
}

__device__ __forceinline__ int32_t q_next(const Ctx &c) {
    // device budget: 0 means "no discharge this cycle"; host budget 0: no cap
    const unsigned budget = c.budget_dev ? *(volatile unsigned *)&c.ctl->budget : c.budget;
    if (c.budget_dev && budget == 0) return -1;
    if (budget && ld_volatile(&c.qctr[QC_HEAD]) + ld_volatile(&c.qctr[QC_CONT]) >= budget) return -1;
    const unsigned hd = atomicAdd(&c.qctr[QC_HEAD], 1u);
    if (budget && hd + ld_volatile(&c.qctr[QC_CONT]) >= budget) return -1;
    return q_wait(c, hd);
}

// Continuation: the CTA that just finished a tile takes an idle neighbour
// it activated straight away (IDLE -> RUNNING), skipping the ring hand-off
// -- the common case in the latency-bound tail, where excess walks from tile
// to tile.  Counts against the pop budget like a pop.
__device__ __forceinline__ bool q_claim(const Ctx &c, int32_t t) {
    const unsigned budget = c.budget_dev ? *(volatile unsigned *)&c.ctl->budget : c.budget;
    if (budget && ld_volatile(&c.qctr[QC_HEAD]) + ld_volatile(&c.qctr[QC_CONT]) >= budget) return false;
    if (atomicCAS(&c.qstate[t], Q_IDLE, Q_RUNNING) != Q_IDLE) return false;
    atomicAdd(&c.qctr[QC_PENDING], 1u);
    atomicAdd(&c.gpend[c.tile_grid[t]], 1);
    atomicAdd(&c.qctr[QC_CONT], 1u);
    return true;
}

// Label-phase kernels act on every grid, or in rolling mode only on the
// grids that finished their lambda in this cycle.
__device__ __forceinline__ bool grid_due(const Ctx &c, int32_t g) { return !c.rolling || c.fin[g]; }

// A batch grid embedded swapped reports its sink side (what split() turns
// into the original graph's minimal source side); everything else needs the
// source-side BFS.
__device__ __forceinline__ bool grid_swapped(const Ctx &c, const GridDesc &gd) {
    return gd.kind == 0 && c.swapflag[gd.prob] != 0;
}

__device__ __forceinline__ int32_t *list_of(const Ctx &c, int k) { return (k & 1) ? c.list1 : c.list0; }
__device__ __forceinline__ int32_t *inq_of(const Ctx &c, int k) { return (k & 1) ? c.inq1 : c.inq0; }

// Append tile t to worklist k (once per list, guarded by its inq flag).
__device__ __forceinline__ void enqueue(const Ctx &c, int k, int32_t t) {
    if (atomicExch(&inq_of(c, k)[t], 1) == 0) {
        int idx = atomicAdd(&c.cnt[k % 3], 1);
        list_of(c, k)[idx] = t;
    }
}

// Seed kernels: put t in the first worklist of the phase (sweep mode) or
// in the persistent queue.
__device__ __forceinline__ void seed_tile(const Ctx &c, int32_t t) {
    if (c.persistent) q_request(c, t);
    else enqueue(c, 0, t);
}

struct TileGeo {
    int32_t g;              // grid id
    int32_t tx, ty;
    int32_t nb[4];          // neighbour tile ids per side, -1 if none
    int32_t x0, y0, W, H;
};

__device__ __forceinline__ TileGeo tile_geo(const Ctx &c, int32_t t) {
    TileGeo o;
    o.g = c.tile_grid[t];
    const GridDesc &gd = c.grids[o.g];
    int32_t l = int32_t(t - gd.tile_base);
    o.tx = l % gd.ntx;
    o.ty = l / gd.ntx;
    o.nb[DL] = o.tx > 0 ? t - 1 : -1;
    o.nb[DR] = o.tx + 1 < gd.ntx ? t + 1 : -1;
    o.nb[DU] = o.ty > 0 ? t - gd.ntx : -1;
    o.nb[DD] = o.ty + 1 < gd.nty ? t + gd.ntx : -1;
    o.x0 = o.tx * TW;
    o.y0 = o.ty * TH;
    o.W = gd.W;
    o.H = gd.H;
    return o;
}

// Neighbour tile on side s (one load from the precomputed table).
__device__ __forceinline__ int32_t tile_nb(const Ctx &c, int32_t t, int s) {
    const int *nb = reinterpret_cast<const int *>(c.tnb + t);
    return __ldg(nb + s);
}

struct TileNb {
    int32_t nb[4];
};
__device__ __forceinline__ TileNb tile_nbs(const Ctx &c, int32_t t) {
    const int4 v = __ldg(c.tnb + t);
    return TileNb{{v.x, v.y, v.z, v.w}};
}

// Index, inside the neighbour tile on side s, of the halo pixel facing
// position j (row for L/R, column for U/D) of this tile.
__device__ __forceinline__ int halo_index(int s, int j) {
    switch (s) {
    case DL: return j * TW + (TW - 1);
    case DR: return j * TW;
    case DU: return (TH - 1) * TW + j;
    default: return j;
    }
}

__device__ __forceinline__ bool on_border(int i) {
    int lx = i & (TW - 1), ly = i / TW;
    return lx == 0 || lx == TW - 1 || ly == 0 || ly == TH - 1;
}

// ---- residual storage policies -------------------------------------------

// Four 8-bit residuals in one word: lane d holds r(p -> d-neighbour).
// Valid when every arc pair satisfies c(p->q) + c(q->p) <= 255, checked on
// the host; all concurrent updates are word-sized atomics of lane deltas
// that keep every lane inside [0, 255].
struct EdgeU8 {
    using Word = uint32_t;
    static constexpr int kBytes = 4;
    __device__ static Word load(const void *R, int64_t p) { return __ldcg(((const uint32_t *)R) + p); }
    __device__ static int lane(Word w, int d) { return int((w >> (8 * d)) & 0xffu); }
    __device__ static Word pack(int a, int b, int c, int d) {
        return uint32_t(a) | (uint32_t(b) << 8) | (uint32_t(c) << 16) | (uint32_t(d) << 24);
    }
    __device__ static void store(void *R, int64_t p, Word w) { ((uint32_t *)R)[p] = w; }
    __device__ static void store_delta(void *R, int64_t p, Word nw, Word ow) {
        if (nw != ow) atomicAdd(((uint32_t *)R) + p, nw - ow);
    }
    __device__ static void add(void *R, int64_t p, int d, int v) {
        atomicAdd(((uint32_t *)R) + p, uint32_t(v) << (8 * d));
    }
};

// Four int32 residuals per pixel (16 B, int4-aligned).
struct EdgeI32 {
    using Word = int4;
    static constexpr int kBytes = 16;
    __device__ static Word load(const void *R, int64_t p) { return __ldcg(((const int4 *)R) + p); }
    __device__ static int lane(Word w, int d) {
        return d == 0 ? w.x : d == 1 ? w.y : d == 2 ? w.z : w.w;
    }
    __device__ static Word pack(int a, int b, int c, int d) { return make_int4(a, b, c, d); }
    __device__ static void store(void *R, int64_t p, Word w) { ((int4 *)R)[p] = w; }
    __device__ static void store_delta(void *R, int64_t p, Word nw, Word ow) {
        int *q = ((int *)R) + 4 * p;
        if (nw.x != ow.x) atomicAdd(q + 0, nw.x - ow.x);
        if (nw.y != ow.y) atomicAdd(q + 1, nw.y - ow.y);
        if (nw.z != ow.z) atomicAdd(q + 2, nw.z - ow.z);
        if (nw.w != ow.w) atomicAdd(q + 3, nw.w - ow.w);
    }
    __device__ static void add(void *R, int64_t p, int d, int v) {
        atomicAdd(((int *)R) + 4 * p + d, v);
    }
};

}  // namespace pmf
