// engine.cu -- host driver and C ABI of the B200 supergraph min-cut engine.
//
// One pmf_solver = one CUDA device + one stream + grow-only device/pinned
// workspaces.  A solve is a fixed sequence of kernel launches on that
// stream; the host synchronises only to read worklist lengths (BFS
// convergence, termination), never per tile.  See DESIGN.md.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <sys/mman.h>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/pmflow_b200.h"
#include "kernels.cuh"
#include "tile.cuh"
#include "warp.cuh"
#include "async.cuh"
#include "wide.cuh"

using namespace pmf;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess)                                                     \
            return fail(PMF_ERR_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap) return 0;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) return fail(PMF_ERR_CUDA, "cudaMalloc(%zu): %s", want, cudaGetErrorString(e));
        cap = want;
        return 0;
    }
    template <class T> T *as() const { return (T *)p; }
    ~DevBuf() { if (p) cudaFree(p); }
};

struct HostBuf {
    void *p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap) return 0;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e != cudaSuccess) return fail(PMF_ERR_CUDA, "cudaMallocHost(%zu): %s", want, cudaGetErrorString(e));
        cap = want;
        return 0;
    }
    template <class T> T *as() const { return (T *)p; }
    ~HostBuf() { if (p) cudaFreeHost(p); }
};

enum Cat { C_BUILD = 0, C_BFS, C_PUSH, C_SEED, C_LAB, C_H2D, C_D2H, C_N };

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Host-side parallel loops (OpenMP) for the conversion / validation of the
// input planes and the copy-out of label masks: the host side of the e2e
// path is memory-bound int64 -> int32 narrowing that one thread cannot
// keep up with.
struct Pool {
    int threads = 1;
    // fn(i) for i in [0, n)
    template <class F>
    void run(int64_t n, F &&fn) {
        if (n <= 0) return;
        const int nt = int(std::min<int64_t>(threads, n));
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
        for (int64_t i = 0; i < n; i++) fn(i);
    }
};

// first error raised by a parallel task (others keep running, result dropped)
struct TaskErr {
    std::atomic<int> code{0};
    std::mutex mu;
    std::string msg;
    void set(int c, const std::string &m) {
        int z = 0;
        if (code.compare_exchange_strong(z, c)) {
            std::lock_guard<std::mutex> g(mu);
            msg = m;
        }
    }
    int raise() {
        if (!code.load()) return 0;
        std::lock_guard<std::mutex> g(mu);
        return fail(code.load(), "%s", msg.c_str());
    }
};

constexpr int64_t kChunk = 1 << 14;   // elements per host task


struct Layout {
    std::vector<GridDesc> grids;
    std::vector<int32_t> tile_grid;
    std::vector<int4> tile_nb;      // neighbour tile per side (L, R, U, D), -1 if none
    int64_t ntiles = 0, out_bytes = 0, pixels = 0;
    void clear() {
        grids.clear();
        tile_grid.clear();
        tile_nb.clear();
        ntiles = out_bytes = pixels = 0;
    }
    void add(int32_t W, int32_t H, int32_t kind, int32_t colswap_off, int32_t prob, int32_t lam,
             int32_t lam_end) {
        GridDesc g{};
        g.W = W;
        g.H = H;
        g.ntx = int32_t(cdiv(W, TW));
        g.nty = int32_t(cdiv(H, TH));
        g.tile_base = ntiles;
        g.out_off = out_bytes;
        g.kind = kind;
        g.colswap_off = colswap_off;
        g.prob = prob;
        g.lam = lam;
        g.lam_end = lam_end;
        g.pitch = W;
        g.xoff = 0;
        int64_t nt = int64_t(g.ntx) * g.nty;
        tile_grid.insert(tile_grid.end(), size_t(nt), int32_t(grids.size()));
        for (int32_t ty = 0; ty < g.nty; ty++)
            for (int32_t tx = 0; tx < g.ntx; tx++) {
                const int32_t t = int32_t(ntiles + int64_t(ty) * g.ntx + tx);
                tile_nb.push_back(make_int4(tx > 0 ? t - 1 : -1, tx + 1 < g.ntx ? t + 1 : -1,
                                            ty > 0 ? t - g.ntx : -1, ty + 1 < g.nty ? t + g.ntx : -1));
            }
        ntiles += nt;
        out_bytes += int64_t(W) * H;
        pixels += int64_t(W) * H;
        grids.push_back(g);
    }
    // One column span [xoff, xoff + W) of a pitch x H composite whose output
    // starts at out_base (reserved by the caller): a grid of its own.
    void add_span(int32_t W, int32_t H, int32_t colswap_off, int32_t comp, int64_t out_base, int32_t pitch,
                  int32_t xoff) {
        const int64_t ob = out_bytes, px = pixels;
        add(W, H, 1, colswap_off, comp, 0, 1);
        out_bytes = ob;
        pixels = px + int64_t(W) * H;
        grids.back().out_off = out_base;
        grids.back().pitch = pitch;
        grids.back().xoff = xoff;
    }
};

// A staged seed batch: converted planes resident on the device, ready to be
// built and solved any number of times (pmf_seed_run).
struct SeedStage {
    bool valid = false;
    int32_t nprob = 0, nlam = 0, W = 0, H = 0, swap_mode = 0;
    bool u8 = true;
    std::vector<int64_t> offs;      // [plane_off(nprob) | pw_off(nprob)]
    std::vector<int64_t> lambdas;
    std::vector<int64_t> slope_sum; // per problem: sum of unary_slope over non-fg pixels
    int32_t chain = 1;              // lambdas per warm-start chain
    bool wide = false;              // excess bound past int32: int64 state variant (wide.cuh)
    bool synth = false;             // planes derived on the device from 8-bit images (pmf_synth_stage)
    int32_t nimg = 0, nseed = 0;    // ... images and seeds per image of such a batch
};

}  // namespace

struct pmf_solver {
    int device = 0;
    cudaStream_t st = nullptr;
    int sms = 148;
    int grid_push = 0, grid_bfs = 0, grid_full = 0;
    // knobs
    int push_iters = 16;
    int push_sweeps = 64;
    int relabel_every = 8;
    // label BFS: warp-per-tile bitset kernel (4, default) or the
    // 1024-thread CTA kernel (0)
    int warp = 4;
    int warp_eff = 0;         // resolved for the current batch
    int warm_active = 0;      // the current run uses warm-start chains
    int grid_wbfs = 0;
    size_t smem_w = 0;
    int persistent = 1;       // discharge phase as one persistent launch
    int persistent_bfs = 0;   // BFS phases as one persistent launch
    int bfs_multi = 1;        // BFS phases as one cooperative launch (grid barriers between sweeps)
    int push_budget = 2;      // persistent push phase: pops <= budget * seeded tiles
    int chain = 0;            // warm-start chain length (0: auto, see warm_min_problems)
    int warm_min_problems = 8;  // auto: one chain per problem (whole ladder) from this many problems
    int push_budget_warm = 3;   // discharge budget factor when the batch runs warm-start chains
    int push_budget_add = 64;   // asynchronous solver: + this many pops per discharge phase
    int verify = 1;             // seed batches: device cut_cost == flow certificate per cut
    int verify_vec = 1;         // 4-pixel-group verify kernel when W % 4 == 0
    int rolling = 1;            // warm-start chains advance per grid as each finishes (no step barrier)
    int fresh_skip = 1;         // first discharge pass after an exact relabel skips its local relabel
    int push_flush = 0;         // discharge: hand border inflow over every this many iterations (0 off; queue modes)
    int async_mode = -1;        // seed batches: one persistent kernel, every grid on its own phase machine
                                // (1), step-synchronous phases (0), or -1: async up to async_max_tiles tiles
    int async_max_tiles = 20000;
    int async_max_grid_tiles = 1024;   // ... and grids of at most this many tiles on average
    int async_cont = 1, async_prefetch = 1;
    int nested_lab = 1;
    int comp_async = 1;         // latency-bound composites on the asynchronous solver         // rolling step mode: seed label closures with the previous lambda's source side
    int async_yield_us = 0;     // asynchronous solver: idle CTAs leave an empty-queue tail after this (0 never)
    int async_yield_keep = 0;   // ... except the first this many CTAs (0: a quarter of the grid)
    bool last_async = false;    // the last launched seed run was asynchronous (no cooperative kernels)
    int async_spec = 1;         // drained discharge -> speculative label closure instead of a confirming relabel
    int adv_keep_h = 1;         // async: unswapped grids enter the next lambda without a relabel
    int phase_log = 0;          // diagnostics: record every grid's phase timeline (async)
    int64_t plog_grids = 0;
    double busy_ms[16] = {0};
    int64_t spec_tries = 0, spec_spoiled = 0;    // async: CTA-busy time per phase kind of the last run (diagnostics)
    int bfs_chunk = 8;
    int timing = 0;
    int64_t max_cycles = 50000;
    int force_wide = 0;         // select the int64 state variant even when int32 bounds hold (tests)
    cudaEvent_t fetch_ev[8] = {};   // seed_fetch: label pieces in flight (created once)
    int wide_pulses = 64;       // int64 variant: lock-step pulses between exact global relabels
    int64_t wide_cycles = 0, wide_pulses_run = 0, wide_relax_launches = 0;   // ... of the last wide run
    // device workspace
    DevBuf d_w, d_h, d_r, d_lab, d_tile_grid, d_tnb, d_fin, d_gpend, d_specg, d_keeph, d_labok, d_seeds, d_sofs, d_gr, d_tflag, d_vacc, d_truth, d_score, d_plog, d_tfresh, d_grids, d_live, d_act, d_list, d_inq, d_cnt,
        d_snk, d_drain, d_err, d_stat, d_colswap, d_out, d_bits, d_in32, d_pw, d_mask, d_off, d_lam,
        d_swapcnt, d_swapflag, d_ring, d_qstate, d_qctr, d_ctl, d_curlam, d_flows, d_slopesum,
        d_we, d_wr, d_wgrid, d_wtile, d_wchg, d_wcnt, d_cv,   // int64 state variant (wide.cuh)
        d_img, d_spix;   // on-device synthesis: images, seed pixel per (image, seed)
    HostBuf h_in32, h_pw, h_mask, h_out, h_small, h_seeds;
    Layout lay;
    std::vector<int32_t> ones, curlam0;
    std::vector<uint8_t> colswap;
    std::vector<int64_t> comp_off, grid_off, comp_out, comp_n;
    int comp_any_split = 0;
    int comp_split = 1;         // composites: one grid per isolated segment span
    SeedStage stage;
    Ctx ctx{};
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_marks;  // (category, event index of start)
    size_t ev_used = 0;
    cudaEvent_t ev_run[2] = {nullptr, nullptr};
    cudaEvent_t ev_tail = nullptr;     // end of the last launched seed run (pmf_seed_launch's `after`)
    bool launched = false;             // a seed run was launched and not yet waited for
    bool prepped = false;              // seed_prep_t ran for the run being launched
    struct Geom {
        int grid_push = 0, grid_bfs = 0, grid_wbfs = 0;
        size_t smem_w = 0;
    } geom[2];                         // launch geometry per residual policy (U8, I32), computed once
    int64_t launch_h2d = 0;
    pmf_stats stats{};
    int edge_bytes = 4;
    Pool *pool = nullptr;
    int use_graph = 1;                 // whole solve as one CUDA graph
    cudaGraphExec_t gexec = nullptr;   // cached instantiated solve graph
    unsigned char gkey[1024] = {0};    // GraphKey it was built for

    int ev_get(cudaEvent_t *e) {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t x;
            CK(cudaEventCreate(&x));
            ev_pool.push_back(x);
        }
        *e = ev_pool[ev_used++];
        return 0;
    }
    // mark the start of a timed region of category cat (timing mode only)
    void tmark(int cat) {
        if (!timing) return;
        cudaEvent_t e;
        if (ev_get(&e)) return;
        cudaEventRecord(e, st);
        ev_marks.push_back({cat, int(ev_used - 1)});
    }
};

// every kernel launch of a run goes through LAUNCH (counted in stats.launches)
#define LAUNCH(s, ...)           \
    do {                         \
        __VA_ARGS__;             \
        (s)->stats.launches++;   \
    } while (0)

namespace {

int setup_state(pmf_solver *s, int edge_bytes) {
    const Layout &L = s->lay;
    const int64_t T = L.ntiles, P = T * TPIX, G = int64_t(L.grids.size());
    if (T >= (int64_t(1) << 31) / 2) return fail(PMF_ERR_ARG, "batch too large (%lld tiles)", (long long)T);
    int rc = 0;
    if ((rc = s->d_w.ensure(P * 4)) || (rc = s->d_h.ensure(P * 4)) ||
        (rc = s->d_r.ensure(P * size_t(edge_bytes))) || (rc = s->d_lab.ensure(P)) ||
        (rc = s->d_tile_grid.ensure(T * 4)) || (rc = s->d_tnb.ensure(T * 16)) || (rc = s->d_grids.ensure(G * sizeof(GridDesc))) ||
        (rc = s->d_live.ensure(G * 4)) || (rc = s->d_fin.ensure(G * 4)) || (rc = s->d_gpend.ensure(G * 4)) || (rc = s->d_specg.ensure(G * 4)) || (rc = s->d_keeph.ensure(G * 4)) || (rc = s->d_labok.ensure(G * 4)) || (rc = s->d_act.ensure(G * 4)) ||
        (rc = s->d_list.ensure(2 * T * 4)) || (rc = s->d_inq.ensure(2 * T * 4)) ||
        (rc = s->d_cnt.ensure(64)) || (rc = s->d_snk.ensure(G * 8)) || (rc = s->d_drain.ensure(G * 8)) ||
        (rc = s->d_err.ensure(64)) || (rc = s->d_stat.ensure(ST_NSTAT * 8)) ||
        (rc = s->d_out.ensure(std::max<int64_t>(L.out_bytes, 1))) || (rc = s->d_colswap.ensure(64)) ||
        (rc = s->d_swapflag.ensure(64)) || (rc = s->d_ring.ensure(T * 4)) ||
        (rc = s->d_qstate.ensure(T * 4)) || (rc = s->d_qctr.ensure(64)) ||
        (rc = s->d_ctl.ensure(sizeof(Ctl))) || (rc = s->d_curlam.ensure(G * 4)))
        return rc;
    s->edge_bytes = edge_bytes;
    s->warp_eff = s->warp;
    // host sources live in the solver (s->lay, s->ones) until the next setup
    CK(cudaMemcpyAsync(s->d_tile_grid.p, L.tile_grid.data(), T * 4, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_tnb.p, L.tile_nb.data(), T * 16, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_grids.p, L.grids.data(), G * sizeof(GridDesc), cudaMemcpyHostToDevice, s->st));
    s->ones.assign(size_t(G), 1);
    CK(cudaMemcpyAsync(s->d_live.p, s->ones.data(), G * 4, cudaMemcpyHostToDevice, s->st));
    s->curlam0.resize(size_t(G));
    for (int64_t g = 0; g < G; g++) s->curlam0[g] = L.grids[g].lam;
    CK(cudaMemcpyAsync(s->d_curlam.p, s->curlam0.data(), G * 4, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemsetAsync(s->d_act.p, 0, G * 4, s->st));
    CK(cudaMemsetAsync(s->d_fin.p, 0, G * 4, s->st));
    CK(cudaMemsetAsync(s->d_gpend.p, 0, G * 4, s->st));
    CK(cudaMemsetAsync(s->d_specg.p, 0, G * 4, s->st));
    CK(cudaMemsetAsync(s->d_keeph.p, 0, G * 4, s->st));
    CK(cudaMemsetAsync(s->d_labok.p, 0, G * 4, s->st));
    CK(cudaMemsetAsync(s->d_snk.p, 0, G * 8, s->st));
    CK(cudaMemsetAsync(s->d_drain.p, 0, G * 8, s->st));
    CK(cudaMemsetAsync(s->d_err.p, 0, 64, s->st));
    CK(cudaMemsetAsync(s->d_stat.p, 0, ST_NSTAT * 8, s->st));
    Ctx &x = s->ctx;
    x = Ctx{};
    x.w = s->d_w.as<int32_t>();
    x.h = s->d_h.as<int32_t>();
    x.r = s->d_r.p;
    x.lab = s->d_lab.as<uint8_t>();
    x.tile_grid = s->d_tile_grid.as<int32_t>();
    x.tnb = s->d_tnb.as<int4>();
    x.grids = s->d_grids.as<GridDesc>();
    x.live = s->d_live.as<int32_t>();
    x.fin = s->d_fin.as<int32_t>();
    x.push_flush = s->push_flush;
    x.tfresh = nullptr;
    if (s->fresh_skip) {
        if ((rc = s->d_tfresh.ensure(size_t(T)))) return rc;
        CK(cudaMemsetAsync(s->d_tfresh.p, 0, size_t(T), s->st));
        x.tfresh = s->d_tfresh.as<uint8_t>();
    }
    x.gpend = s->d_gpend.as<int32_t>();
    x.specg = nullptr;   // set by seed_run_t in rolling mode
    x.keeph = nullptr;   // set by seed_run_t for warm chains
    x.labok = nullptr;   // ... as is the nested label seeding
    x.ngrids = int32_t(G);
    x.rolling = 0;
    x.act = s->d_act.as<int32_t>();
    x.list0 = s->d_list.as<int32_t>();
    x.list1 = x.list0 + T;
    x.inq0 = s->d_inq.as<int32_t>();
    x.inq1 = x.inq0 + T;
    x.cnt = s->d_cnt.as<int32_t>();
    x.snk_sum = s->d_snk.as<int64_t>();
    x.drain = s->d_drain.as<int64_t>();
    x.err = s->d_err.as<int32_t>();
    x.stat = s->d_stat.as<unsigned long long>();
    x.colswap = s->d_colswap.as<uint8_t>();
    x.swapflag = s->d_swapflag.as<int32_t>();
    x.out = s->d_out.as<uint8_t>();
    x.ntiles = T;
    x.ring = s->d_ring.as<int32_t>();
    x.qstate = s->d_qstate.as<int32_t>();
    x.qctr = s->d_qctr.as<unsigned int>();
    x.qcap = int32_t(T);
    x.persistent = s->persistent;
    x.ctl = s->d_ctl.as<Ctl>();
    x.budget_dev = 0;
    x.cur_lam = s->d_curlam.as<int32_t>();
    x.flows = s->d_flows.as<int64_t>();
    x.nlam = s->stage.nlam;
    // BFS phases converge on their own (values only decrease); the cap only
    // guards against a runaway launch
    x.budget = unsigned(std::min<int64_t>(int64_t(4096) * T + 4096, int64_t(0xffffffffu) - 1));
    return 0;
}

int read_count(pmf_solver *s, const Ctx &c, int idx, int32_t *out) {
    int32_t *hp = s->h_small.as<int32_t>();
    CK(cudaMemcpyAsync(hp, c.cnt + idx, 4, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    *out = *hp;
    return 0;
}

int read_ctl(pmf_solver *s, const Ctx &c, Ctl *out) {
    Ctl *hp = s->h_small.as<Ctl>();
    CK(cudaMemcpyAsync(hp, c.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    *out = *hp;
    return 0;
}

// discharge pop budget per seeded tile (warm-start steps start closer to
// the answer and profit from longer discharges between global relabels)
inline int budget_factor(const pmf_solver *s) {
    return s->warm_active ? s->push_budget_warm : s->push_budget;
}

inline LaunchCtl lctl(int stat, cudaGraphConditionalHandle h = 0, int has = 0, int max_k = 0) {
    LaunchCtl l;
    l.stat = stat;
    l.cond = h;
    l.has_cond = has;
    l.max_k = max_k;
    return l;
}

// Per-phase scheduling contexts: the BFS phases and the discharge phase can
// each run as launch-per-sweep worklists or as one persistent launch.
struct PhaseCtx {
    Ctx base, bfs, push, pq;   // pq: persistent discharge with device budget
};

PhaseCtx phase_ctx(pmf_solver *s, const Ctx &c0) {
    PhaseCtx p;
    p.base = c0;
    p.bfs = c0;
    p.bfs.persistent = s->persistent_bfs;
    p.push = c0;
    p.push.persistent = s->persistent;
    p.pq = p.push;
    p.pq.budget_dev = 1;
    return p;
}

// ---- tile-kernel launchers: warp-per-tile kernels (default) or the
// 1024-thread-CTA kernels
// cooperative launch (every CTA co-resident) for the K_MULTI kernels
template <class... KArgs, class... Args>
cudaError_t launch_coop(void (*f)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, f, args...);
}

template <class E>
void launch_bfs(pmf_solver *s, const Ctx &c, bool sink, int k) {
    if (k == K_MULTI) {
        const LaunchCtl lc = lctl(sink ? ST_BFS : ST_LAB);
        cudaError_t e;
        if (!sink && (s->warp_eff & 4))
            e = launch_coop(k_wbfs_src<E>, s->grid_wbfs, WPB * 32, s->smem_w, s->st, c, k, lc);
        else
            e = launch_coop(sink ? k_bfs_sink<E> : k_bfs_src<E>, s->grid_bfs, NTT, 0, s->st, c, k, lc);
        (void)e;   // surfaced by the caller's cudaGetLastError
        s->stats.launches++;
        return;
    }
    if (!sink && (s->warp_eff & 4)) {
        LAUNCH(s, (k_wbfs_src<E><<<s->grid_wbfs, WPB * 32, s->smem_w, s->st>>>(c, k, lctl(ST_LAB))));
    } else {
        if (sink) LAUNCH(s, (k_bfs_sink<E><<<s->grid_bfs, NTT, 0, s->st>>>(c, k, lctl(ST_BFS))));
        else LAUNCH(s, (k_bfs_src<E><<<s->grid_bfs, NTT, 0, s->st>>>(c, k, lctl(ST_LAB))));
    }
}

// CTA discharge kernel: 2 CTAs per SM at 32 registers
template <class E>
void launch_push(pmf_solver *s, const Ctx &c, int k) {
    LAUNCH(s, (k_push<E><<<s->grid_push, NTT, 0, s->st>>>(c, k, s->push_iters, s->relabel_every, lctl(ST_PUSH))));
}

// ---- host-driven loop (graph = 0): the host reads worklist lengths and the
// control block between phases
template <class E>
int host_bfs(pmf_solver *s, const Ctx &c, bool sink) {
    if (c.persistent) {   // one launch; the queue drains on the device
        launch_bfs<E>(s, c, sink, K_PERSISTENT);
        CK(cudaGetLastError());
        return 0;
    }
    if (s->bfs_multi) {   // one cooperative launch runs every sweep
        launch_bfs<E>(s, c, sink, K_MULTI);
        CK(cudaGetLastError());
        return 0;
    }
    int k = 0;
    for (;;) {
        for (int j = 0; j < s->bfs_chunk; j++, k++) launch_bfs<E>(s, c, sink, k);
        CK(cudaGetLastError());
        int32_t left = 0;
        int rc = read_count(s, c, k % 3, &left);
        if (rc) return rc;
        if (left == 0) return 0;
    }
}

template <class E>
int host_solve(pmf_solver *s, const Ctx &c0, int32_t ngrids) {
    PhaseCtx P = phase_ctx(s, c0);
    int rc = 0;
    for (;;) {
        // exact global relabel
        s->tmark(C_BFS);
        LAUNCH(s, (k_phase_begin<<<s->grid_full, 256, 0, s->st>>>(P.bfs, P.bfs.persistent, 0, 0)));
        LAUNCH(s, (k_gr_init<<<s->grid_full, NT, 0, s->st>>>(P.bfs)));
        s->stats.full_passes++;
        if ((rc = host_bfs<E>(s, P.bfs, true))) return rc;
        // list active tiles; retire grids without active pixels
        s->tmark(C_SEED);
        LAUNCH(s, (k_phase_begin<<<s->grid_full, 256, 0, s->st>>>(P.push, P.push.persistent, 0, 0)));
        LAUNCH(s, (k_seed_push<<<s->grid_full, NT, 0, s->st>>>(P.push)));
        LAUNCH(s, (k_cycle_ctl<<<1, 1024, 0, s->st>>>(P.push, ngrids, P.push.persistent,
                                                      unsigned(budget_factor(s)), s->max_cycles, 0, 0, 0, 0)));
        CK(cudaGetLastError());
        s->stats.full_passes++;
        Ctl ctl;
        if ((rc = read_ctl(s, c0, &ctl))) return rc;
        if (ctl.noconv)
            return fail(PMF_ERR_NOCONV, "push-relabel failed to converge within %lld cycles",
                        (long long)s->max_cycles);
        if (ctl.nact == 0) break;
        s->tmark(C_PUSH);
        if (P.push.persistent) {
            launch_push<E>(s, P.pq, K_PERSISTENT);
            CK(cudaGetLastError());
            continue;
        }
        // discharge until no tile is listed (or the per-cycle sweep cap)
        for (int k = 0; k < s->push_sweeps;) {
            int chunk = std::min(s->bfs_chunk, s->push_sweeps - k);
            for (int j = 0; j < chunk; j++, k++) launch_push<E>(s, P.push, k);
            CK(cudaGetLastError());
            int32_t left = 0;
            if ((rc = read_count(s, P.push, k % 3, &left))) return rc;
            if (left == 0) break;
        }
    }
    // labels: source-side closure, then emit
    s->tmark(C_LAB);
    LAUNCH(s, (k_phase_begin<<<s->grid_full, 256, 0, s->st>>>(P.bfs, P.bfs.persistent, 0, 0)));
    LAUNCH(s, (k_lab_seed<<<s->grid_full, NT, 0, s->st>>>(P.bfs)));
    s->stats.full_passes++;
    if ((rc = host_bfs<E>(s, P.bfs, false))) return rc;
    LAUNCH(s, (k_emit<<<s->grid_full, NT, 0, s->st>>>(P.base)));
    s->stats.full_passes++;
    CK(cudaGetLastError());
    return 0;
}

// ---- graph-driven loop (graph = 1): the whole solve is one CUDA graph with
// conditional while nodes; loop decisions are taken on the device
// (k_cycle_ctl, last CTA of every sweep) and the host never synchronises
// mid-solve.
template <class F, class... Args>
int add_kernel_smem(cudaGraph_t g, cudaGraphNode_t *prev, dim3 grid, dim3 block, size_t smem, F func,
                    Args... args) {
    void *ptrs[] = {(void *)&args...};
    cudaKernelNodeParams kp{};
    kp.func = (void *)func;
    kp.gridDim = grid;
    kp.blockDim = block;
    kp.sharedMemBytes = unsigned(smem);
    kp.kernelParams = ptrs;
    cudaGraphNode_t n;
    CK(cudaGraphAddKernelNode(&n, g, *prev ? prev : nullptr, *prev ? 1 : 0, &kp));
    *prev = n;
    return 0;
}

template <class F, class... Args>
int add_kernel(cudaGraph_t g, cudaGraphNode_t *prev, dim3 grid, dim3 block, F func, Args... args) {
    void *ptrs[] = {(void *)&args...};
    cudaKernelNodeParams kp{};
    kp.func = (void *)func;
    kp.gridDim = grid;
    kp.blockDim = block;
    kp.kernelParams = ptrs;
    cudaGraphNode_t n;
    CK(cudaGraphAddKernelNode(&n, g, *prev ? prev : nullptr, *prev ? 1 : 0, &kp));
    *prev = n;
    return 0;
}

// appends a while node to g (after *prev); returns its body graph
int add_while(cudaGraph_t g, cudaGraphNode_t *prev, cudaGraphConditionalHandle h, cudaGraph_t *body) {
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t n;
    CK(cudaGraphAddNode(&n, g, *prev ? prev : nullptr, *prev ? 1 : 0, &p));
    *body = p.conditional.phGraph_out[0];
    *prev = n;
    return 0;
}

// appends an if node to g (after *prev); returns its body graph
int add_if(cudaGraph_t g, cudaGraphNode_t *prev, cudaGraphConditionalHandle h, cudaGraph_t *body) {
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t n;
    CK(cudaGraphAddNode(&n, g, *prev ? prev : nullptr, *prev ? 1 : 0, &p));
    *body = p.conditional.phGraph_out[0];
    *prev = n;
    return 0;
}

template <class E>
int add_bfs_node_raw(pmf_solver *s, cudaGraph_t g, cudaGraphNode_t *prev, bool sink, const Ctx &c, int k,
                     LaunchCtl lc) {
    if (!sink && (s->warp_eff & 4))
        return add_kernel_smem(g, prev, dim3(s->grid_wbfs), dim3(WPB * 32), s->smem_w, k_wbfs_src<E>, c, k, lc);
    if (sink) return add_kernel(g, prev, dim3(s->grid_bfs), dim3(NTT), k_bfs_sink<E>, c, k, lc);
    return add_kernel(g, prev, dim3(s->grid_bfs), dim3(NTT), k_bfs_src<E>, c, k, lc);
}

template <class E>
int add_bfs_node(pmf_solver *s, cudaGraph_t g, cudaGraphNode_t *prev, bool sink, const Ctx &c, int k,
                 LaunchCtl lc) {
    int rc = add_bfs_node_raw<E>(s, g, prev, sink, c, k, lc);
    if (rc || k != K_MULTI) return rc;
    cudaLaunchAttributeValue v{};
    v.cooperative = 1;
    CK(cudaGraphKernelNodeSetAttribute(*prev, cudaLaunchAttributeCooperative, &v));
    return 0;
}

template <class E>
int add_push_node(pmf_solver *s, cudaGraph_t g, cudaGraphNode_t *prev, const Ctx &c, int k, LaunchCtl lc) {
    return add_kernel(g, prev, dim3(s->grid_push), dim3(NTT), k_push<E>, c, k, s->push_iters, s->relabel_every, lc);
}

template <class E>
int build_graph(pmf_solver *s, const Ctx &c0, int32_t ngrids, const SeedArgs *sa, const int64_t *slope_sum,
                cudaGraph_t *out) {
    PhaseCtx P = phase_ctx(s, c0);
    cudaGraph_t root;
    CK(cudaGraphCreate(&root, 0));
    *out = root;
    int rc;
    const dim3 gfull(s->grid_full);
    // warm-start steps: one iteration per lambda of the longest chain
    cudaGraphConditionalHandle h_step;
    CK(cudaGraphConditionalHandleCreate(&h_step, root, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t rprev = nullptr;
    cudaGraph_t g;
    if ((rc = add_while(root, &rprev, h_step, &g))) return rc;
    cudaGraphNode_t prev = nullptr;
    cudaGraphConditionalHandle h_cycle;
    CK(cudaGraphConditionalHandleCreate(&h_cycle, g, 0, 0));
    if ((rc = add_kernel(g, &prev, dim3(1), dim3(1), k_arm, h_cycle))) return rc;
    cudaGraph_t cyc;
    if ((rc = add_while(g, &prev, h_cycle, &cyc))) return rc;
    {   // ---- one cycle: exact global relabel, seeding, discharge
        cudaGraphNode_t q = nullptr;
        cudaGraphConditionalHandle h_bfs = 0, h_push = 0;
        const bool bfs_loop = !P.bfs.persistent && !s->bfs_multi;
        if (bfs_loop) CK(cudaGraphConditionalHandleCreate(&h_bfs, cyc, 0, 0));
        if ((rc = add_kernel(cyc, &q, gfull, dim3(256), k_phase_begin, P.bfs, int(P.bfs.persistent), h_bfs,
                             int(bfs_loop))))
            return rc;
        if ((rc = add_kernel(cyc, &q, gfull, dim3(NT), k_gr_init, P.bfs))) return rc;
        if (P.bfs.persistent) {
            if ((rc = add_bfs_node<E>(s, cyc, &q, true, P.bfs, K_PERSISTENT, lctl(ST_BFS)))) return rc;
        } else if (s->bfs_multi) {
            if ((rc = add_bfs_node<E>(s, cyc, &q, true, P.bfs, K_MULTI, lctl(ST_BFS)))) return rc;
        } else {
            cudaGraph_t body;
            if ((rc = add_while(cyc, &q, h_bfs, &body))) return rc;
            cudaGraphNode_t b = nullptr;
            if ((rc = add_bfs_node<E>(s, body, &b, true, P.bfs, K_DEVICE, lctl(ST_BFS, h_bfs, 1)))) return rc;
        }
        if (!P.push.persistent) CK(cudaGraphConditionalHandleCreate(&h_push, cyc, 0, 0));
        if ((rc = add_kernel(cyc, &q, gfull, dim3(256), k_phase_begin, P.push, int(P.push.persistent), h_push,
                             int(!P.push.persistent))))
            return rc;
        if ((rc = add_kernel(cyc, &q, gfull, dim3(NT), k_seed_push, P.push))) return rc;
        if ((rc = add_kernel(cyc, &q, dim3(1), dim3(1024), k_cycle_ctl, P.push, ngrids, int(P.push.persistent),
                             unsigned(budget_factor(s)), int64_t(s->max_cycles), h_cycle, 1,
                             cudaGraphConditionalHandle(0), 0)))
            return rc;
        if (P.push.persistent) {
            if ((rc = add_push_node<E>(s, cyc, &q, P.pq, K_PERSISTENT, lctl(ST_PUSH)))) return rc;
        } else {
            // k_phase_begin armed h_push = 1; an empty list ends the loop
            // after its first (idle) sweep
            cudaGraph_t body;
            if ((rc = add_while(cyc, &q, h_push, &body))) return rc;
            cudaGraphNode_t b = nullptr;
            if ((rc = add_push_node<E>(s, body, &b, P.push, K_DEVICE, lctl(ST_PUSH, h_push, 1, s->push_sweeps))))
                return rc;
        }
    }
    // ---- labels
    cudaGraphConditionalHandle h_lab = 0;
    const bool lab_loop = !P.bfs.persistent && !s->bfs_multi;
    if (lab_loop) CK(cudaGraphConditionalHandleCreate(&h_lab, g, 0, 0));
    if ((rc = add_kernel(g, &prev, gfull, dim3(256), k_phase_begin, P.bfs, int(P.bfs.persistent), h_lab,
                         int(lab_loop))))
        return rc;
    if ((rc = add_kernel(g, &prev, gfull, dim3(NT), k_lab_seed, P.bfs))) return rc;
    if (P.bfs.persistent) {
        if ((rc = add_bfs_node<E>(s, g, &prev, false, P.bfs, K_PERSISTENT, lctl(ST_LAB)))) return rc;
    } else if (s->bfs_multi) {
        if ((rc = add_bfs_node<E>(s, g, &prev, false, P.bfs, K_MULTI, lctl(ST_LAB)))) return rc;
    } else {
        cudaGraph_t body;
        if ((rc = add_while(g, &prev, h_lab, &body))) return rc;
        cudaGraphNode_t b = nullptr;
        if ((rc = add_bfs_node<E>(s, body, &b, false, P.bfs, K_DEVICE, lctl(ST_LAB, h_lab, 1)))) return rc;
    }
    if ((rc = add_kernel(g, &prev, gfull, dim3(NT), k_emit, P.base))) return rc;
    if ((rc = add_kernel(g, &prev, dim3(std::max(1, int(cdiv(ngrids, 256)))), dim3(256), k_finalize, P.base, ngrids)))
        return rc;
    SeedArgs none{};
    if (sa && (rc = add_kernel(g, &prev, gfull, dim3(NT), k_advance_tiles, P.base, *sa))) return rc;
    if ((rc = add_kernel(g, &prev, dim3(1), dim3(1024), k_advance_grids, P.base, sa ? *sa : none, slope_sum, ngrids,
                         h_step, 1)))
        return rc;
    return 0;
}

// Rolling warm start (graph mode): one cycle loop for the whole batch.
// Every cycle relabels and discharges the live grids; the grids that ran out
// of active pixels in it (k_cycle_ctl marks them `fin`) get their labels,
// flow and next lambda in the same cycle and rejoin the live set -- chains
// no longer wait for the slowest grid of a common step.
template <class E>
int build_graph_rolling(pmf_solver *s, const Ctx &c0, int32_t ngrids, const SeedArgs *sa,
                        const int64_t *slope_sum, cudaGraph_t *out) {
    PhaseCtx P = phase_ctx(s, c0);
    cudaGraph_t root;
    CK(cudaGraphCreate(&root, 0));
    *out = root;
    int rc;
    const dim3 gfull(s->grid_full);
    const int bfs_k = P.bfs.persistent ? K_PERSISTENT : K_MULTI;
    cudaGraphConditionalHandle h_cycle;
    CK(cudaGraphConditionalHandleCreate(&h_cycle, root, 0, 0));
    cudaGraphNode_t prev = nullptr;
    if ((rc = add_kernel(root, &prev, dim3(1), dim3(1), k_arm, h_cycle))) return rc;
    cudaGraph_t cyc;
    if ((rc = add_while(root, &prev, h_cycle, &cyc))) return rc;
    cudaGraphConditionalHandle h_lab;
    CK(cudaGraphConditionalHandleCreate(&h_lab, cyc, 0, cudaGraphCondAssignDefault));
    cudaGraphNode_t q = nullptr;
    const cudaGraphConditionalHandle none = 0;
    // exact global relabel of the live grids
    if ((rc = add_kernel(cyc, &q, gfull, dim3(256), k_phase_begin, P.bfs, int(P.bfs.persistent), none, 0))) return rc;
    if ((rc = add_kernel(cyc, &q, gfull, dim3(NT), k_gr_init, P.bfs))) return rc;
    if ((rc = add_bfs_node<E>(s, cyc, &q, true, P.bfs, bfs_k, lctl(ST_BFS)))) return rc;
    // seeding, retire / finish grids, discharge
    if ((rc = add_kernel(cyc, &q, gfull, dim3(256), k_phase_begin, P.push, 1, none, 0))) return rc;
    if ((rc = add_kernel(cyc, &q, gfull, dim3(NT), k_seed_push, P.push))) return rc;
    if ((rc = add_kernel(cyc, &q, dim3(1), dim3(1024), k_cycle_ctl, P.push, ngrids, 1, unsigned(budget_factor(s)),
                         int64_t(s->max_cycles), h_cycle, 1, h_lab, 1)))
        return rc;
    if ((rc = add_push_node<E>(s, cyc, &q, P.pq, K_PERSISTENT, lctl(ST_PUSH)))) return rc;
    if (c0.specg && (rc = add_kernel(cyc, &q, dim3(1), dim3(1024), k_push_spec, P.base, ngrids, h_cycle, 1, h_lab, 1)))
        return rc;
    // finished grids: labels, flow, next lambda
    cudaGraph_t lab;
    if ((rc = add_if(cyc, &q, h_lab, &lab))) return rc;
    cudaGraphNode_t l = nullptr;
    if ((rc = add_kernel(lab, &l, gfull, dim3(256), k_phase_begin, P.bfs, int(P.bfs.persistent), none, 0))) return rc;
    if ((rc = add_kernel(lab, &l, gfull, dim3(NT), k_lab_seed, P.bfs))) return rc;
    if ((rc = add_bfs_node<E>(s, lab, &l, false, P.bfs, bfs_k, lctl(ST_LAB)))) return rc;
    if (c0.specg && (rc = add_kernel(lab, &l, dim3(1), dim3(1024), k_unspoil, P.base, ngrids))) return rc;
    // label bytes + warm-start advance of the finished grids in one pass
    if ((rc = add_kernel(lab, &l, gfull, dim3(NT), k_emit_advance, P.base, *sa))) return rc;
    if ((rc = add_kernel(lab, &l, dim3(std::max(1, int(cdiv(ngrids, 256)))), dim3(256), k_finalize, P.base, ngrids)))
        return rc;
    if ((rc = add_kernel(lab, &l, dim3(1), dim3(1024), k_advance_grids, P.base, *sa, slope_sum, ngrids, h_cycle, 1)))
        return rc;
    return 0;
}

// knobs + context a cached graph was built for
struct GraphKey {
    Ctx ctx;
    int32_t ngrids, edge, p_push, p_bfs, iters, relabel, budget, sweeps, warp, multi;
    int64_t maxc;
    int32_t gfull, gbfs, gpush;
    SeedArgs sa;
    const int64_t *slope_sum;
    int32_t has_sa;
};

template <class E>
int graph_solve(pmf_solver *s, const Ctx &c0, int32_t ngrids, const SeedArgs *sa, const int64_t *slope_sum) {
    static_assert(sizeof(GraphKey) <= sizeof(pmf_solver::gkey), "graph key buffer too small");
    GraphKey key;
    memset(&key, 0, sizeof key);
    key.ctx = c0;
    key.ngrids = ngrids;
    key.edge = E::kBytes;
    key.p_push = s->persistent;
    key.p_bfs = s->persistent_bfs;
    key.iters = s->push_iters;
    key.relabel = s->relabel_every;
    key.budget = budget_factor(s);
    key.sweeps = s->push_sweeps;
    key.warp = s->warp_eff;
    key.multi = s->bfs_multi;
    key.maxc = s->max_cycles;
    key.gfull = s->grid_full;
    key.gbfs = s->grid_bfs;
    key.gpush = s->grid_push;
    if (sa) key.sa = *sa;
    key.slope_sum = slope_sum;
    key.has_sa = sa != nullptr;
    if (!s->gexec || memcmp(&key, s->gkey, sizeof key) != 0) {
        if (s->gexec) cudaGraphExecDestroy(s->gexec);
        s->gexec = nullptr;
        cudaGraph_t g = nullptr;
        int rc = c0.rolling ? build_graph_rolling<E>(s, c0, ngrids, sa, slope_sum, &g)
                            : build_graph<E>(s, c0, ngrids, sa, slope_sum, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        cudaError_t e = cudaGraphInstantiate(&s->gexec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(PMF_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
        memcpy(s->gkey, &key, sizeof key);
        s->stats.graph_builds++;
    }
    CK(cudaGraphLaunch(s->gexec, s->st));
    s->stats.launches++;
    return 0;
}

// Rolling warm start, host-driven (graph = 0): same kernels and order as
// build_graph_rolling, loop decisions read back from the control block.
template <class E>
int host_solve_rolling(pmf_solver *s, const Ctx &c0, int32_t ngrids, const SeedArgs &sa, const int64_t *slope_sum) {
    PhaseCtx P = phase_ctx(s, c0);
    const int gfin = std::max(1, int(cdiv(ngrids, 256)));
    int rc = 0;
    for (;;) {
        s->tmark(C_BFS);
        LAUNCH(s, (k_phase_begin<<<s->grid_full, 256, 0, s->st>>>(P.bfs, P.bfs.persistent, 0, 0)));
        LAUNCH(s, (k_gr_init<<<s->grid_full, NT, 0, s->st>>>(P.bfs)));
        if ((rc = host_bfs<E>(s, P.bfs, true))) return rc;
        s->tmark(C_SEED);
        LAUNCH(s, (k_phase_begin<<<s->grid_full, 256, 0, s->st>>>(P.push, 1, 0, 0)));
        LAUNCH(s, (k_seed_push<<<s->grid_full, NT, 0, s->st>>>(P.push)));
        LAUNCH(s, (k_cycle_ctl<<<1, 1024, 0, s->st>>>(P.push, ngrids, 1, unsigned(budget_factor(s)), s->max_cycles,
                                                      0, 0, 0, 0)));
        CK(cudaGetLastError());
        Ctl ctl;
        if ((rc = read_ctl(s, c0, &ctl))) return rc;
        if (ctl.noconv)
            return fail(PMF_ERR_NOCONV, "push-relabel failed to converge within %lld cycles",
                        (long long)s->max_cycles);
        if (ctl.nact) {
            s->tmark(C_PUSH);
            launch_push<E>(s, P.pq, K_PERSISTENT);
            if (c0.specg) LAUNCH(s, (k_push_spec<<<1, 1024, 0, s->st>>>(c0, ngrids, 0, 0, 0, 0)));
            CK(cudaGetLastError());
            if ((rc = read_ctl(s, c0, &ctl))) return rc;
        }
        if (!ctl.nfin) {
            if (!ctl.nact) break;
            continue;
        }
        s->tmark(C_LAB);
        LAUNCH(s, (k_phase_begin<<<s->grid_full, 256, 0, s->st>>>(P.bfs, P.bfs.persistent, 0, 0)));
        LAUNCH(s, (k_lab_seed<<<s->grid_full, NT, 0, s->st>>>(P.bfs)));
        if ((rc = host_bfs<E>(s, P.bfs, false))) return rc;
        if (c0.specg) LAUNCH(s, (k_unspoil<<<1, 1024, 0, s->st>>>(c0, ngrids)));
        LAUNCH(s, (k_emit_advance<<<s->grid_full, NT, 0, s->st>>>(P.base, sa)));
        LAUNCH(s, (k_finalize<<<gfin, 256, 0, s->st>>>(c0, ngrids)));
        LAUNCH(s, (k_advance_grids<<<1, 1024, 0, s->st>>>(c0, sa, slope_sum, ngrids, 0, 0)));
        CK(cudaGetLastError());
        if ((rc = read_ctl(s, c0, &ctl))) return rc;
        if (!ctl.more) break;
    }
    return 0;
}

template <class E>
int run_solve(pmf_solver *s, const Ctx &c0, int32_t ngrids, const SeedArgs *sa = nullptr,
              const int64_t *slope_sum = nullptr) {
    CK(cudaMemsetAsync(c0.ctl, 0, sizeof(Ctl), s->st));
    if (c0.rolling && !s->use_graph) return host_solve_rolling<E>(s, c0, ngrids, *sa, slope_sum);
    if (s->use_graph) return graph_solve<E>(s, c0, ngrids, sa, slope_sum);
    const int gfin = std::max(1, int(cdiv(ngrids, 256)));
    for (;;) {   // warm-start steps
        int rc = host_solve<E>(s, c0, ngrids);
        if (rc) return rc;
        LAUNCH(s, (k_finalize<<<gfin, 256, 0, s->st>>>(c0, ngrids)));
        if (!sa) break;
        LAUNCH(s, (k_advance_tiles<<<s->grid_full, NT, 0, s->st>>>(c0, *sa)));
        LAUNCH(s, (k_advance_grids<<<1, 1024, 0, s->st>>>(c0, *sa, slope_sum, ngrids, 0, 0)));
        CK(cudaGetLastError());
        Ctl ctl;
        if ((rc = read_ctl(s, c0, &ctl))) return rc;
        if (ctl.noconv || !ctl.more) break;
    }
    return 0;
}

// Device-side run bracket: always-on events around the whole run give
// ms_device; timing mode adds per-phase marks.
int run_begin(pmf_solver *s) {
    s->stats = pmf_stats{};
    s->ev_used = 0;
    s->ev_marks.clear();
    CK(cudaEventRecord(s->ev_run[0], s->st));
    return 0;
}

int run_end(pmf_solver *s) {
    s->tmark(C_N);
    CK(cudaEventRecord(s->ev_run[1], s->st));
    unsigned long long st[ST_NSTAT];
    int32_t err = 0;
    Ctl ctl;
    CK(cudaMemcpyAsync(st, s->d_stat.p, sizeof st, cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&err, s->d_err.p, 4, cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&ctl, s->d_ctl.p, sizeof ctl, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    const Layout &L = s->lay;
    s->stats.scan_tile_passes = int64_t(st[ST_BINIT] + st[ST_SEED] + st[ST_LINIT] + st[ST_EMIT]);
    s->stats.binit_tile_passes = int64_t(st[ST_BINIT]);
    s->stats.seed_tile_passes = int64_t(st[ST_SEED]);
    s->stats.linit_tile_passes = int64_t(st[ST_LINIT]);
    s->stats.emit_tile_passes = int64_t(st[ST_EMIT]);
    s->stats.ms_async = double(st[ST_ASYNC_NS]) * 1e-6;
    for (int k = 0; k < BUSY_N; k++) s->busy_ms[k] = double(st[ST_BUSY + k]) * 1e-6;
    s->busy_ms[15] = double(st[ST_PUSH_ITERS]);
    s->busy_ms[13] = double(st[ST_RELAX_NS]) * 1e-6;
    s->busy_ms[14] = double(st[ST_RELAX_N]);
    s->busy_ms[12] = double(st[ST_RELAX_SW]);
    s->spec_tries = int64_t(st[ST_SPEC]);
    s->spec_spoiled = int64_t(st[ST_SPOILED]);
    if (!s->stats.async_mode) {   // rolling mode's speculative label rounds
        s->spec_tries = int64_t(st[ST_SPEC_ROLL]);
        s->spec_spoiled = int64_t(st[ST_SPOIL_ROLL]);
    }
    s->stats.push_tile_passes = int64_t(st[ST_PUSH]);
    s->stats.bfs_tile_passes = int64_t(st[ST_BFS]);
    s->stats.label_tile_passes = int64_t(st[ST_LAB]);
    s->stats.push_sweeps = int64_t(st[ST_PUSH_L]);
    s->stats.bfs_sweeps = int64_t(st[ST_BFS_L] + st[ST_LAB_L]);
    s->stats.cycles = ctl.cycles_total;
    s->stats.steps = s->stats.async_mode ? int64_t(st[ST_LAMS]) : std::max(1, ctl.steps);
    // kernels executed on the device: the counted tile-kernel launches plus
    // the fixed per-cycle kernels (2 x phase_begin, gr_init, seed_push,
    // cycle_ctl), the label tail (phase_begin, lab_seed, emit) and the
    // build kernels (host-launched, counted in stats.launches)
    if (s->use_graph && !s->stats.async_mode)
        s->stats.kernels = int64_t(st[ST_PUSH_L] + st[ST_BFS_L] + st[ST_LAB_L]) + 5 * int64_t(ctl.cycles_total) +
                           7 * int64_t(std::max(1, ctl.steps)) + (s->stats.launches - 1);
    else
        s->stats.kernels = s->stats.launches;
    s->stats.grids = int64_t(L.grids.size());
    s->stats.tiles = L.ntiles;
    s->stats.pixels = L.pixels;
    s->stats.edge_bytes = s->edge_bytes;
    // device-clock spans of the tile kernels (always on, graph or not)
    s->stats.ms_push = double(st[ST_PUSH_NS]) * 1e-6;
    s->stats.ms_bfs = double(st[ST_BFS_NS]) * 1e-6;
    s->stats.ms_labels = double(st[ST_LAB_NS]) * 1e-6;
    float dev = 0;
    cudaEventElapsedTime(&dev, s->ev_run[0], s->ev_run[1]);
    s->stats.ms_device = dev;
    if (s->timing && !s->ev_marks.empty()) {
        double cat[C_N] = {0};
        for (size_t i = 0; i + 1 < s->ev_marks.size(); i++) {
            float ms = 0;
            cudaEventElapsedTime(&ms, s->ev_pool[s->ev_marks[i].second], s->ev_pool[s->ev_marks[i + 1].second]);
            cat[s->ev_marks[i].first] += ms;
        }
        s->stats.timed = 1;
        s->stats.ms_total = dev;
        s->stats.ms_build = cat[C_BUILD];
        s->stats.ms_seed = cat[C_SEED];
        s->stats.ms_h2d = cat[C_H2D];
        s->stats.ms_d2h = cat[C_D2H];
    }
    if (ctl.noconv)
        return fail(PMF_ERR_NOCONV, "push-relabel failed to converge within %lld cycles",
                    (long long)s->max_cycles);
    if (err == 4) return fail(PMF_ERR_NONMAX, "source side touches an unsaturated sink edge");
    if (err == 5) return fail(PMF_ERR_NONMAX, "a cut's cost differs from its flow (integrity check)");
    if (err) return fail(PMF_ERR_CUDA, "device error code %d", err);
    return 0;
}

// narrow an int64 plane into int32 staging, clamping into [lo, hi]
inline void narrow(int32_t *dst, const int64_t *src, int64_t n, int64_t lo, int64_t hi) {
    for (int64_t i = 0; i < n; i++) {
        int64_t v = src[i];
        dst[i] = int32_t(v < lo ? lo : v > hi ? hi : v);
    }
}

// largest c(p->q) + c(q->p) over the arc pairs leaving rows [y0, y1) of a
// (4, n) row-major plane set
int64_t max_pair(const int32_t *nb, int W, int H, int y0 = 0, int y1 = -1) {
    const int64_t n = int64_t(W) * H;
    int64_t m = 0;
    if (y1 < 0) y1 = H;
    for (int y = y0; y < y1; y++)
        for (int x = 0; x < W; x++) {
            int64_t p = int64_t(y) * W + x;
            if (x + 1 < W) m = std::max<int64_t>(m, int64_t(nb[1 * n + p]) + nb[0 * n + p + 1]);
            if (y + 1 < H) m = std::max<int64_t>(m, int64_t(nb[3 * n + p]) + nb[2 * n + p + W]);
        }
    return m;
}

template <class E>
int grids_for(pmf_solver *s) {
    // once per solver and residual policy: the occupancy queries and
    // cudaFuncSetAttribute wait for kernels running on the device, which
    // would block a batch stream's launch behind the previous run
    constexpr int kind = E::kBytes == 4 ? 0 : 1;
    if (s->geom[kind].grid_push) {
        s->grid_push = s->geom[kind].grid_push;
        s->grid_bfs = s->geom[kind].grid_bfs;
        s->grid_wbfs = s->geom[kind].grid_wbfs;
        s->smem_w = s->geom[kind].smem_w;
        s->grid_full = 8 * s->sms;
        return 0;
    }
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_push<E>, NTT, 0));
    s->grid_push = std::max(1, occ) * s->sms;
    // BFS grids are co-resident (cooperative K_MULTI launches): the smaller
    // occupancy of the sink and label kernels
    int occ2 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bfs_sink<E>, NTT, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_bfs_src<E>, NTT, 0));
    s->grid_bfs = std::max(1, std::min(occ, occ2)) * s->sms;
    s->smem_w = 0;   // the label closure holds its tile in registers
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_wbfs_src<E>, WPB * 32, s->smem_w));
    s->grid_wbfs = std::max(1, occ2) * s->sms;
    s->grid_full = 8 * s->sms;
    s->geom[kind] = {s->grid_push, s->grid_bfs, s->grid_wbfs, s->smem_w};
    return 0;
}

// --------------------------------------------------------------------------
// seed batches: stage (host convert + H2D) / run (device only) / fetch (D2H)
// --------------------------------------------------------------------------

// Integrity certificate of a seed batch (k_verify): cut cost of every
// emitted mask on the original graph == its flow
template <class E>
int launch_verify(pmf_solver *s, const Ctx &c, const SeedArgs &a) {
    const int64_t planes = int64_t(a.nprob) * a.nlam, n = int64_t(a.W) * a.H;
    // (problem, chunk) CTAs: ~4 rounds of NT * VPX pixels each
    const int64_t want = std::max<int64_t>(cdiv(n, int64_t(NT) * VPX * 4), cdiv(4 * s->sms, a.nprob));
    const int chunks = int(std::max<int64_t>(1, std::min<int64_t>({want, cdiv(n, int64_t(NT) * VPX), 4096})));
    if (n >= (int64_t(1) << 31)) return fail(PMF_ERR_ARG, "image too large for the integrity check (%lld pixels)", (long long)n);
    int rc;
    if ((rc = s->d_vacc.ensure(size_t(planes) * 8))) return rc;
    CK(cudaMemsetAsync(s->d_vacc.p, 0, size_t(planes) * 8, s->st));
    unsigned long long *acc = s->d_vacc.as<unsigned long long>();
    // verify=2 (test hook): flip the label of the centre pixel of (problem 0,
    // lambda 0) so the check must fail
    if (s->verify == 2) LAUNCH(s, (k_flip_label<<<1, 1, 0, s->st>>>(c.out, int64_t(a.H / 2) * a.W + a.W / 2)));
    constexpr bool narrow = std::is_same<E, EdgeU8>::value;
    if (a.W % 4 == 0 && s->verify_vec) {
        // 4-pixel groups: ~4 rounds of NT groups per CTA
        const int64_t n4 = n / 4;
        const int64_t w4 = std::max<int64_t>(cdiv(n4, int64_t(NT) * 4), cdiv(4 * s->sms, a.nprob));
        const int ch4 = int(std::max<int64_t>(1, std::min<int64_t>({w4, cdiv(n4, NT), 4096})));
        LAUNCH(s, (k_verify4<narrow><<<int(std::min<int64_t>(int64_t(a.nprob) * ch4, 32 * s->sms)), NT, 0, s->st>>>(
                       c, a, acc, ch4)));
    } else {
        LAUNCH(s, (k_verify<narrow><<<int(std::min<int64_t>(int64_t(a.nprob) * chunks, 32 * s->sms)), NT, 0, s->st>>>(
                       c, a, acc, chunks)));
    }
    LAUNCH(s, (k_verify_check<<<int(std::max<int64_t>(1, std::min<int64_t>(cdiv(planes, 256), 1024))), 256, 0, s->st>>>(
                   c, planes, acc)));
    CK(cudaGetLastError());
    return 0;
}

// Asynchronous seed batch (async.cuh): queue reset, every grid in BINIT with
// all its tiles queued, then one persistent launch runs every phase of
// every grid.
template <class E>
int async_solve(pmf_solver *s, const Ctx &c0, const SeedArgs &sa) {
    const int64_t G = int64_t(s->lay.grids.size()), T = s->lay.ntiles;
    int rc;
    if ((rc = s->d_gr.ensure(size_t(G) * sizeof(GridRun))) || (rc = s->d_tflag.ensure(size_t(T)))) return rc;
    Ctx c = c0;
    c.persistent = 1;
    c.budget = 0;       // no global pop budget: discharges are capped per grid
    c.budget_dev = 0;
    AsyncArgs A{};
    A.sa = sa;
    A.slope_sum = s->d_slopesum.as<int64_t>();
    A.gr = s->d_gr.as<GridRun>();
    A.tflag = s->d_tflag.as<uint8_t>();
    A.iters = s->push_iters;
    A.relabel_every = s->relabel_every;
    A.budget_factor = unsigned(budget_factor(s));
    A.budget_add = s->push_budget_add;
    A.max_cycles = int32_t(std::min<int64_t>(s->max_cycles, 0x7fffffff));
    A.cont = s->async_cont;
    A.prefetch = s->async_prefetch;
    A.spec = s->async_spec;
    A.keep_h = s->adv_keep_h && s->async_spec;   // kept heights need the speculative closure
    A.yield_ns = (unsigned long long)s->async_yield_us * 1000ull;
    A.yield_keep = s->async_yield_keep ? s->async_yield_keep : std::max(1, s->grid_push / 4);
    if (s->phase_log) {
        if ((rc = s->d_plog.ensure(size_t(G) * PLOG * 8))) return rc;
        CK(cudaMemsetAsync(s->d_plog.p, 0, size_t(G) * PLOG * 8, s->st));
        A.plog = s->d_plog.as<unsigned long long>();
        s->plog_grids = G;
    }
    CK(cudaMemsetAsync(c.ctl, 0, sizeof(Ctl), s->st));
    LAUNCH(s, (k_phase_begin<<<s->grid_full, 256, 0, s->st>>>(c, 1, 0, 0)));
    LAUNCH(s, (k_async_begin<<<s->grid_full, 256, 0, s->st>>>(c, A, int32_t(G))));
    LAUNCH(s, (k_async_queue_all<<<s->grid_full, 256, 0, s->st>>>(c)));
    LAUNCH(s, (k_async<E><<<s->grid_push, NTT, 0, s->st>>>(c, A)));
    CK(cudaGetLastError());
    s->stats.async_mode = 1;
    return 0;
}

// Kernel arguments of the staged seed batch (planes, offsets, lambdas).
SeedArgs seed_args(pmf_solver *s) {
    const SeedStage &S = s->stage;
    const int64_t n = int64_t(S.W) * S.H;
    const int32_t *b32 = s->d_in32.as<int32_t>();
    SeedArgs a{};
    a.base = b32;
    a.slope = b32 + n;
    a.sink = b32 + 2 * n;
    a.pw = s->d_pw.as<int32_t>();
    a.plane_off = s->d_off.as<int64_t>();
    a.pw_off = s->d_off.as<int64_t>() + S.nprob;
    a.lambdas = s->d_lam.as<int64_t>();
    a.nprob = S.nprob;
    a.nlam = S.nlam;
    a.W = S.W;
    a.H = S.H;
    a.mid = (S.nlam - 1) / 2;   // LambdaSchedule.mid_index, parametric.py:65-68
    a.swap_mode = S.swap_mode;
    a.swap_cnt = s->d_swapcnt.as<int32_t>();
    a.swapped = s->d_swapflag.as<int32_t>();
    a.mask = s->d_mask.as<uint8_t>();
    return a;
}

// Swap decision per problem (supergraph.py:210-212, 85-92) into d_swapflag.
int seed_swap_flags(pmf_solver *s, const SeedArgs &a) {
    const SeedStage &S = s->stage;
    const int64_t n = int64_t(S.W) * S.H;
    CK(cudaMemsetAsync(s->d_swapcnt.p, 0, size_t(S.nprob) * 8, s->st));
    if (S.swap_mode == PMF_SWAP_AUTO) {
        if (n >= (int64_t(1) << 31)) return fail(PMF_ERR_ARG, "image too large (%lld pixels)", (long long)n);
        const int chunks = int(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256 * 4), cdiv(8 * s->sms, S.nprob))));
        LAUNCH(s, (k_swap_count<<<int(std::min<int64_t>(int64_t(S.nprob) * chunks, 16 * s->sms)), 256, 0, s->st>>>(
                       a, chunks)));
    }
    LAUNCH(s, (k_swap_decide<<<int(cdiv(S.nprob, 128)), 128, 0, s->st>>>(a)));
    CK(cudaGetLastError());
    return 0;
}

// The staged seed batch runs on the asynchronous solver (one persistent,
// non-cooperative kernel) rather than the step-synchronous graph.
bool seed_uses_async(const pmf_solver *s) {
    if (s->stage.wide) return false;
    const int64_t ngr = std::max<int64_t>(1, int64_t(s->lay.grids.size()));
    return s->async_mode == 1 || (s->async_mode < 0 && s->lay.ntiles <= s->async_max_tiles &&
                                  s->lay.ntiles <= int64_t(s->async_max_grid_tiles) * ngr);
}

// Host-side preparation of a run: launch geometry, device state and the
// layout uploads (pageable copies: issued before a batch stream's wait on
// the previous run, so the launch does not block on it)
template <class E>
int seed_prep_t(pmf_solver *s) {
    int rc = grids_for<E>(s);
    if (rc) return rc;
    if ((rc = setup_state(s, E::kBytes))) return rc;
    if ((rc = s->d_swapflag.ensure(size_t(s->stage.nprob) * 4))) return rc;
    s->ctx.swapflag = s->d_swapflag.as<int32_t>();
    s->prepped = true;
    return 0;
}

template <class E>
int seed_run_t(pmf_solver *s) {
    SeedStage &S = s->stage;
    int rc;
    if (!s->prepped && (rc = seed_prep_t<E>(s))) return rc;
    s->prepped = false;
    const Ctx &c = s->ctx;
    s->tmark(C_BUILD);
    const SeedArgs a = seed_args(s);
    if ((rc = seed_swap_flags(s, a))) return rc;
    LAUNCH(s, (k_build_seed<E><<<s->grid_full, NT, 0, s->st>>>(c, a)));
    CK(cudaGetLastError());
    s->stats.full_passes++;
    const bool chains = S.chain > 1;
    s->warm_active = chains;
    // asynchronous solver for latency-bound batches; large batches keep the
    // GPU full with step-synchronous phases, whose wide scan kernels and
    // multi-sweep relabels cost less per tile than queued tile tasks
    if (seed_uses_async(s)) {
        if ((rc = async_solve<E>(s, c, a))) return rc;
        if (s->verify && (rc = launch_verify<E>(s, c, a))) return rc;
        return 0;
    }
    // rolling warm start needs the persistent discharge and a single-launch BFS
    s->ctx.rolling = chains && s->rolling && s->persistent && (s->bfs_multi || s->persistent_bfs);
    s->ctx.specg = s->ctx.rolling && s->async_spec ? s->d_specg.as<int32_t>() : nullptr;
    // kept heights need the speculative closure as their safety net
    s->ctx.keeph = s->ctx.specg && s->adv_keep_h ? s->d_keeph.as<int32_t>() : nullptr;
    // minimal source sides are nested along the schedule: a chain's next
    // label closure is seeded with the previous lambda's (knob nested_lab)
    s->ctx.labok = s->ctx.rolling && s->nested_lab ? s->d_labok.as<int32_t>() : nullptr;
    int rc2 = run_solve<E>(s, c, int32_t(s->lay.grids.size()), chains ? &a : nullptr,
                           chains ? s->d_slopesum.as<int64_t>() : nullptr);
    if (rc2) return rc2;
    if (s->verify) {
        if ((rc = launch_verify<E>(s, c, a))) return rc;
    }
    return 0;
}

// Common end of the staging paths: offsets, lambdas, chains and the grid
// layout, per-problem slope sums (S.slope_sum, filled by the caller).
int stage_tail(pmf_solver *s, int32_t nprob, int32_t W, int32_t H, int32_t nlam, int32_t swap_mode) {
    SeedStage &S = s->stage;
    const int64_t n = int64_t(W) * H;
    int rc;
    if ((rc = s->d_off.ensure(size_t(nprob) * 16)) || (rc = s->d_lam.ensure(size_t(nlam) * 8)) ||
        (rc = s->d_swapcnt.ensure(size_t(nprob) * 8)) || (rc = s->d_mask.ensure(size_t(nprob) * n)) ||
        (rc = s->d_slopesum.ensure(size_t(nprob) * 8)) || (rc = s->d_flows.ensure(size_t(nprob) * nlam * 8)))
        return rc;
    CK(cudaMemcpyAsync(s->d_off.p, S.offs.data(), S.offs.size() * 8, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_lam.p, S.lambdas.data(), size_t(nlam) * 8, cudaMemcpyHostToDevice, s->st));
    // warm-start chains: nlam lambdas split into chains of S.chain
    // consecutive values; each chain is one grid solved step by step
    // auto: enough problems keep the GPU busy with one grid per problem, so
    // each solves its whole ladder warm; few problems are latency-bound and
    // solve every lambda cold and in parallel
    int32_t chain = s->chain;
    if (chain <= 0) chain = nprob >= s->warm_min_problems ? nlam : 1;
    chain = std::max(1, std::min(chain, nlam));
    S.chain = chain;
    s->lay.clear();
    for (int p = 0; p < nprob; p++)
        for (int j = 0; j < nlam; j += chain) s->lay.add(W, H, 0, 0, p, j, std::min(nlam, j + chain));
    s->lay.out_bytes = int64_t(nprob) * nlam * n;   // one label plane per (problem, lambda)
    CK(cudaMemcpyAsync(s->d_slopesum.p, S.slope_sum.data(), size_t(nprob) * 8, cudaMemcpyHostToDevice, s->st));
    S.nprob = nprob;
    S.nlam = nlam;
    S.W = W;
    S.H = H;
    S.swap_mode = swap_mode;
    S.valid = true;
    return 0;
}

int seed_stage(pmf_solver *s, int32_t nprob, int32_t W, int32_t H, const int64_t *const *ub,
               const int64_t *const *us, const int64_t *const *sb, const int64_t *const *pw,
               const int64_t *const *fg_idx, const int32_t *n_fg, const int64_t *const *bg_idx,
               const int32_t *n_bg, int32_t nlam, const int64_t *lambdas, int32_t swap_mode) {
    s->comp_n.clear();   // a seed batch reuses the output buffer: no composite labels to pack
    SeedStage &S = s->stage;
    S.valid = false;
    if (nprob < 1 || nlam < 1 || W < 1 || H < 1 || !ub || !us || !sb || !pw || !lambdas ||
        swap_mode < 0 || swap_mode > 2)
        return fail(PMF_ERR_ARG, "bad arguments");
    const int64_t n = int64_t(W) * H;
    for (int j = 0; j < nlam; j++)
        if (lambdas[j] < 0 || (j && lambdas[j] <= lambdas[j - 1]))
            return fail(PMF_ERR_ARG, "lambda values must be non-negative and strictly increasing");
    const int64_t lam_max = lambdas[nlam - 1];
    int rc;
    // the previous run may still read the staging buffers
    CK(cudaStreamSynchronize(s->st));
    if ((rc = s->h_in32.ensure(size_t(nprob) * n * 3 * 4)) || (rc = s->h_mask.ensure(size_t(nprob) * n)))
        return rc;
    int32_t *hb = s->h_in32.as<int32_t>();
    uint8_t *hm = s->h_mask.as<uint8_t>();
    S.offs.assign(2 * size_t(nprob), 0);
    std::unordered_map<const int64_t *, int64_t> pw_seen;
    std::vector<const int64_t *> pw_list;
    for (int p = 0; p < nprob; p++) {
        auto it = pw_seen.find(pw[p]);
        if (it == pw_seen.end()) {
            int64_t o = int64_t(pw_list.size()) * 4 * n;
            pw_seen[pw[p]] = o;
            pw_list.push_back(pw[p]);
            S.offs[nprob + p] = o;
        } else {
            S.offs[nprob + p] = it->second;
        }
    }
    if ((rc = s->h_pw.ensure(pw_list.size() * size_t(4 * n) * 4))) return rc;
    int32_t *hp = s->h_pw.as<int32_t>();
    TaskErr terr;
    // seed masks on the host (validation), one task per problem; the device
    // builds its own copy from the index lists (k_seed_masks), so only the
    // lists cross the host link
    TaskErr merr;
    s->pool->run(nprob, [&](int64_t p) {
        uint8_t *m = hm + p * n;
        memset(m, 0, size_t(n));
        for (int32_t i = 0; i < (n_fg ? n_fg[p] : 0); i++) {
            const int64_t q = fg_idx[p][i];
            if (q < 0 || q >= n) return merr.set(PMF_ERR_ARG, "fg seed out of range");
            m[q] = 1;
        }
        for (int32_t i = 0; i < (n_bg ? n_bg[p] : 0); i++) {
            const int64_t q = bg_idx[p][i];
            if (q < 0 || q >= n) return merr.set(PMF_ERR_ARG, "bg seed out of range");
            if (m[q] == 1) return merr.set(PMF_ERR_ARG, "a pixel cannot be both a foreground and background seed");
            m[q] = 2;
        }
    });
    if ((rc = merr.raise())) return rc;
    // index lists for the device: [fg of p0 | bg of p0 | fg of p1 | ...]
    std::vector<int64_t> sofs(size_t(2 * nprob + 1), 0);
    for (int p = 0; p < nprob; p++) {
        sofs[2 * p + 1] = sofs[2 * p] + (n_fg ? n_fg[p] : 0);
        sofs[2 * p + 2] = sofs[2 * p + 1] + (n_bg ? n_bg[p] : 0);
    }
    const int64_t nseeds = sofs.back();
    if ((rc = s->h_seeds.ensure(size_t(nseeds + 1) * 4))) return rc;
    int32_t *hs = s->h_seeds.as<int32_t>();
    s->pool->run(nprob, [&](int64_t p) {
        for (int32_t i = 0; i < (n_fg ? n_fg[p] : 0); i++) hs[sofs[2 * p] + i] = int32_t(fg_idx[p][i]);
        for (int32_t i = 0; i < (n_bg ? n_bg[p] : 0); i++) hs[sofs[2 * p + 1] + i] = int32_t(bg_idx[p][i]);
    });
    // pairwise planes: range check + narrow, chunked
    const int64_t pw_chunks = cdiv(4 * n, kChunk);
    s->pool->run(int64_t(pw_list.size()) * pw_chunks, [&](int64_t task) {
        const int64_t k = task / pw_chunks, lo = (task % pw_chunks) * kChunk, hi = std::min(4 * n, lo + kChunk);
        const int64_t *src = pw_list[k];
        for (int64_t i = lo; i < hi; i++)
            if (src[i] < 0 || src[i] > CAP_MAX) {
                terr.set(PMF_ERR_RANGE, "pairwise capacity outside [0, CAP_MAX]");
                return;
            }
        narrow(hp + k * 4 * n + lo, src + lo, hi - lo, 0, CAP_MAX);
    });
    if ((rc = terr.raise())) return rc;
    const int rows = int(std::max<int64_t>(1, kChunk / W)), row_tasks = int(cdiv(H, rows));
    std::vector<int64_t> mp(pw_list.size() * size_t(row_tasks), 0);
    s->pool->run(int64_t(mp.size()), [&](int64_t task) {
        const int64_t k = task / row_tasks;
        const int y0 = int(task % row_tasks) * rows;
        mp[size_t(task)] = max_pair(hp + k * 4 * n, W, H, y0, std::min(H, y0 + rows));
    });
    int64_t maxpair = 0;
    for (int64_t v : mp) maxpair = std::max(maxpair, v);
    // unary / sink planes.  Problems whose three planes equal those of the
    // previous problem (e.g. the two seed types of one CPMC seed) share one
    // staged copy.  Every problem is range-checked against its own masks
    // (ranges the device relies on; instantiate's own checks are the
    // caller's); only the distinct planes are narrowed and copied, in groups
    // whose H2D overlaps the conversion of the next group.
    std::vector<uint8_t> same(size_t(nprob), 0);
    s->pool->run(nprob, [&](int64_t p) {
        if (p == 0) return;
        const size_t nb = size_t(n) * 8;
        same[p] = (ub[p] == ub[p - 1] || !memcmp(ub[p], ub[p - 1], nb)) &&
                  (us[p] == us[p - 1] || !memcmp(us[p], us[p - 1], nb)) &&
                  (sb[p] == sb[p - 1] || !memcmp(sb[p], sb[p - 1], nb));
    });
    std::vector<int32_t> uniq;   // problems whose planes are staged
    std::vector<int32_t> staged_as(static_cast<size_t>(nprob), 0);
    for (int p = 0; p < nprob; p++) {
        if (!same[p]) uniq.push_back(p);
        staged_as[p] = uniq.back();
        S.offs[p] = 3 * int64_t(uniq.size() - 1) * n;   // base of problem p; slope +n, sink +2n
    }
    // range check of pixel q of problem p (seed masks exempt fg unary / bg sink terms)
    auto check = [&](int p, int64_t q, uint8_t m) -> bool {
        if (m != 1) {
            const int64_t b = ub[p][q], sl = us[p][q];
            if (b < 0 || sl < 0) {
                terr.set(PMF_ERR_RANGE, "negative unary term");
                return false;
            }
            if (b > CAP_MAX || (sl && lam_max > (CAP_MAX - b) / sl)) {
                terr.set(PMF_ERR_RANGE, "unary term exceeds CAP_MAX");
                return false;
            }
        }
        if (m != 2 && (sb[p][q] < 0 || sb[p][q] > CAP_MAX)) {
            terr.set(PMF_ERR_RANGE, "sink term outside [0, CAP_MAX]");
            return false;
        }
        return true;
    };
    // problems sharing planes: only the pixels where their seed masks differ
    // from the staged problem's need their own check
    const int64_t pl_chunks = cdiv(n, kChunk);
    s->pool->run(int64_t(nprob) * pl_chunks, [&](int64_t task) {
        const int p = int(task / pl_chunks);
        if (!same[p]) return;
        const int64_t lo = (task % pl_chunks) * kChunk, hi = std::min(n, lo + kChunk);
        const uint8_t *m = hm + p * n, *mr = hm + int64_t(staged_as[p]) * n;
        for (int64_t q = lo; q < hi; q++)
            if (m[q] != mr[q] && !check(p, q, m[q])) return;
    });
    if ((rc = terr.raise())) return rc;
    S.u8 = maxpair <= 255;
    // a pixel's excess is bounded by its source term plus its incoming arc
    // pairs; past int32 the batch runs on the int64 state variant
    S.wide = s->force_wide || (!S.u8 && CAP_MAX + 8 * maxpair >= (int64_t(1) << 31) - 1);
    S.lambdas.assign(lambdas, lambdas + nlam);
    const int64_t nu = int64_t(uniq.size());
    const size_t bytes_b = size_t(nu) * n * 3 * 4, bytes_pw = pw_list.size() * size_t(4 * n) * 4;
    if ((rc = s->d_in32.ensure(bytes_b)) || (rc = s->d_pw.ensure(bytes_pw)) ||
        (rc = s->d_mask.ensure(size_t(nprob) * n)) || (rc = s->d_off.ensure(size_t(nprob) * 16)) ||
        (rc = s->d_lam.ensure(size_t(nlam) * 8)) || (rc = s->d_swapcnt.ensure(size_t(nprob) * 8)))
        return rc;
    CK(cudaMemcpyAsync(s->d_pw.p, hp, bytes_pw, cudaMemcpyHostToDevice, s->st));
    if ((rc = s->d_seeds.ensure(size_t(nseeds + 1) * 4)) || (rc = s->d_sofs.ensure(sofs.size() * 8))) return rc;
    CK(cudaMemcpyAsync(s->d_seeds.p, hs, size_t(nseeds) * 4, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_sofs.p, sofs.data(), sofs.size() * 8, cudaMemcpyHostToDevice, s->st));
    // (the device seed masks are built at the start of the run, k_seed_masks:
    // staging enqueues copies only, so it overlaps another solver's run)
    // distinct planes: check + narrow in one pass, group by group, each
    // group's H2D overlapping the conversion of the next
    const int64_t group = std::max<int64_t>(1, cdiv(nu, 8));
    for (int64_t g0 = 0; g0 < nu; g0 += group) {
        const int64_t g1 = std::min(nu, g0 + group);
        s->pool->run((g1 - g0) * pl_chunks, [&](int64_t task) {
            const int64_t u = g0 + task / pl_chunks;
            const int p = uniq[size_t(u)];
            const int64_t lo = (task % pl_chunks) * kChunk, hi = std::min(n, lo + kChunk);
            const uint8_t *m = hm + p * n;
            for (int64_t q = lo; q < hi; q++)
                if (!check(p, q, m[q])) return;
            narrow(hb + 3 * u * n + 0 * n + lo, ub[p] + lo, hi - lo, 0, CAP_MAX);
            narrow(hb + 3 * u * n + 1 * n + lo, us[p] + lo, hi - lo, 0, CAP_MAX);
            narrow(hb + 3 * u * n + 2 * n + lo, sb[p] + lo, hi - lo, 0, CAP_MAX);
        });
        if ((rc = terr.raise())) return rc;
        CK(cudaMemcpyAsync(s->d_in32.as<int32_t>() + 3 * g0 * n, hb + 3 * g0 * n, size_t(g1 - g0) * 3 * n * 4,
                           cudaMemcpyHostToDevice, s->st));
    }
    // sums of unary_slope over non-fg pixels (sink capacity growth of swapped grids)
    S.slope_sum.assign(size_t(nprob), 0);
    s->pool->run(nprob, [&](int64_t p) {
        const uint8_t *m = hm + p * n;
        const int32_t *sl = hb + S.offs[p] + n;
        int64_t acc = 0;
        for (int64_t q = 0; q < n; q++)
            if (m[q] != 1) acc += sl[q];
        S.slope_sum[p] = acc;
    });
    S.synth = false;
    if ((rc = stage_tail(s, nprob, W, H, nlam, swap_mode))) return rc;
    s->stats.h2d_bytes = int64_t(bytes_b + bytes_pw) + nseeds * 4 + int64_t(sofs.size()) * 8 + int64_t(nlam) * 8;
    return 0;
}

// Seed batch of synthetic CPMC images whose planes are derived on the
// device (k_synth_planes / k_synth_pw at the start of the run): problems
// image-major, seed, type-minor; type 0 = border background (reference
// problem_for_seed, harness/synth.py:67-100), 1 = border minus the top row.
// Only the 8-bit images, the seed pixels and the seed index lists cross the
// host link.  The admission checks are the caller's (synth_device.py runs
// the reference's checks on image histograms).
int synth_stage(pmf_solver *s, int32_t nimg, int32_t W, int32_t H, const uint8_t *images, int32_t nseed,
                const int32_t *seed_xy, int32_t ntypes, const int32_t *types, int32_t nlam, const int64_t *lambdas,
                int32_t swap_mode) {
    s->comp_n.clear();
    SeedStage &S = s->stage;
    S.valid = false;
    if (nimg < 1 || nseed < 1 || ntypes < 1 || W < 1 || H < 1 || nlam < 1 || !images || !seed_xy || !types ||
        !lambdas || swap_mode < 0 || swap_mode > 2)
        return fail(PMF_ERR_ARG, "bad arguments");
    for (int t = 0; t < ntypes; t++)
        if (types[t] != 0 && types[t] != 1) return fail(PMF_ERR_ARG, "seed type must be 0 (A) or 1 (B)");
    for (int j = 0; j < nlam; j++)
        if (lambdas[j] < 0 || (j && lambdas[j] <= lambdas[j - 1]))
            return fail(PMF_ERR_ARG, "lambda values must be non-negative and strictly increasing");
    const int64_t n = int64_t(W) * H;
    const int64_t nprob64 = int64_t(nimg) * nseed * ntypes;
    if (nprob64 > (int64_t(1) << 30)) return fail(PMF_ERR_ARG, "too many problems");
    const int32_t nprob = int32_t(nprob64);
    // background sets per type (row-major ring; type 1 without the top row)
    std::vector<int32_t> ring[2];
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++)
            if (x == 0 || y == 0 || x == W - 1 || y == H - 1) {
                ring[0].push_back(y * W + x);
                if (y != 0) ring[1].push_back(y * W + x);
            }
    std::vector<int32_t> spix(size_t(nimg) * nseed);
    for (int k = 0; k < nseed; k++) {
        const int32_t x = seed_xy[2 * k], y = seed_xy[2 * k + 1];
        if (x < 0 || x >= W || y < 0 || y >= H) return fail(PMF_ERR_ARG, "seed (%d, %d) outside the image", x, y);
        const bool ring_px = x == 0 || x == W - 1 || y == 0 || y == H - 1;
        for (int t = 0; t < ntypes; t++)
            if (ring_px && (types[t] == 0 || y != 0))
                return fail(PMF_ERR_ARG, "seed (%d, %d) sits on the background border", x, y);
        for (int i = 0; i < nimg; i++) spix[size_t(i) * nseed + k] = y * W + x;
    }
    int rc;
    CK(cudaStreamSynchronize(s->st));   // the previous run may still read the staging buffers
    // seed index lists [fg of p0 | bg of p0 | fg of p1 | ...]
    std::vector<int64_t> sofs(size_t(2 * nprob + 1), 0);
    for (int p = 0; p < nprob; p++) {
        sofs[2 * p + 1] = sofs[2 * p] + 1;
        sofs[2 * p + 2] = sofs[2 * p + 1] + int64_t(ring[types[p % ntypes]].size());
    }
    const int64_t nseeds = sofs.back();
    if ((rc = s->h_seeds.ensure(size_t(nseeds + 1) * 4))) return rc;
    int32_t *hs = s->h_seeds.as<int32_t>();
    s->pool->run(nprob, [&](int64_t p) {
        const std::vector<int32_t> &r = ring[types[p % ntypes]];
        hs[sofs[2 * p]] = spix[size_t(p / ntypes)];
        memcpy(hs + sofs[2 * p + 1], r.data(), r.size() * 4);
    });
    // slope sums over non-fg pixels from one intensity histogram per image
    std::vector<int64_t> hist(size_t(nimg) * 256, 0);
    s->pool->run(nimg, [&](int64_t i) {
        const uint8_t *im = images + i * n;
        int64_t *h = hist.data() + i * 256;
        for (int64_t q = 0; q < n; q++) h[im[q]]++;
    });
    S.slope_sum.assign(size_t(nprob), 0);
    for (int p = 0; p < nprob; p++) {
        const int64_t u = p / ntypes, i = u / nseed;
        const int sv = images[i * n + spix[size_t(u)]];
        int64_t acc = 0;
        for (int v = 0; v < 256; v++) acc += hist[size_t(i) * 256 + v] * (1 + ((255 - std::abs(v - sv)) * 7) / 255);
        S.slope_sum[p] = acc - (1 + (255 * 7) / 255);   // the fg seed (dsim 0)
    }
    S.offs.assign(2 * size_t(nprob), 0);
    for (int p = 0; p < nprob; p++) {
        S.offs[p] = 3 * int64_t(p / ntypes) * n;
        S.offs[nprob + p] = 4 * int64_t(p / (int64_t(nseed) * ntypes)) * n;
    }
    const int64_t nu = int64_t(nimg) * nseed;
    if ((rc = s->d_in32.ensure(size_t(nu) * n * 3 * 4)) || (rc = s->d_pw.ensure(size_t(nimg) * n * 4 * 4)) ||
        (rc = s->d_img.ensure(size_t(nimg) * n)) || (rc = s->d_spix.ensure(spix.size() * 4)) ||
        (rc = s->d_seeds.ensure(size_t(nseeds + 1) * 4)) || (rc = s->d_sofs.ensure(sofs.size() * 8)) ||
        (rc = s->h_mask.ensure(size_t(nimg) * n)) || (rc = s->h_small.ensure(spix.size() * 4 + 64)))
        return rc;
    // images and seed pixels through pinned staging (async copies)
    memcpy(s->h_mask.p, images, size_t(nimg) * n);
    memcpy(s->h_small.p, spix.data(), spix.size() * 4);
    CK(cudaMemcpyAsync(s->d_img.p, s->h_mask.p, size_t(nimg) * n, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_spix.p, s->h_small.p, spix.size() * 4, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_seeds.p, hs, size_t(nseeds) * 4, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_sofs.p, sofs.data(), sofs.size() * 8, cudaMemcpyHostToDevice, s->st));
    S.lambdas.assign(lambdas, lambdas + nlam);
    S.u8 = true;                 // arc pairs <= 2 * 64
    S.wide = s->force_wide;
    S.synth = true;
    S.nimg = nimg;
    S.nseed = nseed;
    if ((rc = stage_tail(s, nprob, W, H, nlam, swap_mode))) return rc;
    s->stats.h2d_bytes = int64_t(nimg) * n + int64_t(spix.size()) * 4 + nseeds * 4 + int64_t(sofs.size()) * 8 +
                         int64_t(nlam) * 8;
    return 0;
}

// 8 output bytes (bit j -> byte j, 0/1) per input byte
struct UnpackLut {
    uint64_t v[256];
    UnpackLut() {
        for (int b = 0; b < 256; b++) {
            uint64_t w = 0;
            for (int j = 0; j < 8; j++) w |= uint64_t((b >> j) & 1) << (8 * j);
            v[b] = w;
        }
    }
};

int seed_fetch(pmf_solver *s, uint8_t *swapped_out, int64_t *flows_out, uint8_t *labels_out) {
    static const UnpackLut lut;
    const SeedStage &S = s->stage;
    const int64_t nf = int64_t(S.nprob) * S.nlam;
    const int64_t out_bytes = nf * int64_t(S.W) * S.H;
    // labels travel as bits (k_pack_bits) and are unpacked on the host
    const int64_t nwords = cdiv(out_bytes, 32), bit_bytes = nwords * 4;
    const size_t lab_bytes = size_t(cdiv(bit_bytes, 64) * 64);
    int rc;
    if ((rc = s->h_out.ensure(lab_bytes + size_t(nf) * 8 + size_t(S.nprob) * 4 + 64))) return rc;
    uint8_t *ho = s->h_out.as<uint8_t>();
    int64_t *hfl = (int64_t *)(ho + lab_bytes);
    int32_t *hsw = (int32_t *)(hfl + nf);
    // (the run packed the labels into d_bits, pmf_seed_launch)
    // the bits cross in pieces of >= 4 MB, each unpacked on the host pool
    // while the next one is in flight (the unpack writes 8x the bytes)
    const int64_t full = labels_out ? out_bytes / 8 : 0;   // whole bit bytes = 8 labels each
    const int npiece = int(std::min<int64_t>(8, std::max<int64_t>(1, full >> 22)));
    const int64_t piece = cdiv(std::max<int64_t>(full, 1), npiece);
    cudaEvent_t *ev = s->fetch_ev;   // created once per solver, reused by every fetch
    if (labels_out) {
        for (int i = 0; i < npiece; i++) {
            const int64_t lo = i * piece, hi = i + 1 == npiece ? int64_t(bit_bytes) : std::min(full, lo + piece);
            if (hi > lo)
                CK(cudaMemcpyAsync(ho + lo, s->d_bits.as<uint8_t>() + lo, size_t(hi - lo), cudaMemcpyDeviceToHost, s->st));
            if (!ev[i]) CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
            CK(cudaEventRecord(ev[i], s->st));
        }
    }
    CK(cudaMemcpyAsync(hfl, s->d_flows.p, nf * 8, cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(hsw, s->d_swapflag.p, size_t(S.nprob) * 4, cudaMemcpyDeviceToHost, s->st));
    if (labels_out) {
        // large outputs: huge pages, so first touch costs one fault per 2 MiB
        if (out_bytes >= (int64_t(64) << 20)) {
            const uintptr_t a = (reinterpret_cast<uintptr_t>(labels_out) + 0x1fffff) & ~uintptr_t(0x1fffff);
            const uintptr_t e = (reinterpret_cast<uintptr_t>(labels_out) + uintptr_t(out_bytes)) & ~uintptr_t(0x1fffff);
            if (e > a) madvise(reinterpret_cast<void *>(a), e - a, MADV_HUGEPAGE);
        }
        // parallel unpack straight into the caller's buffer (64 KiB of bits per task)
        const int64_t per = int64_t(64) << 10;
        for (int i = 0; i < npiece; i++) {
            const cudaError_t e = cudaEventSynchronize(ev[i]);
            if (e != cudaSuccess) return fail(PMF_ERR_CUDA, "label transfer: %s", cudaGetErrorString(e));
            const int64_t lo = i * piece, hi = std::min(full, lo + piece);
            if (hi <= lo) continue;
            s->pool->run(cdiv(hi - lo, per), [&](int64_t t) {
                const int64_t a = lo + t * per, b = std::min(hi, a + per);
                uint64_t *dst = reinterpret_cast<uint64_t *>(labels_out) + a;
                for (int64_t k = a; k < b; k++) {
                    const uint64_t v = lut.v[ho[k]];
                    memcpy(dst + (k - a), &v, 8);
                }
            });
        }
    }
    CK(cudaStreamSynchronize(s->st));
    memcpy(flows_out, hfl, size_t(nf) * 8);
    if (swapped_out)
        for (int p = 0; p < S.nprob; p++) swapped_out[p] = uint8_t(hsw[p] != 0);
    if (labels_out)
        for (int64_t i = full * 8; i < out_bytes; i++) labels_out[i] = uint8_t((ho[i >> 3] >> (i & 7)) & 1);
    s->stats.d2h_bytes = (labels_out ? bit_bytes : 0) + nf * 8 + int64_t(S.nprob) * 4;
    return 0;
}

// --------------------------------------------------------------------------
// int64 state variant (wide.cuh): graphs whose excess bound leaves int32
// --------------------------------------------------------------------------

struct WideBatch {
    std::vector<WGrid> grids;
    std::vector<WTile> tiles;
    int64_t P = 0;
    void add(int32_t W, int32_t H, int64_t out_off, int32_t pitch, int32_t xoff, int32_t cs_off, int32_t flow_idx,
             int32_t prob, int32_t lam) {
        WGrid g{};
        g.base = P;
        g.W = W;
        g.H = H;
        g.out_off = out_off;
        g.pitch = pitch;
        g.xoff = xoff;
        g.cs_off = cs_off;
        g.flow_idx = flow_idx;
        g.prob = prob;
        g.lam = lam;
        const int32_t gi = int32_t(grids.size());
        for (int32_t y = 0; y < H; y += WT)
            for (int32_t x = 0; x < W; x += WT) tiles.push_back(WTile{gi, x, y, 0});
        P += int64_t(W) * H;
        grids.push_back(g);
    }
};

// device state + tables of batch B; returns the kernel context in *c
int wide_setup(pmf_solver *s, const WideBatch &B, WCtx *c) {
    const int64_t P = B.P, G = int64_t(B.grids.size()), T = int64_t(B.tiles.size());
    if (T >= (int64_t(1) << 31)) return fail(PMF_ERR_ARG, "batch too large (%lld tiles)", (long long)T);
    int rc;
    if ((rc = s->d_we.ensure(size_t(P) * 8)) || (rc = s->d_wr.ensure(size_t(P) * 32)) ||
        (rc = s->d_h.ensure(size_t(P) * 4)) || (rc = s->d_lab.ensure(size_t(P))) ||
        (rc = s->d_wgrid.ensure(size_t(G) * sizeof(WGrid))) || (rc = s->d_wtile.ensure(size_t(T) * sizeof(WTile))) ||
        (rc = s->d_snk.ensure(size_t(G) * 8)) || (rc = s->d_drain.ensure(size_t(G) * 8)) ||
        (rc = s->d_wchg.ensure(64)) || (rc = s->d_wcnt.ensure(64)) || (rc = s->d_err.ensure(64)) ||
        (rc = s->d_stat.ensure(ST_NSTAT * 8)) || (rc = s->d_ctl.ensure(sizeof(Ctl))) || (rc = s->d_colswap.ensure(64)))
        return rc;
    CK(cudaMemcpyAsync(s->d_wgrid.p, B.grids.data(), size_t(G) * sizeof(WGrid), cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_wtile.p, B.tiles.data(), size_t(T) * sizeof(WTile), cudaMemcpyHostToDevice, s->st));
    CK(cudaMemsetAsync(s->d_snk.p, 0, size_t(G) * 8, s->st));
    CK(cudaMemsetAsync(s->d_drain.p, 0, size_t(G) * 8, s->st));
    WCtx x{};
    x.e = s->d_we.as<int64_t>();
    x.r = s->d_wr.as<int64_t>();
    x.h = s->d_h.as<int32_t>();
    x.lab = s->d_lab.as<uint8_t>();
    x.P = P;
    x.grids = s->d_wgrid.as<WGrid>();
    x.tiles = s->d_wtile.as<WTile>();
    x.ntiles = int32_t(T);
    x.snk_sum = s->d_snk.as<int64_t>();
    x.drain = s->d_drain.as<int64_t>();
    x.err = s->d_err.as<int32_t>();
    x.colswap = s->d_colswap.as<uint8_t>();
    x.out = s->d_out.as<uint8_t>();
    x.flows = s->d_flows.as<int64_t>();
    x.count = s->d_wcnt.as<unsigned long long>();
    *c = x;
    return 0;
}

// run bracket state of a wide run: no tile-engine counters, no error yet
int wide_bracket(pmf_solver *s) {
    int rc;
    if ((rc = s->d_err.ensure(64)) || (rc = s->d_stat.ensure(ST_NSTAT * 8)) || (rc = s->d_ctl.ensure(sizeof(Ctl))))
        return rc;
    CK(cudaMemsetAsync(s->d_err.p, 0, 64, s->st));
    CK(cudaMemsetAsync(s->d_stat.p, 0, ST_NSTAT * 8, s->st));
    CK(cudaMemsetAsync(s->d_ctl.p, 0, sizeof(Ctl), s->st));
    s->wide_cycles = s->wide_pulses_run = s->wide_relax_launches = 0;
    return 0;
}

inline int wide_grid(const pmf_solver *s, const WCtx &c) {
    return int(std::max<int64_t>(1, std::min<int64_t>(c.ntiles, 2 * int64_t(s->sms))));
}

// relaxation launches until one changes nothing (a fixpoint stays one)
int wide_relax(pmf_solver *s, const WCtx &c, int sink) {
    const int grid = wide_grid(s, c);
    LAUNCH(s, (k_wide_init<<<grid, 1024, 0, s->st>>>(c, sink)));
    int32_t *chg = s->d_wchg.as<int32_t>(), *hp = s->h_small.as<int32_t>();
    for (;;) {
        CK(cudaMemsetAsync(chg, 0, 8 * 4, s->st));
        for (int k = 0; k < 8; k++) LAUNCH(s, (k_wide_relax<<<grid, 1024, 0, s->st>>>(c, sink, chg + k)));
        CK(cudaGetLastError());
        s->wide_relax_launches += 8;
        CK(cudaMemcpyAsync(hp, chg + 7, 4, cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
        if (!*hp) return 0;
    }
}

// phase 1 to a maximum preflow, then labels, flows (per grid into flows[flow_idx])
int wide_solve(pmf_solver *s, const WCtx &c, int32_t ngrids) {
    const int grid = wide_grid(s, c);
    unsigned long long *hc = s->h_small.as<unsigned long long>();
    int rc;
    for (;;) {
        // exact global relabel (solvers.py:54-85) ...
        if ((rc = wide_relax(s, c, 1))) return rc;
        // ... then stop when no pixel that can reach the sink holds excess
        CK(cudaMemsetAsync(c.count, 0, 8, s->st));
        LAUNCH(s, (k_wide_count<<<grid, 1024, 0, s->st>>>(c)));
        CK(cudaMemcpyAsync(hc, c.count, 8, cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
        if (*hc == 0) break;
        if (++s->wide_cycles > s->max_cycles)
            return fail(PMF_ERR_NOCONV, "push-relabel failed to converge within %lld cycles", (long long)s->max_cycles);
        for (int k = 0; k < s->wide_pulses; k++) {
            LAUNCH(s, (k_wide_push<<<grid, 1024, 0, s->st>>>(c)));
            LAUNCH(s, (k_wide_relabel<<<grid, 1024, 0, s->st>>>(c)));
        }
        CK(cudaGetLastError());
        s->wide_pulses_run += s->wide_pulses;
    }
    if ((rc = wide_relax(s, c, 0))) return rc;   // source-side closure
    LAUNCH(s, (k_wide_emit<<<grid, 1024, 0, s->st>>>(c)));
    LAUNCH(s, (k_wide_finalize<<<int(cdiv(ngrids, 256)), 256, 0, s->st>>>(c, ngrids)));
    CK(cudaGetLastError());
    return 0;
}

// seed batch on the int64 state: every (problem, lambda) graph built in
// its original orientation, in chunks that bound the device state
int wide_seed_run(pmf_solver *s) {
    const SeedStage &S = s->stage;
    const int64_t n = int64_t(S.W) * S.H, NG = int64_t(S.nprob) * S.nlam;
    int rc;
    if ((rc = wide_bracket(s))) return rc;
    if ((rc = s->d_swapflag.ensure(size_t(S.nprob) * 4)) || (rc = s->d_out.ensure(size_t(NG * n))) ||
        (rc = s->d_flows.ensure(size_t(NG) * 8)))
        return rc;
    s->tmark(C_BUILD);
    const SeedArgs a = seed_args(s);
    if ((rc = seed_swap_flags(s, a))) return rc;
    const int64_t per = std::max<int64_t>(1, (int64_t(24) << 30) / (45 * n));   // <= ~24 GB of state per chunk
    for (int64_t g0 = 0; g0 < NG; g0 += per) {
        const int64_t g1 = std::min(NG, g0 + per);
        WideBatch B;
        for (int64_t g = g0; g < g1; g++)
            B.add(S.W, S.H, g * n, S.W, 0, -1, int32_t(g), int32_t(g / S.nlam), int32_t(g % S.nlam));
        WCtx c;
        if ((rc = wide_setup(s, B, &c))) return rc;
        LAUNCH(s, (k_wide_build_seed<<<wide_grid(s, c), 1024, 0, s->st>>>(c, a.base, a.slope, a.sink, a.pw, a.mask,
                                                                          a.plane_off, a.pw_off, a.lambdas)));
        CK(cudaGetLastError());
        if ((rc = wide_solve(s, c, int32_t(B.grids.size())))) return rc;
    }
    if (s->verify) {
        Ctx x{};
        x.out = s->d_out.as<uint8_t>();
        x.flows = s->d_flows.as<int64_t>();
        x.err = s->d_err.as<int32_t>();
        if ((rc = launch_verify<EdgeI32>(s, x, a))) return rc;
    }
    return 0;
}

// stats of a wide run (after run_end): cycles, pulses, relaxation launches
void wide_stats(pmf_solver *s) {
    s->stats.cycles = s->wide_cycles;
    s->stats.push_sweeps = s->wide_pulses_run;
    s->stats.bfs_sweeps = s->wide_relax_launches;
    s->stats.wide_mode = 1;
    s->stats.edge_bytes = 32;
}

// composites on the int64 state: one grid per composite, planes from the
// int32 staging (src | snk | nbr per composite at comp_off), already on the
// device (solve_composites_t)
int wide_comp_run(pmf_solver *s, int32_t ncomp, const int32_t *width, const int32_t *height,
                  const std::vector<int32_t> &cs_off, int64_t total_px) {
    int rc;
    if ((rc = wide_bracket(s))) return rc;
    if ((rc = s->d_colswap.ensure(s->colswap.size() + 1)) || (rc = s->d_in32.ensure(size_t(total_px) * 6 * 4)) ||
        (rc = s->d_off.ensure(size_t(ncomp) * 8)) || (rc = s->d_out.ensure(size_t(std::max<int64_t>(s->lay.out_bytes, 1)))))
        return rc;
    s->tmark(C_H2D);
    CK(cudaMemcpyAsync(s->d_colswap.p, s->colswap.data(), s->colswap.size(), cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(s->d_off.p, s->comp_off.data(), size_t(ncomp) * 8, cudaMemcpyHostToDevice, s->st));
    s->tmark(C_BUILD);
    WideBatch B;
    for (int32_t c = 0; c < ncomp; c++)
        B.add(width[c], height[c], s->comp_out[size_t(c)], width[c], 0, cs_off[size_t(c)], c, c, 0);
    WCtx c;
    if ((rc = wide_setup(s, B, &c))) return rc;
    const int32_t *din = s->d_in32.as<int32_t>();
    LAUNCH(s, (k_wide_load_comp<<<wide_grid(s, c), 1024, 0, s->st>>>(c, din, din + total_px, din + 2 * total_px,
                                                                     s->d_off.as<int64_t>())));
    CK(cudaGetLastError());
    return wide_solve(s, c, ncomp);
}

// --------------------------------------------------------------------------
// composites
// --------------------------------------------------------------------------

template <class E>
int comp_run_t(pmf_solver *s, int ncomp, int64_t total_px) {
    s->warm_active = 0;
    int rc = grids_for<E>(s);
    if (rc) return rc;
    if ((rc = setup_state(s, E::kBytes))) return rc;
    if ((rc = s->d_colswap.ensure(s->colswap.size() + 1))) return rc;
    s->ctx.colswap = s->d_colswap.as<uint8_t>();
    CK(cudaMemcpyAsync(s->d_colswap.p, s->colswap.data(), s->colswap.size(), cudaMemcpyHostToDevice, s->st));
    const Ctx &c = s->ctx;
    s->tmark(C_H2D);
    const size_t G = s->lay.grids.size();
    if ((rc = s->d_off.ensure(G * 8))) return rc;
    int32_t *din = s->d_in32.as<int32_t>();   // planes staged by solve_composites_t
    s->grid_off.resize(G);   // per grid: its composite's plane offset
    for (size_t g = 0; g < G; g++) s->grid_off[g] = s->comp_off[size_t(s->lay.grids[g].prob)];
    CK(cudaMemcpyAsync(s->d_off.p, s->grid_off.data(), G * 8, cudaMemcpyHostToDevice, s->st));
    // split composites: bridge / uncovered columns belong to no grid and stay 0
    if (s->comp_any_split) CK(cudaMemsetAsync(s->d_out.p, 0, size_t(s->lay.out_bytes), s->st));
    s->tmark(C_BUILD);
    CompArgs a{din, din + total_px, din + 2 * total_px, s->d_off.as<int64_t>()};
    LAUNCH(s, (k_load_comp<E><<<s->grid_full, NT, 0, s->st>>>(c, a)));
    CK(cudaGetLastError());
    s->stats.full_passes++;
    // latency-bound composites (a wire request, a small join()) run on the
    // asynchronous solver when every grid reports one side: a segment span,
    // or a composite with no swapped column (or only swapped ones)
    bool uniform = true;
    for (const GridDesc &gd : s->lay.grids) {
        const uint8_t *cs = s->colswap.data() + gd.colswap_off;
        for (int32_t x = 1; x < gd.W && uniform; x++) uniform = cs[x] == cs[0];
    }
    const int64_t ngr = std::max<int64_t>(1, int64_t(G));
    const bool use_async = uniform && (s->async_mode == 1 ||
                                       (s->async_mode < 0 && s->lay.ntiles <= s->async_max_tiles &&
                                        s->lay.ntiles <= int64_t(s->async_max_grid_tiles) * ngr));
    if (use_async && s->comp_async) return async_solve<E>(s, c, SeedArgs{});
    return run_solve<E>(s, c, int32_t(s->lay.grids.size()));
}

}  // namespace

// ==========================================================================
// C ABI
// ==========================================================================

extern "C" {

const char *pmf_last_error(void) { return g_err.c_str(); }

int pmf_solver_create(int32_t device, pmf_solver **out) {
    if (!out) return fail(PMF_ERR_ARG, "null output handle");
    *out = nullptr;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(PMF_ERR_ARG, "device %d out of range (%d devices)", device, ndev);
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return fail(PMF_ERR_CUDA, "device %d is sm_%d%d, not sm_100-class", device, prop.major, prop.minor);
    pmf_solver *s = new pmf_solver();
    s->device = device;
    s->sms = prop.multiProcessorCount;
    {
        unsigned hc = std::thread::hardware_concurrency();
        // one process per GPU (torchrun): share the host cores between the local ranks
        if (const char *lw = getenv("LOCAL_WORLD_SIZE")) {
            const int n = atoi(lw);
            if (n > 1) hc = std::max(1u, hc / unsigned(n));
        }
        s->pool = new Pool();
        s->pool->threads = int(std::max(1u, std::min(hc ? hc : 1u, 16u)));
    }
    if (cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&s->ev_run[0]) != cudaSuccess || cudaEventCreate(&s->ev_run[1]) != cudaSuccess ||
        s->h_small.ensure(sizeof(Ctl) + 256)) {
        pmf_solver_destroy(s);
        return fail(PMF_ERR_CUDA, "stream/event/pinned allocation failed");
    }
    *out = s;
    return 0;
}

int pmf_solver_destroy(pmf_solver *s) {
    if (!s) return 0;
    cudaSetDevice(s->device);
    if (s->st) cudaStreamSynchronize(s->st);
    for (auto e : s->ev_pool) cudaEventDestroy(e);
    for (auto e : s->fetch_ev)
        if (e) cudaEventDestroy(e);
    if (s->gexec) cudaGraphExecDestroy(s->gexec);
    delete s->pool;
    for (auto e : s->ev_run)
        if (e) cudaEventDestroy(e);
    if (s->ev_tail) cudaEventDestroy(s->ev_tail);
    if (s->st) cudaStreamDestroy(s->st);
    delete s;
    return 0;
}

int pmf_solver_set(pmf_solver *s, const char *name, int64_t v) {
    if (!s || !name) return fail(PMF_ERR_ARG, "null argument");
    std::string k(name);
    if (k == "push_iters" && v >= 1 && v <= 100000) s->push_iters = int(v);
    else if (k == "push_sweeps" && v >= 1 && v <= 100000) s->push_sweeps = int(v);
    else if (k == "bfs_chunk" && v >= 1 && v <= 100000) s->bfs_chunk = int(v);
    else if (k == "relabel_every" && v >= 0 && v <= 100000) s->relabel_every = int(v);
    else if (k == "persistent") s->persistent = v != 0;
    else if (k == "warp" && (v == 0 || v == 4)) s->warp = int(v);
    else if (k == "chain" && v >= 0 && v <= 1000000) s->chain = int(v);
    else if (k == "warm_min_problems" && v >= 1) s->warm_min_problems = int(v);
    else if (k == "push_budget_warm" && v >= 0) s->push_budget_warm = int(v);
    else if (k == "push_budget_add" && v >= 0 && v < (int64_t(1) << 30)) s->push_budget_add = int(v);
    else if (k == "verify" && v >= 0 && v <= 2) s->verify = int(v);
    else if (k == "verify_vec") s->verify_vec = v != 0;
    else if (k == "comp_split") s->comp_split = v != 0;
    else if (k == "rolling") s->rolling = v != 0;
    else if (k == "push_flush" && v >= 0 && v <= 1024) s->push_flush = int(v);
    else if (k == "nested_lab") s->nested_lab = v != 0;
    else if (k == "comp_async") s->comp_async = v != 0;
    else if (k == "async_yield_us" && v >= 0 && v <= 1000000) s->async_yield_us = int(v);
    else if (k == "async_yield_keep" && v >= 0 && v <= 100000) s->async_yield_keep = int(v);
    else if (k == "fresh_skip") s->fresh_skip = v != 0;
    else if (k == "async" && v >= -1 && v <= 1) s->async_mode = int(v);
    else if (k == "async_max_tiles" && v >= 0) s->async_max_tiles = int(std::min<int64_t>(v, 1 << 30));
    else if (k == "async_max_grid_tiles" && v >= 0) s->async_max_grid_tiles = int(std::min<int64_t>(v, 1 << 30));
    else if (k == "async_cont") s->async_cont = v != 0;
    else if (k == "async_prefetch") s->async_prefetch = v != 0;
    else if (k == "async_spec") s->async_spec = v != 0;
    else if (k == "adv_keep_h") s->adv_keep_h = v != 0;
    else if (k == "phase_log") s->phase_log = v != 0;
    else if (k == "graph") s->use_graph = v != 0;
    else if (k == "persistent_bfs") s->persistent_bfs = v != 0;
    else if (k == "bfs_multi") s->bfs_multi = v != 0;
    else if (k == "push_budget" && v >= 0) s->push_budget = int(v);
    else if (k == "timing") s->timing = v != 0;
    else if (k == "max_cycles" && v >= 1) s->max_cycles = v;
    else if (k == "force_wide") s->force_wide = v != 0;
    else if (k == "wide_pulses" && v >= 1 && v <= 100000) s->wide_pulses = int(v);
    else return fail(PMF_ERR_ARG, "unknown knob or bad value: %s=%lld", name, (long long)v);
    return 0;
}

// Host-side admission statistics of many int64 planes at once (OpenMP over
// planes): min, max, sum and the sum of the entries below CAP_MAX per plane
// (parametric.py _plane_stats; the reductions instantiate's checks need,
// parametric.py:141-165 / grid.py:102-130).
int pmf_plane_stats(int32_t nplanes, const int64_t *const *planes, const int64_t *sizes, int64_t *out) {
    if (nplanes < 0 || (nplanes && (!planes || !sizes || !out))) return fail(PMF_ERR_ARG, "bad arguments");
    int nt = int(std::max(1u, std::min(std::thread::hardware_concurrency(), 16u)));
    if (const char *lw = getenv("LOCAL_WORLD_SIZE")) {   // host cores shared by the local ranks
        const int n = atoi(lw);
        if (n > 1) nt = std::max(1, nt / n);
    }
    // tasks of <= 2^20 elements (a few large planes still use every thread)
    constexpr int64_t kStat = int64_t(1) << 20;
    std::vector<int64_t> first(size_t(nplanes) + 1, 0);
    for (int32_t k = 0; k < nplanes; k++) first[k + 1] = first[k] + std::max<int64_t>(1, cdiv(sizes[k], kStat));
    const int64_t ntask = first[nplanes];
    std::vector<int64_t> part(size_t(ntask) * 4);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t task = 0; task < ntask; task++) {
        const int32_t k = int32_t(std::upper_bound(first.begin(), first.end(), task) - first.begin() - 1);
        const int64_t lo = (task - first[k]) * kStat, hi = std::min(sizes[k], lo + kStat);
        const int64_t *a = planes[k];
        int64_t mn = 0, mx = 0, sum = 0, fin = 0;   // initial=0 semantics of numpy min/max
        for (int64_t i = lo; i < hi; i++) {
            const int64_t v = a[i];
            mn = std::min(mn, v);
            mx = std::max(mx, v);
            sum += v;
            fin += v < CAP_MAX ? v : 0;
        }
        int64_t *o = part.data() + 4 * task;
        o[0] = mn;
        o[1] = mx;
        o[2] = sum;
        o[3] = fin;
    }
    for (int32_t k = 0; k < nplanes; k++) {
        int64_t mn = 0, mx = 0, sum = 0, fin = 0;
        for (int64_t t = first[k]; t < first[k + 1]; t++) {
            const int64_t *o = part.data() + 4 * t;
            mn = std::min(mn, o[0]);
            mx = std::max(mx, o[1]);
            sum += o[2];
            fin += o[3];
        }
        out[4 * k + 0] = mn;
        out[4 * k + 1] = mx;
        out[4 * k + 2] = sum;
        out[4 * k + 3] = fin;
    }
    return 0;
}

int pmf_solver_stream(const pmf_solver *s, void **stream_out) {
    if (!s || !stream_out) return fail(PMF_ERR_ARG, "null argument");
    *stream_out = (void *)s->st;
    return 0;
}

int pmf_solver_stats(const pmf_solver *s, pmf_stats *out) {
    if (!s || !out) return fail(PMF_ERR_ARG, "null argument");
    *out = s->stats;
    return 0;
}

}  // extern "C"

// T = int64_t (GridGraph planes) or int32_t (wire planes, wire.py:19)
template <class T>
static int solve_composites_t(pmf_solver *s, int32_t ncomp, const int32_t *width, const int32_t *height,
                              const T *const *src, const T *const *snk, const T *const *nbr,
                              const int32_t *nseg, const int32_t *const *seg_off, const int32_t *const *seg_w,
                              const uint8_t *const *seg_swapped, int64_t *flow_out, uint8_t *const *labels_out) {
    if (!s || ncomp < 1 || !width || !height || !src || !snk || !nbr || !flow_out || !labels_out)
        return fail(PMF_ERR_ARG, "bad arguments");
    CK(cudaSetDevice(s->device));
    CK(cudaStreamSynchronize(s->st));   // staging buffers are reused below
    // a composite solve overwrites the staged seed batch's layout, planes,
    // offsets, labels and flows (pmf_seed_run/fetch/score refuse until the
    // next pmf_seed_stage), and the previous composites' labels
    s->stage.valid = false;
    s->comp_n.clear();
    s->lay.clear();
    s->colswap.clear();
    s->comp_off.assign(size_t(ncomp), 0);
    std::vector<int32_t> cs_off(size_t(ncomp), 0);
    int64_t total_px = 0;
    for (int c = 0; c < ncomp; c++) {
        if (width[c] < 1 || height[c] < 1) return fail(PMF_ERR_ARG, "composite %d: bad shape", c);
        cs_off[c] = int32_t(s->colswap.size());
        s->colswap.resize(s->colswap.size() + width[c], 0);
        int ns = nseg ? nseg[c] : 0;
        for (int k = 0; k < ns; k++) {
            int o = seg_off[c][k], w = seg_w[c][k];
            if (o < 0 || w < 0 || o + w > width[c])
                return fail(PMF_ERR_ARG, "composite %d: segment %d outside the grid", c, k);
            if (k > 0 && o < seg_off[c][k - 1] + seg_w[c][k - 1])
                return fail(PMF_ERR_ARG, "composite %d: segment %d overlaps its predecessor", c, k);
            if (seg_swapped[c][k])
                for (int x = o; x < o + w; x++) s->colswap[cs_off[c] + x] = 1;
        }
        s->comp_off[c] = total_px;
        total_px += int64_t(width[c]) * height[c];
    }
    // stage inputs as int32: src | snk | nbr (4 planes per composite)
    int rc = s->h_in32.ensure(size_t(total_px) * 6 * 4);
    if (rc) return rc;
    int32_t *hin = s->h_in32.as<int32_t>();
    TaskErr terr;
    // range check + narrow every plane into the pinned staging buffer
    // [src | snk | nbr (4 planes per composite)], in 6 pieces of total_px
    // elements each; a piece's H2D overlaps the narrowing of the next
    // (comp_run_t finds the planes on the device)
    if ((rc = s->d_in32.ensure(size_t(total_px) * 6 * 4))) return rc;
    std::vector<int64_t> off4(size_t(ncomp) + 1, 0);   // 4 * comp_off, plus the end
    for (int c = 0; c < ncomp; c++) off4[size_t(c)] = 4 * s->comp_off[size_t(c)];
    off4[size_t(ncomp)] = 4 * total_px;
    for (int piece = 0; piece < 6; piece++) {
        const int64_t base = int64_t(piece) * total_px, ntask = cdiv(total_px, kChunk);
        s->pool->run(ntask, [&](int64_t task) {
            const int64_t lo = task * kChunk, hi = std::min(total_px, lo + kChunk);
            // element j of this piece: pixel j (src / snk), or element j of
            // the 4-plane neighbour blocks; composite boundaries from `bnd`
            const bool term = piece < 2;
            const int64_t j0 = (term ? 0 : (piece - 2) * total_px) + lo, j1 = j0 + (hi - lo);
            const std::vector<int64_t> &bnd = term ? s->comp_off : off4;
            int c = int(std::upper_bound(bnd.begin(), bnd.begin() + ncomp, j0) - bnd.begin()) - 1;
            for (int64_t j = j0; j < j1;) {
                const int64_t cend = std::min(j1, c + 1 < ncomp ? bnd[size_t(c) + 1] : (term ? total_px : 4 * total_px));
                const int64_t cb = bnd[size_t(c)];
                const T *srcp = term ? (piece == 0 ? src[c] : snk[c]) : nbr[c];
                int32_t *dst = hin + base + (j - j0) + lo;
                for (int64_t k = j; k < cend; k++) {
                    const int64_t v = int64_t(srcp[k - cb]);
                    if (v < 0 || v > CAP_MAX) {
                        terr.set(PMF_ERR_RANGE, "composite capacity outside [0, CAP_MAX]");
                        return;
                    }
                    dst[k - j] = int32_t(v);
                }
                j = cend;
                c++;
            }
        });
        if ((rc = terr.raise())) return rc;
        CK(cudaMemcpyAsync(s->d_in32.as<int32_t>() + base, hin + base, size_t(total_px) * 4, cudaMemcpyHostToDevice,
                           s->st));
    }
    // per (composite, band of rows) task: largest arc pair and the bound on
    // any pixel's excess (its positive terminal plus all arc pairs); bands
    // keep one large composite (a wire request) on every host thread
    constexpr int32_t kBand = 64;
    std::vector<int64_t> band_base(size_t(ncomp) + 1, 0);
    for (int c = 0; c < ncomp; c++) band_base[size_t(c) + 1] = band_base[size_t(c)] + cdiv(height[c], kBand);
    std::vector<int64_t> mp(size_t(band_base[size_t(ncomp)]), 0), mx(mp.size(), 0);
    s->pool->run(band_base[size_t(ncomp)], [&](int64_t task) {
        const int c = int(std::upper_bound(band_base.begin(), band_base.end(), task) - band_base.begin()) - 1;
        const int32_t W = width[c], H = height[c];
        const int32_t y0 = int32_t(task - band_base[size_t(c)]) * kBand, y1 = std::min(H, y0 + kBand);
        const int64_t n = int64_t(W) * H, off = s->comp_off[c];
        const int32_t *nb = hin + 2 * total_px + 4 * off;
        mp[size_t(task)] = max_pair(nb, W, H, y0, y1);
        int64_t m = 0;
        for (int64_t p = int64_t(y0) * W; p < int64_t(y1) * W; p++) {
            int64_t e = std::max<int64_t>(0, int64_t(hin[off + p]) - hin[total_px + off + p]);
            for (int d = 0; d < 4; d++) e += 2 * int64_t(nb[d * n + p]);
            m = std::max(m, e);
        }
        mx[size_t(task)] = m;
    });
    int64_t maxpair = 0, maxexcess = 0;
    for (size_t k = 0; k < mp.size(); k++) {
        maxpair = std::max(maxpair, mp[k]);
        maxexcess = std::max(maxexcess, mx[k]);
    }
    // past int32 the composites run on the int64 state variant (wide.cuh),
    // one grid per composite
    const bool wide = s->force_wide || maxexcess >= (int64_t(1) << 31) - 1;
    // Segments whose spans no arc leaves (bridge / uncovered columns all
    // zero, no LEFT arc on a span's first column, no RIGHT arc on its last)
    // are independent max-flow problems: each becomes a grid of its own
    // (knob comp_split), solved and relabelled separately, writing its
    // columns of the composite's output; the composite's flow is the sum.
    // The reference's join() builds exactly such composites (zero bridge
    // columns, supergraph.py:95-154).
    // column -> segment of every composite (at cs_off), -1: bridge / uncovered
    std::vector<int32_t> colseg(s->colswap.size(), -1);
    std::vector<uint8_t> cand(size_t(ncomp), 0), leak(size_t(band_base[size_t(ncomp)]), 0);
    for (int c = 0; c < ncomp; c++) {
        const int ns = nseg ? nseg[c] : 0;
        if (!s->comp_split || ns < 2 || wide) continue;
        cand[size_t(c)] = 1;
        for (int k = 0; k < ns; k++)
            for (int x = seg_off[c][k]; x < seg_off[c][k] + seg_w[c][k]; x++) colseg[size_t(cs_off[c] + x)] = k;
    }
    s->pool->run(band_base[size_t(ncomp)], [&](int64_t task) {
        const int c = int(std::upper_bound(band_base.begin(), band_base.end(), task) - band_base.begin()) - 1;
        if (!cand[size_t(c)]) return;
        const int32_t *sc = colseg.data() + cs_off[c];
        const int32_t W = width[c], H = height[c];
        const int32_t y0 = int32_t(task - band_base[size_t(c)]) * kBand, y1 = std::min(H, y0 + kBand);
        const int64_t n = int64_t(W) * H, off = s->comp_off[c];
        const int32_t *sp = hin + off, *kp = hin + total_px + off, *nb = hin + 2 * total_px + 4 * off;
        for (int32_t x = 0; x < W; x++) {
            const bool bridge = sc[x] < 0;
            const bool ledge = x > 0 && sc[x - 1] != sc[x];
            const bool redge = x + 1 < W && sc[x + 1] != sc[x];
            if (!bridge && !ledge && !redge) continue;
            for (int32_t y = y0; y < y1; y++) {
                const int64_t q = int64_t(y) * W + x;
                if (bridge ? (sp[q] | kp[q] | nb[q] | nb[n + q] | nb[2 * n + q] | nb[3 * n + q]) != 0
                           : (ledge && nb[q]) || (redge && nb[n + q])) {
                    leak[size_t(task)] = 1;
                    return;
                }
            }
        }
    });
    std::vector<uint8_t> split(size_t(ncomp), 0);
    for (int c = 0; c < ncomp; c++) {
        if (!cand[size_t(c)]) continue;
        split[size_t(c)] = 1;
        for (int64_t k = band_base[size_t(c)]; k < band_base[size_t(c) + 1]; k++)
            if (leak[size_t(k)]) split[size_t(c)] = 0;
    }
    int any_split = 0;
    std::vector<int64_t> &comp_out = s->comp_out;   // output offset per composite (16-byte aligned,
    comp_out.assign(size_t(ncomp), 0);              // so pmf_composite_bits can pack it in place)
    std::vector<int64_t> comp_n(static_cast<size_t>(ncomp), 0);  // published once the solve succeeded
    for (int c = 0; c < ncomp; c++) {
        s->lay.out_bytes = (s->lay.out_bytes + 15) / 16 * 16;
        comp_out[size_t(c)] = s->lay.out_bytes;
        comp_n[size_t(c)] = int64_t(width[c]) * height[c];
        if (split[size_t(c)]) {
            any_split = 1;
            const int64_t base = s->lay.out_bytes;
            s->lay.out_bytes += int64_t(width[c]) * height[c];
            for (int k = 0; k < nseg[c]; k++)
                s->lay.add_span(seg_w[c][k], height[c], cs_off[c] + seg_off[c][k], c, base, width[c],
                                seg_off[c][k]);
        } else {
            s->lay.add(width[c], height[c], 1, cs_off[c], c, 0, 1);
        }
    }
    s->comp_any_split = any_split;
    const int64_t G = int64_t(s->lay.grids.size());
    if ((rc = s->d_flows.ensure(size_t(G) * 8))) return rc;
    if ((rc = run_begin(s))) return rc;
    rc = wide ? wide_comp_run(s, ncomp, width, height, cs_off, total_px)
              : maxpair <= 255 ? comp_run_t<EdgeU8>(s, ncomp, total_px) : comp_run_t<EdgeI32>(s, ncomp, total_px);
    if (rc) return rc;
    // integrity certificate: cut cost of every composite's labels == its flow
    if (s->verify) {
        std::vector<CompV> vdesc(static_cast<size_t>(ncomp));
        int64_t cmax = 0;
        for (int c = 0; c < ncomp; c++) {
            CompV &v = vdesc[size_t(c)];
            v.off = s->comp_off[size_t(c)];
            v.out_off = comp_out[size_t(c)];
            v.W = width[c];
            v.H = height[c];
            cmax = std::max(cmax, int64_t(width[c]) * height[c]);
        }
        if ((rc = s->d_cv.ensure(size_t(ncomp) * sizeof(CompV))) || (rc = s->d_vacc.ensure(size_t(ncomp) * 8)))
            return rc;
        CK(cudaMemcpyAsync(s->d_cv.p, vdesc.data(), size_t(ncomp) * sizeof(CompV), cudaMemcpyHostToDevice, s->st));
        CK(cudaMemsetAsync(s->d_vacc.p, 0, size_t(ncomp) * 8, s->st));
        // verify=2 (test hook): flip the first label of composite 0 whose
        // pixel has src != snk, so the check must fail
        if (s->verify == 2) {
            const int32_t *hin = s->h_in32.as<int32_t>();
            const int64_t n0 = int64_t(width[0]) * height[0];
            for (int64_t q = 0; q < n0; q++)
                if (hin[q] != hin[total_px + q]) {
                    LAUNCH(s, (k_flip_label<<<1, 1, 0, s->st>>>(s->d_out.as<uint8_t>() + comp_out[0], q)));
                    break;
                }
        }
        const int chunks = int(std::max<int64_t>(1, std::min<int64_t>(cdiv(cmax, 8 * NT), 4096)));
        LAUNCH(s, (k_comp_verify<<<int(std::max<int64_t>(1, std::min<int64_t>(int64_t(ncomp) * chunks, 32 * s->sms))),
                                    NT, 0, s->st>>>(s->d_in32.as<int32_t>(), total_px, s->d_cv.as<CompV>(),
                                                    s->d_out.as<uint8_t>(), ncomp, chunks,
                                                    s->d_vacc.as<unsigned long long>())));
        CK(cudaGetLastError());
    }
    // outputs
    s->tmark(C_D2H);
    const Layout &L = s->lay;
    const size_t lab_bytes = size_t((L.out_bytes + 7) / 8) * 8;
    if ((rc = s->h_out.ensure(lab_bytes + size_t(G) * 8 + size_t(ncomp) * 8))) return rc;
    uint8_t *ho = s->h_out.as<uint8_t>();
    int64_t *hsnk = (int64_t *)(ho + lab_bytes);
    int64_t *hcost = hsnk + G;
    if (s->verify) CK(cudaMemcpyAsync(hcost, s->d_vacc.p, size_t(ncomp) * 8, cudaMemcpyDeviceToHost, s->st));
    bool any_labels = false;   // a null labels_out[c]: labels stay on the device (pmf_composite_bits)
    for (int c = 0; c < ncomp; c++) any_labels |= labels_out[c] != nullptr;
    if (any_labels) CK(cudaMemcpyAsync(ho, s->d_out.p, L.out_bytes, cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(hsnk, s->d_flows.p, G * 8, cudaMemcpyDeviceToHost, s->st));
    if ((rc = run_end(s))) return rc;
    if (wide) wide_stats(s);
    s->comp_n = std::move(comp_n);
    for (int c = 0; c < ncomp; c++) flow_out[c] = 0;
    for (int64_t g = 0; g < G; g++) flow_out[L.grids[size_t(g)].prob] += hsnk[g];
    if (s->verify)
        for (int c = 0; c < ncomp; c++)
            if (hcost[c] != flow_out[c]) {
                s->comp_n.clear();
                return fail(PMF_ERR_NONMAX, "composite %d: cut cost %lld differs from its flow %lld (integrity check)",
                            c, (long long)hcost[c], (long long)flow_out[c]);
            }
    for (int c = 0; c < ncomp; c++)
        if (labels_out[c]) memcpy(labels_out[c], ho + comp_out[size_t(c)], size_t(width[c]) * height[c]);
    s->stats.h2d_bytes = total_px * 6 * 4;
    s->stats.d2h_bytes = (any_labels ? L.out_bytes : 0) + G * 8;
    return 0;
}

extern "C" {

int pmf_solve_composites(pmf_solver *s, int32_t ncomp, const int32_t *width, const int32_t *height,
                         const int64_t *const *src, const int64_t *const *snk,
                         const int64_t *const *nbr, const int32_t *nseg,
                         const int32_t *const *seg_off, const int32_t *const *seg_w,
                         const uint8_t *const *seg_swapped, int64_t *flow_out,
                         uint8_t *const *labels_out) {
    return solve_composites_t<int64_t>(s, ncomp, width, height, src, snk, nbr, nseg, seg_off, seg_w,
                                       seg_swapped, flow_out, labels_out);
}

int pmf_solve_composites_i32(pmf_solver *s, int32_t ncomp, const int32_t *width, const int32_t *height,
                             const int32_t *const *src, const int32_t *const *snk,
                             const int32_t *const *nbr, const int32_t *nseg,
                             const int32_t *const *seg_off, const int32_t *const *seg_w,
                             const uint8_t *const *seg_swapped, int64_t *flow_out,
                             uint8_t *const *labels_out) {
    return solve_composites_t<int32_t>(s, ncomp, width, height, src, snk, nbr, nseg, seg_off, seg_w,
                                       seg_swapped, flow_out, labels_out);
}

// Labels of composite c of the last composite solve as LSB-first bits
// (bit i of byte k = pixel 8k + i; the wire's response order, wire.py:26),
// packed on the device: ceil(n / 8) bytes into out.
int pmf_composite_bits(pmf_solver *s, int32_t c, uint8_t *out, int64_t out_bytes) {
    if (!s || !out) return fail(PMF_ERR_ARG, "null argument");
    if (c < 0 || size_t(c) >= s->comp_n.size()) return fail(PMF_ERR_ARG, "no composite %d in the last solve", c);
    const int64_t n = s->comp_n[size_t(c)], need = (n + 7) / 8;
    if (out_bytes < need) return fail(PMF_ERR_ARG, "%lld bytes needed for %lld labels", (long long)need, (long long)n);
    CK(cudaSetDevice(s->device));
    int rc;
    if ((rc = s->d_bits.ensure(size_t(cdiv(n, 32)) * 4))) return rc;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 32 * 256), 16 * s->sms)));
    LAUNCH(s, (k_pack_bits<<<grid, 256, 0, s->st>>>(s->d_out.as<uint8_t>() + s->comp_out[size_t(c)],
                                                     s->d_bits.as<uint32_t>(), n)));
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, s->d_bits.p, size_t(need), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    return 0;
}

// CTA-busy milliseconds of the last asynchronous run, summed over CTAs:
// per phase kind (BINIT, BFS, SEED, PUSH, LINIT, LAB, EMIT, -), queue wait,
// hand-off, grid transitions, then zeros.
int pmf_debug_busy(pmf_solver *s, double *out16) {
    if (!s || !out16) return fail(PMF_ERR_ARG, "null argument");
    for (int k = 0; k < 16; k++) out16[k] = s->busy_ms[k];
    out16[7] = double(s->spec_tries);     // speculative label closures tried
    out16[11] = double(s->spec_spoiled);  // ... and spoiled
    return 0;
}

// Phase timeline of grid g of the last asynchronous run with knob
// phase_log = 1: up to PLOG - 1 entries (phase << 56 | globaltimer ns).
int pmf_debug_phases(pmf_solver *s, int64_t g, uint64_t *out, int32_t *n) {
    if (!s || !out || !n) return fail(PMF_ERR_ARG, "null argument");
    if (g < 0 || g >= s->plog_grids) return fail(PMF_ERR_ARG, "no phase log for grid %lld", (long long)g);
    uint64_t buf[PLOG];
    CK(cudaMemcpy(buf, s->d_plog.as<unsigned long long>() + g * PLOG, sizeof buf, cudaMemcpyDeviceToHost));
    const int k = int(std::min<uint64_t>(buf[0], uint64_t(PLOG - 1)));
    *n = std::min(*n, k);
    for (int j = 0; j < *n; j++) out[j] = buf[j + 1];
    return 0;
}

int pmf_debug_trace(pmf_solver *s, int32_t *kind, double *us, double *start_us, int64_t *tiles,
                    int32_t *n) {
    if (!s || !n) return fail(PMF_ERR_ARG, "null argument");
    CK(cudaSetDevice(s->device));
    Ctl ctl;
    CK(cudaMemcpyAsync(&ctl, s->d_ctl.p, sizeof ctl, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    int m = std::min(*n, ctl.ntrace);
    for (int i = 0; i < m; i++) {
        if (kind) kind[i] = ctl.trace_kind[i];
        if (us) us[i] = double(ctl.trace_ns[i]) * 1e-3;
        if (start_us) start_us[i] = double(ctl.trace_t0[i] - ctl.trace_t0[0]) * 1e-3;
        if (tiles) tiles[i] = int64_t(ctl.trace_tiles[i] & 0xffffffffull);
    }
    *n = m;
    return 0;
}

int pmf_debug_state(pmf_solver *s, int32_t *w, int32_t *h, void *r, uint8_t *lab, int64_t *ntiles) {
    if (!s) return fail(PMF_ERR_ARG, "null solver");
    CK(cudaSetDevice(s->device));
    const int64_t P = s->lay.ntiles * TPIX;
    if (ntiles) *ntiles = s->lay.ntiles;
    if (w) CK(cudaMemcpyAsync(w, s->d_w.p, P * 4, cudaMemcpyDeviceToHost, s->st));
    if (h) CK(cudaMemcpyAsync(h, s->d_h.p, P * 4, cudaMemcpyDeviceToHost, s->st));
    if (r) CK(cudaMemcpyAsync(r, s->d_r.p, P * s->edge_bytes, cudaMemcpyDeviceToHost, s->st));
    if (lab) CK(cudaMemcpyAsync(lab, s->d_lab.p, P, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    return 0;
}

int pmf_seed_stage(pmf_solver *s, int32_t nprob, int32_t W, int32_t H, const int64_t *const *ub,
                   const int64_t *const *us, const int64_t *const *sb, const int64_t *const *pw,
                   const int64_t *const *fg_idx, const int32_t *n_fg,
                   const int64_t *const *bg_idx, const int32_t *n_bg, int32_t nlam,
                   const int64_t *lambdas, int32_t swap_mode) {
    if (!s) return fail(PMF_ERR_ARG, "null solver");
    CK(cudaSetDevice(s->device));
    return seed_stage(s, nprob, W, H, ub, us, sb, pw, fg_idx, n_fg, bg_idx, n_bg, nlam, lambdas, swap_mode);
}

// Enqueue the whole run of the staged batch on the solver's stream: seed
// masks, build, solve, certificate, label bit packing.  `after` (nullable):
// a solver whose last launched run must finish first (device runs of a
// batch stream stay serialised while the host stages and fetches).
int pmf_seed_launch(pmf_solver *s, pmf_solver *after) {
    if (!s || !s->stage.valid) return fail(PMF_ERR_ARG, "no staged seed batch");
    if (after == s) return fail(PMF_ERR_ARG, "a solver cannot wait for itself");
    CK(cudaSetDevice(s->device));
    s->launch_h2d = s->stats.h2d_bytes;
    s->prepped = false;
    if (!s->stage.wide) {
        const int rp = s->stage.u8 ? seed_prep_t<EdgeU8>(s) : seed_prep_t<EdgeI32>(s);
        if (rp) return rp;
    }
    if (after) {   // before run_begin: the run's device time excludes the wait
        if (after->device != s->device) return fail(PMF_ERR_ARG, "solvers on different devices");
        if (after->ev_tail) CK(cudaStreamWaitEvent(s->st, after->ev_tail, 0));
    }
    int rc = run_begin(s);
    if (rc) return rc;
    const SeedStage &S = s->stage;
    const int64_t n = int64_t(S.W) * S.H, out_bytes = int64_t(S.nprob) * S.nlam * n;
    if (S.synth) {   // planes of a synthetic image batch, derived on the device
        const int64_t nu = int64_t(S.nimg) * S.nseed;
        LAUNCH(s, (k_synth_planes<<<int(std::min<int64_t>(cdiv(nu * cdiv(n, 4), 256), 64 * s->sms)), 256, 0,
                                    s->st>>>(s->d_img.as<uint8_t>(), n, S.nseed, s->d_spix.as<int32_t>(), nu,
                                             s->d_in32.as<int32_t>())));
        LAUNCH(s, (k_synth_pw<<<int(std::min<int64_t>(cdiv(int64_t(S.nimg) * n, 256), 64 * s->sms)), 256, 0,
                                s->st>>>(s->d_img.as<uint8_t>(), S.W, S.H, S.nimg, s->d_pw.as<int32_t>())));
        CK(cudaGetLastError());
    }
    CK(cudaMemsetAsync(s->d_mask.p, 0, size_t(S.nprob) * n, s->st));
    LAUNCH(s, (k_seed_masks<<<std::max(1, std::min(S.nprob, 4 * s->sms)), 256, 0, s->st>>>(
                   s->d_mask.as<uint8_t>(), s->d_seeds.as<int32_t>(), s->d_sofs.as<int64_t>(), S.nprob, n)));
    CK(cudaGetLastError());
    rc = S.wide ? wide_seed_run(s) : S.u8 ? seed_run_t<EdgeU8>(s) : seed_run_t<EdgeI32>(s);
    if (rc) return rc;
    // labels leave the device as bits (unpacked on the host by pmf_seed_fetch)
    if ((rc = s->d_bits.ensure(size_t(cdiv(out_bytes, 32)) * 4))) return rc;
    const int grid = int(std::min<int64_t>(cdiv(out_bytes, 32 * 256), 16 * s->sms));
    LAUNCH(s, (k_pack_bits<<<std::max(grid, 1), 256, 0, s->st>>>(s->d_out.as<uint8_t>(), s->d_bits.as<uint32_t>(),
                                                                 out_bytes)));
    CK(cudaGetLastError());
    if (!s->ev_tail) CK(cudaEventCreateWithFlags(&s->ev_tail, cudaEventDisableTiming));
    CK(cudaEventRecord(s->ev_tail, s->st));
    s->launched = true;
    s->last_async = seed_uses_async(s);
    return 0;
}

// The next run of s starts only after `on`'s last launched run (recorded
// before pmf_seed_launch; any number of calls).
int pmf_solver_depend(pmf_solver *s, pmf_solver *on) {
    if (!s || !on || on == s) return fail(PMF_ERR_ARG, "bad arguments");
    if (on->device != s->device) return fail(PMF_ERR_ARG, "solvers on different devices");
    CK(cudaSetDevice(s->device));
    if (on->ev_tail) CK(cudaStreamWaitEvent(s->st, on->ev_tail, 0));
    return 0;
}

// Run kind of the staged batch (1: asynchronous solver, a single
// non-cooperative persistent kernel that may share the device with another
// such run; 0: step-synchronous graph with cooperative launches) and of the
// solver's last launched run.
int pmf_seed_kind(pmf_solver *s, int32_t *staged_async, int32_t *last_async) {
    if (!s || !s->stage.valid) return fail(PMF_ERR_ARG, "no staged seed batch");
    if (staged_async) *staged_async = seed_uses_async(s) ? 1 : 0;
    if (last_async) *last_async = s->last_async ? 1 : 0;
    return 0;
}

// Wait for the launched run; device errors, statistics.
int pmf_seed_wait(pmf_solver *s) {
    if (!s || !s->launched) return fail(PMF_ERR_ARG, "no launched seed run");
    CK(cudaSetDevice(s->device));
    s->launched = false;
    int rc = run_end(s);
    if (s->stage.wide) wide_stats(s);
    s->stats.h2d_bytes = s->launch_h2d;
    return rc;
}

// Diagnostics: the staged planes of the current seed batch as the solver
// holds them on the device (unary / slope / sink per distinct problem, then
// the pairwise planes); sizes in int32 elements, *n_* receive the totals.
int pmf_debug_planes(pmf_solver *s, int32_t *planes_out, int64_t *n_planes, int32_t *pw_out, int64_t *n_pw) {
    if (!s || !s->stage.valid || !n_planes || !n_pw) return fail(PMF_ERR_ARG, "bad arguments");
    CK(cudaSetDevice(s->device));
    const SeedStage &S = s->stage;
    const int64_t n = int64_t(S.W) * S.H;
    int64_t np_ = 0, nw = 0;
    for (int p = 0; p < S.nprob; p++) {
        np_ = std::max(np_, S.offs[p] + 3 * n);
        nw = std::max(nw, S.offs[S.nprob + p] + 4 * n);
    }
    if (planes_out && *n_planes >= np_)
        CK(cudaMemcpyAsync(planes_out, s->d_in32.p, size_t(np_) * 4, cudaMemcpyDeviceToHost, s->st));
    if (pw_out && *n_pw >= nw) CK(cudaMemcpyAsync(pw_out, s->d_pw.p, size_t(nw) * 4, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    *n_planes = np_;
    *n_pw = nw;
    return 0;
}

int pmf_synth_stage(pmf_solver *s, int32_t nimg, int32_t width, int32_t height, const uint8_t *images,
                    int32_t nseed, const int32_t *seed_xy, int32_t ntypes, const int32_t *types, int32_t nlam,
                    const int64_t *lambdas, int32_t swap_mode) {
    if (!s) return fail(PMF_ERR_ARG, "null solver");
    CK(cudaSetDevice(s->device));
    return synth_stage(s, nimg, width, height, images, nseed, seed_xy, ntypes, types, nlam, lambdas, swap_mode);
}

int pmf_seed_run(pmf_solver *s) {
    int rc = pmf_seed_launch(s, nullptr);
    if (rc) return rc;
    return pmf_seed_wait(s);
}

// Device scoring of the last seed run against ground-truth masks (one n-byte
// 0/1 mask per problem): per (problem, lambda) foreground count and the
// exact Jaccard overlap terms |S & G|, |S | G| (harness/bench.py:36-45).
int pmf_seed_score(pmf_solver *s, const uint8_t *const *truths, int64_t *fg_out, int64_t *inter_out,
                   int64_t *union_out) {
    if (!s || !s->stage.valid || !truths || !fg_out || !inter_out || !union_out)
        return fail(PMF_ERR_ARG, "bad arguments");
    CK(cudaSetDevice(s->device));
    const SeedStage &S = s->stage;
    const int64_t n = int64_t(S.W) * S.H, planes = int64_t(S.nprob) * S.nlam;
    int rc;
    if ((rc = s->d_truth.ensure(size_t(S.nprob) * n)) || (rc = s->d_score.ensure(size_t(planes) * 24)) ||
        (rc = s->h_mask.ensure(size_t(S.nprob) * n)) || (rc = s->h_small.ensure(size_t(planes) * 24 + 64)))
        return rc;
    // the previous run may still read the staging masks
    CK(cudaStreamSynchronize(s->st));
    uint8_t *hm = s->h_mask.as<uint8_t>();
    TaskErr terr;
    s->pool->run(S.nprob, [&](int64_t p) {
        if (!truths[p]) {
            terr.set(PMF_ERR_ARG, "a truth mask is missing");
            return;
        }
        memcpy(hm + p * n, truths[p], size_t(n));
    });
    if ((rc = terr.raise())) return rc;
    CK(cudaMemcpyAsync(s->d_truth.p, hm, size_t(S.nprob) * n, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemsetAsync(s->d_score.p, 0, size_t(planes) * 24, s->st));
    const int chunks = int(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 16384), 1024)));
    LAUNCH(s, (k_score<<<int(std::min<int64_t>(planes * chunks, 32 * s->sms)), NT, 0, s->st>>>(
                   s->d_out.as<uint8_t>(), s->d_truth.as<uint8_t>(), S.nprob, S.nlam, n, chunks,
                   s->d_score.as<unsigned long long>())));
    CK(cudaGetLastError());
    int64_t *hs = s->h_small.as<int64_t>();
    CK(cudaMemcpyAsync(hs, s->d_score.p, size_t(planes) * 24, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    for (int64_t k = 0; k < planes; k++) {
        fg_out[k] = hs[3 * k];
        inter_out[k] = hs[3 * k + 1];
        union_out[k] = hs[3 * k + 2];
    }
    return 0;
}

int pmf_seed_fetch(pmf_solver *s, uint8_t *swapped_out, int64_t *flows_out, uint8_t *labels_out) {
    if (!s || !s->stage.valid || !flows_out) return fail(PMF_ERR_ARG, "bad arguments");
    CK(cudaSetDevice(s->device));
    return seed_fetch(s, swapped_out, flows_out, labels_out);
}

int pmf_solve_seed_batch(pmf_solver *s, int32_t nprob, int32_t W, int32_t H,
                         const int64_t *const *ub, const int64_t *const *us,
                         const int64_t *const *sb, const int64_t *const *pw,
                         const int64_t *const *fg_idx, const int32_t *n_fg,
                         const int64_t *const *bg_idx, const int32_t *n_bg, int32_t nlam,
                         const int64_t *lambdas, int32_t swap_mode, uint8_t *swapped_out,
                         int64_t *flows_out, uint8_t *labels_out) {
    if (!flows_out || !labels_out) return fail(PMF_ERR_ARG, "bad arguments");
    int rc = pmf_seed_stage(s, nprob, W, H, ub, us, sb, pw, fg_idx, n_fg, bg_idx, n_bg, nlam, lambdas,
                            swap_mode);
    if (rc) return rc;
    if ((rc = pmf_seed_run(s))) return rc;
    return pmf_seed_fetch(s, swapped_out, flows_out, labels_out);
}

}  // extern "C"
