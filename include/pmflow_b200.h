/*
 * pmflow_b200.h -- C ABI of the B200-native supergraph min-cut engine.
 *
 * Plain pointers and sizes only (no torch / CUDA types in signatures).  Every
 * entry point is reentrant per solver handle; distinct handles may be driven
 * from distinct host threads concurrently (the Python shim calls through
 * ctypes, which drops the GIL).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/pmflow):
 *
 *   pmf_solve_composites   supergraph.py:190-207  solve_composite(g, layout)
 *                          (and, with nseg == 0, solvers.py:188-191
 *                          maxflow_pushrelabel).  Several composites may be
 *                          solved in one device batch; the ThreadedBackend
 *                          default local solver (scheduler.py:141-142) and
 *                          WorkerServer(solve_fn=...) (rpc.py:92-100) call it.
 *   pmf_solve_seed_batch   supergraph.py:227-253 build_seed_supergraph +
 *                          supergraph.py:190-207 solve_composite +
 *                          supergraph.py:157-187 split, fused on device:
 *                          SeedProblem planes in, per-(problem, lambda)
 *                          flows and canonical label masks out.  Also serves
 *                          parametric.py:180-183 solve_schedule_sequential.
 *
 * Status codes map 1:1 onto the reference exception classes (see
 * paper_1509_06004_b200/_native.py): PMF_ERR_NOCONV -> SolverError
 * (solvers.py:137-139), PMF_ERR_NONMAX -> NonMaximalFlowError
 * (solvers.py:156-157,183-184), PMF_ERR_RANGE -> CapacityOverflowError
 * (grid.py:45-46), PMF_ERR_ARG -> ValueError, PMF_ERR_CUDA -> RuntimeError.
 */
#ifndef PMFLOW_B200_H
#define PMFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMF_OK 0
#define PMF_ERR_ARG (-1)
#define PMF_ERR_CUDA (-2)
#define PMF_ERR_NOCONV (-3)
#define PMF_ERR_NONMAX (-4)
#define PMF_ERR_RANGE (-5)

#define PMF_SWAP_AUTO 0
#define PMF_SWAP_ON 1
#define PMF_SWAP_OFF 2

typedef struct pmf_solver pmf_solver;

/* Counters and device timings of the last solve on a handle. */
typedef struct pmf_stats {
    int64_t cycles;             /* global-relabel / discharge cycles          */
    int64_t push_tile_passes;   /* 32x32 tiles discharged                     */
    int64_t bfs_tile_passes;    /* tiles relaxed by the sink-distance BFS     */
    int64_t label_tile_passes;  /* tiles relaxed by the source-side BFS       */
    int64_t push_sweeps;        /* push kernel launches                       */
    int64_t bfs_sweeps;         /* BFS kernel launches (both BFS kinds)       */
    int64_t full_passes;        /* whole-state passes (init/seed/emit)        */
    int64_t grids;              /* independent grids solved                   */
    int64_t tiles;              /* tiles in the batch                         */
    int64_t pixels;             /* real (unpadded) pixels in the batch        */
    int32_t edge_bytes;         /* residual storage per pixel: 4 (u8x4) / 16 */
    int32_t timed;              /* 1 if the ms fields below are valid         */
    double ms_total;            /* device time of the whole solve             */
    double ms_build;            /* build / load kernels                       */
    double ms_push;             /* push-relabel sweeps                        */
    double ms_bfs;              /* sink-distance BFS sweeps + init            */
    double ms_labels;           /* source-side BFS + emit                     */
    double ms_seed;             /* active-tile seeding passes                 */
    double ms_h2d;              /* host->device copies                        */
    double ms_d2h;              /* device->host copies                        */
    double ms_device;           /* device time of the last run (always on)    */
    int64_t launches;           /* host-side launches (kernels + graphs)      */
    int64_t h2d_bytes;          /* host->device bytes of the last stage       */
    int64_t d2h_bytes;          /* device->host bytes of the last fetch       */
    int64_t graph_builds;       /* solve graphs (re)built by the last run     */
    int64_t kernels;            /* kernels executed on the device by the run  */
    int64_t steps;              /* warm-start steps (lambdas per chain); async: lambda-graphs finished */
    int64_t scan_tile_passes;   /* async: init / seed / label-init / emit tile passes */
    double ms_async;            /* async: span of the persistent solve kernel (device clock) */
    int32_t async_mode;         /* 1: the last run used the asynchronous solver */
    int32_t wide_mode;          /* 1: the last run used the int64 state variant */
    int64_t binit_tile_passes;  /* async scan phases, tiles each: relabel init, */
    int64_t seed_tile_passes;   /*   active-tile seeding, label init,           */
    int64_t linit_tile_passes;  /*   emit (+ warm-start advance)                */
    int64_t emit_tile_passes;
} pmf_stats;

/* Create / destroy a solver bound to one CUDA device and its own stream. */
int pmf_solver_create(int32_t device, pmf_solver **out);
int pmf_solver_destroy(pmf_solver *s);

/* Tuning knobs (each covered by a -m gpu parity test, tests/test_gpu_parity.py
 * test_every_knob_keeps_c1_bit_exact):
 *   discharge:  "push_iters" (smem iterations per tile pass), "relabel_every"
 *               (exact local relabel period), "push_budget" / "push_budget_warm"
 *               / "push_budget_add" (pops per discharge phase), "push_sweeps"
 *               (sweep-mode launches per cycle), "push_flush" (mid-pass
 *               hand-off of border inflow), "fresh_skip";
 *   scheduling: "async" (-1 auto / 0 step-synchronous / 1 single-kernel
 *               asynchronous solver) with "async_max_tiles" /
 *               "async_max_grid_tiles" (auto thresholds), "async_cont",
 *               "async_prefetch", "async_spec", "adv_keep_h"; "graph" (0
 *               host-driven loop, 1 whole solve as one CUDA graph),
 *               "persistent", "persistent_bfs", "bfs_multi", "bfs_chunk",
 *               "rolling", "chain" / "warm_min_problems" (warm-start chains);
 *   kernels:    "warp" (label BFS: 4 warp-per-tile bitset kernel, 0 CTA kernel);
 *   int64:      "force_wide" (the int64 state variant even when int32 bounds
 *               hold), "wide_pulses" (pulses between its global relabels);
 *   checks:     "verify" (device cut-cost == flow certificate, default on; 2 =
 *               test hook corrupting one label first), "verify_vec",
 *               "comp_split" (composites: one grid per isolated segment span),
 *               "max_cycles" (non-convergence guard);
 *   diagnostics: "timing", "phase_log".
 * Returns PMF_ERR_ARG if unknown or out of range. */
int pmf_solver_set(pmf_solver *s, const char *name, int64_t value);

/* The solver's CUDA stream (a cudaStream_t) for callers that record their
 * own events or order their own work against the engine. */
int pmf_solver_stream(const pmf_solver *s, void **stream_out);

/* Host-only helper (no device needed): per int64 plane k of sizes[k]
 * entries, out[4k .. 4k+3] = min, max, sum, sum of entries below CAP_MAX
 * (min / max include 0, numpy's initial=0).  The reductions of the seed
 * family admission checks (parametric.py:141-165), over many planes on all
 * host cores. */
int pmf_plane_stats(int32_t nplanes, const int64_t *const *planes, const int64_t *sizes, int64_t *out);

/* Thread-local message describing the last error on this thread. */
const char *pmf_last_error(void);

/* Statistics of the last solve on this handle (copied into *out). */
int pmf_solver_stats(const pmf_solver *s, pmf_stats *out);

/*
 * Solve ncomp independent (composite) grid graphs in one device batch.
 * Composite c: width[c] x height[c] pixels, row-major; src[c], snk[c] are
 * (n) arrays, nbr[c] is (4, n) in direction order LEFT, RIGHT, UP, DOWN --
 * the admitted int64 capacities of GridGraph (grid.py:56-99).  nseg[c]
 * segments with column offset / width / swapped flag describe the layout
 * (supergraph.py:39-64); nseg[c] == 0 means layout None.
 * Outputs: flow_out[c] (int64) and labels_out[c] (n bytes, 1 = source
 * side; swapped spans carry the complement of the sink side over all rows,
 * supergraph.py:201-206).
 */
int pmf_solve_composites(pmf_solver *s, int32_t ncomp,
                         const int32_t *width, const int32_t *height,
                         const int64_t *const *src, const int64_t *const *snk,
                         const int64_t *const *nbr,
                         const int32_t *nseg, const int32_t *const *seg_off,
                         const int32_t *const *seg_w, const uint8_t *const *seg_swapped,
                         int64_t *flow_out, uint8_t *const *labels_out);

/*
 * pmf_solve_composites with int32 planes: the wire request's capacity arrays
 * (wire.py:19 "six i32 arrays", decoded at wire.py:180-186) are read in
 * place, without the int64 GridGraph copies decode_request makes; same
 * checks (PMF_ERR_RANGE outside [0, CAP_MAX]) and outputs.  Serves the
 * GPU worker handler wire.serve_payload (rpc.py:147-162 _solve_and_reply).
 */
int pmf_solve_composites_i32(pmf_solver *s, int32_t ncomp,
                             const int32_t *width, const int32_t *height,
                             const int32_t *const *src, const int32_t *const *snk,
                             const int32_t *const *nbr,
                             const int32_t *nseg, const int32_t *const *seg_off,
                             const int32_t *const *seg_w, const uint8_t *const *seg_swapped,
                             int64_t *flow_out, uint8_t *const *labels_out);

/*
 * Both composite entry points accept a null labels_out[c]: that
 * composite's labels stay on the device, and pmf_composite_bits packs them
 * there into the wire's LSB-first bit order (wire.py:26, bit i of byte k =
 * pixel 8k + i) and copies ceil(n / 8) bytes to out -- the GPU worker's
 * response body without a host-side pack.  c indexes the last solve.
 */
int pmf_composite_bits(pmf_solver *s, int32_t c, uint8_t *out, int64_t out_bytes);

/*
 * Build and solve the lambda families of nprob SeedProblems
 * (parametric.py:80-130) sharing one width x height, over nlam lambda
 * values (strictly increasing, validated by the caller), on device.
 * Per problem p: unary_base[p], unary_slope[p], sink_base[p] (n int64),
 * pairwise[p] ((4, n) int64; identical pointers are uploaded once),
 * fg_idx[p] / bg_idx[p] (seed flat indices, n_fg[p] / n_bg[p] entries).
 * swap_mode: PMF_SWAP_AUTO decides per problem at lambda[(nlam-1)/2]
 * (supergraph.py:210-212, 85-92), ON / OFF force it.
 * Outputs: swapped_out[nprob]; flows_out[nprob*nlam] (problem-major);
 * labels_out: nprob*nlam*n bytes, each the canonical minimal-source-side
 * mask of the ORIGINAL (unswapped) lambda graph -- what split() returns.
 * The caller guarantees admissibility (instantiate's checks,
 * parametric.py:141-165); the engine re-checks the ranges it relies on.
 */
int pmf_solve_seed_batch(pmf_solver *s, int32_t nprob, int32_t width, int32_t height,
                         const int64_t *const *unary_base, const int64_t *const *unary_slope,
                         const int64_t *const *sink_base, const int64_t *const *pairwise,
                         const int64_t *const *fg_idx, const int32_t *n_fg,
                         const int64_t *const *bg_idx, const int32_t *n_bg,
                         int32_t nlam, const int64_t *lambdas, int32_t swap_mode,
                         uint8_t *swapped_out, int64_t *flows_out, uint8_t *labels_out);

/*
 * pmf_solve_seed_batch in three steps, for callers that keep inputs resident
 * on the device across solves (benchmarks, repeated schedules):
 *   pmf_seed_stage  validate + convert the planes and copy them to the device
 *                   (same arguments as pmf_solve_seed_batch minus outputs);
 *   pmf_seed_run    build + solve the staged batch; results stay on device;
 *   pmf_seed_fetch  copy swapped flags, flows and (if labels_out != NULL)
 *                   label masks of the last run to the host.
 * pmf_seed_run = pmf_seed_launch(s, NULL) + pmf_seed_wait(s).  The split
 * lets a batch stream keep the device busy while the host works: launch
 * enqueues the whole run on the solver's stream and returns; with `after`
 * non-NULL (another solver of the same device) the run starts only when
 * `after`'s last launched run has finished, so runs never share the GPU
 * while the next batch is staged and the previous one fetched (staging
 * enqueues copies only).  wait blocks until the run is done and reports
 * its device errors (supergraph.solve_seed_supergraphs).
 */
int pmf_seed_stage(pmf_solver *s, int32_t nprob, int32_t width, int32_t height,
                   const int64_t *const *unary_base, const int64_t *const *unary_slope,
                   const int64_t *const *sink_base, const int64_t *const *pairwise,
                   const int64_t *const *fg_idx, const int32_t *n_fg,
                   const int64_t *const *bg_idx, const int32_t *n_bg,
                   int32_t nlam, const int64_t *lambdas, int32_t swap_mode);
int pmf_seed_run(pmf_solver *s);

/*
 * On-device synthesis (replaces generate_batch's planes,
 * harness/synth.py:52-136): stage a seed batch of `nimg` synthetic CPMC
 * images whose planes are derived on the GPU at the start of the run.
 * images: nimg * width * height intensities (0..255, row-major); seed_xy:
 * `nseed` interior seed pixels (x, y) shared by every image; types[ntypes]:
 * 0 = background = the image border (problem_for_seed, synth.py:67-100),
 * 1 = the border minus its top row.  Problems are image-major, seed,
 * type-minor, with exactly the planes problem_for_seed derives (unary_base
 * 1 + 15(255-d)/255, unary_slope 1 + 7(255-d)/255, sink_base 1 + 63d/255,
 * d = |I - I(seed)|; pairwise 1 + 63(255-|dI|)/255).  Then pmf_seed_run /
 * launch / wait / fetch / score as for pmf_seed_stage.  The admission
 * checks (instantiate's errors) are the caller's.
 */
int pmf_synth_stage(pmf_solver *s, int32_t nimg, int32_t width, int32_t height, const uint8_t *images,
                    int32_t nseed, const int32_t *seed_xy, int32_t ntypes, const int32_t *types,
                    int32_t nlam, const int64_t *lambdas, int32_t swap_mode);
/* Diagnostics: copy the staged planes of the current seed batch off the
 * device (after a run for pmf_synth_stage batches): three int32 planes
 * (unary_base, unary_slope, sink_base) per distinct problem, then four
 * pairwise planes per distinct pairwise plane; pass NULL / too-small
 * buffers to read the sizes (*n_planes, *n_pw, in int32 elements). */
int pmf_debug_planes(pmf_solver *s, int32_t *planes_out, int64_t *n_planes, int32_t *pw_out, int64_t *n_pw);
int pmf_seed_launch(pmf_solver *s, pmf_solver *after);
/* Extra ordering for a batch stream: the next run of s starts only after
 * `on`'s last launched run (any number of calls before pmf_seed_launch). */
int pmf_solver_depend(pmf_solver *s, pmf_solver *on);
/* Kind of the staged batch's run and of the solver's last launched run:
 * 1 = asynchronous solver (one non-cooperative persistent kernel whose idle
 * CTAs may leave its tail to a concurrent run, knob async_yield_us), 0 =
 * step-synchronous graph (cooperative launches: must not share the GPU). */
int pmf_seed_kind(pmf_solver *s, int32_t *staged_async, int32_t *last_async);
int pmf_seed_wait(pmf_solver *s);
int pmf_seed_fetch(pmf_solver *s, uint8_t *swapped_out, int64_t *flows_out, uint8_t *labels_out);

/* Scores of the last seed run on the device (replaces the per-cut host
 * loop of harness/bench.py:95-113, `overlap` :36-45): truths[p] is problem
 * p's 0/1 ground-truth mask (width*height bytes, row-major); for every
 * (problem, lambda), problem-major: fg_out = |S|, inter_out = |S & G|,
 * union_out = |S | G| (overlap = inter / union, exact). */
int pmf_seed_score(pmf_solver *s, const uint8_t *const *truths, int64_t *fg_out, int64_t *inter_out,
                   int64_t *union_out);

/* Diagnostics: the first (up to *n, at most 256) tile-kernel launches of the
 * last run: kind (0 discharge, 1 sink BFS, 2 label BFS; 4-6 one sweep of a
 * multi-sweep launch of kind 0-2), device span in us,
 * start in us after the first traced launch, tile passes.  *n is updated to
 * the number returned. */
int pmf_debug_trace(pmf_solver *s, int32_t *kind, double *us, double *start_us, int64_t *tiles,
                    int32_t *n);

/* Diagnostics: CTA-busy milliseconds of the last asynchronous run, summed
 * over CTAs: per phase kind (BINIT, BFS, SEED, PUSH, LINIT, LAB, EMIT, -),
 * queue wait, hand-off, grid transitions; out16 holds 16 doubles. */
int pmf_debug_busy(pmf_solver *s, double *out16);

/* Diagnostics: phase timeline of grid g of the last asynchronous run made
 * with knob phase_log = 1: up to *n entries, phase << 56 | globaltimer ns;
 * *n is updated to the number returned. */
int pmf_debug_phases(pmf_solver *s, int64_t g, uint64_t *out, int32_t *n);

/* Diagnostics: copy the tile-major device state of the last run (w, h,
 * residual words, source-side flags; any pointer may be NULL) and the tile
 * count.  Buffers hold ntiles*1024 entries (r: edge_bytes each). */
int pmf_debug_state(pmf_solver *s, int32_t *w, int32_t *h, void *r, uint8_t *lab,
                    int64_t *ntiles);

#ifdef __cplusplus
}
#endif

#endif /* PMFLOW_B200_H */
