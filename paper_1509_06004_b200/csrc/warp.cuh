// warp.cuh -- warp-per-tile kernels: one warp owns one 32x32 tile in its own
// slice of shared memory; no CTA barrier anywhere, so an SM keeps 16 tiles
// in flight and a lone tile is not slowed down by 31 idle warps.
//
//   k_wbfs_src  residual closure of the excess pixels (solvers.py:144-158)
//
// (Warp-per-tile discharge and sink-distance kernels were measured against
// the 1024-thread CTA kernels and lost: a lone warp's tile pass is ~3x
// slower; they were removed.)
//
// Bitset representation: lane y holds 32-bit row words (bit x = pixel
// (x, y)); horizontal moves are shifts, vertical moves are shuffles.
#pragma once
#include "engine.cuh"
#include "tile.cuh"

namespace pmf {

constexpr int WPB = 4;   // warps (tiles) per CTA

// ---------------------------------------------------------------------------
// shared-memory residual words per policy
// ---------------------------------------------------------------------------
template <class E> struct SRes;

template <> struct SRes<EdgeU8> {
    static constexpr int kWords = 1;   // uint32 per pixel
    __device__ static int get(const uint32_t *s, int p, int d) { return int((s[p] >> (8 * d)) & 0xffu); }
    __device__ static uint32_t word(const uint32_t *s, int p) { return s[p]; }
    __device__ static int lane(uint32_t w, int d) { return int((w >> (8 * d)) & 0xffu); }
    __device__ static void add(uint32_t *s, int p, int d, int v) { atomicAdd(s + p, uint32_t(v) << (8 * d)); }
    __device__ static void put(uint32_t *s, int p, EdgeU8::Word w) { s[p] = w; }
    __device__ static EdgeU8::Word pack(const uint32_t *s, int p) { return s[p]; }
};

template <> struct SRes<EdgeI32> {
    static constexpr int kWords = 4;
    __device__ static int get(const uint32_t *s, int p, int d) { return int(s[4 * p + d]); }
    __device__ static int4 word(const uint32_t *s, int p) { return *reinterpret_cast<const int4 *>(s + 4 * p); }
    __device__ static int lane(int4 w, int d) { return d == 0 ? w.x : d == 1 ? w.y : d == 2 ? w.z : w.w; }
    __device__ static void add(uint32_t *s, int p, int d, int v) { atomicAdd(reinterpret_cast<int *>(s) + 4 * p + d, v); }
    __device__ static void put(uint32_t *s, int p, int4 w) { *reinterpret_cast<int4 *>(s + 4 * p) = w; }
    __device__ static int4 pack(const uint32_t *s, int p) { return *reinterpret_cast<const int4 *>(s + 4 * p); }
};

template <class E>
struct WarpTile {
    int32_t w[TPIX];                       // excess (> 0) / -sink residual
    int32_t h[TPIX];                       // heights / distances
    uint32_t r[TPIX * SRes<E>::kWords];    // residual words
    int32_t hh[4][TW];                     // halo heights
    int32_t hacc[4][TW];                   // flow pushed into halo pixels
    uint32_t act[TH];                      // active pixels, one word per row
};

__device__ __forceinline__ unsigned lanemask_all() { return 0xffffffffu; }

__device__ __forceinline__ int32_t warp_min(int32_t v) {
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------------------
// tile load / store (lane = column, loop over rows: every access is one
// coalesced 128 B line per plane)
// ---------------------------------------------------------------------------
template <class E>
__device__ __forceinline__ void wt_load(const Ctx &c, int32_t t, WarpTile<E> &T, const TileNb &g, int lane,
                                        bool want_w, bool want_h) {
    const int64_t base = int64_t(t) * TPIX;
#pragma unroll 4
    for (int y = 0; y < TH; y++) {
        const int p = y * TW + lane;
        if (want_w) T.w[p] = __ldcg(c.w + base + p);
        if (want_h) T.h[p] = __ldcg(c.h + base + p);
        SRes<E>::put(T.r, p, E::load(c.r, base + p));
    }
#pragma unroll
    for (int s = 0; s < 4; s++) {
        T.hh[s][lane] = g.nb[s] >= 0 ? __ldcg(c.h + int64_t(g.nb[s]) * TPIX + halo_index(s, lane)) : HINF;
        T.hacc[s][lane] = 0;
    }
    __syncwarp();
}

// Row masks of the pull arcs of lane y's row (bit x: pixel (x, y) has a
// residual arc toward its d-neighbour) -- built with one ballot per row.
template <class E>
__device__ __forceinline__ void wt_arc_masks(const WarpTile<E> &T, int lane, uint32_t m[4]) {
    m[0] = m[1] = m[2] = m[3] = 0;
    for (int y = 0; y < TH; y++) {
        const int p = y * TW + lane;
        uint32_t b0 = __ballot_sync(0xffffffffu, SRes<E>::get(T.r, p, 0) > 0);
        uint32_t b1 = __ballot_sync(0xffffffffu, SRes<E>::get(T.r, p, 1) > 0);
        uint32_t b2 = __ballot_sync(0xffffffffu, SRes<E>::get(T.r, p, 2) > 0);
        uint32_t b3 = __ballot_sync(0xffffffffu, SRes<E>::get(T.r, p, 3) > 0);
        if (lane == y) { m[0] = b0; m[1] = b1; m[2] = b2; m[3] = b3; }
    }
}

__device__ __forceinline__ uint32_t row_ballot_to_lane(bool pred, int y, int lane, uint32_t cur) {
    uint32_t b = __ballot_sync(0xffffffffu, pred);
    return lane == y ? b : cur;
}

// Kogge-Stone fills along a row word: every bit reachable from a set bit of G
// through consecutive propagate bits of P (pull from the left / right).
__device__ __forceinline__ uint32_t fill_from_left(uint32_t G, uint32_t P) {
    P &= ~1u;
    G |= P & (G << 1); P &= P << 1;
    G |= P & (G << 2); P &= P << 2;
    G |= P & (G << 4); P &= P << 4;
    G |= P & (G << 8); P &= P << 8;
    G |= P & (G << 16);
    return G;
}
__device__ __forceinline__ uint32_t fill_from_right(uint32_t G, uint32_t P) {
    P &= ~0x80000000u;
    G |= P & (G >> 1); P &= P >> 1;
    G |= P & (G >> 2); P &= P >> 2;
    G |= P & (G >> 4); P &= P >> 4;
    G |= P & (G >> 8); P &= P >> 8;
    G |= P & (G >> 16);
    return G;
}
// the same across lanes (bit columns independent): pull from the row above
__device__ __forceinline__ uint32_t fill_from_up(uint32_t G, uint32_t P, int lane) {
    if (lane == 0) P = 0;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        uint32_t g = __shfl_up_sync(0xffffffffu, G, s);
        uint32_t p = __shfl_up_sync(0xffffffffu, P, s);
        if (lane >= s) {
            G |= P & g;
            P &= p;
        }
    }
    return G;
}
__device__ __forceinline__ uint32_t fill_from_down(uint32_t G, uint32_t P, int lane) {
    if (lane == 31) P = 0;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        uint32_t g = __shfl_down_sync(0xffffffffu, G, s);
        uint32_t p = __shfl_down_sync(0xffffffffu, P, s);
        if (lane + s < 32) {
            G |= P & g;
            P &= p;
        }
    }
    return G;
}

// ---------------------------------------------------------------------------
// warp-level tile loop: sweep mode (list k / K_DEVICE) or persistent queue
// ---------------------------------------------------------------------------
template <class Body>
__device__ __forceinline__ void warp_loop(const Ctx &c, int k, const LaunchCtl &lc, Body &&body) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * WPB + (threadIdx.x >> 5);
    const int nw = gridDim.x * WPB;
    if (k == K_MULTI) {   // as in tile_loop: all sweeps, grid barriers between them
        if (lane == 0) atomicMin(&c.ctl->t0, gtimer());
        int kk = *(volatile int32_t *)&c.ctl->k, sweeps = 0;
        for (;;) {
            const int32_t n = *(volatile int32_t *)&c.cnt[kk % 3];
            if (n == 0) break;
            const int32_t *lst = list_of(c, kk);
            __syncthreads();   // every warp has read n before block 0 resets a list
            if (gw == 0 && lane == 0) {
                c.cnt[(kk + 2) % 3] = 0;
                atomicAdd(&c.stat[lc.stat], (unsigned long long)n);
            }
            for (int li = gw; li < n; li += nw) {
                const int32_t t = __ldcg(lst + li);
                if (lane == 0) inq_of(c, kk)[t] = 0;
                TileResult r = body(t);
                if (lane < 5) enqueue_follow(c, kk + 1, t, r, lane);
                __syncwarp();
            }
            grid_sync(c.ctl, sweeps);
            kk++;
            sweeps++;
        }
        if (threadIdx.x == 0) {
            if (blockIdx.x == 0) {
                c.ctl->k = kk;
                if (sweeps > 1) atomicAdd(&c.stat[ST_PUSH_L + lc.stat], (unsigned long long)(sweeps - 1));
            }
            launch_exit(c, lc, -1, gridDim.x);
        }
        return;
    }
    if (k != K_PERSISTENT) {
        if (k == K_DEVICE) k = *(volatile int32_t *)&c.ctl->k;
        const int32_t n = *(volatile int32_t *)&c.cnt[k % 3];
        const unsigned parts = unsigned(max(1, min(n, nw)));
        if (unsigned(gw) >= parts) return;
        if (lane == 0) atomicMin(&c.ctl->t0, gtimer());
        const int32_t *lst = list_of(c, k);
        if (gw == 0 && lane == 0) {
            c.cnt[(k + 2) % 3] = 0;
            atomicAdd(&c.stat[lc.stat], (unsigned long long)n);
        }
        for (int li = gw; li < n; li += nw) {
            const int32_t t = lst[li];
            if (lane == 0) inq_of(c, k)[t] = 0;
            TileResult r = body(t);
            if (lane < 5) enqueue_follow(c, k + 1, t, r, lane);
            __syncwarp();
        }
        if (lane == 0) launch_exit(c, lc, k + 1, parts);
        return;
    }
    if (lane == 0) atomicMin(&c.ctl->t0, gtimer());
    // hand-off ordering as in tile_loop: gpu-scope SC fences in every lane
    // on both sides of the warp's hand-off to lane 0
    for (;;) {
        int32_t t = 0;
        if (lane == 0) {
            t = q_next(c);
            __threadfence();
        }
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t < 0) break;
        __threadfence();
        TileResult r = body(t);
        __threadfence();
        __syncwarp();
        q_follow(c, t, r, lane, lc.stat);
        __syncwarp();
    }
    if (lane == 0) launch_exit(c, lc, -1, unsigned(nw));
}

// ---------------------------------------------------------------------------
// source-side closure, warp per tile (cost-0 flood fill with bitsets)
// ---------------------------------------------------------------------------
template <class E>
__global__ void __launch_bounds__(WPB * 32) k_wbfs_src(Ctx c, int k, LaunchCtl lc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpTile<E> &T = reinterpret_cast<WarpTile<E> *>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    warp_loop(c, k, lc, [&](int32_t t) -> TileResult {
        const TileNb g = tile_nbs(c, t);
        const int64_t base = int64_t(t) * TPIX;
        if (c.labok) {   // nested seeding: a tile already inside the closure cannot change
            bool full = true;
#pragma unroll 8
            for (int y = 0; y < TH; y++) full &= __ldcg(c.lab + base + y * TW + lane) != 0;
            if (__all_sync(0xffffffffu, full)) return TileResult{0, 0};
        }
        wt_load<E>(c, t, T, g, lane, true, false);
        uint32_t m[4];   // own arcs: bit x of m[d] = r_d(x, y) > 0
        wt_arc_masks<E>(T, lane, m);
        // pull masks (arcs INTO each pixel) from the neighbours' own arcs
        const uint32_t mD_above = __shfl_up_sync(0xffffffffu, m[3], 1);
        const uint32_t mU_below = __shfl_down_sync(0xffffffffu, m[2], 1);
        uint32_t PL = m[1] << 1, PR = m[0] >> 1;
        uint32_t PU = lane > 0 ? mD_above : 0u, PD = lane < 31 ? mU_below : 0u;
        // sources: excess pixels, previously reached pixels, reached halo
        // pixels whose arc into the tile is residual
        uint32_t R = 0, L0 = 0;
        for (int y = 0; y < TH; y++) {
            const int p = y * TW + lane;
            const bool lab = __ldcg(c.lab + base + p) != 0;
            R = row_ballot_to_lane(lab || T.w[p] > 0, y, lane, R);
            L0 = row_ballot_to_lane(lab, y, lane, L0);
        }
        // halo: left/right pixel of my row, top/bottom rows by ballot
        if (g.nb[DL] >= 0) {
            const int64_t q = int64_t(g.nb[DL]) * TPIX + halo_index(DL, lane);
            if (__ldcg(c.lab + q) && E::lane(E::load(c.r, q), DR) > 0) R |= 1u;
        }
        if (g.nb[DR] >= 0) {
            const int64_t q = int64_t(g.nb[DR]) * TPIX + halo_index(DR, lane);
            if (__ldcg(c.lab + q) && E::lane(E::load(c.r, q), DL) > 0) R |= 0x80000000u;
        }
        bool tu = false, td = false;
        if (g.nb[DU] >= 0) {
            const int64_t q = int64_t(g.nb[DU]) * TPIX + halo_index(DU, lane);
            tu = __ldcg(c.lab + q) && E::lane(E::load(c.r, q), DD) > 0;
        }
        if (g.nb[DD] >= 0) {
            const int64_t q = int64_t(g.nb[DD]) * TPIX + halo_index(DD, lane);
            td = __ldcg(c.lab + q) && E::lane(E::load(c.r, q), DU) > 0;
        }
        const uint32_t bu = __ballot_sync(0xffffffffu, tu), bd = __ballot_sync(0xffffffffu, td);
        if (lane == 0) R |= bu;
        if (lane == 31) R |= bd;
        // flood fill to the fixpoint
        for (;;) {
            uint32_t R0 = R;
            R = fill_from_left(R, PL);
            R = fill_from_right(R, PR);
            R = fill_from_up(R, PU, lane);
            R = fill_from_down(R, PD, lane);
            if (!__any_sync(0xffffffffu, R != R0)) break;
        }
        // write newly reached pixels; reaching a sink-residual pixel means
        // the preflow was not maximal (NonMaximalFlowError)
        const uint32_t fresh = R & ~L0;
        int out = 0;
        for (uint32_t b = fresh; b; b &= b - 1) {
            const int x = __ffs(b) - 1, p = lane * TW + x;
            c.lab[base + p] = 1;
            if (T.w[p] < 0) {
                const int32_t gid = __ldg(c.tile_grid + t);
                if (c.specg && __ldcg(c.specg + gid)) c.specg[gid] = 2;   // speculative: spoiled
                else atomicExch(c.err, 4);
            }
            out |= (x == 0 ? 1 << DL : 0) | (x == TW - 1 ? 1 << DR : 0);
        }
        if (fresh) out |= (lane == 0 ? 1 << DU : 0) | (lane == 31 ? 1 << DD : 0);
        for (int o = 16; o; o >>= 1) out |= __shfl_xor_sync(0xffffffffu, out, o);
        return TileResult{0, out};
    });
}

}  // namespace pmf
