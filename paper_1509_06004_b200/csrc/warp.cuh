// warp.cuh -- warp-per-tile kernels: one warp owns one 32x32 tile in its own
// slice of shared memory; no CTA barrier anywhere, so an SM keeps 16 tiles
// in flight and a lone tile is not slowed down by 31 idle warps.
//
//   k_wpush     push-relabel discharge over the tile's ACTIVE pixels only
//               (row by row, alternating direction: Gauss-Seidel sweeps),
//               with an exact local relabel by bitset BFS
//   k_wbfs_sink exact distance to the sink (global relabel, solvers.py:54-71)
//   k_wbfs_src  residual closure of the excess pixels (solvers.py:144-158)
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

// ---------------------------------------------------------------------------
// bitset BFS: exact distance inside the tile to the sink-residual pixels
// (value 1) or to a halo pixel (its height + 1), over the pixels' own
// residual arcs.  Frozen pixels (blocked) are never reached.  Writes T.h for
// every non-blocked pixel (HINF where unreached).  m[] = own-arc row masks.
// ---------------------------------------------------------------------------
template <class E>
__device__ __forceinline__ void wt_bfs_dist(WarpTile<E> &T, int lane, const uint32_t m[4], uint32_t sinks,
                                            uint32_t blocked) {
    const int y = lane;
    // halo injections: left/right pixels of my row, top row via lane x of
    // the U halo, bottom row via lane x of the D halo
    const int32_t iL = (m[0] & 1u) && T.hh[DL][y] < HINF ? T.hh[DL][y] + 1 : HINF;
    const int32_t iR = (m[1] >> 31) && T.hh[DR][y] < HINF ? T.hh[DR][y] + 1 : HINF;
    const uint32_t m2_row0 = __shfl_sync(0xffffffffu, m[2], 0);
    const uint32_t m3_row31 = __shfl_sync(0xffffffffu, m[3], 31);
    const int32_t iU = ((m2_row0 >> lane) & 1u) && T.hh[DU][lane] < HINF ? T.hh[DU][lane] + 1 : HINF;
    const int32_t iD = ((m3_row31 >> lane) & 1u) && T.hh[DD][lane] < HINF ? T.hh[DD][lane] + 1 : HINF;
    for (int yy = 0; yy < TH; yy++) T.h[yy * TW + lane] = HINF;
    __syncwarp();
    uint32_t V = blocked;
    uint32_t F = sinks & ~V;
    int32_t L = 1;
    for (;;) {
        // injections at level L
        uint32_t inj = (iL == L ? 1u : 0u) | (iR == L ? 0x80000000u : 0u);
        uint32_t mU = __ballot_sync(0xffffffffu, iU == L);
        uint32_t mD = __ballot_sync(0xffffffffu, iD == L);
        if (lane == 0) inj |= mU;
        if (lane == 31) inj |= mD;
        F = (F | inj) & ~V;
        V |= F;
        for (uint32_t b = F; b; b &= b - 1) T.h[y * TW + (__ffs(b) - 1)] = L;
        // expand one level over pull arcs (pixel takes its d-neighbour's level + 1)
        uint32_t up = __shfl_up_sync(0xffffffffu, F, 1);
        uint32_t dn = __shfl_down_sync(0xffffffffu, F, 1);
        if (lane == 0) up = 0;
        if (lane == 31) dn = 0;
        uint32_t N = ((F << 1) & m[0]) | ((F >> 1) & m[1]) | (up & m[2]) | (dn & m[3]);
        F = N & ~V;
        ++L;
        if (!__any_sync(0xffffffffu, F != 0)) {
            // jump to the next pending injection level
            int32_t nx = HINF;
            if (iL >= L) nx = min(nx, iL);
            if (iR >= L) nx = min(nx, iR);
            if (iU >= L) nx = min(nx, iU);
            if (iD >= L) nx = min(nx, iD);
            nx = warp_min(nx);
            if (nx >= HINF) break;
            L = nx;
        }
    }
    __syncwarp();
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
// global relabel (exact distance to the sink), warp per tile
// ---------------------------------------------------------------------------
template <class E>
__global__ void __launch_bounds__(WPB * 32) k_wbfs_sink(Ctx c, int k, LaunchCtl lc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpTile<E> &T = reinterpret_cast<WarpTile<E> *>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    warp_loop(c, k, lc, [&](int32_t t) -> TileResult {
        const TileNb g = tile_nbs(c, t);
        const int64_t base = int64_t(t) * TPIX;
        wt_load<E>(c, t, T, g, lane, true, false);
        uint32_t m[4];
        wt_arc_masks<E>(T, lane, m);
        uint32_t sinks = 0;
        for (int y = 0; y < TH; y++) sinks = row_ballot_to_lane(T.w[y * TW + lane] < 0, y, lane, sinks);
        wt_bfs_dist<E>(T, lane, m, sinks, 0u);
        // relaxation from above: only ever lower the stored distance
        int out = 0;
        for (int y = 0; y < TH; y++) {
            const int p = y * TW + lane;
            const int32_t h0 = __ldcg(c.h + base + p), h1 = T.h[p];
            if (h1 < h0) {
                c.h[base + p] = h1;
                out |= (lane == 0 ? 1 << DL : 0) | (lane == TW - 1 ? 1 << DR : 0) |
                       (y == 0 ? 1 << DU : 0) | (y == TH - 1 ? 1 << DD : 0);
            }
        }
        for (int o = 16; o; o >>= 1) out |= __shfl_xor_sync(0xffffffffu, out, o);
        return TileResult{0, out};
    });
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

// ---------------------------------------------------------------------------
// discharge, warp per tile
// ---------------------------------------------------------------------------
template <class E>
__device__ __forceinline__ void wt_local_relabel(WarpTile<E> &T, int lane) {
    uint32_t m[4];
    wt_arc_masks<E>(T, lane, m);
    uint32_t sinks = 0, frozen = 0;
    for (int y = 0; y < TH; y++) {
        const int p = y * TW + lane;
        sinks = row_ballot_to_lane(T.w[p] < 0, y, lane, sinks);
        frozen = row_ballot_to_lane(T.h[p] >= HINF, y, lane, frozen);
    }
    wt_bfs_dist<E>(T, lane, m, sinks, frozen);   // frozen pixels keep HINF
    uint32_t a = 0;
    for (int y = 0; y < TH; y++) {
        const int p = y * TW + lane;
        a = row_ballot_to_lane(T.w[p] > 0 && T.h[p] < HINF, y, lane, a);
    }
    T.act[lane] = a;
    __syncwarp();
}

template <class E>
__global__ void __launch_bounds__(WPB * 32) k_wpush(Ctx c, int k, int rounds, int relabel_every, LaunchCtl lc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpTile<E> &T = reinterpret_cast<WarpTile<E> *>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    warp_loop(c, k, lc, [&](int32_t t) -> TileResult {
        const TileNb g = tile_nbs(c, t);
        const int64_t base = int64_t(t) * TPIX;
        wt_load<E>(c, t, T, g, lane, true, true);
        // snapshots of the border pixels for delta write-back: lane x keeps
        // (x, 0) and (x, 31); lane y keeps (0, y) and (31, y)
        const int32_t sw_t = T.w[lane], sw_b = T.w[31 * TW + lane];
        const int32_t sw_l = T.w[lane * TW], sw_r = T.w[lane * TW + 31];
        const auto sr_t = SRes<E>::pack(T.r, lane), sr_b = SRes<E>::pack(T.r, 31 * TW + lane);
        const auto sr_l = SRes<E>::pack(T.r, lane * TW), sr_r = SRes<E>::pack(T.r, lane * TW + 31);
        bool any = true;
        for (int rd = 0; rd < rounds && any; rd++) {
            if (relabel_every ? (rd % relabel_every == 0) : (rd == 0)) {
                if (relabel_every) wt_local_relabel<E>(T, lane);
                else {
                    uint32_t a = 0;
                    for (int y = 0; y < TH; y++) {
                        const int p = y * TW + lane;
                        a = row_ballot_to_lane(T.w[p] > 0 && T.h[p] < HINF, y, lane, a);
                    }
                    T.act[lane] = a;
                    __syncwarp();
                }
            }
            // one Gauss-Seidel sweep over the rows holding active pixels
            const bool up = rd & 1;
            for (int yy = 0; yy < TH; yy++) {
                const int y = up ? TH - 1 - yy : yy;
                const uint32_t rowm = T.act[y];
                if (!rowm) continue;
                if ((rowm >> lane) & 1) {
                    atomicAnd(&T.act[y], ~(1u << lane));
                    const int p = y * TW + lane;
                    int32_t e = T.w[p];
                    int32_t hp = T.h[p];
                    if (e > 0 && hp < HINF) {
                        const auto word = SRes<E>::word(T.r, p);
                        int32_t hn[4];
                        hn[DL] = lane > 0 ? T.h[p - 1] : T.hh[DL][y];
                        hn[DR] = lane < TW - 1 ? T.h[p + 1] : T.hh[DR][y];
                        hn[DU] = y > 0 ? T.h[p - TW] : T.hh[DU][lane];
                        hn[DD] = y < TH - 1 ? T.h[p + TW] : T.hh[DD][lane];
                        const int qi[4] = {p - 1, p + 1, p - TW, p + TW};
                        const bool in[4] = {lane > 0, lane < TW - 1, y > 0, y < TH - 1};
                        const int hpos[4] = {y, y, lane, lane};
                        int32_t sent = 0;
                        int32_t mlow = HINF;
#pragma unroll
                        for (int d = 0; d < 4; d++) {
                            const int32_t rr = SRes<E>::lane(word, d);
                            if (rr <= 0) continue;
                            if (e > 0 && hp > hn[d]) {
                                const int32_t dl = min(e, rr);
                                e -= dl;
                                sent += dl;
                                SRes<E>::add(T.r, p, d, -dl);
                                if (in[d]) {
                                    const int q = qi[d];
                                    atomicAdd(&T.w[q], dl);
                                    SRes<E>::add(T.r, q, opp(d), dl);
                                    atomicOr(&T.act[q >> 5], 1u << (q & 31));
                                } else {
                                    T.hacc[d][hpos[d]] += dl;
                                }
                                if (rr > dl) mlow = min(mlow, hn[d]);
                            } else {
                                mlow = min(mlow, hn[d]);
                            }
                        }
                        if (sent) atomicSub(&T.w[p], sent);
                        if (e > 0) {
                            // no residual arc left downhill: relabel over the
                            // current arcs (inflows may have opened reverse arcs)
                            const auto w2 = SRes<E>::word(T.r, p);
                            mlow = HINF;
#pragma unroll
                            for (int d = 0; d < 4; d++)
                                if (SRes<E>::lane(w2, d) > 0) mlow = min(mlow, hn[d]);
                            if (mlow >= hp) {
                                hp = mlow >= HINF ? HINF : mlow + 1;
                                T.h[p] = hp;
                            }
                            if (hp < HINF) atomicOr(&T.act[y], 1u << lane);
                        }
                    }
                }
                __syncwarp();
            }
            any = __any_sync(0xffffffffu, T.act[lane] != 0);
        }
        // ---- write back (interior plainly, border pixels as deltas)
        for (int y = 0; y < TH; y++) {
            const int p = y * TW + lane;
            const int64_t gp = base + p;
            const int32_t e = T.w[p];
            const auto rw = SRes<E>::pack(T.r, p);
            const bool border = y == 0 || y == TH - 1 || lane == 0 || lane == TW - 1;
            if (!border) {
                c.w[gp] = e;
                E::store(c.r, gp, rw);
            }
            c.h[gp] = T.h[p];
        }
        // border pixels: (x, 0) and (x, 31) by lane x; (0, y) and (31, y) by
        // lane y for y in 1..30
        {
            const int pt = lane, pb = 31 * TW + lane;
            if (T.w[pt] != sw_t) atomicAdd(&c.w[base + pt], T.w[pt] - sw_t);
            E::store_delta(c.r, base + pt, SRes<E>::pack(T.r, pt), sr_t);
            if (T.w[pb] != sw_b) atomicAdd(&c.w[base + pb], T.w[pb] - sw_b);
            E::store_delta(c.r, base + pb, SRes<E>::pack(T.r, pb), sr_b);
            if (lane > 0 && lane < TH - 1) {
                const int pl = lane * TW, pr = lane * TW + 31;
                if (T.w[pl] != sw_l) atomicAdd(&c.w[base + pl], T.w[pl] - sw_l);
                E::store_delta(c.r, base + pl, SRes<E>::pack(T.r, pl), sr_l);
                if (T.w[pr] != sw_r) atomicAdd(&c.w[base + pr], T.w[pr] - sw_r);
                E::store_delta(c.r, base + pr, SRes<E>::pack(T.r, pr), sr_r);
            }
        }
        int out = 0;
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const int32_t a = T.hacc[s][lane];
            if (a > 0) {
                const int64_t q = int64_t(g.nb[s]) * TPIX + halo_index(s, lane);
                atomicAdd(&c.w[q], a);
                E::add(c.r, q, opp(s), a);
                out |= 1 << s;
            }
        }
        for (int o = 16; o; o >>= 1) out |= __shfl_xor_sync(0xffffffffu, out, o);
        const int again = __any_sync(0xffffffffu, T.act[lane] != 0);
        __syncwarp();
        return TileResult{again, out};
    });
}

}  // namespace pmf
