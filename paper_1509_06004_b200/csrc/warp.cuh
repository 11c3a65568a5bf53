// warp.cuh -- warp-per-tile kernels: one warp owns one 32x32 tile, held in
// registers as row bitsets; no CTA barrier and no shared memory, so an SM
// keeps as many tiles in flight as its register file allows and a lone tile
// is not slowed down by 31 idle warps.
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

#ifndef PMF_WPB
#define PMF_WPB 4
#endif
constexpr int WPB = PMF_WPB;   // warps (tiles) per CTA

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
        // one pass over the tile's rows (lane = column, every load one
        // coalesced line): lane y receives row y's words -- own arcs
        // (bit x of m[d] = r_d(x, y) > 0), sources (excess or already
        // reached), reached, sink-residual
        uint32_t m[4] = {0u, 0u, 0u, 0u}, R = 0, L0 = 0, NEG = 0;
#pragma unroll 4
        for (int y = 0; y < TH; y++) {
            const int64_t p = base + y * TW + lane;
            const typename E::Word wd = E::load(c.r, p);
            const int32_t wv = __ldcg(c.w + p);
            const bool lab = __ldcg(c.lab + p) != 0;
            const uint32_t b0 = __ballot_sync(0xffffffffu, E::lane(wd, 0) > 0);
            const uint32_t b1 = __ballot_sync(0xffffffffu, E::lane(wd, 1) > 0);
            const uint32_t b2 = __ballot_sync(0xffffffffu, E::lane(wd, 2) > 0);
            const uint32_t b3 = __ballot_sync(0xffffffffu, E::lane(wd, 3) > 0);
            const uint32_t bs = __ballot_sync(0xffffffffu, lab || wv > 0);
            const uint32_t bl = __ballot_sync(0xffffffffu, lab);
            const uint32_t bn = __ballot_sync(0xffffffffu, wv < 0);
            if (lane == y) {
                m[0] = b0; m[1] = b1; m[2] = b2; m[3] = b3;
                R = bs; L0 = bl; NEG = bn;
            }
        }
        // pull masks (arcs INTO each pixel) from the neighbours' own arcs
        const uint32_t mD_above = __shfl_up_sync(0xffffffffu, m[3], 1);
        const uint32_t mU_below = __shfl_down_sync(0xffffffffu, m[2], 1);
        uint32_t PL = m[1] << 1, PR = m[0] >> 1;
        uint32_t PU = lane > 0 ? mD_above : 0u, PD = lane < 31 ? mU_below : 0u;
        // sources also: reached halo pixels whose arc into the tile is residual
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
            const int x = __ffs(b) - 1;
            c.lab[base + lane * TW + x] = 1;
            out |= (x == 0 ? 1 << DL : 0) | (x == TW - 1 ? 1 << DR : 0);
        }
        if (fresh & NEG) {
            const int32_t gid = __ldg(c.tile_grid + t);
            if (c.specg && __ldcg(c.specg + gid)) c.specg[gid] = 2;   // speculative: spoiled
            else atomicExch(c.err, 4);
        }
        if (fresh) out |= (lane == 0 ? 1 << DU : 0) | (lane == 31 ? 1 << DD : 0);
        for (int o = 16; o; o >>= 1) out |= __shfl_xor_sync(0xffffffffu, out, o);
        return TileResult{0, out};
    });
}

}  // namespace pmf
