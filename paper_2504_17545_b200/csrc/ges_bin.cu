// Sort-free tile binning, steps 2 and 3 (step 1, the count, is fused into the
// preprocess kernels).  Replaces the per-tile O(N) selection scan of the
// reference (forward.py:168-169, :294-295) -- the reference's dominant CPU cost.
//
// Bins are (tile, depth slab) pairs: every primitive is counted into the
// NSLAB slab of its conservative depth key in each tile it overlaps.  Within a
// tile the slabs are laid out near to far, so the tile kernel meets near
// primitives first (its depth culling then rejects most of the rest) and can
// stop at the first slab that lies behind everything already drawn.  Results
// never depend on the order (min over packed keys / order-independent sums).
//
//   count (prep) -> k_scan: per-tile slab prefix + prefix sum over tiles
//                -> k_fill: append ids, one atomic per (warp, bin) group
#include <cub/block/block_scan.cuh>

#include "ges_launch.h"

namespace ges {

constexpr int SCAN_T = 256;                   // threads per scan block
constexpr int SCAN_W = 1 << SCAN_CHUNK_SHIFT; // tiles per scan block, SCAN_TPW per warp
constexpr int SCAN_TPW = SCAN_W / (SCAN_T / 32);
static_assert(SCAN_TPW >= 1 && SCAN_TPW * (SCAN_T / 32) == SCAN_W, "tiles per warp");

// Grid (ceil(ntiles / SCAN_W), 2): y selects the pass (0 = surfels, 1 =
// Gaussians).  Each warp turns SCAN_TPW tiles' slab counts into slab prefixes
// (the fill cursors) with two coalesced loads and a shuffle scan per tile; each block
// writes the block-local exclusive prefix of its tiles' totals and its sum;
// the last block of a pass to finish scans the block sums into chunk bases,
// so tile_off(t) = chunk_base[t / SCAN_W] + local_off[t].  One launch, no host
// sync; the ticket is reset with the per-frame counter memset.
__global__ void __launch_bounds__(SCAN_T) k_scan(BinPass p0, BinPass p1, ges_frame_status_t* st) {
    using Scan = cub::BlockScan<uint32_t, SCAN_T>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t wtot[SCAN_W];
    __shared__ bool last;
    const BinPass& p = blockIdx.y ? p1 : p0;
    const int n = p.ntiles;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int R = (NSLAB + 31) / 32;   // 32-slab rounds per tile
    uint32_t v[SCAN_TPW][R];
#pragma unroll
    for (int k = 0; k < SCAN_TPW; ++k) {   // all loads in flight first
        const int t = blockIdx.x * SCAN_W + w * SCAN_TPW + k;
        const uint32_t* c = p.cnt + (size_t)t * NSLAB;
#pragma unroll
        for (int r = 0; r < R; ++r) v[k][r] = (t < n && 32 * r + lane < NSLAB) ? __ldcg(c + 32 * r + lane) : 0u;
    }
#pragma unroll
    for (int k = 0; k < SCAN_TPW; ++k) {
        const int t = blockIdx.x * SCAN_W + w * SCAN_TPW + k;
        uint32_t run = 0;   // slabs of the earlier rounds
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t inc = v[k][r];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += a;
            }
            if (t < n && 32 * r + lane < NSLAB) p.cnt[(size_t)t * NSLAB + 32 * r + lane] = run + inc - v[k][r];
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) wtot[w * SCAN_TPW + k] = run;
    }
    __syncthreads();
    if (w == 0) {   // block-local exclusive prefix of the SCAN_W (<= 32) tile totals
        static_assert(SCAN_W <= 32, "one warp scans the block's tile totals");
        const uint32_t v = lane < SCAN_W ? wtot[lane] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < SCAN_W; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += a;
        }
        const int tl = blockIdx.x * SCAN_W + lane;
        if (lane < SCAN_W && tl < n) {
            p.off[tl] = inc - v;
            if (p.order) p.tot[tl] = v;
        }
        if (lane == SCAN_W - 1) p.chunk[blockIdx.x] = inc;
    }
    // every off/tot/chunk store must be ordered before the ticket: the last
    // block reads them as soon as the ticket says all blocks are done
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(p.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // last block: exclusive scan of the block sums, `per` consecutive ones per thread
    const int nc = gridDim.x;
    const int per = (nc + SCAN_T - 1) / SCAN_T;
    const int c0 = threadIdx.x * per, c1 = min(c0 + per, nc);
    uint32_t run = 0;
    for (int i = c0; i < c1; ++i) run += *((volatile uint32_t*)p.chunk + i);
    uint32_t base, total;
    Scan(tmp).ExclusiveSum(run, base, total);
    for (int i = c0; i < c1; ++i) {
        const uint32_t v = *((volatile uint32_t*)p.chunk + i);
        p.chunk[i] = base;
        base += v;
    }
    if (threadIdx.x == 0) {
        p.chunk[nc] = total;
        if (blockIdx.y) st->gaussian_pairs = total; else st->surfel_pairs = total;
        if ((int64_t)total > p.cap) atomicOr(&st->overflow, 1);
    }
    if (!p.order) return;
    // Tile launch order for the tile kernel: by descending pair count
    // (counting sort over log2 buckets), so the longest tiles start first and
    // do not end up as the last wave's tail.  Any order gives the same
    // results (tiles are independent).
    __shared__ uint32_t bucket[33];
    if (threadIdx.x < 33) bucket[threadIdx.x] = 0;
    constexpr int PER = 8;   // tiles per thread (n <= 2048 here; larger grids loop)
    const unsigned ln = threadIdx.x & 31, lt = (1u << ln) - 1u;
    for (int c0 = 0; c0 < n; c0 += SCAN_T * PER) {
        int bk[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {   // all loads first: one round trip, not PER
            const int i = c0 + k * SCAN_T + threadIdx.x;
            bk[k] = i < n ? (int)*((volatile uint32_t*)p.tot + i) : -1;
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) bk[k] = bk[k] < 0 ? -1 : 32 - __clz((uint32_t)bk[k]);
        __syncthreads();   // (bucket cleared / previous scatter done)
#pragma unroll
        for (int k = 0; k < PER; ++k) {   // one shared atomic per (warp, bucket)
            const unsigned peers = __match_any_sync(0xffffffffu, bk[k]);
            if (bk[k] >= 0 && (peers & lt) == 0) atomicAdd(&bucket[bk[k]], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 32; b >= 0; --b) {
            const uint32_t c = bucket[b];
            bucket[b] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int c0 = 0; c0 < n; c0 += SCAN_T * PER) {
        int bk[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = c0 + k * SCAN_T + threadIdx.x;
            bk[k] = i < n ? (int)*((volatile uint32_t*)p.tot + i) : -1;
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = c0 + k * SCAN_T + threadIdx.x;
            const int b = bk[k] < 0 ? -1 : 32 - __clz((uint32_t)bk[k]);
            const unsigned peers = __match_any_sync(0xffffffffu, b);
            const int leader = __ffs(peers) - 1;
            uint32_t pos = 0;
            if (b >= 0 && (int)ln == leader) pos = atomicAdd(&bucket[b], (uint32_t)__popc(peers));
            pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(peers & lt);
            if (b >= 0) p.order[pos] = (uint32_t)i;
        }
    }
}

cudaError_t launch_scan(const BinPass& s, const BinPass& g, ges_frame_status_t* status, cudaStream_t st) {
    const int nc = (s.ntiles + SCAN_W - 1) / SCAN_W;
    if (nc == 0) return cudaSuccess;
    k_scan<<<dim3(nc, 2), SCAN_T, 0, st>>>(s, g, status);
    return cudaGetLastError();
}

// Append `id` to bin (tile, slab) of every tile of its range.  Called by all
// lanes of a warp whose lanes all belong to the same primitive class; lanes
// that hit the same bin in the same round reserve their slots with a single
// atomic.  The atomics of up to FILL_R rounds are issued back to back (their
// results parked in registers) before any slot is written, so their L2 round
// trips overlap instead of serialising; longer ranges finish in a plain loop.
#ifndef GES_FILL_R
#define GES_FILL_R 4
#endif
constexpr int FILL_R = GES_FILL_R;

__device__ __forceinline__ void fill_one(bool live, uint32_t id, uint32_t sx, uint32_t sy, int slab,
                                         const BinPass& p) {
    const int x0 = span_lo(sx), x1 = span_hi(sx), y0 = span_lo(sy), y1 = span_hi(sy);
    bool more = live && x1 >= x0 && y1 >= y0;
    const int sh = p.tile_shift;   // tiles are 16 or 32 px: shifts, not divisions
    const int tx0 = x0 >> sh, tx1 = x1 >> sh, ty1 = y1 >> sh;
    int ty = y0 >> sh, tx = tx0;
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t base_r[FILL_R], toff_r[FILL_R], peers_r[FILL_R];
    bool act_r[FILL_R];
    // rounds this warp needs (most primitives touch 1-4 tiles): the unrolled
    // batches below stop at the warp's largest tile count
    int ntl = more ? (tx1 - tx0 + 1) * (ty1 - (y0 >> sh) + 1) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) ntl = max(ntl, __shfl_xor_sync(0xffffffffu, ntl, o));
#pragma unroll
    for (int r = 0; r < FILL_R; ++r) {
        act_r[r] = more;
        peers_r[r] = 0u;
        base_r[r] = 0u;
        toff_r[r] = 0u;
        if (r < ntl) {
            const int tile = ty * p.ntx + tx;
            const int key = more ? tile * NSLAB + slab : -1;
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            if (more) {
                peers_r[r] = peers;
                toff_r[r] = p.tile_off(tile);
                if (lane == (unsigned)(__ffs(peers) - 1))
                    base_r[r] = atomicAdd(p.cnt + key, (uint32_t)__popc(peers));
            }
            const bool wrap = tx >= tx1;   // next tile, row-major over the range (branch-free)
            tx = wrap ? tx0 : tx + 1;
            ty += wrap;
            more = more && !(wrap && ty > ty1);
        }
    }
#pragma unroll
    for (int r = 0; r < FILL_R; ++r) {
        if (r >= ntl) break;
        // every lane of a group takes its leader's base (inactive lanes form their own groups)
        const int leader = act_r[r] ? __ffs(peers_r[r]) - 1 : (int)lane;
        const uint32_t b = __shfl_sync(0xffffffffu, base_r[r], leader);
        if (act_r[r]) {
            const uint32_t slot = toff_r[r] + b + __popc(peers_r[r] & lt);
            if ((int64_t)slot < p.cap) p.list[slot] = id;
        }
    }
    while (__any_sync(0xffffffffu, more)) {   // ranges wider than FILL_R tiles
        const int tile = ty * p.ntx + tx;
        const int key = more ? tile * NSLAB + slab : -1;
        const uint32_t toff = more ? p.tile_off(tile) : 0u;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        if (more) {
            const int leader = __ffs(peers) - 1;
            uint32_t base = 0;
            if (lane == (unsigned)leader) base = atomicAdd(p.cnt + key, (uint32_t)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            const uint32_t slot = toff + base + __popc(peers & lt);
            if ((int64_t)slot < p.cap) p.list[slot] = id;
            if (++tx > tx1) { tx = tx0; if (++ty > ty1) more = false; }
        }
    }
}

// Surfel blocks first, then Gaussian blocks, so every warp is one class.
__global__ void __launch_bounds__(256) k_fill(const float4* __restrict__ scull, int64_t ns, BinPass ps,
                                              const float4* __restrict__ gcull, int64_t ng, int g_kind, BinPass pg,
                                              SlabMap sm) {
    // launched as a dependent of the scan: the cull records (preprocess output) are read
    // before pdl_wait, the scan's offsets and cursors only after it
    const unsigned sblocks = (unsigned)((ns + 255) >> 8);   // blockDim.x == 256
    if (blockIdx.x < sblocks) {
        const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        const bool live = i < ns;
        const float4 r3 = live ? __ldg(scull + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        pdl_wait();
        fill_one(live, (uint32_t)i, __float_as_uint(r3.y), __float_as_uint(r3.z), sm.slab(r3.x), ps);
    } else {
        const int64_t j = (int64_t)(blockIdx.x - sblocks) * 256 + threadIdx.x;
        const bool live = j < ng;
        uint32_t sx = 0, sy = 0;
        float key = 0.f;
        if (live) {   // cull fields: c = (depth or key, eps, rect_x, rect_y)
            const float4 c = __ldg(gcull + j);
            sx = __float_as_uint(c.z); sy = __float_as_uint(c.w);
            key = g_kind == 2 ? c.x : gauss_key(c.x, c.y);
        }
        pdl_wait();
        fill_one(live, (uint32_t)j, sx, sy, sm.slab(key), pg);
    }
}

cudaError_t launch_fill(const float4* scull, int64_t ns, const BinPass& ps, const float4* gcull, int64_t ng, int g_kind,
                        const BinPass& pg, const SlabMap& sm, cudaStream_t s) {
    const int64_t nb = (ns + 255) / 256 + (ng + 255) / 256;
    if (nb == 0) return cudaSuccess;
    cudaError_t e = launch_pdl(k_fill, dim3((unsigned)nb), dim3(256), s, scull, ns, ps, gcull, ng, g_kind, pg, sm);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace ges
