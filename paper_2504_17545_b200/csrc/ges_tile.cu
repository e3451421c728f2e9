// K3 + K6 fused: one CTA (8 warps) per tile -- 16x16 base pixels with one
// pixel per thread, or 32x32 with a 2x2 pixel block per thread (PX = 2).
//
// Pass 1 (forward.py:127-209): every thread keeps, per (sub)sample, the hit
// depth and source id of the nearest covering surfel in registers, compared
// lexicographically: argmin over hit depth with ties to the lowest index,
// exactly np.argmin over the ascending candidate list (forward.py:187).
// No atomics: the z-buffer is private per pixel.
//
// Pass 2 (forward.py:248-381): order-independent, depth-gated accumulation of
// Gaussian alpha and alpha*colour in registers against the pass-1 depth that
// never leaves the register file, fused with the composite write
// (forward.py:384-417).
//
// Both passes are warp-independent: each warp owns an 8x4-thread patch of
// the tile and walks the tile's (tile, depth-slab)-binned list itself, 32
// entries at a time, near to far.  Every lane culls one entry against the
// warp's patch from its 16-byte cull record (pixel range; surfels: nearest
// disc depth vs the farthest current hit of the 2 x 2-lane regions of the
// patch its pixel range overlaps; Gaussians: depth - eps vs the patch's
// farthest surfel depth); survivors are transformed into the
// warp's shared slots and every lane then runs the exact per-pixel test for
// each; a warp stops at the first slab behind everything it has drawn.  There
// are no CTA barriers after the prologue.  Culling never changes results: the
// per-pixel tests are exact and order-independent.
#include <math.h>

#include "ges_launch.h"
#include "ges_sh.cuh"

namespace ges {


// Work counters for tuning (compiled in only with -DGES_STATS; read with
// ges_debug_stats).  0 surfel batches, 1 surfel entries staged, 2 staged with
// a live warp mask, 3 surfel warp tests, 4 candidate lanes, 5 Gaussian
// batches, 6 Gaussian entries staged, 7 staged with a live mask, 8 Gaussian
// warp tests, 9 contributing lanes, 10 tiles, 11 tiles with uncovered pixels.
__device__ unsigned long long g_stats[24];
#ifdef GES_STATS
#define GES_STAT(i, v) atomicAdd(&g_stats[i], (unsigned long long)(v))
#else
#define GES_STAT(i, v) ((void)0)
#endif

// Warps per CTA.  The 8 warps of a tile never synchronise after the
// prologue, so a tile can be split over 8 / WPC CTAs: a CTA's registers are
// held until its slowest warp finishes, and small CTAs hand them back warp by
// warp (the warps of one tile have very different amounts of work).
#ifndef GES_TILE_WPC
#define GES_TILE_WPC 1   // 32x32-pixel tiles and ss=4
#endif
#ifndef GES_TILE_WPC1
#define GES_TILE_WPC1 2  // 16x16-pixel tiles (40 registers: 24 two-warp CTAs per SM)
#endif

template <int WPC>
struct __align__(16) TileSmem {
    float4 st[4][32 * WPC];     // per-warp slots (32 each): pass-1 surfel coefficients, pass-2
                                // Gaussian records, then the colour tasks
    uint32_t wpk[4][32 * WPC];  // per lane: packed indices of its samples' winners, parked
                                // in shared memory through the Gaussian pass
    float4 rmax[WPC][2];        // per warp: max best depth of each of its 4 x 2 regions of
                                // 2 x 2 lanes (pass-1 culling)
    uint32_t slab_end[NSLAB];   // this tile's surfel slab ends (relative list positions)
    uint32_t gslab_end[NSLAB];  // this tile's Gaussian slab ends
};

// Lower depth bound of the slab holding relative list position `rel` (slab
// ends are non-decreasing, so the slab index is the number of ends <= rel:
// one vote per 32 slabs); every lane of the warp gets the same answer.
__device__ __forceinline__ float slab_floor(const uint32_t* ends, const SlabMap& m, uint32_t rel, int lane) {
    return m.lower(slab_of_pos(ends, rel, lane));
}
// Max of the per-region depth bounds of a warp (4 x 2 regions of 2 x 2 lanes,
// RW pixels square) over the regions that the pixel range [x0, x1] x [y0, y1]
// (relative to the patch origin, overlapping the patch) touches.
template <int RW>
__device__ __forceinline__ float region_max(const float4* rmax, int x0, int x1, int y0, int y1) {
    const int c0 = max(x0, 0) / RW, c1 = min(x1, 4 * RW - 1) / RW;
    const int q0 = max(y0, 0) / RW, q1 = min(y1, 2 * RW - 1) / RW;
    auto rowmax = [&](const float4& m) {
        float v = -INFINITY;
        v = (c0 <= 0) ? fmaxf(v, m.x) : v;
        v = (c0 <= 1 && c1 >= 1) ? fmaxf(v, m.y) : v;
        v = (c0 <= 2 && c1 >= 2) ? fmaxf(v, m.z) : v;
        v = (c1 >= 3) ? fmaxf(v, m.w) : v;
        return v;
    };
    float r = q0 == 0 ? rowmax(rmax[0]) : -INFINITY;
    if (q1 == 1) r = fmaxf(r, rowmax(rmax[1]));
    return r;
}
// Per-region maxima of v over 2 x 2 lanes (lane = x + 8 y in the warp's 8 x 4
// lane grid) into rm[4 x 2]; returns the max over the warp.
__device__ __forceinline__ float region_reduce(float m, float* rm, int lane) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
    if ((lane & 9) == 0) rm[((lane & 7) >> 1) + 4 * (lane >> 4)] = m;
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
    return fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Layer-selected final colour (forward.py:384-388, :412-417).
__device__ __forceinline__ float3 im_of(const TileArgs& a, float3 cs, float w, float cr, float cg, float cb) {
    if (a.layers == GES_LAYERS_GAUSSIANS_ONLY) {
        if (w > 0.f) {
            const float r = rcp_ftz(fmaxf(w, 1e-12f));   // (1 ulp)
            return make_float3(cr * r, cg * r, cb * r);
        }
        return make_float3(a.bg[0], a.bg[1], a.bg[2]);
    }
    const float r = rcp_ftz(1.0f + w);   // (1 + w >= 1: the approximate reciprocal is within 1 ulp)
    return make_float3((cs.x + cr) * r, (cs.y + cg) * r, (cs.z + cb) * r);
}

// Display/send-buffer form, datasets.py:54-56: clip(x*255+0.5, 0, 255) -> u8.
__device__ __forceinline__ void store_rgba8(uint8_t* dst, int64_t pix, float3 c) {
    auto q = [](float v) -> uint32_t { return (uint32_t)fminf(fmaxf(v * 255.0f + 0.5f, 0.f), 255.f); };
    reinterpret_cast<uint32_t*>(dst)[pix] = q(c.x) | (q(c.y) << 8) | (q(c.z) << 16) | (255u << 24);
}

// Row-pair stores of a thread's two horizontally adjacent pixels (PX = 2):
// one 8-byte store per pair of words when the destination address is 8-byte
// aligned (and both pixels are inside the image), plain stores otherwise --
// the C ABI only requires 4-byte alignment of the output buffers.
__device__ __forceinline__ void put1_pair(float* dst, int64_t pix, float v0, float v1, bool in1) {
    if (in1 && !(reinterpret_cast<uintptr_t>(dst + pix) & 7)) {
        *reinterpret_cast<float2*>(dst + pix) = make_float2(v0, v1);
    } else {
        dst[pix] = v0;
        if (in1) dst[pix + 1] = v1;
    }
}
__device__ __forceinline__ void put1_pair(int32_t* dst, int64_t pix, int32_t v0, int32_t v1, bool in1) {
    if (in1 && !(reinterpret_cast<uintptr_t>(dst + pix) & 7)) {
        *reinterpret_cast<int2*>(dst + pix) = make_int2(v0, v1);
    } else {
        dst[pix] = v0;
        if (in1) dst[pix + 1] = v1;
    }
}
__device__ __forceinline__ void put3_pair(float* dst, int64_t pix, float3 v0, float3 v1, bool in1) {
    float* d = dst + 3 * pix;
    if (in1 && !(reinterpret_cast<uintptr_t>(d) & 7)) {   // the 6 floats start 8-byte aligned
        float2* d2 = reinterpret_cast<float2*>(d);
        d2[0] = make_float2(v0.x, v0.y); d2[1] = make_float2(v0.z, v1.x); d2[2] = make_float2(v1.y, v1.z);
    } else {
        d[0] = v0.x; d[1] = v0.y; d[2] = v0.z;
        if (in1) { d[3] = v1.x; d[4] = v1.y; d[5] = v1.z; }
    }
}

// Camera-facing plane normal of source surfel `sid` (forward.py:148, :152),
// from the packed quaternion in float64 like the reference's frames.
__device__ __forceinline__ float3 surfel_nvis(const TileArgs& a, uint32_t sid) {
    const uint32_t pidx = (uint32_t)__ldg(a.s_pack + sid);
    const float4 qf = __ldg(a.s_quat + pidx), p = __ldg(a.s_pos + pidx);
    double w = qf.x, x = qf.y, y = qf.z, z = qf.w;
    const double inv = 1.0 / sqrt(w * w + x * x + y * y + z * z);
    w *= inv; x *= inv; y *= inv; z *= inv;
    const double c[3] = {2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)};
    double n[3], q[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        n[i] = a.R[3 * i] * c[0] + a.R[3 * i + 1] * c[1] + a.R[3 * i + 2] * c[2];
        q[i] = a.R[3 * i] * p.x + a.R[3 * i + 1] * p.y + a.R[3 * i + 2] * p.z + a.t[i];
    }
    const double sg = n[0] * q[0] + n[1] * q[1] + n[2] * q[2] < 0.0 ? 1.0 : -1.0;
    return make_float3((float)(n[0] * sg), (float)(n[1] * sg), (float)(n[2] * sg));
}

// View colour of packed surfel `pidx` (forward.py:99-103, sh.py:117-133):
// SH at the centre-to-camera direction.  Out of line and scalar-argument so
// the rarely executed, register-hungry evaluation does not raise the
// kernel's register count or copy the kernel parameters to the stack.
static __device__ __noinline__ float3 surfel_color_eval(const float* __restrict__ sh, const float4* __restrict__ pos,
                                                        int deg, float cx, float cy, float cz, uint32_t pidx) {
    const float4 p = __ldg(pos + pidx);
    const float dx = cx - p.x, dy = cy - p.y, dz = cz - p.z;   // |d| ~ scene distance: fp32 is ample
    const float inv = rsqrtf(fmaxf(dx * dx + dy * dy + dz * dz, 1e-24f));   // (2 ulp)
    const int K3 = (deg + 1) * (deg + 1) * 3;
    return sh_color_dyn(deg, sh + (size_t)pidx * K3, dx * inv, dy * inv, dz * inv);
}

// Deferred surfel colour (SURVEY 7 "SH only for winning surfels"): after pass
// 1 each lane knows the winners of its NS samples.  Distinct winners of the
// whole warp are compacted into a task list in the warp's shared-memory slice
// (a winner repeated in a lane's own samples or, per sample slot, in other
// lanes is evaluated once), the list is evaluated 32 tasks per SIMT pass, and
// every sample reads its colour back.  Must be called by all 32 lanes, with
// the warp's slice of sm.st free.
template <int NS, class Smem>
__device__ __forceinline__ void resolve_surfel_colors(const TileArgs& a, Smem& sm, uint32_t covm,
                                                      const uint32_t* bp, int lane, int warp, float3* col) {
    const float3 bg = make_float3(a.bg[0], a.bg[1], a.bg[2]);
    if constexpr (NS == 1) {
        const bool cov = covm & 1u;
        const unsigned peers = __match_any_sync(0xffffffffu, cov ? bp[0] : 0xffffffffu);
        const int leader = __ffs(peers) - 1;
        float3 c = bg;
        if (cov && lane == leader)
            c = surfel_color_eval(a.s_sh, a.s_pos, a.sh_deg, (float)a.cpos[0], (float)a.cpos[1], (float)a.cpos[2],
                                  bp[0]);
        c.x = __shfl_sync(0xffffffffu, c.x, leader);
        c.y = __shfl_sync(0xffffffffu, c.y, leader);
        c.z = __shfl_sync(0xffffffffu, c.z, leader);
        col[0] = cov ? c : bg;
    } else {
        static_assert(NS <= 4, "task slice holds 128 winners per warp");
        int dup[NS], leader[NS];
        uint32_t need = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const bool cov = (covm >> s) & 1u;
            const uint32_t v = cov ? bp[s] : 0xffffffffu;
            dup[s] = -1;
#pragma unroll
            for (int q = s - 1; q >= 0; --q)
                if (cov && bp[q] == v && ((covm >> q) & 1u)) dup[s] = q;
            leader[s] = __ffs(__match_any_sync(0xffffffffu, v)) - 1;
            if (cov && dup[s] < 0 && lane == leader[s]) need |= 1u << s;
        }
        // exclusive prefix of the per-lane task counts
        const int cnt = __popc(need);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        uint32_t* tp = reinterpret_cast<uint32_t*>(&sm.st[0][warp * 32]);   // 128 task slots
        float* tr = reinterpret_cast<float*>(&sm.st[1][warp * 32]);
        float* tg = reinterpret_cast<float*>(&sm.st[2][warp * 32]);
        float* tb = reinterpret_cast<float*>(&sm.st[3][warp * 32]);
        int task[NS];
        int k = incl - cnt;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            int own = -1;
            if ((need >> s) & 1u) { own = k++; tp[own] = bp[s]; }
            else if (dup[s] >= 0) own = task[dup[s]];
            const int lead = __shfl_sync(0xffffffffu, own, leader[s]);
            task[s] = !((covm >> s) & 1u) ? -1 : (dup[s] >= 0 || ((need >> s) & 1u)) ? own : lead;
        }
        __syncwarp();
        for (int i = lane; i < total; i += 32) {
            const float3 c = surfel_color_eval(a.s_sh, a.s_pos, a.sh_deg, (float)a.cpos[0], (float)a.cpos[1],
                                               (float)a.cpos[2], tp[i]);
            tr[i] = c.x; tg[i] = c.y; tb[i] = c.z;
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < NS; ++s) col[s] = task[s] >= 0 ? make_float3(tr[task[s]], tg[task[s]], tb[task[s]]) : bg;
    }
}

#ifndef GES_TILE_MINB2
#define GES_TILE_MINB2 4   // resident CTAs per SM for the 4-sample variants (64 registers)
#endif

// SS: supersampling of the surfel pass (1, or 2 = the 2x2 grid of ss=4);
// PX: base pixels per thread per axis (1: 16x16-pixel tiles; 2: 32x32-pixel
// tiles, each thread a 2x2 pixel block, so every staged surfel and every
// list step is shared by 4 pixels).  A thread owns G x G = (SS*PX)^2 samples
// in pass 1 and PX x PX pixels in pass 2.
template <int SS, int PX>
__host__ __device__ constexpr int tile_wpc() { return (PX == 2 || SS == 2) ? GES_TILE_WPC : GES_TILE_WPC1; }
#ifndef GES_TILE_MINW2
#define GES_TILE_MINW2 (GES_TILE_MINB2 * 8)   // resident warps per SM, 4-sample variants (64 registers)
#endif
template <int SS, int PX>
__host__ __device__ constexpr int tile_min_blocks() {   // resident CTAs per SM (at most 32)
    return ((PX == 2 || SS == 2) ? GES_TILE_MINW2 : 48) / tile_wpc<SS, PX>() > 32
               ? 32 : ((PX == 2 || SS == 2) ? GES_TILE_MINW2 : 48) / tile_wpc<SS, PX>();
}

template <int SS, int PX, int MODE, int GK, bool GEOM>
__global__ void __launch_bounds__(32 * tile_wpc<SS, PX>(), tile_min_blocks<SS, PX>()) k_tile(TileArgs a) {
    constexpr int G = SS * PX, NS = G * G, NP = PX * PX, TP = TILE * PX;
    constexpr int WPC = tile_wpc<SS, PX>(), TPB = 32 * WPC;
    __shared__ TileSmem<WPC> sm;
    pdl_wait();   // (launched as a dependent of the fill: lists, offsets, status)
    if (a.status->overflow) return;   // pair lists incomplete: host re-renders
#ifdef GES_TIMING   // warp lifetimes (tuning builds only, see read_stats / tools/tile_stats.py --timing)
    const long long t_start = clock64();
    unsigned tm_len = 0, tm_b1 = 0, tm_t1 = 0, tm_b2 = 0, tm_t2 = 0;
    long long t_p1 = 0, t_p2 = 0;
#define GES_TM(x) (x)
#else
#define GES_TM(x) ((void)0)
#endif
    // warp: the warp's patch within the tile (0..7); wl: its index within the CTA
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    // CTAs in launch order; with a.order the heaviest tiles come first
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    const int warp = (cta % (NWARP / WPC)) * WPC + wl;
    const int tile = a.order ? (int)__ldg(a.order + cta / (NWARP / WPC)) : cta / (NWARP / WPC);
    // tile / ntx without the integer division: (tile + 0.5) / ntx is >= 0.5 / ntx
    // away from an integer, beyond the float quotient's error (2 ulp of <= nty)
    // while ntx * nty < 2^21 tiles
    const int ty = a.ntx * a.nty < (1 << 21) ? (int)__fdividef((float)tile + 0.5f, (float)a.ntx) : tile / a.ntx;
    const int tx = tile - ty * a.ntx;
    const int plx = (warp & 1) * 8 + (lane & 7), ply = (warp >> 1) * 4 + (lane >> 3);
    const int bx = tx * TP + PX * plx, by = ty * TP + PX * ply;   // first base pixel of the thread

    float ds[NP];                    // surfel depth per pixel (sub-sample 0 of the pixel)
#pragma unroll
    for (int p = 0; p < NP; ++p) ds[p] = INFINITY;
    auto inside_px = [&](int p) { return bx + p % PX < a.W && by + p / PX < a.H; };
    auto pix_of = [&](int p) { return (int64_t)(by + p / PX) * a.W + (bx + p % PX); };

    // Issue every list-position load of both passes now: tile offsets, slab
    // ends and the first batch of Gaussian ids are independent of pass 1, so
    // their latency (and, below, the first Gaussian records via an L2
    // prefetch) overlaps the surfel pass.
    uint32_t gbeg = 0, gend = 0, gid = 0;
    if constexpr ((MODE & 2) != 0) {
        for (int k = threadIdx.x; k < NSLAB; k += TPB) sm.gslab_end[k] = a.gbin.cnt[tile * NSLAB + k];
        gbeg = a.gbin.tile_off(tile);
        gend = gbeg + a.gbin.cnt[tile * NSLAB + NSLAB - 1];
        if (gbeg + warp * 32 + lane < gend) gid = a.g_list[gbeg + warp * 32 + lane];
    }

    // bid[s]: source id of the nearest surfel hit so far (~0u: none); with
    // bt[s] (its hit depth) the pair (bt, bid) is compared lexicographically,
    // == np.argmin with lowest-index ties (forward.py:187); bp[s]: the
    // winner's packed index (SH address of the deferred colour), looked up
    // once after pass 1
    uint32_t bid[NS];
    uint32_t bp[NS];
    uint32_t covm = 0;   // bit s: sample s covered (bt[], bid[] are dead after pass 1)

    // ------------------------------------------------------------ pass 1
    if constexpr (MODE & 1) {
        // bt[s]: the best hit depth (candidate filter with a 1e-5 margin and
        // culling bound; samples outside the image start at 0 so they never
        // take work or block culling)
        // pe: the near-parallel threshold 1e-8|d|, one per thread (the max over
        // its samples: the 2x2 block's |d| differ by < 1e-3 relative, inside the
        // flagged grazing band of the parity rule)
        float bt[NS], pe = 0.f;
        const float lx0 = (float)(G * plx), ly0 = (float)(G * ply);
#pragma unroll
        for (int gy = 0; gy < G; ++gy)
#pragma unroll
            for (int gx = 0; gx < G; ++gx) {
                const int X = bx * SS + gx, Y = by * SS + gy;
                const float dxn = ((float)X + 0.5f - a.rcx) * a.rifx, dyn = ((float)Y + 0.5f - a.rcy) * a.rify;
                pe = fmaxf(pe, fmaf(dxn, dxn, dyn * dyn));
                bid[gy * G + gx] = ~0u;
                const bool in = bx + gx / SS < a.W && by + gy / SS < a.H;
                bt[gy * G + gx] = in ? INFINITY : 0.f;
            }
        pe = PARALLEL_EPS_F * sqrt_ftz(pe + 1.0f);   // max over the samples of 1e-8 |d|
        // Depth culling bounds, refreshed after every chunk: the max over each
        // region of 2 x 2 lanes (one entry of sm.rmax) and over the whole
        // patch (wmx).  A single uncovered sample keeps its bound at +inf, so
        // per-region bounds let covered parts of the patch cull entries long
        // before the whole patch is covered.
        float* const rm = reinterpret_cast<float*>(sm.rmax[wl]);
        auto patch_depth = [&]() {
            float m = bt[0];
#pragma unroll
            for (int s = 1; s < NS; ++s) m = fmaxf(m, bt[s]);
            m *= 1.00001f;   // margin-inflated: culling stays conservative
            return region_reduce(m, rm, lane);
        };
        // max over this warp's samples of the best depth, and per region: +inf
        // for samples in the image, 0 outside, so a patch that lies entirely
        // below the image's last row (the partial bottom tile row) stops at
        // its first slab instead of walking the whole list
        float wmx = patch_depth();
        for (int k = threadIdx.x; k < NSLAB; k += TPB) sm.slab_end[k] = a.sbin.cnt[tile * NSLAB + k];
        __syncthreads();
        const int ox = tx * TP * SS, oy = ty * TP * SS;
        const uint32_t beg = a.sbin.tile_off(tile), end = beg + sm.slab_end[NSLAB - 1];
        GES_TM(tm_len = end - beg);
        uint32_t nid = beg + lane < end ? a.s_list[beg + lane] : 0u;
        if constexpr ((MODE & 2) != 0) {
            if (gbeg + warp * 32 + lane < gend) {
                const char* gp = static_cast<const char*>(a.grec) + (size_t)gid * (GK == 2 ? sizeof(Gauss2Rec) : sizeof(GaussRec));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(gp));
            }
        }
        // Warp-independent, like pass 2: each warp walks the tile's near-to-far
        // surfel list 32 entries at a time, culls every entry against ITS patch
        // from the 16-byte cull record (pixel range; nearest disc depth vs the
        // warp's current max hit depth), transforms the survivors into its own
        // shared slots and tests them, and stops at the first slab behind all
        // of its hits.  No CTA barriers: a warp never waits for the others.
        constexpr int PW = 8 * G, PH = 4 * G;   // patch size in surfel-pass pixels
        const int wx0 = ox + (warp & 1) * PW, wy0 = oy + (warp >> 1) * PH;
        for (uint32_t base = beg; base < end; base += 32) {
            // slabs are near-to-far: stop once the next slab lies behind every hit so far
            if (slab_floor(sm.slab_end, a.slabs, base - beg, lane) > wmx) break;
            const uint32_t e = base + lane;
            const uint32_t id = nid;   // this chunk's ids were loaded one chunk ahead
            if (e + 32 < end) nid = a.s_list[e + 32];
            bool live = false;
            if (e < end) {
                const float4 r3 = __ldg(a.scull + id);
                const uint32_t sxr = __float_as_uint(r3.y), syr = __float_as_uint(r3.z);
                live = span_lo(sxr) < wx0 + PW && span_hi(sxr) >= wx0 && span_lo(syr) < wy0 + PH &&
                       span_hi(syr) >= wy0 && !(r3.x > wmx);
#ifdef GES_STATS
                if (span_lo(sxr) < wx0 + PW && span_hi(sxr) >= wx0 && span_lo(syr) < wy0 + PH && span_hi(syr) >= wy0)
                    GES_STAT(17, 1);
#endif
                // nearest disc depth vs the regions its pixel range overlaps
                if (live) live = !(r3.x > region_max<2 * G>(sm.rmax[wl], span_lo(sxr) - wx0, span_hi(sxr) - wx0,
                                                            span_lo(syr) - wy0, span_hi(syr) - wy0));
                if (live) {
                    const SurfRec* r = a.srec + id;
                    const float4 r0 = __ldg(&r->r0), r1 = __ldg(&r->r1), r2 = __ldg(&r->r2);
                    const float fx = (float)(ox - (int)r1.w), fy = (float)(oy - (int)r2.w);
                    float d0 = fmaf(r0.z, fy, fmaf(r0.y, fx, r0.x));
                    const float u0 = fmaf(r1.z, fy, fmaf(r1.y, fx, r1.x));
                    const float v0 = fmaf(r2.z, fy, fmaf(r2.y, fx, r2.x));
                    // hit depth t = nq / den: orient den so that t > 0 <=> den > 0
                    float nq = r0.w, dx_ = r0.y, dy_ = r0.z;
                    if (nq < 0.f) { nq = -nq; d0 = -d0; dx_ = -dx_; dy_ = -dy_; }
                    live = nq > 0.f;
                    // U, V pre-divided by R: coverage becomes U'^2 + V'^2 <= den^2
                    constexpr float IR = 1.0f / 3.3290429691304455f;
                    const int slot = wl * 32 + lane;
                    sm.st[0][slot] = make_float4(d0, dx_, dy_, nq);
                    sm.st[1][slot] = make_float4(u0 * IR, r1.y * IR, r1.z * IR, v0 * IR);
                    sm.st[2][slot] = make_float4(r2.y * IR, r2.z * IR, r3.w, r3.x);   // r3.w: source id
#ifdef GES_STATS
                    sm.st[3][slot] = make_float4(r3.y, r3.z, 0.f, 0.f);   // spans (work counters only)
#endif
                }
            }
            uint32_t vote = __ballot_sync(0xffffffffu, live);
            GES_TM(++tm_b1);
#ifdef GES_STATS
            if (lane == 0) { GES_STAT(0, 1); GES_STAT(1, min(32u, end - base)); GES_STAT(2, __popc(vote)); }
#endif
            if (!vote) continue;     // nothing tested: the patch depth is unchanged
            __syncwarp();
            while (vote) {
                const int j = wl * 32 + __ffs(vote) - 1;
                vote &= vote - 1;
                // (no depth re-check here: wmx only changes between chunks, and the
                // staging already required the disc's nearest depth <= wmx)
                const float4 C = sm.st[2][j];
                if (lane == 0) GES_STAT(3, 1);
                if (lane == 0) GES_STAT(12, wmx == INFINITY);
#ifdef GES_STATS
                if (lane == 0) {   // survivor's pixel range within one x half / y half / quadrant of the patch
                    const float4 S = sm.st[3][j];
                    const uint32_t sxr = __float_as_uint(S.x), syr = __float_as_uint(S.y);
                    const int ax0 = max(span_lo(sxr) - wx0, 0), ax1 = min(span_hi(sxr) - wx0, PW - 1);
                    const int ay0 = max(span_lo(syr) - wy0, 0), ay1 = min(span_hi(syr) - wy0, PH - 1);
                    const bool xh = (ax0 / (PW / 2)) == (ax1 / (PW / 2)), yh = (ay0 / (PH / 2)) == (ay1 / (PH / 2));
                    GES_STAT(20, xh); GES_STAT(21, yh); GES_STAT(22, xh && yh);
                }
#endif
                GES_TM(++tm_t1);
                const float4 A = sm.st[0][j], B = sm.st[1][j];
                const float Awf = A.w * 0.99999f;   // candidate filter t <= 1.00001 bt (margin vs rounding)
#ifdef GES_STATS
                bool st_any = false;
#endif
                // den, U, V at the thread's first sample, then stepped by the
                // per-sample increments across its G x G block
                const float den0 = fmaf(A.z, ly0, fmaf(A.y, lx0, A.x));
                const float U0 = fmaf(B.z, ly0, fmaf(B.y, lx0, B.x));
                const float V0 = fmaf(C.y, ly0, fmaf(C.x, lx0, B.w));
                float dens[NS];
                bool cand[NS], anyc = false;
#pragma unroll
                for (int gy = 0; gy < G; ++gy)
#pragma unroll
                    for (int gx = 0; gx < G; ++gx) {
                        const int s = gy * G + gx;
                        float den = den0, U = U0, V = V0;
                        if (gx) { den = fmaf(A.y, (float)gx, den); U = fmaf(B.y, (float)gx, U); V = fmaf(C.x, (float)gx, V); }
                        if (gy) { den = fmaf(A.z, (float)gy, den); U = fmaf(B.z, (float)gy, U); V = fmaf(C.y, (float)gy, V); }
                        const float r2 = fmaf(U, U, V * V);
#ifdef GES_STATS
                        {
                            const bool inside = bx + gx / SS < a.W && by + gy / SS < a.H;
                            const bool cov = den > pe && r2 <= den * den;
                            if (inside) GES_STAT(cov ? 14 : 13, 1);
                            if (inside && cov && bid[s] == ~0u) GES_STAT(15, 1);
                            st_any = st_any || (inside && cov);
                        }
#endif
                        // coverage u^2+v^2 <= R^2 and t no later than the current best (all
                        // multiplied out, den > 0 <=> t > 0: with den <= 0 the product
                        // bt*den is <= 0 or NaN and the filter fails); |n.d| > eps|d|, the
                        // exact t > 0.01 and the packed-key comparison run only for candidates
                        dens[s] = den;
                        cand[s] = r2 <= den * den && Awf <= bt[s] * den;
                        anyc = anyc || cand[s];
                    }
                // one branch for the thread's candidates (not one per sample): the
                // re-check is predicated per sample
                if (anyc) {
                    const uint32_t sid = __float_as_uint(C.z);
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        const float t = A.w * rcp_ftz(dens[s]);   // 2 ulp: ties are flagged
                        // (t, sid) < (bt, bid) lexicographically as one 64-bit compare of
                        // (float bits, id): t > 0 and bt >= 0, so the bits order like the values
                        const unsigned long long kt = ((unsigned long long)__float_as_uint(t) << 32) | sid;
                        const unsigned long long kb = ((unsigned long long)__float_as_uint(bt[s]) << 32) | bid[s];
                        const bool take = cand[s] && dens[s] > pe && t > NEAR_F && kt < kb;
                        GES_STAT(4, cand[s]);
                        bt[s] = take ? t : bt[s];
                        bid[s] = take ? sid : bid[s];
                    }
                }
#ifdef GES_STATS
                if (__ballot_sync(0xffffffffu, st_any) == 0u && lane == 0) GES_STAT(16, 1);
#endif
            }
            wmx = patch_depth();
            __syncwarp();   // the slots are rewritten by the next chunk
        }
        // the winners' SH blocks are read at the end (deferred colour): find
        // their packed indices and start pulling them into L2 now, overlapping
        // the Gaussian pass
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            bp[s] = bid[s] != ~0u ? __ldg(a.s_pack + bid[s]) : 0u;
            covm |= (bid[s] != ~0u ? 1u : 0u) << s;
        }
        asm volatile("" : "+r"(covm));   // materialise now so bid[] dies before pass 2
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (bid[s] != ~0u) {
                const char* p = reinterpret_cast<const char*>(a.s_sh) + (size_t)bp[s] * a.sh_bytes;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
                if (a.sh_bytes > 64) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + a.sh_bytes - 4));
            }
            sm.wpk[s][threadIdx.x] = bp[s];   // (reloaded for the deferred colour: no registers in pass 2)
        }
        // depth/normal/winner of each pixel from its sub-sample 0 (forward.py:205-207)
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int s0 = (p / PX) * SS * G + (p % PX) * SS;
            const bool cov = bid[s0] != ~0u;
            ds[p] = cov ? bt[s0] : INFINITY;
            asm volatile("" : "+f"(ds[p]));   // (not rematerialised from bt[] in pass 2)
            if (inside_px(p)) {
                const int64_t pix = pix_of(p);
                if constexpr (PX == 2) {   // depth and winner of the row pair in one store each
                    if (p % 2 == 0) {
                        const int s1 = s0 + SS;
                        const bool in1 = inside_px(p + 1), cov1 = bid[s1] != ~0u;
                        const float d1 = cov1 ? bt[s1] : INFINITY;
                        if (a.out.s_depth) put1_pair(a.out.s_depth, pix, ds[p], d1, in1);
                        if (a.out.s_winner)
                            put1_pair(a.out.s_winner, pix, cov ? (int32_t)bid[s0] : -1,
                                      cov1 ? (int32_t)bid[s1] : -1, in1);
                    }
                } else {
                    if (a.out.s_depth) a.out.s_depth[pix] = ds[p];
                    if (a.out.s_winner) a.out.s_winner[pix] = cov ? (int32_t)bid[s0] : -1;
                }
                if (a.out.s_normal) {
                    const float3 n = cov ? surfel_nvis(a, bid[s0]) : make_float3(0.f, 0.f, 0.f);
                    a.out.s_normal[3 * pix] = n.x; a.out.s_normal[3 * pix + 1] = n.y;
                    a.out.s_normal[3 * pix + 2] = n.z;
                }
            }
        }
    } else {
#pragma unroll
        for (int p = 0; p < NP; ++p)
            if (inside_px(p) && a.ds_in) ds[p] = a.ds_in[pix_of(p)];
    }

    GES_TM(t_p1 = clock64());
    // ------------------------------------------------------------ pass 2
    float wsum[NP], cr[NP], cg[NP], cb[NP], dsum[NP], nx[NP], ny[NP], nz[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        wsum[p] = cr[p] = cg[p] = cb[p] = 0.f;
        dsum[p] = nx[p] = ny[p] = nz[p] = 0.f;
    }
    if constexpr (MODE & 2) {
        // Warp-independent: each warp walks the tile's Gaussian list itself, 32
        // entries at a time, culls against ITS patch (pixel range and the
        // warp's own max surfel depth) from the 16-byte cull record, and
        // evaluates the few survivors lane by lane (the survivor's lane loads
        // its record once and broadcasts it).  No shared staging, no CTA
        // barriers: the pass is latency-bound and warps must not wait on each
        // other.
        if constexpr ((MODE & 1) == 0) __syncthreads();   // gslab_end written in the prologue
        float dm = -INFINITY;
#pragma unroll
        for (int p = 0; p < NP; ++p) dm = fmaxf(dm, inside_px(p) ? ds[p] : -INFINITY);
        const float wdmax = warp_max(dm);
        if (warp == 0 && lane == 0) GES_STAT(10, 1);
        if (lane == 0) GES_STAT(11, wdmax == INFINITY);
        float pe[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            pe[p] = 0.f;
            if constexpr (GK == 2) {
                const float dxn = ((float)(bx + p % PX) + 0.5f - a.gcx) * a.gifx;
                const float dyn = ((float)(by + p / PX) + 0.5f - a.gcy) * a.gify;
                pe[p] = PARALLEL_EPS_F * sqrt_ftz(dxn * dxn + dyn * dyn + 1.0f);
            }
        }
        const int ox = tx * TP, oy = ty * TP;
        const int px0 = (warp & 1) * 8 * PX, py0 = (warp >> 1) * 4 * PX;   // this warp's patch
        float lxs[PX], lys[PX];   // this thread's pixel coordinates in the tile
#pragma unroll
        for (int i = 0; i < PX; ++i) {
            lxs[i] = (float)(PX * plx + i); lys[i] = (float)(PX * ply + i);
            asm volatile("" : "+f"(lxs[i]), "+f"(lys[i]));
        }
        for (uint32_t base = gbeg; base < gend; base += 32) {
            // keys (depth - eps) are binned near-to-far: the rest fail every gate of the patch
            if (slab_floor(sm.gslab_end, a.slabs, base - gbeg, lane) > wdmax) break;
            const uint32_t e = base + lane;
            bool live = false;
            float v[16];
            if (e < gend) {
                const uint32_t id = a.g_list[e];
                if constexpr (GK == 3) {
                    const GaussRec* r = reinterpret_cast<const GaussRec*>(a.grec) + id;
                    const float4 c = __ldg(a.gcull + id);
                    const uint32_t sxr = __float_as_uint(c.z), syr = __float_as_uint(c.w);
                    // exact conservative cull: d < fl(max_ds + eps) is necessary for the gate
                    live = span_lo(sxr) - ox <= px0 + 8 * PX - 1 && span_hi(sxr) - ox >= px0 &&
                           span_lo(syr) - oy <= py0 + 4 * PX - 1 && span_hi(syr) - oy >= py0 &&
                           c.x < wdmax + c.y;
#ifdef GES_STATS
                    if (span_lo(sxr) - ox <= px0 + 8 * PX - 1 && span_hi(sxr) - ox >= px0 &&
                        span_lo(syr) - oy <= py0 + 4 * PX - 1 && span_hi(syr) - oy >= py0)
                        GES_STAT(18, 1);
#endif
                    if (live) {
                        const float4 r0 = __ldg(&r->r0), r1 = __ldg(&r->r1), r2 = __ldg(&r->r2);
                        v[0] = (r0.x - (float)ox) + (r0.y - 0.5f);   // mean relative to the tile
                        v[1] = (r0.z - (float)oy) + (r0.w - 0.5f);
                        v[2] = r1.x; v[3] = r1.y; v[4] = r1.z; v[5] = r1.w;
                        v[6] = c.x; v[7] = c.y; v[8] = r2.x; v[9] = r2.y; v[10] = r2.z; v[11] = r2.w;
                        if constexpr (GEOM) {
                            const float4 nv = __ldg(a.g_nrm + id);
                            v[12] = nv.x; v[13] = nv.y; v[14] = nv.z;
                        }
                    }
                } else {
                    const Gauss2Rec* r = reinterpret_cast<const Gauss2Rec*>(a.grec) + id;
                    const float4 c = __ldg(a.gcull + id);
                    const uint32_t sxr = __float_as_uint(c.z), syr = __float_as_uint(c.w);
                    live = span_lo(sxr) - ox <= px0 + 8 * PX - 1 && span_hi(sxr) - ox >= px0 &&
                           span_lo(syr) - oy <= py0 + 4 * PX - 1 && span_hi(syr) - oy >= py0 && !(c.x > wdmax);
                    if (live) {
                        const float4 r0 = __ldg(&r->r0), r1 = __ldg(&r->r1), r2 = __ldg(&r->r2),
                                     r3 = __ldg(&r->r3), r4 = __ldg(&r->r4);
                        const float fx = (float)(ox - (int)r1.w), fy = (float)(oy - (int)r2.w);
                        v[0] = fmaf(r0.z, fy, fmaf(r0.y, fx, r0.x)); v[1] = r0.y; v[2] = r0.z; v[3] = r0.w;
                        v[4] = fmaf(r1.z, fy, fmaf(r1.y, fx, r1.x)); v[5] = r1.y; v[6] = r1.z;
                        v[7] = fmaf(r2.z, fy, fmaf(r2.y, fx, r2.x)); v[8] = r2.y; v[9] = r2.z;
                        v[10] = r3.x; v[11] = c.y; v[12] = r3.y;          // sigma, eps, r2max
                        v[13] = r4.x; v[14] = r4.y; v[15] = r4.z;         // colour
                    }
                }
            }
            // survivors park their record in this warp's slice of shared memory;
            // every lane then reads each survivor with broadcast loads
            const int slot = wl * 32 + lane;
            if (live) {
                sm.st[0][slot] = make_float4(v[0], v[1], v[2], v[3]);
                sm.st[1][slot] = make_float4(v[4], v[5], v[6], v[7]);
                sm.st[2][slot] = make_float4(v[8], v[9], v[10], v[11]);
                sm.st[3][slot] = make_float4(v[12], v[13], v[14], v[15]);
            }
            uint32_t vote = __ballot_sync(0xffffffffu, live);
            GES_TM(++tm_b2);
            GES_TM(tm_t2 += __popc(vote));
            if (lane == 0) { GES_STAT(6, min(32u, gend - base)); GES_STAT(7, __popc(vote)); GES_STAT(19, 1); }
            __syncwarp();
            while (vote) {
                const int j = __ffs(vote) - 1;
                vote &= vote - 1;
                if (lane == 0) GES_STAT(8, 1);
                float w[16];
                {
                    const float4 q0 = sm.st[0][wl * 32 + j], q1 = sm.st[1][wl * 32 + j],
                                 q2 = sm.st[2][wl * 32 + j];
                    w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
                    w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
                    w[8] = q2.x; w[9] = q2.y; w[10] = q2.z; w[11] = q2.w;
                    if constexpr (GK == 2 || GEOM) {
                        const float4 q3 = sm.st[3][wl * 32 + j];
                        w[12] = q3.x; w[13] = q3.y; w[14] = q3.z; w[15] = q3.w;
                    }
                }
                // power a dx^2 + b dx dy + c dy^2 of the thread's 2 x 2 pixel block:
                // pixel (0,0) directly, its neighbours by the exact finite differences
                // (a (2dx + 1) + b dy, c (2dy + 1) + b dx; the diagonal adds b)
                float pwv[NP];
                if constexpr (GK == 3 && PX == 2) {
                    const float dx = lxs[0] - w[0], dy = lys[0] - w[1];
                    const float bdx = w[3] * dx;
                    const float p00 = fmaf(w[2] * dx, dx, fmaf(w[4] * dy, dy, bdx * dy));
                    const float gx = fmaf(w[2], fmaf(2.f, dx, 1.f), w[3] * dy);
                    const float gy = fmaf(w[4], fmaf(2.f, dy, 1.f), bdx);
                    pwv[0] = p00; pwv[1] = p00 + gx; pwv[2] = p00 + gy; pwv[3] = (p00 + gx) + (gy + w[3]);
                }
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const float lx = lxs[p % PX], ly = lys[p / PX];
                    if constexpr (GK == 3) {
                        // forward.py:301-311; the conic is pre-scaled by log2(e), so
                        // exp is one ex2 (branch-free: most survivors' pixels pass)
                        float pw;
                        if constexpr (PX == 2) {
                            pw = pwv[p];
                        } else {
                            const float dx = lx - w[0], dy = ly - w[1];
                            pw = fmaf(w[2] * dx, dx, fmaf(w[4] * dy, dy, w[3] * dx * dy));
                        }
                        {
                            const float al = w[5] * ex2_ftz(pw);
                            if (al >= ALPHA_CUTOFF_F && w[6] < ds[p] + w[7]) {
                                GES_STAT(9, 1);
                                wsum[p] += al;
                                cr[p] = fmaf(al, w[9], cr[p]); cg[p] = fmaf(al, w[10], cg[p]);
                                cb[p] = fmaf(al, w[11], cb[p]);
                                if constexpr (GEOM) {
                                    dsum[p] = fmaf(al, w[6], dsum[p]);
                                    nx[p] = fmaf(al, w[12], nx[p]); ny[p] = fmaf(al, w[13], ny[p]);
                                    nz[p] = fmaf(al, w[14], nz[p]);
                                }
                            }
                        }
                    } else {
                        // forward.py:361-379
                        const float den = fmaf(w[2], ly, fmaf(w[1], lx, w[0]));
                        const float U = fmaf(w[6], ly, fmaf(w[5], lx, w[4]));
                        const float V = fmaf(w[9], ly, fmaf(w[8], lx, w[7]));
                        const float r2u = fmaf(U, U, V * V);
                        if (r2u <= w[12] * den * den && fabsf(den) > pe[p]) {
                            const float inv = rcp_ftz(den);   // |den| > 1e-8|d|
                            const float t = w[3] * inv;
                            const float q2 = r2u * inv * inv;
                            const float al = w[10] * ex2_ftz(q2 * (-0.5f * LOG2E_F));
                            if (t > NEAR_F && al >= ALPHA_CUTOFF_F && t < ds[p] + w[11]) {
                                wsum[p] += al;
                                cr[p] = fmaf(al, w[13], cr[p]); cg[p] = fmaf(al, w[14], cg[p]);
                                cb[p] = fmaf(al, w[15], cb[p]);
                                if constexpr (GEOM) {
                                    // planar normal: camera-facing plane normal (forward.py:337, :379)
                                    const float4 nv = __ldg(a.g_nrm + a.g_list[base + j]);
                                    dsum[p] = fmaf(al, t, dsum[p]);
                                    nx[p] = fmaf(al, nv.x, nx[p]); ny[p] = fmaf(al, nv.y, ny[p]);
                                    nz[p] = fmaf(al, nv.z, nz[p]);
                                }
                            }
                        }
                    }
                }
            }
            __syncwarp();   // the slots are rewritten by the next step
        }
    }

    GES_TM(t_p2 = clock64());
    // ------------------------------------------------------------ resolve + write
    float3 cs[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) cs[p] = make_float3(a.bg[0], a.bg[1], a.bg[2]);
    if constexpr ((MODE & 1) != 0) {
        float3 col[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) bp[s] = reinterpret_cast<volatile uint32_t*>(sm.wpk[s])[threadIdx.x];
        resolve_surfel_colors<NS>(a, sm, covm, bp, lane, wl, col);
        if constexpr (PX == 1) {   // box mean over the sub-samples (forward.py:201-203)
            float3 acc = make_float3(0.f, 0.f, 0.f);
#pragma unroll
            for (int s = 0; s < NS; ++s) { acc.x += col[s].x; acc.y += col[s].y; acc.z += col[s].z; }
            if (NS > 1) { acc.x /= (float)NS; acc.y /= (float)NS; acc.z /= (float)NS; }
            cs[0] = acc;
        } else {
#pragma unroll
            for (int p = 0; p < NP; ++p) cs[p] = col[p];   // SS == 1: one sample per pixel
        }
    }
    if constexpr (PX == 2 && !GEOM) {
        // row pairs: 8-byte stores (image, colours, weight)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int p0 = 2 * r, p1 = 2 * r + 1;
            if (!inside_px(p0)) continue;
            const bool in1 = inside_px(p1);
            const int64_t pix = pix_of(p0);
            if constexpr ((MODE & 1) != 0)
                if (a.out.s_color) put3_pair(a.out.s_color, pix, cs[p0], cs[p1], in1);
            float3 i0 = cs[p0], i1 = cs[p1];
            if constexpr ((MODE & 2) != 0) {
                if (a.out.g_weight) put1_pair(a.out.g_weight, pix, wsum[p0], wsum[p1], in1);
                if (a.out.g_color)
                    put3_pair(a.out.g_color, pix, make_float3(cr[p0], cg[p0], cb[p0]),
                              make_float3(cr[p1], cg[p1], cb[p1]), in1);
                i0 = im_of(a, cs[p0], wsum[p0], cr[p0], cg[p0], cb[p0]);
                i1 = im_of(a, cs[p1], wsum[p1], cr[p1], cg[p1], cb[p1]);
            } else {   // surfels_only (forward.py:407-410): empty Gaussian buffers
                if (a.out.g_weight) put1_pair(a.out.g_weight, pix, 0.f, 0.f, in1);
                if (a.out.g_color)
                    put3_pair(a.out.g_color, pix, make_float3(0.f, 0.f, 0.f), make_float3(0.f, 0.f, 0.f), in1);
            }
            if (a.out.image) put3_pair(a.out.image, pix, i0, i1, in1);
            if (a.out.image_rgba8) {
                store_rgba8(a.out.image_rgba8, pix, i0);
                if (in1) store_rgba8(a.out.image_rgba8, pix + 1, i1);
            }
        }
    } else {
    #pragma unroll
        for (int p = 0; p < NP; ++p) {
            if (!inside_px(p)) continue;
            const int64_t pix = pix_of(p);
            if constexpr ((MODE & 1) != 0) {
                if (a.out.s_color) {
                    a.out.s_color[3 * pix] = cs[p].x; a.out.s_color[3 * pix + 1] = cs[p].y;
                    a.out.s_color[3 * pix + 2] = cs[p].z;
                }
            }
            if constexpr ((MODE & 2) != 0) {
                if (a.out.g_weight) a.out.g_weight[pix] = wsum[p];
                if (a.out.g_color) {
                    a.out.g_color[3 * pix] = cr[p]; a.out.g_color[3 * pix + 1] = cg[p];
                    a.out.g_color[3 * pix + 2] = cb[p];
                }
                if constexpr (GEOM) {
                    if (a.out.g_depth) a.out.g_depth[pix] = dsum[p];
                    if (a.out.g_normal) {
                        a.out.g_normal[3 * pix] = nx[p]; a.out.g_normal[3 * pix + 1] = ny[p];
                        a.out.g_normal[3 * pix + 2] = nz[p];
                    }
                }
                if (a.out.image || a.out.image_rgba8) {
                    const float3 im = im_of(a, cs[p], wsum[p], cr[p], cg[p], cb[p]);
                    if (a.out.image) {
                        a.out.image[3 * pix] = im.x; a.out.image[3 * pix + 1] = im.y; a.out.image[3 * pix + 2] = im.z;
                    }
                    if (a.out.image_rgba8) store_rgba8(a.out.image_rgba8, pix, im);
                }
            } else {   // surfels_only (forward.py:407-410): empty Gaussian buffers
                if (a.out.image_rgba8) store_rgba8(a.out.image_rgba8, pix, cs[p]);
                if (a.out.image) {
                    a.out.image[3 * pix] = cs[p].x; a.out.image[3 * pix + 1] = cs[p].y;
                    a.out.image[3 * pix + 2] = cs[p].z;
                }
                if (a.out.g_weight) a.out.g_weight[pix] = 0.f;
                if (a.out.g_color) {
                    a.out.g_color[3 * pix] = 0.f; a.out.g_color[3 * pix + 1] = 0.f; a.out.g_color[3 * pix + 2] = 0.f;
                }
            }
        }
    }
#ifdef GES_TIMING
    if (lane == 0) {   // 16: sum of warp cycles, 17: max, 18: max (cycles << 24 | tile << 3 | warp),
                       // 19: warps over 50 us; 12-14: their list lengths, chunks walked, warp tests
        const unsigned long long dt = (unsigned long long)(clock64() - t_start);
        atomicAdd(&g_stats[16], dt);
        atomicMax(&g_stats[17], dt);
        atomicMax(&g_stats[18], (dt << 24) | ((unsigned long long)tile << 3) | (unsigned long long)warp);
        if (dt > 98000ull) {
            atomicAdd(&g_stats[19], 1ull);
            atomicAdd(&g_stats[12], (unsigned long long)tm_len);
            atomicAdd(&g_stats[13], (unsigned long long)tm_b1);
            atomicAdd(&g_stats[14], (unsigned long long)tm_t1);
            atomicAdd(&g_stats[5], (unsigned long long)(t_p1 - t_start));
            atomicAdd(&g_stats[6], (unsigned long long)(t_p2 - t_p1));
            atomicAdd(&g_stats[7], (unsigned long long)tm_b2);
            atomicAdd(&g_stats[8], (unsigned long long)tm_t2);
        }
    }
#endif
}

template <int SS, int PX, int MODE>
static void launch_kind(const TileArgs& a, int g_kind, bool geom, cudaStream_t s) {
    constexpr int WPC = tile_wpc<SS, PX>();
    const dim3 nt((unsigned)(a.ntx * (NWARP / WPC)), (unsigned)a.nty);
    const dim3 tb(32 * WPC);
    if (g_kind == 2) {
        if (geom) launch_pdl(k_tile<SS, PX, MODE, 2, true>, nt, tb, s, a);
        else launch_pdl(k_tile<SS, PX, MODE, 2, false>, nt, tb, s, a);
    } else {
        if (geom) launch_pdl(k_tile<SS, PX, MODE, 3, true>, nt, tb, s, a);
        else launch_pdl(k_tile<SS, PX, MODE, 3, false>, nt, tb, s, a);
    }
}

cudaError_t launch_tile(const TileArgs& a, int ss, int px, int mode, int g_kind, bool geom, cudaStream_t s) {
    if (a.ntx * a.nty == 0) return cudaSuccess;
    if (px == 2) {   // 32x32-pixel tiles, 2x2 pixels per thread (ss=1, no geometry)
        if (mode == 1) launch_kind<1, 2, 1>(a, 3, false, s);
        else if (mode == 2) launch_kind<1, 2, 2>(a, g_kind, false, s);
        else launch_kind<1, 2, 3>(a, g_kind, false, s);
    } else if (mode == 2) {
        launch_kind<1, 1, 2>(a, g_kind, geom, s);
    } else if (ss == 4) {
        if (mode == 1) launch_kind<2, 1, 1>(a, 3, false, s);
        else launch_kind<2, 1, 3>(a, g_kind, geom, s);
    } else {
        if (mode == 1) launch_kind<1, 1, 1>(a, 3, false, s);
        else launch_kind<1, 1, 3>(a, g_kind, geom, s);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- composite / smooth_geometry
__global__ void k_composite(const float* __restrict__ sc, const float* __restrict__ gc,
                            const float* __restrict__ gw, float sw, float* __restrict__ img, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float dn = sw + gw[i];
#pragma unroll
        for (int c = 0; c < 3; ++c) img[3 * i + c] = (sc[3 * i + c] * sw + gc[3 * i + c]) / dn;
    }
}

__global__ void k_smooth(const float* __restrict__ sd, const float* __restrict__ sn, const float* __restrict__ gd,
                         const float* __restrict__ gn, const float* __restrict__ gw, float* __restrict__ dout,
                         float* __restrict__ nout, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float dn = 1.0f + gw[i];
        dout[i] = (sd[i] + gd[i]) / dn;
        float v0 = (sn[3 * i] + gn[3 * i]) / dn, v1 = (sn[3 * i + 1] + gn[3 * i + 1]) / dn,
              v2 = (sn[3 * i + 2] + gn[3 * i + 2]) / dn;
        float nr = sqrtf(v0 * v0 + v1 * v1 + v2 * v2);
        bool ok = nr > 1e-12f;
        float inv = ok ? 1.0f / fmaxf(nr, 1e-12f) : 0.f;
        nout[3 * i] = v0 * inv; nout[3 * i + 1] = v1 * inv; nout[3 * i + 2] = v2 * inv;
    }
}

int read_stats(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, g_stats, sizeof(g_stats)) != cudaSuccess) return 1;
    unsigned long long z[24] = {};
    return cudaMemcpyToSymbol(g_stats, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}

cudaError_t launch_composite(const float* sc, const float* gc, const float* gw, float sw, float* img, int64_t n,
                             cudaStream_t s) {
    if (n > 0) k_composite<<<1184, 256, 0, s>>>(sc, gc, gw, sw, img, n);
    return cudaGetLastError();
}

cudaError_t launch_smooth(const float* sd, const float* sn, const float* gd, const float* gn, const float* gw,
                          float* d_out, float* n_out, int64_t n, cudaStream_t s) {
    if (n > 0) k_smooth<<<1184, 256, 0, s>>>(sd, sn, gd, gn, gw, d_out, n_out, n);
    return cudaGetLastError();
}

}  // namespace ges
