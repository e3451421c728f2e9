// Shared device definitions for the GES sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ges_b200.h"

namespace ges {

constexpr int TILE = 16;                 // base-resolution tile (forward.py:27)
constexpr int TILE_PX = TILE * TILE;     // one thread per base pixel
constexpr int NWARP = TILE_PX / 32;      // 8 warps, each an 8x4 pixel patch
constexpr double R_OPAQUE = 3.3290429691304455;   // sqrt(2 ln 255), filters.py:28-30
constexpr float R2_F = 11.082527f;                // fp32 R^2 (NEP-50 weak scalar)
constexpr double NEAR = 0.01;                     // cameras.py:14
constexpr float NEAR_F = 0.01f;
constexpr float PARALLEL_EPS_F = 1e-8f;           // geometry.py:15
constexpr double SCREEN_VAR = 0.3;                // filters.py:21
constexpr float ALPHA_CUTOFF_F = 1.0f / 255.0f;   // forward.py:26

constexpr float LOG2E_F = 1.4426950408889634f;
constexpr float LN2_F = 0.6931471805599453f;

// 2^x on the SFU, flush-to-zero (results below 2^-126 only ever fail the
// 1/255 alpha cutoff)
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 1/x on the SFU (approximate, ~1 ulp), flush-to-zero; callers guarantee |x| >= 1e-8
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// sqrt on the SFU (approximate, relative error ~2^-22, sqrt(0) = 0); for
// bounds and thresholds that carry their own margins
__device__ __forceinline__ float sqrt_ftz(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Camera in the form the kernels use (double for per-primitive math).
struct CamK {
    double fx, fy, cx, cy;
    double ifx, ify;    // 1/fx, 1/fy
    double R[9];
    double t[3];
    double pos[3];      // world-space camera centre -R^T t (cameras.py:38)
    int W, H;           // resolution of THIS pass (hi-res for ss=4 surfels)
};

// Per-surfel screen record written by the surfel preprocess (48 B).
//   r0 = (D0, Dx, Dy, nq)   den(x,y) = n.d = D0 + Dx*(x-xr) + Dy*(y-yr)
//   r1 = (U0, Ux, Uy, xr)   U = ((n.q) a1 - (a1.q) n).d / s1, u = U/den
//   r2 = (V0, Vx, Vy, yr)   V likewise with a2, s2
// and, in a separate dense array (16 B per surfel, so binning and the tile
// kernel's cull read 16 B instead of a 64-byte DRAM burst per surfel):
//   cull = (zmin, rect_x, rect_y, source id)  rect packed lo | hi << 16 (pixel ranges)
struct __align__(16) SurfRec {
    float4 r0, r1, r2;
};

// Per-Gaussian screen records.  Everything the cull needs (depth test inputs
// and pixel range) is a separate dense array of 16-byte records `c`, so
// binning and the tile kernel's staging read 16 B per entry and fetch the
// rest only for the few entries that survive.
// 3D EWA: c = (depth, eps, rect_x, rect_y), and 48 B
//   r0 = (mx_int, mx_frac, my_int, my_frac)       mean2d split for precision
//   r1 = (pa, pb, pc, sigma)  log2(e) * power = pa dx^2 + pb dx dy + pc dy^2,
//                             alpha = sigma * 2^(pa dx^2 + ...)
//   r2 = (0, r, g, b)         view colour (x unused)
struct __align__(16) GaussRec {
    float4 r0, r1, r2;
};

// Planar 2D Gaussian: c = (slab/cull key, eps, rect_x, rect_y), and 80 B: the
// ray-plane homography r0..r2 like SurfRec, r3 = (sigma, r2max, 0, 0),
// r4 = (r, g, b, 0).
struct __align__(16) Gauss2Rec {
    float4 r0, r1, r2, r3, r4;
};

// Depth slabs of the (tile, slab) bins: NSLAB equal slabs over the view's
// depth range [zlo, zlo + NSLAB/inv_dz); keys outside clamp to the end slabs.
#ifndef GES_NSLAB
#define GES_NSLAB 32
#endif
constexpr int NSLAB = GES_NSLAB;   // multiple of 4
static_assert(NSLAB % 4 == 0, "scan reads slab counters as uint4");

// Slab index of relative list position `rel` of a tile: the number of slab
// ends <= rel (ends are non-decreasing).  One vote per 32 slabs; every lane
// of the warp gets the same answer.
__device__ __forceinline__ int slab_of_pos(const uint32_t* ends, uint32_t rel, int lane) {
    int n = 0;
#pragma unroll
    for (int k = 0; k < NSLAB; k += 32) {
        const bool le = lane + k < NSLAB - 1 && ends[lane + k] <= rel;
        n += __popc(__ballot_sync(0xffffffffu, le));
    }
    return n;
}

struct SlabMap {
    float zlo, inv_dz;
    __device__ __forceinline__ int slab(float key) const {
        float f = floorf((key - zlo) * inv_dz);
        return f > 0.f ? (f < (float)(NSLAB - 1) ? (int)f : NSLAB - 1) : 0;   // NaN -> 0
    }
    float dz;   // 1 / inv_dz
    // every key binned into slab s is >= this bound (slab 0 also takes keys below zlo)
    __device__ __forceinline__ float lower(int s) const {
        if (s == 0 || !(inv_dz > 0.f)) return -INFINITY;
        const float b = fmaf((float)s, dz, zlo);
        return b - (fabsf(b) * 1e-5f + 1e-6f);
    }
};

// Slab key of a 3D Gaussian: it can pass the gate d < D_s + eps only where
// D_s > d - eps (forward.py:310).
__device__ __forceinline__ float gauss_key(float depth, float eps) { return depth - eps; }

// Tiles per scan chunk (k_scan block: 8 warps, 2^SCAN_CHUNK_SHIFT / 8 tiles each).
#ifndef GES_SCAN_CHUNK_SHIFT
#define GES_SCAN_CHUNK_SHIFT 5
#endif
constexpr int SCAN_CHUNK_SHIFT = GES_SCAN_CHUNK_SHIFT;

// One binning pass (surfels or Gaussians).
struct BinPass {
    uint32_t* cnt;      // ntiles * NSLAB: counts -> slab prefix -> slab ends
    uint32_t* off;      // ntiles: first list slot of each tile within its scan chunk
    uint32_t* chunk;    // nchunks + 1: first list slot of each chunk of 2^SCAN_CHUNK_SHIFT tiles; [nchunks] = total
    uint32_t* ticket;   // scan completion counter (zeroed per frame)
    uint32_t* list;     // cap primitive ids (packed indices)
    int64_t cap;
    int ntiles, ntx, tile_px, tile_shift;
    uint32_t* order;    // or NULL; surfel pass: tiles by descending pair count (tile kernel launch order)
    uint32_t* tot;      // with order: per-tile pair totals (scan scratch)
    __device__ __forceinline__ uint32_t tile_off(int t) const { return chunk[t >> SCAN_CHUNK_SHIFT] + off[t]; }
};

__device__ __forceinline__ uint32_t pack_span(int lo, int hi) {
    return (uint32_t)lo | ((uint32_t)hi << 16);
}
__device__ __forceinline__ int span_lo(uint32_t s) { return (int)(s & 0xffffu); }
__device__ __forceinline__ int span_hi(uint32_t s) { return (int)(s >> 16); }

}  // namespace ges
