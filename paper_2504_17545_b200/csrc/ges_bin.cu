// Sort-free tile binning, steps 2 and 3 (step 1, the count, is fused into the
// preprocess kernels): exclusive prefix sum over the per-tile counts, then a
// fill pass that appends each primitive id to every tile its pixel range
// overlaps.  Replaces the per-tile O(N) selection scan of the reference
// (forward.py:168-169, :294-295) -- the reference's dominant CPU cost.
#include <cub/block/block_scan.cuh>

#include "ges_launch.h"

namespace ges {

constexpr int SCAN_T = 1024;

// Block b of the grid scans array b (0 = surfel tiles, 1 = Gaussian tiles).
__global__ void __launch_bounds__(SCAN_T) k_scan(uint32_t* cnt_s, uint32_t* off_s, uint32_t* cur_s, int n_s,
                                                 uint32_t* cnt_g, uint32_t* off_g, uint32_t* cur_g, int n_g,
                                                 int64_t cap_s, int64_t cap_g, ges_frame_status_t* st) {
    using Scan = cub::BlockScan<uint32_t, SCAN_T>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t carry;
    uint32_t* cnt = blockIdx.x ? cnt_g : cnt_s;
    uint32_t* off = blockIdx.x ? off_g : off_s;
    uint32_t* cur = blockIdx.x ? cur_g : cur_s;
    int n = blockIdx.x ? n_g : n_s;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += SCAN_T) {
        int i = base + threadIdx.x;
        uint32_t v = i < n ? cnt[i] : 0u, ex, tot;
        Scan(tmp).ExclusiveSum(v, ex, tot);
        uint32_t c = carry;
        if (i < n) {
            off[i] = c + ex;
            cur[i] = c + ex;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry = c + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        off[n] = carry;
        int64_t cap = blockIdx.x ? cap_g : cap_s;
        if (blockIdx.x) st->gaussian_pairs = carry; else st->surfel_pairs = carry;
        if ((int64_t)carry > cap) atomicOr(&st->overflow, 1);
    }
}

cudaError_t launch_scan(uint32_t* counts_s, uint32_t* off_s, uint32_t* cur_s, int ntiles_s,
                        uint32_t* counts_g, uint32_t* off_g, uint32_t* cur_g, int ntiles_g,
                        int64_t cap_s, int64_t cap_g, ges_frame_status_t* status, cudaStream_t s) {
    k_scan<<<2, SCAN_T, 0, s>>>(counts_s, off_s, cur_s, ntiles_s, counts_g, off_g, cur_g, ntiles_g, cap_s,
                                cap_g, status);
    return cudaGetLastError();
}

__device__ __forceinline__ void fill_one(uint32_t id, uint32_t sx, uint32_t sy, int tile_px, int ntx,
                                         uint32_t* cur, uint32_t* list, int64_t cap) {
    int x0 = span_lo(sx), x1 = span_hi(sx), y0 = span_lo(sy), y1 = span_hi(sy);
    if (x1 < x0 || y1 < y0) return;
    for (int ty = y0 / tile_px; ty <= y1 / tile_px; ++ty)
        for (int tx = x0 / tile_px; tx <= x1 / tile_px; ++tx) {
            uint32_t slot = atomicAdd(cur + ty * ntx + tx, 1u);
            if ((int64_t)slot < cap) list[slot] = id;
        }
}

// One thread per primitive over the concatenated surfel and Gaussian ranges.
__global__ void __launch_bounds__(256) k_fill(const SurfRec* __restrict__ srec, int64_t ns, uint32_t* cur_s,
                                              uint32_t* list_s, int64_t cap_s, int s_tile_px, int s_ntx,
                                              const float4* __restrict__ grec, int64_t ng, int g_kind,
                                              uint32_t* cur_g, uint32_t* list_g, int64_t cap_g, int g_ntx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < ns) {
        float4 r3 = __ldg(&srec[i].r3);
        fill_one((uint32_t)i, __float_as_uint(r3.y), __float_as_uint(r3.z), s_tile_px, s_ntx, cur_s, list_s,
                 cap_s);
    } else if (i < ns + ng) {
        int64_t j = i - ns;
        uint32_t sx, sy;
        if (g_kind == 2) {   // Gauss2Rec: r3 = (sigma, eps, rect_x, rect_y)
            float4 r3 = __ldg(grec + j * 5 + 3);
            sx = __float_as_uint(r3.z); sy = __float_as_uint(r3.w);
        } else {             // GaussRec: r2.w = rect_x, r3.x = rect_y
            sx = __float_as_uint(__ldg(grec + j * 4 + 2).w);
            sy = __float_as_uint(__ldg(grec + j * 4 + 3).x);
        }
        fill_one((uint32_t)j, sx, sy, TILE, g_ntx, cur_g, list_g, cap_g);
    }
}

cudaError_t launch_fill(const void* srec, int64_t ns, uint32_t* cur_s, uint32_t* list_s, int64_t cap_s,
                        int s_tile_px, int s_ntx, const void* grec, int64_t ng, int g_kind,
                        uint32_t* cur_g, uint32_t* list_g, int64_t cap_g, int g_ntx, cudaStream_t s) {
    int64_t n = ns + ng;
    if (n == 0) return cudaSuccess;
    k_fill<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((const SurfRec*)srec, ns, cur_s, list_s, cap_s,
                                                        s_tile_px, s_ntx, (const float4*)grec, ng, g_kind,
                                                        cur_g, list_g, cap_g, g_ntx);
    return cudaGetLastError();
}

}  // namespace ges
