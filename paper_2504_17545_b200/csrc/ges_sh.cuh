// Real spherical harmonics to degree 3, graphics sign convention
// (reference sh.py:13-64, :117-133): rgb = clamp(0.5 + sum_k Y_k(dir) c_k, 0, 1).
#pragma once

#include <cuda_runtime.h>

namespace ges {

// Colour from the K x 3 coefficients of ONE primitive already in registers.
template <int DEG>
__device__ __forceinline__ float3 sh_color_regs(const float* c, float x, float y, float z) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    float b[K];
    b[0] = 0.28209479177387814f;
    if constexpr (DEG >= 1) {
        const float C1 = 0.4886025119029199f;
        b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
    }
    if constexpr (DEG >= 2) {
        float xx = x * x, yy = y * y, zz = z * z;
        b[4] = 1.0925484305920792f * x * y;
        b[5] = -1.0925484305920792f * y * z;
        b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
        b[7] = -1.0925484305920792f * x * z;
        b[8] = 0.5462742152960396f * (xx - yy);
        if constexpr (DEG >= 3) {
            b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
            b[10] = 2.890611442640554f * x * y * z;
            b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
            b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
            b[14] = 1.445305721320277f * z * (xx - yy);
            b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
        }
    }
    float r = 0.f, g = 0.f, bl = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        r = fmaf(b[k], c[3 * k], r);
        g = fmaf(b[k], c[3 * k + 1], g);
        bl = fmaf(b[k], c[3 * k + 2], bl);
    }
    return make_float3(fminf(fmaxf(0.5f + r, 0.f), 1.f), fminf(fmaxf(0.5f + g, 0.f), 1.f),
                       fminf(fmaxf(0.5f + bl, 0.f), 1.f));
}

// sh: K x 3 floats, coefficient-major (DC first), for ONE primitive.
template <int DEG>
__device__ __forceinline__ float3 sh_color(const float* __restrict__ sh, float x, float y, float z) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    float c[K * 3];
    if constexpr ((K * 3) % 4 == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(sh);
#pragma unroll
        for (int j = 0; j < K * 3 / 4; ++j) {
            float4 v = __ldg(s4 + j);
            c[4 * j] = v.x; c[4 * j + 1] = v.y; c[4 * j + 2] = v.z; c[4 * j + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < K * 3; ++j) c[j] = __ldg(sh + j);
    }
    return sh_color_regs<DEG>(c, x, y, z);
}

// ---- TMA form of the warp's coefficient fetch (Gaussian preprocess).
// sh_bulk_issue: one lane starts ONE bulk copy (cp.async.bulk, the TMA
// engine) of the warp's 32 consecutive padded rows into its shared slice,
// completing on the warp's mbarrier.  Issued at kernel entry, so the load
// flies while the caller does its float64 geometry; sh_color_bulk waits on
// the barrier and evaluates from the lane's row with 16-byte shared loads
// (no per-lane global loads or shared stores).  Both must be called by all
// 32 lanes.
// Row stride (floats) of the packed Gaussian SH blocks, in global memory AND
// in the preprocess's shared rows: K*3 rounded up to 16 bytes, plus 16 bytes
// when that is an even number of 16-byte units (4, 12, 28, 52 floats for
// degrees 0-3), so the rows' 16-byte reads by 8 lanes hit distinct bank
// groups and a warp's 32 consecutive rows arrive with ONE bulk copy.
__host__ __device__ constexpr int gsh_stride(int deg) {
    return (((3 * (deg + 1) * (deg + 1) + 3) & ~3) / 4) % 2 == 0 ? ((3 * (deg + 1) * (deg + 1) + 3) & ~3) + 4
                                                                  : ((3 * (deg + 1) * (deg + 1) + 3) & ~3);
}
template <int DEG>
__host__ __device__ constexpr int sh_bulk_stride() { return gsh_stride(DEG); }

// One bulk copy (cp.async.bulk, the TMA engine) of the warp's rows i0 ..
// i0+31 (< n) into its shared slice, completing on the warp's mbarrier.
template <int DEG>
__device__ __forceinline__ void sh_bulk_issue(const float* __restrict__ sh, int64_t i0, int64_t n, float* smw,
                                              uint64_t* bar) {
    constexpr int STR = sh_bulk_stride<DEG>();
    const int lane = threadIdx.x & 31;
    const int cnt = n - i0 < 32 ? (int)(n - i0) : 32;
    if (cnt <= 0) return;   // a warp past the end has nothing to fetch (and never waits)
    if (lane == 0) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(cnt * STR * 4) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(smw)), "l"(sh + i0 * STR), "r"(cnt * STR * 4), "r"(b)
                     : "memory");
    }
}

template <int DEG>
__device__ __forceinline__ float3 sh_color_bulk(const float* smw, uint64_t* bar, int64_t i0, int64_t n, float x,
                                                float y, float z) {
    constexpr int K3 = 3 * (DEG + 1) * (DEG + 1), STR = sh_bulk_stride<DEG>();
    if (n - i0 <= 0) return make_float3(0.f, 0.f, 0.f);   // (no fetch was issued for this warp)
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b) : "memory");
    }
    const float4* row = reinterpret_cast<const float4*>(smw + (threadIdx.x & 31) * STR);
    float c[(K3 + 3) & ~3];
#pragma unroll
    for (int j = 0; j < (K3 + 3) / 4; ++j) {
        const float4 v = row[j];
        c[4 * j] = v.x; c[4 * j + 1] = v.y; c[4 * j + 2] = v.z; c[4 * j + 3] = v.w;
    }
    return sh_color_regs<DEG>(c, x, y, z);
}

__device__ __forceinline__ float3 sh_color_dyn(int deg, const float* __restrict__ sh, float x, float y,
                                               float z) {
    switch (deg) {
        case 0: return sh_color<0>(sh, x, y, z);
        case 1: return sh_color<1>(sh, x, y, z);
        case 2: return sh_color<2>(sh, x, y, z);
        default: return sh_color<3>(sh, x, y, z);
    }
}

}  // namespace ges
