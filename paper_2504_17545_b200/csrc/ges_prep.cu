// K0 scene pack, K1 surfel preprocess, K4 Gaussian preprocess (3D EWA and
// planar 2D).  One thread per primitive; per-primitive geometry in float64
// (as the reference does before casting to dtype, forward.py:148-163), the
// per-pixel coefficients it emits in float32.  Each kernel also counts its
// primitive into the tiles its pixel range overlaps (count pass of the
// sort-free count -> prefix-sum -> fill binning).
#include <math.h>

#include "ges_launch.h"
#include "ges_sh.cuh"

#ifndef GES_PREP_MINB
#define GES_PREP_MINB 5   // resident 256-thread blocks per SM of the surfel preprocess (48 registers)
#endif
#ifndef GES_GPREP_MINB
#define GES_GPREP_MINB 7   // resident 128-thread blocks per SM, Gaussian preprocess (72 registers)
#endif

namespace ges {

CamK make_cam(const ges_camera_t& c, int scale) {
    CamK k{};
    k.fx = c.fx * scale; k.fy = c.fy * scale; k.cx = c.cx * scale; k.cy = c.cy * scale;
    k.ifx = 1.0 / k.fx; k.ify = 1.0 / k.fy;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) k.R[3 * i + j] = c.w2c[4 * i + j];
        k.t[i] = c.w2c[4 * i + 3];
    }
    for (int j = 0; j < 3; ++j)   // -R^T t
        k.pos[j] = -(k.R[j] * k.t[0] + k.R[3 + j] * k.t[1] + k.R[6 + j] * k.t[2]);
    k.W = c.width * scale; k.H = c.height * scale;
    return k;
}

// ---------------------------------------------------------------- helpers
struct d3 { double x, y, z; };
__device__ __forceinline__ d3 mk(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ d3 scl(d3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ d3 sub(d3 a, d3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ d3 rot(const CamK& c, d3 v) {   // W v
    return {c.R[0] * v.x + c.R[1] * v.y + c.R[2] * v.z, c.R[3] * v.x + c.R[4] * v.y + c.R[5] * v.z,
            c.R[6] * v.x + c.R[7] * v.y + c.R[8] * v.z};
}

// Columns of the rotation of quaternion (w,x,y,z), renormalised (geometry.py:18-36).
__device__ __forceinline__ void quat_cols(float4 qf, d3& c0, d3& c1, d3& c2) {
    double w = qf.x, x = qf.y, y = qf.z, z = qf.w;
    double inv = rsqrt(w * w + x * x + y * y + z * z);
    w *= inv; x *= inv; y *= inv; z *= inv;
    c0 = mk(1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y));
    c1 = mk(2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x));
    c2 = mk(2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y));
}

// Screen AABB of the projected disc {q + a m1 + b m2 : a^2+b^2<=1}
// (geometry.py:273-302) -> inclusive ranges of the pixels whose centres it
// contains (forward.py:85-96 pads them by another half pixel).  Returns false
// if the range is empty.
//
// The ranges only cull (every pixel in them still gets the exact coverage
// test), so they need to contain the reference's, not to equal them.  The
// tangent condition is solved relative to the projected centre s0 = q_a/q_z,
// s = s0 + delta: with w = m_a - s0 m_z (per disc axis),
//   delta^2 (q_z^2 - |m_z|^2) + 2 delta (w.m_z) - |w|^2 = 0,
// whose coefficients are of the disc's size, so float32 is accurate to
// ~1e-6 of the disc extent; the bounds are widened by PAD_PX to cover that.
// q_z^2 <= |m_z|^2 (the disc reaches the focal plane) is the reference's
// whole-screen case; it is taken with a relative margin (superset).
__device__ bool disc_ranges(d3 q, d3 m1, d3 m2, const CamK& c, int& x0, int& x1, int& y0, int& y1) {
    constexpr float PAD_PX = 0.01f;
    const float qz = (float)q.z, m1z = (float)m1.z, m2z = (float)m2.z;
    const float A = fmaf(qz, qz, -(m1z * m1z + m2z * m2z));
    const bool whole = !(A > 1e-5f * qz * qz);
    auto clampi = [](float v, int n) -> int {
        if (!(v >= 0.f)) return 0;
        if (v > n - 1.f) return n - 1;
        return (int)v;
    };
    if (whole) {
        x0 = 0; x1 = c.W - 1; y0 = 0; y1 = c.H - 1;
        return c.W > 0 && c.H > 0;
    }
    const float iA = rcp_ftz(A), iz = rcp_ftz(qz);   // (1 ulp: inside the padding)
    float lo[2], hi[2];
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
        const float f = (float)(ax ? c.fy : c.fx), cc = (float)(ax ? c.cy : c.cx);
        const float s0 = (float)(ax ? q.y : q.x) * iz;
        const float w1 = fmaf(-s0, m1z, (float)(ax ? m1.y : m1.x)), w2 = fmaf(-s0, m2z, (float)(ax ? m2.y : m2.x));
        const float B = fmaf(w1, m1z, w2 * m2z), Cw = fmaf(w1, w1, w2 * w2);
        const float root = sqrt_ftz(fmaxf(fmaf(B, B, A * Cw), 0.f));
        const float dlo = (-B - root) * iA, dhi = (-B + root) * iA;
        const float clo = fmaf(f, s0 + dlo, cc), chi = fmaf(f, s0 + dhi, cc);
        const float pad = PAD_PX + 1e-6f * (fabsf(clo) + fabsf(chi));
        lo[ax] = clo - pad;
        hi[ax] = chi + pad;
    }
    // pixels whose centre p + 0.5 lies in [lo, hi]: a covered pixel's centre is
    // inside the projected ellipse, so inside its (padded) box -- the
    // reference's extra half-pixel of padding (forward.py:85-96) only adds
    // pixels that fail the exact test
    const float fx0 = ceilf(lo[0] - 0.5f), fx1 = floorf(hi[0] - 0.5f);
    const float fy0 = ceilf(lo[1] - 0.5f), fy1 = floorf(hi[1] - 0.5f);
    // A disc whose padded box lies entirely beyond an image edge covers no
    // pixel.  The reference's clamp turns its range into the edge row/column
    // (forward.py:85-96), so every off-screen disc is a candidate of the
    // edge tiles there and is rejected pixel by pixel; dropping it here gives
    // the same pixels and keeps the edge tiles' lists short.
    if (fx0 > c.W - 1.f || fx1 < 0.f || fy0 > c.H - 1.f || fy1 < 0.f) return false;
    x0 = clampi(fx0, c.W);
    x1 = clampi(fx1, c.W);
    y0 = clampi(fy0, c.H);
    y1 = clampi(fy1, c.H);
    return x1 >= x0 && y1 >= y0;
}

// Count this primitive into every tile of its pixel range.  Called by ALL
// lanes of the warp (empty ranges allowed); lanes that hit the same tile in
// the same round are merged into one atomic (spatially ordered scenes make
// warps' primitives share tiles).
__device__ __forceinline__ void count_tiles(uint32_t* cnt, const Grid& g, bool live, int x0, int x1, int y0,
                                            int y1, float zkey) {
    const int sh = __ffs(g.tile_px) - 1;   // tiles are 16, 32 or 64 px
    int tx0 = x0 >> sh, tx1 = x1 >> sh, ty0 = y0 >> sh, ty1 = y1 >> sh;
    int tx = tx0, ty = ty0;
    bool more = live;
    const int slab = g.slabs.slab(zkey);
    const unsigned lane = threadIdx.x & 31;
    while (__any_sync(0xffffffffu, more)) {
        int key = more ? (ty * g.ntx + tx) * NSLAB + slab : -1;
        unsigned peers = __match_any_sync(0xffffffffu, key);
        if (more && lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(cnt + key, (uint32_t)__popc(peers));
        const bool wrap = tx >= tx1;   // next tile, row-major over the range (branch-free)
        tx = wrap ? tx0 : tx + 1;
        ty += wrap;
        more = more && !(wrap && ty > ty1);
    }
}

// Ray-plane homography of a planar primitive relative to pixel (xr, yr):
// n.d, U and V as affine functions of the pixel offset (see SurfRec).
__device__ __forceinline__ float4 affine_of(d3 v, const CamK& c, int xr, int yr, float last) {
    double cx = v.x * c.ifx, cy = v.y * c.ify;
    double c0 = cx * (xr + 0.5 - c.cx) + cy * (yr + 0.5 - c.cy) + v.z;
    return make_float4((float)c0, (float)cx, (float)cy, last);
}

// 1/x of a positive normal x to float64 accuracy without the IEEE division's
// slow path: the float32 estimate (rel. error < 2^-22) refined by two Newton
// steps (error squared each), a few float64 ulp.
__device__ __forceinline__ double rcp_pos(double x) {
    double r = (double)rcp_ftz((float)x);
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}

__device__ __forceinline__ void planar_coeffs(d3 q, d3 a1, d3 a2, d3 n, double s1, double s2,
                                              const CamK& c, int x0, int x1, int y0, int y1,
                                              float4& r0, float4& r1, float4& r2) {
    double nq = dot(n, q);
    d3 cu = scl(sub(scl(a1, nq), scl(n, dot(a1, q))), rcp_pos(s1));
    d3 cv = scl(sub(scl(a2, nq), scl(n, dot(a2, q))), rcp_pos(s2));
    int xr = x0, yr = y0;
    if (q.z > 0.0) {   // reference pixel of the coefficients: any pixel of the range works
        const float iz = rcp_ftz((float)q.z);
        const float mx = fmaf((float)c.fx * (float)q.x, iz, (float)c.cx);
        const float my = fmaf((float)c.fy * (float)q.y, iz, (float)c.cy);
        xr = mx >= (float)x1 ? x1 : (mx > (float)x0 ? (int)mx : x0);   // clamp(floor(mx), x0, x1)
        yr = my >= (float)y1 ? y1 : (my > (float)y0 ? (int)my : y0);
    }
    r0 = affine_of(n, c, xr, yr, (float)nq);
    r1 = affine_of(cu, c, xr, yr, (float)xr);
    r2 = affine_of(cv, c, xr, yr, (float)yr);
}

// ---------------------------------------------------------------- K0 pack
__global__ void k_pack_prims(ges_scene_src_t src, ges_scene_t dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < src.n_surfels) {
        const int64_t o = src.s_order ? src.s_order[i] : i;
        const double* p = src.s_pos + 3 * o;
        const double* q = src.s_quat + 4 * o;
        const double* l = src.s_log_scale + 2 * o;
        dst.s_id[i] = (int32_t)o;
        dst.s_pack[o] = (int32_t)i;
        double nrm = 1.0 / sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        reinterpret_cast<float4*>(dst.s_pos_s1)[i] = make_float4(p[0], p[1], p[2], exp(l[0]));
        reinterpret_cast<float4*>(dst.s_quat)[i] =
            make_float4(q[0] * nrm, q[1] * nrm, q[2] * nrm, q[3] * nrm);
        dst.s_s2[i] = (float)exp(l[1]);
    }
    if (i < src.n_gaussians) {
        // primitives.py:113-131: eff_scale = sqrt(s^2 + f3), eff_opacity =
        // sigma * prod(s / eff_s), epsilon = (5/D) sum eff_s.
        int D = src.gaussian_dim;
        const int64_t o = src.g_order ? src.g_order[i] : i;
        const double* p = src.g_pos + 3 * o;
        const double* q = src.g_quat + 4 * o;
        const double* l = src.g_log_scale + D * o;
        double f3 = src.g_filter3d ? src.g_filter3d[o] : 0.0;
        double sig = 1.0 / (1.0 + exp(-src.g_raw_opacity[o]));
        double es[3] = {0.0, 0.0, 0.0}, esum = 0.0;
        for (int k = 0; k < D; ++k) {
            double s = exp(l[k]);
            es[k] = sqrt(s * s + f3);
            sig *= s / es[k];
            esum += es[k];
        }
        double nrm = 1.0 / sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        reinterpret_cast<float4*>(dst.g_pos_op)[i] = make_float4(p[0], p[1], p[2], sig);
        reinterpret_cast<float4*>(dst.g_quat)[i] =
            make_float4(q[0] * nrm, q[1] * nrm, q[2] * nrm, q[3] * nrm);
        reinterpret_cast<float4*>(dst.g_scale_eps)[i] =
            make_float4(es[0], es[1], es[2], (5.0 / D) * esum);
    }
}

// Row-permuted float64 -> float32 copy of the (N, K*3) SH blocks into rows of
// `stride` floats (zero padding after the K*3 coefficients).
__global__ void k_pack_sh(const double* __restrict__ a, float* __restrict__ b, int64_t n, int row, int stride,
                          const int32_t* __restrict__ order) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / stride, c = i - r * stride;
        int64_t src = order ? (int64_t)order[r] : r;
        b[i] = c < row ? (float)a[src * row + c] : 0.f;
    }
}

cudaError_t launch_pack(const ges_scene_src_t& src, const ges_scene_t& dst, cudaStream_t s) {
    int64_t n = src.n_surfels > src.n_gaussians ? src.n_surfels : src.n_gaussians;
    if (n > 0) k_pack_prims<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, dst);
    int K = (src.sh_degree + 1) * (src.sh_degree + 1);
    const int gs = gsh_stride(src.sh_degree);   // Gaussian rows padded for the preprocess's bulk copies
    if (src.n_surfels)
        k_pack_sh<<<1184, 256, 0, s>>>(src.s_sh, dst.s_sh, src.n_surfels * K * 3, K * 3, K * 3, src.s_order);
    if (src.n_gaussians)
        k_pack_sh<<<1184, 256, 0, s>>>(src.g_sh, dst.g_sh, src.n_gaussians * gs, K * 3, gs, src.g_order);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- K1 surfels
// forward.py:148-158 (frames, colour, n_vis, cull, bounds, ranges) for one surfel.
template <int DEG>
__global__ void __launch_bounds__(256, GES_PREP_MINB) k_surfel_prep(ges_scene_t sc, CamK cam, Grid g, PrepOut o) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0 && o.zero_status) *o.zero_status = ges_frame_status_t{0, 0, 0, 0};
    const bool valid_thread = i < sc.n_surfels;
    if (!valid_thread) i = sc.n_surfels - 1;   // idle lanes still join the warp-wide count
    float4 ps = __ldg(reinterpret_cast<const float4*>(sc.s_pos_s1) + i);
    float4 qf = __ldg(reinterpret_cast<const float4*>(sc.s_quat) + i);
    double s1 = ps.w, s2 = __ldg(sc.s_s2 + i);
    d3 r0, r1, r2;
    quat_cols(qf, r0, r1, r2);
    d3 p = mk(ps.x, ps.y, ps.z);
    d3 q = rot(cam, p);
    q.x += cam.t[0]; q.y += cam.t[1]; q.z += cam.t[2];
    d3 a1 = rot(cam, r0), a2 = rot(cam, r1), n = rot(cam, r2);
    SurfRec rec;
    int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
    bool alive = valid_thread && q.z > NEAR;
    if (alive) alive = disc_ranges(q, scl(a1, s1 * R_OPAQUE), scl(a2, s2 * R_OPAQUE), cam, x0, x1, y0, y1);
    // nearest camera depth of the disc, made conservative against the float32
    // evaluation of the per-pixel hit depth (culling and slab key only)
    // (float32 radius, rounded up by 2e-6 relative: the bound stays conservative)
    const float rz = sqrt_ftz((float)(s1 * s1 * a1.z * a1.z + s2 * s2 * a2.z * a2.z)) * (float)(R_OPAQUE * (1.0 + 2e-6));
    double zmin = q.z - (double)rz;
    zmin -= 1e-5 * fabs(zmin) + 1e-6;
    const float zkey = (float)zmin;
    count_tiles(o.bin_count, g, alive, x0, x1, y0, y1, zkey);
    if (!valid_thread) return;
    const int32_t sid = __ldg(sc.s_id + i);
    if (alive) {
        planar_coeffs(q, a1, a2, n, s1, s2, cam, x0, x1, y0, y1, rec.r0, rec.r1, rec.r2);
        o.cull[i] = make_float4(zkey, __uint_as_float(pack_span(x0, x1)), __uint_as_float(pack_span(y0, y1)),
                                __int_as_float(sid));
        reinterpret_cast<SurfRec*>(o.rec)[i] = rec;
        // view colour (forward.py:99-103) and n_vis (:152) are evaluated for
        // winners only, in the tile kernel
    } else {   // empty pixel range: never binned, the coefficients are never read
        o.cull[i] = make_float4(0.f, __uint_as_float(pack_span(1, 0)), __uint_as_float(pack_span(1, 0)),
                                __int_as_float(sid));
    }
}

cudaError_t launch_surfel_prep(const ges_scene_t& sc, const CamK& cam, const Grid& g, const PrepOut& o,
                               cudaStream_t s) {
    if (sc.n_surfels == 0) return cudaSuccess;
    unsigned nb = (unsigned)((sc.n_surfels + 255) / 256);
    switch (sc.sh_degree) {
        case 0: k_surfel_prep<0><<<nb, 256, 0, s>>>(sc, cam, g, o); break;
        case 1: k_surfel_prep<1><<<nb, 256, 0, s>>>(sc, cam, g, o); break;
        case 2: k_surfel_prep<2><<<nb, 256, 0, s>>>(sc, cam, g, o); break;
        default: k_surfel_prep<3><<<nb, 256, 0, s>>>(sc, cam, g, o); break;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- K4 Gaussians
struct GaussCfg {
    int mip, eps_const, geom;
    float eps_value;
};

// Gaussian preprocess blocks: 128 threads (4 warps).
constexpr int GPREP_T = 128;

// Shared state of the warp's SH fetch: its 32 coefficient rows (one TMA bulk
// copy of the packed, row-padded blocks, sh_bulk_issue) + the mbarrier.
template <int DEG>
struct GaussShSmem {
    alignas(16) float rows[GPREP_T / 32][32 * sh_bulk_stride<DEG>()];
    uint64_t bar[GPREP_T / 32];
};

// Start the warp's coefficient fetch at kernel entry.
template <int DEG>
__device__ __forceinline__ void gauss_sh_prefetch(const ges_scene_t& sc, GaussShSmem<DEG>& sm) {
    const int w = threadIdx.x >> 5;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31u);
    sh_bulk_issue<DEG>(sc.g_sh, i0, sc.n_gaussians, sm.rows[w], &sm.bar[w]);
}

// View colour of this lane's Gaussian (forward.py:99-109) from the warp's
// fetched rows; all lanes call it.
template <int DEG>
__device__ __forceinline__ float3 gauss_view_colour(const ges_scene_t& sc, const CamK& cam, d3 p,
                                                    GaussShSmem<DEG>& sm) {
    // (the colour is evaluated in float32: the direction is too)
    const float dx = (float)(cam.pos[0] - p.x), dy = (float)(cam.pos[1] - p.y), dz = (float)(cam.pos[2] - p.z);
    const float inv = rsqrtf(fmaxf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)), 1e-24f));   // (2 ulp)
    const int w = threadIdx.x >> 5;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31u);
    return sh_color_bulk<DEG>(sm.rows[w], &sm.bar[w], i0, sc.n_gaussians, dx * inv, dy * inv, dz * inv);
}

// 3D EWA: geometry.py:114-132 + forward.py:252-290.
template <int DEG>
__global__ void __launch_bounds__(GPREP_T, GES_GPREP_MINB) k_gauss3_prep(ges_scene_t sc, CamK cam, Grid g, GaussCfg cfg,
                                                     PrepOut o) {
    __shared__ GaussShSmem<DEG> shsm;
    gauss_sh_prefetch<DEG>(sc, shsm);   // TMA: the warp's SH blocks fly during the geometry
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid_thread = i < sc.n_gaussians;
    if (!valid_thread) i = sc.n_gaussians - 1;
    float4 po = __ldg(reinterpret_cast<const float4*>(sc.g_pos_op) + i);
    float4 qf = __ldg(reinterpret_cast<const float4*>(sc.g_quat) + i);
    float4 se = __ldg(reinterpret_cast<const float4*>(sc.g_scale_eps) + i);
    d3 p = mk(po.x, po.y, po.z);
    d3 t = rot(cam, p);
    t.x += cam.t[0]; t.y += cam.t[1]; t.z += cam.t[2];
    bool valid = valid_thread && t.z > NEAR;
    d3 ts = valid ? t : mk(0.0, 0.0, 1.0);
    d3 r0, r1, r2;
    quat_cols(qf, r0, r1, r2);
    // camera-space axes scaled: M = sum_k s_k^2 (W r_k)(W r_k)^T
    d3 w0 = scl(rot(cam, r0), se.x), w1 = scl(rot(cam, r1), se.y), w2 = scl(rot(cam, r2), se.z);
    double iz = 1.0 / ts.z;
    // J rows: j0 = (fx/z, 0, -fx x/z^2), j1 = (0, fy/z, -fy y/z^2); cov = sum_k (J w_k)(J w_k)^T
    double jx[3], jy[3];
    const d3 ws[3] = {w0, w1, w2};
    for (int k = 0; k < 3; ++k) {
        jx[k] = cam.fx * iz * ws[k].x - cam.fx * ts.x * iz * iz * ws[k].z;
        jy[k] = cam.fy * iz * ws[k].y - cam.fy * ts.y * iz * iz * ws[k].z;
    }
    double cv00 = jx[0] * jx[0] + jx[1] * jx[1] + jx[2] * jx[2];
    double cv11 = jy[0] * jy[0] + jy[1] * jy[1] + jy[2] * jy[2];
    double cv01 = jx[0] * jy[0] + jx[1] * jy[1] + jx[2] * jy[2];
    double raw_det = cv00 * cv11 - cv01 * cv01;
    double c00 = cv00 + SCREEN_VAR, c11 = cv11 + SCREEN_VAR, c01 = cv01;
    double det = c00 * c11 - c01 * c01;
    const double idet = 1.0 / det;
    double sig = po.w;
    if (cfg.mip) sig *= sqrt(fmax(raw_det, 0.0) * idet);
    valid = valid && det > 0.0;
    double la = c11 * idet, lb = -c01 * idet, lc = c00 * idet;
    // m2max = 2 ln(max(255 sig, 1e-12)) > 0  <=>  255 sig > 1 (exactly, ln is monotone with
    // ln 1 = 0); the support box only culls, so its radius is evaluated in float32 and widened
    valid = valid && 255.0 * sig > 1.0;
    // (__logf: absolute error < 4e-7 near 1, relative 2^-21 elsewhere; inside the widening)
    const float m2 = fmaxf(2.0f * __logf((float)(255.0 * sig)), 0.f) * 1.0001f + 4e-6f;
    const double rx = (double)(sqrt_ftz(m2 * (float)c00) * 1.0001f) + 1e-3;
    const double ry = (double)(sqrt_ftz(m2 * (float)c11) * 1.0001f) + 1e-3;
    double mx = cam.fx * ts.x * iz + cam.cx, my = cam.fy * ts.y * iz + cam.cy;
    GaussRec rec;
    int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
    if (valid) {
        auto clampi = [](double v, int n) -> int {
            if (!(v >= 0.0)) return 0;
            if (v > n - 1.0) return n - 1;
            return (int)v;
        };
        // pixel centres inside the (widened) support box (see disc_ranges)
        const double fx0 = ceil(mx - rx - 0.5), fx1 = floor(mx + rx - 0.5);
        const double fy0 = ceil(my - ry - 0.5), fy1 = floor(my + ry - 0.5);
        // off-screen support box: no pixel of the image reaches alpha >= 1/255
        // (the reference clamps it onto the edge tiles and rejects it per pixel)
        valid = !(fx0 > cam.W - 1.0 || fx1 < 0.0 || fy0 > cam.H - 1.0 || fy1 < 0.0);
        x0 = clampi(fx0, cam.W);
        x1 = clampi(fx1, cam.W);
        y0 = clampi(fy0, cam.H);
        y1 = clampi(fy1, cam.H);
        valid = valid && x1 >= x0 && y1 >= y0;
    }
    const float3 col = gauss_view_colour<DEG>(sc, cam, p, shsm);
    const float depf = (float)t.z, epsf = cfg.eps_const ? cfg.eps_value : se.w;
    count_tiles(o.bin_count, g, valid, x0, x1, y0, y1, gauss_key(depf, epsf));
    if (!valid_thread) return;
    if (valid) {
        double mxi = floor(mx), myi = floor(my);
        o.cull[i] = make_float4(depf, epsf, __uint_as_float(pack_span(x0, x1)), __uint_as_float(pack_span(y0, y1)));
        rec.r0 = make_float4((float)mxi, (float)(mx - mxi), (float)myi, (float)(my - myi));
        // conic pre-scaled by log2(e): the tile kernel evaluates exp as one ex2
        const double L2E = 1.4426950408889634;
        rec.r1 = make_float4((float)(-0.5 * L2E * la), (float)(-L2E * lb), (float)(-0.5 * L2E * lc), (float)sig);
        rec.r2 = make_float4(0.f, col.x, col.y, col.z);
        if (cfg.geom) {   // forward.py:277-284: shortest eff_scale axis, camera-facing
            int k = 0;
            double smin = se.x;
            if (se.y < smin) { k = 1; smin = se.y; }
            if (se.z < smin) { k = 2; }
            d3 nv = rot(cam, k == 0 ? r0 : (k == 1 ? r1 : r2));
            double sgn = dot(nv, t) < 0.0 ? 1.0 : -1.0;
            o.nrm[i] = make_float4((float)(nv.x * sgn), (float)(nv.y * sgn), (float)(nv.z * sgn), 0.f);
        }
        reinterpret_cast<GaussRec*>(o.rec)[i] = rec;
    } else {   // empty pixel range: never binned, the record is never read
        o.cull[i] = make_float4(0.f, 0.f, __uint_as_float(pack_span(1, 0)), __uint_as_float(pack_span(1, 0)));
    }
}

// Planar 2D Gaussians: forward.py:324-351 (+ filters.py:84-109 when mip).
template <int DEG>
__global__ void __launch_bounds__(GPREP_T, GES_GPREP_MINB) k_gauss2_prep(ges_scene_t sc, CamK cam, Grid g, GaussCfg cfg,
                                                     PrepOut o) {
    __shared__ GaussShSmem<DEG> shsm;
    gauss_sh_prefetch<DEG>(sc, shsm);   // TMA: the warp's SH blocks fly during the geometry
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid_thread = i < sc.n_gaussians;
    if (!valid_thread) i = sc.n_gaussians - 1;
    float4 po = __ldg(reinterpret_cast<const float4*>(sc.g_pos_op) + i);
    float4 qf = __ldg(reinterpret_cast<const float4*>(sc.g_quat) + i);
    float4 se = __ldg(reinterpret_cast<const float4*>(sc.g_scale_eps) + i);
    d3 r0, r1, r2;
    quat_cols(qf, r0, r1, r2);
    d3 p = mk(po.x, po.y, po.z);
    d3 q = rot(cam, p);
    q.x += cam.t[0]; q.y += cam.t[1]; q.z += cam.t[2];
    d3 a1 = rot(cam, r0), a2 = rot(cam, r1), n = rot(cam, r2);
    double s1 = se.x, s2 = se.y, sig = po.w;
    bool fvalid = true;
    if (cfg.mip) {   // object_space_filter_2d with r = 0.3 (filters.py:84-109, geometry.py:305-319)
        double z = q.z;
        d3 m1 = scl(a1, s1), m2 = scl(a2, s2);
        double J00 = cam.fx * (m1.x * z - q.x * m1.z) / (z * z);
        double J01 = cam.fx * (m2.x * z - q.x * m2.z) / (z * z);
        double J10 = cam.fy * (m1.y * z - q.y * m1.z) / (z * z);
        double J11 = cam.fy * (m2.y * z - q.y * m2.z) / (z * z);
        double det = J00 * J11 - J01 * J10;
        fvalid = fabs(det) > 1e-12 && z > NEAR;
        double dets = fvalid ? det : 1.0;
        double i00 = J11 / dets, i01 = -J01 / dets, i10 = -J10 / dets, i11 = J00 / dets;
        double sm0 = sqrt(1.0 + SCREEN_VAR * (i00 * i00 + i01 * i01));
        double sm1 = sqrt(1.0 + SCREEN_VAR * (i10 * i10 + i11 * i11));
        s1 *= sm0; s2 *= sm1;
        sig *= 1.0 / (sm0 * sm1);
    }
    double m2max = 2.0 * log(fmax(255.0 * sig, 1e-12));
    bool valid = valid_thread && fvalid && q.z > NEAR && m2max > 0.0;
    double rmax = sqrt(fmax(m2max, 0.0));
    int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
    if (valid) valid = disc_ranges(q, scl(a1, s1 * rmax), scl(a2, s2 * rmax), cam, x0, x1, y0, y1);
    // slab key: nearest depth of the alpha support minus eps (gate t < D_s + eps)
    const float epsf = cfg.eps_const ? cfg.eps_value : se.w;
    double zsup = q.z - rmax * sqrt(s1 * s1 * a1.z * a1.z + s2 * s2 * a2.z * a2.z);
    zsup -= 1e-5 * fabs(zsup) + 1e-6;
    const float gkey = (float)zsup - epsf;
    const float3 col = gauss_view_colour<DEG>(sc, cam, p, shsm);
    count_tiles(o.bin_count, g, valid, x0, x1, y0, y1, gkey);
    if (!valid_thread) return;
    Gauss2Rec rec;
    if (valid) {
        planar_coeffs(q, a1, a2, n, s1, s2, cam, x0, x1, y0, y1, rec.r0, rec.r1, rec.r2);
        o.cull[i] = make_float4(gkey, epsf, __uint_as_float(pack_span(x0, x1)), __uint_as_float(pack_span(y0, y1)));
        rec.r3 = make_float4((float)sig, (float)m2max * 1.0001f + 1e-4f, 0.f, 0.f);
        rec.r4 = make_float4(col.x, col.y, col.z, 0.f);
        if (o.aux) {   // k1 = a1.d/s1, k2 = a2.d/s2 of ray_splat_backward (geometry.py:229-252)
            const int xr = (int)rec.r1.w, yr = (int)rec.r2.w;
            o.aux[2 * i] = affine_of(scl(a1, 1.0 / s1), cam, xr, yr, 0.f);
            o.aux[2 * i + 1] = affine_of(scl(a2, 1.0 / s2), cam, xr, yr, 0.f);
        }
        if (cfg.geom) {
            double sgn = dot(n, q) < 0.0 ? 1.0 : -1.0;   // forward.py:337
            o.nrm[i] = make_float4((float)(n.x * sgn), (float)(n.y * sgn), (float)(n.z * sgn), 0.f);
        }
        reinterpret_cast<Gauss2Rec*>(o.rec)[i] = rec;
    } else {   // empty pixel range: never binned, the record is never read
        o.cull[i] = make_float4(0.f, 0.f, __uint_as_float(pack_span(1, 0)), __uint_as_float(pack_span(1, 0)));
    }
}

cudaError_t launch_gauss_prep(const ges_scene_t& sc, const CamK& cam, const Grid& g,
                              const ges_settings_t& st, const PrepOut& o, cudaStream_t s) {
    if (sc.n_gaussians == 0) return cudaSuccess;
    GaussCfg cfg{st.mip, st.epsilon_mode == 1, st.with_geometry, (float)st.epsilon_value};
    unsigned nb = (unsigned)((sc.n_gaussians + GPREP_T - 1) / GPREP_T);
#define GES_G(KER)                                                              \
    switch (sc.sh_degree) {                                                     \
        case 0: KER<0><<<nb, GPREP_T, 0, s>>>(sc, cam, g, cfg, o); break;      \
        case 1: KER<1><<<nb, GPREP_T, 0, s>>>(sc, cam, g, cfg, o); break;      \
        case 2: KER<2><<<nb, GPREP_T, 0, s>>>(sc, cam, g, cfg, o); break;      \
        default: KER<3><<<nb, GPREP_T, 0, s>>>(sc, cam, g, cfg, o); break;     \
    }
    if (sc.gaussian_dim == 2) {
        GES_G(k_gauss2_prep)
    } else {
        GES_G(k_gauss3_prep)
    }
#undef GES_G
    return cudaGetLastError();
}

}  // namespace ges
