// Training step kernels (reference training.py, joint stage with frozen
// surfel geometry):
//   k_surfel_colors      view colour of every surfel (training.py:100-109)
//   k_gauss_bwd<GK,GEOM> per-tile replay of the Gaussian pass, pushing the
//                        pixel cotangents dL/dC_G, dL/dW_G (, dL/dD_G, dL/dN_G)
//                        to per-Gaussian partial sums (training.py:646-690,
//                        :722-768 up to the bincounts)
//   k_gauss3_finish /    per-Gaussian float64 chain rule from those sums to
//   k_gauss2_finish      the exposed parameters (conic -> covariance -> EWA
//                        projection, ray-plane frame, SH, world filter,
//                        geometry.py:135-190, :229-270, training.py:123-138,
//                        :632-643, :890-911)
//   k_frozen_scatter +   _surfel_backward_frozen (training.py:612-629)
//   k_surfel_sh_bwd
//
// The replay uses exactly the forward's screen records and arithmetic (same
// prep kernels, same tile binning, same alpha/gate tests), so the set of
// contributing (pixel, Gaussian) fragments is the forward's.  Each warp owns
// an 8x4 pixel patch of a 16x16 tile, walks the tile's near-to-far Gaussian
// list, culls whole entries against its patch, and for every surviving
// Gaussian reduces the lanes' per-pixel terms with shuffles: one float64
// atomic per (warp, Gaussian, term).
#include <math.h>

#include "ges_launch.h"
#include "ges_sh.cuh"

namespace ges {

namespace {

constexpr int NACC = 16;   // accumulators per Gaussian (3D uses 10)

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------------------ SH in float64
template <int DEG>
__device__ void sh_basis_d(double x, double y, double z, double* b) {
    b[0] = 0.28209479177387814;
    if (DEG >= 1) {
        const double C1 = 0.4886025119029199;
        b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
    }
    if (DEG >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[4] = 1.0925484305920792 * x * y;
        b[5] = -1.0925484305920792 * y * z;
        b[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
        b[7] = -1.0925484305920792 * x * z;
        b[8] = 0.5462742152960396 * (xx - yy);
        if (DEG >= 3) {
            b[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
            b[10] = 2.890611442640554 * x * y * z;
            b[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
            b[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            b[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
            b[14] = 1.445305721320277 * z * (xx - yy);
            b[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
        }
    }
}

// g_dir += sum_k gb[k] * d basis_k / d dir   (sh.py:67-112 contracted with gb)
template <int DEG>
__device__ void sh_basis_vjp(double x, double y, double z, const double* gb, double* gd) {
    gd[0] = gd[1] = gd[2] = 0.0;
    if (DEG >= 1) {
        const double C1 = 0.4886025119029199;
        gd[1] += -C1 * gb[1]; gd[2] += C1 * gb[2]; gd[0] += -C1 * gb[3];
    }
    if (DEG >= 2) {
        const double A = 1.0925484305920792, B = -1.0925484305920792, Cc = 0.31539156525252005,
                     D = -1.0925484305920792, E = 0.5462742152960396;
        gd[0] += gb[4] * A * y; gd[1] += gb[4] * A * x;
        gd[1] += gb[5] * B * z; gd[2] += gb[5] * B * y;
        gd[0] += gb[6] * Cc * (-2.0 * x); gd[1] += gb[6] * Cc * (-2.0 * y); gd[2] += gb[6] * Cc * (4.0 * z);
        gd[0] += gb[7] * D * z; gd[2] += gb[7] * D * x;
        gd[0] += gb[8] * E * (2.0 * x); gd[1] += gb[8] * E * (-2.0 * y);
    }
    if (DEG >= 3) {
        const double c0 = -0.5900435899266435, c1 = 2.890611442640554, c2 = -0.4570457994644658,
                     c3 = 0.3731763325901154, c4 = -0.4570457994644658, c5 = 1.445305721320277,
                     c6 = -0.5900435899266435;
        const double xx = x * x, yy = y * y, zz = z * z;
        gd[0] += gb[9] * c0 * 6.0 * x * y; gd[1] += gb[9] * c0 * (3.0 * xx - 3.0 * yy);
        gd[0] += gb[10] * c1 * y * z; gd[1] += gb[10] * c1 * x * z; gd[2] += gb[10] * c1 * x * y;
        gd[0] += gb[11] * c2 * (-2.0 * x * y); gd[1] += gb[11] * c2 * (4.0 * zz - xx - 3.0 * yy);
        gd[2] += gb[11] * c2 * (8.0 * y * z);
        gd[0] += gb[12] * c3 * (-6.0 * x * z); gd[1] += gb[12] * c3 * (-6.0 * y * z);
        gd[2] += gb[12] * c3 * (6.0 * zz - 3.0 * xx - 3.0 * yy);
        gd[0] += gb[13] * c4 * (4.0 * zz - 3.0 * xx - yy); gd[1] += gb[13] * c4 * (-2.0 * x * y);
        gd[2] += gb[13] * c4 * (8.0 * x * z);
        gd[0] += gb[14] * c5 * (2.0 * x * z); gd[1] += gb[14] * c5 * (-2.0 * y * z);
        gd[2] += gb[14] * c5 * (xx - yy);
        gd[0] += gb[15] * c6 * (3.0 * xx - 3.0 * yy); gd[1] += gb[15] * c6 * (-6.0 * x * y);
    }
}

// _sh_backward (training.py:123-138) for one primitive: g_sh (K x 3) and the
// positional gradient through the view direction dir = (cam - p)/|cam - p|.
template <int DEG>
__device__ void sh_backward(const double* sh, const double* p, const double* cpos, const double* g_col,
                            double* g_sh, double* g_pos) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    double d[3] = {cpos[0] - p[0], cpos[1] - p[1], cpos[2] - p[2]};
    const double dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    d[0] /= dist; d[1] /= dist; d[2] /= dist;
    double b[K];
    sh_basis_d<DEG>(d[0], d[1], d[2], b);
    double gc[3];
    for (int c = 0; c < 3; ++c) {
        double raw = 0.5;
        for (int k = 0; k < K; ++k) raw += b[k] * sh[3 * k + c];
        gc[c] = (raw > 0.0 && raw < 1.0) ? g_col[c] : 0.0;   // clamp mask
    }
    double gb[K];
    for (int k = 0; k < K; ++k) {
        gb[k] = 0.0;
        for (int c = 0; c < 3; ++c) {
            g_sh[3 * k + c] = b[k] * gc[c];
            gb[k] += sh[3 * k + c] * gc[c];
        }
    }
    double gd[3];
    sh_basis_vjp<DEG>(d[0], d[1], d[2], gb, gd);
    const double dd = gd[0] * d[0] + gd[1] * d[1] + gd[2] * d[2];
    for (int j = 0; j < 3; ++j) g_pos[j] = -(gd[j] - dd * d[j]) / dist;
}

// Rotation of a unit quaternion (geometry.py:23-36) and the contraction of
// dR/dq (geometry.py:39-65) with a 3x3 cotangent G (row-major).
__device__ void quat_rot(const double* q, double* R) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}
__device__ void quat_rot_vjp(const double* q, const double* G, double* gq) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    gq[0] = -2 * z * G[1] + 2 * y * G[2] + 2 * z * G[3] - 2 * x * G[5] - 2 * y * G[6] + 2 * x * G[7];
    gq[1] = 2 * y * G[1] + 2 * z * G[2] + 2 * y * G[3] - 4 * x * G[4] - 2 * w * G[5] + 2 * z * G[6] +
            2 * w * G[7] - 4 * x * G[8];
    gq[2] = -4 * y * G[0] + 2 * x * G[1] + 2 * w * G[2] + 2 * x * G[3] + 2 * z * G[5] - 2 * w * G[6] +
            2 * z * G[7] - 4 * y * G[8];
    gq[3] = -4 * z * G[0] - 2 * w * G[1] + 2 * x * G[2] + 2 * w * G[3] - 4 * z * G[4] + 2 * y * G[5] +
            2 * x * G[6] + 2 * y * G[7];
}

// Per-Gaussian source parameters (float64, source order) and the exposed /
// effective quantities of primitives.py:101-131.
struct GSrc {
    double p[3], qn[4], s[3], s_eff[3], sig, sig_eff;
};
__device__ void load_gsrc(const ges_scene_src_t& src, int64_t o, int any_filter, GSrc& g) {
    const int D = src.gaussian_dim;
    for (int j = 0; j < 3; ++j) g.p[j] = src.g_pos[3 * o + j];
    double qq[4], n2 = 0.0;
    for (int j = 0; j < 4; ++j) { qq[j] = src.g_quat[4 * o + j]; n2 += qq[j] * qq[j]; }
    const double qnrm = sqrt(n2);
    for (int j = 0; j < 4; ++j) g.qn[j] = qq[j] / qnrm;
    const double f3 = (any_filter && src.g_filter3d) ? src.g_filter3d[o] : 0.0;
    g.sig = 1.0 / (1.0 + exp(-src.g_raw_opacity[o]));
    g.sig_eff = g.sig;
    for (int k = 0; k < 3; ++k) { g.s[k] = 0.0; g.s_eff[k] = 0.0; }
    for (int k = 0; k < D; ++k) {
        g.s[k] = exp(src.g_log_scale[D * o + k]);
        if (any_filter) {
            g.s_eff[k] = sqrt(g.s[k] * g.s[k] + f3);
            g.sig_eff *= g.s[k] / g.s_eff[k];
        } else {
            g.s_eff[k] = g.s[k];
        }
    }
}

// _chain_effective (training.py:632-643), screen statistic (:896-911) and the
// tangent projection of the quaternion gradient (:890-893); writes one
// Gaussian's gradients.
__device__ void write_gauss_grads(const ges_gauss_grads_t& out, int64_t o, int D, int K, int any_filter,
                                  const GSrc& g, const CamK& cam, const double* g_pos, const double* g_qu,
                                  const double* g_s_eff, double g_sig_eff, const double* g_sh) {
    double g_scale[3], g_sig = g_sig_eff;
    for (int k = 0; k < D; ++k) g_scale[k] = g_s_eff[k];
    if (any_filter) {
        for (int k = 0; k < D; ++k)
            g_scale[k] = g_s_eff[k] * (g.s[k] / g.s_eff[k]) +
                         g_sig_eff * g.sig_eff * (1.0 / g.s[k] - g.s[k] / (g.s_eff[k] * g.s_eff[k]));
        g_sig = g_sig_eff * (g.sig_eff / g.sig);
    }
    double dq = 0.0;
    for (int j = 0; j < 4; ++j) dq += g.qn[j] * g_qu[j];
    for (int j = 0; j < 3; ++j) out.pos[3 * o + j] = g_pos[j];
    for (int j = 0; j < 4; ++j) out.quat[4 * o + j] = g_qu[j] - dq * g.qn[j];
    for (int k = 0; k < D; ++k) out.scale[D * o + k] = g_scale[k];
    out.opacity[o] = g_sig;
    for (int j = 0; j < K * 3; ++j) out.sh[(int64_t)K * 3 * o + j] = g_sh[j];
    if (out.screen) {
        const double* R = cam.R;
        const double z = fmax(R[6] * g.p[0] + R[7] * g.p[1] + R[8] * g.p[2] + cam.t[2], NEAR);
        const double gx = R[0] * g_pos[0] + R[1] * g_pos[1] + R[2] * g_pos[2];
        const double gy = R[3] * g_pos[0] + R[4] * g_pos[1] + R[5] * g_pos[2];
        out.screen[o] = hypot(gx * z / cam.fx * (cam.W / 2.0), gy * z / cam.fy * (cam.H / 2.0));
    }
}

}  // namespace

// ---------------------------------------------------------------- colours
template <int DEG>
__global__ void k_surfel_colors(ges_scene_t sc, CamK cam, float* rgb) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= sc.n_surfels) return;
    const float4 p = reinterpret_cast<const float4*>(sc.s_pos_s1)[i];
    double d[3] = {cam.pos[0] - p.x, cam.pos[1] - p.y, cam.pos[2] - p.z};
    const double inv = 1.0 / fmax(sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]), 1e-12);
    const float3 c = sh_color<DEG>(sc.s_sh + i * (DEG + 1) * (DEG + 1) * 3, (float)(d[0] * inv),
                                   (float)(d[1] * inv), (float)(d[2] * inv));
    const int64_t o = sc.s_id[i];
    rgb[3 * o] = c.x; rgb[3 * o + 1] = c.y; rgb[3 * o + 2] = c.z;
}

// ---------------------------------------------------------------- tile replay
// CONTRIB: instead of gradients, the per-Gaussian max over its fragments of
// max_c(colour) * alpha / (1 + W_G) (optim.py:526-533; g_wg = W_G then),
// atomically max-ed into a.scores[source id].
template <int GK, bool GEOM, bool CONTRIB = false>
__global__ void __launch_bounds__(256) k_gauss_bwd(BwdArgs a) {
    __shared__ uint32_t gslab_end[NSLAB];
    if (a.status->overflow) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx = blockIdx.x, ty = blockIdx.y, tile = ty * a.ntx + tx;
    const int plx = (warp & 1) * 8 + (lane & 7), ply = (warp >> 1) * 4 + (lane >> 3);
    const int X = tx * TILE + plx, Y = ty * TILE + ply;
    const bool inside = X < a.W && Y < a.H;
    const int64_t pix = (int64_t)Y * a.W + X;
    float ds = INFINITY, gcr = 0.f, gcg = 0.f, gcb = 0.f, gw = 0.f, gd = 0.f, gnx = 0.f, gny = 0.f, gnz = 0.f;
    if (inside) {
        ds = a.ds[pix];
        if (!CONTRIB) { gcr = a.g_cg[3 * pix]; gcg = a.g_cg[3 * pix + 1]; gcb = a.g_cg[3 * pix + 2]; }
        gw = a.g_wg[pix];
        if (a.g_gd) gd = a.g_gd[pix];
        if (a.g_gn) { gnx = a.g_gn[3 * pix]; gny = a.g_gn[3 * pix + 1]; gnz = a.g_gn[3 * pix + 2]; }
    }
    const float cden = CONTRIB ? 1.0f / (1.0f + gw) : 0.f;   // gw = W_G in CONTRIB mode
    if (threadIdx.x < NSLAB) gslab_end[threadIdx.x] = a.gbin.cnt[tile * NSLAB + threadIdx.x];
    const uint32_t gbeg = a.gbin.tile_off(tile), gend = gbeg + a.gbin.cnt[tile * NSLAB + NSLAB - 1];
    __syncthreads();
    const float wdmax = warp_maxf(inside ? ds : -INFINITY);
    float pe = 0.f;
    if (GK == 2) {
        const float dxn = ((float)X + 0.5f - a.gcx) * a.gifx, dyn = ((float)Y + 0.5f - a.gcy) * a.gify;
        pe = PARALLEL_EPS_F * sqrtf(dxn * dxn + dyn * dyn + 1.0f);
    }
    const int ox = tx * TILE, oy = ty * TILE;
    const int px0 = (warp & 1) * 8, py0 = (warp >> 1) * 4;
    const float lx = (float)plx, ly = (float)ply;
    for (uint32_t base = gbeg; base < gend; base += 32) {
        {   // near-to-far slabs: stop once the rest fail every gate of the patch
            if (a.slabs.lower(slab_of_pos(gslab_end, base - gbeg, lane)) > wdmax) break;
        }
        const uint32_t e = base + lane;
        bool live = false;
        uint32_t id = 0;
        if (e < gend) {
            id = a.g_list[e];
            const float4 c = __ldg(a.gcull + id);
            const uint32_t sxr = __float_as_uint(c.z), syr = __float_as_uint(c.w);
            live = span_lo(sxr) - ox <= px0 + 7 && span_hi(sxr) - ox >= px0 && span_lo(syr) - oy <= py0 + 3 &&
                   span_hi(syr) - oy >= py0 && (GK == 3 ? c.x < wdmax + c.y : !(c.x > wdmax));
        }
        uint32_t vote = __ballot_sync(0xffffffffu, live);
        while (vote) {
            const int j = __ffs(vote) - 1;
            vote &= vote - 1;
            const uint32_t gid = __shfl_sync(0xffffffffu, id, j);
            float v[NACC];
#pragma unroll
            for (int k = 0; k < NACC; ++k) v[k] = 0.f;
            bool contrib = false;
            if constexpr (GK == 3) {
                const GaussRec* r = reinterpret_cast<const GaussRec*>(a.grec) + gid;
                const float4 c = a.gcull[gid], r0 = r->r0, r1 = r->r1, r2 = r->r2;
                const float mx = (r0.x - (float)ox) + (r0.y - 0.5f), my = (r0.z - (float)oy) + (r0.w - 0.5f);
                // identical to the forward tile kernel (forward.py:301-311)
                const float dx = lx - mx, dy = ly - my;
                const float pw = fmaf(r1.x * dx, dx, fmaf(r1.z * dy, dy, r1.y * dx * dy));   // log2(e) * power
                if (inside) {
                    const float al = r1.w * ex2_ftz(pw);
                    if (al >= ALPHA_CUTOFF_F && c.x < ds + c.y) {
                        contrib = true;
                        if constexpr (CONTRIB) {
                            v[0] = fmaxf(r2.y, fmaxf(r2.z, r2.w)) * al * cden;
                        } else {
                        // training.py:652-690: g_alpha, then alpha = amp exp(power)
                        float ga = fmaf(r2.y, gcr, fmaf(r2.z, gcg, fmaf(r2.w, gcb, gw)));
                        ga = fmaf(c.x, gd, ga);
                        if (GEOM) {
                            const float4 nv = __ldg(a.g_nrm + gid);
                            ga = fmaf(nv.x, gnx, fmaf(nv.y, gny, fmaf(nv.z, gnz, ga)));
                        }
                        const float gp = ga * al;
                        const float la = -2.f * LN2_F * r1.x, lb = -LN2_F * r1.y, lc = -2.f * LN2_F * r1.z;
                        v[0] = gp;
                        v[1] = gp * fmaf(la, dx, lb * dy);
                        v[2] = gp * fmaf(lb, dx, lc * dy);
                        v[3] = -0.5f * gp * dx * dx;
                        v[4] = -gp * dx * dy;
                        v[5] = -0.5f * gp * dy * dy;
                        v[6] = al * gcr; v[7] = al * gcg; v[8] = al * gcb;
                        v[9] = al * gd;
                        }
                    }
                }
            } else {
                const Gauss2Rec* r = reinterpret_cast<const Gauss2Rec*>(a.grec) + gid;
                const float4 c = a.gcull[gid], r0 = r->r0, r1 = r->r1, r2 = r->r2, r3 = r->r3, r4 = r->r4;
                const float4 k1c = CONTRIB ? float4{} : a.aux[2 * (size_t)gid];
                const float4 k2c = CONTRIB ? float4{} : a.aux[2 * (size_t)gid + 1];
                const float fx = (float)(ox - (int)r1.w), fy = (float)(oy - (int)r2.w);
                const float d0 = fmaf(r0.z, fy, fmaf(r0.y, fx, r0.x));
                const float u0 = fmaf(r1.z, fy, fmaf(r1.y, fx, r1.x));
                const float v0 = fmaf(r2.z, fy, fmaf(r2.y, fx, r2.x));
                // identical to the forward tile kernel (forward.py:361-379)
                const float den = fmaf(r0.z, ly, fmaf(r0.y, lx, d0));
                const float U = fmaf(r1.z, ly, fmaf(r1.y, lx, u0));
                const float V = fmaf(r2.z, ly, fmaf(r2.y, lx, v0));
                const float r2u = fmaf(U, U, V * V);
                if (inside && r2u <= r3.y * den * den && fabsf(den) > pe) {
                    const float inv = rcp_ftz(den);   // |den| > 1e-8|d|
                    const float t = r0.w * inv;
                    const float q2 = r2u * inv * inv;
                    const float G = ex2_ftz(q2 * (-0.5f * LOG2E_F));
                    const float al = r3.x * G;
                    if (t > NEAR_F && al >= ALPHA_CUTOFF_F && t < ds + c.y) {
                        contrib = true;
                        if constexpr (CONTRIB) {
                            v[0] = fmaxf(r4.x, fmaxf(r4.y, r4.z)) * al * cden;
                        } else {
                        // training.py:731-754: g_alpha, g_sigma', g_G, g_u, g_v, g_t
                        float ga = fmaf(r4.x, gcr, fmaf(r4.y, gcg, fmaf(r4.z, gcb, gw)));
                        ga = fmaf(t, gd, ga);
                        float n0 = 0.f, n1 = 0.f, n2 = 0.f;
                        if (GEOM) {
                            const float4 nv = __ldg(a.g_nrm + gid);
                            n0 = nv.x; n1 = nv.y; n2 = nv.z;
                            ga = fmaf(n0, gnx, fmaf(n1, gny, fmaf(n2, gnz, ga)));
                        }
                        const float u = U * inv, vv = V * inv;
                        const float gG = ga * r3.x;
                        const float gu = -u * G * gG, gv = -vv * G * gG;
                        // ray_splat_backward (geometry.py:229-252) reduced to in-plane
                        // coordinates: h = s1 u a1 + s2 v a2 (see the finish kernel)
                        const float k1 = fmaf(k1c.z, ly, fmaf(k1c.y, lx, fmaf(k1c.z, fy, fmaf(k1c.y, fx, k1c.x))));
                        const float k2 = fmaf(k2c.z, ly, fmaf(k2c.y, lx, fmaf(k2c.z, fy, fmaf(k2c.y, fx, k2c.x))));
                        const float gst = fmaf(gu, k1, fmaf(gv, k2, al * gd));
                        const float w = gst * inv;
                        v[0] = w; v[1] = gu; v[2] = gv;
                        v[3] = w * u; v[4] = w * vv;
                        v[5] = gu * u; v[6] = gu * vv; v[7] = gv * u; v[8] = gv * vv;
                        v[9] = ga * G;
                        v[10] = al * gcr; v[11] = al * gcg; v[12] = al * gcb;
                        v[13] = al * gnx; v[14] = al * gny; v[15] = al * gnz;
                        }
                    }
                }
            }
            if (!__any_sync(0xffffffffu, contrib)) continue;
            if constexpr (CONTRIB) {
                const float m = warp_maxf(v[0]);
                if (lane == 0 && m > 0.f)
                    atomicMax(reinterpret_cast<unsigned int*>(a.scores) + (a.order ? a.order[gid] : (int32_t)gid),
                              __float_as_uint(m));   // non-negative floats order like their bits
                continue;
            }
            constexpr int NV = GK == 3 ? 10 : NACC;
            float mine = 0.f;
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const float s = warp_sum(v[k]);
                if (lane == k) mine = s;
            }
            if (lane < NV && mine != 0.f) atomicAdd(a.acc + (size_t)gid * NACC + lane, (double)mine);
        }
    }
}

// ---------------------------------------------------------------- finish 3D
// training.py:692-719 + project_gaussian_backward (geometry.py:135-190).
template <int DEG>
__global__ void k_gauss3_finish(ges_scene_src_t src, int any_filter, int mip, CamK cam, const double* __restrict__ acc,
                                ges_gauss_grads_t out) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= src.n_gaussians) return;
    const int64_t o = src.g_order ? src.g_order[i] : i;
    double A[10];
    bool any = false;
    for (int k = 0; k < 10; ++k) { A[k] = acc[i * NACC + k]; any |= A[k] != 0.0; }
    if (!any) return;   // no fragments: the (zero-initialised) outputs stay zero
    GSrc g;
    load_gsrc(src, o, any_filter, g);
    const double* W = cam.R;
    double t[3];
    for (int r = 0; r < 3; ++r) t[r] = W[3 * r] * g.p[0] + W[3 * r + 1] * g.p[1] + W[3 * r + 2] * g.p[2] + cam.t[r];
    const double x = t[0], y = t[1], z = t[2], fx = cam.fx, fy = cam.fy;
    const double iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    const double J[6] = {fx * iz, 0.0, -fx * x * iz2, 0.0, fy * iz, -fy * y * iz2};
    double R[9];
    quat_rot(g.qn, R);
    // Vw = R diag(s^2) R^T, M = W Vw W^T
    double Vw[9], M[9], T[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += R[3 * r + k] * g.s_eff[k] * g.s_eff[k] * R[3 * c + k];
            Vw[3 * r + c] = acc_;
        }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += W[3 * r + k] * Vw[3 * k + c];
            T[3 * r + c] = acc_;
        }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += T[3 * r + k] * W[3 * c + k];
            M[3 * r + c] = acc_;
        }
    // cov2d = J M J^T (+0.3 I), conic, mip compensation (training.py:401-418)
    double JM[6];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += J[3 * r + k] * M[3 * k + c];
            JM[3 * r + c] = acc_;
        }
    double cr[4];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += JM[3 * r + k] * J[3 * c + k];
            cr[2 * r + c] = acc_;
        }
    const double c00 = cr[0] + SCREEN_VAR, c11 = cr[3] + SCREEN_VAR, c01 = cr[1];
    const double det = c00 * c11 - c01 * c01;
    const double raw_det = cr[0] * cr[3] - cr[1] * cr[1];
    const double kcomp = mip ? sqrt(fmax(raw_det, 1e-300) / det) : 1.0;
    const double amp = g.sig_eff * kcomp;
    const double la = c11 / det, lb = -c01 / det, lc = c00 / det;
    // conic -> covariance: dL/dSigma' = -L gL L (training.py:692-701)
    const double gL[4] = {A[3], 0.5 * A[4], 0.5 * A[4], A[5]};
    const double L[4] = {la, lb, lb, lc};
    double LgL[4], gcov[4];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) LgL[2 * r + c] = L[2 * r] * gL[c] + L[2 * r + 1] * gL[2 + c];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) gcov[2 * r + c] = -(LgL[2 * r] * L[c] + LgL[2 * r + 1] * L[2 + c]);
    const double G_amp = A[0] / amp;
    const double g_sig_eff = G_amp * kcomp;
    if (mip) {   // training.py:704-711
        const double g_k = G_amp * g.sig_eff;
        const double r00 = cr[0] + 1e-12, r11 = cr[3] + 1e-12, r01 = cr[1];
        const double rd = r00 * r11 - r01 * r01;
        const double ir[4] = {r11 / rd, -r01 / rd, -r01 / rd, r00 / rd};
        const double jf[4] = {c11 / det, -c01 / det, -c01 / det, c00 / det};
        for (int k = 0; k < 4; ++k) gcov[k] += 0.5 * kcomp * g_k * (ir[k] - jf[k]);
    }
    // project_gaussian_backward: g_M = J^T gcov J, g_J = 2 gcov J M
    double gM[9], gJ[6], GJ[6];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) GJ[3 * r + c] = gcov[2 * r] * J[c] + gcov[2 * r + 1] * J[3 + c];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) gM[3 * r + c] = J[r] * GJ[c] + J[3 + r] * GJ[3 + c];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += GJ[3 * r + k] * M[3 * k + c];
            gJ[3 * r + c] = 2.0 * acc_;
        }
    double gt[3];
    gt[0] = gJ[2] * (-fx * iz2);
    gt[1] = gJ[5] * (-fy * iz2);
    gt[2] = gJ[0] * (-fx * iz2) + gJ[2] * (2.0 * fx * x * iz3) + gJ[4] * (-fy * iz2) + gJ[5] * (2.0 * fy * y * iz3);
    gt[0] += A[1] * fx * iz;
    gt[1] += A[2] * fy * iz;
    gt[2] += (-fx * x * iz2) * A[1] + (-fy * y * iz2) * A[2];
    gt[2] += A[9];
    double g_pos[3];
    for (int c = 0; c < 3; ++c) g_pos[c] = W[c] * gt[0] + W[3 + c] * gt[1] + W[6 + c] * gt[2];
    // g_Vw = W^T g_M W, symmetrised
    double gV[9], U_[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += W[3 * k + r] * gM[3 * k + c];
            U_[3 * r + c] = acc_;
        }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += U_[3 * r + k] * W[3 * k + c];
            gV[3 * r + c] = acc_;
        }
    for (int r = 0; r < 3; ++r)
        for (int c = r + 1; c < 3; ++c) {
            const double m = 0.5 * (gV[3 * r + c] + gV[3 * c + r]);
            gV[3 * r + c] = gV[3 * c + r] = m;
        }
    // GR = 2 gVw R; g_s_k = s_k (GR[:,k] . R[:,k]); g_R = GR diag(s^2)
    double GR[9], gR[9], g_s[3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc_ = 0.0;
            for (int k = 0; k < 3; ++k) acc_ += gV[3 * r + k] * R[3 * k + c];
            GR[3 * r + c] = 2.0 * acc_;
        }
    for (int k = 0; k < 3; ++k) {
        double d = 0.0;
        for (int r = 0; r < 3; ++r) d += GR[3 * r + k] * R[3 * r + k];
        g_s[k] = g.s_eff[k] * d;
        for (int r = 0; r < 3; ++r) gR[3 * r + k] = GR[3 * r + k] * g.s_eff[k] * g.s_eff[k];
    }
    double g_qu[4];
    quat_rot_vjp(g.qn, gR, g_qu);
    // SH (training.py:713-714)
    const double gcol[3] = {A[6], A[7], A[8]};
    double shs[K * 3], g_sh[K * 3], g_psh[3];
    for (int j = 0; j < K * 3; ++j) shs[j] = src.g_sh[(int64_t)K * 3 * o + j];
    sh_backward<DEG>(shs, g.p, cam.pos, gcol, g_sh, g_psh);
    for (int j = 0; j < 3; ++j) g_pos[j] += g_psh[j];
    write_gauss_grads(out, o, 3, K, any_filter, g, cam, g_pos, g_qu, g_s, g_sig_eff, g_sh);
}

// ---------------------------------------------------------------- finish 2D
// training.py:756-788 with the fragment sums reduced in plane coordinates:
// per fragment h = t d - q = s1 u a1 + s2 v a2 (n.h = 0, orthonormal frame),
// so with w = g_t_total / (n.d):
//   G_q  = n sum(w) - a1 sum(gu)/s1 - a2 sum(gv)/s2
//   G_n  = -(a1 s1 sum(w u) + a2 s2 sum(w v))        (+ sign * sum(alpha dL/dN_G))
//   G_a1 = a1 sum(gu u) + a2 (s2/s1) sum(gu v)
//   G_a2 = a1 (s1/s2) sum(gv u) + a2 sum(gv v)
//   g_s1 = -sum(gu u)/s1, g_s2 = -sum(gv v)/s2
template <int DEG>
__global__ void k_gauss2_finish(ges_scene_src_t src, int any_filter, int mip, CamK cam, const double* __restrict__ acc,
                                ges_gauss_grads_t out) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= src.n_gaussians) return;
    const int64_t o = src.g_order ? src.g_order[i] : i;
    double B[NACC];
    bool any = false;
    for (int k = 0; k < NACC; ++k) { B[k] = acc[i * NACC + k]; any |= B[k] != 0.0; }
    if (!any) return;   // no fragments: the (zero-initialised) outputs stay zero
    GSrc g;
    load_gsrc(src, o, any_filter, g);
    const double* W = cam.R;
    double R[9];
    quat_rot(g.qn, R);
    double q[3], a1[3], a2[3], n[3];
    for (int r = 0; r < 3; ++r) {
        q[r] = W[3 * r] * g.p[0] + W[3 * r + 1] * g.p[1] + W[3 * r + 2] * g.p[2] + cam.t[r];
        a1[r] = W[3 * r] * R[0] + W[3 * r + 1] * R[3] + W[3 * r + 2] * R[6];
        a2[r] = W[3 * r] * R[1] + W[3 * r + 1] * R[4] + W[3 * r + 2] * R[7];
        n[r] = W[3 * r] * R[2] + W[3 * r + 1] * R[5] + W[3 * r + 2] * R[8];
    }
    double smul0 = 1.0, smul1 = 1.0, omul = 1.0;
    if (mip) {   // object_space_filter_2d, filters.py:84-109 (as the forward prep)
        const double zz = q[2];
        const double m1[3] = {a1[0] * g.s_eff[0], a1[1] * g.s_eff[0], a1[2] * g.s_eff[0]};
        const double m2[3] = {a2[0] * g.s_eff[1], a2[1] * g.s_eff[1], a2[2] * g.s_eff[1]};
        const double J00 = cam.fx * (m1[0] * zz - q[0] * m1[2]) / (zz * zz);
        const double J01 = cam.fx * (m2[0] * zz - q[0] * m2[2]) / (zz * zz);
        const double J10 = cam.fy * (m1[1] * zz - q[1] * m1[2]) / (zz * zz);
        const double J11 = cam.fy * (m2[1] * zz - q[1] * m2[2]) / (zz * zz);
        const double det = J00 * J11 - J01 * J10;
        const double dets = (fabs(det) > 1e-12 && zz > NEAR) ? det : 1.0;
        const double i00 = J11 / dets, i01 = -J01 / dets, i10 = -J10 / dets, i11 = J00 / dets;
        smul0 = sqrt(1.0 + SCREEN_VAR * (i00 * i00 + i01 * i01));
        smul1 = sqrt(1.0 + SCREEN_VAR * (i10 * i10 + i11 * i11));
        omul = 1.0 / (smul0 * smul1);
    }
    const double s1 = g.s_eff[0] * smul0, s2 = g.s_eff[1] * smul1;
    const double sign = (n[0] * q[0] + n[1] * q[1] + n[2] * q[2]) < 0.0 ? 1.0 : -1.0;
    double Gq[3], Gn[3], Ga1[3], Ga2[3];
    for (int r = 0; r < 3; ++r) {
        Gq[r] = n[r] * B[0] - a1[r] * B[1] / s1 - a2[r] * B[2] / s2;
        Gn[r] = -(a1[r] * s1 * B[3] + a2[r] * s2 * B[4]) + sign * B[13 + r];
        Ga1[r] = a1[r] * B[5] + a2[r] * (s2 / s1) * B[6];
        Ga2[r] = a1[r] * (s1 / s2) * B[7] + a2[r] * B[8];
    }
    // frame_world_grads (geometry.py:255-270): g_pos = W^T G_q, columns W^T G_*
    double g_pos[3], gR[9];
    for (int c = 0; c < 3; ++c) {
        g_pos[c] = W[c] * Gq[0] + W[3 + c] * Gq[1] + W[6 + c] * Gq[2];
        gR[3 * c + 0] = W[c] * Ga1[0] + W[3 + c] * Ga1[1] + W[6 + c] * Ga1[2];
        gR[3 * c + 1] = W[c] * Ga2[0] + W[3 + c] * Ga2[1] + W[6 + c] * Ga2[2];
        gR[3 * c + 2] = W[c] * Gn[0] + W[3 + c] * Gn[1] + W[6 + c] * Gn[2];
    }
    double g_qu[4];
    quat_rot_vjp(g.qn, gR, g_qu);
    const double gcol[3] = {B[10], B[11], B[12]};
    double shs[K * 3], g_sh[K * 3], g_psh[3];
    for (int j = 0; j < K * 3; ++j) shs[j] = src.g_sh[(int64_t)K * 3 * o + j];
    sh_backward<DEG>(shs, g.p, cam.pos, gcol, g_sh, g_psh);
    for (int j = 0; j < 3; ++j) g_pos[j] += g_psh[j];
    const double g_s_eff[3] = {(-B[5] / s1) * smul0, (-B[8] / s2) * smul1, 0.0};
    write_gauss_grads(out, o, 2, K, any_filter, g, cam, g_pos, g_qu, g_s_eff, B[9] * omul, g_sh);
}

// ---------------------------------------------------------------- frozen surfels
// dL/dC_s (base pixel) * 1/grid^2 to every covered sub-sample's winner
// (training.py:617-625).  One thread per BASE pixel: its grid^2 sub-samples
// usually share one winner, and so do neighbouring pixels, so equal
// (winner, value) contributions are first summed per thread, then across the
// warp's lanes with the same single winner (one float64 atomic per group).
__global__ void k_frozen_scatter(const int32_t* __restrict__ winner, const float* __restrict__ g_cs, int W, int H,
                                 int grid, double* col) {
    const int64_t n = (int64_t)W * H;
    const int WW = W * grid;
    const double share = 1.0 / (grid * grid);
    const unsigned lane = threadIdx.x & 31;
    for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < n; b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = b0 + threadIdx.x;
        int32_t w[4] = {-1, -1, -1, -1};
        double g[3] = {0.0, 0.0, 0.0};
        if (b < n) {
            const int64_t X = b % W, Y = b / W;
            for (int k = 0; k < grid * grid; ++k)
                w[k] = winner[(Y * grid + k / grid) * (int64_t)WW + X * grid + k % grid];
            for (int c = 0; c < 3; ++c) g[c] = (double)g_cs[3 * b + c] * share;
        }
        const bool uni = w[0] >= 0 && (grid == 1 || (w[1] == w[0] && w[2] == w[0] && w[3] == w[0]));
        if (!uni) {
            for (int k = 0; k < grid * grid; ++k)
                if (w[k] >= 0)
                    for (int c = 0; c < 3; ++c) atomicAdd(col + 3 * (int64_t)w[k] + c, g[c]);
        }
        // lanes whose sub-samples all share one winner: one group per distinct
        // winner of the warp (usually 1-3), summed with shuffles, one atomic each
        const double m = (double)(grid * grid);
        unsigned todo = __ballot_sync(0xffffffffu, uni);
        while (todo) {
            const int lead = __ffs(todo) - 1;
            const int32_t key = __shfl_sync(0xffffffffu, w[0], lead);
            const bool mine = uni && w[0] == key;
            todo &= ~__ballot_sync(0xffffffffu, mine);
            double t[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                t[c] = mine ? g[c] * m : 0.0;
#pragma unroll
                for (int o = 16; o; o >>= 1) t[c] += __shfl_xor_sync(0xffffffffu, t[c], o);
            }
            if ((int)lane == lead)
                for (int c = 0; c < 3; ++c) atomicAdd(col + 3 * (int64_t)key + c, t[c]);
        }
    }
}

// Forward of the frozen surfel pass on the cached z-buffer
// (training.py:380-392, :334-346): per base pixel the box mean over its
// grid^2 sub-samples of (winner colour or background), the Gaussian gate depth
// = sub-sample (0,0) depth, and with geometry the box means of the covered
// sub-samples' depth and normal (0 where uncovered).
__global__ void k_frozen_resolve(const int32_t* __restrict__ winner, const float* __restrict__ depth,
                                 const float* __restrict__ normal, const float* __restrict__ colors, int W, int H,
                                 int grid, float bg0, float bg1, float bg2, float* s_color, float* s_depth,
                                 float* b_depth, float* b_normal) {
    const int64_t n = (int64_t)W * H;
    const int WW = W * grid;
    const float inv = 1.0f / (float)(grid * grid);
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t X = b % W, Y = b / W;
        float c[3] = {0.f, 0.f, 0.f}, d = 0.f, nn[3] = {0.f, 0.f, 0.f};
        for (int k = 0; k < grid * grid; ++k) {
            const int64_t P = (Y * grid + k / grid) * (int64_t)WW + X * grid + k % grid;
            const int32_t w = winner[P];
            if (w >= 0) {
                c[0] += __ldg(colors + 3 * (int64_t)w); c[1] += __ldg(colors + 3 * (int64_t)w + 1);
                c[2] += __ldg(colors + 3 * (int64_t)w + 2);
                if (b_depth) d += depth[P];
                if (b_normal) { nn[0] += normal[3 * P]; nn[1] += normal[3 * P + 1]; nn[2] += normal[3 * P + 2]; }
            } else {
                c[0] += bg0; c[1] += bg1; c[2] += bg2;
            }
            if (k == 0) s_depth[b] = depth[P];
        }
        s_color[3 * b] = c[0] * inv; s_color[3 * b + 1] = c[1] * inv; s_color[3 * b + 2] = c[2] * inv;
        if (b_depth) b_depth[b] = d * inv;
        if (b_normal) { b_normal[3 * b] = nn[0] * inv; b_normal[3 * b + 1] = nn[1] * inv; b_normal[3 * b + 2] = nn[2] * inv; }
    }
}

template <int DEG>
__global__ void k_surfel_sh_bwd(ges_scene_src_t src, CamK cam, const double* __restrict__ col, double* g_sh,
                                double* g_pos) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= src.n_surfels) return;
    const double gc[3] = {col[3 * j], col[3 * j + 1], col[3 * j + 2]};
    if (gc[0] == 0.0 && gc[1] == 0.0 && gc[2] == 0.0) return;   // not visible: outputs stay zero
    double p[3] = {src.s_pos[3 * j], src.s_pos[3 * j + 1], src.s_pos[3 * j + 2]};
    double shs[K * 3], gs[K * 3], gp[3];
    for (int k = 0; k < K * 3; ++k) shs[k] = src.s_sh[(int64_t)K * 3 * j + k];
    sh_backward<DEG>(shs, p, cam.pos, gc, gs, gp);
    for (int k = 0; k < K * 3; ++k) g_sh[(int64_t)K * 3 * j + k] = gs[k];
    for (int k = 0; k < 3; ++k) g_pos[3 * j + k] = gp[k];
}

// ---------------------------------------------------------------- launchers
#define GES_DEG_SWITCH(deg, KER, ...)                    \
    switch (deg) {                                       \
        case 0: KER<0><<<__VA_ARGS__>>>; break;          \
        case 1: KER<1><<<__VA_ARGS__>>>; break;          \
        case 2: KER<2><<<__VA_ARGS__>>>; break;          \
        default: KER<3><<<__VA_ARGS__>>>; break;         \
    }

cudaError_t launch_surfel_colors(const ges_scene_t& sc, const CamK& cam, float* rgb, cudaStream_t s) {
    if (sc.n_surfels == 0) return cudaSuccess;
    const unsigned nb = (unsigned)((sc.n_surfels + 255) / 256);
    switch (sc.sh_degree) {
        case 0: k_surfel_colors<0><<<nb, 256, 0, s>>>(sc, cam, rgb); break;
        case 1: k_surfel_colors<1><<<nb, 256, 0, s>>>(sc, cam, rgb); break;
        case 2: k_surfel_colors<2><<<nb, 256, 0, s>>>(sc, cam, rgb); break;
        default: k_surfel_colors<3><<<nb, 256, 0, s>>>(sc, cam, rgb); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_gauss_bwd(const BwdArgs& a, int g_kind, bool geom, cudaStream_t s) {
    const dim3 nt((unsigned)a.ntx, (unsigned)a.nty);
    if (g_kind == 2) {
        if (geom) k_gauss_bwd<2, true><<<nt, 256, 0, s>>>(a);
        else k_gauss_bwd<2, false><<<nt, 256, 0, s>>>(a);
    } else {
        if (geom) k_gauss_bwd<3, true><<<nt, 256, 0, s>>>(a);
        else k_gauss_bwd<3, false><<<nt, 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_gauss_contrib(const BwdArgs& a, int g_kind, cudaStream_t s) {
    const dim3 nt((unsigned)a.ntx, (unsigned)a.nty);
    if (g_kind == 2) k_gauss_bwd<2, false, true><<<nt, 256, 0, s>>>(a);
    else k_gauss_bwd<3, false, true><<<nt, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_gauss_finish(const ges_scene_src_t& src, int any_filter, int mip, const CamK& cam,
                                const double* acc, const ges_gauss_grads_t& out, cudaStream_t s) {
    if (src.n_gaussians == 0) return cudaSuccess;
    const unsigned nb = (unsigned)((src.n_gaussians + 127) / 128);
    if (src.gaussian_dim == 2) {
        switch (src.sh_degree) {
            case 0: k_gauss2_finish<0><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
            case 1: k_gauss2_finish<1><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
            case 2: k_gauss2_finish<2><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
            default: k_gauss2_finish<3><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
        }
    } else {
        switch (src.sh_degree) {
            case 0: k_gauss3_finish<0><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
            case 1: k_gauss3_finish<1><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
            case 2: k_gauss3_finish<2><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
            default: k_gauss3_finish<3><<<nb, 128, 0, s>>>(src, any_filter, mip, cam, acc, out); break;
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_frozen_bwd(const ges_scene_src_t& src, const CamK& cam, int W, int H, int grid,
                              const int32_t* winner, const float* g_cs, double* col, double* g_sh, double* g_pos,
                              cudaStream_t s) {
    if (src.n_surfels == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(col, 0, sizeof(double) * 3 * src.n_surfels, s);
    if (e != cudaSuccess) return e;
    k_frozen_scatter<<<148 * 16, 256, 0, s>>>(winner, g_cs, W, H, grid, col);
    const unsigned nb = (unsigned)((src.n_surfels + 127) / 128);
    switch (src.sh_degree) {
        case 0: k_surfel_sh_bwd<0><<<nb, 128, 0, s>>>(src, cam, col, g_sh, g_pos); break;
        case 1: k_surfel_sh_bwd<1><<<nb, 128, 0, s>>>(src, cam, col, g_sh, g_pos); break;
        case 2: k_surfel_sh_bwd<2><<<nb, 128, 0, s>>>(src, cam, col, g_sh, g_pos); break;
        default: k_surfel_sh_bwd<3><<<nb, 128, 0, s>>>(src, cam, col, g_sh, g_pos); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_frozen_resolve(const int32_t* winner, const float* depth, const float* normal, const float* colors,
                                  int W, int H, int grid, const float* bg, float* s_color, float* s_depth,
                                  float* b_depth, float* b_normal, cudaStream_t s) {
    k_frozen_resolve<<<148 * 16, 256, 0, s>>>(winner, depth, normal, colors, W, H, grid, bg[0], bg[1], bg[2], s_color,
                                              s_depth, b_depth, b_normal);
    return cudaGetLastError();
}

}  // namespace ges
