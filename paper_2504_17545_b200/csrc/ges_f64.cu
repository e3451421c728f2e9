// Float64 render mode (RenderSettings.dtype = float64, forward.py:44): the
// reference's own test suite renders in float64 (pkg/tests/test_forward.py:
// 33-35), so the drop-in computes the per-pixel passes in double precision
// when asked to.
//
// The frame reuses the float32 pipeline's binning (preprocess counts, scan,
// fill: conservative pixel ranges and depth keys, 16x16 tiles) and replaces
// the fused float32 tile kernel by
//   K1d/K4d  float64 per-primitive records from the SOURCE float64 arrays
//            (geometry.py:193-205 frames, :93-132 EWA, filters.py:84-109,
//            primitives.py:113-131, sh.py:117-133 colours), and
//   K6d      one CTA per 16x16 tile, one thread per base pixel (2x2
//            sub-samples at supersample=4): the surfel z-buffer (forward.py:
//            166-207: argmin over the hit depth, lowest source id on ties),
//            deferred view colour of the winners, the depth-gated Gaussian
//            sums (forward.py:248-381) and the composite / layer logic
//            (:384-417), all in float64 with the reference's formulas.
// Culling uses only the float32 records' conservative bounds (tile lists and
// disc depth keys), so it never changes a float64 decision.  This mode is for
// reference-precision callers, not for throughput (B200 float64 issue is half
// the float32 rate, and the kernel is deliberately the simple one).
#include <math.h>

#include "ges_launch.h"

namespace ges {

namespace {

constexpr double ALPHA_CUTOFF = 1.0 / 255.0;   // forward.py:26
constexpr double PARALLEL_EPS = 1e-8;          // geometry.py:15
constexpr int SREC = 16;                       // doubles per surfel record
constexpr int GREC3 = 16;                      // doubles per 3D Gaussian record
constexpr int GREC2 = 24;                      // doubles per planar Gaussian record

struct dv3 { double x, y, z; };
__device__ __forceinline__ double dot3(dv3 a, dv3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// geometry.py:18-36: rotation of the normalised quaternion (w, x, y, z); column k.
__device__ __forceinline__ void rotmat(const double* q4, double R[9]) {
    double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    const double n = sqrt(w * w + x * x + y * y + z * z);
    w /= n; x /= n; y /= n; z /= n;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

// camera-space image of world column k of R (geometry.py:193-205: Rm[:, :, k] @ cam.R^T)
__device__ __forceinline__ dv3 col_cam(const double R[9], int k, const CamK& c) {
    const double v0 = R[k], v1 = R[3 + k], v2 = R[6 + k];
    return {c.R[0] * v0 + c.R[1] * v1 + c.R[2] * v2, c.R[3] * v0 + c.R[4] * v1 + c.R[5] * v2,
            c.R[6] * v0 + c.R[7] * v1 + c.R[8] * v2};
}
__device__ __forceinline__ dv3 to_cam(const double* p, const CamK& c) {   // cameras.py:48-50
    return {c.R[0] * p[0] + c.R[1] * p[1] + c.R[2] * p[2] + c.t[0],
            c.R[3] * p[0] + c.R[4] * p[1] + c.R[5] * p[2] + c.t[1],
            c.R[6] * p[0] + c.R[7] * p[1] + c.R[8] * p[2] + c.t[2]};
}

// View colour (forward.py:99-109, sh.py:117-133): clip(0.5 + sum_k Y_k(dir) c_k, 0, 1)
// with dir = normalised (camera position - centre); sh is (K, 3) coefficient-major.
__device__ void view_colour(const double* sh, int deg, const double* pos, const double* cpos, double out[3]) {
    double dx = cpos[0] - pos[0], dy = cpos[1] - pos[1], dz = cpos[2] - pos[2];
    const double nr = fmax(sqrt(dx * dx + dy * dy + dz * dz), 1e-12);
    const double x = dx / nr, y = dy / nr, z = dz / nr;
    double B[16];
    B[0] = 0.28209479177387814;
    if (deg >= 1) {
        const double C1 = 0.4886025119029199;
        B[1] = -C1 * y; B[2] = C1 * z; B[3] = -C1 * x;
    }
    if (deg >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        B[4] = 1.0925484305920792 * x * y;
        B[5] = -1.0925484305920792 * y * z;
        B[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
        B[7] = -1.0925484305920792 * x * z;
        B[8] = 0.5462742152960396 * (xx - yy);
        if (deg >= 3) {
            B[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
            B[10] = 2.890611442640554 * x * y * z;
            B[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
            B[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            B[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
            B[14] = 1.445305721320277 * z * (xx - yy);
            B[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
        }
    }
    const int K = (deg + 1) * (deg + 1);
    for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += B[k] * sh[3 * k + c];
        out[c] = fmin(fmax(0.5 + s, 0.0), 1.0);
    }
}

// ---------------------------------------------------------------- K1d: surfel records
// rec = n(3) a1(3) a2(3) n.q a1.q a2.q s1 s2 alive 0, per PACKED surfel (the
// tile lists hold packed indices); forward.py:148-158 in float64.
__global__ void k_surfel_rec64(ges_scene_src_t src, const int32_t* s_id, int64_t ns, CamK cam, double* rec) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const int64_t o = s_id[i];
    double R[9];
    rotmat(src.s_quat + 4 * o, R);
    const dv3 q = to_cam(src.s_pos + 3 * o, cam);
    const dv3 a1 = col_cam(R, 0, cam), a2 = col_cam(R, 1, cam), n = col_cam(R, 2, cam);
    double* r = rec + SREC * i;
    r[0] = n.x; r[1] = n.y; r[2] = n.z;
    r[3] = a1.x; r[4] = a1.y; r[5] = a1.z;
    r[6] = a2.x; r[7] = a2.y; r[8] = a2.z;
    r[9] = dot3(n, q); r[10] = dot3(a1, q); r[11] = dot3(a2, q);
    r[12] = exp(src.s_log_scale[2 * o]);
    r[13] = exp(src.s_log_scale[2 * o + 1]);
    r[14] = q.z > NEAR ? 1.0 : 0.0;   // (the range part of `alive` is the tile list)
    r[15] = 0.0;
}

// Effective scale / opacity / adaptive epsilon, primitives.py:113-131 (with
// filter3d = 0 the effective values equal the raw ones exactly).
__device__ __forceinline__ double gauss_eff(const ges_scene_src_t& src, int64_t o, int D, double es[3]) {
    const double f3 = src.g_filter3d ? src.g_filter3d[o] : 0.0;
    double sig = 1.0 / (1.0 + exp(-src.g_raw_opacity[o]));
    for (int k = 0; k < D; ++k) {
        const double s = exp(src.g_log_scale[D * o + k]);
        es[k] = sqrt(s * s + f3);
        sig *= s / es[k];
    }
    return sig;
}

struct GaussCfg64 {
    int mip, eps_const, deg;
    double eps_value;
};

// ---------------------------------------------------------------- K4d: 3D EWA records
// rec = valid mx my la lb lc sig z eps col(3) nrm(3) 0 (forward.py:252-290,
// geometry.py:93-132; nrm: camera-facing normal of the smallest axis, :277-284)
__global__ void k_gauss3_rec64(ges_scene_src_t src, int64_t ng, CamK cam, GaussCfg64 cfg, double* rec) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= ng) return;
    const int64_t o = src.g_order ? src.g_order[j] : j;
    double es[3];
    double sig = gauss_eff(src, o, 3, es);
    const double eps = cfg.eps_const ? cfg.eps_value : (5.0 / 3.0) * (es[0] + es[1] + es[2]);
    double R[9];
    rotmat(src.g_quat + 4 * o, R);
    const double* p = src.g_pos + 3 * o;
    const dv3 t = to_cam(p, cam);
    bool valid = t.z > NEAR;
    const dv3 ts = valid ? t : dv3{0.0, 0.0, 1.0};
    // V = R diag(es^2) R^T; M = W V W^T
    double V[9], M[9], T[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double v = 0.0;
            for (int k = 0; k < 3; ++k) v += R[3 * a + k] * (es[k] * es[k]) * R[3 * b + k];
            V[3 * a + b] = v;
        }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double v = 0.0;
            for (int k = 0; k < 3; ++k) v += cam.R[3 * a + k] * V[3 * k + b];
            T[3 * a + b] = v;
        }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double v = 0.0;
            for (int k = 0; k < 3; ++k) v += T[3 * a + k] * cam.R[3 * b + k];
            M[3 * a + b] = v;
        }
    const double iz = 1.0 / ts.z;
    const double J[6] = {cam.fx * iz, 0.0, -cam.fx * ts.x * iz * iz, 0.0, cam.fy * iz, -cam.fy * ts.y * iz * iz};
    double cov[4];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            double v = 0.0;
            for (int k = 0; k < 3; ++k) {
                double w = 0.0;
                for (int l = 0; l < 3; ++l) w += M[3 * k + l] * J[3 * b + l];
                v += J[3 * a + k] * w;
            }
            cov[2 * a + b] = v;
        }
    const double mx = cam.fx * ts.x / ts.z + cam.cx, my = cam.fy * ts.y / ts.z + cam.cy;
    const double raw_det = cov[0] * cov[3] - cov[1] * cov[1];
    const double c00 = cov[0] + SCREEN_VAR, c11 = cov[3] + SCREEN_VAR, c01 = cov[1];
    const double det = c00 * c11 - c01 * c01;
    if (cfg.mip) sig = sig * sqrt(fmax(raw_det, 0.0) / det);
    valid = valid && det > 0.0;
    const double m2max = 2.0 * log(fmax(255.0 * sig, 1e-12));
    valid = valid && m2max > 0.0;
    double* r = rec + GREC3 * j;
    r[0] = valid ? 1.0 : 0.0;
    // r[15]: exponent below which sig * exp(pw) < 1/255 beyond any rounding (a
    // pre-screen only: the kept cases take the exact test)
    const double lt = log(ALPHA_CUTOFF / fmax(sig, 1e-300));
    r[15] = lt - 1e-9 * (1.0 + fabs(lt));
    r[1] = mx; r[2] = my;
    r[3] = c11 / det; r[4] = -c01 / det; r[5] = c00 / det;
    r[6] = sig; r[7] = t.z; r[8] = eps;
    double col[3];
    view_colour(src.g_sh + (size_t)o * 3 * (cfg.deg + 1) * (cfg.deg + 1), cfg.deg, p, cam.pos, col);
    r[9] = col[0]; r[10] = col[1]; r[11] = col[2];
    const int k = (es[1] < es[0]) ? ((es[2] < es[1]) ? 2 : 1) : ((es[2] < es[0]) ? 2 : 0);   // argmin (first)
    const dv3 nv = col_cam(R, k, cam);
    const double sg = dot3(nv, t) < 0.0 ? 1.0 : -1.0;
    r[12] = nv.x * sg; r[13] = nv.y * sg; r[14] = nv.z * sg;
}

// ---------------------------------------------------------------- K4d: planar records
// rec = n(3) a1(3) a2(3) n.q a1.q a2.q s1 s2 sig eps col(3) nvis(3) valid 0
// (forward.py:324-381 with object_space_filter_2d, filters.py:84-109)
__global__ void k_gauss2_rec64(ges_scene_src_t src, int64_t ng, CamK cam, GaussCfg64 cfg, double* rec) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= ng) return;
    const int64_t o = src.g_order ? src.g_order[j] : j;
    double es[3] = {0.0, 0.0, 0.0};
    double sig = gauss_eff(src, o, 2, es);
    const double eps = cfg.eps_const ? cfg.eps_value : (5.0 / 2.0) * (es[0] + es[1]);
    double R[9];
    rotmat(src.g_quat + 4 * o, R);
    const double* p = src.g_pos + 3 * o;
    const dv3 q = to_cam(p, cam);
    const dv3 a1 = col_cam(R, 0, cam), a2 = col_cam(R, 1, cam), n = col_cam(R, 2, cam);
    double s1 = es[0], s2 = es[1];
    bool valid = true;
    if (cfg.mip) {   // object_filter_2d
        const double z = q.z;
        double J[2][2];
        const double qa[2] = {q.x, q.y}, m1[3] = {a1.x * s1, a1.y * s1, a1.z * s1},
                     m2[3] = {a2.x * s2, a2.y * s2, a2.z * s2};
        for (int ax = 0; ax < 2; ++ax) {
            const double f = ax ? cam.fy : cam.fx;
            J[ax][0] = f * (m1[ax] * z - qa[ax] * m1[2]) / (z * z);
            J[ax][1] = f * (m2[ax] * z - qa[ax] * m2[2]) / (z * z);
        }
        const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        valid = fabs(det) > 1e-12 && z > NEAR;
        const double dets = valid ? det : 1.0;
        const double i00 = J[1][1] / dets, i01 = -J[0][1] / dets, i10 = -J[1][0] / dets, i11 = J[0][0] / dets;
        const double m0 = sqrt(1.0 + SCREEN_VAR * (i00 * i00 + i01 * i01));
        const double mm1 = sqrt(1.0 + SCREEN_VAR * (i10 * i10 + i11 * i11));
        s1 *= m0;
        s2 *= mm1;
        sig *= 1.0 / (m0 * mm1);
    }
    const double m2max = 2.0 * log(fmax(255.0 * sig, 1e-12));
    valid = valid && q.z > NEAR && m2max > 0.0;
    const double nq = dot3(n, q);
    double* r = rec + GREC2 * j;
    r[0] = n.x; r[1] = n.y; r[2] = n.z;
    r[3] = a1.x; r[4] = a1.y; r[5] = a1.z;
    r[6] = a2.x; r[7] = a2.y; r[8] = a2.z;
    r[9] = nq; r[10] = dot3(a1, q); r[11] = dot3(a2, q);
    r[12] = s1; r[13] = s2; r[14] = sig; r[15] = eps;
    double col[3];
    view_colour(src.g_sh + (size_t)o * 3 * (cfg.deg + 1) * (cfg.deg + 1), cfg.deg, p, cam.pos, col);
    r[16] = col[0]; r[17] = col[1]; r[18] = col[2];
    const double sg = nq < 0.0 ? 1.0 : -1.0;
    r[19] = n.x * sg; r[20] = n.y * sg; r[21] = n.z * sg;
    r[22] = valid ? 1.0 : 0.0;
    // r[23]: u^2 + v^2 beyond which sig * exp(-q/2) < 1/255 beyond any rounding (pre-screen)
    const double qm = 2.0 * log(fmax(255.0 * sig, 1e-300));
    r[23] = qm + 1e-9 * (1.0 + fabs(qm));
}

// ---------------------------------------------------------------- K6d: the tile
struct Tile64Args {
    int W, H, ntx, grid, mode, layers, gk, geom, deg;
    double bg[3];
    CamK cs, cg;                  // surfel-pass camera (scaled by grid) and base camera
    SlabMap slabs;
    const double* srec;
    const float4* scull;
    const uint32_t* s_list;
    BinPass sbin;
    const int32_t* s_id;          // packed -> source surfel
    ges_scene_src_t src;
    const double* grec;
    const float4* gcull;
    const uint32_t* g_list;
    BinPass gbin;
    const double* ds_in;          // mode 2: surfel depth (H, W)
    ges_outputs_f64_t out;
    const ges_frame_status_t* status;
};

__device__ __forceinline__ double warp_max64(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ bool span_hits(uint32_t sx, uint32_t sy, int x0, int x1, int y0, int y1) {
    return span_lo(sx) <= x1 && span_hi(sx) >= x0 && span_lo(sy) <= y1 && span_hi(sy) >= y0;
}

// Each warp (16 x 2 pixels of the tile) walks the tile's near-to-far lists 32
// entries at a time: the lanes load the chunk's ids and float32 cull records
// together; entries whose pixel range misses the warp's rows, or whose
// conservative depth key lies behind every pixel's current best, are skipped
// by the whole warp; the walk stops at the first slab behind all of the
// warp's pixels.  That is the float32 path's culling (all bounds
// conservative), so every float64 decision is still the per-pixel test's.
template <int G>   // sub-samples per axis of the surfel pass (1, or 2 at supersample=4)
__global__ void __launch_bounds__(256) k_tile64(Tile64Args a) {
    __shared__ uint32_t s_end[NSLAB], g_end[NSLAB];
    if (a.status->overflow) return;
    const int tile = blockIdx.x;
    for (int k = threadIdx.x; k < NSLAB; k += blockDim.x) {
        if (a.mode & 1) s_end[k] = a.sbin.cnt[tile * NSLAB + k];
        if (a.mode & 2) g_end[k] = a.gbin.cnt[tile * NSLAB + k];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wrow = 2 * (threadIdx.x >> 5);   // the warp's first tile row
    const int tx = tile % a.ntx, ty = tile / a.ntx;
    const int x = tx * TILE + (threadIdx.x & 15), y = ty * TILE + (threadIdx.x >> 4);
    const bool inside = x < a.W && y < a.H;
    const double R2 = R_OPAQUE * R_OPAQUE;
    double ds = INFINITY;
    double s_col[3] = {a.bg[0], a.bg[1], a.bg[2]};
    const int64_t pix = (int64_t)y * a.W + x;

    if (a.mode & 1) {
        // ---- pass 1: float64 z-buffer per sub-sample (forward.py:166-207)
        double bt[G * G];
        int32_t bid[G * G];
        uint32_t bpk[G * G];
        dv3 dvec[G * G];
        double dn[G * G];
#pragma unroll
        for (int s = 0; s < G * G; ++s) { bt[s] = INFINITY; bid[s] = -1; bpk[s] = 0; }
#pragma unroll
        for (int s = 0; s < G * G; ++s) {
            const int X = x * G + (s % G), Y = y * G + (s / G);
            dvec[s] = {((double)X + 0.5 - a.cs.cx) / a.cs.fx, ((double)Y + 0.5 - a.cs.cy) / a.cs.fy, 1.0};
            dn[s] = sqrt(dot3(dvec[s], dvec[s]));
        }
        auto worst_of = [&]() {   // the thread's max best depth (-inf outside the image)
            double wv = bt[0];
#pragma unroll
            for (int s = 1; s < G * G; ++s) wv = fmax(wv, bt[s]);
            return inside ? wv : -INFINITY;
        };
        const int wx0 = tx * TILE * G, wx1 = wx0 + TILE * G - 1;   // the warp's rows in the sample grid
        const int wy0 = (ty * TILE + wrow) * G, wy1 = wy0 + 2 * G - 1;
        const uint32_t beg = a.sbin.tile_off(tile), end = beg + s_end[NSLAB - 1];
        for (uint32_t e0 = beg; e0 < end; e0 += 32) {
            const double wmax = warp_max64(worst_of());
            if ((double)a.slabs.lower(slab_of_pos(s_end, e0 - beg, lane)) > wmax) break;
            uint32_t id = 0;
            float key = INFINITY;
            bool live = false;
            if (e0 + lane < end) {
                id = __ldg(a.s_list + e0 + lane);
                const float4 c = __ldg(a.scull + id);
                key = c.x;
                live = span_hits(__float_as_uint(c.y), __float_as_uint(c.z), wx0, wx1, wy0, wy1) &&
                       !((double)key > wmax);
            }
            uint32_t vote = __ballot_sync(0xffffffffu, live);
            while (vote) {
                const int j = __ffs(vote) - 1;
                vote &= vote - 1;
                const uint32_t i = __shfl_sync(0xffffffffu, id, j);
                const float kj = __shfl_sync(0xffffffffu, key, j);
                if ((double)kj > worst_of()) continue;   // behind every sample's best (-inf: outside)
                const double* r = a.srec + SREC * (size_t)i;
                if (r[14] == 0.0) continue;              // q_z <= NEAR
                const dv3 n = {r[0], r[1], r[2]}, a1 = {r[3], r[4], r[5]}, a2 = {r[6], r[7], r[8]};
                const int32_t sid = a.s_id[i];
#pragma unroll
                for (int s = 0; s < G * G; ++s) {
                    const double ndot = dot3(n, dvec[s]);
                    const double th = r[9] / ndot;
                    // the reference's conditions (geometry.py:216-226, forward.py:183-187),
                    // the depth comparison first: u, v only for samples it would win
                    if (!(th < bt[s] || (th == bt[s] && sid < bid[s]))) continue;
                    if (!(fabs(ndot) > PARALLEL_EPS * dn[s] && th > NEAR)) continue;
                    const double u = (th * dot3(a1, dvec[s]) - r[10]) / r[12];
                    const double v = (th * dot3(a2, dvec[s]) - r[11]) / r[13];
                    if (u * u + v * v <= R2) {
                        bt[s] = th;
                        bid[s] = sid;
                        bpk[s] = i;
                    }
                }
            }
        }
        // winners' view colours (box mean over the sub-samples) and the sample-0 buffers
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int s = 0; s < G * G; ++s) {
            double c[3] = {a.bg[0], a.bg[1], a.bg[2]};
            if (bid[s] >= 0) {
                const int64_t o = bid[s];
                view_colour(a.src.s_sh + (size_t)o * 3 * (a.deg + 1) * (a.deg + 1), a.deg, a.src.s_pos + 3 * o,
                            a.cs.pos, c);
            }
            acc[0] += c[0]; acc[1] += c[1]; acc[2] += c[2];
        }
        const double inv = 1.0 / (double)(G * G);
        s_col[0] = acc[0] * inv; s_col[1] = acc[1] * inv; s_col[2] = acc[2] * inv;
        ds = bid[0] >= 0 ? bt[0] : INFINITY;
        if (inside) {
            if (a.out.s_color) { a.out.s_color[3 * pix] = s_col[0]; a.out.s_color[3 * pix + 1] = s_col[1]; a.out.s_color[3 * pix + 2] = s_col[2]; }
            if (a.out.s_depth) a.out.s_depth[pix] = ds;
            if (a.out.s_winner) a.out.s_winner[pix] = bid[0];
            if (a.out.s_normal) {
                double nv[3] = {0.0, 0.0, 0.0};
                if (bid[0] >= 0) {
                    const double* r = a.srec + SREC * (size_t)bpk[0];
                    const double sg = r[9] < 0.0 ? 1.0 : -1.0;   // n_vis (forward.py:152)
                    nv[0] = r[0] * sg; nv[1] = r[1] * sg; nv[2] = r[2] * sg;
                }
                a.out.s_normal[3 * pix] = nv[0]; a.out.s_normal[3 * pix + 1] = nv[1]; a.out.s_normal[3 * pix + 2] = nv[2];
            }
        }
    } else if (inside) {
        ds = a.ds_in[pix];
    }

    // ---- pass 2: depth-gated float64 Gaussian sums (forward.py:248-381)
    double w = 0.0, cr = 0.0, cg = 0.0, cb = 0.0, gd = 0.0, n0 = 0.0, n1 = 0.0, n2 = 0.0;
    if (a.mode & 2) {
        const uint32_t beg = a.gbin.tile_off(tile), end = beg + g_end[NSLAB - 1];
        const double px = (double)x + 0.5, py = (double)y + 0.5;
        const dv3 d = {(px - a.cg.cx) / a.cg.fx, (py - a.cg.cy) / a.cg.fy, 1.0};
        const double dn = sqrt(dot3(d, d));
        const double wdmax = warp_max64(inside ? ds : -INFINITY);
        const int wx0 = tx * TILE, wx1 = wx0 + TILE - 1, wy0 = ty * TILE + wrow, wy1 = wy0 + 1;
        for (uint32_t e0 = beg; e0 < end; e0 += 32) {
            // keys (depth - eps) are binned near-to-far: the rest fail every gate of the warp
            if ((double)a.slabs.lower(slab_of_pos(g_end, e0 - beg, lane)) > wdmax) break;
            uint32_t id = 0;
            bool live = false;
            if (e0 + lane < end) {
                id = __ldg(a.g_list + e0 + lane);
                const float4 c = __ldg(a.gcull + id);
                live = span_hits(__float_as_uint(c.z), __float_as_uint(c.w), wx0, wx1, wy0, wy1);
            }
            uint32_t vote = __ballot_sync(0xffffffffu, live);
            while (vote) {
                const int jl = __ffs(vote) - 1;
                vote &= vote - 1;
                const uint32_t j = __shfl_sync(0xffffffffu, id, jl);
                if (!inside) continue;
                if (a.gk == 3) {
                    const double* r = a.grec + GREC3 * (size_t)j;
                    if (r[0] == 0.0 || !(r[7] < ds + r[8])) continue;   // invalid, or fails the gate
                    const double dx = px - r[1], dy = py - r[2];
                    const double pw = -0.5 * (r[3] * dx * dx + r[5] * dy * dy) - r[4] * dx * dy;
                    if (pw < r[15]) continue;   // far below the 1/255 cutoff: no exp needed
                    const double al = r[6] * exp(pw);
                    if (al >= ALPHA_CUTOFF) {
                        w += al;
                        cr += al * r[9]; cg += al * r[10]; cb += al * r[11];
                        gd += al * r[7];
                        n0 += al * r[12]; n1 += al * r[13]; n2 += al * r[14];
                    }
                } else {
                    const double* r = a.grec + GREC2 * (size_t)j;
                    if (r[22] == 0.0) continue;
                    const dv3 n = {r[0], r[1], r[2]}, a1 = {r[3], r[4], r[5]}, a2 = {r[6], r[7], r[8]};
                    const double ndot = dot3(n, d);
                    const double th = r[9] / ndot;
                    const bool ok = fabs(ndot) > PARALLEL_EPS * dn && th > NEAR;
                    if (!ok || !(th < ds + r[15])) continue;
                    const double u = (th * dot3(a1, d) - r[10]) / r[12];
                    const double v = (th * dot3(a2, d) - r[11]) / r[13];
                    const double q2 = u * u + v * v;
                    if (q2 > r[23]) continue;   // far outside the 1/255 support: no exp needed
                    const double al = r[14] * exp(-0.5 * q2);
                    if (al >= ALPHA_CUTOFF) {
                        w += al;
                        cr += al * r[16]; cg += al * r[17]; cb += al * r[18];
                        gd += al * th;
                        n0 += al * r[19]; n1 += al * r[20]; n2 += al * r[21];
                    }
                }
            }
        }
    }
    if (!inside) return;
    if (a.mode & 2) {
        if (a.out.g_weight) a.out.g_weight[pix] = w;
        if (a.out.g_color) { a.out.g_color[3 * pix] = cr; a.out.g_color[3 * pix + 1] = cg; a.out.g_color[3 * pix + 2] = cb; }
        if (a.geom) {
            if (a.out.g_depth) a.out.g_depth[pix] = gd;
            if (a.out.g_normal) { a.out.g_normal[3 * pix] = n0; a.out.g_normal[3 * pix + 1] = n1; a.out.g_normal[3 * pix + 2] = n2; }
        }
    } else if (a.mode & 1) {   // surfels_only: empty Gaussian buffers (forward.py:407-410)
        if (a.out.g_weight) a.out.g_weight[pix] = 0.0;
        if (a.out.g_color) { a.out.g_color[3 * pix] = 0.0; a.out.g_color[3 * pix + 1] = 0.0; a.out.g_color[3 * pix + 2] = 0.0; }
    }
    if (a.out.image && (a.mode & 1)) {
        double im[3];
        if (!(a.mode & 2)) {
            im[0] = s_col[0]; im[1] = s_col[1]; im[2] = s_col[2];
        } else if (a.layers == GES_LAYERS_GAUSSIANS_ONLY) {   // forward.py:412-416
            const double dnm = fmax(w, 1e-12);
            im[0] = w > 0.0 ? cr / dnm : a.bg[0];
            im[1] = w > 0.0 ? cg / dnm : a.bg[1];
            im[2] = w > 0.0 ? cb / dnm : a.bg[2];
        } else {                                               // composite, forward.py:384-388
            const double den = 1.0 + w;
            im[0] = (s_col[0] * 1.0 + cr) / den; im[1] = (s_col[1] * 1.0 + cg) / den; im[2] = (s_col[2] * 1.0 + cb) / den;
        }
        a.out.image[3 * pix] = im[0]; a.out.image[3 * pix + 1] = im[1]; a.out.image[3 * pix + 2] = im[2];
    }
}

__global__ void k_composite64(const double* __restrict__ sc, const double* __restrict__ gc,
                              const double* __restrict__ gw, double sw, double* __restrict__ img, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double dn = sw + gw[i];
        for (int c = 0; c < 3; ++c) img[3 * i + c] = (sc[3 * i + c] * sw + gc[3 * i + c]) / dn;
    }
}

__global__ void k_smooth64(const double* __restrict__ sd, const double* __restrict__ sn, const double* __restrict__ gd,
                           const double* __restrict__ gn, const double* __restrict__ gw, double* __restrict__ dout,
                           double* __restrict__ nout, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double dn = 1.0 + gw[i];
        dout[i] = (sd[i] + gd[i]) / dn;
        const double v0 = (sn[3 * i] + gn[3 * i]) / dn, v1 = (sn[3 * i + 1] + gn[3 * i + 1]) / dn,
                     v2 = (sn[3 * i + 2] + gn[3 * i + 2]) / dn;
        const double nr = sqrt(v0 * v0 + v1 * v1 + v2 * v2);   // forward.py:398-400
        const double dv = fmax(nr, 1e-12);
        const bool ok = nr > 1e-12;
        nout[3 * i] = ok ? v0 / dv : 0.0; nout[3 * i + 1] = ok ? v1 / dv : 0.0; nout[3 * i + 2] = ok ? v2 / dv : 0.0;
    }
}

}  // namespace

size_t f64_record_bytes(int64_t ns, int64_t ng, int gdim) {
    const size_t a = ((size_t)ns * SREC * sizeof(double) + 255) & ~size_t(255);
    return a + (size_t)ng * (gdim == 2 ? GREC2 : GREC3) * sizeof(double);
}

cudaError_t launch_f64(const F64Launch& L, cudaStream_t s) {
    const size_t soff = ((size_t)L.ns * SREC * sizeof(double) + 255) & ~size_t(255);
    double* srec = static_cast<double*>(L.records);
    double* grec = reinterpret_cast<double*>(static_cast<char*>(L.records) + soff);
    if ((L.mode & 1) && L.ns > 0)
        k_surfel_rec64<<<(unsigned)((L.ns + 127) / 128), 128, 0, s>>>(L.src, L.s_id, L.ns, L.cs, srec);
    GaussCfg64 gc{L.mip, L.eps_const, L.deg, L.eps_value};
    if ((L.mode & 2) && L.ng > 0) {
        if (L.gdim == 2) k_gauss2_rec64<<<(unsigned)((L.ng + 127) / 128), 128, 0, s>>>(L.src, L.ng, L.cg, gc, grec);
        else k_gauss3_rec64<<<(unsigned)((L.ng + 127) / 128), 128, 0, s>>>(L.src, L.ng, L.cg, gc, grec);
    }
    Tile64Args a{};
    a.W = L.W; a.H = L.H; a.ntx = L.ntx; a.grid = L.grid; a.mode = L.mode; a.layers = L.layers;
    a.gk = L.gdim; a.geom = L.geom; a.deg = L.deg;
    for (int i = 0; i < 3; ++i) a.bg[i] = L.bg[i];
    a.cs = L.cs; a.cg = L.cg; a.slabs = L.slabs;
    a.gcull = L.gcull;
    a.srec = srec; a.scull = L.scull; a.s_list = L.s_list; a.sbin = L.sbin; a.s_id = L.s_id; a.src = L.src;
    a.grec = grec; a.g_list = L.g_list; a.gbin = L.gbin;
    a.ds_in = L.ds_in;
    a.out = L.out;
    a.status = L.status;
    if (L.ntiles > 0) {
        if (L.grid == 2) k_tile64<2><<<(unsigned)L.ntiles, 256, 0, s>>>(a);
        else k_tile64<1><<<(unsigned)L.ntiles, 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_composite64(const double* sc, const double* gc, const double* gw, double sw, double* img,
                               int64_t n, cudaStream_t s) {
    if (n > 0) k_composite64<<<1184, 256, 0, s>>>(sc, gc, gw, sw, img, n);
    return cudaGetLastError();
}

cudaError_t launch_smooth64(const double* sd, const double* sn, const double* gd, const double* gn, const double* gw,
                            double* d_out, double* n_out, int64_t n, cudaStream_t s) {
    if (n > 0) k_smooth64<<<1184, 256, 0, s>>>(sd, sn, gd, gn, gw, d_out, n_out, n);
    return cudaGetLastError();
}

}  // namespace ges
