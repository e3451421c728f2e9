// C-ABI entry points (include/ges_b200.h): argument validation, scene-blob and
// frame-workspace layout, and the per-frame launch sequence
//   memset -> K1 surfel prep(+count) -> K4 Gaussian prep(+count) -> scan -> fill -> fused tile kernel
// Every call is stream-ordered and capturable in a CUDA graph (no host sync).
#include <stdio.h>
#include <string.h>

#include <string>

#include "ges_launch.h"
#include "ges_sh.cuh"

using namespace ges;

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return GES_ECUDA;
}

inline size_t al(size_t v) { return (v + 255) & ~size_t(255); }

// Side lane of a caller stream: the Gaussian preprocess runs on it, forked
// from and joined back into the caller's stream with two events, so it
// overlaps the surfel preprocess of the same frame (both read only the
// scene and write disjoint records/counters).  One side stream per (caller
// stream, device), created on first use and kept for the thread's lifetime;
// works under stream capture (the fork/join become graph edges).
struct SideLane {
    cudaStream_t caller, side;
    cudaEvent_t fork, join;
    int device;
};

SideLane* side_lane(cudaStream_t s) {
    static thread_local SideLane lanes[64];
    static thread_local int n = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    for (int i = 0; i < n; ++i)
        if (lanes[i].caller == s && lanes[i].device == dev) return &lanes[i];
    if (n == 64) return nullptr;   // (more caller streams than lanes: run sequentially)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return nullptr;            // (lanes are made outside capture: the first call of a stream is eager)
    SideLane& l = lanes[n];
    if (cudaStreamCreateWithFlags(&l.side, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (cudaEventCreateWithFlags(&l.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&l.join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    l.caller = s;
    l.device = dev;
    return &lanes[n++];
}

struct Carve {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t n) {
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += al(n * sizeof(T));
        return p;
    }
};

int check_settings(const ges_settings_t* st) {
    if (!st) return fail(GES_EINVAL, "settings is NULL");
    if (st->supersample != 1 && st->supersample != 4) return fail(GES_EINVAL, "supersample must be 1 or 4");
    if (st->layers < 0 || st->layers > 2) return fail(GES_EINVAL, "unknown layer mode");
    if (st->epsilon_mode != 0 && st->epsilon_mode != 1) return fail(GES_EINVAL, "unknown epsilon mode");
    if (st->tile_mode < 0 || st->tile_mode > 2) return fail(GES_EINVAL, "tile_mode must be 0, 1 or 2");
    return GES_OK;
}

int check_scene(const ges_scene_t* sc) {
    if (!sc) return fail(GES_EINVAL, "scene is NULL");
    if (sc->sh_degree < 0 || sc->sh_degree > 3) return fail(GES_EDEGREE, "SH degree must be in [0, 3]");
    if (sc->gaussian_dim != 2 && sc->gaussian_dim != 3) return fail(GES_EINVAL, "gaussian_dim must be 2 or 3");
    if (sc->n_surfels < 0 || sc->n_gaussians < 0) return fail(GES_EINVAL, "negative primitive count");
    if (sc->n_surfels >= (1ll << 31) || sc->n_gaussians >= (1ll << 31))
        return fail(GES_EINVAL, "primitive count exceeds 2^31");
    return GES_OK;
}

int check_cam(const ges_camera_t* c) {
    if (!c) return fail(GES_EINVAL, "camera is NULL");
    if (!(c->fx > 0) || !(c->fy > 0)) return fail(GES_EINVAL, "focal lengths must be positive");
    if (c->width <= 0 || c->height <= 0 || c->width > 32767 || c->height > 32767)
        return fail(GES_EINVAL, "image size out of range");
    return GES_OK;
}

// Frame workspace layout; base == nullptr only measures.
struct Frame {
    SurfRec* srec;
    float4* scull;
    void* grec;
    float4* gcull;
    float4* g_nrm;
    uint32_t *cnt_s, *off_s, *cnt_g, *off_g, *chunk_s, *chunk_g, *tickets;
    size_t zero_bytes;   // counters + tickets, cleared by one memset per frame
    uint32_t *list_s, *list_g;
    uint32_t *order, *tot;
    void* rec64;         // float64 mode: per-primitive float64 records
    ges_frame_status_t* status;
    size_t bytes;
    int ntx, nty, ntiles, px;
};

// Base pixels per tile-kernel thread per axis: 2 (32x32-pixel tiles, 2x2
// pixels per thread) for plain frames large enough to fill the GPU, else 1.
int tile_px_of(const ges_camera_t* cam, const ges_settings_t* st) {
    if (st->supersample != 1 || st->with_geometry) return 1;
    if (st->tile_mode == 1 || st->tile_mode == 2) return st->tile_mode;
    return (int64_t)cam->width * cam->height >= 512 * 512 ? 2 : 1;
}

Frame layout(void* base, const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st, int64_t cap_s,
             int64_t cap_g, bool f64 = false) {
    Frame f{};
    Carve c{static_cast<char*>(base)};
    f.px = tile_px_of(cam, st);
    const int tp = TILE * f.px;
    f.ntx = (cam->width + tp - 1) / tp;
    f.nty = (cam->height + tp - 1) / tp;
    f.ntiles = f.ntx * f.nty;
    size_t ns = (size_t)sc->n_surfels, ng = (size_t)sc->n_gaussians;
    f.status = c.take<ges_frame_status_t>(1);
    const size_t nbins = (size_t)f.ntiles * NSLAB;   // both passes' counters + tickets: one memset
    f.cnt_s = c.take<uint32_t>(2 * nbins + 64);
    f.cnt_g = f.cnt_s ? f.cnt_s + nbins : nullptr;
    f.tickets = f.cnt_s ? f.cnt_s + 2 * nbins : nullptr;
    f.zero_bytes = (2 * nbins + 64) * sizeof(uint32_t);
    const size_t nchunk = ((size_t)f.ntiles >> SCAN_CHUNK_SHIFT) + 2;
    f.order = c.take<uint32_t>(f.ntiles);
    f.tot = c.take<uint32_t>(f.ntiles);
    f.off_s = c.take<uint32_t>(f.ntiles);
    f.off_g = c.take<uint32_t>(f.ntiles);
    f.chunk_s = c.take<uint32_t>(nchunk);
    f.chunk_g = c.take<uint32_t>(nchunk);
    f.srec = c.take<SurfRec>(ns);
    f.scull = c.take<float4>(ns);
    f.grec = c.take<char>(ng * (sc->gaussian_dim == 2 ? sizeof(Gauss2Rec) : sizeof(GaussRec)));
    f.gcull = c.take<float4>(ng);
    f.g_nrm = c.take<float4>(ng);
    f.list_s = c.take<uint32_t>((size_t)cap_s);
    f.list_g = c.take<uint32_t>((size_t)cap_g);
    f.rec64 = f64 ? c.take<char>(f64_record_bytes((int64_t)ns, (int64_t)ng, sc->gaussian_dim)) : nullptr;
    f.bytes = c.off;
    return f;
}

// Depth range of the binning slabs for one view: camera z of the scene's
// bounding-box corners widened by the largest primitive radius.
SlabMap slab_map(const ges_scene_t& sc, const CamK& c) {
    const double* b = sc.bounds;
    double zlo = 1e300, zhi = -1e300;
    for (int k = 0; k < 8; ++k) {
        double p[3] = {b[(k & 1) ? 3 : 0], b[(k & 2) ? 4 : 1], b[(k & 4) ? 5 : 2]};
        double z = c.R[6] * p[0] + c.R[7] * p[1] + c.R[8] * p[2] + c.t[2];
        zlo = z < zlo ? z : zlo;
        zhi = z > zhi ? z : zhi;
    }
    zlo = zlo - b[6];
    zhi = zhi + b[6];
    if (zlo < NEAR) zlo = NEAR;
    SlabMap m;
    if (!(zhi > zlo + 1e-9)) {   // degenerate or missing bounds: everything in slab 0
        m.zlo = 0.f;
        m.inv_dz = 0.f;
        m.dz = 0.f;
    } else {
        m.zlo = (float)zlo;
        m.inv_dz = (float)(NSLAB / (zhi - zlo));
        m.dz = (float)((zhi - zlo) / NSLAB);
    }
    return m;
}

#ifndef GES_TILE_ORDER
#define GES_TILE_ORDER 1   // tile kernel CTAs in descending pair-count order (k_scan computes it)
#endif

// Float64 mode of a frame (ges_render_f64): the source arrays, the float64
// outputs and the external float64 surfel depth of the pass-2-only entry.
struct F64Ctx {
    const ges_scene_src_t* src;
    const ges_outputs_f64_t* out;
    const double* ds_in;
};

// mode: 1 surfel pass, 2 Gaussian pass against ds_in, 3 both.
int run_frame(const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st_in, const ges_outputs_t* out,
              const float* ds_in, int mode, void* ws, size_t ws_bytes, int64_t cap_s, int64_t cap_g,
              ges_frame_status_t* status_dev, cudaStream_t s, void* const* ev = nullptr,
              const F64Ctx* f64 = nullptr) {
    int rc;
    if ((rc = check_scene(sc)) || (rc = check_cam(cam)) || (rc = check_settings(st_in))) return rc;
    if (!out && !f64) return fail(GES_EINVAL, "outputs is NULL");
    if (cap_s < 0 || cap_g < 0 || cap_s >= (1ll << 32) || cap_g >= (1ll << 32))
        return fail(GES_EINVAL, "pair capacity out of range");
    ges_settings_t st64;
    const ges_settings_t* st = st_in;
    if (f64) {   // the float64 tile kernel works on 16x16 tiles, one thread per base pixel
        st64 = *st_in;
        st64.tile_mode = 1;
        st = &st64;
    }
    Frame f = layout(ws, sc, cam, st, cap_s, cap_g, f64 != nullptr);
    if (!ws || ws_bytes < f.bytes) return fail(GES_EWORKSPACE, "workspace too small (see ges_workspace_bytes)");
    ges_frame_status_t* status = status_dev ? status_dev : f.status;
    const int grid = st->supersample == 4 ? 2 : 1;
    const bool do_s = mode & 1;
    const bool do_g = (mode & 2) && st->layers != GES_LAYERS_SURFELS_ONLY;
    cudaError_t e;
    auto mark = [&](int k) {
        if (ev && ev[k]) cudaEventRecord((cudaEvent_t)ev[k], s);
    };
    mark(0);
    if ((e = cudaMemsetAsync(f.cnt_s, 0, f.zero_bytes, s)) != cudaSuccess) return cuda_fail(e, "memset counts");
    // the surfel preprocess zeroes the status word (it is first read by the scan); without
    // surfel work a memset does
    const bool prep_zeroes = (mode & 1) && sc->n_surfels > 0;
    if (!prep_zeroes && (e = cudaMemsetAsync(status, 0, sizeof(ges_frame_status_t), s)) != cudaSuccess)
        return cuda_fail(e, "memset status");
    mark(1);
    CamK cs = make_cam(*cam, grid), cg = make_cam(*cam, 1);
    const SlabMap slabs = slab_map(*sc, cs);
    const int tp = TILE * f.px;   // tile edge in base pixels
    Grid gs{cs.W, cs.H, tp * grid, f.ntx, f.nty, slabs}, gg{cg.W, cg.H, tp, f.ntx, f.nty, slabs};
    ges_scene_t scs = *sc;
    if (!do_s) scs.n_surfels = 0;
    if (!do_g) scs.n_gaussians = 0;
    auto log2i = [](int v) { int k = 0; while ((1 << k) < v) ++k; return k; };
    const BinPass bs{f.cnt_s, f.off_s, f.chunk_s, f.tickets, f.list_s, cap_s, f.ntiles, f.ntx, tp * grid,
                     log2i(tp * grid), (do_s && GES_TILE_ORDER) ? f.order : nullptr, f.tot};
    const BinPass bg{f.cnt_g, f.off_g, f.chunk_g, f.tickets + 32, f.list_g, cap_g, f.ntiles, f.ntx, tp, log2i(tp)};
    // both preprocesses of a full frame run concurrently: Gaussians on the side lane
    SideLane* lane = (do_s && do_g && scs.n_surfels && scs.n_gaussians) ? side_lane(s) : nullptr;
    cudaStream_t gs_stream = s;
    if (lane) {
        if ((e = cudaEventRecord(lane->fork, s)) != cudaSuccess || (e = cudaStreamWaitEvent(lane->side, lane->fork, 0)))
            return cuda_fail(e, "preprocess fork");
        gs_stream = lane->side;
    }
    if (do_s && (e = launch_surfel_prep(scs, cs, gs,
                                        PrepOut{f.srec, nullptr, f.cnt_s, nullptr, f.scull, prep_zeroes ? status : nullptr},
                                        s)))
        return cuda_fail(e, "surfel preprocess");
    if (do_g && (e = launch_gauss_prep(scs, cg, gg, *st, PrepOut{f.grec, f.g_nrm, f.cnt_g, nullptr, f.gcull},
                                       gs_stream)))
        return cuda_fail(e, "gaussian preprocess");
    if (lane) {
        if ((e = cudaEventRecord(lane->join, lane->side)) != cudaSuccess || (e = cudaStreamWaitEvent(s, lane->join, 0)))
            return cuda_fail(e, "preprocess join");
    }
    mark(2);
    if ((e = launch_scan(bs, bg, status, s)))
        return cuda_fail(e, "tile scan");
    mark(3);
    if ((e = launch_fill(f.scull, scs.n_surfels, bs, f.gcull, scs.n_gaussians, sc->gaussian_dim, bg, slabs, s)))
        return cuda_fail(e, "tile fill");
    mark(4);
    if (f64) {
        F64Launch L{};
        L.src = *f64->src;
        L.s_id = sc->s_id;
        L.ns = do_s ? sc->n_surfels : 0;
        L.ng = do_g ? sc->n_gaussians : 0;
        L.gdim = sc->gaussian_dim; L.deg = sc->sh_degree;
        L.mode = (do_s ? 1 : 0) | ((mode & 2) ? 2 : 0);
        L.layers = st->layers; L.geom = st->with_geometry; L.mip = st->mip;
        L.eps_const = st->epsilon_mode; L.eps_value = (double)st->epsilon_value;
        for (int i = 0; i < 3; ++i) L.bg[i] = (double)st->background[i];
        L.W = cam->width; L.H = cam->height; L.ntx = f.ntx; L.ntiles = f.ntiles; L.grid = grid;
        L.cs = cs; L.cg = cg;
        L.scull = f.scull; L.gcull = f.gcull; L.slabs = slabs; L.s_list = f.list_s; L.g_list = f.list_g; L.sbin = bs; L.gbin = bg;
        L.ds_in = f64->ds_in;
        L.out = *f64->out;
        L.records = f.rec64;
        L.status = status;
        if ((e = launch_f64(L, s))) return cuda_fail(e, "float64 tile kernel");
        mark(5);
        return GES_OK;
    }
    TileArgs a{};
    a.W = cam->width; a.H = cam->height; a.ntx = f.ntx; a.nty = f.nty;
    a.layers = st->layers;
    for (int i = 0; i < 3; ++i) a.bg[i] = (float)st->background[i];
    a.rcx = (float)cs.cx; a.rcy = (float)cs.cy; a.rifx = (float)(1.0 / cs.fx); a.rify = (float)(1.0 / cs.fy);
    a.srec = f.srec; a.scull = f.scull; a.s_list = f.list_s; a.sbin = bs;
    a.order = bs.order;
    a.s_sh = sc->s_sh; a.sh_deg = sc->sh_degree; a.sh_bytes = (sc->sh_degree + 1) * (sc->sh_degree + 1) * 12;
    for (int i = 0; i < 3; ++i) a.cpos[i] = cs.pos[i];
    a.s_quat = reinterpret_cast<const float4*>(sc->s_quat);
    a.s_pos = reinterpret_cast<const float4*>(sc->s_pos_s1);
    a.s_pack = sc->s_pack;
    for (int i = 0; i < 9; ++i) a.R[i] = cs.R[i];
    for (int i = 0; i < 3; ++i) a.t[i] = cs.t[i];
    a.slabs = slabs;
    a.gcx = (float)cg.cx; a.gcy = (float)cg.cy; a.gifx = (float)(1.0 / cg.fx); a.gify = (float)(1.0 / cg.fy);
    a.grec = f.grec; a.gcull = f.gcull; a.g_nrm = f.g_nrm; a.g_list = f.list_g; a.gbin = bg;
    a.ds_in = ds_in;
    a.out = *out;
    a.status = status;
    int tmode = (do_s ? 1 : 0) | (do_g ? 2 : 0);
    if (tmode == 0) tmode = 1;   // surfels_only + pass-2-only entry never happens; keep a valid mode
    if (mode == 2 && !do_g) {
        // accumulate_gaussians with layers=surfels_only still accumulates (forward.py:218-245
        // ignores layers); force the Gaussian pass.
        tmode = 2;
    }
    if ((e = launch_tile(a, st->supersample, f.px, tmode, sc->gaussian_dim, st->with_geometry != 0, s)))
        return cuda_fail(e, "tile kernel");
    mark(5);
    return GES_OK;
}

size_t backward_scratch_bytes(int64_t ng) { return al((size_t)ng * 16 * sizeof(double)) + al((size_t)ng * 32); }

ges_settings_t backward_settings(const ges_settings_t* st, bool geom) {
    ges_settings_t s2 = *st;
    s2.supersample = 1;        // the Gaussian pass runs at base resolution (training.py:315-326)
    s2.tile_mode = 1;          // 16 px tiles: the training forward's Gaussian pass uses them too
    s2.layers = GES_LAYERS_FULL;
    s2.with_geometry = geom;   // normals are only needed for a normal cotangent
    return s2;
}

}  // namespace

extern "C" {

int ges_abi_version(void) { return GES_ABI_VERSION; }

const char* ges_last_error(void) { return g_err.c_str(); }

size_t ges_scene_bytes(int64_t ns, int64_t ng, int32_t deg) {
    if (deg < 0 || deg > 3 || ns < 0 || ng < 0) return 0;
    size_t K = (size_t)(deg + 1) * (deg + 1);
    return al(ns * 16) + al(ns * 16) + al(ns * 4) + al(ns * K * 12) + al(ns * 4) * 2 + al(ng * 16) * 3 +
           al(ng * gsh_stride(deg) * 4);
}

int ges_scene_pack(const ges_scene_src_t* src, void* blob, size_t blob_bytes, ges_scene_t* out, void* stream) {
    if (!src || !out) return fail(GES_EINVAL, "NULL argument");
    if (src->sh_degree < 0 || src->sh_degree > 3) return fail(GES_EDEGREE, "SH degree must be in [0, 3]");
    if (src->gaussian_dim != 2 && src->gaussian_dim != 3) return fail(GES_EINVAL, "gaussian_dim must be 2 or 3");
    if (src->n_surfels < 0 || src->n_gaussians < 0) return fail(GES_EINVAL, "negative primitive count");
    size_t need = ges_scene_bytes(src->n_surfels, src->n_gaussians, src->sh_degree);
    if (blob_bytes < need || (need && !blob)) return fail(GES_EWORKSPACE, "scene blob too small");
    size_t ns = src->n_surfels, ng = src->n_gaussians, K = (size_t)(src->sh_degree + 1) * (src->sh_degree + 1);
    Carve c{static_cast<char*>(blob)};
    ges_scene_t sc{};
    sc.n_surfels = src->n_surfels; sc.n_gaussians = src->n_gaussians;
    sc.sh_degree = src->sh_degree; sc.gaussian_dim = src->gaussian_dim;
    sc.s_pos_s1 = c.take<float>(ns * 4);
    sc.s_quat = c.take<float>(ns * 4);
    sc.s_s2 = c.take<float>(ns);
    sc.s_sh = c.take<float>(ns * K * 3);
    sc.s_id = c.take<int32_t>(ns);
    sc.s_pack = c.take<int32_t>(ns);
    for (int k = 0; k < 7; ++k) sc.bounds[k] = src->bounds[k];
    sc.g_pos_op = c.take<float>(ng * 4);
    sc.g_quat = c.take<float>(ng * 4);
    sc.g_scale_eps = c.take<float>(ng * 4);
    sc.g_sh = c.take<float>(ng * gsh_stride(src->sh_degree));   // rows padded (ges_sh.cuh gsh_stride)
    cudaError_t e = launch_pack(*src, sc, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "scene pack");
    *out = sc;
    return GES_OK;
}

size_t ges_workspace_bytes(const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st,
                           int64_t cap_s, int64_t cap_g) {
    if (check_scene(sc) || check_cam(cam) || check_settings(st) || cap_s < 0 || cap_g < 0) return 0;
    return layout(nullptr, sc, cam, st, cap_s, cap_g).bytes;
}

int ges_render(const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st, const ges_outputs_t* out,
               void* ws, size_t ws_bytes, int64_t cap_s, int64_t cap_g, ges_frame_status_t* status_dev,
               void* stream) {
    return run_frame(sc, cam, st, out, nullptr, 3, ws, ws_bytes, cap_s, cap_g, status_dev, (cudaStream_t)stream);
}

int ges_render_profiled(const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st,
                        const ges_outputs_t* out, void* ws, size_t ws_bytes, int64_t cap_s, int64_t cap_g,
                        ges_frame_status_t* status_dev, void* stream, void* const* events) {
    return run_frame(sc, cam, st, out, nullptr, 3, ws, ws_bytes, cap_s, cap_g, status_dev, (cudaStream_t)stream,
                     events);
}

int ges_rasterize_surfels(const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st,
                          const ges_outputs_t* out, void* ws, size_t ws_bytes, int64_t cap_s,
                          ges_frame_status_t* status_dev, void* stream) {
    return run_frame(sc, cam, st, out, nullptr, 1, ws, ws_bytes, cap_s, 0, status_dev, (cudaStream_t)stream);
}

int ges_accumulate_gaussians(const ges_scene_t* sc, const ges_camera_t* cam, const float* surfel_depth,
                             const ges_settings_t* st, const ges_outputs_t* out, void* ws, size_t ws_bytes,
                             int64_t cap_g, ges_frame_status_t* status_dev, void* stream) {
    if (!surfel_depth) return fail(GES_EINVAL, "surfel_depth is NULL");
    ges_settings_t s2 = st ? *st : ges_settings_t{};
    s2.supersample = 1;   // the Gaussian pass always runs at base resolution (forward.py:411)
    if (st && s2.layers == GES_LAYERS_SURFELS_ONLY) s2.layers = GES_LAYERS_FULL;
    return run_frame(sc, cam, st ? &s2 : nullptr, out, surfel_depth, 2, ws, ws_bytes, 0, cap_g, status_dev,
                     (cudaStream_t)stream);
}

size_t ges_workspace_bytes_f64(const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st,
                               int64_t cap_s, int64_t cap_g) {
    if (check_scene(sc) || check_cam(cam) || check_settings(st) || cap_s < 0 || cap_g < 0) return 0;
    ges_settings_t s2 = *st;
    s2.tile_mode = 1;
    return layout(nullptr, sc, cam, &s2, cap_s, cap_g, true).bytes;
}

int ges_render_f64(const ges_scene_t* sc, const ges_scene_src_t* src, const ges_camera_t* cam,
                   const ges_settings_t* st, int32_t mode, const double* surfel_depth,
                   const ges_outputs_f64_t* out, void* ws, size_t ws_bytes, int64_t cap_s, int64_t cap_g,
                   ges_frame_status_t* status_dev, void* stream) {
    if (!src) return fail(GES_EINVAL, "float64 render needs the source scene");
    if (!out) return fail(GES_EINVAL, "outputs is NULL");
    if (mode < 1 || mode > 3) return fail(GES_EINVAL, "mode must be 1, 2 or 3");
    if (mode == 2 && !surfel_depth) return fail(GES_EINVAL, "mode 2 needs the surfel depth");
    if (sc && (src->n_surfels != sc->n_surfels || src->n_gaussians != sc->n_gaussians ||
               src->sh_degree != sc->sh_degree || src->gaussian_dim != sc->gaussian_dim))
        return fail(GES_EINVAL, "source scene does not match the packed scene");
    if (sc && ((sc->n_surfels && (!src->s_pos || !src->s_quat || !src->s_log_scale || !src->s_sh)) ||
               (sc->n_gaussians && (!src->g_pos || !src->g_raw_opacity || !src->g_quat || !src->g_log_scale ||
                                    !src->g_sh))))
        return fail(GES_EINVAL, "source scene arrays missing");
    F64Ctx ctx{src, out, surfel_depth};
    ges_settings_t s2 = st ? *st : ges_settings_t{};
    // accumulate_gaussians ignores `layers` (forward.py:218-245): mode 2 always accumulates
    if (mode == 2 && st && st->layers == GES_LAYERS_SURFELS_ONLY) s2.layers = GES_LAYERS_FULL;
    return run_frame(sc, cam, st ? &s2 : nullptr, nullptr, nullptr, mode, ws, ws_bytes, mode & 1 ? cap_s : 0,
                     mode & 2 ? cap_g : 0, status_dev, (cudaStream_t)stream, nullptr, &ctx);
}

int ges_composite_f64(const double* sc, const double* gc, const double* gw, double sw, double* img, int64_t n,
                      void* stream) {
    if (n < 0 || (n && (!sc || !gc || !gw || !img))) return fail(GES_EINVAL, "bad composite arguments");
    cudaError_t e = launch_composite64(sc, gc, gw, sw, img, n, (cudaStream_t)stream);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "composite");
}

int ges_smooth_geometry_f64(const double* sd, const double* sn, const double* gd, const double* gn, const double* gw,
                            double* d_out, double* n_out, int64_t n, void* stream) {
    if (n < 0 || (n && (!sd || !sn || !gd || !gn || !gw || !d_out || !n_out)))
        return fail(GES_EINVAL, "bad smooth_geometry arguments");
    cudaError_t e = launch_smooth64(sd, sn, gd, gn, gw, d_out, n_out, n, (cudaStream_t)stream);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "smooth_geometry");
}

int ges_composite(const float* sc, const float* gc, const float* gw, float sw, float* img, int64_t n, void* stream) {
    if (n < 0 || (n && (!sc || !gc || !gw || !img))) return fail(GES_EINVAL, "bad composite arguments");
    cudaError_t e = launch_composite(sc, gc, gw, sw, img, n, (cudaStream_t)stream);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "composite");
}

int ges_smooth_geometry(const float* sd, const float* sn, const float* gd, const float* gn, const float* gw,
                        float* d_out, float* n_out, int64_t n, void* stream) {
    if (n < 0 || (n && (!sd || !sn || !gd || !gn || !gw || !d_out || !n_out)))
        return fail(GES_EINVAL, "bad smooth_geometry arguments");
    cudaError_t e = launch_smooth(sd, sn, gd, gn, gw, d_out, n_out, n, (cudaStream_t)stream);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "smooth_geometry");
}

int ges_surfel_colors(const ges_scene_t* sc, const ges_camera_t* cam, float* rgb, void* stream) {
    int rc;
    if ((rc = check_scene(sc)) || (rc = check_cam(cam))) return rc;
    if (sc->n_surfels && !rgb) return fail(GES_EINVAL, "rgb is NULL");
    cudaError_t e = launch_surfel_colors(*sc, make_cam(*cam, 1), rgb, (cudaStream_t)stream);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "surfel colours");
}

size_t ges_backward_scratch_bytes(int64_t ng) { return ng < 0 ? 0 : backward_scratch_bytes(ng); }

size_t ges_backward_workspace_bytes(const ges_scene_t* sc, const ges_camera_t* cam, const ges_settings_t* st,
                                    int64_t cap_g) {
    if (check_scene(sc) || check_cam(cam) || check_settings(st) || cap_g < 0) return 0;
    const ges_settings_t s2 = backward_settings(st, true);
    return layout(nullptr, sc, cam, &s2, 0, cap_g).bytes;
}

int ges_backward_gaussians(const ges_scene_t* sc, const ges_scene_src_t* src, int32_t any_filter,
                           const ges_camera_t* cam, const ges_settings_t* st, const float* surfel_depth,
                           const float* g_color, const float* g_weight, const float* g_depth, const float* g_normal,
                           const ges_gauss_grads_t* grads, void* scratch, size_t scratch_bytes, void* ws,
                           size_t ws_bytes, int64_t cap_g, ges_frame_status_t* status_dev, void* stream) {
    int rc;
    if ((rc = check_scene(sc)) || (rc = check_cam(cam)) || (rc = check_settings(st))) return rc;
    if (!src || !grads) return fail(GES_EINVAL, "NULL argument");
    if (src->n_gaussians != sc->n_gaussians || src->gaussian_dim != sc->gaussian_dim ||
        src->sh_degree != sc->sh_degree)
        return fail(GES_EINVAL, "source arrays do not match the packed scene");
    const int64_t ng = sc->n_gaussians;
    if (ng == 0) return GES_OK;
    if (!surfel_depth || !g_color || !g_weight) return fail(GES_EINVAL, "surfel_depth/g_color/g_weight is NULL");
    if (!src->g_pos || !src->g_quat || !src->g_log_scale || !src->g_raw_opacity || !src->g_sh)
        return fail(GES_EINVAL, "source Gaussian arrays are NULL");
    if (!grads->pos || !grads->opacity || !grads->quat || !grads->scale || !grads->sh)
        return fail(GES_EINVAL, "gradient outputs are NULL");
    if (cap_g < 0 || cap_g >= (1ll << 32)) return fail(GES_EINVAL, "pair capacity out of range");
    if (!scratch || scratch_bytes < backward_scratch_bytes(ng)) return fail(GES_EWORKSPACE, "scratch too small");
    // a normal cotangent reaches 3D Gaussians only when the frame has their
    // normals (training.py:661-664); planar ones always carry n_vis (:736-743)
    const bool geom = g_normal && (sc->gaussian_dim == 2 || st->with_geometry);
    const ges_settings_t s2 = backward_settings(st, geom);
    Frame f = layout(ws, sc, cam, &s2, 0, cap_g);
    if (!ws || ws_bytes < f.bytes) return fail(GES_EWORKSPACE, "workspace too small (see ges_backward_workspace_bytes)");
    cudaStream_t s = (cudaStream_t)stream;
    ges_frame_status_t* status = status_dev ? status_dev : f.status;
    double* acc = static_cast<double*>(scratch);
    float4* aux = reinterpret_cast<float4*>(static_cast<char*>(scratch) + al((size_t)ng * 16 * sizeof(double)));
    cudaError_t e;
    if ((e = cudaMemsetAsync(f.cnt_s, 0, f.zero_bytes, s)) != cudaSuccess) return cuda_fail(e, "memset counts");
    if ((e = cudaMemsetAsync(status, 0, sizeof(ges_frame_status_t), s)) != cudaSuccess)
        return cuda_fail(e, "memset status");
    if ((e = cudaMemsetAsync(acc, 0, (size_t)ng * 16 * sizeof(double), s)) != cudaSuccess)
        return cuda_fail(e, "memset accumulators");
    const CamK cg = make_cam(*cam, 1);
    const SlabMap slabs = slab_map(*sc, cg);
    Grid gg{cg.W, cg.H, TILE, f.ntx, f.nty, slabs};
    ges_scene_t scs = *sc;
    scs.n_surfels = 0;
    const BinPass bs{f.cnt_s, f.off_s, f.chunk_s, f.tickets, f.list_s, 0, f.ntiles, f.ntx, TILE, 4};
    const BinPass bg{f.cnt_g, f.off_g, f.chunk_g, f.tickets + 32, f.list_g, cap_g, f.ntiles, f.ntx, TILE, 4};
    PrepOut po{f.grec, f.g_nrm, f.cnt_g, sc->gaussian_dim == 2 ? aux : nullptr, f.gcull};
    if ((e = launch_gauss_prep(scs, cg, gg, s2, po, s))) return cuda_fail(e, "gaussian preprocess");
    if ((e = launch_scan(bs, bg, status, s))) return cuda_fail(e, "tile scan");
    if ((e = launch_fill(f.scull, 0, bs, f.gcull, ng, sc->gaussian_dim, bg, slabs, s))) return cuda_fail(e, "tile fill");
    BwdArgs a{};
    a.W = cam->width; a.H = cam->height; a.ntx = f.ntx; a.nty = f.nty;
    a.grec = f.grec; a.gcull = f.gcull; a.aux = aux; a.g_nrm = f.g_nrm; a.g_list = f.list_g; a.gbin = bg; a.slabs = slabs;
    a.ds = surfel_depth; a.g_cg = g_color; a.g_wg = g_weight; a.g_gd = g_depth; a.g_gn = geom ? g_normal : nullptr;
    a.gcx = (float)cg.cx; a.gcy = (float)cg.cy; a.gifx = (float)(1.0 / cg.fx); a.gify = (float)(1.0 / cg.fy);
    a.acc = acc;
    a.status = status;
    if ((e = launch_gauss_bwd(a, sc->gaussian_dim, geom, s))) return cuda_fail(e, "gaussian backward");
    if ((e = launch_gauss_finish(*src, any_filter, st->mip, cg, acc, *grads, s)))
        return cuda_fail(e, "gaussian backward finish");
    return GES_OK;
}

int ges_frozen_surfel_buffers(const int32_t* winner, const float* depth, const float* normal, const float* colors,
                              int32_t width, int32_t height, int32_t grid, const float* background, float* s_color,
                              float* s_depth, float* b_depth, float* b_normal, void* stream) {
    if (grid != 1 && grid != 2) return fail(GES_EINVAL, "grid must be 1 or 2");
    if (width <= 0 || height <= 0) return fail(GES_EINVAL, "image size out of range");
    if (!winner || !depth || !colors || !background || !s_color || !s_depth || (b_normal && !normal))
        return fail(GES_EINVAL, "NULL argument");
    cudaError_t e = launch_frozen_resolve(winner, depth, normal, colors, width, height, grid, background, s_color,
                                          s_depth, b_depth, b_normal, (cudaStream_t)stream);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "frozen surfel buffers");
}

int ges_gaussian_contributions(const ges_scene_t* sc, const ges_scene_src_t* src, const ges_camera_t* cam,
                               const ges_settings_t* st, const float* surfel_depth, const float* g_weight,
                               float* scores, void* ws, size_t ws_bytes, int64_t cap_g,
                               ges_frame_status_t* status_dev, void* stream) {
    int rc;
    if ((rc = check_scene(sc)) || (rc = check_cam(cam)) || (rc = check_settings(st))) return rc;
    const int64_t ng = sc->n_gaussians;
    if (ng == 0) return GES_OK;
    if (!surfel_depth || !g_weight || !scores) return fail(GES_EINVAL, "surfel_depth/g_weight/scores is NULL");
    if (src && src->n_gaussians != ng) return fail(GES_EINVAL, "source arrays do not match the packed scene");
    if (cap_g < 0 || cap_g >= (1ll << 32)) return fail(GES_EINVAL, "pair capacity out of range");
    const ges_settings_t s2 = backward_settings(st, false);
    Frame f = layout(ws, sc, cam, &s2, 0, cap_g);
    if (!ws || ws_bytes < f.bytes) return fail(GES_EWORKSPACE, "workspace too small (see ges_backward_workspace_bytes)");
    cudaStream_t s = (cudaStream_t)stream;
    ges_frame_status_t* status = status_dev ? status_dev : f.status;
    cudaError_t e;
    if ((e = cudaMemsetAsync(f.cnt_s, 0, f.zero_bytes, s)) != cudaSuccess) return cuda_fail(e, "memset counts");
    if ((e = cudaMemsetAsync(status, 0, sizeof(ges_frame_status_t), s)) != cudaSuccess)
        return cuda_fail(e, "memset status");
    const CamK cg = make_cam(*cam, 1);
    const SlabMap slabs = slab_map(*sc, cg);
    Grid gg{cg.W, cg.H, TILE, f.ntx, f.nty, slabs};
    ges_scene_t scs = *sc;
    scs.n_surfels = 0;
    const BinPass bs{f.cnt_s, f.off_s, f.chunk_s, f.tickets, f.list_s, 0, f.ntiles, f.ntx, TILE, 4};
    const BinPass bg{f.cnt_g, f.off_g, f.chunk_g, f.tickets + 32, f.list_g, cap_g, f.ntiles, f.ntx, TILE, 4};
    PrepOut po{f.grec, f.g_nrm, f.cnt_g, nullptr, f.gcull};
    if ((e = launch_gauss_prep(scs, cg, gg, s2, po, s))) return cuda_fail(e, "gaussian preprocess");
    if ((e = launch_scan(bs, bg, status, s))) return cuda_fail(e, "tile scan");
    if ((e = launch_fill(f.scull, 0, bs, f.gcull, ng, sc->gaussian_dim, bg, slabs, s))) return cuda_fail(e, "tile fill");
    BwdArgs a{};
    a.W = cam->width; a.H = cam->height; a.ntx = f.ntx; a.nty = f.nty;
    a.grec = f.grec; a.gcull = f.gcull; a.g_nrm = f.g_nrm; a.g_list = f.list_g; a.gbin = bg; a.slabs = slabs;
    a.ds = surfel_depth; a.g_wg = g_weight;
    a.gcx = (float)cg.cx; a.gcy = (float)cg.cy; a.gifx = (float)(1.0 / cg.fx); a.gify = (float)(1.0 / cg.fy);
    a.scores = scores;
    a.order = src ? src->g_order : nullptr;
    a.status = status;
    if ((e = launch_gauss_contrib(a, sc->gaussian_dim, s))) return cuda_fail(e, "gaussian contributions");
    return GES_OK;
}

int ges_backward_surfels_frozen(const ges_scene_src_t* src, const ges_camera_t* cam, int32_t grid,
                                const int32_t* winner, const float* g_color, double* col, double* g_sh,
                                double* g_pos, void* stream) {
    int rc;
    if ((rc = check_cam(cam))) return rc;
    if (!src) return fail(GES_EINVAL, "src is NULL");
    if (grid != 1 && grid != 2) return fail(GES_EINVAL, "grid must be 1 or 2");
    if (src->sh_degree < 0 || src->sh_degree > 3) return fail(GES_EDEGREE, "SH degree must be in [0, 3]");
    if (src->n_surfels == 0) return GES_OK;
    if (!winner || !g_color || !col || !g_sh || !g_pos || !src->s_pos || !src->s_sh)
        return fail(GES_EINVAL, "NULL argument");
    cudaError_t e = launch_frozen_bwd(*src, make_cam(*cam, 1), cam->width, cam->height, grid, winner, g_color, col,
                                      g_sh, g_pos, (cudaStream_t)stream);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "frozen surfel backward");
}

int ges_peer_alloc(size_t bytes, void** dev_ptr, void* ipc_handle) {
    if (!dev_ptr || !ipc_handle || bytes == 0) return fail(GES_EINVAL, "bad peer_alloc arguments");
    cudaError_t e = cudaMalloc(dev_ptr, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "peer buffer cudaMalloc");
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, *dev_ptr)) != cudaSuccess) {
        cudaFree(*dev_ptr);
        *dev_ptr = nullptr;
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(ipc_handle, &h, sizeof(h));
    return GES_OK;
}

int ges_peer_free(void* dev_ptr) {
    cudaError_t e = cudaFree(dev_ptr);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "peer buffer cudaFree");
}

int ges_peer_open(const void* ipc_handle, int32_t device, void** dev_ptr) {
    if (!ipc_handle || !dev_ptr) return fail(GES_EINVAL, "bad peer_open arguments");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    cudaSetDevice(prev);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

int ges_peer_close(void* dev_ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    return e == cudaSuccess ? GES_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

int ges_debug_stats(uint64_t* out24) {
    if (!out24) return fail(GES_EINVAL, "NULL argument");
    if (read_stats(reinterpret_cast<unsigned long long*>(out24))) return fail(GES_ECUDA, "stats copy failed");
    return GES_OK;
}

int ges_render_views_host(const ges_scene_t* sc, const ges_camera_t* host_cams, int32_t n_views,
                          const ges_settings_t* st, int32_t format, void* host_images, int32_t n_lanes,
                          void* const* workspaces, size_t ws_bytes, int64_t cap_s, int64_t cap_g, void* image_dev,
                          ges_frame_status_t* status_dev, void* const* streams, void* copy_stream) {
    if (!host_cams || !host_images || !image_dev || n_views < 0 || !copy_stream || n_lanes < 1 || !workspaces ||
        !streams)
        return fail(GES_EINVAL, "bad view batch arguments");
    if (format != GES_IMAGE_F32_RGB && format != GES_IMAGE_RGBA8) return fail(GES_EINVAL, "unknown image format");
    if (n_views == 0) return GES_OK;
    for (int v = 1; v < n_views; ++v)
        if (host_cams[v].width != host_cams[0].width || host_cams[v].height != host_cams[0].height)
            return fail(GES_EINVAL, "all views of a batch must share one resolution");
    cudaStream_t cs = (cudaStream_t)copy_stream;
    const size_t px = (size_t)host_cams[0].width * host_cams[0].height;
    const size_t bytes = px * (format == GES_IMAGE_RGBA8 ? 4 : 3 * sizeof(float));
    const int nb = 2 * n_lanes;   // image buffers: two per lane
    cudaEvent_t rendered[64], copied[64];
    if (nb > 64) return fail(GES_EINVAL, "at most 32 lanes");
    for (int k = 0; k < nb; ++k) {
        cudaEventCreateWithFlags(&rendered[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming);
    }
    int rc = GES_OK;
    for (int v = 0; v < n_views && rc == GES_OK; ++v) {
        const int lane = v % n_lanes;
        const int b = (v / n_lanes) % 2 * n_lanes + lane;   // buffer of this (lane, parity)
        cudaStream_t s = (cudaStream_t)streams[lane];
        char* buf = static_cast<char*>(image_dev) + b * bytes;
        if (v >= nb) cudaStreamWaitEvent(s, copied[b], 0);   // buffer b free again
        ges_outputs_t out{};
        if (format == GES_IMAGE_RGBA8) out.image_rgba8 = reinterpret_cast<uint8_t*>(buf);
        else out.image = reinterpret_cast<float*>(buf);
        rc = ges_render(sc, &host_cams[v], st, &out, workspaces[lane], ws_bytes, cap_s, cap_g,
                        status_dev ? status_dev + v : nullptr, s);
        if (rc) break;
        cudaEventRecord(rendered[b], s);
        cudaStreamWaitEvent(cs, rendered[b], 0);
        cudaError_t e = cudaMemcpyAsync(static_cast<char*>(host_images) + v * bytes, buf, bytes,
                                        cudaMemcpyDeviceToHost, cs);
        if (e != cudaSuccess) rc = cuda_fail(e, "image copy");
        cudaEventRecord(copied[b], cs);
    }
    for (int l = 0; l < n_lanes; ++l)   // later work on the lanes may reuse image_dev
        for (int k = 0; k < nb; ++k) cudaStreamWaitEvent((cudaStream_t)streams[l], copied[k], 0);
    for (int k = 0; k < nb; ++k) {      // destroy is deferred by the driver until complete
        cudaEventDestroy(rendered[k]);
        cudaEventDestroy(copied[k]);
    }
    return rc;
}

}  // extern "C"
