// Host-side launchers shared between the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include "ges_common.cuh"

namespace ges {

// Programmatic dependent launch (Hopper/Blackwell): the scan -> fill -> tile
// kernels of a frame are launched so the next one's launch overlaps the
// previous one's last CTAs; each dependent waits (griddepcontrol.wait) before
// its first read of the previous kernel's output.
#ifndef GES_PDL
#define GES_PDL 1
#endif
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (GES_PDL) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct PrepOut {
    void* rec;              // SurfRec / GaussRec / Gauss2Rec per primitive
    float4* nrm;            // per-primitive camera-facing normal (surfels; Gaussians if geometry)
    uint32_t* bin_count;    // per-(tile, slab) pair counters (zeroed by the caller)
    float4* aux;            // 2D Gaussians, training backward only: (a1/s1).d and (a2/s2).d
                            // as affine functions of the pixel (2 per Gaussian), or NULL
    float4* cull;           // dense cull records (see SurfRec, GaussRec)
    ges_frame_status_t* zero_status;   // or NULL: zeroed by the kernel's first thread (replaces a memset)
};

// Tile grid for the pass: ntx x nty tiles of `tile_px` pixels at resolution W x H.
struct Grid {
    int W, H, tile_px, ntx, nty;
    SlabMap slabs;
};

CamK make_cam(const ges_camera_t& c, int scale);

cudaError_t launch_pack(const ges_scene_src_t& src, const ges_scene_t& dst, cudaStream_t s);
cudaError_t launch_surfel_prep(const ges_scene_t& sc, const CamK& cam, const Grid& g,
                               const PrepOut& o, cudaStream_t s);
cudaError_t launch_gauss_prep(const ges_scene_t& sc, const CamK& cam, const Grid& g,
                              const ges_settings_t& st, const PrepOut& o, cudaStream_t s);
cudaError_t launch_scan(const BinPass& s, const BinPass& g, ges_frame_status_t* status, cudaStream_t st);
cudaError_t launch_fill(const float4* scull, int64_t ns, const BinPass& ps, const float4* gcull, int64_t ng, int g_kind,
                        const BinPass& pg, const SlabMap& sm, cudaStream_t s);

struct TileArgs {
    int W, H, ntx, nty;           // base resolution and 16x16 tile grid
    int layers;
    float bg[3];
    // surfel pass (resolution = ss * base)
    float rcx, rcy, rifx, rify;   // principal point and 1/f of the surfel pass
    const SurfRec* srec;
    const float4* scull;          // dense surfel cull records
    const uint32_t* order;        // tile launch order (by descending surfel pairs), or NULL
    const float* s_sh;            // packed SH (deferred colour of winners)
    int sh_deg, sh_bytes;
    double cpos[3];               // camera centre (world)
    const float4 *s_quat, *s_pos; // packed scene (n_vis of winners, on demand)
    const int32_t* s_pack;        // source id -> packed index
    double R[9], t[3];            // world -> camera
    const uint32_t* s_list;
    BinPass sbin;                 // tile offsets; cnt = per-(tile, slab) ends relative to the tile
    // Gaussian pass (base resolution)
    float gcx, gcy, gifx, gify;
    const void* grec;
    const float4* gcull;          // dense Gaussian cull records
    const float4* g_nrm;          // with_geometry normals
    const uint32_t* g_list;
    BinPass gbin;
    SlabMap slabs;
    const float* ds_in;           // external surfel depth (pass-2-only entry)
    ges_outputs_t out;
    const ges_frame_status_t* status;
};

// mode: 1 = surfels only, 2 = Gaussians only (external depth), 3 = both;
// px: base pixels per thread per axis (1: 16x16 tiles, 2: 32x32 tiles).
cudaError_t launch_tile(const TileArgs& a, int ss, int px, int mode, int g_kind, bool geom, cudaStream_t s);

int read_stats(unsigned long long* out);   // 16 counters, then reset (GES_STATS builds)

cudaError_t launch_composite(const float* sc, const float* gc, const float* gw, float sw, float* img,
                             int64_t n, cudaStream_t s);
cudaError_t launch_smooth(const float* sd, const float* sn, const float* gd, const float* gn,
                          const float* gw, float* d_out, float* n_out, int64_t n, cudaStream_t s);

// ---------------------------------------------------------------- float64 mode (ges_f64.cu)
struct F64Launch {
    ges_scene_src_t src;
    const int32_t* s_id;          // packed -> source surfel
    int64_t ns, ng;
    int gdim, deg, mode, layers, geom, mip, eps_const;
    double eps_value;
    double bg[3];
    int W, H, ntx, ntiles, grid;
    CamK cs, cg;
    const float4 *scull, *gcull;
    const uint32_t *s_list, *g_list;
    BinPass sbin, gbin;
    SlabMap slabs;
    const double* ds_in;
    ges_outputs_f64_t out;
    void* records;                // f64_record_bytes(ns, ng, gdim)
    const ges_frame_status_t* status;
};
size_t f64_record_bytes(int64_t ns, int64_t ng, int gdim);
cudaError_t launch_f64(const F64Launch& L, cudaStream_t s);
cudaError_t launch_composite64(const double* sc, const double* gc, const double* gw, double sw, double* img,
                               int64_t n, cudaStream_t s);
cudaError_t launch_smooth64(const double* sd, const double* sn, const double* gd, const double* gn, const double* gw,
                            double* d_out, double* n_out, int64_t n, cudaStream_t s);

// ---------------------------------------------------------------- training (ges_train.cu)
struct BwdArgs {
    int W, H, ntx, nty;           // base resolution, 16x16 tiles
    const void* grec;
    const float4* gcull;
    const float4* aux;            // 2D: (k1, k2) affine coefficients per Gaussian
    const float4* g_nrm;          // normal cotangent given: camera-facing normals
    const uint32_t* g_list;
    BinPass gbin;
    SlabMap slabs;
    const float *ds, *g_cg, *g_wg, *g_gd, *g_gn;   // gd, gn may be NULL
    float gcx, gcy, gifx, gify;
    double* acc;                  // 16 float64 partial sums per packed Gaussian
    float* scores;                // contribution mode: per-source-Gaussian max
    const int32_t* order;         // packed -> source index (NULL = identity)
    const ges_frame_status_t* status;
};

cudaError_t launch_surfel_colors(const ges_scene_t& sc, const CamK& cam, float* rgb, cudaStream_t s);
cudaError_t launch_gauss_bwd(const BwdArgs& a, int g_kind, bool geom, cudaStream_t s);
cudaError_t launch_frozen_resolve(const int32_t* winner, const float* depth, const float* normal, const float* colors,
                                  int W, int H, int grid, const float* bg, float* s_color, float* s_depth,
                                  float* b_depth, float* b_normal, cudaStream_t s);
cudaError_t launch_gauss_contrib(const BwdArgs& a, int g_kind, cudaStream_t s);
cudaError_t launch_gauss_finish(const ges_scene_src_t& src, int any_filter, int mip, const CamK& cam,
                                const double* acc, const ges_gauss_grads_t& out, cudaStream_t s);
cudaError_t launch_frozen_bwd(const ges_scene_src_t& src, const CamK& cam, int W, int H, int grid,
                              const int32_t* winner, const float* g_cs, double* col, double* g_sh, double* g_pos,
                              cudaStream_t s);

}  // namespace ges
