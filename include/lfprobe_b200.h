/*
 * lfprobe_b200.h -- C ABI of the B200 probe-grid tracer (sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path
 *   render_frame(ProbeGrid, Camera)          pkg/src/lfprobe/render.py:102-153
 *     -> kernels.render_grid(...)            pkg/src/lfprobe/kernels.py:825-843
 *        -> trace_grid_ray(...)              pkg/src/lfprobe/kernels.py:653-822
 * The reference crosses Python -> numba native code exactly once, at
 * render.py:132-136; these entry points are what that call site binds to
 * instead (see INTEGRATION.md for the ctypes binding).
 *
 * Conventions
 *  - plain C types only; every pointer is caller-owned unless stated;
 *  - array layouts are the reference's (C-contiguous, [ty][tx] texels);
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *  - every call returns LFP_OK (0) or a negative error code and never
 *    throws; lfp_last_error() returns a thread-local message;
 *  - probe sets are immutable after creation and may be used by concurrent
 *    renders on different streams / host threads (the reference kernel is
 *    pure over immutable inputs and is called concurrently by the service,
 *    service.py:136, 189).
 */
#ifndef LFPROBE_B200_H
#define LFPROBE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFP_OK 0
#define LFP_ERR_INVALID -1   /* bad argument (shape, null pointer, dims) */
#define LFP_ERR_CUDA -2      /* CUDA runtime error                       */
#define LFP_ERR_NOMEM -3     /* device allocation failed                 */

/* status codes, kernels.py:18-20 */
#define LFP_MISS 0
#define LFP_HIT 1
#define LFP_UNKNOWN 2

/* lfp_probeset_create flags */
#define LFP_SRC_DEVICE 0x1u     /* source pointers are device pointers       */
#define LFP_FMT_AUTO_HALF 0x2u  /* store dir/irr as half4 when lossless      */
#define LFP_FMT_FORCE_F32 0x4u  /* never compress payloads                   */

typedef struct lfp_probeset lfp_probeset;

/* Trace parameters: grid geometry (grid.py:48-93) + TraceConfig
 * (trace.py:32-40). */
typedef struct {
    double grid_origin[3];
    double cell;            /* scalar cubic cell (grid.py:51-57)          */
    int32_t nx, ny, nz;     /* probe counts per axis                      */
    double eps_start;       /* default 1e-4 (kernels.py:25)               */
    double eps_align;       /* default 1e-4 (kernels.py:27)               */
    double slack;           /* default 1e-3 (kernels.py:23)               */
    int32_t trace_mode;     /* 0 = filtered (default): fp32 decision filters
                               with exact fp64 fallback, outputs identical to
                               the reference; 1 = exact fp64 on every step;
                               2 = filtered + re-check of every filtered
                               decision (counts into lfp_outputs.diag)    */
    int32_t schedule;       /* 0 = entry point default (cameras: nested;
                               explicit rays: wavefront from 2^21 rays,
                               persistent below); 1 = nested: one thread
                               per ray; 2 = persistent: flattened per-lane
                               state machine, lanes pull rays from a global
                               counter; 3 = wavefront (explicit rays): one
                               probe trace per ray per launch, rays
                               re-sorted by (probe, chord ends) between
                               launches; blocks the calling thread        */
    int32_t min_active;     /* persistent: keep stepping while >= this many
                               lanes of a warp step (1..32, 0 = 16)      */
} lfp_grid_params;

/* Pinhole camera (render.py:24-62). `basis` = (right, up, forward) exactly
 * as Camera.basis() returns them; tan_v = tan(radians(vfov)/2),
 * tan_h = tan_v * width / height, all computed on the host. */
typedef struct {
    double eye[3];
    double basis[9];
    double tan_v, tan_h;
} lfp_camera;

/* Per-ray outputs; any pointer may be NULL to skip that output.
 *  status u8[n]      MISS / HIT / UNKNOWN (grid mode never yields UNKNOWN)
 *  rgb    f32[n*3]   see rgb_mode
 *  probe  i32[n]     hit probe, or last-UNKNOWN probe diagnostic, or -1
 *  texel  i32[n]     tx | (ty << 16) of that probe texel, or -1
 *  fetch  i32[n]     reference-equivalent texel fetch count (K:216,341,443,628)
 *  hit_t  f32[n]     HIT: (origin_p + dist_hi[p,ty,tx] * v_texel - eye) . d,
 *                    else +inf (SURVEY.md §8(c) hit-distance definition)
 *  stats  u64[4]     accumulated: {sum fetch, #MISS, #UNKNOWN, #HIT}
 * rgb_mode 0 = frame fill (render.py:147-149): HIT radiance, MISS
 * `background`, UNKNOWN `unknown_color`; rgb_mode 1 = kernel semantics
 * (kernels.py:840-843): only HIT rows are written.
 *  rgb8   u8[n*3]    (optional) the frame-filled colour as Frame.rgb8
 *                    (render.py:70-73): clip(rint(c * 255), 0, 255) --
 *                    what the service PNG-encodes (service.py:101-104) */
typedef struct {
    uint8_t* status;
    float* rgb;
    int32_t* probe;
    int32_t* texel;
    int32_t* fetch;
    float* hit_t;
    unsigned long long* stats;
    unsigned long long* diag;   /* u64[11]: low-res decisions taken by the
                                   filter / by the exact path, hi-res ditto,
                                   filter-vs-exact disagreements (mode 2),
                                   low-res steps cleared by the segment
                                   bound, (reserved, 0), segments traced,
                                   fp32 classification outcomes (march,
                                   occluder, candidate)                   */
    int32_t rgb_mode;
    float background[3];
    float unknown_color[3];
    uint8_t* rgb8;
} lfp_outputs;

/* Library version (major*10000 + minor*100 + patch). */
int lfp_version(void);

/* Thread-local message of the last failing call on this thread. */
const char* lfp_last_error(void);

/* Kernels launched by this thread's last lfp_trace_rays /
 * lfp_trace_rays_ordered / lfp_render_grid call (the wavefront schedule
 * launches one per iteration; the others one). */
int64_t lfp_last_launches(void);

/* Upload + relayout a ProbeSet (grid.py:19-45 arrays):
 *   dist_hi f32[P][R][R], dir_hi f32[P][R][R][3], irr_hi f32[P][R][R][3],
 *   dist_lo f32[P][r][r], origins f64[P][3]
 * into device-resident tracing layouts on `device` (pre-dilated low-res
 * MIN, float4/half4 payloads, texel-centre direction table). Replaces the
 * per-call array hand-off of render.py:132-136 / grid.py:76-80. */
int lfp_probeset_create(int device, const float* dist_hi, const float* dir_hi,
                        const float* irr_hi, const float* dist_lo,
                        const double* origins, int64_t P, int32_t R,
                        int32_t r, uint32_t flags, void* stream,
                        lfp_probeset** out);

/* Same, straight from the .lfp payload sections (bake.py:228-341): per
 * probe (concatenated over P probes, host memory) irradiance RGB565
 * u16[R][R], distance f16[R][R], direction 2 x u8 sub-texel offsets
 * [R][R][2], low-res distance f16[r][r]; origins f64[P][3] may be host or
 * device (`origins` of lfp_probeset_create also accepts either). Uploads 6 B
 * per texel instead of 28 and decodes on the device exactly as load_probe
 * does (f32 RGB565 division, fp64 sub-texel oct_decode, EMPTY texels
 * zeroed). The decoded reference-layout arrays are also written to the
 * optional host buffers (for the Python ProbeSet mirror). Replaces
 * load_probe / load_grid's host decode (bake.py:301-341, grid.py:268-274). */
int lfp_probeset_create_packed(int device, const uint16_t* irr565,
                               const uint16_t* dist_f16, const uint8_t* dir_q8,
                               const uint16_t* dist_lo_f16,
                               const double* origins, int64_t P, int32_t R,
                               int32_t r, uint32_t flags, float* host_dist_hi,
                               float* host_dir_hi, float* host_irr_hi,
                               float* host_dist_lo, void* stream,
                               lfp_probeset** out);

int lfp_probeset_destroy(lfp_probeset* ps);

/* Device bytes held by the probe set, and which payload formats it chose. */
int lfp_probeset_info(const lfp_probeset* ps, int64_t* device_bytes,
                      int32_t* dir_half, int32_t* irr_half);

/* render_frame(ProbeGrid, Camera) for a batch of cameras sharing one
 * resolution (render.py:102-153; ray generation render.py:50-62 fused in).
 * The frame is cut into 8x16-pixel tiles numbered camera-major, row-major;
 * this call traces tiles tile_begin, tile_begin + tile_step, ... (n_tiles of
 * them). compact == 0: outputs are indexed like the frames,
 * cam * H * W + y * W + x (arrays sized n_cams * H * W). compact == 1:
 * outputs are indexed local_tile * 128 + (y % 16) * 8 + (x % 8) (arrays
 * sized n_tiles * 128; pixels past the frame edge are left untouched) --
 * the per-GPU shard layout gathered by lfp_untile. */
int lfp_render_cameras(const lfp_probeset* ps, const lfp_grid_params* grid,
                       const lfp_camera* cams_host, int32_t n_cams,
                       int32_t width, int32_t height, int64_t tile_begin,
                       int64_t tile_step, int64_t n_tiles, int32_t compact,
                       const lfp_outputs* out, void* stream);

/* render_frame(ProbeGrid, Camera) end to end for one camera: ray
 * generation, trace and shade as lfp_render_cameras, plus the copy of the
 * frame into caller HOST buffers (page-locked memory recommended). The
 * frame is traced in row bands on two internal streams and each band is
 * copied while later bands trace, so only the last band's copy is exposed.
 * Blocks until the frame is on the host. host_status (u8 H*W), host_rgb
 * (f32 H*W*3: HIT radiance, MISS background, UNKNOWN unknown_color) and
 * host_rgb8 (u8 H*W*3, Frame.rgb8) may each be NULL; stats_out (u64[4]) =
 * fetch sum, MISS, UNKNOWN, HIT counts; trace_ms_out = device time from the
 * first band's start to the last band's end. Work is ordered after what is
 * queued on `stream`, and later work on `stream` after this frame. */
int lfp_render_frame_host(const lfp_probeset* ps, const lfp_grid_params* grid,
                          const lfp_camera* cam, int32_t width, int32_t height,
                          const float* background, const float* unknown_color,
                          uint8_t* host_status, float* host_rgb,
                          uint8_t* host_rgb8, uint64_t* stats_out,
                          float* trace_ms_out, void* stream);

/* render_frame for the non-grid sources (render.py:118-144), same camera
 * batching, frame-ordered outputs:
 *  LFP_SOURCE_SINGLE  one probe, full marching over the padded bounds
 *                     (render_single_probe, kernels.py:567-596)
 *  LFP_SOURCE_FEW     a probe list in nearest-first `order` (stable by
 *                     squared eye distance, computed by the caller) with
 *                     MISS/UNKNOWN fall-through over the padded union bounds
 *                     (render_few_probes, kernels.py:846-892; returns UNKNOWN)
 *  LFP_SOURCE_LOOKUP  eye at the probe: one octahedral lookup per pixel
 *                     (_lookup_render, render.py:86-99)
 * The probe set holds 1 probe for SINGLE / LOOKUP. Only eps_start,
 * eps_align, slack and trace_mode of `params` are used. */
#define LFP_SOURCE_SINGLE 1
#define LFP_SOURCE_FEW 2
#define LFP_SOURCE_LOOKUP 3
int lfp_render_probes(const lfp_probeset* ps, int32_t source_kind,
                      const int32_t* order, int32_t n_order,
                      const double* bounds_lo, const double* bounds_hi,
                      const lfp_grid_params* params, const lfp_camera* cams_host,
                      int32_t n_cams, int32_t width, int32_t height,
                      const lfp_outputs* out, void* stream);

/* Coarse-to-fine probe hierarchy (config 4): up to 4 probe-grid levels on
 * one device, each with its own lattice (grids[l]); every pixel ray is traced
 * through level 0 (kernels.py:653-822), a MISS falls through to level 1, and
 * so on; the first HIT wins. fetch = sum over the levels tried; the probe
 * output is (level << 24) | probe (HIT, or the last MISS diagnostic); texel,
 * rgb, hit_t refer to that level's probe. Same tiling / compact layout as
 * lfp_render_cameras; all levels share grids[0].trace_mode. */
int lfp_render_hierarchy(const lfp_probeset* const* levels,
                         const lfp_grid_params* grids, int32_t n_levels,
                         const lfp_camera* cams_host, int32_t n_cams,
                         int32_t width, int32_t height, int64_t tile_begin,
                         int64_t tile_step, int64_t n_tiles, int32_t compact,
                         const lfp_outputs* out, void* stream);

/* Number of 8x16 tiles of a batch of n_cams frames of width x height. */
int64_t lfp_num_tiles(int32_t n_cams, int32_t width, int32_t height);

/* kernels.render_grid (kernels.py:825-843): one shared eye, explicit unit
 * directions dirs[n][3] (device, f64 if dirs_f32 == 0 else f32). */
int lfp_render_grid(const lfp_probeset* ps, const lfp_grid_params* grid,
                    const double* eye, const void* dirs, int32_t dirs_f32,
                    int64_t n, const lfp_outputs* out, void* stream);

/* trace_grid_ray (kernels.py:653-822) over n explicit rays with per-ray
 * origins (device arrays [n][3], f64 if f32 == 0 else f32 up-cast
 * exactly). Config 5 and the parity harness. */
int lfp_trace_rays(const lfp_probeset* ps, const lfp_grid_params* grid,
                   const void* ray_origins, const void* ray_dirs, int32_t f32,
                   int64_t n, const lfp_outputs* out, void* stream);

/* Ray binning for incoherent batches (config 5): keys[i] = (lattice cube
 * where ray i enters the grid, 4x4x4 sub-cell of the entry point, 8x8
 * octahedral cell of the direction), 0xffffffff for rays missing the
 * lattice (cubes < 2^20). Sorting rays by key (any stable or unstable device
 * sort) and tracing them in that order with lfp_trace_rays_ordered lets a
 * warp march coherent cubes/segments; results do not depend on the order. */
int lfp_bin_rays(const lfp_grid_params* grid, const void* ray_origins,
                 const void* ray_dirs, int32_t f32, int64_t n, uint32_t* keys,
                 void* stream);

/* lfp_trace_rays where slot s traces ray order[s] (a permutation of
 * 0..n-1, device int32); outputs are written at the ray's input index. */
int lfp_trace_rays_ordered(const lfp_probeset* ps, const lfp_grid_params* grid,
                           const void* ray_origins, const void* ray_dirs,
                           int32_t f32, int64_t n, const int32_t* order,
                           const lfp_outputs* out, void* stream);

/* Scatter compact-tile outputs of `n_ranks` shards back into frame order.
 * Shard k traced tiles k, k + n_ranks, ...; its j-th tile sits at tile slot
 * k * shard_stride + j of the input (shard_stride = 0: shards packed
 * back to back, shard k holding floor(T/n) + (k < T % n) tiles). Any of the
 * array pairs may be NULL. */
int lfp_untile(int32_t n_cams, int32_t width, int32_t height, int32_t n_ranks,
               int64_t shard_stride, const uint8_t* status_in,
               const float* rgb_in, uint8_t* status_out, float* rgb_out,
               void* stream);

/* Diagnostics: ref[i] = a[i] / b[i] (nvcc IEEE division); fast[i] = the
 * tracer's branch-free division of the same operands (LFP_FAST_DIV: the
 * fast-path quotient when nvcc's fast-path test passes, else a / b) and
 * took[i] = 1 when it passed (device arrays). The GPU tests assert fast ==
 * ref bit for bit. */
int lfp_selftest_division(const double* a, const double* b, int64_t n,
                          double* ref, double* fast, uint8_t* took,
                          void* stream);

/* The same for the high-res DDA set-up's division (dda_init_hi): a / b
 * formed from the correctly rounded reciprocal of b, obtained by the exact
 * power-of-two scaling (1 / (b / 4)) / 4 the tracer applies to the low-res
 * DDA increments. */
int lfp_selftest_division_recip(const double* a, const double* b, int64_t n,
                                double* ref, double* fast, uint8_t* took,
                                void* stream);

/* ---- debug instrumentation (bounds-check builds only) ----
 * The library built with -DLFP_CHECK_BOUNDS=1 (liblfprobe_b200_check.so)
 * checks every probe-map / direction-table / payload / origin / ray-order
 * index against its array extent and, when `wcount` (device u32[n_out],
 * zeroed by the caller) is set, counts the writes of every per-ray output
 * record -- the evidence that each ray writes exactly its own row
 * (kernels.py:831-843), standing in for compute-sanitizer, which the GPU
 * pool does not allow. lfp_debug_bounds resets the violation counter and
 * installs `wcount` (NULL: no write counting) for later launches on
 * `device`; lfp_debug_report synchronises the device and returns the number
 * of failed checks and the site id of the first. Release builds return
 * LFP_ERR_INVALID from both. */
int lfp_debug_bounds(int device, uint32_t* wcount, int64_t n_out);
int lfp_debug_report(int device, uint64_t* violations, int32_t* first_site);

/* ---- input production: GPU ray-cast bake ---- */

/* Analytic primitive: kind 0 = axis-aligned box (a = lo, b = hi), kind 1 =
 * sphere (a = centre, b[0] = radius). */
typedef struct {
    int32_t kind;
    double a[3];
    double b[3];
    float albedo[3];
} lfp_prim;

typedef struct {
    double position[3];
    double power;     /* falloff min(1, power / (1 + d^2)) */
    double ambient;
} lfp_light;

/* Bake P probes (origins_host f64[P][3]) of R x R texels by ray-casting the
 * texel-centre directions against the primitives; writes the reference
 * ProbeSet layout into caller-owned DEVICE arrays dist_hi f32[P][R][R],
 * dir_hi / irr_hi f32[P][R][R][3], dist_lo f32[P][r][r] (block MIN,
 * bake.py:94-102). quant_f16 rounds radiance / direction through half.
 * Synchronous on `stream`. Replaces the point-cloud bake of bake.py:140-207
 * for the analytic benchmark scenes. */
int lfp_bake_probes(int device, const lfp_prim* prims_host, int32_t n_prims,
                    const lfp_light* light, const double* origins_host,
                    int64_t P, int32_t R, int32_t r, int32_t quant_f16,
                    int32_t shadows, float* dist_hi, float* dir_hi,
                    float* irr_hi, float* dist_lo, void* stream);

/* ---- the reference's point-cloud bake (bake.py:140-207, grid.py:96-109) ---- */

/* Bake P probes (origins_host f64[P][3]) from one point cloud: positions
 * f64[n][3] and colors f32[n][3] (PointCloud, pointcloud.py:19-45), host
 * pointers or, with LFP_SRC_DEVICE, device pointers. Per texel the nearest
 * point wins (exact-distance ties: smallest (x, y, z, r, g, b),
 * bake.py:116-137); the maps are the reference's in-memory quantised
 * values -- RGB565 radiance, float16 distance, 8-bit sub-texel direction
 * (bake.py:62-91) -- bit-identical to bake_probe, written into caller-owned
 * DEVICE arrays in the ProbeSet layout (dist_hi f32[P][R][R], dir_hi /
 * irr_hi f32[P][R][R][3], dist_lo f32[P][r][r] block MIN). skipped_host
 * (optional, int64[P]) receives the per-probe count of points within 1e-6 of
 * the origin (bake.py:167-174). n < 2^32 - 1. Synchronous on `stream`.
 * Replaces bake_probe / simulate_probe / grid.bake_grid's per-probe loop. */
int lfp_bake_points(int device, const double* positions, const float* colors,
                    int64_t n_points, const double* origins_host, int64_t P,
                    int32_t R, int32_t r, uint32_t flags, float* dist_hi,
                    float* dir_hi, float* irr_hi, float* dist_lo,
                    int64_t* skipped_host, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LFPROBE_B200_H */
