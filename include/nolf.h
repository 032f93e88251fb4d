/*
 * nolf.h -- C ABI of the B200-native i-NOLF render path (libnolf_b200.so).
 *
 * Plain C types only: host pointers for asset creation, device pointers for
 * per-frame buffers, an opaque cudaStream_t passed as void*.  Every entry
 * point returns 0 on success or a negative NOLF_E* status; nolf_last_error()
 * returns a thread-local message for the last failure on the calling thread.
 *
 * Each entry point replaces one reference (radfarm, pure numpy) interface;
 * the Python host mirror paper_2303_04086_b200/ binds these via ctypes and
 * keeps the reference signatures:
 *
 *   nolf_asset_create   <- LightFieldAsset construction / assetio.read_asset
 *                          (lightfield.py:217-248, assetio.py:174-255): uploads
 *                          density atlas, PSH (Phi narrowed to u32), features,
 *                          MLPs, diffuse atlas or hash grid, march params.
 *   nolf_render_rays    <- lightfield.render_rays(asset, origins, dirs, counters)
 *                          (lightfield.py:400-456)
 *   nolf_render_rect    <- renderer.render_range(asset, RayRange, counters)
 *                          (renderer.py:63-93), camera_dirs fused on device
 *   nolf_render_scene   <- renderer.render_frame + farm.compose
 *                          (renderer.py:96-107, farm.py:129-172) fused: march,
 *                          shade and depth-composite every asset of a scene
 *                          over a list of screen tiles of one or more cameras
 *   nolf_compose        <- farm.compose(frames, alpha_vis) (farm.py:129-172)
 *   nolf_march_rays     <- lightfield.march_rays (lightfield.py:129-186)
 *   nolf_eval_diffuse   <- hashgrid_encode + mlp_forward(diffuse_mlp)
 *                          (encoding.py:467-478, lightfield.py:319-327)
 *   nolf_counters layout = RenderCounters {fs_evals, fd_evals, hit_pixels,
 *                          march_samples} (lightfield.py:113-126)
 *
 * Error mapping in the host mirror (errors.py of the reference):
 *   NOLF_EINVAL -> DomainError, NOLF_ESTATE -> StateError,
 *   NOLF_EDATA -> DataError, NOLF_ECAPACITY -> CapacityError,
 *   NOLF_ECUDA / NOLF_ENOMEM -> RuntimeError.
 */
#ifndef NOLF_H_
#define NOLF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NOLF_ABI_VERSION 4

#define NOLF_OK 0
#define NOLF_EINVAL -1
#define NOLF_ESTATE -2
#define NOLF_EDATA -3
#define NOLF_ECUDA -4
#define NOLF_ENOMEM -5
#define NOLF_ECAPACITY -6   /* work was dropped on the device (see nolf_check_errors) */

#define NOLF_HEAD_IDENTITY 0
#define NOLF_HEAD_SIGMOID 1
#define NOLF_HEAD_EXP 2

/* MLP execution mode for the specular network (lightfield.py:632-637). */
#define NOLF_MLP_FP32 0   /* CUDA-core fp32, tolerance 1e-3 vs reference */
#define NOLF_MLP_BF16 1   /* tcgen05 bf16 x bf16 -> fp32 TMEM, tolerance 2/255 */

typedef struct NolfAtlasDesc {        /* CubeAtlas, atlas.py:25-51 */
    int32_t b, r, channels;
    int64_t n_cubes;
    const int32_t *index;             /* (b,b,b), -1 = empty */
    const float *cubes;               /* (n_cubes, r+1, r+1, r+1, channels) */
} NolfAtlasDesc;

typedef struct NolfMlpDesc {          /* Mlp, neural.py:29-86 */
    int32_t n_layers;                 /* number of weight matrices */
    int32_t widths[5];                /* widths[0] = input width */
    const float *w[4];                /* (out, in) row-major */
    const float *b[4];
    int32_t n_heads;
    int32_t head_act[8];              /* NOLF_HEAD_* */
    int32_t head_w[8];
} NolfMlpDesc;

typedef struct NolfAssetDesc {        /* LightFieldAsset, lightfield.py:217-248 */
    NolfAtlasDesc density;
    int32_t has_diffuse_atlas;
    NolfAtlasDesc diffuse;
    /* PshTable, encoding.py:109-140 */
    int32_t psh_resolution;
    int64_t psh_table_size;           /* m */
    int64_t psh_offset_size;          /* m_phi */
    const int64_t *psh_offsets;       /* (m_phi,) */
    uint64_t primes_h0[3], primes_h1[3];
    const float *psh_features;        /* (m, F) */
    int32_t psh_features_dim;         /* F */
    /* HashGridEncoder, encoding.py:405-459 (live diffuse path) */
    int32_t hg_levels, hg_features;
    int64_t hg_table_size;
    int32_t hg_resolution[16];
    int32_t hg_dense[16];
    int64_t hg_rows[16];
    const float *hg_feat[16];
    NolfMlpDesc specular, diffuse_mlp;
    /* MarchParams, lightfield.py:85-90 */
    double step, t_stop, alpha_floor;
    double proxy_min[3], proxy_max[3]; /* Aabb proxy */
    /* ModelWiring, lightfield.py:59-67 */
    int32_t use_hit_point, use_opacity, refine_opacity, use_tint, use_diffuse_color;
    /* Optional triangle-mesh proxy (object space, inside the proxy box):
     * the march starts at its first hit.  No reference counterpart
     * (BASELINE config 2).  mesh_n_triangles == 0: slab proxy only. */
    const double *mesh_vertices;       /* (n_vertices, 3) */
    int64_t mesh_n_vertices;
    const int32_t *mesh_triangles;     /* (n_triangles, 3) vertex indices */
    int64_t mesh_n_triangles;
} NolfAssetDesc;

typedef struct NolfAsset *nolf_asset_t;

/* One placed asset: the scene transform replaces object_to_world
 * (renderer.py:110-113, farm.py:118-122).  w2o = inv(object_to_world) and
 * scale = uniform_scale_of(w2o) are computed on the host exactly as the
 * reference does (lightfield.py:408-409). */
typedef struct NolfInstance {
    nolf_asset_t asset;
    double w2o[16];
    double scale;
} NolfInstance;

typedef struct NolfCamera {            /* Camera, core.py:90-126 */
    double pose[16];                   /* camera-to-world, row-major */
    double fx, fy, cx, cy;
    int32_t width, height;
} NolfCamera;

typedef struct NolfTile {              /* RayRange rect of one camera */
    int32_t cam, x0, y0, x1, y1;
} NolfTile;

/* Scene output.  layout 0 writes pixels in TILE-PACKED order: tile t (in the
 * order given) owns slots [t*tile_stride, t*tile_stride + w_t*h_t); inside a
 * tile whose sides are multiples of 8x4 the slots run over 8x4 pixel blocks
 * (block-row-major, row-major inside a block), other tiles are row-major
 * (render.slot_xy / unpack_index); layout 1 writes the row-major frame of
 * each camera.  Any pointer may be NULL to skip it. */
typedef struct NolfSceneOut {
    float *rgba;                       /* (.., 4) f32, farm.compose Frame.rgba */
    float *depth;                      /* f32, inf = miss */
    uint8_t *rgba8;                    /* protocol.encode_frame RAW rgba8 */
    uint16_t *depth16;                 /* protocol.encode_frame RAW depth u16 */
    int64_t tile_stride;               /* pixels per tile slot (>= max w*h) */
    double depth_far;                  /* encode_frame far plane */
    int32_t layout;                    /* 0: tile-packed (above); 1: row-major frame per
                                          camera, cameras concatenated in order */
    int32_t peer;                      /* 1: outputs live in another GPU's memory (CUDA IPC
                                          mapping); the compose epilogue stores them over
                                          NVLink and ends with a system-scope fence */
    int32_t prefilled;                 /* 1: rgba8 / depth16 already hold the miss encoding
                                          (0 / 65535) for every pixel of these tiles, so
                                          miss pixels are not written (chunks no screen
                                          box reaches, runs of 4 / 8 misses)
                                          (u8/u16 outputs only; rgba/depth must be NULL) */
    /* Sparse frame (end-to-end delivery): with prefilled = 1, 128-slot-aligned
     * tiles in the 8x4-block layout (sides multiples of 8 x 4) and tile_stride
     * a multiple of 128, the compose epilogue also packs the LIVE chunks (128
     * consecutive slots some screen box reaches; every other pixel is a miss)
     * run by run: each 8-pixel run that encodes to anything but the miss
     * encoding goes to `pack` (48 B: 8 rgba8 then 8 depth16), and pack_ids
     * holds per live chunk i {chunk id (slot / 128), mask of its packed runs,
     * index of its first packed run}; pack_count[0] = live chunks,
     * pack_count[1] = packed runs (may be host-mapped memory).  Only these
     * bytes need to cross PCIe: nolf_host_scatter rebuilds the frame.
     * rgba8 / depth16 may then be NULL.  All three NULL: no pack. */
    uint8_t *pack;
    uint32_t *pack_ids;
    uint32_t *pack_count;
    /* With prefilled = 1 and frame layout: a u16 per 128-slot chunk of the
     * tile list (DEVICE, owned by the caller, one array per frame buffer,
     * zero for a buffer that holds only the miss encoding): bit r = the
     * chunk's 8-pixel run r holds non-miss bytes from an earlier frame.  The
     * library rewrites exactly the runs that change (hits now, or dirty and
     * a miss now; dead chunks' dirty runs are reset) and keeps the bits: a
     * frame buffer never needs a full clear between frames.  NULL: the
     * caller re-clears. */
    uint16_t *chunk_state;
} NolfSceneOut;

int nolf_abi_version(void);
const char *nolf_last_error(void);

int nolf_asset_create(const NolfAssetDesc *desc, int device, nolf_asset_t *out);
/* assetio.read_asset (assetio.py:174-255) natively: the ``.nolf`` container
 * (optionally gzip-compressed) is parsed, every section's CRC32 checked, the
 * JSON meta decoded and the asset uploaded; object_to_world (may be NULL)
 * receives the stored transform (row-major 4x4).  Corrupt input ->
 * NOLF_EDATA (DataError). */
int nolf_asset_load(const char *path, int device, nolf_asset_t *out, double object_to_world[16]);
int nolf_asset_load_mem(const void *data, size_t n, int device, nolf_asset_t *out, double object_to_world[16]);
int nolf_asset_destroy(nolf_asset_t asset);
int nolf_asset_set_mlp_mode(nolf_asset_t asset, int mode);
int64_t nolf_asset_device_bytes(nolf_asset_t asset);

/* Workspace bytes sufficient for any call with up to n_rays rays x n_inst
 * placed assets (upper bound). */
size_t nolf_workspace_bytes(int32_t n_inst, int64_t n_rays);
/* Tight workspace bytes for nolf_render_scene with these instances and
 * cameras over n_rays pixel slots (hit queues sized by each instance's
 * screen box, compose layers by the maximum box overlap); 0 on bad input. */
size_t nolf_scene_workspace_bytes(const NolfInstance *inst, int32_t n_inst, const NolfCamera *cams,
                                  int32_t n_cams, int64_t n_rays);

/* counters: device uint64[4] accumulated (not reset). */
int nolf_render_rays(const NolfInstance *inst, const double *origins, int32_t origin_stride,
                     const double *dirs, int64_t n, float *rgba, float *depth,
                     unsigned long long *counters, void *workspace, size_t ws_bytes,
                     void *stream);

int nolf_render_rect(const NolfInstance *inst, const NolfCamera *cam, int32_t x0, int32_t y0,
                     int32_t x1, int32_t y1, float *rgba, float *depth,
                     unsigned long long *counters, void *workspace, size_t ws_bytes,
                     void *stream);

/* tiles: DEVICE pointer to n_tiles NolfTile (uploaded once per tiling). */
int nolf_render_scene(const NolfInstance *inst, int32_t n_inst, const NolfCamera *cams,
                      int32_t n_cams, const NolfTile *tiles, int32_t n_tiles,
                      const NolfSceneOut *out, double alpha_vis, unsigned long long *counters,
                      void *workspace, size_t ws_bytes, void *stream);

/* march_rays (lightfield.py:129-186) on object-space rays (no transform, no
 * renormalisation), slab against the asset proxy: per-ray MarchResult
 * fields.  Used e.g. for hit-shell collection (lightfield.py:475-512). */
int nolf_march_rays(nolf_asset_t asset, const double *origins, int32_t origin_stride, const double *dirs,
                    int64_t n, uint8_t *hit, double *t_hit, double *alpha_c, int64_t *samples, double *p_h,
                    void *workspace, size_t ws_bytes, void *stream);

/* Live diffuse network (hash grid + diffuse MLP, encoding.py:467-478,
 * neural.py:89-108) at n object-space points -> (n, 4) post-activation
 * (c_d, t); what bake_diffuse_cubes caches (lightfield.py:547-576). */
int nolf_eval_diffuse(nolf_asset_t asset, const double *points, int64_t n, float *out, void *stream);

/* Launch-variant knobs of the calling thread (defaults are the measured
 * best; the timed variants are selected by launch size, so tests force each
 * one to run it against the oracle).  Results never depend on them. */
#define NOLF_OPT_MARCH_ORDER 1    /* 0 auto, 1 live chunks in spatial order, 2 heaviest first */
#define NOLF_OPT_COMPOSE_SLOTS 2  /* live-chunk compose slots per thread: 0 auto, 4 or 8 */
#define NOLF_OPT_HEAVY_WAVES 3    /* auto order: heaviest-first below this many CTA waves (3) */
#define NOLF_OPT_MARCH_SPLIT 4    /* CTAs per live 128-slot chunk in the marcher: 1 (128 threads) or 2 (64) */
#define NOLF_OPT_CHUNK_COST 5     /* heaviest-first order: 1 by the previous frame's measured per-chunk
                                     marcher durations (default), 0 by candidate-instance counts */
int nolf_set_option(int32_t key, int64_t value);

/* Device-side failures fail loudly.  The kernels count (never silently
 * blend) work they had to drop: hit records beyond an instance's queue, hits
 * beyond a pixel's compose layers, scene tiles outside their camera's frame
 * (or larger than tile_stride), BVH traversals deeper than the stack -- all
 * impossible for valid inputs.  The counters are read back asynchronously
 * after every render call; an increase makes the NEXT render call on the
 * thread return NOLF_ECAPACITY.  nolf_check_errors synchronises `stream`
 * and reports at once (NOLF_ECAPACITY, message in nolf_last_error). */
int nolf_check_errors(void *stream);

/* The variants the calling thread's last render call launched: info[0] = 1
 * when live 128-slot chunks were compacted and marched (k_cull_chunks +
 * k_march_chunks), info[1] = 1 heaviest-first / 0 spatial order, info[2] =
 * live-chunk compose slots per thread (4 / 8; 0 = full-frame k_compose),
 * info[3] = resident k_shade_tc CTAs per SM (bf16 tcgen05 shading; >= 1) /
 * 0 fp32 (k_shade). */
int nolf_last_launch(int32_t info[4]);

/* Parity read-back (debug): while slots != NULL, every render call on the
 * calling thread makes its shading kernel (k_shade / k_shade_tc) store the
 * 8 PSH corner slots it gathered for each shaded hit -- PshTable.corner_slots
 * (encoding.py:130-140), corner order CORNERS (encoding.py:34-37) -- to
 * slots[8*row + c] (u32, DEVICE), row = the hit's output row (render_rays /
 * render_rect) or layer*P + slot (render_scene's compose layers); rows >=
 * capacity_rows are not written.  NULL turns it off. */
int nolf_debug_psh_slots(uint32_t *slots, int64_t capacity_rows);

/* Per-kernel timing: while enabled, every render call of the calling thread
 * records CUDA events on its stream around k_march, k_shade, k_compose (up to
 * 4096 calls).  nolf_profile_read synchronises and returns, in ms[0..2], the
 * summed durations over all recorded calls; its return value is the call
 * count (negative on error). */
int nolf_profile(int enable);
int nolf_profile_read(float *ms);
/* Host->device bytes a render call copies (instance, camera, cull tables). */
size_t nolf_launch_param_bytes(int32_t n_inst, int32_t n_cams);

/* Frame assembly after gathering every rank's tile-packed encode_frame
 * output (rank r: n_per_rank slots of rgba8, then their depth16) into one
 * buffer: slot_tiles (DEVICE, world*n_per_rank, rank-major) gives each slot's
 * tile; writes the row-major rgba8 (H,W,4) and depth16 (H,W) frame of every
 * camera, camera c at offset c*W*H (all cameras W x H). */
int nolf_unpack_gathered(const uint8_t *gathered, int32_t world, int32_t n_per_rank, int64_t tile_stride,
                         const NolfTile *slot_tiles, int32_t width, int32_t height, uint8_t *rgba8,
                         uint16_t *depth16, void *stream);

/* The specular network alone (numerics tests / microbench): x (n, in) f32
 * device rows -> out (n, 4) f32 post-head, via the tcgen05 bf16 path
 * (NOLF_MLP_BF16) or the fp32 CUDA-core path (NOLF_MLP_FP32). */
int nolf_mlp_eval(nolf_asset_t asset, int mode, const float *x, int64_t n, float *out, void *stream);

/* Device buffers that can be shared across processes (CUDA IPC): the
 * multi-GPU frame composer maps rank 0's frame into every rank so compose
 * kernels store their pixels straight into it over NVLink / NVSwitch. */
int nolf_device_alloc(size_t bytes, void **ptr);
int nolf_device_free(void *ptr);
int nolf_ipc_get_handle(void *ptr, void *handle64);          /* 64-byte handle out */
int nolf_ipc_open_handle(const void *handle64, void **ptr);  /* peer mapping */
int nolf_ipc_close_handle(void *ptr);
/* Frame-completion signalling over NVLink without a collective: set stores
 * `value` into a (possibly peer-mapped) u32 flag after a system-scope fence
 * (everything the stream did before is visible first); wait spins on the
 * device until all n local flags are >= value (sleeping between polls),
 * bounded: after ~4 s it gives up and sets *timed_out (device u32, may be
 * NULL).  Both are stream-ordered, no host sync. */
int nolf_flag_set(uint32_t *flag, uint32_t value, void *stream);
int nolf_flag_wait(const uint32_t *flags, int32_t n, uint32_t value, uint32_t *timed_out, void *stream);
int nolf_memcpy_async(void *dst, const void *src, size_t bytes, void *stream);
/* n (<= 1024) u32 words by a one-warp kernel (plain stores, system fence):
 * e.g. a render's pack_count into host-mapped memory without a copy-engine
 * operation in the stream. */
int nolf_store_u32(uint32_t *dst, const uint32_t *src, int32_t n, void *stream);
int nolf_memset_async(void *dst, int32_t byte_value, size_t bytes, void *stream);
int nolf_memcpy2d_async(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width_bytes,
                        size_t height, void *stream);
/* Page-lock host memory (e.g. a shared-memory frame buffer mapped by every
 * rank) and map it into the device address space: compose kernels then
 * store frames straight into host memory over each GPU's own PCIe link. */
int nolf_host_register(void *host_ptr, size_t bytes, void **dev_ptr);
int nolf_host_unregister(void *host_ptr);

/* protocol.encode_frame (protocol.py:256-279): quantisation of an f32 frame
 * (DEVICE rgba (n,4) / depth (n)) to rgba8 = clip(round(255 x)) and u16 depth
 * = round(min(d, far) / far * 65534), 65535 for misses; and ENC_DEFLATE's
 * zlib stream (HOST, zlib compress2 at `level`, the reference uses 6:
 * byte-identical to Python's zlib.compress(data, 6) when both use the same
 * zlib, see nolf_zlib_version).  dst NULL: *dst_len = the size bound. */
int nolf_encode_frame(const float *rgba, const float *depth, int64_t n, double depth_far, uint8_t *rgba8,
                      uint16_t *depth16, void *stream);
int nolf_deflate(const void *src, size_t n, int32_t level, void *dst, size_t *dst_len);
const char *nolf_zlib_version(void);

/* Stage-2 training step (lightfield.train_light_field, lightfield.py:654-749,
 * after the frozen march).  Trainable tensors live in one flat DEVICE f32
 * buffer `params` in the reference layouts (W (out, in) row-major), at the
 * float offsets `offsets` (HOST, NOLF_TRAIN_OFFSETS entries): psh features
 * (m,F); specular W0,b0,W1,b1,W2,b2; diffuse W0,b0,W1,b1; hash-grid level
 * features (rows_l, F) for l < 16.  `grads` (DEVICE f64, same layout) is
 * ACCUMULATED (zero it first).  For n hit rays (p_h, alpha_c, object-space
 * dirs; targets rgb (n,3) / alpha (n) f32; `batch` = rays in the batch b):
 * shade_batch with the live diffuse network, the loss |c - rgb|^2 +
 * (alpha - alpha_t)^2 (loss, pred = (c, alpha)), d = 2 err / b and
 * shade_backward (MLP weight / bias gradients, psh_backward and
 * hashgrid_backward scatters).  *nonfinite |= 1 on a non-finite loss. */
#define NOLF_TRAIN_OFFSETS 27
int nolf_train_shade(nolf_asset_t asset, const float *params, const int64_t *offsets, double *grads, int64_t n,
                     const double *p_h, const double *alpha_c, const double *dirs, const float *rgb,
                     const float *alpha_t, double batch, float *pred, double *loss, uint32_t *nonfinite,
                     void *stream);
/* adam_step (neural.py:162-177) on n DEVICE params with f64 gradients (used
 * as f32), in the reference's f32 arithmetic; step = the group's step count
 * after increment.  *nonfinite |= 2 on a non-finite gradient (TrainingError). */
int nolf_adam(float *param, const double *grad, float *m, float *v, int64_t n, double lr, double beta1,
              double beta2, double eps, int64_t step, uint32_t *nonfinite, void *stream);

/* frames: rgba (K, P, 4) f32, depth (K, P) f32, all device pointers. */
/* Host side of the sparse frame (NolfSceneOut.pack): writes the packed runs
 * of the n live chunks (HOST copies of pack / pack_ids) into a row-major
 * encode_frame RAW frame in host memory (camera c at c*width*height; tiles =
 * the HOST tile list of the render, tile_stride as rendered).  `dirty`
 * (HOST, one u16 per chunk of the tile list, zero for a buffer holding only
 * the miss encoding) records which runs of this frame buffer hold non-miss
 * bytes: runs that were dirty and are misses now are reset, the rest of the
 * frame is never touched.  Runs on n_threads host threads (0: the pool
 * default). */
int nolf_host_scatter(const uint8_t *runs, const uint32_t *heads, uint32_t n, const NolfTile *tiles, int32_t n_tiles,
                      int64_t tile_stride, int32_t width, int32_t height, uint8_t *rgba8, uint16_t *depth16,
                      uint16_t *dirty, int32_t n_threads);

int nolf_compose(int32_t K, int64_t P, const float *rgba, const float *depth, double alpha_vis,
                 float *out_rgba, float *out_depth, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NOLF_H_ */
