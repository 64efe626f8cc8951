/*
 * gpile_b200.h — C-ABI boundary of the B200-native GaussianPile slice renderer.
 *
 * This is the process/device boundary that replaces the CPU hot path of the
 * reference library (header-only C++20, /root/reference/proj/include/gpile).
 * Every entry point below names the reference interface it stands in for.
 * Nothing here uses C++ or torch types: plain structs, pointers and sizes.
 *
 * Conventions
 *   - Every function returns a gpk_status. No exception ever crosses the ABI.
 *     Status codes map 1:1 to the reference's exception taxonomy
 *     (errors.hpp:9-27 plus std::invalid_argument); the failing primitive
 *     index (when the reference names one, backward.hpp:182-184,
 *     voxelize.hpp:237) is available from gpk_last_error_index().
 *   - Gaussian parameters cross the boundary in the checkpoint record layout:
 *     11 x f32 per primitive, (mu x y z, log-scale x y z, quat w x y z,
 *     raw alpha) (checkpoint.hpp:14-16, docs/FORMATS.md:5-17). On the device
 *     they live as 11 SoA f32 planes.
 *   - Gradients use the same 11-slot order (grad_chain.hpp:12-22 flattened).
 *   - Images are row-major f32, pixels[j*W + i] (image.hpp:17-27); volumes are
 *     z-major f32, data[(k*Y + j)*X + i] (core.hpp:119-121).
 *   - One session per GPU. Calls on a session are issued in order on the
 *     session's CUDA stream. Functions that take or return HOST buffers
 *     synchronize the stream and surface device-side errors, like the
 *     reference's synchronous exceptions; functions whose host pointers are
 *     NULL stay asynchronous (device-resident data) so they can be captured
 *     in a CUDA graph; gpk_session_synchronize() surfaces deferred errors.
 */
#ifndef GPILE_B200_H
#define GPILE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPK_ABI_VERSION 7
#define GPK_RECORD_FLOATS 11

typedef enum {
    GPK_OK = 0,
    GPK_ERR_INVALID_ARGUMENT = 1,      /* std::invalid_argument */
    GPK_ERR_DEGENERATE_COVARIANCE = 2, /* gpile::DegenerateCovariance, errors.hpp:9 */
    GPK_ERR_NUMERIC_FAILURE = 3,       /* gpile::NumericFailure, errors.hpp:14 */
    GPK_ERR_CUDA = 4,                  /* CUDA runtime / launch failure */
    GPK_ERR_NCCL = 5,                  /* NCCL failure */
    GPK_ERR_OUT_OF_MEMORY = 6,         /* device allocation failed */
    GPK_ERR_STATE = 7,                 /* call order violated (e.g. backward before prepare) */
    GPK_ERR_CORRUPT_CONTAINER = 8,     /* gpile::CorruptContainer, errors.hpp:19 */
    GPK_ERR_LOAD = 9                   /* gpile::LoadError, errors.hpp:24 */
} gpk_status;

/* Bounds (core.hpp:50-65): world-space bbox, positions clamped into it by Adam. */
typedef struct {
    double min[3];
    double max[3];
} gpk_bounds;

/* SlicePose (core.hpp:78-105). rotation is R_c, row-major. */
typedef struct {
    double rotation[9];
    double translation[3];
    int32_t width;
    int32_t height;
    double pixel_spacing[2];
    double principal_point[2];
} gpk_slice_pose;

/* PsfSpec (core.hpp:109-117). Only sigma_z enters the renderer. */
typedef struct {
    double sigma_x, sigma_y, sigma_z;
} gpk_psf;

/* RasterConfig (render.hpp:26-31). tile_size must be 16 on this backend. */
typedef struct {
    double tau;
    int32_t tile_size;
    double footprint_sigmas;
    double scale_modifier;
} gpk_raster_config;

/* LearningRates (optimize.hpp:178-180) and AdamState hyper-parameters
 * (optimize.hpp:157). */
typedef struct {
    double position, opacity, scale, rotation;
} gpk_learning_rates;

typedef struct {
    double beta1, beta2, eps;
} gpk_adam_hparams;

/* VoxelizerConfig (voxelize.hpp:16-38). */
typedef struct {
    int32_t dims[3];
    double spacing[3];
    double origin[3];
    int32_t tile_dims[3];
    double support_sigmas;
    double scale_modifier;
} gpk_voxelizer_config;

/* ScreenGradStats (backward.hpp:19-26), host arrays of length n, overwritten. */
typedef struct {
    double* mu2d_grad_norm;   /* n */
    uint8_t* observed;        /* n */
    double* world_pos_grad;   /* 3n, xyz interleaved */
} gpk_screen_stats;

typedef struct gpk_session gpk_session;

/* Device buffers a zero-copy caller may address (gpk_device_buffer). */
typedef enum {
    GPK_BUF_PARAMS = 0,   /* 11 f32 planes x capacity: plane p at p*capacity */
    GPK_BUF_GRADS = 1,    /* 11 f32 planes, dense dL/dparam (backward output) */
    GPK_BUF_IMAGE = 2,    /* W*H f32: rendered slice (rasterize output) */
    GPK_BUF_DL_DI = 3,    /* W*H f32: dL/dI consumed by backward */
    GPK_BUF_TARGET = 4,   /* W*H f32: target slice for the photometric loss */
    GPK_BUF_VOLUME = 5,   /* X*Y*Z f32: voxelize output */
    GPK_BUF_DL_DV = 6,    /* X*Y*Z f32: dL/dV consumed by voxelize_backward */
    GPK_BUF_LOSS = 7,     /* 1 f64: last photometric loss */
    GPK_BUF_UNION_ROWS = 8  /* 11 f32 planes x capacity: a data-parallel step's union gradient rows
                               (rows [0, union capacity) of each plane; gpk_train_step_dp) */
} gpk_buffer;

/* ---- library ------------------------------------------------------------ */
int gpk_abi_version(void);
const char* gpk_last_error_message(void);   /* thread-local, valid until next call */
int64_t gpk_last_error_index(void);          /* primitive index or -1 */
int gpk_device_count(int* count);

/* ---- session lifecycle ---------------------------------------------------- */
/* cuda_stream may be NULL (the session creates its own non-blocking stream) or
 * a caller-owned cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream). */
int gpk_session_create(int device, void* cuda_stream, gpk_session** out);
int gpk_session_destroy(gpk_session* s);
int gpk_session_set_stream(gpk_session* s, void* cuda_stream);
int gpk_session_get_stream(gpk_session* s, void** cuda_stream);
/* Wait for all queued work, then report any device-side error flag. */
int gpk_session_synchronize(gpk_session* s);
/* Reserve (tile, Gaussian) pair capacity up front (avoids growth on first use). */
int gpk_session_reserve_pairs(gpk_session* s, uint64_t pairs);
int gpk_device_buffer(gpk_session* s, int which, void** ptr, uint64_t* bytes);
/* Raw, stream-ordered copies between a device buffer (gpk_buffer) and caller
 * memory (pinned memory makes them asynchronous). bytes must not exceed the
 * buffer size reported by gpk_device_buffer. */
int gpk_upload(gpk_session* s, int which, const void* host, uint64_t bytes);
int gpk_download(gpk_session* s, int which, void* host, uint64_t bytes);

/* ---- live stage timing (CUDA events on the session stream) ------------------ */
typedef enum {
    GPK_STAGE_PREPARE = 0,   /* K_prep: cull, fp64 focus Gaussians, survivor records, gradient clear */
    GPK_STAGE_SORT = 1,      /* radix passes */
    GPK_STAGE_RASTER = 2,    /* forward accumulation */
    GPK_STAGE_BACKWARD = 3,  /* backward pixel accumulation */
    GPK_STAGE_CHAIN = 4,     /* backward chain to world parameters */
    GPK_STAGE_LOSS = 5,
    GPK_STAGE_ADAM = 6,
    GPK_STAGE_VOXEL = 7,
    GPK_STAGE_BIN = 8,       /* K_bin: survivor slots, (tile, candidate) pair emission */
    GPK_STAGE_VOXEL_EVAL = 9,   /* voxelize: the per-tile evaluation (GPK_STAGE_VOXEL: prims + tile lists) */
    GPK_STAGE_ADAM_REST = 10,   /* training step: the non-survivors' Adam beside the render (GPK_STAGE_ADAM: the survivors') */
    GPK_NUM_STAGES = 11
} gpk_stage;
/* Enable/disable event pairs around every stage launch. */
int gpk_stage_timing(gpk_session* s, int enable);
/* Accumulated device milliseconds and launch counts per stage since the last
 * reset (synchronizes). ms and counts have GPK_NUM_STAGES entries. */
int gpk_stage_times(gpk_session* s, double* ms, uint64_t* counts, int reset);

/* ---- parameters (GaussianSet, core.hpp:67-74) ------------------------------ */
/* Upload n primitives (host records, 11 f32 each) and the bbox. Resets Adam. */
int gpk_set_gaussians(gpk_session* s, uint64_t n, const float* records, const gpk_bounds* bbox);
/* Same from f64 records (GaussianPrimitive layout flattened); rounded to f32. */
int gpk_set_gaussians_f64(gpk_session* s, uint64_t n, const double* records,
                          const gpk_bounds* bbox);
int gpk_get_gaussians(gpk_session* s, float* records);
int gpk_gaussian_count(gpk_session* s, uint64_t* n);
/* Dense gradient buffer (GaussianGradients, grad_chain.hpp:12-22) to/from host
 * records (n x 11 f32): the input of adam_step when gradients come from the host. */
int gpk_set_gradients(gpk_session* s, const float* grads);
int gpk_get_gradients(gpk_session* s, float* grads);

/* ---- slice renderer: prepare_gaussians + TileGrid (render.hpp:83-160) ------ */
/* Preprocess every primitive for this slice (focus Gaussian, cull, bounds),
 * then bin survivors to 16x16 tiles with a stable radix sort. Device-resident;
 * asynchronous. Validates pose/psf/cfg on the host (core.hpp:112-116). */
int gpk_prepare(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                const gpk_raster_config* cfg);
/* Survivor and pair counts of the last prepare (synchronizes). */
int gpk_prepared_count(gpk_session* s, uint64_t* survivors, uint64_t* pairs);
/* Counters of the last prepare (synchronizes): K_filter candidates (not
 * certainly culled by the fp32 bound), survivors, (tile, survivor) pairs and
 * survivors whose decision took the reference-order fp64 path. Any pointer
 * may be NULL. */
int gpk_prepare_stats(gpk_session* s, uint64_t* candidates, uint64_t* survivors, uint64_t* pairs,
                      uint64_t* fp64_decided);
/* Survivors in ascending set order (render.hpp:133-137): set index, inclusive
 * pixel bounds (lo_x, hi_x, lo_y, hi_y) and 6 doubles (alpha_tilde, mu_2d.x,
 * mu_2d.y, conic.a, conic.b, conic.d). Any pointer may be NULL. */
int gpk_get_prepared(gpk_session* s, uint32_t* index, int32_t* bounds, double* fields);
/* Every PreparedGaussian field (render.hpp:68-79) of the survivors, in set
 * order, GPK_PREPARED_FIELDS doubles each, in the reference's fp64 operation
 * order: alpha, opacity_r, alpha_tilde, mu_c[3], mu_e[3], sigma_c[9],
 * sigma_c_inv[9], sigma_e[9] (row-major), mu_2d[2], cov2d[4] (a b c d),
 * conic[4], det2. Synchronizes. */
#define GPK_PREPARED_FIELDS 47
int gpk_get_prepared_fields(gpk_session* s, double* fields);
/* Per-tile lists (render.hpp:142-160): offsets[tiles+1], entries[pairs] holding
 * set indices in list order. */
int gpk_get_tile_lists(gpk_session* s, uint32_t* offsets, uint32_t* entries);

/* ---- forward: rasterize_prepared (render.hpp:166-192) ----------------------- */
/* Renders the prepared slice into GPK_BUF_IMAGE; copies to image_out if non-NULL. */
int gpk_rasterize(gpk_session* s, float* image_out);

/* ---- backward: backward_prepared (backward.hpp:97-187) ---------------------- */
/* dl_di: host W*H f32, or NULL to consume GPK_BUF_DL_DI. Writes the dense
 * gradient (exact zeros for culled primitives) into GPK_BUF_GRADS; copies it
 * to grads_out (host, n*11 f32 record order) if non-NULL; fills stats if
 * non-NULL. Non-finite gradients -> GPK_ERR_NUMERIC_FAILURE naming the first
 * primitive (backward.hpp:175-185). */
int gpk_backward(gpk_session* s, const float* dl_di, float* grads_out, gpk_screen_stats* stats);

/* ---- loss: photometric_loss (loss.hpp:13-37) -------------------------------- */
/* target: host W*H f32 or NULL for GPK_BUF_TARGET. Renders must have run.
 * Writes dL/dI into GPK_BUF_DL_DI (and dl_di_out if non-NULL); the loss into
 * GPK_BUF_LOSS (and *loss_out if non-NULL, which synchronizes). */
int gpk_photometric_loss(gpk_session* s, const float* target, double lambda,
                         double dssim_scale, double* loss_out, float* dl_di_out);
/* Stand-alone photometric_loss(rendered, target, lambda, dl_di, dssim_scale)
 * on host images (loss.hpp:13): synchronous; overwrites the session's image,
 * target and dL/dI buffers. */
int gpk_photometric_loss_images(gpk_session* s, int32_t width, int32_t height,
                                const float* rendered, const float* target, double lambda,
                                double dssim_scale, double* loss_out, float* dl_di_out);

/* ---- optimizer: adam_step (optimize.hpp:195-221) ---------------------------- */
/* One bias-corrected Adam step on all n primitives using GPK_BUF_GRADS.
 * hp may be NULL (beta1 0.9, beta2 0.999, eps 1e-8). The step counter lives on
 * the device (AdamState::step). */
int gpk_adam_step(gpk_session* s, const gpk_learning_rates* lrs, const gpk_adam_hparams* hp);
/* Adam step whose learning rates follow lr_at(lr0, step, total) (optimize.hpp:71)
 * evaluated on the device from the device step counter (graph-capturable). */
int gpk_adam_step_scheduled(gpk_session* s, const gpk_learning_rates* lr0, int32_t total,
                            const gpk_adam_hparams* hp);
int gpk_adam_reset(gpk_session* s);
/* Adam moments in record order (n*11 each) and the step counter. */
int gpk_get_adam_state(gpk_session* s, float* m, float* v, int64_t* step);
int gpk_set_adam_state(gpk_session* s, const float* m, const float* v, int64_t step);

/* ---- fused paths for the throughput loop ------------------------------------ */
/* U1: prepare + rasterize + backward(GPK_BUF_DL_DI), all device-resident. */
int gpk_fwd_bwd_slice(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                      const gpk_raster_config* cfg);
/* U2: prepare + rasterize + loss(GPK_BUF_TARGET) + backward + scheduled Adam. */
/* Every later loss evaluation of this session (or slice context) also writes
 * the f64 loss into *host, page-locked host memory (cudaHostAlloc'd or
 * registered), from the loss kernel itself: the value is in host memory when
 * the kernel ends, with no separate device-to-host copy. NULL: off. Graphs
 * captured before a change must be recaptured. */
int gpk_set_loss_sink(gpk_session* s, double* host);
/* Target slots (0 or 1; 0 by default): GPK_BUF_TARGET uploads and downloads,
 * and every later loss evaluation (direct or captured into a graph), use the
 * selected slot's buffer. A caller that alternates slots step by step (and
 * captures its graphs with the matching slot) lets the next slice's target
 * upload run while the previous step still reads the other buffer, instead
 * of after it: the copy no longer waits for the previous step's last target
 * reader. Selecting slot 1 the first time allocates it (image-sized). */
int gpk_set_target_slot(gpk_session* s, int32_t slot);
/* Lazy mode (off by default; measured slower on B200): single-GPU
 * U2 steps run "lazily": Adam updates the slice's
 * survivors and one 1/16 window of the set per step; every other Gaussian's
 * zero-gradient step (optimize.hpp:195-221 with g = 0) is deferred and
 * replayed, in order and with the same fp32 operations, where it is next
 * needed — by the next cull for the Gaussians it cannot reject, by the window,
 * and by every API call that reads or writes parameters or moments — so each
 * result is bit-identical to the eager step. on = 0 (the default): every step
 * updates all n (the deferred steps are replayed first). */
int gpk_set_lazy_adam(gpk_session* s, int on);
int gpk_train_step(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                   const gpk_raster_config* cfg, double lambda, double dssim_scale,
                   const gpk_learning_rates* lr0, int32_t total_iterations);

/* Pipelined U2: as gpk_train_step, with Adam fused with the cull of next_pose
 * (same PSF and raster config): the parameters cross HBM once per step and the
 * next step on next_pose starts at K_decide. Results are bitwise those of
 * gpk_train_step; any other call that changes parameters or gradients in
 * between simply makes the next step cull again. */
int gpk_train_step_next(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                        const gpk_raster_config* cfg, double lambda, double dssim_scale,
                        const gpk_learning_rates* lr0, int32_t total_iterations,
                        const gpk_slice_pose* next_pose);

/* ---- batched slices (SURVEY.md §7.3.7, §8e "B slices per rank per step") ------
 * Context k in [0, 8) of a session: k = 0 is the session itself; k >= 1 is a
 * session handle with its own stream and per-slice buffers (image, dL/dI,
 * target, survivor records, tile lists) whose Gaussian parameters, dense
 * gradient planes and Adam moments are the session's. Upload slice k's target
 * or dL/dI to context k (gpk_upload); per-slice calls (gpk_prepare,
 * gpk_rasterize, gpk_get_prepared, ...) work on a context; calls that change
 * the set or the optimizer state do not (GPK_ERR_STATE). Contexts are owned
 * and destroyed by their session. */
int gpk_slice_context(gpk_session* s, int32_t k, gpk_session** ctx);
/* U1 x B: slices poses[0..B) (B <= 8) rendered concurrently, slice k on
 * context k, each backward of its context's GPK_BUF_DL_DI; GPK_BUF_GRADS
 * holds the SUM of the B slices' gradients, added in slice order. */
int gpk_fwd_bwd_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses, const gpk_psf* psf,
                      const gpk_raster_config* cfg);
/* U2 x B: B slices (targets from the contexts' GPK_BUF_TARGET), their losses
 * (each context's GPK_BUF_LOSS), ONE scheduled Adam step on the sum of the B
 * gradients (slice order). B = 1 is gpk_train_step. */
int gpk_train_step_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses, const gpk_psf* psf,
                         const gpk_raster_config* cfg, double lambda, double dssim_scale,
                         const gpk_learning_rates* lr0, int32_t total_iterations);

/* ---- CUDA graphs of the fused paths ------------------------------------------- */
/* Capture gpk_fwd_bwd_slice / gpk_train_step for a fixed pose into an
 * executable CUDA graph (launch overhead of the ~7 kernels collapses to one
 * submission). Buffers must already be sized (run the path once first and
 * reserve pair capacity). Returns a graph id for gpk_graph_launch. */
int gpk_graph_capture_fwd_bwd(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                              const gpk_raster_config* cfg, int32_t* graph_id);
int gpk_graph_capture_train(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                            const gpk_raster_config* cfg, double lambda, double dssim_scale,
                            const gpk_learning_rates* lr0, int32_t total_iterations,
                            int32_t* graph_id);
/* Graph of gpk_train_step_next (launching it culls its own slice first when the
 * previous launch did not leave it culled). */
int gpk_graph_capture_train_next(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                                 const gpk_raster_config* cfg, double lambda, double dssim_scale,
                                 const gpk_learning_rates* lr0, int32_t total_iterations,
                                 const gpk_slice_pose* next_pose, int32_t* graph_id);
/* Graphs of the batched steps (fixed poses). */
int gpk_graph_capture_fwd_bwd_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses,
                                    const gpk_psf* psf, const gpk_raster_config* cfg, int32_t* graph_id);
int gpk_graph_capture_train_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses,
                                  const gpk_psf* psf, const gpk_raster_config* cfg, double lambda,
                                  double dssim_scale, const gpk_learning_rates* lr0, int32_t total_iterations,
                                  int32_t* graph_id);
int gpk_graph_launch(gpk_session* s, int32_t graph_id);
int gpk_graph_destroy_all(gpk_session* s);

/* ---- voxelizer: voxelize / voxelize_backward (voxelize.hpp:113-240) ---------- */
int gpk_voxelize(gpk_session* s, const gpk_voxelizer_config* cfg, float* volume_out);
/* Per-8^3-tile lists of the last voxelize (VoxelTiles, voxelize.hpp:86-105). */
int gpk_voxel_tile_count(gpk_session* s, uint64_t* tiles, uint64_t* instances);
int gpk_get_voxel_tile_lists(gpk_session* s, uint32_t* offsets, uint32_t* entries);
int gpk_voxelize_backward(gpk_session* s, const gpk_voxelizer_config* cfg, const float* dl_dv,
                          float* grads_out);

/* ---- host utilities of the fit driver (synthetic inputs, schedule) ----------- */
/* init_random (optimize.hpp:94-108) on the reference's seeded mt19937_64 stream
 * (rng.hpp:14-70): n x 11 f64 records, bit-identical to the reference. */
int gpk_init_random(uint64_t n, const gpk_bounds* bbox, double scale_base, uint64_t seed,
                    double* records);
/* slice_pose_for_index (core.hpp:202-211) for a z-major volume geometry. */
int gpk_slice_pose_for_index(const int32_t dims[3], const double spacing[3],
                             const double origin[3], int k, gpk_slice_pose* out);
/* lr_at (optimize.hpp:71-73). */
double gpk_lr_at(double lr0, int iteration, int total);

/* init_grid (optimize.hpp:111-133): ceil(cbrt(n))^3 lattice of cell centres,
 * truncated to n, shapes from the same seeded stream; n x 11 f64 records. */
int gpk_init_grid(uint64_t n, const gpk_bounds* bbox, double scale_base, uint64_t seed,
                  double* records);
/* default_init_count (optimize.hpp:64-66). */
int gpk_default_init_count(uint64_t voxel_count, uint64_t* out);

/* The reference's seeded generator (Rng, rng.hpp:14-70: mt19937_64 with
 * self-contained distributions), for slice sampling and split draws. */
typedef struct gpk_rng gpk_rng;
int gpk_rng_create(uint64_t seed, gpk_rng** out);
int gpk_rng_destroy(gpk_rng* rng);
int gpk_rng_uniform(gpk_rng* rng, double* out);              /* [0, 1) */
int gpk_rng_below(gpk_rng* rng, uint64_t n, uint64_t* out);  /* Rng::below */
int gpk_rng_normal(gpk_rng* rng, double* out);               /* Box-Muller, spare cached */

/* ---- checkpoints: save_checkpoint / load_checkpoint (checkpoint.hpp:38-92) ---- */
/* The reference's uncompressed format byte for byte ("GPILE", u32 version 1,
 * u64 count, 6 f64 bbox, count x 11 f32 records). Load replaces the session's
 * set (Adam reset, as gpk_set_gaussians). Errors: GPK_ERR_LOAD (cannot open /
 * write), GPK_ERR_CORRUPT_CONTAINER (magic, version, truncation). */
int gpk_save_checkpoint(gpk_session* s, const char* path);
int gpk_load_checkpoint(gpk_session* s, const char* path);
uint64_t gpk_checkpoint_bytes(uint64_t count);   /* checkpoint_bytes (checkpoint.hpp:95-97) */
/* The set's world bbox (GaussianSet::bbox, core.hpp:67-74). */
int gpk_get_bounds(gpk_session* s, gpk_bounds* out);

/* ---- codec front half (morton.hpp, quant.hpp, container.hpp:136-230) --------- */
typedef struct {
    int32_t pos_bits;      /* 14, per axis */
    int32_t opacity_bits;  /* 12 */
    int32_t scale_bits;    /* 12, on log-scale */
    int32_t quat_bits;     /* 12, per component */
    int32_t morton_bits;   /* 14, per axis */
} gpk_quant_spec;          /* QuantSpec (quant.hpp:13-26), widths in [4, 21] */

/* morton_sort(set, bits) (morton.hpp:33-48) of the resident set: the stable
 * Z-order permutation (n entries; perm[k] = set index of the k-th). */
int gpk_morton_sort(gpk_session* s, int32_t bits, uint64_t* perm_out);
/* quantize (quant.hpp:67-132) of the resident set — in Morton order
 * (morton_order != 0, as encode() does, container.hpp:203-206) or set order:
 * positions 3n, opacities n, log_scales 3n, quats 4n (u32), and the observed
 * log-scale range. Non-finite / zero-quaternion inputs -> INVALID_ARGUMENT
 * naming the (quantized-order) index, as the reference throws. */
int gpk_quantize(gpk_session* s, const gpk_quant_spec* spec, int32_t morton_order, uint32_t* positions,
                 uint32_t* opacities, uint32_t* log_scales, uint32_t* quats, double scale_min[3],
                 double scale_max[3]);
/* encode()'s front half (container.hpp:203-230): Morton sort, quantize, and
 * the delta + zig-zag packing of each stream (detail::pack_deltas,
 * container.hpp:136-156) — the byte streams LZMA then compresses.
 * Sizes: gpk_stream_bytes(n, 3, pos_bits), (n, 1, opacity_bits),
 * (n, 3, scale_bits), (n, 4, quat_bits). */
int gpk_encode_streams(gpk_session* s, const gpk_quant_spec* spec, uint8_t* positions, uint8_t* opacities,
                       uint8_t* log_scales, uint8_t* quats, double scale_min[3], double scale_max[3]);
uint64_t gpk_stream_bytes(uint64_t count, int32_t components, int32_t bits);
/* The decode side before dequantization (detail::unpack_deltas,
 * container.hpp:158-181, then dequantize, quant.hpp:134-176): the four packed
 * streams of n primitives -> n x 11 f32 records (records_out, host, if
 * non-NULL); load != 0 makes the decoded set the session's (gpk_set_gaussians).
 * An out-of-range delta -> GPK_ERR_CORRUPT_CONTAINER naming the stream. */
int gpk_decode_streams(gpk_session* s, const gpk_quant_spec* spec, uint64_t n, const gpk_bounds* bbox,
                       const double scale_min[3], const double scale_max[3], const uint8_t* positions,
                       const uint8_t* opacities, const uint8_t* log_scales, const uint8_t* quats,
                       float* records_out, int32_t load);

/* ---- adaptive density control (optimize.hpp:228-344) ------------------------ */
typedef struct {
    double tau;                  /* prune exposed alpha < tau (FitConfig::tau) */
    double grad_threshold;       /* mean screen gradient threshold (5e-5) */
    double split_scale_fraction; /* split when max scale > fraction * extent (0.01) */
    double split_scale_divisor;  /* children's scales divided by this (1.6) */
    double scale_modifier;       /* "mod" (1.0) */
} gpk_densify_config;

typedef struct {
    uint64_t pruned, cloned, split;   /* DensifyReport (optimize.hpp:251-253) */
} gpk_densify_report;

/* DensifyAccum (optimize.hpp:228-249) kept on the device: while enabled, every
 * backward (gpk_backward, gpk_train_step, graphs captured afterwards) adds
 * its ScreenGradStats (|dL/dmu_2d|, observed, world dL/dmu) of the survivors.
 * Enabling zeroes it; it is zeroed whenever the set changes size. */
int gpk_densify_accum_enable(gpk_session* s, int on);
int gpk_densify_accum_reset(gpk_session* s);
/* host arrays of n: grad_norm_sum f64, observations i32, world_grad_sum 3n f64 */
int gpk_get_densify_accum(gpk_session* s, double* grad_norm_sum, int32_t* observations,
                          double* world_grad_sum);
int gpk_set_densify_accum(gpk_session* s, const double* grad_norm_sum, const int32_t* observations,
                          const double* world_grad_sum);
/* densify_and_prune(set, adam, accum, cfg, rng) (optimize.hpp:255-344) on the
 * resident set: prune / keep / clone / split decided on the device, the new
 * set ordered as the reference orders it (kept in index order, then the born
 * in their parents' order), Adam moments carried for the kept and zero for
 * the born, the step counter kept; 6 normals per split drawn from rng in
 * parent order. Resets the accumulator. */
int gpk_densify_and_prune(gpk_session* s, const gpk_densify_config* cfg, gpk_rng* rng,
                          gpk_densify_report* report);
/* The same with the normals drawn by the caller's generator (e.g. the
 * reference's own gpile::Rng): normal(user) is called 6 times per split
 * parent, in parent order, before any parameter changes. */
typedef double (*gpk_normal_fn)(void* user);
int gpk_densify_and_prune_draw(gpk_session* s, const gpk_densify_config* cfg, gpk_normal_fn normal,
                               void* user, gpk_densify_report* report);

/* ---- fit driver (optimize.hpp:360-424) --------------------------------------- */
typedef struct {
    int32_t iterations;            /* 30000 */
    double lr_position, lr_opacity, lr_scale, lr_rotation;  /* 6e-4, 0.02, 2e-3, 1e-3 */
    uint64_t init_count;           /* 0 -> default_init_count(voxels) */
    double tau;                    /* 0.02 */
    int32_t densify_start, densify_end;   /* 500, 25000 */
    double grad_threshold;         /* 5e-5 */
    double lambda;                 /* 0.2 */
    int32_t densify_interval;      /* 100 */
    uint64_t rng_seed;             /* 0 */
    int32_t init_mode;             /* 0 random, 1 grid */
    double scale_modifier;         /* 1.0 */
    double split_scale_fraction;   /* 0.01 */
    double split_scale_divisor;    /* 1.6 */
    double dssim_scale;            /* 0.5 */
    int32_t progress_interval;     /* 200 */
    int32_t tile_size;             /* 16 */
    double footprint_sigmas;       /* 3.0 */
} gpk_fit_config;

typedef struct {
    int32_t iteration;
    double loss;          /* photometric loss on this iteration's slice */
    uint64_t count;       /* primitives */
    double psnr2d;        /* monitor slice (Z/2), clamped render */
    double monitor_loss;  /* photometric loss on the monitor slice */
} gpk_fit_progress;       /* FitProgress (optimize.hpp:350-356) */

#define GPK_PSNR_INF 999.0   /* kPsnrInf (metrics.hpp:14) */

typedef void (*gpk_fit_progress_fn)(const gpk_fit_progress* p, void* user);

/* fit(volume, psf, cfg, progress) (optimize.hpp:360-424): volume is host
 * X*Y*Z f32 z-major (data[(k*Y + j)*X + i]). The fitted set stays resident in
 * the session (gpk_get_gaussians). Errors carry "fit: iteration N: ". */
int gpk_fit(gpk_session* s, const float* volume, const int32_t dims[3], const double spacing[3],
            const double origin[3], const gpk_psf* psf, const gpk_fit_config* cfg,
            gpk_fit_progress_fn progress, void* user);

/* ---- multi-GPU: slice-sharded data parallelism ------------------------------ */
/* 128-byte ncclUniqueId produced on rank 0 and broadcast by the caller. */
int gpk_nccl_get_unique_id(void* id_out128);
int gpk_comm_init(gpk_session* s, int nranks, int rank, const void* id128);
int gpk_comm_destroy(gpk_session* s);
/* Sum GPK_BUF_GRADS across ranks (one ncclAllReduce, in place, session stream). */
int gpk_allreduce_grads(gpk_session* s);

/* Data-parallel training step with the union-compacted exchange (SURVEY.md
 * §7.3.8, §8e). Every rank passes the step's `world` slice poses in rank order
 * (the shared schedule) and renders poses[rank]. In its cull pass each rank
 * also evaluates the other poses' certain-cull, so every rank derives the same
 * union of candidates (a superset of every rank's survivors) without a
 * collective; its chain writes the survivors' gradients into rows of that
 * union (GPK_BUF_UNION_ROWS); ONE grouped ncclAllReduce sums the rows; every
 * rank runs the scheduled Adam on all Gaussians from the summed rows, so the
 * replicas stay bitwise equal. phases: a bitmask of GPK_DP_RENDER,
 * GPK_DP_EXCHANGE, GPK_DP_UPDATE (GPK_DP_ALL = the step; the exchange needs
 * gpk_comm_init; the split lets a caller exchange the rows itself). world <= 8.
 * A direct call sizes the row capacity (the all-reduce count) from the union
 * it computed; graphs bake it (gpk_dp_reserve_union before capture). */
#define GPK_DP_RENDER 1
#define GPK_DP_EXCHANGE 2
#define GPK_DP_UPDATE 4
#define GPK_DP_ALL 7
int gpk_train_step_dp(gpk_session* s, int32_t world, int32_t rank, const gpk_slice_pose* poses, const gpk_psf* psf,
                      const gpk_raster_config* cfg, double lambda, double dssim_scale, const gpk_learning_rates* lr0,
                      int32_t total_iterations, int32_t phases);
int gpk_graph_capture_train_dp(gpk_session* s, int32_t world, int32_t rank, const gpk_slice_pose* poses,
                               const gpk_psf* psf, const gpk_raster_config* cfg, double lambda, double dssim_scale,
                               const gpk_learning_rates* lr0, int32_t total_iterations, int32_t* graph_id);
/* Union rows of the last step and the exchange capacity (synchronizes);
 * GPK_ERR_STATE when the union outgrew a captured capacity (that step's
 * update was skipped). */
int gpk_dp_union_rows(gpk_session* s, uint64_t* rows, uint64_t* capacity);
/* Set the exchanged row capacity (every rank the same value). */
int gpk_dp_reserve_union(gpk_session* s, uint64_t rows);

#ifdef __cplusplus
}
#endif

#endif /* GPILE_B200_H */
