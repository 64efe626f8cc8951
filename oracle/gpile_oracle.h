/* gpile_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, fp64 restatement of the reference's hot path (GaussianPile,
 * /root/reference/proj/include/gpile). It is the checker the CUDA path is
 * compared against in tests/ and the "port" CPU baseline; it is never linked
 * into the product. Each function cites the reference code it restates.
 * Pinned against the reference itself (oracle/_ref) and the golden fixtures in
 * tests/golden/ by tests/test_oracle.py.
 *
 * Records are n x 11 doubles: mu xyz, log-scale xyz, quat wxyz, raw alpha.
 */
#ifndef GPILE_ORACLE_H
#define GPILE_ORACLE_H

#include <stdint.h>

#include "../include/gpile_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* gor_last_error(void);
int64_t gor_last_error_index(void);

/* prepare_gaussians (render.hpp:83-138). fields: 19 doubles per survivor, same
 * layout as oracle/ref_shim.cpp gref_prepare. */
int gor_prepare(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                const gpk_raster_config* cfg, uint64_t* count, uint32_t* index, int32_t* bounds,
                double* fields);
/* detail::TileGrid (render.hpp:142-160); entries are set indices. */
int gor_tile_lists(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                   const gpk_raster_config* cfg, uint32_t* offsets, uint32_t* entries,
                   uint64_t capacity, uint64_t* total, uint64_t* tiles);
/* rasterize_slice (render.hpp:194). */
int gor_rasterize(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                  const gpk_raster_config* cfg, double* image);
/* rasterize_naive (render.hpp:203-219). */
int gor_rasterize_naive(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                        const gpk_raster_config* cfg, double* image);
/* backward_slice (backward.hpp:189). */
int gor_backward(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                 const gpk_raster_config* cfg, const double* dl_di, double* grads,
                 double* stat_norm, uint8_t* stat_observed, double* stat_world);
/* photometric_loss (loss.hpp:13). */
int gor_loss(int w, int h, const double* rendered, const double* target, double lambda,
             double dssim_scale, double* dl_di, double* loss);
/* adam_step (optimize.hpp:195); rec, m, v, step updated in place. */
int gor_adam_step(uint64_t n, double* rec, const gpk_bounds* bbox, const double* grads, double* m,
                  double* v, int64_t* step, const gpk_learning_rates* lrs,
                  const gpk_adam_hparams* hp);
/* voxelize (voxelize.hpp:113). out: X*Y*Z, z-major. */
int gor_voxelize(uint64_t n, const double* rec, const gpk_voxelizer_config* cfg, double* out);
/* detail::VoxelTiles (voxelize.hpp:86-105). */
int gor_voxel_tiles(uint64_t n, const double* rec, const gpk_voxelizer_config* cfg,
                    uint32_t* offsets, uint32_t* entries, uint64_t capacity, uint64_t* total,
                    uint64_t* tiles);
/* voxelize_backward (voxelize.hpp:152). */
int gor_voxelize_backward(uint64_t n, const double* rec, const gpk_voxelizer_config* cfg,
                          const double* dl_dv, double* grads);

#ifdef __cplusplus
}
#endif

#endif
