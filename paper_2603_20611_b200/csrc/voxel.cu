// voxel.cu — 3-D voxelizer (voxelize.hpp:113-240). Work in progress: the
// entry points report GPK_ERR_STATE until the kernels land.
#include "../../include/gpile_b200.h"

extern "C" {
int gpk_voxelize(gpk_session*, const gpk_voxelizer_config*, float*) { return GPK_ERR_STATE; }
int gpk_voxel_tile_count(gpk_session*, uint64_t*, uint64_t*) { return GPK_ERR_STATE; }
int gpk_get_voxel_tile_lists(gpk_session*, uint32_t*, uint32_t*) { return GPK_ERR_STATE; }
int gpk_voxelize_backward(gpk_session*, const gpk_voxelizer_config*, const float*, float*) {
    return GPK_ERR_STATE;
}
}
