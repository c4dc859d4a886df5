// Compiled tiled-kernel variants.  Each line instantiates k_tiled for one
// (R, S, KT, NBT, TH, TW) tile and several (io dtype, weight format, mode)
// combinations; the launch tuner (scb_launch_candidates + Python
// tune_launch) picks among the ones matching a layer.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"
#include "sparseconv_b200.h"

namespace scb {

using TiledLauncher = cudaError_t (*)(const TiledParams&, unsigned grid, unsigned threads,
                                      size_t smem, cudaStream_t st);

struct VariantEntry {
    scb_variant_info info;
    TiledLauncher launch;
};

extern const VariantEntry g_variants[];
extern const int g_num_variants;

cudaError_t launch_generic(const GenericParams& p, int dtype, bool fast, cudaStream_t st);
cudaError_t launch_maxpool2(int dtype, const void* x, void* y, int64_t planes, int h, int w,
                            cudaStream_t st);

}  // namespace scb

// (R, S, KT, NBT, TH, TW)
#define SCB_VARIANT_LIST                        \
    SCB_TILE_ALLMODES(3, 3, 8, 1, 4, 4)         \
    SCB_TILE_ALLMODES(3, 3, 4, 1, 4, 4)         \
    SCB_TILE_ALLMODES(3, 3, 8, 1, 2, 4)         \
    SCB_TILE_ALLMODES(3, 3, 4, 2, 2, 4)         \
    SCB_TILE_ALLMODES(3, 3, 8, 2, 2, 4)         \
    SCB_TILE_ALLMODES(3, 3, 4, 2, 4, 4)         \
    SCB_TILE_ALLMODES(3, 3, 8, 2, 2, 2)         \
    SCB_TILE_ALLMODES(3, 3, 8, 1, 2, 2)         \
    SCB_TILE_QUANT(3, 3, 8, 1, 4, 4)            \
    SCB_TILE_QUANT(3, 3, 4, 2, 2, 4)            \
    SCB_TILE_QUANT(3, 3, 8, 2, 2, 2)            \
    SCB_TILE_ALLMODES(1, 1, 8, 1, 4, 4)         \
    SCB_TILE_ALLMODES(1, 1, 8, 2, 2, 4)         \
    SCB_TILE_ALLMODES(5, 5, 4, 1, 4, 4)         \
    SCB_TILE_ALLMODES(5, 5, 4, 2, 2, 4)         \
    SCB_TILE_ALLMODES(1, 2, 8, 2, 1, 8)         \
    SCB_TILE_ALLMODES(1, 3, 8, 2, 1, 8)
